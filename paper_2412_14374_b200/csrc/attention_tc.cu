// Tensor-core causal flash attention for bf16, head_dim 64 or 128.
//
// Semantics: oracle/gpt.py attention / attention_bwd (exact softmax, causal).
// Forward: FlashAttention-2 structure -- one CTA per (128 query rows, head),
// 8 warps x 16 rows, K/V tiles of 64 keys double-buffered in shared memory
// via cp.async, S = Q K^T and O += P V on warp-level bf16 MMAs (m16n8k16,
// fp32 accumulate), online softmax in registers (exp2 with pre-scaled
// logits), log-sum-exp saved for the backward.
// Backward: two kernels, no atomics (bitwise deterministic):
//   dK/dV  one CTA per 64 keys, loops over the causal query blocks,
//   dQ     one CTA per 64 queries, loops over the causal key blocks,
// both recomputing P from the saved log-sum-exp; delta = rowsum(dO * O) first.
//
// Layout as attention_simt.cu: qkv [B*S, ld_qkv] (q | k | v, head h at h*hd),
// o / dO [B*S, ld_o], lse / delta [B, H, S] fp32 (natural log).
#include "common.cuh"

namespace pp200 {

int attention_delta(int dtype, int B, int H, int S, int hd, const void* o, const void* dO,
                    int64_t ld_o, float* delta, cudaStream_t st);

namespace {

using bf16 = __nv_bfloat16;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                        uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                          uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// rows [0, ROWS) of a head slice -> smem [ROWS][LDS]; rows >= valid are zeros.
template <int ROWS, int HD, int NT>
__device__ __forceinline__ void load_tile(bf16* s, const bf16* g, int64_t ldg, int valid) {
  constexpr int LDS = HD + 8, CPR = HD / 8;
  for (int c = threadIdx.x; c < ROWS * CPR; c += NT) {
    const int r = c / CPR, k = c % CPR;
    const bool ok = r < valid;
    cp_async16(s + r * LDS + k * 8, ok ? g + static_cast<int64_t>(r) * ldg + k * 8 : g, ok ? 16 : 0);
  }
}
template <int ROWS, int NT>
__device__ __forceinline__ void load_vec(float* s, const float* g, int valid) {
  for (int r = threadIdx.x; r < ROWS; r += NT) s[r] = r < valid ? g[r] : 0.f;
}

// A fragments (16 rows x HD) of rows [row0, row0+16) of an smem tile.
template <int HD>
__device__ __forceinline__ void load_afrags(uint32_t (*f)[4], const bf16* s, int row0, int lane) {
  constexpr int LDS = HD + 8;
  const int mi = lane >> 3, r = lane & 7;
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk)
    ldsm_x4(f[kk][0], f[kk][1], f[kk][2], f[kk][3],
            smem_u32(s + (row0 + (mi & 1) * 8 + r) * LDS + kk * 16 + (mi >> 1) * 8));
}

// acc[NB/8][4] += A(16 x HD) * rows(NB x HD)^T   (B rows = n index, non-trans)
template <int HD, int NB, bool A_FROM_SMEM>
__device__ __forceinline__ void mma_abt(float (*acc)[4], const uint32_t (*af)[4], const bf16* sa,
                                        int arow0, const bf16* sb, int lane) {
  constexpr int LDS = HD + 8;
  const int mi = lane >> 3, r = lane & 7;
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    uint32_t a[4];
    if (A_FROM_SMEM) {
      ldsm_x4(a[0], a[1], a[2], a[3],
              smem_u32(sa + (arow0 + (mi & 1) * 8 + r) * LDS + kk * 16 + (mi >> 1) * 8));
    } else {
      a[0] = af[kk][0]; a[1] = af[kk][1]; a[2] = af[kk][2]; a[3] = af[kk][3];
    }
#pragma unroll
    for (int np = 0; np < NB / 16; ++np) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4(b0, b1, b2, b3,
              smem_u32(sb + ((2 * np + (mi >> 1)) * 8 + r) * LDS + kk * 16 + (mi & 1) * 8));
      mma16816(acc[2 * np], a, b0, b1);
      mma16816(acc[2 * np + 1], a, b2, b3);
    }
  }
}

// out[HD/8][4] += P(16 x KB, in C-fragment registers) * tile(KB x HD)  (B via .trans)
template <int HD, int KB>
__device__ __forceinline__ void mma_pv(float (*out)[4], const float (*p)[4], const bf16* sv,
                                       int lane) {
  constexpr int LDS = HD + 8;
  const int mi = lane >> 3, r = lane & 7;
#pragma unroll
  for (int k2 = 0; k2 < KB / 16; ++k2) {
    uint32_t a[4] = {pack2(p[2 * k2][0], p[2 * k2][1]), pack2(p[2 * k2][2], p[2 * k2][3]),
                     pack2(p[2 * k2 + 1][0], p[2 * k2 + 1][1]),
                     pack2(p[2 * k2 + 1][2], p[2 * k2 + 1][3])};
#pragma unroll
    for (int dp = 0; dp < HD / 16; ++dp) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(b0, b1, b2, b3,
                smem_u32(sv + (k2 * 16 + (mi & 1) * 8 + r) * LDS + dp * 16 + (mi >> 1) * 8));
      mma16816(out[2 * dp], a, b0, b1);
      mma16816(out[2 * dp + 1], a, b2, b3);
    }
  }
}

__device__ __forceinline__ float quad_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float quad_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// ----------------------------------------------------------------- forward

template <int HD>
struct FwdCfg {
  static constexpr int BM = 128, BN = 64, NT = 256, LDS = HD + 8;
  static constexpr int SMEM = (BM + 4 * BN) * LDS * 2;
};

template <int HD>
__global__ void __launch_bounds__(256) fa_fwd(const bf16* __restrict__ qkv, int64_t ldq,
                                              bf16* __restrict__ o, int64_t ldo,
                                              float* __restrict__ lse, int H, int S, float sl2) {
  using C = FwdCfg<HD>;
  constexpr int BM = C::BM, BN = C::BN, LDS = C::LDS;
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sQ = reinterpret_cast<bf16*>(smraw);
  bf16* sK = sQ + BM * LDS;
  bf16* sV = sK + 2 * BN * LDS;
  const int nqb = (S + BM - 1) / BM;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);  // heavy (late) blocks first
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int d = H * HD;
  const bf16* Qg = qkv + static_cast<int64_t>(b) * S * ldq + h * HD;
  const bf16* Kg = Qg + d;
  const bf16* Vg = Qg + 2 * d;
  const int q0 = qb * BM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  const int kend = min(S, q0 + BM);
  const int nkb = (kend + BN - 1) / BN;

  load_tile<BM, HD, C::NT>(sQ, Qg + static_cast<int64_t>(q0) * ldq, ldq, S - q0);
  cp_commit();
  load_tile<BN, HD, C::NT>(sK, Kg, ldq, S);
  load_tile<BN, HD, C::NT>(sV, Vg, ldq, S);
  cp_commit();
  cp_wait<1>();
  __syncthreads();
  uint32_t qf[HD / 16][4];
  load_afrags<HD>(qf, sQ, warp * 16, lane);

  const int rowA = q0 + warp * 16 + g, rowB = rowA + 8;
  float oacc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;

  for (int kb = 0; kb < nkb; ++kb) {
    if (kb + 1 < nkb) {
      const int n1 = (kb + 1) * BN;
      load_tile<BN, HD, C::NT>(sK + ((kb + 1) & 1) * BN * LDS, Kg + static_cast<int64_t>(n1) * ldq, ldq, S - n1);
      load_tile<BN, HD, C::NT>(sV + ((kb + 1) & 1) * BN * LDS, Vg + static_cast<int64_t>(n1) * ldq, ldq, S - n1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int n0 = kb * BN;
    const bf16* sKb = sK + (kb & 1) * BN * LDS;
    const bf16* sVb = sV + (kb & 1) * BN * LDS;
    if (n0 <= q0 + warp * 16 + 15 && q0 + warp * 16 < S) {
      float s[BN / 8][4];
#pragma unroll
      for (int i = 0; i < BN / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
      mma_abt<HD, BN, false>(s, qf, nullptr, 0, sKb, lane);
      float bmA = -INFINITY, bmB = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = e < 2 ? rowA : rowB;
          const int key = n0 + nt * 8 + tg * 2 + (e & 1);
          float v = s[nt][e] * sl2;
          if (key > row || key >= S) v = -INFINITY;
          s[nt][e] = v;
        }
        bmA = fmaxf(bmA, fmaxf(s[nt][0], s[nt][1]));
        bmB = fmaxf(bmB, fmaxf(s[nt][2], s[nt][3]));
      }
      const float nA = fmaxf(mA, quad_max(bmA)), nB = fmaxf(mB, quad_max(bmB));
      const float refA = nA == -INFINITY ? 0.f : nA, refB = nB == -INFINITY ? 0.f : nB;
      const float cA = exp2f(mA - refA), cB = exp2f(mB - refB);
      mA = nA;
      mB = nB;
      float sumA = 0.f, sumB = 0.f;
#pragma unroll
      for (int nt = 0; nt < BN / 8; ++nt) {
        s[nt][0] = exp2f(s[nt][0] - refA);
        s[nt][1] = exp2f(s[nt][1] - refA);
        s[nt][2] = exp2f(s[nt][2] - refB);
        s[nt][3] = exp2f(s[nt][3] - refB);
        sumA += s[nt][0] + s[nt][1];
        sumB += s[nt][2] + s[nt][3];
      }
      lA = lA * cA + sumA;
      lB = lB * cB + sumB;
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) {
        oacc[i][0] *= cA; oacc[i][1] *= cA;
        oacc[i][2] *= cB; oacc[i][3] *= cB;
      }
      mma_pv<HD, BN>(oacc, s, sVb, lane);
    }
    __syncthreads();
  }
  lA = quad_sum(lA);
  lB = quad_sum(lB);
  const float iA = lA > 0.f ? 1.f / lA : 0.f, iB = lB > 0.f ? 1.f / lB : 0.f;
  bf16* ob = o + static_cast<int64_t>(b) * S * ldo + h * HD;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int col = i * 8 + tg * 2;
    if (rowA < S)
      *reinterpret_cast<uint32_t*>(ob + static_cast<int64_t>(rowA) * ldo + col) = pack2(oacc[i][0] * iA, oacc[i][1] * iA);
    if (rowB < S)
      *reinterpret_cast<uint32_t*>(ob + static_cast<int64_t>(rowB) * ldo + col) = pack2(oacc[i][2] * iB, oacc[i][3] * iB);
  }
  if (tg == 0) {
    float* l = lse + (static_cast<int64_t>(b) * H + h) * S;
    if (rowA < S) l[rowA] = (mA + log2f(lA)) * LN2;
    if (rowB < S) l[rowB] = (mB + log2f(lB)) * LN2;
  }
}

// Forward with 32 query rows per warp (two m16 tiles): every K / V fragment
// loaded from shared memory feeds two MMAs, halving ldmatrix traffic per
// flop.  4 warps x 32 rows = 128 rows per CTA.  Used for head_dim 64.
template <int HD>
struct Fwd2Cfg {
  static constexpr int BM = 128, BN = 64, NT = 128, LDS = HD + 8;
  static constexpr int SMEM = (BM + 4 * BN) * LDS * 2;
};

template <int HD>
__global__ void __launch_bounds__(128) fa_fwd2(const bf16* __restrict__ qkv, int64_t ldq,
                                               bf16* __restrict__ o, int64_t ldo,
                                               float* __restrict__ lse, int H, int S, float sl2) {
  using C = Fwd2Cfg<HD>;
  constexpr int BM = C::BM, BN = C::BN, LDS = C::LDS, NT = C::NT;
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sQ = reinterpret_cast<bf16*>(smraw);
  bf16* sK = sQ + BM * LDS;
  bf16* sV = sK + 2 * BN * LDS;
  const int nqb = (S + BM - 1) / BM;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int d = H * HD;
  const bf16* Qg = qkv + static_cast<int64_t>(b) * S * ldq + h * HD;
  const bf16* Kg = Qg + d;
  const bf16* Vg = Qg + 2 * d;
  const int q0 = qb * BM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  const int mi = lane >> 3, r8 = lane & 7;
  const int kend = min(S, q0 + BM);
  const int nkb = (kend + BN - 1) / BN;
  const int wrow0 = q0 + warp * 32;

  load_tile<BM, HD, NT>(sQ, Qg + static_cast<int64_t>(q0) * ldq, ldq, S - q0);
  cp_commit();
  load_tile<BN, HD, NT>(sK, Kg, ldq, S);
  load_tile<BN, HD, NT>(sV, Vg, ldq, S);
  cp_commit();
  cp_wait<1>();
  __syncthreads();
  uint32_t qf[2][HD / 16][4];
  load_afrags<HD>(qf[0], sQ, warp * 32, lane);
  load_afrags<HD>(qf[1], sQ, warp * 32 + 16, lane);

  float oacc[2][HD / 8][4];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) oacc[t][i][0] = oacc[t][i][1] = oacc[t][i][2] = oacc[t][i][3] = 0.f;
  float m[2][2] = {{-INFINITY, -INFINITY}, {-INFINITY, -INFINITY}};
  float l[2][2] = {{0.f, 0.f}, {0.f, 0.f}};

  for (int kb = 0; kb < nkb; ++kb) {
    if (kb + 1 < nkb) {
      const int n1 = (kb + 1) * BN;
      load_tile<BN, HD, NT>(sK + ((kb + 1) & 1) * BN * LDS, Kg + static_cast<int64_t>(n1) * ldq, ldq, S - n1);
      load_tile<BN, HD, NT>(sV + ((kb + 1) & 1) * BN * LDS, Vg + static_cast<int64_t>(n1) * ldq, ldq, S - n1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int n0 = kb * BN;
    const bf16* sKb = sK + (kb & 1) * BN * LDS;
    const bf16* sVb = sV + (kb & 1) * BN * LDS;
    if (n0 <= wrow0 + 31 && wrow0 < S) {
      float sc[2][BN / 8][4];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int i = 0; i < BN / 8; ++i) sc[t][i][0] = sc[t][i][1] = sc[t][i][2] = sc[t][i][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
        for (int np = 0; np < BN / 16; ++np) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(b0, b1, b2, b3,
                  smem_u32(sKb + ((2 * np + (mi >> 1)) * 8 + r8) * LDS + kk * 16 + (mi & 1) * 8));
          mma16816(sc[0][2 * np], qf[0][kk], b0, b1);
          mma16816(sc[0][2 * np + 1], qf[0][kk], b2, b3);
          mma16816(sc[1][2 * np], qf[1][kk], b0, b1);
          mma16816(sc[1][2 * np + 1], qf[1][kk], b2, b3);
        }
      }
      const bool diag = n0 + BN > wrow0;  // some key > some row in this block
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int rowA = wrow0 + t * 16 + g, rowB = rowA + 8;
        float bmA = -INFINITY, bmB = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float v = sc[t][nt][e] * sl2;
            if (diag || n0 + BN > S) {
              const int row = e < 2 ? rowA : rowB;
              const int key = n0 + nt * 8 + tg * 2 + (e & 1);
              if (key > row || key >= S) v = -INFINITY;
            }
            sc[t][nt][e] = v;
          }
          bmA = fmaxf(bmA, fmaxf(sc[t][nt][0], sc[t][nt][1]));
          bmB = fmaxf(bmB, fmaxf(sc[t][nt][2], sc[t][nt][3]));
        }
        const float nA = fmaxf(m[t][0], quad_max(bmA)), nB = fmaxf(m[t][1], quad_max(bmB));
        const float refA = nA == -INFINITY ? 0.f : nA, refB = nB == -INFINITY ? 0.f : nB;
        const float cA = exp2f(m[t][0] - refA), cB = exp2f(m[t][1] - refB);
        m[t][0] = nA;
        m[t][1] = nB;
        float sumA = 0.f, sumB = 0.f;
#pragma unroll
        for (int nt = 0; nt < BN / 8; ++nt) {
          sc[t][nt][0] = exp2f(sc[t][nt][0] - refA);
          sc[t][nt][1] = exp2f(sc[t][nt][1] - refA);
          sc[t][nt][2] = exp2f(sc[t][nt][2] - refB);
          sc[t][nt][3] = exp2f(sc[t][nt][3] - refB);
          sumA += sc[t][nt][0] + sc[t][nt][1];
          sumB += sc[t][nt][2] + sc[t][nt][3];
        }
        l[t][0] = l[t][0] * cA + sumA;
        l[t][1] = l[t][1] * cB + sumB;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
          oacc[t][i][0] *= cA; oacc[t][i][1] *= cA;
          oacc[t][i][2] *= cB; oacc[t][i][3] *= cB;
        }
      }
      // O += P V for both row tiles, sharing every V fragment
#pragma unroll
      for (int k2 = 0; k2 < BN / 16; ++k2) {
        uint32_t a0[4] = {pack2(sc[0][2 * k2][0], sc[0][2 * k2][1]), pack2(sc[0][2 * k2][2], sc[0][2 * k2][3]),
                          pack2(sc[0][2 * k2 + 1][0], sc[0][2 * k2 + 1][1]),
                          pack2(sc[0][2 * k2 + 1][2], sc[0][2 * k2 + 1][3])};
        uint32_t a1[4] = {pack2(sc[1][2 * k2][0], sc[1][2 * k2][1]), pack2(sc[1][2 * k2][2], sc[1][2 * k2][3]),
                          pack2(sc[1][2 * k2 + 1][0], sc[1][2 * k2 + 1][1]),
                          pack2(sc[1][2 * k2 + 1][2], sc[1][2 * k2 + 1][3])};
#pragma unroll
        for (int dp = 0; dp < HD / 16; ++dp) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(b0, b1, b2, b3,
                    smem_u32(sVb + (k2 * 16 + (mi & 1) * 8 + r8) * LDS + dp * 16 + (mi >> 1) * 8));
          mma16816(oacc[0][2 * dp], a0, b0, b1);
          mma16816(oacc[0][2 * dp + 1], a0, b2, b3);
          mma16816(oacc[1][2 * dp], a1, b0, b1);
          mma16816(oacc[1][2 * dp + 1], a1, b2, b3);
        }
      }
    }
    __syncthreads();
  }
  bf16* ob = o + static_cast<int64_t>(b) * S * ldo + h * HD;
  float* lb = lse + (static_cast<int64_t>(b) * H + h) * S;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int rowA = wrow0 + t * 16 + g, rowB = rowA + 8;
    const float LA = quad_sum(l[t][0]), LB = quad_sum(l[t][1]);
    const float iA = LA > 0.f ? 1.f / LA : 0.f, iB = LB > 0.f ? 1.f / LB : 0.f;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      const int col = i * 8 + tg * 2;
      if (rowA < S)
        *reinterpret_cast<uint32_t*>(ob + static_cast<int64_t>(rowA) * ldo + col) = pack2(oacc[t][i][0] * iA, oacc[t][i][1] * iA);
      if (rowB < S)
        *reinterpret_cast<uint32_t*>(ob + static_cast<int64_t>(rowB) * ldo + col) = pack2(oacc[t][i][2] * iB, oacc[t][i][3] * iB);
    }
    if (tg == 0) {
      if (rowA < S) lb[rowA] = (m[t][0] + log2f(LA)) * LN2;
      if (rowB < S) lb[rowB] = (m[t][1] + log2f(LB)) * LN2;
    }
  }
}

// ---------------------------------------------------------------- backward

template <int HD>
struct BwdCfg {
  static constexpr int BK = 64;                  // keys per CTA (dK/dV) / per iteration (dQ)
  static constexpr int BQ = HD == 64 ? 64 : 32;  // queries per iteration (dK/dV)
  static constexpr int BQ2 = 64;                 // queries per CTA (dQ)
  static constexpr int NT = 128, LDS = HD + 8;
  static constexpr bool KEEP = HD == 64;         // keep K/V (Q/dO) A-fragments in registers
  static constexpr int SMEM_KV = (2 * BK + 4 * BQ) * LDS * 2 + 4 * BQ * 4;
  static constexpr int SMEM_Q = (2 * BQ2 + 4 * BK) * LDS * 2;
};

template <int HD>
__global__ void __launch_bounds__(128) fa_bwd_dkdv(const bf16* __restrict__ qkv, int64_t ldq,
                                                   const bf16* __restrict__ dO, int64_t ldo,
                                                   const float* __restrict__ lse,
                                                   const float* __restrict__ delta,
                                                   bf16* __restrict__ dqkv, int64_t ldd, int H,
                                                   int S, float sl2, float scale) {
  using C = BwdCfg<HD>;
  constexpr int BK = C::BK, BQ = C::BQ, LDS = C::LDS;
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sK = reinterpret_cast<bf16*>(smraw);
  bf16* sV = sK + BK * LDS;
  bf16* sQ = sV + BK * LDS;          // [2][BQ][LDS]
  bf16* sG = sQ + 2 * BQ * LDS;      // dO, [2][BQ][LDS]
  float* sL = reinterpret_cast<float*>(sG + 2 * BQ * LDS);  // lse*log2e [2][BQ]
  float* sD = sL + 2 * BQ;                                  // delta [2][BQ]
  const int nkb = (S + BK - 1) / BK;
  const int kb = nkb - 1 - static_cast<int>(blockIdx.x);  // short (late) blocks last
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int d = H * HD;
  const bf16* Qg = qkv + static_cast<int64_t>(b) * S * ldq + h * HD;
  const bf16* Kg = Qg + d;
  const bf16* Vg = Qg + 2 * d;
  const bf16* Gg = dO + static_cast<int64_t>(b) * S * ldo + h * HD;
  const float* Lg = lse + (static_cast<int64_t>(b) * H + h) * S;
  const float* Dg = delta + (static_cast<int64_t>(b) * H + h) * S;
  const int k0 = kb * BK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  const int qbeg = k0 / BQ, nqb = (S + BQ - 1) / BQ;

  load_tile<BK, HD, C::NT>(sK, Kg + static_cast<int64_t>(k0) * ldq, ldq, S - k0);
  load_tile<BK, HD, C::NT>(sV, Vg + static_cast<int64_t>(k0) * ldq, ldq, S - k0);
  cp_commit();
  auto load_q = [&](int qb, int buf) {
    const int m0 = qb * BQ;
    load_tile<BQ, HD, C::NT>(sQ + buf * BQ * LDS, Qg + static_cast<int64_t>(m0) * ldq, ldq, S - m0);
    load_tile<BQ, HD, C::NT>(sG + buf * BQ * LDS, Gg + static_cast<int64_t>(m0) * ldo, ldo, S - m0);
  };
  load_q(qbeg, 0);
  cp_commit();
  load_vec<BQ, C::NT>(sL, Lg + qbeg * BQ, S - qbeg * BQ);
  load_vec<BQ, C::NT>(sD, Dg + qbeg * BQ, S - qbeg * BQ);
  cp_wait<1>();
  __syncthreads();
  uint32_t kf[C::KEEP ? HD / 16 : 1][4], vf[C::KEEP ? HD / 16 : 1][4];
  if (C::KEEP) {
    load_afrags<HD>(kf, sK, warp * 16, lane);
    load_afrags<HD>(vf, sV, warp * 16, lane);
  }
  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int keyA = k0 + warp * 16 + g, keyB = keyA + 8;

  for (int qb = qbeg; qb < nqb; ++qb) {
    const int buf = (qb - qbeg) & 1;
    if (qb + 1 < nqb) {
      load_q(qb + 1, buf ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int m0 = qb * BQ;
    const bf16* sQb = sQ + buf * BQ * LDS;
    const bf16* sGb = sG + buf * BQ * LDS;
    const float* sLb = sL + buf * BQ;
    const float* sDb = sD + buf * BQ;
    if (m0 + BQ - 1 >= k0 + warp * 16) {
      float st[BQ / 8][4], dpt[BQ / 8][4];
#pragma unroll
      for (int i = 0; i < BQ / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
      mma_abt<HD, BQ, !C::KEEP>(st, kf, sK, warp * 16, sQb, lane);
      mma_abt<HD, BQ, !C::KEEP>(dpt, vf, sV, warp * 16, sGb, lane);
#pragma unroll
      for (int nt = 0; nt < BQ / 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int ql = nt * 8 + tg * 2 + (e & 1);
          const int q = m0 + ql;
          const int key = e < 2 ? keyA : keyB;
          const float p = (q >= key && q < S) ? exp2f(st[nt][e] * sl2 - sLb[ql] * LOG2E) : 0.f;
          st[nt][e] = p;
          dpt[nt][e] = p * (dpt[nt][e] - sDb[ql]);
        }
      }
      mma_pv<HD, BQ>(dv, st, sGb, lane);
      mma_pv<HD, BQ>(dk, dpt, sQb, lane);
    }
    __syncthreads();
    if (qb + 1 < nqb) {
      // lse/delta of the next block go to the other half (plain loads, after the barrier)
      load_vec<BQ, C::NT>(sL + (buf ^ 1) * BQ, Lg + (qb + 1) * BQ, S - (qb + 1) * BQ);
      load_vec<BQ, C::NT>(sD + (buf ^ 1) * BQ, Dg + (qb + 1) * BQ, S - (qb + 1) * BQ);
    }
  }
  bf16* base = dqkv + static_cast<int64_t>(b) * S * ldd + h * HD;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int col = i * 8 + tg * 2;
    if (keyA < S) {
      *reinterpret_cast<uint32_t*>(base + static_cast<int64_t>(keyA) * ldd + d + col) = pack2(dk[i][0] * scale, dk[i][1] * scale);
      *reinterpret_cast<uint32_t*>(base + static_cast<int64_t>(keyA) * ldd + 2 * d + col) = pack2(dv[i][0], dv[i][1]);
    }
    if (keyB < S) {
      *reinterpret_cast<uint32_t*>(base + static_cast<int64_t>(keyB) * ldd + d + col) = pack2(dk[i][2] * scale, dk[i][3] * scale);
      *reinterpret_cast<uint32_t*>(base + static_cast<int64_t>(keyB) * ldd + 2 * d + col) = pack2(dv[i][2], dv[i][3]);
    }
  }
}

template <int HD>
__global__ void __launch_bounds__(128) fa_bwd_dq(const bf16* __restrict__ qkv, int64_t ldq,
                                                 const bf16* __restrict__ dO, int64_t ldo,
                                                 const float* __restrict__ lse,
                                                 const float* __restrict__ delta,
                                                 bf16* __restrict__ dqkv, int64_t ldd, int H,
                                                 int S, float sl2, float scale) {
  using C = BwdCfg<HD>;
  constexpr int BK = C::BK, BQ = C::BQ2, LDS = C::LDS;
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sQ = reinterpret_cast<bf16*>(smraw);
  bf16* sG = sQ + BQ * LDS;
  bf16* sK = sG + BQ * LDS;        // [2][BK][LDS]
  bf16* sV = sK + 2 * BK * LDS;    // [2][BK][LDS]
  const int nqb = (S + BQ - 1) / BQ;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int d = H * HD;
  const bf16* Qg = qkv + static_cast<int64_t>(b) * S * ldq + h * HD;
  const bf16* Kg = Qg + d;
  const bf16* Vg = Qg + 2 * d;
  const bf16* Gg = dO + static_cast<int64_t>(b) * S * ldo + h * HD;
  const int q0 = qb * BQ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  const int rowA = q0 + warp * 16 + g, rowB = rowA + 8;
  const int kend = min(S, q0 + BQ);
  const int nkb = (kend + BK - 1) / BK;

  load_tile<BQ, HD, C::NT>(sQ, Qg + static_cast<int64_t>(q0) * ldq, ldq, S - q0);
  load_tile<BQ, HD, C::NT>(sG, Gg + static_cast<int64_t>(q0) * ldo, ldo, S - q0);
  cp_commit();
  load_tile<BK, HD, C::NT>(sK, Kg, ldq, S);
  load_tile<BK, HD, C::NT>(sV, Vg, ldq, S);
  cp_commit();
  cp_wait<1>();
  __syncthreads();
  uint32_t qf[C::KEEP ? HD / 16 : 1][4], gf[C::KEEP ? HD / 16 : 1][4];
  if (C::KEEP) {
    load_afrags<HD>(qf, sQ, warp * 16, lane);
    load_afrags<HD>(gf, sG, warp * 16, lane);
  }
  const float* Lr = lse + (static_cast<int64_t>(b) * H + h) * S;
  const float* Dr = delta + (static_cast<int64_t>(b) * H + h) * S;
  const float lA = rowA < S ? Lr[rowA] * LOG2E : 0.f, lB = rowB < S ? Lr[rowB] * LOG2E : 0.f;
  const float dA = rowA < S ? Dr[rowA] : 0.f, dB = rowB < S ? Dr[rowB] : 0.f;
  float dq[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int kb = 0; kb < nkb; ++kb) {
    if (kb + 1 < nkb) {
      const int n1 = (kb + 1) * BK;
      load_tile<BK, HD, C::NT>(sK + ((kb + 1) & 1) * BK * LDS, Kg + static_cast<int64_t>(n1) * ldq, ldq, S - n1);
      load_tile<BK, HD, C::NT>(sV + ((kb + 1) & 1) * BK * LDS, Vg + static_cast<int64_t>(n1) * ldq, ldq, S - n1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int n0 = kb * BK;
    const bf16* sKb = sK + (kb & 1) * BK * LDS;
    const bf16* sVb = sV + (kb & 1) * BK * LDS;
    if (n0 <= q0 + warp * 16 + 15 && q0 + warp * 16 < S) {
      float s[BK / 8][4], dp[BK / 8][4];
#pragma unroll
      for (int i = 0; i < BK / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
      mma_abt<HD, BK, !C::KEEP>(s, qf, sQ, warp * 16, sKb, lane);
      mma_abt<HD, BK, !C::KEEP>(dp, gf, sG, warp * 16, sVb, lane);
#pragma unroll
      for (int nt = 0; nt < BK / 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = n0 + nt * 8 + tg * 2 + (e & 1);
          const int row = e < 2 ? rowA : rowB;
          const float p = (key <= row && key < S && row < S)
                              ? exp2f(s[nt][e] * sl2 - (e < 2 ? lA : lB)) : 0.f;
          s[nt][e] = p * (dp[nt][e] - (e < 2 ? dA : dB));
        }
      }
      mma_pv<HD, BK>(dq, s, sKb, lane);
    }
    __syncthreads();
  }
  bf16* base = dqkv + static_cast<int64_t>(b) * S * ldd + h * HD;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int col = i * 8 + tg * 2;
    if (rowA < S)
      *reinterpret_cast<uint32_t*>(base + static_cast<int64_t>(rowA) * ldd + col) = pack2(dq[i][0] * scale, dq[i][1] * scale);
    if (rowB < S)
      *reinterpret_cast<uint32_t*>(base + static_cast<int64_t>(rowB) * ldd + col) = pack2(dq[i][2] * scale, dq[i][3] * scale);
  }
}

// One flag per kernel instantiation (kernels with equal signatures share a
// function-pointer type, so the flag must be keyed on the kernel itself).
template <auto Kernel>
int set_smem(int bytes) {
  static bool done = false;
  if (!done) {
    PP_CUDA_TRY(cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done = true;
  }
  return PC_OK;
}

template <int HD>
int fwd2_impl(int B, int H, int S, const void* qkv, int64_t ldq, void* o, int64_t ldo, float* lse,
              cudaStream_t st) {
  using C = Fwd2Cfg<HD>;
  int rc = set_smem<fa_fwd2<HD>>(C::SMEM);
  if (rc) return rc;
  dim3 grid((S + C::BM - 1) / C::BM, B * H);
  const float sl2 = LOG2E / sqrtf(static_cast<float>(HD));
  fa_fwd2<HD><<<grid, C::NT, C::SMEM, st>>>(static_cast<const bf16*>(qkv), ldq,
                                             static_cast<bf16*>(o), ldo, lse, H, S, sl2);
  return check_launch("fa_fwd2");
}

int g_fwd_variant = 2;

template <int HD>
int fwd_impl(int B, int H, int S, const void* qkv, int64_t ldq, void* o, int64_t ldo, float* lse,
             cudaStream_t st) {
  if constexpr (HD == 64) {
    if (g_fwd_variant == 2) return fwd2_impl<HD>(B, H, S, qkv, ldq, o, ldo, lse, st);
  }
  using C = FwdCfg<HD>;
  int rc = set_smem<fa_fwd<HD>>(C::SMEM);
  if (rc) return rc;
  dim3 grid((S + C::BM - 1) / C::BM, B * H);
  const float sl2 = LOG2E / sqrtf(static_cast<float>(HD));
  fa_fwd<HD><<<grid, C::NT, C::SMEM, st>>>(static_cast<const bf16*>(qkv), ldq,
                                            static_cast<bf16*>(o), ldo, lse, H, S, sl2);
  return check_launch("fa_fwd");
}

template <int HD>
int bwd_impl(int B, int H, int S, const void* qkv, int64_t ldq, const void* o, const void* dO,
             int64_t ldo, const float* lse, float* delta, void* dqkv, int64_t ldd, cudaStream_t st) {
  using C = BwdCfg<HD>;
  int rc = attention_delta(PC_BF16, B, H, S, HD, o, dO, ldo, delta, st);
  if (rc) return rc;
  rc = set_smem<fa_bwd_dkdv<HD>>(C::SMEM_KV);
  if (rc) return rc;
  rc = set_smem<fa_bwd_dq<HD>>(C::SMEM_Q);
  if (rc) return rc;
  const float scale = 1.f / sqrtf(static_cast<float>(HD));
  const float sl2 = scale * LOG2E;
  dim3 g1((S + C::BK - 1) / C::BK, B * H);
  fa_bwd_dkdv<HD><<<g1, C::NT, C::SMEM_KV, st>>>(static_cast<const bf16*>(qkv), ldq,
                                                  static_cast<const bf16*>(dO), ldo, lse, delta,
                                                  static_cast<bf16*>(dqkv), ldd, H, S, sl2, scale);
  rc = check_launch("fa_bwd_dkdv");
  if (rc) return rc;
  dim3 g2((S + C::BQ2 - 1) / C::BQ2, B * H);
  fa_bwd_dq<HD><<<g2, C::NT, C::SMEM_Q, st>>>(static_cast<const bf16*>(qkv), ldq,
                                               static_cast<const bf16*>(dO), ldo, lse, delta,
                                               static_cast<bf16*>(dqkv), ldd, H, S, sl2, scale);
  return check_launch("fa_bwd_dq");
}

}  // namespace

bool attention_tc_supported(int hd, int64_t ld_qkv, int64_t ld_o) {
  return (hd == 64 || hd == 128) && ld_qkv % 8 == 0 && ld_o % 8 == 0;
}

int attention_fwd_tc(int B, int H, int S, int hd, const void* qkv, int64_t ld_qkv, void* o,
                     int64_t ld_o, float* lse, cudaStream_t st) {
  if (hd == 64) return fwd_impl<64>(B, H, S, qkv, ld_qkv, o, ld_o, lse, st);
  return fwd_impl<128>(B, H, S, qkv, ld_qkv, o, ld_o, lse, st);
}

int attention_bwd_tc(int B, int H, int S, int hd, const void* qkv, int64_t ld_qkv, const void* o,
                     const void* dO, int64_t ld_o, const float* lse, float* delta, void* dqkv,
                     int64_t ld_dqkv, cudaStream_t st) {
  if (hd == 64)
    return bwd_impl<64>(B, H, S, qkv, ld_qkv, o, dO, ld_o, lse, delta, dqkv, ld_dqkv, st);
  return bwd_impl<128>(B, H, S, qkv, ld_qkv, o, dO, ld_o, lse, delta, dqkv, ld_dqkv, st);
}

}  // namespace pp200
