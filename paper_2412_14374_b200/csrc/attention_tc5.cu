// tcgen05 causal flash-attention forward (bf16, head_dim 64), sm_100a.
//
// Semantics: oracle/gpt.py `attention` (exact softmax, causal), same layout
// contract as attention_tc.cu (qkv [B*S, ld], o [B*S, ld_o], lse [B,H,S]).
//
// One CTA = 128 query rows of one (batch, head); 8 warps:
//   warp 0      TMA producer: Q tile once, then K/V tiles of 64 keys into a
//               128B-swizzled smem ring
//   warp 1      single-thread tcgen05.mma issuer, one key block ahead:
//                 S_j = Q K_j^T  (M=128, N=64 keys, K=64) -> TMEM S[j % 2]
//                 O  += P_j V_j  (M=128, N=64 dims, K=64) -> TMEM O
//               S_{j+1} is issued before PV_j, so the tensor core computes
//               the next scores while the softmax warps work on block j.
//   warp 2      TMEM allocator (256 columns: S0, S1, O; 2 CTAs fit per SM)
//   warps 4..7  softmax: one thread owns one query row (TMEM lane), so row
//               max / sum need no shuffles; P_j is written as bf16 into the
//               128B-swizzled K-major smem tile P[j % 2] (the MMA's A operand);
//               O is rescaled in TMEM when the running max moves.
// Barriers: s_full[i] (S_j landed), p_full[i] (P_j staged), pv_done[i]
// (PV_j retired: P[i] reusable, O up to date).
#include <cudaTypedefs.h>

#include "common.cuh"

namespace pp200 {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder_fn();

namespace {

using bf16 = __nv_bfloat16;
constexpr int F_BM = 128, F_BN = 64, F_HD = 64, F_STAGES = 3, F_THREADS = 256;
constexpr int F_Q_BYTES = F_BM * F_HD * 2;    // 16 KB
constexpr int F_KV_BYTES = F_BN * F_HD * 2;   // 8 KB
constexpr int F_P_BYTES = F_BM * F_BN * 2;    // 16 KB
constexpr int F_SMEM = F_Q_BYTES + 2 * F_STAGES * F_KV_BYTES + 2 * F_P_BYTES + 1024 + 256;
constexpr float F_LN2 = 0.6931471805599453f;

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// Paired fp32 arithmetic (FFMA2 / FADD2 on sm_100a) on two floats in a b64.
__device__ __forceinline__ uint64_t pack_f2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack_f2(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(F_THREADS, 2)
    fa_fwd_tc5(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ o, int64_t ldo,
               float* __restrict__ lse, int H, int S, float sl2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + F_Q_BYTES;
  uint8_t* sV = sK + F_STAGES * F_KV_BYTES;
  uint8_t* sP = sV + F_STAGES * F_KV_BYTES;
  uint64_t* bar_q = reinterpret_cast<uint64_t*>(sP + 2 * F_P_BYTES);
  uint64_t* kv_full = bar_q + 1;
  uint64_t* kv_empty = kv_full + F_STAGES;
  uint64_t* s_full = kv_empty + F_STAGES;  // [2]
  uint64_t* p_full = s_full + 2;           // [2]
  uint64_t* pv_done = p_full + 2;          // [2]
  uint64_t* o_done = pv_done + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (S + F_BM - 1) / F_BM;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);  // long (late) tiles first
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int d = H * F_HD;
  const int q0 = qb * F_BM;
  const int brow = b * S;  // first row of this batch in the [B*S, ld] tensors
  const int nkb = (min(S, q0 + F_BM) + F_BN - 1) / F_BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    mbar_init(bar_q, 1);
    for (int s = 0; s < F_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 128;  // S[i] at tS + 64 i

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(bar_q, F_Q_BYTES);
      tma_load_2d(sQ, &tm, bar_q, h * F_HD, brow + q0);
      tma_load_2d(sQ + F_Q_BYTES / 2, &tm, bar_q, h * F_HD, brow + q0 + 64);
      for (int j = 0; j < nkb; ++j) {
        const int s = j % F_STAGES;
        const uint32_t ph = (j / F_STAGES) & 1;
        mbar_wait(&kv_empty[s], ph ^ 1);
        mbar_expect_tx(&kv_full[s], 2 * F_KV_BYTES);
        tma_load_2d(sK + s * F_KV_BYTES, &tm, &kv_full[s], d + h * F_HD, brow + j * F_BN);
        tma_load_2d(sV + s * F_KV_BYTES, &tm, &kv_full[s], 2 * d + h * F_HD, brow + j * F_BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t ID_S = umma_idesc_bf16(F_BM, F_BN, 0, 0);  // Q, K both K-major
      constexpr uint32_t ID_O = umma_idesc_bf16(F_BM, F_HD, 0, 1);  // P K-major, V MN-major
      mbar_wait(bar_q, 0);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_s = [&](int j) {  // S_j = Q K_j^T into S[j % 2]
        const int s = j % F_STAGES;
        mbar_wait(&kv_full[s], (j / F_STAGES) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + s * F_KV_BYTES);
#pragma unroll
        for (int k = 0; k < F_HD / 16; ++k)
          tc_mma_f16(tS + (j & 1) * 64, umma_sdesc_sw128(q_addr + k * 32, 16, 1024),
                     umma_sdesc_sw128(k_addr + k * 32, 16, 1024), ID_S, k > 0 ? 1u : 0u);
        tc_commit(&s_full[j & 1]);
      };
      issue_s(0);
      for (int j = 0; j < nkb; ++j) {
        // S[(j+1) % 2] was last read by softmax j-1, which finished before PV_{j-1}
        if (j + 1 < nkb) issue_s(j + 1);
        const int s = j % F_STAGES;
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t p_addr = smem_u32(sP + (j & 1) * F_P_BYTES);
        const uint32_t v_addr = smem_u32(sV + s * F_KV_BYTES);
#pragma unroll
        for (int k = 0; k < F_BN / 16; ++k)
          tc_mma_f16(tO, umma_sdesc_sw128(p_addr + k * 32, 16, 1024),
                     umma_sdesc_sw128(v_addr + k * 2048, 8192, 1024), ID_O,
                     (j > 0 || k > 0) ? 1u : 0u);
        tc_commit(&pv_done[j & 1]);
        tc_commit(&kv_empty[s]);
      }
      tc_commit(o_done);
    }
  } else if (warp >= 4) {
    const int qw = warp & 3;              // TMEM lane quarter
    const int r = qw * 32 + lane;          // row within the tile
    const int row = q0 + r;                // query index within the sequence
    const uint32_t lane_off = static_cast<uint32_t>(qw * 32) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sr[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(tS + (j & 1) * 64 + lane_off + c * 16, sr + c * 16);
      tc_wait_ld();
      float* sv = reinterpret_cast<float*>(sr);
      const int n0 = j * F_BN;
      const bool edge = n0 + F_BN - 1 > q0 || n0 + F_BN > S;  // diagonal or ragged block
      // max of the raw scores (the positive scale commutes with max), 8
      // independent chains; masked entries become -inf
      float mx8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
      if (edge) {
#pragma unroll
        for (int i = 0; i < F_BN; ++i)
          if (n0 + i > row || n0 + i >= S) sv[i] = -INFINITY;
      }
#pragma unroll
      for (int i = 0; i < F_BN; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], sv[i]);
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
      // Lazy rescaling (FA4): keep the running reference max unless the row
      // max grows by more than 8 (log2 units, P <= 256 stays exact enough in
      // bf16); O and l only need a correction when the reference moves.
      const float mn = fmaxf(m, mx);
      float corr = 1.f;
      if (j == 0 || m == -INFINITY) {
        m = mn == -INFINITY ? 0.f : mn;
        corr = 0.f;  // nothing accumulated yet
      } else if (mn > m + 8.f) {
        corr = ex2(m - mn);
        m = mn;
      }
      // p = 2^(s * scale - m): one paired FMA per two scores, paired sums
      const uint64_t sc2 = pack_f2(sl2, sl2), nm2 = pack_f2(-m, -m);
      uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
      for (int i = 0; i < F_BN; i += 2) {
        float p0, p1;
        unpack_f2(ffma2(pack_f2(sv[i], sv[i + 1]), sc2, nm2), p0, p1);
        p0 = ex2(p0);
        p1 = ex2(p1);
        sv[i] = p0;
        sv[i + 1] = p1;
        acc2[(i >> 1) & 3] = fadd2(acc2[(i >> 1) & 3], pack_f2(p0, p1));
      }
      float sa[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) unpack_f2(acc2[k], sa[2 * k], sa[2 * k + 1]);
      const float sum = ((sa[0] + sa[1]) + (sa[2] + sa[3])) + ((sa[4] + sa[5]) + (sa[6] + sa[7]));
      l = l * corr + sum;
      // P[j % 2] was read by PV_{j-2}
      if (j >= 2) mbar_wait(&pv_done[j & 1], ((j - 2) >> 1) & 1);
      // P row -> smem, K-major with 128B swizzle (8 chunks of 8 bf16)
      uint8_t* sPj = sP + (j & 1) * F_P_BYTES;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 u;
        __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int k = 0; k < 4; ++k) hp[k] = __floats2bfloat162_rn(sv[8 * c + 2 * k], sv[8 * c + 2 * k + 1]);
        *reinterpret_cast<uint4*>(sPj + r * 128 + ((c ^ (r & 7)) << 4)) = u;
      }
      fence_proxy_async_smem();
      // rescale O by corr once PV_{j-1} has retired
      if (j > 0 && __any_sync(0xffffffffu, corr != 1.f && l > 0.f)) {
        mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t orr[16];
          tmem_ld16(tO + lane_off + c * 16, orr);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) orr[i] = __float_as_uint(__uint_as_float(orr[i]) * corr);
          tmem_st16(tO + lane_off + c * 16, orr);
        }
        tc_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j & 1]);
    }
    mbar_wait(o_done, 0);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    bf16* orow = o + static_cast<int64_t>(brow + row) * ldo + h * F_HD;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t orr[16];
      tmem_ld16(tO + lane_off + c * 16, orr);
      tc_wait_ld();
      if (row < S) {
        uint4 u[2];
        __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(u);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          hp[k] = __floats2bfloat162_rn(__uint_as_float(orr[2 * k]) * inv,
                                        __uint_as_float(orr[2 * k + 1]) * inv);
        reinterpret_cast<uint4*>(orow + c * 16)[0] = u[0];
        reinterpret_cast<uint4*>(orow + c * 16)[1] = u[1];
      }
    }
    if (row < S) lse[(static_cast<int64_t>(b) * H + h) * S + row] = (m + log2f(l)) * F_LN2;
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 256);
}


// ------------------------------------------------------------------ backward
// Writes 16 bf16 (two 16 B chunks, logical chunk index c2 and c2+1) of row r
// into a 128B-swizzled [rows x 64] K-major tile.
__device__ __forceinline__ void st_row16(uint8_t* tile, int r, int c2, const float* v) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint4 u;
    __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) hp[k] = __floats2bfloat162_rn(v[8 * h + 2 * k], v[8 * h + 2 * k + 1]);
    *reinterpret_cast<uint4*>(tile + r * 128 + (((c2 + h) ^ (r & 7)) << 4)) = u;
  }
}

__device__ __forceinline__ void store_row64(bf16* dst, const uint32_t* acc, float scale) {
  uint4 u[8];
  __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(u);
#pragma unroll
  for (int k = 0; k < 32; ++k)
    hp[k] = __floats2bfloat162_rn(__uint_as_float(acc[2 * k]) * scale, __uint_as_float(acc[2 * k + 1]) * scale);
#pragma unroll
  for (int k = 0; k < 8; ++k) reinterpret_cast<uint4*>(dst)[k] = u[k];
}

constexpr int B_KEYS = 128, B_Q = 64;  // dK/dV: 128 keys per CTA, 64-query blocks
constexpr int BKV_SMEM = 2 * 16384 /*K,V*/ + 2 * 2 * 8192 /*Q,dO stages*/ + 2 * 16384 /*P^T,dS^T*/ + 1024 + 256;

// dK, dV for 128 keys of one (batch, head): S^T = K Q^T and dP^T = V dO^T per
// 64-query block (TMEM), P^T / dS^T built by one thread per key row, then
// dV += P^T dO and dK += dS^T Q (TMEM accumulators).
__global__ void __launch_bounds__(F_THREADS, 2)
    fa_bwd_dkdv_tc5(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tg,
                    const float* __restrict__ lse, const float* __restrict__ delta,
                    bf16* __restrict__ dqkv, int64_t ldd, int H, int S, float sl2, float scale) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + 16384;
  uint8_t* sQ = sV + 16384;      // [2][64 x 64]
  uint8_t* sG = sQ + 2 * 8192;   // dO, [2][64 x 64]
  uint8_t* sPt = sG + 2 * 8192;  // P^T  [128 keys x 64 q]
  uint8_t* sDt = sPt + 16384;    // dS^T [128 keys x 64 q]
  uint64_t* bar_kv = reinterpret_cast<uint64_t*>(sDt + 16384);
  uint64_t* q_full = bar_kv + 1;
  uint64_t* q_empty = q_full + 2;
  uint64_t* s_full = q_empty + 2;
  uint64_t* p_full = s_full + 1;
  uint64_t* done = p_full + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x;  // early key blocks see the most query blocks: launch first
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int d = H * F_HD;
  const int k0 = kb * B_KEYS;
  const int brow = b * S;
  const int qbeg = k0 / B_Q, nqb = (S + B_Q - 1) / B_Q;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tg);
    mbar_init(bar_kv, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tSt = tmem, tPt = tmem + 64, tdV = tmem + 128, tdK = tmem + 192;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(bar_kv, 2 * 16384);
      for (int hf = 0; hf < 2; ++hf) {
        tma_load_2d(sK + hf * 8192, &tq, bar_kv, d + h * F_HD, brow + k0 + hf * 64);
        tma_load_2d(sV + hf * 8192, &tq, bar_kv, 2 * d + h * F_HD, brow + k0 + hf * 64);
      }
      for (int qb = qbeg, i = 0; qb < nqb; ++qb, ++i) {
        const int st = i & 1;
        mbar_wait(&q_empty[st], ((i >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[st], 2 * 8192);
        tma_load_2d(sQ + st * 8192, &tq, &q_full[st], h * F_HD, brow + qb * B_Q);
        tma_load_2d(sG + st * 8192, &tg, &q_full[st], h * F_HD, brow + qb * B_Q);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t ID_T = umma_idesc_bf16(128, B_Q, 0, 0);   // K/V x (Q/dO)^T, N = 64 queries
      constexpr uint32_t ID_A = umma_idesc_bf16(128, F_HD, 0, 1);  // P^T/dS^T x (dO/Q), N = 64 dims
      mbar_wait(bar_kv, 0);
      tc_fence_after();
      const uint32_t ka = smem_u32(sK), va = smem_u32(sV), pa = smem_u32(sPt), da = smem_u32(sDt);
      for (int qb = qbeg, i = 0; qb < nqb; ++qb, ++i) {
        const int st = i & 1;
        mbar_wait(&q_full[st], (i >> 1) & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(sQ + st * 8192), ga = smem_u32(sG + st * 8192);
#pragma unroll
        for (int k = 0; k < F_HD / 16; ++k) {
          tc_mma_f16(tSt, umma_sdesc_sw128(ka + k * 32, 16, 1024), umma_sdesc_sw128(qa + k * 32, 16, 1024), ID_T, k > 0 ? 1u : 0u);
          tc_mma_f16(tPt, umma_sdesc_sw128(va + k * 32, 16, 1024), umma_sdesc_sw128(ga + k * 32, 16, 1024), ID_T, k > 0 ? 1u : 0u);
        }
        tc_commit(s_full);
        mbar_wait(p_full, i & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < B_Q / 16; ++k) {
          const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
          tc_mma_f16(tdV, umma_sdesc_sw128(pa + k * 32, 16, 1024), umma_sdesc_sw128(ga + k * 2048, 8192, 1024), ID_A, acc);
          tc_mma_f16(tdK, umma_sdesc_sw128(da + k * 32, 16, 1024), umma_sdesc_sw128(qa + k * 2048, 8192, 1024), ID_A, acc);
        }
        tc_commit(&q_empty[st]);
      }
      tc_commit(done);
    }
  } else if (warp >= 4) {
    const int qw = warp & 3;
    const int r = qw * 32 + lane;  // key row in the tile
    const int key = k0 + r;
    const uint32_t lo = static_cast<uint32_t>(qw * 32) << 16;
    const float* Lr = lse + (static_cast<int64_t>(b) * H + h) * S;
    const float* Dr = delta + (static_cast<int64_t>(b) * H + h) * S;
    for (int qb = qbeg, i = 0; qb < nqb; ++qb, ++i) {
      mbar_wait(s_full, i & 1);
      tc_fence_after();
      const int m0 = qb * B_Q;
      // lse / delta of this query block: every thread reads the same 64 values
      // (16 B broadcast loads; the block never straddles the end of a batch row
      // range because S is a multiple of 8)
      const bool full = m0 + B_Q <= S && (S % 4) == 0;
#pragma unroll 1
      for (int c = 0; c < B_Q / 16; ++c) {
        uint32_t sr[16], dr[16];
        tmem_ld16(tSt + lo + c * 16, sr);
        tmem_ld16(tPt + lo + c * 16, dr);
        float lq[16], dq[16];
        if (full) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(Lr + m0 + c * 16) + v);
            const float4 g = __ldg(reinterpret_cast<const float4*>(Dr + m0 + c * 16) + v);
            lq[4 * v] = a.x; lq[4 * v + 1] = a.y; lq[4 * v + 2] = a.z; lq[4 * v + 3] = a.w;
            dq[4 * v] = g.x; dq[4 * v + 1] = g.y; dq[4 * v + 2] = g.z; dq[4 * v + 3] = g.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int q = m0 + c * 16 + e;
            lq[e] = q < S ? __ldg(Lr + q) : 0.f;
            dq[e] = q < S ? __ldg(Dr + q) : 0.f;
          }
        }
        tc_wait_ld();
        float pv[16], dv[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int q = m0 + c * 16 + e;
          const bool ok = q >= key && q < S;
          const float p = ok ? ex2(__uint_as_float(sr[e]) * sl2 - lq[e] * 1.4426950408889634f) : 0.f;
          pv[e] = p;
          dv[e] = ok ? p * (__uint_as_float(dr[e]) - dq[e]) : 0.f;
        }
        st_row16(sPt, r, 2 * c, pv);
        st_row16(sDt, r, 2 * c, dv);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(done, 0);
    tc_fence_after();
    uint32_t acc[64];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld16(tdV + lo + c * 16, acc + c * 16);
    tc_wait_ld();
    bf16* base = dqkv + static_cast<int64_t>(brow + key) * ldd + h * F_HD;
    if (key < S) store_row64(base + 2 * d, acc, 1.f);
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld16(tdK + lo + c * 16, acc + c * 16);
    tc_wait_ld();
    if (key < S) store_row64(base + d, acc, scale);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 256);
}

constexpr int BQ_SMEM = 2 * 16384 /*Q,dO*/ + 2 * 2 * 8192 /*K,V stages*/ + 16384 /*dS*/ + 1024 + 256;

// dQ for 128 queries of one (batch, head): S = Q K^T, dP = dO V^T per 64-key
// block, dS by one thread per query row, dQ += dS K (TMEM accumulator).
__global__ void __launch_bounds__(F_THREADS, 1)
    fa_bwd_dq_tc5(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tg,
                  const float* __restrict__ lse, const float* __restrict__ delta,
                  bf16* __restrict__ dqkv, int64_t ldd, int H, int S, float sl2, float scale) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sG = sQ + 16384;
  uint8_t* sK = sG + 16384;       // [2][64 x 64]
  uint8_t* sV = sK + 2 * 8192;    // [2][64 x 64]
  uint8_t* sD = sV + 2 * 8192;    // dS [128 q x 64 keys]
  uint64_t* bar_q = reinterpret_cast<uint64_t*>(sD + 16384);
  uint64_t* kv_full = bar_q + 1;
  uint64_t* kv_empty = kv_full + 2;
  uint64_t* s_full = kv_empty + 2;
  uint64_t* p_full = s_full + 1;
  uint64_t* done = p_full + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (S + F_BM - 1) / F_BM;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int d = H * F_HD;
  const int q0 = qb * F_BM;
  const int brow = b * S;
  const int nkb = (min(S, q0 + F_BM) + F_BN - 1) / F_BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tg);
    mbar_init(bar_q, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tP = tmem + 64, tdQ = tmem + 128;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(bar_q, 2 * 16384);
      for (int hf = 0; hf < 2; ++hf) {
        tma_load_2d(sQ + hf * 8192, &tq, bar_q, h * F_HD, brow + q0 + hf * 64);
        tma_load_2d(sG + hf * 8192, &tg, bar_q, h * F_HD, brow + q0 + hf * 64);
      }
      for (int j = 0; j < nkb; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * 8192);
        tma_load_2d(sK + st * 8192, &tq, &kv_full[st], d + h * F_HD, brow + j * F_BN);
        tma_load_2d(sV + st * 8192, &tq, &kv_full[st], 2 * d + h * F_HD, brow + j * F_BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t ID_T = umma_idesc_bf16(128, F_BN, 0, 0);  // Q/dO x (K/V)^T
      constexpr uint32_t ID_A = umma_idesc_bf16(128, F_HD, 0, 1);  // dS x K (MN-major)
      mbar_wait(bar_q, 0);
      tc_fence_after();
      const uint32_t qa = smem_u32(sQ), ga = smem_u32(sG), dsa = smem_u32(sD);
      for (int j = 0; j < nkb; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(sK + st * 8192), va = smem_u32(sV + st * 8192);
#pragma unroll
        for (int k = 0; k < F_HD / 16; ++k) {
          tc_mma_f16(tS, umma_sdesc_sw128(qa + k * 32, 16, 1024), umma_sdesc_sw128(ka + k * 32, 16, 1024), ID_T, k > 0 ? 1u : 0u);
          tc_mma_f16(tP, umma_sdesc_sw128(ga + k * 32, 16, 1024), umma_sdesc_sw128(va + k * 32, 16, 1024), ID_T, k > 0 ? 1u : 0u);
        }
        tc_commit(s_full);
        mbar_wait(p_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < F_BN / 16; ++k)
          tc_mma_f16(tdQ, umma_sdesc_sw128(dsa + k * 32, 16, 1024), umma_sdesc_sw128(ka + k * 2048, 8192, 1024), ID_A,
                     (j > 0 || k > 0) ? 1u : 0u);
        tc_commit(&kv_empty[st]);
      }
      tc_commit(done);
    }
  } else if (warp >= 4) {
    const int qw = warp & 3;
    const int r = qw * 32 + lane;
    const int row = q0 + r;
    const uint32_t lo = static_cast<uint32_t>(qw * 32) << 16;
    const int64_t vrow = (static_cast<int64_t>(b) * H + h) * S + row;
    const float l2 = row < S ? lse[vrow] * 1.4426950408889634f : 0.f;
    const float dl = row < S ? delta[vrow] : 0.f;
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      const int n0 = j * F_BN;
#pragma unroll
      for (int c = 0; c < F_BN / 16; ++c) {
        uint32_t sr[16], dr[16];
        tmem_ld16(tS + lo + c * 16, sr);
        tmem_ld16(tP + lo + c * 16, dr);
        tc_wait_ld();
        float dsv[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int key = n0 + c * 16 + e;
          const bool ok = key <= row && key < S && row < S;
          const float p = ok ? ex2(__uint_as_float(sr[e]) * sl2 - l2) : 0.f;
          dsv[e] = ok ? p * (__uint_as_float(dr[e]) - dl) : 0.f;
        }
        st_row16(sD, r, 2 * c, dsv);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(done, 0);
    tc_fence_after();
    uint32_t acc[64];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld16(tdQ + lo + c * 16, acc + c * 16);
    tc_wait_ld();
    if (row < S) store_row64(dqkv + static_cast<int64_t>(brow + row) * ldd + h * F_HD, acc, scale);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 256);
}

int make_tmap_rows64(CUtensorMap* m, const void* base, int64_t ld, int64_t rows) {
  auto enc = tmap_encoder_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return PC_ERR_CUDA;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {64u, 64u};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (attention) failed (%d)", static_cast<int>(r));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}
}  // namespace

bool attention_tc5_supported(int hd, int64_t ld_qkv, int64_t ld_o, const void* qkv, const void* o) {
  return hd == F_HD && (ld_qkv * 2) % 16 == 0 && (ld_o * 2) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(qkv) & 15) == 0 && (reinterpret_cast<uintptr_t>(o) & 15) == 0;
}

int attention_fwd_tc5(int B, int H, int S, const void* qkv, int64_t ld_qkv, void* o, int64_t ld_o,
                      float* lse, cudaStream_t st) {
  auto enc = tmap_encoder_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return PC_ERR_CUDA;
  }
  CUtensorMap tm;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld_qkv), static_cast<cuuint64_t>(B) * S};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_qkv * 2)};
  cuuint32_t box[2] = {64u, 64u};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (attention) failed (%d)", static_cast<int>(r));
    return PC_ERR_CUDA;
  }
  static bool attr = false;
  if (!attr) {
    PP_CUDA_TRY(cudaFuncSetAttribute(fa_fwd_tc5, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM));
    attr = true;
  }
  dim3 grid((S + F_BM - 1) / F_BM, B * H);
  const float sl2 = 1.4426950408889634f / sqrtf(static_cast<float>(F_HD));
  fa_fwd_tc5<<<grid, F_THREADS, F_SMEM, st>>>(tm, static_cast<bf16*>(o), ld_o, lse, H, S, sl2);
  return check_launch("fa_fwd_tc5");
}

}  // namespace pp200

namespace pp200 {
int attention_delta(int dtype, int B, int H, int S, int hd, const void* o, const void* dO,
                    int64_t ld_o, float* delta, cudaStream_t st);

int attention_bwd_tc5(int B, int H, int S, const void* qkv, int64_t ld_qkv, const void* o,
                      const void* dO, int64_t ld_o, const float* lse, float* delta, void* dqkv,
                      int64_t ld_dqkv, cudaStream_t st) {
  int rc = attention_delta(PC_BF16, B, H, S, F_HD, o, dO, ld_o, delta, st);
  if (rc) return rc;
  CUtensorMap tq, tg;
  rc = make_tmap_rows64(&tq, qkv, ld_qkv, static_cast<int64_t>(B) * S);
  if (rc) return rc;
  rc = make_tmap_rows64(&tg, dO, ld_o, static_cast<int64_t>(B) * S);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    PP_CUDA_TRY(cudaFuncSetAttribute(fa_bwd_dkdv_tc5, cudaFuncAttributeMaxDynamicSharedMemorySize, BKV_SMEM));
    PP_CUDA_TRY(cudaFuncSetAttribute(fa_bwd_dq_tc5, cudaFuncAttributeMaxDynamicSharedMemorySize, BQ_SMEM));
    attr = true;
  }
  const float scale = 1.f / sqrtf(static_cast<float>(F_HD));
  const float sl2 = scale * 1.4426950408889634f;
  dim3 g1((S + B_KEYS - 1) / B_KEYS, B * H);
  fa_bwd_dkdv_tc5<<<g1, F_THREADS, BKV_SMEM, st>>>(tq, tg, lse, delta, static_cast<bf16*>(dqkv),
                                                    ld_dqkv, H, S, sl2, scale);
  rc = check_launch("fa_bwd_dkdv_tc5");
  if (rc) return rc;
  dim3 g2((S + F_BM - 1) / F_BM, B * H);
  fa_bwd_dq_tc5<<<g2, F_THREADS, BQ_SMEM, st>>>(tq, tg, lse, delta, static_cast<bf16*>(dqkv),
                                                 ld_dqkv, H, S, sl2, scale);
  return check_launch("fa_bwd_dq_tc5");
}
}  // namespace pp200
