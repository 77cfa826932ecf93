// tcgen05 causal flash attention, forward and backward, bf16, sm_100a.
//
// Semantics: oracle/gpt.py `attention` / `attention_bwd` (exact softmax,
// causal) and, with fewer key/value heads than query heads, oracle/llama.py
// `gqa_attention` (query head h reads kv head h / (H / Hkv); a kv head's
// gradient is the sum over its query heads).  Templated on the head dim
// HD in {64, 128} (GPT-2 configs C1-C3: 64; GPT-3 1.3B / Llama-8B, C4 / C5: 128).
//
// Layout contract (the stage activations): one packed
// projection buffer qkv [B*S, ld] holding H query heads, then Hkv key heads,
// then Hkv value heads, each HD columns wide; o [B*S, ld_o]; lse / delta
// [B, H, S] fp32; the gradient dqkv has qkv's layout.  Grouped-query heads
// are addressed in the TMA coordinates: no K/V expansion and no separate
// group reduction (the dK/dV kernel accumulates a kv head's whole group in
// TMEM).
//
// Every operand tile is a set of 128B-swizzled K-major "panels" of 64
// columns (one TMA box is 64 columns x 64 rows); a head of HD columns is
// HD / 64 panels side by side in shared memory.
#include <cudaTypedefs.h>

#include "common.cuh"

namespace pp200 {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder_fn();

namespace {

using bf16 = __nv_bfloat16;
constexpr float F_LN2 = 0.6931471805599453f;
constexpr float F_LOG2E = 1.4426950408889634f;

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
// O += A B with A (bf16, K-major, one row per TMEM lane, two values per
// 32-bit column) read from TMEM and B from shared memory.
__device__ __forceinline__ void tc_mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// 16 fp32 -> 8 packed bf16x2 words (lower K index in the low half)
__device__ __forceinline__ void pack_bf16x16(const float* v, uint32_t* w) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
    w[k] = *reinterpret_cast<uint32_t*>(&h);
  }
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Column of the first element of query head h / kv head hk (K or V) in qkv.
struct Heads {
  int H, Hkv, G, hd;
  __device__ __forceinline__ int qcol(int h) const { return h * hd; }
  __device__ __forceinline__ int kcol(int hk) const { return (H + hk) * hd; }
  __device__ __forceinline__ int vcol(int hk) const { return (H + Hkv + hk) * hd; }
};

// K-major descriptor of k-step k (16 elements of the contraction dim) of a
// tile made of 64-column panels `panel_bytes` apart.
__device__ __forceinline__ uint64_t kmajor_step(uint32_t base, int k, uint32_t panel_bytes) {
  return umma_sdesc_sw128(base + (k >> 2) * panel_bytes + (k & 3) * 32, 16, 1024);
}

// ------------------------------------------------------------------ forward
// One CTA = 128 query rows of one (batch, head); 8 warps:
//   warp 0      TMA producer: Q tile once, then K/V blocks of 64 keys into a
//               128B-swizzled smem ring
//   warp 1      single-thread tcgen05.mma issuer, one key block ahead:
//                 S_j = Q K_j^T  (M=128, N=64 keys, K=HD) -> TMEM S[j % 2]
//                 O  += P_j V_j  (M=128, N=HD dims, K=64) -> TMEM O
//               S_{j+1} is issued before PV_j, so the tensor core computes
//               the next scores while the softmax warps work on block j.
//   warp 2      TMEM allocator (256 columns: S0, S1, O; two CTAs fit per SM
//               and share the tensor core, hiding each other's softmax)
//   warps 4..7  softmax: one thread owns one query row (TMEM lane), so row
//               max / sum need no shuffles; P_j is written back as packed bf16
//               over its own score columns (the PV MMA reads A from TMEM);
//               O is rescaled in TMEM when the running max moves.
template <int HD>
struct Fwd {
  static constexpr int BM = 128, BN = 64, THREADS = 256;
  static constexpr int NP = HD / 64;                   // 64-column panels per head
  static constexpr int STAGES = HD == 64 ? 3 : 2;
  static constexpr int Q_PANEL = BM * 64 * 2;          // 16 KB
  static constexpr int KV_PANEL = BN * 64 * 2;         // 8 KB
  static constexpr int Q_BYTES = NP * Q_PANEL;
  static constexpr int KV_BYTES = NP * KV_PANEL;
  static constexpr int SMEM = Q_BYTES + 2 * STAGES * KV_BYTES + 1024 + 256;
  static constexpr int TMEM_COLS = 256;                // S0 | S1 | O (HD <= 128)
};

template <int HD, int SPLIT = 0>  // SPLIT: S and PV MMAs from two issuing warps (see fa_fwd64_tc5)
__global__ void __launch_bounds__(256, 2)
    fa_fwd_tc5(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ o, int64_t ldo,
               float* __restrict__ lse, Heads hs, int S, float sl2) {
  using K = Fwd<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + K::Q_BYTES;
  uint8_t* sV = sK + K::STAGES * K::KV_BYTES;
  uint64_t* bar_q = reinterpret_cast<uint64_t*>(sV + K::STAGES * K::KV_BYTES);
  uint64_t* kv_full = bar_q + 1;
  uint64_t* kv_empty = kv_full + K::STAGES;
  uint64_t* s_full = kv_empty + K::STAGES;  // [2]
  uint64_t* p_full = s_full + 2;            // [2]
  uint64_t* pv_done = p_full + 2;           // [2]
  uint64_t* o_done = pv_done + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int H = hs.H;
  const int nqb = (S + K::BM - 1) / K::BM;
  // grid (B*H, tiles): x varies fastest, so every head's longest (latest) tile
  // launches before any shorter one -- longest-first across the whole grid
  const int qb = nqb - 1 - static_cast<int>(blockIdx.y);
  const int b = blockIdx.x / H, h = blockIdx.x % H, hk = h / hs.G;
  const int q0 = qb * K::BM;
  const int brow = b * S;  // first row of this batch in the [B*S, ld] tensors
  const int nkb = (min(S, q0 + K::BM) + K::BN - 1) / K::BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    mbar_init(bar_q, 1);
    for (int s = 0; s < K::STAGES; ++s) {
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
  if (warp == 2) tmem_alloc(tslot, K::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 128;  // S[i] at tS + 64 i

  if (warp == 0) {
    // warp-uniform loops, one elected lane issuing (see fa_fwd64_tc5)
    if (elect_one()) {
      mbar_expect_tx(bar_q, K::Q_BYTES);
#pragma unroll
      for (int p = 0; p < K::NP; ++p)
        for (int hf = 0; hf < 2; ++hf)
          tma_load_2d(sQ + p * K::Q_PANEL + hf * (K::Q_PANEL / 2), &tm, bar_q, hs.qcol(h) + 64 * p,
                      brow + q0 + 64 * hf);
    }
    __syncwarp();
    for (int j = 0; j < nkb; ++j) {
      const int s = j % K::STAGES;
      const uint32_t ph = (j / K::STAGES) & 1;
      mbar_wait(&kv_empty[s], ph ^ 1);
      if (elect_one()) {
        mbar_expect_tx(&kv_full[s], 2 * K::KV_BYTES);
#pragma unroll
        for (int p = 0; p < K::NP; ++p) {
          tma_load_2d(sK + s * K::KV_BYTES + p * K::KV_PANEL, &tm, &kv_full[s],
                      hs.kcol(hk) + 64 * p, brow + j * K::BN);
          tma_load_2d(sV + s * K::KV_BYTES + p * K::KV_PANEL, &tm, &kv_full[s],
                      hs.vcol(hk) + 64 * p, brow + j * K::BN);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    constexpr uint32_t ID_S = umma_idesc_bf16(K::BM, K::BN, 0, 0);  // Q, K both K-major
    constexpr uint32_t ID_O = umma_idesc_bf16(K::BM, HD, 0, 1);     // P K-major, V MN-major
    mbar_wait(bar_q, 0);
    tc_fence_after();
    const uint32_t q_addr = smem_u32(sQ);
    auto issue_s = [&](int j) {  // S_j = Q K_j^T into S[j % 2]
      const int s = j % K::STAGES;
      mbar_wait(&kv_full[s], (j / K::STAGES) & 1);
      // S[j % 2] still holds P_{j-2}: wait until PV_{j-2} has read it
      if (j >= 2) mbar_wait(&pv_done[j & 1], ((j - 2) >> 1) & 1);
      tc_fence_after();
      const uint32_t k_addr = smem_u32(sK + s * K::KV_BYTES);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          tc_mma_f16(tS + (j & 1) * 64, kmajor_step(q_addr, k, K::Q_PANEL),
                     kmajor_step(k_addr, k, K::KV_PANEL), ID_S, k > 0 ? 1u : 0u);
        tc_commit(&s_full[j & 1]);
      }
      __syncwarp();
    };
    if (SPLIT) {
      for (int j = 0; j < nkb; ++j) issue_s(j);
    } else {
      issue_s(0);
    }
    for (int j = 0; j < nkb && !SPLIT; ++j) {
      // S[(j+1) % 2] was last read by softmax j-1, which finished before PV_{j-1}
      if (j + 1 < nkb) issue_s(j + 1);
      const int s = j % K::STAGES;
      mbar_wait(&p_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t v_addr = smem_u32(sV + s * K::KV_BYTES);
      const uint32_t tP = tS + (j & 1) * 64;  // P_j packed bf16, key chunk k at column 8 k
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < K::BN / 16; ++k)
          tc_mma_f16_ts(tO, tP + 8 * k, umma_sdesc_sw128(v_addr + k * 2048, K::KV_PANEL, 1024),
                        ID_O, (j > 0 || k > 0) ? 1u : 0u);
        tc_commit(&pv_done[j & 1]);
        tc_commit(&kv_empty[s]);
      }
      __syncwarp();
    }
    if (!SPLIT && elect_one()) tc_commit(o_done);
    __syncwarp();
  } else if (SPLIT && warp == 3) {
    constexpr uint32_t ID_O = umma_idesc_bf16(K::BM, HD, 0, 1);  // P K-major, V MN-major
    for (int j = 0; j < nkb; ++j) {
      const int s = j % K::STAGES;
      mbar_wait(&p_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t v_addr = smem_u32(sV + s * K::KV_BYTES);
      const uint32_t tP = tS + (j & 1) * 64;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < K::BN / 16; ++k)
          tc_mma_f16_ts(tO, tP + 8 * k, umma_sdesc_sw128(v_addr + k * 2048, K::KV_PANEL, 1024),
                        ID_O, (j > 0 || k > 0) ? 1u : 0u);
        tc_commit(&pv_done[j & 1]);
        tc_commit(&kv_empty[s]);  // K_j was read by S_j, retired before softmax j
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(o_done);
    __syncwarp();
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
      const int n0 = j * K::BN;
      const bool edge = n0 + K::BN - 1 > q0 || n0 + K::BN > S;  // diagonal or ragged block
      // max of the raw scores (the positive scale commutes with max), 8
      // independent chains; masked entries become -inf
      float mx8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
      if (edge) {
#pragma unroll
        for (int i = 0; i < K::BN; ++i)
          if (n0 + i > row || n0 + i >= S) sv[i] = -INFINITY;
      }
#pragma unroll
      for (int i = 0; i < K::BN; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], sv[i]);
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
      for (int i = 0; i < K::BN; i += 2) {
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
      // P row as packed bf16 over the first 32 columns of its own score buffer
      {
        uint32_t wv[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) pack_bf16x16(sv + 16 * c, wv + 8 * c);
        tmem_st16(tS + (j & 1) * 64 + lane_off, wv);
        tmem_st16(tS + (j & 1) * 64 + lane_off + 16, wv + 16);
        tc_wait_st();
      }
      // rescale O by corr once PV_{j-1} has retired
      if (j > 0 && __any_sync(0xffffffffu, corr != 1.f && l > 0.f)) {
        mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
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
    bf16* orow = o + static_cast<int64_t>(brow + row) * ldo + hs.qcol(h);
#pragma unroll
    for (int c = 0; c < HD / 16; ++c) {
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
  if (warp == 2) tmem_dealloc(tmem, K::TMEM_COLS);
}

// 2^x on the FMA pipe for a pair of fp32 values (x >= -126: j >= -126 keeps
// the exponent field of p * 2^j non-negative, p >= 2^-1/2): round-to-nearest
// split x = j + f (|f| <= 1/2) with the 1.5 * 2^23 shifter, a degree-3
// minimax polynomial for 2^f (max rel err 7.5e-5, well below the bf16
// rounding of P), then j added to the exponent field.  Takes part of the
// exp2 work off the MUFU unit (16 ex2 / SM / clk), which bounds head_dim 64.
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float& y0, float& y1) {
  constexpr float SH = 12582912.f;
  const uint64_t t = fadd2(pack_f2(x0, x1), pack_f2(SH, SH));
  const uint64_t j = fadd2(t, pack_f2(-SH, -SH));
  const uint64_t f = ffma2(j, pack_f2(-1.f, -1.f), pack_f2(x0, x1));
  uint64_t p = ffma2(f, pack_f2(0.05517166f, 0.05517166f), pack_f2(0.24261114f, 0.24261114f));
  p = ffma2(p, f, pack_f2(0.69326097f, 0.69326097f));
  p = ffma2(p, f, pack_f2(0.99992806f, 0.99992806f));
  float t0, t1, p0, p1;
  unpack_f2(t, t0, t1);
  unpack_f2(p, p0, p1);
  y0 = __uint_as_float(__float_as_uint(p0) + (__float_as_uint(t0) << 23));
  y1 = __uint_as_float(__float_as_uint(p1) + (__float_as_uint(t1) << 23));
}

// Forward, head_dim 64, persistent.  Measured on fa_fwd_tc5<64> (C2 shape,
// clock64 / %globaltimer traces and ablations, profiles/r02_attn_fwd64.txt):
// (1) a one-tile CTA spent ~2.7 us outside its key blocks (setup, Q load, first
// S, epilogue); (2) with P aliased over S, the MMA warp waited for PV_g to
// retire before it could issue S_{g+2} into the same columns, a full
// issue -> execute -> commit round trip per block (the MMA-only pipeline, no
// softmax math, ran 20.9 us); (3) a lane-0-only MMA / TMA branch made every
// wait and issue a divergent slow path.  So: two CTAs per SM walk the query
// tiles longest-first in snake order without draining between tiles (Q
// double-buffered; the next tile's scores are computed while the current tile
// finishes); P_g has its own TMEM buffer, so a score buffer is released as
// soon as the softmax warps have loaded it (s_free) and the MMA warp never
// waits on a PV; the producer / MMA warps run warp-uniform with one elected
// issuing lane.  O leaves through a per-warp TMA store (3-D map: rows clipped
// at the sequence end).  EMU of every 16 score columns take exp2 on the FMA
// pipe (exp2_poly2).  Ring / buffer phases run on CTA-wide block counters.
// TMEM (256 columns): S0 @0, S1 @64, P0 @128, P1 @160 (packed bf16), O @192.
#ifdef PP200_FA_TRACE
// tools/fa_trace.cu: clock64 stamps per (CTA < 64, event < 8, block < 32)
__device__ unsigned long long fa_trace_buf[64 * 8 * 32];
__device__ unsigned long long fa_trace_cta[1024 * 3];  // start / end %globaltimer, smid
#define FA_T(ev, idx)                                                                          \
  do {                                                                                         \
    if (blockIdx.x < 64 && (idx) < 32) fa_trace_buf[(blockIdx.x * 8 + (ev)) * 32 + (idx)] = clock64(); \
  } while (0)
__device__ __forceinline__ unsigned long long fa_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
#define FA_T(ev, idx) \
  do {                \
  } while (0)
#endif

struct Fwd64 {
  static constexpr int BM = 128, BN = 64, THREADS = 256, STAGES = 3;
  static constexpr int Q_BYTES = BM * 64 * 2;    // 16 KB
  static constexpr int KV_BYTES = BN * 64 * 2;   // 8 KB (one of K / V)
  static constexpr int O_WARP = 32 * 128;        // per softmax warp: 32 rows x 64 bf16
  static constexpr int SMEM = 2 * Q_BYTES + 2 * STAGES * KV_BYTES + 4 * O_WARP + 1024 + 256;
};

__device__ __forceinline__ void tma_store_3d(const void* tmap, const void* src, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// SPLIT: the S MMAs (warp 1) and the PV MMAs (warp 3) come from two issuing
// warps, so a PV is never queued behind an S issue that waits for K/V (the
// MMA-only pipeline, no softmax math: 24.1 -> 17.5 us at C2).
template <int EMU, int ABL = 0, int SPLIT = 0>  // ABL (tools/attn_ab.py): 1 no softmax math, 2 no MMAs
__global__ void __launch_bounds__(256, 2)
    fa_fwd64_tc5(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap to,
                 float* __restrict__ lse, int B, Heads hs, int S, float sl2) {
  using K = Fwd64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                                  // [2][128 x 64]
  uint8_t* sK = sQ + 2 * K::Q_BYTES;                   // [ST][64 x 64]
  uint8_t* sV = sK + K::STAGES * K::KV_BYTES;          // [ST][64 x 64]
  uint8_t* sO = sV + K::STAGES * K::KV_BYTES;          // [4 warps][32 x 64] staging
  uint64_t* q_full = reinterpret_cast<uint64_t*>(sO + 4 * K::O_WARP);  // [2]
  uint64_t* q_empty = q_full + 2;                      // [2]
  uint64_t* kv_full = q_empty + 2;                     // [ST]
  uint64_t* kv_empty = kv_full + K::STAGES;            // [ST]
  uint64_t* s_full = kv_empty + K::STAGES;             // [2] S_g landed
  uint64_t* s_free = s_full + 2;                       // [2] S_g loaded by every softmax warp
  uint64_t* p_full = s_free + 2;                       // [2] P_g stored (O rescaled)
  uint64_t* pv_done = p_full + 2;                      // [2] PV_g retired
  uint64_t* o_full = pv_done + 2;                      // a tile's O complete
  uint32_t* tslot = reinterpret_cast<uint32_t*>(o_full + 1);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int H = hs.H, BH = B * H;
  const int nqt = (S + K::BM - 1) / K::BM;
  const int items = BH * nqt;
  const int G = gridDim.x;
  // k-th tile of this CTA, snake order over the longest-first list
  auto tile_of = [&](int k) {
    const int r = k / 2, base = 2 * G * r;
    return (k & 1) ? base + 2 * G - 1 - static_cast<int>(blockIdx.x) : base + static_cast<int>(blockIdx.x);
  };
  auto decode = [&](int w, int& b, int& h, int& q0, int& nkb) {
    const int qt = nqt - 1 - w / BH;
    const int bh = w % BH;
    b = bh / H;
    h = bh % H;
    q0 = qt * K::BM;
    nkb = (min(S, q0 + K::BM) + K::BN - 1) / K::BN;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    tma_prefetch_desc(&to);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_full, 1);
    for (int s = 0; s < K::STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tP = tmem + 128, tO = tmem + 192;
#ifdef PP200_FA_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) {
    fa_trace_cta[blockIdx.x * 3] = fa_gtime();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    fa_trace_cta[blockIdx.x * 3 + 2] = smid;
  }
#endif

  if (warp == 0) {
    uint32_t g = 0;
    for (int k = 0;; ++k) {
      const int w = tile_of(k);
      if (w >= items) break;
      int b, h, q0, nkb;
      decode(w, b, h, q0, nkb);
      const int hk = h / hs.G, brow = b * S;
      const int qb = k & 1;
      mbar_wait(&q_empty[qb], ((k >> 1) & 1) ^ 1);
      if (elect_one()) {
        mbar_expect_tx(&q_full[qb], K::Q_BYTES);
        for (int hf = 0; hf < 2; ++hf)
          tma_load_2d(sQ + qb * K::Q_BYTES + hf * (K::Q_BYTES / 2), &tm, &q_full[qb], hs.qcol(h),
                      brow + q0 + 64 * hf);
      }
      __syncwarp();
      for (int j = 0; j < nkb; ++j, ++g) {
        const int st = g % K::STAGES;
        mbar_wait(&kv_empty[st], ((g / K::STAGES) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&kv_full[st], 2 * K::KV_BYTES);
          tma_load_2d(sK + st * K::KV_BYTES, &tm, &kv_full[st], hs.kcol(hk), brow + j * K::BN);
          tma_load_2d(sV + st * K::KV_BYTES, &tm, &kv_full[st], hs.vcol(hk), brow + j * K::BN);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t ID_S = umma_idesc_bf16(K::BM, K::BN, 0, 0);  // Q, K both K-major
    constexpr uint32_t ID_O = umma_idesc_bf16(K::BM, 64, 0, 1);     // P K-major, V MN-major
    // S_g = Q K_g^T for block g (tile k, block j) into S[g % 2]
    auto issue_s = [&](uint32_t g, int k, int j) {
      const int st = g % K::STAGES, qb = k & 1;
      if (j == 0) mbar_wait(&q_full[qb], (k >> 1) & 1);
      mbar_wait(&kv_full[st], (g / K::STAGES) & 1);
      if (g >= 2) mbar_wait(&s_free[g & 1], ((g - 2) >> 1) & 1);  // S_{g-2} loaded
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sQ + qb * K::Q_BYTES), k_addr = smem_u32(sK + st * K::KV_BYTES);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (ABL != 2)
            tc_mma_f16(tS + (g & 1) * 64, kmajor_step(q_addr, kk, K::Q_BYTES),
                       kmajor_step(k_addr, kk, K::KV_BYTES), ID_S, kk > 0 ? 1u : 0u);
        tc_commit(&s_full[g & 1]);
        FA_T(0, g);
      }
      __syncwarp();
    };
    // (tile, block) pairs in order; S is issued two pairs ahead, across tiles
    int kq[3], jq[3], nq[3];  // pairs g, g+1, g+2
    auto next_pair = [&](int k, int j, int nkb, int& k2, int& j2, int& n2) {
      k2 = k;
      j2 = j + 1;
      n2 = nkb;
      if (j2 == nkb) {
        k2 = k + 1;
        j2 = 0;
        const int w2 = tile_of(k2);
        if (w2 >= items) return false;
        int b2, h2, q02;
        decode(w2, b2, h2, q02, n2);
      }
      return true;
    };
    if (SPLIT) {
      uint32_t g = 0;
      for (int k = 0;; ++k) {
        const int w = tile_of(k);
        if (w >= items) break;
        int b, h, q0, nkb;
        decode(w, b, h, q0, nkb);
        for (int j = 0; j < nkb; ++j, ++g) issue_s(g, k, j);
        if (elect_one()) tc_commit(&q_empty[k & 1]);  // Q is read by the S MMAs only
        __syncwarp();
      }
    } else if (tile_of(0) < items) {
      int b0, h0, q00;
      kq[0] = 0;
      jq[0] = 0;
      decode(tile_of(0), b0, h0, q00, nq[0]);
      bool have1 = next_pair(kq[0], jq[0], nq[0], kq[1], jq[1], nq[1]);
      issue_s(0, kq[0], jq[0]);
      if (have1) issue_s(1, kq[1], jq[1]);
      bool have2 = have1 && next_pair(kq[1], jq[1], nq[1], kq[2], jq[2], nq[2]);
      for (uint32_t g = 0;; ++g) {
        if (have2) issue_s(g + 2, kq[2], jq[2]);  // once softmax g has loaded S_g
        const int k = kq[0], j = jq[0], nkb = nq[0];
        const int st = g % K::STAGES;
        mbar_wait(&p_full[g & 1], (g >> 1) & 1);
        if (lane == 0) FA_T(1, g);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + st * K::KV_BYTES);
        const uint32_t tPg = tP + (g & 1) * 32;  // key chunk c of 16 at column 8 c
        if (elect_one()) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (ABL != 2)
              tc_mma_f16_ts(tO, tPg + 8 * c, umma_sdesc_sw128(v_addr + c * 2048, K::KV_BYTES, 1024), ID_O,
                            (j > 0 || c > 0) ? 1u : 0u);
          tc_commit(&pv_done[g & 1]);
          tc_commit(&kv_empty[st]);
          FA_T(2, g);
          if (j == nkb - 1) {
            tc_commit(o_full);
            tc_commit(&q_empty[k & 1]);
          }
        }
        __syncwarp();
        if (!have1) break;
        kq[0] = kq[1]; jq[0] = jq[1]; nq[0] = nq[1];
        kq[1] = kq[2]; jq[1] = jq[2]; nq[1] = nq[2];
        have1 = have2;
        if (have2) have2 = next_pair(kq[1], jq[1], nq[1], kq[2], jq[2], nq[2]);
      }
    }
  } else if (SPLIT && warp == 3) {
    constexpr uint32_t ID_O = umma_idesc_bf16(K::BM, 64, 0, 1);  // P K-major, V MN-major
    uint32_t g = 0;
    for (int k = 0;; ++k) {
      const int w = tile_of(k);
      if (w >= items) break;
      int b, h, q0, nkb;
      decode(w, b, h, q0, nkb);
      for (int j = 0; j < nkb; ++j, ++g) {
        const int st = g % K::STAGES;
        mbar_wait(&p_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + st * K::KV_BYTES);
        const uint32_t tPg = tP + (g & 1) * 32;
        if (elect_one()) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (ABL != 2)
              tc_mma_f16_ts(tO, tPg + 8 * c, umma_sdesc_sw128(v_addr + c * 2048, K::KV_BYTES, 1024), ID_O,
                            (j > 0 || c > 0) ? 1u : 0u);
          tc_commit(&pv_done[g & 1]);
          // K_g was read by S_g, which retired before the softmax loaded it
          tc_commit(&kv_empty[st]);
          if (j == nkb - 1) tc_commit(o_full);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int qw = warp & 3;
    const int r = qw * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(qw * 32) << 16;
    uint8_t* so = sO + qw * K::O_WARP;
    const uint64_t sc2 = pack_f2(sl2, sl2);
    uint32_t g = 0;
    for (int k = 0;; ++k) {
      const int w = tile_of(k);
      if (w >= items) break;
      int b, h, q0, nkb;
      decode(w, b, h, q0, nkb);
      const int row = q0 + r;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nkb; ++j, ++g) {
        mbar_wait(&s_full[g & 1], (g >> 1) & 1);
        if (threadIdx.x == 128) FA_T(3, g);
        tc_fence_after();
        uint32_t sr[64];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld16(tS + (g & 1) * 64 + lane_off + c * 16, sr + c * 16);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[g & 1]);  // the MMA may overwrite S[g % 2]
        if (threadIdx.x == 128) FA_T(4, g);
        float* sv = reinterpret_cast<float*>(sr);
        const int n0 = j * K::BN;
        if (ABL == 1) {
          if (g >= 2) mbar_wait(&pv_done[g & 1], ((g - 2) >> 1) & 1);
          tc_fence_after();
          tmem_st16(tP + (g & 1) * 32 + lane_off, sr);
          tmem_st16(tP + (g & 1) * 32 + lane_off + 16, sr + 16);
          l = 1.f;
          m = 0.f;
          tc_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[g & 1]);
          continue;
        }
        if (n0 + K::BN - 1 > q0 || n0 + K::BN > S) {  // diagonal or ragged block
#pragma unroll
          for (int i = 0; i < K::BN; ++i)
            if (n0 + i > row || n0 + i >= S) sv[i] = -INFINITY;
        }
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
#pragma unroll
        for (int i = 0; i < K::BN; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], sv[i]);
        const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
        const float mn = fmaxf(m, mx);
        float corr = 1.f;
        if (j == 0 || m == -INFINITY) {
          m = mn == -INFINITY ? 0.f : mn;
          corr = 0.f;
        } else if (mn > m + 8.f) {  // lazy rescale (FA4), see fa_fwd_tc5
          corr = ex2(m - mn);
          m = mn;
        }
        const uint64_t nm2 = pack_f2(-m, -m);
        uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int i = 0; i < K::BN; i += 2) {
          float p0, p1;
          unpack_f2(ffma2(pack_f2(sv[i], sv[i + 1]), sc2, nm2), p0, p1);
          if ((i & 15) < EMU) {
            exp2_poly2(fmaxf(p0, -126.f), fmaxf(p1, -126.f), p0, p1);
          } else {
            p0 = ex2(p0);
            p1 = ex2(p1);
          }
          sv[i] = p0;
          sv[i + 1] = p1;
          acc2[(i >> 1) & 3] = fadd2(acc2[(i >> 1) & 3], pack_f2(p0, p1));
        }
        float sa[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) unpack_f2(acc2[i], sa[2 * i], sa[2 * i + 1]);
        l = l * corr + (((sa[0] + sa[1]) + (sa[2] + sa[3])) + ((sa[4] + sa[5]) + (sa[6] + sa[7])));
        uint32_t wv[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) pack_bf16x16(sv + 16 * c, wv + 8 * c);
        if (threadIdx.x == 128) FA_T(5, __float_as_uint(l) == 7u ? 40 : g);
        // P[g % 2] was last read by PV_{g-2}
        if (g >= 2) mbar_wait(&pv_done[g & 1], ((g - 2) >> 1) & 1);
        if (threadIdx.x == 128) FA_T(6, g);
        tc_fence_after();
        tmem_st16(tP + (g & 1) * 32 + lane_off, wv);
        tmem_st16(tP + (g & 1) * 32 + lane_off + 16, wv + 16);
        // rescale O by corr once PV_{g-1} (same tile) has retired
        if (j > 0 && __any_sync(0xffffffffu, corr != 1.f && l > 0.f)) {
          mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
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
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[g & 1]);
        if (threadIdx.x == 128) FA_T(7, g);
      }
      // epilogue: O / l -> bf16 rows in this warp's staging tile -> TMA store.
      // The next tile's first PV overwrites O only after this warp's next
      // p_full arrival, which follows the load below.
      mbar_wait(o_full, k & 1);
      tc_fence_after();
      uint32_t orr[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(tO + lane_off + c * 16, orr + c * 16);
      tc_wait_ld();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      if (lane == 0) bulk_wait_read0();  // the previous tile's store has left the staging tile
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 u;
        __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          hp[e] = __floats2bfloat162_rn(__uint_as_float(orr[8 * c + 2 * e]) * inv,
                                        __uint_as_float(orr[8 * c + 2 * e + 1]) * inv);
        *reinterpret_cast<uint4*>(so + lane * 128 + ((c ^ (lane & 7)) << 4)) = u;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(&to, so, hs.qcol(h), q0 + qw * 32, b);
        bulk_commit();
      }
      if (row < S) lse[(static_cast<int64_t>(b) * H + h) * S + row] = (m + log2f(l)) * F_LN2;
    }
    if (lane == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 256);
#ifdef PP200_FA_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) fa_trace_cta[blockIdx.x * 3 + 1] = fa_gtime();
#endif
}


// ------------------------------------------------------------------ backward
// NG elementwise warps per TMEM lane quarter.  With SETS = 2 (head_dim 128) they
// form two sets that take alternate score blocks (set = block % 2 = its score
// buffer), so one set's TMEM loads / stores and barrier round trips overlap the
// other set's math (measured: C4 / C5 backward 355 -> 306 / 670 -> 576 us); with
// SETS = 1 (head_dim 64) all of them work on every block and three score
// buffers let the MMA run further ahead (the two-set variant measured slower
// there, 98 -> 113 us at C2).  Each warp owns CW = 64 * SETS / NG score columns
// of its blocks; in the epilogues every warp owns HD / NG output columns.
constexpr int BW_NG = 4;
template <int HD>
struct BwSets {
  static constexpr int SETS = HD == 128 ? 2 : 1;
  static constexpr int CW = 64 * SETS / BW_NG;
};

// NC * 8 fp32 accumulator values -> bf16 (scaled) in global memory.
template <int NC>
__device__ __forceinline__ void store_row_chunks(bf16* dst, const uint32_t* acc, float scale) {
  uint4 u[NC];
  __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(u);
#pragma unroll
  for (int k = 0; k < 4 * NC; ++k)
    hp[k] = __floats2bfloat162_rn(__uint_as_float(acc[2 * k]) * scale, __uint_as_float(acc[2 * k + 1]) * scale);
#pragma unroll
  for (int k = 0; k < NC; ++k) reinterpret_cast<uint4*>(dst)[k] = u[k];
}

// CW fp32 columns of one TMEM lane into registers (CW a multiple of 16).
template <int CW>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
#pragma unroll
  for (int i = 0; i < CW / 16; ++i) tmem_ld16(taddr + 16 * i, r + 16 * i);
}

// dK, dV for 128-key tiles of one (batch, kv head), persistent: one CTA per SM
// walks the tiles longest-first (tile w: key tile w / (B Hkv), kv head w % (B Hkv)).
// A tile's blocks are the 64-query blocks at or after its keys of every query
// head of the kv head's group, so dK / dV accumulate the group sum in TMEM.
// 4 + 16 warps:
//   warp 0      TMA producer: K, V of a tile into one of KVBUF buffers; per
//               block Q, dO (tensor maps) and its lse / delta rows (bulk
//               copies) into a STAGES-deep ring
//   warp 1      MMA issuer, up to SBUF query blocks ahead of the elementwise
//               warps: S^T_i = K Q_i^T, dP^T_i = V dO_i^T -> TMEM buffer i % SBUF;
//               dV += P^T_i dO_i, dK += dS^T_i Q_i -> TMEM accumulators
//   warp 2      TMEM allocator (512 columns: S^T/dP^T x SBUF, dV, dK)
//   warps 4..   elementwise: BW_NG warps per TMEM lane quarter (one key row
//               per thread, 64 / BW_NG queries each) build P^T = exp2(S^T*c - lse)
//               and dS^T = P^T (dP^T - delta) as packed bf16 written back into
//               TMEM over the scores they came from: the dV / dK MMAs read their
//               A operand straight from TMEM (query chunk k of 16 at column 16 k)
// Ring / buffer phases run on tile-global block counters; a score buffer is
// reused once the dV / dK MMAs that read its P^T / dS^T have retired.
template <int HD>
struct BwdKV {
  static constexpr int KEYS = 128, BQ = 64;
  static constexpr int NP = HD / 64;
  static constexpr int SETS = BwSets<HD>::SETS;
  static constexpr int SBUF = SETS == 2 ? 2 : 3;  // two sets: one score buffer each
  static constexpr int STAGES = HD == 64 ? 5 : 4;
  static constexpr int KVBUF = HD == 64 ? 2 : 1;
  static constexpr int KV_PANEL = KEYS * 64 * 2;   // 16 KB
  static constexpr int KV_BYTES = NP * KV_PANEL;   // one of K / V
  static constexpr int Q_PANEL = BQ * 64 * 2;      // 8 KB
  static constexpr int Q_BYTES = NP * Q_PANEL;     // one of Q / dO per stage
  static constexpr int EW = 4 * BW_NG, THREADS = 128 + 32 * EW;
  static constexpr int SMEM = KVBUF * 2 * KV_BYTES + STAGES * 2 * Q_BYTES + STAGES * 512 + 1024 + 256;
};

template <int HD>
__global__ void __launch_bounds__(BwdKV<HD>::THREADS, 1)
    fa_bwd_dkdv_tc5(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tg,
                    const float* __restrict__ lse, const float* __restrict__ delta,
                    bf16* __restrict__ dqkv, int64_t ldd, int B, Heads hs, int S, float sl2,
                    float scale) {
  using K = BwdKV<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sK = smem;                            // [KVBUF][NP][128 keys x 64]
  uint8_t* sV = sK + K::KVBUF * K::KV_BYTES;     // [KVBUF][NP][128 keys x 64]
  uint8_t* sQ = sV + K::KVBUF * K::KV_BYTES;     // [ST][NP][64 x 64]
  uint8_t* sG = sQ + K::STAGES * K::Q_BYTES;     // dO [ST][NP][64 x 64]
  float* sLD = reinterpret_cast<float*>(sG + K::STAGES * K::Q_BYTES);  // [ST][lse 64 | delta 64]
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(sLD + K::STAGES * 128);  // [KVBUF]
  uint64_t* kv_empty = kv_full + K::KVBUF;      // [KVBUF]
  uint64_t* q_full = kv_empty + K::KVBUF;
  uint64_t* q_empty = q_full + K::STAGES;
  uint64_t* s_full = q_empty + K::STAGES;       // [SBUF] scores landed
  uint64_t* p_full = s_full + K::SBUF;          // [SBUF] P^T / dS^T packed in TMEM
  uint64_t* pv_done = p_full + K::SBUF;         // [SBUF] dV / dK MMAs of the buffer retired
  uint64_t* done = pv_done + K::SBUF;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int H = hs.H, G = hs.G;
  const int nkt = (S + K::KEYS - 1) / K::KEYS, nqb = (S + K::BQ - 1) / K::BQ;
  const int BHk = B * hs.Hkv;
  const int items = BHk * nkt;
  // k-th item of this CTA: snake order over the longest-first list (a plain
  // stride left the first CTAs ~15 % more key blocks than the last)
  auto snake_item = [&](int k) {
    const int r = k >> 1, G2 = 2 * static_cast<int>(gridDim.x);
    return (k & 1) ? G2 * r + G2 - 1 - static_cast<int>(blockIdx.x) : G2 * r + static_cast<int>(blockIdx.x);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tg);
    for (int i = 0; i < K::KVBUF; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < K::STAGES; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < K::SBUF; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], K::EW / K::SETS);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // S^T of block i at tmem + 128 (i % SBUF), dP^T at + 64; then dV, dK
  const uint32_t tdV = tmem + 128 * K::SBUF, tdK = tdV + HD;

  // tile w -> (batch, kv head, first key, first query block, query blocks per head)
  auto decode = [&](int w, int& b, int& hk, int& k0, int& qbeg, int& nq) {
    const int kt = w / BHk;  // early key tiles see the most query blocks: first
    const int bhk = w % BHk;
    b = bhk / hs.Hkv;
    hk = bhk % hs.Hkv;
    k0 = kt * K::KEYS;
    qbeg = k0 / K::BQ;
    nq = nqb - qbeg;
  };

  if (warp == 0) {
    // warp-uniform loop, one elected lane issuing (see fa_fwd64_tc5)
    uint32_t g = 0, ic = 0;
    for (int w = snake_item(0); w < items; w = snake_item(++ic)) {
      int b, hk, k0, qbeg, nq;
      decode(w, b, hk, k0, qbeg, nq);
      const int brow = b * S;
      const int kb = ic % K::KVBUF;
      mbar_wait(&kv_empty[kb], ((ic / K::KVBUF) & 1) ^ 1);
      if (elect_one()) {
        mbar_expect_tx(&kv_full[kb], 2 * K::KV_BYTES);
        for (int p = 0; p < K::NP; ++p)
          for (int hf = 0; hf < 2; ++hf) {
            const int off = kb * K::KV_BYTES + p * K::KV_PANEL + hf * (K::KV_PANEL / 2);
            tma_load_2d(sK + off, &tq, &kv_full[kb], hs.kcol(hk) + 64 * p, brow + k0 + hf * 64);
            tma_load_2d(sV + off, &tq, &kv_full[kb], hs.vcol(hk) + 64 * p, brow + k0 + hf * 64);
          }
      }
      __syncwarp();
      for (int i = 0; i < G * nq; ++i, ++g) {
        const int h = hk * G + i / nq;
        const int st = g % K::STAGES;
        const int m0 = (qbeg + i % nq) * K::BQ;
        const int64_t vbase = (static_cast<int64_t>(b) * H + h) * S;
        const uint32_t lbytes = static_cast<uint32_t>(min(K::BQ, S - m0)) * 4;  // S % 4 == 0
        mbar_wait(&q_empty[st], ((g / K::STAGES) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&q_full[st], 2 * K::Q_BYTES + 2 * lbytes);
          for (int p = 0; p < K::NP; ++p) {
            tma_load_2d(sQ + st * K::Q_BYTES + p * K::Q_PANEL, &tq, &q_full[st], hs.qcol(h) + 64 * p, brow + m0);
            tma_load_2d(sG + st * K::Q_BYTES + p * K::Q_PANEL, &tg, &q_full[st], hs.qcol(h) + 64 * p, brow + m0);
          }
          bulk_load(sLD + st * 128, lse + vbase + m0, lbytes, &q_full[st]);
          bulk_load(sLD + st * 128 + 64, delta + vbase + m0, lbytes, &q_full[st]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t ID_T = umma_idesc_bf16(128, K::BQ, 0, 0);  // K/V x (Q/dO)^T, N = 64 queries
    constexpr uint32_t ID_A = umma_idesc_bf16(128, HD, 0, 1);     // P^T/dS^T x (dO/Q), N = HD dims
    const uint64_t qn = umma_sdesc_sw128(smem_u32(sQ), K::Q_PANEL, 1024);  // MN-major views
    const uint64_t gn = umma_sdesc_sw128(smem_u32(sG), K::Q_PANEL, 1024);
    uint32_t g0 = 0, ic = 0;
    for (int w = snake_item(0); w < items; w = snake_item(++ic)) {
      int b, hk, k0, qbeg, nq;
      decode(w, b, hk, k0, qbeg, nq);
      const int n = G * nq;
      const int kb = ic % K::KVBUF;
      mbar_wait(&kv_full[kb], (ic / K::KVBUF) & 1);
      tc_fence_after();
      const uint32_t ka = smem_u32(sK + kb * K::KV_BYTES), va = smem_u32(sV + kb * K::KV_BYTES);
      auto issue_s = [&](uint32_t g) {
        const int st = g % K::STAGES, sb = g % K::SBUF;
        mbar_wait(&q_full[st], (g / K::STAGES) & 1);
        // the buffer's previous P^T / dS^T have been read by their MMAs
        if (g >= K::SBUF) mbar_wait(&pv_done[sb], ((g - K::SBUF) / K::SBUF) & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(sQ + st * K::Q_BYTES), ga = smem_u32(sG + st * K::Q_BYTES);
        const uint32_t tS = tmem + sb * 128;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            tc_mma_f16(tS, kmajor_step(ka, k, K::KV_PANEL), kmajor_step(qa, k, K::Q_PANEL), ID_T,
                       k > 0 ? 1u : 0u);
            tc_mma_f16(tS + 64, kmajor_step(va, k, K::KV_PANEL), kmajor_step(ga, k, K::Q_PANEL), ID_T,
                       k > 0 ? 1u : 0u);
          }
          tc_commit(&s_full[sb]);
        }
        __syncwarp();
      };
      for (int i = 0; i < K::SBUF && i < n; ++i) issue_s(g0 + i);
      for (int i = 0; i < n; ++i) {
        const uint32_t g = g0 + i;
        const int st = g % K::STAGES, sb = g % K::SBUF;
        mbar_wait(&p_full[sb], (g / K::SBUF) & 1);
        tc_fence_after();
        const uint64_t so = static_cast<uint64_t>(st * (K::Q_BYTES >> 4));
        const uint32_t tP = tmem + sb * 128;  // P^T chunk k at column 16 k, dS^T at + 64
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < K::BQ / 16; ++k) {
            const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
            tc_mma_f16_ts(tdV, tP + 16 * k, gn + so + 128 * k, ID_A, acc);
            tc_mma_f16_ts(tdK, tP + 64 + 16 * k, qn + so + 128 * k, ID_A, acc);
          }
          tc_commit(&pv_done[sb]);
          tc_commit(&q_empty[st]);
        }
        __syncwarp();
        if (i + K::SBUF < n) issue_s(g + K::SBUF);  // into the buffer block i released
      }
      if (elect_one()) {
        tc_commit(&kv_empty[kb]);  // K / V of this tile no longer read
        tc_commit(done);           // dV / dK of this tile complete
      }
      __syncwarp();
      g0 += n;
    }
  } else if (warp >= 4) {
    constexpr int CW = BwSets<HD>::CW, CO = HD / BW_NG;
    const int qw = warp & 3;                 // TMEM lane quarter
    const int grp = (warp - 4) >> 2;         // warp group: output columns in the epilogue
    const int set = grp / (BW_NG / K::SETS); // two sets: blocks g with g % 2 == set
    const int cb = (grp % (BW_NG / K::SETS)) * CW;  // first of this warp's CW queries
    const int r = qw * 32 + lane;            // key row in the tile
    const uint32_t lo = static_cast<uint32_t>(qw * 32) << 16;
    const uint64_t sc2 = pack_f2(sl2, sl2);
    uint32_t g0 = 0, ic = 0;
    for (int w = snake_item(0); w < items; w = snake_item(++ic)) {
      int b, hk, k0, qbeg, nq;
      decode(w, b, hk, k0, qbeg, nq);
      const int brow = b * S;
      const int key = k0 + r;
      const int n = G * nq;
      for (int i = 0; i < n; ++i) {
        const uint32_t g = g0 + i;
        const int st = g % K::STAGES, sb = g % K::SBUF;
        if (K::SETS == 2 && sb != set) continue;  // the other set's block
        const int m0 = (qbeg + i % nq) * K::BQ;
        mbar_wait(&s_full[sb], (g / K::SBUF) & 1);
        tc_fence_after();
        uint32_t sr[CW], pr[CW];
        const uint32_t tS = tmem + sb * 128 + lo + cb;
        tmem_ld_cols<CW>(tS, sr);
        tmem_ld_cols<CW>(tS + 64, pr);
        tc_wait_ld();
        mbar_wait(&q_full[st], (g / K::STAGES) & 1);  // lse / delta rows visible
        const float* Ls = sLD + st * 128 + cb;
        const float* Ds = Ls + 64;
        // P^T into sr, dS^T into pr (in place: registers)
        float* pv = reinterpret_cast<float*>(sr);
        float* dv = reinterpret_cast<float*>(pr);
#pragma unroll
        for (int gi = 0; gi < CW / 4; ++gi) {
          const float4 l4 = reinterpret_cast<const float4*>(Ls)[gi];
          const float4 d4 = reinterpret_cast<const float4*>(Ds)[gi];
          const uint64_t nl01 = pack_f2(-l4.x * F_LOG2E, -l4.y * F_LOG2E);
          const uint64_t nl23 = pack_f2(-l4.z * F_LOG2E, -l4.w * F_LOG2E);
          float a0, a1, a2, a3;
          unpack_f2(ffma2(pack_f2(__uint_as_float(sr[4 * gi]), __uint_as_float(sr[4 * gi + 1])), sc2, nl01), a0, a1);
          unpack_f2(ffma2(pack_f2(__uint_as_float(sr[4 * gi + 2]), __uint_as_float(sr[4 * gi + 3])), sc2, nl23), a2, a3);
          const float p0 = ex2(a0), p1 = ex2(a1), p2 = ex2(a2), p3 = ex2(a3);
          float e0, e1, e2, e3;
          unpack_f2(fadd2(pack_f2(__uint_as_float(pr[4 * gi]), __uint_as_float(pr[4 * gi + 1])),
                          pack_f2(-d4.x, -d4.y)), e0, e1);
          unpack_f2(fadd2(pack_f2(__uint_as_float(pr[4 * gi + 2]), __uint_as_float(pr[4 * gi + 3])),
                          pack_f2(-d4.z, -d4.w)), e2, e3);
          float f0, f1, f2, f3;
          unpack_f2(fmul2(pack_f2(p0, p1), pack_f2(e0, e1)), f0, f1);
          unpack_f2(fmul2(pack_f2(p2, p3), pack_f2(e2, e3)), f2, f3);
          pv[4 * gi] = p0; pv[4 * gi + 1] = p1; pv[4 * gi + 2] = p2; pv[4 * gi + 3] = p3;
          dv[4 * gi] = f0; dv[4 * gi + 1] = f1; dv[4 * gi + 2] = f2; dv[4 * gi + 3] = f3;
        }
        // causal / ragged mask: only blocks reaching below the diagonal or past S
        if (m0 + cb < key || m0 + cb + CW > S) {
#pragma unroll
          for (int e = 0; e < CW; ++e) {
            const int q = m0 + cb + e;
            if (q < key || q >= S) {
              pv[e] = 0.f;
              dv[e] = 0.f;
            }
          }
        }
        // packed bf16 back over this group's own score columns (MMA A operands):
        // query chunk k of 16 at column 16 k
        static_assert(CW % 16 == 0, "TMEM-resident P^T: whole 16-query chunks per warp");
#pragma unroll
        for (int c = 0; c < CW / 16; ++c) {
          uint32_t wv[8];
          pack_bf16x16(pv + 16 * c, wv);
          tmem_st8(tS + 16 * c, wv);
          pack_bf16x16(dv + 16 * c, wv);
          tmem_st8(tS + 64 + 16 * c, wv);
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
      }
      mbar_wait(done, ic & 1);
      tc_fence_after();
      uint32_t acc[CO];
      const int64_t rowoff = static_cast<int64_t>(brow + key) * ldd + grp * CO;
      tmem_ld_cols<CO>(tdV + lo + grp * CO, acc);
      tc_wait_ld();
      if (key < S) store_row_chunks<CO / 8>(dqkv + rowoff + hs.vcol(hk), acc, 1.f);
      tmem_ld_cols<CO>(tdK + lo + grp * CO, acc);
      tc_wait_ld();
      if (key < S) store_row_chunks<CO / 8>(dqkv + rowoff + hs.kcol(hk), acc, scale);
      g0 += n;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int HD>
struct BwdQ {
  static constexpr int BM = 128, BN = 64;
  static constexpr int NP = HD / 64;
  static constexpr int SETS = BwSets<HD>::SETS;
  static constexpr int SBUF = SETS == 2 ? 2 : 3;  // two sets: one score buffer each
  static constexpr int STAGES = HD == 64 ? 5 : 3;
  static constexpr int QBUF = HD == 64 ? 2 : 1;
  static constexpr int Q_PANEL = BM * 64 * 2;     // 16 KB
  static constexpr int Q_BYTES = NP * Q_PANEL;    // one of Q / dO / O
  static constexpr int KV_PANEL = BN * 64 * 2;    // 8 KB
  static constexpr int KV_BYTES = NP * KV_PANEL;  // one of K / V per stage
  static constexpr int EW = 4 * BW_NG, THREADS = 128 + 32 * EW;
  static constexpr int SMEM = QBUF * 3 * Q_BYTES + STAGES * 2 * KV_BYTES + 128 * BW_NG * 4 + 1024 + 256;
};

// 16 B chunk j (8 bf16, j < HD / 8) of row r in a [128 x HD] tile stored as
// 64-column panels, each loaded as two 128B-swizzled 64-row TMA boxes.
__device__ __forceinline__ uint4 ld_chunk128(const uint8_t* tile, int r, int j) {
  return *reinterpret_cast<const uint4*>(tile + (j >> 3) * 16384 + (r >> 6) * 8192 + (r & 63) * 128 +
                                         (((j & 7) ^ (r & 7)) << 4));
}

// dQ for 128-query tiles of one (batch, head), persistent: one CTA per SM
// walks the tiles longest-first (tile w: query tile nqt-1 - w/BH, head w%BH).
// Also produces delta = rowsum(dO o O) for its rows (consumed by the dK/dV
// kernel that runs next).  4 + 16 warps:
//   warp 0      TMA producer: Q, dO, O of a tile into one of QBUF buffers,
//               K/V blocks of 64 keys (the head's kv head) through a ring
//   warp 1      MMA issuer, up to three key blocks ahead of the elementwise
//               warps: S_j = Q K_j^T, dP_j = dO V_j^T -> TMEM buffer j % 3,
//               dQ += dS_j K_j -> TMEM accumulator
//   warp 2      TMEM allocator (512 columns)
//   warps 4..   elementwise: BW_NG warps per TMEM lane quarter (one query
//               row per thread, 64 / BW_NG keys each) build
//               dS = exp2(S*c - lse) (dP - delta) as packed bf16 written back
//               over their own score columns: the dQ MMA reads A from TMEM
// Ring / buffer phases run on tile-global block counters, so a tile's first
// blocks reuse buffers the previous tile released.
template <int HD, int SPLIT = 0>  // SPLIT: dQ MMAs from warp 3, S / dP from warp 1
__global__ void __launch_bounds__(BwdQ<HD>::THREADS, 1)
    fa_bwd_dq_tc5(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tg,
                  const __grid_constant__ CUtensorMap to, const float* __restrict__ lse,
                  float* __restrict__ delta, bf16* __restrict__ dqkv, int64_t ldd, int BH, Heads hs,
                  int S, float sl2, float scale) {
  using K = BwdQ<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                              // [QBUF][NP][128 x 64]
  uint8_t* sG = sQ + K::QBUF * K::Q_BYTES;         // dO
  uint8_t* sO = sG + K::QBUF * K::Q_BYTES;         // O
  uint8_t* sK = sO + K::QBUF * K::Q_BYTES;         // [ST][NP][64 x 64]
  uint8_t* sV = sK + K::STAGES * K::KV_BYTES;      // [ST][NP][64 x 64]
  float* sDelta = reinterpret_cast<float*>(sV + K::STAGES * K::KV_BYTES);  // [BW_NG][128] row partials
  uint64_t* q_full = reinterpret_cast<uint64_t*>(sDelta + 128 * BW_NG);  // [QBUF]
  uint64_t* q_empty = q_full + K::QBUF;         // [QBUF]
  uint64_t* kv_full = q_empty + K::QBUF;
  uint64_t* kv_empty = kv_full + K::STAGES;
  uint64_t* s_full = kv_empty + K::STAGES;  // [SBUF] scores landed
  uint64_t* p_full = s_full + K::SBUF;      // [SBUF] dS packed in TMEM
  uint64_t* pv_done = p_full + K::SBUF;     // [SBUF] dQ MMAs of the buffer retired
  uint64_t* done = pv_done + K::SBUF;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int H = hs.H;
  const int nqt = (S + K::BM - 1) / K::BM;
  const int items = BH * nqt;
  auto snake_item = [&](int k) {  // see fa_bwd_dkdv_tc5
    const int r = k >> 1, G2 = 2 * static_cast<int>(gridDim.x);
    return (k & 1) ? G2 * r + G2 - 1 - static_cast<int>(blockIdx.x) : G2 * r + static_cast<int>(blockIdx.x);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tg);
    tma_prefetch_desc(&to);
    for (int i = 0; i < K::QBUF; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1 + K::EW);  // MMA warp (Q, dO) + elementwise warps (O, dO)
    }
    for (int i = 0; i < K::STAGES; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < K::SBUF; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], K::EW / K::SETS);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tdQ = tmem + 128 * K::SBUF;  // S_j at tmem + 128 (j % SBUF), dP_j at + 64

  // tile w -> (batch*head, first query row, key blocks)
  auto decode = [&](int w, int& bh, int& q0, int& nkb) {
    const int qt = nqt - 1 - w / BH;
    bh = w % BH;
    q0 = qt * K::BM;
    nkb = (min(S, q0 + K::BM) + K::BN - 1) / K::BN;
  };

  if (warp == 0) {
    // warp-uniform loop, one elected lane issuing (see fa_fwd64_tc5)
    uint32_t g = 0, ic = 0;
    for (int w = snake_item(0); w < items; w = snake_item(++ic)) {
      int bh, q0, nkb;
      decode(w, bh, q0, nkb);
      const int b = bh / H, h = bh % H, hk = h / hs.G, brow = b * S;
      const int qb = ic % K::QBUF;
      mbar_wait(&q_empty[qb], ((ic / K::QBUF) & 1) ^ 1);
      if (elect_one()) {
        mbar_expect_tx(&q_full[qb], 3 * K::Q_BYTES);
        for (int p = 0; p < K::NP; ++p)
          for (int hf = 0; hf < 2; ++hf) {
            const int off = qb * K::Q_BYTES + p * K::Q_PANEL + hf * (K::Q_PANEL / 2);
            const int x = hs.qcol(h) + 64 * p, y = brow + q0 + hf * 64;
            tma_load_2d(sQ + off, &tq, &q_full[qb], x, y);
            tma_load_2d(sG + off, &tg, &q_full[qb], x, y);
            tma_load_2d(sO + off, &to, &q_full[qb], x, y);
          }
      }
      __syncwarp();
      for (int j = 0; j < nkb; ++j, ++g) {
        const int st = g % K::STAGES;
        mbar_wait(&kv_empty[st], ((g / K::STAGES) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&kv_full[st], 2 * K::KV_BYTES);
          for (int p = 0; p < K::NP; ++p) {
            tma_load_2d(sK + st * K::KV_BYTES + p * K::KV_PANEL, &tq, &kv_full[st],
                        hs.kcol(hk) + 64 * p, brow + j * K::BN);
            tma_load_2d(sV + st * K::KV_BYTES + p * K::KV_PANEL, &tq, &kv_full[st],
                        hs.vcol(hk) + 64 * p, brow + j * K::BN);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t ID_T = umma_idesc_bf16(128, K::BN, 0, 0);  // Q/dO x (K/V)^T
    constexpr uint32_t ID_A = umma_idesc_bf16(128, HD, 0, 1);     // dS x K (MN-major)
    const uint64_t kn = umma_sdesc_sw128(smem_u32(sK), K::KV_PANEL, 1024);   // MN-major view
    uint32_t g0 = 0, ic = 0;
    for (int w = snake_item(0); w < items; w = snake_item(++ic)) {
      int bh, q0, nkb;
      decode(w, bh, q0, nkb);
      const int qb = ic % K::QBUF;
      mbar_wait(&q_full[qb], (ic / K::QBUF) & 1);
      tc_fence_after();
      const uint32_t qa = smem_u32(sQ + qb * K::Q_BYTES), ga = smem_u32(sG + qb * K::Q_BYTES);
      auto issue_s = [&](uint32_t g) {
        const int st = g % K::STAGES, sb = g % K::SBUF;
        mbar_wait(&kv_full[st], (g / K::STAGES) & 1);
        // the buffer's previous dS has been read by its dQ MMAs
        if (g >= K::SBUF) mbar_wait(&pv_done[sb], ((g - K::SBUF) / K::SBUF) & 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(sK + st * K::KV_BYTES), va = smem_u32(sV + st * K::KV_BYTES);
        const uint32_t tS = tmem + sb * 128;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            tc_mma_f16(tS, kmajor_step(qa, k, K::Q_PANEL), kmajor_step(ka, k, K::KV_PANEL), ID_T,
                       k > 0 ? 1u : 0u);
            tc_mma_f16(tS + 64, kmajor_step(ga, k, K::Q_PANEL), kmajor_step(va, k, K::KV_PANEL), ID_T,
                       k > 0 ? 1u : 0u);
          }
          tc_commit(&s_full[sb]);
        }
        __syncwarp();
      };
      if (SPLIT) {
        for (int j = 0; j < nkb; ++j) issue_s(g0 + j);
        if (elect_one()) tc_commit(&q_empty[qb]);  // Q / dO of this tile no longer read by MMAs
        __syncwarp();
        g0 += nkb;
        continue;
      }
      for (int j = 0; j < K::SBUF && j < nkb; ++j) issue_s(g0 + j);
      for (int j = 0; j < nkb; ++j) {
        const uint32_t g = g0 + j;
        const int st = g % K::STAGES, sb = g % K::SBUF;
        mbar_wait(&p_full[sb], (g / K::SBUF) & 1);
        tc_fence_after();
        const uint64_t so = static_cast<uint64_t>(st * (K::KV_BYTES >> 4));
        const uint32_t tD = tmem + sb * 128;  // dS key chunk k at column 16 k
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < K::BN / 16; ++k)
            tc_mma_f16_ts(tdQ, tD + 16 * k, kn + so + 128 * k, ID_A, (j > 0 || k > 0) ? 1u : 0u);
          tc_commit(&pv_done[sb]);
          tc_commit(&kv_empty[st]);
        }
        __syncwarp();
        if (j + K::SBUF < nkb) issue_s(g + K::SBUF);  // into the buffer block j released
      }
      if (elect_one()) {
        tc_commit(&q_empty[qb]);  // Q / dO of this tile no longer read by MMAs
        tc_commit(done);          // dQ of this tile complete
      }
      __syncwarp();
      g0 += nkb;
    }
  } else if (SPLIT && warp == 3) {
    constexpr uint32_t ID_A = umma_idesc_bf16(128, HD, 0, 1);     // dS x K (MN-major)
    const uint64_t kn = umma_sdesc_sw128(smem_u32(sK), K::KV_PANEL, 1024);   // MN-major view
    uint32_t g0 = 0, ic = 0;
    for (int w = snake_item(0); w < items; w = snake_item(++ic)) {
      int bh, q0, nkb;
      decode(w, bh, q0, nkb);
      for (int j = 0; j < nkb; ++j) {
        const uint32_t g = g0 + j;
        const int st = g % K::STAGES, sb = g % K::SBUF;
        mbar_wait(&p_full[sb], (g / K::SBUF) & 1);
        tc_fence_after();
        const uint64_t so = static_cast<uint64_t>(st * (K::KV_BYTES >> 4));
        const uint32_t tD = tmem + sb * 128;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < K::BN / 16; ++k)
            tc_mma_f16_ts(tdQ, tD + 16 * k, kn + so + 128 * k, ID_A, (j > 0 || k > 0) ? 1u : 0u);
          tc_commit(&pv_done[sb]);
          tc_commit(&kv_empty[st]);  // K_j / V_j: the S / dP MMAs retired before p_full
        }
        __syncwarp();
      }
      if (elect_one()) tc_commit(done);  // dQ of this tile complete
      __syncwarp();
      g0 += nkb;
    }
  } else if (warp >= 4) {
    constexpr int CW = BwSets<HD>::CW, CO = HD / BW_NG;
    const int qw = warp & 3;               // TMEM lane quarter
    const int grp = (warp - 4) >> 2;       // warp group: delta / output columns
    const int set = grp / (BW_NG / K::SETS);        // two sets: key blocks with g % 2 == set
    const int cb = (grp % (BW_NG / K::SETS)) * CW;  // first of this warp's CW keys
    const int r = qw * 32 + lane;          // query row in the tile
    const uint32_t lo = static_cast<uint32_t>(qw * 32) << 16;
    const uint64_t sc2 = pack_f2(sl2, sl2);
    uint32_t g0 = 0, ic = 0;
    for (int w = snake_item(0); w < items; w = snake_item(++ic)) {
      int bh, q0, nkb;
      decode(w, bh, q0, nkb);
      const int b = bh / H, h = bh % H, brow = b * S;
      const int row = q0 + r;
      const int64_t vrow = static_cast<int64_t>(bh) * S + row;
      const int qb = ic % K::QBUF;
      // delta = rowsum(dO o O): each column group sums CO head dims, fixed-order combine
      mbar_wait(&q_full[qb], (ic / K::QBUF) & 1);
      float part = 0.f;
#pragma unroll
      for (int jj = 0; jj < CO / 8; ++jj) {
        const uint4 ov = ld_chunk128(sO + qb * K::Q_BYTES, r, grp * (CO / 8) + jj);
        const uint4 gv = ld_chunk128(sG + qb * K::Q_BYTES, r, grp * (CO / 8) + jj);
        const __nv_bfloat162* oh = reinterpret_cast<const __nv_bfloat162*>(&ov);
        const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&gv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 of = __bfloat1622float2(oh[k]), gf = __bfloat1622float2(gh[k]);
          part = fmaf(of.x, gf.x, part);
          part = fmaf(of.y, gf.y, part);
        }
      }
      sDelta[grp * 128 + r] = part;
      asm volatile("bar.sync 1, %0;" ::"n"(K::EW * 32) : "memory");  // elementwise warps only
      float dl = 0.f;
#pragma unroll
      for (int gi = 0; gi < BW_NG; ++gi) dl += sDelta[gi * 128 + r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_empty[qb]);  // O / dO no longer read here
      if (grp == 0 && row < S) delta[vrow] = dl;
      const float nl2 = row < S ? -lse[vrow] * F_LOG2E : 0.f;
      const uint64_t nl22 = pack_f2(nl2, nl2), nd2 = pack_f2(-dl, -dl);
      for (int j = 0; j < nkb; ++j) {
        const uint32_t g = g0 + j;
        const int sb = g % K::SBUF;
        if (K::SETS == 2 && sb != set) continue;  // the other set's block
        const int n0 = j * K::BN;
        mbar_wait(&s_full[sb], (g / K::SBUF) & 1);
        tc_fence_after();
        uint32_t sr[CW], pr[CW];
        const uint32_t tS = tmem + sb * 128 + lo + cb;
        tmem_ld_cols<CW>(tS, sr);
        tmem_ld_cols<CW>(tS + 64, pr);
        tc_wait_ld();
        float* dv = reinterpret_cast<float*>(sr);  // dS in place
#pragma unroll
        for (int e = 0; e < CW; e += 2) {
          float a0, a1, e0, e1, f0, f1;
          unpack_f2(ffma2(pack_f2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])), sc2, nl22), a0, a1);
          const float p0 = ex2(a0), p1 = ex2(a1);
          unpack_f2(fadd2(pack_f2(__uint_as_float(pr[e]), __uint_as_float(pr[e + 1])), nd2), e0, e1);
          unpack_f2(fmul2(pack_f2(p0, p1), pack_f2(e0, e1)), f0, f1);
          dv[e] = f0;
          dv[e + 1] = f1;
        }
        // causal / ragged mask: only blocks crossing the diagonal or the sequence end
        if (n0 + cb + CW - 1 > row || n0 + cb + CW > S || row >= S) {
#pragma unroll
          for (int e = 0; e < CW; ++e) {
            const int key = n0 + cb + e;
            if (key > row || key >= S || row >= S) dv[e] = 0.f;
          }
        }
        // packed bf16 dS back over this group's own score columns (MMA A operand):
        // key chunk k of 16 at column 16 k
        static_assert(CW % 16 == 0, "TMEM-resident dS: whole 16-key chunks per warp");
#pragma unroll
        for (int c = 0; c < CW / 16; ++c) {
          uint32_t wv[8];
          pack_bf16x16(dv + 16 * c, wv);
          tmem_st8(tS + 16 * c, wv);
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
      }
      mbar_wait(done, ic & 1);
      tc_fence_after();
      uint32_t acc[CO];
      tmem_ld_cols<CO>(tdQ + lo + grp * CO, acc);
      tc_wait_ld();
      if (row < S)
        store_row_chunks<CO / 8>(dqkv + static_cast<int64_t>(brow + row) * ldd + hs.qcol(h) + grp * CO,
                                 acc, scale);
      g0 += nkb;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
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

int g_fwd64_design = 3;  // pc_attention_tune key 0
int g_fwd64_emu = 6;     // pc_attention_tune key 1
int g_fwd_split = 1;     // pc_attention_tune key 2: fa_fwd_tc5 with two issuing warps
int g_dq_split = 1;      // pc_attention_tune key 3: fa_bwd_dq_tc5 with two issuing warps

// O as a 3-D tensor [B][S][ld_o] (rows clipped per sequence), box 64 x 32 x 1.
int make_tmap_o3(CUtensorMap* m, const void* base, int64_t ld, int S, int B) {
  auto enc = tmap_encoder_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return PC_ERR_CUDA;
  }
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(B)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 2), static_cast<cuuint64_t>(ld * 2 * S)};
  cuuint32_t box[3] = {64u, 32u, 1u};
  cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (attention O) failed (%d)", static_cast<int>(r));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

template <int EMU, int ABL = 0, int SPLIT = 0>
int fwd64_launch(int B, int S, Heads hs, const CUtensorMap& tm, void* o, int64_t ld_o, float* lse,
                 cudaStream_t st) {
  CUtensorMap to;
  int rc = make_tmap_o3(&to, o, ld_o, S, B);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    PP_CUDA_TRY(cudaFuncSetAttribute(fa_fwd64_tc5<EMU, ABL, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Fwd64::SMEM));
    attr = true;
  }
  const int items = B * hs.H * ((S + Fwd64::BM - 1) / Fwd64::BM);
  const int grid = items < 2 * num_sms() ? items : 2 * num_sms();
  const float sl2 = F_LOG2E / 8.f;  // 1 / sqrt(64)
  fa_fwd64_tc5<EMU, ABL, SPLIT><<<grid, Fwd64::THREADS, Fwd64::SMEM, st>>>(tm, to, lse, B, hs, S, sl2);
  return check_launch("fa_fwd64_tc5");
}

template <int HD>
int fwd_launch(int B, int S, Heads hs, const void* qkv, int64_t ld_qkv, void* o, int64_t ld_o,
               float* lse, cudaStream_t st) {
  CUtensorMap tm;
  int rc = make_tmap_rows64(&tm, qkv, ld_qkv, static_cast<int64_t>(B) * S);
  if (rc) return rc;
  if (HD == 64 && g_fwd64_design == 3) {
    switch (g_fwd64_emu) {
      case 0: return fwd64_launch<0, 0, 1>(B, S, hs, tm, o, ld_o, lse, st);
      case 4: return fwd64_launch<4, 0, 1>(B, S, hs, tm, o, ld_o, lse, st);
      case 8: return fwd64_launch<8, 0, 1>(B, S, hs, tm, o, ld_o, lse, st);
      case 101: return fwd64_launch<0, 1, 1>(B, S, hs, tm, o, ld_o, lse, st);
      case 102: return fwd64_launch<0, 2, 1>(B, S, hs, tm, o, ld_o, lse, st);
      default: return fwd64_launch<6, 0, 1>(B, S, hs, tm, o, ld_o, lse, st);
    }
  }
  if (HD == 64 && g_fwd64_design == 2) {
    switch (g_fwd64_emu) {
      case 0: return fwd64_launch<0>(B, S, hs, tm, o, ld_o, lse, st);
      case 4: return fwd64_launch<4>(B, S, hs, tm, o, ld_o, lse, st);
      case 8: return fwd64_launch<8>(B, S, hs, tm, o, ld_o, lse, st);
      case 101: return fwd64_launch<0, 1>(B, S, hs, tm, o, ld_o, lse, st);
      case 102: return fwd64_launch<0, 2>(B, S, hs, tm, o, ld_o, lse, st);
      default: return fwd64_launch<6>(B, S, hs, tm, o, ld_o, lse, st);
    }
  }
  static bool attr = false;
  if (!attr) {
    PP_CUDA_TRY(cudaFuncSetAttribute(fa_fwd_tc5<HD, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Fwd<HD>::SMEM));
    PP_CUDA_TRY(cudaFuncSetAttribute(fa_fwd_tc5<HD, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Fwd<HD>::SMEM));
    attr = true;
  }
  dim3 grid(B * hs.H, (S + Fwd<HD>::BM - 1) / Fwd<HD>::BM);
  const float sl2 = F_LOG2E / sqrtf(static_cast<float>(HD));
  if (g_fwd_split)
    fa_fwd_tc5<HD, 1><<<grid, Fwd<HD>::THREADS, Fwd<HD>::SMEM, st>>>(tm, static_cast<bf16*>(o), ld_o, lse,
                                                                    hs, S, sl2);
  else
    fa_fwd_tc5<HD, 0><<<grid, Fwd<HD>::THREADS, Fwd<HD>::SMEM, st>>>(tm, static_cast<bf16*>(o), ld_o, lse,
                                                                    hs, S, sl2);
  return check_launch("fa_fwd_tc5");
}

template <int HD>
int bwd_launch(int B, int S, Heads hs, const void* qkv, int64_t ld_qkv, const void* o,
               const void* dO, int64_t ld_o, const float* lse, float* delta, void* dqkv,
               int64_t ld_dqkv, cudaStream_t st) {
  CUtensorMap tq, tg, to;
  int rc = make_tmap_rows64(&tq, qkv, ld_qkv, static_cast<int64_t>(B) * S);
  if (rc) return rc;
  rc = make_tmap_rows64(&tg, dO, ld_o, static_cast<int64_t>(B) * S);
  if (rc) return rc;
  rc = make_tmap_rows64(&to, o, ld_o, static_cast<int64_t>(B) * S);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    PP_CUDA_TRY(cudaFuncSetAttribute(fa_bwd_dkdv_tc5<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     BwdKV<HD>::SMEM));
    PP_CUDA_TRY(cudaFuncSetAttribute(fa_bwd_dq_tc5<HD, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     BwdQ<HD>::SMEM));
    PP_CUDA_TRY(cudaFuncSetAttribute(fa_bwd_dq_tc5<HD, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     BwdQ<HD>::SMEM));
    attr = true;
  }
  const float scale = 1.f / sqrtf(static_cast<float>(HD));
  const float sl2 = scale * F_LOG2E;
  // dQ first: it also writes delta = rowsum(dO o O), which dK/dV consume.
  // Both persistent: one CTA per SM over their work lists.
  const int dq_items = B * hs.H * ((S + BwdQ<HD>::BM - 1) / BwdQ<HD>::BM);
  const int g2 = dq_items < num_sms() ? dq_items : num_sms();
  if (g_dq_split)
    fa_bwd_dq_tc5<HD, 1><<<g2, BwdQ<HD>::THREADS, BwdQ<HD>::SMEM, st>>>(
        tq, tg, to, lse, delta, static_cast<bf16*>(dqkv), ld_dqkv, B * hs.H, hs, S, sl2, scale);
  else
    fa_bwd_dq_tc5<HD, 0><<<g2, BwdQ<HD>::THREADS, BwdQ<HD>::SMEM, st>>>(
        tq, tg, to, lse, delta, static_cast<bf16*>(dqkv), ld_dqkv, B * hs.H, hs, S, sl2, scale);
  rc = check_launch("fa_bwd_dq_tc5");
  if (rc) return rc;
  const int kv_items = B * hs.Hkv * ((S + BwdKV<HD>::KEYS - 1) / BwdKV<HD>::KEYS);
  const int g1 = kv_items < num_sms() ? kv_items : num_sms();
  fa_bwd_dkdv_tc5<HD><<<g1, BwdKV<HD>::THREADS, BwdKV<HD>::SMEM, st>>>(
      tq, tg, lse, delta, static_cast<bf16*>(dqkv), ld_dqkv, B, hs, S, sl2, scale);
  return check_launch("fa_bwd_dkdv_tc5");
}
}  // namespace

int attention_tc5_tune(int key, int value) {
  if (key == 0 && (value >= 1 && value <= 3)) {
    g_fwd64_design = value;
  } else if (key == 2 && (value == 0 || value == 1)) {
    g_fwd_split = value;
  } else if (key == 3 && (value == 0 || value == 1)) {
    g_dq_split = value;
  } else if (key == 1 && (value == 0 || value == 4 || value == 6 || value == 8 || value == 101 || value == 102)) {
    g_fwd64_emu = value;
  } else {
    set_error("pc_attention_tune: unknown key %d or value %d", key, value);
    return PC_ERR_ARG;
  }
  return PC_OK;
}

bool attention_tc5_supported(int hd, int H, int Hkv, int64_t ld_qkv, int64_t ld_o, const void* qkv,
                             const void* o) {
  return (hd == 64 || hd == 128) && Hkv > 0 && H % Hkv == 0 && (ld_qkv * 2) % 16 == 0 &&
         (ld_o * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(o) & 15) == 0;
}

int attention_fwd_tc5(int B, int H, int Hkv, int S, int hd, const void* qkv, int64_t ld_qkv, void* o,
                      int64_t ld_o, float* lse, cudaStream_t st) {
  const Heads hs{H, Hkv, H / Hkv, hd};
  return hd == 64 ? fwd_launch<64>(B, S, hs, qkv, ld_qkv, o, ld_o, lse, st)
                  : fwd_launch<128>(B, S, hs, qkv, ld_qkv, o, ld_o, lse, st);
}

int attention_bwd_tc5(int B, int H, int Hkv, int S, int hd, const void* qkv, int64_t ld_qkv,
                      const void* o, const void* dO, int64_t ld_o, const float* lse, float* delta,
                      void* dqkv, int64_t ld_dqkv, cudaStream_t st) {
  const Heads hs{H, Hkv, H / Hkv, hd};
  return hd == 64 ? bwd_launch<64>(B, S, hs, qkv, ld_qkv, o, dO, ld_o, lse, delta, dqkv, ld_dqkv, st)
                  : bwd_launch<128>(B, S, hs, qkv, ld_qkv, o, dO, ld_o, lse, delta, dqkv, ld_dqkv, st);
}

}  // namespace pp200
