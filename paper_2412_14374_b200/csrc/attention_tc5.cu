// tcgen05 causal flash-attention forward (bf16, head_dim 64), sm_100a.
//
// Semantics: oracle/gpt.py `attention` (exact softmax, causal), same layout
// contract as attention_tc.cu (qkv [B*S, ld], o [B*S, ld_o], lse [B,H,S]).
//
// One CTA = 128 query rows of one (batch, head); 8 warps:
//   warp 0      TMA producer: Q tile once, then K/V tiles of 64 keys into a
//               3-deep 128B-swizzled smem ring
//   warp 1      single-thread tcgen05.mma issuer:
//                 S = Q K^T   (M=128, N=64 keys, K=64)  -> TMEM cols [0, 64)
//                 O += P V    (M=128, N=64 dims, K=64)  -> TMEM cols [64, 128)
//   warp 2      TMEM allocator (128 columns: 2 CTAs fit per SM)
//   warps 4..7  softmax: one thread owns one query row (TMEM lane), so row
//               max / sum need no shuffles; P is written as bf16 into a
//               128B-swizzled K-major smem tile (the MMA's A operand), O is
//               rescaled in TMEM when the running max moves.
// Ordering: the commit after S_{j+1} also covers PV_j, so when the softmax
// warps see S_{j+1} ready they may overwrite P and rescale O.
#include <cudaTypedefs.h>

#include "common.cuh"

namespace pp200 {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder_fn();

namespace {

using bf16 = __nv_bfloat16;
constexpr int F_BM = 128, F_BN = 64, F_HD = 64, F_STAGES = 2, F_THREADS = 256;
constexpr int F_Q_BYTES = F_BM * F_HD * 2;    // 16 KB
constexpr int F_KV_BYTES = F_BN * F_HD * 2;   // 8 KB
constexpr int F_P_BYTES = F_BM * F_BN * 2;    // 16 KB
constexpr int F_SMEM = F_Q_BYTES + 2 * F_STAGES * F_KV_BYTES + F_P_BYTES + 1024 + 256;
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
  uint64_t* bar_q = reinterpret_cast<uint64_t*>(sP + F_P_BYTES);
  uint64_t* kv_full = bar_q + 1;
  uint64_t* kv_empty = kv_full + F_STAGES;
  uint64_t* s_full = kv_empty + F_STAGES;
  uint64_t* p_full = s_full + 1;
  uint64_t* o_done = p_full + 1;
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
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tslot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 64;

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
      const uint32_t q_addr = smem_u32(sQ), p_addr = smem_u32(sP);
      for (int j = 0; j < nkb; ++j) {
        const int s = j % F_STAGES;
        mbar_wait(&kv_full[s], (j / F_STAGES) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + s * F_KV_BYTES);
        const uint32_t v_addr = smem_u32(sV + s * F_KV_BYTES);
#pragma unroll
        for (int k = 0; k < F_HD / 16; ++k)
          tc_mma_f16(tS, umma_sdesc_sw128(q_addr + k * 32, 16, 1024),
                     umma_sdesc_sw128(k_addr + k * 32, 16, 1024), ID_S, k > 0 ? 1u : 0u);
        tc_commit(s_full);
        mbar_wait(p_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < F_BN / 16; ++k)
          tc_mma_f16(tO, umma_sdesc_sw128(p_addr + k * 32, 16, 1024),
                     umma_sdesc_sw128(v_addr + k * 2048, 8192, 1024), ID_O,
                     (j > 0 || k > 0) ? 1u : 0u);
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
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      uint32_t sr[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(tS + lane_off + c * 16, sr + c * 16);
      tc_wait_ld();
      float* sv = reinterpret_cast<float*>(sr);
      const int n0 = j * F_BN;
      const bool edge = n0 + F_BN - 1 > q0 || n0 + F_BN > S;  // diagonal or ragged block
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < F_BN; ++i) {
        float v = sv[i] * sl2;
        if (edge && (n0 + i > row || n0 + i >= S)) v = -INFINITY;
        sv[i] = v;
        mx = fmaxf(mx, v);
      }
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
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < F_BN; ++i) {
        const float p = ex2(sv[i] - m);
        sv[i] = p;
        sum += p;
      }
      l = l * corr + sum;
      // P row -> smem, K-major with 128B swizzle (8 chunks of 8 bf16)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 u;
        __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int k = 0; k < 4; ++k) hp[k] = __floats2bfloat162_rn(sv[8 * c + 2 * k], sv[8 * c + 2 * k + 1]);
        *reinterpret_cast<uint4*>(sP + r * 128 + ((c ^ (r & 7)) << 4)) = u;
      }
      fence_proxy_async_smem();
      // rescale O by corr (PV_{j-1} is complete: covered by the S_j commit)
      if (j > 0 && __any_sync(0xffffffffu, corr != 1.f && l > 0.f)) {
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
      if (lane == 0) mbar_arrive(p_full);
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
  if (warp == 2) tmem_dealloc(tmem, 128);
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
