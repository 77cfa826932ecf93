// Fused LM head + next-token cross-entropy (SURVEY §8(b) pc_lmhead_xent_fwd/bwd),
// replacing the reference's loss node `sub-sample-loss` (executor.py:72-75) in
// the GPT / Llama vocabularies (oracle/gpt.py head_loss).
//
// Forward, two launches:
//   1. the logits GEMM (tcgen05, bf16 out through TMA) whose epilogue also
//      leaves, per row and per (N tile, epilogue column group), the running
//      (max, sum exp(x - max)) of the values it stored -- no pass over the
//      logits is needed for the log-sum-exp;
//   2. one streaming pass per row: combine the partials (fixed order) into
//      lse, row loss = lse - logit[target], and overwrite the logits in place
//      with dlogits = exp(logit - lse) - onehot(target) (one exp per element,
//      read + write once; the last position of each sequence has no target
//      and gets zeros).
// Backward: dh = dlogits W and dW (+)= dlogits^T h, two tcgen05 GEMMs.
#include "common.cuh"

namespace pp200 {

int gemm_bf16_tc(int out_f32, int transA, int transB, int64_t M, int64_t N, int64_t K,
                 const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                 int epi, const void* bias, const void* aux, int64_t ldaux, void* aux_out,
                 int64_t ldaux_out, cudaStream_t st, float2* stats, int64_t ld_stats);

namespace {

constexpr int XF_THREADS = 256;
constexpr int TC_EPI_G = 2;  // epilogue column groups per TMEM lane quarter (gemm_tc.cu)

__device__ __forceinline__ void ms_combine(float& m, float& s, float mo, float so) {
  const float mn = fmaxf(m, mo);
  if (mn == -INFINITY) return;  // both empty
  float a, b;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"((m - mn) * 1.4426950408889634f));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"((mo - mn) * 1.4426950408889634f));
  s = s * a + so * b;
  m = mn;
}

__global__ void __launch_bounds__(XF_THREADS) xent_finish_kernel(
    int V, int seq, __nv_bfloat16* __restrict__ logits, int64_t ld, const int32_t* __restrict__ tok,
    const float2* __restrict__ stats, int nstat, int64_t ld_stats, float* __restrict__ row_loss) {
  __shared__ float sm[XF_THREADS / 32], ss[XF_THREADS / 32];
  __shared__ float s_lse;
  const int64_t r = blockIdx.x;
  uint4* row = reinterpret_cast<uint4*>(logits + r * ld);
  const int nv = V / 8;
  if ((r % seq) == seq - 1) {  // no next token: zero loss, zero gradient
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int c = threadIdx.x; c < nv; c += blockDim.x) row[c] = z;
    if (threadIdx.x == 0) row_loss[r] = 0.f;
    return;
  }
  // fixed-order combine of the GEMM's partial statistics: thread t folds
  // partials t, t + 256, ...; then a shuffle tree; then the warps in order
  float m = -INFINITY, s = 0.f;
  const float2* sr = stats + r * ld_stats;
  for (int i = threadIdx.x; i < nstat; i += blockDim.x) {
    const float2 p = sr[i];
    ms_combine(m, s, p.x, p.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, o), so = __shfl_xor_sync(0xffffffffu, s, o);
    ms_combine(m, s, mo, so);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sm[w] = m;
    ss[w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float mm = sm[0], s2 = ss[0];
    for (int k = 1; k < XF_THREADS / 32; ++k) ms_combine(mm, s2, sm[k], ss[k]);
    const float lse = mm + logf(s2);
    s_lse = lse;
    row_loss[r] = lse - __bfloat162float(logits[r * ld + tok[r + 1]]);
  }
  __syncthreads();
  const float nl = -s_lse * 1.4426950408889634f;
  const int target = tok[r + 1];
  // dlogits in place: 16-byte chunks, two in flight per thread
  for (int c = threadIdx.x; c < nv; c += 2 * blockDim.x) {
    const int c2 = c + blockDim.x;
    uint4 u0 = row[c];
    uint4 u1 = c2 < nv ? row[c2] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int cc = half ? c2 : c;
      if (cc >= nv) break;
      uint4& u = half ? u1 : u0;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        float e0, e1;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(fmaf(f.x, 1.4426950408889634f, nl)));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(fmaf(f.y, 1.4426950408889634f, nl)));
        const int col = cc * 8 + 2 * j;
        if (col == target) e0 -= 1.f;
        if (col + 1 == target) e1 -= 1.f;
        h[j] = __floats2bfloat162_rn(e0, e1);
      }
      row[cc] = u;
    }
  }
}

}  // namespace
}  // namespace pp200

using namespace pp200;

extern "C" int pc_lmhead_xent_workspace(int64_t T, int64_t V, int64_t d, int64_t* ld_stats,
                                        int64_t* bytes) {
  PP_CHECK_ARG(T > 0 && V > 0 && d > 0 && ld_stats && bytes, "lmhead_xent_workspace: bad args");
  int bn, cg, ks;
  if (int rc = pc_gemm_tile_choice(1, T, V, d, 0, &bn, &cg, &ks)) return rc;
  *ld_stats = ((V + bn - 1) / bn) * TC_EPI_G;
  *bytes = T * *ld_stats * static_cast<int64_t>(sizeof(float2));
  return PC_OK;
}

extern "C" int pc_lmhead_xent_fwd(int64_t T, int64_t V, int64_t d, int64_t seq, const void* h,
                                  int64_t ldh, const void* w, int64_t ldw, const int32_t* tokens,
                                  void* logits, int64_t ld_logits, void* ws, int64_t ws_bytes,
                                  float* row_loss, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PP_CHECK_ARG(T > 0 && V > 0 && d > 0 && seq > 0 && T % seq == 0, "lmhead_xent: bad dims");
  PP_CHECK_ARG(V % 8 == 0 && ld_logits % 8 == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0,
               "lmhead_xent: logits rows must be 16 B aligned (V %% 8 == 0)");
  int64_t ld_stats = 0, need = 0;
  if (int rc = pc_lmhead_xent_workspace(T, V, d, &ld_stats, &need)) return rc;
  PP_CHECK_ARG(ws != nullptr && ws_bytes >= need, "lmhead_xent: workspace too small");
  float2* stats = static_cast<float2*>(ws);
  int rc = gemm_bf16_tc(0, 0, 1, T, V, d, h, ldh, w, ldw, logits, ld_logits, 0, nullptr, nullptr,
                        0, nullptr, 0, st, stats, ld_stats);
  if (rc) return rc;
  xent_finish_kernel<<<static_cast<unsigned>(T), XF_THREADS, 0, st>>>(
      static_cast<int>(V), static_cast<int>(seq), static_cast<__nv_bfloat16*>(logits), ld_logits,
      tokens, stats, static_cast<int>(ld_stats), ld_stats, row_loss);
  return check_launch("xent_finish_kernel");
}

extern "C" int pc_lmhead_xent_bwd(int64_t T, int64_t V, int64_t d, const void* dlogits, int64_t ld,
                                  const void* h, int64_t ldh, const void* w_t, int64_t ld_wt,
                                  void* dh, int64_t ld_dh, float* dw, int64_t ld_dw,
                                  int accumulate, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PP_CHECK_ARG(T > 0 && V > 0 && d > 0, "lmhead_xent_bwd: bad dims");
  // dh [T, d] = dlogits [T, V] x W [V, d], B read K-major from W^T [d, V]
  int rc = gemm_bf16_tc(0, 0, 1, T, d, V, dlogits, ld, w_t, ld_wt, dh, ld_dh, 0, nullptr, nullptr,
                        0, nullptr, 0, st, nullptr, 0);
  if (rc) return rc;
  // dW [V, d] (+)= dlogits^T h (fp32; unsplit, one add per element when accumulating)
  return gemm_bf16_tc(1, 1, 0, V, d, T, dlogits, ld, h, ldh, dw, ld_dw,
                      accumulate ? PC_EPI_ACCUM : 0, nullptr, nullptr, 0, nullptr, 0, st, nullptr, 0);
}
