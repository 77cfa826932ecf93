// GPT vocabulary kernels: LayerNorm fwd/bwd, token+position embedding fwd/bwd,
// fused next-token cross-entropy (loss + in-place dlogits).
//
// The reference has no GPT ops (SURVEY.md key fact 5); these implement the
// semantics of oracle/gpt.py (layer_norm, head_loss, embedding) on B200.
// Row-parallel kernels give one warp per row with coalesced, vectorised
// (16 B) loads; parameter reductions (dgamma, dbeta, dwpe, dwte) use fixed
// summation orders so every result is bitwise reproducible.
#include <cub/cub.cuh>

#include "common.cuh"

namespace pp200 {
namespace {

template <typename T> __device__ __forceinline__ float ldf(const T* p, int64_t i) {
  return static_cast<float>(p[i]);
}
template <> __device__ __forceinline__ float ldf(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}
template <typename T> __device__ __forceinline__ void stf(T* p, int64_t i, float v) {
  p[i] = static_cast<T>(v);
}
template <> __device__ __forceinline__ void stf(__nv_bfloat16* p, int64_t i, float v) {
  p[i] = __float2bfloat16_rn(v);
}

constexpr int ROWS_PER_BLOCK = 8;  // one warp per row

template <typename T>
__global__ void __launch_bounds__(256) ln_fwd_kernel(int64_t rows, int d, const T* __restrict__ x,
                                                     const float* __restrict__ g,
                                                     const float* __restrict__ b, T* __restrict__ y,
                                                     float* __restrict__ mean,
                                                     float* __restrict__ rstd, float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)ROWS_PER_BLOCK + (threadIdx.x >> 5);
  if (r >= rows) return;
  const T* xr = x + r * d;
  float s = 0.f;
  for (int c = lane; c < d; c += 32) s += ldf(xr, c);
  const float mu = warp_sum(s) / d;
  float v = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float t = ldf(xr, c) - mu;
    v += t * t;
  }
  const float rs = rsqrtf(warp_sum(v) / d + eps);
  T* yr = y + r * d;
  for (int c = lane; c < d; c += 32) stf(yr, c, (ldf(xr, c) - mu) * rs * g[c] + b[c]);
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

// dx = dres + rstd * (dxh - mean(dxh) - xh * mean(dxh * xh)),  dxh = dy * g
template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_dx_kernel(int64_t rows, int d, const T* __restrict__ dy,
                                                        const T* __restrict__ x,
                                                        const float* __restrict__ g,
                                                        const float* __restrict__ mean,
                                                        const float* __restrict__ rstd,
                                                        const T* __restrict__ dres,
                                                        T* __restrict__ dx) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)ROWS_PER_BLOCK + (threadIdx.x >> 5);
  if (r >= rows) return;
  const T* dyr = dy + r * d;
  const T* xr = x + r * d;
  const float mu = mean[r], rs = rstd[r];
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float dxh = ldf(dyr, c) * g[c];
    const float xh = (ldf(xr, c) - mu) * rs;
    s1 += dxh;
    s2 += dxh * xh;
  }
  const float m1 = warp_sum(s1) / d, m2 = warp_sum(s2) / d;
  T* dxr = dx + r * d;
  const T* rr = dres ? dres + r * d : nullptr;
  for (int c = lane; c < d; c += 32) {
    const float dxh = ldf(dyr, c) * g[c];
    const float xh = (ldf(xr, c) - mu) * rs;
    float v = rs * (dxh - m1 - xh * m2);
    if (rr) v += ldf(rr, c);
    stf(dxr, c, v);
  }
}

// dgamma[c] = sum_r dy[r,c] * xh[r,c]; dbeta[c] = sum_r dy[r,c]  (fixed order)
template <typename T>
__global__ void __launch_bounds__(1024) ln_bwd_param_kernel(int64_t rows, int d,
                                                            const T* __restrict__ dy,
                                                            const T* __restrict__ x,
                                                            const float* __restrict__ mean,
                                                            const float* __restrict__ rstd,
                                                            float* dgamma, float* dbeta) {
  __shared__ float sg[32][33], sb[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  float a = 0.f, bsum = 0.f;
  if (c < d)
    for (int64_t r = ty; r < rows; r += 32) {
      const float gy = ldf(dy, r * d + c);
      a += gy * (ldf(x, r * d + c) - mean[r]) * rstd[r];
      bsum += gy;
    }
  sg[ty][tx] = a;
  sb[ty][tx] = bsum;
  __syncthreads();
  if (ty == 0 && c < d) {
    float ta = 0.f, tb = 0.f;
    for (int k = 0; k < 32; ++k) {
      ta += sg[k][tx];
      tb += sb[k][tx];
    }
    dgamma[c] = ta;
    dbeta[c] = tb;
  }
}

// ---- vectorised LayerNorm (d = 256*NCH, NCH <= 4): the row lives in registers,
// one 16 B load / store per 8 elements.
template <typename T>
__device__ __forceinline__ void ld8(const T* p, float* v) {
  if (sizeof(T) == 2) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h[j]);
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
  } else {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}
template <typename T>
__device__ __forceinline__ void st8(T* p, const float* v) {
  if (sizeof(T) == 2) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  } else {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}
__device__ __forceinline__ void ldf8(const float* p, float* v) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

template <typename T, int NCH>
__global__ void __launch_bounds__(256) ln_fwd_vec(int64_t rows, int d, const T* __restrict__ x,
                                                  const float* __restrict__ g,
                                                  const float* __restrict__ b, T* __restrict__ y,
                                                  float* __restrict__ mean,
                                                  float* __restrict__ rstd, float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)ROWS_PER_BLOCK + (threadIdx.x >> 5);
  if (r >= rows) return;
  float v[NCH][8];
  float s = 0.f;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    ld8(x + r * d + ch * 256 + lane * 8, v[ch]);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[ch][j];
  }
  const float mu = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float t = v[ch][j] - mu;
      q += t * t;
    }
  const float rs = rsqrtf(warp_sum(q) / d + eps);
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    const int c = ch * 256 + lane * 8;
    float gg[8], bb[8], o[8];
    ldf8(g + c, gg);
    ldf8(b + c, bb);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (v[ch][j] - mu) * rs * gg[j] + bb[j];
    st8(y + r * d + c, o);
  }
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

template <typename T, int NCH>
__global__ void __launch_bounds__(256) ln_bwd_dx_vec(int64_t rows, int d, const T* __restrict__ dy,
                                                     const T* __restrict__ x,
                                                     const float* __restrict__ g,
                                                     const float* __restrict__ mean,
                                                     const float* __restrict__ rstd,
                                                     const T* __restrict__ dres,
                                                     T* __restrict__ dx) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)ROWS_PER_BLOCK + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float mu = mean[r], rs = rstd[r];
  float dxh[NCH][8], xh[NCH][8];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    const int c = ch * 256 + lane * 8;
    float gy[8], xv[8], gg[8];
    ld8(dy + r * d + c, gy);
    ld8(x + r * d + c, xv);
    ldf8(g + c, gg);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      dxh[ch][j] = gy[j] * gg[j];
      xh[ch][j] = (xv[j] - mu) * rs;
      s1 += dxh[ch][j];
      s2 += dxh[ch][j] * xh[ch][j];
    }
  }
  const float m1 = warp_sum(s1) / d, m2 = warp_sum(s2) / d;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    const int c = ch * 256 + lane * 8;
    float o[8], rr[8];
    if (dres) ld8(dres + r * d + c, rr);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = rs * (dxh[ch][j] - m1 - xh[ch][j] * m2) + (dres ? rr[j] : 0.f);
    st8(dx + r * d + c, o);
  }
}

// LayerNorm backward that also leaves the parameter-gradient partials: each CTA
// owns a contiguous chunk of rows (warps stride them), computes dx exactly as
// ln_bwd_dx_vec, and adds dy*xhat and dy of every row it handles into its
// warp's private shared-memory accumulators (no atomics); the CTA then folds
// its 8 warps in order and writes one partial row per quantity (pg / pb
// [gridDim.x, d]).  dy and x are read once; a fixed-order column sum of the
// partial rows (pc_col_sum, on any stream) finishes dgamma / dbeta.
template <typename T, int NCH>
__global__ void __launch_bounds__(256) ln_bwd_partials_vec(int64_t rows, int d, int64_t chunk,
                                                           const T* __restrict__ dy,
                                                           const T* __restrict__ x,
                                                           const float* __restrict__ g,
                                                           const float* __restrict__ mean,
                                                           const float* __restrict__ rstd,
                                                           const T* __restrict__ dres,
                                                           T* __restrict__ dx,
                                                           float* __restrict__ pg,
                                                           float* __restrict__ pb) {
  // [8 warps][2][NCH * 256]; column ch*256 + lane*8 + j lives at ch*256 + j*32 + lane
  // (consecutive lanes, consecutive banks: conflict-free read-modify-writes)
  extern __shared__ float acc_sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* ag = acc_sm + w * 2 * NCH * 256;
  float* ab = ag + NCH * 256;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
    for (int j = 0; j < 8; ++j) ag[ch * 256 + j * 32 + lane] = ab[ch * 256 + j * 32 + lane] = 0.f;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  for (int64_t r = r0 + w; r < r1; r += 8) {
    const float mu = mean[r], rs = rstd[r];
    float gy[NCH][8], xh[NCH][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int c = ch * 256 + lane * 8;
      float xv[8], gg[8];
      ld8(dy + r * d + c, gy[ch]);
      ld8(x + r * d + c, xv);
      ldf8(g + c, gg);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        xh[ch][j] = (xv[j] - mu) * rs;
        const float t = gy[ch][j] * gg[j];
        s1 += t;
        s2 += t * xh[ch][j];
        const int k = ch * 256 + j * 32 + lane;
        ag[k] = fmaf(gy[ch][j], xh[ch][j], ag[k]);
        ab[k] += gy[ch][j];
      }
    }
    const float m1 = warp_sum(s1) / d, m2 = warp_sum(s2) / d;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int c = ch * 256 + lane * 8;
      float o[8], rr[8], gg[8];
      ldf8(g + c, gg);
      if (dres) ld8(dres + r * d + c, rr);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        o[j] = rs * (gy[ch][j] * gg[j] - m1 - xh[ch][j] * m2) + (dres ? rr[j] : 0.f);
      st8(dx + r * d + c, o);
    }
  }
  __syncthreads();
  // fold the 8 warps in order
  float* og = pg + static_cast<int64_t>(blockIdx.x) * d;
  float* ob = pb + static_cast<int64_t>(blockIdx.x) * d;
  for (int c = threadIdx.x; c < d; c += 256) {
    const int k0 = (c / 256) * 256 + (c % 8) * 32 + (c % 256) / 8;  // storage slot of column c
    float tg = 0.f, tb = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      tg += acc_sm[k * 2 * NCH * 256 + k0];
      tb += acc_sm[k * 2 * NCH * 256 + NCH * 256 + k0];
    }
    og[c] = tg;
    ob[c] = tb;
  }
}

template <typename T>
bool ln_vec_ok(int64_t d, const void* p0, const void* p1, const void* p2) {
  const uintptr_t m = reinterpret_cast<uintptr_t>(p0) | reinterpret_cast<uintptr_t>(p1) |
                      reinterpret_cast<uintptr_t>(p2);
  return d % 256 == 0 && d / 256 >= 1 && d / 256 <= 4 && (m & 31) == 0;
}

// out[t,:] = wte[tok[t],:] + wpe[t % seq,:]   (fp32 master tables)
template <typename T>
__global__ void __launch_bounds__(256) embed_fwd_kernel(int64_t T_, int d, int seq,
                                                        const int32_t* __restrict__ tok,
                                                        const float* __restrict__ wte,
                                                        const float* __restrict__ wpe,
                                                        T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x * (int64_t)ROWS_PER_BLOCK + (threadIdx.x >> 5);
  if (t >= T_) return;
  const float* a = wte + static_cast<int64_t>(tok[t]) * d;
  const float* p = wpe + static_cast<int64_t>(t % seq) * d;
  T* o = out + t * d;
  for (int c = lane; c < d; c += 32) stf(o, c, a[c] + p[c]);
}

__global__ void iota_kernel(int n, int32_t* v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

// One warp per sorted position; segment heads sum their rows (ascending row
// order from the stable sort) into dwte[token].  Rows of absent tokens are
// zeroed beforehand.
template <typename T>
__global__ void __launch_bounds__(256) embed_bwd_wte_kernel(int n, int d,
                                                            const int32_t* __restrict__ keys,
                                                            const int32_t* __restrict__ rows,
                                                            const T* __restrict__ dh,
                                                            float* __restrict__ dwte,
                                                            int accumulate) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * ROWS_PER_BLOCK + (threadIdx.x >> 5);
  if (i >= n) return;
  const int key = keys[i];
  if (i > 0 && keys[i - 1] == key) return;
  int j = i + 1;
  while (j < n && keys[j] == key) ++j;
  float* out = dwte + static_cast<int64_t>(key) * d;
  for (int c = lane; c < d; c += 32) {
    float s = 0.f;
    for (int k = i; k < j; ++k) s += ldf(dh, static_cast<int64_t>(rows[k]) * d + c);
    out[c] = accumulate ? out[c] + s : s;
  }
}

// dwpe[s,c] = sum_b dh[b*seq + s, c]
template <typename T>
__global__ void embed_bwd_wpe_kernel(int64_t T_, int d, int seq, const T* __restrict__ dh,
                                     float* __restrict__ dwpe, int accumulate) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(seq) * d) return;
  const int64_t s = i / d, c = i % d;
  float acc = 0.f;
  for (int64_t t = s; t < T_; t += seq) acc += ldf(dh, t * d + c);
  dwpe[i] = accumulate ? dwpe[i] + acc : acc;
}

// Per row: online (max, sum) over the vocab, loss = lse - logit[target], then
// overwrite the row with dlogits = softmax - onehot (zeros for the last
// position of each sequence, which has no target).
template <typename T>
__global__ void __launch_bounds__(512) xent_kernel(int64_t rows, int V, int seq, T* logits,
                                                   int64_t ld, const int32_t* __restrict__ tok,
                                                   float* __restrict__ row_loss) {
  __shared__ float sm[32], ss[32];
  const int64_t r = blockIdx.x;
  T* row = logits + r * ld;
  const bool valid = (r % seq) != seq - 1;
  if (!valid) {
    for (int c = threadIdx.x; c < V; c += blockDim.x) stf(row, c, 0.f);
    if (threadIdx.x == 0) row_loss[r] = 0.f;
    return;
  }
  const int target = tok[r + 1];
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x; c < V; c += blockDim.x) {
    const float v = ldf(row, c);
    if (v > m) {
      s = s * __expf(m - v) + 1.f;
      m = v;
    } else {
      s += __expf(v - m);
    }
  }
  // warp combine
  for (int o = 16; o > 0; o >>= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, o), so = __shfl_xor_sync(0xffffffffu, s, o);
    const float mn = fmaxf(m, mo);
    s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (mo == -INFINITY ? 0.f : so * __expf(mo - mn));
    m = mn;
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sm[w] = m;
    ss[w] = s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < nw ? sm[threadIdx.x] : -INFINITY;
    s = threadIdx.x < nw ? ss[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) {
      const float mo = __shfl_xor_sync(0xffffffffu, m, o), so = __shfl_xor_sync(0xffffffffu, s, o);
      const float mn = fmaxf(m, mo);
      s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (mo == -INFINITY ? 0.f : so * __expf(mo - mn));
      m = mn;
    }
    if (threadIdx.x == 0) {
      sm[0] = m;
      ss[0] = s;
    }
  }
  __syncthreads();
  const float lse = sm[0] + logf(ss[0]);
  __syncthreads();
  if (threadIdx.x == 0) row_loss[r] = lse - ldf(row, target);
  __syncthreads();
  for (int c = threadIdx.x; c < V; c += blockDim.x) {
    const float p = __expf(ldf(row, c) - lse);
    stf(row, c, c == target ? p - 1.f : p);
  }
}


// (m, s) running softmax statistics merge
__device__ __forceinline__ void ms_merge(float& m, float& s, float mo, float so) {
  const float mn = fmaxf(m, mo);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (mo == -INFINITY ? 0.f : so * __expf(mo - mn));
  m = mn;
}

// bf16 rows with V % 8 == 0 and 16 B aligned rows: 16-byte loads and stores.
__global__ void __launch_bounds__(512) xent_bf16_vec_kernel(int64_t rows, int V, int seq,
                                                            __nv_bfloat16* logits, int64_t ld,
                                                            const int32_t* __restrict__ tok,
                                                            float* __restrict__ row_loss) {
  __shared__ float sm[16], ss[16];
  __shared__ float s_lse;
  const int64_t r = blockIdx.x;
  uint4* row = reinterpret_cast<uint4*>(logits + r * ld);
  const int nv = V / 8;
  const bool valid = (r % seq) != seq - 1;
  if (!valid) {
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int c = threadIdx.x; c < nv; c += blockDim.x) row[c] = z;
    if (threadIdx.x == 0) row_loss[r] = 0.f;
    return;
  }
  const int target = tok[r + 1];
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x; c < nv; c += blockDim.x) {
    const uint4 u = row[c];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
    float v[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h[j]);
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
    float bm = v[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) bm = fmaxf(bm, v[j]);
    float bs = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) bs += __expf(v[j] - bm);
    ms_merge(m, s, bm, bs);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    ms_merge(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sm[w] = m;
    ss[w] = s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < nw ? sm[threadIdx.x] : -INFINITY;
    s = threadIdx.x < nw ? ss[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      ms_merge(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
    if (threadIdx.x == 0) {
      const float lse = m + logf(s);
      s_lse = lse;
      row_loss[r] = lse - __bfloat162float(logits[r * ld + target]);
    }
  }
  __syncthreads();
  const float lse = s_lse;
  for (int c = threadIdx.x; c < nv; c += blockDim.x) {
    uint4 u = row[c];
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h[j]);
      float p0 = __expf(f.x - lse), p1 = __expf(f.y - lse);
      if (c * 8 + 2 * j == target) p0 -= 1.f;
      if (c * 8 + 2 * j + 1 == target) p1 -= 1.f;
      h[j] = __floats2bfloat162_rn(p0, p1);
    }
    row[c] = u;
  }
}
}  // namespace
}  // namespace pp200

using namespace pp200;

#define PP_DISPATCH_FB(dtype, T, ...)                                 \
  switch (dtype) {                                                    \
    case PC_F32: { using T = float; __VA_ARGS__; break; }            \
    case PC_BF16: { using T = __nv_bfloat16; __VA_ARGS__; break; }   \
    default: set_error("unsupported dtype %d (f32/bf16 only)", dtype); return PC_ERR_UNSUPPORTED; \
  }

static inline unsigned row_blocks(int64_t rows) {
  return static_cast<unsigned>((rows + ROWS_PER_BLOCK - 1) / ROWS_PER_BLOCK);
}

extern "C" int pc_layernorm_fwd(int dtype, int64_t rows, int64_t d, const void* x,
                                const float* gamma, const float* beta, void* y, float* mean,
                                float* rstd, float eps, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0) return PC_OK;
  PP_DISPATCH_FB(dtype, T,
    if (ln_vec_ok<T>(d, x, y, gamma) && (reinterpret_cast<uintptr_t>(beta) & 31) == 0) {
      const unsigned nb = row_blocks(rows);
      switch (d / 256) {
        case 1: ln_fwd_vec<T, 1><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(x), gamma, beta, static_cast<T*>(y), mean, rstd, eps); break;
        case 2: ln_fwd_vec<T, 2><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(x), gamma, beta, static_cast<T*>(y), mean, rstd, eps); break;
        case 3: ln_fwd_vec<T, 3><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(x), gamma, beta, static_cast<T*>(y), mean, rstd, eps); break;
        default: ln_fwd_vec<T, 4><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(x), gamma, beta, static_cast<T*>(y), mean, rstd, eps); break;
      }
    } else {
      ln_fwd_kernel<T><<<row_blocks(rows), 256, 0, st>>>(rows, (int)d, static_cast<const T*>(x), gamma, beta, static_cast<T*>(y), mean, rstd, eps);
    });
  return check_launch("layernorm_fwd");
}

namespace pp200 {
template <typename T>
bool colred_launch(int mode, int64_t rows, int64_t cols, const T* a, int64_t lda, const T* x,
                   const float* mean, const float* rstd, float* out1, float* out2,
                   int accumulate, void* ws, int64_t ws_bytes, cudaStream_t st);
int64_t colred_ws_bytes(int64_t rows, int64_t cols);
}

extern "C" int pc_layernorm_bwd(int dtype, int64_t rows, int64_t d, const void* dy, const void* x,
                                const float* gamma, const float* mean, const float* rstd,
                                const void* dres, void* dx, float* dgamma, float* dbeta,
                                void* ws, int64_t ws_bytes, void* stream) {
  return pc_layernorm_bwd_acc(dtype, rows, d, dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta,
                              0, ws, ws_bytes, stream);
}

extern "C" int pc_layernorm_bwd_acc(int dtype, int64_t rows, int64_t d, const void* dy,
                                    const void* x, const float* gamma, const float* mean,
                                    const float* rstd, const void* dres, void* dx, float* dgamma,
                                    float* dbeta, int accumulate, void* ws, int64_t ws_bytes,
                                    void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0) return PC_OK;
  PP_CHECK_ARG(!accumulate || ws_bytes >= colred_ws_bytes(rows, d),
               "layernorm_bwd: accumulate needs the reduction workspace");
  PP_DISPATCH_FB(dtype, T,
    if (ln_vec_ok<T>(d, dy, x, dx) && ((reinterpret_cast<uintptr_t>(gamma) | reinterpret_cast<uintptr_t>(dres)) & 31) == 0) {
      const unsigned nb = row_blocks(rows);
      const T* dr = static_cast<const T*>(dres);
      switch (d / 256) {
        case 1: ln_bwd_dx_vec<T, 1><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(dy), static_cast<const T*>(x), gamma, mean, rstd, dr, static_cast<T*>(dx)); break;
        case 2: ln_bwd_dx_vec<T, 2><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(dy), static_cast<const T*>(x), gamma, mean, rstd, dr, static_cast<T*>(dx)); break;
        case 3: ln_bwd_dx_vec<T, 3><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(dy), static_cast<const T*>(x), gamma, mean, rstd, dr, static_cast<T*>(dx)); break;
        default: ln_bwd_dx_vec<T, 4><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(dy), static_cast<const T*>(x), gamma, mean, rstd, dr, static_cast<T*>(dx)); break;
      }
    } else {
      ln_bwd_dx_kernel<T><<<row_blocks(rows), 256, 0, st>>>(rows, (int)d, static_cast<const T*>(dy), static_cast<const T*>(x), gamma, mean, rstd, static_cast<const T*>(dres), static_cast<T*>(dx));
    }
    if (dgamma == nullptr && dbeta == nullptr) {
      // dx only: the parameter gradients are reduced elsewhere (pc_layernorm_param_grads)
    } else if (!colred_launch<T>(1, rows, d, static_cast<const T*>(dy), d, static_cast<const T*>(x), mean, rstd, dgamma, dbeta, accumulate, ws, ws_bytes, st)) {
      ln_bwd_param_kernel<T><<<(unsigned)((d + 31) / 32), 1024, 0, st>>>(rows, (int)d, static_cast<const T*>(dy), static_cast<const T*>(x), mean, rstd, dgamma, dbeta);
    });
  return check_launch("layernorm_bwd");
}

extern "C" int pc_layernorm_param_grads(int dtype, int64_t rows, int64_t d, const void* dy,
                                        const void* x, const float* mean, const float* rstd,
                                        float* dgamma, float* dbeta, int accumulate, void* ws,
                                        int64_t ws_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0) return PC_OK;
  PP_CHECK_ARG(dgamma != nullptr && ws_bytes >= colred_ws_bytes(rows, d),
               "layernorm_param_grads: needs dgamma and the reduction workspace");
  bool ok = false;
  PP_DISPATCH_FB(dtype, T,
    ok = colred_launch<T>(1, rows, d, static_cast<const T*>(dy), d, static_cast<const T*>(x),
                          mean, rstd, dgamma, dbeta, accumulate, ws, ws_bytes, st));
  PP_CHECK_ARG(ok, "layernorm_param_grads: reduction not launchable");
  return check_launch("layernorm_param_grads");
}

extern "C" int pc_embedding_fwd(int dtype, int64_t T_, int64_t d, int64_t seq,
                                const int32_t* tokens, const float* wte, const float* wpe,
                                void* out, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (T_ <= 0) return PC_OK;
  PP_DISPATCH_FB(dtype, T, embed_fwd_kernel<T><<<row_blocks(T_), 256, 0, st>>>(T_, (int)d, (int)seq, tokens, wte, wpe, static_cast<T*>(out)));
  return check_launch("embedding_fwd");
}

static size_t cub_sort_bytes(int n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, n);
  return bytes;
}

extern "C" int pc_embedding_bwd_workspace_bytes(int64_t T_, int64_t* bytes) {
  PP_CHECK_ARG(T_ > 0 && T_ < (1ll << 31), "embedding_bwd: bad token count");
  *bytes = static_cast<int64_t>(3 * ((T_ * 4 + 255) / 256 * 256) + cub_sort_bytes((int)T_) + 256);
  return PC_OK;
}

extern "C" int pc_embedding_bwd(int dtype, int64_t T_, int64_t d, int64_t seq, int64_t vocab,
                                const int32_t* tokens, const void* dh, float* dwte, float* dwpe,
                                void* workspace, int64_t ws_bytes, void* stream) {
  return pc_embedding_bwd_acc(dtype, T_, d, seq, vocab, tokens, dh, dwte, dwpe, 0, workspace,
                              ws_bytes, stream);
}

extern "C" int pc_embedding_bwd_acc(int dtype, int64_t T_, int64_t d, int64_t seq,
                                    int64_t vocab, const int32_t* tokens, const void* dh,
                                    float* dwte, float* dwpe, int accumulate, void* workspace,
                                    int64_t ws_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t need = 0;
  int rc = pc_embedding_bwd_workspace_bytes(T_, &need);
  if (rc) return rc;
  PP_CHECK_ARG(ws_bytes >= need, "embedding_bwd: workspace %lld < %lld", (long long)ws_bytes, (long long)need);
  const int n = static_cast<int>(T_);
  const size_t slab = (T_ * 4 + 255) / 256 * 256;
  uint8_t* w = static_cast<uint8_t*>(workspace);
  int32_t* vals = reinterpret_cast<int32_t*>(w);
  int32_t* keys_out = reinterpret_cast<int32_t*>(w + slab);
  int32_t* vals_out = reinterpret_cast<int32_t*>(w + 2 * slab);
  void* temp = w + 3 * slab;
  size_t temp_bytes = cub_sort_bytes(n);
  int end_bit = 1;
  while ((1ll << end_bit) < vocab) ++end_bit;
  iota_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, vals);
  if (cub::DeviceRadixSort::SortPairs(temp, temp_bytes, tokens, keys_out, vals, vals_out, n, 0,
                                      end_bit, st) != cudaSuccess) {
    set_error("embedding_bwd: radix sort failed");
    return PC_ERR_CUDA;
  }
  if (!accumulate) PP_CUDA_TRY(cudaMemsetAsync(dwte, 0, static_cast<size_t>(vocab) * d * 4, st));
  PP_DISPATCH_FB(dtype, T,
    embed_bwd_wte_kernel<T><<<row_blocks(T_), 256, 0, st>>>(n, (int)d, keys_out, vals_out, static_cast<const T*>(dh), dwte, accumulate);
    if (dwpe)  // NULL: no position table (Llama)
      embed_bwd_wpe_kernel<T><<<(unsigned)((seq * d + 255) / 256), 256, 0, st>>>(T_, (int)d, (int)seq, static_cast<const T*>(dh), dwpe, accumulate));
  return check_launch("embedding_bwd");
}

extern "C" int pc_xent_fwd_bwd(int dtype, int64_t rows, int64_t V, int64_t seq, void* logits,
                               int64_t ld, const int32_t* tokens, float* row_loss, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0) return PC_OK;
  PP_CHECK_ARG(rows % seq == 0, "xent: rows must be a multiple of seq");
  if (dtype == PC_BF16 && V % 8 == 0 && ld % 8 == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0) {
    xent_bf16_vec_kernel<<<(unsigned)rows, 512, 0, st>>>(rows, (int)V, (int)seq, static_cast<__nv_bfloat16*>(logits), ld, tokens, row_loss);
    return check_launch("xent_vec");
  }
  PP_DISPATCH_FB(dtype, T, xent_kernel<T><<<(unsigned)rows, 512, 0, st>>>(rows, (int)V, (int)seq, static_cast<T*>(logits), ld, tokens, row_loss));
  return check_launch("xent");
}

namespace pp200 {
template <typename T, int N>
int launch_ln_partials(unsigned nb, size_t smem, cudaStream_t st, int64_t rows, int64_t d,
                       int64_t chunk, const void* dy, const void* x, const float* gamma,
                       const float* mean, const float* rstd, const T* dr, void* dx, float* pg,
                       float* pb) {
  static bool attr = false;
  if (!attr) {
    PP_CUDA_TRY(cudaFuncSetAttribute(ln_bwd_partials_vec<T, N>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    attr = true;
  }
  ln_bwd_partials_vec<T, N><<<nb, 256, smem, st>>>(rows, (int)d, chunk, static_cast<const T*>(dy),
                                                   static_cast<const T*>(x), gamma, mean, rstd, dr,
                                                   static_cast<T*>(dx), pg, pb);
  return PC_OK;
}
}  // namespace pp200

// Number of partial rows pc_layernorm_bwd_partials writes per quantity.
extern "C" int pc_layernorm_partial_rows(int64_t rows, int64_t d, int64_t* n) {
  PP_CHECK_ARG(rows > 0 && d > 0 && n, "layernorm_partial_rows: bad args");
  int64_t r = 4 * static_cast<int64_t>(num_sms());
  const int64_t cap = (rows + 7) / 8;
  *n = r < cap ? r : cap;
  return PC_OK;
}

extern "C" int pc_layernorm_bwd_partials(int dtype, int64_t rows, int64_t d, const void* dy,
                                         const void* x, const float* gamma, const float* mean,
                                         const float* rstd, const void* dres, void* dx,
                                         float* partials, int64_t n_part, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0) return PC_OK;
  PP_CHECK_ARG(dtype == PC_BF16 || dtype == PC_F32, "layernorm_bwd_partials: f32/bf16 only");
  PP_CHECK_ARG(partials != nullptr && n_part > 0, "layernorm_bwd_partials: bad partials");
  const int64_t chunk = (rows + n_part - 1) / n_part;
  bool ok = true;
  PP_DISPATCH_FB(dtype, T,
    if (!ln_vec_ok<T>(d, dy, x, dx) ||
        ((reinterpret_cast<uintptr_t>(gamma) | reinterpret_cast<uintptr_t>(dres)) & 31) != 0) {
      ok = false;
    } else {
      const int nch = static_cast<int>(d / 256);
      const size_t smem = static_cast<size_t>(8) * 2 * nch * 256 * 4;
      const T* dr = static_cast<const T*>(dres);
      float* pg = partials;
      float* pb = partials + n_part * d;
      const unsigned nb = static_cast<unsigned>(n_part);
      int rc = PC_OK;
      switch (nch) {
        case 1: rc = launch_ln_partials<T, 1>(nb, smem, st, rows, d, chunk, dy, x, gamma, mean, rstd, dr, dx, pg, pb); break;
        case 2: rc = launch_ln_partials<T, 2>(nb, smem, st, rows, d, chunk, dy, x, gamma, mean, rstd, dr, dx, pg, pb); break;
        case 3: rc = launch_ln_partials<T, 3>(nb, smem, st, rows, d, chunk, dy, x, gamma, mean, rstd, dr, dx, pg, pb); break;
        default: rc = launch_ln_partials<T, 4>(nb, smem, st, rows, d, chunk, dy, x, gamma, mean, rstd, dr, dx, pg, pb); break;
      }
      if (rc) return rc;
    });
  PP_CHECK_ARG(ok, "layernorm_bwd_partials: needs 32 B aligned rows with d %% 256 == 0 (d <= 1024)");
  return check_launch("layernorm_bwd_partials");
}
