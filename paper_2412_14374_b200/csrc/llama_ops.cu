// Llama-style block pieces (BASELINE config C5): RMSNorm, rotary position
// embedding, SwiGLU, and the grouped-query K/V expand / group-sum used around
// the attention kernels.  Semantics: oracle/llama.py (float64 restatement,
// pinned by finite differences and torch autograd in tests/test_oracle.py).
//
// All kernels are row-parallel and memory-bound (HBM roofline); one warp per
// row for the norms, one thread per (row, frequency) for RoPE.
#include "common.cuh"

namespace pp200 {

template <typename T>
bool colred_launch(int mode, int64_t rows, int64_t cols, const T* a, int64_t lda, const T* x,
                   const float* mean, const float* rstd, float* out1, float* out2,
                   int accumulate, void* ws, int64_t ws_bytes, cudaStream_t st);

namespace {

constexpr int RMS_ROWS_PER_BLOCK = 8;  // one warp per row

template <typename T>
__global__ void __launch_bounds__(256) rms_fwd_kernel(int64_t rows, int d, const T* __restrict__ x,
                                                      const float* __restrict__ g,
                                                      T* __restrict__ y, float* __restrict__ rstd,
                                                      float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * static_cast<int64_t>(RMS_ROWS_PER_BLOCK) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const T* xr = x + r * d;
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float v = Io<T>::ld(xr + c);
    ss = fmaf(v, v, ss);
  }
  ss = warp_sum(ss);
  const float rs = rsqrtf(ss / d + eps);
  T* yr = y + r * d;
  for (int c = lane; c < d; c += 32) Io<T>::st(yr + c, Io<T>::ld(xr + c) * rs * g[c]);
  if (lane == 0) rstd[r] = rs;
}

// dx = dres + rstd * (dy*g - xh * mean(dy*g*xh)),  xh = x * rstd
template <typename T>
__global__ void __launch_bounds__(256) rms_bwd_dx_kernel(int64_t rows, int d, const T* __restrict__ dy,
                                                         const T* __restrict__ x,
                                                         const float* __restrict__ g,
                                                         const float* __restrict__ rstd,
                                                         const T* __restrict__ dres,
                                                         T* __restrict__ dx) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * static_cast<int64_t>(RMS_ROWS_PER_BLOCK) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float rs = rstd[r];
  const T* dyr = dy + r * d;
  const T* xr = x + r * d;
  float s = 0.f;
  for (int c = lane; c < d; c += 32)
    s = fmaf(Io<T>::ld(dyr + c) * g[c], Io<T>::ld(xr + c) * rs, s);
  const float m = warp_sum(s) / d;
  T* dxr = dx + r * d;
  for (int c = lane; c < d; c += 32) {
    float v = rs * (Io<T>::ld(dyr + c) * g[c] - Io<T>::ld(xr + c) * rs * m);
    if (dres) v += Io<T>::ld(dres + r * d + c);
    Io<T>::st(dxr + c, v);
  }
}

// In-place rotate-half RoPE on n_heads consecutive heads of each row:
// (t1, t2) -> (t1 c - t2 s, t2 c + t1 s), angle = pos * theta^(-2i/hd); the
// inverse (transpose) rotation negates s.  Angles in double precision: fp32
// parity holds for large positions.
template <typename T>
__global__ void rope_kernel(int64_t rows, int n_heads, int hd, T* __restrict__ t, int64_t ld,
                            const int32_t* __restrict__ pos, double log2_theta, int inverse) {
  const int half = hd / 2;
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * half) return;
  const int64_t r = idx / half;
  const int i = static_cast<int>(idx % half);
  const double ang = static_cast<double>(pos[r]) * exp2(-2.0 * i / hd * log2_theta);
  double sd, cd;
  sincos(ang, &sd, &cd);
  const float c = static_cast<float>(cd), s = static_cast<float>(inverse ? -sd : sd);
  T* row = t + r * ld;
  for (int h = 0; h < n_heads; ++h) {
    T* p = row + h * hd;
    const float a = Io<T>::ld(p + i), b = Io<T>::ld(p + i + half);
    Io<T>::st(p + i, a * c - b * s);
    Io<T>::st(p + i + half, b * c + a * s);
  }
}

__device__ __forceinline__ float sigmoid_f(float g) { return 1.f / (1.f + expf(-g)); }

// m = silu(g) * u with gu = [g | u] (f columns each)
template <typename T>
__global__ void swiglu_fwd_kernel(int64_t rows, int f, const T* __restrict__ gu, int64_t ld_gu,
                                  T* __restrict__ m, int64_t ld_m) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * f) return;
  const int64_t r = idx / f;
  const int j = static_cast<int>(idx % f);
  const float g = Io<T>::ld(gu + r * ld_gu + j), u = Io<T>::ld(gu + r * ld_gu + f + j);
  Io<T>::st(m + r * ld_m + j, g * sigmoid_f(g) * u);
}

// dg = dm * u * silu'(g), du = dm * silu(g);  silu'(g) = sig(g) (1 + g (1 - sig(g)))
template <typename T>
__global__ void swiglu_bwd_kernel(int64_t rows, int f, const T* __restrict__ gu, int64_t ld_gu,
                                  const T* __restrict__ dm, int64_t ld_dm, T* __restrict__ dgu,
                                  int64_t ld_dgu) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * f) return;
  const int64_t r = idx / f;
  const int j = static_cast<int>(idx % f);
  const float g = Io<T>::ld(gu + r * ld_gu + j), u = Io<T>::ld(gu + r * ld_gu + f + j);
  const float d = Io<T>::ld(dm + r * ld_dm + j);
  const float sg = sigmoid_f(g);
  Io<T>::st(dgu + r * ld_dgu + j, d * u * (sg * (1.f + g * (1.f - sg))));
  Io<T>::st(dgu + r * ld_dgu + f + j, d * g * sg);
}

// Grouped-query K/V: expand [q(H) | k(Hkv) | v(Hkv)] heads to [q(H) | k(H) | v(H)]
// (query head h reads kv head h / G), or reduce the gradient back: dk, dv of
// each kv head = sum over its G query heads in ascending order (deterministic).
template <typename T>
__global__ void gqa_kv_kernel(int64_t rows, int H, int Hkv, int hd, const T* __restrict__ src,
                              int64_t ld_src, T* __restrict__ dst, int64_t ld_dst, int reduce) {
  const int G = H / Hkv;
  const int ncol = reduce ? (H + 2 * Hkv) * hd : 3 * H * hd;  // destination columns
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * ncol) return;
  const int64_t r = idx / ncol;
  const int c = static_cast<int>(idx % ncol);
  const T* s = src + r * ld_src;
  float v;
  if (!reduce) {
    if (c < H * hd) {
      v = Io<T>::ld(s + c);  // q
    } else {
      const int part = (c - H * hd) / (H * hd);  // 0: k, 1: v
      const int cc = (c - H * hd) % (H * hd);
      const int h = cc / hd, e = cc % hd;
      v = Io<T>::ld(s + (H + part * Hkv + h / G) * hd + e);
    }
  } else {
    if (c < H * hd) {
      v = Io<T>::ld(s + c);  // dq
    } else {
      const int part = (c - H * hd) / (Hkv * hd);  // 0: dk, 1: dv
      const int cc = (c - H * hd) % (Hkv * hd);
      const int kvh = cc / hd, e = cc % hd;
      v = 0.f;
      for (int gi = 0; gi < G; ++gi) v += Io<T>::ld(s + (H + part * H + kvh * G + gi) * hd + e);
    }
  }
  Io<T>::st(dst + r * ld_dst + c, v);
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace
}  // namespace pp200

using namespace pp200;

#define PP_DISPATCH_FB2(dtype, T, ...)                                \
  switch (dtype) {                                                    \
    case PC_F32: { using T = float; __VA_ARGS__; break; }            \
    case PC_BF16: { using T = __nv_bfloat16; __VA_ARGS__; break; }   \
    default: set_error("unsupported dtype %d (f32/bf16 only)", dtype); return PC_ERR_UNSUPPORTED; \
  }

extern "C" int pc_rmsnorm_fwd(int dtype, int64_t rows, int64_t d, const void* x, const float* gamma,
                              void* y, float* rstd, float eps, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0) return PC_OK;
  PP_CHECK_ARG(d > 0, "rmsnorm: bad width");
  const unsigned nb = blocks_for(rows, RMS_ROWS_PER_BLOCK);
  PP_DISPATCH_FB2(dtype, T, rms_fwd_kernel<T><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(x), gamma, static_cast<T*>(y), rstd, eps));
  return check_launch("rmsnorm_fwd");
}

extern "C" int pc_rmsnorm_bwd(int dtype, int64_t rows, int64_t d, const void* dy, const void* x,
                              const float* gamma, const float* rstd, const void* dres, void* dx,
                              float* dgamma, void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0) return PC_OK;
  PP_CHECK_ARG(d > 0, "rmsnorm: bad width");
  const unsigned nb = blocks_for(rows, RMS_ROWS_PER_BLOCK);
  bool ok = true;
  PP_DISPATCH_FB2(dtype, T,
    rms_bwd_dx_kernel<T><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(dy), static_cast<const T*>(x), gamma, rstd, static_cast<const T*>(dres), static_cast<T*>(dx));
    // dgamma = sum_rows dy * x * rstd: the LayerNorm-statistics reduction without a mean
    ok = colred_launch<T>(1, rows, d, static_cast<const T*>(dy), d, static_cast<const T*>(x), nullptr, rstd, dgamma, nullptr, 0, ws, ws_bytes, st));
  if (!ok) {
    set_error("rmsnorm_bwd: reduction workspace too small (pc_reduce_workspace_bytes)");
    return PC_ERR_ARG;
  }
  return check_launch("rmsnorm_bwd");
}

extern "C" int pc_rope(int dtype, int64_t rows, int64_t n_heads, int64_t head_dim, void* t,
                       int64_t ld, const int32_t* pos, float theta, int inverse, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0 || n_heads <= 0) return PC_OK;
  PP_CHECK_ARG(head_dim > 0 && head_dim % 2 == 0, "rope: head_dim must be even");
  PP_CHECK_ARG(theta > 1.f, "rope: theta must exceed 1");
  const int64_t n = rows * (head_dim / 2);
  PP_DISPATCH_FB2(dtype, T, rope_kernel<T><<<blocks_for(n, 256), 256, 0, st>>>(rows, (int)n_heads, (int)head_dim, static_cast<T*>(t), ld, pos, log2(static_cast<double>(theta)), inverse));
  return check_launch("rope");
}

extern "C" int pc_swiglu_fwd(int dtype, int64_t rows, int64_t f, const void* gu, int64_t ld_gu,
                             void* m, int64_t ld_m, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0 || f <= 0) return PC_OK;
  PP_DISPATCH_FB2(dtype, T, swiglu_fwd_kernel<T><<<blocks_for(rows * f, 256), 256, 0, st>>>(rows, (int)f, static_cast<const T*>(gu), ld_gu, static_cast<T*>(m), ld_m));
  return check_launch("swiglu_fwd");
}

extern "C" int pc_swiglu_bwd(int dtype, int64_t rows, int64_t f, const void* gu, int64_t ld_gu,
                             const void* dm, int64_t ld_dm, void* dgu, int64_t ld_dgu, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0 || f <= 0) return PC_OK;
  PP_DISPATCH_FB2(dtype, T, swiglu_bwd_kernel<T><<<blocks_for(rows * f, 256), 256, 0, st>>>(rows, (int)f, static_cast<const T*>(gu), ld_gu, static_cast<const T*>(dm), ld_dm, static_cast<T*>(dgu), ld_dgu));
  return check_launch("swiglu_bwd");
}

extern "C" int pc_gqa_kv(int dtype, int64_t rows, int64_t n_heads, int64_t n_kv_heads,
                         int64_t head_dim, const void* src, int64_t ld_src, void* dst,
                         int64_t ld_dst, int reduce, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0) return PC_OK;
  PP_CHECK_ARG(n_kv_heads > 0 && n_heads % n_kv_heads == 0, "gqa: heads must be a multiple of kv heads");
  const int64_t ncol = reduce ? (n_heads + 2 * n_kv_heads) * head_dim : 3 * n_heads * head_dim;
  PP_DISPATCH_FB2(dtype, T, gqa_kv_kernel<T><<<blocks_for(rows * ncol, 256), 256, 0, st>>>(rows, (int)n_heads, (int)n_kv_heads, (int)head_dim, static_cast<const T*>(src), ld_src, static_cast<T*>(dst), ld_dst, reduce));
  return check_launch("gqa_kv");
}
