// Llama-style block pieces (BASELINE config C5): RMSNorm, rotary position
// embedding, SwiGLU, and the grouped-query K/V expand / group-sum used around
// the attention kernels.  Semantics: oracle/llama.py (float64 restatement,
// pinned by finite differences and torch autograd in tests/test_oracle.py).
//
// All kernels are row-parallel and memory-bound (HBM roofline).  bf16 rows
// whose widths are multiples of 8 take vectorised paths (16-byte loads and
// stores, coalesced across a warp): one warp per row for the norms, one block
// per row for RoPE (the row's cos / sin table computed once into shared
// memory from fp64 angles, then 8 frequencies of one head per thread), 8
// columns per thread for SwiGLU.  fp32 (parity mode) keeps the scalar kernels.
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

using bf16 = __nv_bfloat16;

__device__ __forceinline__ void unpack8(const uint4& u, float* v) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(h[k]);
    v[2 * k] = f.x;
    v[2 * k + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
  return u;
}
__device__ __forceinline__ void load_g8(const float* g, float* v) {
  const float4 a = reinterpret_cast<const float4*>(g)[0], b = reinterpret_cast<const float4*>(g)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// bf16, d % 8 == 0: warp per row, 16-byte chunks
__global__ void __launch_bounds__(256) rms_fwd_vec(int64_t rows, int d, const bf16* __restrict__ x,
                                                   const float* __restrict__ g, bf16* __restrict__ y,
                                                   float* __restrict__ rstd, float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * static_cast<int64_t>(RMS_ROWS_PER_BLOCK) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + r * d);
  const int nc = d / 8;
  float ss = 0.f;
  for (int c = lane; c < nc; c += 32) {
    float v[8];
    unpack8(xr[c], v);
#pragma unroll
    for (int k = 0; k < 8; ++k) ss = fmaf(v[k], v[k], ss);
  }
  ss = warp_sum(ss);
  const float rs = rsqrtf(ss / d + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + r * d);
  for (int c = lane; c < nc; c += 32) {
    float v[8], gv[8];
    unpack8(xr[c], v);
    load_g8(g + 8 * c, gv);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = v[k] * rs * gv[k];
    yr[c] = pack8(v);
  }
  if (lane == 0) rstd[r] = rs;
}

// bf16, d % 8 == 0: dx = dres + rstd * (dy*g - xh * mean(dy*g*xh))
__global__ void __launch_bounds__(256) rms_bwd_dx_vec(int64_t rows, int d, const bf16* __restrict__ dy,
                                                      const bf16* __restrict__ x,
                                                      const float* __restrict__ g,
                                                      const float* __restrict__ rstd,
                                                      const bf16* __restrict__ dres,
                                                      bf16* __restrict__ dx) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * static_cast<int64_t>(RMS_ROWS_PER_BLOCK) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float rs = rstd[r];
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + r * d);
  const uint4* xr = reinterpret_cast<const uint4*>(x + r * d);
  const int nc = d / 8;
  float s = 0.f;
  for (int c = lane; c < nc; c += 32) {
    float a[8], b[8], gv[8];
    unpack8(dyr[c], a);
    unpack8(xr[c], b);
    load_g8(g + 8 * c, gv);
#pragma unroll
    for (int k = 0; k < 8; ++k) s = fmaf(a[k] * gv[k], b[k] * rs, s);
  }
  const float m = warp_sum(s) / d;
  uint4* dxr = reinterpret_cast<uint4*>(dx + r * d);
  const uint4* drr = dres ? reinterpret_cast<const uint4*>(dres + r * d) : nullptr;
  for (int c = lane; c < nc; c += 32) {
    float a[8], b[8], gv[8], o[8];
    unpack8(dyr[c], a);
    unpack8(xr[c], b);
    load_g8(g + 8 * c, gv);
    if (drr) {
      unpack8(drr[c], o);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] += rs * (a[k] * gv[k] - b[k] * rs * m);
    dxr[c] = pack8(o);
  }
}

// bf16, head_dim % 16 == 0, ld % 8 == 0: one block per row.  The row's
// (cos, sin) per frequency come from fp64 angles (exact for large positions),
// computed once into shared memory; each thread then rotates 8 frequencies of
// one head with two 16-byte loads and stores.
__global__ void __launch_bounds__(128) rope_row_vec(int n_heads, int hd, bf16* __restrict__ t,
                                                    int64_t ld, const int32_t* __restrict__ pos,
                                                    double log2_theta, int inverse) {
  __shared__ float2 cs[128];  // hd <= 256
  const int half = hd / 2;
  const int64_t r = blockIdx.x;
  const double p = static_cast<double>(pos[r]);
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    double sd, cd;
    sincos(p * exp2(-2.0 * i / hd * log2_theta), &sd, &cd);
    cs[i] = make_float2(static_cast<float>(cd), static_cast<float>(inverse ? -sd : sd));
  }
  __syncthreads();
  const int per_head = half / 8;
  bf16* row = t + r * ld;
  for (int ch = threadIdx.x; ch < n_heads * per_head; ch += blockDim.x) {
    const int h = ch / per_head, i0 = (ch % per_head) * 8;
    uint4* pa = reinterpret_cast<uint4*>(row + h * hd + i0);
    uint4* pb = reinterpret_cast<uint4*>(row + h * hd + half + i0);
    float a[8], b[8], oa[8], ob[8];
    unpack8(*pa, a);
    unpack8(*pb, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float2 q = cs[i0 + k];
      oa[k] = a[k] * q.x - b[k] * q.y;
      ob[k] = b[k] * q.x + a[k] * q.y;
    }
    *pa = pack8(oa);
    *pb = pack8(ob);
  }
}

__device__ __forceinline__ float sigmoid_fast(float g) { return 1.f / (1.f + __expf(-g)); }

// bf16, f % 8 == 0 and 16-byte aligned rows: 8 columns per thread
__global__ void swiglu_fwd_vec(int64_t rows, int f, const bf16* __restrict__ gu, int64_t ld_gu,
                               bf16* __restrict__ m, int64_t ld_m) {
  const int nc = f / 8;
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * nc) return;
  const int64_t r = idx / nc;
  const int c = static_cast<int>(idx % nc) * 8;
  float g[8], u[8], o[8];
  unpack8(*reinterpret_cast<const uint4*>(gu + r * ld_gu + c), g);
  unpack8(*reinterpret_cast<const uint4*>(gu + r * ld_gu + f + c), u);
#pragma unroll
  for (int k = 0; k < 8; ++k) o[k] = g[k] * sigmoid_fast(g[k]) * u[k];
  *reinterpret_cast<uint4*>(m + r * ld_m + c) = pack8(o);
}

__global__ void swiglu_bwd_vec(int64_t rows, int f, const bf16* __restrict__ gu, int64_t ld_gu,
                               const bf16* __restrict__ dm, int64_t ld_dm, bf16* __restrict__ dgu,
                               int64_t ld_dgu) {
  const int nc = f / 8;
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * nc) return;
  const int64_t r = idx / nc;
  const int c = static_cast<int>(idx % nc) * 8;
  float g[8], u[8], d[8], dg[8], du[8];
  unpack8(*reinterpret_cast<const uint4*>(gu + r * ld_gu + c), g);
  unpack8(*reinterpret_cast<const uint4*>(gu + r * ld_gu + f + c), u);
  unpack8(*reinterpret_cast<const uint4*>(dm + r * ld_dm + c), d);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float sg = sigmoid_fast(g[k]);
    dg[k] = d[k] * u[k] * (sg * (1.f + g[k] * (1.f - sg)));
    du[k] = d[k] * g[k] * sg;
  }
  *reinterpret_cast<uint4*>(dgu + r * ld_dgu + c) = pack8(dg);
  *reinterpret_cast<uint4*>(dgu + r * ld_dgu + f + c) = pack8(du);
}

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

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
  if (dtype == PC_BF16 && d % 8 == 0 && al16(x) && al16(y) && al16(gamma)) {
    rms_fwd_vec<<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const bf16*>(x), gamma,
                                    static_cast<bf16*>(y), rstd, eps);
    return check_launch("rmsnorm_fwd");
  }
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
  const bool vec = dtype == PC_BF16 && d % 8 == 0 && al16(dy) && al16(x) && al16(dx) &&
                   al16(gamma) && (dres == nullptr || al16(dres));
  // dgamma == NULL: dx only (the gain gradient then comes from
  // pc_layernorm_param_grads with mean = NULL, e.g. on another stream)
  PP_DISPATCH_FB2(dtype, T,
    if (vec)
      rms_bwd_dx_vec<<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const bf16*>(dy), static_cast<const bf16*>(x), gamma, rstd, static_cast<const bf16*>(dres), static_cast<bf16*>(dx));
    else
      rms_bwd_dx_kernel<T><<<nb, 256, 0, st>>>(rows, (int)d, static_cast<const T*>(dy), static_cast<const T*>(x), gamma, rstd, static_cast<const T*>(dres), static_cast<T*>(dx));
    // dgamma = sum_rows dy * x * rstd: the LayerNorm-statistics reduction without a mean
    if (dgamma)
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
  if (dtype == PC_BF16 && head_dim % 16 == 0 && head_dim <= 256 && ld % 8 == 0 && al16(t)) {
    rope_row_vec<<<static_cast<unsigned>(rows), 128, 0, st>>>(
        (int)n_heads, (int)head_dim, static_cast<bf16*>(t), ld, pos, log2(static_cast<double>(theta)),
        inverse);
    return check_launch("rope");
  }
  PP_DISPATCH_FB2(dtype, T, rope_kernel<T><<<blocks_for(n, 256), 256, 0, st>>>(rows, (int)n_heads, (int)head_dim, static_cast<T*>(t), ld, pos, log2(static_cast<double>(theta)), inverse));
  return check_launch("rope");
}

extern "C" int pc_swiglu_fwd(int dtype, int64_t rows, int64_t f, const void* gu, int64_t ld_gu,
                             void* m, int64_t ld_m, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0 || f <= 0) return PC_OK;
  if (dtype == PC_BF16 && f % 8 == 0 && ld_gu % 8 == 0 && ld_m % 8 == 0 && al16(gu) && al16(m)) {
    swiglu_fwd_vec<<<blocks_for(rows * (f / 8), 256), 256, 0, st>>>(
        rows, (int)f, static_cast<const bf16*>(gu), ld_gu, static_cast<bf16*>(m), ld_m);
    return check_launch("swiglu_fwd");
  }
  PP_DISPATCH_FB2(dtype, T, swiglu_fwd_kernel<T><<<blocks_for(rows * f, 256), 256, 0, st>>>(rows, (int)f, static_cast<const T*>(gu), ld_gu, static_cast<T*>(m), ld_m));
  return check_launch("swiglu_fwd");
}

extern "C" int pc_swiglu_bwd(int dtype, int64_t rows, int64_t f, const void* gu, int64_t ld_gu,
                             const void* dm, int64_t ld_dm, void* dgu, int64_t ld_dgu, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= 0 || f <= 0) return PC_OK;
  if (dtype == PC_BF16 && f % 8 == 0 && ld_gu % 8 == 0 && ld_dm % 8 == 0 && ld_dgu % 8 == 0 &&
      al16(gu) && al16(dm) && al16(dgu)) {
    swiglu_bwd_vec<<<blocks_for(rows * (f / 8), 256), 256, 0, st>>>(
        rows, (int)f, static_cast<const bf16*>(gu), ld_gu, static_cast<const bf16*>(dm), ld_dm,
        static_cast<bf16*>(dgu), ld_dgu);
    return check_launch("swiglu_bwd");
  }
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
