// Causal multi-head attention, exact (SIMT, fp32 math), any head_dim <= 256.
//
// Reference semantics: oracle/gpt.py attention / attention_bwd.  This is the
// generic path used in fp32 mode and as the parity anchor for the
// tensor-core flash-attention kernels (attention_tc.cu).  One warp owns one
// query row (forward, dQ) or one key row (dK, dV); online softmax keeps the
// forward single-pass; the backward recomputes probabilities from the saved
// log-sum-exp, and dQ / dK,dV are separate passes so no atomics are needed
// (bitwise deterministic).
//
// Layout: qkv is [B*S, ld_qkv] with q at columns [h*hd, (h+1)*hd), k at
// d + h*hd, v at 2d + h*hd (d = H*hd); o / dO are [B*S, ld_o] with head h at
// h*hd; lse / delta are [B, H, S] fp32.
#include "common.cuh"

namespace pp200 {
namespace {

constexpr int MAXE = 8;  // head_dim / 32 upper bound (hd <= 256)

template <typename T> __device__ __forceinline__ float lf(const T* p, int64_t i) {
  return static_cast<float>(p[i]);
}
template <> __device__ __forceinline__ float lf(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}
template <typename T> __device__ __forceinline__ void sf(T* p, int64_t i, float v) {
  p[i] = static_cast<T>(v);
}
template <> __device__ __forceinline__ void sf(__nv_bfloat16* p, int64_t i, float v) {
  p[i] = __float2bfloat16_rn(v);
}

struct AttnDims {
  int B, H, S, hd;
  int64_t ld_qkv, ld_o;
  float scale;
};

template <typename T>
__global__ void __launch_bounds__(256) attn_fwd_simt(AttnDims a, const T* __restrict__ qkv,
                                                     T* __restrict__ o, float* __restrict__ lse) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = blockIdx.x * 8ll + (threadIdx.x >> 5);  // global (b, h, i)
  if (gw >= static_cast<int64_t>(a.B) * a.H * a.S) return;
  const int i = static_cast<int>(gw % a.S);
  const int h = static_cast<int>((gw / a.S) % a.H);
  const int b = static_cast<int>(gw / (static_cast<int64_t>(a.S) * a.H));
  const int d = a.H * a.hd;
  const int ne = (a.hd + 31) / 32;
  const T* base = qkv + static_cast<int64_t>(b) * a.S * a.ld_qkv;
  float q[MAXE], acc[MAXE];
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int c = lane + 32 * e;
    q[e] = (e < ne && c < a.hd) ? lf(base, i * a.ld_qkv + h * a.hd + c) * a.scale : 0.f;
    acc[e] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int j = 0; j <= i; ++j) {
    const T* kr = base + j * a.ld_qkv + d + h * a.hd;
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int c = lane + 32 * e;
      if (e < ne && c < a.hd) s += q[e] * lf(kr, c);
    }
    s = warp_sum(s);
    const float mn = fmaxf(m, s);
    const float corr = __expf(m - mn), p = __expf(s - mn);
    l = l * corr + p;
    const T* vr = base + j * a.ld_qkv + 2 * d + h * a.hd;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int c = lane + 32 * e;
      if (e < ne && c < a.hd) acc[e] = acc[e] * corr + p * lf(vr, c);
    }
    m = mn;
  }
  T* orow = o + (static_cast<int64_t>(b) * a.S + i) * a.ld_o + h * a.hd;
  const float inv = 1.f / l;
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int c = lane + 32 * e;
    if (e < ne && c < a.hd) sf(orow, c, acc[e] * inv);
  }
  if (lane == 0) lse[gw] = m + logf(l);
}

// delta[b,h,i] = sum_c dO[i,c] * O[i,c]: one warp per token row walks all
// heads (contiguous, coalesced reads of the whole row).
template <typename T>
__global__ void __launch_bounds__(256) attn_delta(AttnDims a, const T* __restrict__ o,
                                                  const T* __restrict__ dO,
                                                  float* __restrict__ delta) {
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * 8ll + (threadIdx.x >> 5);  // b*S + i
  if (row >= static_cast<int64_t>(a.B) * a.S) return;
  const int b = static_cast<int>(row / a.S), i = static_cast<int>(row % a.S);
  const T* orow = o + row * a.ld_o;
  const T* grow = dO + row * a.ld_o;
  for (int h = 0; h < a.H; ++h) {
    float s = 0.f;
    for (int c = lane; c < a.hd; c += 32) s += lf(orow, h * a.hd + c) * lf(grow, h * a.hd + c);
    s = warp_sum(s);
    if (lane == 0) delta[(static_cast<int64_t>(b) * a.H + h) * a.S + i] = s;
  }
}

// dQ_i = scale * sum_{j<=i} p_ij (dp_ij - delta_i) k_j
template <typename T>
__global__ void __launch_bounds__(256) attn_bwd_dq_simt(AttnDims a, const T* __restrict__ qkv,
                                                        const T* __restrict__ dO,
                                                        const float* __restrict__ lse,
                                                        const float* __restrict__ delta,
                                                        T* __restrict__ dqkv, int64_t ld_dqkv) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = blockIdx.x * 8ll + (threadIdx.x >> 5);
  if (gw >= static_cast<int64_t>(a.B) * a.H * a.S) return;
  const int i = static_cast<int>(gw % a.S);
  const int h = static_cast<int>((gw / a.S) % a.H);
  const int b = static_cast<int>(gw / (static_cast<int64_t>(a.S) * a.H));
  const int d = a.H * a.hd;
  const int ne = (a.hd + 31) / 32;
  const T* base = qkv + static_cast<int64_t>(b) * a.S * a.ld_qkv;
  const T* dob = dO + (static_cast<int64_t>(b) * a.S + i) * a.ld_o + h * a.hd;
  float q[MAXE], g[MAXE], acc[MAXE];
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int c = lane + 32 * e;
    const bool ok = e < ne && c < a.hd;
    q[e] = ok ? lf(base, i * a.ld_qkv + h * a.hd + c) * a.scale : 0.f;
    g[e] = ok ? lf(dob, c) : 0.f;
    acc[e] = 0.f;
  }
  const float L = lse[gw], D = delta[gw];
  for (int j = 0; j <= i; ++j) {
    const T* kr = base + j * a.ld_qkv + d + h * a.hd;
    const T* vr = base + j * a.ld_qkv + 2 * d + h * a.hd;
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int c = lane + 32 * e;
      if (e < ne && c < a.hd) {
        s += q[e] * lf(kr, c);
        dp += g[e] * lf(vr, c);
      }
    }
    s = warp_sum(s);
    dp = warp_sum(dp);
    const float ds = __expf(s - L) * (dp - D);
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int c = lane + 32 * e;
      if (e < ne && c < a.hd) acc[e] += ds * lf(kr, c);
    }
  }
  T* out = dqkv + (static_cast<int64_t>(b) * a.S + i) * ld_dqkv + h * a.hd;
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int c = lane + 32 * e;
    if (e < ne && c < a.hd) sf(out, c, acc[e] * a.scale);
  }
}

// dV_j = sum_{i>=j} p_ij dO_i ;  dK_j = scale * sum_{i>=j} p_ij (dp_ij - delta_i) q_i
template <typename T>
__global__ void __launch_bounds__(256) attn_bwd_dkv_simt(AttnDims a, const T* __restrict__ qkv,
                                                         const T* __restrict__ dO,
                                                         const float* __restrict__ lse,
                                                         const float* __restrict__ delta,
                                                         T* __restrict__ dqkv, int64_t ld_dqkv) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = blockIdx.x * 8ll + (threadIdx.x >> 5);  // (b, h, j)
  if (gw >= static_cast<int64_t>(a.B) * a.H * a.S) return;
  const int j = static_cast<int>(gw % a.S);
  const int h = static_cast<int>((gw / a.S) % a.H);
  const int b = static_cast<int>(gw / (static_cast<int64_t>(a.S) * a.H));
  const int d = a.H * a.hd;
  const int ne = (a.hd + 31) / 32;
  const T* base = qkv + static_cast<int64_t>(b) * a.S * a.ld_qkv;
  float k[MAXE], v[MAXE], dk[MAXE], dv[MAXE];
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int c = lane + 32 * e;
    const bool ok = e < ne && c < a.hd;
    k[e] = ok ? lf(base, j * a.ld_qkv + d + h * a.hd + c) : 0.f;
    v[e] = ok ? lf(base, j * a.ld_qkv + 2 * d + h * a.hd + c) : 0.f;
    dk[e] = dv[e] = 0.f;
  }
  const int64_t row0 = (static_cast<int64_t>(b) * a.H + h) * a.S;
  for (int i = j; i < a.S; ++i) {
    const T* qr = base + i * a.ld_qkv + h * a.hd;
    const T* gr = dO + (static_cast<int64_t>(b) * a.S + i) * a.ld_o + h * a.hd;
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int c = lane + 32 * e;
      if (e < ne && c < a.hd) {
        s += lf(qr, c) * a.scale * k[e];
        dp += lf(gr, c) * v[e];
      }
    }
    s = warp_sum(s);
    dp = warp_sum(dp);
    const float p = __expf(s - lse[row0 + i]);
    const float ds = p * (dp - delta[row0 + i]);
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
      const int c = lane + 32 * e;
      if (e < ne && c < a.hd) {
        dv[e] += p * lf(gr, c);
        dk[e] += ds * lf(qr, c);
      }
    }
  }
  T* ok_ = dqkv + (static_cast<int64_t>(b) * a.S + j) * ld_dqkv + d + h * a.hd;
  T* ov_ = dqkv + (static_cast<int64_t>(b) * a.S + j) * ld_dqkv + 2 * d + h * a.hd;
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int c = lane + 32 * e;
    if (e < ne && c < a.hd) {
      sf(ok_, c, dk[e] * a.scale);
      sf(ov_, c, dv[e]);
    }
  }
}

}  // namespace

int attention_fwd_simt(int dtype, int B, int H, int S, int hd, const void* qkv, int64_t ld_qkv,
                       void* o, int64_t ld_o, float* lse, cudaStream_t st) {
  AttnDims a{B, H, S, hd, ld_qkv, ld_o, 1.f / sqrtf(static_cast<float>(hd))};
  const unsigned blocks = static_cast<unsigned>((static_cast<int64_t>(B) * H * S + 7) / 8);
  if (dtype == PC_F32)
    attn_fwd_simt<float><<<blocks, 256, 0, st>>>(a, static_cast<const float*>(qkv), static_cast<float*>(o), lse);
  else
    attn_fwd_simt<__nv_bfloat16><<<blocks, 256, 0, st>>>(a, static_cast<const __nv_bfloat16*>(qkv), static_cast<__nv_bfloat16*>(o), lse);
  return check_launch("attention_fwd_simt");
}

int attention_delta(int dtype, int B, int H, int S, int hd, const void* o, const void* dO,
                    int64_t ld_o, float* delta, cudaStream_t st) {
  AttnDims a{B, H, S, hd, 0, ld_o, 0.f};
  const unsigned blocks = static_cast<unsigned>((static_cast<int64_t>(B) * S + 7) / 8);
  if (dtype == PC_F32)
    attn_delta<float><<<blocks, 256, 0, st>>>(a, static_cast<const float*>(o), static_cast<const float*>(dO), delta);
  else
    attn_delta<__nv_bfloat16><<<blocks, 256, 0, st>>>(a, static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dO), delta);
  return check_launch("attention_delta");
}

int attention_bwd_simt(int dtype, int B, int H, int S, int hd, const void* qkv, int64_t ld_qkv,
                       const void* dO, int64_t ld_o, const float* lse, const float* delta,
                       void* dqkv, int64_t ld_dqkv, cudaStream_t st) {
  AttnDims a{B, H, S, hd, ld_qkv, ld_o, 1.f / sqrtf(static_cast<float>(hd))};
  const unsigned blocks = static_cast<unsigned>((static_cast<int64_t>(B) * H * S + 7) / 8);
  if (dtype == PC_F32) {
    attn_bwd_dq_simt<float><<<blocks, 256, 0, st>>>(a, static_cast<const float*>(qkv), static_cast<const float*>(dO), lse, delta, static_cast<float*>(dqkv), ld_dqkv);
    attn_bwd_dkv_simt<float><<<blocks, 256, 0, st>>>(a, static_cast<const float*>(qkv), static_cast<const float*>(dO), lse, delta, static_cast<float*>(dqkv), ld_dqkv);
  } else {
    attn_bwd_dq_simt<__nv_bfloat16><<<blocks, 256, 0, st>>>(a, static_cast<const __nv_bfloat16*>(qkv), static_cast<const __nv_bfloat16*>(dO), lse, delta, static_cast<__nv_bfloat16*>(dqkv), ld_dqkv);
    attn_bwd_dkv_simt<__nv_bfloat16><<<blocks, 256, 0, st>>>(a, static_cast<const __nv_bfloat16*>(qkv), static_cast<const __nv_bfloat16*>(dO), lse, delta, static_cast<__nv_bfloat16*>(dqkv), ld_dqkv);
  }
  return check_launch("attention_bwd_simt");
}

}  // namespace pp200

using namespace pp200;

static int g_attn_impl = 0;  // 0 auto (tcgen05 fwd), 1 force SIMT, 2 force mma.sync

extern "C" int pc_attention_set_impl(int impl) {
  g_attn_impl = impl;
  return PC_OK;
}

namespace pp200 {
int attention_tc5_tune(int key, int value);
}

extern "C" int pc_attention_tune(int key, int value) { return pp200::attention_tc5_tune(key, value); }

namespace pp200 {
int attention_fwd_tc(int B, int H, int S, int hd, const void* qkv, int64_t ld_qkv, void* o,
                     int64_t ld_o, float* lse, cudaStream_t st);
int attention_bwd_tc(int B, int H, int S, int hd, const void* qkv, int64_t ld_qkv, const void* o,
                     const void* dO, int64_t ld_o, const float* lse, float* delta, void* dqkv,
                     int64_t ld_dqkv, cudaStream_t st);
bool attention_tc_supported(int hd, int64_t ld_qkv, int64_t ld_o);
bool attention_tc5_supported(int hd, int H, int Hkv, int64_t ld_qkv, int64_t ld_o, const void* qkv,
                             const void* o);
int attention_fwd_tc5(int B, int H, int Hkv, int S, int hd, const void* qkv, int64_t ld_qkv, void* o,
                      int64_t ld_o, float* lse, cudaStream_t st);
int attention_bwd_tc5(int B, int H, int Hkv, int S, int hd, const void* qkv, int64_t ld_qkv,
                      const void* o, const void* dO, int64_t ld_o, const float* lse, float* delta,
                      void* dqkv, int64_t ld_dqkv, cudaStream_t st);
}  // namespace pp200

extern "C" int pc_attention_gqa_fwd(int dtype, int B, int H, int Hkv, int S, int hd,
                                    const void* qkv, int64_t ld_qkv, void* o, int64_t ld_o,
                                    float* lse, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PP_CHECK_ARG(B > 0 && H > 0 && Hkv > 0 && H % Hkv == 0 && S > 0 && hd > 0 && hd <= 32 * 8,
               "attention: bad dims");
  PP_CHECK_ARG(dtype == PC_F32 || dtype == PC_BF16, "attention: f32/bf16 only");
  if (dtype == PC_BF16 && g_attn_impl == 0 &&
      attention_tc5_supported(hd, H, Hkv, ld_qkv, ld_o, qkv, o))
    return attention_fwd_tc5(B, H, Hkv, S, hd, qkv, ld_qkv, o, ld_o, lse, st);
  if (Hkv != H) {
    set_error("attention: grouped-query heads need the tcgen05 path (bf16, head_dim 64/128)");
    return PC_ERR_UNSUPPORTED;
  }
  if (dtype == PC_BF16 && g_attn_impl != 1 && attention_tc_supported(hd, ld_qkv, ld_o))
    return attention_fwd_tc(B, H, S, hd, qkv, ld_qkv, o, ld_o, lse, st);
  return attention_fwd_simt(dtype, B, H, S, hd, qkv, ld_qkv, o, ld_o, lse, st);
}

extern "C" int pc_attention_gqa_bwd(int dtype, int B, int H, int Hkv, int S, int hd,
                                    const void* qkv, int64_t ld_qkv, const void* o, const void* dO,
                                    int64_t ld_o, const float* lse, float* delta, void* dqkv,
                                    int64_t ld_dqkv, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PP_CHECK_ARG(B > 0 && H > 0 && Hkv > 0 && H % Hkv == 0 && S > 0 && hd > 0 && hd <= 32 * 8,
               "attention: bad dims");
  PP_CHECK_ARG(dtype == PC_F32 || dtype == PC_BF16, "attention: f32/bf16 only");
  if (dtype == PC_BF16 && g_attn_impl == 0 &&
      attention_tc5_supported(hd, H, Hkv, ld_qkv, ld_o, qkv, dO) &&
      (reinterpret_cast<uintptr_t>(dqkv) & 15) == 0 && (ld_dqkv * 2) % 16 == 0 && S % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(lse) & 15) == 0 && (reinterpret_cast<uintptr_t>(delta) & 15) == 0)
    return attention_bwd_tc5(B, H, Hkv, S, hd, qkv, ld_qkv, o, dO, ld_o, lse, delta, dqkv, ld_dqkv,
                             st);
  if (Hkv != H) {
    set_error("attention: grouped-query heads need the tcgen05 path (bf16, head_dim 64/128, S %% 4 == 0)");
    return PC_ERR_UNSUPPORTED;
  }
  if (dtype == PC_BF16 && g_attn_impl != 1 && attention_tc_supported(hd, ld_qkv, ld_o))
    return attention_bwd_tc(B, H, S, hd, qkv, ld_qkv, o, dO, ld_o, lse, delta, dqkv, ld_dqkv, st);
  int rc = attention_delta(dtype, B, H, S, hd, o, dO, ld_o, delta, st);
  if (rc) return rc;
  return attention_bwd_simt(dtype, B, H, S, hd, qkv, ld_qkv, dO, ld_o, lse, delta, dqkv, ld_dqkv,
                            st);
}

extern "C" int pc_attention_fwd(int dtype, int B, int H, int S, int hd, const void* qkv,
                                int64_t ld_qkv, void* o, int64_t ld_o, float* lse, void* stream) {
  return pc_attention_gqa_fwd(dtype, B, H, H, S, hd, qkv, ld_qkv, o, ld_o, lse, stream);
}

extern "C" int pc_attention_bwd(int dtype, int B, int H, int S, int hd, const void* qkv,
                                int64_t ld_qkv, const void* o, const void* dO, int64_t ld_o,
                                const float* lse, float* delta, void* dqkv, int64_t ld_dqkv,
                                void* stream) {
  return pc_attention_gqa_bwd(dtype, B, H, H, S, hd, qkv, ld_qkv, o, dO, ld_o, lse, delta, dqkv,
                              ld_dqkv, stream);
}
