// Throughput per SM per clock of MUFU ex2 / tanh (fp32 and packed half
// types) and of the paired FMA pipe (FFMA2), for the attention softmax
// design.  One "op" = one result element.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
__device__ __forceinline__ float tanh_mufu(float x) { float y; asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2_mufu(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2_h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2_bf2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
template <int OP>
__global__ void k(float* out, int iters) {
  float a[8];
  uint32_t h[8];
  uint64_t p[8];
  for (int i = 0; i < 8; ++i) { a[i] = 0.001f * (threadIdx.x + i); h[i] = 0x3c003c00u ^ i; p[i] = (uint64_t)__float_as_uint(a[i]) << 32 | __float_as_uint(a[i]); }
  const uint64_t m = 0x3f8000003f800000ull, c = 0x3a83126f3a83126full;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = tanh_mufu(a[i]);
      else if (OP == 1) a[i] = ex2_mufu(a[i]) - 1.0f;
      else if (OP == 2) h[i] = ex2_h2(h[i]) ^ 0x80008000u;
      else if (OP == 3) h[i] = ex2_bf2(h[i]) ^ 0x80008000u;
      else p[i] = ffma2(p[i], m, c);
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + h[i] + (float)p[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[5] = {"tanh.approx", "ex2.approx.f32", "ex2.f16x2", "ex2.bf16x2", "fma.f32x2"};
  const int per[5] = {1, 1, 2, 2, 2};
  for (int op = 0; op < 5; ++op) {
    const int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(s);
      if (op == 0) k<0><<<blocks, threads>>>(o, iters);
      else if (op == 1) k<1><<<blocks, threads>>>(o, iters);
      else if (op == 2) k<2><<<blocks, threads>>>(o, iters);
      else if (op == 3) k<3><<<blocks, threads>>>(o, iters);
      else k<4><<<blocks, threads>>>(o, iters);
      cudaEventRecord(e); cudaEventSynchronize(e);
      cudaEventElapsedTime(&ms, s, e);
    }
    double ops = double(blocks) * threads * iters * 8 * per[op];
    printf("%-16s %.2f Gop/s = %.2f results per SM per clock (at %d MHz)\n", names[op], ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
