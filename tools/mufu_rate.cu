// Throughput of MUFU tanh.approx vs ex2.approx vs an FMA-pipe tanh (per SM per clock).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float tanh_mufu(float x) { float y; asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2_mufu(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
// tanh(x) = 1 - 2 / (exp(2x) + 1) via ex2 + rcp (two MUFU ops)
__device__ __forceinline__ float tanh_ex2(float x) {
  float e = ex2_mufu(2.8853900817779268f * x);
  float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.f));
  return 1.f - 2.f * r;
}
template <int OP>
__global__ void k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = tanh_mufu(a[i]);
      else if (OP == 1) a[i] = ex2_mufu(a[i]) - 1.0f;
      else a[i] = tanh_ex2(a[i]);
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[3] = {"tanh.approx", "ex2.approx", "ex2+rcp tanh"};
  for (int op = 0; op < 3; ++op) {
    const int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(s);
      if (op == 0) k<0><<<blocks, threads>>>(o, iters);
      else if (op == 1) k<1><<<blocks, threads>>>(o, iters);
      else k<2><<<blocks, threads>>>(o, iters);
      cudaEventRecord(e); cudaEventSynchronize(e);
    }
    float ms; cudaEventElapsedTime(&ms, s, e);
    double ops = double(blocks) * threads * iters * 8;
    printf("%-14s %.2f Gop/s = %.2f per SM per clock (at %d MHz)\n", names[op], ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
