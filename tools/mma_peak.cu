// Legacy warp-level mma.sync (bf16 m16n8k16) throughput on this GPU: the
// ceiling for the FA2-style attention kernels.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int iters = 4096;
  for (int warps : {4, 8, 16}) {
    int blocks = 148 * 4;
    k<<<blocks, warps * 32>>>(o, 16);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    cudaEventRecord(s);
    k<<<blocks, warps * 32>>>(o, iters);
    cudaEventRecord(e); cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * warps * blocks;
    printf("mma.sync bf16 m16n8k16: %d warps/CTA x %d CTAs: %.0f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
  }
  return 0;
}
