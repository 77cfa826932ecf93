// clock64 / %globaltimer timeline of the persistent head_dim-64 forward
// (fa_fwd64_tc5): compiled with the kernel source and PP200_FA_TRACE, linked
// against libpp200.so for the shared helpers.
// usage: tools/fa_trace [B H S emu]
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_2412_14374_b200/csrc --expt-relaxed-constexpr -o tools/fa_trace \
//          tools/fa_trace.cu -L paper_2412_14374_b200 -lpp200 -lcuda \
//          -Xlinker -rpath='$ORIGIN/../paper_2412_14374_b200'
#define PP200_FA_TRACE 1
#include "../paper_2412_14374_b200/csrc/attention_tc5.cu"
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 8, H = argc > 2 ? atoi(argv[2]) : 12;
  const int S = argc > 3 ? atoi(argv[3]) : 1024, emu = argc > 4 ? atoi(argv[4]) : 0;
  pp200::g_fwd64_emu = emu;
  const int hd = 64, ld = 3 * H * hd;
  std::vector<__nv_bfloat16> h(static_cast<size_t>(B) * S * ld);
  srand(1);
  for (auto& v : h) v = __float2bfloat16((rand() / (float)RAND_MAX - 0.5f));
  void *qkv, *o;
  float* lse;
  cudaMalloc(&qkv, h.size() * 2);
  cudaMalloc(&o, static_cast<size_t>(B) * S * H * hd * 2);
  cudaMalloc(&lse, static_cast<size_t>(B) * H * S * 4);
  cudaMemcpy(qkv, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  for (int it = 0; it < 3; ++it)
    if (pp200::attention_fwd_tc5(B, H, H, S, hd, qkv, ld, o, H * hd, lse, 0)) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  pp200::attention_fwd_tc5(B, H, H, S, hd, qkv, ld, o, H * hd, lse, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> t(64 * 8 * 32), c(1024 * 3);
  cudaMemcpyFromSymbol(t.data(), pp200::fa_trace_buf, t.size() * 8);
  cudaMemcpyFromSymbol(c.data(), pp200::fa_trace_cta, c.size() * 8);
  printf("kernel %.2f us (B %d H %d S %d emu %d)\n", ms * 1e3, B, H, S, emu);
  auto T = [&](int cta, int e, int g) { return (long long)t[(cta * 8 + e) * 32 + g]; };
  // events: 0 S_g issued, 1 MMA saw p_full(g), 2 PV_g issued, 3 softmax saw s_full(g),
  // 4 S loaded + s_free, 5 exp done, 6 pv_done(g-2) seen, 7 p_full arrived
  const char* nm[] = {"S issued -> softmax sees it", "s_full seen -> S loaded", "S loaded -> exp done",
                      "exp done -> P buffer free", "P free -> p_full arrive", "p_full arrive -> MMA sees",
                      "MMA sees -> PV issued", "period (p_full to p_full)"};
  double acc[8] = {0};
  int n = 0;
  for (int cta = 0; cta < 64; ++cta)
    for (int g = 3; g < 20; ++g) {
      acc[0] += T(cta, 3, g) - T(cta, 0, g);
      acc[1] += T(cta, 4, g) - T(cta, 3, g);
      acc[2] += T(cta, 5, g) - T(cta, 4, g);
      acc[3] += T(cta, 6, g) - T(cta, 5, g);
      acc[4] += T(cta, 7, g) - T(cta, 6, g);
      acc[5] += T(cta, 1, g) - T(cta, 7, g);
      acc[6] += T(cta, 2, g) - T(cta, 1, g);
      acc[7] += T(cta, 7, g) - T(cta, 7, g - 1);
      ++n;
    }
  for (int i = 0; i < 8; ++i) printf("  %-30s %8.1f cycles\n", nm[i], acc[i] / n);
  const long long s0 = T(0, 0, 0);
  for (int g = 0; g < 24; ++g)
    printf("  g=%2d S %7lld seen %7lld ld %7lld exp %7lld pfree %7lld parr %7lld mma %7lld pv %7lld\n", g,
           T(0, 0, g) - s0, T(0, 3, g) - s0, T(0, 4, g) - s0, T(0, 5, g) - s0, T(0, 6, g) - s0, T(0, 7, g) - s0,
           T(0, 1, g) - s0, T(0, 2, g) - s0);
  const int items = B * H * ((S + 127) / 128);
  int ncta = std::min(items, 2 * 148);
  unsigned long long t0 = ~0ull, t1 = 0;
  double dsum = 0, dmin = 1e30, dmax = 0;
  for (int i = 0; i < ncta; ++i) {
    t0 = std::min(t0, c[i * 3]);
    t1 = std::max(t1, c[i * 3 + 1]);
  }
  for (int i = 0; i < ncta; ++i) {
    double d = (c[i * 3 + 1] - c[i * 3]) * 1e-3, st = (c[i * 3] - t0) * 1e-3;
    dsum += d;
    dmin = std::min(dmin, st + d);
    dmax = std::max(dmax, st + d);
  }
  printf("grid span %.2f us, %d CTAs, mean CTA duration %.2f us, CTA end times %.2f .. %.2f us\n",
         (t1 - t0) * 1e-3, ncta, dsum / ncta, dmin, dmax);
  return 0;
}
