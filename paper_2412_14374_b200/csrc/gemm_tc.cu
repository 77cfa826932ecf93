// tcgen05 / TMEM / TMA bf16 GEMM for sm_100a with fused epilogues.
//
// Replaces the `matmul` rule of the reference interpreter (a @ b,
// pkg/src/pipecraft/executor.py:66-67) and the explicit `transpose` ops the
// backward rules emit before it (ir.py:519-529, executor.py:78-79): a
// transpose is an operand major (K-major vs MN-major shared-memory
// descriptor), never a copy.
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A/B tiles -> 128B-swizzled smem ring (STAGES deep)
//   warp 1      MMA issuer: one thread issues tcgen05.mma 128xBNx16 into TMEM
//   warp 2      TMEM allocator (2 accumulator buffers of BN fp32 columns)
//   warps 4..11 epilogue (2 per TMEM lane quarter, one per column half):
//               tcgen05.ld TMEM -> registers -> fused epilogue -> 128B-swizzled
//               smem stage -> TMA bulk tensor store (cp.async.bulk.tensor)
// The two TMEM accumulators let the epilogue of tile i overlap the MMAs of
// tile i+1.
#include <cudaTypedefs.h>

#include <mutex>

#include <algorithm>

#include "common.cuh"

namespace pp200 {

namespace {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row
// Epilogue: TC_EPI_G warps per TMEM lane quarter, each with TC_EPI_BUFS 4 KB
// staging buffers (a ring when 2: the store of chunk i drains while i+1 stages)
constexpr int TC_EPI_G = 2, TC_EPI_BUFS = 2;
constexpr int TC_EPI_WARPS = 4 * TC_EPI_G;
constexpr int TC_THREADS = 128 + 32 * TC_EPI_WARPS;  // 4 control warps + epilogue warps
constexpr int TC_STAGE_BYTES = 4096 * TC_EPI_BUFS;
constexpr int TC_SMEM_MAX = 232448;   // 227 KB opt-in dynamic smem per block
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;
constexpr int TC_MN_CHUNK_BYTES = TC_BK * 128;  // one 64-wide MN box of BK rows

struct TcEpi {
  int ksplit;  // 1, or 2: two K halves reduce-added (TMA add) onto a zero-filled fp32 C
  int tma_c;  // C written through smem + TMA bulk tensor store
  int tma_u;  // GELU/RELU pre-activation (aux_out) through smem + TMA as well
  int tma_a;  // residual / activation-derivative input (aux) read through TMA boxes
  int cw64;   // plain bf16 C in 64-column chunks (128 B rows, SW128 boxes)
  void* C;
  int64_t ldc;
  const float* bias;
  const void* aux;
  int64_t ldaux;
  void* aux_out;
  int64_t ldaux_out;
  int M, N, flags, out_f32;
  int n_fast;  // tile raster: 1 = consecutive tiles walk N (share the A rows), 0 = walk M
  // LM-head softmax statistics (EK_PLAIN only): per row, per (N tile, epilogue
  // column group), the running (max, sum exp(x - max)) of the bf16-rounded
  // outputs that group stored -- stats[row * ld_stats + n_tile * TC_EPI_G + group]
  float2* stats;
  int ld_stats;
  int m2_row0;  // grouped pair (pc_gemm_wgrad_pair): rows >= m2_row0 are problem 2, 0 = one problem
};

// Second problem of a grouped weight-gradient pair: C2 (+)= op(A2) op(B2) with the
// same N, K, majors and epilogue; its M tiles follow the first problem's.
struct TcGroup {
  CUtensorMap a, b, c;
};


// First k-block of split ``sp`` (sp = ksplit: the end).  Ordered split-K
// staggers the split lengths (each dl = nk / (4 ks) k-blocks longer than the
// previous; ks = 2: 6 % of nk either side of the middle): split s finishes
// after split s-1, so the earlier reduce-adds overlap the later splits'
// last k-blocks instead of making them wait.
__device__ __forceinline__ int k_split_at(int sp, int nk, const TcEpi& ep) {
  if (sp == 0) return 0;
  const int ks = ep.ksplit;
  if (sp >= ks) return nk;
  if (!(ep.flags & PC_EPI_SPLITK_ORDERED)) return sp * nk / ks;
  // split lengths L0 + s * dl, dl = nk / (4 ks): each split starts its add
  // about one epilogue after the previous one's
  const int dl = (nk + 4 * ks - 1) / (4 * ks);
  const int l0 = (nk - dl * ks * (ks - 1) / 2) / ks;
  return sp * l0 + dl * sp * (sp - 1) / 2;
}

// CG = 1: one CTA owns a 128 x BN tile.  CG = 2: a cluster pair owns a
// 256 x BN tile through cta_group::2 MMAs -- each CTA stages its own 128 rows
// of A and half (BN/2 rows) of B, so per-SM operand traffic drops by a third.
template <int BN, int CG>
struct TcCfg {
  static constexpr int B_ROWS = BN / CG;
  static constexpr int B_BYTES = B_ROWS * TC_BK * 2;
  static constexpr int STAGE_BYTES = TC_A_BYTES + B_BYTES;
  static constexpr int STAGES =
      (TC_SMEM_MAX - TC_EPI_WARPS * TC_STAGE_BYTES - 1024 - 512) / STAGE_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + TC_EPI_WARPS * TC_STAGE_BYTES +
                               1024 /*align*/ + 512 /*barriers*/;
  // two accumulators of BN fp32 columns, rounded up to a legal power-of-2 allocation
  static constexpr int TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
};

__device__ __forceinline__ void load16(const void* base, bool f32, int64_t off, int nvalid,
                                       float* v) {
  if (f32) {
    const float* p = static_cast<const float*>(base) + off;
    if (nvalid == 16 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float4 t = reinterpret_cast<const float4*>(p)[i];
        v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = i < nvalid ? p[i] : 0.f;
    }
  } else {
    const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(base) + off;
    if (nvalid == 16 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint4 t = reinterpret_cast<const uint4*>(p)[i];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 f = __bfloat1622float2(h[j]);
          v[8 * i + 2 * j] = f.x;
          v[8 * i + 2 * j + 1] = f.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = i < nvalid ? __bfloat162float(p[i]) : 0.f;
    }
  }
}

__device__ __forceinline__ void store16(void* base, bool f32, int64_t off, int nvalid,
                                        const float* v) {
  if (f32) {
    float* p = static_cast<float*>(base) + off;
    if (nvalid == 16 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        reinterpret_cast<float4*>(p)[i] =
            make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)  // fixed trip count: v stays in registers
        if (i < nvalid) p[i] = v[i];
    }
  } else {
    __nv_bfloat16* p = static_cast<__nv_bfloat16*>(base) + off;
    if (nvalid == 16 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint4 t;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          h[j] = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
        reinterpret_cast<uint4*>(p)[i] = t;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nvalid) p[i] = __float2bfloat16_rn(v[i]);
    }
  }
}

// Applies the fused epilogue to 16 accumulator values of (row, col..col+15).
// store_c: write C here (direct path).  stage_pre: the pre-activation of
// GELU/RELU is returned in pre (staged for a TMA store) instead of stored.
// have_aux: the aux input was already read (TMA box) into aux_pre.  The arrays
// are always real register arrays (never selected against nullptr), so they
// stay out of local memory.
__device__ __forceinline__ void epilogue16(const TcEpi& ep, int row, int col, float* v,
                                           bool store_c, bool stage_pre, float* pre,
                                           bool have_aux, const float* aux_pre) {
  const int nvalid = min(16, ep.N - col);
  const bool f32 = ep.out_f32 != 0;
  const int fl = ep.flags;
  if (fl & PC_EPI_ACCUM) {
    if (!store_c) return;  // staged: the TMA reduce-add does C += v
    float old[16];
    load16(ep.C, true, static_cast<int64_t>(row) * ep.ldc + col, nvalid, old);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] += old[i];
    store16(ep.C, true, static_cast<int64_t>(row) * ep.ldc + col, nvalid, v);
    return;
  }
  if (fl & PC_EPI_BIAS) {
    const float* bp = ep.bias + col;
    if (nvalid == 16 && (reinterpret_cast<uintptr_t>(bp) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 b4 = reinterpret_cast<const float4*>(bp)[i];
        v[4 * i] += b4.x; v[4 * i + 1] += b4.y; v[4 * i + 2] += b4.z; v[4 * i + 3] += b4.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += i < nvalid ? bp[i] : 0.f;
    }
  }
  if (fl & (PC_EPI_GELU | PC_EPI_RELU)) {
    if (stage_pre) {
#pragma unroll
      for (int i = 0; i < 16; ++i) pre[i] = v[i];
    } else {
      store16(ep.aux_out, f32, static_cast<int64_t>(row) * ep.ldaux_out + col, nvalid, v);
    }
    if (fl & PC_EPI_GELU) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) gelu_pair(v[i], v[i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
    }
  }
  if (fl & (PC_EPI_RESIDUAL | PC_EPI_GELU_GRAD | PC_EPI_RELU_GRAD)) {
    float a[16];
    if (have_aux) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = aux_pre[i];
    } else {
      load16(ep.aux, f32, static_cast<int64_t>(row) * ep.ldaux + col, nvalid, a);
    }
    if (fl & PC_EPI_RESIDUAL) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += a[i];
    } else if (fl & PC_EPI_GELU_GRAD) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) mul_gelu_grad_pair(v[i], v[i + 1], a[i], a[i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = a[i] > 0.f ? v[i] : 0.f;
    }
  }
  if (store_c) store16(ep.C, f32, static_cast<int64_t>(row) * ep.ldc + col, nvalid, v);
}

// 16 B chunk `j` of row `r` inside a 128B-swizzled [32 x 128 B] staging tile.
__device__ __forceinline__ uint4* stage_chunk(uint8_t* stg, int r, int j) {
  return reinterpret_cast<uint4*>(stg + r * 128 + ((j ^ (r & 7)) << 4));
}
// ... and inside a 64B-swizzled [32 x 64 B] tile (bf16 boxes of 32 columns).
__device__ __forceinline__ uint4* stage_chunk64(uint8_t* stg, int r, int j) {
  return reinterpret_cast<uint4*>(stg + r * 64 + ((j ^ ((r >> 1) & 3)) << 4));
}
__device__ __forceinline__ void stage_bf16_row32(uint8_t* stg, int r, const float* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[8 * j + 2 * k], v[8 * j + 2 * k + 1]);
    *stage_chunk64(stg, r, j) = u;
  }
}

// Epilogue kinds, one kernel instantiation each so that every kernel carries
// only its own epilogue code (the MMA and producer warps share the SM's
// instruction cache with it):
//   EK_PLAIN    bf16 C (+ bias), 64-column chunks
//   EK_ACT      bf16 C = act(acc + bias) and the pre-activation U, 64-column chunks
//   EK_AUX      bf16 C = (acc + bias) op aux with aux read as TMA boxes, 64-column chunks
//   EK_GENERIC  everything else (fp32 C, split-K, accumulate, direct stores), 32 columns
constexpr int EK_PLAIN = 0, EK_ACT = 1, EK_AUX = 2, EK_GENERIC = 3;

// v[0..63] += bias[col..col+63] (columns >= N get nothing)
__device__ __forceinline__ void add_bias64(float* v, const float* bias, int col, int N) {
  const float* bp = bias + col;
  if (col + 64 <= N) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float4 b4 = reinterpret_cast<const float4*>(bp)[i];
      v[4 * i] += b4.x; v[4 * i + 1] += b4.y; v[4 * i + 2] += b4.z; v[4 * i + 3] += b4.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] += col + i < N ? bp[i] : 0.f;
  }
}
// 64 fp32 -> bf16, one 128 B row of a 128B-swizzled [32 x 128 B] staging tile
__device__ __forceinline__ void stage_bf16_row64(uint8_t* stg, int r, const float* v) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint4 w;
    __nv_bfloat162* hw = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
    for (int k = 0; k < 4; ++k) hw[k] = __floats2bfloat162_rn(v[8 * j + 2 * k], v[8 * j + 2 * k + 1]);
    *stage_chunk(stg, r, j) = w;
  }
}

// Before restaging a buffer: the bulk store that last read it has finished.
__device__ __forceinline__ void bulk_wait_read_ring() {
  if constexpr (TC_EPI_BUFS == 2)
    bulk_wait_read1();
  else
    bulk_wait_read0();
}

// Epilogue warp hands a drained TMEM accumulator back to the (leader's) MMA warp.
template <int CG>
__device__ __forceinline__ void release_acc(uint64_t* bar, int lane) {
  tc_fence_before();
  __syncwarp();
  if (lane == 0) {
    if constexpr (CG == 2)
      mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(bar), 0));
    else
      mbar_arrive_relaxed(bar);
  }
}

template <int BN, bool A_MN, bool B_MN, int CG, int EK>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmU,
                   const __grid_constant__ CUtensorMap tmX, const __grid_constant__ TcGroup g2, int M,
                   int N, int K, TcEpi ep) {
  using Cfg = TcCfg<BN, CG>;
  constexpr int STAGES = Cfg::STAGES;
  static_assert(!B_MN || Cfg::B_ROWS % 64 == 0, "MN-major B needs 64-wide chunks per CTA");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * TC_A_BYTES;
  uint8_t* sEpi = sB + STAGES * Cfg::B_BYTES;  // 1024-aligned: 8 x 4 KB staging tiles
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + TC_EPI_WARPS * TC_STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* xbar = tempty + 2;  // one aux-tile barrier per epilogue warp
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xbar + TC_EPI_WARPS);

  // warp index through a shuffle so the compiler knows it is warp-uniform and
  // keeps the MMA warp's descriptors in uniform registers
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;  // 0 = MMA leader of the pair
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;   // pair (cluster) index / count
  const int num_m = (M + TC_BM * CG - 1) / (TC_BM * CG), num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_units = num_tiles * ep.ksplit;
  const int nk = (K + TC_BK - 1) / TC_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (ep.m2_row0) {
      tma_prefetch_desc(&g2.a);
      tma_prefetch_desc(&g2.b);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG * TC_EPI_WARPS);  // every epilogue warp of the pair
    }
    for (int w = 0; w < TC_EPI_WARPS; ++w) mbar_init(&xbar[w], 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2)
      tmem_alloc_pair(tslot, Cfg::TMEM_COLS);
    else
      tmem_alloc(tslot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote use
  tc_fence_after();
  const uint32_t tmem_base = *tslot;

  if (warp == 0) {
    // warp-uniform producer loop, one elected lane issuing (a lane-0-only
    // branch makes every barrier wait and TMA issue a divergent slow path;
    // measured on the attention kernels, profiles/r02_attn_fwd64.txt)
    {
      int stage = 0;
      uint32_t phase = 0;
      // the leader's full barrier counts both CTAs' bytes (one expect_tx)
      auto load = [&](void* dst, const CUtensorMap* tm, int stg, int x, int y) {
        if constexpr (CG == 2)
          tma_load_2d_pair(dst, tm, mapa_shared(smem_u32(&full[stg]), 0), x, y);
        else
          tma_load_2d(dst, tm, &full[stg], x, y);
      };
      for (int u = cid; u < num_units; u += ncl) {
        const int t = u % num_tiles, sp = u / num_tiles;
        const int mi = ep.n_fast ? t / num_n : t % num_m, ni = ep.n_fast ? t % num_n : t / num_m;
        // grouped pair: tiles past the first problem's rows read the second's operands
        const bool p2 = ep.m2_row0 && mi * TC_BM * CG >= ep.m2_row0;
        const CUtensorMap* pA = p2 ? &g2.a : &tmA;
        const CUtensorMap* pB = p2 ? &g2.b : &tmB;
        const int m0 = mi * TC_BM * CG + static_cast<int>(rank) * TC_BM - (p2 ? ep.m2_row0 : 0);
        const int nb = ni * BN + static_cast<int>(rank) * Cfg::B_ROWS;
        for (int kb = k_split_at(sp, nk, ep), kb_end = k_split_at(sp + 1, nk, ep); kb < kb_end; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (ep.flags & (1 << 17)) {  // profiling ablation: no operand traffic
            if (rank == 0 && elect_one()) mbar_arrive(&full[stage]);
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          if (elect_one()) {
            if (rank == 0) mbar_expect_tx(&full[stage], CG * Cfg::STAGE_BYTES);
            uint8_t* a = sA + stage * TC_A_BYTES;
            uint8_t* b = sB + stage * Cfg::B_BYTES;
            const int k0 = kb * TC_BK;
            if (!A_MN) {
              load(a, pA, stage, k0, m0);
            } else {
#pragma unroll
              for (int j = 0; j < TC_BM / 64; ++j)
                load(a + j * TC_MN_CHUNK_BYTES, pA, stage, m0 + 64 * j, k0);
            }
            if (!B_MN) {
              load(b, pB, stage, k0, nb);
            } else {
#pragma unroll
              for (int j = 0; j < Cfg::B_ROWS / 64; ++j)
                load(b + j * TC_MN_CHUNK_BYTES, pB, stage, nb + 64 * j, k0);
            }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if constexpr (CG == 2) {
        // drain: every MMA commit multicast into this CTA's ring has landed
        for (int i = 0; i < STAGES; ++i) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp walks the ring (warp-uniform control flow), one
    // elected lane issues.  Descriptors are built once; a k-step or a stage is
    // a plain add on the 14-bit start-address field (smem offsets < 256 KB).
    if (rank == 0) {
      constexpr uint32_t IDESC = umma_idesc_bf16(TC_BM * CG, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      constexpr uint64_t A_KSTEP = A_MN ? (2048 >> 4) : (32 >> 4);
      constexpr uint64_t B_KSTEP = B_MN ? (2048 >> 4) : (32 >> 4);
      const uint64_t a_desc0 = A_MN ? umma_sdesc_sw128(smem_u32(sA), TC_MN_CHUNK_BYTES, 1024)
                                    : umma_sdesc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t b_desc0 = B_MN ? umma_sdesc_sw128(smem_u32(sB), TC_MN_CHUNK_BYTES, 1024)
                                    : umma_sdesc_sw128(smem_u32(sB), 16, 1024);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int u = cid; u < num_units; u += ncl) {
        const int sp = u / num_tiles;
        const int kb0 = k_split_at(sp, nk, ep), kb1 = k_split_at(sp + 1, nk, ep);
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = a_desc0 + static_cast<uint64_t>(stage * (TC_A_BYTES >> 4));
          const uint64_t bd = b_desc0 + static_cast<uint64_t>(stage * (Cfg::B_BYTES >> 4));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < TC_BK / 16; ++k) {
              const uint32_t accum = (kb > kb0 || k > 0) ? 1u : 0u;
              if constexpr (CG == 2)
                tc_mma_f16_pair(d, ad + k * A_KSTEP, bd + k * B_KSTEP, IDESC, accum);
              else
                tc_mma_f16(d, ad + k * A_KSTEP, bd + k * B_KSTEP, IDESC, accum);
            }
            if constexpr (CG == 2)
              tc_commit_pair(&empty[stage]);
            else
              tc_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) {
          if constexpr (CG == 2)
            tc_commit_pair(&tfull[acc]);
          else
            tc_commit(&tfull[acc]);
        }
        __syncwarp();
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
      if constexpr (CG == 2) {
        // both CTAs' epilogues have released both accumulators
        for (int i = 0; i < 2; ++i) {
          mbar_wait(&tempty[acc], aphase ^ 1);
          acc ^= 1;
          if (acc == 0) aphase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // 8 epilogue warps: warp & 3 selects the TMEM lane quarter (rows), the
    // warp-group half selects which half of the tile's columns it drains.
    const int q = warp & 3;
    const int grp = (warp - 4) >> 2;  // column group within the lane quarter
    // per-warp ring of two 4 KB staging buffers: the TMA store of chunk i
    // drains while chunk i+1 is staged; a buffer is rewritten only after the
    // store two chunks back has finished reading it.
    uint8_t* stg0 = sEpi + (warp - 4) * TC_STAGE_BYTES;
    const bool f32 = ep.out_f32 != 0;
    const bool tma = ep.tma_c != 0;
    const bool tma_x = ep.tma_a != 0;
    const bool skip_x = (ep.flags & (1 << 18)) != 0;  // profiling ablation: aux never loaded
    const bool stage_u = ep.tma_u != 0;
    // chunks (64 columns as full 128 B rows for the specialised kinds, 32 for
    // the generic one) dealt round-robin to the warp groups of a lane quarter
    constexpr bool wide = EK != EK_GENERIC;
    constexpr int CW = wide ? 64 : 32;
    const int cstart = grp * CW;
    constexpr int cstep = CW * TC_EPI_G;
    const int cstop = BN;
    uint64_t* xb = &xbar[warp - 4];
    uint32_t xphase = 0;
    uint32_t nchunk = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int u = cid; u < num_units; u += ncl) {
      const int t = u % num_tiles;
      const int mi = ep.n_fast ? t / num_n : t % num_m, ni = ep.n_fast ? t % num_n : t / num_m;
      const int m0 = mi * TC_BM * CG + static_cast<int>(rank) * TC_BM;
      const int n0 = ni * BN;
      // grouped pair: the second problem's tiles store to its C at local rows
      const bool p2 = ep.m2_row0 && mi * TC_BM * CG >= ep.m2_row0;
      const CUtensorMap* pC = p2 ? &g2.c : &tmC;
      const int m0s = m0 - (p2 ? ep.m2_row0 : 0);
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const int cend = (ep.flags & (1 << 16)) ? cstart : cstop;  // profiling ablation: no epilogue work
      const uint32_t tb =
          tmem_base + static_cast<uint32_t>(acc * BN) + (static_cast<uint32_t>(q * 32) << 16);
      // the accumulator goes back to the MMA warp as soon as it is in registers
      uint64_t* rel = &tempty[acc];
      if (tma_x && !skip_x && lane == 0 && cend > cstart) {  // prefetch the first aux box of this tile
        if constexpr (EK == EK_AUX) {
          if (nchunk == 0) {  // later tiles: prefetched by the previous tile's last chunk
            mbar_expect_tx(xb, 4096);
            tma_load_2d(stg0, &tmX, xb, n0 + cstart, m0 + q * 32);
          }
        } else {
          mbar_expect_tx(xb, 2048);
          tma_load_2d(stg0 + (TC_EPI_BUFS == 2 ? (nchunk & 1) * 4096 : 0) + 2048, &tmX, xb, n0 + cstart,
                      m0 + q * 32);
        }
      }
      if constexpr (EK == EK_PLAIN) {
        float xm = -INFINITY, xs = 0.f;   // softmax statistics of this row (ep.stats)
#pragma unroll 1
        for (int cc = cstart; cc < cend; cc += cstep) {
          const uint32_t my = nchunk++;
          uint8_t* stg = stg0 + (TC_EPI_BUFS == 2 ? (my & 1) * 4096 : 0);
          uint32_t r[64];
#pragma unroll
          for (int h = 0; h < 4; ++h) tmem_ld16(tb + cc + 16 * h, r + 16 * h);
          tc_wait_ld();
          if (cc + cstep >= cend) release_acc<CG>(rel, lane);
          float* v = reinterpret_cast<float*>(r);
          if (ep.flags & PC_EPI_BIAS) add_bias64(v, ep.bias, n0 + cc, N);
          if (lane == 0) bulk_wait_read_ring();
          __syncwarp();
          stage_bf16_row64(stg, lane, v);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(pC, stg, n0 + cc, m0s + q * 32);
            bulk_commit();
          }
          if (ep.stats != nullptr) {
            // online (max, sum exp) over the values as stored (bf16-rounded),
            // columns past N excluded; exp2 with log2(e) folded into one FMA
            constexpr float L2E = 1.4426950408889634f;
            const int nvalid = N - (n0 + cc);
            float cm = -INFINITY;
#pragma unroll
            for (int i = 0; i < 64; ++i) {
              v[i] = i < nvalid ? __bfloat162float(__float2bfloat16_rn(v[i])) : -INFINITY;
              cm = fmaxf(cm, v[i]);
            }
            const float mn = fmaxf(xm, cm);
            if (mn != -INFINITY) {
              const float nm = -mn * L2E;
              float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
              for (int i = 0; i < 64; ++i) {
                float e;
                asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fmaf(v[i], L2E, nm)));
                part[i & 3] += e;
              }
              float sc;
              asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(sc) : "f"(fmaf(xm, L2E, nm)));
              xs = xs * sc + ((part[0] + part[1]) + (part[2] + part[3]));
              xm = mn;
            }
          }
        }
        if (ep.stats != nullptr && row < M)
          ep.stats[static_cast<int64_t>(row) * ep.ld_stats + ni * TC_EPI_G + grp] = make_float2(xm, xs);
      } else if constexpr (EK == EK_ACT) {
        // U (pre-activation) staged in buffer B, C in buffer A, one bulk group
        // each: before restaging either, the group two back has been read
        uint8_t* sA = stg0;
        uint8_t* sB = stg0 + 4096;
        const bool gelu = (ep.flags & PC_EPI_GELU) != 0;
#pragma unroll 1
        for (int cc = cstart; cc < cend; cc += cstep) {
          uint32_t r[64];
#pragma unroll
          for (int h = 0; h < 4; ++h) tmem_ld16(tb + cc + 16 * h, r + 16 * h);
          tc_wait_ld();
          if (cc + cstep >= cend) release_acc<CG>(rel, lane);
          float* v = reinterpret_cast<float*>(r);
          if (ep.flags & PC_EPI_BIAS) add_bias64(v, ep.bias, n0 + cc, N);
          if (lane == 0) bulk_wait_read1();
          __syncwarp();
          stage_bf16_row64(sB, lane, v);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmU, sB, n0 + cc, m0 + q * 32);
            bulk_commit();
          }
          if (gelu) {
#pragma unroll
            for (int i = 0; i < 64; i += 2) gelu_pair(v[i], v[i + 1]);
          } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) v[i] = fmaxf(v[i], 0.f);
          }
          if (lane == 0) bulk_wait_read1();
          __syncwarp();
          stage_bf16_row64(sA, lane, v);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(pC, sA, n0 + cc, m0s + q * 32);
            bulk_commit();
          }
        }
      } else if constexpr (EK == EK_AUX) {
        // Buffers alternate per chunk: chunk i finds its aux box in X = buf[i&1],
        // consumes it, then stages C(i) in X.  Before computing, it requests the
        // next box (rest of this tile, else the first box of this warp's next
        // tile) into the other buffer, once C(i-1) has left it.
        const int op = (ep.flags & PC_EPI_RESIDUAL) ? 0 : ((ep.flags & PC_EPI_GELU_GRAD) ? 1 : 2);
#pragma unroll 1
        for (int cc = cstart; cc < cend; cc += cstep) {
          const uint32_t my = nchunk++;
          uint8_t* X = stg0 + (my & 1) * 4096;
          uint8_t* Y = stg0 + ((my + 1) & 1) * 4096;
          const bool last = cc + cstep >= cend;
          int nx_n = -1, nx_m = 0;
          if (!last) {
            nx_n = n0 + cc + cstep;
            nx_m = m0 + q * 32;
          } else if (u + ncl < num_units) {
            const int t2 = (u + ncl) % num_tiles;
            nx_n = (t2 / num_m) * BN + cstart;
            nx_m = (t2 % num_m) * TC_BM * CG + static_cast<int>(rank) * TC_BM + q * 32;
          }
          uint32_t r[64];
#pragma unroll
          for (int h = 0; h < 4; ++h) tmem_ld16(tb + cc + 16 * h, r + 16 * h);
          if (!skip_x) mbar_wait(xb, xphase);  // aux(i) has landed in X
          xphase ^= 1;
          if (lane == 0) bulk_wait_read0();  // C(i-1) has left Y
          __syncwarp();
          if (lane == 0 && nx_n >= 0 && !skip_x) {
            mbar_expect_tx(xb, 4096);
            tma_load_2d(Y, &tmX, xb, nx_n, nx_m);
          }
          tc_wait_ld();
          if (last) release_acc<CG>(rel, lane);
          float* v = reinterpret_cast<float*>(r);
          if (ep.flags & PC_EPI_BIAS) add_bias64(v, ep.bias, n0 + cc, N);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 w = *stage_chunk(X, lane, j);
            const __nv_bfloat162* hx = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 a2 = __bfloat1622float2(hx[k]);
              float& v0 = v[8 * j + 2 * k];
              float& v1 = v[8 * j + 2 * k + 1];
              if (op == 0) {
                v0 += a2.x;
                v1 += a2.y;
              } else if (op == 1) {
                mul_gelu_grad_pair(v0, v1, a2.x, a2.y);
              } else {
                v0 = a2.x > 0.f ? v0 : 0.f;
                v1 = a2.y > 0.f ? v1 : 0.f;
              }
            }
          }
          __syncwarp();  // every lane has read X
          stage_bf16_row64(X, lane, v);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(pC, X, n0 + cc, m0s + q * 32);
            bulk_commit();
          }
        }
      } else {
      // ordered split-K accumulate: split s adds its part onto C only after
      // splits 0..s-1 added theirs to the same region (this warp's rows x
      // columns); the region's flag counts the splits that landed
      const bool ordered = (ep.flags & PC_EPI_SPLITK_ORDERED) && ep.ksplit > 1;
      const int sp = u / num_tiles;
      unsigned* oflag = static_cast<unsigned*>(const_cast<void*>(ep.aux)) +
                        ((t * CG + static_cast<int>(rank)) * TC_EPI_WARPS + (warp - 4));
      if (ordered && sp > 0) {
        if (lane == 0) {
          while (ld_acquire_gpu(oflag) != static_cast<unsigned>(sp)) __nanosleep(100);
          if (sp == ep.ksplit - 1) st_release_gpu(oflag, 0u);  // last: re-armed for the next launch
          fence_proxy_async_global();
        }
        __syncwarp();
      }
#pragma unroll 1
      for (int cc = cstart; cc < cend; cc += cstep) {
        const uint32_t my = nchunk++;
        uint8_t* stg = stg0 + (TC_EPI_BUFS == 2 ? (my & 1) * 4096 : 0);
        const bool last = cc + cstep >= cend;
        uint32_t r[32];
        tmem_ld16(tb + cc, r);
        tmem_ld16(tb + cc + 16, r + 16);
        // aux input (TMA box) and staged pre-activation are never both used:
        // one register array serves either role
        float xu[32];
        if (tma_x) {
          uint8_t* xstg = stg + 2048;  // aux box (bf16 32x32, 64B swizzle)
          if (!skip_x) mbar_wait(xb, xphase);
          xphase ^= 1;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 w = *stage_chunk64(xstg, lane, j);
            const __nv_bfloat162* hx = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 f2 = __bfloat1622float2(hx[k]);
              xu[8 * j + 2 * k] = f2.x;
              xu[8 * j + 2 * k + 1] = f2.y;
            }
          }
          __syncwarp();
          if (lane == 0 && !last && !skip_x) {  // prefetch the next chunk's box into the other buffer
            mbar_expect_tx(xb, 2048);
            tma_load_2d(stg0 + (TC_EPI_BUFS == 2 ? ((my + 1) & 1) * 4096 : 0) + 2048, &tmX, xb,
                        n0 + cc + cstep, m0 + q * 32);
          }
        }
        tc_wait_ld();
        if (last) release_acc<CG>(rel, lane);
        float* v = reinterpret_cast<float*>(r);
        if (row < M) {
          if (n0 + cc < N)
            epilogue16(ep, row, n0 + cc, v, !tma, stage_u, xu, tma_x, xu);
          if (n0 + cc + 16 < N)
            epilogue16(ep, row, n0 + cc + 16, v + 16, !tma, stage_u, xu + 16, tma_x, xu + 16);
        }
        if (!tma) continue;
        if (lane == 0) bulk_wait_read_ring();  // the store that last used this buffer has read it
        __syncwarp();
        if (f32) {
          // 32 fp32 = one 128 B row per thread, 128B-swizzled box {32 cols, 32 rows}
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *stage_chunk(stg, lane, j) = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
        } else {
          // 32 bf16 = one 64 B row per thread, 64B-swizzled box {32 cols, 32 rows};
          // the pre-activation goes to the second half of the buffer
          stage_bf16_row32(stg, lane, v);
          if (stage_u) stage_bf16_row32(stg + 2048, lane, xu);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (ep.ksplit > 1 || (ep.flags & PC_EPI_ACCUM))
            tma_reduce_add_2d(pC, stg, n0 + cc, m0s + q * 32);
          else
            tma_store_2d(pC, stg, n0 + cc, m0s + q * 32);
          if (stage_u) tma_store_2d(&tmU, stg + 2048, n0 + cc, m0 + q * 32);
          bulk_commit();
        }
      }
      if (ordered && sp < ep.ksplit - 1 && lane == 0) {  // publish once this split's adds landed
        bulk_wait0();
        fence_proxy_async_global();
        st_release_gpu(oflag, static_cast<unsigned>(sp + 1));
      }
      }
      if (cend <= cstart) release_acc<CG>(rel, lane);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (tma && lane == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();
  tc_fence_after();
  if (warp == 2) {
    if constexpr (CG == 2)
      tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
    else
      tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor map over a row-major [outer, inner] view with leading
// dimension `ld` elements, 128B-swizzled boxes of {64, box_outer}.
int make_tmap(CUtensorMap* m, const void* ptr, int64_t inner, int64_t outer, int64_t ld,
              int box_outer) {
  auto enc = tmap_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return PC_ERR_CUDA;
  }
  PP_CHECK_ARG((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "TMA operand not 16B aligned");
  PP_CHECK_ARG((ld * 2) % 16 == 0, "TMA leading dimension %lld not a multiple of 8", (long long)ld);
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_outer)};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

// Store-side tensor map for C (or the pre-activation): [M, N] row-major, boxes
// of 32 columns x 32 rows: fp32 -> 128 B rows, 128B swizzle; bf16 -> 64 B rows,
// 64B swizzle -- matching the epilogue staging tiles.
int make_tmap_c(CUtensorMap* m, void* ptr, int64_t N, int64_t M, int64_t ldc, bool f32,
                bool wide = false) {
  auto enc = tmap_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return PC_ERR_CUDA;
  }
  const int es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldc * es)};
  // wide: bf16 boxes of 64 columns (128 B rows, 128B swizzle)
  cuuint32_t box[2] = {wide ? 64u : 32u, 32u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (f32 || wide) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (C) failed (%d)", static_cast<int>(r));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

int g_force_bn = 0;
int g_tma_store = 1;
int g_cta_pair = 0;  // 0 auto, 1 never, 2 always (where the tile allows it)
int g_max_split = 4;  // pc_gemm_set_max_split (tuning hook; 4: C2 dW_o 26.4 -> 22.9 us)
int g_ablate = 0;    // profiling: bit0 skip epilogue work, bit1 skip operand loads

template <int BN, bool A_MN, bool B_MN, int CG, int EK>
int launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
              const CUtensorMap& tu, const CUtensorMap& tx, const TcGroup& g2, int M, int N, int K,
              const TcEpi& ep, cudaStream_t st) {
  using Cfg = TcCfg<BN, CG>;
  auto kern = tc_gemm_kernel<BN, A_MN, B_MN, CG, EK>;
  static int max_units = 0;  // benign race: idempotent attribute write / query
  if (!max_units) {
    PP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    int mu = num_sms();
    if (CG == 2) {
      PP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t q{};
      cudaLaunchAttribute qa[1];
      q.gridDim = dim3(2 * (num_sms() / 2));
      q.blockDim = dim3(TC_THREADS);
      q.dynamicSmemBytes = Cfg::SMEM;
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = 2;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      int nc = 0;
      PP_CUDA_TRY(cudaOccupancyMaxActiveClusters(&nc, kern, &q));
      mu = nc > 0 ? nc : num_sms() / 2;  // co-resident pairs
    }
    max_units = mu;
  }
  const int units = ((M + TC_BM * CG - 1) / (TC_BM * CG)) * ((N + BN - 1) / BN) * ep.ksplit;
  const int groups = units < max_units ? units : max_units;
  if constexpr (CG == 1) {
    kern<<<groups, TC_THREADS, Cfg::SMEM, st>>>(ta, tb, tc, tu, tx, g2, M, N, K, ep);
  } else {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(2 * groups);
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tu, tx, g2, M, N, K, ep));
  }
  return check_launch("tc_gemm_kernel");
}

// A_MN is only ever used by weight gradients (fp32 C): generic epilogue only.
template <int BN, int CG, bool B_MN>
int dispatch_ek(bool a_mn, int ek, const CUtensorMap& ta, const CUtensorMap& tb,
                const CUtensorMap& tc, const CUtensorMap& tu, const CUtensorMap& tx, const TcGroup& g2, int M, int N,
                int K, const TcEpi& ep, cudaStream_t st) {
  if (a_mn) return launch_tc<BN, true, B_MN, CG, EK_GENERIC>(ta, tb, tc, tu, tx, g2, M, N, K, ep, st);
  switch (ek) {
    case EK_PLAIN: return launch_tc<BN, false, B_MN, CG, EK_PLAIN>(ta, tb, tc, tu, tx, g2, M, N, K, ep, st);
    case EK_ACT: return launch_tc<BN, false, B_MN, CG, EK_ACT>(ta, tb, tc, tu, tx, g2, M, N, K, ep, st);
    case EK_AUX: return launch_tc<BN, false, B_MN, CG, EK_AUX>(ta, tb, tc, tu, tx, g2, M, N, K, ep, st);
    default: return launch_tc<BN, false, B_MN, CG, EK_GENERIC>(ta, tb, tc, tu, tx, g2, M, N, K, ep, st);
  }
}

template <int BN, int CG>
int dispatch_majors(bool a_mn, bool b_mn, int ek, const CUtensorMap& ta, const CUtensorMap& tb,
                    const CUtensorMap& tc, const CUtensorMap& tu, const CUtensorMap& tx, const TcGroup& g2, int M,
                    int N, int K, const TcEpi& ep, cudaStream_t st) {
  if constexpr ((BN / CG) % 64 != 0) {  // MN-major B needs 64-wide chunks per CTA
    if (b_mn) {
      set_error("gemm: tile %d x cta_group %d needs a K-major B", BN, CG);
      return PC_ERR_ARG;
    }
    return dispatch_ek<BN, CG, false>(a_mn, ek, ta, tb, tc, tu, tx, g2, M, N, K, ep, st);
  } else {
    if (b_mn) return dispatch_ek<BN, CG, true>(a_mn, ek, ta, tb, tc, tu, tx, g2, M, N, K, ep, st);
    return dispatch_ek<BN, CG, false>(a_mn, ek, ta, tb, tc, tu, tx, g2, M, N, K, ep, st);
  }
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder_fn() { return tmap_encoder(); }

// Pick (tile width, CTA pair, K split) minimising a per-SM time model:
//   waves x (mainloop + epilogue) + the split reduce-adds,
// mainloop = K-split length x (tile FLOPs / SM peak) / eff(tile) -- the large
// pair tiles sustain more of the peak on long K (fewer operand bytes per FLOP),
// the narrow ones lose less to a partial last wave -- and epilogue = the tile's
// C bytes per SM at ~30 B / clk plus ~1000 cycles; an ordered split adds one
// epilogue per chain link, an unordered one a single reduce-add.  The factors
// were fit to tools/gemm_sweep_mix.py over the C2-C5 shapes (round 2,
// profiles/r02_gemm_sweep_*.txt).  Deterministic split-K: exactly 2 K halves
// reduce-added onto a zero-filled fp32 C (0 + a + b == 0 + b + a bitwise), or
// the ordered protocol, only when the caller allows it.  c_bytes: bytes moved
// per C element by the epilogue (bf16 store 2, fp32 store 4, fp32 add 8).
static void choose_tiles(bool b_kmajor, int64_t M, int64_t N, int64_t K, bool can_split,
                         int* bn_out, int* cg_out, int* ks_out, int max_split = 2,
                         bool ordered = false, double c_bytes = 2.0) {
  struct Cand { int bn, cg; double eff; };
  const Cand cands[7] = {{256, 2, 0.95}, {192, 2, 0.85}, {256, 1, 0.80}, {192, 1, 0.80},
                         {128, 2, 0.80}, {128, 1, 0.75}, {64, 1, 0.55}};
  const int sms = num_sms();
  can_split = can_split && K >= 2 * TC_BK * 8;
  if (!can_split) max_split = 1;
  int bn = 0, cg = 1, ksplit = 1;
  double best = 1e300;
  for (const Cand& c : cands) {
    if (g_force_bn && c.bn != g_force_bn) continue;
    if (g_cta_pair == 1 && c.cg == 2) continue;
    if (g_cta_pair == 2 && c.cg == 1 && c.bn != 64) continue;
    if (c.cg == 2 && (c.bn / 2) % 64 != 0 && !b_kmajor) continue;
    if (!g_force_bn && c.bn > 64 && N < c.bn / 2) continue;
    if (!g_force_bn && c.cg == 2 && M <= TC_BM) continue;
    // short K and narrow N (C2 attention-output GEMM and its dX, 8192x768x768):
    // the pair's cluster launch / barrier costs outweigh its operand savings
    // (measured 12.7 vs 11.7 us); single-CTA tiles
    if (!g_force_bn && g_cta_pair == 0 && c.cg == 2 && K <= 768 && N <= 768) continue;
    const int64_t tm = TC_BM * c.cg;
    const int64_t tiles = ((M + tm - 1) / tm) * ((N + c.bn - 1) / c.bn);
    const int64_t slots = sms / c.cg;
    const double flop_cycles = static_cast<double>(tm) * c.bn * 2.0 / (c.cg * 8192.0);  // per k
    const double epi = static_cast<double>(tm) * c.bn * c_bytes / c.cg / 30.0 + 1000.0;
    for (int ks = 1; ks <= max_split; ks *= 2) {
      if (K < static_cast<int64_t>(ks) * TC_BK * 8) break;   // >= 8 k-blocks per split
      // Ordered split-K makes split s of a tile wait for split s-1 on another CTA.
      // With more units than co-resident CTAs a resident CTA can wait on a unit
      // whose CTA is not resident yet while every resident CTA waits too (a
      // deadlock, seen on C4's 512-unit weight gradients): one wave only.
      if (ordered && ks > 1 && tiles * ks > slots) break;
      const int64_t waves = (tiles * ks + slots - 1) / slots;
      const double kper = static_cast<double>((K + ks - 1) / ks);
      double t = static_cast<double>(waves) * (kper * flop_cycles / c.eff + epi);
      if (ks > 1) t += (ordered ? ks - 1 : 1) * epi;
      if (t < best * (1.0 - 1e-9)) {
        best = t;
        bn = c.bn;
        cg = c.cg;
        ksplit = ks;
      }
    }
  }
  if (bn == 0) {  // forced combination not realisable (e.g. pair 192 with MN-major B)
    bn = g_force_bn ? g_force_bn : 128;
    cg = 1;
    ksplit = 1;
  }
  *bn_out = bn;
  *cg_out = cg;
  *ks_out = ksplit;
}

// Second problem of a grouped weight-gradient pair (pc_gemm_wgrad_pair).
struct PairArgs {
  int64_t M2;
  const void* A2;
  int64_t lda2;
  const void* B2;
  int64_t ldb2;
  void* C2;
  int64_t ldc2;
};

static int gemm_tc_impl(int out_f32, int transA, int transB, int64_t M, int64_t N, int64_t K,
                        const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                        int epi, const void* bias, const void* aux, int64_t ldaux, void* aux_out,
                        int64_t ldaux_out, cudaStream_t st, float2* stats, int64_t ld_stats,
                        const PairArgs* pair);

int gemm_bf16_tc(int out_f32, int transA, int transB, int64_t M, int64_t N, int64_t K,
                 const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                 int epi, const void* bias, const void* aux, int64_t ldaux, void* aux_out,
                 int64_t ldaux_out, cudaStream_t st, float2* stats, int64_t ld_stats) {
  return gemm_tc_impl(out_f32, transA, transB, M, N, K, A, lda, B, ldb, C, ldc, epi, bias, aux, ldaux,
                      aux_out, ldaux_out, st, stats, ld_stats, nullptr);
}

static int gemm_tc_impl(int out_f32, int transA, int transB, int64_t M, int64_t N, int64_t K,
                        const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                        int epi, const void* bias, const void* aux, int64_t ldaux, void* aux_out,
                        int64_t ldaux_out, cudaStream_t st, float2* stats, int64_t ld_stats,
                        const PairArgs* pair) {
  PP_CHECK_ARG(M > 0 && N > 0 && K > 0, "gemm: empty problem");
  // a grouped pair runs as one problem of M + M2 rows; tiles past M read / write
  // the second problem (the first's rows must fill whole tiles)
  const int64_t Mt = pair ? M + pair->M2 : M;
  PP_CHECK_ARG(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31), "gemm: dims too large");
  PP_CHECK_ARG(!((epi & PC_EPI_ACCUM) && (epi & PC_EPI_SPLITK_ZERO_C)),
               "gemm: accumulate and split-K onto zeros are exclusive");
  const int es = out_f32 ? 4 : 2;
  // C through smem + TMA: plain store, or (fp32 accumulate / split-K) a TMA
  // reduce-add at L2 -- C += tile in one fp32 add per element, so an
  // unsplit accumulate equals storing the product and adding it after
  const bool tma_c = g_tma_store && (!(epi & PC_EPI_ACCUM) || out_f32) &&
                     (reinterpret_cast<uintptr_t>(C) & 15) == 0 && (ldc * es) % 16 == 0;
  const bool ordered = (epi & PC_EPI_SPLITK_ORDERED) && (epi & PC_EPI_ACCUM) && out_f32 && tma_c;
  PP_CHECK_ARG(!(epi & PC_EPI_SPLITK_ORDERED) ||
                   ((epi & PC_EPI_ACCUM) && aux != nullptr &&
                    !(epi & (PC_EPI_RESIDUAL | PC_EPI_GELU_GRAD | PC_EPI_RELU_GRAD))),
               "gemm: ordered split-K needs accumulate and a flag array in aux");
  const bool can_split = ((epi & PC_EPI_SPLITK_ZERO_C) && out_f32 && tma_c) || ordered;
  int bn, cg, ksplit;
  // (up to g_max_split = 4 K splits: re-measured in round 2 after the relaxed
  // accumulator hand-back, a 4-split C2 dW_o [768 x 768 x 8192] runs 22.9 vs
  // 26.4 us and the other weight gradients are unchanged or faster, 8 is slower)
  // unordered split-K onto a zero C is only order-independent for 2 halves
  // (0 + a + b == 0 + b + a): more splits need the ordered protocol
  const double c_bytes = (epi & PC_EPI_ACCUM) ? 8.0 : out_f32 ? 4.0 : 2.0;
  choose_tiles(transB != 0, Mt, N, K, can_split, &bn, &cg, &ksplit, ordered ? g_max_split : std::min(g_max_split, 2),
               ordered, c_bytes);
  if (pair) {
    PP_CHECK_ARG(M % (TC_BM * cg) == 0 && tma_c && out_f32 && transA && !transB && !(epi & ~(PC_EPI_ACCUM | PC_EPI_SPLITK_ORDERED | PC_EPI_SPLITK_ZERO_C)),
                 "gemm pair: first problem must fill whole tiles, fp32 TMA C, weight-gradient majors");
  }
  // raster: an A operand far larger than L2 (the LM-head gradients: 824 MB of
  // logit gradients) is streamed once when the tiles sharing its rows run
  // together; otherwise walk M (B is the large, reused operand)
  const bool n_fast = static_cast<double>(Mt) * K * 2 > 64e6 && Mt * 2 > N;
  if (ordered && ksplit > 1) {
    const int64_t tiles = ((Mt + TC_BM * cg - 1) / (TC_BM * cg)) * ((N + bn - 1) / bn);
    PP_CHECK_ARG(ldaux >= tiles * cg * TC_EPI_WARPS, "gemm: ordered split-K flag array too short");
  }
  // op(A) is [M,K]: transA=0 -> stored [M,K] (K-major); transA=1 -> stored [K,M] (MN-major).
  // op(B) is [K,N]: transB=0 -> stored [K,N] (MN-major); transB=1 -> stored [N,K] (K-major).
  const bool a_mn = transA != 0;
  const bool b_mn = transB == 0;
  CUtensorMap ta, tb;
  int rc;
  if (!a_mn)
    rc = make_tmap(&ta, A, K, M, lda, TC_BM);
  else
    rc = make_tmap(&ta, A, M, K, lda, TC_BK);
  if (rc) return rc;
  if (!b_mn)
    rc = make_tmap(&tb, B, K, N, ldb, bn / cg);
  else
    rc = make_tmap(&tb, B, N, K, ldb, TC_BK);
  if (rc) return rc;
  // C (and a GELU/RELU pre-activation) goes through smem + TMA store when
  // legal (tma_c above: 16 B aligned rows, no read-modify-write epilogue).
  const bool tma_u = tma_c && !out_f32 && (epi & (PC_EPI_GELU | PC_EPI_RELU)) &&
                     (reinterpret_cast<uintptr_t>(aux_out) & 15) == 0 && (ldaux_out * 2) % 16 == 0;
  // aux (residual / activation-derivative input) through TMA boxes in the free
  // half of the bf16 staging tile (never together with a staged pre-activation)
  const bool tma_a = tma_c && !out_f32 && !tma_u &&
                     (epi & (PC_EPI_RESIDUAL | PC_EPI_GELU_GRAD | PC_EPI_RELU_GRAD)) &&
                     (reinterpret_cast<uintptr_t>(aux) & 15) == 0 && (ldaux * 2) % 16 == 0;
  CUtensorMap tc, tu, tx;
  memset(&tc, 0, sizeof(tc));
  memset(&tu, 0, sizeof(tu));
  memset(&tx, 0, sizeof(tx));
  // epilogue kind: the specialised 64-column kinds need bf16 C through TMA, no
  // split / accumulate, a 16 B aligned bias, and U / aux through TMA as well
  const bool bias_ok = !(epi & PC_EPI_BIAS) || (reinterpret_cast<uintptr_t>(bias) & 15) == 0;
  const bool spec = tma_c && !out_f32 && ksplit == 1 && bias_ok && !a_mn;
  const int aux_ops = epi & (PC_EPI_RESIDUAL | PC_EPI_GELU_GRAD | PC_EPI_RELU_GRAD);
  int ek = EK_GENERIC;
  if (spec && (epi & ~PC_EPI_BIAS) == 0)
    ek = EK_PLAIN;
  else if (spec && tma_u && (epi & ~(PC_EPI_BIAS | PC_EPI_GELU | PC_EPI_RELU)) == 0 &&
           (epi & (PC_EPI_GELU | PC_EPI_RELU)) != (PC_EPI_GELU | PC_EPI_RELU))
    ek = EK_ACT;
  else if (spec && tma_a && (epi & ~(PC_EPI_BIAS | aux_ops)) == 0 &&
           (aux_ops == PC_EPI_RESIDUAL || aux_ops == PC_EPI_GELU_GRAD || aux_ops == PC_EPI_RELU_GRAD))
    ek = EK_AUX;
  const bool cw64 = ek != EK_GENERIC;
  if (tma_a) {
    rc = make_tmap_c(&tx, const_cast<void*>(aux), N, M, ldaux, false, cw64);
    if (rc) return rc;
  }
  if (tma_u) {
    rc = make_tmap_c(&tu, aux_out, N, M, ldaux_out, false, cw64);
    if (rc) return rc;
  }
  if (tma_c) {
    rc = make_tmap_c(&tc, C, N, M, ldc, out_f32 != 0, cw64);
    if (rc) return rc;
  }
  if (stats != nullptr) {
    PP_CHECK_ARG(ek == EK_PLAIN, "gemm: softmax statistics need a plain bf16 C through TMA");
    PP_CHECK_ARG(ld_stats >= ((N + bn - 1) / bn) * TC_EPI_G, "gemm: statistics row too short");
  }
  TcEpi ep{ksplit, tma_c ? 1 : 0, tma_u ? 1 : 0, tma_a ? 1 : 0, cw64 ? 1 : 0, C, ldc, static_cast<const float*>(bias), aux, ldaux,
           aux_out, ldaux_out, static_cast<int>(Mt), static_cast<int>(N), epi | (g_ablate << 16), out_f32,
           n_fast ? 1 : 0, stats, static_cast<int>(ld_stats), pair ? static_cast<int>(M) : 0};
  TcGroup g2;
  memset(&g2, 0, sizeof(g2));
  if (pair) {
    rc = make_tmap(&g2.a, pair->A2, pair->M2, K, pair->lda2, TC_BK);  // MN-major A2 [K, M2]
    if (rc) return rc;
    rc = make_tmap(&g2.b, pair->B2, N, K, pair->ldb2, TC_BK);         // MN-major B2 [K, N]
    if (rc) return rc;
    rc = make_tmap_c(&g2.c, pair->C2, N, pair->M2, pair->ldc2, true, cw64);
    if (rc) return rc;
  }
  const int iM = static_cast<int>(Mt), iN = static_cast<int>(N), iK = static_cast<int>(K);
  switch (bn * 4 + cg) {
    case 256 * 4 + 2: return dispatch_majors<256, 2>(a_mn, b_mn, ek, ta, tb, tc, tu, tx, g2, iM, iN, iK, ep, st);
    case 192 * 4 + 2: return dispatch_majors<192, 2>(a_mn, b_mn, ek, ta, tb, tc, tu, tx, g2, iM, iN, iK, ep, st);
    case 128 * 4 + 2: return dispatch_majors<128, 2>(a_mn, b_mn, ek, ta, tb, tc, tu, tx, g2, iM, iN, iK, ep, st);
    case 256 * 4 + 1: return dispatch_majors<256, 1>(a_mn, b_mn, ek, ta, tb, tc, tu, tx, g2, iM, iN, iK, ep, st);
    case 192 * 4 + 1: return dispatch_majors<192, 1>(a_mn, b_mn, ek, ta, tb, tc, tu, tx, g2, iM, iN, iK, ep, st);
    case 128 * 4 + 1: return dispatch_majors<128, 1>(a_mn, b_mn, ek, ta, tb, tc, tu, tx, g2, iM, iN, iK, ep, st);
    case 64 * 4 + 1: return dispatch_majors<64, 1>(a_mn, b_mn, ek, ta, tb, tc, tu, tx, g2, iM, iN, iK, ep, st);
    default: set_error("gemm: bad tile %d x cta_group %d", bn, cg); return PC_ERR_ARG;
  }
}

}  // namespace pp200

extern "C" int pc_gemm_wgrad_pair(int64_t M1, int64_t M2, int64_t N, int64_t K, const void* A1,
                                  int64_t lda1, const void* B1, int64_t ldb1, float* C1, int64_t ldc1,
                                  const void* A2, int64_t lda2, const void* B2, int64_t ldb2, float* C2,
                                  int64_t ldc2, int epilogue, void* aux, int64_t ldaux, void* stream) {
  PP_CHECK_ARG(M1 > 0 && M2 > 0 && N > 0 && K > 0, "gemm pair: empty problem");
  const pp200::PairArgs pa{M2, A2, lda2, B2, ldb2, C2, ldc2};
  return pp200::gemm_tc_impl(1, 1, 0, M1, N, K, A1, lda1, B1, ldb1, C1, ldc1, epilogue, nullptr, aux,
                             ldaux, nullptr, 0, static_cast<cudaStream_t>(stream), nullptr, 0, &pa);
}

extern "C" int pc_gemm_tile_choice(int transB, int64_t M, int64_t N, int64_t K, int split_ok,
                                   int* bn, int* cta_pair, int* ksplit) {
  PP_CHECK_ARG(M > 0 && N > 0 && K > 0 && bn && cta_pair && ksplit, "gemm_tile_choice: bad args");
  pp200::choose_tiles(transB != 0, M, N, K, split_ok != 0, bn, cta_pair, ksplit,
                      split_ok == 2 ? pp200::g_max_split : 2, split_ok == 2,
                      split_ok == 2 ? 8.0 : split_ok ? 4.0 : 2.0);
  return PC_OK;
}

extern "C" int pc_gemm_set_tile_n(int bn) {
  if (bn != 0 && bn != 64 && bn != 128 && bn != 192 && bn != 256) {
    pp200::set_error("tile width must be 0, 64, 128, 192 or 256");
    return PC_ERR_ARG;
  }
  pp200::g_force_bn = bn;
  return PC_OK;
}

extern "C" int pc_gemm_set_max_split(int ks) {
  if (ks != 1 && ks != 2 && ks != 4 && ks != 8) {
    pp200::set_error("max split must be 1, 2, 4 or 8");
    return PC_ERR_ARG;
  }
  pp200::g_max_split = ks;
  return PC_OK;
}

extern "C" int pc_gemm_set_cta_pair(int mode) {
  if (mode < 0 || mode > 2) {
    pp200::set_error("cta pair mode must be 0 (auto), 1 (never) or 2 (always)");
    return PC_ERR_ARG;
  }
  pp200::g_cta_pair = mode;
  return PC_OK;
}

// Profiling ablation (results are garbage while set): bit0 = skip the epilogue
// work, bit1 = skip the operand TMA loads.
extern "C" int pc_gemm_set_ablation(int bits) {
  pp200::g_ablate = bits & 7;
  return PC_OK;
}

extern "C" int pc_gemm_set_tma_store(int on) {
  pp200::g_tma_store = on ? 1 : 0;
  return PC_OK;
}
