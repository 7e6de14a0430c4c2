// gemm_mbar.cuh -- the GEMM main loop with mbarrier-tracked cp.async stages
// instead of a CTA-wide __syncthreads per k-tile.  Same tile body as
// gemm_kernel.cuh (load_tile, mac_step, k = 0 peel, masked epilogue), so the
// per-element order and the results are identical; only the synchronisation
// differs:
//  * "full" mbarrier per stage, expected count THREADS: every thread's
//    cp.async.mbarrier.arrive.noinc fires when that thread's copies of the
//    stage have landed;
//  * "empty" mbarrier per stage, expected count = warps: lane 0 of each warp
//    arrives once the warp has finished reading the stage;
//  * STAGES >= 3 slots, and the tile issued at iteration kt goes into the
//    slot freed at iteration kt-2, so a warp waits only when another warp is
//    two k-tiles behind (with __syncthreads every warp waits for the slowest
//    at every k-tile: ~1.6 % of warp time on DD n=8192, ncu "barrier").
#pragma once

#include "gemm_kernel.cuh"

namespace mpfk {
namespace kern {

__device__ __forceinline__ unsigned mb_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mb_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(mb_addr(bar)) : "memory");
}
// this thread's prior cp.async copies count as one arrival once complete
__device__ __forceinline__ void mb_cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(mb_addr(bar)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "MB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra MB_WAIT_%=;\n"
      "}\n" ::"r"(mb_addr(bar)),
      "r"(parity)
      : "memory");
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) mpgemm_mbar_kernel(const GemmArgs g) {
  constexpr int W = Cfg::W, BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, TX = Cfg::TX, TY = Cfg::TY;
  constexpr int S = Cfg::STAGES, D = S - 3;  // tiles issued ahead of the current one
  constexpr int NWARPS = Cfg::THREADS / 32;
  static_assert(S >= 3, "the mbarrier pipeline needs a spare stage");
  extern __shared__ __align__(16) double smem[];
  __shared__ uint64_t full[S], empty[S];
  double* As0 = smem;
  double* Bs0 = smem + S * Cfg::A_STAGE;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      mb_init(&full[s], Cfg::THREADS);
      mb_init(&empty[s], NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int tiles_m = (g.M + BM - 1) / BM, tiles_n = (g.N + BN - 1) / BN;
  int tile_m, tile_n;
  tile_coords<Cfg::GROUP_M>(blockIdx.x, tiles_m, tiles_n, tile_m, tile_n);
  const int m0 = tile_m * BM, n0 = tile_n * BN;
  const int ktiles = (g.K + BK - 1) / BK;

  double acc[TM][TN][W];
  if (g.accumulate) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int gm = m0 + ty + i * TY, gn = n0 + tx + j * TX;
        const bool ok = gm < g.M && gn < g.N;
#pragma unroll
        for (int w = 0; w < W; ++w) acc[i][j][w] = ok ? g.C[w * g.pc + (long long)gm * g.ldc + gn] : 0.0;
      }
  }

  // prologue: tiles 0..D (first use of their slots: nothing to wait for)
#pragma unroll
  for (int t = 0; t <= D; ++t) {
    if (t < ktiles) {
      load_tile<Cfg>(As0 + t * Cfg::A_STAGE, Bs0 + t * Cfg::B_STAGE, g, m0, n0, t * BK);
      mb_cp_async_arrive(&full[t]);
    }
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    {
      const int nt = kt + D + 1;
      if (nt < ktiles) {
        const int ns = nt % S;
        if (nt >= S) mb_wait(&empty[ns], ((nt - S) / S) & 1);  // tile nt - S = kt - 2 released
        load_tile<Cfg>(As0 + ns * Cfg::A_STAGE, Bs0 + ns * Cfg::B_STAGE, g, m0, n0, nt * BK);
        mb_cp_async_arrive(&full[ns]);
      }
    }
    const int slot = kt % S;
    mb_wait(&full[slot], (kt / S) & 1);
    const double* As = As0 + slot * Cfg::A_STAGE;
    const double* Bs = Bs0 + slot * Cfg::B_STAGE;
    const int kend = min(BK, g.K - kt * BK);
    int kk = 0;
    if (kt == 0 && !g.accumulate) {
      double a[TM][W], b[TN][W];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int w = 0; w < W; ++w) a[i][w] = As[w * BM * Cfg::AS + (ty + i * TY) * Cfg::AS];
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int w = 0; w < W; ++w) b[j][w] = Bs[w * BK * Cfg::BS + tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) arith::mp_mul<W>(a[i], b[j], acc[i][j]);
      kk = 1;
    }
#pragma unroll Cfg::KUNROLL
    for (; kk < kend; ++kk) mac_step<Cfg>(acc, As, Bs, tx, ty, kk);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mb_arrive(&empty[slot]);
  }

  if (ktiles == 0) return;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty + i * TY;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gn = n0 + tx + j * TX;
      if (gn >= g.N) continue;
#pragma unroll
      for (int w = 0; w < W; ++w) g.C[w * g.pc + (long long)gm * g.ldc + gn] = acc[i][j][w];
    }
  }
}

}  // namespace kern
}  // namespace mpfk
