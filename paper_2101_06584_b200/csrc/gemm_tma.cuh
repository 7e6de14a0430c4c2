// gemm_tma.cuh -- the DD/TD/QD GEMM with Blackwell bulk-tensor (TMA) tile
// staging and mbarrier pipelines.  Same arithmetic, same per-element order,
// same register micro-tiles as gemm_kernel.cuh (bit-identical results); only
// the data movement differs:
//  * one elected thread issues cp.async.bulk.tensor.3d loads; a single box
//    carries all W component planes of an A or B tile (the planes are the
//    third tensor dimension of the reference's SoA layout);
//  * A tiles land 128-byte swizzled (16-byte chunk c of row r at c ^ (r & 7))
//    so the two rows a warp reads never share a bank; out-of-range rows and
//    columns arrive as zeros (TMA OOB fill);
//  * "full" mbarriers (transaction-counted) replace the CTA-wide
//    __syncthreads: each warp waits only for its data and releases a stage by
//    arriving on its "empty" mbarrier, so warps drift instead of lock-stepping.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "gemm_kernel.cuh"

namespace mpfk {
namespace kern {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// TMA tile layout: A box {BK, BM, W} -> [W][BM][BK] (BK = 16 doubles = 128 B
// rows, 128B-swizzled); B box {BN, BK, W} -> [W][BK][BN] (unswizzled).
template <class Cfg>
struct TmaLayout {
  static constexpr int W = Cfg::W, BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  static_assert(BK == 16, "128-byte swizzled A rows need BK == 16 doubles");
  static constexpr int A_TILE = W * BM * BK;  // doubles
  static constexpr int B_TILE = W * BK * BN;
  static constexpr int A_BYTES = A_TILE * 8, B_BYTES = B_TILE * 8;
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "keep 1024-byte tile alignment");
  static constexpr size_t SMEM = size_t(STAGES) * (A_BYTES + B_BYTES) + 2 * STAGES * 8 + 1024;
};

template <class Cfg>
__device__ __forceinline__ double lds_a(const double* As, int w, int r, int kk) {
  constexpr int BM = Cfg::BM, BK = Cfg::BK;
  return As[w * BM * BK + r * BK + ((((kk >> 1) ^ (r & 7))) << 1) + (kk & 1)];
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
    mpgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const GemmArgs g) {
  using L = TmaLayout<Cfg>;
  constexpr int W = Cfg::W, BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, TX = Cfg::TX, TY = Cfg::TY, STAGES = Cfg::STAGES;
  constexpr int NWARPS = Cfg::THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double* As0 = reinterpret_cast<double*>(base);
  double* Bs0 = reinterpret_cast<double*>(base + STAGES * L::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * (L::A_BYTES + L::B_BYTES));
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31;
  const int tx = tid % TX, ty = tid / TX;
  const int tiles_m = (g.M + BM - 1) / BM, tiles_n = (g.N + BN - 1) / BN;
  int tile_m, tile_n;
  tile_coords<Cfg::GROUP_M>(blockIdx.x, tiles_m, tiles_n, tile_m, tile_n);
  const int m0 = tile_m * BM, n0 = tile_n * BN;
  const int ktiles = (g.K + BK - 1) / BK;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < STAGES && s < ktiles; ++s) {
      mbar_expect_tx(&full[s], L::A_BYTES + L::B_BYTES);
      tma_load_3d(As0 + s * L::A_TILE, &tmA, &full[s], s * BK, m0, 0);
      tma_load_3d(Bs0 + s * L::B_TILE, &tmB, &full[s], n0, s * BK, 0);
    }
  }

  double acc[TM][TN][W];
  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % STAGES;
    const unsigned parity = (kt / STAGES) & 1;
    mbar_wait(&full[s], parity);
    const double* As = As0 + s * L::A_TILE;
    const double* Bs = Bs0 + s * L::B_TILE;
    const int kend = min(BK, g.K - kt * BK);
    int kk = 0;
    if (kt == 0) {
      double a[TM][W], b[TN][W];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int w = 0; w < W; ++w) a[i][w] = lds_a<Cfg>(As, w, ty + i * TY, 0);
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int w = 0; w < W; ++w) b[j][w] = Bs[w * BK * BN + tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) arith::mp_mul<W>(a[i], b[j], acc[i][j]);
      kk = 1;
    }
#pragma unroll Cfg::KUNROLL
    for (; kk < kend; ++kk) {
      double a[TM][W], b[TN][W];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int w = 0; w < W; ++w) a[i][w] = lds_a<Cfg>(As, w, ty + i * TY, kk);
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int w = 0; w < W; ++w) b[j][w] = Bs[w * BK * BN + kk * BN + tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          double p[W];
          arith::mp_mul<W>(a[i], b[j], p);
          arith::mp_add<W>(acc[i][j], p, acc[i][j]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && kt + STAGES < ktiles) {
      mbar_wait(&empty[s], parity);  // every warp has finished reading stage s
      const int nk = (kt + STAGES) * BK;
      mbar_expect_tx(&full[s], L::A_BYTES + L::B_BYTES);
      tma_load_3d(As0 + s * L::A_TILE, &tmA, &full[s], nk, m0, 0);
      tma_load_3d(Bs0 + s * L::B_TILE, &tmB, &full[s], n0, nk, 0);
    }
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

// Round 2 variant (tuning library): dense (unswizzled) A and B tiles, so the
// shared-memory addressing is the product's (A rows of BK doubles read as
// k pairs, B columns in adjacent pairs: TileCfg::PAIRB), straight-line
// 16-step full k-tiles (TileCfg::FIXK), and no loader code at all in the
// FP64 warps: thread 0 refills a stage with two bulk tensor copies once
// every warp has released it.  Bank conflicts of the dense A rows (the two
// rows a warp reads are 128 B apart) cost shared-memory wavefronts, which
// run at ~10 % of their rate here, not issue slots.
template <class Cfg>
struct TmaLayout2 {
  static constexpr int W = Cfg::W, BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  static constexpr int A_TILE = W * BM * BK;  // doubles, [W][BM][BK]
  static constexpr int B_TILE = W * BK * BN;  // doubles, [W][BK][BN]
  static constexpr int A_BYTES = A_TILE * 8, B_BYTES = B_TILE * 8;
  static_assert(A_BYTES % 128 == 0 && B_BYTES % 128 == 0, "128-byte aligned stages");
  static constexpr size_t SMEM = size_t(STAGES) * (A_BYTES + B_BYTES) + 2 * STAGES * 8 + 1024;
};

template <class Cfg>
__device__ __forceinline__ void tma2_step(double (&acc)[Cfg::TM][Cfg::TN][Cfg::W], const double* As,
                                          const double* Bs, int tx, int ty, int kk) {
  constexpr int W = Cfg::W, BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, TM = Cfg::TM, TN = Cfg::TN;
  constexpr int TY = Cfg::TY;
  double a[TM][W], b[TN][W];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int w = 0; w < W; ++w) a[i][w] = As[w * BM * BK + (ty + i * TY) * BK + kk];
  if constexpr (Cfg::PAIRB) {
#pragma unroll
    for (int jp = 0; jp < TN / 2; ++jp)
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const double2 v = *reinterpret_cast<const double2*>(Bs + w * BK * BN + kk * BN + bcol<Cfg>(tx, 2 * jp));
        b[2 * jp][w] = v.x;
        b[2 * jp + 1][w] = v.y;
      }
  } else {
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int w = 0; w < W; ++w) b[j][w] = Bs[w * BK * BN + kk * BN + bcol<Cfg>(tx, j)];
  }
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      double p[W];
      arith::mp_mul<W>(a[i], b[j], p);
      arith::mp_add<W>(acc[i][j], p, acc[i][j]);
    }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
    mpgemm_tma2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const GemmArgs g) {
  using L = TmaLayout2<Cfg>;
  constexpr int W = Cfg::W, BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, TX = Cfg::TX, TY = Cfg::TY, STAGES = Cfg::STAGES;
  constexpr int NWARPS = Cfg::THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double* As0 = reinterpret_cast<double*>(base);
  double* Bs0 = reinterpret_cast<double*>(base + STAGES * L::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * (L::A_BYTES + L::B_BYTES));
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31;
  const int tx = tid % TX, ty = tid / TX;
  const int tiles_m = (g.M + BM - 1) / BM, tiles_n = (g.N + BN - 1) / BN;
  int tile_m, tile_n;
  tile_coords<Cfg::GROUP_M>(blockIdx.x, tiles_m, tiles_n, tile_m, tile_n);
  const int m0 = tile_m * BM, n0 = tile_n * BN;
  const int ktiles = (g.K + BK - 1) / BK;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < STAGES && s < ktiles; ++s) {
      mbar_expect_tx(&full[s], L::A_BYTES + L::B_BYTES);
      tma_load_3d(As0 + s * L::A_TILE, &tmA, &full[s], s * BK, m0, 0);
      tma_load_3d(Bs0 + s * L::B_TILE, &tmB, &full[s], n0, s * BK, 0);
    }
  }

  double acc[TM][TN][W];
  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % STAGES;
    const unsigned parity = (kt / STAGES) & 1;
    mbar_wait(&full[s], parity);
    const double* As = As0 + s * L::A_TILE;
    const double* Bs = Bs0 + s * L::B_TILE;
    const int kend = min(BK, g.K - kt * BK);
    int kk = 0;
    if (kt == 0) {
      double a[TM][W], b[TN][W];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int w = 0; w < W; ++w) a[i][w] = As[w * BM * BK + (ty + i * TY) * BK];
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int w = 0; w < W; ++w) b[j][w] = Bs[w * BK * BN + bcol<Cfg>(tx, j)];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) arith::mp_mul<W>(a[i], b[j], acc[i][j]);
      kk = 1;
    }
    if (kk == 0 && kend == BK) {
#pragma unroll
      for (int q = 0; q < BK; ++q) tma2_step<Cfg>(acc, As, Bs, tx, ty, q);
    } else {
#pragma unroll 1
      for (; kk < kend; ++kk) tma2_step<Cfg>(acc, As, Bs, tx, ty, kk);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && kt + STAGES < ktiles) {
      mbar_wait(&empty[s], parity);  // every warp has finished reading stage s
      const int nk = (kt + STAGES) * BK;
      mbar_expect_tx(&full[s], L::A_BYTES + L::B_BYTES);
      tma_load_3d(As0 + s * L::A_TILE, &tmA, &full[s], nk, m0, 0);
      tma_load_3d(Bs0 + s * L::B_TILE, &tmB, &full[s], n0, nk, 0);
    }
  }
  if (ktiles == 0) return;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty + i * TY;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gn = n0 + bcol<Cfg>(tx, j);
      if (gn >= g.N) continue;
#pragma unroll
      for (int w = 0; w < W; ++w) g.C[w * g.pc + (long long)gm * g.ldc + gn] = acc[i][j][w];
    }
  }
}

// Host: tensor maps for the A and B operands of one call.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 3-D map over (inner, outer, W planes) with an {bx, by, W} box.
inline bool make_map(CUtensorMap* map, const double* base, uint64_t inner, uint64_t outer, uint64_t ld,
                     uint64_t plane, int W, int bx, int by, bool swizzle128) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  const cuuint64_t dims[3] = {inner, outer, (cuuint64_t)W};
  const cuuint64_t strides[2] = {ld * 8, plane * 8};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)W};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class Cfg>
cudaError_t launch_tma(const GemmArgs& g, cudaStream_t s) {
  using L = TmaLayout<Cfg>;
  CUtensorMap ma, mb;
  if (!make_map(&ma, g.A, g.K, g.M, g.lda, g.pa, Cfg::W, Cfg::BK, Cfg::BM, true) ||
      !make_map(&mb, g.B, g.N, g.K, g.ldb, g.pb, Cfg::W, Cfg::BN, Cfg::BK, false))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(mpgemm_tma_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)L::SMEM);
  if (e != cudaSuccess) return e;
  const long long tiles = (long long)((g.N + Cfg::BN - 1) / Cfg::BN) * ((g.M + Cfg::BM - 1) / Cfg::BM);
  mpgemm_tma_kernel<Cfg><<<(unsigned)tiles, Cfg::THREADS, L::SMEM, s>>>(ma, mb, g);
  return cudaGetLastError();
}

template <class Cfg>
cudaError_t launch_tma2(const GemmArgs& g, cudaStream_t s) {
  using L = TmaLayout2<Cfg>;
  CUtensorMap ma, mb;
  if (!make_map(&ma, g.A, g.K, g.M, g.lda, g.pa, Cfg::W, Cfg::BK, Cfg::BM, false) ||
      !make_map(&mb, g.B, g.N, g.K, g.ldb, g.pb, Cfg::W, Cfg::BN, Cfg::BK, false))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(mpgemm_tma2_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)L::SMEM);
  if (e != cudaSuccess) return e;
  const long long tiles = (long long)((g.N + Cfg::BN - 1) / Cfg::BN) * ((g.M + Cfg::BM - 1) / Cfg::BM);
  mpgemm_tma2_kernel<Cfg><<<(unsigned)tiles, Cfg::THREADS, L::SMEM, s>>>(ma, mb, g);
  return cudaGetLastError();
}

}  // namespace kern
}  // namespace mpfk
