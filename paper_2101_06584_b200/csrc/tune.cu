// tune.cu -- tile-configuration sweep for the GEMM kernel (libmpfk_tune.so).
// Not part of the product library: scripts/tune.py times every entry on the
// B200 on device-resident BASELINE inputs and checks each result bitwise
// against the product kernel, to pick the tiles compiled into capi.cu.
#include <cuda_runtime.h>

#include "gemm_kernel.cuh"
#include "gemm_tma.cuh"

using namespace mpfk::kern;

namespace {
struct Entry {
  int W;
  const char* name;
  cudaError_t (*run)(const GemmArgs&, cudaStream_t);
  cudaError_t (*info)(int*, int*, int*);
};

template <class Cfg>
cudaError_t run_cfg(const GemmArgs& g, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(mpgemm_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Cfg::SMEM);
  if (e != cudaSuccess) return e;
  const long long tiles = (long long)((g.N + Cfg::BN - 1) / Cfg::BN) * ((g.M + Cfg::BM - 1) / Cfg::BM);
  mpgemm_kernel<Cfg><<<(unsigned)tiles, Cfg::THREADS, Cfg::SMEM, s>>>(g);
  return cudaGetLastError();
}

template <class Cfg>
cudaError_t run_tma_cfg(const GemmArgs& g, cudaStream_t s) {
  return launch_tma<Cfg>(g, s);
}

template <class Cfg>
cudaError_t info_tma_cfg(int* regs, int* smem, int* threads) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, mpgemm_tma_kernel<Cfg>);
  *regs = a.numRegs;
  *smem = (int)TmaLayout<Cfg>::SMEM;
  *threads = Cfg::THREADS;
  return e;
}

template <class Cfg>
cudaError_t info_cfg(int* regs, int* smem, int* threads) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, mpgemm_kernel<Cfg>);
  *regs = a.numRegs;
  *smem = (int)Cfg::SMEM;
  *threads = Cfg::THREADS;
  return e;
}

#define E(W, BM, BN, BK, TM, TN, ST, KU, GM, MB)                                                   \
  {W, #W "/" #BM "x" #BN "x" #BK "/" #TM "x" #TN "/st" #ST "/ku" #KU "/g" #GM "/mb" #MB,           \
   run_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB>>, info_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB>>}

#define T(W, BM, BN, BK, TM, TN, ST, KU, GM, MB)                                                   \
  {W, "tma/" #W "/" #BM "x" #BN "x" #BK "/" #TM "x" #TN "/st" #ST "/ku" #KU "/g" #GM "/mb" #MB,     \
   run_tma_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB>>,                                    \
   info_tma_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB>>}

#define F(W, BM, BN, BK, TM, TN, ST, KU, GM, MB, FX)                                                \
  {W, #W "/" #BM "x" #BN "x" #BK "/" #TM "x" #TN "/st" #ST "/ku" #KU "/g" #GM "/mb" #MB "/fixk" #FX,  \
   run_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB, FX>>,                                      \
   info_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB, FX>>}

const Entry kEntries[] = {
    E(2, 64, 64, 16, 4, 4, 2, 2, 16, 2),  // DD product
    E(2, 64, 64, 24, 4, 4, 2, 2, 16, 2),
    E(2, 64, 64, 24, 4, 4, 2, 3, 16, 2),
    E(2, 64, 64, 16, 4, 4, 2, 4, 16, 2),
    E(2, 64, 64, 32, 4, 4, 2, 2, 16, 1),
    E(2, 64, 64, 8, 4, 4, 3, 2, 16, 2),
};
}  // namespace

extern "C" {
int tune_count(void) { return (int)(sizeof(kEntries) / sizeof(kEntries[0])); }
int tune_width(int i) { return kEntries[i].W; }
const char* tune_name(int i) { return kEntries[i].name; }
int tune_info(int i, int* regs, int* smem, int* threads) { return (int)kEntries[i].info(regs, smem, threads); }
int tune_run(int i, int M, int N, int K, const double* A, long long lda, long long pa, const double* B,
             long long ldb, long long pb, double* C, long long ldc, long long pc, void* stream) {
  GemmArgs g;
  g.A = A, g.B = B, g.C = C;
  g.lda = lda, g.ldb = ldb, g.ldc = ldc, g.pa = pa, g.pb = pb, g.pc = pc;
  g.M = M, g.N = N, g.K = K;
  g.accumulate = 0;
  g.batch = 1, g.sa = g.sb = g.sc = 0;
  return (int)kEntries[i].run(g, (cudaStream_t)stream);
}
}
