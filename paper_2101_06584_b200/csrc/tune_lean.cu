// tune_lean.cu -- tile-configuration sweep for the MPFK_LEAN GEMM kernels
// (libmpfk_tune_lean.so; the interface of tune.cu, loaded by scripts/tune.py
// through TUNE_LIB with --lean: results are checked against the bit-exact
// product within the north star's tolerance, not bitwise).  Not part of the
// product library.
#include <cuda_runtime.h>

#include "gemm_kernel.cuh"

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
cudaError_t info_cfg(int* regs, int* smem, int* threads) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, mpgemm_kernel<Cfg>);
  *regs = a.numRegs;
  *smem = (int)Cfg::SMEM;
  *threads = Cfg::THREADS;
  return e;
}

// W, BM, BN, BK, TM, TN, STAGES, KUNROLL, GROUP_M, MINB, FIXK, ONEBAR, FLOAD, PAIRB
#define L(W, BM, BN, BK, TM, TN, ST, KU, GM, MB, FX, OB, FL, PB)                                        \
  {W, "lean/" #W "/" #BM "x" #BN "x" #BK "/" #TM "x" #TN "/st" #ST "/ku" #KU "/mb" #MB "/fx" #FX "/ob" #OB "/fl" #FL "/pb" #PB, \
   run_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB, FX, OB, 0, 0, FL, PB, 0, 1>>,                \
   info_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB, FX, OB, 0, 0, FL, PB, 0, 1>>}

// LEAN_ = 2: DD stage-major rows
#define L2(W, BM, BN, BK, TM, TN, ST, KU, GM, MB, FX, OB, FL, PB)                                       \
  {W, "lean2/" #W "/" #BM "x" #BN "x" #BK "/" #TM "x" #TN "/st" #ST "/ku" #KU "/mb" #MB "/fx" #FX "/ob" #OB "/fl" #FL "/pb" #PB, \
   run_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB, FX, OB, 0, 0, FL, PB, 0, 2>>,                \
   info_cfg<TileCfg<W, BM, BN, BK, TM, TN, ST, KU, GM, MB, FX, OB, 0, 0, FL, PB, 0, 2>>}

const Entry kEntries[] = {
    // DD
    L2(2, 64, 64, 16, 4, 4, 2, 16, 16, 2, 1, 1, 1, 1),
    L2(2, 64, 64, 16, 4, 4, 2, 4, 16, 2, 1, 1, 1, 1),
    L2(2, 64, 64, 16, 4, 4, 2, 1, 16, 2, 0, 0, 1, 1),
    L2(2, 32, 32, 16, 2, 2, 2, 16, 16, 4, 1, 1, 1, 1),
    L2(2, 64, 128, 16, 4, 8, 2, 16, 16, 1, 1, 1, 1, 1),
    L2(2, 64, 32, 16, 4, 2, 2, 16, 16, 3, 1, 1, 1, 1),
    L2(2, 32, 64, 16, 2, 4, 2, 16, 16, 3, 1, 1, 1, 1),
    L(2, 64, 32, 16, 4, 2, 2, 16, 16, 3, 1, 1, 1, 1),
    L(2, 32, 64, 16, 2, 4, 2, 16, 16, 3, 1, 1, 1, 1),
    L(2, 64, 64, 16, 4, 4, 2, 1, 16, 2, 0, 0, 1, 1),
    L(2, 64, 64, 16, 4, 4, 2, 2, 16, 2, 1, 1, 1, 1),
    // fewer accumulators per thread at 2 CTAs/SM: registers left for interleaving
    L(2, 64, 32, 16, 4, 2, 2, 16, 16, 2, 1, 1, 1, 1),
    L2(2, 64, 32, 16, 4, 2, 2, 16, 16, 2, 1, 1, 1, 1),
    L(2, 32, 64, 16, 2, 4, 2, 16, 16, 2, 1, 1, 1, 1),
    L2(2, 32, 64, 16, 2, 4, 2, 16, 16, 2, 1, 1, 1, 1),
    L2(2, 128, 32, 16, 8, 2, 2, 16, 16, 2, 1, 1, 1, 1),
    L2(2, 32, 128, 16, 2, 8, 2, 16, 16, 2, 1, 1, 1, 1),
    L2(2, 64, 64, 8, 4, 4, 2, 8, 16, 2, 1, 1, 1, 1),
    L2(2, 64, 64, 32, 4, 4, 2, 32, 16, 2, 1, 1, 1, 1),
    L(2, 64, 64, 16, 4, 4, 2, 16, 16, 2, 1, 1, 1, 1),
    L(2, 64, 64, 16, 4, 4, 2, 4, 16, 2, 1, 1, 1, 1),
    L(2, 64, 64, 16, 4, 4, 2, 16, 16, 2, 1, 1, 0, 1),
    L(2, 64, 64, 16, 4, 4, 3, 16, 16, 2, 1, 1, 1, 1),
    L(2, 32, 32, 16, 2, 2, 2, 16, 16, 4, 1, 1, 1, 1),
    L(2, 64, 32, 16, 4, 2, 2, 16, 16, 4, 1, 1, 1, 1),
    L(2, 32, 64, 16, 2, 4, 2, 16, 16, 4, 1, 1, 1, 1),
    L(2, 128, 64, 16, 8, 4, 2, 16, 16, 1, 1, 1, 1, 1),
    L(2, 64, 128, 16, 4, 8, 2, 16, 16, 1, 1, 1, 1, 1),
    // TD
    L(3, 32, 32, 16, 2, 2, 2, 16, 16, 2, 1, 1, 1, 1),
    L(3, 32, 32, 16, 2, 2, 2, 4, 16, 2, 1, 1, 1, 1),
    L(3, 32, 32, 16, 2, 2, 2, 1, 16, 2, 0, 0, 1, 1),
    L(3, 32, 32, 16, 2, 2, 2, 16, 16, 3, 1, 1, 1, 1),
    L(3, 32, 32, 16, 2, 2, 2, 16, 16, 4, 1, 1, 1, 1),
    L(3, 64, 32, 16, 4, 2, 2, 16, 16, 2, 1, 1, 1, 1),
    L(3, 32, 64, 16, 2, 4, 2, 16, 16, 2, 1, 1, 1, 1),
    L(3, 64, 64, 16, 4, 4, 2, 16, 16, 1, 1, 1, 1, 1),
    L(3, 64, 64, 16, 4, 4, 2, 4, 16, 2, 1, 1, 1, 1),
    // QD
    L(4, 32, 32, 16, 2, 2, 2, 4, 16, 2, 1, 1, 0, 0),
    L(4, 32, 32, 16, 2, 2, 2, 16, 16, 2, 1, 1, 1, 1),
    L(4, 32, 32, 16, 2, 2, 2, 4, 16, 2, 1, 1, 1, 1),
    L(4, 32, 32, 16, 2, 2, 2, 1, 16, 2, 0, 0, 1, 1),
    L(4, 32, 32, 16, 2, 2, 2, 4, 16, 3, 1, 1, 1, 1),
    L(4, 64, 32, 16, 4, 2, 2, 4, 16, 2, 1, 1, 1, 1),
    L(4, 32, 64, 16, 2, 4, 2, 4, 16, 2, 1, 1, 1, 1),
    L(4, 64, 64, 16, 4, 4, 2, 4, 16, 1, 1, 1, 1, 1),
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
