// capi.cu -- host runtime and C ABI of libmpfk.so (declared in include/mpfk.h);
// the host-buffer GEMM drivers live in host_gemm.inl, the pageable-operand
// staging in host_stage.inl, Strassen in strassen.inl, MPFM I/O in mpfm_io.inl.
//
// Replaces the reference's runtime + GEMM drivers:
//   runtime::verify_fp_environment / active_backend  (runtime.cpp:19-81)
//     -> per-device context with a device FP self-test, lazily initialised
//   linalg::matmul_{naive,block,block_parallel}_into (linalg.hpp:346-433)
//     -> shape/n_min validation with the reference's messages, then the
//        sm_100a GEMM kernel on 1..G GPUs with C sharded by row spans
//   run_on_threads (linalg.hpp:314-334) -> one host thread per GPU
//   count_matmul / op counters (linalg.hpp:160-180, linalg.cpp:10-25)
//   rng + fill generators (random.hpp)
#include <cuda.h>  // driver types only: entry points are resolved at run time
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mpfk.h"
#include "ew_kernel.cuh"
#include "gemm_kernel.cuh"
#include "splitk.cuh"
#include "strassen_kernels.cuh"
#include "mpf_arith.cuh"

namespace {

using namespace mpfk;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
thread_local std::string t_err;
thread_local mpfk_stats t_stats{};

struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear sticky-free errors
    // device or pinned-host memory exhausted: the twin of std::bad_alloc
    // (linalg.hpp:116), not a device failure
    fail(e == cudaErrorMemoryAllocation ? MPFK_ENOMEM : MPFK_ECUDA,
         std::string("mpfk: ") + what + ": " + cudaGetErrorString(e));
  }
}

// op counts of the calling thread's current (outermost) entry point call:
// the C++ shim forwards them to the caller's own counters (mpfk_last_op_counts)
thread_local uint64_t t_ops[3];  // adds, muls, leaf multiplies
thread_local int t_depth = 0;

struct CallScope {
  CallScope() {
    if (t_depth++ == 0) t_ops[0] = t_ops[1] = t_ops[2] = 0;
  }
  ~CallScope() { --t_depth; }
};

template <class F>
int guarded(F&& f) {
  CallScope scope;
  try {
    f();
    return MPFK_OK;
  } catch (const Fail& e) {
    t_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    t_err = "std::bad_alloc";
    return MPFK_ENOMEM;
  } catch (const std::exception& e) {
    t_err = e.what();
    return MPFK_ERUNTIME;
  }
}

// ---------------------------------------------------------------------------
// op counters, linalg.cpp:10-25 / count_matmul linalg.hpp:175-180
// ---------------------------------------------------------------------------
std::atomic<uint64_t> g_adds{0}, g_muls{0}, g_leaf{0};

void tally_adds(uint64_t v) {
  g_adds.fetch_add(v, std::memory_order_relaxed);
  t_ops[0] += v;
}
void tally_muls(uint64_t v) {
  g_muls.fetch_add(v, std::memory_order_relaxed);
  t_ops[1] += v;
}
void tally_leaf(uint64_t v) {
  g_leaf.fetch_add(v, std::memory_order_relaxed);
  t_ops[2] += v;
}

void count_matmul(uint64_t m, uint64_t n, uint64_t k) {
  if (k == 0) return;
  tally_muls(m * n * k);
  tally_adds(m * n * (k - 1));
}

// ---------------------------------------------------------------------------
// device self-test, the twin of runtime.cpp:19-38.  Operands come from
// global memory so nothing is constant-folded by the compiler.
// ---------------------------------------------------------------------------
__global__ void selftest_kernel(const double* in, int* ok) {
  const double one = in[0], tiny = in[1], three_half = in[2], big = in[3], c = in[4];
  bool r = true;
  r &= __dadd_rn(one, tiny) == 1.0;                     // tie -> even
  r &= __dsub_rn(-one, tiny) == -1.0;
  r &= __dadd_rn(one, three_half) == 1.0 + 0x1p-52;     // above the tie rounds away
  r &= __dsub_rn(-one, three_half) == -1.0 - 0x1p-52;
  const bool rn = r;
  const bool fused = __fma_rn(big, big, c) == 1.0;      // (2^27+1)^2 - (2^54+2^28)
  *ok = (rn ? 1 : 0) | (fused ? 2 : 0);
}

constexpr int kMaxChunks = 16;  // row chunks / K panels of a host-buffer GEMM
constexpr int kStagedPanels = 8;  // K panels of mpfk_gemm_device_staged

#include "host_stage.inl"

struct Device {
  int id = -1;
  bool ready = false;
  cudaStream_t stream = nullptr;  // compute
  cudaStream_t up = nullptr;      // host->device copies
  cudaStream_t down = nullptr;    // device->host copies
  cudaStream_t stream2 = nullptr; // second compute stream: chunk c+1 fills chunk c's tail
  cudaEvent_t ev[6] = {};
  cudaEvent_t evB[kMaxChunks] = {};  // B K-panel p resident (single-GPU path)
  cudaEvent_t evJ = nullptr;         // join of the second compute stream
  cudaEvent_t evA[kMaxChunks] = {};  // A row chunk c resident
  cudaEvent_t evC[kMaxChunks] = {};  // C row chunk c computed
  // grow-only operand buffers for the host-buffer path
  double* dA = nullptr;
  double* dB = nullptr;
  double* dC = nullptr;
  size_t capA = 0, capB = 0, capC = 0;
  unsigned* gate = nullptr;  // gated path: K-panel flags + row-band tile counters
  size_t gate_cap = 0;
  cudaStream_t gather = nullptr;   // copy-engine all-gather of B (mpfk_gemm_device_gathered)
  cudaEvent_t evG[3] = {};         // gate reset, gather done, last use of ggate finished
  cudaEvent_t evS[kStagedPanels + 1] = {};  // mpfk_gemm_device_staged: start, K panel p gathered
  unsigned* ggate = nullptr;       // its flags/counters (cudaMalloc'd: stream memory operations
  size_t ggate_cap = 0;            // reject stream-ordered pool memory)
  Stager stage;  // pageable host operands
};

// host<->device pitched copies (strides in doubles): direct DMA for
// page-locked host buffers, the device's staging ring for pageable ones
void copy_h2d(Device& D, bool pinned, double* dst, uint64_t dld, const double* src, uint64_t sld, uint64_t cols,
              uint64_t rows, cudaStream_t st) {
  if (!cols || !rows) return;
  if (pinned)
    ck(cudaMemcpy2DAsync(dst, dld * 8, src, sld * 8, cols * 8, rows, cudaMemcpyHostToDevice, st), "H2D");
  else
    D.stage.h2d(dst, dld * 8, src, sld * 8, cols * 8, rows, st);
}

void copy_d2h(Device& D, bool pinned, double* dst, uint64_t dld, const double* src, uint64_t sld, uint64_t cols,
              uint64_t rows, cudaStream_t st) {
  if (!cols || !rows) return;
  if (pinned)
    ck(cudaMemcpy2DAsync(dst, dld * 8, src, sld * 8, cols * 8, rows, cudaMemcpyDeviceToHost, st), "D2H");
  else
    D.stage.d2h(dst, dld * 8, src, sld * 8, cols * 8, rows, st);
}

std::mutex g_mu;
// Host-buffer calls share each device's grow-only operand buffers, streams
// and events; they are serialised (each call is synchronous, like the
// reference's).  Device-resident entry points run on the caller's stream and
// take no lock.
std::mutex g_call_mu;
// mpfk_gemm_device_gathered: one lock per device for its flag buffer
std::mutex g_gather_mu[64];
std::vector<Device> g_dev;
int g_ndev = -1;

int visible_sm100_devices() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int usable = 0;
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, d) != cudaSuccess) continue;
    if (p.major == 10 && p.minor == 0) ++usable;
  }
  // (a box mixing sm_100 with other GPUs is not supported: the first
  // `usable` ordinals are taken to be the sm_100 devices)
  return usable;
}

// The device table, built once.  Caller holds g_mu.
// Testing hook: MPFK_EMULATED_DEVICES=N presents N logical devices that all
// live on physical device 0 (Device::id is the physical ordinal), so the
// multi-GPU host path -- row shards, B slices gathered with peer copies, one
// host thread per device -- runs on a one-GPU box.  The "peer" copies are
// then device-local copies ordered by events; no kernel waits on another.
void build_device_table_locked() {
  if (g_ndev >= 0) return;
  const int phys = visible_sm100_devices();
  const char* emu = std::getenv("MPFK_EMULATED_DEVICES");
  const int n = (phys > 0 && emu && std::atoi(emu) > 0) ? std::atoi(emu) : phys;
  g_ndev = n;
  g_dev.resize(std::max(n, 0));
  for (int d = 0; d < n; ++d) g_dev[d].id = n == phys ? d : 0;
}

void init_device_table_locked() {
  build_device_table_locked();
  if (g_ndev == 0)
    fail(MPFK_ENODEV, "mpfk: no CUDA sm_100 device is visible; the GPU library has no CPU fallback");
}

void run_selftest_current() {
  const double h_in[5] = {1.0, 0x1p-53, 0x1.8p-53, 0x1p27 + 1.0, -(0x1p54 + 0x1p28)};
  double* d_in = nullptr;
  int* d_ok = nullptr;
  ck(cudaMalloc(&d_in, sizeof h_in), "cudaMalloc(selftest)");
  ck(cudaMalloc(&d_ok, sizeof(int)), "cudaMalloc(selftest)");
  ck(cudaMemcpy(d_in, h_in, sizeof h_in, cudaMemcpyHostToDevice), "selftest H2D");
  selftest_kernel<<<1, 1>>>(d_in, d_ok);
  ck(cudaGetLastError(), "selftest launch");
  int ok = 0;
  ck(cudaMemcpy(&ok, d_ok, sizeof ok, cudaMemcpyDeviceToHost), "selftest D2H");
  cudaFree(d_in);
  cudaFree(d_ok);
  // testing hook: MPFK_SELFTEST_INJECT=rn|fma reports that probe as failed,
  // so the error path (status MPFK_ERUNTIME -> std::runtime_error, as
  // runtime.cpp:73-80 throws) can be exercised on a healthy GPU
  if (const char* inj = std::getenv("MPFK_SELFTEST_INJECT")) {
    if (!std::strcmp(inj, "rn")) ok &= ~1;
    if (!std::strcmp(inj, "fma")) ok &= ~2;
  }
  if (!(ok & 1))
    fail(MPFK_ERUNTIME,
         "mpfk: binary64 arithmetic is not rounding to nearest-even; "
         "the extended-precision kernels are unusable in this environment");
  if (!(ok & 2))
    fail(MPFK_ERUNTIME,
         "mpfk: fma is not a correctly rounded fused multiply-add; "
         "the extended-precision kernels are unusable in this environment");
}

// Lazily initialise `n` devices starting at `first` (wrapping), e.g. the
// caller's current device and its successors.  Only those devices get a
// context, so one process per GPU (torchrun) touches only its own GPU.
// Caller holds no lock.
void ensure_devices(int n, int first = 0) {
  std::lock_guard<std::mutex> lk(g_mu);
  init_device_table_locked();
  if (n > g_ndev) n = g_ndev;
  int prev = 0;
  cudaGetDevice(&prev);
  for (int i = 0; i < n; ++i) {
    const int d = (first + i) % g_ndev;
    Device& D = g_dev[d];
    if (D.ready) continue;
    ck(cudaSetDevice(D.id), "cudaSetDevice");
    run_selftest_current();
    ck(cudaStreamCreateWithFlags(&D.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&D.up, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&D.down, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&D.stream2, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&D.gather, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& e : D.evG) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    for (auto& e : D.evS) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    for (auto& e : D.evB) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&D.evJ, cudaEventDisableTiming), "cudaEventCreate");
    for (auto& e : D.ev) ck(cudaEventCreate(&e), "cudaEventCreate");
    for (auto& e : D.evA) ck(cudaEventCreate(&e), "cudaEventCreate");
    for (auto& e : D.evC) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    // keep stream-ordered scratch (Strassen levels) mapped between calls
    // instead of returning it to the OS at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, D.id) == cudaSuccess) {
      uint64_t keep = ~uint64_t(0);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    D.ready = true;
  }
  cudaSetDevice(prev);
}

// The caller's current device; MPFK_ENODEV (no fallback) when none is usable.
int current_device() {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    init_device_table_locked();
  }
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  return dev;
}

void grow(double*& p, size_t& cap, size_t bytes) {
  if (bytes <= cap) return;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  ck(cudaMalloc(&p, bytes), "cudaMalloc(operand buffer)");
  cap = bytes;
}

// ---------------------------------------------------------------------------
// kernel dispatch per width
// ---------------------------------------------------------------------------
// Tile configurations chosen by the sweep in scripts/tune.py over
// csrc/tune.cu (profiles/r01_tune.log): the occupancy floor (MINB) matters
// most -- it caps registers so 2-3 CTAs share each SM's FP64 pipe.
// DD: full k-tiles as one straight-line 16-step block (FIXK, KUNROLL 16) and
// one barrier per k-tile (ONEBAR): +1 % (profiles/r01_tune_dd_fixk.log)
using Cfg2 = kern::TileCfg<2, 64, 64, 16, 4, 4, 2, 16, 16, 2, 1, 1>;   // DD, large problems
using Cfg2s = kern::TileCfg<2, 32, 32, 16, 2, 2, 2, 16, 16, 4, 1, 1>;  // DD, few waves
// TD / QD: branch- and select-free common paths in the k loop with an exact
// warp-level redo of any k-tile that met an input outside them
// (TileCfg::FASTR / VSEBF; profiles/r01_tune_fastr.log, r01_tune_levels.log):
// TD renorm5 paths A/B + td_mul's vseb common case (n=4096 0.978 -> 1.030 of
// peak in counted ops), QD renorm5 path A only (0.928 -> 0.962).  Path B is
// common for TD (its zero-extended fourth lane), so TD keeps it in the fast form.
// Paired B columns (TileCfg::PAIRB, round 2; profiles/r02/tune_pairb.log,
// tune_tdqd_flpb.log): half the B shared loads -- DD n=4096 +0.5 %, DD n=1024
// +1 %, TD n=4096 +1.2 % with the 32-bit fast-loader state; QD neutral, it
// keeps the strided columns and the general loader.
using Cfg3 = kern::TileCfg<3, 32, 32, 16, 2, 2, 2, 1, 16, 2, 0, 0, 1, 1, 1, 1>;  // TD: renorm5 A/B, vseb fast
// The interior fast loader (TileCfg::FLOAD, round 2; profiles/r02/tune_fload.log):
// DD n=1024 1.330 -> 1.288 ms, DD n=4096 -0.7 %, TD n=4096 -0.5 %; QD keeps the
// general loader (+0.5 % with it: its 128-register budget spills the loader state)
using Cfg4 = kern::TileCfg<4, 32, 32, 16, 2, 2, 2, 4, 16, 2, 1, 1, 2, 0, 0, 0>;  // QD: renorm5 path A, 4-step unroll
// the copy-engine-gated QD launch keeps the 1-step loop: with the 4-step
// straight-line k-tiles and one barrier per k-tile it ran 25 ms slower at
// n=4096 (e2e 891 vs 864 ms; the per-panel flag wait after the k-tile's
// barrier is the culprit -- 4-step tiles with two barriers measure 867 ms)
using Cfg4g = kern::TileCfg<4, 32, 32, 16, 2, 2, 2, 1, 16, 2, 0, 0, 2, 0, 0, 0>;
// MPFK_LEAN (csrc/mpf_lean.cuh: 10 / 42 / 107 FP64 instructions per
// multiply-add, tolerance mode).  Tiles from the sweep of csrc/tune_lean.cu
// (scripts/tune.py --lean, profiles/r02/tune_lean.log): straight-line
// k-tiles, one barrier, fast loader and paired B columns for every width;
// TD at 3 CTAs/SM (80 registers), QD at 2.  DD (LEAN = 2: a micro-tile row's
// operations written stage by stage, +0.4 %) stays at 0.87-0.88 of the FP64
// pipe for every tile, occupancy and instruction order tried (32x32 .. 64x128,
// 1-4 CTAs/SM; TD 0.95, QD 0.97): a quarter of its FP64 instructions are
// three-operand DFMAs (bit-exact DD: one in twenty).
using CfgL2 = kern::TileCfg<2, 64, 64, 16, 4, 4, 2, 16, 16, 2, 1, 1, 0, 0, 1, 1, 0, 2>;
using CfgL2s = kern::TileCfg<2, 32, 32, 16, 2, 2, 2, 16, 16, 4, 1, 1, 0, 0, 1, 1, 0, 1>;  // (element-major: +2 % at n=1024)
using CfgL3 = kern::TileCfg<3, 32, 32, 16, 2, 2, 2, 16, 16, 3, 1, 1, 0, 0, 1, 1, 0, 1>;
using CfgL4 = kern::TileCfg<4, 32, 32, 16, 2, 2, 2, 4, 16, 2, 1, 1, 0, 0, 1, 1, 0, 1>;

template <class Cfg>
void configure_once() {
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    ck(cudaFuncSetAttribute(kern::mpgemm_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)Cfg::SMEM),
       "cudaFuncSetAttribute");
    configured_dev = dev;
  }
}

template <class Cfg>
long long tiles_of(const kern::GemmArgs& g) {
  return (long long)((g.N + Cfg::BN - 1) / Cfg::BN) * ((g.M + Cfg::BM - 1) / Cfg::BM) * std::max(g.batch, 1);
}

// Expected fraction of FP64 peak: steady-state efficiency of the tile shape
// (measured by the sweep) times the per-SM balance of the tile count -- the
// FP64 pipe is shared by all CTAs resident on an SM, so what quantises is
// tiles per SM (tiles / SMs vs its ceiling), e.g. DD n=1024: 256 64x64 tiles
// -> 1.73 per SM (0.86), 1024 32x32 tiles -> 6.92 per SM (0.99) -- times the
// share of tile cells inside the m x n output.
template <class Cfg>
double predicted_eff(const kern::GemmArgs& g, double steady) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const double per_sm = double(tiles_of<Cfg>(g)) / std::max(sms, 1);
  // cells of the tiles that hold output (edge tiles compute masked cells too)
  const double useful = double(g.M) * g.N /
                        (double((g.M + Cfg::BM - 1) / Cfg::BM * Cfg::BM) * ((g.N + Cfg::BN - 1) / Cfg::BN * Cfg::BN));
  return steady * useful * per_sm / std::ceil(per_sm);
}

// DD: the 32x32 tiles when the 64x64 grid would leave SMs unevenly loaded
// (steady-state efficiencies with the interior fast loader at n=4096:
// 0.941 / 0.950, profiles/r02/tune_fload.log); one rule for every
// launch path (plain, split-K, fused all-gather, gated, host chunking)
bool dd_small_tiles(const kern::GemmArgs& g) {
  return predicted_eff<Cfg2s>(g, 0.935) > predicted_eff<Cfg2>(g, 0.948);
}
// the same rule for the lean DD tiles (steady: 0.865 / 0.874 of the pipe at n=4096)
bool dd_small_tiles_lean(const kern::GemmArgs& g) {
  return predicted_eff<CfgL2s>(g, 0.865) > predicted_eff<CfgL2>(g, 0.874);
}

template <class Cfg>
void launch_cfg(const kern::GemmArgs& g, cudaStream_t s) {
  configure_once<Cfg>();
  const long long tiles = tiles_of<Cfg>(g);
  if (tiles > 0x7fffffffLL) fail(MPFK_EINVAL, "mpfk: too many tiles");
  kern::mpgemm_kernel<Cfg><<<(unsigned)tiles, Cfg::THREADS, Cfg::SMEM, s>>>(g);
  ck(cudaGetLastError(), "GEMM kernel launch");
}

__global__ void zero_planes_kernel(double* C, long long ldc, long long pc, int M, int N, int W) {
  const long long total = (long long)W * M * N;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int w = (int)(t / ((long long)M * N));
    const long long r = t % ((long long)M * N);
    C[w * pc + (r / N) * ldc + (r % N)] = 0.0;
  }
}

// Enqueue C = A*B on the current device.  Returns kernel launches.
// lean: the MPFK_LEAN arithmetic (tolerance mode) instead of the reference's.
int dispatch_gemm(int W, const kern::GemmArgs& g, cudaStream_t s, bool lean = false);

// accumulate: continue the chains already in C over this K panel (see
// GemmArgs::accumulate); k == 0 is then a no-op.
int enqueue_gemm(int W, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                 uint64_t pa, const double* B, uint64_t ldb, uint64_t pb, double* C,
                 uint64_t ldc, uint64_t pc, cudaStream_t s, bool accumulate = false, bool lean = false) {
  if (m == 0 || n == 0) return 0;
  if (k == 0 && accumulate) return 0;
  if (m > 0x7fffffffULL || n > 0x7fffffffULL || k > 0x7fffffffULL)
    fail(MPFK_EINVAL, "mpfk: dimension exceeds 2^31-1");
  if (k == 0) {
    zero_planes_kernel<<<std::min<uint64_t>((W * m * n + 255) / 256, 4096), 256, 0, s>>>(
        C, (long long)ldc, (long long)pc, (int)m, (int)n, W);
    ck(cudaGetLastError(), "zero kernel launch");
    return 1;
  }
  kern::GemmArgs g;
  g.A = A, g.B = B, g.C = C;
  g.lda = (long long)lda, g.ldb = (long long)ldb, g.ldc = (long long)ldc;
  g.pa = (long long)pa, g.pb = (long long)pb, g.pc = (long long)pc;
  g.M = (int)m, g.N = (int)n, g.K = (int)k;
  g.accumulate = accumulate ? 1 : 0;
  g.batch = 1, g.sa = g.sb = g.sc = 0;
  return dispatch_gemm(W, g, s, lean);
}

// A strided batch of `batch` products of one shape (Strassen leaves).
int enqueue_gemm_batched(int W, int batch, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                         uint64_t pa, uint64_t sa, const double* B, uint64_t ldb, uint64_t pb, uint64_t sb,
                         double* C, uint64_t ldc, uint64_t pc, uint64_t sc, cudaStream_t s) {
  if (batch <= 0 || m == 0 || n == 0) return 0;
  if (k == 0) {
    for (int b = 0; b < batch; ++b) enqueue_gemm(W, m, n, 0, A, lda, pa, B, ldb, pb, C + b * sc, ldc, pc, s);
    return batch;
  }
  kern::GemmArgs g;
  g.A = A, g.B = B, g.C = C;
  g.lda = (long long)lda, g.ldb = (long long)ldb, g.ldc = (long long)ldc;
  g.pa = (long long)pa, g.pb = (long long)pb, g.pc = (long long)pc;
  g.M = (int)m, g.N = (int)n, g.K = (int)k;
  g.accumulate = 0;
  g.batch = batch, g.sa = (long long)sa, g.sb = (long long)sb, g.sc = (long long)sc;
  return dispatch_gemm(W, g, s);
}

template <class Cfg>
void launch_pull_cfg(const kern::GemmArgs& g, const kern::PullB& P, cudaStream_t s) {
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    ck(cudaFuncSetAttribute(kern::mpgemm_pull_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)Cfg::SMEM),
       "cudaFuncSetAttribute");
    configured_dev = dev;
  }
  if (P.panel_rows % Cfg::BK) fail(MPFK_EINVAL, "mpfk: panel_rows must be a multiple of 16");
  const long long tiles = tiles_of<Cfg>(g);
  if (tiles > 0x7fffffffLL) fail(MPFK_EINVAL, "mpfk: too many tiles");
  kern::mpgemm_pull_kernel<Cfg><<<(unsigned)tiles, Cfg::THREADS, Cfg::SMEM, s>>>(g, P);
  ck(cudaGetLastError(), "fused all-gather GEMM launch");
}

int dispatch_gemm_pull(int W, const kern::GemmArgs& g, const kern::PullB& P, cudaStream_t s) {
  switch (W) {
    case 2:
      if (dd_small_tiles(g))
        launch_pull_cfg<Cfg2s>(g, P, s);
      else
        launch_pull_cfg<Cfg2>(g, P, s);
      break;
    case 3: launch_pull_cfg<Cfg3>(g, P, s); break;
    case 4: launch_pull_cfg<Cfg4>(g, P, s); break;
    default: fail(MPFK_EINVAL, "mpfk: width must be 2, 3 or 4");
  }
  return 1;
}

template <class Cfg>
void launch_splitk_cfg(const kern::GemmArgs& g, int klast, cudaStream_t s) {
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    ck(cudaFuncSetAttribute(kern::mpgemm_splitk_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)Cfg::SMEM),
       "cudaFuncSetAttribute");
    configured_dev = dev;
  }
  const long long tiles = tiles_of<Cfg>(g);
  if (tiles > 0x7fffffffLL) fail(MPFK_EINVAL, "mpfk: too many tiles");
  kern::mpgemm_splitk_kernel<Cfg><<<(unsigned)tiles, Cfg::THREADS, Cfg::SMEM, s>>>(g, klast);
  ck(cudaGetLastError(), "split-K GEMM launch");
}

int dispatch_gemm_splitk(int W, const kern::GemmArgs& g, int klast, cudaStream_t s) {
  switch (W) {
    case 2:
      if (dd_small_tiles(g))
        launch_splitk_cfg<Cfg2s>(g, klast, s);
      else
        launch_splitk_cfg<Cfg2>(g, klast, s);
      break;
    case 3: launch_splitk_cfg<Cfg3>(g, klast, s); break;
    case 4: launch_splitk_cfg<Cfg4>(g, klast, s); break;
    default: fail(MPFK_EINVAL, "mpfk: width must be 2, 3 or 4");
  }
  return 1;
}

// ---------------------------------------------------------------------------
// copy-engine-gated GEMM (host operands streamed in K panels)
// ---------------------------------------------------------------------------
// Stream memory operations (cuStreamWriteValue32 / cuStreamWaitValue32) are
// driver API; their entry points are resolved through the runtime so the
// library does not link libcuda.  Unavailable -> the chunked host path.
using MemOpFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
MemOpFn g_write32 = nullptr, g_wait32 = nullptr;
std::once_flag g_memops_once;

bool memops_available() {
  std::call_once(g_memops_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &f, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_write32 = reinterpret_cast<MemOpFn>(f);
    f = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait32 = reinterpret_cast<MemOpFn>(f);
    cudaGetLastError();
    if (const char* e = std::getenv("MPFK_NO_GATED"); e && std::atoi(e) > 0) g_write32 = g_wait32 = nullptr;
    if (!g_write32 || !g_wait32) return;
    // probe once on the current device: write a value, wait for it, read it back
    unsigned* d = nullptr;
    cudaStream_t st = nullptr;
    unsigned h = 0;
    bool ok = cudaMalloc(reinterpret_cast<void**>(&d), sizeof(unsigned)) == cudaSuccess &&
              cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMemsetAsync(d, 0, sizeof(unsigned), st) == cudaSuccess &&
              g_write32(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(d), 7, 0) == CUDA_SUCCESS &&
              g_wait32(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(d), 7,
                       CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS &&
              cudaMemcpyAsync(&h, d, sizeof(unsigned), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
              cudaStreamSynchronize(st) == cudaSuccess && h == 7;
    if (st) cudaStreamDestroy(st);
    if (d) cudaFree(d);
    cudaGetLastError();
    if (!ok) g_write32 = g_wait32 = nullptr;
  });
  return g_write32 && g_wait32;
}

void cu_ck(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) fail(MPFK_ECUDA, std::string("mpfk: ") + what + " failed (CUresult " + std::to_string(r) + ")");
}

template <class Cfg>
std::pair<int, int> launch_gated_cfg(const kern::GemmArgs& g, const kern::GateArgs& G, cudaStream_t s) {
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    ck(cudaFuncSetAttribute(kern::mpgemm_gated_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)Cfg::SMEM),
       "cudaFuncSetAttribute");
    configured_dev = dev;
  }
  if (G.panel_rows % Cfg::BK || G.band_rows % Cfg::BM) fail(MPFK_EINVAL, "mpfk: gated panel/band size");
  const long long tiles = tiles_of<Cfg>(g);
  if (tiles > 0x7fffffffLL) fail(MPFK_EINVAL, "mpfk: too many tiles");
  kern::mpgemm_gated_kernel<Cfg><<<(unsigned)tiles, Cfg::THREADS, Cfg::SMEM, s>>>(g, G);
  ck(cudaGetLastError(), "gated GEMM launch");
  return {Cfg::BM, Cfg::BN};
}

// the same configuration choice as dispatch_gemm; returns the tile (BM, BN)
std::pair<int, int> dispatch_gemm_gated(int W, const kern::GemmArgs& g, const kern::GateArgs& G, cudaStream_t s) {
  switch (W) {
    case 2:
      if (dd_small_tiles(g)) return launch_gated_cfg<Cfg2s>(g, G, s);
      return launch_gated_cfg<Cfg2>(g, G, s);
    case 3: return launch_gated_cfg<Cfg3>(g, G, s);
    case 4: return launch_gated_cfg<Cfg4g>(g, G, s);
    default: fail(MPFK_EINVAL, "mpfk: width must be 2, 3 or 4");
  }
}

int dispatch_gemm(int W, const kern::GemmArgs& g, cudaStream_t s, bool lean) {
  if (lean) {
    switch (W) {
      case 2:
        if (dd_small_tiles_lean(g))
          launch_cfg<CfgL2s>(g, s);
        else
          launch_cfg<CfgL2>(g, s);
        break;
      case 3: launch_cfg<CfgL3>(g, s); break;
      case 4: launch_cfg<CfgL4>(g, s); break;
      default: fail(MPFK_EINVAL, "mpfk: width must be 2, 3 or 4");
    }
    return 1;
  }
  switch (W) {
    case 2:
      if (dd_small_tiles(g))
        launch_cfg<Cfg2s>(g, s);
      else
        launch_cfg<Cfg2>(g, s);
      break;
    case 3: launch_cfg<Cfg3>(g, s); break;
    case 4: launch_cfg<Cfg4>(g, s); break;
    default: fail(MPFK_EINVAL, "mpfk: width must be 2, 3 or 4");
  }
  return 1;
}

// ---------------------------------------------------------------------------
// MPFK_FAST: split-K (csrc/splitk.cuh)
// ---------------------------------------------------------------------------
struct SplitK {
  int S;        // K segments (1 = the bit-exact path)
  uint64_t ks;  // segment length (multiple of 16: 16-byte A offsets)
};

// Split K only when the bit-exact launch would leave the GPU under-used
// (predicted efficiency < 0.9: fewer tiles than resident CTA slots, or a
// badly quantised last wave) and k >= 512.  The segment count is the
// smallest whose tiles-per-SM balance x slot occupancy reaches 0.98 (else
// the best), with segments of >= 256 k steps and at most 4096 segments.
SplitK splitk_plan(int W, uint64_t m, uint64_t n, uint64_t k) {
  int BM = Cfg2s::BM, BN = Cfg2s::BN, minb = Cfg2s::MINB;
  if (W == 3) BM = Cfg3::BM, BN = Cfg3::BN, minb = Cfg3::MINB;
  if (W == 4) BM = Cfg4::BM, BN = Cfg4::BN, minb = Cfg4::MINB;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const double tiles = double((m + BM - 1) / BM) * double((n + BN - 1) / BN);
  auto eff = [&](double segs) {
    const double per_sm = tiles * segs / sms;
    return per_sm / std::ceil(per_sm) * std::min(1.0, per_sm / minb);
  };
  if (m == 0 || n == 0 || k < 512 || eff(1) >= 0.9) return {1, k};
  const uint64_t smax = std::min<uint64_t>(k / 256, 4096);
  SplitK best{1, k};
  double best_eff = eff(1);
  for (uint64_t S = 2; S <= smax; ++S) {
    const uint64_t ks = ((k + S - 1) / S + 15) / 16 * 16;
    const uint64_t segs = (k + ks - 1) / ks;
    const double e = eff((double)segs);
    if (e > best_eff + 1e-9) best_eff = e, best = {(int)segs, ks};
    if (best_eff >= 0.98) break;
  }
  return best;
}

// C = A*B with MPFK_FAST on the current device: split-K when the plan says
// so (one batched GEMM launch over the segments + one combine launch, the
// partials in stream-ordered scratch), else exactly enqueue_gemm.
int enqueue_gemm_fast(int W, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                      uint64_t pa, const double* B, uint64_t ldb, uint64_t pb, double* C,
                      uint64_t ldc, uint64_t pc, cudaStream_t s) {
  const SplitK p = splitk_plan(W, m, n, k);
  if (p.S <= 1) return enqueue_gemm(W, m, n, k, A, lda, pa, B, ldb, pb, C, ldc, pc, s);
  if (m > 0x7fffffffULL || n > 0x7fffffffULL || k > 0x7fffffffULL)
    fail(MPFK_EINVAL, "mpfk: dimension exceeds 2^31-1");
  const uint64_t ldw = (n + 1) & ~uint64_t(1), pw = m * ldw, sw = W * pw;
  double* ws = nullptr;
  ck(cudaMallocAsync(reinterpret_cast<void**>(&ws), sizeof(double) * sw * p.S, s), "split-K scratch");
  kern::GemmArgs g;
  g.A = A, g.B = B, g.C = ws;
  g.lda = (long long)lda, g.ldb = (long long)ldb, g.ldc = (long long)ldw;
  g.pa = (long long)pa, g.pb = (long long)pb, g.pc = (long long)pw;
  g.M = (int)m, g.N = (int)n, g.K = (int)p.ks;
  g.accumulate = 0;
  g.batch = p.S, g.sa = (long long)p.ks, g.sb = (long long)(p.ks * ldb), g.sc = (long long)sw;
  const uint64_t klast = k - (uint64_t)(p.S - 1) * p.ks;
  int launches = dispatch_gemm_splitk(W, g, klast == p.ks ? 0 : (int)klast, s);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((m * n + 255) / 256, (uint64_t)sms * 8));
  switch (W) {
    case 2: kern::splitk_reduce_kernel<2><<<blocks, 256, 0, s>>>(ws, ldw, pw, sw, p.S, C, ldc, pc, (int)m, (int)n); break;
    case 3: kern::splitk_reduce_kernel<3><<<blocks, 256, 0, s>>>(ws, ldw, pw, sw, p.S, C, ldc, pc, (int)m, (int)n); break;
    default: kern::splitk_reduce_kernel<4><<<blocks, 256, 0, s>>>(ws, ldw, pw, sw, p.S, C, ldc, pc, (int)m, (int)n); break;
  }
  ck(cudaGetLastError(), "split-K combine launch");
  ck(cudaFreeAsync(ws, s), "split-K scratch free");
  return launches + 1;
}

// Enqueue out = op(a, b) elementwise on the current device.
int enqueue_ew(int W, int op, uint64_t rows, uint64_t cols, double* out, uint64_t ldo, uint64_t po,
               const double* a, uint64_t lda, uint64_t pa, const double* b, uint64_t ldb,
               uint64_t pb, cudaStream_t s) {
  if (rows == 0 || cols == 0) return 0;
  if (rows > 0x7fffffffULL || cols > 0x7fffffffULL) fail(MPFK_EINVAL, "mpfk: dimension exceeds 2^31-1");
  kern::EwArgs g;
  g.out = out, g.a = a, g.b = b;
  g.ldo = (long long)ldo, g.lda = (long long)lda, g.ldb = (long long)ldb;
  g.po = (long long)po, g.pa = (long long)pa, g.pb = (long long)pb;
  g.rows = (int)rows, g.cols = (int)cols;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t work = rows * ((cols + 1) / 2);
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, (uint64_t)sms * 8));
#define MPFK_EW(WW, OO) kern::ew_kernel<WW, OO><<<blocks, 256, 0, s>>>(g)
  switch (W * 4 + op) {
    case 8: MPFK_EW(2, kern::EW_ADD); break;
    case 9: MPFK_EW(2, kern::EW_MUL); break;
    case 12: MPFK_EW(3, kern::EW_ADD); break;
    case 13: MPFK_EW(3, kern::EW_MUL); break;
    case 14: MPFK_EW(3, kern::EW_ADD_MERGE); break;
    case 16: MPFK_EW(4, kern::EW_ADD); break;
    case 17: MPFK_EW(4, kern::EW_MUL); break;
    case 11: MPFK_EW(2, kern::EW_SUB); break;
    case 15: MPFK_EW(3, kern::EW_SUB); break;
    case 19: MPFK_EW(4, kern::EW_SUB); break;
    default: fail(MPFK_EINVAL, "ew: add_merge is a triple-width operation");
  }
#undef MPFK_EW
  ck(cudaGetLastError(), "ew kernel launch");
  return 1;
}

void count_ew(int op, uint64_t rows, uint64_t cols) {  // linalg.hpp:682-683
  if (op == kern::EW_MUL)
    tally_muls(rows * cols);
  else
    tally_adds(rows * cols);
}

void check_width(int W) {
  if (W < 2 || W > 4) fail(MPFK_EINVAL, "mpfk: width must be 2, 3 or 4");
}

uint64_t plane_of(const mpfk_mat* M) {
  return M->plane_stride ? M->plane_stride : M->rows * M->stride;
}

void check_mat(const mpfk_mat* M, const char* name) {
  if (!M) fail(MPFK_EINVAL, std::string("mpfk: null matrix ") + name);
  if (M->stride < M->cols) fail(MPFK_EINVAL, std::string("mpfk: stride < cols for ") + name);
  if (M->rows && M->cols && !M->base) fail(MPFK_EINVAL, std::string("mpfk: null data for ") + name);
}

// check_mul_shapes, linalg.hpp:279-286
void check_mul_shapes(const mpfk_mat* A, const mpfk_mat* B, const mpfk_mat* C) {
  if (A->cols != B->rows) fail(MPFK_EINVAL, "matmul: inner dimensions differ");
  if (C->rows != A->rows || C->cols != B->cols)
    fail(MPFK_EINVAL, "matmul: result shape mismatch");
}

// check_n_min, linalg.hpp:290-294
void check_n_min(uint64_t n_min, int variant) {
  if (variant < MPFK_NORMAL || variant > MPFK_SIMD_LOADSTORE)
    fail(MPFK_EINVAL, "matmul: unknown kernel variant");
  if (n_min < 1) fail(MPFK_EINVAL, "matmul: n_min must be at least 1");
  if (variant != MPFK_NORMAL && n_min % 4 != 0)
    fail(MPFK_EINVAL, "matmul: SIMD variants need n_min divisible by 4");
}

uint64_t pad4(uint64_t c) { return (c + 3) & ~uint64_t(3); }

// host pads of C -> +0 (zero_pads, linalg.hpp:99-106)
void zero_host_pads(int W, mpfk_mat* C) {
  if (C->stride == C->cols || !C->base || C->rows == 0) return;
  const uint64_t pc = plane_of(C);
  for (int w = 0; w < W; ++w)
    for (uint64_t i = 0; i < C->rows; ++i)
      std::memset(C->base + w * pc + i * C->stride + C->cols, 0,
                  (C->stride - C->cols) * sizeof(double));
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

#include "host_gemm.inl"

// ---------------------------------------------------------------------------
// elementwise batch kernel for the arithmetic parity sweeps
// ---------------------------------------------------------------------------
template <int W>
__global__ void binop_kernel(int op, long long count, const double* x, const double* y,
                             double* r) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    double a[W], b[W], c[W];
#pragma unroll
    for (int w = 0; w < W; ++w) a[w] = x[i * W + w], b[w] = y[i * W + w];
    if (op == 0)
      arith::mp_add<W>(a, b, c);
    else if (op == 1 || W != 3)
      arith::mp_mul<W>(a, b, c);
    else if (op == 2)
      arith::td_mul_q(a, b, c);
    else {
      double zb[6];  // the ew kernel's ranked form (per-thread scratch here)
      arith::td_add_merge_ranked(a, b, c, zb, 1);
    }
#pragma unroll
    for (int w = 0; w < W; ++w) r[i * W + w] = c[w];
  }
}

// EFT primitives over a batch (acceptance criterion 1): op 0 two_sum,
// 1 quick_two_sum, 2 two_prod (eft.hpp:46-67)
__global__ void eft_kernel(int op, long long count, const double* a, const double* b, double* s, double* e) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    double x, y;
    if (op == 0) arith::two_sum(a[i], b[i], x, y);
    else if (op == 1) arith::qts(a[i], b[i], x, y);
    else arith::two_prod(a[i], b[i], x, y);
    s[i] = x, e[i] = y;
  }
}

// ---------------------------------------------------------------------------
// FP64 pipe microbenchmark: 8 independent DFMA chains per thread
// ---------------------------------------------------------------------------
__global__ void fp64_peak_kernel(double* out, int iters, double m) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __fma_rn(a[j], m, 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.678) out[0] = s;
}

// ---------------------------------------------------------------------------
// host generator; restated independently in
// oracle/mpfk_oracle.c:orc_fill_baseline for cross-checking
// ---------------------------------------------------------------------------
struct SM64 {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1p-53; }
};

// renormalized<W>(c, W): vec_sum then vseb(W) (mpf.hpp:76-88, eft.hpp:103-225)
void renormalize_host(int W, const double* c, double* out) {
  double d[4];
  double s = c[W - 1];
  for (int i = W - 1; i-- > 0;) {
    double ss, e;
    arith::two_sum(c[i], s, ss, e);
    d[i + 1] = e;
    s = ss;
  }
  d[0] = s;
  for (int i = 0; i < W; ++i) out[i] = 0.0;
  int j = 0;
  double eps = d[0];
  for (int i = 0; i + 1 < W; ++i) {
    double ps, pe;
    arith::qts(eps, d[i + 1], ps, pe);
    out[j] = ps;
    if (arith::nz(pe)) {
      if (j >= W - 1) return;
      ++j;
      eps = pe;
    } else {
      eps = ps;
    }
  }
  if (arith::nz(eps) && j < W) out[j] = eps;
}

// rng::random_normalized<W>, random.hpp:54-67: lead in [1, 2), tails at
// 2^(-53 i) scales, renormalised; redraw the lead if the tail pushed it out.
void random_normalized(int W, SM64& g, double* out) {
  double raw[4];
  raw[0] = 1.0 + g.unit();
  for (int i = 1; i < W; ++i) {
    const uint64_t bits = g.next();
    const double u = static_cast<double>(bits >> 11) * 0x1p-53;
    raw[i] = ((bits & 1) ? -u : u) * std::ldexp(1.0, -53 * i);
  }
  for (int guard = 0; guard < 64; ++guard) {
    renormalize_host(W, raw, out);
    if (out[0] >= 1.0 && out[0] < 2.0) return;
    raw[0] = 1.0 + g.unit();
  }
  for (int i = 0; i < W; ++i) out[i] = 0.0;
  out[0] = 1.0;
}

void baseline_elem(int W, int wide, SM64& g, double* v) {
  double c[4];
  if (wide) {
    const uint64_t sbits = g.next();
    const int e = static_cast<int>(g.next() % 61ULL) - 30;
    const double f = 1.0 + g.unit();
    c[0] = std::ldexp((sbits & 1) ? -f : f, e);
  } else {
    c[0] = 2.0 * g.unit() - 1.0;
  }
  for (int i = 1; i < W; ++i) c[i] = (c[i - 1] * 0x1p-53) * (2.0 * g.unit() - 1.0);
  if (W == 2)
    arith::qts(c[0], c[1], v[0], v[1]);
  else
    renormalize_host(W, c, v);
}

#include "mpfm_io.inl"
#include "strassen.inl"

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int mpfk_abi_version(void) { return MPFK_ABI_VERSION; }

const char* mpfk_last_error(void) { return t_err.c_str(); }

int mpfk_device_count(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  build_device_table_locked();
  return g_ndev;
}

int mpfk_init(int n_gpus) {
  return guarded([&] { ensure_devices(n_gpus <= 0 ? 1 << 20 : n_gpus); });
}

void mpfk_shutdown(void) {
  // the same lock order as the calls (host call, gather, table): no host
  // GEMM, gathered/staged GEMM or table change can be in flight
  std::lock_guard<std::mutex> call_lock(g_call_mu);
  std::vector<std::unique_lock<std::mutex>> gather_locks;
  for (auto& m : g_gather_mu) gather_locks.emplace_back(m);
  std::lock_guard<std::mutex> lk(g_mu);
  int prev = 0;
  cudaGetDevice(&prev);
  for (auto& D : g_dev) {
    if (!D.ready) continue;
    cudaSetDevice(D.id);
    // every library stream (compute, copies, gather) and whatever the
    // device-resident entry points queued on callers' streams
    cudaDeviceSynchronize();
    if (D.dA) cudaFree(D.dA);
    if (D.dB) cudaFree(D.dB);
    if (D.dC) cudaFree(D.dC);
    if (D.gate) cudaFree(D.gate);
    if (D.ggate) cudaFree(D.ggate);
    for (auto& e : D.ev) cudaEventDestroy(e);
    for (auto& e : D.evA) cudaEventDestroy(e);
    for (auto& e : D.evC) cudaEventDestroy(e);
    cudaStreamDestroy(D.stream);
    cudaStreamDestroy(D.up);
    cudaStreamDestroy(D.down);
    cudaStreamDestroy(D.stream2);
    cudaStreamDestroy(D.gather);
    for (auto& e : D.evG) cudaEventDestroy(e);
    for (auto& e : D.evS) cudaEventDestroy(e);
    for (auto& e : D.evB) cudaEventDestroy(e);
    cudaEventDestroy(D.evJ);
    D.stage.release();
    D = Device{};
  }
  g_dev.clear();
  g_ndev = -1;
  host_reg_cache().clear();
  cudaSetDevice(prev);
}

int mpfk_set_device(int dev) {
  return guarded([&] {
    const int n = mpfk_device_count();
    if (n == 0) fail(MPFK_ENODEV, "mpfk: no CUDA sm_100 device is visible; the GPU library has no CPU fallback");
    if (dev < 0 || dev >= n) fail(MPFK_EINVAL, "mpfk: device index out of range");
    int phys = dev;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      phys = g_dev[dev].id;
    }
    ck(cudaSetDevice(phys), "cudaSetDevice");
    ensure_devices(1, dev);
  });
}

int mpfk_get_device(void) {
  int d = -1;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return d;
}

int mpfk_selftest(void) {
  return guarded([&] {
    if (mpfk_device_count() == 0)
      fail(MPFK_ENODEV, "mpfk: no CUDA sm_100 device is visible");
    run_selftest_current();
  });
}

int mpfk_matmul_block_parallel_into(int width, mpfk_mat* C, const mpfk_mat* A, const mpfk_mat* B,
                                    uint64_t n_min, int variant, unsigned workers) {
  return guarded([&] {
    check_width(width);
    check_mat(A, "A");
    check_mat(B, "B");
    check_mat(C, "C");
    check_mul_shapes(A, B, C);
    check_n_min(n_min, variant);
    if (workers < 1) fail(MPFK_EINVAL, "matmul: workers must be at least 1");
    host_gemm(width, C, A, B, workers);
  });
}

int mpfk_matmul_block_into(int width, mpfk_mat* C, const mpfk_mat* A, const mpfk_mat* B,
                           uint64_t n_min, int variant) {
  return guarded([&] {
    check_width(width);
    check_mat(A, "A");
    check_mat(B, "B");
    check_mat(C, "C");
    check_mul_shapes(A, B, C);
    check_n_min(n_min, variant);
    host_gemm(width, C, A, B, 1);
  });
}

int mpfk_matmul_naive_into(int width, mpfk_mat* C, const mpfk_mat* A, const mpfk_mat* B,
                           int variant) {
  return guarded([&] {
    check_width(width);
    check_mat(A, "A");
    check_mat(B, "B");
    check_mat(C, "C");
    check_mul_shapes(A, B, C);
    if (variant < MPFK_NORMAL || variant > MPFK_SIMD_LOADSTORE)
      fail(MPFK_EINVAL, "matmul: unknown kernel variant");
    host_gemm(width, C, A, B, 1);
  });
}

int mpfk_matmul_strassen(int width, mpfk_mat* C, const mpfk_mat* A, const mpfk_mat* B,
                         uint64_t cutoff, uint64_t n_min, int variant, unsigned workers) {
  return guarded([&] {
    check_width(width);
    check_mat(A, "A");
    check_mat(B, "B");
    check_mat(C, "C");
    // matmul_strassen[_parallel], linalg.hpp:582-605
    if (A->cols != B->rows) fail(MPFK_EINVAL, "matmul: inner dimensions differ");
    check_n_min(n_min, variant);
    if (cutoff < 1) fail(MPFK_EINVAL, "matmul: cutoff must be at least 1");
    if (workers < 1) fail(MPFK_EINVAL, "matmul: workers must be at least 1");
    if (C->rows != A->rows || C->cols != B->cols) fail(MPFK_EINVAL, "matmul: result shape mismatch");
    host_strassen(width, C, A, B, cutoff);
  });
}

int mpfk_strassen_device(int width, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                         uint64_t a_plane, const double* B, uint64_t ldb, uint64_t b_plane, double* C,
                         uint64_t ldc, uint64_t c_plane, uint64_t cutoff, void* stream, int* launches) {
  return guarded([&] {
    check_width(width);
    if (cutoff < 1) fail(MPFK_EINVAL, "matmul: cutoff must be at least 1");
    if (lda < k || ldb < n || ldc < n) fail(MPFK_EINVAL, "mpfk: leading dimension too small");
    if ((lda | ldb | ldc | a_plane | b_plane | c_plane) & 1)
      fail(MPFK_EINVAL, "mpfk: device strides must be even (16-byte rows)");
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
         reinterpret_cast<uintptr_t>(C)) & 15)
      fail(MPFK_EINVAL, "mpfk: device operands must be 16-byte aligned");
    const int dev = current_device();
    ensure_devices(1, dev);
    const int l = strassen_device(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane, cutoff,
                                  static_cast<cudaStream_t>(stream));
    if (launches) *launches = l;
  });
}

int mpfk_last_stats(mpfk_stats* out) {
  if (!out) return MPFK_EINVAL;
  *out = t_stats;
  return MPFK_OK;
}

int mpfk_gemm_device(int width, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                     uint64_t a_plane, const double* B, uint64_t ldb, uint64_t b_plane, double* C,
                     uint64_t ldc, uint64_t c_plane, void* stream, int* launches) {
  return guarded([&] {
    check_width(width);
    if (lda < k || ldb < n || ldc < n) fail(MPFK_EINVAL, "mpfk: leading dimension too small");
    if ((lda | ldb | ldc | a_plane | b_plane | c_plane) & 1)
      fail(MPFK_EINVAL, "mpfk: device strides must be even (16-byte rows)");
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
         reinterpret_cast<uintptr_t>(C)) & 15)
      fail(MPFK_EINVAL, "mpfk: device operands must be 16-byte aligned");
    const int dev = current_device();
    ensure_devices(1, dev);
    const int l = enqueue_gemm(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane,
                               static_cast<cudaStream_t>(stream));
    count_matmul(m, n, k);
    if (launches) *launches = l;
  });
}

int mpfk_gemm(int width, const mpfk_mat* A, const mpfk_mat* B, mpfk_mat* C, int n_gpus, unsigned flags) {
  return guarded([&] {
    check_width(width);
    check_mat(A, "A");
    check_mat(B, "B");
    check_mat(C, "C");
    check_mul_shapes(A, B, C);
    if (flags & ~unsigned(MPFK_FAST | MPFK_LEAN)) fail(MPFK_EINVAL, "mpfk: unknown flags");
    // n_gpus <= 0: every visible device (host_gemm caps the count)
    host_gemm(width, C, A, B, n_gpus > 0 ? (unsigned)n_gpus : 1u << 20, (flags & MPFK_FAST) != 0,
              (flags & MPFK_LEAN) != 0);
  });
}

int mpfk_gemm_device_ex(int width, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                        uint64_t a_plane, const double* B, uint64_t ldb, uint64_t b_plane, double* C,
                        uint64_t ldc, uint64_t c_plane, unsigned flags, void* stream, int* launches) {
  return guarded([&] {
    check_width(width);
    if (flags & ~unsigned(MPFK_FAST | MPFK_LEAN)) fail(MPFK_EINVAL, "mpfk: unknown flags");
    if (lda < k || ldb < n || ldc < n) fail(MPFK_EINVAL, "mpfk: leading dimension too small");
    if ((lda | ldb | ldc | a_plane | b_plane | c_plane) & 1)
      fail(MPFK_EINVAL, "mpfk: device strides must be even (16-byte rows)");
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
         reinterpret_cast<uintptr_t>(C)) & 15)
      fail(MPFK_EINVAL, "mpfk: device operands must be 16-byte aligned");
    const int dev = current_device();
    ensure_devices(1, dev);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    // MPFK_FAST splits K (segments in the reference's arithmetic) where the
    // output cannot fill the GPU; otherwise MPFK_LEAN picks the arithmetic
    const bool split = (flags & MPFK_FAST) && splitk_plan(width, m, n, k).S > 1;
    const int l = split ? enqueue_gemm_fast(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane, s)
                        : enqueue_gemm(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane, s,
                                       false, (flags & MPFK_LEAN) != 0);
    count_matmul(m, n, k);
    if (launches) *launches = l;
  });
}

int mpfk_splitk_segments(int width, uint64_t m, uint64_t n, uint64_t k) {
  int segs = 1;
  const int rc = guarded([&] {
    check_width(width);
    const int dev = current_device();
    ensure_devices(1, dev);
    segs = splitk_plan(width, m, n, k).S;
  });
  return rc == MPFK_OK ? segs : -rc;
}

int mpfk_ew_apply_into(int width, int op, mpfk_mat* out, const mpfk_mat* a, const mpfk_mat* b,
                       int variant) {
  return guarded([&] {
    check_width(width);
    check_mat(a, "a");
    check_mat(b, "b");
    check_mat(out, "out");
    if (op < kern::EW_ADD || op > kern::EW_ADD_MERGE) fail(MPFK_EINVAL, "ew: unknown operation");
    if (variant < MPFK_NORMAL || variant > MPFK_SIMD_LOADSTORE)
      fail(MPFK_EINVAL, "ew: unknown kernel variant");
    // linalg.hpp:650-653
    if (!(a->rows == b->rows && a->cols == b->cols) || !(a->rows == out->rows && a->cols == out->cols))
      fail(MPFK_EINVAL, "ew: shape mismatch");
    if (op == kern::EW_ADD_MERGE && width != 3)
      fail(MPFK_EINVAL, "ew: add_merge is a triple-width operation");
    const uint64_t rows = a->rows, cols = a->cols;
    std::lock_guard<std::mutex> call_lock(g_call_mu);
    mpfk_stats st{};
    const auto t0 = std::chrono::steady_clock::now();
    if (rows && cols) {
      const int dev = current_device();
      ensure_devices(1, dev);
      Device& D = g_dev[dev];
      const uint64_t ld = pad4(cols), ps = rows * ld;
      grow(D.dA, D.capA, sizeof(double) * width * ps);
      grow(D.dB, D.capB, sizeof(double) * width * ps);
      grow(D.dC, D.capC, sizeof(double) * width * ps);
      const uint64_t pa = plane_of(a), pb = plane_of(b), po = plane_of(out);
      const bool a_pin = host_operand_pinned(a->base, width, a->rows, a->cols, a->stride, pa),
                 b_pin = host_operand_pinned(b->base, width, b->rows, b->cols, b->stride, pb),
                 o_pin = host_operand_pinned(out->base, width, out->rows, out->cols, out->stride, po);
      D.stage.reset();
      ck(cudaEventRecord(D.ev[0], D.stream), "event");
      for (int w = 0; w < width; ++w) {
        copy_h2d(D, a_pin, D.dA + w * ps, ld, a->base + w * pa, a->stride, cols, rows, D.stream);
        copy_h2d(D, b_pin, D.dB + w * ps, ld, b->base + w * pb, b->stride, cols, rows, D.stream);
      }
      ck(cudaEventRecord(D.ev[1], D.stream), "event");
      st.kernel_launches = enqueue_ew(width, op, rows, cols, D.dC, ld, ps, D.dA, ld, ps, D.dB, ld, ps,
                                      D.stream);
      ck(cudaEventRecord(D.ev[2], D.stream), "event");
      for (int w = 0; w < width; ++w)
        copy_d2h(D, o_pin, out->base + w * po, out->stride, D.dC + w * ps, ld, cols, rows, D.stream);
      ck(cudaEventRecord(D.ev[3], D.stream), "event");
      ck(cudaEventSynchronize(D.ev[3]), "ew execution");
      D.stage.drain();
      float x = 0;
      cudaEventElapsedTime(&x, D.ev[0], D.ev[1]);
      st.h2d_ms = x;
      cudaEventElapsedTime(&x, D.ev[1], D.ev[2]);
      st.kernel_ms = x;
      cudaEventElapsedTime(&x, D.ev[2], D.ev[3]);
      st.d2h_ms = x;
      st.h2d_bytes = 16ull * width * rows * cols;
      st.d2h_bytes = 8ull * width * rows * cols;
      st.n_gpus = 1;
    }
    // the SIMD variants run over the padding and restore it to +0
    // (linalg.hpp:663-680); NORMAL leaves out's pads untouched (:654-657)
    if (variant != MPFK_NORMAL) zero_host_pads(width, out);
    count_ew(op, rows, cols);
    st.total_ms = ms_since(t0);
    t_stats = st;
  });
}

int mpfk_ew_device(int width, int op, uint64_t rows, uint64_t cols, double* out, uint64_t ldo,
                   uint64_t o_plane, const double* a, uint64_t lda, uint64_t a_plane, const double* b,
                   uint64_t ldb, uint64_t b_plane, void* stream, int* launches) {
  return guarded([&] {
    check_width(width);
    if (op < kern::EW_ADD || op > kern::EW_ADD_MERGE) fail(MPFK_EINVAL, "ew: unknown operation");
    if (op == kern::EW_ADD_MERGE && width != 3)
      fail(MPFK_EINVAL, "ew: add_merge is a triple-width operation");
    if (ldo < cols || lda < cols || ldb < cols) fail(MPFK_EINVAL, "mpfk: leading dimension too small");
    if ((ldo | lda | ldb | o_plane | a_plane | b_plane) & 1)
      fail(MPFK_EINVAL, "mpfk: device strides must be even (16-byte rows)");
    if ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(a) |
         reinterpret_cast<uintptr_t>(b)) & 15)
      fail(MPFK_EINVAL, "mpfk: device operands must be 16-byte aligned");
    const int dev = current_device();
    ensure_devices(1, dev);
    const int l = enqueue_ew(width, op, rows, cols, out, ldo, o_plane, a, lda, a_plane, b, ldb, b_plane,
                             static_cast<cudaStream_t>(stream));
    count_ew(op, rows, cols);
    if (launches) *launches = l;
  });
}

int mpfk_gemm_device_acc(int width, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                         uint64_t a_plane, const double* B, uint64_t ldb, uint64_t b_plane, double* C,
                         uint64_t ldc, uint64_t c_plane, void* stream, int* launches) {
  return mpfk_gemm_device_acc_ex(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane, MPFK_BIT_EXACT,
                                 stream, launches);
}

int mpfk_gemm_device_acc_ex(int width, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                            uint64_t a_plane, const double* B, uint64_t ldb, uint64_t b_plane, double* C,
                            uint64_t ldc, uint64_t c_plane, unsigned flags, void* stream, int* launches) {
  return guarded([&] {
    check_width(width);
    // a continuation is one launch over this panel: MPFK_FAST (split K) has no meaning here
    if (flags & ~unsigned(MPFK_LEAN)) fail(MPFK_EINVAL, "mpfk: a K-panel continuation takes MPFK_LEAN only");
    if (lda < k || ldb < n || ldc < n) fail(MPFK_EINVAL, "mpfk: leading dimension too small");
    if ((lda | ldb | ldc | a_plane | b_plane | c_plane) & 1)
      fail(MPFK_EINVAL, "mpfk: device strides must be even (16-byte rows)");
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
         reinterpret_cast<uintptr_t>(C)) & 15)
      fail(MPFK_EINVAL, "mpfk: device operands must be 16-byte aligned");
    const int dev = current_device();
    ensure_devices(1, dev);
    const int l = enqueue_gemm(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane,
                               static_cast<cudaStream_t>(stream), true, (flags & MPFK_LEAN) != 0);
    if (k) {  // k more multiply-adds per element: k muls and k adds
      tally_muls(m * n * k);
      tally_adds(m * n * k);
    }
    if (launches) *launches = l;
  });
}

int mpfk_gemm_device_pull(int width, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                          uint64_t a_plane, double* B, uint64_t ldb, uint64_t b_plane, double* C, uint64_t ldc,
                          uint64_t c_plane, int nsrc, const double* const* src, const uint64_t* src_row0,
                          uint64_t panel_rows, uint64_t chunk_rows, void* stream, int* launches) {
  return guarded([&] {
    check_width(width);
    if (nsrc < 1 || nsrc > 8) fail(MPFK_EINVAL, "mpfk: 1..8 source slices");
    if (!src || !src_row0) fail(MPFK_EINVAL, "mpfk: null source table");
    if (src_row0[0] != 0 || src_row0[nsrc] != k) fail(MPFK_EINVAL, "mpfk: source slices must cover rows [0, k)");
    for (int s_ = 0; s_ < nsrc; ++s_)
      if (src_row0[s_ + 1] < src_row0[s_]) fail(MPFK_EINVAL, "mpfk: source slices out of order");
    if (panel_rows < 16 || panel_rows % 16 || chunk_rows < 1)
      fail(MPFK_EINVAL, "mpfk: panel_rows must be a positive multiple of 16 and chunk_rows >= 1");
    if (lda < k || ldb < n || ldc < n) fail(MPFK_EINVAL, "mpfk: leading dimension too small");
    if ((lda | ldb | ldc | a_plane | b_plane | c_plane) & 1)
      fail(MPFK_EINVAL, "mpfk: device strides must be even (16-byte rows)");
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
      fail(MPFK_EINVAL, "mpfk: device operands must be 16-byte aligned");
    for (int s_ = 0; s_ < nsrc; ++s_)
      if (reinterpret_cast<uintptr_t>(src[s_]) & 15) fail(MPFK_EINVAL, "mpfk: source slices must be 16-byte aligned");
    const int dev = current_device();
    ensure_devices(1, dev);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int l = 0;
    if (m && n && k) {
      if (m > 0x7fffffffULL || n > 0x7fffffffULL || k > 0x7fffffffULL)
        fail(MPFK_EINVAL, "mpfk: dimension exceeds 2^31-1");
      kern::PullB P{};
      P.panel_rows = (int)panel_rows;
      P.panels = (int)((k + panel_rows - 1) / panel_rows);
      P.chunk_rows = (int)std::min<uint64_t>(chunk_rows, panel_rows);
      P.chunks = (int)((panel_rows + P.chunk_rows - 1) / P.chunk_rows);
      P.nsrc = nsrc;
      for (int s_ = 0; s_ <= nsrc; ++s_) P.src_row0[s_] = (int)src_row0[s_];
      for (int s_ = 0; s_ < nsrc; ++s_) {
        P.src[s_] = src[s_];
        P.src_plane[s_] = (long long)((src_row0[s_ + 1] - src_row0[s_]) * ldb);
      }
      // the last panel may be short: its tail chunks copy nothing but still count
      int* ctr = nullptr;
      ck(cudaMallocAsync(reinterpret_cast<void**>(&ctr), sizeof(int) * 2 * P.panels, s), "cudaMallocAsync");
      ck(cudaMemsetAsync(ctr, 0, sizeof(int) * 2 * P.panels, s), "cudaMemsetAsync");
      P.next = ctr, P.done = ctr + P.panels;
      kern::GemmArgs g;
      g.A = A, g.B = B, g.C = C;
      g.lda = (long long)lda, g.ldb = (long long)ldb, g.ldc = (long long)ldc;
      g.pa = (long long)a_plane, g.pb = (long long)b_plane, g.pc = (long long)c_plane;
      g.M = (int)m, g.N = (int)n, g.K = (int)k;
      g.accumulate = 0;
      g.batch = 1, g.sa = g.sb = g.sc = 0;
      l = dispatch_gemm_pull(width, g, P, s);
      ck(cudaFreeAsync(ctr, s), "cudaFreeAsync");
    } else {
      l = enqueue_gemm(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane, s);
    }
    count_matmul(m, n, k);
    if (launches) *launches = l;
  });
}


// ---------------------------------------------------------------------------
// B row-sliced across devices (the all-gather -> GEMM entry points)
// ---------------------------------------------------------------------------
// Rows [row0[s], row0[s+1]) of B live in slice s, a W-plane (rows_s x ldb)
// array on this device, a peer device, or CUDA-IPC-mapped peer memory.
struct Slices {
  int n;
  const double* const* src;
  const uint64_t* row0;
  std::vector<char> local;  // slice is on this device (or of unknown placement)
  bool remote_on_copy_engines = true;  // every remote slice is on a P2P-capable peer

  Slices(int nsrc, const double* const* s, const uint64_t* r, uint64_t k, int max_src, int dev_id)
      : n(nsrc), src(s), row0(r), local(nsrc, 0) {
    if (nsrc < 1 || nsrc > max_src) fail(MPFK_EINVAL, "mpfk: 1.." + std::to_string(max_src) + " source slices");
    if (!s || !r) fail(MPFK_EINVAL, "mpfk: null source table");
    if (r[0] != 0 || r[nsrc] != k) fail(MPFK_EINVAL, "mpfk: source slices must cover rows [0, k)");
    for (int i = 0; i < nsrc; ++i)
      if (r[i + 1] < r[i]) fail(MPFK_EINVAL, "mpfk: source slices out of order");
    for (int i = 0; i < nsrc; ++i) {
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, s[i]) != cudaSuccess) {
        cudaGetLastError();
        local[i] = 1;  // unknown: the safe side
        continue;
      }
      local[i] = at.type != cudaMemoryTypeDevice || at.device == dev_id;
      if (!local[i]) {
        // a peer copy runs on the copy engines only over a P2P path; without
        // one the driver stages it, possibly with copy kernels that a GEMM
        // waiting inside the kernel for the data would starve
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, dev_id, at.device) != cudaSuccess) cudaGetLastError(), can = 0;
        if (!can) remote_on_copy_engines = false;
      }
    }
  }

  // rows [k0, k1) of B from the slices that hold them into B (whole rows of
  // ldb doubles per plane) on stream cs; which: 1 local slices, 0 remote, -1 all
  void copy(int W, double* B, uint64_t ldb, uint64_t b_plane, uint64_t k0, uint64_t k1, cudaStream_t cs,
            int which) const {
    for (int i = 0; i < n; ++i) {
      if (which >= 0 && local[i] != which) continue;
      const uint64_t a = std::max(k0, row0[i]), b = std::min(k1, row0[i + 1]);
      if (a >= b) continue;
      const uint64_t rows_s = row0[i + 1] - row0[i];
      for (int w = 0; w < W; ++w)
        ck(cudaMemcpyAsync(B + w * b_plane + a * ldb, src[i] + w * rows_s * ldb + (a - row0[i]) * ldb,
                           sizeof(double) * (b - a) * ldb, cudaMemcpyDefault, cs),
           "gather copy");
    }
  }
};

static void check_device_operands(uint64_t n, uint64_t k, const double* A, uint64_t lda, uint64_t a_plane,
                           const double* B, uint64_t ldb, uint64_t b_plane, const double* C, uint64_t ldc,
                           uint64_t c_plane) {
  if (lda < k || ldb < n || ldc < n) fail(MPFK_EINVAL, "mpfk: leading dimension too small");
  if ((lda | ldb | ldc | a_plane | b_plane | c_plane) & 1)
    fail(MPFK_EINVAL, "mpfk: device strides must be even (16-byte rows)");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
    fail(MPFK_EINVAL, "mpfk: device operands must be 16-byte aligned");
}

// K panel boundaries of the staged all-gather -> GEMM: a short first panel
// (its gather is the only exposed transfer), each next panel 4x the last,
// so every panel's compute covers the gather of the next; the last panel
// runs to k.  head_rows overrides the first panel's height.
static std::vector<uint64_t> staged_panels(uint64_t k, uint64_t head_rows) {
  std::vector<uint64_t> cut{0};
  uint64_t h = head_rows ? head_rows : 64;
  h = std::max<uint64_t>(16, (h + 15) / 16 * 16);
  while ((int)cut.size() < kStagedPanels && cut.back() + h < k && h * 2 <= k - cut.back()) {
    cut.push_back(cut.back() + h);
    h *= 4;
  }
  cut.push_back(k);
  return cut;
}

int mpfk_gemm_device_gathered(int width, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                              uint64_t a_plane, double* B, uint64_t ldb, uint64_t b_plane, double* C, uint64_t ldc,
                              uint64_t c_plane, int nsrc, const double* const* src, const uint64_t* src_row0,
                              uint64_t panel_rows, void* stream, int* launches) {
  return guarded([&] {
    check_width(width);
    if (panel_rows < 16 || panel_rows % 16) fail(MPFK_EINVAL, "mpfk: panel_rows must be a positive multiple of 16");
    check_device_operands(n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane);
    const int dev = current_device();
    ensure_devices(1, dev);
    Device& D = g_dev[dev];
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // panel p of B = rows [p*panel_rows, ...) gathered from the slices that
    // hold them.  A slice on this very device is copied in stream order
    // BEFORE the GEMM: device-local copies may run as copy kernels, which a
    // GEMM that fills every SM slot while it waits on panel flags would
    // starve.  Slices on other GPUs move over NVLink on the copy engines,
    // concurrently -- only when every such peer is P2P-reachable; otherwise
    // (S.remote_on_copy_engines false) the whole gather precedes a plain GEMM.
    const Slices S(nsrc, src, src_row0, k, 64, D.id);
    auto copy_panel = [&](uint64_t k0, uint64_t k1, cudaStream_t cs, int which) {
      S.copy(width, B, ldb, b_plane, k0, k1, cs, which);
    };
    int l = 0;
    if (!(m && n && k) || !memops_available() || !S.remote_on_copy_engines) {
      // no stream memory operations: gather everything, then the plain GEMM
      if (m && n)
        for (uint64_t k0 = 0; k0 < k; k0 += panel_rows) copy_panel(k0, std::min(k, k0 + panel_rows), s, -1);
      l = enqueue_gemm(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane, s);
    } else {
      if (m > 0x7fffffffULL || n > 0x7fffffffULL || k > 0x7fffffffULL)
        fail(MPFK_EINVAL, "mpfk: dimension exceeds 2^31-1");
      const uint64_t npan = (k + panel_rows - 1) / panel_rows, band_rows = 256, nb = (m + band_rows - 1) / band_rows;
      // one flag buffer per device: the previous gathered GEMM on this device
      // must be done with it (host wait; consecutive calls are whole GEMMs)
      std::lock_guard<std::mutex> lk(g_gather_mu[dev % 64]);
      ck(cudaEventSynchronize(D.evG[2]), "previous gathered GEMM");
      const size_t gbytes = sizeof(unsigned) * (npan + nb);
      if (gbytes > D.ggate_cap) {
        if (D.ggate) cudaFree(D.ggate);
        D.ggate = nullptr;
        D.ggate_cap = 0;
        ck(cudaMalloc(reinterpret_cast<void**>(&D.ggate), gbytes), "cudaMalloc(gather gate)");
        D.ggate_cap = gbytes;
      }
      unsigned* gate = D.ggate;
      ck(cudaMemsetAsync(gate, 0, gbytes, s), "cudaMemsetAsync");
      copy_panel(0, k, s, 1);  // this device's own rows, before the launch
      ck(cudaEventRecord(D.evG[0], s), "event");
      // the copy engines gather B panel by panel on the device's gather
      // stream, flagging each panel; the GEMM on the caller's stream waits
      // per panel inside the kernel (kern::GateArgs)
      ck(cudaStreamWaitEvent(D.gather, D.evG[0], 0), "wait gate reset");
      for (uint64_t p = 0; p < npan; ++p) {
        copy_panel(p * panel_rows, std::min(k, (p + 1) * panel_rows), D.gather, 0);
        cu_ck(g_write32(reinterpret_cast<CUstream>(D.gather), reinterpret_cast<CUdeviceptr>(gate + p), 1, 0),
              "cuStreamWriteValue32");
      }
      ck(cudaEventRecord(D.evG[1], D.gather), "event");
      kern::GemmArgs g;
      g.A = A, g.B = B, g.C = C;
      g.lda = (long long)lda, g.ldb = (long long)ldb, g.ldc = (long long)ldc;
      g.pa = (long long)a_plane, g.pb = (long long)b_plane, g.pc = (long long)c_plane;
      g.M = (int)m, g.N = (int)n, g.K = (int)k;
      g.accumulate = 0;
      g.batch = 1, g.sa = g.sb = g.sc = 0;
      // A is resident: every row counts as uploaded with the first panel
      kern::GateArgs gate_args{gate, gate + npan, (int)panel_rows, (int)band_rows, (int)m, nullptr};
      dispatch_gemm_gated(width, g, gate_args, s);
      l = 1;
      ck(cudaStreamWaitEvent(s, D.evG[1], 0), "join gather");  // B complete when the stream is
      ck(cudaEventRecord(D.evG[2], s), "event");
    }
    count_matmul(m, n, k);
    if (launches) *launches = l;
  });
}


int mpfk_gemm_device_staged(int width, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                            uint64_t a_plane, double* B, uint64_t ldb, uint64_t b_plane, double* C, uint64_t ldc,
                            uint64_t c_plane, int nsrc, const double* const* src, const uint64_t* src_row0,
                            uint64_t head_rows, void* stream, int* launches) {
  return mpfk_gemm_device_staged_ex(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane, nsrc, src,
                                    src_row0, head_rows, MPFK_BIT_EXACT, stream, launches);
}

int mpfk_gemm_device_staged_ex(int width, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda,
                               uint64_t a_plane, double* B, uint64_t ldb, uint64_t b_plane, double* C,
                               uint64_t ldc, uint64_t c_plane, int nsrc, const double* const* src,
                               const uint64_t* src_row0, uint64_t head_rows, unsigned flags, void* stream,
                               int* launches) {
  return guarded([&] {
    check_width(width);
    if (flags & ~unsigned(MPFK_LEAN)) fail(MPFK_EINVAL, "mpfk: the staged all-gather GEMM takes MPFK_LEAN only");
    const bool lean = (flags & MPFK_LEAN) != 0;
    check_device_operands(n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane);
    const int dev = current_device();
    ensure_devices(1, dev);
    Device& D = g_dev[dev];
    const Slices S(nsrc, src, src_row0, k, 64, D.id);
    for (int i = 0; i < nsrc; ++i)
      if (reinterpret_cast<uintptr_t>(src[i]) & 15) fail(MPFK_EINVAL, "mpfk: source slices must be 16-byte aligned");
    if (head_rows % 16) fail(MPFK_EINVAL, "mpfk: head_rows must be a multiple of 16 (0: automatic)");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int l = 0;
    if (!(m && n && k)) {
      if (n && k) S.copy(width, B, ldb, b_plane, 0, k, s, -1);
      l = enqueue_gemm(width, m, n, k, A, lda, a_plane, B, ldb, b_plane, C, ldc, c_plane, s, false, lean);
    } else {
      // the gather runs on the device's gather stream -- peer slices on the
      // copy engines over NVLink -- in ascending K panels, one event per
      // panel; panel p's GEMM launch (p > 0 continues the chains kept in C)
      // waits for that event only.  No kernel ever waits on a flag, so the
      // schedule cannot stall whatever engine the driver picks for a copy.
      const std::vector<uint64_t> cut = staged_panels(k, head_rows);
      const int np = (int)cut.size() - 1;
      std::lock_guard<std::mutex> lk(g_gather_mu[dev % 64]);
      ck(cudaEventRecord(D.evS[0], s), "event");  // B's buffer is free in stream order
      ck(cudaStreamWaitEvent(D.gather, D.evS[0], 0), "wait stream");
      for (int p = 0; p < np; ++p) {
        S.copy(width, B, ldb, b_plane, cut[p], cut[p + 1], D.gather, -1);
        ck(cudaEventRecord(D.evS[p + 1], D.gather), "event");
      }
      for (int p = 0; p < np; ++p) {
        ck(cudaStreamWaitEvent(s, D.evS[p + 1], 0), "wait panel");
        l += enqueue_gemm(width, m, n, cut[p + 1] - cut[p], A + cut[p], lda, a_plane, B + cut[p] * ldb, ldb,
                          b_plane, C, ldc, c_plane, s, p > 0, lean);
      }
    }
    count_matmul(m, n, k);
    if (launches) *launches = l;
  });
}

int mpfk_device_alloc(uint64_t bytes, void** ptr) {
  return guarded([&] {
    if (!ptr) fail(MPFK_EINVAL, "mpfk: null output pointer");
    const int dev = current_device();
    ensure_devices(1, dev);
    *ptr = nullptr;
    ck(cudaMalloc(ptr, std::max<uint64_t>(bytes, 1)), "cudaMalloc");
  });
}

int mpfk_device_free(void* ptr) {
  return guarded([&] {
    if (ptr) ck(cudaFree(ptr), "cudaFree");
  });
}

int mpfk_memcpy(void* dst, const void* src, uint64_t bytes) {
  return guarded([&] {
    if (bytes) ck(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault), "cudaMemcpy");
  });
}

int mpfk_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  return guarded([&] {
    if (!handle_out) fail(MPFK_EINVAL, "mpfk: null handle buffer");
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)), "cudaIpcGetMemHandle");
    std::memcpy(handle_out, &h, sizeof h);
  });
}

int mpfk_ipc_open(const void* handle, void** dev_ptr) {
  return guarded([&] {
    if (!handle || !dev_ptr) fail(MPFK_EINVAL, "mpfk: null handle or output pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    *dev_ptr = nullptr;
    ck(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}

int mpfk_ipc_close(void* dev_ptr) {
  return guarded([&] {
    if (dev_ptr) ck(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
  });
}

int mpfk_eft_batch(int op, uint64_t count, const double* a, const double* b, double* s, double* e) {
  return guarded([&] {
    if (op < 0 || op > 2) fail(MPFK_EINVAL, "mpfk: eft op must be 0 (two_sum), 1 (quick_two_sum) or 2 (two_prod)");
    if (count == 0) return;
    const int dev = current_device();
    ensure_devices(1, dev);
    const size_t bytes = sizeof(double) * count;
    double* d = nullptr;
    ck(cudaMalloc(&d, 4 * bytes), "cudaMalloc");
    ck(cudaMemcpy(d, a, bytes, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(d + count, b, bytes, cudaMemcpyHostToDevice), "H2D");
    const int blocks = (int)std::min<uint64_t>((count + 255) / 256, 148 * 16);
    eft_kernel<<<blocks, 256>>>(op, (long long)count, d, d + count, d + 2 * count, d + 3 * count);
    ck(cudaGetLastError(), "eft launch");
    ck(cudaMemcpy(s, d + 2 * count, bytes, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(e, d + 3 * count, bytes, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(d);
  });
}

int mpfk_binop_batch(int width, int op, uint64_t count, const double* x, const double* y,
                     double* r) {
  return guarded([&] {
    check_width(width);
    if (op < 0 || op > 3 || (op >= 2 && width != 3))
      fail(MPFK_EINVAL, "mpfk: op must be 0 (add), 1 (mul), or for width 3 2 (td_mul_q) / 3 (td_add_merge)");
    if (count == 0) return;
    const int dev = current_device();
    ensure_devices(1, dev);
    const size_t bytes = sizeof(double) * width * count;
    double *dx = nullptr, *dy = nullptr, *dr = nullptr;
    ck(cudaMalloc(&dx, bytes), "cudaMalloc");
    ck(cudaMalloc(&dy, bytes), "cudaMalloc");
    ck(cudaMalloc(&dr, bytes), "cudaMalloc");
    ck(cudaMemcpy(dx, x, bytes, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(dy, y, bytes, cudaMemcpyHostToDevice), "H2D");
    const int blocks = (int)std::min<uint64_t>((count + 255) / 256, 148 * 16);
    switch (width) {
      case 2: binop_kernel<2><<<blocks, 256>>>(op, (long long)count, dx, dy, dr); break;
      case 3: binop_kernel<3><<<blocks, 256>>>(op, (long long)count, dx, dy, dr); break;
      case 4: binop_kernel<4><<<blocks, 256>>>(op, (long long)count, dx, dy, dr); break;
    }
    ck(cudaGetLastError(), "binop launch");
    ck(cudaMemcpy(r, dr, bytes, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dr);
  });
}

int mpfk_mpfm_info(const char* path, int* width, uint64_t* rows, uint64_t* cols) {
  return guarded([&] {
    const std::string p = path ? path : "";
    File F;
    F.f = std::fopen(p.c_str(), "rb");
    if (!F.f) io_fail(p, "cannot open");
    const MpfmHeader h = read_header(F.f, p, 0);
    if (width) *width = h.width;
    if (rows) *rows = h.rows;
    if (cols) *cols = h.cols;
  });
}

int mpfk_mpfm_load_device(const char* path, int width, double* dev, uint64_t ld, uint64_t plane,
                          void* stream) {
  return guarded([&] {
    check_width(width);
    const int d = current_device();
    ensure_devices(1, d);
    mpfm_load(path, width, dev, ld, plane, true, static_cast<cudaStream_t>(stream));
  });
}

int mpfk_mpfm_save_device(const char* path, int width, const double* dev, uint64_t rows, uint64_t cols,
                          uint64_t ld, uint64_t plane, void* stream) {
  return guarded([&] {
    check_width(width);
    const int d = current_device();
    ensure_devices(1, d);
    mpfm_save(path, width, dev, rows, cols, ld, plane, true, static_cast<cudaStream_t>(stream));
  });
}

int mpfk_mpfm_load_host(const char* path, int width, mpfk_mat* m) {
  return guarded([&] {
    check_width(width);
    check_mat(m, "m");
    const std::string p = path ? path : "";
    {
      File F;
      F.f = std::fopen(p.c_str(), "rb");
      if (!F.f) io_fail(p, "cannot open");
      const MpfmHeader h = read_header(F.f, p, width);
      if (h.rows != m->rows || h.cols != m->cols) fail(MPFK_EINVAL, "mpfk: matrix shape differs from the file");
    }
    zero_host_pads(width, m);
    mpfm_load(path, width, m->base, m->stride, plane_of(m), false, nullptr);
  });
}

int mpfk_mpfm_save_host(const char* path, int width, const mpfk_mat* m) {
  return guarded([&] {
    check_width(width);
    check_mat(m, "m");
    mpfm_save(path, width, m->base, m->rows, m->cols, m->stride, plane_of(m), false, nullptr);
  });
}

void mpfk_op_counters_reset(void) {
  g_adds.store(0, std::memory_order_relaxed);
  g_muls.store(0, std::memory_order_relaxed);
  g_leaf.store(0, std::memory_order_relaxed);
}

void mpfk_op_counters_read(uint64_t* adds, uint64_t* muls, uint64_t* leaf) {
  if (adds) *adds = g_adds.load(std::memory_order_relaxed);
  if (muls) *muls = g_muls.load(std::memory_order_relaxed);
  if (leaf) *leaf = g_leaf.load(std::memory_order_relaxed);
}

void mpfk_last_op_counts(uint64_t* adds, uint64_t* muls, uint64_t* leaf) {
  if (adds) *adds = t_ops[0];
  if (muls) *muls = t_ops[1];
  if (leaf) *leaf = t_ops[2];
}

int mpfk_gemm_redo_count(uint64_t* count, int reset) {
  return guarded([&] {
    const int dev = current_device();
    ensure_devices(1, dev);
    unsigned long long v = 0;
    ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    ck(cudaMemcpyFromSymbol(&v, kern::g_fastr_redo, sizeof v), "cudaMemcpyFromSymbol");
    if (count) *count = v;
    if (reset) {
      v = 0;
      ck(cudaMemcpyToSymbol(kern::g_fastr_redo, &v, sizeof v), "cudaMemcpyToSymbol");
    }
  });
}

void* mpfk_host_alloc(uint64_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 1;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    t_err = "mpfk: cudaMallocHost failed";
    return nullptr;
  }
  return p;
}

void mpfk_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int mpfk_host_register_cache(uint64_t bytes) {
  return guarded([&] { host_reg_cache().set_capacity(bytes); });
}

int mpfk_host_register_cache_stats(uint64_t* capacity, uint64_t* used, uint64_t* entries) {
  return guarded([&] {
    if (capacity) *capacity = host_reg_cache().capacity();
    if (used) *used = host_reg_cache().used();
    if (entries) *entries = host_reg_cache().entries();
  });
}

int mpfk_host_unregister(const void* base) {
  return guarded([&] { host_reg_cache().unregister(base); });
}

int mpfk_fill_baseline(int width, int wide, uint64_t row0, uint64_t rows, uint64_t cols,
                       uint64_t stride, uint64_t seed, double* planes, int threads) {
  return guarded([&] {
    check_width(width);
    if (stride < cols) fail(MPFK_EINVAL, "mpfk: stride < cols");
    if (rows && cols && !planes) fail(MPFK_EINVAL, "mpfk: null planes");
    unsigned T = threads > 0 ? (unsigned)threads : std::max(1u, std::thread::hardware_concurrency());
    T = (unsigned)std::min<uint64_t>(T, std::max<uint64_t>(rows, 1));
    const uint64_t ps = rows * stride;
    auto body = [&](unsigned t) {
      for (uint64_t i = t; i < rows; i += T) {
        SM64 g{seed ^ ((row0 + i + 1) * 0xd1b54a32d192ed03ULL)};
        for (uint64_t j = 0; j < cols; ++j) {
          double v[4];
          baseline_elem(width, wide, g, v);
          for (int w = 0; w < width; ++w) planes[w * ps + i * stride + j] = v[w];
        }
        for (int w = 0; w < width; ++w)
          for (uint64_t j = cols; j < stride; ++j) planes[w * ps + i * stride + j] = 0.0;
      }
    };
    if (T <= 1) {
      body(0);
      return;
    }
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t) th.emplace_back(body, t);
    for (auto& x : th) x.join();
  });
}

int mpfk_fill_random(int width, uint64_t rows, uint64_t cols, uint64_t stride, uint64_t seed,
                     double* planes) {
  return guarded([&] {
    check_width(width);
    if (stride < cols) fail(MPFK_EINVAL, "mpfk: stride < cols");
    if (rows && cols && !planes) fail(MPFK_EINVAL, "mpfk: null planes");
    SM64 g{seed};
    const uint64_t ps = rows * stride;
    std::memset(planes, 0, sizeof(double) * width * ps);
    for (uint64_t i = 0; i < rows; ++i)
      for (uint64_t j = 0; j < cols; ++j) {
        double v[4];
        random_normalized(width, g, v);
        for (int w = 0; w < width; ++w) planes[w * ps + i * stride + j] = v[w];
      }
  });
}

int mpfk_gen_paper(int width, uint64_t n, uint64_t stride, double* A, double* B) {
  return guarded([&] {
    check_width(width);
    if (n < 1) fail(MPFK_EINVAL, "gen_paper_matrices: n must be at least 1");
    if (stride < n) fail(MPFK_EINVAL, "mpfk: stride < cols");
    const uint64_t ps = n * stride;
    std::memset(A, 0, sizeof(double) * width * ps);
    std::memset(B, 0, sizeof(double) * width * ps);
    double r5[4] = {std::sqrt(5.0), 0, 0, 0}, r3[4] = {std::sqrt(3.0), 0, 0, 0};
    auto mul = [&](const double* x, const double* y, double* r) {
      if (width == 2) arith::mp_mul<2>(x, y, r);
      else if (width == 3) arith::mp_mul<3>(x, y, r);
      else arith::mp_mul<4>(x, y, r);
    };
    for (uint64_t i = 1; i <= n; ++i) {
      double f[4] = {static_cast<double>(n - i), 0, 0, 0}, brow[4];
      mul(r3, f, brow);
      for (uint64_t j = 1; j <= n; ++j) {
        double gv[4] = {static_cast<double>(i + j - 1), 0, 0, 0}, a[4];
        mul(r5, gv, a);
        for (int w = 0; w < width; ++w) {
          A[w * ps + (i - 1) * stride + (j - 1)] = a[w];
          B[w * ps + (i - 1) * stride + (j - 1)] = brow[w];
        }
      }
    }
  });
}

int mpfk_fp64_peak(double* ops_per_s, double* ms_out) {
  return guarded([&] {
    const int dev = current_device();
    ensure_devices(1, dev);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* d = nullptr;
    ck(cudaMalloc(&d, 8), "cudaMalloc");
    // ~5 ms per launch so the launch ramp and tail are < 0.5 % of it
    const int blocks = sms * 8, threads = 256, iters = 1 << 15;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    fp64_peak_kernel<<<blocks, threads>>>(d, iters, 0.999999);  // warm-up
    ck(cudaGetLastError(), "fp64 peak launch");
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      fp64_peak_kernel<<<blocks, threads>>>(d, iters, 0.999999);
      cudaEventRecord(b);
      ck(cudaEventSynchronize(b), "fp64 peak");
      float t = 0;
      cudaEventElapsedTime(&t, a, b);
      best = std::min(best, t);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    const double ops = double(blocks) * threads * iters * 8.0;
    if (ops_per_s) *ops_per_s = ops / (best * 1e-3);
    if (ms_out) *ms_out = best;
  });
}

}  // extern "C"
