// gemm_kernel.cuh -- register-blocked, shared-memory-tiled DD/TD/QD GEMM for
// sm_100a on the FP64 CUDA-core pipe.
//
// Replaces the reference's hot loop: matmul_block*_into -> mul_panel ->
// QuadRow::axpy -> mpf::mul/add<W> (linalg.hpp:250-277, 368-433).
//
// Per-element contract (linalg.hpp:235-248, 338-344): C(i,j) = mul(A(i,0),
// B(0,j)); then C(i,j) = add(C(i,j), mul(A(i,k), B(k,j))) for k = 1..K-1 in
// ascending order.  Each thread owns a TM x TN register micro-tile of all W
// components and walks k in exactly that order, so every C element is
// bit-identical to the reference for any tiling, grid or GPU count.  K is
// never padded (an extra add(C, mul(0, b)) is not a bitwise identity on
// signed zeros), the k loop is bounded by the true K.
//
// Data movement: A and B tiles of all W component planes (the reference's
// SoA layout, linalg.hpp:36-129) are staged into shared memory with 16-byte
// cp.async (LDGSTS) in a STAGES-deep ring; operand traffic is tiny next to
// the 20-218 FP64 operations per multiply-add, so the kernel is bound by the
// FP64 pipe, not by HBM, L2 or shared memory.
//
// One tile body (tile_run, called by gemm_body for one tile per CTA), four
// entry points: mpgemm_kernel (plain), mpgemm_splitk_kernel (MPFK_FAST
// segments), mpgemm_pull_kernel (fused all-gather, PullB) and
// mpgemm_gated_kernel (K panels flagged by the copy engines, GateArgs).  The pull/gate bookkeeping is out of line so every
// variant's main loop is the same instruction stream.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "mpf_arith.cuh"
#include "mpf_lean.cuh"

namespace mpfk {
namespace kern {

struct GemmArgs {
  const double* A;  // W planes, plane stride pa, row stride lda (elements)
  const double* B;
  double* C;
  long long lda, ldb, ldc;
  long long pa, pb, pc;
  int M, N, K;
  // 0: C = A*B (k = 0 initialises, linalg.hpp:242).  1: continue the chains
  // stored in C over this K panel: every k is an add(C, mul(a, b)).  The
  // reference itself carries the chain state in C between k steps
  // (QuadRow::axpy reloads C, linalg.hpp:261), so splitting K into panels
  // and continuing from C is bit-identical.
  int accumulate;
  // Strided batch of independent products (the Strassen leaves, all of one
  // shape): matrix b of A/B/C starts sa/sb/sc doubles after matrix b-1.
  int batch;
  long long sa, sb, sc;
};

// Fused all-gather -> GEMM (mpgemm_pull_kernel, gemm_body mode 1): B is not resident
// yet; its rows live in up to 8 source slices (other ranks' memory reached
// over NVLink peer mappings, or local buffers when emulated on one GPU).
// Before a CTA stages the k-tile of panel p it makes sure panel p has been
// copied into the local B: chunks of the panel are handed out by an atomic
// counter, the CTA copies every chunk it wins (16-byte loads from the
// owning slice, stores into local B), publishes each with a release fence +
// done-counter, then waits for the panel's other chunks -- which are being
// copied by CTAs that are running (they took them), so nothing waits on a
// CTA that is not resident.  Each panel crosses NVLink once per GPU, while
// the rest of the grid computes on the panels already present.
struct PullB {
  int panels, panel_rows;  // K rows per panel (a multiple of BK)
  int chunk_rows, chunks;  // chunks per panel
  int nsrc;                // source slices
  int src_row0[9];         // slice s holds B rows [src_row0[s], src_row0[s+1])
  const double* src[8];    // slice s: W planes of (rows_s x ldb), plane stride src_plane[s]
  long long src_plane[8];
  int* next;               // [panels] chunk tickets handed out
  int* done;               // [panels] chunks copied and published
};

// warp k-tiles recomputed with the exact renormalisation (TileCfg::FASTR);
// read through mpfk_gemm_redo_count
__device__ unsigned long long g_fastr_redo = 0;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;  // src-size 0 -> 16 zero bytes, no global read
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
// 16 bytes, always valid (interior tiles): no src-size operand
__device__ __forceinline__ void cp_async16_full(unsigned smem_addr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr), "l"(gmem));
}

// GROUP_M: tiles are visited in column-major order within bands of GROUP_M
// tile rows, so the CTAs resident at one time cover a near-square block of C
// and share their A and B panels in L2 instead of streaming all of B per
// tile row.
template <int W_, int BM_, int BN_, int BK_, int TM_, int TN_, int STAGES_ = 2, int KUNROLL_ = 1,
          int GROUP_M_ = 16, int MINB_ = 1, int FIXK_ = 0, int ONEBAR_ = 0, int FASTR_ = 0, int VSEBF_ = 0,
          int FLOAD_ = 1, int PAIRB_ = 1, int RAREMIN_ = 0, int LEAN_ = 0, int ROWMAJ_ = 0>
struct TileCfg {
  // bit-exact DD: a micro-tile row's multiply-adds written stage by stage
  // (arith::dd_mac_row: the same operations in another order)
  static constexpr int ROWMAJ = (W_ == 2 && !LEAN_) ? ROWMAJ_ : 0;
  // MPFK_LEAN (mpf_lean.cuh): the tolerance-mode multiply-accumulate --
  // every element is W levels fed by exact two-sum cascades, pulled back to
  // nearly non-overlapping once per k-tile and normalised once at the end.
  // 10 / 42 / 107 FP64 instructions per step; NOT bit-identical to the
  // reference (within the north star's 4*k*u_p).  No data-dependent path, so
  // no FASTR machinery.
  static constexpr int LEAN = LEAN_;
  static constexpr int W = W_, BM = BM_, BN = BN_, BK = BK_, TM = TM_, TN = TN_;
  static constexpr int STAGES = STAGES_, KUNROLL = KUNROLL_, GROUP_M = GROUP_M_, MINB = MINB_;
  static constexpr int FIXK = FIXK_;  // full k-tiles run a constant-trip loop
  // one __syncthreads per k-tile: wait for tile kt, barrier, THEN refill the
  // slot of tile kt-1 (every warp is past it) and compute -- instead of
  // refill, wait, barrier, compute, barrier
  static constexpr int ONEBAR = ONEBAR_;
  // interior tiles load full k-tiles with the precomputed-address loader
  // (FastLoad); 0 keeps the general loader everywhere
  static constexpr int FLOAD = FLOAD_;
  // a thread's micro-tile columns in adjacent pairs (2 tx, 2 tx + 1, then
  // + 2 TX ...) instead of stride TX, so each k step reads its B values with
  // half as many (16-byte) shared loads; same bytes, same bank wavefronts
  static constexpr int PAIRB = (PAIRB_ && TN_ % 2 == 0) ? 1 : 0;
  static constexpr int TX = BN / TN;  // threads along N
  static constexpr int TY = BM / TM;  // threads along M
  static constexpr int THREADS = TX * TY;
  // TD/QD: run each k-tile with the branch-free renorm5 (paths A/B) and a
  // per-thread "rare" flag; a warp that saw any input needing paths C/D
  // restores its chains from a shared-memory snapshot taken at the k-tile
  // start and recomputes the k-tile with the exact form (same smem stage,
  // same order): bit-identical, and the common path has no branch
  static constexpr int FASTR = (W_ >= 3 && !LEAN_) ? FASTR_ : 0;  // renorm5_t level (1: paths A/B, 2: path A)
  static constexpr bool VSEBF = FASTR && VSEBF_;          // td_mul's vseb common case in the fast pass
  // the fast pass's "left the fast form" accumulator: exact LOP3/PLOP3
  // predicates (arith::RareBool, the product) or a running FMNMX3 minimum
  // (arith::RareMin, measured before the ordered two-sums: 14 of TD's 48 and 83 of QD's 205 non-FP64 instructions
  // per loop body fewer, yet 0.3-0.7 % SLOWER on the B200,
  // profiles/r02/tune_raremin.log -- kept as a measured alternative)
  // (RAREMIN_ = 2: arith::RareHi, every test one binary32 compare of the high words)
  using Rare = typename std::conditional<
      RAREMIN_ == 1, arith::RareMin,
      typename std::conditional<RAREMIN_ == 2, arith::RareHi, arith::RareBool>::type>::type;
  static constexpr int SNAP = FASTR ? THREADS * TM * TN * W : 0;  // doubles
  static_assert(!FASTR || THREADS % 32 == 0, "the warp-level redo votes over full warps");
  static constexpr int APAD = 2, BPAD = 2;  // keep 16 B row alignment, spread banks
  static constexpr int AS = BK + APAD;      // A tile row stride (doubles), [BM][AS]
  static constexpr int BS = BN + BPAD;      // B tile row stride, [BK][BS]
  static constexpr int A_STAGE = W * BM * AS;
  static constexpr int B_STAGE = W * BK * BS;
  static constexpr size_t SMEM = sizeof(double) * (size_t(STAGES) * (A_STAGE + B_STAGE) + SNAP);
  static_assert(BK % 2 == 0 && BN % 2 == 0, "16-byte chunks");
  static_assert(BM % TM == 0 && BN % TN == 0, "micro-tile");
};

template <class Cfg>
__device__ __forceinline__ void load_tile(double* As, double* Bs, const GemmArgs& g, int m0,
                                          int n0, int k0) {
  constexpr int W = Cfg::W, BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  const int tid = threadIdx.x;
  // A: BM rows x BK/2 chunks per plane
  constexpr int ACH = BM * (BK / 2);
#pragma unroll
  for (int c = tid; c < W * ACH; c += Cfg::THREADS) {
    const int w = c / ACH, r = (c % ACH) / (BK / 2), kc = (c % ACH) % (BK / 2);
    const int gm = m0 + r, gk = k0 + 2 * kc;
    const bool ok = gm < g.M && gk < g.K;
    const double* src = ok ? g.A + w * g.pa + (long long)gm * g.lda + gk : g.A;
    cp_async16(As + w * BM * Cfg::AS + r * Cfg::AS + 2 * kc, src, ok);
  }
  constexpr int BCH = BK * (BN / 2);
#pragma unroll
  for (int c = tid; c < W * BCH; c += Cfg::THREADS) {
    const int w = c / BCH, r = (c % BCH) / (BN / 2), nc = (c % BCH) % (BN / 2);
    const int gk = k0 + r, gn = n0 + 2 * nc;
    const bool ok = gk < g.K && gn < g.N;
    const double* src = ok ? g.B + w * g.pb + (long long)gk * g.ldb + gn : g.B;
    cp_async16(Bs + w * BK * Cfg::BS + r * Cfg::BS + 2 * nc, src, ok);
  }
}

// Interior-tile loader.  load_tile above is general (any edge, any k0) but
// recomputes every chunk's (plane, row, column), bounds test and 64-bit
// address per k-tile: ~30 instructions per 16-byte copy, ~5 % of a DD
// thread's instruction stream next to its 5,120 FP64 instructions per
// k-tile (profiles/r02: the non-FP64 share is what costs FP64 issue slots).
// For a tile wholly inside M x N and a full k-tile, chunk `it` of a thread
// sits at a fixed offset from the thread's first chunk -- whole planes and
// whole row groups, since THREADS divides the chunks of a plane and is a
// multiple of the chunks of a row -- so the copies reduce to one pointer
// plus uniform offsets each, the pointers stepping by BK per k-tile.
template <class Cfg>
struct FastLoad {
  static constexpr int T = Cfg::THREADS, BK = Cfg::BK, BM = Cfg::BM, BN = Cfg::BN;
  static constexpr int ACH = BM * (BK / 2), BCH = BK * (BN / 2);
  static constexpr bool ok =
      Cfg::FLOAD && T % (BK / 2) == 0 && ACH % T == 0 && T % (BN / 2) == 0 && BCH % T == 0;
  static constexpr int A_IT = ok ? ACH / T : 1;      // copies per plane of A
  static constexpr int A_ROWS = ok ? T / (BK / 2) : 1;  // rows of A per copy round
  static constexpr int B_IT = ok ? BCH / T : 1;
  static constexpr int B_ROWS = ok ? T / (BN / 2) : 1;
};

struct FastLoadState {
  // this thread's first A / B chunk at the current k-tile, in elements from
  // the plane base (32-bit: the fast loader runs only when a plane's
  // offsets fit, fast_load_fits), and their shared-memory byte offsets
  // within a stage -- four registers, so a 128-register kernel keeps them
  unsigned a, b;
  unsigned sa, sb;
};

__device__ __forceinline__ bool fast_load_fits(const GemmArgs& g) {
  return (long long)g.M * g.lda < 0x7fffffffLL && ((long long)g.K + 64) * g.ldb < 0x7fffffffLL;
}

template <class Cfg>
__device__ __forceinline__ FastLoadState fast_load_init(const GemmArgs& g, int m0, int n0, int k0) {
  const int tid = threadIdx.x;
  const int ra = tid / (Cfg::BK / 2), ka = 2 * (tid % (Cfg::BK / 2));
  const int rb = tid / (Cfg::BN / 2), nb = 2 * (tid % (Cfg::BN / 2));
  FastLoadState st;
  st.a = (unsigned)((m0 + ra) * (long long)g.lda + k0 + ka);
  st.b = (unsigned)((k0 + rb) * (long long)g.ldb + n0 + nb);
  st.sa = 8u * (ra * Cfg::AS + ka);
  st.sb = 8u * (rb * Cfg::BS + nb);
  return st;
}

// the k-tile the state points at into stage (As, Bs); then advance one k-tile
template <class Cfg>
__device__ __forceinline__ void fast_load_tile(FastLoadState& st, double* As, double* Bs, const GemmArgs& g) {
  using F = FastLoad<Cfg>;
  constexpr int W = Cfg::W;
  const unsigned as = static_cast<unsigned>(__cvta_generic_to_shared(As)) + st.sa;
  const unsigned bs = static_cast<unsigned>(__cvta_generic_to_shared(Bs)) + st.sb;
#pragma unroll
  for (int w = 0; w < W; ++w)
#pragma unroll
    for (int it = 0; it < F::A_IT; ++it)
      cp_async16_full(as + 8u * (w * Cfg::BM * Cfg::AS + it * F::A_ROWS * Cfg::AS),
                      g.A + w * g.pa + (long long)(it * F::A_ROWS) * g.lda + st.a);
#pragma unroll
  for (int w = 0; w < W; ++w)
#pragma unroll
    for (int it = 0; it < F::B_IT; ++it)
      cp_async16_full(bs + 8u * (w * Cfg::BK * Cfg::BS + it * F::B_ROWS * Cfg::BS),
                      g.B + w * g.pb + (long long)(it * F::B_ROWS) * g.ldb + st.b);
  st.a += Cfg::BK;
  st.b += (unsigned)(Cfg::BK * g.ldb);
}

// linear CTA index -> (tile row, tile col) with GROUP_M-row bands
template <int GROUP_M>
__device__ __forceinline__ void tile_coords(int lin, int tiles_m, int tiles_n, int& tm, int& tn) {
  if (GROUP_M <= 1) {
    tm = lin / tiles_n;
    tn = lin % tiles_n;
    return;
  }
  const int band = lin / (GROUP_M * tiles_n);
  const int first = band * GROUP_M;
  const int rows = min(GROUP_M, tiles_m - first);
  const int local = lin - band * GROUP_M * tiles_n;
  tm = first + local % rows;
  tn = local / rows;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Copy chunk c of panel p from its source slices into the local B.
template <int W>
__device__ __forceinline__ void pull_chunk(const PullB& P, const GemmArgs& g, int p, int c) {
  const int r0 = p * P.panel_rows + c * P.chunk_rows;
  const int r1 = min(min(r0 + P.chunk_rows, (p + 1) * P.panel_rows), g.K);
  if (r1 <= r0) return;
  const int vpr = (int)(g.ldb / 2);  // 16-byte vectors per row (ld is even)
  const long long per_plane = (long long)(r1 - r0) * vpr, total = per_plane * W;
  double* B = const_cast<double*>(g.B);
  for (long long t = threadIdx.x; t < total; t += blockDim.x) {
    const int w = (int)(t / per_plane);
    const long long rem = t - w * per_plane;
    const int row = r0 + (int)(rem / vpr), v = (int)(rem % vpr);
    int s = 0;
    while (s + 1 < P.nsrc && row >= P.src_row0[s + 1]) ++s;
    const double2* src = reinterpret_cast<const double2*>(P.src[s] + w * P.src_plane[s] +
                                                          (long long)(row - P.src_row0[s]) * g.ldb) + v;
    double2* dst = reinterpret_cast<double2*>(B + w * g.pb + (long long)row * g.ldb) + v;
    *dst = *src;
  }
}

// Copy (without waiting) any still-unclaimed chunks of panel p: the
// lookahead that lets CTAs entering panel p-1 stage panel p in advance.
// (help_panel and ensure_panel are out of line: run once per panel, they
// keep their registers out of the GEMM main loop, which then compiles to the
// same instruction stream as the plain kernel's.)
template <int W>
__device__ __noinline__ void help_panel(const PullB& P, const GemmArgs& g, int p) {
  __shared__ int s_ticket;
  if (p >= P.panels) return;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0)
      s_ticket = ld_acquire_gpu(&P.next[p]) >= P.chunks ? P.chunks : atomicAdd(&P.next[p], 1);
    __syncthreads();
    const int c = s_ticket;
    if (c >= P.chunks) break;
    pull_chunk<W>(P, g, p, c);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&P.done[p], 1);
    }
  }
}

// Make panel p of B resident (block-wide; see PullB).
template <int W>
__device__ __noinline__ void ensure_panel(const PullB& P, const GemmArgs& g, int p) {
  __shared__ int s_state;
  if (threadIdx.x == 0) s_state = ld_acquire_gpu(&P.done[p]) >= P.chunks;
  __syncthreads();
  if (s_state) return;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_state = atomicAdd(&P.next[p], 1);
    __syncthreads();
    const int c = s_state;
    if (c >= P.chunks) break;
    pull_chunk<W>(P, g, p, c);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();  // release: the chunk's stores before the count
      atomicAdd(&P.done[p], 1);
    }
  }
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    while (ld_acquire_gpu(&P.done[p]) < P.chunks) {
      __nanosleep(200);
      if (clock64() - t0 > (1ll << 36)) __trap();  // ~30 s: a lost chunk, fail loudly
    }
  }
  __syncthreads();
}

// Copy-engine-gated GEMM (host operands streamed in K panels, see
// capi.cu:host_gemm_gated): panel p of A and B is resident once flags[p] is
// nonzero -- written by the copy stream with a stream memory operation after
// the panel's copies, so no SM time goes into the transfer -- and each
// finished tile adds 1 to band_done[m0 / band_rows], which the download
// stream waits on (stream wait-value) before copying that row band of C.
struct GateArgs {
  const unsigned* flags;
  unsigned* band_done;
  int panel_rows;  // multiple of BK
  int band_rows;   // multiple of BM
  // flags[p] covers B's panel p and A's panel p for rows < a_rows_first
  // only (the rows the first wave of tiles computes, uploaded first); the
  // remaining rows of A arrive after all panels and raise *a_rest
  int a_rows_first = 0x7fffffff;  // default: all of A is resident
  const unsigned* a_rest = nullptr;
};

// out of line: the main loop keeps the plain kernel's code generation
__device__ __noinline__ void wait_flag(const unsigned* f) {
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    while (ld_acquire_gpu(reinterpret_cast<const int*>(f)) == 0) {
      __nanosleep(256);
      if (clock64() - t0 > (1ll << 37)) __trap();  // ~70 s without the copy: fail loudly
    }
  }
  __syncthreads();
}

// column (within the tile) of micro-tile column j of thread column tx
template <class Cfg>
__device__ __forceinline__ int bcol(int tx, int j) {
  if constexpr (Cfg::PAIRB) return 2 * tx + (j & 1) + (j >> 1) * (2 * Cfg::TX);
  return tx + j * Cfg::TX;
}

// the thread's B values of k step kk from the stage
template <class Cfg>
__device__ __forceinline__ void load_b(double (&b)[Cfg::TN][Cfg::W], const double* Bs, int tx, int kk) {
  constexpr int W = Cfg::W, BK = Cfg::BK, TN = Cfg::TN;
  if constexpr (Cfg::PAIRB) {
#pragma unroll
    for (int jp = 0; jp < TN / 2; ++jp)
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const double2 v =
            *reinterpret_cast<const double2*>(Bs + w * BK * Cfg::BS + kk * Cfg::BS + bcol<Cfg>(tx, 2 * jp));
        b[2 * jp][w] = v.x;
        b[2 * jp + 1][w] = v.y;
      }
  } else {
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int w = 0; w < W; ++w) b[j][w] = Bs[w * BK * Cfg::BS + kk * Cfg::BS + bcol<Cfg>(tx, j)];
  }
}

// one k step of the register micro-tile: C (+)= A(:, kk) * B(kk, :)
template <class Cfg>
__device__ __forceinline__ void mac_step(double (&acc)[Cfg::TM][Cfg::TN][Cfg::W], const double* As,
                                         const double* Bs, int tx, int ty, int kk) {
  constexpr int W = Cfg::W, BM = Cfg::BM, TM = Cfg::TM, TN = Cfg::TN;
  constexpr int TY = Cfg::TY;
  double a[TM][W], b[TN][W];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int w = 0; w < W; ++w) a[i][w] = As[w * BM * Cfg::AS + (ty + i * TY) * Cfg::AS + kk];
  load_b<Cfg>(b, Bs, tx, kk);
  if constexpr (Cfg::ROWMAJ) {
#pragma unroll
    for (int i = 0; i < TM; ++i) arith::dd_mac_row<TN>(acc[i], a[i], b);
  } else {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        double p[W];
        arith::mp_mul<W>(a[i], b[j], p);
        arith::mp_add<W>(acc[i][j], p, acc[i][j]);
      }
  }
}

// mac_step with the branch-free renormalisation (Cfg::FASTR); ORs into
// `rare` when an input needed renorm5 paths C/D
template <class Cfg>
__device__ __forceinline__ void mac_step_fast(double (&acc)[Cfg::TM][Cfg::TN][Cfg::W], const double* As,
                                              const double* Bs, int tx, int ty, int kk,
                                              typename Cfg::Rare& rare) {
  constexpr int W = Cfg::W, BM = Cfg::BM, TM = Cfg::TM, TN = Cfg::TN;
  constexpr int TY = Cfg::TY;
  double a[TM][W], b[TN][W];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int w = 0; w < W; ++w) a[i][w] = As[w * BM * Cfg::AS + (ty + i * TY) * Cfg::AS + kk];
  load_b<Cfg>(b, Bs, tx, kk);
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      double p[W];
      arith::mp_mul_f<W, Cfg::FASTR, Cfg::VSEBF>(a[i], b[j], p, rare);
      arith::mp_add_f<W, Cfg::FASTR>(acc[i][j], p, acc[i][j], rare);
    }
}

// one k step in the lean form (Cfg::LEAN): acc holds levels, not a value
template <class Cfg>
__device__ __forceinline__ void mac_step_lean(double (&acc)[Cfg::TM][Cfg::TN][Cfg::W], const double* As,
                                              const double* Bs, int tx, int ty, int kk) {
  constexpr int W = Cfg::W, BM = Cfg::BM, TM = Cfg::TM, TN = Cfg::TN;
  constexpr int TY = Cfg::TY;
  double a[TM][W], b[TN][W];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int w = 0; w < W; ++w) a[i][w] = As[w * BM * Cfg::AS + (ty + i * TY) * Cfg::AS + kk];
  load_b<Cfg>(b, Bs, tx, kk);
  if constexpr (W == 2 && Cfg::LEAN == 2) {
    // stage-major across a micro-tile row (same operations, other order)
#pragma unroll
    for (int i = 0; i < TM; ++i) arith::lean_mac_dd_row<TN>(acc[i], a[i], b);
  } else {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) arith::lean_mac<W>(acc[i][j], a[i], b[j]);
  }
}

// One output tile (rows m0.., columns n0..) over the K range of g: the
// k = 0 step initialises the chains unless g.accumulate, which continues the
// chains stored in C.
// kMode: 0 plain, 1 fused all-gather (PullB), 2 copy-engine gated (GateArgs)
template <class Cfg, int kMode>
__device__ __forceinline__ void tile_run(const GemmArgs& g, int m0, int n0, const PullB& P,
                                         const GateArgs& G) {
  constexpr bool kPull = kMode == 1, kGate = kMode == 2;
  constexpr int W = Cfg::W, BM = Cfg::BM, BK = Cfg::BK;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, TX = Cfg::TX, TY = Cfg::TY;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ __align__(16) double smem[];
  double* As0 = smem;
  double* Bs0 = smem + STAGES * Cfg::A_STAGE;

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int ktiles = (g.K + BK - 1) / BK;

  double acc[TM][TN][W];
  if (Cfg::LEAN && !g.accumulate) {  // the levels start at +0: no peeled first step
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int w = 0; w < W; ++w) acc[i][j][w] = 0.0;
  }
  if (g.accumulate) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int gm = m0 + ty + i * TY, gn = n0 + bcol<Cfg>(tx, j);
        const bool ok = gm < g.M && gn < g.N;
#pragma unroll
        for (int w = 0; w < W; ++w) acc[i][j][w] = ok ? g.C[w * g.pc + (long long)gm * g.ldc + gn] : 0.0;
      }
  }

  // interior tile: every full k-tile takes the fast loader (FastLoad)
  const bool interior = FastLoad<Cfg>::ok && m0 + BM <= g.M && n0 + Cfg::BN <= g.N && fast_load_fits(g);
  const int kfull = g.K / BK;  // k-tiles [0, kfull) are full
  FastLoadState fl{};
  if (interior) fl = fast_load_init<Cfg>(g, m0, n0, 0);

  int ready_panel = -1;  // kPull: panels [0, ready_panel] are resident (visited in order)
  if (kGate && min(m0 + BM, g.M) > G.a_rows_first) wait_flag(G.a_rest);  // rows uploaded after the panels

  // prologue: fill STAGES-1 stages
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) {
      if (kPull && s * BK / P.panel_rows > ready_panel) {
        ready_panel = s * BK / P.panel_rows;
        ensure_panel<W>(P, g, ready_panel);
        help_panel<W>(P, g, ready_panel + 1);
      }
      if (kGate && s * BK / G.panel_rows > ready_panel) {
        ready_panel = s * BK / G.panel_rows;
        wait_flag(G.flags + ready_panel);
      }
      if (interior && s < kfull)
        fast_load_tile<Cfg>(fl, As0 + s * Cfg::A_STAGE, Bs0 + s * Cfg::B_STAGE, g);
      else
        load_tile<Cfg>(As0 + s * Cfg::A_STAGE, Bs0 + s * Cfg::B_STAGE, g, m0, n0, s * BK);
    }
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    if (Cfg::ONEBAR) {
      cp_async_wait<STAGES - 2>();  // tile kt has landed (later ones may be in flight)
      __syncthreads();              // ... for every thread; every warp is done with kt-1
    }
    // issue the tile STAGES-1 ahead into the slot freed last iteration
    {
      const int nt = kt + STAGES - 1;
      if (nt < ktiles) {
        const int slot = nt % STAGES;
        if (kPull && nt * BK / P.panel_rows > ready_panel) {  // a new panel: once per panel
          ready_panel = nt * BK / P.panel_rows;
          ensure_panel<W>(P, g, ready_panel);
          help_panel<W>(P, g, ready_panel + 1);
        }
        if (kGate && nt * BK / G.panel_rows > ready_panel) {
          ready_panel = nt * BK / G.panel_rows;
          wait_flag(G.flags + ready_panel);
        }
        if (interior && nt < kfull)
          fast_load_tile<Cfg>(fl, As0 + slot * Cfg::A_STAGE, Bs0 + slot * Cfg::B_STAGE, g);
        else
          load_tile<Cfg>(As0 + slot * Cfg::A_STAGE, Bs0 + slot * Cfg::B_STAGE, g, m0, n0, nt * BK);
      }
      cp_async_commit();
    }
    if (!Cfg::ONEBAR) {
      cp_async_wait<STAGES - 1>();
      __syncthreads();
    }

    const int slot = kt % STAGES;
    const double* As = As0 + slot * Cfg::A_STAGE;
    const double* Bs = Bs0 + slot * Cfg::B_STAGE;
    const int kend = min(BK, g.K - kt * BK);
    int kk = 0;
    if (!Cfg::LEAN && kt == 0 && !g.accumulate) {
      // k == 0: the product initialises the element (linalg.hpp:242, 260-261)
      double a[TM][W], b[TN][W];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int w = 0; w < W; ++w) a[i][w] = As[w * BM * Cfg::AS + (ty + i * TY) * Cfg::AS];
      load_b<Cfg>(b, Bs, tx, 0);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) arith::mp_mul<W>(a[i], b[j], acc[i][j]);
      kk = 1;
    }
    if constexpr (Cfg::LEAN) {
      if (Cfg::FIXK && kend == BK) {
#pragma unroll Cfg::KUNROLL
        for (int q = 0; q < BK; ++q) mac_step_lean<Cfg>(acc, As, Bs, tx, ty, q);
      } else {
#pragma unroll Cfg::KUNROLL
        for (int q = 0; q < kend; ++q) mac_step_lean<Cfg>(acc, As, Bs, tx, ty, q);
      }
      // once per k-tile: the levels back to nearly non-overlapping
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) arith::lean_renorm_loose<W>(acc[i][j]);
    } else if constexpr (Cfg::FASTR) {
      double* snap = smem + STAGES * (Cfg::A_STAGE + Cfg::B_STAGE) + threadIdx.x;
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int w = 0; w < W; ++w) snap[((i * TN + j) * W + w) * Cfg::THREADS] = acc[i][j][w];
      typename Cfg::Rare rare;
      if (Cfg::FIXK && kk == 0 && kend == BK) {
#pragma unroll Cfg::KUNROLL
        for (int q = 0; q < BK; ++q) mac_step_fast<Cfg>(acc, As, Bs, tx, ty, q, rare);
      } else {
#pragma unroll Cfg::KUNROLL
        for (int q = kk; q < kend; ++q) mac_step_fast<Cfg>(acc, As, Bs, tx, ty, q, rare);
      }
      if (__any_sync(0xffffffffu, rare.any())) {  // rare: this warp redoes the k-tile exactly
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_fastr_redo, 1ull);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int w = 0; w < W; ++w) acc[i][j][w] = snap[((i * TN + j) * W + w) * Cfg::THREADS];
        for (int q = kk; q < kend; ++q) mac_step<Cfg>(acc, As, Bs, tx, ty, q);
      }
    } else if (Cfg::FIXK && kk == 0 && kend == BK) {
#pragma unroll Cfg::KUNROLL
      for (int q = 0; q < BK; ++q) mac_step<Cfg>(acc, As, Bs, tx, ty, q);
    } else {
#pragma unroll Cfg::KUNROLL
      for (; kk < kend; ++kk) mac_step<Cfg>(acc, As, Bs, tx, ty, kk);
    }
    if (!Cfg::ONEBAR) __syncthreads();
  }
  cp_async_wait<0>();
  if (Cfg::ONEBAR) __syncthreads();  // the slots are free again (a persistent caller may refill them)

  if (ktiles == 0) return;  // K == 0 is handled by the host (C = +0)
  if constexpr (Cfg::LEAN) {  // levels -> canonical normalised values
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) arith::lean_finish<W>(acc[i][j], acc[i][j]);
  }
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
  if (kGate) {  // publish the finished tile to the download stream
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(G.band_done + m0 / G.band_rows, 1u);
    }
  }
}

// One CTA = one tile (blockIdx.x in GROUP_M order; batch-major for batches).
template <class Cfg, int kMode>
__device__ __forceinline__ void gemm_body(const GemmArgs& g0, const PullB& P, int klast = 0,
                                          const GateArgs& G = GateArgs{}) {
  const int tiles_m = (g0.M + Cfg::BM - 1) / Cfg::BM, tiles_n = (g0.N + Cfg::BN - 1) / Cfg::BN;
  int lin = blockIdx.x, bz = 0;
  if (g0.batch > 1) {
    bz = lin / (tiles_m * tiles_n);
    lin -= bz * tiles_m * tiles_n;
  }
  GemmArgs g = g0;
  if (klast && bz == g0.batch - 1) g.K = klast;  // split-K: ragged last segment
  g.A += bz * g0.sa;
  g.B += bz * g0.sb;
  g.C += bz * g0.sc;
  int tile_m, tile_n;
  tile_coords<Cfg::GROUP_M>(lin, tiles_m, tiles_n, tile_m, tile_n);
  tile_run<Cfg, kMode>(g, tile_m * Cfg::BM, tile_n * Cfg::BN, P, G);
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) mpgemm_kernel(const GemmArgs g0) {
  gemm_body<Cfg, 0>(g0, PullB{});
}

// MPFK_FAST split-K (csrc/splitk.cuh): the batch is the K segments, the
// last one running over klast k steps (a separate kernel so the product
// kernels keep their code generation).
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) mpgemm_splitk_kernel(const GemmArgs g0, int klast) {
  gemm_body<Cfg, 0>(g0, PullB{}, klast);
}

// The fused all-gather -> GEMM (see PullB); batch must be 1.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) mpgemm_pull_kernel(const GemmArgs g0, const PullB pull) {
  gemm_body<Cfg, 1>(g0, pull);
}

// Host operands streamed by the copy engines in K panels (see GateArgs);
// batch must be 1.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) mpgemm_gated_kernel(const GemmArgs g0, const GateArgs gate) {
  gemm_body<Cfg, 2>(g0, PullB{}, 0, gate);
}

}  // namespace kern
}  // namespace mpfk
