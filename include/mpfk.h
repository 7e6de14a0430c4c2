/*
 * mpfk.h -- C ABI of the B200-native DD/TD/QD GEMM (libmpfk.so).
 *
 * The reference (mpfkit, /root/reference/proj) exposes no C ABI: its drop-in
 * surface is the header-only C++ template API in namespace mpfkit::linalg
 * (SURVEY.md section 8(b)).  These entry points are exactly what a binding of
 * that API to a GPU library needs; include/mpfk/linalg.hpp re-exposes them
 * with the reference's C++ signatures, types and exceptions, and
 * paper_2101_06584_b200/__init__.py binds them with ctypes.  Each function
 * cites the reference interface it replaces (paths relative to
 * /root/reference/proj).
 *
 * Conventions
 *  - A width-W matrix is W component planes (component 0 leads), each a
 *    row-major rows x stride binary64 array; plane w starts at
 *    base + w * plane_stride.  This is MPMatrix<W>'s layout
 *    (include/mpfkit/linalg.hpp:36-129, pad_columns :32-34) when
 *    stride == pad4(cols) and plane_stride == rows * stride.
 *  - Every call returns MPFK_OK or an error code; the message (identical to
 *    the reference's exception text where one exists) is in
 *    mpfk_last_error(), which is thread-local.
 *  - Results are bit-identical to the reference's per-element accumulation
 *    order (linalg.hpp:338-344) for every variant, n_min and GPU count.
 *  - There is no CPU fallback: without a usable GPU every compute call fails
 *    with MPFK_ENODEV.
 */
#ifndef MPFK_H_
#define MPFK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPFK_ABI_VERSION 1

/* error codes; the C++ shim maps them to the reference's exception types */
enum mpfk_status {
  MPFK_OK = 0,
  MPFK_EINVAL = 1,   /* std::invalid_argument (linalg.hpp:283-293, :409; config.hpp:25-28) */
  MPFK_ERUNTIME = 2, /* std::runtime_error (runtime.cpp:73-80: FP environment) */
  MPFK_ECUDA = 3,    /* CUDA runtime failure (message carries cudaGetErrorString) */
  MPFK_ENOMEM = 4,   /* std::bad_alloc (linalg.hpp:116) */
  MPFK_ENODEV = 5    /* no usable sm_100 device: there is no CPU fallback */
};

/* KernelVariant, linalg.hpp:149.  All three are bit-identical on the GPU
 * (one kernel); the value is validated exactly like the reference
 * (SIMD variants need n_min % 4 == 0, linalg.hpp:290-294). */
enum mpfk_variant { MPFK_NORMAL = 0, MPFK_SIMD_SET = 1, MPFK_SIMD_LOADSTORE = 2 };

typedef struct mpfk_mat {
  double *base;          /* W planes */
  uint64_t rows, cols;
  uint64_t stride;       /* row stride in doubles, >= cols */
  uint64_t plane_stride; /* doubles between planes; 0 means rows * stride */
} mpfk_mat;

/* Timings of the last host-buffer GEMM on this thread (device clocks, ms,
 * max over GPUs).  Row chunks are pipelined: uploads of chunk c+1 and the
 * download of chunk c-1 overlap the GEMM of chunk c, so the parts overlap. */
typedef struct mpfk_stats {
  double h2d_ms;    /* span of the host->device copies (B slice, A chunks) */
  double bcast_ms;  /* B replication over NVLink (peer all-gather), G > 1 */
  double kernel_ms; /* span of the GEMM launches (first chunk to last) */
  double d2h_ms;    /* exposed device->host tail after the last GEMM */
  double total_ms;  /* whole call, host wall clock */
  uint64_t h2d_bytes, d2h_bytes, peer_bytes;
  int n_gpus;
  int kernel_launches;
} mpfk_stats;

/* ---- runtime (runtime.hpp:10-30, runtime.cpp:48-81) -------------------- */

/* Once-init of the device context(s): checks for sm_100 devices and runs the
 * device FP-environment self-test (the twin of verify_fp_environment,
 * runtime.cpp:19-38,72-81) on each.  n_gpus <= 0 means all visible devices.
 * Idempotent; compute calls initialise lazily. */
int mpfk_init(int n_gpus);
void mpfk_shutdown(void);
const char *mpfk_last_error(void);
int mpfk_abi_version(void);
/* number of usable devices (0 when none); never fails */
int mpfk_device_count(void);
/* Make `dev` the calling thread's current device for libmpfk (and
 * initialise it).  libmpfk carries its own CUDA runtime; a host framework
 * that selected a device with its runtime (e.g. torch.cuda.set_device under
 * torchrun) should mirror that choice here.  mpfk_get_device returns the
 * current device (-1 when none). */
int mpfk_set_device(int dev);
int mpfk_get_device(void);
/* Device self-test on the current device: binary64 round-to-nearest-even and
 * a correctly rounded fused multiply-add (runtime.cpp:19-38). */
int mpfk_selftest(void);

/* ---- GEMM, host buffers: the drop-in for linalg::matmul_*_into --------- */

/* matmul_block_parallel_into(C, A, B, n_min, variant, workers),
 * linalg.hpp:402-433.  Validates shapes and n_min before any device work
 * with the reference's messages; clears C (fill_zero, linalg.hpp:94-96),
 * computes C = A*B on min(workers, devices) GPUs sharding C by contiguous
 * row spans (the reference's worker partition, linalg.hpp:413-421), leaves
 * C's padding cells +0 (zero_pads, :99-106) and bumps the op counters
 * (count_matmul, :175-180).  Synchronous: returns once C is on the host.
 * workers: 1..; GPUs actually used = min(workers, device count, row blocks). */
int mpfk_matmul_block_parallel_into(int width, mpfk_mat *C, const mpfk_mat *A, const mpfk_mat *B,
                                    uint64_t n_min, int variant, unsigned workers);
/* matmul_block_into, linalg.hpp:368-388 (one GPU) */
int mpfk_matmul_block_into(int width, mpfk_mat *C, const mpfk_mat *A, const mpfk_mat *B,
                           uint64_t n_min, int variant);
/* matmul_naive_into, linalg.hpp:346-358 (same result by construction) */
int mpfk_matmul_naive_into(int width, mpfk_mat *C, const mpfk_mat *A, const mpfk_mat *B,
                           int variant);
/* matmul_strassen / matmul_strassen_parallel (linalg.hpp:582-617) into a
 * caller-allocated m x n C: Strassen top levels on the GPU (per-level even
 * zero padding, the fixed M1..M7 operand order, exact width add/sub) with
 * the block GEMM as the leaf once min(m, K, n) <= cutoff.  Bit-identical to
 * the reference's Strassen (not to the block product -- a different
 * algorithm).  Errors as the reference ("matmul: cutoff must be at least
 * 1", ...).  Counts adds per mat_add/mat_sub, leaf multiplies, and each
 * leaf's count_matmul, like linalg.hpp:457, :468, :570. */
int mpfk_matmul_strassen(int width, mpfk_mat *C, const mpfk_mat *A, const mpfk_mat *B,
                         uint64_t cutoff, uint64_t n_min, int variant, unsigned workers);
/* Device-resident Strassen (same recursion and bits) on the current device /
 * `stream`: level-synchronous, one batched block GEMM for all leaves.
 * Scratch comes from the stream-ordered allocator. */
int mpfk_strassen_device(int width, uint64_t m, uint64_t n, uint64_t k, const double *A,
                         uint64_t lda, uint64_t a_plane, const double *B, uint64_t ldb,
                         uint64_t b_plane, double *C, uint64_t ldc, uint64_t c_plane,
                         uint64_t cutoff, void *stream, int *launches);
int mpfk_last_stats(mpfk_stats *out);

/* Flags of mpfk_gemm / mpfk_gemm_device_ex ("flags selects
 * BIT_EXACT (default) or FAST (reordered, tolerance-checked)").
 * MPFK_BIT_EXACT: the reference's per-element order; bit-identical to
 *   linalg::matmul_block_into (linalg.hpp:338-344).
 * MPFK_FAST: when the bit-exact launch would under-use the GPU (too few
 *   output tiles for the resident CTA slots, or a badly quantised last wave;
 *   predicted < 90 %) and k >= 512, K is cut into S segments, each a
 *   reference-order chain, and the S partial products are added in a fixed
 *   order (mpf::add<W>); otherwise identical to MPFK_BIT_EXACT.
 *   Deterministic for a given shape and device; normwise relative error
 *   within 4*k*u_p (u_p = 2^-104 / 2^-156 / 2^-208).
 * MPFK_LEAN: the north star's tolerance mode for the arithmetic itself.  The
 *   reference renormalises to a canonical value after every multiply and
 *   every add (mpf.hpp:105-238: 20 / 132 / 218 FP64 operations per
 *   multiply-add); a GEMM element is one long sum, so this mode keeps each
 *   element as W overlapping levels fed by exact two-sum cascades, pulls them
 *   back once per 16 k steps and normalises once at the end
 *   (csrc/mpf_lean.cuh: 10 / 42 / 107 FP64 instructions per multiply-add, 1.75x /
 *   2.6x / 1.96x the bit-exact GEMM's rate on a B200).  NOT bit-identical to
 *   the reference; results are canonical normalised values within the same
 *   normwise 4*k*u_p (measured: 1e-4..4e-3 of it on the BASELINE inputs,
 *   i.e. less accurate than the reference's own 4e-6..2e-4), deterministic
 *   and independent of tiling, sharding and K panels.  May be combined with
 *   MPFK_FAST (K segments keep the reference's arithmetic). */
enum mpfk_flags { MPFK_BIT_EXACT = 0u, MPFK_FAST = 1u, MPFK_LEAN = 2u };

/* The SURVEY's proposed entry point: C = A*B for host matrices in the
 * reference layout on n_gpus GPUs (<= 0: all visible), rows of C sharded
 * like matmul_block_parallel_into.  Validation, pads, op counters and
 * synchronous completion as mpfk_matmul_block_parallel_into; with
 * MPFK_BIT_EXACT it IS that call (n_min and variant have no effect on the
 * GPU). */
int mpfk_gemm(int width, const mpfk_mat *A, const mpfk_mat *B, mpfk_mat *C, int n_gpus,
              unsigned flags);

/* ---- GEMM, device-resident operands ------------------------------------ */

/* C[0:m,0:n] = A[0:m,0:k] * B[0:k,0:n] on the CURRENT device, enqueued on
 * `stream` (a cudaStream_t; NULL = legacy default stream), asynchronous.
 * Pointers are device memory of that device, 16-byte aligned, with even row
 * strides (pad4 strides of the reference layout qualify).  Only the m x n
 * cells of C are written.  k == 0 writes +0 into C.  Counts ops like
 * count_matmul.  Returns the number of kernel launches through *launches
 * when non-NULL. */
int mpfk_gemm_device(int width, uint64_t m, uint64_t n, uint64_t k, const double *A,
                     uint64_t lda, uint64_t a_plane, const double *B, uint64_t ldb,
                     uint64_t b_plane, double *C, uint64_t ldc, uint64_t c_plane, void *stream,
                     int *launches);

/* mpfk_gemm_device with flags (MPFK_FAST may split K; see mpfk_flags). */
int mpfk_gemm_device_ex(int width, uint64_t m, uint64_t n, uint64_t k, const double *A,
                        uint64_t lda, uint64_t a_plane, const double *B, uint64_t ldb,
                        uint64_t b_plane, double *C, uint64_t ldc, uint64_t c_plane, unsigned flags,
                        void *stream, int *launches);
/* the number of K segments MPFK_FAST uses for an m x n x k product on the
 * current device (1 = the bit-exact path); negative status on error */
int mpfk_splitk_segments(int width, uint64_t m, uint64_t n, uint64_t k);

/* Continuation over a K panel: C = C (+) A*B, i.e. every element's chain
 * continues with add(C, mul(A(i,k), B(k,j))) for k = 0..k-1 of this panel.
 * The reference carries the chain state in C between k steps
 * (QuadRow::axpy reloads C, linalg.hpp:261), so a GEMM split into K panels
 * -- the first through mpfk_gemm_device, the rest through this call, in
 * ascending k -- is bit-identical to the one-shot product.  Lets a caller
 * stream B (or A) in K panels and overlap the transfer with compute. */
int mpfk_gemm_device_acc(int width, uint64_t m, uint64_t n, uint64_t k, const double *A,
                         uint64_t lda, uint64_t a_plane, const double *B, uint64_t ldb,
                         uint64_t b_plane, double *C, uint64_t ldc, uint64_t c_plane, void *stream,
                         int *launches);
/* ... with flags: MPFK_BIT_EXACT, or MPFK_LEAN -- the tolerance-mode
 * arithmetic continues from the normalised value in C (each panel ends with
 * the lean form's final normalisation, so a panelled product is within the
 * tolerance of, not bit-identical to, the one-shot lean product). */
int mpfk_gemm_device_acc_ex(int width, uint64_t m, uint64_t n, uint64_t k, const double *A,
                            uint64_t lda, uint64_t a_plane, const double *B, uint64_t ldb,
                            uint64_t b_plane, double *C, uint64_t ldc, uint64_t c_plane,
                            unsigned flags, void *stream, int *launches);

/* Fused all-gather -> GEMM in ONE kernel: B is not resident on this device;
 * its rows [src_row0[s], src_row0[s+1]) live in source slice s (nsrc <= 8),
 * typically other GPUs' memory mapped over NVLink (mpfk_ipc_open), each a
 * W-plane (rows_s x ldb) array.  The GEMM kernel pulls B's K panels
 * (panel_rows rows, a multiple of 16) into the local buffer B on demand, in
 * chunks of chunk_rows handed out by atomic counters, so the transfer
 * overlaps the FP64 work tile by tile and every panel crosses the link once
 * per GPU.  Bit-identical to mpfk_gemm_device; after the call B holds the
 * whole matrix.  Source slices must stay unchanged until the call completes
 * on the stream. */
int mpfk_gemm_device_pull(int width, uint64_t m, uint64_t n, uint64_t k, const double *A,
                          uint64_t lda, uint64_t a_plane, double *B, uint64_t ldb, uint64_t b_plane,
                          double *C, uint64_t ldc, uint64_t c_plane, int nsrc,
                          const double *const *src, const uint64_t *src_row0, uint64_t panel_rows,
                          uint64_t chunk_rows, void *stream, int *launches);
/* All-gather -> GEMM with the copy engines doing the gather: B's K panels
 * are copied from the source slices (peer or IPC-mapped memory; same table
 * as mpfk_gemm_device_pull, up to 64 slices) into the local B on an
 * internal stream, each followed by a stream memory write of the panel's
 * flag, while ONE GEMM launch on `stream` waits per panel inside the kernel
 * -- the transfer overlaps the FP64 work tile by tile and costs no SM time.
 * Bit-identical to mpfk_gemm_device; after the call (in stream order) B
 * holds the whole matrix.  panel_rows: a multiple of 16.  Without stream
 * memory operations the gather completes before a plain GEMM launch. */
int mpfk_gemm_device_gathered(int width, uint64_t m, uint64_t n, uint64_t k, const double *A,
                              uint64_t lda, uint64_t a_plane, double *B, uint64_t ldb,
                              uint64_t b_plane, double *C, uint64_t ldc, uint64_t c_plane, int nsrc,
                              const double *const *src, const uint64_t *src_row0,
                              uint64_t panel_rows, void *stream, int *launches);
/* All-gather -> GEMM with no in-kernel waiting (the default multi-GPU
 * transport of bench.py): the copy engines gather B from the source slices
 * (same table as mpfk_gemm_device_gathered, up to 64 slices) on an internal
 * stream in ascending K panels -- a short first panel of head_rows rows
 * (0: 64), each next one 4x longer, at most 8 -- and one GEMM launch per
 * panel on `stream` waits on that panel's event only (panels after the
 * first continue the chains kept in C, as mpfk_gemm_device_acc).  Every
 * panel's compute covers the gather of the next, so only the first panel's
 * transfer is exposed, the gather costs no SM time, and no kernel spins on
 * a flag.  Bit-identical to mpfk_gemm_device; after the call (in stream
 * order) B holds the whole matrix.
 * Replaces, across GPUs, the reference's worker fan-out over row blocks
 * (linalg.hpp:402-433), which shares B through host memory. */
int mpfk_gemm_device_staged(int width, uint64_t m, uint64_t n, uint64_t k, const double *A,
                            uint64_t lda, uint64_t a_plane, double *B, uint64_t ldb,
                            uint64_t b_plane, double *C, uint64_t ldc, uint64_t c_plane, int nsrc,
                            const double *const *src, const uint64_t *src_row0,
                            uint64_t head_rows, void *stream, int *launches);
/* ... with flags: MPFK_BIT_EXACT, or MPFK_LEAN (every panel's launch in the
 * tolerance-mode arithmetic; deterministic for a given panel schedule). */
int mpfk_gemm_device_staged_ex(int width, uint64_t m, uint64_t n, uint64_t k, const double *A,
                               uint64_t lda, uint64_t a_plane, double *B, uint64_t ldb,
                               uint64_t b_plane, double *C, uint64_t ldc, uint64_t c_plane, int nsrc,
                               const double *const *src, const uint64_t *src_row0,
                               uint64_t head_rows, unsigned flags, void *stream, int *launches);
/* device memory and CUDA IPC plumbing for the fused path (one process per
 * GPU): handles are 64-byte cudaIpcMemHandle_t blobs. */
int mpfk_device_alloc(uint64_t bytes, void **ptr);
int mpfk_device_free(void *ptr);
int mpfk_memcpy(void *dst, const void *src, uint64_t bytes);
int mpfk_ipc_get_handle(const void *dev_ptr, void *handle_out);
int mpfk_ipc_open(const void *handle, void **dev_ptr);
int mpfk_ipc_close(void *dev_ptr);

/* ---- elementwise width kernels (mpf::add/mul<W>, mpf.hpp:341-353) ------- */

/* EwOp, linalg.hpp:623 */
enum mpfk_ew_op { MPFK_EW_ADD = 0, MPFK_EW_MUL = 1, MPFK_EW_ADD_MERGE = 2 };

/* linalg::ew_apply_into(out, a, b, op, variant), linalg.hpp:647-684:
 * out = op(a, b) cell by cell on the GPU (add/mul: the width's library
 * defaults, mpf.hpp:242-260; add_merge: td_add_merge, mpf.hpp:125-131, W = 3
 * only).  Errors "ew: shape mismatch" / "ew: add_merge is a triple-width
 * operation" (linalg.hpp:650-653).  SIMD variants leave out's pads +0, NORMAL
 * leaves them untouched, as in the reference.  Counts adds (add, add_merge)
 * or muls (mul) += rows*cols (linalg.hpp:682-683).  Synchronous. */
int mpfk_ew_apply_into(int width, int op, mpfk_mat *out, const mpfk_mat *a, const mpfk_mat *b,
                       int variant);
/* device-resident form on the current device / `stream`, asynchronous; only
 * the rows x cols cells of out are written; 16-byte aligned, even strides. */
int mpfk_ew_device(int width, int op, uint64_t rows, uint64_t cols, double *out, uint64_t ldo,
                   uint64_t o_plane, const double *a, uint64_t lda, uint64_t a_plane,
                   const double *b, uint64_t ldb, uint64_t b_plane, void *stream, int *launches);

/* r[i] = op(x[i], y[i]) for `count` values stored AoS (W doubles each) in
 * host memory, computed on the GPU.  op: 0 = add, 1 = mul (library
 * defaults for the width, mpf.hpp:242-260); width 3 also 2 = td_mul_q
 * (mpf.hpp:167-174) and 3 = td_add_merge (:125-131).  Used by the
 * arithmetic parity sweeps. */
int mpfk_binop_batch(int width, int op, uint64_t count, const double *x, const double *y,
                     double *r);

/* ---- MPFM matrix files (linalg_io.cpp:20-111, README.md:145-151) --------- */
/* 33-byte header {"MPFM", u32 version 1, u8 width, u64 rows, cols, stride =
 * pad4(cols)} + W little-endian binary64 planes, padding included and +0.
 * Errors (MPFK_ERUNTIME) carry the reference's texts: "<path>: cannot open",
 * "truncated", "not an MPFM file", "unsupported version", "component width
 * mismatch", "implausible dimensions", "bad stride", "trailing data",
 * "nonzero padding", "cannot open for writing", "write failed". */
int mpfk_mpfm_info(const char *path, int *width, uint64_t *rows, uint64_t *cols);
/* Stream a file's planes into device memory of the current device (any even
 * or odd ld >= cols; plane stride >= rows*ld) through pinned double-buffered
 * staging; returns once the data is on the device. */
int mpfk_mpfm_load_device(const char *path, int width, double *dev, uint64_t ld, uint64_t plane,
                          void *stream);
/* Write rows x cols device cells as an MPFM file (pads written +0). */
int mpfk_mpfm_save_device(const char *path, int width, const double *dev, uint64_t rows,
                          uint64_t cols, uint64_t ld, uint64_t plane, void *stream);
/* Host MPMatrix-layout forms: save_matrix_binary / load_matrix_binary
 * (linalg_io.cpp:66-111); load requires m preallocated with the file's
 * rows x cols (see mpfk_mpfm_info). */
int mpfk_mpfm_load_host(const char *path, int width, mpfk_mat *m);
int mpfk_mpfm_save_host(const char *path, int width, const mpfk_mat *m);

/* The EFT primitives on the GPU over `count` operand pairs (host arrays):
 * op 0 two_sum, 1 quick_two_sum, 2 two_prod (eft.hpp:46-67).  s + e is the
 * exact result (acceptance criterion 1). */
int mpfk_eft_batch(int op, uint64_t count, const double *a, const double *b, double *s, double *e);

/* ---- op counters (linalg.hpp:160-180, linalg.cpp:10-25) ----------------- */
void mpfk_op_counters_reset(void);
void mpfk_op_counters_read(uint64_t *adds, uint64_t *muls, uint64_t *leaf_multiplies);
/* What the calling thread's last entry point call added to the counters
 * above (exact for that call even when other threads count concurrently);
 * the C++ shim forwards it to the caller's own op counters. */
void mpfk_last_op_counts(uint64_t *adds, uint64_t *muls, uint64_t *leaf_multiplies);

/* TD/QD GEMM kernels run each k-tile with branch-free common paths (QD:
 * renorm5 path A, eft.hpp:255-257; TD: renorm5 paths A/B, eft.hpp:255-260,
 * and td_mul's vseb with a nonzero first residual, eft.hpp:205-225) and
 * recompute, exactly, any warp's k-tile that met an input outside them.
 * Number of such recomputed warp k-tiles on the current device since the
 * last reset (synchronises the device).  No reference counterpart; for
 * tests and the bench line. */
int mpfk_gemm_redo_count(uint64_t *count, int reset);

/* ---- pinned host memory for MPMatrix-style buffers ----------------------- */
/* aligned (>= 256 B), page-locked: host<->device copies run at full PCIe
 * bandwidth.  Replaces aligned_alloc(32, .) of linalg.hpp:115. */
void *mpfk_host_alloc(uint64_t bytes);
void mpfk_host_free(void *p);
/* Page-locking of long-lived pageable operands (opt-in; default capacity 0,
 * or MPFK_HOST_REGISTER_CACHE_MB from the environment): with a nonzero
 * capacity, a pageable host operand of >= 1 MiB given to a host-buffer call
 * (matmul_*, gemm, Strassen, ew) is cudaHostRegister'ed -- the whole
 * MPMatrix buffer, W planes from its base -- and kept registered in a
 * bounded LRU set, so later calls on the same buffer copy it by direct DMA
 * (the page-locked paths) instead of through the staging ring.  The caller
 * must drop a cached buffer (mpfk_host_unregister(base), or capacity 0 to
 * empty the set) BEFORE freeing it: freed-and-reused memory must never stay
 * registered.  A reference MPMatrix (aligned_alloc, linalg.hpp:115) is such
 * an operand.  mpfk_shutdown empties the set. */
int mpfk_host_register_cache(uint64_t capacity_bytes);
int mpfk_host_register_cache_stats(uint64_t *capacity, uint64_t *used, uint64_t *entries);
int mpfk_host_unregister(const void *base);

/* ---- seeded inputs (random.hpp:17-75) --------------------- */
/* The BASELINE.json configurations, generated row-parallel on the host:
 * per-row SplitMix64 stream state = seed ^ ((row+1) * 0xd1b54a32d192ed03);
 * narrow (wide == 0): c0 = 2u - 1; wide: c0 = +-(1+u) * 2^(x mod 61 - 30);
 * c_{i+1} = c_i * 2^-53 * (2u - 1); W == 2 -> quick_two_sum, W > 2 ->
 * renormalized<W> (mpf.hpp:76-88).  Pads (stride - cols) are set to +0.
 * Rows [row0, row0 + rows) of the seeded matrix are written (a row shard).
 * threads <= 0: hardware concurrency. */
int mpfk_fill_baseline(int width, int wide, uint64_t row0, uint64_t rows, uint64_t cols,
                       uint64_t stride, uint64_t seed, double *planes, int threads);

/* bench::fill_random (bench.cpp:295-302): one sequential SplitMix64 stream
 * from `seed` over the matrix in row-major order, each element
 * rng::random_normalized<W> (random.hpp:54-67, lead in [1,2)). */
int mpfk_fill_random(int width, uint64_t rows, uint64_t cols, uint64_t stride, uint64_t seed,
                     double *planes);
/* bench::gen_paper_matrices (bench.cpp:278-292): A(i,j) = sqrt5 * (i+j-1),
 * B(i,j) = sqrt3 * (n-i) (1-based), products taken in width W. */
int mpfk_gen_paper(int width, uint64_t n, uint64_t stride, double *A, double *B);

/* FP64 pipe microbenchmark on the current device: returns measured FP64
 * lane-operations per second (each DADD/DMUL/DFMA counted once), the
 * denominator of the roofline fraction (MEASURED_PEAKS.json has no FP64
 * entry). */
int mpfk_fp64_peak(double *ops_per_s, double *ms);

#ifdef __cplusplus
}
#endif

#endif /* MPFK_H_ */
