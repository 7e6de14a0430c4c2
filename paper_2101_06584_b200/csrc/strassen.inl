// strassen.inl -- Strassen top levels on the GPU with the block GEMM as the
// leaf.  Included by capi.cu inside its anonymous
// namespace.
//
// Restates linalg.hpp:472-617 step for step on device-resident operands:
// per-level zero padding to even sizes (copy_block, :483-498), the 14
// operands in the fixed M1..M7 order (:522-540) built with the width's exact
// add / sub (mat_add/mat_sub, :450-470 -> the ew kernel), the seven products
// recursed until min(m, K, n) <= cutoff where the leaf is the block GEMM
// (:569-571), and the combine (:543-563) with clipping paste.  Every step is
// the reference's operation on the same values in the same order, so the
// result is bit-identical to mpfkit::linalg::matmul_strassen (and to its
// parallel form, which only reorders independent products).  Op counters
// follow the reference: mat_add/mat_sub add rows*cols adds, each leaf adds
// one leaf multiply plus count_matmul of its block GEMM.

struct DMat {
  double* p = nullptr;
  uint64_t rows = 0, cols = 0, ld = 0;
  uint64_t plane() const { return rows * ld; }
};

struct StrassenCtx {
  int W;
  uint64_t cutoff;
  cudaStream_t s;
  std::vector<double*> owned;  // freed stream-ordered at the end of each level

  DMat alloc(uint64_t rows, uint64_t cols) {
    DMat m;
    m.rows = rows, m.cols = cols, m.ld = std::max<uint64_t>(pad4(cols), 4);
    const size_t bytes = sizeof(double) * W * std::max<uint64_t>(m.plane(), 1);
    ck(cudaMallocAsync(reinterpret_cast<void**>(&m.p), bytes, s), "cudaMallocAsync");
    ck(cudaMemsetAsync(m.p, 0, bytes, s), "cudaMemsetAsync");
    return m;
  }
  void release(DMat& m) {
    if (m.p) ck(cudaFreeAsync(m.p, s), "cudaFreeAsync");
    m.p = nullptr;
  }

  // copy_block, linalg.hpp:483-498: window outside the source stays +0
  DMat copy_block(const DMat& src, uint64_t i0, uint64_t j0, uint64_t rows, uint64_t cols) {
    DMat r = alloc(rows, cols);
    if (i0 >= src.rows || j0 >= src.cols) return r;
    const uint64_t ni = std::min(rows, src.rows - i0), nj = std::min(cols, src.cols - j0);
    for (int w = 0; w < W; ++w)
      ck(cudaMemcpy2DAsync(r.p + w * r.plane(), r.ld * 8, src.p + w * src.plane() + i0 * src.ld + j0,
                           src.ld * 8, nj * 8, ni, cudaMemcpyDeviceToDevice, s),
         "copy_block");
    return r;
  }

  // paste_block, linalg.hpp:501-514: clipped to dst's bounds
  void paste_block(DMat& dst, const DMat& src, uint64_t i0, uint64_t j0) {
    if (i0 >= dst.rows || j0 >= dst.cols) return;
    const uint64_t ni = std::min(src.rows, dst.rows - i0), nj = std::min(src.cols, dst.cols - j0);
    for (int w = 0; w < W; ++w)
      ck(cudaMemcpy2DAsync(dst.p + w * dst.plane() + i0 * dst.ld + j0, dst.ld * 8, src.p + w * src.plane(),
                           src.ld * 8, nj * 8, ni, cudaMemcpyDeviceToDevice, s),
         "paste_block");
  }

  // mat_add / mat_sub, linalg.hpp:450-470
  DMat ew(const DMat& a, const DMat& b, int op) {
    DMat r = alloc(a.rows, a.cols);
    enqueue_ew(W, op, a.rows, a.cols, r.p, r.ld, r.plane(), a.p, a.ld, a.plane(), b.p, b.ld, b.plane(), s);
    g_adds.fetch_add(a.rows * a.cols, std::memory_order_relaxed);
    return r;
  }
  DMat add(const DMat& a, const DMat& b) { return ew(a, b, kern::EW_ADD); }
  DMat sub(const DMat& a, const DMat& b) { return ew(a, b, kern::EW_SUB); }
  DMat copy(const DMat& a) { return copy_block(a, 0, 0, a.rows, a.cols); }

  // strassen_rec, linalg.hpp:565-578
  DMat rec(const DMat& A, const DMat& B, int& launches) {
    const uint64_t m = A.rows, K = A.cols, n = B.cols;
    if (std::min({m, K, n}) <= cutoff) {
      g_leaf.fetch_add(1, std::memory_order_relaxed);
      DMat C = alloc(m, n);
      launches += enqueue_gemm(W, m, n, K, A.p, A.ld, A.plane(), B.p, B.ld, B.plane(), C.p, C.ld,
                               C.plane(), s);
      count_matmul(m, n, K);
      return C;
    }
    const uint64_t hm = (m + 1) / 2, hk = (K + 1) / 2, hn = (n + 1) / 2;
    DMat A11 = copy_block(A, 0, 0, hm, hk), A12 = copy_block(A, 0, hk, hm, hk);
    DMat A21 = copy_block(A, hm, 0, hm, hk), A22 = copy_block(A, hm, hk, hm, hk);
    DMat B11 = copy_block(B, 0, 0, hk, hn), B12 = copy_block(B, 0, hn, hk, hn);
    DMat B21 = copy_block(B, hk, 0, hk, hn), B22 = copy_block(B, hk, hn, hk, hn);
    // the 14 operands in the fixed M1..M7 order, linalg.hpp:532-538
    DMat L[7], R[7];
    L[0] = add(A11, A22), R[0] = add(B11, B22);  // M1
    L[1] = add(A21, A22), R[1] = copy(B11);      // M2
    L[2] = copy(A11), R[2] = sub(B12, B22);      // M3
    L[3] = copy(A22), R[3] = sub(B21, B11);      // M4
    L[4] = add(A11, A12), R[4] = copy(B22);      // M5
    L[5] = sub(A21, A11), R[5] = add(B11, B12);  // M6
    L[6] = sub(A12, A22), R[6] = add(B21, B22);  // M7
    for (DMat* x : {&A11, &A12, &A21, &A22, &B11, &B12, &B21, &B22}) release(*x);
    DMat M[7];
    for (int t = 0; t < 7; ++t) {
      M[t] = rec(L[t], R[t], launches);
      release(L[t]);
      release(R[t]);
    }
    // strassen_combine, linalg.hpp:543-563
    DMat t1 = add(M[0], M[3]), t2 = sub(t1, M[4]);
    DMat C11 = add(t2, M[6]);
    DMat C12 = add(M[2], M[4]);
    DMat C21 = add(M[1], M[3]);
    DMat t3 = sub(M[0], M[1]), t4 = add(t3, M[2]);
    DMat C22 = add(t4, M[5]);
    DMat C = alloc(m, n);
    paste_block(C, C11, 0, 0);
    paste_block(C, C12, 0, hn);
    paste_block(C, C21, hm, 0);
    paste_block(C, C22, hm, hn);
    for (DMat* x : {&t1, &t2, &t3, &t4, &C11, &C12, &C21, &C22}) release(*x);
    for (auto& x : M) release(x);
    return C;
  }
};

// Host-buffer matmul_strassen: upload A and B, recurse on the device,
// download C.  `workers` only validates (the seven products are
// independent; the reference's parallel form is bit-identical to serial).
void host_strassen(int W, mpfk_mat* Cm, const mpfk_mat* A, const mpfk_mat* B, uint64_t cutoff) {
  std::lock_guard<std::mutex> call_lock(g_call_mu);
  const auto t0 = std::chrono::steady_clock::now();
  mpfk_stats st{};
  const uint64_t m = A->rows, K = A->cols, n = B->cols;
  if (m == 0 || n == 0) {  // min(m, K, n) <= cutoff: one (empty) leaf
    g_leaf.fetch_add(1, std::memory_order_relaxed);
    zero_host_pads(W, Cm);
    t_stats = st;
    return;
  }
  const int dev = current_device();
  ensure_devices(1, dev);
  Device& D = g_dev[dev];
  StrassenCtx ctx{W, cutoff, D.stream, {}};
  ck(cudaEventRecord(D.ev[0], D.stream), "event");
  DMat dA = ctx.alloc(m, K), dB = ctx.alloc(K, n);
  const uint64_t pa = plane_of(A), pb = plane_of(B), pc = plane_of(Cm);
  for (int w = 0; w < W; ++w) {
    if (K) {
      ck(cudaMemcpy2DAsync(dA.p + w * dA.plane(), dA.ld * 8, A->base + w * pa, A->stride * 8, K * 8, m,
                           cudaMemcpyHostToDevice, D.stream), "H2D A");
      ck(cudaMemcpy2DAsync(dB.p + w * dB.plane(), dB.ld * 8, B->base + w * pb, B->stride * 8, n * 8, K,
                           cudaMemcpyHostToDevice, D.stream), "H2D B");
    }
  }
  ck(cudaEventRecord(D.ev[1], D.stream), "event");
  int launches = 0;
  DMat dC;
  if (K == 0) {
    dC = ctx.alloc(m, n);  // an empty product: every cell +0
    g_leaf.fetch_add(1, std::memory_order_relaxed);
  } else {
    dC = ctx.rec(dA, dB, launches);
  }
  ck(cudaEventRecord(D.ev[2], D.stream), "event");
  for (int w = 0; w < W; ++w)
    ck(cudaMemcpy2DAsync(Cm->base + w * pc, Cm->stride * 8, dC.p + w * dC.plane(), dC.ld * 8, n * 8, m,
                         cudaMemcpyDeviceToHost, D.stream), "D2H C");
  ck(cudaEventRecord(D.ev[3], D.stream), "event");
  ctx.release(dA);
  ctx.release(dB);
  ctx.release(dC);
  ck(cudaEventSynchronize(D.ev[3]), "Strassen execution");
  ck(cudaStreamSynchronize(D.stream), "Strassen execution");
  zero_host_pads(W, Cm);
  float x = 0;
  cudaEventElapsedTime(&x, D.ev[0], D.ev[1]);
  st.h2d_ms = x;
  cudaEventElapsedTime(&x, D.ev[1], D.ev[2]);
  st.kernel_ms = x;
  cudaEventElapsedTime(&x, D.ev[2], D.ev[3]);
  st.d2h_ms = x;
  st.kernel_launches = launches;
  st.n_gpus = 1;
  st.h2d_bytes = 8ull * W * (m * K + K * n);
  st.d2h_bytes = 8ull * W * m * n;
  st.total_ms = ms_since(t0);
  t_stats = st;
}
