// strassen.inl -- Strassen top levels on the GPU with the block GEMM as the
// leaf.  Included by capi.cu inside its anonymous
// namespace.
//
// The reference recurses depth-first (linalg.hpp:565-578), one node at a
// time.  All nodes at one depth have the same padded shape (ceil halves of
// their parent's), so here a whole level runs at once:
//   level d (batch b = 7^d): one strassen_operands launch per side builds
//   all 7b child operands; the next level recurses on them; at the leaf depth
//   (min(m, K, n) <= cutoff) ONE batched GEMM launch computes all 7^D leaf
//   products; on the way back one strassen_combine launch per level builds
//   every parent's C from its children's products.
// A few dozen launches instead of ~10^4.  If a level's operands would not
// fit the memory budget, that level is processed depth-first (children one
// at a time) and the levels below it level-synchronously again.
// Each element sees the reference's operations in the reference's order, so
// the result is bit-identical to mpfkit::linalg::matmul_strassen (and its
// parallel form).  Op counters follow the reference: every mat_add/mat_sub
// adds rows*cols adds (linalg.hpp:457, 468), every leaf one leaf multiply
// (:570) plus count_matmul of its block GEMM (:387).

struct BMat {  // a batch of width-W device matrices
  double* p = nullptr;
  uint64_t rows = 0, cols = 0, ld = 0, plane = 0, bstride = 0;
  int batch = 0;
  kern::BatchRef ref() const {
    return {p, (long long)ld, (long long)plane, (long long)bstride};
  }
  kern::BatchOut out() const { return {p, (long long)ld, (long long)plane, (long long)bstride}; }
};

struct StrassenCtx {
  int W;
  uint64_t cutoff;
  cudaStream_t s;
  uint64_t budget;  // bytes the level-synchronous scratch may use
  int launches = 0;

  BMat alloc(int batch, uint64_t rows, uint64_t cols) {
    BMat m;
    m.rows = rows, m.cols = cols, m.ld = std::max<uint64_t>(pad4(cols), 4);
    m.plane = rows * m.ld, m.bstride = W * m.plane, m.batch = batch;
    const size_t bytes = sizeof(double) * std::max<uint64_t>(uint64_t(batch) * m.bstride, 1);
    ck(cudaMallocAsync(reinterpret_cast<void**>(&m.p), bytes, s), "cudaMallocAsync");
    return m;
  }
  void release(BMat& m) {
    if (m.p) ck(cudaFreeAsync(m.p, s), "cudaFreeAsync");
    m.p = nullptr;
  }
  uint64_t bytes_of(uint64_t batch, uint64_t rows, uint64_t cols) const {
    return 8ull * W * batch * rows * std::max<uint64_t>(pad4(cols), 4);
  }
  // scratch a level-synchronous subtree needs below a node batch
  uint64_t subtree_bytes(uint64_t batch, uint64_t m, uint64_t K, uint64_t n) const {
    if (std::min({m, K, n}) <= cutoff) return 0;
    const uint64_t hm = (m + 1) / 2, hk = (K + 1) / 2, hn = (n + 1) / 2, c = batch * 7;
    return bytes_of(c, hm, hk) + bytes_of(c, hk, hn) + bytes_of(c, hm, hn) + subtree_bytes(c, hm, hk, hn);
  }

  unsigned grid_for(uint64_t elems) const {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((elems + 255) / 256, 148ull * 16));
  }

  template <int SIDE>
  void operands(const BMat& src, const BMat& dst, uint64_t h0, uint64_t h1, int t0, int t1) {
    const uint64_t elems = uint64_t(src.batch) * h0 * h1;
    const unsigned g = grid_for(elems);
#define MPFK_OPS(WW)                                                                               \
  kern::strassen_operands<WW, SIDE><<<g, 256, 0, s>>>(src.ref(), dst.out(), src.batch, (int)src.rows, \
                                                      (int)src.cols, (int)h0, (int)h1, t0, t1)
    if (W == 2) MPFK_OPS(2);
    else if (W == 3) MPFK_OPS(3);
    else MPFK_OPS(4);
#undef MPFK_OPS
    ck(cudaGetLastError(), "strassen operands launch");
    ++launches;
    // mat_add/mat_sub among the 7 (L: t in {0,1,4,5,6}; R: t in {0,2,3,5,6})
    uint64_t ops = 0;
    for (int t = t0; t < t1; ++t) ops += SIDE == 0 ? (t != 2 && t != 3) : (t != 1 && t != 4);
    tally_adds(ops * src.batch * h0 * h1);
  }

  void combine(const BMat& M, const BMat& C) {
    const uint64_t elems = uint64_t(C.batch) * C.rows * C.cols;
    const unsigned g = grid_for(elems);
#define MPFK_CMB(WW) \
  kern::strassen_combine<WW><<<g, 256, 0, s>>>(M.ref(), C.out(), C.batch, (int)C.rows, (int)C.cols, (int)M.rows, (int)M.cols)
    if (W == 2) MPFK_CMB(2);
    else if (W == 3) MPFK_CMB(3);
    else MPFK_CMB(4);
#undef MPFK_CMB
    ck(cudaGetLastError(), "strassen combine launch");
    ++launches;
    tally_adds(8ull * C.batch * M.rows * M.cols);  // 8 adds/subs
  }

  // L: batch of m x K, R: batch of K x n; writes the products into C
  // (batch of m x n, possibly a strided view of a larger buffer).
  void solve(const BMat& L, const BMat& R, const BMat& C) {
    const uint64_t m = L.rows, K = L.cols, n = R.cols;
    const int b = L.batch;
    if (std::min({m, K, n}) <= cutoff) {  // the leaves: one batched block GEMM
      tally_leaf(b);
      launches += enqueue_gemm_batched(W, b, m, n, K, L.p, L.ld, L.plane, L.bstride, R.p, R.ld, R.plane,
                                       R.bstride, C.p, C.ld, C.plane, C.bstride, s);
      if (K) {
        tally_muls(uint64_t(b) * m * n * K);
        tally_adds(uint64_t(b) * m * n * (K - 1));
      }
      return;
    }
    const uint64_t hm = (m + 1) / 2, hk = (K + 1) / 2, hn = (n + 1) / 2;
    BMat M = alloc(b * 7, hm, hn);
    if (subtree_bytes(b, m, K, n) <= budget) {
      BMat L2 = alloc(b * 7, hm, hk), R2 = alloc(b * 7, hk, hn);
      operands<0>(L, L2, hm, hk, 0, 7);
      operands<1>(R, R2, hk, hn, 0, 7);
      solve(L2, R2, M);
      release(L2);
      release(R2);
    } else {  // depth-first over the 7 products of this level
      for (int t = 0; t < 7; ++t) {
        BMat L2 = alloc(b, hm, hk), R2 = alloc(b, hk, hn);
        operands<0>(L, L2, hm, hk, t, t + 1);
        operands<1>(R, R2, hk, hn, t, t + 1);
        BMat Mt = M;  // children b*7 + t: a strided view
        Mt.p = M.p + t * M.bstride;
        Mt.bstride = 7 * M.bstride;
        Mt.batch = b;
        solve(L2, R2, Mt);
        release(L2);
        release(R2);
      }
    }
    combine(M, C);
    release(M);
  }
};

// Strassen on device operands (single matrices) of the current device.
int strassen_device(int W, uint64_t m, uint64_t n, uint64_t k, const double* A, uint64_t lda, uint64_t pa,
                    const double* B, uint64_t ldb, uint64_t pb, double* C, uint64_t ldc, uint64_t pc,
                    uint64_t cutoff, cudaStream_t s) {
  size_t free_b = 0, total_b = 0;
  ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  uint64_t budget = (uint64_t)(0.4 * free_b);
  if (const char* e = std::getenv("MPFK_STRASSEN_BUDGET_BYTES")) budget = std::strtoull(e, nullptr, 10);
  StrassenCtx ctx{W, cutoff, s, budget};
  BMat a, b, c;
  a.p = const_cast<double*>(A), a.rows = m, a.cols = k, a.ld = lda, a.plane = pa, a.bstride = W * pa, a.batch = 1;
  b.p = const_cast<double*>(B), b.rows = k, b.cols = n, b.ld = ldb, b.plane = pb, b.bstride = W * pb, b.batch = 1;
  c.p = C, c.rows = m, c.cols = n, c.ld = ldc, c.plane = pc, c.bstride = W * pc, c.batch = 1;
  if (m == 0 || n == 0) {
    tally_leaf(1);  // min(m, K, n) <= cutoff: one empty leaf
    return 0;
  }
  ctx.solve(a, b, c);
  return ctx.launches;
}

// Host-buffer matmul_strassen: upload A and B, run on the device, download C.
// `workers` only validates (the reference's parallel form reorders
// independent products and is bit-identical to serial).
void host_strassen(int W, mpfk_mat* Cm, const mpfk_mat* A, const mpfk_mat* B, uint64_t cutoff) {
  std::lock_guard<std::mutex> call_lock(g_call_mu);
  const auto t0 = std::chrono::steady_clock::now();
  mpfk_stats st{};
  const uint64_t m = A->rows, K = A->cols, n = B->cols;
  if (m == 0 || n == 0) {
    tally_leaf(1);
    zero_host_pads(W, Cm);
    t_stats = st;
    return;
  }
  const int dev = current_device();
  ensure_devices(1, dev);
  Device& D = g_dev[dev];
  const uint64_t lda = pad4(K), ldb = pad4(n), ldc = pad4(n);
  grow(D.dA, D.capA, sizeof(double) * W * std::max<uint64_t>(m * lda, 1));
  grow(D.dB, D.capB, sizeof(double) * W * std::max<uint64_t>(K * ldb, 1));
  grow(D.dC, D.capC, sizeof(double) * W * std::max<uint64_t>(m * ldc, 1));
  const uint64_t pa = plane_of(A), pb = plane_of(B), pc = plane_of(Cm);
  const bool a_pin = host_operand_pinned(A->base, W, A->rows, A->cols, A->stride, plane_of(A)),
             b_pin = host_operand_pinned(B->base, W, B->rows, B->cols, B->stride, plane_of(B));
  const bool c_pin = host_operand_pinned(Cm->base, W, Cm->rows, Cm->cols, Cm->stride, plane_of(Cm));
  D.stage.reset();
  ck(cudaEventRecord(D.ev[0], D.stream), "event");
  for (int w = 0; w < W; ++w) {
    copy_h2d(D, a_pin, D.dA + w * m * lda, lda, A->base + w * pa, A->stride, K, m, D.stream);
    copy_h2d(D, b_pin, D.dB + w * K * ldb, ldb, B->base + w * pb, B->stride, n, K, D.stream);
  }
  ck(cudaEventRecord(D.ev[1], D.stream), "event");
  st.kernel_launches = strassen_device(W, m, n, K, D.dA, lda, m * lda, D.dB, ldb, K * ldb, D.dC, ldc,
                                       m * ldc, cutoff, D.stream);
  ck(cudaEventRecord(D.ev[2], D.stream), "event");
  for (int w = 0; w < W; ++w)
    copy_d2h(D, c_pin, Cm->base + w * pc, Cm->stride, D.dC + w * m * ldc, ldc, n, m, D.stream);
  ck(cudaEventRecord(D.ev[3], D.stream), "event");
  ck(cudaEventSynchronize(D.ev[3]), "Strassen execution");
  D.stage.drain();
  zero_host_pads(W, Cm);
  float x = 0;
  cudaEventElapsedTime(&x, D.ev[0], D.ev[1]);
  st.h2d_ms = x;
  cudaEventElapsedTime(&x, D.ev[1], D.ev[2]);
  st.kernel_ms = x;
  cudaEventElapsedTime(&x, D.ev[2], D.ev[3]);
  st.d2h_ms = x;
  st.n_gpus = 1;
  st.h2d_bytes = 8ull * W * (m * K + K * n);
  st.d2h_bytes = 8ull * W * m * n;
  st.total_ms = ms_since(t0);
  t_stats = st;
}
