// host_gemm.inl -- the host-buffer GEMM drivers behind mpfk_matmul_*_into /
// mpfk_gemm: the copy-engine-gated single launch and the row-chunked
// multi-GPU pipeline (included by capi.cu inside its anonymous namespace).

// The gated single launch stalls while its first wave of tiles consumes K
// panels faster than PCIe delivers them; it pays when the whole upload fits
// in about two first-wave durations (measured: DD/TD/QD n=1024, TD/QD n=4096
// gain; DD n=8192 -- 2 GiB of operands against an 11 ms first wave -- keeps
// the row-chunked path, whose chunk-0 GEMM walks B panel by panel).
// The tile shape and occupancy the gated launch uses, and the rows of A the
// first wave of tiles covers (whole GROUP_M bands of the tile raster,
// gemm_kernel.cuh:tile_coords): those rows go up with B's panels, the rest
// of A after them.
struct GatePlan {
  int bm, bn, minb;
  uint64_t a_rows_first;
  double waves;
};
GatePlan gate_plan(int W, uint64_t m, uint64_t n) {
  kern::GemmArgs g;
  g.M = (int)std::min<uint64_t>(m, 0x7fffffff), g.N = (int)std::min<uint64_t>(n, 0x7fffffff), g.batch = 1;
  GatePlan p{Cfg3::BM, Cfg3::BN, Cfg3::MINB, 0, 1.0};
  if (W == 4) p.bm = Cfg4::BM, p.bn = Cfg4::BN, p.minb = Cfg4::MINB;
  if (W == 2) {
    if (dd_small_tiles(g))
      p.bm = Cfg2s::BM, p.bn = Cfg2s::BN, p.minb = Cfg2s::MINB;
    else
      p.bm = Cfg2::BM, p.bn = Cfg2::BN, p.minb = Cfg2::MINB;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const double tiles_n = double((n + p.bn - 1) / p.bn);
  const double tiles = double((m + p.bm - 1) / p.bm) * tiles_n;
  const double slots = double(sms) * p.minb;
  p.waves = std::max(1.0, tiles / slots);
  constexpr int kGroupM = 16;  // TileCfg GROUP_M of every product configuration
  const double bands = std::ceil(std::min(slots, tiles) / (kGroupM * tiles_n));
  p.a_rows_first = std::min<uint64_t>(m, (uint64_t)bands * kGroupM * p.bm);
  return p;
}

bool gate_pays(int W, uint64_t m, uint64_t n, uint64_t K, double upload_bw) {
  const GatePlan p = gate_plan(W, m, n);
  const double ops = W == 2 ? 20.0 : W == 3 ? 132.0 : 218.0;
  const double kern_s = double(m) * n * K * ops / 18e12;  // ~FP64 peak
  // what the first wave waits for: B and the first-wave rows of A
  const double upload_s = 8.0 * W * (double(p.a_rows_first) * K + double(K) * n) / upload_bw;
  return upload_s <= 2.0 * kern_s / p.waves;
}

// One GPU: ONE GEMM launch gated by the copy engines.  A and B are uploaded
// in K panels on the copy stream (directly, or through the staging ring for
// pageable operands), each followed by a stream memory write of the panel's
// flag; the kernel, enqueued before the uploads, waits on
// a panel's flag before staging its first k-tile (kern::GateArgs), so it
// starts once the first panel has landed and never waits again while the
// copies stay ahead.  Finished tiles count per 256-row band; the download
// stream waits on each band's count (stream wait-value) and copies it out
// while later bands compute.  No chunking: the kernel keeps its full-size
// tile grid (the chunked path's under-filled launches were the main loss on
// small shapes).
void host_gemm_gated(int W, mpfk_mat* C, const mpfk_mat* A, const mpfk_mat* B, Device& D, mpfk_stats& st,
                     bool a_pin, bool b_pin, bool c_pin) {
  const uint64_t m = A->rows, K = A->cols, n = B->cols;
  const uint64_t lda = pad4(K), ldb = pad4(n), ldc = pad4(n);
  const uint64_t pa_h = plane_of(A), pb_h = plane_of(B), pc_h = plane_of(C);
  ck(cudaSetDevice(D.id), "cudaSetDevice");
  grow(D.dA, D.capA, sizeof(double) * W * std::max<uint64_t>(m * lda, 1));
  grow(D.dB, D.capB, sizeof(double) * W * std::max<uint64_t>(K * ldb, 1));
  grow(D.dC, D.capC, sizeof(double) * W * std::max<uint64_t>(m * ldc, 1));
  // K panels: >= 128 k steps, at most 32, a multiple of BK = 16 rows each.
  // The kernel starts once the first panel has landed, so smaller panels
  // start it sooner, but A's panel is a column slab whose 2D copy slows down
  // with narrow rows (measured: 64-k panels cost DD n=1024 e2e 4 %, helped
  // TD/QD n=1024 2 %; 256-k panels idle the GPU for the first 1/4 of A+B)
  const uint64_t np0 = std::max<uint64_t>(1, std::min<uint64_t>(32, K / 128));
  const uint64_t pk = ((K + np0 - 1) / np0 + 15) / 16 * 16;
  const uint64_t npan = (K + pk - 1) / pk;
  const uint64_t band_rows = 256;  // a multiple of every configuration's BM
  const uint64_t nb = (m + band_rows - 1) / band_rows;
  const size_t gate_bytes = sizeof(unsigned) * (npan + 1 + nb);
  if (gate_bytes > D.gate_cap) {
    if (D.gate) cudaFree(D.gate);
    D.gate = nullptr;
    D.gate_cap = 0;
    ck(cudaMalloc(reinterpret_cast<void**>(&D.gate), gate_bytes), "cudaMalloc(gate)");
    D.gate_cap = gate_bytes;
  }
  unsigned* flags = D.gate;               // [npan] B panel + first-wave rows of A
  unsigned* a_rest = D.gate + npan;       // the other rows of A
  unsigned* band_done = D.gate + npan + 1;
  const uint64_t m1 = gate_plan(W, m, n).a_rows_first;

  D.stage.reset();
  ck(cudaEventRecord(D.ev[0], D.up), "event");
  ck(cudaMemsetAsync(D.gate, 0, gate_bytes, D.up), "cudaMemsetAsync(gate)");
  ck(cudaEventRecord(D.ev[5], D.up), "event");  // flags and counters cleared

  // the kernel is enqueued first: it starts computing as soon as panel 0's
  // flag is written, while this thread is still issuing (or, for pageable
  // operands, staging) the later panels
  ck(cudaStreamWaitEvent(D.stream, D.ev[5], 0), "wait gate reset");
  ck(cudaEventRecord(D.ev[2], D.stream), "event");
  kern::GemmArgs g;
  g.A = D.dA, g.B = D.dB, g.C = D.dC;
  g.lda = (long long)lda, g.ldb = (long long)ldb, g.ldc = (long long)ldc;
  g.pa = (long long)(m * lda), g.pb = (long long)(K * ldb), g.pc = (long long)(m * ldc);
  g.M = (int)m, g.N = (int)n, g.K = (int)K;
  g.accumulate = 0;
  g.batch = 1, g.sa = g.sb = g.sc = 0;
  kern::GateArgs gate{flags, band_done, (int)pk, (int)band_rows, (int)m1, a_rest};
  const auto tile = dispatch_gemm_gated(W, g, gate, D.stream);
  ck(cudaEventRecord(D.ev[3], D.stream), "event");

  for (uint64_t p = 0; p < npan; ++p) {
    const uint64_t k0 = p * pk, k1 = std::min<uint64_t>(K, k0 + pk);
    for (int w = 0; w < W; ++w) {
      copy_h2d(D, a_pin, D.dA + w * m * lda + k0, lda, A->base + w * pa_h + k0, A->stride, k1 - k0, m1, D.up);
      copy_h2d(D, b_pin, D.dB + w * K * ldb + k0 * ldb, ldb, B->base + w * pb_h + k0 * B->stride, B->stride, n,
               k1 - k0, D.up);
    }
    cu_ck(g_write32(reinterpret_cast<CUstream>(D.up), reinterpret_cast<CUdeviceptr>(flags + p), 1, 0),
          "cuStreamWriteValue32");
  }
  if (m1 < m)
    for (int w = 0; w < W; ++w)
      copy_h2d(D, a_pin, D.dA + w * m * lda + m1 * lda, lda, A->base + w * pa_h + m1 * A->stride, A->stride, K,
               m - m1, D.up);
  cu_ck(g_write32(reinterpret_cast<CUstream>(D.up), reinterpret_cast<CUdeviceptr>(a_rest), 1, 0),
        "cuStreamWriteValue32");
  ck(cudaEventRecord(D.ev[1], D.up), "event");

  ck(cudaStreamWaitEvent(D.down, D.ev[5], 0), "wait gate reset");
  const uint64_t tiles_n = (n + tile.second - 1) / tile.second;
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t r0 = b * band_rows, r1 = std::min<uint64_t>(m, r0 + band_rows);
    const uint64_t tiles = (r1 - r0 + tile.first - 1) / tile.first * tiles_n;
    cu_ck(g_wait32(reinterpret_cast<CUstream>(D.down), reinterpret_cast<CUdeviceptr>(band_done + b),
                   (cuuint32_t)tiles, CU_STREAM_WAIT_VALUE_GEQ),
          "cuStreamWaitValue32");
    for (int w = 0; w < W; ++w)
      copy_d2h(D, c_pin, C->base + w * pc_h + r0 * C->stride, C->stride, D.dC + w * m * ldc + r0 * ldc, ldc, n,
               r1 - r0, D.down);
  }
  ck(cudaStreamWaitEvent(D.down, D.ev[3], 0), "join");
  ck(cudaEventRecord(D.ev[4], D.down), "event");
  ck(cudaEventSynchronize(D.ev[4]), "GEMM execution");
  D.stage.drain();
  float x = 0;
  cudaEventElapsedTime(&x, D.ev[0], D.ev[1]);
  st.h2d_ms = x;
  cudaEventElapsedTime(&x, D.ev[2], D.ev[3]);
  st.kernel_ms = x;
  cudaEventElapsedTime(&x, D.ev[3], D.ev[4]);
  st.d2h_ms = x;
  st.h2d_bytes = 8ull * W * (m * K + K * n);
  st.d2h_bytes = 8ull * W * m * n;
  st.kernel_launches = 1;
  st.n_gpus = 1;
}

// One GPU's share of a host-buffer GEMM: rows [r0, r1) of C.
struct Shard {
  int dev;
  uint64_t r0, r1;
  uint64_t b0, b1;  // B rows this GPU uploads itself (G > 1: a 1/G slice)
};

// The multi-GPU host-buffer GEMM.  Device layout: planes packed with
// ld = pad4(cols) (16-byte rows for cp.async), A shard rows only, full B.
// fast: MPFK_FAST -- shards whose output cannot fill the GPU take the
// split-K path (enqueue_gemm_fast); everything else is bit-exact.
// lean: MPFK_LEAN -- every launch that is not a split-K one runs the lean
// arithmetic (csrc/mpf_lean.cuh, tolerance mode); the chunked pipeline below
// (the copy-engine-gated single launch has no lean instantiation).
void host_gemm(int W, mpfk_mat* C, const mpfk_mat* A, const mpfk_mat* B, unsigned gpus, bool fast = false,
               bool lean = false) {
  std::lock_guard<std::mutex> call_lock(g_call_mu);
  const auto t0 = std::chrono::steady_clock::now();
  const uint64_t m = A->rows, K = A->cols, n = B->cols;
  mpfk_stats st{};
  // fill_zero (linalg.hpp:94-96) semantics: every C cell is defined below;
  // pads are cleared on the host.
  if (m == 0 || n == 0) {
    zero_host_pads(W, C);
    count_matmul(m, n, K);
    st.n_gpus = 0;
    st.total_ms = ms_since(t0);
    t_stats = st;
    return;
  }
  const int base = current_device();
  ensure_devices((int)gpus, base);
  int G = std::min<int>((int)gpus, g_ndev);
  // never more GPUs than 64-row blocks, like nt = min(workers, nblocks)
  G = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)G, (m + 63) / 64));
  const uint64_t lda = pad4(K), ldb = pad4(n), ldc = pad4(n);
  const uint64_t pa_h = plane_of(A), pb_h = plane_of(B), pc_h = plane_of(C);

  // contiguous row spans rounded to 64 rows (the DD tile height)
  std::vector<Shard> sh(G);
  const uint64_t per = ((m + G - 1) / G + 63) / 64 * 64;
  const uint64_t bper = (K + G - 1) / G;
  for (int g = 0; g < G; ++g) {
    sh[g].dev = (base + g) % g_ndev;  // the caller's device first
    sh[g].r0 = std::min<uint64_t>(m, g * per);
    sh[g].r1 = std::min<uint64_t>(m, (g + 1) * per);
    sh[g].b0 = G == 1 ? 0 : std::min<uint64_t>(K, g * bper);
    sh[g].b1 = G == 1 ? K : std::min<uint64_t>(K, (g + 1) * bper);
  }
  const bool peer = G > 1;
  if (peer) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (int a = 0; a < G; ++a) {
      const int pa = g_dev[sh[a].dev].id;
      ck(cudaSetDevice(pa), "cudaSetDevice");
      for (int b = 0; b < G; ++b) {
        const int pb = g_dev[sh[b].dev].id;
        if (pa == pb) continue;  // (emulated devices share one GPU)
        int can = 0;
        cudaDeviceCanAccessPeer(&can, pa, pb);
        if (!can) fail(MPFK_ECUDA, "mpfk: GPUs lack peer access for the B all-gather");
        cudaError_t e = cudaDeviceEnablePeerAccess(pb, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "enable peer");
        cudaGetLastError();
      }
    }
  }

  std::vector<float> h2d(G, 0.f), bc(G, 0.f), kms(G, 0.f), d2h(G, 0.f);
  std::vector<int> launches(G, 0);
  std::vector<std::exception_ptr> errs(G);
  std::vector<Fail> fails(G);
  std::vector<int> failed(G, 0);

  // Row chunks of each shard are pipelined over three streams: H2D of chunk
  // c+1 (copy engine) and D2H of chunk c-1 (second copy engine) overlap the
  // GEMM of chunk c.  Rows of C are independent, so chunking cannot change a
  // bit.  A chunk is sized to keep >= 4 64x64 tiles per SM per launch.  A
  // shard too small for two such chunks is cut into chunks that each fill
  // one wave of resident CTAs of the small-tile configuration; failing that,
  // into chunks of >= 1.5 small tiles per SM (the two compute streams fill
  // each other's tails) only when the copies are a large share of the work
  // (DD: 20 FP64 ops per MAC; TD/QD do 6-11x more per byte).  Measured on
  // DD/TD/QD n=1024.
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g_dev[base].id);
  int sBM = Cfg2s::BM, sBN = Cfg2s::BN, sMINB = Cfg2s::MINB;
  if (W == 3) sBM = Cfg3::BM, sBN = Cfg3::BN, sMINB = Cfg3::MINB;
  if (W == 4) sBM = Cfg4::BM, sBN = Cfg4::BN, sMINB = Cfg4::MINB;
  auto split = [](uint64_t rows, uint64_t min_rows) -> std::pair<uint64_t, uint64_t> {
    if (rows == 0) return {0, 0};
    // at most 8 uniform chunks (chunk_bounds may halve the first and last)
    const uint64_t nc = std::max<uint64_t>(1, std::min<uint64_t>(8, rows / std::max<uint64_t>(min_rows, 1)));
    const uint64_t crows = ((rows + nc - 1) / nc + 63) / 64 * 64;
    return std::make_pair((rows + crows - 1) / std::max<uint64_t>(crows, 1), crows);
  };
  auto chunks_of = [&](uint64_t rows) {
    const double big = double(n) / (64.0 * 64.0);
    const uint64_t min_rows = (uint64_t)std::ceil(sms * 4.0 / std::max(big, 1e-9));
    if (rows >= 2 * min_rows) return split(rows, min_rows);
    // chunks that each fill one wave of resident CTAs
    const uint64_t tiles_per_band = (n + sBN - 1) / sBN;
    const uint64_t wave_rows = (uint64_t(sms) * sMINB + tiles_per_band - 1) / tiles_per_band * sBM;
    const auto wave = split(rows, wave_rows);
    if (wave.first >= 2) return wave;
    // under-filled chunks only when the copies are a large share
    const double ops = W == 2 ? 20.0 : W == 3 ? 132.0 : 218.0;
    const double copy_s = 8.0 * W * double(rows * K + K * n + rows * n) / 50e9;  // ~PCIe 5 x16
    const double kern_s = double(rows) * n * K * ops / 18e12;                    // ~FP64 peak
    if (copy_s > 0.3 * kern_s)
      return split(rows, (uint64_t)std::ceil(sms * 1.5 / std::max(double(tiles_per_band) / sBM, 1e-9)));
    return split(rows, rows);
  };
  // Row boundaries of a shard's chunks.  Large shards (the >= 4-tiles-per-SM
  // rule) get a half-size first and last chunk: the first GEMM starts after
  // half the A rows, and the download left exposed after the last GEMM is
  // half a chunk.
  auto chunk_bounds = [&](uint64_t rows) {
    if (rows == 0) return std::vector<uint64_t>{0, 0};  // an empty shard (G > row blocks / per)
    const auto pr = chunks_of(rows);
    const uint64_t nc = pr.first, crows = pr.second;
    std::vector<uint64_t> b{0};
    const double big = double(n) / (64.0 * 64.0);
    const uint64_t min_rows = (uint64_t)std::ceil(sms * 4.0 / std::max(big, 1e-9));
    if (nc >= 2 && rows >= 2 * min_rows && crows >= 128) {
      const uint64_t h = crows / 2 / 64 * 64;
      b.push_back(h);
      while (b.back() + crows < rows) b.push_back(b.back() + crows);
    } else {
      for (uint64_t c = 1; c < nc; ++c) b.push_back(std::min(rows, c * crows));
    }
    if (b.back() < rows) b.push_back(rows);
    return b;
  };
  // Single GPU: B is uploaded in K panels right after the first A chunk, and
  // the first chunk's GEMM runs panel by panel (continuing the chains from C,
  // bit-identical) so compute starts before all of B has landed.
  auto panels_of = [&](uint64_t k) -> std::pair<int, uint64_t> {
    if (peer || k < 1024) return {1, k};
    const int np = (int)std::min<uint64_t>(kMaxChunks, k / 512);
    const uint64_t pk = ((k + np - 1) / np + 15) / 16 * 16;  // even: 16-byte cp.async rows
    return {(int)((k + pk - 1) / pk), pk};
  };
  const bool a_pin = host_operand_pinned(A->base, W, A->rows, A->cols, A->stride, plane_of(A));
  const bool b_pin = host_operand_pinned(B->base, W, B->rows, B->cols, B->stride, plane_of(B));
  const bool c_pin = host_operand_pinned(C->base, W, C->rows, C->cols, C->stride, plane_of(C));
  // (pageable operands keep the chunked path: measured, staging A's narrow
  // K-panel columns through the copy threads costs more than the single
  // launch saves)
  if (G == 1 && a_pin && b_pin && c_pin && K > 0 && !lean && !std::getenv("MPFK_CHUNKED_HOST") &&
      gate_pays(W, m, n, K, 50e9) && memops_available() && !(fast && splitk_plan(W, m, n, K).S > 1)) {
    int prev = 0;
    cudaGetDevice(&prev);
    host_gemm_gated(W, C, A, B, g_dev[sh[0].dev], st, a_pin, b_pin, c_pin);
    cudaSetDevice(prev);
    zero_host_pads(W, C);
    count_matmul(m, n, K);
    st.total_ms = ms_since(t0);
    t_stats = st;
    return;
  }
  for (int g = 0; g < G; ++g) g_dev[sh[g].dev].stage.reset();

  std::vector<int> nchunks(G, 0);
  std::vector<std::vector<uint64_t>> bounds(G);
  // MPFK_FAST splits K only for a shard whose whole output cannot fill the
  // GPU (the same decision mpfk_splitk_segments reports for its shape); such
  // a shard runs as one chunk, every other shard is bit-exact
  std::vector<char> fast_split(G, 0);
  for (int g = 0; g < G; ++g) {
    const uint64_t rows = sh[g].r1 - sh[g].r0;
    fast_split[g] = fast && rows && splitk_plan(W, rows, n, K).S > 1;
    bounds[g] = fast_split[g] ? std::vector<uint64_t>{0, rows} : chunk_bounds(rows);
  }
  // One GPU, page-locked A and B, K long enough for panels: chunk 0's A goes
  // up in the same K panels as B (its narrow column blocks are plain DMA), so
  // the first GEMM starts after one small panel instead of a whole A chunk;
  // the panels grow 4x from 64 k rows, each panel's upload hiding under the
  // previous panel's GEMM (chunk 0 = the first two standard chunks, so its
  // compute per k row is ~5x the upload of a B row plus its A column).
  const bool kpanel0 = G == 1 && a_pin && b_pin && !fast_split[0] && panels_of(K).first > 1 &&
                       bounds[0].size() > 3;
  if (kpanel0) bounds[0].erase(bounds[0].begin() + 1);
  std::vector<uint64_t> cuts{0};
  if (kpanel0) {
    for (uint64_t h = 64; (int)cuts.size() < kMaxChunks && cuts.back() + h < K && h * 2 <= K - cuts.back(); h *= 4)
      cuts.push_back(cuts.back() + h);
    cuts.push_back(K);
  } else {
    const auto pp = panels_of(K);
    for (int p = 1; p <= pp.first; ++p) cuts.push_back(std::min<uint64_t>(K, p * pp.second));
  }
  const int ncuts = (int)cuts.size() - 1;
  auto upload_a = [&](int g, int c) {  // A row chunk c of shard g
    Shard& s = sh[g];
    Device& D = g_dev[s.dev];
    const uint64_t rows = s.r1 - s.r0;
    const uint64_t c0 = bounds[g][c], c1 = bounds[g][c + 1];
    for (int w = 0; w < W; ++w)
      copy_h2d(D, a_pin, D.dA + w * rows * lda + c0 * lda, lda, A->base + w * pa_h + (s.r0 + c0) * A->stride,
          A->stride, K, c1 - c0, D.up);
    ck(cudaEventRecord(D.evA[c], D.up), "event");
  };
  // One GPU with pageable operands: the staged copies occupy the calling
  // thread, so A chunks c >= 1 are staged just before chunk c's GEMM, and
  // chunk 0's K-panel GEMMs are enqueued as each B panel lands, instead of
  // after all uploads (with page-locked buffers the copies are asynchronous
  // and the order of the calls does not matter).
  const bool defer_a = G == 1 && !a_pin;
  const bool panel_split0 = !fast_split[0];
  const bool early0 = G == 1 && !b_pin && panels_of(K).first > 1 && panel_split0;
  auto gemm_chunk0_panel = [&](Device& D, int p) {
    const uint64_t rows = m, c1 = bounds[0][1];
    const uint64_t k0 = cuts[p], k1 = cuts[p + 1];
    if (p == 0) ck(cudaStreamWaitEvent(D.stream, D.evA[0], 0), "wait A chunk");
    ck(cudaStreamWaitEvent(D.stream, D.evB[p], 0), "wait B panel");
    return enqueue_gemm(W, c1, n, k1 - k0, D.dA + k0, lda, rows * lda, D.dB + k0 * ldb, ldb, K * ldb, D.dC, ldc,
                        rows * ldc, D.stream, p > 0, lean);
  };
  auto phase1 = [&](int g) {  // allocate; upload A chunk 0, B (slice or K panels), other A chunks
    Shard& s = sh[g];
    Device& D = g_dev[s.dev];
    ck(cudaSetDevice(D.id), "cudaSetDevice");
    const uint64_t rows = s.r1 - s.r0;
    grow(D.dA, D.capA, sizeof(double) * W * std::max<uint64_t>(rows * lda, 1));
    grow(D.dB, D.capB, sizeof(double) * W * std::max<uint64_t>(K * ldb, 1));
    grow(D.dC, D.capC, sizeof(double) * W * std::max<uint64_t>(rows * ldc, 1));
    nchunks[g] = rows ? (int)bounds[g].size() - 1 : 0;
    ck(cudaEventRecord(D.ev[0], D.up), "event");
    if (early0) ck(cudaEventRecord(D.ev[2], D.stream), "event");
    if (nchunks[g] && !kpanel0) upload_a(g, 0);
    // B's own rows in panels: the K cuts on one GPU, uniform panels of the
    // GPU's 1/G slice otherwise
    std::vector<uint64_t> bc;
    if (G == 1) {
      bc = cuts;
    } else {
      const auto ppair = panels_of(s.b1 - s.b0);
      for (int p = 0; p <= ppair.first; ++p) bc.push_back(std::min<uint64_t>(s.b1, s.b0 + p * ppair.second));
    }
    for (int p = 0; p + 1 < (int)bc.size(); ++p) {
      const uint64_t k0 = bc[p], k1 = bc[p + 1];
      if (kpanel0 && nchunks[g]) {  // chunk 0's A columns [k0, k1) with the panel
        const uint64_t c1 = bounds[g][1];
        for (int w = 0; w < W; ++w)
          copy_h2d(D, a_pin, D.dA + w * rows * lda + k0, lda, A->base + w * pa_h + s.r0 * A->stride + k0,
                   A->stride, k1 - k0, c1, D.up);
      }
      for (int w = 0; w < W; ++w)
        if (k1 > k0)
          copy_h2d(D, b_pin, D.dB + w * K * ldb + k0 * ldb, ldb, B->base + w * pb_h + k0 * B->stride, B->stride, n,
              k1 - k0, D.up);
      ck(cudaEventRecord(D.evB[p], D.up), "event");
      if (early0 && nchunks[g]) launches[g] += gemm_chunk0_panel(D, p);
    }
    if (kpanel0 && nchunks[g]) ck(cudaEventRecord(D.evA[0], D.up), "event");
    ck(cudaEventRecord(D.ev[1], D.up), "event");
    if (!defer_a)
      for (int c = 1; c < nchunks[g]; ++c) upload_a(g, c);
  };
  auto download = [&](int g, int c) {  // C row chunk c of shard g, after its GEMM
    Shard& s = sh[g];
    Device& D = g_dev[s.dev];
    const uint64_t rows = s.r1 - s.r0;
    const uint64_t c0 = bounds[g][c], c1 = bounds[g][c + 1];
    ck(cudaStreamWaitEvent(D.down, D.evC[c], 0), "wait C chunk");
    for (int w = 0; w < W; ++w)
      copy_d2h(D, c_pin, C->base + w * pc_h + (s.r0 + c0) * C->stride, C->stride, D.dC + w * rows * ldc + c0 * ldc,
               ldc, n, c1 - c0, D.down);
  };
  auto phase2 = [&](int g) {  // gather B slices from peers, compute chunks, download chunks
    Shard& s = sh[g];
    Device& D = g_dev[s.dev];
    ck(cudaSetDevice(D.id), "cudaSetDevice");
    const uint64_t rows = s.r1 - s.r0;
    if (!early0) ck(cudaEventRecord(D.ev[2], D.stream), "event");
    if (peer) {
      ck(cudaStreamWaitEvent(D.stream, D.ev[1], 0), "wait B upload");
      for (int o = 0; o < G; ++o) {
        if (o == g || sh[o].b1 == sh[o].b0) continue;
        Device& P = g_dev[sh[o].dev];
        ck(cudaStreamWaitEvent(D.stream, P.ev[1], 0), "wait peer upload");
        for (int w = 0; w < W; ++w)
          ck(cudaMemcpyPeerAsync(D.dB + w * K * ldb + sh[o].b0 * ldb, D.id,
                                 P.dB + w * K * ldb + sh[o].b0 * ldb, P.id,
                                 (sh[o].b1 - sh[o].b0) * ldb * 8, D.stream),
             "peer copy B");
      }
      ck(cudaEventRecord(D.ev[5], D.stream), "event");  // B complete on this GPU
    }
    const cudaEvent_t b_ready = peer ? D.ev[5] : D.ev[1];
    const int np = ncuts;
    for (int c = 0; c < nchunks[g]; ++c) {
      cudaStream_t cs = (c & 1) ? D.stream2 : D.stream;
      const uint64_t c0 = bounds[g][c], c1 = bounds[g][c + 1];
      if (defer_a && c > 0) upload_a(g, c);
      // (kpanel0: chunk 0's A arrives with the B panels; each panel's event covers both)
      if (!(kpanel0 && c == 0)) ck(cudaStreamWaitEvent(cs, D.evA[c], 0), "wait A chunk");
      if (c == 0 && early0) {
        // enqueued panel by panel in phase1
      } else if (fast_split[g]) {  // one chunk: the whole shard
        ck(cudaStreamWaitEvent(cs, b_ready, 0), "wait B");
        launches[g] += enqueue_gemm_fast(W, c1 - c0, n, K, D.dA + c0 * lda, lda, rows * lda, D.dB, ldb,
                                         K * ldb, D.dC + c0 * ldc, ldc, rows * ldc, cs);
      } else if (c == 0 && np > 1) {
        for (int p = 0; p < np; ++p) {
          const uint64_t k0 = cuts[p], k1 = cuts[p + 1];
          ck(cudaStreamWaitEvent(cs, D.evB[p], 0), "wait B panel");
          launches[g] += enqueue_gemm(W, c1 - c0, n, k1 - k0, D.dA + c0 * lda + k0, lda, rows * lda,
                                      D.dB + k0 * ldb, ldb, K * ldb, D.dC + c0 * ldc, ldc, rows * ldc, cs,
                                      p > 0, lean);
        }
      } else {
        ck(cudaStreamWaitEvent(cs, b_ready, 0), "wait B");
        launches[g] += enqueue_gemm(W, c1 - c0, n, K, D.dA + c0 * lda, lda, rows * lda, D.dB, ldb,
                                    K * ldb, D.dC + c0 * ldc, ldc, rows * ldc, cs, false, lean);
      }
      ck(cudaEventRecord(D.evC[c], cs), "event");
      // pageable C: a staged download occupies this thread until its chunk
      // is computed, so it trails by one chunk (GEMM c is already queued)
      if (c_pin) download(g, c);
      else if (c > 0) download(g, c - 1);
    }
    if (!c_pin && nchunks[g]) download(g, nchunks[g] - 1);
    ck(cudaEventRecord(D.evJ, D.stream2), "event");
    ck(cudaStreamWaitEvent(D.stream, D.evJ, 0), "join");
    ck(cudaEventRecord(D.ev[3], D.stream), "event");
    ck(cudaStreamWaitEvent(D.down, D.ev[3], 0), "join");
    ck(cudaEventRecord(D.ev[4], D.down), "event");
    ck(cudaEventSynchronize(D.ev[4]), "GEMM execution");
    D.stage.drain();
    const cudaEvent_t h2d_end = nchunks[g] > 1 ? D.evA[nchunks[g] - 1] : D.ev[1];
    cudaEventElapsedTime(&h2d[g], D.ev[0], h2d_end);
    bc[g] = 0.f;
    cudaEventElapsedTime(&kms[g], D.ev[2], D.ev[3]);  // compute span incl. waits for data
    cudaEventElapsedTime(&d2h[g], D.ev[3], D.ev[4]);  // exposed download tail
  };
  auto run_all = [&](auto&& fn) {
    if (G == 1) {
      fn(0);
      return;
    }
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g)
      th.emplace_back([&, g] {
        try {
          fn(g);
        } catch (const Fail& f) {
          fails[g] = f;
          failed[g] = 1;
        } catch (...) {
          errs[g] = std::current_exception();
        }
      });
    for (auto& t : th) t.join();
    for (int g = 0; g < G; ++g) {
      if (failed[g]) throw fails[g];
      if (errs[g]) std::rethrow_exception(errs[g]);
    }
  };
  int prev = 0;
  cudaGetDevice(&prev);
  run_all(phase1);
  run_all(phase2);
  cudaSetDevice(prev);

  zero_host_pads(W, C);
  count_matmul(m, n, K);
  for (int g = 0; g < G; ++g) {
    const uint64_t rows = sh[g].r1 - sh[g].r0;
    st.h2d_ms = std::max<double>(st.h2d_ms, h2d[g]);
    st.bcast_ms = std::max<double>(st.bcast_ms, bc[g]);
    st.kernel_ms = std::max<double>(st.kernel_ms, kms[g]);
    st.d2h_ms = std::max<double>(st.d2h_ms, d2h[g]);
    st.h2d_bytes += 8ull * W * (rows * K + (sh[g].b1 - sh[g].b0) * n);
    st.d2h_bytes += 8ull * W * rows * n;
    st.peer_bytes += peer ? 8ull * W * (K - (sh[g].b1 - sh[g].b0)) * ldb : 0;
    st.kernel_launches += launches[g];
  }
  st.n_gpus = G;
  st.total_ms = ms_since(t0);
  t_stats = st;
}
