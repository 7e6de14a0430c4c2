// host_stage.inl -- pageable host operands: pinned staging ring + copy-thread
// pool (included by capi.cu inside its anonymous namespace, before Device).

// ---------------------------------------------------------------------------
// pageable host buffers (e.g. the reference's aligned_alloc'd MPMatrix): a
// ring of pinned staging slots filled and drained by a pool of copy threads,
// so the DMA of one slot overlaps the CPU copy of the next and the calling
// thread never sits in the driver's single-threaded staging path.
// ---------------------------------------------------------------------------
bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// persistent workers running one job at a time: f(worker, workers)
class CopyPool {
 public:
  explicit CopyPool(int n) : n_(n) {
    for (int i = 0; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void run(const std::function<void(int, int)>& f) {
    std::unique_lock<std::mutex> lk(mu_);
    job_ = &f;
    pending_ = n_;
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      const auto* f = job_;
      lk.unlock();
      (*f)(i, n_);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)>* job_ = nullptr;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

// rows x width bytes between two pitched host regions, split over the pool
void copy_rows(CopyPool& pool, char* dst, size_t dpitch, const char* src, size_t spitch, size_t width,
               size_t rows) {
  if (rows * width < (size_t(1) << 20)) {  // small: not worth waking the pool
    for (size_t r = 0; r < rows; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, width);
    return;
  }
  pool.run([&](int i, int n) {
    const size_t r0 = rows * i / n, r1 = rows * (i + 1) / n;
    for (size_t r = r0; r < r1; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, width);
  });
}

struct Stager {
  static constexpr int kSlots = 8;
  static constexpr size_t kSlotBytes = size_t(16) << 20;
  char* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  struct Out {  // a finished-or-in-flight download still to be copied out
    bool pending = false;
    char* dst = nullptr;
    size_t dpitch = 0, width = 0, rows = 0;
  } out[kSlots];
  int next = 0;
  std::unique_ptr<CopyPool> pool;

  void init() {  // on the owning device, lazily
    if (pool) return;
    for (int i = 0; i < kSlots; ++i) {
      ck(cudaMallocHost(reinterpret_cast<void**>(&slot[i]), kSlotBytes), "cudaMallocHost(staging)");
      ck(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const char* env = std::getenv("MPFK_COPY_THREADS");
    const int nthr = env && std::atoi(env) > 0 ? std::atoi(env) : (int)std::min(8u, hw);
    pool.reset(new CopyPool(nthr));
  }
  void release() {
    for (int i = 0; i < kSlots; ++i) {
      if (slot[i]) cudaFreeHost(slot[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
      slot[i] = nullptr, ev[i] = nullptr;
    }
    pool.reset();
  }
  void reset() {  // a new call: forget copy-outs of an aborted one
    for (auto& o : out) o.pending = false;
  }
  int acquire() {  // the oldest slot, once its DMA is done and its data copied out
    const int i = next;
    next = (next + 1) % kSlots;
    ck(cudaEventSynchronize(ev[i]), "staging slot");
    if (out[i].pending) {
      copy_rows(*pool, out[i].dst, out[i].dpitch, slot[i], out[i].width, out[i].width, out[i].rows);
      out[i].pending = false;
    }
    return i;
  }
  // host (pageable) -> device, pitched; enqueued on s
  void h2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows, cudaStream_t s) {
    if (!rows || !width) return;
    if (width > kSlotBytes) {  // a row larger than a slot: the driver's path
      ck(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyHostToDevice, s), "H2D");
      return;
    }
    init();
    const size_t per = kSlotBytes / width;
    for (size_t r = 0; r < rows; r += per) {
      const size_t pr = std::min(per, rows - r);
      const int i = acquire();
      copy_rows(*pool, slot[i], width, static_cast<const char*>(src) + r * spitch, spitch, width, pr);
      ck(cudaMemcpy2DAsync(static_cast<char*>(dst) + r * dpitch, dpitch, slot[i], width, width, pr,
                           cudaMemcpyHostToDevice, s),
         "H2D (staged)");
      ck(cudaEventRecord(ev[i], s), "event");
    }
  }
  // device -> host (pageable), pitched; the copy-out happens when the slot
  // is reused or at drain()
  void d2h(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows, cudaStream_t s) {
    if (!rows || !width) return;
    if (width > kSlotBytes) {
      ck(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToHost, s), "D2H");
      return;
    }
    init();
    const size_t per = kSlotBytes / width;
    for (size_t r = 0; r < rows; r += per) {
      const size_t pr = std::min(per, rows - r);
      const int i = acquire();
      ck(cudaMemcpy2DAsync(slot[i], width, static_cast<const char*>(src) + r * spitch, spitch, width, pr,
                           cudaMemcpyDeviceToHost, s),
         "D2H (staged)");
      ck(cudaEventRecord(ev[i], s), "event");
      out[i] = Out{true, static_cast<char*>(dst) + r * dpitch, dpitch, width, pr};
    }
  }
  void drain() {  // every pending copy-out, oldest first
    for (int k = 0; k < kSlots; ++k) {
      const int i = (next + k) % kSlots;
      if (!out[i].pending) continue;
      ck(cudaEventSynchronize(ev[i]), "staging slot");
      copy_rows(*pool, out[i].dst, out[i].dpitch, slot[i], out[i].width, out[i].width, out[i].rows);
      out[i].pending = false;
    }
  }
};
