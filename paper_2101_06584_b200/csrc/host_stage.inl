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

// ---------------------------------------------------------------------------
// page-locking long-lived caller buffers (opt-in): a bounded LRU set of
// cudaHostRegister'ed ranges, keyed by the exact operand buffer (one
// MPMatrix<W> allocation: W planes from its base).  A registered operand
// takes the page-locked paths (direct DMA, the copy-engine-gated launch)
// from its second call on.  The caller promises the buffers stay allocated
// while cached: freeing registered memory and reallocating at the same
// address would leave a stale registration, so a caller that frees an
// operand first drops it (mpfk_host_unregister) or empties the cache
// (mpfk_host_register_cache(0)).  Off by default; mpfk_shutdown empties it.
// ---------------------------------------------------------------------------
class HostRegCache {
 public:
  void set_capacity(size_t bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    cap_ = bytes;
    while (used_ > cap_ && !ents_.empty()) evict_lru_locked();
  }
  size_t capacity() {
    std::lock_guard<std::mutex> lk(mu_);
    return cap_;
  }
  // true when [p, p + bytes) is page-locked after the call (cached, or
  // registered now); false leaves the operand on the staging path
  bool ensure(const void* p, size_t bytes) {
    if (!p || bytes < kMinBytes) return false;
    std::lock_guard<std::mutex> lk(mu_);
    if (!cap_ || bytes > cap_) return false;
    const char* b = static_cast<const char*>(p);
    for (auto& e : ents_)
      if (b >= e.base && b + bytes <= e.base + e.bytes) {
        e.last = ++tick_;
        return true;
      }
    // ranges overlapping the new one cannot stay registered beside it
    for (size_t i = 0; i < ents_.size();)
      if (b < ents_[i].base + ents_[i].bytes && ents_[i].base < b + bytes)
        drop_locked(i);
      else
        ++i;
    while (used_ + bytes > cap_ && !ents_.empty()) evict_lru_locked();
    if (cudaHostRegister(const_cast<char*>(b), bytes, cudaHostRegisterDefault) != cudaSuccess) {
      cudaGetLastError();  // e.g. registered by the caller already: not ours to manage
      return false;
    }
    ents_.push_back(Ent{b, bytes, ++tick_});
    used_ += bytes;
    return true;
  }
  void unregister(const void* p) {
    std::lock_guard<std::mutex> lk(mu_);
    for (size_t i = 0; i < ents_.size();)
      if (ents_[i].base == p)
        drop_locked(i);
      else
        ++i;
  }
  void clear() {
    std::lock_guard<std::mutex> lk(mu_);
    while (!ents_.empty()) drop_locked(ents_.size() - 1);
  }
  size_t used() {
    std::lock_guard<std::mutex> lk(mu_);
    return used_;
  }
  size_t entries() {
    std::lock_guard<std::mutex> lk(mu_);
    return ents_.size();
  }

 private:
  static constexpr size_t kMinBytes = size_t(1) << 20;  // below: the staging ring is as fast
  struct Ent {
    const char* base;
    size_t bytes;
    uint64_t last;
  };
  void drop_locked(size_t i) {
    cudaHostUnregister(const_cast<char*>(ents_[i].base));
    cudaGetLastError();
    used_ -= ents_[i].bytes;
    ents_.erase(ents_.begin() + (long)i);
  }
  void evict_lru_locked() {
    size_t lru = 0;
    for (size_t i = 1; i < ents_.size(); ++i)
      if (ents_[i].last < ents_[lru].last) lru = i;
    drop_locked(lru);
  }
  std::mutex mu_;
  std::vector<Ent> ents_;
  size_t cap_ = 0, used_ = 0;
  uint64_t tick_ = 0;
};

HostRegCache& host_reg_cache() {
  static HostRegCache* c = [] {
    auto* r = new HostRegCache;  // never destroyed: mpfk_shutdown empties it
    if (const char* env = std::getenv("MPFK_HOST_REGISTER_CACHE_MB"))
      r->set_capacity(size_t(std::max(0L, std::atol(env))) << 20);
    return r;
  }();
  return *c;
}

// an operand of W planes (rows x cols, row stride `stride`, plane stride
// `plane_stride`, in doubles) is page-locked, registering it through the
// cache when that is enabled -- exactly the bytes the operand spans, from
// its first cell to the last cell of its last plane, never beyond
bool host_operand_pinned(const void* base, int W, uint64_t rows, uint64_t cols, uint64_t stride,
                         uint64_t plane_stride) {
  if (!base) return true;
  if (is_pinned(base)) return true;
  if (!rows || !cols) return false;
  const uint64_t span = uint64_t(W - 1) * plane_stride + (rows - 1) * stride + cols;
  return host_reg_cache().ensure(base, sizeof(double) * size_t(span));
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
