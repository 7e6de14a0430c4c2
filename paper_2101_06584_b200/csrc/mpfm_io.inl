// mpfm_io.inl -- MPFM matrix files straight to / from device buffers
// (SURVEY.md 8(f) row 2).  Included by capi.cu inside its anonymous
// namespace (uses its error helpers and device context).
//
// Format (linalg_io.cpp:20-23, 66-111; README.md:145-151): a 33-byte header
//   "MPFM" | u32 version = 1 | u8 width | u64 rows | u64 cols | u64 stride
// (little-endian, stride = pad4(cols)), then the W component planes as
// little-endian binary64, rows*stride values each, padding included and +0.
// Errors are the reference's std::runtime_error texts, "<path>: <what>".
//
// The planes stream through two page-locked staging buffers: while chunk i
// is copied host->device (or device->host), chunk i+1 is read from (or
// chunk i-1 written to) the file, and the zero-padding invariant is checked
// on the staged rows, so a multi-GiB matrix reaches HBM at disk speed
// without a host-side MPMatrix.

constexpr char kMpfmMagic[4] = {'M', 'P', 'F', 'M'};
constexpr uint32_t kMpfmVersion = 1;
constexpr uint64_t kMpfmMaxDim = uint64_t{1} << 32;
constexpr size_t kMpfmHeader = 33;
constexpr size_t kStageBytes = size_t(64) << 20;

[[noreturn]] void io_fail(const std::string& path, const std::string& what) {
  fail(MPFK_ERUNTIME, path + ": " + what);
}

uint64_t le_get(const unsigned char* p, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= uint64_t{p[i]} << (8 * i);
  return v;
}

void le_put(unsigned char* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
}

struct File {
  std::FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

struct MpfmHeader {
  int width;
  uint64_t rows, cols, stride;
};

// load_matrix_binary's header checks, linalg_io.cpp:88-102, plus the
// size check that the reference performs while reading (truncated /
// trailing data, :59-61, :104).
MpfmHeader read_header(std::FILE* f, const std::string& path, int want_width) {
  unsigned char h[kMpfmHeader];
  if (std::fread(h, 1, sizeof h, f) != sizeof h) io_fail(path, "truncated");
  if (std::memcmp(h, kMpfmMagic, 4) != 0) io_fail(path, "not an MPFM file");
  if (le_get(h + 4, 4) != kMpfmVersion) io_fail(path, "unsupported version");
  MpfmHeader r;
  r.width = h[8];
  if (want_width > 0 && r.width != want_width) io_fail(path, "component width mismatch");
  r.rows = le_get(h + 9, 8);
  r.cols = le_get(h + 17, 8);
  r.stride = le_get(h + 25, 8);
  if (r.rows > kMpfmMaxDim || r.cols > kMpfmMaxDim) io_fail(path, "implausible dimensions");
  if (r.stride != pad4(r.cols)) io_fail(path, "bad stride");
  if (r.width < 2 || r.width > 4) io_fail(path, "component width mismatch");
  if (std::fseek(f, 0, SEEK_END) != 0) io_fail(path, "cannot seek");
  const long long size = std::ftell(f);
  // 33 + 8 W rows stride without wrapping: a crafted header must not pass
  // the size check with an undersized payload
  unsigned long long cells = 0, need = 0;
  if (__builtin_mul_overflow((unsigned long long)r.rows, (unsigned long long)r.stride, &cells) ||
      __builtin_mul_overflow(cells, 8ull * r.width, &need) ||
      __builtin_add_overflow(need, (unsigned long long)kMpfmHeader, &need))
    io_fail(path, "implausible dimensions");
  if (size < 0 || (unsigned long long)size < need) io_fail(path, "truncated");
  if ((unsigned long long)size > need) io_fail(path, "trailing data");
  std::fseek(f, (long)kMpfmHeader, SEEK_SET);
  return r;
}

void write_header(std::FILE* f, const std::string& path, int W, uint64_t rows, uint64_t cols) {
  unsigned char h[kMpfmHeader];
  std::memcpy(h, kMpfmMagic, 4);
  le_put(h + 4, kMpfmVersion, 4);
  h[8] = static_cast<unsigned char>(W);
  le_put(h + 9, rows, 8);
  le_put(h + 17, cols, 8);
  le_put(h + 25, pad4(cols), 8);
  if (std::fwrite(h, 1, sizeof h, f) != sizeof h) io_fail(path, "write failed");
}

bool pads_zero(const double* rowsbuf, uint64_t nrows, uint64_t cols, uint64_t stride) {
  for (uint64_t i = 0; i < nrows; ++i)
    for (uint64_t j = cols; j < stride; ++j) {
      uint64_t u;
      std::memcpy(&u, rowsbuf + i * stride + j, 8);
      if (u != 0) return false;
    }
  return true;
}

// Pinned double-buffered staging shared by load and save.
// (host-only transfers use plain memory and no events, so they work without
// a GPU)
struct Stage {
  bool pinned;
  double* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  Stage(size_t bytes, bool pinned_) : pinned(pinned_) {
    for (int i = 0; i < 2; ++i) {
      if (pinned) {
        ck(cudaMallocHost(&buf[i], bytes), "cudaMallocHost(staging)");
        ck(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "cudaEventCreate");
      } else {
        buf[i] = static_cast<double*>(std::malloc(bytes));
        if (!buf[i]) throw std::bad_alloc();
      }
    }
  }
  void wait(int i) {
    if (pinned) ck(cudaEventSynchronize(ev[i]), "staging");
  }
  ~Stage() {
    for (int i = 0; i < 2; ++i) {
      if (pinned) {
        if (ev[i]) {
          cudaEventSynchronize(ev[i]);
          cudaEventDestroy(ev[i]);
        }
        if (buf[i]) cudaFreeHost(buf[i]);
      } else {
        std::free(buf[i]);
      }
    }
  }
};

// rows per staging chunk for a row of `stride` doubles
uint64_t chunk_rows(uint64_t stride) {
  return std::max<uint64_t>(1, kStageBytes / (8 * std::max<uint64_t>(stride, 1)));
}

// dst: device (dev != 0) or host planes, row stride ld, plane stride plane.
void mpfm_load(const char* cpath, int W, double* dst, uint64_t ld, uint64_t plane, bool device,
               cudaStream_t s) {
  const std::string path = cpath ? cpath : "";
  File F;
  F.f = std::fopen(path.c_str(), "rb");
  if (!F.f) io_fail(path, "cannot open");
  const MpfmHeader h = read_header(F.f, path, W);
  if (ld < h.cols) fail(MPFK_EINVAL, "mpfk: leading dimension too small");
  uint64_t plane_need = 0;
  if (h.rows && (__builtin_mul_overflow(h.rows, ld, &plane_need) || plane < plane_need))
    fail(MPFK_EINVAL, "mpfk: plane stride too small");
  if (h.rows == 0 || h.stride == 0) return;
  const uint64_t cr = chunk_rows(h.stride);
  Stage st(8 * std::min<uint64_t>(cr, h.rows) * h.stride, device);
  int slot = 0;
  for (int w = 0; w < W; ++w)
    for (uint64_t r0 = 0; r0 < h.rows; r0 += cr) {
      const uint64_t nr = std::min<uint64_t>(cr, h.rows - r0);
      st.wait(slot);
      double* b = st.buf[slot];
      if (std::fread(b, 8, nr * h.stride, F.f) != nr * h.stride) io_fail(path, "truncated");
      if (!pads_zero(b, nr, h.cols, h.stride)) io_fail(path, "nonzero padding");
      double* d = dst + w * plane + r0 * ld;
      if (device) {
        ck(cudaMemcpy2DAsync(d, ld * 8, b, h.stride * 8, h.cols * 8, nr, cudaMemcpyHostToDevice, s),
           "H2D MPFM chunk");
        ck(cudaEventRecord(st.ev[slot], s), "event");
      } else {
        for (uint64_t i = 0; i < nr; ++i) std::memcpy(d + i * ld, b + i * h.stride, h.cols * 8);
      }
      slot ^= 1;
    }
  if (device) ck(cudaStreamSynchronize(s), "MPFM load");
}

void mpfm_save(const char* cpath, int W, const double* src, uint64_t rows, uint64_t cols,
               uint64_t ld, uint64_t plane, bool device, cudaStream_t s) {
  const std::string path = cpath ? cpath : "";
  if (ld < cols) fail(MPFK_EINVAL, "mpfk: leading dimension too small");
  File F;
  F.f = std::fopen(path.c_str(), "wb");
  if (!F.f) io_fail(path, "cannot open for writing");
  write_header(F.f, path, W, rows, cols);
  const uint64_t stride = pad4(cols);
  if (rows && stride) {
    const uint64_t cr = chunk_rows(stride);
    Stage st(8 * std::min<uint64_t>(cr, rows) * stride, device);
    for (int i = 0; i < 2; ++i) std::memset(st.buf[i], 0, 8 * std::min<uint64_t>(cr, rows) * stride);
    // chunk list (plane, first row); download chunk i+1 while writing chunk i
    std::vector<std::pair<int, uint64_t>> chunks;
    for (int w = 0; w < W; ++w)
      for (uint64_t r0 = 0; r0 < rows; r0 += cr) chunks.emplace_back(w, r0);
    auto fetch = [&](size_t c, int slot) {
      const int w = chunks[c].first;
      const uint64_t r0 = chunks[c].second, nr = std::min<uint64_t>(cr, rows - r0);
      const double* p = src + w * plane + r0 * ld;
      if (device) {
        ck(cudaMemcpy2DAsync(st.buf[slot], stride * 8, p, ld * 8, cols * 8, nr, cudaMemcpyDeviceToHost, s),
           "D2H MPFM chunk");
        ck(cudaEventRecord(st.ev[slot], s), "event");
      } else {
        for (uint64_t i = 0; i < nr; ++i) std::memcpy(st.buf[slot] + i * stride, p + i * ld, cols * 8);
      }
    };
    fetch(0, 0);
    for (size_t c = 0; c < chunks.size(); ++c) {
      const int slot = (int)(c & 1);
      if (c + 1 < chunks.size()) fetch(c + 1, slot ^ 1);
      st.wait(slot);
      const uint64_t nr = std::min<uint64_t>(cr, rows - chunks[c].second);
      if (std::fwrite(st.buf[slot], 8, nr * stride, F.f) != nr * stride) io_fail(path, "write failed");
    }
  }
  if (std::fflush(F.f) != 0) io_fail(path, "write failed");
  if (std::fclose(F.f) != 0) {
    F.f = nullptr;
    io_fail(path, "write failed");
  }
  F.f = nullptr;
}
