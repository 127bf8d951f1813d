// staging.cu -- host<->device copies of caller memory that is not pinned.
//
// The drop-in call (tcmis::run_mis(const Graph &, ...)) hands the engine plain
// std::vector storage.  A cudaMemcpyAsync from pageable memory is staged by
// the driver through a small bounce buffer on one CPU thread and is
// synchronous: the 547 MB CSR upload of R-MAT s22 -- the whole cost of the
// drop-in call -- took 53 ms that way against 9.9 ms from pinned memory.
//
// Here every context owns a ring of kSlots pinned staging buffers and a pool
// of host threads.  Piece k of a copy is copied into slot k % kSlots by all
// threads at once (the calling thread takes a share) while the copy engine
// moves piece k-1 to the device on the context stream, so host memcpy and
// DMA overlap.  Measured on the 16-core host of the B200 box at s22: 53 ms
// driver-staged, 15.5 ms with 8 threads and 8 MB pieces (the host memcpy is
// then bound by the host's DRAM: the source read, the slot write and the
// DMA's read of the slot); one stream and large pieces beat per-thread
// streams with small cache-resident slots (22-37 ms: per-piece copy and event
// overheads).  Device-to-host copies into pageable memory (the MIS ids) run
// the same pipeline backwards.  Pinned / registered caller memory goes
// straight to the copy engine.
#include <emmintrin.h>
#include <pthread.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>  // hardware_concurrency
#include <vector>

#include "internal.cuh"

namespace tcmis_b200 {

namespace {

constexpr int kSlots = 4;
constexpr size_t kMinStaged = 2u << 20;   // smaller copies go straight to the driver
constexpr size_t kMinPart = 256u << 10;   // smallest per-thread share of a piece

// ordinary (write-allocate) 16-byte stores: the slot stays cache-resident for
// the copy engine's read (TCMIS_STAGE_COPY=cached); memcpy's large-copy path
// streams past the cache
void copy_cached(char *d, const char *s, size_t len) {
  size_t i = 0;
  for (; i + 64 <= len; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 48));
    _mm_storeu_si128(reinterpret_cast<__m128i *>(d + i), a);
    _mm_storeu_si128(reinterpret_cast<__m128i *>(d + i + 16), b);
    _mm_storeu_si128(reinterpret_cast<__m128i *>(d + i + 32), c);
    _mm_storeu_si128(reinterpret_cast<__m128i *>(d + i + 48), e);
  }
  if (i < len) std::memcpy(d + i, s + i, len - i);
}

// A fixed pool of host threads running one parallel copy at a time.  (POSIX
// threads: nvcc gives anonymous namespaces external linkage, so a
// std::thread instantiation over these types would be exported from the
// library next to the C-ABI.)
class CopyPool {
 public:
  CopyPool(int threads, bool cached) : cached_(cached) {
    args_.resize((size_t)threads);
    for (int i = 0; i < threads; ++i) {
      args_[i] = {this, i};
      pthread_t t;
      if (pthread_create(&t, nullptr, &CopyPool::entry, &args_[i]) == 0) th_.push_back(t);
    }
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (pthread_t t : th_) pthread_join(t, nullptr);
  }
  // dst[0, bytes) = src[0, bytes), split over the pool and the calling thread
  void copy(void *dst, const void *src, size_t bytes) {
    const int parts =
        (int)std::max<size_t>(1, std::min<size_t>(th_.size() + 1, bytes / kMinPart));
    if (parts == 1) {
      one(static_cast<char *>(dst), static_cast<const char *>(src), bytes);
      return;
    }
    const size_t per = (bytes + parts - 1) / parts;
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char *>(dst);
      src_ = static_cast<const char *>(src);
      bytes_ = bytes;
      per_ = per;
      parts_ = parts;
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    const size_t tail = (size_t)(parts - 1) * per;  // the caller's share
    one(dst_ + tail, src_ + tail, bytes - tail);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  struct Arg {
    CopyPool *self;
    int i;
  };
  static void *entry(void *p) {
    const Arg *a = static_cast<const Arg *>(p);
    a->self->loop(a->i);
    return nullptr;
  }
  void one(char *d, const char *s, size_t len) {
    if (cached_) copy_cached(d, s, len);
    else std::memcpy(d, s, len);
  }
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      char *dst;
      const char *src;
      size_t len = 0, off = 0;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (i >= parts_ - 1) continue;  // not needed for this copy
        dst = dst_;
        src = src_;
        off = (size_t)i * per_;
        len = std::min(per_, bytes_ - off);
      }
      one(dst + off, src + off, len);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  bool cached_;
  std::vector<Arg> args_;
  std::vector<pthread_t> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  bool stop_ = false;
  uint64_t gen_ = 0;
  char *dst_ = nullptr;
  const char *src_ = nullptr;
  size_t bytes_ = 0, per_ = 0;
  int parts_ = 0, pending_ = 0;
};

}  // namespace

struct Staging {
  size_t piece = 8u << 20;  // bytes per slot (TCMIS_STAGE_PIECE_KB)
  void *buf[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  bool used[kSlots] = {};
  int next = 0;
  CopyPool *pool = nullptr;
};

void free_staging(tcmis_ctx *ctx) {
  Staging *s = ctx->staging;
  if (!s) return;
  for (int i = 0; i < kSlots; ++i) {
    if (s->ev[i]) cudaEventSynchronize(s->ev[i]);
    if (s->buf[i]) cudaFreeHost(s->buf[i]);
    if (s->ev[i]) cudaEventDestroy(s->ev[i]);
  }
  delete s->pool;
  delete s;
  ctx->staging = nullptr;
}

bool host_pinned(const void *p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear: plain pageable memory on older drivers
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged ||
         a.type == cudaMemoryTypeDevice;
}

namespace {

int staging(tcmis_ctx *ctx, Staging **out) {
  if (!ctx->staging) {
    auto *s = new Staging();
    if (const char *env = std::getenv("TCMIS_STAGE_PIECE_KB"))
      s->piece = std::max<size_t>(256, std::strtoull(env, nullptr, 10)) << 10;
    for (int i = 0; i < kSlots; ++i) {
      if (cudaMallocHost(&s->buf[i], s->piece) != cudaSuccess ||
          cudaEventCreateWithFlags(&s->ev[i], cudaEventDisableTiming) != cudaSuccess) {
        ctx->staging = s;
        free_staging(ctx);
        return set_error(TCMIS_E_CUDA, "pinned staging buffers");
      }
    }
    int threads = (int)std::thread::hardware_concurrency() / 2;
    if (const char *env = std::getenv("TCMIS_STAGE_THREADS")) threads = std::atoi(env);
    threads = std::max(1, std::min(threads, 32));
    const char *mode = std::getenv("TCMIS_STAGE_COPY");
    s->pool = new CopyPool(threads - 1, mode && std::strcmp(mode, "cached") == 0);
    ctx->staging = s;
  }
  *out = ctx->staging;
  return 0;
}

}  // namespace

// Enqueue dst (device) <- src (host, any kind) on `st`.  A pageable source
// has been read completely when the call returns; the device side completes
// in stream order.
int h2d(tcmis_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t st) {
  if (!bytes) return 0;
  if (bytes < kMinStaged || host_pinned(src) || std::getenv("TCMIS_NO_STAGING")) {
    TCMIS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return 0;
  }
  Staging *s = nullptr;
  if (int rc = staging(ctx, &s)) return rc;
  TCMIS_RANGE("staged h2d");
  const char *from = static_cast<const char *>(src);
  char *to = static_cast<char *>(dst);
  for (size_t off = 0; off < bytes; off += s->piece) {
    const size_t len = std::min(s->piece, bytes - off);
    const int k = s->next;
    s->next = (s->next + 1) % kSlots;
    if (s->used[k]) TCMIS_CUDA(cudaEventSynchronize(s->ev[k]));  // its last DMA is done
    s->pool->copy(s->buf[k], from + off, len);
    TCMIS_CUDA(cudaMemcpyAsync(to + off, s->buf[k], len, cudaMemcpyHostToDevice, st));
    TCMIS_CUDA(cudaEventRecord(s->ev[k], st));
    s->used[k] = true;
  }
  return 0;
}

// dst (host, any kind) <- src (device, written in `st` order); complete when
// the call returns.
int d2h(tcmis_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t st) {
  if (!bytes) return 0;
  if (bytes < kMinStaged || host_pinned(dst) || std::getenv("TCMIS_NO_STAGING")) {
    TCMIS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    TCMIS_CUDA(cudaStreamSynchronize(st));
    return 0;
  }
  Staging *s = nullptr;
  if (int rc = staging(ctx, &s)) return rc;
  TCMIS_RANGE("staged d2h");
  const char *from = static_cast<const char *>(src);
  char *to = static_cast<char *>(dst);
  const size_t pieces = (bytes + s->piece - 1) / s->piece;
  // slot j holds pieces j, j + kSlots, ...: DMAs run kSlots pieces ahead of
  // the host's copy-out (the ring is free: every earlier DMA from it is
  // behind these on the same stream)
  auto issue = [&](size_t p) -> int {
    const size_t off = p * s->piece, len = std::min(s->piece, bytes - off);
    const int k = (int)(p % kSlots);
    TCMIS_CUDA(cudaMemcpyAsync(s->buf[k], from + off, len, cudaMemcpyDeviceToHost, st));
    TCMIS_CUDA(cudaEventRecord(s->ev[k], st));
    s->used[k] = true;
    return 0;
  };
  for (size_t p = 0; p < pieces && p < (size_t)kSlots; ++p)
    if (int rc = issue(p)) return rc;
  for (size_t p = 0; p < pieces; ++p) {
    const int k = (int)(p % kSlots);
    const size_t off = p * s->piece, len = std::min(s->piece, bytes - off);
    TCMIS_CUDA(cudaEventSynchronize(s->ev[k]));
    s->pool->copy(to + off, s->buf[k], len);
    if (p + kSlots < pieces)
      if (int rc = issue(p + kSlots)) return rc;
  }
  s->next = 0;
  return 0;
}

}  // namespace tcmis_b200
