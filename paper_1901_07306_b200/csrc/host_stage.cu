// Host-side staging of caller key arrays (no device code).
//
// DetectorState.process_batch from host memory -- the reference's own call
// pattern, 65,536-pair numpy buffers (cli.py:215-217, distributed.py:225-227)
// -- copies each batch into pinned staging memory before returning (the
// caller may reuse its buffer).  One thread copies pageable memory at
// ~8-10 GB/s, far below the 55 GB/s the H2D link then moves, so the copy is
// split across a small persistent worker pool: workers spin briefly between
// batches (the next call arrives within microseconds in a scan loop) and
// sleep on a condition variable when idle.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <pthread.h>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif
#include "sspd_common.cuh"

namespace sspd {
namespace host {

static inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
  __builtin_ia32_pause();
#endif
}

template <typename T>
static void narrow(const T* s, uint64_t n, uint32_t* d) {
  for (uint64_t i = 0; i < n; ++i) d[i] = (uint32_t)s[i];
}

// Streaming (non-temporal) copy of n u32 into the pinned staging buffer:
// the destination is only read again by the H2D DMA, so its lines skip the
// cache and the read-for-ownership a plain store pays (a plain memcpy moves
// 3 bytes of host memory traffic per byte copied, a streaming one 2).  The
// sfence orders the streaming stores before the pool reports the part done.
static bool g_nt = true;
static void copy_u32(uint32_t* d, const uint32_t* s, uint64_t n) {
#if defined(__x86_64__)
  if (g_nt) {
    uint64_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 15u)) d[i] = s[i], ++i;  // head to 16 B
    for (; i + 16 <= n; i += 16) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 4));
      const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 8));
      const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 12));
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 4), b);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 8), c);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 12), e);
    }
    for (; i < n; ++i) d[i] = s[i];
    _mm_sfence();
    return;
  }
#endif
  memcpy(d, s, n * 4);
}

static void pack(const void* src, uint64_t lo, uint64_t hi, uint32_t eb, uint32_t* dst) {
  const uint8_t* s = static_cast<const uint8_t*>(src) + lo * eb;
  switch (eb) {
    case 1: narrow(reinterpret_cast<const uint8_t*>(s), hi - lo, dst + lo); break;
    case 2: narrow(reinterpret_cast<const uint16_t*>(s), hi - lo, dst + lo); break;
    case 4: copy_u32(dst + lo, reinterpret_cast<const uint32_t*>(s), hi - lo); break;
    default: narrow(reinterpret_cast<const uint64_t*>(s), hi - lo, dst + lo); break;
  }
}

struct Job {
  const void* src[2];
  uint32_t* dst[2];
  uint32_t eb[2];
  uint64_t n;
};

class CopyPool;
static std::atomic<CopyPool*> g_pool{nullptr};
static std::mutex g_pool_mu;

// A forked child inherits the pool object but none of its threads: forget
// it there, so the child builds its own pool on first use instead of
// waiting forever for workers that do not exist.
static void forget_pool_in_child() { g_pool.store(nullptr, std::memory_order_relaxed); }

class CopyPool {
 public:
  static CopyPool& get() {
    CopyPool* p = g_pool.load(std::memory_order_acquire);
    if (p) return *p;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    p = g_pool.load(std::memory_order_relaxed);
    if (!p) {
      static bool atfork = (pthread_atfork(nullptr, nullptr, forget_pool_in_child), true);
      (void)atfork;
      p = new CopyPool();  // leaked on purpose: detached workers outlive static destructors
      g_pool.store(p, std::memory_order_release);
    }
    return *p;
  }

  int workers() const { return (int)nworkers_; }

  void run(const Job& job) {
    std::lock_guard<std::mutex> one_at_a_time(run_mu_);
    job_ = job;
    const int parts = (int)nworkers_ + 1;
    pending_.store((int)nworkers_, std::memory_order_relaxed);
    gen_.fetch_add(1, std::memory_order_release);
    if (sleepers_.load(std::memory_order_acquire) > 0) {
      std::lock_guard<std::mutex> lk(mu_);
      cv_.notify_all();
    }
    part(0, parts);
    while (pending_.load(std::memory_order_acquire) != 0) cpu_relax();
  }

 private:
  CopyPool() {
    unsigned hw = std::thread::hardware_concurrency();
    // every host thread up to 16 (measured on the 16-thread GPU host,
    // tools/dropin_probe.py: 8 threads 35-40 GB/s, 16 threads + streaming
    // stores 48.7 GB/s of pageable -> pinned copy)
    unsigned want = hw > 1 ? std::min(hw, 16u) : 1u;
    if (const char* e = getenv("SSPD_HOST_COPY_THREADS")) want = (unsigned)std::max(1, atoi(e));
    if (const char* e = getenv("SSPD_HOST_COPY_NT")) g_nt = atoi(e) != 0;
    nworkers_ = want - 1;  // the calling thread takes part 0
    for (unsigned i = 0; i < nworkers_; ++i) std::thread([this, i] { loop(i + 1); }).detach();
  }

  void part(int p, int parts) {
    const Job& j = job_;
    const uint64_t lo = j.n * (uint64_t)p / (uint64_t)parts, hi = j.n * (uint64_t)(p + 1) / (uint64_t)parts;
    if (hi <= lo) return;
    for (int a = 0; a < 2; ++a) pack(j.src[a], lo, hi, j.eb[a], j.dst[a]);
  }

  void loop(int id) {
    uint64_t seen = 0;  // workers start before the first job (generation 1)
    for (;;) {
      uint64_t g;
      auto t0 = std::chrono::steady_clock::now();
      unsigned spins = 0;
      while ((g = gen_.load(std::memory_order_acquire)) == seen) {
        cpu_relax();
        if ((++spins & 1023u) == 0 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(300)) {
          std::unique_lock<std::mutex> lk(mu_);
          sleepers_.fetch_add(1, std::memory_order_acq_rel);
          cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
          sleepers_.fetch_sub(1, std::memory_order_acq_rel);
          t0 = std::chrono::steady_clock::now();
        }
      }
      seen = g;
      part(id, (int)nworkers_ + 1);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }

  unsigned nworkers_ = 0;
  Job job_{};
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0};
  std::atomic<int> sleepers_{0};
  std::mutex mu_, run_mu_;
  std::condition_variable cv_;
};

}  // namespace host
}  // namespace sspd

using namespace sspd;

// Copy n (hip, oip) keys -- already range-checked (sspd_host_check_u32),
// of elem widths hbytes/obytes (1/2/4/8) -- into u32 staging arrays, on the
// worker pool for batches large enough to amortise the hand-off.
extern "C" int sspd_host_pack_pairs(const void* hips, const void* oips, uint64_t n, uint32_t hbytes,
                                    uint32_t obytes, uint32_t* dst_h, uint32_t* dst_o) {
  if (n == 0) return SSPD_OK;
  if (!hips || !oips || !dst_h || !dst_o) return SSPD_ERR_DATA;
  auto ok = [](uint32_t b) { return b == 1 || b == 2 || b == 4 || b == 8; };
  if (!ok(hbytes) || !ok(obytes)) return SSPD_ERR_CONFIG;
  host::Job job{{hips, oips}, {dst_h, dst_o}, {hbytes, obytes}, n};
  host::CopyPool& pool = host::CopyPool::get();
  if (n < (1u << 14) || pool.workers() == 0) {
    host::pack(hips, 0, n, hbytes, dst_h);
    host::pack(oips, 0, n, obytes, dst_o);
    return SSPD_OK;
  }
  pool.run(job);
  return SSPD_OK;
}

// Worker threads of the staging pool (+1 for the caller), for reporting.
extern "C" int sspd_host_copy_threads(void) { return host::CopyPool::get().workers() + 1; }
