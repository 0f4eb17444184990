// Stable LSD radix sort of u32 keys (with optional u32 values), 4 passes of
// 8 bits: the candidate sort behind SeavSketch.restore (candidates ordered
// by ip, short_sketch.py:398-408) and the finalize's fallback for key sets
// too clustered for its bucket sort.  Library-free (no CUB).
//
// Per pass: (1) every block counts the digits of its contiguous tile into
// hist[digit][block]; (2) one block turns hist into exclusive offsets
// (digit-major, so equal digits keep block order = stability across
// blocks); (3) every block re-reads its tile in 1,024-key chunks and ranks
// each key among equal digits -- lanes by __match_any_sync, warps by a
// per-chunk scan of per-warp digit counts -- so equal keys keep their
// input order within the block as well.
#include <cuda_runtime.h>
#include "sspd_common.cuh"
#include "launch.cuh"

namespace sspd {
namespace radix {

constexpr uint32_t kThreads = 1024;
constexpr uint32_t kWarps = kThreads / 32;
constexpr uint32_t kMaxBlocks = 1024;

struct Geo {
  uint32_t blocks;
  uint64_t tile;  // keys per block (multiple of kThreads)
};

static Geo geometry(uint64_t n) {
  Geo g;
  uint64_t b = (n + 4095) / 4096;
  if (b < 1) b = 1;
  if (b > kMaxBlocks) b = kMaxBlocks;
  g.tile = ((n + b - 1) / b + kThreads - 1) / kThreads * kThreads;
  g.blocks = (uint32_t)((n + g.tile - 1) / g.tile);
  if (g.blocks < 1) g.blocks = 1;
  return g;
}

__global__ void __launch_bounds__(kThreads) hist_kernel(const uint32_t* __restrict__ keys, uint64_t n, uint64_t tile,
                                                         uint32_t shift, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  for (uint32_t i = threadIdx.x; i < 256; i += kThreads) h[i] = 0;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * tile, hi = min(n, lo + tile);
  for (uint64_t j = lo + threadIdx.x; j < hi; j += kThreads) atomicAdd(&h[(keys[j] >> shift) & 255u], 1u);
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < 256; d += kThreads) hist[(uint64_t)d * gridDim.x + blockIdx.x] = h[d];
}

// exclusive scan of m = 256 * blocks counts, in place (one block)
__global__ void __launch_bounds__(kThreads) scan_kernel(uint32_t* __restrict__ hist, uint32_t m) {
  __shared__ uint32_t ws[kWarps];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t per = (m + kThreads - 1) / kThreads;
  const uint32_t lo = min(m, tid * per), hi = min(m, lo + per);
  uint32_t sum = 0;
  for (uint32_t i = lo; i < hi; ++i) sum += hist[i];
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  if (lane == 31) ws[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const uint32_t v = ws[lane];
    uint32_t wi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= (uint32_t)o) wi += y;
    }
    ws[lane] = wi - v;
  }
  __syncthreads();
  uint32_t run = ws[wid] + incl - sum;
  for (uint32_t i = lo; i < hi; ++i) {
    const uint32_t c = hist[i];
    hist[i] = run;
    run += c;
  }
}

template <bool kVals>
__global__ void __launch_bounds__(kThreads) scatter_kernel(const uint32_t* __restrict__ keys,
                                                           const uint32_t* __restrict__ vals, uint64_t n,
                                                           uint64_t tile, uint32_t shift,
                                                           const uint32_t* __restrict__ offs,
                                                           uint32_t* __restrict__ keys_out,
                                                           uint32_t* __restrict__ vals_out) {
  __shared__ uint32_t run[256];              // next output position per digit (this block)
  __shared__ uint16_t wcnt[kWarps][256];     // per-warp digit counts of the chunk, then prefixes
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (uint32_t d = tid; d < 256; d += kThreads) run[d] = offs[(uint64_t)d * gridDim.x + blockIdx.x];
  const uint64_t lo = (uint64_t)blockIdx.x * tile, hi = min(n, lo + tile);
  for (uint64_t base = lo; base < hi; base += kThreads) {
    for (uint32_t i = tid; i < kWarps * 256; i += kThreads) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint64_t j = base + tid;
    const bool live = j < hi;
    const uint32_t key = live ? keys[j] : 0u;
    const uint32_t d = live ? (key >> shift) & 255u : 256u;  // 256: a tail lane, matches no live digit
    const uint32_t same = __match_any_sync(0xFFFFFFFFu, d);
    const uint32_t rank_in_warp = __popc(same & ((1u << lane) - 1u));
    if (live && rank_in_warp == 0) wcnt[wid][d] = (uint16_t)__popc(same);
    __syncthreads();
    // per digit: exclusive prefix over the warps (in warp order); the
    // chunk's total is added to run[] once every key has been placed
    uint32_t total = 0;
    if (tid < 256) {
#pragma unroll 4
      for (uint32_t w = 0; w < kWarps; ++w) {
        const uint32_t c = wcnt[w][tid];
        wcnt[w][tid] = (uint16_t)total;
        total += c;
      }
    }
    __syncthreads();
    if (live) {
      const uint32_t pos = run[d] + wcnt[wid][d] + rank_in_warp;
      keys_out[pos] = key;
      if (kVals) vals_out[pos] = vals[j];
    }
    __syncthreads();
    if (tid < 256) run[tid] += total;
    __syncthreads();
  }
}

}  // namespace radix

// Scratch bytes of radix_sort_u32 for n keys (with values or not).
size_t radix_sort_scratch(uint64_t n, bool with_vals) {
  const radix::Geo g = radix::geometry(n);
  const size_t vec = ((n * 4 + 255) / 256) * 256;
  return vec * (with_vals ? 2 : 1) + 4ull * 256 * g.blocks + 256;
}

// Sort keys[0..n) ascending (vals permuted alike when non-NULL), in place:
// four passes ping-pong through the scratch copies and end in keys/vals.
int radix_sort_u32(uint32_t* keys, uint32_t* vals, uint64_t n, void* scratch, size_t scratch_bytes,
                   cudaStream_t st) {
  if (n <= 1) return SSPD_OK;
  if (n >= (1ull << 32)) return SSPD_ERR_CONFIG;
  if (!scratch || scratch_bytes < radix_sort_scratch(n, vals != nullptr)) return SSPD_ERR_CAPACITY;
  const radix::Geo g = radix::geometry(n);
  const size_t vec = ((n * 4 + 255) / 256) * 256;
  uint8_t* s = static_cast<uint8_t*>(scratch);
  uint32_t* k_alt = reinterpret_cast<uint32_t*>(s);
  uint32_t* v_alt = vals ? reinterpret_cast<uint32_t*>(s + vec) : nullptr;
  uint32_t* hist = reinterpret_cast<uint32_t*>(s + vec * (vals ? 2 : 1));
  uint32_t *kin = keys, *vin = vals, *kout = k_alt, *vout = v_alt;
  for (uint32_t shift = 0; shift < 32; shift += 8) {
    radix::hist_kernel<<<g.blocks, radix::kThreads, 0, st>>>(kin, n, g.tile, shift, hist);
    radix::scan_kernel<<<1, radix::kThreads, 0, st>>>(hist, 256u * g.blocks);
    if (vals)
      radix::scatter_kernel<true><<<g.blocks, radix::kThreads, 0, st>>>(kin, vin, n, g.tile, shift, hist, kout, vout);
    else
      radix::scatter_kernel<false><<<g.blocks, radix::kThreads, 0, st>>>(kin, nullptr, n, g.tile, shift, hist, kout,
                                                                         nullptr);
    uint32_t* t = kin;
    kin = kout;
    kout = t;
    t = vin;
    vin = vout;
    vout = t;
  }
  return check_launch();  // 4 passes: the result is back in keys / vals
}

}  // namespace sspd
