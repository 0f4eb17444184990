// K1 scan_discrete and K2 scan_sliding: the per-packet hot loop.
//
// Reference semantics (one packet = one (hip, oip) pair):
//   LdcaSketch.update_batch  long_sketch.py:125-135
//     b   = H3(oip) % k
//     c_i = LH_i(hip) % lc                     for i < LR
//     data[i, c_i, b>>3] |= 1 << (b & 7)       == flat bit (i*lc + c_i)*k + b
//   SeavSketch.update_batch  short_sketch.py:300-318
//     if lsb(H1(oip) & 0xFFFFFFFF) >= tau:
//        bit = 1 << (H2(oip) % g); rp = hip & (2^r-1); lp = (hip>>r) & (2^w-1)
//        rows[i][rp, index_of(i, lp)] |= bit   for i < SR
//   SlidingDetector.observe_batch sliding.py:156-185 stamps the same slots
//   (one slot per sketch bit) with `now & mask` (plain store, sliding.py:77-79).
//
// B200 mapping: the input is streamed once from HBM with 16-byte
// evict-first loads (4 packets per thread per trip); every sketch bit-set
// is a fire-and-forget `red.relaxed.gpu.global.or.b32` into the
// L2-resident bit arrays (idempotent OR == the paper's "no data conflict"),
// and every sliding stamp is a plain store (all writers of one slice store
// the same value, so no atomic is needed and none would be correct across
// the wrap -- see DESIGN.md).
#include <cooperative_groups.h>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sspd_common.cuh"
#include "launch.cuh"

namespace cg = cooperative_groups;

namespace sspd {

__device__ __forceinline__ void red_or(uint32_t* addr, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// ---------------------------------------------------------------- sinks
struct DiscreteSink {
  uint32_t* seav;  // word view of the SEAV payload (may be null)
  uint32_t* ldca;  // word view of the LDCA payload (may be null)
  __device__ __forceinline__ void le(uint64_t bitpos) const {
    red_or(ldca + (bitpos >> 5), 1u << (bitpos & 31));
  }
  // register byte offset + bit within the (little-endian) register
  __device__ __forceinline__ void se(uint64_t reg_byte, uint32_t bit) const {
    uint64_t abs_bit = reg_byte * 8 + bit;
    red_or(seav + (abs_bit >> 5), 1u << (abs_bit & 31));
  }
};

template <typename T>
struct SlidingSink {
  T* pool;
  T now;
  __device__ __forceinline__ void le_slot(uint64_t slot) const { pool[slot] = now; }
  __device__ __forceinline__ void se_slot(uint64_t slot) const { pool[slot] = now; }
};

// ------------------------------------------------------------ per packet
template <bool kSeav, bool kLdca>
__device__ __forceinline__ void packet_discrete(uint32_t hip, uint32_t oip, const sspd_params& p,
                                                const DiscreteSink& s, uint32_t tmask) {
  if (kLdca) {
    const uint64_t b = hash_range(oip, p.seed_h3, p.div_k);
    const uint64_t k = p.k;
    uint64_t cell = 0;  // i * lc
#pragma unroll 8
    for (uint32_t i = 0; i < p.lr; ++i) {
      const uint64_t c = hash_range(hip, p.seed_lh[i], p.div_lc);
      s.le((cell + c) * k + b);
      cell += p.lc;
    }
  }
  if (kSeav) {
    if (sampled(oip, p.seed_h1, tmask)) {
      const uint32_t bit = (uint32_t)hash_range(oip, p.seed_h2, p.div_g);
      const uint64_t rp = hip & ((1u << p.r) - 1u);
      const uint64_t lp = ((uint64_t)hip >> p.r) & ((1ull << p.lp_bits) - 1ull);
      for (uint32_t i = 0; i < p.sr; ++i) {
        const uint32_t col = index_of(lp, p.isb[i], p.ibn[i], p.lp_bits);
        s.se(p.seav_row_off[i] + (rp * p.sc[i] + col) * p.reg_bytes, bit);
      }
    }
  }
}

template <typename T>
__device__ __forceinline__ void packet_sliding(uint32_t hip, uint32_t oip, const sspd_params& p,
                                               const SlidingSink<T>& s, uint32_t tmask) {
  if (sampled(oip, p.seed_h1, tmask)) {
    const uint64_t bit = hash_range(oip, p.seed_h2, p.div_g);
    const uint64_t rp = hip & ((1u << p.r) - 1u);
    const uint64_t lp = ((uint64_t)hip >> p.r) & ((1ull << p.lp_bits) - 1ull);
    for (uint32_t i = 0; i < p.sr; ++i) {
      const uint32_t col = index_of(lp, p.isb[i], p.ibn[i], p.lp_bits);
      s.se_slot(p.slot_row_base[i] + (rp * p.sc[i] + col) * p.g + bit);
    }
  }
  const uint64_t b = hash_range(oip, p.seed_h3, p.div_k);
  const uint64_t k = p.k;
  uint64_t cell = 0;
#pragma unroll 8
  for (uint32_t i = 0; i < p.lr; ++i) {
    const uint64_t c = hash_range(hip, p.seed_lh[i], p.div_lc);
    s.le_slot(p.slot_ldca_base + (cell + c) * k + b);
    cell += p.lc;
  }
}

// -------------------------------------------------------------- kernels
// Grid-stride over 16-byte quads of hips/oips (both 16-byte aligned, checked
// by the host); the scalar head/tail is handled by the same kernel.
template <bool kSeav, bool kLdca>
__global__ void __launch_bounds__(256) scan_discrete_kernel(const uint32_t* __restrict__ hips,
                                                            const uint32_t* __restrict__ oips,
                                                            uint64_t n, const __grid_constant__ sspd_params p,
                                                            uint32_t* seav, uint32_t* ldca) {
  const DiscreteSink s{seav, ldca};
  const uint32_t tmask = tau_mask(p.tau);
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t nq = n >> 2;
  const uint4* hq = reinterpret_cast<const uint4*>(hips);
  const uint4* oq = reinterpret_cast<const uint4*>(oips);
  for (uint64_t q = tid; q < nq; q += stride) {
    const uint4 h = ld_stream(hq + q);
    const uint4 o = ld_stream(oq + q);
    packet_discrete<kSeav, kLdca>(h.x, o.x, p, s, tmask);
    packet_discrete<kSeav, kLdca>(h.y, o.y, p, s, tmask);
    packet_discrete<kSeav, kLdca>(h.z, o.z, p, s, tmask);
    packet_discrete<kSeav, kLdca>(h.w, o.w, p, s, tmask);
  }
  for (uint64_t j = (nq << 2) + tid; j < n; j += stride)
    packet_discrete<kSeav, kLdca>(hips[j], oips[j], p, s, tmask);
}

// Unaligned inputs (a numpy view at an odd offset): scalar loads only.
template <bool kSeav, bool kLdca>
__global__ void __launch_bounds__(256) scan_discrete_scalar_kernel(const uint32_t* __restrict__ hips,
                                                                   const uint32_t* __restrict__ oips,
                                                                   uint64_t n, const __grid_constant__ sspd_params p,
                                                                   uint32_t* seav, uint32_t* ldca) {
  const DiscreteSink s{seav, ldca};
  const uint32_t tmask = tau_mask(p.tau);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride)
    packet_discrete<kSeav, kLdca>(hips[j], oips[j], p, s, tmask);
}

template <typename T>
__global__ void __launch_bounds__(256) scan_sliding_kernel(const uint32_t* __restrict__ hips,
                                                           const uint32_t* __restrict__ oips, uint64_t n,
                                                           const __grid_constant__ sspd_params p, T* pool,
                                                           T now) {
  const SlidingSink<T> s{pool, now};
  const uint32_t tmask = tau_mask(p.tau);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride)
    packet_sliding<T>(hips[j], oips[j], p, s, tmask);
}

// K2 fast path: u16 stamps, k and lc powers of two, < 2^32 slots, 16-byte
// aligned inputs (config 4).  Four packets per thread from one 16-byte load
// per array, 32-bit slot math (the row modulo is a mask), and the LDCA stamp
// stores carry an L2 evict_last policy for a fraction of the addresses:
// the ~134 MB LDCA stamp region is the re-written working set (8 stores per
// packet), while the input stream and the sparse SEAV stamps are not, so
// keeping most of it L2-resident turns partial-sector misses into hits.
__device__ __forceinline__ void st_u16_hint(uint16_t* addr, uint16_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b16 [%0], %1, %2;" ::"l"(addr), "h"(v), "l"(pol) : "memory");
}

// Incremental SEAV view (optional, `tr.view != nullptr`): every SEAV stamp
// also sets its bit in the maintained active-bit view and appends the slot
// to a ring log, so advance_slice can clear exactly the bits whose slice
// expires (sspd_seav_advance) instead of re-reading the 268 MB SEAV stamp
// region at every detect.
struct SeavTracker {
  uint32_t* view;                // SEAV view as words (seav payload layout)
  uint32_t* log;                 // ring of SEAV slot indexes
  unsigned long long* log_head;  // entries ever appended
  uint32_t log_mask;             // ring size - 1
};

// The log positions are reserved per BLOCK: a sampled packet takes a slot of
// a shared-memory staging area (shared atomic), and the block writes its
// staged entries out with ONE atomic on the global log head when half full
// and at its end.  (Reserving per warp from the single global counter
// serialised every sampled packet at one L2 slice: ~14 k dependent atomics
// per config-4 slice, 80 % of K2's stall samples.)  The ring's order within
// a slice is irrelevant to sspd_seav_advance; only the head per slice is.
constexpr uint32_t kLogPk = 256;  // packets staged per block (x SR entries of dynamic smem)
struct LogStage {
  uint32_t np;
  unsigned long long base;
};

// one sampled packet: where its SR log entries go (staged or, when the
// staging area is full, straight to the ring)
struct LogDst {
  uint32_t* ent;               // staged entries, or nullptr
  unsigned long long base;     // ring position otherwise
};

__device__ __forceinline__ LogDst log_reserve(LogStage* ls, uint32_t* lbuf, const SeavTracker& tr, uint32_t sr) {
  const uint32_t pk = atomicAdd(&ls->np, 1u);
  if (pk < kLogPk) return {lbuf + pk * sr, 0ull};
  return {nullptr, atomicAdd(tr.log_head, (unsigned long long)sr)};
}

__device__ __forceinline__ void log_put(const LogDst& d, const SeavTracker& tr, uint32_t i, uint32_t slot) {
  if (d.ent)
    d.ent[i] = slot;
  else
    tr.log[(d.base + i) & tr.log_mask] = slot;
}

// whole block (uniform call): write the staged entries out once at least
// `thresh` packets are staged
__device__ __forceinline__ void log_flush(LogStage* ls, const uint32_t* lbuf, const SeavTracker& tr, uint32_t sr,
                                          uint32_t thresh) {
  __syncthreads();
  const uint32_t np = min(ls->np, kLogPk);
  __syncthreads();
  if (np == 0 || np < thresh) return;
  if (threadIdx.x == 0) ls->base = atomicAdd(tr.log_head, (unsigned long long)np * sr);
  __syncthreads();
  const unsigned long long base = ls->base;
  for (uint32_t i = threadIdx.x; i < np * sr; i += blockDim.x) tr.log[(base + i) & tr.log_mask] = lbuf[i];
  __syncthreads();
  if (threadIdx.x == 0) ls->np = 0;
}

// Deferred LDCA stamps (optional, `dirty != nullptr`): instead of storing
// `now` into the 134 MB LDCA stamp region (8 random 2-byte stores per
// packet, most of them DRAM read-modify-writes), the scan sets the slot's
// bit in an LDCA-shaped dirty bitmap (8 MiB, L2-resident) with a `red.or`;
// sspd_ldca_fold later writes `now` into every dirty slot in one coalesced
// pass (and can emit the active-bit view in the same pass).  Exact: every
// stamp written during one slice is the same `now`, and the host folds
// before the slice changes or the stamps are read.
template <bool kTrack, bool kDefer>
__global__ void __launch_bounds__(256) scan_sliding_u16_fast_kernel(const uint32_t* __restrict__ hips,
                                                                    const uint32_t* __restrict__ oips, uint64_t n,
                                                                    const __grid_constant__ sspd_params p,
                                                                    uint16_t* pool, uint16_t now, float l2_frac,
                                                                    SeavTracker tr, uint32_t* dirty) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, %1;" : "=l"(pol) : "f"(l2_frac));
  const uint32_t tmask = tau_mask(p.tau);
  const uint32_t k_mask = p.k - 1, lc_mask = p.lc - 1;
  const uint32_t log2k = 31 - __clz(p.k);
  uint16_t* const lpool = pool + p.slot_ldca_base;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // hips/oips share their misalignment (host check): peel the scalar head
  const uint64_t head = min(n, (uint64_t)((16u - (reinterpret_cast<uintptr_t>(hips) & 15u)) & 15u) >> 2);
  const uint64_t nq = (n - head) >> 2;
  const uint4* hq = reinterpret_cast<const uint4*>(hips + head);
  const uint4* oq = reinterpret_cast<const uint4*>(oips + head);
  extern __shared__ uint32_t lbuf[];  // kTrack: kLogPk * SR staged log entries
  __shared__ LogStage ls;
  if (kTrack) {
    if (threadIdx.x == 0) ls.np = 0;
    __syncthreads();
  }
  auto one = [&](uint32_t hip, uint32_t oip) {
    if (sampled(oip, p.seed_h1, tmask)) {
      const uint32_t bit = (uint32_t)hash_range(oip, p.seed_h2, p.div_g);
      const uint64_t rp = hip & ((1u << p.r) - 1u);
      const uint64_t lp = ((uint64_t)hip >> p.r) & ((1ull << p.lp_bits) - 1ull);
      LogDst d{nullptr, 0ull};
      if (kTrack) d = log_reserve(&ls, lbuf, tr, p.sr);
      for (uint32_t i = 0; i < p.sr; ++i) {
        const uint32_t col = index_of(lp, p.isb[i], p.ibn[i], p.lp_bits);
        const uint64_t reg = rp * p.sc[i] + col;
        const uint64_t slot = p.slot_row_base[i] + reg * p.g + bit;
        pool[slot] = now;
        if (kTrack) {
          const uint64_t vbit = (p.seav_row_off[i] + reg * p.reg_bytes) * 8 + bit;
          atomicOr(tr.view + (vbit >> 5), 1u << (vbit & 31));
          log_put(d, tr, i, (uint32_t)slot);
        }
      }
    }
    const uint32_t b = (uint32_t)mix64(oip ^ p.seed_h3) & k_mask;
    uint32_t cell = 0;
#pragma unroll 8
    for (uint32_t i = 0; i < p.lr; ++i) {
      const uint32_t c = (uint32_t)mix64(hip ^ p.seed_lh[i]) & lc_mask;
      const uint32_t slot = ((cell + c) << log2k) | b;
      if (kDefer)
        red_or(dirty + (slot >> 5), 1u << (slot & 31));
      else
        st_u16_hint(lpool + slot, now, pol);
      cell += p.lc;
    }
  };
  // block-uniform trip count (the log flush is a block barrier)
  for (uint64_t qb = tid - threadIdx.x; qb < nq; qb += stride) {
    const uint64_t q = qb + threadIdx.x;
    if (q < nq) {
      const uint4 h = ld_stream(hq + q);
      const uint4 o = ld_stream(oq + q);
      one(h.x, o.x);
      one(h.y, o.y);
      one(h.z, o.z);
      one(h.w, o.w);
    }
    if (kTrack) log_flush(&ls, lbuf, tr, p.sr, kLogPk / 2);
  }
  if (tid < head) one(hips[tid], oips[tid]);
  for (uint64_t j = head + (nq << 2) + tid; j < n; j += stride) one(hips[j], oips[j]);
  if (kTrack) log_flush(&ls, lbuf, tr, p.sr, 1);
}

// K2 for u16 stamps when the fast path does not apply (k or lc not a power
// of two, or hips/oips misaligned relative to each other): scalar loads and
// the exact 64-bit modulo, with the same optional SEAV tracking and deferred
// LDCA stamps as the fast kernel (dirty bit = the LDCA bit index
// (i*lc + c)*k + b), so every u16 scan honours the caller's deferred state.
template <bool kTrack, bool kDefer>
__global__ void __launch_bounds__(256) scan_sliding_u16_generic_kernel(const uint32_t* __restrict__ hips,
                                                                       const uint32_t* __restrict__ oips, uint64_t n,
                                                                       const __grid_constant__ sspd_params p,
                                                                       uint16_t* pool, uint16_t now, SeavTracker tr,
                                                                       uint32_t* dirty) {
  const uint32_t tmask = tau_mask(p.tau);
  uint16_t* const lpool = pool + p.slot_ldca_base;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  extern __shared__ uint32_t lbuf[];  // kTrack: kLogPk * SR staged log entries
  __shared__ LogStage ls;
  if (kTrack) {
    if (threadIdx.x == 0) ls.np = 0;
    __syncthreads();
  }
  // block-uniform trip count (the log flush is a block barrier)
  for (uint64_t jb = (uint64_t)blockIdx.x * blockDim.x; jb < n; jb += stride) {
    const uint64_t j = jb + threadIdx.x;
    if (kTrack) log_flush(&ls, lbuf, tr, p.sr, kLogPk / 2);
    if (j >= n) continue;
    const uint32_t hip = hips[j], oip = oips[j];
    if (sampled(oip, p.seed_h1, tmask)) {
      const uint32_t bit = (uint32_t)hash_range(oip, p.seed_h2, p.div_g);
      const uint64_t rp = hip & ((1u << p.r) - 1u);
      const uint64_t lp = ((uint64_t)hip >> p.r) & ((1ull << p.lp_bits) - 1ull);
      LogDst d{nullptr, 0ull};
      if (kTrack) d = log_reserve(&ls, lbuf, tr, p.sr);
      for (uint32_t i = 0; i < p.sr; ++i) {
        const uint32_t col = index_of(lp, p.isb[i], p.ibn[i], p.lp_bits);
        const uint64_t reg = rp * p.sc[i] + col;
        const uint64_t slot = p.slot_row_base[i] + reg * p.g + bit;
        pool[slot] = now;
        if (kTrack) {
          const uint64_t vbit = (p.seav_row_off[i] + reg * p.reg_bytes) * 8 + bit;
          atomicOr(tr.view + (vbit >> 5), 1u << (vbit & 31));
          log_put(d, tr, i, (uint32_t)slot);
        }
      }
    }
    const uint64_t b = hash_range(oip, p.seed_h3, p.div_k);
    const uint64_t k = p.k;
    uint64_t cell = 0;
    for (uint32_t i = 0; i < p.lr; ++i) {
      const uint64_t c = hash_range(hip, p.seed_lh[i], p.div_lc);
      const uint64_t slot = (cell + c) * k + b;
      if (kDefer)
        red_or(dirty + (slot >> 5), 1u << (slot & 31));
      else
        lpool[slot] = now;
      cell += p.lc;
    }
  }
  if (kTrack) log_flush(&ls, lbuf, tr, p.sr, 1);
}

template <bool S, bool L>
static int launch_discrete(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params& p,
                           uint8_t* seav, uint8_t* ldca, cudaStream_t st) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(hips) | reinterpret_cast<uintptr_t>(oips)) & 15u) == 0;
  if (aligned) {
    const int grid = grid_for(scan_discrete_kernel<S, L>, 256, (n + 3) / 4);
    scan_discrete_kernel<S, L><<<grid, 256, 0, st>>>(hips, oips, n, p, reinterpret_cast<uint32_t*>(seav),
                                                     reinterpret_cast<uint32_t*>(ldca));
  } else {
    const int grid = grid_for(scan_discrete_scalar_kernel<S, L>, 256, n);
    scan_discrete_scalar_kernel<S, L><<<grid, 256, 0, st>>>(hips, oips, n, p, reinterpret_cast<uint32_t*>(seav),
                                                            reinterpret_cast<uint32_t*>(ldca));
  }
  return check_launch();
}

}  // namespace sspd

using namespace sspd;

extern "C" int sspd_scan_discrete(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p,
                                  uint8_t* seav, uint8_t* ldca, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (n == 0 || (!seav && !ldca)) return SSPD_OK;
  if (!hips || !oips) return SSPD_ERR_DATA;
  if ((reinterpret_cast<uintptr_t>(seav) | reinterpret_cast<uintptr_t>(ldca)) & 3u) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (seav && ldca) return launch_discrete<true, true>(hips, oips, n, *p, seav, ldca, st);
  if (seav) return launch_discrete<true, false>(hips, oips, n, *p, seav, ldca, st);
  return launch_discrete<false, true>(hips, oips, n, *p, seav, ldca, st);
}

static int scan_sliding_impl(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p,
                             void* pool, uint32_t ts_bytes, uint64_t now_wrapped, uint32_t max_blocks_per_sm,
                             SeavTracker tracker, uint32_t* dirty, void* stream, bool seav_only = false);

extern "C" int sspd_scan_sliding_capped(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                        const sspd_params* p, void* pool, uint32_t ts_bytes, uint64_t now_wrapped,
                                        uint32_t max_blocks_per_sm, void* stream) {
  return scan_sliding_impl(hips, oips, n, p, pool, ts_bytes, now_wrapped, max_blocks_per_sm,
                           SeavTracker{nullptr, nullptr, nullptr, 0u}, nullptr, stream);
}

extern "C" int sspd_scan_sliding_tracked(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                         const sspd_params* p, void* pool, uint32_t ts_bytes, uint64_t now_wrapped,
                                         uint32_t max_blocks_per_sm, uint8_t* seav_view, uint32_t* log,
                                         uint64_t log_entries, unsigned long long* log_head, void* stream) {
  if (!seav_view || !log || !log_head || log_entries == 0 || (log_entries & (log_entries - 1)) ||
      log_entries > (1ull << 32) || (reinterpret_cast<uintptr_t>(seav_view) & 3u))
    return SSPD_ERR_DATA;
  return scan_sliding_impl(hips, oips, n, p, pool, ts_bytes, now_wrapped, max_blocks_per_sm,
                           SeavTracker{reinterpret_cast<uint32_t*>(seav_view), log, log_head,
                                       (uint32_t)(log_entries - 1)},
                           nullptr, stream);
}

// Tracked (optional: seav_view may be null) scan with deferred LDCA stamps
// (optional: ldca_dirty may be null).  u16 stamps only; when the fast path
// does not apply (geometry, alignment) the generic u16 kernel keeps the same
// tracked / deferred semantics (the ring of dirty bitmaps depends on it).
extern "C" int sspd_scan_sliding_deferred(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                          const sspd_params* p, void* pool, uint32_t ts_bytes, uint64_t now_wrapped,
                                          uint32_t max_blocks_per_sm, uint8_t* seav_view, uint32_t* log,
                                          uint64_t log_entries, unsigned long long* log_head, uint32_t* ldca_dirty,
                                          void* stream) {
  SeavTracker tr{nullptr, nullptr, nullptr, 0u};
  if (seav_view) {
    if (!log || !log_head || log_entries == 0 || (log_entries & (log_entries - 1)) || log_entries > (1ull << 32) ||
        (reinterpret_cast<uintptr_t>(seav_view) & 3u))
      return SSPD_ERR_DATA;
    tr = SeavTracker{reinterpret_cast<uint32_t*>(seav_view), log, log_head, (uint32_t)(log_entries - 1)};
  }
  if (ldca_dirty && (reinterpret_cast<uintptr_t>(ldca_dirty) & 3u)) return SSPD_ERR_DATA;
  return scan_sliding_impl(hips, oips, n, p, pool, ts_bytes, now_wrapped, max_blocks_per_sm, tr, ldca_dirty, stream);
}

// SEAV half of the deferred scan: SEAV stamps (+ optional tracking) only.
// The LDCA half of the same packets goes to the slice's dirty bitmap through
// the partitioned scan (sspd_scan_partitioned with seav = NULL, ldca = the
// bitmap) -- together exactly sspd_scan_sliding_deferred.
extern "C" int sspd_scan_sliding_seav(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p,
                                      void* pool, uint32_t ts_bytes, uint64_t now_wrapped,
                                      uint32_t max_blocks_per_sm, uint8_t* seav_view, uint32_t* log,
                                      uint64_t log_entries, unsigned long long* log_head, void* stream) {
  SeavTracker tr{nullptr, nullptr, nullptr, 0u};
  if (seav_view) {
    if (!log || !log_head || log_entries == 0 || (log_entries & (log_entries - 1)) || log_entries > (1ull << 32) ||
        (reinterpret_cast<uintptr_t>(seav_view) & 3u))
      return SSPD_ERR_DATA;
    tr = SeavTracker{reinterpret_cast<uint32_t*>(seav_view), log, log_head, (uint32_t)(log_entries - 1)};
  }
  return scan_sliding_impl(hips, oips, n, p, pool, ts_bytes, now_wrapped, max_blocks_per_sm, tr, nullptr, stream,
                           true);
}

extern "C" int sspd_scan_sliding(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p,
                                 void* pool, uint32_t ts_bytes, uint64_t now_wrapped, void* stream) {
  return sspd_scan_sliding_capped(hips, oips, n, p, pool, ts_bytes, now_wrapped, 0, stream);
}

static int scan_sliding_impl(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p_in,
                             void* pool, uint32_t ts_bytes, uint64_t now_wrapped, uint32_t max_blocks_per_sm,
                             SeavTracker tracker, uint32_t* dirty, void* stream, bool seav_only) {
  int rc = validate_params(p_in);
  if (rc) return rc;
  // seav_only: the SEAV stamps (and tracking) of the packets, no LDCA slot --
  // the same kernels with zero LDCA rows (the LDCA side is then recorded by
  // the partitioned scan into the dirty bitmap, sspd_scan_sliding_seav)
  sspd_params pv = *p_in;
  if (seav_only) {
    pv.lr = 0;
    dirty = nullptr;
  }
  const sspd_params* p = &pv;
  // tracking and deferred LDCA stamps exist for u16 stamps only
  if ((tracker.view || dirty) && ts_bytes != 2) return SSPD_ERR_CONFIG;
  if (n == 0) return SSPD_OK;
  if (!hips || !oips || !pool) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (ts_bytes) {
    case 1: {
      const int grid = grid_for(scan_sliding_kernel<uint8_t>, 256, n);
      scan_sliding_kernel<uint8_t><<<grid, 256, 0, st>>>(hips, oips, n, *p, (uint8_t*)pool, (uint8_t)now_wrapped);
      break;
    }
    case 2: {
      const bool pow2 = (p->k & (p->k - 1)) == 0 && (p->lc & (p->lc - 1)) == 0;
      const bool aligned = ((reinterpret_cast<uintptr_t>(hips) ^ reinterpret_cast<uintptr_t>(oips)) & 15u) == 0 &&
                           (reinterpret_cast<uintptr_t>(hips) & 3u) == 0;
      if (pow2 && aligned && p->slot_total < (1ull << 32) && getenv("SSPD_SLIDE_GENERIC") == nullptr) {
        float frac = 0.85f;
        if (const char* e = getenv("SSPD_SLIDE_L2_FRAC")) frac = (float)atof(e);
        frac = frac < 0.f ? 0.f : (frac > 1.f ? 1.f : frac);
        auto kern = tracker.view ? (dirty ? scan_sliding_u16_fast_kernel<true, true> : scan_sliding_u16_fast_kernel<true, false>)
                                 : (dirty ? scan_sliding_u16_fast_kernel<false, true> : scan_sliding_u16_fast_kernel<false, false>);
        int grid = grid_for(kern, 256, (n + 3) / 4);
        // optional cap (blocks per SM) so kernels on other streams (the
        // pipelined detect) stay co-resident with this store-bound scan
        uint32_t cap_bps = max_blocks_per_sm;
        if (const char* e = getenv("SSPD_SLIDE_BLOCKS_PER_SM")) cap_bps = (uint32_t)atoi(e);
        if (cap_bps) {
          int dev = 0, sms = 148;
          cudaGetDevice(&dev);
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
          const int cap = (int)cap_bps * sms;
          if (grid > cap) grid = cap;
        }
        const size_t lsm = tracker.view ? (size_t)kLogPk * p->sr * 4 : 0;
        kern<<<grid, 256, lsm, st>>>(hips, oips, n, *p, (uint16_t*)pool, (uint16_t)now_wrapped, frac, tracker, dirty);
        break;
      }
      if (tracker.view || dirty) {  // the caller's tracked / deferred state must be honoured
        if (p->slot_total >= (1ull << 32) && tracker.view) return SSPD_ERR_CONFIG;  // 32-bit log entries
        auto kern = tracker.view
                        ? (dirty ? scan_sliding_u16_generic_kernel<true, true> : scan_sliding_u16_generic_kernel<true, false>)
                        : scan_sliding_u16_generic_kernel<false, true>;
        const int grid = grid_for(kern, 256, n);
        const size_t lsm = tracker.view ? (size_t)kLogPk * p->sr * 4 : 0;
        kern<<<grid, 256, lsm, st>>>(hips, oips, n, *p, (uint16_t*)pool, (uint16_t)now_wrapped, tracker, dirty);
        break;
      }
      const int grid = grid_for(scan_sliding_kernel<uint16_t>, 256, n);
      scan_sliding_kernel<uint16_t><<<grid, 256, 0, st>>>(hips, oips, n, *p, (uint16_t*)pool, (uint16_t)now_wrapped);
      break;
    }
    case 4: {
      const int grid = grid_for(scan_sliding_kernel<uint32_t>, 256, n);
      scan_sliding_kernel<uint32_t><<<grid, 256, 0, st>>>(hips, oips, n, *p, (uint32_t*)pool, (uint32_t)now_wrapped);
      break;
    }
    case 8: {
      const int grid = grid_for(scan_sliding_kernel<uint64_t>, 256, n);
      scan_sliding_kernel<uint64_t><<<grid, 256, 0, st>>>(hips, oips, n, *p, (uint64_t*)pool, (uint64_t)now_wrapped);
      break;
    }
    default:
      return SSPD_ERR_CONFIG;
  }
  return check_launch();
}
