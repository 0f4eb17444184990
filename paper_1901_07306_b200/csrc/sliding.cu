// Sliding-window pool kernels: K3 sweep, K4 materialize, pool ages.
//
// Reference: TimestampPool (sliding.py:33-106) keeps one wrapped
// last-active-slice stamp per sketch bit; a slot is active iff
// ((now - ts) & mask) < window (sliding.py:96-102).  Stamps live in the
// smallest unsigned type whose modulus is >= 2w+2 (sliding.py:24-30), so
// the kernels are templated on the stamp width and do their arithmetic in
// that type (wrap-around == `& mask`).
#include <cuda_runtime.h>
#include "sspd_common.cuh"
#include "launch.cuh"

namespace sspd {

template <typename T>
__device__ __forceinline__ bool active(T ts, T now, uint64_t window) {
  return (uint64_t)(T)(now - ts) < window;
}

// _sweep (sliding.py:88-94): every slot whose age >= window is clamped to
// `clamp` = (now - window) & mask (age == window, i.e. just expired).
template <typename T>
__global__ void __launch_bounds__(256) sweep_kernel(T* pool, uint64_t n, T now, uint64_t window, T clamp) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const T ts = pool[j];
    if (!active<T>(ts, now, window)) pool[j] = clamp;
  }
}

// materialize_seav (sliding.py:191-203): register (rp, col) of row i is
// sum_b active(slot_row_base[i] + (rp*sc_i + col)*g + b) << b.
template <typename T>
__global__ void __launch_bounds__(256) materialize_seav_kernel(const T* __restrict__ pool,
                                                               const __grid_constant__ sspd_params p, T now,
                                                               uint64_t window, uint8_t* out) {
  uint64_t total = 0;
  for (uint32_t i = 0; i < p.sr; ++i) total += ((uint64_t)p.sc[i]) << p.r;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += stride) {
    // locate the row
    uint32_t i = 0;
    uint64_t local = j;
    while (local >= ((uint64_t)p.sc[i] << p.r)) {
      local -= ((uint64_t)p.sc[i] << p.r);
      ++i;
    }
    const T* slots = pool + p.slot_row_base[i] + local * p.g;
    uint64_t reg = 0;
    constexpr uint32_t kVec = 16 / sizeof(T);
    if ((p.g % kVec) == 0 && (reinterpret_cast<uintptr_t>(slots) & 15u) == 0) {
      for (uint32_t b0 = 0; b0 < p.g; b0 += kVec) {  // 16-byte loads of kVec stamps
        union {
          uint4 v;
          T t[kVec];
        } u;
        u.v = __ldg(reinterpret_cast<const uint4*>(slots + b0));
#pragma unroll
        for (uint32_t e = 0; e < kVec; ++e)
          if (active<T>(u.t[e], now, window)) reg |= 1ull << (b0 + e);
      }
    } else {
      for (uint32_t b = 0; b < p.g; ++b)
        if (active<T>(slots[b], now, window)) reg |= 1ull << b;
    }
    uint8_t* dst = out + p.seav_row_off[i] + local * p.reg_bytes;
    switch (p.reg_bytes) {
      case 1: *dst = (uint8_t)reg; break;
      case 2: *reinterpret_cast<uint16_t*>(dst) = (uint16_t)reg; break;
      case 4: *reinterpret_cast<uint32_t*>(dst) = (uint32_t)reg; break;
      default: *reinterpret_cast<uint64_t*>(dst) = reg; break;
    }
  }
}

// Fast path of materialize_seav for the common layout (g = 8 one-byte
// registers, u16 stamps): a thread builds FOUR consecutive registers of one
// row from four independent 16-byte streaming loads (8 stamps each) and
// writes them as one u32, so the pass runs at HBM speed instead of being
// instruction-bound (one register per thread).  `quads` = registers / 4.
__device__ __forceinline__ uint32_t active8_u16(uint4 v, uint16_t now, uint32_t window) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t bits = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t lo = (uint16_t)(now - (uint16_t)(w[e] & 0xFFFFu));
    const uint32_t hi = (uint16_t)(now - (uint16_t)(w[e] >> 16));
    bits |= (lo < window ? 1u : 0u) << (2 * e);
    bits |= (hi < window ? 1u : 0u) << (2 * e + 1);
  }
  return bits;
}

__global__ void __launch_bounds__(256) materialize_seav_g8u16_kernel(const uint16_t* __restrict__ pool,
                                                                     const __grid_constant__ sspd_params p,
                                                                     uint16_t now, uint32_t window, uint64_t quads,
                                                                     uint8_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < quads; q += stride) {
    uint32_t i = 0;
    uint64_t local = q;
    while (local >= (((uint64_t)p.sc[i] << p.r) >> 2)) {
      local -= ((uint64_t)p.sc[i] << p.r) >> 2;
      ++i;
    }
    const uint4* src = reinterpret_cast<const uint4*>(pool + p.slot_row_base[i]) + local * 4;
    const uint4 v0 = __ldcs(src), v1 = __ldcs(src + 1), v2 = __ldcs(src + 2), v3 = __ldcs(src + 3);
    const uint32_t word = active8_u16(v0, now, window) | (active8_u16(v1, now, window) << 8) |
                          (active8_u16(v2, now, window) << 16) | (active8_u16(v3, now, window) << 24);
    *reinterpret_cast<uint32_t*>(out + p.seav_row_off[i] + local * 4) = word;
  }
}

// ---- incremental SEAV view (SlidingDetector, u16 stamps) -----------------
// meta (u64): [0] log head (entries ever appended by the tracked scan),
// [1] "view invalid" flag (sticky: full materialization at every detect),
// [4 + s % nseg] = log head at the end of slice s.
__global__ void seav_record_kernel(unsigned long long* meta, uint32_t seg_slot) {
  meta[4 + seg_slot] = meta[0];
}

// Clear the view bit of every SEAV slot logged during slice e whose stamp is
// still e (not re-touched since): those are exactly the bits that turn
// inactive when `now` reaches e + window (sliding.py:96-102).
__global__ void __launch_bounds__(256) seav_expire_kernel(const uint16_t* __restrict__ pool,
                                                          const __grid_constant__ sspd_params p, uint32_t* view,
                                                          const uint32_t* __restrict__ log, uint64_t log_entries,
                                                          unsigned long long* meta, int32_t start_slot,
                                                          uint32_t end_slot, uint16_t expired) {
  const unsigned long long start = start_slot < 0 ? 0ull : meta[4 + start_slot];
  const unsigned long long end = meta[4 + end_slot];
  if (meta[0] - start > log_entries) {  // the ring overwrote entries of slice e
    if (blockIdx.x == 0 && threadIdx.x == 0) meta[1] = 1ull;
    return;
  }
  const uint64_t mask = log_entries - 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t pos = start + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < end; pos += stride) {
    const uint32_t slot = log[pos & mask];
    if (pool[slot] != expired) continue;
    uint32_t i = 0;
    while (i + 1 < p.sr && p.slot_row_base[i + 1] <= slot) ++i;
    const uint64_t rel = slot - p.slot_row_base[i];
    const uint64_t vbit = (p.seav_row_off[i] + (rel / p.g) * p.reg_bytes) * 8 + rel % p.g;
    atomicAnd(view + (vbit >> 5), ~(1u << (vbit & 31)));
  }
}

__global__ void __launch_bounds__(256) materialize_seav_g8u16_if_kernel(const uint16_t* __restrict__ pool,
                                                                        const __grid_constant__ sspd_params p,
                                                                        uint16_t now, uint32_t window, uint64_t quads,
                                                                        uint8_t* out,
                                                                        const unsigned long long* flag) {
  if (*flag == 0ull) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < quads; q += stride) {
    uint32_t i = 0;
    uint64_t local = q;
    while (local >= (((uint64_t)p.sc[i] << p.r) >> 2)) {
      local -= ((uint64_t)p.sc[i] << p.r) >> 2;
      ++i;
    }
    const uint4* src = reinterpret_cast<const uint4*>(pool + p.slot_row_base[i]) + local * 4;
    const uint4 v0 = __ldcs(src), v1 = __ldcs(src + 1), v2 = __ldcs(src + 2), v3 = __ldcs(src + 3);
    *reinterpret_cast<uint32_t*>(out + p.seav_row_off[i] + local * 4) =
        active8_u16(v0, now, window) | (active8_u16(v1, now, window) << 8) | (active8_u16(v2, now, window) << 16) |
        (active8_u16(v3, now, window) << 24);
  }
}

// materialize_ldca (sliding.py:215-220): byte q of the packed array holds
// the activity of slots ldca_base + 8q .. 8q+7, little bit order.
template <typename T>
__global__ void __launch_bounds__(256) materialize_ldca_kernel(const T* __restrict__ pool, uint64_t base,
                                                               uint64_t nbytes, T now, uint64_t window,
                                                               uint8_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nbytes; q += stride) {
    const T* s = pool + base + q * 8;
    uint32_t v = 0;
    if (sizeof(T) == 2 && (reinterpret_cast<uintptr_t>(s) & 15u) == 0) {  // 8 u16 stamps = one 16-B load
      union {
        uint4 v4;
        T t[8];
      } u;
      u.v4 = __ldg(reinterpret_cast<const uint4*>(s));
#pragma unroll
      for (int b = 0; b < 8; ++b) v |= (active<T>(u.t[b], now, window) ? 1u : 0u) << b;
    } else {
#pragma unroll
      for (int b = 0; b < 8; ++b) v |= (active<T>(s[b], now, window) ? 1u : 0u) << b;
    }
    out[q] = (uint8_t)v;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) ages_kernel(const T* __restrict__ pool, uint64_t n, T now, uint64_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride)
    out[j] = (uint64_t)(T)(now - pool[j]);
}

// TimestampPool.touch_batch (sliding.py:77-79): ts[slot_indexes] = now.
// Duplicates all store the same value, so the scatter needs no ordering.
template <typename T>
__global__ void touch_slots_kernel(T* __restrict__ pool, uint64_t n_slots, const int64_t* __restrict__ idx,
                                   uint64_t n, T now, uint32_t* __restrict__ bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    int64_t s = idx[j];
    if (s < 0) s += (int64_t)n_slots;  // numpy's negative indexes
    if (s < 0 || (uint64_t)s >= n_slots) {
      if (bad) atomicOr(bad, 1u);
    } else {
      pool[s] = now;
    }
  }
}

}  // namespace sspd

using namespace sspd;

#define SSPD_TS_DISPATCH(ts_bytes, ...)          \
  switch (ts_bytes) {                             \
    case 1: { typedef uint8_t T; __VA_ARGS__; break; }   \
    case 2: { typedef uint16_t T; __VA_ARGS__; break; }  \
    case 4: { typedef uint32_t T; __VA_ARGS__; break; }  \
    case 8: { typedef uint64_t T; __VA_ARGS__; break; }  \
    default: return SSPD_ERR_CONFIG;              \
  }

extern "C" int sspd_sweep(void* pool, uint64_t n_slots, uint32_t ts_bytes, uint64_t now_wrapped,
                          uint64_t window_slices, uint64_t clamp_value, void* stream) {
  if (n_slots == 0) return SSPD_OK;
  if (!pool) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SSPD_TS_DISPATCH(ts_bytes, {
    const int grid = grid_for(sweep_kernel<T>, 256, n_slots);
    sweep_kernel<T><<<grid, 256, 0, st>>>((T*)pool, n_slots, (T)now_wrapped, window_slices, (T)clamp_value);
  })
  return check_launch();
}

extern "C" int sspd_touch_slots(void* pool, uint64_t n_slots, uint32_t ts_bytes, const int64_t* slot_indexes,
                                uint64_t n, uint64_t now_wrapped, uint32_t* bad_flag, void* stream) {
  if (n == 0) return SSPD_OK;
  if (!pool || !slot_indexes) return SSPD_ERR_DATA;
  if (n_slots > (uint64_t)INT64_MAX) return SSPD_ERR_CONFIG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SSPD_TS_DISPATCH(ts_bytes, {
    const int grid = grid_for(touch_slots_kernel<T>, 256, n);
    touch_slots_kernel<T><<<grid, 256, 0, st>>>((T*)pool, n_slots, slot_indexes, n, (T)now_wrapped, bad_flag);
  })
  return check_launch();
}

extern "C" int sspd_materialize_seav(const void* pool, uint32_t ts_bytes, const sspd_params* p,
                                     uint64_t now_wrapped, uint64_t window_slices, uint8_t* seav_out,
                                     void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (!pool || !seav_out) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t regs = 0;
  for (uint32_t i = 0; i < p->sr; ++i) regs += ((uint64_t)p->sc[i]) << p->r;
  bool fast = ts_bytes == 2 && p->g == 8 && p->reg_bytes == 1 &&
              (reinterpret_cast<uintptr_t>(pool) & 15u) == 0 && (reinterpret_cast<uintptr_t>(seav_out) & 3u) == 0;
  for (uint32_t i = 0; i < p->sr && fast; ++i)
    fast = ((((uint64_t)p->sc[i]) << p->r) & 3u) == 0 && (p->slot_row_base[i] & 7u) == 0 && (p->seav_row_off[i] & 3u) == 0;
  if (fast) {
    const uint64_t quads = regs >> 2;
    const int grid = grid_for(materialize_seav_g8u16_kernel, 256, quads);
    materialize_seav_g8u16_kernel<<<grid, 256, 0, st>>>((const uint16_t*)pool, *p, (uint16_t)now_wrapped,
                                                        (uint32_t)window_slices, quads, seav_out);
    return check_launch();
  }
  SSPD_TS_DISPATCH(ts_bytes, {
    // one register per thread: a full grid keeps every load independent
    const int grid = (int)((regs + 255) / 256 < 0x7FFFFFFFull ? (regs + 255) / 256 : 0x7FFFFFFF);
    materialize_seav_kernel<T><<<grid, 256, 0, st>>>((const T*)pool, *p, (T)now_wrapped, window_slices, seav_out);
  })
  return check_launch();
}

// materialize_ldca fast path (u16 stamps): four output bytes per thread
// from four independent 16-byte streaming loads, one u32 store.
__global__ void __launch_bounds__(256) materialize_ldca_u16x4_kernel(const uint16_t* __restrict__ pool, uint64_t base,
                                                                     uint64_t nwords, uint16_t now, uint32_t window,
                                                                     uint32_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nwords; q += stride) {
    const uint4* src = reinterpret_cast<const uint4*>(pool + base) + q * 4;
    const uint4 v0 = __ldcs(src), v1 = __ldcs(src + 1), v2 = __ldcs(src + 2), v3 = __ldcs(src + 3);
    out[q] = active8_u16(v0, now, window) | (active8_u16(v1, now, window) << 8) |
             (active8_u16(v2, now, window) << 16) | (active8_u16(v3, now, window) << 24);
  }
}

extern "C" int sspd_materialize_ldca(const void* pool, uint32_t ts_bytes, const sspd_params* p,
                                     uint64_t now_wrapped, uint64_t window_slices, uint8_t* ldca_out,
                                     void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (!pool || !ldca_out) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t nbytes = p->ldca_bytes;
  if (ts_bytes == 2 && (nbytes & 3u) == 0 && (p->slot_ldca_base & 7u) == 0 &&
      (reinterpret_cast<uintptr_t>(pool) & 15u) == 0 && (reinterpret_cast<uintptr_t>(ldca_out) & 3u) == 0) {
    const uint64_t nwords = nbytes >> 2;
    const int grid = grid_for(materialize_ldca_u16x4_kernel, 256, nwords);
    materialize_ldca_u16x4_kernel<<<grid, 256, 0, st>>>((const uint16_t*)pool, p->slot_ldca_base, nwords,
                                                        (uint16_t)now_wrapped, (uint32_t)window_slices,
                                                        reinterpret_cast<uint32_t*>(ldca_out));
    return check_launch();
  }
  SSPD_TS_DISPATCH(ts_bytes, {
    const int grid = (int)((nbytes + 255) / 256 < 0x7FFFFFFFull ? (nbytes + 255) / 256 : 0x7FFFFFFF);
    materialize_ldca_kernel<T><<<grid, 256, 0, st>>>((const T*)pool, p->slot_ldca_base, nbytes, (T)now_wrapped,
                                                     window_slices, ldca_out);
  })
  return check_launch();
}

// Fold of the deferred LDCA stamps (scan.cu, kDefer): every slot whose bit
// is set in `dirty` gets stamp `now`, the bitmap is cleared, and -- when
// `view` is given -- the packed active-bit LDCA view (sliding.py:205-220) is
// written in the same pass: active = dirty | (age(old stamp) < w).  One
// thread per dirty word = 32 slots = 64 B of stamps.  Without a view, clean
// words cost only the 4-byte bitmap read.
__device__ __forceinline__ uint32_t stamp_pairs(uint32_t w, uint32_t m2, uint32_t now) {
  const uint32_t lo = (m2 & 1u) ? now : (w & 0xFFFFu);
  const uint32_t hi = (m2 & 2u) ? now : (w >> 16);
  return lo | (hi << 16);
}

template <bool kView>
__global__ void __launch_bounds__(256) ldca_fold_u16_kernel(uint16_t* __restrict__ pool, uint64_t base,
                                                            uint64_t nwords, uint32_t* __restrict__ dirty,
                                                            uint16_t now, uint32_t window, uint32_t* __restrict__ view) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nwords; q += stride) {
    uint4* src = reinterpret_cast<uint4*>(pool + base) + q * 4;
    const uint32_t d = __ldcg(dirty + q);
    if (kView) {
      // the view needs every stamp: issue the four 16-B loads with the
      // bitmap load instead of after it
      uint4 v[4];
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j) v[j] = __ldcg(src + j);
      uint32_t act = 0;
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j) act |= active8_u16(v[j], now, window) << (8 * j);
      view[q] = act | d;  // a dirty slot is stamped `now`: age 0 < w
      if (d == 0) continue;
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j) {
        const uint32_t m = (d >> (8 * j)) & 0xFFu;
        if (m) {
          uint4 u = v[j];
          u.x = stamp_pairs(u.x, m, now);
          u.y = stamp_pairs(u.y, m >> 2, now);
          u.z = stamp_pairs(u.z, m >> 4, now);
          u.w = stamp_pairs(u.w, m >> 6, now);
          src[j] = u;
        }
      }
      dirty[q] = 0;
    } else {
      if (d == 0) continue;
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j) {
        const uint32_t m = (d >> (8 * j)) & 0xFFu;
        if (m) {
          uint4 u = __ldcg(src + j);
          u.x = stamp_pairs(u.x, m, now);
          u.y = stamp_pairs(u.y, m >> 2, now);
          u.z = stamp_pairs(u.z, m >> 4, now);
          u.w = stamp_pairs(u.w, m >> 6, now);
          src[j] = u;
        }
      }
      dirty[q] = 0;
    }
  }
}

extern "C" int sspd_ldca_fold(void* pool, uint32_t ts_bytes, const sspd_params* p, uint32_t* dirty,
                              uint64_t now_wrapped, uint64_t window_slices, uint8_t* ldca_view, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (!pool || !dirty) return SSPD_ERR_DATA;
  if (ts_bytes != 2 || (p->ldca_bytes & 3u) || (p->slot_ldca_base & 7u) || (reinterpret_cast<uintptr_t>(pool) & 15u) ||
      (reinterpret_cast<uintptr_t>(dirty) & 3u) || (reinterpret_cast<uintptr_t>(ldca_view) & 3u))
    return SSPD_ERR_CONFIG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t nwords = p->ldca_bytes >> 2;
  if (ldca_view) {
    const int grid = grid_for(ldca_fold_u16_kernel<true>, 256, nwords);
    ldca_fold_u16_kernel<true><<<grid, 256, 0, st>>>((uint16_t*)pool, p->slot_ldca_base, nwords, dirty,
                                                     (uint16_t)now_wrapped, (uint32_t)window_slices,
                                                     reinterpret_cast<uint32_t*>(ldca_view));
  } else {
    const int grid = grid_for(ldca_fold_u16_kernel<false>, 256, nwords);
    ldca_fold_u16_kernel<false><<<grid, 256, 0, st>>>((uint16_t*)pool, p->slot_ldca_base, nwords, dirty,
                                                      (uint16_t)now_wrapped, (uint32_t)window_slices, nullptr);
  }
  return check_launch();
}

// ---- ring mode of the deferred LDCA stamps (SlidingDetector._DeferredLdca)
//
// The dirty bitmap of every slice of the window is kept (ring of R = w+1
// LDCA-shaped bitmaps, slot = slice % R).  A slot is active at `now` iff it
// was stamped in one of the slices now-w+1 .. now (sliding.py:98-106: the
// anti-alias sweep keeps wrapped ages exact), so the active-bit LDCA view is
// the OR of those w bitmaps.  It is kept with the two-stack sliding-window
// OR: `acc` = OR of the current block's bitmaps (blocks of w slices), and at
// each block end the block's bitmaps are turned in place into suffix ORs
// (sspd_ldca_suffix_or), so view(now) = suffix[now-w+1] | acc | dirty[now]:
// three bitmap reads and two writes per detect instead of every LDCA stamp.
// Stamps are written lazily (sspd_ldca_fold_ring) when the pool is read and
// at block ends, before the suffix pass overwrites the raw bitmaps.

// acc |= cur; view = acc | suffix (when view); zero = 0 (when zero).  Any of
// cur / suffix / view / zero may be NULL.  Word granularity n32, vectorised.
__global__ void __launch_bounds__(256) ldca_window_or_kernel(const uint32_t* __restrict__ cur,
                                                             uint32_t* __restrict__ acc,
                                                             const uint32_t* __restrict__ suffix,
                                                             uint32_t* __restrict__ view, uint32_t* __restrict__ zero,
                                                             uint64_t n32) {
  const uint64_t n128 = n32 >> 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t i = t0; i < n128; i += stride) {
    uint4 a = reinterpret_cast<const uint4*>(acc)[i];
    if (cur) {
      const uint4 c = __ldcg(reinterpret_cast<const uint4*>(cur) + i);
      a.x |= c.x, a.y |= c.y, a.z |= c.z, a.w |= c.w;
      reinterpret_cast<uint4*>(acc)[i] = a;
    }
    if (view) {
      if (suffix) {
        const uint4 s = __ldcg(reinterpret_cast<const uint4*>(suffix) + i);
        a.x |= s.x, a.y |= s.y, a.z |= s.z, a.w |= s.w;
      }
      reinterpret_cast<uint4*>(view)[i] = a;
    }
    if (zero) reinterpret_cast<uint4*>(zero)[i] = make_uint4(0, 0, 0, 0);
  }
  for (uint64_t i = (n128 << 2) + t0; i < n32; i += stride) {  // tail words
    uint32_t a = acc[i];
    if (cur) acc[i] = a = a | cur[i];
    if (view) view[i] = suffix ? (a | suffix[i]) : a;
    if (zero) zero[i] = 0;
  }
}

// Stamps of the ring slices [lo, hi] into the LDCA slots, the newest slice
// of each slot winning (slice e writes stamp e & 0xFFFF, as the direct scan
// would have at slice e).  One thread per 32 slots; the walk stops once all
// 32 have been seen.
__global__ void __launch_bounds__(256) ldca_fold_ring_kernel(uint16_t* __restrict__ pool, uint64_t base,
                                                             uint64_t nwords, const uint32_t* __restrict__ ring,
                                                             uint64_t slot_words, uint32_t ring_slots, uint64_t lo,
                                                             uint64_t hi) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t slot_hi = (uint32_t)(hi % ring_slots);
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nwords; q += stride) {
    uint4* src = reinterpret_cast<uint4*>(pool + base) + q * 4;
    uint4 v[4];
    uint32_t seen = 0;
    bool loaded = false;
    uint32_t slot = slot_hi;
    for (uint64_t e = hi + 1; e-- > lo && seen != 0xFFFFFFFFu;) {
      const uint32_t d = __ldcg(ring + (uint64_t)slot * slot_words + q);
      slot = slot == 0 ? ring_slots - 1 : slot - 1;
      const uint32_t m = d & ~seen;
      if (!m) continue;
      if (!loaded) {
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) v[j] = __ldcg(src + j);
        loaded = true;
      }
      const uint32_t s16 = (uint32_t)(e & 0xFFFFu);
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j) {
        const uint32_t mj = (m >> (8 * j)) & 0xFFu;
        if (mj) {
          v[j].x = stamp_pairs(v[j].x, mj, s16);
          v[j].y = stamp_pairs(v[j].y, mj >> 2, s16);
          v[j].z = stamp_pairs(v[j].z, mj >> 4, s16);
          v[j].w = stamp_pairs(v[j].w, mj >> 6, s16);
        }
      }
      seen |= m;
    }
    if (loaded) {
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j)
        if ((seen >> (8 * j)) & 0xFFu) src[j] = v[j];
    }
  }
}

// In place: bitmap of slice e <- OR of slices e .. first+count-1 (suffix ORs
// of one block), walking the block from its last slice down.
template <typename V>
__global__ void __launch_bounds__(256) ldca_suffix_or_kernel(V* __restrict__ ring, uint32_t ring_slots, uint64_t nvec,
                                                             uint64_t first, uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t slot_last = (uint32_t)((first + count - 1) % ring_slots);
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nvec; q += stride) {
    V acc{};
    uint32_t slot = slot_last;
    for (uint64_t c = 0; c < count; ++c) {
      V* p = ring + (uint64_t)slot * nvec + q;
      const V x = __ldcg(p);
      if constexpr (sizeof(V) == 16) {
        acc.x |= x.x, acc.y |= x.y, acc.z |= x.z, acc.w |= x.w;
      } else {
        acc |= x;
      }
      if (c) *p = acc;  // the block's last bitmap is its own suffix
      slot = slot == 0 ? ring_slots - 1 : slot - 1;
    }
  }
}

extern "C" int sspd_ldca_window_or(const uint32_t* cur, uint32_t* acc, const uint32_t* suffix, uint32_t* view,
                                   uint32_t* zero, uint64_t nbytes, void* stream) {
  if (nbytes == 0) return SSPD_OK;
  if (!acc || (nbytes & 3u)) return SSPD_ERR_DATA;
  const uintptr_t al = reinterpret_cast<uintptr_t>(cur) | reinterpret_cast<uintptr_t>(acc) |
                       reinterpret_cast<uintptr_t>(suffix) | reinterpret_cast<uintptr_t>(view) |
                       reinterpret_cast<uintptr_t>(zero);
  if (al & 15u) return SSPD_ERR_CONFIG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t n32 = nbytes >> 2;
  const int grid = grid_for(ldca_window_or_kernel, 256, (n32 + 3) >> 2);
  ldca_window_or_kernel<<<grid, 256, 0, st>>>(cur, acc, suffix, view, zero, n32);
  return check_launch();
}

extern "C" int sspd_ldca_fold_ring(void* pool, uint32_t ts_bytes, const sspd_params* p, const uint32_t* ring,
                                   uint64_t slot_stride_bytes, uint32_t ring_slots, uint64_t slice_lo,
                                   uint64_t slice_hi, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (!pool || !ring || ring_slots == 0) return SSPD_ERR_DATA;
  if (ts_bytes != 2 || (p->ldca_bytes & 3u) || (p->slot_ldca_base & 7u) || (reinterpret_cast<uintptr_t>(pool) & 15u) ||
      (reinterpret_cast<uintptr_t>(ring) & 3u))
    return SSPD_ERR_CONFIG;
  // consecutive slices' bitmaps are slot_stride_bytes apart (>= the LDCA
  // bytes, a multiple of 4: the Python ring pads them to 16 B)
  if ((slot_stride_bytes & 3u) || slot_stride_bytes < p->ldca_bytes) return SSPD_ERR_CONFIG;
  if (slice_hi < slice_lo) return SSPD_OK;
  if (slice_hi - slice_lo >= ring_slots) return SSPD_ERR_DATA;  // the ring holds R slices at most
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t nwords = p->ldca_bytes >> 2;
  const int grid = grid_for(ldca_fold_ring_kernel, 256, nwords);
  ldca_fold_ring_kernel<<<grid, 256, 0, st>>>((uint16_t*)pool, p->slot_ldca_base, nwords, ring,
                                              slot_stride_bytes >> 2, ring_slots, slice_lo, slice_hi);
  return check_launch();
}

extern "C" int sspd_ldca_suffix_or(uint32_t* ring, uint32_t ring_slots, uint64_t nbytes, uint64_t first_slice,
                                   uint64_t count, void* stream) {
  if (count == 0 || nbytes == 0) return SSPD_OK;
  if (!ring || (nbytes & 3u) || count > ring_slots) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((nbytes & 15u) == 0 && (reinterpret_cast<uintptr_t>(ring) & 15u) == 0) {
    const uint64_t nvec = nbytes >> 4;
    const int grid = grid_for(ldca_suffix_or_kernel<uint4>, 256, nvec);
    ldca_suffix_or_kernel<uint4><<<grid, 256, 0, st>>>(reinterpret_cast<uint4*>(ring), ring_slots, nvec, first_slice,
                                                       count);
  } else {
    const uint64_t nvec = nbytes >> 2;
    const int grid = grid_for(ldca_suffix_or_kernel<uint32_t>, 256, nvec);
    ldca_suffix_or_kernel<uint32_t><<<grid, 256, 0, st>>>(ring, ring_slots, nvec, first_slice, count);
  }
  return check_launch();
}

static bool seav_fast_layout(const void* pool, const sspd_params* p, const void* out) {
  bool ok = p->g == 8 && p->reg_bytes == 1 && (reinterpret_cast<uintptr_t>(pool) & 15u) == 0 &&
            (reinterpret_cast<uintptr_t>(out) & 3u) == 0;
  for (uint32_t i = 0; i < p->sr && ok; ++i)
    ok = ((((uint64_t)p->sc[i]) << p->r) & 3u) == 0 && (p->slot_row_base[i] & 7u) == 0 && (p->seav_row_off[i] & 3u) == 0;
  return ok;
}

// advance_slice of an incrementally tracked pool (u16 stamps): record the
// log head for slice `now_abs`, then clear the bits of slice now_abs+1-w.
extern "C" int sspd_seav_advance(const void* pool, uint32_t ts_bytes, const sspd_params* p, uint8_t* seav_view,
                                 const uint32_t* log, uint64_t log_entries, unsigned long long* meta, uint32_t nseg,
                                 uint64_t now_abs, uint64_t window_slices, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (ts_bytes != 2 || nseg < window_slices + 2) return SSPD_ERR_CONFIG;
  if (!pool || !seav_view || !log || !meta || log_entries == 0 || (log_entries & (log_entries - 1)))
    return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  seav_record_kernel<<<1, 1, 0, st>>>(meta, (uint32_t)(now_abs % nseg));
  if (now_abs + 1 >= window_slices) {
    const uint64_t e = now_abs + 1 - window_slices;
    const int32_t start_slot = e == 0 ? -1 : (int32_t)((e - 1) % nseg);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    seav_expire_kernel<<<sms * 2, 256, 0, st>>>((const uint16_t*)pool, *p, reinterpret_cast<uint32_t*>(seav_view),
                                                log, log_entries, meta, start_slot, (uint32_t)(e % nseg),
                                                (uint16_t)(e & 0xFFFFu));
  }
  return check_launch();
}

// The SEAV view materialized from the pool only when *flag != 0 (the
// incremental view was invalidated); otherwise a no-op launch.
extern "C" int sspd_materialize_seav_if(const void* pool, uint32_t ts_bytes, const sspd_params* p,
                                        uint64_t now_wrapped, uint64_t window_slices, uint8_t* seav_out,
                                        const unsigned long long* flag, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (ts_bytes != 2 || !seav_fast_layout(pool, p, seav_out)) return SSPD_ERR_CONFIG;
  if (!flag) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t regs = 0;
  for (uint32_t i = 0; i < p->sr; ++i) regs += ((uint64_t)p->sc[i]) << p->r;
  const uint64_t quads = regs >> 2;
  const int grid = grid_for(materialize_seav_g8u16_if_kernel, 256, quads);
  materialize_seav_g8u16_if_kernel<<<grid, 256, 0, st>>>((const uint16_t*)pool, *p, (uint16_t)now_wrapped,
                                                         (uint32_t)window_slices, quads, seav_out, flag);
  return check_launch();
}

extern "C" int sspd_pool_ages(const void* pool, uint64_t n_slots, uint32_t ts_bytes, uint64_t now_wrapped,
                              uint64_t* ages_out, void* stream) {
  if (n_slots == 0) return SSPD_OK;
  if (!pool || !ages_out) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SSPD_TS_DISPATCH(ts_bytes, {
    const int grid = grid_for(ages_kernel<T>, 256, n_slots);
    ages_kernel<T><<<grid, 256, 0, st>>>((const T*)pool, n_slots, (T)now_wrapped, ages_out);
  })
  return check_launch();
}
