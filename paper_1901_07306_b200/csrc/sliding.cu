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

extern "C" int sspd_materialize_seav(const void* pool, uint32_t ts_bytes, const sspd_params* p,
                                     uint64_t now_wrapped, uint64_t window_slices, uint8_t* seav_out,
                                     void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (!pool || !seav_out) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t regs = 0;
  for (uint32_t i = 0; i < p->sr; ++i) regs += ((uint64_t)p->sc[i]) << p->r;
  SSPD_TS_DISPATCH(ts_bytes, {
    // one register per thread: a full grid keeps every load independent
    const int grid = (int)((regs + 255) / 256 < 0x7FFFFFFFull ? (regs + 255) / 256 : 0x7FFFFFFF);
    materialize_seav_kernel<T><<<grid, 256, 0, st>>>((const T*)pool, *p, (T)now_wrapped, window_slices, seav_out);
  })
  return check_launch();
}

extern "C" int sspd_materialize_ldca(const void* pool, uint32_t ts_bytes, const sspd_params* p,
                                     uint64_t now_wrapped, uint64_t window_slices, uint8_t* ldca_out,
                                     void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (!pool || !ldca_out) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t nbytes = p->ldca_bytes;
  SSPD_TS_DISPATCH(ts_bytes, {
    const int grid = (int)((nbytes + 255) / 256 < 0x7FFFFFFFull ? (nbytes + 255) / 256 : 0x7FFFFFFF);
    materialize_ldca_kernel<T><<<grid, 256, 0, st>>>((const T*)pool, p->slot_ldca_base, nbytes, (T)now_wrapped,
                                                     window_slices, ldca_out);
  })
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
