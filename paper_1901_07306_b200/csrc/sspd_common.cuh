// Shared device/host primitives for the sspd B200 kernels.
//
// The hash family is the reference's SplitMix64 finalizer keyed by a
// domain seed (hashing.py:48-53, 102-130).  All arithmetic is unsigned
// 64-bit wrap-around, exactly like the reference's masked Python ints and
// numpy uint64 arrays, so the device produces bit-identical indexes.
#pragma once
#include <stdint.h>
#include "../../include/sspd_b200.h"

#if defined(__CUDACC__)
#define SSPD_HD __host__ __device__ __forceinline__
#else
#define SSPD_HD static inline
#endif

namespace sspd {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;  // hashing.py:32
constexpr uint64_t kMixA = 0xBF58476D1CE4E5B9ull;    // hashing.py:33
constexpr uint64_t kMixB = 0x94D049BB133111EBull;    // hashing.py:34

SSPD_HD uint64_t mix64(uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * kMixA;
  z = (z ^ (z >> 27)) * kMixB;
  return z ^ (z >> 31);
}

#if defined(__CUDACC__)
// Low 32 bits of mix64(key ^ seed) for a 32-bit key, with the seed split on
// the host into s_lo (low word) and hg = s_hi + golden_hi: the first add of
// SplitMix64 then reads both straight from the constant bank (no per-row
// 64-bit seed load).  Same value as (uint32_t)mix64(key ^ seed).
__device__ __forceinline__ uint32_t mix64_lo_split(uint32_t key, uint32_t s_lo, uint32_t hg) {
  uint32_t zl, zh;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;"
      : "=r"(zl), "=r"(zh)
      : "r"(key ^ s_lo), "n"((uint32_t)(kGolden & 0xFFFFFFFFull)), "r"(hg));
  uint64_t z = ((uint64_t)zh << 32) | zl;
  z = (z ^ (z >> 30)) * kMixA;
  z = (z ^ (z >> 27)) * kMixB;
  return (uint32_t)(z ^ (z >> 31));
}
#endif

SSPD_HD uint64_t umulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// x mod d for the full 64-bit x (hashing.py:124 `hash64(...) % m`).
// Granlund-Montgomery round-up division (65-bit multiplier): exact for all
// 64-bit x; the pow2 branch is uniform across a launch.
SSPD_HD uint64_t mod(uint64_t x, const sspd_divisor& dv) {
  if (dv.pow2) return x & (dv.d - 1);
  uint64_t t = umulhi64(dv.magic, x);
  uint64_t q = (t + ((x - t) >> dv.sh1)) >> dv.sh2;
  return x - q * dv.d;
}

// hash_range(key, seed, m) = mix64(key ^ seed) % m   (hashing.py:120-124)
SSPD_HD uint64_t hash_range(uint64_t key, uint64_t seed, const sspd_divisor& dv) {
  return mod(mix64(key ^ seed), dv);
}

// lsb(hash_full(key, h1)) >= tau  <=>  low min(tau,32) bits are zero
// (hashing.py:111-117, 144-153).  tau_mask = (1 << min(tau,32)) - 1.
SSPD_HD bool sampled(uint64_t oip, uint64_t seed_h1, uint32_t tau_mask) {
  return ((uint32_t)mix64(oip ^ seed_h1) & tau_mask) == 0u;
}

SSPD_HD uint32_t tau_mask(uint32_t tau) {
  return tau >= 32 ? 0xFFFFFFFFu : ((1u << tau) - 1u);
}

// SeavConfig.index_of (short_sketch.py:183-193): bit j of the column is bit
// (isb+j) mod w of lp.  Equivalent to rotating the w-bit lp right by isb
// and keeping the low ibn bits (ibn <= w by constraint, short_sketch.py:148).
SSPD_HD uint32_t index_of(uint64_t lp, uint32_t isb, uint32_t ibn, uint32_t w) {
  uint64_t wmask = (w >= 64) ? ~0ull : ((1ull << w) - 1ull);
  lp &= wmask;
  uint64_t rot = isb == 0 ? lp : (((lp >> isb) | (lp << (w - isb))) & wmask);
  return (uint32_t)(rot & ((1ull << ibn) - 1ull));
}

// Inverse scatter of one column into lp bit positions (short_sketch.py:196-205
// lp_from_indexes / _row_scatter short_sketch.py:222-232).
SSPD_HD uint64_t scatter_col(uint32_t col, uint32_t isb, uint32_t ibn, uint32_t w) {
  uint64_t wmask = (w >= 64) ? ~0ull : ((1ull << w) - 1ull);
  uint64_t v = (uint64_t)col & ((1ull << ibn) - 1ull);
  if (isb == 0) return v & wmask;
  return ((v << isb) | (v >> (w - isb))) & wmask;
}

SSPD_HD uint64_t row_mask(uint32_t isb, uint32_t ibn, uint32_t w) {
  return scatter_col((1u << ibn) - 1u, isb, ibn, w);
}

}  // namespace sspd
