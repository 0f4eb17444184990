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

// Per-seed constants of mix64_lo_fast (host-computed once per launch).
struct SplitSeed {
  uint32_t lo;  // low word of the seed
  uint32_t hg;  // high word of the seed + high word of the golden gamma
  uint32_t d;   // T(hg+1) - T(hg), T(h) = (h ^ (h >> 30)) * lo32(kMixA)
  uint32_t e;   // T(hg) - hg * d
};

SSPD_HD SplitSeed split_seed(uint64_t seed) {
  SplitSeed s;
  s.lo = (uint32_t)seed;
  s.hg = (uint32_t)(seed >> 32) + (uint32_t)(kGolden >> 32);
  const uint32_t h1 = s.hg + 1u;
  const uint32_t t0 = (s.hg ^ (s.hg >> 30)) * (uint32_t)kMixA, t1 = (h1 ^ (h1 >> 30)) * (uint32_t)kMixA;
  s.d = t1 - t0;
  s.e = t0 - s.hg * s.d;
  return s;
}

#if defined(__CUDACC__)
// Low 32 bits of mix64(key ^ seed) for a 32-bit key, in 32-bit halves with
// the high-word chain of the first round folded away: after the gamma add
// the high word H0 is hg or hg + 1 (the carry of the low add), so its
// contribution to the first product, (H0 ^ (H0 >> 30)) * lo32(kMixA), is the
// affine H0 * d + e.  18 instructions per hash instead of 21.  Measured B200
// pipe costs (tools/pipe_probe.cu): LOP3/SHF/IADD3 and IMAD take 2 cycles of
// their pipe (alu / fma), IMAD.WIDE and IMAD.HI take 4; this form is 10 alu +
// 8 fma instructions (2 of them WIDE) = 20 + 20 pipe cycles per warp, against
// 24 alu-pipe cycles for the 64-bit form (tools/hash_variants.cu: 129 vs
// 115 Gpps for the scans' ten hashes per packet).  Bit-identical to
// (uint32_t)mix64(key ^ seed) for every key and seed (checked exhaustively
// over the 2^32 keys in tests/test_gpu_hash.py).
__device__ __forceinline__ uint32_t mix64_lo_fast(uint32_t key, uint32_t s_lo, uint32_t hg, uint32_t d, uint32_t e) {
  uint32_t l0, h0;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;"
      : "=r"(l0), "=r"(h0)
      : "r"(key ^ s_lo), "n"((uint32_t)(kGolden & 0xFFFFFFFFull)), "r"(hg));
  const uint32_t yl = l0 ^ __funnelshift_r(l0, h0, 30);
  const uint32_t p = yl * (uint32_t)(kMixA >> 32) + (h0 * d + e);
  const uint64_t w = (uint64_t)yl * (uint32_t)kMixA;
  const uint32_t z1l = (uint32_t)w, z1h = (uint32_t)(w >> 32) + p;
  const uint32_t y2l = z1l ^ __funnelshift_r(z1l, z1h, 27);
  const uint32_t y2h = z1h ^ (z1h >> 27);
  const uint64_t w2 = (uint64_t)y2l * (uint32_t)kMixB;
  uint32_t z2h;  // hi(y2l * lo(B)) + y2l * hi(B) + y2h * lo(B) as one dependent chain (2 IMAD after the wide one)
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(z2h) : "r"(y2l), "n"((uint32_t)(kMixB >> 32)), "r"((uint32_t)(w2 >> 32)));
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(z2h) : "r"(y2h), "n"((uint32_t)kMixB));
  const uint32_t z2l = (uint32_t)w2;
  return z2l ^ __funnelshift_r(z2l, z2h, 31);
}
__device__ __forceinline__ uint32_t mix64_lo_fast(uint32_t key, const SplitSeed& s) {
  return mix64_lo_fast(key, s.lo, s.hg, s.d, s.e);
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
