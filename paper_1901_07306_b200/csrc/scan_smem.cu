// K1p: the partitioned scan -- the LDCA lives in the SMs' shared memory.
//
// Why: every packet sets LR (=8) bits at uniformly random words of the
// 8 MiB LDCA.  Done as L2 atomics that is 8 random `red.or` per packet and
// the scan is capped by the L2 atomic rate (~190-215 G/s measured, ~23.7
// Gpps); random L2 loads cap at ~287 G/s as well.  Shared-memory atomics
// run at ~2,000 G/s per chip, and 148 SMs x 227 KB = 33 MB of shared memory
// holds the whole 8 MiB LDCA.  So:
//
//   * the LDCA word space is cut into P contiguous partitions, one per CTA
//     (one persistent 1024-thread CTA per SM, cooperative launch); each CTA
//     keeps its partition in shared memory for the whole launch;
//   * the stream is processed in chunks.  Producer phase: every CTA hashes
//     its slice of chunk t tile by tile, appends each LDCA update
//     (local word << 5 | bit, one u32) to a per-destination shared-memory
//     staging area, and flushes the staging areas as coalesced runs into
//     its OWN region of each destination's bucket -- region (src, dst) is
//     private to one producer CTA, so no global atomics are needed; the
//     run lengths are published once per chunk;
//   * consumer phase: CTA q ORs every region (src, q) of chunk t-1 into its
//     partition with shared-memory atomics.  Buckets are double-buffered,
//     so ONE grid barrier per chunk separates "chunk t produced" from
//     "chunk t consumed";
//   * at the end each CTA ORs its partition into the global LDCA.
//
// Per packet the L2 sees 32 B of coalesced bucket writes + 32 B of reads
// instead of 8 random atomics.  Anything that does not fit (a staging area
// or a region overflowing under a skewed stream) falls back to a direct L2
// `red.or` on the global LDCA -- exact, because OR is commutative and
// idempotent.  SEAV updates (0.78 % of packets at tau=7) stay direct reds.
//
// Reference semantics are unchanged from K1 (scan.cu): bit (i*lc + c_i)*k + b
// of the LDCA, c_i = LH_i(hip) % lc, b = H3(oip) % k (long_sketch.py:125-135),
// and the SEAV update of short_sketch.py:300-318.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sspd_common.cuh"
#include "launch.cuh"

namespace cg = cooperative_groups;

namespace sspd {

__device__ __forceinline__ void red_or_g(uint32_t* addr, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

// floor(x / d) with the same round-up multiplier as sspd::mod
__device__ __forceinline__ uint64_t div_fast(uint64_t x, const sspd_divisor& dv) {
  if (dv.pow2) return x >> (63 - __clzll(dv.d));
  const uint64_t t = __umul64hi(dv.magic, x);
  return (t + ((x - t) >> dv.sh1)) >> dv.sh2;
}

// Staging overflow (rare, skewed streams): re-apply every LDCA row of the
// packet as a direct L2 red (exact: OR is idempotent).  Out of line so the
// hot loop keeps its registers.
__device__ __noinline__ void reapply_direct(const sspd_params& p, uint32_t lc_mask, uint32_t log2k, uint32_t hip,
                                            uint32_t bb, uint32_t* ldca) {
  for (uint32_t i = 0; i < p.lr; ++i) {
    const uint32_t c = (uint32_t)mix64(hip ^ p.seed_lh[i]) & lc_mask;
    const uint32_t bit = ((i * p.lc + c) << log2k) | bb;
    red_or_g(ldca + (bit >> 5), 1u << (bit & 31u));
  }
}


// SEAV update of one sampled packet (short_sketch.py:300-318): SR direct reds.
__device__ __forceinline__ void seav_update(const sspd_params& p, uint32_t hip, uint32_t oip, uint32_t* seav) {
  const uint32_t sbit = (uint32_t)hash_range(oip, p.seed_h2, p.div_g);
  const uint64_t rp = hip & ((1u << p.r) - 1u);
  const uint64_t lp = ((uint64_t)hip >> p.r) & ((1ull << p.lp_bits) - 1ull);
  for (uint32_t i = 0; i < p.sr; ++i) {
    const uint32_t col = index_of(lp, p.isb[i], p.ibn[i], p.lp_bits);
    const uint64_t abs_bit = (p.seav_row_off[i] + (rp * p.sc[i] + col) * p.reg_bytes) * 8 + sbit;
    red_or_g(seav + (abs_bit >> 5), 1u << (abs_bit & 31));
  }
}
__device__ __noinline__ void seav_update_ool(const sspd_params& p, uint32_t hip, uint32_t oip, uint32_t* seav) {
  seav_update(p, hip, oip, seav);
}

#ifndef SSPD_PART_THREADS
#define SSPD_PART_THREADS 1024
#endif
constexpr uint32_t kThreads = SSPD_PART_THREADS;
constexpr uint32_t kPktPerThread = 4;  // packets per thread per tile (= one uint4 of hips + oips)
constexpr uint32_t kTile = kThreads * kPktPerThread;
// sampled packets (0.78 % at tau = 7, ~32 per tile) are queued in shared
// memory and their SEAV updates applied by all lanes after the tile, instead
// of one divergent lane per warp inside the hashing loop
constexpr uint32_t kSeavQueue = 128;  // per tile parity

// Producer routing modes, chosen per launch by the host plan:
//   kGeneric  64-bit index math, any k / lc (exact 64-bit modulo)
//   kFast32   k, lc powers of two, < 2^32 LDCA bits; partition = magic division
//   kPow2     kFast32 + power-of-two partitions + LR = 8 unrolled with static
//             seeds: q = bit >> pshift, staged entry = bit & pmask
enum : int { kGeneric = 0, kFast32 = 1, kPow2 = 2 };

struct PartPlan {
  uint32_t nparts;        // consumers = partitions (CTAs 0 .. nparts-1)
  uint32_t nsrc;          // producers = gridDim.x (>= nparts)
  uint32_t part_words;    // words per partition (last one may be shorter)
  uint32_t stage_slots;   // staging slots per destination per tile
  uint64_t total_words;   // LDCA words (ceil(bits / 32))
  sspd_divisor div_part;  // divisor by part_words (generic mode)
  uint32_t region_cap;    // entries per (src, dst) region per chunk
  uint32_t w_owner, w_other;  // producer slice weights (consumers vs pure producers)
  uint64_t chunk;         // packets per chunk
  uint64_t n;             // packets
  uint32_t* buckets;      // [2][dst][src][region_cap]
  uint32_t* counts;       // [2][dst][src]
  uint32_t k_mask, lc_mask, log2k;
  uint32_t magic32, sh32;  // floor(w / part_words) for 32-bit w (fast mode)
  uint32_t pshift, pmask;  // pow2 mode: partition of a bit index / its local bit
  uint32_t qshift;         // pow2 mode: partition of a cell index (pshift - log2k)
  uint32_t s_lo[10], s_hg[10];  // split seeds (mix64_lo_split): H3, H1, LH0..7
  uint32_t vec_ok;         // hips/oips 16-byte aligned and chunk % 4 == 0
  uint32_t qstride;        // ns * region_cap: bucket elements per destination
  uint32_t gshift;         // log2 of the flush group size (threads per destination)
};

// Weighted producer slice of CTA s in [c0, c1): pure producers (s >= nparts)
// take w_other/w_owner as much as consumer CTAs; boundaries are 4-aligned.
__device__ __forceinline__ uint64_t slice_start(const PartPlan& P, uint64_t c0, uint64_t c1, uint32_t s) {
  if (s >= P.nsrc) return c1;
  const uint64_t tw = (uint64_t)P.nparts * P.w_owner + (uint64_t)(P.nsrc - P.nparts) * P.w_other;
  const uint64_t cw = (uint64_t)min(s, P.nparts) * P.w_owner + (uint64_t)(s > P.nparts ? s - P.nparts : 0) * P.w_other;
  const uint64_t off = (((c1 - c0) * cw) / tw) & ~3ull;
  return min(c1, c0 + off);
}

// Shared memory: [part_words | nparts*stage_slots staging | nparts cnt | nparts cursor | sink
//                 | sampled-packet queue (count + kSeavQueue (hip, oip) pairs)]
template <bool kSeav, int kMode>
__global__ void __launch_bounds__(kThreads, 1)
    scan_partitioned_kernel(const uint32_t* __restrict__ hips, const uint32_t* __restrict__ oips,
                            const __grid_constant__ sspd_params p, const __grid_constant__ PartPlan P,
                            uint32_t* seav, uint32_t* ldca) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* part = smem;
  uint32_t* stage = smem + P.part_words;
  uint32_t* cnt = stage + (size_t)P.nparts * P.stage_slots;
  uint32_t* cursor = cnt + P.nparts;
  uint32_t* sink = cursor + P.nparts;  // dummy target for overflowing staging writes
  uint32_t* sq_cnt = sink + 4;         // [2] queue counts by tile parity (16-B aligned)
  uint2* sq_base = reinterpret_cast<uint2*>(sq_cnt + 4);  // [2][kSeavQueue]
  cg::grid_group grid = cg::this_grid();
  const uint32_t self = blockIdx.x;
  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31, warp = tid >> 5, nwarps = kThreads >> 5;
  const uint32_t tmask = tau_mask(p.tau);
  const uint32_t np = P.nparts, ns = P.nsrc;
  const bool owner = self < np;

  for (uint32_t i = tid; i < P.part_words; i += kThreads) part[i] = 0;
  for (uint32_t i = tid; i < np; i += kThreads) cnt[i] = cursor[i] = 0;
  if (tid == 0) sq_cnt[0] = sq_cnt[1] = 0;
  __syncthreads();

  const uint64_t nchunks = (P.n + P.chunk - 1) / P.chunk;
  const uint64_t k = p.k;
  for (uint64_t t = 0; t <= nchunks; ++t) {
    // ---------------- consume chunk t-1 into the shared partition --------
    if (t >= 1 && owner) {
      const uint32_t b = (uint32_t)((t - 1) & 1);
      const uint32_t* cnts = P.counts + ((size_t)b * np + self) * ns;
      const uint32_t* regions = P.buckets + ((size_t)b * np + self) * (size_t)ns * P.region_cap;
      // warp w drains sources w, w+W, ... (W = warps per CTA): fetch all of
      // its run lengths at once (lane j holds source w+W*j) so no region
      // waits on its count
      const uint32_t my_src = warp + nwarps * lane;
      const uint32_t my_cnt = my_src < ns ? min(__ldcg(cnts + my_src), P.region_cap) : 0u;
      for (uint32_t src = warp, j = 0; src < ns; src += nwarps, ++j) {
        const uint32_t m = __shfl_sync(0xffffffffu, my_cnt, j);
        const uint32_t* reg = regions + (size_t)src * P.region_cap;  // 128-B aligned
        const uint32_t m4 = m >> 2;
        const uint4* r4 = reinterpret_cast<const uint4*>(reg);
        for (uint32_t j0 = lane; j0 < m4; j0 += 128) {  // 4 independent 16-B loads in flight per lane
          uint4 u[4];
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if (j0 + 32 * g < m4) u[g] = __ldcg(r4 + j0 + 32 * g);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            if (j0 + 32 * g < m4) {
              atomicOr(&part[u[g].x >> 5], 1u << (u[g].x & 31));
              atomicOr(&part[u[g].y >> 5], 1u << (u[g].y & 31));
              atomicOr(&part[u[g].z >> 5], 1u << (u[g].z & 31));
              atomicOr(&part[u[g].w >> 5], 1u << (u[g].w & 31));
            }
          }
        }
        for (uint32_t jj = (m4 << 2) + lane; jj < m; jj += 32) {
          const uint32_t u = __ldcg(reg + jj);
          atomicOr(&part[u >> 5], 1u << (u & 31));
        }
        // the region is dead once read: drop its L2 lines without write-back
        // so bucket traffic stays on-chip instead of spilling to HBM
        __syncwarp();
        for (uint32_t line = lane; line * 32 < m; line += 32)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(reg + line * 32) : "memory");
      }
    }
    // ---------------- produce chunk t ------------------------------------
    if (t < nchunks) {
      const uint32_t b = (uint32_t)(t & 1);
      const uint64_t c0 = t * P.chunk;
      const uint64_t c1 = min(P.n, c0 + P.chunk);
      const uint64_t lo = slice_start(P, c0, c1, self);
      const uint64_t hi = slice_start(P, c0, c1, self + 1);
      // software pipeline: thread tid owns the kPktPerThread consecutive
      // packets base + 4 tid + e, fetched one tile ahead with one 16-byte
      // load per array when the slice is aligned
      auto fetch = [&](uint64_t first, uint32_t* h, uint32_t* o) {
        if (P.vec_ok && first + kPktPerThread <= hi) {
          const uint4 hv = __ldcs(reinterpret_cast<const uint4*>(hips + first));
          const uint4 ov = __ldcs(reinterpret_cast<const uint4*>(oips + first));
          h[0] = hv.x, h[1] = hv.y, h[2] = hv.z, h[3] = hv.w;
          o[0] = ov.x, o[1] = ov.y, o[2] = ov.z, o[3] = ov.w;
        } else {
#pragma unroll
          for (uint32_t e = 0; e < kPktPerThread; ++e) {
            h[e] = first + e < hi ? __ldcs(hips + first + e) : 0u;
            o[e] = first + e < hi ? __ldcs(oips + first + e) : 0u;
          }
        }
      };
      uint32_t nh[kPktPerThread], no[kPktPerThread];
      fetch(lo + (uint64_t)tid * kPktPerThread, nh, no);
      uint32_t par = 0;  // tile parity: selects the sampled-packet queue
      for (uint64_t base = lo; base < hi; base += kTile, par ^= 1u) {
        uint32_t ch[kPktPerThread], co[kPktPerThread];
#pragma unroll
        for (uint32_t e = 0; e < kPktPerThread; ++e) {
          ch[e] = nh[e];
          co[e] = no[e];
        }
        fetch(base + kTile + (uint64_t)tid * kPktPerThread, nh, no);
#pragma unroll
        for (uint32_t e = 0; e < kPktPerThread; ++e) {
          const uint64_t j = base + (uint64_t)tid * kPktPerThread + e;
          const uint32_t hip = ch[e], oip = co[e];
          if (j < hi) {
            if (kMode == kPow2) {
              // LR = 8, k and lc powers of two, partitions of 2^pshift bits:
              // the staged entry is the bit index inside its partition
              const uint32_t bb = mix64_lo_split(oip, P.s_lo[0], P.s_hg[0]) & P.k_mask;
              bool ovf = false;
#pragma unroll
              for (uint32_t i = 0; i < 8; ++i) {
                // partitions hold whole cells and rows hold whole partitions
                // (plan): q = cell >> qshift, entry = (cell << log2k | b) & pmask
                const uint32_t c = mix64_lo_split(hip, P.s_lo[2 + i], P.s_hg[2 + i]) & P.lc_mask;
                const uint32_t q = (i * p.lc + c) >> P.qshift;
                const uint32_t slot = atomicAdd(&cnt[q], 1u);
                const bool fits = slot < P.stage_slots;
                ovf |= !fits;
                *(fits ? &stage[q * P.stage_slots + slot] : sink) = ((c << P.log2k) & P.pmask) | bb;
              }
              if (ovf) reapply_direct(p, P.lc_mask, P.log2k, hip, bb, ldca);
            } else if (kMode == kFast32) {
              // k, lc powers of two and < 2^32 LDCA bits: the modulo is a mask
              // of the low hash word and all index math is 32-bit.
              const uint32_t bb = (uint32_t)mix64(oip ^ p.seed_h3) & P.k_mask;
              uint32_t cellbase = 0;
              bool ovf = false;  // some staging area was full (rare)
#pragma unroll 8
              for (uint32_t i = 0; i < p.lr; ++i) {
                const uint32_t c = (uint32_t)mix64(hip ^ p.seed_lh[i]) & P.lc_mask;
                const uint32_t bit = ((cellbase + c) << P.log2k) | bb;
                const uint32_t w = bit >> 5;
                const uint32_t th = __umulhi(w, P.magic32);
                const uint32_t q = (th + ((w - th) >> 1)) >> P.sh32;
                const uint32_t local = w - q * P.part_words;
                const uint32_t slot = atomicAdd(&cnt[q], 1u);
                const bool fits = slot < P.stage_slots;
                ovf |= !fits;
                // branch-free: an overflowing update is parked in a dummy word
                *(fits ? &stage[q * P.stage_slots + slot] : sink) = (local << 5) | (bit & 31u);
                cellbase += p.lc;
              }
              if (ovf) reapply_direct(p, P.lc_mask, P.log2k, hip, bb, ldca);
            } else {
              const uint64_t bb = hash_range(oip, p.seed_h3, p.div_k);
              uint64_t cell = 0;
#pragma unroll 4
              for (uint32_t i = 0; i < p.lr; ++i) {
                const uint64_t c = hash_range(hip, p.seed_lh[i], p.div_lc);
                const uint64_t bit = (cell + c) * k + bb;
                const uint64_t w = bit >> 5;
                const uint32_t q = (uint32_t)div_fast(w, P.div_part);
                const uint32_t local = (uint32_t)(w - (uint64_t)q * P.part_words);
                const uint32_t slot = atomicAdd(&cnt[q], 1u);
                if (slot < P.stage_slots)
                  stage[q * P.stage_slots + slot] = (local << 5) | (uint32_t)(bit & 31);
                else
                  red_or_g(ldca + w, 1u << (bit & 31));  // staging full: direct (exact)
                cell += p.lc;
              }
            }
            if (kSeav && (kMode == kPow2 ? (mix64_lo_split(oip, P.s_lo[1], P.s_hg[1]) & tmask) == 0u
                                         : sampled(oip, p.seed_h1, tmask))) {
              const uint32_t qs = atomicAdd(sq_cnt + par, 1u);
              if (qs < kSeavQueue)
                sq_base[par * kSeavQueue + qs] = make_uint2(hip, oip);
              else
                seav_update_ool(p, hip, oip, seav);  // queue full (a skewed tile): apply now
            }
          }
        }
        __syncthreads();
        if (kSeav) {  // the tile's sampled packets, all lanes busy
          const uint32_t nq = min(sq_cnt[par], kSeavQueue);
          const uint2* sq = sq_base + par * kSeavQueue;
          for (uint32_t i = tid; i < nq; i += kThreads) seav_update(p, sq[i].x, sq[i].y, seav);
          // the previous tile's queue was fully read before this barrier
          if (tid == 0) sq_cnt[par ^ 1u] = 0;
        }
        // flush: a group of G = 2^gshift threads per destination (8 when
        // there are 128 destinations) copies the run as aligned 16-B stores
        // into this CTA's own region of the destination bucket (no global
        // atomics).  The loop is warp-uniform so __syncwarp is safe.
        {
          const uint32_t gs = P.gshift, G = 1u << gs, gl = tid & (G - 1u);
          const uint32_t boff = (uint32_t)b * np * P.qstride + self * P.region_cap;
          for (uint32_t q0 = 0; q0 < np; q0 += (kThreads >> gs)) {
            const uint32_t q = q0 + (tid >> gs);
            const bool act = q < np;
            const uint32_t m0 = act ? min(cnt[q], P.stage_slots) : 0u;
            uint32_t* src = stage + (act ? q : 0u) * P.stage_slots;
            // pad the run to a multiple of 4 with copies of its last update
            // (idempotent OR) so every copy below is an aligned 16-B store
            const uint32_t m = (m0 + 3u) & ~3u;
            if (gl < m - m0) src[m0 + gl] = src[m0 - 1];
            __syncwarp();
            if (m0) {
              const uint32_t pos = cursor[q];  // multiple of 4; region_cap multiple of 32
              const uint32_t fit = pos < P.region_cap ? min(m, P.region_cap - pos) : 0u;
              uint4* dst4 = reinterpret_cast<uint4*>(P.buckets + (boff + q * P.qstride + pos));
              const uint4* src4 = reinterpret_cast<const uint4*>(src);
              const uint32_t f4 = fit >> 2;
              uint32_t s = gl;
              for (; s + 3u * G < f4; s += 4u * G) {  // 4 shared loads in flight, then 4 stores
                const uint4 a0 = src4[s], a1 = src4[s + G], a2 = src4[s + 2u * G], a3 = src4[s + 3u * G];
                __stcg(dst4 + s, a0);
                __stcg(dst4 + s + G, a1);
                __stcg(dst4 + s + 2u * G, a2);
                __stcg(dst4 + s + 3u * G, a3);
              }
              for (; s < f4; s += G) __stcg(dst4 + s, src4[s]);
              for (s = fit + gl; s < m; s += G) {  // region full: direct (exact)
                const uint32_t u = src[s];
                red_or_g(ldca + (uint64_t)q * P.part_words + (u >> 5), 1u << (u & 31));
              }
              if (gl == 0) {
                cursor[q] = pos + fit;
                cnt[q] = 0;
              }
            }
          }
        }
        __syncthreads();
      }
      if (kSeav) {  // queues restart at parity 0 with the next chunk's slice
        __syncthreads();
        if (tid == 0) sq_cnt[0] = sq_cnt[1] = 0;
      }
      // publish this CTA's run lengths for chunk t and reset the cursors
      for (uint32_t q = tid; q < np; q += kThreads) {
        __stcg(P.counts + ((size_t)b * np + q) * ns + self, cursor[q]);
        cursor[q] = 0;
      }
    }
    grid.sync();  // chunk t produced everywhere; chunk t-1 consumed everywhere
  }
  // fold the shared partition into the global LDCA (after the last barrier
  // no direct reds are in flight, so plain read-modify-write is exact)
  if (!owner) return;
  __syncthreads();
  const uint64_t w0 = (uint64_t)self * P.part_words;
  for (uint32_t i = tid; i < P.part_words; i += kThreads) {
    const uint64_t w = w0 + i;
    if (w < P.total_words && part[i]) ldca[w] |= part[i];
  }
}

static bool bits_fit32(const sspd_params* p) { return (uint64_t)p->lr * p->lc * p->k <= 0xFFFFFFFFull; }

static uint32_t ilog2_ceil(uint64_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  return l;
}

static bool plan_partitioned(const sspd_params* p, uint64_t n, uint64_t chunk, int sms, int max_smem,
                             PartPlan& P, uint64_t& smem, uint64_t& scratch, int& mode) {
  const uint64_t bits = (uint64_t)p->lr * p->lc * p->k;
  const bool pow2_kl = (p->k & (p->k - 1)) == 0 && (p->lc & (p->lc - 1)) == 0 && bits_fit32(p);
  P.total_words = (bits + 31) / 32;
  P.nsrc = (uint32_t)sms;
  auto staging = [&](uint32_t nparts) {
    // expected kTile*lr/nparts per destination per tile + 3-4 sigma, 16-B rows
    const double mean = (double)kTile * p->lr / nparts;
    const double sig = nparts < (uint32_t)sms ? 3.0 : 4.0;
    return ((uint32_t)(mean + sig * __builtin_sqrt(mean) + 8.0) + 3u) & ~3u;
  };
  auto fits = [&](uint32_t nparts, uint32_t pw, uint32_t slots) {
    smem = 4ull * (pw + (uint64_t)nparts * slots + 2ull * nparts + 8 + 4ull * kSeavQueue);
    return (int64_t)smem <= max_smem && pw < (1u << 27);
  };
  mode = pow2_kl ? kFast32 : kGeneric;
  // power-of-two partitions when the LDCA word count is a power of two
  // and the largest power-of-two partition count <= SMs fits in smem
  const uint64_t tw = P.total_words;
  if (pow2_kl && p->lr == 8 && (tw & (tw - 1)) == 0 && getenv("SSPD_PART_NOPOW2") == nullptr) {
    uint32_t np2 = 1;
    while ((uint64_t)np2 * 2 <= (uint64_t)sms) np2 *= 2;
    if (tw >= np2) {
      const uint32_t pw = (uint32_t)(tw / np2);
      const uint32_t slots = staging(np2);
      if (fits(np2, pw, slots)) {
        mode = kPow2;
        P.nparts = np2;
        P.part_words = pw;
        P.stage_slots = slots;
        P.pshift = ilog2_ceil(pw) + 5;
        P.pmask = (uint32_t)((uint64_t)pw * 32 - 1);
      }
    }
  }
  if (mode != kPow2) {
    P.nparts = (uint32_t)sms;
    P.part_words = (uint32_t)(((tw + P.nparts - 1) / P.nparts + 3) & ~3ull);
    P.stage_slots = staging(P.nparts);
    if (!fits(P.nparts, P.part_words, P.stage_slots)) return false;
    P.pshift = 0;
    P.pmask = 0;
  }
  const uint64_t d = P.part_words;
  P.div_part.d = d;
  P.div_part.pad_ = 0;
  if ((d & (d - 1)) == 0) {
    P.div_part.pow2 = 1;
    P.div_part.magic = 0;
    P.div_part.sh1 = P.div_part.sh2 = 0;
  } else {
    const uint32_t l = ilog2_ceil(d);
    const unsigned __int128 num = ((unsigned __int128)1 << 64) * (((unsigned __int128)1 << l) - d);
    P.div_part.magic = (uint64_t)(num / d) + 1;
    P.div_part.sh1 = 1;
    P.div_part.sh2 = l - 1;
    P.div_part.pow2 = 0;
  }
  {  // 32-bit division by part_words (Granlund-Montgomery, N = 32)
    const uint32_t l = ilog2_ceil(d);
    P.magic32 = (d & (d - 1)) == 0 ? 0u : (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
    P.sh32 = l - 1;
  }
  // pure producers (no partition) take a larger slice: consumers also drain
  // their buckets.  Weight ratio (x64) tunable with SSPD_PART_WEIGHT.
  P.w_owner = 64;
  P.w_other = 80;
  if (const char* e = getenv("SSPD_PART_WEIGHT")) P.w_other = (uint32_t)atoi(e);
  // default chunk: 8 tiles per producer (measured best together with w_other = 80),
  // so slices are (nearly) whole tiles
  P.chunk = chunk ? chunk : (uint64_t)P.nsrc * kTile * 8;
  const double share = (double)P.w_other / ((double)P.nparts * P.w_owner + (double)(P.nsrc - P.nparts) * P.w_other);
  const double rmean = (double)P.chunk * p->lr * share / P.nparts;  // largest producer -> one destination
  P.region_cap = (uint32_t)(rmean + 6.0 * __builtin_sqrt(rmean) + 32.0);
  P.region_cap = (P.region_cap + 31u) & ~31u;
  // bucket offsets are 32-bit element indexes
  if (2ull * P.nparts * P.nsrc * P.region_cap >= (1ull << 32)) return false;
  P.qstride = P.nsrc * P.region_cap;
  P.gshift = 0;
  while ((2u << P.gshift) <= 32u && ((kThreads >> (P.gshift + 1)) >= P.nparts)) ++P.gshift;
  if (P.gshift < 2) return false;  // the flush pads runs with up to 3 lanes of a group
  P.n = n;
  scratch = 4ull * (2ull * P.nparts * P.nsrc * P.region_cap + 2ull * P.nparts * P.nsrc);
  P.k_mask = p->k - 1;
  P.lc_mask = p->lc - 1;
  P.log2k = ilog2_ceil(p->k);
  {
    const uint64_t seeds[10] = {p->seed_h3, p->seed_h1, p->seed_lh[0], p->seed_lh[1], p->seed_lh[2],
                                p->seed_lh[3], p->seed_lh[4], p->seed_lh[5], p->seed_lh[6], p->seed_lh[7]};
    for (int i = 0; i < 10; ++i) {
      P.s_lo[i] = (uint32_t)seeds[i];
      P.s_hg[i] = (uint32_t)(seeds[i] >> 32) + (uint32_t)(kGolden >> 32);
    }
  }
  P.qshift = 0;
  if (mode == kPow2) {
    // the cell form of the routing needs whole cells per partition and
    // whole partitions per row
    const uint64_t pbits = 1ull << P.pshift;
    if (P.pshift < P.log2k || ((uint64_t)p->lc << P.log2k) % pbits != 0) {
      mode = kFast32;
    } else {
      P.qshift = P.pshift - P.log2k;
    }
  }
  return true;
}


}  // namespace sspd

using namespace sspd;

// Returns SSPD_ERR_CONFIG when the geometry/device cannot host the
// partitioned scan (the caller then uses the direct kernel).
extern "C" int sspd_scan_partitioned(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p,
                                     uint8_t* seav, uint8_t* ldca, void* scratch, uint64_t scratch_bytes,
                                     uint64_t chunk, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (n == 0) return SSPD_OK;
  if (!hips || !oips || !ldca) return SSPD_ERR_DATA;
  if (scan_bpart_scratch(p, chunk) != 0)
    return scan_bpart_launch(hips, oips, n, p, seav, ldca, scratch, scratch_bytes, chunk, stream);
  int dev = 0, sms = 0, max_smem = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return SSPD_ERR_CONFIG;
  PartPlan P;
  uint64_t smem = 0, need = 0;
  int mode = kGeneric;
  if (!plan_partitioned(p, n, chunk, sms, max_smem, P, smem, need, mode)) return SSPD_ERR_CONFIG;
  if (!scratch || scratch_bytes < need) return SSPD_ERR_CAPACITY;
  P.buckets = static_cast<uint32_t*>(scratch);
  P.counts = P.buckets + 2ull * P.nparts * P.nsrc * P.region_cap;
  P.vec_ok = (((reinterpret_cast<uintptr_t>(hips) | reinterpret_cast<uintptr_t>(oips)) & 15u) == 0 &&
              (P.chunk & 3u) == 0)
                 ? 1u
                 : 0u;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kern = nullptr;
  if (seav)
    kern = mode == kPow2 ? (void*)scan_partitioned_kernel<true, kPow2>
                         : (mode == kFast32 ? (void*)scan_partitioned_kernel<true, kFast32>
                                            : (void*)scan_partitioned_kernel<true, kGeneric>);
  else
    kern = mode == kPow2 ? (void*)scan_partitioned_kernel<false, kPow2>
                         : (mode == kFast32 ? (void*)scan_partitioned_kernel<false, kFast32>
                                            : (void*)scan_partitioned_kernel<false, kGeneric>);
  // the attribute/occupancy answers only change with (kernel, smem, device):
  // cached so a launch costs one driver call (a benign race recomputes)
  static void* c_kern = nullptr;
  static uint64_t c_smem = 0;
  static int c_dev = -1, c_per_sm = 0;
  if (kern != c_kern || smem != c_smem || dev != c_dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    c_kern = kern, c_smem = smem, c_dev = dev, c_per_sm = per_sm;
  }
  if (c_per_sm < 1) return SSPD_ERR_CONFIG;
  const uint32_t* h = hips;
  const uint32_t* o = oips;
  sspd_params pv = *p;
  uint32_t* sv = reinterpret_cast<uint32_t*>(seav);
  uint32_t* lv = reinterpret_cast<uint32_t*>(ldca);
  void* args[] = {(void*)&h, (void*)&o, (void*)&pv, (void*)&P, (void*)&sv, (void*)&lv};
  if (cudaLaunchCooperativeKernel(kern, dim3(P.nsrc), dim3(kThreads), args, smem, st) != cudaSuccess) {
    cudaGetLastError();
    return SSPD_ERR_CUDA;
  }
  return check_launch();
}

// Scratch bytes the partitioned scan needs for a given chunk size (0 when
// the LDCA cannot be partitioned into shared memory on this device).
// sspd_scan_partitioned into an LDCA buffer that holds only zeros (a fresh
// sliding dirty-bitmap slot): K1b's fold then stores instead of
// read-modify-writing.  The result is the same as sspd_scan_partitioned's.
extern "C" int sspd_scan_partitioned_fresh(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                           const sspd_params* p, uint8_t* seav, uint8_t* ldca, void* scratch,
                                           uint64_t scratch_bytes, uint64_t chunk, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (n == 0) return SSPD_OK;
  if (!hips || !oips || !ldca) return SSPD_ERR_DATA;
  if (scan_bpart_scratch(p, chunk) != 0)
    return scan_bpart_launch(hips, oips, n, p, seav, ldca, scratch, scratch_bytes, chunk, stream, true);
  return sspd_scan_partitioned(hips, oips, n, p, seav, ldca, scratch, scratch_bytes, chunk, stream);
}

// Which partitioned scan sspd_scan_partitioned runs for this geometry:
// 2 = K1b (b-axis partitions), 1 = K1p (word-range partitions), 0 = none
// (the LDCA does not fit the SMs' shared memory: SSPD_ERR_CONFIG).
extern "C" int sspd_scan_partitioned_variant(const sspd_params* p, uint64_t chunk) {
  if (!p || validate_params(p)) return 0;
  if (scan_bpart_scratch(p, chunk) != 0) return 2;
  int dev = 0, sms = 148, max_smem = 232448;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
    cudaGetLastError();
    sms = 148;
    max_smem = 232448;
  }
  PartPlan P;
  uint64_t smem = 0, need = 0;
  int mode = 0;
  return plan_partitioned(p, 1, chunk, sms, max_smem, P, smem, need, mode) ? 1 : 0;
}

extern "C" uint64_t sspd_scan_partitioned_scratch(const sspd_params* p, uint64_t chunk) {
  if (!p) return 0;
  if (const uint64_t b = scan_bpart_scratch(p, chunk)) return b;
  int dev = 0, sms = 148, max_smem = 232448;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
    cudaGetLastError();
    sms = 148;
    max_smem = 232448;
  }
  PartPlan P;
  uint64_t smem = 0, need = 0;
  int mode = 0;
  if (!plan_partitioned(p, 1, chunk, sms, max_smem, P, smem, need, mode)) return 0;
  return need;
}
