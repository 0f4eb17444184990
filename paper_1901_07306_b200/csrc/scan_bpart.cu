// K1b: the partitioned scan with the LDCA cut along its b axis.
//
// Same result as K1 (scan.cu) and K1p (scan_smem.cu): bit (i*lc + c_i)*k + b
// of the LDCA with c_i = LH_i(hip) % lc and b = H3(oip) % k
// (long_sketch.py:125-135), plus the SEAV update of short_sketch.py:300-318.
//
// Like K1p, the LDCA lives in the SMs' shared memory for the whole launch
// (one persistent 1,024-thread CTA per SM, cooperative launch, one grid
// barrier per chunk, double-buffered buckets in L2).  The difference is the
// cut.  K1p gives partition q a contiguous word range, so the LR = 8 bits of
// one packet land in 8 different partitions: 8 staged u32 updates, 8 shared
// atomicAdd slot reservations and 32 B of bucket traffic per packet.  K1b
// gives partition q the b range [q*bw, (q+1)*bw) of EVERY cell
// (bw = k / P bits, P = 128 partitions at k = 8192: 64 KB each).  All LR bits
// of a packet share its b, so the packet goes to exactly ONE partition
// q = b / bw as one 16-byte entry:
//
//   eight u16 halves; with w_i = c_i << HB | (b % bw) >> 5 (HB = log2(bw/32))
//   the word of row i inside the partition (rows of rw = lc << HB words):
//     half_0 = w_0 | (b & 31) << log2(rw)        (a word index + the bit)
//     half_i = 4 * (i * rw + w_i), i = 1..7      (shared-memory byte offsets)
//
// which the owner of q turns into 8 shared-memory atomicOr (bit b & 31 of
// word i*rw + w_i of its partition; 8*rw*4 <= 2^16 by plan).  Per packet: one
// shared atomicAdd instead of 8, one 16-byte staging store instead of 8
// scalar ones, 16 B of bucket writes + 16 B of reads instead of 32 + 32.
//
// Anything that does not fit (a destination's staging row or bucket region
// full, e.g. one opposite IP sending a large share of the window) is applied
// as direct L2 `red.or` on the global LDCA -- exact, because OR is
// commutative and idempotent.  SEAV updates (0.78 % of packets at tau = 7)
// are queued per tile and applied by all lanes as direct reds (as K1p).
#include <algorithm>
#include <type_traits>
#include <cooperative_groups.h>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sspd_common.cuh"
#include "launch.cuh"

namespace cg = cooperative_groups;

namespace sspd {
namespace bpart {

constexpr uint32_t kThreads = 1024;
constexpr uint32_t kPkt = 4;  // packets per thread per tile (one uint4 of hips + oips)
constexpr uint32_t kTile = kThreads * kPkt;
constexpr uint32_t kLR = 8;
constexpr uint32_t kSeavQueue = 1024;  // sampled packets per CTA per chunk (expected ~570 at tau = 7)
constexpr uint32_t kMaxSrc = 256;     // producer CTAs (SMs) the plan supports

struct Plan {
  uint32_t nparts;       // partitions = consumer CTAs 0 .. nparts-1 (power of two)
  uint32_t nsrc;         // producers = gridDim.x (>= nparts)
  uint32_t bshift;       // log2(bw): partition of b = b >> bshift
  uint32_t row_words;    // rw = lc << HB: words of one LDCA row inside a partition (<= 2048)
  uint32_t part_words;   // kLR * row_words
  uint32_t lowm;         // rw - 1: half 0 without the bit position
  uint32_t bsh_shift;    // log2(rw): where half 0 keeps b & 31
  uint32_t rowc[4];      // per entry word: the row byte offsets of its halves (4*i*rw << 16*(i&1))
  uint32_t stage_slots;  // 16-B entries per destination per tile (owner CTAs)
  uint32_t stage_slots_pure;  // dbuf: the same for pure producers (their staging takes the partition's room)
  uint32_t dbuf;         // 1: two staging buffers, one producer barrier per tile
  uint32_t cnt_off_words;  // dbuf: shared-memory word offset of cnt[2][nparts]
  uint32_t region_cap;   // entries per (src, dst) region per chunk
  uint32_t w_owner, w_other;  // producer slice weights (owners vs pure producers)
  uint64_t chunk;        // packets per chunk
  uint64_t n;            // packets
  uint4* buckets;        // [2][dst][src][region_cap]
  uint32_t* counts;      // [2][dst][src]
  uint32_t k_mask, lc_mask, log2k, lc;
  uint32_t kw;           // k / 32: words per cell in the global LDCA
  SplitSeed ss[10];     // split seeds (mix64_lo_fast): H3, H1, LH0..7
  uint32_t vec_ok;       // hips/oips 16-byte aligned and chunk % 4 == 0
  uint32_t qstride;      // nsrc * region_cap: bucket entries per destination
  uint32_t gshift;       // log2 of the flush group (threads per destination)
  uint32_t tau_mask;
  uint32_t cons_warps;   // kWarpLdg / kWarpTma: consumer warps of an owner CTA
  uint32_t tma_flush;    // 1: staging runs leave shared memory as TMA bulk stores
  uint32_t dst_zero;     // 1: the LDCA holds only zeros on entry: the fold stores, no read-modify-write
  uint32_t fold_red;     // 1: the fold ORs with red.or (fire and forget), 0: load-OR-store
  uint32_t* ready;       // kWarpFlag: [dst][src] = chunks of src published to dst (zeroed per launch)
  uint32_t* drained;     // kWarpFlag: [dst] = chunks dst has drained
  uint32_t slice_off[kMaxSrc + 1];  // producer s starts at chunk start + slice_off[s] (full chunks)
  // sliding SEAV sink (kSm == 2): u16 stamps of the sampled packets (+ the
  // optional incremental view and slot log), as K2 (scan.cu) writes them
  uint16_t* spool;
  uint32_t snow;
  uint32_t* sview;               // nullptr: no tracking
  uint32_t* slog;
  unsigned long long* slog_head;
  uint32_t slog_mask;
};

__device__ __forceinline__ void red_or_g(uint32_t* addr, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
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

// Sliding SEAV half of one sampled packet (sliding.py:156-185, as K2's
// scan_sliding_u16_fast_kernel): u16 stamp `now` into its SR slots, and with
// tracking the view bit + the slot's log entry at ring position lpos + i.
__device__ __forceinline__ void seav_stamp(const sspd_params& p, const Plan& P, uint32_t hip, uint32_t oip,
                                           unsigned long long lpos) {
  const uint32_t bit = (uint32_t)hash_range(oip, p.seed_h2, p.div_g);
  const uint64_t rp = hip & ((1u << p.r) - 1u);
  const uint64_t lp = ((uint64_t)hip >> p.r) & ((1ull << p.lp_bits) - 1ull);
  for (uint32_t i = 0; i < p.sr; ++i) {
    const uint32_t col = index_of(lp, p.isb[i], p.ibn[i], p.lp_bits);
    const uint64_t reg = rp * p.sc[i] + col;
    const uint64_t slot = p.slot_row_base[i] + reg * p.g + bit;
    P.spool[slot] = (uint16_t)P.snow;
    if (P.sview) {
      const uint64_t vbit = (p.seav_row_off[i] + reg * p.reg_bytes) * 8 + bit;
      atomicOr(P.sview + (vbit >> 5), 1u << (vbit & 31));
      P.slog[(lpos + i) & P.slog_mask] = (uint32_t)slot;
    }
  }
}
__device__ __noinline__ void seav_stamp_ool(const sspd_params& p, const Plan& P, uint32_t hip, uint32_t oip) {
  seav_stamp(p, P, hip, oip, P.sview ? atomicAdd(P.slog_head, (unsigned long long)p.sr) : 0ull);
}

// Staging row full (rare): the packet's LR bits as direct L2 reds (exact).
__device__ __noinline__ void direct_packet(const Plan& P, uint32_t hip, uint32_t b, uint32_t* ldca) {
  for (uint32_t i = 0; i < kLR; ++i) {
    const uint32_t c = mix64_lo_fast(hip, P.ss[2 + i]) & P.lc_mask;
    const uint32_t bit = ((i * P.lc + c) << P.log2k) | b;
    red_or_g(ldca + (bit >> 5), 1u << (bit & 31u));
  }
}

// Bucket region full (rare): decode a staged entry of partition q back to
// its LR bits and apply them as direct L2 reds (exact).
template <int HB>
__device__ __noinline__ void direct_entry(const Plan& P, uint32_t q, uint4 e, uint32_t* ldca) {
  const uint32_t bsh = (e.x >> P.bsh_shift) & 31u;
  const uint32_t h[kLR] = {e.x & P.lowm, e.x >> 16, e.y & 0xFFFFu, e.y >> 16,
                           e.z & 0xFFFFu, e.z >> 16, e.w & 0xFFFFu, e.w >> 16};
  for (uint32_t i = 0; i < kLR; ++i) {
    const uint32_t w = (i ? h[i] >> 2 : h[i]) & (P.row_words - 1u);  // strip the row offset
    const uint32_t c = w >> HB;
    const uint32_t b = (q << P.bshift) | ((w & ((1u << HB) - 1u)) << 5) | bsh;
    const uint32_t bit = ((i * P.lc + c) << P.log2k) | b;
    red_or_g(ldca + (bit >> 5), 1u << (bit & 31u));
  }
}

// ---- TMA bulk-copy pipeline of the consumer warps (kWarpTma) -------------
// One lane of the first consumer warp streams the chunk's bucket regions
// into a ring of kRing shared-memory slots with cp.async.bulk (completion
// on the slot's `full` mbarrier, transaction bytes); the other consumer
// warps OR the entries out of shared memory and release the slot on its
// `empty` mbarrier.  No consumer lane waits on a global load.
constexpr uint32_t kRing = 4;
constexpr uint32_t kSlot = 256;  // entries (16 B) per ring slot

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both 16-B aligned),
// completing `bytes` transactions on mbarrier `b`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// shared -> global bulk copy (TMA store) in this thread's bulk group
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Weighted producer slice of CTA s in [c0, c1): pure producers (s >= nparts)
// take w_other/w_owner as much as owners; boundaries are 4-aligned.  Full
// chunks read the host-computed table (no 64-bit division per chunk).
__device__ __forceinline__ uint64_t slice_start(const Plan& P, uint64_t c0, uint64_t c1, uint32_t s) {
  if (s >= P.nsrc) return c1;
  if (c1 - c0 == P.chunk) return c0 + P.slice_off[s];
  const uint64_t tw = (uint64_t)P.nparts * P.w_owner + (uint64_t)(P.nsrc - P.nparts) * P.w_other;
  const uint64_t cw =
      (uint64_t)min(s, P.nparts) * P.w_owner + (uint64_t)(s > P.nparts ? s - P.nparts : 0) * P.w_other;
  const uint64_t off = (((c1 - c0) * cw) / tw) & ~3ull;
  return min(c1, c0 + off);
}

// Shared memory: [part_words | nparts*stage_slots uint4 staging | nparts cnt |
//                 4 sq_cnt | kSeavQueue (hip, oip) | kWarpTma: kRing*kSlot uint4
//                 ring | 2*kRing mbarriers]
// Warp-specialised owner CTAs (kWarpLdg / kWarpTma): P.cons_warps warps consume chunk t-1
// (the bucket entries into the shared partition: LSU/shared-atomic work)
// while the other warps hash and stage chunk t (ALU/FMA work), so the two
// overlap instead of alternating; the producers synchronise on named
// barrier 1.  Pure-producer CTAs (no partition) hash with all warps.
// Consumer modes: kInline = every warp drains chunk t-1, then produces;
// kWarpLdg = P.cons_warps warps drain with 16-B global loads (4 in flight
// per lane) while the rest produce (default: 4.60 vs 4.80 ms per config-2
// window); kWarpTma = the same split, fed by TMA bulk copies into a
// shared-memory ring (1 issuing lane + draining warps; bit-exact but
// measured slower on B200: 6.3-6.9 ms -- the 16 KB ring the shared-memory
// budget leaves keeps too few bytes in flight); kWarpFlag = kWarpLdg with
// the per-chunk grid barrier replaced by point-to-point release/acquire
// flags (ready[dst][src] per published chunk, drained[dst] per drained
// chunk; producers wait only before reusing a bucket buffer) -- bit-exact,
// 4.23 vs 4.19 ms: the barrier share of the stall samples is the drain's
// pace, not the barrier itself.
enum : int { kInline = 0, kWarpLdg = 1, kWarpTma = 2, kWarpFlag = 3 };
#ifndef SSPD_BPART_DIAG  // timing diagnostics (tools builds only): 1 drain w/o atomics, 2 no staging,
                         // 4 no per-tile barriers, 8 no SEAV sampling, 16 no drain
#define SSPD_BPART_DIAG 0
#endif
#ifndef SSPD_BPART_DRAIN_LOADS
#define SSPD_BPART_DRAIN_LOADS 4
#endif
constexpr uint32_t kConsWarpsLdg = 8;  // measured: 4 -> 5.48 ms, 6 -> 4.70, 8 -> 4.60, 10 -> 4.75
constexpr uint32_t kConsWarpsTma = 6;

template <int kSm, int HB, int kCons>
__global__ void __launch_bounds__(kThreads, 1)
    scan_bpart_kernel(const uint32_t* __restrict__ hips, const uint32_t* __restrict__ oips,
                      const __grid_constant__ sspd_params p, const __grid_constant__ Plan P, uint32_t* seav,
                      uint32_t* ldca) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* part = smem;
  const bool owner = blockIdx.x < P.nparts;
  // staging: [part | stage[np][S]] or, double-buffered (P.dbuf), owners
  // [part | stage[2][np][S_o]] and pure producers [stage[2][np][S_p]] (no
  // partition), cnt[2][np] at a common offset
  uint4* const stage = reinterpret_cast<uint4*>(smem + (P.dbuf && !owner ? 0u : P.part_words));
  const uint32_t slots = P.dbuf && !owner ? P.stage_slots_pure : P.stage_slots;
  uint32_t* cnt = P.dbuf ? smem + P.cnt_off_words
                         : reinterpret_cast<uint32_t*>(stage + (size_t)P.nparts * P.stage_slots);
  uint32_t* sq_cnt = cnt + (P.dbuf ? 2u : 1u) * P.nparts;  // [1] (+3 pad); nparts % 4 == 0
  uint2* sq_base = reinterpret_cast<uint2*>(sq_cnt + 4);  // [kSeavQueue]
  uint4* ring = reinterpret_cast<uint4*>(sq_base + kSeavQueue);  // kWarpTma: [kRing][kSlot]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(ring + kRing * kSlot);
  uint64_t* empty_bar = full_bar + kRing;
  cg::grid_group grid = cg::this_grid();
  const uint32_t self = blockIdx.x;
  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31, warp = tid >> 5, nwarps = kThreads >> 5;
  const uint32_t np = P.nparts, ns = P.nsrc;
  constexpr uint32_t kHMask = (1u << HB) - 1u;
  // producer threads of this CTA and their tile (packets per tile barrier)
  constexpr bool kSpec = kCons != kInline;
  const uint32_t nprod = (kSpec && owner) ? kThreads - 32u * P.cons_warps : kThreads;
  const bool producer = tid < nprod;
  const uint32_t tile = nprod * kPkt;
  auto pbar = [&]() {  // the producers' barrier
    if (SSPD_BPART_DIAG & 4) return;  // timing diagnostic: no per-tile barriers
    if (kSpec)
      asm volatile("bar.sync 1, %0;" ::"r"(nprod) : "memory");
    else
      __syncthreads();
  };

  for (uint32_t i = tid; i < P.part_words; i += kThreads) part[i] = 0;
  for (uint32_t i = tid; i < (P.dbuf ? 2u : 1u) * np; i += kThreads) cnt[i] = 0;
  // flush role, fixed for the launch: group q = tid >> gshift of G threads
  // copies destination q's staging row (one pass covers every destination)
  uint32_t gs = P.gshift;
  while (gs && (nprod >> gs) < np) --gs;
  const uint32_t G = 1u << gs, gl = tid & (G - 1u), fq = tid >> gs;
  const bool flusher = producer && fq < np;
  if (tid == 0) sq_cnt[0] = 0;
  if (kCons == kWarpTma && tid == 0) {
    for (uint32_t r = 0; r < kRing; ++r) {
      mbar_init(full_bar + r, 1);                     // the issuing lane's expect_tx
      mbar_init(empty_bar + r, P.cons_warps - 1u);    // every draining warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t ring_s = 0, ring_ph = 0;  // consumer pipeline position (kept across chunks)
  uint32_t tb = 0;                   // dbuf: the staging buffer of the current tile (kept across chunks)
#if SSPD_BPART_DIAG
  uint32_t diag = 0;
#endif

  const uint64_t nchunks = (P.n + P.chunk - 1) / P.chunk;
  for (uint64_t t = 0; t <= nchunks; ++t) {
    // ---------------- consume chunk t-1 into the shared partition --------
    if (kCons == kWarpTma && t >= 1 && owner && !producer) {
      // TMA-fed drain of chunk t-1: consumer warp 0 issues, warps 1.. OR
      const uint32_t cw = warp - nprod / 32u, nk = P.cons_warps - 1u;
      const uint32_t bb = (uint32_t)((t - 1) & 1);
      const uint32_t* cnts = P.counts + ((size_t)bb * np + self) * ns;
      const uint4* regions = P.buckets + ((size_t)bb * np + self) * (size_t)P.qstride;
      const uint32_t lowm = P.lowm, bss = P.bsh_shift;
      char* const pb = reinterpret_cast<char*>(part);
      if (cw == 0) {
        if (lane == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");  // peers' bucket stores -> TMA reads
          for (uint32_t src = 0; src < ns; ++src) {
            const uint32_t m = min(__ldcg(cnts + src), P.region_cap);
            const uint4* reg = regions + (size_t)src * P.region_cap;
            for (uint32_t off = 0; off < m; off += kSlot) {
              const uint32_t len = min(kSlot, m - off);
              mbar_wait(empty_bar + ring_s, ring_ph ^ 1u);
              mbar_expect_tx(full_bar + ring_s, len * 16u);
              bulk_g2s(ring + ring_s * kSlot, reg + off, len * 16u, full_bar + ring_s);
              if (++ring_s == kRing) ring_s = 0, ring_ph ^= 1u;
            }
          }
        }
        __syncwarp();
      } else {
        const uint32_t k = cw - 1u;
        for (uint32_t src = 0; src < ns; ++src) {
          const uint32_t m = min(__ldcg(cnts + src), P.region_cap);
          for (uint32_t off = 0; off < m; off += kSlot) {
            const uint32_t len = min(kSlot, m - off);
            mbar_wait(full_bar + ring_s, ring_ph);
            const uint4* slot = ring + ring_s * kSlot;
            for (uint32_t e = k * 32u + lane; e < len; e += nk * 32u) {
              const uint4 u = slot[e];
              const uint32_t bit = 1u << ((u.x >> bss) & 31u);
              atomicOr(part + (u.x & lowm), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (u.x >> 16)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (u.y & 0xFFFFu)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (u.y >> 16)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (u.z & 0xFFFFu)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (u.z >> 16)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (u.w & 0xFFFFu)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (u.w >> 16)), bit);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_bar + ring_s);
            if (++ring_s == kRing) ring_s = 0, ring_ph ^= 1u;
          }
          if (k == 0) {  // the region is dead once read: drop its L2 lines without write-back
            const uint4* reg = regions + (size_t)src * P.region_cap;
            for (uint32_t line = lane; line * 8 < m; line += 32)
              asm volatile("discard.global.L2 [%0], 128;" ::"l"(reg + line * 8) : "memory");
          }
        }
      }
    }
    if (kCons != kWarpTma && t >= 1 && owner && !producer == kSpec) {
      const uint32_t cw = kSpec ? warp - nprod / 32u : warp;  // draining warp index
      const uint32_t ncw = kSpec ? P.cons_warps : nwarps;
      const uint32_t bb = (uint32_t)((t - 1) & 1);
      const uint32_t* cnts = P.counts + ((size_t)bb * np + self) * ns;
      const uint4* regions = P.buckets + ((size_t)bb * np + self) * (size_t)P.qstride;
      const uint32_t lowm = P.lowm, bss = P.bsh_shift;
      char* const pb = reinterpret_cast<char*>(part);
      // warp w drains sources w, w+W, ...: lane j holds the run length of
      // source w+W*j, fetched at once so no region waits on its count
      for (uint32_t src0 = cw; src0 < ((SSPD_BPART_DIAG & 16) ? 0u : ns); src0 += 32u * ncw) {
      const uint32_t my_src = src0 + ncw * lane;
      if (kCons == kWarpFlag && my_src < ns) {  // chunk t-1 of this source published to us?
        const uint32_t* f = P.ready + (size_t)self * ns + my_src;
        while (ld_acquire(f) < (uint32_t)t) __nanosleep(64);
      }
      const uint32_t my_cnt = my_src < ns ? min(__ldcg(cnts + my_src), P.region_cap) : 0u;
      for (uint32_t src = src0, j = 0; src < ns && j < 32u; src += ncw, ++j) {
        const uint32_t m = __shfl_sync(0xffffffffu, my_cnt, j);
        const uint4* reg = regions + (size_t)src * P.region_cap;  // 128-B aligned
        // kInFlight independent 16-B loads in flight per lane (8 measured
        // 5.4 vs 4.2 ms: the kernel's 64-register budget is shared with the
        // producers, which then spill)
        constexpr int kInFlight = kSpec ? SSPD_BPART_DRAIN_LOADS : 4;
        for (uint32_t j0 = lane; j0 < m; j0 += 32 * kInFlight) {
          uint4 u[kInFlight];
#pragma unroll
          for (int g = 0; g < kInFlight; ++g)
            if (j0 + 32 * g < m) u[g] = __ldcg(reg + j0 + 32 * g);
#pragma unroll
          for (int g = 0; g < kInFlight; ++g) {
            if (j0 + 32 * g < m) {
              const uint4 e = u[g];
#if SSPD_BPART_DIAG & 1
              diag ^= e.x ^ e.y ^ e.z ^ e.w;  // timing diagnostic: drain without the shared atomics
              continue;
#endif
              const uint32_t bit = 1u << ((e.x >> bss) & 31u);
              atomicOr(part + (e.x & lowm), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (e.x >> 16)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (e.y & 0xFFFFu)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (e.y >> 16)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (e.z & 0xFFFFu)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (e.z >> 16)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (e.w & 0xFFFFu)), bit);
              atomicOr(reinterpret_cast<uint32_t*>(pb + (e.w >> 16)), bit);
            }
          }
        }
        // the region is dead once read: drop its L2 lines without write-back
        // so the bucket exchange stays on chip
        __syncwarp();
        for (uint32_t line = lane; line * 8 < m; line += 32)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(reg + line * 8) : "memory");
      }
      }
    }
    if (kCons == kWarpFlag && t >= 1 && owner && !producer) {
      // every draining warp is done reading chunk t-1's buckets: tell the
      // producers that buffer (t-1)&1 may be overwritten
      asm volatile("bar.sync 2, %0;" ::"r"(kThreads - nprod) : "memory");
      if (tid == nprod) st_release(P.drained + self, (uint32_t)t);
    }
    // ---------------- produce chunk t ------------------------------------
    if (t < nchunks && producer) {
      const uint32_t bb = (uint32_t)(t & 1);
      if (kCons == kWarpFlag && t >= 2) {
        // buffer bb last held chunk t-2: every destination must have drained it
        if (warp == 0) {
          for (uint32_t q0 = 0; q0 < np; q0 += 32) {
            const uint32_t q = q0 + lane;
            if (q < np)
              while (ld_acquire(P.drained + q) < (uint32_t)(t - 1)) __nanosleep(64);
          }
          __syncwarp();
        }
        pbar();
      }
      const uint64_t c0 = t * P.chunk;
      const uint64_t c1 = min(P.n, c0 + P.chunk);
      const uint64_t lo = slice_start(P, c0, c1, self);
      const uint64_t hi = slice_start(P, c0, c1, self + 1);
      // thread tid owns packets base + 4 tid + e, fetched one tile ahead
      // with one 16-byte streaming load per array when aligned
      auto fetch = [&](uint64_t first, uint32_t* h, uint32_t* o) {
        if (P.vec_ok && first + kPkt <= hi) {
          const uint4 hv = __ldcs(reinterpret_cast<const uint4*>(hips + first));
          const uint4 ov = __ldcs(reinterpret_cast<const uint4*>(oips + first));
          h[0] = hv.x, h[1] = hv.y, h[2] = hv.z, h[3] = hv.w;
          o[0] = ov.x, o[1] = ov.y, o[2] = ov.z, o[3] = ov.w;
        } else {
#pragma unroll
          for (uint32_t e = 0; e < kPkt; ++e) {
            h[e] = first + e < hi ? __ldcs(hips + first + e) : 0u;
            o[e] = first + e < hi ? __ldcs(oips + first + e) : 0u;
          }
        }
      };
      // this thread's flush destination: region (self -> fq) of bucket bb,
      // filled up to `pos` (identical in the G lanes of the group)
      uint4* const dstq = P.buckets + ((size_t)bb * np + fq) * P.qstride + (size_t)self * P.region_cap;
      uint32_t pos = 0;
      uint32_t nh[kPkt], no[kPkt];
      fetch(lo + (uint64_t)tid * kPkt, nh, no);
      // one tile; TB = its staging buffer (compile-time: the buffer offsets fold
      // into the addresses); single-buffered launches always use buffer 0
      auto tile_body = [&](uint64_t base, auto tb_c) {
        constexpr uint32_t TB = decltype(tb_c)::value;
        uint32_t ch[kPkt], co[kPkt];
#pragma unroll
        for (uint32_t e = 0; e < kPkt; ++e) {
          ch[e] = nh[e];
          co[e] = no[e];
        }
        fetch(base + tile + (uint64_t)tid * kPkt, nh, no);
#pragma unroll
        for (uint32_t e = 0; e < kPkt; ++e) {
          const uint64_t j = base + (uint64_t)tid * kPkt + e;
          const uint32_t hip = ch[e], oip = co[e];
          if (j < hi) {
            const uint32_t b = mix64_lo_fast(oip, P.ss[0]) & P.k_mask;
            const uint32_t q = b >> P.bshift;
            const uint32_t bhi = (b >> 5) & kHMask;
            // the word bits shared by all halves (half 0: word index, 1..7: byte offsets)
            const uint32_t both = (bhi << 2) * 0x10001u;
            uint32_t c[kLR];
#pragma unroll
            for (uint32_t i = 0; i < kLR; ++i) c[i] = mix64_lo_fast(hip, P.ss[2 + i]) & P.lc_mask;
            uint4 ent;
            ent.x = (c[0] << HB) + bhi + ((b & 31u) << P.bsh_shift) + c[1] * (1u << (18 + HB)) + (both & 0xFFFF0000u) +
                    P.rowc[0];
            ent.y = c[2] * (1u << (2 + HB)) + c[3] * (1u << (18 + HB)) + (both + P.rowc[1]);
            ent.z = c[4] * (1u << (2 + HB)) + c[5] * (1u << (18 + HB)) + (both + P.rowc[2]);
            ent.w = c[6] * (1u << (2 + HB)) + c[7] * (1u << (18 + HB)) + (both + P.rowc[3]);
#if SSPD_BPART_DIAG & 2
            diag ^= ent.x ^ ent.y ^ ent.z ^ ent.w ^ q;  // timing diagnostic: no staging
#else
            const uint32_t slot = atomicAdd(&cnt[TB * np + q], 1u);
            if (slot < slots)
              stage[(TB * np + q) * slots + slot] = ent;
            else
              direct_entry<HB>(P, q, ent, ldca);  // staging row full: direct (exact)
#endif
            if (kSm && !(SSPD_BPART_DIAG & 8) && (mix64_lo_fast(oip, P.ss[1]) & P.tau_mask) == 0u) {
              const uint32_t qs = atomicAdd(sq_cnt, 1u);
              if (qs < kSeavQueue)
                sq_base[qs] = make_uint2(hip, oip);
              else if (kSm == 1)
                seav_update_ool(p, hip, oip, seav);  // queue full (a skewed slice): apply now
              else
                seav_stamp_ool(p, P, hip, oip);
            }
          }
        }
        // dbuf: the previous tile's bulk copies (out of the other buffer,
        // which the next tile writes) must have read shared memory before
        // this barrier releases the producers
        if (P.dbuf && flusher && gl == 0) bulk_wait_read();
        pbar();
        const uint4* const srcq = stage + (TB * np + fq) * slots;
        uint32_t* const cntq = cnt + TB * np + fq;
        // flush: the G = 2^gshift threads of group fq copy destination fq's
        // run of 16-B entries into this CTA's own region of that bucket (no
        // global atomics); `pos` lives in registers, identical in the group
        if (P.tma_flush) {
          // one TMA bulk store per destination run (its lane group's lane 0);
          // the run must have been read out of shared memory before the next
          // tile's staging writes: wait_group.read ahead of the barrier
          if (flusher && gl == 0) {
            const uint32_t m = min(*cntq, slots);
            const uint32_t fit = pos < P.region_cap ? min(m, P.region_cap - pos) : 0u;
            if (fit) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging writes -> TMA reads
              bulk_s2g(dstq + pos, srcq, fit * 16u);
              bulk_commit();
            }
            for (uint32_t s2 = fit; s2 < m; ++s2) direct_entry<HB>(P, fq, srcq[s2], ldca);  // region full (exact)
            pos += fit;
            *cntq = 0;
            if (!P.dbuf) bulk_wait_read();
          }
          if (flusher) pos = __shfl_sync(__activemask(), pos, 0, G);  // keep the group's copies equal
        } else if (flusher) {
          const uint32_t m = min(*cntq, slots);
          const uint32_t fit = pos < P.region_cap ? min(m, P.region_cap - pos) : 0u;
          uint4* dst = dstq + pos;
          uint32_t s = gl;
          for (; s + G < fit; s += 2u * G) {  // 2 shared loads in flight, then 2 stores
            const uint4 a0 = srcq[s], a1 = srcq[s + G];
            __stcg(dst + s, a0);
            __stcg(dst + s + G, a1);
          }
          if (s < fit) __stcg(dst + s, srcq[s]);
          for (s = fit + gl; s < m; s += G) direct_entry<HB>(P, fq, srcq[s], ldca);  // region full (exact)
          pos += fit;
          __syncwarp();  // the group's lanes read cnt[fq] before it is reset
          if (gl == 0) *cntq = 0;
        }
        if (!P.dbuf) pbar();
      };
      for (uint64_t base = lo; base < hi;) {
        if (tb == 0 || !P.dbuf) {
          tile_body(base, std::integral_constant<uint32_t, 0>{});
        } else {
          tile_body(base, std::integral_constant<uint32_t, 1>{});
        }
        tb ^= P.dbuf;
        base += tile;
      }
      if (kSm) {
        // the slice's sampled packets (0.78 % at tau = 7), queued per chunk
        // and applied here by consecutive producer lanes (full warps): a
        // per-tile pass left one warp updating while the others waited at
        // the tile barrier (-0.3 ms per config-2 window).  Sliding stamps
        // with tracking reserve the chunk's log run with one atomic.
        pbar();
        const uint32_t nq = min(sq_cnt[0], kSeavQueue);
        unsigned long long* lbase = reinterpret_cast<unsigned long long*>(sq_cnt + 2);
        if (kSm == 2 && P.sview) {
          if (tid == 0) *lbase = nq ? atomicAdd(P.slog_head, (unsigned long long)nq * p.sr) : 0ull;
          pbar();
        }
        for (uint32_t i = tid; i < nq; i += nprod) {
          if (kSm == 1)
            seav_update(p, sq_base[i].x, sq_base[i].y, seav);
          else
            seav_stamp(p, P, sq_base[i].x, sq_base[i].y, P.sview ? *lbase + (unsigned long long)i * p.sr : 0ull);
        }
        pbar();
        if (tid == 0) sq_cnt[0] = 0;
      }
      // publish this CTA's run lengths for chunk t
      if (flusher && gl == 0) {
        if (P.tma_flush) {  // the bulk stores must be complete and visible before the grid barrier
          bulk_wait_all();
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __stcg(P.counts + ((size_t)bb * np + fq) * ns + self, pos);
        if (kCons == kWarpFlag) st_release(P.ready + (size_t)fq * ns + self, (uint32_t)(t + 1));
      }
    }
    // chunk t produced everywhere; chunk t-1 consumed everywhere -- or, with
    // point-to-point flags, only before the fold.  No barrier after the last
    // drain when the fold is a red.or: it commutes with every other CTA's
    // direct reds, so each owner folds as soon as its own drain is done
    if (t < nchunks ? kCons != kWarpFlag : !P.fold_red) grid.sync();
  }
  // fold the partition into the global LDCA: word (row, cell, j) of
  // partition q is global word (row*lc + cell)*k/32 + q*2^HB + j.  After the
  // last barrier no direct reds are in flight and the partitions are
  // disjoint, so a fire-and-forget red.or is exact (with
  // SSPD_BPART_FOLD_RED=0, after a last grid barrier: a load-OR-store, or
  // into an all-zero destination -- a fresh sliding dirty bitmap -- a plain
  // store).  Each CTA
  // starts its walk at a different cell (rotated by part_words / nparts
  // words): the 2^HB words of one cell that the partitions own share 128-B
  // lines, and walking in lockstep sent all owners to the same lines at once
  // (a 1.8 M-packet launch spent ~40 of its 110 us in this loop, as
  // load-OR-store round trips queued on those lines).
#if SSPD_BPART_DIAG
  if (diag == 0x9E3779B9u) ldca[tid] = diag;  // keep the diagnostic work alive
#endif
  if (!owner) return;
  __syncthreads();
  const uint32_t rshift = 31 - __clz(P.row_words);  // row_words is a power of two
  const uint32_t rot = self * (P.part_words / P.nparts), wmask = P.part_words - 1u;
  for (uint32_t k = tid; k < P.part_words; k += kThreads) {
    const uint32_t i = (k + rot) & wmask;
    const uint32_t v = part[i];
    if (v) {
      const uint32_t row = i >> rshift, within = i & (P.row_words - 1u);
      const uint64_t cell = (uint64_t)row * P.lc + (within >> HB);
      uint32_t* dst = ldca + cell * P.kw + ((uint64_t)self << HB) + (within & kHMask);
      if (P.fold_red)
        red_or_g(dst, v);
      else if (P.dst_zero)
        __stcg(dst, v);
      else
        *dst |= v;
    }
  }
}

static uint32_t ilog2_exact(uint64_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  return l;
}

// Plan for the b-axis partitioned scan; false when the geometry or device
// cannot host it (the caller then uses K1p or K1).
static bool plan(const sspd_params* p, uint64_t n, uint64_t chunk, int sms, int max_smem, Plan& P, uint64_t& smem,
                 uint64_t& scratch, int& hb, int& cons) {
  const bool pow2 = (p->k & (p->k - 1)) == 0 && (p->lc & (p->lc - 1)) == 0;
  if (p->lr != kLR || !pow2 || (uint64_t)p->lr * p->lc * p->k > 0xFFFFFFFFull) return false;
  if (getenv("SSPD_PART_LEGACY") != nullptr) return false;
  uint32_t np = 1;
  while ((uint64_t)np * 2 <= (uint64_t)sms) np *= 2;
  while (np > 1 && p->k / np < 32) np >>= 1;  // >= one word of b per cell and partition
  if (np < 16 || p->k / np < 32) return false;
  const uint32_t bw = p->k / np;
  hb = (int)ilog2_exact(bw / 32);
  if (hb > 3) return false;  // kernels are instantiated for 32..256 b values per cell
  const uint32_t log2lc = ilog2_exact(p->lc);
  if (log2lc + hb > 11) return false;  // 8 rows of rw <= 2048 words: byte offsets fit a u16 half
  if (sms > (int)kMaxSrc) return false;
  P.nparts = np;
  P.nsrc = (uint32_t)sms;
  P.bshift = ilog2_exact(bw);
  P.row_words = p->lc << hb;
  P.part_words = kLR * P.row_words;
  P.bsh_shift = log2lc + hb;
  P.lowm = (1u << P.bsh_shift) - 1u;
  for (uint32_t w = 0; w < 4; ++w)
    P.rowc[w] = (w ? (4u * (2 * w) * P.row_words) : 0u) | ((4u * (2 * w + 1) * P.row_words) << 16);
  {  // staging per destination per tile: mean kTile/np + 4 sigma + 8
    const double mean = (double)kTile / np;
    P.stage_slots = (uint32_t)(mean + 4.0 * __builtin_sqrt(mean) + 8.0);
  }
  P.stage_slots_pure = P.stage_slots;
  P.dbuf = 0;
  P.cnt_off_words = 0;
  smem = 4ull * P.part_words + 16ull * np * P.stage_slots + 4ull * np + 16 + 8ull * kSeavQueue;
  // consumer mode (SSPD_BPART_CONS = 0 in line / 1 warp-specialised, global
  // loads (default) / 2 warp-specialised, TMA ring)
  // producer tiles per chunk: 16 measured best on B200 (fewer grid barriers
  // outweigh the part of the bucket exchange that then spills from L2)
  uint32_t tiles = 16;
  if (const char* e = getenv("SSPD_BPART_TILES")) tiles = (uint32_t)atoi(e) > 0 ? (uint32_t)atoi(e) : 16;
  P.chunk = chunk ? ((chunk + 3) & ~3ull) : (uint64_t)P.nsrc * kTile * tiles;
  if (P.chunk >= (1ull << 32)) return false;  // slice offsets are 32-bit
  cons = kWarpLdg;
  // a single-chunk launch (a sliding slice, a small batch) has no chunk to
  // drain while the next is produced: every warp produces, then drains
  // (config-4 slice: 66 vs 73 us)
  if (n <= P.chunk) cons = kInline;
  if (const char* e = getenv("SSPD_BPART_CONS")) cons = std::min(3, std::max(0, atoi(e)));
  P.cons_warps = cons == kWarpTma ? kConsWarpsTma : kConsWarpsLdg;
  if (const char* e = getenv("SSPD_BPART_CONS_WARPS")) P.cons_warps = (uint32_t)std::min(16, std::max(2, atoi(e)));
  const uint64_t ring_bytes = 16ull * kRing * kSlot + 16ull * kRing;  // TMA ring + full/empty mbarriers
  if (cons == kWarpTma && (int64_t)(smem + ring_bytes) > max_smem) cons = kWarpLdg;  // no room for the ring
  if (cons == kWarpTma) smem += ring_bytes;
  if ((int64_t)smem > max_smem) return false;
  const bool spec = cons != kInline;
  // staging runs leave shared memory as TMA bulk stores (default; 4.36 vs
  // 4.65 ms per config-2 window: no per-entry LDS/STG, no short-scoreboard
  // stalls in the flush) or as 16-B stores by 2^gshift threads each
  P.tma_flush = 1;
  if (const char* e = getenv("SSPD_BPART_FLUSH_TMA")) P.tma_flush = atoi(e) != 0;
  if (cons == kWarpFlag && !P.tma_flush) cons = kWarpLdg;  // flags are released by the one flushing lane
  // double-buffered staging (warp-specialised TMA-flush launches): the
  // flush of tile t overlaps the staging of tile t+1, one producer barrier
  // per tile instead of two.  Two buffers fit because the rows are sized to
  // each role's tile -- owners stage (1024 - 32 * cons_warps) * 4 packets
  // per tile, pure producers 4,096 but hold no partition -- with a 2.5-3
  // sigma margin (a full row sends the entry straight to L2, exact)
  if (cons == kWarpLdg && P.tma_flush && !(getenv("SSPD_BPART_DB") && atoi(getenv("SSPD_BPART_DB")) == 0)) {
    const double mo = (double)(kThreads - 32u * P.cons_warps) * kPkt / np, mp = (double)kTile / np;
    const uint64_t tail = 4ull * 2 * np + 16 + 8ull * kSeavQueue;
    const int64_t room_o = (int64_t)max_smem - (int64_t)tail - 4ll * P.part_words;
    uint32_t so = (uint32_t)(mo + 3.0 * __builtin_sqrt(mo) + 2.0);
    uint32_t sp = (uint32_t)(mp + 3.0 * __builtin_sqrt(mp) + 2.0);
    if (room_o > 0) so = std::min<uint32_t>(so, (uint32_t)(room_o / (32ll * np)));
    sp = std::min<uint32_t>(sp, (uint32_t)(((int64_t)max_smem - (int64_t)tail) / (32ll * np)));
    const uint64_t end_o = 4ull * P.part_words + 32ull * np * so, end_p = 32ull * np * sp;
    const uint64_t cnt_off = (std::max(end_o, end_p) + 15) & ~15ull;
    if (room_o > 0 && so >= mo + 2.0 * __builtin_sqrt(mo) && sp >= mp + 2.5 * __builtin_sqrt(mp) &&
        cnt_off + tail <= (uint64_t)max_smem) {
      P.dbuf = 1;
      P.stage_slots = so;
      P.stage_slots_pure = sp;
      P.cnt_off_words = (uint32_t)(cnt_off / 4);
      smem = cnt_off + tail;
    }
  }
  // producer slice weights: pure producers hash with all 32 warps; owners
  // with 28 (spec) or pause to consume (in line)
  P.w_owner = 64;
  // measured with the TMA flush, 16-tile chunks: 64-70 -> 4.27 ms, 72-73 ->
  // 4.18, 74-76 -> 4.30-4.35, 82 -> 4.58 (slices are whole tiles, so the
  // optimum is a step, not a slope)
  // in line (one chunk: everybody produces, then the owners drain) equal
  // slices are best -- a 1.8 M-packet launch: 80 -> 54.6 us, 64 -> 49.1
  P.w_other = spec ? 72 : 64;
  if (const char* e = getenv("SSPD_PART_WEIGHT")) P.w_other = (uint32_t)atoi(e);
  // the largest producer's share of a chunk -- over the weights of BOTH
  // consumer modes, so the scratch size a caller queries (which cannot know
  // the batch size, and plans one chunk in line) covers every launch
  auto share_of = [&](uint32_t wo) {
    return (double)std::max(P.w_owner, wo) / ((double)np * P.w_owner + (double)(P.nsrc - np) * wo);
  };
  const double share = std::max({share_of(P.w_other), share_of(72), share_of(64)});
  const double rmean = (double)P.chunk * share / np;  // largest producer -> one destination
  P.region_cap = (uint32_t)(rmean + 6.0 * __builtin_sqrt(rmean) + 32.0);
  P.region_cap = (P.region_cap + 7u) & ~7u;  // regions start on 128-B lines
  P.qstride = P.nsrc * P.region_cap;
  if (2ull * np * P.qstride >= (1ull << 32)) return false;
  P.gshift = 0;  // one pass of the flush covers every destination: np << gshift <= kThreads
  while ((2u << P.gshift) <= 32u && ((kThreads >> (P.gshift + 1)) >= np)) ++P.gshift;
  {  // producer slice offsets inside a full chunk (slice_start)
    const uint64_t tw = (uint64_t)np * P.w_owner + (uint64_t)(P.nsrc - np) * P.w_other;
    for (uint32_t sidx = 0; sidx <= P.nsrc; ++sidx) {
      const uint64_t cw = (uint64_t)std::min(sidx, np) * P.w_owner + (uint64_t)(sidx > np ? sidx - np : 0) * P.w_other;
      P.slice_off[sidx] = (uint32_t)std::min<uint64_t>(P.chunk, ((P.chunk * cw) / tw) & ~3ull);
    }
  }
  P.n = n;
  // [buckets | counts | ready flags [np][ns] | drained flags [np]]
  scratch = 16ull * 2 * np * P.qstride + 4ull * 2 * np * P.nsrc + 4ull * np * P.nsrc + 4ull * np;
  P.k_mask = p->k - 1;
  P.lc_mask = p->lc - 1;
  P.log2k = ilog2_exact(p->k);
  P.lc = p->lc;
  P.kw = p->k / 32;
  P.tau_mask = tau_mask(p->tau);
  const uint64_t seeds[10] = {p->seed_h3,    p->seed_h1,    p->seed_lh[0], p->seed_lh[1], p->seed_lh[2],
                              p->seed_lh[3], p->seed_lh[4], p->seed_lh[5], p->seed_lh[6], p->seed_lh[7]};
  for (int i = 0; i < 10; ++i) P.ss[i] = split_seed(seeds[i]);
  return true;
}

template <int kSm, int kCons>
static void* kernel_hb(int hb) {
  switch (hb) {
    case 0: return (void*)scan_bpart_kernel<kSm, 0, kCons>;
    case 1: return (void*)scan_bpart_kernel<kSm, 1, kCons>;
    case 2: return (void*)scan_bpart_kernel<kSm, 2, kCons>;
    default: return (void*)scan_bpart_kernel<kSm, 3, kCons>;
  }
}

template <int kSm>
static void* kernel_for(int hb, int cons) {
  if (kSm == 2) return cons == kInline ? kernel_hb<2, kInline>(hb) : kernel_hb<2, kWarpLdg>(hb);
  switch (cons) {
    case kWarpTma: return kernel_hb<kSm == 2 ? 0 : kSm, kWarpTma>(hb);
    case kWarpLdg: return kernel_hb<kSm, kWarpLdg>(hb);
    case kWarpFlag: return kernel_hb<kSm == 2 ? 0 : kSm, kWarpFlag>(hb);
    default: return kernel_hb<kSm, kInline>(hb);
  }
}

static void device_limits(int& dev, int& sms, int& max_smem) {
  dev = 0;
  sms = 148;
  max_smem = 232448;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
    cudaGetLastError();
    sms = 148;
    max_smem = 232448;
  }
  // A/B knob: fewer CTAs than SMs (the rest stay free for kernels of other
  // streams while the cooperative scan runs)
  if (const char* e = getenv("SSPD_BPART_GRID")) sms = std::max(16, std::min(sms, atoi(e)));
}

}  // namespace bpart

// Scratch bytes of the b-axis partitioned scan (0 = not applicable).
uint64_t scan_bpart_scratch(const sspd_params* p, uint64_t chunk) {
  int dev, sms, max_smem;
  bpart::device_limits(dev, sms, max_smem);
  bpart::Plan P;
  uint64_t smem = 0, need = 0;
  int hb = 0;
  int cons = 0;
  if (!bpart::plan(p, 1, chunk, sms, max_smem, P, smem, need, hb, cons)) return 0;
  return need;
}

// Launch; SSPD_ERR_CONFIG when not applicable (the caller tries K1p).
int scan_bpart_launch(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p, uint8_t* seav,
                      uint8_t* ldca, void* scratch, uint64_t scratch_bytes, uint64_t chunk, void* stream,
                      bool dst_zero, const SlideSeavSink* slide) {
  int dev, sms, max_smem, coop = 0;
  bpart::device_limits(dev, sms, max_smem);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return SSPD_ERR_CONFIG;
  bpart::Plan P;
  uint64_t smem = 0, need = 0;
  int hb = 0;
  int cons = 0;
  if (!bpart::plan(p, n, chunk, sms, max_smem, P, smem, need, hb, cons)) return SSPD_ERR_CONFIG;
  if (!scratch || scratch_bytes < need) return SSPD_ERR_CAPACITY;
  P.spool = nullptr, P.snow = 0, P.sview = nullptr, P.slog = nullptr, P.slog_head = nullptr, P.slog_mask = 0;
  if (slide) {
    P.spool = slide->pool, P.snow = slide->now, P.sview = slide->view, P.slog = slide->log;
    P.slog_head = slide->log_head, P.slog_mask = slide->log_mask;
    if (cons != bpart::kInline) cons = bpart::kWarpLdg;
  }
  P.dst_zero = dst_zero ? 1u : 0u;
  P.fold_red = !(getenv("SSPD_BPART_FOLD_RED") && atoi(getenv("SSPD_BPART_FOLD_RED")) == 0);
  P.buckets = static_cast<uint4*>(scratch);
  P.counts = reinterpret_cast<uint32_t*>(P.buckets + 2ull * P.nparts * P.qstride);
  P.ready = P.counts + 2ull * P.nparts * P.nsrc;
  P.drained = P.ready + (uint64_t)P.nparts * P.nsrc;
  if (cons == bpart::kWarpFlag &&
      cudaMemsetAsync(P.ready, 0, 4ull * P.nparts * (P.nsrc + 1), static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return SSPD_ERR_CUDA;
  P.vec_ok = (((reinterpret_cast<uintptr_t>(hips) | reinterpret_cast<uintptr_t>(oips)) & 15u) == 0 &&
              (P.chunk & 3u) == 0)
                 ? 1u
                 : 0u;
  void* kern = slide ? bpart::kernel_for<2>(hb, cons) : seav ? bpart::kernel_for<1>(hb, cons) : bpart::kernel_for<0>(hb, cons);
  // attribute/occupancy answers only change with (kernel, smem, device)
  static void* c_kern = nullptr;
  static uint64_t c_smem = 0;
  static int c_dev = -1, c_per_sm = 0;
  if (kern != c_kern || smem != c_smem || dev != c_dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, bpart::kThreads, smem);
    c_kern = kern, c_smem = smem, c_dev = dev, c_per_sm = per_sm;
  }
  if (c_per_sm < 1) return SSPD_ERR_CONFIG;
  const uint32_t* h = hips;
  const uint32_t* o = oips;
  sspd_params pv = *p;
  uint32_t* sv = reinterpret_cast<uint32_t*>(seav);
  uint32_t* lv = reinterpret_cast<uint32_t*>(ldca);
  void* args[] = {(void*)&h, (void*)&o, (void*)&pv, (void*)&P, (void*)&sv, (void*)&lv};
  if (cudaLaunchCooperativeKernel(kern, dim3(P.nsrc), dim3(bpart::kThreads), args, smem,
                                  static_cast<cudaStream_t>(stream)) != cudaSuccess) {
    cudaGetLastError();
    return SSPD_ERR_CUDA;
  }
  return check_launch();
}


}  // namespace sspd

using namespace sspd;

// One pass of a sliding slice (u16 stamps): the LDCA half into the slice's
// dirty bitmap (K1b's fold, `dirty_fresh`: the bitmap holds only zeros) and
// the SEAV half -- stamps of the sampled packets, with the optional view and
// slot log -- applied from K1b's per-chunk sampled-packet queue.  The same
// state as sspd_scan_partitioned(_fresh)(seav = NULL, ldca = dirty) followed
// by sspd_scan_sliding_seav, in one launch instead of two (the second
// re-read the slice and re-hashed every packet for its 0.78 % sample).
// SSPD_ERR_CONFIG when K1b does not apply (the caller uses the two calls).
extern "C" int sspd_scan_sliding_partitioned(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                             const sspd_params* p, void* pool, uint32_t ts_bytes,
                                             uint64_t now_wrapped, uint8_t* seav_view, uint32_t* log,
                                             uint64_t log_entries, unsigned long long* log_head, uint8_t* dirty,
                                             int dirty_fresh, void* scratch, uint64_t scratch_bytes, uint64_t chunk,
                                             void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (ts_bytes != 2) return SSPD_ERR_CONFIG;
  if (n == 0) return SSPD_OK;
  if (!hips || !oips || !pool || !dirty) return SSPD_ERR_DATA;
  SlideSeavSink sink{static_cast<uint16_t*>(pool), (uint32_t)(now_wrapped & 0xFFFFu), nullptr, nullptr, nullptr, 0u};
  if (seav_view) {
    if (!log || !log_head || log_entries == 0 || (log_entries & (log_entries - 1)) || log_entries > (1ull << 32) ||
        (reinterpret_cast<uintptr_t>(seav_view) & 3u) || p->slot_total >= (1ull << 32))
      return SSPD_ERR_DATA;
    sink.view = reinterpret_cast<uint32_t*>(seav_view);
    sink.log = log;
    sink.log_head = log_head;
    sink.log_mask = (uint32_t)(log_entries - 1);
  }
  if (scan_bpart_scratch(p, chunk) == 0) return SSPD_ERR_CONFIG;
  return scan_bpart_launch(hips, oips, n, p, nullptr, dirty, scratch, scratch_bytes, chunk, stream, dirty_fresh != 0,
                           &sink);
}
