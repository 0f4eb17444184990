// End-of-window estimate path: K5 restore, candidate sort, K6 filter,
// report compaction.
//
// Reference: SeavSketch.restore_sea / restore   short_sketch.py:347-408
//            LdcaSketch.union_register/estimate long_sketch.py:137-148
//            DetectorState.finalize_window      window_detector.py:105-125
//
// Restore on the device.  One CTA owns one register array (SEA, index rp).
// The reference walks rows depth-first and prunes a partial tuple as soon
// as a row's column disagrees with already-fixed left-part (LP) bits
// (`(acc_lp ^ v) & acc_mask & mask`, short_sketch.py:379-388).  The set of
// LP positions that are already fixed when row i is reached,
//     fixed_i = (mask_0 | ... | mask_{i-1}) & mask_i,
// does not depend on the path, so the CTA buckets row i's hot columns by
// their bits on fixed_i (counting sort in shared memory).  A walk then
// reads exactly the consistent columns of each row as one contiguous
// bucket -- no rejected candidates are ever visited.  Rows 0 and 1 are
// flattened into one balanced work list (a prefix sum over row-0 entries
// of their row-1 bucket sizes); deeper rows are walked with an explicit
// stack.
//
// Cap semantics (short_sketch.py:373-376, 398-407): `survivors` counts
// every complete consistent tuple, whatever its AND weight; more than `cap`
// of them drops the whole SEA.  A tuple is one-to-one with an LP whose
// registers are all hot, so the count is order-independent: pass 1 counts
// (stopping early once the shared total exceeds cap), pass 2 emits the
// weight >= 3 tuples only for SEAs that did not overflow.
#include <cooperative_groups.h>
#include <cooperative_groups/details/partitioning.h>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <cuda_runtime.h>
#include "sspd_common.cuh"
#include "launch.cuh"

namespace cg = cooperative_groups;

namespace sspd {

struct RestorePlan {
  uint32_t sr, w, r, reg_bytes;
  uint32_t full_bits_lo, full_bits_hi;  // (1<<g)-1
  uint32_t isb[SSPD_MAX_SR], ibn[SSPD_MAX_SR], sc[SSPD_MAX_SR];
  uint32_t keymask[SSPD_MAX_SR];  // column bits that sit on fixed_i
  uint32_t nk[SSPD_MAX_SR];       // popcount(keymask)
  uint32_t off_regs[SSPD_MAX_SR], off_cols[SSPD_MAX_SR], off_bstart[SSPD_MAX_SR];
  uint32_t off_pref0, off_misc, smem_bytes, hshift;
  uint64_t seav_row_off[SSPD_MAX_SR];
  uint32_t* hist;  // optional: per-bucket candidate counts (bucket = ip >> hshift) for the bucket sort
  // one-load staging of a whole SEA by a warp (g = 8 one-byte registers,
  // rows of multiples of 8 bytes, <= 256 bytes per SEA, e.g. r = 16): lane l
  // loads 8 bytes of row lane_row[l] at byte lane_off[l] (lane_row >= sr: idle)
  uint32_t lane_fast;
  uint32_t row_lanes[SSPD_MAX_SR];  // ballot mask of the lanes holding row i
  uint8_t lane_row[32], lane_off[32];
  // ... and, when every row has <= 64 registers, the tuples are enumerated
  // straight from per-row hot-column masks (no bucket tables) as long as
  // their number is <= kEnumMax and <= cap
  uint32_t lane_enum, enum_max;
  uint32_t row_lane0[SSPD_MAX_SR];  // first lane of row i
  uint32_t row_bits[SSPD_MAX_SR];   // LP positions row i fixes (row_mask), w <= 32
  uint32_t rows8;  // enumeration with every row 64 registers = 8 aligned lanes (SR <= 4)
};

__device__ __forceinline__ uint32_t pext32(uint32_t x, uint32_t m) {
  uint32_t r = 0, bb = 1;
  while (m) {
    const uint32_t low = m & (0u - m);
    if (x & low) r |= bb;
    bb <<= 1;
    m &= m - 1;
  }
  return r;
}

__device__ __forceinline__ uint64_t load_reg(const uint8_t* base, uint32_t idx, uint32_t rb) {
  switch (rb) {
    case 1: return base[idx];
    case 2: return reinterpret_cast<const uint16_t*>(base)[idx];
    case 4: return reinterpret_cast<const uint32_t*>(base)[idx];
    default: return reinterpret_cast<const uint64_t*>(base)[idx];
  }
}

// Shared-memory copy of the plan fields the warp path indexes by lane or by
// walk depth: indexed constant-bank loads with lane-divergent indices are
// serialised (ncu: ADU pipe 80 % busy), shared-memory loads are not.
struct WarpTab {
  uint64_t lane_src[32];  // seav_row_off[row] + lane_off of the lane's 8 bytes
  uint32_t lane_sc[32];   // sc[row] (the SEA stride of the lane's row); 0 = idle lane
  uint32_t lane_dst[32];  // off_regs[row] + lane_off (staging offset)
  uint32_t isb[SSPD_MAX_SR], ibn[SSPD_MAX_SR], sc[SSPD_MAX_SR], keymask[SSPD_MAX_SR], off_regs[SSPD_MAX_SR];
  uint32_t off_bstart[SSPD_MAX_SR], off_cols[SSPD_MAX_SR], row_lane0[SSPD_MAX_SR];
};

// Enumeration path (warp kernel only): ctab[i][x] = the columns of row i
// (<= 64) whose bits on keymask[i] equal x's (x = the walk's LP bits at row
// i, masked to keymask[i] < 64) -- col_match() as one shared-memory load.
struct EnumTab {
  uint64_t ctab[SSPD_MAX_SR][64];
  uint32_t scol[SSPD_MAX_SR][64];  // scatter_col(c, row i): column c's LP bits (w <= 32)
  uint32_t rd[SSPD_MAX_SR];        // row descriptor: isb | ibn << 8 | keymask << 16
  uint32_t wmask;                  // (1 << w) - 1
};

__device__ __forceinline__ uint64_t col_match(uint32_t km, uint32_t v, uint32_t sc);

__device__ void fill_enum_tab(const RestorePlan& P, EnumTab* E) {
  if (!P.lane_enum) return;
  for (uint32_t x = threadIdx.x; x < P.sr * 64u; x += blockDim.x) {
    const uint32_t i = x >> 6, c = x & 63;
    E->ctab[i][c] = col_match(P.keymask[i], c, P.sc[i]);
    E->scol[i][c] = c < P.sc[i] ? (uint32_t)scatter_col(c, P.isb[i], P.ibn[i], P.w) : 0u;
  }
  if (threadIdx.x < P.sr) E->rd[threadIdx.x] = P.isb[threadIdx.x] | P.ibn[threadIdx.x] << 8 | P.keymask[threadIdx.x] << 16;
  if (threadIdx.x == 0) E->wmask = P.w >= 32 ? 0xFFFFFFFFu : ((1u << P.w) - 1u);
}

// index_of on a w <= 32 bit LP, masked to the row's key bits: the ctab row
// index of the columns consistent with lp at row `rd`
__device__ __forceinline__ uint32_t key32(uint32_t lp, uint32_t rd, uint32_t w, uint32_t wmask) {
  const uint32_t isb = rd & 255u;
  const uint32_t rot = isb == 0 ? lp : (((lp >> isb) | (lp << (w - isb))) & wmask);
  return rot & (rd >> 16);  // keymask bits lie inside the column's ibn bits
}

__device__ void fill_warp_tab(const RestorePlan& P, WarpTab* T) {
  const uint32_t t = threadIdx.x;
  if (t < 32) {
    if (!P.lane_fast) return;
    const uint32_t row = P.lane_row[t];
    const bool act = row < P.sr;
    T->lane_src[t] = act ? P.seav_row_off[row] + P.lane_off[t] : 0;
    T->lane_sc[t] = act ? P.sc[row] : 0u;
    T->lane_dst[t] = act ? P.off_regs[row] + P.lane_off[t] : 0u;
  } else if (t < 32 + P.sr) {
    const uint32_t i = t - 32;
    T->isb[i] = P.isb[i];
    T->ibn[i] = P.ibn[i];
    T->sc[i] = P.sc[i];
    T->keymask[i] = P.keymask[i];
    T->off_regs[i] = P.off_regs[i];
    T->off_bstart[i] = P.off_bstart[i];
    T->off_cols[i] = P.off_cols[i];
    T->row_lane0[i] = P.row_lane0[i];
  }
}

struct Misc {
  unsigned long long total;  // consistent complete tuples counted so far
  uint32_t abort;
  uint32_t pairs;
  uint32_t hot[SSPD_MAX_SR];
  uint8_t hmask[32];  // one-load path: per-lane hot-byte masks (8 registers each)
  unsigned long long rmask[SSPD_MAX_SR];  // ... assembled per row (enumeration path)
};

// In-place exclusive scan of a[0..m) by one warp; returns the total.
__device__ uint32_t warp_exclusive_scan(uint32_t* a, uint32_t m) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < m; base += 32) {
    const uint32_t i = base + lane;
    const uint32_t v = i < m ? a[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (i < m) a[i] = carry + x - v;
    carry += __shfl_sync(0xFFFFFFFFu, x, 31);
  }
  return carry;
}

// Emit one candidate (weight >= 3 already checked by the caller): the lanes
// emitting together take one slot range from the shared counter.
__device__ __forceinline__ void emit_candidate(const RestorePlan& P, uint64_t lp, uint32_t rp, uint32_t wgt,
                                               uint32_t* out_ip, uint32_t* out_aux, uint64_t out_capacity,
                                               unsigned long long* out_count) {
  cg::coalesced_group g = cg::coalesced_threads();
  unsigned long long base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(out_count, (unsigned long long)g.size());
  const unsigned long long slot = g.shfl(base, 0) + g.thread_rank();
  if (slot < out_capacity) {
    const uint32_t ip = (uint32_t)((lp << P.r) | rp);
    out_ip[slot] = ip;
    out_aux[slot] = (rp << 8) | wgt;
    if (P.hist) atomicAdd(P.hist + (ip >> P.hshift), 1u);
  }
}

// Columns c < sc (<= 64) whose bits on `km` equal those of v: per bit j of
// km, intersect with the columns whose bit j is v's bit j.
__device__ __forceinline__ uint64_t col_match(uint32_t km, uint32_t v, uint32_t sc) {
  constexpr uint64_t kBit[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull, 0xF0F0F0F0F0F0F0F0ull,
                                0xFF00FF00FF00FF00ull, 0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
  uint64_t m = sc >= 64 ? ~0ull : ((1ull << sc) - 1ull);
#pragma unroll
  for (uint32_t j = 0; j < 6; ++j)
    if ((km >> j) & 1u) m &= ((v >> j) & 1u) ? kBit[j] : ~kBit[j];
  return m;
}

// k-th (0-based) set bit of a 64-bit mask (k < popcount(m))
__device__ __forceinline__ uint32_t nth_bit64(uint64_t m, uint32_t k) {
  const uint32_t lo = (uint32_t)m, nlo = __popc(lo);
  return k < nlo ? __fns(lo, 0, (int)k + 1) : 32u + __fns((uint32_t)(m >> 32), 0, (int)(k - nlo) + 1);
}

// the same by popcount halving: ~20 ALU ops, where __fns is a loop
__device__ __forceinline__ uint32_t select64(uint64_t m, uint32_t k) {
  uint32_t pos = 0, c = __popc((uint32_t)m);
  if (k >= c) k -= c, m >>= 32, pos = 32;
  uint32_t x = (uint32_t)m;
  c = __popc(x & 0xFFFFu);
  if (k >= c) k -= c, x >>= 16, pos += 16;
  c = __popc(x & 0xFFu);
  if (k >= c) k -= c, x >>= 8, pos += 8;
  c = __popc(x & 0xFu);
  if (k >= c) k -= c, x >>= 4, pos += 4;
  c = __popc(x & 0x3u);
  if (k >= c) k -= c, x >>= 2, pos += 2;
  return pos + (k >= (x & 1u) ? 1u : 0u);
}

// Candidates of the enumeration path are staged per warp in shared memory
// and leave with ONE global counter atomic per flush (a warp restores many
// SEAs): per-candidate-group atomics on the single shared counter were
// round trips to one L2 slice that every emitting lane waited on.
constexpr uint32_t kEmitBuf = 128;
struct EmitBuf {
  uint32_t n;
  uint32_t ip[kEmitBuf], aux[kEmitBuf];
};

__device__ __forceinline__ void emit_buffered(const RestorePlan& P, EmitBuf* eb, uint64_t lp, uint32_t rp,
                                              uint32_t wgt, uint32_t* out_ip, uint32_t* out_aux,
                                              uint64_t out_capacity, unsigned long long* out_count) {
  const uint32_t ip = (uint32_t)((lp << P.r) | rp), aux = (rp << 8) | wgt;
  const uint32_t pos = atomicAdd(&eb->n, 1u);
  if (pos < kEmitBuf) {
    eb->ip[pos] = ip;
    eb->aux[pos] = aux;
    return;
  }
  const unsigned long long slot = atomicAdd(out_count, 1ull);  // buffer full (rare): straight out
  if (slot < out_capacity) {
    out_ip[slot] = ip;
    out_aux[slot] = aux;
    if (P.hist) atomicAdd(P.hist + (ip >> P.hshift), 1u);
  }
}

// whole warp, converged: write the staged candidates out once there are at
// least `thresh` of them
__device__ __forceinline__ void flush_emit(const RestorePlan& P, EmitBuf* eb, uint32_t thresh, uint32_t* out_ip,
                                           uint32_t* out_aux, uint64_t out_capacity,
                                           unsigned long long* out_count) {
  __syncwarp();
  const uint32_t n = eb->n;
  if (n < thresh || n == 0) return;
  const uint32_t lane = threadIdx.x & 31, m = min(n, kEmitBuf);
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(out_count, (unsigned long long)m);
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  for (uint32_t i = lane; i < m; i += 32) {
    const unsigned long long slot = base + i;
    if (slot < out_capacity) {
      const uint32_t ip = eb->ip[i];
      out_ip[slot] = ip;
      out_aux[slot] = eb->aux[i];
      if (P.hist) atomicAdd(P.hist + (ip >> P.hshift), 1u);
    }
  }
  __syncwarp();
  if (lane == 0) eb->n = 0;
  __syncwarp();
}

template <bool kEmit>
__device__ void restore_walk(const RestorePlan& P, uint8_t* sm, uint32_t rp, uint64_t cap, uint32_t* out_ip,
                             uint32_t* out_aux, uint64_t out_capacity, unsigned long long* out_count,
                             uint32_t gtid, uint32_t gsize, const WarpTab* T) {
  Misc* misc = reinterpret_cast<Misc*>(sm + P.off_misc);
  const uint32_t* pref0 = reinterpret_cast<const uint32_t*>(sm + P.off_pref0);
  const uint32_t npairs = misc->pairs;
  const uint32_t h0 = misc->hot[0];
  const uint64_t full_bits = ((uint64_t)P.full_bits_hi << 32) | P.full_bits_lo;
  const uint32_t sr = P.sr, w = P.w;
  const uint16_t* cols0 = reinterpret_cast<const uint16_t*>(sm + T->off_cols[0]);
  const uint16_t* cols1 = reinterpret_cast<const uint16_t*>(sm + T->off_cols[1]);
  const uint32_t* b1 = reinterpret_cast<const uint32_t*>(sm + T->off_bstart[1]);

  uint64_t since_flush = 0;
  volatile uint32_t* abort_flag = &misc->abort;

  for (uint32_t t = gtid; t < npairs; t += gsize) {
    if (!kEmit && *abort_flag) break;
    // locate the row-0 entry owning pair t: last j with pref0[j] <= t
    uint32_t lo = 0, hi = h0;  // pref0 has h0+1 entries, pref0[h0] = npairs
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (pref0[mid] <= t) lo = mid; else hi = mid;
    }
    const uint32_t j0 = lo;
    const uint32_t c0 = cols0[j0];
    const uint64_t v0 = scatter_col(c0, T->isb[0], T->ibn[0], w);
    const uint32_t key1 = pext32(index_of(v0, T->isb[1], T->ibn[1], w) & T->keymask[1], T->keymask[1]);
    const uint32_t c1 = cols1[b1[key1] + (t - pref0[j0])];
    const uint64_t v1 = scatter_col(c1, T->isb[1], T->ibn[1], w);
    uint64_t lp_stack[SSPD_MAX_SR];
    uint64_t and_stack[SSPD_MAX_SR];
    uint32_t lo_stack[SSPD_MAX_SR], hi_stack[SSPD_MAX_SR];
    const uint64_t and01 = full_bits & load_reg(sm + T->off_regs[0], c0, P.reg_bytes) &
                           load_reg(sm + T->off_regs[1], c1, P.reg_bytes);
    const uint64_t lp01 = v0 | v1;

    auto leaf = [&](uint64_t lp, uint64_t acc_and) {
      if (kEmit) {
        const uint32_t wgt = (uint32_t)__popcll(acc_and);
        // warp-aggregated slot reservation: the lanes that reach a leaf
        // together take one global atomic (a single counter is shared by
        // every SEA, so per-candidate atomics would serialise at L2)
        cg::coalesced_group leaves = cg::coalesced_threads();
        const cg::coalesced_group keep = cg::binary_partition(leaves, wgt >= 3);
        if (wgt >= 3) {
          unsigned long long base = 0;
          if (keep.thread_rank() == 0) base = atomicAdd(out_count, (unsigned long long)keep.size());
          const unsigned long long slot = keep.shfl(base, 0) + keep.thread_rank();
          if (slot < out_capacity) {
            const uint32_t ip = (uint32_t)((lp << P.r) | rp);
            out_ip[slot] = ip;
            out_aux[slot] = (rp << 8) | wgt;
            if (P.hist) atomicAdd(P.hist + (ip >> P.hshift), 1u);
          }
        }
      } else {
        if (++since_flush == 64) {
          const unsigned long long before = atomicAdd(&misc->total, since_flush);
          since_flush = 0;
          if (before + 64 > cap) *abort_flag = 1u;
        }
      }
    };

    if (sr == 2) {
      leaf(lp01, and01);
      continue;
    }
    // explicit-stack walk over rows 2 .. sr-1
    uint32_t lvl = 2;
    lp_stack[2] = lp01;
    and_stack[2] = and01;
    {
      const uint32_t* bs = reinterpret_cast<const uint32_t*>(sm + T->off_bstart[2]);
      const uint32_t key = pext32(index_of(lp01, T->isb[2], T->ibn[2], w) & T->keymask[2], T->keymask[2]);
      lo_stack[2] = bs[key];
      hi_stack[2] = bs[key + 1];
    }
    while (true) {
      if (lo_stack[lvl] < hi_stack[lvl]) {
        const uint16_t* cols = reinterpret_cast<const uint16_t*>(sm + T->off_cols[lvl]);
        const uint32_t c = cols[lo_stack[lvl]++];
        const uint64_t nlp = lp_stack[lvl] | scatter_col(c, T->isb[lvl], T->ibn[lvl], w);
        const uint64_t nand = and_stack[lvl] & load_reg(sm + T->off_regs[lvl], c, P.reg_bytes);
        if (lvl + 1 == sr) {
          leaf(nlp, nand);
          if (!kEmit && *abort_flag) break;
        } else {
          ++lvl;
          lp_stack[lvl] = nlp;
          and_stack[lvl] = nand;
          const uint32_t* bs = reinterpret_cast<const uint32_t*>(sm + T->off_bstart[lvl]);
          const uint32_t key =
              pext32(index_of(nlp, T->isb[lvl], T->ibn[lvl], w) & T->keymask[lvl], T->keymask[lvl]);
          lo_stack[lvl] = bs[key];
          hi_stack[lvl] = bs[key + 1];
        }
      } else {
        if (--lvl < 2) break;
      }
    }
  }
  if (!kEmit && since_flush) {
    const unsigned long long before = atomicAdd(&misc->total, since_flush);
    if (before + since_flush > cap) *abort_flag = 1u;
  }
}

// A "group" restores one SEA: the whole CTA (large arrays) or one warp
// (small arrays, e.g. r=16 with 256 registers per SEA, where a CTA per SEA
// would spend its life in barriers).  Only the synchronisation differs.
template <bool kWarp>
struct Group {
  uint32_t tid, size, warp, nwarps;
  __device__ __forceinline__ void sync() const {
    if (kWarp)
      __syncwarp();
    else
      __syncthreads();
  }
  __device__ __forceinline__ bool any(bool v) const {
    if (kWarp) return __any_sync(0xFFFFFFFFu, v);
    return __syncthreads_or(v) != 0;
  }
};

template <bool kWarp>
__device__ void restore_sea_group(const uint8_t* __restrict__ seav, const RestorePlan& P, uint8_t* sm, uint32_t rp,
                                  uint32_t slot, uint64_t cap, uint32_t* out_ip, uint32_t* out_aux,
                                  uint64_t out_capacity, unsigned long long* out_count, uint8_t* overflow,
                                  const Group<kWarp> G, const WarpTab* T, uint64_t pre = 0,
                                  EmitBuf* eb = nullptr, const EnumTab* E = nullptr) {
  Misc* misc = reinterpret_cast<Misc*>(sm + P.off_misc);
  const uint32_t sr = P.sr;

  // fast reject: a row without a hot register admits no complete tuple
  // (short_sketch.py:360-361), so the SEA has no candidates and no
  // survivors (it cannot overflow either).  Most SEAs of a large, sparse
  // SEAV end here without touching shared memory.
  bool staged = false;
  if (kWarp && P.lane_fast) {
    // the whole SEA in ONE independent 8-byte load per lane (instead of a
    // dependent round trip per row, which is what a restore co-running with
    // the L2-atomic-bound sliding scan waits on); hot = a byte of weight >= 3
    // (loaded by the caller one SEA ahead: `pre`)
    const bool act = T->lane_sc[G.tid] != 0;
    const uint64_t v = pre;
    uint64_t c = v - ((v >> 1) & 0x5555555555555555ull);
    c = (c & 0x3333333333333333ull) + ((c >> 2) & 0x3333333333333333ull);
    c = (c + (c >> 4)) & 0x0F0F0F0F0F0F0F0Full;                      // per-byte popcounts (<= 8)
    const bool hot = act && ((c + 0x7D7D7D7D7D7D7D7Dull) & 0x8080808080808080ull) != 0;  // some byte >= 3
    const uint32_t hb = __ballot_sync(0xFFFFFFFFu, hot);
    for (uint32_t i = 0; i < sr; ++i)
      if ((hb & P.row_lanes[i]) == 0) return;
    if (act) *reinterpret_cast<uint64_t*>(sm + T->lane_dst[G.tid]) = v;
    staged = true;
    if (P.lane_enum) {
      // per-row hot-column masks: lane l's 8 hot bits are bits lane_off..+7
      // of its row's mask (bytes in lane order = little-endian mask bytes)
      const uint64_t hb8 = ((c + 0x7D7D7D7D7D7D7D7Dull) >> 7) & 0x0101010101010101ull;
      const uint32_t hbyte = act ? (uint32_t)((hb8 * 0x0102040810204080ull) >> 56) : 0u;
      uint64_t tuples = 1;
      if (P.rows8) {
        // row i = lanes 8i .. 8i+7: OR the bytes within each 8-lane group
        uint64_t x = (uint64_t)hbyte << (8 * (G.tid & 7));
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 1);
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 2);
        x |= __shfl_xor_sync(0xFFFFFFFFu, x, 4);
        if ((G.tid & 7) == 0 && (G.tid >> 3) < sr) misc->rmask[G.tid >> 3] = x;
        const uint32_t pc = (uint32_t)__popcll(x);
        uint32_t t32 = 1;  // <= 64^4
        for (uint32_t i = 0; i < sr; ++i) t32 *= __shfl_sync(0xFFFFFFFFu, pc, 8 * i);
        tuples = t32;
        __syncwarp();
      } else {
        misc->hmask[G.tid] = (uint8_t)hbyte;
        __syncwarp();
        if (G.tid < sr) {
          uint64_t m = 0;
          for (uint32_t j = 0; j < (T->sc[G.tid] >> 3); ++j)
            m |= (uint64_t)misc->hmask[T->row_lane0[G.tid] + j] << (8 * j);
          misc->rmask[G.tid] = m;
        }
        __syncwarp();
        for (uint32_t i = 0; i < sr && tuples <= cap; ++i) tuples *= (uint64_t)__popcll(misc->rmask[i]);
      }
      if (tuples <= cap && tuples <= P.enum_max) {
        // every complete tuple is one LP, so the survivors (<= tuples) cannot
        // exceed the cap: no counting pass.  Depth-first walk straight from
        // the hot masks: lane t takes the t-th hot column of row 0; at row i
        // the consistent hot columns are hot_i & (columns whose bits on the
        // already-fixed LP positions equal the walk's) -- the prune of
        // short_sketch.py:379-388 as one 64-bit mask, no bucket tables
        const uint32_t hot0_lo = (uint32_t)misc->rmask[0], hot0_hi = (uint32_t)(misc->rmask[0] >> 32);
        const uint32_t lane = G.tid, w = P.w, wmask = E->wmask;
        const uint8_t* reg0 = sm + T->off_regs[0];
        const uint8_t* reg1 = sm + T->off_regs[1];
        const uint32_t rd1 = E->rd[1];
        const uint64_t hot1 = misc->rmask[1];
        // the walk is spread over consistent (row-0, row-1) PAIRS, not row-0
        // columns: a SEA with few hot row-0 columns but many pairs (a busy
        // late-trace SEA) keeps all 32 lanes walking.  Row-0 columns lane and
        // lane + 32 and the sizes of their consistent hot row-1 sets (a cold
        // column counts 0):
        auto row1_of = [&](uint32_t c0) { return hot1 & E->ctab[1][key32(E->scol[0][c0], rd1, w, wmask)]; };
        const uint32_t cnt_a = (hot0_lo >> lane) & 1u ? (uint32_t)__popcll(row1_of(lane)) : 0u;
        const uint32_t cnt_b = (hot0_hi >> lane) & 1u ? (uint32_t)__popcll(row1_of(lane + 32)) : 0u;
        uint32_t inc_a = cnt_a, inc_b = cnt_b;  // inclusive prefixes over columns 0..63
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t ya = __shfl_up_sync(0xFFFFFFFFu, inc_a, o), yb = __shfl_up_sync(0xFFFFFFFFu, inc_b, o);
          if (lane >= (uint32_t)o) inc_a += ya, inc_b += yb;
        }
        inc_b += __shfl_sync(0xFFFFFFFFu, inc_a, 31);
        const uint32_t npairs = __shfl_sync(0xFFFFFFFFu, inc_b, 31);
        auto incl_at = [&](uint32_t j) {  // every lane takes part (per-lane source j)
          const uint32_t a = __shfl_sync(0xFFFFFFFFu, inc_a, j & 31), b = __shfl_sync(0xFFFFFFFFu, inc_b, j & 31);
          return j < 32 ? a : b;
        };
        auto emit = [&](uint32_t lp, uint32_t a) {
          const uint32_t wgt = (uint32_t)__popc(a);
          if (wgt >= 3) emit_buffered(P, eb, lp, rp, wgt, out_ip, out_aux, out_capacity, out_count);
        };
        // rows 2 and 3 (the reference default SR = 4) walked in registers
        const uint64_t hot2 = sr > 2 ? misc->rmask[2] : 0ull, hot3 = sr > 3 ? misc->rmask[3] : 0ull;
        const uint32_t rd2 = sr > 2 ? E->rd[2] : 0u, rd3 = sr > 3 ? E->rd[3] : 0u;
        for (uint32_t base = 0; base < npairs; base += 32) {
          const uint32_t t = base + lane;
          // row-0 column of pair t: the first j with incl(j) > t
          uint32_t lo = 0, hi = 63;
#pragma unroll
          for (int it = 0; it < 6; ++it) {
            const uint32_t mid = (lo + hi) >> 1;
            if (incl_at(mid) > t) hi = mid; else lo = mid + 1;
          }
          const uint32_t c0 = lo;
          const uint32_t excl = incl_at(c0 == 0 ? 0 : c0 - 1);
          if (t >= npairs) continue;
          const uint32_t c1 = select64(row1_of(c0), t - (c0 == 0 ? 0u : excl));
          const uint32_t lp1 = E->scol[0][c0] | E->scol[1][c1];
          const uint32_t and1 = (uint32_t)reg0[c0] & reg1[c1];
          if (sr == 2) {
            emit(lp1, and1);
            continue;
          }
          if (sr == 4) {
            const uint8_t* reg2 = sm + T->off_regs[2];
            const uint8_t* reg3 = sm + T->off_regs[3];
            for (uint64_t rem2 = hot2 & E->ctab[2][key32(lp1, rd2, w, wmask)]; rem2; rem2 &= rem2 - 1) {
              const uint32_t c2 = (uint32_t)__ffsll((long long)rem2) - 1;
              const uint32_t lp2 = lp1 | E->scol[2][c2];
              const uint32_t and2 = and1 & reg2[c2];
              for (uint64_t rem3 = hot3 & E->ctab[3][key32(lp2, rd3, w, wmask)]; rem3; rem3 &= rem3 - 1) {
                const uint32_t c3 = (uint32_t)__ffsll((long long)rem3) - 1;
                emit(lp2 | E->scol[3][c3], and2 & reg3[c3]);
              }
            }
            continue;
          }
          // any other SR: explicit-stack walk over rows 2 .. sr-1
          uint32_t lp_st[SSPD_MAX_SR], and_st[SSPD_MAX_SR];
          uint64_t rem_st[SSPD_MAX_SR];
          lp_st[1] = lp1;
          and_st[1] = and1;
          uint32_t lvl = 2;
          rem_st[2] = hot2 & E->ctab[2][key32(lp1, rd2, w, wmask)];
          while (lvl >= 2) {
            const uint64_t rem = rem_st[lvl];
            if (rem == 0) {
              --lvl;
              continue;
            }
            const uint32_t c = (uint32_t)__ffsll((long long)rem) - 1;
            rem_st[lvl] = rem & (rem - 1);
            const uint32_t nlp = lp_st[lvl - 1] | E->scol[lvl][c];
            const uint32_t nand = and_st[lvl - 1] & sm[T->off_regs[lvl] + c];
            if (lvl + 1 == sr) {
              emit(nlp, nand);
              continue;
            }
            lp_st[lvl] = nlp;
            and_st[lvl] = nand;
            ++lvl;
            rem_st[lvl] = misc->rmask[lvl] & E->ctab[lvl][key32(nlp, E->rd[lvl], w, wmask)];
          }
        }
        return;
      }
    }
  } else {
    for (uint32_t i = 0; i < sr; ++i) {
      const uint8_t* src = seav + P.seav_row_off[i] + (uint64_t)rp * P.sc[i] * P.reg_bytes;
      bool hot = false;
      for (uint32_t c = G.tid; c < P.sc[i]; c += G.size) hot |= __popcll(load_reg(src, c, P.reg_bytes)) >= 3;
      if (!G.any(hot)) return;
    }
  }

  // stage the SEA's registers (unless the one-load path did) and clear the
  // bucket tables
  for (uint32_t i = 0; i < sr; ++i) {
    const uint32_t nbytes = P.sc[i] * P.reg_bytes;
    const uint8_t* src = seav + P.seav_row_off[i] + (uint64_t)rp * nbytes;
    uint8_t* dst = sm + P.off_regs[i];
    if (!staged && (nbytes & 15u) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15u) == 0)) {
      for (uint32_t o = G.tid * 16; o < nbytes; o += G.size * 16)
        *reinterpret_cast<uint4*>(dst + o) = __ldg(reinterpret_cast<const uint4*>(src + o));
    } else if (!staged) {
      for (uint32_t o = G.tid; o < nbytes; o += G.size) dst[o] = src[o];
    }
    uint32_t* bs = reinterpret_cast<uint32_t*>(sm + P.off_bstart[i]);
    for (uint32_t o = G.tid; o <= (1u << P.nk[i]); o += G.size) bs[o] = 0;
  }
  if (G.tid == 0) {
    misc->total = 0;
    misc->abort = 0;
    misc->pairs = 0;
    for (uint32_t i = 0; i < SSPD_MAX_SR; ++i) misc->hot[i] = 0;
  }
  G.sync();

  // hot registers (weight >= 3, short_sketch.py:355-362) counted per bucket
  for (uint32_t i = 0; i < sr; ++i) {
    uint32_t* bs = reinterpret_cast<uint32_t*>(sm + P.off_bstart[i]);
    const uint8_t* regs = sm + P.off_regs[i];
    for (uint32_t c = G.tid; c < P.sc[i]; c += G.size) {
      if (__popcll(load_reg(regs, c, P.reg_bytes)) >= 3) {
        atomicAdd(&bs[pext32(c, P.keymask[i]) + 1], 1u);
        atomicAdd(&misc->hot[i], 1u);
      }
    }
  }
  G.sync();
  for (uint32_t i = 0; i < sr; ++i)
    if (misc->hot[i] == 0) return;  // a row without hot registers: no tuple (short_sketch.py:360-361)

  // bucket starts: exclusive scan of counts stored at [1 .. 2^nk]
  for (uint32_t i = G.warp; i < sr; i += G.nwarps) {
    uint32_t* bs = reinterpret_cast<uint32_t*>(sm + P.off_bstart[i]);
    warp_exclusive_scan(bs + 1, 1u << P.nk[i]);
  }
  G.sync();
  // scatter hot columns into their buckets; bs[key+1] advances to the end
  // of bucket key, leaving bs[key] = start of bucket key for every key.
  for (uint32_t i = 0; i < sr; ++i) {
    uint32_t* bs = reinterpret_cast<uint32_t*>(sm + P.off_bstart[i]);
    uint16_t* cols = reinterpret_cast<uint16_t*>(sm + P.off_cols[i]);
    const uint8_t* regs = sm + P.off_regs[i];
    for (uint32_t c = G.tid; c < P.sc[i]; c += G.size) {
      if (__popcll(load_reg(regs, c, P.reg_bytes)) >= 3) {
        const uint32_t pos = atomicAdd(&bs[pext32(c, P.keymask[i]) + 1], 1u);
        cols[pos] = (uint16_t)c;
      }
    }
  }
  G.sync();

  // flatten rows 0 x 1: pref0[j] = number of row-1 partners of row-0 entry j
  {
    uint32_t* pref0 = reinterpret_cast<uint32_t*>(sm + P.off_pref0);
    const uint16_t* cols0 = reinterpret_cast<const uint16_t*>(sm + P.off_cols[0]);
    const uint32_t* b1 = reinterpret_cast<const uint32_t*>(sm + P.off_bstart[1]);
    const uint32_t h0 = misc->hot[0];
    for (uint32_t j = G.tid; j < h0; j += G.size) {
      const uint64_t v0 = scatter_col(cols0[j], P.isb[0], P.ibn[0], P.w);
      const uint32_t key = pext32(index_of(v0, P.isb[1], P.ibn[1], P.w) & P.keymask[1], P.keymask[1]);
      pref0[j] = b1[key + 1] - b1[key];
    }
    G.sync();
    if (G.warp == 0) {
      const uint32_t total = warp_exclusive_scan(pref0, h0);
      if (G.tid == 0) {
        pref0[h0] = total;
        misc->pairs = total;
      }
    }
    G.sync();
  }

  // The counting pass only matters when the SEA could exceed the cap: the
  // complete tuples are at most (row-0 x row-1 pairs) x hot(2) x ... x
  // hot(SR-1); when that bound is <= cap the emit pass alone is exact.
  uint64_t bound = misc->pairs;
  for (uint32_t i = 2; i < sr && bound <= cap; ++i) bound *= misc->hot[i];
  if (bound > cap) {
    restore_walk<false>(P, sm, rp, cap, out_ip, out_aux, out_capacity, out_count, G.tid, G.size, T);
    G.sync();
    if (misc->total > cap) {
      if (G.tid == 0) overflow[slot] = 1;
      return;
    }
  }
  restore_walk<true>(P, sm, rp, cap, out_ip, out_aux, out_capacity, out_count, G.tid, G.size, T);
}

// one SEA at a time per warp, 4 warps per CTA, each warp with its own smem
// slice; persistent (the grid is what fits on the GPU at once, each warp
// strides over the SEAs), the next SEA's registers loaded one SEA ahead
__global__ void __launch_bounds__(128) restore_warp_kernel(const uint8_t* __restrict__ seav,
                                                           const __grid_constant__ RestorePlan P, uint32_t rp_begin,
                                                           uint32_t rp_count, uint64_t cap, uint32_t* out_ip,
                                                           uint32_t* out_aux, uint64_t out_capacity,
                                                           unsigned long long* out_count, uint8_t* overflow) {
  extern __shared__ __align__(16) uint8_t smw[];
  __shared__ WarpTab tab;
  __shared__ EmitBuf ebuf[4];
  __shared__ EnumTab etab;
  fill_warp_tab(P, &tab);
  fill_enum_tab(P, &etab);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  if (lane == 0) ebuf[warp].n = 0;
  __syncthreads();
  const Group<true> G{lane, 32u, 0u, 1u};
  const uint32_t stride = gridDim.x * (blockDim.x >> 5);
  const uint32_t lsc = tab.lane_sc[lane];
  const uint64_t lsrc = tab.lane_src[lane];
  auto load = [&](uint32_t slot) -> uint64_t {
    return (P.lane_fast && lsc && slot < rp_count)
               ? __ldg(reinterpret_cast<const uint64_t*>(seav + lsrc + (uint64_t)(rp_begin + slot) * lsc))
               : 0ull;
  };
  uint32_t slot = blockIdx.x * (blockDim.x >> 5) + warp;
  uint64_t next = load(slot);
  for (; slot < rp_count; slot += stride) {
    const uint64_t v = next;
    next = load(slot + stride);
    restore_sea_group<true>(seav, P, smw + (size_t)warp * P.smem_bytes, rp_begin + slot, slot, cap, out_ip, out_aux,
                            out_capacity, out_count, overflow, G, &tab, v, &ebuf[warp], &etab);
    flush_emit(P, &ebuf[warp], kEmitBuf / 2, out_ip, out_aux, out_capacity, out_count);
  }
  flush_emit(P, &ebuf[warp], 1, out_ip, out_aux, out_capacity, out_count);
}

__global__ void __launch_bounds__(128) restore_kernel(const uint8_t* __restrict__ seav,
                                                      const __grid_constant__ RestorePlan P, uint32_t rp_begin,
                                                      uint64_t cap, uint32_t* out_ip, uint32_t* out_aux,
                                                      uint64_t out_capacity, unsigned long long* out_count,
                                                      uint8_t* overflow) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ WarpTab tab;
  fill_warp_tab(P, &tab);
  __syncthreads();
  const Group<false> G{threadIdx.x, blockDim.x, threadIdx.x >> 5, blockDim.x >> 5};
  restore_sea_group<false>(seav, P, sm, rp_begin + blockIdx.x, blockIdx.x, cap, out_ip, out_aux, out_capacity,
                           out_count, overflow, G, &tab);
}

// ---------------------------------------------------------- cell summary
// zeros[c] = k - popcount(cell c) for every LDCA cell (LR x LC of them), one
// warp per cell.  The filter's z0 is the zero count of the AND of a
// candidate's LR cells; a full cell (zeros = 0) is the AND identity, so the
// filter reads only the non-full cells, and none at all when every cell is
// full (a saturated LDCA: z0 = 0) or only one is not (z0 = its zeros).
__global__ void __launch_bounds__(256) cell_zeros_kernel(const uint8_t* __restrict__ ldca,
                                                         const __grid_constant__ sspd_params p,
                                                         uint32_t* __restrict__ zeros) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t cells = (uint64_t)p.lr * p.lc, cell_bytes = p.k >> 3;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (cell_bytes & 15u) == 0 && (reinterpret_cast<uintptr_t>(ldca) & 15u) == 0;
  for (uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < cells; c += nwarps) {
    const uint8_t* cell = ldca + c * cell_bytes;
    uint32_t pop = 0;
    if (vec) {
      for (uint64_t v = lane; v < (cell_bytes >> 4); v += 32) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(cell) + v);
        pop += __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
      }
    } else {
      for (uint64_t b = lane; b < cell_bytes; b += 32) pop += __popc((uint32_t)cell[b]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) pop += __shfl_xor_sync(0xFFFFFFFFu, pop, o);
    if (lane == 0) zeros[c] = p.k - pop;
  }
}

// ------------------------------------------------------------------ filter
// popcount of the AND of candidate ip's LR row cells, by the whole warp
// (every lane calls it with the same ip; the result is warp-uniform).
// rows: the rows to AND (bit i = row i; rows >= 32 always taken) -- the
// others are full cells, the AND identity.  lane i (and i+32) hashes row i
// once; the cell offsets are broadcast by shuffle.
__device__ __forceinline__ uint32_t and_popcount(const uint8_t* __restrict__ ldca, const sspd_params& p,
                                                 uint32_t ip, uint32_t rows, uint32_t lane, uint64_t seed_a,
                                                 uint64_t seed_b) {
  const uint64_t cell_bytes = p.k >> 3;
  const uint64_t off_a = lane < p.lr ? ((uint64_t)lane * p.lc + hash_range(ip, seed_a, p.div_lc)) * cell_bytes : 0;
  const uint64_t off_b =
      lane + 32 < p.lr ? ((uint64_t)(lane + 32) * p.lc + hash_range(ip, seed_b, p.div_lc)) * cell_bytes : 0;
  uint32_t pop = 0;
  if (p.lr == 8 && cell_bytes == 1024 && (reinterpret_cast<uintptr_t>(ldca) & 15u) == 0) {
    // the BASELINE geometry (LR = 8, k = 8192): all 8 cell offsets first,
    // then the 8 rows' 16-byte loads of each half in flight at once (the
    // generic loop below issues one row's loads per shuffle round trip).
    // A full row's loads are redirected to the first taken row's cell (AND
    // is idempotent; the repeat hits L1, not L2).
    const uint32_t first = __ffs(rows) - 1;
    uint64_t off[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) off[i] = __shfl_sync(0xFFFFFFFFu, off_a, ((rows >> i) & 1u) ? i : first);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two halves of the 1 KB cells, 8 loads in flight each
      uint4 w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = __ldg(reinterpret_cast<const uint4*>(ldca + off[i]) + 32 * h + lane);
      uint4 a = w[0];
#pragma unroll
      for (int i = 1; i < 8; ++i) a.x &= w[i].x, a.y &= w[i].y, a.z &= w[i].z, a.w &= w[i].w;
      pop += __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w);
    }
  } else if ((cell_bytes & 15u) == 0 && (reinterpret_cast<uintptr_t>(ldca) & 15u) == 0) {
    // 16-byte loads: lane l ANDs words 4l..4l+3 of each 128-word stripe
    const uint32_t vecs = (uint32_t)(cell_bytes >> 4);
    for (uint32_t base = 0; base < vecs; base += 32) {
      const uint32_t v = base + lane;
      uint4 acc = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
      for (uint32_t i = 0; i < p.lr; ++i) {
        if (i < 32 && !((rows >> i) & 1u)) continue;  // a full cell (warp-uniform)
        const uint64_t off = __shfl_sync(0xFFFFFFFFu, i < 32 ? off_a : off_b, i & 31);
        if (v < vecs) {
          const uint4 w = __ldg(reinterpret_cast<const uint4*>(ldca + off) + v);
          acc.x &= w.x, acc.y &= w.y, acc.z &= w.z, acc.w &= w.w;
        }
      }
      if (v < vecs) pop += __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
    }
  } else if ((p.k & 31u) == 0) {
    const uint32_t words = p.k >> 5;
    for (uint32_t base = 0; base < words; base += 32) {
      const uint32_t wd = base + lane;
      uint32_t acc = 0xFFFFFFFFu;
      for (uint32_t i = 0; i < p.lr; ++i) {
        if (i < 32 && !((rows >> i) & 1u)) continue;
        const uint64_t off = __shfl_sync(0xFFFFFFFFu, i < 32 ? off_a : off_b, i & 31);
        if (wd < words) acc &= __ldg(reinterpret_cast<const uint32_t*>(ldca + off) + wd);
      }
      if (wd < words) pop += __popc(acc);
    }
  } else {
    for (uint32_t base = 0; base < cell_bytes; base += 32) {
      const uint32_t by = base + lane;
      uint32_t acc = 0xFFu;
      for (uint32_t i = 0; i < p.lr; ++i) {
        if (i < 32 && !((rows >> i) & 1u)) continue;
        const uint64_t off = __shfl_sync(0xFFFFFFFFu, i < 32 ? off_a : off_b, i & 31);
        if (by < cell_bytes) acc &= ldca[off + by];
      }
      if (by < cell_bytes) pop += __popc(acc);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) pop += __shfl_xor_sync(0xFFFFFFFFu, pop, o);
  return pop;
}

// K6: z0 = k - popcount(AND of the LR row cells) per candidate, keep =
// keep_table[z0]; one warp per candidate.  n_dev (optional): the live count
// lives in device memory (<= n); entries at or beyond it get keep = 0 so a
// fixed-capacity compaction skips them.  work / work_rows / work_n
// (optional, from filter_summary_kernel): the candidates left to AND are
// work[0 .. *work_n), each over its non-full rows work_rows[t] only.
__global__ void __launch_bounds__(256) filter_kernel(const uint8_t* __restrict__ ldca,
                                                     const __grid_constant__ sspd_params p,
                                                     const uint32_t* __restrict__ ips, uint64_t n,
                                                     const uint8_t* __restrict__ keep_table, uint32_t* z0_out,
                                                     uint8_t* keep_out, const unsigned long long* n_dev,
                                                     const uint32_t* __restrict__ work,
                                                     const uint32_t* __restrict__ work_rows,
                                                     const unsigned long long* work_n) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t live = n_dev ? min(n, (uint64_t)*n_dev) : n;
  const uint64_t items = work ? min(n, (uint64_t)*work_n) : n;
  const uint32_t all_rows = p.lr >= 32 ? 0xFFFFFFFFu : ((1u << p.lr) - 1u);
  // lane i (and i+32) owns row i: its seed is loaded once (a lane-indexed
  // constant load is serialised across the warp's distinct addresses)
  const uint64_t seed_a = lane < p.lr ? p.seed_lh[lane] : 0, seed_b = lane + 32 < p.lr ? p.seed_lh[lane + 32] : 0;
  for (uint64_t t = warp; t < items; t += nwarps) {
    const uint64_t j = work ? work[t] : t;
    if (j >= live) {
      if (lane == 0 && keep_out) keep_out[j] = 0;
      continue;
    }
    const uint32_t pop = and_popcount(ldca, p, ips[j], work ? work_rows[t] : all_rows, lane, seed_a, seed_b);
    if (lane == 0) {
      const uint32_t z0 = p.k - pop;
      z0_out[j] = z0;
      if (keep_out) keep_out[j] = keep_table ? keep_table[z0] : 1;
    }
  }
}

// K6 first pass over the cell summary (LR <= 32), one thread per candidate:
// hash the LR cells, read their zero counts; with at most one non-full cell
// z0 is known without touching the LDCA (every candidate of a saturated
// LDCA), otherwise the candidate and its non-full rows go to the work list
// that filter_kernel ANDs (full cells are the AND identity: exact).
// Candidates past the live count get keep = 0.
__global__ void __launch_bounds__(256) filter_summary_kernel(const __grid_constant__ sspd_params p,
                                                             const uint32_t* __restrict__ ips, uint64_t n,
                                                             const unsigned long long* n_dev,
                                                             const uint32_t* __restrict__ cell_zeros,
                                                             const uint8_t* __restrict__ keep_table,
                                                             uint32_t* z0_out, uint8_t* keep_out, uint32_t* work,
                                                             uint32_t* work_rows, unsigned long long* work_n) {
  const uint64_t live = n_dev ? min(n, (uint64_t)*n_dev) : n;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    if (j >= live) {
      if (keep_out) keep_out[j] = 0;
      continue;
    }
    const uint32_t ip = ips[j];
    uint32_t rows = 0, zlast = 0;
    for (uint32_t i = 0; i < p.lr; ++i) {  // row index uniform across the warp: broadcast constant loads
      const uint32_t z = __ldg(cell_zeros + (uint64_t)i * p.lc + hash_range(ip, p.seed_lh[i], p.div_lc));
      if (z) rows |= 1u << i, zlast = z;
    }
    if (__popc(rows) <= 1) {
      z0_out[j] = zlast;
      if (keep_out) keep_out[j] = keep_table ? keep_table[zlast] : 1;
    } else {
      const uint32_t t = (uint32_t)atomicAdd(work_n, 1ull);
      work[t] = (uint32_t)j;
      work_rows[t] = rows;
    }
  }
}

// Sliding variant: a slot is a set bit iff ((now - ts) & mask) < window.
template <typename T>
__global__ void __launch_bounds__(256) filter_sliding_kernel(const T* __restrict__ pool,
                                                             const __grid_constant__ sspd_params p, T now,
                                                             uint64_t window, const uint32_t* __restrict__ ips,
                                                             uint64_t n, const uint8_t* __restrict__ keep_table,
                                                             uint32_t* z0_out, uint8_t* keep_out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  constexpr uint32_t kVec = 16 / sizeof(T);  // stamps per 16-byte load
  const uint64_t seed_a = lane < p.lr ? p.seed_lh[lane] : 0, seed_b = lane + 32 < p.lr ? p.seed_lh[lane + 32] : 0;
  for (uint64_t j = warp; j < n; j += nwarps) {
    const uint32_t ip = ips[j];
    // lane i (and i+32) hashes row i once; cell bases are broadcast by shuffle
    const uint64_t base_a =
        lane < p.lr ? p.slot_ldca_base + ((uint64_t)lane * p.lc + hash_range(ip, seed_a, p.div_lc)) * p.k : 0;
    const uint64_t base_b =
        lane + 32 < p.lr
            ? p.slot_ldca_base + ((uint64_t)(lane + 32) * p.lc + hash_range(ip, seed_b, p.div_lc)) * p.k
            : 0;
    uint32_t pop = 0;
    bool vec = (p.k % (32 * kVec)) == 0;
    for (uint32_t i = 0; i < p.lr && vec; ++i)
      vec = ((__shfl_sync(0xFFFFFFFFu, i < 32 ? base_a : base_b, i & 31) * sizeof(T)) & 15u) == 0;
    if (vec) {
      // each lane ANDs kVec consecutive stamps of every row with one 16-B load per row
      for (uint32_t s0 = lane * kVec; s0 < p.k; s0 += 32 * kVec) {
        uint32_t live = (1u << kVec) - 1u;
        for (uint32_t i = 0; i < p.lr; ++i) {
          const uint64_t base = __shfl_sync(0xFFFFFFFFu, i < 32 ? base_a : base_b, i & 31);
          union {
            uint4 v;
            T t[kVec];
          } u;
          u.v = __ldg(reinterpret_cast<const uint4*>(pool + base + s0));
#pragma unroll
          for (uint32_t e = 0; e < kVec; ++e)
            if ((uint64_t)(T)(now - u.t[e]) >= window) live &= ~(1u << e);
        }
        pop += __popc(live);
      }
    } else {
      for (uint32_t s0 = 0; s0 < p.k; s0 += 32) {
        const uint32_t s = s0 + lane;
        bool all = s < p.k;
        for (uint32_t i = 0; i < p.lr; ++i) {
          const uint64_t base = __shfl_sync(0xFFFFFFFFu, i < 32 ? base_a : base_b, i & 31);
          if (all) all = (uint64_t)(T)(now - pool[base + s]) < window;
        }
        pop += all ? 1u : 0u;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) pop += __shfl_xor_sync(0xFFFFFFFFu, pop, o);
    if (lane == 0) {
      const uint32_t z0 = p.k - pop;
      z0_out[j] = z0;
      if (keep_out) keep_out[j] = keep_table ? keep_table[z0] : 1;
    }
  }
}

// Stable compaction of the kept candidates.  Segment b of kSeg entries is
// owned by block b: pass 1 counts each segment, pass 2 gets the number of
// kept entries before it -- by summing the preceding counts when there are
// at most kSegDirect segments, else from one exclusive scan of the counts --
// and scatters its segment in order with a ballot-based block scan.
constexpr uint32_t kSeg = 1024;  // one 1,024-thread pass per segment (many blocks in flight)

__device__ void compact_segment(const uint32_t* __restrict__ ip, const uint32_t* __restrict__ z0,
                                const uint8_t* __restrict__ keep, uint64_t lo, uint64_t hi, uint32_t* ip_out,
                                uint32_t* z0_out, unsigned long long base) {
  __shared__ uint32_t warp_pre[32];
  __shared__ uint32_t tile_total;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint64_t start = lo; start < hi; start += blockDim.x) {
    const uint64_t j = start + threadIdx.x;
    const uint32_t f = (j < hi && keep[j]) ? 1u : 0u;
    const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, f);
    if (lane == 0) warp_pre[wid] = __popc(ballot);
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the per-warp counts (lane i owns entry i)
      const uint32_t v = lane < nw ? warp_pre[lane] : 0u;
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      if (lane < nw) warp_pre[lane] = incl - v;
      if (lane == 31) tile_total = incl;
    }
    __syncthreads();
    const uint32_t before = warp_pre[wid] + __popc(ballot & ((1u << lane) - 1u));
    if (f) {
      ip_out[base + before] = ip[j];
      z0_out[base + before] = z0[j];
    }
    base += tile_total;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) compact_count_kernel(const uint8_t* __restrict__ keep, uint64_t n,
                                                             uint32_t* seg_counts) {
  const uint64_t lo = (uint64_t)blockIdx.x * kSeg, hi = min(n, lo + kSeg);
  uint32_t c = 0;
  for (uint64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) c += keep[j] ? 1u : 0u;
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  __shared__ uint32_t ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) t += ws[w];
    seg_counts[blockIdx.x] = t;
  }
}

// Exclusive prefix of the segment counts (one 1,024-thread block; thread t
// owns a contiguous run of ceil(segs/1024) counts): used when there are more
// than kSegDirect segments, so the scatter reads its base in O(1) instead of
// summing every earlier segment (O(segs^2) work over the grid).
constexpr uint64_t kSegDirect = 1024;

__global__ void __launch_bounds__(1024) compact_seg_scan_kernel(const uint32_t* __restrict__ seg_counts,
                                                                uint64_t segs, uint32_t* __restrict__ seg_pre) {
  __shared__ uint32_t ws[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t per = (segs + 1023) / 1024;
  const uint64_t lo = min(segs, tid * per), hi = min(segs, lo + per);
  uint32_t sum = 0;
  for (uint64_t b = lo; b < hi; ++b) sum += seg_counts[b];
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
  for (uint64_t b = lo; b < hi; ++b) {
    const uint32_t c = seg_counts[b];
    seg_pre[b] = run;
    run += c;
  }
}

// kPre: seg_pre holds the exclusive prefix (compact_seg_scan_kernel); else the
// block sums the counts before it (<= kSegDirect of them).
template <bool kPre>
__global__ void __launch_bounds__(1024) compact_scatter_kernel(const uint32_t* __restrict__ ip,
                                                               const uint32_t* __restrict__ z0,
                                                               const uint8_t* __restrict__ keep, uint64_t n,
                                                               const uint32_t* __restrict__ seg_counts,
                                                               const uint32_t* __restrict__ seg_pre,
                                                               uint32_t* ip_out, uint32_t* z0_out,
                                                               unsigned long long* out_count) {
  __shared__ unsigned long long base_s;
  __shared__ uint32_t ws[32];
  if (kPre) {
    if (threadIdx.x == 0) {
      base_s = seg_pre[blockIdx.x];
      if (blockIdx.x == gridDim.x - 1) *out_count = base_s + seg_counts[blockIdx.x];
    }
  } else {
    uint32_t pre = 0;
    for (uint32_t b = threadIdx.x; b < blockIdx.x; b += blockDim.x) pre += seg_counts[b];
#pragma unroll
    for (int o = 16; o; o >>= 1) pre += __shfl_xor_sync(0xFFFFFFFFu, pre, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = pre;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
      for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) t += ws[w];
      base_s = t;
      if (blockIdx.x == gridDim.x - 1) *out_count = t + seg_counts[blockIdx.x];
    }
  }
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * kSeg, hi = min(n, lo + kSeg);
  compact_segment(ip, z0, keep, lo, hi, ip_out, z0_out, base_s);
}

__global__ void __launch_bounds__(1024) compact_single_kernel(const uint32_t* __restrict__ ip,
                                                              const uint32_t* __restrict__ z0,
                                                              const uint8_t* __restrict__ keep, uint64_t n,
                                                              uint32_t* ip_out, uint32_t* z0_out,
                                                              unsigned long long* out_count) {
  __shared__ uint32_t cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  compact_segment(ip, z0, keep, 0, n, ip_out, z0_out, 0);
  uint32_t c = 0;
  for (uint64_t j = threadIdx.x; j < n; j += blockDim.x) c += keep[j] ? 1u : 0u;
  atomicAdd(&cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) *out_count = cnt;
}

static int build_plan(const sspd_params& p, RestorePlan& P) {
  memset(&P, 0, sizeof(P));
  P.sr = p.sr;
  P.w = p.lp_bits;
  P.r = p.r;
  P.reg_bytes = p.reg_bytes;
  const uint64_t full = p.g >= 64 ? ~0ull : ((1ull << p.g) - 1ull);
  P.full_bits_lo = (uint32_t)full;
  P.full_bits_hi = (uint32_t)(full >> 32);
  uint64_t seen = 0;
  uint32_t off = 0;
  auto align = [](uint32_t v, uint32_t a) { return (v + a - 1) / a * a; };
  off = align(sizeof(Misc), 16);
  P.off_misc = 0;
  for (uint32_t i = 0; i < p.sr; ++i) {
    P.isb[i] = p.isb[i];
    P.ibn[i] = p.ibn[i];
    P.sc[i] = p.sc[i];
    P.seav_row_off[i] = p.seav_row_off[i];
    const uint64_t mask = row_mask(p.isb[i], p.ibn[i], p.lp_bits);
    const uint64_t fixed = seen & mask;
    seen |= mask;
    P.keymask[i] = index_of(fixed, p.isb[i], p.ibn[i], p.lp_bits);
    P.nk[i] = (uint32_t)__builtin_popcount(P.keymask[i]);
    P.off_bstart[i] = off;
    off = align(off + 4u * ((1u << P.nk[i]) + 1u), 16);
  }
  P.off_pref0 = off;
  off = align(off + 4u * (p.sc[0] + 1u), 16);
  for (uint32_t i = 0; i < p.sr; ++i) {
    P.off_regs[i] = off;
    off = align(off + p.sc[i] * p.reg_bytes, 16);
  }
  for (uint32_t i = 0; i < p.sr; ++i) {
    P.off_cols[i] = off;
    off = align(off + 2u * p.sc[i], 16);
  }
  P.smem_bytes = off;
  P.hist = nullptr;
  P.hshift = 0;
  // one-load warp staging (see RestorePlan::lane_fast)
  P.lane_fast = 0;
  {
    bool ok = p.reg_bytes == 1 && p.sr <= 32;
    uint32_t lane = 0;
    for (uint32_t i = 0; i < p.sr && ok; ++i) {
      ok = (p.sc[i] % 8) == 0 && (p.seav_row_off[i] % 8) == 0 && (P.off_regs[i] % 8) == 0;
      P.row_lanes[i] = 0;
      for (uint32_t o = 0; ok && o < p.sc[i]; o += 8, ++lane) {
        if (lane >= 32) {
          ok = false;
          break;
        }
        P.lane_row[lane] = (uint8_t)i;
        P.lane_off[lane] = (uint8_t)o;
        P.row_lanes[i] |= 1u << lane;
      }
    }
    for (uint32_t l = lane; l < 32; ++l) {
      P.lane_row[l] = 0xFF;
      P.lane_off[l] = 0;
    }
    P.lane_fast = ok ? 1u : 0u;
    bool en = ok && p.lp_bits <= 32;
    uint32_t l0 = 0;
    for (uint32_t i = 0; i < p.sr && en; ++i) {
      en = p.sc[i] <= 64;
      P.row_lane0[i] = l0;
      l0 += p.sc[i] / 8;
      P.row_bits[i] = (uint32_t)row_mask(p.isb[i], p.ibn[i], p.lp_bits);
    }
    P.lane_enum = en ? 1u : 0u;
    P.rows8 = en && p.sr <= 4 ? 1u : 0u;
    for (uint32_t i = 0; i < p.sr && P.rows8; ++i) P.rows8 = p.sc[i] == 64 ? 1u : 0u;
    // mask walk whenever the tuple bound allows it (<= cap); the knob caps
    // it further for A/B against the bucket tables
    P.enum_max = 0xFFFFFFFFu;
    if (const char* e = getenv("SSPD_RESTORE_ENUM_MAX")) P.enum_max = (uint32_t)atoi(e);
  }
  return SSPD_OK;
}

// ---- bucket sort of the candidates (sspd_finalize) -----------------------
// The candidates are unique IPv4 keys, uniformly spread for random traffic.
// The restore counts them per bucket (bucket = ip >> hshift, nb buckets,
// ~16 keys per bucket at full capacity); one pass turns the counts into
// bucket starts and scatters the keys into their buckets, and one warp per
// bucket then orders its <= 64 keys in registers (rank = number of smaller
// keys).  Two launches instead of a radix sort's six.  A bucket with more
// than kBucketMax keys (skewed addresses) raises *too_big: the caller
// re-runs the finalize with the radix sort (exact either way).
constexpr uint32_t kBucketMax = 64;

__global__ void __launch_bounds__(1024) bucket_scatter_kernel(const uint32_t* __restrict__ ip,
                                                              const unsigned long long* __restrict__ found,
                                                              uint64_t cap, const uint32_t* __restrict__ hist,
                                                              uint32_t nb, uint32_t hshift, uint32_t* cursor,
                                                              uint32_t* start_out, uint32_t* __restrict__ bucketed) {
  extern __shared__ uint32_t pre[];  // [nb] bucket starts
  __shared__ uint32_t wsum[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t per = (nb + 1023) / 1024;  // contiguous counts per thread
  uint32_t tsum = 0;
  for (uint32_t e = 0; e < per; ++e) {
    const uint32_t i = tid * per + e;
    if (i < nb) tsum += hist[i];
  }
  uint32_t x = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= (uint32_t)o) w += y;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  uint32_t run = x - tsum + (warp ? wsum[warp - 1] : 0u);
  for (uint32_t e = 0; e < per; ++e) {
    const uint32_t i = tid * per + e;
    if (i < nb) {
      pre[i] = run;
      run += hist[i];
    }
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (uint32_t i = tid; i < nb; i += blockDim.x) start_out[i] = pre[i];
    if (tid == 0) start_out[nb] = wsum[31];
  }
  const uint64_t n = min((uint64_t)*found, cap);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + tid; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = ip[i];
    const uint32_t b = k >> hshift;
    bucketed[pre[b] + atomicAdd(cursor + b, 1u)] = k;
  }
}

__global__ void __launch_bounds__(256) bucket_sort_kernel(const uint32_t* __restrict__ bucketed,
                                                          const uint32_t* __restrict__ start, uint32_t nb,
                                                          uint32_t* __restrict__ out, uint8_t* too_big) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb; b += nwarps) {
    const uint32_t lo = start[b], n = start[b + 1] - lo;
    if (n == 0) continue;
    if (n > kBucketMax) {
      if (lane == 0) *too_big = 1;
      continue;
    }
    const uint32_t k0 = lane < n ? bucketed[lo + lane] : 0xFFFFFFFFu;
    const uint32_t k1 = lane + 32 < n ? bucketed[lo + 32 + lane] : 0xFFFFFFFFu;
    uint32_t r0 = 0, r1 = 0;
    for (uint32_t j = 0; j < n; ++j) {  // n is warp-uniform
      const uint32_t kj = __shfl_sync(0xFFFFFFFFu, j < 32 ? k0 : k1, j & 31);
      r0 += (kj < k0) | ((kj == k0) & (j < lane));
      r1 += (kj < k1) | ((kj == k1) & (j < lane + 32));
    }
    if (lane < n) out[lo + r0] = k0;
    if (lane + 32 < n) out[lo + r1] = k1;
  }
}

}  // namespace sspd

using namespace sspd;

static int restore_launch(const uint8_t* seav, const sspd_params* p, uint32_t rp_begin, uint32_t rp_count,
                          uint64_t cap, uint32_t* out_ip, uint32_t* out_aux, uint64_t out_capacity,
                          unsigned long long* out_count, uint8_t* overflow, uint32_t* hist, uint32_t hshift,
                          void* stream);

extern "C" int sspd_restore(const uint8_t* seav, const sspd_params* p, uint32_t rp_begin, uint32_t rp_count,
                            uint64_t cap, uint32_t* out_ip, uint32_t* out_aux, uint64_t out_capacity,
                            unsigned long long* out_count, uint8_t* overflow, void* stream) {
  return restore_launch(seav, p, rp_begin, rp_count, cap, out_ip, out_aux, out_capacity, out_count, overflow,
                        nullptr, 0, stream);
}

static int restore_launch(const uint8_t* seav, const sspd_params* p, uint32_t rp_begin, uint32_t rp_count,
                          uint64_t cap, uint32_t* out_ip, uint32_t* out_aux, uint64_t out_capacity,
                          unsigned long long* out_count, uint8_t* overflow, uint32_t* hist, uint32_t hshift,
                          void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if ((uint64_t)rp_begin + rp_count > (1ull << p->r)) return SSPD_ERR_CONFIG;
  if (!seav || !out_count || !overflow) return SSPD_ERR_DATA;
  if (rp_count == 0) return SSPD_OK;
  RestorePlan P;
  build_plan(*p, P);
  P.hist = hist;
  P.hshift = hshift;
  int dev = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if ((int)P.smem_bytes > max_smem) return SSPD_ERR_CONFIG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t regs = 0;
  for (uint32_t i = 0; i < p->sr; ++i) regs += p->sc[i];
  // arrays up to this many registers: one warp per SEA (r = 16 geometry,
  // 65,536 small arrays); larger ones (r = 12: 512 registers) split each
  // array's work list over a CTA -- measured 93 vs 213 us at config 2
  uint32_t warp_regs = 256;
  if (const char* e = getenv("SSPD_RESTORE_WARP_REGS")) warp_regs = (uint32_t)atoi(e);
  if (regs <= warp_regs && 4 * P.smem_bytes <= 48 * 1024) {  // small arrays: one warp per SEA
    static int per_sm = 0, sms = 0;
    static uint32_t per_sm_smem = 0;
    if (per_sm == 0 || per_sm_smem != P.smem_bytes) {
      // dynamic + the static tables (WarpTab, EmitBuf) may pass the 48 KB default
      cudaFuncSetAttribute(restore_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4 * P.smem_bytes));
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, restore_warp_kernel, 128, 4 * P.smem_bytes);
      if (per_sm < 1) per_sm = 1;
      per_sm_smem = P.smem_bytes;
    }
    const uint32_t blocks = std::min<uint32_t>((rp_count + 3) / 4, (uint32_t)(sms * per_sm));
    restore_warp_kernel<<<blocks, 128, 4 * P.smem_bytes, st>>>(seav, P, rp_begin, rp_count, cap, out_ip, out_aux,
                                                               out_capacity, out_count, overflow);
    return check_launch();
  }
  if (P.smem_bytes > 48 * 1024)
    cudaFuncSetAttribute(restore_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem_bytes);
  restore_kernel<<<rp_count, 128, P.smem_bytes, st>>>(seav, P, rp_begin, cap, out_ip, out_aux, out_capacity,
                                                      out_count, overflow);
  return check_launch();
}

// csrc/radix.cu: library-free stable LSD radix sort of u32 keys (+ values)
namespace sspd {
size_t radix_sort_scratch(uint64_t n, bool with_vals);
int radix_sort_u32(uint32_t* keys, uint32_t* vals, uint64_t n, void* scratch, size_t scratch_bytes,
                   cudaStream_t st);
}  // namespace sspd

extern "C" int sspd_sort_candidates(uint32_t* ip, uint32_t* aux, uint64_t n, void* scratch, size_t* scratch_bytes,
                                    void* stream) {
  if (!scratch_bytes) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t need = radix_sort_scratch(n ? n : 1, true);
  if (!scratch) {
    *scratch_bytes = need;
    return SSPD_OK;
  }
  if (*scratch_bytes < need) return SSPD_ERR_CAPACITY;
  if (n <= 1) return SSPD_OK;
  return radix_sort_u32(ip, aux, n, scratch, *scratch_bytes, st);
}

extern "C" int sspd_filter(const uint8_t* ldca, const sspd_params* p, const uint32_t* ips, uint64_t n,
                           const uint8_t* keep_table, uint32_t* z0_out, uint8_t* keep_out, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (n == 0) return SSPD_OK;
  if (!ldca || !ips || !z0_out) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(filter_kernel, 256, n * 32);
  filter_kernel<<<grid, 256, 0, st>>>(ldca, *p, ips, n, keep_table, z0_out, keep_out, nullptr, nullptr, nullptr,
                                      nullptr);
  return check_launch();
}

extern "C" int sspd_filter_sliding(const void* pool, uint32_t ts_bytes, const sspd_params* p, uint64_t now_wrapped,
                                   uint64_t window_slices, const uint32_t* ips, uint64_t n,
                                   const uint8_t* keep_table, uint32_t* z0_out, uint8_t* keep_out, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (n == 0) return SSPD_OK;
  if (!pool || !ips || !z0_out) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (ts_bytes) {
#define SSPD_FS(T)                                                                                       \
  {                                                                                                      \
    const int grid = grid_for(filter_sliding_kernel<T>, 256, n * 32);                                   \
    filter_sliding_kernel<T><<<grid, 256, 0, st>>>((const T*)pool, *p, (T)now_wrapped, window_slices, ips, n, \
                                                   keep_table, z0_out, keep_out);                        \
    break;                                                                                               \
  }
    case 1: SSPD_FS(uint8_t)
    case 2: SSPD_FS(uint16_t)
    case 4: SSPD_FS(uint32_t)
    case 8: SSPD_FS(uint64_t)
#undef SSPD_FS
    default:
      return SSPD_ERR_CONFIG;
  }
  return check_launch();
}

extern "C" int sspd_compact_reports(const uint32_t* ip, const uint32_t* z0, const uint8_t* keep, uint64_t n,
                                    uint32_t* ip_out, uint32_t* z0_out, unsigned long long* out_count, void* scratch,
                                    size_t* scratch_bytes, void* stream) {
  if (!out_count) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t segs = (n + kSeg - 1) / kSeg;
  // [seg counts | exclusive prefix (more than kSegDirect segments only)]
  const size_t need = 4 * (segs ? segs : 1) * (segs > kSegDirect ? 2 : 1);
  if (!scratch) {
    if (scratch_bytes) {  // size query
      *scratch_bytes = need;
      return SSPD_OK;
    }
    compact_single_kernel<<<1, 1024, 0, st>>>(ip, z0, keep, n, ip_out, z0_out, out_count);
    return check_launch();
  }
  if (!scratch_bytes || *scratch_bytes < need) return SSPD_ERR_CAPACITY;
  if (n == 0) return cudaMemsetAsync(out_count, 0, sizeof(unsigned long long), st) == cudaSuccess ? SSPD_OK
                                                                                                 : SSPD_ERR_CUDA;
  uint32_t* seg_counts = static_cast<uint32_t*>(scratch);
  compact_count_kernel<<<(unsigned)segs, 1024, 0, st>>>(keep, n, seg_counts);
  if (segs > kSegDirect) {
    uint32_t* seg_pre = seg_counts + segs;
    compact_seg_scan_kernel<<<1, 1024, 0, st>>>(seg_counts, segs, seg_pre);
    compact_scatter_kernel<true><<<(unsigned)segs, 1024, 0, st>>>(ip, z0, keep, n, seg_counts, seg_pre, ip_out,
                                                                  z0_out, out_count);
  } else {
    compact_scatter_kernel<false><<<(unsigned)segs, 1024, 0, st>>>(ip, z0, keep, n, seg_counts, nullptr, ip_out,
                                                                   z0_out, out_count);
  }
  return check_launch();
}

// One finalize without host round trips (restore -> sort -> filter ->
// compaction), every count kept on the device.  The candidate buffers have a
// fixed capacity C; slots past the live count (counts[0], on the device) are
// never reported: the filter marks them not kept and the compaction runs over
// C.  Sort: bucket sort (above) for C <= kBucketSortMaxCap unless `flags` bit
// 0 asks for the radix sort, which sorts all C slots of a key buffer
// pre-filled with 0xFFFFFFFF (the live candidates come first).  counts[0] =
// candidates found (may exceed C: the outputs are then incomplete and the
// caller retries with a larger C), counts[1] = reports kept; overflow[2^r] = 1
// when a bucket was too large for the bucket sort (the caller re-runs with
// the radix sort).
constexpr uint64_t kBucketSortMaxCap = 1ull << 18;

// The finalize's zero-initialised state in one launch instead of one memset
// per region: the two counts, the per-SEA overflow flags + the bucket flag
// byte, the bucket histogram + cursors (bucket path) and the filter's
// work-list count -- each a graph node otherwise.
namespace sspd {
__global__ void __launch_bounds__(256) finalize_init_kernel(unsigned long long* counts, uint8_t* overflow,
                                                            uint32_t nflags, uint32_t* hist, uint32_t nhist,
                                                            unsigned long long* work_n) {
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 2) counts[t] = 0;
  if (t == 2 && work_n) *work_n = 0;
  for (uint32_t i = t; i < nflags; i += stride) overflow[i] = 0;
  if (hist)
    for (uint32_t i = t; i < nhist; i += stride) hist[i] = 0;
}
}  // namespace sspd

extern "C" int sspd_finalize(const uint8_t* seav, const uint8_t* ldca, const sspd_params* p, uint64_t restore_cap,
                             const uint8_t* keep_table, uint64_t capacity, uint32_t* out_ip, uint32_t* out_z0,
                             unsigned long long* counts, uint8_t* overflow, void* scratch, size_t* scratch_bytes,
                             uint32_t flags, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (!scratch_bytes || capacity == 0 || capacity >= (1ull << 31)) return SSPD_ERR_CONFIG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t C = (size_t)capacity;
  const size_t vec = ((C * 4 + 255) / 256) * 256;
  const bool bucket = (flags & 1u) == 0 && C <= kBucketSortMaxCap;
  // bucket count: ~16 keys per bucket at full capacity, power of two
  uint32_t nb = 256;
  while ((uint64_t)nb * 16 < C && nb < 16384) nb <<= 1;
  const uint32_t hshift = 32 - (31 - __builtin_clz(nb));
  // the filter and the report list need the candidate IPs only: sort keys
  // (restore's AND-weights are not part of a report)
  const size_t sort_tmp = radix_sort_scratch(C, false);
  const size_t segs = (C + kSeg - 1) / kSeg;
  // [ip | aux | ip_alt | aux_alt | z0 | keep | sort temp | compaction segs | hist, cursor | starts]
  const size_t o_aux = vec, o_ipa = 2 * vec, o_z0 = 4 * vec, o_keep = 5 * vec;  // [3 vec, 4 vec): spare
  const size_t o_tmp = o_keep + ((C + 255) / 256) * 256;
  const size_t o_seg = o_tmp + ((sort_tmp + 255) / 256) * 256;
  const size_t seg_bytes = 4 * segs * (segs > kSegDirect ? 2 : 1);  // sspd_compact_reports scratch
  const size_t o_hist = o_seg + ((seg_bytes + 255) / 256) * 256;
  const size_t o_start = o_hist + 8ull * 16384;
  const size_t o_cz = o_start + ((4ull * (16384 + 1) + 255) / 256) * 256;  // cell summary (LR <= 32)
  const uint64_t cells = p->lr <= 32 ? (uint64_t)p->lr * p->lc : 0;
  const size_t o_wn = o_cz + ((4 * cells + 255) / 256) * 256;  // work-list count (u64)
  const size_t need = o_wn + 256;
  if (!scratch) {
    *scratch_bytes = need;
    return SSPD_OK;
  }
  if (*scratch_bytes < need) return SSPD_ERR_CAPACITY;
  if (!seav || !ldca || !out_ip || !out_z0 || !counts || !overflow) return SSPD_ERR_DATA;
  uint8_t* s8 = static_cast<uint8_t*>(scratch);
  uint32_t* ip = reinterpret_cast<uint32_t*>(s8);
  uint32_t* aux = reinterpret_cast<uint32_t*>(s8 + o_aux);
  uint32_t* ipa = reinterpret_cast<uint32_t*>(s8 + o_ipa);
  uint32_t* z0 = reinterpret_cast<uint32_t*>(s8 + o_z0);
  uint8_t* keep = s8 + o_keep;
  uint32_t* hist = reinterpret_cast<uint32_t*>(s8 + o_hist);
  uint32_t* cursor = hist + nb;
  uint32_t* starts = reinterpret_cast<uint32_t*>(s8 + o_start);
  const uint32_t rp_count = 1u << p->r;
  {
    unsigned long long* wn = cells ? reinterpret_cast<unsigned long long*>(s8 + o_wn) : nullptr;
    const uint32_t nflags = rp_count + 1, nhist = bucket ? 2u * nb : 0u;  // hist + cursor: 8 B per bucket
    const uint32_t work = std::max(nflags, nhist);
    finalize_init_kernel<<<std::min<uint32_t>(148u * 4u, (work + 255) / 256), 256, 0, st>>>(
        counts, overflow, nflags, bucket ? hist : nullptr, nhist, wn);
  }
  const uint32_t* sorted = ip;
  if (bucket) {
    rc = restore_launch(seav, p, 0, rp_count, restore_cap, ip, aux, C, counts, overflow, hist, hshift, stream);
    if (rc) return rc;
    const uint32_t smem = 4u * nb;
    if (smem > 48u * 1024u)
      cudaFuncSetAttribute(bucket_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint32_t grid = (uint32_t)std::min<size_t>(296, (C + 1023) / 1024);  // ~1 key per thread
    bucket_scatter_kernel<<<grid, 1024, smem, st>>>(ip, counts, C, hist, nb, hshift, cursor, starts, ipa);
    bucket_sort_kernel<<<(nb * 32 + 255) / 256, 256, 0, st>>>(ipa, starts, nb, ip, overflow + rp_count);
  } else {
    if (cudaMemsetAsync(ip, 0xFF, C * 4, st) != cudaSuccess) return SSPD_ERR_CUDA;
    rc = restore_launch(seav, p, 0, rp_count, restore_cap, ip, aux, C, counts, overflow, nullptr, 0, stream);
    if (rc) return rc;
    rc = radix_sort_u32(ip, nullptr, C, s8 + o_tmp, sort_tmp, st);
    if (rc) return rc;
    sorted = ip;
  }
  const int grid = grid_for(filter_kernel, 256, C * 32);
  if (cells) {
    // the cell summary, then the thread-per-candidate pass; the warps AND
    // only the candidates it could not settle (work list in the free
    // [2 vec, 4 vec) of the scratch: ip_alt and the spare vector)
    uint32_t* cz = reinterpret_cast<uint32_t*>(s8 + o_cz);
    uint32_t* work_rows = reinterpret_cast<uint32_t*>(s8 + o_ipa);
    uint32_t* work = reinterpret_cast<uint32_t*>(s8 + 3 * vec);
    unsigned long long* work_n = reinterpret_cast<unsigned long long*>(s8 + o_wn);  // zeroed by finalize_init_kernel
    cell_zeros_kernel<<<grid_for(cell_zeros_kernel, 256, cells * 32), 256, 0, st>>>(ldca, *p, cz);
    filter_summary_kernel<<<grid_for(filter_summary_kernel, 256, C), 256, 0, st>>>(
        *p, sorted, C, counts, cz, keep_table, z0, keep, work, work_rows, work_n);
    filter_kernel<<<grid, 256, 0, st>>>(ldca, *p, sorted, C, keep_table, z0, keep, counts, work, work_rows, work_n);
  } else {
    filter_kernel<<<grid, 256, 0, st>>>(ldca, *p, sorted, C, keep_table, z0, keep, counts, nullptr, nullptr,
                                        nullptr);
  }
  size_t cb = seg_bytes;
  rc = sspd_compact_reports(sorted, z0, keep, C, out_ip, out_z0, counts + 1, s8 + o_seg, &cb, stream);
  if (rc) return rc;
  return check_launch();
}
