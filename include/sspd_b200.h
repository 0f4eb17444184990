/*
 * sspd_b200.h -- C ABI of the B200 packet-scan / estimate path for the
 * super-point detector of arXiv 1901.07306 (reference package `sspd`).
 *
 * Every entry point takes caller-owned DEVICE buffers (plain pointers and
 * sizes), an explicit cudaStream_t passed as `void*`, and a host pointer to a
 * POD `sspd_params` block that it copies by value into the kernel launch.
 * Nothing allocates behind the caller's back and there is no global mutable
 * state.  The return value is an `sspd_status`; the Python host layer maps
 * it onto the reference exception classes (errors.py:7-53):
 *   SSPD_ERR_CONFIG  -> ConfigError      (bad geometry / argument)
 *   SSPD_ERR_DATA    -> DataError        (malformed input)
 *   SSPD_ERR_CUDA    -> SspdError        (launch / runtime failure)
 *
 * The reference has no FFI layer: each function below
 * replaces one Python method of the reference, cited per function.
 */
#ifndef SSPD_B200_H
#define SSPD_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SSPD_API __attribute__((visibility("default")))
#else
#define SSPD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SSPD_ABI_VERSION 1
#define SSPD_MAX_SR 16   /* SEAV rows supported by the kernels        */
#define SSPD_MAX_LR 64   /* LDCA rows supported by the kernels        */

typedef enum sspd_status {
  SSPD_OK = 0,
  SSPD_ERR_CONFIG = 2,
  SSPD_ERR_DATA = 3,
  SSPD_ERR_CUDA = 4,
  SSPD_ERR_CAPACITY = 5 /* output buffer too small; *count holds the need */
} sspd_status;

/* Exact `x % d` for 64-bit x by a runtime divisor 1 <= d < 2^32
 * (hashing.py:120-130 reduces the FULL 64-bit hash modulo m).  pow2 != 0
 * means d is a power of two and the mask path is used; otherwise the
 * Granlund-Montgomery round-up multiplier `magic` (65-bit, top bit implicit)
 * with shifts sh1/sh2 gives the quotient.  Built by the host layer. */
typedef struct sspd_divisor {
  uint64_t d;
  uint64_t magic;
  uint32_t sh1;
  uint32_t sh2;
  uint32_t pow2;
  uint32_t pad_;
} sspd_divisor;

/* Resolved detector geometry + hash family.  Field meanings follow the
 * reference: SeedFamily (hashing.py:82-99), SeavConfig
 * (short_sketch.py:116-181), LdcaConfig (long_sketch.py:72-90). */
typedef struct sspd_params {
  /* hash family: derive_seed(master, tag) for H1/H2/H3/ROUTE/LH_i */
  uint64_t seed_h1, seed_h2, seed_h3, seed_route;
  uint64_t seed_lh[SSPD_MAX_LR];
  /* SEAV (short estimator array vector) */
  uint32_t r, sr, a, g;
  uint32_t addr_bits, lp_bits, tau, reg_bytes; /* reg_bytes: 1/2/4/8 */
  uint32_t isb[SSPD_MAX_SR];
  uint32_t ibn[SSPD_MAX_SR];
  uint32_t sc[SSPD_MAX_SR];
  uint64_t seav_row_off[SSPD_MAX_SR]; /* byte offset of row i (flat payload) */
  uint64_t seav_bytes;                /* payload bytes = memory_bytes()      */
  /* LDCA (linear distinct counter array) */
  uint32_t lr, lc, k, pad0_;
  uint64_t ldca_bytes;                /* lr*lc*k/8                           */
  sspd_divisor div_g, div_k, div_lc;
  /* sliding layout (sliding.py:119-146): slot bases, in timestamp slots */
  uint64_t slot_row_base[SSPD_MAX_SR];
  uint64_t slot_ldca_base;
  uint64_t slot_total;
} sspd_params;

/* ---- library identity ------------------------------------------------- */
SSPD_API int sspd_abi_version(void);
SSPD_API size_t sspd_params_size(void);          /* sizeof(sspd_params) for checking  */
SSPD_API int sspd_device_sm_count(int device);   /* -1 when no device is available     */

/* ---- host-side helpers (no device work; used by the CPU test suite) ---- */
/* hash_range(key, seed, d) exactly as hashing.py:120-124, via the same
 * fast-modulo code the kernels run. */
SSPD_API uint64_t sspd_hash_range_host(uint64_t key, uint64_t seed, const sspd_divisor* d);
SSPD_API uint64_t sspd_mix64_host(uint64_t x);                   /* hashing.py:48-53 */

/* ---- host staging of caller key arrays (no device work) ----------------
 * DetectorState.process_batch from host memory (the reference's own call
 * pattern: 65,536-pair numpy buffers, cli.py:215-217) stages the keys in
 * pinned memory and scans them in large batches.  sspd_host_check_u32 =
 * SSPD_ERR_DATA if any of n keys (elem_bytes 1/2/4/8, signed or not) lies
 * outside [0, 2^32) -- the IPv4-only contract, checked before anything is
 * staged; sspd_host_pack_u32 = narrow n checked keys into dst (u32). */
SSPD_API int sspd_host_check_u32(const void* src, uint64_t n, uint32_t elem_bytes, int is_signed);
SSPD_API int sspd_host_pack_u32(const void* src, uint64_t n, uint32_t elem_bytes, int is_signed, uint32_t* dst);
/* Both key arrays of a batch at once (widths hbytes/obytes), split over a
 * persistent host worker pool (SSPD_HOST_COPY_THREADS, default min(cores/2, 8));
 * sspd_host_copy_threads = the threads a pack uses (pool workers + caller). */
SSPD_API int sspd_host_pack_pairs(const void* hips, const void* oips, uint64_t n, uint32_t hbytes,
                                  uint32_t obytes, uint32_t* dst_h, uint32_t* dst_o);
SSPD_API int sspd_host_copy_threads(void);

/* ---- K1 discrete scan --------------------------------------------------
 * Replaces DetectorState.process_batch (window_detector.py:100-103) =
 * SeavSketch.update_batch (short_sketch.py:300-318) +
 * LdcaSketch.update_batch (long_sketch.py:125-135).
 * hips/oips: n uint32 host/opposite IPs (device).  seav: p->seav_bytes,
 * ldca: p->ldca_bytes (both rounded up to 16 B by the caller, zero-padded).
 * Either sketch pointer may be NULL to skip that sketch. */
SSPD_API int sspd_scan_discrete(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                       const sspd_params* p, uint8_t* seav, uint8_t* ldca,
                       void* stream);

/* ---- K1b / K1p partitioned scan (same result as sspd_scan_discrete) -----
 * Replaces the same reference call as sspd_scan_discrete
 * (window_detector.py:100-103).  The LDCA is partitioned across the SMs'
 * shared memory for the duration of the launch (one persistent CTA per SM,
 * cooperative launch); updates are routed through per-partition buckets in
 * `scratch` (size from sspd_scan_partitioned_scratch(p, chunk)).  K1b cuts
 * the LDCA along its b axis (one 16-byte entry per packet; LR = 8, k and lc
 * powers of two) and is used whenever it applies; K1p cuts it into word
 * ranges (any geometry whose LDCA fits).  sspd_scan_partitioned_variant
 * tells which one runs: 2 = K1b, 1 = K1p, 0 = neither.  Returns
 * SSPD_ERR_CONFIG when the LDCA does not fit in shared memory (use
 * sspd_scan_discrete), and SSPD_ERR_CAPACITY when scratch is too small.
 * ldca must be non-NULL. */
SSPD_API int sspd_scan_partitioned(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                   const sspd_params* p, uint8_t* seav, uint8_t* ldca,
                                   void* scratch, uint64_t scratch_bytes, uint64_t chunk,
                                   void* stream);
/* The same into an LDCA buffer that holds only zeros on entry (a fresh
 * sliding dirty-bitmap slot, see sspd_scan_sliding_seav): K1b's final fold
 * then stores its words instead of read-modify-writing them.  Same result
 * as sspd_scan_partitioned on a zeroed buffer. */
SSPD_API int sspd_scan_partitioned_fresh(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                   const sspd_params* p, uint8_t* seav, uint8_t* ldca,
                                   void* scratch, uint64_t scratch_bytes, uint64_t chunk,
                                   void* stream);
SSPD_API uint64_t sspd_scan_partitioned_scratch(const sspd_params* p, uint64_t chunk);
SSPD_API int sspd_scan_partitioned_variant(const sspd_params* p, uint64_t chunk);

/* ---- K2 sliding scan ---------------------------------------------------
 * Replaces SlidingDetector.observe_batch (sliding.py:156-185) with
 * TimestampPool.touch_batch (sliding.py:77-79): plain store of
 * `now_wrapped` into every slot the discrete path would set.
 * pool: p->slot_total timestamps of ts_bytes (1/2/4/8) each. */
SSPD_API int sspd_scan_sliding(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                      const sspd_params* p, void* pool, uint32_t ts_bytes,
                      uint64_t now_wrapped, void* stream);
/* The same with the scan's grid capped at max_blocks_per_sm resident blocks
 * per SM (0 = no cap), leaving room for kernels of another stream -- the
 * pipelined detect of SlidingDetector.detect_async. */
SSPD_API int sspd_scan_sliding_capped(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                      const sspd_params* p, void* pool, uint32_t ts_bytes,
                                      uint64_t now_wrapped, uint32_t max_blocks_per_sm, void* stream);

/* ---- incremental SEAV view of a sliding pool (u16 stamps) ---------------
 * Instead of re-reading the whole SEAV stamp region at every detect
 * (materialize_seav, sliding.py:191-203), SlidingDetector keeps the active
 * SEAV bits up to date:
 *   sspd_scan_sliding_tracked  = sspd_scan_sliding_capped that also ORs
 *       every SEAV stamp's bit into `seav_view` and appends the slot to the
 *       ring `log` (log_entries, a power of two; *log_head counts appends);
 *   sspd_seav_advance          = before TimestampPool.advance_slice
 *       (sliding.py:81-86): records the log head of slice now_abs in
 *       meta[4 + now_abs % nseg] and clears the view bit of every slot of
 *       slice now_abs + 1 - window whose stamp was not renewed (the bits
 *       that turn inactive); sets meta[1] if the ring overwrote live entries;
 *   sspd_materialize_seav_if   = full materialization into seav_view only
 *       when *flag (meta[1]) is set -- the invalidated view stays exact.
 * meta (u64): [0] log head, [1] invalid flag, [4 + s % nseg] segment ends;
 * nseg >= window + 2. */
SSPD_API int sspd_scan_sliding_tracked(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                       const sspd_params* p, void* pool, uint32_t ts_bytes,
                                       uint64_t now_wrapped, uint32_t max_blocks_per_sm,
                                       uint8_t* seav_view, uint32_t* log, uint64_t log_entries,
                                       unsigned long long* log_head, void* stream);
SSPD_API int sspd_seav_advance(const void* pool, uint32_t ts_bytes, const sspd_params* p,
                               uint8_t* seav_view, const uint32_t* log, uint64_t log_entries,
                               unsigned long long* meta, uint32_t nseg, uint64_t now_abs,
                               uint64_t window_slices, void* stream);
SSPD_API int sspd_materialize_seav_if(const void* pool, uint32_t ts_bytes, const sspd_params* p,
                                      uint64_t now_wrapped, uint64_t window_slices, uint8_t* seav_out,
                                      const unsigned long long* flag, void* stream);

/* ---- deferred LDCA stamps of a sliding pool (u16 stamps) ---------------
 * touch_batch (sliding.py:77-79) stores `now` into every LDCA slot a packet
 * selects -- 8 random 2-byte stores per packet into a region larger than L2.
 * Within one slice every such store writes the same value, so the scan may
 * instead record the slot in an LDCA-shaped dirty bitmap (ldca_bytes):
 *   sspd_scan_sliding_deferred = sspd_scan_sliding_tracked (seav_view may be
 *       NULL: no tracking) whose LDCA stamps go to `ldca_dirty` (may be
 *       NULL: stored directly) -- for every geometry and input alignment
 *       (a generic u16 kernel when the fast path does not apply);
 *   sspd_ldca_fold             = stamp now_wrapped into every dirty slot and
 *       clear the bitmap; with ldca_view != NULL also write the packed
 *       active-bit LDCA (as sspd_materialize_ldca after the fold) in the
 *       same pass.  Must run before the slice advances or the stamps are
 *       read (SlidingDetector does; TimestampPool.flush).
 * SSPD_ERR_CONFIG when the stamps are not u16 / the layout is not 8-slot
 * aligned. */
/* sspd_scan_sliding_seav = the SEAV half of sspd_scan_sliding_deferred
 *       (SEAV stamps + optional tracking, no LDCA slot); with
 *       sspd_scan_partitioned(seav = NULL, ldca = the slice's dirty bitmap)
 *       for the LDCA half it records exactly what the deferred scan does. */
SSPD_API int sspd_scan_sliding_seav(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                    const sspd_params* p, void* pool, uint32_t ts_bytes, uint64_t now_wrapped,
                                    uint32_t max_blocks_per_sm, uint8_t* seav_view, uint32_t* log,
                                    uint64_t log_entries, unsigned long long* log_head, void* stream);
/* sspd_scan_sliding_partitioned = both halves of one sliding slice in ONE
 *       launch of the partitioned scan K1b: the LDCA half into the slice's
 *       dirty bitmap `dirty` (dirty_fresh: it holds only zeros), the SEAV
 *       stamps (+ optional view and slot log) from K1b's sampled-packet
 *       queue.  Same state as sspd_scan_partitioned(seav = NULL, ldca =
 *       dirty) + sspd_scan_sliding_seav (observe_batch, sliding.py:156-185);
 *       u16 stamps only; SSPD_ERR_CONFIG when K1b does not apply. */
SSPD_API int sspd_scan_sliding_partitioned(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                           const sspd_params* p, void* pool, uint32_t ts_bytes,
                                           uint64_t now_wrapped, uint8_t* seav_view, uint32_t* log,
                                           uint64_t log_entries, unsigned long long* log_head, uint8_t* dirty,
                                           int dirty_fresh, void* scratch, uint64_t scratch_bytes,
                                           uint64_t chunk, void* stream);
SSPD_API int sspd_scan_sliding_deferred(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                        const sspd_params* p, void* pool, uint32_t ts_bytes,
                                        uint64_t now_wrapped, uint32_t max_blocks_per_sm,
                                        uint8_t* seav_view, uint32_t* log, uint64_t log_entries,
                                        unsigned long long* log_head, uint32_t* ldca_dirty, void* stream);
SSPD_API int sspd_ldca_fold(void* pool, uint32_t ts_bytes, const sspd_params* p, uint32_t* ldca_dirty,
                            uint64_t now_wrapped, uint64_t window_slices, uint8_t* ldca_view, void* stream);

/* Ring mode of the deferred LDCA stamps (SlidingDetector keeps the dirty
 * bitmap of every slice of the window, slot = slice % ring_slots; a slot is
 * active iff stamped in one of the last w slices, sliding.py:98-106, so the
 * packed view of materialize_ldca (sliding.py:215-220) is an OR of bitmaps):
 *   sspd_ldca_window_or = acc |= cur; view = acc | suffix; zero[:] = 0 (each
 *       pointer may be NULL; 16-byte aligned, nbytes % 4 == 0);
 *   sspd_ldca_fold_ring = TimestampPool.touch_batch of the LDCA slots for the
 *       ring slices [slice_lo, slice_hi], newest slice winning (stamp =
 *       slice & 0xFFFF); slice e's bitmap starts at byte
 *       (e % ring_slots) * slot_stride_bytes of `ring` (stride >= ldca_bytes,
 *       a multiple of 4); slice_hi - slice_lo < ring_slots;
 *   sspd_ldca_suffix_or = in place, bitmap of slice e <- OR of slices
 *       e .. first_slice + count - 1 (the two-stack suffix pass at a block end). */
SSPD_API int sspd_ldca_window_or(const uint32_t* cur, uint32_t* acc, const uint32_t* suffix, uint32_t* view,
                                 uint32_t* zero, uint64_t nbytes, void* stream);
SSPD_API int sspd_ldca_fold_ring(void* pool, uint32_t ts_bytes, const sspd_params* p, const uint32_t* ring,
                                 uint64_t slot_stride_bytes, uint32_t ring_slots, uint64_t slice_lo,
                                 uint64_t slice_hi, void* stream);
SSPD_API int sspd_ldca_suffix_or(uint32_t* ring, uint32_t ring_slots, uint64_t nbytes, uint64_t first_slice,
                                 uint64_t count, void* stream);

/* ---- K3 sweep: TimestampPool._sweep (sliding.py:88-94) ---------------- */
SSPD_API int sspd_sweep(void* pool, uint64_t n_slots, uint32_t ts_bytes,
               uint64_t now_wrapped, uint64_t window_slices,
               uint64_t clamp_value, void* stream);

/* TimestampPool.touch_batch (sliding.py:77-79): pool[slot_indexes[j]] =
 * now_wrapped for j < n (int64 device indexes; negative ones count from
 * the end, as numpy's).  An index outside [-n_slots, n_slots) is skipped
 * and ORs 1 into *bad_flag (device u32, may be NULL).  The Python host
 * checks the bounds first and raises IndexError before any store, as the
 * reference's numpy fancy-index store does. */
SSPD_API int sspd_touch_slots(void* pool, uint64_t n_slots, uint32_t ts_bytes,
               const int64_t* slot_indexes, uint64_t n, uint64_t now_wrapped,
               uint32_t* bad_flag, void* stream);

/* ---- K4 materialize ----------------------------------------------------
 * materialize_seav (sliding.py:191-203): active slots -> SEAV payload.
 * materialize_ldca (sliding.py:215-220): active slots -> packed LDCA bytes.
 * active  <=>  ((now_wrapped - ts) & mask) < window_slices. */
SSPD_API int sspd_materialize_seav(const void* pool, uint32_t ts_bytes,
                          const sspd_params* p, uint64_t now_wrapped,
                          uint64_t window_slices, uint8_t* seav_out,
                          void* stream);
SSPD_API int sspd_materialize_ldca(const void* pool, uint32_t ts_bytes,
                          const sspd_params* p, uint64_t now_wrapped,
                          uint64_t window_slices, uint8_t* ldca_out,
                          void* stream);
/* pool ages: ((now_wrapped - ts) & mask) as uint64 (TimestampPool.ages,
 * sliding.py:96-98) */
SSPD_API int sspd_pool_ages(const void* pool, uint64_t n_slots, uint32_t ts_bytes,
                   uint64_t now_wrapped, uint64_t* ages_out, void* stream);

/* ---- K5 restore --------------------------------------------------------
 * Replaces SeavSketch.restore_sea / restore (short_sketch.py:347-408).
 * For every register array rp in [rp_begin, rp_begin+rp_count):
 *   counts the consistent all-hot tuples (exact up to cap+1),
 *   sets overflow[rp-rp_begin]=1 when the count exceeds `cap`,
 *   otherwise emits every tuple whose register AND has weight >= 3 as
 *   (ip, (rp<<8)|weight) -- unsorted.
 * out_count (device uint64) receives the number of candidates found; when
 * it exceeds out_capacity nothing beyond capacity is written and the host
 * retries with a larger buffer.  Entries are sorted by ip by
 * sspd_sort_candidates. */
SSPD_API int sspd_restore(const uint8_t* seav, const sspd_params* p,
                 uint32_t rp_begin, uint32_t rp_count, uint64_t cap,
                 uint32_t* out_ip, uint32_t* out_aux, uint64_t out_capacity,
                 unsigned long long* out_count, uint8_t* overflow,
                 void* stream);

/* Sort (ip, aux) pairs by ip ascending on the device (restore's
 * `sorted(found)`, short_sketch.py:408).  scratch may be NULL to query
 * *scratch_bytes. */
SSPD_API int sspd_sort_candidates(uint32_t* ip, uint32_t* aux, uint64_t n,
                         void* scratch, size_t* scratch_bytes, void* stream);

/* ---- K6 filter ---------------------------------------------------------
 * Replaces LdcaSketch.union_register/estimate (long_sketch.py:137-148) and
 * the keep test of finalize_window (window_detector.py:105-125):
 *   z0[j] = k - popcount(AND_i data[i, c_i(ip_j)])
 *   keep[j] = keep_table[z0[j]]   (host-built table of k+1 bytes that holds
 *             the reference float test `saturated or est >= beta*theta`
 *             evaluated once per possible z0, so the device stays integer)
 * keep may be NULL. */
SSPD_API int sspd_filter(const uint8_t* ldca, const sspd_params* p,
                const uint32_t* ips, uint64_t n, const uint8_t* keep_table,
                uint32_t* z0_out, uint8_t* keep_out, void* stream);

/* Sliding filter: the same on the active view of the timestamp pool
 * (SlidingDetector._estimate, sliding.py:222-230). */
SSPD_API int sspd_filter_sliding(const void* pool, uint32_t ts_bytes,
                        const sspd_params* p, uint64_t now_wrapped,
                        uint64_t window_slices, const uint32_t* ips,
                        uint64_t n, const uint8_t* keep_table,
                        uint32_t* z0_out, uint8_t* keep_out, void* stream);

/* Stable compaction of (ip, z0) by keep flag; *out_count (device). */
SSPD_API int sspd_compact_reports(const uint32_t* ip, const uint32_t* z0,
                         const uint8_t* keep, uint64_t n, uint32_t* ip_out,
                         uint32_t* z0_out, unsigned long long* out_count,
                         void* scratch, size_t* scratch_bytes, void* stream);

/* ---- fused finalize (K5 + sort + K6 + compaction, no host round trip) ----
 * DetectorState.finalize_window (window_detector.py:105-125) /
 * SlidingDetector.detect on a materialised LDCA view (sliding.py:232-248):
 * restore with cap `restore_cap` into `capacity` candidate slots, sort by
 * ip, filter against `ldca` with the host-built keep table, stable
 * compaction into out_ip/out_z0 (capacity entries each).  counts (device,
 * 2 x u64): [0] candidates found -- if it exceeds `capacity` the outputs
 * are incomplete and the caller re-runs with a larger capacity -- and [1]
 * reports kept.  overflow (device, 2^r + 1 bytes): 1 for every register
 * array dropped by the cap; byte [2^r] = 1 when the bucket sort met a
 * bucket it cannot order (skewed addresses): the outputs are then invalid
 * and the caller re-runs with flags bit 0 (radix sort).  scratch NULL
 * queries *scratch_bytes. */
SSPD_API int sspd_finalize(const uint8_t* seav, const uint8_t* ldca, const sspd_params* p,
                           uint64_t restore_cap, const uint8_t* keep_table, uint64_t capacity,
                           uint32_t* out_ip, uint32_t* out_z0, unsigned long long* counts,
                           uint8_t* overflow, void* scratch, size_t* scratch_bytes, uint32_t flags,
                           void* stream);

/* ---- K7 merge ----------------------------------------------------------
 * Bytewise OR of n_src equal-length buffers into dst (dst may alias
 * srcs[0]).  Sources may be peer-GPU pointers (CUDA IPC / P2P mapped):
 * replaces merge_frames' payload OR (distributed.py:167-169),
 * SeavSketch.merge (short_sketch.py:326-331), LdcaSketch.merge
 * (long_sketch.py:150-153).  srcs is a HOST array of device pointers. */
SSPD_API int sspd_merge_or(const void* const* srcs, int n_src, void* dst,
                  uint64_t bytes, void* stream);

/* ---- K8 merge_age_min --------------------------------------------------
 * merge_timestamp_pools (distributed.py:176-192): per slot, the smallest
 * wrapped age over all pools wins; dst = (now - min_age) & mask. */
SSPD_API int sspd_merge_age_min(const void* const* srcs, int n_src, void* dst,
                       uint64_t n_slots, uint32_t ts_bytes,
                       uint64_t now_wrapped, void* stream);

/* ---- route_pairs on the device (distributed.py:195-210) ---------------
 * mode 0 = "hash": mix64(((hip<<32)|oip) ^ seed_route) % n_wp
 * mode 1 = "round-robin": (index_base + j) % n_wp */
SSPD_API int sspd_route_pairs(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                     const sspd_params* p, const sspd_divisor* n_wp,
                     int mode, uint64_t index_base, int64_t* lanes_out,
                     void* stream);

/* ---- roofline microbenchmark ------------------------------------------
 * Random red.global.or.b32 over `bytes` of device memory (pow2), issued the
 * way the scan issues them; returns achieved ops/s in *ops_per_s.  Used by
 * bench.py for the L2-atomic term of the scan roofline. */
SSPD_API int sspd_microbench_red(void* buf, uint64_t bytes, int blocks_per_sm,
                        int iters, double* ops_per_s, void* stream);
/* The scans' compute floor: packets/s of streaming the caller's (16-B
 * aligned) pairs and evaluating every per-packet hash the partitioned scans
 * evaluate (H3 % k, the H1 sampling test, LR row hashes % lc; k and lc
 * powers of two), with no sketch update -- at blocks_per_sm = 1 or 2
 * CTAs of 1,024 threads per SM (1 = the scans' launch shape, 2 = full
 * occupancy).  sink: >= 2048 x SMs
 * words.  The binding roofline of K1b (bench.py `roofline.binding`). */
SSPD_API int sspd_microbench_hash(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                  const sspd_params* p, int blocks_per_sm, uint32_t* sink,
                                  double* pkts_per_s, void* stream);
/* Self-check of the scans' 32-bit-key hash (mix64_lo_fast: low word of
 * SplitMix64, hashing.py:48-53, evaluated in 32-bit halves) against the
 * 64-bit definition for every key in [key0, key0 + nkeys) (<= 2^32):
 * *mismatches = count, *first_bad = smallest mismatching key (~0 if none). */
SSPD_API int sspd_check_hash32(uint64_t seed, uint64_t key0, uint64_t nkeys, uint64_t* mismatches,
                               uint64_t* first_bad, void* stream);
/* Random st.global.u16 rate over a `bytes` (power of two) footprint -- the
 * measured roofline term of the sliding scan K2. */
SSPD_API int sspd_microbench_store16(void* buf, uint64_t bytes, int blocks_per_sm,
                                     int iters, double* ops_per_s, void* stream);

/* ---- multi-GPU plumbing (CUDA IPC) -------------------------------------
 * One cudaMalloc block per rank holds SEAV+LDCA; its 64-byte IPC handle is
 * exchanged over torch.distributed and opened by the peers, whose merge
 * kernels (sspd_merge_or) then read it over NVLink.  Replaces the
 * in-process frame list of simulate_window (distributed.py:231-271). */
SSPD_API int sspd_ipc_alloc(uint64_t bytes, void** ptr);
SSPD_API int sspd_ipc_free(void* ptr);
SSPD_API int sspd_ipc_get_handle(void* ptr, uint8_t* handle_out /* 64 B */);
SSPD_API int sspd_ipc_open(const uint8_t* handle /* 64 B */, void** ptr);
SSPD_API int sspd_ipc_close(void* ptr);
SSPD_API int sspd_copy_async(void* dst, const void* src, uint64_t bytes, void* stream);

/* ---- ingest and frames ---------------------------------
 * sspd_unpack_records: the reference trace format, n little-endian 12-byte
 * records (slice u32, hip u32, oip u32) (evaluation.py:21, read_trace
 * :235-254), into SoA device arrays; slices may be NULL.
 * sspd_crc32: zlib.crc32 of a device buffer (the frame checksum of
 * serialize/parse_frame, distributed.py:81-126); scratch NULL queries
 * *scratch_bytes; *out (device uint32) receives the CRC. */
SSPD_API int sspd_unpack_records(const uint8_t* records, uint64_t n, uint32_t* slices,
                                 uint32_t* hips, uint32_t* oips, void* stream);
SSPD_API int sspd_crc32(const uint8_t* data, uint64_t n, uint32_t* out, void* scratch,
                        uint64_t* scratch_bytes, void* stream);

/* ---- exact oracle --------------------------------
 * Replaces ExactOracle.__init__ (evaluation.py:35-40): sort-unique of the
 * keys (hip << 32 | oip), then distinct keys counted per host.  Writes the
 * hosts ascending to hosts_out and their distinct-peer counts to
 * counts_out (both sized n by the caller: at most n hosts), and the host
 * count to *n_hosts_out (device).  scratch NULL queries *scratch_bytes
 * (about 24 B per packet).  n < 2^31.  Evaluation infrastructure, not on
 * the scan path. */
SSPD_API int sspd_exact_cardinalities(const uint32_t* hips, const uint32_t* oips, uint64_t n,
                                      uint32_t* hosts_out, uint32_t* counts_out,
                                      unsigned long long* n_hosts_out, void* scratch,
                                      size_t* scratch_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSPD_B200_H */
