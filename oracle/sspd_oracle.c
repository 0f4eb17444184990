/*
 * sspd_oracle.c -- CPU restatement of the reference algorithm for the
 * packet-scan / estimate path.  TEST INFRASTRUCTURE ONLY: it is the checker
 * for the CUDA kernels (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline / --impl reference legs).  The product never links it.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function below
 * against golden vectors produced by running the reference package itself
 * (tests/golden/make_golden.py).
 *
 * Written as plain loops over the reference's own definitions -- `%` for
 * hash_range, the bit-by-bit index_of, a recursive depth-first restore with
 * the reference's prune test -- deliberately NOT sharing code with the
 * device kernels.  Geometry is read from the same POD parameter block the
 * product uses (include/sspd_b200.h), which is only data.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/sspd_b200.h"

/* hashing.py:48-53 */
uint64_t or_mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* hashing.py:64-67 */
uint64_t or_derive_seed(uint64_t master, uint32_t tag) {
  return or_mix64(master ^ ((uint64_t)(tag & 0xFFu) * 0x9E3779B97F4A7C15ull));
}

/* hashing.py:120-124: hash64(key, seed) % m, full 64-bit value */
uint64_t or_hash_range(uint64_t key, uint64_t seed, uint64_t m) { return or_mix64(key ^ seed) % m; }

/* hashing.py:133-141 */
static int or_lsb32(uint32_t x) {
  if (x == 0) return 32;
  int i = 0;
  while (!((x >> i) & 1u)) ++i;
  return i;
}

/* short_sketch.py:183-193, bit by bit */
static uint64_t or_index_of(const sspd_params* p, uint32_t row, uint64_t lp) {
  uint64_t idx = 0;
  for (uint32_t j = 0; j < p->ibn[row]; ++j) idx |= ((lp >> ((p->isb[row] + j) % p->lp_bits)) & 1ull) << j;
  return idx;
}

static uint64_t or_get_reg(const uint8_t* base, uint32_t rb) {
  uint64_t v = 0;
  for (uint32_t b = 0; b < rb; ++b) v |= (uint64_t)base[b] << (8 * b); /* little-endian */
  return v;
}
static void or_put_reg(uint8_t* base, uint32_t rb, uint64_t v) {
  for (uint32_t b = 0; b < rb; ++b) base[b] = (uint8_t)(v >> (8 * b));
}

/* SeavSketch.update (short_sketch.py:289-298) for one pair */
static void or_seav_pair(const sspd_params* p, uint64_t hip, uint64_t oip, uint8_t* seav) {
  uint32_t h1 = (uint32_t)(or_mix64(oip ^ p->seed_h1) & 0xFFFFFFFFull);
  if (or_lsb32(h1) < (int)p->tau) return;
  uint64_t bit = 1ull << or_hash_range(oip, p->seed_h2, p->g);
  uint64_t rp = hip & ((1ull << p->r) - 1ull);
  uint64_t lp = (hip >> p->r) & ((1ull << p->lp_bits) - 1ull);
  for (uint32_t i = 0; i < p->sr; ++i) {
    uint64_t col = or_index_of(p, i, lp);
    uint8_t* reg = seav + p->seav_row_off[i] + (rp * p->sc[i] + col) * p->reg_bytes;
    or_put_reg(reg, p->reg_bytes, or_get_reg(reg, p->reg_bytes) | bit);
  }
}

/* LdcaSketch.update (long_sketch.py:116-123): data[i, c, b>>3] |= 1<<(b&7) */
static void or_ldca_pair(const sspd_params* p, uint64_t hip, uint64_t oip, uint8_t* ldca) {
  uint64_t b = or_hash_range(oip, p->seed_h3, p->k);
  uint64_t kb = p->k / 8;
  for (uint32_t i = 0; i < p->lr; ++i) {
    uint64_t c = or_hash_range(hip, p->seed_lh[i], p->lc);
    ldca[((uint64_t)i * p->lc + c) * kb + (b >> 3)] |= (uint8_t)(1u << (b & 7));
  }
}

void or_seav_update(const sspd_params* p, const uint32_t* hips, const uint32_t* oips, uint64_t n, uint8_t* seav) {
  for (uint64_t j = 0; j < n; ++j) or_seav_pair(p, hips[j], oips[j], seav);
}

void or_ldca_update(const sspd_params* p, const uint32_t* hips, const uint32_t* oips, uint64_t n, uint8_t* ldca) {
  for (uint64_t j = 0; j < n; ++j) or_ldca_pair(p, hips[j], oips[j], ldca);
}

/* DetectorState.process_batch (window_detector.py:100-103) on nthreads.
 * Work is split by SKETCH ROW (LDCA row i, or the whole SEAV) so each
 * thread's working set is one 1 MiB row that stays in its private cache;
 * the (row task x packet) space is cut into nthreads equal ranges, and a
 * task shared by several threads is OR-ed with relaxed atomics (exact: OR
 * is monotone). */
typedef struct {
  const sspd_params* p;
  const uint32_t* hips;
  const uint32_t* oips;
  uint64_t lo, hi;
  int row;      /* LDCA row, or -1 for the SEAV task */
  uint8_t* out; /* the LDCA row / the SEAV, or a private zeroed copy of it */
  uint8_t* dst; /* where a private copy is OR-ed after the join (NULL: out is dst) */
  uint64_t bytes;
} or_job;

static void* or_scan_job(void* arg) {
  or_job* j = (or_job*)arg;
  const sspd_params* p = j->p;
  if (j->row < 0) {
    for (uint64_t t = j->lo; t < j->hi; ++t) or_seav_pair(p, j->hips[t], j->oips[t], j->out);
    return NULL;
  }
  const uint64_t kb = p->k / 8;
  const uint64_t seed = p->seed_lh[j->row];
  for (uint64_t t = j->lo; t < j->hi; ++t) {
    uint64_t b = or_hash_range(j->oips[t], p->seed_h3, p->k);
    uint64_t c = or_hash_range(j->hips[t], seed, p->lc);
    j->out[c * kb + (b >> 3)] |= (uint8_t)(1u << (b & 7));
  }
  return NULL;
}

/* one thread's jobs (at most a few), run in order */
typedef struct {
  or_job* jobs;
  int count;
} or_run;

static void* or_run_jobs(void* a) {
  or_run* r = (or_run*)a;
  for (int i = 0; i < r->count; ++i) or_scan_job(&r->jobs[i]);
  return NULL;
}

int or_scan(const sspd_params* p, const uint32_t* hips, const uint32_t* oips, uint64_t n, uint8_t* seav,
            uint8_t* ldca, int nthreads) {
  if (nthreads <= 1 || n < 4096) {
    for (uint64_t t = 0; t < n; ++t) {
      if (seav) or_seav_pair(p, hips[t], oips[t], seav);
      if (ldca) or_ldca_pair(p, hips[t], oips[t], ldca);
    }
    return 0;
  }
  /* the (task, packet) work space is cut into nthreads equal contiguous
   * ranges, so every thread is busy; a task covered by several ranges is
   * scanned into private zeroed copies that are OR-ed in after the join
   * (exact: OR is commutative and idempotent) */
  const int tasks = (ldca ? (int)p->lr : 0) + (seav ? 1 : 0);
  if (tasks == 0) return 0;
  const uint64_t units = (uint64_t)tasks * n;
  const uint64_t row_bytes = (uint64_t)p->lc * (p->k / 8);
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  or_job* jobs = (or_job*)calloc((size_t)nthreads + (size_t)tasks + 1, sizeof(or_job));  /* pieces <= tasks + nthreads - 1 */
  int* first = (int*)calloc((size_t)nthreads + 1, sizeof(int));
  int nj = 0;
  for (int t = 0; t < nthreads; ++t) {
    const uint64_t u0 = units * (uint64_t)t / (uint64_t)nthreads, u1 = units * (uint64_t)(t + 1) / (uint64_t)nthreads;
    first[t] = nj;
    for (uint64_t u = u0; u < u1;) {
      const int task = (int)(u / n);
      const uint64_t lo = u - (uint64_t)task * n;
      const uint64_t hi = (u1 - (uint64_t)task * n) < n ? (u1 - (uint64_t)task * n) : n;
      or_job* j = &jobs[nj++];
      j->p = p;
      j->hips = hips;
      j->oips = oips;
      j->lo = lo;
      j->hi = hi;
      j->row = (ldca && task < (int)p->lr) ? task : -1;
      uint8_t* target = j->row >= 0 ? ldca + (uint64_t)j->row * row_bytes : seav;
      j->bytes = j->row >= 0 ? row_bytes : p->seav_bytes;
      if (lo == 0 && hi == n) {
        j->out = target;
        j->dst = NULL;
      } else {
        j->out = (uint8_t*)calloc(j->bytes, 1);
        j->dst = target;
      }
      u = (uint64_t)task * n + hi;
    }
  }
  first[nthreads] = nj;
  or_run* runs = (or_run*)calloc((size_t)nthreads, sizeof(or_run));
  for (int t = 0; t < nthreads; ++t) {
    runs[t].jobs = &jobs[first[t]];
    runs[t].count = first[t + 1] - first[t];
  }
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, or_run_jobs, &runs[t]);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  for (int q = 0; q < nj; ++q) {
    if (!jobs[q].dst) continue;
    uint64_t* d = (uint64_t*)jobs[q].dst;
    const uint64_t* s8 = (const uint64_t*)jobs[q].out;
    uint64_t words = jobs[q].bytes / 8, tail = jobs[q].bytes % 8;
    for (uint64_t i = 0; i < words; ++i) d[i] |= s8[i];
    for (uint64_t i = 0; i < tail; ++i) jobs[q].dst[words * 8 + i] |= jobs[q].out[words * 8 + i];
    free(jobs[q].out);
  }
  free(runs);
  free(first);
  free(th);
  free(jobs);
  return 0;
}

/* ---- restore (short_sketch.py:347-408) -------------------------------- */
typedef struct {
  const sspd_params* p;
  uint32_t rp;
  uint64_t cap;
  uint64_t survivors;
  int overflow;
  uint32_t* hot_col[SSPD_MAX_SR];
  uint64_t* hot_reg[SSPD_MAX_SR];
  uint32_t nhot[SSPD_MAX_SR];
  uint64_t* scatter[SSPD_MAX_SR]; /* _row_scatter vals (short_sketch.py:224-235) */
  uint64_t row_mask[SSPD_MAX_SR];
  uint32_t* out_ip;
  uint32_t* out_w;
  uint64_t nout, out_cap;
} or_walk;

static void or_walk_rec(or_walk* W, uint32_t i, uint64_t acc_mask, uint64_t acc_lp, uint64_t acc_and) {
  if (W->overflow) return;
  const sspd_params* p = W->p;
  if (i == p->sr) {
    W->survivors += 1;
    if (W->survivors > W->cap) { /* SeaOverflowError (short_sketch.py:375-376) */
      W->overflow = 1;
      return;
    }
    int w = __builtin_popcountll(acc_and);
    if (w >= 3) {
      if (W->nout < W->out_cap) {
        W->out_ip[W->nout] = (uint32_t)((acc_lp << p->r) | W->rp);
        W->out_w[W->nout] = (uint32_t)w;
      }
      W->nout += 1;
    }
    return;
  }
  for (uint32_t h = 0; h < W->nhot[i]; ++h) {
    uint64_t v = W->scatter[i][W->hot_col[i][h]];
    if ((acc_lp ^ v) & (acc_mask & W->row_mask[i])) continue;
    or_walk_rec(W, i + 1, acc_mask | W->row_mask[i], acc_lp | v, acc_and & W->hot_reg[i][h]);
    if (W->overflow) return;
  }
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y);
}

/* Candidates of rp in [rp_begin, rp_begin+rp_count), sorted by ip.  Returns
 * the number of candidates (may exceed out_cap: caller retries).
 * overflow[rp - rp_begin] = 1 for SEAs whose tuple count exceeds cap; they
 * contribute nothing (restore(on_overflow="warn"), short_sketch.py:398-407). */
int64_t or_restore(const sspd_params* p, const uint8_t* seav, uint32_t rp_begin, uint32_t rp_count, uint64_t cap,
                   uint32_t* out_ip, uint32_t* out_w, uint64_t out_cap, uint8_t* overflow) {
  or_walk W;
  memset(&W, 0, sizeof(W));
  W.p = p;
  W.cap = cap;
  const uint64_t full = p->g >= 64 ? ~0ull : ((1ull << p->g) - 1ull);
  for (uint32_t i = 0; i < p->sr; ++i) {
    W.hot_col[i] = (uint32_t*)malloc(sizeof(uint32_t) * p->sc[i]);
    W.hot_reg[i] = (uint64_t*)malloc(sizeof(uint64_t) * p->sc[i]);
    W.scatter[i] = (uint64_t*)malloc(sizeof(uint64_t) * p->sc[i]);
    W.row_mask[i] = 0;
    for (uint32_t j = 0; j < p->ibn[i]; ++j) W.row_mask[i] |= 1ull << ((p->isb[i] + j) % p->lp_bits);
    for (uint64_t c = 0; c < p->sc[i]; ++c) {
      uint64_t v = 0;
      for (uint32_t j = 0; j < p->ibn[i]; ++j)
        if ((c >> j) & 1ull) v |= 1ull << ((p->isb[i] + j) % p->lp_bits);
      W.scatter[i][c] = v;
    }
  }
  /* all candidates of all SEAs, collected then sorted by ip */
  uint64_t cap_all = 1024, nall = 0;
  uint64_t* all = (uint64_t*)malloc(sizeof(uint64_t) * cap_all);
  uint32_t* tmp_ip = NULL;
  uint32_t* tmp_w = NULL;
  uint64_t tmp_cap = 0;
  for (uint32_t k = 0; k < rp_count; ++k) {
    uint32_t rp = rp_begin + k;
    int empty = 0;
    for (uint32_t i = 0; i < p->sr; ++i) {
      W.nhot[i] = 0;
      const uint8_t* row = seav + p->seav_row_off[i] + (uint64_t)rp * p->sc[i] * p->reg_bytes;
      for (uint32_t c = 0; c < p->sc[i]; ++c) {
        uint64_t reg = or_get_reg(row + (uint64_t)c * p->reg_bytes, p->reg_bytes);
        if (__builtin_popcountll(reg) >= 3) {
          W.hot_col[i][W.nhot[i]] = c;
          W.hot_reg[i][W.nhot[i]] = reg;
          W.nhot[i]++;
        }
      }
      if (W.nhot[i] == 0) empty = 1;
    }
    if (overflow) overflow[k] = 0;
    if (empty) continue;
    W.rp = rp;
    W.survivors = 0;
    W.overflow = 0;
    for (;;) {
      W.nout = 0;
      W.out_ip = tmp_ip;
      W.out_w = tmp_w;
      W.out_cap = tmp_cap;
      W.survivors = 0;
      W.overflow = 0;
      or_walk_rec(&W, 0, 0, 0, full);
      if (W.overflow || W.nout <= tmp_cap) break;
      tmp_cap = W.nout;
      tmp_ip = (uint32_t*)realloc(tmp_ip, sizeof(uint32_t) * tmp_cap);
      tmp_w = (uint32_t*)realloc(tmp_w, sizeof(uint32_t) * tmp_cap);
    }
    if (W.overflow) {
      if (overflow) overflow[k] = 1;
      continue;
    }
    for (uint64_t t = 0; t < W.nout; ++t) {
      if (nall == cap_all) {
        cap_all *= 2;
        all = (uint64_t*)realloc(all, sizeof(uint64_t) * cap_all);
      }
      all[nall++] = ((uint64_t)tmp_ip[t] << 32) | ((uint64_t)rp << 8) | tmp_w[t];
    }
  }
  qsort(all, nall, sizeof(uint64_t), cmp_u64);
  for (uint64_t t = 0; t < nall && t < out_cap; ++t) {
    out_ip[t] = (uint32_t)(all[t] >> 32);
    out_w[t] = (uint32_t)(all[t] & 0xFFFFFFFFu); /* (rp << 8) | weight */
  }
  for (uint32_t i = 0; i < p->sr; ++i) {
    free(W.hot_col[i]);
    free(W.hot_reg[i]);
    free(W.scatter[i]);
  }
  free(all);
  free(tmp_ip);
  free(tmp_w);
  return (int64_t)nall;
}

/* LdcaSketch.union_register / estimate (long_sketch.py:137-148): z0 */
void or_filter(const sspd_params* p, const uint8_t* ldca, const uint32_t* ips, uint64_t n, uint32_t* z0) {
  uint64_t kb = p->k / 8;
  for (uint64_t j = 0; j < n; ++j) {
    uint64_t cell[SSPD_MAX_LR];
    for (uint32_t i = 0; i < p->lr; ++i) cell[i] = (uint64_t)i * p->lc + or_hash_range(ips[j], p->seed_lh[i], p->lc);
    uint32_t pop = 0;
    for (uint64_t by = 0; by < kb; ++by) {
      uint8_t acc = 0xFF;
      for (uint32_t i = 0; i < p->lr; ++i) acc &= ldca[cell[i] * kb + by];
      pop += (uint32_t)__builtin_popcount(acc);
    }
    z0[j] = p->k - pop;
  }
}

/* ---- the same restore / filter on nthreads (CPU baseline) --------------
 * Restore: SEAs are independent, so the rp range is cut into nthreads
 * contiguous pieces restored concurrently, then the candidates are merged
 * and sorted by ip exactly as or_restore does.  Filter: candidates cut into
 * nthreads pieces. */
typedef struct {
  const sspd_params* p;
  const uint8_t* seav;
  uint32_t rp_begin, rp_count;
  uint64_t cap;
  uint8_t* overflow;
  uint32_t* ip;
  uint32_t* w;
  int64_t n;
} or_restore_job;

static void* or_restore_run(void* a) {
  or_restore_job* j = (or_restore_job*)a;
  uint64_t capacity = 1024;
  for (;;) {
    j->ip = (uint32_t*)realloc(j->ip, sizeof(uint32_t) * capacity);
    j->w = (uint32_t*)realloc(j->w, sizeof(uint32_t) * capacity);
    j->n = or_restore(j->p, j->seav, j->rp_begin, j->rp_count, j->cap, j->ip, j->w, capacity, j->overflow);
    if ((uint64_t)j->n <= capacity) break;
    capacity = (uint64_t)j->n;
  }
  return NULL;
}

int64_t or_restore_mt(const sspd_params* p, const uint8_t* seav, uint32_t rp_begin, uint32_t rp_count, uint64_t cap,
                      uint32_t* out_ip, uint32_t* out_w, uint64_t out_cap, uint8_t* overflow, int nthreads) {
  if (nthreads <= 1 || rp_count < 2 * (uint32_t)nthreads)
    return or_restore(p, seav, rp_begin, rp_count, cap, out_ip, out_w, out_cap, overflow);
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  or_restore_job* jobs = (or_restore_job*)calloc((size_t)nthreads, sizeof(or_restore_job));
  for (int t = 0; t < nthreads; ++t) {
    const uint32_t a = (uint32_t)((uint64_t)rp_count * t / nthreads), b = (uint32_t)((uint64_t)rp_count * (t + 1) / nthreads);
    jobs[t].p = p;
    jobs[t].seav = seav;
    jobs[t].rp_begin = rp_begin + a;
    jobs[t].rp_count = b - a;
    jobs[t].cap = cap;
    jobs[t].overflow = overflow ? overflow + a : NULL;
    pthread_create(&th[t], NULL, or_restore_run, &jobs[t]);
  }
  uint64_t nall = 0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    nall += (uint64_t)jobs[t].n;
  }
  uint64_t* all = (uint64_t*)malloc(sizeof(uint64_t) * (nall ? nall : 1));
  uint64_t q = 0;
  for (int t = 0; t < nthreads; ++t) {
    for (int64_t i = 0; i < jobs[t].n; ++i) all[q++] = ((uint64_t)jobs[t].ip[i] << 32) | jobs[t].w[i];
    free(jobs[t].ip);
    free(jobs[t].w);
  }
  qsort(all, nall, sizeof(uint64_t), cmp_u64);
  for (uint64_t t = 0; t < nall && t < out_cap; ++t) {
    out_ip[t] = (uint32_t)(all[t] >> 32);
    out_w[t] = (uint32_t)(all[t] & 0xFFFFFFFFu);
  }
  free(all);
  free(jobs);
  free(th);
  return (int64_t)nall;
}

typedef struct {
  const sspd_params* p;
  const uint8_t* ldca;
  const uint32_t* ips;
  uint64_t n;
  uint32_t* z0;
} or_filter_job;

static void* or_filter_run(void* a) {
  or_filter_job* j = (or_filter_job*)a;
  or_filter(j->p, j->ldca, j->ips, j->n, j->z0);
  return NULL;
}

void or_filter_mt(const sspd_params* p, const uint8_t* ldca, const uint32_t* ips, uint64_t n, uint32_t* z0,
                  int nthreads) {
  if (nthreads <= 1 || n < 64) {
    or_filter(p, ldca, ips, n, z0);
    return;
  }
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  or_filter_job* jobs = (or_filter_job*)calloc((size_t)nthreads, sizeof(or_filter_job));
  for (int t = 0; t < nthreads; ++t) {
    const uint64_t a = n * (uint64_t)t / (uint64_t)nthreads, b = n * (uint64_t)(t + 1) / (uint64_t)nthreads;
    jobs[t] = (or_filter_job){p, ldca, ips + a, b - a, z0 + a};
    pthread_create(&th[t], NULL, or_filter_run, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(jobs);
  free(th);
}

/* ---- sliding (sliding.py:24-248) -------------------------------------- */
static uint64_t or_ts_get(const void* pool, uint32_t tb, uint64_t s) {
  switch (tb) {
    case 1: return ((const uint8_t*)pool)[s];
    case 2: return ((const uint16_t*)pool)[s];
    case 4: return ((const uint32_t*)pool)[s];
    default: return ((const uint64_t*)pool)[s];
  }
}
static void or_ts_set(void* pool, uint32_t tb, uint64_t s, uint64_t v) {
  switch (tb) {
    case 1: ((uint8_t*)pool)[s] = (uint8_t)v; break;
    case 2: ((uint16_t*)pool)[s] = (uint16_t)v; break;
    case 4: ((uint32_t*)pool)[s] = (uint32_t)v; break;
    default: ((uint64_t*)pool)[s] = v; break;
  }
}
static uint64_t or_ts_mask(uint32_t tb) { return tb >= 8 ? ~0ull : ((1ull << (8 * tb)) - 1ull); }

/* SlidingDetector.observe_batch (sliding.py:156-185) + touch_batch (:77-79) */
void or_observe(const sspd_params* p, const uint32_t* hips, const uint32_t* oips, uint64_t n, void* pool,
                uint32_t tb, uint64_t now_wrapped) {
  for (uint64_t j = 0; j < n; ++j) {
    uint64_t hip = hips[j], oip = oips[j];
    uint32_t h1 = (uint32_t)(or_mix64(oip ^ p->seed_h1) & 0xFFFFFFFFull);
    if (or_lsb32(h1) >= (int)p->tau) {
      uint64_t bitpos = or_hash_range(oip, p->seed_h2, p->g);
      uint64_t rp = hip & ((1ull << p->r) - 1ull);
      uint64_t lp = (hip >> p->r) & ((1ull << p->lp_bits) - 1ull);
      for (uint32_t i = 0; i < p->sr; ++i) {
        uint64_t col = or_index_of(p, i, lp);
        or_ts_set(pool, tb, p->slot_row_base[i] + (rp * p->sc[i] + col) * p->g + bitpos, now_wrapped);
      }
    }
    uint64_t b = or_hash_range(oip, p->seed_h3, p->k);
    for (uint32_t i = 0; i < p->lr; ++i) {
      uint64_t c = or_hash_range(hip, p->seed_lh[i], p->lc);
      or_ts_set(pool, tb, p->slot_ldca_base + ((uint64_t)i * p->lc + c) * p->k + b, now_wrapped);
    }
  }
}

/* TimestampPool._sweep (sliding.py:88-94) */
void or_sweep(void* pool, uint64_t n, uint32_t tb, uint64_t now_wrapped, uint64_t window, uint64_t clamp) {
  uint64_t m = or_ts_mask(tb);
  for (uint64_t s = 0; s < n; ++s)
    if (((now_wrapped - or_ts_get(pool, tb, s)) & m) >= window) or_ts_set(pool, tb, s, clamp);
}

/* materialize_seav (sliding.py:191-203) */
void or_materialize_seav(const sspd_params* p, const void* pool, uint32_t tb, uint64_t now_wrapped,
                         uint64_t window, uint8_t* seav_out) {
  uint64_t m = or_ts_mask(tb);
  for (uint32_t i = 0; i < p->sr; ++i) {
    uint64_t regs = ((uint64_t)p->sc[i]) << p->r;
    for (uint64_t q = 0; q < regs; ++q) {
      uint64_t v = 0;
      for (uint32_t b = 0; b < p->g; ++b) {
        uint64_t ts = or_ts_get(pool, tb, p->slot_row_base[i] + q * p->g + b);
        if (((now_wrapped - ts) & m) < window) v |= 1ull << b;
      }
      or_put_reg(seav_out + p->seav_row_off[i] + q * p->reg_bytes, p->reg_bytes, v);
    }
  }
}

/* materialize_ldca (sliding.py:215-220), packbits little */
void or_materialize_ldca(const sspd_params* p, const void* pool, uint32_t tb, uint64_t now_wrapped,
                         uint64_t window, uint8_t* ldca_out) {
  uint64_t m = or_ts_mask(tb);
  uint64_t nbits = (uint64_t)p->lr * p->lc * p->k;
  memset(ldca_out, 0, nbits / 8);
  for (uint64_t s = 0; s < nbits; ++s) {
    uint64_t ts = or_ts_get(pool, tb, p->slot_ldca_base + s);
    if (((now_wrapped - ts) & m) < window) ldca_out[s >> 3] |= (uint8_t)(1u << (s & 7));
  }
}

/* merge_timestamp_pools (distributed.py:176-192) */
void or_merge_age_min(const void* const* pools, int npools, void* out, uint64_t n, uint32_t tb,
                      uint64_t now_wrapped) {
  uint64_t m = or_ts_mask(tb);
  for (uint64_t s = 0; s < n; ++s) {
    uint64_t best = (now_wrapped - or_ts_get(pools[0], tb, s)) & m;
    for (int q = 1; q < npools; ++q) {
      uint64_t a = (now_wrapped - or_ts_get(pools[q], tb, s)) & m;
      if (a < best) best = a;
    }
    or_ts_set(out, tb, s, (now_wrapped - best) & m);
  }
}

/* route_pairs "hash" (distributed.py:195-210) */
void or_route_hash(const uint32_t* hips, const uint32_t* oips, uint64_t n, uint64_t seed_route, uint64_t n_wp,
                   int64_t* lanes) {
  for (uint64_t j = 0; j < n; ++j)
    lanes[j] = (int64_t)or_hash_range(((uint64_t)hips[j] << 32) | oips[j], seed_route, n_wp);
}
