"""Seeded synthetic packet streams for the BASELINE.json configs.

The paper's CAIDA traces are not available (no network), so
seeded synthetic streams with the configs' shapes stand in for them.  The
generator is counter-based: every random draw is mix64 of a (tag, seed,
index) counter, all arithmetic is int64 bit patterns with explicit logical
shifts, so the numpy backend (small streams, CPU oracle checks) and the
torch/CUDA backend (full-size bench streams, generated in HBM) produce
BIT-IDENTICAL streams for the same spec.

Config resolutions (BASELINE.md §5 asks the builder to record them):
* background cardinalities are rank-size Zipf, c_i = clip(floor(C i^-s),
  1, c_max), C solved by bisection so distinct pairs x mean duplicates
  fills the packet budget (SURVEY.md §8d recommendation);
* duplicates are geometric(p) on {1, 2, ...} (mean 1/p), drawn by integer
  inverse-CDF lookup; the stream is cut/padded to EXACTLY n packets while
  every distinct pair is kept at least once;
* source IPs are distinct (a keyed 32-bit bijection of the source index);
  destination IPs are distinct per source (the same bijection of a
  per-source random offset plus a counter).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
T_SRC, T_OFF, T_CARD, T_DUP, T_PICK, T_ORDER, T_PAD, T_DST, T_SPLIT, T_TIME = range(1, 11)


def mix64_int(x: int) -> int:
    z = (x + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _signed(v: int) -> int:
    v &= M64
    return v - (1 << 64) if v >= (1 << 63) else v


@dataclass(frozen=True)
class StreamSpec:
    name: str
    n_packets: int
    n_sources: int
    n_super: int
    super_card: tuple[int, int]          # inclusive range
    zipf_s: float
    zipf_max: int
    dup_p: float
    seed: int = 0
    super_log_uniform: bool = False


CONFIG1 = StreamSpec("config1", 1 << 20, 65_536, 32, (2048, 2048), 1.1, 200, 0.4, seed=0)
CONFIG2 = StreamSpec("config2", 1 << 28, 16_777_216, 512, (1500, 50_000), 1.05, 1000, 0.3, seed=2)


def scaled(spec: StreamSpec, factor: int) -> StreamSpec:
    """The same law at 1/factor size (packets and sources), for CPU checks."""
    return replace(spec, name=f"{spec.name}/{factor}", n_packets=spec.n_packets // factor,
                   n_sources=max(spec.n_super + 1, spec.n_sources // factor),
                   n_super=max(1, spec.n_super // factor))


# ---------------------------------------------------------------- backends
class _Backend:
    def shr(self, x, s):
        return (x >> s) & ((1 << (64 - s)) - 1)

    def mix64(self, x):
        z = x + _signed(GOLDEN)
        z = (z ^ self.shr(z, 30)) * _signed(0xBF58476D1CE4E5B9)
        z = (z ^ self.shr(z, 27)) * _signed(0x94D049BB133111EB)
        return z ^ self.shr(z, 31)

    def draw(self, tag: int, seed: int, idx):
        key = _signed(mix64_int(((seed & 0xFFFFFFFF) << 8) | tag))
        return self.mix64(idx ^ key)

    def perm32(self, x, key: int):
        m = 0xFFFFFFFF
        x = (x ^ (key & m)) & m
        for mul in (0x7FEB352D, 0x846CA68B, 0x9E3779B1):
            x = (x ^ (x >> 16)) & m
            x = (x * mul) & m
        return (x ^ (x >> 16)) & m


class _NP(_Backend):
    def __init__(self):
        import warnings

        warnings.filterwarnings("ignore", "overflow encountered", RuntimeWarning)

    def arange(self, n):
        return np.arange(n, dtype=np.int64)

    def host(self, a):
        return np.asarray(a, dtype=np.int64)

    def repeat(self, v, c):
        return np.repeat(v, c)

    def cumsum(self, x):
        return np.cumsum(x)

    def argsort(self, k):
        return np.argsort(k, kind="stable")

    def searchsorted_left(self, t, x):
        return np.searchsorted(t, x, side="left")

    def cat(self, xs):
        return np.concatenate(xs)

    def total(self, x):
        return int(x.sum())


class _Torch(_Backend):
    def __init__(self, device):
        import torch

        self.t = torch
        self.dev = device

    def arange(self, n):
        return self.t.arange(n, dtype=self.t.int64, device=self.dev)

    def host(self, a):
        return self.t.as_tensor(np.asarray(a, dtype=np.int64), device=self.dev)

    def repeat(self, v, c):
        return self.t.repeat_interleave(v, c)

    def cumsum(self, x):
        return self.t.cumsum(x, 0)

    def argsort(self, k):
        return self.t.sort(k, stable=True).indices

    def searchsorted_left(self, t, x):
        return self.t.searchsorted(t, x, right=False)

    def cat(self, xs):
        return self.t.cat(xs)

    def total(self, x):
        return int(x.sum().item())


# ------------------------------------------------------------ host tables
def zipf_rank_size(n: int, s: float, cmax: int, target_total: int) -> np.ndarray:
    ranks = np.arange(1, n + 1, dtype=np.float64) ** (-s)

    def total(c):
        return int(np.clip(np.floor(c * ranks), 1, cmax).sum())

    lo, hi = 0.0, 1.0
    while total(hi) < target_total and hi < 1e18:
        hi *= 2
    for _ in range(200):
        mid = (lo + hi) / 2
        if total(mid) < target_total:
            lo = mid
        else:
            hi = mid
    return np.clip(np.floor(hi * ranks), 1, cmax).astype(np.int64)


def geometric_table(p: float, kmax: int = 96) -> np.ndarray:
    """-floor((1-p)^k 2^53) for k = 1..kmax, ascending.  With u uniform on
    [0, 2^53): count = 1 + #{k : u < t_k} = 1 + searchsorted_left(table, -u)."""
    return np.array([-int(math.floor((1.0 - p) ** k * (1 << 53))) for k in range(1, kmax + 1)],
                    dtype=np.int64)


def cardinalities(spec: StreamSpec) -> np.ndarray:
    """Per-source distinct-peer counts: supers first, then background."""
    lo, hi = spec.super_card
    key = mix64_int(((spec.seed & 0xFFFFFFFF) << 8) | T_CARD)
    draws = np.array([mix64_int(i ^ key) for i in range(spec.n_super)], dtype=np.uint64)
    if spec.super_log_uniform:
        u = (draws >> np.uint64(11)).astype(np.float64) / float(1 << 53)
        sup = np.floor(np.exp(math.log(lo) + u * (math.log(hi + 1) - math.log(lo)))).astype(np.int64)
        sup = np.clip(sup, lo, hi)
    else:
        sup = lo + (draws % np.uint64(hi - lo + 1)).astype(np.int64)
    budget = int(spec.n_packets * spec.dup_p) - int(sup.sum())
    n_bg = spec.n_sources - spec.n_super
    if budget < n_bg:
        raise ValueError(f"{spec.name}: packet budget too small for {n_bg} background sources")
    return np.concatenate([sup, zipf_rank_size(n_bg, spec.zipf_s, spec.zipf_max, budget)])


# -------------------------------------------------------------- generator
def generate(spec: StreamSpec, backend: str = "numpy", device=None, timing=None):
    """(hips, oips, supers): exactly spec.n_packets pairs.

    numpy backend -> uint32 arrays; torch backend -> int32 device tensors
    holding the uint32 bit patterns.  `supers` = sorted planted IPs (numpy).
    With `timing` (config 4) a fourth array of non-decreasing millisecond
    timestamps is returned and the stream is in arrival order.
    """
    xp = _NP() if backend == "numpy" else _Torch(device)
    seed = spec.seed
    cards_h = cardinalities(spec)
    n_src = spec.n_sources
    n_edges = int(cards_h.sum())
    if n_edges > spec.n_packets:
        raise ValueError(f"{spec.name}: {n_edges} distinct pairs exceed {spec.n_packets} packets")
    src_ip = xp.perm32(xp.arange(n_src), mix64_int(seed ^ (T_SRC << 40)))
    cards = xp.host(cards_h)
    host_of = xp.repeat(xp.arange(n_src), cards)
    starts = xp.cumsum(cards) - cards
    eidx = xp.arange(n_edges)
    rank = eidx - starts[host_of]
    off = xp.draw(T_OFF, seed, host_of) & 0xFFFFFFFF
    dst = xp.perm32((off + rank) & 0xFFFFFFFF, mix64_int(seed ^ (T_DST << 40)))
    table = xp.host(geometric_table(spec.dup_p))
    u53 = xp.shr(xp.draw(T_DUP, seed, eidx), 11)
    counts = 1 + xp.searchsorted_left(table, -u53)
    extra_pool = xp.repeat(eidx, counts - 1)
    need = spec.n_packets - n_edges
    pool_n = int(extra_pool.shape[0])
    if pool_n >= need:
        pri = xp.shr(xp.draw(T_PICK, seed, xp.arange(pool_n)), 1)
        extra = extra_pool[xp.argsort(pri)[:need]]
    else:
        pad = xp.shr(xp.draw(T_PAD, seed, xp.arange(need - pool_n)), 1) % n_edges
        extra = xp.cat([extra_pool, pad])
    edges = xp.cat([eidx, extra])
    ts_ms = None
    if timing is None:
        order = xp.argsort(xp.shr(xp.draw(T_ORDER, seed, xp.arange(spec.n_packets)), 1))
    else:
        # config 4: every packet gets an integer-microsecond arrival time --
        # background uniform over the trace, planted supers uniform inside
        # their own active interval -- and the stream is sorted by time
        # (sorted uniform arrivals = a Poisson stream of the given rate).
        span_us = int(round(spec.n_packets / timing.rate_pps * 1e6))
        u = xp.shr(xp.draw(T_TIME, seed, xp.arange(spec.n_packets)), 11)
        host = host_of[edges]
        is_sup = host < spec.n_super
        lo_h, len_h = super_intervals(spec, timing, span_us)
        lo_t, len_t = xp.host(lo_h), xp.host(len_h)
        hs = host * is_sup  # index 0 for background (masked below)
        t_sup = lo_t[hs] + u % len_t[hs]
        t_bg = u % span_us
        t_us = t_sup * is_sup + t_bg * (1 - is_sup * 1)
        order = xp.argsort(t_us * (1 << 24) + (xp.arange(spec.n_packets) & ((1 << 24) - 1)))
        ts_ms = (t_us[order] // 1000)
    stream = edges[order]
    hips = src_ip[host_of[stream]]
    oips = dst[stream]
    supers = src_ip[: spec.n_super]
    if backend == "numpy":
        out = (hips.astype(np.uint32), oips.astype(np.uint32), np.sort(supers.astype(np.uint32)))
        return out if ts_ms is None else out + (ts_ms.astype(np.uint32),)
    t = xp.t
    to32 = lambda x: t.where(x >= 2**31, x - 2**32, x).to(t.int32)  # noqa: E731
    out = (to32(hips), to32(oips), np.sort(supers.cpu().numpy().astype(np.uint32)))
    return out if ts_ms is None else out + (ts_ms.to(t.int32),)


@dataclass(frozen=True)
class TimingSpec:
    """Config 4: Poisson arrivals, planted supers active on sub-ranges."""

    rate_pps: float = 1.8e6
    active_s: tuple[int, int] = (60, 600)


CONFIG4 = StreamSpec("config4", 1 << 29, 1_740_000, 256, (2048, 2048), 1.1, 200, 0.4, seed=4)
CONFIG4_TIMING = TimingSpec()


def super_intervals(spec: StreamSpec, timing: TimingSpec, span_us: int):
    """[lo, lo+len) activity interval (microseconds) of every planted super,
    lengths U[active_s] clipped to the trace span (BASELINE configs[3])."""
    key = mix64_int(((spec.seed & 0xFFFFFFFF) << 8) | T_SPLIT)
    lo = np.zeros(max(1, spec.n_super), dtype=np.int64)
    ln = np.ones(max(1, spec.n_super), dtype=np.int64)
    a, b = timing.active_s
    for s in range(spec.n_super):
        d1, d2 = mix64_int(2 * s ^ key), mix64_int((2 * s + 1) ^ key)
        length = min(span_us, (a + d1 % (b - a + 1)) * 1_000_000)
        start = d2 % max(1, span_us - length + 1)
        lo[s], ln[s] = start, max(1, length)
    return lo, ln


# ----------------------------------------------------- config 3 (sharded)
@dataclass(frozen=True)
class ShardedSpec:
    """Config 3: n_shards routers over one global source population; every
    planted super's peers are split evenly over 2..8 distinct routers so no
    router sees more than 1,023 of them (BASELINE configs[2])."""

    name: str = "config3"
    n_shards: int = 8
    packets_per_shard: int = 1 << 27
    n_sources: int = 33_554_432
    n_super: int = 1024
    routers: tuple[int, int] = (2, 8)
    zipf_s: float = 1.05
    zipf_max: int = 1000
    dup_p: float = 0.3
    seed: int = 3
    super_log_range: tuple[int, int] | None = None


CONFIG3 = ShardedSpec()
# Config 5, one 300 s window: 8 routers x one 2^26-packet batch each; the
# 4,096 supers are spread over the 8 windows (512 per window, log-uniform
# cardinality 1,024 .. 2^20); 67,108,864 sources / 8 windows per window.
CONFIG5_WINDOW = ShardedSpec(name="config5-window", n_shards=8, packets_per_shard=1 << 26, n_sources=8_388_608,
                             n_super=512, routers=(1, 8), zipf_s=1.05, zipf_max=1000, dup_p=0.3, seed=5,
                             super_log_range=(1024, 1 << 20))
T_SHARD = 11


def sharded_scaled(spec: ShardedSpec, factor: int) -> ShardedSpec:
    return replace(spec, name=f"{spec.name}/{factor}", packets_per_shard=spec.packets_per_shard // factor,
                   n_sources=max(spec.n_super + 1, spec.n_sources // factor),
                   n_super=max(1, spec.n_super // factor))


def super_routing(spec: ShardedSpec):
    """(cardinality, router list) of every planted super (host-side tables)."""
    key = mix64_int(((spec.seed & 0xFFFFFFFF) << 8) | T_SHARD)
    a, b = spec.routers
    cards, routers = [], []
    for s in range(spec.n_super):
        d = [mix64_int((8 * s + t) ^ key) for t in range(3)]
        m = min(spec.n_shards, a + d[0] % (b - a + 1))
        if spec.super_log_range:  # config 5: log-uniform cardinality, any split
            lo, hi = spec.super_log_range
            u = (d[1] >> 11) / float(1 << 53)
            c = int(min(hi, max(lo, math.floor(math.exp(math.log(lo) + u * (math.log(hi + 1) - math.log(lo)))))))
        else:
            c = 1024 + d[1] % (1023 * m - 1024 + 1)  # c ~ U[1024, 1023 m]: >= theta globally, <= 1023 per router
        perm = sorted(range(spec.n_shards), key=lambda r: mix64_int((d[2] << 4) ^ r))
        cards.append(c)
        routers.append(perm[:m])
    return np.array(cards, dtype=np.int64), routers


def generate_shard(spec: ShardedSpec, shard: int, backend: str = "numpy", device=None):
    """(hips, oips, supers) of one router's shard: exactly packets_per_shard pairs.

    Background pairs of the global population go to router hash(pair) % n;
    super s's j-th peer goes to routers_s[j % m_s]."""
    return generate_shards(spec, [shard], backend, device)[0]


def generate_shards(spec: ShardedSpec, shards, backend: str = "numpy", device=None):
    """[(hips, oips, supers)] for several routers of one population: the
    global edge set and its routing are built once (bit-identical to
    calling generate_shard per router)."""
    xp = _NP() if backend == "numpy" else _Torch(device)
    seed = spec.seed
    sup_cards, routers = super_routing(spec)
    total = spec.n_shards * spec.packets_per_shard
    budget = int(total * spec.dup_p) - int(sup_cards.sum())
    n_bg = spec.n_sources - spec.n_super
    cards_h = np.concatenate([sup_cards, zipf_rank_size(n_bg, spec.zipf_s, spec.zipf_max, budget)])
    n_src = spec.n_sources
    src_ip = xp.perm32(xp.arange(n_src), mix64_int(seed ^ (T_SRC << 40)))
    cards = xp.host(cards_h)
    host_of = xp.repeat(xp.arange(n_src), cards)
    starts = xp.cumsum(cards) - cards
    n_edges = int(cards_h.sum())
    eidx = xp.arange(n_edges)
    rank = eidx - starts[host_of]
    off = xp.draw(T_OFF, seed, host_of) & 0xFFFFFFFF
    dst = xp.perm32((off + rank) & 0xFFFFFFFF, mix64_int(seed ^ (T_DST << 40)))
    # router of every edge
    m_h = np.array([len(r) for r in routers] + [1], dtype=np.int64)
    tab_h = np.full((spec.n_super + 1, spec.n_shards), -1, dtype=np.int64)
    for s, rs in enumerate(routers):
        tab_h[s, : len(rs)] = rs
    is_sup = host_of < spec.n_super
    hs = host_of * is_sup + spec.n_super * (1 - is_sup * 1)  # row n_super = background
    m = xp.host(m_h)[hs]
    tab = xp.host(tab_h.reshape(-1))
    sup_router = tab[hs * spec.n_shards + rank % m]
    bg_router = xp.shr(xp.draw(T_SHARD, seed, eidx), 1) % spec.n_shards
    router = sup_router * is_sup + bg_router * (1 - is_sup * 1)
    del rank, off, m, sup_router, bg_router, hs, is_sup
    supers = src_ip[: spec.n_super]
    table = xp.host(geometric_table(spec.dup_p))
    out = []
    for shard in shards:
        mine = eidx[router == shard]
        n_mine = int(mine.shape[0])
        if n_mine > spec.packets_per_shard:
            raise ValueError(f"{spec.name}: shard {shard} has {n_mine} pairs > {spec.packets_per_shard} packets")
        sseed = seed * 131 + shard + 1
        counts = 1 + xp.searchsorted_left(table, -xp.shr(xp.draw(T_DUP, sseed, mine), 11))
        extra_pool = xp.repeat(mine, counts - 1)
        need = spec.packets_per_shard - n_mine
        pool_n = int(extra_pool.shape[0])
        if pool_n >= need:
            extra = extra_pool[xp.argsort(xp.shr(xp.draw(T_PICK, sseed, xp.arange(pool_n)), 1))[:need]]
        else:
            pad = mine[xp.shr(xp.draw(T_PAD, sseed, xp.arange(need - pool_n)), 1) % n_mine]
            extra = xp.cat([extra_pool, pad])
        edges = xp.cat([mine, extra])
        del mine, counts, extra_pool, extra
        order = xp.argsort(xp.shr(xp.draw(T_ORDER, sseed, xp.arange(spec.packets_per_shard)), 1))
        stream = edges[order]
        del edges, order
        hips = src_ip[host_of[stream]]
        oips = dst[stream]
        del stream
        if backend == "numpy":
            out.append((hips.astype(np.uint32), oips.astype(np.uint32), np.sort(supers.astype(np.uint32))))
        else:
            t = xp.t
            to32 = lambda x: t.where(x >= 2**31, x - 2**32, x).to(t.int32)  # noqa: E731
            out.append((to32(hips), to32(oips), np.sort(supers.cpu().numpy().astype(np.uint32))))
    return out
