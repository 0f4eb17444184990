#!/usr/bin/env python
"""Headline benchmark: packets/s of scan + detect (BASELINE.json `metric`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1], "config 2"): one discrete window of
268,435,456 (src,dst) uint32 pairs -- 16,777,216 sources, 512 planted super
points with 1,500-50,000 peers, Zipf(1.05) background clipped to 1,000,
geometric(0.3) duplicates -- seeded synthetic data generated on the GPU
(tools/workloads.py).  Threshold 1,024; LDCA 8 MiB (LR=8, LC=1024,
k=8192); SEAV r=12 (2 MiB) because the reference default r=4 overflows
every register array at this scale.

One step = the scan of the whole window (K1b: the LDCA in shared memory,
cut along its b axis) + finalize (K5 restore, sort, K6 filter, compaction,
report D2H) + reset.  `value` is timed with the inputs resident in HBM;
`e2e` is the same step through the public API from pinned HOST buffers
(DetectorState.process_host_stream: H2D inside the timed region,
double-buffered) with the report list read back; `e2e.dropin` is the
reference's own call pattern (65,536-pair numpy process_batch calls).

--gpus N > 1: the N ranks are launched by this script (torch.distributed.run
on 127.0.0.1) unless it already runs under torchrun.  Config 2 = weak
scaling: every rank is one border router scanning its own config-2-sized
window (seed 2 + rank); the per-rank sketches are OR-merged on rank 0
(multigpu.py: CUDA-IPC peer reads over NVLink, NCCL gather as fallback)
and rank 0 detects once.  --config 3 / 4 / 5 have multi-rank modes too
(DESIGN.md §6).  --same-device puts every rank on GPU 0 (gloo; a protocol
check).

--impl reference: the reference path on the host CPU (the oracle port,
oracle/sspd_oracle.c, on all host threads) over the full config-2 window,
plus the reference package itself on a bounded sample (reference_python),
printed on the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "packets/sec (Mpps) scan+detect"
UNIT = "Mpps"
WORKLOAD = "config2: 1 window x 268,435,456 pkts, 16.8M sources, 512 supers, LDCA 8 MiB, SEAV r=12"


def detector_params():
    from paper_1901_07306_b200 import DetectorParams

    # LDCA 8 MiB (LR=8, LC=1024, k=8192) as the config states; SEAV r=12
    return DetectorParams(theta=1024, r=12, k=8192, lr=8, lc=1024, design_n=80.5e6)


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "fallback": True}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    NVML polled from a thread every 2 ms (a timed region of ~80 ms gets ~40
    samples); falls back to `nvidia-smi -lms 100` when NVML is unavailable."""

    # NVML clocks-event (throttle) reason bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x for x in vis.split(",") if x.strip()]
        self.index = int(ids[index]) if index < len(ids) and ids[index].strip().isdigit() else index
        self.proc = None
        self.nvml = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, float, int]] = []
        self._stop = threading.Event()
        self._mark = 0

    def mark(self):
        """Start of the timed region: stop() reports the samples from here on
        (the sampler is started before the warm-up so that NVML's start-up
        does not overlap the timed steps)."""
        self._mark = len(self.samples) if self.nvml is not None else len(self.lines)

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.nvml = (pynvml, h, reasons)
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            return
        except Exception:  # noqa: BLE001 - fall back to nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _poll(self):
        nv, h, reasons = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                     float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)), int(reasons(h))))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.nvml is not None:
            self._stop.set()
            self._t.join(timeout=2)
            samples = self.samples[self._mark:] or self.samples[-1:]
            sm = [a for a, _, _ in samples]
            mx = [b for _, b, _ in samples]
            found = {name for bit, name in self.REASONS.items() for _, _, r in samples if r & bit}
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                    "reasons": sorted(found), "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines[self._mark:] or self.lines[-1:]:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


# ---------------------------------------------------------- reference arm
def reference_python(hips, oips, dp) -> dict | None:
    """The reference package itself (baseline/_ref, pure Python + numpy) on
    the host: one process over a 2^20-pair prefix, and P = host-core
    processes, each a watch point over 1/P of the sample, merged with
    serialize -> merge_frames -> finalize_window."""
    from oracle import oracle
    from tools import reference_cpu

    if not reference_cpu.available():
        return None
    geom = dict(theta=dp.theta, r=dp.r, k=dp.k, lr=dp.lr, lc=dp.lc, design_n=dp.design_n)
    n1 = min(len(hips), 1 << 20)
    single = reference_cpu.time_single(geom, hips[:n1], oips[:n1])
    procs = max(1, min(oracle.cpu_threads(), 64))
    n = len(hips) - len(hips) % procs
    per = n // procs
    multi = reference_cpu.time_multi(geom, [(hips[i * per:(i + 1) * per], oips[i * per:(i + 1) * per])
                                            for i in range(procs)], procs)
    return {"single_process": single, "processes": multi,
            "source": "baseline/_ref: the reference sspd package (pip-installed from its source), "
                      "DetectorState.process_batch in 65,536-pair buffers + finalize_window; "
                      "P processes: serialize -> merge_frames -> finalize_window",
            "sample": f"config-2 law, single: first {n1} pairs; processes: {procs} x {per} pairs"}


def _config2_host(scale: int):
    """The config-2 stream at 1/scale on the host (generated on the GPU when
    one is present -- the torch and numpy generators are bit-identical --
    because the numpy generator needs ~80 s for the full window)."""
    import numpy as np

    from tools.workloads import CONFIG2, generate, scaled

    spec = scaled(CONFIG2, scale) if scale > 1 else CONFIG2
    try:
        import torch

        if torch.cuda.is_available():
            h, o, _ = generate(spec, "torch", torch.device("cuda", 0))
            out = h.cpu().numpy().view(np.uint32).copy(), o.cpu().numpy().view(np.uint32).copy()
            del h, o
            torch.cuda.empty_cache()
            return spec, out[0], out[1]
    except Exception:  # noqa: BLE001 - no usable GPU: numpy generator
        pass
    h, o, _ = generate(spec)
    return spec, h, o


def run_reference(args) -> dict:
    """The reference path on the host: the oracle port (C restatement of the
    reference's algorithm, oracle/sspd_oracle.c) on all host threads over
    the FULL config-2 window (same workload as the GPU arm), plus the
    reference package itself timed on a bounded prefix (reference_python)."""
    import numpy as np

    from oracle import oracle
    from paper_1901_07306_b200._abi import build_params
    from paper_1901_07306_b200.hashing import SeedFamily

    dp = detector_params()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        p = build_params(dp.seav_config(), dp.ldca_config(), SeedFamily(dp.master_seed))
    spec, hips, oips = _config2_host(args.ref_scale)
    threads = oracle.cpu_threads()
    seav = np.zeros(p.seav_bytes, dtype=np.uint8)
    ldca = np.zeros(p.ldca_bytes, dtype=np.uint8)

    def step():
        seav.fill(0)
        ldca.fill(0)
        oracle.scan(p, hips, oips, seav, ldca, threads=threads)
        ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap, threads=threads)
        oracle.filter_z0(p, ldca, ips, threads=threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    mpps = len(hips) / dt / 1e6
    full = args.ref_scale <= 1
    sample = (f"the full config-2 window ({len(hips)} pairs) per step" if full else
              f"{len(hips)} pairs of the config-2 law (1/{args.ref_scale}) per step") + \
        ", scan + restore + filter, oracle port on all host threads"
    return {
        "metric": METRIC, "value": round(mpps, 3), "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32/u8 (integer)",
        "data": "synthetic (seeded, tools/workloads.py)",
        "config": {"workload": WORKLOAD, "global_batch": len(hips), "parallelism": "host threads",
                   "same_config": full},
        "cpu_baseline": {"value": round(mpps, 3), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "reference_python": reference_python(hips, oips, dp)},
        "e2e": {"value": round(mpps, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline_quick(scale: int) -> dict:
    """Bounded CPU sample for the b200 line's cpu_baseline (rank 0, N=1):
    the oracle port on all host threads, plus the reference package itself."""
    import numpy as np

    from oracle import oracle
    from paper_1901_07306_b200._abi import build_params
    from paper_1901_07306_b200.hashing import SeedFamily

    dp = detector_params()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        p = build_params(dp.seav_config(), dp.ldca_config(), SeedFamily(dp.master_seed))
    spec, hips, oips = _config2_host(scale)
    threads = oracle.cpu_threads()
    best = None
    for _ in range(2):
        seav = np.zeros(p.seav_bytes, dtype=np.uint8)
        ldca = np.zeros(p.ldca_bytes, dtype=np.uint8)
        t0 = time.perf_counter()
        oracle.scan(p, hips, oips, seav, ldca, threads=threads)
        ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap, threads=threads)
        oracle.filter_z0(p, ldca, ips, threads=threads)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return {"value": round(len(hips) / best / 1e6, 3), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(hips)} pkts of the config-2 law (1/{scale} scale), scan+restore+filter on "
                      f"{threads} threads, best of 2",
            "reference_python": reference_python(hips, oips, dp)}


def run_dropin(st, h_host, o_host, args, timed, stream_value) -> dict:
    """The reference's own call pattern end to end: the window fed from
    pageable numpy memory as 65,536-pair process_batch calls (cli.py:215-217,
    distributed.py:225-227), then finalize_window with the report list read
    back.  The host batches are staged in pinned memory and scanned in
    8 Mi-pair batches (DetectorState._stage_host)."""
    import numpy as np

    B = 65_536
    h_np = np.array(h_host.numpy().view(np.uint32))  # pageable copies, as a caller's arrays
    o_np = np.array(o_host.numpy().view(np.uint32))
    n = len(h_np)
    out = [0]

    def step():
        for lo in range(0, n, B):
            st.process_batch(h_np[lo:lo + B], o_np[lo:lo + B])
        reps = st.finalize_window()
        out[0] = len(reps.ips)
        st.reset()

    step()
    ms = timed(step, max(1, args.steps // 4))
    v = n / (ms * 1e-3) / 1e6
    # the path's own bound: the host copy of every call's keys from pageable
    # memory into the pinned staging buffers (sspd_host_pack_pairs on the
    # staging pool), measured alone over the same window
    from paper_1901_07306_b200._abi import lib

    L = lib()
    stage = st._hstage
    pa, pb, cap = stage["ph_addr"][0], stage["po_addr"][0], stage["cap"]
    fast = stage.get("fast")  # the CPython staging binding process_batch uses (csrc/hostfast.c)
    t0 = time.perf_counter()
    for lo in range(0, n, B):
        off = 4 * (lo % cap)
        if fast is not None:
            fast(h_np[lo:lo + B], o_np[lo:lo + B], pa + off, pb + off, cap - lo % cap)
        else:
            L.sspd_host_pack_pairs(h_np.ctypes.data + 4 * lo, o_np.ctypes.data + 4 * lo, min(B, n - lo), 4, 4,
                                   pa + off, pb + off)
    pack_s = time.perf_counter() - t0
    pack_pps = n / pack_s
    return {"value": round(v, 3), "unit": UNIT, "ms_per_step": round(ms, 3), "calls_per_step": -(-n // B),
            "host_copy_bound": {"value": round(pack_pps / 1e6, 3), "unit": UNIT,
                                "gbs": round(8 * n / pack_s / 1e9, 2), "threads": int(L.sspd_host_copy_threads()),
                                "frac": round(v * 1e6 / pack_pps, 4),
                                "binding": "cpython" if fast is not None else "ctypes",
                                "note": "pageable -> pinned copy of the keys alone, same 65,536-pair calls"},
            "pairs_per_call": B, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * out[0] + 16,
            "frac_of_host_stream": round(v / stream_value, 4) if stream_value else None,
            "note": "process_batch(numpy uint32 views of 65,536 pairs) x calls + finalize_window + reset; "
                    "host batches staged in pinned memory, scanned in 8 Mi-pair batches"}


def merge_summary(merger, merge_ms: list[float], dist, dev, args) -> dict:
    """Per-window OR-merge cost (multigpu.OrMerger.merge_to_root), max over
    ranks of each rank's median, with the bytes it moves over NVLink."""
    import torch

    med = statistics.median(merge_ms) if merge_ms else 0.0
    t = torch.tensor([med, max(merge_ms) if merge_ms else 0.0], dtype=torch.float64,
                     device=dev if args.backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    med, worst = float(t[0]), float(t[1])
    tr = merger.traffic()
    moved = tr["peer_read_bytes_this_rank"] + tr["root_gather_bytes"]
    return {"merge_ms_median": round(med, 4), "merge_ms_max": round(worst, 4), **tr,
            "achieved_gbs": round(moved / (med * 1e-3) / 1e9, 2) if med > 0 else None,
            "note": "host wall time of merge_to_root after the post-scan barrier: reduce-scatter of the "
                    "SEAV||LDCA block by stripes over CUDA-IPC peer reads, gather onto rank 0, three barriers; "
                    "achieved_gbs = (this rank's peer reads + root gather) / median"}


# ---------------------------------------------------------------- GPU arm
def run_gpu(args) -> dict | None:
    import torch

    from paper_1901_07306_b200 import DetectorState
    from paper_1901_07306_b200._abi import lib
    from tools.workloads import CONFIG2, generate

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:  # protocol test: all ranks share GPU 0 (host barriers only)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_ranks(args, local)
    lib()

    from dataclasses import replace

    spec = replace(CONFIG2, seed=CONFIG2.seed + rank)
    if args.packets:
        from tools.workloads import scaled

        spec = scaled(spec, max(1, CONFIG2.n_packets // args.packets))
    t_gen = time.perf_counter()
    hips, oips, supers = generate(spec, "torch", dev)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    n = int(hips.numel())
    dp = detector_params()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(dp)
    st.scan_mode = args.scan_mode
    if args.part_chunk:
        st.partitioned_chunk = args.part_chunk
    merger = None
    if world > 1:
        from paper_1901_07306_b200.multigpu import OrMerger

        merger = OrMerger(st, dist)

    stream = torch.cuda.current_stream()
    scan_ev = []
    merge_ms: list[float] = []

    def step(reports_out=None, time_scan=False):
        if time_scan:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        st.process_batch(hips, oips)
        if time_scan:
            b.record(stream)
            scan_ev.append((a, b))
        if merger is not None:
            merger.merge_to_root()
            if time_scan:
                merge_ms.append(merger.last_merge_ms)
        if rank != 0:
            st.reset()
            return []
        if args.sync_finalize:
            reps = st.finalize_window()
            st.reset()
            if reports_out is not None:
                reports_out.append(len(reps))
            return reps
        # pipelined windows: this window's finalize runs on a device snapshot
        # and is resolved after the next window's scan has been enqueued, so
        # the GPU never waits for the host between windows
        reps = st.finalize_window_async()
        st.reset()
        drain_all()  # the previous window's list (its finalize ran before this scan)
        pending.append((reps, reports_out))
        return reps

    pending: list = []

    def drain_all():
        """Resolve the pending report lists (counts read back)."""
        while pending:
            r, out = pending.pop(0)
            n_r = len(r)
            if out is not None:
                out.append(n_r)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        drain_all()  # every window's list is resolved inside the timed region
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if dist is not None:
            t = torch.tensor([ms], device=dev if args.backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # warm-up (also checks the planted supers come out)
    clocks = ClockSampler(local)
    clocks.start()
    first = None
    for _ in range(args.warmup):
        r = step()
        first = first if first is not None else r
    drain_all()
    found = {x.ip for x in first} if first else set()
    planted_found = len(set(supers.tolist()) & found) if rank == 0 else None

    clocks.mark()
    counts: list[int] = []
    ms = timed(lambda: step(counts, time_scan=True), args.steps)
    clk = clocks.stop()
    scan_ms = statistics.mean(a.elapsed_time(b) for a, b in scan_ev)
    scan_share = scan_ms / ms

    # e2e: same step through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        h_host = hips.cpu().pin_memory()
        o_host = oips.cpu().pin_memory()
        h2d = [0]
        d2h = [0]

        def step_e2e():
            h2d[0] = st.process_host_stream(h_host, o_host, chunk_pairs=args.chunk)
            if merger is not None:
                merger.merge_to_root()
            reps = st.finalize_window() if rank == 0 else []
            if rank == 0 and len(reps):
                reps.ips  # the super-point list itself comes back to the host (lazy otherwise)
            d2h[0] = 8 * len(reps) + 16 + (1 << dp.r)  # (ip, z0) pairs + counts + overflow flags
            st.reset()

        for _ in range(max(1, args.warmup // 2)):
            step_e2e()
        e2e_ms = timed(step_e2e, args.steps)
        e2e = {"value": round(world * n / (e2e_ms * 1e-3) / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": h2d[0], "d2h_bytes_per_step": d2h[0], "ms_per_step": round(e2e_ms, 3)}
        # the e2e bound is the host link: measured pinned H2D copy rate, same size as one step
        dst = torch.empty_like(hips)
        best = None
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dst.copy_(h_host, non_blocking=True)
            dst.copy_(o_host, non_blocking=True)
            b.record(stream)
            b.synchronize()
            t = a.elapsed_time(b)
            best = t if best is None else min(best, t)
        h2d_gbs = 2 * hips.numel() * 4 / (best * 1e-3) / 1e9
        e2e["h2d_roofline"] = {"bound": "pcie_h2d", "peak_gbs_measured": round(h2d_gbs, 2),
                               "achieved_gbs": round(h2d[0] / (e2e_ms * 1e-3) / 1e9, 2),
                               "frac": round(h2d[0] / (e2e_ms * 1e-3) / 1e9 / h2d_gbs, 4)}
        del dst
        if world == 1:
            e2e["dropin"] = run_dropin(st, h_host, o_host, args, timed, e2e["value"])

    merge = merge_summary(merger, merge_ms, dist, dev, args) if merger is not None else None
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None

    # roofline of the dominant kernel, the scan.  Algorithmic bytes = the 8 B
    # input per packet.  Bounds measured live in this
    # process: the hash floor (every per-packet index hash, no sketch
    # update: the work K1b is issue-bound on), and the SURVEY's L2-red term.
    import ctypes

    peaks = measured_peaks()
    p_blk = st.seav._params
    buf = torch.empty(8 << 20, dtype=torch.uint8, device=dev)
    red = ctypes.c_double(0.0)
    lib().sspd_microbench_red(buf.data_ptr(), 8 << 20, 8, 256, ctypes.byref(red), stream.cuda_stream)
    red_per_s = red.value
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.empty(2048 * sms, dtype=torch.int32, device=dev)
    hash_pps = {}
    for bps in (1, 2):
        v = ctypes.c_double(0.0)
        rc = lib().sspd_microbench_hash(hips.data_ptr(), oips.data_ptr(), n, p_blk, bps, sink.data_ptr(),
                                        ctypes.byref(v), stream.cuda_stream)
        hash_pps[bps] = v.value if rc == 0 else None
    del buf, sink
    reds_per_pkt = dp.ldca_config().lr + dp.seav_config().sr / (1 << dp.seav_config().tau)
    scan_pps = n / (scan_ms * 1e-3)
    hbm_gbs = peaks.get("hbm_gbs", 6650.0)
    achieved_gbs = 8 * n / (scan_ms * 1e-3) / 1e9
    roof_pps = min(hbm_gbs * 1e9 / 8, red_per_s / reds_per_pkt)
    kernel = getattr(st, "last_scan", "direct")
    variant = int(lib().sspd_scan_partitioned_variant(p_blk, 0)) if kernel == "partitioned" else 0
    kkey = {2: "bpart", 1: "partitioned"}.get(variant, "direct")
    kname = {"bpart": "scan_bpart_kernel<true, 1> (K1b: LDCA in shared memory, cut along b)",
             "partitioned": "scan_partitioned_kernel<true, kPow2> (K1p, LDCA in shared memory)",
             "direct": "scan_discrete_kernel<true,true> (K1, L2 red.or)"}[kkey]
    # per-kernel ncu evidence committed under profiles/ (bytes and issue slots per packet)
    prof = {}
    pf = ROOT / "profiles" / "scan_ncu_summary.json"
    if pf.exists():
        try:
            prof = json.loads(pf.read_text()).get(kkey, {})
        except ValueError:
            prof = {}
    traffic = prof.get("dram_bytes_per_packet")
    traffic = round(traffic * n) if traffic else None
    issue = None
    if prof.get("warp_inst_per_packet"):
        clk_hz = (clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)) * 1e6
        issue_pps = sms * 4 * clk_hz / prof["warp_inst_per_packet"]  # 4 schedulers x 1 warp-inst/clk
        issue = {"bound": "sm_issue", "warp_inst_per_packet": round(prof["warp_inst_per_packet"], 3),
                 "roofline_gpps": round(issue_pps / 1e9, 3), "frac": round(scan_pps / issue_pps, 4),
                 "issue_slots_busy_pct": prof.get("issue_active_pct"),
                 "source": prof.get("source")}
    ceiling = hash_pps.get(2) or hash_pps.get(1)
    binding = None
    if ceiling:
        binding = {"bound": "sm_issue: per-packet index hashes (sspd_microbench_hash, live)",
                   "ceiling_gpps": round(ceiling / 1e9, 3),
                   "ceiling_gpps_scan_launch_shape": round(hash_pps[1] / 1e9, 3) if hash_pps.get(1) else None,
                   "achieved_gpps": round(scan_pps / 1e9, 3), "frac": round(scan_pps / ceiling, 4),
                   "note": ("streaming the same pairs and computing H3 % k, the H1 test and the LR row hashes "
                            "(10 SplitMix64 per packet, the scans' 32-bit-half form, rows unrolled) with no sketch update, at full occupancy (2 x 1,024 "
                            "threads per SM); the scan adds the shared-memory partition exchange to this floor")}

    value = world * n / (ms * 1e-3) / 1e6
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 keys / u8 bit arrays (integer)",
        "data": "synthetic (seeded counter-based generator, tools/workloads.py; no CAIDA traces offline)",
        "config": {"workload": WORKLOAD if n == CONFIG2.n_packets else WORKLOAD.replace("268,435,456", f"{n:,}"),
                   "global_batch": world * n, "packets_per_gpu": n,
                   "parallelism": f"dp{world} (one border router per GPU, OR-merge to rank 0)",
                   "l2": "inputs (2 GiB/window) exceed the 126 MB L2; no flush needed",
                   "seav_r": dp.r, "ldca": "LR=8 LC=1024 k=8192 (8 MiB)"},
        "e2e": e2e,
        # per step: the scan, then the fused finalize -- state init, K5
        # restore, bucket sort (scatter + per-bucket rank), cell summary,
        # K6 filter (summary pass + AND pass), compaction (count + scatter)
        # = 10 launches of libsspd_b200.so (+ the merge kernels at N > 1);
        # matches the ncu launch list of the step (profiles/r02f_launches_config2_final.csv)
        "gpu_launches": args.steps * (10 + (2 if merger else 0)),
        "roofline": {"bound": "hbm", "achieved": round(achieved_gbs, 2), "peak": hbm_gbs, "unit": "GB/s",
                     "frac": round(achieved_gbs / hbm_gbs, 5), "traffic": traffic,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "fallback" not in peaks else "fallback",
                     "kernel": kname, "algorithmic_bytes_per_packet": 8,
                     "binding": binding,
                     "note": ("the packet stream is 8 B/pkt, so HBM is far from binding; the scan is bound by "
                              "SM instruction issue on the ten SplitMix64 index hashes per packet -- `binding` "
                              "is that floor measured live in this process; `traffic` (ncu, per launch) is the "
                              "8 B/pkt input plus the part of the 16 B/pkt shared-memory bucket exchange that "
                              "spills from L2 with 16-tile chunks (DESIGN.md §3)")},
        "scan_roofline": {"bound": "l2_red", "l2_red_ops_per_s": round(red_per_s / 1e9, 2),
                          "reds_per_packet": round(reds_per_pkt, 4), "roofline_gpps": round(roof_pps / 1e9, 3),
                          "achieved_gpps": round(scan_pps / 1e9, 3), "frac": round(scan_pps / roof_pps, 4),
                          "scan_ms": round(scan_ms, 4), "scan_share_of_step": round(scan_share, 4),
                          "l2_red_requests_per_packet_ncu": prof.get("l2_red_requests_per_packet"),
                          "note": ("SURVEY.md §8d roofline min(HBM 8 B/pkt, L2 red.or rate / reds per pkt), red "
                                   "rate measured live -- the bound of the L2-atomic scan K1; the partitioned "
                                   "scan keeps the LDCA in shared memory and issues only the SEAV reds to L2 "
                                   "(~0.03 per packet), so this term does not bind it")},
        "issue_roofline": issue,
        "merge": merge,
        "clocks": clk,
        "detect": {"reports_per_window": counts[0] if counts else None,
                   "planted_supers_found": planted_found, "planted": len(supers)},
        "gen_s": round(t_gen, 2),
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_quick(args.cpu_scale)
    if dist is not None:
        dist.destroy_process_group()
    return line


def run_sliding(args) -> dict:
    """Config 4 (BASELINE configs[3]): 2^29 packets with millisecond
    timestamps (Poisson 1.8 M pkt/s, ~298 one-second slices), w = 300
    slices, super-point list at EVERY slide.  One step = the whole trace:
    per slice K2 observe (plain u16 stores) + detect (K4 materialize,
    K5 restore, K6 filter on the pool) + advance."""
    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector
    from tools.workloads import CONFIG4, CONFIG4_TIMING, TimingSpec, generate, scaled

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        return run_sliding_ranks(args)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    spec, timing = CONFIG4, CONFIG4_TIMING
    if args.packets:
        spec = scaled(CONFIG4, max(1, CONFIG4.n_packets // args.packets))
        timing = TimingSpec(rate_pps=spec.n_packets / (CONFIG4.n_packets / CONFIG4_TIMING.rate_pps))
    t_gen = time.perf_counter()
    hips, oips, supers, ts = generate(spec, "torch", dev, timing=timing)
    slices = ts // 1000
    n_sl = int(slices[-1].item()) + 1
    bounds = torch.searchsorted(slices, torch.arange(n_sl + 1, device=dev, dtype=slices.dtype)).cpu().tolist()
    t_gen = time.perf_counter() - t_gen
    n = int(hips.numel())
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=2.15e8),
                              window_slices=300)
    if args.direct_stamps:
        det.defer_ldca_stamps = False
    if args.no_finalize_graphs:
        det.finalize_graphs = False  # the fused finalize launched op by op from the host
    if args.no_ldca_ring:
        det.ldca_ring_max_bytes = 0  # deferred single-bitmap mode (one fold + view per slide)
    if os.environ.get("SSPD_PIPELINE_DEPTH"):
        det.pipeline_depth = int(os.environ["SSPD_PIPELINE_DEPTH"])
    stream = torch.cuda.current_stream()
    counts = []

    def step(record=None):
        det.reset()
        pending = []
        total = 0
        for s in range(n_sl):
            lo, hi = bounds[s], bounds[s + 1]
            if hi > lo:
                det.observe_batch(hips[lo:hi], oips[lo:hi])
            # every slide's super-point list is computed inside the step; the
            # async form overlaps restore/filter of slide s with the scan of s+1
            pending.append(det.detect() if args.sync_detect else det.detect_async())
            det.advance_slice()
            # consume lists as a monitor would (the pipeline has already
            # resolved those older than its depth): their device report
            # buffers are released instead of 299 being held to the end
            while len(pending) > det.pipeline_depth:
                total += len(pending.pop(0))
        total += sum(len(r) for r in pending)  # all lists resolved before the step ends
        if record is not None:
            record.append(total)

    clocks = ClockSampler(0)
    clocks.start()
    for _ in range(args.warmup):
        step()
    clocks.mark()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    marks = []
    for _ in range(args.steps):
        step(counts)
        marks.append(torch.cuda.Event(enable_timing=True))
        marks[-1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    step_ms = [round(a.elapsed_time(b), 3) for a, b in zip([e0] + marks[:-1], marks)]
    # K2 alone over the same trace.  Deferred stamps (default): observe
    # every slice without advancing (the dirty bitmap absorbs it, no fold),
    # against the live-measured random L2 red.or rate -- the scan's bound;
    # direct stamps: observe + advance against the random u16 store rate at
    # the LDCA stamp footprint.
    import ctypes

    from paper_1901_07306_b200._abi import lib

    deferred = not args.direct_stamps
    det.reset()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for s in range(n_sl):
        lo, hi = bounds[s], bounds[s + 1]
        if hi > lo:
            det.observe_batch(hips[lo:hi], oips[lo:hi])
        if not deferred:
            det.advance_slice()
    s1.record(stream)
    torch.cuda.synchronize()
    scan_ms = s0.elapsed_time(s1)
    det.reset()
    lcfg = det.ldca_config
    scan_gpps = n / (scan_ms * 1e-3) / 1e9
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    seav_pp = det.seav_config.sr / (1 << det.seav_config.tau)
    if deferred:
        buf = torch.empty(8 << 20, dtype=torch.uint8, device=dev)
        rate = ctypes.c_double(0.0)
        lib().sspd_microbench_red(buf.data_ptr(), 8 << 20, 8, 256, ctypes.byref(rate), stream.cuda_stream)
        del buf
        ops_pp = lcfg.lr + 2 * seav_pp  # LDCA dirty bits + SEAV view bits (+ SEAV stamps, stores)
        scan_roof = {"bound": "l2_red", "l2_red_ops_per_s": round(rate.value / 1e9, 2), "reds_per_packet": ops_pp,
                     "note": "K2 (deferred) over the whole trace alone: 8 dirty-bitmap red.or + the SEAV view "
                             "atomics per packet into L2-resident bitmaps, vs the live-measured random red.or rate"}
    else:
        foot = 1 << max(1, (2 * lcfg.lr * lcfg.lc * lcfg.k - 1).bit_length())  # LDCA stamp bytes, pow2
        sbuf = torch.empty(foot, dtype=torch.uint8, device=dev)
        rate = ctypes.c_double(0.0)
        lib().sspd_microbench_store16(sbuf.data_ptr(), foot, 8, 256, ctypes.byref(rate), stream.cuda_stream)
        del sbuf
        ops_pp = lcfg.lr + seav_pp
        scan_roof = {"bound": "random_u16_store", "store_rate_gops": round(rate.value / 1e9, 2),
                     "footprint_bytes": foot, "stores_per_packet": round(ops_pp, 4),
                     "note": "K2 over the whole trace alone vs the live-measured random st.global.u16 rate at "
                             "the LDCA stamp footprint"}
    roof_gpps = rate.value / ops_pp / 1e9
    scan_roof.update({"roofline_gpps": round(roof_gpps, 3), "achieved_gpps": round(scan_gpps, 3),
                      "frac": round(scan_gpps / roof_gpps, 4), "scan_ms_per_trace": round(scan_ms, 3)})
    # whole-trace HBM model: the input (8 B/pkt) plus, per slide, deferred
    # in ring mode the sliding-window OR of the bitmaps (read the slice's
    # bitmap and the block OR, write the block OR and the view, clear the next
    # slot: 5 x LDCA bytes; the stamps are folded lazily, when read), deferred
    # single-bitmap one fold that reads and rewrites the LDCA stamp region
    # (2 B/slot) + reads/clears the bitmap + writes the view; direct, one 32-B
    # sector read-modify-write per scattered stamp (8 + 8.031 x 32 B)
    ldca_bytes = lcfg.lr * lcfg.lc * lcfg.k // 8
    dfr = det._deferred()
    ring = deferred and dfr is not None and dfr.ring is not None
    if ring:
        bytes_pp = 8 + 5 * ldca_bytes * n_sl / n
    elif deferred:
        fold_bytes = 2 * (2 * lcfg.lr * lcfg.lc * lcfg.k) + 3 * ldca_bytes
        bytes_pp = 8 + fold_bytes * n_sl / n
    else:
        bytes_pp = 8 + 8.031 * 32
    value = n / (ms * 1e-3) / 1e6
    return {
        "metric": "packets/sec (Mpps) sliding scan+detect at every slide", "value": round(value, 3), "unit": UNIT,
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 keys / u16 stamps",
        "data": "synthetic (seeded, tools/workloads.py CONFIG4)",
        "config": {"workload": f"config4: {n} pkts, {n_sl} slices, w=300, r=16, LDCA 8x1024x8192, detect every slide",
                   "detect": "synchronous detect()" if args.sync_detect else
                             "detect_async(): K5/K6 of slide s on a side stream, overlapping K2 of slide s+1",
                   "ldca_stamps": "direct u16 stores" if args.direct_stamps else
                                  ("deferred, ring mode: per-slice dirty bitmaps (red.or in the scan) kept for the "
                                   "window; LDCA view = two-stack sliding-window OR; stamps folded when read"
                                   if ring else "deferred: dirty-bitmap red.or in the scan, one fold per slide "
                                                "fused with the LDCA view"),
                   "pool_bytes": det.pool.memory_bytes(), "l2": "pool 403 MB exceeds L2; inputs 4 GiB"},
        "roofline": {"bound": "hbm", "achieved": round(value * 1e6 * bytes_pp / 1e9, 2), "peak": hbm, "unit": "GB/s",
                     "frac": round(value * 1e6 * bytes_pp / 1e9 / hbm, 4), "traffic": None,
                     "kernel": "whole trace (K2 + per-slide LDCA view/K4/K5/K6)",
                     "bytes_per_packet_model": round(bytes_pp, 2)},
        "scan_roofline": {**scan_roof, "scan_share_of_step": round(scan_ms / ms, 4)},
        "step_ms": step_ms,
        "clocks": clk, "detect": {"reports_total": counts[0] if counts else None, "slides": n_sl,
                                  "planted": len(supers)},
        "gen_s": round(t_gen, 2),
    }


def run_sliding_ranks(args) -> dict | None:
    """Config 4 on N ranks: N routers share the one sliding window; every
    slice's packets are split into N contiguous parts (rank r observes part
    r, slices advanced in lockstep) and every slide is detected through
    multigpu.SlidingMerger (the ranks' active-bit views OR-merged onto rank
    0 over peer memory, finalized there).  Strong scaling: the trace is
    fixed.  The value is packets / (max over ranks of the trace time)."""
    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector
    from paper_1901_07306_b200.multigpu import SlidingMerger
    from tools.workloads import CONFIG4, CONFIG4_TIMING, TimingSpec, generate, scaled

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_ranks(args, local)
    spec, timing = CONFIG4, CONFIG4_TIMING
    if args.packets:
        spec = scaled(CONFIG4, max(1, CONFIG4.n_packets // args.packets))
        timing = TimingSpec(rate_pps=spec.n_packets / (CONFIG4.n_packets / CONFIG4_TIMING.rate_pps))
    t_gen = time.perf_counter()
    hips, oips, supers, ts = generate(spec, "torch", dev, timing=timing)
    slices = ts // 1000
    del ts
    n_sl = int(slices[-1].item()) + 1
    bounds = torch.searchsorted(slices, torch.arange(n_sl + 1, device=dev, dtype=slices.dtype)).cpu().tolist()
    del slices
    parts = []
    for s_ in range(n_sl):  # this rank's contiguous part of every slice
        lo, hi = bounds[s_], bounds[s_ + 1]
        parts.append((lo + (hi - lo) * rank // world, lo + (hi - lo) * (rank + 1) // world))
    t_gen = time.perf_counter() - t_gen
    n = int(hips.numel())
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=2.15e8),
                              window_slices=300)
    merger = SlidingMerger(det, dist)
    stream = torch.cuda.current_stream()
    counts = []
    merge_ms: list[float] = []

    def step(record=None):
        det.reset()
        total = 0
        for s_ in range(n_sl):
            lo, hi = parts[s_]
            if hi > lo:
                det.observe_batch(hips[lo:hi], oips[lo:hi])
            total += len(merger.detect())
            if record is not None:
                merge_ms.append(merger.last_merge_ms)
            det.advance_slice()
        if record is not None:
            record.append(total)

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    clocks.mark()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(counts)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device=dev if args.backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    merge = merge_summary(merger, merge_ms, dist, dev, args)
    dist.destroy_process_group()
    if rank != 0:
        return None
    value = n / (ms * 1e-3) / 1e6
    return {
        "metric": "packets/sec (Mpps) sliding scan+detect at every slide", "value": round(value, 3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32 keys / u16 stamps",
        "data": "synthetic (seeded, tools/workloads.py CONFIG4)",
        "config": {"workload": f"config4: {n} pkts, {n_sl} slices, w=300, r=16, LDCA 8x1024x8192, detect every slide",
                   "parallelism": f"dp{world} (each slice split over {world} routers; per-slide OR of the "
                                  "active-bit views onto rank 0, finalize there)",
                   "detect": "SlidingMerger.detect() at every slide (synchronous)"},
        "merge": merge, "clocks": clk,
        "detect": {"reports_total": counts[0] if counts else None, "slides": n_sl, "planted": len(supers)},
        "gen_s": round(t_gen, 2),
    }


def run_sharded(args) -> dict | None:
    """Config 3 (BASELINE configs[2]): 8 router shards x 2^27 packets over one
    33.5 M-source population; each of 1,024 planted super points has its
    peers split over 2-8 routers so no router sees it above threshold.  The
    shards are folded onto the N ranks (rank r scans shards r, r+N, ...
    into ONE local sketch: OR idempotence), the per-rank sketches are
    OR-merged onto rank 0 (multigpu.OrMerger: CUDA-IPC peer reads), and
    rank 0 detects once.  Strong scaling: the 2^30 packets are fixed.
    A step = every local shard's scan (K1b) + merge + finalize + reset."""
    import torch

    from paper_1901_07306_b200 import DetectorParams, DetectorState
    from paper_1901_07306_b200._abi import lib
    from tools.workloads import CONFIG3, generate_shards, sharded_scaled

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_ranks(args, local)
    lib()
    spec = CONFIG3
    if args.packets:
        spec = sharded_scaled(spec, max(1, spec.packets_per_shard // args.packets))
    mine = list(range(rank, spec.n_shards, world))
    t_gen = time.perf_counter()
    gen = generate_shards(spec, mine, "torch", dev)
    shards = [(h, o) for h, o, _ in gen]
    supers = gen[0][2]
    del gen
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    n_local = sum(int(h.numel()) for h, _ in shards)
    n_total = spec.n_shards * spec.packets_per_shard
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=1.0e8))
    merger = None
    if world > 1:
        from paper_1901_07306_b200.multigpu import OrMerger

        merger = OrMerger(st, dist)
    stream = torch.cuda.current_stream()

    merge_ms: list[float] = []

    def step(out=None):
        for h, o in shards:
            st.process_batch(h, o)
        if merger is not None:
            merger.merge_to_root()
            if out is None:
                merge_ms.append(merger.last_merge_ms)
        reps = st.finalize_window() if rank == 0 else []
        st.reset()
        if out is not None:
            out.append(reps)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    first: list = []
    for i in range(max(1, args.warmup)):
        step(first if i == 0 else None)
    found = {r.ip for r in first[0]} if rank == 0 else set()
    barrier()
    clocks.mark()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    merge = merge_summary(merger, merge_ms, dist, dev, args) if merger is not None else None
    if dist is not None:
        dist.destroy_process_group()
    if rank != 0:
        return None
    value = n_total / (ms * 1e-3) / 1e6
    return {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32 keys / u8 bit arrays (integer)",
        "data": "synthetic (seeded, tools/workloads.py CONFIG3 shard generator)",
        "config": {"workload": f"config3: {spec.n_shards} router shards x {spec.packets_per_shard} pkts, "
                               f"{spec.n_sources} sources, {spec.n_super} split supers, LDCA 8 MiB, SEAV r=16",
                   "global_batch": n_total, "shards_per_rank": len(mine),
                   "parallelism": f"dp{world} (shards folded onto ranks, OR-merge to rank 0)",
                   "l2": "inputs (8 GiB) exceed the 126 MB L2; no flush needed"},
        # one scan per shard + the fused finalize's 9 launches (as config 2)
        "e2e": None, "gpu_launches": args.steps * (len(mine) + 9 + (2 if merger else 0)),
        "merge": merge,
        "clocks": clk,
        "detect": {"reports_per_window": len(first[0]), "planted_supers_found": len(set(supers.tolist()) & found),
                   "planted": len(supers),
                   "note": "no router sees a planted super above threshold; they are found only after the merge"},
        "gen_s": round(t_gen, 2),
    }


def run_streaming(args) -> dict | None:
    """Config 5 (BASELINE configs[4]): 2^32 packets streamed from pinned host
    memory in 2^26-packet batches (double-buffered H2D, process_host_stream);
    8 discrete windows x 8 router batches, LDCA 64 MiB (LR=8, LC=8192),
    SEAV r=16, finalize once per window.  At N ranks, rank r is the border
    router(s) r, r+N, ... of every window: it streams only its own batches
    over its own PCIe link, the per-rank sketches are OR-merged onto rank 0
    (multigpu.OrMerger) and rank 0 finalizes each window.  At N = 1 one GPU
    plays all 8 routers (the OR-merge is the sketch itself).  The router
    batches are generated once and re-streamed by every window."""
    import torch

    from paper_1901_07306_b200 import DetectorParams, DetectorState
    from tools.workloads import CONFIG5_WINDOW, generate_shard, sharded_scaled

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_ranks(args, local)
    spec = CONFIG5_WINDOW
    if args.packets:
        spec = sharded_scaled(spec, max(1, spec.packets_per_shard // args.packets))
    mine = list(range(rank, spec.n_shards, world))
    t_gen = time.perf_counter()
    batches = []
    for r in mine:
        h, o, _ = generate_shard(spec, r, "torch", dev)
        batches.append((h.cpu().pin_memory(), o.cpu().pin_memory()))
        del h, o
    torch.cuda.empty_cache()
    t_gen = time.perf_counter() - t_gen
    windows = 8
    per_batch = int(batches[0][0].numel())
    n = windows * spec.n_shards * per_batch
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=8192, design_n=1.6e8))
    merger = None
    if dist is not None:
        from paper_1901_07306_b200.multigpu import OrMerger

        merger = OrMerger(st, dist)
    stream = torch.cuda.current_stream()
    reps = []
    merge_ms: list[float] = []

    def step(record=None):
        total = 0
        for _ in range(windows):
            for h, o in batches:
                st.process_host_stream(h, o, chunk_pairs=args.chunk)
            if merger is not None:
                merger.merge_to_root()
                if record is not None:
                    merge_ms.append(merger.last_merge_ms)
            if rank == 0:
                total += len(st.finalize_window())
            st.reset()
        if record is not None:
            record.append(total)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    clocks.mark()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(reps)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # bound: the host links -- measured pinned H2D rate on one batch (per GPU)
    dst = torch.empty(per_batch, dtype=torch.int32, device=dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(3):
        a.record(stream)
        dst.copy_(batches[0][0], non_blocking=True)
        b.record(stream)
        b.synchronize()
        best = a.elapsed_time(b) if best is None else min(best, a.elapsed_time(b))
    h2d = per_batch * 4 / (best * 1e-3) / 1e9
    merge = merge_summary(merger, merge_ms, dist, dev, args) if merger is not None else None
    if dist is not None:
        dist.destroy_process_group()
    if rank != 0:
        return None
    achieved = 8 * n / (ms * 1e-3) / 1e9
    value = n / (ms * 1e-3) / 1e6
    return {
        "metric": "packets/sec (Mpps) streamed scan+detect (pinned host batches)", "value": round(value, 3),
        "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32 keys / u8 bit arrays",
        "data": "synthetic (seeded, tools/workloads.py CONFIG5_WINDOW)",
        "config": {"workload": f"config5: {windows} windows x {spec.n_shards} batches x {per_batch} pkts = {n}",
                   "ldca": "LR=8 LC=8192 k=8192 (64 MiB, L2 red.or scan)", "seav_r": 16,
                   "routers_per_rank": len(mine),
                   "parallelism": f"dp{world} (router batches over each GPU's own PCIe link, OR-merge to rank 0)",
                   "ingest": f"process_host_stream, {args.chunk}-pair double-buffered H2D chunks"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": None},
        "roofline": {"bound": "pcie_h2d", "achieved": round(achieved, 2), "peak": round(h2d * world, 2),
                     "unit": "GB/s", "frac": round(achieved / (h2d * world), 4), "traffic": None,
                     "peak_source": f"measured pinned H2D copy x {world} GPU link(s)"},
        "merge": merge,
        "clocks": clk, "detect": {"reports_total": reps[0] if reps else None, "windows": windows},
        "gen_s": round(t_gen, 2),
    }


# ------------------------------------------------------------ rank launcher
def _free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launch_cmd(argv: list[str], nproc: int, port: int) -> list[str]:
    """torchrun command that re-runs this script as `nproc` ranks (one process
    per GPU) on this node, rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *argv]


def self_launch(args, argv: list[str]) -> int | None:
    """`--gpus N` (N > 1) without a torchrun environment: spawn the N ranks
    ourselves so the run really times N GPUs (rank 0 prints the line)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if not args.launcher_selftest and not args.same_device:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} GPU(s) visible "
                             "(use --same-device to run the ranks on GPU 0 as a protocol test)")
    print(f"[bench] launching {args.gpus} ranks via torch.distributed.run", file=sys.stderr, flush=True)
    return subprocess.call(launch_cmd(argv, args.gpus, _free_port()))


def init_ranks(args, local: int):
    """Process group of the torchrun ranks (None at N = 1); logs the
    communicator so the driver can check ranks and backend."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist

    if args.same_device:  # NCCL refuses two ranks on one GPU: protocol runs use gloo
        args.backend = "gloo"
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    dev = f"cuda:{local}" if args.backend == "nccl" or torch.cuda.is_available() else "cpu"
    print(f"[bench] rank {dist.get_rank()}/{dist.get_world_size()} backend={dist.get_backend()} device={dev} "
          f"nccl={'.'.join(map(str, torch.cuda.nccl.version())) if args.backend == 'nccl' else '-'}",
          file=sys.stderr, flush=True)
    return dist


def run_launcher_selftest(args) -> dict | None:
    """CPU check of the launcher: every rank joins a gloo group and
    all-reduces its rank; rank 0 reports the world it saw."""
    import torch

    args.backend = "gloo"
    dist = init_ranks(args, 0)
    world = dist.get_world_size() if dist else 1
    rank = dist.get_rank() if dist else 0
    t = torch.tensor([rank + 1], dtype=torch.int64)
    if dist:
        dist.all_reduce(t)
        dist.destroy_process_group()
    if rank != 0:
        return None
    return {"selftest": "launcher", "n_gpus": world, "rank_sum": int(t.item()),
            "world_env": int(os.environ.get("WORLD_SIZE", "1"))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--packets", type=int, default=0, help="override packets per window (debug)")
    ap.add_argument("--chunk", type=int, default=1 << 23, help="e2e staging chunk (pairs)")
    ap.add_argument("--cpu-scale", type=int, default=32, help="CPU sample = config 2 / scale")
    ap.add_argument("--ref-scale", type=int, default=1,
                    help="--impl reference: config 2 / scale per step (1 = the full window)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--scan-mode", default="auto", choices=["auto", "direct", "partitioned"])
    ap.add_argument("--part-chunk", type=int, default=0, help="partitioned-scan chunk (packets); 0 = default")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"], help="process-group backend (N > 1)")
    ap.add_argument("--same-device", action="store_true", help="all ranks on GPU 0 (multi-rank protocol test)")
    ap.add_argument("--sync-detect", action="store_true", help="config 4: synchronous detect() per slide")
    ap.add_argument("--no-finalize-graphs", action="store_true",
                    help="config 4: launch the per-slide finalize op by op instead of replaying its CUDA graph")
    ap.add_argument("--no-ldca-ring", action="store_true",
                    help="config 4: deferred LDCA stamps without the ring of per-slice bitmaps (fold per slide)")
    ap.add_argument("--direct-stamps", action="store_true",
                    help="config 4: store LDCA stamps directly instead of the deferred dirty bitmap + fold")
    ap.add_argument("--sync-finalize", action="store_true",
                    help="config 2: synchronous finalize_window() per window (default: pipelined windows)")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="2 = headline discrete window; 3 = 8 router shards OR-merged (strong scaling); "
                         "4 = sliding window, detect every slide; 5 = 2^32 pkts streamed from host")
    ap.add_argument("--launcher-selftest", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.impl != "reference":
        rc = self_launch(args, sys.argv[1:])
        if rc is not None:
            sys.exit(rc)
    if args.launcher_selftest:
        line = run_launcher_selftest(args)
        if line is not None:
            print(json.dumps(line))
        return
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        print(json.dumps(run_reference(args)))
        return
    line = {3: run_sharded, 4: run_sliding, 5: run_streaming}.get(args.config, run_gpu)(args)
    if line is not None:
        print(json.dumps(line))


if __name__ == "__main__":
    main()
