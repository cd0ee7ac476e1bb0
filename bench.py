"""Benchmark of the sketch pass (BASELINE.json metric: sketch-pass GB/s of A,
% of roofline, end-to-end PCA seconds).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--scaling auto|weak|strong] [--precision auto|simt|tc]

A step = one full sketch pass (Algorithm 4 steps 4-8) over the config's A,
resident in HBM: every row pushed through libspca, H flushed, G widened, the
state finished on the device; with N > 1 ranks each rank owns a contiguous
row shard and the step ends with the NCCL all-reduce of [H | col_sums | rows].
Scaling: config 2 (a one-GPU config) is weak — every rank a full 100 000-row
matrix; configs 3 and 5 (fixed matrices, BASELINE.json) are strong — the
config's m rows split over the ranks.  ``--gpus N`` without WORLD_SIZE in the
environment re-launches itself under torch.distributed.run with N ranks.

The JSON line (rank 0) carries: value (whole-job GB/s of A), e2e (same
metric through the public API with A in pinned host memory, H2D and the D2H
of the sketch inside the timed region; e2e_pageable the same from a plain
numpy array), roofline (the pass kernel, CUDA events on its stream),
pca_seconds (A in HBM) and pca_seconds_host (numpy input), parity (our U, S, V
against the unmodified reference's single_pass_pca on the same A and Omega,
N = 1), cpu_baseline (the reference timed on this host's cores on the full A),
clocks sampled during the timed region, gpu_launches.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sketch-pass GB/s of A"
UNIT = "GB/s"
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="cfg2")
    p.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                   help="auto: weak for cfg1/cfg2 (one-GPU configs), strong for cfg3/cfg5")
    p.add_argument("--precision", default="auto")
    p.add_argument("--rows", type=int, default=None, help="override m (debug)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-pca", action="store_true")
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--ref-budget-s", type=float, default=240.0,
                   help="--impl reference: bound on the whole timed run (rows sampled above it)")
    p.add_argument("--ring-gb", type=float, default=16.0, help="cfg4: pinned host ring size")
    p.add_argument("--dtype", default="f32", choices=["f32", "f64"],
                   help="element type of A (f64: the config's values widened, DFMA path)")
    return p.parse_args()


def workload_config(workload: str, cs: dict, m_total: int, m_rank: int, world: int, mode: str) -> dict:
    """The `config` object of a bench line: the workload alone, so both arms
    (ours and --impl reference) print the same object for the same run."""
    return {"workload": workload, "m": int(m_total), "m_per_gpu": int(m_rank), "n": cs["n"], "l": cs["l"],
            "k": cs["k"], "rank": cs["rank"], "spectrum": cs["spectrum"], "noise": cs["noise"],
            "parallelism": f"row-shard x{world} ({mode})",
            "l2": "inputs larger than L2" if m_rank * cs["n"] * 4 >= (512 << 20)
                  else "L2 flushed before every timed step"}


def scaling_mode(args) -> str:
    if args.scaling != "auto":
        return args.scaling
    return "strong" if args.config in ("cfg3", "cfg5") else "weak"


def host_cores():
    """(threads usable by this process, physical cores)."""
    try:
        logical = len(os.sched_getaffinity(0))
    except Exception:
        logical = os.cpu_count() or 1
    try:
        import psutil
        phys = psutil.cpu_count(logical=False) or logical
    except Exception:
        phys = logical
    return logical, phys


def ref_module():
    """The unmodified reference package, installed into baseline/_ref by
    tools/install_reference.sh (pip --target; travels with the repo
    snapshot), or None when it is absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "streampca")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import streampca
    return streampca


def max_angle(x, y) -> float:
    """Largest principal angle between the column spaces of x and y."""
    from scipy.linalg import subspace_angles
    return float(np.max(subspace_angles(np.asarray(x, dtype=np.float64), np.asarray(y, dtype=np.float64))))


def peaks():
    """(hbm GB/s, bf16 dense TF/s burst, kind) from MEASURED_PEAKS.json."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, streamed every 50 ms while the
    timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self._t = None

    def _reader(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._reader, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self._t:
            self._t.join(timeout=5)

    def summary(self):
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(s[0]) for s in self.samples) if v]
        mx = [v for v in (num(s[1]) for s in self.samples) if v]
        pw = [v for v in (num(s[2]) for s in self.samples) if v]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        busy = [v for v in sm if v > 0]
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_max": max(pw) if pw else None}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_oracle_rate(n_rows: int, n: int, l: int, seed: int, threads: int):
    """Time the numpy oracle (blocked sketch_pass, fp32 rows widened to fp64
    as FileRowStream does) on a sample of rows; returns (GB/s of fp32 A, s)."""
    from threadpoolctl import threadpool_limits
    import oracle as O
    rng = np.random.Generator(np.random.Philox(key=np.array([seed, 99], dtype=np.uint64)))
    a = (rng.standard_normal((n_rows, n), dtype=np.float32) * np.float32(1e-2))
    om = O.gaussian(n, l, 1)
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        blocks = ((r0, a[r0:r0 + 4096].astype(np.float64)) for r0 in range(0, n_rows, 4096))
        O.oracle_sketch(blocks, om)
        dt = time.perf_counter() - t0
    return a.nbytes / dt / 1e9, dt


def host_config_matrix(config: str, rows: int):
    """The config's A (first ``rows`` rows) generated on the host for the
    reference arm, which runs without the GPU: configs 2-5 by the same
    block-seeded construction as synth.config_matrix (torch CPU generator,
    so the values differ from the GPU-generated matrix, the distribution does
    not); config 1 by the reference's own synth_matrix (seed 100)."""
    import math
    import torch
    from paper_1704_07669_b200 import synth
    torch.set_num_threads(host_cores()[0])
    if config == "cfg1":
        ref = ref_module()
        m, n = synth.CONFIGS["cfg1"][:2]
        spec_vals = tuple(10.0 ** (-4.0 * np.arange(n) / (n - 1)))
        if ref is not None:
            return ref.synth_matrix(m, n, ref.SpectrumSpec("custom", values=spec_vals), seed=100).materialize()
        import oracle as O
        return O.reference_synth_matrix(m, n, spec_vals, 100)
    m, n, r, kind, noise, _, _ = synth.CONFIGS[config]
    dev = torch.device("cpu")
    w = synth.right_factor(n, r, kind, 2024, dev)
    out = torch.empty((rows, n), dtype=torch.float32)
    synth.fill_rows(out, 0, m, n, r, noise, 2024, w)
    return out.numpy()


def run_reference(args):
    """Reference arm: the unmodified reference package (baseline/_ref, its
    public API: ``sketch_pass(ArrayRowStream(A), Omega, block_rows)``,
    sketch.py:52-116, streams.py:55-80) on this host's cores, every step one
    pass over the config's A (fp32, widened to fp64 inside the timed step by
    ArrayRowStream as for any numpy input), W warm-up + K timed steps. A config
    whose K + W passes would exceed --ref-budget-s passes a stated row prefix
    instead. Falls back to the numpy oracle port when baseline/_ref is absent.
    Under torchrun only rank 0 runs."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits
    from paper_1704_07669_b200.synth import config_shape
    cs = config_shape(args.config)
    n, l = cs["n"], cs["l"]
    es = 8 if args.config == "cfg1" else 4
    threads, phys = host_cores()
    ref = ref_module()
    kind = "reference" if ref is not None else "port"
    m = args.rows or cs["m"]
    if args.config != "cfg1":
        # ~1 GB/s of fp32 A per pass on 16 cores (measured): bound the run
        per_step_cap = max(4096, int(args.ref_budget_s / max(1, args.steps + args.warmup) * 1.0e9 / (n * es)))
        m = min(m, (per_step_cap // 4096) * 4096 or 4096)
    a = host_config_matrix(args.config, m)
    br = 200 if args.config == "cfg1" else 4096
    if ref is not None:
        omega = ref.linalg.gaussian_matrix(n, l, 1)

        def one_pass():
            return ref.sketch_pass(ref.ArrayRowStream(a), omega, block_rows=br)
    else:
        import oracle as O
        omega = O.gaussian(n, l, 1)

        def one_pass():
            return O.oracle_sketch(((r0, a[r0:r0 + br].astype(np.float64)) for r0 in range(0, m, br)), omega)
    times = []
    with threadpool_limits(limits=threads):
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            one_pass()
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
    sec = float(np.mean(times))
    value = m * n * es / sec / 1e9
    full = m == cs["m"]
    sample = (f"{'full' if full else 'row prefix of the'} config A: {m} x {n} "
              f"{'fp64' if es == 8 else 'fp32 widened to fp64 by ArrayRowStream'} per step, "
              f"block_rows {br}, {'unmodified reference streampca (baseline/_ref)' if ref else 'numpy oracle port'}")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sec,
        "higher_is_better": True, "scaling": scaling_mode(args), "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": workload_config(args.config if full else f"{args.config} row prefix", cs, m, m, world,
                                  scaling_mode(args)),
        "precision": "fp64 (numpy / BLAS)", "block_rows": br,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "cores_physical": phys, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def profile_traffic(rows: float, config: str):
    """(dram read+write bytes of the pass kernel over `rows` rows, source):
    scaled from the committed ncu --set full capture (profiles/ncu_summary.json)
    of the same config — a profile figure, not measured in this run."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            prof = json.load(fh)
        src = "ncu --set full capture, profiles/ncu_summary.json (%s), per-row bytes x rows" % prof.get(
            "capture", "committed profile")
        per = prof.get("per_config", {}).get(config)
        if per is not None:
            return per["dram_bytes_per_row"] * rows, src
        if prof.get("config", "cfg2") != config:
            return None, None
        return prof["dram_bytes_per_row"] * rows, src
    except Exception:
        return None, None


def run_stream(args):
    """Config 4 (out-of-HBM host streaming): A = 5 000 000 x 10 000 fp32 (200 GB,
    more than HBM) lives in page-locked host memory and every step streams all
    of it through the library (pinned double-buffered H2D on a copy stream,
    overlapped with the pass kernel). Host memory holds a ring of `--ring-gb`
    of distinct 4096-row blocks generated from seed(block index); block j of
    the stream is ring slot j mod R (rows repeat with period R blocks), so the
    bytes crossing the link per step are the full 200 GB. Bound: the host link."""
    import torch
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    from paper_1704_07669_b200 import GpuSketch, gaussian_matrix, synth
    from paper_1704_07669_b200.parallel import allreduce_sketch
    cs = synth.config_shape(args.config)
    m_total = args.rows or cs["m"]
    m = m_total // world
    n, l = cs["n"], cs["l"]
    B = synth.BLOCK
    nblk = (m + B - 1) // B
    ring = max(1, min(nblk, int(args.ring_gb * 1e9) // (B * n * 4)))
    host = torch.empty((ring, B, n), dtype=torch.float32, pin_memory=True)
    b0 = (rank * m) // B
    for j in range(ring):  # generated on the device from seed(block), parked in pinned memory
        blk = synth.config_matrix(args.config, device=dev, rows=((b0 + j) * B, (b0 + j + 1) * B),
                                  m_override=m_total)
        host[j].copy_(blk)
    torch.cuda.synchronize()
    # link peak: one large pinned H2D copy
    probe = torch.empty((min(ring, 6), B, n), dtype=torch.float32, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(3):
        e0.record()
        probe.copy_(host[:probe.shape[0]], non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, probe.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del probe
    omega = gaussian_matrix(n, l, 1)
    sk = GpuSketch(n, omega, np.float32, precision=args.precision, device=dev, rows_hint=m)
    stream = torch.cuda.current_stream(dev)

    def step():
        sk.reset()
        for j in range(nblk):
            r0 = j * B
            rows = min(B, m - r0)
            sk.push(host[j % ring][:rows], r0, final=(j == nblk - 1))
        g, h, c, rows = sk.finish(on_device=True)
        if pg is not None:
            allreduce_sketch(h, c, pg, rows=rows)
        return h

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    sk.enable_timing(True)
    launches0 = sk.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            h = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        hh = h.cpu()  # D2H of the step's result (e2e)
    if pg is not None:
        pg.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = sk.kernel_launches() - launches0
    kern_ms, _ = sk.kernel_time()
    sk.close()
    if pg is not None:
        t = torch.tensor([ms, wall], device=dev, dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms, wall = float(t[0]), float(t[1])
    ms_step = ms / args.steps
    value = world * m * n * 4 / (ms_step * 1e-3) / 1e9
    extra = {}
    if rank == 0 and world == 1 and not (args.no_cpu and args.no_parity):
        # config-4 prefix: the first P distinct blocks of the host ring (4 GB),
        # PCA through the streaming path (PinnedRowStream: H2D inside the
        # pass) against the unmodified reference on the same rows
        from paper_1704_07669_b200 import PcaConfig, PinnedRowStream, single_pass_pca
        pblk = min(ring, max(1, (4 << 30) // (B * n * 4)))
        pre = host[:pblk].reshape(pblk * B, n)
        cfg = PcaConfig(k=cs["k"], oversample=cs["l"] - cs["k"], seed=1)
        single_pass_pca(PinnedRowStream(pre), cfg, precision=args.precision, device=dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = single_pass_pca(PinnedRowStream(pre), cfg, precision=args.precision, device=dev)
        torch.cuda.synchronize()
        extra["pca_seconds_prefix"] = {"value": time.perf_counter() - t0, "unit": "s", "rows": int(pre.shape[0]),
                                       "includes": "Omega draw, pass streamed from pinned host memory, QB, SVD, "
                                                   "U/S/V to host"}
        extra.update(reference_leg(args, pre, res, cs, what=f"config-4 prefix of {pblk} blocks"))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "m": m_total, "m_per_gpu": m, "n": n, "l": l, "k": cs["k"],
                       "rank": cs["rank"], "spectrum": cs["spectrum"], "noise": cs["noise"],
                       "source": f"pinned host ring of {ring} distinct 4096-row blocks "
                                 f"({ring * B * n * 4 / 1e9:.1f} GB), block j = slot j mod {ring}",
                       "precision": "3xTF32 tcgen05" if sk.precision == "tc" else "FFMA",
                       "parallelism": f"row-shard x{world}",
                       "l2": "inputs larger than L2 (streamed from host)"},
            "roofline": {"bound": "host_link", "achieved": value / world, "peak": best, "unit": "GB/s",
                         "frac": value / world / best, "traffic": None,
                         "peak_desc": "measured pinned H2D copy (torch, 1 GB), this GPU",
                         "kernel_ms_per_pass": kern_ms / max(1, args.steps),
                         "kernel_share": kern_ms / max(1e-9, ms)},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "e2e": {"value": world * m * n * 4 / (wall / args.steps) / 1e9, "unit": UNIT,
                    "h2d_bytes_per_step": m * n * 4, "d2h_bytes_per_step": int(hh.numel() * 8),
                    "seconds_per_step": wall / args.steps},
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


def run_ours(args):
    import torch
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist

    from paper_1704_07669_b200 import GpuSketch, gaussian_matrix, synth
    from paper_1704_07669_b200.parallel import allreduce_sketch, shard_rows

    cs = synth.config_shape(args.config)
    mode = scaling_mode(args)
    n, l = cs["n"], cs["l"]
    if mode == "weak":  # every rank a full config matrix: rows [rank m, (rank + 1) m) of a world*m job
        m_total = (args.rows or cs["m"]) * world
        r0, r1 = rank * (m_total // world), (rank + 1) * (m_total // world)
    else:  # the config's fixed matrix split over the ranks
        m_total = args.rows or cs["m"]
        r0, r1 = shard_rows(m_total, world, rank)
    m = r1 - r0
    if args.config == "cfg1":  # the reference's fp64 case
        args.dtype = "f64"
    es = 8 if args.dtype == "f64" else 4
    npdt = np.float64 if args.dtype == "f64" else np.float32
    bytes_per_rank = m * n * es
    hbm_peak, bf16_peak, peak_kind = peaks()

    a = synth.config_matrix(args.config, device=dev, rows=(r0, r1), m_override=m_total)
    if args.dtype == "f64" and a.dtype != torch.float64:
        a = a.double()
    omega = gaussian_matrix(n, l, 1)
    sk = GpuSketch(n, omega, npdt, precision=args.precision, device=dev, rows_hint=m)
    stream = torch.cuda.current_stream(dev)

    def step():
        sk.reset()
        sk.push(a, 0, final=True)
        g, h, c, rows = sk.finish(on_device=True)
        if pg is not None:
            allreduce_sketch(h, c, pg, rows=rows)
        return g, h, c

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    sk.enable_timing(True)
    launches0 = sk.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # inputs smaller than L2 (config 1): flush L2 before every timed step and
    # sum the per-step event times (the flush itself is not timed)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if bytes_per_rank < (512 << 20) else None
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if flush is None:
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
        else:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for e_s, e_e in evs:
                flush.fill_(1)
                e_s.record(stream)
                step()
                e_e.record(stream)
            torch.cuda.synchronize()
            ms = sum(e_s.elapsed_time(e_e) for e_s, e_e in evs)
    if pg is not None:
        pg.barrier()
    launches = sk.kernel_launches() - launches0
    kern_ms, kern_chunks = sk.kernel_time()
    sk.enable_timing(False)
    if pg is not None:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = m_total * n * es / (ms_step * 1e-3) / 1e9

    # Roofline of the dominant kernel: the pass kernel (tc_pass_kernel, one
    # persistent launch per push) timed with CUDA events around its launches on
    # the library's stream over the timed region (spca_kernel_time_ms).
    chunk_rows = sk.chunk_rows()
    pass_ms = kern_ms / max(1, args.steps)
    pass_bytes = m * n * es
    flops = 4.0 * m * n * l
    used_tc = sk.precision == "tc"
    if used_tc:
        peak_tf = bf16_peak / 2.0 / 3.0   # 3xTF32: tf32 = bf16/2, three products
        peak_desc = "3xTF32 effective = measured bf16 burst / 2 (tf32) / 3 (products)"
    elif args.dtype == "f64":
        peak_tf = 148 * 64 * 2 * 1.965e9 / 1e12  # fp64: DMMA = DFMA on B200 (tools/dmma_bench.cu: 37.2 TF)
        peak_desc = "fp64 tensor (DMMA) = DFMA rate, 148 SMs x 64 x 2 x 1965 MHz (measured 37.2 TF/s)"
    else:
        peak_tf = 148 * 128 * 2 * 1.965e9 / 1e12  # FFMA nominal
        peak_desc = "FFMA nominal (148 SMs x 128 lanes x 2 x 1965 MHz)"
    hbm_floor = pass_bytes / (hbm_peak * 1e9)
    tc_floor = flops / (peak_tf * 1e12)
    achieved_tf = flops / (pass_ms * 1e-3) / 1e12
    achieved_gbs = pass_bytes / (pass_ms * 1e-3) / 1e9
    if tc_floor >= hbm_floor:
        roofline = {"bound": "tensor", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": achieved_tf / peak_tf}
    else:
        roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved_gbs / hbm_peak}
    traffic, traffic_src = profile_traffic(m, args.config) if used_tc else (None, None)
    roofline.update({
        "traffic": traffic, "traffic_source": traffic_src,
        "peak_kind": peak_kind, "peak_desc": peak_desc,
        "kernel": "tc_pass_kernel (persistent, CTA pairs; G + H + column sums of all chunks)" if used_tc
                  else "sketch chunk: simt_g_kernel + simt_h_kernel + colsum (DMMA for fp64)",
        "kernel_ms_per_pass": pass_ms, "kernel_share": kern_ms / max(1e-9, ms), "chunk_rows": chunk_rows,
        "hbm": {"achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_gbs / hbm_peak},
        "algorithmic_bytes_per_pass": pass_bytes, "flops_per_pass": flops,
        "floors_ms_per_pass": {"hbm": hbm_floor * 1e3, "tensor": tc_floor * 1e3},
    })
    sk.close()

    out = {}
    if not args.no_e2e:
        out.update(e2e_leg(args, a, omega, dev, pg, world, rank))
    res_dev = None
    if not args.no_pca:
        pca, res_dev = pca_leg(args, a, dev, pg, world, rank)
        out.update(pca)
    if rank == 0 and world == 1 and not (args.no_cpu and args.no_parity):
        out.update(reference_leg(args, a, res_dev, cs))
    if pg is not None:
        pg.barrier()
    if rank != 0:
        if pg is not None:
            pg.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": mode, "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        # the workload only (identical in the reference arm's line); how this arm
        # computes it is in "precision"
        "config": workload_config(args.config, cs, m_total, m, world, mode),
        "precision": "3xTF32 tcgen05" if used_tc else ("DMMA fp64" if args.dtype == "f64" else "FFMA"),
        "l2": ("inputs larger than L2 (A is %.1f GB per GPU)" % (bytes_per_rank / 1e9)
               if flush is None else
               "L2 flushed before every timed step (512 MB write, untimed; A is %.0f MB)"
               % (bytes_per_rank / 1e6)),
        "roofline": roofline,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "tflops": 4.0 * m_total * n * l / (ms_step * 1e-3) / 1e12,
    }
    line.update(out)
    print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


def _max_over_ranks(x: float, pg, dev) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def e2e_leg(args, a_dev, omega, dev, pg, world, rank):
    """Same metric through the public API (GpuSketch.push / finish), every
    step from HOST memory: (e2e) A in page-locked memory, (e2e_pageable) A in a
    plain numpy array — the reference's own input type. Each step pushes all
    of A (H2D inside the library, overlapped with the pass), finishes, reads
    G, H and the column sums back to the host, and (N > 1) all-reduces the
    sketch. K timed steps after one warm-up; wall clock, max over ranks."""
    import torch
    from paper_1704_07669_b200 import GpuSketch
    from paper_1704_07669_b200.parallel import allreduce_sketch
    m, n = a_dev.shape
    es = a_dev.element_size()
    host = torch.empty((m, n), dtype=a_dev.dtype, pin_memory=True)
    host.copy_(a_dev)
    torch.cuda.synchronize()
    npdt = np.float64 if a_dev.dtype == torch.float64 else np.float32
    sk = GpuSketch(n, omega, npdt, precision=args.precision, device=dev, rows_hint=m)
    out = {}
    for key, src in (("e2e", host), ("e2e_pageable", None)):
        if src is None:
            src = host.numpy().copy()  # plain pageable numpy array
        d2h = 0

        def one():
            sk.reset()
            sk.push(src, 0, final=True)
            g, h, c, rows = sk.finish(on_device=pg is not None)
            if pg is not None:
                allreduce_sketch(h, c, pg, rows=rows)
                g, h, c = g.cpu(), h.cpu(), c.cpu()
            return int(g.nbytes + h.nbytes + c.nbytes) if hasattr(g, "nbytes") else 0

        one()
        torch.cuda.synchronize()
        if pg is not None:
            pg.barrier()
        steps = args.steps if key == "e2e" else max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(steps):
            d2h = one()
        torch.cuda.synchronize()
        t = _max_over_ranks((time.perf_counter() - t0) / steps, pg, dev)
        out[key] = {"value": world * m * n * es / t / 1e9, "unit": UNIT, "h2d_bytes_per_step": m * n * es,
                    "d2h_bytes_per_step": int(d2h), "seconds_per_step": t, "steps": steps,
                    "source": "page-locked host tensor" if key == "e2e" else "pageable numpy array"}
        del src
    sk.close()
    del host
    return out


def pca_leg(args, a_dev, dev, pg, world, rank):
    """End-to-end PCA seconds through the public entry point: with A resident
    in HBM (DeviceRowStream), and (N = 1) from a plain numpy array as the
    reference receives it (H2D inside). N > 1: sharded_single_pass_pca (the
    row-sum of Eq. 10, one all-reduce, gathered G), max over ranks.
    Returns (fields, the HBM-resident result)."""
    import torch
    from paper_1704_07669_b200 import DeviceRowStream, PcaConfig, single_pass_pca
    from paper_1704_07669_b200.parallel import sharded_single_pass_pca
    from paper_1704_07669_b200.synth import config_shape
    cs = config_shape(args.config)
    cfg = PcaConfig(k=cs["k"], oversample=cs["l"] - cs["k"], seed=1)
    out = {}
    if pg is not None:
        sharded_single_pass_pca(a_dev, cfg, pg, precision=args.precision, device=dev)
        torch.cuda.synchronize()
        pg.barrier()
        t0 = time.perf_counter()
        res = sharded_single_pass_pca(a_dev, cfg, pg, precision=args.precision, device=dev)
        torch.cuda.synchronize()
        t = _max_over_ranks(time.perf_counter() - t0, pg, dev)
        out["pca_seconds"] = {"value": t, "unit": "s", "k": cfg.k, "l": cfg.l, "s0": float(res.s[0]),
                              "includes": "Omega draw, sharded sketch pass, all-reduce, G gather, QB, SVD, "
                                          "U/S/V to host (max over ranks)"}
        return out, res
    single_pass_pca(DeviceRowStream(a_dev), cfg, precision=args.precision, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = single_pass_pca(DeviceRowStream(a_dev), cfg, precision=args.precision, device=dev)
    torch.cuda.synchronize()
    out["pca_seconds"] = {"value": time.perf_counter() - t0, "unit": "s", "k": cfg.k, "l": cfg.l,
                          "s0": float(res.s[0]),
                          "includes": "Omega draw, sketch pass (A in HBM), QB, SVD, U/S/V to host"}
    a_np = a_dev.cpu().numpy()
    single_pass_pca(a_np, cfg, precision=args.precision, device=dev)
    t0 = time.perf_counter()
    single_pass_pca(a_np, cfg, precision=args.precision, device=dev)
    torch.cuda.synchronize()
    out["pca_seconds_host"] = {"value": time.perf_counter() - t0, "unit": "s",
                               "includes": "same, A a pageable numpy array (H2D of A inside)"}
    del a_np
    return out, res


def reference_leg(args, a_dev, res, cs, what: str = "full config A"):
    """N = 1: the unmodified reference (baseline/_ref) on this host's cores
    over the SAME A (the device matrix copied to the host, fp32 widened to
    fp64 by the reference's ArrayRowStream) and the same seeded Omega:
    (cpu_baseline) its sketch_pass GB/s over the full A and its
    single_pass_pca seconds; (parity) our U, S, V against its U, S, V —
    max relative S error and the largest principal angles of U and V
    (BASELINE.json bar: 1e-4 fp32, 1e-10 fp64)."""
    from threadpoolctl import threadpool_limits
    ref = ref_module()
    threads, phys = host_cores()
    out = {}
    if ref is None:
        if not args.no_cpu:
            r, dt = cpu_oracle_rate(8192, cs["n"], cs["l"], seed=0, threads=threads)
            out["cpu_baseline"] = {"value": r, "unit": UNIT, "cores": threads, "cores_physical": phys,
                                   "kind": "port", "sample": f"8192 rows x {cs['n']} fp32 (widened to fp64), "
                                   f"numpy oracle sketch, {dt:.1f} s (baseline/_ref absent)"}
        return out
    a_host = a_dev.cpu().numpy()
    m, n = a_host.shape
    l = cs["l"]
    br = 200 if args.config == "cfg1" else 4096
    cfg = ref.PcaConfig(k=cs["k"], oversample=l - cs["k"], seed=1)
    # A above 6 GB goes through the reference's GeneratorRowStream over fp32
    # row blocks (widened to fp64 per block, as FileRowStream does at
    # streams.py:128) instead of ArrayRowStream's whole fp64 copy, which
    # would not fit host memory beside A at config 5 (40 GB -> 80 GB)
    streamed = a_host.nbytes > (6 << 30)

    def src():
        if streamed:
            return ref.GeneratorRowStream((a_host[r:r + br] for r in range(0, m, br)), n)
        return ref.ArrayRowStream(a_host)
    with threadpool_limits(limits=threads):
        omega = ref.linalg.gaussian_matrix(n, l, 1)
        t0 = time.perf_counter()
        ref.sketch_pass(src(), omega, block_rows=br)
        t_sketch = time.perf_counter() - t0
        t0 = time.perf_counter()
        rs = ref.single_pass_pca(src() if streamed else a_host, cfg, block_rows=br)
        t_pca = time.perf_counter() - t0
    del a_host
    out["cpu_baseline"] = {
        "value": m * n * a_dev.element_size() / t_sketch / 1e9, "unit": UNIT, "cores": threads,
        "cores_physical": phys, "kind": "reference", "pass_seconds": t_sketch, "pca_seconds": t_pca,
        "sample": f"{what} ({m} x {n} {'fp64' if a_dev.element_size() == 8 else 'fp32 widened to fp64'}), "
                  f"unmodified reference streampca (baseline/_ref): sketch_pass("
                  f"{'GeneratorRowStream(fp32 row blocks)' if streamed else 'ArrayRowStream(A)'}, Omega, "
                  f"block_rows={br}) and single_pass_pca(A, PcaConfig(k={cs['k']}, oversample={l - cs['k']}, "
                  f"seed=1), block_rows={br}), threadpoolctl {threads} threads"}
    if res is not None and not args.no_parity:
        s_ours = np.asarray(res.s, dtype=np.float64)
        s_ref = np.asarray(rs.s, dtype=np.float64)
        out["parity"] = {
            "s_rel_max": float(np.max(np.abs(s_ours - s_ref) / np.abs(s_ref))),
            "angle_u_max": max_angle(res.u, rs.u), "angle_v_max": max_angle(res.v, rs.v),
            "k": int(cs["k"]), "bar": 1e-10 if a_dev.element_size() == 8 else 1e-4,
            "against": "reference single_pass_pca (baseline/_ref) on the same A and seeded Omega, "
                       "this host, this run"}
        p = out["parity"]
        p["pass"] = bool(max(p["s_rel_max"], p["angle_u_max"], p["angle_v_max"]) <= p["bar"])
    return out


def spawn(args) -> int:
    """--gpus N without a launcher: re-run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "cfg4":
        run_stream(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
