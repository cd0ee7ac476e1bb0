"""Benchmark of the sketch pass (BASELINE.json metric: sketch-pass GB/s of A).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--precision auto|simt|tc]

A step = one full sketch pass (Algorithm 4 steps 4-8) over the config's A,
resident in HBM: every row pushed through libspca, H flushed, G widened, the
state finished on the device; with N > 1 ranks each rank owns its own row
shard (weak scaling: the per-GPU shard is the config's full m) and the step
ends with the NCCL all-reduce of [H | col_sums | rows].

The JSON line (rank 0) carries: value (whole-job GB/s of A), e2e (same
metric through the public API with A in pinned host memory, H2D and the D2H
of the sketch inside the timed region), roofline (dominant kernel group),
cpu_baseline (the numpy oracle port on this host's cores, bounded sample),
clocks sampled during the timed region, gpu_launches.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sketch-pass GB/s of A"
UNIT = "GB/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="cfg2")
    p.add_argument("--precision", default="auto")
    p.add_argument("--rows", type=int, default=None, help="override m (debug)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-pca", action="store_true")
    p.add_argument("--ring-gb", type=float, default=16.0, help="cfg4: pinned host ring size")
    p.add_argument("--dtype", default="f32", choices=["f32", "f64"],
                   help="element type of A (f64: the config's values widened, DFMA path)")
    return p.parse_args()


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


def run_reference(args):
    """Reference arm: the CPU implementation of the path (the oracle port —
    the reference is pure Python/numpy, nothing to compile), all host
    threads, a bounded sample of the same workload per step."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    from paper_1704_07669_b200.synth import config_shape
    cs = config_shape(args.config)
    threads = os.cpu_count() or 1
    sample_rows = 8192
    rates, times = [], []
    for i in range(min(args.warmup, 3) + min(args.steps, 10)):
        r, dt = cpu_oracle_rate(sample_rows, cs["n"], cs["l"], seed=i, threads=threads)
        if i >= min(args.warmup, 3):
            rates.append(r)
            times.append(dt)
    value = float(np.mean(rates))
    one_thread, _ = cpu_oracle_rate(sample_rows // 2, cs["n"], cs["l"], seed=7, threads=1)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": len(rates),
        "warmup": min(args.warmup, 3), "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{args.config} sample", "m": sample_rows, "n": cs["n"], "l": cs["l"],
                   "block_rows": 4096},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "value_1_thread": one_thread,
                         "sample": f"{sample_rows} rows x {cs['n']} fp32 widened to fp64 per step "
                                   "(numpy oracle of sketch.py:52-116, blocked path)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def profile_traffic(rows: float, config: str):
    """dram read+write bytes of the pass kernel over `rows` rows, scaled from the
    committed ncu --set full capture (profiles/ncu_summary.json) of the same config."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            prof = json.load(fh)
        per = prof.get("per_config", {}).get(config)
        if per is not None:
            return per["dram_bytes_per_row"] * rows
        if prof.get("config", "cfg2") != config:
            return None
        return prof["dram_bytes_per_row"] * rows
    except Exception:
        return None


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
    from paper_1704_07669_b200.parallel import allreduce_sketch

    cs = synth.config_shape(args.config)
    m = args.rows or cs["m"]
    n, l = cs["n"], cs["l"]
    if args.config == "cfg1":  # the reference's fp64 case
        args.dtype = "f64"
    es = 8 if args.dtype == "f64" else 4
    npdt = np.float64 if args.dtype == "f64" else np.float32
    bytes_per_rank = m * n * es
    hbm_peak, bf16_peak, peak_kind = peaks()

    # this rank's shard: rows [rank*m, (rank+1)*m) of the job's matrix
    a = synth.config_matrix(args.config, device=dev, rows=(rank * m, (rank + 1) * m),
                            m_override=m * world)
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
    value = world * bytes_per_rank / (ms_step * 1e-3) / 1e9

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
    roofline.update({
        "traffic": profile_traffic(m, args.config) if used_tc else None,
        "peak_kind": peak_kind, "peak_desc": peak_desc,
        "kernel": "tc_pass_kernel (persistent, CTA pairs; G + H + column sums of all chunks)" if used_tc
                  else "sketch chunk: simt_g_kernel + simt_h_kernel + colsum (DMMA for fp64)",
        "kernel_ms_per_pass": pass_ms, "chunk_rows": chunk_rows,
        "hbm": {"achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_gbs / hbm_peak},
        "algorithmic_bytes_per_pass": pass_bytes, "flops_per_pass": flops,
        "floors_ms_per_pass": {"hbm": hbm_floor * 1e3, "tensor": tc_floor * 1e3},
    })

    out = {}
    if rank == 0 and not args.no_e2e:
        out["e2e"] = e2e_leg(args, a, omega, dev)
    if rank == 0 and not args.no_pca:
        out["pca_seconds"] = pca_leg(args, a, dev)
    if rank == 0 and not args.no_cpu:
        r, dt = cpu_oracle_rate(4096 * 2, n, l, seed=0, threads=os.cpu_count() or 1)
        out["cpu_baseline"] = {"value": r, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
                               "sample": f"8192 rows x {n} fp32 (widened to fp64), numpy oracle sketch, "
                                         f"{dt:.1f} s"}
    sk.close()
    if pg is not None:
        pg.barrier()
    if rank != 0:
        if pg is not None:
            pg.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": args.config, "m_per_gpu": m, "n": n, "l": l, "k": cs["k"],
                   "rank": cs["rank"], "spectrum": cs["spectrum"], "noise": cs["noise"],
                   "precision": "3xTF32 tcgen05" if used_tc else ("DMMA fp64" if args.dtype == "f64" else "FFMA"),
                   "parallelism": f"row-shard x{world}",
                   "l2": ("inputs larger than L2 (A is %.1f GB per GPU)" % (bytes_per_rank / 1e9)
                          if flush is None else
                          "L2 flushed before every timed step (512 MB write, untimed; A is %.0f MB)"
                          % (bytes_per_rank / 1e6))},
        "roofline": roofline,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "tflops": 4.0 * m * n * l * world / (ms_step * 1e-3) / 1e12,
    }
    line.update(out)
    print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


def e2e_leg(args, a_dev, omega, dev, steps=3):
    """Same metric through the public API: A in pinned host memory; each
    step pushes it (H2D inside the library, overlapped with compute) and
    reads the finished sketch back to the host."""
    import torch
    from paper_1704_07669_b200 import GpuSketch
    m, n = a_dev.shape
    host = torch.empty((m, n), dtype=a_dev.dtype, pin_memory=True)
    host.copy_(a_dev)
    torch.cuda.synchronize()
    sk = GpuSketch(n, omega, np.float64 if a_dev.dtype == torch.float64 else np.float32,
                   precision=args.precision, device=dev, rows_hint=m)
    times = []
    d2h = 0
    for i in range(steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sk.reset()
        sk.push(host, 0, final=True)
        g, h, c, rows = sk.finish(on_device=False)
        dt = time.perf_counter() - t0
        d2h = g.nbytes + h.nbytes + c.nbytes
        if i:
            times.append(dt)
    sk.close()
    del host
    t = float(np.median(times))
    es = a_dev.element_size()
    return {"value": m * n * es / t / 1e9, "unit": UNIT, "h2d_bytes_per_step": m * n * es,
            "d2h_bytes_per_step": int(d2h), "seconds_per_step": t}


def pca_leg(args, a_dev, dev):
    """End-to-end PCA seconds (sketch + GPU post-pass) on the resident A."""
    import torch
    from paper_1704_07669_b200 import DeviceRowStream, PcaConfig, single_pass_pca
    from paper_1704_07669_b200.synth import config_shape
    cs = config_shape(args.config)
    cfg = PcaConfig(k=cs["k"], oversample=cs["l"] - cs["k"], seed=1)
    single_pass_pca(DeviceRowStream(a_dev), cfg, precision=args.precision, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = single_pass_pca(DeviceRowStream(a_dev), cfg, precision=args.precision, device=dev)
    torch.cuda.synchronize()
    return {"value": time.perf_counter() - t0, "unit": "s", "k": cfg.k, "l": cfg.l,
            "s0": float(res.s[0]), "includes": "Omega draw, sketch pass, QB, SVD, U/S/V to host"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "cfg4":
        run_stream(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
