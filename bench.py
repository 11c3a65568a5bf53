"""Benchmark: lambda-graph min-cuts/sec of the supergraph path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
                    [--impl b200|reference] [--no-cpu-baseline] [--no-cpmc]

One step = one pass of the hot path over one batch: the seed supergraph of
BASELINE.json config 2 (synthetic 500x375 image, 1 seed, 20-lambda ladder,
integer capacities) built, solved and decoded on one GPU = 20 lambda-cuts.
Under torchrun (N > 1) every rank solves its own supergraph per step (weak
scaling, independent supergraphs, no data-path collective); ranks only
meet in barriers and a max-reduction of their times.

value : whole-job lambda-cuts/s with the seed planes already resident in
        HBM (pmf_seed_run), device time from CUDA events on the engine's
        stream, L2 flushed (256 MiB memset) between steps, max over ranks.
e2e   : the same metric through the public API (solve_seed_supergraph)
        from host SeedProblem objects: conversion + H2D + solve + D2H of
        every label mask + CutResult construction, wall clock per step.
--impl reference : the reference solver's algorithm (oracle/, a C
        restatement of pmflow's push-relabel) on the host cores, same
        config, same metric.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "lambda-graph min-cuts/sec"
UNIT = "lambda-cuts/s"
CONFIGS = {
    "c1": dict(w=160, h=120, rows=1, cols=1, types=("A",), lams="default",
               desc="C1: synthetic 160x120, 1 seed, DEFAULT 20-lambda ladder, one supergraph"),
    "c2": dict(w=500, h=375, rows=1, cols=1, types=("A",), lams="L20",
               desc="C2: synthetic 500x375 (VOC-sized), 1 seed, 20-lambda ladder L20, "
                    "one supergraph (20 lambda-graphs) per GPU per step"),
    "c3": dict(w=500, h=375, rows=5, cols=5, types=("A", "B"), lams="L20",
               desc="C3: one CPMC-style image per GPU per step -- synthetic 500x375, 25 seeds x "
                    "2 seed types x 20 lambdas = 1000 lambda-graphs in one device batch "
                    "(warm-start chains along the schedule)"),
    "c4": dict(w=1920, h=1080, rows=1, cols=1, types=("A",), lams="C4",
               desc="C4: synthetic 1920x1080, 1 seed, 8 lambdas per supergraph"),
    "c5": dict(w=500, h=375, rows=5, cols=5, types=("A", "B"), lams="L20", images=8,
               desc="C5: batch throughput -- 8 synthetic CPMC images (500x375, 25 seeds x 2 types "
                    "x 20 lambdas) per GPU per step, images independent across GPUs"),
}
# CPU reference sample per step for the big configs (the full C3 image is
# ~3,400 CPU-s on the reference algorithm): the first problems' lambda graphs
REF_SAMPLE_PROBLEMS = {"c3": 2, "c5": 2, "c4": 1}
BYTES_PER_PIXEL_PASS = {4: 24, 16: 48}   # load+store of w, h and the residual word(s)
# algorithmic bytes per pixel of one tile pass of each kind of the
# asynchronous solver, by residual word size 4 / 16:
#   push  load+store w, h, r          bfs   load h, r; store h
#   lab   load lab, r; store lab      binit load w; store h
#   seed  load w, h                   linit load w; store lab
#   emit  load w, lab|h, mask, slope; store out, w, h (next lambda's init)
ASYNC_BYTES = {"push_tile_passes": (24, 48), "bfs_tile_passes": (12, 24), "label_tile_passes": (6, 18),
               "binit_tile_passes": (8, 8), "seed_tile_passes": (8, 8), "linit_tile_passes": (5, 5),
               "emit_tile_passes": (22, 22)}


# ----------------------------------------------------------------- helpers

def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def shard(n_units: int, rank: int, world: int):
    """Contiguous block of unit indices owned by ``rank`` (independent
    supergraphs; no exchange between ranks)."""
    base, extra = divmod(n_units, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def reduce_max(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(device=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        if device is not None and dist.get_backend() == "nccl":
            dist.barrier(device_ids=[device])
        else:
            dist.barrier()


def lambdas_for(name):
    from paper_1509_06004_b200 import synth
    from paper_1509_06004_b200.parametric import DEFAULT_LAMBDA_VALUES
    return {"default": DEFAULT_LAMBDA_VALUES, "L20": synth.L20, "C4": synth.C4_LAMBDAS}[name]


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def committed_traffic(kernel, config):
    """Per-launch DRAM bytes (ncu dram__bytes_read + write) of `kernel` on
    `config` from the committed capture in profiles/traffic.json, or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return d.get(kernel, {}).get("per_config", {}).get(config, {}).get("dram_bytes_per_launch")


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    every 5 ms from a thread (short regions still get samples), nvidia-smi
    as the fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.nvml = index, [], None, None
        self._stop = threading.Event()

    def _nvml_loop(self):
        nv, h = self.nvml
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for b in bits])
            except Exception:  # noqa: BLE001
                pass
            if self._stop.wait(0.005):
                return

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = (nv, nv.nvmlDeviceGetHandleByIndex(self.index))
            self._t = threading.Thread(target=self._nvml_loop, daemon=True)
            self._t.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        self._stop.set()
        if self.nvml is not None:
            self._t.join(timeout=5)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


# ------------------------------------------------------------- CPU baseline

def cpu_solve_config(cfg, rng_seed, threads, max_problems=None):
    """The reference's solver (C restatement in oracle/) on every lambda graph
    of one supergraph (or of the first ``max_problems`` problems), per lambda
    as solve_schedule_sequential does; returns (n_cuts, seconds, total_flow)."""
    import oracle
    from paper_1509_06004_b200 import synth
    lams = lambdas_for(cfg["lams"])
    batch = synth.generate(cfg["w"], cfg["h"], cfg["rows"], cfg["cols"], rng_seed=rng_seed,
                           types=cfg["types"])
    jobs = []
    for p in batch.problems[:max_problems]:
        for lam in lams:
            s, t, nb = oracle.instantiate(p.unary_base, p.unary_slope, p.sink_base, p.pairwise,
                                          p.fg_seeds, p.bg_seeds, lam)
            jobs.append((cfg["w"], cfg["h"], s, t, nb))
    t0 = time.perf_counter()
    res = oracle.solve_many(jobs, threads=threads)
    dt = time.perf_counter() - t0
    return len(jobs), dt, sum(r[0] for r in res)


def run_reference(args, cfg):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import oracle
    oracle.build()
    threads = os.cpu_count() or 1
    mp = REF_SAMPLE_PROBLEMS.get(args.config)
    for _ in range(args.warmup):
        cpu_solve_config(cfg, 0, threads, mp)
    tot_cuts, tot_s = 0, 0.0
    for _ in range(args.steps):
        n, dt, _ = cpu_solve_config(cfg, 0, threads, mp)
        tot_cuts += n
        tot_s += dt
    value = tot_cuts / tot_s
    what = (f"the lambda-graphs of the first {mp} seed problems" if mp else
            "all lambda-graphs of one supergraph")
    sample = (f"{cfg['desc']}: {what} per step ({tot_cuts // args.steps} graphs), solved with the "
              f"reference push-relabel restated in C (oracle/pmflow_oracle.c), per lambda as "
              f"solve_schedule_sequential, {threads} host threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": {"workload": cfg["desc"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU arm

def run_b200(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1509_06004_b200 import LambdaSchedule, _native, solve_seed_supergraph, synth
    from paper_1509_06004_b200.supergraph import check_seed_supergraph

    rank, local, world = dist_env()
    ndev = torch.cuda.device_count()
    dev = local % ndev          # one GPU per rank (shared only when testing N > #GPUs)
    torch.cuda.set_device(dev)
    if world > 1:
        if ndev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:   # NCCL cannot put two ranks on one GPU: plumbing-only test mode
            dist.init_process_group("gloo")
    sched = LambdaSchedule(lambdas_for(cfg["lams"]))
    # weak scaling with fixed per-GPU work: every rank solves the same
    # synthetic image(s) (rng_seed = i), so the max over ranks measures the
    # system, not the spread of data-dependent difficulty between images
    nimg = cfg.get("images", 1)
    problems = []
    for i in range(nimg):
        batch = synth.generate(cfg["w"], cfg["h"], cfg["rows"], cfg["cols"],
                               rng_seed=i, types=cfg["types"])
        problems += check_seed_supergraph(batch.problems, sched, "auto")
    cuts_per_step = len(problems) * len(sched)

    solver = _native.solver_for_thread(dev)
    stream = torch.cuda.ExternalStream(solver.stream_handle(), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    solver.seed_stage(cfg["w"], cfg["h"], problems, sched.values, "auto")
    for _ in range(args.warmup):
        solver.seed_run()
    _, ref_flows, _ = solver.seed_fetch(labels=False)

    # ---- device-resident timed region
    barrier(dev)
    torch.cuda.synchronize()
    steps_ms, stats = [], []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()                      # L2 flush, outside the timed events
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            solver.seed_run()
            with torch.cuda.stream(stream):
                e1.record(stream)
            e1.synchronize()
            steps_ms.append(e0.elapsed_time(e1))
            stats.append(solver.stats())
    torch.cuda.synchronize()
    barrier(dev)
    _, flows, _ = solver.seed_fetch(labels=False)
    assert (flows == ref_flows).all(), "flows changed between runs"
    dev_s = sum(steps_ms) / 1e3
    dev_s_max = reduce_max(dev_s, torch.device("cuda", dev))
    value = world * cuts_per_step * args.steps / dev_s_max

    # roofline of the dominant kernel: the asynchronous solve kernel (every
    # phase of every grid, one launch per step) or, step-synchronous, the
    # push-relabel discharge
    peak, peak_kind = measured_peaks()
    edge_bytes = stats[-1]["edge_bytes"]
    total_ms = sum(s["ms_device"] for s in stats)
    if stats[-1]["async_mode"]:
        col = 0 if edge_bytes == 4 else 1
        kern_ms = sum(s["ms_async"] for s in stats)
        alg_bytes = sum(s[k] * 1024 * v[col] for s in stats for k, v in ASYNC_BYTES.items())
        achieved = alg_bytes / args.steps / (kern_ms / 1e3 / args.steps) / 1e9 if kern_ms else 0.0
        roofline = {"bound": "hbm", "kernel": "k_async (asynchronous solve: relabel, discharge, labels, "
                                              "emit of every grid in one persistent launch)",
                    "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": committed_traffic("k_async", args.config), "peak_kind": peak_kind,
                    "bytes_per_pixel_pass": {k.replace("_tile_passes", ""): v[col] for k, v in ASYNC_BYTES.items()},
                    "tile_passes_per_step": {k.replace("_tile_passes", ""): stats[-1][k] for k in ASYNC_BYTES},
                    "avg_launch_us": kern_ms * 1e3 / args.steps,
                    "time_share": {"k_async": round(kern_ms / total_ms, 4) if total_ms else None}}
    else:
        push_ms = sum(s["ms_push"] for s in stats)
        push_launches = sum(s["push_sweeps"] for s in stats)
        tile_passes = sum(s["push_tile_passes"] for s in stats)
        bpp = BYTES_PER_PIXEL_PASS[edge_bytes]
        alg_bytes_per_launch = tile_passes * 1024 * bpp / max(push_launches, 1)
        avg_launch_s = push_ms / 1e3 / max(push_launches, 1)
        achieved = alg_bytes_per_launch / avg_launch_s / 1e9 if avg_launch_s else 0.0
        share = {k: round(sum(s[k] for s in stats) / total_ms, 4) for k in
                 ("ms_push", "ms_bfs", "ms_labels")} if total_ms else {}
        roofline = {"bound": "hbm", "kernel": "k_push (push-relabel tile discharge)",
                    "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": committed_traffic("k_push", args.config), "peak_kind": peak_kind,
                    "bytes_per_pixel_pass": bpp,
                    "pixel_passes_per_s": tile_passes * 1024 / (push_ms / 1e3) if push_ms else 0,
                    "avg_launch_us": avg_launch_s * 1e6,
                    "time_share": share}

    # ---- end to end through the public API (host SeedProblems in, CutResults out)
    e2e_s, h2d, d2h = 0.0, 0, 0
    barrier(dev)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        res = solve_seed_supergraph(problems, sched, "auto", device=dev)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_s += dt
            st = solver.stats()
            h2d += st["h2d_bytes"]
            d2h += st["d2h_bytes"]
    assert [c.flow for c in res.cuts] == [int(f) for f in ref_flows.reshape(-1)]
    e2e_s_max = reduce_max(e2e_s, torch.device("cuda", dev))
    e2e_value = world * cuts_per_step * args.steps / e2e_s_max

    # ---- CPMC image (C3) device time, reported beside the headline
    cpmc = None
    if args.cpmc and rank == 0 and args.config not in ("c3", "c5"):
        c3 = synth.generate(500, 375, 5, 5, rng_seed=0, types=("A", "B"))
        s3sched = LambdaSchedule(synth.L20)      # C3's ladder, whatever the headline config
        c3p = check_seed_supergraph(c3.problems, s3sched, "auto")
        s3 = _native.Solver(dev)
        s3.seed_stage(500, 375, c3p, s3sched.values, "auto")
        s3.seed_run()
        s3.seed_run()
        st3 = s3.stats()
        cpmc = {"ms_per_image": round(st3["ms_device"], 3), "lambda_cuts": len(c3p) * len(s3sched),
                "lambda_cuts_per_s": round(len(c3p) * len(s3sched) / st3["ms_device"] * 1e3, 1),
                "image": "500x375, 25 seeds x 2 types x 20 lambdas, one device batch"}
        s3.close()

    # ---- CPU baseline (rank 0, N == 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        threads = os.cpu_count() or 1
        mp = REF_SAMPLE_PROBLEMS.get(args.config)
        n, dt, flow = cpu_solve_config(cfg, 0, threads, mp)
        if mp is None:
            assert flow == int(ref_flows.sum()), "oracle and engine disagree on the flow"
        else:
            assert flow == int(ref_flows.reshape(-1)[:n].sum()), "oracle and engine disagree"
        cpu = {"value": n / dt, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{n} lambda-graphs of the rank-0 batch ({cfg['desc'].split(':')[0]}"
                         f"{', first %d problems' % mp if mp else ''}), "
                         "reference push-relabel restated in C (oracle/pmflow_oracle.c), "
                         f"per lambda, {threads} threads; took {dt:.2f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dev_s_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": cfg["desc"], "lambda_cuts_per_step_per_gpu": cuts_per_step,
                       "image": f"{cfg['w']}x{cfg['h']}", "rng_seed": "0.. per image, the same on every rank",
                       "l2": "flushed between steps (256 MiB memset, outside the timed events)",
                       "parallelism": f"{world} GPU(s), independent supergraphs, no collectives"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                    "d2h_bytes_per_step": d2h // args.steps},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": int(sum(s["kernels"] for s in stats)),
            "solver": {k: stats[-1][k] for k in ("async_mode", "cycles", "steps", "push_sweeps",
                                                  "push_tile_passes", "bfs_sweeps", "bfs_tile_passes",
                                                  "label_tile_passes", "scan_tile_passes", "tiles",
                                                  "edge_bytes", "grids")},
            "cpmc": cpmc,
        }
        if args.config in ("c3", "c5"):
            line["ms_per_image"] = 1e3 * dev_s_max / args.steps / nimg
            line["e2e"]["ms_per_image"] = 1e3 * e2e_s_max / args.steps / nimg
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpmc", dest="cpmc", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
