"""Benchmark: lambda-graph min-cuts/sec of the supergraph path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5]
                    [--impl b200|reference] [--no-cpu-baseline] [--no-secondary]

Default workload (BASELINE.json config 5, the multi-GPU headline; its unit
of work is config 3's CPMC image): a pool of 256 distinct synthetic CPMC
images (500x375, rng_seed 0..255; 25 seeds x 2 seed types x 20 lambdas =
1,000 lambda-graphs each), cut into 8 batches of 32 images.  One step of a
rank = one batch, CLAIMED DYNAMICALLY: the rank takes the next batch of the
shared FIFO (a counter on the process group's store, the torchrun
analogue of run_dynamic's token queue, scheduler.py:253-292) and solves it
as one device batch (32,000 lambda-cuts; a larger batch amortises the
latency-bound tail of its slowest chains: 24.3 / 22.5 / 19.9 ms per image
at 8 / 16 / 32 images).  Per-GPU work per step is fixed, so scaling is weak; no
data-path collective exists (ranks share only the claim counter, barriers
and a max-reduction, over gloo -- no NCCL).

value : whole-job lambda-cuts/s with the batch's seed planes already
        resident in HBM (pmf_seed_stage before the timed events), device
        time of pmf_seed_run from CUDA events on the engine's stream, L2
        flushed between steps, max over ranks.
e2e   : the same metric through the public API on FRESH SeedProblem objects
        of the same batches the device-resident loop solved (generated
        before the timed region): a stream of `steps` batches
        through solve_seed_supergraphs -- per batch admission checks, int64
        -> int32 narrowing, H2D, solve, D2H of every label mask, CutResult
        construction; the host work of batch k+1 / k-1 overlaps the device
        solve of batch k -- wall clock from the first call to the last
        result, max over ranks.  e2e.single_call: one solve_seed_supergraph
        call per step (no overlap).
--impl reference : the reference solver's algorithm (oracle/, a C
        restatement of pmflow's push-relabel) on the host cores, same
        workload, a bounded sample per step, same metric.
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
POOL_IMAGES = 256            # C5: rng_seed 0..255
CONFIGS = {
    "c1": dict(w=160, h=120, rows=1, cols=1, types=("A",), lams="default", images=1,
               desc="C1: synthetic 160x120, 1 seed, DEFAULT 20-lambda ladder, one supergraph per step"),
    "c2": dict(w=500, h=375, rows=1, cols=1, types=("A",), lams="L20", images=1,
               desc="C2: synthetic 500x375 (VOC-sized), 1 seed, 20-lambda ladder L20, "
                    "one supergraph (20 lambda-graphs) per GPU per step"),
    "c3": dict(w=500, h=375, rows=5, cols=5, types=("A", "B"), lams="L20", images=1,
               desc="C3: one CPMC-style image per GPU per step -- synthetic 500x375, 25 seeds x "
                    "2 seed types x 20 lambdas = 1000 lambda-graphs in one device batch"),
    "c4": dict(w=1920, h=1080, rows=1, cols=1, types=("A",), lams="C4", images=1,
               desc="C4: synthetic 1920x1080, 1 seed, 8 lambdas per supergraph"),
    "c5": dict(w=500, h=375, rows=5, cols=5, types=("A", "B"), lams="L20", images=32,
               desc="C5: batch throughput over 256 distinct CPMC images (500x375, 25 seeds x 2 types "
                    "x 20 lambdas; rng_seed 0..255) in batches of 32 images claimed dynamically "
                    "(FIFO) by the GPUs; one batch per GPU per step"),
}
# CPU reference sample per step for the big configs (the full C3 image is
# ~3,400 CPU-s on the reference algorithm): the first problems' lambda graphs
REF_SAMPLE_PROBLEMS = {"c3": 1, "c5": 1, "c4": 1}
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


def reduce_max(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


class Claims:
    """Shared FIFO of batch ids: rank r takes the next id with one atomic
    add on the process group's store (torchrun), or a local counter."""

    KEY = "pmf_bench_claims"

    def __init__(self, shared: bool):
        self.store, self.k = None, 0
        if shared:
            import torch.distributed as dist
            self.store = dist.distributed_c10d._get_default_store()

    def next(self) -> int:
        if self.store is None:
            self.k += 1
            return self.k - 1
        return int(self.store.add(self.KEY, 1)) - 1


def mem_available() -> float:
    """Host MemAvailable in bytes (Linux), or a large default."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024.0
    except OSError:
        pass
    return 1e12


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
        self._stop.clear()   # re-entered for each timed region; rows accumulate
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




# ------------------------------------------------------------- workload

def batch_problems(cfg, b: int, sched):
    """Fresh SeedProblem objects of batch b (images b*k .. b*k + k - 1 of
    the pool, rng_seed = image index); generated on the host, untimed."""
    from paper_1509_06004_b200 import synth
    k = cfg["images"]
    probs = []
    for i in range(b * k, b * k + k):
        probs += synth.generate(cfg["w"], cfg["h"], cfg["rows"], cfg["cols"], rng_seed=i % POOL_IMAGES,
                                types=cfg["types"]).problems
    return probs


# ------------------------------------------------------------- CPU baseline

def cpu_solve(cfg, problems, threads):
    """The reference's solver (C restatement in oracle/) on every lambda graph
    of the given problems, per lambda as solve_schedule_sequential does;
    returns (n_cuts, seconds, flows)."""
    import oracle
    lams = lambdas_for(cfg["lams"])
    jobs = []
    for p in problems:
        for lam in lams:
            s, t, nb = oracle.instantiate(p.unary_base, p.unary_slope, p.sink_base, p.pairwise,
                                          p.fg_seeds, p.bg_seeds, lam)
            jobs.append((cfg["w"], cfg["h"], s, t, nb))
    t0 = time.perf_counter()
    res = oracle.solve_many(jobs, threads=threads)
    dt = time.perf_counter() - t0
    return len(jobs), dt, [r[0] for r in res]


def ref_sample(cfg, step: int):
    """Bounded CPU sample of one step: the problems of one seed supergraph
    (C1/C2/C4), or REF_SAMPLE_PROBLEMS of them, rotating through the pool."""
    from paper_1509_06004_b200 import synth
    img = step % POOL_IMAGES
    b = synth.generate(cfg["w"], cfg["h"], cfg["rows"], cfg["cols"], rng_seed=img, types=cfg["types"])
    mp = REF_SAMPLE_PROBLEMS.get(args_config(cfg))
    if mp is None:
        return b.problems, img
    k = (step * mp) % len(b.problems)
    return (b.problems + b.problems)[k:k + mp], img


def args_config(cfg):
    return next(k for k, v in CONFIGS.items() if v is cfg)


def run_reference(args, cfg):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import oracle
    oracle.build()
    threads = os.cpu_count() or 1
    for i in range(args.warmup):
        cpu_solve(cfg, ref_sample(cfg, i)[0], threads)
    tot_cuts, tot_s = 0, 0.0
    for i in range(args.steps):
        n, dt, _ = cpu_solve(cfg, ref_sample(cfg, args.warmup + i)[0], threads)
        tot_cuts += n
        tot_s += dt
    value = tot_cuts / tot_s
    mp = REF_SAMPLE_PROBLEMS.get(args.config)
    what = (f"the lambda-graphs of {mp} seed problem(s) of one pool image, rotating" if mp else
            "all lambda-graphs of one supergraph")
    sample = (f"{cfg['desc']}: {what} per step ({tot_cuts // args.steps} graphs), solved with the "
              f"reference push-relabel restated in C (oracle/pmflow_oracle.c), per lambda as "
              f"solve_schedule_sequential, {threads} host threads ({cpu_model()})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": {"workload": cfg["desc"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU arm

def roofline_of(stats, steps, config):
    """Roofline of the dominant kernel: the asynchronous solve kernel (one
    launch per step: every phase of every grid) or, step-synchronous, the
    push-relabel discharge k_push.  achieved = algorithmic bytes per launch
    (declared layout) / average launch time; the
    SURVEY section 8(d) canonical 64 B push / 24 B BFS pixel-pass figure and
    the layout-independent pixel-passes/s are reported beside it."""
    peak, peak_kind = measured_peaks()
    edge_bytes = stats[-1]["edge_bytes"]
    total_ms = sum(s["ms_device"] for s in stats)
    if stats[-1]["async_mode"]:
        col = 0 if edge_bytes == 4 else 1
        kern_ms = sum(s["ms_async"] for s in stats)
        alg = sum(s[k] * 1024 * v[col] for s in stats for k, v in ASYNC_BYTES.items())
        canon = sum(s["push_tile_passes"] * 1024 * 64 + (s["bfs_tile_passes"] + s["label_tile_passes"]) * 1024 * 24
                    for s in stats)
        pp = sum((s["push_tile_passes"] + s["bfs_tile_passes"] + s["label_tile_passes"]) * 1024 for s in stats)
        sec = kern_ms / 1e3 if kern_ms else float("inf")
        achieved = alg / sec / 1e9
        return {"bound": "hbm", "kernel": "k_async (asynchronous solve: relabel, discharge, labels, "
                                          "emit of every grid in one persistent launch)",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": committed_traffic("k_async", config), "peak_kind": peak_kind,
                "frac_canonical_64_24": canon / sec / 1e9 / peak,
                "pixel_passes_per_s": pp / sec,
                "bytes_per_pixel_pass": {k.replace("_tile_passes", ""): v[col] for k, v in ASYNC_BYTES.items()},
                "tile_passes_per_step": {k.replace("_tile_passes", ""): stats[-1][k] for k in ASYNC_BYTES},
                "avg_launch_us": kern_ms * 1e3 / steps,
                "time_share": {"k_async": round(kern_ms / total_ms, 4) if total_ms else None},
                "limiter": "latency / issue, not HBM: working set L2-resident (profiles/r02n_ncu_full.md: "
                           "k_async C3 DRAM 0.9 %, issue slots 42 %, barrier 58 % of stall samples, most of it idle CTAs "
                           "waiting for work in the single-image tail)"}
    push_ms = sum(s["ms_push"] for s in stats)
    launches = max(1, sum(s["push_sweeps"] for s in stats))
    passes = sum(s["push_tile_passes"] for s in stats)
    bpp = BYTES_PER_PIXEL_PASS[edge_bytes]
    sec = push_ms / 1e3 if push_ms else float("inf")
    achieved = passes * 1024 * bpp / launches / (sec / launches) / 1e9
    share = {k: round(sum(s[k] for s in stats) / total_ms, 4) for k in ("ms_push", "ms_bfs", "ms_labels")} \
        if total_ms else {}
    return {"bound": "hbm", "kernel": "k_push (push-relabel tile discharge)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": committed_traffic("k_push", config), "peak_kind": peak_kind,
            "frac_canonical_64_24": passes * 1024 * 64 / sec / 1e9 / peak,
            "bytes_per_pixel_pass": bpp, "pixel_passes_per_s": passes * 1024 / sec,
            "avg_launch_us": sec / launches * 1e6, "launches_per_step": launches / steps,
            "time_share": share,
            "limiter": "instruction issue, not HBM (profiles/r02n_ncu_full.md: k_push C5 issue slots 64 %, "
                       "IPC 2.6, DRAM 3.9 %, barrier 42 % of stall samples): up to 16 shared-memory "
                       "push-relabel iterations per pixel-pass"}


def measure(cfg, steps, warmup, dev, claims, sampler=None):
    """Run warmup + steps batches claimed from the shared FIFO; per step the
    e2e call on fresh problems (wall clock) and the device-resident run
    (CUDA events).  Returns the per-rank sums and the last batch's data."""
    import torch

    from paper_1509_06004_b200 import LambdaSchedule, _native, solve_seed_supergraph

    sched = LambdaSchedule(lambdas_for(cfg["lams"]))
    nbatch = POOL_IMAGES // cfg["images"]
    solver = _native.solver_for_thread(dev)
    stream = torch.cuda.ExternalStream(solver.stream_handle(), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = dict(dev_ms=0.0, e2e_s=0.0, h2d=0, d2h=0, cuts=0, stats=[], batches=[])

    def one(timed):
        b = claims.next() % nbatch
        probs = batch_problems(cfg, b, sched)
        # end to end through the public API, fresh objects (admission included)
        t0 = time.perf_counter()
        res = solve_seed_supergraph(probs, sched, "auto", device=dev)
        dt = time.perf_counter() - t0
        st_e2e = solver.stats()
        # device-resident: stage (untimed), L2 flush, timed run
        solver.seed_stage(cfg["w"], cfg["h"], probs, sched.values, "auto")
        with torch.cuda.stream(stream):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        solver.seed_run()
        with torch.cuda.stream(stream):
            e1.record(stream)
        e1.synchronize()
        st = solver.stats()
        _, flows, _ = solver.seed_fetch(labels=False)
        assert [c.flow for c in res.cuts] == [int(f) for f in flows.reshape(-1)], "e2e and device runs disagree"
        if timed:
            out["dev_ms"] += e0.elapsed_time(e1)
            out["e2e_s"] += dt
            out["h2d"] += st_e2e["h2d_bytes"]
            out["d2h"] += st_e2e["d2h_bytes"]
            out["cuts"] += len(res.cuts)
            out["stats"].append(st)
            out["batches"].append(b)
            out["last"] = (probs, flows)

    for _ in range(warmup):
        one(False)
    barrier()
    torch.cuda.synchronize()
    if sampler is not None:
        with sampler:
            for _ in range(steps):
                one(True)
    else:
        for _ in range(steps):
            one(True)
    torch.cuda.synchronize()
    barrier()
    return out


def measure_stream(cfg, steps, warmup, dev, claims, sampler=None, ids=None):
    """e2e leg: `steps` fresh batches -- the batch ids the device-resident
    loop of this rank solved (`ids`, so both legs do the same work), else
    claimed from the shared FIFO; problems generated before the timed
    region -- through the public batch stream
    solve_seed_supergraphs -- per batch: admission, narrowing, H2D, solve,
    D2H of every label mask, CutResults -- wall clock from the first call
    to the last result, stager / runner / fetch of neighbouring batches
    overlapped.  A warm-up stream of `warmup` batches (>= 2) runs first."""
    from paper_1509_06004_b200 import LambdaSchedule, _native, solve_seed_supergraphs

    sched = LambdaSchedule(lambdas_for(cfg["lams"]))
    nbatch = POOL_IMAGES // cfg["images"]

    def batches(n, given=None):
        got = list(given) if given is not None else [claims.next() % nbatch for _ in range(n)]
        return got, [batch_problems(cfg, b, sched) for b in got]

    _, warm = batches(max(2, warmup))
    for _ in solve_seed_supergraphs(warm, sched, "auto", device=dev):
        pass
    del warm
    # host memory: the timed batches are generated up front (~120 MB of
    # int64 planes per CPMC image); ranks sharing the node split 40 % of the
    # available memory (with 8 ranks on a small node the stream is shorter)
    per_batch = 0.125e9 * cfg["images"]
    budget = 0.4 * mem_available() / int(os.environ.get("LOCAL_WORLD_SIZE", 1))
    n = max(2, min(steps, int(budget // (2 * per_batch))))
    ids, todo = batches(n, ids[:n] if ids is not None else None)
    barrier()
    cuts = 0
    ctx = sampler if sampler is not None else _Null()
    with ctx:
        t0 = time.perf_counter()
        for res in solve_seed_supergraphs(todo, sched, "auto", device=dev):
            cuts += len(res.cuts)
            del res
        dt = time.perf_counter() - t0
    barrier()
    st = _native.pipeline_solvers(dev, 1)[0].stats()   # the last stream's solver: same shape as every batch
    return dict(e2e_s=dt, cuts=cuts, h2d=st["h2d_bytes"], d2h=st["d2h_bytes"], batches=ids, steps=len(ids))


def measure_stream_synth(cfg, steps, warmup, dev, ids):
    """Harness path with on-device synthesis (synth_device): per batch the
    host draws the images from their rng seeds (the reference generator's
    stream, inside the timed region, on the stager thread), the device
    derives every plane, solves, and the host receives every flow and label
    mask -- generate_batch + solve + split of harness/bench.py:79-120."""
    from paper_1509_06004_b200 import LambdaSchedule, solve_seed_supergraphs
    from paper_1509_06004_b200.synth_device import generate_images

    sched = LambdaSchedule(lambdas_for(cfg["lams"]))
    k = cfg["images"]

    def gen(bids):
        for b in bids:
            yield generate_images(cfg["w"], cfg["h"], cfg["rows"], cfg["cols"],
                                  [(b * k + i) % POOL_IMAGES for i in range(k)], cfg["types"])

    for _ in solve_seed_supergraphs(gen(ids[:max(2, warmup)]), sched, "auto", device=dev):
        pass
    barrier()
    cuts = 0
    t0 = time.perf_counter()
    for res in solve_seed_supergraphs(gen(ids), sched, "auto", device=dev):
        cuts += len(res.cuts)
        del res
    dt = time.perf_counter() - t0
    barrier()
    return dict(e2e_s=dt, cuts=cuts)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def c2_per_lambda(dev):
    """Critical path of C2 (one supergraph, 20 cold lambda-graphs solved in
    parallel by the asynchronous solver): per lambda-graph the exact global
    relabels and discharge phases it needed and when it finished (device
    phase log of one untimed solve of pool image 0)."""
    from paper_1509_06004_b200 import LambdaSchedule, _native
    cfg = CONFIGS["c2"]
    sched = LambdaSchedule(lambdas_for(cfg["lams"]))
    s = _native.Solver(dev, phase_log=1)
    try:
        s.solve_seed_batch(cfg["w"], cfg["h"], batch_problems(cfg, 0, sched), sched.values, "auto")
        out = []
        for g, lam in enumerate(sched.values):
            ph = s.phases(g)
            out.append({"lambda": int(lam), "global_relabels": sum(1 for n, _ in ph if n == "bfs"),
                        "discharges": sum(1 for n, _ in ph if n == "push"), "finish_us": ph[-1][1]})
        return {"device_ms": round(s.stats()["ms_device"], 3), "image": 0, "lambdas": out}
    finally:
        s.close()


def run_b200(args, cfg):
    import torch
    import torch.distributed as dist

    rank, local, world = dist_env()
    ndev = torch.cuda.device_count()
    dev = local % ndev          # one GPU per rank (shared only when testing N > #GPUs)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("gloo")   # plumbing only: claims, barriers, max-reduce
    clk = ClockSampler(dev)
    claims = Claims(world > 1)
    m = measure(cfg, args.steps, args.warmup, dev, claims, clk)
    sm = measure_stream(cfg, args.steps, args.warmup, dev, claims, clk, ids=m["batches"])
    sy = measure_stream_synth(cfg, args.steps, args.warmup, dev, m["batches"])
    synth_s_max = reduce_max(sy["e2e_s"])
    synth_cuts_all = int(reduce_sum(sy["cuts"]))
    dev_s_max = reduce_max(m["dev_ms"] / 1e3)
    single_s_max = reduce_max(m["e2e_s"])
    e2e_s_max = reduce_max(sm["e2e_s"])
    cuts_all = int(reduce_sum(m["cuts"]))
    stream_cuts_all = int(reduce_sum(sm["cuts"]))
    value = cuts_all / dev_s_max
    e2e_value = stream_cuts_all / e2e_s_max
    stats = m["stats"]
    nimg = cfg["images"]

    # ---- CPU baseline (rank 0, N == 1 only): the oracle on a bounded
    # sample of the last timed batch, checked against the device flows
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        threads = os.cpu_count() or 1
        probs, flows = m["last"]
        mp = REF_SAMPLE_PROBLEMS.get(args.config) or len(probs)
        n, dt, fl = cpu_solve(cfg, probs[:mp], threads)
        assert fl == [int(f) for f in flows[:mp].reshape(-1)], "oracle and engine disagree"
        cpu = {"value": n / dt, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"{n} lambda-graphs ({mp} seed problem(s) of the last timed batch, "
                         f"{cfg['desc'].split(':')[0]}), reference push-relabel restated in C "
                         f"(oracle/pmflow_oracle.c), per lambda, {threads} threads; took {dt:.2f} s"}

    # ---- secondary workloads (N == 1): C3 (ms per CPMC image) and C2
    secondary = None
    if rank == 0 and world == 1 and args.secondary and args.config == "c5":
        secondary = {}
        for name, st_, wu in (("c3", 5, 3), ("c2", 10, 3)):
            c = CONFIGS[name]
            cl = Claims(False)
            s2 = measure(c, st_, wu, dev, cl)
            ss = measure_stream(c, st_, wu, dev, cl, ids=s2["batches"])
            k = s2["cuts"]
            secondary[name] = {
                "workload": c["desc"], "steps": st_, "value": k / (s2["dev_ms"] / 1e3), "unit": UNIT,
                "ms_per_image": s2["dev_ms"] / st_ / c["images"],
                "e2e": {"value": ss["cuts"] / ss["e2e_s"],
                        "ms_per_image": 1e3 * ss["e2e_s"] / ss["steps"] / c["images"],
                        "h2d_bytes_per_step": ss["h2d"], "d2h_bytes_per_step": ss["d2h"],
                        "api": "solve_seed_supergraphs (batch stream)",
                        "single_call": {"value": k / s2["e2e_s"],
                                        "ms_per_image": 1e3 * s2["e2e_s"] / st_ / c["images"]}},
                "roofline": roofline_of(s2["stats"], st_, name)}
        secondary["c2"]["per_lambda"] = c2_per_lambda(dev)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dev_s_max / args.steps,
            "ms_per_image": 1e3 * dev_s_max / args.steps / nimg,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": cfg["desc"], "images_per_step_per_gpu": nimg,
                       "lambda_cuts_per_step_per_gpu": cuts_all // world // args.steps,
                       "image": f"{cfg['w']}x{cfg['h']}",
                       "pool": f"{POOL_IMAGES} distinct images (rng_seed 0..{POOL_IMAGES - 1}), "
                               f"batches of {nimg} claimed FIFO across ranks",
                       "l2": "flushed between steps (256 MiB memset, outside the timed events); "
                             "each step also stages a new batch",
                       "parallelism": f"{world} GPU(s), one process each, dynamic batch claims "
                                      "(store counter), no data-path collective, gloo plumbing"},
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_image": 1e3 * e2e_s_max / sm["steps"] / nimg,
                    "steps": sm["steps"],
                    "h2d_bytes_per_step": sm["h2d"], "d2h_bytes_per_step": sm["d2h"],
                    "api": "solve_seed_supergraphs (batch stream: staging of batch k+1 and the fetch of "
                           "batch k-1 overlap the solve of batch k; fresh problems of the device loop's "
                           "batches, generated untimed)",
                    "synthetic_path": {
                        "value": synth_cuts_all / synth_s_max,
                        "ms_per_image": 1e3 * synth_s_max / args.steps / nimg,
                        "api": "solve_seed_supergraphs over synth_device.ImageBatch: images drawn from "
                               "their rng seeds on the host inside the timed region, planes derived on "
                               "the device (pmf_synth_stage), every flow and label mask to the host"},
                    "single_call": {"value": cuts_all / single_s_max,
                                    "ms_per_image": 1e3 * single_s_max / args.steps / nimg,
                                    "api": "solve_seed_supergraph, one batch per call",
                                    "h2d_bytes_per_step": m["h2d"] // args.steps,
                                    "d2h_bytes_per_step": m["d2h"] // args.steps}},
            "roofline": roofline_of(stats, args.steps, args.config),
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": int(sum(s["kernels"] for s in stats)),
            "solver": {k: stats[-1][k] for k in ("async_mode", "cycles", "steps", "push_sweeps",
                                                  "push_tile_passes", "bfs_sweeps", "bfs_tile_passes",
                                                  "label_tile_passes", "scan_tile_passes", "tiles",
                                                  "edge_bytes", "grids")},
            "batches_rank0": m["batches"],

            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def reduce_sum(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", dest="secondary", action="store_false")
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
