import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1509_06004_b200 import synth, wire, _native
from paper_1509_06004_b200.parametric import LambdaSchedule
from paper_1509_06004_b200.supergraph import build_lambda_supergraph, family_swap_decision
p = synth.generate(500, 375, 1, 1, rng_seed=0).problems[0]
sched = LambdaSchedule(synth.L20)
comp, layout, _ = build_lambda_supergraph(p, sched, family_swap_decision(p, sched))
payload = wire.encode_request(wire.WireRequest(9, comp, layout))
s = _native.solver_for_thread(0)
for r in range(5):
    t = time.perf_counter(); wire.serve_payload(payload); dt = time.perf_counter() - t
    st = s.stats()
    print(json.dumps({"wall_ms": round(1e3*dt, 2), "device_ms": round(st["ms_device"], 3), "async": st["async_mode"], "cycles": st["cycles"], "push": st["push_tile_passes"], "bfs": st["bfs_tile_passes"]}))
# seed path for the same problem
for r in range(3):
    s.solve_seed_batch(500, 375, [p], sched.values, "auto")
    print("seed path device ms", round(s.stats()["ms_device"], 3), "async", s.stats()["async_mode"])
