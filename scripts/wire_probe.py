"""Wire worker step on the C2 composite (500x375 problem, L20 ladder joined
into one 10,019x375 request): serve_payload (int32 planes in place) vs the
reference worker's steps on the engine (decode_request -> int64 GridGraph,
gpu_solve_fn, encode_response).  Wall ms per request, median of --reps."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1509_06004_b200 import synth, wire
from paper_1509_06004_b200.parametric import LambdaSchedule
from paper_1509_06004_b200.supergraph import build_lambda_supergraph, family_swap_decision

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=7)
a = ap.parse_args()
p = synth.generate(500, 375, 1, 1, rng_seed=0).problems[0]
sched = LambdaSchedule(synth.L20)
comp, layout, _ = build_lambda_supergraph(p, sched, family_swap_decision(p, sched))
payload = wire.encode_request(wire.WireRequest(9, comp, layout))


def ref_steps(pl):
    req = wire.decode_request(pl)
    cut = wire.gpu_solve_fn(req.graph, req.layout)
    return wire.encode_response(wire.WireResponse(req.task_id, wire.Status.OK, cut.flow, cut.labels))


out = {"request_bytes": len(payload), "pixels": comp.n}
for name, fn in (("serve_payload", wire.serve_payload), ("decode_request+gpu_solve_fn", ref_steps)):
    fn(payload)
    ts = []
    for _ in range(a.reps):
        t = time.perf_counter()
        r = fn(payload)
        ts.append(1e3 * (time.perf_counter() - t))
    out[name + "_ms"] = round(float(np.median(ts)), 2)
    out[name + "_flow"] = wire.decode_response(r, comp.n).flow
print(json.dumps(out))
