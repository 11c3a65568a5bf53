"""Async busy breakdown per pass kind for one config (CTA-summed us per pass)."""
import json, os, subprocess, sys
cfg = sys.argv[1]
args = sys.argv[2:]
out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "probe.py"), cfg, "--reps", "2", *args],
                     capture_output=True, text=True).stdout.splitlines()
busy = [l for l in out if l.startswith("busy")][-1]
b = eval(busy[busy.index("{"):busy.index("}") + 1])
d = json.loads([l for l in out if l.startswith("{")][-1])
per = lambda k, n: round(1e3 * b[k] / max(1, d[n]), 2)
print(cfg, " ".join(args), "dev", d["med_dev_ms"], "| us/pass push", per("push", "push_tile_passes"),
      "bfs", per("bfs", "bfs_tile_passes"), "lab", per("lab", "label_tile_passes"),
      "| CTA-ms push", b["push"], "bfs", b["bfs"], "lab", b["lab"], "scan", round(b["binit"] + b["seed"] + b["linit"] + b["emit"], 1),
      "handoff", b["handoff"], "wait", b["wait"], "trans", b["transition"],
      "| iters/push pass", round(b.get("push_iterations", 0) / max(1, d["push_tile_passes"]), 2),
      "relax us/call", round(1e3 * b.get("relax_ms", 0) / max(1, b.get("relax_calls", 0)), 2),
      "relax calls/pass", round(b.get("relax_calls", 0) / max(1, d["push_tile_passes"]), 2),
      "sweeps/relax", round(b.get("relax_sweeps", 0) / max(1, b.get("relax_calls", 0)), 2),
      "| spec", b.get("spec_tries"), "spoiled", b.get("spec_spoiled"))
