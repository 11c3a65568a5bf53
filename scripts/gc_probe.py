import gc, time, sys, os
sys.path.insert(0, os.getcwd())
import bench
gt = {"n": 0, "t": 0.0, "gen2": 0}
t0 = [0.0]
def cb(phase, info):
    if phase == "start":
        t0[0] = time.perf_counter()
    else:
        gt["n"] += 1
        gt["t"] += time.perf_counter() - t0[0]
        if info["generation"] == 2:
            gt["gen2"] += 1
gc.callbacks.append(cb)
cfg = bench.CONFIGS["c5"]
claims = bench.Claims(False)
m = bench.measure(cfg, 10, 3, 0, claims)
gt.update(n=0, t=0.0, gen2=0)
sm = bench.measure_stream(cfg, 10, 3, 0, claims, ids=m["batches"])
print("stream ms/image", 1e3 * sm["e2e_s"] / 160, "gc", gt)
gt.update(n=0, t=0.0, gen2=0)
gc.freeze()
sm = bench.measure_stream(cfg, 10, 3, 0, claims, ids=m["batches"])
print("after freeze: stream ms/image", 1e3 * sm["e2e_s"] / 160, "gc", gt)
