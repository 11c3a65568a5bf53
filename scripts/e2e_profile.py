"""cProfile of one public-API seed supergraph call (host side of e2e)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_06004_b200 import LambdaSchedule, solve_seed_supergraph, synth
imgs = int(sys.argv[1]) if len(sys.argv) > 1 else 8
probs = []
for i in range(imgs):
    probs += synth.generate(500, 375, 5, 5, rng_seed=i, types=("A", "B")).problems
sched = LambdaSchedule(synth.L20)
for _ in range(3):
    res = solve_seed_supergraph(probs, sched, "auto")
t = time.perf_counter(); res = solve_seed_supergraph(probs, sched, "auto"); print("wall ms", 1e3 * (time.perf_counter() - t))
pr = cProfile.Profile(); pr.enable(); res = solve_seed_supergraph(probs, sched, "auto"); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
