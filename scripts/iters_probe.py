import sys; sys.path.insert(0,'.')
from paper_1509_06004_b200 import _native, synth
for imgs in (8, 1):
    probs=[]
    for i in range(imgs): probs+=synth.generate(500,375,5,5,rng_seed=i,types=('A','B')).problems
    s=_native.Solver(0)
    for r in range(2): s.solve_seed_batch(500,375,probs,synth.L20,'auto')
    st=s.stats(); b=s.busy()
    print(imgs, 'push passes', st['push_tile_passes'], 'iters', b['push_iterations'], 'iters/pass', round(b['push_iterations']/st['push_tile_passes'],2),
          'relax calls', b['relax_calls'], 'sweeps', b['relax_sweeps'], 'relax ms(sum)', b['relax_ms'], 'ms', st['ms_device'])
