"""Diagnose intermittent label mismatches: repeat C1 solves per mode and
check the residual-pair invariant r(p->q) + r(q->p) == c(p->q) + c(q->p)
on the downloaded device state."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_synth
from paper_1509_06004_b200 import _native, synth

g = load_synth("c1_160x120.npz")
probs = synth.generate(160, 120, rng_seed=0).problems
p = probs[0]
W, H = 160, 120
ntx, nty = 5, 4
pw = p.pairwise.reshape(4, H, W)

def untile(a):
    # tile-major (G, nty, ntx, 32, 32) -> (G, H, W)
    G = a.shape[0] // (ntx * nty * 1024)
    t = a.reshape(G, nty, ntx, 32, 32).transpose(0, 1, 3, 2, 4).reshape(G, nty * 32, ntx * 32)
    return t[:, :H, :W]

def closure(wg, lanes, j):
    """host BFS from excess pixels along residual arcs (grid j)"""
    from collections import deque
    reach = wg[j] > 0
    q = deque(zip(*np.nonzero(reach)))
    dirs = ((0, 0, -1), (1, 0, 1), (2, -1, 0), (3, 1, 0))
    while q:
        y, x = q.popleft()
        for d, dy, dx in dirs:
            if lanes[d][j, y, x] > 0:
                yy, xx = y + dy, x + dx
                if 0 <= yy < H and 0 <= xx < W and not reach[yy, xx]:
                    reach[yy, xx] = True
                    q.append((yy, xx))
    return reach

def check(s, bad):
    w, h, r, lab = s.debug_state()
    wg = untile(w.astype(np.int64))
    labg = untile(lab)
    r0 = r.astype(np.int64)
    lanes = [untile((r0 >> (8 * d)) & 0xff) for d in range(4)]
    for (j, _, _) in bad:
        lam = g["lambdas"][j]
        src = (p.unary_base + lam * p.unary_slope).copy(); src[p._fg_idx] = 1 << 30
        snk = p.sink_base.copy(); snk[p._bg_idx] = 1 << 30
        t = (src - snk).reshape(H, W)
        out = sum(pw[d] - lanes[d][j] for d in range(4))
        exc_bad = int((wg[j] != t - out).sum())
        cl = closure(wg, lanes, j).reshape(-1)
        gold = g["labels"][j].astype(bool)
        print("   grid", j, "excess-invariant violations", exc_bad, "host-closure vs gold diff", int((cl != gold).sum()),
              "device lab vs host closure diff", int((labg[j].reshape(-1).astype(bool) != cl).sum()),
              "n excess px", int((wg[j] > 0).sum()), "alive excess (h<INF)", int(((wg[j] > 0) & (untile(h)[j] < 0x3fffffff)).sum()))
    r = r.astype(np.int64)
    lanes = [untile((r >> (8 * d)) & 0xff) for d in range(4)]
    bad = 0
    # horizontal pairs: R(p) + L(p+1) == pw_R(p) + pw_L(p+1)
    hs = lanes[1][:, :, :-1] + lanes[0][:, :, 1:]
    hc = pw[1][:, :-1] + pw[0][:, 1:]
    vs = lanes[3][:, :-1, :] + lanes[2][:, 1:, :]
    vc = pw[3][:-1, :] + pw[2][1:, :]
    return int((hs != hc[None]).sum()), int((vs != vc[None]).sum()), int((lanes[0][:, :, 0] != 0).sum())

for persistent in (1, 0):
    s = _native.Solver(0, persistent=persistent)
    fails = 0
    for rep in range(25):
        sw, flows, labels = s.solve_seed_batch(W, H, probs, g["lambdas"], "auto")
        bad = [(j, int(flows[0][j]) - g["flows"][j], int((labels[0][j] != g["labels"][j]).sum()))
               for j in range(20) if flows[0][j] != g["flows"][j] or not np.array_equal(labels[0][j], g["labels"][j])]
        inv = (0,)
        if bad:
            check(s, bad)
        if bad or any(inv):
            fails += 1
            print("persistent", persistent, "rep", rep, "mismatch", bad, "pair-invariant violations (h, v, border)", inv)
    print("persistent", persistent, "fails", fails, "/ 25")
