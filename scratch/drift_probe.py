import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1311_2661_b200 as th
from tests.test_parity_gpu import rand_graph
src, dst = rand_graph(800, 4000, 3)
vw = np.random.default_rng(2).uniform(1, 10, 800).astype(np.float32)
for prob in (1, 2):
    for mode in (0, 1):
        g = th.LP.from_graph(prob, 800, src, dst, vertex_w=vw)
        for e in range(5):
            g.solve(10.0, 1, mode=mode, seed=3)
            o = g.objective(10.0)
            z = g.get_x().cpu().numpy().astype(np.float64); r = g.get_r().cpu().numpy()
            eu, ev = g.edges()
            n = 800; m = g.m
            sig = -1 if prob == 1 else 1
            rr = z[eu] + z[ev] + sig * z[n:n+m] - 1
            bad = np.nonzero(np.abs(rr - r) > 1e-4)[0]
            print(prob, mode, e, o['drift_inf'], len(bad), bad[:5], (r-rr)[bad[:5]], z[n+bad[:5]])
