import os, sys, numpy as np
sys.path.insert(0, '.')
import paper_1311_2661_b200 as th, inputs
from oracle import RefLP
from tests.test_parity_gpu import rand_graph, grid
def run(problem, n, src, dst, vw=None, ew=None, k=0, terms=None, t=0, epochs=20, rule=0):
    g = th.LP.from_graph(problem, n, src, dst, vertex_w=vw, edge_w=ew, k=k, terminals=terms, t_per_label=t)
    g.solve(10.0, epochs, mode=1, seed=71, step_rule=rule)
    o = g.objective(10.0); x = g.get_x().cpu().numpy()
    out = [os.environ.get('THETIS_ASYNC_SERIAL','0'), problem, round(o['f_beta'],4)]
    for mode in (1, 3):
        r = RefLP.graph(problem, n, src, dst, vertex_w=vw, edge_w=ew, k=k, terminals=terms, t_per_label=t, bits=64)
        r.solve(10.0, epochs, mode=mode, seed=71, step_rule=rule)
        ro = r.objective(10.0)
        out += [mode, round(ro['f_beta'],4), float(np.abs(x - r.x()).max())]
    print(*out, flush=True)
cfg = inputs.CONFIGS['vc_er_1k']; gi = inputs.make_graph(cfg)
run(1, gi.n, gi.src, gi.dst, vw=gi.vertex_w)
run(2, gi.n, gi.src, gi.dst, vw=gi.vertex_w)
src, dst = grid(40); ew = np.random.default_rng(5).exponential(1.0, len(src)).astype(np.float32)
run(3, 1600, src, dst, ew=ew, k=5, terms=inputs.terminals(1600, 25, 6), t=5, epochs=30)
rng = np.random.default_rng(2); n = 20000
src = np.concatenate([rng.integers(0, 64, 60000), rng.integers(0, n, 40000)]).astype(np.int32)
dst = np.concatenate([rng.integers(0, n, 60000), rng.integers(0, n, 40000)]).astype(np.int32)
run(1, n, src, dst, vw=rng.uniform(1, 10, n).astype(np.float32), epochs=15)
