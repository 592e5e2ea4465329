import numpy as np, sys
sys.path.insert(0,'.')
import inputs
from oracle import RefLP
from tests.test_parity_gpu import grid
def spread(name, problem, n, src, dst, vw=None, ew=None, k=0, terms=None, t=0, epochs=20):
    fs=[]; ls=[]
    for seed in (71,72,73,74,75):
        r = RefLP.graph(problem, n, src, dst, vertex_w=vw, edge_w=ew, k=k, terminals=terms, t_per_label=t)
        r.solve(10.0, epochs, mode=1, seed=seed); o = r.objective(10.0); fs.append(o['f_beta']); ls.append(o['lp_obj'])
    fs=np.array(fs); ls=np.array(ls)
    print(name, 'f rel spread', (fs.max()-fs.min())/abs(fs.mean()), 'lp rel spread', (ls.max()-ls.min())/abs(ls.mean()))
src, dst = grid(40); ew = np.random.default_rng(5).exponential(1.0, len(src)).astype(np.float32)
spread('mwc40', 3, 1600, src, dst, ew=ew, k=5, terms=inputs.terminals(1600, 25, 6), t=5, epochs=30)
rng = np.random.default_rng(2); n = 20000
src = np.concatenate([rng.integers(0, 64, 60000), rng.integers(0, n, 40000)]).astype(np.int32)
dst = np.concatenate([rng.integers(0, n, 60000), rng.integers(0, n, 40000)]).astype(np.int32)
spread('hubs', 1, n, src, dst, vw=rng.uniform(1, 10, n).astype(np.float32), epochs=15)
cfg = inputs.CONFIGS['vc_er_1k']; gi = inputs.make_graph(cfg)
spread('cfg1-vc', 1, gi.n, gi.src, gi.dst, vw=gi.vertex_w)
spread('cfg1-mis', 2, gi.n, gi.src, gi.dst, vw=gi.vertex_w)
