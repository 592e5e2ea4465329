"""One deterministic epoch of a config under ncu (launch list): which class launches dominate.
  ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/det_profile.py vc_chunglu_10m"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1311_2661_b200 as th  # noqa: E402

cfg = inputs.CONFIGS[sys.argv[1]]
g = inputs.make_graph(cfg)
lp = th.LP.from_graph(cfg.problem, g.n, g.src, g.dst, vertex_w=g.vertex_w, device="cuda:0")
lp.solve(cfg.beta, 1, mode=0, seed=cfg.solve_seed)  # colouring + graph capture
st = lp.solve(cfg.beta, 2, mode=0, seed=cfg.solve_seed)
print("det ms per epoch", st["ms_per_epoch"], "classes", st["n_colours"])
