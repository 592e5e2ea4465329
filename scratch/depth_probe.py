import sys, os, numpy as np
sys.path.insert(0,'.')
import paper_1311_2661_b200 as th
from tests.test_parity_gpu import async_cases, build_case
for name in ('vc_hubs', 'mwc_grid40'):
    c = async_cases()[name]
    g = build_case(th, c)
    g.solve(10.0, c['epochs'], mode=1, seed=71)
    o = g.objective(10.0)
    print(os.environ.get('THETIS_ASYNC_MAX_BLOCKS'), name, o['f_beta'], o['lp_obj'], flush=True)
