import numpy as np, sys, time
sys.path.insert(0,'.')
import inputs, oracle
s=18
src, dst = inputs.rmat(s, 16 << s, 0.57, 0.19, 0.19, 13115)
w = inputs.uniform_weights(1 << s, 26615)
for mode in (1, 3, 0):
    for rule in (0, 1):
        lp = oracle.RefLP.graph(1, 1 << s, src, dst, vertex_w=w)
        t=time.time(); lp.solve(10.0, 20, mode=mode, seed=75, step_rule=rule); o = lp.objective(10.0)
        print('mode', mode, 'rule', rule, 'f', round(o['f_beta'],1), 'lp', round(o['lp_obj'],1), 'eps', round(o['max_violation_eps'],4), round(time.time()-t,1),'s', flush=True)
