import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1311_2661_b200 as th
np.set_printoptions(linewidth=200, precision=5)
n=40
for prob in (1,2):
  g = th.LP.from_graph(prob, n, np.arange(n-1, dtype=np.int32), np.arange(1,n, dtype=np.int32), vertex_w=np.ones(n, np.float32))
  print('r0', g.get_r().cpu().numpy()[:5])
  g.solve(10.0, 1, mode=1, seed=3)
  z = g.get_x().cpu().numpy(); r = g.get_r().cpu().numpy()
  sig = -1 if prob==1 else 1
  rr = z[:n-1] + z[1:n] + sig*z[n:] - 1
  print('x', z[:n]); print('s', z[n:]); print('r', r); print('rr', rr)
