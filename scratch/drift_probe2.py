import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1311_2661_b200 as th
for prob in (2,):
    g = th.LP.from_graph(prob, 2, np.array([0], np.int32), np.array([1], np.int32), vertex_w=np.ones(2, np.float32))
    print('U', g.U, 'N', g.N)
    for e in range(4):
        g.solve(10.0, 1, mode=1, seed=3)
        z = g.get_x().cpu().numpy(); r = g.get_r().cpu().numpy()
        print(e, z, r, 'expected r', z[0]+z[1]+z[2]-1)
    # 40 vertices path
    n=40
    g = th.LP.from_graph(prob, n, np.arange(n-1, dtype=np.int32), np.arange(1,n, dtype=np.int32), vertex_w=np.ones(n, np.float32))
    g.solve(10.0, 1, mode=1, seed=3)
    z = g.get_x().cpu().numpy(); r = g.get_r().cpu().numpy()
    rr = z[:n-1] + z[1:n] + z[n:] - 1
    print('path', np.abs(r-rr).max(), (r-rr)[:8], z[n:n+8])
