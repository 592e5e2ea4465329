#!/usr/bin/env python
"""Can the hub-lag variant's synchronous hub step be repaired by grouping?  (TEST INFRASTRUCTURE:
runs the oracle.)  After a slack-first sweep the hub vertices are split into G groups; the
groups step one after the other (Gauss-Seidel across groups), synchronously inside a group
(Jacobi), then the light tiles in the permuted order -- tests/experiments/sched_variants.c
exp_groups.  Prints the deviation of f_beta, c^T x and the rounded cover from Alg. 1's
permuted sweep (oracle MODE_ASYNC) on the config-5 recipe at a reduced R-MAT scale, 1/L_max.

  python tests/experiments/grouped_hubs.py [scale]      (results: profiles/r02_grouped_hubs.txt)
"""
import ctypes, os, sys, time
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE))); sys.path.insert(0, HERE)
import numpy as np
import inputs, oracle
import schedule_sensitivity as ss
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 18
cfg = inputs.CONFIGS["vc_rmat_26"]
g = inputs.make_graph(cfg, scale=scale, samples=16 << scale)
L = ss.lib()
L.exp_groups.argtypes = [ctypes.c_void_p, ctypes.c_float, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
beta, ep, seed = cfg.beta, cfg.epochs, cfg.solve_seed
def fresh():
    h = ctypes.c_void_p()
    src, dst = np.ascontiguousarray(g.src, np.int32), np.ascontiguousarray(g.dst, np.int32)
    vw = np.ascontiguousarray(g.vertex_w, np.float32)
    rc = L.thetis_ref_build_graph_lp(ctypes.byref(h), 1, g.n, len(src), src.ctypes.data, dst.ctypes.data, vw.ctypes.data, None, 0, None, 0)
    assert rc == 0
    return oracle.RefLP(h, L, 64, None)
def res(lp):
    o = lp.objective(beta); _, rr = lp.round(oracle.ROUND_VC_HALF)
    return o["f_beta"], o["lp_obj"], rr["cost"]
lp = fresh()
n = g.n
deg = np.diff(np.asarray(lp.colptr()[: n + 1])) if hasattr(lp, "colptr") else None
if deg is None:
    # degrees from the unique edge list
    e = lp.edges() if hasattr(lp, "edges") else None
print("n", n, "U", lp.U)
rule = oracle.STEP_LMAX
lp.solve(beta, ep, mode=oracle.MODE_ASYNC, seed=seed, step_rule=rule)
base = res(lp)
print("base", base)
def run(name, grp, G, permute=1, jac=1):
    lp = fresh(); grp = np.ascontiguousarray(grp, np.int32)
    t = time.time(); L.exp_groups(lp._h, beta, ep, seed, rule, grp.ctypes.data, G, permute, jac)
    v = res(lp); d = [(v[i] - base[i]) / abs(base[i]) for i in range(3)]
    print(f"{name:60s} {d[0]:+10.2e} {d[1]:+10.2e} {d[2]:+10.2e}  ({time.time()-t:.1f}s)", flush=True)
# tile degrees
u_ = np.minimum(g.src, g.dst); v_ = np.maximum(g.src, g.dst); keep = u_ != v_
key = np.unique(u_[keep].astype(np.int64) * n + v_[keep])
uu, vv = key // n, key % n
deg = np.bincount(uu, minlength=n) + np.bincount(vv, minlength=n)
nt = (n + 31) // 32
tdeg = np.add.reduceat(np.pad(deg, (0, nt * 32 - n)), np.arange(0, nt * 32, 32))
hubtile = tdeg > 512
hub = np.repeat(hubtile, 32)[:n]
print("hub vertices", hub.sum(), "hub nnz frac", deg[hub].sum() / deg.sum(), "max deg", deg.max())
def h32(x):
    x = x.astype(np.uint64); x = (x ^ (x >> 16)) * 0x85EBCA6B & 0xFFFFFFFF; x = (x ^ (x >> 13)) * 0xC2B2AE35 & 0xFFFFFFFF; return x ^ (x >> 16)
tile = np.arange(n) // 32
for G in (1, 2, 4, 8, 16, 32):
    grp = np.where(hub, (h32(tile) % G).astype(np.int64), -1)
    run(f"hub tiles hashed into {G} groups, Jacobi in group", grp, G)
grp = np.where(hub, (h32(tile) % 16).astype(np.int64), -1)
run("16 groups, sequential in group (the order itself)", grp, 16, jac=0)
# all structural units grouped (no light sweep)
for G in (8, 16):
    run(f"ALL tiles hashed into {G} groups, Jacobi", (h32(tile) % G).astype(np.int64), G)
# degree-threshold: top vertices in G-1 hashed groups, the rest of hubs in the last group
for T in (64, 256, 1024):
    for G in (8, 16):
        top = deg > T
        grp = np.where(top, (h32(np.arange(n)) % (G - 1)).astype(np.int64), np.where(hub, G - 1, -1))
        lp_ = None
        run(f"deg>{T} vertices ({top.sum()}) in {G-1} groups, other hubs last group; fixed order", grp, G, permute=0)
