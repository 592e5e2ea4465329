"""Distinct 32-byte sectors of r per structural nonzero that a column-by-column sweep (Alg. 1's
order: each column gathers and scatters its rows) touches, under the R-17 row layout and three
alternatives, on the config-5 recipe at a reduced R-MAT scale.  TEST INFRASTRUCTURE (builds the
LP with the oracle).  python tests/experiments/layout_sectors.py 22
"""
import sys, numpy as np, time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import inputs, oracle
sc = int(sys.argv[1])
cfg = inputs.CONFIGS["vc_rmat_26"]
g = inputs.make_graph(cfg, scale=sc, samples=16 << sc)
t = time.time()
ref = oracle.RefLP.graph(1, g.n, g.src, g.dst, vertex_w=g.vertex_w)
cp, ri, _ = ref.csc(); eu, ev = ref.edges()
print("build", time.time() - t, "rows", ref.m, "nnz", ref.nnz_struct)
def sectors(cp, rows):
    # distinct 32-B sectors (8 rows) per column, summed
    col = np.repeat(np.arange(len(cp) - 1), np.diff(cp))
    key = col.astype(np.int64) * (1 << 40) + (rows.astype(np.int64) >> 3)
    return len(np.unique(key))
nnz = len(ri)
print("R-17 order: sectors per nnz %.3f" % (sectors(cp, ri) / nnz))
# alternative: rows sorted by (higher-degree endpoint, other endpoint)
deg = np.bincount(eu, minlength=g.n) + np.bincount(ev, minlength=g.n)
hi = np.where(deg[eu] >= deg[ev], eu, ev); lo = np.where(deg[eu] >= deg[ev], ev, eu)
order = np.lexsort((lo, hi)); newid = np.empty(len(order), np.int64); newid[order] = np.arange(len(order))
# CSC in new row ids: column j rows = rows where j is an endpoint, ascending by new id
u2 = np.concatenate([eu, ev]); r2 = np.concatenate([newid, newid])
o = np.lexsort((r2, u2)); cp2 = np.concatenate([[0], np.cumsum(np.bincount(u2, minlength=g.n))])
print("by higher-degree endpoint: sectors per nnz %.3f" % (sectors(cp2, r2[o]) / nnz))
# CSR-upper (u, v) order
order = np.lexsort((ev, eu)); newid = np.empty(len(order), np.int64); newid[order] = np.arange(len(order))
r2 = np.concatenate([newid, newid]); o = np.lexsort((r2, u2))
print("(min, max) order: sectors per nnz %.3f" % (sectors(cp2, r2[o]) / nnz))
order = np.lexsort((eu, ev)); newid = np.empty(len(order), np.int64); newid[order] = np.arange(len(order))
r2 = np.concatenate([newid, newid]); o = np.lexsort((r2, u2))
print("(max, min) order: sectors per nnz %.3f" % (sectors(cp2, r2[o]) / nnz))
