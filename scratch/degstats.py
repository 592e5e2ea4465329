import numpy as np, sys
sys.path.insert(0,'.')
import inputs
for s in (20, 22, 24):
    src, dst = inputs.rmat(s, 16 << s, 0.57, 0.19, 0.19, 13115)
    n = 1 << s
    lo = np.minimum(src, dst).astype(np.int64); hi = np.maximum(src, dst).astype(np.int64)
    k = np.unique((lo << 32 | hi)[lo != hi])
    u = (k >> 32); v = k & 0xffffffff
    deg = np.bincount(u, minlength=n) + np.bincount(v, minlength=n)
    tiles = deg.reshape(-1, 32).sum(1)
    tot = deg.sum()
    for H in (2048, 8192, 65536):
        h = tiles > H
        print(s, 'm', len(k), 'H', H, 'heavy tiles', h.sum(), 'heavy nnz frac', tiles[h].sum()/tot, 'max tile nnz', tiles.max(), 'max deg', deg.max())
