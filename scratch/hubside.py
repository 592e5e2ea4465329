import numpy as np, sys
sys.path.insert(0,'.')
import inputs
s=24
src, dst = inputs.rmat(s, 16 << s, 0.57, 0.19, 0.19, 13115)
n = 1 << s
lo = np.minimum(src, dst).astype(np.int64); hi = np.maximum(src, dst).astype(np.int64)
k = np.unique((hi << 32 | lo)[lo != hi])   # (max, min) order
u = (k & 0xffffffff); v = (k >> 32)
deg = np.bincount(u, minlength=n) + np.bincount(v, minlength=n)
tiles = deg.reshape(-1, 32).sum(1)
hub_tile = tiles > 2048
hub = hub_tile[np.arange(n) // 32]
hu = hub[u]; hv = hub[v]
m = len(k)
print('rows', m, 'rows with hub u', hu.mean(), 'hub v', hv.mean(), 'both', (hu&hv).mean(), 'neither', (~hu&~hv).mean())
print('hub vertices', hub.sum(), 'hub u ids < 8192 frac', (u[hu] < 8192).mean(), '< 65536', (u[hu] < 65536).mean())
# concentration: share of hub-u incidences on top-K vertices
cnt = np.bincount(u[hu], minlength=n)
srt = np.sort(cnt)[::-1]
for K in (1, 32, 1024, 8192, 65536):
    print('top', K, 'share', srt[:K].sum()/srt.sum())
