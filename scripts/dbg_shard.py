import numpy as np, sys
sys.path.insert(0, '.')
from paper_2404_03226_b200 import abi, api
from paper_2404_03226_b200 import platform as P
costs = P.default_cost_table()
hb = api.HostBatch().add_layered(12288, 96, 1.0 / 32, [5])
b = hb.view()
ctx = api.Context(0); ctx.set_large_graph_threshold(1000)
db = ctx.upload(b)
want = ctx.attributes(db, costs, abi.ATTR_ALL)
lay = ctx.attributes(db, costs, abi.ATTR_LAYERS)["layer"]
n = b.n_tasks
L = lay.max() + 1
cnt = np.bincount(lay, minlength=L)
lstart = np.concatenate([[0], np.cumsum(cnt)])
# level-order positions: within a level arbitrary on device; words only depend on level ranges
nw = (n + 63) // 64
dens = np.zeros(nw + 1)
for l in range(L):
    lo = min(lstart[l + 1] >> 6, nw)
    dens[lo] += cnt[l]
cum = np.concatenate([[0], np.cumsum(np.cumsum(dens[:nw]))])
world = 2
b1 = np.searchsorted(cum, cum[-1] * 1 / world)
print("nw", nw, "b1", b1, "lstart near", [(l, lstart[l+1] >> 6) for l in range(55, 70)])
ctxs = [api.Context(0) for _ in range(world)]
parts = []
for r, c in enumerate(ctxs):
    c.set_large_graph_threshold(1000)
    d = c.upload(b)
    parts.append(c.attributes_shard_partial(d, costs, r, world))
ab = sum(p[0] for p in parts)
bad = np.nonzero(ab != want["ability"])[0]
print("bad", len(bad))
for u in bad[:8]:
    print(u, "level", lay[u], "lo", lstart[lay[u] + 1] >> 6, "want", want["ability"][u], "r0", parts[0][0][u], "r1", parts[1][0][u])
