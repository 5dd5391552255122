"""Locate differences between the GPU exact join and the oracle at C1."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_21230_b200 as F
from paper_2508_21230_b200 import engine
from oracle import oracle as O
n, d, eps = 16384, 128, 3.973260466174982
hd = F.to_half(F.generate_synthetic(n, d, seed=12345))
oi, oj, od = O.join(hd.values, hd.norms, n, eps)
for mode in ("exact", "tc"):
    rs = F.self_join(hd, eps, mode=mode)
    print(mode, "count", len(rs), len(oi))
    if len(rs) == len(oi):
        bad = np.nonzero((rs.i != oi) | (rs.j != oj) | (rs.dist_sq.view(np.uint32) != od.view(np.uint32)))[0]
        print(" mismatches", len(bad))
        for b in bad[:10]:
            print("  ", b, (rs.i[b], rs.j[b], rs.dist_sq[b]), (oi[b], oj[b], od[b]))
    key = rs.i.astype(np.int64) * (1 << 32) + rs.j
    print(" sorted", bool(np.all(np.diff(key) > 0)), "dups", len(key) - len(np.unique(key)))
# unsorted raw exact output vs oracle set
dd = engine.upload(hd, 0)
es = float(O.eps_sq_of(eps))
res = engine.join_device(dd, es, exact=True, sort=False)
i, j, dv = engine.to_host(res)
k1 = i.astype(np.int64) * (1 << 32) + j; k2 = oi.astype(np.int64) * (1 << 32) + oj
print("raw exact: count", len(i), "set equal", np.array_equal(np.sort(k1), np.sort(k2)))
order = np.argsort(k1)
print("raw exact d equal", np.array_equal(dv[order].view(np.uint32), od.view(np.uint32)))
