"""Debug: TC filter vs exact path on a deterministic single-CTA flat scan."""
import math, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_17229_b200 as gp
from oracle import Oracle

dim, dd, k = 64, 16, 10
g = np.random.default_rng(dim + dd)
n, nq = 3000, 64
lam = np.arange(1, dim + 1) ** -1.2
centers = g.standard_normal((8, dim)) * 3
data = (centers[g.integers(0, 8, n)] + g.standard_normal((n, dim)) * np.sqrt(lam * dim / lam.sum())).astype(np.float32)
qs = (data[g.integers(0, n, nq)] + 0.3 * g.standard_normal((nq, dim))).astype(np.float32)
os.environ["DADE_GPU_FLAT_BLOCKS"] = "1"
dev = gp.Device(0)
fi = gp.FlatIndex(dev, data)
s = gp.AdsamplingStrategy(dim, dd, 1.0, dev=dev)
res = {}
for tc in ["0", "1", "0", "1"]:
    os.environ["DADE_GPU_NO_TC"] = "1" if tc == "0" else "0"
    st = gp.DcoStats()
    ids, d, cnt = fi.search_batch(qs, k, s, st)
    key = tc + ("b" if tc in res else "")
    res[key] = (ids, d, cnt, st.total_dco, st.dims_accumulated)
    print(tc, st.total_dco, st.dims_accumulated)
print("det0", np.array_equal(res["0"][0], res["0b"][0]), "det1", np.array_equal(res["1"][0], res["1b"][0]))
a, b = res["0"], res["1"]
o = Oracle()
cps, co, sc = o.ads_tables(dim, dd, 1.0)
for q in range(nq):
    if not np.array_equal(a[0][q], b[0][q]):
        print("q", q, "exact", a[0][q], a[1][q])
        print("    tc", b[0][q], b[1][q])
        # which ids missing in tc
        miss = set(a[0][q]) - set(b[0][q])
        for m in miss:
            pr = [o.partial_sqdist(data[m], qs[q], 0, dd)]
            print("   missing", m, "partial16", pr, "full", math.sqrt(o.partial_sqdist(data[m], qs[q], 0, dim)))
        break
