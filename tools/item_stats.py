"""Work-item census of the streaming passes on a BASELINE workload (diagnostic).
    python tools/item_stats.py [config1]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_17229_b200 as gp
from paper_2411_17229_b200 import workloads as W

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config1"]
dev = gp.Device(0)
art = W.build(cfg, dev, torch.device("cuda:0"), with_gt=False, log=print)
cen = torch.from_numpy(art.centroids).cuda().double()
q = art.q_rot.double()
d = torch.cdist(q, cen)
near = d.topk(cfg.nprobe, largest=False).indices.cpu().numpy()
sizes = np.diff(art.offsets.astype(np.int64))
K, SEED, PIECE, QC = cfg.k, int(os.environ.get("SEED_ROWS", 512)), 1024, 64
for rank_lo, rank_hi, name in [(0, 1, "nearest"), (1, cfg.nprobe, "others")]:
    cnt = np.zeros(cfg.nlist, np.int64)
    for r in range(rank_lo, rank_hi):
        np.add.at(cnt, near[:, r], 1)
    used = cnt > 0
    skip = np.where((rank_lo == 0) & (sizes >= K), np.minimum(sizes, SEED), 0)
    rem = sizes - skip
    pieces = np.maximum(1, (rem + PIECE - 1) // PIECE)
    qch = (cnt + QC - 1) // QC
    items = (qch * pieces * (rem > 0))[used].sum()
    pairs = (cnt * rem)[used].sum()
    p0 = (cnt * np.minimum(rem, PIECE))[used].sum()
    print(f"{name}: lists {used.sum()} items {items} pairs {pairs:.3e} piece0-pairs {p0:.3e} "
          f"q/list max {cnt.max()} mean {cnt[used].mean():.1f} rem rows max {rem[used].max()} "
          f"pieces max {pieces[used].max()} lists<K {(sizes[used] < K).sum()}")
print("list sizes: min/median/mean/max", sizes.min(), np.median(sizes), sizes.mean(), sizes.max())
print("size percentiles 50/90/99/99.9:", np.percentile(sizes, [50, 90, 99, 99.9]))
# seed census: groups of <= 16 queries per nearest list, rows min(size, 1024)
cnt0 = np.zeros(cfg.nlist, np.int64)
np.add.at(cnt0, near[:, 0], 1)
g = (cnt0 + 15) // 16
rows = np.minimum(sizes, 1024)
print(f"seed: groups {g.sum()} lists {(cnt0 > 0).sum()} q/group mean {cnt0.sum() / max(1, g.sum()):.2f} "
      f"tile bytes {(g * rows).sum() * cfg.dim * 4 / 1e9:.3f} GB (unique {(rows * (cnt0 > 0)).sum() * cfg.dim * 4 / 1e9:.3f} GB) "
      f"pair-dims {(cnt0 * rows).sum() * cfg.dim:.3e} padded {(((cnt0 + 1) // 2 * 2) * rows).sum() * cfg.dim:.3e}")
print("q per nearest list histogram:", np.bincount(np.minimum(cnt0, 40)))
