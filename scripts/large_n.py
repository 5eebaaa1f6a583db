"""Scaling check beyond the BASELINE sizes (dev aid; GPU): build an n-point tree
(default 100M 3D uniform), all-points k-NN, timings, and sampled rows vs the oracle's
brute force.

  python scripts/large_n.py [n_millions] [dim] [k] [rows]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402

n = int(float(sys.argv[1]) * 1e6) if len(sys.argv) > 1 else 100_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 3
k = int(sys.argv[3]) if len(sys.argv) > 3 else 10
rows = int(sys.argv[4]) if len(sys.argv) > 4 else 48
t0 = time.time()
pts = zdgen.uniform(n, dim, seed=123)
gen_s = time.time() - t0
d = torch.from_numpy(pts).cuda()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {"n": n, "dim": dim, "k": k, "gen_s": round(gen_s, 1)}
for rep in range(2):
    e0, e1, e2 = ev(), ev(), ev()
    torch.cuda.synchronize()
    e0.record()
    t = zd.zd_build(d)
    e1.record()
    oi, od = t.zd_knn(k)
    e2.record()
    torch.cuda.synchronize()
    res.update(build_ms=round(e0.elapsed_time(e1), 2), knn_ms=round(e1.elapsed_time(e2), 2),
               build_mpts_s=round(n / e0.elapsed_time(e1) / 1e3, 1),
               queries_s=round(n / e1.elapsed_time(e2) * 1e3))
    if rep == 0:
        t.zd_free()
        del oi, od
res["gpu_mem_peak_gb"] = round(torch.cuda.max_memory_allocated() / 1e9, 2)
free, total = torch.cuda.mem_get_info()
res["device_used_gb"] = round((total - free) / 1e9, 1)
sel = np.random.default_rng(1).choice(n, size=rows, replace=False).astype(np.int32)
t0 = time.time()
bi, bd = oracle.brute_knn(pts, None, pts[sel], sel, k)
res["brute_s"] = round(time.time() - t0, 1)
gi = oi[torch.from_numpy(sel).long().cuda()].cpu().numpy()
gd = od[torch.from_numpy(sel).long().cuda()].cpu().numpy()
res["rows_checked"] = rows
res["rows_equal"] = int(np.sum(np.all(gi == bi, axis=1) & np.all(gd == bd, axis=1)))
print(json.dumps(res), flush=True)
