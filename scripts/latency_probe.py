"""Fixed-cost floor of one small synchronous update call on this box (dev aid for the
NEXT-2 analysis): wall time of an empty torch kernel + sync, of a 4-byte
device->host copy + sync, and of zd_insert / zd_delete of 1 and 10 points on a 10^7
uniform 3D tree, with the library's per-phase device times."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402


def wall(f, reps=20):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6


x = torch.zeros(1, device="cuda")
h = torch.zeros(1).pin_memory()
print("empty kernel + sync us", round(wall(lambda: (x.add_(1), torch.cuda.synchronize())), 1))
print("4-byte D2H + sync us", round(wall(lambda: (h.copy_(x, non_blocking=True), torch.cuda.synchronize())), 1))
t = zd.zd_build(torch.from_numpy(zdgen.uniform(10_000_000, 3, seed=43)).cuda(), timing=True)
rng = np.random.default_rng(3)
for m in (1, 10):
    ins, dels = [], []
    for rep in range(12):
        b = torch.from_numpy(zdgen.uniform(m, 3, seed=777 * m + rep)).cuda()
        live = t.zd_live_ids()
        kill = live[torch.from_numpy(rng.choice(live.numel(), size=m, replace=False)).cuda()]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t.zd_insert(b)
        t1 = time.perf_counter()
        pi = t.zd_get_timing()
        t.zd_delete(kill)
        t2 = time.perf_counter()
        pd = t.zd_get_timing()
        if rep >= 2:
            ins.append(t1 - t0)
            dels.append(t2 - t1)
    print(f"m={m} insert us {statistics.median(ins) * 1e6:.1f} delete us {statistics.median(dels) * 1e6:.1f}",
          "last insert phases", {k: round(v * 1e3, 1) for k, v in pi.items() if v},
          "last delete phases", {k: round(v * 1e3, 1) for k, v in pd.items() if v}, t.zd_get_info())
