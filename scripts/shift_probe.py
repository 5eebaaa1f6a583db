"""NEXT-4: 2D random shift — build and all-points k=10 times with and without
a shift on the 2D configs (dev aid; GPU).  One JSON line per (config, shift)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, r


rng = np.random.default_rng(2111)
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "K2"]):
    pts = torch.from_numpy(zdgen.config_points(name)).cuda()
    n = pts.shape[0]
    ref = None
    for shift in [None] + [tuple(int(v) for v in rng.integers(0, 1 << 30, size=2)) for _ in range(3)]:
        bms, t = timed(lambda: zd.zd_build(pts, shift=shift))
        oi = torch.empty((n, 10), dtype=torch.int32, device="cuda")
        od = torch.empty((n, 10), dtype=torch.int64, device="cuda")
        kms, _ = timed(lambda: t.zd_knn(10, out_idx=oi, out_dist2=od))
        same = None
        if ref is None:
            ref = (oi.clone(), od.clone())
        else:
            same = bool(torch.equal(ref[0], oi) and torch.equal(ref[1], od))
        info = t.zd_get_info()
        print(json.dumps({"config": name, "shift": shift, "build_ms": round(bms, 3), "knn_ms": round(kms, 3),
                          "leaves": info["n_leaves"], "same_answer_as_unshifted": same}), flush=True)
        t.zd_free()
