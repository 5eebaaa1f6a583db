"""Time all-points k-NN at given k (dev aid; also an ncu target).

  python scripts/knn_bigk.py C3 16,32,100 [reps] [warp]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402

ks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16, 32]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
warp = len(sys.argv) > 4 and sys.argv[4] == "warp"
for name in sys.argv[1].split(","):
    pts = torch.from_numpy(zdgen.config_points(name)).cuda()
    n = pts.shape[0]
    t = zd.zd_build(pts)
    for k in ks:
        oi = torch.empty((n, k), dtype=torch.int32, device="cuda")
        od = torch.empty((n, k), dtype=torch.int64, device="cuda")
        t.zd_knn(k, out_idx=oi, out_dist2=od, warp=warp)
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t.zd_knn(k, out_idx=oi, out_dist2=od, warp=warp)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(name, k, round(best, 3), flush=True)
