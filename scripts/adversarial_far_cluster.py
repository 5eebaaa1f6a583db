"""Worst case of a coarse bound list (dev aid; GPU): a dense cluster plus a few far
outliers whose k nearest neighbours are cluster points at nearly equal distances.
  python scripts/adversarial_far_cluster.py [n] [outliers] [k]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402


def points(n, m, dim=3, seed=3):
    rng = np.random.default_rng(seed)
    c = 1 << 20
    core = rng.normal(0.0, 600.0, size=(n - m, dim))
    v = rng.normal(size=(m, dim))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    out = v * (0.9 * c)
    pts = np.concatenate([core, out]) + c
    return np.clip(np.rint(pts), 0, (1 << 21) - 1).astype(np.int32)


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    t = zd.zd_build(torch.from_numpy(points(n, m)).cuda())
    oi = torch.empty((n, k), dtype=torch.int32, device="cuda")
    od = torch.empty((n, k), dtype=torch.int64, device="cuda")
    for i in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t.zd_knn(k, out_idx=oi, out_dist2=od)
        e1.record()
        torch.cuda.synchronize()
        print(f"n={n} outliers={m} k={k} knn_ms {e0.elapsed_time(e1):.3f}", flush=True)
