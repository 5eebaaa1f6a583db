"""Per-point update cost vs batch size (the paper's Fig. 4; NEXT-2).

Base: 10^7 uniform points (2D as in Fig. 4, and 3D).  For batch sizes 1 .. 10^6: the
wall time of one zd_insert of m fresh uniform points and of one zd_delete of m random
original ids (each call is synchronous: one host sync), median of 5, on a tree that
has already absorbed a warm-up update of the same size.  One JSON line per (dim, m).
  python scripts/fig4_curve.py [2,3]
"""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402

# Fig. 4's printed per-point seconds, context only (reading R27: every
# value is as printed; 144 threads, Dell R930)
PAPER_INSERT = {1: 3.35e-5, 10: 9.4e-6, 100: 5.3e-6}
N = 10_000_000


def main():
    dims = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2", "3"])]
    zd.load()
    for dim in dims:
        base = torch.from_numpy(zdgen.uniform(N, dim, seed=40 + dim)).cuda()
        t = zd.zd_build(base)
        rng = np.random.default_rng(7)
        for m in (1, 10, 100, 1000, 10_000, 100_000, 1_000_000):
            ins, dels, fast_i, fast_d = [], [], 0, 0
            for rep in range(6):
                b = torch.from_numpy(zdgen.uniform(m, dim, seed=1000 * m + rep)).cuda()
                live = t.zd_live_ids()
                kill = live[torch.from_numpy(rng.choice(live.numel(), size=m, replace=False)).cuda()]
                torch.cuda.synchronize()
                f0 = t.zd_get_info()
                t0 = time.perf_counter()
                t.zd_insert(b)
                t1 = time.perf_counter()
                t.zd_delete(kill)
                t2 = time.perf_counter()
                f1 = t.zd_get_info()
                if rep > 0:   # rep 0 warms the pool for this batch size
                    ins.append(t1 - t0)
                    dels.append(t2 - t1)
                    fast_i += f1["fast_inserts"] - f0["fast_inserts"]
                    fast_d += f1["fast_deletes"] - f0["fast_deletes"]
            mi, md = statistics.median(ins), statistics.median(dels)
            print(json.dumps({"dim": dim, "n": N, "batch": m, "insert_ms": round(mi * 1e3, 4),
                              "delete_ms": round(md * 1e3, 4), "insert_s_per_point": mi / m,
                              "delete_s_per_point": md / m, "fast_inserts": fast_i, "fast_deletes": fast_d,
                              "paper_insert_s_per_point_144thr": PAPER_INSERT.get(m)}), flush=True)
        t.zd_free()


if __name__ == "__main__":
    main()
