"""NEXT-1 measurement: external ("dynamic") k-NN queries (App. B, Fig. 5):
build on n points, query n other points of the same distribution (Morton sort of the
queries + bit-based leaf location + packet search).  One JSON line per config."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402


def main():
    for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["C3", "C2", "C4a"]):
        c = zdgen.CONFIGS[name]
        n = c["n"]
        pts = torch.from_numpy(zdgen.config_points(name)).cuda()
        q = torch.from_numpy(zdgen.points(c["dist"], n, c["dim"], c["seed"] + 1000)).cuda()
        t = zd.zd_build(pts)
        oi = torch.empty((n, 10), dtype=torch.int32, device="cuda")
        od = torch.empty((n, 10), dtype=torch.int64, device="cuda")
        t.zd_knn(10, queries=q, out_idx=oi, out_dist2=od)
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t.zd_knn(10, queries=q, out_idx=oi, out_dist2=od)
            e1.record()
            torch.cuda.synchronize()
            best = e0.elapsed_time(e1) if best is None else min(best, e0.elapsed_time(e1))
        print(json.dumps({"config": name, "n_tree": n, "n_queries": n, "k": 10, "ms": round(best, 3),
                          "queries_per_s": round(n / (best / 1e3)), "note": "includes query Morton sort + leaf location"}),
              flush=True)
        t.zd_free()


if __name__ == "__main__":
    main()
