"""Per-packet / per-query work of the k-NN kernel (profiling build; development aid).

  ZD_LIB=stats python scripts/knn_stats.py --configs C1,C3
"""
import argparse
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("ZD_LIB", "stats")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4a,C4b")
    ap.add_argument("--k", type=int, default=10)
    args = ap.parse_args()
    zd.load()
    for name in args.configs.split(","):
        pts = torch.from_numpy(zdgen.config_points(name)).cuda()
        t = zd.zd_build(pts)
        zd.zd_knn_stats(reset=True)
        t.zd_knn(args.k)
        torch.cuda.synchronize()
        s = zd.zd_knn_stats(reset=True)
        p, q = s["packets"], s["queries"]
        hist = {i: s.pop(f"hist{i}") for i in range(32) if s.get(f"hist{i}")}
        cyc = s["cycles"]
        mp = s.pop("max_packet")
        s["slowest_packet"] = {"packet": mp & 0xFFFFFF, "cycles": mp >> 24}
        # share of all packet-cycles spent in packets of 2^i .. 2^(i+1) cycles
        out = {"config": name, "k": args.k, "cycle_hist_log2": hist,
               "mean_cycles_per_packet": round(cyc / s["packets"]), **s,
               "per_packet": {k: round(v / p, 2) for k, v in s.items()
                              if k not in ("packets", "queries", "slowest_packet")},
               "per_query": {"candidates_per_lane": round(s["candidates"] / p, 1), "hits": round(s["hits"] / q, 2),
                             "survivors": round(s["survivors"] / q, 2)}}
        print(json.dumps(out), flush=True)
        t.zd_free()


if __name__ == "__main__":
    main()
