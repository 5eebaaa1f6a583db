"""Quick per-phase timing probe (development aid, not the bench contract)."""
import argparse
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2111_04182_b200 as zd
import zdgen


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4a,C4b,C5")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    zd.load()
    for name in args.configs.split(","):
        c = zdgen.CONFIGS[name]
        t0 = time.time()
        pts = torch.from_numpy(zdgen.config_points(name)).cuda()
        gen_s = time.time() - t0
        res = []
        for r in range(args.reps):
            torch.cuda.synchronize()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            t = zd.zd_build(pts, timing=True)
            e1.record()
            torch.cuda.synchronize()
            row = dict(build_ms=round(e0.elapsed_time(e1), 3), build_phases=t.zd_get_timing())
            e1.record()
            oi, od = t.zd_knn(10)
            e2.record()
            torch.cuda.synchronize()
            row["knn_ms"] = round(e1.elapsed_time(e2), 3)
            row["leaves"] = t.zd_get_info()["n_leaves"]
            if "insert_m" in c:
                b = torch.from_numpy(zdgen.insert_batch(c["insert_m"], 3, c["insert_seed"])).cuda()
                kill = torch.from_numpy(zdgen.delete_ids(c["n"], c["delete_m"], c["delete_seed"])).cuda()
                torch.cuda.synchronize()
                e0.record()
                t.zd_insert(b)
                e1.record()
                torch.cuda.synchronize()
                row["insert_ms"] = round(e0.elapsed_time(e1), 3)
                row["insert_phases"] = t.zd_get_timing()
                e0.record()
                t.zd_delete(kill)
                e1.record()
                torch.cuda.synchronize()
                row["delete_ms"] = round(e0.elapsed_time(e1), 3)
                row["delete_phases"] = t.zd_get_timing()
                e0.record()
                oi, od = t.zd_knn(10)
                e1.record()
                torch.cuda.synchronize()
                row["knn2_ms"] = round(e0.elapsed_time(e1), 3)
            res.append(row)
            t.zd_free()
        print(json.dumps(dict(config=name, n=c["n"], gen_s=round(gen_s, 2), runs=res)), flush=True)


if __name__ == "__main__":
    main()
