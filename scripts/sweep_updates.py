"""NEXT-2 measurement: batch insert / delete cost vs batch size on a 10M-point base
(the paper's Fig. 4 shape: per-point update time vs batch size; 2D uniform
as in the paper, and 3D uniform).  One JSON line per (dim, batch, op)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402


def main():
    n = 10_000_000
    for dim in (2, 3):
        base = torch.from_numpy(zdgen.uniform(n, dim, seed=40 + dim)).cuda()
        for m in (1_000, 10_000, 100_000, 1_000_000, 5_000_000):
            batch = torch.from_numpy(zdgen.uniform(m, dim, seed=50 + dim, first_index=n)).cuda()
            kill = torch.from_numpy(zdgen.delete_ids(n, m, seed=60 + dim)).cuda()
            ins, dele = [], []
            for rep in range(4):
                t = zd.zd_build(base)
                torch.cuda.synchronize()
                for op, arg, acc in (("insert", batch, ins), ("delete", kill, dele)):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    (t.zd_insert if op == "insert" else t.zd_delete)(arg)
                    e1.record()
                    torch.cuda.synchronize()
                    if rep:
                        acc.append(e0.elapsed_time(e1))
                t.zd_free()
            for op, acc in (("insert", ins), ("delete", dele)):
                ms = float(np.median(acc))
                print(json.dumps({"dim": dim, "n": n, "batch": m, "op": op, "ms": round(ms, 4),
                                  "ns_per_point": round(ms * 1e6 / m, 2), "mpts_per_s": round(m / ms / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
