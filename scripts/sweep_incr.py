"""NEXT-2 (part): the insert fast path (csrc/incr.cu) on a 10M-point base (dev aid; GPU).

For batches that keep the canonical topology (points placed in leaves with room:
copies of a leaf's point with the lowest bit of one coordinate flipped), time the
insert with the fast path and with ZD_INCR=0 (full rebuild), m = 100 .. 64K, and the
delete of those points again; and the fraction of random single-point inserts and
deletes that keep the topology.  One JSON line
per measurement."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402


def fitting(ex, dim, m, rng):
    ls = ex["leaf_start"]
    sizes = np.diff(ls)
    leaves = rng.choice(np.nonzero(sizes <= 15)[0], size=m, replace=False)
    p = ex["recs"][ls[leaves], :dim].astype(np.int64)
    p[np.arange(m), rng.integers(0, dim, size=m)] ^= 1
    return np.ascontiguousarray(p.astype(np.int32))


def timed_insert(pts, b, incr):
    os.environ["ZD_INCR"] = "1" if incr else "0"
    best, fast = 1e9, None
    for _ in range(3):
        t = zd.zd_build(pts)
        t.zd_insert(b[:1])          # grow the capacity outside the timed call
        f0 = t.zd_get_info()["fast_inserts"]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        t.zd_insert(b[1:])
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
        fast = t.zd_get_info()["fast_inserts"] - f0
        t.zd_free()
    return best, fast


for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["C3", "C2"]):
    pts_np = zdgen.config_points(name)
    dim = pts_np.shape[1]
    pts = torch.from_numpy(pts_np).cuda()
    t = zd.zd_build(pts)
    ex = t.zd_export()
    rng = np.random.default_rng(5)
    for m in (100, 1000, 10000, 65536):
        b = torch.from_numpy(fitting(ex, dim, m + 1, rng)).cuda()
        ms_f, nf = timed_insert(pts, b, True)
        ms_r, _ = timed_insert(pts, b, False)
        print(json.dumps({"config": name, "batch": m, "fast_ms": round(ms_f, 4), "rebuild_ms": round(ms_r, 4),
                          "fast_path_taken": bool(nf), "fast_ns_per_point": round(ms_f * 1e6 / m, 1),
                          "rebuild_ns_per_point": round(ms_r * 1e6 / m, 1)}), flush=True)
    # deletes that undo a fitting insert (keep the topology) vs the rebuild
    for m in (100, 1000, 10000):
        b = torch.from_numpy(fitting(ex, dim, m, rng)).cuda()
        res = {}
        for incr in (True, False):
            os.environ["ZD_INCR"] = "1" if incr else "0"
            best, fd = 1e9, 0
            for _ in range(3):
                t3 = zd.zd_build(pts)
                first = t3.zd_insert(b)
                ids = torch.arange(first, first + m, dtype=torch.int32, device="cuda")
                d0 = t3.zd_get_info()["fast_deletes"]
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                t3.zd_delete(ids)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
                fd = t3.zd_get_info()["fast_deletes"] - d0
                t3.zd_free()
            res[incr] = (best, fd)
        print(json.dumps({"config": name, "delete_batch": m, "fast_ms": round(res[True][0], 4),
                          "rebuild_ms": round(res[False][0], 4), "fast_path_taken": bool(res[True][1])}), flush=True)
    # how often does a random single point keep the topology?
    os.environ["ZD_INCR"] = "1"
    t2 = zd.zd_build(pts)
    q = zdgen.uniform(300, dim, seed=77)
    f0 = t2.zd_get_info()["fast_inserts"]
    for i in range(len(q)):
        t2.zd_insert(torch.from_numpy(q[i:i + 1]).cuda())
    frac = (t2.zd_get_info()["fast_inserts"] - f0) / len(q)
    print(json.dumps({"config": name, "random_single_point_inserts": len(q), "fraction_fast": round(frac, 3)}), flush=True)
    d0 = t2.zd_get_info()["fast_deletes"]
    kill = np.random.default_rng(9).choice(pts_np.shape[0], size=300, replace=False).astype(np.int32)
    for i in range(len(kill)):
        t2.zd_delete(torch.from_numpy(kill[i:i + 1]).cuda())
    frac = (t2.zd_get_info()["fast_deletes"] - d0) / len(kill)
    print(json.dumps({"config": name, "random_single_point_deletes": len(kill), "fraction_fast": round(frac, 3)}), flush=True)
