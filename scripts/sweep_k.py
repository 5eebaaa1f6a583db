"""NEXT-3 measurements: k sweep (the paper's Fig. 3(e), time per neighbour vs k) and the
root-based vs leaf-based search ablation (Fig. 2, P:243 vs P:248) on one B200.
Prints one JSON line per (config, k, variant): steady-state k-NN ms (CUDA events).

  python scripts/sweep_k.py [configs] [ks] [kernels]
  kernels: comma list of packet (k <= 32; the default kernel there), warp (the
  warp-per-query kernel, forced for k <= 32, the only one above), root (root-based)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402


def timed(t, k, root, n, warp=False, reps=3):
    oi = torch.empty((n, k), dtype=torch.int32, device="cuda")
    od = torch.empty((n, k), dtype=torch.int64, device="cuda")
    t.zd_knn(k, out_idx=oi, out_dist2=od, root_based=root, warp=warp)
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t.zd_knn(k, out_idx=oi, out_dist2=od, root_based=root, warp=warp)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best


def main():
    configs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C3", "C4a", "C4b", "C2", "K2"]
    ks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 4, 8, 10, 16, 32]
    kernels = sys.argv[3].split(",") if len(sys.argv) > 3 else ["packet", "root"]
    for name in configs:
        pts = torch.from_numpy(zdgen.config_points(name)).cuda()
        n = pts.shape[0]
        t = zd.zd_build(pts)
        for k in ks:
            for kern in kernels:
                if kern == "root" and k not in (1, 10):
                    continue
                if kern == "packet" and k > 32:
                    continue
                ms = timed(t, k, kern == "root", n, warp=kern == "warp")
                print(json.dumps({"config": name, "k": k, "search": "root" if kern == "root" else "leaf",
                                  "kernel": "warp" if (kern == "warp" or k > 32) else "packet",
                                  "knn_ms": round(ms, 3), "ns_per_neighbor": round(ms * 1e6 / (n * k), 3),
                                  "queries_per_s": round(n / (ms / 1e3))}), flush=True)
        t.zd_free()


if __name__ == "__main__":
    main()
