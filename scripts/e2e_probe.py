"""Time the pieces of the e2e (host-buffer) path (dev aid)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402

c = zdgen.CONFIGS["C5"]
pts = torch.from_numpy(zdgen.config_points("C5")).pin_memory()
batch = torch.from_numpy(zdgen.insert_batch(c["insert_m"], 3, c["insert_seed"])).pin_memory()
kill = torch.from_numpy(zdgen.delete_ids(c["n"], c["delete_m"], c["delete_seed"])).pin_memory()
n_live = c["n"]
oi = torch.empty((n_live, 10), dtype=torch.int32).pin_memory()
od = torch.empty((n_live, 10), dtype=torch.int64).pin_memory()
for it in range(4):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    tr = zd.zd_build(pts); torch.cuda.synchronize(); t.append(time.perf_counter())
    tr.zd_insert(batch); torch.cuda.synchronize(); t.append(time.perf_counter())
    tr.zd_delete(kill); torch.cuda.synchronize(); t.append(time.perf_counter())
    tr.zd_knn(10, out_idx=oi, out_dist2=od); torch.cuda.synchronize(); t.append(time.perf_counter())
    tr.zd_free(); torch.cuda.synchronize(); t.append(time.perf_counter())
    print(it, "build %.1f insert %.1f delete %.1f knn %.1f free %.1f ms" % tuple((b - a) * 1e3 for a, b in zip(t[:-1], t[1:])), flush=True)
