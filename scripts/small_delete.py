"""Small deletes on a 10^7 uniform 3D tree (profiling target for the delete path; dev
aid): builds once, then deletes m random live ids per call, `reps` times.
  python scripts/small_delete.py [m] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t = zd.zd_build(torch.from_numpy(zdgen.uniform(10_000_000, 3, seed=43)).cuda())
rng = np.random.default_rng(5)
for _ in range(reps):
    live = t.zd_live_ids()
    kill = live[torch.from_numpy(rng.choice(live.numel(), size=m, replace=False)).cuda()]
    t.zd_delete(kill)
    torch.cuda.synchronize()
print("ok", t.zd_get_info()["fast_deletes"])
