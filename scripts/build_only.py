"""Repeated zd_build on a config with event timing (profiling target; dev aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
pts = torch.from_numpy(zdgen.config_points(name)).cuda()
for i in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    t = zd.zd_build(pts, timing=True)
    e1.record()
    torch.cuda.synchronize()
    print(name, i, "build_ms %.3f" % e0.elapsed_time(e1), {k: round(v, 3) for k, v in t.zd_get_timing().items() if v}, flush=True)
    t.zd_free()
