"""Repeat zd_build on one config (profiling target; dev aid)."""
import sys
sys.path.insert(0, '/root/repo')
import torch, paper_2111_04182_b200 as zd, zdgen
pts = torch.from_numpy(zdgen.config_points(sys.argv[1])).cuda()
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = zd.zd_build(pts, timing=True)
    e1.record()
    torch.cuda.synchronize()
    print(sys.argv[1], i, "build_ms %.3f" % e0.elapsed_time(e1), {k: round(v, 3) for k, v in t.zd_get_timing().items() if v}, flush=True)
    t.zd_free()
