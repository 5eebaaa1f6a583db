"""Repeat the all-points k-NN on one config (profiling target; dev aid)."""
import sys; sys.path.insert(0,'/root/repo')
import torch, paper_2111_04182_b200 as zd, zdgen
pts=torch.from_numpy(zdgen.config_points(sys.argv[1])).cuda()
t=zd.zd_build(pts)
oi = torch.empty((pts.shape[0], 10), dtype=torch.int32, device="cuda")
od = torch.empty((pts.shape[0], 10), dtype=torch.int64, device="cuda")
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t.zd_knn(10, out_idx=oi, out_dist2=od)
    e1.record()
    torch.cuda.synchronize()
    print(sys.argv[1], i, "knn_ms %.3f" % e0.elapsed_time(e1), flush=True)
