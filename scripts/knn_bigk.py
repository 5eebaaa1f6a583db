"""Time k = 16 and 32 all-points k-NN (dev aid)."""
import sys; sys.path.insert(0,'/root/repo')
import json, torch, paper_2111_04182_b200 as zd, zdgen
for name in sys.argv[1].split(','):
    pts=torch.from_numpy(zdgen.config_points(name)).cuda(); n=pts.shape[0]; t=zd.zd_build(pts)
    for k in (16, 32):
        oi=torch.empty((n,k),dtype=torch.int32,device='cuda'); od=torch.empty((n,k),dtype=torch.int64,device='cuda')
        t.zd_knn(k,out_idx=oi,out_dist2=od); best=1e9
        for _ in range(3):
            e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record(); t.zd_knn(k,out_idx=oi,out_dist2=od); e1.record(); torch.cuda.synchronize(); best=min(best,e0.elapsed_time(e1))
        print(name, k, round(best,3), flush=True)
