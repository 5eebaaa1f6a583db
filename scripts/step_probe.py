"""C5 step phase times over repeated steps (dev aid: pool / sync-order experiments)."""
import sys
import time
sys.path.insert(0, '/root/repo')
import torch, bench, paper_2111_04182_b200 as zd
zd.load()
pts_np, batch_np, kill_np = bench.workload_inputs()
pts, batch, kill = (torch.from_numpy(a).cuda() for a in (pts_np, batch_np, kill_np))
n_live = 10_000_000
oi = torch.empty((n_live, 10), dtype=torch.int32, device="cuda")
od = torch.empty((n_live, 10), dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    h = [time.perf_counter()]
    ev[0].record(st); t = zd.zd_build(pts, timing=True); ev[1].record(st); h.append(time.perf_counter())
    tb = t.zd_get_timing()
    t.zd_insert(batch); ev[2].record(st); h.append(time.perf_counter())
    ti = t.zd_get_timing()
    t.zd_delete(kill); ev[3].record(st); h.append(time.perf_counter())
    t.zd_knn(10, out_idx=oi, out_dist2=od); ev[4].record(st)
    torch.cuda.synchronize(); h.append(time.perf_counter())
    print(i, "dev", " ".join("%.3f" % ev[j].elapsed_time(ev[j + 1]) for j in range(4)),
          "host", " ".join("%.3f" % ((h[j + 1] - h[j]) * 1e3) for j in range(4)),
          "build", {k: round(v, 3) for k, v in tb.items() if v}, "ins", {k: round(v, 3) for k, v in ti.items() if v},
          flush=True)
    t.zd_free()
