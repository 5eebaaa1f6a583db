#!/usr/bin/env python
"""bench.py — zd-tree hot path on B200 (one JSON line on rank 0).

A step = one pass of the whole hot path over config C5
(BASELINE.json configs[4]): zd_build on 10^7 uniform 3D points, zd_insert of 10^6
points, zd_delete of 10^6 original ids, then the all-points exact k=10 query over
the 10^7 live points.  Metric: all-points kNN queries/s (k=10, 10M 3D pts) of the
whole step (build + updates + query); the build Mpts/s and per-phase throughputs
are reported beside it.

Timing: inputs resident in HBM; W untimed warm-up steps; K timed steps, each
bracketed by CUDA events on the working stream with a 256 MB L2 flush (> 126 MB L2)
between steps outside the timed region; barrier + synchronize around the timed
loop; max over ranks.  Multi-GPU (the parallel-for over queries
of P:53 / P:543): every rank holds a replica of the tree (it runs the build and both
updates itself: no exchange) and answers one contiguous Morton range of the 10^7
queries (zd_knn_range); value = the 10^7 queries / max time over ranks ("strong").

Beside the headline (rank 0, one GPU): a per-config report for C1-C4b (build and
k-NN throughput with their roofline fractions, every row compared with the oracle),
the oracle timed on the host cores at full size (all cores; one thread for C1 and a
10^6-point C3 sample) and the CPU model.

--impl reference: the CPU oracle (oracle/, the only other place bench.py executes
it) on the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import zdgen  # noqa: E402

METRIC = "all-points kNN queries/s (k=10, 10M 3D pts)"
UNIT = "queries/s"
K_NN = 10
WORKLOAD = "C5"
PAPER_CONTEXT = {
    "build_plus_knn_3DinCube_10M_k10_qps": 22.1e6,
    "build_3DinCube_10M_mpts_s": 140.0,
    "hardware": "Dell R930, 4x Xeon E7-8867 v4, 144 threads (PAPER.md P:1022, P:1127, P:1209)",
    "note": "context only: the paper reports no k=10 numbers with batch updates (BASELINE.md)",
}


# ----------------------------------------------------------------- helpers

def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class Dist:
    """torch.distributed plumbing for N>1 (barrier + max over ranks)."""

    def __init__(self, backend: str | None = None):
        self.world = env_int("WORLD_SIZE", 1)
        self.rank = env_int("RANK", 0)
        self.local_rank = env_int("LOCAL_RANK", 0)
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            if backend is None:
                import torch
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = dist
            self.backend = backend

    def barrier(self):
        if self.pg:
            if getattr(self, "backend", "") == "nccl":
                import torch
                self.pg.barrier(device_ids=[torch.cuda.current_device()])
            else:
                self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        dev = "cuda" if getattr(self, "backend", "") == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_id: str | None):
        self.gpu_id = gpu_id
        self.rows = []
        self.proc = None

    def start(self):
        cmd = ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits", "-lms", "100"]
        if self.gpu_id:
            cmd[1:1] = ["-i", self.gpu_id]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def _hbm_peak_gbs() -> float:
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0   # B200_PROFILING.md fallback


HBM_PEAK_GBS = _hbm_peak_gbs()


def workload_inputs(scale_n: int | None = None):
    c = zdgen.CONFIGS[WORKLOAD]
    n = c["n"] if scale_n is None else scale_n
    frac = n / c["n"]
    m_ins = int(round(c["insert_m"] * frac))
    m_del = int(round(c["delete_m"] * frac))
    pts = zdgen.points(c["dist"], n, c["dim"], c["seed"])
    batch = zdgen.insert_batch(m_ins, c["dim"], c["insert_seed"])
    kill = zdgen.delete_ids(n, m_del, c["delete_seed"])
    return pts, batch, kill


def config_block(extra=None):
    c = zdgen.CONFIGS[WORKLOAD]
    d = {"workload": f"{WORKLOAD}: build 10M 3D uniform [0,2^21)^3, insert 1M, delete 1M originals, "
                     f"all-points exact k=10 NN over the 10M live points",
         "n": c["n"], "dim": c["dim"], "k": K_NN, "insert_m": c["insert_m"], "delete_m": c["delete_m"],
         "leaf_max": 16, "seeds": {"base": c["seed"], "insert": c["insert_seed"], "delete": c["delete_seed"]},
         "l2": "flushed between timed steps (256 MB write, outside the timed region)",
         "parallelism": "query shards (contiguous Morton ranges), tree replicated per GPU"}
    if extra:
        d.update(extra)
    return d


# -------------------------------------------------------- oracle (CPU) legs

def oracle_step(pts, batch, kill, nthreads=0):
    """One C5 step on the CPU oracle (as it stands): build, insert, delete, knn."""
    import oracle
    t0 = time.perf_counter()
    live = oracle.LiveSet(pts)
    live.tree()                           # build (canonical tree of the base set)
    live.insert(batch)
    live.tree()                           # insert = rebuild of the live set
    live.delete(kill)
    t = live.tree()                       # delete = rebuild of the live set
    oi, od, cnt = t.knn_all(K_NN, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return dt, t.n, cnt


def cpu_baseline(sample_n: int):
    import oracle
    pts, batch, kill = workload_inputs(sample_n)
    dt, nq, cnt = oracle_step(pts, batch, kill)
    per_q = {k: v / nq for k, v in cnt.items()}
    full = sample_n == zdgen.CONFIGS[WORKLOAD]["n"]
    what = "one full C5 step" if full else f"one C5 step scaled to n={sample_n:,}"
    return {"value": nq / dt, "unit": UNIT, "cores": oracle.num_cores(), "kind": "oracle",
            "sample": f"{what} (insert {len(batch):,}, delete {len(kill):,}): 3 sequential oracle builds + "
                      f"leaf-based k=10 query of the {nq:,} live points on all cores",
            "seconds": dt, "cpu_model": cpu_model()}, per_q


def run_reference(args, D: Dist):
    if D.rank != 0:
        return
    import oracle
    n = args.ref_sample
    pts, batch, kill = workload_inputs(n)
    for _ in range(args.warmup):
        oracle_step(pts, batch, kill)
    times = []
    for _ in range(args.steps):
        dt, nq, _ = oracle_step(pts, batch, kill)
        times.append(dt)
    tot = sum(times)
    value = nq * args.steps / tot
    sample = (f"each step = full C5 step scaled to n={n:,} (insert {len(batch):,}, delete {len(kill):,}) "
              f"on the host cores")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": config_block({"reference_sample_n": n}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_cores(), "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU leg

# Algorithmic work per query, in lane-instructions: the oracle's counters (the paper's
# Alg. 3 + Alg. 2 on the same input) times the SASS cost of each operation as the k-NN
# kernel implements it (scripts/op_costs.py -> profiles/r02_op_costs.json: distance
# test per candidate, box test per child box, k-best insertion, ascent stop test).
# Fallback (no file): the survey's hand estimates.
def _op_costs():
    try:
        d = json.loads((ROOT / "profiles" / "r02_op_costs.json").read_text())["ops"]
        # the final kernel's forms where the file has them (sign-bit hit masks, packed
        # bf16 bound list), else the first round-2 forms
        pick = {k: (k + "_final" if k + "_final" in d else k) for k in ("dist", "box", "insert", "ascent")}
        return ({k: d[pick[k]]["lane_instructions"] for k in pick},
                {k: d[pick[k]]["half_rate_instructions"] for k in pick},
                "profiles/r02_op_costs.json (cuobjdump -sass of scripts/op_costs.cu; ops: " +
                ", ".join(sorted(pick.values())) + ")")
    except Exception:
        return (dict(SURVEY_OP_COSTS), dict(dist=0, box=0, insert=0, ascent=0), "SURVEY §8(d) estimates")


# SURVEY §8(d)'s hand estimates per operation (its ~2,670 thread-instructions per 3D query)
SURVEY_OP_COSTS = dict(dist=10, box=20, insert=50, ascent=15)
OP_COSTS, OP_HALF, OP_SOURCE = _op_costs()


def alu_ops_per_query(per_q: dict, costs: dict | None = None) -> float:
    c = OP_COSTS if costs is None else costs
    return (per_q["dist_evals"] * c["dist"] + per_q["box_tests"] * c["box"] +
            per_q["replacements"] * c["insert"] + per_q["ascents"] * c["ascent"])


def mix_peak_factor(per_q: dict) -> float:
    """Issue ceiling of the op mix relative to the full-rate one: half-rate
    instructions (FMNMX, HMNMX2, PRMT, VIMNMX, IMAD.WIDE: 0.5 of full rate measured,
    profiles/r01_alu_rates.json, r02_alu_rates_v2.json) occupy two issue slots' worth of their pipe."""
    tot = alu_ops_per_query(per_q)
    half = alu_ops_per_query(per_q, OP_HALF)
    return tot / (tot + half) if tot > 0 else 1.0


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


# Algorithmic bytes: build 274.6 B/pt (3D) / 270.6 (2D); insert (the
# full-rebuild model) 268 m + 24 n + 58.6 (n + m); delete 4 m + 28 n_before (records +
# alive lookups) + 24 n_after (compacted records) + 30.6 n_after (topology + boxes);
# k-NN compulsory 16 + 6.6 + 12 k B/query.
def build_bytes(n: int, dim: int) -> float:
    return (274.6 if dim == 3 else 270.6) * n


def insert_bytes(n: int, m: int) -> float:
    return 268.0 * m + 24.0 * n + 58.6 * (n + m)


def delete_bytes(n_before: int, m: int) -> float:
    n_after = n_before - m
    return 4.0 * m + 28.0 * n_before + 24.0 * n_after + 30.6 * n_after


def knn_bytes(nq: int, k: int = K_NN) -> float:
    return (16 + 6.6 + 12 * k) * nq


def load_traffic():
    """Per-launch DRAM bytes of the bench's k-NN kernel (the packet kernel at k=10, its
    longest captured launch) from the newest committed `rNN_ncu_knn_vMM.json` summary
    under profiles/ (highest round, then version; file times are not trusted)."""
    import re
    pat = re.compile(r"r(\d+)_ncu_knn_v(\d+)\.json$")
    files = []
    for p in (ROOT / "profiles").glob("r*_ncu_knn_v*.json"):
        m = pat.search(p.name)
        if m:
            files.append(((int(m.group(1)), int(m.group(2))), p))
    for _, p in sorted(files, reverse=True):
        try:
            d = json.loads(p.read_text())
            ks = [k for k in d.get("kernels", []) if "dram_bytes_per_launch" in k
                  and "knn_packet_kernel<3, 10" in k.get("kernel", "").replace("(int)", "")]
            if not ks:
                continue
            main = max(ks, key=lambda k: k.get("gpu__time_duration.sum", [0])[0])
            return main["dram_bytes_per_launch"], p.name
        except Exception:
            continue
    return None, None


def load_work_inflation(per_q):
    """K6's work against the oracle's (the round-1 verdict's inflation ratios): staged
    candidates tested per lane and post-seed hits per lane, from the newest committed
    profiling-build counters `rNN_knn_stats_vMM.jsonl` (scripts/knn_stats.py, config C3,
    which has the C5 step's point distribution), over the oracle's distance evaluations
    and k-best insertions per query."""
    import re
    pat = re.compile(r"r(\d+)_knn_stats_v(\d+)\.jsonl$")
    files = []
    for p in (ROOT / "profiles").glob("r*_knn_stats_v*.jsonl"):
        m = pat.search(p.name)
        if m:
            files.append(((int(m.group(1)), int(m.group(2))), p))
    for _, p in sorted(files, reverse=True):
        try:
            for line in p.read_text().splitlines():
                if not line.startswith("{"):
                    continue
                d = json.loads(line)
                if d.get("config") != "C3" or d.get("k") != 10:
                    continue
                cand = d["per_query"]["candidates_per_lane"]
                hits = d["per_query"]["hits"]
                return {"candidates_per_lane": cand, "oracle_dist_evals": per_q["dist_evals"],
                        "candidates_ratio": cand / per_q["dist_evals"],
                        "hits_per_lane": hits, "oracle_insertions": per_q["replacements"],
                        "hits_ratio": hits / per_q["replacements"],
                        "hit_rounds_per_packet": d["per_packet"]["rounds"],
                        "source": p.name + " (profiling build, C3) vs the oracle counters of this line"}
        except Exception:
            continue
    return None


def run_gpu(args, D: Dist):
    import torch
    import paper_2111_04182_b200 as zd

    torch.cuda.set_device(D.local_rank)
    zd.load()
    dev = torch.device("cuda", D.local_rank)
    pts_np, batch_np, kill_np = workload_inputs()
    pts = torch.from_numpy(pts_np).to(dev)
    batch = torch.from_numpy(batch_np).to(dev)
    kill = torch.from_numpy(kill_np).to(dev)
    c = zdgen.CONFIGS[WORKLOAD]
    n_live = c["n"] + c["insert_m"] - c["delete_m"]
    oi = torch.empty((n_live, K_NN), dtype=torch.int32, device=dev)
    od = torch.empty((n_live, K_NN), dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # this rank's shard of the queries: a contiguous Morton range (whole 32-query packets)
    q_lo, q_hi = zd.query_partition(n_live, D.world, D.rank)
    st = torch.cuda.current_stream()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e

    def step():
        e0 = ev()
        t = zd.zd_build(pts)
        e1 = ev()
        t.zd_insert(batch)
        e2 = ev()
        t.zd_delete(kill)
        e3 = ev()
        t.zd_set_timing(True)
        t.zd_knn_range(K_NN, q_lo, q_hi, oi, od)
        e4 = ev()
        return t, (e0, e1, e2, e3, e4)

    for _ in range(args.warmup):
        t, _ = step()
        t.zd_free()
    torch.cuda.synchronize()

    def measure():
        uuid = None
        try:
            uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
        except Exception:
            pass
        sampler = ClockSampler(uuid)
        sampler.start()
        time.sleep(0.3)
        l0 = zd.zd_kernel_launches()
        evs, knn_kernel = [], []
        D.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1)                      # L2 flush, outside the timed events
            t, e = step()
            knn_kernel.append(None)
            evs.append((t, e))
            torch.cuda.synchronize()
            knn_kernel[-1] = t.zd_get_timing()["knn"]
            t.zd_free()
        torch.cuda.synchronize()
        D.barrier()
        launches = zd.zd_kernel_launches() - l0
        clocks = sampler.stop()
        ph = np.array([[a.elapsed_time(b) for a, b in zip(e[:-1], e[1:])] for _, e in evs])
        return ph, knn_kernel, launches, clocks

    ph, knn_kernel, launches, clocks = measure()
    remeasured = False
    if set(clocks["reasons"]) & BAD_REASONS:
        remeasured = True
        ph, knn_kernel, launches, clocks = measure()

    step_ms = ph.sum(1)
    tot_ms = D.max(float(step_ms.sum()))
    ms_per_step = tot_ms / args.steps
    value = n_live * args.steps / (tot_ms / 1e3)   # one problem: the 10^7 queries, max time over ranks
    mean_ph = ph.mean(0)
    knn_ms = float(np.mean(knn_kernel))

    # ---- CPU oracle and per-config report (rank 0 at N=1), measured before the e2e
    # section: its extra streams and host threads would slow later default-stream
    # builds (observed +60 us per build), so nothing on the GPU follows it
    per_q, cpu, per_config = None, None, None
    if D.rank == 0 and D.world == 1:
        if args.cpu_baseline:
            cpu, per_q = cpu_baseline(args.cpu_sample or c["n"])
        if args.per_config:
            per_config = run_per_config(zd, dev, clocks)
    if per_q is None:   # oracle counters of 3D uniform at 10^6 (tests/test_oracle_pins.py App. A pin)
        per_q = dict(dist_evals=92.0, box_tests=45.0, ascents=9.02, replacements=23.1, evictions=13.1)

    # ---- e2e: the same step through the C ABI with pinned HOST buffers
    pts_h = torch.from_numpy(pts_np).pin_memory()
    batch_h = torch.from_numpy(batch_np).pin_memory()
    kill_h = torch.from_numpy(kill_np).pin_memory()
    oi_h = torch.empty((n_live, K_NN), dtype=torch.int32).pin_memory()
    od_h = torch.empty((n_live, K_NN), dtype=torch.int64).pin_memory()
    h2d = pts_h.numel() * 4 + batch_h.numel() * 4 + kill_h.numel() * 4
    d2h = oi_h.numel() * 4 + od_h.numel() * 8

    def e2e_step():
        e0 = ev()
        t = zd.zd_build(pts_h)
        t.zd_insert(batch_h)
        t.zd_delete(kill_h)
        if D.world == 1:
            t.zd_knn(K_NN, out_idx=oi_h, out_dist2=od_h)   # host outputs: the library stages them
        else:   # this rank's shard into device rows, then the row arrays to the host
            t.zd_knn_range(K_NN, q_lo, q_hi, oi, od)
            oi_h.copy_(oi, non_blocking=True)
            od_h.copy_(od, non_blocking=True)
        e1 = ev()
        torch.cuda.synchronize()
        t.zd_free()
        return e0.elapsed_time(e1)

    # Pipelined e2e (one GPU): two host threads, each running whole steps through the
    # public API on its own CUDA stream with its own pinned output rows (concurrent calls
    # on different handles are allowed, include/zd.h).  One step's 1.2 GB of rows going
    # over PCIe overlaps the next step's uploads and kernels; every step still copies its
    # inputs in and its rows out inside the timed region.
    n_pipe = 2 if (D.world == 1 and args.e2e_pipeline) else 1
    pipes = []
    if n_pipe == 2:
        for j in range(2):
            pipes.append({"stream": torch.cuda.Stream(),
                          "oi": oi_h if j == 0 else torch.empty_like(oi_h).pin_memory(),
                          "od": od_h if j == 0 else torch.empty_like(od_h).pin_memory()})

    def pipe_steps(j, count):
        pp = pipes[j]
        with torch.cuda.stream(pp["stream"]):
            for _ in range(count):
                t = zd.zd_build(pts_h, stream=pp["stream"])
                t.zd_insert(batch_h)
                t.zd_delete(kill_h)
                t.zd_knn(K_NN, out_idx=pp["oi"], out_dist2=pp["od"])   # returns when the rows are on the host
                t.zd_free()

    def e2e_pipelined(steps):
        from concurrent.futures import ThreadPoolExecutor
        torch.cuda.synchronize()
        e0 = ev()
        counts = [(steps + 1 - j) // 2 for j in range(2)]
        with ThreadPoolExecutor(2) as ex:
            list(ex.map(lambda j: pipe_steps(j, counts[j]), range(2)))
        for pp in pipes:
            st.wait_stream(pp["stream"])   # the end event follows both streams' last copies
        e1 = ev()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    e2e_value, e2e_tot, same = None, 0.0, None
    if args.e2e_steps > 0:   # (0: development runs, e.g. under a profiler)
        for _ in range(max(3, args.warmup)):   # warm the host-staging paths (pool growth on first use)
            e2e_step()
        if n_pipe == 2:
            e2e_pipelined(2)   # warm both streams' pools
        e2e_ms = []
        D.barrier()
        if n_pipe == 2:
            flush.fill_(1)
            e2e_ms.append(e2e_pipelined(args.e2e_steps))
        else:
            for _ in range(args.e2e_steps):
                flush.fill_(1)
                e2e_ms.append(e2e_step())
        e2e_tot = D.max(float(sum(e2e_ms)))
        e2e_value = n_live * args.e2e_steps / (e2e_tot / 1e3)
        # e2e parity spot check: host rows of this shard == the device-timed run's rows
        if D.world == 1:
            same = bool(torch.equal(oi_h, oi.cpu()) and torch.equal(od_h, od.cpu()))
        else:
            same = None

    if D.rank != 0:
        return

    # ---- roofline of the dominant kernel (k-NN): issue-bound integer/fp32 ALU work
    sm_max = clocks.get("sm_max_mhz") or 1965.0
    knn_roof = knn_roofline(per_q, n_live, knn_ms, sm_max)
    traffic, traffic_src = load_traffic()
    knn_roof.update({"kernel": "knn_packet_kernel<3,10>", "traffic": traffic, "traffic_source": traffic_src,
                     "work_inflation": load_work_inflation(per_q)})
    n_before_delete = c["n"] + c["insert_m"]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": D.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": config_block({"parallelism": f"query shards: {D.world} x contiguous Morton range, tree replicated",
                                "query_shard_rank0": [q_lo, q_hi]}),
        "phases_ms": {"build": float(mean_ph[0]), "insert": float(mean_ph[1]), "delete": float(mean_ph[2]),
                      "knn_call": float(mean_ph[3]), "knn_kernel": knn_ms},
        "build_mpts_s": c["n"] / (mean_ph[0] / 1e3) / 1e6,
        "build_roofline": hbm_roof(build_bytes(c["n"], 3), mean_ph[0], "274.6 B/pt (SURVEY §8(d))"),
        "insert_mpts_s": c["insert_m"] / (mean_ph[1] / 1e3) / 1e6,
        "insert_roofline": hbm_roof(insert_bytes(c["n"], c["insert_m"]), mean_ph[1],
                                    "268 m + 24 n + 58.6 (n+m) B (full-rebuild model, SURVEY §8(d))"),
        "delete_mpts_s": c["delete_m"] / (mean_ph[2] / 1e3) / 1e6,
        "delete_roofline": hbm_roof(delete_bytes(n_before_delete, c["delete_m"]), mean_ph[2],
                                    "4 m + 28 n_before + 24 n_after + 30.6 n_after B"),
        "knn_qps": n_live / (mean_ph[3] / 1e3),
        "roofline": knn_roof,
        "per_config": per_config,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_tot / max(1, args.e2e_steps), "matches_device_result": same,
                "pipelined_streams": n_pipe},
        "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "clocks": clocks, "remeasured": remeasured,
        "paper_context": PAPER_CONTEXT,
    }
    print(json.dumps(line), flush=True)


def hbm_roof(nbytes: float, ms: float, model: str) -> dict:
    ach = nbytes / (ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": HBM_PEAK_GBS, "unit": "GB/s", "frac": ach / HBM_PEAK_GBS,
            "algorithmic_bytes": nbytes, "bytes_model": model,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)"}


def knn_roofline(per_q: dict, nq: int, knn_ms: float, sm_max: float) -> dict:
    ops_q = alu_ops_per_query(per_q)
    achieved = ops_q * nq / (knn_ms / 1e3) / 1e12
    peak = 148 * 4 * 32 * sm_max * 1e6 / 1e12   # lane-instr/s: 148 SMs x 4 SMSPs x 32 lanes x clock
    mixf = mix_peak_factor(per_q)
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "T lane-instr/s", "frac": achieved / peak,
            "peak_mix": peak * mixf, "frac_mix": achieved / (peak * mixf),
            "ops_per_query": ops_q,
            # the same counters at SURVEY §8(d)'s hand-estimated costs (implementation-independent yardstick)
            "ops_per_query_survey_costs": alu_ops_per_query(per_q, SURVEY_OP_COSTS),
            "frac_survey_costs": alu_ops_per_query(per_q, SURVEY_OP_COSTS) * nq / (knn_ms / 1e3) / 1e12 / peak,
            "op_costs": OP_COSTS, "op_costs_half_rate": OP_HALF, "op_costs_source": OP_SOURCE,
            "counters_per_query": per_q,
            "peak_note": "full-rate issue ceiling 148 SMs x 4 SMSPs x 32 lanes x sm_max clock (B200_PROFILING.md); "
                         "peak_mix weights the op mix's half-rate share: FMNMX, HMNMX2, PRMT (profiles/r01_alu_rates.json, r02_alu_rates_v2.json)",
            "hbm_frac_compulsory": knn_bytes(nq) / (knn_ms / 1e3) / (HBM_PEAK_GBS * 1e9)}


PER_CONFIGS = ("C1", "C2", "C3", "C4a", "C4b")
C3_SHIFT = (1234567, 765432, 1048577)   # a fixed 3D shift in [0, 2^21)^3 for the C3+shift row


def run_per_config(zd, dev, clocks) -> list:
    """Per-config rows on one GPU (BASELINE.json configs[0..3]): build and k=10
    all-points throughput with roofline fractions, every row compared with the CPU
    oracle at full size (timed on all host cores), plus one-thread oracle runs for C1
    and for a 10^6-point sample of the C3 recipe."""
    import torch
    import oracle
    sm_max = clocks.get("sm_max_mhz") or 1965.0
    rows = []
    for name in PER_CONFIGS:
        cfg = zdgen.CONFIGS[name]
        n, dim = cfg["n"], cfg["dim"]
        pts_np = zdgen.config_points(name)
        pts = torch.from_numpy(pts_np).to(dev)
        oi = torch.empty((n, K_NN), dtype=torch.int32, device=dev)
        od = torch.empty((n, K_NN), dtype=torch.int64, device=dev)
        st = torch.cuda.current_stream()
        b_ms, k_ms, kk_ms = [], [], []
        for rep in range(6):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(st)
            t = zd.zd_build(pts)
            e1.record(st)
            t.zd_set_timing(True)
            t.zd_knn(K_NN, out_idx=oi, out_dist2=od)
            e2.record(st)
            torch.cuda.synchronize()
            if rep > 0:   # rep 0 warms the pool and the caches
                b_ms.append(e0.elapsed_time(e1))
                k_ms.append(e1.elapsed_time(e2))
                kk_ms.append(t.zd_get_timing()["knn"])
            t.zd_free()
        bm, km, kkm = statistics.median(b_ms), statistics.median(k_ms), statistics.median(kk_ms)
        # oracle at full size on all host cores (its build is sequential, P:235 sort + Alg. 1)
        t0 = time.perf_counter()
        T = oracle.Tree(pts_np)
        t1 = time.perf_counter()
        ri, rd, cnt = T.knn_all(K_NN)
        t2 = time.perf_counter()
        per_q = {k: v / n for k, v in cnt.items()}
        gi, gd = oi.cpu().numpy(), od.cpu().numpy()
        exact = int(np.count_nonzero(np.all(gi == ri, axis=1) & np.all(gd == rd, axis=1)))
        row = {"config": name, "n": n, "dim": dim, "dist": cfg["dist"], "k": K_NN,
               "build_ms": bm, "build_mpts_s": n / (bm / 1e3) / 1e6,
               "build_roofline": hbm_roof(build_bytes(n, dim), bm, f"{274.6 if dim == 3 else 270.6} B/pt"),
               "knn_call_ms": km, "knn_kernel_ms": kkm, "knn_qps": n / (km / 1e3),
               "knn_roofline": knn_roofline(per_q, n, kkm, sm_max),
               "bit_exact_rows": f"{exact}/{n}",
               "oracle_all_cores": {"cores": oracle.num_cores(), "build_s": t1 - t0, "knn_s": t2 - t1,
                                    "knn_qps": n / (t2 - t1), "build_plus_knn_qps": n / (t2 - t0)}}
        for key in ("knn_roofline",):   # keep the row compact
            for drop in ("op_costs", "op_costs_half_rate", "op_costs_source", "peak_note"):
                row[key].pop(drop, None)
        if name in ("C1", "C3"):
            n1 = n if name == "C1" else 1_000_000
            p1 = pts_np if name == "C1" else zdgen.config_points(name, n1)
            t0 = time.perf_counter()
            T1 = oracle.Tree(p1)
            t1 = time.perf_counter()
            T1.knn_all(K_NN, nthreads=1)
            t2 = time.perf_counter()
            row["oracle_1_thread"] = {"n": n1, "sample": "full config" if n1 == n else
                                      f"the {name} recipe at n={n1:,} (per-query work is flat in n, SURVEY App. A)",
                                      "build_s": t1 - t0, "knn_s": t2 - t1, "knn_qps": n1 / (t2 - t1)}
        rows.append(row)
        if name == "C3":   # NEXT-4: the same config with the 3D random shift (reading R31)
            sh = C3_SHIFT
            b_ms, k_ms = [], []
            for rep in range(4):
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record(st)
                t = zd.zd_build(pts, shift=sh)
                e1.record(st)
                t.zd_set_timing(True)
                t.zd_knn(K_NN, out_idx=oi, out_dist2=od)
                e2.record(st)
                torch.cuda.synchronize()
                if rep > 0:
                    b_ms.append(e0.elapsed_time(e1))
                    k_ms.append(t.zd_get_timing()["knn"])
                t.zd_free()
            gi, gd = oi.cpu().numpy(), od.cpu().numpy()
            exact = int(np.count_nonzero(np.all(gi == ri, axis=1) & np.all(gd == rd, axis=1)))
            bm, kkm = statistics.median(b_ms), statistics.median(k_ms)
            rows.append({"config": "C3+shift", "shift": list(sh), "n": n, "dim": dim, "k": K_NN,
                         "build_ms": bm, "build_mpts_s": n / (bm / 1e3) / 1e6, "knn_kernel_ms": kkm,
                         "knn_qps_kernel": n / (kkm / 1e3),
                         "bit_exact_rows_vs_unshifted_oracle": f"{exact}/{n}"})
        del pts, oi, od, T, ri, rd, gi, gd
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-e2e-pipeline", dest="e2e_pipeline", action="store_false",
                    help="e2e steps one after another instead of two overlapping host threads")
    ap.add_argument("--cpu-sample", type=int, default=0, help="C5 points for the oracle baseline (0 = full 10^7)")
    ap.add_argument("--no-per-config", dest="per_config", action="store_false")
    ap.add_argument("--ref-sample", type=int, default=1_000_000)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    D = Dist(backend="gloo" if args.impl == "reference" else None)
    try:
        if args.impl == "reference":
            run_reference(args, D)
        else:
            run_gpu(args, D)
    finally:
        D.close()


if __name__ == "__main__":
    main()
