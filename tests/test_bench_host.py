"""Host-side logic of bench.py on CPU: the multi-rank plumbing (gloo, world_size 2),
the reference arm's JSON contract, and the workload recipe."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    D = bench.Dist(backend="gloo")
    D.barrier()
    m = D.max(1.5 + rank)
    D.barrier()
    q.put((rank, m))
    D.close()


def test_dist_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res == [(0, 2.5), (1, 2.5)]


def test_workload_recipe_scaled():
    pts, batch, kill = bench.workload_inputs(50_000)
    assert pts.shape == (50_000, 3) and batch.shape == (5_000, 3) and kill.shape == (5_000,)
    assert np.array_equal(pts, bench.zdgen.uniform(50_000, 3, 6))
    assert kill.max() < 50_000 and np.unique(kill).size == kill.size


def test_alu_ops_model():
    per_q = dict(dist_evals=10, box_tests=1, ascents=1, replacements=1)
    assert bench.alu_ops_per_query(per_q) == 10 * 9 + 22 + 30 + 15


def _check_line(line):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_reference_arm_single():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--ref-sample", "20000"], capture_output=True, text=True,
                         timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    _check_line(json.loads(lines[0]))


def test_reference_arm_torchrun_two_ranks():
    port = _free_port()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                          "--ref-sample", "10000"], capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1                       # rank 0 alone prints
    _check_line(json.loads(lines[0]))
