"""CPU, world_size 2 over gloo: the replica (N>1) host logic of bench.py —
barrier, max-over-ranks device time, summed proposals, rank-0-only output,
and the reference arm exiting 0 without work on ranks > 0."""
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    w, r, local, dist = bench.dist_init()
    assert (w, r) == (ws, rank) and dist.get_backend() == "gloo"
    bench.barrier(dist)
    t = bench.reduce_max(dist, 10.0 + rank)       # per-rank device ms
    n = bench.reduce_sum(dist, 1000 * (rank + 1))  # per-rank proposals
    out[rank] = (t, n)
    dist.destroy_process_group()


def test_replica_reductions_gloo():
    ws = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    for r in range(ws):
        assert out[r] == (11.0, 3000.0)


def test_reference_arm_nonzero_rank_exits_clean():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1", MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(_free_port()))
    # rank 1 of a 2-rank reference run must exit 0 without doing work; it joins
    # the process group, so run rank 0 alongside it
    env0 = dict(env, RANK="0", LOCAL_RANK="0")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
           "--steps", "1", "--warmup", "3", "--ref-seconds", "0.3", "--config", "0"]
    p0 = subprocess.Popen(cmd, env=env0, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    p1 = subprocess.Popen(cmd, env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    o1, e1 = p1.communicate(timeout=600)
    o0, e0 = p0.communicate(timeout=600)
    assert p1.returncode == 0, e1
    assert o1.strip() == ""
    assert p0.returncode == 0, e0
    import json
    line = json.loads(o0.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    if "unavailable" not in line:
        assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "reference"
        # the reference arm builds its world with the reference's generator and
        # never loads the engine
        assert line["detail"]["engine_imported"] is False
