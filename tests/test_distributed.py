"""Multi-rank host logic on CPU (gloo, world_size 2) and the block-range shard geometry.
No GPU: the per-rank compute is the oracle, which only tests/ may call."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import distributed as D


@pytest.fixture(scope="module", autouse=True)
def lib():
    from paper_1201_3018_b200 import build as B
    B.build_library()
    pcb.load()


@pytest.mark.parametrize("L,N,W_block", [(1000, 9, 40), (777, 10, 34), (5, 1, 4), (70000, 65, 1024),
                                         (1 << 22, 512, 4096), (1 << 24, 4096, 16384)])
@pytest.mark.parametrize("mode", [0, 1])
def test_shards_cover_outputs_and_inputs(L, N, W_block, mode):
    if mode == 1 and L < N:
        return
    g = O.Geometry(L, N, W_block)
    L_out = g.L_out if mode == 0 else L - N + 1
    for world in (1, 2, 3, 8, 13):
        cover = []
        for r in range(world):
            sh = D.shard(L, N, W_block, mode, r, world)
            assert sh["block_begin"] == g.P * r // world and sh["block_end"] == g.P * (r + 1) // world
            for w in range(sh["block_begin"], sh["block_end"]):      # inputs of every owned block present
                a = g.block_start(w)
                assert sh["in_begin"] <= a and min(a + W_block, L) <= sh["in_end"]
            cover.append((sh["out_begin"], sh["out_end"]))
        pos = 0
        for a, b in cover:                                            # disjoint, in order, complete
            if a == b:
                continue
            assert a == pos
            pos = b
        assert pos == L_out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker_sharded(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    L, N, W_block, Q = 20000, 33, 200, 31
    s, k = rng.laplace(0, 0.3, L), rng.uniform(-1, 1, N)
    g = O.Geometry(L, N, W_block)
    ks = O.prepare_kernel(k, g, O.ASYM2, Q)
    sh = D.shard(L, N, W_block, 0, rank, world)
    s_local = np.zeros(L)                                  # this rank only sees its input range
    s_local[sh["in_begin"]:sh["in_end"]] = s[sh["in_begin"]:sh["in_end"]]
    out = np.full(g.L_out, np.nan)
    for w in range(sh["block_begin"], sh["block_end"]):
        br = O.process_block(s_local, w, g, ks, Q)
        o0, n = g.kept(w)
        lo = g.block_start(w) + o0
        n = min(n, g.L_out - lo)
        out[lo:lo + n] = br.out[:n]
    piece = out[sh["out_begin"]:sh["out_end"]].copy()
    parts = [None] * world
    dist.all_gather_object(parts, piece)
    if rank == 0:
        full = np.concatenate(parts)
        ref = O.conv_pipeline(s, k, W_block, O.ASYM2, Q).out
        q.put(bool(np.array_equal(full, ref)))
    dist.destroy_process_group()


def test_gloo_block_sharded_pipeline_equals_single_run():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sharded, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


def _cpu_best_match(out, n, scores=None, lags=None, cand=None, first=0):
    """Stand-in for the conv_best_match kernel on CPU: the C17 rule written out."""
    rows = cand.view(-1, 3).tolist() if cand is not None else \
        [[float(scores[i]), float(lags[i]), float(first + i)] for i in range(n)]
    best = None
    for sc, lg, idx in rows[:n]:
        if best is None or sc > best[0] or (sc == best[0] and idx < best[2]):
            best = [sc, lg, idx]
    out.copy_(torch.tensor(best, dtype=torch.float64))


def _worker_gather(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 11
    a, b = D.signal_range(n, rank, world)
    scores = torch.tensor([float((i * 7) % 5) for i in range(a, b)], dtype=torch.float64)  # ties: max 4 at i=2,7
    lags = torch.tensor([100 + i for i in range(a, b)], dtype=torch.int64)
    best = D.gather_best_match(scores, lags, a, reduce=_cpu_best_match)
    q.put((rank, D.best_match_tuple(best)))
    dist.destroy_process_group()


def test_gloo_score_gather_ties_to_lowest_signal():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_gather, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res[0] == res[1] == (2, 4.0, 102)


@pytest.mark.slow
def test_bench_launcher_relaunches_with_torchrun():
    """bench.py --gpus 2 outside torchrun re-launches itself through torch.distributed.run (one
    process per rank); the reference arm runs on rank 0 and reports n_gpus = the world size."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "1", "--workload", "cfg1"], capture_output=True, text=True,
                         timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
