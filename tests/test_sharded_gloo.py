"""The N > 1 (sequence-sharded) host path on CPU: world_size-2 gloo process
group, each rank owning a contiguous token range of every head. Ranks scan
their shard (oracle scores), all-gather the per-head score histograms (the
collective bench.py runs over NCCL), derive the plan with the C-ABI's host
planner, select locally, and the rank-order concatenation must equal the
reference's top_k_indices over the whole cache. The log-sum-exp combine of
per-rank attention partials is checked against one-shot attention."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    from oracle_lib import Oracle
    from paper_2508_19740_b200 import capi

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    rng = np.random.default_rng(7)
    H, N, W = 4, 6000, 4
    L = 32 * W
    codes = rng.integers(0, 2**32, (H, N, W), dtype=np.uint64).astype(np.uint32)
    codes[1] = codes[1][rng.integers(0, 3, N)]  # ties straddling the shard cut
    q = codes[:, 11].copy()
    k = 777
    lo, hi = rank * N // world, (rank + 1) * N // world
    hist = np.zeros((H, L + 1), np.int64)
    local_scores = []
    for h in range(H):
        s = orc.nxor_scores(q[h], np.ascontiguousarray(codes[h, lo:hi]))
        local_scores.append(s)
        hist[h] = np.bincount(s, minlength=L + 1)
    gathered = [torch.zeros((H, L + 1), dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(hist))
    all_hist = np.stack([g.numpy() for g in gathered]).astype(np.uint32)  # [R][H][L+1]
    sel = []
    for h in range(H):
        pl = capi.plan_shard_host(all_hist[:, h, :], rank, k)
        s = local_scores[h]
        gt = np.nonzero(s > pl["T"])[0]
        eq = np.nonzero(s == pl["T"])[0][: pl["take_eq"]]
        mine = np.sort(np.concatenate([gt, eq])) + lo
        assert len(mine) == pl["count"]
        sel.append((pl["offset"], mine))
    # attention partials (m, l, o) per rank over its selected rows, combined
    d = 16
    Kc = np.random.default_rng(1).standard_normal((N, d)).astype(np.float64)
    Vc = np.random.default_rng(2).standard_normal((N, d)).astype(np.float64)
    qv = np.random.default_rng(3).standard_normal(d)
    rows = sel[0][1]
    if len(rows):
        lg = Kc[rows] @ qv
        m = lg.max()
        w = np.exp(lg - m)
        part = np.concatenate([[m, w.sum()], w @ Vc[rows]])
    else:
        part = np.concatenate([[-np.inf, 0.0], np.zeros(d)])
    parts = [torch.zeros(d + 2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(part))
    objs = [None] * world
    dist.all_gather_object(objs, [(off, m.tolist()) for off, m in sel])
    if rank == 0:
        P = np.stack([p.numpy() for p in parts])
        M = P[:, 0].max()
        sc = np.where(np.isfinite(P[:, 0]), np.exp(P[:, 0] - M), 0.0)
        out = (sc[:, None] * P[:, 2:]).sum(0) / (sc * P[:, 1]).sum()
        result_q.put((objs, out))
    dist.destroy_process_group()


def test_sequence_sharded_two_ranks_gloo(oracle):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    qres = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, qres)) for r in range(world)]
    for p in procs:
        p.start()
    objs, out = qres.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    H, N, W = 4, 6000, 4
    codes = rng.integers(0, 2**32, (H, N, W), dtype=np.uint64).astype(np.uint32)
    codes[1] = codes[1][rng.integers(0, 3, N)]
    q = codes[:, 11].copy()
    want = oracle.retrieve_batch(codes, q, np.full(H, N, np.uint32), 777)
    for h in range(H):
        cat = np.concatenate([np.asarray(objs[r][h][1], np.uint32) for r in range(world)])
        assert np.array_equal(cat, want[h])
        assert objs[0][h][0] == 0 and objs[1][h][0] == len(objs[0][h][1])
    # combine == one-shot softmax attention over all selected rows of head 0
    d = 16
    Kc = np.random.default_rng(1).standard_normal((N, d))
    Vc = np.random.default_rng(2).standard_normal((N, d))
    qv = np.random.default_rng(3).standard_normal(d)
    rows = want[0]
    lg = Kc[rows] @ qv
    w = np.exp(lg - lg.max())
    ref = (w @ Vc[rows]) / w.sum()
    assert np.abs(out - ref).max() < 1e-12
