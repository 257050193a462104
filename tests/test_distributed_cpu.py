"""Multi-rank host logic on CPU with the gloo backend (world size 2):
shard splits, the owner-computes record exchange (all-to-all of the halo
records, counts first) and the all-gathers of the row blocks
(paper_2302_07499_b200/distributed.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2302_07499_b200 import distributed as D


def test_shard_range_covers_contiguously():
    for n in (0, 1, 7, 3072, 5308416):
        for w in (1, 2, 3, 8):
            parts = [D.shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_shard_by_weight_balances():
    rng = np.random.default_rng(0)
    w = rng.integers(100, 2000, size=1000)
    off = np.concatenate([[0], np.cumsum(w)])
    parts = [D.shard_by_weight(off, r, 4) for r in range(4)]
    assert parts[0][0] == 0 and parts[-1][1] == 1000
    loads = [off[b] - off[a] for a, b in parts]
    assert max(loads) <= off[-1] / 4 + w.max()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _csr(n, seed):
    rng = np.random.default_rng(seed)
    rows = [np.sort(rng.choice(n, size=rng.integers(1, 6), replace=False)) for _ in range(n)]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)
    return {"row_ptr": rp, "col_idx": np.concatenate(rows).astype(np.int32),
            "values": rng.standard_normal(rp[-1]), "rhs": rng.standard_normal(n)}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = _csr(37, 3)
        r0, r1 = D.shard_range(37, rank, world)
        s0, s1 = full["row_ptr"][r0], full["row_ptr"][r1]
        block = {"row_ptr": full["row_ptr"][r0:r1 + 1] - s0, "col_idx": full["col_idx"][s0:s1],
                 "values": full["values"][s0:s1], "rhs": full["rhs"][r0:r1]}
        got = D.allgather_csr(block)
        ok_gather = all(np.array_equal(got[k], full[k]) for k in full)
        # variable-length all-gather (the row-block gather of device_step)
        mine = torch.arange(3 + 4 * rank, dtype=torch.int64) + 100 * rank
        g = D.allgather_var(mine, device=torch.device("cpu")).numpy()
        want = np.concatenate([np.arange(3 + 4 * r) + 100 * r for r in range(world)])
        ok_var = np.array_equal(g, want)
        q.put((rank, ok_gather, ok_var, True))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_reduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for (_, a, b, c) in res for ok in (a, b, c)), res


def _records(rank, world, dest):
    """Rank `rank`'s records for rank `dest`: (key, 4 words) with key
    = row << 32 | col, rows in dest's block, count 2 + rank + dest."""
    n = 2 + rank + dest
    keys = (np.int64(dest) << 32) + 1000 * rank + np.arange(n, dtype=np.int64)
    words = np.arange(4 * n, dtype=np.int64) * (rank + 1) - 7 * dest
    return keys, words


def _exchange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ks, ws = zip(*[_records(rank, world, d) for d in range(world)])
        cnt = np.array([len(k) for k in ks], np.int64)
        # rhs records: one per destination (position, 32 doubles)
        ridx = np.array([10 * rank + d for d in range(world)], np.int32)
        rvals = np.repeat(ridx.astype(np.float64), 32) + 0.5
        got = D.exchange_records(
            {"keys": (torch.from_numpy(np.concatenate(ks)), 1),
             "words": (torch.from_numpy(np.concatenate(ws)), 4),
             "ridx": (torch.from_numpy(ridx), 1), "rvals": (torch.from_numpy(rvals), 32)},
            {"keys": cnt, "words": cnt, "ridx": np.ones(world, np.int64),
             "rvals": np.ones(world, np.int64)}, device=torch.device("cpu"))
        wk = np.concatenate([_records(r, world, rank)[0] for r in range(world)])
        ww = np.concatenate([_records(r, world, rank)[1] for r in range(world)])
        wi = np.array([10 * r + rank for r in range(world)], np.int32)
        ok = (np.array_equal(got["keys"].numpy(), wk) and np.array_equal(got["words"].numpy(), ww)
              and np.array_equal(got["ridx"].numpy(), wi)
              and np.array_equal(got["rvals"].numpy(), np.repeat(wi.astype(np.float64), 32) + 0.5))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_halo_records_reach_their_owners():
    # the owner-computes exchange (device_step step 2): every rank's records
    # for rank d arrive at d, concatenated in sender order, counts first
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_row_bounds_split_unknowns():
    for u in (0, 5, 857375):
        for w in (1, 2, 8):
            b = D.row_bounds(u, w)
            assert b[0] == 0 and b[-1] == u and len(b) == w + 1
            assert all(b[i] <= b[i + 1] for i in range(w))
