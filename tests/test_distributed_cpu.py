"""Multi-rank host logic on CPU with the gloo backend (world size 2):
shard splits, the exact integer reduction of fixed-point partials, and the
all-gather of CSR row blocks (paper_2302_07499_b200/distributed.py)."""
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
        # exact integer reduction with wrap-around (two's complement words)
        rng = np.random.default_rng(100 + rank)
        part = rng.integers(-2**62, 2**62, size=1000, dtype=np.int64)
        V = torch.from_numpy(part.copy())
        R = torch.zeros(8, dtype=torch.float64)
        R[rank] = 1.5 + rank  # each rhs partial written by one rank only
        D.allreduce_partials(V, R)
        parts = [np.random.default_rng(100 + r).integers(-2**62, 2**62, size=1000, dtype=np.int64)
                 for r in range(world)]
        with np.errstate(over="ignore"):
            want = parts[0].copy()
            for p in parts[1:]:
                want = want + p
        ok_reduce = np.array_equal(V.numpy(), want)
        ok_rhs = R[:world].tolist() == [1.5 + r for r in range(world)]
        q.put((rank, ok_gather, ok_reduce, ok_rhs))
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


class _FakePairsSession:
    """Stand-in for Session's sharded-pair API: outer element i has (i % 5) + 1
    partners with ids 1000 * i + j."""

    def __init__(self, ki):
        self.ki = ki
        self.installed = None

    def _lists(self, lo, hi):
        counts = np.array([(i % 5) + 1 for i in range(lo, hi)], np.int32)
        partners = np.array([1000 * i + j for i in range(lo, hi) for j in range((i % 5) + 1)],
                            np.int32)
        return counts, partners

    def pairs_shard(self, lo, hi):
        self._c, self._p = self._lists(lo, hi)
        return len(self._p)

    def pairs_shard_out(self):
        return self._c, self._p

    def pairs_install(self, counts, partners, total, stream=None):
        self.installed = (np.asarray(counts).copy(), np.asarray(partners).copy(), total)


def _pairs_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ki = 23
        s = _FakePairsSession(ki)
        lo, hi = D.shard_range(ki, rank, world)
        total = D.gather_pairs(s, lo, hi, device="cpu")
        wc, wp = s._lists(0, ki)
        c, p, t = s.installed
        q.put((rank, t == total == len(wp), np.array_equal(c, wc), np.array_equal(p, wp)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_pairs_concatenates_in_outer_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pairs_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for (_, a, b, c) in res for ok in (a, b, c)), res
