"""Sharded assembly on one B200: the per-shard fixed-point partials summed as
integers give a system bit-identical to the unsharded run (the property the
NCCL all-reduce relies on across 1/2/4/8 GPUs)."""
import os
import socket

import numpy as np
import pytest

import paper_2302_07499_b200 as P
from paper_2302_07499_b200 import distributed as D
from tests.helpers import SEED, U2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strat,mc,nshard", [("nocaps", 1, 3), ("fullcaps", 8, 2),
                                             ("barycenter", 1, 4)])
def test_shards_sum_to_single_gpu_bitwise(strat, mc, nshard):
    import torch
    m = P.generate_mesh(3, 6, 0.34, jitter_seed=5)
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    s = P.Session(t, 0.34, strat, "moment2", U2, seed=SEED, mc_samples=mc)
    s.run()
    want = s.download()
    KI = s.interior_count
    Vsum = Rsum = None
    for r in range(nshard):
        lo, hi = D.shard_range(KI, r, nshard)
        s.run_shard(lo, hi)
        vv, rv = s.partials()
        V = torch.as_tensor(vv, device="cuda").cpu().numpy().copy()
        R = torch.as_tensor(rv, device="cuda").cpu().numpy().copy()
        with np.errstate(over="ignore"):
            Vsum = V if Vsum is None else Vsum + V
        Rsum = R if Rsum is None else Rsum + R
    vv, rv = s.partials()
    torch.as_tensor(vv, device="cuda").copy_(torch.from_numpy(Vsum))
    torch.as_tensor(rv, device="cuda").copy_(torch.from_numpy(Rsum))
    torch.cuda.synchronize()
    blocks = []
    for r in range(nshard):
        r0, r1 = D.shard_range(s.unknowns, r, nshard)
        s.finalize(r0, r1)
        blocks.append(s.download_rows(r0, r1))
    got = D.concat_csr(blocks)
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        assert np.array_equal(got[k], want[k]), (strat, k)


def test_assemble_distributed_world1_nccl():
    import torch
    import torch.distributed as dist
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        m = P.generate_mesh(3, 4, 0.3)
        t = P.ElementTable(m["coords"], m["cells"], m["region"])
        s = P.Session(t, 0.3, "fullcaps", "moment2", U2, seed=SEED, mc_samples=8)
        full, st = D.assemble_distributed(s)
        ref, _ = P.assemble(t, 0.3, "fullcaps", "moment2", U2, seed=SEED, mc_samples=8)
        for k in ("row_ptr", "col_idx", "values", "rhs"):
            assert np.array_equal(full[k], ref[k]), k
        assert st["shard_pairs"] == st["element_pairs"]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("strat,mc,nshard", [("nocaps", 1, 3), ("fullcaps", 8, 2),
                                             ("barycenter", 1, 4)])
def test_sharded_pairs_sum_to_single_gpu_bitwise(strat, mc, nshard):
    # nshard "ranks" as nshard sessions on one GPU: each builds only its own
    # outer elements' pairs; the concatenated lists are installed everywhere
    # (what gather_pairs does over NCCL), each integrates its range, and the
    # integer partials summed give the unsharded system bit for bit
    import torch
    m = P.generate_mesh(3, 6, 0.34, jitter_seed=5)
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    ref = P.Session(t, 0.34, strat, "moment2", U2, seed=SEED, mc_samples=mc)
    ref.run()
    want = ref.download()
    KI = ref.interior_count
    ranks = [P.Session(t, 0.34, strat, "moment2", U2, seed=SEED, mc_samples=mc)
             for _ in range(nshard)]
    counts, partners, total = [], [], 0
    for r, s in enumerate(ranks):
        lo, hi = D.shard_range(KI, r, nshard)
        n = s.pairs_shard(lo, hi)
        cv, pv = s.pairs_shard_out()
        counts.append(torch.as_tensor(cv, device="cuda").clone())
        partners.append(torch.as_tensor(pv, device="cuda").clone() if n else
                        torch.zeros(0, dtype=torch.int32, device="cuda"))
        total += n
    allc, allp = torch.cat(counts), torch.cat(partners)
    assert total == ref.stats.element_pairs
    Vsum = Rsum = None
    for r, s in enumerate(ranks):
        lo, hi = D.shard_range(KI, r, nshard)
        s.pairs_install(allc, allp, total)
        st = s.run_shard(lo, hi)
        assert st.element_pairs == total
        vv, rv = s.partials()
        V = torch.as_tensor(vv, device="cuda").cpu().numpy().copy()
        R = torch.as_tensor(rv, device="cuda").cpu().numpy().copy()
        with np.errstate(over="ignore"):
            Vsum = V if Vsum is None else Vsum + V
        Rsum = R if Rsum is None else Rsum + R
    s0 = ranks[0]
    vv, rv = s0.partials()
    torch.as_tensor(vv, device="cuda").copy_(torch.from_numpy(Vsum))
    torch.as_tensor(rv, device="cuda").copy_(torch.from_numpy(Rsum))
    torch.cuda.synchronize()
    s0.finalize(0, s0.unknowns)
    got = s0.download_rows(0, s0.unknowns)
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        assert np.array_equal(got[k], want[k]), (strat, k)


def test_interleaved_sessions_on_one_device():
    # the device parameter block is per device: a session whose pairs were
    # built before another session ran must rebind its own state for
    # run_shard / finalize (different meshes, so a stale binding would show)
    import torch
    mA = P.generate_mesh(3, 5, 0.34, jitter_seed=3)
    tA = P.ElementTable(mA["coords"], mA["cells"], mA["region"])
    mB = P.generate_mesh(3, 6, 0.3)
    tB = P.ElementTable(mB["coords"], mB["cells"], mB["region"])
    a = P.Session(tA, 0.34, "fullcaps", "moment2", U2, seed=SEED, mc_samples=8)
    a.run()
    want = a.download()
    b = P.Session(tB, 0.3, "nocaps", "moment2", U2, seed=SEED)
    KI = a.interior_count
    n = a.pairs_shard(0, KI)
    cv, pv = a.pairs_shard_out()
    counts = torch.as_tensor(cv, device="cuda").clone()
    partners = torch.as_tensor(pv, device="cuda").clone()
    b.run()                      # another session binds its state in between
    a.pairs_install(counts, partners, n)
    a.run_shard(0, KI)
    b.run()
    a.finalize(0, a.unknowns)
    got = a.download_rows(0, a.unknowns)
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        assert np.array_equal(got[k], want[k]), k


def test_session_reset_equals_fresh_session():
    # the workspace reuse behind repeated one-shot calls: a session reloaded
    # with another mesh gives that mesh's system bit for bit
    mA = P.generate_mesh(3, 5, 0.34, jitter_seed=3)
    tA = P.ElementTable(mA["coords"], mA["cells"], mA["region"])
    mB = P.generate_mesh(3, 6, 0.3)
    tB = P.ElementTable(mB["coords"], mB["cells"], mB["region"])
    s = P.Session(tA, 0.3, "fullcaps", "moment2", U2, seed=SEED, mc_samples=8)
    s.run()
    s.reset(tB)
    s.run()
    got = s.download()
    f = P.Session(tB, 0.3, "fullcaps", "moment2", U2, seed=SEED, mc_samples=8)
    f.run()
    want = f.download()
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        assert np.array_equal(got[k], want[k]), k
    # the device pair list equals the host download
    import torch
    pd, ph = f.pairs_device(), f.pairs()
    assert np.array_equal(torch.as_tensor(pd["offsets"], device="cuda").cpu().numpy(),
                          ph["offsets"])
    assert np.array_equal(torch.as_tensor(pd["partner"], device="cuda").cpu().numpy(),
                          ph["partner"])
    assert np.array_equal(torch.as_tensor(pd["info"], device="cuda").cpu().numpy(), ph["info"])


def _owner_computes(t, strat, mc, nrank, delta=0.34, chunk_env=None):
    """nrank "ranks" as sessions on one GPU running the owner-computes plan
    (distributed.device_step without the collectives): local pairs / pattern /
    integration per rank, records routed by destination in rank order (what
    the all-to-all delivers), merged finalize of each row block."""
    import torch
    ranks = [P.Session(t, delta, strat, "moment2", U2, seed=SEED, mc_samples=mc)
             for _ in range(nrank)]
    KI, U = ranks[0].interior_count, ranks[0].unknowns
    bounds = D.row_bounds(U, nrank)
    sent, pairs = [], 0
    for r, s in enumerate(ranks):
        lo, hi = D.shard_range(KI, r, nrank)
        st = s.run_local(lo, hi)
        pairs += st.element_pairs
        k, w, kc = s.halo_records(bounds)
        ri, rv, rc = s.rhs_records(bounds)
        k, w = torch.as_tensor(k, device="cuda").clone(), torch.as_tensor(w, device="cuda").clone()
        ri, rv = torch.as_tensor(ri, device="cuda").clone(), torch.as_tensor(rv, device="cuda").clone()
        ko, ro = np.concatenate([[0], np.cumsum(kc)]), np.concatenate([[0], np.cumsum(rc)])
        sent.append([(k[ko[d]:ko[d + 1]], w[4 * ko[d]:4 * ko[d + 1]], ri[ro[d]:ro[d + 1]],
                      rv[32 * ro[d]:32 * ro[d + 1]]) for d in range(nrank)])
    blocks = []
    for d, s in enumerate(ranks):
        parts = [sent[r][d] for r in range(nrank)]
        keys, words, ridx, rvals = (torch.cat([p[i] for p in parts]) for i in range(4))
        s.finalize_merged(bounds[d], bounds[d + 1], keys, words, ridx, rvals)
        blocks.append(s.download_rows(bounds[d], bounds[d + 1]))
    for s in ranks:
        s.close()
    return D.concat_csr(blocks), pairs


@pytest.mark.parametrize("strat,mc,nrank", [("nocaps", 1, 3), ("fullcaps", 8, 2),
                                            ("barycenter", 1, 4), ("fullcaps", 8, 1)])
def test_owner_computes_equals_single_gpu_bitwise(strat, mc, nrank):
    m = P.generate_mesh(3, 6, 0.34, jitter_seed=5)
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    ref = P.Session(t, 0.34, strat, "moment2", U2, seed=SEED, mc_samples=mc)
    ref.run()
    want = ref.download()
    got, pairs = _owner_computes(t, strat, mc, nrank)
    assert pairs == ref.stats.element_pairs
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        assert np.array_equal(got[k], want[k]), (strat, nrank, k)


def test_owner_computes_eight_ranks_lattice():
    # thin slabs (N = 8 lattice, 8 ranks: one cube layer of outer elements
    # each, delta = 2h): every rank's rows take records from several others
    m = P.generate_mesh(3, 8, 0.25)
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    ref = P.Session(t, 0.25, "fullcaps", "moment2", U2, seed=SEED, mc_samples=16)
    ref.run()
    want = ref.download()
    got, _ = _owner_computes(t, "fullcaps", 16, 8, delta=0.25)
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        assert np.array_equal(got[k], want[k]), k


def test_owner_computes_chunked_units():
    # the local path through the chunked units / combine (several chunks per
    # rank, two alternating unit-buffer sets): same system bit for bit
    code = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2302_07499_b200 as P
from tests.test_gpu_distributed import _owner_computes
from tests.helpers import SEED, U2
m = P.generate_mesh(3, 6, 0.34, jitter_seed=5)
t = P.ElementTable(m["coords"], m["cells"], m["region"])
got, _ = _owner_computes(t, "fullcaps", 8, 3)
np.savez(sys.argv[2], **got)
"""
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "c.npz")
        env = dict(os.environ, NLFEM_PAIRS_PER_CHUNK="2000")
        subprocess.run([sys.executable, "-c", code, root, out], env=env, cwd=root, check=True,
                       timeout=600)
        got = np.load(out)
        m = P.generate_mesh(3, 6, 0.34, jitter_seed=5)
        t = P.ElementTable(m["coords"], m["cells"], m["region"])
        ref = P.Session(t, 0.34, "fullcaps", "moment2", U2, seed=SEED, mc_samples=8)
        ref.run()
        want = ref.download()
        for k in ("row_ptr", "col_idx", "values", "rhs"):
            assert np.array_equal(got[k], want[k]), k
