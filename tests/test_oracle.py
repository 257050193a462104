"""The CPU oracle (oracle/restated.cpp) pinned against the reference.

Mode R must reproduce the unmodified reference bit for bit: against the
committed golden fixtures (generated from oracle/_ref by
tests/golden/make_golden.py) everywhere, and against the live reference
library when it is present.  Mode P (the GPU's Philox stream) shares every
line except the sampler."""
import numpy as np
import pytest

import paper_2302_07499_b200 as P
from oracle import port, ref
from tests.helpers import SEED, U2, golden_names, load_golden, rhs_rel_err, row_rel_err, same_pattern


def _table(g):
    return P.ElementTable(g["coords"], g["cells"], g["region"])


def _run(table, delta, strat, mc, sampler, threads=0):
    return port.assemble(table, delta, strat, P.kernel_constant(delta, "moment2"),
                         P.forcing_terms(delta, U2, "moment2"), P.normalize_terms(U2),
                         seed=SEED, mc_samples=mc, sampler=sampler, threads=threads)


def test_philox_known_answers():
    # Random123 Philox4x32-10 KATs
    assert [hex(x) for x in port.philox([0, 0, 0, 0], (0, 0))] == \
        ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    assert [hex(x) for x in port.philox([0xFFFFFFFF] * 4, (0xFFFFFFFF, 0xFFFFFFFF))] == \
        ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]
    assert [hex(x) for x in port.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                                        (0xA4093822, 0x299F31D0))] == \
        ["0xd16cfe09", "0x94fdcceb", "0x5001e420", "0x24126ea1"]


def _philox_py(ctr, k0, k1, rounds):
    """Philox4x32-R in plain Python (Salmon et al. 2011; Random123 constants)."""
    M = 0xFFFFFFFF
    c0, c1, c2, c3 = ctr
    for _ in range(rounds):
        p0, p1 = 0xD2511F53 * c0, 0xCD9E8D57 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & M, p1 & M, ((p0 >> 32) ^ c3 ^ k1) & M, p0 & M
        k0, k1 = (k0 + 0x9E3779B9) & M, (k1 + 0xBB67AE85) & M
    return [c0, c1, c2, c3]


def test_mc_stream_is_philox4x32_7():
    # the 3D stream's words are Philox4x32-7 of (T, T', q | sub << 2, 2j + c)
    # under key (seed lo, seed hi), cut into 21-bit fields as the header says;
    # the 10-round function under it is pinned by the Random123 KATs above
    assert _philox_py([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], 0xA4093822,
                      0x299F31D0, 10) == [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]
    seed, T, Tp, q, sub = 0x0123456789ABCDEF, 77, 123456, 3, 2
    f = port.mc_fields(seed, T, Tp, q, sub, 5, 3)
    for b in range(3):
        j = 5 + b
        W = sum((_philox_py([T, Tp, q | (sub << 2), 2 * j + c], seed & 0xFFFFFFFF, seed >> 32, 7)
                 for c in range(2)), [])
        for i in range(4):
            w = W[4 * (i >> 1):4 * (i >> 1) + 4]
            if i % 2 == 0:
                want = [w[t] >> 11 for t in range(3)]
            else:
                want = [((w[t] & 0x7FF) << 10) | ((w[3] >> (22 - 10 * t)) & 0x3FF) for t in range(3)]
            assert list(f[4 * b + i]) == want, (b, i)


def test_mc_stream_uniform_and_independent():
    # statistical sanity of the 7-round stream over the counter patterns the
    # kernel uses: consecutive blocks, neighbouring inner elements, the quad
    # points and sub-simplices of one item.  Each coordinate (even and odd
    # samples separately) chi-square over 64 bins, correlations between the
    # three fields of a sample and between consecutive samples, and the sorted
    # spacings' means (1/4, 1/2, 3/4: a uniform point in the tetrahedron)
    from scipy import stats
    F = np.concatenate([port.mc_fields(SEED, 1000 + t, 5000 + tp, q, sub, 0, 256)
                        for t in range(4) for tp in range(4) for q in range(4) for sub in range(3)])
    U = (F.astype(np.float64) + 0.5) / 2.0**21                    # (196608, 3)
    for par in (0, 1):
        for c in range(3):
            h = np.bincount((F[par::2, c] >> 15).astype(np.int64), minlength=64)
            assert stats.chisquare(h).pvalue > 1e-4, (par, c)
    n = len(U)
    for a, b in ((0, 1), (0, 2), (1, 2)):
        assert abs(np.corrcoef(U[:, a], U[:, b])[0, 1]) < 5.0 / np.sqrt(n)
    for c in range(3):
        assert abs(np.corrcoef(U[:-1, c], U[1:, c])[0, 1]) < 5.0 / np.sqrt(n)
    Us = np.sort(U, axis=1).mean(axis=0)
    assert np.allclose(Us, [0.25, 0.5, 0.75], atol=5.0 * 0.25 / np.sqrt(n))


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("strat", ["inside", "overlap", "barycenter", "nocaps", "approxcaps",
                                   "fullcaps"])
def test_mode_r_matches_reference_golden(name, strat):
    g = load_golden(name)
    o = _run(_table(g), float(g["delta"]), strat, int(g["mc_samples"]), "R", threads=2)
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        assert np.array_equal(o[k], g[f"{strat}_{k}"]), (name, strat, k)
    assert [o["mc_samples"], o["mc_hits"]] == list(g[f"{strat}_mc"])


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_mode_r_matches_live_reference():
    m = P.generate_mesh(3, 5, 0.3, jitter_seed=3)
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    r = ref.Problem(m["coords"], m["cells"], m["region"])
    for strat, mc in (("inside", 1), ("overlap", 1), ("nocaps", 1), ("approxcaps", 1),
                      ("fullcaps", 12)):
        o = _run(t, 0.3, strat, mc, "R")
        s = r.assemble(0.3, strat, U2, threads=3, seed=SEED, mc_samples=mc)
        for k in ("row_ptr", "col_idx", "values", "rhs"):
            assert np.array_equal(o[k], s[k]), (strat, k)
        assert (o["mc_samples"], o["mc_hits"]) == (s["mc_samples"], s["mc_hits"])


def test_mode_p_same_regions_and_thread_invariant():
    g = load_golden("lat4_d030")
    t = _table(g)
    a = _run(t, 0.3, "fullcaps", 16, "P", threads=1)
    b = _run(t, 0.3, "fullcaps", 16, "P", threads=5)
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        assert np.array_equal(a[k], b[k])
    assert same_pattern(a, {"row_ptr": g["fullcaps_row_ptr"], "col_idx": g["fullcaps_col_idx"]})
    # same Monte Carlo regions as the reference: identical draw count
    assert a["mc_samples"] == int(g["fullcaps_mc"][0])
    hit_ref = int(g["fullcaps_mc"][1]) / int(g["fullcaps_mc"][0])
    assert abs(a["mc_hits"] / a["mc_samples"] - hit_ref) < 0.01


def test_mode_p_solution_error_close_to_reference():
    g = load_golden("lat6_d025")
    t = _table(g)
    o = _run(t, 0.25, "fullcaps", 8, "P")
    sol = port.solve_l2(t, o, U2)
    assert sol["converged"]
    assert abs(sol["l2"] / float(g["fullcaps_l2"]) - 1) < 0.01


def test_oracle_l2_matches_reference_harness():
    g = load_golden("lat4_d030")
    t = _table(g)
    s = {k: g[f"nocaps_{k}"] for k in ("row_ptr", "col_idx", "values", "rhs")}
    sol = port.solve_l2(t, s, U2)
    assert abs(sol["l2"] - float(g["nocaps_l2"])) <= 1e-9 * float(g["nocaps_l2"])


def test_ball_exits_mesh():
    m = P.generate_mesh(3, 4, 0.25)   # layer of 1 cell = 0.25
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    with pytest.raises(port.OracleError) as ei:
        _run(t, 0.3, "nocaps", 1, "R")
    assert ei.value.code == 5 and "unglued facet" in str(ei.value)


def test_bad_config():
    g = load_golden("lat4_d030")
    t = _table(g)
    with pytest.raises(port.OracleError) as ei:
        _run(t, 0.3, "fullcaps", 0, "P")
    assert ei.value.code == 8


def test_outer_subset_rows_are_complete():
    # the sampled-row parity at full sizes (tests/test_gpu_fullsize_values.py)
    # relies on affecting_outer() covering every outer element that touches a
    # row: on a delta = 3h mesh the oracle's rows from that subset equal its
    # rows of the whole system (pattern exact, values to rounding of the
    # different block merge order)
    import paper_2302_07499_b200 as P
    from tests.helpers import affecting_outer, cluster_rows, U2
    res, delta = 10, 0.3
    m = P.generate_mesh(3, res, delta, jitter_seed=7)
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    full = _run(t, delta, "nocaps", 1, "R")
    rows, nodes = cluster_rows(t, res, 2, np.random.default_rng(5))
    assert len(rows) >= 4
    outer = affecting_outer(t, delta, nodes)
    assert 0 < len(outer) < int((t.region == 0).sum())
    sub = port.assemble(t, delta, "nocaps", P.kernel_constant(delta, "moment2"),
                        P.forcing_terms(delta, U2, "moment2"), P.normalize_terms(U2),
                        seed=1234, mc_samples=1, sampler="R", outer=outer)
    for r in rows:
        a, b = full["row_ptr"][r], full["row_ptr"][r + 1]
        c, d = sub["row_ptr"][r], sub["row_ptr"][r + 1]
        assert np.array_equal(full["col_idx"][a:b], sub["col_idx"][c:d]), r
        rm = np.abs(full["values"][a:b]).max()
        assert np.abs(full["values"][a:b] - sub["values"][c:d]).max() <= 1e-13 * rm, r
        assert abs(full["rhs"][r] - sub["rhs"][r]) <= 1e-13 * np.abs(full["rhs"]).max(), r
    # dropping the outer elements at one sampled node changes its row (the
    # comparison has teeth)
    v = nodes[0]
    keep = outer[~np.any(t.verts[outer] == v, axis=1)]
    assert len(keep) < len(outer)
    sub2 = port.assemble(t, delta, "nocaps", P.kernel_constant(delta, "moment2"),
                         P.forcing_terms(delta, U2, "moment2"), P.normalize_terms(U2),
                         seed=1234, mc_samples=1, sampler="R", outer=keep)
    r = int(t.dof_of_node[v])
    a, b = full["row_ptr"][r], full["row_ptr"][r + 1]
    c, d = sub2["row_ptr"][r], sub2["row_ptr"][r + 1]
    assert (b - a != d - c) or np.abs(full["values"][a:b] - sub2["values"][c:d]).max() > 1e-8
