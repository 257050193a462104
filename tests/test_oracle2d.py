"""The 2D checker (oracle/port2d.py, test infrastructure) pinned against the
unmodified reference (oracle/_ref) on its own 2D meshes: mode R is the
reference itself for the random-free strategies, so the restatement must give
the reference's pattern and values; for fullcaps the pattern and the number of
Monte Carlo draws (the regions) must be the reference's, and the Philox
function is pinned by the Random123 known answers."""
import numpy as np
import pytest

from oracle import port2d, ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

U2D = np.array([[1, 2, 0, 0], [1, 0, 2, 0]], float)  # u = x^2 + y^2


def table2d(R):
    import paper_2302_07499_b200 as P
    t = R.table()
    return P.ElementTable2D(R.coords, t["verts"], t["neighbor"], t["center"], t["radius"],
                            t["volume"], t["diam"], t["region"], t["inv_edges"],
                            t["dof_of_node"])


def problem2d(res, delta):
    import paper_2302_07499_b200 as P
    R = ref.Problem.generated(2, res, delta)
    Cc, f = ref.forcing(delta, U2D, dim=2)
    return R, table2d(R), Cc, f, P.normalize_terms(U2D)


def rownorm_err(a, b):
    assert np.array_equal(a["row_ptr"], b["row_ptr"]) and np.array_equal(a["col_idx"], b["col_idx"])
    rows = np.repeat(np.arange(len(b["rhs"])), np.diff(b["row_ptr"]))
    rmax = np.zeros(len(b["rhs"]))
    np.maximum.at(rmax, rows, np.abs(b["values"]))
    err = float((np.abs(a["values"] - b["values"]) / rmax[rows]).max()) if len(rows) else 0.0
    rerr = float(np.abs(a["rhs"] - b["rhs"]).max() / max(np.abs(b["rhs"]).max(), 1e-300))
    return err, rerr


def test_philox_known_answers_python():
    assert port2d.philox4x32_10((0, 0, 0, 0), 0, 0) == (0x6627e8d5, 0xe169c58d, 0xbc57ac4c,
                                                        0x9b00dbd8)
    f = 0xFFFFFFFF
    assert port2d.philox4x32_10((f, f, f, f), f, f) == (0x408f276d, 0x41c83b0e, 0xa20bc7c6,
                                                        0x6d5451fd)
    assert port2d.philox4x32_10((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), 0xa4093822,
                                0x299f31d0) == (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)


@pytest.mark.parametrize("strat", ["barycenter", "nocaps", "inside", "overlap", "approxcaps"])
@pytest.mark.parametrize("res,delta", [(4, 0.5), (6, 0.34)])
def test_port2d_equals_reference(strat, res, delta):
    R, t, Cc, f, g = problem2d(res, delta)
    want = R.assemble(delta, strat, U2D)
    got = port2d.assemble(t, delta, strat, Cc, f, g)
    err, rerr = rownorm_err(got, want)
    assert err <= 1e-13 and rerr <= 1e-13, (err, rerr)


def test_port2d_fullcaps_regions_equal_reference():
    R, t, Cc, f, g = problem2d(4, 0.5)
    want = R.assemble(0.5, "fullcaps", U2D, mc_samples=16)
    got = port2d.assemble(t, 0.5, "fullcaps", Cc, f, g, seed=1234, mc_samples=16)
    assert np.array_equal(got["row_ptr"], want["row_ptr"])
    assert np.array_equal(got["col_idx"], want["col_idx"])
    assert got["mc_samples"] == want["mc_samples"]
    # different streams, same estimator: the hit rates agree statistically
    assert abs(got["mc_hits"] / got["mc_samples"] - want["mc_hits"] / want["mc_samples"]) < 0.03
