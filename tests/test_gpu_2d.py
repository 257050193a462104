"""The reference's 2D path (nlfem::assemble with et.n == 2) on the B200
(nlfem_gpu_assemble_2d) against the checkers on the reference's own 2D meshes
and element tables: the unmodified reference (oracle/_ref) for the random-free
strategies -- pattern bit-exact, values within 1e-12 of the row's largest
entry -- and the 2D restatement on the same Philox stream (oracle/port2d.py)
for fullcaps -- pattern bit-exact, identical draws and hits, values within
1e-11; the solved L2 error against the reference's."""
import numpy as np
import pytest

import paper_2302_07499_b200 as P
from oracle import port2d, ref
from tests.test_oracle2d import U2D, problem2d, rownorm_err

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]

SEED = 1234


@pytest.mark.parametrize("strat", ["barycenter", "nocaps", "inside", "overlap", "approxcaps"])
@pytest.mark.parametrize("res,delta", [(4, 0.5), (8, 0.25), (16, 3 / 16)])
def test_2d_matches_reference(strat, res, delta):
    R, t, Cc, f, g = problem2d(res, delta)
    want = R.assemble(delta, strat, U2D)
    got, st = P.assemble_2d(t, delta, strat, Cc, f, g, seed=SEED, device=0)
    err, rerr = rownorm_err(got, want)
    assert err <= 1e-12 and rerr <= 1e-12, (strat, res, err, rerr)
    if res <= 8:
        o = port2d.assemble(t, delta, strat, Cc, f, g)
        assert st["element_pairs"] == o["element_pairs"]


@pytest.mark.parametrize("res,delta,mc", [(4, 0.5, 16), (8, 0.25, 32)])
def test_2d_fullcaps_matches_oracle_same_stream(res, delta, mc):
    R, t, Cc, f, g = problem2d(res, delta)
    got, st = P.assemble_2d(t, delta, "fullcaps", Cc, f, g, seed=SEED, mc_samples=mc, device=0)
    o = port2d.assemble(t, delta, "fullcaps", Cc, f, g, seed=SEED, mc_samples=mc)
    assert (st["mc_samples"], st["mc_hits"]) == (o["mc_samples"], o["mc_hits"])
    assert st["element_pairs"] == o["element_pairs"]
    err, rerr = rownorm_err(got, o)
    assert err <= 1e-11 and rerr <= 1e-11, (err, rerr)
    # the regions and the pattern are the reference's
    want = R.assemble(delta, "fullcaps", U2D, mc_samples=mc)
    assert np.array_equal(got["row_ptr"], want["row_ptr"])
    assert np.array_equal(got["col_idx"], want["col_idx"])
    assert st["mc_samples"] == want["mc_samples"]


def test_2d_fullcaps_solved_error_close_to_reference():
    # north star (d): the solved error of u = x^2 + y^2 within 1% of the
    # reference's (its own xoshiro stream vs our Philox stream, same estimator)
    R, t, Cc, f, g = problem2d(32, 3 / 32)
    got, _ = P.assemble_2d(t, 3 / 32, "fullcaps", Cc, f, g, seed=SEED, mc_samples=128, device=0)
    want = R.assemble(3 / 32, "fullcaps", U2D, mc_samples=128)
    a, b = R.solve_l2(got, U2D), R.solve_l2(want, U2D)
    assert a["converged"] and b["converged"]
    assert abs(a["l2"] - b["l2"]) <= 0.01 * b["l2"], (a["l2"], b["l2"])


def test_2d_deterministic_and_bad_config():
    R, t, Cc, f, g = problem2d(8, 0.25)
    a, _ = P.assemble_2d(t, 0.25, "fullcaps", Cc, f, g, seed=SEED, mc_samples=16, device=0)
    b, _ = P.assemble_2d(t, 0.25, "fullcaps", Cc, f, g, seed=SEED, mc_samples=16, device=0)
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        assert np.array_equal(a[k], b[k]), k
    with pytest.raises(P.NlfemError) as e:
        P.assemble_2d(t, 0.25, "fullcaps", Cc, f, g, mc_samples=0, device=0)
    assert e.value.code == 8
    # a ball wider than the interaction layer reaches past the mesh boundary
    with pytest.raises(P.NlfemError) as e:
        P.assemble_2d(t, 0.6, "nocaps", Cc, f, g, device=0)
    assert e.value.code == 5 and "unglued facet" in str(e.value)
