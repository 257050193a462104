"""Conjugate gradients on the GPU (reference cg_solve, proj/src/solver.cpp:26-66;
python binding nlfem.cg, nlfem_module.cpp:228-256) against the oracle's
reference-style CG on the assembled C1 system."""
import numpy as np
import pytest

import paper_2302_07499_b200 as P
from oracle import port
from tests.helpers import SEED, U2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    m = P.generate_mesh(3, 8, 0.25)
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    sys, _ = P.assemble(t, 0.25, "nocaps", "moment2", U2, seed=SEED)
    return t, {k: np.array(v) for k, v in sys.items()}


def test_cg_matches_reference_style_oracle(c1):
    t, sys = c1
    got = P.cg(sys["row_ptr"], sys["col_idx"], sys["values"], sys["rhs"], tol=1e-12,
               max_iterations=100 * len(sys["rhs"]))
    ref = port.solve_l2(t, sys, U2, tol=1e-12)
    assert got["converged"] and ref["converged"]
    x, xr = got["x"], ref["u"]
    assert np.abs(x - xr).max() <= 1e-8 * np.abs(xr).max()
    # same algorithm, different summation order: iteration counts within a few
    assert abs(got["iterations"] - ref["iterations"]) <= 3
    assert got["relative_residual"] <= 1e-12


def test_cg_on_device_session_equals_host_call_and_is_deterministic(c1):
    t, sys = c1
    s = P.Session(t, 0.25, "nocaps", "moment2", U2, seed=SEED)
    s.run()
    a = s.cg(tol=1e-11)
    b = s.cg(tol=1e-11)
    h = P.cg(sys["row_ptr"], sys["col_idx"], sys["values"], sys["rhs"], tol=1e-11)
    assert np.array_equal(a["x"], b["x"]) and a["iterations"] == b["iterations"]
    assert np.array_equal(a["x"], h["x"]) and a["iterations"] == h["iterations"]


def test_cg_edge_cases(c1):
    _, sys = c1
    z = P.cg(sys["row_ptr"], sys["col_idx"], sys["values"], np.zeros_like(sys["rhs"]))
    assert z["converged"] and z["iterations"] == 0 and not z["x"].any()
    n0 = P.cg(sys["row_ptr"], sys["col_idx"], sys["values"], sys["rhs"], max_iterations=0)
    assert not n0["converged"] and n0["iterations"] == 0 and not n0["x"].any()
    assert n0["relative_residual"] == pytest.approx(1.0)
    capped = P.cg(sys["row_ptr"], sys["col_idx"], sys["values"], sys["rhs"], tol=1e-14,
                  max_iterations=5)
    assert capped["iterations"] == 5 and not capped["converged"]
    with pytest.raises(ValueError):
        P.cg(sys["row_ptr"][:-1], sys["col_idx"], sys["values"], sys["rhs"])
