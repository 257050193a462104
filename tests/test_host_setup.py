"""Host-side setup (restated mesh / element table / dof map / forcing) is
bit-identical to the reference's upstream (upstream unchanged)."""
import math

import numpy as np
import pytest

import paper_2302_07499_b200 as P
from oracle import ref
from tests.helpers import U2, load_golden

FIELDS = ("verts", "neighbor", "center", "radius", "volume", "diam", "inv_edges")


@pytest.mark.parametrize("name,res,delta,jit", [("lat4_d030", 4, 0.3, None),
                                                ("lat6_d025", 6, 0.25, None),
                                                ("jit5_d040", 5, 0.4, 7)])
def test_generate_mesh_matches_fixture(name, res, delta, jit):
    g = load_golden(name)
    m = P.generate_mesh(3, res, delta, jitter_seed=jit)
    assert np.array_equal(m["coords"], g["coords"])
    assert np.array_equal(m["cells"], g["cells"])
    assert np.array_equal(m["region"], g["region"])


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("res,delta", [(4, 0.3), (5, 0.4), (6, 0.25), (7, 0.3), (8, 0.25),
                                       (8, 0.375)])
def test_generate_mesh_matches_reference(res, delta):
    # the restated lattice generator against the reference's own
    # generate_mesh (mesh.cpp:115-121) -- not against fixtures it produced
    coords, cells, region = ref.generate_mesh(res, delta)
    m = P.generate_mesh(3, res, delta)
    assert np.array_equal(m["coords"], coords)
    assert np.array_equal(m["cells"], cells)
    assert np.array_equal(m["region"], region)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("res,delta", [(5, 0.4), (10, 0.3), (24, 0.125)])
def test_jittered_mesh_matches_reference_rng(res, delta):
    # the config-3 jitter, drawn with the reference's own nlfem::Rng
    coords, cells, region = ref.generate_mesh(res, delta, jitter_seed=7)
    m = P.generate_mesh(3, res, delta, jitter_seed=7)
    assert np.array_equal(m["coords"], coords)
    assert np.array_equal(m["cells"], cells)
    assert np.array_equal(m["region"], region)


def test_mesh_sizes():
    # K = 6 (N+2L)^3, nodes (N+2L+1)^3
    for N, d in ((8, 0.25), (32, 0.1)):
        L = math.ceil(d * N - 1e-9)
        m = P.generate_mesh(3, N, d)
        assert len(m["cells"]) == 6 * (N + 2 * L) ** 3
        assert len(m["coords"]) == (N + 2 * L + 1) ** 3
        assert int((m["region"] == 0).sum()) == 6 * N ** 3


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["lat4_d030", "jit5_d040", "perm4_d030"])
def test_element_table_bit_identical(name):
    g = load_golden(name)
    t = P.ElementTable(g["coords"], g["cells"], g["region"])
    r = ref.Problem(g["coords"], g["cells"], g["region"]).table()
    for f in FIELDS:
        assert np.array_equal(getattr(t, f), r[f]), f
    assert np.array_equal(t.dof_of_node, r["dof_of_node"])
    assert np.array_equal(t.constrained, r["constrained"])


def test_orientation_flips_consistent():
    g = load_golden("perm4_d030")
    t = P.ElementTable(g["coords"], g["cells"], g["region"])
    v = t.coords[t.verts]
    det = np.einsum("ij,ij->i", np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), v[:, 3] - v[:, 0])
    assert (np.sign(det) == np.sign(det[0])).all()
    # neighbour symmetry
    for e in range(0, len(t.verts), 97):
        for f in range(4):
            nb = t.neighbor[e, f]
            if nb >= 0:
                assert e in t.neighbor[nb]


def test_kernel_and_forcing():
    for d in (0.25, 0.1, 1 / 16, 1 / 32):
        C = P.kernel_constant(d, "moment2")
        assert abs(C / (15 / (4 * math.pi * d ** 5)) - 1) < 1e-14
        f = P.forcing_terms(d, U2, "moment2")
        assert f.shape == (1, 4) and f[0, 0] == -6.0 and (f[0, 1:] == 0).all()
        if ref.available():
            Cr, fr = ref.forcing(d, U2, True)
            assert C == Cr and np.array_equal(f, fr)


def test_default_problem_terms():
    t = P.default_problem_terms()
    assert len(t) == 8 and set(np.abs(t[:, 0])) == {1.0}


def test_bad_mesh_rejected():
    g = load_golden("lat4_d030")
    c, k, r = g["coords"], g["cells"], g["region"]
    with pytest.raises(ValueError):
        P.ElementTable(c, k[:, :3], r)
    with pytest.raises(ValueError):
        P.ElementTable(c, k, r + 5)
    bad = k.copy()
    bad[0, 0] = bad[0, 1]
    with pytest.raises(P.NlfemError) as ei:
        P.ElementTable(c, bad, r)
    assert ei.value.name == "BadIndex"
    extra = np.vstack([c, [[9.0, 9.0, 9.0]]])
    with pytest.raises(P.NlfemError) as ei:
        P.ElementTable(extra, k, r)
    assert ei.value.name == "DanglingVertex"
