"""Upstream setup on the GPU: nlfem_gpu_element_table
writes the same ElementTable / DofMap arrays as the host restatement (itself
bit-identical to the reference, tests/test_host_setup.py), and the same errors."""
import numpy as np
import pytest

import paper_2302_07499_b200 as P
from tests.helpers import load_golden

FIELDS = ("verts", "neighbor", "center", "radius", "volume", "diam", "inv_edges",
          "dof_of_node", "constrained")


def _same(a, b):
    for f in FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.unknowns == b.unknowns


def _err(coords, cells, region, device):
    with pytest.raises(P.NlfemError) as ei:
        P.ElementTable(coords, cells, region, device=device)
    return ei.value


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["lat4_d030", "lat6_d025", "jit5_d040", "perm4_d030"])
def test_gpu_table_bit_identical_to_host(name):
    g = load_golden(name)
    _same(P.ElementTable(g["coords"], g["cells"], g["region"], device=0),
          P.ElementTable(g["coords"], g["cells"], g["region"]))


@pytest.mark.gpu
def test_gpu_table_large_jittered_and_shuffled():
    m = P.generate_mesh(3, 24, 3 / 24, jitter_seed=7)
    c, k, r = m["coords"], m["cells"].copy(), m["region"]
    rng = np.random.default_rng(3)
    order = rng.permutation(len(k))
    k, r = k[order], r[order]
    flip = rng.random(len(k)) < 0.5          # random orientation flips
    k[flip, 0], k[flip, 1] = k[flip, 1].copy(), k[flip, 0].copy()
    _same(P.ElementTable(c, k, r, device=0), P.ElementTable(c, k, r))


def _ring(n, closure):
    """Cyclic tet strip, cell i = seq[i:i+4]; a twisted closure (odd
    permutation of the first three vertices) is not orientable -- the
    reference raises NonManifold for it, as the host restatement does."""
    seq = list(range(n)) + list(closure)
    k = np.array([seq[i:i + 4] for i in range(n)], np.int32)
    return np.random.default_rng(n).random((n, 3)), k, np.zeros(n, np.uint8)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [8, 11])
def test_gpu_orientation_rings(n):
    _same(P.ElementTable(*_ring(n, [0, 1, 2]), device=0), P.ElementTable(*_ring(n, [0, 1, 2])))
    for twist in ([1, 0, 2], [2, 1, 0]):
        eh, eg = _err(*_ring(n, twist), None), _err(*_ring(n, twist), 0)
        assert (eg.code, str(eg)) == (eh.code, str(eh)) == (3, "NonManifold: mesh is not orientable")


@pytest.mark.gpu
def test_gpu_table_two_components_with_flips():
    # each component's flips are relative to its own lowest-id cell
    g = load_golden("perm4_d030")
    c, k, r = g["coords"], g["cells"], g["region"]
    k2 = k + len(c)
    k2[::3, 2], k2[::3, 3] = k2[::3, 3].copy(), k2[::3, 2].copy()
    cc = np.vstack([c, c + 5.0])
    kk = np.vstack([k2[:50], k, k2[50:]]).astype(np.int32)
    rr = np.concatenate([r[:50], r, r[50:]])
    _same(P.ElementTable(cc, kk, rr, device=0), P.ElementTable(cc, kk, rr))


@pytest.mark.gpu
def test_gpu_table_errors_match_host():
    g = load_golden("lat4_d030")
    c, k, r = g["coords"], g["cells"], g["region"]
    cases = []
    bad = k.copy()
    bad[7, 2] = bad[7, 0]                    # repeated vertex (first in cell order)
    bad[9, 1] = bad[9, 3]
    cases.append((c, bad, r))
    bad = k.copy()
    bad[11, 3] = bad[11, 2]
    cases.append((c, bad, r))
    cases.append((np.vstack([c, [[9.0, 9.0, 9.0]]]), k, r))        # dangling vertex
    # a third cell on an interior facet
    f = k[100, :3]
    c3 = np.vstack([c, [[0.31, 0.27, 0.29]]])
    cases.append((c3, np.vstack([k, [[f[0], f[1], f[2], len(c)]]]), np.append(r, 0)))
    # degenerate element: one node moved into its cell's opposite face plane
    cd = c.copy()
    t = 500
    a, b, d, e = cd[k[t]]
    cd[k[t][3]] = a + 0.5 * (b - a) + 0.25 * (d - a)
    cases.append((cd, k, r))
    for cc, kk, rr in cases:
        eh, eg = _err(cc, kk, rr, None), _err(cc, kk, rr, 0)
        assert (eg.code, str(eg)) == (eh.code, str(eh))


def test_gpu_table_fails_loudly_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    g = load_golden("lat4_d030")
    e = _err(g["coords"], g["cells"], g["region"], 0)
    assert e.code == 100
