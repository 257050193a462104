"""Shared test helpers: fixtures, CSR comparisons, set extraction."""
from __future__ import annotations

import glob
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
U2 = np.array([[1, 2, 0, 0], [1, 0, 2, 0], [1, 0, 0, 2]], float)   # u = |x|^2
SEED = 1234


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def csr_rows(s):
    return np.repeat(np.arange(len(s["row_ptr"]) - 1), np.diff(s["row_ptr"]))


def same_pattern(a, b):
    return np.array_equal(a["row_ptr"], b["row_ptr"]) and np.array_equal(a["col_idx"], b["col_idx"])


def row_rel_err(a, b):
    """max_i max_k |a_ik - b_ik| / max_k |b_ik| (row-normwise)."""
    assert same_pattern(a, b)
    rows = csr_rows(b)
    rmax = np.zeros(len(b["row_ptr"]) - 1)
    np.maximum.at(rmax, rows, np.abs(b["values"]))
    rmax[rmax == 0] = 1.0
    return float((np.abs(a["values"] - b["values"]) / rmax[rows]).max()) if len(rows) else 0.0


def rhs_rel_err(a, b):
    s = max(np.abs(b["rhs"]).max(), 1e-300) if len(b["rhs"]) else 1.0
    return float(np.abs(a["rhs"] - b["rhs"]).max() / s) if len(b["rhs"]) else 0.0


def gpu_sets(pairs, q_filter=None):
    """{(T, q): {(parent, 'W'|'P')}} from the GPU pair list (5-bit codes)."""
    out = {}
    off, partner, info, interior = pairs["offsets"], pairs["partner"], pairs["info"], pairs["interior"]
    for ii, T in enumerate(interior):
        for p in range(off[ii], off[ii + 1]):
            for q in range(4):
                c = (int(info[p]) >> (5 * q)) & 31
                if c:
                    out.setdefault((int(T), q), set()).add((int(partner[p]), "W" if c == 1 else "P"))
    return out


def walk_sets(rows):
    """Same structure from the reference's walk_ball piece lists (T, q, parent, kind)."""
    tmp = {}
    for T, q, par, kind in rows:
        tmp.setdefault((int(T), int(q)), {}).setdefault(int(par), []).append(int(kind))
    out = {}
    for key, d in tmp.items():
        out[key] = {(par, "W" if kinds == [0] else "P") for par, kinds in d.items()}
    return out


def cluster_rows(t, res, nclusters, rng):
    """Seeded clusters of unknowns of a lattice (or jittered lattice) mesh: a
    node and its +x / +y lattice neighbours when they are unknowns; the first
    cluster in the bulk (>= 0.3 from the boundary of [0,1]^3), the second next
    to the boundary.  Returns (sorted unknown rows, their node ids)."""
    dof = t.dof_of_node
    xyz = t.coords
    unk = np.nonzero(dof >= 0)[0]
    h = 1.0 / res
    dist = np.min(np.minimum(xyz[unk], 1.0 - xyz[unk]), axis=1)
    picks = [rng.choice(unk[dist > 0.3])]
    if nclusters > 1:
        picks.append(rng.choice(unk[dist < 1.5 * h]))
    nodes = []
    for v in picks:
        for off in ((0, 0, 0), (h, 0, 0), (0, h, 0)):
            p = xyz[v] + np.array(off)
            j = int(np.argmin(np.abs(xyz - p).sum(axis=1)))
            if dof[j] >= 0 and np.abs(xyz[j] - p).max() < 0.45 * h:
                nodes.append(j)
    nodes = sorted(set(nodes))
    return sorted({int(dof[j]) for j in nodes}), nodes


def affecting_outer(t, delta, nodes):
    """Every interior (outer) element whose element pairs can put an entry in
    the rows of `nodes`: v in T gives |c_T - x_v| <= r_T; v in T' with T'
    meeting B_delta(x_q), x_q in T, gives |c_T - x_v| <= delta + 2 r_T' + r_T.
    So centre within delta + 3 r_max (a superset; extra elements only add to
    other rows)."""
    interior = np.nonzero(t.region == 0)[0]
    reach = (delta + 3.0 * float(t.radius.max())) * (1 + 1e-6) + 1e-12
    c = t.center[interior]
    keep = np.zeros(len(interior), bool)
    for v in nodes:
        keep |= np.sum((c - t.coords[v]) ** 2, axis=1) <= reach * reach
    return interior[keep].astype(np.int32)
