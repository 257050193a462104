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
