"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run here (needs /root/reference compiled by `make -C oracle ref`):
    python tests/golden/make_golden.py
Each fixture holds a small 3D mesh, the reference's assemble() output for
inside / overlap / barycenter / nocaps / approxcaps / fullcaps (reference xoshiro sampler, seed 1234) with the
moment2 kernel and u = |x|^2, and the per-(T, q) pieces the reference's public
walk_ball emits for a seeded sample of outer points.  These pin the oracle
restatement (tests/test_oracle.py) and the GPU sets/pattern (tests/test_gpu_*.py)
on machines without /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402

U = np.array([[1, 2, 0, 0], [1, 0, 2, 0], [1, 0, 0, 2]], float)
SEED = 1234
STRATS = ("inside", "overlap", "barycenter", "nocaps", "approxcaps", "fullcaps")


def lattice(res, delta, jitter=None):
    import paper_2302_07499_b200 as P
    m = P.generate_mesh(3, res, delta, jitter_seed=jitter)
    return m["coords"], m["cells"], m["region"]


def permuted(res, delta, seed):
    """Lattice mesh with relabelled nodes, shuffled cells and random flips
    (the reference's random_mesh idea, tests/support/test_meshes.cpp:189-221)."""
    c, k, r = lattice(res, delta)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(len(c))
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(c))
    c2 = c[inv]                      # new id j holds old node inv[j]
    k2 = perm[k].astype(np.int32)    # old id -> new id
    order = rng.permutation(len(k2))
    k2, r2 = k2[order], r[order]
    flip = rng.random(len(k2)) < 0.5
    k2[flip, 2], k2[flip, 3] = k2[flip, 3].copy(), k2[flip, 2].copy()
    return c2, k2, r2


CASES = {
    "lat4_d030": (lambda: lattice(4, 0.3), 0.3, 16),
    "lat6_d025": (lambda: lattice(6, 0.25), 0.25, 8),
    "jit5_d040": (lambda: lattice(5, 0.4, jitter=7), 0.4, 8),
    "perm4_d030": (lambda: permuted(4, 0.3, 11), 0.3, 16),
}


def main():
    for name, (mk, delta, mc) in CASES.items():
        c, k, r = mk()
        P = ref.Problem(c, k, r)
        out = dict(coords=c, cells=k.astype(np.int32), region=r.astype(np.uint8),
                   delta=np.float64(delta), mc_samples=np.int32(mc), seed=np.int64(SEED),
                   uterms=U)
        tab = P.table()
        interior = np.nonzero(tab["region"] == 0)[0]
        for strat in STRATS:
            s = P.assemble(delta, strat, U, threads=1, seed=SEED, mc_samples=mc)
            for key in ("row_ptr", "col_idx", "values", "rhs"):
                out[f"{strat}_{key}"] = s[key]
            out[f"{strat}_mc"] = np.array([s["mc_samples"], s["mc_hits"]], np.uint64)
            sol = P.solve_l2(s, U)
            out[f"{strat}_l2"] = np.float64(sol["l2"])
            # walk_ball piece lists for a seeded sample of outer points
            rng = np.random.default_rng(5)
            pick = rng.choice(interior, size=min(24, len(interior)), replace=False)
            rows = []
            for t in pick:
                for q in range(4):
                    par, kind = P.walk_pieces(int(t), q, delta, strat)
                    rows += [(int(t), q, int(a), int(b)) for a, b in zip(par, kind)]
            out[f"{strat}_walk"] = np.array(rows, np.int32)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, len(c), "nodes", len(k), "cells",
              {s: len(out[f"{s}_values"]) for s in STRATS})


if __name__ == "__main__":
    main()
