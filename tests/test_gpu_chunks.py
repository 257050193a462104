"""The units / combine pipeline over many chunks (two alternating unit-buffer
sets, the combine of one chunk overlapping the units of the next) gives the
same system bit for bit as one chunk.  Chunking is forced small through
NLFEM_PAIRS_PER_CHUNK in a child process (the library reads it once)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2302_07499_b200 as P
from tests.helpers import SEED, U2
m = P.generate_mesh(3, 6, 0.34, jitter_seed=5)
t = P.ElementTable(m["coords"], m["cells"], m["region"])
out = {}
for strat, mc in (("fullcaps", 8), ("nocaps", 1), ("approxcaps", 1)):
    s = P.Session(t, 0.34, strat, "moment2", U2, seed=SEED, mc_samples=mc)
    st = s.run()
    d = s.download()
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        out[f"{strat}_{k}"] = d[k]
    out[f"{strat}_mc"] = np.array([st.mc_samples, st.mc_hits], np.uint64)
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, name, chunk, overlap=None):
    env = dict(os.environ)
    if chunk:
        env["NLFEM_PAIRS_PER_CHUNK"] = str(chunk)
    else:
        env.pop("NLFEM_PAIRS_PER_CHUNK", None)
    env.pop("NLFEM_COMB_OVERLAP", None)
    if overlap is not None:
        env["NLFEM_COMB_OVERLAP"] = str(overlap)
    f = tmp_path / f"{name}.npz"
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(f)], check=True, env=env, cwd=ROOT)
    return np.load(f)


def test_many_chunks_bitwise_equal_one_chunk(tmp_path):
    one = _run(tmp_path, "one", None)
    many = _run(tmp_path, "many", 3000)   # ~10-20 chunks on this mesh
    for k in one.files:
        assert np.array_equal(one[k], many[k]), k


def test_overlap_modes_bitwise_equal(tmp_path):
    # Overlap mode of Monte Carlo runs (the combine of a chunk as one resident
    # CTA per SM beside the next chunk's units, their launches padded to three
    # CTAs per SM): on (the default), off and chosen by the run's own
    # measurement (many small chunks) all give the same bits as one chunk.
    one = _run(tmp_path, "one", None)
    on = _run(tmp_path, "on", 3000, overlap=3)
    off = _run(tmp_path, "off", 3000, overlap=0)
    probe = _run(tmp_path, "probe", 700, overlap=-1)   # > 20 chunks: the measured choice
    for k in one.files:
        assert np.array_equal(one[k], on[k]), k
        assert np.array_equal(one[k], off[k]), k
        assert np.array_equal(one[k], probe[k]), k
