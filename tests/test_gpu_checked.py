"""Memory checking without compute-sanitizer (closed on this GPU pool): the
library built with -DNLFEM_CHECKED=1 (4-KiB canaries on both sides of every
device buffer, verified at the end of every run) must catch a deliberate
one-element overrun, and the whole pipeline -- one chunk and many chunks
(two alternating unit-buffer sets over four streams), fullcaps / nocaps /
approxcaps, the owner-computes path -- must run clean and give the default
build's system bit for bit.  Skipped unless the checked library is built
(scripts/build_variant.sh checked -DNLFEM_CHECKED=1)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2302_07499_b200", "libnlfem_gpu_checked.so")

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2302_07499_b200 as P
from paper_2302_07499_b200 import distributed as D
from tests.helpers import SEED, U2
from tests.test_gpu_distributed import _owner_computes
L = P.lib()
r1, r0 = L.nlfem_gpu_debug_guard_selftest(1), L.nlfem_gpu_debug_guard_selftest(0)
want = (1, 0) if sys.argv[3] == "checked" else (-1, -1)
assert (r1, r0) == want, ("canary self-test", r1, r0, P.LIB_PATH)
out = {}
m = P.generate_mesh(3, 6, 0.34, jitter_seed=5)
t = P.ElementTable(m["coords"], m["cells"], m["region"])
for strat, mc in (("fullcaps", 8), ("nocaps", 1), ("approxcaps", 1), ("barycenter", 1)):
    s = P.Session(t, 0.34, strat, "moment2", U2, seed=SEED, mc_samples=mc)
    s.run()
    r = s.download()
    for k in r:
        out[f"{strat}_{k}"] = np.array(r[k])
    s.close()
got, _ = _owner_computes(t, "fullcaps", 8, 3)
for k in got:
    out[f"oc_{k}"] = got[k]
np.savez(sys.argv[2], **out)
"""


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked library not built")
@pytest.mark.parametrize("chunk", [None, "3000"])
def test_checked_build_runs_clean_and_equal(chunk, tmp_path):
    res = {}
    for tag, lib in (("checked", CHECKED), ("default", None)):
        env = dict(os.environ)
        env.pop("NLFEM_GPU_LIB", None)
        if lib:
            env["NLFEM_GPU_LIB"] = lib
        if chunk:
            env["NLFEM_PAIRS_PER_CHUNK"] = chunk
        out = str(tmp_path / f"{tag}.npz")
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT, out, tag], env=env, cwd=ROOT,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        res[tag] = np.load(out)
    for k in res["default"].files:
        assert np.array_equal(res["checked"][k], res["default"][k]), k
