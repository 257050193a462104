"""Acceptance checks at C4 (N=96, delta=3h, fullcaps M=128):
the sets of a seeded sample of 10^4 outer elements against the reference's
walk_ball (oracle/_ref), exact symmetry and bitwise repeatability of the
assembled matrix, checked on the device.  Too long for the test suite (two C4
assemblies plus the reference's host setup of a 6.4M-element mesh); its output
is kept in profiles/r1_c4_check.txt.

usage: python scripts/c4_check.py [NSAMPLE]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2302_07499_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402
from tests.test_gpu_fullsize import _outputs, _reference_sets, _sampled_gpu_sets, _symmetric  # noqa: E402

nsample = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
cfg = bench.CONFIGS["C4"]
t0 = time.time()
m = P.generate_mesh(3, cfg["res"], cfg["delta"], jitter_seed=cfg["jitter"])
t = P.ElementTable(m["coords"], m["cells"], m["region"], device=0)
s = P.Session(t, cfg["delta"], cfg["strategy"], "moment2", bench.U2, seed=bench.SEED,
              mc_samples=cfg["mc"], device=0)
st = s.run()
print(f"C4: elements {t.elem_count}, interior {s.interior_count}, unknowns {s.unknowns}, "
      f"element pairs {st.element_pairs}, items {st.items}, MC samples {st.mc_samples}, "
      f"device {st.device_ms:.0f} ms", flush=True)
ro, ci, va, rh = (x.clone() for x in _outputs(s))
print(f"nnz {int(ro[-1])}; exactly symmetric: {_symmetric(ro, ci, va)}", flush=True)
interior = np.nonzero(t.region == 0)[0]
sample = np.random.default_rng(2024).choice(interior, size=nsample, replace=False)
got = _sampled_gpu_sets(s, sample)
s.run()
ro2, ci2, va2, rh2 = _outputs(s)
same = (torch.equal(ro, ro2) and torch.equal(ci, ci2) and torch.equal(va, va2) and
        torch.equal(rh, rh2))
print(f"second run bitwise identical: {same}", flush=True)
s.close()
del ro, ci, va, rh, ro2, ci2, va2, rh2
if not ref.available():
    print("oracle/_ref not built: sets not compared")
    sys.exit(0)
t1 = time.time()
want = _reference_sets(m, sample, cfg["delta"], cfg["strategy"])
keys = set(want) | set(got)
bad = [k for k in keys if got.get(k, set()) != want.get(k, set())]
npieces = sum(len(v) for v in want.values())
print(f"sets: {nsample} outer elements, {len(want)} (T, q) keys, {npieces} (T, q, T') items "
      f"with pieces; mismatches: {len(bad)} (reference walk {time.time() - t1:.0f} s)")
print(f"total {time.time() - t0:.0f} s")
sys.exit(1 if bad or not same else 0)
