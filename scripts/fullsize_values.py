"""North-star criteria (a)-(c) on the full-size workloads, against the CPU
checkers run on the box's host cores (minutes each, so outside the test suite;
output kept in profiles/r1_fullsize_values.txt):

  nocaps / barycenter configs: the unmodified reference (oracle/_ref) --
      pattern bit-exact, values <= 1e-12 row-normwise, rhs <= 1e-12;
  fullcaps configs: the restated oracle drawing the same Philox stream
      (oracle/restated.cpp, sampler P) -- pattern bit-exact, values <= 1e-11
      row-normwise, identical draw and hit counts.

usage: python scripts/fullsize_values.py CONFIG [CONFIG ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2302_07499_b200 as P  # noqa: E402
from oracle import port, ref  # noqa: E402
from tests.helpers import rhs_rel_err, row_rel_err, same_pattern  # noqa: E402

rc = 0
cores = os.cpu_count() or 1
for name in sys.argv[1:] or ["C3n"]:
    cfg = bench.CONFIGS[name]
    m = P.generate_mesh(3, cfg["res"], cfg["delta"], jitter_seed=cfg["jitter"])
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    out, st = P.assemble(t, cfg["delta"], cfg["strategy"], "moment2", bench.U2, seed=bench.SEED,
                         mc_samples=cfg["mc"], device=0)
    t0 = time.time()
    if cfg["strategy"] == "fullcaps":
        o = port.assemble(t, cfg["delta"], cfg["strategy"], P.kernel_constant(cfg["delta"], "moment2"),
                          P.forcing_terms(cfg["delta"], bench.U2, "moment2"),
                          P.normalize_terms(bench.U2), seed=bench.SEED, mc_samples=cfg["mc"],
                          sampler="P", threads=cores)
        what, tol = "restated oracle (Philox stream P)", 1e-11
    else:
        R = ref.Problem(m["coords"], m["cells"], m["region"])
        o = R.assemble(cfg["delta"], cfg["strategy"], bench.U2, threads=cores, seed=bench.SEED,
                       mc_samples=cfg["mc"])
        what, tol = "unmodified reference", 1e-12
    tc = time.time() - t0
    pat = same_pattern(out, o)
    ev = row_rel_err(out, o) if pat else float("nan")
    er = rhs_rel_err(out, o)
    line = (f"{name} ({cfg['strategy']}): nnz {len(out['values'])}; {what} on {cores} threads "
            f"{tc:.0f} s; pattern bit-exact {pat}; values max row-normwise rel err {ev:.2e} "
            f"(tol {tol:g}); rhs rel err {er:.2e}")
    if cfg["strategy"] == "fullcaps":
        same_mc = (st["mc_samples"], st["mc_hits"]) == (o["mc_samples"], o["mc_hits"])
        line += f"; draws/hits {st['mc_samples']}/{st['mc_hits']} identical {same_mc}"
        rc |= not same_mc
    print(line, flush=True)
    rc |= not (pat and ev <= tol and er <= tol)
sys.exit(rc)
