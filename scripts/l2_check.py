"""North-star criterion (d) at full size: the solved L2 error against the
manufactured solution u = |x|^2, GPU (assembly + Session.solve on the device)
against the unmodified reference (oracle/_ref: assemble() on all host cores,
then the reference harness's CG + l2_error).  nocaps is deterministic (the two
agree to the CG tolerance); fullcaps differs only by the Monte Carlo stream
(Philox vs the reference's xoshiro), so within 1%.  Minutes of CPU time per
config: kept out of the test suite, output in profiles/r1_l2_check.txt.

usage: python scripts/l2_check.py CONFIG [CONFIG ...]   (bench.py config names)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2302_07499_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402

for name in sys.argv[1:] or ["C3n"]:
    cfg = bench.CONFIGS[name]
    m = P.generate_mesh(3, cfg["res"], cfg["delta"], jitter_seed=cfg["jitter"])
    t = P.ElementTable(m["coords"], m["cells"], m["region"], device=0)
    s = P.Session(t, cfg["delta"], cfg["strategy"], "moment2", bench.U2, seed=bench.SEED,
                  mc_samples=cfg["mc"], device=0)
    st = s.run()
    g = s.solve(tol=1e-12)
    s.close()
    print(f"{name}: GPU assembly {st.device_ms:.0f} ms, solve {g['device_ms']:.0f} ms "
          f"({g['iterations']} CG iterations): L2 {g['l2']:.6e}, max nodal {g['max_nodal_error']:.6e}",
          flush=True)
    t0 = time.time()
    R = ref.Problem(m["coords"], m["cells"], m["region"])
    r = R.assemble(cfg["delta"], cfg["strategy"], bench.U2, threads=os.cpu_count() or 1,
                   seed=bench.SEED, mc_samples=cfg["mc"])
    ta = time.time() - t0
    rs = R.solve_l2(r, bench.U2, tol=1e-12)
    print(f"{name}: reference assembly {ta:.0f} s on {os.cpu_count()} threads, solve "
          f"({rs['iterations']} CG iterations): L2 {rs['l2']:.6e}, max nodal {rs['max_nodal']:.6e}")
    print(f"{name}: L2 ratio GPU / reference - 1 = {g['l2'] / rs['l2'] - 1:+.3e}; max nodal "
          f"ratio - 1 = {g['max_nodal_error'] / rs['max_nodal'] - 1:+.3e}", flush=True)
