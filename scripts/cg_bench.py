"""Time GPU CG on an assembled system (device-resident) against the oracle's
reference-style CPU CG (single thread) on the same system."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_07499_b200 as P
from oracle import port
U2 = np.array([[1, 2, 0, 0], [1, 0, 2, 0], [1, 0, 0, 2]], float)
res, delta, strat = int(sys.argv[1]), float(sys.argv[2]), sys.argv[3]
m = P.generate_mesh(3, res, delta, jitter_seed=7 if res == 48 else None)
t = P.ElementTable(m["coords"], m["cells"], m["region"])
s = P.Session(t, delta, strat, "moment2", U2, seed=1234, mc_samples=16)
s.run()
s.cg(tol=1e-10)  # warm-up
t0 = time.perf_counter(); g = s.cg(tol=1e-10); t1 = time.perf_counter()
sysd = s.download()
nnz = len(sysd["values"])
print(f"N={res} delta={delta} {strat}: unknowns {len(sysd['rhs'])}, nnz {nnz}, GPU CG {1e3*(t1-t0):.1f} ms, "
      f"{g['iterations']} it, rel res {g['relative_residual']:.2e}, {1e3*(t1-t0)/max(g['iterations'],1):.3f} ms/it")
if len(sysd["rhs"]) < 200000:
    t0 = time.perf_counter(); r = port.solve_l2(t, sysd, U2, tol=1e-10); t1 = time.perf_counter()
    d = np.abs(g["x"] - r["u"]).max() / np.abs(r["u"]).max()
    print(f"oracle CPU CG (1 thread) + L2: {1e3*(t1-t0):.1f} ms, {r['iterations']} it; max rel diff {d:.1e}; L2 error {r['l2']:.3e}")
