"""Where does the one-shot C-ABI call spend host time? (profiling helper)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_07499_b200 as P
U = np.array([[1, 2, 0, 0], [1, 0, 2, 0], [1, 0, 0, 2]], float)
m = P.generate_mesh(3, 8, 0.25)
t = P.ElementTable(m["coords"], m["cells"], m["region"])
for i in range(4):
    t0 = time.perf_counter()
    out, st = P.assemble(t, 0.25, "fullcaps", "moment2", U, seed=1234, mc_samples=64)
    t1 = time.perf_counter()
    print(f"call {i}: wall {1e3*(t1-t0):.2f} ms, C-ABI seconds {1e3*st['seconds']:.2f} ms, device {st['device_ms']:.2f} ms, phases {[round(x,2) for x in st['phase_ms'][:6]]}")
s = P.Session(t, 0.25, "fullcaps", "moment2", U, seed=1234, mc_samples=64)
for i in range(3):
    t0 = time.perf_counter(); st = s.run(); t1 = time.perf_counter()
    print(f"session run {i}: wall {1e3*(t1-t0):.2f} ms device {st.device_ms:.2f}")
t0 = time.perf_counter(); o = s.download(); print("download", 1e3*(time.perf_counter()-t0), "ms")
