"""The 2D path (nlfem_gpu_assemble_2d) timed against the unmodified reference
on the same box: the reference's own 2D mesh / element table (oracle/_ref),
u = x^2 + y^2, delta = 3h, fullcaps M = 128 and nocaps; GPU: the one-shot
C-ABI call (host arrays in, host CSR out; device time from its CUDA events);
reference: assemble() on all host cores (AssemblyStats.seconds).
  python scripts/bench2d.py [N ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2302_07499_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402
from tests.test_oracle2d import U2D, problem2d  # noqa: E402

for res in [int(a) for a in sys.argv[1:]] or [128, 256]:
    delta = 3.0 / res
    R, t, Cc, f, g = problem2d(res, delta)
    for strat, mc in (("nocaps", 1), ("fullcaps", 128)):
        P.assemble_2d(t, delta, strat, Cc, f, g, seed=1234, mc_samples=mc, device=0)  # warm-up
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            out, st = P.assemble_2d(t, delta, strat, Cc, f, g, seed=1234, mc_samples=mc,
                                    device=0)
            ts.append(time.perf_counter() - t0)
        r = R.assemble(delta, strat, U2D, mc_samples=mc, seed=1234)
        pairs = st["element_pairs"]
        print(json.dumps({"res": res, "strategy": strat, "mc": mc, "elements": t.elem_count,
                          "element_pairs": pairs, "nnz": int(len(out["values"])),
                          "gpu_device_ms": st["device_ms"], "gpu_phase_ms": [round(x, 2) for x in st["phase_ms"][:4]], "mc_samples": st["mc_samples"], "gpu_e2e_ms": 1e3 * min(ts),
                          "gpu_pairs_per_s_e2e": pairs / min(ts),
                          "ref_s": r["seconds"], "ref_threads": r["threads"],
                          "ref_pairs_per_s": pairs / r["seconds"],
                          "e2e_speedup": r["seconds"] / min(ts)}), flush=True)
