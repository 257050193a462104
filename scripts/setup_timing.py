"""Upstream setup time: host restatement vs nlfem_gpu_element_table (C3/C4 meshes)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2302_07499_b200 as P  # noqa: E402

out = []
for N, jit in ((48, 7), (96, None)):
    m = P.generate_mesh(3, N, 3 / N, jitter_seed=jit)
    c, k, r = m["coords"], m["cells"], m["region"]
    P.ElementTable(c[:0 + len(c)], k, r, device=0) if N == 48 else None  # warm the context
    t0 = time.perf_counter()
    g = P.ElementTable(c, k, r, device=0)
    t1 = time.perf_counter()
    h = P.ElementTable(c, k, r)
    t2 = time.perf_counter()
    same = all(np.array_equal(getattr(g, f), getattr(h, f)) for f in
               ("verts", "neighbor", "center", "radius", "volume", "diam", "inv_edges",
                "dof_of_node", "constrained"))
    out.append({"N": N, "cells": len(k), "gpu_s": round(t1 - t0, 4), "host_s": round(t2 - t1, 3),
                "identical": same})
    print(json.dumps(out[-1]), flush=True)
