"""Per-element-pair rate of the unmodified reference assemble() (oracle/_ref)
against mesh size at fixed delta/h and M: justifies timing the reference arm
on a smaller mesh than the benchmarked one.

    python scripts/ref_rate_vs_n.py --ratio 3 --mc 128 --res 8 12 16 24

Pairs are counted by the restated oracle (oracle/port.py) on the reference's
own element table; nothing from paper_2302_07499_b200 is imported."""
import argparse
import json
import os
import sys
import time
import types

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import port, ref  # noqa: E402

U2 = np.array([[1, 2, 0, 0], [1, 0, 2, 0], [1, 0, 0, 2]], float)


def ref_table(coords, cells, region):
    R = ref.Problem(coords, cells, region)
    t = R.table()
    ns = types.SimpleNamespace(**t)
    ns.coords = np.ascontiguousarray(coords, np.float64)
    ns.elem_count, ns.node_count, ns.unknowns = R.elems, R.nodes, R.unknowns
    return R, ns


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ratio", type=float, default=3.0)
    ap.add_argument("--mc", type=int, default=128)
    ap.add_argument("--strategy", default="fullcaps")
    ap.add_argument("--res", type=int, nargs="+", default=[8, 12, 16])
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    for res in a.res:
        delta = a.ratio / res
        coords, cells, region = ref.generate_mesh(res, delta)
        R, t = ref_table(coords, cells, region)
        Cc, f = ref.forcing(delta, U2)
        o = port.assemble(t, delta, a.strategy, Cc, f, U2, seed=1234, mc_samples=1,
                          sampler="R", threads=a.threads)
        t0 = time.perf_counter()
        out = R.assemble(delta, a.strategy, U2, threads=a.threads, seed=1234,
                         mc_samples=a.mc)
        wall = time.perf_counter() - t0
        interior = int((region == 0).sum())
        print(json.dumps({"res": res, "delta": delta, "strategy": a.strategy, "M": a.mc,
                          "threads": a.threads, "outer_elements": interior,
                          "element_pairs": int(o["element_pairs"]),
                          "seconds": out["seconds"], "wall": wall,
                          "pairs_per_s": o["element_pairs"] / out["seconds"],
                          "mc_samples": out["mc_samples"],
                          "samples_per_pair": out["mc_samples"] / o["element_pairs"]}),
              flush=True)


if __name__ == "__main__":
    main()
