"""Per-rank cost of the sharded (multi-GPU) step, emulated on one GPU.

For n shards of the outer elements, times what ONE rank does for its shard
(the collectives themselves excluded -- they need n GPUs):
  pairs   build the element pairs of the rank's range (pairs_shard: prep + K1)
  run     pattern from the full pair list (installed, as after the all-gather)
          + units / combine of the rank's range (run_shard)
  final   finalize of the rank's row block
Usage: python scripts/shard_timing.py [CONFIG] (bench.py config names)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2302_07499_b200 as P  # noqa: E402
from paper_2302_07499_b200.distributed import shard_range  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = bench.CONFIGS[name]
m = P.generate_mesh(3, cfg["res"], cfg["delta"], jitter_seed=cfg["jitter"])
t = P.ElementTable(m["coords"], m["cells"], m["region"], device=0)
s = P.Session(t, cfg["delta"], cfg["strategy"], "moment2", bench.U2, seed=bench.SEED,
              mc_samples=cfg["mc"], device=0)
KI = s.interior_count
# full pair list (what every rank holds after the all-gather)
s.pairs_shard(0, KI)
cv, pv = s.pairs_shard_out()
counts = torch.as_tensor(cv, device="cuda").clone()
partners = torch.as_tensor(pv, device="cuda").clone()
total = int(partners.numel())


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return float(np.median(ts))


print(f"{name}: KI={KI} pairs={total}")
print(f"{'shards':>6s} {'pairs ms':>9s} {'run ms':>8s} {'final ms':>9s} {'sum ms':>8s}")
for n in (1, 2, 4, 8):
    lo, hi = shard_range(KI, 0, n)
    r0, r1 = shard_range(s.unknowns, 0, n)
    tp = timed(lambda: s.pairs_shard(lo, hi))

    def run():
        s.pairs_install(counts, partners, total)
        s.run_shard(lo, hi, finalize=False)
    tr = timed(run)
    tf = timed(lambda: s.finalize(r0, r1))
    print(f"{n:6d} {tp:9.3f} {tr:8.3f} {tf:9.3f} {tp + tr + tf:8.3f}")
