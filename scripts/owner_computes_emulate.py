"""Owner-computes multi-GPU step emulated rank by rank on ONE GPU (the ranks'
kernels never wait on each other: each rank's work runs alone, the all-to-all
is replaced by slicing the records by destination).  Per rank and world size:
run_local time (pairs + local pattern + units + combine of its outer
elements), local pattern size, records and bytes it sends to other ranks,
finalize_merged time; the assembled system's SHA-256 equals the one-GPU run.

  python scripts/owner_computes_emulate.py [CONFIG] [WORLDS]   e.g. C4 2,4,8
"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2302_07499_b200 as P  # noqa: E402
from paper_2302_07499_b200 import distributed as D  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
worlds = [int(w) for w in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
cfg = bench.CONFIGS[name]
m = P.generate_mesh(3, cfg["res"], cfg["delta"], jitter_seed=cfg["jitter"])
t = P.ElementTable(m["coords"], m["cells"], m["region"], device=0)


def session():
    return P.Session(t, cfg["delta"], cfg["strategy"], "moment2", bench.U2, seed=bench.SEED,
                     mc_samples=cfg["mc"], device=0)


def sha(blocks):
    h = hashlib.sha256()
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        h.update(np.ascontiguousarray(blocks[k]).tobytes())
    return h.hexdigest()


s = session()
s.run()  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
s.run()
torch.cuda.synchronize()
one_ms = 1e3 * (time.perf_counter() - t0)
ref = s.download()
ref_sha = sha(ref)
KI, U = s.interior_count, s.unknowns
s.close()
del ref
torch.cuda.empty_cache()
print(json.dumps({"config": name, "one_gpu_ms": one_ms, "interior": KI, "unknowns": U}),
      flush=True)

for world in worlds:
    bounds = D.row_bounds(U, world)
    # phase 1: every rank's local run; its outgoing records parked on the host
    # (pinned) so one session at a time holds HBM
    inbox = [[] for _ in range(world)]
    ranks = []
    for r in range(world):
        lo, hi = D.shard_range(KI, r, world)
        s = session()
        s.run_local(lo, hi)  # warm-up: the session's buffers are allocated here
        s.halo_records(bounds)
        s.rhs_records(bounds)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = s.run_local(lo, hi)
        torch.cuda.synchronize()
        t_local = 1e3 * (time.perf_counter() - t0)
        t0 = time.perf_counter()
        k, w, kc = s.halo_records(bounds)
        ri, rv, rc = s.rhs_records(bounds)
        torch.cuda.synchronize()
        t_rec = 1e3 * (time.perf_counter() - t0)
        k, w = torch.as_tensor(k, device="cuda"), torch.as_tensor(w, device="cuda")
        ri, rv = torch.as_tensor(ri, device="cuda"), torch.as_tensor(rv, device="cuda")
        ko, ro = np.concatenate([[0], np.cumsum(kc)]), np.concatenate([[0], np.cumsum(rc)])
        for d in range(world):
            inbox[d].append(tuple(x.cpu() for x in (k[ko[d]:ko[d + 1]], w[4 * ko[d]:4 * ko[d + 1]],
                                                    ri[ro[d]:ro[d + 1]],
                                                    rv[32 * ro[d]:32 * ro[d + 1]])))
        sent = int(kc.sum() - kc[r]), int(rc.sum() - rc[r])
        ranks.append({"rank": r, "outer": hi - lo, "pairs": int(st.element_pairs),
                      "local_nnz": int(st.nnz_ext), "run_local_ms": round(t_local, 2),
                      "records_ms": round(t_rec, 2), "records_out": sent[0],
                      "rhs_records_out": sent[1],
                      "bytes_out": 40 * sent[0] + (4 + 256) * sent[1]})
        s.close()
        torch.cuda.empty_cache()
    # phase 2: every owner merges what it received and finalizes its block
    blocks = []
    for d in range(world):
        s = session()
        lo, hi = D.shard_range(KI, d, world)
        s.run_local(lo, hi)  # the owner's own state (its V is replaced below)
        keys, words, ridx, rvals = (torch.cat([p[i] for p in inbox[d]]).cuda() for i in range(4))
        s.finalize_merged(bounds[d], bounds[d + 1], keys, words, ridx, rvals)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.finalize_merged(bounds[d], bounds[d + 1], keys, words, ridx, rvals)
        torch.cuda.synchronize()
        ranks[d]["finalize_merged_ms"] = round(1e3 * (time.perf_counter() - t0), 2)
        ranks[d]["records_in"] = int(keys.numel())
        blocks.append(s.download_rows(bounds[d], bounds[d + 1]))
        s.close()
        del keys, words, ridx, rvals
        torch.cuda.empty_cache()
    full = D.concat_csr(blocks)
    step = max(x["run_local_ms"] + x["records_ms"] + x["finalize_merged_ms"] for x in ranks)
    print(json.dumps({"config": name, "world": world, "bitwise_equal_one_gpu": sha(full) == ref_sha,
                      "max_rank_ms_excl_collectives": round(step, 2),
                      "speedup_vs_one_gpu": round(one_ms / step, 2), "ranks": ranks}), flush=True)
