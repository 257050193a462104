"""The N>1 path end to end on one GPU: two ranks (processes) over gloo, both on
cuda:0, each building its own outer elements' pairs, all-gathering them,
integrating its shard, all-reducing the fixed-point partials, finalizing its
row block and all-gathering the blocks (distributed.device_step /
assemble_distributed).  gloo's collectives are driven by the host, so the two
ranks' kernels never wait on each other; the result must be the one-GPU system
bit for bit.  (On a multi-GPU box the same code runs over NCCL, one GPU each.)"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, sys, numpy as np
sys.path.insert(0, sys.argv[1])
import torch, torch.distributed as dist
import paper_2302_07499_b200 as P
from paper_2302_07499_b200 import distributed as D
from tests.helpers import SEED, U2
rank, world, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
torch.cuda.set_device(0)
dist.init_process_group("gloo", rank=rank, world_size=world)
m = P.generate_mesh(3, 6, 0.34, jitter_seed=5)
t = P.ElementTable(m["coords"], m["cells"], m["region"])
res = {}
for strat, mc in (("fullcaps", 8), ("nocaps", 1)):
    s = P.Session(t, 0.34, strat, "moment2", U2, seed=SEED, mc_samples=mc)
    full, st = D.assemble_distributed(s)
    for k in ("row_ptr", "col_idx", "values", "rhs"):
        res[f"{strat}_{k}"] = full[k]
    s.close()
dist.destroy_process_group()
np.savez(out + f".{rank}.npz", **res)
"""


def _port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def test_two_ranks_gloo_one_gpu_bitwise(tmp_path):
    import paper_2302_07499_b200 as P
    from tests.helpers import SEED, U2
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    out = str(tmp_path / "mr")
    procs = [subprocess.Popen([sys.executable, "-c", CHILD, ROOT, str(r), "2", out], env=env,
                              cwd=ROOT) for r in range(2)]
    assert all(p.wait(timeout=600) == 0 for p in procs)
    m = P.generate_mesh(3, 6, 0.34, jitter_seed=5)
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    for r in range(2):
        got = np.load(f"{out}.{r}.npz")
        for strat, mc in (("fullcaps", 8), ("nocaps", 1)):
            s = P.Session(t, 0.34, strat, "moment2", U2, seed=SEED, mc_samples=mc)
            s.run()
            want = s.download()
            s.close()
            for k in ("row_ptr", "col_idx", "values", "rhs"):
                assert np.array_equal(got[f"{strat}_{k}"], want[k]), (r, strat, k)
