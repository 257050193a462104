"""Precision of the one-word fixed-point scatter: the
same C4 (or CONFIG) assembly with the default library (unknown x unknown
entries keep the high word only) and with a -DNLFEM_FIXED_TWO=1 build (every
entry keeps both words, ~101 bits: the exact sum of the FP64 contributions up
to one final rounding).  Prints the row-normwise difference over the whole
matrix (|a - b| / max_k |a_ik|), computed on the device.

  python scripts/fixed_point_precision.py [CONFIG]     (needs both .so files)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TWO = os.path.join(ROOT, "paper_2302_07499_b200", "libnlfem_gpu_two.so")

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2302_07499_b200 as P
import bench
cfg = bench.CONFIGS[sys.argv[2]]
m = P.generate_mesh(3, cfg["res"], cfg["delta"], jitter_seed=cfg["jitter"])
t = P.ElementTable(m["coords"], m["cells"], m["region"], device=0)
s = P.Session(t, cfg["delta"], cfg["strategy"], "moment2", bench.U2, seed=bench.SEED,
              mc_samples=cfg["mc"], device=0)
s.run()
ro, ci, va, rh = (torch.as_tensor(x, device="cuda") for x in s.outputs())
torch.save({"values": va.cpu(), "rhs": rh.cpu(), "row_off": ro.cpu()}, sys.argv[3])
"""


def run(lib, out, cfg):
    env = dict(os.environ)
    if lib:
        env["NLFEM_GPU_LIB"] = lib
    subprocess.run([sys.executable, "-c", CHILD, ROOT, cfg, out], env=env, check=True)


def main():
    import torch
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    a, b = "/tmp/fp_one.pt", "/tmp/fp_two.pt"
    run(None, a, cfg)
    run(TWO, b, cfg)
    A, B = torch.load(a), torch.load(b)
    ro = A["row_off"].cuda()
    va, vb = A["values"].cuda(), B["values"].cuda()
    n = ro.numel() - 1
    rows = torch.repeat_interleave(torch.arange(n, device="cuda"), ro[1:] - ro[:-1])
    rmax = torch.zeros(n, dtype=torch.float64, device="cuda").scatter_reduce(
        0, rows, vb.abs(), "amax")
    rel = (va - vb).abs() / rmax[rows]
    rr = (A["rhs"] - B["rhs"]).abs().max() / B["rhs"].abs().max()
    print(json.dumps({"config": cfg, "nnz": int(va.numel()),
                      "max_row_rel_diff": float(rel.max()),
                      "mean_row_rel_diff": float(rel.mean()),
                      "p99_row_rel_diff": float(torch.quantile(rel[::97].float(), 0.99)),
                      "identical_entries": int((va == vb).sum()),
                      "rhs_rel_diff": float(rr)}))


if __name__ == "__main__":
    main()
