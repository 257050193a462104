"""bench.py --impl reference on the CPU: the unmodified reference (oracle/_ref)
through its own mesh generator and element table, the same `config` object as
the GPU arm, and nothing from paper_2302_07499_b200 loaded."""
import json
import os
import subprocess
import sys

import pytest

from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import io, json, os, runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--config", "C0", "--steps", "1", "--warmup", "0"]
try:
    runpy.run_path(os.path.join(sys.argv_root, "bench.py"), run_name="__main__")
except SystemExit:
    pass
loaded = sorted(m for m in sys.modules if m.startswith("paper_2302_07499_b200"))
maps = open("/proc/self/maps").read()
print("PROBE " + json.dumps({"modules": loaded, "gpu_so": "libnlfem_gpu.so" in maps}),
      file=sys.stderr)
"""


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_reference_arm_is_clean_and_shares_config():
    code = "import sys; sys.argv_root = %r\n" % ROOT + PROBE
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    probe = json.loads(r.stderr.split("PROBE ", 1)[1].splitlines()[0])
    assert probe == {"modules": [], "gpu_so": False}, probe
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    sys.path.insert(0, ROOT)
    import bench
    assert line["config"] == bench.bench_config("C0", bench.CONFIGS["C0"])
    assert line["e2e"]["h2d_bytes_per_step"] == 0
