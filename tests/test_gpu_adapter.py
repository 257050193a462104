"""The drop-in, end to end: the reference's own C++ upstream feeds both the
unmodified nlfem::assemble and nlfem::gpu::assemble (include/nlfem_gpu_adapter.hpp),
compiled into oracle/_ref/adapter_demo (needs the reference build)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "adapter_demo")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DEMO), reason="oracle/_ref/adapter_demo not built")
@pytest.mark.parametrize("strat", ["inside", "overlap", "barycenter", "nocaps", "approxcaps",
                                   "fullcaps"])
def test_adapter_drop_in_matches_reference(strat):
    out = subprocess.run([DEMO, "6", "0.34", strat], capture_output=True, text=True, timeout=600)
    rec = json.loads(out.stdout.strip().splitlines()[-1])
    assert rec.get("pattern_equal") is True, rec
    if strat != "fullcaps":
        assert rec["max_row_rel_err"] <= 1e-12, rec
        assert rec["rhs_rel_err"] <= 1e-12, rec
    else:
        # same Monte Carlo regions: identical number of draws
        assert rec["mc_samples_gpu"] == rec["mc_samples_ref"], rec


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DEMO), reason="oracle/_ref/adapter_demo not built")
@pytest.mark.parametrize("strat", ["inside", "overlap", "barycenter", "nocaps", "approxcaps",
                                   "fullcaps"])
def test_adapter_drop_in_2d_matches_reference(strat):
    # a 2D ElementTable (et.n == 2) through the same nlfem::gpu::assemble call
    out = subprocess.run([DEMO, "16", str(3 / 16), strat, "2"], capture_output=True, text=True,
                         timeout=600)
    rec = json.loads(out.stdout.strip().splitlines()[-1])
    assert rec.get("pattern_equal") is True, rec
    if strat != "fullcaps":
        assert rec["max_row_rel_err"] <= 1e-12, rec
        assert rec["rhs_rel_err"] <= 1e-12, rec
    else:
        assert rec["mc_samples_gpu"] == rec["mc_samples_ref"], rec


def test_adapter_header_compiles_against_reference_types():
    # CPU-side check: the adapter builds against the reference headers
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference headers not present")
    src = "#include \"nlfem/assembly.hpp\"\n#include \"nlfem_gpu_adapter.hpp\"\nint main(){return 0;}\n"
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-x", "c++", "-",
                        "-I/root/reference/proj/include", "-I" + os.path.join(ROOT, "include")],
                       input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
