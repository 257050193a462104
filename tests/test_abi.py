"""The C-ABI library loads, exports every symbol include/*.h declares, and
fails loudly (no CPU fallback) when it cannot run on a B200."""
import ctypes
import os
import re

import pytest

import paper_2302_07499_b200 as P
from tests.helpers import U2, load_golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("nlfem_gpu.h", "nlfem_host.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(nlfem_(?:gpu|host)_\w+)\s*\(", src))
    return names


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(P.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 15
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(P.EXPORTED_SYMBOLS)


def test_version_names_arch():
    assert b"sm_100a" in P.lib().nlfem_gpu_version()


def test_sm100a_only_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def _table():
    g = load_golden("lat4_d030")
    return P.ElementTable(g["coords"], g["cells"], g["region"])


def test_bad_config_codes():
    t = _table()
    with pytest.raises(P.NlfemError) as ei:
        P.assemble(t, 0.3, "fullcaps", "moment2", U2, mc_samples=0)
    assert ei.value.name == "BadConfig"
    with pytest.raises(P.NlfemError) as ei:
        P.assemble(t, -1.0, "nocaps", "moment2", U2)
    assert ei.value.name == "BadConfig"
    with pytest.raises(P.NlfemError):
        P.assemble(t, 0.3, "nosuch", "moment2", U2)
    with pytest.raises(ValueError):
        P.assemble(t, 0.3, "nocaps", "nosuchnorm", U2)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.NlfemError) as ei:
        P.assemble(_table(), 0.3, "nocaps", "moment2", U2)
    assert ei.value.code == 100
