"""ctypes wrapper over oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

The restated CPU assembly (oracle/restated.cpp) consuming the same element
table arrays as the GPU C-ABI.  sampler="P" draws the Philox stream of
include/nlfem_mc_stream.h (the GPU's); sampler="R" reproduces the unmodified
reference's xoshiro stream (pinned against oracle/_ref by tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
STRATEGY = {"inside": 0, "overlap": 1, "barycenter": 2, "nocaps": 3, "approxcaps": 4,
            "fullcaps": 5}
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "restated.cpp")
    hdr = os.path.join(os.path.dirname(_HERE), "include", "nlfem_mc_stream.h")
    if force or not os.path.exists(LIB_PATH) or max(os.path.getmtime(src), os.path.getmtime(hdr)) > os.path.getmtime(LIB_PATH):
        subprocess.run(["make", "-C", _HERE, "port"], check=True, capture_output=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
        L.oracle_assemble.restype = vp
        L.oracle_assemble.argtypes = [C.c_int, C.c_int] + [vp] * 10 + [C.c_int, dbl, dbl, vp, C.c_int,
                                      vp, C.c_int, C.c_int, u64, C.c_int, C.c_int, C.c_int,
                                      vp, i64, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.oracle_result_sizes.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.oracle_result_copy.argtypes = [vp, vp, vp, vp, vp]
        L.oracle_result_stats.argtypes = [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(i32),
                                          C.POINTER(u64)]
        L.oracle_result_free.argtypes = [vp]
        L.oracle_philox.argtypes = [vp, C.c_uint32, C.c_uint32, vp]
        L.oracle_mc_fields.argtypes = [u64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_int, vp]
        L.oracle_cg.restype = C.c_int
        L.oracle_cg.argtypes = [C.c_int, vp, vp, vp, vp, dbl, C.c_int, vp, C.POINTER(i32)]
        L.oracle_l2_error.restype = dbl
        L.oracle_l2_error.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, C.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def assemble(table, delta, strategy, C_kernel, fterms, gterms, *, seed=0x5EED,
             mc_samples=200, sampler="P", threads=0, outer=None) -> dict:
    """Restated nlfem::assemble on a paper_2302_07499_b200.ElementTable-like object.

    outer: optional interior element ids -- integrate only these outer elements
    (the partial system of a sample, for parity at full mesh sizes)."""
    L = lib()
    f = np.ascontiguousarray(fterms, np.float64)
    g = np.ascontiguousarray(gterms, np.float64)
    code = C.c_int()
    err = C.create_string_buffer(512)
    threads = threads or os.cpu_count() or 1
    t = table
    ov = None if outer is None else np.ascontiguousarray(outer, np.int32)
    h = L.oracle_assemble(t.elem_count, t.node_count, _p(t.coords), _p(t.verts), _p(t.neighbor),
                          _p(t.center), _p(t.radius), _p(t.volume), _p(t.diam), _p(t.region),
                          _p(t.inv_edges), _p(t.dof_of_node), t.unknowns, C_kernel, delta,
                          _p(f), len(f), _p(g), len(g), STRATEGY[strategy], seed & (2**64 - 1),
                          mc_samples, {"P": 0, "R": 1}[sampler], threads,
                          None if ov is None else _p(ov), 0 if ov is None else len(ov),
                          C.byref(code), err, 512)
    if not h:
        raise OracleError(code.value, err.value.decode())
    rows, nnz = C.c_int64(), C.c_int64()
    L.oracle_result_sizes(h, C.byref(rows), C.byref(nnz))
    out = dict(row_ptr=np.empty(rows.value + 1, np.int32), col_idx=np.empty(nnz.value, np.int32),
               values=np.empty(nnz.value), rhs=np.empty(rows.value))
    L.oracle_result_copy(h, _p(out["row_ptr"]), _p(out["col_idx"]), _p(out["values"]), _p(out["rhs"]))
    md, mh, bl, npr = C.c_uint64(), C.c_uint64(), C.c_int32(), C.c_uint64()
    L.oracle_result_stats(h, C.byref(md), C.byref(mh), C.byref(bl), C.byref(npr))
    out.update(mc_samples=md.value, mc_hits=mh.value, blocks=bl.value, element_pairs=npr.value)
    L.oracle_result_free(h)
    return out


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    o = np.empty(4, np.uint32)
    lib().oracle_philox(_p(c), int(key[0]), int(key[1]), _p(o))
    return o


def mc_fields(seed, T, Tp, q, sub, j0, nblocks):
    """Unsorted 21-bit fields of the 3D Monte Carlo stream, shape (4 nblocks, 3)."""
    o = np.empty((4 * nblocks, 3), np.uint32)
    lib().oracle_mc_fields(int(seed), T, Tp, q, sub, j0, nblocks, _p(o))
    return o


def solve_l2(table, sys, uterms, tol=1e-12):
    """Reference-style CG from zero + L2 error of the P1 solution (harness check)."""
    L = lib()
    n = len(sys["rhs"])
    x = np.zeros(n)
    it = C.c_int32()
    rc = L.oracle_cg(n, _p(np.ascontiguousarray(sys["row_ptr"], np.int32)),
                     _p(np.ascontiguousarray(sys["col_idx"], np.int32)),
                     _p(np.ascontiguousarray(sys["values"], np.float64)),
                     _p(np.ascontiguousarray(sys["rhs"], np.float64)), tol, 100 * max(n, 1),
                     _p(x), C.byref(it))
    u = np.ascontiguousarray(uterms, np.float64)
    nv = np.empty(table.node_count)
    from math import prod  # noqa: F401  (keeps eval order explicit below)
    for v in range(table.node_count):
        if table.dof_of_node[v] >= 0:
            nv[v] = x[table.dof_of_node[v]]
        else:
            p = table.coords[v]
            acc = 0.0
            for c, e0, e1, e2 in u:
                val = c
                for _ in range(int(e0)):
                    val *= p[0]
                for _ in range(int(e1)):
                    val *= p[1]
                for _ in range(int(e2)):
                    val *= p[2]
                acc += val
            nv[v] = acc
    l2 = L.oracle_l2_error(table.elem_count, _p(table.coords), _p(table.verts), _p(table.region),
                           _p(table.volume), _p(nv), _p(u), len(u))
    return dict(l2=l2, iterations=it.value, converged=rc == 0, u=x)
