"""ctypes wrapper over oracle/_ref/libnlfem_ref.so -- TEST INFRASTRUCTURE ONLY.

Drives the *unmodified* reference library (compiled from /root/reference by
oracle/Makefile) through its own public API: generate_mesh, build_cmap,
build_element_table, build_dofmap, make_kernel, make_problem_from, assemble,
walk_ball, cg_solve, l2_error (see oracle/ref_driver.cpp for the file:line of
each).  Only tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libnlfem_ref.so")
STRATEGY = {"inside": 0, "overlap": 1, "barycenter": 2, "nocaps": 3,
            "approxcaps": 4, "fullcaps": 5}

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, u64, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double
        P = C.POINTER
        L.ref_mesh_generate.restype = vp
        L.ref_mesh_generate.argtypes = [C.c_int, dbl]
        L.ref_mesh_generate_n.restype = vp
        L.ref_mesh_generate_n.argtypes = [C.c_int, C.c_int, dbl]
        L.ref_mesh_dim.restype = C.c_int
        L.ref_mesh_dim.argtypes = [vp]
        L.ref_forcing_n.restype = C.c_int
        L.ref_forcing_n.argtypes = [C.c_int, dbl, C.c_int, vp, C.c_int, P(dbl), vp, C.c_int]
        L.ref_mesh_generate_jittered.restype = vp
        L.ref_mesh_generate_jittered.argtypes = [C.c_int, dbl, i64]
        L.ref_mesh_from_arrays.restype = vp
        L.ref_mesh_from_arrays.argtypes = [vp, i64, vp, vp, i64]
        L.ref_mesh_sizes.argtypes = [vp, P(i64), P(i64)]
        L.ref_mesh_copy.argtypes = [vp, vp, vp, vp]
        L.ref_mesh_free.argtypes = [vp]
        L.ref_problem_build.restype = vp
        L.ref_problem_build.argtypes = [vp, C.c_char_p, C.c_int]
        L.ref_problem_sizes.argtypes = [vp, P(i64), P(i64), P(i64)]
        L.ref_problem_copy.argtypes = [vp] * 12
        L.ref_problem_free.argtypes = [vp]
        L.ref_forcing.restype = C.c_int
        L.ref_forcing.argtypes = [dbl, C.c_int, vp, C.c_int, P(dbl), vp, C.c_int]
        L.ref_assemble.restype = vp
        L.ref_assemble.argtypes = [vp, dbl, C.c_int, C.c_int, vp, C.c_int, C.c_int,
                                   u64, C.c_int, C.c_char_p, C.c_int]
        L.ref_result_sizes.argtypes = [vp, P(i64), P(i64)]
        L.ref_result_copy.argtypes = [vp, vp, vp, vp, vp]
        L.ref_result_stats.argtypes = [vp, P(dbl), P(i32), P(i64), P(u64), P(u64)]
        L.ref_result_free.argtypes = [vp]
        L.ref_walk_pieces.restype = C.c_int
        L.ref_walk_pieces.argtypes = [vp, i32, C.c_int, dbl, C.c_int, vp, vp, C.c_int]
        L.ref_solve_l2.restype = C.c_int
        L.ref_solve_l2.argtypes = [vp, vp, vp, vp, vp, vp, C.c_int, dbl,
                                   P(dbl), P(dbl), P(i32)]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def generate_mesh(res: int, delta: float, jitter_seed: int | None = None):
    """Reference generate_mesh(3, res, delta) -> (coords, cells, region);
    jitter_seed: the config-3 interior-vertex jitter drawn with the
    reference's own nlfem::Rng (oracle/ref_driver.cpp)."""
    L = lib()
    h = (L.ref_mesh_generate(res, delta) if jitter_seed is None
         else L.ref_mesh_generate_jittered(res, delta, int(jitter_seed)))
    nn, nc = C.c_int64(), C.c_int64()
    L.ref_mesh_sizes(h, C.byref(nn), C.byref(nc))
    coords = np.empty((nn.value, 3), np.float64)
    cells = np.empty((nc.value, 4), np.int32)
    region = np.empty(nc.value, np.uint8)
    L.ref_mesh_copy(h, _p(coords), _p(cells), _p(region))
    L.ref_mesh_free(h)
    return coords, cells, region


class Problem:
    """Reference ElementTable + DofMap built from mesh arrays (3D), or from the
    reference's own generate_mesh in dimension n (Problem.generated)."""

    def __init__(self, coords, cells, region, _mesh_handle=None):
        L = lib()
        if _mesh_handle is None:
            coords = np.ascontiguousarray(coords, np.float64)
            cells = np.ascontiguousarray(cells, np.int32)
            region = np.ascontiguousarray(region, np.uint8)
            mh = L.ref_mesh_from_arrays(_p(coords), len(coords), _p(cells), _p(region),
                                        len(cells))
        else:
            mh = _mesh_handle
        self.n = L.ref_mesh_dim(mh)
        err = C.create_string_buffer(512)
        self.h = L.ref_problem_build(mh, err, 512)
        L.ref_mesh_free(mh)
        if not self.h:
            raise RuntimeError(err.value.decode())
        n, k, u = C.c_int64(), C.c_int64(), C.c_int64()
        L.ref_problem_sizes(self.h, C.byref(n), C.byref(k), C.byref(u))
        self.nodes, self.elems, self.unknowns = n.value, k.value, u.value

    @classmethod
    def generated(cls, n: int, res: int, delta: float):
        """The reference's generate_mesh(n, res, delta) -> cmap -> element table
        -> dof map (n = 2: the triangle path); also keeps the mesh arrays."""
        L = lib()
        mh = L.ref_mesh_generate_n(n, res, delta)
        nn, nc = C.c_int64(), C.c_int64()
        L.ref_mesh_sizes(mh, C.byref(nn), C.byref(nc))
        coords = np.empty((nn.value, 3), np.float64)
        cells = np.empty((nc.value, 4), np.int32)
        region = np.empty(nc.value, np.uint8)
        L.ref_mesh_copy(mh, _p(coords), _p(cells), _p(region))
        self = cls(None, None, None, _mesh_handle=mh)
        self.coords, self.cells, self.region = coords, cells[:, :n + 1].copy(), region
        return self

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_problem_free(self.h)
            self.h = None

    def table(self) -> dict:
        K, V = self.elems, self.nodes
        t = dict(verts=np.empty((K, 4), np.int32), neighbor=np.empty((K, 4), np.int32),
                 center=np.empty((K, 3)), radius=np.empty(K), volume=np.empty(K),
                 diam=np.empty(K), region=np.empty(K, np.uint8),
                 inv_edges=np.empty((K, 9)), simplex=np.empty((K, 4, 3)),
                 dof_of_node=np.empty(V, np.int32), constrained=np.empty(V, np.uint8))
        lib().ref_problem_copy(self.h, *[_p(t[k]) for k in (
            "verts", "neighbor", "center", "radius", "volume", "diam", "region",
            "inv_edges", "simplex", "dof_of_node", "constrained")])
        return t

    def assemble(self, delta, strategy, uterms, *, moment2=True, threads=0,
                 seed=0x5EED, mc_samples=200) -> dict:
        L = lib()
        ut = np.ascontiguousarray(uterms, np.float64)
        err = C.create_string_buffer(512)
        h = L.ref_assemble(self.h, delta, STRATEGY[strategy], int(moment2), _p(ut),
                           len(ut), threads, seed, mc_samples, err, 512)
        if not h:
            raise RuntimeError(err.value.decode())
        rows, nnz = C.c_int64(), C.c_int64()
        L.ref_result_sizes(h, C.byref(rows), C.byref(nnz))
        out = dict(row_ptr=np.empty(rows.value + 1, np.int32),
                   col_idx=np.empty(nnz.value, np.int32),
                   values=np.empty(nnz.value), rhs=np.empty(rows.value))
        L.ref_result_copy(h, _p(out["row_ptr"]), _p(out["col_idx"]), _p(out["values"]),
                          _p(out["rhs"]))
        s, th, bl, smp, hit = C.c_double(), C.c_int32(), C.c_int64(), C.c_uint64(), C.c_uint64()
        L.ref_result_stats(h, C.byref(s), C.byref(th), C.byref(bl), C.byref(smp), C.byref(hit))
        out.update(seconds=s.value, threads=th.value, blocks=bl.value,
                   mc_samples=smp.value, mc_hits=hit.value)
        L.ref_result_free(h)
        return out

    def walk_pieces(self, t, k, delta, strategy, maxout=200000):
        par = np.empty(maxout, np.int32)
        kind = np.empty(maxout, np.int32)
        n = lib().ref_walk_pieces(self.h, t, k, delta, STRATEGY[strategy], _p(par),
                                  _p(kind), maxout)
        if n < 0:
            raise RuntimeError(f"walk_ball failed ({n})")
        return par[:n].copy(), kind[:n].copy()

    def solve_l2(self, sys: dict, uterms, tol=1e-12):
        ut = np.ascontiguousarray(uterms, np.float64)
        l2, mx, it = C.c_double(), C.c_double(), C.c_int32()
        rc = lib().ref_solve_l2(self.h, _p(np.ascontiguousarray(sys["row_ptr"], np.int32)),
                                _p(np.ascontiguousarray(sys["col_idx"], np.int32)),
                                _p(np.ascontiguousarray(sys["values"], np.float64)),
                                _p(np.ascontiguousarray(sys["rhs"], np.float64)),
                                _p(ut), len(ut), tol, C.byref(l2), C.byref(mx), C.byref(it))
        return dict(l2=l2.value, max_nodal=mx.value, iterations=it.value, converged=rc == 0)


def forcing(delta, uterms, moment2=True, dim=3):
    """Reference make_kernel + make_problem_from -> (C, f terms)."""
    ut = np.ascontiguousarray(uterms, np.float64)
    Cc = C.c_double()
    f = np.empty((64, 4))
    n = lib().ref_forcing_n(dim, delta, int(moment2), _p(ut), len(ut), C.byref(Cc), _p(f), 64)
    return Cc.value, f[:n].copy()
