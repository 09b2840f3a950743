"""CPU oracle of the Parthenon-hydro per-cycle update (arXiv 2202.12309, §4.1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2202_12309_b200``) never imports it, and the
two share no code: this is a ctypes wrapper around ``oracle/liboracle.so``, which
is built from ``oracle/oracle.cpp`` alone (plain scalar C++, ``-O2
-ffp-contract=off``).

Parity status per function ("Oracle pins"):
  cons<->prim, PLM (minmod, van Leer, MC), HLLE (Davis and Einfeldt), restriction, prolongation,
  Morton, partition, tree/2:1, neighbours, exchange, flux correction, dt, totals, RK2, VL2
                                                           -> pinned (tests/test_oracle_*.py)
  AMR refinement criterion (A14: closed form on a linear pressure)  -> pinned
  physical BCs on fine ghosts and coarse staging, staging geometry at walls (A12)
                                                           -> pinned (method of images)
  derefinement (A16 gate, family rule, 2:1 on derefinement) -> pinned (closed-form block counts,
                                                              tests/test_oracle_exchange.py)
  PPM / WENO-Z (A37 / A38; the paper names neither)        -> pinned by their textbook definitions
                                                              (tests/test_oracle_highorder.py)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

PERIODIC, OUTFLOW, REFLECT = 0, 1, 2
MINMOD, VANLEER, MC, PPM, WENOZ = 0, 1, 2, 3, 4
RK2, VL2 = 0, 1
LINEAR_WAVE, SOD, BLAST, KH = 0, 1, 2, 3
REF_NONE, REF_STATIC, REF_ADAPTIVE = 0, 1, 2
DAVIS, EINFELDT = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -ffp-contract=off -fopenmp)."""
    hdr = os.path.join(_HERE, "oracle.h")
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= max(os.path.getmtime(_SRC), os.path.getmtime(hdr))):
        return _LIB
    cmd = ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-std=c++17",
           "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC]
    subprocess.check_call(cmd, cwd=_HERE)
    os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Cfg(C.Structure):
    _fields_ = [
        ("mesh_nx", C.c_int64 * 3), ("block_nx", C.c_int64 * 3),
        ("nghost", C.c_int32), ("max_level", C.c_int32),
        ("xmin", C.c_double * 3), ("xmax", C.c_double * 3),
        ("bc_inner", C.c_int32 * 3), ("bc_outer", C.c_int32 * 3),
        ("gamma", C.c_double), ("cfl", C.c_double),
        ("recon", C.c_int32), ("integrator", C.c_int32),
        ("refinement", C.c_int32),
        ("refine_tol", C.c_double), ("derefine_tol", C.c_double),
        ("derefine_interval", C.c_int32),
        ("nregions", C.c_int32), ("regions", C.POINTER(C.c_double)),
        ("nranks", C.c_int32), ("nthreads", C.c_int32),
        ("wavespeed", C.c_int32),
    ]


class OrcBlock(C.Structure):
    _fields_ = [("gid", C.c_int64), ("level", C.c_int32), ("rank", C.c_int32),
                ("lx", C.c_int64 * 3), ("xmin", C.c_double * 3), ("xmax", C.c_double * 3)]


class OrcNeighbor(C.Structure):
    _fields_ = [("gid", C.c_int64), ("rank", C.c_int32), ("off", C.c_int8 * 3),
                ("dlevel", C.c_int8), ("fine", C.c_int8 * 2)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        dp = C.POINTER(C.c_double)
        L.orc_last_error.restype = C.c_char_p
        L.orc_cons_to_prim.argtypes = [dp, C.c_double, dp]
        L.orc_prim_to_cons.argtypes = [dp, C.c_double, dp]
        L.orc_prim_to_cons.restype = None
        L.orc_plm.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int32, dp, dp]
        L.orc_plm.restype = None
        L.orc_recon5.argtypes = [dp, C.c_int32, dp, dp]
        L.orc_recon5.restype = None
        L.orc_hlle.argtypes = [dp, dp, C.c_double, dp]
        L.orc_hlle.restype = None
        L.orc_hlle_ws.argtypes = [dp, dp, C.c_double, C.c_int32, dp]
        L.orc_hlle_ws.restype = None
        L.orc_flux_phys.argtypes = [dp, C.c_double, dp]
        L.orc_flux_phys.restype = None
        L.orc_restrict8.argtypes = [dp]
        L.orc_restrict8.restype = C.c_double
        L.orc_prolong.argtypes = [C.c_double, dp, dp, dp]
        L.orc_prolong.restype = None
        L.orc_morton_key.argtypes = [C.c_int32, C.POINTER(C.c_int64), C.c_int32]
        L.orc_morton_key.restype = C.c_uint64
        L.orc_partition.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_partition.restype = None
        L.orc_pairwise_sum.argtypes = [dp, C.c_int64]
        L.orc_pairwise_sum.restype = C.c_double
        L.orc_mesh_create.argtypes = [C.POINTER(_Cfg), C.POINTER(C.c_void_p)]
        for name in ("orc_mesh_destroy", "orc_exchange", "orc_tag_and_remesh"):
            getattr(L, name).argtypes = [C.c_void_p]
        L.orc_set_problem.argtypes = [C.c_void_p, C.c_int32, dp, C.c_int32]
        for name in ("orc_set_state", "orc_get_state", "orc_get_state_full", "orc_set_state_full"):
            getattr(L, name).argtypes = [C.c_void_p, C.c_int64, dp, C.c_int64]
        L.orc_compute_dt.argtypes = [C.c_void_p, dp]
        L.orc_step.argtypes = [C.c_void_p, C.c_int32, C.c_double]
        L.orc_get_time.argtypes = [C.c_void_p, dp, dp, C.POINTER(C.c_int64)]
        L.orc_num_blocks.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.orc_get_blocks.argtypes = [C.c_void_p, C.POINTER(OrcBlock), C.c_int64, C.POINTER(C.c_int64)]
        L.orc_get_neighbors.argtypes = [C.c_void_p, C.c_int64, C.POINTER(OrcNeighbor), C.c_int32,
                                        C.POINTER(C.c_int32)]
        L.orc_get_refine_flags.argtypes = [C.c_void_p, C.POINTER(C.c_int8), C.c_int64, C.POINTER(C.c_int64)]
        L.orc_get_indicators.argtypes = [C.c_void_p, dp, C.c_int64, C.POINTER(C.c_int64)]
        L.orc_get_history.argtypes = [C.c_void_p, dp, C.c_int64, C.POINTER(C.c_int64)]
        L.orc_totals.argtypes = [C.c_void_p, dp]
        L.orc_level_counts.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int32]
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class OracleError(RuntimeError):
    pass


def _check(rc: int):
    if rc != 0:
        raise OracleError(f"oracle error {rc}: {lib().orc_last_error().decode()}")


# ---------------------------------------------------------------- point functions
def cons_to_prim(U, gamma):
    U = np.ascontiguousarray(U, dtype=np.float64)
    W = np.zeros(5)
    rc = lib().orc_cons_to_prim(_dp(U), gamma, _dp(W))
    return W, rc


def prim_to_cons(W, gamma):
    W = np.ascontiguousarray(W, dtype=np.float64)
    U = np.zeros(5)
    lib().orc_prim_to_cons(_dp(W), gamma, _dp(U))
    return U


def plm(qm, q0, qp, recon=MINMOD):
    a, b = C.c_double(), C.c_double()
    lib().orc_plm(qm, q0, qp, recon, C.byref(a), C.byref(b))
    return a.value, b.value


def recon5(q, recon):
    q = np.ascontiguousarray(q, dtype=np.float64)
    a, b = C.c_double(), C.c_double()
    lib().orc_recon5(_dp(q), recon, C.byref(a), C.byref(b))
    return a.value, b.value


def hlle(WL, WR, gamma, wavespeed=DAVIS):
    WL = np.ascontiguousarray(WL, dtype=np.float64)
    WR = np.ascontiguousarray(WR, dtype=np.float64)
    F = np.zeros(5)
    if wavespeed == DAVIS:
        lib().orc_hlle(_dp(WL), _dp(WR), gamma, _dp(F))
    else:
        lib().orc_hlle_ws(_dp(WL), _dp(WR), gamma, wavespeed, _dp(F))
    return F


def flux_phys(W, gamma):
    W = np.ascontiguousarray(W, dtype=np.float64)
    F = np.zeros(5)
    lib().orc_flux_phys(_dp(W), gamma, _dp(F))
    return F


def restrict8(v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    return lib().orc_restrict8(_dp(v))


def prolong(c, cm, cp):
    cm = np.ascontiguousarray(cm, dtype=np.float64)
    cp = np.ascontiguousarray(cp, dtype=np.float64)
    out = np.zeros(8)
    lib().orc_prolong(c, _dp(cm), _dp(cp), _dp(out))
    return out


def morton_key(level, lx, max_level):
    a = (C.c_int64 * 3)(*lx)
    return lib().orc_morton_key(level, a, max_level)


def partition(nblocks, nranks, rank):
    lo, hi = C.c_int64(), C.c_int64()
    lib().orc_partition(nblocks, nranks, rank, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def pairwise_sum(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().orc_pairwise_sum(_dp(a), a.size)


# ---------------------------------------------------------------- mesh
DEFAULTS = dict(
    mesh_nx=(32, 32, 32), block_nx=(32, 32, 32), nghost=2, max_level=0,
    xmin=(0.0, 0.0, 0.0), xmax=(1.0, 1.0, 1.0),
    bc_inner=(PERIODIC,) * 3, bc_outer=(PERIODIC,) * 3,
    gamma=5.0 / 3.0, cfl=0.3, recon=MINMOD, integrator=RK2,
    refinement=REF_NONE, refine_tol=0.1, derefine_tol=0.025, derefine_interval=8,
    regions=(), nranks=1, nthreads=0, wavespeed=DAVIS,
)


class Mesh:
    """One oracle mesh (all simulated ranks in one address space)."""

    def __init__(self, **kw):
        c = dict(DEFAULTS)
        unknown = set(kw) - set(c) - {"pack_size"}
        if unknown:
            raise TypeError(f"unknown config keys {unknown}")
        c.update({k: v for k, v in kw.items() if k in c})
        self.cfgdict = c
        cfg = _Cfg()
        cfg.mesh_nx[:] = list(c["mesh_nx"])
        cfg.block_nx[:] = list(c["block_nx"])
        cfg.nghost = c["nghost"]
        cfg.max_level = c["max_level"]
        cfg.xmin[:] = list(c["xmin"])
        cfg.xmax[:] = list(c["xmax"])
        cfg.bc_inner[:] = list(c["bc_inner"])
        cfg.bc_outer[:] = list(c["bc_outer"])
        cfg.gamma = c["gamma"]
        cfg.cfl = c["cfl"]
        cfg.recon = c["recon"]
        cfg.integrator = c["integrator"]
        cfg.refinement = c["refinement"]
        cfg.refine_tol = c["refine_tol"]
        cfg.derefine_tol = c["derefine_tol"]
        cfg.derefine_interval = c["derefine_interval"]
        regs = np.ascontiguousarray(np.asarray(c["regions"], dtype=np.float64).reshape(-1))
        self._regs = regs
        cfg.nregions = regs.size // 7
        cfg.regions = _dp(regs) if regs.size else None
        cfg.nranks = c["nranks"]
        cfg.nthreads = c["nthreads"]
        cfg.wavespeed = c["wavespeed"]
        self._cfg = cfg
        h = C.c_void_p()
        _check(lib().orc_mesh_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self.n = tuple(int(x) for x in c["block_nx"])
        self.g = int(c["nghost"])

    def close(self):
        if getattr(self, "_h", None):
            lib().orc_mesh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- state
    def set_problem(self, problem, params=()):
        p = np.ascontiguousarray(params, dtype=np.float64)
        _check(lib().orc_set_problem(self._h, problem, _dp(p) if p.size else None, p.size))

    def num_blocks(self):
        n = C.c_int64()
        lib().orc_num_blocks(self._h, C.byref(n))
        return n.value

    def get_state(self, gid):
        n1, n2, n3 = self.n
        out = np.zeros((5, n3, n2, n1))
        _check(lib().orc_get_state(self._h, gid, _dp(out), out.size))
        return out

    def set_state(self, gid, cons):
        a = np.ascontiguousarray(cons, dtype=np.float64)
        _check(lib().orc_set_state(self._h, gid, _dp(a), a.size))

    def get_state_full(self, gid):
        n1, n2, n3 = self.n
        g = self.g
        out = np.zeros((5, n3 + 2 * g, n2 + 2 * g, n1 + 2 * g))
        _check(lib().orc_get_state_full(self._h, gid, _dp(out), out.size))
        return out

    def set_state_full(self, gid, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        _check(lib().orc_set_state_full(self._h, gid, _dp(a), a.size))

    def all_states(self):
        return np.stack([self.get_state(b) for b in range(self.num_blocks())])

    def exchange(self):
        _check(lib().orc_exchange(self._h))

    def compute_dt(self):
        d = C.c_double()
        _check(lib().orc_compute_dt(self._h, C.byref(d)))
        return d.value

    def step(self, ncycles, tlim=0.0):
        _check(lib().orc_step(self._h, ncycles, tlim))

    def tag_and_remesh(self):
        _check(lib().orc_tag_and_remesh(self._h))

    def time(self):
        t, dt, cyc = C.c_double(), C.c_double(), C.c_int64()
        lib().orc_get_time(self._h, C.byref(t), C.byref(dt), C.byref(cyc))
        return t.value, dt.value, cyc.value

    # --- mesh queries
    def blocks(self):
        n = self.num_blocks()
        arr = (OrcBlock * max(n, 1))()
        cnt = C.c_int64()
        lib().orc_get_blocks(self._h, arr, n, C.byref(cnt))
        return [dict(gid=b.gid, level=b.level, rank=b.rank, lx=tuple(b.lx),
                     xmin=tuple(b.xmin), xmax=tuple(b.xmax)) for b in arr[:n]]

    def neighbors(self, gid):
        arr = (OrcNeighbor * 64)()
        cnt = C.c_int32()
        _check(lib().orc_get_neighbors(self._h, gid, arr, 64, C.byref(cnt)))
        return [dict(gid=e.gid, rank=e.rank, off=tuple(e.off), dlevel=e.dlevel, fine=tuple(e.fine))
                for e in arr[:cnt.value]]

    def refine_flags(self):
        n = self.num_blocks() * 8 + 8
        arr = (C.c_int8 * n)()
        cnt = C.c_int64()
        lib().orc_get_refine_flags(self._h, arr, n, C.byref(cnt))
        return np.array(arr[:cnt.value], dtype=np.int8)

    def indicators(self):
        n = self.num_blocks() * 8 + 8
        out = np.zeros(n)
        cnt = C.c_int64()
        lib().orc_get_indicators(self._h, _dp(out), n, C.byref(cnt))
        return out[:cnt.value]

    def history(self):
        cap = 100000
        out = np.zeros((cap, 7))
        n = C.c_int64()
        lib().orc_get_history(self._h, _dp(out), cap, C.byref(n))
        return out[:n.value].copy()

    def totals(self):
        out = np.zeros(5)
        lib().orc_totals(self._h, _dp(out))
        return out

    def level_counts(self, cap=12):
        out = (C.c_int64 * cap)()
        lib().orc_level_counts(self._h, out, cap)
        return list(out)
