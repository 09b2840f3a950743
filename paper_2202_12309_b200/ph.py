"""ctypes binding of include/ph.h (argument marshalling only).

Names follow the C ABI.  PyTorch provides device memory (caching allocator), the CUDA
stream and, for multi-GPU runs, the process group used to broadcast the NCCL unique id.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.environ.get("PH_LIB") or os.path.join(_HERE, "libph.so")  # PH_LIB: A/B builds

PERIODIC, OUTFLOW, REFLECT = 0, 1, 2
MINMOD, VANLEER, MC, PPM, WENOZ = 0, 1, 2, 3, 4
RK2, VL2 = 0, 1
LINEAR_WAVE, SOD, BLAST, KH = 0, 1, 2, 3
REF_NONE, REF_STATIC, REF_ADAPTIVE = 0, 1, 2
ABI_VERSION = 3
DAVIS, EINFELDT = 0, 1
HALO_AUTO, HALO_NCCL, HALO_PEER = 0, 1, 2

_ALLOC = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
_FREE = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class _Cfg(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("nghost", C.c_int32),
        ("mesh_nx", C.c_int64 * 3), ("block_nx", C.c_int64 * 3),
        ("max_level", C.c_int32), ("refinement", C.c_int32),
        ("xmin", C.c_double * 3), ("xmax", C.c_double * 3),
        ("bc_inner", C.c_int32 * 3), ("bc_outer", C.c_int32 * 3),
        ("gamma", C.c_double), ("cfl", C.c_double),
        ("recon", C.c_int32), ("integrator", C.c_int32),
        ("refine_tol", C.c_double), ("derefine_tol", C.c_double),
        ("derefine_interval", C.c_int32),
        ("nregions", C.c_int32), ("regions", C.POINTER(C.c_double)),
        ("pack_size", C.c_int32),
        ("rank", C.c_int32), ("nranks", C.c_int32), ("device", C.c_int32), ("host_only", C.c_int32),
        ("no_direct_halo", C.c_int32),
        ("stream", C.c_void_p), ("nccl_id", C.c_void_p),
        ("dev_alloc", _ALLOC), ("dev_free", _FREE), ("alloc_ctx", C.c_void_p),
        ("halo_transport", C.c_int32), ("wavespeed", C.c_int32),
    ]


class PhBlock(C.Structure):
    _fields_ = [("gid", C.c_int64), ("level", C.c_int32), ("rank", C.c_int32),
                ("lx", C.c_int64 * 3), ("xmin", C.c_double * 3), ("xmax", C.c_double * 3)]


class PhNeighbor(C.Structure):
    _fields_ = [("gid", C.c_int64), ("rank", C.c_int32), ("off", C.c_int8 * 3),
                ("dlevel", C.c_int8), ("fine", C.c_int8 * 2)]


class PhStepInfo(C.Structure):
    _fields_ = [("cycle", C.c_int64), ("t", C.c_double), ("dt", C.c_double), ("zone_cycles", C.c_int64)]


class PhPlanInfo(C.Structure):
    _fields_ = [("n_local_tasks", C.c_int64), ("n_send_tasks", C.c_int64), ("n_recv_tasks", C.c_int64),
                ("send_doubles_to", C.c_int64 * 64), ("recv_doubles_from", C.c_int64 * 64),
                ("send_hash_to", C.c_uint64 * 64), ("recv_hash_from", C.c_uint64 * 64),
                ("cyc_send_doubles_to", C.c_int64 * 64), ("cyc_recv_doubles_from", C.c_int64 * 64),
                ("cyc_send_hash_to", C.c_uint64 * 64), ("cyc_recv_hash_from", C.c_uint64 * 64),
                ("direct_halo", C.c_int32), ("n_cyc_local_tasks", C.c_int64), ("peer_halo", C.c_int32)]


EXPORTS = ["ph_nccl_unique_id", "ph_mesh_create", "ph_mesh_destroy", "ph_set_problem", "ph_set_state",
           "ph_refresh", "ph_get_state", "ph_get_state_full", "ph_set_state_full", "ph_exchange", "ph_step",
           "ph_step_host", "ph_num_blocks", "ph_get_blocks", "ph_get_neighbors", "ph_get_refine_flags",
           "ph_get_history", "ph_get_time", "ph_totals", "ph_get_plan_info", "ph_launch_count",
           "ph_kernel_timing", "ph_last_error", "ph_step_host_async", "ph_sync"]

_lib = None
_LIVE = __import__("weakref").WeakSet()


def _close_all():
    for m in list(_LIVE):
        try:
            m.close()
        except Exception:
            pass


__import__("atexit").register(_close_all)


def lib():
    """Load libph.so (fails loudly if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIBPATH):
            raise ImportError(f"{_LIBPATH} is missing: run `python -m paper_2202_12309_b200._build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(_LIBPATH)
        dp = C.POINTER(C.c_double)
        vp = C.c_void_p
        L.ph_last_error.restype = C.c_char_p
        L.ph_nccl_unique_id.argtypes = [vp, C.c_int32]
        L.ph_mesh_create.argtypes = [C.POINTER(_Cfg), C.POINTER(vp)]
        L.ph_mesh_destroy.argtypes = [vp]
        L.ph_set_problem.argtypes = [vp, C.c_int32, dp, C.c_int32]
        for n in ("ph_set_state", "ph_get_state", "ph_get_state_full", "ph_set_state_full"):
            getattr(L, n).argtypes = [vp, C.c_int64, dp, C.c_int64]
        L.ph_refresh.argtypes = [vp]
        L.ph_exchange.argtypes = [vp]
        L.ph_step.argtypes = [vp, C.c_int32, C.c_double, C.POINTER(PhStepInfo)]
        L.ph_step_host.argtypes = [vp, vp, vp, C.c_int64, C.c_int32, C.c_double]
        L.ph_step_host_async.argtypes = [vp, vp, vp, C.c_int64, C.c_int32, C.c_double]
        L.ph_sync.argtypes = [vp]
        L.ph_num_blocks.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ph_get_blocks.argtypes = [vp, C.POINTER(PhBlock), C.c_int64, C.POINTER(C.c_int64)]
        L.ph_get_neighbors.argtypes = [vp, C.c_int64, C.POINTER(PhNeighbor), C.c_int32, C.POINTER(C.c_int32)]
        L.ph_get_refine_flags.argtypes = [vp, C.POINTER(C.c_int8), C.c_int64, C.POINTER(C.c_int64)]
        L.ph_get_history.argtypes = [vp, dp, C.c_int64, C.POINTER(C.c_int64)]
        L.ph_get_time.argtypes = [vp, dp, dp, C.POINTER(C.c_int64)]
        L.ph_totals.argtypes = [vp, dp]
        L.ph_get_plan_info.argtypes = [vp, C.POINTER(PhPlanInfo)]
        L.ph_launch_count.argtypes = [vp, C.POINTER(C.c_int64)]
        L.ph_kernel_timing.argtypes = [vp, C.c_int32, dp, C.POINTER(C.c_int64), dp, C.POINTER(C.c_int64)]
        _lib = L
    return _lib


class PhError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"ph error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise PhError(rc, lib().ph_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


DEFAULTS = dict(
    mesh_nx=(32, 32, 32), block_nx=(32, 32, 32), nghost=2, max_level=0, refinement=REF_NONE,
    xmin=(0.0, 0.0, 0.0), xmax=(1.0, 1.0, 1.0),
    bc_inner=(PERIODIC,) * 3, bc_outer=(PERIODIC,) * 3,
    gamma=5.0 / 3.0, cfl=0.3, recon=MINMOD, integrator=RK2,
    refine_tol=0.1, derefine_tol=0.025, derefine_interval=8, regions=(), pack_size=0,
    direct_halo=True, halo_transport=HALO_AUTO, wavespeed=DAVIS,
)


class Mesh:
    """Handle of one ph_mesh (one rank).  Config keys as in include/ph.h."""

    def __init__(self, device=0, rank=0, nranks=1, host_only=False, stream=None, torch_alloc=True,
                 process_group=None, nccl_id=None, **kw):
        c = dict(DEFAULTS)
        unknown = set(kw) - set(c) - {"nranks_sim", "nthreads"}
        if unknown:
            raise TypeError(f"unknown config keys {unknown}")
        c.update({k: v for k, v in kw.items() if k in c})
        self.cfgdict = c
        cfg = _Cfg()
        cfg.abi_version = ABI_VERSION
        cfg.nghost = c["nghost"]
        cfg.mesh_nx[:] = list(c["mesh_nx"])
        cfg.block_nx[:] = list(c["block_nx"])
        cfg.max_level = c["max_level"]
        cfg.refinement = c["refinement"]
        cfg.xmin[:] = list(c["xmin"])
        cfg.xmax[:] = list(c["xmax"])
        cfg.bc_inner[:] = list(c["bc_inner"])
        cfg.bc_outer[:] = list(c["bc_outer"])
        cfg.gamma = c["gamma"]
        cfg.cfl = c["cfl"]
        cfg.recon = c["recon"]
        cfg.integrator = c["integrator"]
        cfg.refine_tol = c["refine_tol"]
        cfg.derefine_tol = c["derefine_tol"]
        cfg.derefine_interval = c["derefine_interval"]
        regs = np.ascontiguousarray(np.asarray(c["regions"], dtype=np.float64).reshape(-1))
        self._regs = regs
        cfg.nregions = regs.size // 7
        cfg.regions = _dp(regs) if regs.size else None
        cfg.pack_size = c["pack_size"]
        cfg.rank, cfg.nranks, cfg.device = rank, nranks, device
        cfg.host_only = 1 if host_only else 0
        cfg.no_direct_halo = 0 if c["direct_halo"] else 1
        cfg.halo_transport = c["halo_transport"]
        cfg.wavespeed = c["wavespeed"]
        self._keep = []
        if not host_only:
            import torch
            torch.cuda.set_device(device)
            if stream is None:
                stream = torch.cuda.current_stream(device)
            self.stream = stream
            cfg.stream = C.c_void_p(stream.cuda_stream)
            if torch_alloc:
                dev = device
                _calloc = torch.cuda.caching_allocator_alloc
                _cfree = torch.cuda.caching_allocator_delete

                def _alloc(nbytes, ctx, _s=stream):
                    try:
                        return _calloc(int(nbytes), dev, _s)
                    except Exception:
                        return None

                def _free(ptr, ctx):
                    try:
                        _cfree(ptr)
                    except Exception:
                        pass  # interpreter shutdown: the process is exiting anyway

                a, f = _ALLOC(_alloc), _FREE(_free)
                self._keep += [a, f]
                cfg.dev_alloc, cfg.dev_free = a, f
            if nranks > 1:
                if nccl_id is None:
                    nccl_id = Mesh.make_nccl_id(rank, process_group)
                idbuf = C.create_string_buffer(bytes(nccl_id), 128)
                self._keep.append(idbuf)
                cfg.nccl_id = C.cast(idbuf, C.c_void_p)
        self._cfg = cfg
        h = C.c_void_p()
        _check(lib().ph_mesh_create(C.byref(cfg), C.byref(h)))
        self._h = h
        _LIVE.add(self)
        self.n = tuple(int(x) for x in c["block_nx"])
        self.g = int(c["nghost"])
        self.rank, self.nranks = rank, nranks
        self.host_only = host_only

    @staticmethod
    def make_nccl_id(rank, process_group=None):
        """rank 0 creates the ncclUniqueId; torch.distributed broadcasts it (plumbing only)."""
        import torch.distributed as dist
        buf = C.create_string_buffer(128)
        if rank == 0:
            _check(lib().ph_nccl_unique_id(buf, 128))
        obj = [bytes(buf.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=process_group)
        return obj[0]

    def close(self):
        if getattr(self, "_h", None):
            lib().ph_mesh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ state
    def set_problem(self, problem, params=()):
        p = np.ascontiguousarray(params, dtype=np.float64)
        _check(lib().ph_set_problem(self._h, problem, _dp(p) if p.size else None, p.size))

    def num_blocks(self):
        g, l = C.c_int64(), C.c_int64()
        lib().ph_num_blocks(self._h, C.byref(g), C.byref(l))
        return g.value

    def num_local(self):
        g, l = C.c_int64(), C.c_int64()
        lib().ph_num_blocks(self._h, C.byref(g), C.byref(l))
        return l.value

    def set_state(self, gid, cons):
        a = np.ascontiguousarray(cons, dtype=np.float64)
        _check(lib().ph_set_state(self._h, gid, _dp(a), a.size))

    def refresh(self):
        _check(lib().ph_refresh(self._h))

    def get_state(self, gid):
        n1, n2, n3 = self.n
        out = np.zeros((5, n3, n2, n1))
        _check(lib().ph_get_state(self._h, gid, _dp(out), out.size))
        return out

    def get_state_full(self, gid):
        n1, n2, n3 = self.n
        g = self.g
        out = np.zeros((5, n3 + 2 * g, n2 + 2 * g, n1 + 2 * g))
        _check(lib().ph_get_state_full(self._h, gid, _dp(out), out.size))
        return out

    def set_state_full(self, gid, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        _check(lib().ph_set_state_full(self._h, gid, _dp(a), a.size))

    def exchange(self):
        _check(lib().ph_exchange(self._h))

    def step(self, ncycles, tlim=0.0, info=False):
        if info:
            si = PhStepInfo()
            _check(lib().ph_step(self._h, ncycles, tlim, C.byref(si)))
            return dict(cycle=si.cycle, t=si.t, dt=si.dt, zone_cycles=si.zone_cycles)
        _check(lib().ph_step(self._h, ncycles, tlim, None))
        return None

    @staticmethod
    def _host_pair(host_in, host_out, pinned):
        """Both buffers: contiguous float64 of the same size (torch CPU tensors or numpy arrays);
        pinned=True (the async form) also requires page-locked torch tensors."""
        def info(x):
            if hasattr(x, "data_ptr"):
                import torch
                if x.device.type != "cpu" or x.dtype != torch.float64 or not x.is_contiguous():
                    raise ValueError("host buffers must be contiguous float64 CPU tensors")
                if pinned and not x.is_pinned():
                    raise ValueError("step_host_async needs pinned host buffers (tensor.pin_memory())")
                return x.data_ptr(), x.numel()
            a = np.asarray(x)
            if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
                raise ValueError("host buffers must be C-contiguous float64 arrays")
            if pinned:
                raise ValueError("step_host_async needs pinned torch tensors, not numpy arrays")
            return a.ctypes.data, a.size
        pi, ni = info(host_in)
        po, no = info(host_out)
        if ni != no:
            raise ValueError(f"host_in has {ni} elements, host_out {no}")
        return pi, po, ni

    def step_host(self, host_in, host_out, ncycles, tlim=0.0):
        """End-to-end call with host buffers ([nlocal][5][n3][n2][n1]); pinned torch tensors or numpy."""
        pi, po, n = self._host_pair(host_in, host_out, pinned=False)
        _check(lib().ph_step_host(self._h, C.c_void_p(pi), C.c_void_p(po), n, ncycles, tlim))

    def step_host_async(self, host_in, host_out, ncycles, tlim=0.0):
        """Enqueue step_host on the mesh's stream and return (pinned buffers; call sync())."""
        pi, po, n = self._host_pair(host_in, host_out, pinned=True)
        _check(lib().ph_step_host_async(self._h, C.c_void_p(pi), C.c_void_p(po), n, ncycles, tlim))

    def sync(self):
        _check(lib().ph_sync(self._h))

    def time(self):
        t, dt, cyc = C.c_double(), C.c_double(), C.c_int64()
        _check(lib().ph_get_time(self._h, C.byref(t), C.byref(dt), C.byref(cyc)))
        return t.value, dt.value, cyc.value

    def totals(self):
        out = np.zeros(5)
        _check(lib().ph_totals(self._h, _dp(out)))
        return out

    def history(self):
        cap = 1 << 16
        out = np.zeros((cap, 7))
        n = C.c_int64()
        _check(lib().ph_get_history(self._h, _dp(out), cap, C.byref(n)))
        return out[:n.value].copy()

    # ------------------------------------------------------------------ mesh queries
    def blocks(self):
        n = self.num_blocks()
        arr = (PhBlock * max(n, 1))()
        cnt = C.c_int64()
        _check(lib().ph_get_blocks(self._h, arr, n, C.byref(cnt)))
        return [dict(gid=b.gid, level=b.level, rank=b.rank, lx=tuple(b.lx),
                     xmin=tuple(b.xmin), xmax=tuple(b.xmax)) for b in arr[:n]]

    def neighbors(self, gid):
        arr = (PhNeighbor * 64)()
        cnt = C.c_int32()
        _check(lib().ph_get_neighbors(self._h, gid, arr, 64, C.byref(cnt)))
        return [dict(gid=e.gid, rank=e.rank, off=tuple(e.off), dlevel=e.dlevel, fine=tuple(e.fine))
                for e in arr[:cnt.value]]

    def refine_flags(self):
        n = self.num_blocks() * 8 + 8
        arr = (C.c_int8 * n)()
        cnt = C.c_int64()
        _check(lib().ph_get_refine_flags(self._h, arr, n, C.byref(cnt)))
        return np.array(arr[:cnt.value], dtype=np.int8)

    def plan_info(self):
        p = PhPlanInfo()
        _check(lib().ph_get_plan_info(self._h, C.byref(p)))
        R = self.nranks
        return dict(n_local_tasks=p.n_local_tasks, n_send_tasks=p.n_send_tasks, n_recv_tasks=p.n_recv_tasks,
                    send_doubles_to=list(p.send_doubles_to[:R]), recv_doubles_from=list(p.recv_doubles_from[:R]),
                    send_hash_to=list(p.send_hash_to[:R]), recv_hash_from=list(p.recv_hash_from[:R]),
                    cyc_send_doubles_to=list(p.cyc_send_doubles_to[:R]),
                    cyc_recv_doubles_from=list(p.cyc_recv_doubles_from[:R]),
                    cyc_send_hash_to=list(p.cyc_send_hash_to[:R]), cyc_recv_hash_from=list(p.cyc_recv_hash_from[:R]),
                    direct_halo=bool(p.direct_halo), n_cyc_local_tasks=p.n_cyc_local_tasks,
                    peer_halo=bool(p.peer_halo))

    def launch_count(self):
        n = C.c_int64()
        _check(lib().ph_launch_count(self._h, C.byref(n)))
        return n.value

    def kernel_timing(self, enable=True):
        """Return (stage_ms, stage_launches, exch_ms, exch_launches) since the last call; (re)arm."""
        s, x = C.c_double(), C.c_double()
        ns, nx = C.c_int64(), C.c_int64()
        _check(lib().ph_kernel_timing(self._h, 1 if enable else 0, C.byref(s), C.byref(ns), C.byref(x), C.byref(nx)))
        return s.value, ns.value, x.value, nx.value
