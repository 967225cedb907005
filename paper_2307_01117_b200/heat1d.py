"""Thin ctypes binding of libheat1d (include/heat1d.h): argument marshalling only.

Every step of the path runs in the library's CUDA kernels; nothing here
computes the stencil.  If libheat1d.so is missing this module raises -- there
is no CPU fallback.

    h = Heat1D(nx, np, nt, k, dt, dx, T=0, mode="matched")
    h.set_initial(u0)          # numpy array / torch tensor (host or cuda), COPIED
    h.run()                    # nt steps (or h.run(n))
    u = h.get()                # numpy array of this rank's slab

Names follow the paper (§2): nx cells per partition, np partitions,
nt steps, diffusivity k (alpha), time step dt, grid spacing dx (h).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEAT1D_LIB") or os.path.join(_HERE, "libheat1d.so")  # override: A/B builds (tools/)

OK, EINVAL, EUNSTABLE, ESTATE, ENOMEM, ECUDA, ENCCL, EUNSUPPORTED = range(8)
MODES = {"matched": 0, "fast": 1}
DENOMINATORS = {"dx2": 0, "paper_2dx": 1}
KERNELS = {"auto": 0, "naive": 1}


class Heat1DError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("heat1d status %d: %s" % (status, msg))
        self.status = status


class Opts(ctypes.Structure):
    _fields_ = [
        ("size", ctypes.c_uint32),
        ("device", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("T", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("denominator", ctypes.c_int32),
        ("allow_unstable", ctypes.c_int32),
        ("virtual_slabs", ctypes.c_int32),
        ("kernel", ctypes.c_int32),
        ("blocking", ctypes.c_int32),
        ("use_graphs", ctypes.c_int32),
        ("resident", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("comm_stream", ctypes.c_void_p),
        ("transport", ctypes.c_int32),
        ("dev_buf", ctypes.c_void_p),
        ("window_cells", ctypes.c_int64),
    ]


class Info(ctypes.Structure):
    _fields_ = [
        ("size", ctypes.c_uint32),
        ("T", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("denominator", ctypes.c_int32),
        ("kernel", ctypes.c_int32),
        ("dp_ops", ctypes.c_int32),
        ("nslabs", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("r", ctypes.c_double),
        ("N", ctypes.c_int64),
        ("first", ctypes.c_int64),
        ("count", ctypes.c_int64),
        ("steps_done", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("pad", ctypes.c_int64),
        ("tile_cells", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("pass_kind", ctypes.c_int32),
        ("pass_V", ctypes.c_int32),
        ("pass_NW", ctypes.c_int32),
        ("pass_S", ctypes.c_int32),
        ("resident", ctypes.c_int32),
        ("resident_warps", ctypes.c_int32),
        ("stream_windows", ctypes.c_int64),
        ("transport", ctypes.c_int32),
        ("resident_V", ctypes.c_int32),
        ("pass_feed", ctypes.c_int32),
        ("reserved1", ctypes.c_int32),
    ]


class TraceEvent(ctypes.Structure):
    _fields_ = [("stream", ctypes.c_int32), ("kind", ctypes.c_int32), ("t0_ms", ctypes.c_double),
                ("t1_ms", ctypes.c_double)]


TRACE_KINDS = {1: "K1", 2: "K2", 3: "halo", 6: "K6"}


class ExchangePlan(ctypes.Structure):
    _fields_ = [
        ("left", ctypes.c_int32),
        ("right", ctypes.c_int32),
        ("send_right_off", ctypes.c_int64),
        ("send_left_off", ctypes.c_int64),
        ("recv_left_off", ctypes.c_int64),
        ("recv_right_off", ctypes.c_int64),
        ("cells", ctypes.c_int64),
    ]


# Every symbol include/heat1d.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "heat1d_opts_default", "heat1d_version", "heat1d_strerror", "heat1d_partition",
    "heat1d_plan_exchange", "heat1d_buffer_len", "heat1d_get_unique_id", "heat1d_create",
    "heat1d_local_range", "heat1d_set_initial", "heat1d_init_uniform", "heat1d_run",
    "heat1d_get", "heat1d_steps_done", "heat1d_info", "heat1d_set_profiling",
    "heat1d_profile", "heat1d_stream", "heat1d_destroy", "heat1d_last_error", "heat1d_solve_host",
    "heat1d_solve_host_halo", "heat1d_trace",
)

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libheat1d.so (torch is imported first so that its libnccl.so.2 is the one in the process)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError("libheat1d.so not built: run `python -m paper_2307_01117_b200._build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    try:
        import torch  # noqa: F401  (load order: one libnccl.so.2, torch's)
    except Exception:
        pass
    lib = ctypes.CDLL(path)
    i64, i32, dp, vp = ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
    H = ctypes.c_void_p
    sig = {
        "heat1d_opts_default": (None, [ctypes.POINTER(Opts)]),
        "heat1d_version": (ctypes.c_int, []),
        "heat1d_strerror": (ctypes.c_char_p, [ctypes.c_int]),
        "heat1d_partition": (ctypes.c_int, [i64, i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "heat1d_plan_exchange": (ctypes.c_int, [i64, i64, i32, i32, i32, ctypes.POINTER(ExchangePlan)]),
        "heat1d_buffer_len": (i64, [i64, i64, ctypes.POINTER(Opts)]),
        "heat1d_get_unique_id": (ctypes.c_int, [vp]),
        "heat1d_create": (ctypes.c_int, [ctypes.POINTER(H), i64, i64, i64, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.POINTER(Opts)]),
        "heat1d_local_range": (ctypes.c_int, [H, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "heat1d_set_initial": (ctypes.c_int, [H, vp, i64]),
        "heat1d_init_uniform": (ctypes.c_int, [H, ctypes.c_uint64, ctypes.c_double, ctypes.c_double]),
        "heat1d_run": (ctypes.c_int, [H, i64]),
        "heat1d_get": (ctypes.c_int, [H, vp, i64]),
        "heat1d_solve_host": (ctypes.c_int, [H, vp, i64, i64, vp]),
        "heat1d_solve_host_halo": (ctypes.c_int, [H, vp, vp, vp, i64, i64, vp]),
        "heat1d_steps_done": (i64, [H]),
        "heat1d_info": (ctypes.c_int, [H, ctypes.POINTER(Info)]),
        "heat1d_set_profiling": (ctypes.c_int, [H, ctypes.c_int]),
        "heat1d_profile": (ctypes.c_int, [H, ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double)]),
        "heat1d_stream": (vp, [H]),
        "heat1d_trace": (ctypes.c_int, [H, ctypes.POINTER(TraceEvent), i64, ctypes.POINTER(i64)]),
        "heat1d_destroy": (ctypes.c_int, [H]),
        "heat1d_last_error": (ctypes.c_char_p, [H]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    del dp
    _lib = lib
    return lib


def _check(st: int, h=None):
    if st != OK:
        lib = load()
        msg = lib.heat1d_last_error(h).decode() or lib.heat1d_strerror(st).decode()
        raise Heat1DError(st, msg)


def strerror(st: int) -> str:
    return load().heat1d_strerror(st).decode()


def default_opts() -> Opts:
    o = Opts()
    load().heat1d_opts_default(ctypes.byref(o))
    return o


def partition(nx: int, np_: int, nranks: int, rank: int):
    """(first, count) of `rank`'s slab; pure host logic (no GPU needed)."""
    f, c = ctypes.c_int64(), ctypes.c_int64()
    _check(load().heat1d_partition(nx, np_, nranks, rank, ctypes.byref(f), ctypes.byref(c)))
    return f.value, c.value


def plan_exchange(nx: int, np_: int, nranks: int, rank: int, T: int) -> ExchangePlan:
    """The four halo messages of `rank` for depth T, in issue order (pure host logic)."""
    p = ExchangePlan()
    _check(load().heat1d_plan_exchange(nx, np_, nranks, rank, T, ctypes.byref(p)))
    return p


def buffer_len(nx: int, np_: int, opts: Optional[Opts] = None) -> int:
    return load().heat1d_buffer_len(nx, np_, ctypes.byref(opts) if opts is not None else None)


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().heat1d_get_unique_id(buf))
    return buf.raw


def _data_ptr(a, out: bool = False):
    """(pointer, count, keepalive) for a numpy array or torch tensor of float64.  Inputs may
    be converted (a contiguous float64 copy); an output (`out`) must already be one, since
    the library writes through the pointer."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64 or not a.is_contiguous():
                raise TypeError("tensor must be contiguous float64")
            return a.data_ptr(), a.numel(), a
    except ImportError:
        pass
    if out:
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.flags.writeable):
            raise TypeError("out must be a writeable C-contiguous float64 array or tensor")
        return a.ctypes.data, a.size, a
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return arr.ctypes.data, arr.size, arr


class Heat1D:
    """One rank's handle on the periodic ring N = nx*np (§2)."""

    def __init__(self, nx: int, np_: int, nt: int, k: float, dt: float, dx: float, *, T: int = 0,
                 mode: str = "matched", denominator: str = "dx2", allow_unstable: bool = False,
                 rank: int = 0, nranks: int = 1, nccl_id: Optional[bytes] = None, virtual_slabs: int = 1,
                 kernel: str = "auto", device: int = -1, stream=None, comm_stream=None,
                 blocking: bool = True, use_graphs: bool = True, resident: Optional[bool] = None,
                 transport: str = "p2p", dev_buf=None, window_cells: int = 0):
        self._lib = load()
        o = default_opts()
        o.device = device
        o.rank, o.nranks = rank, nranks
        self._id = None
        if nccl_id is not None:
            self._id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = ctypes.cast(self._id, ctypes.c_void_p)
        o.T = T
        o.mode = MODES[mode]
        o.denominator = DENOMINATORS[denominator]
        o.allow_unstable = 1 if allow_unstable else 0
        o.virtual_slabs = virtual_slabs
        o.kernel = KERNELS[kernel]
        o.blocking = 1 if blocking else 0
        o.use_graphs = 1 if use_graphs else 0
        o.resident = -1 if resident is None else (1 if resident else 0)
        o.stream = _stream_ptr(stream)
        o.comm_stream = _stream_ptr(comm_stream)
        o.transport = {"nccl": 0, "p2p": 1}[transport]
        o.window_cells = window_cells
        self._dev_buf = dev_buf  # caller-owned state memory (torch tensor): kept alive with the handle
        if dev_buf is not None:
            import torch
            if not (isinstance(dev_buf, torch.Tensor) and dev_buf.is_cuda):
                raise TypeError("dev_buf must be a CUDA tensor (device memory the handle computes in)")
            ptr, n, _ = _data_ptr(dev_buf, out=True)
            need = buffer_len(nx, np_, o)
            if n < need:
                raise ValueError("dev_buf holds %d doubles, the handle needs %d (buffer_len)" % (n, need))
            o.dev_buf = ptr
        h = ctypes.c_void_p()
        st = self._lib.heat1d_create(ctypes.byref(h), nx, np_, nt, float(k), float(dt), float(dx), ctypes.byref(o))
        _check(st, None)
        self._h = h
        self.nx, self.np, self.nt = nx, np_, nt
        self.N = nx * np_

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            self._lib.heat1d_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- queries
    @property
    def local_range(self):
        f, c = ctypes.c_int64(), ctypes.c_int64()
        _check(self._lib.heat1d_local_range(self._h, ctypes.byref(f), ctypes.byref(c)), self._h)
        return f.value, c.value

    @property
    def count(self) -> int:
        return self.local_range[1]

    @property
    def steps_done(self) -> int:
        return self._lib.heat1d_steps_done(self._h)

    def info(self) -> dict:
        i = Info()
        i.size = ctypes.sizeof(Info)
        _check(self._lib.heat1d_info(self._h, ctypes.byref(i)), self._h)
        return {name: getattr(i, name) for name, _ in Info._fields_ if name != "size"}

    @property
    def stream_ptr(self) -> int:
        return self._lib.heat1d_stream(self._h) or 0

    # -- state
    def set_initial(self, u0):
        ptr, n, keep = _data_ptr(u0)
        _check(self._lib.heat1d_set_initial(self._h, ctypes.c_void_p(ptr), n), self._h)
        del keep

    def init_uniform(self, seed: int, lo: float = 0.0, hi: float = 1.0):
        _check(self._lib.heat1d_init_uniform(self._h, seed & 0xFFFFFFFFFFFFFFFF, float(lo), float(hi)), self._h)

    def run(self, nt: Optional[int] = None):
        _check(self._lib.heat1d_run(self._h, -1 if nt is None else int(nt)), self._h)

    def get(self, out=None):
        if out is None:
            out = np.empty(self.count, dtype=np.float64)
        ptr, n, keep = _data_ptr(out, out=True)
        _check(self._lib.heat1d_get(self._h, ctypes.c_void_p(ptr), n), self._h)
        return out

    def solve_host(self, u0, nt: Optional[int] = None, out=None):
        """set_initial(u0) + run(nt) + get(out) for HOST arrays with the transfers
        overlapped by light-cone windows (heat1d_solve_host); pinned tensors overlap best."""
        if out is None:
            out = np.empty(self.count, dtype=np.float64)
        pi, n, keep_in = _data_ptr(u0)
        po, m, keep_out = _data_ptr(out, out=True)
        if n != self.count or m != self.count:
            raise ValueError("u0 and out must hold the local slab (%d cells)" % self.count)
        _check(self._lib.heat1d_solve_host(self._h, ctypes.c_void_p(pi), n, -1 if nt is None else nt,
                                           ctypes.c_void_p(po)), self._h)
        return out

    def solve_host_halo(self, u0, left, right, nt: Optional[int] = None, out=None):
        """Streamed solve of this slab given the nt cells before (`left`) and after (`right`)
        it (heat1d_solve_host_halo): no communication needed."""
        if out is None:
            out = np.empty(self.count, dtype=np.float64)
        pi, n, k1 = _data_ptr(u0)
        pl, nl, k2 = _data_ptr(left)
        pr, nr, k3 = _data_ptr(right)
        po, m, k4 = _data_ptr(out, out=True)
        steps = -1 if nt is None else nt
        if n != self.count or m != self.count or (nt is not None and (nl < nt or nr < nt)):
            raise ValueError("u0/out must hold the slab and left/right at least nt cells")
        _check(self._lib.heat1d_solve_host_halo(self._h, ctypes.c_void_p(pi), ctypes.c_void_p(pl),
                                                ctypes.c_void_p(pr), n, steps, ctypes.c_void_p(po)), self._h)
        return out

    # -- profiling of the pass kernel (CUDA events on the compute stream)
    def set_profiling(self, on: bool):
        _check(self._lib.heat1d_set_profiling(self._h, 1 if on else 0), self._h)

    def profile(self):
        n, ms = ctypes.c_int64(), ctypes.c_double()
        _check(self._lib.heat1d_profile(self._h, ctypes.byref(n), ctypes.byref(ms)), self._h)
        return n.value, ms.value

    def trace(self):
        """[(stream, kind, t0_ms, t1_ms), ...] of the profiling session (heat1d_trace)."""
        n = ctypes.c_int64()
        _check(self._lib.heat1d_trace(self._h, None, 0, ctypes.byref(n)), self._h)
        buf = (TraceEvent * max(1, n.value))()
        _check(self._lib.heat1d_trace(self._h, buf, n.value, ctypes.byref(n)), self._h)
        return [(e.stream, TRACE_KINDS.get(e.kind, str(e.kind)), e.t0_ms, e.t1_ms) for e in buf[:n.value]]


def _stream_ptr(s) -> Optional[int]:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return int(s.cuda_stream)  # torch.cuda.Stream
