"""Python binding of libcpsel.so — exact k-th order statistics by Kelley's cutting-plane method
(Beliakov, arXiv:1104.2732) on B200.

Argument marshalling only: every step of the path (init reduction, cutting-plane passes,
compaction, radix select, LMS residuals, NCCL exchange) runs inside libcpsel.so (C ABI in
include/cpsel.h).  PyTorch supplies device memory, the current CUDA stream and process groups.
There is no CPU fallback: if the shared library is missing or CUDA is unavailable the calls
raise.  Names follow the C ABI: select_kth, median, lms_objective, eval, ...
"""
from __future__ import annotations

import ctypes as C
import os
import threading

__all__ = [
    "select_kth", "median", "select_kth_host", "lms_objective", "lms_residuals", "select_kth_batched",
    "eval", "init_stats", "small_select", "get_trace", "set_config", "get_config", "nccl_unique_id",
    "comm_init", "select_kth_sharded", "drive_host", "library_path", "load", "CpselError",
    "LoopbackGroup", "comm_init_loopback", "knn_regress", "knn_classify",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libcpsel.so")

F32, F64 = 0, 1
OK, EINVAL, ERANK, ENONFINITE, ECUDA, ENCCL, ENOMEM, EINTERNAL = range(8)
EXIT_REASONS = ["init_min", "init_max", "hit", "pred", "succ", "compact_select", "direct_select"]


class CpselError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"cpsel status {status}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("z_cap", C.c_uint64), ("direct_threshold", C.c_uint64), ("select_cap", C.c_uint64),
                ("max_iters", C.c_uint32),
                ("force_cp", C.c_int32), ("record_trace", C.c_int32), ("record_timing", C.c_int32),
                ("init_cut", C.c_int32), ("objective", C.c_int32),
                ("pass_cuts", C.c_int32), ("lms_fused", C.c_int32), ("device_loop", C.c_int32),
                ("driver", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("passes", C.c_uint32), ("cp_iters", C.c_uint32), ("fallback_steps", C.c_uint32),
                ("exit_reason", C.c_uint32), ("z_count", C.c_uint64), ("bytes_moved", C.c_uint64),
                ("ms_total", C.c_double), ("launches", C.c_uint32), ("reserved", C.c_uint32),
                ("kernel_ms_init", C.c_double), ("kernel_ms_passes", C.c_double), ("kernel_ms_select", C.c_double),
                ("init_written", C.c_uint64), ("kernel_ms_sample", C.c_double)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["exit"] = EXIT_REASONS[self.exit_reason] if self.exit_reason < len(EXIT_REASONS) else "?"
        return d


class PassStats(C.Structure):
    _fields_ = [("c_lt", C.c_uint64), ("c_eq", C.c_uint64), ("c_lo", C.c_uint64), ("c_hi", C.c_uint64),
                ("L_lo", C.c_double), ("L_hi", C.c_double), ("P", C.c_double), ("N", C.c_double),
                ("pred", C.c_double), ("succ", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class InitStats(C.Structure):
    _fields_ = [("vmin", C.c_double), ("vmax", C.c_double), ("cnt_min", C.c_uint64), ("cnt_max", C.c_uint64),
                ("nonfinite", C.c_uint64), ("x0", C.c_double), ("S", C.c_double), ("has_cut", C.c_uint64),
                ("t_lo", C.c_double), ("t_hi", C.c_double), ("c_le_lo", C.c_uint64), ("c_lt_hi", C.c_uint64),
                ("t_est", C.c_double), ("reserved_cut", C.c_uint64), ("N_lo", C.c_double), ("P_hi", C.c_double),
                ("I_in", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class TraceRow(C.Structure):
    _fields_ = [("t", C.c_double), ("F", C.c_double), ("c_lt", C.c_uint64), ("c_eq", C.c_uint64),
                ("interior", C.c_uint64), ("scanned", C.c_uint64), ("written", C.c_uint64), ("kind", C.c_uint32),
                ("compacted", C.c_uint32),
                ("kernel_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_INIT_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(InitStats))
_PASS_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_int, C.POINTER(PassStats))
_SEL_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_uint64, C.POINTER(C.c_double))
_ADOPT_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int)


class CutStats(C.Structure):
    _fields_ = [("t_a", C.c_double), ("t_b", C.c_double), ("t_est", C.c_double), ("le_a", C.c_uint64),
                ("inner", C.c_uint64)]


_CUT_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.POINTER(CutStats))


class HostBackend(C.Structure):
    _fields_ = [("user", C.c_void_p), ("init", _INIT_CB), ("pass_", _PASS_CB), ("adopt", _ADOPT_CB),
                ("select", _SEL_CB), ("cut", _CUT_CB)]


# every symbol the header declares (tests check the library exports exactly these)
SYMBOLS = [
    "cpsel_create", "cpsel_destroy", "cpsel_last_error", "cpsel_status_string", "cpsel_config_default",
    "cpsel_set_config", "cpsel_get_config", "cpsel_set_stream", "cpsel_select_kth", "cpsel_median",
    "cpsel_select_kth_host", "cpsel_lms_objective", "cpsel_lms_residuals", "cpsel_select_kth_batched",
    "cpsel_eval", "cpsel_init", "cpsel_small_select", "cpsel_get_trace", "cpsel_init_timings", "cpsel_nccl_unique_id",
    "cpsel_comm_init", "cpsel_select_kth_sharded", "cpsel_drive_host", "cpsel_pooled_cuts",
    "cpsel_lts_objective", "cpsel_loopback_create", "cpsel_loopback_destroy", "cpsel_comm_init_loopback",
    "cpsel_knn_regress", "cpsel_knn_classify",
]

_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return _LIB_PATH


def load():
    """Load libcpsel.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: build it with `python -m paper_1104_2732_b200.build`")
        lib = C.CDLL(_LIB_PATH)
        P, U64, U32, I, D = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double
        sig = {
            "cpsel_create": (I, [I, P, C.POINTER(P)]),
            "cpsel_destroy": (None, [P]),
            "cpsel_last_error": (C.c_char_p, [P]),
            "cpsel_status_string": (C.c_char_p, [I]),
            "cpsel_config_default": (None, [C.POINTER(Config)]),
            "cpsel_set_config": (I, [P, C.POINTER(Config)]),
            "cpsel_get_config": (I, [P, C.POINTER(Config)]),
            "cpsel_set_stream": (I, [P, P]),
            "cpsel_select_kth": (I, [P, P, U64, I, U64, P, C.POINTER(Info)]),
            "cpsel_median": (I, [P, P, U64, I, P, C.POINTER(Info)]),
            "cpsel_select_kth_host": (I, [P, P, U64, I, U64, P, C.POINTER(Info)]),
            "cpsel_lms_objective": (I, [P, P, P, U64, U32, P, U32, P, C.POINTER(Info)]),
            "cpsel_lms_residuals": (I, [P, P, P, U64, U32, P, U32, P]),
            "cpsel_select_kth_batched": (I, [P, P, U64, U32, U64, P, C.POINTER(Info)]),
            "cpsel_eval": (I, [P, P, U64, I, D, D, D, C.POINTER(PassStats)]),
            "cpsel_init": (I, [P, P, U64, I, C.POINTER(InitStats)]),
            "cpsel_small_select": (I, [P, P, U64, I, U64, P]),
            "cpsel_get_trace": (I, [P, C.POINTER(TraceRow), U32, C.POINTER(U32)]),
            "cpsel_init_timings": (I, [P, C.POINTER(D), U32, C.POINTER(U32), C.c_int32]),
            "cpsel_nccl_unique_id": (I, [P]),
            "cpsel_comm_init": (I, [P, P, I, I]),
            "cpsel_select_kth_sharded": (I, [P, P, U64, I, U64, P, C.POINTER(Info)]),
            "cpsel_drive_host": (I, [C.POINTER(HostBackend), U64, I, U64, C.POINTER(Config), C.POINTER(D),
                                     C.POINTER(Info), C.POINTER(TraceRow), U32, C.POINTER(U32)]),
            "cpsel_pooled_cuts": (I, [P, P, U32, U64, I, C.POINTER(D)]),
            "cpsel_lts_objective": (I, [P, P, P, U64, U32, P, U32, U64, P, P, C.POINTER(Info)]),
            "cpsel_loopback_create": (I, [I, C.POINTER(P)]),
            "cpsel_loopback_destroy": (None, [P]),
            "cpsel_comm_init_loopback": (I, [P, P, I]),
            "cpsel_knn_regress": (I, [P, P, P, U64, U32, P, U32, U64, C.c_int32, P, P, C.POINTER(Info)]),
            "cpsel_knn_classify": (I, [P, P, P, U64, U32, P, U32, U64, U32, C.c_int32, P, P, C.POINTER(Info)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


# ------------------------------------------------------------------------------------------ ctx
class _Ctx:
    def __init__(self, device: int):
        lib = load()
        self.device = device
        self.handle = C.c_void_p()
        st = lib.cpsel_create(device, None, C.byref(self.handle))
        if st != OK:
            raise CpselError(st, "cpsel_create failed (see stderr)")
        self._stream = None

    def bind_stream(self, stream_ptr: int):
        # torch's default stream has handle 0 = the legacy default stream, which the C ABI
        # takes as NULL; any other handle is used as given
        if stream_ptr != self._stream:
            _check(self, load().cpsel_set_stream(self.handle, C.c_void_p(stream_ptr)))
            self._stream = stream_ptr

    def __del__(self):
        try:
            if self.handle and _lib is not None:
                _lib.cpsel_destroy(self.handle)
        except Exception:
            pass


# One ctx per (thread, device): a ctx is not thread-safe (include/cpsel.h) and ctypes releases the
# GIL during every call, so threads never share one.  A thread's ctxs are destroyed when it ends.
_tls = threading.local()


def _ctxs() -> dict:
    d = getattr(_tls, "ctxs", None)
    if d is None:
        d = _tls.ctxs = {}
    return d


def _current_stream(dev: int) -> int:
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # the cheap form of current_stream()
    return raw(dev) if raw is not None else torch.cuda.current_stream(dev).cuda_stream


def _ctx_device(dev: int) -> _Ctx:
    d = _ctxs()
    c = d.get(dev)
    if c is None:
        c = d[dev] = _Ctx(dev)
    c.bind_stream(_current_stream(dev))
    return c


def _ctx_for(t) -> _Ctx:
    if not getattr(t, "is_cuda", False):
        raise ValueError("expected a CUDA tensor (no CPU fallback)")
    return _ctx_device(t.get_device())


def _check(ctx: _Ctx, st: int):
    if st == OK:
        return
    msg = load().cpsel_last_error(ctx.handle).decode(errors="replace")
    if st in (EINVAL, ERANK, ENONFINITE):
        raise ValueError(f"cpsel status {st}: {msg}")
    raise CpselError(st, msg)


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float64:
        return F64
    raise ValueError(f"unsupported dtype {t.dtype} (float32 / float64)")


def _flat(t):
    if t.dim() != 1:
        t = t.reshape(-1)
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t


def _out_value(buf, dt: int) -> float:
    return float(C.cast(buf, C.POINTER(C.c_float if dt == F32 else C.c_double))[0])


# ------------------------------------------------------------------------------------------ API
def select_kth(x, k: int, return_info=False):
    """k-th smallest element (1-based) of the CUDA tensor x (float32/float64).  return_info: True
    adds the call's report as a dict, "raw" as the ctypes `Info` struct."""
    x = _flat(x)
    ctx = _ctx_for(x)
    dt = _dtype_code(x)
    lib = _lib or load()
    if dt == F32:
        out = C.c_float()
    else:
        out = C.c_double()
    info = Info() if return_info else None
    _check(ctx, lib.cpsel_select_kth(ctx.handle, x.data_ptr(), x.numel(), dt, k, C.byref(out),
                                     C.byref(info) if info is not None else None))
    v = out.value
    if return_info == "raw":  # the ctypes struct itself (no dict built: for tight timing loops)
        return v, info
    return (v, info.as_dict()) if return_info else v


def median(x, return_info: bool = False):
    """Lower median x_((n+1)//2)."""
    x = _flat(x)
    return select_kth(x, (x.numel() + 1) // 2, return_info)


def select_kth_host(x, k: int, device: int = 0, return_info: bool = False):
    """k-th smallest of a HOST tensor (pinned recommended); the H2D copy is inside the call."""
    import torch
    if x.is_cuda:
        raise ValueError("select_kth_host expects a CPU tensor")
    x = _flat(x)
    ctx = _ctx_device(device)
    dt = _dtype_code(x)
    out = C.create_string_buffer(8)
    info = Info()
    _check(ctx, load().cpsel_select_kth_host(ctx.handle, C.c_void_p(x.data_ptr()), x.numel(), dt, int(k), out,
                                            C.byref(info)))
    v = _out_value(out, dt)
    return (v, info.as_dict()) if return_info else v


def eval(x, t: float, y_lo: float, y_hi: float) -> dict:  # noqa: A001  (C ABI name)
    """One cutting-plane pass at t over bracket (y_lo, y_hi): counts, local sums, P, N, pred, succ."""
    x = _flat(x)
    ctx = _ctx_for(x)
    s = PassStats()
    _check(ctx, load().cpsel_eval(ctx.handle, C.c_void_p(x.data_ptr()), x.numel(), _dtype_code(x), float(t),
                                  float(y_lo), float(y_hi), C.byref(s)))
    return s.as_dict()


def init_stats(x) -> dict:
    x = _flat(x)
    ctx = _ctx_for(x)
    s = InitStats()
    _check(ctx, load().cpsel_init(ctx.handle, C.c_void_p(x.data_ptr()), x.numel(), _dtype_code(x), C.byref(s)))
    return s.as_dict()


def small_select(z, r: int) -> float:
    z = _flat(z)
    ctx = _ctx_for(z)
    dt = _dtype_code(z)
    out = C.create_string_buffer(8)
    _check(ctx, load().cpsel_small_select(ctx.handle, C.c_void_p(z.data_ptr()), z.numel(), dt, int(r), out))
    return _out_value(out, dt)


def init_timings(device: int = 0, reset: bool = True) -> list:
    """record_timing=2: the init-kernel durations (ms, CUDA events) of the selections since the last
    reset, in call order."""
    c = _ctx_device(device)
    n = C.c_uint32()
    _check(c, load().cpsel_init_timings(c.handle, None, 0, C.byref(n), 0))
    buf = (C.c_double * max(n.value, 1))()
    _check(c, load().cpsel_init_timings(c.handle, buf, n.value, C.byref(n), 1 if reset else 0))
    return [buf[i] for i in range(n.value)]


def get_trace(device: int = 0) -> list:
    c = _ctxs().get(device)
    if c is None:
        return []
    n = C.c_uint32()
    load().cpsel_get_trace(c.handle, None, 0, C.byref(n))
    rows = (TraceRow * max(n.value, 1))()
    load().cpsel_get_trace(c.handle, rows, n.value, C.byref(n))
    return [rows[i].as_dict() for i in range(n.value)]


def set_config(device: int = 0, **kw) -> None:
    c = _ctx_device(device)
    cfg = Config()
    _check(c, load().cpsel_get_config(c.handle, C.byref(cfg)))
    for k, v in kw.items():
        if not hasattr(cfg, k):
            raise ValueError(f"unknown config field {k}")
        setattr(cfg, k, int(v))
    _check(c, load().cpsel_set_config(c.handle, C.byref(cfg)))


def get_config(device: int = 0) -> dict:
    c = _ctx_device(device)
    cfg = Config()
    _check(c, load().cpsel_get_config(c.handle, C.byref(cfg)))
    return {f: getattr(cfg, f) for f, _ in cfg._fields_}


def default_config() -> dict:
    cfg = Config()
    load().cpsel_config_default(C.byref(cfg))
    return {f: getattr(cfg, f) for f, _ in cfg._fields_}


# ------------------------------------------------------------------------------------------ LMS
def _check_lms(X, y, thetas):
    import torch
    for t in (X, y, thetas):
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("X, y, thetas must be contiguous float32 CUDA tensors")
    n, p = X.shape
    if y.numel() != n:
        raise ValueError("y must have n elements")
    if thetas.dim() != 2 or thetas.shape[1] != p:
        raise ValueError("thetas must be (C, p): row j is theta_j (= p x C column-major)")
    return n, p, thetas.shape[0]


def lms_objective(X, y, thetas, return_info: bool = False):
    """Med_i (x_i . theta_j - y_i)^2 for every candidate theta_j (rows of thetas)."""
    import torch
    n, p, Cn = _check_lms(X, y, thetas)
    ctx = _ctx_for(X)
    out = torch.empty(Cn, device=X.device, dtype=torch.float32)
    info = Info()
    _check(ctx, load().cpsel_lms_objective(ctx.handle, C.c_void_p(X.data_ptr()), C.c_void_p(y.data_ptr()), n, p,
                                           C.c_void_p(thetas.data_ptr()), Cn, C.c_void_p(out.data_ptr()),
                                           C.byref(info)))
    return (out, info.as_dict()) if return_info else out


def lms_residuals(X, y, thetas, out=None):
    """S[j, i] = (x_i . theta_j - y_i)^2 as a (C, n) tensor (= n x C column-major)."""
    import torch
    n, p, Cn = _check_lms(X, y, thetas)
    ctx = _ctx_for(X)
    if out is None:
        out = torch.empty((Cn, n), device=X.device, dtype=torch.float32)
    _check(ctx, load().cpsel_lms_residuals(ctx.handle, C.c_void_p(X.data_ptr()), C.c_void_p(y.data_ptr()), n, p,
                                           C.c_void_p(thetas.data_ptr()), Cn, C.c_void_p(out.data_ptr())))
    return out


def lts_objective(X, y, thetas, h: int, return_info: bool = False):
    """LTS objective per candidate (NEXT row): the sum of the h smallest squared
    residuals (float64) and the h-th smallest itself (float32), for every row theta_j of thetas."""
    import torch
    n, p, Cn = _check_lms(X, y, thetas)
    ctx = _ctx_for(X)
    out = torch.empty(Cn, device=X.device, dtype=torch.float64)
    m = torch.empty(Cn, device=X.device, dtype=torch.float32)
    info = Info()
    _check(ctx, load().cpsel_lts_objective(ctx.handle, C.c_void_p(X.data_ptr()), C.c_void_p(y.data_ptr()), n, p,
                                           C.c_void_p(thetas.data_ptr()), Cn, int(h), C.c_void_p(out.data_ptr()),
                                           C.c_void_p(m.data_ptr()), C.byref(info)))
    return (out, m, info.as_dict()) if return_info else (out, m)


def select_kth_batched(S, k: int, return_info: bool = False):
    """Row-wise k-th smallest of a (C, n) float32 CUDA tensor (columns of an n x C column-major S)."""
    import torch
    if S.dtype != torch.float32 or not S.is_cuda or not S.is_contiguous() or S.dim() != 2:
        raise ValueError("S must be a contiguous (C, n) float32 CUDA tensor")
    ctx = _ctx_for(S)
    Cn, n = S.shape
    out = torch.empty(Cn, device=S.device, dtype=torch.float32)
    info = Info()
    _check(ctx, load().cpsel_select_kth_batched(ctx.handle, C.c_void_p(S.data_ptr()), n, Cn, int(k),
                                                C.c_void_p(out.data_ptr()), C.byref(info)))
    return (out, info.as_dict()) if return_info else out


# ------------------------------------------------------------------------------------------ kNN
def knn_regress(X, f, Q, k: int, weighting: int = 0, return_dk: bool = False, return_info: bool = False):
    """kNN regression via d_(k): for each query row of Q (nq, p), the rho-weighted mean
    of f over the k nearest rows of X (n, p) — see cpsel_knn_regress.  Returns a float32 (nq,)
    tensor (and d2_(k) per query, and the report, if asked)."""
    import torch
    for t in (X, f, Q):
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("X, f, Q must be contiguous float32 CUDA tensors")
    if X.dim() != 2 or Q.dim() != 2 or Q.shape[1] != X.shape[1] or f.numel() != X.shape[0]:
        raise ValueError("X (n, p), f (n,), Q (nq, p)")
    n, p = X.shape
    nq = Q.shape[0]
    ctx = _ctx_for(X)
    out = torch.empty(nq, device=X.device, dtype=torch.float32)
    dk = torch.empty(nq, device=X.device, dtype=torch.float32)
    info = Info()
    _check(ctx, load().cpsel_knn_regress(ctx.handle, C.c_void_p(X.data_ptr()), C.c_void_p(f.data_ptr()), n, p,
                                         C.c_void_p(Q.data_ptr()), nq, int(k), int(weighting),
                                         C.c_void_p(out.data_ptr()), C.c_void_p(dk.data_ptr()), C.byref(info)))
    res = (out, dk) if return_dk else (out,)
    if return_info:
        res = res + (info.as_dict(),)
    return res if len(res) > 1 else res[0]


def knn_classify(X, labels, Q, k: int, n_classes: int, weighting: int = 0, return_votes: bool = False):
    """kNN classification via d_(k): the rho-weighted majority vote of the k nearest rows of
    X for every query row of Q; labels: int32 (n,) in [0, n_classes).  Returns int32 (nq,) classes
    (and the (nq, n_classes) float64 votes if asked)."""
    import torch
    for t in (X, Q):
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("X, Q must be contiguous float32 CUDA tensors")
    if labels.dtype != torch.int32 or not labels.is_cuda or not labels.is_contiguous():
        raise ValueError("labels must be a contiguous int32 CUDA tensor")
    if X.dim() != 2 or Q.dim() != 2 or Q.shape[1] != X.shape[1] or labels.numel() != X.shape[0]:
        raise ValueError("X (n, p), labels (n,), Q (nq, p)")
    n, p = X.shape
    nq = Q.shape[0]
    ctx = _ctx_for(X)
    out = torch.empty(nq, device=X.device, dtype=torch.int32)
    votes = torch.empty((nq, n_classes), device=X.device, dtype=torch.float64) if return_votes else None
    info = Info()
    _check(ctx, load().cpsel_knn_classify(ctx.handle, C.c_void_p(X.data_ptr()), C.c_void_p(labels.data_ptr()), n, p,
                                          C.c_void_p(Q.data_ptr()), nq, int(k), int(n_classes), int(weighting),
                                          C.c_void_p(out.data_ptr()),
                                          C.c_void_p(votes.data_ptr()) if votes is not None else None,
                                          C.byref(info)))
    return (out, votes) if return_votes else out


# ------------------------------------------------------------------------------------------ multi-GPU
def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = load().cpsel_nccl_unique_id(buf)
    if st != OK:
        raise CpselError(st, "ncclGetUniqueId failed / NCCL not loadable")
    return buf.raw


def comm_init(uid: bytes, rank: int, world: int, device: int) -> None:
    c = _ctx_device(device)
    buf = C.create_string_buffer(uid, 128)
    _check(c, load().cpsel_comm_init(c.handle, buf, int(rank), int(world)))


class LoopbackGroup:
    """`world` virtual ranks on one device inside this process: each rank is a thread
    that calls comm_init_loopback(group, rank, device) and then select_kth_sharded on its shard —
    the real sharded driver, its all-gathers as device-to-device copies."""

    def __init__(self, world: int):
        self.world = int(world)
        self.handle = C.c_void_p()
        st = load().cpsel_loopback_create(self.world, C.byref(self.handle))
        if st != OK:
            raise CpselError(st, "cpsel_loopback_create failed")

    def __del__(self):
        try:
            if self.handle and _lib is not None:
                _lib.cpsel_loopback_destroy(self.handle)
        except Exception:
            pass


def comm_init_loopback(group: LoopbackGroup, rank: int, device: int = 0) -> None:
    """Attach the calling thread's ctx on `device` to the loopback group as `rank`."""
    c = _ctx_device(device)
    _check(c, load().cpsel_comm_init_loopback(c.handle, group.handle, int(rank)))


def select_kth_sharded(shard, k: int, return_info: bool = False):
    """Collective: k-th smallest of the concatenation (rank order) of every rank's shard."""
    shard = _flat(shard)
    ctx = _ctx_for(shard)
    dt = _dtype_code(shard)
    out = C.create_string_buffer(8)
    info = Info()
    ptr = C.c_void_p(shard.data_ptr()) if shard.numel() else C.c_void_p(0)
    _check(ctx, load().cpsel_select_kth_sharded(ctx.handle, ptr, shard.numel(), dt, int(k), out, C.byref(info)))
    v = _out_value(out, dt)
    return (v, info.as_dict()) if return_info else v


def pooled_cuts(keys, m, r: int, dtype: str):
    """R28 host step: cuts (t_a, t_b, estimate) common to all ranks from their pooled sample keys
    (keys: G x 1024 uint64 order-preserving keys, each block sorted with min(m[g],1024) valid first)."""
    import numpy as np
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    mm = np.ascontiguousarray(m, dtype=np.uint64)
    out = (C.c_double * 3)()
    st = load().cpsel_pooled_cuts(k.ctypes.data_as(C.c_void_p), mm.ctypes.data_as(C.c_void_p), int(mm.size), int(r),
                                   F32 if dtype == "f32" else F64, out)
    if st != OK:
        raise CpselError(st, load().cpsel_status_string(st).decode())
    return out[0], out[1], out[2]


# ------------------------------------------------------------------------------------------ host driver
def drive_host(n: int, k: int, dtype: str, init_fn, pass_fn, adopt_fn, select_fn, config: dict | None = None,
               cut_fn=None):
    """Run libcpsel's cutting-plane driver with Python callbacks for the data steps
    (init_fn() -> dict of InitStats fields; pass_fn(t, y_lo, y_hi, compact) -> dict of PassStats
    fields over the current array; adopt_fn(side); select_fn(side, r) -> float; optional
    cut_fn(r) -> dict of CutStats fields, the R26 cut pass).  No GPU
    involved: used to test the host logic."""
    lib = load()
    errors = []

    def _init(_u, out):
        try:
            d = init_fn()
            for f, _ in InitStats._fields_:
                setattr(out.contents, f, d.get(f, 0))
            return 0
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            return 1

    def _pass(_u, t, lo, hi, compact, out):
        try:
            d = pass_fn(t, lo, hi, bool(compact))
            for f, _ in PassStats._fields_:
                setattr(out.contents, f, d.get(f, 0))
            return 0
        except Exception as e:  # pragma: no cover
            errors.append(e)
            return 1

    def _sel(_u, side, r, out):
        try:
            out[0] = float(select_fn(side, r))
            return 0
        except Exception as e:  # pragma: no cover
            errors.append(e)
            return 1

    def _adopt(_u, side):
        try:
            adopt_fn(side)
            return 0
        except Exception as e:  # pragma: no cover
            errors.append(e)
            return 1

    def _cut(_u, r, out):
        try:
            d = cut_fn(r)
            for f, _ in CutStats._fields_:
                setattr(out.contents, f, d[f])
            return 0
        except Exception as e:  # pragma: no cover
            errors.append(e)
            return 1

    cbs = (_INIT_CB(_init), _PASS_CB(_pass), _ADOPT_CB(_adopt), _SEL_CB(_sel),
           _CUT_CB(_cut) if cut_fn is not None else C.cast(None, _CUT_CB))
    be = HostBackend(None, *cbs)
    cfg = Config()
    lib.cpsel_config_default(C.byref(cfg))
    for key, v in (config or {}).items():
        setattr(cfg, key, int(v))
    val = C.c_double()
    info = Info()
    rows = (TraceRow * 512)()
    nrows = C.c_uint32()
    st = lib.cpsel_drive_host(C.byref(be), int(n), F32 if dtype == "f32" else F64, int(k), C.byref(cfg),
                              C.byref(val), C.byref(info), rows, 512, C.byref(nrows))
    if errors:
        raise errors[0]
    if st != OK:
        raise CpselError(st, lib.cpsel_status_string(st).decode())
    return val.value, info.as_dict(), [rows[i].as_dict() for i in range(min(nrows.value, 512))]
