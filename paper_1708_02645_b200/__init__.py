"""paper_1708_02645_b200 -- B200-native hot path of arXiv 1708.02645.

Thin Python binding over the C ABI in include/qmcj2.h (libqmcj2.so, built
in-tree by _build.py).  This module only marshals arguments: every step of the
hot path runs in the CUDA kernels of csrc/.  PyTorch provides device memory and
streams.  There is no CPU fallback: importing this package without the built
library raises, and every call goes to the GPU library.

Public API (names follow include/qmcj2.h):
    eval(R, k, r_trial, fn, n_total, n_up, ...)   -> out [W][P][5] fp64 (and row, ratio)
    eval_j1(ions, species_start, r_trial, fn1)    -> NEXT-1: J1 over the AB row
    accept(R, state, k, r_new, acc, out_new, fn, ...) -> NEXT-2: accept-side update of R and the 5N J2 state
    metropolis(ratio, u)                          -> NEXT-2: accept flags (u < rho^2)
    SpoTable, spo_eval(tab, pos, ...)             -> NEXT-4: Bspline-v/vgh + determinant ratio
    eval_host(R, k, r_trial, fn, ...)             -> host-buffer end-to-end path
    ratio(out, V_cur=None)                        -> [W][P][2] (dJ2, exp(dJ2))
    functor_eval_vgl(fn, channel, r)              -> [n][3] (U, U', U'')
    min_image_disp(L, a, b)                       -> [n][4] (|d|, dx, dy, dz)
    check_inputs(...), padded_size(n, block), gen_positions(...)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _build

__all__ = ["QJ2Error", "Functor", "J1Functor", "Workspace", "eval", "eval_j1", "accept", "metropolis",
           "metropolis_accept", "sweep", "state_init", "SpoTable",
           "spo_eval", "gen_spo_table", "eval_host", "ratio", "functor_eval_vgl",
           "min_image_disp", "check_inputs", "padded_size", "gen_positions", "lib_path",
           "workspace_size", "host_workspace_size", "version", "device_check"]

QJ2_FP32, QJ2_FP64 = 0, 1
QJ2_MAX_M = 64
QJ2_MAX_P = 64
QJ2_MAX_SPECIES = 4


class QJ2Error(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status


class _Functor(ctypes.Structure):
    _fields_ = [("L", ctypes.c_double * 3),
                ("r_cut", ctypes.c_double),
                ("m", ctypes.c_int32),
                ("reserved", ctypes.c_int32),
                ("coef", (ctypes.c_double * (QJ2_MAX_M + 3)) * 2)]


class _SpoTable(ctypes.Structure):
    _fields_ = [("L", ctypes.c_double * 3),
                ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("n_orb", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("coef", ctypes.c_void_p)]


class _SweepJ1(ctypes.Structure):
    _fields_ = [("fn", ctypes.c_void_p), ("species_start", ctypes.POINTER(ctypes.c_int64)),
                ("ions", ctypes.c_void_p), ("Np_ion", ctypes.c_int64), ("state", ctypes.c_void_p)]


class _J1Functor(ctypes.Structure):
    _fields_ = [("L", ctypes.c_double * 3),
                ("n_species", ctypes.c_int32),
                ("reserved", ctypes.c_int32),
                ("r_cut", ctypes.c_double * QJ2_MAX_SPECIES),
                ("m", ctypes.c_int32 * QJ2_MAX_SPECIES),
                ("coef", (ctypes.c_double * (QJ2_MAX_M + 3)) * QJ2_MAX_SPECIES)]


def lib_path() -> str:
    return os.environ.get("QJ2_LIB") or _build.LIB


def _load():
    path = lib_path()   # QJ2_LIB: load another build of the library (A/B measurements)
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    i64, i32, vp, dp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)
    F = ctypes.POINTER(_Functor)
    sz = ctypes.c_size_t
    sigs = {
        "qj2_version": (i32, []),
        "qj2_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "qj2_last_error": (ctypes.c_char_p, []),
        "qj2_device_check": (ctypes.c_int, []),
        "qj2_padded_size": (ctypes.c_int, [i64, i64, ctypes.POINTER(i64)]),
        "qj2_eval_workspace_size": (ctypes.c_int, [i64, i32, i64, ctypes.c_int, ctypes.POINTER(sz)]),
        "qj2_eval": (ctypes.c_int, [F, ctypes.c_int, i64, i64, i64, i64, i64, i64, vp, vp, i32, vp,
                                    vp, vp, vp, vp, vp, sz, vp]),
        "qj2_ratio": (ctypes.c_int, [i64, i32, vp, vp, vp, vp]),
        "qj2_accept_workspace_size": (ctypes.c_int, [i64, ctypes.c_int, ctypes.POINTER(sz)]),
        "qj2_accept": (ctypes.c_int, [F, ctypes.c_int, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp, i64, vp,
                                      vp, vp, i64, vp, sz, vp]),
        "qj2_metropolis": (ctypes.c_int, [i64, vp, i64, vp, vp, vp]),
        "qj2_sweep": (ctypes.c_int, [F, i64, i64, i64, i64, vp, vp, i64, vp, vp, vp, vp, vp,
                                     ctypes.POINTER(_SweepJ1), vp]),
        "qj2_state_init": (ctypes.c_int, [F, i64, i64, i64, i64, vp, vp, ctypes.POINTER(_SweepJ1), vp]),
        "qj2_metropolis_accept": (ctypes.c_int, [F, ctypes.c_int, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp, vp, i64,
                                                 vp, vp, i64, i64, vp, vp, vp]),
        "qj2_spo_eval": (ctypes.c_int, [ctypes.POINTER(_SpoTable), i32, ctypes.c_int, i64, vp, i64, vp, i64, i64,
                                        vp, i64, vp, vp, vp]),
        "qj2gen_spo_table": (ctypes.c_int, [ctypes.c_uint64, i64, i64, i64, i64, i64, vp, vp]),
        "qj2_eval_j1": (ctypes.c_int, [ctypes.POINTER(_J1Functor), ctypes.c_int, i64, ctypes.POINTER(i64), i64,
                                       vp, i32, vp, vp, vp, vp, vp, vp, sz, vp]),
        "qj2_eval_host_workspace_size": (ctypes.c_int, [i64, i32, i64, ctypes.c_int, i64, ctypes.POINTER(sz)]),
        "qj2_eval_host": (ctypes.c_int, [F, ctypes.c_int, i64, i64, i64, i64, i64, i64, vp, vp, i32, vp,
                                         vp, vp, vp, i64, vp, sz, vp]),
        "qj2_functor_eval_vgl": (ctypes.c_int, [F, ctypes.c_int, i32, i64, vp, vp, vp]),
        "qj2_min_image_disp": (ctypes.c_int, [dp, ctypes.c_int, i64, vp, vp, vp, vp]),
        "qj2_check_inputs": (ctypes.c_int, [F, ctypes.c_int, i64, i64, i64, i64, vp, vp, i32, vp, vp, vp]),
        "qj2gen_positions": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, i64, i64, i64, i64, i64,
                                            ctypes.c_double, vp, vp]),
    }
    for name, (res, args) in sigs.items():
        if not hasattr(lib, name) and os.environ.get("QJ2_LIB"):
            continue          # an older A/B build may lack newer entry points
        fnc = getattr(lib, name)
        fnc.restype = res
        fnc.argtypes = args
    return lib


_lib = _load()
EXPORTS = ("qj2_version", "qj2_status_string", "qj2_last_error", "qj2_device_check", "qj2_padded_size",
           "qj2_eval_workspace_size", "qj2_eval", "qj2_ratio", "qj2_eval_j1", "qj2_accept_workspace_size",
           "qj2_accept", "qj2_metropolis", "qj2_metropolis_accept", "qj2_sweep", "qj2_state_init", "qj2_spo_eval", "qj2gen_spo_table", "qj2_eval_host_workspace_size",
           "qj2_eval_host", "qj2_functor_eval_vgl", "qj2_min_image_disp", "qj2_check_inputs",
           "qj2gen_positions")


def _check(st: int, where: str):
    if st != 0:
        detail = _lib.qj2_last_error().decode() or _lib.qj2_status_string(st).decode()
        raise QJ2Error(st, where, detail)


def version() -> int:
    return _lib.qj2_version()


def device_check():
    _check(_lib.qj2_device_check(), "qj2_device_check")


class Functor:
    """Functor + cell in the C layout (qj2_functor)."""

    def __init__(self, L, r_cut: float, m: int, coef):
        coef = np.asarray(coef, dtype=np.float64)
        if coef.shape != (2, m + 3):
            raise ValueError(f"coef must be [2][m+3], got {coef.shape}")
        self.L = tuple(float(x) for x in (L if np.ndim(L) else (L, L, L)))
        self.r_cut, self.m, self.coef = float(r_cut), int(m), coef
        c = _Functor()
        for d in range(3):
            c.L[d] = self.L[d]
        c.r_cut, c.m, c.reserved = self.r_cut, self.m, 0
        for s in range(2):
            for j in range(m + 3):
                c.coef[s][j] = float(coef[s, j])
        self._c = c

    @classmethod
    def of(cls, fn) -> "Functor":
        return fn if isinstance(fn, Functor) else cls(fn.L, fn.r_cut, fn.m, fn.coef)

    @property
    def ptr(self):
        return ctypes.byref(self._c)


def _dtype_code(t: torch.dtype) -> int:
    if t == torch.float32:
        return QJ2_FP32
    if t == torch.float64:
        return QJ2_FP64
    raise TypeError(f"positions must be float32 or float64, got {t}")


def _stream_ptr(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _keep(stream, *tensors):
    """A call on a stream other than the current one: tensors this call allocated
    itself (workspaces, outputs it created) were allocated on the current stream,
    so the caching allocator must not hand their memory to that stream again
    before the kernels using them on `stream` have run (torch's record_stream)."""
    if stream is None or stream == torch.cuda.current_stream():
        return
    for t in tensors:
        if t is not None and t.is_cuda:
            t.record_stream(stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _req(t: torch.Tensor, name: str, dtype=None, ndim=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must have {ndim} dims, got {t.dim()}")


def _shape(t: torch.Tensor, name: str, shape):
    if tuple(t.shape) != tuple(int(x) for x in shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


def padded_size(n: int, block: int) -> int:
    out = ctypes.c_int64()
    _check(_lib.qj2_padded_size(int(n), int(block), ctypes.byref(out)), "qj2_padded_size")
    return out.value


def workspace_size(W: int, P: int, n_local: int, dtype: torch.dtype) -> int:
    b = ctypes.c_size_t()
    _check(_lib.qj2_eval_workspace_size(W, P, n_local, _dtype_code(dtype), ctypes.byref(b)),
           "qj2_eval_workspace_size")
    return b.value


class Workspace:
    """Reusable device scratch for qj2_eval / qj2_eval_host (grown on demand;
    the library initialises what it needs on every call)."""

    def __init__(self, nbytes: int = 0, device=None):
        self.device = device
        self.buf = None
        self.reserve(nbytes)

    def reserve(self, nbytes: int):
        if nbytes > 0 and (self.buf is None or self.buf.numel() < nbytes):
            self.buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8,
                                   device=self.device or torch.cuda.current_device())
        return self

    @property
    def nbytes(self) -> int:
        return 0 if self.buf is None else self.buf.numel()


def eval(R, k, r_trial, fn, n_total: int, n_up: int, *, i_offset: int = 0, n_local: int | None = None,
         row: bool = False, V_cur=None, ratio: bool = False, out=None, row_out=None, ratio_out=None,
         workspace: Workspace | None = None, stream=None):
    """qj2_eval on torch tensors (see include/qmcj2.h).

    R [W][3][Np] f32/f64, k [W] int32, r_trial [W][P][3] (same dtype as R).
    Returns out [W][P][5] fp64, plus row [W][P][4][Np] if row=True and
    ratio [W][P][2] if ratio=True.
    """
    _req(R, "R", ndim=3)
    W, three, Np = R.shape
    if three != 3:
        raise ValueError("R must be [W][3][Np]")
    _req(k, "k", torch.int32, 1)
    _req(r_trial, "r_trial", R.dtype, 3)
    P = r_trial.shape[1]
    if k.shape[0] != W or r_trial.shape[0] != W or r_trial.shape[2] != 3:
        raise ValueError("shape mismatch between R, k and r_trial")
    n_local = min(Np, n_total - i_offset) if n_local is None else int(n_local)
    f = Functor.of(fn)
    dev = R.device
    if out is None:
        out = torch.empty((W, P, 5), dtype=torch.float64, device=dev)
    _req(out, "out", torch.float64)
    _shape(out, "out", (W, P, 5))
    if row and row_out is None:
        row_out = torch.empty((W, P, 4, Np), dtype=R.dtype, device=dev)
    if row:
        _req(row_out, "row_out", R.dtype)
        _shape(row_out, "row_out", (W, P, 4, Np))
    if ratio and ratio_out is None:
        ratio_out = torch.empty((W, P, 2), dtype=torch.float64, device=dev)
    if ratio:
        _req(ratio_out, "ratio_out", torch.float64)
        _shape(ratio_out, "ratio_out", (W, P, 2))
    if V_cur is not None:
        _req(V_cur, "V_cur", torch.float64, 1)
        _shape(V_cur, "V_cur", (W,))
    need = workspace_size(max(W, 0), P, max(n_local, 1), R.dtype) if W > 0 and n_local >= 1 else 0
    ws = workspace if workspace is not None else Workspace(device=dev)
    ws.reserve(need)
    st = _lib.qj2_eval(f.ptr, _dtype_code(R.dtype), W, n_total, n_up, i_offset, n_local, Np,
                       _ptr(R), _ptr(k), P, _ptr(r_trial), _ptr(out),
                       _ptr(row_out) if row else None, _ptr(V_cur), _ptr(ratio_out) if ratio else None,
                       _ptr(ws.buf), ws.nbytes, ctypes.c_void_p(_stream_ptr(stream)))
    _check(st, "qj2_eval")
    _keep(stream, out, row_out, ratio_out, ws.buf)
    res = [out]
    if row:
        res.append(row_out)
    if ratio:
        res.append(ratio_out)
    return res[0] if len(res) == 1 else tuple(res)


class J1Functor:
    """Per-species one-body functors in the C layout (qj2_j1_functor)."""

    def __init__(self, L, r_cut, m, coef):
        r_cut = [float(x) for x in r_cut]
        m = [int(x) for x in m]
        coef = np.asarray(coef, dtype=np.float64)
        S = len(m)
        if not (1 <= S <= QJ2_MAX_SPECIES) or len(r_cut) != S or coef.shape[0] != S:
            raise ValueError("need 1..4 species with matching r_cut, m, coef")
        self.L = tuple(float(x) for x in (L if np.ndim(L) else (L, L, L)))
        self.r_cut, self.m, self.coef = tuple(r_cut), tuple(m), coef
        c = _J1Functor()
        for d in range(3):
            c.L[d] = self.L[d]
        c.n_species, c.reserved = S, 0
        for s in range(S):
            c.r_cut[s] = r_cut[s]
            c.m[s] = m[s]
            for j in range(min(coef.shape[1], QJ2_MAX_M + 3)):
                c.coef[s][j] = float(coef[s, j])
        self._c = c

    @classmethod
    def of(cls, fn) -> "J1Functor":
        return fn if isinstance(fn, J1Functor) else cls(fn.L, fn.r_cut, fn.m, fn.coef)

    @property
    def ptr(self):
        return ctypes.byref(self._c)


def eval_j1(ions, species_start, r_trial, fn1, *, row: bool = False, V_cur=None, ratio: bool = False,
            out=None, row_out=None, ratio_out=None, workspace: Workspace | None = None, stream=None):
    """qj2_eval_j1 (NEXT-1): one-body Jastrow over the AB row.

    ions [3][Np] (f32/f64, sorted by species), species_start [S+1] (host ints),
    r_trial [W][P][3] (same dtype).  Returns out [W][P][5] fp64 (and row
    [W][P][4][Np], ratio [W][P][2])."""
    _req(ions, "ions", ndim=2)
    _req(r_trial, "r_trial", ions.dtype, 3)
    W, P = r_trial.shape[0], r_trial.shape[1]
    if ions.shape[0] != 3 or r_trial.shape[2] != 3:
        raise ValueError("ions must be [3][Np] and r_trial [W][P][3]")
    Np = ions.shape[1]
    f = J1Functor.of(fn1)
    if len(species_start) != len(f.m) + 1 or int(species_start[-1]) > Np:
        raise ValueError("species_start must have n_species + 1 entries and end <= Np")
    st = (ctypes.c_int64 * (len(f.m) + 1))(*[int(x) for x in species_start])
    n_ions = int(species_start[-1])
    dev = ions.device
    if out is None:
        out = torch.empty((W, P, 5), dtype=torch.float64, device=dev)
    _req(out, "out", torch.float64)
    _shape(out, "out", (W, P, 5))
    if row and row_out is None:
        row_out = torch.empty((W, P, 4, Np), dtype=ions.dtype, device=dev)
    if row:
        _req(row_out, "row_out", ions.dtype)
        _shape(row_out, "row_out", (W, P, 4, Np))
    if ratio and ratio_out is None:
        ratio_out = torch.empty((W, P, 2), dtype=torch.float64, device=dev)
    if ratio:
        _req(ratio_out, "ratio_out", torch.float64)
        _shape(ratio_out, "ratio_out", (W, P, 2))
    if V_cur is not None:
        _req(V_cur, "V_cur", torch.float64, 1)
        _shape(V_cur, "V_cur", (W,))
    need = workspace_size(W, P, max(n_ions, 1), ions.dtype) if W > 0 else 0
    ws = workspace if workspace is not None else Workspace(device=dev)
    ws.reserve(need)
    _check(_lib.qj2_eval_j1(f.ptr, _dtype_code(ions.dtype), W, st, Np, _ptr(ions), P, _ptr(r_trial), _ptr(out),
                            _ptr(row_out) if row else None, _ptr(V_cur), _ptr(ratio_out) if ratio else None,
                            _ptr(ws.buf), ws.nbytes, ctypes.c_void_p(_stream_ptr(stream))), "qj2_eval_j1")
    _keep(stream, out, row_out, ratio_out, ws.buf)
    res = [out]
    if row:
        res.append(row_out)
    if ratio:
        res.append(ratio_out)
    return res[0] if len(res) == 1 else tuple(res)


def ratio(out, V_cur=None, ratio_out=None, stream=None):
    """qj2_ratio: (dJ2, exp(dJ2)) per (w, p) from (reduced) `out`."""
    _req(out, "out", torch.float64, 3)
    W, P, _ = out.shape
    if ratio_out is None:
        ratio_out = torch.empty((W, P, 2), dtype=torch.float64, device=out.device)
    _req(ratio_out, "ratio_out", torch.float64)
    _shape(ratio_out, "ratio_out", (W, P, 2))
    if V_cur is not None:
        _req(V_cur, "V_cur", torch.float64, 1)
        _shape(V_cur, "V_cur", (W,))
    _check(_lib.qj2_ratio(W, P, _ptr(out), _ptr(V_cur), _ptr(ratio_out), ctypes.c_void_p(_stream_ptr(stream))),
           "qj2_ratio")
    _keep(stream, ratio_out)
    return ratio_out


def _row_ptr(t: torch.Tensor, trial: int, width: int, W: int | None = None):
    """(pointer, stride in elements) of trial `trial` of a [W][P][width]
    (or [W][width]) contiguous tensor (W checked when given)."""
    if t.dim() not in (2, 3) or t.shape[-1] != width or (W is not None and t.shape[0] != W):
        raise ValueError(f"expected a [W={W}][P][{width}] or [W][{width}] tensor, got {tuple(t.shape)}")
    if t.dim() == 2:
        if trial != 0:
            raise ValueError("trial index on a [W][width] tensor")
        return ctypes.c_void_p(t.data_ptr()), width
    P = t.shape[1]
    if not 0 <= trial < P:
        raise ValueError(f"trial {trial} out of range [0, {P})")
    return ctypes.c_void_p(t.data_ptr() + trial * width * t.element_size()), width * P


def accept(R, state, k, r_new, acc, out_new, fn, n_total: int, n_up: int, *, trial: int = 0, i_offset: int = 0,
           n_local: int | None = None, r_old=None, workspace: Workspace | None = None, stream=None):
    """qj2_accept (NEXT-2): in place on R [W][3][Np] and state [W][5][Np]
    (same dtype).  k [W] int32, acc [W] int32 (nonzero = accepted); r_new
    [W][P][3] (or [W][3]) and out_new (qj2_eval's out [W][P][5] fp64, or
    [W][5]): trial `trial` is the accepted move.  Returns (R, state)."""
    _req(R, "R", ndim=3)
    W, _, Np = R.shape
    _req(state, "state", R.dtype, 3)
    if tuple(state.shape) != (W, 5, Np):
        raise ValueError("state must be [W][5][Np]")
    _req(k, "k", torch.int32, 1)
    _shape(k, "k", (W,))
    _req(acc, "acc", torch.int32, 1)
    _shape(acc, "acc", (W,))
    _req(r_new, "r_new", R.dtype)
    if r_old is not None:
        _req(r_old, "r_old", R.dtype, 2)
        _shape(r_old, "r_old", (W, 3))
    _req(out_new, "out_new", torch.float64)
    rp, rs = _row_ptr(r_new, trial, 3, W)
    op, os_ = _row_ptr(out_new, trial, 5, W)
    n_local = min(Np, n_total - i_offset) if n_local is None else int(n_local)
    f = Functor.of(fn)
    b = ctypes.c_size_t()
    _check(_lib.qj2_accept_workspace_size(W, _dtype_code(R.dtype), ctypes.byref(b)), "qj2_accept_workspace_size")
    ws = workspace if workspace is not None else Workspace(device=R.device)
    if r_old is None:
        ws.reserve(b.value)
    _check(_lib.qj2_accept(f.ptr, _dtype_code(R.dtype), W, n_total, n_up, i_offset, n_local, Np,
                           _ptr(R), _ptr(state), _ptr(k), rp, rs, _ptr(r_old), _ptr(acc),
                           op, os_, _ptr(ws.buf), ws.nbytes,
                           ctypes.c_void_p(_stream_ptr(stream))), "qj2_accept")
    _keep(stream, ws.buf)
    return R, state


def metropolis_accept(R, state, k, r_trial, out, u, fn, n_total: int, n_up: int, *, acc=None, trial_new: int = 1,
                      trial_old: int = 0, V_cur=None, i_offset: int = 0, n_local: int | None = None, stream=None):
    """qj2_metropolis_accept: the Metropolis test (u < exp(2 (V_new - V_ref)))
    fused into the accept-side update, one launch.  r_trial [W][P][3] holds
    r_k (trial_old) and r'_k (trial_new), out is qj2_eval's [W][P][5];
    V_ref = V_cur [W] if given, else out[:, trial_old, 0].  Returns acc [W]."""
    _req(R, "R", ndim=3)
    W, _, Np = R.shape
    _req(state, "state", R.dtype, 3)
    _shape(state, "state", (W, 5, Np))
    _req(k, "k", torch.int32, 1)
    _shape(k, "k", (W,))
    _req(r_trial, "r_trial", R.dtype, 3)
    _req(out, "out", torch.float64, 3)
    if out.shape[1] != r_trial.shape[1]:
        raise ValueError("out and r_trial must have the same number of trials")
    _req(u, "u", torch.float64, 1)
    _shape(u, "u", (W,))
    rn, rs = _row_ptr(r_trial, trial_new, 3, W)
    ro, _ = _row_ptr(r_trial, trial_old, 3, W)
    on, os_ = _row_ptr(out, trial_new, 5, W)
    if V_cur is not None:
        _req(V_cur, "V_cur", torch.float64, 1)
        _shape(V_cur, "V_cur", (W,))
        vr, vrs = _ptr(V_cur), 1
    else:
        vr, vrs = _row_ptr(out, trial_old, 5, W)
    if acc is None:
        acc = torch.empty(W, dtype=torch.int32, device=R.device)
    _req(acc, "acc", torch.int32, 1)
    _shape(acc, "acc", (W,))
    n_local = min(Np, n_total - i_offset) if n_local is None else int(n_local)
    f = Functor.of(fn)
    _check(_lib.qj2_metropolis_accept(f.ptr, _dtype_code(R.dtype), W, n_total, n_up, i_offset, n_local, Np,
                                      _ptr(R), _ptr(state), _ptr(k), rn, ro, rs, on, vr, os_, vrs, _ptr(u),
                                      _ptr(acc), ctypes.c_void_p(_stream_ptr(stream))), "qj2_metropolis_accept")
    _keep(stream, acc)
    return acc


def _sweep_j1(j1, W, Np):
    """(ctypes qj2_sweep_j1, objects to keep alive) for j1 = (ions [3][Np_ion] fp32,
    species_start, fn1, state_j1 [W][5][Np] fp32) or None."""
    if j1 is None:
        return None, []
    ions, start, fn1, state_j1 = j1
    _req(ions, "ions", torch.float32, 2)
    if ions.shape[0] != 3:
        raise ValueError("ions must be [3][Np_ion]")
    _req(state_j1, "state_j1", torch.float32, 3)
    _shape(state_j1, "state_j1", (W, 5, Np))
    f1 = J1Functor.of(fn1)
    if len(start) != len(f1.m) + 1 or int(start[-1]) > ions.shape[1]:
        raise ValueError("species_start must have n_species + 1 entries and end <= Np_ion")
    st = (ctypes.c_int64 * (len(f1.m) + 1))(*[int(x) for x in start])
    s1 = _SweepJ1(ctypes.addressof(f1._c), st, ions.data_ptr(), ions.shape[1], state_j1.data_ptr())
    return ctypes.byref(s1), [f1, st, s1]


def sweep(R, state, ks, delta, u, fn, n: int, n_up: int, *, acc=None, dj=None, j1=None, stream=None):
    """qj2_sweep: S particle-by-particle moves of every walker in one launch,
    walkers resident in shared memory (N <= 1024, fp32, functor m <= 16).
    R [W][3][Np], state [W][5][Np] fp32 (in place, consistent with R: see
    state_init); ks [S][W] int32, delta [S][W][3] fp32 (r'_k = wrap(r_k + delta)
    from the walker's current r_k), u [S][W] fp64.  j1 = (ions [3][Np_ion] fp32,
    species_start, fn1, state_j1 [W][5][Np] fp32) adds the one-body Jastrow to
    every move's ratio.  Returns (acc [S][W] int32, dj [S][W] fp64)."""
    _req(R, "R", torch.float32, 3)
    W, three, Np = R.shape
    if three != 3:
        raise ValueError("R must be [W][3][Np]")
    _req(state, "state", torch.float32, 3)
    _shape(state, "state", (W, 5, Np))
    _req(ks, "ks", torch.int32, 2)
    S = ks.shape[0]
    _shape(ks, "ks", (S, W))
    _req(delta, "delta", torch.float32, 3)
    _shape(delta, "delta", (S, W, 3))
    _req(u, "u", torch.float64, 2)
    _shape(u, "u", (S, W))
    if acc is None:
        acc = torch.empty((S, W), dtype=torch.int32, device=R.device)
    _req(acc, "acc", torch.int32, 2)
    _shape(acc, "acc", (S, W))
    if dj is None:
        dj = torch.empty((S, W), dtype=torch.float64, device=R.device)
    _req(dj, "dj", torch.float64, 2)
    _shape(dj, "dj", (S, W))
    f = Functor.of(fn)
    j1p, keep = _sweep_j1(j1, W, Np)
    _check(_lib.qj2_sweep(f.ptr, W, n, n_up, Np, _ptr(R), _ptr(state), S, _ptr(ks), _ptr(delta), _ptr(u),
                          _ptr(acc), _ptr(dj), j1p, ctypes.c_void_p(_stream_ptr(stream))), "qj2_sweep")
    _keep(stream, acc, dj)
    del keep
    return acc, dj


def state_init(R, state, fn, n: int, n_up: int, *, j1=None, stream=None):
    """qj2_state_init: the 5N J2 state of every electron from scratch into
    state [W][5][Np] fp32 (and, with j1 as for sweep(), every electron's J1 row
    into state_j1).  R [W][3][Np] fp32.  Returns state."""
    _req(R, "R", torch.float32, 3)
    W, three, Np = R.shape
    if three != 3:
        raise ValueError("R must be [W][3][Np]")
    _req(state, "state", torch.float32, 3)
    _shape(state, "state", (W, 5, Np))
    f = Functor.of(fn)
    j1p, keep = _sweep_j1(j1, W, Np)
    _check(_lib.qj2_state_init(f.ptr, W, n, n_up, Np, _ptr(R), _ptr(state), j1p,
                               ctypes.c_void_p(_stream_ptr(stream))), "qj2_state_init")
    del keep
    return state


def metropolis(ratio_out, u, acc=None, *, trial: int = 0, stream=None):
    """qj2_metropolis: acc[w] = u[w] < rho^2 with rho = ratio_out[w][trial][1]
    (ratio_out [W][P][2] or [W][2] fp64; u [W] fp64 uniforms in [0, 1))."""
    _req(ratio_out, "ratio_out", torch.float64)
    _req(u, "u", torch.float64, 1)
    W = u.shape[0]
    rp, rs = _row_ptr(ratio_out, trial, 2, W)
    if acc is None:
        acc = torch.empty(W, dtype=torch.int32, device=u.device)
    _req(acc, "acc", torch.int32, 1)
    _shape(acc, "acc", (W,))
    _check(_lib.qj2_metropolis(W, rp, rs, _ptr(u), _ptr(acc), ctypes.c_void_p(_stream_ptr(stream))),
           "qj2_metropolis")
    _keep(stream, acc)
    return acc


QJ2_SPO_V, QJ2_SPO_VGH, QJ2_SPO_GATHER = 0, 1, 0x10


class SpoTable:
    """A read-only 3D B-spline SPO table (qj2_spo_table): coef is a CUDA fp32
    tensor [nx][ny][nz][ld] (ld % 4 == 0) holding n_orb orbitals per row."""

    def __init__(self, coef: torch.Tensor, n_orb: int, L):
        _req(coef, "coef", torch.float32, 4)
        self.coef = coef
        self.n_orb = int(n_orb)
        self.L = tuple(float(x) for x in (L if np.ndim(L) else (L, L, L)))
        nx, ny, nz, ld = coef.shape
        c = _SpoTable()
        for d in range(3):
            c.L[d] = self.L[d]
        c.nx, c.ny, c.nz, c.n_orb, c.ld = nx, ny, nz, self.n_orb, ld
        c.coef = coef.data_ptr()
        self._c = c

    @property
    def ptr(self):
        return ctypes.byref(self._c)


def spo_eval(tab: SpoTable, pos, *, vgh: bool = True, Ainv=None, krow=None, trial: int = 0, all_trials: bool = False,
             out=None, spo_out=None, want_spo: bool = False, kernel: str = "auto", stream=None):
    """qj2_spo_eval (NEXT-4): Bspline-vgh (vgh=True) or Bspline-v at pos
    ([W][3], or [W][P][3]: trial `trial`, or every trial with all_trials=True --
    then the P points of a walker share its A^{-1} row, e.g. the NLPP
    quadrature), fused with the determinant ratio against Ainv (fp32,
    [W][n][lda] with krow [W] int32, or [W][lda] rows).  Returns out
    [W*P or W][5] fp64 (rho, G, L) (None without Ainv) and, if want_spo, spo
    [evaluations][10 or 1][ld] fp32.  kernel="gather" selects the per-thread-gather
    kernel (QJ2_SPO_GATHER) instead of the automatic choice."""
    if kernel not in ("auto", "gather"):
        raise ValueError("kernel must be 'auto' or 'gather'")
    _req(pos, "pos")
    ppw = 1
    if all_trials and pos.dim() == 3:
        ppw = pos.shape[1]
        pos = pos.reshape(-1, 3)
    W = pos.shape[0]
    pp, ps = _row_ptr(pos, trial if not all_trials else 0, 3)
    ldv = tab.coef.shape[3]
    dev = pos.device
    a_ptr, a_stride, a_ld = None, 0, 0
    if Ainv is not None:
        _req(Ainv, "Ainv", torch.float32)
        n_walk = W // ppw                # walkers owning an A^{-1} row (points_per_walker points each)
        if W % ppw:
            raise ValueError("the evaluation count must be a multiple of points_per_walker")
        if Ainv.dim() == 3:
            if krow is None:
                raise ValueError("krow is required with a [W][n][lda] Ainv")
            _req(krow, "krow", torch.int32, 1)
            _shape(krow, "krow", (n_walk,))
            if Ainv.shape[0] != n_walk or Ainv.shape[2] < tab.n_orb:
                raise ValueError(f"Ainv must be [{n_walk}][n][>= {tab.n_orb}], got {tuple(Ainv.shape)}")
            a_stride, a_ld = Ainv.shape[1] * Ainv.shape[2], Ainv.shape[2]
        elif Ainv.dim() == 2:
            if Ainv.shape[0] != n_walk or Ainv.shape[1] < tab.n_orb:
                raise ValueError(f"Ainv must be [{n_walk}][>= {tab.n_orb}], got {tuple(Ainv.shape)}")
            a_stride, a_ld = Ainv.shape[1], Ainv.shape[1]
            krow = None
        else:
            raise ValueError("Ainv must be [W][n][lda] (with krow) or [W][lda]")
        a_ptr = _ptr(Ainv)
        if out is None:
            out = torch.empty((W, 5), dtype=torch.float64, device=dev)
        _req(out, "out", torch.float64)
        _shape(out, "out", (W, 5))
    if want_spo and spo_out is None:
        spo_out = torch.empty((W, 10 if vgh else 1, ldv), dtype=torch.float32, device=dev)
    if spo_out is not None:
        _req(spo_out, "spo_out", torch.float32)
        _shape(spo_out, "spo_out", (W, 10 if vgh else 1, ldv))
    what = (QJ2_SPO_VGH if vgh else QJ2_SPO_V) | (QJ2_SPO_GATHER if kernel == "gather" else 0)
    _check(_lib.qj2_spo_eval(tab.ptr, what, _dtype_code(pos.dtype), W, pp, ps,
                             a_ptr, a_stride, a_ld, _ptr(krow), ppw, _ptr(out) if Ainv is not None else None,
                             _ptr(spo_out), ctypes.c_void_p(_stream_ptr(stream))), "qj2_spo_eval")
    _keep(stream, out if Ainv is not None else None, spo_out)
    if want_spo:
        return out, spo_out
    return out


def gen_spo_table(seed: int, nx: int, ny: int, nz: int, n_orb: int, ld: int | None = None, stream=None,
                  device=None) -> torch.Tensor:
    """Device synthetic SPO table (harness; same recipe as qmcgen.spo_table)."""
    ld = n_orb if ld is None else ld
    coef = torch.empty((nx, ny, nz, ld), dtype=torch.float32, device=device or torch.cuda.current_device())
    _check(_lib.qj2gen_spo_table(int(seed) & 0xFFFFFFFFFFFFFFFF, nx, ny, nz, n_orb, ld, _ptr(coef),
                                 ctypes.c_void_p(_stream_ptr(stream))), "qj2gen_spo_table")
    return coef


def host_workspace_size(W, P, Np, dtype, chunk_walkers) -> int:
    b = ctypes.c_size_t()
    _check(_lib.qj2_eval_host_workspace_size(W, P, Np, _dtype_code(dtype), chunk_walkers, ctypes.byref(b)),
           "qj2_eval_host_workspace_size")
    return b.value


def eval_host(R, k, r_trial, fn, n_total: int, n_up: int, *, i_offset: int = 0, n_local: int | None = None,
              V_cur=None, ratio: bool = False, chunk_walkers: int = 16, out=None, ratio_out=None,
              workspace: Workspace | None = None, stream=None):
    """qj2_eval_host: HOST tensors in (pinned for full PCIe rate), host out.

    R [W][3][Np] (CPU torch tensor), k [W] int32, r_trial [W][P][3]; returns
    out [W][P][5] fp64 CPU tensor (and ratio [W][P][2])."""
    for t, nm in ((R, "R"), (k, "k"), (r_trial, "r_trial")):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{nm} must be a contiguous host tensor")
    if R.dim() != 3 or R.shape[1] != 3:
        raise ValueError("R must be [W][3][Np]")
    W, _, Np = R.shape
    if r_trial.dim() != 3 or r_trial.shape[0] != W or r_trial.shape[2] != 3 or r_trial.dtype != R.dtype:
        raise ValueError("r_trial must be [W][P][3] of R's dtype")
    if tuple(k.shape) != (W,) or k.dtype != torch.int32:
        raise ValueError("k must be [W] int32")
    P = r_trial.shape[1]
    n_local = min(Np, n_total - i_offset) if n_local is None else int(n_local)
    if out is None:
        out = torch.empty((W, P, 5), dtype=torch.float64, pin_memory=R.is_pinned())
    if ratio and ratio_out is None:
        ratio_out = torch.empty((W, P, 2), dtype=torch.float64, pin_memory=R.is_pinned())
    for t, nm, shp in ((out, "out", (W, P, 5)), (ratio_out if ratio else None, "ratio_out", (W, P, 2)),
                       (V_cur, "V_cur", (W,))):
        if t is not None and (t.is_cuda or not t.is_contiguous() or t.dtype != torch.float64 or tuple(t.shape) != shp):
            raise ValueError(f"{nm} must be a contiguous fp64 host tensor of shape {shp}")
    f = Functor.of(fn)
    need = host_workspace_size(W, P, Np, R.dtype, chunk_walkers)
    ws = workspace if workspace is not None else Workspace(device=torch.cuda.current_device())
    ws.reserve(need)
    st = _lib.qj2_eval_host(f.ptr, _dtype_code(R.dtype), W, n_total, n_up, i_offset, n_local, Np,
                            _ptr(R), _ptr(k), P, _ptr(r_trial), _ptr(out), _ptr(V_cur),
                            _ptr(ratio_out) if ratio else None, chunk_walkers,
                            _ptr(ws.buf), ws.nbytes, ctypes.c_void_p(_stream_ptr(stream)))
    _check(st, "qj2_eval_host")
    return (out, ratio_out) if ratio else out


def functor_eval_vgl(fn, channel: int, r, stream=None):
    _req(r, "r", ndim=1)
    f = Functor.of(fn)
    out = torch.empty((r.shape[0], 3), dtype=torch.float64, device=r.device)
    _check(_lib.qj2_functor_eval_vgl(f.ptr, _dtype_code(r.dtype), channel, r.shape[0], _ptr(r), _ptr(out),
                                     ctypes.c_void_p(_stream_ptr(stream))), "qj2_functor_eval_vgl")
    return out


def min_image_disp(L, a, b, stream=None):
    _req(a, "a", ndim=2)
    _req(b, "b", a.dtype, 2)
    Ls = (ctypes.c_double * 3)(*[float(x) for x in (L if np.ndim(L) else (L, L, L))])
    out = torch.empty((a.shape[0], 4), dtype=a.dtype, device=a.device)
    _check(_lib.qj2_min_image_disp(Ls, _dtype_code(a.dtype), a.shape[0], _ptr(a), _ptr(b), _ptr(out),
                                   ctypes.c_void_p(_stream_ptr(stream))), "qj2_min_image_disp")
    return out


def check_inputs(R, k, r_trial, fn, n_total: int, n_local: int | None = None, stream=None) -> int:
    """Device precondition scan; returns the flag bits (0 = clean)."""
    W, _, Np = R.shape
    n_local = min(Np, n_total) if n_local is None else n_local
    flag = torch.zeros(1, dtype=torch.int32, device=R.device)
    f = Functor.of(fn)
    _check(_lib.qj2_check_inputs(f.ptr, _dtype_code(R.dtype), W, n_total, n_local, Np, _ptr(R), _ptr(k),
                                 r_trial.shape[1], _ptr(r_trial), _ptr(flag),
                                 ctypes.c_void_p(_stream_ptr(stream))), "qj2_check_inputs")
    return int(flag.item())


def gen_positions(seed: int, W: int, N_local: int, Np: int, L: float, dtype=torch.float32, *,
                  w_offset: int = 0, i_offset: int = 0, out=None, stream=None, device=None):
    """Device synthetic-input generator (harness; same recipe as qmcgen)."""
    if out is None:
        out = torch.empty((W, 3, Np), dtype=dtype, device=device or torch.cuda.current_device())
    _check(_lib.qj2gen_positions(_dtype_code(out.dtype), int(seed) & 0xFFFFFFFFFFFFFFFF, W, w_offset,
                                 i_offset, N_local, Np, float(L), _ptr(out),
                                 ctypes.c_void_p(_stream_ptr(stream))), "qj2gen_positions")
    return out
