"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper over oracle/oracle.c, the plain fp64 CPU oracle of the J2 /
distance-row hot path (see oracle.c for the citations of every function).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this package.  It shares no code with
paper_1708_02645_b200/ and never imports it.

Parity status: pinned (tests/test_oracle_pins.py, test_oracle_accept.py,
test_oracle_spo.py, test_inputs.py; mutation check in
test_oracle_mutations.py); nothing is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GCC_FLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared",
             "-std=c11", "-pthread"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no SIMD pragmas, no fast-math, no FMA
    contraction so every product/sum rounds once as written)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *GCC_FLAGS, "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        # ORACLE_LIB: a deliberately mutated build, loaded by tests/test_oracle_mutations.py
        # to show that the pins catch plausible mistakes (test infrastructure only)
        _lib = ctypes.CDLL(os.environ.get("ORACLE_LIB") or build())
        dp = ctypes.POINTER(ctypes.c_double)
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64 = ctypes.c_int64
        _lib.orc_eval.restype = i64
        _lib.orc_eval.argtypes = [dp, ctypes.c_double, ctypes.c_int, dp,
                                  i64, i64, i64, i64, i64, i64,
                                  dp, i32p, ctypes.c_int32, dp,
                                  dp, dp, dp, ctypes.c_int]
        _lib.orc_eval_f32.restype = i64
        _lib.orc_eval_f32.argtypes = [dp, ctypes.c_double, ctypes.c_int, dp,
                                      i64, i64, i64, i64, i64, i64,
                                      ctypes.c_void_p, i32p, ctypes.c_int32, ctypes.c_void_p,
                                      dp, dp, dp, ctypes.c_int]
        _lib.orc_gen_positions.restype = None
        _lib.orc_gen_positions.argtypes = [ctypes.c_uint64, i64, i64, i64, i64, ctypes.c_double,
                                           ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
        _lib.orc_eval_j1.restype = i64
        _lib.orc_eval_j1.argtypes = [dp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), dp,
                                     ctypes.POINTER(ctypes.c_int), dp, ctypes.c_int,
                                     i64, i64, i64, dp, ctypes.c_int32, dp, dp, dp]
        _lib.orc_j2_total.restype = ctypes.c_double
        _lib.orc_j2_total.argtypes = [dp, ctypes.c_double, ctypes.c_int, dp,
                                      i64, i64, i64, dp]
        _lib.orc_bspline_batch.restype = None
        _lib.orc_bspline_batch.argtypes = [dp, ctypes.c_int, ctypes.c_double, i64, dp, dp]
        _lib.orc_min_image_batch.restype = None
        _lib.orc_min_image_batch.argtypes = [dp, i64, dp, dp, dp]
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class CoincidentError(ValueError):
    """r == 0 inside the cutoff (reading R9: undefined; the oracle refuses)."""


def eval_j2(R, k, r_trial, fn, n_total: int, n_up: int, i_offset: int = 0,
            row: bool = False, threads: int = 1, n_local: int | None = None):
    """Oracle of qj2_eval.

    R: [W][3][Np] (fp32 or fp64; promoted exactly), k: [W] global indices,
    r_trial: [W][P][3], fn: qmcgen.Functor-like (L, r_cut, m, coef[2][m+3]).
    Returns (out[W][P][5], abs[W][P][5], row[W][P][4][Np] or None), fp64.
    """
    f32 = (np.asarray(R).dtype == np.float32 and np.asarray(r_trial).dtype == np.float32)
    if f32:   # promoted element by element inside the oracle (exact)
        R = np.ascontiguousarray(R)
        rt = np.ascontiguousarray(r_trial)
    else:
        R = _f64(R)
        rt = _f64(r_trial)
    W, three, Np = R.shape
    assert three == 3
    N_local = min(Np, n_total - i_offset) if n_local is None else int(n_local)
    P = rt.shape[1]
    k = np.ascontiguousarray(np.asarray(k, dtype=np.int32))
    L = _f64(fn.L)
    coef = _f64(fn.coef)
    out = np.zeros((W, P, 5))
    absout = np.zeros((W, P, 5))
    rowout = np.full((W, P, 4, Np), np.nan) if row else None
    entry = lib().orc_eval_f32 if f32 else lib().orc_eval
    st = entry(_dp(L), float(fn.r_cut), int(fn.m), _dp(coef),
               W, n_total, n_up, i_offset, N_local, Np,
               R.ctypes.data_as(ctypes.c_void_p) if f32 else _dp(R),
               k.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
               P, rt.ctypes.data_as(ctypes.c_void_p) if f32 else _dp(rt), _dp(out), _dp(absout),
               _dp(rowout) if row else ctypes.POINTER(ctypes.c_double)(),
               int(threads))
    if st:
        raise CoincidentError(f"coincident source at (w*P+p) = {st - 1}")
    return out, absout, rowout


def eval_j1(ions, species_start, r_trial, fn1):
    """Oracle of qj2_eval_j1 (NEXT-1).  ions: [3][Np] sorted by species,
    species_start: [S+1], r_trial [W][P][3], fn1: qmcgen.J1Functor-like
    (L, r_cut[S], m[S], coef[S][max_m+3]).  Returns (out, abs) [W][P][5]."""
    ions = _f64(ions)
    rt = _f64(r_trial)
    W, P = rt.shape[0], rt.shape[1]
    S = len(fn1.m)
    st = np.ascontiguousarray(np.asarray(species_start, dtype=np.int64))
    rc = _f64(fn1.r_cut)
    mm = np.ascontiguousarray(np.asarray(fn1.m, dtype=np.int32))
    coef = _f64(fn1.coef)
    out = np.zeros((W, P, 5))
    absout = np.zeros((W, P, 5))
    r = lib().orc_eval_j1(_dp(_f64(fn1.L)), S, st.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(rc),
                          mm.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _dp(coef), coef.shape[1],
                          W, int(st[-1]), ions.shape[1], _dp(ions), P, _dp(rt), _dp(out), _dp(absout))
    if r:
        raise CoincidentError(f"ion coincides with trial (w*P+p) = {r - 1}")
    return out, absout


def normalized_error_j1(gpu, orc, absout, fn1) -> np.ndarray:
    """Parity metric for J1: as normalized_error with the functor scale taken
    over all species (max|c|, max|c|/delta_s, max|c|/delta_s^2)."""
    cmax = float(np.max(np.abs(fn1.coef)))
    dmin = min(rc / m for rc, m in zip(fn1.r_cut, fn1.m))
    F = np.array([cmax, cmax / dmin, cmax / dmin, cmax / dmin, cmax / dmin ** 2])
    return np.abs(np.asarray(gpu, dtype=np.float64) - orc) / np.maximum(absout, F)


def gen_positions(seed: int, walkers_begin: int, n_walkers: int, N: int, Np: int, L: float,
                  dtype, threads: int = 1) -> np.ndarray:
    """Oracle-side C twin of qmcgen.positions for contiguous global walker ids
    [walkers_begin, walkers_begin + n_walkers) (input generation only)."""
    f32 = np.dtype(dtype) == np.float32
    out = np.empty((n_walkers, 3, Np), dtype=np.float32 if f32 else np.float64)
    lib().orc_gen_positions(int(seed) & 0xFFFFFFFFFFFFFFFF, walkers_begin, n_walkers, N, Np, float(L),
                            1 if f32 else 0, out.ctypes.data_as(ctypes.c_void_p), int(threads))
    return out


def j2_total(R1, n: int, n_up: int, fn) -> float:
    """Brute-force J2 = sum_{i<j} U(r_ij) of one configuration R1[3][Np]."""
    R1 = _f64(R1)
    return lib().orc_j2_total(_dp(_f64(fn.L)), float(fn.r_cut), int(fn.m),
                              _dp(_f64(fn.coef)), n, n_up, R1.shape[1], _dp(R1))


def bspline(coef_channel, m: int, r_cut: float, r) -> np.ndarray:
    """[n][3] = (U, U', U'') of one channel at distances r."""
    r = _f64(np.atleast_1d(r))
    c = _f64(coef_channel)
    out = np.zeros((r.size, 3))
    lib().orc_bspline_batch(_dp(c), int(m), float(r_cut), r.size, _dp(r), _dp(out))
    return out


def min_image(L, a, b) -> np.ndarray:
    """[n][4] = (dist, dx, dy, dz) of b - a wrapped (a, b: [n][3])."""
    a = _f64(np.atleast_2d(a))
    b = _f64(np.atleast_2d(b))
    out = np.zeros((a.shape[0], 4))
    lib().orc_min_image_batch(_dp(_f64(L)), a.shape[0], _dp(a), _dp(b), _dp(out))
    return out


def normalized_error(gpu, orc, absout, fn) -> np.ndarray:
    """Parity metric (reading R14): per component
    |s_gpu - s_orc| / max(A_s, F_s), F = max|c| (V), max|c|/delta (G),
    max|c|/delta^2 (L)."""
    cmax = float(np.max(np.abs(fn.coef)))
    delta = fn.r_cut / fn.m
    F = np.array([cmax, cmax / delta, cmax / delta, cmax / delta, cmax / delta ** 2])
    denom = np.maximum(absout, F)
    return np.abs(np.asarray(gpu, dtype=np.float64) - orc) / denom


def plain_relative_error(gpu, orc, absout, floor: float = 1e-3):
    """The plain relative error SURVEY 8(c) asks to report beside the normalized
    one: max |s_gpu - s_orc| / |s_orc| over components with |s_orc| >= floor * A_s
    (per component V, Gx, Gy, Gz, L; None where no component qualifies)."""
    g = np.asarray(gpu, dtype=np.float64)
    out = []
    for c in range(orc.shape[-1]):
        o, a, x = orc[..., c], absout[..., c], g[..., c]
        m = (np.abs(o) >= floor * a) & (np.abs(o) > 0)
        out.append(float(np.max(np.abs(x[m] - o[m]) / np.abs(o[m]))) if m.any() else None)
    return out


def _lib_next2():
    L = lib()
    if not getattr(L, "_next2", False):
        dp = ctypes.POINTER(ctypes.c_double)
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64 = ctypes.c_int64
        L.orc_j2_state.restype = i64
        L.orc_j2_state.argtypes = [dp, ctypes.c_double, ctypes.c_int, dp, i64, i64, i64, dp, dp, dp]
        L.orc_accept.restype = i64
        L.orc_accept.argtypes = [dp, ctypes.c_double, ctypes.c_int, dp, i64, i64, i64, i64,
                                 dp, dp, i32p, dp, i32p, dp]
        L._next2 = True
    return L


def j2_state(R1, n: int, n_up: int, fn):
    """NEXT-2: per-electron J2 state of one configuration R1[3][Np] from
    scratch: (state[5][Np], abs[5][Np]) with rows V, Gx, Gy, Gz, L (see
    orc_j2_state).  Slots >= n are 0."""
    R1 = _f64(R1)
    Np = R1.shape[1]
    st = np.zeros((5, Np))
    ab = np.zeros((5, Np))
    r = _lib_next2().orc_j2_state(_dp(_f64(fn.L)), float(fn.r_cut), int(fn.m), _dp(_f64(fn.coef)),
                                  n, n_up, Np, _dp(R1), _dp(st), _dp(ab))
    if r:
        raise CoincidentError(f"electron {r - 1} has a coincident partner")
    return st, ab


def accept(R, state, k, r_new, acc, fn, n: int, n_up: int):
    """NEXT-2 oracle of qj2_accept (orc_accept): returns (R', state', abs)
    as fp64 copies; inputs (fp32 or fp64) are promoted exactly.
    R [W][3][Np], state [W][5][Np], k [W], r_new [W][3], acc [W] (nonzero =
    accepted).  abs is NaN for rejected walkers."""
    R2 = _f64(R).copy()
    S2 = _f64(state).copy()
    W, _, Np = R2.shape
    ab = np.full((W, 5, Np), np.nan)
    k = np.ascontiguousarray(np.asarray(k, dtype=np.int32))
    a = np.ascontiguousarray(np.asarray(acc, dtype=np.int32))
    rn = _f64(np.asarray(r_new).reshape(W, 3))
    r = _lib_next2().orc_accept(_dp(_f64(fn.L)), float(fn.r_cut), int(fn.m), _dp(_f64(fn.coef)),
                                W, n, n_up, Np, _dp(R2), _dp(S2),
                                k.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _dp(rn),
                                a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _dp(ab))
    if r:
        raise CoincidentError(f"walker {r - 1} has a coincident pair")
    return R2, S2, ab


def propose_f32(L, r, delta) -> np.ndarray:
    """Oracle of the in-kernel proposal r' = wrap(r + delta) in fp32
    (orc_propose_f32; Alg. 1 L5 without drift, reading R24).  r, delta [n][3]."""
    r = np.ascontiguousarray(np.asarray(r, dtype=np.float32).reshape(-1, 3))
    d = np.ascontiguousarray(np.asarray(delta, dtype=np.float32).reshape(-1, 3))
    out = np.empty_like(r)
    Lb = lib()
    Lb.orc_propose_f32.restype = None
    Lb.orc_propose_f32.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p]
    Lb.orc_propose_f32(_dp(_f64(np.broadcast_to(np.asarray(L, dtype=np.float64), (3,)))), r.shape[0],
                       r.ctypes.data_as(ctypes.c_void_p), d.ctypes.data_as(ctypes.c_void_p),
                       out.ctypes.data_as(ctypes.c_void_p))
    return out


def sweep(R, state, ks, delta, u, fn, n: int, n_up: int, *, forced=None, j1=None, threads: int = 1):
    """Oracle of qj2_sweep (orc_sweep): S ordered particle-by-particle moves per
    walker with the ratio from the stored state.

    R [W][3][Np] fp32 (copied), state [W][5][Np] (promoted to fp64, copied),
    ks [S][W], delta [S][W][3] fp32, u [S][W] fp64, forced [S][W] int (decisions
    to apply; None = the oracle's own), j1 = (ions [3][Np_ion], species_start,
    fn1, state_j1 [W][5][Np]) or None.
    Returns (R', state', acc [S][W] (the oracle's own decisions, -1 for an
    invalid k), dj [S][W], state_j1' or None)."""
    R2 = np.ascontiguousarray(np.asarray(R, dtype=np.float32)).copy()
    S2 = _f64(state).copy()
    W, _, Np = R2.shape
    ks = np.ascontiguousarray(np.asarray(ks, dtype=np.int32))
    S = ks.shape[0]
    dl = np.ascontiguousarray(np.asarray(delta, dtype=np.float32).reshape(S, W, 3))
    uu = _f64(np.asarray(u).reshape(S, W))
    fc = None if forced is None else np.ascontiguousarray(np.asarray(forced, dtype=np.int32).reshape(S, W))
    acc = np.zeros((S, W), dtype=np.int32)
    dj = np.zeros((S, W))
    i32p = ctypes.POINTER(ctypes.c_int32)
    dp = ctypes.POINTER(ctypes.c_double)
    Lb = lib()
    Lb.orc_sweep.restype = ctypes.c_int64
    Lb.orc_sweep.argtypes = [dp, ctypes.c_double, ctypes.c_int, dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                             ctypes.c_int64, ctypes.c_void_p, dp, ctypes.c_int64, i32p, ctypes.c_void_p, dp, i32p,
                             i32p, dp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), dp, ctypes.POINTER(ctypes.c_int),
                             dp, ctypes.c_int, ctypes.c_int64, dp, dp, ctypes.c_int]
    keep = []
    if j1 is not None:
        ions, start, fn1, sj1 = j1
        ions = _f64(ions)
        st = np.ascontiguousarray(np.asarray(start, dtype=np.int64))
        rc = _f64(fn1.r_cut)
        mm = np.ascontiguousarray(np.asarray(fn1.m, dtype=np.int32))
        c1 = _f64(fn1.coef)
        S1 = _f64(sj1).copy()
        keep = [ions, st, rc, mm, c1, S1]
        j1args = (len(fn1.m), st.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(rc),
                  mm.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _dp(c1), c1.shape[1], ions.shape[1], _dp(ions),
                  _dp(S1))
    else:
        S1 = None
        j1args = (0, None, None, None, None, 0, 0, None, None)
    r = Lb.orc_sweep(_dp(_f64(fn.L)), float(fn.r_cut), int(fn.m), _dp(_f64(fn.coef)), W, n, n_up, Np,
                     R2.ctypes.data_as(ctypes.c_void_p), _dp(S2), S, ks.ctypes.data_as(i32p),
                     dl.ctypes.data_as(ctypes.c_void_p), _dp(uu), None if fc is None else fc.ctypes.data_as(i32p),
                     acc.ctypes.data_as(i32p), _dp(dj), *j1args, int(threads))
    del keep
    if r:
        raise CoincidentError(f"walker {r - 1} has a coincident pair")
    return R2, S2, acc, dj, S1


def normalized_error_state(gpu, orc, absst, fn) -> np.ndarray:
    """Parity metric for the 5N state (NEXT-2): per entry
    |s_gpu - s_orc| / max(A, F) with A the oracle's absolute-term bound and F
    the functor scale of normalized_error (rows V, Gx, Gy, Gz, L)."""
    cmax = float(np.max(np.abs(fn.coef)))
    delta = fn.r_cut / fn.m
    F = np.array([cmax, cmax / delta, cmax / delta, cmax / delta, cmax / delta ** 2])[:, None]
    return np.abs(np.asarray(gpu, dtype=np.float64) - orc) / np.maximum(np.nan_to_num(absst, nan=0.0), F)


def _lib_next4():
    L = lib()
    if not getattr(L, "_next4", False):
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        L.orc_spo_vgh.restype = None
        L.orc_spo_vgh.argtypes = [i64, i64, i64, i64, i64, ctypes.c_void_p, dp, dp, dp, dp, dp, dp]
        L.orc_det_ratio.restype = None
        L.orc_det_ratio.argtypes = [i64, dp, dp, dp, dp, dp, dp]
        L._next4 = True
    return L


def spo_vgh(table, n_orb: int, L, pos):
    """NEXT-4 oracle of the tricubic B-spline SPOs (orc_spo_vgh).
    table: fp32 [nx][ny][nz][ld]; pos [M][3].  Returns v [M][n_orb],
    g [M][3][n_orb], h [M][6][n_orb] (xx, xy, xz, yy, yz, zz) and abs
    [M][10][n_orb], fp64."""
    T = np.ascontiguousarray(np.asarray(table, dtype=np.float32))
    nx, ny, nz, ld = T.shape
    pos = _f64(np.atleast_2d(pos))
    M = pos.shape[0]
    v = np.zeros((M, n_orb)); g = np.zeros((M, 3, n_orb)); h = np.zeros((M, 6, n_orb))
    ab = np.zeros((M, 10, n_orb))
    Lv = _f64(np.broadcast_to(np.asarray(L, dtype=np.float64), (3,)))
    lb = _lib_next4()
    for m in range(M):
        vm, gm, hm, am = v[m], g[m], h[m], ab[m]
        lb.orc_spo_vgh(nx, ny, nz, n_orb, ld, T.ctypes.data_as(ctypes.c_void_p), _dp(Lv),
                       _dp(np.ascontiguousarray(pos[m])), _dp(vm), _dp(gm), _dp(hm), _dp(am))
    return v, g, h, ab


def det_ratio(Ainv_rows, v, g, h):
    """NEXT-4 oracle of the determinant ratio (orc_det_ratio): per row m,
    (rho, G, L) = (sum a.phi, sum a.grad phi / rho, sum a.lap phi / rho) and the
    absolute-term sums.  Ainv_rows [M][n], v [M][n], g [M][3][n], h [M][6][n]."""
    A = _f64(np.atleast_2d(Ainv_rows))
    M, n = A.shape
    out = np.zeros((M, 5)); ab = np.zeros((M, 5))
    lb = _lib_next4()
    for m in range(M):
        lb.orc_det_ratio(n, _dp(np.ascontiguousarray(A[m])), _dp(_f64(v[m])), _dp(_f64(g[m])),
                         _dp(_f64(h[m])), _dp(out[m]), _dp(ab[m]))
    return out, ab


def det_ratio_scale(Ainv_rows, ab_vgh, F):
    """Parity scale of the determinant-ratio numerators (rho, rho G, rho L) in the
    form of DESIGN.md section 4, max(A_s, F_s) per term: sum_o |a_o| max(ab_o, F)
    with ab_vgh [M][10][n] the SPO absolute-term sums (spo_vgh) and F [10] the
    table scale per component (value, 3 gradient, 6 Hessian lanes).  Without the
    F floor a near-zero sum of |a . grad phi| (few orbitals) would leave no room
    for the fp32 rounding of grad phi itself."""
    A = np.abs(_f64(np.atleast_2d(Ainv_rows)))
    m = np.maximum(_f64(ab_vgh), np.asarray(F, dtype=np.float64)[None, :, None])
    out = np.empty((A.shape[0], 5))
    out[:, 0] = (A * m[:, 0]).sum(-1)
    out[:, 1:4] = (A[:, None, :] * m[:, 1:4]).sum(-1)
    out[:, 4] = (A * (m[:, 4] + m[:, 7] + m[:, 9])).sum(-1)
    return out


def gen_spo_table(seed: int, nx: int, ny: int, nz: int, n_orb: int, ld: int | None = None,
                  threads: int = 1) -> np.ndarray:
    """Oracle-side C twin of qmcgen.spo_table (input generation only)."""
    ld = n_orb if ld is None else ld
    L = lib()
    L.orc_gen_spo_table.restype = None
    L.orc_gen_spo_table.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
    out = np.empty((nx, ny, nz, ld), dtype=np.float32)
    L.orc_gen_spo_table(int(seed) & 0xFFFFFFFFFFFFFFFF, nx, ny, nz, n_orb, ld,
                        out.ctypes.data_as(ctypes.c_void_p), int(threads))
    return out
