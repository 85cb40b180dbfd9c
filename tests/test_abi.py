"""C-ABI library: loads on CPU and exports every symbol include/qmcj2.h
declares; host-side validation paths that return before any CUDA call.
No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "qmcj2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(qj2\w*)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def q():
    from paper_1708_02645_b200 import _build
    _build.build()
    import paper_1708_02645_b200 as q
    return q


def test_header_symbols_exported(q):
    lib = ctypes.CDLL(q.lib_path())
    names = _declared_symbols()
    assert len(names) >= 14, names
    for n in names:
        assert hasattr(lib, n), f"{n} declared in qmcj2.h but not exported"
    assert set(names) == set(q.EXPORTS)


def test_version_and_status_strings(q):
    assert q.version() == 20000
    lib = q._lib
    assert lib.qj2_status_string(0) == b"ok"
    assert lib.qj2_status_string(1) == b"invalid-argument"
    assert lib.qj2_status_string(2) == b"out-of-range"


def test_padded_size_examples(q):
    # SPEC:38-40
    assert q.padded_size(5, 8) == 8
    assert q.padded_size(16, 8) == 16
    assert q.padded_size(768, 16) == 768
    assert q.padded_size(0, 32) == 32
    with pytest.raises(q.QJ2Error) as ei:
        q.padded_size(5, 0)
    assert ei.value.status == 1


def _functor(q, **kw):
    import qmcgen
    fn = qmcgen.make_functor(0, 10.0)
    f = q.Functor(fn.L, fn.r_cut, fn.m, fn.coef)
    for a, v in kw.items():
        setattr(f._c, a, v)
    return f


def _call_eval(q, f, **over):
    args = dict(dtype=0, W=4, N_total=100, N_up=50, i_offset=0, N_local=100, Np=128,
                R=ctypes.c_void_p(4096), k=ctypes.c_void_p(4096), P=1, rt=ctypes.c_void_p(4096),
                out=ctypes.c_void_p(4096), row=None, vcur=None, ratio=None, ws=ctypes.c_void_p(4096),
                wsb=1 << 30)
    args.update(over)
    st = q._lib.qj2_eval(f.ptr, args["dtype"], args["W"], args["N_total"], args["N_up"], args["i_offset"],
                         args["N_local"], args["Np"], args["R"], args["k"], args["P"], args["rt"],
                         args["out"], args["row"], args["vcur"], args["ratio"], args["ws"], args["wsb"], None)
    return st, q._lib.qj2_last_error().decode()


def test_eval_host_validation(q):
    f = _functor(q)
    assert _call_eval(q, f, N_total=1)[0] == 1
    assert _call_eval(q, f, N_up=101)[0] == 2
    assert _call_eval(q, f, i_offset=50, N_local=60)[0] == 2
    assert _call_eval(q, f, Np=99)[0] == 1           # not a multiple of 4
    assert _call_eval(q, f, Np=64)[0] == 1           # Np < N_local
    assert _call_eval(q, f, P=0)[0] == 1
    assert _call_eval(q, f, dtype=7)[0] == 1
    assert _call_eval(q, f, R=None)[0] == 1
    assert _call_eval(q, f, R=ctypes.c_void_p(4100))[0] == 1     # misaligned
    assert _call_eval(q, f, i_offset=10, N_local=20, ratio=ctypes.c_void_p(4096))[0] == 1
    # any P may fuse the ratio relative to trial 0 (a second launch when P > 1): passes validation
    assert _call_eval(q, f, P=8, ratio=ctypes.c_void_p(4096))[0] != 1
    assert _call_eval(q, f, W=0) == (0, _call_eval(q, f, W=0)[1])      # no-op
    st, msg = _call_eval(q, f, N_local=1 << 20, Np=1 << 20, N_total=1 << 20, wsb=16)
    assert st == 1 and "workspace" in msg


def test_functor_validation(q):
    assert _call_eval(q, _functor(q, m=3))[0] == 1
    assert _call_eval(q, _functor(q, m=65))[0] == 1
    assert _call_eval(q, _functor(q, r_cut=5.01))[0] == 1       # > L/2
    f = _functor(q)
    f._c.coef[0][f.m] = 0.5                                     # tail must be zero
    assert _call_eval(q, f)[0] == 1
    assert _call_eval(q, _functor(q, reserved=1))[0] == 1


def test_workspace_size(q):
    import torch
    assert q.workspace_size(1024, 1, 1400, torch.float32) == 0            # one tile per walker
    b = q.workspace_size(1024, 1, 614400, torch.float32)
    assert b >= 1024 * 3 * 6 * 8 + 1024 * 4                            # 3 tiles of 204800 sources, 6 fp64 partials
    assert q.workspace_size(8, 3, 40000, torch.float64) == 0            # fp64 tiles hold 102400 sources
    assert q.workspace_size(8, 3, 102401, torch.float64) > 0


def test_package_has_no_cpu_fallback():
    """The product package must not import the oracle (no CPU path)."""
    pkg = os.path.join(ROOT, "paper_1708_02645_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, fn
                assert "liboracle" not in txt, fn


def test_no_runtime_switches_in_the_product():
    """Kernel variants are chosen from the arguments alone: no source of the
    library reads the environment (the measured alternatives are compile-time
    A/B builds, tools/ab), and the binding reads only QJ2_LIB (which library
    file to load)."""
    import re
    csrc = os.path.join(ROOT, "paper_1708_02645_b200", "csrc")
    for fn in os.listdir(csrc):
        if fn.endswith((".cu", ".cuh", ".h", ".cpp")):
            assert "getenv" not in open(os.path.join(csrc, fn)).read(), fn
    txt = open(os.path.join(ROOT, "paper_1708_02645_b200", "__init__.py")).read()
    assert set(re.findall(r"environ(?:\.get)?\(?\[?[\"']([A-Z0-9_]+)", txt)) <= {"QJ2_LIB"}


def test_oracle_is_independent_of_the_product():
    """The oracle imports nothing from the product package, includes none of its
    headers, and the product's binding, kernels and bench timing path never
    load it (bench.py only in its cpu_baseline / --impl reference legs)."""
    import re
    odir = os.path.join(ROOT, "oracle")
    for fn in os.listdir(odir):
        txt = open(os.path.join(odir, fn)).read() if fn.endswith((".py", ".c", ".h")) else ""
        if fn.endswith(".py"):      # its imports: stdlib and numpy only
            mods = re.findall(r"^\s*(?:from|import)\s+([\w.]+)", txt, re.M)
            assert set(mods) <= {"__future__", "ctypes", "os", "subprocess", "numpy"}, (fn, mods)
        elif txt:                   # its includes: the C library only
            incs = re.findall(r'#include\s*[<"]([^>"]+)[>"]', txt)
            assert set(incs) <= {"math.h", "stdint.h", "stdlib.h", "string.h", "pthread.h"}, (fn, incs)
    txt = open(os.path.join(ROOT, "qmcgen", "__init__.py")).read()   # the shared input generator
    mods = re.findall(r"^\s*(?:from|import)\s+([\w.]+)", txt, re.M)
    assert not any(m.startswith(("oracle", "paper_1708_02645_b200")) for m in mods), mods


def _call_accept(q, f, **over):
    P = ctypes.c_void_p(4096)
    args = dict(dtype=0, W=4, N_total=100, N_up=50, i_offset=0, N_local=100, Np=128, R=P, S=P, k=P, rn=P,
                rs=3, ro=None, acc=P, out=P, os=5, ws=P, wsb=1 << 20)
    args.update(over)
    st = q._lib.qj2_accept(f.ptr, args["dtype"], args["W"], args["N_total"], args["N_up"], args["i_offset"],
                           args["N_local"], args["Np"], args["R"], args["S"], args["k"], args["rn"], args["rs"],
                           args["ro"], args["acc"], args["out"], args["os"], args["ws"], args["wsb"], None)
    return st, q._lib.qj2_last_error().decode()


def test_accept_host_validation(q):
    """qj2_accept (NEXT-2): argument checks that return before any CUDA call."""
    f = _functor(q)
    assert _call_accept(q, f, N_total=1)[0] == 1
    assert _call_accept(q, f, N_up=101)[0] == 2
    assert _call_accept(q, f, i_offset=50, N_local=60)[0] == 2
    assert _call_accept(q, f, Np=99)[0] == 1
    assert _call_accept(q, f, os=4)[0] == 1                   # out_stride < 5
    assert _call_accept(q, f, rs=2)[0] == 1                   # r_stride < 3
    assert _call_accept(q, f, S=None)[0] == 1
    assert _call_accept(q, f, acc=None)[0] == 1
    assert _call_accept(q, f, S=ctypes.c_void_p(4104))[0] == 1     # misaligned state
    st, msg = _call_accept(q, f, ws=None, wsb=0)
    assert st == 1 and "workspace" in msg                     # r_old NULL needs the gather workspace
    assert _call_accept(q, f, W=0)[0] == 0
    assert _call_accept(q, _functor(q, m=3))[0] == 1
    b = ctypes.c_size_t()
    assert q._lib.qj2_accept_workspace_size(1024, 0, ctypes.byref(b)) == 0 and b.value >= 1024 * 12


def test_metropolis_accept_host_validation(q):
    f = _functor(q)
    P = ctypes.c_void_p(4096)

    def call(**over):
        a = dict(W=4, N_total=100, N_up=50, i_offset=0, N_local=100, Np=128, R=P, S=P, k=P, rn=P, ro=P, rs=6,
                 on=P, vr=P, os=10, vrs=10, u=P, acc=P)
        a.update(over)
        return q._lib.qj2_metropolis_accept(f.ptr, 0, a["W"], a["N_total"], a["N_up"], a["i_offset"], a["N_local"],
                                            a["Np"], a["R"], a["S"], a["k"], a["rn"], a["ro"], a["rs"], a["on"],
                                            a["vr"], a["os"], a["vrs"], a["u"], a["acc"], None)
    assert call(ro=None) == 1                     # r_old is required (no gather in the fused path)
    assert call(u=None) == 1
    assert call(rs=2) == 1
    assert call(vrs=0) == 1
    assert call(N_up=101) == 2
    assert call(W=0) == 0


def test_sweep_host_validation(q):
    f = _functor(q)
    P = ctypes.c_void_p(4096)

    def call(fn=f, W=4, N=100, N_up=50, Np=128, S=3):
        return q._lib.qj2_sweep(fn.ptr, W, N, N_up, Np, P, P, S, P, P, P, P, None, None, None)
    assert call(N=1025, Np=1056) == 1            # walker must fit shared memory
    assert call(N=1) == 1
    assert call(Np=64) == 1
    assert call(N_up=101) == 2
    assert call(fn=_functor(q, m=17)) == 1       # fp32 pair terms: m <= 16
    assert call(S=0) == 0 and call(W=0) == 0
    assert call(S=-1) == 1


def test_state_init_host_validation(q):
    f = _functor(q)
    P = ctypes.c_void_p(4096)

    def call(fn=f, W=4, N=100, N_up=50, Np=128):
        return q._lib.qj2_state_init(fn.ptr, W, N, N_up, Np, P, P, None, None)
    assert call(N=1025, Np=1056) == 1
    assert call(N=1) == 1
    assert call(Np=64) == 1
    assert call(N_up=-1) == 2
    assert call(fn=_functor(q, m=17)) == 1
    assert call(W=0) == 0


def test_metropolis_and_spo_host_validation(q):
    P = ctypes.c_void_p(4096)
    lib = q._lib
    assert lib.qj2_metropolis(-1, P, 2, P, P, None) == 1
    assert lib.qj2_metropolis(4, P, 1, P, P, None) == 1         # ratio_stride < 2
    assert lib.qj2_metropolis(4, None, 2, P, P, None) == 1
    assert lib.qj2_metropolis(0, None, 2, None, None, None) == 0

    def tab(**kw):
        t = q._SpoTable()
        for d in range(3):
            t.L[d] = 3.0
        t.nx = t.ny = t.nz = 8
        t.n_orb, t.ld, t.coef = 10, 12, 4096
        for a, v in kw.items():
            setattr(t, a, v)
        return t

    def spo(t, what=1, dt=0, W=5, pos=P, ps=3, ainv=P, out=P, spo_out=None, ppw=1):
        return lib.qj2_spo_eval(ctypes.byref(t), what, dt, W, pos, ps, ainv, 12, 12, None, ppw, out, spo_out, None)

    assert spo(tab(), what=2) == 1
    assert spo(tab(), dt=5) == 1
    assert spo(tab(nx=3)) == 1                                  # grid >= 4
    assert spo(tab(ld=10)) == 1                                 # ld % 4
    assert spo(tab(ld=8)) == 1                                  # ld < n_orb
    assert spo(tab(nx=1024, ny=1024, nz=1024)) == 1             # >= 2^31 floats
    assert spo(tab(), ps=2) == 1
    assert spo(tab(coef=4100)) == 1                             # misaligned table
    assert spo(tab(), pos=None) == 1
    assert spo(tab(), W=0) == 0
    assert spo(tab(), ppw=0) == 1
    L = tab()
    L.L[1] = 0.0
    assert spo(L) == 1
