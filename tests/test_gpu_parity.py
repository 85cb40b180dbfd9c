"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element on the same seeded inputs (-m gpu; needs a B200).

Tolerance: per output component
|s_gpu - s_orc| / max(A_s, F_s) <= 1e-5 (fp32 path) or 1e-12 (fp64 path),
A_s the oracle's absolute-term sum, F_s the functor scale.  Row output:
dx, dy, dz bit-exact in fp32 (except exact |d| = L/2 ties), r within 3 ulp.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import qmcgen

pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}
THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def q():
    import paper_1708_02645_b200 as q
    assert torch.cuda.is_available()
    q.device_check()
    return q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def instance(N, W, seed, dtype, P=1, mode="move", Np=None, m=8, n_up=None):
    L = qmcgen.cell_length(N)
    vw = 4 if dtype == np.float32 else 2
    Np = Np or qmcgen.padded_size(N, vw)
    walkers = np.arange(W)
    R = qmcgen.positions(seed, walkers, N, Np, L, dtype)
    k = qmcgen.make_k(seed, W, N) if W else np.zeros(0, np.int32)
    rt = (qmcgen.make_trials(seed, walkers, k, N, L, dtype, P=P, mode=mode) if W
          else np.zeros((0, P, 3), dtype))
    fn = qmcgen.make_functor(seed, L, m)
    return R, k, rt, fn, (N // 2 if n_up is None else n_up)


def check(q, R, k, rt, fn, N, n_up, dtype, i_offset=0, n_local=None, row=False):
    res = q.eval(dev(R), dev(k), dev(rt), fn, N, n_up, i_offset=i_offset, n_local=n_local, row=row)
    torch.cuda.synchronize()
    out = (res[0] if row else res).cpu().numpy()
    orc, absout, orow = oracle.eval_j2(R, k, rt, fn, N, n_up, i_offset=i_offset, n_local=n_local,
                                       row=row, threads=THREADS)
    err = oracle.normalized_error(out, orc, absout, fn)
    assert np.all(np.isfinite(out))
    assert err.max() <= TOL[dtype], f"max normalized error {err.max():.3e}"
    print(f"N={N} {np.dtype(dtype).name}: normalized {err.max():.2e}, plain relative (V, Gx, Gy, Gz, L) "
          f"{oracle.plain_relative_error(out, orc, absout)}")
    if row:
        return out, orc, res[1].cpu().numpy(), orow
    return out, orc


# ---------------------------------------------------------------------------
# Configs C1, C2 (fp32 and fp64) in full
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["C1", "C2", "C2f64"])
def test_config_full(q, name):
    cfg = qmcgen.CONFIGS[name]
    R, k, rt, fn = qmcgen.host_instance(cfg)
    check(q, R, k, rt, fn, cfg.N, cfg.n_up, cfg.np_dtype)


# ---------------------------------------------------------------------------
# Edge cases: tiny / ragged / tile boundaries / spin boundary / P groups
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("N", [2, 3, 5, 17, 1023, 2048, 2049, 4095, 4096, 4097, 8191, 8192, 8193, 20001, 32769, 70001,
                               102401, 204801])   # and both sides of the mapping / tile boundaries
def test_ragged_sizes(q, dtype, N):
    R, k, rt, fn, n_up = instance(N, 37, seed=100 + N, dtype=dtype)
    check(q, R, k, rt, fn, N, n_up, dtype)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_k_at_tile_and_spin_boundaries(q, dtype):
    # sub-tiles of 8192 (fp32) / 4096 (fp64) sources, CTA tiles of 25 sub-tiles (204800 / 102400)
    N = 2 * 204800 + 77
    ks = np.array([0, 1, 4095, 4096, 8191, 8192, 8193, 16383, 102399, 102400, 102401, 204799, 204800,
                   204801, 307199, 307200, 409599, 409600, N - 2, N - 1, N // 2], np.int32)
    W = ks.size
    R, k, rt, fn, _ = instance(N, W, seed=7, dtype=dtype)
    L = qmcgen.cell_length(N)
    rt = qmcgen.make_trials(7, np.arange(W), ks, N, L, dtype)
    for n_up in (N // 2, 204800, 102400, 8192, 8190, 0, N, 1):   # spin boundary inside / on a tile edge / degenerate
        check(q, R, ks, rt, fn, N, n_up, dtype)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("P", [2, 3, 4, 5, 9])
def test_multi_trial(q, dtype, P):
    R, k, rt, fn, n_up = instance(9000, 9, seed=200 + P, dtype=dtype, P=P)
    check(q, R, k, rt, fn, 9000, n_up, dtype)


def test_empty_batch(q):
    R, k, rt, fn, n_up = instance(100, 0, seed=1, dtype=np.float32)
    out = q.eval(dev(R), dev(k), dev(rt), fn, 100, n_up)
    assert out.shape == (0, 1, 5)


def test_single_walker_and_larger_m(q):
    for m in (4, 13, 64):
        R, k, rt, fn, n_up = instance(4000, 1, seed=300 + m, dtype=np.float32, m=m)
        check(q, R, k, rt, fn, 4000, n_up, np.float32)


@pytest.mark.parametrize("m", [17, 36, 64])
def test_fine_functors_fp32(q, m):
    """fp32 functors finer than m = 16 take the fp64 geometry:
    the 1e-5 bar holds where one or two terms make the whole sum (tiny N: the
    short-row warp kernel), in the compact warp kernel (long rows, many walkers),
    in the CTA kernel (one and several tiles per walker), and the row output keeps
    the fp32 single-rounding displacements bitwise."""
    for N, W in ((2, 512), (4, 512), (8, 256), (4100, 4096), (5000, 64), (300000, 2)):
        R, k, rt, fn, n_up = instance(N, W, seed=400 + m + N, dtype=np.float32, m=m)
        check(q, R, k, rt, fn, N, n_up, np.float32)
    N = 3000
    R, k, rt, fn, n_up = instance(N, 8, seed=450 + m, dtype=np.float32, m=m)
    out, orc, row, orow = check(q, R, k, rt, fn, N, n_up, np.float32, row=True)
    L = np.float64(fn.L[0])
    for w in range(8):
        i = np.array([j for j in range(N) if j != k[w]])
        d_gpu = row[w, 0, 1:, i].astype(np.float64)
        d_orc = orow[w, 0, 1:, i]
        tie = np.abs(np.abs(d_orc) - L / 2) <= 4 * np.spacing(np.float32(L))
        assert ((d_gpu == d_orc.astype(np.float32)) | tie).all()
        rg, ro = row[w, 0, 0, i], orow[w, 0, 0, i].astype(np.float32)
        assert np.all(np.abs(rg - ro) <= 3 * np.spacing(ro))


def test_noop_move_ratio_exactly_one(q):
    """P = 2 with r_trial[0] == r_trial[1] (no-op move): dJ2 = 0 bitwise,
    ratio 1."""
    for dtype in (np.float32, np.float64):
        R, k, rt, fn, n_up = instance(30000, 16, seed=11, dtype=dtype, P=2, mode="noop")
        out, ratio = q.eval(dev(R), dev(k), dev(rt), fn, 30000, n_up, ratio=True)
        ratio = ratio.cpu().numpy()
        assert np.all(ratio[:, :, 0] == 0.0) and np.all(ratio[:, :, 1] == 1.0)


def test_ratio_against_oracle_delta_j2(q):
    """P = 2 drift variant: dJ2 = V(r'_k) - V(r_k) (Eq. 5) and exp(dJ2) (Eq. 4)."""
    R, k, rt, fn, n_up = instance(20000, 32, seed=12, dtype=np.float64, P=2, mode="drift")
    out, ratio = q.eval(dev(R), dev(k), dev(rt), fn, 20000, n_up, ratio=True)
    orc, absout, _ = oracle.eval_j2(R, k, rt, fn, 20000, n_up, threads=THREADS)
    dj = orc[:, 1, 0] - orc[:, 0, 0]
    r = ratio.cpu().numpy()
    scale = np.maximum(absout[:, :, 0].max(1), 1.0)
    assert np.max(np.abs(r[:, 1, 0] - dj) / scale) < 1e-12
    np.testing.assert_allclose(r[:, 1, 1], np.exp(dj), rtol=1e-11)
    # V_cur variant and the standalone qj2_ratio kernel agree
    vcur = dev(out[:, 0, 0].cpu().numpy().copy())
    _, r2 = q.eval(dev(R), dev(k), dev(rt), fn, 20000, n_up, V_cur=vcur, ratio=True)
    r3 = q.ratio(out, V_cur=vcur)
    assert torch.equal(r2, r3)


def test_determinism(q):
    R, k, rt, fn, n_up = instance(50000, 64, seed=13, dtype=np.float32)
    a = q.eval(dev(R), dev(k), dev(rt), fn, 50000, n_up)
    b = q.eval(dev(R), dev(k), dev(rt), fn, 50000, n_up)
    assert torch.equal(a, b)


# ---------------------------------------------------------------------------
# Row output (Fig. 6's v)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_row_output(q, dtype):
    N = 9001
    R, k, rt, fn, n_up = instance(N, 8, seed=21, dtype=dtype, P=2)
    out, orc, row, orow = check(q, R, k, rt, fn, N, n_up, dtype, row=True)
    L = np.float64(fn.L[0])
    for w in range(8):
        for p in range(2):
            i = np.array([j for j in range(N) if j != k[w]])
            d_gpu = row[w, p, 1:, i].astype(np.float64)
            d_orc = orow[w, p, 1:, i]
            tie = np.abs(np.abs(d_orc) - L / 2) <= 4 * np.spacing(np.float32(L))
            if dtype == np.float32:
                ok = (d_gpu == d_orc.astype(np.float32)) | tie
                assert ok.all()
                rg, ro = row[w, p, 0, i], orow[w, p, 0, i].astype(np.float32)
                assert np.all(np.abs(rg - ro) <= 3 * np.spacing(ro))
            else:
                assert np.all((np.abs(d_gpu - d_orc) <= 2 * np.spacing(L)) | tie)
                # the fp64 oracle wraps with two roundings (|err| <= ulp(L)); the kernel rounds once
                assert np.all(np.abs(row[w, p, 0, i] - orow[w, p, 0, i]) <= 4 * np.spacing(L))


# ---------------------------------------------------------------------------
# Sharding along the electron axis (the per-rank path of C5)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_fake_shard_partial_sums(q, dtype):
    N, W = 40000, 24
    R, k, rt, fn, n_up = instance(N, W, seed=31, dtype=dtype)
    full = q.eval(dev(R), dev(k), dev(rt), fn, N, n_up).cpu().numpy()
    orc, absout, _ = oracle.eval_j2(R, k, rt, fn, N, n_up, threads=THREADS)
    for G in (2, 3, 8):
        tot = np.zeros_like(full)
        bounds = [N * g // G for g in range(G + 1)]
        for a, b in zip(bounds[:-1], bounds[1:]):
            vw = 4 if dtype == np.float32 else 2
            Np = qmcgen.padded_size(b - a, vw)
            Rs = np.zeros((W, 3, Np), dtype)
            Rs[:, :, :b - a] = R[:, :, a:b]
            part = q.eval(dev(Rs), dev(k), dev(rt), fn, N, n_up, i_offset=a, n_local=b - a)
            tot += part.cpu().numpy()
        assert oracle.normalized_error(tot, orc, absout, fn).max() <= TOL[dtype]
        assert oracle.normalized_error(tot, full, absout, fn).max() <= TOL[dtype]


# ---------------------------------------------------------------------------
# Building blocks
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_functor_eval_vgl(q, dtype):
    fn = qmcgen.make_functor(5, 20.0, m=8)
    r = (np.random.default_rng(0).random(100000) * 12.0).astype(dtype)
    for ch in (0, 1):
        g = q.functor_eval_vgl(fn, ch, dev(r)).cpu().numpy()
        o = oracle.bspline(fn.coef[ch], fn.m, fn.r_cut, r.astype(np.float64))
        cmax, delta = np.abs(fn.coef).max(), fn.r_cut / fn.m
        tol = 4e-6 if dtype == np.float32 else 1e-13
        # compare away from the cutoff (fp32 r/delta may round across r_cut)
        inside = r.astype(np.float64) < fn.r_cut * (1 - 1e-6)
        for nu in range(3):
            assert np.max(np.abs(g[inside, nu] - o[inside, nu])) <= tol * cmax / delta ** nu
        assert np.all(g[r.astype(np.float64) >= fn.r_cut] == 0.0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_min_image_disp(q, dtype):
    rng = np.random.default_rng(1)
    L = np.float32(17.5)
    a = (rng.random((50000, 3)) * L).astype(dtype)
    b = (rng.random((50000, 3)) * L).astype(dtype)
    g = q.min_image_disp([float(L)] * 3, dev(a), dev(b)).cpu().numpy()
    o = oracle.min_image([float(L)] * 3, a, b)
    if dtype == np.float32:
        assert np.array_equal(g[:, 1:], o[:, 1:].astype(np.float32))   # single rounding
        assert np.all(np.abs(g[:, 0] - o[:, 0]) <= 3 * np.spacing(o[:, 0].astype(np.float32)))
    else:
        np.testing.assert_allclose(g[:, 1:], o[:, 1:], atol=4 * np.spacing(17.5))
        assert np.all(np.abs(g[:, 0] - o[:, 0]) <= 4 * np.spacing(17.5))   # oracle wraps with 2 roundings


def test_check_inputs_flags(q):
    R, k, rt, fn, n_up = instance(1000, 4, seed=3, dtype=np.float32)
    assert q.check_inputs(dev(R), dev(k), dev(rt), fn, 1000) == 0
    R2 = R.copy(); R2[1, 2, 5] = np.float32(fn.L[0])
    k2 = k.copy(); k2[3] = 1000
    rt2 = rt.copy(); rt2[0, 0, 1] = -1.0
    assert q.check_inputs(dev(R2), dev(k), dev(rt), fn, 1000) == 1
    assert q.check_inputs(dev(R), dev(k2), dev(rt), fn, 1000) == 2
    assert q.check_inputs(dev(R), dev(k), dev(rt2), fn, 1000) == 4


def test_device_generator_matches_host_generator(q):
    for dtype, tdt in ((np.float32, torch.float32), (np.float64, torch.float64)):
        N, Np, L = 5000, 5008, qmcgen.cell_length(5000)
        g = q.gen_positions(42, 6, N, Np, L, tdt, w_offset=100).cpu().numpy()
        h = qmcgen.positions(42, np.arange(100, 106), N, Np, L, dtype)
        assert np.array_equal(g, h)
        # a slice of the source axis (C5 per-rank generation)
        g2 = q.gen_positions(42, 2, 1000, 1000, L, tdt, w_offset=100, i_offset=3000).cpu().numpy()
        assert np.array_equal(g2, h[:2, :, 3000:4000])


def test_eval_host_matches_device_path(q):
    R, k, rt, fn, n_up = instance(30000, 40, seed=41, dtype=np.float32)
    d = q.eval(dev(R), dev(k), dev(rt), fn, 30000, n_up).cpu()
    Rh = torch.from_numpy(R).pin_memory()
    kh = torch.from_numpy(k).pin_memory()
    th = torch.from_numpy(rt).pin_memory()
    h = q.eval_host(Rh, kh, th, fn, 30000, n_up, chunk_walkers=7)
    assert torch.equal(d, h)
    vcur = torch.from_numpy(d[:, 0, 0].numpy().copy())
    h2, rat = q.eval_host(Rh, kh, th, fn, 30000, n_up, V_cur=vcur, ratio=True, chunk_walkers=16)
    assert torch.equal(h2, d)
    assert torch.all(rat[:, 0, 0] == 0) and torch.all(rat[:, 0, 1] == 1)


# ---------------------------------------------------------------------------
# Full-size configs in the launch configuration bench.py times (sampled)
# ---------------------------------------------------------------------------
def _sampled_check(q, cfg, seed, Rdev, walkers_sample, n_local=None, i_offset=0, out=None):
    L = cfg.L
    k = qmcgen.make_k(seed, cfg.W, cfg.N)
    rt = qmcgen.make_trials(seed, np.arange(cfg.W), k, cfg.N, L, cfg.np_dtype)
    fn = qmcgen.make_functor(cfg.seed, L, cfg.m)
    if out is None:
        out = q.eval(Rdev, dev(k), dev(rt), fn, cfg.N, cfg.n_up).cpu().numpy()
    assert np.all(np.isfinite(out))
    Rs = qmcgen.positions(seed, walkers_sample, cfg.N, cfg.Np, L, cfg.np_dtype)
    orc, absout, _ = oracle.eval_j2(Rs, k[walkers_sample], rt[walkers_sample], fn, cfg.N, cfg.n_up,
                                    threads=THREADS)
    err = oracle.normalized_error(out[walkers_sample], orc, absout, fn)
    assert err.max() <= TOL[cfg.np_dtype], err.max()
    return out


def test_C3_full_size_sampled(q):
    cfg = qmcgen.CONFIGS["C3"]
    R = q.gen_positions(cfg.seed, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32)
    sample = np.array([0, 1, 77, 511, 512, 1000, 1023])
    _sampled_check(q, cfg, cfg.seed, R, sample)
    del R
    torch.cuda.empty_cache()


def test_C3_full_size_every_walker(q):
    """The default bench workload in its launch configuration, every one of the 1024
    walkers against the oracle (the oracle's own C twin of the position generator
    builds the 7.55 GB host copy; ~2 s of oracle time on the box's cores)."""
    cfg = qmcgen.CONFIGS["C3"]
    R = q.gen_positions(cfg.seed, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32)
    k = qmcgen.make_k(cfg.seed, cfg.W, cfg.N)
    rt = qmcgen.make_trials(cfg.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32)
    fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
    out = q.eval(R, dev(k), dev(rt), fn, cfg.N, cfg.n_up).cpu().numpy()
    del R
    torch.cuda.empty_cache()
    Rh = oracle.gen_positions(cfg.seed, 0, cfg.W, cfg.N, cfg.Np, cfg.L, np.float32, threads=THREADS)
    orc, absout, _ = oracle.eval_j2(Rh, k, rt, fn, cfg.N, cfg.n_up, threads=THREADS)
    del Rh
    assert np.all(np.isfinite(out))
    err = oracle.normalized_error(out, orc, absout, fn)
    assert err.max() <= TOL[np.float32], err.max()
    # the plain relative error: fp32 per-term arithmetic (rounded functor table and 1/delta)
    # leaves a per-interval bias of ~1e-7 of the term scale that cancelling G sums do not average away,
    # so near |G| = 1e-3 A it reaches ~1e-4; V (all terms >= 0) stays at ~1e-7
    rel = oracle.plain_relative_error(out, orc, absout)
    print(f"C3 every walker: normalized {err.max():.2e}, plain relative (V, Gx, Gy, Gz, L) {rel}")
    assert rel[0] <= 1e-6 and max(rel[1:]) <= 1e-3


def test_C4_instances_every_walker(q):
    """Three of C4's 4096 instances (first, second, last) in the bench's launch
    configuration (warp-per-walker kernel), every walker vs the oracle."""
    cfg = qmcgen.CONFIGS["C4"]
    fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
    for inst in (0, 1, 4095):
        seed = cfg.seed + inst
        R = q.gen_positions(seed, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32)
        k = qmcgen.make_k(seed, cfg.W, cfg.N)
        rt = qmcgen.make_trials(seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32)
        out = q.eval(R, dev(k), dev(rt), fn, cfg.N, cfg.n_up).cpu().numpy()
        Rh = oracle.gen_positions(seed, 0, cfg.W, cfg.N, cfg.Np, cfg.L, np.float32, threads=THREADS)
        orc, absout, _ = oracle.eval_j2(Rh, k, rt, fn, cfg.N, cfg.n_up, threads=THREADS)
        assert np.all(np.isfinite(out))
        assert oracle.normalized_error(out, orc, absout, fn).max() <= TOL[np.float32], inst


@pytest.fixture(scope="module")
def c5_reference():
    """The oracle's C5 values for every 8th walker (and the last): the unsplit
    source sum over all N = 4,915,200 electrons (~1.6 s of oracle time; 7.6 GB of
    host positions from the oracle's own generator)."""
    cfg = qmcgen.CONFIGS["C5"]
    k = qmcgen.make_k(cfg.seed, cfg.W, cfg.N)
    rt = qmcgen.make_trials(cfg.seed, np.arange(cfg.W), k, cfg.N, cfg.L, cfg.np_dtype)
    fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
    ws = np.r_[0:cfg.W:8, cfg.W - 1]
    Rh = np.concatenate([oracle.gen_positions(cfg.seed, int(w), 1, cfg.N, cfg.Np, cfg.L, np.float32, threads=THREADS)
                         for w in ws])
    orc, absout, _ = oracle.eval_j2(Rh, k[ws], rt[ws], fn, cfg.N, cfg.n_up, threads=THREADS)
    # one rank's slice checked on its own as well: the oracle's partial sum over [a, b)
    a, b = cfg.N // 4, cfg.N // 2
    sub = ws[:17]
    po, pa, _ = oracle.eval_j2(Rh[:17, :, a:b], k[sub], rt[sub], fn, cfg.N, cfg.n_up, i_offset=a, n_local=b - a,
                               threads=THREADS)
    del Rh
    return dict(k=k, rt=rt, fn=fn, ws=ws, orc=orc, absout=absout, slice=(a, b, sub, po, pa))


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_C5_rank_slices_as_benched(q, c5_reference, G):
    """C5 (N = 4,915,200, W = 1024) split along the electron axis into G slices,
    each evaluated exactly as the rank of a G-GPU run calls it (qj2_eval with
    i_offset over a device-generated slice; G = 1 is one 60 GB launch with 24
    tiles per walker and 5e9 > 2^31 elements), partials summed on the host (the
    all-reduce); every 8th walker and the last vs the unsplit oracle sum, and the
    slice [N/4, N/2) of the G = 4 split vs the oracle's own partial sum."""
    cfg = qmcgen.CONFIGS["C5"]
    ref = c5_reference
    fn = ref["fn"]
    kd, td = dev(ref["k"]), dev(ref["rt"])
    tot = np.zeros((cfg.W, 1, 5))
    ws = q.Workspace()
    for g in range(G):
        a, b = cfg.N * g // G, cfg.N * (g + 1) // G
        Np = qmcgen.padded_size(b - a, 32)
        R = q.gen_positions(cfg.seed, cfg.W, b - a, Np, cfg.L, torch.float32, i_offset=a)
        part = q.eval(R, kd, td, fn, cfg.N, cfg.n_up, i_offset=a, n_local=b - a, workspace=ws).cpu().numpy()
        del R
        assert np.all(np.isfinite(part))
        tot += part
        sa, sb, sub, po, pa = ref["slice"]
        if (a, b) == (sa, sb):
            assert oracle.normalized_error(part[sub], po, pa, fn).max() <= TOL[np.float32]
    torch.cuda.empty_cache()
    err = oracle.normalized_error(tot[ref["ws"]], ref["orc"], ref["absout"], fn)
    assert err.max() <= TOL[np.float32], err.max()


def _c4_wave(q, cfg, first, count, fn):
    """One C4 wave as bench.py launches it: `count` instances (1024 walkers each)
    concatenated into ONE qj2_eval (warp-per-walker kernel); returns out, k, rt."""
    W = cfg.W
    R = torch.empty((count * W, 3, cfg.Np), dtype=torch.float32, device="cuda")
    ks, rts = [], []
    for j in range(count):
        seed = cfg.seed + first + j
        q.gen_positions(seed, W, cfg.N, cfg.Np, cfg.L, torch.float32, out=R[j * W:(j + 1) * W])
        k = qmcgen.make_k(seed, W, cfg.N)
        ks.append(k)
        rts.append(qmcgen.make_trials(seed, np.arange(W), k, cfg.N, cfg.L, np.float32))
    k, rt = np.concatenate(ks), np.concatenate(rts)
    out = q.eval(R, dev(k), dev(rt), fn, cfg.N, cfg.n_up).cpu().numpy()
    del R
    torch.cuda.empty_cache()
    return out, k, rt


def test_C4_full_wave_as_benched(q):
    """One full C4 wave exactly as benched: 1024 instances = 1,048,576 walkers
    (77 GB, 6.4e9 > 2^31 elements) in one qj2_eval; three walkers (first, last,
    a middle one) of each of 65 instances spread over the wave (every 16th and
    the last) vs the oracle."""
    cfg = qmcgen.CONFIGS["C4"]
    fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
    out, k, rt = _c4_wave(q, cfg, 0, 1024, fn)
    assert np.all(np.isfinite(out))
    for inst in list(range(0, 1024, 16)) + [1023]:
        seed = cfg.seed + inst
        for wl in (0, 1 + (inst * 37) % 1022, 1023):
            Rs = oracle.gen_positions(seed, wl, 1, cfg.N, cfg.Np, cfg.L, np.float32)
            g = inst * cfg.W + wl
            orc, absout, _ = oracle.eval_j2(Rs, k[g:g + 1], rt[g:g + 1], fn, cfg.N, cfg.n_up)
            assert oracle.normalized_error(out[g:g + 1], orc, absout, fn).max() <= TOL[np.float32], (inst, wl)


@pytest.mark.slow
def test_C4_all_instances_every_walker(q):
    """All 4096 C4 instances in the bench's four waves of 1024, every walker of
    every instance vs the oracle (every config checked in full;
    ~2 min of oracle time on the box's cores)."""
    cfg = qmcgen.CONFIGS["C4"]
    fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
    worst = 0.0
    for first in range(0, cfg.instances, 1024):
        out, k, rt = _c4_wave(q, cfg, first, 1024, fn)
        assert np.all(np.isfinite(out))
        for j in range(1024):
            seed = cfg.seed + first + j
            sl = slice(j * cfg.W, (j + 1) * cfg.W)
            Rh = oracle.gen_positions(seed, 0, cfg.W, cfg.N, cfg.Np, cfg.L, np.float32, threads=THREADS)
            orc, absout, _ = oracle.eval_j2(Rh, k[sl], rt[sl], fn, cfg.N, cfg.n_up, threads=THREADS)
            e = oracle.normalized_error(out[sl], orc, absout, fn).max()
            worst = max(worst, e)
            assert e <= TOL[np.float32], (first + j, e)
    print(f"C4: all 4096 instances, worst normalized error {worst:.3e}")


# ---------------------------------------------------------------------------
# Warp-per-walker mapping (>= 4096 walker units, one tile per walker): the
# kernel C4's bench waves run.  Positions generated on the device; the oracle
# side regenerates sampled walkers with its own C generator.
# ---------------------------------------------------------------------------
def _warp_case(q, N, W, seed, dtype, row=False, P=1, sample=(0, 1, 97, 2048, 4095)):
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 32 if dtype == np.float32 else 16)
    R = q.gen_positions(seed, W, N, Np, L, tdt)
    k = qmcgen.make_k(seed, W, N)
    rt = qmcgen.make_trials(seed, np.arange(W), k, N, L, dtype, P=P)
    fn = qmcgen.make_functor(seed, L)
    res = q.eval(R, dev(k), dev(rt), fn, N, N // 2, row=row)
    out = (res[0] if row else res).cpu().numpy()
    w = np.array(sample)
    Rs = np.concatenate([oracle.gen_positions(seed, int(i), 1, N, Np, L, dtype) for i in w])
    orc, absout, orow = oracle.eval_j2(Rs, k[w], rt[w], fn, N, N // 2, row=row, threads=THREADS)
    assert oracle.normalized_error(out[w], orc, absout, fn).max() <= TOL[dtype]
    assert np.all(np.isfinite(out))
    if row:
        rowg = res[1].cpu().numpy()[w]
        for a in range(w.size):
            i = np.array([j for j in range(N) if j != k[w[a]]])
            if dtype == np.float32:
                tie = np.abs(np.abs(orow[a, 0, 1:, i]) - L / 2) <= 4 * np.spacing(np.float32(L))
                assert np.all((rowg[a, 0, 1:, i] == orow[a, 0, 1:, i].astype(np.float32)) | tie)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("N", [1000, 5003, 6144, 10001])
def test_warp_mapping_parity(q, dtype, N):
    _warp_case(q, N, 4096, seed=400 + N, dtype=dtype)


def test_warp_mapping_row_and_multi_trial(q):
    _warp_case(q, 3001, 4096, seed=77, dtype=np.float32, row=True)
    _warp_case(q, 2500, 4096, seed=78, dtype=np.float32, P=2)
    _warp_case(q, 2500, 2048, seed=79, dtype=np.float64, P=3, sample=(0, 1, 97, 2047))


def test_C4_batched_waves_as_benched(q):
    """C4 exactly as bench.py runs it: instances concatenated into one launch
    (here 5 instances = 5120 walkers, warp mapping), shared functor (R16)."""
    cfg = qmcgen.CONFIGS["C4"]
    insts = [0, 1, 2, 3, 4095]
    W = cfg.W
    R = torch.empty((len(insts) * W, 3, cfg.Np), dtype=torch.float32, device="cuda")
    ks, rts = [], []
    for j, inst in enumerate(insts):
        seed = cfg.seed + inst
        q.gen_positions(seed, W, cfg.N, cfg.Np, cfg.L, torch.float32, out=R[j * W:(j + 1) * W])
        k = qmcgen.make_k(seed, W, cfg.N)
        ks.append(k)
        rts.append(qmcgen.make_trials(seed, np.arange(W), k, cfg.N, cfg.L, np.float32))
    k = np.concatenate(ks)
    rt = np.concatenate(rts)
    fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
    out = q.eval(R, dev(k), dev(rt), fn, cfg.N, cfg.n_up).cpu().numpy()
    for j, inst in enumerate(insts):
        seed = cfg.seed + inst
        for wl in (0, 511, 1023):
            Rs = oracle.gen_positions(seed, wl, 1, cfg.N, cfg.Np, cfg.L, np.float32)
            g = j * W + wl
            orc, absout, _ = oracle.eval_j2(Rs, k[g:g + 1], rt[g:g + 1], fn, cfg.N, cfg.n_up)
            assert oracle.normalized_error(out[g:g + 1], orc, absout, fn).max() <= TOL[np.float32]


# ---------------------------------------------------------------------------
# NEXT-3: multi-trial batches (one trial per CTA, the P trials of a tile on
# consecutive CTAs): P = 12 NLPP quadrature virtual moves, P = 2 drift, ratios
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_nlpp_P12(q, dtype):
    N, W = 20001, 16
    L = qmcgen.cell_length(N)
    R, k, _, fn, n_up = instance(N, W, seed=61, dtype=dtype)
    rt = qmcgen.make_trials(61, np.arange(W), k, N, L, dtype, P=12, mode="nlpp")
    out, orc = check(q, R, k, rt, fn, N, n_up, dtype)
    # ratios relative to the caller's V_cur and relative to trial 0 (second launch)
    vcur = dev(orc[:, 0, 0].copy())
    _, r1 = q.eval(dev(R), dev(k), dev(rt), fn, N, n_up, V_cur=vcur, ratio=True)
    _, r0 = q.eval(dev(R), dev(k), dev(rt), fn, N, n_up, ratio=True)
    r1, r0 = r1.cpu().numpy(), r0.cpu().numpy()
    np.testing.assert_allclose(r1[:, :, 0], out[:, :, 0] - orc[:, :1, 0], rtol=0, atol=1e-9 * np.abs(out).max())
    assert np.all(r0[:, 0, 0] == 0.0) and np.all(r0[:, 0, 1] == 1.0)
    np.testing.assert_allclose(r0[:, :, 1], np.exp(out[:, :, 0] - out[:, :1, 0]), rtol=1e-12)


@pytest.mark.parametrize("name", ["C3P2", "C3P12"])
def test_multi_trial_full_size_every_walker(q, name):
    """The NEXT-3 bench workloads at full C3 size (N = 614,400, W = 1024, fp32)
    in the bench launch configuration; every walker vs the oracle."""
    cfg = qmcgen.config(name)
    P, mode = qmcgen.trial_spec(name)
    R = q.gen_positions(cfg.seed, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32)
    k = qmcgen.make_k(cfg.seed, cfg.W, cfg.N)
    rt = qmcgen.make_trials(cfg.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32, P=P, mode=mode)
    fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
    out = q.eval(R, dev(k), dev(rt), fn, cfg.N, cfg.n_up).cpu().numpy()
    del R
    torch.cuda.empty_cache()
    Rh = oracle.gen_positions(cfg.seed, 0, cfg.W, cfg.N, cfg.Np, cfg.L, np.float32, threads=THREADS)
    orc, absout, _ = oracle.eval_j2(Rh, k, rt, fn, cfg.N, cfg.n_up, threads=THREADS)
    del Rh
    assert np.all(np.isfinite(out))
    err = oracle.normalized_error(out, orc, absout, fn)
    assert err.max() <= TOL[np.float32], err.max()
