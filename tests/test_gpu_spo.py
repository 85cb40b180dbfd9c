"""GPU parity of NEXT-4 (qj2_spo_eval: Bspline-v / Bspline-vgh fused with the
determinant ratio of Eq. 6) against the CPU oracle (oracle.spo_vgh,
oracle.det_ratio), through the C ABI (-m gpu; needs a B200).

Tolerance (fp32 table, fp32 per-term arithmetic): per output
|x_gpu - x_orc| / max(A, F) <= 1e-5, A the oracle's sum of |weight * coef|
(or |a_o phi_o| for the ratio), F the table scale (max|P| times n/L per
derivative order).  The ratio's G and L are compared as rho*G and rho*L (the
lemma's numerators) so that a small rho does not amplify the comparison.
"""

import os

import numpy as np
import pytest
import torch

import oracle
import qmcgen

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def q():
    import paper_1708_02645_b200 as q
    assert torch.cuda.is_available()
    q.device_check()
    return q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _F(L, n):
    s = np.array(n, dtype=np.float64) / np.array(L, dtype=np.float64)
    # v, gx, gy, gz, hxx, hxy, hxz, hyy, hyz, hzz
    return np.array([1, s[0], s[1], s[2], s[0] ** 2, s[0] * s[1], s[0] * s[2], s[1] ** 2, s[1] * s[2], s[2] ** 2])


@pytest.fixture(params=["tma", "ldg"])
def kernel(request):
    """Both SPO kernels: the TMA-pipelined default ("auto") and the per-thread LDG gather
    kernel (QJ2_SPO_GATHER)."""
    return "auto" if request.param == "tma" else "gather"


def check_spo(q, nx, ny, nz, n_orb, ld, W, seed, pos_dtype=np.float32, L=(3.0, 3.5, 4.0), krow_mode=False,
              shift=0.0, kernel="auto"):
    T = qmcgen.spo_table(seed, nx, ny, nz, n_orb, ld)
    tab = q.SpoTable(dev(T), n_orb, L)
    rng = np.random.default_rng(seed)
    pos = (rng.random((W, 3)) * np.asarray(L) + shift).astype(pos_dtype)
    A = qmcgen.make_ainv_rows(seed, W, n_orb)
    if krow_mode:                        # full [W][n][lda] inverse, row krow[w]
        lda = n_orb + 3
        full = np.random.default_rng(seed + 1).random((W, n_orb, lda)).astype(np.float32)
        krow = rng.integers(0, n_orb, W).astype(np.int32)
        full[np.arange(W), krow, :n_orb] = A
        out, spo = q.spo_eval(tab, dev(pos), Ainv=dev(full), krow=dev(krow), want_spo=True, kernel=kernel)
    else:
        out, spo = q.spo_eval(tab, dev(pos), Ainv=dev(A), want_spo=True, kernel=kernel)
    out, spo = out.cpu().numpy(), spo.cpu().numpy()
    v, g, h, ab = oracle.spo_vgh(T, n_orb, L, pos.astype(np.float64))
    ref = np.concatenate([v[:, None, :], g, h], axis=1)               # [W][10][n_orb]
    F = np.abs(T).max() * _F(L, (nx, ny, nz))[None, :, None]
    err = np.abs(spo[:, :, :n_orb] - ref) / np.maximum(ab, F)
    assert np.all(np.isfinite(spo[:, :, :n_orb]))
    assert err.max() <= TOL, f"spo max normalized error {err.max():.3e}"
    orc, aab = oracle.det_ratio(A, v, g, h)
    scale = np.maximum(aab, oracle.det_ratio_scale(A, ab, np.abs(T).max() * _F(L, (nx, ny, nz))))
    rho_g, rho_o = out[:, 0], orc[:, 0]
    assert np.max(np.abs(rho_g - rho_o) / scale[:, 0]) <= TOL
    num_g = out[:, 1:] * rho_g[:, None]
    num_o = orc[:, 1:] * rho_o[:, None]
    assert np.max(np.abs(num_g - num_o) / scale[:, 1:]) <= TOL
    return T, tab, pos, out, spo


@pytest.mark.parametrize("n_orb,ld", [(1, 4), (3, 4), (10, 12), (64, 64), (130, 132), (384, 384), (600, 600)])
def test_spo_vgh_and_ratio(q, kernel, n_orb, ld):
    check_spo(q, 6, 7, 8, n_orb, ld, 37, seed=10 + n_orb, kernel=kernel)


def test_spo_z_wrap_and_many_walkers(q, kernel):
    """nz = 4: every walker's z rows wrap (split bulk copies); W > 32 * SMs
    exercises several producer batches per CTA."""
    check_spo(q, 5, 6, 4, 40, 40, 10000, seed=8, kernel=kernel)


def test_spo_fp64_positions_krow_and_wrapping(q, kernel):
    check_spo(q, 5, 9, 4, 48, 48, 29, seed=3, pos_dtype=np.float64, krow_mode=True, kernel=kernel)
    # positions outside [0, L): wrapped into the cell (periodic table)
    check_spo(q, 5, 9, 4, 48, 48, 29, seed=4, shift=-7.25, kernel=kernel)
    check_spo(q, 5, 9, 4, 48, 48, 29, seed=5, shift=11.5, kernel=kernel)


def test_spo_v_equals_vgh_values_bitwise(q, kernel):
    """Bspline-v and the value lanes of Bspline-vgh: the same sums in the same
    order (SPEC: 'vs spo_eval_vgh value lanes: identical'); the ratio rho is
    the same dot product reduced over a different thread grouping (1e-12)."""
    T, tab, pos, out, spo = check_spo(q, 8, 8, 8, 96, 96, 64, seed=21, kernel=kernel)
    A = qmcgen.make_ainv_rows(21, 64, 96)
    out_v, spo_v = q.spo_eval(tab, dev(pos), vgh=False, Ainv=dev(A), want_spo=True, kernel=kernel)
    assert torch.equal(spo_v[:, 0].cpu(), torch.from_numpy(spo[:, 0]))
    np.testing.assert_allclose(out_v.cpu().numpy()[:, 0], out[:, 0], rtol=1e-12, atol=1e-14)
    assert np.all(out_v.cpu().numpy()[:, 1:] == 0)


def test_spo_no_ratio_and_empty(q):
    T = qmcgen.spo_table(1, 4, 4, 4, 8, 8)
    tab = q.SpoTable(dev(T), 8, 2.0)
    pos = torch.rand((5, 3), device="cuda") * 2
    out, spo = q.spo_eval(tab, pos, want_spo=True)
    assert out is None and spo.shape == (5, 10, 8)
    e = q.spo_eval(tab, torch.zeros((0, 3), device="cuda"), Ainv=torch.zeros((0, 8), device="cuda"))
    assert e.shape == (0, 5)


def test_spo_device_generator_matches_host(q):
    g = q.gen_spo_table(77, 6, 5, 7, 30, 32).cpu().numpy()
    assert np.array_equal(g, qmcgen.spo_table(77, 6, 5, 7, 30, 32))


def test_spo_kernels_agree(q):
    """The TMA-pipelined and the LDG kernels: identical per-orbital sums (same
    order), ratios equal to rounding."""
    T = qmcgen.spo_table(31, 9, 8, 7, 200, 200)
    tab = q.SpoTable(dev(T), 200, (2.0, 2.5, 3.0))
    pos = dev((np.random.default_rng(1).random((3000, 3)) * 3).astype(np.float32))
    A = dev(qmcgen.make_ainv_rows(31, 3000, 200))
    o1, s1 = q.spo_eval(tab, pos, Ainv=A, want_spo=True)
    o2, s2 = q.spo_eval(tab, pos, Ainv=A, want_spo=True, kernel="gather")
    assert torch.equal(s1, s2)
    torch.testing.assert_close(o1, o2, rtol=1e-10, atol=1e-12)


def test_spo_nio64_full_size_sampled(q):
    """The bench workload: NiO-64-shaped table (80^3 grid, 384 orbitals = N/2
    for N = 768, fp32, 786 MB) generated on the device, 65,536 walkers'
    Bspline-vgh + ratio in the bench launch configuration; ~8300 walkers (both ends
    and every 8th) vs the oracle on the oracle side's own copy of the table."""
    cfg = qmcgen.SPO_CONFIGS["S1"]
    coef = q.gen_spo_table(cfg.seed, cfg.nx, cfg.ny, cfg.nz, cfg.n_orb, cfg.ld)
    tab = q.SpoTable(coef, cfg.n_orb, cfg.L)
    pos = qmcgen.spo_positions(cfg.seed, cfg.W, cfg.L)
    A = qmcgen.make_ainv_rows(cfg.seed, cfg.W, cfg.n_orb)
    out = q.spo_eval(tab, dev(pos), Ainv=dev(A)).cpu().numpy()
    del coef
    torch.cuda.empty_cache()
    T = oracle.gen_spo_table(cfg.seed, cfg.nx, cfg.ny, cfg.nz, cfg.n_orb, cfg.ld, threads=os.cpu_count() or 1)
    ws = np.r_[0:64, 64:cfg.W - 64:8, cfg.W - 64:cfg.W]          # ~8300 walkers: both ends, every 8th
    v, g, h, ab = oracle.spo_vgh(T, cfg.n_orb, cfg.L, pos[ws].astype(np.float64))
    orc, aab = oracle.det_ratio(A[ws], v, g, h)
    scale = np.maximum(aab, oracle.det_ratio_scale(A[ws], ab, np.abs(T).max() *
                                                   _F(cfg.L, (cfg.nx, cfg.ny, cfg.nz))))
    assert np.max(np.abs(out[ws, 0] - orc[:, 0]) / scale[:, 0]) <= TOL
    assert np.max(np.abs(out[ws, 1:] * out[ws, :1] - orc[:, 1:] * orc[:, :1]) / scale[:, 1:]) <= TOL


def test_spo_v_nlpp_points_share_the_walkers_row(q, kernel):
    """Bspline-v at the 12 NLPP quadrature points of each walker (all_trials,
    points_per_walker = 12): every point's ratio uses its walker's A^{-1} row."""
    n_orb, W = 48, 40
    L = (3.0, 3.0, 3.0)
    T = qmcgen.spo_table(51, 6, 6, 6, n_orb)
    tab = q.SpoTable(dev(T), n_orb, L)
    k = qmcgen.make_k(51, W, 200)
    pts = qmcgen.make_trials(51, np.arange(W), k, 200, 3.0, np.float32, P=12, mode="nlpp")     # [W][12][3]
    A = qmcgen.make_ainv_rows(51, W, n_orb)
    out, spo = q.spo_eval(tab, dev(pts), vgh=False, Ainv=dev(A), all_trials=True, want_spo=True, kernel=kernel)
    out, spo = out.cpu().numpy(), spo.cpu().numpy()
    assert out.shape == (W * 12, 5)
    v, g, h, ab = oracle.spo_vgh(T, n_orb, L, pts.reshape(-1, 3).astype(np.float64))
    err = np.abs(spo[:, 0, :n_orb] - v) / np.maximum(ab[:, 0], np.abs(T).max())
    assert err.max() <= TOL
    orc, aab = oracle.det_ratio(np.repeat(A, 12, axis=0), v, g, h)
    assert np.max(np.abs(out[:, 0] - orc[:, 0]) / aab[:, 0]) <= TOL


def test_spo_S1V_full_size_sampled(q):
    """The S1V bench workload at full size (NiO-64 table, 8192 walkers x 12 NLPP
    points, Bspline-v + ratio) in the bench launch configuration; sampled
    walkers' 12 points vs the oracle on its own C-generated table."""
    cfg = qmcgen.SPO_CONFIGS["S1V"]
    coef = q.gen_spo_table(cfg.seed, cfg.nx, cfg.ny, cfg.nz, cfg.n_orb, cfg.ld)
    tab = q.SpoTable(coef, cfg.n_orb, cfg.L)
    k = qmcgen.make_k(cfg.seed, cfg.W, cfg.N)
    pts = qmcgen.make_trials(cfg.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32, P=12, mode="nlpp")
    A = qmcgen.make_ainv_rows(cfg.seed, cfg.W, cfg.n_orb)
    out = q.spo_eval(tab, dev(pts), vgh=False, Ainv=dev(A), all_trials=True).cpu().numpy()
    del coef
    torch.cuda.empty_cache()
    T = oracle.gen_spo_table(cfg.seed, cfg.nx, cfg.ny, cfg.nz, cfg.n_orb, cfg.ld, threads=os.cpu_count() or 1)
    ws = np.r_[0:16, 16:cfg.W - 16:8, cfg.W - 16:cfg.W]           # ~1050 walkers x 12 points
    v, g, h, ab = oracle.spo_vgh(T, cfg.n_orb, cfg.L, pts[ws].reshape(-1, 3).astype(np.float64))
    orc, aab = oracle.det_ratio(np.repeat(A[ws], 12, axis=0), v, g, h)
    scale = np.maximum(aab, oracle.det_ratio_scale(np.repeat(A[ws], 12, axis=0), ab, np.abs(T).max() *
                                                   _F(cfg.L, (cfg.nx, cfg.ny, cfg.nz))))
    rows = (ws[:, None] * 12 + np.arange(12)[None, :]).reshape(-1)
    assert np.max(np.abs(out[rows, 0] - orc[:, 0]) / scale[:, 0]) <= TOL


def test_spo_tma_kernel_deterministic(q, kernel):
    """The bulk-copy ring (full/empty mbarriers) and the deferred ratio finalize leave
    no race: repeated evaluations over many walkers are bitwise identical."""
    T = qmcgen.spo_table(77, 20, 20, 20, 384, 384)
    tab = q.SpoTable(dev(T), 384, (4.0, 4.0, 4.0))
    rng = np.random.default_rng(77)
    pos = dev((rng.random((20000, 3)) * 4.0).astype(np.float32))
    A = dev(qmcgen.make_ainv_rows(77, 20000, 384))
    ref = q.spo_eval(tab, pos, Ainv=A, want_spo=True, kernel=kernel)
    for _ in range(4):
        out = q.spo_eval(tab, pos, Ainv=A, want_spo=True, kernel=kernel)
        assert torch.equal(out[0], ref[0]) and torch.equal(out[1], ref[1])


@pytest.mark.parametrize("kernel", ["auto", "gather"])
def test_spo_non_finite_positions_give_nan_not_faults(q, kernel):
    """A NaN or infinite coordinate gathers an in-range row with NaN weights: that
    walker's outputs are NaN, every other walker is unaffected, no device fault."""
    T = qmcgen.spo_table(91, 8, 8, 8, 64, 64)
    tab = q.SpoTable(dev(T), 64, (3.0, 3.0, 3.0))
    pos = (np.random.default_rng(5).random((40, 3)) * 3).astype(np.float32)
    bad = [3, 17, 31]
    pos[3, 0], pos[17, 1], pos[31, 2] = np.nan, np.inf, -np.inf
    A = qmcgen.make_ainv_rows(91, 40, 64)
    out, spo = q.spo_eval(tab, dev(pos), Ainv=dev(A), want_spo=True, kernel=kernel)
    torch.cuda.synchronize()
    out, spo = out.cpu().numpy(), spo.cpu().numpy()
    good = np.setdiff1d(np.arange(40), bad)
    assert np.all(np.isnan(out[bad, 0])) and np.all(np.isnan(spo[bad, 0, :64]))
    assert np.all(np.isfinite(out[good])) and np.all(np.isfinite(spo[good, :, :64]))
    ref, _ = q.spo_eval(tab, dev(pos[good]), Ainv=dev(A[good]), want_spo=True, kernel=kernel)
    assert np.array_equal(ref.cpu().numpy(), out[good])
