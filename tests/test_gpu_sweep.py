"""GPU parity of the resident-walker sweep (qj2_sweep) and the from-scratch
state (qj2_state_init) against the oracle (-m gpu; needs a B200).

qj2_sweep follows Alg. 1 L4-L9 with the ratio from the stored
5N state and the proposal r'_k = wrap(r_k + delta) formed
from the walker's current r_k (reading R24).  Every case runs the GPU sweep and
replays it with oracle.sweep (tests/sweep_check.py: decisions where clear,
dJ, positions bitwise, final state, J1 rows).
"""
import numpy as np
import pytest
import torch

import oracle
import qmcgen
from sweep_check import check_sweep, dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1708_02645_b200 as q
    q.device_check()
    return q


def _system(N, W, seed, n_up=None, m=8):
    L = qmcgen.cell_length(N)
    Np = qmcgen.padded_size(N, 32)
    R = qmcgen.positions(seed, np.arange(W), N, Np, L, np.float32)
    fn = qmcgen.make_functor(seed, L, m)
    return R, fn, L, Np, (N // 2 if n_up is None else n_up)


def _init_state(q, R, fn, N, n_up, j1=None):
    """qj2_state_init on the device (checked against the oracle in its own test)."""
    W, _, Np = R.shape
    Sd = torch.zeros((W, 5, Np), dtype=torch.float32, device="cuda")
    j1d = None
    if j1 is not None:
        ions, start, fn1 = j1
        j1d = (dev(ions), start, fn1, torch.zeros((W, 5, Np), dtype=torch.float32, device="cuda"))
    q.state_init(dev(R), Sd, fn, N, n_up, j1=j1d)
    return Sd.cpu().numpy(), (j1d[3].cpu().numpy() if j1d else None)


@pytest.mark.parametrize("N,n_up", [(2, 1), (33, 16), (256, 128), (385, 192), (600, 300), (768, 384), (1024, 512),
                                    (130, 0), (130, 130), (130, 47)])
def test_state_init_vs_oracle(q, N, n_up):
    """qj2_state_init == the oracle's from-scratch state (orc_j2_state), normalized
    by its absolute sums and the functor scale; padding
    untouched."""
    W = 6
    R, fn, L, Np, _ = _system(N, W, 10 + N)
    Sd = torch.full((W, 5, Np), 7.0, dtype=torch.float32, device="cuda")
    q.state_init(dev(R), Sd, fn, N, n_up)
    Sg = Sd.cpu().numpy()
    for w in range(W):
        st, ab = oracle.j2_state(R[w].astype(np.float64), N, n_up, fn)
        assert oracle.normalized_error_state(Sg[w][:, :N], st[:, :N], ab[:, :N], fn).max() <= 1e-5
    assert np.all(Sg[:, :, N:] == 7.0)


def test_state_init_j1_rows_vs_oracle(q):
    """With ions, every electron's J1 row == oracle.eval_j1 at its position."""
    N, W, n_ions = 300, 4, 37
    R, fn, L, Np, n_up = _system(N, W, 31)
    ions, start = qmcgen.make_ions(31, n_ions, qmcgen.padded_size(n_ions, 4), L, np.float32, n_species=3)
    fn1 = qmcgen.make_j1_functor(31, L, n_species=3, m=(8, 10, 6), rcut_frac=(0.5, 0.4, 0.3))
    _, S1 = _init_state(q, R, fn, N, n_up, j1=(ions, start, fn1))
    for w in range(W):
        o1, a1 = oracle.eval_j1(ions.astype(np.float64), start, R[w][:, :N].T.reshape(-1, 1, 3).astype(np.float64), fn1)
        err = oracle.normalized_error_j1(S1[w][:, :N].T.reshape(-1, 1, 5), o1, a1, fn1).max()
        assert err <= 1e-5


@pytest.mark.parametrize("N", [2, 33, 256, 257, 300, 384, 385, 512, 513, 600, 640, 641, 768, 769, 1000, 1024])
# every tier, full and ragged, and both sides of each tier boundary
def test_sweep_one_sweep_vs_oracle(q, N):
    """One ordered sweep (N moves) in one launch from the from-scratch state."""
    W = 12
    R, fn, L, Np, n_up = _system(N, W, 60 + N)
    ks, delta, u = qmcgen.make_sweep_moves(60 + N, W, N, N)
    state, _ = _init_state(q, R, fn, N, n_up)
    acc, _ = check_sweep(q, R, state, ks, delta, u, fn, N, n_up)
    assert 0 < (acc == 1).sum() < acc.size


@pytest.mark.parametrize("N,order", [(256, "ordered"), (768, "ordered"), (385, "random"), (768, "random"),
                                     (1024, "random")])
def test_sweep_three_sweeps_and_repeated_k(q, N, order):
    """S = 3N moves in one launch: three ordered sweeps, or k drawn at random with
    repeats -- every move starts from the walker's current r_k, so an electron
    that already moved is proposed from its new position (Alg. 1 L4-L9)."""
    W = 8
    R, fn, L, Np, n_up = _system(N, W, 70 + N)
    ks, delta, u = qmcgen.make_sweep_moves(70 + N, W, N, 3 * N, order=order)
    state, _ = _init_state(q, R, fn, N, n_up)
    check_sweep(q, R, state, ks, delta, u, fn, N, n_up)


def test_sweep_same_electron_back_to_back(q):
    """Runs of consecutive moves of the same electron (the owner of slot k writes
    r'_k and the next move reads it: the kernel's extra barrier)."""
    N, W, S = 768, 6, 400
    R, fn, L, Np, n_up = _system(N, W, 81)
    ks, delta, u = qmcgen.make_sweep_moves(81, W, N, S, order="random")
    ks[1::2] = ks[0::2][:ks[1::2].shape[0]]          # every odd move repeats the previous electron
    ks[100:140] = ks[100]                            # and a run of 40 moves of one electron
    state, _ = _init_state(q, R, fn, N, n_up)
    check_sweep(q, R, state, ks, delta, u, fn, N, n_up)


@pytest.mark.parametrize("n_up_case", ["zero", "all", "odd"])
def test_sweep_spin_boundaries(q, n_up_case):
    N, W = 130, 6
    n_up = {"zero": 0, "all": N, "odd": 47}[n_up_case]
    R, fn, L, Np, _ = _system(N, W, 90 + n_up)
    ks, delta, u = qmcgen.make_sweep_moves(90 + n_up, W, N, 2 * N, order="random")
    state, _ = _init_state(q, R, fn, N, n_up)
    check_sweep(q, R, state, ks, delta, u, fn, N, n_up)


def test_sweep_out_of_range_k(q):
    """A move whose k is outside [0, N) is never accepted, flagged -1, dj 0; the
    walker's other moves go on as the oracle says; padding is untouched."""
    for N in (130, 600, 768):          # 64 x 4, 64 x 10, 64 x 12 with the compile-time layout
        W = 6
        R, fn, L, Np, n_up = _system(N, W, 120 + N)
        ks, delta, u = qmcgen.make_sweep_moves(120 + N, W, N, N)
        for s_, w_, k_ in [(3, 2, -5), (7, 4, N), (11, 0, N + 1000), (12, 5, -(1 << 30)), (0, 1, N)]:
            ks[s_, w_] = k_
        state, _ = _init_state(q, R, fn, N, n_up)
        R[:, :, N:] = 3.0
        acc, dj = check_sweep(q, R, state, ks, delta, u, fn, N, n_up)
        for s_, w_ in [(3, 2), (7, 4), (11, 0), (12, 5), (0, 1)]:
            assert acc[s_, w_] == -1 and dj[s_, w_] == 0.0


def test_sweep_and_state_init_empty_calls(q):
    """W = 0 walkers or S = 0 moves: no launch, nothing touched, status OK."""
    N, W = 100, 3
    R, fn, L, Np, n_up = _system(N, W, 7)
    Rd, Sd = dev(R), torch.full((W, 5, Np), 2.5, dtype=torch.float32, device="cuda")
    ks, delta, u = qmcgen.make_sweep_moves(7, W, N, 0)
    q.sweep(Rd, Sd, dev(ks), dev(delta), dev(u), fn, N, n_up)                      # S = 0
    assert torch.equal(Rd.cpu(), torch.from_numpy(R)) and bool((Sd == 2.5).all())
    R0 = torch.zeros((0, 3, Np), dtype=torch.float32, device="cuda")
    S0 = torch.zeros((0, 5, Np), dtype=torch.float32, device="cuda")
    ks0, d0, u0 = qmcgen.make_sweep_moves(7, 0, N, 4)
    q.sweep(R0, S0, dev(ks0), dev(d0), dev(u0), fn, N, n_up)                        # W = 0
    q.state_init(R0, S0, fn, N, n_up)
    torch.cuda.synchronize()


@pytest.mark.parametrize("n_ions,S,N", [(64, 2, 200), (37, 3, 200), (256, 1, 200), (64, 2, 300), (256, 3, 450),
                                         (256, 2, 520), (64, 2, 640), (64, 2, 768), (100, 2, 1000), (100, 2, 1024)])
def test_sweep_with_j1_vs_oracle(q, n_ions, S, N):
    """J1 joined to every move: dJ = dJ2 + dJ1, the J1 rows of accepted electrons
    (two sweeps, random order), in every thread x partner tier (64 x 4 / 6 / 8 /
    10 / 12, 128 x 8; 256 ions: four per thread at 64 threads); 640, 768 and 1024
    fill the threads exactly."""
    W = 8
    R, fn, L, Np, n_up = _system(N, W, 300 + n_ions)
    ions, start = qmcgen.make_ions(300 + n_ions, n_ions, qmcgen.padded_size(n_ions, 4), L, np.float32, n_species=S)
    fn1 = qmcgen.make_j1_functor(300 + n_ions, L, n_species=S, m=(8, 10, 6), rcut_frac=(0.5, 0.4, 0.3))
    ks, delta, u = qmcgen.make_sweep_moves(300 + n_ions, W, N, 2 * N, order="random")
    state, S1 = _init_state(q, R, fn, N, n_up, j1=(ions, start, fn1))
    check_sweep(q, R, state, ks, delta, u, fn, N, n_up, j1=(ions, start, fn1), state_j1=S1)


def test_sweep_N64S_full_size_every_walker(q):
    """The N64S bench workload at full size (W = 1024 walkers of N = 768, one
    ordered sweep from the qj2_state_init state) in the bench launch
    configuration; every walker replayed by the oracle (the O(N^2) from-scratch
    state check on every 64th)."""
    cfg = qmcgen.config("N64S")
    N, W, n_up = cfg.N, cfg.W, cfg.n_up
    fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
    R = q.gen_positions(cfg.seed, W, N, cfg.Np, cfg.L, torch.float32).cpu().numpy()
    ks, delta, u = qmcgen.make_sweep_moves(cfg.seed, W, N, N)
    state, _ = _init_state(q, R, fn, N, n_up)
    check_sweep(q, R, state, ks, delta, u, fn, N, n_up, walkers_state=range(0, W, 64))


@pytest.mark.parametrize("with_j1", [False, True])
def test_sweep_deterministic(q, with_j1):
    """One barrier per move (double-buffered partials, U^2_k and move chunks;
    every thread writing only its own slots): five runs of a NiO-64-sized sweep
    from the same inputs are bitwise identical."""
    cfg = qmcgen.config("N64S")
    N, W, n_up = cfg.N, cfg.W, cfg.n_up
    fn = q.Functor.of(qmcgen.make_functor(cfg.seed, cfg.L, cfg.m))
    R0 = q.gen_positions(cfg.seed, W, N, cfg.Np, cfg.L, torch.float32)
    S0 = torch.zeros((W, 5, cfg.Np), dtype=torch.float32, device="cuda")
    ks, delta, u = qmcgen.make_sweep_moves(cfg.seed, W, N, 2 * N, order="random")
    kd, dd, ud = dev(ks), dev(delta), dev(u)
    j1 = None
    if with_j1:
        ions, start = qmcgen.make_ions(cfg.seed, 64, 64, cfg.L, np.float32, n_species=2)
        fn1 = q.J1Functor.of(qmcgen.make_j1_functor(cfg.seed, cfg.L, n_species=2))
    q.state_init(R0, S0, fn, N, n_up)
    results = []
    for _ in range(5):
        R, S = R0.clone(), S0.clone()
        if with_j1:
            j1 = (dev(ions), start, fn1, torch.zeros((W, 5, cfg.Np), dtype=torch.float32, device="cuda"))
        acc, dj = q.sweep(R, S, kd, dd, ud, fn, N, n_up, j1=j1)
        results.append((R, S, acc, dj) + ((j1[3],) if with_j1 else ()))
    torch.cuda.synchronize()
    for other in results[1:]:
        for a, b in zip(results[0], other):
            assert torch.equal(a, b)


def test_sweep_binding_rejects_bad_shapes(q):
    """The binding validates every tensor's shape before the C call."""
    N, W, S = 64, 4, 8
    R, fn, L, Np, n_up = _system(N, W, 5)
    ks, delta, u = qmcgen.make_sweep_moves(5, W, N, S)
    Rd, Sd = dev(R), torch.zeros((W, 5, Np), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        q.sweep(Rd, Sd, dev(ks[:, :2]), dev(delta), dev(u), fn, N, n_up)
    with pytest.raises(ValueError):
        q.sweep(Rd, Sd, dev(ks), dev(delta[:4]), dev(u), fn, N, n_up)
    with pytest.raises(ValueError):
        q.sweep(Rd, Sd[:, :4], dev(ks), dev(delta), dev(u), fn, N, n_up)
    with pytest.raises(ValueError):
        q.sweep(Rd, Sd, dev(ks), dev(delta), dev(u[:, :3]), fn, N, n_up)
