"""qmcgen -- seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no minimum image, no spline,
no reduction).  It only draws numbers.  Both the tests/oracle and the product
path may import it; it imports neither.

Input recipe:

* Cell: cubic, periodic, density 1: L = fl32(N ** (1/3)) (chosen exactly
  representable in fp32 so fp32 and fp64 paths share the same cell), r_cut = L/2
  (reading R4).
* Positions R[w][d][i]: counter-based hash (splitmix64 finaliser) of
  (seed, walker, coordinate, electron) -> u in [0,1) -> x = fl_T(L * u), kept
  below L.  The device generator in the CUDA library implements the same integer
  recipe independently (a test checks bit equality on samples).
* Active electron k_w ~ U{0..N-1}; trial r' = wrap(r_k + delta),
  delta ~ N(0, 0.01 I) (reading R13); NumPy default_rng.
* Functor: m = 8 intervals, per spin channel c[0..m-1] ~ U[0,1), c[m..m+2] = 0
  (C2 cutoff, reading R3).
* N_up = N / 2.

The paper's workloads (Table 1) need QMCPACK orbital,
pseudopotential and Jastrow files that are not available; these synthetic
inputs stand in for them with the paper's shape parameters (N, W).
"""
from __future__ import annotations

import dataclasses

import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = 0x9E3779B97F4A7C15
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def seed_key(seed: int) -> np.uint64:
    """Per-instance key: mix64(seed * GOLDEN + GOLDEN) (mod 2^64)."""
    s = (int(seed) * GOLDEN + GOLDEN) & 0xFFFFFFFFFFFFFFFF
    return mix64(np.array([s], dtype=np.uint64))[0]


def hash_u64(seed: int, w, d, i) -> np.ndarray:
    """h = mix64(key ^ ((w*3 + d) << 32 | i)) for broadcastable int arrays."""
    key = seed_key(seed)
    w = np.asarray(w, dtype=np.uint64)
    d = np.asarray(d, dtype=np.uint64)
    i = np.asarray(i, dtype=np.uint64)
    with np.errstate(over="ignore"):
        ctr = ((w * np.uint64(3) + d) << np.uint64(32)) | i
    return mix64(ctr ^ key)


def _scale(h: np.ndarray, L: float, dtype) -> np.ndarray:
    if np.dtype(dtype) == np.float32:
        u = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
        Lf = np.float32(L)
        x = (Lf * u).astype(np.float32)
        below = np.nextafter(Lf, np.float32(0))
        return np.where(x >= Lf, below, x).astype(np.float32)
    u = (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    x = np.float64(L) * u
    below = np.nextafter(np.float64(L), 0.0)
    return np.where(x >= L, below, x)


def cell_length(N: int) -> float:
    """L = fl32(N^(1/3)): density 1, exactly representable in fp32."""
    return float(np.float32(float(N) ** (1.0 / 3.0)))


def positions(seed: int, walkers, N: int, Np: int, L: float, dtype) -> np.ndarray:
    """R[len(walkers)][3][Np] (dtype); walkers are GLOBAL walker ids; padding 0."""
    walkers = np.asarray(walkers, dtype=np.int64).reshape(-1)
    out = np.zeros((walkers.size, 3, Np), dtype=dtype)
    i = np.arange(N, dtype=np.uint64)
    for a, w in enumerate(walkers):
        for d in range(3):
            out[a, d, :N] = _scale(hash_u64(seed, w, d, i), L, dtype)
    return out


def position_at(seed: int, w, d, i, L: float, dtype) -> np.ndarray:
    """Single coordinates R[w][d][i] for broadcastable index arrays."""
    return _scale(hash_u64(seed, w, d, i), L, dtype)


def padded_size(n: int, block: int) -> int:
    """Smallest multiple of block >= max(n, 1)."""
    if block < 1:
        raise ValueError("block must be >= 1")
    n = max(int(n), 1)
    return ((n + block - 1) // block) * block


@dataclasses.dataclass(frozen=True)
class Functor:
    """J2 radial functor data: cell, cutoff and two channels of m+3 B-spline
    coefficients ([0] same spin, [1] opposite spin)."""
    L: tuple
    r_cut: float
    m: int
    coef: np.ndarray  # [2][m+3] float64

    @property
    def delta(self) -> float:
        return self.r_cut / self.m


def make_functor(seed: int, L: float, m: int = 8, r_cut: float | None = None,
                 zero_tail: bool = True) -> Functor:
    rng = np.random.default_rng([int(seed), 2])
    coef = np.zeros((2, m + 3), dtype=np.float64)
    coef[:, :m] = rng.random((2, m))
    if not zero_tail:
        coef[:, m:] = rng.random((2, 3))
    rc = L / 2.0 if r_cut is None else float(r_cut)
    return Functor(L=(float(L),) * 3, r_cut=rc, m=int(m), coef=coef)


def make_k(seed: int, W: int, N: int, w_offset: int = 0) -> np.ndarray:
    """Active electron per walker, uniform on [0, N)."""
    rng = np.random.default_rng([int(seed), 1])
    k = rng.integers(0, N, size=w_offset + W, dtype=np.int64)[w_offset:]
    return k.astype(np.int32)


def make_trials(seed: int, walkers, k: np.ndarray, N: int, L: float, dtype,
                P: int = 1, mode: str = "move") -> np.ndarray:
    """r_trial[W][P][3] (dtype).

    mode="move":  every p is r'_k = wrap(r_k + delta_p), delta ~ N(0, 0.01 I).
    mode="drift": p = 0 is r_k itself (current position), p >= 1 are moves
                  (the P = 2 variant: value at R and at R' in one pass).
    mode="noop":  every p is r_k (no-op move).
    mode="nlpp":  P = 12 virtual moves of electron k onto the 12-point
                  icosahedral quadrature sphere about a nearby "ion" point
                  r_I ("quadrature on a spherical
                  shell"): r_q = wrap(r_I + |r_k - r_I| R v_q), v_q the unit
                  icosahedron vertices, R a random rotation per walker,
                  |r_k - r_I| ~ U[0.3, 1.0) (density-1 units).
    """
    if mode == "nlpp":
        return _nlpp_trials(seed, walkers, k, N, L, dtype, P)
    walkers = np.asarray(walkers, dtype=np.int64).reshape(-1)
    W = walkers.size
    rng = np.random.default_rng([int(seed), 3])
    # draw for the whole walker range up to max id so draws do not depend on
    # which subset is requested
    nmax = int(walkers.max()) + 1 if W else 0
    delta = rng.normal(0.0, 0.1, size=(nmax, P, 3))[walkers] if W else np.zeros((0, P, 3))
    rk = np.stack([position_at(seed, walkers, d, k.astype(np.int64), L, dtype)
                   for d in range(3)], axis=-1).astype(np.float64)  # [W][3]
    out = np.empty((W, P, 3), dtype=dtype)
    for p in range(P):
        if mode == "noop" or (mode == "drift" and p == 0):
            out[:, p, :] = rk.astype(dtype)
            continue
        t = np.mod(rk + delta[:, p, :], L)
        t = t.astype(dtype)
        below = np.nextafter(np.asarray(L, dtype=dtype), np.asarray(0, dtype=dtype))
        t = np.where(t >= np.asarray(L, dtype=dtype), below, t)
        out[:, p, :] = t
    return out


def _icosahedron() -> np.ndarray:
    g = (1.0 + 5.0 ** 0.5) / 2.0
    v = []
    for a in (-1.0, 1.0):
        for b in (-g, g):
            v += [(0.0, a, b), (a, b, 0.0), (b, 0.0, a)]
    v = np.array(v)
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _nlpp_trials(seed, walkers, k, N, L, dtype, P):
    if P != 12:
        raise ValueError("mode='nlpp' is the 12-point icosahedral rule (P = 12)")
    walkers = np.asarray(walkers, dtype=np.int64).reshape(-1)
    W = walkers.size
    nmax = int(walkers.max()) + 1 if W else 0
    # one stream per quantity, so a walker's draws do not depend on which walkers are requested
    rq, rd, rr = (np.random.default_rng([int(seed), 6, j]) for j in range(3))
    q = rq.normal(size=(nmax, 4))[walkers] if W else np.zeros((0, 4))          # random rotations
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    u_dir = rd.normal(size=(nmax, 3))[walkers] if W else np.zeros((0, 3))       # ion direction
    u_dir /= np.linalg.norm(u_dir, axis=1, keepdims=True)
    rad = rr.uniform(0.3, 1.0, size=nmax)[walkers] if W else np.zeros(0)
    rk = np.stack([position_at(seed, walkers, d, k.astype(np.int64), L, dtype) for d in range(3)],
                  axis=-1).astype(np.float64)
    rI = rk + rad[:, None] * u_dir
    a, b, c, d = q.T
    Rm = np.stack([np.stack([1 - 2 * (c * c + d * d), 2 * (b * c - a * d), 2 * (b * d + a * c)], -1),
                   np.stack([2 * (b * c + a * d), 1 - 2 * (b * b + d * d), 2 * (c * d - a * b)], -1),
                   np.stack([2 * (b * d - a * c), 2 * (c * d + a * b), 1 - 2 * (b * b + c * c)], -1)], 1)
    v = np.einsum("wij,qj->wqi", Rm, _icosahedron())
    t = np.mod(rI[:, None, :] + rad[:, None, None] * v, L).astype(dtype)
    below = np.nextafter(np.asarray(L, dtype=dtype), np.asarray(0, dtype=dtype))
    return np.where(t >= np.asarray(L, dtype=dtype), below, t)


def trial_spec(name: str):
    """(P, make_trials mode) of a bench configuration."""
    return {"C3P2": (2, "drift"), "C3P12": (12, "nlpp")}.get(name, (1, "move"))


def make_sweep(seed: int, W: int, N: int, L: float, dtype, steps: int):
    """NEXT-2 sweep inputs (harness draws, no method arithmetic): for sweep step
    s < steps, walker w moves electron k[s][w] = (k0_w + s) mod N (an ordered
    particle-by-particle sweep, Alg. 1 L4; every electron moves at most once
    while steps <= N, so its current position is still the generated one).
    Returns ks [S][W] int32, trials [S][W][2][3] dtype (trial 0 = r_k, trial 1
    = r'_k = wrap(r_k + delta), delta ~ N(0, 0.01 I)), u [S][W] fp64 uniforms
    in [0, 1) for the Metropolis test."""
    k0 = make_k(seed, W, N).astype(np.int64)
    s = np.arange(steps, dtype=np.int64)[:, None]
    ks = ((k0[None, :] + s) % N).astype(np.int32)
    rng = np.random.default_rng([int(seed), 5])
    delta = rng.normal(0.0, 0.1, size=(steps, W, 3))
    u = rng.random((steps, W))
    w = np.broadcast_to(np.arange(W, dtype=np.int64)[None, :], ks.shape)
    rk = np.stack([position_at(seed, w, d, ks.astype(np.int64), L, dtype) for d in range(3)], axis=-1)
    t = np.mod(rk.astype(np.float64) + delta, L).astype(dtype)
    below = np.nextafter(np.asarray(L, dtype=dtype), np.asarray(0, dtype=dtype))
    t = np.where(t >= np.asarray(L, dtype=dtype), below, t)
    trials = np.stack([rk.astype(dtype), t], axis=2)
    return ks, np.ascontiguousarray(trials), u


def make_sweep_moves(seed: int, W: int, N: int, steps: int, order: str = "ordered", sigma: float = 0.1,
                     stream: int = 0):
    """Inputs of qj2_sweep (harness draws, no method arithmetic): for move s <
    steps of walker w, the electron ks[s][w] and the proposal displacement
    delta[s][w] ~ N(0, sigma^2 I) (reading R13: sigma^2 = 0.01), fp32; u[s][w]
    fp64 uniforms in [0, 1) for the Metropolis test.  The kernel forms r'_k =
    wrap(r_k + delta) from the walker's CURRENT r_k, so any number of moves
    and any k sequence is valid.
    order="ordered": k = (k0_w + s) mod N (particle-by-particle sweeps, Alg. 1
    L4; steps = n*N is n full sweeps); order="random": k ~ U{0..N-1}
    independently per move (repeats included).  stream selects an independent
    draw of the same shape (consecutive sweeps of a Markov chain); an ordered
    sweep's k sequence is the same for every stream."""
    rng = np.random.default_rng([int(seed), 9, int(stream)])
    if order == "ordered":
        k0 = make_k(seed, W, N).astype(np.int64)
        s = np.arange(steps, dtype=np.int64)[:, None]
        ks = ((k0[None, :] + s) % N).astype(np.int32)
    elif order == "random":
        ks = rng.integers(0, N, size=(steps, W)).astype(np.int32)
    else:
        raise ValueError(order)
    delta = rng.normal(0.0, sigma, size=(steps, W, 3)).astype(np.float32)
    u = rng.random((steps, W))
    return ks, np.ascontiguousarray(delta), u


# ---------------------------------------------------------------------------
# NEXT-4 inputs: a synthetic 3D B-spline SPO coefficient table (Table 1 grid
# and orbital counts; the real DFT orbitals are not available)
# and A^{-1} rows.  Coefficient (ix, iy, iz, o) = u*2 - 1 with u the top 24
# bits of mix64(key' ^ flat index) times 2^-24 (exact in fp32); lanes
# [n_orb, ld) are 0.  The device twin is qj2gen_spo_table.
# ---------------------------------------------------------------------------
SPO_SALT = 0x5A0C0EFF1C1E17A5


def spo_key(seed: int) -> np.uint64:
    return mix64(np.array([int(seed_key(seed)) ^ SPO_SALT], dtype=np.uint64))[0]


def spo_table(seed: int, nx: int, ny: int, nz: int, n_orb: int, ld: int | None = None) -> np.ndarray:
    """fp32 [nx][ny][nz][ld] coefficient table (small grids: host generation)."""
    ld = n_orb if ld is None else ld
    key = spo_key(seed)
    idx = np.arange(nx * ny * nz * ld, dtype=np.uint64)
    h = mix64(idx ^ key)
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)
    t = u.reshape(nx, ny, nz, ld)
    t[..., n_orb:] = 0.0
    return t


def spo_table_rows(seed: int, nx: int, ny: int, nz: int, ld: int, n_orb: int, rows) -> np.ndarray:
    """Rows (ix, iy, iz) of the table, [len(rows)][ld] fp32, for sampled checks of big tables."""
    rows = np.asarray(rows, dtype=np.int64).reshape(-1, 3)
    flat = ((rows[:, 0] * ny + rows[:, 1]) * nz + rows[:, 2]).astype(np.uint64)
    idx = flat[:, None] * np.uint64(ld) + np.arange(ld, dtype=np.uint64)[None, :]
    h = mix64(idx ^ spo_key(seed))
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)
    u[:, n_orb:] = 0.0
    return u


@dataclasses.dataclass(frozen=True)
class SpoConfig:
    """NEXT-4 workload: a Table-1-shaped SPO set and W walker
    positions (one Bspline-vgh + determinant ratio each)."""
    name: str
    nx: int
    ny: int
    nz: int
    n_orb: int
    ld: int
    W: int
    N: int            # electrons of the system (cell: density 1)
    seed: int

    @property
    def L(self) -> float:
        return cell_length(self.N)

    @property
    def table_bytes(self) -> int:
        return self.nx * self.ny * self.nz * self.ld * 4


SPO_CONFIGS = {
    # NiO-64 (Table 1): N = 768, FFT grid 80^3; the determinant needs N/2 = 384 orbitals per spin
    "S1": SpoConfig("S1", 80, 80, 80, 384, 384, 65536, 768, seed=11),
    # NLPP ratios (Bspline-v): 8192 (walker, electron near an ion) pairs x 12 quadrature points
    "S1V": SpoConfig("S1V", 80, 80, 80, 384, 384, 8192, 768, seed=11),
}


@dataclasses.dataclass(frozen=True)
class J1Config:
    """NEXT-1 workload: the J1 share of one full PbyP sweep of a walker
    population, batched (DeltaJ1 of a move depends only on r_k and r'_k, so
    all proposals of a sweep are independent): W walkers x N electrons trial
    points against N_ion ions of S species (Table 1)."""
    name: str
    N: int
    n_ions: int
    n_species: int
    walkers: int
    seed: int

    @property
    def W(self) -> int:
        return self.walkers * self.N            # trial points (one per electron move)

    @property
    def L(self) -> float:
        return cell_length(self.N)


J1_CONFIGS = {
    # NiO-64 (Table 1): N = 768 electrons, 64 ions (Ni, O), the paper's 1024-walker population
    "J1S": J1Config("J1S", N=768, n_ions=64, n_species=2, walkers=1024, seed=13),
}


def spo_positions(seed: int, W: int, L: float) -> np.ndarray:
    """W positions uniform in the cell (fp32), the r'_k of one move per walker."""
    rng = np.random.default_rng([int(seed), 8])
    p = (rng.random((W, 3)) * L).astype(np.float32)
    return np.where(p >= np.float32(L), np.float32(0), p)


def make_ainv_rows(seed: int, W: int, n: int) -> np.ndarray:
    """Synthetic rows k of A^{-1} per walker, fp32 [W][n], U[-1, 1)/sqrt(n)."""
    rng = np.random.default_rng([int(seed), 7])
    return ((rng.random((W, n)) * 2 - 1) / np.sqrt(n)).astype(np.float32)


# ---------------------------------------------------------------------------
# NEXT-1 inputs: ions and per-species one-body functors.
# Table 1: N / N_ion = 12 for NiO (2 species, Ni and O, 1:1),
# 4 for graphite (1 species).  Ions are a fixed set shared by all walkers
# (PAPER:1306-1308), drawn from the same hash with a walker id no walker uses.
# ---------------------------------------------------------------------------
ION_WALKER_ID = (1 << 31) - 1


@dataclasses.dataclass(frozen=True)
class J1Functor:
    """Per-species one-body functors: r_cut[s], m[s], coef[s][max_m+3] (tail 0)."""
    L: tuple
    r_cut: tuple
    m: tuple
    coef: np.ndarray


def make_j1_functor(seed: int, L: float, n_species: int = 2, m=(8, 10), rcut_frac=(0.5, 0.4)) -> J1Functor:
    rng = np.random.default_rng([int(seed), 4])
    ms = tuple(int(m[s % len(m)]) for s in range(n_species))
    rcs = tuple(float(L) * float(rcut_frac[s % len(rcut_frac)]) for s in range(n_species))
    coef = np.zeros((n_species, max(ms) + 3))
    for s in range(n_species):
        coef[s, :ms[s]] = rng.random(ms[s])
    return J1Functor(L=(float(L),) * 3, r_cut=rcs, m=ms, coef=coef)


def make_ions(seed: int, n_ions: int, Np: int, L: float, dtype, n_species: int = 2):
    """ions [3][Np] (dtype, padding 0) sorted by species, and species_start [S+1]
    (species as equal as possible, NiO-like 1:1 for S = 2)."""
    R = positions(seed, [ION_WALKER_ID], n_ions, Np, L, dtype)[0]
    start = np.array([n_ions * s // n_species for s in range(n_species + 1)], dtype=np.int64)
    return R, start


# ---------------------------------------------------------------------------
# Configurations (BASELINE.json configs; concrete instances SURVEY.md 8(d)).
# ---------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    N: int
    W: int
    dtype: str          # "f32" | "f64"
    seed: int
    instances: int = 1  # C4: independent instances with seeds seed..seed+instances-1
    m: int = 8

    @property
    def np_dtype(self):
        return np.float32 if self.dtype == "f32" else np.float64

    @property
    def Np(self) -> int:
        # 128-byte padded lanes: 32 fp32 or 16 fp64 elements
        return padded_size(self.N, 32 if self.dtype == "f32" else 16)

    @property
    def L(self) -> float:
        return cell_length(self.N)

    @property
    def n_up(self) -> int:
        return self.N // 2

    @property
    def items(self) -> int:
        """(walker, trial, source i != k) terms per instance at P = 1."""
        return self.W * (self.N - 1)

    def functor(self, seed: int | None = None) -> Functor:
        return make_functor(self.seed if seed is None else seed, self.L, self.m)


CONFIGS = {
    "C1": Config("C1", N=14, W=1024, dtype="f64", seed=0),
    "C2": Config("C2", N=1400, W=1024, dtype="f32", seed=1),
    "C2f64": Config("C2f64", N=1400, W=1024, dtype="f64", seed=1),
    "C3": Config("C3", N=614400, W=1024, dtype="f32", seed=2),
    # C3's instance in fp64 (15.1 GB of positions): the fp64 path at the HBM roofline
    "C3f64": Config("C3f64", N=614400, W=1024, dtype="f64", seed=2),
    "C4": Config("C4", N=6144, W=1024, dtype="f32", seed=3, instances=4096),
    "C5": Config("C5", N=4915200, W=1024, dtype="f32", seed=5),
    # the paper's own NiO-64 size (Table 1: N = 768) and population (1024 walkers): one full
    # particle-by-particle sweep (768 moves per walker) as one CUDA graph
    "N64S": Config("N64S", N=768, W=1024, dtype="f32", seed=14),
    # the same sweep with the one-body Jastrow over NiO-64's 64 ions (Ni, O) in every move's ratio
    "N64SJ": Config("N64SJ", N=768, W=1024, dtype="f32", seed=14),
}


def config(name: str):
    """CONFIGS[name]; "C3S" (the NEXT-2 sweep-step bench) and "C3P2" / "C3P12"
    (NEXT-3 multi-trial benches: P = 2 drift variant, P = 12 NLPP quadrature)
    run on C3's instance."""
    if name in ("C3S", "C3P2", "C3P12"):
        return dataclasses.replace(CONFIGS["C3"], name=name)
    if name in SPO_CONFIGS:
        return SPO_CONFIGS[name]
    if name in J1_CONFIGS:
        return J1_CONFIGS[name]
    return CONFIGS[name]


def host_instance(cfg: Config, seed: int | None = None, walkers=None, P: int = 1,
                  mode: str = "move"):
    """Generate (R, k, r_trial, functor) on the host for the given walkers
    (default all).  Used for small configs and for sampled checks of large
    ones."""
    seed = cfg.seed if seed is None else seed
    walkers = np.arange(cfg.W) if walkers is None else np.asarray(walkers)
    L = cfg.L
    k_all = make_k(seed, cfg.W, cfg.N)
    k = k_all[walkers]
    R = positions(seed, walkers, cfg.N, cfg.Np, L, cfg.np_dtype)
    rt = make_trials(seed, walkers, k, cfg.N, L, cfg.np_dtype, P=P, mode=mode)
    # the functor is a property of the system: one per config (C4's 4096
    # instances share it; their seeds only change positions and moves)
    return R, k, rt, make_functor(cfg.seed, L, cfg.m)
