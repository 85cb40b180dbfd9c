"""Mutation check of the oracle's pins (-m "not gpu").

Each case applies one plausible mistake to a copy of oracle/oracle.c (a
flipped sign, a dropped term, a wrong index, spin boundary, basis derivative,
tie rule, scale or update direction), builds it, and runs the oracle pin
suites against it (ORACLE_LIB); the mutant must fail at least one pin.  This
is the automated form of DESIGN.md's mutation check.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_accept.py", "tests/test_oracle_spo.py",
        "tests/test_oracle_sweep.py"]

MUTANTS = {
    "eval_G_sign": ("nsum_add(&G[c], -g);", "nsum_add(&G[c], g);", 0),
    "eval_drop_2U'/r": ("nsum_add(&Lp, u[2] + 2.0 * u[1] / rho);", "nsum_add(&Lp, u[2]);", 0),
    "j1_G_sign": ("nsum_add(&G[c], -g);", "nsum_add(&G[c], g);", 1),
    "j1_drop_2U'/r": ("nsum_add(&Lp, u[2] + 2.0 * u[1] / rho);", "nsum_add(&Lp, u[2]);", 1),
    "self_exclusion_index": ("if (i == kw) continue;                 /* i != k, Eq. (5) */",
                             "if (i == kw + 1 || i == kw) continue;"),
    "spin_boundary": ("return ((i < n_up) == (k < n_up)) ? 0 : 1;", "return ((i <= n_up) == (k < n_up)) ? 0 : 1;"),
    "basis_derivative": ("double D1 = 0.5 * (3.0 * f * f - 4.0 * f);", "double D1 = 0.5 * (3.0 * f * f - 3.0 * f);"),
    "basis_second_derivative": ("double S2 = 1.0 - 3.0 * f;", "double S2 = 1.0 - 2.0 * f;"),
    "min_image_tie": ("else if (t <= -0.5 * L[c]) t += L[c];", "else if (t < -0.5 * L[c]) t += L[c];"),
    "cutoff_inclusive_wrong_radius": ("if (!(r < r_cut)) { out[0] = out[1] = out[2] = 0.0; return; }",
                                      "if (!(r < 0.9 * r_cut)) { out[0] = out[1] = out[2] = 0.0; return; }"),
    "accept_update_direction": ("Sw[c * Np + i] = old + (tn[c] - to[c]);", "Sw[c * Np + i] = old + (to[c] - tn[c]);"),
    "state_gradient_sign": ("for (int c = 0; c < 3; ++c) t[1 + c] = u[1] * d[c] / rho;",
                            "for (int c = 0; c < 3; ++c) t[1 + c] = -u[1] * d[c] / rho;"),
    "accept_commit_position": ("for (int c = 0; c < 3; ++c) Rw[c * Np + kw] = rn[c];", ""),
    "spo_axis_scale": ("Dx[a] * By[b] * Bz[c] * sx,                  /* gx  */",
                       "Dx[a] * By[b] * Bz[c] * sy,                  /* gx  */"),
    "spo_control_point_shift": ("for (int a = 0; a < 4; ++a) idx[a] = ((i - 1 + a) % n + n) % n;",
                                "for (int a = 0; a < 4; ++a) idx[a] = ((i + a) % n + n) % n;"),
    "spo_hessian_cross_term": ("Dx[a] * Dy[b] * Bz[c] * sx * sy,             /* hxy */",
                               "Dx[a] * By[b] * Dz[c] * sx * sy,             /* hxy */"),
    "det_ratio_laplacian_not_divided": ("out[4] = nsum_get(&Lp) / rho;", "out[4] = nsum_get(&Lp);"),
    "j1_species_functor": ("orc_bspline(coef + s * coef_stride, m[s], r_cut[s], rho, u);",
                           "orc_bspline(coef, m[s], r_cut[s], rho, u);", 0),
    "sweep_j1_species_functor": ("orc_bspline(coef + s * coef_stride, m[s], r_cut[s], rho, u);",
                                 "orc_bspline(coef, m[s], r_cut[s], rho, u);", 1),
    "sweep_ratio_sign": ("double dj = nsum_get(&Tk[0]) - Sw[k];", "double dj = Sw[k] - nsum_get(&Tk[0]);"),
    "sweep_decision_not_squared": ("J->u[sw] < rho * rho ? 1 : 0;", "J->u[sw] < rho ? 1 : 0;"),
    "sweep_commit_position": ("for (int c = 0; c < 3; ++c) Rw[c * Np + k] = rnf[c];", ""),
    "sweep_j1_sign": ("dj += o1n[0] - o1o[0];", "dj -= o1n[0] - o1o[0];"),
    "propose_wrap_direction": ("if (x < 0.0f) x = x + Lf;", "if (x < 0.0f) x = x - Lf;"),
}


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_pins_catch_mutant(name, tmp_path):
    old, new, *occ = MUTANTS[name]
    src = open(SRC).read()
    sites = [i for i in range(len(src)) if src.startswith(old, i)]
    if occ:
        assert len(sites) > occ[0], f"mutation site {occ[0]} for {name} not found"
        at = sites[occ[0]]
    else:
        assert len(sites) == 1, f"mutation site for {name} not found exactly once"
        at = sites[0]
    mut = tmp_path / "oracle_mut.c"
    mut.write_text(src[:at] + new + src[at + len(old):])
    so = tmp_path / "liboracle_mut.so"
    subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11",
                           "-pthread", "-o", str(so), str(mut), "-lm"])
    env = dict(os.environ, ORACLE_LIB=str(so))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *PINS],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"mutant {name} passed every pin:\n{r.stdout[-2000:]}"
