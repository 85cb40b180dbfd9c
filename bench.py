#!/usr/bin/env python
"""bench.py -- hot-path items/s and HBM-roofline fraction on B200, next to the
CPU oracle (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config NAME] [--dist-backend nccl|gloo] [--same-device]

One step = one pass of the whole hot path (staged
SoA rows -> on-the-fly distance row -> functor -> fp64 reduction -> out and
e^{dJ2}) over one batch: a single qj2_eval launch for all W walkers.

Workload (N=1 default): C3 = one instance of N = 614,400 electrons x W = 1024
walkers, P = 1, fp32 (7.55 GB of positions: larger than the 126 MB L2, so no
L2 flush is needed between steps).  BASELINE.json names C3 the "single-GPU
roofline measurement"; C2 (17 MB) is L2-resident and is a parity case.
N>1 (torchrun): the default is C5 -- one N = 4,915,200 instance split along
the electron axis, the partial sums combined with an NCCL all-reduce (strong
scaling; at N = 1 C5's per-GPU rate equals C3's, both streaming one pass of
positions at the HBM roofline).  --config C4 shards 4096 independent instances
by rank (strong); --config C3 runs one distinct C3 instance per rank (weak
scaling, no collective on the data path).

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hot-path items/sec and fraction of roofline at 1/2/4/8 B200 vs CPU oracle"
UNIT = "items/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=None,
                    choices=["C1", "C2", "C2f64", "C3", "C3f64", "C4", "C5", "C3S", "C3P2", "C3P12", "S1", "S1V", "J1S",
                             "N64S", "N64SJ"],
                    help="default: C3 at N = 1, C5 (source split + all-reduce) at N > 1")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend at N > 1 (gloo: functional runs of several ranks on one GPU)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 (functional multi-rank runs on a one-GPU box; not a measurement)")
    ap.add_argument("--c4-instances", type=int, default=0, help="C4 instance count override (functional runs)")
    ap.add_argument("--row", action="store_true",
                    help="C1/C2/C2f64/C3/C3f64: also write the candidate row (r, dx, dy, dz) per item (row a5)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-walkers", type=int, default=0, help="0 = auto")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def dist_init(world, device, backend="nccl"):
    import torch
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
    return dist if world > 1 else None


def allreduce_max(x: float, dist_mod) -> float:
    """max over ranks of a host number (per-rank device-timed spans, e2e times)."""
    if dist_mod is None:
        return x
    import torch
    dev = "cuda" if dist_mod.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist_mod.all_reduce(t, op=dist_mod.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------
class ClockSampler:
    BAD = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "hw_power_brake")

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.period = period_s
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            log(f"[bench] NVML unavailable: {e}")
            self.max_mhz = None

    def _names(self, mask):
        nv = self.nv
        table = {
            "gpu_idle": nv.nvmlClocksEventReasonGpuIdle,
            "applications_clocks_setting": nv.nvmlClocksEventReasonApplicationsClocksSetting,
            "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
            "hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
            "sync_boost": nv.nvmlClocksEventReasonSyncBoost,
            "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
            "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
            "hw_power_brake": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown,
        }
        return {n for n, b in table.items() if mask & b}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self._names(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}

    def rejected(self):
        s = self.summary()
        if any(r in s["reasons"] for r in self.BAD):
            return True
        if s["sm_mhz"] and s["sm_max_mhz"] and s["sm_mhz"] < 0.6 * s["sm_max_mhz"] and not s["reasons"]:
            return True
        return False


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy_ of 1 Gi bf16)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


ALU_PEAKS = os.path.join(ROOT, "profiles", "r02_alu_peaks.json")


def alu_peaks():
    """The measured ALU ceilings (tools/probe/alu_peaks.cu, committed as
    profiles/r02_alu_peaks.json): FP32 / FP64 TFLOP/s (FMA = 2 flops) and the
    thread-instruction issue rate, or None."""
    if os.path.exists(ALU_PEAKS):
        return json.load(open(ALU_PEAKS))
    return None


def kernel_record(config_name: str):
    """The committed ncu record of a configuration's dominant kernel
    (profiles/r02_kernels.json, else round 1's profiles/ncu_traffic.json): DRAM
    bytes and thread instructions per launch."""
    for name in ("r02_kernels.json", "ncu_traffic.json"):
        p = os.path.join(ROOT, "profiles", name)
        if os.path.exists(p):
            e = json.load(open(p)).get(config_name)
            if e:
                return e
    return {}


def committed_traffic(config_name: str):
    """dram read+write bytes per launch of the dominant kernel from the committed
    ncu --set full capture (profiles/), or None."""
    return kernel_record(config_name).get("dram_bytes_per_launch")


FLOPS_PER_TERM = 36       # algorithmic flops of one functor term (FMA = 2 flops)


def alu_roofline(cfg_name, kernel, kms, terms, fp64=False, extra=None, thread_inst=None):
    """Roofline of an issue/ALU-bound kernel: algorithmic flops (36 per functor term,
    FMA = 2) per launch / launch time against the measured FP32 (or FP64) FMA peak;
    beside it the issue fraction: the kernel's thread instructions per launch (the
    committed ncu record, or thread_inst = (count, how) derived from it by the
    caller) / launch time against the measured issue rate."""
    pk = alu_peaks()
    flops = terms * FLOPS_PER_TERM
    achieved = flops / (kms / 1e3) / 1e12
    if pk:
        peak = pk["fp64_tflops" if fp64 else "fp32_tflops"]
        src = (f"measured: {'DFMA' if fp64 else 'FFMA'} throughput, FMA = 2 flops (profiles/r02_alu_peaks.json, "
               f"{pk['sm_clock_mhz_median']:.0f} MHz)")
    else:
        peak = 148 * 128 * 2 * 1.965e9 / 1e12 / (2 if fp64 else 1)
        src = "derived: 148 SMs x 128 FP32 lanes x 2 flops x 1.965 GHz (no committed measurement)"
    r = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
         "traffic": committed_traffic(cfg_name), "kernel": kernel, "kernel_ms": kms, "alg_flops_per_launch": flops,
         "flops_per_term": FLOPS_PER_TERM, "terms_per_launch": terms, "peak_source": src}
    rec = kernel_record(cfg_name)
    if pk and (thread_inst or rec.get("thread_inst_per_launch")):
        ti, how = thread_inst or (rec["thread_inst_per_launch"], rec.get("source"))
        r["issue"] = {"thread_inst_per_launch": ti, "sass_per_term": ti / terms,
                      "achieved_tinst_per_s": ti / (kms / 1e3) / 1e12, "peak_tinst_per_s": pk["issue_tinst_per_s"],
                      "frac": ti / (kms / 1e3) / 1e12 / pk["issue_tinst_per_s"], "source": how}
    if extra:
        r.update(extra)
    return r


# ---------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------
class OracleSample:
    """The CPU oracle (as it stands) on walkers [0, n) of cfg.  Inputs are drawn
    by the oracle side's own C generator (untimed); run() times one evaluation
    (C3S: one sweep step -- eval at (r_k, r'_k), the Metropolis test and the
    accept-side update of R and the fp64 state)."""

    MAX_SWEEP_WALKERS = 48     # the oracle's fp64 state is 5 * 8 * N bytes per walker

    def __init__(self, cfg, n_walkers, threads):
        import oracle
        import qmcgen
        self.cfg, self.n, self.threads = cfg, int(n_walkers), threads
        self.sweep = cfg.name in ("C3S", "N64S", "N64SJ")
        self.moves = cfg.N if cfg.name in ("N64S", "N64SJ") else 1   # N64S(J): one full sweep per step
        self.j1 = None
        if cfg.name == "N64SJ":
            ions, start = qmcgen.make_ions(cfg.seed, 64, 64, cfg.L, np.float32, n_species=2)
            self.j1 = (ions.astype(np.float64), start, qmcgen.make_j1_functor(cfg.seed, cfg.L, n_species=2))
        if self.sweep and cfg.name in ("N64S", "N64SJ"):
            self.n = min(self.n, self.MAX_SWEEP_WALKERS)
            self.ks, self.delta, self.us = [a[:, :self.n] for a in qmcgen.make_sweep_moves(cfg.seed, cfg.W, cfg.N, self.moves)]
            self.rt = np.zeros((self.n, 1, 3), np.float32)
        elif self.sweep:
            self.n = min(self.n, self.MAX_SWEEP_WALKERS)
            ks, tr, u = qmcgen.make_sweep(cfg.seed, cfg.W, cfg.N, cfg.L, cfg.np_dtype, self.moves)
            self.ks, self.trs, self.us = ks[:, :self.n], tr[:, :self.n], u[:, :self.n]
            self.k, self.rt = self.ks[0], self.trs[0]
            self.S = np.zeros((self.n, 5, cfg.Np))
        else:
            P, mode = qmcgen.trial_spec(cfg.name)
            k_all = qmcgen.make_k(cfg.seed, cfg.W, cfg.N)
            self.k = k_all[:self.n]
            self.rt = qmcgen.make_trials(cfg.seed, np.arange(self.n), self.k, cfg.N, cfg.L, cfg.np_dtype, P=P,
                                         mode=mode)
        self.P = self.rt.shape[1]
        self.fn = qmcgen.make_functor(cfg.seed, cfg.L, cfg.m)
        self.R = oracle.gen_positions(cfg.seed, 0, self.n, cfg.N, cfg.Np, cfg.L, cfg.np_dtype, threads)
        if self.sweep and cfg.name in ("N64S", "N64SJ"):      # the state of the start configuration (untimed)
            self.S = np.stack([oracle.j2_state(self.R[w].astype(np.float64), cfg.N, cfg.n_up, self.fn)[0]
                               for w in range(self.n)])
            self.S1 = None
            if self.j1 is not None:
                ions, start, fn1 = self.j1
                self.S1 = np.zeros((self.n, 5, cfg.Np))
                for w in range(self.n):
                    o1, _ = oracle.eval_j1(ions, start, self.R[w][:, :cfg.N].T.reshape(-1, 1, 3).astype(np.float64), fn1)
                    self.S1[w][:, :cfg.N] = o1[:, 0].T
        # items in the bench's unit: (walker, trial, partner) terms; the sweep configs count one per
        # (move, partner) like their GPU lines
        self.items = self.n * (self.moves if self.sweep else self.P) * (cfg.N - 1 + (64 if self.j1 else 0))

    forced = None          # N64S(J): the GPU's decisions to replay (the parity field), else its own

    def run(self):
        """Time one pass; its outputs stay in self.result for the parity field."""
        import oracle
        t0 = time.perf_counter()
        if not self.sweep:
            out, ab, _ = oracle.eval_j2(self.R, self.k, self.rt, self.fn, self.cfg.N, self.cfg.n_up,
                                        threads=self.threads)
            dt = time.perf_counter() - t0
            self.result = (out, ab)
            return dt
        if self.cfg.name in ("N64S", "N64SJ"):           # oracle.sweep: the whole sweep, as it stands
            j1 = None if self.j1 is None else (self.j1[0], self.j1[1], self.j1[2], self.S1)
            res = oracle.sweep(self.R, self.S, self.ks, self.delta, self.us, self.fn, self.cfg.N, self.cfg.n_up,
                               j1=j1, forced=self.forced, threads=self.threads)
            dt = time.perf_counter() - t0
            self.result = res
            return dt
        R, S = self.R, self.S
        for m in range(self.moves):
            k, rt, u = self.ks[m], self.trs[m], self.us[m]
            out, ab, _ = oracle.eval_j2(R, k, rt, self.fn, self.cfg.N, self.cfg.n_up, threads=self.threads)
            if m == 0:
                self.result = (out, ab)
            d = out[:, 1, 0] - out[:, 0, 0]
            acc = (u < np.exp(d) ** 2).astype(np.int32)
            R, S, _ = oracle.accept(R, S, k, rt[:, 1], acc, self.fn, self.cfg.N, self.cfg.n_up)
        return time.perf_counter() - t0


_SPO_TABLE_CACHE = {}


class OracleSampleSpo:
    """NEXT-4 CPU oracle sample: Bspline-vgh of every orbital at the first n
    walkers' positions and the determinant ratio (oracle.spo_vgh + det_ratio,
    single-threaded as the oracle stands).  The table is generated once by the
    oracle side's own C generator (untimed)."""

    def __init__(self, cfg, n_walkers, threads):
        import oracle
        import qmcgen
        self.cfg, self.n = cfg, int(max(1, min(n_walkers, cfg.W)))
        if cfg.name not in _SPO_TABLE_CACHE:
            _SPO_TABLE_CACHE[cfg.name] = oracle.gen_spo_table(cfg.seed, cfg.nx, cfg.ny, cfg.nz, cfg.n_orb, cfg.ld,
                                                              threads=threads)
        self.T = _SPO_TABLE_CACHE[cfg.name]
        self.A = qmcgen.make_ainv_rows(cfg.seed, cfg.W, cfg.n_orb)[:self.n]
        if cfg.name == "S1V":          # 12 NLPP points per walker, each with its walker's A^-1 row
            k = qmcgen.make_k(cfg.seed, cfg.W, cfg.N)[:self.n]
            pts = qmcgen.make_trials(cfg.seed, np.arange(self.n), k, cfg.N, cfg.L, np.float32, P=12, mode="nlpp")
            self.pos = pts.reshape(-1, 3).astype(np.float64)
            self.A = np.repeat(self.A, 12, axis=0)
        else:
            self.pos = qmcgen.spo_positions(cfg.seed, cfg.W, cfg.L)[:self.n].astype(np.float64)
        self.items = self.pos.shape[0] * cfg.n_orb

    def run(self):
        import oracle
        t0 = time.perf_counter()
        v, g, h, ab = oracle.spo_vgh(self.T, self.cfg.n_orb, self.cfg.L, self.pos)
        out, aab = oracle.det_ratio(self.A, v, g, h)
        dt = time.perf_counter() - t0
        self.result = (out, aab, ab)
        return dt


class OracleSampleJ1:
    """NEXT-1 CPU oracle sample: oracle.eval_j1 (single-threaded as it stands)
    on the first n trial points of the J1S sweep batch."""

    def __init__(self, cfg, n, threads):
        self.cfg, self.n = cfg, int(max(1, min(n, cfg.W)))
        self.ions, self.start, self.rt, self.fn1 = j1_inputs(cfg, self.n)
        self.ions = self.ions.astype(np.float64)
        self.rt = self.rt.astype(np.float64)
        self.items = self.n * cfg.n_ions

    def run(self):
        import oracle
        t0 = time.perf_counter()
        out, ab = oracle.eval_j1(self.ions, self.start, self.rt, self.fn1)
        dt = time.perf_counter() - t0
        self.result = (out, ab)
        return dt


def j1_inputs(cfg, n=None, rank=0):
    """ions [3][Np], species_start, trial points [n][1][3] (fp32), J1 functor of a J1 config
    (the ions and functor are the system's; the trial points are rank-specific)."""
    import qmcgen
    n = cfg.W if n is None else n
    ions, start = qmcgen.make_ions(cfg.seed, cfg.n_ions, qmcgen.padded_size(cfg.n_ions, 4), cfg.L, np.float32,
                                   n_species=cfg.n_species)
    fn1 = qmcgen.make_j1_functor(cfg.seed, cfg.L, n_species=cfg.n_species)
    ids = np.arange(n)
    k = (ids % cfg.N).astype(np.int32)                 # electron of each trial point
    rt = qmcgen.make_trials(cfg.seed + rank, ids, k, cfg.N, cfg.L, np.float32)
    return ions, start, rt, fn1


def make_oracle_sample(cfg, n, threads):
    if cfg.name.startswith("S"):
        return OracleSampleSpo(cfg, n, threads)
    if cfg.name.startswith("J"):
        return OracleSampleJ1(cfg, n, threads)
    return OracleSample(cfg, n, threads)


def _what(cfg):
    import qmcgen
    if cfg.name.startswith("J"):
        return f"J1 over {cfg.n_ions} ions of {cfg.n_species} species, one trial point per row"
    if cfg.name == "S1V":
        return f"Bspline-v of {cfg.n_orb} orbitals at 12 NLPP points per walker + determinant ratios"
    if cfg.name.startswith("S"):
        return f"Bspline-vgh of {cfg.n_orb} orbitals + determinant ratio, {cfg.nx}x{cfg.ny}x{cfg.nz} grid"
    if cfg.name == "C3S":
        return "eval P=2 + Metropolis + accept update"
    if cfg.name in ("N64S", "N64SJ"):
        return (f"one sweep of {cfg.N} moves: eval P=2 + Metropolis + accept update"
                + (" + J1 over 64 ions" if cfg.name == "N64SJ" else ""))
    P, mode = qmcgen.trial_spec(cfg.name)
    return f"P={P} {mode}" if P > 1 else "P=1"


def oracle_sample_size(cfg, cores, budget_s):
    """Walkers such that one oracle pass takes about budget_s on `cores` threads
    (calibrated on one walker per core), capped at the whole workload."""
    n0 = min(cfg.W, cores)
    s0 = make_oracle_sample(cfg, n0, cores)
    dt0 = s0.run()
    per_round = max(dt0, 1e-6)              # one walker per core
    n = int(budget_s / per_round) * cores
    if cfg.name[0] in "SJ":                 # the SPO and J1 oracles run on one thread
        n = int(budget_s / per_round * n0)
    return max(n0, min(cfg.W, n)), s0.items / dt0


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def config_name(args, world):
    """--config, else the default workload: C3 (BASELINE.json's single-GPU roofline
    configuration) at N = 1 and C5 (the source-axis split whose partial sums meet
    in an all-reduce) at N > 1."""
    return args.config or ("C3" if world == 1 else "C5")


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    import qmcgen
    cfg = qmcgen.config(config_name(args, world))
    cores = cpu_cores()
    budget_total = 120.0
    per_step = max(0.2, min(10.0, budget_total / max(1, args.steps + args.warmup)))
    ws, rate0 = oracle_sample_size(cfg, cores, per_step)
    log(f"[reference] oracle {rate0:.3e} items/s (calibration); {ws} walkers per step")
    smp = make_oracle_sample(cfg, ws, cores)
    for _ in range(args.warmup):
        smp.run()
    times = [smp.run() for _ in range(args.steps)]
    t = float(np.mean(times))
    value = smp.items / t
    used = 1 if cfg.name[0] in "SJ" else cores
    sample = (f"{smp.n} of {cfg.W} walkers of {cfg.name} (N={cfg.N}, {_what(cfg)}) per step, fp32 inputs promoted "
              f"exactly to fp64, plain C oracle, {used} threads ({cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg.name in ("C4", "C5") else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(cfg, world):
    name = cfg.name
    if name.startswith("J"):
        return {"workload": f"{name} (NEXT-1): the J1 share of one PbyP sweep of {cfg.walkers} walkers of a NiO-64-"
                            f"shaped system (N={cfg.N} electrons, {cfg.n_ions} ions of {cfg.n_species} species), "
                            f"W={cfg.W} independent trial points per rank, fp32",
                "N": cfg.N, "n_ions": cfg.n_ions, "W": cfg.W, "parallelism": f"walker-batch x{world}",
                "l2": "inputs + outputs (~41 MB) < 126 MB L2: 256 MB L2 flush before every timed step"}
    if name.startswith("S"):
        what = ("12 NLPP quadrature points each (Bspline-v + determinant ratio, one A^-1 row per walker)"
                if name == "S1V" else "one Bspline-vgh + determinant ratio each")
        return {"workload": f"{name} (NEXT-4): NiO-64-shaped SPO set (Table 1: {cfg.nx}x{cfg.ny}x{cfg.nz} grid, "
                            f"{cfg.n_orb} orbitals = N/2 for N={cfg.N}, fp32 table {cfg.table_bytes / 1e6:.0f} MB), "
                            f"W={cfg.W} walkers per rank, {what}",
                "nx": cfg.nx, "n_orb": cfg.n_orb, "ld": cfg.ld, "W": cfg.W, "N": cfg.N,
                "parallelism": f"walker-batch x{world}",
                "l2": "table 786 MB > 126 MB L2; random gathers (no flush needed)"}
    sz = 8 if cfg.dtype == "f64" else 4
    rbytes = cfg.W * 3 * cfg.Np * sz
    desc = {
        "C1": f"C1: SPEC's tiny instance, N={cfg.N} electrons x W={cfg.W} walkers, P=1, fp64, seed 0(+rank)",
        "C2": f"C2: N={cfg.N} x W={cfg.W} (100 x C1's N), P=1, fp32, seed 1(+rank)",
        "C2f64": f"C2f64: N={cfg.N} x W={cfg.W} (100 x C1's N), P=1, fp64, seed 1(+rank)",
        "C3": f"C3: one instance per rank, N={cfg.N} electrons x W={cfg.W} walkers, P=1, fp32, seed 2(+rank)",
        "C3f64": f"C3f64: C3's instance in fp64 (N={cfg.N} x W={cfg.W}, P=1, seed 2(+rank)): the fp64 path",
        "C4": f"C4: {cfg.instances} instances of N={cfg.N} x W={cfg.W}, P=1, fp32, seeds 3.., sharded by instance",
        "C5": f"C5: one instance N={cfg.N} x W={cfg.W}, P=1, fp32, seed 5, split along N + NCCL all-reduce",
        "C3P2": f"C3P2 (NEXT-3): C3 instance per rank (N={cfg.N} x W={cfg.W}, fp32, seed 2(+rank)), P=2 drift "
                f"variant (U^2_k at r_k and r'_k in one step, ratio fused)",
        "C3P12": f"C3P12 (NEXT-3): C3 instance per rank (N={cfg.N} x W={cfg.W}, fp32, seed 2(+rank)), P=12 NLPP "
                 f"virtual moves (icosahedral quadrature sphere about a nearby ion point), ratios vs V_cur",
        "N64SJ": f"N64SJ: as N64S with the one-body Jastrow over NiO-64's 64 ions (Ni, O) joined to every move's "
                 f"ratio (dJ1 + dJ2) and state, one qj2_sweep launch per sweep",
        "N64S": f"N64S: the paper's NiO-64 size (N={cfg.N} electrons, Table 1) x W={cfg.W} walkers, fp32: one full "
                f"particle-by-particle sweep per step ({cfg.N} moves: r'_k = wrap(r_k + delta) -> U^2_k(R') on the "
                f"fly -> ratio against the stored U^2_k(R) -> Metropolis -> on acceptance the update of R and the "
                f"5N state) in one qj2_sweep launch, continuing the Markov chain from step to step",
        "C3S": f"C3S (NEXT-2 sweep step): C3 instance per rank (N={cfg.N} x W={cfg.W}, fp32, seed 2(+rank)), "
               f"one PbyP move per walker: eval at (r_k, r'_k) -> Metropolis -> accept-side update of R and "
               f"the 5N fp32 J2 state",
    }[name]
    if name in ("N64S", "N64SJ"):
        l2 = "R, state and moves (~53 MB) < 126 MB L2: 256 MB L2 flush before every timed step"
    elif name == "C4":
        l2 = (f"positions {rbytes / 1e6:.1f} MB per instance, {rbytes * 1024 / 1e9:.1f} GB per wave launch of 1024 "
              f"instances > 126 MB L2 (no flush needed)")
    elif rbytes < (126 << 20):
        l2 = f"positions {rbytes / 1e6:.1f} MB < 126 MB L2: 256 MB L2 flush before every timed step"
    else:
        l2 = f"inputs ({rbytes / 1e9:.2f} GB of positions per instance) > 126 MB L2 (no flush needed)"
    return {"workload": desc, "N": cfg.N, "W": cfg.W,
            "P": {"C3S": 2, "C3P2": 2, "C3P12": 12}.get(name, 1), "m": cfg.m, "Np": cfg.Np, "dtype": cfg.dtype,
            "parallelism": f"{'source-axis' if name == 'C5' else ('instance' if name == 'C4' else 'walker-instance')} x{world}",
            "l2": l2}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class EvalPlan:
    """The hot path on one instance per rank (C1, C2, C2f64, C3, C3f64; weak
    scaling, no collective on the data path): one qj2_eval launch over all W
    walkers, P = 1, ratio fused against the caller's 5N-state value V_cur."""
    launches_per_step = 1      # one j2_eval kernel (multi-tile rows add a 4 KB cudaMemsetAsync of the counters)
    roofline_from_timed = True  # a step is the eval launch: its roofline from the timed region's spans

    row = False                # --row: the optional row output (Fig. 6's v, 16 / 32 B per item more)
    row_out = None

    def __init__(self, cfg, rank, world):
        import torch
        self.cfg = cfg
        self.mode = cfg.name
        self.seed = cfg.seed + rank
        self.items_per_step = cfg.W * (cfg.N - 1)
        self.f64 = cfg.dtype == "f64"
        self.tdt = torch.float64 if self.f64 else torch.float32
        self.sz = 8 if self.f64 else 4
        # inputs that fit in the 126 MB L2 (C1, C2, C2f64) are flushed before every timed step
        self.flush_l2 = cfg.W * 3 * cfg.Np * self.sz < (126 << 20)
        self.ch = 204800 if not self.f64 else 102400          # tile of the CTA kernel (sources)
        self.warp_kernel = cfg.N <= 2048 or (cfg.N <= self.ch and cfg.W >= 4096)

    def items_total(self, world):
        return self.items_per_step * world

    def _alg(self):
        cfg = self.cfg
        # algorithmic bytes: x, y, z of every source i != k once per walker, plus per
        # walker k (4 B), r_trial (3 sz), V_cur (8 B), out (40 B), ratio (16 B)
        return cfg.W * (cfg.N - 1) * (3 + (4 if self.row else 0)) * self.sz + cfg.W * (4 + 3 * self.sz + 8 + 40 + 16)

    @property
    def alg_bytes_per_launch(self):
        return self._alg()

    def prepare(self, q):
        import torch
        import qmcgen
        cfg = self.cfg
        self.fn = q.Functor.of(qmcgen.make_functor(cfg.seed, cfg.L, cfg.m))
        self.R = q.gen_positions(self.seed, cfg.W, cfg.N, cfg.Np, cfg.L, self.tdt)
        k = qmcgen.make_k(self.seed, cfg.W, cfg.N)
        rt = qmcgen.make_trials(self.seed, np.arange(cfg.W), k, cfg.N, cfg.L, cfg.np_dtype)
        rk = qmcgen.make_trials(self.seed, np.arange(cfg.W), k, cfg.N, cfg.L, cfg.np_dtype, mode="noop")
        self.k = torch.from_numpy(k).cuda()
        self.rt = torch.from_numpy(rt).cuda()
        self.ws = q.Workspace(q.workspace_size(cfg.W, 1, cfg.N, self.tdt))
        # the caller's 5N state: U^2_k(R) at the current positions (untimed)
        v0 = q.eval(self.R, self.k, torch.from_numpy(rk).cuda(), self.fn, cfg.N, cfg.n_up, workspace=self.ws)
        self.V_cur = v0[:, 0, 0].contiguous()
        self.out = torch.empty((cfg.W, 1, 5), dtype=torch.float64, device="cuda")
        self.ratio = torch.empty((cfg.W, 1, 2), dtype=torch.float64, device="cuda")
        self.row_out = (torch.empty((cfg.W, 1, 4, cfg.Np), dtype=self.tdt, device="cuda") if self.row else None)
        torch.cuda.synchronize()

    def step(self, q, dist_mod):
        cfg = self.cfg
        q.eval(self.R, self.k, self.rt, self.fn, cfg.N, cfg.n_up, V_cur=self.V_cur, ratio=True, row=self.row,
               out=self.out, row_out=self.row_out, ratio_out=self.ratio, workspace=self.ws)

    def kernel_ms(self, q, stream, reps):
        if self.flush_l2:
            return self.flusher.event_ms(lambda: self.step(q, None), stream, reps)
        return _event_ms(lambda: self.step(q, None), stream, reps)

    def gpu_sample(self, n):
        """(out [n][P][5]) of walkers [0, n) from the last step, for the parity field."""
        return self.out[:n].cpu().numpy()

    def roofline(self, kms, peak_hbm):
        cfg = self.cfg
        achieved = self._alg() / (kms / 1e3) / 1e9
        kern = ("j2_eval_warp_kernel" if self.warp_kernel else "j2_eval_kernel") + \
            f"<{'double' if self.f64 else 'float'}>"
        r = {"bound": "hbm", "achieved": achieved, "peak": peak_hbm, "unit": "GB/s", "frac": achieved / peak_hbm,
             "traffic": committed_traffic(self.mode), "kernel": kern, "kernel_ms": kms,
             "alg_bytes_per_launch": self._alg(), "bytes_per_item": 3 * self.sz}
        if self.flush_l2:
            r["regime"] = (f"launch/latency-bound: {cfg.W * 3 * cfg.Np * self.sz / 1e6:.1f} MB of positions per step "
                           f"(L2 flushed before every step); not an HBM measurement (SURVEY 8(d))")
        if self.f64:      # the fp64 path also against the measured DFMA peak (36 flops per term)
            pk = alu_peaks()
            if pk:
                fl = cfg.W * (cfg.N - 1) * FLOPS_PER_TERM / (kms / 1e3) / 1e12
                r["fp64_alu"] = {"achieved": fl, "peak": pk["fp64_tflops"], "unit": "TFLOP/s",
                                 "frac": fl / pk["fp64_tflops"], "source": "profiles/r02_alu_peaks.json (DFMA)"}
        return r

    def e2e(self, q, steps, dist_mod):
        """Same metric through the public host-buffer API (qj2_eval_host): every step copies the
        step's inputs from pinned host memory and reads the result back."""
        import torch
        cfg = self.cfg
        try:
            Rh = torch.empty(self.R.shape, dtype=self.R.dtype, pin_memory=True)
            pinned = True
        except RuntimeError as e:       # host without room to pin the positions: pageable copies
            log(f"[bench] pinned host buffer unavailable ({e}); e2e uses pageable memory")
            Rh = torch.empty(self.R.shape, dtype=self.R.dtype)
            pinned = False
        Rh.copy_(self.R)
        kh = self.k.cpu().pin_memory()
        th = self.rt.cpu().pin_memory()
        vh = self.V_cur.cpu().pin_memory() if self.V_cur is not None else None
        P = th.shape[1]
        outh = torch.empty((cfg.W, P, 5), dtype=torch.float64, pin_memory=True)
        rath = torch.empty((cfg.W, P, 2), dtype=torch.float64, pin_memory=True)
        chunk = 32 if cfg.N > 100000 else max(32, min(cfg.W, 256))
        ws = q.Workspace(q.host_workspace_size(cfg.W, P, cfg.Np, self.tdt, chunk))
        run = lambda: q.eval_host(Rh, kh, th, self.fn, cfg.N, cfg.n_up, V_cur=vh, ratio=True,  # noqa: E731
                                  chunk_walkers=chunk, out=outh, ratio_out=rath, workspace=ws)
        run()
        torch.cuda.synchronize()
        if dist_mod:
            dist_mod.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            run()
        dt = (time.perf_counter() - t0) / steps
        dt = allreduce_max(dt, dist_mod)
        same = bool(torch.equal(outh, self.out.cpu()))
        world = dist_mod.get_world_size() if dist_mod else 1
        h2d = Rh.numel() * self.sz + kh.numel() * 4 + th.numel() * self.sz + (vh.numel() * 8 if vh is not None else 0)
        d2h = outh.numel() * 8 + rath.numel() * 8
        del Rh
        return {"value": self.items_per_step * world / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3, "steps": steps,
                "api": f"qj2_eval_host ({'pinned' if pinned else 'pageable'} host buffers, 2-stage H2D/compute pipeline)",
                "matches_device_path": same}


def _event_ms(fn, stream, reps=1):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


L2_FLUSH_BYTES = 256 << 20     # > the 126 MB L2
SPIN_CYCLES = 400_000          # ~0.2 ms of device spin before each separately timed step


class L2Flusher:
    """For workloads whose inputs fit in L2: a 256 MB write before every timed
    step evicts the previous step's lines; each step is timed on its own events
    (the flush is outside them) and the step time is their mean."""

    def __init__(self):
        import torch
        self.buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def flush(self):
        self.buf.fill_(1.0)

    def event_ms(self, fn, stream, reps=1, spans=None):
        """Mean span of reps flushed launches of fn (spans, if given, receives each)."""
        import torch
        evs = []
        for _ in range(reps):
            self.flush()
            # keep the GPU busy (untimed) while the host prepares the launch, so that the
            # events time the kernel and not the host's launch latency
            torch.cuda._sleep(SPIN_CYCLES)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        t = [a.elapsed_time(b) for a, b in evs]
        if spans is not None:
            spans[:] = t
        return sum(t) / reps


class C5Plan:
    """One instance N = 4,915,200 x W = 1024 split along the electron axis: rank g
    evaluates sources [g*N/G, (g+1)*N/G) (qj2_eval with i_offset), then one NCCL
    all_reduce(SUM) of the 40 KB fp64 partials and qj2_ratio (strong scaling)."""
    mode = "C5"
    launches_per_step = 2      # j2_eval_kernel + ratio_kernel (+ the counter memset and the NCCL all-reduce)

    def __init__(self, cfg, rank, world):
        from paper_1708_02645_b200 import parallel
        self.cfg, self.rank, self.world = cfg, rank, world
        self.a, self.b = parallel.shard_bounds(cfg.N, rank, world)
        self.n_local = self.b - self.a
        self.Np = ((self.n_local + 31) // 32) * 32
        self.items_per_step = cfg.W * (cfg.N - 1)      # global: every rank reports the whole job
        self.alg_bytes_per_launch = cfg.W * self.n_local * 12 + cfg.W * (4 + 12 + 40)

    def items_total(self, world):
        return self.items_per_step

    def prepare(self, q):
        import torch
        import qmcgen
        from paper_1708_02645_b200 import parallel
        self.parallel = parallel
        cfg = self.cfg
        self.fn = q.Functor.of(qmcgen.make_functor(cfg.seed, cfg.L, cfg.m))
        self.R = q.gen_positions(cfg.seed, cfg.W, self.n_local, self.Np, cfg.L, torch.float32, i_offset=self.a)
        k = qmcgen.make_k(cfg.seed, cfg.W, cfg.N)
        rt = qmcgen.make_trials(cfg.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32)
        rk = qmcgen.make_trials(cfg.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32, mode="noop")
        self.k = torch.from_numpy(k).cuda()
        self.rt = torch.from_numpy(rt).cuda()
        self.ws = q.Workspace(q.workspace_size(cfg.W, 1, self.n_local, torch.float32))
        v0 = parallel.eval_sharded(self.R, self.k, torch.from_numpy(rk).cuda(), self.fn, cfg.N, cfg.n_up,
                                   self.a, self.n_local, workspace=self.ws)
        self.V_cur = v0[:, 0, 0].contiguous()
        self.out = torch.empty((cfg.W, 1, 5), dtype=torch.float64, device="cuda")
        self.ratio = torch.empty((cfg.W, 1, 2), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

    def step(self, q, dist_mod):
        cfg = self.cfg
        self.parallel.eval_sharded(self.R, self.k, self.rt, self.fn, cfg.N, cfg.n_up, self.a, self.n_local,
                                   V_cur=self.V_cur, ratio=True, out=self.out, ratio_out=self.ratio,
                                   workspace=self.ws)

    def kernel_ms(self, q, stream, reps):
        """The eval kernel alone; spans() adds the kernel + all-reduce + ratio span."""
        cfg = self.cfg
        kms = _event_ms(lambda: q.eval(self.R, self.k, self.rt, self.fn, cfg.N, cfg.n_up, i_offset=self.a,
                                       n_local=self.n_local, out=self.out, workspace=self.ws), stream, reps)
        full = _event_ms(lambda: self.step(q, None), stream, reps)
        self.span = {"kernel_ms": kms, "kernel_allreduce_ratio_ms": full,
                     "allreduce": "torch.distributed all_reduce(SUM) of W*5 fp64 (40 KB) on the "
                                  + (self.parallel_backend() or "(one rank: none)")}
        return kms

    def parallel_backend(self):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return dist.get_backend()
        return None

    def gpu_sample(self, n):
        return self.out[:n].cpu().numpy()

    def e2e(self, q, steps, dist_mod):
        # 60 GB of positions per step cannot sit in pinned host memory: the host-buffer
        # path is measured on C3 / C3f64 (same kernel, same access pattern)
        return {"value": None, "reason": "the step's inputs (60.4 GB of positions over all ranks) exceed pinned "
                                         "host memory; end to end is measured on C3 (same kernel)"}


class C4Plan:
    """4096 independent instances (N = 6144, W = 1024, seeds 3..4098, one functor)
    sharded by instance; each rank evaluates its instances as one batch of
    n_inst * 1024 walkers per launch, in waves that fit HBM (generation of a
    wave is outside the timed spans; the step time is the sum of the waves'
    kernel spans).  No collective on the data path."""
    mode = "C4"
    launches_per_step = 1      # per wave: one j2_eval_warp_kernel (one tile per walker: no memset)
    MAX_RESIDENT = 1024        # instances per wave (77 GB)

    def __init__(self, cfg, rank, world):
        from paper_1708_02645_b200 import parallel
        self.cfg, self.rank, self.world = cfg, rank, world
        self.i0, self.i1 = parallel.instance_range(cfg.instances, rank, world)
        self.n_inst = self.i1 - self.i0
        self.waves = parallel.waves(self.i0, self.n_inst, self.MAX_RESIDENT)
        self.launches_per_step = len(self.waves)
        self.items_per_step = self.n_inst * cfg.W * (cfg.N - 1)
        self.timed_wave_ms = None
        n_first = self.waves[0][1] if self.waves else 0
        self.alg_bytes_per_launch = n_first * cfg.W * ((cfg.N - 1) * 12 + 4 + 12 + 8 + 40 + 16)

    def items_total(self, world):
        return self.cfg.instances * self.cfg.W * (self.cfg.N - 1)

    def _gen_wave(self, q, first, count):
        import torch
        cfg = self.cfg
        for j in range(count):
            q.gen_positions(cfg.seed + first + j, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32,
                            out=self.R[j * cfg.W:(j + 1) * cfg.W])

    def prepare(self, q):
        import torch
        import qmcgen
        cfg = self.cfg
        self.q = q
        self.fn = q.Functor.of(qmcgen.make_functor(cfg.seed, cfg.L, cfg.m))
        nmax = max((c for _, c in self.waves), default=0)
        self.R = torch.empty((nmax * cfg.W, 3, cfg.Np), dtype=torch.float32, device="cuda")
        ks, rts, rks = [], [], []
        for inst in range(self.i0, self.i1):
            seed = cfg.seed + inst
            k = qmcgen.make_k(seed, cfg.W, cfg.N)
            ks.append(k)
            rts.append(qmcgen.make_trials(seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32))
            rks.append(qmcgen.make_trials(seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32, mode="noop"))
        self.k = torch.from_numpy(np.concatenate(ks)).cuda()
        self.rt = torch.from_numpy(np.concatenate(rts)).cuda()
        rk = torch.from_numpy(np.concatenate(rks)).cuda()
        self.ws = q.Workspace(0)
        self.out = torch.empty((self.n_inst * cfg.W, 1, 5), dtype=torch.float64, device="cuda")
        self.ratio = torch.empty((self.n_inst * cfg.W, 1, 2), dtype=torch.float64, device="cuda")
        self.V_cur = torch.empty((self.n_inst * cfg.W,), dtype=torch.float64, device="cuda")
        for first, count in self.waves:
            self._gen_wave(q, first, count)
            sl = self._slice(first, count)
            v0 = q.eval(self.R[:count * cfg.W], self.k[sl], rk[sl], self.fn, cfg.N, cfg.n_up, workspace=self.ws)
            self.V_cur[sl] = v0[:, 0, 0]
        self.resident = self.waves[-1] if self.waves else None
        torch.cuda.synchronize()

    def _slice(self, first, count):
        W = self.cfg.W
        return slice((first - self.i0) * W, (first - self.i0 + count) * W)

    def _eval_wave(self, q, first, count):
        cfg = self.cfg
        sl = self._slice(first, count)
        q.eval(self.R[:count * cfg.W], self.k[sl], self.rt[sl], self.fn, cfg.N, cfg.n_up, V_cur=self.V_cur[sl],
               ratio=True, out=self.out[sl], ratio_out=self.ratio[sl], workspace=self.ws)

    def step(self, q, dist_mod):
        # warm-up form: evaluate the resident wave(s) only
        if len(self.waves) == 1:
            self._eval_wave(q, *self.waves[0])
        else:
            self._eval_wave(q, *self.resident)

    def timed(self, K, stream, local, dist_mod):
        """Sum over waves of the kernel spans (generation between waves untimed)."""
        import torch
        q = self.q
        if dist_mod:
            dist_mod.barrier()
        torch.cuda.synchronize()
        total = 0.0
        with ClockSampler(local) as clk:
            if len(self.waves) == 1:
                total = _event_ms(lambda: self._eval_wave(q, *self.waves[0]), stream, K) * K
            else:
                for _ in range(K):
                    for first, count in self.waves:
                        if (first, count) != self.resident:
                            self._gen_wave(q, first, count)
                            self.resident = (first, count)
                            torch.cuda.synchronize()
                        total += _event_ms(lambda: self._eval_wave(q, first, count), stream, 1)
        if dist_mod:
            dist_mod.barrier()
        self.timed_wave_ms = total / (K * len(self.waves)) if self.waves else None
        return total / K, clk

    def kernel_ms(self, q, stream, reps):
        """The wave kernel's mean launch span over the timed region (each timed span is
        exactly one wave launch); the same launch repeated back to back, where the
        power cap lowers the clock further, is reported beside it."""
        b2b = _event_ms(lambda: self._eval_wave(q, *self.resident), stream, reps)
        self.span = {"wave_kernel_ms_timed_region": self.timed_wave_ms, "wave_kernel_ms_back_to_back": b2b,
                     "note": "roofline from the timed region's wave spans; back to back (no generation between "
                             "waves) the 1000 W cap holds the kernel lower"}
        return self.timed_wave_ms if self.timed_wave_ms else b2b

    def gpu_sample(self, n):
        """instance i0's first n walkers (evaluated in the rank's first wave)."""
        first, count = self.waves[0]
        if self.resident != self.waves[0]:
            self._gen_wave(self.q, first, count)
            self.resident = self.waves[0]
            self._eval_wave(self.q, first, count)
        return self.out[:n].cpu().numpy()

    def e2e(self, q, steps, dist_mod):
        return {"value": None, "reason": "the step's inputs (309 GB of positions over 4096 instances) exceed pinned "
                                         "host memory; end to end is measured on C3 (same kernel family)"}


class MultiTrialPlan(EvalPlan):
    """NEXT-3: the hot path with P trial positions per walker (P = 2 drift
    variant, P = 12 NLPP quadrature), one eval launch per step; the P trials
    of a tile run on consecutive CTAs (one HBM read, L2 hits for the rest).
    Issue-bound (FP32 ALU) rather than HBM-bound."""
    launches_per_step = 1      # j2_eval_kernel (+ the ratio kernel when V_cur is not given: drift)

    def __init__(self, cfg, rank, world):
        import qmcgen
        super().__init__(cfg, rank, world)
        self.mode = cfg.name
        self.P, self.tmode = qmcgen.trial_spec(cfg.name)
        self.items_per_step = cfg.W * self.P * (cfg.N - 1)
        if self.tmode == "drift":
            self.launches_per_step = 2

    def _alg(self):
        cfg = self.cfg
        return cfg.W * (cfg.N - 1) * 12 + cfg.W * (4 + 12 * self.P + 8 + 56 * self.P)

    def prepare(self, q):
        import torch
        import qmcgen
        cfg = self.cfg
        self.fn = q.Functor.of(qmcgen.make_functor(cfg.seed, cfg.L, cfg.m))
        self.R = q.gen_positions(self.seed, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32)
        k = qmcgen.make_k(self.seed, cfg.W, cfg.N)
        rt = qmcgen.make_trials(self.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32, P=self.P, mode=self.tmode)
        rk = qmcgen.make_trials(self.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32, mode="noop")
        self.k = torch.from_numpy(k).cuda()
        self.rt = torch.from_numpy(rt).cuda()
        self.ws = q.Workspace(q.workspace_size(cfg.W, self.P, cfg.N, torch.float32))
        self.V_cur = None
        if self.tmode != "drift":       # NLPP ratios are relative to the current U^2_k (the caller's 5N state)
            v0 = q.eval(self.R, self.k, torch.from_numpy(rk).cuda(), self.fn, cfg.N, cfg.n_up, workspace=self.ws)
            self.V_cur = v0[:, 0, 0].contiguous()
        self.out = torch.empty((cfg.W, self.P, 5), dtype=torch.float64, device="cuda")
        self.ratio = torch.empty((cfg.W, self.P, 2), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

    def roofline(self, kms, peak_hbm):
        cfg = self.cfg
        hbm = self._alg() / (kms / 1e3) / 1e9
        return alu_roofline(self.mode, "j2_eval_kernel<float,false,2,3> (one trial per CTA, the P trials of a tile "
                            "on consecutive CTAs)", kms, cfg.W * self.P * (cfg.N - 1),
                            extra={"hbm": {"achieved": hbm, "peak": peak_hbm, "unit": "GB/s", "frac": hbm / peak_hbm,
                                           "alg_bytes_per_launch": self._alg()}})


class SweepPlan:
    """NEXT-2: one particle-by-particle move per walker and step on a C3 instance
    (Alg. 1 L5-L9 for the J2 factor): qj2_eval with P = 2 (U^2_k at r_k and
    r'_k in one pass, ratio e^{dJ2} fused) -> qj2_metropolis (u < rho^2) ->
    qj2_accept (R[:, k] and the 5N fp32 state of every partner).  Electron
    k = (k0 + s) mod N at step s (ordered sweep), inputs pre-drawn by qmcgen."""
    mode = "C3S"
    launches_per_step = 5      # eval kernel + ratio + metropolis + r_k gather + accept kernel (+ the counter memset)

    def __init__(self, cfg, rank, world):
        self.cfg = cfg
        self.seed = cfg.seed + rank
        self.items_per_step = cfg.W * (cfg.N - 1)
        self.s = 0

    def items_total(self, world):
        return self.items_per_step * world

    def prepare(self, q, n_steps):
        import torch
        import qmcgen
        cfg = self.cfg
        self.fn = q.Functor.of(qmcgen.make_functor(cfg.seed, cfg.L, cfg.m))
        self.R = q.gen_positions(self.seed, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32)
        self.S_ = torch.zeros((cfg.W, 5, cfg.Np), dtype=torch.float32, device="cuda")   # 5N state
        ks, tr, u = qmcgen.make_sweep(self.seed, cfg.W, cfg.N, cfg.L, np.float32, n_steps)
        self.ks, self.tr, self.u = (torch.from_numpy(ks).cuda(), torch.from_numpy(tr).cuda(),
                                    torch.from_numpy(u).cuda())
        self.n = n_steps
        self.ws = q.Workspace(q.workspace_size(cfg.W, 2, cfg.N, torch.float32))
        self.wsa = q.Workspace(4096 * 16)
        self.out = torch.empty((cfg.W, 2, 5), dtype=torch.float64, device="cuda")
        self.ratio = torch.empty((cfg.W, 2, 2), dtype=torch.float64, device="cuda")
        self.acc = torch.empty((cfg.W,), dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()

    def step(self, q, dist_mod):
        cfg = self.cfg
        s = self.s % self.n
        self.s += 1
        k = self.ks[s]
        q.eval(self.R, k, self.tr[s], self.fn, cfg.N, cfg.n_up, ratio=True, out=self.out,
               ratio_out=self.ratio, workspace=self.ws)
        if self.s == 1:               # the first move's values (the parity field's sample)
            self.first_out = self.out.clone()
        q.metropolis(self.ratio, self.u[s], self.acc, trial=1)
        q.accept(self.R, self.S_, k, self.tr[s], self.acc, self.out, self.fn, cfg.N, cfg.n_up, trial=1,
                 workspace=self.wsa)

    def kernel_ms(self, q, stream, reps):
        """The dominant kernel: qj2_accept on the last step's decisions (one
        launch per call with the caller's r_old)."""
        import torch
        cfg = self.cfg
        s = (self.s - 1) % self.n
        k = self.ks[s]
        r_old = self.tr[s][:, 0, :].contiguous()
        self.n_acc = int(self.acc.sum().item())
        torch.cuda.synchronize()
        return _event_ms(lambda: q.accept(self.R, self.S_, k, self.tr[s], self.acc, self.out, self.fn, cfg.N,
                                          cfg.n_up, trial=1, r_old=r_old), stream, reps)

    def gpu_sample(self, n):
        return self.first_out[:n].cpu().numpy()

    def e2e(self, q, steps, dist_mod):
        """Through the public API with host buffers: each step uploads its move (k, the
        (r_k, r'_k) pair, u) from pinned host memory and reads the step's results back
        (the (V, G, L) pair, the ratios and the decisions); R and the 5N state are the
        walkers' resident Markov-chain state (7.55 + 12.6 GB), not per-step inputs."""
        import torch
        cfg = self.cfg
        kh = [self.ks[s].cpu().pin_memory() for s in range(self.n)]
        th = [self.tr[s].cpu().pin_memory() for s in range(self.n)]
        uh = [self.u[s].cpu().pin_memory() for s in range(self.n)]
        kd, td, ud = torch.empty_like(self.ks[0]), torch.empty_like(self.tr[0]), torch.empty_like(self.u[0])
        oh = torch.empty(tuple(self.out.shape), dtype=torch.float64, pin_memory=True)
        rh = torch.empty(tuple(self.ratio.shape), dtype=torch.float64, pin_memory=True)
        ah = torch.empty(tuple(self.acc.shape), dtype=torch.int32, pin_memory=True)

        def run(i):
            s = i % self.n
            kd.copy_(kh[s], non_blocking=True)
            td.copy_(th[s], non_blocking=True)
            ud.copy_(uh[s], non_blocking=True)
            q.eval(self.R, kd, td, self.fn, cfg.N, cfg.n_up, ratio=True, out=self.out, ratio_out=self.ratio,
                   workspace=self.ws)
            q.metropolis(self.ratio, ud, self.acc, trial=1)
            q.accept(self.R, self.S_, kd, td, self.acc, self.out, self.fn, cfg.N, cfg.n_up, trial=1,
                     workspace=self.wsa)
            oh.copy_(self.out, non_blocking=True)
            rh.copy_(self.ratio, non_blocking=True)
            ah.copy_(self.acc, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        run(self.s)
        if dist_mod:
            dist_mod.barrier()
        t0 = time.perf_counter()
        for i in range(steps):
            run(self.s + 1 + i)
        dt = allreduce_max((time.perf_counter() - t0) / steps, dist_mod)
        world = dist_mod.get_world_size() if dist_mod else 1
        return {"value": self.items_per_step * world / dt, "unit": UNIT,
                "h2d_bytes_per_step": kh[0].numel() * 4 + th[0].numel() * 4 + uh[0].numel() * 8,
                "d2h_bytes_per_step": oh.numel() * 8 + rh.numel() * 8 + ah.numel() * 4, "ms_per_step": dt * 1e3,
                "steps": steps,
                "api": "qj2_eval + qj2_metropolis + qj2_accept with each step's move copied from pinned host memory "
                       "and its values, ratios and decisions read back (R and the 5N state resident)"}

    @property
    def alg_bytes_per_launch(self):
        # per accepted walker: x, y, z of every partner (12 B) + 5 fp32 state lanes read and written
        # (40 B) per partner, + k, accept, r_new, r_old, out_new row (4+4+12+12+40 B); 4 B accept flag
        # per rejected walker
        cfg = self.cfg
        return self.n_acc * ((cfg.N - 1) * 52 + 72) + (cfg.W - self.n_acc) * 4

class GraphSweepPlan(SweepPlan):
    """A full particle-by-particle sweep of the paper's NiO-64 size (N = 768,
    1024 walkers): N moves per walker (Alg. 1 L4-L9), each r'_k = wrap(r_k +
    delta) from the walker's current r_k -> U^2_k(R') on the fly -> ratio with
    the stored U^2_k(R) -> Metropolis -> on acceptance the update of R and the 5N
    state.  The timed step is ONE qj2_sweep launch (walkers resident in shared
    memory); consecutive steps continue the Markov chain from the evolved
    configuration (the state starts from qj2_state_init), with the moves of
    step i drawn from a pool of POOL pre-drawn sweeps.  For context prepare()
    also times one sweep's moves as per-move launches (qj2_eval + qj2_metropolis_
    accept, 2 per move), eagerly and captured in a CUDA graph."""
    mode = "N64S"
    flush_l2 = True                     # R, state and the moves (~53 MB) fit in L2
    # the roofline from separately timed sweeps (kernel_ms): a sweep's time depends on its
    # acceptance, which drifts along the chain, and the issue model needs the acceptance of
    # the very sweeps that were timed
    POOL = 4

    N_IONS = 64                         # NiO-64 (Table 1): 64 ions of 2 species

    def __init__(self, cfg, rank, world):
        super().__init__(cfg, rank, world)
        self.mode = cfg.name
        self.with_j1 = cfg.name == "N64SJ"
        self.S = cfg.N
        self.launches_per_step = 1
        self.items_per_step = self.S * cfg.W * (cfg.N - 1 + (self.N_IONS if self.with_j1 else 0))
        self.i = 0

    def prepare(self, q, n_steps=None):
        import torch
        import qmcgen
        cfg = self.cfg
        self.q = q
        self.fn = q.Functor.of(qmcgen.make_functor(cfg.seed, cfg.L, cfg.m))
        self.R = q.gen_positions(self.seed, cfg.W, cfg.N, cfg.Np, cfg.L, torch.float32)
        self.S_ = torch.zeros((cfg.W, 5, cfg.Np), dtype=torch.float32, device="cuda")
        self.j1 = None
        if self.with_j1:
            ions, start = qmcgen.make_ions(cfg.seed, self.N_IONS, self.N_IONS, cfg.L, np.float32, n_species=2)
            fn1 = q.J1Functor.of(qmcgen.make_j1_functor(cfg.seed, cfg.L, n_species=2))
            self.j1 = (torch.from_numpy(ions).cuda(), start, fn1,
                       torch.zeros((cfg.W, 5, cfg.Np), dtype=torch.float32, device="cuda"))
        q.state_init(self.R, self.S_, self.fn, cfg.N, cfg.n_up, j1=self.j1)       # untimed
        self.moves = [tuple(torch.from_numpy(a).cuda()
                            for a in qmcgen.make_sweep_moves(self.seed, cfg.W, cfg.N, self.S, stream=i))
                      for i in range(self.POOL)]
        self.acc_all = torch.empty((self.S, cfg.W), dtype=torch.int32, device="cuda")
        self.dj_all = torch.empty((self.S, cfg.W), dtype=torch.float64, device="cuda")
        # context: one sweep's moves as per-move launches on copies (pre-drawn (r_k, r'_k) pairs of an
        # ordered sweep from the start configuration), eager and as one CUDA graph
        pks, ptr, pu = qmcgen.make_sweep(self.seed, cfg.W, cfg.N, cfg.L, np.float32, self.S)
        self.pks, self.ptr, self.pu = torch.from_numpy(pks).cuda(), torch.from_numpy(ptr).cuda(), torch.from_numpy(pu).cuda()
        self.Rc, self.Sc = self.R.clone(), self.S_.clone()
        self.ws = q.Workspace(q.workspace_size(cfg.W, 2, cfg.N, torch.float32))
        self.out = torch.empty((cfg.W, 2, 5), dtype=torch.float64, device="cuda")
        self.acc = torch.empty((cfg.W,), dtype=torch.int32, device="cuda")
        for _ in range(2):
            self._per_move(q)
        torch.cuda.synchronize()
        self.eager_ms = _event_ms(lambda: self._per_move(q), torch.cuda.current_stream(), 1)
        graph = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            self._per_move(q)
        torch.cuda.current_stream().wait_stream(cs)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph):
            self._per_move(q)
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        self.graph_ms = _event_ms(lambda: graph.replay(), torch.cuda.current_stream(), 3)
        del graph, self.Rc, self.Sc
        log(f"[bench] {self.mode}: per-move launches {self.eager_ms:.3f} ms eager, {self.graph_ms:.3f} ms as one CUDA "
            f"graph ({self.S} moves x 2 launches); the timed step is one qj2_sweep launch")
        torch.cuda.synchronize()

    def _per_move(self, q):
        cfg = self.cfg
        for s in range(self.S):
            k = self.pks[s]
            q.eval(self.Rc, k, self.ptr[s], self.fn, cfg.N, cfg.n_up, out=self.out, workspace=self.ws)
            q.metropolis_accept(self.Rc, self.Sc, k, self.ptr[s], self.out, self.pu[s], self.fn, cfg.N, cfg.n_up,
                                acc=self.acc)

    def step(self, q, dist_mod):
        ks, dl, u = self.moves[self.i % self.POOL]
        self.i += 1
        q.sweep(self.R, self.S_, ks, dl, u, self.fn, self.cfg.N, self.cfg.n_up, acc=self.acc_all,
                dj=self.dj_all, j1=self.j1)
        if self.i == 1:               # the first sweep (from the start configuration): the parity sample
            self.first_acc = self.acc_all.cpu().numpy()
            self.first_dj = self.dj_all.cpu().numpy()
            self.first_R = self.R[:64].cpu().numpy()

    def e2e(self, q, steps, dist_mod):
        """Through the public API with host buffers: each step uploads the walkers'
        positions and 5N state (and J1 state), the sweep's moves (k, r_k, r'_k, u)
        from pinned memory, runs qj2_sweep and reads the accept flags back (the
        functor tables and the ions are model data, resident on the device)."""
        import torch
        cfg = self.cfg
        ks, dl, u = self.moves[0]
        dev = [self.R, self.S_, ks, dl, u] + ([self.j1[3]] if self.j1 else [])
        host = [t.cpu().pin_memory() for t in dev]
        dbuf = [torch.empty_like(t) for t in dev]
        acc_h = torch.empty(tuple(self.acc_all.shape), dtype=torch.int32, pin_memory=True)
        j1 = (self.j1[0], self.j1[1], self.j1[2], dbuf[5]) if self.j1 else None

        def run():
            for d, h in zip(dbuf, host):
                d.copy_(h, non_blocking=True)
            q.sweep(dbuf[0], dbuf[1], dbuf[2], dbuf[3], dbuf[4], self.fn, cfg.N, cfg.n_up, acc=self.acc_all,
                    dj=self.dj_all, j1=j1)
            acc_h.copy_(self.acc_all, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        run()
        if dist_mod:
            dist_mod.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            run()
        dt = allreduce_max((time.perf_counter() - t0) / steps, dist_mod)
        world = dist_mod.get_world_size() if dist_mod else 1
        return {"value": self.items_per_step * world / dt, "unit": UNIT,
                "h2d_bytes_per_step": sum(h.numel() * h.element_size() for h in host),
                "d2h_bytes_per_step": acc_h.numel() * 4, "ms_per_step": dt * 1e3, "steps": steps,
                "api": "qj2_sweep with R, the 5N state and the sweep's moves (k, delta, u) copied from pinned "
                       "host memory every step, accept flags read back"}

    @property
    def alg_bytes_per_launch(self):
        cfg = self.cfg
        return cfg.W * cfg.Np * 8 * 4 * 2 + self.S * cfg.W * (4 + 12 + 8 + 4 + 8)   # R + state in/out, moves

    def kernel_ms(self, q, stream, reps):
        return self.flusher.event_ms(lambda: self.step(q, None), stream, max(1, reps // 5))

    def roofline(self, kms, peak_hbm):
        cfg = self.cfg
        acc = (self.acc_all == 1).float().mean().item()    # acceptance of the last timed sweep
        # functor terms per move: N - 1 at r'_k, N - 1 more at r_k when accepted; J1: 2 per ion
        terms = self.S * cfg.W * ((cfg.N - 1) * (1.0 + acc) + (2 * self.N_IONS if self.with_j1 else 0))
        # the ncu-captured launch sits at another point of the chain (another acceptance): its
        # instructions split into a per-move and a per-accepted-move part (tools/sweep_model.py)
        # give this launch's count
        sm = kernel_record(self.mode).get("sweep_model")
        ti = None
        if sm:
            per_mp = sm["per_move_partner"] + acc * sm["per_accepted_move_partner"]
            ti = (self.S * cfg.W * cfg.N * per_mp,
                  f"ncu SASS source page split into per-move ({sm['per_move_partner']:.1f}) and per-accepted-move "
                  f"({sm['per_accepted_move_partner']:.1f}) thread instructions per (move, partner) "
                  f"(tools/sweep_model.py, profiles/r02/ncu_{self.mode}.json, captured at acceptance "
                  f"{sm['acceptance_captured']:.3f}), at this launch's acceptance: {per_mp:.1f}")
        return alu_roofline(self.mode, "j2_sweep_kernel (one launch per sweep, walkers resident in shared memory"
                            + (", J1 over 64 ions in every move)" if self.with_j1 else ")"), kms, terms,
                            extra={"acceptance": acc, "per_move_launches_eager_ms": self.eager_ms,
                                   "per_move_launches_graph_ms": self.graph_ms}, thread_inst=ti)


class SpoPlan:
    """NEXT-4: one Bspline-vgh + determinant ratio per walker (qj2_spo_eval) over a
    NiO-64-shaped shared table; item = one (walker, orbital) pair."""
    mode = "S1"
    launches_per_step = 1
    roofline_from_timed = True  # a step is the spo_eval launch

    def __init__(self, cfg, rank, world):
        self.cfg = cfg
        self.mode = cfg.name
        self.seed = cfg.seed + rank
        self.nlpp = cfg.name == "S1V"                 # Bspline-v at 12 quadrature points per walker
        self.ppw = 12 if self.nlpp else 1
        self.items_per_step = cfg.W * self.ppw * cfg.n_orb

    def items_total(self, world):
        return self.items_per_step * world

    @property
    def alg_bytes_per_launch(self):
        cfg = self.cfg
        # per evaluation the position and the 5 fp64 outputs; per walker the A^{-1} row and the
        # DISTINCT coefficient rows of n_orb fp32 its points need: 64 for one point (S1); for the 12
        # NLPP points of a walker (S1V) the union of their 4x4x4 control blocks, since points of one
        # walker that share a row need it once (counted from the positions: self.rows_per_walker)
        rows = 64 * cfg.W if not self.nlpp else self.unique_rows
        return rows * cfg.n_orb * 4 + cfg.W * self.ppw * (12 + 40) + cfg.W * cfg.n_orb * 4

    def _count_unique_rows(self, pts):
        """Distinct (ix, iy, iz) control rows per walker over its points [W][ppw][3] (the
        table's uniform periodic grid, reading R22), summed over walkers."""
        cfg = self.cfg
        n = np.array([cfg.nx, cfg.ny, cfg.nz])
        u = np.mod(pts.astype(np.float64), cfg.L) / cfg.L * n
        i = np.minimum(np.floor(u).astype(np.int64), n - 1)                      # [W][ppw][3]
        off = np.arange(-1, 3)
        ix = np.mod(i[..., 0, None] + off, n[0])
        iy = np.mod(i[..., 1, None] + off, n[1])
        iz = np.mod(i[..., 2, None] + off, n[2])
        flat = ((ix[..., :, None, None] * n[1] + iy[..., None, :, None]) * n[2] + iz[..., None, None, :])
        flat = flat.reshape(pts.shape[0], -1)
        flat.sort(axis=1)
        return int((np.diff(flat, axis=1) != 0).sum() + flat.shape[0])

    def prepare(self, q):
        import torch
        import qmcgen
        cfg = self.cfg
        self.coef = q.gen_spo_table(cfg.seed, cfg.nx, cfg.ny, cfg.nz, cfg.n_orb, cfg.ld)
        self.tab = q.SpoTable(self.coef, cfg.n_orb, cfg.L)
        if self.nlpp:
            k = qmcgen.make_k(self.seed, cfg.W, cfg.N)
            pts = qmcgen.make_trials(self.seed, np.arange(cfg.W), k, cfg.N, cfg.L, np.float32, P=12, mode="nlpp")
            self.pos = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
            self.unique_rows = self._count_unique_rows(pts)
        else:
            self.pos = torch.from_numpy(qmcgen.spo_positions(self.seed, cfg.W, cfg.L)).cuda()
        self.A = torch.from_numpy(qmcgen.make_ainv_rows(self.seed, cfg.W, cfg.n_orb)).cuda()
        self.out = torch.empty((cfg.W * self.ppw, 5), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

    def step(self, q, dist_mod):
        if self.nlpp:
            q.spo_eval(self.tab, self.pos, vgh=False, Ainv=self.A, all_trials=True, out=self.out)
        else:
            q.spo_eval(self.tab, self.pos, Ainv=self.A, out=self.out)

    def kernel_ms(self, q, stream, reps):
        return _event_ms(lambda: self.step(q, None), stream, reps)

    def gpu_sample(self, n):
        return self.out[:n].cpu().numpy()

    def e2e(self, q, steps, dist_mod):
        """Through the public API with host buffers: each step uploads the walkers'
        positions and A^{-1} rows from pinned memory and reads the ratios back (the
        shared table is model data, resident on the device)."""
        import torch
        cfg = self.cfg
        ph = self.pos.cpu().pin_memory()
        ah = self.A.cpu().pin_memory()
        oh = torch.empty((cfg.W * self.ppw, 5), dtype=torch.float64, pin_memory=True)
        pd, ad = torch.empty_like(self.pos), torch.empty_like(self.A)

        def run():
            pd.copy_(ph, non_blocking=True)
            ad.copy_(ah, non_blocking=True)
            if self.nlpp:
                q.spo_eval(self.tab, pd, vgh=False, Ainv=ad, all_trials=True, out=self.out)
            else:
                q.spo_eval(self.tab, pd, Ainv=ad, out=self.out)
            oh.copy_(self.out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        run()
        if dist_mod:
            dist_mod.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            run()
        dt = allreduce_max((time.perf_counter() - t0) / steps, dist_mod)
        world = dist_mod.get_world_size() if dist_mod else 1
        return {"value": self.items_per_step * world / dt, "unit": UNIT,
                "h2d_bytes_per_step": ph.numel() * 4 + ah.numel() * 4, "d2h_bytes_per_step": oh.numel() * 8,
                "ms_per_step": dt * 1e3, "steps": steps,
                "api": "qj2_spo_eval with positions and A^-1 rows copied from pinned host memory every step "
                       "(the shared table stays resident)"}


class J1Plan:
    """NEXT-1: one qj2_eval_j1 launch over a full sweep's trial points (ions in
    shared memory, one thread per trial point).  Issue-bound: ALU roofline."""
    mode = "J1S"
    launches_per_step = 1
    flush_l2 = True                     # trial points + outputs (~41 MB) fit in L2
    roofline_from_timed = True          # a step is the eval_j1 launch

    def __init__(self, cfg, rank, world):
        self.cfg = cfg
        self.rank = rank
        self.items_per_step = cfg.W * cfg.n_ions

    def items_total(self, world):
        return self.items_per_step * world

    @property
    def alg_bytes_per_launch(self):
        cfg = self.cfg
        return cfg.W * (12 + 40 + 16) + cfg.n_ions * 12

    def prepare(self, q):
        import torch
        cfg = self.cfg
        ions, self.start, rt, fn1 = j1_inputs(cfg, rank=self.rank)
        self.fn1 = q.J1Functor.of(fn1)
        self.ions = torch.from_numpy(ions).cuda()
        self.rt = torch.from_numpy(rt).cuda()
        self.out = torch.empty((cfg.W, 1, 5), dtype=torch.float64, device="cuda")
        self.ratio = torch.empty((cfg.W, 1, 2), dtype=torch.float64, device="cuda")
        self.V_cur = torch.zeros((cfg.W,), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

    def step(self, q, dist_mod):
        q.eval_j1(self.ions, self.start, self.rt, self.fn1, V_cur=self.V_cur, ratio=True, out=self.out,
                  ratio_out=self.ratio)

    def kernel_ms(self, q, stream, reps):
        return self.flusher.event_ms(lambda: self.step(q, None), stream, reps)

    def roofline(self, kms, peak_hbm):
        cfg = self.cfg
        return alu_roofline("J1S", "j1_thread_kernel<float>", kms, cfg.W * cfg.n_ions)

    def gpu_sample(self, n):
        return self.out[:n].cpu().numpy()

    def e2e(self, q, steps, dist_mod):
        """Through the public API with host buffers: each step uploads the sweep's
        trial points from pinned memory, runs qj2_eval_j1 (ratio fused) and reads
        the (V, G, L) rows and ratios back (the ions are model data, resident)."""
        import torch
        cfg = self.cfg
        rh = self.rt.cpu().pin_memory()
        rd = torch.empty_like(self.rt)
        oh = torch.empty(tuple(self.out.shape), dtype=torch.float64, pin_memory=True)
        qh = torch.empty(tuple(self.ratio.shape), dtype=torch.float64, pin_memory=True)

        def run():
            rd.copy_(rh, non_blocking=True)
            q.eval_j1(self.ions, self.start, rd, self.fn1, V_cur=self.V_cur, ratio=True, out=self.out,
                      ratio_out=self.ratio)
            oh.copy_(self.out, non_blocking=True)
            qh.copy_(self.ratio, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        run()
        if dist_mod:
            dist_mod.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            run()
        dt = allreduce_max((time.perf_counter() - t0) / steps, dist_mod)
        world = dist_mod.get_world_size() if dist_mod else 1
        return {"value": self.items_per_step * world / dt, "unit": UNIT,
                "h2d_bytes_per_step": rh.numel() * 4, "d2h_bytes_per_step": (oh.numel() + qh.numel()) * 8,
                "ms_per_step": dt * 1e3, "steps": steps,
                "api": "qj2_eval_j1 with the trial points copied from pinned host memory every step, (V, G, L) "
                       "and the ratios read back"}


def make_plan(cfg, rank, world):
    if cfg.name in ("N64S", "N64SJ"):
        return GraphSweepPlan(cfg, rank, world)
    if cfg.name.startswith("J"):
        return J1Plan(cfg, rank, world)
    if cfg.name.startswith("S"):
        return SpoPlan(cfg, rank, world)
    if cfg.name in ("C3P2", "C3P12"):
        return MultiTrialPlan(cfg, rank, world)
    if cfg.name == "C3S":
        return SweepPlan(cfg, rank, world)
    if cfg.name in ("C1", "C2", "C2f64", "C3", "C3f64"):
        return EvalPlan(cfg, rank, world)
    if cfg.name == "C4":
        return C4Plan(cfg, rank, world)
    if cfg.name == "C5":
        return C5Plan(cfg, rank, world)
    raise NotImplementedError(cfg.name)


def plan_kernel_name(plan):
    return {"C3S": "j2_accept_kernel<float>", "S1": "spo_tma_kernel<vgh>", "S1V": "spo_tma_kernel<v>",
            "C4": "j2_eval_warp_kernel<float> (one warp per walker, compact masked loop)",
            "C5": "j2_eval_kernel<float> (CTA tiles, cross-CTA fp64 partials)"}.get(plan.mode, "j2_eval_kernel<float>")


def _plain_rel(gpu, orc, absout):
    """max |gpu - orc| / |orc| over components with |orc| >= 1e-3 A."""
    m = (np.abs(orc) >= 1e-3 * absout) & (np.abs(orc) > 0)
    if not m.any():
        return None
    return float(np.max(np.abs(np.asarray(gpu, np.float64)[m] - orc[m]) / np.abs(orc[m])))


def parity_field(cfg, plan, smp):
    """Sampled parity of this run's GPU outputs against the oracle sample the
    cpu_baseline leg just ran (the same walkers [0, n) of rank 0's instance, the
    same seeded inputs), computed outside the timed region: the max normalized
    error of DESIGN.md section 4 and the max plain relative error."""
    import oracle
    n = smp.n
    try:
        if cfg.name in ("N64S", "N64SJ"):
            R2, S2, own, dj, _ = smp.result
            acc = plan.first_acc[:, :n]
            ok = acc >= 0
            rho2 = np.exp(2.0 * dj)
            clear = ok & (np.abs(smp.us - rho2) > 1e-3 * rho2)
            scale = np.maximum(np.abs(S2[:, 0, :cfg.N]).max(1), 1.0)[None, :]
            e = np.abs(plan.first_dj[:, :n] - dj) / scale
            return {"walkers": n, "moves": int(acc.shape[0]), "max_normalized_dj_err": float(e[ok].max()),
                    "decisions_agree_where_clear": bool(np.array_equal(acc[clear], own[clear])),
                    "positions_bitwise": bool(np.array_equal(plan.first_R[:n, :, :cfg.N], R2[:, :, :cfg.N])),
                    "what": "the oracle replays the first timed-run sweep of walkers [0, n) on the GPU's decisions"}
        if cfg.name.startswith("S"):
            out, aab, ab = smp.result
            g = plan.gpu_sample(out.shape[0])
            T = smp.T
            s = np.array((cfg.nx, cfg.ny, cfg.nz), np.float64) / cfg.L
            F = np.abs(T).max() * np.array([1, s[0], s[1], s[2], s[0] ** 2, s[0] * s[1], s[0] * s[2], s[1] ** 2,
                                            s[1] * s[2], s[2] ** 2])
            scale = np.maximum(aab, oracle.det_ratio_scale(smp.A, ab, F))
            e0 = np.abs(g[:, 0] - out[:, 0]) / scale[:, 0]
            e = e0.max()
            if cfg.name != "S1V":       # Bspline-vgh: also the numerators rho G and rho L (S1V computes rho only)
                e = max(e, (np.abs(g[:, 1:] * g[:, :1] - out[:, 1:] * out[:, :1]) / scale[:, 1:]).max())
            return {"evaluations": int(out.shape[0]), "max_normalized_err": float(e),
                    "max_plain_rel_err_rho": _plain_rel(g[:, 0], out[:, 0], aab[:, 0])}
        out, ab = smp.result
        g = plan.gpu_sample(out.shape[0])
        if cfg.name.startswith("J"):
            e = oracle.normalized_error_j1(g, out, ab, smp.fn1)
        else:
            e = oracle.normalized_error(g, out, ab, smp.fn)
        pr = {"walkers": int(out.shape[0]), "max_normalized_err": float(e.max()),
              "max_plain_rel_err": _plain_rel(g, out, ab)}
        for c, name in enumerate(("V", "Gx", "Gy", "Gz", "L")):
            pr[f"max_plain_rel_err_{name}"] = _plain_rel(g[..., c], out[..., c], ab[..., c])
        return pr
    except Exception as exc:        # the parity field must never take the bench line down
        return {"error": repr(exc)}


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if world != args.gpus:
        log(f"[bench] warning: --gpus {args.gpus} but WORLD_SIZE {world}")
    device = 0 if args.same_device else local
    torch.cuda.set_device(device)
    dist_mod = dist_init(world, device, args.dist_backend)
    import qmcgen
    import paper_1708_02645_b200 as q
    q.device_check()
    cfg = qmcgen.config(config_name(args, world))
    if cfg.name == "C4" and args.c4_instances:
        import dataclasses
        cfg = dataclasses.replace(cfg, instances=args.c4_instances)

    plan = make_plan(cfg, rank, world)
    if args.row:
        if not isinstance(plan, EvalPlan) or isinstance(plan, MultiTrialPlan):
            raise SystemExit("--row applies to C1, C2, C2f64, C3, C3f64")
        plan.row = True
    nvtx = torch.cuda.nvtx                            # phase ranges for nsys / ncu --nvtx
    with nvtx.range(f"prepare {cfg.name}"):
        if plan.mode in ("N64S", "N64SJ"):
            plan.prepare(q)                           # state_init, pools of pre-drawn moves
        elif plan.mode == "C3S":                      # pre-drawn sweep inputs for every step
            plan.prepare(q, args.warmup + 2 * args.steps + 2)
        else:
            plan.prepare(q)                           # device-resident inputs (generation untimed)

    stream = torch.cuda.current_stream()
    with nvtx.range("warmup"):
        for _ in range(args.warmup):
            plan.step(q, dist_mod)
        torch.cuda.synchronize()

    flusher = L2Flusher() if getattr(plan, "flush_l2", False) else None

    timed_spans = []

    def timed(K):
        if dist_mod:
            dist_mod.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(device) as clk:
            if flusher is not None:          # inputs < L2: flush before every step, time steps alone
                ms = flusher.event_ms(lambda: plan.step(q, dist_mod), stream, K, spans=timed_spans)
            else:
                # an event between consecutive steps: the same K-step span, and each step's own span
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
                evs[0].record(stream)
                for i in range(K):
                    plan.step(q, dist_mod)
                    evs[i + 1].record(stream)
                torch.cuda.synchronize()
                ms = evs[0].elapsed_time(evs[K]) / K
                timed_spans[:] = [evs[i].elapsed_time(evs[i + 1]) for i in range(K)]
        if dist_mod:
            dist_mod.barrier()
        return ms, clk

    run_timed = (lambda K: plan.timed(K, stream, device, dist_mod)) if hasattr(plan, "timed") else timed
    with nvtx.range(f"timed {args.steps} steps"):
        ms, clk = run_timed(args.steps)
    if clk.rejected():
        log(f"[bench] clocks rejected ({clk.summary()}); re-measuring once")
        ms, clk = run_timed(args.steps)
    ms_max = allreduce_max(ms, dist_mod)
    items_total = plan.items_total(world)
    value = items_total / (ms_max / 1e3)

    # roofline of the dominant kernel, timed on its launching stream: where a step is that
    # kernel's launch (plus at most a 4 KB counter memset and a W-thread ratio kernel), the mean
    # of the timed region's per-step spans; otherwise (several large kernels per step) the
    # kernel alone, launched back to back after the timed region.  The back-to-back figure is
    # reported beside it either way.
    plan.flusher = flusher
    with nvtx.range("kernel_ms"):
        kms_b2b = plan.kernel_ms(q, stream, reps=max(5, min(args.steps, 50)))
    if getattr(plan, "roofline_from_timed", False) and timed_spans:
        kms = float(np.mean(timed_spans))
        kms_how = f"timed region: mean of the {len(timed_spans)} per-step event spans"
    else:
        kms = kms_b2b
        kms_how = ("timed region: the wave launches' spans" if hasattr(plan, "timed") else
                   "the dominant kernel alone, after the timed region")
    alg_bytes = plan.alg_bytes_per_launch
    peak, peak_src = measured_peaks()
    achieved = alg_bytes / (kms / 1e3) / 1e9
    traffic = committed_traffic(cfg.name)

    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        with nvtx.range("e2e"):
            e2e = plan.e2e(q, args.e2e_steps, dist_mod)

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = cpu_cores()
        nw = args.cpu_sample_walkers or oracle_sample_size(cfg, cores, 15.0)[0]
        smp = make_oracle_sample(cfg, nw, cores)
        if cfg.name in ("N64S", "N64SJ"):
            smp.forced = plan.first_acc[:, :smp.n]
        dt = smp.run()
        used = 1 if cfg.name[0] in "SJ" else cores
        cpu = {"value": smp.items / dt, "unit": UNIT, "cores": used, "kind": "oracle",
               "sample": f"{smp.n} of {cfg.W} walkers of {cfg.name} (N={cfg.N}, {_what(cfg)}), one pass, "
                         f"{'fp64' if getattr(cfg, 'dtype', 'f32') == 'f64' else 'fp32'} inputs (promoted exactly to fp64), plain C "
                         f"oracle, {used} threads ({cpu_model()}), {dt:.1f} s wall"}
        parity = parity_field(cfg, plan, smp)
        # the T = 1 oracle on a sub-sample, for the per-core rate
        if used > 1:
            n1 = max(1, min(smp.n, 4 if cfg.N > 100000 else 16))
            s1 = make_oracle_sample(cfg, n1, 1)
            dt1 = s1.run()
            cpu["single_thread"] = {"value": s1.items / dt1, "unit": UNIT, "cores": 1,
                                    "sample": f"{s1.n} walkers, one thread, {dt1:.2f} s wall"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong" if plan.mode in ("C4", "C5") else "weak",
            "vs_baseline": None, "dtype": getattr(cfg, "dtype", "f32"), "data": "synthetic",
            "config": dict(workload_config(cfg, world), **({"row_out": "r, dx, dy, dz per item (SoA)"} if args.row
                                                           else {})),
            "roofline": dict(plan.roofline(kms, peak) if hasattr(plan, "roofline") else
                             {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                              "frac": achieved / peak, "traffic": traffic,
                              "kernel": plan_kernel_name(plan), "kernel_ms": kms,
                              "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src},
                             kernel_ms_source=kms_how, kernel_ms_back_to_back=kms_b2b),
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": e2e,
            "gpu_launches": plan.launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        if getattr(plan, "span", None):
            line["spans"] = plan.span
        print(json.dumps(line), flush=True)
    if dist_mod:
        dist_mod.barrier()
        dist_mod.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
