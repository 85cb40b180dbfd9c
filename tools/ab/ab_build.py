"""A/B of compile-time kernel variants: build the library with extra -D flags
(paper_1708_02645_b200/_build.py keys the objects and the library by the flags'
hash, so a variant never replaces the product build), then time one bench
configuration with it (QJ2_LIB) next to the product build.

    python tools/ab/ab_build.py --config C3 --steps 30 -- -DQJ2_EVAL_PF=1 -DQJ2_EVAL_MINB=4

Knobs (defaults in csrc/): QJ2_EVAL_PF / QJ2_EVAL_MINB (fp32 CTA kernel),
QJ2_WARP_PF / QJ2_WARP_MINB (warp kernel), QJ2_ITERS / QJ2_SUB (sub-tile
shape), QJ2_SPO_RING_KB (SPO ring budget per CTA).  j2_tma.cuh in this
directory is the TMA-pipelined eval kernel measured against the LDG kernel in
round 1 (52-60% of roofline) -- archived, not built.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--bench-args", default="", help="extra bench.py arguments, e.g. '--c4-instances 1024'")
    ap.add_argument("flags", nargs="*")
    a = ap.parse_args()
    from paper_1708_02645_b200 import _build
    libs = {"product": _build.build()}
    if a.flags:
        libs["variant"] = _build.build(extra=a.flags)
    for name, lib in libs.items():
        env = dict(os.environ, QJ2_LIB=lib)
        out = subprocess.run([sys.executable, "bench.py", "--config", a.config, "--steps", str(a.steps), "--warmup", "5",
                              "--no-cpu-baseline", "--no-e2e", *a.bench_args.split()], cwd=ROOT, env=env,
                             capture_output=True, text=True)
        d = json.loads(out.stdout.strip().splitlines()[-1])
        print(json.dumps({"build": name, "flags": a.flags if name == "variant" else [], "config": a.config,
                          "ms_per_step": d["ms_per_step"], "kernel_ms": d["roofline"]["kernel_ms"],
                          "frac": d["roofline"]["frac"]}))


if __name__ == "__main__":
    main()
