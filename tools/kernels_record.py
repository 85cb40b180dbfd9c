"""Collect the ncu summaries of each configuration's dominant kernel
(tools/gpu/r02_ncu.sh -> gpurun_out/ncu_r02/<config>.json, tools/ncu_summary.py)
into profiles/r02_kernels.json, the record bench.py reads for `roofline.traffic`
(DRAM read + write bytes per launch) and for the issue fraction of the ALU rows
(thread-instruction slots per launch = 32 x warp instructions, the unit of the
measured issue rate in profiles/r02_alu_peaks.json).

    python tools/kernels_record.py [gpurun_out/ncu_r02] [profiles/r02_kernels.json] [--only=C3,N64S]

With --only the named configurations' entries are replaced and the others kept.
The sweep configurations (N64S, N64SJ) also get their `sweep_model`
(tools/sweep_model.py) from the trimmed SASS source page <config>_source_trim.csv
when it is there.
"""
import json
import os
import re
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def num(v):
    m = re.match(r"([0-9.eE+-]+)\s*(\S*)", v.replace(",", ""))
    x = float(m.group(1))
    return x * UNITS.get(m.group(2), 1)


SWEEPS = {"N64S": (1024, 768, 768), "N64SJ": (1024, 768, 768)}   # W, S, N of the bench launch


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--only")]
    only = [a.split("=", 1)[1].split(",") for a in sys.argv[1:] if a.startswith("--only=")]
    only = set(only[0]) if only else None
    src = args[0] if len(args) > 0 else "gpurun_out/ncu_r02"
    out = args[1] if len(args) > 1 else "profiles/r02_kernels.json"
    rec = json.load(open(out)) if only and os.path.exists(out) else {}
    for f in sorted(os.listdir(src)):
        if not f.endswith(".json"):
            continue
        cfg = f[:-5]
        if only is not None and cfg not in only:
            continue
        d = json.load(open(os.path.join(src, f)))
        if not d:
            continue
        k = d[0]
        m = k["metrics"]
        t = num(m["gpu__time_duration.sum"].replace(" ms", "")) * 1e-3 if "ms" in m["gpu__time_duration.sum"] \
            else num(m["gpu__time_duration.sum"].replace(" us", "")) * 1e-6
        wi = num(m["smsp__inst_executed.sum"].split()[0])
        rec[cfg] = {
            "kernel": k["kernel"],
            "ncu_time_s": t,
            "dram_bytes_per_launch": num(m["dram__bytes_read.sum"]) + num(m["dram__bytes_write.sum"]),
            "warp_inst_per_launch": wi,
            "thread_inst_per_launch": 32 * wi,
            "issue_active_pct": num(m["smsp__issue_active.avg.pct_of_peak_sustained_active"].split()[0]),
            "warps_active_pct": num(m["sm__warps_active.avg.pct_of_peak_sustained_active"].split()[0]),
            "registers": num(m["launch__registers_per_thread"].split()[0]),
            "sm_clock_hz": num(m["sm__cycles_elapsed.avg.per_second"].split()[0]) * 1e9,
            "top_stalls": k.get("top_stalls", {}),
            "source": f"profiles/r02/ncu_{cfg}.json (ncu --set full --clock-control none, one launch of "
                      f"bench.py --config {cfg} --steps 4 --warmup 3)",
        }
        trim = os.path.join(src, f"{cfg}_source_trim.csv")
        if cfg in SWEEPS and os.path.exists(trim):
            sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
            from sweep_model import model
            m = model(trim, *SWEEPS[cfg])
            m.pop("kernel")
            m["source"] = f"profiles/r02/ncu_{cfg}_source.csv"
            rec[cfg]["sweep_model"] = m
    json.dump(rec, open(out, "w"), indent=1)
    for c, r in rec.items():
        print(f"{c:6s} {r['ncu_time_s'] * 1e3:8.3f} ms  dram {r['dram_bytes_per_launch'] / 1e9:8.3f} GB  "
              f"warp-inst {r['warp_inst_per_launch']:.3e}  issue {r['issue_active_pct']:.1f}%  "
              f"warps {r['warps_active_pct']:.1f}%  regs {r['registers']:.0f}  {r['top_stalls']}")


if __name__ == "__main__":
    main()
