"""Collect the ncu summaries of each configuration's dominant kernel
(tools/gpu/r02_ncu.sh -> gpurun_out/ncu_r02/<config>.json, tools/ncu_summary.py)
into profiles/r02_kernels.json, the record bench.py reads for `roofline.traffic`
(DRAM read + write bytes per launch) and for the issue fraction of the ALU rows
(thread-instruction slots per launch = 32 x warp instructions, the unit of the
measured issue rate in profiles/r02_alu_peaks.json).

    python tools/kernels_record.py [gpurun_out/ncu_r02] [profiles/r02_kernels.json]
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


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu_r02"
    out = sys.argv[2] if len(sys.argv) > 2 else "profiles/r02_kernels.json"
    rec = {}
    for f in sorted(os.listdir(src)):
        if not f.endswith(".json"):
            continue
        cfg = f[:-5]
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
    json.dump(rec, open(out, "w"), indent=1)
    for c, r in rec.items():
        print(f"{c:6s} {r['ncu_time_s'] * 1e3:8.3f} ms  dram {r['dram_bytes_per_launch'] / 1e9:8.3f} GB  "
              f"warp-inst {r['warp_inst_per_launch']:.3e}  issue {r['issue_active_pct']:.1f}%  "
              f"warps {r['warps_active_pct']:.1f}%  regs {r['registers']:.0f}  {r['top_stalls']}")


if __name__ == "__main__":
    main()
