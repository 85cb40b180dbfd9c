"""Summarise an ncu --set full report (raw page) into the metrics we track.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--json OUT.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum",
    "launch__grid_size", "launch__block_size",
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        kernels.append(d)
    return kernels


def main():
    rep = sys.argv[1]
    res = []
    for d in raw(rep):
        name = d.get("Kernel Name", ("?", ""))[0]
        m = {k: d[k][0] + (" " + d[k][1] if d[k][1] else "") for k in KEYS if k in d}
        stalls = {}
        for k in d:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(d[k][0].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        top = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
        res.append({"kernel": name, "metrics": m, "top_stalls": top})
    txt = json.dumps(res, indent=1)
    print(txt)
    if "--json" in sys.argv:
        open(sys.argv[sys.argv.index("--json") + 1], "w").write(txt)


if __name__ == "__main__":
    main()
