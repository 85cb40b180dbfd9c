"""Run tools/probe/alu_peaks.cu on the GPU box and write the measured ALU
ceilings (FP32 FFMA, FP64 DFMA, warp-instruction issue, MUFU.RSQ) with the SM
clock sampled by NVML during the run:

    python tools/probe/alu_peaks.py [out.json]      (default gpurun_out/alu_peaks.json)

bench.py reads the committed copy (profiles/r02_alu_peaks.json) for the
denominators of its ALU-bound roofline rows; DESIGN.md section 9 quotes it.
"""
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "alu_peaks.cu")
BIN = os.path.join(HERE, "alu_peaks")


def build():
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-o", BIN, SRC])


def issue_body():
    """SASS instructions per iteration of k_issue's loop (backward branch span)."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", BIN], capture_output=True, text=True).stdout
    block = sass.split("k_issue")[1].split("Function :")[0]
    for m in re.finditer(r"/\*([0-9a-f]{4})\*/\s+BRA(?:\.U)?\s+U?P\d+,\s*0x([0-9a-f]+)", block):
        at, tgt = int(m.group(1), 16), int(m.group(2), 16)
        if tgt < at:
            return (at - tgt) // 16 + 1
    raise RuntimeError("k_issue loop not found")


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/alu_peaks.json"
    build()
    body = issue_body()
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            time.sleep(0.005)
    t = threading.Thread(target=sample, daemon=True)
    t.start()
    r = subprocess.run([BIN, "5", str(body)], capture_output=True, text=True, check=True)
    stop.set()
    t.join()
    rows = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    meta = rows[-1]
    kern = {x["kernel"]: x for x in rows[:-1]}
    busy = [s for s in samples if s > 1000] or samples
    clk = statistics.median(busy) * 1e6
    sms = meta["sms"]
    res = {
        "what": "measured ALU ceilings of this B200 (tools/probe/alu_peaks.cu; best of 5 launches, grid = 8 CTAs x "
                "256 threads per SM, 8 independent chains per thread)",
        "sm_clock_mhz_median": clk / 1e6, "sms": sms, "issue_body_sass": body,
        "fp32_tflops": kern["ffma"]["per_s"] * 2 / 1e12,
        "fp64_tflops": kern["dfma"]["per_s"] * 2 / 1e12,
        "issue_tinst_per_s": kern["issue"]["per_s"] / 1e12,
        "rsqrt_t_per_s": kern["rsqrt"]["per_s"] / 1e12,
        "per_sm_per_clock": {"ffma_lanes": kern["ffma"]["per_s"] / (sms * clk),
                             "dfma_lanes": kern["dfma"]["per_s"] / (sms * clk),
                             "issue_thread_inst": kern["issue"]["per_s"] / (sms * clk),
                             "rsqrt_lanes": kern["rsqrt"]["per_s"] / (sms * clk)},
        "raw": rows,
    }
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "raw"}))


if __name__ == "__main__":
    main()
