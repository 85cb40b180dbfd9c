#!/bin/bash
# sweep kernel: parity tests + N64S / N64SJ bench lines (10 steps)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_accept.py -q -k "sweep" > gpurun_out/pytest_sweep.log 2>&1
tail -1 gpurun_out/pytest_sweep.log
for cfg in N64S N64SJ; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sw_${cfg}.json 2> gpurun_out/sw_${cfg}.err
  python -c "import json;d=json.load(open('gpurun_out/sw_${cfg}.json'));print('$cfg', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"
done
