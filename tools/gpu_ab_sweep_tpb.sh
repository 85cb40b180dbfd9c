#!/bin/bash
# A/B of the sweep kernel's threads per walker (QJ2_SWEEP_TPB) on N64S / N64SJ
mkdir -p gpurun_out
for tpb in ${TPBS:-128 96 64}; do
  QJ2_SWEEP_TPB=$tpb timeout 900 python -m pytest tests/test_gpu_accept.py -q -k "N64S or (sweep and 768)" > gpurun_out/pytest_sweep_$tpb.log 2>&1
  echo "tpb=$tpb $(tail -1 gpurun_out/pytest_sweep_$tpb.log)"
done
for cfg in N64S N64SJ; do
  for tpb in ${TPBS:-128 96 64}; do
    QJ2_SWEEP_TPB=$tpb timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${cfg}_${tpb}.json 2> gpurun_out/ab_${cfg}_${tpb}.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${cfg}_${tpb}.json'));print('$cfg tpb=$tpb', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"
  done
done
