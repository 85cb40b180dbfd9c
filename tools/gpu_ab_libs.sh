#!/bin/bash
# A/B of library builds: LIBS="name=path ..." CFGS="N64S ..." bench lines per build
mkdir -p gpurun_out
for cfg in ${CFGS:-N64S N64SJ}; do
  for spec in $LIBS; do
    name=${spec%%=*}; lib=${spec#*=}
    QJ2_LIB=$lib timeout 600 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${name}.json 2> gpurun_out/ab_${cfg}_${name}.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${cfg}_${name}.json'));print('$cfg $name', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"
  done
done
