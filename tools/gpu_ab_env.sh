#!/bin/bash
# A/B of environment switches: ENVS="name=VAR=value ..." CFGS="N64S ..."; "base" = no variable
mkdir -p gpurun_out
for cfg in ${CFGS:-N64S}; do
  for spec in ${ENVS:-base}; do
    name=${spec%%=*}; kv=${spec#*=}
    if [ "$kv" = "base" ]; then envset=""; else envset="$kv"; fi
    env $envset timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abe_${cfg}_${name}.json 2> gpurun_out/abe_${cfg}_${name}.err
    python -c "import json;d=json.load(open('gpurun_out/abe_${cfg}_${name}.json'));print('$cfg $name', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"
  done
done
