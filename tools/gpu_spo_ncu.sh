mkdir -p gpurun_out
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:spo_ -s 3 -c 1 -o gpurun_out/s1_tma python bench.py --config S1 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_s1.log 2>&1
