mkdir -p gpurun_out
timeout 900 python bench.py --config C4 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_warp.json 2> /dev/null
QJ2_NOWARP=1 timeout 900 python bench.py --config C4 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_cta.json 2> /dev/null
