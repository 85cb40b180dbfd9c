mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_j1.py -x -q > gpurun_out/pytest_j1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_j1.log
timeout 900 python bench.py --config J1S --steps 50 --warmup 5 > gpurun_out/bench_J1S.json 2> gpurun_out/bench_J1S.err
QJ2_J1_WARP=1 timeout 900 python bench.py --config J1S --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_J1S_warp.json 2>/dev/null
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:j1_ -s 3 -c 1 -o gpurun_out/j1s_full python bench.py --config J1S --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_j1s.log 2>&1
