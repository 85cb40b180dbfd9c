mkdir -p gpurun_out
export AB_VARIANTS=default
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_accept.py tests/test_gpu_j1.py -x -q > gpurun_out/pytest_ab7.log 2>&1
timeout 600 python tools/ab_multitrial.py 1 2 12 2> gpurun_out/ab7.txt > /dev/null
timeout 900 ncu -f --set full --clock-control none -k regex:j2_eval -s 3 -c 1 -o gpurun_out/c3x python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
