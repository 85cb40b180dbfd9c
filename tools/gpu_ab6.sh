mkdir -p gpurun_out
export AB_VARIANTS=default
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_accept.py tests/test_gpu_j1.py -x -q > gpurun_out/pytest_ab6.log 2>&1
timeout 900 python bench.py --config C4 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4.json 2>/dev/null
timeout 600 python tools/ab_multitrial.py 1 2 12 2> gpurun_out/ab6.txt > /dev/null
