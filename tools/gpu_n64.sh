mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_accept.py -q -k "graph or sweep" > gpurun_out/pytest_n64.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_n64.log
timeout 900 python bench.py --config N64S --steps 10 --warmup 3 > gpurun_out/bench_N64S.json 2> gpurun_out/bench_N64S.err
