set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g1_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_randomized.py -k "sweep or state_init" -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/g1_pytest.log
timeout 600 python bench.py --config N64S --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/g1_n64s.json 2> gpurun_out/g1_n64s.err; echo "bench rc $?"
timeout 600 python bench.py --config N64SJ --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/g1_n64sj.json 2> gpurun_out/g1_n64sj.err; echo "bench rc $?"
cat gpurun_out/g1_n64s.json gpurun_out/g1_n64sj.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:j2_sweep_kernel -c 1 -o gpurun_out/g1_sweep python bench.py --config N64S --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g1_ncu.log 2>&1; echo "ncu rc $?"
