set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_accept.py -x -q > gpurun_out/pytest_accept.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_accept.log
timeout 600 python bench.py --config C3S --steps 50 --warmup 5 > gpurun_out/bench_c3s.json 2> gpurun_out/bench_c3s.err; echo "rc=$?" >> gpurun_out/bench_c3s.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3s.csv python bench.py --config C3S --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c3s.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:j2_accept -s 3 -c 1 -o gpurun_out/c3s_accept_full python bench.py --config C3S --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c3s.log 2>&1
ls -la gpurun_out
