mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spo.py -x -q > gpurun_out/pytest_spo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spo.log
timeout 900 python bench.py --config S1 --steps 50 --warmup 5 > gpurun_out/bench_S1.json 2> gpurun_out/bench_S1.err; echo "rc=$?" >> gpurun_out/bench_S1.err
timeout 900 ncu --set full --clock-control none --import-source on -f -k regex:spo_ -s 3 -c 1 -o gpurun_out/s1_full python bench.py --config S1 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_s1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches_s1.csv python bench.py --config S1 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
