mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spo.py -q > gpurun_out/pytest_spo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spo.log
timeout 900 python bench.py --config S1V --steps 30 --warmup 5 > gpurun_out/bench_S1V.json 2> gpurun_out/bench_S1V.err
timeout 900 ncu -f --set full --clock-control none -k regex:spo_ -s 3 -c 1 -o gpurun_out/s1v_full python bench.py --config S1V --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
