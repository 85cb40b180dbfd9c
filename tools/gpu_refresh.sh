mkdir -p gpurun_out/refresh
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/refresh/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/refresh/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/refresh/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/refresh/smoke.log
timeout 900 python bench.py > gpurun_out/refresh/bench_C3.json 2> gpurun_out/refresh/bench_C3.err
for c in C3P2 C3P12 C3S S1 S1V J1S N64S N64SJ C5; do
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/refresh/bench_$c.json 2> gpurun_out/refresh/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/refresh/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:j2_eval -s 3 -c 1 -o gpurun_out/refresh/c3_full python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
