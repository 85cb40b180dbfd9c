set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
for c in C3 C3P2 C3P12 C3S; do
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "rc=$?" >> gpurun_out/bench_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:j2_eval -s 3 -c 1 -o gpurun_out/c3p12_full python bench.py --config C3P12 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c3p12.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:j2_eval -s 3 -c 1 -o gpurun_out/c3p2_full python bench.py --config C3P2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c3p2.log 2>&1
ls gpurun_out
