# quick A/B for the sweep kernel: parity subset + N64S/N64SJ bench lines (+ optional ncu)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/q_pytest.log
for c in N64S N64SJ; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err; echo "bench $c rc $?"
  python -c "import json;d=json.load(open('gpurun_out/q_$c.json'));r=d['roofline'];print('$c', d['ms_per_step'], r['kernel_ms'], r['frac'])"
done
if [ "$1" = "ncu" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:j2_sweep_kernel -s 2 -c 1 -o gpurun_out/q_sweep python bench.py --config N64S --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/q_ncu.log 2>&1; echo "ncu rc $?"
fi
