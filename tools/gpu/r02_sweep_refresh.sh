# sweep kernel change: its parity tests, ncu captures (+ the per-move / per-accept instruction split into the
# record the bench reads), then the N64S / N64SJ bench lines and the N64S launch list
mkdir -p gpurun_out/ncu_r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sr_build.log 2>&1 || { tail gpurun_out/sr_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_randomized.py tests/test_gpu_check_build.py -x -q > gpurun_out/sr_pytest.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/sr_pytest.log
for c in N64S N64SJ; do   # each bench command exits 0 without ncu first
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "pre $c rc $?"
done
SKIP_LAUNCHES=1 KEEP_SRC="N64S N64SJ" CAPS="N64S:j2_sweep N64SJ:j2_sweep" bash tools/gpu/r02_ncu.sh
python tools/kernels_record.py gpurun_out/ncu_r02 profiles/r02_kernels.json --only=N64S,N64SJ
SKIP_ALU=1 CFGS="N64S N64SJ" bash tools/gpu/r02_bench_all.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed 3 steps/" --csv \
  --log-file gpurun_out/ncu_r02/launches_N64S.csv \
  python bench.py --config N64S --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launches N64S rc $?"
rm -f gpurun_out/ncu_r02/N64S_source.csv gpurun_out/ncu_r02/N64SJ_source.csv
