# timed-region launch lists (NVTX-filtered) of N64S and N64SJ
mkdir -p gpurun_out/ncu_r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu_r02/build.log 2>&1
for c in N64S N64SJ; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "pre $c rc $?"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed 3 steps/" --csv \
    --log-file gpurun_out/ncu_r02/launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launches $c rc $?"
  grep -c "sweep" gpurun_out/ncu_r02/launches_$c.csv
done
