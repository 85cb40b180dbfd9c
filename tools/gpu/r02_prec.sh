# the fp64-geometry path for fp32 functors finer than m = 16: its tests, the randomized campaign, perf at m = 8 unchanged
mkdir -p gpurun_out/prec
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/prec/build.log 2>&1 || { tail gpurun_out/prec/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_j1.py tests/test_gpu_accept.py -q -x -k "fine or larger_m or accept" 2>&1 | tail -3
for sh in 0 1 2 3 4 5 6 7 8; do
  QJ2_RANDOM_SHIFT=$sh timeout 1500 python -m pytest tests/test_gpu_randomized.py -q 2>&1 | tail -1 | sed "s/^/shift $sh: /"
done
timeout 900 python tools/ab/ab_build.py --config C3 --steps 30 -- -DQJ2_DUMMY_FLAG=1 2>&1 | tail -2
