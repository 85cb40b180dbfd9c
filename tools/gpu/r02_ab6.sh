# A/B: fp64 rsqrt without ::rsqrt's out-of-range branch (product) -- C3f64 with the fp64 pipeline knobs, the ring
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build6.log 2>&1
for v in "-DQJ2_EVAL64_PF=3" "-DQJ2_EVAL64_PF=1 -DQJ2_EVAL64_MINB=3" "-DQJ2_RING64=8 -DQJ2_RING64_MINB=2"; do
  timeout 900 python tools/ab/ab_build.py --config C3f64 --steps 30 -- $v 2>&1 | tail -2
done
timeout 900 python tools/ab/ab_build.py --config C2f64 --steps 50 -- -DQJ2_EVAL64_PF=3 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_j1.py -q -x -k "not slow" 2>&1 | tail -2
