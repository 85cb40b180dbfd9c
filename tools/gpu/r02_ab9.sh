# A/B: the warp kernel in small CTAs (1 / 2 / 4 warps) when its units fill fewer than 2 x 148 8-warp CTAs (C1, C2, C2f64)
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build9.log 2>&1
for w in 1 2 4; do
  for c in C1 C2 C2f64; do
    timeout 900 python tools/ab/ab_build.py --config $c --steps 50 -- -DQJ2_WARP_SMALL_WPC=$w 2>&1 | tail -2
  done
done
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_WARP_SMALL_WPC=2']))")
QJ2_LIB=$LIB timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_j1.py -q -x -k "not slow" 2>&1 | tail -2
