# A/B: rows of 2-3 sub-tiles split over 2 warps at 128 registers (2 CTAs/SM, one wave at C2), parity
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build27.log 2>&1
for v in "-DQJ2_WARP_SPLIT=2 -DQJ2_WARP_SPLIT_PF=4" "-DQJ2_WARP_SPLIT=2 -DQJ2_WARP_SPLIT_PF=2"; do
  for c in C2 C2f64; do
    timeout 900 python tools/ab/ab_build.py --config $c --steps 50 -- $v 2>&1 | tail -2
  done
done
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra='-DQJ2_WARP_SPLIT=2 -DQJ2_WARP_SPLIT_PF=4'.split()))")
QJ2_LIB=$LIB timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_j1.py -q -x -k "not slow" 2>&1 | tail -2
