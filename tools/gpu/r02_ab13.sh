# A/B: warp kernel -- lane 0 prefetches the walker's later sub-tiles into L2 (C1, C2, C2f64, C4)
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build13.log 2>&1
for v in 2 8; do
  for c in C2 C2f64; do
    timeout 900 python tools/ab/ab_build.py --config $c --steps 50 -- -DQJ2_WARP_L2PF=$v 2>&1 | tail -2
  done
done
timeout 1500 python tools/ab/ab_build.py --config C4 --steps 3 -- -DQJ2_WARP_L2PF=8 2>&1 | tail -2
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_WARP_L2PF=8']))")
QJ2_LIB=$LIB timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py -q -x -k "not slow" 2>&1 | tail -2
