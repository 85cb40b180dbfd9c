# A/B: TMA L2 prefetch of the sub-tile QJ2_L2PF ahead in the CTA kernel (C3f64, C3, C5, C3P2)
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build12.log 2>&1
for v in 1 2 3; do
  timeout 900 python tools/ab/ab_build.py --config C3f64 --steps 30 -- -DQJ2_L2PF=$v 2>&1 | tail -2
done
for v in 1 2; do
  timeout 900 python tools/ab/ab_build.py --config C3 --steps 30 -- -DQJ2_L2PF=$v 2>&1 | tail -2
done
timeout 900 python tools/ab/ab_build.py --config C5 --steps 10 -- -DQJ2_L2PF=2 2>&1 | tail -2
timeout 900 python tools/ab/ab_build.py --config C3P2 --steps 30 -- -DQJ2_L2PF=2 2>&1 | tail -2
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_L2PF=2']))")
QJ2_LIB=$LIB timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py -q -x -k "not slow" 2>&1 | tail -2
