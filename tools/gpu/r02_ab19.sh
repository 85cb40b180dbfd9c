# A/B: J1 thread kernel with its last, partial wave split TAIL lanes per unit (J1S), parity
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build19.log 2>&1
for v in 2 4; do
  timeout 900 python tools/ab/ab_build.py --config J1S --steps 50 -- -DQJ2_J1_TAIL_SPLIT=$v 2>&1 | tail -2
done
for v in 2 4; do
  LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_J1_TAIL_SPLIT=$v']))")
  QJ2_LIB=$LIB timeout 900 python -m pytest tests/test_gpu_j1.py -q -x 2>&1 | tail -2
done
timeout 900 python -m pytest tests/test_gpu_j1.py -q -x 2>&1 | tail -2
