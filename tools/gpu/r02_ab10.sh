# A/B: J1 thread kernel -- lanes per unit (SPLIT) and threads per CTA (J1S), parity of the variants
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build10.log 2>&1
for v in "-DQJ2_J1_SPLIT=2" "-DQJ2_J1_SPLIT=4" "-DQJ2_J1_SPLIT=8"; do
  timeout 900 python tools/ab/ab_build.py --config J1S --steps 50 -- $v 2>&1 | tail -2
done
for v in "-DQJ2_J1_SPLIT=4" "-DQJ2_J1_SPLIT=8"; do
  LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra='$v'.split()))")
  echo "parity $v"
  QJ2_LIB=$LIB timeout 900 python -m pytest tests/test_gpu_j1.py tests/test_gpu_randomized.py -q -x -k "j1" 2>&1 | tail -2
done
