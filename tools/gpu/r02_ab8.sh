# A/B: sweep tiers (64 x 4/8/12, 128 x 8) vs the product tiers across N, then parity of the variant
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build8.log 2>&1
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_SWEEP_T64=1']))")
for j in "" "--j1"; do
  timeout 600 python tools/ab/sweep_n.py $j 2>&1 | grep '^{'
  QJ2_LIB=$LIB timeout 600 python tools/ab/sweep_n.py $j 2>&1 | grep '^{'
done
QJ2_LIB=$LIB timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_randomized.py -q -x -k "sweep" 2>&1 | tail -2
