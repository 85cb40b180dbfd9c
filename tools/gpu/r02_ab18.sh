# A/B: the NiO-64 sweep at 96 threads x 8 partners (7 CTAs/SM: 21 warps) vs 64 x 12 (14 warps)
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build18.log 2>&1
for c in N64S N64SJ; do
  timeout 900 python tools/ab/ab_build.py --config $c --steps 20 -- -DQJ2_SWEEP_T96=1 2>&1 | tail -2
done
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_SWEEP_T96=1']))")
QJ2_LIB=$LIB timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x 2>&1 | tail -2
