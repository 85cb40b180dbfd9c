# A/B: short rows (C1, C2, C2f64) on the CTA kernel instead of the warp kernel
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build4.log 2>&1
for c in C1 C2 C2f64; do
  timeout 1200 python tools/ab/ab_build.py --config $c --steps 50 -- -DQJ2_WARP_SHORT_N=0 2>&1 | tail -2
done
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_WARP_SHORT_N=0']))")
QJ2_LIB=$LIB timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config_full or ragged or multi_trial" 2>&1 | tail -1
