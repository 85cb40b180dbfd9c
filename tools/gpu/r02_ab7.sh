# A/B: the sweep kernel at 64 threads x 12 partners per walker (N64S, N64SJ), and its parity
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build7.log 2>&1
for v in "-DQJ2_SWEEP_TPB64=1 -DQJ2_SWEEP_MINB64=7" "-DQJ2_SWEEP_TPB64=1 -DQJ2_SWEEP_MINB64=8"; do
  for c in N64S N64SJ; do
    timeout 900 python tools/ab/ab_build.py --config $c --steps 20 -- $v 2>&1 | tail -2
  done
done
v="-DQJ2_SWEEP_TPB64=1 -DQJ2_SWEEP_MINB64=7"
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra='$v'.split()))")
QJ2_LIB=$LIB timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x 2>&1 | tail -2
