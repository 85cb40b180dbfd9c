# A/B: multi-trial fp32 J2 kernel (PT trials per CTA share each loaded vector) on C3P2 / C3P12 / C3S, and its parity
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build11.log 2>&1
for v in "-DQJ2_EVAL_PT=2" "-DQJ2_EVAL_PT=2 -DQJ2_EVAL_PT_PF=1" "-DQJ2_EVAL_PT=2 -DQJ2_EVAL_PT_PF=3"; do
  timeout 900 python tools/ab/ab_build.py --config C3P2 --steps 30 -- $v 2>&1 | tail -2
done
for v in "-DQJ2_EVAL_PT=2" "-DQJ2_EVAL_PT=3" "-DQJ2_EVAL_PT=4"; do
  timeout 900 python tools/ab/ab_build.py --config C3P12 --steps 20 -- $v 2>&1 | tail -2
done
timeout 900 python tools/ab/ab_build.py --config C3S --steps 30 -- -DQJ2_EVAL_PT=2 2>&1 | tail -2
for v in "-DQJ2_EVAL_PT=2" "-DQJ2_EVAL_PT=3"; do
  LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra='$v'.split()))")
  echo "parity $v"
  QJ2_LIB=$LIB timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_accept.py -q -x -k "not slow" 2>&1 | tail -2
done
