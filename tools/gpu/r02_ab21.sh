# A/B: 256-bit loads in the CTA kernel's clean fp32 sub-tiles (C3, C5, C3P2, C3P12), parity
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build21.log 2>&1
for v in "-DQJ2_EVAL_V8=1" "-DQJ2_EVAL_V8=1 -DQJ2_EVAL_PF=4 -DQJ2_EVAL_MINB=2"; do
  timeout 900 python tools/ab/ab_build.py --config C3 --steps 30 -- $v 2>&1 | tail -2
done
timeout 900 python tools/ab/ab_build.py --config C5 --steps 10 -- -DQJ2_EVAL_V8=1 2>&1 | tail -2
timeout 900 python tools/ab/ab_build.py --config C3P2 --steps 30 -- -DQJ2_EVAL_V8=1 2>&1 | tail -2
timeout 900 python tools/ab/ab_build.py --config C3P12 --steps 10 -- -DQJ2_EVAL_V8=1 2>&1 | tail -2
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_EVAL_V8=1']))")
QJ2_LIB=$LIB timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_padding.py tests/test_gpu_cells.py -q -x -k "not slow" 2>&1 | tail -2
