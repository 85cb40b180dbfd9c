# A/B: 256-bit loads (v4.f64) in the fp64 CTA kernel's clean sub-tiles (C3f64), parity
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build23.log 2>&1
timeout 900 python tools/ab/ab_build.py --config C3f64 --steps 30 -- -DQJ2_EVAL64_V8=1 2>&1 | tail -2
timeout 900 python tools/ab/ab_build.py --config C3f64 --steps 30 -- -DQJ2_EVAL64_V8=1 2>&1 | tail -2
timeout 900 python tools/ab/ab_build.py --config C3 --steps 30 -- -DQJ2_EVAL64_V8=1 2>&1 | tail -2
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_EVAL64_V8=1']))")
QJ2_LIB=$LIB timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_padding.py -q -x -k "not slow" 2>&1 | tail -2
