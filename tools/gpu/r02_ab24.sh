# A/B: 256-bit loads/stores in the fp32 accept kernel (C3S), parity
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build24.log 2>&1
timeout 900 python tools/ab/ab_build.py --config C3S --steps 30 -- -DQJ2_ACCEPT_V8=1 2>&1 | tail -2
timeout 900 python tools/ab/ab_build.py --config C3S --steps 30 -- -DQJ2_ACCEPT_V8=1 2>&1 | tail -2
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_ACCEPT_V8=1']))")
QJ2_LIB=$LIB timeout 1200 python -m pytest tests/test_gpu_accept.py tests/test_gpu_randomized.py tests/test_gpu_padding.py tests/test_gpu_cells.py -q -x -k "accept" 2>&1 | tail -2
