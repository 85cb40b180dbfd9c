# A/B: 256-bit loads in the compact warp kernel's clean sub-tiles (C4), parity
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build22.log 2>&1
timeout 1500 python tools/ab/ab_build.py --config C4 --steps 3 -- -DQJ2_WARP_V8=1 2>&1 | tail -2
timeout 1500 python tools/ab/ab_build.py --config C4 --steps 3 -- -DQJ2_WARP_V8=1 -DQJ2_WARP_PF=4 2>&1 | tail -2
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_WARP_V8=1']))")
QJ2_LIB=$LIB timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "warp or C4" 2>&1 | tail -2
