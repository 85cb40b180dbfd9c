# A/B: compact masked sub-tile loop in the warp kernel (icache) on C4 / C2 / C2f64, with its parity tests
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build3.log 2>&1
LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra=['-DQJ2_WARP_COMPACT_GEN=1']))")
QJ2_LIB=$LIB timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "warp or C4_full or ragged or config_full" 2>&1 | tail -2
timeout 1200 python tools/ab/ab_build.py --config C4 --steps 10 --bench-args="--c4-instances 1024" -- -DQJ2_WARP_COMPACT_GEN=1 2>&1 | tail -2
timeout 1200 python tools/ab/ab_build.py --config C2 --steps 50 -- -DQJ2_WARP_COMPACT_GEN=1 2>&1 | tail -2
timeout 1200 python tools/ab/ab_build.py --config C2f64 --steps 50 -- -DQJ2_WARP_COMPACT_GEN=1 2>&1 | tail -2
