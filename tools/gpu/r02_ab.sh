# A/B of compile-time kernel variants (tools/ab/ab_build.py): the warp kernel on one resident C4 wave,
# the fp64 CTA kernel on C3f64
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build.log 2>&1
for fl in "-DQJ2_EVAL64_PF=1 -DQJ2_EVAL64_MINB=2" "-DQJ2_EVAL64_PF=1 -DQJ2_EVAL64_MINB=3" "-DQJ2_EVAL64_PF=3 -DQJ2_EVAL64_MINB=1" "-DQJ2_EVAL64_PF=2 -DQJ2_EVAL64_MINB=1"; do
  timeout 1200 python tools/ab/ab_build.py --config C3f64 --steps 20 -- $fl 2>&1 | tail -2
done
for fl in "-DQJ2_WARP_PF=2 -DQJ2_WARP_MINB=3" "-DQJ2_WARP_PF=4 -DQJ2_WARP_MINB=2" "-DQJ2_WARP_PF=2 -DQJ2_WARP_MINB=2" "-DQJ2_ITERS=16"; do
  timeout 1200 python tools/ab/ab_build.py --config C4 --steps 10 --bench-args="--c4-instances 1024" -- $fl 2>&1 | tail -2
done
