# A/B: fp64 CTA kernel residency / depth / rsqrt with the L2 prefetch in place (C3f64)
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build14.log 2>&1
for v in "-DQJ2_EVAL64_PF=1 -DQJ2_EVAL64_MINB=3" "-DQJ2_EVAL64_PF=1 -DQJ2_EVAL64_MINB=3 -DQJ2_L2PF64=2" "-DQJ2_RSQRT64_INLINE=1" "-DQJ2_RSQRT64_INLINE=1 -DQJ2_EVAL64_PF=1 -DQJ2_EVAL64_MINB=3" "-DQJ2_EVAL64_PF=3" "-DQJ2_L2PF64=2"; do
  timeout 900 python tools/ab/ab_build.py --config C3f64 --steps 30 -- $v 2>&1 | tail -2
done
