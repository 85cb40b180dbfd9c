# A/B: the V8 CTA kernel at 4 CTAs/SM (C3)
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build25.log 2>&1
for v in "-DQJ2_EVAL_MINB=4" "-DQJ2_EVAL_PF=1 -DQJ2_EVAL_MINB=4"; do
  timeout 900 python tools/ab/ab_build.py --config C3 --steps 30 -- $v 2>&1 | tail -2
done
