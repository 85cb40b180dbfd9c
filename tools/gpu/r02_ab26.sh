# A/B: the sweep kernel under a 144-register cap (64 x 12 keeps 7 CTAs/SM) instead of the launch bounds' 128
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build26.log 2>&1
for c in N64S N64SJ; do
  timeout 900 python tools/ab/ab_build.py --config $c --steps 20 -- -DQJ2_SWEEP_MAXNREG=144 2>&1 | tail -2
done
