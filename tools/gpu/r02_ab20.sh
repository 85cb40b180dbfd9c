# A/B: streaming-load cache hints of the fp32 kernels (C3, C4 wave)
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build20.log 2>&1
for v in 1 3; do
  timeout 900 python tools/ab/ab_build.py --config C3 --steps 30 -- -DQJ2_LD_HINT=$v 2>&1 | tail -2
done
timeout 1500 python tools/ab/ab_build.py --config C4 --steps 3 -- -DQJ2_LD_HINT=1 2>&1 | tail -2
