# A/B: J1 thread kernel compiled for 6 CTAs/SM (40 registers) vs 5 (48): the tail wave of J1S
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build15.log 2>&1
timeout 900 python tools/ab/ab_build.py --config J1S --steps 50 -- -DQJ2_J1_MINB=6 2>&1 | tail -2
timeout 900 python tools/ab/ab_build.py --config J1S --steps 50 -- -DQJ2_J1_MINB=6 2>&1 | tail -2
