# A/B: the shared-memory ring (cp.async) CTA kernel against the register pipeline (C3f64, C3, C3P2)
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build5.log 2>&1
for v in "-DQJ2_RING64=4 -DQJ2_RING64_MINB=2" "-DQJ2_RING64=4 -DQJ2_RING64_MINB=3"; do
  timeout 900 python tools/ab/ab_build.py --config C3f64 --steps 30 -- $v 2>&1 | tail -2
done
for v in "-DQJ2_RING32=4 -DQJ2_RING32_MINB=3" "-DQJ2_RING32=4 -DQJ2_RING32_MINB=4"; do
  timeout 900 python tools/ab/ab_build.py --config C3 --steps 30 -- $v 2>&1 | tail -2
done
for v in "-DQJ2_RING64=8 -DQJ2_RING64_MINB=2 -DQJ2_RING32=4 -DQJ2_RING32_MINB=3" "-DQJ2_RING64=4 -DQJ2_RING64_MINB=3 -DQJ2_RING32=8 -DQJ2_RING32_MINB=2"; do
  LIB=$(python -c "from paper_1708_02645_b200 import _build; print(_build.build(extra='$v'.split()))")
  echo "parity $v"
  QJ2_LIB=$LIB timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py -q -x -k "not slow" 2>&1 | tail -8
done
timeout 600 python -m pytest tests/test_gpu_j1.py -q -x -k thread_kernel_many 2>&1 | tail -2
