# extended randomized parity campaign: the seeded randomized suite redrawn with shifts FROM..TO (default 1..5);
# PYTEST_K selects a subset
mkdir -p gpurun_out/campaign
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/campaign/build.log 2>&1
for sh in $(seq ${1:-1} ${2:-5}); do
  QJ2_RANDOM_SHIFT=$sh timeout 1500 python -m pytest tests/test_gpu_randomized.py -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/campaign/shift_$sh.log 2>&1
  tail -1 gpurun_out/campaign/shift_$sh.log | sed "s/^/shift $sh: /"
  grep -q " failed" gpurun_out/campaign/shift_$sh.log || rm -f gpurun_out/campaign/shift_$sh.log
done
