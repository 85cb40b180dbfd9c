# extended randomized parity campaign: the seeded randomized suite redrawn with shifts 1..$1 (default 5)
mkdir -p gpurun_out/campaign
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/campaign/build.log 2>&1
for sh in $(seq 1 ${1:-5}); do
  QJ2_RANDOM_SHIFT=$sh timeout 1500 python -m pytest tests/test_gpu_randomized.py -q 2>&1 | tail -1 | sed "s/^/shift $sh: /"
done
