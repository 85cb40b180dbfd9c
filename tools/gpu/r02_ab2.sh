# A/B: persistent warps in the warp kernel (one C4 wave resident), plus fp64 variants if given
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build2.log 2>&1
for fl in ${AB_FLAGS:-"-DQJ2_WARP_PERSIST=1"}; do
  timeout 1200 python tools/ab/ab_build.py --config ${AB_CFG:-C4} --steps 10 --bench-args="${AB_ARGS:---c4-instances 1024}" -- $fl 2>&1 | tail -2
done
