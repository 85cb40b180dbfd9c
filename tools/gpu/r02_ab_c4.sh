# A/B of the warp kernel's pipeline depth / residency on one resident C4 wave (1024 instances)
mkdir -p gpurun_out/ab_c4
for fl in "-DQJ2_WARP_PF=2 -DQJ2_WARP_MINB=3" "-DQJ2_WARP_PF=4 -DQJ2_WARP_MINB=2" "-DQJ2_WARP_PF=2 -DQJ2_WARP_MINB=2" "-DQJ2_ITERS=16"; do
  timeout 1200 python tools/ab/ab_build.py --config C4 --steps 10 --bench-args="--c4-instances 1024" -- $fl 2>&1 | tail -2
done
