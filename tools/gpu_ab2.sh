mkdir -p gpurun_out
export AB_VARIANTS=default
for lib in paper_1708_02645_b200/libqmcj2.so abtest/libqmcj2_sub8.so; do
  echo "== $lib" >> gpurun_out/ab2.txt
  QJ2_LIB=$lib timeout 600 python tools/ab_multitrial.py 1 2 12 2>> gpurun_out/ab2.txt > /dev/null
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:j2_eval -s 3 -c 1 -o gpurun_out/c3p12_fast python bench.py --config C3P12 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
