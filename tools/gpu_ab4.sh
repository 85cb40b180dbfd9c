mkdir -p gpurun_out
export AB_VARIANTS=default
rm -f gpurun_out/ab4.txt
for lib in paper_1708_02645_b200/libqmcj2.so abtest/libqmcj2_sub8.so abtest/libqmcj2_sub16.so; do
  echo "== $lib" >> gpurun_out/ab4.txt
  QJ2_LIB=$lib timeout 600 python tools/ab_multitrial.py 1 2 12 2>> gpurun_out/ab4.txt > /dev/null
done
