mkdir -p gpurun_out
export AB_VARIANTS=default
rm -f gpurun_out/ab3.txt
for lib in paper_1708_02645_b200/libqmcj2.so abtest/libqmcj2_it16.so; do
  echo "== $lib" >> gpurun_out/ab3.txt
  QJ2_LIB=$lib timeout 600 python tools/ab_multitrial.py 1 2 12 2>> gpurun_out/ab3.txt > /dev/null
done
QJ2_LIB=abtest/libqmcj2_it16.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_it16.log 2>&1
