mkdir -p gpurun_out
export AB_VARIANTS=default
rm -f gpurun_out/ab5.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_accept.py -x -q > gpurun_out/pytest_ab5.log 2>&1
for lib in abtest/libqmcj2_sub8.so paper_1708_02645_b200/libqmcj2.so; do
  echo "== $lib" >> gpurun_out/ab5.txt
  QJ2_LIB=$lib timeout 600 python tools/ab_multitrial.py 1 2 12 2>> gpurun_out/ab5.txt > /dev/null
done
