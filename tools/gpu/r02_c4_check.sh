mkdir -p gpurun_out/bench_r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bench_r02/build_c4.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py -q -x -k "warp or C4 or ragged or config_full or eval_random" 2>&1 | tail -2
for c in C4 C2 C2f64; do
  timeout 1500 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_r02/$c.json 2> gpurun_out/bench_r02/$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_r02/$c.json'));r=d['roofline'];print('$c',d['ms_per_step'],r['kernel_ms'],r['frac'],d['parity'].get('max_normalized_err'),d['clocks'])"
done
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:j2_eval_warp -s 3 -c 1 -o gpurun_out/bench_r02/C4 \
    python bench.py --config C4 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/bench_r02/C4.ncu-rep --json gpurun_out/bench_r02/ncu_C4.json > /dev/null; rm -f gpurun_out/bench_r02/C4.ncu-rep
