# ALU ceilings + one bench line per configuration (cpu_baseline, parity, e2e), logs in gpurun_out/bench_r02/
mkdir -p gpurun_out/bench_r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bench_r02/build.log 2>&1 || { tail gpurun_out/bench_r02/build.log; exit 1; }
if [ -z "$SKIP_ALU" ]; then
  python tools/probe/alu_peaks.py gpurun_out/bench_r02/alu_peaks.json; echo "alu rc $?"
  mkdir -p profiles && cp gpurun_out/bench_r02/alu_peaks.json profiles/r02_alu_peaks.json
fi
for c in ${CFGS:-C3 C1 C2 C2f64 C3f64 C3P2 C3P12 C3S C5 C4 S1 S1V J1S N64S N64SJ}; do
  steps=${STEPS:-30}
  timeout 1500 python bench.py --config $c --steps $steps --warmup 5 > gpurun_out/bench_r02/$c.json 2> gpurun_out/bench_r02/$c.err
  echo "bench $c rc $?"
  python - <<PY
import json
try:
    d=json.load(open('gpurun_out/bench_r02/$c.json'))
    r=d['roofline']; p=d.get('parity') or {}; e=d.get('e2e') or {}
    print('$c', round(d['ms_per_step'],4), '%.3e'%d['value'], r['bound'], round(r['frac'],3), 'cpu', (d.get('cpu_baseline') or {}).get('value'),
          'par', {k:v for k,v in p.items() if k.startswith('max')}, 'e2e', e.get('value'), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
except Exception as ex:
    print('$c parse failed', ex)
PY
done
