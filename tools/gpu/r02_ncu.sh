# launch lists + one `ncu --set full` capture of each configuration's dominant kernel (gpurun_out/ncu_r02/)
# each bench command ran to exit 0 without ncu first (r02_bench_all.sh); ncu numbers are never bench values
mkdir -p gpurun_out/ncu_r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu_r02/build.log 2>&1
if [ -z "$SKIP_LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed 5 steps/" --csv \
  --log-file gpurun_out/ncu_r02/launches_C3.csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launches C3 rc $?"
# N64S: the timed region only (its prepare() times 1536 per-move launches for context first)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed 3 steps/" --csv \
  --log-file gpurun_out/ncu_r02/launches_N64S.csv \
  python bench.py --config N64S --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launches N64S rc $?"
fi
cap() {  # config kernel-regex skip
  timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:$2 -s ${3:-3} -c 1 -o gpurun_out/ncu_r02/$1 \
    python bench.py --config $1 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r02/$1.log 2>&1
  echo "ncu $1 rc $?"
  python tools/ncu_summary.py gpurun_out/ncu_r02/$1.ncu-rep --json gpurun_out/ncu_r02/$1.json > /dev/null
  # gpurun brings back <= 64 MiB: keep the summary (and the SASS-level source page of the key kernels)
  case " ${KEEP_SRC:-C3 N64S N64SJ} " in *" $1 "*)
    ncu -i gpurun_out/ncu_r02/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_r02/$1_source.csv 2>/dev/null
    python tools/trim_source.py gpurun_out/ncu_r02/$1_source.csv gpurun_out/ncu_r02/$1_source_trim.csv;;
  esac
  rm -f gpurun_out/ncu_r02/$1.ncu-rep
}
# CAPS: config:kernel-regex[:skip] specs
for spec in ${CAPS:-C3:j2_eval_kernel C3f64:j2_eval_kernel C2:j2_eval_warp C2f64:j2_eval_warp C3P2:j2_eval_kernel C3P12:j2_eval_kernel C3S:j2_accept C4:j2_eval_warp C5:j2_eval_kernel S1:spo_tma S1V:spo_tma J1S:j1_thread N64S:j2_sweep N64SJ:j2_sweep}; do
  IFS=: read -r c k sk <<< "$spec"; cap $c $k $sk
done
