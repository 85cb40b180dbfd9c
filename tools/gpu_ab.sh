set -x
mkdir -p gpurun_out
timeout 600 python tools/ab_multitrial.py 1 2 4 12 > gpurun_out/ab_multitrial.json 2> gpurun_out/ab_multitrial.err
QJ2_PB1=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:j2_eval -c 1 -o gpurun_out/p2pb1_full python tools/ab_multitrial.py 2 > /dev/null 2> gpurun_out/ncu_p2pb1.log
ls gpurun_out
