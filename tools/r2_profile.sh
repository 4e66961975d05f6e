# Throughput-mode evidence for round 2: launch list + ncu --set full of every
# kapsm kernel of one 1024-frame pipeline launch (tools/tp_launches.py).
set -x

timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2q_launches.csv python tools/tp_launches.py 1024 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"band_kernel|screen_tc|apsm_train_tp|detect_finish" -s 0 -c 5 -o gpurun_out/r2q_full python tools/tp_launches.py 1024 > gpurun_out/r2q_ncu.log 2>&1
tail -2 gpurun_out/r2q_ncu.log
