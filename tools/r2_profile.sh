# Round-2 evidence: launch list + ncu --set full of every kapsm kernel of one
# 1024-frame throughput pipeline launch and of one single-frame latency
# pipeline launch (tools/tp_launches.py).
set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2z_launches_tp.csv python tools/tp_launches.py 1024 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2z_launches_lat.csv python tools/tp_launches.py 1 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"band_kernel|screen_tc|apsm_train_tp|detect_finish" -s 0 -c 5 -o gpurun_out/r2z_full_tp python tools/tp_launches.py 1024 > gpurun_out/r2z_ncu_tp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pilot_gram|apsm_train_kernel|screen_tc|detect_finish" -s 0 -c 4 -o gpurun_out/r2z_full_lat python tools/tp_launches.py 1 > gpurun_out/r2z_ncu_lat.log 2>&1
ls -la gpurun_out | grep r2z
