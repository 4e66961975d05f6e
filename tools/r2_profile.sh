# Round-2 evidence: launch list + ncu --set full of every kapsm kernel of one
# throughput pipeline launch (F = 1184 frames) and of one single-frame latency
# pipeline launch (tools/tp_launches.py), plus the band trainers of the
# single-frame C3 / C4-full-band configs (tools/cfg_time.py).  usage: TAG
T=${1:-r2f}
set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_tp.csv python tools/tp_launches.py 1184 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_lat.csv python tools/tp_launches.py 1 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"band_tile_kernel|screen_tc|apsm_train_tp|detect_finish" -s 0 -c 5 -o gpurun_out/${T}_full_tp python tools/tp_launches.py 1184 > gpurun_out/${T}_ncu_tp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pilot_gram|apsm_train_kernel|screen_tc|detect_finish" -s 0 -c 4 -o gpurun_out/${T}_full_lat python tools/tp_launches.py 1 > gpurun_out/${T}_ncu_lat.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"apsm_train_tpl" -s 0 -c 1 -o gpurun_out/${T}_full_c4fb python tools/cfg_time.py C4_full_band 1 > gpurun_out/${T}_ncu_c4fb.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"apsm_train_tpl" -s 0 -c 1 -o gpurun_out/${T}_full_c3 python tools/cfg_time.py C3_n2048_W64 1 > gpurun_out/${T}_ncu_c3.log 2>&1
ls -la gpurun_out | grep ${T}
