set -x
python tools/time_stages.py 256 C1 > gpurun_out/r2c_stages256.txt 2>&1
python tools/time_stages.py 1 C1 > gpurun_out/r2c_stages1.txt 2>&1
python tools/time_stages.py 16 C4 > gpurun_out/r2c_stages16_c4.txt 2>&1
cat > /tmp/tp1.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2201_05024_b200 as K
F = int(sys.argv[1])
rx, pil, tx, _ = K.host_frames(range(F), 6, 16, 685, 3840, "QPSK")
p = K.FramePipeline(F, 6, 16, 685, 3840, "QPSK", precision="f32", store_est=False)
p.load(rx, pil, tx)
p.launch(); p.launch(); torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_tp_launches.csv python /tmp/tp1.py 256 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"screen|apsm_train|finish|gram" -s 4 -c 4 -o gpurun_out/r2c_tp_full python /tmp/tp1.py 256 > gpurun_out/r2c_ncu.log 2>&1
ls -la gpurun_out
