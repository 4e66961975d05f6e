set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2f_tests.log 2>&1; tail -5 gpurun_out/r2f_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.log 2>&1; tail -c 1500 gpurun_out/r2f_bench.log
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
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"screen_tc" -s 1 -c 1 -o gpurun_out/r2f_screen_tc python /tmp/tp1.py 256 > gpurun_out/r2f_ncu.log 2>&1
tail -3 gpurun_out/r2f_ncu.log
