"""Time a single-frame pipeline (C1 or one of bench.py's OTHER_CONFIGS) with
each trainer: AUTO, 1 Gram, 2 band (critical-warp form in latency mode),
3 band (plain one-warp form); CUDA events around one launch.
usage: python tools/cfg_time.py NAME [reps] [gram]"""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2201_05024_b200 as K

CFGS = dict(bench.OTHER_CONFIGS)
CFGS["C1"] = dict(K=6, M=16, n_train=685, n_data=3840, scheme="QPSK", W=20)
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = CFGS[name]
rx, pil, tx, _ = K.host_frames([3], c["K"], c["M"], c["n_train"], c["n_data"], c["scheme"])
p = K.FramePipeline(1, c["K"], c["M"], c["n_train"], c["n_data"], c["scheme"],
                    cfg=K.ApsmConfig(window=c["W"]), precision="f32", store_est=False,
                    full_workspace="gram" in sys.argv)
p.load(rx, pil, tx)
modes = [("auto", p.launch)] + [(f"mode{md}", (lambda md=md: p.launch_trainer(md))) for md in (1, 2, 3)]
for label, fn in modes:
    try:
        fn()
    except Exception as e:            # noqa: BLE001
        print(name, label, "unavailable:", str(e)[:80])
        continue
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    r = p.results()
    print(name, label, "us", [round(t) for t in ts], "bit_err", int(r["bit_err"].sum()),
          "atoms", r["n_active"][0].tolist()[:4], flush=True)
