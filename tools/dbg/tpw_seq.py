import sys, glob, os, numpy as np, torch
sys.path.insert(0, '.')
import paper_2201_05024_b200 as K
from oracle import kapsm_oracle as O
SMALL = sorted(glob.glob('tests/golden/small_*.npz'))
def run(path, W, reps=2):
    g = np.load(path)
    Kn, M, nt, nd, sch = int(g["K"]), int(g["M"]), int(g["n_train"]), int(g["n_data"]), str(g["scheme"])
    rx, pil, tx, _ = K.host_frames([int(g["seed"])], Kn, M, nt, nd, sch)
    pipe = K.FramePipeline(1, Kn, M, nt, nd, sch, cfg=K.ApsmConfig(window=W), precision="f32")
    pipe.load(rx, pil, tx)
    out = []
    for _ in range(reps):
        pipe.launch_trainer(2); r = pipe.results(); out.append(r["n_active"][0].copy())
    return out
for W in [int(a) for a in sys.argv[1].split(',')]:
    for p in SMALL:
        o = run(p, W)
        print(W, os.path.basename(p), [list(x) for x in o], flush=True)
