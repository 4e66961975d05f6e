import sys, numpy as np, glob
sys.path.insert(0, '.')
import paper_2201_05024_b200 as K
from oracle import kapsm_oracle as O
g = np.load('tests/golden/small_s4_K6_M16_QPSK.npz')
Kn, M, nt, nd, sch = int(g["K"]), int(g["M"]), int(g["n_train"]), int(g["n_data"]), str(g["scheme"])
for W in [int(a) for a in sys.argv[1:]]:
    fr = O.make_frame(int(g["seed"]), Kn, M, nt, nd, sch)
    rx, pil, tx, _ = K.host_frames([int(g["seed"])], Kn, M, nt, nd, sch)
    pipe = K.FramePipeline(1, Kn, M, nt, nd, sch, cfg=K.ApsmConfig(window=W), precision="f32")
    pipe.load(rx, pil, tx); pipe.launch_trainer(2); r = pipe.results()
    R = O.realify(fr["rx"][:nt])
    ref = O.train_user(R, O.realify_targets(fr["symbols"][0, :nt]), W=W)
    fsg, fso = r["first_step"][0, 0], ref["first_step"]
    bad = np.nonzero(fsg != fso)[0]
    cg, co = r["coeff"][0, 0], ref["coeff"]
    badc = np.nonzero(np.abs(cg - co) > 1e-4 * np.abs(co).max())[0]
    print("W", W, "nact", r["n_active"][0, 0], ref["n_atoms"], "first fs mismatch", bad[:5], fsg[bad[:5]], fso[bad[:5]],
          "first coeff mismatch", badc[:8])
    print(" theta rel", np.abs(r["theta"][0, 0] - ref["theta"]).max() / np.abs(ref["theta"]).max())
