"""n_active of the one-warp-per-chain trainer vs the Gram trainer vs the
reference table (C1 seeds 0..19) and the oracle (mismatching chains)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2201_05024_b200 as K
from oracle import kapsm_oracle as O
g = np.load("tests/golden/c1_seeds20.npz")
rx, pil, tx, _ = K.host_frames(range(20), 6, 16, 685, 3840, "QPSK")
res = {}
for mode in (1, 2):
    p = K.FramePipeline(20, 6, 16, 685, 3840, "QPSK", precision="f32", full_workspace=True)
    p.load(rx, pil, tx); p.launch_trainer(mode); res[mode] = p.results()
for mode in (1, 2):
    r = res[mode]
    print("mode", mode, "n_active mismatches vs reference:", int((r["n_active"] != g["n_atoms"]).sum()),
          "labels equal:", bool(np.array_equal(r["labels"], g["labels"])),
          "bit_err equal:", bool(np.array_equal(r["bit_err"], g["bit_err"])))
seeds = list(range(50, 90))
rx, pil, tx, _ = K.host_frames(seeds, 6, 16, 685, 3840, "QPSK")
for mode in (1, 2):
    p = K.FramePipeline(40, 6, 16, 685, 3840, "QPSK", precision="f32", full_workspace=True)
    p.load(rx, pil, tx); p.launch_trainer(mode); res[mode] = p.results()
bad = np.argwhere(res[1]["n_active"] != res[2]["n_active"])
print("gram vs tp mismatches at seeds 50..89:", bad.tolist())
for f, u in bad[:3]:
    R = O.realify(rx[f][:685]); ref = O.train_user(R, O.realify_targets(pil[f][u]))
    fs1, fs2 = res[1]["first_step"][f, u], res[2]["first_step"][f, u]
    print(f"seed {seeds[f]} user {u}: oracle {ref['n_atoms']} gram {res[1]['n_active'][f, u]} tp {res[2]['n_active'][f, u]};",
          "first_step diffs gram:", np.argwhere(fs1 != ref['first_step']).ravel()[:5].tolist(),
          "tp:", np.argwhere(fs2 != ref['first_step']).ravel()[:5].tolist())
