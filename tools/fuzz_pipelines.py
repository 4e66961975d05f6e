"""Randomised cross-check of the FP32 pipeline forms (band trainers: one-warp,
ring warps + helpers, wide; Gram cluster trainer) against the FP64 pipeline on
random shapes: decisions and bit errors identical up to rare eps-boundary
flips, estimates close.  usage: python tools/fuzz_pipelines.py [n_cases] [seed]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for case in range(n_cases):
    Kn = int(rng.integers(1, 9)); M = int(rng.choice([2, 3, 4, 7, 8, 12, 16, 19, 32, 33, 48, 64]))
    sch = str(rng.choice(["BPSK", "QPSK", "QAM16"]))
    nt = int(rng.integers(8, 400)); nd = int(rng.integers(1, 300))
    W = int(rng.choice([1, 3, 7, 20, 21, 22, 25, 40, 64, 100, 132]))
    F = int(rng.choice([1, 1, 2, 30]))
    seeds = [int(s) for s in rng.integers(0, 10**6, F)]
    rx, pil, tx, _ = K.host_frames(seeds, Kn, M, nt, nd, sch)
    out = {}
    for prec in ("f32", "f64"):
        p = K.FramePipeline(F, Kn, M, nt, nd, sch, cfg=K.ApsmConfig(window=W), precision=prec)
        p.load(rx, pil, tx); p.launch()
        out[prec] = p.results()
    a, b = out["f32"], out["f64"]
    # user 0 / frame F-1 against the oracle (both precisions)
    from oracle import kapsm_oracle as O
    f = F - 1
    ref = O.train_user(O.realify(rx[f, :nt]), O.realify_targets(pil[f, 0]), W=W)
    est = O.detect_batch(ref["theta"], ref["atoms"], ref["coeffs"], rx[f, nt:])
    o_err = max(np.max(np.abs(out[pr]["est"][f, 0] - est)) / max(1e-30, np.max(np.abs(est)))
                for pr in ("f32", "f64"))
    o_lab = max(np.mean(out[pr]["labels"][f, 0] != O.demap_indices(est, sch)) for pr in ("f32", "f64"))
    lab_mis = np.mean(a["labels"] != b["labels"])
    at_mis = np.mean(a["n_active"] != b["n_active"])
    est_rel = np.max(np.abs(a["est"] - b["est"])) / max(1e-30, np.max(np.abs(b["est"])))
    ok = lab_mis <= 1e-3 and est_rel < 1e-3 and o_err < 1e-3 and o_lab <= 1e-2
    bad += not ok
    print(f"case {case}: F={F} K={Kn} M={M} {sch} nt={nt} nd={nd} W={W}: label mismatch {lab_mis:.2e}, "
          f"atoms mismatch {at_mis:.2f}, est rel {est_rel:.1e}, vs oracle est {o_err:.1e} labels {o_lab:.1e} "
          f"{'OK' if ok else 'BAD'}", flush=True)
print("bad cases:", bad)
