"""Randomised check of the engine API (train -> FilterState, batch_detect,
ApsmTrainer incremental observe) against the oracle on random shapes, windows
and both precisions.  usage: python tools/fuzz_engine.py [n_cases] [seed]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2201_05024_b200 as K
from oracle import kapsm_oracle as O

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for case in range(n_cases):
    Kn = int(rng.integers(1, 7)); M = int(rng.choice([1, 2, 3, 5, 8, 16, 31, 32, 64]))
    sch = str(rng.choice(["BPSK", "QPSK", "QAM16"]))
    nt = int(rng.integers(1, 300)); nd = int(rng.integers(1, 200))
    W = int(rng.choice([1, 2, 5, 20, 23, 24, 50, 100, 132]))
    prec = str(rng.choice(["f32", "f64"]))
    seed = int(rng.integers(0, 10**6))
    fr = O.make_frame(seed, Kn, M, nt, nd, sch)
    cfg = K.ApsmConfig(window=W)
    u = int(rng.integers(0, Kn))
    try:
        f = K.train(None, zip(fr["rx"][:nt], fr["symbols"][u, :nt]), cfg, precision=prec)
        est = K.batch_detect(f, fr["rx"][nt:], cfg.params, K.EngineConfig(precision=prec))
    except Exception as e:  # noqa: BLE001
        print(f"case {case}: K={Kn} M={M} {sch} nt={nt} W={W} {prec}: raised {type(e).__name__}: {str(e)[:80]}")
        continue
    ref = O.train_user(O.realify(fr["rx"][:nt]), O.realify_targets(fr["symbols"][u, :nt]), W=W)
    e_ref = O.detect_batch(ref["theta"], ref["atoms"], ref["coeffs"], fr["rx"][nt:])
    tol = 1e-4 if prec == "f32" else 1e-9
    atoms_ok = f.n_atoms == ref["n_atoms"] or prec == "f32"
    er = np.max(np.abs(est - e_ref)) / max(1e-30, np.max(np.abs(e_ref)))
    ok = atoms_ok and er < (1e-3 if prec == "f32" else 1e-8)
    bad += not ok
    print(f"case {case}: K={Kn} M={M} {sch} nt={nt} nd={nd} W={W} {prec}: atoms {f.n_atoms}/{ref['n_atoms']} "
          f"est rel {er:.1e} {'OK' if ok else 'BAD'}", flush=True)
print("bad cases:", bad)
