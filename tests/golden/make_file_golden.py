"""Container files written by the UNMODIFIED reference (kapsm/modelio.py), to
pin the byte layout of paper_2201_05024_b200.modelio.  Run in the build
container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_file_golden.py
"""
import os
import numpy as np
from kapsm import FilterState, KernelParams
from kapsm.modelio import save_iq, save_model, save_symbols

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "files")
os.makedirs(HERE, exist_ok=True)
rng = np.random.default_rng(77)
rx = (rng.standard_normal((9, 3)) + 1j * rng.standard_normal((9, 3))) * 0.7
save_iq(os.path.join(HERE, "ref.iq"), rx)
f = FilterState(rng.standard_normal(6), rng.standard_normal((4, 6)), rng.standard_normal(4))
save_model(os.path.join(HERE, "ref.mdl"), f, KernelParams(0.3, 0.7, 0.11))
save_symbols(os.path.join(HERE, "ref.sym"), rx[:, 0])
np.savez(os.path.join(HERE, "ref_values.npz"), rx=rx, theta=f.theta, atoms=f.atoms,
         coeffs=f.coeffs, params=np.array([0.3, 0.7, 0.11]))
print("wrote", sorted(os.listdir(HERE)))
