"""File containers (modelio.py) and the file-driven CLI: byte compatibility
with files written by the unmodified reference (tests/golden/files, made by
make_file_golden.py), validation errors with offsets, exit codes
(reference tests/test_cli.py:179-275, test_modelio.py)."""

import os

import numpy as np
import pytest

import paper_2201_05024_b200 as K
from paper_2201_05024_b200 import cli
from paper_2201_05024_b200.modelio import (FileFormatError, load_iq, load_model, load_symbols,
                                           save_iq, save_model, save_symbols)

FILES = os.path.join(os.path.dirname(__file__), "golden", "files")


def test_reads_reference_files_and_writes_identical_bytes(tmp_path):
    g = np.load(os.path.join(FILES, "ref_values.npz"))
    rx = load_iq(os.path.join(FILES, "ref.iq"))
    assert np.array_equal(rx, g["rx"].astype(np.complex64).astype(np.complex128))
    f, p = load_model(os.path.join(FILES, "ref.mdl"))
    assert np.array_equal(f.theta, g["theta"]) and np.array_equal(f.atoms, g["atoms"])
    assert np.array_equal(f.coeffs, g["coeffs"])
    assert (p.w_l, p.w_g, p.sigma_sq) == tuple(g["params"])
    sym = load_symbols(os.path.join(FILES, "ref.sym"))
    assert np.array_equal(sym, g["rx"][:, 0].astype(np.complex64).astype(np.complex128))
    save_iq(tmp_path / "a.iq", g["rx"])
    save_model(tmp_path / "a.mdl", K.FilterState(g["theta"], g["atoms"], g["coeffs"]),
               K.KernelParams(*g["params"]))
    save_symbols(tmp_path / "a.sym", g["rx"][:, 0])
    for ours, ref in (("a.iq", "ref.iq"), ("a.mdl", "ref.mdl"), ("a.sym", "ref.sym")):
        assert (tmp_path / ours).read_bytes() == open(os.path.join(FILES, ref), "rb").read()


def test_validation_errors(tmp_path):
    good = open(os.path.join(FILES, "ref.iq"), "rb").read()
    p = tmp_path / "x.iq"
    p.write_bytes(b"NOTMAGIC" + good[8:])
    with pytest.raises(FileFormatError, match="magic at offset 0"):
        load_iq(p)
    p.write_bytes(good[:-3])
    with pytest.raises(FileFormatError, match="offset 16"):
        load_iq(p)
    p.write_bytes(good + b"\0")
    with pytest.raises(FileFormatError, match="trailing"):
        load_iq(p)
    p.write_bytes(good[:8] + np.array([0, 5], "<u4").tobytes())
    with pytest.raises(FileFormatError, match="M=0"):
        load_iq(p)
    m = open(os.path.join(FILES, "ref.mdl"), "rb").read()
    q = tmp_path / "x.mdl"
    q.write_bytes(m[:32] + np.array([-1.0], "<f8").tobytes() + m[40:])   # sigma^2 < 0
    with pytest.raises(FileFormatError, match="kernel parameters"):
        load_model(q)
    q.write_bytes(m[:100])
    with pytest.raises(FileFormatError, match="truncated"):
        load_model(q)
    s = tmp_path / "x.sym"
    s.write_bytes(b"\0" * 13)
    with pytest.raises(FileFormatError, match="offset 8"):
        load_symbols(s)
    assert issubclass(FileFormatError, ValueError)


def test_cli_exit_codes(tmp_path, capsys):
    assert cli.main(["--help"]) == 0
    assert cli.main(["detect"]) == 2                                  # usage
    assert cli.main(["detect", "nope.mdl", "nope.iq", str(tmp_path / "o")]) == 2
    good = open(os.path.join(FILES, "ref.iq"), "rb").read()
    (tmp_path / "t.iq").write_bytes(good[:-5])
    assert cli.main(["detect", os.path.join(FILES, "ref.mdl"), str(tmp_path / "t.iq"),
                     str(tmp_path / "o")]) == 2
    assert "offset" in capsys.readouterr().err
    (tmp_path / "e.sym").write_bytes(b"")
    assert cli.main(["train", "--iq", os.path.join(FILES, "ref.iq"), "--pilots",
                     str(tmp_path / "e.sym"), "--out", str(tmp_path / "m.mdl")]) == 2
    big = np.zeros(20, np.complex128)
    save_symbols(tmp_path / "b.sym", big)
    assert cli.main(["train", "--iq", os.path.join(FILES, "ref.iq"), "--pilots",
                     str(tmp_path / "b.sym"), "--out", str(tmp_path / "m.mdl")]) == 2
    # antenna mismatch: ref.mdl has M = 3, a 2-antenna capture
    save_iq(tmp_path / "m2.iq", np.ones((4, 2)))
    assert cli.main(["detect", os.path.join(FILES, "ref.mdl"), str(tmp_path / "m2.iq"),
                     str(tmp_path / "o")]) == 2


@pytest.mark.gpu
def test_train_then_detect_flow(tmp_path, capsys):
    """File-based detection == the in-process path at the file's float32
    output precision (test_cli.py:179-197); the model recovers the pilots."""
    fr = K.seeded_frame(5, 2, 4, 60, 40, "QPSK")
    save_iq(tmp_path / "c.iq", fr["rx"])
    save_symbols(tmp_path / "p.sym", fr["symbols"][0, :60])
    assert cli.main(["train", "--iq", str(tmp_path / "c.iq"), "--pilots",
                     str(tmp_path / "p.sym"), "--out", str(tmp_path / "f.mdl")]) == 0
    assert "trained" in capsys.readouterr().err
    assert cli.main(["detect", str(tmp_path / "f.mdl"), str(tmp_path / "c.iq"),
                     str(tmp_path / "e.sym")]) == 0
    f, p = load_model(tmp_path / "f.mdl")
    rx = load_iq(tmp_path / "c.iq")
    exp = K.batch_detect(f, rx, p, K.EngineConfig())
    exp32 = exp.real.astype(np.float32).astype(np.float64) + \
        1j * exp.imag.astype(np.float32).astype(np.float64)
    assert np.array_equal(load_symbols(tmp_path / "e.sym"), exp32)
    # the trained filter recovers its own pilot symbols
    lab = K.demodulate_hard(exp[:60], "QPSK")
    ref = K.demodulate_hard(fr["symbols"][0, :60], "QPSK")
    assert np.mean(lab == ref) > 0.9
