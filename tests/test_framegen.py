"""Parallel live frame generation (paper_2201_05024_b200/framegen.py): the
frames the worker pool writes into the shared ring are the seeded frames of
host_frames (the reference's generator in run_trial's RNG order), byte for
byte in the device layout.  CPU only (the ring is not pinned here)."""

import numpy as np

from paper_2201_05024_b200 import get_constellation
from paper_2201_05024_b200.framegen import FrameGenerator
from paper_2201_05024_b200.frames import host_frames


def test_generator_matches_host_frames():
    F, K, M, nt, nd = 5, 6, 16, 40, 64
    gen = FrameGenerator(F, K, M, nt, nd, "QPSK", slots=2, workers=2, pin=False)
    try:
        seeds = [11, 12, 13, 14, 15]
        gen.fill(1, seeds).wait()
        rx, pil, tx, _ = host_frames(seeds, K, M, nt, nd, "QPSK")
        ref_rx = np.stack([rx.real, rx.imag], -1).astype(np.float32)
        ref_pil = np.stack([pil.real, pil.imag], -1).astype(np.float32)
        assert np.array_equal(gen.views["rx"][1], ref_rx)
        assert np.array_equal(gen.views["pilots"][1], ref_pil)
        assert np.array_equal(gen.views["tx"][1], tx.astype(np.uint8))
        # pilot labels: the constellation points of their labels are the pilots
        pts = get_constellation("QPSK").points
        assert np.array_equal(pts[gen.views["plab"][1]].astype(np.complex64),
                              pil.astype(np.complex64))
        # the other slot is untouched (zeros)
        assert not gen.views["rx"][0].any()
        # a second fill of the same slot with other seeds replaces it
        gen.fill(1, [21, 22, 23, 24, 25]).wait()
        rx2, _, _, _ = host_frames([21, 22, 23, 24, 25], K, M, nt, nd, "QPSK")
        assert np.array_equal(gen.views["rx"][1], np.stack([rx2.real, rx2.imag], -1).astype(np.float32))
    finally:
        gen.close()


def test_generator_qam16_massive():
    F, K, M, nt, nd = 2, 16, 64, 20, 30
    gen = FrameGenerator(F, K, M, nt, nd, "QAM16", slots=1, workers=1, pin=False)
    try:
        gen.fill(0, [3, 4]).wait()
        rx, pil, tx, _ = host_frames([3, 4], K, M, nt, nd, "QAM16")
        assert np.array_equal(gen.views["rx"][0], np.stack([rx.real, rx.imag], -1).astype(np.float32))
        assert np.array_equal(gen.views["tx"][0], tx.astype(np.uint8))
        pts = get_constellation("QAM16").points
        assert np.array_equal(pts[gen.views["plab"][0]].astype(np.complex64),
                              pil.astype(np.complex64))
    finally:
        gen.close()
