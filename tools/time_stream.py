"""Frames/s of FrameStream at several depths (device-resident pool or pinned host)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
P = 64
rx, pil, tx, _ = K.host_frames(range(P), 6, 16, 685, 3840, "QPSK")
rx_p = torch.from_numpy(np.stack([rx.real, rx.imag], -1).astype(np.float32)).pin_memory()
pil_p = torch.from_numpy(np.stack([pil.real, pil.imag], -1).astype(np.float32)).pin_memory()
tx_p = torch.from_numpy(tx.astype(np.uint8)).pin_memory()
src = {"host": (rx_p, pil_p, tx_p), "device": (rx_p.cuda(), pil_p.cuda(), tx_p.cuda())}
for where in ("device", "host"):
    r, p_, t_ = src[where]
    for depth, conc in ((4, True), (6, True), (8, True), (12, True)):
        fs = K.FrameStream(6, 16, 685, 3840, depth=depth, concurrent=conc)
        for i in range(8):
            last = fs.submit(r[i % P:i % P + 1], p_[i % P:i % P + 1], t_[i % P:i % P + 1])
        torch.cuda.synchronize()
        N = 200
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lat = []
        for i in range(N):
            j = i % P
            last = fs.submit(r[j:j + 1], p_[j:j + 1], t_[j:j + 1], start_event=a if i == 0 else None)
        cur = torch.cuda.current_stream()
        for k in range(last - depth + 1, last + 1):
            cur.wait_event(fs.done_event(k))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        errs = int(fs.result(last)[1].sum())
        print(f"{where:6s} depth {depth} concurrent {conc!s:5s}: {N / ms * 1e3:8.0f} frames/s, "
              f"last frame compute {fs.compute_us(last):6.1f} us, bit err {errs}", flush=True)
        del fs
