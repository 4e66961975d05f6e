import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2201_05024_b200 as K
P = 64
rx, pil, tx, _ = K.host_frames(range(P), 6, 16, 685, 3840, "QPSK")
rx_p = torch.from_numpy(np.stack([rx.real, rx.imag], -1).astype(np.float32)).pin_memory()
pil_p = torch.from_numpy(np.stack([pil.real, pil.imag], -1).astype(np.float32)).pin_memory()
tx_p = torch.from_numpy(tx.astype(np.uint8)).pin_memory()
src = {"host": (rx_p, pil_p, tx_p), "device": (rx_p.cuda(), pil_p.cuda(), tx_p.cuda())}
import time
for where in ("device", "host", "device"):
    r, p_, t_ = src[where]
    for post, timing in ((None, False), (lambda p: None, False), (lambda p: None, True)):
        fs = K.FrameStream(6, 16, 685, 3840, depth=4, concurrent=True, post=post)
        for i in range(8):
            last = fs.submit(r[i % P:i % P + 1], p_[i % P:i % P + 1], t_[i % P:i % P + 1])
        torch.cuda.synchronize()
        N = 200
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        c0 = time.perf_counter()
        for i in range(N):
            j = i % P
            last = fs.submit(r[j:j + 1], p_[j:j + 1], t_[j:j + 1], start_event=a if i == 0 else None,
                             timing=ev[i] if timing else None)
        c1 = time.perf_counter()
        cur = torch.cuda.current_stream()
        for k in range(last - 3, last + 1):
            cur.wait_event(fs.done_event(k))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(f"{where:6s} post {post is not None!s:5s} timing {timing!s:5s}: {N / ms * 1e3:8.0f} frames/s, host submit {(c1-c0)/N*1e6:6.1f} us/frame", flush=True)
        del fs
