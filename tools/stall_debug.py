import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
F = 16
rx, pil, tx, _ = K.host_frames(range(F), 6, 16, 685, 3840, "QPSK")
pipe = K.FramePipeline(F, 6, 16, 685, 3840, "QPSK", precision="f32")
pipe.load(rx, pil, tx); pipe.launch(); torch.cuda.synchronize()
st = pipe.status.cpu().numpy(); print("status\n", st)
bad = np.argwhere(st != 0)
print("bad (frame,user):", bad.tolist())
for f in sorted(set(bad[:, 0].tolist()))[:3]:
    p1 = K.FramePipeline(1, 6, 16, 685, 3840, "QPSK", precision="f32")
    p1.load(rx[f:f+1], pil[f:f+1], tx[f:f+1]); p1.launch(); torch.cuda.synchronize()
    print("frame", f, "alone status", p1.status.cpu().numpy())
# repeat F=16 a few times
for i in range(3):
    pipe.launch(); torch.cuda.synchronize()
    print("rerun", i, "bad", int((pipe.status.cpu().numpy() != 0).sum()))
for F2 in (2, 4, 8, 24, 32):
    p2 = K.FramePipeline(F2, 6, 16, 685, 3840, "QPSK", precision="f32")
    p2.load(rx[:F2] if F2 <= 16 else np.concatenate([rx]*2)[:F2], pil[:F2] if F2 <= 16 else np.concatenate([pil]*2)[:F2], tx[:F2] if F2 <= 16 else np.concatenate([tx]*2)[:F2])
    p2.launch(); torch.cuda.synchronize()
    print("F", F2, "bad", int((p2.status.cpu().numpy() != 0).sum()))
