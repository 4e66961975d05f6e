import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, time
import paper_2201_05024_b200 as K
F = int(sys.argv[1])
rx, pil, tx, _ = K.host_frames(range(F), 6, 16, 685, 3840, "QPSK")
pipe = K.FramePipeline(F, 6, 16, 685, 3840, "QPSK", precision="f32")
pipe.load(rx, pil, tx)
t = time.time(); pipe.launch(); torch.cuda.synchronize(); print("time", time.time() - t)
st = pipe.status.cpu().numpy().ravel()
bad = np.nonzero(st)[0]
print("codes", sorted(set(st.tolist()))); print("tasks", st.size, "stalled", bad.size, "first", bad[:20].tolist(), "last", bad[-5:].tolist())
print("bit errors", int(pipe.bit_err.sum()))
