"""Frame-batched device pipeline: F frames x K users, train on each frame's
pilots, detect its payload, decide and count errors -- all on the GPU.

This is the throughput/latency entry point (the reference composes the same
work per user in ``run_trial``, noma.py:249-281).  Buffers are allocated once
per shape; ``launch`` issues the one-call C pipeline (``kapsm_run_frames_*``:
K1 Gram -> K2 persistent trainer -> K3 fused detect/demap/count) on the current
stream; ``capture`` records it into a CUDA graph replayed by ``replay``.

Layout (HBM): rx (F, T, M, 2) interleaved complex, pilots (F, K, n_train, 2),
tx labels (F, K, n_data) uint8; Gram workspace (F, Np, ld).
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .apsm import ApsmConfig, qtab_device
from .noma import get_constellation, points_device

__all__ = ["FramePipeline", "FrameStream", "host_frames"]


def _ld(n: int) -> int:
    """Gram row stride: 128-byte aligned rows with >= 16 zero columns past the
    last sample (the trainer's TMA copies read whole 16-byte granules and the
    staged column segments run up to 11 columns past the last sample)."""
    return (n + 16 + 31) // 32 * 32


class FramePipeline:
    def __init__(self, F: int, K: int, M: int, n_train: int, n_data: int, scheme: str = "QPSK",
                 cfg: Optional[ApsmConfig] = None, precision: str = "f32",
                 store_est: bool = True, device=None, overlap: bool = True,
                 full_workspace: bool = False, pilot_labels: bool = False):
        if precision not in dv.DTYPES:
            raise ValueError(f"precision must be 'f64' or 'f32', got {precision!r}")
        self.cfg = cfg or ApsmConfig()
        self.F, self.K, self.M, self.n_train, self.n_data = F, K, M, n_train, n_data
        self.T = n_train + n_data
        self.Np = 2 * n_train
        self.scheme = scheme
        self.prec = precision
        con = get_constellation(scheme)
        self.n_points, self.bps = con.points.size, con.bits_per_symbol
        lib = _lib.load()
        if self.cfg.window > lib.kapsm_max_window() or self.Np > lib.kapsm_max_samples():
            raise NotImplementedError(
                f"window {self.cfg.window} / {self.Np} pilot samples exceed the trainer limits "
                f"(window <= {lib.kapsm_max_window()}, samples <= {lib.kapsm_max_samples()})")
        dev = dv.device() if device is None else device
        tdt = dv.DTYPES[precision][0]
        z = lambda *s, dt=tdt: torch.zeros(s, dtype=dt, device=dev)
        self.rx = z(F, self.T, M, 2)
        # a spread-out placeholder frame (not zeros): a warm-up launch before the
        # first load (capture()) then sees no coincident pilots/payload (all
        # kernels live, the screen's slowest case)
        gen = torch.Generator(device=dev).manual_seed(0)
        self.rx.normal_(generator=gen)
        self.pilots = z(F, K, n_train, 2)
        # pilot_labels: the pilots arrive as constellation labels (uint8,
        # F x K x n_train) and the launch expands them into the targets on the
        # device (kapsm_targets_from_labels) -- 1 byte per pilot and user to copy
        self.pilot_labels = pilot_labels
        self.pilot_lab = z(F, K, n_train, dt=torch.uint8) if pilot_labels else None
        self.tx = z(F, K, n_data, dt=torch.uint8)
        self.ld = _ld(self.Np)
        # trainer workspace (kapsm_pipeline_workspace_bytes): the pilot Gram +
        # the trainer's zero tail rows, or in FP32 throughput mode the
        # one-warp trainer's band rows + pilot screen; full_workspace keeps
        # the Gram either way (``gram`` view; launch_trainer(1), stage timing)
        esz = 4 if precision == "f32" else 8
        ws = int(lib.kapsm_pipeline_workspace_bytes(F, K, n_train, M, self.cfg.window, esz))
        full = (F * self.Np + 32) * self.ld * esz
        need = max(ws, full) if full_workspace else ws
        self._gram_buf = z((need + esz * self.ld - 1) // (esz * self.ld), self.ld)
        self.gram = (self._gram_buf[: F * self.Np].view(F, self.Np, self.ld)
                     if self._gram_buf.shape[0] >= F * self.Np + 32 else None)
        self.coeff = z(F, K, self.Np)
        self.first_step = z(F, K, self.Np, dt=torch.int32)
        self.theta = z(F, K, 2 * M)
        self.n_active = z(F, K, dt=torch.int32)
        self.status = z(F, K, dt=torch.int32)
        self.est = z(F, K, n_data, 2) if store_est else None
        self.labels = z(F, K, n_data, dt=torch.uint8)
        self.bit_err = z(F, K, dt=torch.int64)
        self.sym_err = z(F, K, dt=torch.int64)
        self.qtab = qtab_device(self.cfg.window, precision)
        self.points = points_device(scheme, precision)
        self.graph = None
        # latency pipeline: the detection kernel screen (independent of the
        # filters) runs on a side stream, overlapping the Gram and the trainer
        self.overlap = overlap
        if overlap:
            nbytes = int(lib.kapsm_screen_workspace_bytes(F, n_train, n_data))
            self.live = torch.zeros(((nbytes + 15) // 16 * 4,), dtype=torch.int32, device=dev)
            self._side = dv.new_stream()
            self._fn = dv.fn("kapsm_run_frames_overlap", precision)
        else:
            self.live = None
            self._side = None
            self._fn = dv.fn("kapsm_run_frames", precision)

    # -- inputs -------------------------------------------------------------
    def load(self, rx, pilots, tx_labels, non_blocking: bool = False):
        """Copy one batch (host complex arrays or device tensors) into the static buffers."""
        def put(dst, src, cplx):
            if isinstance(src, torch.Tensor):
                dst.copy_(src, non_blocking=non_blocking)
            else:
                a = np.asarray(src)
                if cplx:
                    a = np.stack([a.real, a.imag], axis=-1)
                dst.copy_(torch.from_numpy(np.ascontiguousarray(a)).to(dst.dtype),
                          non_blocking=non_blocking)
        put(self.rx, rx, True)
        if self.pilot_labels:
            put(self.pilot_lab, pilots, False)
        else:
            put(self.pilots, pilots, True)
        put(self.tx, tx_labels, False)

    # -- compute ------------------------------------------------------------
    def _args(self, rx=None, pilots=None, tx=None):
        c = self.cfg
        rx = self.rx if rx is None else rx
        pilots = self.pilots if pilots is None else pilots
        tx = self.tx if tx is None else tx
        head = (dv.ptr(rx), self.T * self.M * 2, dv.ptr(pilots), dv.ptr(tx),
                self.F, self.K, self.n_train, self.n_data, self.M, c.window, float(c.epsilon),
                _lib.params(c.params), dv.ptr(self.qtab), dv.ptr(self.points), self.n_points,
                self.bps, dv.ptr(self._gram_buf), self.ld)
        tail = (dv.ptr(self.coeff), dv.ptr(self.first_step), dv.ptr(self.theta),
                dv.ptr(self.n_active), dv.ptr(self.status), dv.ptr(self.est),
                dv.ptr(self.labels), dv.ptr(self.bit_err), dv.ptr(self.sym_err))
        if self.overlap:
            return head + (dv.ptr(self.live),) + tail
        return head + tail

    def launch_on(self, rx, pilots, tx_labels):
        """Run the pipeline on device-resident inputs in place (no copy into
        the static buffers): tensors shaped and typed like ``rx``/``pilots``/
        ``tx`` (contiguous, same device).  Outputs land in this pipeline's
        buffers.  Stream-ordered on the current stream; not graph-captured.
        (Complex-target pipelines only: pilot labels go through ``load``.)"""
        if self.pilot_labels:
            raise ValueError("launch_on takes target pilots; this pipeline takes pilot labels")
        for name, t, ref in (("rx", rx, self.rx), ("pilots", pilots, self.pilots),
                             ("tx_labels", tx_labels, self.tx)):
            if (not isinstance(t, torch.Tensor) or t.shape != ref.shape or t.dtype != ref.dtype
                    or t.device != ref.device or not t.is_contiguous()):
                raise ValueError(f"{name}: expected a contiguous {ref.dtype} tensor of shape "
                                 f"{tuple(ref.shape)} on {ref.device}")
        args = self._args(rx, pilots, tx_labels)
        if self.overlap:
            _lib.check(self._fn(*args, dv.stream(), C.c_void_p(self._side.cuda_stream)),
                       "run_frames_overlap")
        else:
            _lib.check(self._fn(*args, dv.stream()), "run_frames")

    def launch_trainer(self, mode: int):
        """Internal (tests, A/B timing): the overlapped FP32 pipeline with the
        trainer forced -- 1: Gram-based (train.cu), 2: band trainer
        (train_tp.cu) at any number of chains (its critical-warp + helpers form
        in latency mode), 3: as 2 with the plain one-warp form."""
        if self.prec != "f32" or not self.overlap:
            raise ValueError("launch_trainer needs the overlapped FP32 pipeline")
        if mode == 1 and self.gram is None:
            raise ValueError("the Gram-based trainer needs FramePipeline(full_workspace=True)")
        lib = _lib.load()
        if mode in (2, 3) and int(lib.kapsm_internal_train_tp_ws_bytes(self.F, self.n_train, self.cfg.window)) > \
                self._gram_buf.numel() * self._gram_buf.element_size():
            raise ValueError("workspace too small for the one-warp trainer")
        self._expand_pilots()
        _lib.check(_lib.load().kapsm_internal_run_frames_overlap_mode_f32(
            int(mode), *self._args(), dv.stream(), C.c_void_p(self._side.cuda_stream)),
            "run_frames_overlap_mode")

    def _expand_pilots(self):
        if self.pilot_labels:
            _lib.check(dv.fn("kapsm_targets_from_labels", self.prec)(
                dv.ptr(self.pilot_lab), self.pilot_lab.numel(), dv.ptr(self.points),
                self.n_points, dv.ptr(self.pilots), dv.stream()), "targets_from_labels")

    def launch(self):
        """Enqueue the whole pipeline on the current stream."""
        self._expand_pilots()
        if self.overlap:
            _lib.check(self._fn(*self._args(), dv.stream(), C.c_void_p(self._side.cuda_stream)),
                       "run_frames_overlap")
        else:
            _lib.check(self._fn(*self._args(), dv.stream()), "run_frames")

    def capture(self):
        """Record one launch into a CUDA graph (static shapes and buffers)."""
        self.launch()                       # warm-up: sets kernel attributes outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch()
        self.graph = g
        return g

    def replay(self):
        if self.graph is None:
            self.capture()
        self.graph.replay()

    # -- outputs ------------------------------------------------------------
    def check_status(self, status=None):
        """Raise if any (frame, user) trainer reported a failure in its status
        word: DegenerateSampleError (apsm.py:325-328) or a RuntimeError when
        the trainer's pipeline watchdog cut the chain short."""
        st = self.status.cpu().numpy() if status is None else np.asarray(status)
        raise_for_status(st)

    def results(self, est: bool = True, check: bool = True) -> dict:
        out = dict(labels=self.labels.cpu().numpy(), bit_err=self.bit_err.cpu().numpy(),
                   sym_err=self.sym_err.cpu().numpy(), n_active=self.n_active.cpu().numpy(),
                   status=self.status.cpu().numpy(), theta=self.theta.cpu().numpy(),
                   coeff=self.coeff.cpu().numpy(), first_step=self.first_step.cpu().numpy())
        if check:
            self.check_status(out["status"])
        if est and self.est is not None:
            e = self.est.cpu().numpy().astype(np.float64)
            out["est"] = e[..., 0] + 1j * e[..., 1]
        return out


def raise_for_status(status):
    """Trainer status words (F x K int32) -> the reference's exceptions."""
    st = np.asarray(status)
    if np.any(st & _lib.TRAIN_DEGENERATE):
        from .apsm import DegenerateSampleError
        raise DegenerateSampleError(
            "kappa(r, r) = 0: zero sample vector with a weightless Gaussian kernel")
    if np.any(st & _lib.TRAIN_STALLED):
        raise RuntimeError("kapsm trainer pipeline watchdog fired: training was cut short "
                           f"for (frame, user) {np.argwhere(st & _lib.TRAIN_STALLED).tolist()}")
    if np.any(st):
        raise RuntimeError(f"kapsm trainer status {sorted(set(st.ravel().tolist()))}")


def _event_handle(ev) -> int:
    """Raw cudaEvent_t of a torch event (created by a first record if needed)."""
    h = ev.cuda_event
    if not h:
        ev.record(torch.cuda.current_stream())
        h = ev.cuda_event
    return h


class FrameStream:
    """Streaming frames from pinned host memory with copy/compute overlap
    (pinned, double-buffered H2D).  Each submission is one
    frame, or a batch of ``frames`` frames (throughput mode, one captured
    multi-frame pipeline per slot).

    ``depth`` FramePipelines (each captured into its own CUDA graph) are used
    round-robin.  Frame i's host->device copy runs on an H2D stream while frame
    i-1 computes; its decisions and error counters come back on a D2H stream
    while frame i+1 computes.  With ``concurrent`` each slot computes on its own
    stream, so up to ``depth`` frames are in flight at once (a frame's trainer
    occupies a few SMs for most of its latency).  Every copy and launch is
    stream-ordered through events, nothing blocks the host until ``result``::

        fs = FrameStream(6, 16, 685, 3840)
        t = fs.submit(rx_pin, pilots_pin, tx_pin)     # pinned host tensors, 1 frame
        labels, bit_err, sym_err = fs.result(t)       # host tensors (pinned)
    """

    def __init__(self, K: int, M: int, n_train: int, n_data: int, scheme: str = "QPSK",
                 cfg: Optional[ApsmConfig] = None, precision: str = "f32", depth: int = 2,
                 device=None, post=None, concurrent: bool = False, frames: int = 1,
                 pilot_labels: bool = False):
        if depth < 1:
            raise ValueError(f"depth must be >= 1, got {depth}")
        if frames < 1:
            raise ValueError(f"frames must be >= 1, got {frames}")
        dev = dv.device() if device is None else device
        self.depth = depth
        self.frames = frames
        self.pipes = [FramePipeline(frames, K, M, n_train, n_data, scheme, cfg=cfg,
                                    precision=precision, store_est=False, device=dev,
                                    pilot_labels=pilot_labels)
                      for _ in range(depth)]
        self.pilot_labels = pilot_labels
        for p in self.pipes:
            p.capture()
        torch.cuda.synchronize(dev)
        self.h2d = dv.new_stream()
        self.d2h = dv.new_stream()
        pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        self.labels_h = [pin(p.labels) for p in self.pipes]
        self.counts_h = [pin(torch.stack([p.bit_err, p.sym_err])) for p in self.pipes]
        self.status_h = [pin(p.status) for p in self.pipes]
        ev = lambda: [torch.cuda.Event() for _ in range(depth)]
        self.ev_in, self.ev_comp, self.ev_out = ev(), ev(), ev()
        self.used = [False] * depth
        self.post = post          # optional callable(pipe) on the compute stream (collectives)
        self.comp = [dv.new_stream() for _ in range(depth)] if concurrent else None
        self.coll = dv.new_stream() if (concurrent and post is not None) else None
        self.ev_start = [torch.cuda.Event(enable_timing=True) for _ in range(depth)]
        self.ev_end = [torch.cuda.Event(enable_timing=True) for _ in range(depth)]
        lib = _lib.load()
        self._fin, self._fout = lib.kapsm_stream_frame_in, lib.kapsm_stream_frame_out
        VP, UL, VP4, UL4 = C.c_void_p * 3, C.c_ulonglong * 3, C.c_void_p * 4, C.c_ulonglong * 4
        self._slot = []
        for k, p in enumerate(self.pipes):
            # with no collectives the slot's "inputs free" point is the graph's end
            comp_ev = self.ev_comp[k] if post is not None else self.ev_end[k]
            pin_t = p.pilot_lab if pilot_labels else p.pilots
            self._slot.append({
                "dst_in": VP(p.rx.data_ptr(), pin_t.data_ptr(), p.tx.data_ptr()),
                "bytes_in": UL(*(t.numel() * t.element_size() for t in (p.rx, pin_t, p.tx))),
                "src_in": VP(0, 0, 0),
                "dst_out": VP4(self.labels_h[k].data_ptr(), self.counts_h[k][0].data_ptr(),
                               self.counts_h[k][1].data_ptr(), self.status_h[k].data_ptr()),
                "src_out": VP4(p.labels.data_ptr(), p.bit_err.data_ptr(), p.sym_err.data_ptr(),
                               p.status.data_ptr()),
                "bytes_out": UL4(p.labels.numel(), p.bit_err.numel() * 8, p.sym_err.numel() * 8,
                                 p.status.numel() * 4),
                "graph": p.graph.raw_cuda_graph_exec(),
                "ev_in": _event_handle(self.ev_in[k]), "ev_comp": _event_handle(comp_ev),
                "ev_out": _event_handle(self.ev_out[k]), "ev_end": _event_handle(self.ev_end[k]),
                "ev_start": _event_handle(self.ev_start[k]),
            })
        self.n = 0

    def submit(self, rx, pilots, tx_labels, start_event=None, timing=None) -> int:
        """Queue one batch of ``frames`` frames (one frame by default): tensors
        shaped like FramePipeline.load's inputs for F = ``frames``
        (float32/float64 interleaved rx and pilots -- or uint8 pilot labels
        with ``pilot_labels`` -- uint8 payload labels), pinned
        host or device-resident; they are copied into the slot's buffers on the
        copy stream and the slot's captured graph runs on its compute stream --
        one library call (``kapsm_stream_frame_in``), results come back with a
        second (``kapsm_stream_frame_out``).  ``start_event``: the first copy
        waits for it; ``timing``: a (start, end) pair of timing events recorded
        around the frame's compute.  Returns a ticket for ``result``."""
        i, slot = self.n, self.n % self.depth
        p = self.pipes[slot]
        sl = self._slot[slot]
        for t, ref in ((rx, p.rx), (pilots, p.pilot_lab if self.pilot_labels else p.pilots),
                       (tx_labels, p.tx)):
            if t.dtype != ref.dtype or t.numel() != ref.numel() or not t.is_contiguous():
                raise ValueError(f"frame tensor {tuple(t.shape)} {t.dtype} does not match "
                                 f"{tuple(ref.shape)} {ref.dtype}")
        src = sl["src_in"]
        src[0], src[1], src[2] = rx.data_ptr(), pilots.data_ptr(), tx_labels.data_ptr()
        used = self.used[slot]
        t0, t1 = sl["ev_start"], None
        if timing is not None:          # torch events or their raw handles
            t0, t1 = (h if isinstance(h, int) else _event_handle(h) for h in timing)
        comp = self.comp[slot] if self.comp else torch.cuda.current_stream(p.rx.device)
        _lib.check(self._fin(
            self.h2d.cuda_stream, comp.cuda_stream,
            _event_handle(start_event) if start_event is not None else None,
            sl["ev_comp"] if used else None, sl["ev_out"] if used else None, sl["ev_in"],
            3, sl["dst_in"], src, sl["bytes_in"], sl["graph"], t0, t1, sl["ev_end"]),
            "stream_frame_in")
        ready = sl["ev_end"]
        if self.post is not None:
            coll = self.coll if self.coll is not None else comp
            coll.wait_event(self.ev_end[slot])
            with torch.cuda.stream(coll):
                self.post(p)
            self.ev_comp[slot].record(coll)
            ready = sl["ev_comp"]
        else:
            ready = sl["ev_end"]
        _lib.check(self._fout(self.d2h.cuda_stream, ready, 4, sl["dst_out"], sl["src_out"],
                              sl["bytes_out"], sl["ev_out"]), "stream_frame_out")
        self.used[slot] = True
        self.n += 1
        return i

    def compute_us(self, ticket: int) -> float:
        """Device time of the ticket's frame on its compute stream (after it completed)."""
        slot = ticket % self.depth
        self.ev_end[slot].synchronize()
        return self.ev_start[slot].elapsed_time(self.ev_end[slot]) * 1e3

    def done_event(self, ticket: int):
        """Event recorded after the ticket's results reached host memory."""
        return self.ev_out[ticket % self.depth]

    def result(self, ticket: int):
        """(labels, bit_err, sym_err) of a submitted frame, as host tensors.
        Valid until the slot is reused (``depth`` submissions later)."""
        if ticket < self.n - self.depth or ticket >= self.n:
            raise ValueError(f"ticket {ticket} is no longer (or not yet) held")
        slot = ticket % self.depth
        self.ev_out[slot].synchronize()
        raise_for_status(self.status_h[slot].numpy())
        return self.labels_h[slot], self.counts_h[slot][0], self.counts_h[slot][1]


def host_frames(seeds, K, M, n_train, n_data, scheme="QPSK", snr_db=20.0):
    """Seeded host frames in the reference's RNG order -> (rx, pilots, tx_labels, bits)."""
    from .noma import seeded_frame, symbol_labels
    rxs, pils, txs, bits = [], [], [], []
    for s in seeds:
        fr = seeded_frame(int(s), K, M, n_train, n_data, scheme, snr_db)
        k = fr["bps"]
        rxs.append(fr["rx"])
        pils.append(fr["symbols"][:, :n_train])
        txs.append(symbol_labels(fr["bits"][:, n_train * k:], k))
        bits.append(fr["bits"])
    return np.stack(rxs), np.stack(pils), np.stack(txs), np.stack(bits)
