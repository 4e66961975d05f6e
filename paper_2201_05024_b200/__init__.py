"""B200-native (sm_100a) APSM partially linear multiuser detector.

Drop-in for the hot path of the reference ``kapsm`` package
(/root/reference/pkg/src/kapsm): the same detector API -- train on pilots,
detect a frame, the same configuration and result objects -- backed by
hand-written CUDA kernels behind the C ABI in ``include/kapsm_b200.h``:

* K1 pilot Gram (``csrc/gram.cu``),
* K2 persistent APSM trainer, one CTA per (frame, user) (``csrc/train.cu``),
* K3 fused detection + hard decision + error count (``csrc/detect.cu``),
* the one-call frame pipeline captured into CUDA graphs (``csrc/pipeline.cu``,
  ``frames.py``).

There is no CPU fallback: compute calls raise if the library or a CUDA device
is missing.
"""

from .apsm import (ApsmConfig, ApsmTrainer, DegenerateSampleError, DictionaryCapacityError,
                   TrainingSample, apsm_step, beta, complex_to_real_pair, detect_symbol,
                   realify_batch, train, uniform_weights, window_indices)
from .bench import BenchReport, BenchRow, bench_detection, report_to_csv, report_to_json
from .engine import STAGES, EngineConfig, batch_detect, batch_evaluate
from .frames import FramePipeline, FrameStream, host_frames
from .kernels import (FilterState, KernelParams, evaluate, from_expansion, inner_product,
                      kernel_gaussian, kernel_linear, kernel_sum, norm_sq, self_kernel, zero_filter)
from .modelio import (IQ_MAGIC, MODEL_MAGIC, FileFormatError, load_iq, load_model, load_symbols,
                      save_iq, save_model, save_symbols)
from .noma import (SCHEMES, ChannelModel, Constellation, FrameSpec, TrialReport, ber,
                   demodulate_hard, draw_channel, get_constellation, modulate, noise_var_for_snr,
                   run_trial, seeded_frame, symbol_labels, synthesize_received)

__version__ = "0.1.0"
