// One-call frame pipeline: K1 (pilot Gram) -> K2 (persistent trainer, all K
// users of all F frames) -> K3 (fused detection + demap + error count), all on
// one stream, no host synchronisation, no allocation -- the unit that the
// host captures into a CUDA graph.  Composition of run_trial
// (noma.py:249-281) for every target user of each frame.
#include "kapsm_common.cuh"

namespace kapsm {
bool train_tp_supported(int n_train, int M, int W);
template <typename T>
bool train_takes_general(int Np, int W);
size_t train_tp_ws_bytes(int F, int n_train, int W);
int train_tp(const float* rx, long long rx_stride, const float* targets, int F, int K,
             int n_train, int M, int W, double eps, kapsm_kernel_params p, const float* qtab,
             void* ws, float* coeff, int* first_step, float* theta, int* n_active, int* status,
             cudaStream_t s, int stages = 7);
}  // namespace kapsm

static int pipe_num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

// Throughput mode (more chains than SMs): the one-warp-per-chain trainer
// (train_tp.cu) replaces K1 + K2 in FP32 when its limits hold (W <= 25,
// M <= 64) and its workspace (band rows + pilot screen) fits in the caller's
// Gram workspace.  Latency mode keeps the Gram-based trainer, whose critical
// warp is the shorter per-step chain when a chain has SMs to itself.
// trainer choice: AUTO as above, or forced (internal entry points: tests, A/B)
enum TrainerMode { TRAINER_AUTO = 0, TRAINER_GRAM = 1, TRAINER_TP = 2, TRAINER_TP1 = 3 };

template <typename T>
static bool use_tp(int F, int K, int n_train, int M, int window, long long ld,
                   int mode = TRAINER_AUTO) {
  (void)ld;
  if constexpr (sizeof(T) != 4) {
    return false;
  } else {
    if (mode == TRAINER_GRAM || !kapsm::train_tp_supported(n_train, M, window)) return false;
    return mode == TRAINER_TP || mode == TRAINER_TP1 || (long long)F * K > pipe_num_sms() ||
           kapsm::train_takes_general<float>(2 * n_train, window);
  }
}

// Bytes of gram_ws the pipeline needs: the one-warp trainer's workspace (band
// rows + pilot screen) when it runs, else the pilot Gram F x Np x ld plus the
// 32 zero tail rows (ld = Np rounded as below).  The caller allocates this.
extern "C" long long kapsm_pipeline_workspace_bytes(int F, int K, int n_train, int M, int window,
                                                    int elem_bytes) {
  if (F < 0 || K < 1 || n_train < 1 || M < 1 || window < 1 || (elem_bytes != 4 && elem_bytes != 8))
    return -1;
  const long long Np = 2LL * n_train, ld = (Np + 16 + 31) / 32 * 32;
  const long long gram = ((long long)F * Np + 32) * ld * elem_bytes;
  if (elem_bytes == 4 && use_tp<float>(F, K, n_train, M, window, ld))
    return (long long)kapsm::train_tp_ws_bytes(F, n_train, window);
  return gram;
}

template <typename T> struct Fns;
template <> struct Fns<float> {
  static constexpr auto gram = kapsm_pilot_gram_f32;
  static constexpr auto train = kapsm_train_f32;
  static constexpr auto detect = kapsm_detect_frames_f32;
  static constexpr auto screen = kapsm_detect_screen_f32;
  static constexpr auto finish = kapsm_detect_finish_f32;
};
template <> struct Fns<double> {
  static constexpr auto gram = kapsm_pilot_gram_f64;
  static constexpr auto train = kapsm_train_f64;
  static constexpr auto detect = kapsm_detect_frames_f64;
  static constexpr auto screen = kapsm_detect_screen_f64;
  static constexpr auto finish = kapsm_detect_finish_f64;
};

template <typename T>
static int run_frames(const T* rx, long long rx_stride, const T* pilots,
                      const unsigned char* tx_labels, int F, int K, int n_train, int n_data, int M,
                      int window, double eps, kapsm_kernel_params p, const T* qtab,
                      const T* points, int n_points, int bps, T* gram_ws, long long ld, T* coeff,
                      int* first_step, T* theta, int* n_active, int* status, T* est,
                      unsigned char* labels, unsigned long long* bit_err,
                      unsigned long long* sym_err, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (F < 0 || K < 1 || n_train < 1 || n_data < 0 || M < 1) return KAPSM_ERR_INVALID;
  if (F == 0) return KAPSM_OK;
  const int Np = 2 * n_train;
  if (bit_err && cudaMemsetAsync(bit_err, 0, sizeof(unsigned long long) * F * K, s) != cudaSuccess)
    return KAPSM_ERR_CUDA;
  if (sym_err && cudaMemsetAsync(sym_err, 0, sizeof(unsigned long long) * F * K, s) != cudaSuccess)
    return KAPSM_ERR_CUDA;
  int r;
  if constexpr (sizeof(T) == 4) {
    if (use_tp<T>(F, K, n_train, M, window, ld)) {
      r = kapsm::train_tp(rx, rx_stride, pilots, F, K, n_train, M, window, eps, p, qtab, gram_ws,
                          coeff, first_step, theta, n_active, status, s);
      if (r) return r;
      return Fns<T>::detect(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p, points,
                            n_points, bps, tx_labels, est, labels, bit_err, sym_err, stream);
    }
  }
  const long long gstride = (long long)Np * ld;
  r = Fns<T>::gram(rx, rx_stride, F, n_train, M, p, gram_ws, ld, gstride, stream);
  if (r) return r;
  r = Fns<T>::train(gram_ws, ld, gstride, rx, rx_stride, nullptr, 0, 2 * M, pilots, F, K, Np,
                    window, eps, p, qtab, nullptr, nullptr, coeff, first_step, theta, n_active,
                    status, stream);
  if (r) return r;
  return Fns<T>::detect(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p, points,
                        n_points, bps, tx_labels, est, labels, bit_err, sym_err, stream);
}

#define KAPSM_RUN_ENTRY(NAME, T)                                                               \
  extern "C" int NAME(const T* rx, long long rx_stride, const T* pilots,                       \
                      const unsigned char* tx_labels, int F, int K, int n_train, int n_data,   \
                      int M, int window, double eps, kapsm_kernel_params p, const T* qtab,     \
                      const T* points, int n_points, int bps, T* gram_ws, long long ld,        \
                      T* coeff, int* first_step, T* theta, int* n_active, int* status, T* est, \
                      unsigned char* labels, unsigned long long* bit_err,                      \
                      unsigned long long* sym_err, void* stream) {                             \
    return run_frames<T>(rx, rx_stride, pilots, tx_labels, F, K, n_train, n_data, M, window,   \
                         eps, p, qtab, points, n_points, bps, gram_ws, ld, coeff, first_step,  \
                         theta, n_active, status, est, labels, bit_err, sym_err, stream);      \
  }
KAPSM_RUN_ENTRY(kapsm_run_frames_f32, float)
KAPSM_RUN_ENTRY(kapsm_run_frames_f64, double)

// Latency pipeline: K1 first, then K3a (kernel screen, independent of the
// filters) on a side stream while K2 runs on the main stream; K3b finishes
// once both are done.  Stream-ordered fork/join through events, so it captures into one
// CUDA graph.
template <typename T, int MODE = TRAINER_AUTO>
static int run_frames_overlap(const T* rx, long long rx_stride, const T* pilots,
                              const unsigned char* tx_labels, int F, int K, int n_train,
                              int n_data, int M, int window, double eps, kapsm_kernel_params p,
                              const T* qtab, const T* points, int n_points, int bps, T* gram_ws,
                              long long ld, unsigned* live_ws, T* coeff, int* first_step,
                              T* theta, int* n_active, int* status, T* est,
                              unsigned char* labels, unsigned long long* bit_err,
                              unsigned long long* sym_err, void* stream, void* side_stream) {
  cudaStream_t s = (cudaStream_t)stream, s2 = (cudaStream_t)side_stream;
  if (F < 0 || K < 1 || n_train < 1 || n_data < 0 || M < 1 || !live_ws) return KAPSM_ERR_INVALID;
  if (F == 0) return KAPSM_OK;
  if (!s2 || s2 == s) return KAPSM_ERR_INVALID;
  const int Np = 2 * n_train;
  cudaEvent_t fork, join;
  if (cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess) return KAPSM_ERR_CUDA;
  if (cudaEventCreateWithFlags(&join, cudaEventDisableTiming) != cudaSuccess) {
    cudaEventDestroy(fork);
    return KAPSM_ERR_CUDA;
  }
  int r = KAPSM_OK;
  do {
    if constexpr (sizeof(T) == 4) {
      if (use_tp<T>(F, K, n_train, M, window, ld, MODE)) {
        // detection screen forked at once (the band kernel is short); the
        // one-warp-per-chain trainer on the main stream
        if (cudaEventRecord(fork, s) != cudaSuccess ||
            cudaStreamWaitEvent(s2, fork, 0) != cudaSuccess) {
          r = KAPSM_ERR_CUDA;
          break;
        }
        if ((r = Fns<T>::screen(rx, rx_stride, F, n_train, n_data, M, p, live_ws, s2))) break;
        if (cudaEventRecord(join, s2) != cudaSuccess) { r = KAPSM_ERR_CUDA; break; }
        if ((r = kapsm::train_tp(rx, rx_stride, pilots, F, K, n_train, M, window, eps, p, qtab,
                                 gram_ws, coeff, first_step, theta, n_active, status, s,
                                 MODE == TRAINER_TP1 ? 15 : 7)))
          break;
        goto finish;
      }
    }
    if (false) goto finish;           // (the label is unused in the FP64 instantiation)
    {
    const long long gstride = (long long)Np * ld;
    if ((r = Fns<T>::gram(rx, rx_stride, F, n_train, M, p, gram_ws, ld, gstride, stream))) break;
    // fork after K1: the screen then shares the GPU only with the trainer's
    // few SMs instead of slowing the Gram down
    if (cudaEventRecord(fork, s) != cudaSuccess || cudaStreamWaitEvent(s2, fork, 0) != cudaSuccess) {
      r = KAPSM_ERR_CUDA;
      break;
    }
    if ((r = Fns<T>::screen(rx, rx_stride, F, n_train, n_data, M, p, live_ws, s2))) break;
    if (cudaEventRecord(join, s2) != cudaSuccess) { r = KAPSM_ERR_CUDA; break; }
    if ((r = Fns<T>::train(gram_ws, ld, gstride, rx, rx_stride, nullptr, 0, 2 * M, pilots, F, K,
                           Np, window, eps, p, qtab, nullptr, nullptr, coeff, first_step, theta,
                           n_active, status, stream)))
      break;
    }
  finish:
    if (bit_err && cudaMemsetAsync(bit_err, 0, sizeof(unsigned long long) * F * K, s) != cudaSuccess) {
      r = KAPSM_ERR_CUDA;
      break;
    }
    if (sym_err && cudaMemsetAsync(sym_err, 0, sizeof(unsigned long long) * F * K, s) != cudaSuccess) {
      r = KAPSM_ERR_CUDA;
      break;
    }
    if (cudaStreamWaitEvent(s, join, 0) != cudaSuccess) { r = KAPSM_ERR_CUDA; break; }
    r = Fns<T>::finish(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p, points, n_points,
                       bps, tx_labels, live_ws, est, labels, bit_err, sym_err, stream);
  } while (false);
  cudaEventDestroy(fork);
  cudaEventDestroy(join);
  return r;
}

#define KAPSM_RUN2_ENTRY(NAME, T)                                                              \
  extern "C" int NAME(const T* rx, long long rx_stride, const T* pilots,                       \
                      const unsigned char* tx_labels, int F, int K, int n_train, int n_data,   \
                      int M, int window, double eps, kapsm_kernel_params p, const T* qtab,     \
                      const T* points, int n_points, int bps, T* gram_ws, long long ld,        \
                      unsigned* live_ws, T* coeff, int* first_step, T* theta, int* n_active,   \
                      int* status, T* est, unsigned char* labels, unsigned long long* bit_err, \
                      unsigned long long* sym_err, void* stream, void* side_stream) {          \
    return run_frames_overlap<T>(rx, rx_stride, pilots, tx_labels, F, K, n_train, n_data, M,   \
                                 window, eps, p, qtab, points, n_points, bps, gram_ws, ld,     \
                                 live_ws, coeff, first_step, theta, n_active, status, est,     \
                                 labels, bit_err, sym_err, stream, side_stream);               \
  }
KAPSM_RUN2_ENTRY(kapsm_run_frames_overlap_f32, float)
KAPSM_RUN2_ENTRY(kapsm_run_frames_overlap_f64, double)

// Internal (tests / A-B timing, not in the public header): the overlapped
// pipeline in FP32 with the trainer forced -- mode 1: the Gram-based trainer
// (K1 pilot Gram + K2 train.cu), mode 2: the one-warp-per-chain trainer
// (train_tp.cu) whenever its limits hold, at any number of chains (its
// critical-warp form in latency mode), mode 3: as 2 without that form.
extern "C" int kapsm_internal_run_frames_overlap_mode_f32(
    int mode, const float* rx, long long rx_stride, const float* pilots,
    const unsigned char* tx_labels, int F, int K, int n_train, int n_data, int M, int window,
    double eps, kapsm_kernel_params p, const float* qtab, const float* points, int n_points,
    int bps, float* gram_ws, long long ld, unsigned* live_ws, float* coeff, int* first_step,
    float* theta, int* n_active, int* status, float* est, unsigned char* labels,
    unsigned long long* bit_err, unsigned long long* sym_err, void* stream, void* side_stream) {
#define KAPSM_MODE_CALL(MD)                                                                        \
  return run_frames_overlap<float, MD>(rx, rx_stride, pilots, tx_labels, F, K, n_train, n_data, M, \
                                       window, eps, p, qtab, points, n_points, bps, gram_ws, ld,   \
                                       live_ws, coeff, first_step, theta, n_active, status, est,   \
                                       labels, bit_err, sym_err, stream, side_stream)
  if (mode == TRAINER_GRAM) KAPSM_MODE_CALL(TRAINER_GRAM);
  if (mode == TRAINER_TP) KAPSM_MODE_CALL(TRAINER_TP);
  if (mode == TRAINER_TP1) KAPSM_MODE_CALL(TRAINER_TP1);
#undef KAPSM_MODE_CALL
  return KAPSM_ERR_INVALID;
}

extern "C" int kapsm_stream_create(void** stream) {
  if (!stream) return KAPSM_ERR_INVALID;
  cudaStream_t t;
  if (cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking) != cudaSuccess) return KAPSM_ERR_CUDA;
  *stream = t;
  return KAPSM_OK;
}

extern "C" int kapsm_stream_destroy(void* stream) {
  return cudaStreamDestroy((cudaStream_t)stream) == cudaSuccess ? KAPSM_OK : KAPSM_ERR_CUDA;
}

// Streaming frames: one call enqueues a frame's input copies (cudaMemcpyDefault:
// pinned host or device sources) on the copy stream and its captured pipeline
// graph on the slot's compute stream, ordered through the caller's events; a
// second call enqueues the result copies.  The host cost per frame is one
// library call each way instead of a dozen framework calls.
extern "C" int kapsm_stream_frame_in(void* h2d, void* comp, void* ev_wait0, void* ev_inputs_free,
                                     void* ev_outputs_free, void* ev_in, int n, void* const* dst,
                                     const void* const* src, const unsigned long long* bytes,
                                     void* graph_exec, void* ev_t0, void* ev_t1, void* ev_comp) {
  cudaStream_t hs = (cudaStream_t)h2d, cs = (cudaStream_t)comp;
  if (!ev_in || !ev_comp || !graph_exec || n < 0 || (n && (!dst || !src || !bytes)))
    return KAPSM_ERR_INVALID;
  if (ev_wait0 && cudaStreamWaitEvent(hs, (cudaEvent_t)ev_wait0, 0) != cudaSuccess) return KAPSM_ERR_CUDA;
  if (ev_inputs_free && cudaStreamWaitEvent(hs, (cudaEvent_t)ev_inputs_free, 0) != cudaSuccess)
    return KAPSM_ERR_CUDA;
  for (int i = 0; i < n; ++i)
    if (cudaMemcpyAsync(dst[i], src[i], bytes[i], cudaMemcpyDefault, hs) != cudaSuccess)
      return KAPSM_ERR_CUDA;
  if (cudaEventRecord((cudaEvent_t)ev_in, hs) != cudaSuccess ||
      cudaStreamWaitEvent(cs, (cudaEvent_t)ev_in, 0) != cudaSuccess)
    return KAPSM_ERR_CUDA;
  if (ev_outputs_free && cudaStreamWaitEvent(cs, (cudaEvent_t)ev_outputs_free, 0) != cudaSuccess)
    return KAPSM_ERR_CUDA;
  if (ev_t0 && cudaEventRecord((cudaEvent_t)ev_t0, cs) != cudaSuccess) return KAPSM_ERR_CUDA;
  if (cudaGraphLaunch((cudaGraphExec_t)graph_exec, cs) != cudaSuccess) return KAPSM_ERR_CUDA;
  if (ev_t1 && cudaEventRecord((cudaEvent_t)ev_t1, cs) != cudaSuccess) return KAPSM_ERR_CUDA;
  return cudaEventRecord((cudaEvent_t)ev_comp, cs) == cudaSuccess ? KAPSM_OK : KAPSM_ERR_CUDA;
}

extern "C" int kapsm_stream_frame_out(void* d2h, void* ev_ready, int n, void* const* dst,
                                      const void* const* src, const unsigned long long* bytes,
                                      void* ev_out) {
  cudaStream_t ds = (cudaStream_t)d2h;
  if (!ev_ready || !ev_out || n < 0 || (n && (!dst || !src || !bytes)))
    return KAPSM_ERR_INVALID;
  if (cudaStreamWaitEvent(ds, (cudaEvent_t)ev_ready, 0) != cudaSuccess) return KAPSM_ERR_CUDA;
  for (int i = 0; i < n; ++i)
    if (cudaMemcpyAsync(dst[i], src[i], bytes[i], cudaMemcpyDefault, ds) != cudaSuccess)
      return KAPSM_ERR_CUDA;
  return cudaEventRecord((cudaEvent_t)ev_out, ds) == cudaSuccess ? KAPSM_OK : KAPSM_ERR_CUDA;
}
