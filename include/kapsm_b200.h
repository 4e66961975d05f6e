/*
 * kapsm_b200.h -- C ABI of the B200 (sm_100a) APSM partially linear multiuser
 * detector.  Plain pointers and sizes only; every pointer argument is a CUDA
 * device pointer unless stated otherwise; `stream` is a cudaStream_t passed as
 * void*.  All entry points are stream-ordered, allocate nothing and return a
 * kapsm_status code (KAPSM_OK == 0).
 *
 * The reference (/root/reference/pkg/src/kapsm) is pure Python/numpy and has no
 * FFI of its own.  Each entry point below replaces one reference operation on
 * the hot path; the cited file:line is the function whose semantics it keeps.
 * The Python host layer (paper_2201_05024_b200/) binds these with ctypes and
 * re-exposes the reference API (train, ApsmTrainer, batch_evaluate,
 * batch_detect, run_trial, demodulate_hard, ber); see INTEGRATION.md.
 *
 * Data layout (HBM):
 *   complex vectors are interleaved (re, im) pairs of the element type;
 *   a frame's received block is T x M complex, T = n_train + n_data symbols,
 *   pilots first (run_trial, noma.py:267-277);
 *   realified sample n of a complex stream is row 2t + l (apsm.py:156-182):
 *   r(2t) = [Re x_t ; Im x_t], r(2t+1) = [Im x_t ; -Re x_t];
 *   realified targets are the interleaved pilot symbols read as a real array.
 */
#ifndef KAPSM_B200_H
#define KAPSM_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KAPSM_OK = 0,
  KAPSM_ERR_INVALID = 1,      /* bad argument (shape, null, range)          */
  KAPSM_ERR_CUDA = 2,         /* CUDA launch / runtime error                */
  KAPSM_ERR_UNSUPPORTED = 3   /* configuration outside the built variants   */
} kapsm_status;

/* Per-(frame, user) status word written by the training kernel. */
enum {
  KAPSM_TRAIN_OK = 0,
  KAPSM_TRAIN_DEGENERATE = 1, /* kappa(r,r) <= 0  -> DegenerateSampleError (apsm.py:325-328) */
  KAPSM_TRAIN_STALLED = 2     /* internal pipeline watchdog fired (should never happen)       */
};

/* Sum-space kernel parameters (KernelParams, kernels.py:46-70). */
typedef struct {
  double w_l;
  double w_g;
  double sigma_sq;
} kapsm_kernel_params;

/* Human-readable text for a kapsm_status (host pointer, static storage). */
const char* kapsm_strerror(int code);
/* ABI version (major*100 + minor). */
int kapsm_abi_version(void);
/* A fresh non-blocking CUDA stream (host frameworks that pool their streams
 * can hand out aliases; the overlapped pipeline needs two distinct ones). */
int kapsm_stream_create(void** stream);
int kapsm_stream_destroy(void* stream);
/* Streaming frames (FrameStream): enqueue one frame's input copies
 * (cudaMemcpyDefault: pinned host or device sources) on `h2d`, then its
 * captured pipeline graph on `comp`; optional events: ev_wait0 (first copy
 * waits), ev_inputs_free (the slot's previous graph read its inputs),
 * ev_outputs_free (the slot's previous results were copied out), ev_t0/ev_t1
 * (timing around the graph).  ev_in / ev_comp are recorded.  kapsm_stream_
 * frame_out enqueues the result copies on `d2h` after ev_ready and records
 * ev_out. */
int kapsm_stream_frame_in(void* h2d, void* comp, void* ev_wait0, void* ev_inputs_free,
                          void* ev_outputs_free, void* ev_in, int n, void* const* dst,
                          const void* const* src, const unsigned long long* bytes,
                          void* graph_exec, void* ev_t0, void* ev_t1, void* ev_comp);
int kapsm_stream_frame_out(void* d2h, void* ev_ready, int n, void* const* dst,
                           const void* const* src, const unsigned long long* bytes, void* ev_out);
/* Largest APSM window W supported by kapsm_train_* in this build. */
int kapsm_max_window(void);
/* Upper bound on realified training samples per (frame, user); the
 * trainer's shared-memory footprint (the final-coefficient array, n_samples
 * words per chain) sets the effective limit: KAPSM_ERR_UNSUPPORTED beyond. */
int kapsm_max_samples(void);

/* ---------------------------------------------------------------------------
 * K1  Pilot sum-kernel Gram matrix.
 * Replaces the repeated window re-evaluation of ApsmTrainer._window_response
 * (apsm.py:288-302): Kmat[i][j] = w_l r_i.r_j + w_g exp(-||r_i - r_j||^2 / 2s^2)
 * over the 2*n_train realified pilot samples of each frame, computed once per
 * frame and shared by all users.  Exactly symmetric; diagonal = self_kernel
 * (kernels.py:181-184).
 *   rx      : F frames, frame f at rx + f*rx_stride elements, first n_train
 *             complex symbols of length M are the pilots.
 *   gram    : F x (Np x ld), Np = 2*n_train, frame stride gram_stride elements,
 *             ld >= Np.
 * ------------------------------------------------------------------------- */
int kapsm_pilot_gram_f32(const float* rx, long long rx_stride, int F, int n_train, int M,
                         kapsm_kernel_params p, float* gram, long long ld,
                         long long gram_stride, void* stream);
int kapsm_pilot_gram_f64(const double* rx, long long rx_stride, int F, int n_train, int M,
                         kapsm_kernel_params p, double* gram, long long ld,
                         long long gram_stride, void* stream);
/* Same Gram for arbitrary realified sample rows S (F x N x D, frame stride
 * s_stride elements): the stream an ApsmTrainer (apsm.py:241-372) observes. */
int kapsm_sample_gram_f32(const float* S, long long s_stride, int F, int N, int D,
                          kapsm_kernel_params p, float* gram, long long ld,
                          long long gram_stride, void* stream);
int kapsm_sample_gram_f64(const double* S, long long s_stride, int F, int N, int D,
                          kapsm_kernel_params p, double* gram, long long ld,
                          long long gram_stride, void* stream);

/* ---------------------------------------------------------------------------
 * K2  Persistent APSM trainer, one CTA per (frame, user).
 * Replaces ApsmTrainer.observe/observe_symbol/state and train()
 * (apsm.py:254-396): n_samples strictly sequential window updates per user,
 * three-case beta (apsm.py:185-191, 329-332), uniform weights
 * (apsm.py:139-153), theta update (apsm.py:338) and first-activation slot
 * bookkeeping (apsm.py:341-359), with no per-step launch.
 *   gram      : K1 output (kapsm_pilot_gram_* or kapsm_sample_gram_*);
 *               ld >= n_samples + 16 (16-byte aligned rows), and 32 x ld zero
 *               elements must follow the last frame's matrix.
 *   sample source for the final theta, exactly one non-NULL:
 *     rx / rx_stride            complex pilots (n_samples = 2*n_train, dim = 2M)
 *     samples / samples_stride  realified rows F x n_samples x dim
 *   targets   : F x K x n_samples realified targets ((frame,user) at
 *               targets + (f*K+u)*n_samples); for complex pilots this is the
 *               interleaved pilot symbol array read as reals (apsm.py:167-169).
 *   qtab      : 2*W values: qtab[2*(J-1)] = weight of every window entry but the
 *               newest for |J_n| = J, qtab[2*(J-1)+1] = newest entry's weight
 *               (uniform_weights' defect-absorbing last entry); NULL -> 1/J.
 *   base0     : optional F x K x n_samples warm-start responses f0(r_n)
 *               (NULL = zero filter, the case of run_trial, noma.py:271-275).
 *   theta0    : optional F x K x dim warm-start linear part (NULL = 0).
 * Outputs (leading dims F x K):
 *   coeff     : x n_samples  accumulated projection coefficient per sample
 *               (0 if it never became an atom)
 *   first_step: x n_samples  step of its first nonzero beta, -1 if never (slot
 *               order = sort by (first_step, index), apsm.py:341-358)
 *   theta     : x dim        collapsed linear part
 *   n_active  : x 1          number of activated samples (new atoms)
 *   status    : x 1          KAPSM_TRAIN_* flags
 * Limits: window <= kapsm_max_window(), n_samples <= kapsm_max_samples().
 * window <= 23 and n_samples <= 3072 run the latency-scheduled trainer (one
 * critical warp per chain); larger configurations run the general trainer
 * (train_wide.cu: one CTA per chain, the Gram band in shared memory).
 * ------------------------------------------------------------------------- */
int kapsm_train_f32(const float* gram, long long ld, long long gram_stride, const float* rx,
                    long long rx_stride, const float* samples, long long samples_stride, int dim,
                    const float* targets, int F, int K, int n_samples, int window,
                    double epsilon, kapsm_kernel_params p, const float* qtab,
                    const float* base0, const float* theta0, float* coeff, int* first_step,
                    float* theta, int* n_active, int* status, void* stream);
int kapsm_train_f64(const double* gram, long long ld, long long gram_stride, const double* rx,
                    long long rx_stride, const double* samples, long long samples_stride,
                    int dim, const double* targets, int F, int K, int n_samples, int window,
                    double epsilon, kapsm_kernel_params p, const double* qtab,
                    const double* base0, const double* theta0, double* coeff, int* first_step,
                    double* theta, int* n_active, int* status, void* stream);

/* The general trainer (train_wide.cu) at any size: same arguments and
 * results as kapsm_train_*, which selects it by itself beyond the latency
 * kernel's window / shared-memory limits.  Exported so its parity can be
 * tested on the small golden frames. */
int kapsm_train_general_f32(const float* gram, long long ld, long long gram_stride,
                            const float* rx, long long rx_stride, const float* samples,
                            long long samples_stride, int dim, const float* targets, int F, int K,
                            int n_samples, int window, double epsilon, kapsm_kernel_params p,
                            const float* qtab, const float* base0, const float* theta0,
                            float* coeff, int* first_step, float* theta, int* n_active,
                            int* status, void* stream);
int kapsm_train_general_f64(const double* gram, long long ld, long long gram_stride,
                            const double* rx, long long rx_stride, const double* samples,
                            long long samples_stride, int dim, const double* targets, int F,
                            int K, int n_samples, int window, double epsilon,
                            kapsm_kernel_params p, const double* qtab, const double* base0,
                            const double* theta0, double* coeff, int* first_step, double* theta,
                            int* n_active, int* status, void* stream);

/* ---------------------------------------------------------------------------
 * K3  Fused frame detection.
 * Replaces batch_detect / batch_evaluate (engine.py:206-261) for the filters
 * trained by K2 on the frame's own pilots, fused with demodulate_hard
 * (noma.py:125-135) and the bit/symbol error count of ber (noma.py:284-292):
 *   est_u(t) = theta_u . r1(y_t) + w_g sum_i coeff_u[i] kG(r_i, r1(y_t))
 *            + i ( theta_u . r2(y_t) + w_g sum_i coeff_u[i] kG(r_i, r2(y_t)) )
 * for every payload symbol t < n_data and user u < K of every frame.
 *   points     : n_points complex constellation points (host-built table,
 *                get_constellation order, noma.py:86-107), device memory.
 *   tx_labels  : optional F x K x n_data transmitted symbol labels (uint8);
 *                required when bit_err / sym_err are given.
 *   est        : optional F x K x n_data complex soft estimates.
 *   labels     : optional F x K x n_data decided labels (uint8; MSB-first Gray
 *                label bits of the nearest point, ties -> lowest index).
 *   bit_err, sym_err : optional F x K counters (accumulated, caller zeroes).
 * ------------------------------------------------------------------------- */
int kapsm_detect_frames_f32(const float* rx, long long rx_stride, int F, int K, int n_train,
                            int n_data, int M, const float* coeff, const float* theta,
                            kapsm_kernel_params p, const float* points, int n_points,
                            int bits_per_symbol, const unsigned char* tx_labels, float* est,
                            unsigned char* labels, unsigned long long* bit_err,
                            unsigned long long* sym_err, void* stream);
int kapsm_detect_frames_f64(const double* rx, long long rx_stride, int F, int K, int n_train,
                            int n_data, int M, const double* coeff, const double* theta,
                            kapsm_kernel_params p, const double* points, int n_points,
                            int bits_per_symbol, const unsigned char* tx_labels, double* est,
                            unsigned char* labels, unsigned long long* bit_err,
                            unsigned long long* sym_err, void* stream);

/* ---------------------------------------------------------------------------
 * Generic filter evaluation: batch_evaluate (engine.py:206-243) of one
 * FilterState (kernels.py:73-120) on n_inputs realified rows of length dim.
 *   out[n] = theta . u_n + w_g sum_a coeffs[a] exp(-||atoms[a] - u_n||^2 / 2s^2)
 * (kernels.py:194-206).  atoms row-major n_atoms x dim.
 * ------------------------------------------------------------------------- */
int kapsm_batch_evaluate_f32(const float* theta, const float* atoms, const float* coeffs,
                             int n_atoms, int dim, const float* inputs, int n_inputs,
                             kapsm_kernel_params p, float* out, void* stream);
int kapsm_batch_evaluate_f64(const double* theta, const double* atoms, const double* coeffs,
                             int n_atoms, int dim, const double* inputs, int n_inputs,
                             kapsm_kernel_params p, double* out, void* stream);

/* batch_detect (engine.py:246-261): complex estimates f(r1(y_t)) + i f(r2(y_t))
 * of one FilterState (dim = 2M) on n complex inputs rx (n x M interleaved);
 * out is n complex values. */
int kapsm_batch_detect_f32(const float* theta, const float* atoms, const float* coeffs,
                           int n_atoms, int dim, const float* rx, int n, kapsm_kernel_params p,
                           float* out, void* stream);
int kapsm_batch_detect_f64(const double* theta, const double* atoms, const double* coeffs,
                           int n_atoms, int dim, const double* rx, int n, kapsm_kernel_params p,
                           double* out, void* stream);

/* Hard decisions for n complex estimates (demodulate_hard, noma.py:125-135):
 * labels[i] = argmin_q |est[i] - points[q]|, ties -> lowest q. */
int kapsm_demap_f32(const float* est, long long n, const float* points, int n_points,
                    unsigned char* labels, void* stream);
int kapsm_demap_f64(const double* est, long long n, const double* points, int n_points,
                    unsigned char* labels, void* stream);

/* Pilot targets from their constellation labels (the receiver knows the
 * pilot sequence): targets[2i], targets[2i+1] = points[2 labels[i]],
 * points[2 labels[i] + 1] for n labels (realified targets, apsm.py:156-169);
 * a label >= n_points gives NaN targets.  Lets a host ship 1 byte per pilot
 * and user instead of a complex value (FramePipeline(pilot_labels=True)). */
int kapsm_targets_from_labels_f32(const unsigned char* labels, long long n, const float* points,
                                  int n_points, float* targets, void* stream);
int kapsm_targets_from_labels_f64(const unsigned char* labels, long long n, const double* points,
                                  int n_points, double* targets, void* stream);

/* Count differing elements of two equal-length streams of elem_bytes (1, 4, 8)
 * wide integers (ber numerator, noma.py:284-292).  *count is accumulated. */
int kapsm_count_mismatch(const void* a, const void* b, long long n, int elem_bytes,
                         unsigned long long* count, void* stream);

/* ---------------------------------------------------------------------------
 * Whole frame pipeline on one stream: zero the counters, K1, K2, K3 for all K
 * users of F frames (run_trial, noma.py:249-281, once per target user).
 * gram_ws: workspace of kapsm_pipeline_workspace_bytes() bytes -- the pilot
 *          Gram F x (2*n_train) x ld, ld = 2*n_train + 16 rounded up to 32,
 *          followed by 32 x ld zero elements (the trainer's staged reads run
 *          past the last sample into them); in FP32, when the
 *          one-warp-per-chain trainer runs instead (M <= 64 and window <= 149,
 *          with more chains than SMs, or with a window / pilot block beyond
 *          the Gram trainer's fast schedule: window > 23, the C3 sweep, or
 *          the C4 full band), its band rows and pilot screen.  Other
 *          arguments as for the three stages.  Captured into a CUDA graph by the host.
 * ------------------------------------------------------------------------- */
/* Bytes of gram_ws the pipelines need for this shape (elem_bytes 4: FP32,
 * 8: FP64); -1 on invalid arguments. */
long long kapsm_pipeline_workspace_bytes(int F, int K, int n_train, int M, int window,
                                         int elem_bytes);
int kapsm_run_frames_f32(const float* rx, long long rx_stride, const float* pilots,
                         const unsigned char* tx_labels, int F, int K, int n_train, int n_data,
                         int M, int window, double epsilon, kapsm_kernel_params p,
                         const float* qtab, const float* points, int n_points,
                         int bits_per_symbol, float* gram_ws, long long ld, float* coeff,
                         int* first_step, float* theta, int* n_active, int* status, float* est,
                         unsigned char* labels, unsigned long long* bit_err,
                         unsigned long long* sym_err, void* stream);
int kapsm_run_frames_f64(const double* rx, long long rx_stride, const double* pilots,
                         const unsigned char* tx_labels, int F, int K, int n_train, int n_data,
                         int M, int window, double epsilon, kapsm_kernel_params p,
                         const double* qtab, const double* points, int n_points,
                         int bits_per_symbol, double* gram_ws, long long ld, double* coeff,
                         int* first_step, double* theta, int* n_active, int* status, double* est,
                         unsigned char* labels, unsigned long long* bit_err,
                         unsigned long long* sym_err, void* stream);

/* ---------------------------------------------------------------------------
 * Split detection for the latency pipeline (csrc/screen.cu).
 * kapsm_detect_screen_*: the pilot/payload kernel screen of F frames, which
 *   does not depend on the filters (it can run concurrently with training).
 *   live: workspace of kapsm_screen_workspace_bytes(F, n_train, n_data) bytes
 *   (16-byte aligned); it starts with F x ceil(n_train/32) x n_data uint32
 *   bits: bit p%32 of live[f][p/32][t] is set when some realified kernel of
 *   (pilot p, payload t) does not underflow (the screen the fused kernel
 *   applies per pair), followed by per-symbol compact lists of the live
 *   pilots' kernel values.
 * kapsm_detect_finish_*: the fused detection epilogue (linear part, the
 *   Gaussian part over the live pilots recomputed with explicit differences,
 *   demap, error counts) from the screen's live bits; other arguments as for
 *   kapsm_detect_frames_*.
 * ------------------------------------------------------------------------- */
long long kapsm_screen_workspace_bytes(int F, int n_train, int n_data);
int kapsm_detect_screen_f32(const float* rx, long long rx_stride, int F, int n_train, int n_data,
                            int M, kapsm_kernel_params p, unsigned* live, void* stream);
int kapsm_detect_screen_f64(const double* rx, long long rx_stride, int F, int n_train,
                            int n_data, int M, kapsm_kernel_params p, unsigned* live,
                            void* stream);
int kapsm_detect_finish_f32(const float* rx, long long rx_stride, int F, int K, int n_train,
                            int n_data, int M, const float* coeff, const float* theta,
                            kapsm_kernel_params p, const float* points, int n_points,
                            int bits_per_symbol, const unsigned char* tx_labels,
                            const unsigned* live, float* est, unsigned char* labels,
                            unsigned long long* bit_err, unsigned long long* sym_err,
                            void* stream);
int kapsm_detect_finish_f64(const double* rx, long long rx_stride, int F, int K, int n_train,
                            int n_data, int M, const double* coeff, const double* theta,
                            kapsm_kernel_params p, const double* points, int n_points,
                            int bits_per_symbol, const unsigned char* tx_labels,
                            const unsigned* live, double* est, unsigned char* labels,
                            unsigned long long* bit_err, unsigned long long* sym_err,
                            void* stream);

/* Latency pipeline: kapsm_run_frames_* with the kernel screen on side_stream
 * (fork/join through events, capturable into one CUDA graph) overlapping K1
 * and K2, then the detection finish.  live_ws as for kapsm_detect_screen_*. */
int kapsm_run_frames_overlap_f32(const float* rx, long long rx_stride, const float* pilots,
                                 const unsigned char* tx_labels, int F, int K, int n_train,
                                 int n_data, int M, int window, double epsilon,
                                 kapsm_kernel_params p, const float* qtab, const float* points,
                                 int n_points, int bits_per_symbol, float* gram_ws, long long ld,
                                 unsigned* live_ws, float* coeff, int* first_step, float* theta,
                                 int* n_active, int* status, float* est, unsigned char* labels,
                                 unsigned long long* bit_err, unsigned long long* sym_err,
                                 void* stream, void* side_stream);
int kapsm_run_frames_overlap_f64(const double* rx, long long rx_stride, const double* pilots,
                                 const unsigned char* tx_labels, int F, int K, int n_train,
                                 int n_data, int M, int window, double epsilon,
                                 kapsm_kernel_params p, const double* qtab, const double* points,
                                 int n_points, int bits_per_symbol, double* gram_ws,
                                 long long ld, unsigned* live_ws, double* coeff, int* first_step,
                                 double* theta, int* n_active, int* status, double* est,
                                 unsigned char* labels, unsigned long long* bit_err,
                                 unsigned long long* sym_err, void* stream, void* side_stream);

#ifdef __cplusplus
}
#endif
#endif /* KAPSM_B200_H */
