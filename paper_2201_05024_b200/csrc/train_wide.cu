// K2w: general APSM trainer for the configurations beyond the latency
// kernel's schedule (window W > 23 or Np > 3072): the C3 dictionary / window
// sweep (n_train up to 8192, W up to 128) and the C4 full-band frame.
//
// Same reference semantics and restatement as train.cu (ApsmTrainer.observe,
// apsm.py:304-359, on the pilot Gram K from K1): at step n the window
// J_n = [lo_n, n] (apsm.py:132-136) gets
//   delta_j = q_j/den_j * shrink(b_j - f(r_j), eps)   (apsm.py:323-336)
//   c_j += delta_j,   first_step_j = first n with delta_j != 0 (apsm.py:341-358)
// with f(r_m) = init_m + Y_m:
//   * ring position i (one CHAIN thread) owns sample m = i (mod S) from step
//     m-P (its takeover) until the task ends or the position is reused;
//     Y_m accumulates every later window update  Y_m += sum_j delta_j K[j][m]
//     from a shared-memory band of the Gram matrix (Kb[j mod S][m mod S]);
//   * init_m = f0(r_m) + sum_{l<m} c_l K[m][l] with the coefficients as they
//     stood at the end of step t_m = m-P-1 is computed by a HELPER warp: the
//     final coefficients (l <= t_m - W, a shared array filled as samples leave
//     the window) and the per-step snapshot of the window's coefficients
//     (ring of R steps) dotted with Gram row m read from global memory.  The
//     part l <= t_m - W - E only needs coefficients final E steps earlier, so
//     the helper streams it ahead; the chain waits for init_m (a tagged shared
//     word) only when m enters the window P steps after its takeover.
// One step of the chain threads: delta (own slot) -> shared -> one named
// barrier -> band dot over the window -> Y.  The band rows of the samples
// taken over Q steps later arrive by cp.async; only pairs at distance < W+P
// (the ones a window update meets) are written, so two in-flight copies never
// target the same word.  Ring sizes make every reuse safe by construction:
//   S >= W + P + E + Q + 1 (band / init / final-coefficient reuse),
//   R >= P + 2 (snapshot reuse: the chain cannot pass step m+1 before the
//   helper that read snapshot t_m published init_m).
#include "kapsm_common.cuh"

namespace kapsm {

constexpr int TW_P = 4;                  // takeover lookahead (steps)
constexpr int TW_E = 4;                  // helpers' slack on final coefficients
constexpr int TW_Q = 2;                  // band prefetch distance (steps)
constexpr int TW_R = 8;                  // snapshot ring (>= P + 2)
constexpr int TW_HW = 12;                // helper warps
constexpr int TW_MAX_THREADS = 1024;
constexpr long long TW_SPIN = 1LL << 26;
static_assert(TW_R >= TW_P + 2, "snapshot ring too short");

__host__ __device__ constexpr int tw_slots(int W) { return W + TW_P + TW_E + TW_Q + 1; }
__host__ __device__ constexpr int tw_chain_threads(int W) { return (tw_slots(W) + 31) / 32 * 32; }

template <typename T>
struct WideSmem {
  size_t kb, snap, dv, cfin, initr, qsm, ctl, total;
  __host__ __device__ WideSmem(int W, int Np) {
    using Slot = typename Tagged<T>::slot_t;
    const size_t S = tw_slots(W);
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 15) & ~size_t(15); return r; };
    kb = take(S * S * sizeof(T));
    snap = take((size_t)TW_R * S * sizeof(T));
    dv = take(2 * S * sizeof(T));
    cfin = take((size_t)Np * sizeof(T));
    initr = take(S * sizeof(Slot));
    qsm = take(2 * (size_t)(W + 1) * sizeof(T));
    ctl = take(16 * sizeof(int));
    total = (o + 127) & ~size_t(127);
  }
};

// named barrier with an OR vote over the participating threads
KAPSM_DEV bool named_bar_or(int id, int nthreads, bool p) {
  unsigned r;
  asm volatile(
      "{\n .reg .pred q, o;\n setp.ne.u32 q, %1, 0;\n bar.red.or.pred o, %2, %3, q;\n"
      " selp.u32 %0, 1, 0, o;\n}"
      : "=r"(r)
      : "r"((unsigned)p), "r"(id), "r"(nthreads)
      : "memory");
  return r != 0;
}

template <typename T>
__global__ void __launch_bounds__(TW_MAX_THREADS, 1)
    apsm_train_wide_kernel(const T* __restrict__ gram, long long ld, long long gram_stride,
                           const T* __restrict__ rx, long long rx_stride,
                           const T* __restrict__ samples, long long samples_stride, int dim,
                           const T* __restrict__ targets, int F, int K, int Np, int W, T eps,
                           T w_l, const T* __restrict__ qtab, const T* __restrict__ base0,
                           const T* __restrict__ theta0, T* __restrict__ coeff_out,
                           int* __restrict__ fs_out, T* __restrict__ theta_out,
                           int* __restrict__ nact_out, int* __restrict__ status_out) {
  using Slot = typename Tagged<T>::slot_t;
  constexpr int P = TW_P, E = TW_E, Q = TW_Q, R = TW_R;
  extern __shared__ __align__(128) unsigned char smem[];
  const WideSmem<T> L(W, Np);
  const int S = tw_slots(W), NC = tw_chain_threads(W);
  T* Kb = reinterpret_cast<T*>(smem + L.kb);         // [S][S] Gram band, ring-indexed
  T* snap = reinterpret_cast<T*>(smem + L.snap);     // [R][S] window coefficients per step
  T* dv = reinterpret_cast<T*>(smem + L.dv);         // [2][S] the step's deltas
  T* cfin = reinterpret_cast<T*>(smem + L.cfin);     // [Np] final coefficients
  Slot* initr = reinterpret_cast<Slot*>(smem + L.initr);   // [S] tagged init_m
  T* qsm = reinterpret_cast<T*>(smem + L.qsm);       // [W+1][2] (q_mid, q_last)
  int* ctl = reinterpret_cast<int*>(smem + L.ctl);   // [0] steps done [1] abort [2] status [3] nact
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nthreads = blockDim.x;

  for (int fu = blockIdx.x; fu < F * K; fu += gridDim.x) {
    const int f = fu / K;
    const T* G = gram + (long long)f * gram_stride;
    const T* B = targets + (long long)fu * Np;
    const T* P0 = base0 ? base0 + (long long)fu * Np : nullptr;

    // ---------------- per-task state ----------------
    for (int i = tid; i < S * S; i += nthreads) Kb[i] = T(0);
    for (int i = tid; i < S; i += nthreads) Tagged<T>::store(&initr[i], T(0), -1);
    for (int i = tid; i < Np; i += nthreads) cfin[i] = T(0);
    for (int i = tid; i <= W; i += nthreads) {
      T qm = T(1) / T(i + 1), ql = qm;
      if (qtab && i < W) { qm = qtab[2 * i]; ql = qtab[2 * i + 1]; }
      qsm[2 * i] = i < W ? qm : T(0);
      qsm[2 * i + 1] = i < W ? ql : T(0);
    }
    if (tid < 16) ctl[tid] = 0;
    __syncthreads();
    // band rows of the samples taken over before step 0 (0 .. P+Q-1)
    for (int e = tid; e < (P + Q) * S; e += nthreads) {
      const int m = e / S, i = e % S;
      const int l = m - ((m - i) % S + S) % S;
      if (m < Np && l >= 0 && l > m - W - P) {
        const T v = G[(long long)m * ld + l];
        Kb[(m % S) * S + i] = v;
        Kb[i * S + m % S] = v;
      }
    }
    __syncthreads();

    if (tid < NC) {
      // =========================== CHAIN THREADS ===========================
      const int i = tid;
      const bool pos = i < S;
      int s = i <= P ? i : i - S;                 // owned sample
      bool valid = pos && s >= 0 && s < Np;
      T Y = T(0), c = T(0), bm = T(0), bp = T(0), invden = T(0);
      T bv = valid ? B[s] : T(0);
      int fs = 0x7fffffff;
      int degen = 0, nact = 0;
      bool abort = false;
      const unsigned kb_s = smem_u32(Kb);
      for (int n = 0; n < Np && !abort; ++n) {
        // band row of sample n+P+Q (used from step n+Q on)
        cp_async_wait<Q - 1>();
        {
          const int m = n + P + Q;
          if (pos && m < Np) {
            const int l = m - ((m - i) % S + S) % S;
            if (l >= 0 && l > m - W - P) {    // only pairs a window update can meet
              const T* src = G + (long long)m * ld + l;
              cp_async_s(kb_s + (unsigned)(((m % S) * S + i) * sizeof(T)), src);
              cp_async_s(kb_s + (unsigned)((i * S + m % S) * sizeof(T)), src);
            }
          }
          cp_async_commit();
        }
        const int lo = n - W + 1 > 0 ? n - W + 1 : 0;
        bool stalled = false;
        if (valid && s == n) {                    // entering: init_m from the helpers
          T iv = T(0);
          long long spins = 0;
          while (!Tagged<T>::load(&initr[s % S], s, iv))
            if (++spins > TW_SPIN || ((spins & 1023) == 0 && ld_volatile(&ctl[1]))) {
              stalled = true;
              break;
            }
          const T den = Kb[(s % S) * S + s % S];
          if (!(den > T(0))) degen = 1;
          invden = den > T(0) ? T(1) / den : T(0);
          bm = bv - eps - iv;
          bp = bv + eps - iv;
        }
        T delta = T(0);
        if (valid && s >= lo && s <= n) {
          const int J = n - lo + 1;
          const T q = s == n ? qsm[2 * (J - 1) + 1] : qsm[2 * (J - 1)];
          const T qi = q * invden;
          const T v1 = fma(-qi, Y, qi * bm), v2 = fma(-qi, Y, qi * bp);
          delta = fmax(v1, T(0)) + fmin(v2, T(0));
          c += delta;
          if (delta != T(0) && fs > n) fs = n;
          snap[(n % R) * S + i] = c;
          if (n == s + W - 1 || n == Np - 1) {    // leaves the window: final
            cfin[s] = c;
            fs_out[(long long)fu * Np + s] = fs == 0x7fffffff ? -1 : fs;
            nact += fs != 0x7fffffff;
          }
        }
        if (pos) dv[(n & 1) * S + i] = delta;
        abort = named_bar_or(1, NC, stalled);
        if (i == 0) {
          __threadfence_block();
          st_volatile(&ctl[0], n + 1);
        }
        // window update of every owned sample that is (or will be) in a window
        if (valid && s >= lo) {
          const T* d = dv + (n & 1) * S;
          T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
          int j = lo % S;
          int cnt = n - lo + 1;
          while (cnt > 0) {
            const int run = cnt < S - j ? cnt : S - j;    // up to the ring's end
            const T* kp = Kb + j * S + i;
            const T* dp = d + j;
            int k = 0;
            for (; k + 4 <= run; k += 4) {
              a0 = fma(dp[k], kp[k * S], a0);
              a1 = fma(dp[k + 1], kp[(k + 1) * S], a1);
              a2 = fma(dp[k + 2], kp[(k + 2) * S], a2);
              a3 = fma(dp[k + 3], kp[(k + 3) * S], a3);
            }
            for (; k < run; ++k) a0 = fma(dp[k], kp[k * S], a0);
            cnt -= run;
            j = 0;
          }
          Y += (a0 + a1) + (a2 + a3);
        }
        // takeover after step n: sample n+P+1 at ring position (n+P+1) mod S
        if (pos && i == (n + P + 1) % S) {
          s = n + P + 1;
          valid = s < Np;
          Y = T(0);
          c = T(0);
          fs = 0x7fffffff;
          bv = valid ? B[s] : T(0);
        }
      }
      cp_async_wait<0>();
      if (abort || degen || nact) {
        if (abort && i == 0) { atomicOr(&ctl[2], KAPSM_TRAIN_STALLED); st_volatile(&ctl[1], 1); }
        if (degen) atomicOr(&ctl[2], KAPSM_TRAIN_DEGENERATE);
        if (nact) atomicAdd(&ctl[3], nact);
      }
      if (abort && i == 0) st_volatile(&ctl[0], 0x3fffffff);   // release the helpers
    } else {
      // =========================== HELPER WARPS ===========================
      const int h = warp - NC / 32, nh = (nthreads - NC) / 32;
      auto wait_steps = [&](int x) -> bool {    // until ctl[0] >= x; false on abort
        long long spins = 0;
        while (ld_volatile(&ctl[0]) < x)
          if (++spins > TW_SPIN || ((spins & 1023) == 0 && ld_volatile(&ctl[1]))) return false;
        __threadfence_block();
        return true;
      };
      bool ok = true;
      for (int m = h; m < Np && ok; m += nh) {
        const int t = m - P - 1;                // coefficients as of the end of step t
        const T* row = G + (long long)m * ld;
        T acc = T(0);
        if (t >= 0) {
          const int le = t - W - E;               // early part: l <= le, final since step t-E-1
          if (le >= 0) {
            ok = wait_steps(t - E);
            if (!ok) break;
            T a1 = T(0), a2 = T(0), a3 = T(0);
            int l = lane;
            for (; l + 96 <= le; l += 128) {
              acc = fma(cfin[l], row[l], acc);
              a1 = fma(cfin[l + 32], row[l + 32], a1);
              a2 = fma(cfin[l + 64], row[l + 64], a2);
              a3 = fma(cfin[l + 96], row[l + 96], a3);
            }
            for (; l <= le; l += 32) acc = fma(cfin[l], row[l], acc);
            acc += (a1 + a2) + a3;
          }
          ok = wait_steps(t + 1);
          if (!ok) break;
          const T* sn = snap + (t % R) * S;
          for (int l = (le + 1 > 0 ? le + 1 : 0) + lane; l <= t; l += 32) {
            const T cv = l <= t - W ? cfin[l] : sn[l % S];
            acc = fma(cv, row[l], acc);
          }
        }
        acc = warp_sum(acc);
        if (lane == 0) Tagged<T>::store(&initr[m % S], acc + (P0 ? P0[m] : T(0)), m);
      }
      if (!ok && lane == 0) {
        atomicOr(&ctl[2], KAPSM_TRAIN_STALLED);
        st_volatile(&ctl[1], 1);
      }
    }
    __syncthreads();

    // ---------------- outputs ----------------
    for (int i = tid; i < Np; i += nthreads) coeff_out[(long long)fu * Np + i] = cfin[i];
    {
      T* th = theta_out + (long long)fu * dim;
      const T* t0 = theta0 ? theta0 + (long long)fu * dim : nullptr;
      const int nw = nthreads / 32;
      if (rx) {
        // complex pilots: Theta = theta[:M] + i theta[M:] = w_l sum_p (c_2p - i c_2p+1) x_p
        const int M = dim / 2, n_train = Np / 2;
        const T* X = rx + (long long)f * rx_stride;
        for (int kk = warp; kk < M; kk += nw) {
          T tr = T(0), ti = T(0);
          for (int p = lane; p < n_train; p += 32) {
            const T c1 = cfin[2 * p], c2 = cfin[2 * p + 1];
            const T xr = X[(long long)p * 2 * M + 2 * kk], xi = X[(long long)p * 2 * M + 2 * kk + 1];
            tr = fma(c1, xr, fma(c2, xi, tr));
            ti = fma(c1, xi, fma(-c2, xr, ti));
          }
          tr = warp_sum(tr);
          ti = warp_sum(ti);
          if (lane == 0) {
            th[kk] = w_l * tr + (t0 ? t0[kk] : T(0));
            th[M + kk] = w_l * ti + (t0 ? t0[M + kk] : T(0));
          }
        }
      } else {
        const T* Sm = samples + (long long)f * samples_stride;
        for (int kk = warp; kk < dim; kk += nw) {
          T acc = T(0);
          for (int i = lane; i < Np; i += 32) acc = fma(cfin[i], Sm[(long long)i * dim + kk], acc);
          acc = warp_sum(acc);
          if (lane == 0) th[kk] = w_l * acc + (t0 ? t0[kk] : T(0));
        }
      }
    }
    if (tid == 0) {
      status_out[fu] = ctl[2];
      nact_out[fu] = ctl[3];
    }
    __syncthreads();                              // state reused by the next task
  }
}

static int wide_num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

template <typename T>
int train_wide(const T* gram, long long ld, long long gram_stride, const T* rx,
               long long rx_stride, const T* samples, long long samples_stride, int dim,
               const T* targets, int F, int K, int Np, int W, double eps, kapsm_kernel_params p,
               const T* qtab, const T* base0, const T* theta0, T* coeff, int* first_step,
               T* theta, int* n_active, int* status, cudaStream_t s) {
  const int NC = tw_chain_threads(W);
  if (NC + 32 * TW_HW > TW_MAX_THREADS) return KAPSM_ERR_UNSUPPORTED;
  const WideSmem<T> L(W, Np);
  if (L.total > 227 * 1024) return KAPSM_ERR_UNSUPPORTED;
  auto kern = apsm_train_wide_kernel<T>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  const int tasks = F * K;
  const int grid = tasks < wide_num_sms() ? tasks : wide_num_sms();
  kern<<<grid, NC + 32 * TW_HW, L.total, s>>>(gram, ld, gram_stride, rx, rx_stride, samples,
                                              samples_stride, dim, targets, F, K, Np, W, (T)eps,
                                              (T)p.w_l, qtab, base0, theta0, coeff, first_step,
                                              theta, n_active, status);
  return status_from(cudaGetLastError());
}

template int train_wide<float>(const float*, long long, long long, const float*, long long,
                               const float*, long long, int, const float*, int, int, int, int,
                               double, kapsm_kernel_params, const float*, const float*,
                               const float*, float*, int*, float*, int*, int*, cudaStream_t);
template int train_wide<double>(const double*, long long, long long, const double*, long long,
                                const double*, long long, int, const double*, int, int, int, int,
                                double, kapsm_kernel_params, const double*, const double*,
                                const double*, double*, int*, double*, int*, int*, cudaStream_t);

// largest window / sample count the general trainer accepts at this precision
// (the FP64 band with room for 2048 samples: the bound both precisions honour)
int train_wide_max_window() {
  int W = 1;
  while (tw_chain_threads(W + 1) + 32 * TW_HW <= TW_MAX_THREADS &&
         WideSmem<double>(W + 1, 2048).total <= 227 * 1024)
    ++W;
  return W;
}

}  // namespace kapsm
