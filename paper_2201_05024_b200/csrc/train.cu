// K2: persistent APSM trainer -- one CTA per (frame, user), the whole
// 2*n_train-step sequential pilot loop in one launch.
//
// Reference semantics: ApsmTrainer.observe (apsm.py:304-359) driven by
// train()/observe_symbol (apsm.py:361-396).  At step n (realified sample n),
// with window J_n = [lo_n, n], lo_n = max(0, n-W+1) (apsm.py:132-136):
//   y_j   = f_n(r_j)                                 j in J_n   (apsm.py:288-302)
//   beta_j three-case on res_j = y_j - b_j, den_j = kappa(r_j,r_j)  (apsm.py:323-332)
//   c_j  += q_j beta_j, q = uniform_weights(|J_n|)   (apsm.py:336-359)
// where f_n = f0 + sum_i c_i kappa(r_i, .).  The represented function is the
// reference's (collapsed theta + one atom per activated sample); theta is
// formed at the end as w_l sum_i c_i r_i (the reference accumulates it per
// step, apsm.py:338 -- same value up to summation order).
//
// Restatement used here (pilot Gram K from K1, all sums exact rearrangements):
//   * every CRITICAL lane owns one sample m (32 slots) from step m-1 to step
//     m+S-2 and keeps Y_m = response, c_m, first_step_m in registers;
//   * incremental window update ("matvec"): after step n's betas,
//       Y_m += sum_{a in J_n} delta_a K[a][m]   for owned m <= n+1;
//   * the newly entering sample n+1 gets, at step n (off the critical chain),
//       red_{n+1} = sum_{owned i} c_i^(n) K[i][n+1]   (warp butterfly)
//     and at step n+1:  Y_{n+1} += red_{n+1} + P_{n+1},
//       P_m = f0(r_m) + sum_{i <= m-S} cfinal_i K[i][m]
//     which BACKGROUND warps stream from Gram rows as soon as c_i is final
//     (sample i leaves the window after step i+W-1), LB+1 steps ahead.
// Per step the critical warp does O(W) work with one __syncwarp; it never
// waits on global memory: its columns K[.][m] are cp.async-prefetched 8 steps
// ahead into shared memory, and P values arrive as tagged 64-bit words.
#include "kapsm_common.cuh"

namespace kapsm {

constexpr int TR_S = 32;           // critical slots (one warp)
constexpr int TR_NB = 3;           // background warps (warps 0..2); critical = warp 3
constexpr int TR_G = TR_NB * 32;   // background lanes
constexpr int TR_NJ = 16;          // P accumulators per background lane (registers)
constexpr int TR_PD = 4;           // Gram-row prefetch depth of the background ring
constexpr int TR_DELTA = 8;        // column prefetch distance (steps)
constexpr int TR_PBN = 64;         // P slots (ring)
constexpr int TR_MIN_LB = 7;       // minimum look-behind (background slack)
constexpr int TR_MAX_W = TR_S - 1 - TR_MIN_LB;
constexpr int TR_MAX_NP = TR_G * TR_NJ;
constexpr long long TR_SPIN_LIMIT = 1LL << 25;

template <typename T>
struct TrainSmem {
  // byte offsets into dynamic shared memory
  size_t col, bsm, dbuf, qsm, cfin, pbuf, ctl, total;
  int CS;
  __host__ __device__ TrainSmem(int W, int Np) {
    CS = W + TR_S;
    if (CS & 1) CS += 1;  // even row stride -> conflict-free column reads
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 15) & ~size_t(15); return r; };
    pbuf = take(TR_PBN * sizeof(typename Tagged<T>::slot_t));
    col = take(2 * TR_S * (size_t)CS * sizeof(T));
    bsm = take(2 * TR_S * sizeof(T));
    dbuf = take(2 * TR_S * sizeof(T));
    qsm = take(2 * (size_t)W * sizeof(T));
    cfin = take((size_t)Np * sizeof(T));
    ctl = take(16 * sizeof(int));
    total = o;
  }
};

template <typename T>
__global__ void __launch_bounds__((TR_NB + 1) * 32)
    apsm_train_kernel(const T* __restrict__ gram, long long ld, long long gram_stride,
                      const T* __restrict__ rx, long long rx_stride,
                      const T* __restrict__ samples, long long samples_stride, int dim,
                      const T* __restrict__ targets, int K, int Np, int W, T eps,
                      T w_l, const T* __restrict__ qtab, const T* __restrict__ base0,
                      const T* __restrict__ theta0, T* __restrict__ coeff_out,
                      int* __restrict__ fs_out, T* __restrict__ theta_out,
                      int* __restrict__ nact_out, int* __restrict__ status_out) {
  using Slot = typename Tagged<T>::slot_t;
  extern __shared__ __align__(16) unsigned char smem[];
  const TrainSmem<T> L(W, Np);
  const int CS = L.CS;
  Slot* pbuf = reinterpret_cast<Slot*>(smem + L.pbuf);
  T* col = reinterpret_cast<T*>(smem + L.col);     // [2][S][CS]
  T* bsm = reinterpret_cast<T*>(smem + L.bsm);     // [2][S]
  T* dbuf = reinterpret_cast<T*>(smem + L.dbuf);   // [2][S]
  T* qsm = reinterpret_cast<T*>(smem + L.qsm);     // [W][2]
  T* cfin = reinterpret_cast<T*>(smem + L.cfin);   // [Np]
  int* ctl = reinterpret_cast<int*>(smem + L.ctl); // [0]=progress [1]=abort [2]=status

  const int fu = blockIdx.x;                 // frame * K + user
  const int f = fu / K;
  const T* G = gram + (long long)f * gram_stride;
  const T* B = targets + (long long)fu * Np;  // realified targets (interleaved pilot symbols)
  const T* P0 = base0 ? base0 + (long long)fu * Np : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int LB = TR_S - W - 1;

  for (int i = threadIdx.x; i < TR_PBN; i += blockDim.x) Tagged<T>::store(&pbuf[i], T(0), -1);
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    T qm = T(1) / T(i + 1), ql = qm;
    if (qtab) { qm = qtab[2 * i]; ql = qtab[2 * i + 1]; }
    qsm[2 * i] = qm;
    qsm[2 * i + 1] = ql;
  }
  for (int i = threadIdx.x; i < Np; i += blockDim.x) cfin[i] = T(0);
  if (threadIdx.x == 0) { ctl[0] = -1; ctl[1] = 0; ctl[2] = 0; }
  __syncthreads();

  if (warp == TR_NB) {
    // =========================== CRITICAL WARP ===========================
    const int slot = lane;
    int m = slot;                // owned sample
    int buf = 0;
    // prologue: columns of the initial samples 0..S-1 (buffer 0)
    for (int s2 = 0; s2 < TR_S; ++s2) {
      if (s2 >= Np) break;
      T* dst = col + (size_t)s2 * CS;          // buffer 0, slot s2
      for (int j = lane; j < CS; j += 32) {
        int a = s2 - W + j;
        if (a >= 0 && a < Np && j < W + TR_S) cp_async_scalar(dst + j, G + (long long)s2 * ld + a);
      }
    }
    cp_async_commit();
    T b = (m < Np) ? B[m] : T(0);
    cp_async_wait<0>();
    __syncwarp();
    T Y = T(0), c = T(0), red_hold = T(0);
    int fs = -1, nact = 0;
    T den = (m < Np) ? col[(size_t)slot * CS + W] : T(1);
    if (m < Np && !(den > T(0))) atomicOr(&ctl[2], KAPSM_TRAIN_DEGENERATE);
    T invden = T(1) / den;
    if (m == 0) Y = P0 ? P0[0] : T(0);
    bool aborted = false;

    for (int n = 0; n < Np; ++n) {
      const int lo = n - W + 1 > 0 ? n - W + 1 : 0;
      const int J = n - lo + 1;
      const T* mycol = col + ((size_t)buf * TR_S + slot) * CS;
      const int cbase = m - W;                // column index j = a - cbase
      // (R) reduction for the next entering sample (independent of this step's chain)
      T red = T(0);
      if (n + 1 < Np) {
        T prod = (m <= n && m < Np) ? c * mycol[n + 1 - cbase] : T(0);
        red = warp_sum(prod);
        if (m == n + 1) red_hold = red;
      }
      // (E) sample n enters the window
      if (m == n && n > 0) {
        T pv;
        long long spins = 0;
        while (!Tagged<T>::load(&pbuf[n % TR_PBN], n, pv)) {
          if (++spins > TR_SPIN_LIMIT) { aborted = true; break; }
        }
        Y += red_hold + pv;
      }
      if (__any_sync(0xffffffffu, aborted)) { aborted = true; break; }
      // (B) three-case beta on the window (apsm.py:323-335)
      T delta = T(0);
      if (m >= lo && m <= n) {
        const T res = Y - b;
        T beta = T(0);
        if (res < -eps) beta = (-res - eps) * invden;
        else if (res > eps) beta = (-res + eps) * invden;
        const T q = qsm[2 * (J - 1) + (m == n ? 1 : 0)];
        delta = q * beta;
        c += delta;
        if (beta != T(0) && fs < 0) fs = n;
      }
      T* db = dbuf + (n & 1) * TR_S;
      db[slot] = delta;
      __syncwarp();
      // (M) incremental response update for owned samples m <= n+1
      if (m <= n + 1 && m < Np) {
        T acc0 = T(0), acc1 = T(0);
        int k = 0;
        for (; k + 1 < J; k += 2) {
          const int a0 = lo + k, a1 = lo + k + 1;
          acc0 = fma(db[a0 & (TR_S - 1)], mycol[a0 - cbase], acc0);
          acc1 = fma(db[a1 & (TR_S - 1)], mycol[a1 - cbase], acc1);
        }
        if (k < J) acc0 = fma(db[(lo + k) & (TR_S - 1)], mycol[lo + k - cbase], acc0);
        Y += acc0 + acc1;
      }
      // (L) sample lo leaves the window after this step: c is final
      if (n >= W - 1 && m == lo) {
        cfin[m] = c;
        coeff_out[(long long)fu * Np + m] = c;
        fs_out[(long long)fu * Np + m] = fs;
        nact += (fs >= 0);
      }
      // (P) prefetch the column (and target) of the sample taken over TR_DELTA steps later
      {
        const int mp = n + 2 + TR_DELTA;
        if (mp >= TR_S && mp < Np) {
          const int pb = (mp / TR_S) & 1, ps = mp & (TR_S - 1);
          T* dst = col + ((size_t)pb * TR_S + ps) * CS;
          const T* srow = G + (long long)mp * ld;
          for (int j = lane; j < W + TR_S; j += 32) {
            const int a = mp - W + j;
            if (a >= 0 && a < Np) cp_async_scalar(dst + j, srow + a);
          }
          if (lane == 0) cp_async_scalar(bsm + pb * TR_S + ps, B + mp);
        }
        cp_async_commit();
      }
      // (T) release sample n+2-S, take over sample n+2
      const int mt = n + 2;
      if (mt >= TR_S && mt < Np) {
        cp_async_wait<TR_DELTA>();
        __syncwarp();
        if (slot == (mt & (TR_S - 1))) {
          m = mt;
          buf = (mt / TR_S) & 1;
          Y = T(0); c = T(0); fs = -1; red_hold = T(0);
          b = bsm[buf * TR_S + slot];
          den = col[((size_t)buf * TR_S + slot) * CS + W];
          if (!(den > T(0))) atomicOr(&ctl[2], KAPSM_TRAIN_DEGENERATE);
          invden = T(1) / den;
        }
      }
      // (G) publish progress for the background warps
      if ((n & 3) == 3) {
        __syncwarp();
        if (lane == 0) { __threadfence_block(); st_volatile(&ctl[0], n); }
      }
    }
    // remaining window samples
    const int last_left = (Np - 1 >= W - 1) ? Np - W : -1;   // written by (L) at the last step
    if (!aborted && m < Np && m > last_left && m >= Np - W) {
      cfin[m] = c;
      coeff_out[(long long)fu * Np + m] = c;
      fs_out[(long long)fu * Np + m] = fs;
      nact += (fs >= 0);
    }
    nact = (int)warp_sum((T)nact);
    __syncwarp();
    if (lane == 0) {
      if (aborted) { atomicOr(&ctl[2], KAPSM_TRAIN_STALLED); st_volatile(&ctl[1], 1); }
      __threadfence_block();
      st_volatile(&ctl[0], Np + 64);
      nact_out[fu] = nact;
    }
  } else {
    // ========================== BACKGROUND WARPS =========================
    // lane g owns P accumulators for samples m = g + G*j (j < TR_NJ).
    const int g = warp * 32 + lane;
    T pacc[TR_NJ];
#pragma unroll
    for (int j = 0; j < TR_NJ; ++j) pacc[j] = T(0);
    // P_m = f0(r_m) for the first samples (no final predecessors yet)
    for (int mm = 1 + g; mm < TR_S && mm < Np; mm += TR_G)
      Tagged<T>::store(&pbuf[mm % TR_PBN], P0 ? P0[mm] : T(0), mm);
    const int fmax = Np - TR_S;   // f contributes to m >= f + S
    T ring[TR_PD][TR_NJ];
#pragma unroll
    for (int r = 0; r < TR_PD; ++r) {
#pragma unroll
      for (int j = 0; j < TR_NJ; ++j) {
        const int mm = g + TR_G * j;
        ring[r][j] = (r < fmax && mm >= r + TR_S && mm < Np) ? G[(long long)r * ld + mm] : T(0);
      }
    }
    bool stop = false;
    for (int f0 = 0; f0 < fmax && !stop; f0 += TR_PD) {
#pragma unroll
      for (int r = 0; r < TR_PD; ++r) {
        const int fi = f0 + r;
        if (fi < fmax && !stop) {
          const int need = fi + W - 1;
          long long spins = 0;
          while (ld_volatile(&ctl[0]) < need) {
            if (ld_volatile(&ctl[1]) || ++spins > TR_SPIN_LIMIT) { stop = true; break; }
            __nanosleep(32);
          }
          if (!stop) {
            __threadfence_block();
            const T cf = cfin[fi];
            if (cf != T(0)) {
#pragma unroll
              for (int j = 0; j < TR_NJ; ++j) pacc[j] = fma(cf, ring[r][j], pacc[j]);
            }
            const int mpub = fi + TR_S;
            if (mpub < Np && (mpub % TR_G) == g) {
              const int jp = mpub / TR_G;
              T v = T(0);
#pragma unroll
              for (int j = 0; j < TR_NJ; ++j) v = (j == jp) ? pacc[j] : v;
              Tagged<T>::store(&pbuf[mpub % TR_PBN], v + (P0 ? P0[mpub] : T(0)), mpub);
            }
            // refill this ring entry with row fi + PD
            const int fn = fi + TR_PD;
#pragma unroll
            for (int j = 0; j < TR_NJ; ++j) {
              const int mm = g + TR_G * j;
              ring[r][j] = (fn < fmax && mm >= fn + TR_S && mm < Np) ? G[(long long)fn * ld + mm]
                                                                     : T(0);
            }
          }
        }
      }
    }
    (void)LB;
  }
  __syncthreads();
  // ======================= theta = theta0 + w_l sum_i c_i r_i =====================
  // (collapsed linear part, kernels.py:130-141 / apsm.py:338)
  const int nw = blockDim.x >> 5;
  T* th = theta_out + (long long)fu * dim;
  const T* t0 = theta0 ? theta0 + (long long)fu * dim : nullptr;
  if (rx) {
    // complex pilots: theta (as Theta = theta[:M] + i theta[M:]) = w_l sum_p (c_2p - i c_2p+1) x_p
    const int M = dim / 2, n_train = Np / 2;
    const T* X = rx + (long long)f * rx_stride;
    for (int k = warp; k < M; k += nw) {
      T tr = T(0), ti = T(0);
      for (int p = lane; p < n_train; p += 32) {
        const T c1 = cfin[2 * p], c2 = cfin[2 * p + 1];
        const T xr = X[(long long)p * 2 * M + 2 * k], xi = X[(long long)p * 2 * M + 2 * k + 1];
        tr = fma(c1, xr, fma(c2, xi, tr));
        ti = fma(c1, xi, fma(-c2, xr, ti));
      }
      tr = warp_sum(tr);
      ti = warp_sum(ti);
      if (lane == 0) {
        th[k] = w_l * tr + (t0 ? t0[k] : T(0));
        th[M + k] = w_l * ti + (t0 ? t0[M + k] : T(0));
      }
    }
  } else {
    const T* S = samples + (long long)f * samples_stride;
    for (int k = warp; k < dim; k += nw) {
      T acc = T(0);
      for (int i = lane; i < Np; i += 32) acc = fma(cfin[i], S[(long long)i * dim + k], acc);
      acc = warp_sum(acc);
      if (lane == 0) th[k] = w_l * acc + (t0 ? t0[k] : T(0));
    }
  }
  if (threadIdx.x == 0) status_out[fu] = ctl[2];
}

template <typename T>
int train(const T* gram, long long ld, long long gram_stride, const T* rx, long long rx_stride,
          const T* samples, long long samples_stride, int dim, const T* targets, int F, int K,
          int Np, int W, double eps, kapsm_kernel_params p, const T* qtab, const T* base0,
          const T* theta0, T* coeff, int* first_step, T* theta, int* n_active, int* status,
          cudaStream_t s) {
  if (F < 0 || K < 1 || Np < 1 || dim < 1 || W < 1 || !(eps > 0)) return KAPSM_ERR_INVALID;
  if (F == 0) return KAPSM_OK;
  if (!gram || !targets || !coeff || !first_step || !theta || !n_active || !status)
    return KAPSM_ERR_INVALID;
  if ((rx == nullptr) == (samples == nullptr)) return KAPSM_ERR_INVALID;  // exactly one source
  if (rx && ((Np & 1) || (dim & 1))) return KAPSM_ERR_INVALID;
  if (W > TR_MAX_W || Np > TR_MAX_NP) return KAPSM_ERR_UNSUPPORTED;
  if (ld < Np) return KAPSM_ERR_INVALID;
  TrainSmem<T> L(W, Np);
  if (L.total > 227 * 1024) return KAPSM_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(apsm_train_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)L.total) != cudaSuccess)
    return KAPSM_ERR_CUDA;
  apsm_train_kernel<T><<<F * K, (TR_NB + 1) * 32, L.total, s>>>(
      gram, ld, gram_stride, rx, rx_stride, samples, samples_stride, dim, targets, K, Np, W,
      (T)eps, (T)p.w_l, qtab, base0, theta0, coeff, first_step, theta, n_active, status);
  return status_from(cudaGetLastError());
}

}  // namespace kapsm

extern "C" int kapsm_max_window(void) { return kapsm::TR_MAX_W; }

extern "C" int kapsm_max_samples(void) { return kapsm::TR_MAX_NP; }

#define KAPSM_TRAIN_ENTRY(NAME, T)                                                             \
  extern "C" int NAME(const T* gram, long long ld, long long gram_stride, const T* rx,         \
                      long long rx_stride, const T* samples, long long samples_stride, int dim, \
                      const T* targets, int F, int K, int n_samples, int window,               \
                      double epsilon, kapsm_kernel_params p, const T* qtab, const T* base0,    \
                      const T* theta0, T* coeff, int* first_step, T* theta, int* n_active,     \
                      int* status, void* stream) {                                             \
    return kapsm::train<T>(gram, ld, gram_stride, rx, rx_stride, samples, samples_stride, dim, \
                           targets, F, K, n_samples, window, epsilon, p, qtab, base0, theta0,  \
                           coeff, first_step, theta, n_active, status, (cudaStream_t)stream);  \
  }
KAPSM_TRAIN_ENTRY(kapsm_train_f32, float)
KAPSM_TRAIN_ENTRY(kapsm_train_f64, double)
