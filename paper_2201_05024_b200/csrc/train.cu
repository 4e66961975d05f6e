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
// Restatement used here (pilot Gram K from K1; all sums exact rearrangements
// of the reference's window response):
//   * every CRITICAL lane x owns one sample m (m = x mod 32) from step m-1 to
//     step m+30, keeping Y_m (response), c_m, first_step_m in registers, and
//     the slot-indexed column col2[x][l] = K[sample(l)][m] in shared memory;
//   * window update after step n's betas (one 32-term LDS.128 dot per lane):
//       Y_m += sum_l delta_l K[l][m]                      (m in J_n)
//   * the entering sample n+1 gets its full response from the same dot with
//     the coefficient vector instead of delta:
//       Y_{n+1} = sum_l c_l^(n+1) K[l][n+1] + P_{n+1},
//       P_m = f0(r_m) + sum_{i <= m-32} cfinal_i K[i][m]
//     P is streamed from Gram rows by BACKGROUND warps as soon as c_i is final
//     (sample i leaves the window after step i+W-1), several steps ahead;
//   * taking over sample n+2 needs one Gram row segment (32 values), staged by
//     cp.async TR_DELTA steps ahead; it refreshes one entry of every lane's
//     column and the whole column of the new lane (symmetry).
// Per step the critical warp runs ~130 instructions and one __syncwarp; it
// never waits on global memory, and P values arrive as tagged 64-bit words.
#include <type_traits>
#include "kapsm_common.cuh"

namespace kapsm {

constexpr int TR_S = 32;           // critical slots (one warp)
constexpr int TR_NB = 3;           // background warps (warps 0..2); critical = warp 3
constexpr int TR_G = TR_NB * 32;   // background lanes
constexpr int TR_NJ = 16;          // P accumulators per background lane (registers)
constexpr int TR_PD = 4;           // Gram-row prefetch depth of the background ring
constexpr int TR_DELTA = 8;        // column prefetch distance (steps)
constexpr int TR_PBN = 64;         // P slots (ring)
constexpr int TR_CR = 64;          // final-coefficient slots (ring, power of 2)
constexpr int TR_CSTR = TR_S + 4;  // col2 row stride: 16B rows, conflict-free LDS.128
constexpr int TR_STG = 16;         // staged Gram rows (ring, power of 2 >= DELTA+2)
constexpr int TR_MIN_LB = 7;       // minimum look-behind (background slack)
constexpr int TR_MAX_W = TR_S - 1 - TR_MIN_LB;
constexpr int TR_MAX_NP = TR_G * TR_NJ;
constexpr long long TR_SPIN_LIMIT = 1LL << 25;

// 32-term dot of two 16-byte aligned shared-memory vectors (LDS.128, 4 chains)
KAPSM_DEV float dot32(const float* a, const float* b) {
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 u = a4[q], w = b4[q];
    s0 = fmaf(u.x, w.x, s0);
    s1 = fmaf(u.y, w.y, s1);
    s2 = fmaf(u.z, w.z, s2);
    s3 = fmaf(u.w, w.w, s3);
  }
  return (s0 + s1) + (s2 + s3);
}
KAPSM_DEV double dot32(const double* a, const double* b) {
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
  for (int q = 0; q < 16; q += 2) {
    const double2 u = a2[q], w = b2[q], u2 = a2[q + 1], w2 = b2[q + 1];
    s0 = fma(u.x, w.x, s0);
    s1 = fma(u.y, w.y, s1);
    s2 = fma(u2.x, w2.x, s2);
    s3 = fma(u2.y, w2.y, s3);
  }
  return (s0 + s1) + (s2 + s3);
}

template <typename T>
struct TrainSmem {
  // byte offsets into dynamic shared memory
  size_t col, stage, bstage, dbuf, qsm, cfin, fsfin, pbuf, cring, ctl, total;
  __host__ __device__ TrainSmem(int W, int Np) {
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 15) & ~size_t(15); return r; };
    pbuf = take(TR_PBN * sizeof(typename Tagged<T>::slot_t));
    cring = take((TR_CR + 32) * sizeof(typename Tagged<T>::slot_t));
    col = take((size_t)TR_S * TR_CSTR * sizeof(T));
    stage = take((size_t)TR_STG * TR_S * sizeof(T));
    bstage = take((size_t)TR_STG * sizeof(T));
    dbuf = take(2 * 2 * TR_S * sizeof(T));
    qsm = take(2 * (size_t)W * sizeof(T));
    cfin = take((size_t)(Np + 32) * sizeof(T));
    fsfin = take((size_t)(Np + 32) * sizeof(int));
    ctl = take(16 * sizeof(int));
    total = o;
  }
};

template <typename T, int VAR = 0>
__global__ void __launch_bounds__((TR_NB + 1) * 32)
    apsm_train_kernel(const T* __restrict__ gram, long long ld, long long gram_stride,
                      const T* __restrict__ rx, long long rx_stride,
                      const T* __restrict__ samples, long long samples_stride, int dim,
                      const T* __restrict__ targets, int K, int Np, int W, T eps,
                      T w_l, const T* __restrict__ qtab, const T* __restrict__ base0,
                      const T* __restrict__ theta0, T* __restrict__ coeff_out,
                      int* __restrict__ fs_out, T* __restrict__ theta_out,
                      int* __restrict__ nact_out, int* __restrict__ status_out,
                      long long* __restrict__ dbg) {
  using Slot = typename Tagged<T>::slot_t;
  extern __shared__ __align__(16) unsigned char smem[];
  const TrainSmem<T> L(W, Np);
  Slot* pbuf = reinterpret_cast<Slot*>(smem + L.pbuf);   // [PBN]   tagged P_m
  Slot* cring = reinterpret_cast<Slot*>(smem + L.cring); // [CR+32] tagged final c_m (+junk)
  T* col2 = reinterpret_cast<T*>(smem + L.col);          // [S][CSTR]
  T* stage = reinterpret_cast<T*>(smem + L.stage);       // [STG][S]
  T* bstage = reinterpret_cast<T*>(smem + L.bstage);     // [STG]
  T* dbuf = reinterpret_cast<T*>(smem + L.dbuf);         // [2][2S]
  T* qsm = reinterpret_cast<T*>(smem + L.qsm);           // [W][2]
  T* cfin = reinterpret_cast<T*>(smem + L.cfin);         // [Np + 32]  (+junk)
  int* fsfin = reinterpret_cast<int*>(smem + L.fsfin);   // [Np + 32]  (+junk)
  int* ctl = reinterpret_cast<int*>(smem + L.ctl);       // [1]=abort [2]=status [3]=nact

  const int fu = blockIdx.x;                 // frame * K + user
  const int f = fu / K;
  const T* G = gram + (long long)f * gram_stride;
  const T* B = targets + (long long)fu * Np;  // realified targets (interleaved pilot symbols)
  const T* P0 = base0 ? base0 + (long long)fu * Np : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < TR_PBN; i += blockDim.x) Tagged<T>::store(&pbuf[i], T(0), -1);
  for (int i = threadIdx.x; i < TR_CR + 32; i += blockDim.x) Tagged<T>::store(&cring[i], T(0), -1);
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    T qm = T(1) / T(i + 1), ql = qm;
    if (qtab) { qm = qtab[2 * i]; ql = qtab[2 * i + 1]; }
    qsm[2 * i] = qm;
    qsm[2 * i + 1] = ql;
  }
  for (int i = threadIdx.x; i < Np + 32; i += blockDim.x) { cfin[i] = T(0); fsfin[i] = -1; }
  if (threadIdx.x < 16) ctl[threadIdx.x] = 0;
  __syncthreads();

  if (warp == TR_NB) {
    // =========================== CRITICAL WARP ===========================
    // Lane x owns sample m (m = x mod S) from step m-1 to step m+S-2; d = n-m
    // is its position relative to the current step (d = -1: enters next,
    // 0 <= d < W: in the window J_n, d = W-1: leaves after this step,
    // d = S-2: released, slot taken over by m+S).
    // col2[x][l] = K[sample(l)][m] for every owned sample(l).
    const int x = lane;
    for (int e = x; e < TR_S * TR_S; e += 32) {       // K[0..31][0..31]
      const int r = e / TR_S, l = e - r * TR_S;
      T* dst = col2 + r * TR_CSTR + l;
      if (r < Np && l < Np) cp_async_scalar(dst, G + (long long)r * ld + l);
      else *dst = T(0);
    }
    cp_async_commit();
    int m = x;
    T b = (m < Np) ? B[m] : T(0);
    cp_async_wait<0>();
    __syncwarp();
    T Y = (m == 0 && P0) ? P0[0] : T(0), c = T(0);
    int fs = -1, degen = 0;
    int d = (m < Np) ? -1 - x : -(1 << 29);
    const T den0 = (m < Np) ? col2[x * TR_CSTR + x] : T(1);
    degen |= (m < Np && !(den0 > T(0)));
    T invden = T(1) / den0;
    const T* myrow = col2 + x * TR_CSTR;
    const T qm_ss = qsm[2 * (W - 1)], ql_ss = qsm[2 * (W - 1) + 1];
    bool aborted = false;

    auto step = [&](const int n, auto steady_tag) {
      constexpr bool ST = decltype(steady_tag)::value;   // steady state: all branches known
      if (dbg && lane == 0 && fu == 0) dbg[n] = clock64();
      ++d;
      int J;
      T qm, ql;
      if constexpr (ST) {
        J = W; qm = qm_ss; ql = ql_ss;
      } else {
        J = n + 1 < W ? n + 1 : W;
        qm = qsm[2 * (J - 1)];
        ql = qsm[2 * (J - 1) + 1];
      }
      // (B) three-case beta on the window (apsm.py:323-335), branch-free
      const bool inwin = (unsigned)d < (unsigned)J;
      const T res = Y - b;
      const T bl = (-res - eps) * invden, bh = (-res + eps) * invden;
      T beta = res < -eps ? bl : (res > eps ? bh : T(0));
      beta = inwin ? beta : T(0);
      const T delta = (d == 0 ? ql : qm) * beta;
      c += delta;
      fs = (fs < 0 && beta != T(0)) ? n : fs;
      const bool enter = (d == -1);
      // (M) Y_m += sum_l delta_l K[l][m]; the entering sample n+1 instead gets
      //     its full response sum_l c_l K[l][n+1] (+ P_{n+1} below).  The two
      //     vectors are broadcast through shared memory (one STS each, one
      //     __syncwarp, LDS.128 reads) -- measured faster than 32 shuffles.
      T* vecs = dbuf + (n & 1) * 2 * TR_S;     // [0,S): delta, [S,2S): c
      vecs[x] = delta;
      vecs[TR_S + x] = c;
      __syncwarp();
      const T acc = (VAR & 4) ? T(0) : dot32(vecs + (enter ? TR_S : 0), myrow);
      T pv = T(0);
      if (ST || n + 1 < Np) {
        const int me = n + 1;
        if (!Tagged<T>::load(&pbuf[me % TR_PBN], me, pv)) {   // warp-uniform, rare
          long long spins = 0;
          while (!Tagged<T>::load(&pbuf[me % TR_PBN], me, pv))
            if (++spins > TR_SPIN_LIMIT) { aborted = true; break; }
          if (dbg && lane == 0 && fu == 0) dbg[Np + n] = spins + 1;
        }
      }
      Y = enter ? acc + pv : Y + acc;
      // (L) sample lo leaves the window after this step: c is final.  Every lane
      //     stores (non-leaving lanes into junk slots), so there is no branch.
      {
        const bool leave = (d == W - 1);
        const int li = leave ? m : Np + x;
        cfin[li] = c;
        fsfin[li] = fs;
        Tagged<T>::store(&cring[leave ? (m & (TR_CR - 1)) : TR_CR + x], c, leave ? m : -1);
      }
      // (P) stage the Gram row of the sample taken over TR_DELTA steps later,
      //     restricted to the samples owned after that takeover
      {
        const int t = n + TR_DELTA, mt = t + 2;
        if (!(VAR & 2) && (ST || (mt >= TR_S && mt < Np))) {
          const int sx = mt - ((mt - x) & (TR_S - 1));      // owned by slot x after takeover
          T* dst = stage + (t & (TR_STG - 1)) * TR_S + x;
          if (ST || sx >= 0) cp_async_scalar(dst, G + (long long)mt * ld + sx);
          if (x == 0) cp_async_scalar(bstage + (t & (TR_STG - 1)), B + mt);
        }
        cp_async_commit();
      }
      // (T) release sample n+2-S, take over sample n+2
      const int mt = n + 2;
      if (!(VAR & 2) && (ST || (mt >= TR_S && mt < Np))) {
        cp_async_wait<TR_DELTA>();
        __syncwarp();
        const int r = mt & (TR_S - 1);
        const T v = stage[(n & (TR_STG - 1)) * TR_S + x];   // K[mt][sample(x)]
        const T bn = bstage[n & (TR_STG - 1)];
        col2[x * TR_CSTR + r] = v;
        col2[r * TR_CSTR + x] = v;
        const T dnew = __shfl_sync(0xffffffffu, v, r);      // K[mt][mt], warp-uniform
        degen |= !(dnew > T(0));
        const bool take = (x == r);
        T inew;
        if constexpr (sizeof(T) == 4) inew = __fdividef(1.0f, dnew);
        else inew = T(1) / dnew;
        m = take ? mt : m;
        d = take ? -2 : d;
        c = take ? T(0) : c;
        fs = take ? -1 : fs;
        b = take ? bn : b;
        invden = take ? inew : invden;
      }
    };

    // steady phase: full window, prefetch and takeover always in range
    const int nB0 = (TR_S - 2 > W - 1 ? TR_S - 2 : W - 1) < Np ? (TR_S - 2 > W - 1 ? TR_S - 2 : W - 1) : Np;
    int nB1 = Np - TR_DELTA - 2;
    if (nB1 < nB0) nB1 = nB0;
    int n = 0;
    for (; n < nB0 && !aborted; ++n) step(n, std::false_type{});
    for (; n < nB1 && !aborted; ++n) step(n, std::true_type{});
    for (; n < Np && !aborted; ++n) step(n, std::false_type{});
    // remaining window samples (those that did not leave at the last step)
    if (!aborted && m < Np && d >= 0 && d < W - 1) {
      cfin[m] = c;
      fsfin[m] = fs;
    }
    const bool any_degen = __any_sync(0xffffffffu, degen != 0);
    __syncwarp();
    if (lane == 0) {
      if (any_degen) atomicOr(&ctl[2], KAPSM_TRAIN_DEGENERATE);
      if (aborted) { atomicOr(&ctl[2], KAPSM_TRAIN_STALLED); st_volatile(&ctl[1], 1); }
    }
  } else {
    // ========================== BACKGROUND WARPS =========================
    // lane g owns P accumulators for samples m = g + G*j (j < TR_NJ); for every
    // final coefficient c_f (tagged ring, in order) it streams Gram row f:
    //   P_m += c_f K[f][m]   (m >= f + S),   and publishes P_{f+S}.
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
          T cf;
          long long spins = 0;
          while (!Tagged<T>::load(&cring[fi & (TR_CR - 1)], fi, cf)) {
            if (((++spins) & 1023) == 0 && (spins > TR_SPIN_LIMIT || ld_volatile(&ctl[1]))) {
              stop = true;
              break;
            }
          }
          if (!stop) {
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
    if (stop && lane == 0) { atomicOr(&ctl[2], KAPSM_TRAIN_STALLED); st_volatile(&ctl[1], 1); }
  }
  __syncthreads();
  // ---- outputs: coefficients, first steps (coalesced), activation count ----
  {
    int na = 0;
    for (int i = threadIdx.x; i < Np; i += blockDim.x) {
      coeff_out[(long long)fu * Np + i] = cfin[i];
      const int v = fsfin[i];
      fs_out[(long long)fu * Np + i] = v;
      na += (v >= 0);
    }
    na = (int)warp_sum((float)na);
    if (lane == 0) atomicAdd(&ctl[3], na);
  }
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
  __syncthreads();
  if (threadIdx.x == 0) {
    status_out[fu] = ctl[2];
    nact_out[fu] = ctl[3];
  }
}

template <typename T, int VAR>
int launch_train(dim3 grid, size_t smem, cudaStream_t s, const T* gram, long long ld,
                 long long gram_stride, const T* rx, long long rx_stride, const T* samples,
                 long long samples_stride, int dim, const T* targets, int K, int Np, int W,
                 double eps, kapsm_kernel_params p, const T* qtab, const T* base0,
                 const T* theta0, T* coeff, int* first_step, T* theta, int* n_active, int* status,
                 long long* dbg) {
  auto kern = apsm_train_kernel<T, VAR>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  kern<<<grid, (TR_NB + 1) * 32, smem, s>>>(gram, ld, gram_stride, rx, rx_stride, samples,
                                            samples_stride, dim, targets, K, Np, W, (T)eps,
                                            (T)p.w_l, qtab, base0, theta0, coeff, first_step,
                                            theta, n_active, status, dbg);
  return status_from(cudaGetLastError());
}

template <typename T>
int train(const T* gram, long long ld, long long gram_stride, const T* rx, long long rx_stride,
          const T* samples, long long samples_stride, int dim, const T* targets, int F, int K,
          int Np, int W, double eps, kapsm_kernel_params p, const T* qtab, const T* base0,
          const T* theta0, T* coeff, int* first_step, T* theta, int* n_active, int* status,
          cudaStream_t s, long long* dbg = nullptr, int variant = 0) {
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
#define KAPSM_LT(V)                                                                          \
  return launch_train<T, V>(dim3(F * K), L.total, s, gram, ld, gram_stride, rx, rx_stride,   \
                            samples, samples_stride, dim, targets, K, Np, W, eps, p, qtab,   \
                            base0, theta0, coeff, first_step, theta, n_active, status, dbg)
  switch (variant) {
    case 1: KAPSM_LT(1);
    case 2: KAPSM_LT(2);
    case 3: KAPSM_LT(3);
    case 4: KAPSM_LT(4);
    case 8: KAPSM_LT(8);
    case 15: KAPSM_LT(15);
    default: KAPSM_LT(0);
  }
#undef KAPSM_LT
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

// Internal instrumentation entry (not part of the public ABI): as
// kapsm_train_f32, plus clock64() at the top of every step of (frame 0, user 0).
extern "C" int kapsm_internal_train_clock_f32(const float* gram, long long ld,
                                              long long gram_stride, const float* rx,
                                              long long rx_stride, const float* targets, int F,
                                              int K, int n_samples, int dim, int window,
                                              double epsilon, kapsm_kernel_params p,
                                              const float* qtab, float* coeff, int* first_step,
                                              float* theta, int* n_active, int* status,
                                              long long* clocks, int variant, void* stream) {
  return kapsm::train<float>(gram, ld, gram_stride, rx, rx_stride, nullptr, 0, dim, targets, F, K,
                             n_samples, window, epsilon, p, qtab, nullptr, nullptr, coeff,
                             first_step, theta, n_active, status, (cudaStream_t)stream, clocks,
                             variant);
}
