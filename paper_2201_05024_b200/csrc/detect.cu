// K3: fused frame detection + generic filter evaluation, demap, error count.
//
// Frame mode (kapsm_detect_frames_*): every user's trained filter has its
// Gaussian atoms on the frame's own realified pilots (apsm.py:341-359), so the
// pilot/payload kernel block is SHARED by all K users of a frame.  One pass
// over (pilot symbol p, payload symbol t) pairs computes, from ONE complex dot
// x_p^H y_t, the four realified kernel values (apsm.py:156-182 structure):
//   kG(r1x,r1y) = kG(r2x,r2y) = exp(-(|x|^2+|y|^2-2Re x^H y)/2s^2)
//   kG(r1x,r2y) = exp(-(|x|^2+|y|^2-2Im x^H y)/2s^2)
//   kG(r2x,r1y) = exp(-(|x|^2+|y|^2+2Im x^H y)/2s^2)
// and contracts them with all K users' coefficients.  The epilogue adds the
// linear part theta_u . r(y) (kernels.py:194-206), recombines
// g(r) = f(r1) + i f(r2) (engine.py:261), takes the hard decision
// (demodulate_hard, noma.py:125-135: nearest point, ties to the lowest index)
// and counts bit / symbol errors against the transmitted labels
// (ber, noma.py:284-292).  No intermediate touches HBM.
//
// Precision: the distance uses the norm expansion (one complex FMA chain per
// pair); pairs whose kernel is live at large norms (cancellation-prone) are
// recomputed with explicit differences, pairs whose kernel underflows for the
// whole warp skip the exponentials and the user contraction.
#include "kapsm_common.cuh"

namespace kapsm {

constexpr int DT_WARPS = 8;     // pilot split inside a CTA

template <typename T> struct Thresh;
template <> struct Thresh<float> {
  static constexpr float dead = 88.0f;     // exp(-88) underflows FP32 (ftz)
  static constexpr float live = 12.0f;     // kernel > 6e-6: refine if norms are large
  static constexpr float bignorm = 64.0f;  // (|x|^2+|y|^2)/2s^2 above which expansion loses digits
  static constexpr bool refine = true;
};
template <> struct Thresh<double> {
  static constexpr double dead = 745.0;
  static constexpr double live = 0.0;
  static constexpr double bignorm = 1e300;
  static constexpr bool refine = false;
};

template <typename T, int MT>
KAPSM_DEV void cdot(const T* __restrict__ x, const T (&y)[2 * MT], T& cr, T& ci) {
  // x^H y for MT complex entries; x is a 16-byte aligned shared-memory row
  T r0 = T(0), r1 = T(0), i0 = T(0), i1 = T(0);
  if constexpr (sizeof(T) == 4) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll
    for (int q = 0; q < MT / 2; ++q) {
      const float4 v = x4[q];            // (xr_k, xi_k, xr_k+1, xi_k+1)
      r0 = fmaf(v.x, y[4 * q], r0);     r1 = fmaf(v.y, y[4 * q + 1], r1);
      i0 = fmaf(v.x, y[4 * q + 1], i0); i1 = fmaf(v.y, y[4 * q], i1);
      r0 = fmaf(v.z, y[4 * q + 2], r0); r1 = fmaf(v.w, y[4 * q + 3], r1);
      i0 = fmaf(v.z, y[4 * q + 3], i0); i1 = fmaf(v.w, y[4 * q + 2], i1);
    }
  } else {
    const double2* x2 = reinterpret_cast<const double2*>(x);
#pragma unroll
    for (int k = 0; k < MT; ++k) {
      const double2 v = x2[k];
      r0 = fma(v.x, y[2 * k], r0);     r1 = fma(v.y, y[2 * k + 1], r1);
      i0 = fma(v.x, y[2 * k + 1], i0); i1 = fma(v.y, y[2 * k], i1);
    }
  }
  cr = r0 + r1;
  ci = i0 - i1;
}

// One (pilot, payload) pair: distances from the expansion, refine when a live
// kernel meets large norms, exp, contract with every user's coefficients.
template <typename T, int MT, int KT>
KAPSM_DEV void pair_update(const T* x, T nx, const T* cp, const T (&y)[2 * MT], T ny, T cr, T ci,
                           bool tvalid, T inv2s, T (&are)[KT], T (&aim)[KT]) {
  const T s = nx + ny;
  T da = s - T(2) * cr, db = s - T(2) * ci, dc = s + T(2) * ci;
  const T dmin = fmin(da, fmin(db, dc));
  const bool live = tvalid && dmin * inv2s < Thresh<T>::dead;
  if (Thresh<T>::refine && live && dmin * inv2s < Thresh<T>::live && s * inv2s > Thresh<T>::bignorm) {
    T ea = T(0), eb = T(0), ec = T(0);
#pragma unroll
    for (int k = 0; k < MT; ++k) {
      const T xr = x[2 * k], xi = x[2 * k + 1], yr = y[2 * k], yi = y[2 * k + 1];
      T a0 = xr - yr, a1 = xi - yi;
      ea = fma(a0, a0, fma(a1, a1, ea));
      a0 = xr - yi; a1 = xi + yr;
      eb = fma(a0, a0, fma(a1, a1, eb));
      a0 = xr + yi; a1 = xi - yr;
      ec = fma(a0, a0, fma(a1, a1, ec));
    }
    da = ea; db = eb; dc = ec;
  }
  T ka = T(0), kb = T(0), kc = T(0);
  if (live) {
    ka = exp_fast(-fmax(da, T(0)) * inv2s);
    kb = exp_fast(-fmax(db, T(0)) * inv2s);
    kc = exp_fast(-fmax(dc, T(0)) * inv2s);
  }
#pragma unroll
  for (int u = 0; u < KT; ++u) {
    const T c1 = cp[2 * u], c2 = cp[2 * u + 1];
    are[u] = fma(c1, ka, fma(c2, kc, are[u]));
    aim[u] = fma(c1, kb, fma(c2, ka, aim[u]));
  }
}

template <typename T, int MT, int KT>
__global__ void __launch_bounds__(DT_WARPS * 32)
    detect_frames_kernel(const T* __restrict__ rx, long long rx_stride, int K, int n_train,
                         int n_data, int M, int PC, const T* __restrict__ coeff,
                         const T* __restrict__ theta, T w_g, T inv2s,
                         const T* __restrict__ points, int n_points, int bps,
                         const unsigned char* __restrict__ tx_labels, T* __restrict__ est_out,
                         unsigned char* __restrict__ labels_out,
                         unsigned long long* __restrict__ bit_err,
                         unsigned long long* __restrict__ sym_err) {
  extern __shared__ __align__(16) unsigned char smem[];
  // layout: pts[64][2] | xs[PC][2*MT] | nxs[PC] | cs[PC][2*KT]; the epilogue's
  // reduction buffer reuses the chunk area (never the points)
  T* pts = reinterpret_cast<T*>(smem);
  T* xs = pts + 128;
  T* nxs = xs + (size_t)PC * 2 * MT;
  T* cs = nxs + PC;
  const int f = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 32 + lane;
  const bool tvalid = t < n_data;
  const T* Xf = rx + (long long)f * rx_stride;
  const int Np = 2 * n_train;

  for (int i = threadIdx.x; i < 2 * n_points; i += blockDim.x) pts[i] = points[i];

  T y[2 * MT];
  T ny = T(0);
  {
    const T* yp = Xf + (long long)(n_train + (tvalid ? t : 0)) * 2 * M;
#pragma unroll
    for (int k = 0; k < MT; ++k) {
      const bool in = tvalid && k < M;
      y[2 * k] = in ? yp[2 * k] : T(0);
      y[2 * k + 1] = in ? yp[2 * k + 1] : T(0);
      ny = fma(y[2 * k], y[2 * k], fma(y[2 * k + 1], y[2 * k + 1], ny));
    }
  }
  T are[KT], aim[KT];
#pragma unroll
  for (int u = 0; u < KT; ++u) { are[u] = T(0); aim[u] = T(0); }

  for (int c0 = 0; c0 < n_train; c0 += PC) {
    const int pc = min(PC, n_train - c0);
    __syncthreads();
    // ---- stage the chunk: pilots (async copies), coefficients of all users ----
    if (M == MT) {
      const int nvec = pc * 2 * MT * (int)sizeof(T) / 16;
      const char* src = reinterpret_cast<const char*>(Xf + (long long)c0 * 2 * M);
      char* dst = reinterpret_cast<char*>(xs);
      for (int e = threadIdx.x; e < nvec; e += blockDim.x) {
        unsigned d = (unsigned)__cvta_generic_to_shared(dst + 16 * e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + 16 * (long long)e)
                     : "memory");
      }
      cp_async_commit();
    } else {
      for (int e = threadIdx.x; e < pc * MT; e += blockDim.x) {
        const int p = e / MT, k = e - p * MT;
        T xr = T(0), xi = T(0);
        if (k < M) {
          const T* xp = Xf + (long long)(c0 + p) * 2 * M + 2 * k;
          xr = xp[0]; xi = xp[1];
        }
        xs[p * 2 * MT + 2 * k] = xr;
        xs[p * 2 * MT + 2 * k + 1] = xi;
      }
    }
    using V2 = typename Vec2<T>::type;
    for (int e = threadIdx.x; e < pc * KT; e += blockDim.x) {
      const int u = e / pc, p = e - u * pc;          // consecutive threads -> consecutive pilots
      V2 cc;
      cc.x = T(0); cc.y = T(0);
      if (u < K) cc = *reinterpret_cast<const V2*>(coeff + ((long long)f * K + u) * Np + 2 * (c0 + p));
      *reinterpret_cast<V2*>(cs + p * 2 * KT + 2 * u) = cc;
    }
    if (M == MT) cp_async_wait<0>();
    __syncthreads();
    for (int p = threadIdx.x; p < pc; p += blockDim.x) {
      T sacc = T(0);
#pragma unroll 8
      for (int k = 0; k < 2 * MT; ++k) sacc = fma(xs[p * 2 * MT + k], xs[p * 2 * MT + k], sacc);
      nxs[p] = sacc;
    }
    __syncthreads();
    // ---- pairs: two pilots per iteration for ILP ----
    int p = warp;
    for (; p + DT_WARPS < pc; p += 2 * DT_WARPS) {
      const int q = p + DT_WARPS;
      const T* xp = xs + p * 2 * MT;
      const T* xq = xs + q * 2 * MT;
      T crp, cip, crq, ciq;
      cdot<T, MT>(xp, y, crp, cip);
      cdot<T, MT>(xq, y, crq, ciq);
      const T np_ = nxs[p], nq_ = nxs[q];
      const T dp = np_ + ny - T(2) * fmax(crp, fabs(cip));
      const T dq = nq_ + ny - T(2) * fmax(crq, fabs(ciq));
      const bool lp = tvalid && dp * inv2s < Thresh<T>::dead;
      const bool lq = tvalid && dq * inv2s < Thresh<T>::dead;
      if (__any_sync(0xffffffffu, lp))
        pair_update<T, MT, KT>(xp, np_, cs + p * 2 * KT, y, ny, crp, cip, tvalid, inv2s, are, aim);
      if (__any_sync(0xffffffffu, lq))
        pair_update<T, MT, KT>(xq, nq_, cs + q * 2 * KT, y, ny, crq, ciq, tvalid, inv2s, are, aim);
    }
    for (; p < pc; p += DT_WARPS) {
      const T* xp = xs + p * 2 * MT;
      T crp, cip;
      cdot<T, MT>(xp, y, crp, cip);
      const T np_ = nxs[p];
      const T dp = np_ + ny - T(2) * fmax(crp, fabs(cip));
      const bool lp = tvalid && dp * inv2s < Thresh<T>::dead;
      if (__any_sync(0xffffffffu, lp))
        pair_update<T, MT, KT>(xp, np_, cs + p * 2 * KT, y, ny, crp, cip, tvalid, inv2s, are, aim);
    }
  }
  __syncthreads();
  // ---- cross-warp reduction (fixed order -> deterministic) ----
  T* red = xs;   // [DT_WARPS][KT][2][32]
#pragma unroll
  for (int u = 0; u < KT; ++u) {
    red[((warp * KT + u) * 2 + 0) * 32 + lane] = are[u];
    red[((warp * KT + u) * 2 + 1) * 32 + lane] = aim[u];
  }
  __syncthreads();
  unsigned long long be = 0, se = 0;
  for (int u = warp; u < K; u += DT_WARPS) {
    T gr = T(0), gi = T(0);
    for (int w = 0; w < DT_WARPS; ++w) {
      gr += red[((w * KT + u) * 2 + 0) * 32 + lane];
      gi += red[((w * KT + u) * 2 + 1) * 32 + lane];
    }
    // linear part: conj(Theta_u) . y  (Theta = theta[:M] + i theta[M:])
    const T* th = theta + ((long long)f * K + u) * 2 * M;
    T lr = T(0), li = T(0);
#pragma unroll
    for (int k = 0; k < MT; ++k) {
      if (k < M) {
        const T tr = th[k], ti = th[M + k];
        lr = fma(tr, y[2 * k], fma(ti, y[2 * k + 1], lr));
        li = fma(tr, y[2 * k + 1], fma(-ti, y[2 * k], li));
      }
    }
    const T er = lr + w_g * gr, ei = li + w_g * gi;
    // hard decision: nearest constellation point, ties -> lowest index
    int best = 0;
    T bd = T(0);
    for (int q = 0; q < n_points; ++q) {
      const T dr = er - pts[2 * q], di = ei - pts[2 * q + 1];
      const T d = dr * dr + di * di;
      if (q == 0 || d < bd) { bd = d; best = q; }
    }
    if (tvalid) {
      const long long o = ((long long)f * K + u) * n_data + t;
      if (est_out) { est_out[2 * o] = er; est_out[2 * o + 1] = ei; }
      if (labels_out) labels_out[o] = (unsigned char)best;
      if (tx_labels) {
        const unsigned tx = tx_labels[o];
        be = __popc((unsigned)best ^ tx);
        se = ((unsigned)best != tx) ? 1ull : 0ull;
      }
    }
    if (tx_labels && (bit_err || sym_err)) {
      const unsigned long long bsum = warp_sum_u64(be), ssum = warp_sum_u64(se);
      if (lane == 0) {
        if (bit_err && bsum) atomicAdd(&bit_err[(long long)f * K + u], bsum);
        if (sym_err && ssum) atomicAdd(&sym_err[(long long)f * K + u], ssum);
      }
    }
    be = se = 0;
  }
  (void)bps;
}

template <typename T, int MT, int KT>
int launch_detect(const T* rx, long long rx_stride, int F, int K, int n_train, int n_data, int M,
                  const T* coeff, const T* theta, kapsm_kernel_params p, const T* points,
                  int n_points, int bps, const unsigned char* tx, T* est, unsigned char* labels,
                  unsigned long long* be, unsigned long long* se, cudaStream_t s) {
  // pilot chunk: as many pilots as fit in ~100 KB (two CTAs per SM), multiple of 8
  const size_t per_pilot = (2 * MT + 1 + 2 * KT) * sizeof(T);
  int PC = (int)((100 * 1024 - 128 * sizeof(T)) / per_pilot);
  PC = PC / 8 * 8;
  if (PC > n_train) PC = (n_train + 7) / 8 * 8;
  if (PC < 8) PC = 8;
  size_t chunk = (size_t)PC * per_pilot + 16;
  size_t redb = (size_t)DT_WARPS * KT * 2 * 32 * sizeof(T);
  size_t smem = 128 * sizeof(T) + (chunk > redb ? chunk : redb);
  auto kern = detect_frames_kernel<T, MT, KT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  dim3 grid((n_data + 31) / 32, F);
  kern<<<grid, DT_WARPS * 32, smem, s>>>(rx, rx_stride, K, n_train, n_data, M, PC, coeff, theta,
                                         (T)p.w_g, (T)(1.0 / (2.0 * p.sigma_sq)), points,
                                         n_points, bps, tx, est, labels, be, se);
  return status_from(cudaGetLastError());
}

template <typename T, int MT>
int dispatch_k(int K, const T* rx, long long rx_stride, int F, int n_train, int n_data, int M,
               const T* coeff, const T* theta, kapsm_kernel_params p, const T* points,
               int n_points, int bps, const unsigned char* tx, T* est, unsigned char* labels,
               unsigned long long* be, unsigned long long* se, cudaStream_t s) {
  if (K <= 2)
    return launch_detect<T, MT, 2>(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p,
                                   points, n_points, bps, tx, est, labels, be, se, s);
  if (K <= 4)
    return launch_detect<T, MT, 4>(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p,
                                   points, n_points, bps, tx, est, labels, be, se, s);
  if (K <= 8)
    return launch_detect<T, MT, 8>(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p,
                                   points, n_points, bps, tx, est, labels, be, se, s);
  if (K <= 16)
    return launch_detect<T, MT, 16>(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p,
                                    points, n_points, bps, tx, est, labels, be, se, s);
  return KAPSM_ERR_UNSUPPORTED;
}

template <typename T>
int detect_frames(const T* rx, long long rx_stride, int F, int K, int n_train, int n_data, int M,
                  const T* coeff, const T* theta, kapsm_kernel_params p, const T* points,
                  int n_points, int bps, const unsigned char* tx, T* est, unsigned char* labels,
                  unsigned long long* be, unsigned long long* se, cudaStream_t s) {
  if (F < 0 || K < 1 || n_train < 0 || n_data < 0 || M < 1 || !rx || !coeff || !theta ||
      !points || n_points < 1 || n_points > 64)
    return KAPSM_ERR_INVALID;
  if ((be || se) && !tx) return KAPSM_ERR_INVALID;
  if (F == 0 || n_data == 0) return KAPSM_OK;
#define KAPSM_DK(MTV) \
  return dispatch_k<T, MTV>(K, rx, rx_stride, F, n_train, n_data, M, coeff, theta, p, points, \
                            n_points, bps, tx, est, labels, be, se, s)
  if (M <= 4) KAPSM_DK(4);
  if (M <= 8) KAPSM_DK(8);
  if (M <= 16) KAPSM_DK(16);
  if (M <= 32) KAPSM_DK(32);
  if (M <= 64) KAPSM_DK(64);       // FP64 at M = 64 spills its row registers: the
                                   // parity twin of the C4 config, not a fast path
#undef KAPSM_DK
  return KAPSM_ERR_UNSUPPORTED;
}

// ---------------------------------------------------------------------------
// Generic batch_evaluate (engine.py:206-243) of one filter on realified rows.
// Thread per input row; atoms streamed through shared memory in chunks; the
// squared distance uses explicit differences (kernels.py:187-191) so there is
// no cancellation at any norm.
// ---------------------------------------------------------------------------
constexpr int EV_THREADS = 128;
constexpr int EV_AC = 64;   // atoms per chunk

template <typename T, int DT>
__global__ void __launch_bounds__(EV_THREADS)
    evaluate_kernel(const T* __restrict__ theta, const T* __restrict__ atoms,
                    const T* __restrict__ coeffs, int n_atoms, int dim,
                    const T* __restrict__ inputs, int n_inputs, T w_g, T inv2s,
                    T* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* as = reinterpret_cast<T*>(smem);    // [EV_AC][DT]
  T* gs = as + EV_AC * DT;               // [EV_AC]
  const int n = blockIdx.x * EV_THREADS + threadIdx.x;
  const bool valid = n < n_inputs;
  T u[DT];
  T lin = T(0);
#pragma unroll
  for (int k = 0; k < DT; ++k) {
    const bool in = valid && k < dim;
    u[k] = in ? inputs[(long long)n * dim + k] : T(0);
    lin = fma(in ? theta[k] : T(0), u[k], lin);
  }
  T acc = T(0);
  if (w_g != T(0)) {
    for (int a0 = 0; a0 < n_atoms; a0 += EV_AC) {
      const int ac = min(EV_AC, n_atoms - a0);
      __syncthreads();
      for (int e = threadIdx.x; e < EV_AC * DT; e += EV_THREADS) {
        const int a = e / DT, k = e - a * DT;
        as[e] = (a < ac && k < dim) ? atoms[(long long)(a0 + a) * dim + k] : T(0);
      }
      for (int a = threadIdx.x; a < EV_AC; a += EV_THREADS) gs[a] = a < ac ? coeffs[a0 + a] : T(0);
      __syncthreads();
      for (int a = 0; a < ac; ++a) {
        const T* ap = as + a * DT;
        T d0 = T(0), d1 = T(0);
#pragma unroll
        for (int k = 0; k < DT; k += 2) {
          const T e0 = ap[k] - u[k];
          d0 = fma(e0, e0, d0);
          if (k + 1 < DT) {
            const T e1 = ap[k + 1] - u[k + 1];
            d1 = fma(e1, e1, d1);
          }
        }
        const T d2 = d0 + d1;
        if (d2 * inv2s < Thresh<T>::dead) acc = fma(gs[a], exp_acc(-d2 * inv2s), acc);
      }
    }
  }
  if (valid) out[n] = lin + w_g * acc;
}

template <typename T, int DT>
int launch_evaluate(const T* theta, const T* atoms, const T* coeffs, int n_atoms, int dim,
                    const T* inputs, int n_inputs, kapsm_kernel_params p, T* out,
                    cudaStream_t s) {
  size_t smem = (size_t)EV_AC * (DT + 1) * sizeof(T);
  auto kern = evaluate_kernel<T, DT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  kern<<<(n_inputs + EV_THREADS - 1) / EV_THREADS, EV_THREADS, smem, s>>>(
      theta, atoms, coeffs, n_atoms, dim, inputs, n_inputs, (T)p.w_g,
      (T)(1.0 / (2.0 * p.sigma_sq)), out);
  return status_from(cudaGetLastError());
}

template <typename T>
int batch_evaluate(const T* theta, const T* atoms, const T* coeffs, int n_atoms, int dim,
                   const T* inputs, int n_inputs, kapsm_kernel_params p, T* out, cudaStream_t s) {
  if (dim < 1 || n_atoms < 0 || n_inputs < 0 || !theta || !out || (n_inputs && !inputs) ||
      (n_atoms && (!atoms || !coeffs)))
    return KAPSM_ERR_INVALID;
  if (n_inputs == 0) return KAPSM_OK;
  if (dim <= 8) return launch_evaluate<T, 8>(theta, atoms, coeffs, n_atoms, dim, inputs, n_inputs, p, out, s);
  if (dim <= 16) return launch_evaluate<T, 16>(theta, atoms, coeffs, n_atoms, dim, inputs, n_inputs, p, out, s);
  if (dim <= 32) return launch_evaluate<T, 32>(theta, atoms, coeffs, n_atoms, dim, inputs, n_inputs, p, out, s);
  if (dim <= 64) return launch_evaluate<T, 64>(theta, atoms, coeffs, n_atoms, dim, inputs, n_inputs, p, out, s);
  if (dim <= 128) return launch_evaluate<T, 128>(theta, atoms, coeffs, n_atoms, dim, inputs, n_inputs, p, out, s);
  return KAPSM_ERR_UNSUPPORTED;
}


// batch_detect (engine.py:246-261) of one FilterState on complex inputs:
// out[t] = f(r1(y_t)) + i f(r2(y_t)), r1 = [Re y; Im y], r2 = [Im y; -Re y]
// (realify_batch, apsm.py:172-182) -- the realification is done in registers.
template <typename T, int MT>
__global__ void __launch_bounds__(EV_THREADS)
    detect_complex_kernel(const T* __restrict__ theta, const T* __restrict__ atoms,
                          const T* __restrict__ coeffs, int n_atoms, int M,
                          const T* __restrict__ rx, int n_inputs, T w_g, T inv2s,
                          T* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* as = reinterpret_cast<T*>(smem);    // [EV_AC][2*MT]  (re block, im block)
  T* gs = as + EV_AC * 2 * MT;           // [EV_AC]
  const int t = blockIdx.x * EV_THREADS + threadIdx.x;
  const bool valid = t < n_inputs;
  const int D = 2 * M;
  T yr[MT], yi[MT];
  T l1 = T(0), l2 = T(0);
#pragma unroll
  for (int k = 0; k < MT; ++k) {
    const bool in = valid && k < M;
    yr[k] = in ? rx[(long long)t * D + 2 * k] : T(0);
    yi[k] = in ? rx[(long long)t * D + 2 * k + 1] : T(0);
    const T tr = k < M ? theta[k] : T(0), ti = k < M ? theta[M + k] : T(0);
    l1 = fma(tr, yr[k], fma(ti, yi[k], l1));
    l2 = fma(tr, yi[k], fma(-ti, yr[k], l2));
  }
  T acc1 = T(0), acc2 = T(0);
  if (w_g != T(0)) {
    for (int a0 = 0; a0 < n_atoms; a0 += EV_AC) {
      const int ac = min(EV_AC, n_atoms - a0);
      __syncthreads();
      for (int e = threadIdx.x; e < EV_AC * 2 * MT; e += EV_THREADS) {
        const int a = e / (2 * MT), r = e - a * 2 * MT;
        const int half = r / MT, k = r - half * MT;
        as[e] = (a < ac && k < M) ? atoms[(long long)(a0 + a) * D + half * M + k] : T(0);
      }
      for (int a = threadIdx.x; a < EV_AC; a += EV_THREADS) gs[a] = a < ac ? coeffs[a0 + a] : T(0);
      __syncthreads();
      for (int a = 0; a < ac; ++a) {
        const T* ar = as + a * 2 * MT;
        const T* ai = ar + MT;
        T d1 = T(0), d2 = T(0);
#pragma unroll
        for (int k = 0; k < MT; ++k) {
          T e0 = ar[k] - yr[k], e1 = ai[k] - yi[k];
          d1 = fma(e0, e0, fma(e1, e1, d1));
          e0 = ar[k] - yi[k]; e1 = ai[k] + yr[k];
          d2 = fma(e0, e0, fma(e1, e1, d2));
        }
        const T g = gs[a];
        if (d1 * inv2s < Thresh<T>::dead) acc1 = fma(g, exp_acc(-d1 * inv2s), acc1);
        if (d2 * inv2s < Thresh<T>::dead) acc2 = fma(g, exp_acc(-d2 * inv2s), acc2);
      }
    }
  }
  if (valid) {
    out[2 * (long long)t] = l1 + w_g * acc1;
    out[2 * (long long)t + 1] = l2 + w_g * acc2;
  }
}

template <typename T, int MT>
int launch_detect_complex(const T* theta, const T* atoms, const T* coeffs, int n_atoms, int M,
                          const T* rx, int n, kapsm_kernel_params p, T* out, cudaStream_t s) {
  size_t smem = (size_t)EV_AC * (2 * MT + 1) * sizeof(T);
  auto kern = detect_complex_kernel<T, MT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  kern<<<(n + EV_THREADS - 1) / EV_THREADS, EV_THREADS, smem, s>>>(
      theta, atoms, coeffs, n_atoms, M, rx, n, (T)p.w_g, (T)(1.0 / (2.0 * p.sigma_sq)), out);
  return status_from(cudaGetLastError());
}

template <typename T>
int batch_detect(const T* theta, const T* atoms, const T* coeffs, int n_atoms, int dim,
                 const T* rx, int n, kapsm_kernel_params p, T* out, cudaStream_t s) {
  if (dim < 2 || (dim & 1) || n_atoms < 0 || n < 0 || !theta || !out || (n && !rx) ||
      (n_atoms && (!atoms || !coeffs)))
    return KAPSM_ERR_INVALID;
  if (n == 0) return KAPSM_OK;
  const int M = dim / 2;
  if (M <= 4) return launch_detect_complex<T, 4>(theta, atoms, coeffs, n_atoms, M, rx, n, p, out, s);
  if (M <= 8) return launch_detect_complex<T, 8>(theta, atoms, coeffs, n_atoms, M, rx, n, p, out, s);
  if (M <= 16) return launch_detect_complex<T, 16>(theta, atoms, coeffs, n_atoms, M, rx, n, p, out, s);
  if (M <= 32) return launch_detect_complex<T, 32>(theta, atoms, coeffs, n_atoms, M, rx, n, p, out, s);
  if (M <= 64) return launch_detect_complex<T, 64>(theta, atoms, coeffs, n_atoms, M, rx, n, p, out, s);
  return KAPSM_ERR_UNSUPPORTED;
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void demap_kernel(const T* __restrict__ est, long long n, const T* __restrict__ points,
                             int n_points, unsigned char* __restrict__ labels) {
  __shared__ T pts[128];
  for (int i = threadIdx.x; i < 2 * n_points; i += blockDim.x) pts[i] = points[i];
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const T er = est[2 * i], ei = est[2 * i + 1];
    int best = 0;
    T bd = T(0);
    for (int q = 0; q < n_points; ++q) {
      const T dr = er - pts[2 * q], di = ei - pts[2 * q + 1];
      const T d = dr * dr + di * di;
      if (q == 0 || d < bd) { bd = d; best = q; }
    }
    labels[i] = (unsigned char)best;
  }
}

template <typename T>
int demap(const T* est, long long n, const T* points, int n_points, unsigned char* labels,
          cudaStream_t s) {
  if (n < 0 || n_points < 1 || n_points > 64 || !points || (n && (!est || !labels)))
    return KAPSM_ERR_INVALID;
  if (n == 0) return KAPSM_OK;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  demap_kernel<T><<<(int)blocks, 256, 0, s>>>(est, n, points, n_points, labels);
  return status_from(cudaGetLastError());
}

template <typename E>
__global__ void mismatch_kernel(const E* __restrict__ a, const E* __restrict__ b, long long n,
                                unsigned long long* __restrict__ count) {
  unsigned long long c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    c += (a[i] != b[i]);
  c = warp_sum_u64(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

}  // namespace kapsm

using namespace kapsm;

extern "C" int kapsm_detect_frames_f32(const float* rx, long long rx_stride, int F, int K,
                                       int n_train, int n_data, int M, const float* coeff,
                                       const float* theta, kapsm_kernel_params p,
                                       const float* points, int n_points, int bps,
                                       const unsigned char* tx, float* est,
                                       unsigned char* labels, unsigned long long* be,
                                       unsigned long long* se, void* stream) {
  return detect_frames<float>(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p, points,
                              n_points, bps, tx, est, labels, be, se, (cudaStream_t)stream);
}
extern "C" int kapsm_detect_frames_f64(const double* rx, long long rx_stride, int F, int K,
                                       int n_train, int n_data, int M, const double* coeff,
                                       const double* theta, kapsm_kernel_params p,
                                       const double* points, int n_points, int bps,
                                       const unsigned char* tx, double* est,
                                       unsigned char* labels, unsigned long long* be,
                                       unsigned long long* se, void* stream) {
  return detect_frames<double>(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p, points,
                               n_points, bps, tx, est, labels, be, se, (cudaStream_t)stream);
}
extern "C" int kapsm_batch_evaluate_f32(const float* theta, const float* atoms,
                                        const float* coeffs, int n_atoms, int dim,
                                        const float* inputs, int n_inputs, kapsm_kernel_params p,
                                        float* out, void* stream) {
  return batch_evaluate<float>(theta, atoms, coeffs, n_atoms, dim, inputs, n_inputs, p, out,
                               (cudaStream_t)stream);
}
extern "C" int kapsm_batch_evaluate_f64(const double* theta, const double* atoms,
                                        const double* coeffs, int n_atoms, int dim,
                                        const double* inputs, int n_inputs,
                                        kapsm_kernel_params p, double* out, void* stream) {
  return batch_evaluate<double>(theta, atoms, coeffs, n_atoms, dim, inputs, n_inputs, p, out,
                                (cudaStream_t)stream);
}
extern "C" int kapsm_demap_f32(const float* est, long long n, const float* points, int n_points,
                               unsigned char* labels, void* stream) {
  return demap<float>(est, n, points, n_points, labels, (cudaStream_t)stream);
}
extern "C" int kapsm_demap_f64(const double* est, long long n, const double* points,
                               int n_points, unsigned char* labels, void* stream) {
  return demap<double>(est, n, points, n_points, labels, (cudaStream_t)stream);
}
// Pilot targets from their constellation labels (the receiver knows the
// pilot sequence; a host that ships labels moves 1 byte per pilot and user
// instead of a complex value): targets[2i], targets[2i+1] = points[2 labels[i]],
// points[2 labels[i] + 1], the realified targets of apsm.py:156-169.
// (a label outside the constellation gives NaN targets)
template <typename T>
__global__ void targets_from_labels_kernel(const unsigned char* __restrict__ labels, long long n,
                                           const T* __restrict__ points, int n_points,
                                           T* __restrict__ targets) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int l = labels[i];
  const bool ok = l < n_points;
  targets[2 * i] = ok ? points[2 * l] : T(NAN);
  targets[2 * i + 1] = ok ? points[2 * l + 1] : T(NAN);
}
template <typename T>
static int targets_from_labels(const unsigned char* labels, long long n, const T* points,
                               int n_points, T* targets, void* stream) {
  if (n < 0 || n_points < 1 || n_points > 64 || (n && (!labels || !points || !targets)))
    return KAPSM_ERR_INVALID;
  if (n == 0) return KAPSM_OK;
  targets_from_labels_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      labels, n, points, n_points, targets);
  return status_from(cudaGetLastError());
}
extern "C" int kapsm_targets_from_labels_f32(const unsigned char* labels, long long n,
                                             const float* points, int n_points, float* targets,
                                             void* stream) {
  return targets_from_labels<float>(labels, n, points, n_points, targets, stream);
}
extern "C" int kapsm_targets_from_labels_f64(const unsigned char* labels, long long n,
                                             const double* points, int n_points, double* targets,
                                             void* stream) {
  return targets_from_labels<double>(labels, n, points, n_points, targets, stream);
}

extern "C" int kapsm_count_mismatch(const void* a, const void* b, long long n, int elem_bytes,
                                    unsigned long long* count, void* stream) {
  if (n < 0 || !count || (n && (!a || !b))) return KAPSM_ERR_INVALID;
  if (n == 0) return KAPSM_OK;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaStream_t s = (cudaStream_t)stream;
  switch (elem_bytes) {
    case 1: mismatch_kernel<unsigned char><<<(int)blocks, 256, 0, s>>>((const unsigned char*)a, (const unsigned char*)b, n, count); break;
    case 4: mismatch_kernel<unsigned int><<<(int)blocks, 256, 0, s>>>((const unsigned int*)a, (const unsigned int*)b, n, count); break;
    case 8: mismatch_kernel<unsigned long long><<<(int)blocks, 256, 0, s>>>((const unsigned long long*)a, (const unsigned long long*)b, n, count); break;
    default: return KAPSM_ERR_INVALID;
  }
  return status_from(cudaGetLastError());
}
extern "C" int kapsm_batch_detect_f32(const float* theta, const float* atoms, const float* coeffs,
                                      int n_atoms, int dim, const float* rx, int n,
                                      kapsm_kernel_params p, float* out, void* stream) {
  return batch_detect<float>(theta, atoms, coeffs, n_atoms, dim, rx, n, p, out,
                             (cudaStream_t)stream);
}
extern "C" int kapsm_batch_detect_f64(const double* theta, const double* atoms,
                                      const double* coeffs, int n_atoms, int dim,
                                      const double* rx, int n, kapsm_kernel_params p, double* out,
                                      void* stream) {
  return batch_detect<double>(theta, atoms, coeffs, n_atoms, dim, rx, n, p, out,
                              (cudaStream_t)stream);
}

extern "C" const char* kapsm_strerror(int code) {
  switch (code) {
    case KAPSM_OK: return "ok";
    case KAPSM_ERR_INVALID: return "invalid argument";
    case KAPSM_ERR_CUDA: return "CUDA error";
    case KAPSM_ERR_UNSUPPORTED: return "configuration not supported by this build";
    default: return "unknown kapsm status";
  }
}
extern "C" int kapsm_abi_version(void) { return 100; }

// ---------------------------------------------------------------------------
// Internal instrumentation: FP32 FFMA throughput probe (the SIMT roofline
// denominator; MEASURED_PEAKS.json has only HBM and bf16 tensor peaks).
// Each thread runs 8 independent FFMA chains, 64 FFMA per iteration.
__global__ void __launch_bounds__(256) fp32_peak_kernel(float* out, int iters) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0f + 1e-6f * (threadIdx.x + k);
  // register operands (3-register FFMA form, as in the real kernels)
  const float b = 0.999999f - 1e-9f * threadIdx.x, c = 1e-7f * (1 + (threadIdx.x & 3));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[blockIdx.x] = s;   // keep the work alive
}
extern "C" int kapsm_internal_fp32_peak(float* out, int iters, int blocks, void* stream) {
  if (!out || iters < 1 || blocks < 1) return KAPSM_ERR_INVALID;
  fp32_peak_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, iters);
  return status_from(cudaGetLastError());
}
