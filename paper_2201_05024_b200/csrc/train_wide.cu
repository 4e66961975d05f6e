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

// KAPSM_WIDE_EXP (timing experiments only, 0 in every product build): bits
// 1 = the chain does not wait for init, 2 = no window update, 4 = no band copies
#ifndef KAPSM_WIDE_EXP
#define KAPSM_WIDE_EXP 0
#endif

namespace kapsm {

constexpr int TW_P = 8;                  // takeover lookahead (steps)
constexpr int TW_E = 4;                  // helpers' slack on final coefficients
constexpr int TW_Q = 2;                  // band prefetch distance (steps)
constexpr int TW_R = 16;                 // snapshot ring (>= P + 2, pow2)
constexpr int TW_HW = 12;                // helper warps
constexpr int TW_TR = 16;                // theta ring (>= P + E + 2)
constexpr int TW_LCAP = KAPSM_LIVE_CAP;  // live early Gaussian terms kept per row
constexpr int TW_MAX_DIM = 128;          // realified dimension (theta in registers)
constexpr int TW_MAX_LATE = 160;         // late-part terms W + E (registers)
constexpr int TW_MAX_THREADS = 640;
constexpr long long TW_SPIN = 1LL << 26;
static_assert(TW_R >= TW_P + 2 && (TW_R & (TW_R - 1)) == 0, "snapshot ring");
static_assert(TW_TR >= TW_P + TW_E + 2, "theta ring too short");

__host__ __device__ constexpr int tw_slots(int W) { return W + TW_P + TW_E + TW_Q + 1; }
// one thread past the ring (no memory traffic of its own) publishes progress
__host__ __device__ constexpr int tw_chain_threads(int W) { return (tw_slots(W) + 32) / 32 * 32; }

template <typename T>
struct WideSmem {
  size_t kb, snap, dv, cfin, thr, initr, qsm, ctl, total;
  __host__ __device__ WideSmem(int W, int Np, int dim) {
    using Slot = typename Tagged<T>::slot_t;
    const size_t S = tw_slots(W);
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 15) & ~size_t(15); return r; };
    kb = take(S * S * sizeof(T));
    snap = take((size_t)TW_R * S * sizeof(T));
    dv = take(2 * S * sizeof(T));
    cfin = take((size_t)Np * sizeof(T));
    thr = take((size_t)TW_TR * dim * sizeof(T));
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
                           int* __restrict__ nact_out, int* __restrict__ status_out,
                           const int* __restrict__ live_cnt, const int* __restrict__ live_idx,
                           const T* __restrict__ live_val) {
  using Slot = typename Tagged<T>::slot_t;
  constexpr int P = TW_P, E = TW_E, Q = TW_Q, R = TW_R;
  extern __shared__ __align__(128) unsigned char smem[];
  const WideSmem<T> L(W, Np, dim);
  const int S = tw_slots(W), NC = tw_chain_threads(W);
  T* Kb = reinterpret_cast<T*>(smem + L.kb);         // [S][S] Gram band, ring-indexed
  T* snap = reinterpret_cast<T*>(smem + L.snap);     // [R][S] window coefficients per step
  T* dv = reinterpret_cast<T*>(smem + L.dv);         // [2][S] the step's deltas
  T* cfin = reinterpret_cast<T*>(smem + L.cfin);     // [Np] final coefficients
  T* thr = reinterpret_cast<T*>(smem + L.thr);       // [TR][dim] running linear part
  Slot* initr = reinterpret_cast<Slot*>(smem + L.initr);   // [S] tagged init_m
  T* qsm = reinterpret_cast<T*>(smem + L.qsm);       // [W+1][2] (q_mid, q_last)
  int* ctl = reinterpret_cast<int*>(smem + L.ctl);   // [0] steps done [1] abort [2] status
                                                     // [3] nact [4] theta_l done
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
      // 32-bit shared addresses from one opaque base; ring positions advance
      // incrementally (no divisions in the loop)
      constexpr unsigned TS = sizeof(T), SS = sizeof(Slot);
      const unsigned sb = opaque_u32(smem_u32(smem));
      const unsigned kb_s = sb + (unsigned)L.kb, snap_s = sb + (unsigned)L.snap;
      const unsigned dv_s = sb + (unsigned)L.dv, cfin_s = sb + (unsigned)L.cfin;
      const unsigned qsm_s = sb + (unsigned)L.qsm;
      const unsigned init_a = sb + (unsigned)L.initr + (unsigned)i * SS;
      const unsigned kcol = kb_s + (unsigned)i * TS;                 // Kb[.][i]
      const unsigned krow = kb_s + (unsigned)(i * S) * TS;           // Kb[i][.]
      const unsigned rowstep = (unsigned)S * TS;
      const T qmW = lds_t<T>(qsm_s + (unsigned)(2 * (W - 1)) * TS);
      const T qlW = lds_t<T>(qsm_s + (unsigned)(2 * (W - 1) + 1) * TS);
      int mq = (P + Q) % S;                       // ring position of sample n+P+Q
      int dq = ((P + Q - i) % S + S) % S;         // (n+P+Q - i) mod S
      int jlo = 0;                                // ring position of lo_n
      int tk = (P + 1) % S;                       // ring position of sample n+P+1
      long long ck0 = 0;
      auto ck = [&](int n, int p) {             // KAPSM_WIDE_EXP & 8: step phase clocks
        if ((KAPSM_WIDE_EXP & 8) && fu == 0 && i == 0 && n >= 1000 && n < 1064) {
          const long long c = clock64();
          if (p == 0) ck0 = c;
          else fs_out[100 + 4 * (n - 1000) + p - 1] = (int)(c - ck0);
        }
      };
      for (int n = 0; n < Np && !abort; ++n) {
        ck(n, 0);
        // band row of sample m = n+P+Q (used from step n+Q on)
        cp_async_wait<Q - 1>();
        {
          const int m = n + P + Q;
          const int l = m - dq;                   // this position's sample in (m-S, m]
          if (pos && m < Np && l >= 0 && l > m - W - P && !(KAPSM_WIDE_EXP & 4)) {   // pairs a window update meets
            const T* src = G + (long long)m * ld + l;
            cp_async_s(kcol + (unsigned)mq * rowstep, src);
            cp_async_s(krow + (unsigned)mq * TS, src);
          }
          cp_async_commit();
        }
        const int lo = n - W + 1 > 0 ? n - W + 1 : 0;
        bool stalled = false;
        if (valid && s == n + 1) {                // one step ahead: 1/kappa(r_s, r_s) off the entry step
          const T den = lds_t<T>(krow + (unsigned)i * TS);   // band row of s landed at step s-P
          if (!(den > T(0))) degen = 1;
          invden = den > T(0) ? T(1) / den : T(0);
        }
        if (valid && s == n) {                    // entering: init_m from the helpers
          T iv = T(0);
          long long spins = 0;
          while (!(KAPSM_WIDE_EXP & 1) && !ld_tag(init_a, s, iv))
            if (++spins > TW_SPIN || ((spins & 1023) == 0 && ld_volatile(&ctl[1]))) {
              stalled = true;
              break;
            }
          if (s == 0) {                           // (no step before sample 0)
            const T den = lds_t<T>(krow + (unsigned)i * TS);
            if (!(den > T(0))) degen = 1;
            invden = den > T(0) ? T(1) / den : T(0);
          }
          bm = bv - eps - iv;
          bp = bv + eps - iv;
        }
        T delta = T(0);
        if (valid && s >= lo && s <= n) {
          const int J = n - lo + 1;
          // full windows (J = W) after warm-up: the two weights live in registers
          const T q = J == W ? (s == n ? qlW : qmW)
                             : lds_t<T>(qsm_s + (unsigned)(2 * (J - 1) + (s == n)) * TS);
          const T qi = q * invden;
          const T v1 = fma(-qi, Y, qi * bm), v2 = fma(-qi, Y, qi * bp);
          delta = fmax(v1, T(0)) + fmin(v2, T(0));
          c += delta;
          if (delta != T(0) && fs > n) fs = n;
          sts(snap_s + (unsigned)((n & (R - 1)) * S + i) * TS, c);
          if (n == s + W - 1 || n == Np - 1) {    // leaves the window: final
            sts(cfin_s + (unsigned)s * TS, c);
            fs_out[(long long)fu * Np + s] = fs == 0x7fffffff ? -1 : fs;
            nact += fs != 0x7fffffff;
          }
        }
        const unsigned d_s = dv_s + (unsigned)((n & 1) * S) * TS;
        if (pos) sts(d_s + (unsigned)i * TS, delta);
        ck(n, 1);
        abort = named_bar_or(1, NC, stalled);
        ck(n, 2);
        if (i == NC - 1) {                        // idle position: its fence waits on nothing
          if (!(KAPSM_WIDE_EXP & 32)) __threadfence_block();
          st_volatile(&ctl[0], n + 1);
        }
        // window update of every owned sample that is (or will be) in a window
        if (valid && s >= lo && !(KAPSM_WIDE_EXP & 2)) {
          // plain shared loads (schedulable; the barrier's clobber orders them)
          const T* dpp = dv + (n & 1) * S;
          T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
          int j = jlo;
          int cnt = n - lo + 1;
          while (cnt > 0) {
            const int run = cnt < S - j ? cnt : S - j;    // up to the ring's end
            const T* kp = Kb + j * S + i;
            const T* dp = dpp + j;
            int k = 0;
#pragma unroll 2
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
        ck(n, 3);
        // takeover after step n: sample n+P+1 at ring position tk
        if (pos && i == tk) {
          s = n + P + 1;
          valid = s < Np;
          Y = T(0);
          c = T(0);
          fs = 0x7fffffff;
          bv = valid ? B[s] : T(0);
        }
        mq = mq + 1 == S ? 0 : mq + 1;
        dq = dq + 1 == S ? 0 : dq + 1;
        tk = tk + 1 == S ? 0 : tk + 1;
        if (n >= W - 1) jlo = jlo + 1 == S ? 0 : jlo + 1;
        ck(n, 4);
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
      // warp 0 of the helpers: the running linear part theta_l = sum_{i<=l}
      // c_i r_i (ring of TR); the others: init_m, one sample per warp.
      const int h = warp - NC / 32, nh = (nthreads - NC) / 32;
      const T* X = rx ? rx + (long long)f * rx_stride : nullptr;
      const T* Sm = rx ? nullptr : samples + (long long)f * samples_stride;
      const int M = dim / 2;
      auto rcomp = [&](int m, int k) -> T {     // component k of realified sample m
        if (!X) return Sm[(long long)m * dim + k];
        const int kk = k < M ? k : k - M;
        const T re = X[(long long)(m >> 1) * 2 * M + 2 * kk];
        const T im = X[(long long)(m >> 1) * 2 * M + 2 * kk + 1];
        return (m & 1) ? (k < M ? im : -re) : (k < M ? re : im);
      };
      auto wait_ge = [&](const int* ctr, int x) -> bool {   // until *ctr >= x; false on abort
        long long spins = 0;
        while (ld_volatile(ctr) < x) {          // back off: the chain warps share the SM
          __nanosleep(32);
          if (++spins > TW_SPIN / 16 || ((spins & 255) == 0 && ld_volatile(&ctl[1]))) return false;
        }
        __threadfence_block();
        return true;
      };
      constexpr int DK = TW_MAX_DIM / 32;
      bool ok = !(KAPSM_WIDE_EXP & 16);
      if (!ok) {
      } else if (h == 0) {
        T th[DK], rn[DK];
#pragma unroll
        for (int q = 0; q < DK; ++q) {
          th[q] = T(0);
          rn[q] = (lane + 32 * q < dim && Np > 0) ? rcomp(0, lane + 32 * q) : T(0);
        }
        for (int l = 0; l < Np && ok; ++l) {
          T rc[DK];
#pragma unroll
          for (int q = 0; q < DK; ++q) {         // prefetch the next sample
            rc[q] = rn[q];
            rn[q] = (lane + 32 * q < dim && l + 1 < Np) ? rcomp(l + 1, lane + 32 * q) : T(0);
          }
          ok = wait_ge(&ctl[0], l + W < Np ? l + W : Np);     // c_l final
          if (!ok) break;
          const T cl = cfin[l];
          T* tr = thr + (l % TW_TR) * dim;
#pragma unroll
          for (int q = 0; q < DK; ++q)
            if (lane + 32 * q < dim) {
              th[q] = fma(cl, rc[q], th[q]);
              tr[lane + 32 * q] = th[q];
            }
          __syncwarp();
          if (lane == 0) {
            __threadfence_block();
            st_volatile(&ctl[4], l + 1);
          }
        }
      } else {
        const int* lcnt = live_cnt + (long long)f * Np;
        const int* lidx = live_idx + (long long)f * Np * TW_LCAP;
        const T* lval = live_val + (long long)f * Np * TW_LCAP;
        constexpr int LK = (TW_MAX_LATE + 31) / 32;
        for (int m = h - 1; m < Np && ok; m += nh - 1) {
          const int t = m - P - 1;              // coefficients as of the end of step t
          const T* row = G + (long long)m * ld;
          const int le = t - W - E;             // early part: l <= le, final since step t-E-1
          const int l0 = le + 1 > 0 ? le + 1 : 0;
          // the late part's Gram entries do not depend on the chain: load them first
          T kr[LK];
#pragma unroll
          for (int q = 0; q < LK; ++q) {
            const int l = l0 + lane + 32 * q;
            kr[q] = l <= t ? row[l] : T(0);
          }
          T acc = T(0);
          if (t >= 0) {
            if (le >= 0) {
              const int nl = lcnt[m];
              if (nl <= TW_LCAP) {
                // w_l theta_le . r_m + the live Gaussian terms (K1's list)
                T rm[DK];
#pragma unroll
                for (int q = 0; q < DK; ++q)
                  rm[q] = lane + 32 * q < dim ? rcomp(m, lane + 32 * q) : T(0);
                const int li = lane < nl ? lidx[(long long)m * TW_LCAP + lane] : 0;
                const T lv = lane < nl ? lval[(long long)m * TW_LCAP + lane] : T(0);
                ok = wait_ge(&ctl[4], le + 1);
                if (!ok) break;
                const T* tr = thr + (le % TW_TR) * dim;
                T lin = T(0);
#pragma unroll
                for (int q = 0; q < DK; ++q)
                  if (lane + 32 * q < dim) lin = fma(tr[lane + 32 * q], rm[q], lin);
                acc = w_l * lin;
                if (lane < nl && li <= le) acc = fma(cfin[li], lv, acc);
              } else {                            // list overflow: dense row
                ok = wait_ge(&ctl[0], t - E);
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
            }
            ok = wait_ge(&ctl[0], t + 1);
            if (!ok) break;
            const T* sn = snap + (t & (R - 1)) * S;
#pragma unroll
            for (int q = 0; q < LK; ++q) {
              const int l = l0 + lane + 32 * q;
              if (l <= t) acc = fma(l <= t - W ? cfin[l] : sn[l % S], kr[q], acc);
            }
          }
          acc = warp_sum(acc);
          if (lane == 0) Tagged<T>::store(&initr[m % S], acc + (P0 ? P0[m] : T(0)), m);
        }
      }
      if (!ok && lane == 0 && !(KAPSM_WIDE_EXP & 16)) {
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
          // unrolled: 8 pilots' strided loads in flight per lane (same sum order)
#pragma unroll 8
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
#pragma unroll 8
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

// Live early Gaussian terms of every pilot row: for row m the columns
// l <= m - gap (gap = P + 1 + W + E, the helpers' early region) whose term
// w_g exp(-||r_l - r_m||^2 / 2 sigma^2) does not underflow, in increasing l
// (deterministic order), with the value.  More than TW_LCAP: the count is
// kept and the helper falls back to the dense Gram row.  One CTA per 32 rows,
// column tiles of 32 samples staged in shared memory.
template <typename T>
__global__ void __launch_bounds__(256)
    live_lists_kernel(const T* __restrict__ rx, long long rx_stride,
                      const T* __restrict__ samples, long long samples_stride, int dim, int Np,
                      int gap, T w_g, T inv2s, int* __restrict__ cnt, int* __restrict__ idx,
                      T* __restrict__ val) {
  extern __shared__ __align__(16) unsigned char lsm[];
  const int Dp = dim + 1;
  T* Rm = reinterpret_cast<T*>(lsm);            // [32][Dp] this block's rows
  T* Rl = Rm + 32 * Dp;                         // [32][Dp] column tile
  const int f = blockIdx.y, m0 = blockIdx.x * 32;
  cnt += (long long)f * Np;                     // this frame's rows
  idx += (long long)f * Np * TW_LCAP;
  val += (long long)f * Np * TW_LCAP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T* X = rx ? rx + (long long)f * rx_stride : nullptr;
  const T* Sm = rx ? nullptr : samples + (long long)f * samples_stride;
  const int M = dim / 2;
  auto rcomp = [&](int m, int k) -> T {
    if (!X) return Sm[(long long)m * dim + k];
    const int kk = k < M ? k : k - M;
    const T re = X[(long long)(m >> 1) * 2 * M + 2 * kk];
    const T im = X[(long long)(m >> 1) * 2 * M + 2 * kk + 1];
    return (m & 1) ? (k < M ? im : -re) : (k < M ? re : im);
  };
  for (int e = threadIdx.x; e < 32 * dim; e += blockDim.x) {
    const int r = e / dim, k = e % dim;
    Rm[r * Dp + k] = m0 + r < Np ? rcomp(m0 + r, k) : T(0);
  }
  int c[4] = {0, 0, 0, 0};
  const int lmax = m0 + 31 - gap;
  for (int l0 = 0; l0 <= lmax && w_g != T(0); l0 += 32) {
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * dim; e += blockDim.x) {
      const int r = e / dim, k = e % dim;
      Rl[r * Dp + k] = l0 + r < Np ? rcomp(l0 + r, k) : T(0);
    }
    __syncthreads();
    const int l = l0 + lane;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int mr = warp * 4 + r, m = m0 + mr;
      const bool cand = m < Np && l <= m - gap;
      T g = T(0);
      if (cand) {
        T d2 = T(0);
        for (int k = 0; k < dim; ++k) {
          const T e = Rm[mr * Dp + k] - Rl[lane * Dp + k];
          d2 = fma(e, e, d2);
        }
        g = w_g * exp_acc(-d2 * inv2s);
      }
      const bool live = cand && g != T(0);
      const unsigned mask = __ballot_sync(0xffffffffu, live);
      const int pos = c[r] + __popc(mask & ((1u << lane) - 1u));
      if (live && pos < TW_LCAP) {
        idx[(long long)m * TW_LCAP + pos] = l;
        val[(long long)m * TW_LCAP + pos] = g;
      }
      c[r] += __popc(mask);
    }
  }
  if (lane == 0)
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (m0 + warp * 4 + r < Np) cnt[m0 + warp * 4 + r] = c[r];
}

// Live lists of every pilot row (l <= m - gap) in stream-ordered scratch
// memory (cudaMallocAsync; free with cudaFreeAsync(ll.ws) on the same stream).
template <typename T>
int build_live_lists(const T* rx, long long rx_stride, const T* samples, long long samples_stride,
                     int dim, int F, int Np, int gap, kapsm_kernel_params p, cudaStream_t s,
                     LiveLists<T>& ll) {
  const size_t rows = (size_t)F * Np;
  const size_t b_cnt = (rows * sizeof(int) + 255) & ~size_t(255);
  const size_t b_idx = (rows * TW_LCAP * sizeof(int) + 255) & ~size_t(255);
  const size_t b_val = rows * TW_LCAP * sizeof(T);
  ll.ws = nullptr;
  if (cudaMallocAsync(&ll.ws, b_cnt + b_idx + b_val, s) != cudaSuccess) return KAPSM_ERR_CUDA;
  ll.cnt = static_cast<int*>(ll.ws);
  ll.idx = reinterpret_cast<int*>(static_cast<char*>(ll.ws) + b_cnt);
  ll.val = reinterpret_cast<T*>(static_cast<char*>(ll.ws) + b_cnt + b_idx);
  const size_t lsm = 2 * 32 * (size_t)(dim + 1) * sizeof(T);
  if (cudaFuncSetAttribute(live_lists_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)lsm) != cudaSuccess)
    return KAPSM_ERR_CUDA;
  live_lists_kernel<T><<<dim3((Np + 31) / 32, F), 256, lsm, s>>>(
      rx, rx_stride, samples, samples_stride, dim, Np, gap, (T)p.w_g,
      (T)(1.0 / (2.0 * p.sigma_sq)), ll.cnt, ll.idx, ll.val);
  return status_from(cudaGetLastError());
}
template int build_live_lists<float>(const float*, long long, const float*, long long, int, int,
                                     int, int, kapsm_kernel_params, cudaStream_t,
                                     LiveLists<float>&);
template int build_live_lists<double>(const double*, long long, const double*, long long, int,
                                      int, int, int, kapsm_kernel_params, cudaStream_t,
                                      LiveLists<double>&);

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
  if (dim > TW_MAX_DIM || W + TW_E > TW_MAX_LATE) return KAPSM_ERR_UNSUPPORTED;
  const WideSmem<T> L(W, Np, dim);
  if (L.total > 227 * 1024) return KAPSM_ERR_UNSUPPORTED;
  auto kern = apsm_train_wide_kernel<T>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  // live-term lists (stream-ordered scratch: F x Np rows)
  LiveLists<T> ll;
  int r = build_live_lists<T>(rx, rx_stride, samples, samples_stride, dim, F, Np,
                              TW_P + 1 + W + TW_E, p, s, ll);
  int* lcnt = ll.cnt;
  int* lidx = ll.idx;
  T* lval = ll.val;
  void* ws = ll.ws;
  if (r == KAPSM_OK) {
    const int tasks = F * K;
    const int grid = tasks < wide_num_sms() ? tasks : wide_num_sms();
    kern<<<grid, NC + 32 * TW_HW, L.total, s>>>(gram, ld, gram_stride, rx, rx_stride, samples,
                                                samples_stride, dim, targets, F, K, Np, W,
                                                (T)eps, (T)p.w_l, qtab, base0, theta0, coeff,
                                                first_step, theta, n_active, status, lcnt, lidx,
                                                lval);
    r = status_from(cudaGetLastError());
  }
  if (cudaFreeAsync(ws, s) != cudaSuccess && r == KAPSM_OK) r = KAPSM_ERR_CUDA;
  return r;
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
  while (tw_chain_threads(W + 1) + 32 * TW_HW <= TW_MAX_THREADS && W + 1 + TW_E <= TW_MAX_LATE &&
         WideSmem<double>(W + 1, 2048, TW_MAX_DIM).total <= 227 * 1024)
    ++W;
  return W;
}

}  // namespace kapsm
