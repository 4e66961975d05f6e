// K2: persistent APSM trainer.  One chain group trains one (frame, user) at a
// time: a CRITICAL warp runs the strictly sequential pilot loop, BACKGROUND
// warps compute everything that does not depend on the current step.
//
// Reference semantics: ApsmTrainer.observe (apsm.py:304-359) driven by
// train()/observe_symbol (apsm.py:361-396).  At step n (realified sample n),
// with window J_n = [lo_n, n], lo_n = max(0, n-W+1) (apsm.py:132-136):
//   y_j   = f_n(r_j)                                 j in J_n   (apsm.py:288-302)
//   beta_j three-case on res_j = y_j - b_j, den_j = kappa(r_j,r_j)  (apsm.py:323-332)
//   c_j  += q_j beta_j, q = uniform_weights(|J_n|)   (apsm.py:336-359)
// where f_n = f0 + sum_i c_i kappa(r_i, .).  The represented function is the
// reference's (collapsed theta + one atom per activated sample); theta is
// formed at the end as theta0 + w_l sum_i c_i r_i (the reference accumulates it
// per step, apsm.py:338 -- same value up to summation order).
//
// Restatement (pilot sum-kernel Gram K from K1; exact rearrangements):
//   * slot x (= lane x of the critical warp) owns sample m = x (mod 32) from
//     step m-L-1 (L = TC_L, the lookahead) until m leaves the window;
//   * every owned sample accumulates the step's window update
//         Y_m += sum_{l in J_n} delta_l K[l][m]            (one dot per lane)
//     from its first owned step on, so that when it enters the window
//         f(r_m) = init_m + Y_m,
//         init_m = f0(r_m) + sum_{i<m} c_i^(n_m) K[i][m],  n_m = m-L-1,
//     the coefficients c^(n_m) being those at the start of step n_m;
//   * init_m is computed by the BACKGROUND warps: final coefficients
//     (i <= m-32, published as tagged words when the sample leaves the window)
//     dotted with the TMA-staged Gram row m, plus the 31 slot coefficients
//     from a tagged per-step snapshot.  It is needed L+1 steps later;
//   * the critical warp's step is therefore one chain
//         Y -> delta = max(q/den (b-eps-f), 0) + min(q/den (b+eps-f), 0)
//           -> smem broadcast -> window dot (registers x broadcast) -> Y
//     with the slot rotation unrolled 32-wide so that every register index is
//     static; the entering slot's Gram column arrives by cp.async TC_DELTA
//     steps ahead.
// Scheduling: one CTA per SM.  Latency mode (NG = 1): the critical warp is the
// only warp on its SM sub-partition, six background warps on the other three.
// Throughput mode (NG = 4): group g lives on sub-partition g, its critical
// warp has the highest warp id there (the issue arbiter favours it).
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include "kapsm_common.cuh"

// KAPSM_FEAT (experiments only): bits that compile parts of the critical warp
// out of the instrumentation kernel, to time them; 0 in every product build.
#ifndef KAPSM_FEAT
#define KAPSM_FEAT 0
#endif

namespace kapsm {

constexpr int TC_S = 32;                    // slots (one warp)
constexpr int TC_BT = 4;                    // batch: takeover / entry / publication every 4 steps
constexpr int TC_MAX_W = 23;                // lookahead D = 8 with D + W <= 31
constexpr int TC_PF = 2;                    // column prefetch distance (batches)
constexpr int TC_SRING = 4;                 // staged column batches (ring, pow2 > PF)
constexpr int TC_INIT = 64;                 // init values (ring, pow2)
constexpr int TC_ERING = 128;               // early init parts in flight (tagged ring, pow2)
constexpr int TC_Q = 61;                    // init: early part i <= m - Q, late part <= 32 elements
constexpr int TC_MAX_NP = 16384;            // (and the shared-memory footprint)
// slot reuse: the batch taken over after step n+1 (samples n+D..n+D+3)
// reuses the slots of samples that left the window by step n+1:
// D + 3 + W - 33 <= 1.
__host__ __device__ constexpr int lookahead(int wm) {
  return ((31 - wm) & ~3) > 8 ? 8 : ((31 - wm) & ~3);
}
constexpr long long TC_SPIN_LIMIT = 1LL << 20;

template <int K> using ic = std::integral_constant<int, K>;

// ---- window dot: Yz + sum over the window lanes of delta_l * row[l] ----
// Lanes of the window at step k (mod 32): (k - j) & 31, j = 0..WM-1.  Lanes
// outside the true window hold delta = 0, so whole 4-lane blocks are used.
template <int k, int WM>
struct WinBlocks {
  static constexpr bool in(int l) { return ((k - l) & 31) < WM; }
  static constexpr bool blk(int b) { return in(4 * b) || in(4 * b + 1) || in(4 * b + 2) || in(4 * b + 3); }
};


// The broadcast deltas are stored rotated: lane x writes position
// (x - k - 1) & 31 at step k, so the window lanes (k - j) & 31, j < WM,
// always occupy positions 32-WM .. 31 (whole 16-byte blocks for WM % 4 == 0),
// and position p belongs to lane (p + k + 1) & 31 (static per unrolled step).
template <typename T> struct WinLoad;
template <> struct WinLoad<float> { using type = float4; };
template <> struct WinLoad<double> { using type = double4; };

template <int WM>
KAPSM_DEV void window_load(unsigned dvb, float4 (&wl)[8]) {
#pragma unroll
  for (int b = (TC_S - WM) / 4; b < 8; ++b) wl[b] = lds_f4(dvb + 16 * b);
}
template <int WM>
KAPSM_DEV void window_load(unsigned dvb, double4 (&wl)[8]) {
#pragma unroll
  for (int b = (TC_S - WM) / 4; b < 8; ++b) {
    const double2 u = lds_d2(dvb + 32 * b), v = lds_d2(dvb + 32 * b + 16);
    wl[b] = make_double4(u.x, u.y, v.x, v.y);
  }
}
KAPSM_DEV float w4(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
KAPSM_DEV double w4(const double4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
// yz + sum over the window positions of delta * row[lane(position)]; scalar
// FMAs in 4 accumulators (lower latency than FFMA2 on this chain)
template <int k, int WM, typename T>
KAPSM_DEV T window_fma(const typename WinLoad<T>::type (&wl)[8], const T (&row)[TC_S], T yz) {
  T a[4] = {yz, T(0), T(0), T(0)};
#pragma unroll
  for (int p = TC_S - WM; p < TC_S; ++p)
    a[p & 3] = fma(w4(wl[p >> 2], p & 3), row[(p + k + 1) & (TC_S - 1)], a[p & 3]);
  return (a[0] + a[1]) + (a[2] + a[3]);
}

KAPSM_DEV void load_row32(unsigned p, float (&r)[TC_S]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 v = lds_f4(p + 16 * q);
    r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
  }
}
KAPSM_DEV void load_row32(unsigned p, double (&r)[TC_S]) {
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const double2 v = lds_d2(p + 16 * q);
    r[2 * q] = v.x; r[2 * q + 1] = v.y;
  }
}
KAPSM_DEV void warp_sync_full() { asm volatile("bar.warp.sync 0xffffffff;" ::: "memory"); }
KAPSM_DEV float recip(float v) {   // MUFU.RCP (FP32 path tolerance is 1e-4)
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
KAPSM_DEV double recip(double v) { return 1.0 / v; }


// 16-byte vectors for the background row dots
template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; };
template <> struct Vec16<double> { using type = double2; };
KAPSM_DEV float4 ldg16(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
KAPSM_DEV double2 ldg16(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
template <typename T> KAPSM_DEV typename Vec16<T>::type lds16(unsigned a);
template <> KAPSM_DEV float4 lds16<float>(unsigned a) { return lds_f4(a); }
template <> KAPSM_DEV double2 lds16<double>(unsigned a) { return lds_d2(a); }
KAPSM_DEV float elem16(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
KAPSM_DEV double elem16(const double2& v, int e) { return e == 0 ? v.x : v.y; }

// acc + sum_e c[i0+e] * r.e over EPV tagged coefficient slots at address a
template <typename T>
KAPSM_DEV T tagged_dot16(unsigned a, int i0, const typename Vec16<T>::type& r, T acc, bool& bad);
template <>
KAPSM_DEV float tagged_dot16<float>(unsigned a, int i0, const float4& r, float acc, bool& bad) {
  uint4 p, q;
  asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(p.x), "=r"(p.y), "=r"(p.z), "=r"(p.w) : "r"(a) : "memory");
  asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(a + 16) : "memory");
  bad |= (int)p.y != i0 || (int)p.w != i0 + 1 || (int)q.y != i0 + 2 || (int)q.w != i0 + 3;
  acc = fmaf(__uint_as_float(p.x), r.x, acc);
  acc = fmaf(__uint_as_float(p.z), r.y, acc);
  acc = fmaf(__uint_as_float(q.x), r.z, acc);
  return fmaf(__uint_as_float(q.z), r.w, acc);
}
template <>
KAPSM_DEV double tagged_dot16<double>(unsigned a, int i0, const double2& r, double acc, bool& bad) {
  double v0, v1;
  int t0, t1;
  ld_tagged(a, v0, t0);
  ld_tagged(a + 16, v1, t1);
  bad |= t0 != i0 || t1 != i0 + 1;
  return fma(v1, r.y, fma(v0, r.x, acc));
}


template <typename T>
KAPSM_DEV T slot_value(const typename Tagged<T>::slot_t& w);
template <>
KAPSM_DEV float slot_value<float>(const unsigned long long& w) {
  return __uint_as_float((unsigned)(w & 0xffffffffu));
}
template <>
KAPSM_DEV double slot_value<double>(const Tagged<double>::slot_t& w) {
  return __longlong_as_double((long long)w.v);
}

// Role layout.  CL = cluster size (CTAs per task group).
//   NG = 1, CL = 2 (latency): a 2-CTA cluster per task.  CTA rank 0 runs only
//          the critical warp (warp 7; the other warps wait for the
//          epilogue), CTA rank 1 runs 8 background warps on another SM, so
//          nothing competes with the critical warp for issue slots or the
//          shared-memory pipe.  They exchange snapshots, final coefficients
//          and init values through distributed shared memory.
//   NG = 4, CL = 1 (throughput): group g = w % 4 on sub-partition g, role
//          w / 4 (3 = critical).
template <int NG, int CL> struct Roles;
// Every role: NB = id of the critical role; NA A workers, NBH B helpers.
// Roles: NB = id of the critical role; workers are early (kind 1: the early
// init parts, far ahead of need) or late (kind 2: the short deadline path).
template <> struct Roles<1, 2> {
  static constexpr int NE = 8, NL = 4, NB = NE + NL, ACH = 12, WARPS = 8;  // ACH: row vectors/lane
  static KAPSM_DEV int group(int) { return 0; }
  // rank 0: warp 7 critical; warps 0,1,2,4 late finishers (next to the
  // critical warp: local latency; one per sample of a batch, off its
  // sub-partition), warps 3,5,6 idle until the epilogue; rank 1: early workers
  static KAPSM_DEV int role(int w, unsigned rank) {
    if (rank) return w;
    if (w == 7) return NB;
    if (w < 3) return NE + w;
    return w == 4 ? NE + 3 : -1;
  }
};
template <> struct Roles<4, 1> {
  static constexpr int NE = 2, NL = 1, NB = NE + NL, ACH = 4, WARPS = 16;
  static KAPSM_DEV int group(int w) { return w & 3; }
  static KAPSM_DEV int role(int w, unsigned) { return w >> 2; }   // 0,1 early  2 late  3 critical
};

template <typename T, int NG, int CL>
struct GroupSmem {
  // byte offsets of one group's region in dynamic shared memory
  size_t dv, snap, stage, tst, bsm, initr, ering, ctag, cfin, fsfin, qsm, ctl, total;
  // staged: the batch targets arrive with the staged columns instead of a
  // per-sample array (larger Np fits in shared memory)
  __host__ __device__ GroupSmem(int W, int Np, bool staged = false) {
    using Slot = typename Tagged<T>::slot_t;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 15) & ~size_t(15); return r; };
    dv = take(2 * TC_S * sizeof(T));
    snap = take((size_t)2 * TC_S * sizeof(T));   // slot coefficients after a block's 1st step
    stage = take((size_t)TC_SRING * TC_BT * TC_S * sizeof(T));
    tst = take((size_t)TC_SRING * TC_BT * sizeof(T));   // the staged batches' targets
    bsm = take(staged ? 0 : (size_t)(Np + 2 * TC_S) * sizeof(T));   // all targets (zero padded)
    initr = take((size_t)TC_INIT * sizeof(Slot));
    ering = take((size_t)TC_ERING * sizeof(Slot));
    ctag = take((size_t)(Np + TC_S) * sizeof(Slot));
    cfin = take((size_t)(Np + TC_S) * sizeof(T));
    fsfin = take((size_t)(Np + TC_S) * sizeof(int));
    qsm = take(2 * (size_t)(W + 1) * sizeof(T));
    ctl = take(16 * sizeof(int));
    total = (o + 127) & ~size_t(127);
  }
};

// slow path of the entry check (the background warps are late): out of line,
// so the hot loop carries only a predicated call
template <typename T>
__device__ __noinline__ void init_spin(unsigned a, bool isent, int me, int Np, T* iv, int* ctl,
                                       int* nend) {
  long long spins = 0;
  for (;;) {
    bool ok = true;
    if (isent) ok = ld_tag(a, me, *iv) || me >= Np;
    if (vote_all(ok)) break;
    if (++spins > TC_SPIN_LIMIT || ((spins & 4095) == 0 && ld_volatile(&ctl[1]))) {
      *nend = 0;
      atomicOr(&ctl[2], 4);
      break;
    }
  }
}

template <typename T, int NG, int CL, int WM, bool DBG, bool STG = false>
__global__ void __launch_bounds__(Roles<NG, CL>::WARPS * 32, 1)
    apsm_train_kernel(const T* __restrict__ gram, long long ld, long long gram_stride,
                      const T* __restrict__ rx, long long rx_stride,
                      const T* __restrict__ samples, long long samples_stride, int dim,
                      const T* __restrict__ targets, int F, int K, int Np, int W, T eps,
                      T w_l, const T* __restrict__ qtab, const T* __restrict__ base0,
                      const T* __restrict__ theta0, T* __restrict__ coeff_out,
                      int* __restrict__ fs_out, T* __restrict__ theta_out,
                      int* __restrict__ nact_out, int* __restrict__ status_out,
                      long long* __restrict__ dbg) {
  using Slot = typename Tagged<T>::slot_t;
  using R = Roles<NG, CL>;
  constexpr int NB = R::NB, ACH = sizeof(T) == 8 ? R::ACH / 2 : R::ACH;
  constexpr int D = lookahead(WM);            // takeover lookahead (steps)
  constexpr int FEAT = KAPSM_FEAT;            // experiments only: parts compiled out
  constexpr int FIRST = D;                    // first sample whose init needs coefficients
  constexpr unsigned TS = sizeof(T), SS = sizeof(Slot);
  extern __shared__ __align__(128) unsigned char smem[];
  const GroupSmem<T, NG, CL> L(W, Np, STG);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned rank = CL > 1 ? cluster_rank() : 0u;
  const int grp = R::group(warp);
  const int role = R::role(warp, rank);        // 0..NB-1: background, NB: critical, -1: idle
  // threads sharing this group's shared-memory region (per-task init, epilogue)
  const int gt = NG == 1 ? (int)threadIdx.x : role * 32 + lane;
  constexpr int GT = NG == 1 ? R::WARPS * 32 : (NB + 1) * 32;
  unsigned char* gs = smem + (size_t)grp * L.total;
  // shared::cluster bases of this group's region in the critical CTA and in
  // the background CTA (the same CTA unless CL = 2)
  const unsigned lbase = smem_u32(gs);
  const unsigned cw_base = CL > 1 ? map_rank(lbase, 0) : lbase;
  const unsigned bg_base = CL > 1 ? map_rank(lbase, CL - 1) : lbase;
  Slot* initr = reinterpret_cast<Slot*>(gs + L.initr);   // [INIT] tagged init_m
  Slot* ctag = reinterpret_cast<Slot*>(gs + L.ctag);     // [Np+S] tagged final c_m
  T* cfin = reinterpret_cast<T*>(gs + L.cfin);           // [Np+S] final c_m (stored before ctag)
  int* fsfin = reinterpret_cast<int*>(gs + L.fsfin);     // [Np+S] first-activation step
  T* qsm = reinterpret_cast<T*>(gs + L.qsm);             // [W+1][2] (q_mid, q_last), row W = 0
  int* ctl = reinterpret_cast<int*>(gs + L.ctl);         // [1]=abort [2]=status [3]=nact
  const int group_bar = 1 + grp;
  const int dbgvar = DBG ? (int)dbg[5 * Np] : 0;
  auto group_sync = [&] {
    if constexpr (CL > 1) cluster_sync();
    else named_bar(group_bar, GT);
  };
  // abort: raise the flag in both CTAs
  auto raise_abort = [&](int code) {
    red_or_cl(cw_base + (unsigned)L.ctl + 8u, code);
    st_cl_s32(cw_base + (unsigned)L.ctl + 4u, 1);
    if (CL > 1) st_cl_s32(bg_base + (unsigned)L.ctl + 4u, 1);
  };
  const int ncl = CL > 1 ? (int)gridDim.x / CL : (int)gridDim.x;
  const int cid = CL > 1 ? (int)blockIdx.x / CL : (int)blockIdx.x;

  for (int task = cid * NG + grp; task < F * K; task += ncl * NG) {
    const int fu = task;                        // frame * K + user
    const int f = fu / K;
    const T* G = gram + (long long)f * gram_stride;
    const T* B = targets + (long long)fu * Np;  // realified targets (interleaved pilots)
    const T* P0 = base0 ? base0 + (long long)fu * Np : nullptr;

    // ---------------- per-task group state ----------------
    for (int i = gt; i < TC_INIT; i += GT) Tagged<T>::store(&initr[i], T(0), -1);
    {
      Slot* ering = reinterpret_cast<Slot*>(gs + L.ering);
      for (int i = gt; i < TC_ERING; i += GT) Tagged<T>::store(&ering[i], T(0), -1);
    }
    for (int i = gt; i < Np + TC_S; i += GT) { Tagged<T>::store(&ctag[i], T(0), -1); fsfin[i] = -1; }
    if (!STG) {
      T* bsm = reinterpret_cast<T*>(gs + L.bsm);         // [Np+2S] targets (zero padded)
      for (int i = gt; i < Np + 2 * TC_S; i += GT) bsm[i] = i < Np ? B[i] : T(0);
    }
    for (int i = gt; i <= W; i += GT) {
      T qm = T(1) / T(i + 1), ql = qm;
      if (qtab) { qm = qtab[2 * i]; ql = qtab[2 * i + 1]; }
      if (i == W) { qm = T(0); ql = T(0); }     // steps past the last sample: no update
      qsm[2 * i] = qm;
      qsm[2 * i + 1] = ql;
    }
    if (gt < 16) ctl[gt] = 0;
    group_sync();

    if (role == NB) {
      // =========================== CRITICAL WARP ===========================
      // Slot x owns sample m = x (mod 32).  Samples 0..D-1 are owned from the
      // start; after the first step of block j (steps n = 4j .. 4j+3) the
      // samples that left the window are published, the coefficients are
      // snapshot, and the batch n+D .. n+D+3 is taken over (it accumulates
      // from step n+1).  Every shared access goes through 32-bit addresses
      // from one opaque base.
      const int x = lane;
      const unsigned gbase = opaque_u32(smem_u32(gs));
      const unsigned dv_s = gbase + (unsigned)L.dv, stage_s = gbase + (unsigned)L.stage;
      const unsigned snap_s = gbase + (unsigned)L.snap;
      const unsigned initr_s = gbase + (unsigned)L.initr, ctag_s = gbase + (unsigned)L.ctag;
      const unsigned fsfin_s = gbase + (unsigned)L.fsfin, tst_s = gbase + (unsigned)L.tst;
      const unsigned bsm_s = gbase + (unsigned)L.bsm;
      const unsigned qsm_s = gbase + (unsigned)L.qsm, cfin_s = gbase + (unsigned)L.cfin;
      // the background CTA's copies (shared::cluster addresses)
      // the A workers' copy of the final coefficients (shared::cluster address)
      const unsigned bctag_s = opaque_u32(bg_base + (unsigned)L.ctag);
      const int Wm1 = W - 1;
      constexpr int NOWN = D;                   // samples owned from the start

      int m = x < NOWN ? x : x - TC_S;          // owned sample
      bool valid = m >= 0 && m < Np;
      T row[TC_S];                               // row[l] = K[sample(l)][m]
#pragma unroll
      for (int l = 0; l < TC_S; ++l)
        row[l] = (valid && l < NOWN && l < Np) ? G[(long long)l * ld + m] : T(0);
      const T den0 = valid ? G[(long long)m * ld + m] : T(1);
      int degen = valid && !(den0 > T(0));
      T invden = valid ? T(1) / den0 : T(0);
      const T b0 = valid ? B[m] : T(0);
      T bme = b0 - eps, bpe = b0 + eps;        // b -/+ eps of the owned sample
      T bm = T(0), bp = T(0);                    // ... minus init_m, once entered
      T Y = T(0), c = T(0);
      int fs = 0x7fffffff;                       // first step with delta != 0 (min)
      int mleave = m + Wm1;                      // step after which m leaves the window
      unsigned cta = ctag_s + (unsigned)m * SS, fsa = fsfin_s + 4u * (unsigned)m;
      unsigned cfa = cfin_s + (unsigned)m * TS;
      int nend = Np;                             // set to 0 by the watchdog
      int nlast = -1;

      // Stage the entering columns of batch j (samples n+D+i, n = 4j): lane x
      // copies K[n+D+i][sx] (cp.async, 4 bytes each) with sx = x's sample after
      // the batch, into stage[slot][i][x].  Reads before a row start or past
      // the last sample land in finite Gram entries or the workspace's zero
      // tail rows: they only meet invalid slots.
      auto stage_issue = [&](int jb) {
        const int mb = jb * TC_BT + D + TC_BT - 1;
        const int sx = mb - ((mb - x) & (TC_S - 1));
        const T* src = G + ((long long)(mb - (TC_BT - 1)) * ld + sx);
        const unsigned dst = stage_s + ((jb & (TC_SRING - 1)) * TC_BT * TC_S + x) * TS;
#pragma unroll
        for (int i = 0; i < TC_BT; ++i) cp_async_s(dst + i * TC_S * TS, src + i * ld);
        if (STG && x < TC_BT) {                      // the batch's targets (clamped past the end)
          const int mi = mb - (TC_BT - 1) + x;
          cp_async_s(tst_s + ((jb & (TC_SRING - 1)) * TC_BT + x) * TS, B + (mi < Np ? mi : Np - 1));
        }
        cp_async_commit();
      };
#pragma unroll 1
      for (int p = 0; p < TC_PF; ++p) stage_issue(p);

      // init_m of the samples entering in the next block: issued one step
      // before it is checked (hidden under the window loads)
      T iv = T(0);
      int itag = 0;
      auto init_load = [&](int e0) {                // the load only; the tag is tested later
        const int rel = (x - e0) & (TC_S - 1);
        const int me = e0 + rel;
        ld_tagged(initr_s + (me & (TC_INIT - 1)) * SS, iv, itag);
      };
      auto init_check = [&](int e0) {
        const int rel = (x - e0) & (TC_S - 1);
        const bool isent = rel < TC_BT;
        const int me = e0 + rel;
        bool iok = !isent || itag == me || me >= Np;
        if ((DBG && (dbgvar & 1)) || (FEAT & 256)) iok = true;
        if (!vote_all(iok)) {                   // rare: the background warps are late
          init_spin<T>(initr_s + (me & (TC_INIT - 1)) * SS, isent, me, Np, &iv, ctl, &nend);
          if (DBG && lane == 0 && fu == 0 && e0 >= 0) dbg[Np + e0] = 1;
        }
        if (isent) { bm = bme - iv; bp = bpe - iv; }
      };
      init_load(0);
      init_check(0);

      T qi, qbm, qbp;
      // weights of step s (uniform_weights, apsm.py:139-153): (qm, ql) = the
      // table row min(s, W-1), or zeros past the last sample
      auto qload = [&](int s, T& qm, T& ql) {
        int idx = s < Wm1 ? s : Wm1;
        idx = s < Np ? idx : W;
        lds_nv_pair(qsm_s + 2 * idx * TS, qm, ql);       // immutable table: hoistable
      };
      auto weights = [&](int s, T qm, T ql) {
        const int d = s - m;
        const T qsel = d == 0 ? ql : ((unsigned)d < (unsigned)W ? qm : T(0));
        qi = qsel * invden;
        qbm = qi * bm;
        qbp = qi * bp;
      };
      {
        T qm, ql;
        qload(0, qm, ql);
        weights(0, qm, ql);
      }
      T qcm[TC_BT], qcl[TC_BT];                  // table rows of the current block's steps 1..4
#pragma unroll
      for (int i = 0; i < TC_BT; ++i) qload(1 + i, qcm[i], qcl[i]);

      // one step: the chain (beta -> broadcast -> window dot) with `mid`
      // issued while the window loads are in flight, then the bookkeeping
      auto step = [&](const int n, auto kc, const bool fresh, auto&& mid) {
        constexpr int k = decltype(kc)::value;
        if (DBG && !(dbgvar & 8) && lane == 0 && fu == 0) dbg[n] = clock64();
        const T v1 = fma(-qi, Y, qbm), v2 = fma(-qi, Y, qbp);
        const T delta = fmax(v1, T(0)) + fmin(v2, T(0));   // q/den * shrink(b - f, eps)
        const unsigned dvb = dv_s + (k & 1) * TC_S * TS;
        sts(dvb + ((x + (TC_S - 1 - k)) & (TC_S - 1)) * TS, delta);   // rotated position
        warp_sync_full();
        typename WinLoad<T>::type wl[8];
        window_load<WM>(dvb, wl);
        const T yz = fresh ? T(0) : Y;                       // a new slot starts from 0
        mid();
        Y = window_fma<k, WM, T>(wl, row, yz);
        if (!(FEAT & 64)) {
          c += delta;
          fs = min(fs, delta != T(0) ? n : 0x7fffffff);
        }
      };
      auto nothing = [] {};

      auto block = [&](const int n0, auto bc) -> bool {
        constexpr int k0 = decltype(bc)::value * TC_BT;      // first step of the block mod 32
        const int n = n0 + k0;
        if (n >= nend) return false;
        const int jb = n >> 2;
        auto mark = [&](int idx) {
          if (DBG && (dbgvar & 4) && lane == 0 && fu == 0) dbg[7 * Np + jb * 8 + idx] = clock64();
        };
        const int rel = (x - (k0 + D)) & (TC_S - 1);
        const bool isnew = rel < TC_BT;                       // slot taken over in this block
        const int mt = n + D + rel;
        const unsigned sb = stage_s + (jb & (TC_SRING - 1)) * TC_BT * TC_S * TS;
        // ---- step n; under its window loads: next step's weights (each
        //      step's weights are formed under the previous step's loads, off
        //      the chain) and this block's staged batch ----
        step(n, ic<(k0 + 0) & 31>{}, false, [&] {
          if (!(FEAT & 32)) weights(n + 1, qcm[0], qcl[0]);
          if (!(FEAT & 8)) cp_async_wait<TC_PF - 1>();
        });
        mark(0);
        // ---- step n+1 ----
        step(n + 1, ic<(k0 + 1) & 31>{}, false, [&] {
          if (!(FEAT & 32)) weights(n + 2, qcm[1], qcl[1]);
          if (!(FEAT & 16)) init_load(n + TC_BT);
        });
        mark(1);
        if (!(FEAT & 1)) {
          // ---- publish samples that left during steps n-2..n+1 (c final) ----
          if ((unsigned)(n + 1 - mleave) < (unsigned)TC_BT && m >= 0) {
            sts(cfa, c);
            st_tag(cta, c, m);
            if (CL > 1) st_tag_cl(bctag_s + (cta - ctag_s), c, m);
            sts_i(fsa, fs == 0x7fffffff ? -1 : fs);
          }
          // ---- c^(n+2) of the slots that stay (the batch's slots give 0):
          //      the new samples' responses to them are formed in this warp ----
          sts(snap_s + ((jb & 1) * TC_S + x) * TS, isnew ? T(0) : c);
        }
        warp_sync_full();                                     // staged batch visible to all
        // ---- takeover of the batch n+D .. n+D+3: the staged columns (the new
        //      slots accumulate from step n+2; the loads land under its chain) ----
        T diag = T(0), bt = T(0);
        if (!(FEAT & 2)) {
#pragma unroll
          for (int i = 0; i < TC_BT; ++i)
            row[(k0 + D + i) & (TC_S - 1)] = lds_t<T>(sb + (i * TC_S + x) * TS);
          if (isnew) load_row32(sb + (rel & (TC_BT - 1)) * TC_S * TS, row);
        }
        if (!(FEAT & 4)) {
          diag = lds_t<T>(sb + ((rel & (TC_BT - 1)) * TC_S + x) * TS);
          if constexpr (STG)
            bt = lds_t<T>(tst_s + ((jb & (TC_SRING - 1)) * TC_BT + (rel & (TC_BT - 1))) * TS);
          else
            bt = lds_nv(bsm_s + (unsigned)mt * TS, T(0));
        }
        mark(2);
        // ---- step n+2: the new slots start from 0; entry check of the next
        //      block's samples; the slot coefficients for the in-slot init ----
        T cs[TC_S];
        step(n + 2, ic<(k0 + 2) & 31>{}, isnew, [&] {
          if (!(FEAT & 32)) weights(n + 3, qcm[2], qcl[2]);
          if (!(FEAT & 16)) init_check(n + TC_BT);
          if (!(FEAT & 2)) {
            const unsigned csa = snap_s + (jb & 1) * TC_S * TS;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              T c4[4];
              lds_quad<T>(csa + 4 * q * TS, c4);
              cs[4 * q] = c4[0]; cs[4 * q + 1] = c4[1]; cs[4 * q + 2] = c4[2]; cs[4 * q + 3] = c4[3];
            }
          }
        });
        mark(3);
        if (!(FEAT & 4)) {                                    // takeover state
          const bool v = mt < Np;
          const T inv = v ? recip(diag) : T(0);
          degen |= isnew && v && !(diag > T(0));
          m = isnew ? mt : m;
          c = isnew ? T(0) : c;
          fs = isnew ? 0x7fffffff : fs;
          invden = isnew ? inv : invden;
          bme = isnew ? bt - eps : bme;
          bpe = isnew ? bt + eps : bpe;
          mleave = isnew ? mt + Wm1 : mleave;
          cta = isnew ? ctag_s + (unsigned)mt * SS : cta;
          fsa = isnew ? fsfin_s + 4u * (unsigned)mt : fsa;
          cfa = isnew ? cfin_s + (unsigned)mt * TS : cfa;
        }
        if (!(FEAT & 8)) stage_issue(jb + TC_PF);
        // ---- step n+3; after it: the in-slot part of the new samples' init,
        //      sum_l c_l^(n+2) K[sample(l)][mt], folded into their targets ----
        step(n + 3, ic<(k0 + 3) & 31>{}, false, [&] {
          if (!(FEAT & 32)) {
            weights(n + TC_BT, qcm[3], qcl[3]);
#pragma unroll
            for (int i = 0; i < TC_BT; ++i) qload(n + TC_BT + 1 + i, qcm[i], qcl[i]);
          }
        });
        mark(4);
        if (!(FEAT & 2)) {
          T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            a0 = fma(cs[4 * q], row[4 * q], a0);
            a1 = fma(cs[4 * q + 1], row[4 * q + 1], a1);
            a2 = fma(cs[4 * q + 2], row[4 * q + 2], a2);
            a3 = fma(cs[4 * q + 3], row[4 * q + 3], a3);
          }
          const T yinit = (a0 + a1) + (a2 + a3);
          if (isnew) { bme -= yinit; bpe -= yinit; bm -= yinit; bp -= yinit; }
        }
        mark(5);
        nlast = n + 1;                             // last publication point
        return true;
      };

#pragma unroll 1
      for (int n0 = 0; n0 < nend; n0 += TC_S) {
        block(n0, ic<0>{}) && block(n0, ic<1>{}) && block(n0, ic<2>{}) && block(n0, ic<3>{}) &&
            block(n0, ic<4>{}) && block(n0, ic<5>{}) && block(n0, ic<6>{}) &&
            block(n0, ic<7>{});
      }
      cp_async_wait<0>();                       // outstanding staged batches
      const bool aborted = nend == 0;
      // samples still in the window after the last step: coefficients final now
      if (!aborted && nlast >= 0 && m >= 0 && m < Np && mleave > nlast) {
        sts(cfa, c);
        sts_i(fsa, fs == 0x7fffffff ? -1 : fs);
      }
      const bool any_degen = __any_sync(0xffffffffu, degen != 0);
      __syncwarp();
      if (lane == 0) {
        if (any_degen) atomicOr(&ctl[2], KAPSM_TRAIN_DEGENERATE);
        if (aborted) raise_abort(KAPSM_TRAIN_STALLED);
      }
    } else if (role >= 0 && !(DBG && (dbgvar & 2)) && !(FEAT & 128)) {
      // ============================ INIT WORKERS ============================
      // The batch of sample m is taken over after step n_m = (m-D) & ~3; the
      // critical warp itself forms the new slot's response to the coefficients
      // that stay in the slots (samples n_m+D-28 .. n_m).  Everything older is
      // final by then, and the init workers (the other CTA of the cluster when
      // CL = 2) supply
      //   init_m = f0(r_m) + sum_{i <= lastF} cfinal_i K[m][i],  lastF = n_m + D - 29,
      // as an early part over i <= m - Q (final ~Q-W steps before m is taken
      // over: its Gram row is streamed from L2 into registers, double
      // buffered) plus a late part over (m - Q, lastF] (one element per lane)
      // once c_lastF is published, and push it into the critical CTA's ring.
      // Early workers (NE warps) compute the early part far ahead into a local
      // tagged ring; late finishers (NL warps) wait for c_lastF, add the late
      // part and push init_m: the deadline path is short and never queued
      // behind a long dot.
      constexpr int NE = R::NE, NL = R::NL;
      const bool early = role < NE;                        // roles 0..NE-1 early, NE.. late
      const int j = early ? role : role - NE;
      const int nw = early ? NE : NL;
      const unsigned gbase = smem_u32(gs);
      const unsigned ctag_s = gbase + (unsigned)L.ctag, ering_s = gbase + (unsigned)L.ering;
      const unsigned cinitr_s = cw_base + (unsigned)L.initr;   // the critical CTA's rings
      const unsigned cering_s = cw_base + (unsigned)L.ering;
      auto mtask = [&](int t) { return FIRST + j + t * nw; };
      bool stop = false;
      if (early && j == 0)                                 // f0 only before any update
        for (int i = lane; i < FIRST && i < Np; i += 32)
          st_tag_cl(cinitr_s + (i & (TC_INIT - 1)) * SS, P0 ? P0[i] : T(0), i);
      auto wait_final = [&](int i) {                      // c_i published?
        T cl;
        long long spins = 0;
        while (!stop && !ld_tag(ctag_s + i * SS, i, cl))
          if (((++spins) & 1023) == 0 && (spins > TC_SPIN_LIMIT || ld_volatile(&ctl[1])))
          { stop = true; red_or_cl(cw_base + (unsigned)L.ctl + 8u, 32); }
        if (__any_sync(0xffffffffu, stop)) stop = true;
      };
      // the critical warp covers the slots that stay through the takeover:
      // samples n_m+D-28 .. n_m; the taken-over slots' old samples and all
      // older ones are final by then
      auto lastf = [&](int mt) { return ((mt - D) & ~(TC_BT - 1)) + D - TC_S + TC_BT - 1; };
      if (early) {
        // ------------------------- early part: i <= m - Q -------------------------
        using V16 = typename Vec16<T>::type;               // 16-byte vector of T
        constexpr int EPV = 16 / sizeof(T);
        constexpr int CH = 32 * EPV * ACH;                 // row elements per register chunk
        V16 ra0[ACH], ra1[ACH];
        auto a_issue = [&](V16 (&ra)[ACH], int mt, int lastA, int c0) {
          const T* rowp = G + (long long)mt * ld;
#pragma unroll
          for (int u = 0; u < ACH; ++u) {
            const int i = c0 + (u * 32 + lane) * EPV;
            if (i <= lastA) ra[u] = ldg16(rowp + i);
          }
        };
        // chunk c0 against the published final coefficients (tagged; a tag not
        // yet visible makes the chunk redo)
        auto a_dot = [&](const V16 (&ra)[ACH], int lastA, int c0) -> T {
          for (;;) {
            T acc0 = T(0), acc1 = T(0);
            bool bad = false;
#pragma unroll
            for (int u = 0; u < ACH; ++u) {
              const int i = c0 + (u * 32 + lane) * EPV;
              if (i + EPV - 1 <= lastA) {
                acc0 = tagged_dot16<T>(ctag_s + i * SS, i, ra[u], acc0, bad);
              } else if (i <= lastA) {
                for (int e = 0; e < EPV && i + e <= lastA; ++e) {
                  T cv;
                  bad |= !ld_tag(ctag_s + (i + e) * SS, i + e, cv);
                  acc1 = fma(cv, elem16(ra[u], e), acc1);
                }
              }
            }
            if (!__any_sync(0xffffffffu, bad)) return acc0 + acc1;
          }
        };
        auto a_start = [&](V16 (&ra)[ACH], int t) {
          const int mt = mtask(t);
          if (mt < Np && mt - TC_Q >= 0) a_issue(ra, mt, mt - TC_Q, 0);
        };
        auto a_finish = [&](V16 (&ra)[ACH], int t) -> bool {
          const int mt = mtask(t);
          if (mt >= Np) return false;
          const int lastA = mt - TC_Q;
          T part = T(0);
          if (lastA >= 0) {
            wait_final(lastA);
            if (stop) return false;
            part = a_dot(ra, lastA, 0);
            for (int c0 = CH; c0 <= lastA; c0 += CH) {      // rows longer than one chunk
              a_issue(ra, mt, lastA, c0);                   // (the consumed buffer is reused)
              part += a_dot(ra, lastA, c0);
            }
            part = warp_sum(part);
          }
          if (lane == 0) st_tag_cl(cering_s + (mt & (TC_ERING - 1)) * SS, part + (P0 ? P0[mt] : T(0)), mt);
          return true;
        };
        a_start(ra0, 0);
        for (int t = 0; !stop; t += 2) {                    // unrolled by 2: buffers swap
          a_start(ra1, t + 1);
          if (!a_finish(ra0, t)) break;
          a_start(ra0, t + 2);
          if (!a_finish(ra1, t + 1)) break;
        }
      } else {
        // ---------------- late part (m - Q, lastF], then publish ----------------
        const unsigned initr_s_loc = gbase + (unsigned)L.initr;   // (the critical CTA)
        auto l_load = [&](int t) -> T {                   // one Gram entry per lane
          const int mt = mtask(t);
          const int i = mt - TC_Q + 1 + lane;
          return (mt < Np && i >= 0 && i <= lastf(mt)) ? G[(long long)mt * ld + i] : T(0);
        };
        auto l_task = [&](int t, T kl) -> bool {
          const int mt = mtask(t);
          if (mt >= Np) return false;
          const int lastF = lastf(mt);
          T part = T(0);
          if (DBG && lane == 0 && fu == 0) dbg[3 * Np + mt] = clock64();
          if (lastF >= 0) {
            wait_final(lastF);
            if (stop) return false;
            if (DBG && lane == 0 && fu == 0) dbg[5 * Np + 1 + mt] = clock64();
            const int i = mt - TC_Q + 1 + lane;
            for (;;) {
              T cv = T(0);
              bool bad = false;
              if (i >= 0 && i <= lastF) bad = !ld_tag(ctag_s + i * SS, i, cv);
              if (!__any_sync(0xffffffffu, bad)) { part = cv * kl; break; }
            }
            part = warp_sum(part);
          }
          if (lane == 0) {
            T e;
            long long spins = 0;
            while (!ld_tag(ering_s + (mt & (TC_ERING - 1)) * SS, mt, e))
              if (((++spins) & 1023) == 0 && (spins > TC_SPIN_LIMIT || ld_volatile(&ctl[1]))) {
                stop = true; red_or_cl(cw_base + (unsigned)L.ctl + 8u, 16);
                break;
              }
            if (DBG && fu == 0) dbg[4 * Np + mt] = clock64();
            st_tag(initr_s_loc + (mt & (TC_INIT - 1)) * SS, e + part, mt);
          }
          stop = __shfl_sync(0xffffffffu, stop, 0);
          return !stop;
        };
        T kl0 = l_load(0), kl1;
        for (int t = 0; !stop; t += 2) {                    // unrolled by 2: entries swap
          kl1 = l_load(t + 1);
          if (!l_task(t, kl0)) break;
          kl0 = l_load(t + 2);
          if (!l_task(t + 1, kl1)) break;
        }
      }
      if (stop && lane == 0) raise_abort(KAPSM_TRAIN_STALLED);
    }
    group_sync();
    if (CL > 1 && rank != 0) continue;          // the epilogue runs in the critical CTA
    // ---- outputs: coefficients, first steps (coalesced), activation count ----
    {
      int na = 0;
      for (int i = gt; i < Np; i += GT) {
        coeff_out[(long long)fu * Np + i] = cfin[i];
        const int v = fsfin[i];
        fs_out[(long long)fu * Np + i] = v;
        na += (v >= 0);
      }
      na = (int)warp_sum((float)na);
      if (lane == 0) atomicAdd(&ctl[3], na);
    }
    // ---- theta = theta0 + w_l sum_i c_i r_i (kernels.py:130-141 / apsm.py:338) ----
    {
      T* th = theta_out + (long long)fu * dim;
      const T* t0 = theta0 ? theta0 + (long long)fu * dim : nullptr;
      constexpr int nw = NG == 1 ? R::WARPS : NB + 1;
      const int ew = NG == 1 ? warp : role;
      // the chain's tagged coefficient words are dead now: they hold the
      // cross-warp partial sums of the coalesced form below
      T* red = reinterpret_cast<T*>(ctag);
      const bool coalesced = dim <= 128 && (size_t)nw * dim * sizeof(T) <= (size_t)(Np + TC_S) * SS;
      if (rx && coalesced) {
        // complex pilots: Theta = theta[:M] + i theta[M:] = w_l sum_p (c_2p - i c_2p+1) x_p.
        // Lanes run over a pilot row's 2M interleaved components (coalesced
        // rows), warps over pilots; pairs of lanes and then the warps (fixed
        // order) are summed.
        const int M = dim / 2, n_train = Np / 2;
        const T* X = rx + (long long)f * rx_stride;
        T A[4] = {T(0), T(0), T(0), T(0)}, Bq[4] = {T(0), T(0), T(0), T(0)};
        const bool odd = lane & 1;
#pragma unroll 4
        for (int p = ew; p < n_train; p += nw) {
          const T c1 = cfin[2 * p], c2 = cfin[2 * p + 1];
          const T ca = odd ? c2 : c1, cb = odd ? c1 : -c2;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e = lane + 32 * q;
            if (e < dim) {
              const T v = X[(long long)p * dim + e];
              A[q] = fma(ca, v, A[q]);
              Bq[q] = fma(cb, v, Bq[q]);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const T a1 = __shfl_down_sync(0xffffffffu, A[q], 1);
          const T b1 = __shfl_down_sync(0xffffffffu, Bq[q], 1);
          const int e = lane + 32 * q;
          if (!odd && e < dim) {
            red[ew * dim + e / 2] = A[q] + a1;           // real part of component e/2
            red[ew * dim + M + e / 2] = Bq[q] + b1;      // imaginary part
          }
        }
        named_bar(group_bar, GT);
        for (int e = gt; e < dim; e += GT) {
          T acc = T(0);
          for (int w = 0; w < nw; ++w) acc += red[w * dim + e];
          th[e] = w_l * acc + (t0 ? t0[e] : T(0));
        }
      } else if (rx) {
        // complex pilots, strided form (reduction buffer too small)
        const int M = dim / 2, n_train = Np / 2;
        const T* X = rx + (long long)f * rx_stride;
        for (int kk = ew; kk < M; kk += nw) {
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
        const T* S = samples + (long long)f * samples_stride;
        for (int kk = ew; kk < dim; kk += nw) {
          T acc = T(0);
#pragma unroll 8
          for (int i = lane; i < Np; i += 32) acc = fma(cfin[i], S[(long long)i * dim + kk], acc);
          acc = warp_sum(acc);
          if (lane == 0) th[kk] = w_l * acc + (t0 ? t0[kk] : T(0));
        }
      }
    }
    named_bar(group_bar, GT);
    if (gt == 0) {
      status_out[fu] = ctl[2];
      nact_out[fu] = ctl[3];
    }
    named_bar(group_bar, GT);                      // state reused by the next task
  }
}

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

template <typename T, int NG, int CL, int WM, bool STG>
int launch_train(int tasks, cudaStream_t s, const T* gram, long long ld, long long gram_stride,
                 const T* rx, long long rx_stride, const T* samples, long long samples_stride,
                 int dim, const T* targets, int F, int K, int Np, int W, double eps,
                 kapsm_kernel_params p, const T* qtab, const T* base0, const T* theta0, T* coeff,
                 int* first_step, T* theta, int* n_active, int* status, long long* dbg) {
  auto kern = apsm_train_kernel<T, NG, CL, WM, false, STG>;
  if constexpr (sizeof(T) == 4 && NG == 1 && WM == 20 && !STG) {   // clock instrumentation build
    if (dbg) kern = apsm_train_kernel<T, NG, CL, WM, true, false>;
  } else if (dbg) {
    return KAPSM_ERR_UNSUPPORTED;
  }
  const GroupSmem<T, NG, CL> L(W, Np, STG);
  size_t smem = L.total * NG;
  // NG = 1: pad shared memory so that the two CTAs of a cluster land on
  // different SMs (the latency pipeline's concurrent detection screen asks
  // for more than the rest of an SM, so it cannot share them either)
  if (NG == 1 && smem < 120 * 1024) smem = 120 * 1024;
  if (smem > 227 * 1024) return KAPSM_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  int groups = (tasks + NG - 1) / NG;                 // CTAs (CL = 1) or clusters (CL = 2)
  const int max_groups = num_sms() / CL;
  if (groups > max_groups) groups = max_groups;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(groups * CL);
  cfg.blockDim = dim3(Roles<NG, CL>::WARPS * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(
      &cfg, kern, gram, ld, gram_stride, rx, rx_stride, samples, samples_stride, dim, targets, F,
      K, Np, W, (T)eps, (T)p.w_l, qtab, base0, theta0, coeff, first_step, theta, n_active, status,
      dbg);
  if (e != cudaSuccess) return KAPSM_ERR_CUDA;
  return status_from(cudaGetLastError());
}

template <typename T, int NG, int CL>
int launch_train_w(int tasks, cudaStream_t s, const T* gram, long long ld, long long gram_stride,
                   const T* rx, long long rx_stride, const T* samples, long long samples_stride,
                   int dim, const T* targets, int F, int K, int Np, int W, double eps,
                   kapsm_kernel_params p, const T* qtab, const T* base0, const T* theta0, T* coeff,
                   int* first_step, T* theta, int* n_active, int* status, long long* dbg,
                   bool stg = false) {
#define KAPSM_LT(WMV)                                                                          \
  do {                                                                                         \
    if (NG == 1 && stg)                                                                        \
      return launch_train<T, NG, CL, WMV, true>(tasks, s, gram, ld, gram_stride, rx, rx_stride, \
                                                samples, samples_stride, dim, targets, F, K, Np, \
                                                W, eps, p, qtab, base0, theta0, coeff,           \
                                                first_step, theta, n_active, status, dbg);       \
    return launch_train<T, NG, CL, WMV, false>(tasks, s, gram, ld, gram_stride, rx, rx_stride,  \
                                               samples, samples_stride, dim, targets, F, K, Np,  \
                                               W, eps, p, qtab, base0, theta0, coeff,            \
                                               first_step, theta, n_active, status, dbg);        \
  } while (0)
  // the window dot covers the WM newest slots (static per unrolled step)
#ifdef KAPSM_EXP_ONLY
  if (W == 20) KAPSM_LT(20);
  return KAPSM_ERR_UNSUPPORTED;
#endif
  if (W <= 8) KAPSM_LT(8);
  if (W <= 16) KAPSM_LT(16);
  if (W <= 20) KAPSM_LT(20);
  KAPSM_LT(TC_MAX_W);
  static_assert(lookahead(TC_MAX_W) == 8, "the entry/takeover schedule assumes D = 8");
#undef KAPSM_LT
}

// the general trainer (train_wide.cu) for windows / pilot counts beyond the
// latency kernel's schedule
template <typename T>
int train_wide(const T* gram, long long ld, long long gram_stride, const T* rx,
               long long rx_stride, const T* samples, long long samples_stride, int dim,
               const T* targets, int F, int K, int Np, int W, double eps, kapsm_kernel_params p,
               const T* qtab, const T* base0, const T* theta0, T* coeff, int* first_step,
               T* theta, int* n_active, int* status, cudaStream_t s);
int train_wide_max_window();

template <typename T>
int train(const T* gram, long long ld, long long gram_stride, const T* rx, long long rx_stride,
          const T* samples, long long samples_stride, int dim, const T* targets, int F, int K,
          int Np, int W, double eps, kapsm_kernel_params p, const T* qtab, const T* base0,
          const T* theta0, T* coeff, int* first_step, T* theta, int* n_active, int* status,
          cudaStream_t s, long long* dbg = nullptr, bool general = false) {
  if (F < 0 || K < 1 || Np < 1 || dim < 1 || W < 1 || !(eps > 0)) return KAPSM_ERR_INVALID;
  if (F == 0) return KAPSM_OK;
  if (!gram || !targets || !coeff || !first_step || !theta || !n_active || !status)
    return KAPSM_ERR_INVALID;
  if ((rx == nullptr) == (samples == nullptr)) return KAPSM_ERR_INVALID;  // exactly one source
  if (rx && ((Np & 1) || (dim & 1))) return KAPSM_ERR_INVALID;
  // rows: 16-byte aligned with >= 16 padding columns (kapsm_b200.h)
  if (ld < Np + 16 || (ld * (long long)sizeof(T)) % 16 ||
      (gram_stride * (long long)sizeof(T)) % 16 || ((size_t)gram & 15))
    return KAPSM_ERR_INVALID;
  const int tasks = F * K;
  // the general trainer beyond the latency schedule's window or its
  // shared-memory footprint (per-sample words in the chain's CTAs), or at any
  // size through kapsm_train_general_* (parity tests of that kernel)
  // targets staged with the columns once the per-sample target array no
  // longer fits beside the tagged coefficients
  const bool stg = GroupSmem<T, 1, 2>(W, Np, false).total > 227 * 1024;
  if (W > TC_MAX_W || Np > TC_MAX_NP || GroupSmem<T, 1, 2>(W, Np, true).total > 227 * 1024 ||
      general) {
    if (dbg) return KAPSM_ERR_UNSUPPORTED;
    return train_wide<T>(gram, ld, gram_stride, rx, rx_stride, samples, samples_stride, dim,
                         targets, F, K, Np, W, eps, p, qtab, base0, theta0, coeff, first_step,
                         theta, n_active, status, s);
  }
  // latency mode (a 2-CTA cluster per chain) while the chains fit twice on the
  // SMs; throughput mode (4 chains per SM) beyond.  FP64 (the parity/test
  // precision) always runs in latency mode.
  const bool lat = stg || sizeof(T) == 8 || tasks <= num_sms() ||
                   GroupSmem<T, 4, 1>(W, Np).total * 4 > 227 * 1024;
  if (lat)
    return launch_train_w<T, 1, 2>(tasks, s, gram, ld, gram_stride, rx, rx_stride, samples,
                                   samples_stride, dim, targets, F, K, Np, W, eps, p, qtab, base0,
                                   theta0, coeff, first_step, theta, n_active, status, dbg, stg);
#ifdef KAPSM_EXP_ONLY
  return KAPSM_ERR_UNSUPPORTED;
#endif
  if constexpr (sizeof(T) == 8) return KAPSM_ERR_UNSUPPORTED;
  else
    return launch_train_w<T, 4, 1>(tasks, s, gram, ld, gram_stride, rx, rx_stride, samples,
                                   samples_stride, dim, targets, F, K, Np, W, eps, p, qtab, base0,
                                   theta0, coeff, first_step, theta, n_active, status, dbg);
}

// true when train<T> leaves its fast schedule at this shape: the general
// trainer, or the latency schedule with its targets staged beside the Gram
// columns (long pilot blocks); the FP32 pipeline prefers the one-warp
// trainer there (pipeline.cu)
template <typename T>
bool train_takes_general(int Np, int W) {
  return W > TC_MAX_W || Np > TC_MAX_NP || GroupSmem<T, 1, 2>(W, Np, true).total > 227 * 1024 ||
         GroupSmem<T, 1, 2>(W, Np, false).total > 227 * 1024;
}
template bool train_takes_general<float>(int, int);
template bool train_takes_general<double>(int, int);

}  // namespace kapsm

extern "C" int kapsm_max_window(void) { return kapsm::train_wide_max_window(); }

// beyond this the shared-memory footprint decides (KAPSM_ERR_UNSUPPORTED)
extern "C" int kapsm_max_samples(void) { return 1 << 20; }

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

#define KAPSM_TRAIN_GENERAL_ENTRY(NAME, T)                                                     \
  extern "C" int NAME(const T* gram, long long ld, long long gram_stride, const T* rx,         \
                      long long rx_stride, const T* samples, long long samples_stride, int dim, \
                      const T* targets, int F, int K, int n_samples, int window,               \
                      double epsilon, kapsm_kernel_params p, const T* qtab, const T* base0,    \
                      const T* theta0, T* coeff, int* first_step, T* theta, int* n_active,     \
                      int* status, void* stream) {                                             \
    return kapsm::train<T>(gram, ld, gram_stride, rx, rx_stride, samples, samples_stride, dim, \
                           targets, F, K, n_samples, window, epsilon, p, qtab, base0, theta0,  \
                           coeff, first_step, theta, n_active, status, (cudaStream_t)stream,   \
                           nullptr, true);                                                     \
  }
KAPSM_TRAIN_GENERAL_ENTRY(kapsm_train_general_f32, float)
KAPSM_TRAIN_GENERAL_ENTRY(kapsm_train_general_f64, double)

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
  (void)variant;
  return kapsm::train<float>(gram, ld, gram_stride, rx, rx_stride, nullptr, 0, dim, targets, F, K,
                             n_samples, window, epsilon, p, qtab, nullptr, nullptr, coeff,
                             first_step, theta, n_active, status, (cudaStream_t)stream, clocks);
}
