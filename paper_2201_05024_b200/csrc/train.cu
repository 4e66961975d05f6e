// K2: persistent APSM trainer.  One CTA per SM runs 4 independent chain
// groups (one per SM sub-partition); each group trains one (frame, user) at a
// time and loops over its share of the F*K tasks.
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
//   * window update after step n's betas (one 32-term dot per lane):
//       Y_m += sum_l delta_l K[l][m]                      (m in J_n)
//   * the entering sample n+1 gets its full response from the same dot with
//     the coefficient vector instead of delta:
//       Y_{n+1} = sum_l c_l^(n+1) K[l][n+1] + P_{n+1},
//       P_m = f0(r_m) + sum_{i <= m-32} cfinal_i K[i][m];
//   * P is computed by 3 BACKGROUND warps per group: final coefficients are
//     published as tagged 64-bit words (value + index, no fence needed); warp
//     k computes P_m for m = 32+k (mod 3) as one coalesced warp-wide dot over
//     Gram row m as soon as c_{m-32} is final, and publishes it tagged, about
//     S-W steps before the critical warp needs it;
//   * taking over sample n+2 needs one Gram row segment (32 values), staged by
//     cp.async TR_DELTA steps ahead; it refreshes one entry of every lane's
//     column and the whole column of the new lane (symmetry).
// Scheduling: group g = warp % 4 lives on sub-partition g; its critical warp
// has the highest warp id there (the issue arbiter favours it) and there is
// exactly one CTA per SM, so no foreign warp can starve a critical warp.
#include <type_traits>
#include "kapsm_common.cuh"

namespace kapsm {

constexpr int TR_S = 32;           // critical slots (one warp)
constexpr int TR_BGW = 3;          // background warps per group
constexpr int TR_BGL = TR_BGW * 32;   // background lanes per group
constexpr int TR_NJ = 16;          // P accumulators per background lane (registers)
constexpr int TR_RB = 4;           // Gram rows in the TMA ring
constexpr int TR_DELTA = 8;        // column prefetch distance (steps)
constexpr int TR_PBN = 64;         // P slots (ring)
constexpr int TR_CR = 64;          // final-coefficient slots (ring, power of 2)
constexpr int TR_CSTR = TR_S + 4;  // col2 row stride: 16B rows, conflict-free LDS.128
constexpr int TR_STG = 16;         // staged Gram rows (ring, power of 2 >= DELTA+2)
constexpr int TR_MIN_LB = 7;       // minimum look-behind (background slack)
constexpr int TR_MAX_W = TR_S - 1 - TR_MIN_LB;
constexpr int TR_MAX_NP = TR_BGL * TR_NJ;
constexpr long long TR_SPIN_LIMIT = 1LL << 26;

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

// the lane's 32-entry Gram row (16-byte aligned smem) into registers
KAPSM_DEV void load_row32(const float* p, float (&r)[32]) {
  const float4* p4 = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 v = p4[q];
    r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
  }
}
KAPSM_DEV void load_row32(const double* p, double (&r)[32]) {
  const double2* p2 = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const double2 v = p2[q];
    r[2 * q] = v.x; r[2 * q + 1] = v.y;
  }
}
// 32-term dot of a broadcast smem vector (LDS.128) with a register row
KAPSM_DEV float dot32_reg(const float* a, const float (&r)[32]) {
  const float4* a4 = reinterpret_cast<const float4*>(a);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 u = a4[q];
    s0 = fmaf(u.x, r[4 * q], s0);
    s1 = fmaf(u.y, r[4 * q + 1], s1);
    s2 = fmaf(u.z, r[4 * q + 2], s2);
    s3 = fmaf(u.w, r[4 * q + 3], s3);
  }
  return (s0 + s1) + (s2 + s3);
}
KAPSM_DEV double dot32_reg(const double* a, const double (&r)[32]) {
  const double2* a2 = reinterpret_cast<const double2*>(a);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
  for (int q = 0; q < 16; q += 2) {
    const double2 u = a2[q], u2 = a2[q + 1];
    s0 = fma(u.x, r[2 * q], s0);
    s1 = fma(u.y, r[2 * q + 1], s1);
    s2 = fma(u2.x, r[2 * q + 2], s2);
    s3 = fma(u2.y, r[2 * q + 3], s3);
  }
  return (s0 + s1) + (s2 + s3);
}

// sum_{i=0..last} c_i row[i] over a warp, with c_i read from the tagged array
// (value, index) and a mismatch flag instead of a per-element wait.  float:
// each lane takes 4 consecutive columns per LDS.128 (row) + 2 LDS.128 (tags).
template <typename T>
KAPSM_DEV T tagged_dot(const T* row, const typename Tagged<T>::slot_t* ctag, int last, int lane,
                       bool& bad);
template <>
KAPSM_DEV float tagged_dot<float>(const float* row, const unsigned long long* ctag, int last,
                                  int lane, bool& bad) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  const int n = last + 1;
  int i = 4 * lane;
  for (; i + 3 < n; i += 128) {
    const float4 r = *reinterpret_cast<const float4*>(row + i);
    const uint4 t01 = *reinterpret_cast<const uint4*>(ctag + i);
    const uint4 t23 = *reinterpret_cast<const uint4*>(ctag + i + 2);
    bad |= (int)t01.y != i || (int)t01.w != i + 1 || (int)t23.y != i + 2 || (int)t23.w != i + 3;
    s0 = fmaf(__uint_as_float(t01.x), r.x, s0);
    s1 = fmaf(__uint_as_float(t01.z), r.y, s1);
    s2 = fmaf(__uint_as_float(t23.x), r.z, s2);
    s3 = fmaf(__uint_as_float(t23.z), r.w, s3);
  }
  for (int k = i; k < i + 4 && k < n; ++k) {      // ragged tail of this lane's block
    const unsigned long long w = ctag[k];
    bad |= (int)(w >> 32) != k;
    s0 = fmaf(__uint_as_float((unsigned)(w & 0xffffffffu)), row[k], s0);
  }
  return warp_sum((s0 + s1) + (s2 + s3));
}
template <>
KAPSM_DEV double tagged_dot<double>(const double* row, const Tagged<double>::slot_t* ctag,
                                    int last, int lane, bool& bad) {
  double s0 = 0.0, s1 = 0.0;
  int i = lane;
  for (; i + 32 <= last; i += 64) {
    const Tagged<double>::slot_t a = ctag[i], b = ctag[i + 32];
    bad |= (int)a.t != i || (int)b.t != i + 32;
    s0 = fma(__longlong_as_double((long long)a.v), row[i], s0);
    s1 = fma(__longlong_as_double((long long)b.v), row[i + 32], s1);
  }
  if (i <= last) {
    const Tagged<double>::slot_t a = ctag[i];
    bad |= (int)a.t != i;
    s0 = fma(__longlong_as_double((long long)a.v), row[i], s0);
  }
  return warp_sum(s0 + s1);
}

template <typename T>
struct GroupSmem {
  // byte offsets of one group's region in dynamic shared memory
  size_t mbar, pbuf, cring, col, stage, bstage, dbuf, qsm, cfin, fsfin, ring, ctl, total;
  int npr;   // elements per ring row
  __host__ __device__ GroupSmem(int W, int Np) {
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 15) & ~size_t(15); return r; };
    npr = (Np + 8 + 7) & ~7;
    mbar = take(TR_BGW * sizeof(unsigned long long));
    pbuf = take(TR_PBN * sizeof(typename Tagged<T>::slot_t));
    cring = take((size_t)(Np + 32) * sizeof(typename Tagged<T>::slot_t));
    col = take((size_t)TR_S * TR_CSTR * sizeof(T));
    stage = take((size_t)TR_STG * TR_S * sizeof(T));
    bstage = take((size_t)TR_STG * sizeof(T));
    dbuf = take(2 * 2 * TR_S * sizeof(T));
    qsm = take(2 * (size_t)W * sizeof(T));
    cfin = take((size_t)(Np + 32) * sizeof(T));
    fsfin = take((size_t)(Np + 32) * sizeof(int));
    ring = take((size_t)TR_BGW * npr * sizeof(T));      // one Gram-row buffer per bg warp
    ctl = take(16 * sizeof(int));
    total = (o + 127) & ~size_t(127);
  }
};

// NG chain groups per CTA.  Warp w belongs to group w % NG with role w / NG:
//   NG = 4 (throughput): group g owns sub-partition g (warps g, g+4, g+8, g+12),
//          its critical warp (role 3) has the highest id there;
//   NG = 1 (latency): background warps 0-2 on sub-partitions 0-2, the critical
//          warp alone on sub-partition 3.
// Either way exactly one CTA runs per SM (registers for NG=4, shared-memory
// padding for NG=1), so no foreign warp competes with a critical warp.
template <typename T, int NG, int VAR = 0>
__global__ void __launch_bounds__(NG * (TR_BGW + 1) * 32, 1)
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
  extern __shared__ __align__(128) unsigned char smem[];
  const GroupSmem<T> L(W, Np);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp % NG;                   // chain group of this warp
  const int role = warp / NG;                  // 0..BGW-1: background, BGW: critical
  const int gt = role * 32 + lane;             // thread index inside the group
  unsigned char* gs = smem + (size_t)grp * L.total;
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(gs + L.mbar);
  Slot* pbuf = reinterpret_cast<Slot*>(gs + L.pbuf);    // [PBN]   tagged P_m
  Slot* ctag = reinterpret_cast<Slot*>(gs + L.cring);   // [Np+32] tagged final c_m (+junk)
  T* col2 = reinterpret_cast<T*>(gs + L.col);           // [S][CSTR]
  T* stage = reinterpret_cast<T*>(gs + L.stage);        // [STG][S]
  T* bstage = reinterpret_cast<T*>(gs + L.bstage);      // [STG]
  T* dbuf = reinterpret_cast<T*>(gs + L.dbuf);          // [2][2S]
  T* qsm = reinterpret_cast<T*>(gs + L.qsm);            // [W][2]
  T* cfin = reinterpret_cast<T*>(gs + L.cfin);          // [Np + 32]  (+junk)
  int* fsfin = reinterpret_cast<int*>(gs + L.fsfin);    // [Np + 32]  (+junk)
  T* rowbuf = reinterpret_cast<T*>(gs + L.ring);        // [BGW][npr] Gram rows (TMA)
  int* ctl = reinterpret_cast<int*>(gs + L.ctl);        // [1]=abort [2]=status [3]=nact
  const int group_bar = 1 + grp;
  const int GT = (TR_BGW + 1) * 32;

  for (int task = blockIdx.x * NG + grp; task < F * K; task += gridDim.x * NG) {
    const int fu = task;                        // frame * K + user
    const int f = fu / K;
    const T* G = gram + (long long)f * gram_stride;
    const T* B = targets + (long long)fu * Np;  // realified targets (interleaved pilots)
    const T* P0 = base0 ? base0 + (long long)fu * Np : nullptr;

    // ---------------- per-task group state ----------------
    for (int i = gt; i < TR_PBN; i += GT) Tagged<T>::store(&pbuf[i], T(0), -1);
    for (int i = gt; i < Np + 32; i += GT) Tagged<T>::store(&ctag[i], T(0), -1);
    if (gt == 0) {
      for (int r = 0; r < TR_BGW; ++r) mbar_init(&mbar[r], 1);
      mbar_fence_init();
    }
    for (int i = gt; i < W; i += GT) {
      T qm = T(1) / T(i + 1), ql = qm;
      if (qtab) { qm = qtab[2 * i]; ql = qtab[2 * i + 1]; }
      qsm[2 * i] = qm;
      qsm[2 * i + 1] = ql;
    }
    for (int i = gt; i < Np + 32; i += GT) { cfin[i] = T(0); fsfin[i] = -1; }
    if (gt < 16) ctl[gt] = 0;
    named_bar(group_bar, GT);

    if (role == TR_BGW) {
      // =========================== CRITICAL WARP ===========================
      // Lane x owns sample m (m = x mod S) from step m-1 to step m+S-2; d = n-m
      // (d = -1: enters next, 0 <= d < W: in the window J_n, d = W-1: leaves
      // after this step, d = S-2: released, slot taken over by m+S).
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
        constexpr bool ST = decltype(steady_tag)::value;   // steady state: branches known
        if (dbg && lane == 0 && fu == 0) dbg[n] = clock64();
        ++d;
        // loads independent of this step's chain, issued first
        T row[TR_S];
        load_row32(myrow, row);
        const int me = n + 1;
        T pv = T(0);
        const bool pok = Tagged<T>::load(&pbuf[me % TR_PBN], me, pv);
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
        // (M) Y_m += sum_l delta_l K[l][m]; the entering sample n+1 instead gets
        //     its full response sum_l c_l K[l][n+1] + P_{n+1}
        const bool enter = (d == -1);
        T* vecs = dbuf + (n & 1) * 2 * TR_S;     // [0,S): delta, [S,2S): c
        vecs[x] = delta;
        vecs[TR_S + x] = c;
        __syncwarp();
        const T acc = (VAR & 4) ? T(0) : dot32_reg(vecs + (enter ? TR_S : 0), row);
        if ((ST || me < Np) && !pok) {             // warp-uniform, rare: P not yet published
          long long spins = 0;
          while (!Tagged<T>::load(&pbuf[me % TR_PBN], me, pv))
            if (++spins > TR_SPIN_LIMIT || (spins & 4095) == 0 && ld_volatile(&ctl[1])) {
              aborted = true;
              break;
            }
          if (dbg && lane == 0 && fu == 0) dbg[Np + n] = spins + 1;
        }
        Y = enter ? acc + pv : Y + acc;
        // (L) sample lo leaves the window after this step: c is final.  Every
        //     lane stores (non-leaving lanes into junk slots): no branch.
        {
          const bool leave = (d == W - 1);
          const int li = leave ? m : Np + x;
          cfin[li] = c;
          fsfin[li] = fs;
          Tagged<T>::store(&ctag[li], c, leave ? m : -1);
        }
        // (P) stage the Gram row of the sample taken over TR_DELTA steps later,
        //     restricted to the samples owned after that takeover; its target
        //     is staged by the lane that will own it
        {
          const int t = n + TR_DELTA, mt = t + 2;
          if (!(VAR & 2) && (ST || (mt >= TR_S && mt < Np))) {
            const int sx = mt - ((mt - x) & (TR_S - 1));      // owned by slot x after takeover
            T* dst = stage + (t & (TR_STG - 1)) * TR_S + x;
            if (ST || sx >= 0) cp_async_scalar(dst, G + (long long)mt * ld + sx);
            if (x == (mt & (TR_S - 1))) cp_async_scalar(bstage + (t & (TR_STG - 1)), B + mt);
          }
          cp_async_commit();
        }
        // (T) release sample n+2-S, take over sample n+2
        const int mt = n + 2;
        if (!(VAR & 2) && (ST || (mt >= TR_S && mt < Np))) {
          cp_async_wait<TR_DELTA>();               // own copies only: no warp sync needed
          const int r = mt & (TR_S - 1);
          const T v = stage[(n & (TR_STG - 1)) * TR_S + x];   // K[mt][sample(x)]
          const T bn = bstage[n & (TR_STG - 1)];               // valid in lane r
          col2[x * TR_CSTR + r] = v;
          col2[r * TR_CSTR + x] = v;
          const T dnew = __shfl_sync(0xffffffffu, v, r);      // K[mt][mt], warp-uniform
          degen |= !(dnew > T(0));
          T inew;
          if constexpr (sizeof(T) == 4) inew = __fdividef(1.0f, dnew);
          else inew = T(1) / dnew;
          const bool take = (x == r);
          m = take ? mt : m;
          d = take ? -2 : d;
          c = take ? T(0) : c;
          fs = take ? -1 : fs;
          b = take ? bn : b;
          invden = take ? inew : invden;
          __syncwarp();                            // col2 writes before next step's row loads
        }
      };

      // steady phase: full window, prefetch and takeover always in range
      const int a0 = TR_S - 2 > W - 1 ? TR_S - 2 : W - 1;
      const int nB0 = a0 < Np ? a0 : Np;
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
      // Background warp k computes P_m for m = S + k, S + k + BGW, ...:
      //   P_m = f0(r_m) + sum_{i <= m-S} c_i K[m][i]
      // one warp-wide dot over Gram row m (coalesced, independent loads) with
      // the final coefficients from the tagged array, as soon as c_{m-S} is
      // final (sample m-S leaves the window S-W+1 steps before P_m is needed).
      for (int mm = 1 + gt; mm < TR_S && mm < Np; mm += TR_BGL)
        Tagged<T>::store(&pbuf[mm % TR_PBN], P0 ? P0[mm] : T(0), mm);
      bool stop = false;
      T* buf = rowbuf + (size_t)role * L.npr;
      unsigned long long* bar = &mbar[role];
      // TMA bulk copy of Gram row mm, columns 0..mm-S (16-byte rounded)
      auto issue_row = [&](int mm) {
        const unsigned bytes = (unsigned)(((mm - TR_S + 1) * (int)sizeof(T) + 15) & ~15);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, bytes);
        tma_bulk_g2s(buf, G + (long long)mm * ld, bytes, bar);
      };
      unsigned phase = 0;
      if (lane == 0 && TR_S + role < Np) issue_row(TR_S + role);
      for (int mm = TR_S + role; mm < Np && !stop; mm += TR_BGW) {
        const int last = mm - TR_S;                  // dot over i = 0..last
        // wait for c_last (coefficients are finalised in index order)
        {
          T cl;
          long long spins = 0;
          while (!Tagged<T>::load(&ctag[last], last, cl))
            if (((++spins) & 1023) == 0 && (spins > TR_SPIN_LIMIT || ld_volatile(&ctl[1]))) {
              stop = true;
              break;
            }
        }
        if (stop) break;
        {
          long long spins = 0;
          while (!mbar_try_wait(bar, phase))
            if (++spins > TR_SPIN_LIMIT) { stop = true; break; }
          phase ^= 1u;
        }
        if (stop) break;
        T pm_part;
        for (;;) {
          bool bad = false;
          pm_part = tagged_dot<T>(buf, ctag, last, lane, bad);
          if (!__any_sync(0xffffffffu, bad)) break;     // a coefficient not yet visible: redo
        }
        const T acc0 = pm_part, acc1 = T(0);
        const T pm = acc0 + acc1;
        if (lane == 0) Tagged<T>::store(&pbuf[mm % TR_PBN], pm + (P0 ? P0[mm] : T(0)), mm);
        __syncwarp();                                // every lane is done with buf
        if (lane == 0 && mm + TR_BGW < Np) issue_row(mm + TR_BGW);
      }
      if (stop && lane == 0) { atomicOr(&ctl[2], KAPSM_TRAIN_STALLED); st_volatile(&ctl[1], 1); }
    }
    named_bar(group_bar, GT);
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
      const int nw = TR_BGW + 1;
      if (rx) {
        // complex pilots: Theta = theta[:M] + i theta[M:] = w_l sum_p (c_2p - i c_2p+1) x_p
        const int M = dim / 2, n_train = Np / 2;
        const T* X = rx + (long long)f * rx_stride;
        for (int k = role; k < M; k += nw) {
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
        for (int k = role; k < dim; k += nw) {
          T acc = T(0);
          for (int i = lane; i < Np; i += 32) acc = fma(cfin[i], S[(long long)i * dim + k], acc);
          acc = warp_sum(acc);
          if (lane == 0) th[k] = w_l * acc + (t0 ? t0[k] : T(0));
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

static int num_sms_impl();
static int num_sms() { return num_sms_impl(); }
static int num_sms_impl() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

template <typename T, int NG, int VAR>
int launch_train(int tasks, size_t group_smem, cudaStream_t s, const T* gram, long long ld,
                 long long gram_stride, const T* rx, long long rx_stride, const T* samples,
                 long long samples_stride, int dim, const T* targets, int F, int K, int Np,
                 int W, double eps, kapsm_kernel_params p, const T* qtab, const T* base0,
                 const T* theta0, T* coeff, int* first_step, T* theta, int* n_active, int* status,
                 long long* dbg) {
  auto kern = apsm_train_kernel<T, NG, VAR>;
  size_t smem = group_smem * NG;
  // NG = 1: pad shared memory so that only one CTA fits per SM
  if (NG == 1 && smem < 120 * 1024) smem = 120 * 1024;
  if (smem > 227 * 1024) return KAPSM_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  int grid = (tasks + NG - 1) / NG;
  if (grid > num_sms()) grid = num_sms();
  kern<<<grid, NG * (TR_BGW + 1) * 32, smem, s>>>(
      gram, ld, gram_stride, rx, rx_stride, samples, samples_stride, dim, targets, F, K, Np, W,
      (T)eps, (T)p.w_l, qtab, base0, theta0, coeff, first_step, theta, n_active, status, dbg);
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
  // TMA row copies read up to 16 bytes past Np inside each (16-byte aligned) row
  if (ld < Np + 16 / (long long)sizeof(T) || (ld * (long long)sizeof(T)) % 16 ||
      (gram_stride * (long long)sizeof(T)) % 16 || ((size_t)gram & 15))
    return KAPSM_ERR_INVALID;
  GroupSmem<T> L(W, Np);
  if (L.total > 227 * 1024) return KAPSM_ERR_UNSUPPORTED;
  const int tasks = F * K;
  // latency mode (one chain per SM) when the tasks fit on the SMs, else 4 per SM
  const bool lat = tasks <= num_sms() || L.total * 4 > 227 * 1024;
#define KAPSM_LT(NGV, V)                                                                     \
  return launch_train<T, NGV, V>(tasks, L.total, s, gram, ld, gram_stride, rx, rx_stride,    \
                                 samples, samples_stride, dim, targets, F, K, Np, W, eps, p, \
                                 qtab, base0, theta0, coeff, first_step, theta, n_active,    \
                                 status, dbg)
  if (lat) {
    switch (variant) {
      case 4: KAPSM_LT(1, 4);
      default: KAPSM_LT(1, 0);
    }
  }
  KAPSM_LT(4, 0);
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
