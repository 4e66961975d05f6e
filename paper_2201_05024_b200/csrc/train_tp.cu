// K2t: the APSM trainer as one warp per (frame, user) chain, for the frame
// pipeline in FP32 (latency and throughput mode alike).
//
// Reference semantics: ApsmTrainer.observe (apsm.py:304-359) over the
// realified pilots of the frame -- at step n the window J_n = [lo_n, n]
// (apsm.py:132-136) gets
//     delta_j = q_j / den_j * shrink(b_j - f_n(r_j), eps)   (apsm.py:323-336)
//     c_j += delta_j, first activation = first n with delta_j != 0 (apsm.py:341-358)
//     f_{n+1} = f_n + sum_j delta_j kappa(r_j, .)            (theta update, apsm.py:338)
// with uniform weights q from the reference's own table (apsm.py:139-153).
//
// Restatement (exact algebra, FP32 rounding):
//   * lane l of the warp owns ring slot l: sample m lives in slot m mod 32 from
//     its takeover at step m - P (P = 28 - W) until it leaves the window after
//     step m + W - 1.  Its response Y_m = f_n(r_m) is a register, updated each
//     step by the window's deltas:  Y_m += sum_j delta_j K[j][m];
//   * K[j][m] (sum kernel, w_l r.r + w_g kappa_G, explicit differences) for
//     all ring pairs is a 32 x 32 shared matrix; a takeover writes the new
//     sample's row and column from the band K[m][m-d], d < 32, made by
//     band_tile_kernel below (no pilot Gram matrix is materialised);
//   * at takeover, f_{m-P}(r_m) = w_l theta_fin . r_m + sum_{j in window} c_j K[j][m]
//       + w_g sum_{a <= m-P-W live} c_a kappa_G(r_a, r_m),
//     theta_fin = sum of c_a r_a over the samples that already left the window
//     (their coefficients are final; the linear part of every older sample),
//     the window part from the band, and the older Gaussian terms from the
//     live list of row m (the tensor-core screen on pilot x pilot pairs,
//     screen_tc.cu: at the paper's channels the list is almost always empty);
//   * theta = w_l theta_fin at the end (apsm.py:338 summed once per sample).
// Global loads run two steps ahead with cp.async (a sample's pilot row, band
// row, target and live count), so the chain never waits on memory.
#include "kapsm_common.cuh"

#include <type_traits>

namespace kapsm {

constexpr int TP_RING = 32;
constexpr int TP_STG = 8;                // cp.async stages (power of 2, > TP_AHEAD)
constexpr int TP_AHEAD = 6;              // prefetch distance (steps): hides a global-memory
                                         // round trip behind ~6 chain steps
constexpr int TP_LIVE_LAG = 2;           // live terms of a sample: 2 steps after its takeover
constexpr int TP_CAP = 8;                // screen list entries per row (SC_CAP)
constexpr int TP_KS = 36;                // row stride of the ring's K matrix: 16-byte rows
                                         // whose LDS.128 phases hit distinct banks

constexpr int TP_SPAN = 28;              // P + W (< 32: slack for the live-term loads)
__host__ __device__ constexpr int tp_lead(int W) { return TP_SPAN - W; }   // takeover lead P

// per-warp shared memory, a compile-time layout for DPL components per lane
// (rows of up to 32 DPL floats); the stage of step n = m - P holds the
// prefetched inputs of that step: the pilot row of the sample taken over (m)
// and of the sample leaving the window (m - TP_SPAN + 1), XR floats each, then
// the band row (32), the target and the live count (8 KB per chain at M <= 16;
// 6 CTAs of 4 chains per SM, bound by the 80 registers)
template <int DPL>
struct TpL {
  static constexpr int XR = 32 * DPL;
  static constexpr int SSTR = 2 * XR + 36;                  // floats per stage
  static constexpr int OKB = 2 * XR, OB = OKB + 32, OLC = OB + 1;
  static constexpr int KS = 0;                              // [32][TP_KS] K over ring pairs
  static constexpr int DSM = KS + TP_RING * TP_KS * 4;      // [32] deltas
  static constexpr int QS = DSM + TP_RING * 4;              // [32][2] (q_mid, q_last)
  static constexpr int STG = QS + 64 * 4;                   // [STG][SSTR] stages
  static constexpr int TOTAL = (STG + TP_STG * SSTR * 4 + 127) & ~127;
};
__host__ __device__ constexpr int tp_dpl(int M) { return (2 * M + 31) / 32; }
__host__ __device__ constexpr int tp_total(int M) {
  return tp_dpl(M) == 1 ? TpL<1>::TOTAL : tp_dpl(M) == 2 ? TpL<2>::TOTAL : TpL<4>::TOTAL;
}

KAPSM_DEV void cpa16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
KAPSM_DEV void cpa4(unsigned dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
// predicated forms (no branch in the chain's loop)
KAPSM_DEV void cpa16_if(bool p, unsigned dst, const void* src) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
               "@q cp.async.cg.shared.global [%0], [%1], 16;\n\t}"
               ::"r"(dst), "l"(src), "r"((int)p) : "memory");
}
KAPSM_DEV void cpa4_if(bool p, unsigned dst, const void* src) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
               "@q cp.async.ca.shared.global [%0], [%1], 4;\n\t}"
               ::"r"(dst), "l"(src), "r"((int)p) : "memory");
}
template <typename V>
KAPSM_DEV void stg_if(bool p, V* dst, V v);
template <>
KAPSM_DEV void stg_if<float>(bool p, float* dst, float v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f32 [%0], %1;\n\t}"
               ::"l"(dst), "f"(v), "r"((int)p) : "memory");
}
template <>
KAPSM_DEV void stg_if<int>(bool p, int* dst, int v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.s32 [%0], %1;\n\t}"
               ::"l"(dst), "r"(v), "r"((int)p) : "memory");
}

// K[m][m-d] for d = 0..R-1 (0 where m - d < 0): the band of the realified
// pilot Gram that a chain's ring of R slots can meet (R = 32, or 32 NW for
// the wide trainer below).  Realified sample m = 2t + beta is
// r1(x_t) (beta = 0) or r2(x_t) (beta = 1) of pilot x_t (apsm.py:156-182).
// One thread per complex pilot pair (t, t - dt), dt = 0..R/2: one pass over the
// antennas gives c = x^H y (y = x_t, x = x_{t-dt}) and the three distinct
// distances |x - y|, |x + iy|, |x - iy| by explicit differences, hence the
// 2 x 2 realified block: linear parts Re c, Im c, -Im c, Re c and Gaussian
// parts of the matching distances (as screen.cu's list values).
// Tiled: a CTA stages TT pilot rows of a frame plus the R/2 rows before them
// in shared memory with contiguous 16-byte loads (padded rows: the 16-byte
// reads of 8 different rows hit different banks), forms every pair (t, t - dt)
// of the tile from shared memory (one thread per pair), collects the tile's
// 2 TT band rows in shared memory and writes them out as one contiguous block.  Global traffic is the compulsory rows and
// band, with many requests in flight per CTA (a thread-per-pair kernel reading
// rows from global memory waited a DRAM round trip per thread: 2x slower).
__global__ void __launch_bounds__(256)
    band_tile_kernel(const float* __restrict__ rx, long long rx_stride, int n_train, int M,
                     float w_l, float w_g, float inv2s, float* __restrict__ kband, int R, int TT) {
  extern __shared__ __align__(16) float bsm[];
  const int Np = 2 * n_train, D = 2 * M, H = R / 2;
  const int DS = ((D + 3) & ~3) + 4;                      // padded row stride (floats)
  const int f = blockIdx.y, t0 = blockIdx.x * TT;
  const int r0 = max(0, t0 - H), r1 = min(n_train, t0 + TT);   // staged rows [r0, r1)
  float* rows = bsm;                                      // [(TT + H)][DS]
  float* out = bsm + (size_t)(TT + H) * DS;               // [2 TT][R]
  const float* X = rx + (long long)f * rx_stride;
  const bool v16 = (D & 3) == 0 && (rx_stride & 3) == 0 && ((size_t)rx & 15) == 0;
  if (v16) {
    const int q4 = D / 4, n4 = (r1 - r0) * q4;
    const float4* src = reinterpret_cast<const float4*>(X + (long long)r0 * D);
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
      const int r = q4 == 8 ? i / 8 : i / q4, c = i - r * q4;      // (M = 16: a shift)
      *reinterpret_cast<float4*>(rows + r * DS + 4 * c) = __ldg(src + i);
    }
  } else {
    const int n = (r1 - r0) * D;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int r = i / D;
      rows[r * DS + (i - r * D)] = X[(long long)r0 * D + i];
    }
  }
  __syncthreads();
  const int pairs = TT * (H + 1);
  const bool gauss = w_g != 0.f;
  for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
    // (the one-warp ring's R = 32: a division by a constant)
    const int tt = H == 16 ? i / 17 : i / (H + 1), dt = i - tt * (H + 1), t = t0 + tt, tp = t - dt;
    if (t >= n_train) continue;
    float vals[2][2] = {{0.f, 0.f}, {0.f, 0.f}};          // [alpha][beta]
    if (tp >= 0) {
      const float* y = rows + (t - r0) * DS;
      const float* x = rows + (tp - r0) * DS;
      float cr = 0.f, ci = 0.f, ea = 0.f, eb = 0.f, ec = 0.f;
      auto acc = [&](float xr, float xi, float yr, float yi) {
        cr = fmaf(xr, yr, fmaf(xi, yi, cr));
        ci = fmaf(xr, yi, fmaf(-xi, yr, ci));
        float a0 = xr - yr, a1 = xi - yi;
        ea = fmaf(a0, a0, fmaf(a1, a1, ea));
        a0 = xr - yi; a1 = xi + yr;
        eb = fmaf(a0, a0, fmaf(a1, a1, eb));
        a0 = xr + yi; a1 = xi - yr;
        ec = fmaf(a0, a0, fmaf(a1, a1, ec));
      };
      if (D == 32) {                          // 16 antennas: unrolled
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 xv = *reinterpret_cast<const float4*>(x + 4 * q);
          const float4 yv = *reinterpret_cast<const float4*>(y + 4 * q);
          acc(xv.x, xv.y, yv.x, yv.y);
          acc(xv.z, xv.w, yv.z, yv.w);
        }
      } else if ((D & 3) == 0) {
        for (int q = 0; q < D / 4; ++q) {
          const float4 xv = *reinterpret_cast<const float4*>(x + 4 * q);
          const float4 yv = *reinterpret_cast<const float4*>(y + 4 * q);
          acc(xv.x, xv.y, yv.x, yv.y);
          acc(xv.z, xv.w, yv.z, yv.w);
        }
      } else {
        for (int k = 0; k < M; ++k) acc(x[2 * k], x[2 * k + 1], y[2 * k], y[2 * k + 1]);
      }
      const float ka = gauss ? (dt == 0 ? 1.f : exp_fast(-ea * inv2s)) : 0.f;
      const float kbv = gauss ? exp_fast(-eb * inv2s) : 0.f;
      const float kc = gauss ? exp_fast(-ec * inv2s) : 0.f;
      vals[0][0] = vals[1][1] = w_l * cr + w_g * ka;
      vals[0][1] = w_l * ci + w_g * kbv;                  // r1(x) . r2(y) = Im(x^H y)
      vals[1][0] = -w_l * ci + w_g * kc;                  // r2(x) . r1(y) = -Im(x^H y)
    }
    for (int be = 0; be < 2; ++be)
      for (int al = 0; al < 2; ++al) {
        const int d = 2 * dt + be - al;
        if (d >= 0 && d < R) out[(2 * tt + be) * R + d] = vals[al][be];
      }
  }
  __syncthreads();
  // the tile's band rows 2 t0 .. 2 min(t0 + TT, n_train) - 1: one contiguous block
  const int nrow = 2 * (min(t0 + TT, n_train) - t0);
  float* kb = kband + (long long)f * Np * R + (long long)2 * t0 * R;
  const int n4 = nrow * R / 4;                            // R is a multiple of 32
  for (int i = threadIdx.x; i < n4; i += blockDim.x)
    reinterpret_cast<float4*>(kb)[i] = reinterpret_cast<const float4*>(out)[i];
}

KAPSM_DEV float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

KAPSM_DEV float2 ffma2(float2 a, float2 b, float2 c) {     // packed FP32x2 FMA (FFMA2)
  unsigned long long ra, rb, rc;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(rc) : "l"(ra), "l"(rb));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(rc));
  return r;
}

// realified component e of sample (beta) from its interleaved pilot row x
KAPSM_DEV float rcomp(const float* x, int e, int beta) {
  if (!beta) return x[e];
  return (e & 1) ? -x[e - 1] : x[e + 1];
}

template <int DPL, bool VEC>
__global__ void __launch_bounds__(128, 6)
    apsm_train_tp_kernel(const float* __restrict__ rx, long long rx_stride,
                         const float* __restrict__ targets, const float* __restrict__ kband,
                         const unsigned* __restrict__ plive, const int* __restrict__ pcnt,
                         const float4* __restrict__ pvals, int F, int K, int n_train, int M, int W,
                         float eps, float w_l, float w_g, float inv2s,
                         const float* __restrict__ qtab, float* __restrict__ coeff_out,
                         int* __restrict__ fs_out, float* __restrict__ theta_out,
                         int* __restrict__ nact_out, int* __restrict__ status_out) {
  extern __shared__ __align__(128) unsigned char smem_tp[];
  using L = TpL<DPL>;
  const int Np = 2 * n_train, D = 2 * M, P = tp_lead(W);
  const int wpc = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * wpc + warp;
  if (task >= F * K) return;                    // warps are independent: no CTA barrier below
  unsigned char* base = smem_tp + (size_t)warp * L::TOTAL;
  const unsigned sbase = smem_u32(base);
  float* Ks = reinterpret_cast<float*>(base + L::KS);      // [32][TP_KS] K over ring pairs
  float* dsm = reinterpret_cast<float*>(base + L::DSM);    // [32] the step's deltas
  const float* Sg = reinterpret_cast<const float*>(base + L::STG);  // [STG][SSTR] stages
  float* qs = reinterpret_cast<float*>(base + L::QS);      // [W][2] (q_mid, q_last)
  constexpr int XR = L::XR, SSTR = L::SSTR;
  constexpr int OKB = L::OKB, OB = L::OB, OLC = L::OLC;   // stage offsets
  const int f = task / K;
  const float* X = rx + (long long)f * rx_stride;
  const float* Bt = targets + (long long)task * Np;
  const float* KB = kband + (long long)f * Np * 32;
  const int NWp = (n_train + 31) / 32;
  const unsigned* LW = plive + (long long)f * NWp * n_train;
  const int* LC = pcnt + (long long)f * n_train;
  const float4* LV = pvals + (long long)f * n_train * TP_CAP;
  float* Cout = coeff_out + (long long)task * Np;
  int* FSout = fs_out + (long long)task * Np;
  constexpr bool vec = VEC;       // 16-byte rows (host: D % 4 == 0, aligned rows)
  const bool gauss = w_g != 0.f;

  for (int i = lane; i < TP_RING * TP_KS; i += 32) Ks[i] = 0.f;
  for (int i = lane; i < W; i += 32) {
    qs[2 * i] = qtab ? qtab[2 * i] : 1.f / (float)(i + 1);
    qs[2 * i + 1] = qtab ? qtab[2 * i + 1] : 1.f / (float)(i + 1);
  }
  dsm[lane] = 0.f;

  // prefetch pieces into stage m mod STG (one cp.async group per step): the
  // pilot rows of sample m and of the leaving sample m - SPAN + 1 (16-byte
  // pieces, or 4-byte ones when rows are not 16-byte aligned), the band row
  // (8 pieces), the target and the row's live count (the live-list row itself
  // is read from global memory in the rare steps whose count is nonzero).  A
  // lane owns up to 3 pieces for the whole chain; each keeps a running global
  // pointer for its sample mm (m or m - SPAN + 1): g + mm * gm + (mm >> 1) * gt,
  // advanced by gm + (mm odd) gt per step.
  const int XP = vec ? D / 4 : D;               // row pieces (pieces: 2 XP + 10)
  const unsigned sg_s = sbase + L::STG;
  // pieces per lane (compile time): 2 rows of up to 8 DPL 16-byte pieces (or
  // 32 DPL 4-byte ones) + 8 band pieces + target + live count
  constexpr int NRP = VEC ? (16 * DPL + 10 + 31) / 32 : (64 * DPL + 10 + 31) / 32;
  const char* pp[NRP];
  long long pgm[NRP], pgt[NRP];
  unsigned ps[NRP];
  int psz[NRP], poff[NRP];       // poff: the piece's sample is m - poff
#pragma unroll
  for (int r = 0; r < NRP; ++r) {
    int pc = lane + 32 * r;
    const char* g = nullptr;
    pgm[r] = 0; pgt[r] = 0; ps[r] = sg_s; psz[r] = 0; poff[r] = 0;
    if (pc < 2 * XP) {
      const int lv = pc >= XP;
      if (lv) pc -= XP;
      g = reinterpret_cast<const char*>(X + (vec ? 4 * pc : pc));
      pgt[r] = (long long)D * 4;
      ps[r] = sg_s + (unsigned)(lv * XR + (vec ? 4 * pc : pc)) * 4;
      psz[r] = vec ? 16 : 4;
      poff[r] = lv ? TP_SPAN - 1 : 0;
    } else if (pc < 2 * XP + 8) {
      const int q = pc - 2 * XP;
      g = reinterpret_cast<const char*>(KB + 4 * q);
      pgm[r] = 128;
      ps[r] = sg_s + (unsigned)(OKB + 4 * q) * 4;
      psz[r] = 16;
    } else if (pc == 2 * XP + 8) {
      g = reinterpret_cast<const char*>(Bt);
      pgm[r] = 4;
      ps[r] = sg_s + (unsigned)OB * 4;
      psz[r] = 4;
    } else if (pc == 2 * XP + 9) {
      g = reinterpret_cast<const char*>(LC);
      pgt[r] = 4;
      ps[r] = sg_s + (unsigned)OLC * 4;
      psz[r] = gauss ? 4 : 0;
    }
    // pointer for the piece of prefetch(0): sample -poff (may be negative: never issued)
    const long long mm0 = -poff[r];
    pp[r] = g ? g + mm0 * pgm[r] + (mm0 >> 1) * pgt[r] : nullptr;
  }
  int pm = 0;                    // the sample index m of the next prefetch
  auto prefetch = [&]() {        // stage of sample pm (steps are prefetched in order)
    const unsigned so = (unsigned)((pm & (TP_STG - 1)) * SSTR) * 4;
#pragma unroll
    for (int r = 0; r < NRP; ++r) {
      const int mm = pm - poff[r];
      const bool go = (unsigned)mm < (unsigned)Np;
      cpa16_if(go && psz[r] == 16, ps[r] + so, pp[r]);
      cpa4_if(go && psz[r] == 4, ps[r] + so, pp[r]);
      pp[r] += pgm[r] + ((mm & 1) ? pgt[r] : 0);            // -> sample mm + 1
    }
    ++pm;
  };
  for (int i = 0; i < TP_AHEAD; ++i) {
    prefetch();
    cp_async_commit();
  }

  int samp = -(1 << 30);          // sample held by this lane's slot
  float Y = 0.f, c = 0.f, idn = 0.f, bl = 0.f, bh = 0.f;
  int fs = -1, nact = 0, status = 0;
  // theta_fin as (Re, Im) pairs: lane k (+ 32 i) holds antenna k, i.e.
  // components k and M + k of the reference's block layout [Re; Im]
  constexpr int KPL = (DPL + 1) / 2;
  float2 th[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) th[i] = make_float2(0.f, 0.f);
  const unsigned krow = sbase + L::KS + (unsigned)(lane * TP_KS) * 4;   // K[.][my sample]
  const unsigned dsa = sbase + L::DSM;
  const float qmc = qs[2 * (W - 1)], qlc = qs[2 * (W - 1) + 1];

  // one step; MAIN: n >= W - 1 and m = n + P < Np (every part present, q
  // constant), compile-time so the steady state is straight-line code
  auto step = [&](const int n, auto main_) {
    constexpr bool MAIN = decltype(main_)::value;
    const int m = n + P;                        // taken over this step
    cp_async_wait<TP_AHEAD - 1>();              // m's stage (issued TP_AHEAD steps ago) landed
    __syncwarp();
    // ---- live Gaussian terms of sample ml = m - 2: older samples, final c ----
    const int ml = m - TP_LIVE_LAG;
    if (gauss && (MAIN || (ml >= 0 && ml < Np))) {
      const float* sl = Sg + (ml & (TP_STG - 1)) * SSTR;
      const int cnt = __float_as_int(sl[OLC]);
      if (cnt != 0) {
        const int bt = ml & 1;
        float part = 0.f;
        if (cnt > 0) {                          // the list row (rare: from global)
          if (lane < 2 * cnt) {
            const float4 v4 = __ldg(LV + (long long)(ml >> 1) * TP_CAP + (lane >> 1));
            const int al = lane & 1, a = 2 * __float_as_int(v4.w) + al;
            if (a <= ml - TP_SPAN) {
              const float kap = al == 0 ? (bt == 0 ? v4.x : v4.y) : (bt == 0 ? v4.z : v4.x);
              part = w_g * __ldcg(Cout + a) * kap;
            }
          }
        } else {                                // more live pilots than the list holds
          const int tl = ml >> 1;
          const float* xm = X + (long long)tl * D;
          for (int w = lane; w < NWp; w += 32) {
            unsigned bits = LW[(long long)w * n_train + tl];
            while (bits) {
              const int p = w * 32 + __ffs(bits) - 1;
              bits &= bits - 1;
              const float* xa = X + (long long)p * D;
              for (int al = 0; al < 2; ++al) {
                const int a = 2 * p + al;
                if (a > ml - TP_SPAN) continue;
                float dist = 0.f;
                for (int e = 0; e < D; ++e) {
                  const float z = rcomp(xa, e, al) - rcomp(xm, e, bt);
                  dist = fmaf(z, z, dist);
                }
                part = fmaf(w_g * __ldcg(Cout + a), exp_fast(-dist * inv2s), part);
              }
            }
          }
        }
        part = warp_sum_f(part);
        if (lane == (ml & 31)) Y += part;
      }
    }
    // ---- takeover of sample m into slot sm ----
    const float* sg = Sg + (m & (TP_STG - 1)) * SSTR;     // this step's stage
    if (MAIN || m < Np) {
      const int sm = m & 31, bt = m & 1;
      const float v = sg[OKB + ((sm - lane) & 31)];        // K[m][this lane's sample]
      Ks[sm * TP_KS + lane] = v;                           // K is symmetric: row and column
      Ks[lane * TP_KS + sm] = v;
      float pf = 0.f;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int k = lane + 32 * i;
        if (k < M) {                            // r1 = [Re; Im], r2 = [Im; -Re] (apsm.py:156-169)
          const float2 x = *reinterpret_cast<const float2*>(sg + 2 * k);
          pf = fmaf(th[i].x, bt ? x.y : x.x, pf);
          pf = fmaf(th[i].y, bt ? -x.x : x.y, pf);
        }
      }
      pf *= w_l;
      const bool win = (unsigned)(samp - (n - W + 1)) < (unsigned)(W - 1);   // samp in [n-W+1, n-1]
      pf = fmaf(win ? c : 0.f, v, pf);
      const float init = warp_sum_f(pf);
      const float b = sg[OB];
      const bool mine = lane == sm;             // this lane's slot takes sample m
      samp = mine ? m : samp;
      Y = mine ? init : Y;
      c = mine ? 0.f : c;
      fs = mine ? -1 : fs;
      status |= (mine && !(v > 0.f)) ? (int)KAPSM_TRAIN_DEGENERATE : 0;   // kappa(r, r) = K[m][m]
      float rv;                                 // MUFU on every lane (tolerance 1e-4), no branch
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rv) : "f"(v));
      idn = mine ? (v > 0.f ? rv : 0.f) : idn;
      bl = mine ? b - eps : bl;
      bh = mine ? b + eps : bh;
    }
    __syncwarp();                               // stage reads done before it is refilled
    prefetch();                                 // sample m + TP_AHEAD
    cp_async_commit();
    if (!MAIN && n < 0) return;
    // ---- step n: the window's deltas, then the window update ----
    const int lo = MAIN ? n - W + 1 : (n - W + 1 > 0 ? n - W + 1 : 0);
    const int cj = MAIN ? W - 1 : n - lo;
    float qm = qmc, ql = qlc;
    if (!MAIN) {
      qm = qs[2 * cj];
      ql = qs[2 * cj + 1];
    }
    const float q = samp == n ? ql : qm;
    const bool inw = (unsigned)(samp - lo) <= (unsigned)cj;              // samp in [lo, n]
    float dl = q * idn * (fmaxf(bl - Y, 0.f) + fminf(bh - Y, 0.f));
    dl = inw ? dl : 0.f;
    c += dl;
    fs = (dl != 0.f && fs < 0) ? n : fs;
    dsm[lane] = dl;
    __syncwarp();                               // deltas and the takeover's K row/column
    float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
    for (int s = 0; s < 32; s += 8) {
      const float4 d0 = lds_f4(dsa + 4u * s), k0 = lds_f4(krow + 4u * s);
      const float4 d1 = lds_f4(dsa + 4u * (s + 4)), k1 = lds_f4(krow + 4u * (s + 4));
      a0 = ffma2(make_float2(d0.x, d0.y), make_float2(k0.x, k0.y), a0);
      a1 = ffma2(make_float2(d0.z, d0.w), make_float2(k0.z, k0.w), a1);
      a2 = ffma2(make_float2(d1.x, d1.y), make_float2(k1.x, k1.y), a2);
      a3 = ffma2(make_float2(d1.z, d1.w), make_float2(k1.z, k1.w), a3);
    }
    Y += ((a0.x + a0.y) + (a1.x + a1.y)) + ((a2.x + a2.y) + (a3.x + a3.y));
    // ---- the sample leaving after this step: its coefficient is final ----
    const int a = n - W + 1;                    // == m - TP_SPAN + 1: its row is in the stage
    if (MAIN || a >= 0) {
      const float ca = __shfl_sync(0xffffffffu, c, a & 31);
      const bool odd = a & 1;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int k = lane + 32 * i;
        if (k < M) {
          const float2 x = *reinterpret_cast<const float2*>(sg + XR + 2 * k);
          th[i].x = fmaf(ca, odd ? x.y : x.x, th[i].x);
          th[i].y = fmaf(ca, odd ? -x.x : x.y, th[i].y);
        }
      }
      const bool own = lane == (a & 31);
      stg_if(own, Cout + a, c);
      stg_if(own, FSout + a, fs);
      nact += (own && fs >= 0) ? 1 : 0;
    }
  };
  using T_ = std::true_type;
  using F_ = std::false_type;
  int n = -P;
  for (; n < W - 1 && n < Np; ++n) step(n, F_{});
  for (; n + P < Np; ++n) step(n, T_{});
  for (; n < Np; ++n) step(n, F_{});
  cp_async_wait<0>();
  __syncwarp();
  // ---- samples still in the window after the last step (rows from global) ----
  for (int a = (Np - W + 1 > 0 ? Np - W + 1 : 0); a < Np; ++a) {
    const float ca = __shfl_sync(0xffffffffu, c, a & 31);
    const float* xa = X + (long long)(a >> 1) * D;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int k = lane + 32 * i;
      if (k < M) {
        const float xr = xa[2 * k], xi = xa[2 * k + 1];
        th[i].x = fmaf(ca, (a & 1) ? xi : xr, th[i].x);
        th[i].y = fmaf(ca, (a & 1) ? -xr : xi, th[i].y);
      }
    }
    if (lane == (a & 31)) {
      Cout[a] = c;
      FSout[a] = fs;
      nact += fs >= 0;
    }
  }
  // theta = w_l theta_fin in the reference's block layout [Re; Im] (apsm.py:172-182)
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int k = lane + 32 * i;
    if (k < M) {
      theta_out[(long long)task * D + k] = w_l * th[i].x;
      theta_out[(long long)task * D + M + k] = w_l * th[i].y;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    nact += __shfl_xor_sync(0xffffffffu, nact, o);
    status |= __shfl_xor_sync(0xffffffffu, status, o);
  }
  if (lane == 0) {
    nact_out[task] = nact;
    status_out[task] = status;
  }
}

// ---------------------------------------------------------------------------
// K2w: the same restatement for windows beyond the one-warp ring (W > 21, the
// C3 sweep): one CTA of NW warps per chain, thread j owns ring slot j of
// R = 32 NW slots (P = R - 4 - W).  Per step, one CTA barrier:
//   phase A  live terms of sample m - 2 (its owner warp), takeover of sample m
//            (every thread writes its entry of K's new row / column; the owner
//            warp forms f(r_m) from its theta replica, the previous step's
//            coefficients and the band row), the prefetch of sample m + 6, and
//            each slot's delta -> dsm[n & 1], coefficient -> csm[n & 1];
//   barrier  (publishes K, deltas, coefficients and the next stage);
//   phase B  Y_j += sum over the window's slots s of delta_s K[s][j] (16-byte
//            rows of K, packed FP32x2 FMAs), then the leaving sample's
//            coefficient is final: every warp adds c_a r_a to its theta replica.
// Double-buffered deltas / coefficients make the one barrier sufficient.  The
// step is bound by the shared-memory reads of the window update:
// W x (W + P) x 4 bytes per step (128 B/clk per SM).
constexpr int TPW_STG = 16;              // stages: read up to 2 steps back, 6 ahead
constexpr int TPW_MAX_NW = 5;            // W <= 32 NW - 4 - TP_AHEAD - 1 = 149

template <int DPL, int NW>
struct TpwL {
  static constexpr int R = 32 * NW, KS = R + 4, XR = 32 * DPL;
  static constexpr int SSTR = 2 * XR + R + 36;              // floats per stage
  static constexpr int OKB = 2 * XR, OLV = OKB + R, OB = OLV + 32, OLC = OB + 1;
  static constexpr int KSO = 0;                             // [R][KS] K over ring pairs
  static constexpr int DSM = KSO + R * KS * 4;              // [2][R] deltas
  static constexpr int CSM = DSM + 2 * R * 4;               // [2][R] coefficients
  static constexpr int QS = CSM + 2 * R * 4;                // [R][2] (q_mid, q_last)
  static constexpr int RED = QS + 2 * R * 4;                // nact, status
  static constexpr int STG = RED + 16;                      // [TPW_STG][SSTR] stages
  static constexpr int TOTAL = (STG + TPW_STG * SSTR * 4 + 127) & ~127;
};
__host__ __device__ constexpr int tpw_nw(int W) {          // smallest ring with P > TP_AHEAD
  return (W + 4 + TP_AHEAD + 1 + 31) / 32 < 2 ? 2 : (W + 4 + TP_AHEAD + 1 + 31) / 32;
}
template <int NW>
__host__ __device__ constexpr int tpw_total(int M) {
  return tp_dpl(M) == 1 ? TpwL<1, NW>::TOTAL
                        : tp_dpl(M) == 2 ? TpwL<2, NW>::TOTAL : TpwL<4, NW>::TOTAL;
}
static int tpw_total_rt(int NW, int M) {
  switch (NW) {
    case 2: return tpw_total<2>(M);
    case 3: return tpw_total<3>(M);
    case 4: return tpw_total<4>(M);
    default: return tpw_total<5>(M);
  }
}


template <int DPL, int NW>
__global__ void __launch_bounds__(32 * NW, 1)
    apsm_train_tpw_kernel(const float* __restrict__ rx, long long rx_stride,
                          const float* __restrict__ targets, const float* __restrict__ kband,
                          const unsigned* __restrict__ plive, const int* __restrict__ pcnt,
                          const float4* __restrict__ pvals, int F, int K, int n_train, int M,
                          int W, float eps, float w_l, float w_g, float inv2s,
                          const float* __restrict__ qtab, float* __restrict__ coeff_out,
                          int* __restrict__ fs_out, float* __restrict__ theta_out,
                          int* __restrict__ nact_out, int* __restrict__ status_out) {
  extern __shared__ __align__(128) unsigned char smem_tp[];
  using L = TpwL<DPL, NW>;
  constexpr int R = L::R, KS = L::KS, NT = 32 * NW, XR = L::XR, SSTR = L::SSTR;
  constexpr int OKB = L::OKB, OLV = L::OLV, OB = L::OB, OLC = L::OLC;
  constexpr int SPAN = R - 4;
  const int Np = 2 * n_train, D = 2 * M, P = SPAN - W;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, j = tid;   // j: my slot
  const int task = blockIdx.x;
  if (task >= F * K) return;
  float* Ks = reinterpret_cast<float*>(smem_tp + L::KSO);
  float* dsm = reinterpret_cast<float*>(smem_tp + L::DSM);
  float* csm = reinterpret_cast<float*>(smem_tp + L::CSM);
  float* qs = reinterpret_cast<float*>(smem_tp + L::QS);
  int* red = reinterpret_cast<int*>(smem_tp + L::RED);
  const float* Sg = reinterpret_cast<const float*>(smem_tp + L::STG);
  const int f = task / K;
  const float* X = rx + (long long)f * rx_stride;
  const float* Bt = targets + (long long)task * Np;
  const float* KB = kband + (long long)f * Np * R;
  const int NWp = (n_train + 31) / 32;
  const unsigned* LW = plive + (long long)f * NWp * n_train;
  const int* LC = pcnt + (long long)f * n_train;
  const float4* LV = pvals + (long long)f * n_train * TP_CAP;
  float* Cout = coeff_out + (long long)task * Np;
  int* FSout = fs_out + (long long)task * Np;
  const bool vec = (D % 4) == 0 && (rx_stride % 4) == 0 && ((size_t)rx & 15) == 0;
  const bool gauss = w_g != 0.f;

  for (int i = tid; i < R * KS; i += NT) Ks[i] = 0.f;
  for (int i = tid; i < 2 * R; i += NT) dsm[i] = csm[i] = 0.f;
  for (int i = tid; i < W; i += NT) {
    qs[2 * i] = qtab ? qtab[2 * i] : 1.f / (float)(i + 1);
    qs[2 * i + 1] = qtab ? qtab[2 * i + 1] : 1.f / (float)(i + 1);
  }
  if (tid == 0) red[0] = red[1] = 0;

  // prefetch pieces of step m's stage, spread over the CTA:
  // pilot rows of m and of the leaving sample m - SPAN + 1, the band row (R/4
  // pieces), the live-list row (8), the target, the live count
  const int XP = vec ? D / 4 : D, NPC = 2 * XP + R / 4 + 10;
  const unsigned sg_s = smem_u32(smem_tp) + L::STG;
  // rounds of pieces per thread: enough for 4-byte pieces of the widest row
  constexpr int PRW = (2 * 32 * DPL + R / 4 + 10 + NT - 1) / NT;
  const char* pp[PRW];
  long long pgm[PRW], pgt[PRW];
  unsigned ps[PRW];
  int psz[PRW], poff[PRW];
#pragma unroll
  for (int r = 0; r < PRW; ++r) {
    int pc = tid + NT * r;
    const char* g = nullptr;
    pgm[r] = 0; pgt[r] = 0; ps[r] = sg_s; psz[r] = 0; poff[r] = 0;
    if (pc < 2 * XP) {
      const int lv = pc >= XP;
      if (lv) pc -= XP;
      g = reinterpret_cast<const char*>(X + (vec ? 4 * pc : pc));
      pgt[r] = (long long)D * 4;
      ps[r] = sg_s + (unsigned)(lv * XR + (vec ? 4 * pc : pc)) * 4;
      psz[r] = vec ? 16 : 4;
      poff[r] = lv ? SPAN - 1 : 0;
    } else if (pc < 2 * XP + R / 4) {
      const int q = pc - 2 * XP;
      g = reinterpret_cast<const char*>(KB + 4 * q);
      pgm[r] = (long long)R * 4;
      ps[r] = sg_s + (unsigned)(OKB + 4 * q) * 4;
      psz[r] = 16;
    } else if (pc < 2 * XP + R / 4 + 8) {
      const int q = pc - 2 * XP - R / 4;
      g = reinterpret_cast<const char*>(LV + q);
      pgt[r] = (long long)TP_CAP * 16;
      ps[r] = sg_s + (unsigned)(OLV + 4 * q) * 4;
      psz[r] = gauss ? 16 : 0;
    } else if (pc == 2 * XP + R / 4 + 8) {
      g = reinterpret_cast<const char*>(Bt);
      pgm[r] = 4;
      ps[r] = sg_s + (unsigned)OB * 4;
      psz[r] = 4;
    } else if (pc == 2 * XP + R / 4 + 9) {
      g = reinterpret_cast<const char*>(LC);
      pgt[r] = 4;
      ps[r] = sg_s + (unsigned)OLC * 4;
      psz[r] = gauss ? 4 : 0;
    }
    const long long mm0 = -poff[r];
    pp[r] = g ? g + mm0 * pgm[r] + (mm0 >> 1) * pgt[r] : nullptr;
  }
  const int nr = (NPC + NT - 1) / NT;
  int pm = 0;
  auto prefetch = [&]() {
    const unsigned so = (unsigned)((pm & (TPW_STG - 1)) * SSTR) * 4;
#pragma unroll
    for (int r = 0; r < PRW; ++r) {
      if (r < nr) {
        const int mm = pm - poff[r];
        const bool go = (unsigned)mm < (unsigned)Np;
        cpa16_if(go && psz[r] == 16, ps[r] + so, pp[r]);
        cpa4_if(go && psz[r] == 4, ps[r] + so, pp[r]);
        pp[r] += pgm[r] + ((mm & 1) ? pgt[r] : 0);
      }
    }
    ++pm;
  };
  for (int i = 0; i < TP_AHEAD; ++i) {
    prefetch();
    cp_async_commit();
  }
  cp_async_wait<TP_AHEAD - 1>();
  __syncthreads();

  float Y = 0.f, c = 0.f, idn = 0.f, bl = 0.f, bh = 0.f;
  int samp = -(1 << 30), fs = -1, nact = 0, status = 0;
  float th[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) th[i] = 0.f;
  int sm = 0;                                   // slot of m = (n + P) mod R
  const unsigned krow = smem_u32(Ks) + (unsigned)(j * KS) * 4;   // K[.][my sample]

  for (int n = -P; n < Np; ++n) {
    const int m = n + P;
    // ---- phase A: live Gaussian terms of sample ml = m - 2 (final, older c) ----
    const int ml = m - TP_LIVE_LAG;
    int sml = sm - TP_LIVE_LAG;
    sml += sml < 0 ? R : 0;
    if (gauss && ml >= 0 && ml < Np && warp == (sml >> 5)) {
      const float* sl = Sg + (ml & (TPW_STG - 1)) * SSTR;
      const int cnt = __float_as_int(sl[OLC]);
      const int bt = ml & 1;
      float part = 0.f;
      if (cnt > 0) {
        if (lane < 2 * cnt) {
          const float4 v4 = reinterpret_cast<const float4*>(sl + OLV)[lane >> 1];
          const int al = lane & 1, a = 2 * __float_as_int(v4.w) + al;
          if (a <= ml - SPAN) {
            const float kap = al == 0 ? (bt == 0 ? v4.x : v4.y) : (bt == 0 ? v4.z : v4.x);
            part = w_g * __ldcg(Cout + a) * kap;
          }
        }
      } else if (cnt < 0) {                     // more live pilots than the list holds
        const int tl = ml >> 1;
        const float* xm = X + (long long)tl * D;
        for (int w = lane; w < NWp; w += 32) {
          unsigned bits = LW[(long long)w * n_train + tl];
          while (bits) {
            const int p = w * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            const float* xa = X + (long long)p * D;
            for (int al = 0; al < 2; ++al) {
              const int a = 2 * p + al;
              if (a > ml - SPAN) continue;
              float dist = 0.f;
              for (int e = 0; e < D; ++e) {
                const float z = rcomp(xa, e, al) - rcomp(xm, e, bt);
                dist = fmaf(z, z, dist);
              }
              part = fmaf(w_g * __ldcg(Cout + a), exp_fast(-dist * inv2s), part);
            }
          }
        }
      }
      if (__any_sync(0xffffffffu, part != 0.f)) {
        part = warp_sum_f(part);
        if (j == sml) Y += part;
      }
    }
    // ---- takeover of sample m into slot sm ----
    const float* sg = Sg + (m & (TPW_STG - 1)) * SSTR;
    if (m < Np) {
      int d = sm - j;                           // m - (the sample in my slot)
      d += d < 0 ? R : 0;
      const float v = sg[OKB + d];
      Ks[sm * KS + j] = v;                      // K is symmetric: row and column
      Ks[j * KS + sm] = v;
      if (warp == (sm >> 5)) {                  // the owner warp forms f_n(r_m)
        const int bt = m & 1;
        float pf = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          const int e = lane + 32 * i;
          if (e < D) {
            const float x0 = sg[e], x1 = sg[e ^ 1];
            pf = fmaf(th[i], bt ? ((e & 1) ? -x1 : x1) : x0, pf);
          }
        }
        pf *= w_l;
        const float* cprev = csm + ((n - 1) & 1) * R;
        for (int dd = P + 1 + lane; dd < P + W; dd += 32) {   // the window [n-W+1, n-1]
          int s = sm - dd;
          s += s < 0 ? R : 0;
          pf = fmaf(cprev[s], sg[OKB + dd], pf);
        }
        const float init = warp_sum_f(pf);
        if (j == sm) {
          const float kd = sg[OKB], b = sg[OB];
          samp = m;
          Y = init;
          c = 0.f;
          fs = -1;
          status |= !(kd > 0.f) ? (int)KAPSM_TRAIN_DEGENERATE : 0;   // kappa(r, r)
          idn = kd > 0.f ? __fdividef(1.f, kd) : 0.f;
          bl = b - eps;
          bh = b + eps;
        }
      }
    }
    prefetch();                                 // sample m + TP_AHEAD
    cp_async_commit();
    const int lo = n - W + 1 > 0 ? n - W + 1 : 0, cj = n - lo;
    if (n >= 0) {                               // ---- step n: my slot's delta ----
      const float qm = qs[2 * cj], ql = qs[2 * cj + 1];
      const float q = samp == n ? ql : qm;
      const bool inw = (unsigned)(samp - lo) <= (unsigned)cj;
      float dl = q * idn * (fmaxf(bl - Y, 0.f) + fminf(bh - Y, 0.f));
      dl = inw ? dl : 0.f;
      c += dl;
      fs = (dl != 0.f && fs < 0) ? n : fs;
      dsm[(n & 1) * R + j] = dl;
      csm[(n & 1) * R + j] = c;
    }
    cp_async_wait<TP_AHEAD - 1>();              // my pieces of sample m + 1 landed
    __syncthreads();
    if (n >= 0) {
      // ---- phase B: Y_j += sum over the window's slots of delta_s K[s][j] ----
      int sn = sm - P;
      sn += sn < 0 ? R : 0;                     // slot of n
      int slo = sn - cj;
      slo += slo < 0 ? R : 0;                   // slot of lo
      const int c0 = slo >> 2, nch = (n >> 2) - (lo >> 2) + 1;
      const int e1 = c0 + nch < R / 4 ? c0 + nch : R / 4;
      const float4* dd4 = reinterpret_cast<const float4*>(dsm + (n & 1) * R);
      const float4* kk4 = reinterpret_cast<const float4*>(Ks + j * KS);
      float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
      int k = c0;
#pragma unroll 2
      for (; k + 1 < e1; k += 2) {
        const float4 d0 = dd4[k], k0 = kk4[k], d1 = dd4[k + 1], k1 = kk4[k + 1];
        a0 = ffma2(make_float2(d0.x, d0.y), make_float2(k0.x, k0.y), a0);
        a1 = ffma2(make_float2(d0.z, d0.w), make_float2(k0.z, k0.w), a1);
        a2 = ffma2(make_float2(d1.x, d1.y), make_float2(k1.x, k1.y), a2);
        a3 = ffma2(make_float2(d1.z, d1.w), make_float2(k1.z, k1.w), a3);
      }
      if (k < e1) {
        const float4 d0 = dd4[k], k0 = kk4[k];
        a0 = ffma2(make_float2(d0.x, d0.y), make_float2(k0.x, k0.y), a0);
        a1 = ffma2(make_float2(d0.z, d0.w), make_float2(k0.z, k0.w), a1);
      }
      const int rest = nch - (e1 - c0);         // wrapped part: chunks 0 .. rest-1
      k = 0;
#pragma unroll 2
      for (; k + 1 < rest; k += 2) {
        const float4 d0 = dd4[k], k0 = kk4[k], d1 = dd4[k + 1], k1 = kk4[k + 1];
        a0 = ffma2(make_float2(d0.x, d0.y), make_float2(k0.x, k0.y), a0);
        a1 = ffma2(make_float2(d0.z, d0.w), make_float2(k0.z, k0.w), a1);
        a2 = ffma2(make_float2(d1.x, d1.y), make_float2(k1.x, k1.y), a2);
        a3 = ffma2(make_float2(d1.z, d1.w), make_float2(k1.z, k1.w), a3);
      }
      if (k < rest) {
        const float4 d0 = dd4[k], k0 = kk4[k];
        a0 = ffma2(make_float2(d0.x, d0.y), make_float2(k0.x, k0.y), a0);
        a1 = ffma2(make_float2(d0.z, d0.w), make_float2(k0.z, k0.w), a1);
      }
      Y += ((a0.x + a0.y) + (a1.x + a1.y)) + ((a2.x + a2.y) + (a3.x + a3.y));
      // ---- the sample leaving after this step: its coefficient is final ----
      const int a = n - W + 1;                  // == m - SPAN + 1: its row is in the stage
      if (a >= 0) {
        int sa = sm - (SPAN - 1);
        sa += sa < 0 ? R : 0;
        const float ca = csm[(n & 1) * R + sa];
        const int ba = a & 1;
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          const int e = lane + 32 * i;
          if (e < D) {
            const float x0 = sg[XR + e], x1 = sg[XR + (e ^ 1)];
            th[i] = fmaf(ca, ba ? ((e & 1) ? -x1 : x1) : x0, th[i]);
          }
        }
        if (j == sa) {
          Cout[a] = c;
          FSout[a] = fs;
          nact += fs >= 0;
        }
      }
    }
    sm = sm + 1 == R ? 0 : sm + 1;
  }
  cp_async_wait<0>();
  // ---- samples still in the window after the last step ----
  const int a0 = Np - W + 1 > 0 ? Np - W + 1 : 0;
  if (samp >= a0 && samp < Np) {
    Cout[samp] = c;
    FSout[samp] = fs;
    nact += fs >= 0;
  }
  atomicAdd(&red[0], nact);
  atomicOr(&red[1], status);
  __syncthreads();
  if (warp == 0) {
    const float* cl = csm + ((Np - 1) & 1) * R;
    for (int a = a0; a < Np; ++a) {
      const float ca = cl[a % R];
      const float* xa = X + (long long)(a >> 1) * D;
#pragma unroll
      for (int i = 0; i < DPL; ++i) {
        const int e = lane + 32 * i;
        if (e < D) th[i] = fmaf(ca, rcomp(xa, e, a & 1), th[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int e = lane + 32 * i;
      if (e < D)
        theta_out[(long long)task * D + ((e & 1) ? M + (e >> 1) : (e >> 1))] = w_l * th[i];
    }
    if (lane == 0) {
      nact_out[task] = red[0];
      status_out[task] = red[1];
    }
  }
}

// ---------------------------------------------------------------------------
// K2l: the band trainer for latency mode (a chain per SM): the same restated
// recurrence as K2t / K2w, with the work that does not feed the next step
// moved off the ring warps.
//   * ring warps (NW of them; thread j owns ring slot j of R = 32 NW; takeover
//     lead P = 28 - W for NW = 1, else 7).  Per step: the delta of its slot, one barrier among the ring
//     warps (a __syncwarp for NW = 1), the window update of every slot's
//     response (K over ring pairs in shared memory), the takeover of sample
//     m = n + P (K's new row/column from the band row, and c_j K[j][m] of the
//     window's current coefficients -> the p ring), the init of the sample
//     entering at step n + 1 added to its response, and the leaving sample's
//     final coefficient -> the cfin ring (shared) and the outputs;
//   * TPL_NH helper warps (sample m handled by helper m mod TPL_NH) prefetch
//     every stage (pilot row of m and of the sample leaving at m's takeover,
//     band row, live list, target) with cp.async 21 samples ahead, publish it
//     by tag 14 samples ahead of their own work, keep a replica of theta_fin
//     (final coefficients of the samples that left the window, times their
//     rows), and form sample m's init
//         w_l theta_fin . r_m + sum_j p[m][j] + w_g sum_live c_a kappa(r_a, r_m)
//     once m is taken over (an mbarrier the ring warps arrive on: the helpers
//     sleep in hardware instead of polling shared memory), published as a
//     tagged value, added by the ring warps one step before m enters the
//     window (P - 1 steps of slack).
// A slot's response restarts at 0 at the takeover and gathers the window
// updates from there, so the init only has to arrive before step m.
constexpr int TPL_STG = 64;              // stages (samples) in flight
constexpr int TPL_NH = 7;                // helper warps
constexpr int TPL_J = 3;                 // prefetch depth per helper (TPL_NH x TPL_J samples);
                                         // stages published 2 own samples ahead
constexpr int TPL_CFR = 256;             // ring of final coefficients (theta catch-up)

template <int KPL, int NW>
struct TplL {
  static constexpr int R = 32 * NW, KS = NW == 1 ? TP_KS : R + 4;
  static constexpr int XR = 64 * KPL;                       // pilot row (2M <= 64 KPL floats)
  static constexpr int SSTR = 2 * XR + R + 36;              // 2 rows, band R, live list 32, B, LC
  static constexpr int OLR = XR, OKB = 2 * XR, OLV = OKB + R, OB = OLV + 32, OLC = OB + 1;
  static constexpr int KSO = 0;                             // [R][KS] K over ring pairs
  static constexpr int DSM = KSO + R * KS * 4;              // [2][R] deltas (by step parity)
  static constexpr int QS = DSM + 2 * R * 4;                // [R][2] (q_mid, q_last)
  static constexpr int INIT = QS + 2 * R * 4;               // [32] tagged inits
  static constexpr int PR = INIT + 32 * 8;                  // [32][R] c_j K[j][m]
  static constexpr int CFR = PR + 32 * R * 4;               // [TPL_CFR] final coefficients
  static constexpr int STAG = CFR + TPL_CFR * 4;            // [TPL_STG] stage tags
  static constexpr int RED = STAG + TPL_STG * 4;            // nact, status
  static constexpr int TKB = RED + 16;                      // [32] mbarriers: m taken over
  static constexpr int STG = TKB + 32 * 8;                  // [TPL_STG][SSTR] stages
  static constexpr int TOTAL = STG + TPL_STG * SSTR * 4;
};
__host__ __device__ constexpr int tpl_kpl(int M) { return (M + 31) / 32; }
__host__ __device__ constexpr int tpl_span(int NW, int W) { return NW == 1 ? TP_SPAN : W + 7; }
template <int NW>
static size_t tpl_bytes(int M) {
  return tpl_kpl(M) == 1 ? (size_t)TplL<1, NW>::TOTAL : (size_t)TplL<2, NW>::TOTAL;
}

template <int KPL, int NW>
__global__ void __launch_bounds__(32 * (NW + TPL_NH), 1)
    apsm_train_tpl_kernel(const float* __restrict__ rx, long long rx_stride,
                          const float* __restrict__ targets, const float* __restrict__ kband,
                          const unsigned* __restrict__ plive, const int* __restrict__ pcnt,
                          const float4* __restrict__ pvals, int F, int K, int n_train, int M,
                          int W, float eps, float w_l, float w_g, float inv2s,
                          const float* __restrict__ qtab, float* __restrict__ coeff_out,
                          int* __restrict__ fs_out, float* __restrict__ theta_out,
                          int* __restrict__ nact_out, int* __restrict__ status_out) {
  extern __shared__ __align__(128) unsigned char smem_tp[];
  using L = TplL<KPL, NW>;
  constexpr int R = L::R, KS = L::KS, XR = L::XR, SSTR = L::SSTR;
  constexpr int OLR = L::OLR, OKB = L::OKB, OLV = L::OLV, OB = L::OB, OLC = L::OLC;
  constexpr int NT = 32 * (NW + TPL_NH);
  // takeover lead P: the one-warp ring keeps K2t's P = 28 - W; wider rings
  // take over 7 steps ahead (P < 32: the init / p / mbarrier rings are 32 deep)
  const int SPAN = tpl_span(NW, W);
  const int Np = 2 * n_train, D = 2 * M, P = SPAN - W;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x;
  if (task >= F * K) return;
  const unsigned sb = smem_u32(smem_tp);
  float* Ks = reinterpret_cast<float*>(smem_tp + L::KSO);
  float* dsm = reinterpret_cast<float*>(smem_tp + L::DSM);
  float* qs = reinterpret_cast<float*>(smem_tp + L::QS);
  float* prg = reinterpret_cast<float*>(smem_tp + L::PR);
  float* cfr = reinterpret_cast<float*>(smem_tp + L::CFR);
  int* stag = reinterpret_cast<int*>(smem_tp + L::STAG);
  int* red = reinterpret_cast<int*>(smem_tp + L::RED);
  const float* Sg = reinterpret_cast<const float*>(smem_tp + L::STG);
  const unsigned s_init = sb + L::INIT, s_tkb = sb + L::TKB;
  const int f = task / K;
  const float* X = rx + (long long)f * rx_stride;
  const float* Bt = targets + (long long)task * Np;
  const float* KB = kband + (long long)f * Np * R;
  const int NWp = (n_train + 31) / 32;
  const unsigned* LW = plive + (long long)f * NWp * n_train;
  const int* LC = pcnt + (long long)f * n_train;
  const float4* LV = pvals + (long long)f * n_train * TP_CAP;
  float* Cout = coeff_out + (long long)task * Np;
  int* FSout = fs_out + (long long)task * Np;
  const bool gauss = w_g != 0.f;

  for (int i = threadIdx.x; i < R * KS; i += NT) Ks[i] = 0.f;
  for (int i = threadIdx.x; i < 2 * R; i += NT) dsm[i] = 0.f;
  for (int i = threadIdx.x; i < 32; i += NT) st_tag(s_init + 8u * i, 0.f, -1);
  for (int i = threadIdx.x; i < TPL_STG; i += NT) stag[i] = -1;
  for (int i = threadIdx.x; i < W; i += NT) {
    qs[2 * i] = qtab ? qtab[2 * i] : 1.f / (float)(i + 1);
    qs[2 * i + 1] = qtab ? qtab[2 * i + 1] : 1.f / (float)(i + 1);
  }
  if (threadIdx.x == 0) {
    red[0] = red[1] = 0;
    for (int i = 0; i < 32; ++i)
      mbar_init(reinterpret_cast<unsigned long long*>(smem_tp + L::TKB) + i, 1);
    mbar_fence_init();
  }
  __syncthreads();

  if (warp < NW) {
    // ================= ring warps =================
    // steps as straight-line code (takeover / delta parts selected at compile
    // time for the warm-up, window-filling, main and tail ranges); the tags a
    // step depends on are tested after its deltas are out
    constexpr int TPL_LA = 2;
    const int j = threadIdx.x;                   // my slot
    float Y = 0.f, c = 0.f, idn = 0.f, bl = 0.f, bh = 0.f;
    int samp = -(1 << 30), fs = -1, nact = 0, status = 0;
    const float qmc = qs[2 * (W - 1)], qlc = qs[2 * (W - 1) + 1];
    const float4* kk4 = reinterpret_cast<const float4*>(Ks + j * KS);
    for (int s = 0; s < TPL_LA && s < Np; ++s)
      while (ld_volatile(stag + s) != s) {
      }
    int sm = 0;                                  // slot of m = n + P   (mod R)
    int sn = (R - P % R) % R;                    // slot of n
    auto ring_sync = [&]() {
      if constexpr (NW == 1) __syncwarp();
      else named_bar(2, 32 * NW);
    };
    auto step = [&](const int n, auto tk, auto dl_on, auto qconst) {
      const int m = n + P, e = n + 1, a = n - W + 1;
      float* dcur = dsm + (NW == 1 ? 0 : (n & 1) * R);
      // ---- step n: my slot's delta (the critical chain starts here) ----
      const float c_prev = c;
      if constexpr (decltype(dl_on)::value) {
        const int lo = n - W + 1 > 0 ? n - W + 1 : 0, cj = n - lo;
        float qm, ql;
        if constexpr (decltype(qconst)::value) {
          qm = qmc;
          ql = qlc;
        } else {
          qm = qs[2 * cj];
          ql = qs[2 * cj + 1];
        }
        const float q = samp == n ? ql : qm;
        const bool inw = (unsigned)(samp - lo) <= (unsigned)cj;
        float dl = q * idn * (fmaxf(bl - Y, 0.f) + fminf(bh - Y, 0.f));
        dl = inw ? dl : 0.f;
        c += dl;
        fs = (dl != 0.f && fs < 0) ? n : fs;
        dcur[j] = dl;
      }
      float iv;
      int itag;
      ld_tagged(s_init + 8u * (unsigned)(e & 31), iv, itag);
      const int la = m + TPL_LA;
      const int sgtag = ld_volatile(stag + (la & (TPL_STG - 1)));
      bool mine = false;
      if constexpr (decltype(tk)::value) {       // ---- takeover of sample m ----
        const float* sg = Sg + (m & (TPL_STG - 1)) * SSTR;
        int d = sm - j;                          // m - (the sample in my slot)
        d += d < 0 ? R : 0;
        const float v = sg[OKB + d];             // K[m][my sample]
        Ks[sm * KS + j] = v;
        Ks[j * KS + sm] = v;
        // c_j K[j][m] of the window [n-W+1, n-1] before step n's deltas
        const bool win = (unsigned)(samp - (n - W + 1)) < (unsigned)(W - 1);
        prg[(m & 31) * R + j] = win ? c_prev * v : 0.f;
        const float b = sg[OB];
        mine = j == sm;
        samp = mine ? m : samp;
        c = mine ? 0.f : c;
        fs = mine ? -1 : fs;
        status |= (mine && !(v > 0.f)) ? (int)KAPSM_TRAIN_DEGENERATE : 0;
        float rv;                                // MUFU on every lane: no branch
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rv) : "f"(v));
        idn = mine ? (v > 0.f ? rv : 0.f) : idn;
        bl = mine ? b - eps : bl;
        bh = mine ? b + eps : bh;
      }
      ring_sync();                               // deltas and the takeover's K row/column
      if constexpr (decltype(tk)::value) {       // m taken over: wake its helper
        if (j == 0)
          asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];"
                       ::"r"(s_tkb + 8u * (unsigned)(m & 31)) : "memory");
      }
      if (e >= 0 && e < Np && __any_sync(0xffffffffu, itag != e)) {
        do {                                     // (a helper is late: rare)
          ld_tagged(s_init + 8u * (unsigned)(e & 31), iv, itag);
        } while (__any_sync(0xffffffffu, itag != e));
      }
      int se = sn + 1;
      se -= se >= R ? R : 0;                     // slot of e
      const float add = (e >= 0 && e < Np && j == se) ? iv : 0.f;
      if constexpr (decltype(dl_on)::value) {
        const float4* dd4 = reinterpret_cast<const float4*>(dcur);
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
        if constexpr (NW == 1) {
          // the whole ring, unrolled and branch-free (deltas outside the
          // window are zero, K is finite everywhere): every load can be in
          // flight at once, at (R - W - P) / R extra shared-memory traffic
#pragma unroll
          for (int k = 0; k < R / 4; k += 2) {
            const float4 d0 = dd4[k], k0 = kk4[k], d1 = dd4[k + 1], k1 = kk4[k + 1];
            a0 = ffma2(make_float2(d0.x, d0.y), make_float2(k0.x, k0.y), a0);
            a1 = ffma2(make_float2(d0.z, d0.w), make_float2(k0.z, k0.w), a1);
            a2 = ffma2(make_float2(d1.x, d1.y), make_float2(k1.x, k1.y), a2);
            a3 = ffma2(make_float2(d1.z, d1.w), make_float2(k1.z, k1.w), a3);
          }
        } else {
          // wide rings: K only over the 8-slot groups the window [n-W+1, n]
          // touches (a rotating run of the ring); the other groups hold zero
          // deltas, so the sum is unchanged.
          constexpr int G = R / 8;
          int sw = sn - (W - 1);
          sw += sw < 0 ? R : 0;                  // slot of the oldest window sample
          const int g0 = sw >> 3, ng = ((sw & 7) + W + 7) >> 3;
          unsigned gm = ng >= G ? 0xffffffffu : (1u << ng) - 1u;
          gm = ng >= G ? gm : ((gm << g0) | (gm >> (G - g0)));
#pragma unroll
          for (int k = 0; k < R / 4; k += 2) {
            // outside the window: K's chunk is replaced by the (zero) delta
            // chunk itself -- a broadcast read, 1 wavefront instead of 4
            const float4* kr = ((gm >> (k >> 1)) & 1u) ? kk4 : dd4;
            const float4 d0 = dd4[k], k0 = kr[k], d1 = dd4[k + 1], k1 = kr[k + 1];
            a0 = ffma2(make_float2(d0.x, d0.y), make_float2(k0.x, k0.y), a0);
            a1 = ffma2(make_float2(d0.z, d0.w), make_float2(k0.z, k0.w), a1);
            a2 = ffma2(make_float2(d1.x, d1.y), make_float2(k1.x, k1.y), a2);
            a3 = ffma2(make_float2(d1.z, d1.w), make_float2(k1.z, k1.w), a3);
          }
        }
        const float upd = ((a0.x + a0.y) + (a1.x + a1.y)) + ((a2.x + a2.y) + (a3.x + a3.y));
        Y = (mine ? 0.f : Y) + (upd + add);      // the taken-over slot restarts at 0
      } else {
        Y = (mine ? 0.f : Y) + add;
      }
      int sa = sn - (W - 1);
      sa += sa < 0 ? R : 0;                      // slot of a
      const bool own = a >= 0 && j == sa;        // leaves after this step: c is final
      if (own) cfr[a & (TPL_CFR - 1)] = c;
      stg_if(own, Cout + a, c);
      stg_if(own, FSout + a, fs);
      nact += (own && fs >= 0) ? 1 : 0;
      if (la < Np && __any_sync(0xffffffffu, sgtag != la)) {
        while (ld_volatile(stag + (la & (TPL_STG - 1))) != la) {
        }
      }
      if constexpr (NW == 1) __syncwarp();       // delta reads done before the next writes
      sm = sm + 1 == R ? 0 : sm + 1;
      sn = se;
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    int n = -P;
    for (; n < 0 && n + P < Np; ++n) step(n, T_{}, F_{}, F_{});             // warm-up: takeovers
    for (; n < W - 1 && n + P < Np; ++n) step(n, T_{}, T_{}, F_{});         // window filling
    for (; n + P < Np; ++n) step(n, T_{}, T_{}, T_{});                      // main
    for (; n < 0; ++n) step(n, F_{}, F_{}, F_{});                           // (Np <= P)
    for (; n < Np; ++n) step(n, F_{}, T_{}, F_{});                          // tail: no takeover
    if (samp >= 0 && samp < Np && samp > Np - W) {   // still in the window after the last step
      Cout[samp] = c;
      FSout[samp] = fs;
      nact += fs >= 0;
    }
    atomicAdd(&red[0], nact);
    atomicOr(&red[1], status);
    named_bar(1, NT);
  } else {
    // ================= helper warps =================
    const int h = warp - NW;
    const bool vec = (D % 4) == 0 && (rx_stride % 4) == 0 && ((size_t)rx & 15) == 0;
    const int XP = vec ? D / 4 : D, NPC = 2 * XP + R / 4 + 10;
    const unsigned sg_s = sb + L::STG;
    // stage of sample s: pilot rows of s and of s - SPAN + 1, band row, live
    // list, target, live count; lane piece r: shared offset, size, global
    // address g + mm * gs + (mm >> 1) * gt for the piece's sample mm = s - off
    constexpr int PR_MAX = (2 * 64 * KPL + 32 * NW / 4 + 10 + 31) / 32;
    const char* pg[PR_MAX];
    int pgs[PR_MAX], pgt[PR_MAX], pof[PR_MAX], psz[PR_MAX];
    unsigned pso[PR_MAX];
#pragma unroll
    for (int r = 0; r < PR_MAX; ++r) {
      int pc = lane + 32 * r;
      pg[r] = nullptr; pgs[r] = 0; pgt[r] = 0; pso[r] = 0; psz[r] = 0; pof[r] = 0;
      if (pc < 2 * XP) {
        const int lv = pc >= XP;
        if (lv) pc -= XP;
        pg[r] = reinterpret_cast<const char*>(X + (vec ? 4 * pc : pc));
        pgt[r] = D * 4;
        pso[r] = (unsigned)(lv * OLR + (vec ? 4 * pc : pc)) * 4;
        psz[r] = vec ? 16 : 4;
        pof[r] = lv ? SPAN - 1 : 0;
      } else if (pc < 2 * XP + R / 4) {
        const int q = pc - 2 * XP;
        pg[r] = reinterpret_cast<const char*>(KB + 4 * q);
        pgs[r] = R * 4;
        pso[r] = (unsigned)(OKB + 4 * q) * 4;
        psz[r] = 16;
      } else if (pc < 2 * XP + R / 4 + 8) {
        const int q = pc - 2 * XP - R / 4;
        pg[r] = reinterpret_cast<const char*>(LV + q);
        pgt[r] = TP_CAP * 16;
        pso[r] = (unsigned)(OLV + 4 * q) * 4;
        psz[r] = gauss ? 16 : 0;
      } else if (pc == 2 * XP + R / 4 + 8) {
        pg[r] = reinterpret_cast<const char*>(Bt);
        pgs[r] = 4;
        pso[r] = (unsigned)OB * 4;
        psz[r] = 4;
      } else if (pc == 2 * XP + R / 4 + 9) {
        pg[r] = reinterpret_cast<const char*>(LC);
        pgt[r] = 4;
        pso[r] = (unsigned)OLC * 4;
        psz[r] = gauss ? 4 : 0;
      }
    }
    const int nr = (NPC + 31) / 32;
    auto prefetch = [&](int s) {
      const unsigned so = sg_s + (unsigned)((s & (TPL_STG - 1)) * SSTR) * 4;
#pragma unroll
      for (int r = 0; r < PR_MAX; ++r) {
        if (r < nr) {
          const int mm = s - pof[r];
          const bool in = s < Np && mm >= 0;
          const char* g = pg[r] + (long long)mm * pgs[r] + (long long)(mm >> 1) * pgt[r];
          cpa16_if(in && psz[r] == 16, so + pso[r], g);
          cpa4_if(in && psz[r] == 4, so + pso[r], g);
        }
      }
      cp_async_commit();
    };
    for (int jj = 0; jj < TPL_J; ++jj) prefetch(h + TPL_NH * jj);
    cp_async_wait<TPL_J - 2>();                 // my stages of h and h + NH landed
    __syncwarp();
    __threadfence_block();
    if (lane == 0 && h < Np) st_volatile(stag + (h & (TPL_STG - 1)), h);
    if (lane == 0 && h + TPL_NH < Np)
      st_volatile(stag + ((h + TPL_NH) & (TPL_STG - 1)), h + TPL_NH);
    float2 th[KPL];                              // (Re, Im) of antenna lane + 32 i
#pragma unroll
    for (int i = 0; i < KPL; ++i) th[i] = make_float2(0.f, 0.f);
    int next_a = 0;
    for (int m = h; m < Np; m += TPL_NH) {
      prefetch(m + TPL_NH * TPL_J);
      cp_async_wait<TPL_J - 2>();               // my stage of sample m + 2 NH landed
      __syncwarp();
      __threadfence_block();
      if (lane == 0 && m + 2 * TPL_NH < Np)
        st_volatile(stag + ((m + 2 * TPL_NH) & (TPL_STG - 1)), m + 2 * TPL_NH);
      // wait (suspended in hardware: no issue slots or shared-memory traffic
      // taken from the ring warps) for m's takeover
      while (!mbar_try_wait_s(s_tkb + 8u * (unsigned)(m & 31), (unsigned)((m >> 5) & 1))) {
      }
      float part = 0.f;
#pragma unroll
      for (int i = 0; i < NW; ++i) part += prg[(m & 31) * R + lane + 32 * i];
      // theta_fin: the samples a <= m - SPAN (left the window by m's takeover);
      // the row of a is the leaving row of stage a + SPAN - 1.  (Samples 2t
      // and 2t + 1 share the pilot row of t; a adds c_a r1(x) (a even) or
      // c_a r2(x) (a odd), r1 = [Re; Im], r2 = [Im; -Re], apsm.py:156-169.)
      for (; next_a <= m - SPAN; ++next_a) {
        const int a = next_a;
        const float ca = cfr[a & (TPL_CFR - 1)];
        const bool pair = (a & 1) == 0 && a + 1 <= m - SPAN;
        const float cb = pair ? cfr[(a + 1) & (TPL_CFR - 1)] : 0.f;
        const float ce = (a & 1) ? 0.f : ca, co = (a & 1) ? ca : cb;
        const float* xa = Sg + ((a + SPAN - 1) & (TPL_STG - 1)) * SSTR + OLR;
#pragma unroll
        for (int i = 0; i < KPL; ++i) {
          const int k = lane + 32 * i;
          if (k < M) {
            const float2 x = *reinterpret_cast<const float2*>(xa + 2 * k);
            th[i].x = fmaf(ce, x.x, fmaf(co, x.y, th[i].x));
            th[i].y = fmaf(ce, x.y, fmaf(-co, x.x, th[i].y));
          }
        }
        next_a += pair ? 1 : 0;
      }
      const float* sm_ = Sg + (m & (TPL_STG - 1)) * SSTR;
      float lin = 0.f;
      const int bt = m & 1;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int k = lane + 32 * i;
        if (k < M) {
          const float2 x = *reinterpret_cast<const float2*>(sm_ + 2 * k);
          lin = fmaf(th[i].x, bt ? x.y : x.x, lin);
          lin = fmaf(th[i].y, bt ? -x.x : x.y, lin);
        }
      }
      part = fmaf(w_l, lin, part);
      if (gauss) {                              // live Gaussian terms of older samples
        const int cnt = __float_as_int(sm_[OLC]);
        if (cnt > 0) {
          if (lane < 2 * cnt) {
            const float4 v4 = reinterpret_cast<const float4*>(sm_ + OLV)[lane >> 1];
            const int al = lane & 1, a = 2 * __float_as_int(v4.w) + al;
            if (a <= m - SPAN) {
              const float kap = al == 0 ? (bt == 0 ? v4.x : v4.y) : (bt == 0 ? v4.z : v4.x);
              part = fmaf(w_g * __ldcg(Cout + a), kap, part);
            }
          }
        } else if (cnt < 0) {                   // more live pilots than the list holds
          const int tl = m >> 1;
          const float* xm = X + (long long)tl * D;
          for (int w = lane; w < NWp; w += 32) {
            unsigned bits = LW[(long long)w * n_train + tl];
            while (bits) {
              const int p = w * 32 + __ffs(bits) - 1;
              bits &= bits - 1;
              const float* xa = X + (long long)p * D;
              for (int al = 0; al < 2; ++al) {
                const int a = 2 * p + al;
                if (a > m - SPAN) continue;
                float dist = 0.f;
                for (int e2 = 0; e2 < D; ++e2) {
                  const float z = rcomp(xa, e2, al) - rcomp(xm, e2, bt);
                  dist = fmaf(z, z, dist);
                }
                part = fmaf(w_g * __ldcg(Cout + a), exp_fast(-dist * inv2s), part);
              }
            }
          }
        }
      }
      const float init = warp_sum_f(part);
      if (lane == 0) st_tag(s_init + 8u * (unsigned)(m & 31), init, m);
    }
    cp_async_wait<0>();
    named_bar(1, NT);
    if (h == 0) {                               // theta = w_l (all final c_a r_a)
      for (; next_a < Np; ++next_a) {
        const int a = next_a;
        const float ca = __ldcg(Cout + a);
        const float* xa = X + (long long)(a >> 1) * D;
#pragma unroll
        for (int i = 0; i < KPL; ++i) {
          const int k = lane + 32 * i;
          if (k < M) {
            const float xr = xa[2 * k], xi = xa[2 * k + 1];
            th[i].x = fmaf(ca, (a & 1) ? xi : xr, th[i].x);
            th[i].y = fmaf(ca, (a & 1) ? -xr : xi, th[i].y);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int k = lane + 32 * i;
        if (k < M) {
          theta_out[(long long)task * D + k] = w_l * th[i].x;
          theta_out[(long long)task * D + M + k] = w_l * th[i].y;
        }
      }
      if (lane == 0) {
        nact_out[task] = red[0];
        status_out[task] = red[1];
      }
    }
  }
}

static int tp_num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

int screen_tc_rows(const float* rx, long long rx_stride, int F, int n_train, int n_rows,
                   int y_row0, int list_max_off, int M, kapsm_kernel_params p, unsigned* live,
                   int* cnt, float4* vals, cudaStream_t s);

// ring size of the chain's trainer: 32 (one warp) while P = 28 - W > TP_AHEAD,
// else the wide trainer's 32 NW
static int tp_ring(int W) { return tp_lead(W) > TP_AHEAD ? TP_RING : 32 * tpw_nw(W); }

// workspace carved out of the pipeline's Gram workspace: band rows (R per
// realified pilot), then the pilot x pilot screen (live words, counts, lists)
size_t train_tp_ws_bytes(int F, int n_train, int W) {
  const size_t Np = 2 * (size_t)n_train, NWp = (n_train + 31) / 32, R = tp_ring(W);
  const size_t band = (F * Np * R * 4 + 255) / 256 * 256;
  const size_t live = (F * NWp * n_train * 4 + 255) / 256 * 256;
  const size_t cnt = (F * (size_t)n_train * 4 + 255) / 256 * 256;
  return band + live + cnt + F * (size_t)n_train * TP_CAP * 16;
}

bool train_tp_supported(int n_train, int M, int W) {
  // the live terms of a sample are added TP_AHEAD steps after its takeover, which
  // must precede its entry into the window: P = SPAN - W > TP_AHEAD
  if (W < 1 || M < 1 || M > 64 || n_train < 1) return false;
  if (tp_lead(W) > TP_AHEAD) return tp_total(M) <= 200 * 1024;
  return tpw_nw(W) <= TPW_MAX_NW && tpw_total_rt(tpw_nw(W), M) <= 227 * 1024;
}

// stages (bit mask, all by default): 1 band rows, 2 pilot screen, 4 trainer --
// separate launches so the bench can time each on its stream; 8: no
// critical-warp form in latency mode (A/B)
int train_tp(const float* rx, long long rx_stride, const float* targets, int F, int K,
             int n_train, int M, int W, double eps, kapsm_kernel_params p, const float* qtab,
             void* ws, float* coeff, int* first_step, float* theta, int* n_active, int* status,
             cudaStream_t s, int stages = 7) {
  if (!train_tp_supported(n_train, M, W)) return KAPSM_ERR_UNSUPPORTED;
  const int Np = 2 * n_train, NWp = (n_train + 31) / 32, R = tp_ring(W), SPAN = R - 4;
  char* w = reinterpret_cast<char*>(ws);
  float* kband = reinterpret_cast<float*>(w);
  w += ((size_t)F * Np * R * 4 + 255) / 256 * 256;
  unsigned* plive = reinterpret_cast<unsigned*>(w);
  w += ((size_t)F * NWp * n_train * 4 + 255) / 256 * 256;
  int* pcnt = reinterpret_cast<int*>(w);
  w += ((size_t)F * n_train * 4 + 255) / 256 * 256;
  float4* pvals = reinterpret_cast<float4*>(w);
  const float inv2s = (float)(1.0 / (2.0 * p.sigma_sq));
  if (stages & 1) {
    // tiles of TT pilots: shared rows (TT + R/2) x (2M + 4) floats + band 2 TT x R
    const int DS = ((2 * M + 3) & ~3) + 4;
    int TT = 128;
    while (TT > 16 && ((size_t)(TT + R / 2) * DS + (size_t)2 * TT * R) * 4 > 100 * 1024) TT >>= 1;
    const size_t smem = ((size_t)(TT + R / 2) * DS + (size_t)2 * TT * R) * 4;
    if (cudaFuncSetAttribute(band_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return KAPSM_ERR_CUDA;
    dim3 grid((unsigned)((n_train + TT - 1) / TT), F);
    band_tile_kernel<<<grid, 256, smem, s>>>(rx, rx_stride, n_train, M, (float)p.w_l,
                                             (float)p.w_g, inv2s, kband, R, TT);
    if (cudaGetLastError() != cudaSuccess) return KAPSM_ERR_CUDA;
  }
  const int tasks = F * K;
  // latency (chains <= SMs): one chain per CTA with >= 120 KB of shared memory,
  // so no other CTA (the concurrent detection screen) shares its SM, and the
  // ring-warps + helpers form when its shared memory fits
  const bool lat = tasks <= tp_num_sms();
  const int NWr = R / 32, KPL = tpl_kpl(M);
  size_t tpl_smem = 0;
  switch (NWr) {
    case 1: tpl_smem = tpl_bytes<1>(M); break;
    case 2: tpl_smem = tpl_bytes<2>(M); break;
    case 3: tpl_smem = tpl_bytes<3>(M); break;
    case 4: tpl_smem = tpl_bytes<4>(M); break;
    default: tpl_smem = tpl_bytes<5>(M); break;
  }
  const bool tpl = lat && !(stages & 8) && tpl_smem <= 227 * 1024;
  const int span = tpl ? tpl_span(NWr, W) : SPAN;
  if ((stages & 2) && p.w_g != 0.0) {
    // lists only hold pilots p <= t - span / 2 of row t: the trainer's live
    // terms are the samples a <= m - span (the band rows cover the rest)
    const int r = screen_tc_rows(rx, rx_stride, F, n_train, n_train, 0, -(span / 2), M, p,
                                 plive, pcnt, pvals, s);
    if (r) return r;
  }
  if (!(stages & 4)) return KAPSM_OK;
  const int DPL = (2 * M + 31) / 32;
  auto launch = [&](auto kern, int wpc, int threads, size_t smem) -> int {
    if (lat && smem < 120 * 1024) smem = 120 * 1024;
    if (smem > 227 * 1024) return (int)KAPSM_ERR_UNSUPPORTED;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return (int)KAPSM_ERR_CUDA;
    kern<<<(tasks + wpc - 1) / wpc, threads, smem, s>>>(
        rx, rx_stride, targets, kband, plive, pcnt, pvals, F, K, n_train, M, W, (float)eps,
        (float)p.w_l, (float)p.w_g, inv2s, qtab, coeff, first_step, theta, n_active, status);
    return status_from(cudaGetLastError());
  };
  if (tpl) {                                   // latency: ring warps + helpers
    const size_t smem = tpl_smem;
#define KAPSM_TPL(NWV)                                                                        \
  if (NWr == NWV) {                                                                           \
    if (KPL == 1) return launch(apsm_train_tpl_kernel<1, NWV>, 1, 32 * (NWV + TPL_NH), smem); \
    return launch(apsm_train_tpl_kernel<2, NWV>, 1, 32 * (NWV + TPL_NH), smem);               \
  }
    KAPSM_TPL(1)
    KAPSM_TPL(2)
    KAPSM_TPL(3)
    KAPSM_TPL(4)
    KAPSM_TPL(5)
#undef KAPSM_TPL
  }
  if (R == TP_RING) {
    int wpc = lat ? 1 : 4;
    while (wpc > 1 && (size_t)tp_total(M) * wpc > 227 * 1024) wpc >>= 1;
    const size_t smem = (size_t)tp_total(M) * wpc;
    const bool vec = (2 * M) % 4 == 0 && rx_stride % 4 == 0 && ((size_t)rx & 15) == 0;
    if (vec) {
      if (DPL == 1) return launch(apsm_train_tp_kernel<1, true>, wpc, 32 * wpc, smem);
      if (DPL == 2) return launch(apsm_train_tp_kernel<2, true>, wpc, 32 * wpc, smem);
      return launch(apsm_train_tp_kernel<4, true>, wpc, 32 * wpc, smem);
    }
    if (DPL == 1) return launch(apsm_train_tp_kernel<1, false>, wpc, 32 * wpc, smem);
    if (DPL == 2) return launch(apsm_train_tp_kernel<2, false>, wpc, 32 * wpc, smem);
    return launch(apsm_train_tp_kernel<4, false>, wpc, 32 * wpc, smem);
  }
  // wide windows: one CTA of R / 32 warps per chain
  const int NW = R / 32;
  const size_t smem = (size_t)tpw_total_rt(NW, M);
#define KAPSM_TPW(NWV)                                                                   \
  if (NW == NWV) {                                                                       \
    if (DPL == 1) return launch(apsm_train_tpw_kernel<1, NWV>, 1, 32 * NWV, smem);       \
    if (DPL == 2) return launch(apsm_train_tpw_kernel<2, NWV>, 1, 32 * NWV, smem);       \
    return launch(apsm_train_tpw_kernel<4, NWV>, 1, 32 * NWV, smem);                     \
  }
  KAPSM_TPW(2)
  KAPSM_TPW(3)
  KAPSM_TPW(4)
  KAPSM_TPW(5)
#undef KAPSM_TPW
  return KAPSM_ERR_UNSUPPORTED;
}

}  // namespace kapsm

// Internal (bench stage timing, not in the public header): the throughput
// trainer's stages alone -- band rows (1), pilot screen (2), trainer (4) -- on a
// workspace of kapsm_internal_train_tp_ws_bytes bytes.
extern "C" long long kapsm_internal_train_tp_ws_bytes(int F, int n_train, int W) {
  return (long long)kapsm::train_tp_ws_bytes(F, n_train, W);
}
extern "C" int kapsm_internal_train_tp_f32(int stages, const float* rx, long long rx_stride,
                                           const float* targets, int F, int K, int n_train, int M,
                                           int W, double eps, kapsm_kernel_params p,
                                           const float* qtab, void* ws, float* coeff,
                                           int* first_step, float* theta, int* n_active,
                                           int* status, void* stream) {
  return kapsm::train_tp(rx, rx_stride, targets, F, K, n_train, M, W, eps, p, qtab, ws, coeff,
                         first_step, theta, n_active, status, (cudaStream_t)stream, stages);
}
