// K3 split for the latency pipeline: the pilot/payload kernel screen does not
// depend on the trained coefficients, so it runs on the SMs the trainer leaves
// idle, concurrently with it; only the (rare) live pairs are revisited once the
// filters exist.
//
//   K3a detect_screen : for every (pilot p, payload t) pair of a frame, one
//       complex dot x_p^H y_t gives the three realified distances from the norm
//       expansion (same screen as the fused kernel, detect.cu); a pair whose
//       smallest kernel does not underflow sets bit p of live[f][p/32][t].
//   K3b detect_finish : per payload symbol and user, the linear part
//       conj(Theta_u) . y, plus the Gaussian part over the live pilots in
//       pilot order, recomputed with explicit differences (kernels.py:187-191),
//       g(r) = f(r1) + i f(r2) (engine.py:261), the hard decision
//       (noma.py:125-135, ties to the lowest index) and the bit / symbol error
//       counts (noma.py:284-292).
#include "kapsm_common.cuh"

namespace kapsm {

constexpr int SC_WARPS = 8;
constexpr int SC_CAP = 8;       // live pilots kept per payload symbol (else recomputed)

// workspace: live bits F x NW x n_data | counts F x n_data | lists F x n_data x CAP
__host__ __device__ inline size_t ws_live(int F, int n_train, int n_data) {
  return (size_t)F * ((n_train + 31) / 32) * n_data * 4;
}
__host__ __device__ inline size_t ws_cnt(int F, int n_data) { return (size_t)F * n_data * 4; }
__host__ __device__ inline size_t ws_bytes(int F, int n_train, int n_data) {
  return (ws_live(F, n_train, n_data) + ws_cnt(F, n_data) + 15) / 16 * 16 +
         (size_t)F * n_data * SC_CAP * 16;
}

template <typename T> struct ScreenThresh;
template <> struct ScreenThresh<float> { static constexpr float dead = 88.0f; };
template <> struct ScreenThresh<double> { static constexpr double dead = 745.0; };

template <typename T, int MT>
KAPSM_DEV void cdot_s(const T* __restrict__ x, const T (&y)[2 * MT], T& cr, T& ci) {
  T r0 = T(0), r1 = T(0), i0 = T(0), i1 = T(0);
  if constexpr (sizeof(T) == 4) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll
    for (int q = 0; q < MT / 2; ++q) {
      const float4 v = x4[q];
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

// CTA = 32 payload symbols x all pilots (pilot range split over 8 warps),
// pilots staged in shared memory chunk by chunk; the live bits of the tile
// gather in shared memory and leave coalesced.
template <typename T, int MT>
__global__ void __launch_bounds__(SC_WARPS * 32)
    detect_screen_kernel(const T* __restrict__ rx, long long rx_stride, int n_train, int n_data,
                         int M, int PC, T inv2s, unsigned* __restrict__ live,
                         int* __restrict__ cnt, float4* __restrict__ vals) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int NW = (n_train + 31) / 32;
  unsigned* bits = reinterpret_cast<unsigned*>(smem);          // [NW][32]
  T* xs = reinterpret_cast<T*>(smem + ((size_t)NW * 32 * 4 + 15) / 16 * 16);
  T* nxs = xs + (size_t)PC * 2 * MT;
  const int f = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 32 + lane;
  const bool tvalid = t < n_data;
  const T* Xf = rx + (long long)f * rx_stride;
  for (int i = threadIdx.x; i < NW * 32; i += blockDim.x) bits[i] = 0u;

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
  for (int c0 = 0; c0 < n_train; c0 += PC) {
    const int pc = min(PC, n_train - c0);
    __syncthreads();
    if (M == MT) {
      const int nvec = pc * 2 * MT * (int)sizeof(T) / 16;
      const char* src = reinterpret_cast<const char*>(Xf + (long long)c0 * 2 * M);
      char* dst = reinterpret_cast<char*>(xs);
      for (int e = threadIdx.x; e < nvec; e += blockDim.x) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst + 16 * e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + 16 * (long long)e)
                     : "memory");
      }
      cp_async_commit();
      cp_async_wait<0>();
    } else {
      for (int e = threadIdx.x; e < pc * MT; e += blockDim.x) {
        const int p = e / MT, k = e - p * MT;
        T xr = T(0), xi = T(0);
        if (k < M) {
          const T* xp = Xf + (long long)(c0 + p) * 2 * M + 2 * k;
          xr = xp[0];
          xi = xp[1];
        }
        xs[p * 2 * MT + 2 * k] = xr;
        xs[p * 2 * MT + 2 * k + 1] = xi;
      }
    }
    __syncthreads();
    for (int p = threadIdx.x; p < pc; p += blockDim.x) {
      T sacc = T(0);
#pragma unroll 8
      for (int k = 0; k < 2 * MT; ++k) sacc = fma(xs[p * 2 * MT + k], xs[p * 2 * MT + k], sacc);
      nxs[p] = sacc;
    }
    __syncthreads();
    int p = warp;
    for (; p + SC_WARPS < pc; p += 2 * SC_WARPS) {        // two pilots per iteration (ILP)
      const int q = p + SC_WARPS;
      T crp, cip, crq, ciq;
      cdot_s<T, MT>(xs + p * 2 * MT, y, crp, cip);
      cdot_s<T, MT>(xs + q * 2 * MT, y, crq, ciq);
      const T dp = nxs[p] + ny - T(2) * fmax(crp, fabs(cip));
      const T dq = nxs[q] + ny - T(2) * fmax(crq, fabs(ciq));
      if (tvalid && dp * inv2s < ScreenThresh<T>::dead) {
        const int g = c0 + p;
        atomicOr(&bits[(g >> 5) * 32 + lane], 1u << (g & 31));
      }
      if (tvalid && dq * inv2s < ScreenThresh<T>::dead) {
        const int g = c0 + q;
        atomicOr(&bits[(g >> 5) * 32 + lane], 1u << (g & 31));
      }
    }
    for (; p < pc; p += SC_WARPS) {
      T crp, cip;
      cdot_s<T, MT>(xs + p * 2 * MT, y, crp, cip);
      const T dp = nxs[p] + ny - T(2) * fmax(crp, fabs(cip));
      if (tvalid && dp * inv2s < ScreenThresh<T>::dead) {
        const int g = c0 + p;
        atomicOr(&bits[(g >> 5) * 32 + lane], 1u << (g & 31));
      }
    }
  }
  __syncthreads();
  // live[f][w][t]: word-major, coalesced over the payload symbols
  unsigned* lf = live + (long long)f * NW * n_data;
  for (int i = threadIdx.x; i < NW * 32; i += blockDim.x) {
    const int w = i >> 5, l = i & 31, tt = blockIdx.x * 32 + l;
    if (tt < n_data) lf[(long long)w * n_data + tt] = bits[i];
  }
  // ---- compact list of the live pilots of each payload symbol, in pilot
  //      order, with the three kernel values recomputed from explicit
  //      differences (kernels.py:187-191): the finish only contracts them.
  //      Warp w takes words w, w+8, ...; per-(symbol, word) popcounts give the
  //      write offsets.  More than SC_CAP live pilots: count = -1 (the finish
  //      recomputes that symbol from the bits). ----
  int* offs = reinterpret_cast<int*>(nxs + PC);          // [NW][32] (reuses the chunk area)
  for (int i = threadIdx.x; i < NW * 32; i += blockDim.x) offs[i] = __popc(bits[i]);
  __syncthreads();
  if (warp == 0) {                                       // exclusive prefix over words, per symbol
    int run = 0;
    for (int w = 0; w < NW; ++w) {
      const int c = offs[w * 32 + lane];
      offs[w * 32 + lane] = run;
      run += c;
    }
    // (FP64, the parity precision, always recomputes: the lists hold FP32)
    if (tvalid) cnt[(long long)f * n_data + t] = (sizeof(T) == 4 && run <= SC_CAP) ? run : -1;
  }
  __syncthreads();
  if (sizeof(T) == 4 && tvalid) {
    float4* vt = vals + ((long long)f * n_data + t) * SC_CAP;
    for (int w = warp; w < NW; w += SC_WARPS) {
      unsigned b = bits[w * 32 + lane];
      int j = offs[w * 32 + lane];
      while (b) {
        const int p = w * 32 + __ffs(b) - 1;
        b &= b - 1;
        if (j < SC_CAP) {
          const T* x = Xf + (long long)p * 2 * M;
          T ea = T(0), eb = T(0), ec = T(0);
#pragma unroll
          for (int k = 0; k < MT; ++k) {
            if (k < M) {
              const T xr = x[2 * k], xi = x[2 * k + 1], yr = y[2 * k], yi = y[2 * k + 1];
              T a0 = xr - yr, a1 = xi - yi;
              ea = fma(a0, a0, fma(a1, a1, ea));
              a0 = xr - yi; a1 = xi + yr;
              eb = fma(a0, a0, fma(a1, a1, eb));
              a0 = xr + yi; a1 = xi - yr;
              ec = fma(a0, a0, fma(a1, a1, ec));
            }
          }
          vt[j] = make_float4((float)exp_fast(-ea * inv2s), (float)exp_fast(-eb * inv2s),
                              (float)exp_fast(-ec * inv2s), __int_as_float(p));
        }
        ++j;
      }
    }
  }
}

// One thread per (payload symbol, user): linear part, the live pilots (their
// words prefetched together), demap, counts.  A CTA holds up to 8 users (all
// of a frame's at the paper's K = 6: the payload rows are staged once per
// frame; 4 users for the wide rows of M > 16) and walks nb blocks of 32
// symbols: theta is loaded once, and the next block's rows are loaded into
// registers while the current block is finished (FP32, 16-byte rows), so a
// CTA pays one memory latency instead of one per block.
template <typename T, int MT>
__global__ void __launch_bounds__(256)
    detect_finish_kernel(const T* __restrict__ rx, long long rx_stride, int K, int n_train,
                         int n_data, int M, const T* __restrict__ coeff,
                         const T* __restrict__ theta, T w_g, T inv2s,
                         const T* __restrict__ points, int n_points,
                         const unsigned char* __restrict__ tx_labels,
                         const unsigned* __restrict__ live, T* __restrict__ est_out,
                         unsigned char* __restrict__ labels_out,
                         unsigned long long* __restrict__ bit_err,
                         unsigned long long* __restrict__ sym_err, int nb) {
  __shared__ T pts[128];
  // 32 payload rows per buffer, two buffers; odd row stride in (re, im)
  // pairs: conflict-free pair reads
  constexpr int YS = 2 * MT + 2;
  constexpr int NBUF = sizeof(T) == 4 ? 2 : 1;             // FP64: one buffer (48 KB static)
  __shared__ __align__(16) T ys[NBUF][32 * YS];
  __shared__ __align__(16) T tvs[8][2 * MT];               // theta of the CTA's users
  const int f = blockIdx.z;
  const int lane = threadIdx.x;
  const int u = blockIdx.y * blockDim.y + threadIdx.y;
  const int NW = (n_train + 31) / 32, Np = 2 * n_train;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int nthr = blockDim.x * blockDim.y;
  const int rl = 2 * M;
  for (int i = tid; i < 2 * n_points; i += nthr) pts[i] = points[i];
  const T* Xf = rx + (long long)f * rx_stride;
  const int blk0 = blockIdx.x * nb;
  const int nblk = min(nb, (n_data + 31) / 32 - blk0);
  const T* src0 = Xf + (long long)(n_train + blk0 * 32) * rl;
  const bool vec = sizeof(T) == 4 && (rl & 3) == 0 && ((size_t)src0 & 15) == 0 &&
                   ((rx_stride & 3) == 0);
  constexpr int PER = (32 * 2 * MT / 4 + 127) / 128;        // float4 per thread at >= 128 threads
  float4 v[PER];
  auto rows_of = [&](int b) { return min(32, n_data - (blk0 + b) * 32); };
  auto load_regs = [&](int b) {                             // FP32 16-byte path
    const float4* s4 = reinterpret_cast<const float4*>(src0 + (long long)b * 32 * rl);
    const int n = rows_of(b) * rl;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e4 = tid + i * nthr;
      v[i] = 4 * e4 < n ? __ldg(s4 + e4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto store_regs = [&](int b, T* buf) {
    const int n = rows_of(b) * rl;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = 4 * (tid + i * nthr);
      if (e < n) {
        // rows of exactly 2 MT floats (M == MT): a shift, not a division
        const int r = rl == 2 * MT ? e / (2 * MT) : e / rl, c = e - r * rl;
        T* d = buf + r * YS + c;
        d[0] = (T)v[i].x; d[1] = (T)v[i].y; d[2] = (T)v[i].z; d[3] = (T)v[i].w;
      }
    }
    const T* src = src0 + (long long)b * 32 * rl;
    for (int e = 4 * (tid + PER * nthr); e < n; e += 4 * nthr) {   // (< 128 threads)
      const int r = e / rl, c = e - r * rl;
      for (int j = 0; j < 4; ++j) buf[r * YS + c + j] = src[e + j];
    }
  };
  auto stage_plain = [&](int b, T* buf) {                  // FP64 / unaligned rows
    const T* src = src0 + (long long)b * 32 * rl;
    const int n = rows_of(b) * rl;
    for (int e = tid; e < n; e += nthr) {
      const int r = e / rl;
      buf[r * YS + (e - r * rl)] = src[e];
    }
  };
  if (nblk > 0) {
    if (vec) {
      load_regs(0);
      store_regs(0, ys[0]);
    } else {
      stage_plain(0, ys[0]);
    }
  }
  // theta of user u once (shared, broadcast reads): conj(Theta_u) . y with
  // Theta = theta[:M] + i theta[M:]
  const bool uvalid = u < K;
  {
    const T* th = theta + ((long long)f * K + (uvalid ? u : 0)) * 2 * M;
    for (int k = lane; k < MT; k += 32) {
      tvs[threadIdx.y][k] = (uvalid && k < M) ? th[k] : T(0);
      tvs[threadIdx.y][MT + k] = (uvalid && k < M) ? th[M + k] : T(0);
    }
  }
  const T* tv = tvs[threadIdx.y];
  const T* cu = coeff + ((long long)f * K + (uvalid ? u : 0)) * Np;
  const char* ws = reinterpret_cast<const char*>(live);
  const int* cntp = reinterpret_cast<const int*>(ws + ws_live(gridDim.z, n_train, n_data));
  const float4* vals = reinterpret_cast<const float4*>(
      ws + (ws_live(gridDim.z, n_train, n_data) + ws_cnt(gridDim.z, n_data) + 15) / 16 * 16);
  unsigned long long be = 0, se = 0;
  for (int b = 0; b < nblk; ++b) {
    if constexpr (NBUF == 1) {
      if (b > 0) {
        __syncthreads();                                    // block b - 1 finished
        stage_plain(b, ys[0]);
      }
    }
    __syncthreads();                                        // rows of block b staged
    const bool more = b + 1 < nblk;
    if constexpr (NBUF == 2) {
      if (more) {
        if (vec) load_regs(b + 1);                          // in flight during block b
        else stage_plain(b + 1, ys[(b + 1) & 1]);
      }
    }
    const T* yb = ys[NBUF == 2 ? (b & 1) : 0];
    const int t = (blk0 + b) * 32 + lane;
    const bool tvalid = t < n_data && uvalid;
    const int nl = tvalid ? cntp[(long long)f * n_data + t] : 0;
    const unsigned txl = (tvalid && tx_labels) ? tx_labels[((long long)f * K + u) * n_data + t] : 0u;
    // the symbol's row straight from shared memory (no register copy: the
    // CTA keeps its occupancy); theta entries past M are zero
    const T* yp = yb + lane * YS;
    T lr = T(0), li = T(0);
#pragma unroll
    for (int k = 0; k < MT; ++k) {
      const T tr = tv[k], ti = tv[MT + k];
      const T yr = k < M ? yp[2 * k] : T(0), yi = k < M ? yp[2 * k + 1] : T(0);
      lr = fma(tr, yr, fma(ti, yi, lr));
      li = fma(tr, yi, fma(-ti, yr, li));
    }
    T gr = T(0), gi = T(0);
    if (tvalid && w_g != T(0) && nl >= 0) {                 // the screen's compact list
      const float4* vt = vals + ((long long)f * n_data + t) * SC_CAP;
      // entries 4 at a time: the list loads, then the coefficient loads they
      // index, in flight together (two memory round trips per 4 entries
      // instead of two per entry); accumulated in list order as before
      for (int j0 = 0; j0 < nl; j0 += 4) {
        float4 vv[4];
        T c1[4], c2[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          vv[i] = j0 + i < nl ? vt[j0 + i] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int p = __float_as_int(vv[i].w);
          c1[i] = j0 + i < nl ? cu[2 * p] : T(0);
          c2[i] = j0 + i < nl ? cu[2 * p + 1] : T(0);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (j0 + i < nl) {
            const T ka = (T)vv[i].x, kb = (T)vv[i].y, kc = (T)vv[i].z;
            gr = fma(c1[i], ka, fma(c2[i], kc, gr));
            gi = fma(c1[i], kb, fma(c2[i], ka, gi));
          }
        }
      }
    } else if (tvalid && w_g != T(0)) {                     // too many live pilots: recompute
      const unsigned* lf = live + (long long)f * NW * n_data + t;
      for (int w0 = 0; w0 < NW; w0 += 8) {
        unsigned wb[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) wb[q] = (w0 + q < NW) ? lf[(long long)(w0 + q) * n_data] : 0u;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          unsigned bb = wb[q];
          while (bb) {
            const int p = (w0 + q) * 32 + __ffs(bb) - 1;
            bb &= bb - 1;
            const T* x = Xf + (long long)p * 2 * M;
            const T c1 = cu[2 * p], c2 = cu[2 * p + 1];
            T ea = T(0), eb = T(0), ec = T(0);
#pragma unroll
            for (int k = 0; k < MT; ++k) {
              if (k < M) {
                const T xr = x[2 * k], xi = x[2 * k + 1], yr = yp[2 * k], yi = yp[2 * k + 1];
                T a0 = xr - yr, a1 = xi - yi;
                ea = fma(a0, a0, fma(a1, a1, ea));
                a0 = xr - yi; a1 = xi + yr;
                eb = fma(a0, a0, fma(a1, a1, eb));
                a0 = xr + yi; a1 = xi - yr;
                ec = fma(a0, a0, fma(a1, a1, ec));
              }
            }
            const T ka = exp_fast(-ea * inv2s), kb = exp_fast(-eb * inv2s), kc = exp_fast(-ec * inv2s);
            gr = fma(c1, ka, fma(c2, kc, gr));
            gi = fma(c1, kb, fma(c2, ka, gi));
          }
        }
      }
    }
    const T er = lr + w_g * gr, ei = li + w_g * gi;
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
        be += __popc((unsigned)best ^ txl);
        se += ((unsigned)best != txl) ? 1ull : 0ull;
      }
    }
    if constexpr (NBUF == 2) {
      if (more && vec) store_regs(b + 1, ys[(b + 1) & 1]); // (read after the next barrier)
    }
  }
  if (uvalid && tx_labels && (bit_err || sym_err)) {
    const unsigned long long bsum = warp_sum_u64(be), ssum = warp_sum_u64(se);
    if (lane == 0) {
      if (bit_err && bsum) atomicAdd(&bit_err[(long long)f * K + u], bsum);
      if (sym_err && ssum) atomicAdd(&sym_err[(long long)f * K + u], ssum);
    }
  }
}

template <typename T, int MT>
int launch_screen(const T* rx, long long rx_stride, int F, int n_train, int n_data, int M,
                  kapsm_kernel_params p, unsigned* live, cudaStream_t s) {
  const int NW = (n_train + 31) / 32;
  const size_t bitsb = ((size_t)NW * 32 * 4 + 15) / 16 * 16;
  const size_t per_pilot = (2 * MT + 1) * sizeof(T);
  int PC = (int)((110 * 1024 - bitsb - (size_t)NW * 32 * 4) / per_pilot);
  PC = PC / 16 * 16;
  if (PC > n_train) PC = (n_train + 15) / 16 * 16;
  if (PC < 16) PC = 16;
  size_t smem = bitsb + (size_t)PC * per_pilot + 16 + (size_t)NW * 32 * 4;
  // more than an SM holding a latency-mode trainer CTA (120 KB) has left:
  // the screen never shares an SM with a critical warp
  if (smem < 112 * 1024) smem = 112 * 1024;
  auto kern = detect_screen_kernel<T, MT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  dim3 grid((n_data + 31) / 32, F);
  char* ws = reinterpret_cast<char*>(live);
  int* cnt = reinterpret_cast<int*>(ws + ws_live(F, n_train, n_data));
  float4* vals = reinterpret_cast<float4*>(
      ws + (ws_live(F, n_train, n_data) + ws_cnt(F, n_data) + 15) / 16 * 16);
  kern<<<grid, SC_WARPS * 32, smem, s>>>(rx, rx_stride, n_train, n_data, M, PC,
                                         (T)(1.0 / (2.0 * p.sigma_sq)), live, cnt, vals);
  return status_from(cudaGetLastError());
}

template <typename T, int MT>
int launch_finish(const T* rx, long long rx_stride, int F, int K, int n_train, int n_data, int M,
                  const T* coeff, const T* theta, kapsm_kernel_params p, const T* points,
                  int n_points, const unsigned char* tx, const unsigned* live, T* est,
                  unsigned char* labels, unsigned long long* be, unsigned long long* se,
                  cudaStream_t s) {
  // users per CTA: all of a frame's (up to 8) for batches of frames -- the
  // payload rows staged once; 4 for a few frames, where more, smaller CTAs
  // shorten the single-frame latency
  const int ku = (MT <= 16 && sizeof(T) == 4 && F >= 8) ? (K < 8 ? K : 8) : 4;
  // symbol blocks per CTA: 4 for batches (one latency per 128 symbols), 1 for
  // a few frames (more CTAs: a shorter single-frame critical path)
  const int nb = (F >= 8 && sizeof(T) == 4) ? 8 : 1;       // (FP64: one staging buffer)
  const int nblocks = (n_data + 31) / 32;
  dim3 block(32, ku);
  dim3 grid((nblocks + nb - 1) / nb, (K + ku - 1) / ku, F);
  detect_finish_kernel<T, MT><<<grid, block, 0, s>>>(
      rx, rx_stride, K, n_train, n_data, M, coeff, theta, (T)p.w_g,
      (T)(1.0 / (2.0 * p.sigma_sq)), points, n_points, tx, live, est, labels, be, se, nb);
  return status_from(cudaGetLastError());
}

int screen_tc(const float* rx, long long rx_stride, int F, int n_train, int n_data, int M,
              kapsm_kernel_params p, unsigned* live, int* cnt, float4* vals, cudaStream_t s);

template <typename T>
int screen(const T* rx, long long rx_stride, int F, int n_train, int n_data, int M,
           kapsm_kernel_params p, unsigned* live, cudaStream_t s, bool tensor_cores = true) {
  if (F < 0 || n_train < 0 || n_data < 0 || M < 1 || !rx || !live) return KAPSM_ERR_INVALID;
  if (F == 0 || n_data == 0 || n_train == 0) return KAPSM_OK;
  if constexpr (sizeof(T) == 4) {
    // FP32: the tensor-core screen (screen_tc.cu) up to M = 64; FP64 (the
    // parity precision) keeps the SIMT screen with the FP64 threshold
    if (tensor_cores) {
      char* ws = reinterpret_cast<char*>(live);
      int* cnt = reinterpret_cast<int*>(ws + ws_live(F, n_train, n_data));
      float4* vals = reinterpret_cast<float4*>(
          ws + (ws_live(F, n_train, n_data) + ws_cnt(F, n_data) + 15) / 16 * 16);
      const int r = screen_tc(rx, rx_stride, F, n_train, n_data, M, p, live, cnt, vals, s);
      if (r != KAPSM_ERR_UNSUPPORTED) return r;
    }
  }
  if (M <= 4) return launch_screen<T, 4>(rx, rx_stride, F, n_train, n_data, M, p, live, s);
  if (M <= 8) return launch_screen<T, 8>(rx, rx_stride, F, n_train, n_data, M, p, live, s);
  if (M <= 16) return launch_screen<T, 16>(rx, rx_stride, F, n_train, n_data, M, p, live, s);
  if (M <= 32) return launch_screen<T, 32>(rx, rx_stride, F, n_train, n_data, M, p, live, s);
  if (M <= 64) return launch_screen<T, 64>(rx, rx_stride, F, n_train, n_data, M, p, live, s);
  return KAPSM_ERR_UNSUPPORTED;
}

template <typename T>
int finish(const T* rx, long long rx_stride, int F, int K, int n_train, int n_data, int M,
           const T* coeff, const T* theta, kapsm_kernel_params p, const T* points, int n_points,
           const unsigned char* tx, const unsigned* live, T* est, unsigned char* labels,
           unsigned long long* be, unsigned long long* se, cudaStream_t s) {
  if (F < 0 || K < 1 || n_train < 0 || n_data < 0 || M < 1 || !rx || !coeff || !theta ||
      !points || n_points < 1 || n_points > 64 || !live)
    return KAPSM_ERR_INVALID;
  if ((be || se) && !tx) return KAPSM_ERR_INVALID;
  if (F == 0 || n_data == 0) return KAPSM_OK;
#define KAPSM_FM(MTV) \
  return launch_finish<T, MTV>(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p, points, \
                               n_points, tx, live, est, labels, be, se, s)
  if (M <= 4) KAPSM_FM(4);
  if (M <= 8) KAPSM_FM(8);
  if (M <= 16) KAPSM_FM(16);
  if (M <= 32) KAPSM_FM(32);
  if (M <= 64) KAPSM_FM(64);
#undef KAPSM_FM
  return KAPSM_ERR_UNSUPPORTED;
}

}  // namespace kapsm

#define KAPSM_SCREEN_ENTRY(NAME, T)                                                           \
  extern "C" int NAME(const T* rx, long long rx_stride, int F, int n_train, int n_data, int M, \
                      kapsm_kernel_params p, unsigned* live, void* stream) {                   \
    return kapsm::screen<T>(rx, rx_stride, F, n_train, n_data, M, p, live,                     \
                            (cudaStream_t)stream);                                             \
  }
KAPSM_SCREEN_ENTRY(kapsm_detect_screen_f32, float)
KAPSM_SCREEN_ENTRY(kapsm_detect_screen_f64, double)

// Internal (tests, not in the public header): the FP32 SIMT screen, the
// reference point of the tensor-core classifier's superset property.
extern "C" int kapsm_internal_screen_simt_f32(const float* rx, long long rx_stride, int F,
                                              int n_train, int n_data, int M,
                                              kapsm_kernel_params p, unsigned* live,
                                              void* stream) {
  return kapsm::screen<float>(rx, rx_stride, F, n_train, n_data, M, p, live,
                              (cudaStream_t)stream, false);
}

#define KAPSM_FINISH_ENTRY(NAME, T)                                                             \
  extern "C" int NAME(const T* rx, long long rx_stride, int F, int K, int n_train, int n_data,  \
                      int M, const T* coeff, const T* theta, kapsm_kernel_params p,             \
                      const T* points, int n_points, int bits_per_symbol,                       \
                      const unsigned char* tx_labels, const unsigned* live, T* est,             \
                      unsigned char* labels, unsigned long long* bit_err,                       \
                      unsigned long long* sym_err, void* stream) {                              \
    (void)bits_per_symbol;                                                                      \
    return kapsm::finish<T>(rx, rx_stride, F, K, n_train, n_data, M, coeff, theta, p, points,   \
                            n_points, tx_labels, live, est, labels, bit_err, sym_err,           \
                            (cudaStream_t)stream);                                              \
  }
KAPSM_FINISH_ENTRY(kapsm_detect_finish_f32, float)
KAPSM_FINISH_ENTRY(kapsm_detect_finish_f64, double)

extern "C" long long kapsm_screen_workspace_bytes(int F, int n_train, int n_data) {
  if (F < 0 || n_train < 0 || n_data < 0) return -1;
  return (long long)kapsm::ws_bytes(F, n_train, n_data);
}
