// K3a on the 5th-generation tensor cores: the (pilot x payload) kernel screen
// of the detection (engine.py:137-147 restated as a dead/live classifier, see
// screen.cu) with its cross term x_p^H y_t computed by tcgen05.mma (TF32
// operands from shared memory, FP32 accumulators in TMEM).
//
// Per payload symbol t and pilot p of a frame the three realified Gaussian
// distances of the 2x2 kernel block are nx + ny - 2 Re c and nx + ny -+ 2 Im c,
// c = x_p^H y_t; the block is dead when even the smallest one underflows the
// FP32 exponential.  With realified rows in the rx layout (re, im interleaved
// per antenna), Re c = x . y and Im c = x . rot(y), rot(y) = (im, -re) per
// antenna, so one real GEMM A[pilots x 2M] . B[2 NT x 2M]^T gives both: B
// holds NT payload rows and their NT rotated copies (MMA N = 2 NT).
//
// TF32 keeps 10 mantissa bits, so the cross term carries an error of at most
// 2^-9 |x||y| <= 2^-10 (nx + ny) per component: a pair is declared live when
//      nx + ny - 2 max(Re c, |Im c|) < T0 + (nx + ny) / 128,   T0 = dead / inv2s,
// a margin of 4x that bound.  The classifier is therefore conservative (it can
// only add live pairs), and every live pair is recomputed exactly with
// explicit differences (kernels.py:187-191) -- here for the compact list, in
// detect_finish otherwise -- so the detector's outputs do not depend on TF32.
//
// CTA = NT payload symbols of one frame x all pilots:
//   * B (2 NT rows) and two M-tile buffers of A (128 pilots each) in shared
//     memory, K-major with the 128-byte swizzle (1024-byte atoms of 8 rows),
//     one atom column per 32 floats of the row (KC chunks);
//   * thread 0 issues KC x 4 MMAs (M = 128, N = 2 NT, K = 8) per pilot tile and
//     commits them to an mbarrier; the next tile's cp.async copies overlap;
//   * 8 epilogue warps read the accumulators (tcgen05.ld 32x32b.x32: warp w
//     reads TMEM lanes 32 (w % 4) .. +31 = 32 pilots, half of the columns),
//     test each (pilot, symbol) pair and ballot the results into the live-bit
//     words (bit = pilot, word per symbol) -- the word layout of screen.cu;
//   * the live words and the compact per-symbol lists go out as in screen.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kapsm_common.cuh"

namespace kapsm {

constexpr int TC_THREADS = 256;
constexpr int TC_MROWS = 128;            // pilots per MMA tile (M)
constexpr int TC_CAP = 8;                // == SC_CAP (screen.cu): list entries per symbol

// ---- tcgen05 / descriptor helpers ----
KAPSM_DEV unsigned long long umma_desc_sw128(unsigned saddr) {
  // K-major, SWIZZLE_128B: start >> 4 (bits 0-13), LBO (unused) = 1, SBO = 1024 B
  // between 8-row groups (bits 32-45), version 1 (bits 46-47), layout 2 (61-63)
  const unsigned lo = ((saddr >> 4) & 0x3FFFu) | (1u << 16);
  const unsigned hi = (1024u >> 4) | (1u << 14) | (2u << 29);
  return ((unsigned long long)hi << 32) | lo;
}

KAPSM_DEV void umma_tf32(unsigned tmem_d, unsigned long long a, unsigned long long b,
                         unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

KAPSM_DEV void umma_commit(unsigned mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(mbar) : "memory");
}

KAPSM_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
KAPSM_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
KAPSM_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

KAPSM_DEV void tmem_ld32(unsigned taddr, unsigned (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
KAPSM_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// TMA: one 3-D tile {32 floats, 128 rows, 1 frame} of the pilot rows into a
// 128-byte-swizzled shared buffer (the UMMA K-major SW128 layout), completing
// on an mbarrier
KAPSM_DEV void tma_load_3d(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2,
                           unsigned mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
      : "memory");
}
KAPSM_DEV void mbar_arrive_tx(unsigned mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
               : "memory");
}

KAPSM_DEV void sts_f4(unsigned a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// byte offset of 16-byte unit j (0..7) of row r inside a K chunk of 8-row
// 1024-byte atoms (the SWIZZLE_128B pattern: unit index XOR row-in-atom)
KAPSM_DEV unsigned sw128_off(int r, int j) {
  return (unsigned)((r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4));
}

// float4 number q (4 q .. 4 q + 3) of a row of n = 2M floats, zero beyond n
KAPSM_DEV float4 row_f4(const float* row, int q, int n, bool vec) {
  const int e = 4 * q;
  if (vec && e + 4 <= n) return __ldg(reinterpret_cast<const float4*>(row + e));
  float4 v;
  v.x = e < n ? row[e] : 0.f;
  v.y = e + 1 < n ? row[e + 1] : 0.f;
  v.z = e + 2 < n ? row[e + 2] : 0.f;
  v.w = e + 3 < n ? row[e + 3] : 0.f;
  return v;
}

template <int NT, int KC, bool GB = false>
struct TcSmem {
  static constexpr int B_BYTES = 2 * NT * 128 * KC;
  static constexpr int A_BYTES = TC_MROWS * 128 * KC;
  static constexpr int OFF_B = 0;
  static constexpr int OFF_A = B_BYTES;                  // two buffers
  static constexpr int OFF_BITS = OFF_A + 2 * A_BYTES;
  // GB: the live words go straight to global memory (long pilot blocks,
  // whose NW x NT words would not fit beside the tiles)
  static size_t bytes(int NW) {
    return 1024 + (size_t)OFF_BITS + (GB ? 0 : (size_t)NW * NT * 4) + NT * 4 + 96 + TC_MROWS * 4;
  }
};

template <int NT, int KC, bool GB>
__global__ void __launch_bounds__(TC_THREADS)
    detect_screen_tc_kernel(const float* __restrict__ rx, long long rx_stride, int n_train,
                            int n_data, int y_row0, int list_max_off, int M, float inv2s,
                            float dead, unsigned* __restrict__ live, int* __restrict__ cnt,
                            float4* __restrict__ vals, const __grid_constant__ CUtensorMap tmap,
                            int use_tma) {
  using L = TcSmem<NT, KC, GB>;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned base for the swizzle atoms
  const unsigned raw_s = smem_u32(smem_raw);
  const unsigned base_s = (raw_s + 1023u) & ~1023u;
  unsigned char* base = smem_raw + (base_s - raw_s);
  const int NW = (n_train + 31) / 32;
  const int f = blockIdx.y, t0 = blockIdx.x * NT;
  // live words [NW][NT] in shared memory, or (GB) in place in the output
  // [NW][n_data] (word w of symbol t0 + s at bits[w * BST + s])
  unsigned* lf = live + (long long)f * NW * n_data;
  unsigned* bits = GB ? lf + t0 : reinterpret_cast<unsigned*>(base + L::OFF_BITS);
  const long long BST = GB ? n_data : NT;
  float* nyb = reinterpret_cast<float*>(base + L::OFF_BITS + (GB ? 0 : (size_t)NW * NT * 4));
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(nyb + NT);
  unsigned long long* tbar = mbar + 1;                     // [2] TMA arrivals per A buffer
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(mbar + 3);
  float* ath = reinterpret_cast<float*>(mbar + 4);          // [128] pilot thresholds of a tile
  const unsigned sB = base_s + L::OFF_B, sA = base_s + L::OFF_A;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int D = 2 * M;
  const bool vec = (D % 4) == 0 && (rx_stride % 4) == 0 && ((size_t)rx & 15) == 0;
  const float* Xf = rx + (long long)f * rx_stride;
  const float* Yf = Xf + (long long)y_row0 * D;           // the "payload" rows
  // pilot tiles this CTA needs: all of them for the detection; for the
  // trainer's pilot screen (list_max_off < 0) only those holding pilots
  // p <= t + list_max_off of its rows (the lower triangle); the live words of
  // the skipped tiles are written as zeros
  const int n_mt_all = (n_train + TC_MROWS - 1) / TC_MROWS;
  const int n_mt = list_max_off < 0
                       ? max(0, min(n_mt_all, (t0 + NT - 1 + list_max_off) / TC_MROWS + 1))
                       : n_mt_all;

  if (tid == 0) {
    mbar_init(mbar, 1);
    mbar_init(tbar, 1);
    mbar_init(tbar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(2 * NT) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }

  // ---- B: NT payload rows (Re) and their rotations (Im), zero past n_data;
  //      a thread's loads are all issued before its stores (one memory
  //      latency per CTA instead of one per piece) ----
  {
    constexpr int PER = NT * KC * 8 / TC_THREADS;
    float4 v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = tid + i * TC_THREADS;
      const int r = e / (KC * 8), rem = e - r * (KC * 8), kc = rem >> 3, j = rem & 7;
      const int t = t0 + r;
      v[i] = t < n_data ? row_f4(Yf + (long long)t * D, kc * 8 + j, D, vec)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = tid + i * TC_THREADS;
      const int r = e / (KC * 8), rem = e - r * (KC * 8), kc = rem >> 3, j = rem & 7;
      const unsigned chunk = (unsigned)kc * (2 * NT) * 128;
      sts_f4(sB + chunk + sw128_off(r, j), v[i]);
      sts_f4(sB + chunk + sw128_off(NT + r, j), make_float4(v[i].y, -v[i].x, v[i].w, -v[i].z));
    }
  }

  // ---- A tile loader: pilots p0 .. p0 + 127 into buffer b ----
  auto load_a = [&](int mt, int b) {
    const int p0 = mt * TC_MROWS;
    const unsigned sa = sA + (unsigned)b * L::A_BYTES;
    if (use_tma) {                          // one thread: KC boxes of 128 rows x 128 bytes
      if (tid == 0) {
        const unsigned bar = smem_u32(tbar + b);
        mbar_arrive_tx(bar, (unsigned)(KC * TC_MROWS * 128));
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
          tma_load_3d(sa + (unsigned)kc * TC_MROWS * 128, &tmap, 32 * kc, p0, f, bar);
      }
      return;
    }
    for (int e = tid; e < TC_MROWS * KC * 8; e += TC_THREADS) {
      const int r = e / (KC * 8), rem = e - r * (KC * 8), kc = rem >> 3, j = rem & 7;
      const int p = p0 + r;
      const unsigned d = sa + (unsigned)kc * TC_MROWS * 128 + sw128_off(r, j);
      const float* src = Xf + (long long)p * D + 4 * (kc * 8 + j);
      if (p < n_train && vec && 4 * (kc * 8 + j) + 4 <= D) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
      } else {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p < n_train) v = row_f4(Xf + (long long)p * D, kc * 8 + j, D, vec);
        sts_f4(d, v);
      }
    }
    cp_async_commit();
  };
  if (n_mt > 0) load_a(0, 0);

  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = *tmem_slot;
  // symbol norms (scaled half, see the live test below)
  const float shrink = 0.5f * (1.0f - 1.0f / 128.0f);
  for (int r = tid; r < NT; r += TC_THREADS) {
    float s = 0.f;
#pragma unroll
    for (int kc = 0; kc < KC; ++kc)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = lds_f4(sB + (unsigned)kc * (2 * NT) * 128 + sw128_off(r, j));
        s = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, s))));
      }
    nyb[r] = shrink * s;
  }

  const float half_t0 = 0.5f * dead / inv2s;
  const int q = warp & 3;                   // TMEM lane quarter of this warp
  if constexpr (NT == 128) {
    // ---- transposed form: MMA M = 128 payload symbols (A = their rows, then
    //      their rotations), N = 128 pilots (B = the pilot tile) -> TMEM lane =
    //      symbol, column = pilot: Re c in columns 0..127, Im c in 128..255.
    //      A thread tests its symbol against 32 pilots per TMEM load and
    //      builds their live word in the same pass. ----
    const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(128 >> 3) << 17) |
                           ((unsigned)(128 >> 4) << 24);
    const int sym = 32 * q + lane;                                 // this thread's symbol
    float bsym = 0.f;                                              // (read after a barrier)
    const int ph = (warp >> 2) * 64;                               // its half of the pilots
    for (int mt = 0; mt < n_mt; ++mt) {
      if (use_tma) {
        while (!mbar_try_wait(tbar + (mt & 1), (unsigned)((mt >> 1) & 1))) {
        }
      } else {
        cp_async_wait<0>();
        fence_async_smem();
      }
      __syncthreads();                      // pilot tile visible; previous epilogue done
      if (mt == 0) bsym = nyb[sym];
      const unsigned sa = sA + (unsigned)(mt & 1) * L::A_BYTES;
      if (tid == 0) {
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < 2; ++h) {       // Re (payload rows), Im (rotated rows)
#pragma unroll
          for (int kc = 0; kc < KC; ++kc)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const unsigned long long a =
                  umma_desc_sw128(sB + kc * (2 * NT) * 128 + h * NT * 128 + ks * 32);
              const unsigned long long b = umma_desc_sw128(sa + kc * TC_MROWS * 128 + ks * 32);
              umma_tf32(tmem + 128 * h, a, b, idesc, (kc | ks) ? 1u : 0u);
            }
        }
        umma_commit(smem_u32(mbar));
      }
      // pilot thresholds of this tile while the MMAs run (the buffer of the next
      // tile was read by the previous MMA, complete by now)
      if (tid < TC_MROWS) {
        const int p = mt * TC_MROWS + tid;
        float sx = 0.f;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 v = lds_f4(sa + (unsigned)kc * TC_MROWS * 128 + sw128_off(tid, j));
            sx = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, sx))));
          }
        // live <=> max(Re c, |Im c|) > shrink (nx + ny) - T0 / 2
        ath[tid] = p < n_train ? fmaf(shrink, sx, -half_t0) : __int_as_float(0x7f800000);
      }
      if (mt + 1 < n_mt) load_a(mt + 1, (mt + 1) & 1);
      __syncthreads();                      // thresholds visible
      while (!mbar_try_wait(mbar, (unsigned)(mt & 1))) {
      }
      tc_fence_after();
      const unsigned lane_sel = (unsigned)(32 * q) << 16;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int pb = ph + 32 * c;                                // tile column = pilot
        unsigned re[32], im[32];
        tmem_ld32(tmem + lane_sel + (unsigned)pb, re);
        tmem_ld32(tmem + lane_sel + (unsigned)(128 + pb), im);
        float4 th4[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) th4[k] = lds_f4(smem_u32(ath + pb + 4 * k));
        tmem_wait_ld();
        const float* thp = reinterpret_cast<const float*>(th4);
        // the word in one pass: a warp meets a live pair in most chunks (32
        // symbols x 32 pilots), so an any-test + rebuild pass costs more
        unsigned w = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float m = fmaxf(__uint_as_float(re[j]), fabsf(__uint_as_float(im[j])));
          w |= m > thp[j] + bsym ? (1u << j) : 0u;
        }
        const int wrd = (mt * TC_MROWS + pb) >> 5;
        if (wrd < NW && (!GB || t0 + sym < n_data)) bits[wrd * BST + sym] = w;
      }
      tc_fence_before();
    }
  } else {
  // instruction descriptor: F32 accumulate, TF32 A and B, both K-major,
  // N = 2 NT (bits 17-22, >> 3), M = 128 (bits 24-28, >> 4)
  const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(2 * NT >> 3) << 17) |
                         ((unsigned)(TC_MROWS >> 4) << 24);
  constexpr int CH = NT / 64;               // 32-symbol column chunks per warp
  const int col0 = (warp >> 2) * (NT / 2);

  for (int mt = 0; mt < n_mt; ++mt) {
    if (use_tma) {
      while (!mbar_try_wait(tbar + (mt & 1), (unsigned)((mt >> 1) & 1))) {
      }
    } else {
      cp_async_wait<0>();
      fence_async_smem();
    }
    __syncthreads();                        // A[mt] visible; previous epilogue done with TMEM
    if (tid == 0) {
      tc_fence_after();
      const unsigned sa = sA + (unsigned)(mt & 1) * L::A_BYTES;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const unsigned long long a = umma_desc_sw128(sa + kc * TC_MROWS * 128 + ks * 32);
          const unsigned long long b = umma_desc_sw128(sB + kc * (2 * NT) * 128 + ks * 32);
          umma_tf32(tmem, a, b, idesc, (kc | ks) ? 1u : 0u);
        }
      umma_commit(smem_u32(mbar));
    }
    if (mt + 1 < n_mt) load_a(mt + 1, (mt + 1) & 1);

    // this lane's pilot norm (row 32q + lane of the tile) while the MMAs run
    const int prow = 32 * q + lane, p = mt * TC_MROWS + prow;
    float a_thr;
    {
      const unsigned sa = sA + (unsigned)(mt & 1) * L::A_BYTES;
      float s = 0.f;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = lds_f4(sa + (unsigned)kc * TC_MROWS * 128 + sw128_off(prow, j));
          s = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, s))));
        }
      // live <=> max(Re c, |Im c|) > shrink (nx + ny) - T0 / 2
      a_thr = p < n_train ? fmaf(shrink, s, -half_t0) : __int_as_float(0x7f800000);
    }
    while (!mbar_try_wait(mbar, (unsigned)(mt & 1))) {
    }
    tc_fence_after();
    const int wrd = mt * (TC_MROWS / 32) + q;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int cb = col0 + 32 * c;
      unsigned re[32], im[32];
      const unsigned lane_sel = (unsigned)(32 * q) << 16;
      tmem_ld32(tmem + lane_sel + (unsigned)cb, re);
      tmem_ld32(tmem + lane_sel + (unsigned)(NT + cb), im);
      tmem_wait_ld();
      unsigned mine = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float m = fmaxf(__uint_as_float(re[j]), fabsf(__uint_as_float(im[j])));
        const unsigned bj = __ballot_sync(0xffffffffu, m > a_thr + nyb[cb + j]);
        mine = lane == j ? bj : mine;
      }
      if (wrd < NW && (!GB || t0 + cb + lane < n_data)) bits[wrd * BST + cb + lane] = mine;
    }
    tc_fence_before();
  }
  }
  // live words of the skipped pilot tiles (pilot screen's upper triangle)
  for (int i = tid; i < (NW - n_mt * (TC_MROWS / 32)) * NT; i += TC_THREADS) {
    const int w = n_mt * (TC_MROWS / 32) + i / NT, sy = i % NT;
    if (!GB || t0 + sy < n_data) bits[w * BST + sy] = 0u;
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * NT)
                 : "memory");

  // ---- live words out (word-major, coalesced over the symbols) ----
  if (!GB) {
    for (int i = tid; i < NW * NT; i += TC_THREADS) {
      const int w = i / NT, tt = t0 + (i - w * NT);
      if (tt < n_data) lf[(long long)w * n_data + tt] = bits[i];
    }
  }
  // ---- compact list of each symbol's live pilots in pilot order (those
  //      with p <= t + list_max_off), kernel values from explicit differences
  //      (kernels.py:187-191); more than TC_CAP: count -1, the consumer
  //      recomputes from the words.  Phase 1: a thread per symbol gathers the
  //      indices; phase 2: every thread takes (symbol, entry) items. ----
  int* lp = reinterpret_cast<int*>(base + L::OFF_A);       // [NT][CAP] (A tiles are dead)
  int* lnum = lp + NT * TC_CAP;                            // [NT]
  for (int r = tid; r < NT; r += TC_THREADS) {
    const int t = t0 + r;
    int j = 0;
    if (t < n_data) {
      const int pmax = t + list_max_off;
      const int nwl = pmax < 0 ? 0 : min(NW, pmax / 32 + 1);   // words with w * 32 <= pmax
      for (int w0 = 0; w0 < nwl; w0 += 8) {
        unsigned bw[8];                     // 8 words in flight, then their bits
#pragma unroll
        for (int k = 0; k < 8; ++k) bw[k] = w0 + k < nwl ? bits[(w0 + k) * BST + r] : 0u;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          unsigned b = bw[k];
          while (b) {
            const int pp = (w0 + k) * 32 + __ffs(b) - 1;
            b &= b - 1;
            if (pp > pmax) break;
            if (j < TC_CAP) lp[r * TC_CAP + j] = pp;
            ++j;
          }
        }
      }
      cnt[(long long)f * n_data + t] = j <= TC_CAP ? j : -1;
    }
    lnum[r] = j <= TC_CAP ? j : 0;
  }
  __syncthreads();
  for (int it = tid; it < NT * TC_CAP; it += TC_THREADS) {
    // entry-major: the first entries of all NT symbols go to NT different
    // threads (lists are short: symbol-major put a symbol's entries, and
    // every eighth symbol, on one thread, one memory round trip after another)
    const int j = it / NT, r = it - j * NT;
    if (j >= lnum[r]) continue;
    const int t = t0 + r, pp = lp[r * TC_CAP + j];
    const float* x = Xf + (long long)pp * D;
    const float* y = Yf + (long long)t * D;
    float ea = 0.f, eb = 0.f, ec = 0.f;
    auto acc = [&](float xr, float xi, float yr, float yi) {
      float a0 = xr - yr, a1 = xi - yi;
      ea = fmaf(a0, a0, fmaf(a1, a1, ea));
      a0 = xr - yi; a1 = xi + yr;
      eb = fmaf(a0, a0, fmaf(a1, a1, eb));
      a0 = xr + yi; a1 = xi - yr;
      ec = fmaf(a0, a0, fmaf(a1, a1, ec));
    };
    if (vec) {
#pragma unroll 4
      for (int q = 0; q < D / 4; ++q) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(x) + q);
        const float4 yv = __ldg(reinterpret_cast<const float4*>(y) + q);
        acc(xv.x, xv.y, yv.x, yv.y);
        acc(xv.z, xv.w, yv.z, yv.w);
      }
    } else {
      for (int k = 0; k < M; ++k) acc(x[2 * k], x[2 * k + 1], y[2 * k], y[2 * k + 1]);
    }
    vals[((long long)f * n_data + t) * TC_CAP + j] =
        make_float4(exp_fast(-ea * inv2s), exp_fast(-eb * inv2s), exp_fast(-ec * inv2s),
                    __int_as_float(pp));
  }
}

// The 3-D tensor map {2M floats, rows per frame, frames} of rx for TMA loads of
// pilot tiles (box {32 floats, 128 rows, 1}, 128-byte swizzle); 0 when the
// layout does not allow it (rows not 16-byte multiples) -- the kernel then
// stages the tiles with cp.async.
static int make_pilot_map(CUtensorMap* map, const float* rx, long long rx_stride, int F, int M) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  memset(map, 0, sizeof(*map));
  const long long D = 2LL * M;
  if (!encode || D % 4 || rx_stride % D || rx_stride % 4 || ((size_t)rx & 15)) return 0;
  const cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)(rx_stride / D), (cuuint64_t)F};
  const cuuint64_t strides[2] = {(cuuint64_t)D * 4, (cuuint64_t)rx_stride * 4};
  const cuuint32_t box[3] = {32, (cuuint32_t)TC_MROWS, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(rx), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 1 : 0;
}

template <int NT, int KC>
static int launch_screen_tc(const float* rx, long long rx_stride, int F, int n_train, int n_data,
                            int y_row0, int list_max_off, int M, kapsm_kernel_params p,
                            unsigned* live, int* cnt, float4* vals, cudaStream_t s) {
  const int NW = (n_train + 31) / 32;
  const bool gb = TcSmem<NT, KC>::bytes(NW) > 227 * 1024;   // long pilot blocks (C4 full band)
  size_t smem = gb ? TcSmem<NT, KC, true>::bytes(NW) : TcSmem<NT, KC>::bytes(NW);
  // at least 112 KB: never co-resident with a latency-mode trainer CTA (120 KB),
  // so the concurrent screen does not slow a critical warp down (screen.cu)
  if (smem < 112 * 1024) smem = 112 * 1024;
  if (smem > 227 * 1024) return KAPSM_ERR_UNSUPPORTED;
  auto kern = gb ? detect_screen_tc_kernel<NT, KC, true> : detect_screen_tc_kernel<NT, KC, false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return KAPSM_ERR_CUDA;
  dim3 grid((n_data + NT - 1) / NT, F);
  CUtensorMap tmap;
  const int use_tma = make_pilot_map(&tmap, rx, rx_stride, F, M);
  kern<<<grid, TC_THREADS, smem, s>>>(rx, rx_stride, n_train, n_data, y_row0, list_max_off, M,
                                      (float)(1.0 / (2.0 * p.sigma_sq)), 88.0f, live, cnt, vals,
                                      tmap, use_tma);
  return status_from(cudaGetLastError());
}

// the tensor-core screen for M <= 64 (2M <= 128 floats per row) of the pilots
// against n_rows rows starting at row y_row0 of each frame (the payload for
// the detection; the pilots themselves for the trainer's live lists, which
// only need pilots p <= t + list_max_off of row t); KAPSM_ERR_UNSUPPORTED
// beyond (the caller keeps the SIMT screen)
int screen_tc_rows(const float* rx, long long rx_stride, int F, int n_train, int n_rows,
                   int y_row0, int list_max_off, int M, kapsm_kernel_params p, unsigned* live,
                   int* cnt, float4* vals, cudaStream_t s) {
#define KAPSM_TC(NT, KC)                                                                   \
  return launch_screen_tc<NT, KC>(rx, rx_stride, F, n_train, n_rows, y_row0, list_max_off, \
                                  M, p, live, cnt, vals, s)
  if (M <= 16) KAPSM_TC(128, 1);
  if (M <= 32) KAPSM_TC(128, 2);
  if (M <= 64) KAPSM_TC(64, 4);
#undef KAPSM_TC
  return KAPSM_ERR_UNSUPPORTED;
}

int screen_tc(const float* rx, long long rx_stride, int F, int n_train, int n_data, int M,
              kapsm_kernel_params p, unsigned* live, int* cnt, float4* vals, cudaStream_t s) {
  return screen_tc_rows(rx, rx_stride, F, n_train, n_data, n_train, 1 << 30, M, p, live, cnt,
                        vals, s);
}

}  // namespace kapsm
