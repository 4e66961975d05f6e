// K1: pilot sum-kernel Gram matrix (replaces the per-step window
// re-evaluation of ApsmTrainer._window_response, apsm.py:288-302).
//
// The 2x2 realified block of each (pilot p, pilot q) pair comes from complex
// arithmetic (apsm.py:156-182 realification), one thread per 2 x 2 pairs:
//   r1(x).r1(y) = r2(x).r2(y) = Re(x^H y),  r1(x).r2(y) = Im(x^H y) = -r2(x).r1(y)
//   ||r1(x)-r1(y)|| = ||r2(x)-r2(y)|| = ||x-y||,
//   ||r1(x)-r2(y)|| = ||x+iy||,  ||r2(x)-r1(y)|| = ||x-iy||.
// Distances use explicit differences (kernels.py:187-191), never the
// ||a||^2+||b||^2-2ab expansion, so near-coincident pilots keep full
// precision.  Only the upper-triangular tiles are computed; off-diagonal tiles
// also store their transpose (staged through shared memory), and inside a
// diagonal tile every sum is formed in an order that makes thread (q,p)
// reproduce thread (p,q)'s transpose bit for bit: the matrix is exactly
// symmetric.
#include "kapsm_common.cuh"

namespace kapsm {

constexpr int GRAM_TILE = 16;

// A CTA of 16 x 16 threads covers a 32 x 32 pilot tile, each thread a 2 x 2
// block of pairs (p0+ty+16a, q0+tx+16b): every staged element feeds 4 pairs;
// pilot norms are formed once per tile.  One thread's pair sums run over k
// in the same order for (p,q) and (q,p), so diagonal tiles are exactly
// symmetric; off-diagonal tiles store their transposed block.
constexpr int GRAM_T2 = 2 * GRAM_TILE;

template <typename T>
__global__ void __launch_bounds__(GRAM_TILE* GRAM_TILE)
    pilot_gram_kernel(const T* __restrict__ rx, long long rx_stride, int n_train, int M,
                       T w_l, T w_g, T inv2s, T* __restrict__ gram, long long ld,
                       long long gram_stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int rs = 2 * M + 1;                       // odd row stride: conflict-free
  T* xa = reinterpret_cast<T*>(smem_raw);        // [32][rs]
  T* xb = xa + GRAM_T2 * rs;                     // [32][rs]
  T* na = xb + GRAM_T2 * rs;                     // [32] pilot norms
  T* nb = na + GRAM_T2;
  const int f = blockIdx.z;
  const T* X = rx + (long long)f * rx_stride;
  const int nt = (n_train + GRAM_T2 - 1) / GRAM_T2;
  int tr = 0, rem = (int)blockIdx.x;
  while (rem >= nt - tr) { rem -= nt - tr; ++tr; }
  const int tcol = tr + rem;
  const int p0 = tr * GRAM_T2, q0 = tcol * GRAM_T2;
  const bool offdiag = tcol != tr;
  const int tid = threadIdx.y * GRAM_TILE + threadIdx.x;
  const int nthr = GRAM_TILE * GRAM_TILE;
  const int row_elems = 2 * M;
  for (int e = tid; e < GRAM_T2 * row_elems; e += nthr) {
    const int r = e / row_elems, c = e - r * row_elems;
    xa[r * rs + c] = (p0 + r < n_train) ? X[(long long)(p0 + r) * row_elems + c] : T(0);
    xb[r * rs + c] = (q0 + r < n_train) ? X[(long long)(q0 + r) * row_elems + c] : T(0);
  }
  __syncthreads();
  if (tid < 2 * GRAM_T2) {                       // norms, in the one-pair form's order
    const T* x = (tid < GRAM_T2 ? xa : xb) + (tid % GRAM_T2) * rs;
    T n = 0;
    for (int k = 0; k < M; ++k) n = fma(x[2 * k], x[2 * k], fma(x[2 * k + 1], x[2 * k + 1], n));
    (tid < GRAM_T2 ? na : nb)[tid % GRAM_T2] = n;
  }
  __syncthreads();
  const int ty = threadIdx.y, tx = threadIdx.x;
  T srr[2][2] = {}, sii[2][2] = {}, sri[2][2] = {}, sir[2][2] = {};
  {
    const T* x0 = xa + ty * rs;
    const T* x1 = xa + (ty + GRAM_TILE) * rs;
    const T* y0 = xb + tx * rs;
    const T* y1 = xb + (tx + GRAM_TILE) * rs;
#pragma unroll 4
    for (int k = 0; k < M; ++k) {
      const T xr[2] = {x0[2 * k], x1[2 * k]}, xi[2] = {x0[2 * k + 1], x1[2 * k + 1]};
      const T yr[2] = {y0[2 * k], y1[2 * k]}, yi[2] = {y0[2 * k + 1], y1[2 * k + 1]};
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          srr[a][b] = fma(xr[a], yr[b], srr[a][b]);
          sii[a][b] = fma(xi[a], yi[b], sii[a][b]);
          sri[a][b] = fma(xr[a], yi[b], sri[a][b]);
          sir[a][b] = fma(xi[a], yr[b], sir[a][b]);
        }
    }
  }
  T* G = gram + (long long)f * gram_stride;
  T kv[2][2][3];                                 // (k11, k12, k21) per pair
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int lp = ty + GRAM_TILE * a, lq = tx + GRAM_TILE * b;
      const T lin_re = srr[a][b] + sii[a][b];
      const T lin_12 = sri[a][b] - sir[a][b];
      const T lin_21 = sir[a][b] - sri[a][b];
      T g_a = 0, g_b = 0, g_c = 0;
      if (w_g != T(0)) {
        const T nn = na[lp] + nb[lq];
        const T dmin = nn - T(2) * fmax(lin_re, fmax(lin_12, lin_21));
        const T slack = nn * (sizeof(T) == 4 ? T(1e-5) : T(1e-12));
        const T dead = sizeof(T) == 4 ? T(104) : T(746);
        if ((dmin - slack) * inv2s < dead) {
          const T* x = xa + lp * rs;
          const T* y = xb + lq * rs;
          T d_a = 0, d_b = 0, d_c = 0;
          for (int k = 0; k < M; ++k) {
            const T xr = x[2 * k], xi = x[2 * k + 1], yr = y[2 * k], yi = y[2 * k + 1];
            T a0, a1;
            if constexpr (sizeof(T) == 4) {
              a0 = __fsub_rn(xr, yr); a1 = __fsub_rn(xi, yi);
              d_a = __fadd_rn(d_a, __fadd_rn(__fmul_rn(a0, a0), __fmul_rn(a1, a1)));
              a0 = __fsub_rn(xr, yi); a1 = __fadd_rn(xi, yr);
              d_b = __fadd_rn(d_b, __fadd_rn(__fmul_rn(a0, a0), __fmul_rn(a1, a1)));
              a0 = __fadd_rn(xr, yi); a1 = __fsub_rn(xi, yr);
              d_c = __fadd_rn(d_c, __fadd_rn(__fmul_rn(a0, a0), __fmul_rn(a1, a1)));
            } else {
              a0 = __dsub_rn(xr, yr); a1 = __dsub_rn(xi, yi);
              d_a = __dadd_rn(d_a, __dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1)));
              a0 = __dsub_rn(xr, yi); a1 = __dadd_rn(xi, yr);
              d_b = __dadd_rn(d_b, __dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1)));
              a0 = __dadd_rn(xr, yi); a1 = __dsub_rn(xi, yr);
              d_c = __dadd_rn(d_c, __dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1)));
            }
          }
          g_a = exp_acc(-d_a * inv2s);
          g_b = exp_acc(-d_b * inv2s);
          g_c = exp_acc(-d_c * inv2s);
        }
      }
      kv[a][b][0] = w_l * lin_re + w_g * g_a;
      kv[a][b][1] = w_l * lin_12 + w_g * g_b;
      kv[a][b][2] = w_l * lin_21 + w_g * g_c;
      const int p = p0 + lp, q = q0 + lq;
      if (p < n_train && q < n_train) {
        using V2 = typename Vec2<T>::type;
        V2 top, bot;
        top.x = kv[a][b][0]; top.y = kv[a][b][1];
        bot.x = kv[a][b][2]; bot.y = kv[a][b][0];
        *reinterpret_cast<V2*>(G + (long long)(2 * p) * ld + 2 * q) = top;
        *reinterpret_cast<V2*>(G + (long long)(2 * p + 1) * ld + 2 * q) = bot;
      }
    }
  if (!offdiag) return;
  // transposed 64 x 64 realified block through shared memory (coalesced rows)
  __syncthreads();
  constexpr int RT = 2 * GRAM_T2;
  T* tb = reinterpret_cast<T*>(smem_raw);        // [RT][RT + 1]
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int lp = 2 * (ty + GRAM_TILE * a), lq = 2 * (tx + GRAM_TILE * b);
      tb[lq * (RT + 1) + lp] = kv[a][b][0];
      tb[lq * (RT + 1) + lp + 1] = kv[a][b][2];
      tb[(lq + 1) * (RT + 1) + lp] = kv[a][b][1];
      tb[(lq + 1) * (RT + 1) + lp + 1] = kv[a][b][0];
    }
  __syncthreads();
  for (int e = tid; e < RT * RT; e += nthr) {
    const int r = e / RT, c = e % RT;
    const int gr = 2 * q0 + r, gc = 2 * p0 + c;
    if (gr < 2 * n_train && gc < 2 * n_train) G[(long long)gr * ld + gc] = tb[r * (RT + 1) + c];
  }
}

template <typename T>
int pilot_gram(const T* rx, long long rx_stride, int F, int n_train, int M,
               kapsm_kernel_params p, T* gram, long long ld, long long gram_stride,
               cudaStream_t s) {
  if (F < 0 || n_train < 0 || M < 1 || ld < 2LL * n_train || (ld & 1) || !rx || !gram)
    return KAPSM_ERR_INVALID;
  if (F == 0 || n_train == 0) return KAPSM_OK;
  const int nt = (n_train + GRAM_T2 - 1) / GRAM_T2;
  dim3 grid(nt * (nt + 1) / 2, 1, F), block(GRAM_TILE, GRAM_TILE);
  size_t smem = (2 * GRAM_T2 * (2 * (size_t)M + 1) + 2 * GRAM_T2) * sizeof(T);
  const size_t tsm = (size_t)(2 * GRAM_T2) * (2 * GRAM_T2 + 1) * sizeof(T);
  if (smem < tsm) smem = tsm;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(pilot_gram_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return KAPSM_ERR_CUDA;
  pilot_gram_kernel<T><<<grid, block, smem, s>>>(rx, rx_stride, n_train, M, (T)p.w_l,
                                                     (T)p.w_g, (T)(1.0 / (2.0 * p.sigma_sq)),
                                                     gram, ld, gram_stride);
  return status_from(cudaGetLastError());
}


// Generic variant for arbitrary realified sample rows (ApsmTrainer.observe on
// any real stream, apsm.py:304): samples F x (N x D), row-major.
template <typename T>
__global__ void __launch_bounds__(GRAM_TILE* GRAM_TILE)
    sample_gram_kernel(const T* __restrict__ S, long long s_stride, int N, int D, T w_l, T w_g,
                       T inv2s, T* __restrict__ gram, long long ld, long long gram_stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int rs = D | 1;                     // odd row stride: conflict-free
  T* sa = reinterpret_cast<T*>(smem_raw);   // [GRAM_TILE][rs]
  T* sb = sa + GRAM_TILE * rs;
  const int f = blockIdx.z;
  const T* Sf = S + (long long)f * s_stride;
  const int i0 = blockIdx.y * GRAM_TILE, j0 = blockIdx.x * GRAM_TILE;
  const int tid = threadIdx.y * GRAM_TILE + threadIdx.x;
  for (int e = tid; e < GRAM_TILE * D; e += GRAM_TILE * GRAM_TILE) {
    int r = e / D, c = e - r * D;
    sa[r * rs + c] = (i0 + r < N) ? Sf[(long long)(i0 + r) * D + c] : T(0);
    sb[r * rs + c] = (j0 + r < N) ? Sf[(long long)(j0 + r) * D + c] : T(0);
  }
  __syncthreads();
  const int i = i0 + threadIdx.y, j = j0 + threadIdx.x;
  if (i >= N || j >= N) return;
  const T* a = sa + threadIdx.y * rs;
  const T* b = sb + threadIdx.x * rs;
  T dot = T(0), d2 = T(0);
  for (int k = 0; k < D; ++k) {
    dot = fma(a[k], b[k], dot);
    const T e = a[k] - b[k];
    d2 = fma(e, e, d2);
  }
  T g = T(0);
  if (w_g != T(0)) g = exp_acc(-d2 * inv2s);
  gram[(long long)f * gram_stride + (long long)i * ld + j] = w_l * dot + w_g * g;
}

template <typename T>
int sample_gram(const T* S, long long s_stride, int F, int N, int D, kapsm_kernel_params p,
                T* gram, long long ld, long long gram_stride, cudaStream_t s) {
  if (F < 0 || N < 0 || D < 1 || ld < N || !S || !gram) return KAPSM_ERR_INVALID;
  if (F == 0 || N == 0) return KAPSM_OK;
  const int nt = (N + GRAM_TILE - 1) / GRAM_TILE;
  dim3 grid(nt, nt, F), block(GRAM_TILE, GRAM_TILE);
  size_t smem = 2 * GRAM_TILE * (size_t)(D | 1) * sizeof(T);
  if (smem > 227 * 1024) return KAPSM_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(sample_gram_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return KAPSM_ERR_CUDA;
  sample_gram_kernel<T><<<grid, block, smem, s>>>(S, s_stride, N, D, (T)p.w_l, (T)p.w_g,
                                                  (T)(1.0 / (2.0 * p.sigma_sq)), gram, ld,
                                                  gram_stride);
  return status_from(cudaGetLastError());
}

}  // namespace kapsm

extern "C" int kapsm_sample_gram_f32(const float* S, long long s_stride, int F, int N, int D,
                                     kapsm_kernel_params p, float* gram, long long ld,
                                     long long gram_stride, void* stream) {
  return kapsm::sample_gram<float>(S, s_stride, F, N, D, p, gram, ld, gram_stride,
                                   (cudaStream_t)stream);
}
extern "C" int kapsm_sample_gram_f64(const double* S, long long s_stride, int F, int N, int D,
                                     kapsm_kernel_params p, double* gram, long long ld,
                                     long long gram_stride, void* stream) {
  return kapsm::sample_gram<double>(S, s_stride, F, N, D, p, gram, ld, gram_stride,
                                    (cudaStream_t)stream);
}

extern "C" int kapsm_pilot_gram_f32(const float* rx, long long rx_stride, int F, int n_train,
                                    int M, kapsm_kernel_params p, float* gram, long long ld,
                                    long long gram_stride, void* stream) {
  return kapsm::pilot_gram<float>(rx, rx_stride, F, n_train, M, p, gram, ld, gram_stride,
                                  (cudaStream_t)stream);
}
extern "C" int kapsm_pilot_gram_f64(const double* rx, long long rx_stride, int F, int n_train,
                                    int M, kapsm_kernel_params p, double* gram, long long ld,
                                    long long gram_stride, void* stream) {
  return kapsm::pilot_gram<double>(rx, rx_stride, F, n_train, M, p, gram, ld, gram_stride,
                                   (cudaStream_t)stream);
}
