// Shared device helpers for the sm_100a APSM kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/kapsm_b200.h"

#define KAPSM_DEV __device__ __forceinline__

namespace kapsm {

template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

KAPSM_DEV float exp_fast(float x) {  // x <= 0; MUFU.EX2 path
  return exp2f(x * 1.4426950408889634f);
}
KAPSM_DEV double exp_fast(double x) { return exp(x); }
KAPSM_DEV float exp_acc(float x) { return expf(x); }
KAPSM_DEV double exp_acc(double x) { return exp(x); }

template <typename T>
KAPSM_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

KAPSM_DEV unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

KAPSM_DEV int ld_volatile(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "l"(__cvta_generic_to_shared(p)));
  return v;
}
KAPSM_DEV void st_volatile(int* p, int v) {
  asm volatile("st.volatile.shared.s32 [%0], %1;" ::"l"(__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
}

// Tagged value slots: (value, tag) published with ONE shared-memory store so a
// reader that sees the tag also sees the value (no reader-side fence).
template <typename T> struct Tagged;
template <> struct Tagged<float> {
  using slot_t = unsigned long long;
  static KAPSM_DEV void store(slot_t* p, float v, int tag) {
    unsigned long long w = ((unsigned long long)(unsigned)tag << 32) | __float_as_uint(v);
    asm volatile("st.volatile.shared.u64 [%0], %1;" ::"l"(__cvta_generic_to_shared(p)), "l"(w)
                 : "memory");
  }
  static KAPSM_DEV bool load(const slot_t* p, int tag, float& v) {
    unsigned long long w;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(w) : "l"(__cvta_generic_to_shared(p)));
    v = __uint_as_float((unsigned)(w & 0xffffffffu));
    return (int)(w >> 32) == tag;
  }
};
template <> struct Tagged<double> {
  struct __align__(16) slot_t { unsigned long long v, t; };
  static KAPSM_DEV void store(slot_t* p, double v, int tag) {
    asm volatile("st.volatile.shared.v2.u64 [%0], {%1, %2};" ::"l"(__cvta_generic_to_shared(p)),
                 "l"(__double_as_longlong(v)), "l"((unsigned long long)(unsigned)tag)
                 : "memory");
  }
  static KAPSM_DEV bool load(const slot_t* p, int tag, double& v) {
    unsigned long long a, b;
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];"
                 : "=l"(a), "=l"(b)
                 : "l"(__cvta_generic_to_shared(p)));
    v = __longlong_as_double((long long)a);
    return (int)b == tag;
  }
};

// cp.async of one scalar (4 or 8 bytes) global -> shared.
KAPSM_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
KAPSM_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

inline int status_from(cudaError_t e) { return e == cudaSuccess ? KAPSM_OK : KAPSM_ERR_CUDA; }

}  // namespace kapsm

namespace kapsm {

KAPSM_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// ---- named barriers (a subset of the CTA's warps) ----
KAPSM_DEV void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- mbarrier (tcgen05 commit targets, the trainers' pipelines) ----
KAPSM_DEV void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
KAPSM_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
KAPSM_DEV bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

}  // namespace kapsm

namespace kapsm {

// ---- explicit shared-space accesses (32-bit shared addresses; no generic
//      address materialisation on the trainer's critical path) ----
KAPSM_DEV void sts(unsigned a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
KAPSM_DEV void sts(unsigned a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
KAPSM_DEV float4 lds_f4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
KAPSM_DEV double2 lds_d2(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
KAPSM_DEV float lds_f(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
KAPSM_DEV double lds_d(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
template <typename T> KAPSM_DEV T lds_t(unsigned a);
template <> KAPSM_DEV float lds_t<float>(unsigned a) { return lds_f(a); }
template <> KAPSM_DEV double lds_t<double>(unsigned a) { return lds_d(a); }

// cp.async of one scalar to a 32-bit shared address
template <typename T>
KAPSM_DEV void cp_async_s(unsigned d, const T* gmem_src) {
  if (sizeof(T) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem_src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}

}  // namespace kapsm

namespace kapsm {

// opaque copy: the compiler can neither rematerialise nor fold the value
KAPSM_DEV unsigned opaque_u32(unsigned v) {
  unsigned r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
KAPSM_DEV void sts_i(unsigned a, int v) {
  asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
KAPSM_DEV int lds_i(unsigned a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
KAPSM_DEV float2 lds_f2(unsigned a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
template <typename T> KAPSM_DEV void lds_pair(unsigned a, T& x, T& y);
template <> KAPSM_DEV void lds_pair<float>(unsigned a, float& x, float& y) {
  const float2 v = lds_f2(a); x = v.x; y = v.y;
}
template <> KAPSM_DEV void lds_pair<double>(unsigned a, double& x, double& y) {
  const double2 v = lds_d2(a); x = v.x; y = v.y;
}

// tagged slots addressed by 32-bit shared addresses (layout as Tagged<T>)
KAPSM_DEV void st_tag(unsigned a, float v, int tag) {
  unsigned long long w = ((unsigned long long)(unsigned)tag << 32) | __float_as_uint(v);
  asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(a), "l"(w) : "memory");
}
KAPSM_DEV void st_tag(unsigned a, double v, int tag) {
  asm volatile("st.volatile.shared.v2.u64 [%0], {%1, %2};" ::"r"(a), "l"(__double_as_longlong(v)),
               "l"((unsigned long long)(unsigned)tag)
               : "memory");
}
KAPSM_DEV bool ld_tag(unsigned a, int tag, float& v) {
  unsigned long long w;
  asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(w) : "r"(a) : "memory");
  v = __uint_as_float((unsigned)(w & 0xffffffffu));
  return (int)(w >> 32) == tag;
}
KAPSM_DEV bool ld_tag(unsigned a, int tag, double& v) {
  unsigned long long x, t;
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(t) : "r"(a) : "memory");
  v = __longlong_as_double((long long)x);
  return (int)t == tag;
}

}  // namespace kapsm

namespace kapsm {
KAPSM_DEV bool mbar_try_wait_s(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
}  // namespace kapsm

namespace kapsm {
// tagged slot read without the tag test (the caller compares later)
KAPSM_DEV void ld_tagged(unsigned a, float& v, int& tag) {
  unsigned long long w;
  asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(w) : "r"(a) : "memory");
  v = __uint_as_float((unsigned)(w & 0xffffffffu));
  tag = (int)(w >> 32);
}
KAPSM_DEV void ld_tagged(unsigned a, double& v, int& tag) {
  unsigned long long x, t;
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(t) : "r"(a) : "memory");
  v = __longlong_as_double((long long)x);
  tag = (int)t;
}
}  // namespace kapsm

namespace kapsm {
// loads of shared data that is immutable while they run (no volatile, no
// memory clobber: the compiler may hoist and schedule them freely)
KAPSM_DEV float lds_nv(unsigned a, float) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
KAPSM_DEV double lds_nv(unsigned a, double) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
KAPSM_DEV void lds_nv_pair(unsigned a, float& x, float& y) {
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
}
KAPSM_DEV void lds_nv_pair(unsigned a, double& x, double& y) {
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
// warp-wide vote without the compiler's divergence guard (callers are converged)
KAPSM_DEV bool vote_all(bool p) {
  unsigned r;
  asm volatile(
      "{\n\t.reg .pred a, b;\n\t"
      "setp.ne.u32 a, %1, 0;\n\t"
      "vote.sync.all.pred b, a, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, b;\n\t}"
      : "=r"(r)
      : "r"((unsigned)p));
  return r != 0;
}
}  // namespace kapsm

namespace kapsm {
// ---- thread-block clusters / distributed shared memory ----
KAPSM_DEV unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same offset in CTA `rank` of this cluster
KAPSM_DEV unsigned map_rank(unsigned local_addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
KAPSM_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// tagged stores through a shared::cluster address (local or a peer CTA)
KAPSM_DEV void st_tag_cl(unsigned a, float v, int tag) {
  unsigned long long w = ((unsigned long long)(unsigned)tag << 32) | __float_as_uint(v);
  asm volatile("st.volatile.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(w) : "memory");
}
KAPSM_DEV void st_tag_cl(unsigned a, double v, int tag) {
  asm volatile("st.volatile.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(a),
               "l"(__double_as_longlong(v)), "l"((unsigned long long)(unsigned)tag)
               : "memory");
}
KAPSM_DEV void st_cl_s32(unsigned a, int v) {
  asm volatile("st.volatile.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
}  // namespace kapsm

namespace kapsm {
KAPSM_DEV void red_or_cl(unsigned a, int v) {
  asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
KAPSM_DEV int ld_cl_s32(unsigned a) {
  int v;
  asm volatile("ld.volatile.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
}  // namespace kapsm

namespace kapsm {
template <typename T> KAPSM_DEV void lds_quad(unsigned a, T (&v)[4]);
template <> KAPSM_DEV void lds_quad<float>(unsigned a, float (&v)[4]) {
  const float4 q = lds_f4(a);
  v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
}
template <> KAPSM_DEV void lds_quad<double>(unsigned a, double (&v)[4]) {
  const double2 p = lds_d2(a), q = lds_d2(a + 16);
  v[0] = p.x; v[1] = p.y; v[2] = q.x; v[3] = q.y;
}
// Live early Gaussian terms per pilot row (train_wide.cu builds them; both
// trainers read them): count, then up to KAPSM_LIVE_CAP (column, value) pairs.
constexpr int KAPSM_LIVE_CAP = 32;
template <typename T>
struct LiveLists {
  void* ws;
  int* cnt;
  int* idx;
  T* val;
};
template <typename T>
int build_live_lists(const T* rx, long long rx_stride, const T* samples, long long samples_stride,
                     int dim, int F, int Np, int gap, kapsm_kernel_params p, cudaStream_t s,
                     LiveLists<T>& ll);
}  // namespace kapsm
