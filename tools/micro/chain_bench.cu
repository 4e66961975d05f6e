// Microbenchmark: cycles per step of the bare APSM critical-warp chain
// (beta -> broadcast -> window dot over 24 lanes), one warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void chain(float* out, long long* cyc, int steps) {
  __shared__ __align__(16) float dv[64];
  const int x = threadIdx.x;
  float row[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) row[l] = 0.001f * ((l * 7 + x) % 13);
  float Y = 0.1f * x, qi = 0.01f, qbm = 0.02f, qbp = 0.03f;
  unsigned base = (unsigned)__cvta_generic_to_shared(dv);
  long long t0 = clock64();
  for (int n = 0; n < steps; n += 2) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float v1 = fmaf(-qi, Y, qbm), v2 = fmaf(-qi, Y, qbp);
      const float delta = fmaxf(v1, 0.f) + fminf(v2, 0.f);
      if (V & 4) {            // shuffle broadcast
        float a[8] = {Y, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int l = 0; l < 24; ++l) a[l & 7] = fmaf(__shfl_sync(0xffffffffu, delta, l), row[l], a[l & 7]);
        Y = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
        continue;
      }
      const unsigned dvb = base + h * 128;
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(dvb + 4 * x), "f"(delta) : "memory");
      asm volatile("bar.warp.sync 0xffffffff;" ::: "memory");
      float4 w[6];
#pragma unroll
      for (int b = 0; b < 6; ++b)
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(w[b].x), "=f"(w[b].y), "=f"(w[b].z), "=f"(w[b].w) : "r"(dvb + 16 * b) : "memory");
      if (V & 2) {            // 8 accumulators
        float a[8] = {Y, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 6; ++b) {
          a[(4 * b) & 7] = fmaf(w[b].x, row[4 * b], a[(4 * b) & 7]);
          a[(4 * b + 1) & 7] = fmaf(w[b].y, row[4 * b + 1], a[(4 * b + 1) & 7]);
          a[(4 * b + 2) & 7] = fmaf(w[b].z, row[4 * b + 2], a[(4 * b + 2) & 7]);
          a[(4 * b + 3) & 7] = fmaf(w[b].w, row[4 * b + 3], a[(4 * b + 3) & 7]);
        }
        Y = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
      } else if (V & 8) {     // 12 accumulators (depth 2)
        float a[12] = {Y, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 6; ++b) {
          a[(4 * b) % 12] = fmaf(w[b].x, row[4 * b], a[(4 * b) % 12]);
          a[(4 * b + 1) % 12] = fmaf(w[b].y, row[4 * b + 1], a[(4 * b + 1) % 12]);
          a[(4 * b + 2) % 12] = fmaf(w[b].z, row[4 * b + 2], a[(4 * b + 2) % 12]);
          a[(4 * b + 3) % 12] = fmaf(w[b].w, row[4 * b + 3], a[(4 * b + 3) % 12]);
        }
        Y = (((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]))) + ((a[8] + a[9]) + (a[10] + a[11]));
      } else {
        float a0 = Y, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
        for (int b = 0; b < 6; ++b) {
          a0 = fmaf(w[b].x, row[4 * b], a0); a1 = fmaf(w[b].y, row[4 * b + 1], a1);
          a2 = fmaf(w[b].z, row[4 * b + 2], a2); a3 = fmaf(w[b].w, row[4 * b + 3], a3);
        }
        Y = (a0 + a1) + (a2 + a3);
      }
    }
  }
  long long t1 = clock64();
  out[x] = Y;
  if (x == 0) cyc[0] = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  const int steps = 4096;
  auto run = [&](auto k, const char* name) {
    for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, c, steps);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %.1f cycles/step\n", name, (double)h / steps);
  };
  run(chain<0>, "smem, 4 acc");
  run(chain<2>, "smem, 8 acc");
  run(chain<8>, "smem, 12 acc");
  run(chain<4>, "shfl x24, 8 acc");
  return 0;
}
