// FFMA2 operand-pattern microbenchmark: does a scalar-broadcast multiplicand (the ray parameter
// in the sphere scan: FFMA2 Rd, Rpair, Rscalar.F32, Racc) issue at the same rate as all-pair
// operands? Tool only.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kC = 8;
template <int kMode>
__global__ void k(float* out, int iters, float s0) {
  float2 a[kC], b[kC];
  float sc[kC];
#pragma unroll
  for (int i = 0; i < kC; ++i) {
    a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    b[i] = make_float2(s0 + i * 1e-7f, s0 - i * 1e-7f);
    sc[i] = s0 + i * 3e-7f + threadIdx.x * 1e-9f;  // per-lane (vector register) scalar
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < kC; ++i) {
        if (kMode == 0) a[i] = __ffma2_rn(b[i], a[i], a[(i + 1) % kC]);                 // pair x pair + pair
        if (kMode == 1) a[i] = __ffma2_rn(b[i], make_float2(sc[i], sc[i]), a[i]);         // pair x scalar + pair
        if (kMode == 2) a[i] = __ffma2_rn(b[(i + u) % kC], make_float2(sc[i], sc[i]), a[i]);  // rotating pair x scalar
        if (kMode == 3) a[i] = __ffma2_rn(b[i], make_float2(sc[u % kC], sc[u % kC]), a[i]);   // same scalar for all chains
        if (kMode == 4) {  // FFMA2 chain + independent scalar FFMA chain (does scalar FFMA co-issue on the lite pipe?)
          a[i] = __ffma2_rn(b[i], make_float2(sc[i], sc[i]), a[i]);
          sc[i] = fmaf(sc[i], 1.0001f, 0.5f);
        }
        if (kMode == 5) {  // 2 FFMA2 + 1 scalar FFMA
          a[i] = __ffma2_rn(b[i], make_float2(sc[i], sc[i]), a[i]);
          b[i] = __ffma2_rn(a[i], make_float2(sc[i], sc[i]), b[i]);
          sc[i] = fmaf(sc[i], 1.0001f, 0.5f);
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kC; ++i) s += a[i].x + a[i].y + sc[i] + b[i].x;
  if (s == 12345.678f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 2048;
  auto run = [&](auto kern, const char* name, double per = 2.0) {
    const double fmas = per * blocks * threads * iters * 16 * kC;
    kern<<<blocks, threads>>>(d, iters, 0.999f);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); kern<<<blocks, threads>>>(d, iters, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-28s %.3f ms  %.1f FMA-lanes/clk/SM\n", name, best, fmas / (best * 1e-3) / sms / (clk * 1e3));
  };
  run(k<0>, "pair*pair+pair");
  run(k<1>, "pair*scalar+pair");
  run(k<2>, "rot pair*scalar+pair");
  run(k<3>, "pair*shared-scalar+pair");
  run(k<4>, "FFMA2 + scalar FFMA-imm", 3.0);
  run(k<5>, "2 FFMA2 + scalar FFMA-imm", 5.0);
  return 0;
}
