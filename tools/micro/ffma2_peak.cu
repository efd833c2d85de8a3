// Measured FP32 peak for bench.py's roofline (SURVEY §8(d).2 "measure it in the same run"):
// dependent FFMA2 (packed f32x2) chains on every SM, 8 independent chains per thread, 8 CTAs x
// 256 threads per SM. Prints one JSON line: best TFLOP/s over the repetitions (2 flops per FMA
// lane) and the launch geometry. Runs for ~0.3-0.5 s so nvidia-smi can sample the clock under
// FP32 load. Measurement tool only: not part of the product path.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_peak ffma2_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_ffma2(float* out, int iters, float b0, float c0) {
  float2 a[kChains], b[kChains], c[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    a[i] = make_float2(threadIdx.x * 1e-3f + i, threadIdx.x * 2e-3f + i);
    b[i] = make_float2(b0 + i * 1e-7f, b0 - i * 1e-7f);
    c[i] = make_float2(c0 - i * 1e-7f, c0 + i * 1e-7f);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < kChains; ++i) a[i] = __ffma2_rn(a[i], b[i], c[i]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678f) out[0] = s;  // keeps the chains live
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 20;
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float* d;
  CK(cudaMalloc(&d, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  const double flops = 2.0 * 2.0 * blocks * threads * (double)iters * 16 * kChains;  // FFMA2 = 2 FMA = 4 flops
  k_ffma2<<<blocks, threads>>>(d, iters, 0.999f, 0.001f);  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f, sum = 0.f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    k_ffma2<<<blocks, threads>>>(d, iters, 0.999f, 0.001f);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
    sum += ms;
  }
  printf("{\"tflops\": %.4f, \"tflops_mean\": %.4f, \"best_ms\": %.4f, \"reps\": %d, \"sms\": %d, "
         "\"grid\": \"%d x %d, 8 FFMA2 chains per thread\"}\n",
         flops / (best * 1e-3) / 1e12, flops / (sum / reps * 1e-3) / 1e12, best, reps, sms, blocks, threads);
  return 0;
}
