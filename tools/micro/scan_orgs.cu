// Sphere-scan organisations microbenchmark (tool only; not the product path).
//   A  ray-stationary  : one ray per lane, scene from shared memory (warp-uniform LDS.128)
//   B  sphere-stationary: 32 spheres per lane resident in registers (1024 per warp), rays
//                         broadcast from shared memory (one ray per warp per step)
//   C  as B, rays from the constant bank (LDCU -> uniform-register FFMA2 operands)
// All evaluate the expanded-form filter value v = tc^2 + s1 (7 FFMA per sphere) and keep a
// running max, so the FMA work per sphere test is identical. Prints sphere tests / clk / SM.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kNS = 1024;        // spheres
constexpr int kNP = kNS / 64;    // pairs per lane in B/C (16)
constexpr int kRaysC = 1024;     // rays in the constant bank (32 KB)
__constant__ float c_rays[kRaysC * 8];

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

__global__ void __launch_bounds__(256, 3) kA(const float4* __restrict__ pairs, const float* __restrict__ rays, int nrays, float* out) {
  extern __shared__ float4 sp[];
  for (int i = threadIdx.x; i < kNS / 2 * 2; i += blockDim.x) sp[i] = pairs[i];
  __syncthreads();
  float acc = 0.f;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrays; r += gridDim.x * blockDim.x) {
    const float* R = rays + (size_t)(r & 4095) * 8;
    const float a1 = R[0], a2 = R[1], a3 = R[2], dx = R[3], dy = R[4], dz = R[5], b1 = R[6], cut = R[7];
    float vmax = -3e38f;
    for (int base = 0; base < kNS / 2; base += 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 a = sp[2 * (base + i)], b = sp[2 * (base + i) + 1];
        const float2 CX = make_float2(a.x, a.y), CY = make_float2(a.z, a.w), CZ = make_float2(b.x, b.y), K = make_float2(b.z, b.w);
        const float2 s1 = __ffma2_rn(CX, f2(a1), __ffma2_rn(CY, f2(a2), __ffma2_rn(CZ, f2(a3), K)));
        const float2 tc = __ffma2_rn(CX, f2(dx), __ffma2_rn(CY, f2(dy), __ffma2_rn(CZ, f2(dz), f2(b1))));
        const float2 v = __ffma2_rn(tc, tc, s1);
        vmax = fmaxf(vmax, fmaxf(v.x, v.y));
      }
      if (__any_sync(0xffffffffu, vmax >= cut)) acc += 1.f;
    }
    acc += vmax;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <bool kConst>
__global__ void __launch_bounds__(kConst ? 32 : 128) kB(const float4* __restrict__ pairs, const float* __restrict__ rays, int nrays, float* out) {
  __shared__ float sr[4][32][8];
  const int lane = threadIdx.x & 31, w = kConst ? 0 : threadIdx.x >> 5;  // C: one warp per CTA (uniform ray index)
  float2 CX[kNP], CY[kNP], CZ[kNP], K[kNP];
#pragma unroll
  for (int i = 0; i < kNP; ++i) {
    const float4 a = pairs[2 * (i * 32 + lane)], b = pairs[2 * (i * 32 + lane) + 1];
    CX[i] = make_float2(a.x, a.y); CY[i] = make_float2(a.z, a.w); CZ[i] = make_float2(b.x, b.y); K[i] = make_float2(b.z, b.w);
  }
  float acc = 0.f;
  const int wpb = kConst ? 1 : 4;
  const int warps = gridDim.x * wpb, gw = blockIdx.x * wpb + w;
  for (int r0 = gw * 32; r0 < nrays; r0 += warps * 32) {
    if (!kConst) {
#pragma unroll
      for (int c = 0; c < 8; ++c) sr[w][lane][c] = rays[(size_t)((r0 + lane) & 4095) * 8 + c];
      __syncwarp();
    }
    for (int j = 0; j < 32; ++j) {
      const float* R = kConst ? c_rays + ((r0 + j) & (kRaysC - 1)) * 8 : sr[w][j];
      const float a1 = R[0], a2 = R[1], a3 = R[2], dx = R[3], dy = R[4], dz = R[5], b1 = R[6], cut = R[7];
      float vmax = -3e38f;
#pragma unroll
      for (int i = 0; i < kNP; ++i) {
        const float2 s1 = __ffma2_rn(CX[i], f2(a1), __ffma2_rn(CY[i], f2(a2), __ffma2_rn(CZ[i], f2(a3), K[i])));
        const float2 tc = __ffma2_rn(CX[i], f2(dx), __ffma2_rn(CY[i], f2(dy), __ffma2_rn(CZ[i], f2(dz), f2(b1))));
        const float2 v = __ffma2_rn(tc, tc, s1);
        vmax = fmaxf(vmax, fmaxf(v.x, v.y));
      }
      if (__any_sync(0xffffffffu, vmax >= cut)) acc += 1.f;
      acc += vmax;
    }
    if (!kConst) __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float4* pairs; float* rays; float* out;
  cudaMalloc(&pairs, kNS * 16); cudaMalloc(&rays, 4096 * 32); cudaMalloc(&out, 1 << 24);
  float* h = new float[4096 * 8];
  for (int i = 0; i < 4096 * 8; ++i) h[i] = 0.001f * (i % 97) - 0.05f;
  for (int i = 0; i < 4096; ++i) h[i * 8 + 7] = 1e30f;  // cut: no candidates
  cudaMemcpy(rays, h, 4096 * 32, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_rays, h, kRaysC * 32);
  float* hp = new float[kNS * 4];
  for (int i = 0; i < kNS * 4; ++i) hp[i] = 0.01f * (i % 31);
  cudaMemcpy(pairs, hp, kNS * 16, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int nrays = 148 * 24 * 32 * 64;
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double tests = (double)nrays * kNS;
    printf("%-34s %.3f ms  %.2f tests/clk/SM  (%.1f%% of the FFMA2 peak 18.3 at 7 FMA/test)  %s\n", name, best,
           tests / (best * 1e-3) / sms / (clk * 1e3), 100.0 * tests / (best * 1e-3) / sms / (clk * 1e3) / (128.0 / 7.0),
           cudaGetErrorString(cudaGetLastError()));
  };
  cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, kNS * 16);
  run("A ray-stationary smem (3x256)", [&] { kA<<<sms * 3, 256, kNS * 16>>>(pairs, rays, nrays, out); });
  for (int bpm : {4, 6, 8}) {
    char nm[64];
    snprintf(nm, 64, "B sphere-stationary smem rays (%dx128)", bpm);
    run(nm, [&] { kB<false><<<sms * bpm, 128>>>(pairs, rays, nrays, out); });
    snprintf(nm, 64, "C sphere-stationary const rays (%dx128)", bpm);
    run(nm, [&] { kB<true><<<sms * bpm * 4, 32>>>(pairs, rays, nrays, out); });
  }
  return 0;
}
