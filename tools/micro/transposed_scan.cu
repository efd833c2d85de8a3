// Transposed sphere scan microbenchmark: lanes = spheres (a pair per lane), the warp walks R
// rays whose parameters are warp-uniform (uniform registers), vs the current lanes = rays layout.
// Tool only: decides whether the scan layout is worth changing.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int R>
__global__ void __launch_bounds__(256) k_transposed(const float4* __restrict__ pairs_g, int n_pairs, const float* __restrict__ rays,
                                                     int n_groups, int* out) {
  extern __shared__ float4 sp[];
  for (int i = threadIdx.x; i < 2 * n_pairs; i += blockDim.x) sp[i] = pairs_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int hits = 0;
  for (int g = warp; g < n_groups; g += nwarps) {
    float a1[R], a2[R], a3[R], d1[R], d2[R], d3[R], b1[R], cut[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float* q = rays + (size_t)(g * R + r) * 8;
      a1[r] = __shfl_sync(0xffffffff, q[0], 0); a2[r] = __shfl_sync(0xffffffff, q[1], 0);
      a3[r] = __shfl_sync(0xffffffff, q[2], 0); d1[r] = __shfl_sync(0xffffffff, q[3], 0);
      d2[r] = __shfl_sync(0xffffffff, q[4], 0); d3[r] = __shfl_sync(0xffffffff, q[5], 0);
      b1[r] = __shfl_sync(0xffffffff, q[6], 0); cut[r] = __shfl_sync(0xffffffff, q[7], 0);
    }
    for (int c = 0; c < n_pairs / 32; ++c) {
      const float4 A = sp[2 * (c * 32 + lane)], B = sp[2 * (c * 32 + lane) + 1];
      const float2 CX = make_float2(A.x, A.y), CY = make_float2(A.z, A.w), CZ = make_float2(B.x, B.y), K = make_float2(B.z, B.w);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float2 s1 = __ffma2_rn(CX, make_float2(a1[r], a1[r]), __ffma2_rn(CY, make_float2(a2[r], a2[r]), __ffma2_rn(CZ, make_float2(a3[r], a3[r]), K)));
        const float2 tc = __ffma2_rn(CX, make_float2(d1[r], d1[r]), __ffma2_rn(CY, make_float2(d2[r], d2[r]), __ffma2_rn(CZ, make_float2(d3[r], d3[r]), make_float2(b1[r], b1[r]))));
        const float2 v = __ffma2_rn(tc, tc, s1);
        const bool cand = fmaxf(v.x, v.y) >= cut[r];
        if (__any_sync(0xffffffff, cand)) hits += cand ? 1 : 0;
      }
    }
  }
  if (hits == 0x7fffffff) out[0] = hits;
}

__global__ void __launch_bounds__(256) k_lanes_rays(const float4* __restrict__ pairs_g, int n_pairs, const float* __restrict__ rays,
                                                    int n_rays, int* out) {
  extern __shared__ float4 sp[];
  for (int i = threadIdx.x; i < 2 * n_pairs; i += blockDim.x) sp[i] = pairs_g[i];
  __syncthreads();
  int hits = 0;
  const int nthreads = gridDim.x * blockDim.x;
  for (int ray = blockIdx.x * blockDim.x + threadIdx.x; ray < n_rays; ray += nthreads) {
    const float* q = rays + (size_t)ray * 8;
    const float2 A1 = make_float2(q[0], q[0]), A2 = make_float2(q[1], q[1]), A3 = make_float2(q[2], q[2]);
    const float2 D1 = make_float2(q[3], q[3]), D2 = make_float2(q[4], q[4]), D3 = make_float2(q[5], q[5]);
    const float2 B1 = make_float2(q[6], q[6]);
    const float cut = q[7];
    for (int base = 0; base < n_pairs; base += 8) {
      float vmax = -3e38f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 a = sp[2 * (base + i)], b = sp[2 * (base + i) + 1];
        const float2 CX = make_float2(a.x, a.y), CY = make_float2(a.z, a.w), CZ = make_float2(b.x, b.y), K = make_float2(b.z, b.w);
        const float2 s1 = __ffma2_rn(CX, A1, __ffma2_rn(CY, A2, __ffma2_rn(CZ, A3, K)));
        const float2 tc = __ffma2_rn(CX, D1, __ffma2_rn(CY, D2, __ffma2_rn(CZ, D3, B1)));
        const float2 v = __ffma2_rn(tc, tc, s1);
        vmax = fmaxf(vmax, fmaxf(v.x, v.y));
      }
      if (__any_sync(0xffffffff, vmax >= cut)) hits++;
    }
  }
  if (hits == 0x7fffffff) out[0] = hits;
}

int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int n_pairs = 512, n_rays = 1 << 20;
  float4* pg; CK(cudaMalloc(&pg, 2 * n_pairs * sizeof(float4)));
  float* rays; CK(cudaMalloc(&rays, (size_t)n_rays * 8 * sizeof(float)));
  float4 hp[2 * 512]; for (int i = 0; i < 2 * n_pairs; ++i) hp[i] = make_float4(0.1f * i, 0.2f, 0.3f, -1e30f);
  CK(cudaMemcpy(pg, hp, sizeof hp, cudaMemcpyHostToDevice));
  CK(cudaMemset(rays, 0, (size_t)n_rays * 8 * sizeof(float)));
  int* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const size_t smem = 2 * n_pairs * sizeof(float4);
  double tests = (double)n_rays * 2 * n_pairs;
  auto timeit = [&](auto launch, const char* nm) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf("%-26s %.3f ms  %.2f tests/clk/SM (FFMA2 peak 18.3 at 7 FMA/test)  err=%s\n", nm, best, tests / (best * 1e-3) / sms / (clk * 1e3), cudaGetErrorString(cudaGetLastError()));
  };
  for (int bps : {2, 3, 4}) {
    const int grid = sms * bps;
    timeit([&] { k_lanes_rays<<<grid, 256, smem>>>(pg, n_pairs, rays, n_rays, out); }, bps == 2 ? "lanes=rays (2 CTA/SM)" : bps == 3 ? "lanes=rays (3 CTA/SM)" : "lanes=rays (4 CTA/SM)");
    timeit([&] { k_transposed<4><<<grid, 256, smem>>>(pg, n_pairs, rays, n_rays / 4, out); }, "transposed R=4");
    timeit([&] { k_transposed<8><<<grid, 256, smem>>>(pg, n_pairs, rays, n_rays / 8, out); }, "transposed R=8");
  }
  return 0;
}
