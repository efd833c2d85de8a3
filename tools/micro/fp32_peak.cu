// FP32 issue-rate microbenchmarks for the ray-sphere hot loop on sm_100a.
//
// Measures, on all SMs:
//   1. FFMA dependent chains, 3 distinct register operands      -> FP32 FMA lanes / clk / SM
//   2. FFMA with an immediate operand                            -> same, imm form
//   3. FFMA2 (packed f32x2) chains                               -> FMA lanes / clk / SM
//   4. prototype reject-path sphere loops (scene in __constant__ vs shared, scalar vs FFMA2)
//      -> sphere tests / clk / SM
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o fp32_peak fp32_peak.cu
// Tool only: not part of the product path.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void k_ffma_reg(float* out, int iters, float b0, float c0) {
  float a[kChains], b[kChains], c[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { a[i] = threadIdx.x * 1e-3f + i; b[i] = b0 + i * 1e-7f; c[i] = c0 - i * 1e-7f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < kChains; ++i) a[i] = fmaf(a[i], b[i], c[i]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 12345.678f) out[0] = s;
}

__global__ void k_ffma_imm(float* out, int iters) {
  float a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < kChains; ++i) a[i] = fmaf(a[i], 0.999f, 0.001f);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 12345.678f) out[0] = s;
}

__global__ void k_ffma2(float* out, int iters, float b0, float c0) {
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
  if (s == 12345.678f) out[0] = s;
}

__global__ void k_dfma(double* out, int iters, double b0, double c0) {
  double a[kChains], b[kChains], c[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { a[i] = threadIdx.x * 1e-3 + i; b[i] = b0 + i * 1e-7; c[i] = c0 - i * 1e-7; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < kChains; ++i) a[i] = fma(a[i], b[i], c[i]);
    }
  }
  double s = 0.;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

// ---- prototype sphere loops -------------------------------------------------------------
constexpr int kMaxS = 2048;
__constant__ float4 c_sph[kMaxS];         // cx, cy, cz, r^2
__constant__ float4 c_pair[kMaxS];        // pair p: [2p] = (cxA, cxB, cyA, cyB), [2p+1] = (czA, czB, r2A, r2B)

struct Ray { float ox, oy, oz, dx, dy, dz; };

__device__ __forceinline__ void make_ray(int gid, Ray& r) {
  // pseudo-random primary-like direction toward +z
  uint32_t h = gid * 2654435761u;
  float u = ((h >> 8) & 0xffff) / 65535.f - 0.5f;
  float v = ((h >> 20) & 0xfff) / 4095.f - 0.5f;
  float inv = rsqrtf(u * u + v * v + 1.f);
  r.ox = 0.f; r.oy = 0.f; r.oz = 0.f; r.dx = u * inv; r.dy = v * inv; r.dz = inv;
}

// basis-projection reject test: x' = (c-o).u1, y' = (c-o).u2, disc = r2 - x'^2 - y'^2
__device__ __forceinline__ void basis(const Ray& r, float& u1x, float& u1y, float& u1z,
                                      float& u2x, float& u2y, float& u2z) {
  float sgn = copysignf(1.f, r.dz);
  float a = -1.f / (sgn + r.dz);
  float b = r.dx * r.dy * a;
  u1x = 1.f + sgn * r.dx * r.dx * a; u1y = sgn * b; u1z = -sgn * r.dx;
  u2x = b; u2y = sgn + r.dy * r.dy * a; u2z = -r.dy;
}

template <bool kSmem>
__global__ void k_sphere_scalar(int* out, int n, int rays_per_thread) {
  __shared__ float4 s_sph[kMaxS];
  if (kSmem) { for (int i = threadIdx.x; i < n; i += blockDim.x) s_sph[i] = c_sph[i]; __syncthreads(); }
  int hits = 0;
  for (int rr = 0; rr < rays_per_thread; ++rr) {
    Ray r; make_ray((blockIdx.x * blockDim.x + threadIdx.x) * rays_per_thread + rr, r);
    float u1x, u1y, u1z, u2x, u2y, u2z; basis(r, u1x, u1y, u1z, u2x, u2y, u2z);
    float ou1 = -(r.ox * u1x + r.oy * u1y + r.oz * u1z);
    float ou2 = -(r.ox * u2x + r.oy * u2y + r.oz * u2z);
    float od = -(r.ox * r.dx + r.oy * r.dy + r.oz * r.dz);
    float tbest = 1e30f; int best = -1;
#pragma unroll 4
    for (int k = 0; k < n; ++k) {
      float4 s = kSmem ? s_sph[k] : c_sph[k];
      float x = fmaf(s.x, u1x, fmaf(s.y, u1y, fmaf(s.z, u1z, ou1)));
      float y = fmaf(s.x, u2x, fmaf(s.y, u2y, fmaf(s.z, u2z, ou2)));
      float disc = fmaf(-x, x, fmaf(-y, y, s.w));
      if (disc >= 0.f) {
        float tc = fmaf(s.x, r.dx, fmaf(s.y, r.dy, fmaf(s.z, r.dz, od)));
        float q = disc * rsqrtf(disc);
        float t0 = tc - q, t1 = tc + q;
        float t = t0 >= 1e-4f ? t0 : t1;
        if (t >= 1e-4f && t < tbest) { tbest = t; best = k; }
      }
    }
    hits += best;
  }
  if (hits == 0x7fffffff) out[0] = hits;
}

template <bool kSmem>
__global__ void k_sphere_pair(int* out, int n, int rays_per_thread) {
  __shared__ float4 s_pair[kMaxS];
  int np = (n + 1) / 2;
  if (kSmem) { for (int i = threadIdx.x; i < 2 * np; i += blockDim.x) s_pair[i] = c_pair[i]; __syncthreads(); }
  int hits = 0;
  for (int rr = 0; rr < rays_per_thread; ++rr) {
    Ray r; make_ray((blockIdx.x * blockDim.x + threadIdx.x) * rays_per_thread + rr, r);
    float u1x, u1y, u1z, u2x, u2y, u2z; basis(r, u1x, u1y, u1z, u2x, u2y, u2z);
    float ou1 = -(r.ox * u1x + r.oy * u1y + r.oz * u1z);
    float ou2 = -(r.ox * u2x + r.oy * u2y + r.oz * u2z);
    float od = -(r.ox * r.dx + r.oy * r.dy + r.oz * r.dz);
    float2 U1x = make_float2(u1x, u1x), U1y = make_float2(u1y, u1y), U1z = make_float2(u1z, u1z);
    float2 U2x = make_float2(u2x, u2x), U2y = make_float2(u2y, u2y), U2z = make_float2(u2z, u2z);
    float2 OU1 = make_float2(ou1, ou1), OU2 = make_float2(ou2, ou2);
    float tbest = 1e30f; int best = -1;
#pragma unroll 2
    for (int p = 0; p < np; ++p) {
      float4 a = kSmem ? s_pair[2 * p] : c_pair[2 * p];
      float4 b = kSmem ? s_pair[2 * p + 1] : c_pair[2 * p + 1];
      float2 cx = make_float2(a.x, a.y), cy = make_float2(a.z, a.w);
      float2 cz = make_float2(b.x, b.y), r2 = make_float2(b.z, b.w);
      float2 x = __ffma2_rn(cx, U1x, __ffma2_rn(cy, U1y, __ffma2_rn(cz, U1z, OU1)));
      float2 y = __ffma2_rn(cx, U2x, __ffma2_rn(cy, U2y, __ffma2_rn(cz, U2z, OU2)));
      float2 nx = make_float2(-x.x, -x.y), ny = make_float2(-y.x, -y.y);
      float2 disc = __ffma2_rn(nx, x, __ffma2_rn(ny, y, r2));
      if (disc.x >= 0.f || disc.y >= 0.f) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float dd = h ? disc.y : disc.x;
          float sx = h ? cx.y : cx.x, sy = h ? cy.y : cy.x, sz = h ? cz.y : cz.x;
          if (dd >= 0.f) {
            float tc = fmaf(sx, r.dx, fmaf(sy, r.dy, fmaf(sz, r.dz, od)));
            float q = dd * rsqrtf(dd);
            float t0 = tc - q, t1 = tc + q;
            float t = t0 >= 1e-4f ? t0 : t1;
            if (t >= 1e-4f && t < tbest) { tbest = t; best = 2 * p + h; }
          }
        }
      }
    }
    hits += best;
  }
  if (hits == 0x7fffffff) out[0] = hits;
}

template <typename F>
static float time_ms(F launch, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  launch(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    CK(cudaEventRecord(a)); launch(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock_attr %d MHz\n", p.name, sms, clk_khz / 1000);
  float* dout; CK(cudaMalloc(&dout, 64));
  int* iout; CK(cudaMalloc(&iout, 64));
  const int threads = 256, blocks = sms * 8, iters = 4096;
  double fmas = double(blocks) * threads * iters * 16 * kChains;
  float ms = time_ms([&] { k_ffma_reg<<<blocks, threads>>>(dout, iters, 0.999f, 0.001f); });
  printf("FFMA reg : %.3f ms  %.2f TFLOP/s  %.1f FMA-lanes/clk/SM @%dMHz-attr\n", ms, 2 * fmas / ms / 1e9,
         fmas / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
  ms = time_ms([&] { k_ffma_imm<<<blocks, threads>>>(dout, iters); });
  printf("FFMA imm : %.3f ms  %.2f TFLOP/s  %.1f FMA-lanes/clk/SM\n", ms, 2 * fmas / ms / 1e9,
         fmas / (ms * 1e-3) / sms / (clk_khz * 1e3));
  ms = time_ms([&] { k_ffma2<<<blocks, threads>>>(dout, iters, 0.999f, 0.001f); });
  printf("FFMA2    : %.3f ms  %.2f TFLOP/s  %.1f FMA-lanes/clk/SM\n", ms, 2 * 2 * fmas / ms / 1e9,
         2 * fmas / (ms * 1e-3) / sms / (clk_khz * 1e3));

  {
    double* dd; CK(cudaMalloc(&dd, 64));
    int it2 = iters / 8;
    double dfmas = double(blocks) * threads * it2 * 16 * kChains;
    float m = time_ms([&] { k_dfma<<<blocks, threads>>>(dd, it2, 0.999, 0.001); });
    printf("DFMA     : %.3f ms  %.2f TFLOP/s(fp64)  %.1f DFMA-lanes/clk/SM\n", m, 2 * dfmas / m / 1e9,
           dfmas / (m * 1e-3) / sms / (clk_khz * 1e3));
  }
  // sphere field: 1000 spheres in [-30,30]x[-15,15]x[10,70], r in [0.3,1.2]
  int n = 1000;
  std::vector<float4> sph(n), pair(kMaxS);
  uint64_t s = 12345;
  auto rnd = [&] { s = s * 6364136223846793005ull + 1442695040888963407ull; return (s >> 40) / 16777216.0f; };
  for (int i = 0; i < n; ++i) {
    float r = 0.3f + 0.9f * rnd();
    sph[i] = make_float4(-30 + 60 * rnd(), -15 + 30 * rnd(), 10 + 60 * rnd(), r * r);
  }
  for (int q = 0; q < n / 2; ++q) {
    float4 A = sph[2 * q], B = sph[2 * q + 1];
    pair[2 * q] = make_float4(A.x, B.x, A.y, B.y);
    pair[2 * q + 1] = make_float4(A.z, B.z, A.w, B.w);
  }
  CK(cudaMemcpyToSymbol(c_sph, sph.data(), n * sizeof(float4)));
  CK(cudaMemcpyToSymbol(c_pair, pair.data(), n * sizeof(float4)));
  for (int tpb : {128, 256}) {
    int rpt = 4, bl = sms * (2048 / tpb);
    double tests = double(bl) * tpb * rpt * n;
    float m1 = time_ms([&] { k_sphere_scalar<false><<<bl, tpb>>>(iout, n, rpt); });
    float m2 = time_ms([&] { k_sphere_scalar<true><<<bl, tpb>>>(iout, n, rpt); });
    float m3 = time_ms([&] { k_sphere_pair<false><<<bl, tpb>>>(iout, n, rpt); });
    float m4 = time_ms([&] { k_sphere_pair<true><<<bl, tpb>>>(iout, n, rpt); });
    auto rep = [&](const char* nm, float m) {
      printf("%-22s tpb %d: %.3f ms  %.2f Gtests/s  %.2f tests/clk/SM  counted(19) %.1f TFLOP/s\n", nm, tpb, m,
             tests / m / 1e6, tests / (m * 1e-3) / sms / (clk_khz * 1e3), 19 * tests / m / 1e9);
    };
    rep("scalar const", m1); rep("scalar smem", m2); rep("ffma2 const", m3); rep("ffma2 smem", m4);
  }
  CK(cudaGetLastError());
  return 0;
}
