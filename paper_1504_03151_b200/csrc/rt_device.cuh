// rt_device.cuh — device helpers shared by the megakernel and the wavefront kernels
// (included by rt_kernels.cu only: one translation unit, one copy of the constant bank).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "rt_internal.h"

namespace rt {

__constant__ DevPlane c_planes[kMaxPlanes];
// sub-pixel offsets {ox, oy} of samples 0..spp-1 for spp <= kOffTable (sample_offset's values,
// computed on the host with the same IEEE double operations: rt_kernels.cu upload_sample_offsets)
constexpr int kOffTable = 256;
__constant__ double2 c_sample_off[kOffTable];
__device__ unsigned g_rt_check;  // first failed RT_CHECK id (checked builds)

constexpr double kEps = 1e-4;          // EPS_T
constexpr double kInf = 1.0e300;
constexpr unsigned kFull = 0xffffffffu;
constexpr float kInvPi = 0.318309886183790671538f;
constexpr float kInv2Pi = 0.159154943091895335769f;
constexpr float kUlp = 5.9604644775390625e-08f;  // 2^-24

enum : int { Q_NONE = 0, Q_CLOSEST = 1, Q_SHADOW = 2 };

struct d3 { double x, y, z; };
__device__ __forceinline__ d3 mk(double x, double y, double z) { d3 r; r.x = x; r.y = y; r.z = z; return r; }
__device__ __forceinline__ d3 operator+(d3 a, d3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ d3 operator-(d3 a, d3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ d3 operator*(d3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ d3 normalize(d3 a) { return a * (1.0 / sqrt(dot(a, a))); }
__device__ __forceinline__ float3 f3(float x, float y, float z) { return make_float3(x, y, z); }
__device__ __forceinline__ float3 add(float3 a, float3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ float3 mul(float3 a, float3 b) { return f3(a.x * b.x, a.y * b.y, a.z * b.z); }

// splitmix64 finalizer and the per-decision counter RNG
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
__device__ __forceinline__ double rng_u(unsigned long long seed, unsigned long long pix, int s, int depth) {
  const unsigned long long G = 0x9E3779B97F4A7C15ull;
  unsigned long long x = seed ^ ((pix + 1ull) * G);
  x = mix64(x);
  x = mix64(x ^ ((((unsigned long long)(unsigned)s) << 32) + (unsigned long long)(unsigned)depth) * G);
  return (double)(x >> 40) * (1.0 / 16777216.0);
}

// draw k of (pixel, sample, depth): counter word s*2^32 + k*2^8 + depth (R#42);
// stream 0 is rng_u. Streams: 1/2 jitter, 3/4 diffuse bounce, 5+2e/6+2e emitter e's point.
__device__ __forceinline__ double rng_stream(unsigned long long seed, unsigned long long pix, unsigned s,
                                             int depth, unsigned k) {
  const unsigned long long G = 0x9E3779B97F4A7C15ull;
  unsigned long long x = seed ^ ((pix + 1ull) * G);
  x = mix64(x);
  x = mix64(x ^ (((unsigned long long)s << 32) + ((unsigned long long)k << 8) + (unsigned long long)(unsigned)depth) * G);
  return (double)(x >> 40) * (1.0 / 16777216.0);
}

// uniform point on a sphere (R#41): cos(theta) = 1 - 2 u1, phi = 2 pi u2, pole +z
__device__ __forceinline__ d3 sphere_point(double u1, double u2) {
  const double ct = 1.0 - 2.0 * u1;
  const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
  double sp, cp;
  sincospi(2.0 * u2, &sp, &cp);
  return mk(st * cp, st * sp, ct);
}

// cosine-weighted direction about unit n in the Duff et al. (2017) basis (R#40)
__device__ __forceinline__ d3 cosine_dir(d3 n, double u1, double u2) {
  const double sg = copysign(1.0, n.z);
  const double a = -1.0 / (sg + n.z);
  const double b = n.x * n.y * a;
  const d3 t1 = mk(1.0 + sg * n.x * n.x * a, sg * b, -sg * n.x);
  const d3 t2 = mk(b, sg + n.y * n.y * a, -n.y);
  const double rr = sqrt(u1);
  double sp, cp;
  sincospi(2.0 * u2, &sp, &cp);
  return t1 * (rr * cp) + t2 * (rr * sp) + n * sqrt(fmax(0.0, 1.0 - u1));
}

// Phong lobe max(0, r.wo)^s (Eq. 5, R#3) for alpha in [0, 1], s >= 1: exp2(s log2 alpha) with the
// accurate (non-intrinsic) log2f / exp2f. The relative error stays below ln2 |s log2 alpha| 2^-23
// <= 1e-5 over the range before underflow (|s log2 alpha| <= 126), inside the 1e-4 radiance
// tolerance; powf's extended-precision log and special cases cost twice the instructions.
__device__ __forceinline__ float phong_lobe(float alpha, float s) {
  return alpha > 0.f ? exp2f(s * log2f(alpha)) : 0.f;
}

// ---- ray generation (a2): §8(c).1 steps 1-2 ------------------------------------
__device__ __forceinline__ void sample_offset(int s, int spp, double& ox, double& oy) {
  if (spp <= kOffTable) {  // the same values, precomputed per spp (no divisions here)
    const double2 o = c_sample_off[s];
    ox = o.x;
    oy = o.y;
    return;
  }
  int n = 1;
  while ((n + 1) * (n + 1) <= spp) ++n;
  if (n * n == spp) {
    const int i = s % n, j = s / n;
    ox = (i + 0.5) / n;
    oy = (j + 0.5) / n;
  } else {
    const double radinv = (double)__brev((unsigned)s) * (1.0 / 4294967296.0);
    const double y = radinv + 0.5 / spp;
    ox = (s + 0.5) / spp;
    oy = y - floor(y);
  }
}

// camera ray of sample s of pixel (px, py): d = normalize(F + (2sx-1) R + (1-2sy) U)
// sub-pixel position of sample s of pixel (px, py)
__device__ __forceinline__ void sample_xy(const DevParams& P, int px, int py, int s, double& ox, double& oy) {
  if (P.jitter) {  // progressive passes: random offset of sample (pass) sample_base + s (R#42)
    const unsigned long long pix = (unsigned long long)py * P.W + px;
    const unsigned sg = (unsigned)(P.sample_base + s);
    ox = rng_stream(P.seed, pix, sg, 0, 1u);
    oy = rng_stream(P.seed, pix, sg, 0, 2u);
  } else {
    sample_offset(s, P.spp, ox, oy);
  }
}
__device__ __forceinline__ d3 camera_dir(const DevParams& P, int px, int py, int s) {
  double ox, oy;
  sample_xy(P, px, py, s, ox, oy);
  const double sx = (px + ox) / P.W, sy = (py + oy) / P.H;
  const double a = 2.0 * sx - 1.0, b = 1.0 - 2.0 * sy;
  return normalize(mk(P.F[0] + a * P.R[0] + b * P.U[0], P.F[1] + a * P.R[1] + b * P.U[1],
                      P.F[2] + a * P.R[2] + b * P.U[2]));
}

// The same camera ray for a float filter only (the camera-ray scan): the divisions by W and H
// become products with 1/W, 1/H and the normalisation an FP64 rsqrt, so the direction is within
// a few FP64 ulps of camera_dir's — far inside the filter's bound for d rounded to float (eta,
// slack: 2^-24 per component), while every decision uses camera_dir itself (wf_shade).
__device__ __forceinline__ void camera_dir_filter(const DevParams& P, int px, int py, int s, float& dx, float& dy,
                                                  float& dz) {
  double ox, oy;
  sample_xy(P, px, py, s, ox, oy);
  const double a = 2.0 * ((px + ox) * P.inv_w) - 1.0, b = 1.0 - 2.0 * ((py + oy) * P.inv_h);
  const double vx = P.F[0] + a * P.R[0] + b * P.U[0], vy = P.F[1] + a * P.R[1] + b * P.U[1],
               vz = P.F[2] + a * P.R[2] + b * P.U[2];
  const double k = rsqrt(vx * vx + vy * vy + vz * vz);
  dx = (float)(vx * k);
  dy = (float)(vy * k);
  dz = (float)(vz * k);
}

// global tile of a rank's local tile j: one tile of every group of `world` consecutive tiles,
// the slot rotating with the group (rank_tile_slot), so a rank's tiles do not line up in tile
// columns (tiles_x is often a multiple of world) and every rank sees the same mix of the image
__host__ __device__ __forceinline__ int rank_tile(int j, int rank, int world) { return j * world + (rank + j) % world; }
// work item w (tile-major, 8x4 tiles; shard mode maps local tile j to global tile rank_tile(j))
// -> pixel; returns false for pixels outside the image / tiles past the end
__device__ __forceinline__ bool item_pixel(const DevParams& P, int w, int& px, int& py) {
  int t = w / kTilePx;
  const int i = w % kTilePx;
  if (P.mode >= 1) {  // shard (1) or direct shard (2): local tile j is global tile rank_tile(j)
    t = rank_tile(t, P.rank, P.world);
    if (t >= P.n_tiles) return false;
  }
  const int ty = (int)fdiv(P.div_tiles_x, (unsigned)t);  // t / tiles_x
  px = (t - ty * P.tiles_x) * kTileW + (i % kTileW);
  py = ty * kTileH + (i / kTileW);
  return px < P.W && py < P.H;
}

__device__ __forceinline__ d3 reflect(d3 d, d3 n) { return d - n * (2.0 * dot(d, n)); }

// ---- scene staging (a1): one TMA bulk copy global -> shared per CTA -------------------------
// The pair array (32 B per two spheres) is copied into dynamic shared memory with
// cp.async.bulk (UBLKCP) completing on an mbarrier; every warp then reads each pair as a
// warp-uniform LDS.128 broadcast. Scenes larger than the shared-memory budget stay in global
// memory in TMA-loaded tiles (SRC_TILE below).
__device__ __forceinline__ void stage_scene(float4* s_pairs, const float4* g_pairs, uint32_t bytes,
                                            uint64_t* mbar) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s_pairs);
    constexpr uint32_t kChunk = 1u << 15;
    for (uint32_t off = 0; off < bytes; off += kChunk) {
      const uint32_t n = (bytes - off) < kChunk ? (bytes - off) : kChunk;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + off),
          "l"(reinterpret_cast<const char*>(g_pairs) + off), "r"(n), "r"(mb)
          : "memory");
    }
  }
  __syncthreads();  // barrier initialised before anyone waits on it
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(mb), "r"(0u)
        : "memory");
  }
}

// ---- intersection (a3 closest-hit + a5 any-hit), one loop for the whole warp -----------------
extern __shared__ float4 s_pairs[];

// where the sphere-pair array is read from inside the scans: the whole scene staged in shared
// memory (SRC_SMEM), a ring of two TMA-loaded tiles of kTilePairs pairs in shared memory for
// scenes beyond the shared-memory budget (SRC_TILE: global float4 index i lives at ring slot
// i mod 4 kTilePairs while its tile is resident), or global memory (SRC_GLOBAL: the short-queue
// split scans of such scenes)
enum : int { SRC_GLOBAL = 0, SRC_SMEM = 1, SRC_TILE = 2 };
constexpr int kTilePairs = 512;  // 16 KB per tile, two tiles in flight per CTA

template <int kSrc>
__device__ __forceinline__ float4 load_pair(const float4* __restrict__ gp, int i) {
  if constexpr (kSrc == SRC_SMEM) return s_pairs[i];  // warp-uniform address: LDS.128 broadcast
  else if constexpr (kSrc == SRC_TILE) return s_pairs[i & (4 * kTilePairs - 1)];
  else return __ldg(gp + i);
}

// ---- tiled staging for scenes beyond shared memory: TMA bulk copies completing on mbarriers ----
__device__ __forceinline__ void mbar_init(uint64_t* mbar) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one thread: copy `bytes` (multiple of 16, <= 32 KB) from global to shared memory, completing on mbar
__device__ __forceinline__ void tile_load(float4* dst, const float4* src, uint32_t bytes, uint64_t* mbar) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"(mb)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(mb), "r"(parity)
        : "memory");
  }
}

// Exact decision for one sphere (float64, from the float inputs): smallest root >= EPS_T of
// Eq. 11 with a = 1, precise discriminant r^2 - |oc - (oc.d) d|^2, stable roots.
__device__ __forceinline__ double sphere_root(const float4 cr, const d3 o, const d3 d) {
  const d3 oc = o - mk(cr.x, cr.y, cr.z);
  const double r = cr.w;
  const double b = dot(oc, d);
  const d3 perp = oc - d * b;
  const double disc = r * r - dot(perp, perp);
  if (disc < 0.0) return -1.0;
  const double q = sqrt(disc);
  double t0 = -b - q, t1 = -b + q;
  // stable form: a root that cancels (origin near the surface) is recomputed from the
  // product of the roots, c' = |oc|^2 - r^2
  const double cancel = 1e-3 * fabs(b);
  if (fabs(t0) < cancel || fabs(t1) < cancel) {
    const double cprime = dot(oc, oc) - r * r;
    if (fabs(t0) < cancel) t0 = cprime / t1;
    else t1 = cprime / t0;
    if (t0 > t1) { const double tmp = t0; t0 = t1; t1 = tmp; }
  }
  return t0 >= kEps ? t0 : t1;
}

// max of 16 filter values as a depth-3 tree of 3-input maxima (FMNMX3): the same 8 instructions
// as the running max, whose chain of 8 dependent FMNMX3 ends every batch (the 7-FMA scan: 1.665
// -> 1.631 ms at C4; the shared-origin scans keep the running max, which interleaves better)
__device__ __forceinline__ float max16(const float2 (&v)[8]) {
  const float m0 = fmaxf(fmaxf(v[0].x, v[0].y), v[1].x), m1 = fmaxf(fmaxf(v[1].y, v[2].x), v[2].y);
  const float m2 = fmaxf(fmaxf(v[3].x, v[3].y), v[4].x), m3 = fmaxf(fmaxf(v[4].y, v[5].x), v[5].y);
  const float m4 = fmaxf(fmaxf(v[6].x, v[6].y), v[7].x);
  return fmaxf(fmaxf(fmaxf(m0, m1), m2), fmaxf(fmaxf(m3, m4), v[7].y));
}

// Float32 filter state of one ray. Per sphere the filter value v is
// compared with `cut`; a sphere with v >= cut is a candidate, decided later in float64.
// Pair data {c', K = r^2 - |c'|^2} in scene-centred coordinates c' = c - centre:
// s1 = K + 2 c'.o', tc = (c' - o').d, v = tc^2 + s1 = disc + |o'|^2 (Eq. 11's discriminant
// b^2 - (|oc|^2 - r^2) with a = 1 and |oc|^2 expanded): 7 FMA per sphere, two spheres per FFMA2.
// `slack` bounds |v_float - v_exact| (first-order FP32 error analysis), `eta` bounds the error
// of tc; both make the filter conservative: no true intersection is ever dropped.
struct RayFilter {
  float dx, dy, dz, a1, a2, a3, b1, eta, neg_slack, cut;
  __device__ __forceinline__ void init(const d3& o, const d3& d, const DevParams& P) {
    init(o, (float)d.x, (float)d.y, (float)d.z, P);
  }
  // direction already rounded to float (the same values as the FP64 overload's conversion)
  __device__ __forceinline__ void init(const d3& o, float fdx, float fdy, float fdz, const DevParams& P) {
    dx = fdx; dy = fdy; dz = fdz;
    const float ox = (float)(o.x - P.centre[0]), oy = (float)(o.y - P.centre[1]), oz = (float)(o.z - P.centre[2]);
    const float on = sqrtf(fmaf(ox, ox, fmaf(oy, oy, oz * oz)));
    a1 = 2.0f * ox; a2 = 2.0f * oy; a3 = 2.0f * oz;                 // 2 o'
    b1 = -fmaf(ox, dx, fmaf(oy, dy, oz * dz));                       // -o'.d
    const float span = P.cmax + on + P.rmax;
    const float slack = 24.0f * kUlp * span * span;
    eta = 8.0f * kUlp * (P.cmax + on);
    neg_slack = -slack;
    cut = on * on - slack;
  }
  // filter values of 16 spheres (pairs base..base+7), two spheres per FFMA2; returns their max
  template <int kSrc>
  __device__ __forceinline__ float batch(const float4* __restrict__ gp, int base, float2 (&v)[kPairsPerBatch]) const {
    const float2 A1 = make_float2(a1, a1), A2 = make_float2(a2, a2), A3 = make_float2(a3, a3);
    const float2 D1 = make_float2(dx, dx), D2 = make_float2(dy, dy), D3 = make_float2(dz, dz);
    const float2 B1 = make_float2(b1, b1);
#pragma unroll
    for (int i = 0; i < kPairsPerBatch; ++i) {
      const float4 a = load_pair<kSrc>(gp, 2 * (base + i));
      const float4 b = load_pair<kSrc>(gp, 2 * (base + i) + 1);
      const float2 CX = make_float2(a.x, a.y), CY = make_float2(a.z, a.w);
      const float2 CZ = make_float2(b.x, b.y), K = make_float2(b.z, b.w);
      const float2 s1 = __ffma2_rn(CX, A1, __ffma2_rn(CY, A2, __ffma2_rn(CZ, A3, K)));
      const float2 tc = __ffma2_rn(CX, D1, __ffma2_rn(CY, D2, __ffma2_rn(CZ, D3, B1)));
      v[i] = __ffma2_rn(tc, tc, s1);
    }
    static_assert(kPairsPerBatch == 8, "max16");
    return max16(v);
  }
  // Shared-origin scans (camera rays, light-origin shadow rays) test the tangent condition
  // c'.d - h >= o'.d instead of v >= cut (rt_kernels.cu neg_tangent: h per sphere precomputed): a hit
  // at t > 0 from o outside the sphere needs tc >= h, and tc - h is 3 FMA per sphere. Its error
  // (the FMA chain over |c'| + h <= 2 (cmax + |o'|), c' and d rounded to float, -h and o'.d
  // rounded) stays below 11 kUlp (cmax + |o'|) <= 2 eta: candidates are the spheres with
  // c'.d - h >= tangent_cut().
  __device__ __forceinline__ float tangent_cut() const { return -b1 - 2.0f * eta; }
  // dd and tc of sphere k for a shared origin whose s1 = K + 2 c'.o' comes precomputed (s1p, one
  // float2 per pair, FP64 rounded once: more accurate than the FMA chain the slack covers)
  template <int kSrc>
  __device__ __forceinline__ void sphere_s1(const float4* __restrict__ gp, const float2* __restrict__ s1p, int k,
                                            float& dd, float& tc) const {
    const float4 pa = load_pair<kSrc>(gp, 2 * (k >> 1));
    const float4 pb = load_pair<kSrc>(gp, 2 * (k >> 1) + 1);
    const float2 sv = s1p[k >> 1];
    const bool h = k & 1;
    const float cx = h ? pa.y : pa.x, cy = h ? pa.w : pa.z, cz = h ? pb.y : pb.x, s1 = h ? sv.y : sv.x;
    tc = fmaf(cx, dx, fmaf(cy, dy, fmaf(cz, dz, b1)));
    dd = fmaf(tc, tc, s1) - (cut - neg_slack);  // v - |o'|^2
  }
  // the same as sphere() for a table whose K slots hold something else (a light's -h): c' from
  // the table gt (kSrc), K from the float2-per-pair column kp
  template <int kSrc>
  __device__ __forceinline__ void sphere_k(const float4* __restrict__ gt, const float2* __restrict__ kp, int k,
                                           float& dd, float& tc) const {
    const float4 pa = load_pair<kSrc>(gt, 2 * (k >> 1));
    const float4 pb = load_pair<kSrc>(gt, 2 * (k >> 1) + 1);
    const float2 kk = kp[k >> 1];
    const bool h = k & 1;
    const float cx = h ? pa.y : pa.x, cy = h ? pa.w : pa.z, cz = h ? pb.y : pb.x, w = h ? kk.y : kk.x;
    const float s1 = fmaf(cx, a1, fmaf(cy, a2, fmaf(cz, a3, w)));
    tc = fmaf(cx, dx, fmaf(cy, dy, fmaf(cz, dz, b1)));
    dd = fmaf(tc, tc, s1) - (cut - neg_slack);  // v - |o'|^2
  }
  // float discriminant estimate dd (|dd - disc| <= slack) and chord centre tc (|err| <= eta) of
  // one sphere k (rare path)
  template <int kSrc>
  __device__ __forceinline__ void sphere(const float4* __restrict__ gp, int k, float& dd, float& tc) const {
    const float4 pa = load_pair<kSrc>(gp, 2 * (k >> 1));
    const float4 pb = load_pair<kSrc>(gp, 2 * (k >> 1) + 1);
    const bool h = k & 1;
    const float cx = h ? pa.y : pa.x, cy = h ? pa.w : pa.z, cz = h ? pb.y : pb.x, w = h ? pb.w : pb.z;
    const float s1 = fmaf(cx, a1, fmaf(cy, a2, fmaf(cz, a3, w)));
    tc = fmaf(cx, dx, fmaf(cy, dy, fmaf(cz, dz, b1)));
    dd = fmaf(tc, tc, s1) - (cut - neg_slack);  // v - |o'|^2
  }
};

__device__ __forceinline__ unsigned batch_mask(const float2 (&v)[kPairsPerBatch], float cut) {
  unsigned cand = 0u;
#pragma unroll
  for (int i = 0; i < kPairsPerBatch; ++i)
    cand |= ((v[i].x >= cut) ? 1u : 0u) << (2 * i) | ((v[i].y >= cut) ? 1u : 0u) << (2 * i + 1);
  return cand;
}

}  // namespace rt
