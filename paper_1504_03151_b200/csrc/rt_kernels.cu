// rt_kernels.cu — sm_100a kernels of the ray-tracing hot path (arXiv 1504.03151).
//
// One persistent "wavefront-in-a-warp" megakernel:
//   * every lane owns one pixel at a time (all spp samples, summed in order s = 0..spp-1);
//     finished lanes refill from a global work counter with one warp-aggregated atomicAdd
//     (ballot + popc + shfl), so warps stay full until the queue drains (path regeneration);
//   * each round, every lane has exactly one ray query — a closest-hit query (primary or
//     secondary ray) or an any-hit shadow query — and the whole warp runs ONE intersection
//     loop over the scene: sphere data is warp-uniform (constant bank) and two spheres are
//     tested per FFMA2 instruction by a conservative float32 filter; the rare candidates are
//     decided in float64 from the exact float inputs (same decisions as a double-precision
//     reference up to double rounding);
//   * between rounds each lane advances its own small state machine (float64 geometry):
//     ray generation (a2), shading with emission/ambient/Lambert/Phong (a4), shadow-ray set-up
//     (a5), the stack-free reflection/refraction continuation (a6), and the 16-byte store (a7).
// Paper: "each kernel thread traces a single light"; recursion becomes iteration
// (P:226); ray–sphere per Eq. 9–12; shading per Eq. 3–7 for point
// lights; Alg. 1 any-hit with early exit.
#include <cuda_runtime.h>
#include <cstdint>

#include "rt_internal.h"

namespace rt {

__constant__ DevPlane c_planes[kMaxPlanes];

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

// ---- per-lane state ------------------------------------------------------------------------
struct Lane {
  int item;                 // work item, -1 = needs work
  int px, py, s, depth, light;
  float3 Lpix, Ls, T;       // pixel sum, sample radiance, throughput
  d3 o, d;                  // current path segment
  d3 p, n;                  // shading point, facing normal
  int hit_sph, hit_pl;      // packed sphere index / plane index of the hit (-1 if not)
  int mat, entering;
  // query
  int qkind;
  d3 qo, qd;
  double tmax;
  int qs, qp;               // query result: packed sphere / plane index (-1 none)
  float3 contrib;
  // stats
  unsigned n_primary, n_shadow, n_secondary;
  unsigned long long n_stests, n_ptests;
};

// ---- ray generation (a2): §8(c).1 steps 1-2 ------------------------------------
__device__ __forceinline__ void sample_offset(int s, int spp, double& ox, double& oy) {
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

__device__ __forceinline__ void start_sample(Lane& L, const DevParams& P) {
  double ox, oy;
  sample_offset(L.s, P.spp, ox, oy);
  const double sx = (L.px + ox) / P.W, sy = (L.py + oy) / P.H;
  const double a = 2.0 * sx - 1.0, b = 1.0 - 2.0 * sy;
  const d3 dir = mk(P.F[0] + a * P.R[0] + b * P.U[0], P.F[1] + a * P.R[1] + b * P.U[1],
                    P.F[2] + a * P.R[2] + b * P.U[2]);
  L.o = mk(P.eye[0], P.eye[1], P.eye[2]);
  L.d = normalize(dir);
  L.T = f3(1.f, 1.f, 1.f);
  L.Ls = f3(0.f, 0.f, 0.f);
  L.depth = 0;
  L.qkind = Q_CLOSEST;
  L.qo = L.o; L.qd = L.d; L.tmax = kInf;
  L.n_primary++;
}

__device__ __forceinline__ bool start_item(Lane& L, const DevParams& P, int w, float4* out) {
  int t = w / kTilePx;
  const int i = w % kTilePx;
  if (P.mode == 1) {
    t = t * P.world + P.rank;
    if (t >= P.n_tiles) { out[w] = make_float4(0.f, 0.f, 0.f, 0.f); return false; }
  }
  const int px = (t % P.tiles_x) * kTileW + (i % kTileW);
  const int py = (t / P.tiles_x) * kTileH + (i / kTileW);
  if (px >= P.W || py >= P.H) {
    if (P.mode == 1) out[w] = make_float4(0.f, 0.f, 0.f, 0.f);
    return false;
  }
  L.item = w; L.px = px; L.py = py; L.s = 0;
  L.Lpix = f3(0.f, 0.f, 0.f);
  start_sample(L, P);
  return true;
}

// ---- scene staging (a1): one TMA bulk copy global -> shared per CTA -------------------------
// The pair array (32 B per two spheres) is copied into dynamic shared memory with
// cp.async.bulk (UBLKCP) completing on an mbarrier; every warp then reads each pair as a
// warp-uniform LDS.128 broadcast. Scenes larger than the shared-memory budget stay in global
// memory (uniform LDG through L1).
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
template <bool kSmem>
__device__ __forceinline__ float4 load_pair(const float4* __restrict__ sp, int i) {
  if constexpr (kSmem) return sp[i];     // warp-uniform address: LDS.128 broadcast
  else return __ldg(sp + i);
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
  const double cprime = dot(oc, oc) - r * r;
  double t0, t1;
  if (b < 0.0) {
    t1 = -b + q;
    t0 = t1 != 0.0 ? cprime / t1 : -b - q;
  } else {
    t0 = -b - q;
    t1 = t0 != 0.0 ? cprime / t0 : -b + q;
  }
  if (t0 > t1) { const double tmp = t0; t0 = t1; t1 = tmp; }
  return t0 >= kEps ? t0 : t1;
}

template <bool kSmem>
__device__ __forceinline__ void intersect(Lane& L, const DevParams& P, const DevScene& S,
                                          const float4* __restrict__ pairs) {
  bool act = (L.qkind != Q_NONE);
  const bool shadow = (L.qkind == Q_SHADOW);
  double tmax = L.tmax;
  int hs = -1, hp = -1;
  const d3 o = L.qo, d = L.qd;

  // planes first (index order == planes, then spheres for generated scenes); float64
  for (int j = 0; j < P.n_planes; ++j) {
    const DevPlane pl = c_planes[j];
    if (act) {
      const double den = pl.nx * d.x + pl.ny * d.y + pl.nz * d.z;
      if (fabs(den) >= 1e-12) {
        const double t = (pl.d - (pl.nx * o.x + pl.ny * o.y + pl.nz * o.z)) / den;
        if (t >= kEps && t < tmax) {
          hp = j;
          if (shadow) act = false; else tmax = t;
        }
      }
    }
  }

  // Spheres, float32 filter: orthonormal basis (u1, u2) of d (Duff et al. 2017); lateral
  // coordinates x = (c - o).u1, y = (c - o).u2 of each centre; disc = r^2 - x^2 - y^2 (the
  // precise discriminant of Eq. 11-12 with a = 1), two spheres per FFMA2. A sphere is a
  // candidate when disc >= -slack, slack bounding the float error.
  const float ox = (float)o.x, oy = (float)o.y, oz = (float)o.z;
  const float dx = (float)d.x, dy = (float)d.y, dz = (float)d.z;
  const float sg = copysignf(1.0f, dz);
  const float ia = -1.0f / (sg + dz);
  const float bb = dx * dy * ia;
  const float u1x = fmaf(sg * dx * dx, ia, 1.0f), u1y = sg * bb, u1z = -sg * dx;
  const float u2x = bb, u2y = fmaf(dy * dy, ia, sg), u2z = -dy;
  const float ou1 = -fmaf(ox, u1x, fmaf(oy, u1y, oz * u1z));
  const float ou2 = -fmaf(ox, u2x, fmaf(oy, u2y, oz * u2z));
  const float eta = 32.0f * kUlp * (fabsf(ox) + fabsf(oy) + fabsf(oz) + P.cmax);
  const float neg_slack = -(4.0f * eta * P.rmax + 4.0f * eta * eta + 4.0f * kUlp * P.rmax * P.rmax);
  const float2 U1x = make_float2(u1x, u1x), U1y = make_float2(u1y, u1y), U1z = make_float2(u1z, u1z);
  const float2 U2x = make_float2(u2x, u2x), U2y = make_float2(u2y, u2y), U2z = make_float2(u2z, u2z);
  const float2 OU1 = make_float2(ou1, ou1), OU2 = make_float2(ou2, ou2);
  // a warp without closest-hit lanes may leave the loop once every shadow lane found an occluder
  const bool may_exit = !__any_sync(kFull, L.qkind == Q_CLOSEST);

  if (__any_sync(kFull, act)) {
    for (int base = 0; base < P.n_pairs_pad; base += kPairsPerBatch) {
      float2 disc[kPairsPerBatch];
#pragma unroll
      for (int i = 0; i < kPairsPerBatch; ++i) {
        const float4 a = load_pair<kSmem>(pairs, 2 * (base + i));
        const float4 b = load_pair<kSmem>(pairs, 2 * (base + i) + 1);
        const float2 CX = make_float2(a.x, a.y), CY = make_float2(a.z, a.w);
        const float2 CZ = make_float2(b.x, b.y), R2 = make_float2(b.z, b.w);
        const float2 x = __ffma2_rn(CX, U1x, __ffma2_rn(CY, U1y, __ffma2_rn(CZ, U1z, OU1)));
        const float2 y = __ffma2_rn(CX, U2x, __ffma2_rn(CY, U2y, __ffma2_rn(CZ, U2z, OU2)));
        const float2 nx = make_float2(-x.x, -x.y), ny = make_float2(-y.x, -y.y);
        disc[i] = __ffma2_rn(nx, x, __ffma2_rn(ny, y, R2));
      }
      // candidate detection: one max-reduction per batch (FMNMX3 tree), the per-sphere mask is
      // only built on the rare path where some lane has a candidate
      float dmax = fmaxf(disc[0].x, disc[0].y);
#pragma unroll
      for (int i = 1; i < kPairsPerBatch; ++i) dmax = fmaxf(dmax, fmaxf(disc[i].x, disc[i].y));
      const bool any_cand = act && dmax >= neg_slack;
      if (__any_sync(kFull, any_cand)) {
        unsigned cand = 0u;
        if (any_cand) {
#pragma unroll
          for (int i = 0; i < kPairsPerBatch; ++i)
            cand |= ((disc[i].x >= neg_slack) ? 1u : 0u) << (2 * i) | ((disc[i].y >= neg_slack) ? 1u : 0u) << (2 * i + 1);
        }
        while (cand != 0u && act) {  // per-lane candidates, in index order (float64 decision)
          const int i = __ffs(cand) - 1;
          cand &= cand - 1u;
          const int k = 2 * base + i;  // pair (base + i/2), half i&1
          if (k >= P.n_spheres) break;  // padding (only reachable when the slack exceeds r^2 = 1)
          const double t = sphere_root(__ldg(S.sph_cr + k), o, d);
          if (t >= kEps && t < tmax) {
            hs = k; hp = -1;
            if (shadow) act = false; else tmax = t;
          }
        }
      }
      if (may_exit && !__any_sync(kFull, act)) break;  // Alg. 1 `break`, warp-wide
    }
  }
  // algorithmic test counts
  if (L.qkind == Q_CLOSEST) {
    L.n_stests += (unsigned)P.n_spheres;
    L.n_ptests += (unsigned)P.n_planes;
  } else if (L.qkind == Q_SHADOW) {
    if (hp >= 0) {
      L.n_ptests += (unsigned)(hp + 1);
    } else {
      L.n_ptests += (unsigned)P.n_planes;
      L.n_stests += (unsigned)(hs >= 0 ? hs + 1 : P.n_spheres);
    }
  }
  L.tmax = tmax;
  L.qs = hs;
  L.qp = hp;
}

// ---- shading, shadow setup, continuation (a4-a7) --------------------------------------------
template <bool kDebug>
__device__ void finish_sample(Lane& L, const DevParams& P, const DevOutputs& O) {
  L.Lpix = add(L.Lpix, L.Ls);
  if constexpr (kDebug) {
    const long long si = ((long long)L.py * P.W + L.px) * P.spp + L.s;
    O.dbg_bounces[si] = L.depth;  // secondary rays traced = depth of the last segment
    for (int k = L.depth + 1; k <= P.max_depth; ++k) O.dbg_hits[si * (P.max_depth + 1) + k] = -2;
  }
  L.s++;
  if (L.s < P.spp) {
    start_sample(L, P);
    return;
  }
  const float inv = 1.0f / (float)P.spp;
  const float4 v = make_float4(L.Lpix.x * inv, L.Lpix.y * inv, L.Lpix.z * inv, 1.0f);
  if (P.mode == 0) O.out[(long long)L.py * P.W + L.px] = v;  // 16-byte vector store
  else O.out[L.item] = v;
  L.item = -1;
  L.qkind = Q_NONE;
}

__device__ __forceinline__ d3 reflect(d3 d, d3 n) { return d - n * (2.0 * dot(d, n)); }

template <bool kDebug>
__device__ void bounce(Lane& L, const DevParams& P, const DevScene& S, const DevOutputs& O) {
  if (L.depth == P.max_depth) { finish_sample<kDebug>(L, P, O); return; }
  const DevMat m = S.mats[L.mat];
  d3 dn;
  if (m.kind == 1) {  // SPECULAR: mirror, T *= rho
    dn = reflect(L.d, L.n);
    L.T = mul(L.T, f3(m.ar, m.ag, m.ab));
  } else if (m.kind == 0) {  // DIFFUSE: mirror with weight kr when kr > 0 (R#8)
    if (!(m.kr > 0.f)) { finish_sample<kDebug>(L, P, O); return; }
    dn = reflect(L.d, L.n);
    L.T = f3(L.T.x * m.kr, L.T.y * m.kr, L.T.z * m.kr);
  } else {  // REFRACTIVE: Schlick-chosen reflect / refract, TIR -> reflect (R#9-R#11)
    const double ior = m.ior;
    const double eta = L.entering ? 1.0 / ior : ior;
    const double ci = -dot(L.d, L.n);
    const double sin2t = eta * eta * (1.0 - ci * ci);
    bool refl = sin2t > 1.0;
    if (!refl) {
      const double cosT = sqrt(1.0 - sin2t);
      const double c = L.entering ? ci : cosT;
      double r0 = (1.0 - ior) / (1.0 + ior);
      r0 *= r0;
      const double mm = 1.0 - c;
      const double F = r0 + (1.0 - r0) * (mm * mm * mm * mm * mm);
      const double u = rng_u(P.seed, (unsigned long long)L.py * P.W + L.px, L.s, L.depth);
      refl = u < F;
      if (!refl) dn = L.d * eta + L.n * (eta * ci - cosT);
    }
    if (refl) dn = reflect(L.d, L.n);
    L.T = mul(L.T, f3(m.ar, m.ag, m.ab));
  }
  L.o = L.p;
  L.d = normalize(dn);
  L.depth++;
  L.n_secondary++;
  L.qkind = Q_CLOSEST;
  L.qo = L.o; L.qd = L.d; L.tmax = kInf;
}

template <bool kDebug>
__device__ void next_light_or_bounce(Lane& L, const DevParams& P, const DevScene& S,
                                     const DevOutputs& O) {
  const DevMat m = S.mats[L.mat];
  if (m.kind == 0) {
    while (L.light < P.n_lights) {
      const DevLight lt = S.lights[L.light];
      L.light++;
      const d3 Pl = mk(lt.px, lt.py, lt.pz);
      const d3 w = Pl - L.p;
      const double d2 = dot(w, w);
      if (d2 < 1e-12) continue;                    // R#28
      const d3 wi = w * (1.0 / sqrt(d2));
      const double cosT = dot(L.n, wi);
      if (cosT <= 0.0) continue;                   // no shadow ray
      // shadow ray from p + EPS_T n toward the light (Alg. 1 "emit a shadow light")
      const d3 os = L.p + L.n * kEps;
      const d3 ws = Pl - os;
      const double tl = sqrt(dot(ws, ws));
      L.qo = os;
      L.qd = ws * (1.0 / tl);
      L.tmax = tl;
      L.qkind = Q_SHADOW;
      L.n_shadow++;
      // f_r = rho/pi + ks (s+2)/(2 pi) max(0, r.wo)^s (Eq. 5, R#3); E = I cos / d^2 (Eq. 3)
      const d3 rl = L.n * (2.0 * cosT) - wi;
      const float alpha = (float)fmax(0.0, -dot(rl, L.d));
      const float spec = m.ks * (m.shin + 2.0f) * kInv2Pi * powf(alpha, m.shin);
      const float g = (float)(cosT / d2);
      L.contrib = mul(L.T, f3(fmaf(m.ar, kInvPi, spec) * lt.ix * g, fmaf(m.ag, kInvPi, spec) * lt.iy * g,
                              fmaf(m.ab, kInvPi, spec) * lt.iz * g));
      return;
    }
  }
  bounce<kDebug>(L, P, S, O);
}

template <bool kDebug>
__device__ void on_closest(Lane& L, const DevParams& P, const DevScene& S, const DevOutputs& O) {
  const int hs = L.qs, hp = L.qp;
  int prim = -1;
  if (hp >= 0) prim = c_planes[hp].prim;
  else if (hs >= 0) prim = S.sph_prim[hs];
  if constexpr (kDebug) {
    const long long si = ((long long)L.py * P.W + L.px) * P.spp + L.s;
    O.dbg_hits[si * (P.max_depth + 1) + L.depth] = prim;
  }
  if (prim < 0) {  // miss -> background
    L.Ls = add(L.Ls, mul(L.T, f3(P.bg[0], P.bg[1], P.bg[2])));
    finish_sample<kDebug>(L, P, O);
    return;
  }
  L.p = L.o + L.d * L.tmax;
  d3 ng;
  if (hp >= 0) {
    const DevPlane pl = c_planes[hp];
    ng = mk(pl.nx, pl.ny, pl.nz);
    L.mat = pl.mat;
  } else {
    const float4 cr = __ldg(S.sph_cr + hs);
    ng = (L.p - mk(cr.x, cr.y, cr.z)) * (1.0 / (double)cr.w);
    L.mat = S.sph_mat[hs];
  }
  L.hit_sph = hs; L.hit_pl = hp;
  L.entering = dot(L.d, ng) < 0.0;
  L.n = L.entering ? ng : ng * -1.0;
  const DevMat m = S.mats[L.mat];
  L.Ls = add(L.Ls, mul(L.T, f3(m.er, m.eg, m.eb)));             // Eq. 7 emission
  if (m.kind == 0) L.Ls = add(L.Ls, mul(L.T, f3(m.ar * P.amb[0], m.ag * P.amb[1], m.ab * P.amb[2])));
  L.light = 0;
  next_light_or_bounce<kDebug>(L, P, S, O);
}

template <bool kDebug>
__device__ __forceinline__ void advance(Lane& L, const DevParams& P, const DevScene& S, const DevOutputs& O) {
  if (L.qkind == Q_CLOSEST) {
    on_closest<kDebug>(L, P, S, O);
  } else if (L.qkind == Q_SHADOW) {
    if (L.qs < 0 && L.qp < 0) L.Ls = add(L.Ls, L.contrib);  // visible: add f_r I cos / d^2
    next_light_or_bounce<kDebug>(L, P, S, O);
  }
}

// ---- the persistent megakernel --------------------------------------------------------------
template <bool kSmem, bool kDebug>
__global__ void __launch_bounds__(256, 2)
render_kernel(const DevParams P, const DevScene S, const DevOutputs O) {
  extern __shared__ float4 s_pairs[];
  __shared__ uint64_t s_mbar;
  if constexpr (kSmem) stage_scene(s_pairs, S.pairs, (uint32_t)P.n_pairs_pad * 32u, &s_mbar);
  const float4* pairs = kSmem ? s_pairs : S.pairs;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  Lane L;
  L.item = -1; L.qkind = Q_NONE;
  L.n_primary = L.n_shadow = L.n_secondary = 0;
  L.n_stests = L.n_ptests = 0ull;
  L.hit_sph = L.hit_pl = -1;
  bool exhausted = false;

  while (true) {
    // refill idle lanes: one atomicAdd per warp (ballot/popc/shfl)
    while (true) {
      const unsigned need = __ballot_sync(kFull, L.qkind == Q_NONE && !exhausted);
      if (need == 0u) break;
      const int leader = __ffs(need) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(O.work_counter, (unsigned)__popc(need));
      base = __shfl_sync(kFull, base, leader);
      if (need & (1u << lane)) {
        const unsigned w = base + __popc(need & lt_mask);
        if (w >= (unsigned)P.n_items) exhausted = true;
        else start_item(L, P, (int)w, O.out);
      }
    }
    if (!__any_sync(kFull, L.qkind != Q_NONE)) break;
    intersect<kSmem>(L, P, S, pairs);
    advance<kDebug>(L, P, S, O);
  }

  // stats: warp reduction, one atomic per warp
  unsigned long long v[5] = {L.n_primary, L.n_shadow, L.n_secondary, L.n_stests, L.n_ptests};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(kFull, v[k], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) atomicAdd(O.stats + k, v[k]);
  }
}

// ---- assemble (rank slabs -> row-major framebuffer) and tone map ---------------------------
__global__ void assemble_kernel(const float4* __restrict__ g, int W, int H, int world, int tpr,
                                int tiles_x, float4* __restrict__ out) {
  const long long slab_f4 = (long long)tpr * kTilePx + 4;  // + 64-byte stats record
  const long long n = (long long)W * H;
  for (long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x; pix < n;
       pix += (long long)gridDim.x * blockDim.x) {
    const int px = (int)(pix % W), py = (int)(pix / W);
    const int t = (py / kTileH) * tiles_x + px / kTileW;
    const int r = t % world, j = t / world;
    const int i = (py % kTileH) * kTileW + (px % kTileW);
    out[pix] = g[r * slab_f4 + (long long)j * kTilePx + i];
  }
}

__global__ void sum_stats_kernel(const float4* __restrict__ g, int world, int tpr,
                                 unsigned long long* stats) {
  if (threadIdx.x < 5) {
    const long long slab_f4 = (long long)tpr * kTilePx + 4;
    unsigned long long s = 0;
    for (int r = 0; r < world; ++r) {
      const unsigned long long* rec =
          reinterpret_cast<const unsigned long long*>(g + r * slab_f4 + (long long)tpr * kTilePx);
      s += rec[threadIdx.x];
    }
    stats[threadIdx.x] = s;
  }
}

__global__ void tonemap_kernel(const float4* __restrict__ in, uchar4* __restrict__ out, long long n,
                               float exposure, float inv_gamma) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = in[i];
    auto tm = [&](float x) -> unsigned char {
      double y = (double)exposure * (double)x;
      y = y > 0.0 ? (y < 1.0 ? y : 1.0) : 0.0;
      return (unsigned char)floor(255.0 * pow(y, (double)inv_gamma) + 0.5);
    };
    out[i] = make_uchar4(tm(v.x), tm(v.y), tm(v.z), 255);
  }
}

// ---- launchers ------------------------------------------------------------------------------
cudaError_t upload_const_scene(const DevPlane* planes, int n_planes, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  if (n_planes > 0)
    e = cudaMemcpyToSymbolAsync(c_planes, planes, sizeof(DevPlane) * n_planes, 0,
                                cudaMemcpyHostToDevice, st);
  return e;
}

template <bool kSmem, bool kDebug>
static cudaError_t launch_t(const DevParams& p, const DevScene& sc, const DevOutputs& o, int num_sms,
                           cudaStream_t st, int* blocks_per_sm_out) {
  const size_t smem = kSmem ? (size_t)p.n_pairs_pad * 32u : 0u;
  cudaError_t e = cudaFuncSetAttribute(render_kernel<kSmem, kDebug>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(smem > 0 ? smem : 1));
  if (e != cudaSuccess) return e;
  int bps = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, render_kernel<kSmem, kDebug>, 256, smem);
  if (e != cudaSuccess) return e;
  if (bps < 1) bps = 1;
  if (blocks_per_sm_out) *blocks_per_sm_out = bps;
  const long long want = (long long)num_sms * bps;
  const long long max_useful = ((long long)p.n_items + 255) / 256;  // no idle CTAs on tiny frames
  const int grid = (int)(want < max_useful ? want : (max_useful > 0 ? max_useful : 1));
  render_kernel<kSmem, kDebug><<<grid, 256, smem, st>>>(p, sc, o);
  return cudaGetLastError();
}

cudaError_t launch_render(const DevParams& p, const DevScene& sc, const DevOutputs& o, bool smem_scene,
                          int num_sms, cudaStream_t st) {
  const bool dbg = o.dbg_hits != nullptr;
  if (smem_scene) return dbg ? launch_t<true, true>(p, sc, o, num_sms, st, nullptr)
                             : launch_t<true, false>(p, sc, o, num_sms, st, nullptr);
  return dbg ? launch_t<false, true>(p, sc, o, num_sms, st, nullptr)
             : launch_t<false, false>(p, sc, o, num_sms, st, nullptr);
}

cudaError_t launch_assemble(const float4* gathered, int W, int H, int world, int tiles_per_rank,
                            float4* out, unsigned long long* stats, cudaStream_t st) {
  const int tiles_x = (W + kTileW - 1) / kTileW;
  const long long n = (long long)W * H;
  int grid = (int)((n + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  assemble_kernel<<<grid, 256, 0, st>>>(gathered, W, H, world, tiles_per_rank, tiles_x, out);
  sum_stats_kernel<<<1, 32, 0, st>>>(gathered, world, tiles_per_rank, stats);
  return cudaGetLastError();
}

cudaError_t launch_tonemap(const float4* rgba, uint8_t* out, int64_t n, float exposure, float gamma,
                           cudaStream_t st) {
  int grid = (int)((n + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  tonemap_kernel<<<grid, 256, 0, st>>>(rgba, reinterpret_cast<uchar4*>(out), n, exposure, 1.0f / gamma);
  return cudaGetLastError();
}

}  // namespace rt
