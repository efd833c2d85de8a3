// rt_kernels.cu — sm_100a kernels of the ray-tracing hot path (arXiv 1504.03151).
//
// One persistent "wavefront-in-a-warp" megakernel:
//   * every lane owns one pixel at a time (all spp samples, summed in order s = 0..spp-1);
//     finished lanes refill from a global work counter with one warp-aggregated atomicAdd
//     (ballot + popc + shfl), so warps stay full until the queue drains (path regeneration);
//   * each round, every lane has exactly one ray query — a closest-hit query (primary or
//     secondary ray) or an any-hit shadow query — and the whole warp runs ONE intersection
//     loop over the scene: the sphere data is warp-uniform (constant bank -> LDCU.128 into
//     uniform registers) and two spheres are tested per FFMA2 instruction;
//   * between rounds each lane advances its own small state machine: ray generation (a2),
//     shading with emission/ambient/Lambert/Phong (a4), shadow-ray setup (a5) and the
//     stack-free reflection/refraction continuation (a6), accumulation + 16-byte store (a7).
// Paper: "each kernel thread traces a single light" and recursion becomes iteration
// (P:226); ray–sphere per Eq. 9–12; shading per Eq. 3–7 for point
// lights; Alg. 1 any-hit with early exit.
#include <cuda_runtime.h>
#include <cstdint>

#include "rt_internal.h"

namespace rt {

__constant__ float4 c_pairs[2 * kMaxConstPairs];
__constant__ DevPlane c_planes[kMaxPlanes];

constexpr float kEps = 1e-4f;          // EPS_T
constexpr float kInf = 3.0e38f;
constexpr unsigned kFull = 0xffffffffu;
constexpr float kInvPi = 0.318309886183790671538f;
constexpr float kInv2Pi = 0.159154943091895335769f;

enum : int { Q_NONE = 0, Q_CLOSEST = 1, Q_SHADOW = 2 };

__device__ __forceinline__ float3 f3(float x, float y, float z) { return make_float3(x, y, z); }
__device__ __forceinline__ float3 operator+(float3 a, float3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ float3 operator-(float3 a, float3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ float3 operator*(float3 a, float s) { return f3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ float3 mul(float3 a, float3 b) { return f3(a.x * b.x, a.y * b.y, a.z * b.z); }
__device__ __forceinline__ float dot3(float3 a, float3 b) { return fmaf(a.x, b.x, fmaf(a.y, b.y, a.z * b.z)); }
__device__ __forceinline__ float3 fma3(float3 a, float s, float3 b) {
  return f3(fmaf(a.x, s, b.x), fmaf(a.y, s, b.y), fmaf(a.z, s, b.z));
}
__device__ __forceinline__ float3 normalize3(float3 a) { return a * rsqrtf(dot3(a, a)); }

// splitmix64 finalizer and the per-decision counter RNG
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
__device__ __forceinline__ float rng_u(unsigned long long seed, unsigned long long pix, int s, int depth) {
  const unsigned long long G = 0x9E3779B97F4A7C15ull;
  unsigned long long x = seed ^ ((pix + 1ull) * G);
  x = mix64(x);
  x = mix64(x ^ ((((unsigned long long)(unsigned)s) << 32) + (unsigned long long)(unsigned)depth) * G);
  return (float)(unsigned)(x >> 40) * (1.0f / 16777216.0f);
}

// ---- per-lane state ------------------------------------------------------------------------
struct Lane {
  int item;                 // work item, -1 = needs work
  int px, py, s, depth, light;
  float3 Lpix, Ls, T;       // pixel sum, sample radiance, throughput
  float3 o, d;              // current path segment
  float3 p, n, ng;          // shading point, facing normal, geometric normal
  int hit_prim;             // original primitive index of the current hit
  int hit_sph, hit_pl;      // packed sphere index / plane index of the hit (-1 if not)
  int mat, entering;
  // query
  int qkind;
  float3 qo, qd;
  float tmax;
  int qs, qp;               // query result: packed sphere / plane index (-1 none)
  int self_s, self_p, self_in;
  float3 contrib;
  // stats
  unsigned n_primary, n_shadow, n_secondary;
  unsigned long long n_stests, n_ptests;
};

// ---- ray generation (a2): §8(c).1 steps 1-2 ------------------------------------
__device__ __forceinline__ void sample_offset(int s, int spp, float& ox, float& oy) {
  int n = (int)sqrtf((float)spp);
  while ((n + 1) * (n + 1) <= spp) ++n;
  while (n * n > spp) --n;
  if (n * n == spp) {
    int i = s % n, j = s / n;
    ox = (i + 0.5f) / n;
    oy = (j + 0.5f) / n;
  } else {
    float radinv = (float)__brev((unsigned)s) * 2.3283064365386963e-10f;  // 2^-32
    float y = radinv + 0.5f / spp;
    ox = (s + 0.5f) / spp;
    oy = y - floorf(y);
  }
}

__device__ __forceinline__ void start_sample(Lane& L, const DevParams& P) {
  float ox, oy;
  sample_offset(L.s, P.spp, ox, oy);
  float sx = (L.px + ox) / (float)P.W;
  float sy = (L.py + oy) / (float)P.H;
  float a = 2.0f * sx - 1.0f, b = 1.0f - 2.0f * sy;
  float3 F = f3(P.F[0], P.F[1], P.F[2]), R = f3(P.R[0], P.R[1], P.R[2]), U = f3(P.U[0], P.U[1], P.U[2]);
  float3 dir = fma3(U, b, fma3(R, a, F));
  L.o = f3(P.eye[0], P.eye[1], P.eye[2]);
  L.d = normalize3(dir);
  L.T = f3(1.f, 1.f, 1.f);
  L.Ls = f3(0.f, 0.f, 0.f);
  L.depth = 0;
  L.qkind = Q_CLOSEST;
  L.qo = L.o; L.qd = L.d; L.tmax = kInf;
  L.self_s = -1; L.self_p = -1; L.self_in = 0;
  L.n_primary++;
}

__device__ __forceinline__ bool start_item(Lane& L, const DevParams& P, int w, float4* out) {
  int t = w / kTilePx, i = w % kTilePx;
  if (P.mode == 1) {
    t = t * P.world + P.rank;
    if (t >= P.n_tiles) { out[w] = make_float4(0.f, 0.f, 0.f, 0.f); return false; }
  }
  int px = (t % P.tiles_x) * kTileW + (i % kTileW);
  int py = (t / P.tiles_x) * kTileH + (i / kTileW);
  if (px >= P.W || py >= P.H) {
    if (P.mode == 1) out[w] = make_float4(0.f, 0.f, 0.f, 0.f);
    return false;
  }
  L.item = w; L.px = px; L.py = py; L.s = 0;
  L.Lpix = f3(0.f, 0.f, 0.f);
  start_sample(L, P);
  return true;
}

// ---- intersection (a3 closest-hit + a5 any-hit), one loop for the whole warp -----------------
template <bool kConst>
__device__ __forceinline__ float4 load_pair(const float4* __restrict__ g, int i) {
  if constexpr (kConst) return c_pairs[i];
  else return __ldg(g + i);
}

template <bool kConst>
__device__ __forceinline__ void intersect(Lane& L, const DevParams& P, const DevScene& S) {
  bool act = (L.qkind != Q_NONE);
  const bool shadow = (L.qkind == Q_SHADOW);
  float tmax = L.tmax;
  int hs = -1, hp = -1;
  const float3 o = L.qo, d = L.qd;

  // planes first (index order == planes, then spheres for generated scenes)
  for (int j = 0; j < P.n_planes; ++j) {
    DevPlane pl = c_planes[j];
    if (act && j != L.self_p) {
      float den = fmaf(pl.nx, d.x, fmaf(pl.ny, d.y, pl.nz * d.z));
      if (fabsf(den) >= 1e-12f) {
        float num = pl.d - fmaf(pl.nx, o.x, fmaf(pl.ny, o.y, pl.nz * o.z));
        float t = num / den;
        if (t >= kEps && t < tmax) {
          hp = j;
          if (shadow) act = false; else tmax = t;
        }
      }
    }
  }

  // spheres: basis (u1, u2) orthonormal to d (Duff et al. 2017); lateral coordinates of each
  // centre x = (c - o).u1, y = (c - o).u2 and disc = r^2 - x^2 - y^2 (= r^2 - |oc x d|^2, the
  // precise discriminant of Eq. 11-12 with a = 1), two spheres per FFMA2.
  const float sg = copysignf(1.0f, d.z);
  const float ia = -1.0f / (sg + d.z);
  const float bb = d.x * d.y * ia;
  const float u1x = fmaf(sg * d.x * d.x, ia, 1.0f), u1y = sg * bb, u1z = -sg * d.x;
  const float u2x = bb, u2y = fmaf(d.y * d.y, ia, sg), u2z = -d.y;
  const float ou1 = -fmaf(o.x, u1x, fmaf(o.y, u1y, o.z * u1z));
  const float ou2 = -fmaf(o.x, u2x, fmaf(o.y, u2y, o.z * u2z));
  const float od = -fmaf(o.x, d.x, fmaf(o.y, d.y, o.z * d.z));
  const float2 U1x = make_float2(u1x, u1x), U1y = make_float2(u1y, u1y), U1z = make_float2(u1z, u1z);
  const float2 U2x = make_float2(u2x, u2x), U2y = make_float2(u2y, u2y), U2z = make_float2(u2z, u2z);
  const float2 OU1 = make_float2(ou1, ou1), OU2 = make_float2(ou2, ou2);
  const int self_s = L.self_s, self_in = L.self_in;
  // a warp without closest-hit lanes may leave the loop once every shadow lane found an occluder
  const bool may_exit = !__any_sync(kFull, L.qkind == Q_CLOSEST);

  if (__any_sync(kFull, act)) {
    for (int base = 0; base < P.n_pairs_pad; base += kPairsPerBatch) {
      float2 disc[kPairsPerBatch], CX[kPairsPerBatch], CY[kPairsPerBatch], CZ[kPairsPerBatch];
#pragma unroll
      for (int i = 0; i < kPairsPerBatch; ++i) {
        const float4 a = load_pair<kConst>(S.pairs, 2 * (base + i));
        const float4 b = load_pair<kConst>(S.pairs, 2 * (base + i) + 1);
        CX[i] = make_float2(a.x, a.y);
        CY[i] = make_float2(a.z, a.w);
        CZ[i] = make_float2(b.x, b.y);
        const float2 R2 = make_float2(b.z, b.w);
        const float2 x = __ffma2_rn(CX[i], U1x, __ffma2_rn(CY[i], U1y, __ffma2_rn(CZ[i], U1z, OU1)));
        const float2 y = __ffma2_rn(CX[i], U2x, __ffma2_rn(CY[i], U2y, __ffma2_rn(CZ[i], U2z, OU2)));
        const float2 ny = make_float2(-y.x, -y.y), nx = make_float2(-x.x, -x.y);
        disc[i] = __ffma2_rn(nx, x, __ffma2_rn(ny, y, R2));
      }
      bool cand = false;
#pragma unroll
      for (int i = 0; i < kPairsPerBatch; ++i) cand |= (disc[i].x >= 0.f) | (disc[i].y >= 0.f);
      cand &= act;
      if (__any_sync(kFull, cand)) {
#pragma unroll
        for (int i = 0; i < 2 * kPairsPerBatch; ++i) {
          const int pi = i >> 1;
          const float dd = (i & 1) ? disc[pi].y : disc[pi].x;
          if (act && dd >= 0.f) {
            const int k = 2 * (base + pi) + (i & 1);
            const float cx = (i & 1) ? CX[pi].y : CX[pi].x;
            const float cy = (i & 1) ? CY[pi].y : CY[pi].x;
            const float cz = (i & 1) ? CZ[pi].y : CZ[pi].x;
            const float tc = fmaf(cx, d.x, fmaf(cy, d.y, fmaf(cz, d.z, od)));
            const float q = sqrtf(dd);
            float t0 = tc - q, t1 = tc + q;
            if (k == self_s) {  // leaving this sphere: only its far root can be real (R#12)
              t0 = -kInf;
              if (!self_in) t1 = -kInf;
            }
            const float ts = (t0 >= kEps) ? t0 : t1;
            if (ts >= kEps && ts < tmax) {
              hs = k; hp = -1;
              if (shadow) act = false; else tmax = ts;
            }
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
  L.Lpix = L.Lpix + L.Ls;
  if constexpr (kDebug) {
    const long long si = (long long)(L.py * P.W + L.px) * P.spp + L.s;
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

template <bool kDebug>
__device__ void bounce(Lane& L, const DevParams& P, const DevScene& S, const DevOutputs& O) {
  if (L.depth == P.max_depth) { finish_sample<kDebug>(L, P, O); return; }
  const DevMat m = S.mats[L.mat];
  float3 dn;
  if (m.kind == 1) {  // SPECULAR: mirror, T *= rho
    dn = L.d - L.n * (2.0f * dot3(L.d, L.n));
    L.T = mul(L.T, f3(m.ar, m.ag, m.ab));
  } else if (m.kind == 0) {  // DIFFUSE: mirror with weight kr when kr > 0 (R#8)
    if (!(m.kr > 0.f)) { finish_sample<kDebug>(L, P, O); return; }
    dn = L.d - L.n * (2.0f * dot3(L.d, L.n));
    L.T = L.T * m.kr;
  } else {  // REFRACTIVE: Schlick-chosen reflect / refract, TIR -> reflect (R#9-R#11)
    const float eta = L.entering ? 1.0f / m.ior : m.ior;
    const float ci = -dot3(L.d, L.n);
    const float sin2t = eta * eta * (1.0f - ci * ci);
    bool refl = sin2t > 1.0f;
    if (!refl) {
      const float cosT = sqrtf(fmaxf(1.0f - sin2t, 0.f));
      const float c = L.entering ? ci : cosT;
      float r0 = (1.0f - m.ior) / (1.0f + m.ior);
      r0 *= r0;
      const float mm = 1.0f - c;
      const float F = r0 + (1.0f - r0) * (mm * mm * mm * mm * mm);
      const float u = rng_u(P.seed, (unsigned long long)L.py * P.W + L.px, L.s, L.depth);
      refl = u < F;
      if (!refl) dn = L.d * eta + L.n * (eta * ci - cosT);
    }
    if (refl) dn = L.d - L.n * (2.0f * dot3(L.d, L.n));
    L.T = mul(L.T, f3(m.ar, m.ag, m.ab));
  }
  L.o = L.p;
  L.d = normalize3(dn);
  L.depth++;
  L.n_secondary++;
  L.qkind = Q_CLOSEST;
  L.qo = L.o; L.qd = L.d; L.tmax = kInf;
  L.self_s = L.hit_sph; L.self_p = L.hit_pl;
  L.self_in = (L.hit_sph >= 0) && (dot3(L.d, L.ng) < 0.f);
}

template <bool kDebug>
__device__ void next_light_or_bounce(Lane& L, const DevParams& P, const DevScene& S,
                                     const DevOutputs& O) {
  const DevMat m = S.mats[L.mat];
  if (m.kind == 0) {
    while (L.light < P.n_lights) {
      const DevLight lt = S.lights[L.light];
      L.light++;
      const float3 Pl = f3(lt.px, lt.py, lt.pz);
      const float3 w = Pl - L.p;
      const float d2 = dot3(w, w);
      if (d2 < 1e-12f) continue;                   // R#28
      const float3 wi = w * rsqrtf(d2);
      const float cosT = dot3(L.n, wi);
      if (cosT <= 0.f) continue;                   // no shadow ray
      // shadow ray from p + EPS_T n toward the light (Alg. 1 "emit a shadow light")
      const float3 os = fma3(L.n, kEps, L.p);
      const float3 ws = Pl - os;
      const float tl = sqrtf(dot3(ws, ws));
      L.qo = os;
      L.qd = ws * (1.0f / tl);
      L.tmax = tl;
      L.qkind = Q_SHADOW;
      L.self_s = L.hit_sph; L.self_p = L.hit_pl;
      L.self_in = (L.hit_sph >= 0) && !L.entering;
      L.n_shadow++;
      // f_r = rho/pi + ks (s+2)/(2 pi) max(0, r.wo)^s (Eq. 5, R#3); E = I cos / d^2 (Eq. 3)
      const float3 rl = L.n * (2.0f * cosT) - wi;
      const float alpha = fmaxf(0.f, -dot3(rl, L.d));
      const float spec = m.ks * (m.shin + 2.0f) * kInv2Pi * powf(alpha, m.shin);
      const float g = cosT / d2;
      L.contrib = mul(L.T, f3((fmaf(m.ar, kInvPi, spec)) * lt.ix * g, (fmaf(m.ag, kInvPi, spec)) * lt.iy * g,
                              (fmaf(m.ab, kInvPi, spec)) * lt.iz * g));
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
    const long long si = (long long)(L.py * P.W + L.px) * P.spp + L.s;
    O.dbg_hits[si * (P.max_depth + 1) + L.depth] = prim;
  }
  if (prim < 0) {  // miss -> background
    L.Ls = L.Ls + mul(L.T, f3(P.bg[0], P.bg[1], P.bg[2]));
    finish_sample<kDebug>(L, P, O);
    return;
  }
  const float t = L.tmax;
  L.p = fma3(L.d, t, L.o);
  if (hp >= 0) {
    const DevPlane pl = c_planes[hp];
    L.ng = f3(pl.nx, pl.ny, pl.nz);
    L.mat = pl.mat;
  } else {
    const float4 cr = S.sph_cr[hs];
    const float3 oc = L.o - f3(cr.x, cr.y, cr.z);
    L.ng = normalize3(fma3(L.d, t, oc));
    L.mat = S.sph_mat[hs];
  }
  L.hit_prim = prim; L.hit_sph = hs; L.hit_pl = hp;
  L.entering = dot3(L.d, L.ng) < 0.f;
  L.n = L.entering ? L.ng : L.ng * -1.0f;
  const DevMat m = S.mats[L.mat];
  L.Ls = L.Ls + mul(L.T, f3(m.er, m.eg, m.eb));                 // Eq. 7 emission
  if (m.kind == 0) L.Ls = L.Ls + mul(L.T, f3(m.ar * P.amb[0], m.ag * P.amb[1], m.ab * P.amb[2]));
  L.light = 0;
  next_light_or_bounce<kDebug>(L, P, S, O);
}

template <bool kDebug>
__device__ __forceinline__ void advance(Lane& L, const DevParams& P, const DevScene& S, const DevOutputs& O) {
  if (L.qkind == Q_CLOSEST) {
    on_closest<kDebug>(L, P, S, O);
  } else if (L.qkind == Q_SHADOW) {
    if (L.qs < 0 && L.qp < 0) L.Ls = L.Ls + L.contrib;  // visible: add f_r I cos / d^2
    next_light_or_bounce<kDebug>(L, P, S, O);
  }
}

// ---- the persistent megakernel --------------------------------------------------------------
template <bool kConst, bool kDebug>
__global__ void __launch_bounds__(256, 2)
render_kernel(const DevParams P, const DevScene S, const DevOutputs O) {
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
    intersect<kConst>(L, P, S);
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
cudaError_t upload_const_scene(const float4* pairs, int n_pair_float4, const DevPlane* planes,
                               int n_planes, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  if (n_pair_float4 > 0)
    e = cudaMemcpyToSymbolAsync(c_pairs, pairs, sizeof(float4) * n_pair_float4, 0,
                                cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && n_planes > 0)
    e = cudaMemcpyToSymbolAsync(c_planes, planes, sizeof(DevPlane) * n_planes, 0,
                                cudaMemcpyHostToDevice, st);
  return e;
}

template <bool kConst, bool kDebug>
static int blocks_per_sm_t() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, render_kernel<kConst, kDebug>, 256, 0);
  return n > 0 ? n : 1;
}

int render_blocks_per_sm(bool const_scene, bool debug) {
  if (const_scene) return debug ? blocks_per_sm_t<true, true>() : blocks_per_sm_t<true, false>();
  return debug ? blocks_per_sm_t<false, true>() : blocks_per_sm_t<false, false>();
}

cudaError_t launch_render(const DevParams& p, const DevScene& sc, const DevOutputs& o,
                          bool const_scene, int num_sms, cudaStream_t st) {
  const bool dbg = o.dbg_hits != nullptr;
  const int bps = render_blocks_per_sm(const_scene, dbg);
  long long want = (long long)num_sms * bps;
  const long long max_useful = ((long long)p.n_items + 255) / 256;  // no idle CTAs on tiny frames
  const int grid = (int)(want < max_useful ? want : (max_useful > 0 ? max_useful : 1));
  if (const_scene) {
    if (dbg) render_kernel<true, true><<<grid, 256, 0, st>>>(p, sc, o);
    else render_kernel<true, false><<<grid, 256, 0, st>>>(p, sc, o);
  } else {
    if (dbg) render_kernel<false, true><<<grid, 256, 0, st>>>(p, sc, o);
    else render_kernel<false, false><<<grid, 256, 0, st>>>(p, sc, o);
  }
  return cudaGetLastError();
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
