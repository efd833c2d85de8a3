// rt_kernels.cu — sm_100a kernels of the ray-tracing hot path (arXiv 1504.03151).
//
// One persistent "wavefront-in-a-warp" megakernel:
//   * every lane owns one pixel at a time (all spp samples, summed in order s = 0..spp-1);
//     finished lanes refill from a global work counter with one warp-aggregated atomicAdd
//     (ballot + popc + shfl), so warps stay full until the queue drains (path regeneration);
//   * each round, every lane has exactly one ray query — a closest-hit query (primary or
//     secondary ray) or an any-hit shadow query — and the whole warp runs ONE intersection
//     loop over the scene: sphere data is warp-uniform (shared memory) and two spheres are
//     tested per FFMA2 instruction by a conservative float32 filter; the rare candidates are
//     decided in float64 from the exact float inputs (same decisions as a double-precision
//     reference up to double rounding);
//   * between rounds each lane advances its own small state machine (float64 geometry):
//     ray generation (a2), shading with emission/ambient/Lambert/Phong (a4), shadow-ray set-up
//     (a5), the stack-free reflection/refraction continuation (a6), and the 16-byte store (a7).
// Paper: "each kernel thread traces a single light"; recursion becomes iteration
// (P:226); ray–sphere per Eq. 9–12; shading per Eq. 3–7 for point
// lights; Alg. 1 any-hit with early exit.
#include <cmath>
#include <cuda_runtime.h>
#include <cstdint>

#include "rt_device.cuh"
#include "rt_wavefront.cuh"

namespace rt {

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
  // NEXT-1 / NEXT-2 (kExt kernels only): emitter a shadow query must not test, cosine-bounce
  // flag (R#43), float64 progressive sums of the pixel (R#42)
  int qskip, prevd;
  double acc0, acc1, acc2;
  // stats
  unsigned n_primary, n_shadow, n_secondary;
  unsigned long long n_stests, n_ptests, n_ctests;
};

__device__ __forceinline__ void start_sample(Lane& L, const DevParams& P) {
  L.o = mk(P.eye[0], P.eye[1], P.eye[2]);
  L.d = camera_dir(P, L.px, L.py, L.s);  // stratified / Hammersley, or random jitter (R#42)
  L.T = f3(1.f, 1.f, 1.f);
  L.Ls = f3(0.f, 0.f, 0.f);
  L.depth = 0;
  L.prevd = 0;
  L.qskip = -1;
  L.qkind = Q_CLOSEST;
  L.qo = L.o; L.qd = L.d; L.tmax = kInf;
  L.n_primary++;
}

__device__ __forceinline__ bool start_item(Lane& L, const DevParams& P, int w, float4* out) {
  int t = w / kTilePx;
  const int i = w % kTilePx;
  if (P.mode >= 1) {
    t = rank_tile(t, P.rank, P.world);
    if (t >= P.n_tiles) {
      if (P.mode == 1) out[w] = make_float4(0.f, 0.f, 0.f, 0.f);
      return false;
    }
  }
  const int ty = (int)fdiv(P.div_tiles_x, (unsigned)t);  // t / tiles_x
  const int px = (t - ty * P.tiles_x) * kTileW + (i % kTileW);
  const int py = ty * kTileH + (i / kTileW);
  if (px >= P.W || py >= P.H) {
    if (P.mode == 1) out[w] = make_float4(0.f, 0.f, 0.f, 0.f);
    return false;
  }
  L.item = w; L.px = px; L.py = py; L.s = 0;
  L.Lpix = f3(0.f, 0.f, 0.f);
  start_sample(L, P);
  return true;
}

template <bool kExt>
__device__ __forceinline__ void load_accum(Lane& L, const DevParams& P, const DevOutputs& O) {
  if constexpr (kExt) {
    if (O.accum) {
      const double* a = O.accum + 3 * ((long long)L.py * P.W + L.px);
      L.acc0 = a[0]; L.acc1 = a[1]; L.acc2 = a[2];
    }
  }
}

template <bool kSmem, bool kExt>
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

  // Spheres: float32 filter (RayFilter), candidates decided in float64.
  RayFilter F;
  F.init(o, d, P);
  constexpr int kSrc = kSmem ? SRC_SMEM : SRC_GLOBAL;
  // Candidates of one 16-sphere batch (mask bit i = sphere 2*base + i), in index order:
  // float range prefilter (the chord [tc - q, tc + q] lies before EPS_T or beyond tmax with
  // margin: tc error <= eta, q <= sqrt(disc_f + slack)), then the float64 decision.
  auto process = [&](unsigned cand, int base) {
    const float tmax_hi = (float)tmax * 1.000001f + F.eta;
    while (cand != 0u && act) {
      const int i = __ffs(cand) - 1;
      cand &= cand - 1u;
      const int k = 2 * base + i;  // pair (base + i/2), half i&1
      if (k >= P.n_spheres) break;  // padding (only reachable when the slack exceeds the dummy margin)
      if (kExt && shadow && k == L.qskip) continue;  // the emitter a shadow ray aims at (R#41)
      float dd, tc;
      F.sphere<kSrc>(pairs, k, dd, tc);
      const float qh = sqrtf(fmaxf(dd - F.neg_slack, 0.f));
      if (tc + qh < (float)kEps - F.eta || tc - qh > tmax_hi) continue;
      const double t = sphere_root(__ldg(S.sph_cr + k), o, d);
      // closest hits: a sphere at the same t as the plane found first wins iff its primitive
      // index is lower; shadow rays stop at any occluder (the counts are fixed below)
      if (t >= kEps && (t < tmax || (!shadow && t == tmax && hp >= 0 && S.sph_prim[k] < c_planes[hp].prim))) {
        hs = k; hp = -1;
        if (shadow) act = false; else tmax = t;
      }
    }
  };
  // A warp without closest-hit lanes decides candidates inside the loop and leaves it once
  // every shadow lane found an occluder (Alg. 1 `break`). Otherwise the loop runs over the whole
  // scene for the closest-hit lanes anyway, so candidates are queued (batch | mask, FIFO of 4)
  // and decided after the loop with all lanes in parallel instead of one batch at a time.
  const bool may_exit = !__any_sync(kFull, L.qkind == Q_CLOSEST);
  unsigned long long qa = 0ull, qb = 0ull;
  int nq = 0;
  auto pop = [&]() -> unsigned {
    const unsigned e = (unsigned)qa;
    qa = (qa >> 32) | (qb << 32);
    qb >>= 32;
    --nq;
    return e;
  };

  if (__any_sync(kFull, act)) {
    for (int base = 0; base < P.n_pairs_pad; base += kPairsPerBatch) {
      float2 disc[kPairsPerBatch];
      const float dmax = F.batch<kSrc>(pairs, base, disc);
      const bool any_cand = act && dmax >= F.cut;
      if (__any_sync(kFull, any_cand)) {
        if (any_cand) {
          const unsigned cand = batch_mask(disc, F.cut);
          if (may_exit) {
            process(cand, base);
          } else {
            if (nq == 4) {  // FIFO full (rare): decide the queued batches now
              while (nq > 0) { const unsigned e = pop(); process(e & 0xffffu, (int)(e >> 16) * kPairsPerBatch); }
            }
            const unsigned long long e = ((unsigned long long)(base / kPairsPerBatch) << 16) | cand;
            if (nq < 2) qa |= e << (32 * nq); else qb |= e << (32 * (nq - 2));
            ++nq;
          }
        }
      }
      if (may_exit && !__any_sync(kFull, act)) break;  // Alg. 1 `break`, warp-wide
    }
    while (nq > 0) {  // deferred candidates, in index order
      const unsigned e = pop();
      process(e & 0xffffu, (int)(e >> 16) * kPairsPerBatch);
    }
  }
  // algorithmic test counts
  if (L.qkind == Q_CLOSEST) {
    L.n_stests += (unsigned)P.n_spheres;
    L.n_ctests += (unsigned)P.n_spheres;
    L.n_ptests += (unsigned)P.n_planes;
  } else if (L.qkind == Q_SHADOW) {  // up to the first occluder in primitive index order
    unsigned long long ns = 0, np = 0;
    shadow_counts(P, S, o, d, L.tmax, hp, hs, -1, kExt ? L.qskip : -1, ns, np);
    L.n_stests += ns;
    L.n_ptests += np;
  }
  L.tmax = tmax;
  L.qs = hs;
  L.qp = hp;
}

// ---- shading, shadow setup, continuation (a4-a7) --------------------------------------------
template <bool kDebug, bool kExt>
__device__ void finish_sample(Lane& L, const DevParams& P, const DevOutputs& O) {
  L.Lpix = add(L.Lpix, L.Ls);
  if constexpr (kExt) {  // progressive sums in pass order, as wf_resolve
    L.acc0 += (double)L.Ls.x;
    L.acc1 += (double)L.Ls.y;
    L.acc2 += (double)L.Ls.z;
  }
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
  if constexpr (kExt) {
    if (O.accum) {
      const long long pix = (long long)L.py * P.W + L.px;
      double* a = O.accum + 3 * pix;
      a[0] = L.acc0; a[1] = L.acc1; a[2] = L.acc2;
      if (O.out) {
        const double inv = 1.0 / (double)(P.sample_base + P.spp);
        O.out[pix] = make_float4((float)(L.acc0 * inv), (float)(L.acc1 * inv), (float)(L.acc2 * inv), 1.0f);
      }
      L.item = -1;
      L.qkind = Q_NONE;
      return;
    }
  }
  const float inv = 1.0f / (float)P.spp;
  const float4 v = make_float4(L.Lpix.x * inv, L.Lpix.y * inv, L.Lpix.z * inv, 1.0f);
  if (P.mode != 1) O.out[(long long)L.py * P.W + L.px] = v;  // 16-byte vector store (row-major)
  else O.out[L.item] = v;
  L.item = -1;
  L.qkind = Q_NONE;
}

template <bool kDebug, bool kExt>
__device__ void bounce(Lane& L, const DevParams& P, const DevScene& S, const DevOutputs& O) {
  if (L.depth == P.max_depth) { finish_sample<kDebug, kExt>(L, P, O); return; }
  const DevMat m = S.mats[L.mat];
  const unsigned long long pix = (unsigned long long)L.py * P.W + L.px;
  const unsigned sg = (unsigned)(P.sample_base + L.s);  // R#42
  d3 dn;
  bool cosine = false;
  if (m.kind == 1) {  // SPECULAR: mirror, T *= rho
    dn = reflect(L.d, L.n);
    L.T = mul(L.T, f3(m.ar, m.ag, m.ab));
  } else if (kExt && m.kind == 0 && P.integrator == 1) {  // global: cosine-weighted bounce (R#40)
    dn = cosine_dir(L.n, rng_stream(P.seed, pix, sg, L.depth, 3u), rng_stream(P.seed, pix, sg, L.depth, 4u));
    L.T = mul(L.T, f3(m.ar, m.ag, m.ab));
    cosine = true;
  } else if (m.kind == 0) {  // DIFFUSE: mirror with weight kr when kr > 0 (R#8)
    if (!(m.kr > 0.f)) { finish_sample<kDebug, kExt>(L, P, O); return; }
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
      const double u = rng_u(P.seed, pix, (int)sg, L.depth);
      refl = u < F;
      if (!refl) dn = L.d * eta + L.n * (eta * ci - cosT);
    }
    if (refl) dn = reflect(L.d, L.n);
    L.T = mul(L.T, f3(m.ar, m.ag, m.ab));
  }
  L.o = L.p;
  L.d = normalize(dn);
  L.depth++;
  L.prevd = cosine ? 1 : 0;
  L.n_secondary++;
  L.qkind = Q_CLOSEST;
  L.qo = L.o; L.qd = L.d; L.tmax = kInf;
}

template <bool kDebug, bool kExt>
__device__ void next_light_or_bounce(Lane& L, const DevParams& P, const DevScene& S,
                                     const DevOutputs& O) {
  const DevMat m = S.mats[L.mat];
  if (kExt && m.kind == 0) {  // point lights, then one surface sample per emitter (R#41)
    const unsigned long long pix = (unsigned long long)L.py * P.W + L.px;
    const unsigned sg = (unsigned)(P.sample_base + L.s);
    while (L.light < P.n_lights + P.n_emitters) {
      const int l = L.light++;
      LightSample ls;
      if (!light_sample(P, S, l, L.p, L.n, pix, sg, L.depth, ls)) continue;
      double tl;
      d3 os, ds;
      if (l < P.n_lights) {
        shadow_ray(S, L.p, L.n, l, os, ds, tl);
        L.qskip = -1;
      } else {
        shadow_ray_to(L.p, L.n, ls.x, os, ds, tl);
        L.qskip = S.emit_sph[l - P.n_lights];
      }
      L.qo = os;
      L.qd = ds;
      L.tmax = tl;
      L.qkind = Q_SHADOW;
      L.n_shadow++;
      const d3 rl = L.n * (2.0 * ls.cos_s) - ls.wi;
      const float alpha = (float)fmax(0.0, -dot(rl, L.d));
      const float spec = m.ks * (m.shin + 2.0f) * kInv2Pi * phong_lobe(alpha, m.shin);
      const float g = (float)ls.g;
      L.contrib = mul(L.T, f3(fmaf(m.ar, kInvPi, spec) * ls.ir * g, fmaf(m.ag, kInvPi, spec) * ls.ig * g,
                              fmaf(m.ab, kInvPi, spec) * ls.ib * g));
      return;
    }
  } else if (m.kind == 0) {
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
      const float spec = m.ks * (m.shin + 2.0f) * kInv2Pi * phong_lobe(alpha, m.shin);
      const float g = (float)(cosT / d2);
      L.contrib = mul(L.T, f3(fmaf(m.ar, kInvPi, spec) * lt.ix * g, fmaf(m.ag, kInvPi, spec) * lt.iy * g,
                              fmaf(m.ab, kInvPi, spec) * lt.iz * g));
      return;
    }
  }
  bounce<kDebug, kExt>(L, P, S, O);
}

template <bool kDebug, bool kExt>
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
    finish_sample<kDebug, kExt>(L, P, O);
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
  // Eq. 7 emission, except an emitter already sampled from the previous diffuse vertex (R#43)
  if (!(kExt && L.prevd && P.n_emitters > 0 && hs >= 0)) L.Ls = add(L.Ls, mul(L.T, f3(m.er, m.eg, m.eb)));
  if (m.kind == 0) L.Ls = add(L.Ls, mul(L.T, f3(m.ar * P.amb[0], m.ag * P.amb[1], m.ab * P.amb[2])));
  L.light = 0;
  next_light_or_bounce<kDebug, kExt>(L, P, S, O);
}

template <bool kDebug, bool kExt>
__device__ __forceinline__ void advance(Lane& L, const DevParams& P, const DevScene& S, const DevOutputs& O) {
  if (L.qkind == Q_CLOSEST) {
    on_closest<kDebug, kExt>(L, P, S, O);
  } else if (L.qkind == Q_SHADOW) {
    if (L.qs < 0 && L.qp < 0) L.Ls = add(L.Ls, L.contrib);  // visible: add f_r I cos / d^2
    next_light_or_bounce<kDebug, kExt>(L, P, S, O);
  }
}

// ---- the persistent megakernel --------------------------------------------------------------
constexpr int kMegaMinBlocks = 2;  // 128 registers per lane state machine: 2 CTAs x 8 warps per SM
template <bool kSmem, bool kDebug, bool kExt>
__global__ void __launch_bounds__(256, kMegaMinBlocks)
render_kernel(const DevParams P, const DevScene S, const DevOutputs O) {
  __shared__ uint64_t s_mbar;
  if constexpr (kSmem) stage_scene(s_pairs, S.pairs, (uint32_t)P.n_pairs_pad * 32u, &s_mbar);
  const float4* pairs = S.pairs;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  Lane L;
  L.item = -1; L.qkind = Q_NONE;
  L.n_primary = L.n_shadow = L.n_secondary = 0;
  L.n_stests = L.n_ptests = L.n_ctests = 0ull;
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
        else if (start_item(L, P, (int)w, O.out)) load_accum<kExt>(L, P, O);
      }
    }
    if (!__any_sync(kFull, L.qkind != Q_NONE)) break;
    intersect<kSmem, kExt>(L, P, S, pairs);
    advance<kDebug, kExt>(L, P, S, O);
  }

  // stats: warp reduction, one atomic per warp
  unsigned long long v[6] = {L.n_primary, L.n_shadow, L.n_secondary, L.n_stests, L.n_ptests, L.n_ctests};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(kFull, v[k], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) atomicAdd(O.stats + k, v[k]);
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
    const int j = t / world, r = ((t % world) - j % world + world) % world;  // inverse of rank_tile
    const int i = (py % kTileH) * kTileW + (px % kTileW);
    out[pix] = g[r * slab_f4 + (long long)j * kTilePx + i];
  }
}

__global__ void sum_stats_kernel(const float4* __restrict__ g, int world, int tpr,
                                 unsigned long long* stats) {
  if (threadIdx.x < 6) {
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

// ---- shared-origin tables (rt_api.cu: the eye's after rt_camera_set, the lights' after upload) -
// Tangent test: -h = -sqrt((|c - o| - r)(|c - o| + r)) per sphere in FP64 from the
// float inputs, rounded once; +3e38 (always a candidate) when o is inside the sphere or within
// 1e-6 S of its surface; -1e30 for the padding slots (never a candidate).
__device__ __forceinline__ float neg_tangent(const float4 cr, double ox, double oy, double oz, double S) {
  const double x = (double)cr.x - ox, y = (double)cr.y - oy, z = (double)cr.z - oz;
  const double dist = sqrt(x * x + y * y + z * z), r = cr.w;
  if (dist - r <= 1e-6 * S) return 3.0e38f;
  return (float)-sqrt((dist - r) * (dist + r));
}
// The eye's table: pair q = {c'x, c'y | c'z, -h}, then s1 = K + 2 c'.o' (FP64, rounded once) for
// the candidates' chord bounds. One thread per pair.
__global__ void build_eye_table(const float4* __restrict__ pairs, const float4* __restrict__ sph_cr, int ns, int npp,
                                double ox, double oy, double oz, double cx, double cy, double cz, double S,
                                float4* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npp) return;
  const float4 a = pairs[2 * q], b = pairs[2 * q + 1];
  const double px = ox - cx, py = oy - cy, pz = oz - cz;  // o' = o - centre
  float4 nb = b;
  nb.z = 2 * q < ns ? neg_tangent(sph_cr[2 * q], ox, oy, oz, S) : -1e30f;
  nb.w = 2 * q + 1 < ns ? neg_tangent(sph_cr[2 * q + 1], ox, oy, oz, S) : -1e30f;
  out[2 * q] = a;
  out[2 * q + 1] = nb;
  float2* s1 = reinterpret_cast<float2*>(out + 2 * npp);
  s1[q] = make_float2((float)((double)b.z + 2.0 * ((double)a.x * px + (double)a.z * py + (double)b.x * pz)),
                      (float)((double)b.w + 2.0 * ((double)a.y * px + (double)a.w * py + (double)b.y * pz)));
}
// The light-origin tables: the pairs, then -h of light l for every sphere slot k
// (out + 2 npp as floats, [l][2 npp]: the short-list scan stages all of them); and per light the
// pair layout with -h in place of K (out_pl, [l][2 npp] float4: the long-list scan stages one).
// One thread per (light, sphere slot).
__global__ void build_light_tables(const float4* __restrict__ pairs, const float4* __restrict__ sph_cr,
                                   const DevLight* __restrict__ lights, int ns, int npp, int n_lights, double cx,
                                   double cy, double cz, float cmax, float rmax, float4* __restrict__ out,
                                   float4* __restrict__ out_pl) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 2 * npp) out[i] = pairs[i];
  if (i >= n_lights * 2 * npp) return;
  const int l = i / (2 * npp), k = i - l * 2 * npp;
  const DevLight L = lights[l];
  const double ox = L.px, oy = L.py, oz = L.pz;
  const double px = ox - cx, py = oy - cy, pz = oz - cz;
  const double S = (double)cmax + sqrt(px * px + py * py + pz * pz) + (double)rmax;
  const float nh = k < ns ? neg_tangent(sph_cr[k], ox, oy, oz, S) : -1e30f;
  reinterpret_cast<float*>(out + 2 * npp)[i] = nh;
  // per-light pair layout: pair q = k / 2, float4 {cx0, cx1, cy0, cy1} then {cz0, cz1, nh0, nh1};
  // after the 2 npp float4, K as {K0, K1} per pair
  const int q = k >> 1, h = k & 1;
  float4* T = out_pl + (size_t)l * lt_table_stride(npp);
  if (h == 0) T[2 * q] = pairs[2 * q];
  float* b = reinterpret_cast<float*>(&T[2 * q + 1]);
  const float* pb = reinterpret_cast<const float*>(&pairs[2 * q + 1]);
  b[h] = pb[h];  // c'z
  b[2 + h] = nh;
  reinterpret_cast<float*>(T + 2 * npp)[k] = pb[2 + h];  // K
}

cudaError_t launch_eye_table(const float4* pairs, const float4* sph_cr, int ns, int npp, const double o[3],
                             const double centre[3], double S, float4* out, cudaStream_t st) {
  build_eye_table<<<(npp + 255) / 256, 256, 0, st>>>(pairs, sph_cr, ns, npp, o[0], o[1], o[2], centre[0], centre[1],
                                                     centre[2], S, out);
  return cudaGetLastError();
}
cudaError_t launch_light_tables(const float4* pairs, const float4* sph_cr, const DevLight* lights, int ns, int npp,
                                int n_lights, const double centre[3], float cmax, float rmax, float4* out,
                                float4* out_per_light, cudaStream_t st) {
  const int n = (n_lights > 1 ? n_lights : 1) * 2 * npp;
  build_light_tables<<<(n + 255) / 256, 256, 0, st>>>(pairs, sph_cr, lights, ns, npp, n_lights, centre[0], centre[1],
                                                      centre[2], cmax, rmax, out, out_per_light);
  return cudaGetLastError();
}

// sample_offset's values for spp <= kOffTable, in the same IEEE double operations (x86-64 SSE2,
// no FMA contraction: the device table then holds exactly what sample_offset computes)
cudaError_t upload_sample_offsets(int spp, cudaStream_t st) {
  if (spp < 1 || spp > kOffTable) return cudaSuccess;
  static double2 off[kOffTable];
  int n = 1;
  while ((n + 1) * (n + 1) <= spp) ++n;
  for (int s = 0; s < spp; ++s) {
    if (n * n == spp) {
      const int i = s % n, j = s / n;
      off[s] = make_double2((i + 0.5) / n, (j + 0.5) / n);
    } else {
      unsigned v = (unsigned)s, r = 0;
      for (int b = 0; b < 32; ++b) { r = (r << 1) | (v & 1u); v >>= 1; }
      const double radinv = (double)r * (1.0 / 4294967296.0);
      const double y = radinv + 0.5 / spp;
      off[s] = make_double2((s + 0.5) / spp, y - std::floor(y));
    }
  }
  return cudaMemcpyToSymbolAsync(c_sample_off, off, sizeof(double2) * spp, 0, cudaMemcpyHostToDevice, st);
}

// ---- launchers ------------------------------------------------------------------------------
cudaError_t upload_planes(const DevPlane* planes, int n_planes, cudaStream_t st) {
  if (n_planes <= 0) return cudaSuccess;
  return cudaMemcpyToSymbolAsync(c_planes, planes, sizeof(DevPlane) * n_planes, 0, cudaMemcpyHostToDevice, st);
}

template <bool kSmem, bool kDebug, bool kExt>
static cudaError_t launch_t(const DevParams& p, const DevScene& sc, const DevOutputs& o, int num_sms,
                           cudaStream_t st, int* blocks_per_sm_out) {
  const size_t smem = kSmem ? (size_t)p.n_pairs_pad * 32u : 0u;
  auto kern = render_kernel<kSmem, kDebug, kExt>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem > 0 ? smem : 1));
  if (e != cudaSuccess) return e;
  int bps = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, smem);
  if (e != cudaSuccess) return e;
  if (bps < 1) bps = 1;
  if (blocks_per_sm_out) *blocks_per_sm_out = bps;
  const long long want = (long long)num_sms * bps;
  const long long max_useful = ((long long)p.n_items + 255) / 256;  // no idle CTAs on tiny frames
  const int grid = (int)(want < max_useful ? want : (max_useful > 0 ? max_useful : 1));
  kern<<<grid, 256, smem, st>>>(p, sc, o);
  return cudaGetLastError();
}

template <bool kExt>
static cudaError_t launch_x(const DevParams& p, const DevScene& sc, const DevOutputs& o, bool smem_scene, int num_sms,
                            cudaStream_t st) {
  const bool dbg = o.dbg_hits != nullptr;
  if (smem_scene) return dbg ? launch_t<true, true, kExt>(p, sc, o, num_sms, st, nullptr)
                             : launch_t<true, false, kExt>(p, sc, o, num_sms, st, nullptr);
  return dbg ? launch_t<false, true, kExt>(p, sc, o, num_sms, st, nullptr)
             : launch_t<false, false, kExt>(p, sc, o, num_sms, st, nullptr);
}

// kExt: the NEXT-1 / NEXT-2 modes (global integrator, area lights, progressive passes); the
// plain instantiation keeps the hot path's register budget
cudaError_t launch_render(const DevParams& p, const DevScene& sc, const DevOutputs& o, bool smem_scene,
                          int num_sms, cudaStream_t st) {
  const bool ext = p.integrator != 0 || p.n_emitters > 0 || p.jitter != 0 || o.accum != nullptr;
  return ext ? launch_x<true>(p, sc, o, smem_scene, num_sms, st) : launch_x<false>(p, sc, o, smem_scene, num_sms, st);
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

__global__ void sum_records_kernel(const unsigned long long* __restrict__ rec, int world, unsigned long long* stats) {
  if (threadIdx.x < 8) {
    unsigned long long v = 0;
    for (int r = 0; r < world; ++r) v += rec[r * 8 + threadIdx.x];
    stats[threadIdx.x] = v;
  }
}

cudaError_t launch_sum_records(const unsigned long long* rec, int world, unsigned long long* stats, cudaStream_t st) {
  sum_records_kernel<<<1, 32, 0, st>>>(rec, world, stats);
  return cudaGetLastError();
}

cudaError_t read_check_status(unsigned* first_failed) {
  cudaError_t e = cudaMemcpyFromSymbol(first_failed, g_rt_check, sizeof(unsigned));
  if (e != cudaSuccess) return e;
  const unsigned zero = 0;
  return cudaMemcpyToSymbol(g_rt_check, &zero, sizeof(unsigned));
}

cudaError_t launch_tonemap(const float4* rgba, uint8_t* out, int64_t n, float exposure, float gamma,
                           cudaStream_t st) {
  int grid = (int)((n + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  tonemap_kernel<<<grid, 256, 0, st>>>(rgba, reinterpret_cast<uchar4*>(out), n, exposure, 1.0f / gamma);
  return cudaGetLastError();
}

// ---- wavefront launcher ---------------------------------------------------------------------
static int lt_sub_cap(int cap) {  // slots per sub-list: the 256-path blocks of one residue class
  return ((cap + 256 * kLtSub - 1) / (256 * kLtSub)) * 256;
}

size_t wf_bytes(int cap, int scap, int gcap, int lt_lists, int xctas) {
  const size_t q = 4 + 6 * 8 + 3 * 4 + 3 * 4 + 4 + 4;  // one WfQueue entry
  const size_t slots = (size_t)lt_lists * lt_sub_cap(cap);
  return (size_t)cap * (2 * q + 3 * 4 + 3 * 4 + kCandMax * 4 + 4 + 3 * 8) + (size_t)scap * (3 * 4 + 4) +
         slots * (16 + 8 + 8 + kCandMax * 4) + (size_t)gcap * (7 * 8 + 4 + 4 + kCandMax * 4 + 4 + 4) +
         (size_t)xctas * 8 * (32 * 2 + 64) * kCandMax * 4 + 64 * 256;
}

void wf_carve(WfBuffers& B, void* base, int cap, int scap, int gcap, int lt_lists, int xctas, unsigned* ctr) {
  char* p = static_cast<char*>(base);
  auto take = [&](size_t bytes) { char* r = p; p += (bytes + 255) & ~size_t(255); return r; };
  B.cap = cap;
  B.scap = scap;
  B.gcap = gcap;
  B.lt_cap = lt_sub_cap(cap);
  const size_t slots = (size_t)lt_lists * B.lt_cap;
  for (int k = 0; k < 2; ++k) {
    WfQueue& Q = B.q[k];
    Q.path = reinterpret_cast<int*>(take(4 * (size_t)cap));
    Q.ray = reinterpret_cast<double*>(take(6 * 8 * (size_t)cap));
    Q.T = reinterpret_cast<float*>(take(3 * 4 * (size_t)cap));
    Q.L = reinterpret_cast<float*>(take(3 * 4 * (size_t)cap));
    Q.depth = reinterpret_cast<int*>(take(4 * (size_t)cap));
    Q.skip = reinterpret_cast<int*>(take(4 * (size_t)cap));
  }
  B.Lr = reinterpret_cast<float*>(take(3 * 4 * (size_t)cap));
  B.nxt = reinterpret_cast<int*>(take(4 * (size_t)cap));
  B.shoff = reinterpret_cast<int*>(take(4 * (size_t)cap));
  B.shcnt = reinterpret_cast<int*>(take(4 * (size_t)cap));
  B.ccand = reinterpret_cast<int*>(take(4 * (size_t)kCandMax * cap));
  B.cn = reinterpret_cast<int*>(take(4 * (size_t)cap));
  B.sorg = reinterpret_cast<double*>(take(3 * 8 * (size_t)cap));
  B.sq_c = reinterpret_cast<float*>(take(3 * 4 * (size_t)scap));
  B.spos = reinterpret_cast<int*>(take(4 * (size_t)scap));
  B.lt_dir = reinterpret_cast<float4*>(take(16 * (slots ? slots : 1)));
  B.lt_rec = reinterpret_cast<int2*>(take(8 * (slots ? slots : 1)));
  B.lt_res = reinterpret_cast<int2*>(take(8 * (slots ? slots : 1)));
  B.lt_cand = reinterpret_cast<int*>(take(4 * (size_t)kCandMax * (slots ? slots : 1)));
  B.sray = reinterpret_cast<double*>(take(7 * 8 * (size_t)gcap));
  B.sskip = reinterpret_cast<int*>(take(4 * (size_t)gcap));
  B.sskip2 = reinterpret_cast<int*>(take(4 * (size_t)gcap));
  B.scand = reinterpret_cast<int*>(take(4 * (size_t)kCandMax * gcap));
  B.sn = reinterpret_cast<int*>(take(4 * (size_t)gcap));
  B.srob = reinterpret_cast<int*>(take(4 * (size_t)gcap));
  B.xctas = xctas;
  B.solo = 0;
  B.force_parts = -1;
  B.xcand_c = reinterpret_cast<int*>(take(4 * (size_t)xctas * 8 * 32 * kCandMax));
  B.xlo_c = reinterpret_cast<float*>(take(4 * (size_t)xctas * 8 * 32 * kCandMax));
  B.xcand_s = reinterpret_cast<int*>(take(4 * (size_t)xctas * 8 * 64 * kCandMax));
  B.ctr = ctr;
}

// Chunks of whole work items (pixels): at most 2^22 paths per chunk; a frame that would fill
// fewer chunks than max(slots, p.min_chunks) is cut into that many (each >= 2^17 paths), so the
// chunks overlap (DESIGN.md §7 "chunk pipelining"). A host framebuffer (p.min_chunks > 0) cut
// into exactly 2 x slots chunks gets chunks of falling size (the first `slots` chunks share
// kHostHead of the frame): their rows are copied while the smaller last ones render (C4,
// rt_render into pinned memory: head 0.5 (uniform) / 0.7 / 0.8 / 0.9 / 0.95 -> 6.39 / 6.29 /
// 6.24 / 6.17 / 6.32 ms; device-buffer renders keep uniform chunks).
constexpr double kHostHead = 0.9;
static long long wf_uniform_chunks(const DevParams& p, int nslots) {
  const long long paths = (long long)p.n_items * p.spp;
  const int max_items = (1 << 22) / p.spp > 0 ? (1 << 22) / p.spp : 1;
  long long chunks = (p.n_items + max_items - 1) / max_items;
  const long long want_min = nslots > p.min_chunks ? nslots : p.min_chunks;
  if (want_min > 1 && chunks < want_min) {
    long long want = want_min;
    while (want > 1 && paths / want < (1 << 17)) --want;
    if (want > chunks) chunks = want;
  }
  return chunks < 1 ? 1 : chunks;
}
int wf_chunk_count(const DevParams& p, int nslots) {
  const long long chunks = wf_uniform_chunks(p, nslots);
  const long long items = (p.n_items + chunks - 1) / chunks;
  return (int)((p.n_items + items - 1) / items);
}
// first work item of chunk k (k = wf_chunk_count: n_items)
int wf_chunk_begin(const DevParams& p, int nslots, int k) {
  const long long chunks = wf_uniform_chunks(p, nslots);
  const long long items = (p.n_items + chunks - 1) / chunks;
  const int n = (int)((p.n_items + items - 1) / items);
  if (k >= n) return p.n_items;
  const long long rows = p.n_items / ((long long)p.tiles_x * kTilePx);
  if (p.min_chunks > 0 && nslots > 1 && n == 2 * nslots && kHostHead > 0.0 && rows >= 8LL * n) {
    // falling sizes, boundaries on whole tile rows
    const long long row = (long long)p.tiles_x * kTilePx;
    const double f = k <= nslots ? kHostHead * k / nslots : kHostHead + (1.0 - kHostHead) * (k - nslots) / nslots;
    long long b = (long long)(f * (double)p.n_items / (double)row + 0.5) * row;
    return (int)(b < p.n_items ? b : p.n_items);
  }
  const long long b = (long long)k * items;
  return (int)(b < p.n_items ? b : p.n_items);
}
// the largest chunk (the buffer sets' capacity)
int wf_chunk_max_items(const DevParams& p, int nslots) {
  const int n = wf_chunk_count(p, nslots);
  int m = 1;
  for (int k = 0; k < n; ++k) {
    const int w = wf_chunk_begin(p, nslots, k + 1) - wf_chunk_begin(p, nslots, k);
    if (w > m) m = w;
  }
  return m;
}

int wf_timing_pairs(const DevParams& p, int nslots) { return wf_chunk_count(p, nslots) * (p.max_depth + 1); }

template <typename... KArgs, typename... Args>
static void launch(void (*k)(KArgs...), int grid, size_t smem, cudaStream_t st, Args... args) {
  k<<<grid, 256, smem, st>>>(static_cast<KArgs>(args)...);
}

constexpr int kLogicGridPerSm = 6;  // logic kernels: grid-stride loops (measured C4 world 1 / 8:
                                    // 4 -> 7.00 / 1.10 ms, 6 -> 7.03 / 1.084, 8 -> 7.04 / 1.082)

template <int kSrc>
static cudaError_t wf_run(const DevParams& p, const DevScene& sc, const DevOutputs& o, int num_sms, WfTiming& tm,
                          cudaStream_t st0) {
  WfBuffers& B0 = *tm.slot_B[0];
  const cudaStream_t st = st0;  // setup launches (debug fill) go on the caller's stream
  const bool dbg = o.dbg_hits != nullptr;
  const bool ext = p.n_emitters > 0 || p.integrator != 0;  // wf_shade with the NEXT-1/NEXT-2 paths
  // SRC_TILE (scenes beyond shared memory): the long-queue scans stream TMA tiles; the camera-ray
  // scan and the short-queue split scans read the pairs from global memory
  constexpr int kScan = kSrc == SRC_TILE ? SRC_GLOBAL : kSrc;
  const size_t smem = kSrc == SRC_SMEM ? (size_t)p.n_pairs_pad * 32u : 0u;
  const size_t smem_long = kSrc == SRC_TILE ? (size_t)2 * kTilePairs * 32u : smem;
  cudaError_t e;
  int occ_c = 0, occ_s = 0;
  using IsectFn = void (*)(const DevParams, const DevScene, WfBuffers, int);
  const IsectFn kcl = kSrc == SRC_TILE ? (IsectFn)wf_isect_tiled<false> : (IsectFn)wf_isect<kScan, false>;
  const IsectFn ksl = kSrc == SRC_TILE ? (IsectFn)wf_isect_tiled<true> : (IsectFn)wf_isect<kScan, true>;
  // camera rays (depth 0): two per thread through the shared-origin filter on the eye's pair table
  const IsectFn kc0 = kSrc == SRC_TILE ? (IsectFn)wf_isect_eye2_tiled : (IsectFn)wf_isect_eye2<kScan>;
  const size_t smem_eye = smem_long;  // the eye's pairs (its s1 column stays in global memory)
  // point lights' shadow rays scanned from the light (shared-memory scene with the light tables)
  IsectFn klt = nullptr, klts = nullptr;
  size_t smem_lt = 0, smem_ltl = 0;  // the short-list scan's staging, the long-list scan's (one light's table)
  int grid_lt = 0;
  if constexpr (kSrc == SRC_SMEM) {
    if (p.lt_lights > 0) {
      klt = wf_isect_lt<kSrc>;
      // short lists: every light's column beside the pairs while they fit 64 KB, else light by light
      const bool cols = (size_t)p.lt_lights * p.n_pairs_pad * 8u <= 65536u;
      klts = cols ? (IsectFn)wf_isect_lt_split<kSrc, false> : (IsectFn)wf_isect_lt_split<kSrc, true>;
      smem_ltl = (size_t)lt_table_stride(p.n_pairs_pad) * 16u;  // one light's table
      smem_lt = cols ? (size_t)p.n_pairs_pad * 32u + (size_t)p.lt_lights * p.n_pairs_pad * 8u : smem_ltl;
      if ((e = cudaFuncSetAttribute(klt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_ltl)) != cudaSuccess) return e;
      if ((e = cudaFuncSetAttribute(klts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_lt)) != cudaSuccess) return e;
      int occ = 0;
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, klt, 256, smem_ltl)) != cudaSuccess) return e;
      grid_lt = num_sms * (occ > 0 ? occ : 1);
    }
  }
  for (auto fn : {(IsectFn)wf_isect_split<kScan, false>, (IsectFn)wf_isect_split<kScan, true>}) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem > 0 ? smem : 1));
    if (e != cudaSuccess) return e;
  }
  for (auto fn : {kcl, ksl}) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem_long > 0 ? smem_long : 1));
    if (e != cudaSuccess) return e;
  }
  e = cudaFuncSetAttribute(kc0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem_eye > 0 ? smem_eye : 1));
  if (e != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, kcl, 256, smem_long)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, ksl, 256, smem_long)) != cudaSuccess) return e;
  const int grid_c = num_sms * (occ_c > 0 ? occ_c : 1), grid_s = num_sms * (occ_s > 0 ? occ_s : 1);
  const int grid_l = num_sms * kLogicGridPerSm;
  // the device's split_parts (rt_wavefront.cuh) evaluated on a hinted queue length
  auto host_parts = [&](unsigned tasks, int grid) -> int {
    if (grid > B0.xctas) return 1;
    if (B0.force_parts > 0) return B0.force_parts;
    return split_rule(tasks, (unsigned)grid * 8u);
  };
  using ShadeFn = void (*)(const DevParams, const DevScene, WfBuffers, int, long long, int*, int*);
  const ShadeFn shade = ext ? (dbg ? wf_shade<true, true> : wf_shade<false, true>)
                            : (dbg ? wf_shade<true, false> : wf_shade<false, false>);
  int* dh = dbg ? o.dbg_hits : nullptr;
  int* db = dbg ? o.dbg_bounces : nullptr;
  const int nslots = tm.nslots;  // slots that receive chunks (<= the count the chunking used)
  const int n_chunks_plan = wf_chunk_count(p, tm.nslots_req);
  // schedule fuzzing: a spin of 0-40 us (or none) on a stream at each fork, join and slot start
  auto jitter = [&](cudaStream_t s) {
    if (!tm.jitter || !s) return;
    tm.jitter = tm.jitter * 6364136223846793005ull + 1442695040888963407ull;
    const unsigned r = (unsigned)(tm.jitter >> 33);
    if (r & 1u) launch(spin_ns, 1, 0, s, (r >> 1) % 40000u);
  };
  tm.n = 0;
  tm.launches = 0;
  tm.n_chunks = 0;
  if (dbg) {
    const long long nh = (long long)p.W * p.H * p.spp * (p.max_depth + 1);
    launch(fill_int, num_sms * 8, 0, st, o.dbg_hits, nh, -2);
    ++tm.launches;
  }
  if (nslots > 1) {  // the other slots' streams start after everything issued on st so far
    cudaEventRecord(tm.start_ev, st);
    for (int k = 1; k < nslots; ++k) {
      cudaStreamWaitEvent(tm.slot_main[k], tm.start_ev, 0);
      jitter(tm.slot_main[k]);
    }
  }
  int chunk = 0;
  for (; chunk < n_chunks_plan; ++chunk) {
    const int w0 = wf_chunk_begin(p, tm.nslots_req, chunk);
    const int sl = chunk % nslots;
    WfBuffers& Bset = *tm.slot_B[sl];
    const cudaStream_t st = sl == 0 ? st0 : tm.slot_main[sl];
    const cudaStream_t side = tm.slot_side[sl];
    cudaEvent_t* fork = tm.slot_fork[sl];
    cudaEvent_t* join = tm.slot_join[sl];
    // this chunk's queue counters in the render before the capture (null: launch the pairs)
    const unsigned* hint = tm.hints ? tm.hints + (size_t)chunk * tm.hint_stride : nullptr;
    WfBuffers Bc = Bset;  // this chunk's launches: the buffer set with the chunk's first sample
    Bc.g0 = (long long)w0 * p.spp;
    Bc.w0 = w0;
    WfBuffers Bs = Bc;  // the copy passed to a single (solo) kernel launch
    Bs.solo = 1;
    const int nw = wf_chunk_begin(p, tm.nslots_req, chunk + 1) - w0;
    const int npaths = nw * p.spp;
    const long long g0 = (long long)w0 * p.spp;
    if ((e = cudaMemsetAsync(Bc.ctr, 0, sizeof(unsigned) * kWfCtrPerDepth * (p.max_depth + 2), st)) != cudaSuccess) return e;
    launch(wf_q0_len, 1, 0, st, Bc, npaths);  // camera rays are computed on use (implicit queue)
    // per depth d: closest scan (d) -> shade (d) -> { shadow scan (d) -> accumulate (d) on the side
    // stream  ||  closest scan (d + 1) on the main stream } -> join -> shade (d + 1) ...
    // (independent: the shadow side reads the shadow entries and writes L into Q[d+1]; the closest
    // scan reads Q[d+1]'s rays and writes the candidate lists)
    const int t0 = tm.n;
    auto closest_scan = [&](int dd) {
      const int ti = t0 + dd;
      const bool rec = ti < tm.cap;
      if (rec) tm.record(tm.closest[2 * ti], st);
      if (dd == 0) {
        launch(kc0, grid_c, smem_eye, st, p, sc, Bc, dd);
      } else if (hint) {  // one kernel, chosen from the previous frame's queue of this chunk
        // (grids stay full: a hint that underestimates the queue, e.g. after a camera move, may
        // then cost the split kernel's merges, never a starved grid)
        const unsigned tasks = (hint[wf_ctr_q(dd)] + 31u) / 32u;
        if (host_parts(tasks, grid_c) > 1) launch(wf_isect_split<kScan, false>, grid_c, smem, st, p, sc, Bs, dd);
        else launch(kcl, grid_c, smem_long, st, p, sc, Bs, dd);
      } else {  // the self-selecting pair: both read the queue length, exactly one works
        launch(kcl, grid_c, smem_long, st, p, sc, Bc, dd);
        launch(wf_isect_split<kScan, false>, grid_c, smem, st, p, sc, Bc, dd);
        tm.launches += 1;
      }
      tm.launches += 1;
      if (rec) tm.record(tm.closest[2 * ti + 1], st);
    };
    closest_scan(0);
    for (int d = 0; d <= p.max_depth; ++d) {
      const int ti = t0 + d;
      const bool rec = ti < tm.cap;
      if (rec && tm.shade) tm.record(tm.shade[2 * ti], st);
      const int grid_q = grid_l;  // logic kernels: grid-stride loops
      // wf_shade: one wave of its resident CTAs for large chunks (C4: 3 / 6 / 9 / 12 CTAs per SM
      // 5.603 / 5.618 / 5.629 / 5.633 ms per frame), the logic grid for small ones (a world-8 shard
      // is 0.8 % slower with one wave)
      launch(shade, npaths >= (1 << 21) ? num_sms * kShadeMinBlocks : grid_q, 0, st, p, sc, Bc, d, g0, dh, db);
      if (rec && tm.shade) tm.record(tm.shade[2 * ti + 1], st);
      cudaStream_t ss = st;
      if (side) {
        cudaEventRecord(fork[d], st);
        cudaStreamWaitEvent(side, fork[d], 0);
        ss = side;
        jitter(side);
      }
      if (rec) tm.record(tm.shadow[2 * ti], ss);
      int scan_launches = 0;
      if (klt) {  // point lights, from the light
        if (hint) {
          unsigned chunks = 0;
          for (int i = 0; i < p.lt_lights * kLtSub; ++i) chunks += (hint[wf_ctr_lt(d, 0, 0) + i] + 63u) / 64u;
          if (host_parts(chunks, grid_lt) > 1) launch(klts, grid_lt, smem_lt, ss, p, sc, Bs, d);
          else launch(klt, grid_lt, smem_ltl, ss, p, sc, Bs, d);
          scan_launches += 1;
        } else {
          launch(klt, grid_lt, smem_ltl, ss, p, sc, Bc, d);
          launch(klts, grid_lt, smem_lt, ss, p, sc, Bc, d);
          scan_launches += 2;
        }
      }
      if (!klt || p.n_emitters > 0) {  // every other shadow ray
        if (hint) {
          const unsigned tasks = (hint[wf_ctr_so(d)] + 31u) / 32u;
          if (host_parts(tasks, grid_s) > 1) launch(wf_isect_split<kScan, true>, grid_s, smem, ss, p, sc, Bs, d);
          else launch(ksl, grid_s, smem_long, ss, p, sc, Bs, d);
          scan_launches += 1;
        } else {
          launch(ksl, grid_s, smem_long, ss, p, sc, Bc, d);
          launch(wf_isect_split<kScan, true>, grid_s, smem, ss, p, sc, Bc, d);
          scan_launches += 2;
        }
      }
      if (rec) tm.record(tm.shadow[2 * ti + 1], ss);
      // wf_accumulate<false> when no entry aims at an emitter and wf_shade skips the skip2
      // column (the same condition as there: no extensions, light-origin scans on)
      if (rec && tm.accum) tm.record(tm.accum[2 * ti], ss);
      if (ext || p.lt_lights == 0) launch(wf_accumulate<true>, grid_q, 0, ss, p, sc, Bc, d, o.stats);
      else launch(wf_accumulate<false>, grid_q, 0, ss, p, sc, Bc, d, o.stats);
      if (rec && tm.accum) tm.record(tm.accum[2 * ti + 1], ss);
      if (d < p.max_depth) closest_scan(d + 1);
      if (side) {
        jitter(side);
        jitter(st);
        cudaEventRecord(join[d], side);
        cudaStreamWaitEvent(st, join[d], 0);
      }
      tm.launches += 2 + scan_launches;  // shade, accumulate, the shadow scans
    }
    tm.n = t0 + p.max_depth + 1 < tm.cap ? t0 + p.max_depth + 1 : tm.cap;
    const int grid_w = (nw + 255) / 256 < grid_l ? (nw + 255) / 256 : grid_l;
    launch(wf_resolve, grid_w, 0, st, p, Bc, w0, nw, o.out, o.accum, o.stats);
    tm.launches += 2;  // wf_q0_len, wf_resolve
    if (tm.hint_dev)  // keep this chunk's queue counters: the hints of a later capture
      cudaMemcpyAsync(tm.hint_dev + (size_t)chunk * tm.hint_stride, Bc.ctr, sizeof(unsigned) * tm.hint_stride,
                      cudaMemcpyDeviceToDevice, st);
    if (tm.chunk_done && tm.n_chunks < tm.chunk_cap) {
      tm.record(tm.chunk_done[tm.n_chunks], st);
      tm.chunk_items[tm.n_chunks] = w0 + nw;
      ++tm.n_chunks;
    }
  }
  for (int k = 1; k < nslots; ++k) {  // the caller's stream resumes after every slot's last chunk
    cudaEventRecord(tm.slot_done[k], tm.slot_main[k]);
    cudaStreamWaitEvent(st0, tm.slot_done[k], 0);
  }
  return cudaGetLastError();
}

cudaError_t launch_render_wavefront(const DevParams& p, const DevScene& sc, const DevOutputs& o, int src,
                                    int num_sms, WfTiming& tm, cudaStream_t st) {
  if (src == SRC_SMEM) return wf_run<SRC_SMEM>(p, sc, o, num_sms, tm, st);
  if (src == SRC_TILE) return wf_run<SRC_TILE>(p, sc, o, num_sms, tm, st);
  return wf_run<SRC_GLOBAL>(p, sc, o, num_sms, tm, st);
}

}  // namespace rt
