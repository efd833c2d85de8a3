// rt_wavefront.cuh — wavefront variant of the hot path (included by rt_kernels.cu).
//
// The megakernel keeps every lane's path state in registers and runs one divergent state
// machine per round. The wavefront variant splits the same computation
// into kernels over compacted queues in HBM, so the FP32 intersection loop runs at high
// occupancy with no divergent logic inside, and the FP64 logic runs at full SIMD width:
//
//   Q[0] is implicit: entry e is the chunk's path e; its camera ray is computed where
//   it is used (wf_isect_eye2, wf_shade at depth 0)                                 (a2)
//   per depth d = 0..max_depth:
//     isect_closest   Q[d]: FP32 FFMA2 filter over all spheres -> candidate lists     (a3)
//                     (depth 0: two camera rays per thread, shared-origin tangent test)
//     shade           Q[d]: FP64 nearest hit (planes + candidates), emission/ambient,
//                     shadow entries with their Lambert/Phong contribution, bounce   (a4, a6)
//                     -> Q[d+1]
//     isect_shadow    shadow entries: FP64 planes, FP32 filter with early exit on a
//                     robust (float-certain) occluder -> candidate lists; point
//                     lights' rays are scanned from the light, tangent test (wf_isect_lt) (a5)
//     accumulate      Q[d]: FP64 occlusion decisions in light order, L += contribution
//   resolve           sum of the spp sample radiances in order s = 0..spp-1 -> float4 (a7)
//
// Per path the radiance receives the same terms in the same order as the megakernel
// (emission, ambient, lights 0..L-1 of depth 0, then depth 1, ...), so the two variants
// produce bit-identical framebuffers.
#pragma once
#include "rt_device.cuh"

namespace rt {

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// warp-aggregated reservation of `cnt` (< 64) slots on a global counter: exclusive prefix of
// the counts by bit-plane ballots (valid for any set of active lanes), one atomicAdd per warp
__device__ __forceinline__ unsigned warp_reserve(unsigned cnt, unsigned* counter) {
  const unsigned act = __activemask();
  const unsigned lt = lanemask_lt();
  unsigned prefix = 0, total = 0;
#pragma unroll
  for (int b = 0; b < 6; ++b) {
    const unsigned m = __ballot_sync(act, (cnt >> b) & 1u);
    prefix += (unsigned)__popc(m & lt) << b;
    total += (unsigned)__popc(m) << b;
  }
  const int leader = __ffs(act) - 1;
  unsigned base = 0;
  if ((int)(threadIdx.x & 31) == leader && total) base = atomicAdd(counter, total);
  return __shfl_sync(act, base, leader) + prefix;
}

// one slot per predicated lane, in lane order, one atomicAdd per warp
__device__ __forceinline__ unsigned warp_reserve1(bool take, unsigned* counter) {
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, take);
  const int leader = __ffs(act) - 1;
  unsigned base = 0;
  if ((int)(threadIdx.x & 31) == leader && m) base = atomicAdd(counter, (unsigned)__popc(m));
  return __shfl_sync(act, base, leader) + (unsigned)__popc(m & lanemask_lt());
}

// warp-aggregated statistics for ANY set of active lanes (a butterfly of shuffles would read
// inactive lanes, e.g. the work items outside the image between valid ones): two 32-bit
// reductions over the active mask (low 20 bits and the rest; per-lane values < 2^47)
__device__ __forceinline__ void warp_stat(unsigned long long* stats, int k, unsigned long long v) {
  const unsigned act = __activemask();
  const unsigned lo = __reduce_add_sync(act, (unsigned)(v & 0xFFFFFull));
  const unsigned hi = __reduce_add_sync(act, (unsigned)(v >> 20));
  const unsigned long long sum = ((unsigned long long)hi << 20) + lo;
  if ((threadIdx.x & 31) == (__ffs(act) - 1) && sum) atomicAdd(stats + k, sum);
}

__device__ __forceinline__ d3 ld3(const double* a, int cap, int i, int c0) {
  return mk(a[(c0 + 0) * (size_t)cap + i], a[(c0 + 1) * (size_t)cap + i], a[(c0 + 2) * (size_t)cap + i]);
}
__device__ __forceinline__ void st3(double* a, int cap, int i, int c0, d3 v) {
  a[(c0 + 0) * (size_t)cap + i] = v.x;
  a[(c0 + 1) * (size_t)cap + i] = v.y;
  a[(c0 + 2) * (size_t)cap + i] = v.z;
}
// origin / skipped sphere of closest-hit entry e of Q[d] (depth 0: the eye, none)
__device__ __forceinline__ d3 q_origin(const DevParams& P, const WfQueue& Q, int cap, unsigned e, int d) {
  return d == 0 ? mk(P.eye[0], P.eye[1], P.eye[2]) : ld3(Q.ray, cap, (int)e, 0);
}
__device__ __forceinline__ int q_skip(const WfQueue& Q, unsigned e, int d) { return d == 0 ? -1 : Q.skip[e]; }
// direction of closest-hit entry e of Q[d]. Depth 0 (the implicit camera queue): entry e is the
// chunk's path e, whose camera ray is computed here; false for a work item outside the image
// (partial edge tiles, shard tiles past the end)
__device__ __forceinline__ bool q_dir(const DevParams& P, const WfBuffers& B, const WfQueue& Q, unsigned e, int d,
                                      d3& dir) {
  if (d == 0) {
    const unsigned we = fdiv(P.div_spp, e);  // g0 + e = (w0 + we) * spp + sample
    int px = 0, py = 0;
    if (!item_pixel(P, B.w0 + (int)we, px, py)) return false;
    dir = camera_dir(P, px, py, (int)(e - we * (unsigned)P.spp));
    return true;
  }
  dir = ld3(Q.ray, B.cap, (int)e, 3);
  return true;
}
// the camera-ray scan's filter direction of path e of the chunk (camera_dir_filter); false for a
// work item outside the image
__device__ __forceinline__ bool eye_filter_dir(const DevParams& P, const WfBuffers& B, unsigned e, float& dx, float& dy,
                                               float& dz) {
  const unsigned we = fdiv(P.div_spp, e);
  int px = 0, py = 0;
  if (!item_pixel(P, B.w0 + (int)we, px, py)) return false;
  camera_dir_filter(P, px, py, (int)(e - we * (unsigned)P.spp), dx, dy, dz);
  return true;
}
__device__ __forceinline__ int q_path(const WfQueue& Q, unsigned e, int d) {
  return d == 0 ? (int)e : Q.path[e];
}
__device__ __forceinline__ float3 lf3(const float* a, int cap, int i) {
  return f3(a[i], a[(size_t)cap + i], a[2 * (size_t)cap + i]);
}
__device__ __forceinline__ void sf3(float* a, int cap, int i, float3 v) {
  a[i] = v.x;
  a[(size_t)cap + i] = v.y;
  a[2 * (size_t)cap + i] = v.z;
}

// shadow ray from o_s toward the point x: direction and t_max = |x - o_s|
__device__ __forceinline__ void shadow_dir(d3 os, d3 x, d3& ds, double& tl) {
  const d3 ws = x - os;
  tl = sqrt(dot(ws, ws));
  ds = ws * (1.0 / tl);
}
__device__ __forceinline__ d3 light_pos(const DevScene& S, int l) {
  const DevLight lt = S.lights[l];
  return mk(lt.px, lt.py, lt.pz);
}
// shadow ray of light l from the shading point: o = p + EPS_T n toward the light
__device__ __forceinline__ void shadow_ray(const DevScene& S, d3 p, d3 n, int l, d3& os, d3& ds, double& tl) {
  os = p + n * kEps;
  shadow_dir(os, light_pos(S, l), ds, tl);
}

// A shadow ray from a point hit on the outside of sphere `out` (origin p + EPS_T n, outside)
// that heads away from it (n.d > 0) cannot hit it (convexity): that sphere is skipped exactly.
__device__ __forceinline__ int shadow_skip(int out, d3 n, d3 ds) { return (out >= 0 && dot(n, ds) > 0.0) ? out : -1; }

// shadow ray toward a sampled emitter point x (R#41): o = p + EPS_T n, t_max = |x - o|
__device__ __forceinline__ void shadow_ray_to(d3 p, d3 n, d3 x, d3& os, d3& ds, double& tl) {
  os = p + n * kEps;
  shadow_dir(os, x, ds, tl);
}

// Light l seen from shading point p: point light l < n_lights (R#2: g = cos / d^2), else
// emitter e = l - n_lights with one uniform surface point (R#41: g = cos_s cos_l / (d^2 pdf)).
// False when it sends no shadow ray (d^2 < 1e-12, cos_s <= 0, or cos_l <= 0 for an emitter).
struct LightSample {
  d3 x, wi;
  double cos_s, g;
  float ir, ig, ib;
};
constexpr double kPiD = 3.14159265358979323846;
template <bool kExt = true>  // kExt = false: point lights only (no emitters sampled)
__device__ __forceinline__ bool light_sample(const DevParams& P, const DevScene& S, int l, d3 p, d3 nrm,
                                             unsigned long long pix, unsigned sg, int depth, LightSample& ls) {
  d3 nl = mk(0, 0, 0);
  double r = 0.0;
  const bool emitter = kExt && l >= P.n_lights;
  if (!emitter) {
    const DevLight lt = S.lights[l];
    ls.x = mk(lt.px, lt.py, lt.pz);
    ls.ir = lt.ix; ls.ig = lt.iy; ls.ib = lt.iz;
  } else {
    const unsigned e = (unsigned)(l - P.n_lights);
    const int ks = S.emit_sph[e];
    const float4 cr = __ldg(S.sph_cr + ks);
    nl = sphere_point(rng_stream(P.seed, pix, sg, depth, 5u + 2u * e), rng_stream(P.seed, pix, sg, depth, 6u + 2u * e));
    r = (double)cr.w;
    ls.x = mk((double)cr.x + r * nl.x, (double)cr.y + r * nl.y, (double)cr.z + r * nl.z);
    const DevMat m = S.mats[S.sph_mat[ks]];
    ls.ir = m.er; ls.ig = m.eg; ls.ib = m.eb;
  }
  const d3 w = ls.x - p;
  const double d2 = dot(w, w);
  if (d2 < 1e-12) return false;
  const double inv = 1.0 / sqrt(d2);
  ls.wi = w * inv;
  ls.cos_s = dot(nrm, ls.wi);
  if (ls.cos_s <= 0.0) return false;  // no shadow ray
  if (emitter) {
    const double cos_l = -dot(ls.wi, nl);
    if (cos_l <= 0.0) return false;
    ls.g = ls.cos_s * cos_l / (d2 * (1.0 / (4.0 * kPiD * r * r)));
  } else {
    ls.g = ls.cos_s * (inv * inv);  // cos / d^2 within 2 ulp of FP64, and g is used as a float
  }
  return true;
}

// Does light l send a shadow ray from p (light_sample returns true)? The same decision without
// normalising w when its sign is certain: light_sample tests cos_s = n.(w * (1/|w|)), whose
// rounding error is below 8u |w|_1 / |w| (u = 2^-53: the reciprocal, the products and the sum),
// while the unnormalised t = n.w is within 3u |w|_1 of the exact value. Outside the band
// |t| <= 1e-14 |w|_1 (~90u) both therefore have the sign of the exact n.w; inside it (and for
// emitters) light_sample itself decides. Bit-identical decisions, no FP64 sqrt or division
// in the count pass for almost every light.
template <bool kExt>
__device__ __forceinline__ bool sends_shadow_ray(const DevParams& P, const DevScene& S, int l, d3 p, d3 nrm,
                                                 unsigned long long pix, unsigned sg, int depth) {
  if (l < P.n_lights) {
    const DevLight lt = S.lights[l];
    const d3 w = mk(lt.px, lt.py, lt.pz) - p;
    if (dot(w, w) < 1e-12) return false;  // the same d^2 test as light_sample
    const double t = dot(nrm, w);
    const double band = 1e-14 * (fabs(w.x) + fabs(w.y) + fabs(w.z));
    if (t > band) return true;
    if (t < -band) return false;
  }
  LightSample ls;
  return light_sample<kExt>(P, S, l, p, nrm, pix, sg, depth, ls);
}

// ---- a2 with the implicit camera queue: only its length (the rays are computed on use) ---------
__global__ void wf_q0_len(WfBuffers B, int n) {
  if (threadIdx.x == 0) B.ctr[wf_ctr_q(0)] = (unsigned)n;
}

// ---- a3 / a5: FP32 filter over all spheres (persistent, one warp = 32 rays) -----------------
constexpr int kIsectMinBlocks = 3;  // 80 registers: 3 CTAs x 8 warps per SM (4 CTAs spill)
// One ray's scan over the sphere pairs [pb, pe): FP32 filter, candidate list in index order
// (closest: pruned by the certain upper bound tub; shadow: up to the first certain occluder rob).
// lo_row != nullptr: also store each closest candidate's lower root bound (split scans merge their
// parts' lists with the smallest tub of all parts).
template <int kSrc, bool kShadow>
__device__ __forceinline__ void isect_scan(const DevParams& P, const DevScene& S, const float4* __restrict__ gp,
                                           const RayFilter& F, int pb, int pe, bool& act, int skip,
                                           int skip2, float tl_f, float& tub, int& nc, int& rob, int* cand_row,
                                           float* lo_row) {
  const float eps_f = (float)kEps;
  for (int base = pb; base < pe; base += kPairsPerBatch) {
    float2 disc[kPairsPerBatch];
    float dmax;
    dmax = F.template batch<kSrc>(gp, base, disc);
    const bool any = act && dmax >= F.cut;
    if (__any_sync(kFull, any)) {
      if (any) {
        unsigned m = batch_mask(disc, F.cut);
        while (m != 0u) {
          const int i = __ffs(m) - 1;
          m &= m - 1u;
          const int k = 2 * base + i;
          if (k >= P.n_spheres) break;
          if (k == skip) continue;  // the sphere the ray leaves (exact, see shadow_skip / skip_c)
          if (kShadow && k == skip2) continue;
          float dd, tc;
          F.template sphere<kSrc>(gp, k, dd, tc);
          const float qh = sqrtf(fmaxf(dd - F.neg_slack, 0.f));  // >= true q
          const float ql = sqrtf(fmaxf(dd + F.neg_slack, 0.f));  // <= true q
          const bool sure = dd + F.neg_slack > 0.f;               // certainly intersects
          if (tc + qh < eps_f - F.eta) continue;                  // chord certainly behind
          if constexpr (kShadow) {
            if (tc - qh - F.eta >= tl_f * 1.000001f) continue;   // certainly beyond the light
            if (sure) {
              const float t0lo = tc - qh - F.eta, t0hi = tc - ql + F.eta;
              const float t1lo = tc + ql - F.eta, t1hi = tc + qh + F.eta;
              const float tlo = tl_f * 0.999999f;
              if ((t0lo >= eps_f && t0hi < tlo) || (t0hi < eps_f && t1lo >= eps_f && t1hi < tlo)) {
                rob = k;  // certain occluder: earlier ambiguous candidates are decided in FP64 later
                act = false;
                break;
              }
            }
          } else {
            if (tc - qh - F.eta > tub) continue;  // certainly farther than a certain hit
            if (sure) {
              const float t0lo = tc - qh - F.eta, t0hi = tc - ql + F.eta;
              const float t1lo = tc + ql - F.eta, t1hi = tc + qh + F.eta;
              if (t0lo >= eps_f) tub = fminf(tub, t0hi);
              else if (t0hi < eps_f && t1lo >= eps_f) tub = fminf(tub, t1hi);
            }
          }
          if (nc < kCandMax) {
            cand_row[nc] = k;
            if (!kShadow && lo_row != nullptr) lo_row[nc] = tc - qh - F.eta;
          }
          ++nc;
        }
      }
    }
    if constexpr (kShadow) {
      if (!__any_sync(kFull, act)) break;  // Alg. 1 `break`, warp-wide
    }
  }
}

// Split scans for short queues. A queue of a few hundred 32-ray tasks leaves most of the GPU
// idle while each warp scans all spheres serially (the deep depths of a small shard: 30-40 us per
// launch for a few thousand rays). Then `parts` (2, 4 or 8) warps of one CTA scan disjoint,
// batch-aligned sphere ranges of the same rays; after a CTA barrier the part-0 warp merges the
// per-part lists in part (= sphere index) order:
//  * closest: every part's candidates whose lower root bound does not exceed the smallest
//    certain upper bound tub of all parts (a candidate beyond a certain hit cannot be nearest;
//    every sphere attaining the minimum root survives, so wf_shade's FP64 decision is unchanged);
//  * shadow: the parts' candidates up to and including the first part that found a certain
//    occluder, which becomes the ray's rob: exactly the list of the unsplit index-order scan.
// A merged list longer than kCandMax overflows into the FP64 full scan, as an unsplit one does.
constexpr int kSplitMax = 8, kSplitSlack = 4;
// split while tasks x parts x kSplitSlack <= resident warps (measured slack 2, 4, 8, 16 -> world-8
// rank 1.105, 1.082, 1.082, 1.095 ms); the same rule is evaluated on the host for hinted launches
__host__ __device__ __forceinline__ int split_rule(unsigned tasks, unsigned warps) {
  int p = 1;
  while (p < kSplitMax && tasks * (unsigned)p * kSplitSlack <= warps) p <<= 1;
  return p;
}
__device__ __forceinline__ int split_parts(unsigned tasks, const WfBuffers& B) {
  if ((int)gridDim.x > B.xctas || blockDim.x != 256) return 1;
  if (B.force_parts > 0) return B.force_parts;
  return split_rule(tasks, gridDim.x * 8u);
}
// batch-aligned pair range of part `part` of `parts`
__device__ __forceinline__ void split_range(const DevParams& P, int part, int parts, int& pb, int& pe) {
  const int per = ((P.n_pairs_pad + parts - 1) / parts + kPairsPerBatch - 1) / kPairsPerBatch * kPairsPerBatch;
  pb = part * per < P.n_pairs_pad ? part * per : P.n_pairs_pad;
  pe = pb + per < P.n_pairs_pad ? pb + per : P.n_pairs_pad;
}
// merged shadow list of one ray from the parts' lists (rows of the CTA's warps w0 .. w0+parts-1)
__device__ __forceinline__ void split_merge_shadow(int parts, const int* s_nc, const int* s_rob, int stride,
                                                   const int* xrow0, size_t xstride, int* cand_row, int& nc_out,
                                                   int& rob_out) {
  int tot = 0, rob = -1;
  for (int q = 0; q < parts; ++q) {
    const int nq = s_nc[q * stride];
    const int* xr = xrow0 + q * xstride;
    for (int i = 0; i < nq && i < kCandMax; ++i) {
      if (tot + i < kCandMax) cand_row[tot + i] = xr[i];
    }
    tot += nq;
    const int rq = s_rob[q * stride];
    if (rq != -1) { rob = rq; break; }
  }
  nc_out = tot;
  rob_out = rob;
}

template <int kSrc, bool kShadow>
__global__ void __launch_bounds__(256, kIsectMinBlocks)
wf_isect(const DevParams P, const DevScene S, WfBuffers B, int d) {
  __shared__ uint64_t s_mbar;
  // shadow rays: the generic entries (every shadow ray not scanned from a point light), dense in
  // [0, ctr_so)
  const unsigned n = kShadow ? B.ctr[wf_ctr_so(d)] : B.ctr[wf_ctr_q(d)];
  if (!B.solo && split_parts((n + 31u) / 32u, B) > 1) return;  // a short queue: wf_isect_split scans it
  // CTAs beyond ceil(n / blockDim) would find no work: leave before staging the scene (deep
  // depths and small shards have short queues; the remaining warps take every 32-ray chunk)
  if ((unsigned long long)blockIdx.x * blockDim.x >= n) return;
  const float4* gp = S.pairs;
  if constexpr (kSrc == SRC_SMEM) stage_scene(s_pairs, gp, (uint32_t)P.n_pairs_pad * 32u, &s_mbar);
  unsigned* work = B.ctr + (kShadow ? wf_ctr_ws(d) : wf_ctr_wc(d));
  const WfQueue Q = B.q[d & 1];
  int* cand = kShadow ? B.scand : B.ccand;
  int* cn = kShadow ? B.sn : B.cn;
  const int lane = threadIdx.x & 31;
  const float eps_f = (float)kEps;
  while (true) {
    unsigned e0 = 0;
    if (lane == 0) e0 = atomicAdd(work, 32u);
    e0 = __shfl_sync(kFull, e0, 0);
    if (e0 >= n) break;
    const unsigned e = e0 + lane;
    bool act = e < n;
    const bool mine = act;
    d3 o = mk(0, 0, 0), dir = mk(0, 0, 1);
    double tl = 0.0;
    int rob = -1, skip = -1, skip2 = -1;  // skip2: the emitter a shadow ray aims at (R#41)
    if (act) {
      if constexpr (kShadow) {
        o = ld3(B.sray, B.gcap, (int)e, 0);
        dir = ld3(B.sray, B.gcap, (int)e, 3);
        tl = B.sray[6 * (size_t)B.gcap + e];
        skip = B.sskip[e];
        skip2 = B.sskip2[e];
        // planes first, exactly (FP64): the first plane in index order that occludes decides
        for (int j = 0; j < P.n_planes; ++j) {
          const DevPlane pl = c_planes[j];
          const double den = pl.nx * dir.x + pl.ny * dir.y + pl.nz * dir.z;
          if (fabs(den) >= 1e-12) {
            const double t = (pl.d - (pl.nx * o.x + pl.ny * o.y + pl.nz * o.z)) / den;
            if (t >= kEps && t < tl) { rob = -2 - j; act = false; break; }
          }
        }
      } else {
        o = q_origin(P, Q, B.cap, e, d);
        if (!q_dir(P, B, Q, e, d, dir)) act = false;  // outside the image: no candidates
        skip = q_skip(Q, e, d);
      }
    }
    RayFilter F;
    F.init(o, dir, P);
    const float tl_f = (float)tl;
    float tub = 3.0e38f;  // closest: certain upper bound of the nearest accepted root
    int nc = 0;
    for (int base = 0; base < P.n_pairs_pad; base += kPairsPerBatch) {
      float2 disc[kPairsPerBatch];
      float dmax;
      dmax = F.template batch<kSrc>(gp, base, disc);
      const bool any = act && dmax >= F.cut;
      if (__any_sync(kFull, any)) {
        if (any) {
          unsigned m = batch_mask(disc, F.cut);
          while (m != 0u) {
            const int i = __ffs(m) - 1;
            m &= m - 1u;
            const int k = 2 * base + i;
            if (k >= P.n_spheres) break;
            if (k == skip) continue;  // the sphere the ray leaves (exact, see shadow_skip / skip_c)
            if (kShadow && k == skip2) continue;
            float dd, tc;
            F.template sphere<kSrc>(gp, k, dd, tc);
            const float qh = sqrtf(fmaxf(dd - F.neg_slack, 0.f));  // >= true q
            const float ql = sqrtf(fmaxf(dd + F.neg_slack, 0.f));  // <= true q
            const bool sure = dd + F.neg_slack > 0.f;               // certainly intersects
            if (tc + qh < eps_f - F.eta) continue;                  // chord certainly behind
            if constexpr (kShadow) {
              if (tc - qh - F.eta >= tl_f * 1.000001f) continue;   // certainly beyond the light
              if (sure) {
                const float t0lo = tc - qh - F.eta, t0hi = tc - ql + F.eta;
                const float t1lo = tc + ql - F.eta, t1hi = tc + qh + F.eta;
                const float tlo = tl_f * 0.999999f;
                if ((t0lo >= eps_f && t0hi < tlo) || (t0hi < eps_f && t1lo >= eps_f && t1hi < tlo)) {
                  rob = k;  // certain occluder: earlier ambiguous candidates are decided in FP64 later
                  act = false;
                  break;
                }
              }
            } else {
              if (tc - qh - F.eta > tub) continue;  // certainly farther than a certain hit
              if (sure) {
                const float t0lo = tc - qh - F.eta, t0hi = tc - ql + F.eta;
                const float t1lo = tc + ql - F.eta, t1hi = tc + qh + F.eta;
                if (t0lo >= eps_f) tub = fminf(tub, t0hi);
                else if (t0hi < eps_f && t1lo >= eps_f) tub = fminf(tub, t1hi);
              }
            }
            if (nc < kCandMax) cand[(size_t)e * kCandMax + nc] = k;
            ++nc;
          }
        }
      }
      if constexpr (kShadow) {
        if (!__any_sync(kFull, act)) break;  // Alg. 1 `break`, warp-wide
      }
    }
    if (mine) {
      cn[e] = nc;
      if constexpr (kShadow) B.srob[e] = rob;
    }
  }
}

template <int kSrc, bool kShadow>
__device__ __forceinline__ void wf_isect_split_body(const DevParams& P, const DevScene& S, const WfBuffers& B, int d) {
  __shared__ uint64_t s_mbar;
  __shared__ int s_nc[8][32];
  __shared__ int s_x[8][32];  // closest: tub (float bits); shadow: rob
  __shared__ unsigned s_unit;
  const unsigned n = kShadow ? B.ctr[wf_ctr_so(d)] : B.ctr[wf_ctr_q(d)];
  const unsigned tasks = (n + 31u) / 32u;  // 32 rays each
  const int parts = split_parts(tasks, B);
  if (parts == 1 && !B.solo) return;  // a long queue: wf_isect scans it (solo: one part here)
  const float4* gp = S.pairs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tpc = 8 / parts;  // tasks per CTA unit
  const unsigned units = (tasks + tpc - 1) / tpc;
  if (blockIdx.x >= units) return;  // CTAs without work leave before staging the scene
  if constexpr (kSrc == SRC_SMEM) stage_scene(s_pairs, gp, (uint32_t)P.n_pairs_pad * 32u, &s_mbar);
  const int slot = warp / parts, part = warp % parts;
  int pb, pe;
  split_range(P, part, parts, pb, pe);
  const size_t xs = (size_t)32 * kCandMax;  // between the scratch rows of consecutive warps
  const size_t row = ((size_t)(blockIdx.x * 8 + warp) * 32 + lane) * kCandMax;
  int* xc = (kShadow ? B.xcand_s : B.xcand_c) + row;
  float* xl = B.xlo_c + row;
  unsigned* work = B.ctr + (kShadow ? wf_ctr_ws(d) : wf_ctr_wc(d));
  const WfQueue Q = B.q[d & 1];
  while (true) {
    if (threadIdx.x == 0) s_unit = atomicAdd(work, 1u);
    __syncthreads();
    const unsigned u = s_unit;
    if (u >= units) break;  // CTA-uniform
    const unsigned e = (u * tpc + slot) * 32u + lane;
    bool act = e < n;
    const bool mine = act;
    d3 o = mk(0, 0, 0), dir = mk(0, 0, 1);
    double tl = 0.0;
    int rob = -1, skip = -1, skip2 = -1;
    if (act) {
      if constexpr (kShadow) {
        o = ld3(B.sray, B.gcap, (int)e, 0);
        dir = ld3(B.sray, B.gcap, (int)e, 3);
        tl = B.sray[6 * (size_t)B.gcap + e];
        skip = B.sskip[e];
        skip2 = B.sskip2[e];
        for (int j = 0; j < P.n_planes; ++j) {  // planes first, exactly (every part alike)
          const DevPlane pl = c_planes[j];
          const double den = pl.nx * dir.x + pl.ny * dir.y + pl.nz * dir.z;
          if (fabs(den) >= 1e-12) {
            const double t = (pl.d - (pl.nx * o.x + pl.ny * o.y + pl.nz * o.z)) / den;
            if (t >= kEps && t < tl) { rob = -2 - j; act = false; break; }
          }
        }
      } else {
        o = q_origin(P, Q, B.cap, e, d);
        if (!q_dir(P, B, Q, e, d, dir)) act = false;  // outside the image: no candidates
        skip = q_skip(Q, e, d);
      }
    }
    RayFilter F;
    F.init(o, dir, P);
    float tub = 3.0e38f;
    int nc = 0;
    isect_scan<kSrc, kShadow>(P, S, gp, F, pb, pe, act, skip, skip2, (float)tl, tub, nc, rob, xc, xl);
    s_nc[warp][lane] = nc;
    s_x[warp][lane] = kShadow ? rob : __float_as_int(tub);
    __syncthreads();
    if (part == 0 && mine) {
      if constexpr (kShadow) {
        int nco, robo;
        split_merge_shadow(parts, &s_nc[warp][lane], &s_x[warp][lane], 32, xc, xs, B.scand + (size_t)e * kCandMax, nco, robo);
        B.sn[e] = nco;
        B.srob[e] = robo;
      } else {
        float tm = __int_as_float(s_x[warp][lane]);
        for (int q = 1; q < parts; ++q) tm = fminf(tm, __int_as_float(s_x[warp + q][lane]));
        int* crow = B.ccand + (size_t)e * kCandMax;
        int tot = 0;
        for (int q = 0; q < parts; ++q) {
          const int nq = s_nc[warp + q][lane];
          if (nq > kCandMax) { tot = kCandMax + 1; break; }  // a part overflowed: FP64 full scan
          for (int i = 0; i < nq; ++i) {
            if (xl[q * xs + i] > tm) continue;  // certainly farther than a certain hit
            if (tot < kCandMax) crow[tot] = xc[q * xs + i];
            ++tot;
          }
        }
        B.cn[e] = tot;
      }
    }
    __syncthreads();  // s_unit / s_nc / s_x / scratch rows are rewritten by the next unit
  }
}

template <int kSrc, bool kShadow>
__global__ void __launch_bounds__(256, kIsectMinBlocks)
wf_isect_split(const DevParams P, const DevScene S, WfBuffers B, int d) {
  wf_isect_split_body<kSrc, kShadow>(P, S, B, d);
}

// The ring of two TMA-loaded tiles of the pair array (SRC_TILE) a CTA streams through: tile t
// lives in buffer t & 1 (ring slot i mod 4 kTilePairs of global float4 index i), its copy completes
// on mbarrier t & 1; the barrier phases are tracked per buffer in registers (CTA-uniform).
struct TileRing {
  uint64_t* full;  // [2] mbarriers in shared memory
  const float4* gp;
  int n_pairs, ntiles;
  uint32_t phases;  // bit b: the parity the next completion of buffer b's barrier will have
  __device__ __forceinline__ void init(uint64_t* bars, const float4* g, int np) {  // every thread
    full = bars;
    gp = g;
    n_pairs = np;
    ntiles = (np + kTilePairs - 1) / kTilePairs;
    phases = 0u;
    if (threadIdx.x == 0) {
      mbar_init(&full[0]);
      mbar_init(&full[1]);
    }
    __syncthreads();
  }
  __device__ __forceinline__ int begin(int t) const { return t * kTilePairs; }
  __device__ __forceinline__ int end(int t) const {
    return (t + 1) * kTilePairs < n_pairs ? (t + 1) * kTilePairs : n_pairs;
  }
  __device__ __forceinline__ void issue(int t) const {  // one thread
    tile_load(s_pairs + 2 * kTilePairs * (t & 1), gp + 2 * begin(t), (uint32_t)(end(t) - begin(t)) * 32u, &full[t & 1]);
  }
  __device__ __forceinline__ void wait(int t) {  // every thread
    mbar_wait(&full[t & 1], (phases >> (t & 1)) & 1u);
    phases ^= 1u << (t & 1);
  }
};

// ---- a3 / a5 for scenes beyond shared memory: the scan over TMA-loaded tiles ------------------
// A CTA takes 256 rays (8 warps x 32) and streams the pair array through a ring of two tiles of
// kTilePairs pairs: one elected thread issues the bulk copy of tile t + 2 into the buffer tile t
// used as soon as every warp is done with it (CTA barrier), so a copy is in flight while the warps
// scan the other tile. Every warp runs the same FP32 filter over the tile as the staged kernels
// (isect_scan), so candidate lists, robust occluders and every decision are those of wf_isect.
// Shadow rays: the CTA stops streaming once none of its rays is active (Alg. 1 `break`).
template <bool kShadow>
__global__ void __launch_bounds__(256, kIsectMinBlocks)
wf_isect_tiled(const DevParams P, const DevScene S, WfBuffers B, int d) {
  __shared__ uint64_t s_full[2];
  __shared__ unsigned s_task;
  const unsigned n = kShadow ? B.ctr[wf_ctr_so(d)] : B.ctr[wf_ctr_q(d)];
  if (!B.solo && split_parts((n + 31u) / 32u, B) > 1) return;  // a short queue: wf_isect_split scans it
  if ((unsigned long long)blockIdx.x * blockDim.x >= n) return;
  const float4* gp = S.pairs;
  TileRing ring;
  ring.init(s_full, gp, P.n_pairs_pad);
  const int ntiles = ring.ntiles;
  unsigned* work = B.ctr + (kShadow ? wf_ctr_ws(d) : wf_ctr_wc(d));
  const WfQueue Q = B.q[d & 1];
  while (true) {
    if (threadIdx.x == 0) {
      s_task = atomicAdd(work, 256u);
      ring.issue(0);  // the previous task drained every copy it issued: both buffers are free
      if (ntiles > 1) ring.issue(1);
    }
    __syncthreads();
    const unsigned e = s_task + threadIdx.x;
    const bool task_ok = s_task < n;  // CTA-uniform
    if (!task_ok) {  // drain the copies just issued (the ring must be idle when the kernel exits)
      ring.wait(0);
      if (ntiles > 1) ring.wait(1);
      break;
    }
    bool act = e < n;
    const bool mine = act;
    d3 o = mk(0, 0, 0), dir = mk(0, 0, 1);
    double tl = 0.0;
    int rob = -1, skip = -1, skip2 = -1;
    if (act) {
      if constexpr (kShadow) {
        o = ld3(B.sray, B.gcap, (int)e, 0);
        dir = ld3(B.sray, B.gcap, (int)e, 3);
        tl = B.sray[6 * (size_t)B.gcap + e];
        skip = B.sskip[e];
        skip2 = B.sskip2[e];
        for (int j = 0; j < P.n_planes; ++j) {  // planes first, exactly (FP64), in index order
          const DevPlane pl = c_planes[j];
          const double den = pl.nx * dir.x + pl.ny * dir.y + pl.nz * dir.z;
          if (fabs(den) >= 1e-12) {
            const double t = (pl.d - (pl.nx * o.x + pl.ny * o.y + pl.nz * o.z)) / den;
            if (t >= kEps && t < tl) { rob = -2 - j; act = false; break; }
          }
        }
      } else {
        o = q_origin(P, Q, B.cap, e, d);
        if (!q_dir(P, B, Q, e, d, dir)) act = false;  // outside the image: no candidates
        skip = q_skip(Q, e, d);
      }
    }
    RayFilter F;
    F.init(o, dir, P);
    float tub = 3.0e38f;
    int nc = 0;
    int* cand_row = (kShadow ? B.scand : B.ccand) + (size_t)(mine ? e : 0u) * kCandMax;
    for (int t = 0; t < ntiles; ++t) {
      ring.wait(t);
      isect_scan<SRC_TILE, kShadow>(P, S, gp, F, ring.begin(t), ring.end(t), act, skip, skip2, (float)tl, tub, nc, rob,
                                    cand_row, nullptr);
      const bool any_left = kShadow ? (__syncthreads_or(act) != 0) : (__syncthreads(), true);  // buffer t & 1 is free
      if (any_left) {
        if (threadIdx.x == 0 && t + 2 < ntiles) ring.issue(t + 2);
      } else {  // every ray of the CTA is settled: wait for the copy still in flight, then stop
        if (t + 1 < ntiles) ring.wait(t + 1);
        break;
      }
    }
    if (mine) {
      (kShadow ? B.sn : B.cn)[e] = nc;
      if constexpr (kShadow) B.srob[e] = rob;
    }
    __syncthreads();  // s_task and the ring are reused by the next task
  }
}

// ---- a3 for camera rays, two rays per thread --------------------------------------------------
// Camera rays share the origin (the eye), so the scan tests the tangent condition
// c'.d - h >= o'.d (RayFilter::tangent_cut; -h per sphere in the eye's table, rt_kernels.cu
// build_eye_table): 3 FMA per sphere and ray. One ray per thread would leave the kernel co-limited
// by the shared-memory pipe (2 LDS.128 per 2 spheres); here every lane carries two camera rays (a
// warp = 64 rays): each pair of spheres read from shared memory serves both, and the FFMA2 stream
// is again the only limit. Candidates get the chord bounds of wf_isect (s1 precomputed, one
// float2 per pair after the pairs), so the candidate lists hold the same decisions.
constexpr int kEyePB = 8;
static_assert(kPairsPerBatch % kEyePB == 0, "n_pairs_pad is padded to kPairsPerBatch");

struct EyeRay {
  RayFilter F;
  float cu;  // F.tangent_cut()
  float tub;
  int nc;
  bool act;
};

template <int kSrc>
__device__ __forceinline__ void eye_candidates(const DevParams& P, const float4* __restrict__ gp,
                                               const float2* __restrict__ s1p, unsigned m, int kbase, EyeRay& R,
                                               int* cand_row) {
  const float eps_f = (float)kEps;
  while (m != 0u) {
    const int i = __ffs(m) - 1;
    m &= m - 1u;
    const int k = kbase + i;
    if (k >= P.n_spheres) break;
    float dd, tc;
    R.F.template sphere_s1<kSrc>(gp, s1p, k, dd, tc);
    if (dd < R.F.neg_slack) continue;            // certainly no real root
    const float qh = sqrtf(fmaxf(dd - R.F.neg_slack, 0.f));
    const float ql = sqrtf(fmaxf(dd + R.F.neg_slack, 0.f));
    const bool sure = dd + R.F.neg_slack > 0.f;
    if (tc + qh < eps_f - R.F.eta) continue;     // chord certainly behind
    if (tc - qh - R.F.eta > R.tub) continue;     // certainly farther than a certain hit
    if (sure) {
      const float t0lo = tc - qh - R.F.eta, t0hi = tc - ql + R.F.eta;
      const float t1lo = tc + ql - R.F.eta, t1hi = tc + qh + R.F.eta;
      if (t0lo >= eps_f) R.tub = fminf(R.tub, t0hi);
      else if (t0hi < eps_f && t1lo >= eps_f) R.tub = fminf(R.tub, t1hi);
    }
    if (R.nc < kCandMax) cand_row[R.nc] = k;
    ++R.nc;
  }
}

// the shared-origin scan of two camera rays (one thread) over the sphere pairs [pb, pe)
template <int kSrc>
__device__ __forceinline__ void eye2_scan(const DevParams& P, const float4* __restrict__ gp,
                                          const float2* __restrict__ s1p, int pb, int pe, EyeRay& Ra, EyeRay& Rb,
                                          int* rowa, int* rowb) {
  const float2 D1a = make_float2(Ra.F.dx, Ra.F.dx), D2a = make_float2(Ra.F.dy, Ra.F.dy);
  const float2 D3a = make_float2(Ra.F.dz, Ra.F.dz);
  const float2 D1b = make_float2(Rb.F.dx, Rb.F.dx), D2b = make_float2(Rb.F.dy, Rb.F.dy);
  const float2 D3b = make_float2(Rb.F.dz, Rb.F.dz);
  for (int base = pb; base < pe; base += kEyePB) {
    float2 ua[kEyePB], ub[kEyePB];
#pragma unroll
    for (int i = 0; i < kEyePB; ++i) {
      const float4 a = load_pair<kSrc>(gp, 2 * (base + i));
      const float4 b = load_pair<kSrc>(gp, 2 * (base + i) + 1);
      const float2 CX = make_float2(a.x, a.y), CY = make_float2(a.z, a.w);
      const float2 CZ = make_float2(b.x, b.y), NH = make_float2(b.z, b.w);
      ua[i] = __ffma2_rn(CX, D1a, __ffma2_rn(CY, D2a, __ffma2_rn(CZ, D3a, NH)));  // c'.d - h
      ub[i] = __ffma2_rn(CX, D1b, __ffma2_rn(CY, D2b, __ffma2_rn(CZ, D3b, NH)));
    }
    float ma = fmaxf(ua[0].x, ua[0].y), mb = fmaxf(ub[0].x, ub[0].y);
#pragma unroll
    for (int i = 1; i < kEyePB; ++i) {  // a running max: interleaves with the FFMA2 stream (a max16
      ma = fmaxf(ma, fmaxf(ua[i].x, ua[i].y));   // tree measured 7 % / 3 % slower here)
      mb = fmaxf(mb, fmaxf(ub[i].x, ub[i].y));
    }
    const bool ca = Ra.act && ma >= Ra.cu, cb = Rb.act && mb >= Rb.cu;
    if (__any_sync(kFull, ca || cb)) {
      if (ca) {
        unsigned m = 0u;
#pragma unroll
        for (int i = 0; i < kEyePB; ++i)
          m |= ((ua[i].x >= Ra.cu) ? 1u : 0u) << (2 * i) | ((ua[i].y >= Ra.cu) ? 1u : 0u) << (2 * i + 1);
        eye_candidates<kSrc>(P, gp, s1p, m, 2 * base, Ra, rowa);
      }
      if (cb) {
        unsigned m = 0u;
#pragma unroll
        for (int i = 0; i < kEyePB; ++i)
          m |= ((ub[i].x >= Rb.cu) ? 1u : 0u) << (2 * i) | ((ub[i].y >= Rb.cu) ? 1u : 0u) << (2 * i + 1);
        eye_candidates<kSrc>(P, gp, s1p, m, 2 * base, Rb, rowb);
      }
    }
  }
}

template <int kSrc>
__global__ void __launch_bounds__(256, kIsectMinBlocks)
wf_isect_eye2(const DevParams P, const DevScene S, WfBuffers B, int d) {
  __shared__ uint64_t s_mbar;
  const unsigned n = B.ctr[wf_ctr_q(d)];
  if ((unsigned long long)blockIdx.x * blockDim.x * 2ull >= n) return;  // CTAs without work
  const float4* gp = S.pairs_eye;
  // the pairs are staged (32 B per pair); the candidates read their s1 column from global memory
  // (rare; 8 KB less shared memory per CTA for the kernels running beside it: 5.518 -> 5.508 ms)
  if constexpr (kSrc == SRC_SMEM) stage_scene(s_pairs, gp, (uint32_t)P.n_pairs_pad * 32u, &s_mbar);
  const float2* s1p = reinterpret_cast<const float2*>(gp + 2 * P.n_pairs_pad);
  unsigned* work = B.ctr + wf_ctr_wc(d);  // (camera rays: d == 0, the implicit queue)
  const int lane = threadIdx.x & 31;
  while (true) {
    unsigned e0 = 0;
    if (lane == 0) e0 = atomicAdd(work, 64u);
    e0 = __shfl_sync(kFull, e0, 0);
    if (e0 >= n) break;
    const unsigned ea = e0 + lane, eb = e0 + 32 + lane;
    EyeRay Ra, Rb;
    {  // camera rays (depth 0): the eye and the filter direction (decisions: wf_shade, camera_dir)
      const d3 o = mk(P.eye[0], P.eye[1], P.eye[2]);
      float ax = 0.f, ay = 0.f, az = 1.f, bx = 0.f, by = 0.f, bz = 1.f;
      Ra.act = ea < n && eye_filter_dir(P, B, ea, ax, ay, az);
      Rb.act = eb < n && eye_filter_dir(P, B, eb, bx, by, bz);
      Ra.F.init(o, ax, ay, az, P);
      Rb.F.init(o, bx, by, bz, P);
    }
    Ra.cu = Ra.F.tangent_cut();
    Rb.cu = Rb.F.tangent_cut();
    Ra.tub = Rb.tub = 3.0e38f;
    Ra.nc = Rb.nc = 0;
    eye2_scan<kSrc>(P, gp, s1p, 0, P.n_pairs_pad, Ra, Rb, B.ccand + (size_t)ea * kCandMax,
                    B.ccand + (size_t)eb * kCandMax);
    if (ea < n) B.cn[ea] = Ra.nc;
    if (eb < n) B.cn[eb] = Rb.nc;
  }
}

// camera rays of scenes beyond shared memory: the same two-rays-per-thread scan over the eye's
// pair table streamed through the TMA tile ring; a CTA takes 512 rays (8 warps x 64)
__global__ void __launch_bounds__(256, kIsectMinBlocks)
wf_isect_eye2_tiled(const DevParams P, const DevScene S, WfBuffers B, int d) {
  __shared__ uint64_t s_full[2];
  __shared__ unsigned s_task;
  const unsigned n = B.ctr[wf_ctr_q(d)];
  if ((unsigned long long)blockIdx.x * blockDim.x * 2ull >= n) return;  // CTAs without work
  const float4* gp = S.pairs_eye;
  const float2* s1p = reinterpret_cast<const float2*>(gp + 2 * P.n_pairs_pad);  // candidates: from global
  TileRing ring;
  ring.init(s_full, gp, P.n_pairs_pad);
  const int ntiles = ring.ntiles;
  unsigned* work = B.ctr + wf_ctr_wc(d);  // (camera rays: d == 0, the implicit queue)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    if (threadIdx.x == 0) {
      s_task = atomicAdd(work, 512u);
      ring.issue(0);
      if (ntiles > 1) ring.issue(1);
    }
    __syncthreads();
    const unsigned e0 = s_task + 64u * warp;
    if (s_task >= n) {  // CTA-uniform: drain the copies just issued
      ring.wait(0);
      if (ntiles > 1) ring.wait(1);
      break;
    }
    const unsigned ea = e0 + lane, eb = e0 + 32 + lane;
    EyeRay Ra, Rb;
    {  // camera rays (depth 0): the eye and the filter direction (decisions: wf_shade, camera_dir)
      const d3 o = mk(P.eye[0], P.eye[1], P.eye[2]);
      float ax = 0.f, ay = 0.f, az = 1.f, bx = 0.f, by = 0.f, bz = 1.f;
      Ra.act = ea < n && eye_filter_dir(P, B, ea, ax, ay, az);
      Rb.act = eb < n && eye_filter_dir(P, B, eb, bx, by, bz);
      Ra.F.init(o, ax, ay, az, P);
      Rb.F.init(o, bx, by, bz, P);
    }
    Ra.cu = Ra.F.tangent_cut();
    Rb.cu = Rb.F.tangent_cut();
    Ra.tub = Rb.tub = 3.0e38f;
    Ra.nc = Rb.nc = 0;
    int* rowa = B.ccand + (size_t)(ea < n ? ea : 0u) * kCandMax;
    int* rowb = B.ccand + (size_t)(eb < n ? eb : 0u) * kCandMax;
    for (int t = 0; t < ntiles; ++t) {
      ring.wait(t);
      eye2_scan<SRC_TILE>(P, gp, s1p, ring.begin(t), ring.end(t), Ra, Rb, rowa, rowb);
      __syncthreads();  // buffer t & 1 is free
      if (threadIdx.x == 0 && t + 2 < ntiles) ring.issue(t + 2);
    }
    if (ea < n) B.cn[ea] = Ra.nc;
    if (eb < n) B.cn[eb] = Rb.nc;
    __syncthreads();  // s_task and the ring are reused by the next task
  }
}

// ---- a5 for point lights: the shadow scan from the light -------------------------------------
// The segment [p + EPS_T n, P_l) is the same line whichever end it is traced from, and the scan
// only filters (FP64 decides on the original ray in wf_accumulate). Traced from the light, every
// shadow ray of light l shares the origin P_l, and an occluder lies on the reversed half-line
// s = t_l - t > 0: the tangent test c'.d' - h_l >= o'.d' (RayFilter::tangent_cut; -h_l per
// sphere and light precomputed, rt_kernels.cu neg_tangent: light l's own table in S.pairs_ltl for
// the long lists, every light's column after the pairs in S.pairs_lt for the short-list split
// scan) costs 3 FMA per sphere instead of 7, and a thread carries two rays of the same light (one
// shared-memory read serves both). Work comes in chunks of 64 entries of one list. The chord [tc' - q, tc' + q] along the
// reversed ray maps back to t = t_l - tc' -/+ q on the original one; the bounds add the error of
// t_l and of the reversal.
// Why the half-line is safe: a sphere the test drops (light outside it by more than 1e-6 S, else
// it is always a candidate) meets the reversed line, if at all, at s < -(gap)/2 <= -5e-7 S, i.e.
// at t > t_l + 5e-7 S on the original ray, while the FP64 roots there are off by ~1e-15 (t_l + S);
// a ray with t_l > 1e6 S (a far plane point) drops nothing (cu = -3e38).
//
// Input: light l's rays are listed in kLtSub sub-lists (wf_shade reserves slots per warp group,
// the sub-list chosen by the iteration's 256-path block, so no single hot counter); a
// slot holds the ray's direction and t_max rounded to float (what the filter reads; wf_shade
// computed them in FP64) and {shading entry e of Q[d], skip}: skip = the sphere the ray provably
// leaves or -1, or -2 - j when wf_shade already found plane j to occlude (planes are decided in
// FP64 first, in index order). Where an FP64 decision needs the ray, wf_accumulate rebuilds it
// from the shading point's o_s = p + EPS_T n (B.sorg[e]) with the same arithmetic (shadow_dir).
// Output per slot: {rob, nc} + candidates.
constexpr int kLtPB = 8;
static_assert(kPairsPerBatch % kLtPB == 0, "n_pairs_pad is padded to kPairsPerBatch");

struct LtRay {
  RayFilter F;  // filter of the reversed ray (origin P_l, direction -d)
  float cu;     // F.tangent_cut(), or -3e38 (every sphere a candidate) for t_l > 1e6 S
  float tl_f, tlerr;
  int nc, rob, skip;
  bool act;
};

// FP64 shadow ray of list slot g of light l (rebuilt from the shading point's o_s)
__device__ __forceinline__ void lt_ray(const DevScene& S, const WfBuffers& B, int e, int l, d3& os, d3& ds, double& tl) {
  os = ld3(B.sorg, B.cap, e, 0);
  shadow_dir(os, light_pos(S, l), ds, tl);
}

__device__ __forceinline__ void lt_setup(const DevParams& P, const DevScene& S, const WfBuffers& B, unsigned g, bool valid,
                                         int l, LtRay& R) {
  float4 dt = make_float4(0.f, 0.f, 1.f, 1.f);  // direction, t_max (float)
  R.act = valid;
  R.rob = -1;
  R.skip = -1;
  R.nc = 0;
  if (valid) {
    dt = B.lt_dir[g];
    const int skip = B.lt_rec[g].y;
    RT_CHECK(B.lt_rec[g].x >= 0 && B.lt_rec[g].x < B.cap && skip < P.n_spheres, 401);
    if (skip <= -2) {  // plane -2-skip occludes (decided by wf_shade in FP64)
      R.rob = skip;
      R.act = false;
    } else {
      R.skip = skip;
    }
  }
  R.F.init(light_pos(S, l), -dt.x, -dt.y, -dt.z, P);
  // S = cmax + |o'| + rmax = eta / (8 kUlp) + rmax (RayFilter::init)
  R.cu = dt.w > 1.0e6f * (R.F.eta * (1.0f / (8.0f * kUlp)) + P.rmax) ? -3.0e38f : R.F.tangent_cut();
  R.tl_f = dt.w;
  R.tlerr = 4.0e-7f * R.tl_f + 1.0e-6f * R.F.eta;  // t_l to float, P_l vs o + t_l d, the subtraction
}

// gk == nullptr: gp is the shared pair layout (K in place); else gp is a light's table (-h in
// place of K) and K comes from the float2-per-pair column gk
template <int kSrc>
__device__ __forceinline__ void lt_candidates(const DevParams& P, const float4* __restrict__ gp,
                                              const float2* __restrict__ gk, unsigned m, int kbase, LtRay& R,
                                              int* cand_row) {
  const float eps_f = (float)kEps;
  while (m != 0u) {
    const int i = __ffs(m) - 1;
    m &= m - 1u;
    const int k = kbase + i;
    if (k >= P.n_spheres) break;
    if (k == R.skip) continue;
    float dd, tc;  // tc along -d from P_l
    if (gk) R.F.template sphere_k<kSrc>(gp, gk, k, dd, tc);
    else R.F.template sphere<kSrc>(gp, k, dd, tc);
    if (dd < R.F.neg_slack) continue;                  // certainly no real root
    const float qh = sqrtf(fmaxf(dd - R.F.neg_slack, 0.f));
    const float ql = sqrtf(fmaxf(dd + R.F.neg_slack, 0.f));
    const bool sure = dd + R.F.neg_slack > 0.f;
    const float err = R.F.eta + R.tlerr;
    // original-ray roots: t0 = t_l - tc - q, t1 = t_l - tc + q
    const float t0lo = R.tl_f - (tc + qh) - err, t0hi = R.tl_f - (tc + ql) + err;
    const float t1lo = R.tl_f - (tc - ql) - err, t1hi = R.tl_f - (tc - qh) + err;
    if (t1hi < eps_f) continue;                        // chord certainly behind the shading point
    if (t0lo >= R.tl_f * 1.000001f) continue;          // certainly beyond the light
    if (sure) {
      const float tlo = R.tl_f * 0.999999f;
      if ((t0lo >= eps_f && t0hi < tlo) || (t0hi < eps_f && t1lo >= eps_f && t1hi < tlo)) {
        R.rob = k;  // certain occluder (earlier ambiguous candidates are decided in FP64 later)
        R.act = false;
        return;
      }
    }
    if (R.nc < kCandMax) cand_row[R.nc] = k;
    ++R.nc;
  }
}

// the light-origin scan of two rays of light l (one thread) over the sphere pairs [pb, pe):
// kTable = false: the shared pair layout gp + light l's -h column nhp (the short-list scan stages
// every light's column); true: light l's own table gp ({c'x, c'y | c'z, -h}, two LDS.128 per pair
// like the camera-ray scan), K for the candidates from its column gk
template <int kSrc, bool kTable = false>
__device__ __forceinline__ void lt_scan(const DevParams& P, const float4* __restrict__ gp, const float2* __restrict__ nhp,
                                        const float2* __restrict__ gk, int pb, int pe, LtRay& Ra, LtRay& Rb, int* rowa,
                                        int* rowb) {
  const float2 D1a = make_float2(Ra.F.dx, Ra.F.dx), D2a = make_float2(Ra.F.dy, Ra.F.dy);
  const float2 D3a = make_float2(Ra.F.dz, Ra.F.dz);
  const float2 D1b = make_float2(Rb.F.dx, Rb.F.dx), D2b = make_float2(Rb.F.dy, Rb.F.dy);
  const float2 D3b = make_float2(Rb.F.dz, Rb.F.dz);
  for (int base = pb; base < pe; base += kLtPB) {
    float2 ua[kLtPB], ub[kLtPB];
#pragma unroll
    for (int i = 0; i < kLtPB; ++i) {
      const float4 a = load_pair<kSrc>(gp, 2 * (base + i));
      const float4 b = load_pair<kSrc>(gp, 2 * (base + i) + 1);
      const float2 NH = kTable ? make_float2(b.z, b.w) : nhp[base + i];
      const float2 CX = make_float2(a.x, a.y), CY = make_float2(a.z, a.w), CZ = make_float2(b.x, b.y);
      ua[i] = __ffma2_rn(CX, D1a, __ffma2_rn(CY, D2a, __ffma2_rn(CZ, D3a, NH)));  // c'.d' - h_l
      ub[i] = __ffma2_rn(CX, D1b, __ffma2_rn(CY, D2b, __ffma2_rn(CZ, D3b, NH)));
    }
    float ma = fmaxf(ua[0].x, ua[0].y), mb = fmaxf(ub[0].x, ub[0].y);
#pragma unroll
    for (int i = 1; i < kLtPB; ++i) {  // a running max: interleaves with the FFMA2 stream (a max16
      ma = fmaxf(ma, fmaxf(ua[i].x, ua[i].y));   // tree measured 7 % / 3 % slower here)
      mb = fmaxf(mb, fmaxf(ub[i].x, ub[i].y));
    }
    const bool ca = Ra.act && ma >= Ra.cu, cb = Rb.act && mb >= Rb.cu;
    if (__any_sync(kFull, ca || cb)) {
      if (ca) {
        unsigned m = 0u;
#pragma unroll
        for (int i = 0; i < kLtPB; ++i)
          m |= ((ua[i].x >= Ra.cu) ? 1u : 0u) << (2 * i) | ((ua[i].y >= Ra.cu) ? 1u : 0u) << (2 * i + 1);
        lt_candidates<kSrc>(P, gp, kTable ? gk : nullptr, m, 2 * base, Ra, rowa);
      }
      if (cb) {
        unsigned m = 0u;
#pragma unroll
        for (int i = 0; i < kLtPB; ++i)
          m |= ((ub[i].x >= Rb.cu) ? 1u : 0u) << (2 * i) | ((ub[i].y >= Rb.cu) ? 1u : 0u) << (2 * i + 1);
        lt_candidates<kSrc>(P, gp, kTable ? gk : nullptr, m, 2 * base, Rb, rowb);
      }
    }
    if (!__any_sync(kFull, Ra.act || Rb.act)) break;  // Alg. 1 `break`, warp-wide
  }
}

// Prefix sums of the lists' 64-entry chunk counts (list i = light i / kLtSub, sub-list i % kLtSub;
// their counters are contiguous); every thread of the CTA takes part (blockDim = 256 >= lists)
__device__ __forceinline__ unsigned lt_chunk_prefix(const DevParams& P, const WfBuffers& B, int d, unsigned* s_end,
                                                    unsigned* s_warp) {
  const int nl = P.lt_lights * kLtSub;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  unsigned v = t < nl ? (B.ctr[wf_ctr_lt(d, 0, 0) + t] + 63u) / 64u : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned u = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) s_warp[warp] = v;
  __syncthreads();
  unsigned before = 0;
  for (int w = 0; w < warp; ++w) before += s_warp[w];
  if (t < nl) s_end[t] = v + before;
  __syncthreads();
  return nl > 0 ? s_end[nl - 1] : 0u;
}
// list of chunk k: the first list whose prefix end exceeds k (binary search)
__device__ __forceinline__ int lt_list_of(const unsigned* s_end, int nl, unsigned k) {
  int lo = 0, hi = nl - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (s_end[mid] > k) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// thread 0 of wf_isect_lt: the next light (after *light) whose chunks are not all taken, its
// chunk range, and its table staged on the barrier (the previous table is free: every warp
// passed the CTA barrier); *light = -1 when every light's chunks are taken. Out of line: the
// scan's registers are not spent on it.
__device__ __noinline__ void lt_pick_stage(const DevParams& P, const DevScene& S, const WfBuffers& B, int d,
                                           const unsigned* s_chunk_end, uint64_t* mbar, int* light, unsigned* lo_out,
                                           unsigned* hi_out, unsigned tpc) {
  const int LT = P.lt_lights;
  int pick = -1;
  unsigned plo = 0u, phi = 0u;
  for (int t = 1; t <= LT && pick < 0; ++t) {  // the light's head counts units of tpc chunks
    const int l = (*light + t) % LT;
    const unsigned lo = l > 0 ? s_chunk_end[l * kLtSub - 1] : 0u, hi = s_chunk_end[l * kLtSub + kLtSub - 1];
    if (*(volatile unsigned*)(B.ctr + wf_ctr_wltl(d, l)) < (hi - lo + tpc - 1u) / tpc) { pick = l; plo = lo; phi = hi; }
  }
  *light = pick;
  *lo_out = plo;
  *hi_out = phi;
  if (pick < 0) return;
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  const uint32_t table_bytes = (uint32_t)lt_table_stride(P.n_pairs_pad) * 16u;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(table_bytes) : "memory");
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s_pairs);
  const char* src = reinterpret_cast<const char*>(S.pairs_ltl + (size_t)pick * lt_table_stride(P.n_pairs_pad));
  constexpr uint32_t kChunk = 1u << 15;
  for (uint32_t off = 0; off < table_bytes; off += kChunk) {
    const uint32_t n = (table_bytes - off) < kChunk ? (table_bytes - off) : kChunk;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + off),
                 "l"(src + off), "r"(n), "r"(mb)
                 : "memory");
  }
}

// Long lists: a CTA works on one light at a time and stages only that light's table (the pair
// layout with -h in place of K: two LDS.128 per pair and no column load, 32 B per pair of shared
// memory whatever the number of lights). It starts on light blockIdx % lights, takes 64-entry
// chunks of that light's sub-lists (one head per light) and, when they run out, moves to the next
// light with chunks left, restaging after a CTA barrier.
template <int kSrc>
__global__ void __launch_bounds__(256, kIsectMinBlocks)
wf_isect_lt(const DevParams P, const DevScene S, WfBuffers B, int d) {
  static_assert(kSrc == SRC_SMEM, "light-origin scan stages the light tables in smem");
  __shared__ uint64_t s_mbar;
  __shared__ unsigned s_chunk_end[kMaxLtLights * kLtSub];
  __shared__ unsigned s_warp[8];
  __shared__ int s_light;                  // the light being scanned (thread 0 picks it), -1: done
  __shared__ unsigned s_lo, s_hi, s_phase;  // its chunk range, the staging barrier's parity
  const unsigned n_chunks = lt_chunk_prefix(P, B, d, s_chunk_end, s_warp);
  if (!B.solo && split_parts(n_chunks, B) > 1) return;  // a short list: wf_isect_lt_split scans it
  if ((unsigned long long)blockIdx.x * (blockDim.x / 32u) >= n_chunks) return;  // CTAs without work
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&s_mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_light = (int)(blockIdx.x % (unsigned)P.lt_lights) - 1;  // the first pick starts at blockIdx % lights
    s_phase = 0u;
  }
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) lt_pick_stage(P, S, B, d, s_chunk_end, &s_mbar, &s_light, &s_lo, &s_hi, 1u);
    __syncthreads();
    const int L = s_light;
    if (L < 0) break;
    mbar_wait(&s_mbar, s_phase);
#if RT_CHECKS
    for (int q = threadIdx.x; q < P.n_pairs_pad; q += blockDim.x) {
      const float4 a = s_pairs[2 * q], b = s_pairs[2 * q + 1], ga = S.pairs[2 * q], gb = S.pairs[2 * q + 1];
      const float2 nh = reinterpret_cast<const float2*>(S.pairs_lt + 2 * P.n_pairs_pad)[(size_t)L * P.n_pairs_pad + q];
      RT_CHECK(a.x == ga.x && a.y == ga.y && a.z == ga.z && a.w == ga.w, 405);
      RT_CHECK(b.x == gb.x && b.y == gb.y, 406);
      RT_CHECK(b.z == nh.x && b.w == nh.y, 407);
    }
#endif
    while (true) {
      unsigned k = 0;
      if (lane == 0) k = atomicAdd(B.ctr + wf_ctr_wltl(d, L), 1u);
      k = __shfl_sync(kFull, k, 0) + s_lo;  // a chunk of light L's sub-lists
      if (k >= s_hi) break;
      const int li = lt_list_of(s_chunk_end, P.lt_lights * kLtSub, k);
      const unsigned c = k - (li > 0 ? s_chunk_end[li - 1] : 0u);
      const unsigned cnt = B.ctr[wf_ctr_lt(d, 0, 0) + li];
      RT_CHECK(cnt <= (unsigned)B.lt_cap && li / kLtSub == L, 402);
      const unsigned oa = 64u * c + (unsigned)lane, ob = oa + 32u;
      const bool va_ = oa < cnt, vb_ = ob < cnt;
      const unsigned ga = (unsigned)li * B.lt_cap + oa, gb = ga + 32u;  // list slots
      LtRay Ra, Rb;
      lt_setup(P, S, B, ga, va_, L, Ra);
      lt_setup(P, S, B, gb, vb_, L, Rb);
      lt_scan<kSrc, true>(P, s_pairs, nullptr, reinterpret_cast<const float2*>(s_pairs + 2 * P.n_pairs_pad), 0,
                          P.n_pairs_pad, Ra, Rb, B.lt_cand + (size_t)ga * kCandMax, B.lt_cand + (size_t)gb * kCandMax);
#if RT_CHECKS
      {  // the same rays through the shared-layout scan from global memory
        LtRay Ra2, Rb2;
        lt_setup(P, S, B, ga, va_, L, Ra2);
        lt_setup(P, S, B, gb, vb_, L, Rb2);
        int* xa = B.xcand_s + ((size_t)(blockIdx.x * 8 + (threadIdx.x >> 5)) * 64 + lane) * kCandMax;
        lt_scan<SRC_GLOBAL, false>(P, S.pairs_lt, reinterpret_cast<const float2*>(S.pairs_lt + 2 * P.n_pairs_pad) +
                                   (size_t)L * P.n_pairs_pad, nullptr, 0, P.n_pairs_pad, Ra2, Rb2, xa, xa + 32 * kCandMax);
        RT_CHECK(!va_ || (Ra.rob == Ra2.rob && Ra.nc == Ra2.nc), 408);
        RT_CHECK(!vb_ || (Rb.rob == Rb2.rob && Rb.nc == Rb2.nc), 409);
      }
#endif
      if (va_) B.lt_res[ga] = make_int2(Ra.rob, Ra.nc);
      if (vb_) B.lt_res[gb] = make_int2(Rb.rob, Rb.nc);
    }
    __syncthreads();  // every warp is done with light L's table (and has read s_phase)
    if (threadIdx.x == 0) s_phase ^= 1u;
  }
}

// the light-origin scan of a short list: parts warps of a CTA share a 64-entry chunk (sphere
// ranges), merged in part order as in wf_isect_split
// Two organisations of the short-list scan: every light's -h column staged beside the pairs (a
// CTA unit may mix lights; up to 64 KB of columns: C4 frame 5.490 vs 5.501 ms, world-8 shard
// 0.93 vs 0.95 ms), or one light's table at a time (any number of lights x spheres)
template <int kSrc>
__device__ __forceinline__ void wf_isect_lt_split_cols(const DevParams& P, const DevScene& S, const WfBuffers& B, int d) {
  static_assert(kSrc == SRC_SMEM, "light-origin scan stages the light tables in smem");
  __shared__ uint64_t s_mbar;
  __shared__ unsigned s_chunk_end[kMaxLtLights * kLtSub];
  __shared__ unsigned s_warp[8];
  __shared__ int s_nc[8][64];
  __shared__ int s_rob[8][64];
  __shared__ unsigned s_unit;
  const unsigned n_chunks = lt_chunk_prefix(P, B, d, s_chunk_end, s_warp);
  const int parts = split_parts(n_chunks, B);
  if (parts == 1 && !B.solo) return;  // a long list: wf_isect_lt scans it (solo: one part here)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tpc = 8 / parts;  // chunks per CTA unit
  const unsigned units = (n_chunks + tpc - 1) / tpc;
  if (blockIdx.x >= units) return;  // CTAs without work leave before staging the scene
  stage_scene(s_pairs, S.pairs_lt, (uint32_t)P.n_pairs_pad * 32u + (uint32_t)P.lt_lights * P.n_pairs_pad * 8u, &s_mbar);
  const float4* gp = S.pairs_lt;
  const float2* nh_all = reinterpret_cast<const float2*>(s_pairs + 2 * P.n_pairs_pad);
  const int slot = warp / parts, part = warp % parts;
  const int nl = P.lt_lights * kLtSub;
  int pb, pe;
  split_range(P, part, parts, pb, pe);
  const size_t xs = (size_t)64 * kCandMax;
  int* xa = B.xcand_s + ((size_t)(blockIdx.x * 8 + warp) * 64 + lane) * kCandMax;
  int* xb = xa + 32 * kCandMax;
  while (true) {
    if (threadIdx.x == 0) s_unit = atomicAdd(B.ctr + wf_ctr_wlt(d), 1u);
    __syncthreads();
    const unsigned u = s_unit;
    if (u >= units) break;  // CTA-uniform
    const unsigned k = u * tpc + slot;
    const bool valid_chunk = k < n_chunks;
    const int li = valid_chunk ? lt_list_of(s_chunk_end, nl, k) : 0;
    const int l = li / kLtSub;
    const unsigned c = k - (li > 0 ? s_chunk_end[li - 1] : 0u);
    const unsigned cnt = valid_chunk ? B.ctr[wf_ctr_lt(d, 0, 0) + li] : 0u;
    const unsigned oa = 64u * c + (unsigned)lane, ob = oa + 32u;
    const bool va_ = oa < cnt, vb_ = ob < cnt;
    const unsigned ga = (unsigned)li * B.lt_cap + oa, gb = ga + 32u;
    LtRay Ra, Rb;
    lt_setup(P, S, B, ga, va_, l, Ra);
    lt_setup(P, S, B, gb, vb_, l, Rb);
    lt_scan<kSrc>(P, gp, nh_all + (size_t)l * P.n_pairs_pad, nullptr, pb, pe, Ra, Rb, xa, xb);
    s_nc[warp][lane] = Ra.nc;
    s_nc[warp][lane + 32] = Rb.nc;
    s_rob[warp][lane] = Ra.rob;
    s_rob[warp][lane + 32] = Rb.rob;
    __syncthreads();
    if (part == 0) {
      int nco, robo;
      if (va_) {
        split_merge_shadow(parts, &s_nc[warp][lane], &s_rob[warp][lane], 64, xa, xs, B.lt_cand + (size_t)ga * kCandMax, nco,
                           robo);
        B.lt_res[ga] = make_int2(robo, nco);
      }
      if (vb_) {
        split_merge_shadow(parts, &s_nc[warp][lane + 32], &s_rob[warp][lane + 32], 64, xb, xs,
                           B.lt_cand + (size_t)gb * kCandMax, nco, robo);
        B.lt_res[gb] = make_int2(robo, nco);
      }
    }
    __syncthreads();  // s_unit / s_nc / s_rob / scratch rows are rewritten by the next unit
  }
}

template <int kSrc>
__device__ __forceinline__ void wf_isect_lt_split_body(const DevParams& P, const DevScene& S, const WfBuffers& B, int d) {
  static_assert(kSrc == SRC_SMEM, "light-origin scan stages the light tables in smem");
  __shared__ uint64_t s_mbar;
  __shared__ unsigned s_chunk_end[kMaxLtLights * kLtSub];
  __shared__ unsigned s_warp[8];
  __shared__ int s_nc[8][64];
  __shared__ int s_rob[8][64];
  __shared__ unsigned s_unit;
  __shared__ int s_light;                  // as in wf_isect_lt: one light's table at a time
  __shared__ unsigned s_lo, s_hi, s_phase;
  const unsigned n_chunks = lt_chunk_prefix(P, B, d, s_chunk_end, s_warp);
  const int parts = split_parts(n_chunks, B);
  if (parts == 1 && !B.solo) return;  // a long list: wf_isect_lt scans it (solo: one part here)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tpc = 8 / parts;  // chunks per CTA unit (units never straddle two lights)
  if (blockIdx.x >= (n_chunks + tpc - 1) / tpc + (unsigned)P.lt_lights) return;  // CTAs without work
  const int slot = warp / parts, part = warp % parts;
  const int nl = P.lt_lights * kLtSub;
  int pb, pe;
  split_range(P, part, parts, pb, pe);
  const size_t xs = (size_t)64 * kCandMax;
  int* xa = B.xcand_s + ((size_t)(blockIdx.x * 8 + warp) * 64 + lane) * kCandMax;
  int* xb = xa + 32 * kCandMax;
  if (threadIdx.x == 0) {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&s_mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_light = (int)(blockIdx.x % (unsigned)P.lt_lights) - 1;
    s_phase = 0u;
  }
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) lt_pick_stage(P, S, B, d, s_chunk_end, &s_mbar, &s_light, &s_lo, &s_hi, (unsigned)tpc);
    __syncthreads();
    const int l = s_light;
    if (l < 0) break;
    mbar_wait(&s_mbar, s_phase);
    const unsigned units = (s_hi - s_lo + tpc - 1) / tpc;
    while (true) {
      if (threadIdx.x == 0) s_unit = atomicAdd(B.ctr + wf_ctr_wltl(d, l), 1u);
      __syncthreads();
      const unsigned u = s_unit;
      if (u >= units) break;  // CTA-uniform
      const unsigned k = s_lo + u * tpc + slot;
      const bool valid_chunk = k < s_hi;
      const int li = valid_chunk ? lt_list_of(s_chunk_end, nl, k) : l * kLtSub;
      RT_CHECK(li / kLtSub == l, 404);
      const unsigned c = k - (li > 0 ? s_chunk_end[li - 1] : 0u);
      const unsigned cnt = valid_chunk ? B.ctr[wf_ctr_lt(d, 0, 0) + li] : 0u;
      const unsigned oa = 64u * c + (unsigned)lane, ob = oa + 32u;
      const bool va_ = oa < cnt, vb_ = ob < cnt;
      const unsigned ga = (unsigned)li * B.lt_cap + oa, gb = ga + 32u;
      LtRay Ra, Rb;
      lt_setup(P, S, B, ga, va_, l, Ra);
      lt_setup(P, S, B, gb, vb_, l, Rb);
      lt_scan<kSrc, true>(P, s_pairs, nullptr, reinterpret_cast<const float2*>(s_pairs + 2 * P.n_pairs_pad), pb, pe, Ra,
                          Rb, xa, xb);
      s_nc[warp][lane] = Ra.nc;
      s_nc[warp][lane + 32] = Rb.nc;
      s_rob[warp][lane] = Ra.rob;
      s_rob[warp][lane + 32] = Rb.rob;
      __syncthreads();
      if (part == 0) {
        int nco, robo;
        if (va_) {
          split_merge_shadow(parts, &s_nc[warp][lane], &s_rob[warp][lane], 64, xa, xs, B.lt_cand + (size_t)ga * kCandMax,
                             nco, robo);
          B.lt_res[ga] = make_int2(robo, nco);
        }
        if (vb_) {
          split_merge_shadow(parts, &s_nc[warp][lane + 32], &s_rob[warp][lane + 32], 64, xb, xs,
                             B.lt_cand + (size_t)gb * kCandMax, nco, robo);
          B.lt_res[gb] = make_int2(robo, nco);
        }
      }
      __syncthreads();  // s_unit / s_nc / s_rob / scratch rows are rewritten by the next unit
    }
    __syncthreads();  // every warp is done with light l's table (and has read s_phase)
    if (threadIdx.x == 0) s_phase ^= 1u;
  }
}

template <int kSrc, bool kPerLight>
__global__ void __launch_bounds__(256, 2)  // two rays per thread plus the merge: no spills at 2 CTAs/SM
wf_isect_lt_split(const DevParams P, const DevScene S, WfBuffers B, int d) {
  if constexpr (kPerLight) wf_isect_lt_split_body<kSrc>(P, S, B, d);
  else wf_isect_lt_split_cols<kSrc>(P, S, B, d);
}

// FP64 nearest sphere among the candidate list (index order, strict <), or a full scan when
// the list overflowed. The planes were decided first (tbest, hp): a sphere at exactly the same t
// wins the tie when its primitive index is lower (ties -> lowest index, whatever the
// interleaving of spheres and planes in the input)
__device__ __forceinline__ bool beats(const DevScene& S, double t, int k, double tbest, int hp) {
  return t < tbest || (t == tbest && hp >= 0 && S.sph_prim[k] < c_planes[hp].prim);
}
__device__ __forceinline__ void nearest_sphere(const DevParams& P, const DevScene& S, const int* cand, int nc,
                                               int skip, d3 o, d3 d, double& tbest, int& hs, int& hp) {
  if (nc <= kCandMax) {
    for (int c = 0; c < nc; ++c) {
      const int k = cand[c];
      RT_CHECK(k >= 0 && k < P.n_spheres, 301);
      const double t = sphere_root(__ldg(S.sph_cr + k), o, d);
      if (t >= kEps && beats(S, t, k, tbest, hp)) { tbest = t; hs = k; hp = -1; }
    }
  } else {
    for (int k = 0; k < P.n_spheres; ++k) {
      if (k == skip) continue;
      const double t = sphere_root(__ldg(S.sph_cr + k), o, d);
      if (t >= kEps && beats(S, t, k, tbest, hp)) { tbest = t; hs = k; hp = -1; }
    }
  }
}

// Test counts of one shadow ray in primitive index order (§8(c).1 step 11; Alg. 1 `break`). The
// scans test planes first: hp = the first occluding plane (or -1); otherwise hs = the first
// occluding sphere in sphere order (or -1). Spheres precede a plane in index order when the input
// interleaves them (sph_prim / DevPlane::prim): if plane hp occludes, a sphere listed before it may
// be the first occluder in index order, decided here in FP64 (a loop over those spheres only; the
// generated scenes list planes first, where it is empty). skip: the sphere the ray leaves (tested,
// never an occluder); skip2: the aimed-at emitter (not tested, R#41).
// the first occluder among spheres 0..n-1 (FP64), or -1: a rare path (interleaved inputs only),
// kept out of line so the callers' register budgets stay those of the planes-first case
__device__ __noinline__ int first_occluder_before(const DevScene& S, d3 o, d3 d, double tl, int n, int skip, int skip2) {
  for (int k = 0; k < n; ++k) {
    if (k == skip || k == skip2) continue;
    const double t = sphere_root(__ldg(S.sph_cr + k), o, d);
    if (t >= kEps && t < tl) return k;
  }
  return -1;
}
__device__ __forceinline__ void shadow_counts(const DevParams& P, const DevScene& S, d3 o, d3 d, double tl, int hp,
                                              int hs, int skip, int skip2, unsigned long long& nsph,
                                              unsigned long long& npl) {
  int first = hs;
  if (hp >= 0) {
    const int before = c_planes[hp].prim - hp;  // spheres listed before plane hp
    if (before > 0) first = first_occluder_before(S, o, d, tl, before, skip, skip2);
    if (first < 0) {
      npl = (unsigned long long)(hp + 1);
      nsph = (unsigned long long)before - ((skip2 >= 0 && skip2 < before) ? 1ull : 0ull);
      return;
    }
  }
  if (first >= 0) {
    nsph = (unsigned long long)(first + 1) - ((skip2 >= 0 && skip2 < first) ? 1ull : 0ull);
    npl = (unsigned long long)(S.sph_prim[first] - first);  // planes listed before sphere `first`
  } else {
    nsph = (unsigned long long)P.n_spheres - (skip2 >= 0 ? 1ull : 0ull);
    npl = (unsigned long long)P.n_planes;
  }
}

// ---- a4 + a6: nearest hit, emission/ambient, shadow entries, continuation -------------------
// wf_accumulate: 40 registers (160 B spilled: the rare FP64 decisions), 6 CTAs per SM = the logic kernels' grid of 6 CTAs
// per SM in one wave (C4 in order: 4 CTAs / 64 registers 0.550 ms, 5 / 48 (1.2 waves) 0.589,
// 6 / 40 0.514, 8 / 32 (52 B spilled) 0.555)
constexpr int kLogicMinBlocks = 6;
constexpr int kShadeMinBlocks = 3;  // wf_shade: 80 registers, no spills (64: ~190 B spilled, 10 % slower)
// warps that reserve light-origin list slots together (C4 frame: 8 -> 5.842, 4 -> 5.832,
// 2 -> 5.876, 1 -> 5.907 ms: smaller groups wait less, but their list ranges are less coherent)
constexpr int kResWarps = 4;
static_assert(8 % kResWarps == 0, "groups of a 256-thread CTA");
// barrier of the n threads of named barrier `id` (a group of whole warps)
__device__ __forceinline__ void group_sync(int id, int n) {
  if (n == 256) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// kExt: the NEXT-1/NEXT-2 extensions (emitters sampled as area lights, the global integrator)
// are compiled in; the §8(a) hot path (Whitted, point lights) runs the kExt = false instance.
//
// Shadow entries: entry j (path-major: the entries of Q[d]'s entry e are shoff[e] .. + shcnt[e],
// sources in order) carries its contribution sq_c[j] and spos[j], where its scan lives:
//  * point light l < lt_lights (light-origin scans): a slot g of one of light l's sub-lists,
//    holding {e, skip}; the ray is rebuilt from B.sorg[e] = p + EPS_T n by the scan and, when an
//    FP64 decision needs it, by wf_accumulate (spos[j] = g >= 0);
//  * any other source (emitters, or every light when the scene is not in shared memory): a dense
//    generic slot o (spos[j] = -2 - o) holding the FP64 shadow ray, its skips and the scan results.
// Every slot a warp needs is reserved in one round trip: lane-parallel atomics for the shadow
// entries, the continuations and the generic slots; the light-origin lists per group of kResWarps
// warps (one atomic per light and group iteration, warps in order, so a list keeps the group's
// 128 neighbouring paths together: coherent early exits in the scan). The group barrier of that
// reservation sits before the light loop, so warps wait for the slowest warp's hit and bounce,
// not for its light loop.
template <bool kDebug, bool kExt>
__global__ void __launch_bounds__(256, kShadeMinBlocks) wf_shade(const DevParams P, const DevScene S, WfBuffers B, int d,
                                                long long g0, int* dbg_hits, int* dbg_bounces) {
  const unsigned n = B.ctr[wf_ctr_q(d)];
  RT_CHECK(n <= (unsigned)B.cap, 100);
  const WfQueue Q = B.q[d & 1], Qn = B.q[(d + 1) & 1];
  const int w0 = B.w0;  // first work item of the chunk (g0 = w0 * spp)
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask_lane = lanemask_lt();
  const int n_src = P.n_lights + (kExt ? P.n_emitters : 0);  // point lights, then emitters (R#41)
  const int LT = P.lt_lights;                                // point lights 0..LT-1: light-origin lists
  const int nres = n_src < 30 ? n_src : 30;                  // sources whose slots are reserved together
  // warp-uniform iterations: every lane of a warp takes part in the ballots of the slot reservations
  const unsigned stride = gridDim.x * blockDim.x;
  __shared__ unsigned s_cnt[8][kMaxLtLights];  // per warp and light-origin light: entries, then first slot
  for (unsigned cb = blockIdx.x * blockDim.x; cb < n; cb += stride) {  // CTA-uniform (CTA barriers below)
    const unsigned e0 = cb + (threadIdx.x & ~31u);
    const unsigned e = e0 + lane;
    const int warp = threadIdx.x >> 5;
    // the CTA's sub-list of every light list: a list keeps the CTA's 256 neighbouring paths
    // together, in warp order (coherent early exits in the light-origin scan)
    const int sub = (int)((cb >> 8) % kLtSub);
    d3 dir = mk(0, 0, 1);
    const bool valid = e < n && q_dir(P, B, Q, e, d, dir);
    if (e < n && !valid) B.shcnt[e] = 0;  // a work item outside the image (depth 0): nothing to shade
    int path = 0, depth = 0, dword = 0, hs = -1, mi = 0;
    unsigned long long lmask = 0ull;  // sources 0..63 that send a shadow ray
    unsigned nsh = 0;
    d3 p = mk(0, 0, 0), nrm = mk(0, 0, 1);
    bool entering = false, hit = false;
    float3 T = f3(1.f, 1.f, 1.f), L = f3(0.f, 0.f, 0.f);
    // pixel index and global sample index of the path (RNG keys, R#42): 32-bit arithmetic on the
    // chunk-local path id (path = local item * spp + s), computed only when a draw needs them
    unsigned long long pix = 0;
    unsigned sg = 0;
    auto pixel_sample = [&]() {
      const int wl = (int)fdiv(P.div_spp, (unsigned)path);
      int px = 0, py = 0;
      item_pixel(P, w0 + wl, px, py);
      pix = (unsigned long long)py * P.W + px;
      sg = (unsigned)(P.sample_base + (path - wl * P.spp));
    };
    long long si = 0;
    // part 1: FP64 nearest hit, hit geometry, emission/ambient, which sources send a shadow ray
    if (valid) {
      path = q_path(Q, e, d);
      const d3 o = q_origin(P, Q, B.cap, e, d);
      double tbest = kInf;
      int hp = -1;
      for (int j = 0; j < P.n_planes; ++j) {
        const DevPlane pl = c_planes[j];
        const double den = pl.nx * dir.x + pl.ny * dir.y + pl.nz * dir.z;
        if (fabs(den) >= 1e-12) {
          const double t = (pl.d - (pl.nx * o.x + pl.ny * o.y + pl.nz * o.z)) / den;
          if (t >= kEps && t < tbest) { tbest = t; hp = j; }
        }
      }
      nearest_sphere(P, S, B.ccand + (size_t)e * kCandMax, B.cn[e], q_skip(Q, e, d), o, dir, tbest, hs, hp);
      dword = d == 0 ? 0 : Q.depth[e];
      depth = dword & 0xff;
      int prim = -1;
      if (hp >= 0) prim = c_planes[hp].prim;
      else if (hs >= 0) prim = S.sph_prim[hs];
      if constexpr (kDebug) {
        const long long g = g0 + path;
        int px = 0, py = 0;
        item_pixel(P, (int)(g / P.spp), px, py);
        si = ((long long)py * P.W + px) * P.spp + (int)(g % P.spp);
        dbg_hits[si * (P.max_depth + 1) + depth] = prim;
      }
      if (d > 0) {
        T = lf3(Q.T, B.cap, (int)e);
        L = lf3(Q.L, B.cap, (int)e);
      }
      if (kExt && (P.n_emitters > 0 || P.integrator != 0)) pixel_sample();
      if (prim < 0) {  // miss -> background
        L = add(L, mul(T, f3(P.bg[0], P.bg[1], P.bg[2])));
      } else {
        hit = true;
        p = o + dir * tbest;
        d3 ng;
        if (hp >= 0) {
          const DevPlane pl = c_planes[hp];
          ng = mk(pl.nx, pl.ny, pl.nz);
          mi = pl.mat;
        } else {
          const float4 cr = __ldg(S.sph_cr + hs);
          ng = (p - mk(cr.x, cr.y, cr.z)) * (1.0 / (double)cr.w);
          mi = S.sph_mat[hs];
        }
        entering = dot(dir, ng) < 0.0;
        nrm = entering ? ng : ng * -1.0;
        const DevMat m = S.mats[mi];
        // Eq. 7 emission, except an emitter already sampled from the previous diffuse vertex (R#43)
        const bool sampled = kExt && (dword & kPrevDiffuse) && P.n_emitters > 0 && hs >= 0;
        if (!sampled) L = add(L, mul(T, f3(m.er, m.eg, m.eb)));
        if (m.kind == 0) {
          L = add(L, mul(T, f3(m.ar * P.amb[0], m.ag * P.amb[1], m.ab * P.amb[2])));
          for (int l = 0; l < n_src; ++l) {  // count shadow rays (none if cos <= 0)
            if (sends_shadow_ray<kExt>(P, S, l, p, nrm, pix, sg, depth)) {
              ++nsh;
              if (l < 64) lmask |= 1ull << l;
            }
          }
        }
      }
    }
    // part 3 (before the entries, so the continuation's temporaries are dead during the light
    // loop): stack-free continuation; Tn = the throughput after the bounce
    bool cont = false;
    unsigned base = 0, off = 0;  // lane l: the first slot of source l's entries (see below); off: lane's first entry
    {
      float3 Tn = T;
      d3 dn = mk(0, 0, 0);
      bool diffuse_global = false;
      if (hit && depth < P.max_depth) {
        const DevMat m = S.mats[mi];
        diffuse_global = kExt && m.kind == 0 && P.integrator == 1;
        if (m.kind == 1) {  // SPECULAR: mirror, T *= rho
          dn = reflect(dir, nrm);
          Tn = mul(Tn, f3(m.ar, m.ag, m.ab));
          cont = true;
        } else if (kExt && m.kind == 0 && P.integrator == 1) {  // global: cosine-weighted bounce (R#40)
          dn = cosine_dir(nrm, rng_stream(P.seed, pix, sg, depth, 3u), rng_stream(P.seed, pix, sg, depth, 4u));
          Tn = mul(Tn, f3(m.ar, m.ag, m.ab));
          cont = true;
        } else if (m.kind == 0) {  // DIFFUSE: mirror with weight kr when kr > 0 (R#8)
          if (m.kr > 0.f) {
            dn = reflect(dir, nrm);
            Tn = f3(Tn.x * m.kr, Tn.y * m.kr, Tn.z * m.kr);
            cont = true;
          }
        } else {  // REFRACTIVE: Schlick-chosen reflect / refract, TIR -> reflect (R#9-R#11)
          const double ior = m.ior;
          const double eta = entering ? 1.0 / ior : ior;
          const double ci = -dot(dir, nrm);
          const double sin2t = eta * eta * (1.0 - ci * ci);
          bool refl = sin2t > 1.0;
          if (!refl) {
            const double cosT = sqrt(1.0 - sin2t);
            const double c = entering ? ci : cosT;
            double r0 = (1.0 - ior) / (1.0 + ior);
            r0 *= r0;
            const double mm = 1.0 - c;
            const double F = r0 + (1.0 - r0) * (mm * mm * mm * mm * mm);
            if (!kExt || (P.n_emitters == 0 && P.integrator == 0)) pixel_sample();
            const double u = rng_u(P.seed, pix, (int)sg, depth);
            refl = u < F;
            if (!refl) dn = dir * eta + nrm * (eta * ci - cosT);
          }
          if (refl) dn = reflect(dir, nrm);
          Tn = mul(Tn, f3(m.ar, m.ag, m.ab));
          cont = true;
        }
        if (cont) dn = normalize(dn);
      }
      // every slot the warp needs, reserved in ONE round trip to L2 (the atomics' latency, not their
      // number, bounded this kernel): lane l < nres takes source l's slots (its light-origin
      // sub-list, or generic slots), lane 30 the warp's shadow entries, lane 31 its continuations
      unsigned pre_sh = 0, tot_sh = 0;  // warp-exclusive prefix / total of nsh (< 64) by bit planes
#pragma unroll
      for (int b = 0; b < 6; ++b) {
        const unsigned m = __ballot_sync(kFull, (nsh >> b) & 1u);
        pre_sh += (unsigned)__popc(m & lt_mask_lane) << b;
        tot_sh += (unsigned)__popc(m) << b;
      }
      const unsigned mc = __ballot_sync(kFull, cont);
      unsigned cnt = 0;
      for (int l = 0; l < nres; ++l) {
        const unsigned bl = __ballot_sync(kFull, ((lmask >> l) & 1ull) != 0ull);
        if (lane == l) cnt = (unsigned)__popc(bl);
      }
      unsigned* ctr = nullptr;
      if (lane < LT) s_cnt[warp][lane] = cnt;  // light-origin lists: reserved per CTA below
      else if (lane < nres) ctr = B.ctr + wf_ctr_so(d);
      else if (lane == 30) { ctr = B.ctr + wf_ctr_s(d); cnt = tot_sh; }
      else if (lane == 31) { ctr = B.ctr + wf_ctr_q(d + 1); cnt = (unsigned)__popc(mc); }
      base = (ctr != nullptr && cnt != 0u) ? atomicAdd(ctr, cnt) : 0u;
      RT_CHECK(lane != 30 || base + cnt <= (unsigned)B.scap, 101);  // shadow entries fit scap
      RT_CHECK(lane != 31 || base + cnt <= (unsigned)B.cap, 102);   // continuations fit Q[d+1]
      RT_CHECK(lane >= nres || lane < LT || base + cnt <= (unsigned)B.gcap, 103);  // generic slots fit gcap
      // the group's warps (kResWarps of them, named barrier 1 + group) reserve together
      const int grp = warp / kResWarps, w0g = grp * kResWarps;
      group_sync(1 + grp, 32 * kResWarps);
      if (warp == w0g && lane < LT) {  // one atomic per light and group; warps in order
        const int l = lane;
        unsigned tot = 0;
        for (int w = w0g; w < w0g + kResWarps; ++w) tot += s_cnt[w][l];
        unsigned b0 = tot ? atomicAdd(B.ctr + wf_ctr_lt(d, l, sub), tot) : 0u;
        RT_CHECK(b0 + tot <= (unsigned)B.lt_cap, 104);  // a light-origin sub-list fits lt_cap
        for (int w = w0g; w < w0g + kResWarps; ++w) {
          const unsigned c = s_cnt[w][l];
          s_cnt[w][l] = b0;
          b0 += c;
        }
      }
      group_sync(1 + grp, 32 * kResWarps);
      if (lane < LT) base = s_cnt[warp][lane];
      off = __shfl_sync(kFull, base, 30) + pre_sh;
      const unsigned slot = __shfl_sync(kFull, base, 31) + (unsigned)__popc(mc & lt_mask_lane);
      if (valid) {
        B.shcnt[e] = (int)nsh;
        B.shoff[e] = (int)off;
        if constexpr (kDebug) {
          if (!cont) dbg_bounces[si] = depth;
        }
        if (cont) {  // the path moves to slot `slot` of Q[d+1] with its whole state
          Qn.path[slot] = path;
          st3(Qn.ray, B.cap, (int)slot, 0, p);
          st3(Qn.ray, B.cap, (int)slot, 3, dn);
          sf3(Qn.T, B.cap, (int)slot, Tn);
          sf3(Qn.L, B.cap, (int)slot, L);
          Qn.depth[slot] = (depth + 1) | (diffuse_global ? kPrevDiffuse : 0);
          // the new ray starts on sphere hs; heading outward it cannot hit it again (its roots are
          // 0 and negative), so the scans skip it exactly; inward (refraction, TIR) it may
          // (the outward normal ng = entering ? nrm : -nrm)
          const double dng = dot(dn, nrm);
          Qn.skip[slot] = (hs >= 0 && (entering ? dng > 0.0 : dng < 0.0)) ? hs : -1;
          B.nxt[e] = (int)slot;
        } else {  // the path ends here: its radiance (lights of this depth still to come) by path id
          RT_CHECK(path >= 0 && path < B.cap, 105);
          sf3(B.Lr, B.cap, path, L);
          B.nxt[e] = -1 - path;
        }
      }
    }
    // part 2 (after the continuation): shadow entries — the contribution T f_r I cos / d^2
    // (Eq. 3, 5, 6) or the emitter estimator, and the shadow ray or its list slot. A shadow
    // ray leaving a sphere hit from outside skips it exactly (convexity): o_s is EPS_T outside and
    // the ray heads away from the tangent plane, so it cannot meet the sphere again.
    if (__any_sync(kFull, nsh != 0u)) {
      const DevMat m = S.mats[mi];
      const int out_sph = (hs >= 0 && entering) ? hs : -1;
      if (nsh != 0u && LT > 0 && (lmask & ((LT >= 64) ? ~0ull : ((1ull << LT) - 1ull))) != 0ull)
        st3(B.sorg, B.cap, (int)e, 0, p + nrm * kEps);  // the light-origin entries' rays start here
      unsigned k = off;
      for (int l = 0; l < n_src; ++l) {  // warp-uniform trip count: the slot ballots need every lane
        const bool has = l < 64 ? ((lmask >> l) & 1ull) != 0ull : false;
        int g = -1;
        const unsigned bal = __ballot_sync(kFull, has);
        if (bal == 0u) continue;
        unsigned first;  // the warp's first slot for source l
        if (l < nres) {
          first = __shfl_sync(kFull, base, l);
        } else {  // sources beyond lane 29 (more than 30 sources): one more round trip each
          first = 0;
          if (lane == 0) first = atomicAdd(B.ctr + (l < LT ? wf_ctr_lt(d, l, sub) : wf_ctr_so(d)), (unsigned)__popc(bal));
          first = __shfl_sync(kFull, first, 0);
        }
        const unsigned pos = first + (unsigned)__popc(bal & lt_mask_lane);
        if (l < LT) g = (l * kLtSub + sub) * B.lt_cap + (int)pos;  // a slot in light l's sub-list `sub`
        else g = -2 - (int)pos;                                     // a dense generic slot
        if (!has) continue;
        LightSample ls;
        light_sample<kExt>(P, S, l, p, nrm, pix, sg, depth, ls);  // true: the count pass decided
        // f_r = rho/pi + ks (s+2)/(2 pi) max(0, r.wo)^s (Eq. 5, R#3); E = I cos / d^2 (Eq. 3),
        // or L_e cos_s cos_l / (d^2 pdf) for an emitter sample (Eq. 8, R#41)
        const d3 rl = nrm * (2.0 * ls.cos_s) - ls.wi;
        const float alpha = (float)fmax(0.0, -dot(rl, dir));
        const float spec = m.ks * (m.shin + 2.0f) * kInv2Pi * phong_lobe(alpha, m.shin);
        const float gg = (float)ls.g;
        sf3(B.sq_c, B.scap, (int)k, mul(T, f3(fmaf(m.ar, kInvPi, spec) * ls.ir * gg, fmaf(m.ag, kInvPi, spec) * ls.ig * gg,
                                             fmaf(m.ab, kInvPi, spec) * ls.ib * gg)));
        RT_CHECK(k < (unsigned)B.scap, 106);
        RT_CHECK(g < 0 || (g >= (l * kLtSub + sub) * B.lt_cap && g < (l * kLtSub + sub + 1) * B.lt_cap), 107);
        RT_CHECK(g >= 0 || -2 - g < B.gcap, 108);
        B.spos[k] = g;
        if (g >= 0) {
          const d3 os = p + nrm * kEps;
          const d3 ws = ls.x - os;
          float4 rec;
          int skip = -1;
          const double t_n = dot(nrm, ws);  // the sign of n.d_s (shadow_skip) is the sign of n.w_s...
          const double band = 1e-14 * (fabs(ws.x) + fabs(ws.y) + fabs(ws.z));
          if (P.n_planes == 0 && (out_sph < 0 || fabs(t_n) > band)) {
            // ...outside the rounding band (sends_shadow_ray's argument); with no plane to decide
            // in FP64 the direction only feeds the float record, which the filter's bounds cover
            // within a few FP64 ulps: an FP64 rsqrt instead of shadow_dir's sqrt and division
            const double d2 = dot(ws, ws), k = rsqrt(d2);
            rec = make_float4((float)(ws.x * k), (float)(ws.y * k), (float)(ws.z * k), (float)(d2 * k));
            skip = (out_sph >= 0 && t_n > 0.0) ? out_sph : -1;
          } else {
            d3 ds;
            double tl;
            shadow_dir(os, ls.x, ds, tl);
            skip = shadow_skip(out_sph, nrm, ds);
            for (int q = 0; q < P.n_planes; ++q) {  // planes first, exactly (FP64), in index order
              const DevPlane pl = c_planes[q];
              const double den = pl.nx * ds.x + pl.ny * ds.y + pl.nz * ds.z;
              if (fabs(den) >= 1e-12) {
                const double t = (pl.d - (pl.nx * os.x + pl.ny * os.y + pl.nz * os.z)) / den;
                if (t >= kEps && t < tl) { skip = -2 - q; break; }
              }
            }
            rec = make_float4((float)ds.x, (float)ds.y, (float)ds.z, (float)tl);
          }
          B.lt_dir[g] = rec;
          B.lt_rec[g] = make_int2((int)e, skip);
#if RT_CHECKS
          B.lt_res[g] = make_int2(-77, -77);  // every slot must be scanned before wf_accumulate reads it
#endif
        } else {
          const int o = -2 - g;
          d3 os2, ds;
          double tl;
          shadow_ray_to(p, nrm, ls.x, os2, ds, tl);
          st3(B.sray, B.gcap, o, 0, os2);
          st3(B.sray, B.gcap, o, 3, ds);
          B.sray[6 * (size_t)B.gcap + o] = tl;
          B.sskip[o] = shadow_skip(out_sph, nrm, ds);
          B.sskip2[o] = (kExt && l >= P.n_lights) ? S.emit_sph[l - P.n_lights] : -1;  // not tested (R#41)
        }
        ++k;
      }
    }
  }
}

// ---- a5 decision + accumulation of the visible lights, in light order ----------------------
// Per shading entry e of Q[d]: its shadow entries in source order; the scan left each one's
// certain occluder rob (sphere k >= 0, plane -2-j, or -1) and candidate list; an occlusion that
// the float filter could not settle is decided here in FP64 on the original ray, exactly as the
// oracle's step 7 (first accepted root in [EPS_T, t_max) in index order).
template <bool kExt>  // false: no emitters, every skip2 is -1 (not read)
__global__ void __launch_bounds__(256, kLogicMinBlocks) wf_accumulate(const DevParams P, const DevScene S, WfBuffers B, int d,
                                                     unsigned long long* stats) {
  const unsigned n = B.ctr[wf_ctr_q(d)];
  const WfQueue Qn = B.q[(d + 1) & 1];
  unsigned long long st_sph = 0, st_pl = 0;  // this thread's test counts, reduced once at the end
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int cnt = B.shcnt[e];
    if (cnt > 0) {
      const int off = B.shoff[e];
      const int loc = B.nxt[e];  // where the path's radiance lives now: Q[d+1] slot or Lr[path]
      float* Ls = loc >= 0 ? Qn.L : B.Lr;
      const int li = loc >= 0 ? loc : -1 - loc;
      float3 L = lf3(Ls, B.cap, li);
      RT_CHECK(off >= 0 && off + cnt <= B.scap && li >= 0 && li < B.cap, 201);
      for (int j = off; j < off + cnt; ++j) {
        const int g = B.spos[j];
        RT_CHECK(g < 0 || g < B.lt_cap * kLtSub * P.lt_lights, 202);
        RT_CHECK(g >= 0 || -2 - g < B.gcap, 203);
        const bool lt = g >= 0;  // a light-origin list slot, else generic slot o = -2 - g
        const int o = lt ? 0 : -2 - g;
        int rob, nc, skip2 = -1;
        const int* cand;
        if (lt) {
          const int2 r = B.lt_res[g];
          RT_CHECK(r.x != -77, 205);
          rob = r.x;
          nc = r.y;
          cand = B.lt_cand + (size_t)g * kCandMax;
        } else {
          rob = B.srob[o];
          nc = B.sn[o];
          cand = B.scand + (size_t)o * kCandMax;
          if (kExt) skip2 = B.sskip2[o];
        }
        // the FP64 shadow ray and the sphere it leaves (only when an FP64 decision needs them)
        auto ray = [&](d3& os, d3& ds, double& tl, int& skip) {
          if (lt) {
            skip = max(B.lt_rec[g].y, -1);  // (a plane occluder's code is not a sphere to skip)
            lt_ray(S, B, (int)e, g / B.lt_cap / kLtSub, os, ds, tl);
          } else {
            os = ld3(B.sray, B.gcap, o, 0);
            ds = ld3(B.sray, B.gcap, o, 3);
            tl = B.sray[6 * (size_t)B.gcap + o];
            skip = B.sskip[o];
          }
        };
        int hp = -1, first = -1;
        if (rob <= -2) {  // plane -2-rob occludes (planes are tested first, in index order)
          hp = -2 - rob;
        } else if (nc > 0) {
          d3 os, ds;
          double tl;
          int skip;
          ray(os, ds, tl, skip);
          if (nc <= kCandMax) {
            for (int i = 0; i < nc; ++i) {
              RT_CHECK(cand[i] >= 0 && cand[i] < P.n_spheres, 204);
              const double t = sphere_root(__ldg(S.sph_cr + cand[i]), os, ds);
              if (t >= kEps && t < tl) { first = cand[i]; break; }
            }
            if (first < 0) first = rob;
          } else {
            for (int k = 0; k < P.n_spheres; ++k) {
              if (k == skip || k == skip2) continue;
              const double t = sphere_root(__ldg(S.sph_cr + k), os, ds);
              if (t >= kEps && t < tl) { first = k; break; }
            }
          }
        } else {
          first = rob;  // a certain occluder with no ambiguous candidate before it, or none
        }
        const bool occluded = hp >= 0 || first >= 0;
        // tests up to the first occluder in index order; the aimed-at emitter is not tested
        unsigned long long ns = 0, np = 0;
        if (hp >= 0 && c_planes[hp].prim != hp) {  // spheres listed before the occluding plane
          d3 os, ds;
          double tl;
          int skip;
          ray(os, ds, tl, skip);
          shadow_counts(P, S, os, ds, tl, hp, -1, skip, skip2, ns, np);
        } else {
          shadow_counts(P, S, mk(0, 0, 0), mk(0, 0, 1), 0.0, hp, first, -1, skip2, ns, np);
        }
        st_sph += ns;
        st_pl += np;
        if (!occluded) L = add(L, lf3(B.sq_c, B.scap, j));
      }
      sf3(Ls, B.cap, li, L);
    }
  }
  warp_stat(stats, 3, st_sph);
  warp_stat(stats, 4, st_pl);
}

// ---- a7: mean over samples in order, 16-byte store ------------------------------------------
// Also the chunk's ray statistics that need no per-ray work (§8(c).1 step 11): primary rays =
// the valid samples, secondary = the continuations queued at depths 1..max_depth, shadow = the
// shadow entries reserved, closest-hit tests = (primary + secondary) x every sphere / plane; the
// shadow rays' test counts come from wf_accumulate.
__global__ void __launch_bounds__(256) wf_resolve(const DevParams P, WfBuffers B, int w0, int nw, float4* out,
                                                  double* accum, unsigned long long* stats) {
  unsigned long long nvalid = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += gridDim.x * blockDim.x) {
    const int w = w0 + i;
    int px = 0, py = 0;
    const bool valid = item_pixel(P, w, px, py);
    if (!valid) {
      if (P.mode == 1) out[w] = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    ++nvalid;
    if (accum) {  // progressive passes: double sums in pass order, mean = sum / passes so far
      double* a = accum + 3 * ((long long)py * P.W + px);
      double a0 = a[0], a1 = a[1], a2 = a[2];
      for (int s = 0; s < P.spp; ++s) {
        const float3 v = lf3(B.Lr, B.cap, i * P.spp + s);
        a0 += (double)v.x;
        a1 += (double)v.y;
        a2 += (double)v.z;
      }
      a[0] = a0; a[1] = a1; a[2] = a2;
      if (out) {
        const double inv = 1.0 / (double)(P.sample_base + P.spp);
        out[(long long)py * P.W + px] = make_float4((float)(a0 * inv), (float)(a1 * inv), (float)(a2 * inv), 1.0f);
      }
      continue;
    }
    float3 acc = f3(0.f, 0.f, 0.f);
    RT_CHECK((i + 1) * P.spp <= B.cap, 501);
    for (int s = 0; s < P.spp; ++s) acc = add(acc, lf3(B.Lr, B.cap, i * P.spp + s));
    const float inv = 1.0f / (float)P.spp;
    const float4 v = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, 1.0f);
    if (P.mode != 1) out[(long long)py * P.W + px] = v;  // frame (mode 0) or peer frame (mode 2)
    else out[w] = v;
  }
  const unsigned long long prim = nvalid * (unsigned long long)P.spp;
  warp_stat(stats, 0, prim);
  warp_stat(stats, 3, prim * (unsigned long long)P.n_spheres);
  warp_stat(stats, 4, prim * (unsigned long long)P.n_planes);
  warp_stat(stats, 5, prim * (unsigned long long)P.n_spheres);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long sec = 0, sh = 0;
    for (int dd = 0; dd <= P.max_depth; ++dd) {
      sh += B.ctr[wf_ctr_s(dd)];
      if (dd > 0) sec += B.ctr[wf_ctr_q(dd)];
    }
    atomicAdd(stats + 1, sh);
    atomicAdd(stats + 2, sec);
    atomicAdd(stats + 3, sec * (unsigned long long)P.n_spheres);
    if (P.n_planes) atomicAdd(stats + 4, sec * (unsigned long long)P.n_planes);
    atomicAdd(stats + 5, sec * (unsigned long long)P.n_spheres);
  }
}

// schedule fuzzing (rt_set_schedule_jitter): one thread spins for `ns` nanoseconds of global time
__global__ void spin_ns(unsigned ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(500);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

__global__ void fill_int(int* p, long long n, int v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace rt
