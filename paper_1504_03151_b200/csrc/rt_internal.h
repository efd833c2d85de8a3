// rt_internal.h — device-side data layout shared by the host runtime (rt_api.cu) and the
// kernels (rt_kernels.cu). Not part of the public ABI (include/rt.h).
//
// HBM / on-chip layout:
//   spheres : AoSoA pairs, 32 B per pair of spheres in scene-centred coordinates c' = c - centre:
//             float4 {c'xA, c'xB, c'yA, c'yB}, float4 {c'zA, c'zB, KA, KB} with K = r^2 - |c'|^2;
//             padded with K = -1e30 dummies to a multiple of kPairsPerBatch pairs. Global memory;
//             staged per CTA into shared memory with one TMA bulk copy when <= kMaxSmemPairs
//             pairs (warp-uniform LDS.128 broadcasts), else read from global memory.
//   pairs_eye / pairs_lt : the same layout with s1 = K + 2 c'.o' of the eye / of each point light
//   sph_cr  : float4 {cx, cy, cz, r} per sphere (shading only), global
//   sph_prim/sph_mat : int per sphere (original primitive index / material), global
//   planes  : DevPlane[n_planes] (double) in the constant bank (tested before spheres)
//   lights  : DevLight[n_lights], global (lane-divergent index in the shading code)
//   mats    : DevMat[n_mats], global
//
// Precision split: the sphere scan is a conservative float32 filter
// (FFMA2, two spheres per instruction) whose candidates are re-decided in float64 from the exact
// float inputs; rays, hit points, normals, shadow-ray set-up and the bounce are float64.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>


// bounds / capacity checks of the checked build (-DRT_CHECKS=1, test support): the first failing
// check's id is recorded in g_rt_check (rt_check_status); compiled out by default
#ifndef RT_CHECKS
#define RT_CHECKS 0
#endif
#if RT_CHECKS
#define RT_CHECK(cond, id)                                                    \
  do {                                                                        \
    if (!(cond)) atomicCAS(&::rt::g_rt_check, 0u, (unsigned)(id));          \
  } while (0)
#else
#define RT_CHECK(cond, id) \
  do {                     \
  } while (0)
#endif

namespace rt {

constexpr int kWarp = 32;
constexpr int kPairsPerBatch = 8;  // 2x spheres per unrolled batch of the scans
constexpr int kMaxSmemPairs = 5120;  // 10240 spheres = 160 KB of dynamic shared memory per CTA
constexpr int kMaxPlanes = 32;
constexpr int kMaxLights = 32;
constexpr int kTileW = 8, kTileH = 4, kTilePx = kTileW * kTileH;

struct DevPlane {
  double nx, ny, nz, d;  // unit normal (normalised in double from the float input), n.x = d
  int prim, mat, pad0, pad1;
};

struct DevLight {
  float px, py, pz, ix, iy, iz, pad0, pad1;
};

struct DevMat {
  float ar, ag, ab;     // albedo rho
  float er, eg, eb;     // emission L_e
  float ior, ks, shin, kr;
  int kind;
  float pad;
};

// Exact unsigned 32-bit division by a runtime divisor d >= 1 (Granlund-Montgomery, round-up
// multiplier): t = umulhi(x, m), q = (t + ((x - t) >> 1)) >> (l - 1), l = ceil(log2 d), for every
// 32-bit x; d = 1 passes x through. Host-initialised once per render (DevParams).
struct FastDiv {
  unsigned d, m, s;
};
inline FastDiv make_fastdiv(unsigned d) {
  FastDiv f{d, 0u, 0u};
  if (d <= 1u) return f;
  unsigned l = 0;
  while ((1ull << l) < d) ++l;  // l = ceil(log2 d) >= 1
  f.m = (unsigned)((((1ull << 32) * ((1ull << l) - d)) / d) + 1ull);
  f.s = l - 1u;
  return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ unsigned fdiv(const FastDiv& f, unsigned x) {
  if (f.d <= 1u) return x;
  const unsigned t = __umulhi(x, f.m);
  return (t + ((x - t) >> 1)) >> f.s;
}
#endif

struct DevParams {
  // camera (basis in double): d = normalize(F + (2sx-1) R + (1-2sy) U)
  double eye[3], F[3], R[3], U[3];
  float bg[3], amb[3];
  double centre[3];  // scene centre (bounding box of the spheres): origin of the filter frame
  float cmax;   // filter error bound: max over spheres of |c'| (c' = c - centre)
  float rmax;   // max sphere radius
  int W, H, max_depth, spp;
  int n_spheres, n_pairs_pad, n_planes, n_lights;
  unsigned long long seed;
  // SURVEY §8(f) NEXT-1 / NEXT-2 (all zero = the §8(a) hot path; R#40-R#43)
  int integrator;     // 0 Whitted, 1 global (cosine-weighted diffuse bounce)
  int lt_lights;      // point lights whose shadow rays are scanned from the light (0 = off)
  int n_emitters;     // emissive spheres sampled as area lights (0 = area lights off)
  int jitter;         // 1: random sub-pixel offsets from RNG streams 1/2 (progressive passes)
  int min_chunks;     // host side: cut the frame into at least this many chunks (0: no minimum)
  long long sample_base;  // global index of sample 0 (pass index of the first pass)
  // job: full frame (mode 0, tile-major work items, row-major output) or shard (mode 1)
  // mode 0: full frame, tile-major items, row-major output; 1: shard, slab output (tile-major);
  // 2: direct shard, the rank's tiles stored row-major into a (possibly peer) frame
  int mode, rank, world, tiles_x, n_tiles, n_items;
  FastDiv div_spp, div_tiles_x;  // exact divisions by spp and tiles_x (camera rays, pixels)
  double inv_w, inv_h;           // 1/W, 1/H: the camera-ray scan's filter directions (not decisions)
};

struct DevScene {
  const float4* pairs;     // the pair layout in global memory (staged into shared memory per CTA)
  const float4* sph_cr;
  const int* sph_prim;
  const int* sph_mat;
  const DevMat* mats;
  const DevLight* lights;
  const int* emit_sph;     // [n_emitters] sphere index of emitter e (prim order), or null
  // camera rays: the pair layout with -h(eye) in place of K (rt_kernels.cu neg_tangent), followed by
  // s1 = K + 2 c'.o'(eye), float2 per sphere pair [n_pairs_pad]
  const float4* pairs_eye;
  // light-origin shadow scans of short lists (wf_isect_lt_split): the pair layout followed by
  // -h(P_l) per point light, float2 per sphere pair, [lt_lights][n_pairs_pad] (one TMA bulk copy
  // stages both)
  const float4* pairs_lt;
  // per point light l: the pair layout with -h(P_l) in place of K, followed by K as one float2 per
  // pair (for the candidates' chord bounds): lt_table_stride(n_pairs_pad) float4 per light; the
  // long-list light-origin scan stages one light's table at a time
  const float4* pairs_ltl;
};

__host__ __device__ constexpr int lt_table_stride(int npp) { return 2 * npp + (npp + 1) / 2; }  // float4 per light

struct DevOutputs {
  float4* out;                  // framebuffer (mode 0) or slab (mode 1)
  unsigned int* work_counter;   // persistent work queue head
  unsigned long long* stats;    // [6] primary, shadow, secondary, sphere_tests, plane_tests,
                                //     closest_sphere_tests
  int* dbg_hits;                // optional [n_px * spp * (max_depth+1)]
  int* dbg_bounces;             // optional [n_px * spp]
  double* accum;                // optional [H][W][3] progressive sums (rt_render_passes)
};

// ---- wavefront variant buffers (rt_wavefront.cuh) ----
constexpr int kCandMax = 6;  // candidates stored per ray; more -> overflow -> FP64 full scan

// Closest-hit queue of one depth, compacted by copy: entry e carries its path's whole state, so
// every wavefront kernel reads and writes its entries with coalesced accesses.
struct WfQueue {
  int* path;       // [cap]     path id (chunk-local: g0 + path = pixel item * spp + sample)
  double* ray;     // [6][cap]  o, d
  float* T;        // [3][cap]  throughput
  float* L;        // [3][cap]  radiance so far
  int* depth;      // [cap]     segment depth | kPrevDiffuse when the ray left a cosine bounce
  int* skip;       // [cap]     sphere the ray leaves (provably not hit: convexity) or -1
};

struct WfBuffers {
  WfQueue q[2];    // Q[d & 1]: the closest-hit rays of depth d
  float* Lr;       // [3][cap]  final radiance per path (written when the path ends)
  int* nxt;        // [cap]  per entry of Q[d]: its slot in Q[d+1], or -1 - path if the path ended
  int* shoff;      // [cap]  per entry of Q[d]: first shadow entry
  int* shcnt;      // [cap]  per entry of Q[d]: number of shadow entries (lights in order)
  int* ccand;      // [cap * kCandMax] closest-hit candidates per entry of Q[d]
  int* cn;         // [cap]
  // shadow entries j (path-major: entry e of Q[d] owns shoff[e] .. shoff[e] + shcnt[e] - 1)
  float* sq_c;     // [3][scap] contribution T f_r I cos / d^2 (or the emitter estimator)
  int* spos;       // [scap] where entry j is scanned: light-origin list slot g >= 0, or -2 - o
  double* sorg;    // [3][cap] per entry of Q[d] with light-origin entries: o_s = p + EPS_T n
  // light-origin lists (point light l < lt_lights): kLtSub sub-lists per light, lt_cap slots each;
  // slot g = (l * kLtSub + sub) * lt_cap + position
  float4* lt_dir;  // [slots] the shadow ray's direction and t_max, rounded to float
  int2* lt_rec;    // [slots] {entry e of Q[d], skip: sphere the ray leaves or -1; -2-j plane j occludes}
  int2* lt_res;    // [slots] {robust occluder rob, candidate count nc}, written by the scan
  int* lt_cand;    // [slots * kCandMax]
  int lt_cap;
  // generic shadow entries (every other source: emitters, or all lights when the scene is not in
  // shared memory), dense slots o in [0, ctr_so)
  double* sray;    // [7][gcap] o_s (3), d_s (3), t_max
  int* sskip;      // [gcap] sphere the shadow ray leaves (exact skip) or -1
  int* sskip2;     // [gcap] emitter sphere the ray aims at (not tested, R#41) or -1
  int* scand;      // [gcap * kCandMax]
  int* sn;         // [gcap]
  int* srob;       // [gcap] robust occluder: sphere index, -1 none, -2-j plane j
  unsigned* ctr;   // counters, see wf_ctr_*
  int cap, scap, gcap;
  // split scans (short queues): per-part candidate lists of the warps of up to xctas CTAs, one
  // row of kCandMax per ray; closest scans (32 rays per warp) and shadow scans (64 rays per
  // warp) have their own rows because they run concurrently on two streams
  int* xcand_c;    // [xctas * 8 * 32 * kCandMax]
  float* xlo_c;    // [xctas * 8 * 32 * kCandMax] lower bound of each closest candidate's root
  int* xcand_s;    // [xctas * 8 * 64 * kCandMax]
  int xctas;
  // 0: a scan kernel and its split variant are launched as a pair and exactly one works;
  // 1 (set on the copy passed to a launch): the kernel is the only one launched and works
  // whatever the queue length (the host chose it from the previous frame's queue lengths)
  int solo;
  // rt_set_scan_split: -1 = by queue length (split_parts); 1, 2, 4 or 8 = that many parts for
  // every scan (a test and tuning knob)
  int force_parts;
  // set per chunk on the copies passed to its launches: global sample index of the chunk's path 0
  // (the camera rays of depth 0 are implicit: entry e of Q[0] is path e, its ray computed on use)
  long long g0;    // the chunk's first path (w0 * spp)
  int w0;          // the chunk's first work item
};

// counter layout (zeroed per chunk): queue lengths and persistent-kernel work heads per depth
// point lights scanned from the light: at most 30, lane l of wf_shade's one-round-trip slot
// reservation takes light l's slots, lanes 30 / 31 the shadow entries / the continuations (more
// point lights: every shadow ray goes through the general scan)
constexpr int kMaxLtLights = 30;
constexpr int kLtSub = 8;         // sub-lists per light (slot reservations spread over 8 counters)
constexpr int kWfCtrPerDepth = 8 + kMaxLtLights * kLtSub + 32;
__host__ __device__ constexpr int wf_ctr_q(int d) { return kWfCtrPerDepth * d; }       // closest queue
__host__ __device__ constexpr int wf_ctr_s(int d) { return kWfCtrPerDepth * d + 1; }   // shadow entries
__host__ __device__ constexpr int wf_ctr_wc(int d) { return kWfCtrPerDepth * d + 2; }  // work heads
__host__ __device__ constexpr int wf_ctr_ws(int d) { return kWfCtrPerDepth * d + 3; }
__host__ __device__ constexpr int wf_ctr_so(int d) { return kWfCtrPerDepth * d + 4; }  // generic shadow slots
__host__ __device__ constexpr int wf_ctr_wlt(int d) { return kWfCtrPerDepth * d + 5; } // light-scan chunks
__host__ __device__ constexpr int wf_ctr_lt(int d, int l, int sub) {  // light l's sub-list `sub`
  return kWfCtrPerDepth * d + 8 + l * kLtSub + sub;
}
__host__ __device__ constexpr int wf_ctr_wltl(int d, int l) {  // light l's chunk head (wf_isect_lt)
  return kWfCtrPerDepth * d + 8 + kMaxLtLights * kLtSub + l;
}
constexpr int kPrevDiffuse = 0x100;  // flag in WfBuffers::depth (R#43)

// launchers (rt_kernels.cu)
cudaError_t upload_planes(const DevPlane* planes, int n_planes, cudaStream_t st);
cudaError_t upload_sample_offsets(int spp, cudaStream_t st);
cudaError_t launch_eye_table(const float4* pairs, const float4* sph_cr, int ns, int npp, const double o[3],
                             const double centre[3], double S, float4* out, cudaStream_t st);
cudaError_t launch_light_tables(const float4* pairs, const float4* sph_cr, const DevLight* lights, int ns, int npp,
                                int n_lights, const double centre[3], float cmax, float rmax, float4* out,
                                float4* out_per_light, cudaStream_t st);
cudaError_t launch_render(const DevParams& p, const DevScene& sc, const DevOutputs& o,
                          bool smem_scene, int num_sms, cudaStream_t st);
// buffer sizes of one chunk: cap paths, scap = cap x sources shadow entries, gcap generic
// shadow slots, lt_lists = lt_lights x kLtSub light-origin sub-lists
size_t wf_bytes(int cap, int scap, int gcap, int lt_lists, int xctas);
void wf_carve(WfBuffers& B, void* base, int cap, int scap, int gcap, int lt_lists, int xctas, unsigned* ctr);
// per-launch CUDA events around the intersection kernels (pairs: [2i] before, [2i+1] after)
struct WfTiming {
  cudaEvent_t* closest;
  cudaEvent_t* shadow;
  int cap;        // pairs available in each array
  int n;          // pairs recorded (output)
  int launches;   // kernels launched (output)
  cudaEvent_t* shade = nullptr;  // [2 * cap] events around each wf_shade launch
  cudaEvent_t* accum = nullptr;  // [2 * cap] events around each wf_accumulate launch
  // chunk pipelining: chunk i runs on slot i % nslots, each slot a buffer set with its own stream
  // pair, so one chunk's sparse deep depths overlap the next chunks' dense depth 0. Within a slot,
  // the shadow scan + accumulate of depth d run on the side stream, concurrently with the
  // closest-hit scan of depth d + 1 on the main stream (fork/join events per depth; side = null:
  // everything in order on the main stream). Slot 0's main stream is the caller's.
  static constexpr int kMaxSlots = 4;
  int nslots = 1;
  WfBuffers* slot_B[kMaxSlots] = {};
  cudaStream_t slot_main[kMaxSlots] = {}, slot_side[kMaxSlots] = {};
  cudaEvent_t* slot_fork[kMaxSlots] = {};  // [max_depth + 1] each
  cudaEvent_t* slot_join[kMaxSlots] = {};
  cudaEvent_t start_ev = nullptr;           // the other slots start after the caller's prior work
  cudaEvent_t slot_done[kMaxSlots] = {};    // the caller's stream resumes after every slot
  // optional: an event recorded after each chunk's resolve, and the work items resolved so far,
  // so the host can copy finished framebuffer rows while later chunks render
  // queue counters of the previous render with the same launch sequence, per buffer set (host
  // copies; null = unknown): each scan is then launched as one kernel, the long-queue scan or
  // its split variant, instead of the pair
  // (hints: host copy, hint_stride counters per chunk, of the chunks' counters saved in hint_dev
  // by the previous render with this sequence)
  const unsigned* hints = nullptr;
  unsigned* hint_dev = nullptr;
  size_t hint_stride = 0;
  int nslots_req = 1;  // the slot count the chunking was computed for (wf_chunk_count / _begin)
  cudaEvent_t* chunk_done = nullptr;
  int* chunk_items = nullptr;
  int chunk_cap = 0;
  int n_chunks = 0;  // output
  // while the launch sequence is captured into a CUDA graph, the timing and chunk events become
  // event-record nodes (cudaEventRecordExternal), so every replay records them
  bool ext_events = false;
  // schedule fuzzing (rt_set_schedule_jitter): state of the generator of the spin lengths, 0 = off
  unsigned long long jitter = 0;
  void record(cudaEvent_t ev, cudaStream_t s) const {
    cudaEventRecordWithFlags(ev, s, ext_events ? cudaEventRecordExternal : cudaEventRecordDefault);
  }
};
// scene source of the wavefront intersection kernels: 0 global, 1 shared memory
cudaError_t launch_render_wavefront(const DevParams& p, const DevScene& sc, const DevOutputs& o, int src,
                                    int num_sms, WfTiming& tm, cudaStream_t st);
// work items (pixels) per chunk of a frame rendered over nslots buffer-set slots
int wf_chunk_count(const DevParams& p, int nslots);
int wf_chunk_begin(const DevParams& p, int nslots, int k);
int wf_chunk_max_items(const DevParams& p, int nslots);
int wf_timing_pairs(const DevParams& p, int nslots);
cudaError_t launch_assemble(const float4* gathered, int W, int H, int world, int tiles_per_rank,
                            float4* out, unsigned long long* stats, cudaStream_t st);
cudaError_t launch_sum_records(const unsigned long long* rec, int world, unsigned long long* stats, cudaStream_t st);
cudaError_t read_check_status(unsigned* first_failed);
cudaError_t launch_tonemap(const float4* rgba, uint8_t* out, int64_t n, float exposure,
                           float gamma, cudaStream_t st);

}  // namespace rt

// host-side error reporting shared by the runtime translation units (rt_api.cu, rt_scene_io.cpp)
int rt_fail(int code, const char* msg);
void rt_clear_error();
