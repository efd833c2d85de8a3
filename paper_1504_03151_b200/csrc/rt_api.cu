// rt_api.cu — host runtime behind include/rt.h: validation, structure-of-arrays packing,
// device buffers, stream binding, launches, statistics and error reporting.
// Every computational step of the path runs in the kernels of rt_kernels.cu; this file only
// validates, packs and launches.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rt.h"
#include "rt_internal.h"

namespace {

thread_local std::string g_err;

// an NVTX range around each public call (named in ncu --nvtx / nsys timelines; no cost without
// a tool attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-free errors
  if (e == cudaErrorMemoryAllocation) return fail(RT_ERR_OOM, "%s: %s", what, cudaGetErrorString(e));
  return fail(RT_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace

// shared with rt_scene_io.cpp (declared in rt_internal.h)
int rt_fail(int code, const char* msg) {
  g_err = msg;
  return code;
}
void rt_clear_error() { g_err.clear(); }

namespace {

#define CU(call, what)                          \
  do {                                          \
    cudaError_t e_ = (call);                    \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

bool finite3(const float* v) { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); }

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaError_t reserve(size_t count) {
    if (count <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, sizeof(T) * (count ? count : 1));
    if (e == cudaSuccess) n = count;
    return e;
  }
};

// pinned host staging for the scene copies: from pinned memory an async copy is a plain DMA
// (from pageable memory every call first copies into a driver buffer); the next upload waits for
// the previous one's copies before it rewrites the buffer
struct PinnedStage {
  char* p = nullptr;
  size_t n = 0;
  cudaEvent_t done = nullptr;
  bool pending = false;
  cudaError_t reserve(size_t bytes) {
    if (pending) {
      cudaError_t e = cudaEventSynchronize(done);
      if (e != cudaSuccess) return e;
      pending = false;
    }
    if (!done) {
      cudaError_t e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    if (bytes <= n && p) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&p), bytes ? bytes : 1);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
};

struct Context {
  int device = -1;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  unsigned long long seed = 0;
  // scene
  bool has_scene = false;
  bool smem_scene = true;
  int n_spheres = 0, n_pairs_pad = 0, n_planes = 0, n_lights = 0, n_mats = 0;
  float cmax = 0.f, rmax = 0.f;
  double centre[3] = {0, 0, 0};
  float bg[3] = {0, 0, 0}, amb[3] = {0, 0, 0};
  DevBuf<float4> pairs, sph_cr, stage, pairs_eye, pairs_lt, pairs_ltl;
  PinnedStage upload;  // host staging of rt_scene_upload's copies
  int lt_lights = 0;  // point lights with light-origin shadow scans (0 = off)
  bool eye_ready = false;
  DevBuf<int> sph_prim, sph_mat, emit_sph;
  int n_emitters = 0;  // emissive spheres (prim order)
  // integrator settings (rt_set_integrator)
  int integrator = RT_INTEGRATOR_WHITTED, area_lights = 0;
  DevBuf<rt::DevMat> mats;
  DevBuf<rt::DevLight> lights;
  DevBuf<unsigned int> counter;
  DevBuf<unsigned long long> stats;
  DevBuf<int> dbg_hits, dbg_bounces;
  // wavefront variant
  int off_spp = 0;  // spp whose sub-pixel offsets are in the constant table (0: none)
  int variant = RT_VARIANT_AUTO;
  int concurrent = 1;  // shadow scans || next closest scan on a side stream (rt_set_concurrency)
  // chunk pipelining over buffer-set slots (rt_set_pipeline): chunk i on slot i % pipeline, each
  // slot with its own buffers, counters and stream pair (main, side: shadow scans || next closest
  // scan); slot 0's main stream is the library stream
  static constexpr int kSlots = rt::WfTiming::kMaxSlots;
  int pipeline = 0;  // 0: AUTO
  DevBuf<unsigned char> wf_mem[kSlots];
  DevBuf<unsigned> wf_ctr[kSlots];
  rt::WfBuffers wf[kSlots]{};
  cudaStream_t slot_main[kSlots] = {}, slot_side[kSlots] = {};
  std::vector<cudaEvent_t> ev_fork[kSlots], ev_join[kSlots];
  cudaEvent_t ev_start = nullptr, ev_done[kSlots] = {};
  std::vector<cudaEvent_t> ev_c, ev_s, ev_h, ev_a;  // per-launch scan / shade / accumulate timing
  int n_timed = 0, last_launches = 0, last_variant = 0, last_depth = 0;
  // camera (double basis)
  bool has_camera = false;
  double eye[3], f[3], r[3], u[3], h = 0;
  // last statistics
  rt_ray_stats last{};
  bool stats_pending = false, stats_timed = false;  // resolved lazily by rt_stats
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // host framebuffers: finished rows are copied on a second stream while later chunks render
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> ev_chunk;
  std::vector<int> chunk_items;
  // CUDA graph of the wavefront launch sequence (rt_set_graphs): captured on the second of two
  // consecutive renders with the same launch key, replayed while the key stays the same
  int graphs = 1;
  int scan_split = -1;  // rt_set_scan_split
  int tiled = 1;        // scenes beyond shared memory: TMA-tiled scans (1) or global loads (0; A/B)
  unsigned long long jitter = 0;  // rt_set_schedule_jitter: generator state (0 = off)
  cudaStream_t cap_stream = nullptr;  // capture happens here (the legacy stream cannot be captured)
  cudaEvent_t ev_cap = nullptr;
  // a few instantiated graphs, one per launch key (e.g. frames alternating between two output
  // buffers, as the multi-GPU double-buffered frame does), least recently used evicted; a key is
  // captured on its second plain render among the last kRecentKeys renders
  struct Graph {
    std::string key;
    cudaGraphExec_t exec = nullptr;
    int n = 0, launches = 0, chunks = 0;
    std::vector<int> chunk_items;
    unsigned long long used = 0;
  };
  std::vector<Graph> graph_cache;
  std::vector<std::string> recent_keys;
  unsigned long long graph_clock = 0;
  int last_graph = 0;  // how the last wavefront render was launched: 0 plain, 1 captured, 2 replayed
  std::vector<unsigned> hints;     // queue counters of every chunk of the render before a capture
  DevBuf<unsigned> hint_dev;        // where each render leaves its chunks' counters
};
constexpr size_t kGraphCache = 4, kRecentKeys = 8;

Context g_ctx;
// AUTO picks the wavefront kernels for scenes where the sphere scan dominates (measured on B200,
// C4 truncated to n spheres, round 2 kernels, ms per frame wavefront / megakernel: n = 32: 0.67 /
// 0.43; 64: 0.77 / 0.78; 128: 0.97 / 1.48; 1000: 6.23 / 14.2; C3 (100 spheres): 0.87 / 1.02)
constexpr int kAutoWavefrontSpheres = 64;

int ensure_device() {
  int dev = 0;
  CU(cudaGetDevice(&dev), "cudaGetDevice");
  if (g_ctx.device != dev) {
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
    if (prop.major < 10) return fail(RT_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a", dev, prop.major, prop.minor);
    g_ctx = Context();
    g_ctx.device = dev;
    g_ctx.num_sms = prop.multiProcessorCount;
    CU(cudaEventCreate(&g_ctx.ev0), "cudaEventCreate");
    CU(cudaEventCreate(&g_ctx.ev1), "cudaEventCreate");
    CU(g_ctx.counter.reserve(1), "cudaMalloc(counter)");
    CU(g_ctx.stats.reserve(8), "cudaMalloc(stats)");
  }
  return RT_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void norm3(double* v) {
  double l = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  v[0] /= l; v[1] /= l; v[2] /= l;
}

rt::DevParams make_params(int W, int H, int max_depth, int spp) {
  rt::DevParams p{};
  const Context& c = g_ctx;
  const double aspect = (double)W / (double)H;
  for (int i = 0; i < 3; ++i) {
    p.eye[i] = c.eye[i];
    p.F[i] = c.f[i];
    p.R[i] = c.r[i] * c.h * aspect;
    p.U[i] = c.u[i] * c.h;
    p.bg[i] = c.bg[i];
    p.amb[i] = c.amb[i];
  }
  p.cmax = c.cmax;
  p.rmax = c.rmax;
  for (int i = 0; i < 3; ++i) p.centre[i] = c.centre[i];
  p.W = W; p.H = H; p.max_depth = max_depth; p.spp = spp;
  p.n_spheres = c.n_spheres; p.n_pairs_pad = c.n_pairs_pad; p.n_planes = c.n_planes; p.n_lights = c.n_lights;
  p.seed = c.seed;
  p.integrator = c.integrator;
  // light lists need every source in the 64-bit light mask (point lights + sampled emitters <= 64)
  p.n_emitters = c.area_lights ? c.n_emitters : 0;
  p.lt_lights = (c.smem_scene && p.n_lights + p.n_emitters <= 64) ? c.lt_lights : 0;
  p.tiles_x = (W + rt::kTileW - 1) / rt::kTileW;
  p.n_tiles = p.tiles_x * ((H + rt::kTileH - 1) / rt::kTileH);
  p.div_spp = rt::make_fastdiv((unsigned)spp);
  p.div_tiles_x = rt::make_fastdiv((unsigned)p.tiles_x);
  p.inv_w = 1.0 / W;
  p.inv_h = 1.0 / H;
  return p;
}

// Shared-origin tables (rt_wavefront.cuh eye2_scan, lt_scan): built on the device from the
// uploaded pairs and spheres (rt_kernels.cu build_eye_table / build_light_tables: -h of the
// tangent test per sphere, FP64 rounded once). S = cmax + |o'| + rmax bounds the
// scene seen from o.
static double view_scale(const Context& c, const double o[3]) {
  const double x = o[0] - c.centre[0], y = o[1] - c.centre[1], z = o[2] - c.centre[2];
  return (double)c.cmax + std::sqrt(x * x + y * y + z * z) + (double)c.rmax;
}

// Camera rays share the origin `eye`. The table (wf_isect_eye2): the pair layout with -h of the
// eye in place of K, then s1 = K + 2 c'.o'(eye) per sphere (one float2 per pair) for the
// candidates' chord bounds.
int build_eye_pairs() {
  Context& c = g_ctx;
  c.eye_ready = false;
  if (!c.has_scene || !c.has_camera || c.n_pairs_pad == 0) return RT_OK;
  const int npp = c.n_pairs_pad;
  CU(c.pairs_eye.reserve(2 * (size_t)npp + (npp + 1) / 2), "cudaMalloc(eye pairs)");
  CU(rt::launch_eye_table(c.pairs.p, c.sph_cr.p, c.n_spheres, npp, c.eye, c.centre, view_scale(c, c.eye),
                          c.pairs_eye.p, c.stream), "eye table kernel");
  c.eye_ready = true;
  return RT_OK;
}

int check_frame(int32_t W, int32_t H, int32_t D, int32_t spp) {
  if (W < 1 || H < 1) return fail(RT_ERR_INVALID_ARG, "width/height must be >= 1 (got %d x %d)", W, H);
  if ((long long)W * H > 2147483647LL) return fail(RT_ERR_INVALID_ARG, "width*height exceeds 2^31-1");
  if (D < 0 || D > 64) return fail(RT_ERR_INVALID_ARG, "max_depth must be in [0, 64] (got %d)", D);
  if (spp < 1 || spp > 4096) return fail(RT_ERR_INVALID_ARG, "spp must be in [1, 4096] (got %d)", spp);
  if (!g_ctx.has_scene) return fail(RT_ERR_NO_SCENE, "no scene: call rt_scene_upload first");
  if (!g_ctx.has_camera) return fail(RT_ERR_NO_CAMERA, "no camera: call rt_camera_set first");
  return RT_OK;
}

// Everything the wavefront launch sequence depends on: the kernel arguments (parameters — the
// camera and the geometry's bounds included —, scene and output pointers, buffer layout), the
// scene source, the timing/stream configuration. The contents behind the scene pointers
// (materials, lights, sphere data of the same bounds) are read at run time and do not enter it.
template <class T>
void key_add(std::string& k, const T& v) {
  k.append(reinterpret_cast<const char*>(&v), sizeof(T));
}
std::string wf_launch_key(const rt::DevParams& p, const rt::DevScene& sc, const rt::DevOutputs& o, int src,
                          const rt::WfTiming& tm, const Context& c) {
  std::string k;
  key_add(k, p);
  key_add(k, sc);
  key_add(k, o);
  key_add(k, src);
  key_add(k, c.num_sms);
  key_add(k, c.wf);
  key_add(k, tm.nslots);
  key_add(k, tm.slot_B);
  key_add(k, tm.slot_main);
  key_add(k, tm.slot_side);
  key_add(k, tm.slot_fork);
  key_add(k, tm.slot_join);
  key_add(k, tm.slot_done);
  const void* ptrs[] = {tm.closest, tm.shadow, tm.shade, tm.accum, tm.start_ev, tm.chunk_done, tm.chunk_items};
  key_add(k, ptrs);
  key_add(k, tm.cap);
  key_add(k, tm.chunk_cap);
  return k;
}

void drop_graphs(Context& c) {
  for (auto& g : c.graph_cache)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  c.graph_cache.clear();
  c.recent_keys.clear();
}

// Launch the wavefront sequence: replay a cached graph when one matches the key, capture one when
// the key was launched plainly in one of the last kRecentKeys renders (a frame loop, or frames
// alternating between a few output buffers), else launch stream by stream (one-off renders,
// progressive passes whose pass index changes every call).
int launch_wavefront(Context& c, const rt::DevParams& p, const rt::DevScene& sc, const rt::DevOutputs& o, int src,
                     rt::WfTiming& tm) {
  c.last_graph = 0;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CU(cudaStreamIsCapturing(c.stream, &cs), "cudaStreamIsCapturing");
  if (!c.graphs || cs != cudaStreamCaptureStatusNone) {  // the caller captures: plain launches into it
    CU(rt::launch_render_wavefront(p, sc, o, src, c.num_sms, tm, c.stream), "wavefront launch");
    return RT_OK;
  }
  std::string key = wf_launch_key(p, sc, o, src, tm, c);
  for (auto& g : c.graph_cache) {
    if (g.key != key) continue;
    CU(cudaGraphLaunch(g.exec, c.stream), "cudaGraphLaunch");
    g.used = ++c.graph_clock;
    tm.n = g.n;
    tm.launches = g.launches;
    tm.n_chunks = g.chunks;
    if (tm.chunk_items) std::copy(g.chunk_items.begin(), g.chunk_items.end(), tm.chunk_items);
    c.last_graph = 2;
    return RT_OK;
  }
  if (std::find(c.recent_keys.begin(), c.recent_keys.end(), key) == c.recent_keys.end()) {
    // first render with this key (recently): plain launches
    CU(rt::launch_render_wavefront(p, sc, o, src, c.num_sms, tm, c.stream), "wavefront launch");
    c.recent_keys.push_back(key);
    if (c.recent_keys.size() > kRecentKeys) c.recent_keys.erase(c.recent_keys.begin());
    return RT_OK;
  }
  // second render with this key: capture on cap_stream (forked from c.stream so the capture sees
  // the same order), instantiate, launch on c.stream. The previous render left its queue lengths in
  // the counters of each buffer set: with them, each scan is captured as one kernel (long-queue scan
  // or split variant) instead of the self-selecting pair (a stale hint costs speed, never results).
  {
    const size_t nctr = (size_t)rt::kWfCtrPerDepth * (p.max_depth + 2);
    CU(cudaStreamSynchronize(c.stream), "cudaStreamSynchronize");
    (void)nctr;
    const size_t n = tm.hint_stride * (size_t)rt::wf_chunk_count(p, tm.nslots_req);
    c.hints.assign(n, 0u);
    CU(cudaMemcpy(c.hints.data(), c.hint_dev.p, n * sizeof(unsigned), cudaMemcpyDeviceToHost), "counters D2H");
    tm.hints = c.hints.data();
  }
  if (!c.cap_stream) CU(cudaStreamCreateWithFlags(&c.cap_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  // per-launch timing events become event-record nodes, which serialise the graph around every
  // scan and shade launch: kept for the in-order timing mode (rt_set_concurrency(0)), dropped
  // when the launches overlap (their per-launch times would share the GPU anyway)
  if (c.concurrent) tm.cap = 0;
  tm.ext_events = true;
  tm.jitter = 0;  // a captured graph keeps no spins
  CU(cudaStreamBeginCapture(c.cap_stream, cudaStreamCaptureModeRelaxed), "cudaStreamBeginCapture");
  const cudaError_t le = rt::launch_render_wavefront(p, sc, o, src, c.num_sms, tm, c.cap_stream);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(c.cap_stream, &g);
  tm.ext_events = false;
  CU(le, "wavefront launch (capture)");
  CU(ce, "cudaStreamEndCapture");
  cudaGraphExec_t x = nullptr;
  // (the side stream's priority carries over into the replays)
  const cudaError_t ie = cudaGraphInstantiate(&x, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  CU(ie, "cudaGraphInstantiate");
  if (c.graph_cache.size() >= kGraphCache) {  // evict the least recently used graph
    auto lru = std::min_element(c.graph_cache.begin(), c.graph_cache.end(),
                                [](const Context::Graph& a, const Context::Graph& b) { return a.used < b.used; });
    cudaGraphExecDestroy(lru->exec);
    c.graph_cache.erase(lru);
  }
  Context::Graph e;
  e.key = key;
  e.exec = x;
  e.n = tm.n;
  e.launches = tm.launches;
  e.chunks = tm.n_chunks;
  if (tm.chunk_items) e.chunk_items.assign(tm.chunk_items, tm.chunk_items + tm.n_chunks);
  e.used = ++c.graph_clock;
  c.graph_cache.push_back(std::move(e));
  CU(cudaGraphLaunch(x, c.stream), "cudaGraphLaunch");
  c.last_graph = 1;
  return RT_OK;
}

constexpr int kHostMinChunks = 4;
// host_out (optional): the caller's host framebuffer for a mode-0 render into the staging buffer
// `out`; the wavefront variant then copies each chunk's finished rows as soon as it resolves
// (RT_OK with *copied = true), else the caller copies the whole frame after the render
int run_render(const rt::DevParams& p, float4* out, int* dbg_hits, int* dbg_bounces, double* accum = nullptr,
               float* host_out = nullptr, bool* copied = nullptr) {
  if (copied) *copied = false;
  Context& c = g_ctx;
  if (c.off_spp != p.spp) {  // stream-ordered before this render's launches (or graph replay)
    CU(rt::upload_sample_offsets(p.spp, c.stream), "constant upload (sample offsets)");
    c.off_spp = p.spp;
  }
  CU(cudaMemsetAsync(c.counter.p, 0, sizeof(unsigned), c.stream), "cudaMemsetAsync");
  CU(cudaMemsetAsync(c.stats.p, 0, sizeof(unsigned long long) * 8, c.stream), "cudaMemsetAsync");
  rt::DevScene sc{c.pairs.p, c.sph_cr.p, c.sph_prim.p, c.sph_mat.p, c.mats.p, c.lights.p, c.emit_sph.p,
                  c.eye_ready ? c.pairs_eye.p : nullptr, c.lt_lights > 0 ? c.pairs_lt.p : nullptr,
                  c.lt_lights > 0 ? c.pairs_ltl.p : nullptr};
  rt::DevOutputs o{out, c.counter.p, c.stats.p, dbg_hits, dbg_bounces, accum};
  // AUTO: the wavefront kernels for large scenes, and for the NEXT-1 / NEXT-2 modes, whose long
  // divergent paths (every diffuse hit continues; one lane per pixel walks all its passes) leave
  // the megakernel's lanes idle (C0 progressive, 16 passes: 9.7 ms wavefront, 15.2 ms megakernel)
  const bool extended = p.integrator != 0 || p.n_emitters > 0 || p.jitter != 0 || accum != nullptr;
  const bool wavefront = c.variant == RT_VARIANT_WAVEFRONT ||
                         (c.variant == RT_VARIANT_AUTO && (extended || c.n_spheres >= kAutoWavefrontSpheres));
  if (wavefront) {
    // chunks of whole pixels, at most 2^22 paths each; a frame that fills fewer chunks than
    // pipeline slots (or than p.min_chunks, host framebuffers) is cut into that many
    // AUTO (0): two slots, three for frames of >= 8 chunks (C5: 227.4 -> 225.3 ms per frame;
    // C4's two chunks: 2 slots 5.83, 3 slots 5.89 ms)
    const int nslots = !c.concurrent ? 1 : c.pipeline > 0 ? c.pipeline : (rt::wf_chunk_count(p, 2) >= 8 ? 3 : 2);
    const int cap = rt::wf_chunk_max_items(p, nslots) * p.spp;
    const int n_src = p.n_lights + p.n_emitters;  // shadow rays per shading point <= n_src
    const int scap = cap * (n_src > 0 ? n_src : 1);
    // point lights with light-origin scans get list slots; every other source a generic slot
    const int n_gen = n_src - p.lt_lights;
    const int gcap = cap * (n_gen > 0 ? n_gen : 1);
    const int lt_lists = p.lt_lights * rt::kLtSub;
    const int n_chunks = rt::wf_chunk_count(p, nslots);
    const int used = n_chunks < nslots ? n_chunks : nslots;  // slots that receive a chunk
    rt::WfTiming tm{nullptr, nullptr, 0, 0, 0};
    tm.nslots = used;
    for (int k = 0; k < used; ++k) {  // (re)carve each slot's buffers for this frame's chunk size
      CU(c.wf_mem[k].reserve(rt::wf_bytes(cap, scap, gcap, lt_lists, 4 * c.num_sms)), "cudaMalloc(wavefront)");
      CU(c.wf_ctr[k].reserve(rt::kWfCtrPerDepth * 80), "cudaMalloc(wavefront counters)");
      rt::wf_carve(c.wf[k], c.wf_mem[k].p, cap, scap, gcap, lt_lists, 4 * c.num_sms, c.wf_ctr[k].p);
      c.wf[k].force_parts = c.scan_split;
      tm.slot_B[k] = &c.wf[k];
      if (k > 0 && !c.slot_main[k]) CU(cudaStreamCreateWithFlags(&c.slot_main[k], cudaStreamNonBlocking), "cudaStreamCreate");
      if (!c.slot_side[k]) {  // the side stream (shadow scan + accumulate of depth d) at the highest
        // priority: it is the longer branch before the join (C4 5.522 -> 5.477 ms, C5 215.9 -> 214.6)
        int lo = 0, hi = 0;
        CU(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
        CU(cudaStreamCreateWithPriority(&c.slot_side[k], cudaStreamNonBlocking, hi), "cudaStreamCreate");
      }
      if (k > 0 && !c.ev_done[k]) CU(cudaEventCreateWithFlags(&c.ev_done[k], cudaEventDisableTiming), "cudaEventCreate");
      while ((int)c.ev_fork[k].size() < p.max_depth + 1) {
        cudaEvent_t f, j;
        CU(cudaEventCreateWithFlags(&f, cudaEventDisableTiming), "cudaEventCreate");
        CU(cudaEventCreateWithFlags(&j, cudaEventDisableTiming), "cudaEventCreate");
        c.ev_fork[k].push_back(f);
        c.ev_join[k].push_back(j);
      }
      tm.slot_main[k] = c.slot_main[k];
      tm.slot_done[k] = c.ev_done[k];
      if (c.concurrent) {
        tm.slot_side[k] = c.slot_side[k];
        tm.slot_fork[k] = c.ev_fork[k].data();
        tm.slot_join[k] = c.ev_join[k].data();
      }
    }
    if (used > 1 && !c.ev_start) CU(cudaEventCreateWithFlags(&c.ev_start, cudaEventDisableTiming), "cudaEventCreate");
    tm.start_ev = c.ev_start;
    const int pairs = rt::wf_timing_pairs(p, nslots);
    while ((int)c.ev_c.size() < 2 * pairs) {
      cudaEvent_t a, b, h, m;
      CU(cudaEventCreate(&a), "cudaEventCreate");
      CU(cudaEventCreate(&b), "cudaEventCreate");
      CU(cudaEventCreate(&h), "cudaEventCreate");
      CU(cudaEventCreate(&m), "cudaEventCreate");
      c.ev_c.push_back(a);
      c.ev_s.push_back(b);
      c.ev_h.push_back(h);
      c.ev_a.push_back(m);
    }
    tm.closest = c.ev_c.data();
    tm.shadow = c.ev_s.data();
    tm.cap = pairs;
    tm.shade = c.ev_h.data();
    tm.accum = c.ev_a.data();
    tm.jitter = c.jitter;
    tm.nslots_req = nslots;
    tm.hint_stride = (size_t)rt::kWfCtrPerDepth * (p.max_depth + 2);
    CU(c.hint_dev.reserve(tm.hint_stride * n_chunks), "cudaMalloc(hints)");
    tm.hint_dev = c.hint_dev.p;
    const bool overlap = host_out != nullptr && p.mode == 0;
    if (overlap) {
      const int max_chunks = n_chunks;
      if (!c.copy_stream) CU(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
      while ((int)c.ev_chunk.size() < max_chunks) {
        cudaEvent_t ev;
        CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
        c.ev_chunk.push_back(ev);
      }
      c.chunk_items.assign(max_chunks, 0);
      tm.chunk_done = c.ev_chunk.data();
      tm.chunk_items = c.chunk_items.data();
      tm.chunk_cap = max_chunks;
    }
    CU(cudaEventRecord(c.ev0, c.stream), "cudaEventRecord");
    // the scans' scene source: staged whole in shared memory, else streamed in TMA tiles
    const int src = c.smem_scene ? 1 : (c.tiled ? 2 : 0);
    {
      const int lrc = launch_wavefront(c, p, sc, o, src, tm);
      if (lrc) return lrc;
    }
    CU(cudaEventRecord(c.ev1, c.stream), "cudaEventRecord");
    if (overlap) {  // rows of complete tile rows, in order, each after its chunk's resolve
      const long long row_items = (long long)p.tiles_x * rt::kTilePx;
      int rows_done = 0;
      for (int k = 0; k < tm.n_chunks; ++k) {
        long long rows = (long long)(tm.chunk_items[k] / row_items) * rt::kTileH;
        if (k == tm.n_chunks - 1 || rows > p.H) rows = p.H;
        if (rows <= rows_done) continue;
        CU(cudaStreamWaitEvent(c.copy_stream, c.ev_chunk[k], 0), "cudaStreamWaitEvent");
        CU(cudaMemcpyAsync(host_out + (size_t)rows_done * p.W * 4, out + (size_t)rows_done * p.W,
                           sizeof(float4) * (size_t)(rows - rows_done) * p.W, cudaMemcpyDeviceToHost, c.copy_stream),
           "framebuffer D2H");
        rows_done = (int)rows;
      }
      if (copied) *copied = rows_done == p.H;
    }
    c.n_timed = tm.n;
    c.last_depth = p.max_depth;
    c.last_launches = tm.launches;
    c.last_variant = RT_VARIANT_WAVEFRONT;
    return RT_OK;
  }
  CU(cudaEventRecord(c.ev0, c.stream), "cudaEventRecord");
  CU(rt::launch_render(p, sc, o, c.smem_scene, c.num_sms, c.stream), "render kernel launch");
  CU(cudaEventRecord(c.ev1, c.stream), "cudaEventRecord");
  c.n_timed = 0;
  c.last_launches = 1;
  c.last_variant = RT_VARIANT_MEGAKERNEL;
  return RT_OK;
}

// Statistics stay on the device until rt_stats (or a host-output render) needs them, so a
// render into a device buffer is fully asynchronous on the library stream.
void defer_stats(bool timed) {
  g_ctx.stats_pending = true;
  g_ctx.stats_timed = timed;
}

int collect_stats(bool timed) {
  Context& c = g_ctx;
  c.stats_pending = false;
  unsigned long long h[8];
  CU(cudaMemcpyAsync(h, c.stats.p, sizeof h, cudaMemcpyDeviceToHost, c.stream), "stats D2H");
  CU(cudaStreamSynchronize(c.stream), "cudaStreamSynchronize");
  float ms = 0.f;
  if (timed) CU(cudaEventElapsedTime(&ms, c.ev0, c.ev1), "cudaEventElapsedTime");
  c.last.primary = h[0];
  c.last.shadow = h[1];
  c.last.secondary = h[2];
  c.last.sphere_tests = h[3];
  c.last.plane_tests = h[4];
  c.last.closest_sphere_tests = h[5];
  c.last.last_render_ms = ms;
  double tc = 0.0, ts = 0.0, tsh = 0.0, te = 0.0, tac = 0.0;
  if (timed) {
    for (int i = 0; i < c.n_timed; ++i) {
      float a = 0.f, b = 0.f, m = 0.f, ac = 0.f;
      CU(cudaEventElapsedTime(&a, c.ev_c[2 * i], c.ev_c[2 * i + 1]), "cudaEventElapsedTime");
      CU(cudaEventElapsedTime(&b, c.ev_s[2 * i], c.ev_s[2 * i + 1]), "cudaEventElapsedTime");
      CU(cudaEventElapsedTime(&m, c.ev_h[2 * i], c.ev_h[2 * i + 1]), "cudaEventElapsedTime");
      CU(cudaEventElapsedTime(&ac, c.ev_a[2 * i], c.ev_a[2 * i + 1]), "cudaEventElapsedTime");
      tc += a;
      ts += b;
      tsh += m;
      tac += ac;
      if (i % (c.last_depth + 1) == 0) te += a;  // depth 0: the camera-ray scan
    }
  }
  c.last.isect_closest_ms = tc;
  c.last.isect_shadow_ms = ts;
  c.last.shade_ms = tsh;
  c.last.isect_eye_ms = te;
  c.last.accumulate_ms = tac;
  c.last.launches = timed ? (uint32_t)c.last_launches : 2u;
  c.last.variant = c.last_variant;
  c.last.graph = c.last_variant == RT_VARIANT_WAVEFRONT ? c.last_graph : 0;
  return RT_OK;
}

int render_common(int32_t W, int32_t H, int32_t D, int32_t spp, float* out_rgba, int32_t* hit_ids,
                  int32_t* bounces, double* accum = nullptr, long long sample_base = 0) {
  int rc = ensure_device();
  if (rc) return rc;
  if (!out_rgba && !accum) return fail(RT_ERR_INVALID_ARG, "out_rgba is NULL");
  rc = check_frame(W, H, D, spp);
  if (rc) return rc;
  Context& c = g_ctx;
  const long long npx = (long long)W * H;
  if (accum) {
    if (!is_device_ptr(accum)) return fail(RT_ERR_INVALID_ARG, "accum_rgb must be a device pointer");
    if ((reinterpret_cast<uintptr_t>(accum) & 7u) != 0) return fail(RT_ERR_INVALID_ARG, "accum_rgb must be 8-byte aligned");
    if (sample_base < 0 || sample_base + spp > 4294967296LL)
      return fail(RT_ERR_INVALID_ARG, "passes: need 0 <= pass_begin and pass_begin + n_passes <= 2^32");
  }
  if (!out_rgba) {  // accumulation only: resolve writes no framebuffer
    rt::DevParams p = make_params(W, H, D, spp);
    p.mode = 0;
    p.n_items = p.n_tiles * rt::kTilePx;
    p.jitter = 1;
    p.sample_base = sample_base;
    rc = run_render(p, nullptr, nullptr, nullptr, accum);
    if (rc) return rc;
    defer_stats(true);
    return RT_OK;
  }
  const bool dev_out = is_device_ptr(out_rgba);
  if (dev_out && (reinterpret_cast<uintptr_t>(out_rgba) & 15u) != 0)
    return fail(RT_ERR_INVALID_ARG, "device out_rgba must be 16-byte aligned");
  float4* out = reinterpret_cast<float4*>(out_rgba);
  if (!dev_out) {
    CU(c.stage.reserve(npx), "cudaMalloc(staging)");
    out = c.stage.p;
  }
  const bool dbg = hit_ids != nullptr;
  int* dh = nullptr;
  int* db = nullptr;
  const long long nsamp = npx * spp;
  bool dev_dbg = false;
  if (dbg) {
    if (!bounces) return fail(RT_ERR_INVALID_ARG, "bounces is NULL");
    dev_dbg = is_device_ptr(hit_ids) && is_device_ptr(bounces);
    if (dev_dbg) {
      dh = hit_ids;
      db = bounces;
    } else {
      CU(c.dbg_hits.reserve(nsamp * (D + 1)), "cudaMalloc(debug)");
      CU(c.dbg_bounces.reserve(nsamp), "cudaMalloc(debug)");
      dh = c.dbg_hits.p;
      db = c.dbg_bounces.p;
    }
  }
  rt::DevParams p = make_params(W, H, D, spp);
  p.mode = 0;
  p.n_items = p.n_tiles * rt::kTilePx;
  // a host framebuffer: at least kHostMinChunks chunks of falling size (rt_kernels.cu
  // wf_chunk_begin), so the first chunks' rows are copied while the last ones render (two equal
  // chunks start and finish together, and the whole 33 MB D2H of a C4 frame came after the
  // render: rt_render into pinned memory 6.51 ms -> 6.40 with 4 equal chunks, 6.17 falling)
  if (!dev_out && !dbg && !accum) p.min_chunks = kHostMinChunks;
  if (accum) {  // progressive passes (R#42)
    p.jitter = 1;
    p.sample_base = sample_base;
  }
  bool copied = false;
  rc = run_render(p, out, dh, db, accum, (!dev_out && !dbg && !accum) ? out_rgba : nullptr, &copied);
  if (rc) return rc;
  if (!dev_out && !copied)
    CU(cudaMemcpyAsync(out_rgba, out, sizeof(float4) * npx, cudaMemcpyDeviceToHost, c.stream), "framebuffer D2H");
  if (copied) CU(cudaStreamSynchronize(c.copy_stream), "cudaStreamSynchronize(copy)");
  if (dbg && !dev_dbg) {
    CU(cudaMemcpyAsync(hit_ids, dh, sizeof(int) * nsamp * (D + 1), cudaMemcpyDeviceToHost, c.stream), "debug D2H");
    CU(cudaMemcpyAsync(bounces, db, sizeof(int) * nsamp, cudaMemcpyDeviceToHost, c.stream), "debug D2H");
  }
  if (!dev_out || (dbg && !dev_dbg)) return collect_stats(true);  // host outputs: complete on return
  defer_stats(true);
  return RT_OK;
}

}  // namespace

extern "C" {

const char* rt_last_error(void) { return g_err.c_str(); }

int rt_set_stream(void* cuda_stream) {
  int rc = ensure_device();
  if (rc) return rc;
  g_ctx.stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  return RT_OK;
}

int rt_set_variant(int32_t variant) {
  int rc = ensure_device();
  if (rc) return rc;
  if (variant != RT_VARIANT_MEGAKERNEL && variant != RT_VARIANT_WAVEFRONT && variant != RT_VARIANT_AUTO)
    return fail(RT_ERR_INVALID_ARG, "variant %d not in {-1 auto, 0 megakernel, 1 wavefront}", variant);
  g_ctx.variant = variant;
  return RT_OK;
}

int rt_set_integrator(int32_t integrator, int32_t area_lights) {
  int rc = ensure_device();
  if (rc) return rc;
  if (integrator != RT_INTEGRATOR_WHITTED && integrator != RT_INTEGRATOR_GLOBAL)
    return fail(RT_ERR_INVALID_ARG, "integrator %d not in {0 whitted, 1 global}", integrator);
  if (area_lights != 0 && area_lights != 1) return fail(RT_ERR_INVALID_ARG, "area_lights must be 0 or 1");
  g_ctx.integrator = integrator;
  g_ctx.area_lights = area_lights;
  return RT_OK;
}

int rt_render_passes(int32_t width, int32_t height, int32_t max_depth, int64_t pass_begin, int32_t n_passes,
                     double* accum_rgb, float* out_rgba) {
  NvtxRange nvtx_range("rt_render_passes");
  g_err.clear();
  if (!accum_rgb) return fail(RT_ERR_INVALID_ARG, "accum_rgb is NULL");
  return render_common(width, height, max_depth, n_passes, out_rgba, nullptr, nullptr, accum_rgb, pass_begin);
}

int rt_render_passes_debug(int32_t width, int32_t height, int32_t max_depth, int64_t pass_begin, int32_t n_passes,
                           double* accum_rgb, float* out_rgba, int32_t* hit_ids, int32_t* bounces) {
  NvtxRange nvtx_range("rt_render_passes_debug");
  g_err.clear();
  if (!accum_rgb) return fail(RT_ERR_INVALID_ARG, "accum_rgb is NULL");
  if (!out_rgba || !hit_ids || !bounces) return fail(RT_ERR_INVALID_ARG, "out_rgba/hit_ids/bounces must not be NULL");
  return render_common(width, height, max_depth, n_passes, out_rgba, hit_ids, bounces, accum_rgb, pass_begin);
}

int rt_set_concurrency(int32_t on) {
  int rc = ensure_device();
  if (rc) return rc;
  if (on != 0 && on != 1) return fail(RT_ERR_INVALID_ARG, "concurrency must be 0 or 1");
  g_ctx.concurrent = on;
  return RT_OK;
}

int rt_set_pipeline(int32_t slots) {
  int rc = ensure_device();
  if (rc) return rc;
  if (slots < 0 || slots > Context::kSlots) return fail(RT_ERR_INVALID_ARG, "pipeline slots must be in [0, %d]", Context::kSlots);
  g_ctx.pipeline = slots;
  return RT_OK;
}

int rt_set_schedule_jitter(uint64_t seed) {
  int rc = ensure_device();
  if (rc) return rc;
  g_ctx.jitter = seed;
  return RT_OK;
}

int rt_check_status(uint32_t* first_failed, int32_t* compiled) {
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (!first_failed || !compiled) return fail(RT_ERR_INVALID_ARG, "check_status: NULL argument");
  CU(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  unsigned v = 0;
  CU(rt::read_check_status(&v), "read check status");
  *first_failed = v;
  *compiled = RT_CHECKS;
  return RT_OK;
}

int rt_set_tiled_scan(int32_t on) {
  int rc = ensure_device();
  if (rc) return rc;
  if (on != 0 && on != 1) return fail(RT_ERR_INVALID_ARG, "tiled scan must be 0 or 1");
  g_ctx.tiled = on;
  return RT_OK;
}

int rt_set_scan_split(int32_t parts) {
  int rc = ensure_device();
  if (rc) return rc;
  if (parts != -1 && parts != 1 && parts != 2 && parts != 4 && parts != 8)
    return fail(RT_ERR_INVALID_ARG, "scan split must be -1, 1, 2, 4 or 8 (got %d)", parts);
  g_ctx.scan_split = parts;
  return RT_OK;
}

int rt_set_graphs(int32_t on) {
  int rc = ensure_device();
  if (rc) return rc;
  if (on != 0 && on != 1) return fail(RT_ERR_INVALID_ARG, "graphs must be 0 or 1");
  g_ctx.graphs = on;
  drop_graphs(g_ctx);
  return RT_OK;
}

int rt_set_seed(uint64_t seed) {
  int rc = ensure_device();
  if (rc) return rc;
  g_ctx.seed = seed;
  return RT_OK;
}

int rt_scene_upload(const rt_primitive* prims, int32_t n_prims, const rt_material* mats, int32_t n_mats,
                    const rt_light* lights, int32_t n_lights, const rt_env* env) {
  NvtxRange nvtx_range("rt_scene_upload");
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (n_prims < 0 || (n_prims > 0 && !prims)) return fail(RT_ERR_INVALID_ARG, "prims: NULL or n_prims < 0");
  if (n_mats < 1 || !mats) return fail(RT_ERR_INVALID_ARG, "mats: need n_mats >= 1");
  if (n_lights < 0 || n_lights > RT_MAX_LIGHTS || (n_lights > 0 && !lights))
    return fail(RT_ERR_INVALID_ARG, "lights: need 0 <= n_lights <= %d", (int)RT_MAX_LIGHTS);
  // validate materials
  for (int i = 0; i < n_mats; ++i) {
    const rt_material& m = mats[i];
    if (m.kind > 2) return fail(RT_ERR_INVALID_ARG, "material %d: kind %u not in {0,1,2}", i, m.kind);
    for (int k = 0; k < 3; ++k) {
      if (!(m.albedo[k] >= 0.f && m.albedo[k] <= 1.f)) return fail(RT_ERR_INVALID_ARG, "material %d: albedo outside [0,1]", i);
      if (!(m.emission[k] >= 0.f) || !std::isfinite(m.emission[k])) return fail(RT_ERR_INVALID_ARG, "material %d: emission must be finite and >= 0", i);
    }
    if (m.kind == RT_MAT_REFRACTIVE && !(m.ior >= 1.f && std::isfinite(m.ior))) return fail(RT_ERR_INVALID_ARG, "material %d: ior must be >= 1", i);
    if (!(m.ks >= 0.f && m.ks <= 1.f)) return fail(RT_ERR_INVALID_ARG, "material %d: ks outside [0,1]", i);
    if (!(m.shininess >= 1.f && m.shininess <= 1e4f)) return fail(RT_ERR_INVALID_ARG, "material %d: shininess outside [1,1e4]", i);
    if (!(m.kr >= 0.f && m.kr <= 1.f)) return fail(RT_ERR_INVALID_ARG, "material %d: kr outside [0,1]", i);
  }
  int ns = 0, np = 0;
  for (int i = 0; i < n_prims; ++i) {
    const rt_primitive& q = prims[i];
    if (q.material >= (uint32_t)n_mats) return fail(RT_ERR_INVALID_ARG, "prim %d: material %u >= n_mats %d", i, q.material, n_mats);
    for (int k = 0; k < 4; ++k)
      if (!std::isfinite(q.p[k])) return fail(RT_ERR_INVALID_ARG, "prim %d: non-finite parameter", i);
    if (q.type == RT_PRIM_SPHERE) {
      if (!(q.p[3] > 0.f)) return fail(RT_ERR_INVALID_ARG, "prim %d: radius <= 0", i);
      ++ns;
    } else if (q.type == RT_PRIM_PLANE) {
      if (q.p[0] == 0.f && q.p[1] == 0.f && q.p[2] == 0.f) return fail(RT_ERR_INVALID_ARG, "prim %d: plane normal is zero", i);
      ++np;
    } else {
      return fail(RT_ERR_INVALID_ARG, "prim %d: type %u not in {0 sphere, 1 plane}", i, q.type);
    }
  }
  if (np > RT_MAX_PLANES) return fail(RT_ERR_INVALID_ARG, "too many planes (%d > %d)", np, (int)RT_MAX_PLANES);
  if (ns > RT_MAX_SPHERES) return fail(RT_ERR_INVALID_ARG, "too many spheres (%d > %d)", ns, (int)RT_MAX_SPHERES);
  for (int i = 0; i < n_lights; ++i) {
    if (!finite3(lights[i].position)) return fail(RT_ERR_INVALID_ARG, "light %d: non-finite position", i);
    for (int k = 0; k < 3; ++k)
      if (!(lights[i].intensity[k] >= 0.f) || !std::isfinite(lights[i].intensity[k])) return fail(RT_ERR_INVALID_ARG, "light %d: intensity must be finite and >= 0", i);
  }
  if (env) {
    for (int k = 0; k < 3; ++k)
      if (!(env->background[k] >= 0.f && std::isfinite(env->background[k])) || !(env->ambient[k] >= 0.f && std::isfinite(env->ambient[k])))
        return fail(RT_ERR_INVALID_ARG, "env: background/ambient must be finite and >= 0");
  }

  // pack: spheres in index order into AoSoA pairs; planes in index order
  const int npairs = (ns + 1) / 2;
  const int npairs_pad = ((npairs + rt::kPairsPerBatch - 1) / rt::kPairsPerBatch) * rt::kPairsPerBatch;
  std::vector<float4> pairs(2 * (size_t)npairs_pad);
  // filter frame: centre of the spheres' bounding box (expanded form works in c' = c - centre)
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int i = 0; i < n_prims; ++i)
    if (prims[i].type == RT_PRIM_SPHERE)
      for (int k = 0; k < 3; ++k) {
        lo[k] = std::fmin(lo[k], (double)prims[i].p[k]);
        hi[k] = std::fmax(hi[k], (double)prims[i].p[k]);
      }
  double centre[3] = {0, 0, 0};
  if (ns > 0)
    for (int k = 0; k < 3; ++k) centre[k] = (double)(float)(0.5 * (lo[k] + hi[k]));
  for (int q = 0; q < npairs_pad; ++q) {  // dummies never pass the filter
    pairs[2 * q] = make_float4(0.f, 0.f, 0.f, 0.f);
    pairs[2 * q + 1] = make_float4(0.f, 0.f, -1e30f, -1e30f);
  }
  std::vector<float4> cr(ns > 0 ? ns : 1);
  std::vector<int> sprim(ns > 0 ? ns : 1), smat(ns > 0 ? ns : 1);
  std::vector<rt::DevPlane> planes(np > 0 ? np : 1);
  int ks = 0, kp = 0;
  double cmax = 0.0, rmax = 0.0;
  for (int i = 0; i < n_prims; ++i) {
    const rt_primitive& q = prims[i];
    if (q.type == RT_PRIM_SPHERE) {
      if (q.p[3] > rmax) rmax = q.p[3];
      // c' = c - centre (float), K = r^2 - |c'|^2 (double, rounded once)
      const float f0 = (float)((double)q.p[0] - centre[0]);
      const float f1 = (float)((double)q.p[1] - centre[1]);
      const float f2 = (float)((double)q.p[2] - centre[2]);
      const double r = q.p[3];
      const float f3 = (float)(r * r - ((double)f0 * f0 + (double)f1 * f1 + (double)f2 * f2));
      const double cn = std::sqrt((double)f0 * f0 + (double)f1 * f1 + (double)f2 * f2);
      if (cn > cmax) cmax = cn;
      float* A = reinterpret_cast<float*>(&pairs[2 * (ks / 2)]);
      float* B = reinterpret_cast<float*>(&pairs[2 * (ks / 2) + 1]);
      const int h = ks & 1;
      A[0 + h] = f0; A[2 + h] = f1; B[0 + h] = f2; B[2 + h] = f3;
      cr[ks] = make_float4(q.p[0], q.p[1], q.p[2], q.p[3]);
      sprim[ks] = i;
      smat[ks] = (int)q.material;
      ++ks;
    } else {
      double n[3] = {q.p[0], q.p[1], q.p[2]};
      const double l = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
      rt::DevPlane pl{};
      pl.nx = n[0] / l; pl.ny = n[1] / l; pl.nz = n[2] / l;
      pl.d = (double)q.p[3] / l;
      pl.prim = i;
      pl.mat = (int)q.material;
      planes[kp++] = pl;
    }
  }
  // emitters (R#41): spheres whose material emits in some channel, in prim (= sphere) order
  std::vector<int> emit;
  for (int k = 0; k < ns; ++k) {
    const rt_material& m = mats[smat[k]];
    if (m.emission[0] > 0.f || m.emission[1] > 0.f || m.emission[2] > 0.f) emit.push_back(k);
  }
  if (emit.size() > (size_t)RT_MAX_EMITTERS)
    return fail(RT_ERR_INVALID_ARG, "too many emissive spheres (%d > %d)", (int)emit.size(), (int)RT_MAX_EMITTERS);
  std::vector<rt::DevMat> dm(n_mats);
  for (int i = 0; i < n_mats; ++i) {
    const rt_material& m = mats[i];
    dm[i] = rt::DevMat{m.albedo[0], m.albedo[1], m.albedo[2], m.emission[0], m.emission[1], m.emission[2],
                       m.ior, m.ks, m.shininess, m.kr, (int)m.kind, 0.f};
  }
  std::vector<rt::DevLight> dl(n_lights > 0 ? n_lights : 1);
  for (int i = 0; i < n_lights; ++i) {
    const rt_light& L = lights[i];
    dl[i] = rt::DevLight{L.position[0], L.position[1], L.position[2], L.intensity[0], L.intensity[1], L.intensity[2], 0.f, 0.f};
  }

  Context& c = g_ctx;
  CU(c.pairs.reserve(pairs.size()), "cudaMalloc(pairs)");
  CU(c.sph_cr.reserve(cr.size()), "cudaMalloc(spheres)");
  CU(c.sph_prim.reserve(sprim.size()), "cudaMalloc(spheres)");
  CU(c.sph_mat.reserve(smat.size()), "cudaMalloc(spheres)");
  CU(c.mats.reserve(dm.size()), "cudaMalloc(materials)");
  CU(c.lights.reserve(dl.size()), "cudaMalloc(lights)");
  CU(c.emit_sph.reserve(emit.size() > 0 ? emit.size() : 1), "cudaMalloc(emitters)");
  {  // every array through the pinned staging buffer, then async copies (no stream sync: the
     // tables below are built on the device from these copies)
    struct Part { void* dst; const void* src; size_t bytes; };
    const Part parts[] = {{c.pairs.p, pairs.data(), sizeof(float4) * pairs.size()},
                          {c.sph_cr.p, cr.data(), sizeof(float4) * cr.size()},
                          {c.sph_prim.p, sprim.data(), sizeof(int) * sprim.size()},
                          {c.sph_mat.p, smat.data(), sizeof(int) * smat.size()},
                          {c.mats.p, dm.data(), sizeof(rt::DevMat) * dm.size()},
                          {c.lights.p, dl.data(), sizeof(rt::DevLight) * dl.size()},
                          {c.emit_sph.p, emit.data(), sizeof(int) * emit.size()},
                          {nullptr, planes.data(), sizeof(rt::DevPlane) * (size_t)np}};
    size_t total = 0;
    for (const Part& q : parts) total += (q.bytes + 255) & ~size_t(255);
    CU(c.upload.reserve(total), "cudaMallocHost(upload staging)");
    size_t off = 0;
    for (const Part& q : parts) {
      if (q.bytes == 0) continue;
      std::memcpy(c.upload.p + off, q.src, q.bytes);
      if (q.dst) CU(cudaMemcpyAsync(q.dst, c.upload.p + off, q.bytes, cudaMemcpyHostToDevice, c.stream), "H2D");
      else CU(rt::upload_planes(reinterpret_cast<const rt::DevPlane*>(c.upload.p + off), np, c.stream), "constant upload (planes)");
      off += (q.bytes + 255) & ~size_t(255);
    }
    CU(cudaEventRecord(c.upload.done, c.stream), "cudaEventRecord");
    c.upload.pending = true;
  }
  const bool in_smem = npairs_pad <= rt::kMaxSmemPairs;
  c.smem_scene = in_smem;
  c.cmax = (float)(cmax * (1.0 + 1e-6));  // rounded up: the float filter bound must not shrink
  for (int k = 0; k < 3; ++k) c.centre[k] = centre[k];
  c.rmax = (float)(rmax * (1.0 + 1e-6));
  c.n_spheres = ns;
  c.n_pairs_pad = npairs_pad;
  c.n_planes = np;
  c.n_lights = n_lights;
  c.n_emitters = (int)emit.size();
  c.n_mats = n_mats;
  for (int k = 0; k < 3; ++k) {
    c.bg[k] = env ? env->background[k] : 0.f;
    c.amb[k] = env ? env->ambient[k] : 0.f;
  }
  c.has_scene = true;
  // light-origin shadow scans (rt_wavefront.cuh wf_isect_lt / _split): per point light its own
  // table (the pairs with -h in place of K, then K; the scans stage one light's at a time), and
  // the pairs followed by every light's -h column (the checked build's reference); built on the
  // device; on for up to 30 point lights (wf_shade's reservation lanes) in a shared-memory scene
  c.lt_lights = 0;
  const size_t lt_bytes = (size_t)n_lights * npairs_pad * 8;
  if (n_lights > 0 && n_lights <= rt::kMaxLtLights && ns > 0 && in_smem) {
    CU(c.pairs_lt.reserve(2 * (size_t)npairs_pad + lt_bytes / 16 + 1), "cudaMalloc(light pairs)");
    CU(c.pairs_ltl.reserve((size_t)rt::lt_table_stride(npairs_pad) * n_lights), "cudaMalloc(light pairs)");
    CU(rt::launch_light_tables(c.pairs.p, c.sph_cr.p, c.lights.p, ns, npairs_pad, n_lights, c.centre, c.cmax, c.rmax,
                               c.pairs_lt.p, c.pairs_ltl.p, c.stream), "light table kernel");
    c.lt_lights = n_lights;
  }
  return build_eye_pairs();
}

int rt_camera_set(const float eye[3], const float look_at[3], const float up[3], float vfov_deg) {
  NvtxRange nvtx_range("rt_camera_set");
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (!eye || !look_at || !up) return fail(RT_ERR_INVALID_ARG, "camera: NULL vector");
  if (!finite3(eye) || !finite3(look_at) || !finite3(up) || !std::isfinite(vfov_deg))
    return fail(RT_ERR_INVALID_ARG, "camera: non-finite value");
  if (!(vfov_deg > 0.f && vfov_deg < 180.f)) return fail(RT_ERR_INVALID_ARG, "camera: vfov must be in (0, 180)");
  double f[3] = {(double)look_at[0] - eye[0], (double)look_at[1] - eye[1], (double)look_at[2] - eye[2]};
  double fl = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
  if (!(fl > 0.0)) return fail(RT_ERR_INVALID_ARG, "camera: eye == look_at");
  norm3(f);
  double u0[3] = {up[0], up[1], up[2]};
  double r[3] = {f[1] * u0[2] - f[2] * u0[1], f[2] * u0[0] - f[0] * u0[2], f[0] * u0[1] - f[1] * u0[0]};
  double rl = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  double ul = std::sqrt(u0[0] * u0[0] + u0[1] * u0[1] + u0[2] * u0[2]);
  if (!(rl > 1e-12 * (ul > 0 ? ul : 1.0))) return fail(RT_ERR_INVALID_ARG, "camera: up is zero or parallel to the view direction");
  norm3(r);
  double u[3] = {r[1] * f[2] - r[2] * f[1], r[2] * f[0] - r[0] * f[2], r[0] * f[1] - r[1] * f[0]};
  Context& c = g_ctx;
  for (int k = 0; k < 3; ++k) { c.eye[k] = eye[k]; c.f[k] = f[k]; c.r[k] = r[k]; c.u[k] = u[k]; }
  c.h = std::tan(0.5 * (double)vfov_deg * 3.14159265358979323846 / 180.0);
  c.has_camera = true;
  return build_eye_pairs();
}

int rt_render(int32_t width, int32_t height, int32_t max_depth, int32_t spp, float* out_rgba) {
  NvtxRange nvtx_range("rt_render");
  g_err.clear();
  return render_common(width, height, max_depth, spp, out_rgba, nullptr, nullptr);
}

int rt_render_debug(int32_t width, int32_t height, int32_t max_depth, int32_t spp, float* out_rgba,
                    int32_t* hit_ids, int32_t* bounces) {
  NvtxRange nvtx_range("rt_render_debug");
  g_err.clear();
  if (!hit_ids || !bounces) return fail(RT_ERR_INVALID_ARG, "hit_ids/bounces must not be NULL");
  return render_common(width, height, max_depth, spp, out_rgba, hit_ids, bounces);
}

int rt_stats(rt_ray_stats* rays_cast) {
  g_err.clear();
  if (!rays_cast) return fail(RT_ERR_INVALID_ARG, "rays_cast is NULL");
  if (g_ctx.stats_pending) {
    int rc = collect_stats(g_ctx.stats_timed);
    if (rc) return rc;
  }
  *rays_cast = g_ctx.last;
  return RT_OK;
}

int rt_shard_layout(int32_t width, int32_t height, int32_t world, int32_t* tiles_per_rank, int64_t* slab_bytes) {
  g_err.clear();
  if (width < 1 || height < 1 || world < 1) return fail(RT_ERR_INVALID_ARG, "shard layout: width, height, world must be >= 1");
  const long long tiles = (long long)((width + rt::kTileW - 1) / rt::kTileW) * ((height + rt::kTileH - 1) / rt::kTileH);
  const long long tpr = (tiles + world - 1) / world;
  if (tiles_per_rank) *tiles_per_rank = (int32_t)tpr;
  if (slab_bytes) *slab_bytes = tpr * rt::kTilePx * 16 + 64;
  return RT_OK;
}

int rt_render_shard(int32_t width, int32_t height, int32_t max_depth, int32_t spp, int32_t rank, int32_t world,
                    float* slab_dev) {
  NvtxRange nvtx_range("rt_render_shard");
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (world < 1 || rank < 0 || rank >= world) return fail(RT_ERR_INVALID_ARG, "shard: need 0 <= rank < world");
  if (!slab_dev || !is_device_ptr(slab_dev)) return fail(RT_ERR_INVALID_ARG, "shard: slab must be a device pointer");
  if ((reinterpret_cast<uintptr_t>(slab_dev) & 15u) != 0) return fail(RT_ERR_INVALID_ARG, "shard: slab must be 16-byte aligned");
  rc = check_frame(width, height, max_depth, spp);
  if (rc) return rc;
  int32_t tpr = 0;
  rt_shard_layout(width, height, world, &tpr, nullptr);
  rt::DevParams p = make_params(width, height, max_depth, spp);
  p.mode = 1;
  p.rank = rank;
  p.world = world;
  p.n_items = tpr * rt::kTilePx;
  Context& c = g_ctx;
  float4* slab = reinterpret_cast<float4*>(slab_dev);
  rc = run_render(p, slab, nullptr, nullptr);
  if (rc) return rc;
  // stats record at the slab tail (device to device, stays on the stream)
  CU(cudaMemcpyAsync(slab + (size_t)tpr * rt::kTilePx, c.stats.p, 64, cudaMemcpyDeviceToDevice, c.stream), "stats record");
  defer_stats(true);
  return RT_OK;
}

int rt_render_shard_direct(int32_t width, int32_t height, int32_t max_depth, int32_t spp, int32_t rank,
                           int32_t world, float* frame_dev, uint64_t* records_dev) {
  NvtxRange nvtx_range("rt_render_shard_direct");
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (world < 1 || rank < 0 || rank >= world) return fail(RT_ERR_INVALID_ARG, "shard: need 0 <= rank < world");
  if (!frame_dev || !records_dev || !is_device_ptr(frame_dev) || !is_device_ptr(records_dev))
    return fail(RT_ERR_INVALID_ARG, "direct shard: frame and records must be device (or peer) pointers");
  if ((reinterpret_cast<uintptr_t>(frame_dev) & 15u) != 0 || (reinterpret_cast<uintptr_t>(records_dev) & 7u) != 0)
    return fail(RT_ERR_INVALID_ARG, "direct shard: frame must be 16-byte and records 8-byte aligned");
  rc = check_frame(width, height, max_depth, spp);
  if (rc) return rc;
  int32_t tpr = 0;
  rt_shard_layout(width, height, world, &tpr, nullptr);
  rt::DevParams p = make_params(width, height, max_depth, spp);
  p.mode = 2;
  p.rank = rank;
  p.world = world;
  p.n_items = tpr * rt::kTilePx;
  Context& c = g_ctx;
  rc = run_render(p, reinterpret_cast<float4*>(frame_dev), nullptr, nullptr);
  if (rc) return rc;
  // this rank's 8-uint64 stats record into slot `rank` (peer memory over NVLink when remote)
  CU(cudaMemcpyAsync(records_dev + 8 * (size_t)rank, c.stats.p, 64, cudaMemcpyDefault, c.stream), "stats record");
  defer_stats(true);
  return RT_OK;
}

int rt_sum_shard_stats(const uint64_t* records_dev, int32_t world) {
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (world < 1 || !records_dev || !is_device_ptr(records_dev)) return fail(RT_ERR_INVALID_ARG, "records: device pointer, world >= 1");
  CU(rt::launch_sum_records(reinterpret_cast<const unsigned long long*>(records_dev), world, g_ctx.stats.p, g_ctx.stream),
     "sum stats records");
  defer_stats(false);
  return RT_OK;
}

int rt_ipc_alloc(int64_t bytes, void** dev_ptr, uint8_t handle[64]) {
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (bytes < 1 || !dev_ptr || !handle) return fail(RT_ERR_INVALID_ARG, "ipc_alloc: bytes >= 1 and non-NULL outputs");
  void* p = nullptr;
  CU(cudaMalloc(&p, (size_t)bytes), "cudaMalloc(ipc)");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(e, "cudaIpcGetMemHandle");
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  std::memcpy(handle, &h, 64);
  *dev_ptr = p;
  return RT_OK;
}

int rt_ipc_open(const uint8_t handle[64], void** dev_ptr) {
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (!handle || !dev_ptr) return fail(RT_ERR_INVALID_ARG, "ipc_open: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  CU(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return RT_OK;
}

int rt_ipc_close(void* dev_ptr) {
  g_err.clear();
  if (!dev_ptr) return fail(RT_ERR_INVALID_ARG, "ipc_close: NULL");
  CU(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
  return RT_OK;
}

int rt_ipc_free(void* dev_ptr) {
  g_err.clear();
  if (!dev_ptr) return fail(RT_ERR_INVALID_ARG, "ipc_free: NULL");
  CU(cudaFree(dev_ptr), "cudaFree(ipc)");
  return RT_OK;
}

int rt_assemble_tiles(const float* gathered_dev, int32_t width, int32_t height, int32_t world, float* out_rgba_dev) {
  NvtxRange nvtx_range("rt_assemble_tiles");
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (width < 1 || height < 1 || world < 1) return fail(RT_ERR_INVALID_ARG, "assemble: width, height, world must be >= 1");
  if (!gathered_dev || !out_rgba_dev || !is_device_ptr(gathered_dev) || !is_device_ptr(out_rgba_dev))
    return fail(RT_ERR_INVALID_ARG, "assemble: both pointers must be device pointers");
  int32_t tpr = 0;
  rt_shard_layout(width, height, world, &tpr, nullptr);
  Context& c = g_ctx;
  CU(rt::launch_assemble(reinterpret_cast<const float4*>(gathered_dev), width, height, world, tpr,
                         reinterpret_cast<float4*>(out_rgba_dev), c.stats.p, c.stream), "assemble launch");
  defer_stats(false);
  return RT_OK;
}

int rt_tonemap_rgba8(const float* rgba, uint8_t* out, int64_t n_px, float exposure, float gamma) {
  NvtxRange nvtx_range("rt_tonemap_rgba8");
  g_err.clear();
  int rc = ensure_device();
  if (rc) return rc;
  if (n_px < 0 || !rgba || !out) return fail(RT_ERR_INVALID_ARG, "tonemap: NULL pointer or n_px < 0");
  if (!(exposure > 0.f) || !(gamma > 0.f)) return fail(RT_ERR_INVALID_ARG, "tonemap: exposure and gamma must be > 0");
  if (!is_device_ptr(rgba) || !is_device_ptr(out)) return fail(RT_ERR_INVALID_ARG, "tonemap: device pointers required");
  if (n_px == 0) return RT_OK;
  CU(rt::launch_tonemap(reinterpret_cast<const float4*>(rgba), out, n_px, exposure, gamma, g_ctx.stream), "tonemap launch");
  return RT_OK;
}

}  // extern "C"
