/*
 * rt.h — C ABI of the B200-native hot path of arXiv 1504.03151 ("Massively Parallel Ray Tracing
 * Algorithm Using GPU"): per-pixel iterative ray tracing of spheres and planes with
 * Lambert/Phong point-light shading, one shadow ray per light, and a stack-free
 * reflection/refraction loop up to max_depth, written to a float RGBA framebuffer.
 *
 * Library: paper_1504_03151_b200/libb200rt.so (CUDA, sm_100a). No torch types cross this
 * boundary; pointers are plain host or device pointers.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n; BJ = BASELINE.json
 * north_star; §8 = SURVEY.md §8; R#n = DESIGN.md reading n.
 *
 * Conventions shared by every entry point:
 *  - Return value: RT_OK (0) on success, a negative rt_status on error. The library never
 *    aborts. rt_last_error() returns a message for the last failing call of the calling
 *    thread ("prim 7: radius <= 0", cf. the ParseError line + reason of S:221).
 *  - On error, caller-owned outputs are left untouched and library state is unchanged.
 *  - Ownership: inputs are deep-copied during the call; the caller keeps its arrays. The
 *    library owns device copies of the scene until the next rt_scene_upload or process exit.
 *  - Output pointers may be host or device memory (detected with cudaPointerGetAttributes).
 *    With a host pointer the call returns after the data is complete; with a device pointer
 *    the call is asynchronous on the library stream (rt_set_stream).
 *  - One context per process and current CUDA device (one rank = one process = one GPU).
 *    Calls are not thread-safe.
 */
#ifndef B200_RT_H
#define B200_RT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RT_OK = 0,
  RT_ERR_INVALID_ARG = -1, /* a parameter or scene element violates the documented contract */
  RT_ERR_NO_SCENE = -2,    /* rt_render* before a successful rt_scene_upload */
  RT_ERR_NO_CAMERA = -3,   /* rt_render* before a successful rt_camera_set */
  RT_ERR_CUDA = -4,        /* CUDA runtime error (message carries cudaGetErrorString) */
  RT_ERR_OOM = -5,         /* device allocation failed */
  RT_ERR_STATE = -6,       /* call not valid in the current state */
  RT_ERR_PARSE = -7,       /* scene text: rt_last_error() = "line N: reason" */
  RT_ERR_IO = -8           /* file could not be read or written */
} rt_status;

enum { RT_PRIM_SPHERE = 0, RT_PRIM_PLANE = 1 };
/* Material kinds (Fig. 3). */
enum { RT_MAT_DIFFUSE = 0, RT_MAT_SPECULAR = 1, RT_MAT_REFRACTIVE = 2 };

enum {
  RT_MAX_LIGHTS = 32,        /* point lights per scene */
  RT_MAX_EMITTERS = 64,      /* emissive spheres sampled as area lights (rt_set_integrator) */
  RT_MAX_PLANES = 32,        /* planes per scene */
  RT_MAX_SPHERES = 1 << 20,  /* spheres per scene; > RT_SMEM_SPHERES uses the global-memory path */
  RT_SMEM_SPHERES = 10240,   /* spheres staged per CTA in shared memory (TMA bulk copy, 160 KB) */
  RT_TILE_W = 8,             /* shard tile: 8 x 4 pixels = one warp of primary rays */
  RT_TILE_H = 4
};

/* Primitive (S:37-41 sphere; planes per BJ north_star).
 *   type = RT_PRIM_SPHERE: p = {cx, cy, cz, radius}, radius > 0            (Eq. 9)
 *   type = RT_PRIM_PLANE:  p = {nx, ny, nz, d}, n != 0, points x with n.x = d (normalised on
 *                          upload; two-sided)
 * material indexes the rt_material array. 24 bytes, 4-byte aligned. */
typedef struct {
  uint32_t type;
  uint32_t material;
  float p[4];
} rt_primitive;

/* Material (S:199-204 + reading R#3, R#8): albedo rho in [0,1]; emission L_e >= 0 (Eq. 7,
 * P:128); ior >= 1 (REFRACTIVE); DIFFUSE adds a normalised Phong lobe
 * ks (s+2)/(2 pi) max(0, r.wo)^s with ks in [0,1], shininess s in [1, 1e4], and mirrors
 * with weight kr in [0,1] when kr > 0. 48 bytes. */
typedef struct {
  uint32_t kind;
  float albedo[3];
  float emission[3];
  float ior;
  float ks;
  float shininess;
  float kr;
  float _pad;
} rt_material;

/* Point light (reading R#2): position and RGB intensity I (>= 0); irradiance I cos/d^2
 * (Eq. 3, for a delta source). 24 bytes. */
typedef struct {
  float position[3];
  float intensity[3];
} rt_light;

/* Environment (readings R#4, R#5): radiance returned by rays that miss everything, and the
 * ambient term added as rho * ambient at DIFFUSE hits. NULL = all zero. */
typedef struct {
  float background[3];
  float ambient[3];
} rt_env;

/* Ray statistics of the last rt_render / rt_render_shard / rt_assemble_tiles (BJ "rt_stats
 * (rays_cast)"). primary + shadow + secondary = rays cast (BJ metric). sphere_tests and
 * plane_tests are the algorithmic test counts of SURVEY §8(c).1 step 11 (closest-hit rays
 * test every primitive; shadow rays count the primitives up to and including the first
 * occluder in primitive index order, for any interleaving of spheres and planes).
 * last_render_ms: device time of the render kernel (CUDA events on the library stream; 0 for
 * rt_assemble_tiles). 112 bytes. */
typedef struct {
  uint64_t primary;
  uint64_t shadow;
  uint64_t secondary;
  uint64_t sphere_tests;
  uint64_t plane_tests;
  double last_render_ms;
  uint64_t closest_sphere_tests; /* part of sphere_tests done by closest-hit (primary/secondary) rays */
  double isect_closest_ms;       /* wavefront: summed device time of the closest-hit intersection
                                    kernels (CUDA events around each launch); 0 for the megakernel
                                    and for graph replays with concurrency on (rt_set_graphs), whose
                                    launches overlap: time them with rt_set_concurrency(0) */
  double isect_shadow_ms;        /* wavefront: same for the shadow-ray intersection kernels */
  uint32_t launches;             /* kernels of this library launched by the call */
  int32_t variant;               /* RT_VARIANT_MEGAKERNEL or RT_VARIANT_WAVEFRONT actually used */
  double shade_ms;               /* wavefront: summed device time of the wf_shade launches (a4/a6:
                                    FP64 nearest hit, shading, shadow set-up, bounce) */
  double isect_eye_ms;           /* wavefront: the part of isect_closest_ms spent on camera rays
                                    (depth 0, shared-origin tangent test) */
  int32_t graph;                 /* wavefront launch of the call: 0 kernel by kernel, 1 captured
                                    into a CUDA graph and launched, 2 replay of a cached graph
                                    (rt_set_graphs; up to 4 launch keys are cached) */
  int32_t _pad;
  double accumulate_ms;          /* wavefront: summed device time of the wf_accumulate launches
                                    (a5 FP64 occlusion decisions, a4 light sums) */
} rt_ray_stats;

/* Upload the scene: validates every element, normalises plane
 * normals, packs spheres into a structure-of-arrays pair layout in device memory (each render
 * CTA stages it into shared memory with a TMA bulk copy up to RT_SMEM_SPHERES spheres), planes
 * into the constant bank, materials and lights into global memory. Replaces any previous
 * scene. n_prims >= 0, 1 <= n_mats, 0 <= n_lights <= RT_MAX_LIGHTS. env may be NULL. Errors: RT_ERR_INVALID_ARG (message names the element),
 * RT_ERR_OOM, RT_ERR_CUDA. */
int rt_scene_upload(const rt_primitive* prims, int32_t n_prims, const rt_material* mats,
                    int32_t n_mats, const rt_light* lights, int32_t n_lights, const rt_env* env);

/* Pinhole camera: forward = normalize(look_at - eye), right =
 * normalize(forward x up), up' = right x forward; vfov in (0, 180) degrees. Requires
 * eye != look_at and up not parallel to the view direction. */
int rt_camera_set(const float eye[3], const float look_at[3], const float up[3], float vfov_deg);

/* Render one frame: for every pixel (row-major, row 0 =
 * top) and sample s = 0..spp-1 (stratified n x n when spp = n^2, else Hammersley, R#19):
 * primary ray -> nearest hit over all primitives -> emission + (DIFFUSE) ambient + per-light
 * shadow ray and Lambert/Phong term -> stack-free reflection/refraction continuation for up to
 * max_depth secondary segments. out_rgba receives width*height float4 (R, G, B, 1) = the mean
 * over samples summed in order s = 0..spp-1; 16 bytes per pixel, caller-owned, host or device.
 * width, height >= 1; width*height <= 2^31-1; 0 <= max_depth <= 64; 1 <= spp <= 4096. */
int rt_render(int32_t width, int32_t height, int32_t max_depth, int32_t spp, float* out_rgba);

/* Copy the statistics of the last render into *rays_cast. */
int rt_stats(rt_ray_stats* rays_cast);

/* ---- helpers (multi-GPU sharding, parity, plumbing) ---------------------------------------- */

/* Bind the library to a cudaStream_t (NULL = legacy default stream). Kernels and copies are
 * issued on it. */
int rt_set_stream(void* cuda_stream);

/* Kernel organisation (same results, bit for bit):
 *   RT_VARIANT_WAVEFRONT: queue-based kernels — an FP32 FFMA2 intersection kernel per depth for
 *     closest-hit rays and one for shadow rays, FP64 shade/accumulate kernels between;
 *   RT_VARIANT_MEGAKERNEL: one persistent kernel, each lane carries a pixel's path state;
 *   RT_VARIANT_AUTO (default): wavefront for scenes of >= 64 spheres, else megakernel. */
enum { RT_VARIANT_AUTO = -1, RT_VARIANT_MEGAKERNEL = 0, RT_VARIANT_WAVEFRONT = 1 };
int rt_set_variant(int32_t variant);

/* Wavefront kernels: 1 (default) runs the shadow-ray scan + accumulation of depth d on a second
 * stream, concurrently with the closest-hit scan of depth d+1; 0 runs every launch in order on
 * the library stream (same results bit for bit; used to time each kernel alone). */
int rt_set_concurrency(int32_t on);

/* Wavefront kernels: chunk pipelining over `slots` buffer sets (1..4; 0 = AUTO, the default: 2, or
 * 3 when the frame has at least 8 chunks of 2^22 paths). A frame is cut
 * into chunks of at most 2^22 paths, and into at least `slots` chunks when it has >= 2^17 paths
 * per chunk; chunk i runs on slot i % slots, each slot with its own buffers and stream pair, so
 * one chunk's short deep-depth queues overlap the next chunks' dense first depths. 1 renders the
 * chunks one after another. Ignored (1) when concurrency is off. Same results bit for bit for
 * every value. RT_ERR_INVALID_ARG outside 0..4. */
int rt_set_pipeline(int32_t slots);

/* Wavefront kernels, scenes beyond RT_SMEM_SPHERES (the shared-memory budget): 1 (default) the
 * long-queue scans stream the sphere pairs through a ring of two TMA-loaded 16 KB tiles per CTA
 * (cp.async.bulk on mbarriers, a copy in flight while the warps scan the other tile); 0 reads them
 * from global memory (A/B knob). Same results bit for bit. RT_ERR_INVALID_ARG unless 0/1. */
int rt_set_tiled_scan(int32_t on);

/* Test support. Schedule fuzzing: seed != 0 makes every later wavefront render that is launched
 * kernel by kernel (not a graph replay) insert short spin kernels of pseudo-random length (0-40
 * us, drawn from the seed) on its streams at every fork, join and slot start, so the concurrent
 * kernels interleave differently; a missing stream dependency then shows up as a different frame
 * (the results must equal the in-order render bit for bit). 0 (default) turns it off. */
int rt_set_schedule_jitter(uint64_t seed);

/* Test support. In a library built with -DRT_CHECKS=1 (build.py --checks) every kernel checks its
 * queue, list and slot indices and capacities; *first_failed receives the id of the first check
 * that failed since the last call (0 = none) and the record is cleared; *compiled = 1. In the
 * default build the checks are compiled out: *first_failed = 0, *compiled = 0. */
int rt_check_status(uint32_t* first_failed, int32_t* compiled);

/* Wavefront kernels: 1 (default) replays a CUDA graph of the launch sequence. The sequence of a
 * render (frame or shard size, max_depth, spp, output pointers, buffers, concurrency) is captured
 * the second time it is requested within the last 8 renders and replayed whenever it comes again
 * (up to 4 sequences cached, least recently used evicted: e.g. frames alternating between two
 * output buffers), so a frame loop pays one graph launch per frame instead of ~6 kernel launches
 * per depth; materials, lights and the environment may change between replays (the kernels read
 * them at run time; each scan's kernel was chosen from the previous frame's queue lengths, so a
 * large change costs some speed, never results), while a new camera or new geometry bounds change
 * the kernel arguments and start a new capture. 0 launches every kernel from the host and empties the cache (calling it with 1 empties
 * it too). Same results bit for bit either way. RT_ERR_INVALID_ARG unless 0/1. */
int rt_set_graphs(int32_t on);

/* Wavefront kernels, test and tuning knob: -1 (default) splits a scan over 2-8 warps per ray
 * group only when its queue is short (split scans); 1, 2, 4 or 8 forces that many
 * parts on every intersection scan (1: never split). Results are bit-identical for every value.
 * RT_ERR_INVALID_ARG otherwise. */
int rt_set_scan_split(int32_t parts);

/* Seed of the counter-based RNG that picks reflection vs refraction (R#9). */
int rt_set_seed(uint64_t seed);

/* Message of the last failing call on this thread ("" if none). Owned by the library. */
const char* rt_last_error(void);

/* Shard layout for `world` ranks: the image is cut into RT_TILE_W x RT_TILE_H tiles; rank r owns
 * one tile of every group of `world` consecutive tiles, its local tile j being the global tile
 * j * world + (r + j) % world (cyclic, the slot rotating per group so a rank's tiles do not line
 * up in image columns). tiles_per_rank = ceil(n_tiles / world); slab_bytes =
 * tiles_per_rank * 32 * 16 + 64 (pixel slab, tile-major, then a 64-byte stats record of 8
 * uint64: primary, shadow, secondary, sphere_tests, plane_tests, closest_sphere_tests, 0, 0). */
int rt_shard_layout(int32_t width, int32_t height, int32_t world, int32_t* tiles_per_rank,
                    int64_t* slab_bytes);

/* Render this rank's tiles into slab_dev (device pointer, slab_bytes from rt_shard_layout).
 * Pixels of partial edge tiles outside the image are written as 0. Tiles inside the rank are
 * taken dynamically by persistent CTAs. The framebuffer assembled from all ranks is
 * bit-identical to rt_render for any world size. */
int rt_render_shard(int32_t width, int32_t height, int32_t max_depth, int32_t spp, int32_t rank,
                    int32_t world, float* slab_dev);

/* gathered_dev: world slabs back to back (e.g. the output of an NCCL all-gather / gather).
 * Writes the row-major framebuffer to out_rgba_dev and sums the ranks' stats records into the
 * library statistics (rt_stats). Both pointers are device pointers. */
int rt_assemble_tiles(const float* gathered_dev, int32_t width, int32_t height, int32_t world,
                      float* out_rgba_dev);

/* ---- fused render + gather over NVLink peer memory (SURVEY §8(e) ablation) -------------------
 * Direct shard: render this rank's tiles (the rotated cyclic assignment of rt_shard_layout) and store
 * each finished pixel straight into the row-major frame `frame_dev` — rank 0's framebuffer, a
 * peer pointer (rt_ipc_open) on the other ranks, so the pixels cross NVLink inside the resolve
 * kernel instead of through a slab and an all-gather. The rank's 8-uint64 stats record goes to
 * records_dev[8 * rank ..]. No pixel of another rank is touched; after every rank's call has
 * completed (a barrier), the frame equals rt_render's bit for bit. Rank 0 then calls
 * rt_sum_shard_stats(records_dev, world) so rt_stats reports the whole frame. */
int rt_render_shard_direct(int32_t width, int32_t height, int32_t max_depth, int32_t spp, int32_t rank,
                           int32_t world, float* frame_dev, uint64_t* records_dev);
int rt_sum_shard_stats(const uint64_t* records_dev, int32_t world);
/* CUDA IPC for the direct shard (one process per GPU): rt_ipc_alloc cudaMallocs `bytes` and
 * returns the pointer and its 64-byte handle; another process maps it with rt_ipc_open (peer
 * access enabled lazily) and unmaps with rt_ipc_close; the owner frees with rt_ipc_free. */
int rt_ipc_alloc(int64_t bytes, void** dev_ptr, uint8_t handle[64]);
int rt_ipc_open(const uint8_t handle[64], void** dev_ptr);
int rt_ipc_close(void* dev_ptr);
int rt_ipc_free(void* dev_ptr);

/* rt_render plus per-sample records for parity tests: hit_ids[((py*W+px)*spp + s)*(max_depth+1)
 * + segment] = primitive index hit by that segment, -1 on a miss, -2 if the segment was not
 * traced; bounces[(py*W+px)*spp + s] = number of secondary rays. Host or device pointers. */
int rt_render_debug(int32_t width, int32_t height, int32_t max_depth, int32_t spp,
                    float* out_rgba, int32_t* hit_ids, int32_t* bounces);

/* ---- area lights, global illumination, progressive passes ----
 * Integrator for every following render call (R#40-R#43):
 *   integrator RT_INTEGRATOR_WHITTED (default): the §8(a) hot path — DIFFUSE hits stop unless
 *     kr > 0 (mirror term); RT_INTEGRATOR_GLOBAL: DIFFUSE hits continue with a cosine-weighted
 *     direction (pdf cos/pi), T *= albedo (Fig. 7 P:290 "global illumination").
 *   area_lights 1: every sphere whose material emits (emission > 0 in some channel; at most
 *     RT_MAX_EMITTERS) is also a light: one uniform point on its surface per shading point
 *     (pdf 1/(4 pi r^2)), contribution f_r L_e cos_s cos_l / (d^2 pdf), shadow ray to the point
 *     with the emitter itself non-blocking (Eq. 8, Fig. 2). A cosine bounce that
 *     hits a sampled emitter does not add its emission again.
 * Non-default settings run the wavefront kernels (RT_VARIANT_MEGAKERNEL is overridden).
 * Errors: RT_ERR_INVALID_ARG for values outside the enums. */
enum { RT_INTEGRATOR_WHITTED = 0, RT_INTEGRATOR_GLOBAL = 1 };
int rt_set_integrator(int32_t integrator, int32_t area_lights);

/* Progressive passes (§IV.A P:226-229 "the same kernel function should be launched
 * iteratively", "overlapping new color value onto the pixel"). Pass p traces one
 * camera ray per pixel with a random sub-pixel offset and random light / bounce samples, all
 * keyed by (seed, pixel, p) (R#42). For p = pass_begin .. pass_begin + n_passes - 1, in order:
 *   accum_rgb[(py*W + px)*3 + c] += radiance of pass p   (double, device pointer, caller-owned;
 *                                                         zero it before pass 0)
 * then, if out_rgba != NULL (host or device, float4 row-major), out = accum / (pass_begin +
 * n_passes), alpha 1. Splitting a run of passes over several calls is bit-identical to one
 * call. 1 <= n_passes <= 4096, pass_begin + n_passes <= 2^32. Stats (rt_stats) cover this
 * call's passes. Asynchronous unless out_rgba is a host pointer. */
int rt_render_passes(int32_t width, int32_t height, int32_t max_depth, int64_t pass_begin,
                     int32_t n_passes, double* accum_rgb, float* out_rgba);
/* rt_render_passes plus the per-sample records of rt_render_debug (sample index = pass -
 * pass_begin). out_rgba, hit_ids, bounces must not be NULL. */
int rt_render_passes_debug(int32_t width, int32_t height, int32_t max_depth, int64_t pass_begin,
                           int32_t n_passes, double* accum_rgb, float* out_rgba, int32_t* hit_ids,
                           int32_t* bounces);

/* ---- scene files and images ---------------------------------------------
 * Scene text (extended to the primitives of this library), one
 * directive per line, fields separated by whitespace, '#' comments and blank lines ignored:
 *   camera ex ey ez  lx ly lz  ux uy uz  vfov                         (exactly one)
 *   sphere radius  cx cy cz  er eg eb  ar ag ab  kind [ior] [opts]     (SPEC grammar)
 *   plane  nx ny nz d  er eg eb  ar ag ab  kind [ior] [opts]           (n.x = d)
 *   light  px py pz  ir ig ib                                          (point light)
 *   background r g b | ambient r g b
 * kind in {diffuse, specular, refractive}; ior (refractive only) defaults to 1.5; opts are
 * ks=K shininess=S kr=R (defaults 0, 1, 0). Numbers are read as float32 (strtof). Every
 * sphere/plane line defines its own material. The whole text is parsed and validated before any
 * device call; then the scene is uploaded (rt_scene_upload) and the camera set (rt_camera_set).
 * Errors: RT_ERR_PARSE with rt_last_error() = "line N: reason" (unknown directive, bad arity,
 * non-numeric or non-finite field, radius <= 0, albedo outside [0,1], emission < 0, ior < 1,
 * unknown kind or option, zero plane normal, missing camera, duplicate camera, invalid camera);
 * errors of rt_scene_upload / rt_camera_set otherwise. Never reads past text[n_bytes - 1]. */
int rt_scene_parse(const char* text, int64_t n_bytes);
/* rt_scene_parse of a file's bytes. RT_ERR_IO if it cannot be read (message names the path). */
int rt_scene_load(const char* path);
/* SPEC write_ppm: binary PPM P6, header "P6\n<W> <H>\n255\n", then W*H RGB bytes,
 * row 0 = top, tone-mapped on the device (rt_tonemap_rgba8). rgba: W*H float4, device pointer.
 * RT_ERR_IO if the file cannot be written. */
int rt_write_ppm(const float* rgba, int32_t width, int32_t height, float exposure, float gamma,
                 const char* path);

/* SPEC tone_map on the device: per channel round_half_up(255 clamp(exposure v, 0,
 * 1)^(1/gamma)), alpha = 255. rgba: n_px float4 (device); out: n_px * 4 bytes (device). */
int rt_tonemap_rgba8(const float* rgba, uint8_t* out, int64_t n_px, float exposure, float gamma);

#ifdef __cplusplus
}
#endif
#endif /* B200_RT_H */
