/*
 * oracle.h — plain, slow, single-threaded CPU oracle of the per-pixel iterative ray tracer
 * of arXiv 1504.03151 ("Massively Parallel Ray Tracing Algorithm Using GPU").
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * (and `bench.py --impl reference`) may load this library. The product path
 * (paper_1504_03151_b200/, include/rt.h) never includes, links or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Arithmetic is IEEE double. Every scene value is read as float32 (the shared input contract
 * written by scenegen/) and widened to double, so both sides see identical inputs.
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n, §8(c).k = SURVEY.md §8(c) step k,
 * R#n = reading n in DESIGN.md §"Readings of the paper".
 *
 * Pinned-by (tests/test_oracle_*.py): SPEC worked examples (S:56-59, S:65-69, S:83-94,
 * S:141-144), closed forms W1-W6 (tests/golden/worked_examples.json),
 * brute-force bisection of Eq. 9 along the ray, BRDF/Phong hemisphere normalisation
 * quadrature, splitmix64 reference vector, invariants (miss -> background bit-exact,
 * linearity, depth monotonicity, partition invariance).
 * Continuation and shadow arithmetic (tests/test_oracle_continuation.py): Schlick closed forms
 * and the exit-side cosine, DIFFUSE-kr and coloured-glass weights,
 * the p + EPS_T n shadow origin, the [EPS_T, t_max) interval, ambient at DIFFUSE hits
 * only (R#4), ties to the lowest index, the inclusive EPS_T threshold, the RNG
 * composition against an independent splitmix64 stream, hand-counted test counts in
 * index order (§8(c).1 step 11). tools/oracle_mutations.py applies 16 plausible mistakes to this
 * file; each one fails at least one of these tests (profiles/r02_oracle_mutations.txt).
 * NEXT-1 / NEXT-2 extensions (tests/test_oracle_next.py): sphere-irradiance closed form and an
 * independent quadrature for the area-light estimator, cosine-lobe moments, furnace and
 * constant-sky closed forms for the global bounce, SPEC S:148-150 / S:166-168 / S:302-303
 * examples, the NEE double-count rule, progressive resume.
 */
#ifndef RT_ORACLE_H
#define RT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scene as flat float32 arrays (layout documented in scenegen/__init__.py).
 * prim_type: 0 sphere (p = cx,cy,cz,radius), 1 plane (p = nx,ny,nz,d with n.x = d).
 * mat_kind: 0 DIFFUSE, 1 SPECULAR, 2 REFRACTIVE. */
typedef struct {
  int32_t n_prims;
  const int32_t* prim_type;
  const int32_t* prim_mat;
  const float* prim_p;          /* [n_prims][4] */
  int32_t n_mats;
  const int32_t* mat_kind;
  const float* mat_albedo;      /* [n_mats][3] */
  const float* mat_emission;    /* [n_mats][3] */
  const float* mat_ior;
  const float* mat_ks;
  const float* mat_shininess;
  const float* mat_kr;
  int32_t n_lights;
  const float* light_pos;       /* [n_lights][3] */
  const float* light_intensity; /* [n_lights][3] */
  const float* background;      /* [3] */
  const float* ambient;         /* [3] */
  const float* eye;             /* [3] */
  const float* look_at;         /* [3] */
  const float* up;              /* [3] */
  float vfov_deg;
} orc_scene;

typedef struct {
  int32_t width, height, max_depth, spp;
  uint64_t seed;
  /* Classification only (not the method): when > 0, every ray origin/direction component is
   * multiplied by (1 + perturb * u), u in [-1, 1] from a hash of (perturb_seed, pixel, sample,
   * segment, component). Used to detect samples that are ill-conditioned in float32
   * (Monte Carlo arithmetic). perturb = 0 is the method exactly. */
  double perturb;
  uint64_t perturb_seed;
  /* SURVEY §8(f) NEXT-1 / NEXT-2 (0 = the §8(a) hot path exactly):
   * integrator  0 Whitted (DIFFUSE stops unless kr > 0); 1 global: DIFFUSE continues with a
   *             cosine-weighted direction, T *= albedo (R#40)
   * area_lights 1: every emissive sphere is also sampled as a light, one uniform point on its
   *             surface per emitter per shading point (R#41)
   * jitter      0: stratified / Hammersley sub-pixel offsets; 1: random offsets from the
   *             pixel's RNG stream (progressive passes; R#42)
   * sample_base global index of sample 0: sample s of this call is sample (pass)
   *             sample_base + s of the pixel's sequence (keys every RNG draw) */
  int32_t integrator;
  int32_t area_lights;
  int32_t jitter;
  int32_t pad_;
  int64_t sample_base;
} orc_frame;

typedef struct {
  uint64_t primary, shadow, secondary, sphere_tests, plane_tests;
} orc_counts;

/* Render n_pixels pixels (pixel index = py*width + px; NULL = all pixels, row-major).
 * Outputs (each may be NULL):
 *   rgb        [n_pixels][3]  mean radiance over spp samples (§8(c).10)
 *   hit_ids    [n_pixels][spp][max_depth+1]  prim index per segment; -1 miss; -2 not traced
 *   bounces    [n_pixels][spp]  number of secondary rays
 *   margin     [n_pixels][spp]  min normalised decision margin over the sample
 *   sample_rgb [n_pixels][spp][3]
 * Returns 0, or -1 on invalid arguments. */
int orc_render(const orc_scene* scene, const orc_frame* frame, const int64_t* pixels,
               int64_t n_pixels, double* rgb, int32_t* hit_ids, int32_t* bounces,
               double* margin, double* sample_rgb, orc_counts* counts);

/* Literal Alg. 1 (SPEC oracle_render_local S:416-423): local
 * illumination, serial nested loops. Per pixel, per ray (rays_per_pixel sub-pixel offsets of
 * orc_sample_offset), nearest hit; emission of the hit; at DIFFUSE hits ambient, the point
 * lights (as orc_render) and, per emissive sphere, per cell of a light_grid x light_grid
 * latitude-longitude grid (theta in [i pi/n, (i+1) pi/n], phi in [2 pi j/n, 2 pi (j+1)/n],
 * pole +z): a shadow ray to the cell's midpoint (the emitter itself does not block; `break` at
 * the first occluder) and the Eq. 8 term f_r L_e cos_s cos_l / d^2 times the cell's exact area
 * r^2 (cos theta_i - cos theta_i+1) dphi. No continuation (local mode = depth 0). Mean over the
 * rays of the pixel. rgb: [width*height][3]. Returns 0, or -1 on invalid arguments. */
int orc_render_local_grid(const orc_scene* scene, int32_t width, int32_t height, int32_t light_grid,
                          int32_t rays_per_pixel, double* rgb);

/* Building blocks, exported for the unit pins. */
int orc_solve_quadratic(double a, double b, double c, double roots[2]);
int orc_intersect_sphere(const double o[3], const double d[3], const double c[3], double r,
                         double* t);
int orc_intersect_plane(const double o[3], const double d[3], const double n[3], double dp,
                        double* t);
void orc_reflect(const double d[3], const double n[3], double out[3]);
int orc_refract(const double d[3], const double n[3], double eta, double out[3]);
void orc_sample_offset(int32_t s, int32_t spp, double* ox, double* oy);
void orc_camera_ray(const orc_scene* scene, int32_t width, int32_t height, int32_t px,
                    int32_t py, int32_t s, int32_t spp, double o[3], double d[3]);
uint64_t orc_mix64(uint64_t x);
double orc_rng(uint64_t seed, uint64_t pixel_index, uint32_t sample, uint32_t depth);
/* stream k of the counter-based RNG: counter word (sample << 32) + (k << 8) + depth, depth <
 * 256; k = 0 is orc_rng (R#42). Streams: 0 Fresnel, 1/2 jitter x/y, 3/4 diffuse bounce,
 * 5 + 2e / 6 + 2e the surface sample of emitter e. */
double orc_rng_stream(uint64_t seed, uint64_t pixel_index, uint32_t sample, uint32_t depth,
                      uint32_t stream);
/* uniform point on a sphere: cos(theta) = 1 - 2 u1, phi = 2 pi u2, z = pole;
 * writes the point and the outward unit normal, returns pdf_area = 1 / (4 pi r^2) */
double orc_sample_sphere(const double c[3], double r, double u1, double u2, double x[3],
                         double nl[3]);
/* orthonormal basis (t1, t2, n) of a unit vector n (branchless form, Duff et al. 2017) */
void orc_onb(const double n[3], double t1[3], double t2[3]);
/* cosine-weighted direction about unit n: r = sqrt(u1), phi = 2 pi u2,
 * local (r cos phi, r sin phi, sqrt(1 - u1)) in orc_onb(n); pdf = cos(theta) / pi */
void orc_cosine_direction(const double n[3], double u1, double u2, double out[3]);
void orc_brdf(int32_t kind, const double albedo[3], double ks, double shininess,
              const double wi[3], const double wo[3], const double n[3], double f[3]);
double orc_schlick(double ior, double cos_outside);
int32_t orc_tonemap8(double v, double exposure, double gamma);

#ifdef __cplusplus
}
#endif
#endif
