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
void orc_brdf(int32_t kind, const double albedo[3], double ks, double shininess,
              const double wi[3], const double wo[3], const double n[3], double f[3]);
double orc_schlick(double ior, double cos_outside);
int32_t orc_tonemap8(double v, double exposure, double gamma);

#ifdef __cplusplus
}
#endif
#endif
