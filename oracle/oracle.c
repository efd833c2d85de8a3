/*
 * oracle.c — plain, slow, single-threaded, double-precision CPU oracle of the hot path of
 * arXiv 1504.03151: per-pixel iterative (stack-free) Whitted-style ray tracing of spheres and
 * planes with Lambert + normalised-Phong point-light shading, one shadow ray per light, and a
 * reflection/refraction continuation loop up to max_depth.
 *
 * TEST INFRASTRUCTURE ONLY — see oracle.h. Nothing here is shared with the CUDA path.
 *
 * The code follows §8(c).1 step by step, in the paper's order and notation:
 *   ray o + t d (Eq. 10); sphere (p-c).(p-c) - r^2 = 0 (Eq. 9);
 *   substituted quadratic (Eq. 11) solved per Eq. 12 with a = d.d = 1
 *   (S:35); radiance L_o = L_e + f_r L_i cos(theta) (Eq. 6-8) for delta
 *   (point) lights; Alg. 1 shadow loop with `break` at the first occluder;
 *   recursion replaced by iteration.
 * Margin/classification code (clearly separated, suffix _margin) is NOT part of the method:
 * it only labels samples as exact-class or edge-class for the parity rule in DESIGN.md.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define EPS_T 1e-4 /* minimum accepted hit parameter (self-intersection epsilon) */
static const double PI = 3.14159265358979323846264338327950288;

/* ----------------------------------------------------------------------------------------
 * Vector algebra
 * -------------------------------------------------------------------------------------- */
typedef struct { double x, y, z; } v3;

static v3 mk(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 ld3(const float* p) { return mk((double)p[0], (double)p[1], (double)p[2]); }
static v3 ldd(const double* p) { return mk(p[0], p[1], p[2]); }
static void st3(double* out, v3 a) { out[0] = a.x; out[1] = a.y; out[2] = a.z; }
static v3 add(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 sub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 scl(v3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); }
static v3 mulv(v3 a, v3 b) { return mk(a.x * b.x, a.y * b.y, a.z * b.z); }
static double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 cross(v3 a, v3 b) {
  return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double len(v3 a) { return sqrt(dot(a, a)); }
static v3 normalize(v3 a) { return scl(a, 1.0 / len(a)); }

/* ----------------------------------------------------------------------------------------
 * Geometry (Eq. 9-12)
 * -------------------------------------------------------------------------------------- */

/* solve_quadratic: real roots of a t^2 + b t + c = 0, ascending, stable form. */
int orc_solve_quadratic(double a, double b, double c, double roots[2]) {
  double disc = b * b - 4.0 * a * c; /* Eq. 12 discriminant */
  if (disc < 0.0) return 0;
  if (disc == 0.0) { roots[0] = -b / (2.0 * a); return 1; }
  double q = -0.5 * (b + copysign(sqrt(disc), b));
  double r0 = q / a, r1 = c / q;
  roots[0] = r0 < r1 ? r0 : r1;
  roots[1] = r0 < r1 ? r1 : r0;
  return 2;
}

/* Both roots of Eq. 11 with a = d.d = 1 and half-b = (o-c).d (§8(c).1 step 3).
 * disc uses the precise form r^2 - |oc - b d|^2 (equal to b^2 - (|oc|^2 - r^2) exactly).
 * Returns 0 if disc < 0 (miss), else 1 with t0 <= t1. */
static int sphere_roots(v3 o, v3 d, v3 c, double r, double* t0, double* t1) {
  v3 oc = sub(o, c);
  double b = dot(oc, d);
  v3 perp = sub(oc, scl(d, b));
  double disc = r * r - dot(perp, perp);
  if (disc < 0.0) return 0;
  double q = sqrt(disc);
  double cprime = dot(oc, oc) - r * r; /* product of the roots (a = 1) */
  if (b < 0.0) {                       /* -b + q has no cancellation */
    double far = -b + q;
    *t1 = far;
    *t0 = far != 0.0 ? cprime / far : -b - q;
  } else {
    double near = -b - q;
    *t0 = near;
    *t1 = near != 0.0 ? cprime / near : -b + q;
  }
  if (*t0 > *t1) { double tmp = *t0; *t0 = *t1; *t1 = tmp; }
  return 1;
}

/* intersect_sphere: smallest root >= EPS_T; inside -> exit root; tangent -> hit. */
static int sphere_hit(v3 o, v3 d, v3 c, double r, double* t) {
  double t0, t1;
  if (!sphere_roots(o, d, c, r, &t0, &t1)) return 0;
  if (t0 >= EPS_T) { *t = t0; return 1; }
  if (t1 >= EPS_T) { *t = t1; return 1; }
  return 0;
}

/* Ray-plane: n.(o + t d) = dp, accept t >= EPS_T; |n.d| < 1e-12 is a miss (§8(c).1 step 3). */
static int plane_hit(v3 o, v3 d, v3 n, double dp, double* t) {
  double den = dot(n, d);
  if (fabs(den) < 1e-12) return 0;
  double tt = (dp - dot(n, o)) / den;
  if (tt >= EPS_T) { *t = tt; return 1; }
  return 0;
}

int orc_intersect_sphere(const double o[3], const double d[3], const double c[3], double r,
                         double* t) {
  return sphere_hit(ldd(o), ldd(d), ldd(c), r, t);
}

int orc_intersect_plane(const double o[3], const double d[3], const double n[3], double dp,
                        double* t) {
  return plane_hit(ldd(o), ldd(d), ldd(n), dp, t);
}

/* reflect: d - 2 (d.n) n */
static v3 reflect(v3 d, v3 n) { return sub(d, scl(n, 2.0 * dot(d, n))); }

/* refract: Snell with eta = n1/n2, n opposing d; TIR -> absent (return 0). */
static int refract(v3 d, v3 n, double eta, v3* out) {
  double ci = -dot(d, n);
  double sin2t = eta * eta * (1.0 - ci * ci);
  if (sin2t > 1.0) return 0;
  double ct = sqrt(1.0 - sin2t);
  *out = normalize(add(scl(d, eta), scl(n, eta * ci - ct)));
  return 1;
}

void orc_reflect(const double d[3], const double n[3], double out[3]) {
  st3(out, reflect(ldd(d), ldd(n)));
}

int orc_refract(const double d[3], const double n[3], double eta, double out[3]) {
  v3 r;
  if (!refract(ldd(d), ldd(n), eta, &r)) return 0;
  st3(out, r);
  return 1;
}

/* ----------------------------------------------------------------------------------------
 * Radiometry (Eq. 3, 5-7)
 * -------------------------------------------------------------------------------------- */

/* ----------------------------------------------------------------------------------------
 * Light-surface and diffuse-bounce sampling
 * -------------------------------------------------------------------------------------- */

/* sample_light_point (Fig. 2 "sampling points on the surface of light source"):
 * uniform on the whole sphere: cos(theta) = 1 - 2 u1, phi = 2 pi u2, pole = +z. */
double orc_sample_sphere(const double c[3], double r, double u1, double u2, double x[3],
                         double nl[3]) {
  double ct = 1.0 - 2.0 * u1;
  double st = sqrt(fmax(0.0, 1.0 - ct * ct));
  double ph = 2.0 * PI * u2;
  nl[0] = st * cos(ph);
  nl[1] = st * sin(ph);
  nl[2] = ct;
  for (int i = 0; i < 3; ++i) x[i] = c[i] + r * nl[i];
  return 1.0 / (4.0 * PI * r * r);
}

/* Orthonormal basis of unit n (Duff et al. 2017, "Building an Orthonormal Basis, Revisited"):
 * s = sign(n.z) (sign(-0) = -1), a = -1 / (s + n.z), b = n.x n.y a,
 * t1 = (1 + s n.x^2 a, s b, -s n.x), t2 = (b, s + n.y^2 a, -n.y). */
void orc_onb(const double n[3], double t1[3], double t2[3]) {
  double sg = copysign(1.0, n[2]);
  double a = -1.0 / (sg + n[2]);
  double b = n[0] * n[1] * a;
  t1[0] = 1.0 + sg * n[0] * n[0] * a; t1[1] = sg * b; t1[2] = -sg * n[0];
  t2[0] = b; t2[1] = sg + n[1] * n[1] * a; t2[2] = -n[1];
}

/* cosine_weighted_direction: pdf cos(theta)/pi about n. */
void orc_cosine_direction(const double n[3], double u1, double u2, double out[3]) {
  double t1[3], t2[3];
  orc_onb(n, t1, t2);
  double rr = sqrt(u1), ph = 2.0 * PI * u2;
  double lx = rr * cos(ph), ly = rr * sin(ph), lz = sqrt(fmax(0.0, 1.0 - u1));
  for (int i = 0; i < 3; ++i) out[i] = t1[i] * lx + t2[i] * ly + n[i] * lz;
}

/* f_r (Eq. 5): DIFFUSE = rho/pi + normalised Phong ks (s+2)/(2 pi) max(0, r.wo)^s with
 * r = 2 (n.wi) n - wi (reading R#3); delta materials -> 0. */
void orc_brdf(int32_t kind, const double albedo[3], double ks, double shininess,
              const double wi_[3], const double wo_[3], const double n_[3], double f[3]) {
  if (kind != 0) { f[0] = f[1] = f[2] = 0.0; return; }
  v3 wi = ldd(wi_), wo = ldd(wo_), n = ldd(n_);
  v3 rl = sub(scl(n, 2.0 * dot(n, wi)), wi);
  double alpha = dot(rl, wo);
  if (alpha < 0.0) alpha = 0.0;
  double spec = ks * (shininess + 2.0) / (2.0 * PI) * pow(alpha, shininess);
  for (int i = 0; i < 3; ++i) f[i] = albedo[i] / PI + spec;
}

/* Schlick's approximation F = R0 + (1 - R0)(1 - c)^5, R0 = ((1 - ior)/(1 + ior))^2. */
double orc_schlick(double ior, double c) {
  double r0 = (1.0 - ior) / (1.0 + ior);
  r0 = r0 * r0;
  double m = 1.0 - c;
  return r0 + (1.0 - r0) * m * m * m * m * m;
}

/* ----------------------------------------------------------------------------------------
 * RNG (§8(c).1 step 9) — exact 64-bit integer arithmetic.
 * -------------------------------------------------------------------------------------- */
#define GOLDEN 0x9E3779B97F4A7C15ULL

uint64_t orc_mix64(uint64_t x) { /* splitmix64 finalizer */
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27; x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

double orc_rng(uint64_t seed, uint64_t pixel_index, uint32_t sample, uint32_t depth) {
  uint64_t x = seed ^ ((pixel_index + 1ULL) * GOLDEN);
  x = orc_mix64(x);
  x = orc_mix64(x ^ ((((uint64_t)sample << 32) + (uint64_t)depth) * GOLDEN));
  return (double)(x >> 40) * (1.0 / 16777216.0); /* exact in float and double */
}

/* Further draws of the same (pixel, sample, depth): stream k in bits 8..31 of the counter
 * word (reading R#42); k = 0 reproduces orc_rng. */
double orc_rng_stream(uint64_t seed, uint64_t pixel_index, uint32_t sample, uint32_t depth,
                      uint32_t stream) {
  uint64_t x = seed ^ ((pixel_index + 1ULL) * GOLDEN);
  x = orc_mix64(x);
  uint64_t word = ((uint64_t)sample << 32) + ((uint64_t)stream << 8) + (uint64_t)depth;
  x = orc_mix64(x ^ (word * GOLDEN));
  return (double)(x >> 40) * (1.0 / 16777216.0);
}

/* ----------------------------------------------------------------------------------------
 * Camera (§8(c).1 steps 1-2)
 * -------------------------------------------------------------------------------------- */

/* Sub-pixel sample positions (reading R#19): stratified n x n grid when spp = n^2, else the
 * shifted Hammersley point ((s + 1/2)/spp, frac(radinv2(s) + 1/(2 spp))). */
void orc_sample_offset(int32_t s, int32_t spp, double* ox, double* oy) {
  int32_t n = 1;
  while ((n + 1) * (n + 1) <= spp) ++n;
  if (n * n == spp) {
    int32_t i = s % n, j = s / n;
    *ox = (i + 0.5) / n;
    *oy = (j + 0.5) / n;
    return;
  }
  uint32_t bits = (uint32_t)s, rev = 0;
  for (int k = 0; k < 32; ++k) { rev = (rev << 1) | (bits & 1u); bits >>= 1; }
  double radinv = (double)rev / 4294967296.0;
  double y = radinv + 0.5 / spp;
  *ox = (s + 0.5) / spp;
  *oy = y - floor(y);
}

typedef struct { v3 eye, f, r, u; double h; } camera;

static camera build_camera(const orc_scene* sc) {
  camera cam;
  cam.eye = ld3(sc->eye);
  cam.f = normalize(sub(ld3(sc->look_at), cam.eye)); /* forward */
  cam.r = normalize(cross(cam.f, ld3(sc->up)));      /* right = normalize(forward x up) */
  cam.u = cross(cam.r, cam.f);                       /* up' = right x forward */
  cam.h = tan(0.5 * (double)sc->vfov_deg * PI / 180.0);
  return cam;
}

/* generate_camera_ray: pinhole, vertical fov, aspect W/H, py = 0 is the top row. */
static void camera_ray_at(const camera* cam, int32_t W, int32_t H, int32_t px, int32_t py,
                          double ox, double oy, v3* o, v3* d) {
  double sx = (px + ox) / W, sy = (py + oy) / H;
  double aspect = (double)W / (double)H;
  v3 dir = add(cam->f, add(scl(cam->r, (2.0 * sx - 1.0) * cam->h * aspect),
                           scl(cam->u, (1.0 - 2.0 * sy) * cam->h)));
  *o = cam->eye;
  *d = normalize(dir);
}

static void camera_ray(const camera* cam, int32_t W, int32_t H, int32_t px, int32_t py,
                       int32_t s, int32_t spp, v3* o, v3* d) {
  double ox, oy;
  orc_sample_offset(s, spp, &ox, &oy);
  camera_ray_at(cam, W, H, px, py, ox, oy, o, d);
}

void orc_camera_ray(const orc_scene* scene, int32_t width, int32_t height, int32_t px,
                    int32_t py, int32_t s, int32_t spp, double o[3], double d[3]) {
  camera cam = build_camera(scene);
  v3 oo, dd;
  camera_ray(&cam, width, height, px, py, s, spp, &oo, &dd);
  st3(o, oo);
  st3(d, dd);
}

/* tone_map: clamp(exposure v, 0, 1)^(1/gamma) * 255, rounded half-up. */
int32_t orc_tonemap8(double v, double exposure, double gamma) {
  double x = exposure * v;
  if (!(x > 0.0)) x = 0.0;
  if (x > 1.0) x = 1.0;
  return (int32_t)floor(255.0 * pow(x, 1.0 / gamma) + 0.5);
}

/* ----------------------------------------------------------------------------------------
 * Scene access
 * -------------------------------------------------------------------------------------- */
typedef struct {
  const orc_scene* sc;
  int n;
  int n_spheres, n_planes;
  int* type;
  int* mat;
  v3* c;      /* sphere centre, or plane normal */
  double* r;  /* sphere radius, or plane d */
  double* cn; /* |centre| (classification scales) */
  int n_emit;     /* emissive spheres, in prim index order (R#41) */
  int* emit;      /* [n_emit] prim index */
} prims;

static void prims_load(prims* P, const orc_scene* sc) {
  P->sc = sc;
  P->n = sc->n_prims;
  P->n_spheres = P->n_planes = 0;
  P->type = (int*)malloc(sizeof(int) * (P->n + 1));
  P->mat = (int*)malloc(sizeof(int) * (P->n + 1));
  P->c = (v3*)malloc(sizeof(v3) * (P->n + 1));
  P->r = (double*)malloc(sizeof(double) * (P->n + 1));
  P->cn = (double*)malloc(sizeof(double) * (P->n + 1));
  for (int k = 0; k < P->n; ++k) {
    const float* p = sc->prim_p + 4 * k;
    P->type[k] = sc->prim_type[k];
    P->mat[k] = sc->prim_mat[k];
    if (P->type[k] == 1) {
      v3 nn = ld3(p);
      double l = len(nn);
      P->c[k] = scl(nn, 1.0 / l);      /* normalised on load, n.x = d scaled alike */
      P->r[k] = (double)p[3] / l;
      P->cn[k] = fabs(P->r[k]);
      P->n_planes++;
    } else {
      P->c[k] = ld3(p);
      P->r[k] = (double)p[3];
      P->cn[k] = len(P->c[k]);
      P->n_spheres++;
    }
  }
  P->n_emit = 0;
  P->emit = (int*)malloc(sizeof(int) * (P->n + 1));
  for (int k = 0; k < P->n; ++k) {
    const float* le = sc->mat_emission + 3 * P->mat[k];
    if (P->type[k] == 0 && (le[0] > 0.0f || le[1] > 0.0f || le[2] > 0.0f)) P->emit[P->n_emit++] = k;
  }
}

static void prims_free(prims* P) {
  free(P->type); free(P->mat); free(P->c); free(P->r); free(P->cn); free(P->emit);
}

static int prim_hit(const prims* P, int k, v3 o, v3 d, double* t) {
  if (P->type[k] == 1) return plane_hit(o, d, P->c[k], P->r[k], t);
  return sphere_hit(o, d, P->c[k], P->r[k], t);
}

/* ----------------------------------------------------------------------------------------
 * Classification (NOT the method): normalised decision margins, DESIGN.md "Parity rule".
 * Every margin is slack / E, where E is the first-order absolute error scale of the decision
 * for a unit relative perturbation of the float inputs and of every intermediate point
 * (position scale Ps in scene units, direction scale Ad in radians).
 * -------------------------------------------------------------------------------------- */
static double fmin2(double a, double b) { return a < b ? a : b; }

/* closest-hit decisions of one segment: grazing silhouettes, EPS_T acceptance, t ordering */
static double closest_margin(const prims* P, v3 o, v3 d, double Ps, double Ad, int self,
                             int self_inside, int best, double tbest) {
  double m = INFINITY;
  double cos_best = 1.0;
  if (best >= 0) {
    if (P->type[best] == 1) cos_best = fabs(dot(P->c[best], d));
    else {
      v3 p = add(o, scl(d, tbest));
      cos_best = fabs(dot(sub(p, P->c[best]), d)) / P->r[best];
    }
    if (cos_best < 1e-9) cos_best = 1e-9;
  }
  for (int k = 0; k < P->n; ++k) {
    if (P->type[k] == 1) {
      double den = dot(P->c[k], d);
      if (fabs(den) < 1e-12) continue;
      double t = (P->r[k] - dot(P->c[k], o)) / den;
      double E = Ps + fabs(t) * Ad + P->cn[k] + 1.0;
      if (k == self) continue; /* leaving this plane: never re-hit */
      m = fmin2(m, fabs(t - EPS_T) / (E / fabs(den)));
      if (t >= EPS_T && k != best && best >= 0) {
        double Et = E / fabs(den) + (Ps + tbest * Ad + P->cn[best] + 1.0) / cos_best;
        m = fmin2(m, fabs(t - tbest) / Et);
      }
      continue;
    }
    v3 c = P->c[k];
    double r = P->r[k];
    v3 oc = sub(o, c);
    double b = dot(oc, d);
    double tc = -b; /* parameter of closest approach */
    v3 perp = sub(oc, scl(d, b));
    double dp = len(perp);
    double E = Ps + fabs(tc) * Ad + P->cn[k] + 1.0;
    double t0, t1;
    int has = sphere_roots(o, d, c, r, &t0, &t1);
    if (k == self) {
      if (self_inside && has) m = fmin2(m, fabs(t1 - EPS_T) / E);
      if (self_inside && has && k != best && best >= 0) {
        double cosk = sqrt(fmax(r * r - dp * dp, 0.0)) / r;
        if (cosk < 1e-9) cosk = 1e-9;
        double Et = E / cosk + (Ps + tbest * Ad + P->cn[best] + 1.0) / cos_best;
        m = fmin2(m, fabs(t1 - tbest) / Et);
      }
      continue;
    }
    /* grazing: the line passes within the silhouette band of a sphere that is in play */
    if (tc + r >= 0.0 && tc - r <= tbest) m = fmin2(m, fabs(r - dp) / E);
    if (!has) continue;
    double cosk = sqrt(fmax(r * r - dp * dp, 0.0)) / r;
    if (cosk < 1e-9) cosk = 1e-9;
    m = fmin2(m, fabs(t0 - EPS_T) / (E / cosk));
    m = fmin2(m, fabs(t1 - EPS_T) / (E / cosk));
    double tsel = t0 >= EPS_T ? t0 : t1;
    if (tsel >= EPS_T && k != best && best >= 0) {
      double Et = E / cosk + (Ps + tbest * Ad + P->cn[best] + 1.0) / cos_best;
      m = fmin2(m, fabs(tsel - tbest) / Et);
    }
  }
  return m;
}

/* robustness of one prim's occlusion decision on the shadow segment [EPS_T, tmax) */
static double shadow_prim_margin(const prims* P, int k, v3 o, v3 d, double tmax, double Ps,
                                 double Ad, double El, int* occludes) {
  *occludes = 0;
  double m = INFINITY;
  if (P->type[k] == 1) {
    double den = dot(P->c[k], d);
    if (fabs(den) < 1e-12) return INFINITY;
    double t = (P->r[k] - dot(P->c[k], o)) / den;
    double Et = (Ps + fabs(t) * Ad + P->cn[k] + 1.0) / fabs(den);
    *occludes = (t >= EPS_T && t < tmax);
    m = fmin2(m, fabs(t - EPS_T) / Et);
    m = fmin2(m, fabs(t - tmax) / (Et + El));
    return m;
  }
  v3 c = P->c[k];
  double r = P->r[k];
  v3 oc = sub(o, c);
  double b = dot(oc, d);
  double tc = -b;
  double dp = len(sub(oc, scl(d, b)));
  double E = Ps + fabs(tc) * Ad + P->cn[k] + 1.0;
  if (tc + r >= 0.0 && tc - r <= tmax) m = fmin2(m, fabs(r - dp) / E);
  double t0, t1;
  if (sphere_roots(o, d, c, r, &t0, &t1)) {
    double cosk = sqrt(fmax(r * r - dp * dp, 0.0)) / r;
    if (cosk < 1e-9) cosk = 1e-9;
    double Et = E / cosk;
    double tsel = t0 >= EPS_T ? t0 : t1;
    *occludes = (tsel >= EPS_T && tsel < tmax);
    m = fmin2(m, fabs(t0 - EPS_T) / Et);
    m = fmin2(m, fabs(t1 - EPS_T) / Et);
    m = fmin2(m, fabs(t0 - tmax) / (Et + El));
    m = fmin2(m, fabs(t1 - tmax) / (Et + El));
  }
  return m;
}

/* Occluded -> robust if at least one occluder is robust; visible -> robust if every prim is. */
static double shadow_margin(const prims* P, v3 o, v3 d, double tmax, double Ps, double Ad,
                            double El, int self, int self_inside, int emitter) {
  double m_vis = INFINITY, m_occ = 0.0;
  int any = 0;
  for (int k = 0; k < P->n; ++k) {
    if (k == self && !self_inside) continue;
    if (k == emitter) continue; /* the sampled emitter never blocks its own sample (R#41) */
    int occ;
    double mk_ = shadow_prim_margin(P, k, o, d, tmax, Ps, Ad, El, &occ);
    if (occ) { any = 1; if (mk_ > m_occ) m_occ = mk_; }
    else m_vis = fmin2(m_vis, mk_);
  }
  return any ? m_occ : m_vis;
}

/* Monte Carlo arithmetic perturbation of a vector (classification replicas only). */
static v3 perturb_v3(v3 a, double u, uint64_t key) {
  double q[3] = {a.x, a.y, a.z};
  for (int i = 0; i < 3; ++i) {
    uint64_t h = orc_mix64(key + (uint64_t)(i + 1) * GOLDEN);
    double z = (double)(h >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
    q[i] *= (1.0 + u * z);
  }
  return mk(q[0], q[1], q[2]);
}

/* ----------------------------------------------------------------------------------------
 * The method: one sample path (§8(c).1 steps 2-9; Alg. 1; §IV.A)
 * -------------------------------------------------------------------------------------- */
typedef struct {
  double L[3];
  int bounces;
  double margin;
} sample_result;

static sample_result trace_sample(const prims* P, const camera* cam, const orc_frame* fr,
                                  int32_t px, int32_t py, int32_t s, int32_t* hit_ids,
                                  int want_margin, orc_counts* cnt) {
  const orc_scene* sc = P->sc;
  sample_result res;
  uint64_t pixel_index = (uint64_t)py * (uint64_t)fr->width + (uint64_t)px;
  /* the sample's global index keys every random draw (progressive passes, R#42) */
  const uint32_t sg = (uint32_t)(fr->sample_base + s);
  v3 o, d;
  if (fr->jitter) { /* random sub-pixel offset from streams 1, 2 (R#42) */
    double ox = orc_rng_stream(fr->seed, pixel_index, sg, 0, 1);
    double oy = orc_rng_stream(fr->seed, pixel_index, sg, 0, 2);
    camera_ray_at(cam, fr->width, fr->height, px, py, ox, oy, &o, &d); /* step 2 */
  } else {
    camera_ray(cam, fr->width, fr->height, px, py, s, fr->spp, &o, &d); /* step 2 */
  }
  int prev_diffuse = 0; /* the current ray left a DIFFUSE hit by a cosine-weighted bounce */
  v3 T = mk(1, 1, 1);  /* throughput */
  v3 L = mk(0, 0, 0);  /* radiance */
  v3 bg = ld3(sc->background), amb = ld3(sc->ambient);
  int bounces = 0;
  cnt->primary++;

  /* classification state */
  double margin = INFINITY;
  double Ps = len(o) + 1.0, Ad = 1.0;
  int self = -1, self_inside = 0;
  uint64_t pkey = fr->perturb_seed ^ orc_mix64(pixel_index * 0x100000001B3ULL + (uint64_t)sg);

  for (int depth = 0; depth <= fr->max_depth; ++depth) {
    if (hit_ids) hit_ids[depth] = -1;
    if (fr->perturb > 0.0) {
      o = perturb_v3(o, fr->perturb, pkey + 2 * depth);
      d = normalize(perturb_v3(d, fr->perturb, pkey + 2 * depth + 1));
    }
    /* step 3: nearest hit, index order, strict < so ties go to the lowest index */
    int best = -1;
    double tbest = INFINITY;
    for (int k = 0; k < P->n; ++k) {
      double t;
      if (prim_hit(P, k, o, d, &t) && t < tbest) { tbest = t; best = k; }
    }
    cnt->sphere_tests += (uint64_t)P->n_spheres;
    cnt->plane_tests += (uint64_t)P->n_planes;
    if (want_margin)
      margin = fmin2(margin, closest_margin(P, o, d, Ps, Ad, self, self_inside, best, tbest));

    /* step 4: miss -> background */
    if (best < 0) { L = add(L, mulv(T, bg)); break; }
    if (hit_ids) hit_ids[depth] = best;

    /* step 5: hit geometry, normal flipped to oppose the ray */
    v3 p = add(o, scl(d, tbest));
    v3 ng = P->type[best] == 1 ? P->c[best] : scl(sub(p, P->c[best]), 1.0 / P->r[best]);
    int entering = dot(d, ng) < 0.0;
    v3 n = entering ? ng : scl(ng, -1.0);
    v3 wo = scl(d, -1.0);
    int mi = P->mat[best];
    int kind = sc->mat_kind[mi];
    v3 rho = ld3(sc->mat_albedo + 3 * mi);
    double Phit = Ps + tbest * Ad + len(p) + 1.0;
    double An = P->type[best] == 1 ? 1.0 : (Phit + P->cn[best]) / P->r[best];

    /* step 6: emission at every hit (Eq. 7; reading R#6) — except an
     * emitter that next-event estimation already sampled from the previous diffuse bounce
     * (S:299 double-count rule; R#43) */
    {
      int sampled_emitter = 0;
      if (fr->area_lights && prev_diffuse)
        for (int e = 0; e < P->n_emit; ++e) sampled_emitter |= (P->emit[e] == best);
      if (!sampled_emitter) L = add(L, mulv(T, ld3(sc->mat_emission + 3 * mi)));
    }

    /* step 7: direct lighting at DIFFUSE hits (Alg. 1; Eq. 3, 5, 6) */
    if (kind == 0) {
      L = add(L, mulv(T, mulv(rho, amb))); /* ambient, unshadowed (reading R#4) */
      for (int l = 0; l < sc->n_lights; ++l) {
        v3 Pl = ld3(sc->light_pos + 3 * l);
        v3 w = sub(Pl, p);
        double d2 = dot(w, w);
        if (d2 < 1e-12) continue; /* reading R#28 */
        v3 wi = scl(w, 1.0 / sqrt(d2));
        double cos_t = dot(n, wi);
        double El = len(Pl) + 1.0;
        margin = fmin2(margin, fabs(cos_t) / (An + (Phit + El) / sqrt(d2)));
        if (cos_t <= 0.0) continue; /* no shadow ray */
        /* shadow ray from p + EPS_T n toward the light, "emit a shadow light r" */
        v3 os = add(p, scl(n, EPS_T));
        v3 ws = sub(Pl, os);
        double tmax = len(ws);
        v3 ds = scl(ws, 1.0 / tmax);
        if (fr->perturb > 0.0) {
          uint64_t key = pkey + 0x51ED27ULL * (uint64_t)(depth * 64 + l + 1);
          os = perturb_v3(os, fr->perturb, key);
          ds = normalize(perturb_v3(ds, fr->perturb, key + 7));
        }
        cnt->shadow++;
        int occluded = 0;
        for (int k = 0; k < P->n; ++k) { /* Alg. 1 lines 6-11: break at the first occluder */
          double t;
          if (P->type[k] == 1) cnt->plane_tests++; else cnt->sphere_tests++;
          if (prim_hit(P, k, os, ds, &t) && t < tmax) { occluded = 1; break; }
        }
        if (want_margin) {
          int self_in = (P->type[best] == 0) && !entering; /* shading from inside a sphere */
          margin = fmin2(margin, shadow_margin(P, os, ds, tmax, Phit + EPS_T, (Phit + El) / tmax,
                                               El, best, self_in, -1));
        }
        if (!occluded) {
          double f[3], wi_a[3], wo_a[3], n_a[3], alb[3];
          st3(wi_a, wi); st3(wo_a, wo); st3(n_a, n); st3(alb, rho);
          orc_brdf(kind, alb, (double)sc->mat_ks[mi], (double)sc->mat_shininess[mi], wi_a, wo_a,
                   n_a, f);
          v3 I = ld3(sc->light_intensity + 3 * l);
          double g = cos_t / d2; /* Eq. 3 for a point source: E = I cos(theta) / d^2 */
          L = add(L, mulv(T, scl(mulv(mk(f[0], f[1], f[2]), I), g)));
        }
      }
      /* spherical area lights (NEXT-1; Eq. 8 as a one-sample estimator, Fig. 2):
       * one uniform surface point per emitter, in emitter order after the point lights */
      for (int e = 0; fr->area_lights && e < P->n_emit; ++e) {
        int ke = P->emit[e];
        double u1 = orc_rng_stream(fr->seed, pixel_index, sg, (uint32_t)depth, 5u + 2u * e);
        double u2 = orc_rng_stream(fr->seed, pixel_index, sg, (uint32_t)depth, 6u + 2u * e);
        double ca[3], xa[3], nla[3];
        st3(ca, P->c[ke]);
        double pdf = orc_sample_sphere(ca, P->r[ke], u1, u2, xa, nla);
        v3 X = ldd(xa), NL = ldd(nla);
        v3 w = sub(X, p);
        double d2 = dot(w, w);
        if (d2 < 1e-12) continue;
        v3 wi = scl(w, 1.0 / sqrt(d2));
        double cos_s = dot(n, wi);      /* cos(theta) at the shading point (Eq. 3) */
        double cos_l = -dot(wi, NL);    /* cos(theta) at the light sample */
        double El = len(X) + 1.0;
        margin = fmin2(margin, fabs(cos_s) / (An + (Phit + El) / sqrt(d2)));
        margin = fmin2(margin, fabs(cos_l) / (1.0 + (Phit + El) / sqrt(d2)));
        if (cos_s <= 0.0 || cos_l <= 0.0) continue; /* no shadow ray (S:160 analogue) */
        v3 os = add(p, scl(n, EPS_T));
        v3 ws = sub(X, os);
        double tmax = len(ws);
        v3 ds = scl(ws, 1.0 / tmax);
        if (fr->perturb > 0.0) {
          uint64_t key = pkey + 0xA5E1ULL * (uint64_t)(depth * 4096 + e + 1);
          os = perturb_v3(os, fr->perturb, key);
          ds = normalize(perturb_v3(ds, fr->perturb, key + 7));
        }
        cnt->shadow++;
        int occluded = 0;
        for (int k = 0; k < P->n; ++k) { /* index order, break at the first occluder */
          double t;
          if (k == ke) continue; /* the emitter itself is not tested (S:174 ledger) */
          if (P->type[k] == 1) cnt->plane_tests++; else cnt->sphere_tests++;
          if (prim_hit(P, k, os, ds, &t) && t < tmax) { occluded = 1; break; }
        }
        if (want_margin) {
          int self_in = (P->type[best] == 0) && !entering;
          margin = fmin2(margin, shadow_margin(P, os, ds, tmax, Phit + EPS_T, (Phit + El) / tmax,
                                               El, best, self_in, ke));
        }
        if (!occluded) {
          double f[3], wi_a[3], wo_a[3], n_a[3], alb[3];
          st3(wi_a, wi); st3(wo_a, wo); st3(n_a, n); st3(alb, rho);
          orc_brdf(kind, alb, (double)sc->mat_ks[mi], (double)sc->mat_shininess[mi], wi_a, wo_a,
                   n_a, f);
          v3 Le = ld3(sc->mat_emission + 3 * P->mat[ke]);
          double g = cos_s * cos_l / (d2 * pdf); /* f L_e cos_s cos_l / (dist^2 pdf_area) */
          L = add(L, mulv(T, scl(mulv(mk(f[0], f[1], f[2]), Le), g)));
        }
      }
    }

    /* step 8: stack-free continuation */
    if (depth == fr->max_depth) break;
    v3 dn;
    double An_next;
    if (kind == 1) { /* SPECULAR: mirror, T *= rho */
      dn = reflect(d, n);
      T = mulv(T, rho);
      An_next = Ad + 2.0 * An;
    } else if (kind == 0 && fr->integrator == 1) { /* global: cosine-weighted (NEXT-2, R#40) */
      double u1 = orc_rng_stream(fr->seed, pixel_index, sg, (uint32_t)depth, 3u);
      double u2 = orc_rng_stream(fr->seed, pixel_index, sg, (uint32_t)depth, 4u);
      double n_a[3], dn_a[3];
      st3(n_a, n);
      /* sign(n.z) selects the basis branch: a decision for a sphere normal; a plane's normal is
       * exact on both sides (normalised from the same floats), signed zero included */
      if (P->type[best] == 0) margin = fmin2(margin, fabs(n.z) / An);
      orc_cosine_direction(n_a, u1, u2, dn_a);
      dn = ldd(dn_a);
      T = mulv(T, rho); /* f_r cos / pdf = albedo */
      An_next = Ad + 2.0 * An;
    } else if (kind == 0) { /* DIFFUSE: mirror iff kr > 0 (reading R#8) */
      double kr = (double)sc->mat_kr[mi];
      if (!(kr > 0.0)) break;
      dn = reflect(d, n);
      T = scl(T, kr);
      An_next = Ad + 2.0 * An;
    } else { /* REFRACTIVE: Schlick-chosen reflect/refract, TIR -> reflect (R#9-R#11) */
      double ior = (double)sc->mat_ior[mi];
      double eta = entering ? 1.0 / ior : ior;
      double ci = -dot(d, n);
      double sin2t = eta * eta * (1.0 - ci * ci);
      margin = fmin2(margin, fabs(1.0 - sin2t) / (2.0 * eta * eta * (Ad + An)));
      if (sin2t > 1.0) {
        dn = reflect(d, n);
      } else {
        double c = entering ? ci : sqrt(1.0 - sin2t);
        double F = orc_schlick(ior, c);
        double u = orc_rng(fr->seed, pixel_index, sg, (uint32_t)depth);
        margin = fmin2(margin, fabs(u - F) / (5.0 * (Ad + An)));
        if (u < F) dn = reflect(d, n);
        else refract(d, n, eta, &dn);
      }
      T = mulv(T, rho);
      An_next = eta * Ad + 2.0 * (1.0 + eta) * An;
    }
    /* new ray: o' = p (no offset; EPS_T rejects self hits), d' normalised */
    o = p;
    d = normalize(dn);
    prev_diffuse = (kind == 0 && fr->integrator == 1);
    bounces++;
    cnt->secondary++;
    self = best;
    /* the new ray is inside its origin sphere iff it points against the outward normal */
    self_inside = (P->type[best] == 0) && (dot(d, ng) < 0.0);
    Ps = Phit;
    Ad = An_next;
  }
  res.L[0] = L.x; res.L[1] = L.y; res.L[2] = L.z;
  res.bounces = bounces;
  res.margin = margin;
  return res;
}

int orc_render(const orc_scene* scene, const orc_frame* frame, const int64_t* pixels,
               int64_t n_pixels, double* rgb, int32_t* hit_ids, int32_t* bounces,
               double* margin, double* sample_rgb, orc_counts* counts) {
  if (!scene || !frame || frame->width < 1 || frame->height < 1 || frame->max_depth < 0 ||
      frame->spp < 1 || frame->max_depth > 255 || frame->sample_base < 0 ||
      frame->sample_base + frame->spp > 4294967296LL)
    return -1;
  int64_t npx_total = (int64_t)frame->width * frame->height;
  if (!pixels) n_pixels = npx_total;
  orc_counts cnt;
  memset(&cnt, 0, sizeof(cnt));
  prims P;
  prims_load(&P, scene);
  camera cam = build_camera(scene);
  const int D = frame->max_depth + 1;
  for (int64_t i = 0; i < n_pixels; ++i) {
    int64_t pix = pixels ? pixels[i] : i;
    if (pix < 0 || pix >= npx_total) { prims_free(&P); return -1; }
    int32_t px = (int32_t)(pix % frame->width), py = (int32_t)(pix / frame->width);
    double acc[3] = {0, 0, 0};
    for (int32_t s = 0; s < frame->spp; ++s) { /* samples summed in order s = 0..spp-1 */
      int64_t si = i * frame->spp + s;
      int32_t* ids = hit_ids ? hit_ids + si * D : NULL;
      if (ids) for (int k = 0; k < D; ++k) ids[k] = -2;
      sample_result r = trace_sample(&P, &cam, frame, px, py, s, ids, margin != NULL, &cnt);
      for (int c = 0; c < 3; ++c) acc[c] += r.L[c];
      if (bounces) bounces[si] = r.bounces;
      if (margin) margin[si] = r.margin;
      if (sample_rgb) for (int c = 0; c < 3; ++c) sample_rgb[3 * si + c] = r.L[c];
    }
    if (rgb) for (int c = 0; c < 3; ++c) rgb[3 * i + c] = acc[c] / frame->spp; /* step 10 */
  }
  prims_free(&P);
  if (counts) *counts = cnt;
  return 0;
}

/* ----------------------------------------------------------------------------------------
 * NEXT-3: the literal Alg. 1 light-grid form. Test infrastructure that
 * cross-checks the one-sample estimator of trace_sample (NEXT-1) against the paper's serial
 * quadrature over "each sampling point of each source light".
 * -------------------------------------------------------------------------------------- */
int orc_render_local_grid(const orc_scene* scene, int32_t width, int32_t height, int32_t light_grid,
                          int32_t rays_per_pixel, double* rgb) {
  if (!scene || !rgb || width < 1 || height < 1 || light_grid < 1 || rays_per_pixel < 1) return -1;
  prims P;
  prims_load(&P, scene);
  camera cam = build_camera(scene);
  const int n = light_grid;
  for (int32_t py = 0; py < height; ++py) {
    for (int32_t px = 0; px < width; ++px) {
      v3 acc = mk(0, 0, 0);
      for (int32_t s = 0; s < rays_per_pixel; ++s) { /* Alg. 1 line 1: each light of each pixel */
        v3 o, d;
        camera_ray(&cam, width, height, px, py, s, rays_per_pixel, &o, &d);
        int best = -1; /* lines 2-3: each object, nearest intersection */
        double tbest = INFINITY;
        for (int k = 0; k < P.n; ++k) {
          double t;
          if (prim_hit(&P, k, o, d, &t) && t < tbest) { tbest = t; best = k; }
        }
        v3 col = mk(0, 0, 0);
        if (best < 0) {
          col = ld3(scene->background);
        } else {
          v3 p = add(o, scl(d, tbest));
          v3 ng = P.type[best] == 1 ? P.c[best] : scl(sub(p, P.c[best]), 1.0 / P.r[best]);
          v3 nrm = dot(d, ng) < 0.0 ? ng : scl(ng, -1.0);
          v3 wo = scl(d, -1.0);
          int mi = P.mat[best];
          int kind = scene->mat_kind[mi];
          v3 rho = ld3(scene->mat_albedo + 3 * mi);
          col = ld3(scene->mat_emission + 3 * mi); /* Eq. 7 */
          if (kind == 0) {
            double f[3], wi_a[3], wo_a[3], n_a[3], alb[3];
            st3(wo_a, wo); st3(n_a, nrm); st3(alb, rho);
            col = add(col, mulv(rho, ld3(scene->ambient)));
            v3 os = add(p, scl(nrm, EPS_T));
            for (int l = 0; l < scene->n_lights; ++l) { /* point lights, as orc_render */
              v3 Pl = ld3(scene->light_pos + 3 * l);
              v3 w = sub(Pl, p);
              double d2 = dot(w, w);
              if (d2 < 1e-12) continue;
              v3 wi = scl(w, 1.0 / sqrt(d2));
              double cs = dot(nrm, wi);
              if (cs <= 0.0) continue;
              v3 ws = sub(Pl, os);
              double tmax = len(ws);
              v3 ds = scl(ws, 1.0 / tmax);
              int occ = 0;
              for (int k = 0; k < P.n; ++k) {
                double t;
                if (prim_hit(&P, k, os, ds, &t) && t < tmax) { occ = 1; break; }
              }
              if (occ) continue;
              st3(wi_a, wi);
              orc_brdf(kind, alb, (double)scene->mat_ks[mi], (double)scene->mat_shininess[mi], wi_a, wo_a, n_a, f);
              col = add(col, scl(mulv(mk(f[0], f[1], f[2]), ld3(scene->light_intensity + 3 * l)), cs / d2));
            }
            for (int e = 0; e < P.n_emit; ++e) { /* line 4: each sampling point of each source light */
              int ke = P.emit[e];
              v3 c = P.c[ke];
              double r = P.r[ke];
              v3 Le = ld3(scene->mat_emission + 3 * P.mat[ke]);
              for (int i = 0; i < n; ++i) {
                double th0 = PI * i / n, th1 = PI * (i + 1) / n, thm = 0.5 * (th0 + th1);
                for (int j = 0; j < n; ++j) {
                  double phm = 2.0 * PI * (j + 0.5) / n;
                  double dA = r * r * (cos(th0) - cos(th1)) * (2.0 * PI / n); /* exact cell area */
                  v3 nl = mk(sin(thm) * cos(phm), sin(thm) * sin(phm), cos(thm));
                  v3 X = add(c, scl(nl, r));
                  v3 w = sub(X, p);
                  double d2 = dot(w, w);
                  if (d2 < 1e-12) continue;
                  v3 wi = scl(w, 1.0 / sqrt(d2));
                  double cs = dot(nrm, wi), cl = -dot(wi, nl);
                  if (cs <= 0.0 || cl <= 0.0) continue;
                  v3 ws = sub(X, os); /* line 5: emit a shadow light r from p to that point */
                  double tmax = len(ws);
                  v3 ds = scl(ws, 1.0 / tmax);
                  int occ = 0;
                  for (int k = 0; k < P.n; ++k) { /* lines 6-11: break at an occluder */
                    double t;
                    if (k == ke) continue;
                    if (prim_hit(&P, k, os, ds, &t) && t < tmax) { occ = 1; break; }
                  }
                  if (occ) continue;
                  st3(wi_a, wi);
                  orc_brdf(kind, alb, (double)scene->mat_ks[mi], (double)scene->mat_shininess[mi], wi_a, wo_a,
                           n_a, f);
                  /* Eq. 8 over the cell, accumulated (line 12) */
                  col = add(col, scl(mulv(mk(f[0], f[1], f[2]), Le), cs * cl / d2 * dA));
                }
              }
            }
          }
        }
        acc = add(acc, col); /* line 16: accumulate the colour of each light */
      }
      st3(rgb + 3 * ((int64_t)py * width + px), scl(acc, 1.0 / rays_per_pixel)); /* line 18: average */
    }
  }
  prims_free(&P);
  return 0;
}

