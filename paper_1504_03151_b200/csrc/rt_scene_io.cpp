// rt_scene_io.cpp — SURVEY §8(f) NEXT-4: scene text parser (extended
// to planes / point lights / environment, grammar in include/rt.h) and the P6 PPM writer (SPEC
// S:487-494). Host code: the parser validates everything before the first device call, then
// hands the arrays to rt_scene_upload / rt_camera_set; the PPM writer tone-maps on the device.
#include <cuda_runtime.h>

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rt.h"
#include "rt_internal.h"

namespace {

struct Parsed {
  std::vector<rt_primitive> prims;
  std::vector<rt_material> mats;
  std::vector<rt_light> lights;
  rt_env env{};
  bool has_camera = false;
  int camera_line = 0;
  float eye[3], look[3], up[3], vfov = 0.f;
};

int perr(int line, std::string why) {
  for (char& ch : why)  // the message quotes input bytes: keep it printable ASCII
    if ((unsigned char)ch < 0x20 || (unsigned char)ch > 0x7e) ch = '?';
  char buf[400];
  snprintf(buf, sizeof buf, "line %d: %s", line, why.c_str());
  return rt_fail(RT_ERR_PARSE, buf);
}

// one whitespace-separated field as a finite float32 (the whole token must be consumed)
bool to_float(const std::string& tok, float& out) {
  if (tok.empty() || tok.size() > 64) return false;
  char* end = nullptr;
  errno = 0;
  const float v = std::strtof(tok.c_str(), &end);
  if (end != tok.c_str() + tok.size() || !std::isfinite(v)) return false;
  out = v;
  return true;
}

int parse_kind(const std::string& t) {
  if (t == "diffuse") return RT_MAT_DIFFUSE;
  if (t == "specular") return RT_MAT_SPECULAR;
  if (t == "refractive") return RT_MAT_REFRACTIVE;
  return -1;
}

// fields f[first ..] = er eg eb ar ag ab kind [ior] [ks= shininess= kr=] -> material
int parse_material(const std::vector<std::string>& f, size_t first, int line, rt_material& m) {
  if (f.size() < first + 7) return perr(line, "bad arity: expected emission (3), albedo (3) and a kind");
  float v[6];
  for (int i = 0; i < 6; ++i)
    if (!to_float(f[first + i], v[i])) return perr(line, "non-numeric field '" + f[first + i] + "'");
  std::memset(&m, 0, sizeof m);
  for (int i = 0; i < 3; ++i) {
    m.emission[i] = v[i];
    m.albedo[i] = v[3 + i];
    if (!(v[i] >= 0.f)) return perr(line, "emission must be >= 0");
    if (!(v[3 + i] >= 0.f && v[3 + i] <= 1.f)) return perr(line, "albedo outside [0,1]");
  }
  const int kind = parse_kind(f[first + 6]);
  if (kind < 0) return perr(line, "unknown kind '" + f[first + 6] + "' (diffuse, specular, refractive)");
  m.kind = (uint32_t)kind;
  m.ior = 1.5f;
  m.ks = 0.f;
  m.shininess = 1.f;
  m.kr = 0.f;
  size_t i = first + 7;
  if (kind == RT_MAT_REFRACTIVE && i < f.size() && f[i].find('=') == std::string::npos) {
    if (!to_float(f[i], m.ior)) return perr(line, "non-numeric ior '" + f[i] + "'");
    if (!(m.ior >= 1.f)) return perr(line, "ior must be >= 1");
    ++i;
  }
  for (; i < f.size(); ++i) {
    const size_t eq = f[i].find('=');
    if (eq == std::string::npos) return perr(line, "bad arity: unexpected field '" + f[i] + "'");
    const std::string key = f[i].substr(0, eq), val = f[i].substr(eq + 1);
    float x;
    if (!to_float(val, x)) return perr(line, "non-numeric option value '" + f[i] + "'");
    if (key == "ks") {
      if (!(x >= 0.f && x <= 1.f)) return perr(line, "ks outside [0,1]");
      m.ks = x;
    } else if (key == "shininess") {
      if (!(x >= 1.f && x <= 1e4f)) return perr(line, "shininess outside [1,1e4]");
      m.shininess = x;
    } else if (key == "kr") {
      if (!(x >= 0.f && x <= 1.f)) return perr(line, "kr outside [0,1]");
      m.kr = x;
    } else {
      return perr(line, "unknown option '" + key + "' (ks, shininess, kr)");
    }
  }
  return RT_OK;
}

int parse_floats(const std::vector<std::string>& f, size_t n, int line, float* out) {
  if (f.size() != n + 1) {
    char buf[96];
    snprintf(buf, sizeof buf, "bad arity: '%s' takes %zu numbers, got %zu", f[0].c_str(), n, f.size() - 1);
    return perr(line, buf);
  }
  for (size_t i = 0; i < n; ++i)
    if (!to_float(f[1 + i], out[i])) return perr(line, "non-numeric field '" + f[1 + i] + "'");
  return RT_OK;
}

int parse_text(const char* text, int64_t n, Parsed& S) {
  int line = 0;
  int64_t pos = 0;
  while (pos < n) {
    int64_t end = pos;
    while (end < n && text[end] != '\n') ++end;
    ++line;
    // split the line [pos, end) on ASCII whitespace; a '#' starts a comment
    std::vector<std::string> f;
    std::string cur;
    for (int64_t i = pos; i < end; ++i) {
      const char ch = text[i];
      if (ch == '#') break;
      if (ch == ' ' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f') {
        if (!cur.empty()) { f.push_back(cur); cur.clear(); }
      } else {
        if (cur.size() > 256) return perr(line, "field too long");
        cur.push_back(ch);
      }
    }
    if (!cur.empty()) f.push_back(cur);
    pos = end + 1;
    if (f.empty()) continue;
    const std::string& d = f[0];
    int rc = RT_OK;
    if (d == "camera") {
      if (S.has_camera) return perr(line, "duplicate camera");
      float v[10];
      if ((rc = parse_floats(f, 10, line, v))) return rc;
      for (int i = 0; i < 3; ++i) { S.eye[i] = v[i]; S.look[i] = v[3 + i]; S.up[i] = v[6 + i]; }
      S.vfov = v[9];
      S.has_camera = true;
      S.camera_line = line;
    } else if (d == "sphere" || d == "plane") {
      const bool sph = d == "sphere";
      const size_t ng = 4;  // sphere: radius cx cy cz; plane: nx ny nz d
      if (f.size() < 1 + ng) return perr(line, "bad arity: '" + d + "' needs its geometry fields");
      float g[4];
      for (size_t i = 0; i < ng; ++i)
        if (!to_float(f[1 + i], g[i])) return perr(line, "non-numeric field '" + f[1 + i] + "'");
      rt_primitive p{};
      if (sph) {
        if (!(g[0] > 0.f)) return perr(line, "radius <= 0");
        p.type = RT_PRIM_SPHERE;
        p.p[0] = g[1]; p.p[1] = g[2]; p.p[2] = g[3]; p.p[3] = g[0];
      } else {
        if (g[0] == 0.f && g[1] == 0.f && g[2] == 0.f) return perr(line, "plane normal is zero");
        p.type = RT_PRIM_PLANE;
        for (int i = 0; i < 4; ++i) p.p[i] = g[i];
      }
      rt_material m;
      if ((rc = parse_material(f, 1 + ng, line, m))) return rc;
      if (S.mats.size() >= (size_t)1 << 24 || S.prims.size() >= (size_t)RT_MAX_SPHERES + RT_MAX_PLANES)
        return perr(line, "too many primitives");
      p.material = (uint32_t)S.mats.size();
      S.mats.push_back(m);
      S.prims.push_back(p);
    } else if (d == "light") {
      float v[6];
      if ((rc = parse_floats(f, 6, line, v))) return rc;
      for (int i = 0; i < 3; ++i)
        if (!(v[3 + i] >= 0.f)) return perr(line, "light intensity must be >= 0");
      if (S.lights.size() >= (size_t)RT_MAX_LIGHTS) return perr(line, "too many lights");
      rt_light l;
      for (int i = 0; i < 3; ++i) { l.position[i] = v[i]; l.intensity[i] = v[3 + i]; }
      S.lights.push_back(l);
    } else if (d == "background" || d == "ambient") {
      float v[3];
      if ((rc = parse_floats(f, 3, line, v))) return rc;
      for (int i = 0; i < 3; ++i) {
        if (!(v[i] >= 0.f)) return perr(line, d + " must be >= 0");
        (d == "background" ? S.env.background : S.env.ambient)[i] = v[i];
      }
    } else {
      return perr(line, "unknown directive '" + (d.size() > 32 ? d.substr(0, 32) + "..." : d) + "'");
    }
  }
  if (!S.has_camera) return perr(line > 0 ? line : 1, "missing camera");
  // camera invariants, checked here so the error carries the camera's line
  double f3[3] = {(double)S.look[0] - S.eye[0], (double)S.look[1] - S.eye[1], (double)S.look[2] - S.eye[2]};
  const double fl = std::sqrt(f3[0] * f3[0] + f3[1] * f3[1] + f3[2] * f3[2]);
  if (!(fl > 0.0)) return perr(S.camera_line, "camera: eye == look_at");
  if (!(S.vfov > 0.f && S.vfov < 180.f)) return perr(S.camera_line, "camera: vfov must be in (0, 180)");
  const double u[3] = {S.up[0], S.up[1], S.up[2]};
  const double c[3] = {f3[1] * u[2] - f3[2] * u[1], f3[2] * u[0] - f3[0] * u[2], f3[0] * u[1] - f3[1] * u[0]};
  const double cl = std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
  const double ul = std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  if (!(cl > 1e-12 * fl * (ul > 0 ? ul : 1.0))) return perr(S.camera_line, "camera: up is zero or parallel to the view direction");
  return RT_OK;
}

}  // namespace

extern "C" {

int rt_scene_parse(const char* text, int64_t n_bytes) {
  rt_clear_error();
  if (n_bytes < 0 || (n_bytes > 0 && !text)) return rt_fail(RT_ERR_INVALID_ARG, "scene text: NULL or n_bytes < 0");
  Parsed S;
  int rc = parse_text(text, n_bytes, S);
  if (rc) return rc;
  if (S.mats.empty()) {  // a scene of lights only still needs one material record
    rt_material m{};
    m.kind = RT_MAT_DIFFUSE;
    m.ior = 1.5f;
    m.shininess = 1.f;
    S.mats.push_back(m);
  }
  rc = rt_scene_upload(S.prims.empty() ? nullptr : S.prims.data(), (int32_t)S.prims.size(), S.mats.data(),
                       (int32_t)S.mats.size(), S.lights.empty() ? nullptr : S.lights.data(), (int32_t)S.lights.size(),
                       &S.env);
  if (rc) return rc;
  return rt_camera_set(S.eye, S.look, S.up, S.vfov);
}

int rt_scene_load(const char* path) {
  rt_clear_error();
  if (!path) return rt_fail(RT_ERR_INVALID_ARG, "scene path is NULL");
  FILE* fp = std::fopen(path, "rb");
  if (!fp) return rt_fail(RT_ERR_IO, (std::string("cannot read scene file '") + path + "': " + std::strerror(errno)).c_str());
  std::vector<char> buf;
  char chunk[65536];
  size_t got;
  while ((got = std::fread(chunk, 1, sizeof chunk, fp)) > 0) {
    buf.insert(buf.end(), chunk, chunk + got);
    if (buf.size() > ((size_t)1 << 30)) {
      std::fclose(fp);
      return rt_fail(RT_ERR_IO, (std::string("scene file '") + path + "' exceeds 1 GiB").c_str());
    }
  }
  const bool err = std::ferror(fp) != 0;
  std::fclose(fp);
  if (err) return rt_fail(RT_ERR_IO, (std::string("error reading scene file '") + path + "'").c_str());
  return rt_scene_parse(buf.data(), (int64_t)buf.size());
}

int rt_write_ppm(const float* rgba, int32_t width, int32_t height, float exposure, float gamma, const char* path) {
  rt_clear_error();
  if (!rgba || !path || width < 1 || height < 1)
    return rt_fail(RT_ERR_INVALID_ARG, "write_ppm: NULL pointer or empty image");
  const long long n = (long long)width * height;
  uint8_t* d8 = nullptr;
  cudaError_t e = cudaMalloc(&d8, (size_t)n * 4);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return rt_fail(RT_ERR_CUDA, (std::string("write_ppm: cudaMalloc: ") + cudaGetErrorString(e)).c_str());
  }
  int rc = rt_tonemap_rgba8(rgba, d8, n, exposure, gamma);  // validates rgba (device) and the params
  std::vector<uint8_t> h((size_t)n * 4);
  if (rc == RT_OK) {
    e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(h.data(), d8, (size_t)n * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      cudaGetLastError();
      rc = rt_fail(RT_ERR_CUDA, (std::string("write_ppm: ") + cudaGetErrorString(e)).c_str());
    }
  }
  cudaFree(d8);
  if (rc) return rc;
  FILE* fp = std::fopen(path, "wb");
  if (!fp) return rt_fail(RT_ERR_IO, (std::string("cannot write '") + path + "': " + std::strerror(errno)).c_str());
  std::string hdr = "P6\n" + std::to_string(width) + " " + std::to_string(height) + "\n255\n";
  bool ok = std::fwrite(hdr.data(), 1, hdr.size(), fp) == hdr.size();
  std::vector<uint8_t> rgb((size_t)n * 3);
  for (long long i = 0; i < n; ++i) {  // drop alpha (byte shuffling only; the tone map ran on the device)
    rgb[3 * i + 0] = h[4 * i + 0];
    rgb[3 * i + 1] = h[4 * i + 1];
    rgb[3 * i + 2] = h[4 * i + 2];
  }
  ok = ok && std::fwrite(rgb.data(), 1, rgb.size(), fp) == rgb.size();
  ok = (std::fclose(fp) == 0) && ok;
  if (!ok) return rt_fail(RT_ERR_IO, (std::string("error writing '") + path + "'").c_str());
  return RT_OK;
}

}  // extern "C"
