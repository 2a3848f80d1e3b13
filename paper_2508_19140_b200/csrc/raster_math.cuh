// raster_math.cuh — per-point / per-fragment arithmetic of the rasterizer,
// in the pinned fp32 op order of DESIGN.md §3 (R1).  Every operation is an
// explicitly rounded intrinsic (__fmul_rn / __fadd_rn / __fdiv_rn /
// __fsqrt_rn) so nvcc cannot contract it into an FMA: depth keys, pixel
// sets, alpha and the termination decisions are bit-identical to the
// independent CPU oracle.  No fast-math anywhere in this library.
#pragma once
#include <cstdint>

namespace inpc {

constexpr int kTile = 8;  // 8x8 tiles

struct DevCam {
  float R[9];
  float t[3];
  float fx, fy, cx, cy, z_near;
  float cw[3];  // camera centre in world space, -R^T t (SH view directions)
};

struct DevCfg {
  int H, W, C, mode;
  float sigma, dil, amax, tmin;
  int tiles_x, tiles_y, ty0, ty1;
  unsigned flags;
  int env_h, env_w;
};

constexpr unsigned kFlagSigmaPx = 1u;
constexpr unsigned kFlagSkipZero = 2u;
constexpr unsigned kFlagSH = 4u;
constexpr unsigned kFlagEnv = 8u;
constexpr unsigned kFlagRec16 = 1u << 29;  // internal: bilinear records are 16-byte {u, v, z, o}, features read from feat

struct Proj {
  float xc, yc, zc, u, v, xz, yz;
};

// H1: x_c = R x + t, near-plane / finiteness cull (R9), pinhole (R2).
__device__ __forceinline__ bool project_point(const DevCam& c, float X, float Y, float Z,
                                              Proj& p) {
  p.xc = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.R[0], X), __fmul_rn(c.R[1], Y)),
                             __fmul_rn(c.R[2], Z)), c.t[0]);
  p.yc = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.R[3], X), __fmul_rn(c.R[4], Y)),
                             __fmul_rn(c.R[5], Z)), c.t[1]);
  p.zc = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.R[6], X), __fmul_rn(c.R[7], Y)),
                             __fmul_rn(c.R[8], Z)), c.t[2]);
  if (!(p.zc > c.z_near) || !isfinite(p.xc) || !isfinite(p.yc) || !isfinite(p.zc)) return false;
  p.xz = __fdiv_rn(p.xc, p.zc);
  p.yz = __fdiv_rn(p.yc, p.zc);
  p.u = __fadd_rn(__fmul_rn(c.fx, p.xz), c.cx);
  p.v = __fadd_rn(__fmul_rn(c.fy, p.yz), c.cy);
  return true;
}

// Footprint of one point: clipped pixel rectangle + mode parameters.
struct Foot {
  int xlo, xhi, ylo, yhi;
  // bilinear
  int x0, y0;
  float fa, fb;
  // Gaussian
  float ca, cb, cc;
};

// H2 bilinear (R3): block floor(u-1/2) + {0,1}.
__device__ __forceinline__ bool foot_bilinear(const DevCfg& g, float u, float v, Foot& f) {
  float ax = __fsub_rn(u, 0.5f), ay = __fsub_rn(v, 0.5f);
  if (!(ax >= -1.0f && ax < (float)g.W && ay >= -1.0f && ay < (float)g.H)) return false;
  float flx = floorf(ax), fly = floorf(ay);
  f.fa = __fsub_rn(ax, flx);
  f.fb = __fsub_rn(ay, fly);
  f.x0 = (int)flx;
  f.y0 = (int)fly;
  f.xlo = max(f.x0, 0);
  f.xhi = min(f.x0 + 1, g.W - 1);
  f.ylo = max(f.y0, 0);
  f.yhi = min(f.y0 + 1, g.H - 1);
  return true;
}

// H2 Gaussian, part 1 (R15-R19): conic of the dilated EWA
// covariance of an isotropic world Gaussian, and its 3-sigma radius.
__device__ __forceinline__ bool gauss_conic(const DevCam& c, const DevCfg& g, const Proj& p,
                                            float& ca, float& cb, float& cc, float& r) {
  float a, b, c2;
  if (g.flags & kFlagSigmaPx) {
    a = __fadd_rn(__fmul_rn(g.sigma, g.sigma), g.dil);
    b = 0.0f;
    c2 = a;
  } else {
    float s = g.sigma > 0.0f ? g.sigma : __fdiv_rn(__fmul_rn(5.0f, c.z_near), fmaxf(c.fx, c.fy));
    float jx = __fdiv_rn(c.fx, p.zc), jy = __fdiv_rn(c.fy, p.zc);
    float s2 = __fmul_rn(s, s);
    a = __fadd_rn(__fmul_rn(s2, __fmul_rn(__fmul_rn(jx, jx), __fadd_rn(1.0f, __fmul_rn(p.xz, p.xz)))),
                  g.dil);
    b = __fmul_rn(s2, __fmul_rn(__fmul_rn(jx, jy), __fmul_rn(p.xz, p.yz)));
    c2 = __fadd_rn(__fmul_rn(s2, __fmul_rn(__fmul_rn(jy, jy), __fadd_rn(1.0f, __fmul_rn(p.yz, p.yz)))),
                   g.dil);
  }
  float det = __fsub_rn(__fmul_rn(a, c2), __fmul_rn(b, b));
  if (!(det > 0.0f) || !isfinite(det)) return false;
  ca = __fdiv_rn(c2, det);
  cb = __fdiv_rn(-b, det);
  cc = __fdiv_rn(a, det);
  float mid = __fmul_rn(0.5f, __fadd_rn(a, c2)), hd = __fmul_rn(0.5f, __fsub_rn(a, c2));
  float lmax = __fadd_rn(mid, __fsqrt_rn(__fadd_rn(__fmul_rn(hd, hd), __fmul_rn(b, b))));
  r = __fmul_rn(3.0f, __fsqrt_rn(lmax));
  return isfinite(r) && isfinite(ca) && isfinite(cb) && isfinite(cc);
}

// H2 Gaussian, part 2: clipped pixel bbox of radius r around (u, v) (R17).
__device__ __forceinline__ bool gauss_rect(const DevCfg& g, float u, float v, float r, Foot& f) {
  float ax = __fsub_rn(u, 0.5f), ay = __fsub_rn(v, 0.5f);
  float xlo = ceilf(__fsub_rn(ax, r)), xhi = floorf(__fadd_rn(ax, r));
  float ylo = ceilf(__fsub_rn(ay, r)), yhi = floorf(__fadd_rn(ay, r));
  if (!(xhi >= 0.0f && xlo <= (float)(g.W - 1) && yhi >= 0.0f && ylo <= (float)(g.H - 1)))
    return false;
  if (!(xlo <= xhi && ylo <= yhi)) return false;
  f.xlo = xlo < 0.0f ? 0 : (int)xlo;
  f.xhi = xhi > (float)(g.W - 1) ? g.W - 1 : (int)xhi;
  f.ylo = ylo < 0.0f ? 0 : (int)ylo;
  f.yhi = yhi > (float)(g.H - 1) ? g.H - 1 : (int)yhi;
  return true;
}

// Gaussian Mahalanobis distance of pixel (px, py), pinned order.
__device__ __forceinline__ float gauss_q(float ca, float cb, float cc, float u, float v, int px,
                                         int py) {
  float dx = __fsub_rn(__fadd_rn((float)px, 0.5f), u);
  float dy = __fsub_rn(__fadd_rn((float)py, 0.5f), v);
  return __fadd_rn(__fadd_rn(__fmul_rn(__fmul_rn(ca, dx), dx),
                             __fmul_rn(__fmul_rn(__fmul_rn(cb, dx), dy), 2.0f)),
                   __fmul_rn(__fmul_rn(cc, dy), dy));
}

// ---- NEXT f1: degree-2 SH features, values only (no decisions).
// Real basis, standard constants; d = unit vector camera centre -> point (R26).
__device__ __forceinline__ void sh_basis(float x, float y, float z, float* Y) {
  const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
  Y[0] = C0;
  Y[1] = -C1 * y;
  Y[2] = C1 * z;
  Y[3] = -C1 * x;
  Y[4] = 1.0925484305920792f * x * y;
  Y[5] = -1.0925484305920792f * y * z;
  Y[6] = 0.31539156525252005f * (2.0f * z * z - x * x - y * y);
  Y[7] = -1.0925484305920792f * x * z;
  Y[8] = 0.5462742152960396f * (x * x - y * y);
}

__device__ __forceinline__ void sh_dir_basis(const DevCam& c, float X, float Y, float Z, float* B) {
  const float dx = X - c.cw[0], dy = Y - c.cw[1], dz = Z - c.cw[2];
  const float n2 = dx * dx + dy * dy + dz * dz;
  const float inv = n2 > 0.0f ? rsqrtf(n2) : 0.0f;
  sh_basis(dx * inv, dy * inv, dz * inv, B);
}

// f_c = sum_k sh[c*9 + k] B_k for the point's coefficient block sh [C, 9]
__device__ __forceinline__ float sh_feature(const float* __restrict__ sh, int c, const float* B) {
  float f = 0.0f;
#pragma unroll
  for (int k = 0; k < 9; ++k) f += __ldg(sh + c * 9 + k) * B[k];
  return f;
}

// ---- NEXT f2: equirectangular environment background (R27).
// Pixel-centre ray rotated to world space (recomputed: a few flops instead
// of the paper's cached direction buffer, 12 B/pixel of HBM on B200);
// u = (atan2(dx, dz)/2pi + 1/2) We, v = acos(dy)/pi He, texel centres at
// +1/2, bilinear with azimuthal wrap and polar clamp.  The texel coordinate
// is computed in fp64: in fp32 a 2048-texel coordinate carries 1.2e-4 texel
// of rounding (and atan2f another ~1e-4), which on a high-frequency map
// exceeds the 1e-4 image tolerance; per pixel this is ~100 DP instructions.
__device__ __forceinline__ void env_weights(const DevCam& c, const DevCfg& g, int px, int py,
                                            int* idx4, float* w4) {
  const double xc = ((double)px + 0.5 - (double)c.cx) / (double)c.fx;
  const double yc = ((double)py + 0.5 - (double)c.cy) / (double)c.fy;
  const double inv = 1.0 / sqrt(xc * xc + yc * yc + 1.0);
  double d[3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
    d[k] = ((double)c.R[k] * xc + (double)c.R[3 + k] * yc + (double)c.R[6 + k]) * inv;
  const double PI = 3.14159265358979323846;
  const double u = (atan2(d[0], d[2]) / (2.0 * PI) + 0.5) * g.env_w;
  const double v = acos(fmin(fmax(d[1], -1.0), 1.0)) / PI * g.env_h;
  const double x = u - 0.5, y = v - 0.5;
  const double fx0 = floor(x), fy0 = floor(y);
  const double a = x - fx0, b = y - fy0;
  int i0 = (int)fx0, j0 = (int)fy0;  // u in [0, We]: x in [-1/2, We - 1/2]
  int i1 = i0 + 1, j1 = j0 + 1;
  i0 = i0 < 0 ? i0 + g.env_w : (i0 >= g.env_w ? i0 - g.env_w : i0);  // azimuthal wrap
  i1 = i1 < 0 ? i1 + g.env_w : (i1 >= g.env_w ? i1 - g.env_w : i1);
  j0 = min(max(j0, 0), g.env_h - 1);
  j1 = min(max(j1, 0), g.env_h - 1);
  idx4[0] = j0 * g.env_w + i0; w4[0] = (float)((1.0 - a) * (1.0 - b));
  idx4[1] = j0 * g.env_w + i1; w4[1] = (float)(a * (1.0 - b));
  idx4[2] = j1 * g.env_w + i0; w4[2] = (float)((1.0 - a) * b);
  idx4[3] = j1 * g.env_w + i1; w4[3] = (float)(a * b);
}

}  // namespace inpc
