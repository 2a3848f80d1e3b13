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
};

struct DevCfg {
  int H, W, C, mode;
  float sigma, dil, amax, tmin;
  int tiles_x, tiles_y, ty0, ty1;
  unsigned flags;
};

constexpr unsigned kFlagSigmaPx = 1u;
constexpr unsigned kFlagSkipZero = 2u;

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

// H2 bilinear (R3).
__device__ __forceinline__ bool foot_bilinear(const DevCfg& g, const Proj& p, Foot& f) {
  float ax = __fsub_rn(p.u, 0.5f), ay = __fsub_rn(p.v, 0.5f);
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

// H2 Gaussian (R15-R19): isotropic world std s, EWA Jacobian,
// dilation, 3-sigma bbox.
__device__ __forceinline__ bool foot_gauss(const DevCam& c, const DevCfg& g, const Proj& p,
                                           Foot& f) {
  float a, b, cc;
  if (g.flags & kFlagSigmaPx) {
    a = __fadd_rn(__fmul_rn(g.sigma, g.sigma), g.dil);
    b = 0.0f;
    cc = a;
  } else {
    float s = g.sigma > 0.0f ? g.sigma : __fdiv_rn(__fmul_rn(5.0f, c.z_near), fmaxf(c.fx, c.fy));
    float jx = __fdiv_rn(c.fx, p.zc), jy = __fdiv_rn(c.fy, p.zc);
    float s2 = __fmul_rn(s, s);
    a = __fadd_rn(__fmul_rn(s2, __fmul_rn(__fmul_rn(jx, jx), __fadd_rn(1.0f, __fmul_rn(p.xz, p.xz)))),
                  g.dil);
    b = __fmul_rn(s2, __fmul_rn(__fmul_rn(jx, jy), __fmul_rn(p.xz, p.yz)));
    cc = __fadd_rn(__fmul_rn(s2, __fmul_rn(__fmul_rn(jy, jy), __fadd_rn(1.0f, __fmul_rn(p.yz, p.yz)))),
                   g.dil);
  }
  float det = __fsub_rn(__fmul_rn(a, cc), __fmul_rn(b, b));
  if (!(det > 0.0f) || !isfinite(det)) return false;
  f.ca = __fdiv_rn(cc, det);
  f.cb = __fdiv_rn(-b, det);
  f.cc = __fdiv_rn(a, det);
  float mid = __fmul_rn(0.5f, __fadd_rn(a, cc)), hd = __fmul_rn(0.5f, __fsub_rn(a, cc));
  float lmax = __fadd_rn(mid, __fsqrt_rn(__fadd_rn(__fmul_rn(hd, hd), __fmul_rn(b, b))));
  float r = __fmul_rn(3.0f, __fsqrt_rn(lmax));
  if (!isfinite(r) || !isfinite(f.ca) || !isfinite(f.cb) || !isfinite(f.cc)) return false;
  float ax = __fsub_rn(p.u, 0.5f), ay = __fsub_rn(p.v, 0.5f);
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

template <int MODE>
__device__ __forceinline__ bool point_foot(const DevCam& c, const DevCfg& g, const float* xyz,
                                           int64_t i, Proj& p, Foot& f) {
  float X = __ldg(xyz + 3 * i), Y = __ldg(xyz + 3 * i + 1), Z = __ldg(xyz + 3 * i + 2);
  if (!project_point(c, X, Y, Z, p)) return false;
  return MODE == 0 ? foot_bilinear(g, p, f) : foot_gauss(c, g, p, f);
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

}  // namespace inpc
