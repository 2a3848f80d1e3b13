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

}  // namespace inpc
