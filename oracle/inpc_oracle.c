/*
 * inpc_oracle.c — CPU ORACLE for the INPC neural point rasterizer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2508_19140_b200/) never includes, links or calls it,
 * and this file includes nothing from the product path.
 *
 * What it computes is the plain definition of the rasterizer
 * ("Rendering Feature Maps", Eq. 1 at P:474-479, the
 * corrected Eq. 2 at P:482-491, the Gaussian footprint at P:196-204):
 *   for every pixel, gather every fragment of every point that covers it,
 *   sort the fragments by (depth, point index), and composite them front to
 *   back with alpha blending.
 * No tiling, no two-stage sort, no blocking: the tile lists exported by
 * or_tile_lists() are only the definition of what the tiled method must
 * produce, built by a plain per-tile qsort.
 *
 * Precision (readings R1, R4-R6, R23):
 *   - positions, projected coordinates, bilinear weights / Gaussian conics,
 *     alpha and the transmittance recurrence that decides early termination
 *     are fp32 in the pinned op order of DESIGN.md §3 (every op rounded, no
 *     FMA: compiled with -ffp-contract=off on x86-64 SSE);
 *   - the composited values F, A, D and all gradients are accumulated in
 *     fp64 over exactly the fragments the fp32 decisions keep.
 *
 * Parity pins: see tests/test_oracle_pins.py (Q1-Q16 of DESIGN.md §4).
 * Parity unpinned: agreement with INPC's own code/images (unavailable);
 * the constants alpha_max, t_min (R5, R6) are this build's definitions.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- own copies of the parameter records (no shared headers) ---------- */
typedef struct {
  float R[9];     /* world->camera rotation, row-major: x_c = R x + t     */
  float t[3];
  float fx, fy, cx, cy; /* pinhole, pixel (i,j) centre at (i+0.5, j+0.5)  */
  float z_near;
} or_camera;

typedef struct {
  int32_t H, W, C;
  int32_t mode;     /* 0 bilinear 2x2, 1 Gaussian */
  float sigma;      /* Gaussian world std; <=0: 5 px at near plane  */
  float dilation;   /* px^2 added to the 2D covariance          */
  float alpha_max;  /* alpha clamp (R5)                                     */
  float t_min;      /* early-termination threshold (R6), 0 = off            */
  uint32_t flags;   /* bit0 SIGMA_IS_PIXELS (R15), bit1 SKIP_ZERO_ALPHA_GRAD (R13) */
} or_cfg;

#define OR_SIGMA_IS_PIXELS 1u
#define OR_SKIP_ZERO_ALPHA_GRAD 2u
#define OR_TILE 8 /* 8x8 tiles */

/* One fragment = (pixel, point) pair with its footprint weight. */
typedef struct {
  uint32_t key;  /* float bits of camera-space z (R7, "32-bit depth") */
  uint32_t idx;  /* point index (tie-break, R8)                             */
  int32_t pix;   /* y*W + x                                                 */
  float w32;     /* footprint weight, fp32 pinned (decisions)               */
  double w64;    /* footprint weight, fp64 (values)                         */
} frag_t;

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* ---- projection (H1 / O1): pinned fp32 order, DESIGN.md §3 R1 ---------- */
/* returns 1 if the point survives the near-plane / finiteness cull (R9). */
static int project(const or_camera* c, const float* p, float* xc, float* yc,
                   float* zc, float* u, float* v) {
  float X = p[0], Y = p[1], Z = p[2];
  float x = ((c->R[0] * X + c->R[1] * Y) + c->R[2] * Z) + c->t[0];
  float y = ((c->R[3] * X + c->R[4] * Y) + c->R[5] * Z) + c->t[1];
  float z = ((c->R[6] * X + c->R[7] * Y) + c->R[8] * Z) + c->t[2];
  *xc = x; *yc = y; *zc = z;
  if (!(z > c->z_near) || !isfinite(x) || !isfinite(y) || !isfinite(z)) return 0;
  *u = c->fx * (x / z) + c->cx;   /* contraction off: mul then add */
  *v = c->fy * (y / z) + c->cy;
  return 1;
}

/* ---- footprints (H2 / O2) --------------------------------------------- */
typedef struct {
  int ok;                /* touches at least one in-image pixel          */
  int xlo, xhi, ylo, yhi; /* clipped pixel rectangle that may hold frags  */
  /* bilinear */
  int x0, y0; float fa, fb;
  /* Gaussian */
  float ca, cb, cc, r, u, v;
  float a2, b2, c2; /* 2D covariance, for the pins */
} footprint_t;

/* Bilinear 2x2 splat (R3): the pixel block
 * {x0,x0+1} x {y0,y0+1} with x0 = floor(u - 1/2); in-image pixels kept,
 * including weight-0 ones; weights (1-a)(1-b), a(1-b), (1-a)b, ab. */
static void fp_bilinear(const or_cfg* g, float u, float v, footprint_t* f) {
  memset(f, 0, sizeof *f);
  float ax = u - 0.5f, ay = v - 0.5f;
  if (!(ax >= -1.0f && ax < (float)g->W && ay >= -1.0f && ay < (float)g->H)) return;
  float flx = floorf(ax), fly = floorf(ay);
  f->fa = ax - flx; f->fb = ay - fly;
  f->x0 = (int)flx; f->y0 = (int)fly;
  f->xlo = f->x0 < 0 ? 0 : f->x0;
  f->xhi = f->x0 + 1 > g->W - 1 ? g->W - 1 : f->x0 + 1;
  f->ylo = f->y0 < 0 ? 0 : f->y0;
  f->yhi = f->y0 + 1 > g->H - 1 ? g->H - 1 : f->y0 + 1;
  f->ok = 1;
}

/* Isotropic Gaussian of world std s projected with the affine (EWA)
 * approximation, dilated by `dilation` px^2, cut at 3 sigma
 * (R15-R19). */
static void fp_gauss(const or_camera* c, const or_cfg* g, float xc, float yc,
                     float zc, float u, float v, footprint_t* f) {
  memset(f, 0, sizeof *f);
  float a, b, cc;
  if (g->flags & OR_SIGMA_IS_PIXELS) {
    a = g->sigma * g->sigma + g->dilation; b = 0.0f; cc = a;
  } else {
    /* std of a Gaussian at the near plane, projected to the image
     * centre, is five pixels -> s = 5 z_near / max(fx, fy) (R16). */
    float s = g->sigma > 0.0f ? g->sigma
                              : (5.0f * c->z_near) / fmaxf(c->fx, c->fy);
    float xz = xc / zc, yz = yc / zc;      /* same rounded quotients as u,v */
    float jx = c->fx / zc, jy = c->fy / zc; /* J = [[jx,0,-jx*xz],[0,jy,-jy*yz]] */
    float s2 = s * s;
    /* Sigma2D = s^2 J J^T + dilation I */
    a = s2 * ((jx * jx) * (1.0f + xz * xz)) + g->dilation;
    b = s2 * ((jx * jy) * (xz * yz));
    cc = s2 * ((jy * jy) * (1.0f + yz * yz)) + g->dilation;
  }
  f->a2 = a; f->b2 = b; f->c2 = cc;
  float det = a * cc - b * b;
  if (!(det > 0.0f) || !isfinite(det)) return; /* R19 */
  f->ca = cc / det; f->cb = -b / det; f->cc = a / det;
  float mid = 0.5f * (a + cc), hd = 0.5f * (a - cc);
  float lmax = mid + sqrtf(hd * hd + b * b);
  float r = 3.0f * sqrtf(lmax);
  if (!isfinite(r) || !isfinite(f->ca) || !isfinite(f->cb) || !isfinite(f->cc)) return;
  f->r = r; f->u = u; f->v = v;
  float ax = u - 0.5f, ay = v - 0.5f;
  float xlo = ceilf(ax - r), xhi = floorf(ax + r);
  float ylo = ceilf(ay - r), yhi = floorf(ay + r);
  if (!(xhi >= 0.0f && xlo <= (float)(g->W - 1) && yhi >= 0.0f && ylo <= (float)(g->H - 1)))
    return;
  if (!(xlo <= xhi && ylo <= yhi)) return;
  f->xlo = xlo < 0.0f ? 0 : (int)xlo;
  f->xhi = xhi > (float)(g->W - 1) ? g->W - 1 : (int)xhi;
  f->ylo = ylo < 0.0f ? 0 : (int)ylo;
  f->yhi = yhi > (float)(g->H - 1) ? g->H - 1 : (int)yhi;
  f->ok = 1;
}

/* Weight of pixel (px,py) under footprint f; returns 1 if it is a fragment. */
static int frag_weight(const or_cfg* g, const footprint_t* f, int px, int py,
                       float* w32, double* w64) {
  if (px < f->xlo || px > f->xhi || py < f->ylo || py > f->yhi) return 0;
  if (g->mode == 0) {
    int dx = px - f->x0, dy = py - f->y0; /* each 0 or 1 */
    float wx = dx ? f->fa : 1.0f - f->fa;
    float wy = dy ? f->fb : 1.0f - f->fb;
    *w32 = wx * wy;
    double wx64 = dx ? (double)f->fa : 1.0 - (double)f->fa;
    double wy64 = dy ? (double)f->fb : 1.0 - (double)f->fb;
    *w64 = wx64 * wy64;
    return 1;
  }
  float dx = ((float)px + 0.5f) - f->u, dy = ((float)py + 0.5f) - f->v;
  float q = ((f->ca * dx) * dx + ((f->cb * dx) * dy) * 2.0f) + (f->cc * dy) * dy;
  if (!(q <= 9.0f)) return 0;         /* 3-sigma ellipse, R17 */
  *w32 = expf(-0.5f * q);
  double q64 = (double)f->ca * dx * dx + 2.0 * (double)f->cb * dx * dy +
               (double)f->cc * dy * dy;
  *w64 = exp(-0.5 * q64);
  return 1;
}

/* Project one point and build its footprint; returns 1 if it has any. */
static int point_footprint(const or_camera* c, const or_cfg* g, const float* p,
                           uint32_t* key, float* zc_out, footprint_t* f) {
  float xc, yc, zc, u = 0, v = 0;
  memset(f, 0, sizeof *f);
  if (!project(c, p, &xc, &yc, &zc, &u, &v)) return -1; /* culled */
  *key = f2u(zc); *zc_out = zc;
  if (g->mode == 0) fp_bilinear(g, u, v, f);
  else fp_gauss(c, g, xc, yc, zc, u, v, f);
  return f->ok;
}

/* ---- per-point info: depth keys and tile counts (pins H1/H2) ----------- */
/* depth_key[i] = 0xFFFFFFFF for culled points. tiles_touched[i] = number of
 * 8x8 tiles that hold the point's (possible) fragments.  uvz/gauss optional. */
int or_point_info(const or_camera* c, const or_cfg* g, int64_t N, const float* xyz,
                  uint32_t* depth_key, uint32_t* tiles_touched, float* uvz,
                  float* gauss /* [N,7]: ca,cb,cc,r,a2,b2,c2 */) {
  for (int64_t i = 0; i < N; i++) {
    float xc, yc, zc, u = 0, v = 0;
    footprint_t f; memset(&f, 0, sizeof f);
    int vis = project(c, xyz + 3 * i, &xc, &yc, &zc, &u, &v);
    if (vis) {
      if (g->mode == 0) fp_bilinear(g, u, v, &f);
      else fp_gauss(c, g, xc, yc, zc, u, v, &f);
    }
    if (depth_key) depth_key[i] = vis ? f2u(zc) : 0xFFFFFFFFu;
    if (tiles_touched)
      tiles_touched[i] = f.ok ? (uint32_t)((f.xhi / OR_TILE - f.xlo / OR_TILE + 1) *
                                           (f.yhi / OR_TILE - f.ylo / OR_TILE + 1))
                              : 0u;
    if (uvz) { uvz[3 * i] = u; uvz[3 * i + 1] = v; uvz[3 * i + 2] = zc; }
    if (gauss) {
      gauss[7 * i + 0] = f.ca; gauss[7 * i + 1] = f.cb; gauss[7 * i + 2] = f.cc;
      gauss[7 * i + 3] = f.r; gauss[7 * i + 4] = f.a2; gauss[7 * i + 5] = f.b2;
      gauss[7 * i + 6] = f.c2;
    }
  }
  return 0;
}

/* ---- fragment gather (O2) ---------------------------------------------- */
typedef struct { frag_t* a; int64_t n, cap; } fvec;
static int fpush(fvec* v, frag_t f) {
  if (v->n == v->cap) {
    int64_t nc = v->cap ? 2 * v->cap : 1024;
    frag_t* na = (frag_t*)realloc(v->a, (size_t)nc * sizeof(frag_t));
    if (!na) return -1;
    v->a = na; v->cap = nc;
  }
  v->a[v->n++] = f;
  return 0;
}

/* All fragments of all points, in (point index, row, column) order; only
 * pixels with pixel_mask[pix] != 0 are kept when a mask is given. */
static int gather_fragments(const or_camera* c, const or_cfg* g, int64_t N,
                            const float* xyz, const uint8_t* pixel_mask, fvec* out) {
  for (int64_t i = 0; i < N; i++) {
    footprint_t f; uint32_t key = 0; float zc;
    if (point_footprint(c, g, xyz + 3 * i, &key, &zc, &f) != 1) continue;
    for (int py = f.ylo; py <= f.yhi; py++)
      for (int px = f.xlo; px <= f.xhi; px++) {
        int32_t pix = py * g->W + px;
        if (pixel_mask && !pixel_mask[pix]) continue;
        frag_t fr; fr.key = key; fr.idx = (uint32_t)i; fr.pix = pix;
        if (!frag_weight(g, &f, px, py, &fr.w32, &fr.w64)) continue;
        if (fpush(out, fr)) return -1;
      }
  }
  return 0;
}

static int cmp_depth_idx(const void* A, const void* B) {
  const frag_t* a = (const frag_t*)A; const frag_t* b = (const frag_t*)B;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;
  return 0;
}

/* Group fragments per pixel (counting pass) and sort each pixel's list by
 * (depth key, point index) -> O3.  ranges has P+1 entries. */
static int per_pixel_lists(const or_cfg* g, fvec* fr, int64_t** ranges_out,
                           frag_t** sorted_out, int nthreads) {
  int64_t P = (int64_t)g->H * g->W;
  int64_t* ranges = (int64_t*)calloc((size_t)P + 1, sizeof(int64_t));
  frag_t* s = (frag_t*)malloc((size_t)(fr->n ? fr->n : 1) * sizeof(frag_t));
  int64_t* cur = (int64_t*)malloc((size_t)P * sizeof(int64_t));
  if (!ranges || !s || !cur) { free(ranges); free(s); free(cur); return -1; }
  for (int64_t k = 0; k < fr->n; k++) ranges[fr->a[k].pix + 1]++;
  for (int64_t p = 0; p < P; p++) ranges[p + 1] += ranges[p];
  memcpy(cur, ranges, (size_t)P * sizeof(int64_t));
  for (int64_t k = 0; k < fr->n; k++) s[cur[fr->a[k].pix]++] = fr->a[k];
  free(cur);
  (void)nthreads;
#pragma omp parallel for schedule(dynamic, 4096) num_threads(nthreads)
  for (int64_t p = 0; p < P; p++)
    qsort(s + ranges[p], (size_t)(ranges[p + 1] - ranges[p]), sizeof(frag_t), cmp_depth_idx);
  *ranges_out = ranges; *sorted_out = s;
  return 0;
}

/* ---- compositing (O4): Eq. 1 + background ---------- */
/* Decision pass in fp32 (alpha clamp, early termination R5/R6) -> number of
 * fragments composited; the values are then accumulated in fp64. */
static int decide_fp32(const or_cfg* g, const frag_t* fr, int64_t K,
                       const double* opacity, float* T_out) {
  float T = 1.0f; int n = 0;
  for (int64_t k = 0; k < K; k++) {
    float o = (float)opacity[fr[k].idx];
    float alpha = fminf(o * fr[k].w32, g->alpha_max);
    float Tn = T * (1.0f - alpha);
    if (Tn < g->t_min) break;
    T = Tn; n = (int)(k + 1);
  }
  *T_out = T;
  return n;
}

static double alpha64(const or_cfg* g, double o, double w) {
  double a = o * w;
  return a < (double)g->alpha_max ? a : (double)g->alpha_max;
}

/* camera-space z of a fragment, recovered from its depth key (R7) */
static double key_depth(uint32_t key) { float z; memcpy(&z, &key, 4); return (double)z; }

/* Forward render.  Outputs (any may be NULL): F [H,W,C], A [H,W], D [H,W]
 * (fp64 values), T32 [H,W] (fp32 decision transmittance), n_contrib,
 * n_frag [H,W].  bg [H,W,C] or NULL (R11).  pixel_mask selects pixels
 * (others are left untouched). */
int or_render(const or_camera* c, const or_cfg* g, int64_t N, const float* xyz,
              const double* feat, const double* opacity, const double* bg,
              const uint8_t* pixel_mask, double* F, double* A, double* D,
              float* T32, int32_t* n_contrib, int32_t* n_frag, int nthreads) {
  fvec fr = {0, 0, 0};
  if (gather_fragments(c, g, N, xyz, pixel_mask, &fr)) { free(fr.a); return -1; }
  int64_t* ranges; frag_t* s;
  if (per_pixel_lists(g, &fr, &ranges, &s, nthreads)) { free(fr.a); return -1; }
  free(fr.a);
  int64_t P = (int64_t)g->H * g->W; int C = g->C;
#pragma omp parallel for schedule(dynamic, 4096) num_threads(nthreads)
  for (int64_t p = 0; p < P; p++) {
    if (pixel_mask && !pixel_mask[p]) continue;
    const frag_t* L = s + ranges[p];
    int64_t K = ranges[p + 1] - ranges[p];
    float Tf; int n = decide_fp32(g, L, K, opacity, &Tf);
    double T = 1.0, Dv = 0.0;
    double Fv[256];
    for (int ch = 0; ch < C; ch++) Fv[ch] = 0.0;
    for (int k = 0; k < n; k++) {
      uint32_t i = L[k].idx;
      double a = alpha64(g, opacity[i], L[k].w64);
      for (int ch = 0; ch < C; ch++) Fv[ch] += T * a * feat[(int64_t)i * C + ch];
      Dv += T * a * key_depth(L[k].key);
      T *= (1.0 - a);
    }
    for (int ch = 0; ch < C; ch++) {
      double b = bg ? bg[p * C + ch] : 0.0;
      if (F) F[p * C + ch] = Fv[ch] + T * b;
    }
    if (A) A[p] = 1.0 - T;
    if (D) D[p] = Dv;
    if (T32) T32[p] = Tf;
    if (n_contrib) n_contrib[p] = n;
    if (n_frag) n_frag[p] = (int32_t)K;
  }
  free(ranges); free(s);
  return 0;
}

/* ---- backward (O5): Eq. 2 with the sign of the background term corrected
 * (R12, R13).  fp64.  Gradients ACCUMULATE (+=). ---- */
int or_backward(const or_camera* c, const or_cfg* g, int64_t N, const float* xyz,
                const double* feat, const double* opacity, const double* bg,
                const uint8_t* pixel_mask, const double* gF, const double* gA,
                const double* gD, double* g_feat, double* g_opacity, int nthreads) {
  fvec fr = {0, 0, 0};
  if (gather_fragments(c, g, N, xyz, pixel_mask, &fr)) { free(fr.a); return -1; }
  int64_t* ranges; frag_t* s;
  if (per_pixel_lists(g, &fr, &ranges, &s, nthreads)) { free(fr.a); return -1; }
  free(fr.a);
  int64_t P = (int64_t)g->H * g->W; int C = g->C;
  /* per-pixel work in parallel; accumulation into points serialised with
   * atomics (order of fp64 sums differs by rounding only) */
#pragma omp parallel for schedule(dynamic, 4096) num_threads(nthreads)
  for (int64_t p = 0; p < P; p++) {
    if (pixel_mask && !pixel_mask[p]) continue;
    const frag_t* L = s + ranges[p];
    int64_t K = ranges[p + 1] - ranges[p];
    float Tf; int n = decide_fp32(g, L, K, opacity, &Tf);
    if (n == 0) continue;
    double* Tk = (double*)malloc(sizeof(double) * (size_t)n);
    double* ak = (double*)malloc(sizeof(double) * (size_t)n);
    double T = 1.0;
    for (int k = 0; k < n; k++) {   /* T_k = prod_{j<k} (1 - alpha_j), Eq. 1 */
      Tk[k] = T; ak[k] = alpha64(g, opacity[L[k].idx], L[k].w64);
      T *= (1.0 - ak[k]);
    }
    double R[256], RD = 0.0, Pr = 1.0;   /* R = bg after the last fragment */
    for (int ch = 0; ch < C; ch++) R[ch] = bg ? bg[p * C + ch] : 0.0;
    double GA = gA ? gA[p] : 0.0, GD = gD ? gD[p] : 0.0;
    for (int k = n - 1; k >= 0; k--) {
      uint32_t i = L[k].idx;
      double a = ak[k], z = key_depth(L[k].key);
      const double* f = feat + (int64_t)i * C;
      int skip = (g->flags & OR_SKIP_ZERO_ALPHA_GRAD) && a == 0.0;
      if (!skip) {
        /* dF/dalpha_k = T_k (f_k - R_k): R_k is everything behind k
         * (later fragments and background) normalised by T_{k+1}. */
        double dA = 0.0;
        for (int ch = 0; ch < C; ch++) {
          double G = gF ? gF[p * C + ch] : 0.0;
          double gf = Tk[k] * a * G;                 /* dF/df_k = T_k alpha_k */
#pragma omp atomic
          g_feat[(int64_t)i * C + ch] += gf;
          dA += G * (f[ch] - R[ch]);
        }
        dA += GD * (z - RD) + GA * Pr;               /* A = 1 - T_{K+1} */
        dA *= Tk[k];
        double o = opacity[i];
        if (o * L[k].w64 < (double)g->alpha_max) {   /* clamp has zero slope */
#pragma omp atomic
          g_opacity[i] += L[k].w64 * dA;
        }
      }
      for (int ch = 0; ch < C; ch++) R[ch] = a * f[ch] + (1.0 - a) * R[ch];
      RD = a * z + (1.0 - a) * RD;
      Pr *= (1.0 - a);
    }
    free(Tk); free(ak);
  }
  free(ranges); free(s);
  return 0;
}

/* ---- per-tile lists (definition of H4-H6's output) ---------- */
typedef struct { uint32_t key, idx; } ent_t;
static int cmp_ent(const void* A, const void* B) {
  const ent_t* a = (const ent_t*)A; const ent_t* b = (const ent_t*)B;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;
  return 0;
}

/* Every point is listed in every 8x8 tile that holds its footprint
 * rectangle; each list sorted by (depth key, point index).
 * Tiles whose row ty is outside [ty0, ty1) are left empty (screen bands).
 * tile_ranges [T+1]; writes at most cap indices; returns F_t or -1. */
int64_t or_tile_lists(const or_camera* c, const or_cfg* g, int64_t N, const float* xyz,
                      int32_t ty0, int32_t ty1, uint32_t* tile_ranges,
                      uint32_t* sorted_idx, int64_t cap) {
  int tx_n = (g->W + OR_TILE - 1) / OR_TILE, ty_n = (g->H + OR_TILE - 1) / OR_TILE;
  int64_t T = (int64_t)tx_n * ty_n;
  int64_t* cnt = (int64_t*)calloc((size_t)T + 1, sizeof(int64_t));
  if (!cnt) return -1;
  for (int pass = 0; pass < 2; pass++) {
    ent_t* e = NULL; int64_t* cur = NULL;
    if (pass == 1) {
      for (int64_t t = 0; t < T; t++) cnt[t + 1] += cnt[t];
      e = (ent_t*)malloc((size_t)(cnt[T] ? cnt[T] : 1) * sizeof(ent_t));
      cur = (int64_t*)malloc((size_t)T * sizeof(int64_t));
      if (!e || !cur) { free(e); free(cur); free(cnt); return -1; }
      memcpy(cur, cnt, (size_t)T * sizeof(int64_t));
    }
    for (int64_t i = 0; i < N; i++) {
      footprint_t f; uint32_t key = 0; float zc;
      if (point_footprint(c, g, xyz + 3 * i, &key, &zc, &f) != 1) continue;
      for (int ty = f.ylo / OR_TILE; ty <= f.yhi / OR_TILE; ty++) {
        if (ty < ty0 || ty >= ty1) continue;
        for (int tx = f.xlo / OR_TILE; tx <= f.xhi / OR_TILE; tx++) {
          int64_t t = (int64_t)ty * tx_n + tx;
          if (pass == 0) cnt[t + 1]++;
          else { e[cur[t]].key = key; e[cur[t]].idx = (uint32_t)i; cur[t]++; }
        }
      }
    }
    if (pass == 1) {
      for (int64_t t = 0; t < T; t++)
        qsort(e + cnt[t], (size_t)(cnt[t + 1] - cnt[t]), sizeof(ent_t), cmp_ent);
      for (int64_t t = 0; t <= T; t++) tile_ranges[t] = (uint32_t)cnt[t];
      for (int64_t k = 0; k < cnt[T] && k < cap; k++) sorted_idx[k] = e[k].idx;
      free(e); free(cur);
    }
  }
  int64_t Ft = cnt[T];
  free(cnt);
  return Ft;
}

/* ---- O7: the original single-sort ordering ----------
 * All fragments keyed by 64-bit (pixel << 32 | depth key), in point-index
 * emission order, stably merge-sorted.  Used to cross-check O3. */
static void msort64(uint64_t* k, uint32_t* v, uint64_t* tk, uint32_t* tv, int64_t n) {
  for (int64_t w = 1; w < n; w *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
      int64_t i = lo, j = mid, o = lo;
      while (i < mid && j < hi) {
        if (k[j] < k[i]) { tk[o] = k[j]; tv[o++] = v[j++]; }   /* stable */
        else { tk[o] = k[i]; tv[o++] = v[i++]; }
      }
      while (i < mid) { tk[o] = k[i]; tv[o++] = v[i++]; }
      while (j < hi) { tk[o] = k[j]; tv[o++] = v[j++]; }
    }
    memcpy(k, tk, (size_t)n * 8); memcpy(v, tv, (size_t)n * 4);
  }
}

/* method 0: per-pixel qsort by (depth, idx) (O3); method 1: single stable
 * 64-bit sort (O7).  pixel_ranges [P+1]; returns #fragments or -1. */
int64_t or_pixel_lists(const or_camera* c, const or_cfg* g, int64_t N, const float* xyz,
                       int method, uint32_t* pixel_ranges, uint32_t* idx, int64_t cap) {
  fvec fr = {0, 0, 0};
  if (gather_fragments(c, g, N, xyz, NULL, &fr)) { free(fr.a); return -1; }
  int64_t P = (int64_t)g->H * g->W, n = fr.n;
  if (method == 0) {
    int64_t* ranges; frag_t* s;
    if (per_pixel_lists(g, &fr, &ranges, &s, 1)) { free(fr.a); return -1; }
    for (int64_t p = 0; p <= P; p++) pixel_ranges[p] = (uint32_t)ranges[p];
    for (int64_t k = 0; k < n && k < cap; k++) idx[k] = s[k].idx;
    free(ranges); free(s);
  } else {
    uint64_t* k = (uint64_t*)malloc((size_t)(n + 1) * 8);
    uint64_t* tk = (uint64_t*)malloc((size_t)(n + 1) * 8);
    uint32_t* v = (uint32_t*)malloc((size_t)(n + 1) * 4);
    uint32_t* tv = (uint32_t*)malloc((size_t)(n + 1) * 4);
    if (!k || !tk || !v || !tv) { free(k); free(tk); free(v); free(tv); free(fr.a); return -1; }
    for (int64_t q = 0; q < n; q++) {
      k[q] = ((uint64_t)(uint32_t)fr.a[q].pix << 32) | fr.a[q].key;
      v[q] = fr.a[q].idx;
    }
    msort64(k, v, tk, tv, n);
    for (int64_t p = 0; p <= P; p++) pixel_ranges[p] = 0;
    for (int64_t q = 0; q < n; q++) pixel_ranges[(k[q] >> 32) + 1]++;
    for (int64_t p = 0; p < P; p++) pixel_ranges[p + 1] += pixel_ranges[p];
    for (int64_t q = 0; q < n && q < cap; q++) idx[q] = v[q];
    free(k); free(tk); free(v); free(tv);
  }
  free(fr.a);
  return n;
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Raw fragment list (O2) in emission order (point index, row, column), for
 * the footprint pins.  Returns the number of fragments; writes <= cap. */
int64_t or_fragments(const or_camera* c, const or_cfg* g, int64_t N, const float* xyz,
                     int32_t* pix, uint32_t* idx, uint32_t* key, float* w32, double* w64,
                     int64_t cap) {
  fvec fr = {0, 0, 0};
  if (gather_fragments(c, g, N, xyz, NULL, &fr)) { free(fr.a); return -1; }
  for (int64_t k = 0; k < fr.n && k < cap; k++) {
    pix[k] = fr.a[k].pix; idx[k] = fr.a[k].idx; key[k] = fr.a[k].key;
    w32[k] = fr.a[k].w32; w64[k] = fr.a[k].w64;
  }
  int64_t n = fr.n;
  free(fr.a);
  return n;
}

/* ---- NEXT f1: degree-2 spherical-harmonics features -------------
 * f_c = sum_k coeff[c][k] Y_k(d), d = unit vector from the camera centre to
 * the point, real SH basis with the standard constants (SPEC S:~455 design
 * decision; R26).  fp64. */
static const double OR_SH_C0 = 0.28209479177387814;
static const double OR_SH_C1 = 0.4886025119029199;
static const double OR_SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                   -1.0925484305920792, 0.5462742152960396};

void or_sh_basis(const double* d, double* Y) {
  double x = d[0], y = d[1], z = d[2];
  Y[0] = OR_SH_C0;
  Y[1] = -OR_SH_C1 * y;
  Y[2] = OR_SH_C1 * z;
  Y[3] = -OR_SH_C1 * x;
  Y[4] = OR_SH_C2[0] * x * y;
  Y[5] = OR_SH_C2[1] * y * z;
  Y[6] = OR_SH_C2[2] * (2.0 * z * z - x * x - y * y);
  Y[7] = OR_SH_C2[3] * x * z;
  Y[8] = OR_SH_C2[4] * (x * x - y * y);
}

/* camera centre in world space: x_cam = R x + t = 0  ->  c = -R^T t */
static void cam_centre(const or_camera* c, double* ctr) {
  for (int k = 0; k < 3; k++)
    ctr[k] = -((double)c->R[0 * 3 + k] * c->t[0] + (double)c->R[1 * 3 + k] * c->t[1] +
               (double)c->R[2 * 3 + k] * c->t[2]);
}

/* feat [N, C] (fp64) from sh [N, C, 9]; Ybuf [N, 9] optional (the basis per point) */
void or_sh_features(const or_camera* c, int64_t N, int C, const float* xyz, const double* sh,
                    double* feat, double* Ybuf) {
  double ctr[3];
  cam_centre(c, ctr);
  for (int64_t i = 0; i < N; i++) {
    double d[3] = {xyz[3 * i] - ctr[0], xyz[3 * i + 1] - ctr[1], xyz[3 * i + 2] - ctr[2]};
    double n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (n > 0) { d[0] /= n; d[1] /= n; d[2] /= n; }
    double Y[9];
    or_sh_basis(d, Y);
    for (int ch = 0; ch < C; ch++) {
      double s = 0;
      for (int k = 0; k < 9; k++) s += sh[(i * C + ch) * 9 + k] * Y[k];
      feat[i * C + ch] = s;
    }
    if (Ybuf) for (int k = 0; k < 9; k++) Ybuf[i * 9 + k] = Y[k];
  }
}

/* ---- NEXT f2: equirectangular environment-map background ---
 * Pixel ray through the pixel centre, rotated to world space; u =
 * (atan2(dx, dz) / 2 pi + 1/2) We, v = acos(dy) / pi He; texel (i, j) centre
 * at (i + 1/2, j + 1/2); bilinear with azimuthal wrap and polar clamp
 * (R27).  bg [H, W, C] fp64 from env [He, We, C]. */
void or_env_background(const or_camera* c, int H, int W, int C, const float* env, int He, int We,
                       double* bg) {
  const double PI = 3.14159265358979323846;
  for (int py = 0; py < H; py++)
    for (int px = 0; px < W; px++) {
      double dc[3] = {((px + 0.5) - c->cx) / c->fx, ((py + 0.5) - c->cy) / c->fy, 1.0};
      double n = sqrt(dc[0] * dc[0] + dc[1] * dc[1] + dc[2] * dc[2]);
      double d[3];
      for (int k = 0; k < 3; k++)   /* world = R^T cam */
        d[k] = (c->R[0 * 3 + k] * dc[0] + c->R[1 * 3 + k] * dc[1] + c->R[2 * 3 + k] * dc[2]) / n;
      double u = (atan2(d[0], d[2]) / (2 * PI) + 0.5) * We;
      double dy = d[1] < -1 ? -1 : (d[1] > 1 ? 1 : d[1]);
      double v = acos(dy) / PI * He;
      double x = u - 0.5, y = v - 0.5;
      double fx0 = floor(x), fy0 = floor(y);
      double a = x - fx0, b = y - fy0;
      long i0 = (long)fx0, j0 = (long)fy0;
      long i1 = i0 + 1, j1 = j0 + 1;
      i0 = ((i0 % We) + We) % We; i1 = ((i1 % We) + We) % We;
      if (j0 < 0) j0 = 0;
      if (j0 > He - 1) j0 = He - 1;
      if (j1 < 0) j1 = 0;
      if (j1 > He - 1) j1 = He - 1;
      for (int ch = 0; ch < C; ch++) {
        double t00 = env[((size_t)j0 * We + i0) * C + ch], t10 = env[((size_t)j0 * We + i1) * C + ch];
        double t01 = env[((size_t)j1 * We + i0) * C + ch], t11 = env[((size_t)j1 * We + i1) * C + ch];
        bg[((size_t)py * W + px) * C + ch] =
            (1 - a) * (1 - b) * t00 + a * (1 - b) * t10 + (1 - a) * b * t01 + a * b * t11;
      }
    }
}
