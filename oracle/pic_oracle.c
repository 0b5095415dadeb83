/* TEST INFRASTRUCTURE ONLY — see pic_oracle.h.
 *
 * Plain-C fp32 restatement of the reference hot path.  Each function names
 * the reference lines it restates; expression association order is kept
 * exactly (the build uses -ffp-contract=off, like proj/src/CMakeLists.txt:20)
 * so results are bit-identical to the reference's scalar / AVX2 lanes.
 */
#include "pic_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
const char* orc_last_error(void) { return g_err; }

/* ---- grid (proj/include/minipic/grid.hpp:15-56, proj/src/grid.cpp) ------ */
static inline int pnx(const orc_grid* g) { return g->nx + 2; }
static inline int pny(const orc_grid* g) { return g->ny + 2; }
static inline int pnz(const orc_grid* g) { return g->nz + 2; }
static inline size_t padded(const orc_grid* g) {
  return (size_t)pnx(g) * (size_t)pny(g) * (size_t)pnz(g);
}
static inline int32_t vox(const orc_grid* g, int ix, int iy, int iz) {
  return (int32_t)(ix + pnx(g) * (iy + pny(g) * iz)); /* grid.hpp:53-56 */
}

float orc_cfl_limit(const orc_grid* g) { /* grid.cpp:7-11 */
  const float s = 1.0f / (g->hx * g->hx) + 1.0f / (g->hy * g->hy) + 1.0f / (g->hz * g->hz);
  return 1.0f / sqrtf(s);
}

/* lane indices (proj/include/minipic/lanes.hpp) */
enum { F_EX = 0, F_EY, F_EZ, F_DIVE, F_BX, F_BY, F_BZ, F_DIVB, F_JX, F_JY, F_JZ, F_RHO };
enum {
  I_EX = 0, I_DEXDY, I_DEXDZ, I_D2EX, I_EY, I_DEYDZ, I_DEYDX, I_D2EY,
  I_EZ, I_DEZDX, I_DEZDY, I_D2EZ, I_BX, I_DBXDX, I_BY, I_DBYDY, I_BZ, I_DBZDZ
};
#define FL(f, V, lane, v) ((f)[(size_t)(lane) * (V) + (size_t)(v)])

/* ---- load_interpolators (proj/src/particles.cpp:42-111) ----------------- */
void orc_load_interpolators(const orc_grid* g, const float* f, float* c) {
  const size_t V = padded(g);
  const size_t sx = 1, sy = (size_t)pnx(g), sz = (size_t)pnx(g) * (size_t)pny(g);
  for (int iz = 1; iz <= g->nz; ++iz)
    for (int iy = 1; iy <= g->ny; ++iy)
      for (int ix = 1; ix <= g->nx; ++ix) {
        const size_t v = (size_t)vox(g, ix, iy, iz);
        float w0, w1, w2, w3;
        w0 = FL(f, V, F_EX, v); w1 = FL(f, V, F_EX, v + sy);
        w2 = FL(f, V, F_EX, v + sz); w3 = FL(f, V, F_EX, v + sy + sz);
        FL(c, V, I_EX, v) = 0.25f * ((w3 + w0) + (w1 + w2));
        FL(c, V, I_DEXDY, v) = 0.25f * ((w3 - w0) + (w1 - w2));
        FL(c, V, I_DEXDZ, v) = 0.25f * ((w3 - w0) - (w1 - w2));
        FL(c, V, I_D2EX, v) = 0.25f * ((w3 + w0) - (w1 + w2));
        w0 = FL(f, V, F_EY, v); w1 = FL(f, V, F_EY, v + sz);
        w2 = FL(f, V, F_EY, v + sx); w3 = FL(f, V, F_EY, v + sz + sx);
        FL(c, V, I_EY, v) = 0.25f * ((w3 + w0) + (w1 + w2));
        FL(c, V, I_DEYDZ, v) = 0.25f * ((w3 - w0) + (w1 - w2));
        FL(c, V, I_DEYDX, v) = 0.25f * ((w3 - w0) - (w1 - w2));
        FL(c, V, I_D2EY, v) = 0.25f * ((w3 + w0) - (w1 + w2));
        w0 = FL(f, V, F_EZ, v); w1 = FL(f, V, F_EZ, v + sx);
        w2 = FL(f, V, F_EZ, v + sy); w3 = FL(f, V, F_EZ, v + sx + sy);
        FL(c, V, I_EZ, v) = 0.25f * ((w3 + w0) + (w1 + w2));
        FL(c, V, I_DEZDX, v) = 0.25f * ((w3 - w0) + (w1 - w2));
        FL(c, V, I_DEZDY, v) = 0.25f * ((w3 - w0) - (w1 - w2));
        FL(c, V, I_D2EZ, v) = 0.25f * ((w3 + w0) - (w1 + w2));
        w0 = FL(f, V, F_BX, v); w1 = FL(f, V, F_BX, v + sx);
        FL(c, V, I_BX, v) = 0.5f * (w1 + w0);
        FL(c, V, I_DBXDX, v) = 0.5f * (w1 - w0);
        w0 = FL(f, V, F_BY, v); w1 = FL(f, V, F_BY, v + sy);
        FL(c, V, I_BY, v) = 0.5f * (w1 + w0);
        FL(c, V, I_DBYDY, v) = 0.5f * (w1 - w0);
        w0 = FL(f, V, F_BZ, v); w1 = FL(f, V, F_BZ, v + sz);
        FL(c, V, I_BZ, v) = 0.5f * (w1 + w0);
        FL(c, V, I_DBZDZ, v) = 0.5f * (w1 - w0);
      }
}

/* ---- push math (proj/include/minipic/kernels/push_math.hpp:22-82) ------- */
static inline float gamma_of(float ux, float uy, float uz) {
  const float usq = (ux * ux + uy * uy) + uz * uz;
  return sqrtf(1.0f + usq);
}

typedef struct { float ex, ey, ez, bx, by, bz; } eb_t;

static inline void eval_eb(const float* c, size_t V, int32_t v, float x, float y, float z,
                           eb_t* f) {
  const size_t o = (size_t)v;
  f->ex = ((FL(c, V, I_EX, o) + y * FL(c, V, I_DEXDY, o)) + z * FL(c, V, I_DEXDZ, o)) +
          (y * z) * FL(c, V, I_D2EX, o);
  f->ey = ((FL(c, V, I_EY, o) + z * FL(c, V, I_DEYDZ, o)) + x * FL(c, V, I_DEYDX, o)) +
          (z * x) * FL(c, V, I_D2EY, o);
  f->ez = ((FL(c, V, I_EZ, o) + x * FL(c, V, I_DEZDX, o)) + y * FL(c, V, I_DEZDY, o)) +
          (x * y) * FL(c, V, I_D2EZ, o);
  f->bx = FL(c, V, I_BX, o) + x * FL(c, V, I_DBXDX, o);
  f->by = FL(c, V, I_BY, o) + y * FL(c, V, I_DBYDY, o);
  f->bz = FL(c, V, I_BZ, o) + z * FL(c, V, I_DBZDZ, o);
}

static inline void boris(float* ux, float* uy, float* uz, const eb_t* f, float qdt_2m,
                         int exact_gyration) {
  const float emx = qdt_2m * f->ex, emy = qdt_2m * f->ey, emz = qdt_2m * f->ez;
  const float umx = *ux + emx, umy = *uy + emy, umz = *uz + emz;
  const float gm = gamma_of(umx, umy, umz);
  const float rg = qdt_2m / gm;
  float tx = f->bx * rg, ty = f->by * rg, tz = f->bz * rg;
  if (exact_gyration) {
    const float tl = sqrtf((tx * tx + ty * ty) + tz * tz);
    if (tl > 0) {
      const float sc = tanf(tl) / tl;
      tx = tx * sc; ty = ty * sc; tz = tz * sc;
    }
  }
  const float upx = umx + (umy * tz - umz * ty);
  const float upy = umy + (umz * tx - umx * tz);
  const float upz = umz + (umx * ty - umy * tx);
  const float tsq = (tx * tx + ty * ty) + tz * tz;
  const float sf = 2.0f / (1.0f + tsq);
  const float sx = tx * sf, sy = ty * sf, sz = tz * sf;
  *ux = (umx + (upy * sz - upz * sy)) + emx;
  *uy = (umy + (upz * sx - upx * sz)) + emy;
  *uz = (umz + (upx * sy - upy * sx)) + emz;
}

/* ---- deposit_weights (proj/src/particles.cpp:141-158) ------------------- */
static inline void dep_dir(float da, float m1, float m2, float d1, float d2, float qw,
                           float* four) {
  const float twelfth = 1.0f / 12.0f;
  const float base = 0.25f * (qw * da);
  const float p1l = 1 - m1, p1h = 1 + m1, p2l = 1 - m2, p2h = 1 + m2;
  const float cc = (d1 * d2) * twelfth;
  four[0] = base * (p1l * p2l + cc);
  four[1] = base * (p1h * p2l - cc);
  four[2] = base * (p1l * p2h - cc);
  four[3] = base * (p1h * p2h + cc);
}
static inline void deposit(float* acc, int32_t v, const float mid[3], const float disp[3],
                           float qw) {
  float w[12];
  dep_dir(disp[0], mid[1], mid[2], disp[1], disp[2], qw, w + 0);
  dep_dir(disp[1], mid[2], mid[0], disp[2], disp[0], qw, w + 4);
  dep_dir(disp[2], mid[0], mid[1], disp[0], disp[1], qw, w + 8);
  float* row = acc + (size_t)v * 12; /* ScatterBuffer::contribute_row, layout.cpp:159-179 */
  for (int l = 0; l < 12; ++l) row[l] += w[l];
}

/* ---- run_mover (proj/src/particles.cpp:186-241) ------------------------- */
static int run_mover(const orc_grid* g, int32_t v0, const float s[3], const float d[3],
                     float qw, float* acc, float out_q[3], int32_t* out_v) {
  for (int a = 0; a < 3; ++a)
    if (!(fabsf(d[a]) < 2)) {
      snprintf(g_err, sizeof g_err,
               "advance_particles: particle crossed more than one cell along axis %d (CFL violation)", a);
      return 2;
    }
  const int32_t stride[3] = {1, pnx(g), pnx(g) * pny(g)};
  float q[3] = {s[0], s[1], s[2]};
  float r[3] = {d[0], d[1], d[2]};
  int32_t v = v0;
  for (int pass = 0; pass < 8; ++pass) {
    int axis = -1;
    float fmin = 1;
    for (int a = 0; a < 3; ++a) {
      const float e = q[a] + r[a];
      if (e > 1 || e < -1) {
        const float sigma = r[a] > 0 ? 1.0f : -1.0f;
        const float fa = (sigma - q[a]) / r[a];
        if (axis < 0 || fa < fmin) { axis = a; fmin = fa; }
      }
    }
    if (axis < 0) {
      const float mid[3] = {q[0] + 0.5f * r[0], q[1] + 0.5f * r[1], q[2] + 0.5f * r[2]};
      if (acc) deposit(acc, v, mid, r, qw);
      out_q[0] = q[0] + r[0];
      out_q[1] = q[1] + r[1];
      out_q[2] = q[2] + r[2];
      *out_v = v;
      return 0;
    }
    const float sigma = r[axis] > 0 ? 1.0f : -1.0f;
    const float seg[3] = {fmin * r[0], fmin * r[1], fmin * r[2]};
    const float mid[3] = {q[0] + 0.5f * seg[0], q[1] + 0.5f * seg[1], q[2] + 0.5f * seg[2]};
    if (acc) deposit(acc, v, mid, seg, qw);
    for (int a = 0; a < 3; ++a) { q[a] = q[a] + seg[a]; r[a] = r[a] - seg[a]; }
    q[axis] = -sigma;
    v += sigma > 0 ? stride[axis] : -stride[axis];
  }
  snprintf(g_err, sizeof g_err, "advance_particles: mover failed to terminate");
  return 2;
}

/* wrap_axis (proj/src/grid.cpp:40-52) */
static int wrap_axis(int i, int n, int* ok) {
  if (i < 0 || i > n + 1) { *ok = 0; return i; }
  if (i == 0) return n;
  if (i == n + 1) return 1;
  return i;
}

/* ---- advance_particles + push_chunk_scalar (proj/src/particles.cpp:255-360,
 *      proj/src/kernels/scalar.cpp:7-34), single worker / sequential order -- */
int orc_advance_particles(const orc_grid* g, float q, float m, long n, float* p,
                          int32_t* ids, const float* c, float* acc, int exact_gyration) {
  const size_t V = padded(g);
  const size_t N = (size_t)n;
  const float cx = 2 * g->dt / g->hx, cy = 2 * g->dt / g->hy, cz = 2 * g->dt / g->hz;
  const float qdt_2m = q * g->dt / (2 * m);
  for (size_t i = 0; i < N; ++i) {
    float* dx = &FL(p, N, 0, i); float* dy = &FL(p, N, 1, i); float* dz = &FL(p, N, 2, i);
    float* ux = &FL(p, N, 3, i); float* uy = &FL(p, N, 4, i); float* uz = &FL(p, N, 5, i);
    const float w = FL(p, N, 6, i);
    const int32_t v0 = ids[i];
    float u0 = *ux, u1 = *uy, u2 = *uz;
    eb_t f;
    eval_eb(c, V, v0, *dx, *dy, *dz, &f);
    boris(&u0, &u1, &u2, &f, qdt_2m, exact_gyration);
    const float gm = gamma_of(u0, u1, u2);
    const float rg = 1.0f / gm;
    const float e[3] = {*dx + (u0 * rg) * cx, *dy + (u1 * rg) * cy, *dz + (u2 * rg) * cz};
    *ux = u0; *uy = u1; *uz = u2;
    const float s[3] = {*dx, *dy, *dz};
    const float d[3] = {e[0] - s[0], e[1] - s[1], e[2] - s[2]};
    const float qw = q * w;
    float qf[3];
    int32_t vf;
    const int rc = run_mover(g, v0, s, d, qw, acc, qf, &vf);
    if (rc) return rc;
    *dx = qf[0]; *dy = qf[1]; *dz = qf[2];
    /* coords_of -> wrap_periodic -> voxel_of_unchecked (particles.cpp:348-350) */
    if (vf < 0 || (size_t)vf >= V) {
      snprintf(g_err, sizeof g_err, "coords_of: voxel id out of range");
      return 1;
    }
    const int ix = vf % pnx(g), rest = vf / pnx(g);
    const int iy = rest % pny(g), iz = rest / pny(g);
    int ok = 1;
    const int wx = wrap_axis(ix, g->nx, &ok), wy = wrap_axis(iy, g->ny, &ok),
              wz = wrap_axis(iz, g->nz, &ok);
    if (!ok) {
      snprintf(g_err, sizeof g_err, "wrap_periodic: displacement beyond one cell (CFL violation)");
      return 2;
    }
    ids[i] = vox(g, wx, wy, wz);
  }
  return 0;
}

/* ---- ghost_fold_currents (proj/src/grid.cpp:59-99) ---------------------- */
static inline void fold_slot(float* a, const orc_grid* g, int fx, int fy, int fz, int tx,
                             int ty, int tz) {
  float* from = a + (size_t)vox(g, fx, fy, fz) * 12;
  float* to = a + (size_t)vox(g, tx, ty, tz) * 12;
  for (int l = 0; l < 12; ++l) { to[l] += from[l]; from[l] = 0; }
}
void orc_ghost_fold(const orc_grid* g, float* a) {
  for (int iz = 0; iz < pnz(g); ++iz)
    for (int iy = 0; iy < pny(g); ++iy) {
      fold_slot(a, g, 0, iy, iz, g->nx, iy, iz);
      fold_slot(a, g, g->nx + 1, iy, iz, 1, iy, iz);
    }
  for (int iz = 0; iz < pnz(g); ++iz)
    for (int ix = 1; ix <= g->nx; ++ix) {
      fold_slot(a, g, ix, 0, iz, ix, g->ny, iz);
      fold_slot(a, g, ix, g->ny + 1, iz, ix, 1, iz);
    }
  for (int iy = 1; iy <= g->ny; ++iy)
    for (int ix = 1; ix <= g->nx; ++ix) {
      fold_slot(a, g, ix, iy, 0, ix, iy, g->nz);
      fold_slot(a, g, ix, iy, g->nz + 1, ix, iy, 1);
    }
}

/* ---- clear_currents / unload_currents (proj/src/fields.cpp:195-251) ----- */
void orc_clear_currents(const orc_grid* g, float* f) {
  const size_t V = padded(g);
  for (int lane = F_JX; lane <= F_JZ; ++lane)
    for (size_t v = 0; v < V; ++v) FL(f, V, lane, v) = 0;
}
static inline int wrap_hi(int i, int n) { return i > n ? 1 : i; }
void orc_unload(const orc_grid* g, const float* red, float* f) {
  const size_t V = padded(g);
  const float two_dt_v = 2 * g->dt * (g->hx * g->hy * g->hz);
  const float fx = g->hx / two_dt_v, fy = g->hy / two_dt_v, fz = g->hz / two_dt_v;
  for (int iz = 1; iz <= g->nz; ++iz)
    for (int iy = 1; iy <= g->ny; ++iy)
      for (int ix = 1; ix <= g->nx; ++ix) {
        const float* L = red + (size_t)vox(g, ix, iy, iz) * 12;
        const int yhi = wrap_hi(iy + 1, g->ny), zhi = wrap_hi(iz + 1, g->nz),
                  xhi = wrap_hi(ix + 1, g->nx);
        FL(f, V, F_JX, vox(g, ix, iy, iz)) += fx * L[0];
        FL(f, V, F_JX, vox(g, ix, yhi, iz)) += fx * L[1];
        FL(f, V, F_JX, vox(g, ix, iy, zhi)) += fx * L[2];
        FL(f, V, F_JX, vox(g, ix, yhi, zhi)) += fx * L[3];
        FL(f, V, F_JY, vox(g, ix, iy, iz)) += fy * L[4];
        FL(f, V, F_JY, vox(g, ix, iy, zhi)) += fy * L[5];
        FL(f, V, F_JY, vox(g, xhi, iy, iz)) += fy * L[6];
        FL(f, V, F_JY, vox(g, xhi, iy, zhi)) += fy * L[7];
        FL(f, V, F_JZ, vox(g, ix, iy, iz)) += fz * L[8];
        FL(f, V, F_JZ, vox(g, xhi, iy, iz)) += fz * L[9];
        FL(f, V, F_JZ, vox(g, ix, yhi, iz)) += fz * L[10];
        FL(f, V, F_JZ, vox(g, xhi, yhi, iz)) += fz * L[11];
      }
}

/* ---- advance_b / advance_e (proj/src/fields.cpp:113-193, curl_line(_j) at
 *      proj/src/kernels/scalar.cpp:36-49) --------------------------------- */
void orc_advance_b(const orc_grid* g, float* f, float frac) {
  const size_t V = padded(g);
  const float fdt = frac * g->dt;
  const float rhx = 1.0f / g->hx, rhy = 1.0f / g->hy, rhz = 1.0f / g->hz;
  const size_t sx = 1, sy = (size_t)pnx(g), sz = (size_t)pnx(g) * (size_t)pny(g);
  const float c1x = -fdt * rhy, c2x = fdt * rhz;
  const float c1y = -fdt * rhz, c2y = fdt * rhx;
  const float c1z = -fdt * rhx, c2z = fdt * rhy;
  for (int iz = 1; iz <= g->nz; ++iz)
    for (int iy = 1; iy <= g->ny; ++iy)
      for (int ix = 1; ix <= g->nx; ++ix) {
        const size_t v = (size_t)vox(g, ix, iy, iz);
        FL(f, V, F_BX, v) = (FL(f, V, F_BX, v) + c1x * (FL(f, V, F_EZ, v + sy) - FL(f, V, F_EZ, v))) +
                            c2x * (FL(f, V, F_EY, v + sz) - FL(f, V, F_EY, v));
        FL(f, V, F_BY, v) = (FL(f, V, F_BY, v) + c1y * (FL(f, V, F_EX, v + sz) - FL(f, V, F_EX, v))) +
                            c2y * (FL(f, V, F_EZ, v + sx) - FL(f, V, F_EZ, v));
        FL(f, V, F_BZ, v) = (FL(f, V, F_BZ, v) + c1z * (FL(f, V, F_EY, v + sx) - FL(f, V, F_EY, v))) +
                            c2z * (FL(f, V, F_EX, v + sy) - FL(f, V, F_EX, v));
      }
}
void orc_advance_e(const orc_grid* g, float* f) {
  const size_t V = padded(g);
  const float dt = g->dt;
  const float rhx = 1.0f / g->hx, rhy = 1.0f / g->hy, rhz = 1.0f / g->hz;
  const size_t sx = 1, sy = (size_t)pnx(g), sz = (size_t)pnx(g) * (size_t)pny(g);
  const float c1x = dt * rhy, c2x = -dt * rhz;
  const float c1y = dt * rhz, c2y = -dt * rhx;
  const float c1z = dt * rhx, c2z = -dt * rhy;
  const float c3 = -dt;
  for (int iz = 1; iz <= g->nz; ++iz)
    for (int iy = 1; iy <= g->ny; ++iy)
      for (int ix = 1; ix <= g->nx; ++ix) {
        const size_t v = (size_t)vox(g, ix, iy, iz);
        FL(f, V, F_EX, v) = ((FL(f, V, F_EX, v) + c1x * (FL(f, V, F_BZ, v) - FL(f, V, F_BZ, v - sy))) +
                             c2x * (FL(f, V, F_BY, v) - FL(f, V, F_BY, v - sz))) +
                            c3 * FL(f, V, F_JX, v);
        FL(f, V, F_EY, v) = ((FL(f, V, F_EY, v) + c1y * (FL(f, V, F_BX, v) - FL(f, V, F_BX, v - sz))) +
                             c2y * (FL(f, V, F_BZ, v) - FL(f, V, F_BZ, v - sx))) +
                            c3 * FL(f, V, F_JY, v);
        FL(f, V, F_EZ, v) = ((FL(f, V, F_EZ, v) + c1z * (FL(f, V, F_BY, v) - FL(f, V, F_BY, v - sx))) +
                             c2z * (FL(f, V, F_BX, v) - FL(f, V, F_BX, v - sy))) +
                            c3 * FL(f, V, F_JZ, v);
      }
}

/* ---- ghost_sync_fields (proj/src/fields.cpp:19-58) ---------------------- */
static inline void copy_ghost(float* f, size_t V, int32_t to, int32_t from) {
  static const int lanes[6] = {F_EX, F_EY, F_EZ, F_BX, F_BY, F_BZ};
  for (int k = 0; k < 6; ++k) FL(f, V, lanes[k], to) = FL(f, V, lanes[k], from);
}
void orc_ghost_sync(const orc_grid* g, float* f) {
  const size_t V = padded(g);
  for (int iz = 0; iz < pnz(g); ++iz)
    for (int iy = 0; iy < pny(g); ++iy) {
      copy_ghost(f, V, vox(g, 0, iy, iz), vox(g, g->nx, iy, iz));
      copy_ghost(f, V, vox(g, g->nx + 1, iy, iz), vox(g, 1, iy, iz));
    }
  for (int iz = 0; iz < pnz(g); ++iz)
    for (int ix = 0; ix < pnx(g); ++ix) {
      copy_ghost(f, V, vox(g, ix, 0, iz), vox(g, ix, g->ny, iz));
      copy_ghost(f, V, vox(g, ix, g->ny + 1, iz), vox(g, ix, 1, iz));
    }
  for (int iy = 0; iy < pny(g); ++iy)
    for (int ix = 0; ix < pnx(g); ++ix) {
      copy_ghost(f, V, vox(g, ix, iy, 0), vox(g, ix, iy, g->nz));
      copy_ghost(f, V, vox(g, ix, iy, g->nz + 1), vox(g, ix, iy, 1));
    }
}

/* ---- sort_particles (proj/src/particles.cpp:412-458) -------------------- */
int orc_sort(long n_, float* p, int32_t* ids, int interleaved) {
  const size_t n = (size_t)n_;
  if (n == 0) return 0;
  int32_t max_id = ids[0];
  for (size_t i = 1; i < n; ++i) if (ids[i] > max_id) max_id = ids[i];
  const size_t buckets = (size_t)max_id + 1;
  size_t* start = calloc(buckets + 1, sizeof(size_t));
  size_t* cursor = malloc(buckets * sizeof(size_t));
  size_t* perm = malloc(n * sizeof(size_t));
  size_t* within = malloc(n * sizeof(size_t));
  for (size_t i = 0; i < n; ++i) ++start[(size_t)ids[i] + 1];
  for (size_t b = 1; b <= buckets; ++b) start[b] += start[b - 1];
  memcpy(cursor, start, buckets * sizeof(size_t));
  for (size_t i = 0; i < n; ++i) {
    const size_t b = (size_t)ids[i];
    const size_t slot = cursor[b]++;
    perm[slot] = i;
    within[slot] = slot - start[b];
  }
  if (interleaved) {
    size_t max_k = 0;
    for (size_t j = 0; j < n; ++j) if (within[j] > max_k) max_k = within[j];
    size_t* kstart = calloc(max_k + 2, sizeof(size_t));
    size_t* perm2 = malloc(n * sizeof(size_t));
    for (size_t j = 0; j < n; ++j) ++kstart[within[j] + 1];
    for (size_t b = 1; b <= max_k + 1; ++b) kstart[b] += kstart[b - 1];
    for (size_t j = 0; j < n; ++j) perm2[kstart[within[j]]++] = perm[j];
    free(perm);
    perm = perm2;
    free(kstart);
  }
  float* tmp = malloc(n * sizeof(float));
  for (int lane = 0; lane < 7; ++lane) {
    for (size_t j = 0; j < n; ++j) tmp[j] = FL(p, n, lane, perm[j]);
    memcpy(p + (size_t)lane * n, tmp, n * sizeof(float));
  }
  int32_t* tid = malloc(n * sizeof(int32_t));
  for (size_t j = 0; j < n; ++j) tid[j] = ids[perm[j]];
  memcpy(ids, tid, n * sizeof(int32_t));
  free(tid); free(tmp); free(start); free(cursor); free(perm); free(within);
  return 0;
}

/* ---- SimState::step (proj/src/sim.cpp:143-183) -------------------------- */
int orc_step(const orc_grid* g, int nspecies, const float* q, const float* m, const long* n,
             float** lanes7, int32_t** ids, float* f, float* interp, float* acc,
             int exact_gyration) {
  const size_t V = padded(g);
  memset(acc, 0, V * 12 * sizeof(float));
  orc_clear_currents(g, f);
  orc_load_interpolators(g, f, interp);
  for (int s = 0; s < nspecies; ++s) {
    const int rc = orc_advance_particles(g, q[s], m[s], n[s], lanes7[s], ids[s], interp, acc,
                                         exact_gyration);
    if (rc) return rc;
  }
  orc_ghost_fold(g, acc);
  orc_unload(g, acc, f);
  orc_advance_b(g, f, 0.5f);
  orc_ghost_sync(g, f);
  orc_advance_e(g, f);
  orc_ghost_sync(g, f);
  orc_advance_b(g, f, 0.5f);
  orc_ghost_sync(g, f);
  return 0;
}

/* ---- particle load: SimState::initialize (proj/src/sim.cpp:74-112) with the
 *      Rng of proj/include/minipic/rng.hpp:17-51 (std::mt19937_64, whose
 *      output sequence the C++ standard fixes) -------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} orc_rng;

static void mt_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->have_spare = 0;
  r->spare = 0.0;
}
static uint64_t mt_next(orc_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}
static double rng_uniform(orc_rng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }
static double rng_pm1(orc_rng* r) { return 2.0 * rng_uniform(r) - 1.0; }
static double rng_normal(orc_rng* r) {
  if (r->have_spare) { r->have_spare = 0; return r->spare; }
  double u1 = rng_uniform(r);
  double u2 = rng_uniform(r);
  while (u1 == 0.0) u1 = rng_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double t = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rr * sin(t);
  r->have_spare = 1;
  return rr * cos(t);
}

void orc_load_species(const orc_grid* g, uint64_t seed, int si, int ppc, float u_th,
                      const float drift[3], float perturb_ux, int perturb_kmode, float* p,
                      int32_t* ids) {
  static orc_rng rng; /* 2.5 KB state; not re-entrant (test helper) */
  mt_seed(&rng, seed + 0x9e3779b9ULL * (uint64_t)(si + 1));
  const size_t N = (size_t)ppc * (size_t)g->nx * (size_t)g->ny * (size_t)g->nz;
  const double pi = 3.14159265358979323846;
  const float lx = g->hx * (float)g->nx;
  size_t i = 0;
  for (int iz = 1; iz <= g->nz; ++iz)
    for (int iy = 1; iy <= g->ny; ++iy)
      for (int ix = 1; ix <= g->nx; ++ix) {
        const int32_t v = vox(g, ix, iy, iz);
        for (int k = 0; k < ppc; ++k, ++i) {
          const float dx = (float)rng_pm1(&rng);
          const float dy = (float)rng_pm1(&rng);
          const float dz = (float)rng_pm1(&rng);
          float ux = drift[0] + u_th * (float)rng_normal(&rng);
          float uy = drift[1] + u_th * (float)rng_normal(&rng);
          float uz = drift[2] + u_th * (float)rng_normal(&rng);
          if (perturb_ux != 0) {
            const float xg = ((float)(ix - 1) + (dx + 1) * 0.5f) * g->hx;
            ux += perturb_ux * sinf((float)(2 * pi * perturb_kmode) * xg / lx);
          }
          FL(p, N, 0, i) = dx; FL(p, N, 1, i) = dy; FL(p, N, 2, i) = dz;
          FL(p, N, 3, i) = ux; FL(p, N, 4, i) = uy; FL(p, N, 5, i) = uz;
          FL(p, N, 6, i) = 1;
          ids[i] = v;
        }
      }
}

/* ---- diagnostics --------------------------------------------------------- */
/* deposit_rho (proj/src/particles.cpp:384-410) */
void orc_deposit_rho(const orc_grid* g, float q, long n_, const float* p, const int32_t* ids,
                     float* f) {
  const size_t V = padded(g), n = (size_t)n_;
  const float scale = 0.125f / (g->hx * g->hy * g->hz);
  for (size_t i = 0; i < n; ++i) {
    const float x = FL(p, n, 0, i), y = FL(p, n, 1, i), z = FL(p, n, 2, i);
    const float qw = q * FL(p, n, 6, i) * scale;
    const int cx_ = ids[i] % pnx(g), rest = ids[i] / pnx(g);
    const int cy_ = rest % pny(g), cz_ = rest / pny(g);
    const int xh = cx_ + 1 > g->nx ? 1 : cx_ + 1;
    const int yh = cy_ + 1 > g->ny ? 1 : cy_ + 1;
    const int zh = cz_ + 1 > g->nz ? 1 : cz_ + 1;
    const float wxl = 1 - x, wxh = 1 + x, wyl = 1 - y, wyh = 1 + y, wzl = 1 - z, wzh = 1 + z;
    FL(f, V, F_RHO, vox(g, cx_, cy_, cz_)) += qw * (wxl * wyl * wzl);
    FL(f, V, F_RHO, vox(g, xh, cy_, cz_)) += qw * (wxh * wyl * wzl);
    FL(f, V, F_RHO, vox(g, cx_, yh, cz_)) += qw * (wxl * wyh * wzl);
    FL(f, V, F_RHO, vox(g, xh, yh, cz_)) += qw * (wxh * wyh * wzl);
    FL(f, V, F_RHO, vox(g, cx_, cy_, zh)) += qw * (wxl * wyl * wzh);
    FL(f, V, F_RHO, vox(g, xh, cy_, zh)) += qw * (wxh * wyl * wzh);
    FL(f, V, F_RHO, vox(g, cx_, yh, zh)) += qw * (wxl * wyh * wzh);
    FL(f, V, F_RHO, vox(g, xh, yh, zh)) += qw * (wxh * wyh * wzh);
  }
}
/* compute_div_errors (proj/src/fields.cpp:253-274) */
void orc_compute_div_errors(const orc_grid* g, float* f) {
  const size_t V = padded(g);
  const float rhx = 1.0f / g->hx, rhy = 1.0f / g->hy, rhz = 1.0f / g->hz;
  const size_t sx = 1, sy = (size_t)pnx(g), sz = (size_t)pnx(g) * (size_t)pny(g);
  for (int iz = 1; iz <= g->nz; ++iz)
    for (int iy = 1; iy <= g->ny; ++iy)
      for (int ix = 1; ix <= g->nx; ++ix) {
        const size_t v = (size_t)vox(g, ix, iy, iz);
        const float dive = ((FL(f, V, F_EX, v) - FL(f, V, F_EX, v - sx)) * rhx +
                            (FL(f, V, F_EY, v) - FL(f, V, F_EY, v - sy)) * rhy) +
                           (FL(f, V, F_EZ, v) - FL(f, V, F_EZ, v - sz)) * rhz;
        FL(f, V, F_DIVE, v) = dive - FL(f, V, F_RHO, v);
        FL(f, V, F_DIVB, v) = ((FL(f, V, F_BX, v + sx) - FL(f, V, F_BX, v)) * rhx +
                               (FL(f, V, F_BY, v + sy) - FL(f, V, F_BY, v)) * rhy) +
                              (FL(f, V, F_BZ, v + sz) - FL(f, V, F_BZ, v)) * rhz;
      }
}
/* field_energy + sum_squares_scalar (proj/src/fields.cpp:276-299,
 * proj/src/kernels/scalar.cpp:51-59, impl.hpp:30-34; simd_block = 8 in fp32) */
static float sum_squares(const float* x, size_t n) {
  float p[8] = {0};
  for (size_t k = 0; k < n; ++k) { const float v = x[k]; p[k % 8] += v * v; }
  for (int h = 4; h > 0; h >>= 1)
    for (int j = 0; j < h; ++j) p[j] += p[j + h];
  return p[0];
}
void orc_field_energy(const orc_grid* g, const float* f, float* e_b) {
  const size_t V = padded(g);
  float se = 0, sb = 0;
  for (int lane = F_EX; lane <= F_EZ; ++lane)
    for (int iz = 1; iz <= g->nz; ++iz)
      for (int iy = 1; iy <= g->ny; ++iy)
        se += sum_squares(f + (size_t)lane * V + (size_t)vox(g, 1, iy, iz), (size_t)g->nx);
  for (int lane = F_BX; lane <= F_BZ; ++lane)
    for (int iz = 1; iz <= g->nz; ++iz)
      for (int iy = 1; iy <= g->ny; ++iy)
        sb += sum_squares(f + (size_t)lane * V + (size_t)vox(g, 1, iy, iz), (size_t)g->nx);
  const float hv = 0.5f * (g->hx * g->hy * g->hz);
  e_b[0] = hv * se;
  e_b[1] = hv * sb;
}
/* kinetic_energy_centered (proj/src/particles.cpp:468-501) */
float orc_kinetic_energy_centered(const orc_grid* g, float q, float m, long n_,
                                  const float* p, const int32_t* ids, const float* c) {
  const size_t V = padded(g), n = (size_t)n_;
  if (n == 0) return 0;
  const float qdt_2m = q * g->dt / (2 * m);
  float acc[8] = {0};
  for (size_t i = 0; i < n; ++i) {
    eb_t f;
    eval_eb(c, V, ids[i], FL(p, n, 0, i), FL(p, n, 1, i), FL(p, n, 2, i), &f);
    const float cx_ = FL(p, n, 3, i) + qdt_2m * f.ex;
    const float cy_ = FL(p, n, 4, i) + qdt_2m * f.ey;
    const float cz_ = FL(p, n, 5, i) + qdt_2m * f.ez;
    const float gm = gamma_of(cx_, cy_, cz_);
    acc[i % 8] += (FL(p, n, 6, i) * m) * (gm - 1.0f);
  }
  for (int h = 4; h > 0; h >>= 1)
    for (int j = 0; j < h; ++j) acc[j] += acc[j + h];
  return acc[0];
}
/* max_abs_lane (proj/src/fields.cpp:301-313) */
float orc_max_abs_lane(const orc_grid* g, const float* f, int lane) {
  const size_t V = padded(g);
  float mx = 0;
  for (int iz = 1; iz <= g->nz; ++iz)
    for (int iy = 1; iy <= g->ny; ++iy)
      for (int ix = 1; ix <= g->nx; ++ix) {
        const float v = fabsf(FL(f, V, lane, vox(g, ix, iy, iz)));
        if (v > mx) mx = v;
      }
  return mx;
}
