// Non-periodic x boundaries, laser source, particle emitter, slab loader
// (SURVEY §8f item 4).  NOT IN REFERENCE: minipic is periodic in every
// direction (proj/src/grid.cpp:32-99, proj/src/fields.cpp:19-58), so this
// is designed fresh on top of the x-open machinery of the decomposition
// (the x faces neither wrap nor fold), and checked by self-consistency
// tests (tests/test_gpu_boundaries.py): mirror symmetry of reflected
// particles against the periodic run, exact removal of absorbed particles,
// Gauss's law under reflection, conductor / absorbing wave tests, laser
// amplitude and arrival time.
//
// Layout reminders (lanes.hpp:23-91): E_y(ix), E_z(ix) sit on the x = (ix-1)
// hx node plane of voxel ix, so the low wall (x = 0) is voxel 1's plane and
// the high wall (x = nx hx) the ghost voxel nx+1's; B_x(ix) is on the same
// planes, B_y / B_z at cell centres in x.  Accumulator lanes: jx_k on x
// edges (y, z positions), jy (z, x) and jz (x, y) with x lo / hi.
#include <algorithm>

#include "pic_device.cuh"
#include "pic_internal.hpp"

namespace picb {

namespace {

// ---- generic plane addressing ------------------------------------------------
// Axis a's plane c_a = k, addressed by the two other axes in cyclic order
// (a + 1, a + 2): u in [u0, u0 + nu), w in [w0, w0 + nw).
__device__ __forceinline__ int plane_voxel(const GridC& g, int a, int k, int u, int w) {
  return a == 0 ? voxel_of(g, k, u, w) : (a == 1 ? voxel_of(g, w, k, u) : voxel_of(g, u, w, k));
}
__device__ __forceinline__ int axis_n(const GridC& g, int a) { return a == 0 ? g.nx : (a == 1 ? g.ny : g.nz); }

// Accumulator ghost planes of one walled axis: reflect -> the mirror image
// of the current beyond the wall folded into the boundary cell (the normal
// direction's lanes negated, lo / hi edges across the axis swapped in the
// two transverse directions), absorb -> the part beyond the wall dropped.
// Ranges and order follow ghost_fold_currents (grid.cpp:59-99): x planes over
// all (y, z), y planes over interior x and all z, z planes over interior x, y.
__global__ void wall_fold_kernel(GridC g, float* __restrict__ acc, int a, int u0, int nu, int w0, int nw) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long P = (long long)nu * nw;
  if (t >= 2 * P) return;
  const int side = (int)(t / P);
  const int pb = g.wall_p[2 * a + side];
  if (pb == PIC_PBC_PERIODIC) return;  // an exchange side (x, decomposed)
  const long long r = t - side * P;
  const int u = u0 + (int)(r % nu), w = w0 + (int)(r / nu);
  const int n = axis_n(g, a);
  float* G = acc + (size_t)plane_voxel(g, a, side ? n + 1 : 0, u, w) * 12;
  if (pb == PIC_PBC_REFLECT) {
    float* B = acc + (size_t)plane_voxel(g, a, side ? n : 1, u, w) * 12;
    // lanes: jx0..3 (y, z), jy0..3 (z, x), jz0..3 (x, y); index 2 t + s of a
    // direction's four = (lo / hi of its first, lo / hi of its second axis)
    int perm[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) perm[k] = k;
    float sg[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) sg[k] = 1.f;
    if (a == 0) {
      sg[0] = sg[1] = sg[2] = sg[3] = -1.f;
      perm[4] = 6; perm[6] = 4; perm[5] = 7; perm[7] = 5;    // jy: x is its second axis
      perm[8] = 9; perm[9] = 8; perm[10] = 11; perm[11] = 10; // jz: x is its first axis
    } else if (a == 1) {
      sg[4] = sg[5] = sg[6] = sg[7] = -1.f;
      perm[0] = 1; perm[1] = 0; perm[2] = 3; perm[3] = 2;     // jx: y is its first axis
      perm[8] = 10; perm[10] = 8; perm[9] = 11; perm[11] = 9; // jz: y is its second axis
    } else {
      sg[8] = sg[9] = sg[10] = sg[11] = -1.f;
      perm[0] = 2; perm[2] = 0; perm[1] = 3; perm[3] = 1;     // jx: z is its second axis
      perm[4] = 5; perm[5] = 4; perm[6] = 7; perm[7] = 6;     // jy: z is its first axis
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) B[perm[k]] = B[perm[k]] + sg[k] * G[k];
  }
#pragma unroll
  for (int k = 0; k < 12; ++k) G[k] = 0.f;
}

// Tangential E lanes of a wall normal to axis a, and the normal one.
__device__ __forceinline__ int tan_lane(int a, int i) {
  return a == 0 ? (i ? F_EZ : F_EY) : (a == 1 ? (i ? F_EX : F_EZ) : (i ? F_EY : F_EX));
}

// Mur's saved planes: for each face [wall plane (t0, t1), inner plane (t0, t1)]
// in save + face * 4 * Pmax.
__global__ void wall_save_kernel(GridC g, const float* __restrict__ f, float* __restrict__ save, int a, int side,
                                 int nu, int nw, long long pmax) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long P = (long long)nu * nw;
  if (t >= 2 * P) return;
  const int inner = (int)(t / P);
  const long long r = t - inner * P;
  const int u = (int)(r % nu), w = (int)(r / nu);
  const int n = axis_n(g, a);
  const int k = side ? n + 1 - inner : 1 + inner;
  const size_t v = (size_t)plane_voxel(g, a, k, u, w);
  float* sv = save + (size_t)(2 * a + side) * 4 * pmax + (size_t)(2 * inner) * pmax;
  sv[r] = f[(size_t)tan_lane(a, 0) * g.V + v];
  sv[pmax + r] = f[(size_t)tan_lane(a, 1) * g.V + v];
}

// After the E update: PEC -> tangential E = 0 on the wall plane; Mur ->
// E_w^{n+1} = E_i^n + k (E_i^{n+1} - E_w^n), k = (c dt - h_a) / (c dt + h_a).
// The normal E in the ghost cells beyond the wall (outside) is zeroed.
__global__ void wall_e_kernel(GridC g, float* __restrict__ f, const float* __restrict__ save, int a, int side,
                              int nu, int nw, long long pmax, float kmur) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long P = (long long)nu * nw;
  if (t >= P) return;
  const int u = (int)(t % nu), w = (int)(t / nu);
  const int n = axis_n(g, a);
  const int fb = g.wall_f[2 * a + side];
  const size_t vw = (size_t)plane_voxel(g, a, side ? n + 1 : 1, u, w);
  const size_t vi = (size_t)plane_voxel(g, a, side ? n : 2, u, w);
  float* e0 = f + (size_t)tan_lane(a, 0) * g.V;
  float* e1 = f + (size_t)tan_lane(a, 1) * g.V;
  if (fb == PIC_FBC_PEC) {
    e0[vw] = 0.f;
    e1[vw] = 0.f;
  } else if (fb == PIC_FBC_MUR) {
    const float* sv = save + (size_t)(2 * a + side) * 4 * pmax;
    e0[vw] = sv[2 * pmax + t] + kmur * (e0[vi] - sv[t]);
    e1[vw] = sv[3 * pmax + t] + kmur * (e1[vi] - sv[pmax + t]);
  }
  f[(size_t)(F_EX + a) * g.V + (size_t)plane_voxel(g, a, side ? n + 1 : 0, u, w)] = 0.f;
}

// B normal to the high wall plane (ghost plane n_a + 1, never touched by the
// interior advance_b): the same curl of the wall-plane tangential E
// (fields.cpp:113-151 expression order), interior (u, w).
__global__ void wall_bn_kernel(GridC g, float* __restrict__ f, int a, float c1, float c2) {
  const int n = axis_n(g, a);
  const int nu = a == 0 ? g.ny : (a == 1 ? g.nz : g.nx), nw = a == 0 ? g.nz : (a == 1 ? g.nx : g.ny);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)nu * nw) return;
  const size_t v = (size_t)plane_voxel(g, a, n + 1, 1 + (int)(t % nu), 1 + (int)(t / nu));
  const size_t sx = 1, sy = (size_t)g.sy, sz = (size_t)g.sz;
  const float* ex = f + (size_t)F_EX * g.V;
  const float* ey = f + (size_t)F_EY * g.V;
  const float* ez = f + (size_t)F_EZ * g.V;
  if (a == 0) {
    float* bx = f + (size_t)F_BX * g.V;
    bx[v] = (bx[v] + c1 * (ez[v + sy] - ez[v])) + c2 * (ey[v + sz] - ey[v]);
  } else if (a == 1) {
    float* by = f + (size_t)F_BY * g.V;
    by[v] = (by[v] + c1 * (ex[v + sz] - ex[v])) + c2 * (ez[v + sx] - ez[v]);
  } else {
    float* bz = f + (size_t)F_BZ * g.V;
    bz[v] = (bz[v] + c1 * (ey[v + sx] - ey[v])) + c2 * (ex[v + sy] - ex[v]);
  }
}

__global__ void laser_kernel(GridC g, float* __restrict__ f, int ix, int lanei, float amp, float y0, float z0,
                             float inv_w2) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.ny * g.nz) return;
  const int iy = 1 + (int)(t % g.ny), iz = 1 + (int)(t / g.ny);
  float prof = 1.0f;
  if (inv_w2 > 0.f) {
    // E_y sits at y cell centres, E_z at z cell centres
    const float y = (lanei == F_EY ? (float)iy - 0.5f : (float)(iy - 1)) * g.hy;
    const float z = (lanei == F_EZ ? (float)iz - 0.5f : (float)(iz - 1)) * g.hz;
    prof = __expf(-((y - y0) * (y - y0) + (z - z0) * (z - z0)) * inv_w2);
  }
  float* e = f + (size_t)lanei * g.V;
  e[(size_t)voxel_of(g, ix, iy, iz)] += amp * prof;
}

__device__ __forceinline__ uint64_t mix64b(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float u01b(uint64_t h) { return (float)(h >> 40) * (1.0f / 16777216.0f); }

// per_cell particles in every (iy, iz) boundary cell of the side; cell =
// i / per_cell in (y, z) order.  x offset uniform in [-1, 1); u = drift +
// u_th N(0, 1) with the x component directed into the domain.
__global__ void emit_kernel(GridC g, int side, int per_cell, float u_th, float dx0, float dy0, float dz0,
                            uint64_t seed, size_t n, float4* __restrict__ pos, float4* __restrict__ mom) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long cell = (long long)(i / (size_t)per_cell);
  const int iy = 1 + (int)(cell % g.ny), iz = 1 + (int)(cell / g.ny);
  const int ix = side ? g.nx : 1;
  const uint64_t base = mix64b(seed ^ (0x632be59bd9b4e019ULL * (uint64_t)(i + 1)));
  float nrm[4];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float a = 1.0f - u01b(mix64b(base + 4 + 2 * k));
    const float b = u01b(mix64b(base + 5 + 2 * k));
    const float rr = sqrtf(-2.0f * logf(a));
    nrm[2 * k] = rr * cospif(2.0f * b);
    nrm[2 * k + 1] = rr * sinpif(2.0f * b);
  }
  float ux = fabsf(dx0 + u_th * nrm[0]);
  if (side) ux = -ux;
  pos[i] = make_float4(2.0f * u01b(mix64b(base + 1)) - 1.0f, 2.0f * u01b(mix64b(base + 2)) - 1.0f,
                       2.0f * u01b(mix64b(base + 3)) - 1.0f, __int_as_float(voxel_of(g, ix, iy, iz)));
  mom[i] = make_float4(ux, dy0 + u_th * nrm[1], dz0 + u_th * nrm[2], 1.0f);
}

// load_synthetic over the cells with ix in [lo, hi] (x fastest, then y, z)
__global__ void load_slab_kernel(GridC g, int lo, int nxr, int ppc, float u_th, float dx0, float dy0, float dz0,
                                 uint64_t seed, size_t n, float4* __restrict__ pos, float4* __restrict__ mom) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long cell = (long long)(i / (size_t)ppc);
  const int ix = lo + (int)(cell % nxr);
  const long long r = cell / nxr;
  const int iy = 1 + (int)(r % g.ny), iz = 1 + (int)(r / g.ny);
  const uint64_t base = mix64b(seed ^ (0x632be59bd9b4e019ULL * (uint64_t)(i + 1)));
  float nrm[4];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float a = 1.0f - u01b(mix64b(base + 4 + 2 * k));
    const float b = u01b(mix64b(base + 5 + 2 * k));
    const float rr = sqrtf(-2.0f * logf(a));
    nrm[2 * k] = rr * cospif(2.0f * b);
    nrm[2 * k + 1] = rr * sinpif(2.0f * b);
  }
  pos[i] = make_float4(2.0f * u01b(mix64b(base + 1)) - 1.0f, 2.0f * u01b(mix64b(base + 2)) - 1.0f,
                       2.0f * u01b(mix64b(base + 3)) - 1.0f, __int_as_float(voxel_of(g, ix, iy, iz)));
  mom[i] = make_float4(dx0 + u_th * nrm[0], dy0 + u_th * nrm[1], dz0 + u_th * nrm[2], 1.0f);
}

inline unsigned nblk(long long n) { return (unsigned)((n + 255) / 256); }

}  // namespace

bool has_walls(const Context& c) {
  for (int k = 0; k < 6; ++k)
    if (c.gc.wall_p[k] || c.gc.wall_f[k]) return true;
  return false;
}

static bool axis_walled(const GridC& g, int a) { return g.wall_p[2 * a] || g.wall_p[2 * a + 1]; }

void set_boundary(Context& c, int face, int pbc, int fbc) {
  if (face < 0 || face > 5) throw UsageError("boundary: face must be 0-5 (x low, x high, y low, ..., z high)");
  if (pbc < PIC_PBC_PERIODIC || pbc > PIC_PBC_REFLECT) throw UsageError("boundary: unknown particle bc");
  if (fbc < PIC_FBC_PERIODIC || fbc > PIC_FBC_MUR) throw UsageError("boundary: unknown field bc");
  if ((pbc == PIC_PBC_PERIODIC) != (fbc == PIC_FBC_PERIODIC))
    throw UsageError("boundary: particles and fields must both be periodic or both walls");
  if (face >= 2 && c.decomposed && pbc != PIC_PBC_PERIODIC)
    throw UsageError("boundary: y / z walls on an x-decomposed slab");
  c.gc.wall_p[face] = pbc;
  c.gc.wall_f[face] = fbc;
  // one face may be set before the other; check_walls refuses a pic_step
  // with a single wall on an axis.  On a decomposed (x-open) slab an x wall
  // side is the global boundary, the other side keeps exchanging.
  const bool xw = axis_walled(c.gc, 0);
  c.gc.xopen = (xw || c.decomposed) ? 1 : 0;
  if (xw && c.gc.wall_p[0]) c.gc.x_low_wraps = 0;
  c.gc.ywall = axis_walled(c.gc, 1) ? 1 : 0;
  c.gc.zwall = axis_walled(c.gc, 2) ? 1 : 0;
  if (has_walls(c))
    for (auto& s : c.species) ensure_mig_lists(c, s);
}

void set_x_boundary(Context& c, int side, int pbc, int fbc) {
  if (side != 0 && side != 1) throw UsageError("x boundary: side must be 0 (low) or 1 (high)");
  set_boundary(c, side, pbc, fbc);
}

void check_walls(const Context& c, bool deterministic) {
  if (!has_walls(c)) return;
  for (int a = 0; a < 3; ++a)
    if (axis_walled(c.gc, a) && (!c.gc.wall_p[2 * a] || !c.gc.wall_p[2 * a + 1]))
      throw UsageError("boundary: both faces of an axis must be walls (or both periodic)");
  if (!deterministic && (c.push_variant < 42 || c.push_variant > 55))
    throw UsageError("boundary: walls are supported by push variants 42-55 and the deterministic path");
}

bool absorbing_walls(const Context& c) {
  for (int k = 0; k < 6; ++k)
    if (c.gc.wall_p[k] == PIC_PBC_ABSORB) return true;
  return false;
}

// The wall / laser / emitter pieces of the step, for hosts that sequence the
// step themselves (the decomposed driver, domain.py); pic_step calls them in
// the same places.  (The accumulator's wall folds run inside
// pic_ghost_fold_currents, in the x -> y -> z order; FOLD is kept for hosts
// written against it and does nothing.)
void wall_stage(Context& c, int stage, float frac) {
  const bool walls = has_walls(c);
  switch (stage) {
    case PIC_STAGE_FOLD:
      break;
    case PIC_STAGE_AFTER_B:
      if (walls) launch_wall_b(c, frac);
      break;
    case PIC_STAGE_BEFORE_E:
      if (walls) launch_wall_e_save(c);
      break;
    case PIC_STAGE_AFTER_E:
      launch_laser(c);
      if (walls) launch_wall_e(c);
      ++c.steps_done;
      break;
    case PIC_STAGE_EMIT:
      if (!c.emitters.empty()) run_emitters(c);
      break;
    default:
      throw UsageError("wall_stage: unknown stage");
  }
}

// After a species' push: absorbed particles (recorded in the emigrant lists:
// low faces in the first, high faces in the second) are removed; the store
// is compacted in index order (domain.cu).
void absorb_compact(Context& c, Species& s) {
  size_t cnt[2];
  migrate_counts(c, s, cnt);
  if (cnt[0] + cnt[1] == 0) return;
  c.absorbed[0] += cnt[0];
  c.absorbed[1] += cnt[1];
  migrate_pack(c, s, nullptr, nullptr);
}

// The accumulator's ghost planes of walled axis a (fields.cu launch_ghost_fold
// calls this in place of the periodic fold of that axis).
void launch_wall_fold(Context& c, int a) {
  const GridC& g = c.gc;
  int u0, nu, w0, nw;
  if (a == 0) { u0 = 0; nu = g.pny; w0 = 0; nw = g.pnz; }       // (y, z) padded
  else if (a == 1) { u0 = 0; nu = g.pnz; w0 = 1; nw = g.nx; }   // (z padded, x interior)
  else { u0 = 1; nu = g.nx; w0 = 1; nw = g.ny; }                // (x, y) interior
  wall_fold_kernel<<<nblk(2LL * nu * nw), 256, 0, c.stream>>>(g, c.acc, a, u0, nu, w0, nw);
  c.count_launch();
}

static void plane_dims(const GridC& g, int a, int& nu, int& nw) {
  nu = a == 0 ? g.pny : (a == 1 ? g.pnz : g.pnx);
  nw = a == 0 ? g.pnz : (a == 1 ? g.pnx : g.pny);
}
static long long plane_max(const GridC& g) {
  return std::max({(long long)g.pny * g.pnz, (long long)g.pnz * g.pnx, (long long)g.pnx * g.pny});
}

void launch_wall_e_save(Context& c) {
  const GridC& g = c.gc;
  const long long pmax = plane_max(g);
  float* save = nullptr;
  for (int face = 0; face < 6; ++face) {
    if (g.wall_f[face] != PIC_FBC_MUR) continue;
    if (!save) save = static_cast<float*>(c.scratch_bytes(Context::kScrWall, (size_t)24 * pmax * sizeof(float)));
    int nu, nw;
    plane_dims(g, face / 2, nu, nw);
    wall_save_kernel<<<nblk(2LL * nu * nw), 256, 0, c.stream>>>(g, c.f, save, face / 2, face & 1, nu, nw, pmax);
    c.count_launch();
  }
}

void launch_wall_e(Context& c) {
  const GridC& g = c.gc;
  const long long pmax = plane_max(g);
  float* save = static_cast<float*>(c.scratch_bytes(Context::kScrWall, (size_t)24 * pmax * sizeof(float)));
  const float cdt = c.grid.dt;
  const float h[3] = {c.grid.hx, c.grid.hy, c.grid.hz};
  for (int face = 0; face < 6; ++face) {
    if (g.wall_f[face] == PIC_FBC_PERIODIC) continue;
    const int a = face / 2;
    int nu, nw;
    plane_dims(g, a, nu, nw);
    wall_e_kernel<<<nblk((long long)nu * nw), 256, 0, c.stream>>>(g, c.f, save, a, face & 1, nu, nw, pmax,
                                                                  (cdt - h[a]) / (cdt + h[a]));
    c.count_launch();
  }
}

void launch_wall_b(Context& c, float frac) {
  const GridC& g = c.gc;
  const float fdt = frac * c.grid.dt;
  const float rhx = 1.0f / c.grid.hx, rhy = 1.0f / c.grid.hy, rhz = 1.0f / c.grid.hz;
  const float c1[3] = {-fdt * rhy, -fdt * rhz, -fdt * rhx}, c2[3] = {fdt * rhz, fdt * rhx, fdt * rhy};
  for (int a = 0; a < 3; ++a) {
    if (g.wall_f[2 * a + 1] == PIC_FBC_PERIODIC) continue;  // B normal to the high wall plane only
    const long long n = a == 0 ? (long long)g.ny * g.nz : (a == 1 ? (long long)g.nz * g.nx : (long long)g.nx * g.ny);
    wall_bn_kernel<<<nblk(n), 256, 0, c.stream>>>(g, c.f, a, c1[a], c2[a]);
    c.count_launch();
  }
}

void launch_laser(Context& c) {
  const pic_laser& L = c.laser;
  if (L.e0 == 0.f) return;
  const double t = (double)c.steps_done * c.grid.dt;  // E^{n+1} time level minus dt/2 (source centred)
  double s = std::sin((double)L.omega * (t + 0.5 * c.grid.dt));
  if (L.ramp_steps > 0 && c.steps_done < L.ramp_steps) {
    const double q = std::sin(0.5 * 3.14159265358979323846 * (double)c.steps_done / L.ramp_steps);
    s *= q * q;
  }
  const float amp = (float)((double)c.grid.dt * 2.0 * L.e0 / c.grid.hx * s);
  const float inv_w2 = L.waist > 0.f ? 1.0f / (L.waist * L.waist) : 0.f;
  laser_kernel<<<nblk((long long)c.gc.ny * c.gc.nz), 256, 0, c.stream>>>(c.gc, c.f, L.ix, L.pol == 2 ? F_EZ : F_EY,
                                                                         amp, L.y0, L.z0, inv_w2);
  c.count_launch();
}

void run_emitters(Context& c) {
  for (auto& e : c.emitters) {
    Species& s = c.species.at((size_t)e.species);
    const size_t n = (size_t)e.per_cell * (size_t)c.gc.ny * c.gc.nz;
    if (s.n + n > s.cap) throw RunAbort("emitter: species capacity exceeded");
    emit_kernel<<<nblk((long long)n), 256, 0, c.stream>>>(c.gc, e.side, e.per_cell, e.u_th, e.drift[0], e.drift[1],
                                                          e.drift[2], e.seed + 0x9e3779b97f4a7c15ULL * (uint64_t)(c.steps_done + 1),
                                                          n, s.pos + s.n, s.mom + s.n);
    c.count_launch();
    s.n += n;
  }
}

void load_slab(Context& c, Species& s, int ppc, float u_th, const float drift[3], uint64_t seed, int lo, int hi) {
  if (ppc < 0) throw UsageError("load_slab: ppc must be >= 0");
  if (lo < 1 || hi > c.gc.nx || lo > hi) throw UsageError("load_slab: need 1 <= ix_lo <= ix_hi <= nx");
  const int nxr = hi - lo + 1;
  const size_t n = (size_t)ppc * nxr * (size_t)c.gc.ny * c.gc.nz;
  if (n > s.cap) throw UsageError("load_slab: ppc * slab cells exceeds species capacity");
  s.n = n;
  if (n == 0) return;
  load_slab_kernel<<<nblk((long long)n), 256, 0, c.stream>>>(c.gc, lo, nxr, ppc, u_th, drift[0], drift[1], drift[2],
                                                             seed, n, s.pos, s.mom);
  c.count_launch();
}

}  // namespace picb
