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

// Accumulator x ghost planes: reflect -> mirror image folded into the
// boundary cell (x currents negated, x lo / hi edges swapped), absorb -> the
// part beyond the wall dropped.  Every (iy, iz) of the padded plane, before
// the y / z folds (the x -> y -> z order of ghost_fold_currents).
__global__ void wall_fold_kernel(GridC g, float* __restrict__ acc) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long P = (long long)g.pny * g.pnz;
  if (t >= 2 * P) return;
  const int side = (int)(t / P);
  if (g.wall_p[side] == PIC_PBC_PERIODIC) return;  // an exchange side (decomposed)
  const long long r = t - side * P;
  const int iy = (int)(r % g.pny), iz = (int)(r / g.pny);
  const int gx = side ? g.nx + 1 : 0, bx = side ? g.nx : 1;
  float* G = acc + (size_t)voxel_of(g, gx, iy, iz) * 12;
  if (g.wall_p[side] == PIC_PBC_REFLECT) {
    float* B = acc + (size_t)voxel_of(g, bx, iy, iz) * 12;
    // jx0..3: same (y, z) edge, reversed
    B[0] = B[0] - G[0];
    B[1] = B[1] - G[1];
    B[2] = B[2] - G[2];
    B[3] = B[3] - G[3];
    // jy0 (z lo, x lo) <-> jy2 (z lo, x hi), jy1 <-> jy3
    B[6] = B[6] + G[4];
    B[7] = B[7] + G[5];
    B[4] = B[4] + G[6];
    B[5] = B[5] + G[7];
    // jz0 (x lo, y lo) <-> jz1 (x hi, y lo), jz2 <-> jz3
    B[9] = B[9] + G[8];
    B[8] = B[8] + G[9];
    B[11] = B[11] + G[10];
    B[10] = B[10] + G[11];
  }
#pragma unroll
  for (int k = 0; k < 12; ++k) G[k] = 0.f;
}

// Wall planes of (E_y, E_z): [side][0] = the wall node plane, [side][1] = the
// node plane one cell inside.  Saved before the E update for Mur.
__device__ __forceinline__ int wall_plane_ix(const GridC& g, int side, int inner) {
  return side ? g.nx + 1 - inner : 1 + inner;
}

__global__ void wall_save_kernel(GridC g, const float* __restrict__ f, float* __restrict__ save) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long P = (long long)g.pny * g.pnz;
  if (t >= 4 * P) return;
  const int plane = (int)(t / P);  // side * 2 + inner
  const long long r = t - plane * P;
  const int iy = (int)(r % g.pny), iz = (int)(r / g.pny);
  const size_t v = (size_t)voxel_of(g, wall_plane_ix(g, plane >> 1, plane & 1), iy, iz);
  save[(size_t)(2 * plane) * P + r] = f[(size_t)F_EY * g.V + v];
  save[(size_t)(2 * plane + 1) * P + r] = f[(size_t)F_EZ * g.V + v];
}

// After the E update: PEC -> tangential E = 0 on the wall plane; Mur ->
// E_w^{n+1} = E_i^n + k (E_i^{n+1} - E_w^n), k = (c dt - h) / (c dt + h).
// E_x in the x ghost cells (outside the domain) is zeroed.
__global__ void wall_e_kernel(GridC g, float* __restrict__ f, const float* __restrict__ save, float kmur) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long P = (long long)g.pny * g.pnz;
  if (t >= 2 * P) return;
  const int side = (int)(t / P);
  const int fb = g.wall_f[side];
  if (fb == PIC_FBC_PERIODIC) return;  // an exchange side (decomposed)
  const long long r = t - side * P;
  const int iy = (int)(r % g.pny), iz = (int)(r / g.pny);
  const size_t vw = (size_t)voxel_of(g, wall_plane_ix(g, side, 0), iy, iz);
  const size_t vi = (size_t)voxel_of(g, wall_plane_ix(g, side, 1), iy, iz);
  float* ey = f + (size_t)F_EY * g.V;
  float* ez = f + (size_t)F_EZ * g.V;
  if (fb == PIC_FBC_PEC) {
    ey[vw] = 0.f;
    ez[vw] = 0.f;
  } else if (fb == PIC_FBC_MUR) {
    const float* sw = save + (size_t)(4 * side) * P;   // wall plane (ey, ez)
    const float* si = save + (size_t)(4 * side + 2) * P;  // inner plane
    ey[vw] = si[r] + kmur * (ey[vi] - sw[r]);
    ez[vw] = si[P + r] + kmur * (ez[vi] - sw[P + r]);
  }
  f[(size_t)F_EX * g.V + (size_t)voxel_of(g, side ? g.nx + 1 : 0, iy, iz)] = 0.f;
}

// B_x on the high wall plane (ghost voxel nx+1, never touched by the
// interior advance_b): the same curl of the wall-plane tangential E
// (fields.cpp:113-151 expression order), interior (iy, iz).
__global__ void wall_bx_kernel(GridC g, float* __restrict__ f, float c1x, float c2x) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.ny * g.nz) return;
  const int iy = 1 + (int)(t % g.ny), iz = 1 + (int)(t / g.ny);
  const size_t v = (size_t)voxel_of(g, g.nx + 1, iy, iz);
  const float* ey = f + (size_t)F_EY * g.V;
  const float* ez = f + (size_t)F_EZ * g.V;
  float* bx = f + (size_t)F_BX * g.V;
  bx[v] = (bx[v] + c1x * (ez[v + g.sy] - ez[v])) + c2x * (ey[v + g.sz] - ey[v]);
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

bool has_walls(const Context& c) { return c.gc.wall_p[0] || c.gc.wall_p[1] || c.gc.wall_f[0] || c.gc.wall_f[1]; }

void set_x_boundary(Context& c, int side, int pbc, int fbc) {
  if (side != 0 && side != 1) throw UsageError("x boundary: side must be 0 (low) or 1 (high)");
  if (pbc < PIC_PBC_PERIODIC || pbc > PIC_PBC_REFLECT) throw UsageError("x boundary: unknown particle bc");
  if (fbc < PIC_FBC_PERIODIC || fbc > PIC_FBC_MUR) throw UsageError("x boundary: unknown field bc");
  if ((pbc == PIC_PBC_PERIODIC) != (fbc == PIC_FBC_PERIODIC))
    throw UsageError("x boundary: particles and fields must both be periodic or both walls");
  c.gc.wall_p[side] = pbc;
  c.gc.wall_f[side] = fbc;
  // one side may be set before the other; check_walls refuses a pic_step
  // with a single wall.  On a decomposed (x-open) slab a wall side is the
  // global boundary, the other side keeps exchanging.
  const bool any = has_walls(c);
  c.gc.xopen = (any || c.decomposed) ? 1 : 0;
  if (any) {
    if (c.gc.wall_p[0]) c.gc.x_low_wraps = 0;
    for (auto& s : c.species) ensure_mig_lists(c, s);
  }
}

void check_walls(const Context& c, bool deterministic) {
  if (!has_walls(c)) return;
  if (!c.gc.wall_p[0] || !c.gc.wall_p[1])
    throw UsageError("x boundary: both x sides must be walls (or both periodic)");
  if (!deterministic && (c.push_variant < 42 || c.push_variant > 52))
    throw UsageError("x boundary: supported by push variants 42-52 and the deterministic path");
}

// The wall / laser / emitter pieces of the step, for hosts that sequence the
// step themselves (the decomposed driver, domain.py); pic_step calls them in
// the same places.
void wall_stage(Context& c, int stage, float frac) {
  const bool walls = has_walls(c);
  switch (stage) {
    case PIC_STAGE_FOLD:
      if (walls) launch_wall_fold(c);
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

// After a species' push: absorbed particles (recorded as x emigrants) are
// removed; the store is compacted in index order (domain.cu).
void absorb_compact(Context& c, Species& s) {
  size_t cnt[2];
  migrate_counts(c, s, cnt);
  if (cnt[0] + cnt[1] == 0) return;
  c.absorbed[0] += cnt[0];
  c.absorbed[1] += cnt[1];
  migrate_pack(c, s, nullptr, nullptr);
}

void launch_wall_fold(Context& c) {
  const long long P = (long long)c.gc.pny * c.gc.pnz;
  wall_fold_kernel<<<nblk(2 * P), 256, 0, c.stream>>>(c.gc, c.acc);
  c.count_launch();
}

void launch_wall_e_save(Context& c) {
  if (c.gc.wall_f[0] != PIC_FBC_MUR && c.gc.wall_f[1] != PIC_FBC_MUR) return;
  const long long P = (long long)c.gc.pny * c.gc.pnz;
  float* save = static_cast<float*>(c.scratch_bytes(Context::kScrWall, (size_t)8 * P * sizeof(float)));
  wall_save_kernel<<<nblk(4 * P), 256, 0, c.stream>>>(c.gc, c.f, save);
  c.count_launch();
}

void launch_wall_e(Context& c) {
  const long long P = (long long)c.gc.pny * c.gc.pnz;
  float* save = static_cast<float*>(c.scratch_bytes(Context::kScrWall, (size_t)8 * P * sizeof(float)));
  const float cdt = c.grid.dt, h = c.grid.hx;
  wall_e_kernel<<<nblk(2 * P), 256, 0, c.stream>>>(c.gc, c.f, save, (cdt - h) / (cdt + h));
  c.count_launch();
}

void launch_wall_b(Context& c, float frac) {
  if (c.gc.wall_f[1] == PIC_FBC_PERIODIC) return;  // B_x of the high wall plane only
  const float fdt = frac * c.grid.dt;
  wall_bx_kernel<<<nblk((long long)c.gc.ny * c.gc.nz), 256, 0, c.stream>>>(c.gc, c.f, -fdt / c.grid.hy,
                                                                           fdt / c.grid.hz);
  c.count_launch();
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
