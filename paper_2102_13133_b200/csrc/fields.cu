// Field-side kernels for sm_100a: the per-voxel stencils of the step.
//
// Reference path restated (all /root/reference/proj):
//   load_interpolators   src/particles.cpp:42-111
//   advance_b            src/fields.cpp:113-151 (+ curl_line, src/kernels/scalar.cpp:36-41)
//   advance_e            src/fields.cpp:153-193 (+ curl_line_j, scalar.cpp:43-49)
//   unload_currents      src/fields.cpp:208-251
//   ghost_sync_fields    src/fields.cpp:35-58
//   ghost_fold_currents  src/grid.cpp:59-99
//   clear_currents       src/fields.cpp:195-201
//
// Fields live lane-major (16 lanes x padded voxels, the reference's
// field_major layout) so every stencil reads/writes unit-stride along x and
// a warp's accesses coalesce.  All of these kernels are HBM-bound
// streaming stencils; each does one pass with neighbours served from L1/L2.
// unload_currents is restated in gather form: each interior edge sums its
// <= 4 contributor voxels in ascending contributor index, which is exactly
// the order the reference's z,y,x scatter loop adds them, so J is
// bit-identical while no two threads write one edge.
#include "pic_device.cuh"
#include "pic_internal.hpp"

namespace picb {

namespace {

struct Lanes {
  float* p[F_COUNT];
};

__host__ Lanes lanes_of(Context& c) {
  Lanes L;
  for (int l = 0; l < F_COUNT; ++l) L.p[l] = c.f + (size_t)l * (size_t)c.gc.V;
  return L;
}

__device__ __forceinline__ bool interior_coords(const GridC& g, long long idx, int& ix, int& iy,
                                                int& iz) {
  const long long nxy = (long long)g.nx * g.ny;
  if (idx >= nxy * g.nz) return false;
  iz = (int)(idx / nxy);
  const int r = (int)(idx - (long long)iz * nxy);
  iy = r / g.nx;
  ix = r - iy * g.nx;
  ++ix;
  ++iy;
  ++iz;
  return true;
}

unsigned interior_blocks(const GridC& g, int threads) {
  const long long n = (long long)g.nx * g.ny * g.nz;
  return (unsigned)((n + threads - 1) / threads);
}

// ---- load_interpolators (particles.cpp:48-110) ----------------------------
// Each thread builds one voxel's record; the CTA's 256 records are staged in
// shared memory and leave as contiguous 128-bit stores (a record per thread
// stored directly is five 16-B stores 80 B apart per warp instruction: the
// LSU throttled at half the DRAM bandwidth).
// kClear: the step prologue in one launch — the accumulator (scatter_->clear)
// and the J lanes (clear_currents) zeroed by a grid-stride sweep beside the
// interpolators (disjoint data)
template <bool kClear>
__global__ void __launch_bounds__(256)
load_interpolators_kernel(GridC g, Lanes L, float4* __restrict__ out, float4* __restrict__ acc) {
  if (kClear) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (long long i = t0; i < 3 * g.V; i += stride) acc[i] = z4;
    float* __restrict__ j = L.p[F_JX];
    for (long long i = t0; i < 3 * g.V; i += stride) j[i] = 0.f;
  }
  __shared__ float4 buf[256 * kInterpF4];
  __shared__ long long sv[256];
  int ix, iy, iz;
  const bool valid = interior_coords(g, (long long)blockIdx.x * blockDim.x + threadIdx.x, ix, iy, iz);
  sv[threadIdx.x] = valid ? (long long)voxel_of(g, ix, iy, iz) : -1;
  if (valid) {
  const size_t v = (size_t)voxel_of(g, ix, iy, iz);
  const size_t sx = 1, sy = (size_t)g.sy, sz = (size_t)g.sz;
  const float* __restrict__ fex = L.p[F_EX];
  const float* __restrict__ fey = L.p[F_EY];
  const float* __restrict__ fez = L.p[F_EZ];
  float w0, w1, w2, w3;
  float4 r0, r1, r2, r3, r4;  // the paired record layout (pic_device.cuh)
  w0 = fex[v]; w1 = fex[v + sy]; w2 = fex[v + sz]; w3 = fex[v + sy + sz];
  r0.x = 0.25f * ((w3 + w0) + (w1 + w2));  // ex
  r0.z = 0.25f * ((w3 - w0) + (w1 - w2));  // dexdy
  r1.x = 0.25f * ((w3 - w0) - (w1 - w2));  // dexdz
  r1.z = 0.25f * ((w3 + w0) - (w1 + w2));  // d2exdydz
  w0 = fey[v]; w1 = fey[v + sz]; w2 = fey[v + sx]; w3 = fey[v + sz + sx];
  r0.y = 0.25f * ((w3 + w0) + (w1 + w2));  // ey
  r0.w = 0.25f * ((w3 - w0) + (w1 - w2));  // deydz
  r1.y = 0.25f * ((w3 - w0) - (w1 - w2));  // deydx
  r1.w = 0.25f * ((w3 + w0) - (w1 + w2));  // d2eydzdx
  w0 = fez[v]; w1 = fez[v + sx]; w2 = fez[v + sy]; w3 = fez[v + sx + sy];
  r2.x = 0.25f * ((w3 + w0) + (w1 + w2));
  r2.y = 0.25f * ((w3 - w0) + (w1 - w2));
  r2.z = 0.25f * ((w3 - w0) - (w1 - w2));
  r2.w = 0.25f * ((w3 + w0) - (w1 + w2));
  w0 = L.p[F_BX][v]; w1 = L.p[F_BX][v + sx];
  r3.x = 0.5f * (w1 + w0);  // cbx
  r3.z = 0.5f * (w1 - w0);  // dcbxdx
  w0 = L.p[F_BY][v]; w1 = L.p[F_BY][v + sy];
  r3.y = 0.5f * (w1 + w0);  // cby
  r3.w = 0.5f * (w1 - w0);  // dcbydy
  w0 = L.p[F_BZ][v]; w1 = L.p[F_BZ][v + sz];
  r4.x = 0.5f * (w1 + w0);
  r4.y = 0.5f * (w1 - w0);
  r4.z = 0.f;
  r4.w = 0.f;
  float4* o = buf + threadIdx.x * kInterpF4;
  o[0] = r0; o[1] = r1; o[2] = r2; o[3] = r3; o[4] = r4;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256 * kInterpF4; i += 256) {
    const long long vv = sv[i / kInterpF4];
    if (vv >= 0) out[vv * kInterpF4 + i % kInterpF4] = buf[i];
  }
}

// Periodic ghost images of one interior voxel's three lanes: every ghost
// voxel whose wrapped image is (ix, iy, iz) — what ghost_sync_kernel would
// copy there (fully periodic boxes only).  Interior cells off the faces
// have none.
__device__ __forceinline__ void write_ghost_images(const GridC& g, int ix, int iy, int iz, float* a, float* b,
                                                   float* c, float va, float vb, float vc) {
  if (ix != 1 && ix != g.nx && iy != 1 && iy != g.ny && iz != 1 && iz != g.nz) return;
  int lx[3], ly[3], lz[3], nxl = 1, nyl = 1, nzl = 1;
  lx[0] = ix; ly[0] = iy; lz[0] = iz;
  if (ix == g.nx) lx[nxl++] = 0;
  if (ix == 1) lx[nxl++] = g.nx + 1;
  if (iy == g.ny) ly[nyl++] = 0;
  if (iy == 1) ly[nyl++] = g.ny + 1;
  if (iz == g.nz) lz[nzl++] = 0;
  if (iz == 1) lz[nzl++] = g.nz + 1;
  for (int k = 0; k < nzl; ++k)
    for (int j = 0; j < nyl; ++j)
      for (int i = 0; i < nxl; ++i) {
        if (i == 0 && j == 0 && k == 0) continue;
        const size_t w = (size_t)voxel_of(g, lx[i], ly[j], lz[k]);
        a[w] = va;
        b[w] = vb;
        c[w] = vc;
      }
}

// ---- advance_b (fields.cpp:113-151) -----------------------------------------
struct BCoef {
  float c1x, c2x, c1y, c2y, c1z, c2z;
};
// kVox voxels per thread, 256 apart (each round coalesced), every load of
// every round issued before the first store: the one-voxel-per-thread form
// stalled on load latency at half the DRAM bandwidth.
constexpr int kBVox = 4;
// kImages: the step's periodic ghost sync after this update is fused in
// (B's ghost images written here; E's ghosts are unchanged since the last
// sync)
template <bool kImages, int kBVox = picb::kBVox>
__device__ __forceinline__ void advance_b_chunk(const GridC& g, const Lanes& L, const BCoef& k, long long base) {
  const size_t sx = 1, sy = (size_t)g.sy, sz = (size_t)g.sz;
  const float* __restrict__ ex = L.p[F_EX];
  const float* __restrict__ ey = L.p[F_EY];
  const float* __restrict__ ez = L.p[F_EZ];
  float* __restrict__ bx = L.p[F_BX];
  float* __restrict__ by = L.p[F_BY];
  float* __restrict__ bz = L.p[F_BZ];
  size_t v[kBVox];
  bool ok[kBVox];
  float e0[kBVox][3], e1[kBVox][6], b0[kBVox][3];
  int cx[kBVox], cy[kBVox], cz[kBVox];
#pragma unroll
  for (int r = 0; r < kBVox; ++r) {
    int ix, iy, iz;
    ok[r] = interior_coords(g, base + r * 256, ix, iy, iz);
    cx[r] = ix;
    cy[r] = iy;
    cz[r] = iz;
    v[r] = ok[r] ? (size_t)voxel_of(g, ix, iy, iz) : (size_t)g.sz + (size_t)g.sy + 1;  // a valid interior address
    const size_t w = v[r];
    e0[r][0] = ex[w]; e0[r][1] = ey[w]; e0[r][2] = ez[w];
    e1[r][0] = ez[w + sy]; e1[r][1] = ey[w + sz]; e1[r][2] = ex[w + sz];
    e1[r][3] = ez[w + sx]; e1[r][4] = ey[w + sx]; e1[r][5] = ex[w + sy];
    b0[r][0] = bx[w]; b0[r][1] = by[w]; b0[r][2] = bz[w];
  }
#pragma unroll
  for (int r = 0; r < kBVox; ++r) {
    if (!ok[r]) continue;
    const size_t w = v[r];
    // dst = (dst + c1 * (p1 - p0)) + c2 * (q1 - q0)
    const float nbx = (b0[r][0] + k.c1x * (e1[r][0] - e0[r][2])) + k.c2x * (e1[r][1] - e0[r][1]);
    const float nby = (b0[r][1] + k.c1y * (e1[r][2] - e0[r][0])) + k.c2y * (e1[r][3] - e0[r][2]);
    const float nbz = (b0[r][2] + k.c1z * (e1[r][4] - e0[r][1])) + k.c2z * (e1[r][5] - e0[r][0]);
    bx[w] = nbx;
    by[w] = nby;
    bz[w] = nbz;
    if (kImages) write_ghost_images(g, cx[r], cy[r], cz[r], bx, by, bz, nbx, nby, nbz);
  }
}

template <bool kImages, int kVox = kBVox>
__global__ void __launch_bounds__(256)
advance_b_kernel(GridC g, Lanes L, BCoef k) {
  advance_b_chunk<kImages, kVox>(g, L, k, (long long)blockIdx.x * (256 * kVox) + threadIdx.x);
}
// a box small enough that kBVox voxels per thread leave the SMs short of
// warps (C1: 287 k voxels = 281 CTAs): one voxel per thread
inline int b_vox_for(const GridC& g) {
  return (long long)g.nx * g.ny * g.nz <= 148LL * 8 * 256 * kBVox ? 1 : kBVox;
}

// ---- unload_currents (gather form) + advance_e --------------------------------
struct ECoef {
  float c1x, c2x, c1y, c2y, c1z, c2z, c3;
  float fx, fy, fz;  // unload scales h_a / (2 dt V) (fields.cpp:216-219)
};

// Adds f * val[o][i] onto jf in the order the reference's (z, y, x) voxel
// loop visits the contributors: outer axis ascending, then inner axis
// ascending.  o/i index 0 = the edge's own coordinate, 1 = the (wrapped)
// minus-one neighbour; *_minus_first tells whether the neighbour's
// coordinate is the smaller one (false only when wrapping at coordinate 1).
__device__ __forceinline__ float gather4(float jf, float f, float v00, float v01, float v10,
                                         float v11, bool outer_minus_first,
                                         bool inner_minus_first) {
  const float a0 = outer_minus_first ? (inner_minus_first ? v11 : v10) : (inner_minus_first ? v01 : v00);
  const float a1 = outer_minus_first ? (inner_minus_first ? v10 : v11) : (inner_minus_first ? v00 : v01);
  const float a2 = outer_minus_first ? (inner_minus_first ? v01 : v00) : (inner_minus_first ? v11 : v10);
  const float a3 = outer_minus_first ? (inner_minus_first ? v00 : v01) : (inner_minus_first ? v10 : v11);
  jf = jf + f * a0;
  jf = jf + f * a1;
  jf = jf + f * a2;
  jf = jf + f * a3;
  return jf;
}

template <bool kUnload, bool kAdvanceE, bool kImages>
__device__ __forceinline__ void unload_e_voxel(const GridC& g, const Lanes& L, const float* acc, const ECoef& k,
                                               long long idx) {
  int ix, iy, iz;
  if (!interior_coords(g, idx, ix, iy, iz)) return;
  const size_t v = (size_t)voxel_of(g, ix, iy, iz);
  float jx = L.p[F_JX][v], jy = L.p[F_JY][v], jz = L.p[F_JZ][v];
  if (kUnload) {
    // x-decomposed: the x-1 neighbour of ix = 1 is the ghost plane filled
    // from the low neighbour; it precedes in the reference's sum order
    // unless this slab's low face is the global periodic boundary
    // walled y / z: the -1 neighbour of the first cell is the ghost row,
    // emptied by the wall fold
    const int xm = (ix == 1 && !g.xopen) ? g.nx : ix - 1;
    const int ym = (iy == 1 && !g.ywall) ? g.ny : iy - 1;
    const int zm = (iz == 1 && !g.zwall) ? g.nz : iz - 1;
    const bool xmf = ix != 1 || (g.xopen && !g.x_low_wraps), ymf = iy != 1 || g.ywall, zmf = iz != 1 || g.zwall;
    const float* a_000 = acc + (size_t)v * 12;
    const float* a_0y0 = acc + (size_t)voxel_of(g, ix, ym, iz) * 12;
    const float* a_00z = acc + (size_t)voxel_of(g, ix, iy, zm) * 12;
    const float* a_0yz = acc + (size_t)voxel_of(g, ix, ym, zm) * 12;
    const float* a_x00 = acc + (size_t)voxel_of(g, xm, iy, iz) * 12;
    const float* a_x0z = acc + (size_t)voxel_of(g, xm, iy, zm) * 12;
    const float* a_xy0 = acc + (size_t)voxel_of(g, xm, ym, iz) * 12;
    // jfx: outer z, inner y (jx0 own, jx1 y-minus, jx2 z-minus, jx3 both)
    jx = gather4(jx, k.fx, a_000[0], a_0y0[1], a_00z[2], a_0yz[3], zmf, ymf);
    // jfy: outer z, inner x (jy0 own, jy2 x-minus, jy1 z-minus, jy3 both)
    jy = gather4(jy, k.fy, a_000[4], a_x00[6], a_00z[5], a_x0z[7], zmf, xmf);
    // jfz: outer y, inner x (jz0 own, jz1 x-minus, jz2 y-minus, jz3 both)
    jz = gather4(jz, k.fz, a_000[8], a_x00[9], a_0y0[10], a_xy0[11], ymf, xmf);
    L.p[F_JX][v] = jx;
    L.p[F_JY][v] = jy;
    L.p[F_JZ][v] = jz;
  }
  if (kAdvanceE) {
    const size_t sx = 1, sy = (size_t)g.sy, sz = (size_t)g.sz;
    const float* __restrict__ bx = L.p[F_BX];
    const float* __restrict__ by = L.p[F_BY];
    const float* __restrict__ bz = L.p[F_BZ];
    const float bxv = bx[v], byv = by[v], bzv = bz[v];
    // dst = ((dst + c1 * (p1 - p0)) + c2 * (q1 - q0)) + c3 * r
    const float nex = ((L.p[F_EX][v] + k.c1x * (bzv - bz[v - sy])) + k.c2x * (byv - by[v - sz])) + k.c3 * jx;
    const float ney = ((L.p[F_EY][v] + k.c1y * (bxv - bx[v - sz])) + k.c2y * (bzv - bz[v - sx])) + k.c3 * jy;
    const float nez = ((L.p[F_EZ][v] + k.c1z * (byv - by[v - sx])) + k.c2z * (bxv - bx[v - sy])) + k.c3 * jz;
    L.p[F_EX][v] = nex;
    L.p[F_EY][v] = ney;
    L.p[F_EZ][v] = nez;
    // the step's periodic ghost sync fused in: E's images (B's are current)
    if (kImages) write_ghost_images(g, ix, iy, iz, L.p[F_EX], L.p[F_EY], L.p[F_EZ], nex, ney, nez);
  }
}
template <bool kUnload, bool kAdvanceE, bool kImages = false>
__global__ void __launch_bounds__(256)
unload_advance_e_kernel(GridC g, Lanes L, const float* __restrict__ acc, ECoef k) {
  unload_e_voxel<kUnload, kAdvanceE, kImages>(g, L, acc, k, (long long)blockIdx.x * blockDim.x + threadIdx.x);
}

// ---- ghost_sync_fields (fields.cpp:35-58) -----------------------------------
// The reference's x -> y -> z plane copies leave every ghost voxel equal to
// its fully wrapped interior image, so one pass over the six ghost faces
// (edge/corner voxels written more than once with the same value) is
// bit-identical.
__device__ __forceinline__ int wrapc(int i, int n) { return i == 0 ? n : (i == n + 1 ? 1 : i); }

__global__ void __launch_bounds__(256)
ghost_sync_kernel(GridC g, Lanes L) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // x-decomposed: the x faces come from the neighbours (halo exchange)
  const long long fx = g.xopen ? 0 : 2LL * g.pny * g.pnz, fy = g.ywall ? 0 : 2LL * g.pnx * g.pnz,
                  fz = g.zwall ? 0 : 2LL * g.pnx * g.pny;  // walled faces: wall conditions (boundary.cu)
  int ix, iy, iz;
  if (t < fx) {
    const int side = (int)(t & 1);
    const long long r = t >> 1;
    ix = side ? g.nx + 1 : 0;
    iy = (int)(r % g.pny);
    iz = (int)(r / g.pny);
  } else if ((t -= fx) < fy) {
    const int side = (int)(t & 1);
    const long long r = t >> 1;
    iy = side ? g.ny + 1 : 0;
    ix = (int)(r % g.pnx);
    iz = (int)(r / g.pnx);
  } else if ((t -= fy) < fz) {
    const int side = (int)(t & 1);
    const long long r = t >> 1;
    iz = side ? g.nz + 1 : 0;
    ix = (int)(r % g.pnx);
    iy = (int)(r / g.pnx);
  } else {
    return;
  }
  const size_t to = (size_t)voxel_of(g, ix, iy, iz);
  const size_t from = (size_t)voxel_of(g, g.xopen ? ix : wrapc(ix, g.nx), g.ywall ? iy : wrapc(iy, g.ny),
                                      g.zwall ? iz : wrapc(iz, g.nz));
  L.p[F_EX][to] = L.p[F_EX][from];
  L.p[F_EY][to] = L.p[F_EY][from];
  L.p[F_EZ][to] = L.p[F_EZ][from];
  L.p[F_BX][to] = L.p[F_BX][from];
  L.p[F_BY][to] = L.p[F_BY][from];
  L.p[F_BZ][to] = L.p[F_BZ][from];
}

// ---- ghost_fold_currents (grid.cpp:59-99): three ordered passes ---------------
__device__ __forceinline__ void fold_slot(float* acc, size_t from, size_t to) {
  float4* a = reinterpret_cast<float4*>(acc);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float4 t = a[to * 3 + k];
    const float4 s = a[from * 3 + k];
    t.x = t.x + s.x; t.y = t.y + s.y; t.z = t.z + s.z; t.w = t.w + s.w;
    a[to * 3 + k] = t;
    a[from * 3 + k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}
__global__ void fold_x_kernel(GridC g, float* acc) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.pny * g.pnz) return;
  const int iy = (int)(t % g.pny), iz = (int)(t / g.pny);
  fold_slot(acc, voxel_of(g, 0, iy, iz), voxel_of(g, g.nx, iy, iz));
  fold_slot(acc, voxel_of(g, g.nx + 1, iy, iz), voxel_of(g, 1, iy, iz));
}
__global__ void fold_y_kernel(GridC g, float* acc) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nx * g.pnz) return;
  const int ix = (int)(t % g.nx) + 1, iz = (int)(t / g.nx);
  fold_slot(acc, voxel_of(g, ix, 0, iz), voxel_of(g, ix, g.ny, iz));
  fold_slot(acc, voxel_of(g, ix, g.ny + 1, iz), voxel_of(g, ix, 1, iz));
}
__global__ void fold_z_kernel(GridC g, float* acc) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.nx * g.ny) return;
  const int ix = (int)(t % g.nx) + 1, iy = (int)(t / g.nx) + 1;
  fold_slot(acc, voxel_of(g, ix, iy, 0), voxel_of(g, ix, iy, g.nz));
  fold_slot(acc, voxel_of(g, ix, iy, g.nz + 1), voxel_of(g, ix, iy, 1));
}

// The three passes of ghost_fold_currents (grid.cpp:78-99) in one launch
// for a fully periodic box: each ghost element folds into exactly one
// interior element (its periodic image, through the x -> y -> z chain), so
// one thread per interior element on the box's boundary shell gathers its
// sources with the passes' own additions in their order — the x pass's
// (A + A[x ghost]), then the y pass's (X + X[y ghost]), then the z pass's
// (Y + Y[z ghost]) — and zeroes every ghost it read: bit-identical to the
// sequential passes.
struct Acc12 {
  float4 a, b, c;
};
__device__ __forceinline__ Acc12 acc_ld(const float4* a, size_t v) { return {a[3 * v], a[3 * v + 1], a[3 * v + 2]}; }
__device__ __forceinline__ void acc_add(Acc12& t, const Acc12& s) {
  t.a.x = t.a.x + s.a.x; t.a.y = t.a.y + s.a.y; t.a.z = t.a.z + s.a.z; t.a.w = t.a.w + s.a.w;
  t.b.x = t.b.x + s.b.x; t.b.y = t.b.y + s.b.y; t.b.z = t.b.z + s.b.z; t.b.w = t.b.w + s.b.w;
  t.c.x = t.c.x + s.c.x; t.c.y = t.c.y + s.c.y; t.c.z = t.c.z + s.c.z; t.c.w = t.c.w + s.c.w;
}
__device__ __forceinline__ void acc_zero(float4* a, size_t v) {
  a[3 * v] = a[3 * v + 1] = a[3 * v + 2] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__device__ __forceinline__ void fold_shell_item(const GridC& g, float* acc, long long t) {
  const long long fx = 2LL * g.ny * g.nz;              // ix = 1, nx
  const long long fy = 2LL * (g.nx - 2) * g.nz;        // iy = 1, ny (2 <= ix <= nx - 1)
  const long long fz = 2LL * (g.nx - 2) * (g.ny - 2);  // iz = 1, nz (interior ix, iy)
  int ix, iy, iz;
  if (t < fx) {
    const long long r = t >> 1;
    ix = (t & 1) ? g.nx : 1;
    iy = 1 + (int)(r % g.ny);
    iz = 1 + (int)(r / g.ny);
  } else if (t < fx + fy) {
    const long long u = t - fx, r = u >> 1;
    iy = (u & 1) ? g.ny : 1;
    ix = 2 + (int)(r % (g.nx - 2));
    iz = 1 + (int)(r / (g.nx - 2));
  } else if (t < fx + fy + fz) {
    const long long u = t - fx - fy, r = u >> 1;
    iz = (u & 1) ? g.nz : 1;
    ix = 2 + (int)(r % (g.nx - 2));
    iy = 2 + (int)(r / (g.nx - 2));
  } else {
    return;
  }
  float4* a = reinterpret_cast<float4*>(acc);
  // the x pass's value at (ix, y, z): A + the x ghost that folds onto it
  auto X = [&](int y, int z) {
    Acc12 v = acc_ld(a, (size_t)voxel_of(g, ix, y, z));
    const int gx = ix == g.nx ? 0 : (ix == 1 ? g.nx + 1 : -1);
    if (gx >= 0) {
      const size_t s = (size_t)voxel_of(g, gx, y, z);
      acc_add(v, acc_ld(a, s));
      acc_zero(a, s);
    }
    return v;
  };
  // the y pass's value at (ix, iy, z)
  auto Y = [&](int z) {
    Acc12 v = X(iy, z);
    const int gy = iy == g.ny ? 0 : (iy == 1 ? g.ny + 1 : -1);
    if (gy >= 0) {
      acc_add(v, X(gy, z));
      acc_zero(a, (size_t)voxel_of(g, ix, gy, z));
    }
    return v;
  };
  Acc12 v = Y(iz);
  const int gz = iz == g.nz ? 0 : (iz == 1 ? g.nz + 1 : -1);
  if (gz >= 0) {
    acc_add(v, Y(gz));
    // the z ghost row at (ix, iy) and the ghosts of its x / y passes
    acc_zero(a, (size_t)voxel_of(g, ix, iy, gz));
  }
  const size_t tv = (size_t)voxel_of(g, ix, iy, iz);
  a[3 * tv] = v.a;
  a[3 * tv + 1] = v.b;
  a[3 * tv + 2] = v.c;
}
__global__ void fold_fused_kernel(GridC g, float* acc) {
  fold_shell_item(g, acc, (long long)blockIdx.x * blockDim.x + threadIdx.x);
}
// The periodic fold and the first B half step in one launch: they touch
// disjoint data (the accumulator; E and B), CTAs [0, nfold) fold, the rest
// advance B (sim.cpp:173-176 order kept: both precede unload + E).
template <int kVox>
__global__ void __launch_bounds__(256)
fold_advance_b_kernel(GridC g, Lanes L, float* acc, BCoef k, unsigned nfold) {
  if (blockIdx.x < nfold)
    fold_shell_item(g, acc, (long long)blockIdx.x * 256 + threadIdx.x);
  else
    advance_b_chunk<true, kVox>(g, L, k, (long long)(blockIdx.x - nfold) * (256 * kVox) + threadIdx.x);
}
__host__ __device__ __forceinline__ long long fold_shell_items(const GridC& g) {
  return 2LL * g.ny * g.nz + 2LL * (g.nx - 2) * g.nz + 2LL * (g.nx - 2) * (g.ny - 2);
}

// ---- layout conversion --------------------------------------------------------
__global__ void pack_species_kernel(const float* __restrict__ l7, const int32_t* __restrict__ ids,
                                    size_t n, float4* __restrict__ pos, float4* __restrict__ mom) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  pos[i] = make_float4(l7[i], l7[n + i], l7[2 * n + i], __int_as_float(ids[i]));
  mom[i] = make_float4(l7[3 * n + i], l7[4 * n + i], l7[5 * n + i], l7[6 * n + i]);
}
// records -> 7 lanes + ids; with lidx (a voxel-ordered store) record i
// lands at its logical index lidx[i] (the store keeps its own order)
__global__ void unpack_species_kernel(const float4* __restrict__ pos, const float4* __restrict__ mom,
                                      const unsigned* __restrict__ lidx, size_t n, float* __restrict__ l7,
                                      int32_t* __restrict__ ids) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 p = pos[i], u = mom[i];
  const size_t d = lidx ? (size_t)lidx[i] : i;
  l7[d] = p.x; l7[n + d] = p.y; l7[2 * n + d] = p.z;
  l7[3 * n + d] = u.x; l7[4 * n + d] = u.y; l7[5 * n + d] = u.z; l7[6 * n + d] = u.w;
  ids[d] = __float_as_int(p.w);
}
__global__ void interp_to_lanes_kernel(const float4* __restrict__ c, size_t V, float* __restrict__ o) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const float4* r = c + v * kInterpF4;
  const float4 a = r[0], b = r[1], d = r[2], e = r[3], h = r[4];
  const float slots[18] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w,
                           e.x, e.y, e.z, e.w, h.x, h.y};
#pragma unroll
  for (int l = 0; l < 18; ++l) o[(size_t)l * V + v] = slots[interp_slot(l)];
}
__global__ void lanes_to_interp_kernel(const float* __restrict__ in, size_t V, float4* __restrict__ c) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  float x[20];
#pragma unroll
  for (int l = 0; l < 18; ++l) x[interp_slot(l)] = in[(size_t)l * V + v];
  x[18] = 0.f;
  x[19] = 0.f;
  float4* r = c + v * kInterpF4;
#pragma unroll
  for (int k = 0; k < 5; ++k) r[k] = make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
}

// ---- synthetic load (benchmark decks): counter-based RNG ---------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float u01(uint64_t h) {  // [0, 1)
  return (float)(h >> 40) * (1.0f / 16777216.0f);
}
// Density profile of a synthetic load (uniform: bg 1, amp 0): particle
// weight w(z) = bg + amp (sech^2((z - z1) / L) + sech^2((z - z2) / L)), and
// with flip the drift changes sign for particles nearer z2 than z1 (the
// counter-propagating currents of a double Harris sheet).  z is the physical
// coordinate of the particle, (iz - 1 + (oz + 1) / 2) hz.
struct Sheet {
  float bg, amp, z1, z2, L, hz;
  int flip;
};
__global__ void load_synthetic_kernel(GridC g, int ppc, float u_th, float dx0, float dy0, float dz0,
                                      uint64_t seed, size_t n, float4* __restrict__ pos,
                                      float4* __restrict__ mom, Sheet sh) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long cell = (long long)(i / (size_t)ppc);
  int ix, iy, iz;
  interior_coords(g, cell, ix, iy, iz);
  const uint64_t base = mix64(seed ^ (0x632be59bd9b4e019ULL * (uint64_t)(i + 1)));
  const float x = 2.0f * u01(mix64(base + 1)) - 1.0f;
  const float y = 2.0f * u01(mix64(base + 2)) - 1.0f;
  const float z = 2.0f * u01(mix64(base + 3)) - 1.0f;
  float nrm[4];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float a = 1.0f - u01(mix64(base + 4 + 2 * k));  // (0, 1]
    const float b = u01(mix64(base + 5 + 2 * k));
    const float r = sqrtf(-2.0f * logf(a));
    nrm[2 * k] = r * cospif(2.0f * b);
    nrm[2 * k + 1] = r * sinpif(2.0f * b);
  }
  float w = 1.0f, sgn = 1.0f;
  if (sh.amp != 0.0f || sh.bg != 1.0f) {
    const float zp = ((float)(iz - 1) + 0.5f * (z + 1.0f)) * sh.hz;
    const float c1 = coshf((zp - sh.z1) / sh.L), c2 = coshf((zp - sh.z2) / sh.L);
    w = sh.bg + sh.amp * (1.0f / (c1 * c1) + 1.0f / (c2 * c2));
    if (sh.flip && fabsf(zp - sh.z2) < fabsf(zp - sh.z1)) sgn = -1.0f;
  }
  pos[i] = make_float4(x, y, z, __int_as_float(voxel_of(g, ix, iy, iz)));
  mom[i] = make_float4(sgn * dx0 + u_th * nrm[0], sgn * dy0 + u_th * nrm[1], sgn * dz0 + u_th * nrm[2], w);
}

}  // namespace

// ---- launchers -----------------------------------------------------------------
void launch_load_interpolators(Context& c) {
  load_interpolators_kernel<false>
      <<<interior_blocks(c.gc, 256), 256, 0, c.stream>>>(c.gc, lanes_of(c), c.interp, nullptr);
  c.count_launch();
}

// clear_accumulator + clear_currents + load_interpolators in one launch
void launch_step_prologue_fused(Context& c) {
  load_interpolators_kernel<true><<<interior_blocks(c.gc, 256), 256, 0, c.stream>>>(
      c.gc, lanes_of(c), c.interp, reinterpret_cast<float4*>(c.acc));
  c.count_launch();
}

void launch_advance_b(Context& c, float frac, bool images) {
  // constants computed on the host in real_t (fields.cpp:115-118, 133-138)
  const float fdt = frac * c.grid.dt;
  const float rhx = 1.0f / c.grid.hx, rhy = 1.0f / c.grid.hy, rhz = 1.0f / c.grid.hz;
  BCoef k;
  k.c1x = -fdt * rhy; k.c2x = fdt * rhz;
  k.c1y = -fdt * rhz; k.c2y = fdt * rhx;
  k.c1z = -fdt * rhx; k.c2z = fdt * rhy;
  const bool one = b_vox_for(c.gc) == 1;
  const unsigned nb = interior_blocks(c.gc, 256 * (one ? 1 : kBVox));
  if (images && one)
    advance_b_kernel<true, 1><<<nb, 256, 0, c.stream>>>(c.gc, lanes_of(c), k);
  else if (images)
    advance_b_kernel<true><<<nb, 256, 0, c.stream>>>(c.gc, lanes_of(c), k);
  else if (one)
    advance_b_kernel<false, 1><<<nb, 256, 0, c.stream>>>(c.gc, lanes_of(c), k);
  else
    advance_b_kernel<false><<<nb, 256, 0, c.stream>>>(c.gc, lanes_of(c), k);
  c.count_launch();
}

// fold + advance_b(1/2) of a fully periodic box in one launch
void launch_fold_advance_b(Context& c) {
  const float fdt = 0.5f * c.grid.dt;
  const float rhx = 1.0f / c.grid.hx, rhy = 1.0f / c.grid.hy, rhz = 1.0f / c.grid.hz;
  BCoef k;  // as launch_advance_b(c, 0.5f, ...)
  k.c1x = -fdt * rhy; k.c2x = fdt * rhz;
  k.c1y = -fdt * rhz; k.c2y = fdt * rhx;
  k.c1z = -fdt * rhx; k.c2z = fdt * rhy;
  const unsigned nfold = (unsigned)((fold_shell_items(c.gc) + 255) / 256);
  if (b_vox_for(c.gc) == 1)
    fold_advance_b_kernel<1><<<nfold + interior_blocks(c.gc, 256), 256, 0, c.stream>>>(c.gc, lanes_of(c), c.acc,
                                                                                       k, nfold);
  else
    fold_advance_b_kernel<kBVox><<<nfold + interior_blocks(c.gc, 256 * kBVox), 256, 0, c.stream>>>(
        c.gc, lanes_of(c), c.acc, k, nfold);
  c.count_launch();
}

void launch_unload_advance_e(Context& c, bool unload, bool advance_e, bool images) {
  const float dt = c.grid.dt;
  const float rhx = 1.0f / c.grid.hx, rhy = 1.0f / c.grid.hy, rhz = 1.0f / c.grid.hz;
  ECoef k;
  k.c1x = dt * rhy; k.c2x = -dt * rhz;   // fields.cpp:175-180
  k.c1y = dt * rhz; k.c2y = -dt * rhx;
  k.c1z = dt * rhx; k.c2z = -dt * rhy;
  k.c3 = -dt;
  const float two_dt_v = 2.0f * dt * (c.grid.hx * c.grid.hy * c.grid.hz);  // fields.cpp:216-219
  k.fx = c.grid.hx / two_dt_v;
  k.fy = c.grid.hy / two_dt_v;
  k.fz = c.grid.hz / two_dt_v;
  const unsigned b = interior_blocks(c.gc, 256);
  if (unload && advance_e && images)
    unload_advance_e_kernel<true, true, true><<<b, 256, 0, c.stream>>>(c.gc, lanes_of(c), c.acc, k);
  else if (unload && advance_e)
    unload_advance_e_kernel<true, true><<<b, 256, 0, c.stream>>>(c.gc, lanes_of(c), c.acc, k);
  else if (unload)
    unload_advance_e_kernel<true, false><<<b, 256, 0, c.stream>>>(c.gc, lanes_of(c), c.acc, k);
  else if (advance_e)
    unload_advance_e_kernel<false, true><<<b, 256, 0, c.stream>>>(c.gc, lanes_of(c), c.acc, k);
  else
    return;
  c.count_launch();
}

void launch_ghost_sync(Context& c) {
  const GridC& g = c.gc;
  const long long n = 2LL * g.pny * g.pnz + 2LL * g.pnx * g.pnz + 2LL * g.pnx * g.pny;  // >= the faces synced
  ghost_sync_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(g, lanes_of(c));
  c.count_launch();
}

void launch_ghost_fold(Context& c) {
  const GridC& g = c.gc;
  const long long nx = (long long)g.pny * g.pnz, ny = (long long)g.nx * g.pnz, nz = (long long)g.nx * g.ny;
  // x -> y -> z; a walled axis folds its mirror images / drops (boundary.cu);
  // x-decomposed: the shared x planes were folded into the neighbours by
  // exchange (a global x wall is folded here)
  if (!g.xopen && !g.ywall && !g.zwall) {
    // fully periodic: the three passes in one launch (bit-identical)
    const long long shell = fold_shell_items(g);
    fold_fused_kernel<<<(unsigned)((shell + 255) / 256), 256, 0, c.stream>>>(g, c.acc);
    c.count_launch();
    return;
  }
  if (g.xopen) {
    if (g.wall_p[0] || g.wall_p[1]) launch_wall_fold(c, 0);
  } else {
    fold_x_kernel<<<(unsigned)((nx + 255) / 256), 256, 0, c.stream>>>(g, c.acc);
    c.count_launch();
  }
  if (g.ywall) {
    launch_wall_fold(c, 1);
  } else {
    fold_y_kernel<<<(unsigned)((ny + 255) / 256), 256, 0, c.stream>>>(g, c.acc);
    c.count_launch();
  }
  if (g.zwall) {
    launch_wall_fold(c, 2);
  } else {
    fold_z_kernel<<<(unsigned)((nz + 255) / 256), 256, 0, c.stream>>>(g, c.acc);
    c.count_launch();
  }
}

void launch_clear_currents(Context& c) {
  CUDA_OK(cudaMemsetAsync(c.f + (size_t)F_JX * c.gc.V, 0, 3 * (size_t)c.gc.V * sizeof(float), c.stream));
}

void launch_clear_accumulator(Context& c) {
  CUDA_OK(cudaMemsetAsync(c.acc, 0, 12 * (size_t)c.gc.V * sizeof(float), c.stream));
}

void launch_pack_species(Context& c, Species& s, const float* l7, const int32_t* ids, size_t n) {
  if (n == 0) return;
  pack_species_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(l7, ids, n, s.pos, s.mom);
  c.count_launch();
}

void launch_unpack_species(Context& c, Species& s, float* l7, int32_t* ids) {
  if (s.n == 0) return;
  unpack_species_kernel<<<(unsigned)((s.n + 255) / 256), 256, 0, c.stream>>>(s.pos, s.mom, nullptr, s.n, l7,
                                                                              ids);
  c.count_launch();
}
void launch_unpack_logical(Context& c, const Species& s, float* l7, int32_t* ids) {
  if (s.n == 0) return;
  unpack_species_kernel<<<(unsigned)((s.n + 255) / 256), 256, 0, c.stream>>>(s.pos, s.mom, s.lidx, s.n, l7, ids);
  c.count_launch();
}

void launch_load_synthetic(Context& c, Species& s, int ppc, float u_th, const float drift[3],
                           uint64_t seed, const pic_sheet* sheet) {
  const size_t n = (size_t)ppc * (size_t)c.gc.nx * c.gc.ny * c.gc.nz;
  if (n > s.cap) throw UsageError("load_synthetic: ppc * interior voxels exceeds species capacity");
  Sheet sh{1.0f, 0.0f, 0.0f, 0.0f, 1.0f, c.grid.hz, 0};
  if (sheet) {
    if (!(sheet->half_width > 0.0f)) throw UsageError("load_harris: half_width must be > 0");
    if (sheet->background < 0.0f || sheet->amplitude < 0.0f)
      throw UsageError("load_harris: background and amplitude must be >= 0");
    sh = Sheet{sheet->background, sheet->amplitude, sheet->z1, sheet->z2, sheet->half_width, c.grid.hz,
               sheet->flip_drift ? 1 : 0};
  }
  s.n = n;
  if (n == 0) return;
  load_synthetic_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(
      c.gc, ppc, u_th, drift[0], drift[1], drift[2], seed, n, s.pos, s.mom, sh);
  c.count_launch();
}

void launch_interp_to_lanes(Context& c, float* out18) {
  interp_to_lanes_kernel<<<(unsigned)((c.gc.V + 255) / 256), 256, 0, c.stream>>>(c.interp, (size_t)c.gc.V, out18);
  c.count_launch();
}

void launch_lanes_to_interp(Context& c, const float* in18) {
  lanes_to_interp_kernel<<<(unsigned)((c.gc.V + 255) / 256), 256, 0, c.stream>>>(in18, (size_t)c.gc.V, c.interp);
  c.count_launch();
}

}  // namespace picb
