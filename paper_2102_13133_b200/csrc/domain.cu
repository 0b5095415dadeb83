// Domain decomposition in x: the device side of the three
// per-step exchanges of a slab-decomposed run, replacing the periodic
// x-wrap of the single-domain reference path:
//
//   particle migration   replaces wrap_periodic in x     (particles.cpp:348-350, grid.cpp:32-52)
//   accumulator halo-add replaces ghost_fold_currents' x  (grid.cpp:78-86)
//   field halo copy      replaces ghost_sync_fields' x    (fields.cpp:35-44)
//
// The library only packs / unpacks device buffers; the transport (NCCL
// send/recv through torch.distributed, or an in-process copy) is the host's
// (paper_2102_13133_b200/domain.py).  Everything here is deterministic: the
// emigrant lists appended by the push (atomics, arbitrary order) are sorted
// before use, holes left by emigrants are filled from the tail in index
// order, and immigrants are appended in the order received.
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "pic_device.cuh"
#include "pic_internal.hpp"

namespace picb {

namespace {

// (iy, iz) of plane element t, iy fastest, padded ranges
__device__ __forceinline__ size_t plane_voxel(const GridC& g, int ix, long long t) {
  const int iy = (int)(t % g.pny), iz = (int)(t / g.pny);
  return (size_t)voxel_of(g, ix, iy, iz);
}

__global__ void pack_acc_plane(GridC g, int ix, float4* __restrict__ acc, float4* __restrict__ dst, int zero) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.pny * g.pnz) return;
  const size_t v = plane_voxel(g, ix, t);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    dst[t * 3 + k] = acc[v * 3 + k];
    if (zero) acc[v * 3 + k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}
__global__ void unpack_acc_plane(GridC g, int ix, float4* __restrict__ acc, const float4* __restrict__ src,
                                 int accumulate) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)g.pny * g.pnz) return;
  const size_t v = plane_voxel(g, ix, t);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float4 s = src[t * 3 + k];
    if (accumulate) {  // fold_slot's `to += from` (grid.cpp:66-75)
      float4 a = acc[v * 3 + k];
      a.x = a.x + s.x; a.y = a.y + s.y; a.z = a.z + s.z; a.w = a.w + s.w;
      acc[v * 3 + k] = a;
    } else {
      acc[v * 3 + k] = s;
    }
  }
}
// field lanes: 6 (E, B) or 1 (rhof), lane-major source, plane-major buffer
__global__ void pack_field_plane(GridC g, int ix, float* __restrict__ f, int lane0, int nl, int stride,
                                 float* __restrict__ dst, int zero) {
  const long long P = (long long)g.pny * g.pnz;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P) return;
  const size_t v = plane_voxel(g, ix, t);
  for (int l = 0; l < nl; ++l) {
    float* a = f + (size_t)(lane0 + l * stride) * (size_t)g.V + v;
    dst[l * P + t] = *a;
    if (zero) *a = 0.f;
  }
}
__global__ void unpack_field_plane(GridC g, int ix, float* __restrict__ f, int lane0, int nl, int stride,
                                   const float* __restrict__ src, int accumulate) {
  const long long P = (long long)g.pny * g.pnz;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P) return;
  const size_t v = plane_voxel(g, ix, t);
  for (int l = 0; l < nl; ++l) {
    float* a = f + (size_t)(lane0 + l * stride) * (size_t)g.V + v;
    *a = accumulate ? *a + src[l * P + t] : src[l * P + t];
  }
}

// Migration.  e[0..nl) = sorted low-face emigrants, e[nl..nl+nh) = sorted
// high-face emigrants.  Records go to the buffers with the x coordinate
// moved into the receiver's frame (equal slabs: low-face emigrants land in
// the receiver's ix = nx, high-face ones in ix = 1).
__global__ void mig_pack_kernel(GridC g, const unsigned* __restrict__ e, unsigned nl, unsigned nh,
                                const float4* __restrict__ pos, const float4* __restrict__ mom,
                                float4* __restrict__ low, float4* __restrict__ high) {
  const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl + nh) return;
  const unsigned i = e[k];
  float4 p = pos[i];
  const int v = __float_as_int(p.w);
  const unsigned rest = fast_div((unsigned)v, g.mag_pnx);
  const int ix = v - (int)rest * g.pnx;
  const int nxr = ix == 0 ? g.nx : 1;
  p.w = __int_as_float(v - ix + nxr);
  float4* d = k < nl ? low + 2 * (size_t)k : high + 2 * (size_t)(k - nl);
  d[0] = p;
  d[1] = mom[i];
}

// Hole filling: the store shrinks to n' = n - E.  hole k = k-th emigrant
// index below n'; filler k = k-th non-emigrant index in [n', n).  all[] is
// the merged sorted list of the E emigrant indices.  One thread per slot of
// the tail [n', n) computes its filler ordinal by counting (E is small).
__global__ void mig_fill_kernel(const unsigned* __restrict__ all, unsigned E, unsigned long long nnew,
                                unsigned nholes, float4* __restrict__ pos, float4* __restrict__ mom) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= E) return;
  const unsigned long long idx = nnew + t;
  // is idx an emigrant? binary search in all[nholes, E)
  unsigned lo = nholes, hi = E;
  while (lo < hi) {
    const unsigned mid = (lo + hi) >> 1;
    if (all[mid] < idx) lo = mid + 1;
    else hi = mid;
  }
  if (lo < E && all[lo] == idx) return;
  // filler ordinal = t - (#emigrants in [nnew, idx)) = t - (lo - nholes)
  const unsigned k = t - (lo - nholes);
  if (k >= nholes) return;
  const unsigned hole = all[k];
  pos[hole] = pos[idx];
  mom[hole] = mom[idx];
}

}  // namespace

void ensure_mig_lists(Context& c, Species& s) {
  // a slab's particles leave only from its two boundary cell planes (one
  // cell per step at most, CFL); size for four times the uniform share
  const size_t nxl = (size_t)std::max(c.gc.nx, 1);
  const size_t want = std::min<size_t>(std::max<size_t>(s.cap, 1), 4 * s.cap / nxl + 65536);
  if (s.mig_idx && s.mig_cap >= want) return;
  CUDA_OK(cudaStreamSynchronize(c.stream));
  cudaFree(s.mig_idx);
  cudaFree(s.mig_count);
  s.mig_idx = nullptr;
  s.mig_count = nullptr;
  CUDA_OK(cudaMalloc(&s.mig_idx, 2 * want * sizeof(unsigned)));
  CUDA_OK(cudaMalloc(&s.mig_count, 2 * sizeof(unsigned)));
  CUDA_OK(cudaMemsetAsync(s.mig_count, 0, 2 * sizeof(unsigned), c.stream));
  s.mig_cap = (unsigned)want;
}

void set_x_open(Context& c, bool open, bool low_wraps) {
  if (!open && (c.gc.wall_p[0] || c.gc.wall_p[1])) throw UsageError("x-open: the context has x walls (pic_set_x_boundary)");
  if (open && (c.gc.ywall || c.gc.zwall)) throw UsageError("x-open: y / z walls are single-domain only");
  c.decomposed = open;
  c.gc.xopen = (open || has_walls(c)) ? 1 : 0;
  c.gc.x_low_wraps = low_wraps ? 1 : 0;
  if (open)
    for (auto& s : c.species) ensure_mig_lists(c, s);
}

size_t halo_plane_bytes(const Context& c, int kind) {
  const size_t P = (size_t)c.gc.pny * (size_t)c.gc.pnz;
  switch (kind) {
    case 0: return P * 12 * sizeof(float);
    case 1: return P * 6 * sizeof(float);
    case 2: return P * sizeof(float);
    default: throw UsageError("halo: kind must be 0 (accumulator), 1 (E, B) or 2 (rhof)");
  }
}

static void check_plane(const Context& c, int ix) {
  if (ix < 0 || ix > c.gc.nx + 1) throw UsageError("halo: plane index outside [0, nx + 1]");
}

void halo_pack(Context& c, int kind, int ix, void* dst, bool zero_after) {
  halo_plane_bytes(c, kind);
  check_plane(c, ix);
  const long long P = (long long)c.gc.pny * c.gc.pnz;
  const unsigned b = (unsigned)((P + 255) / 256);
  if (kind == 0)
    pack_acc_plane<<<b, 256, 0, c.stream>>>(c.gc, ix, reinterpret_cast<float4*>(c.acc),
                                            static_cast<float4*>(dst), zero_after);
  else if (kind == 1)  // ex, ey, ez (lanes 0-2) and cbx, cby, cbz (4-6)
    pack_field_plane<<<b, 256, 0, c.stream>>>(c.gc, ix, c.f, 0, 3, 1, static_cast<float*>(dst), zero_after),
    pack_field_plane<<<b, 256, 0, c.stream>>>(c.gc, ix, c.f, F_BX, 3, 1, static_cast<float*>(dst) + 3 * P,
                                              zero_after);
  else
    pack_field_plane<<<b, 256, 0, c.stream>>>(c.gc, ix, c.f, F_RHO, 1, 1, static_cast<float*>(dst), zero_after);
  c.count_launch(kind == 1 ? 2 : 1);
}

void halo_unpack(Context& c, int kind, int ix, const void* src, bool accumulate) {
  halo_plane_bytes(c, kind);
  check_plane(c, ix);
  const long long P = (long long)c.gc.pny * c.gc.pnz;
  const unsigned b = (unsigned)((P + 255) / 256);
  if (kind == 0)
    unpack_acc_plane<<<b, 256, 0, c.stream>>>(c.gc, ix, reinterpret_cast<float4*>(c.acc),
                                              static_cast<const float4*>(src), accumulate);
  else if (kind == 1)
    unpack_field_plane<<<b, 256, 0, c.stream>>>(c.gc, ix, c.f, 0, 3, 1, static_cast<const float*>(src), accumulate),
    unpack_field_plane<<<b, 256, 0, c.stream>>>(c.gc, ix, c.f, F_BX, 3, 1,
                                                static_cast<const float*>(src) + 3 * P, accumulate);
  else
    unpack_field_plane<<<b, 256, 0, c.stream>>>(c.gc, ix, c.f, F_RHO, 1, 1, static_cast<const float*>(src),
                                                accumulate);
  c.count_launch(kind == 1 ? 2 : 1);
}

void migrate_counts(Context& c, Species& s, size_t out[2]) {
  out[0] = out[1] = 0;
  if ((!c.gc.xopen && !c.gc.ywall && !c.gc.zwall) || !s.mig_count) return;
  unsigned h[2];
  CUDA_OK(cudaMemcpyAsync(h, s.mig_count, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
  if (h[0] > s.mig_cap || h[1] > s.mig_cap)
    throw RunAbort("migration: emigrant list overflow (more particles left the slab than its capacity)");
  out[0] = h[0];
  out[1] = h[1];
}

// Sorts the two emigrant lists (ascending particle index), packs them, and
// compacts the store.  Requires migrate_counts first (same push).
void migrate_pack(Context& c, Species& s, void* low_dst, void* high_dst) {
  size_t cnt[2];
  migrate_counts(c, s, cnt);
  const unsigned nl = (unsigned)cnt[0], nh = (unsigned)cnt[1], E = nl + nh;
  if (E == 0) return;
  // sorted copies: e = [low sorted | high sorted], all = merged sorted
  unsigned* e = reinterpret_cast<unsigned*>(c.scratch_bytes(Context::kScrMigA, (size_t)E * 4));
  unsigned* all = reinterpret_cast<unsigned*>(c.scratch_bytes(Context::kScrMigB, (size_t)E * 4));
  size_t tmp_bytes = 0;
  CUDA_OK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, s.mig_idx, e, (int)E, 0, 32, c.stream));
  size_t need = tmp_bytes;
  void* tmp = c.scratch_bytes(Context::kScrMigT, need + 256);
  if (nl) {
    tmp_bytes = need;
    CUDA_OK(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, s.mig_idx, e, (int)nl, 0, 32, c.stream));
  }
  if (nh) {
    tmp_bytes = need;
    CUDA_OK(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, s.mig_idx + s.mig_cap, e + nl, (int)nh, 0, 32,
                                           c.stream));
  }
  // all = sort([raw low | raw high])
  unsigned* raw = reinterpret_cast<unsigned*>(c.scratch_bytes(Context::kScrMigC, (size_t)E * 4));
  CUDA_OK(cudaMemcpyAsync(raw, s.mig_idx, (size_t)nl * 4, cudaMemcpyDeviceToDevice, c.stream));
  CUDA_OK(cudaMemcpyAsync(raw + nl, s.mig_idx + s.mig_cap, (size_t)nh * 4, cudaMemcpyDeviceToDevice, c.stream));
  tmp_bytes = need;
  CUDA_OK(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, raw, all, (int)E, 0, 32, c.stream));
  if (low_dst || high_dst)  // absorbing walls discard (boundary.cu)
    mig_pack_kernel<<<(E + 255) / 256, 256, 0, c.stream>>>(c.gc, e, nl, nh, s.pos, s.mom,
                                                           static_cast<float4*>(low_dst),
                                                           static_cast<float4*>(high_dst));
  // holes below n' = n - E: the emigrants with index < n' (a prefix of all[])
  const unsigned long long nnew = (unsigned long long)s.n - E;
  std::vector<unsigned> h_all(E);
  CUDA_OK(cudaMemcpyAsync(h_all.data(), all, (size_t)E * 4, cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
  const unsigned nholes = (unsigned)(std::lower_bound(h_all.begin(), h_all.end(), nnew,
                                                      [](unsigned a, unsigned long long b) { return a < b; }) -
                                     h_all.begin());
  if (nholes)
    mig_fill_kernel<<<(E + 255) / 256, 256, 0, c.stream>>>(all, E, nnew, nholes, s.pos, s.mom);
  c.count_launch(nholes ? 2 : 1);
  s.n = (size_t)nnew;
  CUDA_OK(cudaMemsetAsync(s.mig_count, 0, 2 * sizeof(unsigned), c.stream));
}

void migrate_append(Context& c, Species& s, const void* src, size_t count) {
  if (count == 0) return;
  if (s.n + count > s.cap) throw RunAbort("migration: species capacity exceeded by immigrants");
  // src = count x (pos, mom) pairs
  CUDA_OK(cudaMemcpy2DAsync(s.pos + s.n, 16, src, 32, 16, count, cudaMemcpyDeviceToDevice, c.stream));
  CUDA_OK(cudaMemcpy2DAsync(s.mom + s.n, 16, static_cast<const char*>(src) + 16, 32, 16, count,
                            cudaMemcpyDeviceToDevice, c.stream));
  s.n += count;
}

}  // namespace picb
