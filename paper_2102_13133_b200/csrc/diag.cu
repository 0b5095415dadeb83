// Diagnostics on the device: the quantities
// SimState::current_diagnostics / refresh_charge_diagnostics compute on the
// diagnostic cadence (proj/src/sim.cpp:236-266, 230-234).
//
// Reference path restated (all /root/reference/proj):
//   clear_rho                 src/fields.cpp:203-206
//   deposit_rho               src/particles.cpp:384-410
//   compute_div_errors        src/fields.cpp:253-274
//   field_energy              src/fields.cpp:276-299 (+ sum_squares, kernels/scalar.cpp:51-59)
//   max_abs_lane              src/fields.cpp:301-313
//   kinetic_energy_centered   src/particles.cpp:468-501
//   kinetic_energy            src/particles.cpp:460-466 (+ kinetic_sum, scalar.cpp:61-71)
//
// Parity: compute_div_errors and max_abs_lane are bit-exact (a stencil and an
// order-free max).  The energies have two modes (pic_diagnostics_order):
//   * fast (default): fp64 device sums of the reference's fp32 terms;
//   * reference order (deterministic decks): the reference's own fp32
//     summation — field energy as the serial sum over (lane, z, y) lines of
//     each line's 8 interleaved partials collapsed pairwise (sum_squares,
//     kernels/scalar.cpp:51-59, impl.hpp:24-28; the AVX2 lane sums the same
//     partials, avx2.cpp:192-205), kinetic energy as 8 interleaved partials
//     over the particles in their order, collapsed pairwise
//     (particles.cpp:468-501) — bit-identical to the reference.  The 8
//     partial chains are serial by definition: ~n/8 dependent adds.
// rho: float atomics (fast), or in reference-order mode the reference's
// serial order (every node's contributions sorted stably by node, added in
// particle order) — bit-identical.
// Per-particle / per-voxel terms keep the reference's fp32 expressions.
#include <algorithm>
#include <cstring>

#include "pic_device.cuh"
#include "pic_internal.hpp"

namespace picb {

namespace {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Block reduction of two doubles into out[0..1] with one fp64 atomic each.
__device__ __forceinline__ void block_add2(double a, double b, double* out) {
  __shared__ double sa[32], sb[32];
  a = warp_sum_d(a);
  b = warp_sum_d(b);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sa[w] = a;
    sb[w] = b;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    a = l < nw ? sa[l] : 0.0;
    b = l < nw ? sb[l] : 0.0;
    a = warp_sum_d(a);
    b = warp_sum_d(b);
    if (l == 0) {
      atomicAdd(out, a);
      atomicAdd(out + 1, b);
    }
  }
}

__device__ __forceinline__ void interior_of(const GridC& g, long long idx, int& ix, int& iy, int& iz) {
  const long long nxy = (long long)g.nx * g.ny;
  iz = (int)(idx / nxy);
  const int r = (int)(idx - (long long)iz * nxy);
  iy = r / g.nx;
  ix = r - iy * g.nx + 1;
  ++iy;
  ++iz;
}

// field_energy: per interior voxel e = ex^2+ey^2+ez^2 (each v*v in fp32 as
// sum_squares does), accumulated in fp64.
__global__ void __launch_bounds__(256)
field_energy_kernel(GridC g, const float* __restrict__ f, double* __restrict__ out) {
  const long long n = (long long)g.nx * g.ny * g.nz;
  const size_t V = (size_t)g.V;
  double se = 0.0, sb = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    interior_of(g, t, ix, iy, iz);
    const size_t v = (size_t)voxel_of(g, ix, iy, iz);
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const float e = f[(size_t)(F_EX + l) * V + v];
      const float b = f[(size_t)(F_BX + l) * V + v];
      se += (double)(e * e);
      sb += (double)(b * b);
    }
  }
  block_add2(se, sb, out);
}

// max_abs_lane over the interior: |x| >= 0 orders like its bit pattern.
__global__ void __launch_bounds__(256)
max_abs_kernel(GridC g, const float* __restrict__ lane, unsigned* __restrict__ out) {
  const long long n = (long long)g.nx * g.ny * g.nz;
  unsigned m = 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    interior_of(g, t, ix, iy, iz);
    const float a = fabsf(lane[voxel_of(g, ix, iy, iz)]);
    const unsigned u = __float_as_uint(a);
    m = (a > __uint_as_float(m)) ? u : m;  // NaN never replaces (fields.cpp:309 `v > m`)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// compute_div_errors (fields.cpp:253-274), same expression order.
__global__ void __launch_bounds__(256)
div_errors_kernel(GridC g, float* __restrict__ f, float rhx, float rhy, float rhz) {
  const long long n = (long long)g.nx * g.ny * g.nz;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int ix, iy, iz;
  interior_of(g, t, ix, iy, iz);
  const size_t V = (size_t)g.V;
  const size_t v = (size_t)voxel_of(g, ix, iy, iz);
  const size_t sx = 1, sy = (size_t)g.sy, sz = (size_t)g.sz;
  const float* ex = f + (size_t)F_EX * V;
  const float* ey = f + (size_t)F_EY * V;
  const float* ez = f + (size_t)F_EZ * V;
  const float* bx = f + (size_t)F_BX * V;
  const float* by = f + (size_t)F_BY * V;
  const float* bz = f + (size_t)F_BZ * V;
  const float dive = ((ex[v] - ex[v - sx]) * rhx + (ey[v] - ey[v - sy]) * rhy) + (ez[v] - ez[v - sz]) * rhz;
  f[(size_t)F_DIVE * V + v] = dive - f[(size_t)F_RHO * V + v];
  f[(size_t)F_DIVB * V + v] =
      ((bx[v + sx] - bx[v]) * rhx + (by[v + sy] - by[v]) * rhy) + (bz[v + sz] - bz[v]) * rhz;
}

// deposit_rho (particles.cpp:384-410): eight trilinear weights per particle
// into the rhof lane (float atomics, order not fixed: tolerance parity).
// A CTA takes 2048 consecutive records; each lane sums runs of equal voxels
// over 8 consecutive records of its own (staged through shared memory from
// coalesced loads), so a voxel-ordered store adds once per node per lane
// and run, with fire-and-forget reductions in L2.
// Measured at C1 (8.4 M records, ncu): 132 us for the previous form (a
// segmented shuffle scan of one record per lane, then shared-memory windows
// whose float atomics compile to a CAS loop: issue-bound), 98 us with the
// lane runs of 4 and scalar REDs, 108 us with red.v2 for the x-adjacent
// node pairs when 8-B aligned; refresh_charge at C1 (two species + div
// errors) 0.205 ms with runs of 4 per lane, 0.157 ms with 8, 0.39 with 2.
#ifndef PIC_RHO_LANE
#define PIC_RHO_LANE 8
#define PIC_RHO_ROUNDS 1
#endif
constexpr int kRhoLane = PIC_RHO_LANE;      // consecutive records per lane and round
constexpr int kRhoRounds = PIC_RHO_ROUNDS;  // rounds per CTA: 256 * 8 = 2048 records
__device__ __forceinline__ void rho_flush(const GridC& g, int key, const float* w, float* __restrict__ rho) {
  const unsigned rest = fast_div((unsigned)key, g.mag_pnx);
  const int ix = key - (int)rest * g.pnx;
  const unsigned izu = fast_div(rest, g.mag_pny);
  const int iy = (int)rest - (int)izu * g.pny, iz = (int)izu;
  const int xh = (ix + 1 > g.nx && !g.xopen) ? 1 : ix + 1;  // x-decomposed: ghost, halo-added
  const int yh = (iy + 1 > g.ny && !g.ywall) ? 1 : iy + 1;  // walled: the wall node plane
  const int zh = (iz + 1 > g.nz && !g.zwall) ? 1 : iz + 1;
  const int node[8] = {voxel_of(g, ix, iy, iz), voxel_of(g, xh, iy, iz), voxel_of(g, ix, yh, iz),
                       voxel_of(g, xh, yh, iz), voxel_of(g, ix, iy, zh), voxel_of(g, xh, iy, zh),
                       voxel_of(g, ix, yh, zh), voxel_of(g, xh, yh, zh)};
#pragma unroll
  for (int k = 0; k < 8; ++k) atomicAdd(rho + node[k], w[k]);
}

__global__ void __launch_bounds__(256)
deposit_rho_kernel(GridC g, const float4* __restrict__ pos, const float4* __restrict__ mom, long long n,
                   float q, float scale, float* __restrict__ rho) {
  constexpr int kPad = kRhoLane + 1;  // staging stride per lane (bank-conflict free)
  __shared__ float4 sp[8][32 * kPad];
  __shared__ float sw[8][32 * kPad];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long i0 = (long long)blockIdx.x * (256 * kRhoLane * kRhoRounds);
  int cur = -1;
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 0.f;
#pragma unroll
  for (int round = 0; round < kRhoRounds; ++round) {
    // the warp's 128 records of this round, coalesced, into lane-major staging
    const long long wb = i0 + ((long long)round * 8 + warp) * (32 * kRhoLane);
    if (round) __syncwarp();  // the previous round's staging read by every lane
#pragma unroll
    for (int r = 0; r < kRhoLane; ++r) {
      const int k = r * 32 + lane;
      const long long i = wb + k;
      float4 p = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
      float w = 0.f;
      if (i < n) {
        p = pos[i];
        w = mom[i].w;
      }
      const int at = (k / kRhoLane) * kPad + k % kRhoLane;
      sp[warp][at] = p;
      sw[warp][at] = w;
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < kRhoLane; ++t) {
      const float4 p = sp[warp][lane * kPad + t];
      const int key = __float_as_int(p.w);
      if (key != cur) {
        if (cur >= 0) rho_flush(g, cur, a, rho);
        cur = key;
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = 0.f;
      }
      if (key >= 0) {
        const float qw = (q * sw[warp][lane * kPad + t]) * scale;  // sp.q * w * scale (particles.cpp:393)
        const float wxl = 1 - p.x, wxh = 1 + p.x;
        const float wyl = 1 - p.y, wyh = 1 + p.y;
        const float wzl = 1 - p.z, wzh = 1 + p.z;
        a[0] += qw * (wxl * wyl * wzl);
        a[1] += qw * (wxh * wyl * wzl);
        a[2] += qw * (wxl * wyh * wzl);
        a[3] += qw * (wxh * wyh * wzl);
        a[4] += qw * (wxl * wyl * wzh);
        a[5] += qw * (wxh * wyl * wzh);
        a[6] += qw * (wxl * wyh * wzh);
        a[7] += qw * (wxh * wyh * wzh);
      }
    }
  }
  if (cur >= 0) rho_flush(g, cur, a, rho);
}

// kinetic_energy_centered (particles.cpp:468-501): momentum recentred by a
// half electric kick with the current interpolators, (w m)(gamma - 1) per
// particle in fp32, summed in fp64.  kCentered=false is kinetic_energy
// (kinetic_sum, scalar.cpp:61-71).
template <bool kCentered>
__global__ void __launch_bounds__(256)
kinetic_kernel(const float4* __restrict__ pos, const float4* __restrict__ mom, long long n,
               const float4* __restrict__ interp, float qdt_2m, float m, double* __restrict__ out) {
  // four particles per iteration, their loads (and gathers) issued together
  constexpr int kPer = 4;
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += kPer * stride) {
    float4 u[kPer], p[kPer];
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const long long i = i0 + r * stride;
      u[r] = i < n ? mom[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      if (kCentered) p[r] = i < n ? pos[i] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
    }
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      float cx = u[r].x, cy = u[r].y, cz = u[r].z;
      if (kCentered && __float_as_int(p[r].w) >= 0) {
        const float4* c = interp + (size_t)__float_as_int(p[r].w) * kInterpF4;
        const float4 c0 = __ldg(c), c1 = __ldg(c + 1), c2 = __ldg(c + 2);
        float ex, ey, ez;
        interp_eval_e(c0, c1, c2, p[r].x, p[r].y, p[r].z, ex, ey, ez);
        cx = cx + qdt_2m * ex;
        cy = cy + qdt_2m * ey;
        cz = cz + qdt_2m * ez;
      }
      const float gm = __fsqrt_rn(1.0f + ((cx * cx + cy * cy) + cz * cz));
      acc += (double)((u[r].w * m) * (gm - 1.0f));  // w = 0 past the end: adds 0
    }
  }
  block_add2(acc, 0.0, out);
}

// sum_squares of one x line (interior ix = 1..nx) per thread, for lanes
// lane0..lane0+2: the reference's 8 interleaved partials, collapsed pairwise.
__global__ void __launch_bounds__(128)
line_sum_squares_kernel(GridC g, const float* __restrict__ f, int lane0, float* __restrict__ out) {
  const long long lines = 3LL * g.ny * g.nz;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= lines) return;
  const int l = (int)(t / ((long long)g.ny * g.nz));
  const long long r = t - (long long)l * g.ny * g.nz;
  const int iz = 1 + (int)(r / g.ny), iy = 1 + (int)(r % g.ny);
  const float* x = f + (size_t)(lane0 + l) * (size_t)g.V + (size_t)voxel_of(g, 1, iy, iz);
  float p[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int k = 0; k < g.nx; ++k) {
    const float v = x[k];
    p[k & 7] = p[k & 7] + v * v;
  }
#pragma unroll
  for (int h = 4; h > 0; h >>= 1)
#pragma unroll
    for (int j = 0; j < h; ++j) p[j] = p[j] + p[j + h];
  out[t] = p[0];
}

// se / sb: the serial fp32 sums over the lines in (lane, z, y) order.
__global__ void serial_line_sum_kernel(const float* __restrict__ lines, long long n, float* __restrict__ out) {
  if (threadIdx.x >= 2) return;
  const float* x = lines + (size_t)threadIdx.x * (size_t)n;
  float s = 0.f;
  for (long long i = 0; i < n; ++i) s = s + x[i];
  out[threadIdx.x] = s;
}

// kinetic_energy_centered's per-particle terms, in particle order.
__global__ void __launch_bounds__(256)
kinetic_terms_kernel(const float4* __restrict__ pos, const float4* __restrict__ mom, long long n,
                     const float4* __restrict__ interp, float qdt_2m, float m, float* __restrict__ term) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 u = mom[i];
  const float4 p = pos[i];
  const float4* c = interp + (size_t)__float_as_int(p.w) * kInterpF4;
  const float4 c0 = __ldg(c), c1 = __ldg(c + 1), c2 = __ldg(c + 2);
  float ex, ey, ez;
  interp_eval_e(c0, c1, c2, p.x, p.y, p.z, ex, ey, ez);
  const float cx = u.x + qdt_2m * ex, cy = u.y + qdt_2m * ey, cz = u.z + qdt_2m * ez;
  const float gm = __fsqrt_rn(1.0f + ((cx * cx + cy * cy) + cz * cz));
  term[i] = (u.w * m) * (gm - 1.0f);
}

// p[i % 8] += term[i] in particle order (8 serial chains), collapsed pairwise.
__global__ void partials8_kernel(const float* __restrict__ term, long long n, float* __restrict__ out) {
  __shared__ float p[8];
  const int j = threadIdx.x;
  if (j < 8) {
    float s = 0.f;
    long long i = j;
    for (; i + 24 < n; i += 32) {  // four loads in flight, the adds in order
      const float a = term[i], b = term[i + 8], cc = term[i + 16], dd = term[i + 24];
      s = s + a;
      s = s + b;
      s = s + cc;
      s = s + dd;
    }
    for (; i < n; i += 8) s = s + term[i];
    p[j] = s;
  }
  __syncthreads();
  if (j == 0) {
    float q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = p[k];
#pragma unroll
    for (int h = 4; h > 0; h >>= 1)
#pragma unroll
      for (int k = 0; k < h; ++k) q[k] = q[k] + q[k + h];
    out[0] = q[0];
  }
}

// deposit_rho in the reference's order (particles.cpp:384-410): every
// particle's 8 node contributions, emitted in (particle, corner) order ...
__global__ void __launch_bounds__(256)
emit_rho_kernel(GridC g, const float4* __restrict__ pos, const float4* __restrict__ mom, long long i0,
                long long n, float q, float scale, unsigned* __restrict__ key, float* __restrict__ w) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const float4 p = pos[i0 + t];
  const float4 u = mom[i0 + t];
  const int v = __float_as_int(p.w);
  const unsigned rest = fast_div((unsigned)v, g.mag_pnx);
  const int ix = v - (int)rest * g.pnx;
  const unsigned izu = fast_div(rest, g.mag_pny);
  const int iy = (int)rest - (int)izu * g.pny, iz = (int)izu;
  const int xh = ix + 1 > g.nx ? 1 : ix + 1, yh = iy + 1 > g.ny ? 1 : iy + 1, zh = iz + 1 > g.nz ? 1 : iz + 1;
  const float qw = (q * u.w) * scale;
  const float wxl = 1 - p.x, wxh = 1 + p.x, wyl = 1 - p.y, wyh = 1 + p.y, wzl = 1 - p.z, wzh = 1 + p.z;
  unsigned* k = key + 8 * t;
  float* o = w + 8 * t;
  k[0] = (unsigned)voxel_of(g, ix, iy, iz);  o[0] = qw * (wxl * wyl * wzl);
  k[1] = (unsigned)voxel_of(g, xh, iy, iz);  o[1] = qw * (wxh * wyl * wzl);
  k[2] = (unsigned)voxel_of(g, ix, yh, iz);  o[2] = qw * (wxl * wyh * wzl);
  k[3] = (unsigned)voxel_of(g, xh, yh, iz);  o[3] = qw * (wxh * wyh * wzl);
  k[4] = (unsigned)voxel_of(g, ix, iy, zh);  o[4] = qw * (wxl * wyl * wzh);
  k[5] = (unsigned)voxel_of(g, xh, iy, zh);  o[5] = qw * (wxh * wyl * wzh);
  k[6] = (unsigned)voxel_of(g, ix, yh, zh);  o[6] = qw * (wxl * wyh * wzh);
  k[7] = (unsigned)voxel_of(g, xh, yh, zh);  o[7] = qw * (wxh * wyh * wzh);
}

// ... sorted stably by node, then added onto each node in that order.
__global__ void __launch_bounds__(256)
ordered_rho_kernel(const unsigned* __restrict__ start, const unsigned* __restrict__ idx,
                   const float* __restrict__ w, float* __restrict__ rho, long long V) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const unsigned b = start[v], e = start[v + 1];
  if (b == e) return;
  float r = rho[v];
  for (unsigned t = b; t < e; ++t) r = r + w[idx[t]];
  rho[v] = r;
}

unsigned grid_stride_blocks(const Context& c, long long n) {
  const long long want = (n + 255) / 256;
  const long long cap = (long long)c.num_sms * 8;
  return (unsigned)std::max<long long>(1, std::min(want, cap));
}

}  // namespace

void launch_clear_rho(Context& c) {
  CUDA_OK(cudaMemsetAsync(c.f + (size_t)F_RHO * c.gc.V, 0, (size_t)c.gc.V * sizeof(float), c.stream));
}

void launch_deposit_rho(Context& c, Species& s) {
  if (s.n == 0) return;
  const float scale = 0.125f / ((c.grid.hx * c.grid.hy) * c.grid.hz);
  if (c.reference_order_sums && !s.ordered) {
    // the reference's serial order, in chunks of particles (8 contributions
    // each; a chunk's node sums continue the previous chunk's)
    const long long V = c.gc.V;
    const long long chunk = 1LL << 26;
    for (long long i0 = 0; i0 < (long long)s.n; i0 += chunk) {
      const long long n = std::min<long long>(chunk, (long long)s.n - i0);
      unsigned* key = static_cast<unsigned*>(c.scratch_bytes(Context::kScrSegKey, (size_t)(8 * n) * 4));
      float* w = static_cast<float*>(c.scratch_bytes(Context::kScrSegW, (size_t)(8 * n) * 4));
      emit_rho_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(c.gc, s.pos, s.mom, i0, n, s.q, scale,
                                                                       key, w);
      c.count_launch();
      unsigned *skey = nullptr, *sval = nullptr;
      radix_sort_pairs(c, key, nullptr, (size_t)(8 * n), key_bits_for(V), &skey, &sval);
      unsigned* start = static_cast<unsigned*>(c.scratch_bytes(Context::kScrStart, (size_t)(V + 1) * 4));
      key_run_starts(c, skey, (size_t)(8 * n), (size_t)V, start);
      ordered_rho_kernel<<<(unsigned)((V + 255) / 256), 256, 0, c.stream>>>(start, sval, w,
                                                                          c.f + (size_t)F_RHO * c.gc.V, V);
      c.count_launch();
    }
    return;
  }
  constexpr long long kPerCta = 256 * kRhoLane * kRhoRounds;
  deposit_rho_kernel<<<(unsigned)((s.n + kPerCta - 1) / kPerCta), 256, 0, c.stream>>>(
      c.gc, s.pos, s.mom, (long long)s.n, s.q, scale, c.f + (size_t)F_RHO * c.gc.V);
  c.count_launch();
}

void launch_compute_div_errors(Context& c) {
  const long long n = (long long)c.gc.nx * c.gc.ny * c.gc.nz;
  div_errors_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(c.gc, c.f, 1.0f / c.grid.hx,
                                                                      1.0f / c.grid.hy, 1.0f / c.grid.hz);
  c.count_launch();
}

double* diag_slots(Context& c) {
  return reinterpret_cast<double*>(c.scratch_bytes(Context::kScrDiag, 64 * sizeof(double)));
}

void field_energy(Context& c, float e_b[2]) {
  if (c.reference_order_sums) {
    // field_energy (fields.cpp:276-299) in the reference's summation order
    const long long lines = 3LL * c.gc.ny * c.gc.nz;
    float* ls = static_cast<float*>(c.scratch_bytes(Context::kScrDiagLines, (size_t)(2 * lines + 2) * sizeof(float)));
    line_sum_squares_kernel<<<(unsigned)((lines + 127) / 128), 128, 0, c.stream>>>(c.gc, c.f, F_EX, ls);
    line_sum_squares_kernel<<<(unsigned)((lines + 127) / 128), 128, 0, c.stream>>>(c.gc, c.f, F_BX, ls + lines);
    serial_line_sum_kernel<<<1, 32, 0, c.stream>>>(ls, lines, ls + 2 * lines);
    c.count_launch(3);
    float h[2];
    CUDA_OK(cudaMemcpyAsync(h, ls + 2 * lines, sizeof h, cudaMemcpyDeviceToHost, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
    const float hv = 0.5f * ((c.grid.hx * c.grid.hy) * c.grid.hz);
    e_b[0] = hv * h[0];
    e_b[1] = hv * h[1];
    return;
  }
  double* d = diag_slots(c);
  CUDA_OK(cudaMemsetAsync(d, 0, 2 * sizeof(double), c.stream));
  const long long n = (long long)c.gc.nx * c.gc.ny * c.gc.nz;
  field_energy_kernel<<<grid_stride_blocks(c, n), 256, 0, c.stream>>>(c.gc, c.f, d);
  c.count_launch();
  double h[2];
  CUDA_OK(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
  const double hv = 0.5 * (double)((c.grid.hx * c.grid.hy) * c.grid.hz);
  e_b[0] = (float)(hv * h[0]);
  e_b[1] = (float)(hv * h[1]);
}

float max_abs_lane(Context& c, int lane) {
  unsigned* d = reinterpret_cast<unsigned*>(diag_slots(c) + 8);
  CUDA_OK(cudaMemsetAsync(d, 0, sizeof(unsigned), c.stream));
  const long long n = (long long)c.gc.nx * c.gc.ny * c.gc.nz;
  max_abs_kernel<<<grid_stride_blocks(c, n), 256, 0, c.stream>>>(c.gc, c.f + (size_t)lane * c.gc.V, d);
  c.count_launch();
  unsigned h = 0;
  CUDA_OK(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
  float r;
  std::memcpy(&r, &h, sizeof r);
  return r;
}

float kinetic_energy(Context& c, Species& s, bool centered) {
  if (s.n == 0) return 0.0f;
  if (c.reference_order_sums && centered && !s.ordered) {
    // kinetic_energy_centered (particles.cpp:468-501) in the reference's order
    float* term = static_cast<float*>(c.scratch_bytes(Context::kScrDiagLines, (s.n + 8) * sizeof(float)));
    const float qdt_2m = (s.q * c.grid.dt) / (2.0f * s.m);
    kinetic_terms_kernel<<<(unsigned)((s.n + 255) / 256), 256, 0, c.stream>>>(s.pos, s.mom, (long long)s.n,
                                                                             c.interp, qdt_2m, s.m, term);
    partials8_kernel<<<1, 32, 0, c.stream>>>(term, (long long)s.n, term + s.n);
    c.count_launch(2);
    float h = 0.f;
    CUDA_OK(cudaMemcpyAsync(&h, term + s.n, sizeof h, cudaMemcpyDeviceToHost, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
    return h;
  }
  double* d = diag_slots(c) + 16;
  CUDA_OK(cudaMemsetAsync(d, 0, 2 * sizeof(double), c.stream));
  const float qdt_2m = (s.q * c.grid.dt) / (2.0f * s.m);
  const unsigned b = grid_stride_blocks(c, (long long)s.n);
  if (centered)
    kinetic_kernel<true><<<b, 256, 0, c.stream>>>(s.pos, s.mom, (long long)s.n, c.interp, qdt_2m, s.m, d);
  else
    kinetic_kernel<false><<<b, 256, 0, c.stream>>>(s.pos, s.mom, (long long)s.n, c.interp, qdt_2m, s.m, d);
  c.count_launch();
  double h = 0;
  CUDA_OK(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
  return (float)h;
}

// SimState::current_diagnostics' reductions (sim.cpp:236-266) with one
// readback: field energy, centred kinetic energy per species (with fresh
// interpolators) and the two max div errors launched back to back into
// device slots, one copy, one synchronisation (the synchronous functions
// above cost a round trip each: 0.58 ms a row at C1).  The fp32 results are
// those of field_energy / kinetic_energy / max_abs_lane in fast mode; the
// reference-order sums (deterministic decks) take those functions instead.
void diagnostics_batch(Context& c, float e_b[2], float* kinetic, float mdiv[2]) {
  const size_t ns = c.species.size();
  if (c.reference_order_sums || ns > 24) {
    field_energy(c, e_b);
    launch_load_interpolators(c);
    for (size_t i = 0; i < ns; ++i) kinetic[i] = kinetic_energy(c, c.species[i], true);
    mdiv[0] = max_abs_lane(c, F_DIVE);
    mdiv[1] = max_abs_lane(c, F_DIVB);
    return;
  }
  // slots: [0, 2) field energy, [2, 4) max |div e|, |div b| (as u32), [8, 8 + ns) kinetic
  double* d = reinterpret_cast<double*>(c.scratch_bytes(Context::kScrDiag, 64 * sizeof(double)));
  CUDA_OK(cudaMemsetAsync(d, 0, (8 + ns) * sizeof(double), c.stream));
  const long long n = (long long)c.gc.nx * c.gc.ny * c.gc.nz;
  field_energy_kernel<<<grid_stride_blocks(c, n), 256, 0, c.stream>>>(c.gc, c.f, d);
  unsigned* mx = reinterpret_cast<unsigned*>(d + 2);
  max_abs_kernel<<<grid_stride_blocks(c, n), 256, 0, c.stream>>>(c.gc, c.f + (size_t)F_DIVE * c.gc.V, mx);
  max_abs_kernel<<<grid_stride_blocks(c, n), 256, 0, c.stream>>>(c.gc, c.f + (size_t)F_DIVB * c.gc.V,
                                                               reinterpret_cast<unsigned*>(d + 3));
  launch_load_interpolators(c);  // fresh coefficients (sim.cpp:245-246)
  c.count_launch(3);
  for (size_t i = 0; i < ns; ++i) {
    Species& s = c.species[i];
    if (s.n == 0) continue;
    const float qdt_2m = (s.q * c.grid.dt) / (2.0f * s.m);
    kinetic_kernel<true><<<grid_stride_blocks(c, (long long)s.n), 256, 0, c.stream>>>(
        s.pos, s.mom, (long long)s.n, c.interp, qdt_2m, s.m, d + 8 + i);
    c.count_launch();
  }
  double h[8 + 24];
  CUDA_OK(cudaMemcpyAsync(h, d, (8 + ns) * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
  const double hv = 0.5 * (double)((c.grid.hx * c.grid.hy) * c.grid.hz);
  e_b[0] = (float)(hv * h[0]);
  e_b[1] = (float)(hv * h[1]);
  unsigned u[2];
  std::memcpy(u, &h[2], sizeof(unsigned));
  std::memcpy(u + 1, &h[3], sizeof(unsigned));
  std::memcpy(&mdiv[0], &u[0], sizeof(float));
  std::memcpy(&mdiv[1], &u[1], sizeof(float));
  for (size_t i = 0; i < ns; ++i) kinetic[i] = c.species[i].n ? (float)h[8 + i] : 0.0f;
}

}  // namespace picb
