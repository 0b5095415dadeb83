// Device-side vocabulary shared by the sm_100a kernels.
//
// All arithmetic on the parity path is IEEE fp32 with no contraction: the
// library is compiled with --fmad=false, -prec-div=true, -prec-sqrt=true and
// without FTZ, and the few places that matter use the explicit __f*_rn
// intrinsics so the association order of the reference
// (proj/include/minipic/kernels/push_math.hpp:22-82) is kept bit for bit.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace picb {

constexpr unsigned kFull = 0xffffffffu;

// Device error latch bits (raised as run_abort at quiescence points).
enum ErrBits : int {
  kErrCfl = 1,       // |d| >= 2 on some axis (proj/src/particles.cpp:190-194)
  kErrMover = 2,     // mover did not terminate in 8 passes (:240)
  kErrWrap = 4,      // final voxel beyond one cell (proj/src/grid.cpp:42-43)
  kErrVoxel = 8,     // voxel id outside the padded lattice (grid.cpp:33-34)
  kErrMigCap = 16,   // emigrant list overflow (domain decomposition)
};

// GridDescriptor (proj/include/minipic/grid.hpp:15-38) plus derived strides.
struct GridC {
  int nx, ny, nz;
  int pnx, pny, pnz;
  int sy, sz;          // +y / +z padded strides (stride_x == 1)
  long long V;         // padded voxels
  float hx, hy, hz, dt;
  // exact division by pnx / pny: floor(v / d) == __umul64hi(v, m) with
  // m = ceil(2^64 / d), valid for 0 <= v < 2^31 (host computes m).
  unsigned long long mag_pnx, mag_pny;
  // Domain decomposition in x: with xopen the x faces are not
  // periodic — particles leaving through them become emigrants, the x ghost
  // planes are filled / folded by neighbour exchange instead of wrap-around.
  // x_low_wraps: this slab's low face is the global periodic boundary
  // (rank 0), which fixes the summation order of the wrapped unload edge.
  int xopen, x_low_wraps;
  // Non-periodic walls (pic_set_boundary), per face 2 axis + side (x low,
  // x high, y low, ...): particle bc (PIC_PBC_*; on an x face 0 = exchange
  // with a neighbour when decomposed) and field bc (PIC_FBC_*).  An x wall
  // sets xopen; ywall / zwall: that axis has walls (both faces).
  int wall_p[6], wall_f[6];
  int ywall, zwall;
};

__device__ __forceinline__ unsigned fast_div(unsigned v, unsigned long long m) {
  return (unsigned)__umul64hi((unsigned long long)v, m);
}

// Interpolator record: the 18 coefficients of the reference's lanes
// (lanes.hpp:48-69: ex dexdy dexdz d2exdydz, ey deydz deydx d2eydzdx,
// ez dezdx dezdy d2ezdxdy, cbx dcbxdx, cby dcbydy, cbz dcbzdz) padded to 5
// float4 (80 B), arranged so the push evaluates E_x, E_y and B_x, B_y as
// register pairs (packed FP32, push.cu):
//   [0] ex ey dexdy deydz          [1] dexdz deydx d2exdydz d2eydzdx
//   [2] ez dezdx dezdy d2ezdxdy    [3] cbx cby dcbxdx dcbydy   [4] cbz dcbzdz 0 0
constexpr int kInterpF4 = 5;
// float slot of the record holding reference lane l (0..17)
__host__ __device__ constexpr int interp_slot(int l) {
  return l < 4 ? (l == 0 ? 0 : l == 1 ? 2 : l == 2 ? 4 : 6)
       : l < 8 ? (l == 4 ? 1 : l == 5 ? 3 : l == 6 ? 5 : 7)
       : l < 12 ? l
       : l < 16 ? (l == 12 ? 12 : l == 13 ? 14 : l == 14 ? 13 : 15)
       : l;
}
// E at offsets (x, y, z) in the reference's association order
// (eval_eb_lanes, push_math.hpp:22-39)
__device__ __forceinline__ void interp_eval_e(const float4 F0, const float4 F1, const float4 F2, float x, float y,
                                              float z, float& ex, float& ey, float& ez) {
  ex = ((F0.x + y * F0.z) + z * F1.x) + (y * z) * F1.z;
  ey = ((F0.y + z * F0.w) + x * F1.y) + (z * x) * F1.w;
  ez = ((F2.x + x * F2.y) + y * F2.z) + (x * y) * F2.w;
}
// Accumulator record: 12 lanes (accum_var, lanes.hpp:72-91) = 3 float4.
constexpr int kAccF4 = 3;

// Field lanes (field_var, lanes.hpp:23-43), stored lane-major on device.
enum FieldLane : int {
  F_EX = 0, F_EY, F_EZ, F_DIVE, F_BX, F_BY, F_BZ, F_DIVB,
  F_JX, F_JY, F_JZ, F_RHO, F_TCAX, F_TCAY, F_TCAZ, F_RHOB, F_COUNT
};

__device__ __forceinline__ int voxel_of(const GridC& g, int ix, int iy, int iz) {
  return ix + g.pnx * (iy + g.pny * iz);  // grid.hpp:53-56
}

// Streaming 128-bit loads/stores for the particle records (each record is
// touched exactly once per kernel).
// Read-only gather that bypasses L1 (keeps L1 for the interpolator records).
__device__ __forceinline__ float4 ld_na(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
// Stores / loads that do not allocate in L1 (the ordered push's scattered
// output must not evict the interpolator records the gathers reuse).
__device__ __forceinline__ void st_na(float4* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_na_u32(unsigned* p, unsigned v) {
  asm volatile("st.global.L1::no_allocate.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_na_u32(const unsigned* p) {
  unsigned r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c,
                                           float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(addr), "f"(a),
               "f"(b), "f"(c), "f"(d)
               : "memory");
}

// ---- TMA bulk copies + mbarriers (sm_90+; the sm_100a TMA engine) ----------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// A converged global load ahead of a divergent loop whose only earlier
// global traffic is TMA: it makes ptxas keep the global memory descriptor
// in a uniform register instead of re-materialising it (R2UR) before every
// load and reduction of the loop.  Reads one L2-hot word; the OR of 0 never
// changes the flag.
__device__ __forceinline__ void pin_global_descriptor(const float4* __restrict__ p, int* __restrict__ flag) {
  const float4 w = __ldg(p);
  if (w.x == 1.2345e-38f && w.y == 3.25e-38f) atomicOr(flag, 0);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, unsigned bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// global -> L2 bulk prefetch (no completion; bytes % 16 == 0)
__device__ __forceinline__ void bulk_prefetch_l2(const void* gmem_src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem_src), "r"(bytes) : "memory");
}

// shared -> global bulk copy (bulk-group completion; bytes % 16 == 0)
__device__ __forceinline__ void tma_store_1d(void* gmem_dst, const void* smem_src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// waits until the smem sources of every committed bulk store have been read
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// orders this thread's generic-proxy smem writes before later async-proxy
// (TMA) reads of the same smem
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace picb
