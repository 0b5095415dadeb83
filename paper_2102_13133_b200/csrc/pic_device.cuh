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
};

// GridDescriptor (proj/include/minipic/grid.hpp:15-38) plus derived strides.
struct GridC {
  int nx, ny, nz;
  int pnx, pny, pnz;
  int sy, sz;          // +y / +z padded strides (stride_x == 1)
  long long V;         // padded voxels
  float hx, hy, hz, dt;
};

// Interpolator record: 18 coefficients padded to 5 float4 (80 B), in the
// reference lane order (lanes.hpp:48-69):
//   [0] ex dexdy dexdz d2exdydz  [1] ey deydz deydx d2eydzdx
//   [2] ez dezdx dezdy d2ezdxdy  [3] cbx dcbxdx cby dcbydy  [4] cbz dcbzdz 0 0
constexpr int kInterpF4 = 5;
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
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c,
                                           float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(addr), "f"(a),
               "f"(b), "f"(c), "f"(d)
               : "memory");
}

}  // namespace picb
