/* TEST INFRASTRUCTURE ONLY — the CPU checker for the CUDA path.
 *
 * Plain-C (C11, fp32, no FP contraction) restatement of the reference's
 * particle-in-cell hot path (minipic, /root/reference/proj).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * oracle/liborc.so; the product path (paper_2102_13133_b200/) never does.
 *
 * Parity pinning: every function is checked bit-for-bit against the
 * unmodified reference compiled from its sources (oracle/_ref, see
 * oracle/Makefile) by tests/test_oracle_vs_ref.py, and against the committed
 * golden vectors in tests/golden/ (made by tests/golden/make_golden.py from
 * the reference itself).
 *
 * Array conventions (all field-major, i.e. lane * records + record, the
 * reference's default Layout::field_major, proj/include/minipic/layout.hpp:18):
 *   fields16 : 16 lanes x padded voxels   (lanes.hpp:23-43)
 *   interp18 : 18 lanes x padded voxels   (lanes.hpp:48-69)
 *   lanes7   :  7 lanes x particles       (lanes.hpp:8-19) + int32 ids
 *   acc12    : padded voxels x 12 (record-major, the ScatterBuffer's dense
 *              form, proj/src/layout.cpp:181-197)
 */
#ifndef PIC_ORACLE_H
#define PIC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_grid {
  int nx, ny, nz;
  float hx, hy, hz, dt;
} orc_grid;

/* status codes: 0 ok, 1 usage_error, 2 run_abort */
const char* orc_last_error(void);

float orc_cfl_limit(const orc_grid* g);
void orc_load_interpolators(const orc_grid* g, const float* fields16, float* interp18);
int orc_advance_particles(const orc_grid* g, float q, float m, long n, float* lanes7,
                          int32_t* ids, const float* interp18, float* acc12,
                          int exact_gyration);
void orc_ghost_fold(const orc_grid* g, float* acc12);
void orc_clear_currents(const orc_grid* g, float* fields16);
void orc_unload(const orc_grid* g, const float* acc12, float* fields16);
void orc_advance_b(const orc_grid* g, float* fields16, float frac);
void orc_advance_e(const orc_grid* g, float* fields16);
void orc_ghost_sync(const orc_grid* g, float* fields16);
int orc_sort(long n, float* lanes7, int32_t* ids, int interleaved);

/* One SimState::step (proj/src/sim.cpp:143-183) over nspecies species that
 * share one accumulator; acc12 / interp18 are caller scratch. */
int orc_step(const orc_grid* g, int nspecies, const float* q, const float* m,
             const long* n, float** lanes7, int32_t** ids, float* fields16,
             float* interp18, float* acc12, int exact_gyration);

/* Particle load of SimState::initialize (proj/src/sim.cpp:74-112) for one
 * species: mt19937_64 + Box-Muller (proj/include/minipic/rng.hpp:17-51). */
void orc_load_species(const orc_grid* g, uint64_t seed, int species_index, int ppc,
                      float u_th, const float drift[3], float perturb_ux,
                      int perturb_kmode, float* lanes7, int32_t* ids);

/* Diagnostics. */
void orc_deposit_rho(const orc_grid* g, float q, long n, const float* lanes7,
                     const int32_t* ids, float* fields16);
void orc_compute_div_errors(const orc_grid* g, float* fields16);
void orc_field_energy(const orc_grid* g, const float* fields16, float* e_b);
float orc_kinetic_energy_centered(const orc_grid* g, float q, float m, long n,
                                  const float* lanes7, const int32_t* ids,
                                  const float* interp18);
float orc_max_abs_lane(const orc_grid* g, const float* fields16, int lane);

#ifdef __cplusplus
}
#endif
#endif
