/*
 * pic_b200.h — C-ABI drop-in boundary for the particle-in-cell hot path of
 * arXiv 2102.13133 (VPIC 2.0; reference implementation "minipic",
 * /root/reference/proj), re-implemented as hand-written sm_100a CUDA.
 *
 * Plain pointers, sizes and POD structs only; no C++ or torch types cross
 * this boundary.  Every entry point returns a pic_status; the message of the
 * most recent failure on the calling thread is pic_last_error().
 *
 * Array conventions match the reference's default storage
 * (Layout::field_major, proj/include/minipic/layout.hpp:18-30), so a host
 * that holds minipic buffers can hand their data() pointers straight in:
 *   fields16 : 16 lanes x padded voxels, lane-major   (lanes.hpp:23-43)
 *   interp18 : 18 lanes x padded voxels, lane-major   (lanes.hpp:48-69)
 *   lanes7   :  7 lanes x n particles, lane-major     (lanes.hpp:8-19)
 *   ids      :  n int32 voxel ids                     (types.hpp:20)
 *   acc12    : padded voxels x 12 (record-major; the ScatterBuffer's dense
 *              reduce() form, proj/src/layout.cpp:181-197)
 * Device-side the data live in B200-native layouts; the
 * upload / download calls convert.
 *
 * Error classes mirror proj/include/minipic/types.hpp:26-36 and
 * proj/include/minipic/sim.hpp:66-69.  Device-detected failures (CFL
 * violation, mover non-termination) are latched in a device flag and raised
 * as PIC_RUN_ABORT at the next quiescence point (pic_synchronize, any
 * download, pic_sim_step).
 */
#ifndef PIC_B200_H
#define PIC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PIC_B200_ABI_VERSION 1

typedef enum pic_status {
  PIC_OK = 0,
  PIC_USAGE_ERROR = 1,      /* minipic::usage_error      (types.hpp:27-30)  */
  PIC_RUN_ABORT = 2,        /* minipic::run_abort        (types.hpp:33-36)  */
  PIC_DECK_PARSE_ERROR = 3, /* minipic::deck_parse_error (sim.hpp:66-69)    */
  PIC_CUDA_ERROR = 4,       /* CUDA runtime failure                          */
  PIC_INTERNAL_ERROR = 5
} pic_status;

/* GridDescriptor (proj/include/minipic/grid.hpp:15-38), fp32. */
typedef struct pic_grid {
  int nx, ny, nz;
  float hx, hy, hz, dt;
} pic_grid;

/* advance_p flags (proj/src/particles.cpp:255-262 exact_gyration / stage). */
#define PIC_EXACT_GYRATION 0x1u
#define PIC_DETERMINISTIC 0x2u /* DepositStage + replay_deposits order */

/* sort orders (proj/include/minipic/particles.hpp:35) */
#define PIC_SORT_BLOCKED 0
#define PIC_SORT_INTERLEAVED 1

typedef struct pic_context pic_context;

int pic_version(void);
const char* pic_last_error(void);

/* ---- lifecycle ------------------------------------------------------------
 * Replaces the device-side state SimState builds in its constructor
 * (proj/src/sim.cpp:49-72): FieldArray, InterpolatorArray, ScatterBuffer.
 * validate_grid (proj/src/grid.cpp:13-20) is applied. */
int pic_context_create(int device, const pic_grid* grid, pic_context** out);
int pic_context_destroy(pic_context* ctx);
int pic_context_grid(pic_context* ctx, pic_grid* out);
/* Quiescence point: waits for the context stream and raises latched device
 * errors (proj/src/particles.cpp:190-194,240; proj/src/grid.cpp:42-43). */
int pic_synchronize(pic_context* ctx);
/* Pins (cudaHostRegister) / unpins a host range used for uploads/downloads. */
int pic_host_register(void* ptr, size_t bytes);
int pic_host_unregister(void* ptr);

/* ---- species: Species / ParticleStore (proj/include/minipic/particles.hpp:18-45)
 * capacity >= the largest count ever uploaded. */
int pic_species_create(pic_context* ctx, const char* name, float q, float m,
                       size_t capacity, int* out_species);
int pic_species_count(pic_context* ctx, int species, size_t* out_n);
/* copy_between host -> device mirror (proj/src/layout.cpp:99-118). */
int pic_species_upload(pic_context* ctx, int species, size_t n,
                       const float* lanes7, const int32_t* ids);
int pic_species_download(pic_context* ctx, int species, float* lanes7,
                         int32_t* ids);
/* Native-record upload/download: two float4 streams per particle,
 * pos = (dx, dy, dz, bits(id)) and mom = (ux, uy, uz, w) — the 32-byte
 * device record, no layout conversion.  The pointers may be host or device
 * memory (unified addressing: device-to-device copies stay on the GPU). */
int pic_species_upload_records(pic_context* ctx, int species, size_t n,
                               const void* pos16, const void* mom16);
int pic_species_download_records(pic_context* ctx, int species, void* pos16,
                                 void* mom16);
/* Device-side synthetic load (counter-based RNG, NOT the reference's
 * mt19937_64 stream): uniform offsets, drift + u_th * N(0,1) momenta, w = 1,
 * ppc particles per interior voxel in voxel order (proj/src/sim.cpp:84-111
 * shape).  For large benchmark decks; parity tests upload host-generated
 * reference streams instead. */
int pic_species_load_synthetic(pic_context* ctx, int species, int ppc,
                               float u_th, const float drift[3],
                               uint64_t seed);

/* Double Harris current sheet (BASELINE configs[2]; built through the API,
 * as SURVEY §8d C3 notes the reference cannot express it as deck text): the
 * synthetic load with particle weights w(z) = background + amplitude *
 * (sech^2((z - z1)/L) + sech^2((z - z2)/L)), z = (iz - 1 + (oz + 1)/2) hz,
 * and, with flip_drift, the drift reversed for particles nearer z2 (the two
 * sheets carry opposite currents).  Fields (B_x = B0 tanh profile) are
 * uploaded by the caller (paper_2102_13133_b200/decks.py). */
typedef struct pic_sheet {
  float z1, z2, half_width;
  float background, amplitude;
  int flip_drift;
} pic_sheet;
int pic_species_load_harris(pic_context* ctx, int species, int ppc,
                            float u_th, const float drift[3], uint64_t seed,
                            const pic_sheet* sheet);

/* ---- fields: FieldArray (proj/include/minipic/fields.hpp:21-38) --------- */
int pic_fields_upload(pic_context* ctx, const float* fields16);
int pic_fields_download(pic_context* ctx, float* fields16);
int pic_interpolators_download(pic_context* ctx, float* interp18);
int pic_interpolators_upload(pic_context* ctx, const float* interp18);
int pic_accumulator_download(pic_context* ctx, float* acc12);
int pic_accumulator_upload(pic_context* ctx, const float* acc12);

/* ---- the hot path ---------------------------------------------------------*/
/* ScatterBuffer::clear (proj/src/layout.cpp:205-207). */
int pic_clear_accumulator(pic_context* ctx);
/* clear_currents (proj/src/fields.cpp:195-201). */
int pic_clear_currents(pic_context* ctx);
/* load_interpolators (proj/src/particles.cpp:42-111). */
int pic_load_interpolators(pic_context* ctx);
/* advance_particles (+ replay_deposits with PIC_DETERMINISTIC)
 * (proj/src/particles.cpp:255-382): interpolator gather, Boris kick, face-
 * splitting mover, charge-conserving deposit into the accumulator, periodic
 * wrap of the final voxel. */
int pic_advance_p(pic_context* ctx, int species, unsigned flags);
/* ghost_fold_currents (proj/src/grid.cpp:78-99). */
int pic_ghost_fold_currents(pic_context* ctx);
/* unload_currents (proj/src/fields.cpp:208-251), jf += f_a * lane. */
int pic_unload_currents(pic_context* ctx);
/* advance_b (proj/src/fields.cpp:113-151) and advance_e (:153-193). */
int pic_advance_b(pic_context* ctx, float frac);
int pic_advance_e(pic_context* ctx);
/* unload_currents fused with advance_e (identical results to calling
 * pic_unload_currents then pic_advance_e). */
int pic_unload_advance_e(pic_context* ctx);
/* ghost_sync_fields (proj/src/fields.cpp:35-58). */
int pic_ghost_sync_fields(pic_context* ctx);
/* sort_particles (proj/src/particles.cpp:412-458). */
int pic_sort_particles(pic_context* ctx, int species, int order);
/* SimState::step (proj/src/sim.cpp:143-183) over every species of the
 * context in creation order. */
int pic_step(pic_context* ctx, unsigned flags);
/* NOT IN REFERENCE (executor preparation): pic_step replays one CUDA graph
 * per step configuration (buffer pair, reorder cadence, owed relabel).
 * This captures, without running anything, the graphs of the next `steps`
 * fast steps, assuming a blocked pic_sort_particles of every species after
 * each step whose running count (steps_taken + k) is a multiple of
 * sort_interval (0: no sorts) — the run loop's cadence
 * (proj/src/sim.cpp:217-222) — so those steps replay from the first.
 * Species state is left as it was.  A no-op (captured = 0) unless every
 * species is already in continuous voxel order (after one fast step). */
int pic_prepare_step_graphs(pic_context* ctx, unsigned flags, int steps, int sort_interval,
                            long long steps_taken, int* captured);
/* The same step with host-resident species (the reference's host
 * advance_particles contract): uploads every species from lanes7[s]/ids[s],
 * steps, downloads back into the same buffers (the weight lane, which the
 * step never modifies, is not copied back).  Species stream through the
 * device in chunks with H2D, compute and D2H overlapped; pin the buffers
 * (pic_host_register) for the copies to overlap. */
int pic_step_host(pic_context* ctx, unsigned flags, float* const* lanes7,
                  int32_t* const* ids);

/* ---- domain decomposition in x -------------------------------
 * A slab of a global periodic box decomposed along x.  With x_open set the
 * context's x faces stop being periodic (the single-domain wrap of
 * particles.cpp:348-350 / grid.cpp:32-52, the x pass of ghost_fold_currents,
 * grid.cpp:78-86, and the x pass of ghost_sync_fields, fields.cpp:35-44);
 * the host exchanges x planes and migrating particles with its neighbours
 * (NCCL through torch.distributed in paper_2102_13133_b200/domain.py) using
 * the pack / unpack calls below.  low_wraps: this slab's low x face is the
 * global periodic boundary (fixes the reference's unload sum order there).
 * Slabs must have equal nx.  pic_step / pic_step_host refuse an x-open
 * context: the host sequences the step around the exchanges. */
int pic_set_x_open(pic_context* ctx, int x_open, int low_wraps);

/* ---- non-periodic x boundaries (NOT IN REFERENCE: the
 * reference is periodic only, so these are designed fresh and checked by
 * self-consistency tests, tests/test_gpu_boundaries.py) ------------------
 * side 0 = low x face (x = 0), 1 = high x face (x = nx hx).  A wall side
 * replaces the periodic wrap / fold / ghost copy on that face:
 *   particles  PIC_PBC_ABSORB   leave the domain: removed after the push
 *                               (store compacted in index order), the part
 *                               of their last segment beyond the wall is
 *                               not deposited;
 *              PIC_PBC_REFLECT  specular: mirrored back into the boundary
 *                               cell (x offset -> -x offset, u_x -> -u_x),
 *                               the current beyond the wall folded back as
 *                               its mirror image (charge-conserving);
 *   fields     PIC_FBC_PEC      conductor: tangential E = 0 on the wall;
 *              PIC_FBC_MUR      first-order Mur absorbing condition on the
 *                               tangential E at the wall (normal incidence).
 * pic_step needs both sides periodic or both walls; on an x-decomposed
 * slab (pic_set_x_open) a wall side is the global boundary and the host
 * sequences the step (pic_wall_stage).  The default push (and variants
 * 42-52) and the deterministic path. */
#define PIC_PBC_PERIODIC 0
#define PIC_PBC_ABSORB 1
#define PIC_PBC_REFLECT 2
#define PIC_FBC_PERIODIC 0
#define PIC_FBC_PEC 1
#define PIC_FBC_MUR 2
int pic_set_x_boundary(pic_context* ctx, int side, int particle_bc, int field_bc);
/* Any face: 0 = x low, 1 = x high, 2 = y low, 3 = y high, 4 = z low,
 * 5 = z high (same conditions; the wall plane of a y / z face is the y / z
 * node plane, tangential E = (E_z, E_x) / (E_x, E_y)).  y / z walls are
 * single-domain only (not on an x-decomposed slab); pic_absorbed_counts
 * then counts the low / high faces of every axis together. */
int pic_set_boundary(pic_context* ctx, int face, int particle_bc, int field_bc);
/* particles absorbed through the low / high x wall since the last call
 * (synchronises) */
int pic_absorbed_counts(pic_context* ctx, uint64_t out[2], int reset);
/* The wall / laser / emitter pieces of the step for hosts that sequence it
 * themselves (the decomposed driver: on an x-open slab a wall side is the
 * global boundary, the other side keeps exchanging).  pic_step runs them at:
 *   FOLD      after the pushes, before the y/z current folds (accumulator x
 *             ghost planes of wall sides: mirror fold / drop)
 *   AFTER_B   after each advance_b(frac) (B_x on the high wall plane)
 *   BEFORE_E  before the E update (Mur's saved planes)
 *   AFTER_E   after the E update (laser source, wall E; advances the
 *             laser / emitter clock by one step)
 *   EMIT      after the pushes (emitter hooks) */
#define PIC_STAGE_FOLD 0
#define PIC_STAGE_AFTER_B 1
#define PIC_STAGE_BEFORE_E 2
#define PIC_STAGE_AFTER_E 3
#define PIC_STAGE_EMIT 4
int pic_wall_stage(pic_context* ctx, int stage, float frac);

/* Laser: a soft source on the node plane x = (ix - 1) hx — after every E
 * update E_pol += dt (2 e0 / hx) s(t) g(y, z) on that plane (a current sheet
 * radiating amplitude ~e0 each way), s(t) = sin(omega t) ramped in over
 * ramp_steps steps (sin^2), g = exp(-((y - y0)^2 + (z - z0)^2) / waist^2)
 * (waist <= 0: plane wave).  pol 1 = E_y, 2 = E_z.  e0 = 0 removes it. */
typedef struct pic_laser {
  int ix, pol;
  float e0, omega, ramp_steps, y0, z0, waist;
} pic_laser;
int pic_set_laser(pic_context* ctx, const pic_laser* laser);

/* Emitter hook: after every push, per_cell new particles of `species` are
 * injected into each boundary cell of x side `side` (uniform offsets,
 * Maxwellian u_th momenta, drift[0] directed into the domain).  Injected
 * particles deposit no current in their first step (they appear, as in a
 * loader).  per_cell = 0 removes the species' emitter on that side. */
int pic_set_emitter(pic_context* ctx, int species, int side, int per_cell, float u_th,
                    const float drift[3], uint64_t seed);

/* Synthetic load restricted to the cells with x index in [ix_lo, ix_hi]
 * (a plasma slab, e.g. the LPI deck's target). */
int pic_species_load_slab(pic_context* ctx, int species, int ppc, float u_th,
                          const float drift[3], uint64_t seed, int ix_lo, int ix_hi);
/* Runs the context's work on a caller-provided cudaStream_t (a created
 * stream, e.g. torch's current stream, so NCCL send/recv order with the
 * kernels); NULL restores the context's own stream (the legacy default
 * stream cannot be borrowed). */
int pic_set_stream(pic_context* ctx, void* cuda_stream);
/* Halo planes: kind 0 = accumulator rows (12 floats per voxel), 1 = E and B
 * (6 floats), 2 = rhof (1 float); a plane is every (iy, iz) of the padded
 * y-z range at x index ix in [0, nx + 1].  Device buffers. */
#define PIC_HALO_ACCUMULATOR 0
#define PIC_HALO_FIELDS 1
#define PIC_HALO_RHO 2
int pic_halo_plane_bytes(pic_context* ctx, int kind, size_t* out);
int pic_halo_pack(pic_context* ctx, int kind, int ix, void* dst_dev, int zero_after);
int pic_halo_unpack(pic_context* ctx, int kind, int ix, const void* src_dev, int accumulate);
/* Migration after an x-open pic_advance_p: emigrant counts through the low
 * and high x faces (a quiescence point), then pack them — 32-byte device
 * records (pos float4, mom float4), voxel ids already in the receiving
 * slab's frame, ascending particle index — into two device buffers while
 * the store is compacted (holes filled from the tail in index order), then
 * append received records at the end of the store. */
int pic_migrate_counts(pic_context* ctx, int species, size_t out_counts[2]);
int pic_migrate_pack(pic_context* ctx, int species, void* low_dev, void* high_dev);
int pic_migrate_append(pic_context* ctx, int species, const void* records_dev, size_t count);

/* ---- diagnostics -------------------------------------
 * The diagnostic-cadence quantities of SimState::refresh_charge_diagnostics /
 * current_diagnostics (proj/src/sim.cpp:230-266).  compute_div_errors and
 * max_abs_lane are bit-exact; energies are summed in fp64 on the device and
 * rho with float atomics (the reference reassociates these sums itself with
 * its SIMD width / worker count), returned in fp32 like real_t. */
/* clear_rho (proj/src/fields.cpp:203-206). */
int pic_clear_rho(pic_context* ctx);
/* deposit_rho (proj/src/particles.cpp:384-410). */
int pic_deposit_rho(pic_context* ctx, int species);
/* compute_div_errors (proj/src/fields.cpp:253-274). */
int pic_compute_div_errors(pic_context* ctx);
/* SimState::refresh_charge_diagnostics (proj/src/sim.cpp:230-234):
 * clear_rho, deposit_rho of every species, compute_div_errors. */
int pic_refresh_charge_diagnostics(pic_context* ctx);
/* field_energy (proj/src/fields.cpp:276-299): e_b = {E energy, B energy}. */
int pic_field_energy(pic_context* ctx, float e_b[2]);
/* max_abs_lane (proj/src/fields.cpp:301-313), lane in [0, 16). */
int pic_max_abs_lane(pic_context* ctx, int lane, float* out);
/* kinetic_energy_centered (proj/src/particles.cpp:468-501) with the
 * context's current interpolators when centered != 0, else kinetic_energy
 * (proj/src/particles.cpp:460-466). */
int pic_kinetic_energy(pic_context* ctx, int species, int centered, float* out);
/* DiagnosticsRecord (proj/include/minipic/sim.hpp:88-100) minus the wall
 * clock fields; kinetic[] receives one entry per species (kinetic_cap >=
 * species count). */
typedef struct pic_diag {
  float e_energy, b_energy, total_energy, max_div_e_err, max_div_b_err;
  uint64_t particle_count;
} pic_diag;
/* SimState::current_diagnostics (proj/src/sim.cpp:236-266): field energy,
 * load_interpolators, centred kinetic energy per species, total, max div
 * errors, particle count.  Call pic_refresh_charge_diagnostics first for
 * current div errors, as SimState::run does on the diag cadence. */
int pic_diagnostics(pic_context* ctx, pic_diag* out, float* kinetic, size_t kinetic_cap);
/* Energy summation order of pic_diagnostics / pic_field_energy /
 * pic_kinetic_energy (centered): 0 (default) = fp64 device sums of the
 * reference's fp32 terms; 1 = the reference's own fp32 order (sum_squares'
 * 8 interleaved partials per x line, lines summed serially in (lane, z, y)
 * order, fields.cpp:276-299, kernels/scalar.cpp:51-59; kinetic: 8 interleaved
 * partials over the particles in order, particles.cpp:468-501) —
 * bit-identical to the reference in deterministic mode, serial chains of
 * n/8 adds.  pic_sim sets 1 for decks with run.deterministic = true. */
int pic_diagnostics_order(pic_context* ctx, int reference_order);

/* ---- the x-slab decomposed fast step over NCCL --------------
 * One process per GPU; each owns an x-open context (pic_set_x_open, with
 * low_wraps on rank 0) for its slab of a global periodic box of world slabs.
 * pic_dd_step runs SimState::step over the slab with the three x exchanges
 * of the single-domain wrap — particle migration (particles.cpp:348-350),
 * the accumulator halo-add (grid.cpp:78-86) and the E / B halo copy
 * (fields.cpp:35-44) — as grouped ncclSend / ncclRecv on the context stream
 * with no host synchronisation (counts stay on the device; migration
 * buffers hold mig_frac x a boundary plane's share of the capacity, 0 =
 * 1/8; an overflow is a run_abort), captured as a CUDA graph after its first
 * steps.  Fast mode, periodic boxes; walled decks and deterministic mode use
 * the host-sequenced exchanges (halo / migrate entry points below).  NCCL
 * is loaded at run time (the process's libnccl.so.2); world 1 sends to
 * itself. */
typedef struct pic_dd pic_dd;
int pic_dd_unique_id(void* out128); /* ncclGetUniqueId, 128 bytes, on rank 0 */
int pic_dd_create(pic_context* ctx, int rank, int world, const void* unique_id128, double mig_frac, pic_dd** out);
int pic_dd_step(pic_dd* dd, unsigned flags);
/* pic_prepare_step_graphs for pic_dd_step (same arguments; every rank must
 * call it with the same values, as every rank captures the same exchange
 * sequence).  A no-op until one pic_dd_step has run. */
int pic_dd_prepare_graphs(pic_dd* dd, unsigned flags, int steps, int sort_interval, long long steps_taken,
                          int* captured);
int pic_dd_destroy(pic_dd* dd);

/* ---- decks and the SimState run surface ---------------
 * The reference's host API above the step: the deck text format
 * (proj/src/deck.cpp:20-395), SimState::initialize / step / run /
 * emit_diagnostics (proj/src/sim.cpp:25-47, 74-134, 143-306) and the binary
 * field dump (proj/src/fields.cpp:315-344).  Particles are loaded on the
 * host with the reference's Rng (std::mt19937_64 + its uniform and
 * Box-Muller mappings, proj/include/minipic/rng.hpp:17-51), so the initial
 * state is bit-identical to SimState::initialize's.  Deck keys that pick CPU
 * strategies (run.workers, layout, scatter_backend, chunk_size, kernel) are
 * validated and ignored; run.deterministic / exact_gyration map to the
 * PIC_* flags. */
typedef struct pic_deck pic_deck;
typedef struct pic_sim pic_sim;
/* parse_deck (deck.cpp:200-293): PIC_DECK_PARSE_ERROR names key and line. */
int pic_deck_parse(const char* text, pic_deck** out);
int pic_deck_destroy(pic_deck* deck);
/* apply_override (deck.cpp:361-395), e.g. "species.electron.ppc=4"; a
 * failed override leaves the deck unchanged. */
int pic_deck_override(pic_deck* deck, const char* key_eq_value);
/* serialize_deck (deck.cpp:321-359): canonical text; *len = full length
 * (the copy into buf is truncated to cap - 1 and NUL-terminated). */
int pic_deck_serialize(const pic_deck* deck, char* buf, size_t cap, size_t* len);
/* make_grid (deck.cpp:188-198): spacings from extents, dt resolved. */
int pic_deck_grid(const pic_deck* deck, pic_grid* out);
int pic_deck_steps(const pic_deck* deck, long* out);
/* SimState::initialize on a device. */
int pic_sim_create(int device, const pic_deck* deck, pic_sim** out);
int pic_sim_destroy(pic_sim* sim);
/* The sim's device state as a (borrowed) pic_context: species in deck
 * order; valid until pic_sim_destroy; do not pic_context_destroy it. */
int pic_sim_context(pic_sim* sim, pic_context** out);
/* SimState::step followed by sort_due_species (sim.cpp:217-222). */
int pic_sim_step(pic_sim* sim);
int pic_sim_step_count(pic_sim* sim, long* out);
int pic_sim_refresh_charge_diagnostics(pic_sim* sim);
/* SimState::emit_diagnostics: the CSV header on first use, then one row.
 * A call with a null or short buffer computes the row, reports its length
 * and keeps it: the next call returns that same row. */
int pic_sim_emit_diagnostics(pic_sim* sim, char* buf, size_t cap, size_t* len);
/* SimState::run: deck.grid.steps steps with the diagnostic / sort / dump
 * cadences; CSV to csv_path unless NULL; dumps into run.out_dir. */
int pic_sim_run(pic_sim* sim, const char* csv_path);
int pic_sim_dump_fields(pic_sim* sim, const char* path);
/* SimState::warnings (sim.hpp:171), newline-separated. */
int pic_sim_warnings(pic_sim* sim, char* buf, size_t cap, size_t* len);

/* Hooks (HookRegistration / HookFlags / HookContext, proj/include/minipic/
 * sim.hpp:102-127; SimState::run_hooks, proj/src/sim.cpp:185-215): run by
 * pic_sim_run after the step, the due sorts and the due charge refresh,
 * every `interval` steps (never at step 0).  The flags say which host
 * mirrors are refreshed from the device before the callback
 * (particles_to_host: every species' 7 lanes + ids in the reference's order;
 * fields_to_host: the 16 field lanes) and copied back after it
 * (particles_back, fields_back; particle counts are fixed).  Every mirror
 * copy is one copy in pic_sim_copies_performed (copy_between's count,
 * proj/src/layout.cpp:99-118): the legacy flags (all four; flags == NULL)
 * cost 2 x species + 2 copies per invocation, none cost nothing.  A callback
 * returning nonzero aborts the run: PIC_RUN_ABORT "hook '<name>' failed at
 * step <n>: ...". */
typedef struct pic_hook_flags {
  int particles_to_host, fields_to_host, particles_back, fields_back;
} pic_hook_flags;
typedef struct pic_hook_view {
  pic_sim* sim;
  long step;
  float* fields16;        /* 16 x V, lane-major (the reference's field-major layout) */
  size_t nspecies;
  float* const* lanes7;   /* per species: 7 x n, lane-major */
  int32_t* const* ids;    /* per species: n voxel ids */
  const size_t* counts;   /* per species: n */
} pic_hook_view;
typedef int (*pic_hook_fn)(pic_hook_view* view, void* user);
int pic_sim_register_hook(pic_sim* sim, const char* name, long interval, const pic_hook_flags* flags,
                          pic_hook_fn fn, void* user);
/* SimState::copies_performed (sim.hpp:175): mirror copies since initialize. */
int pic_sim_copies_performed(pic_sim* sim, uint64_t* out);

/* ---- timing: CUDA events on the context stream --------------------------*/
int pic_event_record(pic_context* ctx, int slot); /* slot in [0, 64) */
int pic_event_elapsed_ms(pic_context* ctx, int a, int b, float* ms);
/* PhaseTimings (proj/include/minipic/sim.hpp:129-136) measured on the
 * device with CUDA events: when enabled, pic_step / pic_sort_particles
 * bracket their phases; pic_phase_timings returns cumulative milliseconds
 * {interpolate, push, scatter, field, sort} (reset != 0 zeroes them). */
int pic_phase_timing(pic_context* ctx, int enable);
int pic_phase_timings(pic_context* ctx, double out_ms[5], int reset);
/* Kernel launches issued by this context since creation. */
int pic_launch_count(pic_context* ctx, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* PIC_B200_H */
