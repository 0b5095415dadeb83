// Host-side internal API of the sm_100a PIC library: the device-resident
// context (the B200 replacement for SimState's FieldArray / InterpolatorArray
// / ScatterBuffer / Species storage, proj/src/sim.cpp:49-72) and the kernel
// launchers.  Not part of the public C-ABI (include/pic_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pic_b200.h"
#include "pic_device.cuh"

namespace picb {

// Error classes of proj/include/minipic/types.hpp:26-36 / sim.hpp:66-69.
struct UsageError : std::logic_error {
  using std::logic_error::logic_error;
};
struct RunAbort : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeckParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CUDA_OK(expr)                                                              \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      throw ::picb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// Species / ParticleStore (proj/include/minipic/particles.hpp:18-45) with the
// 32-byte device record split in two float4 streams.
struct Species {
  std::string name;
  float q = 0, m = 1;
  size_t n = 0, cap = 0;
  float4* pos = nullptr;  // (dx, dy, dz, bits(id))
  float4* mom = nullptr;  // (ux, uy, uz, w)
  float4* pos_alt = nullptr;  // permutation target of the sort (lazy)
  float4* mom_alt = nullptr;
  // x-decomposition: emigrant index lists of the last push (low / high
  // face), capacity mig_cap each; mig_count[2] on the device (lazy)
  unsigned* mig_count = nullptr;
  unsigned* mig_idx = nullptr;
  unsigned mig_cap = 0;
  // Deferred sort permutation (sort.cu): after a blocked sort the records
  // stay where they are and perm[j] names the record that belongs at j; the
  // next default push gathers through it and writes the sorted store, any
  // other consumer materialises it first (materialize()).
  unsigned* perm = nullptr;  // cap entries (lazy)
  bool perm_pending = false;
  // the decomposed C++ step (dd.cu) keeps the count on the device across
  // its migrations: dn is authoritative while n_on_device (s.n stale);
  // species_ref() settles it back to the host
  unsigned long long* dn = nullptr;
  bool n_on_device = false;
  bool resort_pending = false;  // physical-order contexts: a blocked sort owed to the next push
  // Voxel order of the fast push's store (order.cu): physical record i is
  // logical (reference-order) record lidx[i]; vcnt = records per voxel,
  // vcur = chunk cursors of the reordering push (lazy; V entries), vscan =
  // the count scan's tile sums.
  unsigned* lidx = nullptr;
  unsigned* lidx_alt = nullptr;
  unsigned* vcur = nullptr;
  unsigned* vcnt = nullptr;
  unsigned* vscan = nullptr;  // tile sums of the count scan
  bool ordered = false;          // physical order != logical; lidx valid
  bool relabel_pending = false;  // a blocked sort is owed (applied by the next push, a reordering one)
  bool counts_ready = false;     // vcur = chunk starts of the stored voxels (the last push counted)
  unsigned since_reorder = 0;    // pushes since the last reordering one
};

struct Context {
  int device = 0;
  pic_grid grid{};
  GridC gc{};
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;  // set when pic_set_stream borrowed a stream
  float* f = nullptr;         // 16 lanes x V, lane-major
  float4* interp = nullptr;   // V x 5 float4
  float* acc = nullptr;       // V x 12
  int* d_err = nullptr;
  int* h_err = nullptr;       // pinned
  std::vector<Species> species;
  uint64_t launches = 0;
  // advance_p strategy (push.cu): 52 = advance_p_lean (run-per-lane, TMA in /
  // out, two voxel slots of first-segment moments, call-free IEEE loop body,
  // index-only crosser queue; the default); 43 = the same with the full queue;
  // 42 = advance_p_run capped at 85 registers (exact_gyration and
  // out-of-range decks use it); 30 / 20 = earlier run-per-lane forms;
  // 7 = TMA-staged CTA rounds with warp reduction; 0 = one particle per
  // thread; the rest are measured ablations, 99 a timing probe
  int push_variant = 52;
  // sort_particles (blocked): 0 = LSD radix over (voxel, index), 1 = tiled counting sort (ablation)
  int sort_variant = 0;
  int sort_radix_bits = 9;  // LSD digit width (passes = ceil(key bits / width), widths evened out)
  int sort_match = 1;       // group equal digits with match.any (0: per-bit ballots)
  bool sort_defer = true;   // blocked sorts leave the permutation to the next push
  bool reference_order_sums = false;
  // the decomposed fast step's contexts keep no logical order (particles
  // migrate between ranks): a blocked sort is a reordering push (dd.cu)
  bool physical_order = false;  // energies in the reference's fp32 order (pic_diagnostics_order)
  bool voxel_order = true;  // fast periodic pushes keep the store near voxel order (order.cu)
  int reorder_interval = 5;  // every m-th ordered push reorders the store (PIC_REORDER_INTERVAL)
  int order_probe = 0;       // tools library only (PIC_ABLATIONS): timing probes of the reordering push
  int relabel_variant = 0;   // 0 = voxel blocks staged in shared memory, 1 = a warp per chunk (ablation)
  int num_sms = 148;
  // non-periodic x boundaries (boundary.cu): absorbed particle counts per
  // side, the laser source, emitter hooks, steps taken (laser clock)
  uint64_t absorbed[2] = {0, 0};
  pic_laser laser{};
  struct Emitter {
    int species, side, per_cell;
    float u_th, drift[3];
    uint64_t seed;
  };
  std::vector<Emitter> emitters;
  long long steps_done = 0;
  bool decomposed = false;  // pic_set_x_open: x faces exchanged by the host
  // pic_step as CUDA graphs (capi.cu step_graphed): a few configurations
  // The species' host-side state a step leaves behind (buffer swaps of the
  // ordered push / gathering push, order flags): a graph replay re-applies
  // the state its capture produced.
  struct SpeciesState {
    float4 *pos, *mom, *pos_alt, *mom_alt;
    unsigned *lidx, *lidx_alt;
    bool perm_pending, ordered, relabel_pending, counts_ready;
    unsigned since_reorder;
  };
  struct Graph {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;
    std::vector<SpeciesState> post;
  };
  std::vector<Graph> graphs;
  std::vector<std::vector<uint64_t>> graph_seen;  // recent keys (captured on their second occurrence)
  uint64_t graph_captures = 0, graph_replays = 0, graph_plain = 0;
  bool use_graphs = true;
  cudaEvent_t events[64] = {};
  // fast-mode step: species after the first push on side streams (their
  // CTAs fill the first push's tail; the pushes share only the atomically
  // updated accumulator)
  static constexpr int kSide = 3;
  bool fork_species = true;
  bool batch_species = true;  // one advance_p launch per push form for all species (push.cu)
  bool interleave_species = true;  // batched push: species CTAs round robin (push.cu)
  uint64_t batched_launches = 0;  // advance_p_lean launches issued for several species at once
  // fully periodic step: the accumulator / J clears beside the interpolators
  // in one launch, the fold beside the first B half step in one launch
  // (fields.cu)
  bool fuse_fields = true;
  cudaStream_t side[kSide] = {};
  cudaEvent_t fork_ev[kSide] = {}, join_ev[kSide] = {};

  enum ScratchSlot {
    kScrStage = 0, kScrNseg, kScrOff, kScrSegKey, kScrSegW,
    kScrKeyA, kScrValA, kScrKeyB, kScrValB, kScrHist, kScrScan,
    kScrCount, kScrStart, kScrWithin, kScrStaging, kScrSmall, kScrDiag, kScrMigA, kScrMigB, kScrMigC, kScrMigT,
    kScrWall, kScrDiagLines, kScrN
  };
  void* scratch[kScrN] = {};
  size_t scratch_size[kScrN] = {};

  // PhaseTimings (proj/include/minipic/sim.hpp:129-136) on the device clock:
  // CUDA events bracket each phase when enabled; resolved lazily.
  enum Phase { kPhInterp = 0, kPhPush, kPhScatter, kPhField, kPhSort, kPhN };
  bool phase_timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_marks;  // (phase, event index of phase start)
  size_t ev_used = 0;
  double phase_ms[kPhN] = {};
  int phase_open = -1;
  bool nvtx_open = false;  // an NVTX phase range is pushed
  void phase_begin(int ph);
  void phase_end();
  void resolve_phases();
  // the push kernels alone (every advance_p launch bracketed by events on
  // its own stream while phase_timing is on): the roofline's denominator
  std::vector<int> kev;  // event index of each push launch's start (end = +1)
  double push_kernel_ms = 0;
  uint64_t push_kernel_launches = 0;
  int kernel_begin();
  void kernel_end(int idx);

  // host-buffer step pipeline (pic_step_host): copy-in / copy-out streams,
  // double-buffered staging, ordering events
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  static constexpr int kMaxStage = 4;
  int host_bufs = 2;  // staging buffers per direction (PIC_HOST_BUFS: 2-4; 3, 4 measured no faster)
  cudaEvent_t ev_in[kMaxStage] = {}, ev_packed[kMaxStage] = {}, ev_unpacked[kMaxStage] = {},
              ev_out[kMaxStage] = {};
  void* hstage[2 * kMaxStage] = {};  // in[0..kMaxStage), out[0..kMaxStage)
  size_t hstage_bytes = 0;
  size_t host_chunk = (size_t)1 << 24;  // particles per pipelined chunk (16 M: measured best on B200/PCIe5)

  void count_launch(uint64_t k = 1) { launches += k; }
  void* scratch_bytes(int slot, size_t bytes);
  void release();
};

Context* make_context(int device, const pic_grid& g);
void destroy_context(Context* c);
// Waits for the stream, raises latched device errors as RunAbort.
void quiesce(Context& c);
Species& species_at(Context& c, int sid);
// the host count from the device one (decomposed step), synchronous
void settle_count(Context& c, Species& s);

// ---- launchers -------------------------------------------------------------
// ordered: the fast push may keep the store in continuous voxel order (not
// for chunk views of a species, pic_step_host)
void launch_advance_p(Context& c, Species& s, bool exact_gyration, bool ordered = true);
bool launch_advance_p_batch(Context& c, bool exact_gyration);
void launch_advance_p_deterministic(Context& c, Species& s, bool exact_gyration);
// the decomposed step's push (dd.cu): mode 0 in place, 1 in place counting
// the new voxels, 2 reordering into voxel chunks (physical order only);
// false: the lean push cannot run (exact_gyration, ranges) and the store
// was pushed in place without counts
bool launch_advance_p_dd(Context& c, Species& s, bool exact_gyration, int mode);
void launch_load_interpolators(Context& c);
// images: also write B's periodic ghost images (the step's fused ghost sync)
void launch_advance_b(Context& c, float frac, bool images = false);
// unload (jf += f_a * lane, gather form) and/or advance_e in one pass.
void launch_unload_advance_e(Context& c, bool unload, bool advance_e, bool images = false);
void launch_ghost_sync(Context& c);
void launch_ghost_fold(Context& c);
void launch_step_prologue_fused(Context& c);
void launch_fold_advance_b(Context& c);
void launch_clear_currents(Context& c);
void launch_clear_accumulator(Context& c);
void launch_pack_species(Context& c, Species& s, const float* lanes7_dev, const int32_t* ids_dev,
                         size_t n);
void launch_unpack_species(Context& c, Species& s, float* lanes7_dev, int32_t* ids_dev);
// a voxel-ordered store (no relabel / permutation pending) to lanes in logical order
void launch_unpack_logical(Context& c, const Species& s, float* l7, int32_t* ids);
void launch_load_synthetic(Context& c, Species& s, int ppc, float u_th, const float drift[3],
                           uint64_t seed, const pic_sheet* sheet);
void launch_interp_to_lanes(Context& c, float* out18);
void launch_lanes_to_interp(Context& c, const float* in18);

// ---- domain decomposition in x (domain.cu) -----------------------
void ensure_mig_lists(Context& c, Species& s);
// boundary.cu
bool has_walls(const Context& c);
void set_x_boundary(Context& c, int side, int pbc, int fbc);
void set_boundary(Context& c, int face, int pbc, int fbc);
bool absorbing_walls(const Context& c);
void check_walls(const Context& c, bool deterministic);
void absorb_compact(Context& c, Species& s);
void launch_wall_fold(Context& c, int axis);
void launch_wall_e_save(Context& c);
void launch_wall_e(Context& c);
void launch_wall_b(Context& c, float frac);
void launch_laser(Context& c);
void run_emitters(Context& c);
void load_slab(Context& c, Species& s, int ppc, float u_th, const float drift[3], uint64_t seed, int lo, int hi);
void wall_stage(Context& c, int stage, float frac);
void set_x_open(Context& c, bool open, bool low_wraps);
// halo planes: kind 0 = accumulator (12 lanes / voxel), 1 = E and B
// (6 lanes), 2 = rhof; one x plane covers all (iy, iz) incl. ghosts
size_t halo_plane_bytes(const Context& c, int kind);
void halo_pack(Context& c, int kind, int ix, void* dst, bool zero_after);
void halo_unpack(Context& c, int kind, int ix, const void* src, bool accumulate);
// migration after an x-open push: counts of emigrants through the low /
// high face (synchronous), then pack (32 B device records, ids translated
// to the neighbour's frame) + compact, then append received records
void migrate_counts(Context& c, Species& s, size_t out[2]);
void migrate_pack(Context& c, Species& s, void* low_dst, void* high_dst);
void migrate_append(Context& c, Species& s, const void* src, size_t count);

// ---- diagnostics (diag.cu) -----------------------------------------------------
void launch_clear_rho(Context& c);
void launch_deposit_rho(Context& c, Species& s);
void launch_compute_div_errors(Context& c);
void field_energy(Context& c, float e_b[2]);  // synchronous
float max_abs_lane(Context& c, int lane);     // synchronous
float kinetic_energy(Context& c, Species& s, bool centered);  // synchronous
// current_diagnostics' reductions with one readback (fast mode; the
// reference-order sums otherwise): e_b, kinetic[species], max |div e|, |div b|
void diagnostics_batch(Context& c, float e_b[2], float* kinetic, float mdiv[2]);

// ---- sort / scan primitives --------------------------------------------------
int key_bits_for(long long max_key_exclusive);
void exclusive_scan_u32(Context& c, const unsigned* in, unsigned* out, size_t n);
// start[v] = first position of key v in the sorted keys, start[V] = n
void key_run_starts(Context& c, const unsigned* skey, size_t n, size_t V, unsigned* start);
// Stable LSD radix sort of (key, value) pairs on the context stream.  vals ==
// nullptr means values are the identity 0..n-1.  Results are in
// *keys_out / *vals_out (scratch buffers owned by the context).
void radix_sort_pairs(Context& c, const unsigned* keys, const unsigned* vals, size_t n,
                      int key_bits, unsigned** keys_out, unsigned** vals_out);
void sort_species(Context& c, Species& s, int order);
// continuous voxel order (order.cu)
bool voxel_order_usable(const Context& c);
bool copy_logical(Context& c, Species& s, float4* pos, float4* mom);  // order.cu
void enter_voxel_order(Context& c, Species& s);  // logical indices of the current store
void ensure_count_buffers(Context& c, Species& s);  // vcnt / vcur / scan, pos_alt (physical order)
void count_stored_voxels(Context& c, Species& s);   // vcnt += records per stored voxel
void scan_voxel_counts(Context& c, Species& s);     // vcnt -> vcur, vcnt cleared
void prepare_reorder(Context& c, Species& s);    // chunk cursors of the stored voxels
void after_ordered_push(Context& c, Species& s, bool reordered, bool counted);
void leave_voxel_order(Context& c, Species& s);   // records back into logical order
// apply a deferred sort permutation (no-op when none is pending)
void materialize(Context& c, Species& s);
void materialize_all(Context& c);
void materialize_for_sums(Context& c);
// Sort strategies (benchmarking): 0 = LSD radix, 9-bit digits, equal digits
// grouped with match.any (default); 1 = tiled counting sort; 2 = radix,
// 8-bit digits; 3 = radix, 9-bit, per-bit ballot grouping; 4 = 8-bit, ballot.
// Measured on B200, 2^29 particles 19 steps after a sort: 17.6 / 28 / 17.9 /
// 23.0 / 20.6 ms.
inline bool ablations_built() {
#ifdef PIC_ABLATIONS
  return true;
#else
  return false;
#endif
}
inline void set_sort_variant(Context& c, int v) {
  if (v != 0 && !(ablations_built() && v >= 0 && v <= 4))
    throw UsageError("sort variant " + std::to_string(v) +
                     " is not in this build (ablations: libpic_b200_ablate.so)");
  c.sort_variant = v == 1 ? 1 : 0;
  c.sort_radix_bits = (v == 2 || v == 4) ? 8 : 9;
  c.sort_match = (v == 3 || v == 4) ? 0 : 1;
}

// advance_p strategy: the product library holds 52 (advance_p_lean, the
// default) and 42 (advance_p_run: exact_gyration, decks outside the
// call-free ranges); the measured ablations (0-55) and the timing probes
// (90-93, 99: not valid pushes) exist only in libpic_b200_ablate.so.
inline void set_push_variant(Context& c, int v) {
  const bool product = v == 42 || v == 52;
  const bool ablation = (v >= 0 && v <= 55) || (v >= 90 && v <= 93) || v == 99;
  if (!product && !(ablations_built() && ablation))
    throw UsageError("push variant " + std::to_string(v) +
                     " is not in this build (ablations: libpic_b200_ablate.so)");
  c.push_variant = v;
}

// ---- the step --------------------------------------------------------------
void step(Context& c, unsigned flags);
void step_graphed(Context& c, unsigned flags);  // pic_step: one CUDA graph per step configuration
// the graphs of the next `steps` steps (a blocked sort of every species after
// each sort_interval-th) captured ahead without running; returns the count
int prepare_step_graphs(Context& c, unsigned flags, int steps, int sort_interval, long long taken);

// C-ABI error translation (capi.cu): runs fn, maps the exception classes to
// pic_status codes and records the message for pic_last_error().
int capi_guard(const std::function<void()>& fn);

}  // namespace picb

// The C-ABI handle: owns its context unless borrowed (a pic_sim's view).
struct pic_context {
  picb::Context* c;
  bool borrowed;
};
