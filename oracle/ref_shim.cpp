// TEST INFRASTRUCTURE ONLY — never linked into, loaded by, or called from the
// product path (paper_2102_13133_b200/).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load the library
// this file builds (oracle/_ref/libminipic_ref.so).
//
// A thin C-ABI over the *unmodified* reference implementation (minipic,
// /root/reference/proj, compiled from its own sources by oracle/Makefile with
// -DMINIPIC_SINGLE_PRECISION=1, the fp32 build SURVEY.md §0 names as the
// parity oracle).  Every function below only marshals flat field-major
// arrays into the reference's own types and calls the reference function
// named in its comment; no arithmetic of the path lives here.
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "minipic/fields.hpp"
#include "minipic/grid.hpp"
#include "minipic/kernels/dispatch.hpp"
#include "minipic/layout.hpp"
#include "minipic/particles.hpp"
#include "minipic/sim.hpp"
#include "minipic/thread_pool.hpp"

using namespace minipic;

namespace {

thread_local std::string g_err;

struct mref_grid {
  int nx, ny, nz;
  float hx, hy, hz, dt;
};

GridDescriptor to_grid(const mref_grid* g) {
  GridDescriptor d;
  d.nx = g->nx;
  d.ny = g->ny;
  d.nz = g->nz;
  d.hx = g->hx;
  d.hy = g->hy;
  d.hz = g->hz;
  d.dt = g->dt;
  return d;
}

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const usage_error& e) {
    g_err = e.what();
    return 1;
  } catch (const run_abort& e) {
    g_err = e.what();
    return 2;
  } catch (const deck_parse_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

// Field-major (lane * records + record) flat copies into / out of a buffer.
void load_buffer(FieldedBuffer& b, const float* src) {
  for (std::size_t l = 0; l < b.num_fields(); ++l)
    for (std::size_t r = 0; r < b.num_records(); ++r)
      b(r, l) = src[l * b.num_records() + r];
}
void store_buffer(const FieldedBuffer& b, float* dst) {
  for (std::size_t l = 0; l < b.num_fields(); ++l)
    for (std::size_t r = 0; r < b.num_records(); ++r)
      dst[l * b.num_records() + r] = b(r, l);
}

struct SimHandle {
  std::unique_ptr<SimState> s;
};

}  // namespace

extern "C" {

int mref_real_size() { return static_cast<int>(sizeof(real_t)); }
const char* mref_last_error() { return g_err.c_str(); }

// ---- ScatterBuffer (proj/src/layout.cpp:120-207) -------------------------
void* mref_scatter_new(const mref_grid* g, int backend, int workers) {
  const GridDescriptor d = to_grid(g);
  return new ScatterBuffer(d.padded_voxels(), accum_var::count,
                           static_cast<ScatterBackend>(backend), workers);
}
void mref_scatter_free(void* h) { delete static_cast<ScatterBuffer*>(h); }
int mref_scatter_clear(void* h) {
  return guard([&] { static_cast<ScatterBuffer*>(h)->clear(); });
}
int mref_scatter_reduce(void* h, float* dense) {
  return guard([&] {
    auto* sb = static_cast<ScatterBuffer*>(h);
    sb->reduce(std::span<real_t>(dense, sb->num_slots() * sb->num_lanes()));
  });
}

// ---- load_interpolators (proj/src/particles.cpp:42-111) ------------------
int mref_load_interpolators(const mref_grid* g, const float* fields16,
                            float* interp18, int workers) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    InterpolatorArray ia(d, Layout::field_major);
    ThreadPool pool(workers);
    load_interpolators(fa, d, ia, &pool);
    store_buffer(ia.c, interp18);
  });
}

// ---- advance_particles / replay_deposits (proj/src/particles.cpp:255-382) -
int mref_advance_particles(const mref_grid* g, float q, float m, long n,
                           float* lanes7, int* ids, const float* interp18,
                           void* scatter, long chunk, int workers,
                           int exact_gyration, int deterministic) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    Species sp{"s", q, m, 0, SortOrder::blocked,
               ParticleStore(static_cast<std::size_t>(n), Layout::field_major)};
    load_buffer(sp.store.r, lanes7);
    std::memcpy(sp.store.id.data(), ids, sizeof(int) * static_cast<std::size_t>(n));
    InterpolatorArray ia(d, Layout::field_major);
    load_buffer(ia.c, interp18);
    ThreadPool pool(workers);
    DepositStage stage;
    auto* sb = static_cast<ScatterBuffer*>(scatter);
    try {
      advance_particles(sp, ia, *sb, d, static_cast<std::size_t>(chunk),
                        kernels::kernels_for(kernels::detect_arch()), &pool,
                        exact_gyration != 0, deterministic ? &stage : nullptr);
      if (deterministic) replay_deposits(sp, stage, *sb, d);
    } catch (...) {
      store_buffer(sp.store.r, lanes7);
      std::memcpy(ids, sp.store.id.data(), sizeof(int) * static_cast<std::size_t>(n));
      throw;
    }
    store_buffer(sp.store.r, lanes7);
    std::memcpy(ids, sp.store.id.data(), sizeof(int) * static_cast<std::size_t>(n));
  });
}

// ---- ghost_fold_currents (proj/src/grid.cpp:78-99) -----------------------
int mref_ghost_fold(const mref_grid* g, float* dense12) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    ghost_fold_currents(std::span<real_t>(dense12, d.padded_voxels() * 12), 12, d);
  });
}

// ---- clear_currents + unload_currents (proj/src/fields.cpp:195-251) ------
int mref_unload(const mref_grid* g, const float* dense12, float* fields16) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    unload_currents(std::span<const real_t>(dense12, d.padded_voxels() * 12), 12,
                    fa, d);
    store_buffer(fa.f, fields16);
  });
}
int mref_clear_currents(const mref_grid* g, float* fields16) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    clear_currents(fa);
    store_buffer(fa.f, fields16);
  });
}

// ---- advance_b / advance_e / ghost_sync_fields (proj/src/fields.cpp) -----
int mref_advance_b(const mref_grid* g, float* fields16, float frac, int workers) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    ThreadPool pool(workers);
    advance_b(fa, d, frac, kernels::kernels_for(kernels::detect_arch()), &pool);
    store_buffer(fa.f, fields16);
  });
}
int mref_advance_e(const mref_grid* g, float* fields16, int workers) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    ThreadPool pool(workers);
    advance_e(fa, d, kernels::kernels_for(kernels::detect_arch()), &pool);
    store_buffer(fa.f, fields16);
  });
}
int mref_ghost_sync(const mref_grid* g, float* fields16) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    ghost_sync_fields(fa, d);
    store_buffer(fa.f, fields16);
  });
}

// ---- sort_particles (proj/src/particles.cpp:412-458) ---------------------
int mref_sort(long n, float* lanes7, int* ids, int order) {
  return guard([&] {
    Species sp{"s", -1, 1, 0, SortOrder::blocked,
               ParticleStore(static_cast<std::size_t>(n), Layout::field_major)};
    load_buffer(sp.store.r, lanes7);
    std::memcpy(sp.store.id.data(), ids, sizeof(int) * static_cast<std::size_t>(n));
    sort_particles(sp, order ? SortOrder::interleaved : SortOrder::blocked);
    store_buffer(sp.store.r, lanes7);
    std::memcpy(ids, sp.store.id.data(), sizeof(int) * static_cast<std::size_t>(n));
  });
}

// ---- diagnostics (proj/src/particles.cpp:384-501, proj/src/fields.cpp:253-313)
int mref_deposit_rho(const mref_grid* g, float q, long n, const float* lanes7,
                     const int* ids, float* fields16) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    Species sp{"s", q, 1, 0, SortOrder::blocked,
               ParticleStore(static_cast<std::size_t>(n), Layout::field_major)};
    load_buffer(sp.store.r, lanes7);
    std::memcpy(sp.store.id.data(), ids, sizeof(int) * static_cast<std::size_t>(n));
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    deposit_rho(sp, fa, d);
    store_buffer(fa.f, fields16);
  });
}
int mref_compute_div_errors(const mref_grid* g, float* fields16) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    compute_div_errors(fa, d);
    store_buffer(fa.f, fields16);
  });
}
int mref_field_energy(const mref_grid* g, const float* fields16, float* e_b) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    const FieldEnergy fe =
        field_energy(fa, d, kernels::kernels_for(kernels::detect_arch()));
    e_b[0] = fe.e;
    e_b[1] = fe.b;
  });
}
int mref_kinetic_energy_centered(const mref_grid* g, float q, float m, long n,
                                 const float* lanes7, const int* ids,
                                 const float* interp18, float* out) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    Species sp{"s", q, m, 0, SortOrder::blocked,
               ParticleStore(static_cast<std::size_t>(n), Layout::field_major)};
    load_buffer(sp.store.r, lanes7);
    std::memcpy(sp.store.id.data(), ids, sizeof(int) * static_cast<std::size_t>(n));
    InterpolatorArray ia(d, Layout::field_major);
    load_buffer(ia.c, interp18);
    *out = kinetic_energy_centered(sp, ia, d);
  });
}
int mref_max_abs_lane(const mref_grid* g, const float* fields16, int lane,
                      float* out) {
  return guard([&] {
    const GridDescriptor d = to_grid(g);
    FieldArray fa(d, Layout::field_major);
    load_buffer(fa.f, fields16);
    *out = max_abs_lane(fa, d, lane);
  });
}

// ---- deck text (proj/src/deck.cpp) ---------------------------------------
// parse + serialize; with an override applied when kv != NULL.
int mref_deck_roundtrip(const char* text, const char* kv, char* buf, long buflen) {
  return guard([&] {
    Deck d = parse_deck(text);
    if (kv) apply_override(d, kv);
    const std::string t = serialize_deck(d);
    if (static_cast<long>(t.size()) + 1 > buflen) throw usage_error("deck buffer too small");
    std::memcpy(buf, t.c_str(), t.size() + 1);
  });
}

// ---- SimState (proj/src/sim.cpp) -----------------------------------------
void* mref_sim_new(const char* deck_text) {
  void* out = nullptr;
  const int rc = guard([&] {
    auto h = std::make_unique<SimHandle>();
    h->s = std::make_unique<SimState>(SimState::initialize(parse_deck(deck_text)));
    out = h.release();
  });
  return rc == 0 ? out : nullptr;
}
void mref_sim_free(void* h) { delete static_cast<SimHandle*>(h); }

int mref_sim_grid(void* h, mref_grid* out) {
  return guard([&] {
    const GridDescriptor& d = static_cast<SimHandle*>(h)->s->grid();
    *out = {d.nx, d.ny, d.nz, d.hx, d.hy, d.hz, d.dt};
  });
}
int mref_sim_nspecies(void* h) {
  return static_cast<int>(static_cast<SimHandle*>(h)->s->species().size());
}
long mref_sim_species_size(void* h, int s) {
  return static_cast<long>(
      static_cast<SimHandle*>(h)->s->species()[static_cast<std::size_t>(s)].store.size());
}
int mref_sim_species_get(void* h, int s, float* lanes7, int* ids) {
  return guard([&] {
    const Species& sp = static_cast<SimHandle*>(h)->s->species()[static_cast<std::size_t>(s)];
    store_buffer(sp.store.r, lanes7);
    std::memcpy(ids, sp.store.id.data(), sizeof(int) * sp.store.size());
  });
}
int mref_sim_species_set(void* h, int s, const float* lanes7, const int* ids) {
  return guard([&] {
    Species& sp = static_cast<SimHandle*>(h)->s->species()[static_cast<std::size_t>(s)];
    load_buffer(sp.store.r, lanes7);
    std::memcpy(sp.store.id.data(), ids, sizeof(int) * sp.store.size());
  });
}
int mref_sim_fields_get(void* h, float* f16) {
  return guard([&] { store_buffer(static_cast<SimHandle*>(h)->s->fields().f, f16); });
}
int mref_sim_fields_set(void* h, const float* f16) {
  return guard([&] { load_buffer(static_cast<SimHandle*>(h)->s->fields().f, f16); });
}
// SimState::step (proj/src/sim.cpp:143-183), nsteps times, no cadence work.
int mref_sim_step(void* h, long nsteps) {
  return guard([&] {
    for (long i = 0; i < nsteps; ++i) static_cast<SimHandle*>(h)->s->step();
  });
}
// One iteration of SimState::run's loop body without diagnostics / hooks
// (proj/src/sim.cpp:290-295): step() then the due sorts.
int mref_sim_step_and_sort(void* h, long nsteps) {
  return guard([&] {
    SimState& s = *static_cast<SimHandle*>(h)->s;
    for (long i = 0; i < nsteps; ++i) {
      s.step();
      for (auto& sp : s.species())
        if (sp.sort_interval > 0 && s.step_count() % sp.sort_interval == 0)
          sort_particles(sp, sp.sort_order);
    }
  });
}
long mref_sim_step_count(void* h) { return static_cast<SimHandle*>(h)->s->step_count(); }
// SimState::refresh_charge_diagnostics (optional) + current_diagnostics
// (proj/src/sim.cpp:230-266): out = e_energy, b_energy, total_energy,
// max_div_e_err, max_div_b_err, particle_count, kinetic[0..k)
int mref_sim_diagnostics(void* h, int refresh, double* out, int cap) {
  return guard([&] {
    SimState& s = *static_cast<SimHandle*>(h)->s;
    if (refresh) s.refresh_charge_diagnostics();
    const DiagnosticsRecord d = s.current_diagnostics();
    if (cap < 6 + static_cast<int>(d.kinetic.size())) throw usage_error("diagnostics buffer too small");
    out[0] = d.e_energy;
    out[1] = d.b_energy;
    out[2] = d.total_energy;
    out[3] = d.max_div_e_err;
    out[4] = d.max_div_b_err;
    out[5] = static_cast<double>(d.particle_count);
    for (std::size_t k = 0; k < d.kinetic.size(); ++k) out[6 + k] = d.kinetic[k];
  });
}
int mref_sim_run_csv(void* h, char* buf, long buflen) {
  return guard([&] {
    std::ostringstream os;
    static_cast<SimHandle*>(h)->s->run(&os);
    const std::string t = os.str();
    if (static_cast<long>(t.size()) + 1 > buflen) throw usage_error("csv buffer too small");
    std::memcpy(buf, t.c_str(), t.size() + 1);
  });
}
// PhaseTimings (proj/include/minipic/sim.hpp:129-136): interpolate, push,
// scatter, field accumulated seconds.
int mref_sim_timings(void* h, double* out4) {
  return guard([&] {
    const PhaseTimings& t = static_cast<SimHandle*>(h)->s->timings();
    out4[0] = t.interpolate;
    out4[1] = t.push;
    out4[2] = t.scatter;
    out4[3] = t.field;
  });
}

}  // extern "C"
