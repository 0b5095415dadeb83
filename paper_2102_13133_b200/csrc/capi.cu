// Device context and the C-ABI (include/pic_b200.h).
//
// The context owns the device-resident state SimState builds in its
// constructor (proj/src/sim.cpp:49-72) — fields, interpolators, the current
// accumulator, the species stores — on one CUDA stream, plus a device error
// latch that replaces the reference's immediate throws from inside the push
// (proj/src/particles.cpp:190-194,240; proj/src/grid.cpp:42-43).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "pic_internal.hpp"

namespace picb {

namespace {
thread_local std::string g_last_error;
// NVTX range names of the PhaseTimings phases (header-only NVTX3: no cost
// unless a tool is attached)
const char* const kPhaseName[Context::kPhN] = {"interpolate", "push", "scatter", "field", "sort"};
}

void* Context::scratch_bytes(int slot, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (scratch_size[slot] < bytes) {
    if (scratch[slot]) {
      CUDA_OK(cudaStreamSynchronize(stream));
      CUDA_OK(cudaFree(scratch[slot]));
      scratch[slot] = nullptr;
      scratch_size[slot] = 0;
    }
    // slack for slots whose size varies step to step (segments, movers):
    // a new maximum by a few percent must not free and reallocate tens of GB
    const size_t want = ((bytes + bytes / 8) + (2u << 20) - 1) / (2u << 20) * (2u << 20);
    CUDA_OK(cudaMalloc(&scratch[slot], want));
    scratch_size[slot] = want;
  }
  return scratch[slot];
}

void Context::phase_begin(int ph) {
  nvtxRangePushA(kPhaseName[ph]);
  nvtx_open = true;
  if (!phase_timing) return;
  if (ev_used + 2 > ev_pool.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
  }
  CUDA_OK(cudaEventRecord(ev_pool[ev_used], stream));
  ev_marks.emplace_back(ph, (int)ev_used);
  ev_used += 2;
  phase_open = ph;
}

void Context::phase_end() {
  if (nvtx_open) {
    nvtxRangePop();
    nvtx_open = false;
  }
  if (!phase_timing || phase_open < 0) return;
  CUDA_OK(cudaEventRecord(ev_pool[(size_t)ev_marks.back().second + 1], stream));
  phase_open = -1;
  if (ev_used > 4096 && kev.empty()) resolve_phases();
}

int Context::kernel_begin() {
  if (!phase_timing) return -1;
  if (ev_used + 2 > ev_pool.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
  }
  const int idx = (int)ev_used;
  CUDA_OK(cudaEventRecord(ev_pool[(size_t)idx], stream));
  ev_used += 2;
  return idx;
}

void Context::kernel_end(int idx) {
  if (idx < 0) return;
  CUDA_OK(cudaEventRecord(ev_pool[(size_t)idx + 1], stream));
  kev.push_back(idx);
}

void Context::resolve_phases() {
  if (ev_marks.empty() && kev.empty()) return;
  CUDA_OK(cudaDeviceSynchronize());  // push launches may sit on the side streams
  for (const auto& m : ev_marks) {
    float ms = 0;
    CUDA_OK(cudaEventElapsedTime(&ms, ev_pool[(size_t)m.second], ev_pool[(size_t)m.second + 1]));
    phase_ms[m.first] += ms;
  }
  for (int i : kev) {
    float ms = 0;
    CUDA_OK(cudaEventElapsedTime(&ms, ev_pool[(size_t)i], ev_pool[(size_t)i + 1]));
    push_kernel_ms += ms;
    ++push_kernel_launches;
  }
  ev_marks.clear();
  kev.clear();
  ev_used = 0;
}

void Context::release() {
  if (stream) cudaStreamSynchronize(stream);
  if (own_stream && stream != own_stream) cudaStreamSynchronize(own_stream);
  for (auto& s : species) {
    cudaFree(s.pos);
    cudaFree(s.mom);
    cudaFree(s.pos_alt);
    cudaFree(s.mom_alt);
    cudaFree(s.perm);
    cudaFree(s.dn);
    cudaFree(s.lidx);
    cudaFree(s.lidx_alt);
    cudaFree(s.vcur);
    cudaFree(s.vcnt);
    cudaFree(s.vscan);
    cudaFree(s.mig_idx);
    cudaFree(s.mig_count);
  }
  species.clear();
  for (int i = 0; i < kScrN; ++i) {
    cudaFree(scratch[i]);
    scratch[i] = nullptr;
  }
  cudaFree(f);
  cudaFree(interp);
  cudaFree(acc);
  cudaFree(d_err);
  if (h_err) cudaFreeHost(h_err);
  for (auto& e : events)
    if (e) cudaEventDestroy(e);
  for (auto& e : ev_pool) cudaEventDestroy(e);
  ev_pool.clear();
  for (int b = 0; b < kMaxStage; ++b) {
    if (ev_in[b]) cudaEventDestroy(ev_in[b]);
    if (ev_packed[b]) cudaEventDestroy(ev_packed[b]);
    if (ev_unpacked[b]) cudaEventDestroy(ev_unpacked[b]);
    if (ev_out[b]) cudaEventDestroy(ev_out[b]);
  }
  for (auto& p : hstage) {
    cudaFree(p);
    p = nullptr;
  }
  if (cs_in) cudaStreamDestroy(cs_in);
  if (cs_out) cudaStreamDestroy(cs_out);
  cs_in = cs_out = nullptr;
  for (int k = 0; k < kSide; ++k) {
    if (side[k]) cudaStreamDestroy(side[k]);
    if (fork_ev[k]) cudaEventDestroy(fork_ev[k]);
    if (join_ev[k]) cudaEventDestroy(join_ev[k]);
    side[k] = nullptr;
    fork_ev[k] = join_ev[k] = nullptr;
  }
  if (own_stream) stream = own_stream;  // never destroy a borrowed stream
  if (stream) cudaStreamDestroy(stream);
  f = nullptr;
  interp = nullptr;
  acc = nullptr;
  d_err = nullptr;
  h_err = nullptr;
  stream = nullptr;
  own_stream = nullptr;
}

// validate_grid / cfl_limit (proj/src/grid.cpp:7-20), in fp32.
static void validate_grid(const pic_grid& g) {
  if (g.nx < 2 || g.ny < 2 || g.nz < 2) throw UsageError("grid: interior counts must be >= 2");
  if (!(g.hx > 0) || !(g.hy > 0) || !(g.hz > 0)) throw UsageError("grid: spacings must be positive");
  const float s = 1.0f / (g.hx * g.hx) + 1.0f / (g.hy * g.hy) + 1.0f / (g.hz * g.hz);
  const float cfl = 1.0f / std::sqrt(s);
  if (!(g.dt > 0) || g.dt > 0.99f * cfl)
    throw UsageError("grid: dt must satisfy 0 < dt <= 0.99 * cfl_limit");
  const long long V = (long long)(g.nx + 2) * (g.ny + 2) * (g.nz + 2);
  if (V >= (1LL << 31)) throw UsageError("grid: padded voxel count must fit int32 voxel ids");
}

Context* make_context(int device, const pic_grid& g) {
  validate_grid(g);
  auto* c = new Context();
  try {
    c->device = device;
    c->grid = g;
    GridC& gc = c->gc;
    gc.nx = g.nx; gc.ny = g.ny; gc.nz = g.nz;
    gc.pnx = g.nx + 2; gc.pny = g.ny + 2; gc.pnz = g.nz + 2;
    gc.sy = gc.pnx;
    gc.sz = gc.pnx * gc.pny;
    gc.V = (long long)gc.pnx * gc.pny * gc.pnz;
    gc.hx = g.hx; gc.hy = g.hy; gc.hz = g.hz; gc.dt = g.dt;
    // m = ceil(2^64 / d) for d >= 2 (pnx, pny >= 4)
    auto magic = [](unsigned d) {
      const unsigned __int128 one = (unsigned __int128)1 << 64;
      return (unsigned long long)((one + d - 1) / d);
    };
    gc.mag_pnx = magic((unsigned)gc.pnx);
    gc.mag_pny = magic((unsigned)gc.pny);
    CUDA_OK(cudaSetDevice(device));
    CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CUDA_OK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    if (const char* v = std::getenv("PIC_PUSH_VARIANT")) set_push_variant(*c, std::atoi(v));  // profiling knob
    if (const char* v = std::getenv("PIC_FORK_SPECIES")) c->fork_species = std::atoi(v) != 0;  // profiling knob
    if (const char* v = std::getenv("PIC_BATCH_SPECIES")) c->batch_species = std::atoi(v) != 0;  // A/B knob
    if (const char* v = std::getenv("PIC_INTERLEAVE_SPECIES")) c->interleave_species = std::atoi(v) != 0;  // A/B
    if (const char* v = std::getenv("PIC_FUSE_FIELDS")) c->fuse_fields = std::atoi(v) != 0;  // A/B knob
    if (const char* v = std::getenv("PIC_SORT_VARIANT")) set_sort_variant(*c, std::atoi(v));  // profiling knob
    if (const char* v = std::getenv("PIC_SORT_DEFER")) c->sort_defer = std::atoi(v) != 0;     // profiling knob
    if (const char* v = std::getenv("PIC_VOXEL_ORDER")) c->voxel_order = std::atoi(v) != 0;   // profiling knob
    if (const char* v = std::getenv("PIC_REORDER_INTERVAL")) c->reorder_interval = std::atoi(v);  // profiling knob
#ifdef PIC_ABLATIONS
    if (const char* v = std::getenv("PIC_ORDER_PROBE")) c->order_probe = std::atoi(v);  // timing probe
#endif
    if (const char* v = std::getenv("PIC_RELABEL_VARIANT")) c->relabel_variant = std::atoi(v) == 1;  // profiling knob
    if (const char* v = std::getenv("PIC_HOST_BUFS")) c->host_bufs = std::atoi(v);            // profiling knob
    const size_t V = (size_t)gc.V;
    CUDA_OK(cudaMalloc(&c->f, F_COUNT * V * sizeof(float)));
    CUDA_OK(cudaMalloc(&c->interp, kInterpF4 * V * sizeof(float4)));
    CUDA_OK(cudaMalloc(&c->acc, 12 * V * sizeof(float)));
    CUDA_OK(cudaMalloc(&c->d_err, sizeof(int)));
    CUDA_OK(cudaMallocHost(&c->h_err, sizeof(int)));
    CUDA_OK(cudaMemsetAsync(c->f, 0, F_COUNT * V * sizeof(float), c->stream));
    CUDA_OK(cudaMemsetAsync(c->interp, 0, kInterpF4 * V * sizeof(float4), c->stream));
    CUDA_OK(cudaMemsetAsync(c->acc, 0, 12 * V * sizeof(float), c->stream));
    CUDA_OK(cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
  } catch (...) {
    c->release();
    delete c;
    throw;
  }
  return c;
}

void destroy_context(Context* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
  c->release();
  delete c;
}

void quiesce(Context& c) {
  CUDA_OK(cudaMemcpyAsync(c.h_err, c.d_err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
  const int e = *c.h_err;
  if (e) {
    CUDA_OK(cudaMemsetAsync(c.d_err, 0, sizeof(int), c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
    std::string msg;
    if (e & kErrCfl) msg += "advance_particles: particle crossed more than one cell (CFL violation); ";
    if (e & kErrMover) msg += "advance_particles: mover failed to terminate; ";
    if (e & kErrWrap) msg += "wrap_periodic: displacement beyond one cell (CFL violation); ";
    if (e & kErrVoxel) msg += "coords_of: voxel id out of range; ";
    if (e & kErrMigCap) msg += "advance_particles: emigrant / absorbed list overflow (raise the species capacity); ";
    throw RunAbort(msg);
  }
}

// A species for an entry point: any deferred sort permutation is applied
// first (the reference's order is what every caller observes); the push and
// the count take it as it is (species_ref).
void settle_count(Context& c, Species& s) {
  if (!s.n_on_device) return;
  unsigned long long n = 0;
  CUDA_OK(cudaMemcpyAsync(&n, s.dn, sizeof n, cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
  s.n = (size_t)n;
  s.n_on_device = false;
}

static Species& species_ref(Context& c, int sid) {
  if (sid < 0 || sid >= (int)c.species.size()) throw UsageError("species index out of range");
  Species& s = c.species[(size_t)sid];
  settle_count(c, s);
  return s;
}
Species& species_at(Context& c, int sid) {
  Species& s = species_ref(c, sid);
  materialize(c, s);
  return s;
}

// SimState::step (proj/src/sim.cpp:143-183).  unload_currents is fused into
// advance_e: the first advance_b and ghost sync touch neither jf nor the
// accumulator, so moving the unload past them changes no value.
// Phases as PhaseTimings: interpolate / push / scatter (clear + fold) /
// field (B, E with the fused unload, B, three ghost syncs).
static bool fully_periodic(const Context& c) {
  return !c.gc.xopen && !c.gc.ywall && !c.gc.zwall && !has_walls(c);
}

static void step_prologue(Context& c) {
  if (fully_periodic(c) && c.fuse_fields) {  // the clears beside the interpolators, one launch
    c.phase_begin(Context::kPhInterp);
    launch_step_prologue_fused(c);
    c.phase_end();
    return;
  }
  c.phase_begin(Context::kPhScatter);
  launch_clear_accumulator(c);  // scatter_->clear()
  launch_clear_currents(c);     // clear_currents(fields_)
  c.phase_end();
  c.phase_begin(Context::kPhInterp);
  launch_load_interpolators(c);
  c.phase_end();
}

// With x walls (boundary.cu) the x face work changes: wall fold of the
// accumulator's x ghost planes before the y / z folds, the wall-plane B_x
// after each B half step, Mur's saved planes, the laser source and the wall
// E condition around the E update.
static void step_epilogue(Context& c) {
  if (fully_periodic(c) && c.fuse_fields && c.gc.nx >= 3 && c.gc.ny >= 3) {
    // fold + first B half step in one launch, then unload + E, B half step;
    // ghost syncs fused into the updates
    c.phase_begin(Context::kPhField);
    launch_fold_advance_b(c);
    launch_unload_advance_e(c, true, true, true);
    launch_advance_b(c, 0.5f, true);
    c.phase_end();
    return;
  }
  c.phase_begin(Context::kPhScatter);
  wall_stage(c, PIC_STAGE_FOLD, 0.f);
  launch_ghost_fold(c);
  c.phase_end();
  c.phase_begin(Context::kPhField);
  // a fully periodic box: each ghost sync is fused into the update before it
  // (the updated lanes write their own ghost images; the other lanes' ghosts
  // are unchanged since the previous sync) — bit-identical ghosts, three
  // launches fewer per step
  const bool fused = !c.gc.xopen && !c.gc.ywall && !c.gc.zwall && !has_walls(c);
  launch_advance_b(c, 0.5f, fused);
  wall_stage(c, PIC_STAGE_AFTER_B, 0.5f);
  if (!fused) launch_ghost_sync(c);
  wall_stage(c, PIC_STAGE_BEFORE_E, 0.f);
  launch_unload_advance_e(c, true, true, fused);
  wall_stage(c, PIC_STAGE_AFTER_E, 0.f);
  if (!fused) launch_ghost_sync(c);
  launch_advance_b(c, 0.5f, fused);
  wall_stage(c, PIC_STAGE_AFTER_B, 0.5f);
  if (!fused) launch_ghost_sync(c);
  c.phase_end();
}

void step(Context& c, unsigned flags) {
  for (auto& s : c.species) settle_count(c, s);
  const bool det = (flags & PIC_DETERMINISTIC) != 0;
  const bool exact = (flags & PIC_EXACT_GYRATION) != 0;
  const bool walls = has_walls(c);
  check_walls(c, det);
  step_prologue(c);
  c.phase_begin(Context::kPhPush);
  // fast mode without walls: species 1.. on side streams (fork / join; also
  // inside a graph capture), so the small decks' pushes overlap their tails
  const size_t ns = c.species.size();
  // every species in one launch per push form where the deck allows it
  const bool batched = !det && !walls && c.batch_species && launch_advance_p_batch(c, exact);
  // (not while timing phases: each push launch is then timed alone)
  const bool fork = !batched && !det && !walls && c.fork_species && ns > 1 && !c.phase_timing;
  if (fork && !c.side[0]) {
    for (int k = 0; k < Context::kSide; ++k) {
      CUDA_OK(cudaStreamCreateWithFlags(&c.side[k], cudaStreamNonBlocking));
      CUDA_OK(cudaEventCreateWithFlags(&c.fork_ev[k], cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&c.join_ev[k], cudaEventDisableTiming));
    }
  }
  const size_t nside = fork ? std::min<size_t>(ns - 1, Context::kSide) : 0;
  if (nside) CUDA_OK(cudaEventRecord(c.fork_ev[0], c.stream));
  for (size_t k = 0; k < nside; ++k) CUDA_OK(cudaStreamWaitEvent(c.side[k], c.fork_ev[0], 0));
  for (size_t i = 0; i < ns && !batched; ++i) {
    Species& s = c.species[i];
    if (det) {
      launch_advance_p_deterministic(c, s, exact);
    } else if (nside && i > 0) {
      cudaStream_t main = c.stream;
      c.stream = c.side[(i - 1) % nside];
      try {
        launch_advance_p(c, s, exact);
      } catch (...) {
        c.stream = main;
        throw;
      }
      c.stream = main;
    } else {
      launch_advance_p(c, s, exact);
    }
    if (walls && absorbing_walls(c)) absorb_compact(c, s);
  }
  for (size_t k = 0; k < nside; ++k) {
    CUDA_OK(cudaEventRecord(c.join_ev[k], c.side[k]));
    CUDA_OK(cudaStreamWaitEvent(c.stream, c.join_ev[k], 0));
  }
  wall_stage(c, PIC_STAGE_EMIT, 0.f);
  c.phase_end();
  step_epilogue(c);
}

// The step with host-resident species (pic_step_host).  The push of a
// particle needs only the interpolators (built in the prologue) and writes
// only its own record plus the accumulator, so species are streamed through
// the device in chunks: H2D of chunk k+1, pack/push/unpack of chunk k and
// D2H of chunk k-1 run concurrently on three streams with double-buffered
// staging; the field epilogue follows the last push.  Host buffers should be
// pinned (pic_host_register) for the copies to overlap.
static void step_host(Context& c, unsigned flags, float* const* lanes7, int32_t* const* ids) {
  const bool exact = (flags & PIC_EXACT_GYRATION) != 0;
  for (auto& s : c.species) {  // the host arrays replace the device records
    s.perm_pending = false;
    s.ordered = false;
    s.relabel_pending = false;
    s.counts_ready = false;
  }
  size_t nmax = 0;
  for (auto& s : c.species) nmax = std::max(nmax, s.n);
  const size_t chunk = std::max<size_t>(1, std::min<size_t>(nmax, c.host_chunk));
  if (!c.cs_in) {
    CUDA_OK(cudaStreamCreateWithFlags(&c.cs_in, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&c.cs_out, cudaStreamNonBlocking));
    for (int b = 0; b < Context::kMaxStage; ++b) {
      CUDA_OK(cudaEventCreateWithFlags(&c.ev_in[b], cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&c.ev_packed[b], cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&c.ev_unpacked[b], cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&c.ev_out[b], cudaEventDisableTiming));
    }
  }
  const int nb = std::min(std::max(c.host_bufs, 2), (int)Context::kMaxStage);
  if (c.hstage_bytes < chunk * 32 || !c.hstage[nb - 1]) {
    CUDA_OK(cudaStreamSynchronize(c.stream));
    for (auto& p : c.hstage) {
      cudaFree(p);
      p = nullptr;
    }
    for (int b = 0; b < nb; ++b) {
      CUDA_OK(cudaMalloc(&c.hstage[b], chunk * 32));
      CUDA_OK(cudaMalloc(&c.hstage[Context::kMaxStage + b], chunk * 32));
    }
    c.hstage_bytes = chunk * 32;
  }
  step_prologue(c);
  c.phase_begin(Context::kPhPush);
  size_t it = 0;
  for (size_t si = 0; si < c.species.size(); ++si) {
    Species& sp = c.species[si];
    const size_t n = sp.n;
    for (size_t start = 0; start < n; start += chunk, ++it) {
      const size_t cnt = std::min(chunk, n - start);
      const int b = (int)(it % (size_t)nb);
      char* in = static_cast<char*>(c.hstage[b]);
      char* out = static_cast<char*>(c.hstage[Context::kMaxStage + b]);
      // H2D: 7 lane rows (host pitch n) + ids into in[b] once its last pack is done
      CUDA_OK(cudaStreamWaitEvent(c.cs_in, c.ev_packed[b], 0));
      CUDA_OK(cudaMemcpy2DAsync(in, cnt * 4, lanes7[si] + start, n * 4, cnt * 4, 7, cudaMemcpyHostToDevice,
                                c.cs_in));
      CUDA_OK(cudaMemcpyAsync(in + cnt * 28, ids[si] + start, cnt * 4, cudaMemcpyHostToDevice, c.cs_in));
      CUDA_OK(cudaEventRecord(c.ev_in[b], c.cs_in));
      // compute on the context stream
      Species view = sp;
      view.pos = sp.pos + start;
      view.mom = sp.mom + start;
      view.n = cnt;
      CUDA_OK(cudaStreamWaitEvent(c.stream, c.ev_in[b], 0));
      launch_pack_species(c, view, reinterpret_cast<float*>(in), reinterpret_cast<int32_t*>(in + cnt * 28), cnt);
      CUDA_OK(cudaEventRecord(c.ev_packed[b], c.stream));
      launch_advance_p(c, view, exact, false);
      CUDA_OK(cudaStreamWaitEvent(c.stream, c.ev_out[b], 0));
      launch_unpack_species(c, view, reinterpret_cast<float*>(out), reinterpret_cast<int32_t*>(out + cnt * 28));
      CUDA_OK(cudaEventRecord(c.ev_unpacked[b], c.stream));
      // D2H
      CUDA_OK(cudaStreamWaitEvent(c.cs_out, c.ev_unpacked[b], 0));
      // the push never changes the weight lane (particles.cpp:255-360): rows
      // 0-5 (offsets, momenta) and the ids come back, w stays as the host has it
      CUDA_OK(cudaMemcpy2DAsync(lanes7[si] + start, n * 4, out, cnt * 4, cnt * 4, 6, cudaMemcpyDeviceToHost,
                                c.cs_out));
      CUDA_OK(cudaMemcpyAsync(ids[si] + start, out + cnt * 28, cnt * 4, cudaMemcpyDeviceToHost, c.cs_out));
      CUDA_OK(cudaEventRecord(c.ev_out[b], c.cs_out));
    }
  }
  c.phase_end();
  step_epilogue(c);
  CUDA_OK(cudaStreamSynchronize(c.cs_out));
}

}  // namespace picb

// ===========================================================================
// C-ABI
using namespace picb;

namespace {
template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return PIC_OK;
  } catch (const UsageError& e) {
    g_last_error = e.what();
    return PIC_USAGE_ERROR;
  } catch (const RunAbort& e) {
    g_last_error = e.what();
    return PIC_RUN_ABORT;
  } catch (const DeckParseError& e) {
    g_last_error = e.what();
    return PIC_DECK_PARSE_ERROR;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return PIC_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PIC_INTERNAL_ERROR;
  }
}
}  // namespace

int picb::capi_guard(const std::function<void()>& fn) { return guard(fn); }

namespace {
// Every entry point runs on its context's device: contexts on several GPUs
// may share one host thread (the scratch allocations, streams, events and
// launches of a call all follow the current device).
Context& C_(pic_context* p) {
  if (!p || !p->c) throw UsageError("null pic_context");
  CUDA_OK(cudaSetDevice(p->c->device));
  return *p->c;
}
void check_launch() {
  CUDA_OK(cudaGetLastError());
}
}  // namespace

extern "C" {

int pic_version(void) { return PIC_B200_ABI_VERSION; }
const char* pic_last_error(void) { return g_last_error.c_str(); }

int pic_context_create(int device, const pic_grid* grid, pic_context** out) {
  return guard([&] {
    if (!grid || !out) throw UsageError("pic_context_create: null argument");
    *out = nullptr;
    Context* c = make_context(device, *grid);
    *out = new pic_context{c, false};
  });
}

int pic_context_destroy(pic_context* ctx) {
  return guard([&] {
    if (!ctx) return;
    if (ctx->borrowed) throw UsageError("pic_context_destroy: the context belongs to a pic_sim; destroy the sim");
    destroy_context(ctx->c);
    delete ctx;
  });
}

int pic_context_grid(pic_context* ctx, pic_grid* out) {
  return guard([&] { *out = C_(ctx).grid; });
}

int pic_synchronize(pic_context* ctx) {
  return guard([&] {
    check_launch();
    quiesce(C_(ctx));
  });
}

int pic_host_register(void* ptr, size_t bytes) {
  return guard([&] { CUDA_OK(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault)); });
}
int pic_host_unregister(void* ptr) {
  return guard([&] { CUDA_OK(cudaHostUnregister(ptr)); });
}

int pic_species_create(pic_context* ctx, const char* name, float q, float m, size_t capacity,
                       int* out_species) {
  return guard([&] {
    Context& c = C_(ctx);
    if (!(m > 0)) throw UsageError("species: m must be positive");
    Species s;
    s.name = name ? name : "";
    s.q = q;
    s.m = m;
    s.cap = capacity;
    const size_t cap = capacity ? capacity : 1;
    CUDA_OK(cudaMalloc(&s.pos, cap * sizeof(float4)));
    CUDA_OK(cudaMalloc(&s.mom, cap * sizeof(float4)));
    CUDA_OK(cudaMemsetAsync(s.pos, 0, cap * sizeof(float4), c.stream));
    CUDA_OK(cudaMemsetAsync(s.mom, 0, cap * sizeof(float4), c.stream));
    c.species.push_back(s);
    *out_species = (int)c.species.size() - 1;
  });
}

int pic_species_count(pic_context* ctx, int species, size_t* out_n) {
  return guard([&] { *out_n = species_ref(C_(ctx), species).n; });
}

static void validate_ids(const pic_grid& g, const int32_t* ids, size_t n) {
  const int pnx = g.nx + 2, pny = g.ny + 2;
  for (size_t i = 0; i < n; ++i) {
    const int v = ids[i];
    const int ix = v % pnx, rest = v / pnx, iy = rest % pny, iz = rest / pny;
    if (v < 0 || ix < 1 || ix > g.nx || iy < 1 || iy > g.ny || iz < 1 || iz > g.nz)
      throw UsageError("species upload: voxel id " + std::to_string(v) + " (particle " +
                       std::to_string(i) + ") is not an interior voxel");
  }
}

int pic_species_upload(pic_context* ctx, int species, size_t n, const float* lanes7,
                       const int32_t* ids) {
  return guard([&] {
    Context& c = C_(ctx);
    Species& s = species_at(c, species);
    if (n > s.cap) throw UsageError("species upload: count exceeds capacity");
    validate_ids(c.grid, ids, n);
    s.n = n;
    if (n == 0) return;
    char* stg = static_cast<char*>(c.scratch_bytes(Context::kScrStaging, n * 32));
    float* d7 = reinterpret_cast<float*>(stg);
    int32_t* did = reinterpret_cast<int32_t*>(stg + n * 28);
    CUDA_OK(cudaMemcpyAsync(d7, lanes7, n * 28, cudaMemcpyHostToDevice, c.stream));
    CUDA_OK(cudaMemcpyAsync(did, ids, n * 4, cudaMemcpyHostToDevice, c.stream));
    launch_pack_species(c, s, d7, did, n);
    check_launch();
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_species_download(pic_context* ctx, int species, float* lanes7, int32_t* ids) {
  return guard([&] {
    Context& c = C_(ctx);
    // a voxel-ordered store is copied out in logical order and keeps its
    // own order (hooks and dumps do not force a regrouping)
    Species& sr = species_ref(c, species);
    settle_count(c, sr);
    const bool logical = sr.ordered && !sr.relabel_pending && !sr.perm_pending;
    Species& s = logical ? sr : species_at(c, species);
    quiesce(c);
    const size_t n = s.n;
    if (n == 0) return;
    char* stg = static_cast<char*>(c.scratch_bytes(Context::kScrStaging, n * 32));
    float* d7 = reinterpret_cast<float*>(stg);
    int32_t* did = reinterpret_cast<int32_t*>(stg + n * 28);
    if (logical)
      launch_unpack_logical(c, s, d7, did);
    else
      launch_unpack_species(c, s, d7, did);
    check_launch();
    CUDA_OK(cudaMemcpyAsync(lanes7, d7, n * 28, cudaMemcpyDeviceToHost, c.stream));
    CUDA_OK(cudaMemcpyAsync(ids, did, n * 4, cudaMemcpyDeviceToHost, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_species_upload_records(pic_context* ctx, int species, size_t n, const void* pos16,
                               const void* mom16) {
  return guard([&] {
    Context& c = C_(ctx);
    Species& s = species_at(c, species);
    if (n > s.cap) throw UsageError("species upload: count exceeds capacity");
    s.n = n;
    if (n == 0) return;
    CUDA_OK(cudaMemcpyAsync(s.pos, pos16, n * 16, cudaMemcpyDefault, c.stream));
    CUDA_OK(cudaMemcpyAsync(s.mom, mom16, n * 16, cudaMemcpyDefault, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_species_download_records(pic_context* ctx, int species, void* pos16, void* mom16) {
  return guard([&] {
    Context& c = C_(ctx);
    // device buffers of a voxel-ordered store: scattered into logical order
    // directly, the store keeps its order (no regrouping after a download)
    Species& sr = species_ref(c, species);
    cudaPointerAttributes ap{}, am{};
    if (cudaPointerGetAttributes(&ap, pos16) == cudaSuccess && cudaPointerGetAttributes(&am, mom16) == cudaSuccess &&
        ap.type == cudaMemoryTypeDevice && am.type == cudaMemoryTypeDevice) {
      settle_count(c, sr);
      if (copy_logical(c, sr, static_cast<float4*>(pos16), static_cast<float4*>(mom16))) {
        quiesce(c);
        return;
      }
    }
    cudaGetLastError();  // a host pointer: attributes may report an error on older drivers
    Species& s = species_at(c, species);
    quiesce(c);
    if (s.n == 0) return;
    CUDA_OK(cudaMemcpyAsync(pos16, s.pos, s.n * 16, cudaMemcpyDefault, c.stream));
    CUDA_OK(cudaMemcpyAsync(mom16, s.mom, s.n * 16, cudaMemcpyDefault, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_species_load_synthetic(pic_context* ctx, int species, int ppc, float u_th,
                               const float drift[3], uint64_t seed) {
  return guard([&] {
    Context& c = C_(ctx);
    if (ppc < 0) throw UsageError("load_synthetic: ppc must be >= 0");
    const float zero[3] = {0, 0, 0};
    launch_load_synthetic(c, species_at(c, species), ppc, u_th, drift ? drift : zero,
                          seed + 0x9e3779b9ULL * (uint64_t)(species + 1), nullptr);
    check_launch();
  });
}

int pic_species_load_harris(pic_context* ctx, int species, int ppc, float u_th, const float drift[3],
                            uint64_t seed, const pic_sheet* sheet) {
  return guard([&] {
    Context& c = C_(ctx);
    if (ppc < 0) throw UsageError("load_harris: ppc must be >= 0");
    if (!sheet) throw UsageError("load_harris: sheet is null");
    const float zero[3] = {0, 0, 0};
    launch_load_synthetic(c, species_at(c, species), ppc, u_th, drift ? drift : zero,
                          seed + 0x9e3779b9ULL * (uint64_t)(species + 1), sheet);
    check_launch();
  });
}

int pic_fields_upload(pic_context* ctx, const float* fields16) {
  return guard([&] {
    Context& c = C_(ctx);
    CUDA_OK(cudaMemcpyAsync(c.f, fields16, F_COUNT * (size_t)c.gc.V * sizeof(float),
                            cudaMemcpyHostToDevice, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_fields_download(pic_context* ctx, float* fields16) {
  return guard([&] {
    Context& c = C_(ctx);
    quiesce(c);
    CUDA_OK(cudaMemcpyAsync(fields16, c.f, F_COUNT * (size_t)c.gc.V * sizeof(float),
                            cudaMemcpyDeviceToHost, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_interpolators_download(pic_context* ctx, float* interp18) {
  return guard([&] {
    Context& c = C_(ctx);
    quiesce(c);
    const size_t bytes = 18 * (size_t)c.gc.V * sizeof(float);
    float* d = static_cast<float*>(c.scratch_bytes(Context::kScrStaging, bytes));
    launch_interp_to_lanes(c, d);
    check_launch();
    CUDA_OK(cudaMemcpyAsync(interp18, d, bytes, cudaMemcpyDeviceToHost, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_interpolators_upload(pic_context* ctx, const float* interp18) {
  return guard([&] {
    Context& c = C_(ctx);
    const size_t bytes = 18 * (size_t)c.gc.V * sizeof(float);
    float* d = static_cast<float*>(c.scratch_bytes(Context::kScrStaging, bytes));
    CUDA_OK(cudaMemcpyAsync(d, interp18, bytes, cudaMemcpyHostToDevice, c.stream));
    launch_lanes_to_interp(c, d);
    check_launch();
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_accumulator_download(pic_context* ctx, float* acc12) {
  return guard([&] {
    Context& c = C_(ctx);
    quiesce(c);
    CUDA_OK(cudaMemcpyAsync(acc12, c.acc, 12 * (size_t)c.gc.V * sizeof(float), cudaMemcpyDeviceToHost,
                            c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_accumulator_upload(pic_context* ctx, const float* acc12) {
  return guard([&] {
    Context& c = C_(ctx);
    CUDA_OK(cudaMemcpyAsync(c.acc, acc12, 12 * (size_t)c.gc.V * sizeof(float), cudaMemcpyHostToDevice,
                            c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int pic_clear_accumulator(pic_context* ctx) {
  return guard([&] { launch_clear_accumulator(C_(ctx)); });
}
int pic_clear_currents(pic_context* ctx) {
  return guard([&] { launch_clear_currents(C_(ctx)); });
}
int pic_load_interpolators(pic_context* ctx) {
  return guard([&] {
    launch_load_interpolators(C_(ctx));
    check_launch();
  });
}
int pic_advance_p(pic_context* ctx, int species, unsigned flags) {
  return guard([&] {
    Context& c = C_(ctx);
    Species& s = species_ref(c, species);  // the push applies a deferred sort itself
    if (flags & PIC_DETERMINISTIC)
      launch_advance_p_deterministic(c, s, (flags & PIC_EXACT_GYRATION) != 0);
    else
      launch_advance_p(c, s, (flags & PIC_EXACT_GYRATION) != 0);
    check_launch();
  });
}
int pic_ghost_fold_currents(pic_context* ctx) {
  return guard([&] {
    launch_ghost_fold(C_(ctx));
    check_launch();
  });
}
int pic_unload_currents(pic_context* ctx) {
  return guard([&] {
    launch_unload_advance_e(C_(ctx), true, false);
    check_launch();
  });
}
int pic_advance_b(pic_context* ctx, float frac) {
  return guard([&] {
    launch_advance_b(C_(ctx), frac);
    check_launch();
  });
}
int pic_advance_e(pic_context* ctx) {
  return guard([&] {
    launch_unload_advance_e(C_(ctx), false, true);
    check_launch();
  });
}
int pic_unload_advance_e(pic_context* ctx) {
  return guard([&] {
    launch_unload_advance_e(C_(ctx), true, true);
    check_launch();
  });
}
int pic_ghost_sync_fields(pic_context* ctx) {
  return guard([&] {
    launch_ghost_sync(C_(ctx));
    check_launch();
  });
}
int pic_sort_particles(pic_context* ctx, int species, int order) {
  return guard([&] {
    if (order != PIC_SORT_BLOCKED && order != PIC_SORT_INTERLEAVED) throw UsageError("sort: bad order");
    Context& c = C_(ctx);
    c.phase_begin(Context::kPhSort);
    sort_species(c, species_ref(c, species), order);  // resolves any pending order itself
    c.phase_end();
    check_launch();
  });
}
// SimState::step as one CUDA graph launch.  The fast step
// has no host synchronisation, so it is captured once per configuration —
// flags, push variant and every species' (pos, mom, n); the sort swaps the
// record buffers, so two graphs alternate — and relaunched.  Steps with host
// work between kernels run as plain launches: deterministic replay (segment
// count read back), absorbing walls (compaction counts), emitters (n grows),
// the laser (host-computed amplitude), phase timing (host events).
static bool graph_ok(const Context& c, unsigned flags) {
  if (flags & PIC_DETERMINISTIC) return false;
  if (c.phase_timing || !c.emitters.empty() || c.laser.e0 != 0.f) return false;
  if (absorbing_walls(c)) return false;
  return c.use_graphs;
}

static std::vector<uint64_t> graph_key(const Context& c, unsigned flags) {
  std::vector<uint64_t> k{flags, (uint64_t)c.push_variant, (uint64_t)(uintptr_t)c.stream};
  for (int f = 0; f < 6; ++f) k.push_back(((uint64_t)c.gc.wall_p[f] << 8) | (uint64_t)c.gc.wall_f[f]);
  for (const auto& s : c.species) {
    k.push_back((uint64_t)(uintptr_t)s.pos);
    k.push_back((uint64_t)(uintptr_t)s.mom);
    k.push_back((uint64_t)(uintptr_t)s.lidx);
    k.push_back((uint64_t)s.n);
    k.push_back((s.perm_pending ? 1u : 0u) | (s.ordered ? 2u : 0u) | (s.relabel_pending ? 4u : 0u) |
                (s.counts_ready ? 8u : 0u) | ((uint64_t)s.since_reorder << 8));
  }
  return k;
}

static std::vector<Context::SpeciesState> species_state(const Context& c) {
  std::vector<Context::SpeciesState> v;
  for (const auto& s : c.species)
    v.push_back({s.pos, s.mom, s.pos_alt, s.mom_alt, s.lidx, s.lidx_alt, s.perm_pending, s.ordered,
                 s.relabel_pending, s.counts_ready, s.since_reorder});
  return v;
}

static void apply_species_state(Context& c, const std::vector<Context::SpeciesState>& v) {
  for (size_t i = 0; i < v.size() && i < c.species.size(); ++i) {
    Species& s = c.species[i];
    const auto& t = v[i];
    s.pos = t.pos;
    s.mom = t.mom;
    s.pos_alt = t.pos_alt;
    s.mom_alt = t.mom_alt;
    s.lidx = t.lidx;
    s.lidx_alt = t.lidx_alt;
    s.perm_pending = t.perm_pending;
    s.ordered = t.ordered;
    s.relabel_pending = t.relabel_pending;
    s.counts_ready = t.counts_ready;
    s.since_reorder = t.since_reorder;
  }
}

static const Context::Graph& capture_step(Context& c, unsigned flags, const std::vector<uint64_t>& key);

static void step_graphed_impl(Context& c, unsigned flags) {
  for (auto& s : c.species) settle_count(c, s);
  if (!graph_ok(c, flags)) {
    step(c, flags);
    return;
  }
  const auto key = graph_key(c, flags);
  for (auto& g : c.graphs) {
    if (g.key == key) {
      CUDA_OK(cudaGraphLaunch(g.exec, c.stream));
      ++c.graph_replays;
      apply_species_state(c, g.post);
      c.count_launch(g.launches);
      ++c.steps_done;
      return;
    }
  }
  if (std::find(c.graph_seen.begin(), c.graph_seen.end(), key) == c.graph_seen.end()) {
    // first step of a configuration: plain (allocates scratch, sets attributes)
    c.graph_seen.push_back(key);
    if (c.graph_seen.size() > 128) c.graph_seen.erase(c.graph_seen.begin());
    ++c.graph_plain;
    step(c, flags);
    return;
  }
  const Context::Graph& g = capture_step(c, flags, key);
  CUDA_OK(cudaGraphLaunch(g.exec, c.stream));
  c.count_launch(g.launches);
  ++c.steps_done;
}

// Records one step into a new cached graph (nothing runs; the species' host
// state advances as the step would advance it).
static const Context::Graph& capture_step(Context& c, unsigned flags, const std::vector<uint64_t>& key) {
  const uint64_t l0 = c.launches;
  const long long sd = c.steps_done;
  cudaGraph_t graph = nullptr;
  CUDA_OK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  try {
    step(c, flags);
  } catch (...) {
    cudaStreamEndCapture(c.stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  CUDA_OK(cudaStreamEndCapture(c.stream, &graph));
  Context::Graph g;
  g.key = key;
  g.launches = c.launches - l0;
  g.post = species_state(c);
  ++c.graph_captures;
  CUDA_OK(cudaGraphInstantiate(&g.exec, graph, 0));
  CUDA_OK(cudaGraphDestroy(graph));
  c.launches = l0;
  c.steps_done = sd;
  if (c.graphs.size() >= 64) {
    CUDA_OK(cudaGraphExecDestroy(c.graphs.front().exec));
    c.graphs.erase(c.graphs.begin());
  }
  c.graphs.push_back(g);
  return c.graphs.back();
}

// Captures the graphs of the next `steps` fast steps ahead of time, with a
// blocked sort of every species after every step whose count (taken before
// + k) is a multiple of sort_interval (the run loop's cadence,
// proj/src/sim.cpp:217-222): the host state machine (buffer
// pairs, reorder cadence, owed relabels) is walked without running a
// kernel, then restored, so later pic_step calls replay from the first.
// Only for stores already in continuous voxel order (their buffers and
// sort scratch exist; a blocked sort is then host-only): otherwise a no-op.
static int prepare_step_graphs_impl(Context& c, unsigned flags, int steps, int sort_interval, long long taken) {
  if (!graph_ok(c, flags) || steps <= 0) return 0;
  for (auto& s : c.species) {
    settle_count(c, s);
    if (s.n && !s.ordered) return 0;
  }
  const auto saved = species_state(c);
  const uint64_t l0 = c.launches;
  const long long sd = c.steps_done;
  int made = 0;
  try {
    for (int k = 1; k <= steps; ++k) {
      const auto key = graph_key(c, flags);
      const Context::Graph* hit = nullptr;
      for (const auto& g : c.graphs)
        if (g.key == key) hit = &g;
      if (!hit) {
        if (c.graphs.size() >= 63) break;  // keep the cache from evicting what it just made
        hit = &capture_step(c, flags, key);
        ++made;
      }
      apply_species_state(c, hit->post);
      if (sort_interval > 0 && (taken + k) % sort_interval == 0)
        for (auto& s : c.species)
          if (s.n) sort_species(c, s, PIC_SORT_BLOCKED);  // ordered: host-only (relabel owed)
    }
  } catch (...) {
    apply_species_state(c, saved);
    c.launches = l0;
    c.steps_done = sd;
    throw;
  }
  apply_species_state(c, saved);
  c.launches = l0;
  c.steps_done = sd;
  return made;
}

int pic_step(pic_context* ctx, unsigned flags) {
  return guard([&] {
    if (C_(ctx).gc.xopen && !has_walls(C_(ctx)))
      throw UsageError("pic_step: x-open (decomposed) context; the host sequences the step");
    step_graphed_impl(C_(ctx), flags);
    check_launch();
  });
}

int pic_prepare_step_graphs(pic_context* ctx, unsigned flags, int steps, int sort_interval, long long steps_taken,
                            int* captured) {
  return guard([&] {
    Context& c = C_(ctx);
    if (c.gc.xopen && !has_walls(c))
      throw UsageError("pic_prepare_step_graphs: x-open (decomposed) context");
    const int made = prepare_step_graphs_impl(c, flags, steps, sort_interval, steps_taken);
    if (captured) *captured = made;
    check_launch();
  });
}

// Not in the public header: CUDA graphs for pic_step on / off (benchmarking).
int pic_internal_set_graphs(pic_context* ctx, int on) {
  return guard([&] { C_(ctx).use_graphs = on != 0; });
}

int pic_step_host(pic_context* ctx, unsigned flags, float* const* lanes7, int32_t* const* ids) {
  return guard([&] {
    Context& c = C_(ctx);
    // host arrays keep their length: no exchange, absorption or emission
    if (c.gc.xopen || has_walls(c) || !c.emitters.empty())
      throw UsageError("pic_step_host: x-open (decomposed), walled or emitting context (use pic_step)");
    if (!lanes7 || !ids) throw UsageError("pic_step_host: null buffer list");
    for (size_t s = 0; s < c.species.size(); ++s)
      if (c.species[s].n && (!lanes7[s] || !ids[s])) throw UsageError("pic_step_host: null species buffer");
    if (flags & PIC_DETERMINISTIC) {
      // ordered replay needs whole-species passes: upload, step, download
      for (size_t s = 0; s < c.species.size(); ++s) {
        Species& sp = c.species[s];
        const size_t n = sp.n;
        if (n == 0) continue;
        char* stg = static_cast<char*>(c.scratch_bytes(Context::kScrStaging, n * 32));
        CUDA_OK(cudaMemcpyAsync(stg, lanes7[s], n * 28, cudaMemcpyHostToDevice, c.stream));
        CUDA_OK(cudaMemcpyAsync(stg + n * 28, ids[s], n * 4, cudaMemcpyHostToDevice, c.stream));
        launch_pack_species(c, sp, reinterpret_cast<float*>(stg), reinterpret_cast<int32_t*>(stg + n * 28), n);
      }
      step(c, flags);
      for (size_t s = 0; s < c.species.size(); ++s) {
        Species& sp = c.species[s];
        const size_t n = sp.n;
        if (n == 0) continue;
        char* stg = static_cast<char*>(c.scratch_bytes(Context::kScrStaging, n * 32));
        launch_unpack_species(c, sp, reinterpret_cast<float*>(stg), reinterpret_cast<int32_t*>(stg + n * 28));
        CUDA_OK(cudaMemcpyAsync(lanes7[s], stg, n * 28, cudaMemcpyDeviceToHost, c.stream));
        CUDA_OK(cudaMemcpyAsync(ids[s], stg + n * 28, n * 4, cudaMemcpyDeviceToHost, c.stream));
      }
    } else {
      step_host(c, flags, lanes7, ids);
    }
    check_launch();
    quiesce(c);
  });
}

int pic_set_x_boundary(pic_context* ctx, int side, int particle_bc, int field_bc) {
  return guard([&] { set_x_boundary(C_(ctx), side, particle_bc, field_bc); });
}

int pic_set_boundary(pic_context* ctx, int face, int particle_bc, int field_bc) {
  return guard([&] { set_boundary(C_(ctx), face, particle_bc, field_bc); });
}

int pic_wall_stage(pic_context* ctx, int stage, float frac) {
  return guard([&] {
    wall_stage(C_(ctx), stage, frac);
    check_launch();
  });
}

int pic_absorbed_counts(pic_context* ctx, uint64_t out[2], int reset) {
  return guard([&] {
    Context& c = C_(ctx);
    if (!out) throw UsageError("absorbed_counts: out is null");
    CUDA_OK(cudaStreamSynchronize(c.stream));
    out[0] = c.absorbed[0];
    out[1] = c.absorbed[1];
    if (reset) c.absorbed[0] = c.absorbed[1] = 0;
  });
}

int pic_set_laser(pic_context* ctx, const pic_laser* laser) {
  return guard([&] {
    Context& c = C_(ctx);
    if (!laser) throw UsageError("laser: null");
    if (laser->e0 != 0.f) {
      if (laser->ix < 1 || laser->ix > c.gc.nx) throw UsageError("laser: plane ix outside [1, nx]");
      if (laser->pol != 1 && laser->pol != 2) throw UsageError("laser: pol must be 1 (E_y) or 2 (E_z)");
    }
    c.laser = *laser;
  });
}

int pic_set_emitter(pic_context* ctx, int species, int side, int per_cell, float u_th, const float drift[3],
                    uint64_t seed) {
  return guard([&] {
    Context& c = C_(ctx);
    species_at(c, species);
    if (side != 0 && side != 1) throw UsageError("emitter: side must be 0 or 1");
    if (per_cell < 0) throw UsageError("emitter: per_cell must be >= 0");
    auto& E = c.emitters;
    E.erase(std::remove_if(E.begin(), E.end(),
                           [&](const Context::Emitter& e) { return e.species == species && e.side == side; }),
            E.end());
    if (per_cell > 0) {
      Context::Emitter e{species, side, per_cell, u_th, {0.f, 0.f, 0.f}, seed};
      if (drift) std::copy(drift, drift + 3, e.drift);
      E.push_back(e);
    }
  });
}

int pic_species_load_slab(pic_context* ctx, int species, int ppc, float u_th, const float drift[3], uint64_t seed,
                          int ix_lo, int ix_hi) {
  return guard([&] {
    Context& c = C_(ctx);
    const float zero[3] = {0, 0, 0};
    load_slab(c, species_at(c, species), ppc, u_th, drift ? drift : zero,
              seed + 0x9e3779b9ULL * (uint64_t)(species + 1), ix_lo, ix_hi);
    check_launch();
  });
}

int pic_set_x_open(pic_context* ctx, int x_open, int low_wraps) {
  return guard([&] { set_x_open(C_(ctx), x_open != 0, low_wraps != 0); });
}
int pic_set_stream(pic_context* ctx, void* cuda_stream) {
  return guard([&] {
    Context& c = C_(ctx);
    CUDA_OK(cudaStreamSynchronize(c.stream));
    if (!c.own_stream) c.own_stream = c.stream;
    c.stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : c.own_stream;
  });
}
int pic_halo_plane_bytes(pic_context* ctx, int kind, size_t* out) {
  return guard([&] { *out = halo_plane_bytes(C_(ctx), kind); });
}
int pic_halo_pack(pic_context* ctx, int kind, int ix, void* dst_dev, int zero_after) {
  return guard([&] {
    halo_pack(C_(ctx), kind, ix, dst_dev, zero_after != 0);
    check_launch();
  });
}
int pic_halo_unpack(pic_context* ctx, int kind, int ix, const void* src_dev, int accumulate) {
  return guard([&] {
    halo_unpack(C_(ctx), kind, ix, src_dev, accumulate != 0);
    check_launch();
  });
}
int pic_migrate_counts(pic_context* ctx, int species, size_t out_counts[2]) {
  return guard([&] {
    Context& c = C_(ctx);
    quiesce(c);
    migrate_counts(c, species_at(c, species), out_counts);
  });
}
int pic_migrate_pack(pic_context* ctx, int species, void* low_dev, void* high_dev) {
  return guard([&] {
    Context& c = C_(ctx);
    migrate_pack(c, species_at(c, species), low_dev, high_dev);
    check_launch();
  });
}
int pic_migrate_append(pic_context* ctx, int species, const void* records_dev, size_t count) {
  return guard([&] {
    Context& c = C_(ctx);
    migrate_append(c, species_at(c, species), records_dev, count);
  });
}

int pic_clear_rho(pic_context* ctx) {
  return guard([&] { launch_clear_rho(C_(ctx)); });
}
int pic_deposit_rho(pic_context* ctx, int species) {
  return guard([&] {
    Context& c = C_(ctx);
    launch_deposit_rho(c, species_at(c, species));
    check_launch();
  });
}
int pic_compute_div_errors(pic_context* ctx) {
  return guard([&] {
    launch_compute_div_errors(C_(ctx));
    check_launch();
  });
}
int pic_refresh_charge_diagnostics(pic_context* ctx) {
  return guard([&] {
    Context& c = C_(ctx);
    for (auto& s : c.species) settle_count(c, s);
    materialize_for_sums(c);
    launch_clear_rho(c);
    for (auto& s : c.species) launch_deposit_rho(c, s);
    launch_compute_div_errors(c);
    check_launch();
  });
}
int pic_field_energy(pic_context* ctx, float e_b[2]) {
  return guard([&] {
    Context& c = C_(ctx);
    quiesce(c);
    field_energy(c, e_b);
  });
}
int pic_max_abs_lane(pic_context* ctx, int lane, float* out) {
  return guard([&] {
    Context& c = C_(ctx);
    if (lane < 0 || lane >= F_COUNT) throw UsageError("max_abs_lane: lane out of range");
    quiesce(c);
    *out = max_abs_lane(c, lane);
  });
}
int pic_kinetic_energy(pic_context* ctx, int species, int centered, float* out) {
  return guard([&] {
    Context& c = C_(ctx);
    Species& s = species_ref(c, species);
    if (!s.ordered) materialize(c, s);  // order-free sum
    quiesce(c);
    *out = kinetic_energy(c, s, centered != 0);
  });
}
int pic_diagnostics(pic_context* ctx, pic_diag* out, float* kinetic, size_t kinetic_cap) {
  return guard([&] {
    Context& c = C_(ctx);
    if (!out) throw UsageError("diagnostics: null output");
    for (auto& s : c.species) settle_count(c, s);
    materialize_for_sums(c);
    if (kinetic_cap < c.species.size() || (!kinetic && !c.species.empty()))
      throw UsageError("diagnostics: kinetic[] smaller than the species count");
    quiesce(c);
    float eb[2], mdiv[2];
    diagnostics_batch(c, eb, kinetic, mdiv);
    out->e_energy = eb[0];
    out->b_energy = eb[1];
    float total = eb[0] + eb[1];
    uint64_t count = 0;
    for (size_t i = 0; i < c.species.size(); ++i) {
      total += kinetic[i];
      count += c.species[i].n;
    }
    out->total_energy = total;
    out->max_div_e_err = mdiv[0];
    out->max_div_b_err = mdiv[1];
    out->particle_count = count;
  });
}

int pic_diagnostics_order(pic_context* ctx, int reference_order) {
  return guard([&] { C_(ctx).reference_order_sums = reference_order != 0; });
}

int pic_event_record(pic_context* ctx, int slot) {
  return guard([&] {
    Context& c = C_(ctx);
    if (slot < 0 || slot >= 64) throw UsageError("event slot out of range");
    if (!c.events[slot]) CUDA_OK(cudaEventCreate(&c.events[slot]));
    CUDA_OK(cudaEventRecord(c.events[slot], c.stream));
  });
}

int pic_event_elapsed_ms(pic_context* ctx, int a, int b, float* ms) {
  return guard([&] {
    Context& c = C_(ctx);
    if (a < 0 || a >= 64 || b < 0 || b >= 64 || !c.events[a] || !c.events[b])
      throw UsageError("event slot not recorded");
    CUDA_OK(cudaEventSynchronize(c.events[b]));
    CUDA_OK(cudaEventElapsedTime(ms, c.events[a], c.events[b]));
  });
}

int pic_phase_timing(pic_context* ctx, int enable) {
  return guard([&] {
    Context& c = C_(ctx);
    c.resolve_phases();
    c.phase_timing = enable != 0;
  });
}

int pic_phase_timings(pic_context* ctx, double out_ms[5], int reset) {
  return guard([&] {
    Context& c = C_(ctx);
    c.resolve_phases();
    for (int k = 0; k < Context::kPhN; ++k) {
      out_ms[k] = c.phase_ms[k];
      if (reset) c.phase_ms[k] = 0;
    }
  });
}

// Not in the public header: cumulative device ms of the push kernels alone
// and their launch count (phase timing on), the roofline's denominator.
int pic_internal_push_kernel_ms(pic_context* ctx, double* ms, uint64_t* launches, int reset) {
  return guard([&] {
    Context& c = C_(ctx);
    c.resolve_phases();
    *ms = c.push_kernel_ms;
    *launches = c.push_kernel_launches;
    if (reset) {
      c.push_kernel_ms = 0;
      c.push_kernel_launches = 0;
    }
  });
}

// Not in the public header: graph captures / replays / plain steps of pic_step.
int pic_internal_graph_stats(pic_context* ctx, uint64_t out[3]) {
  return guard([&] {
    Context& c = C_(ctx);
    out[0] = c.graph_captures;
    out[1] = c.graph_replays;
    out[2] = c.graph_plain;
  });
}

// Not in the public header: advance_p_lean launches that pushed several
// species at once (host-side count: captures and plain steps, not replays).
int pic_internal_batched_launches(pic_context* ctx, uint64_t* out) {
  return guard([&] { *out = C_(ctx).batched_launches; });
}

// Not in the public header: sort strategy (benchmarking).
int pic_internal_set_sort_variant(pic_context* ctx, int variant) {
  return guard([&] { set_sort_variant(C_(ctx), variant); });
}
// Not in the public header: selects an advance_p strategy (benchmarking).
int pic_internal_set_push_variant(pic_context* ctx, int variant) {
  return guard([&] { set_push_variant(C_(ctx), variant); });
}

// Not in the public header: continuous voxel order of the fast push on / off
// (benchmarking and A/B tests); off leaves every species in logical order.
int pic_internal_set_voxel_order(pic_context* ctx, int on) {
  return guard([&] {
    Context& c = C_(ctx);
    c.voxel_order = on != 0;
    if (!c.voxel_order)
      for (auto& s : c.species) leave_voxel_order(c, s);
  });
}
// Not in the public header: pushes between reorderings of the store.
int pic_internal_set_reorder_interval(pic_context* ctx, int m) {
  return guard([&] {
    if (m < 1) throw UsageError("reorder interval must be >= 1");
    C_(ctx).reorder_interval = m;
  });
}
// Not in the public header: 1 when the species is held in continuous voxel order.
int pic_internal_species_ordered(pic_context* ctx, int species, int* out) {
  return guard([&] { *out = species_ref(C_(ctx), species).ordered ? 1 : 0; });
}

// Not in the public header: the species' records as they lie (no order
// applied) plus, in continuous voxel order, the logical index of each
// (diagnostics of the physical layout).
int pic_internal_download_physical(pic_context* ctx, int species, void* pos16, void* mom16, unsigned* lidx) {
  return guard([&] {
    Context& c = C_(ctx);
    Species& s = species_ref(c, species);
    quiesce(c);
    if (s.n == 0) return;
    CUDA_OK(cudaMemcpyAsync(pos16, s.pos, s.n * 16, cudaMemcpyDefault, c.stream));
    CUDA_OK(cudaMemcpyAsync(mom16, s.mom, s.n * 16, cudaMemcpyDefault, c.stream));
    if (lidx && s.ordered) CUDA_OK(cudaMemcpyAsync(lidx, s.lidx, s.n * 4, cudaMemcpyDefault, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

// Not in the public header: particles per chunk of the pic_step_host pipeline.
int pic_internal_set_host_chunk(pic_context* ctx, size_t particles) {
  return guard([&] { C_(ctx).host_chunk = particles ? particles : 1; });
}

int pic_launch_count(pic_context* ctx, uint64_t* out) {
  return guard([&] { *out = C_(ctx).launches; });
}

}  // extern "C"

void picb::step_graphed(Context& c, unsigned flags) { step_graphed_impl(c, flags); }
int picb::prepare_step_graphs(Context& c, unsigned flags, int steps, int sort_interval, long long taken) {
  return prepare_step_graphs_impl(c, flags, steps, sort_interval, taken);
}
