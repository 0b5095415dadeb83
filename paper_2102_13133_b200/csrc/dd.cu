// The x-slab decomposed fast step in C++ over NCCL: one
// process per GPU, each owning an x-open context (pic_set_x_open) for its
// slab of a global periodic box.  Replaces, per step, the three places where
// the single-domain reference wraps x —
//
//   particle migration   wrap_periodic in x   (proj/src/particles.cpp:348-350, grid.cpp:32-52)
//   accumulator halo-add ghost_fold_currents' x pass   (proj/src/grid.cpp:78-86)
//   E / B halo copy      ghost_sync_fields' x pass     (proj/src/fields.cpp:35-44)
//
// — with grouped ncclSend / ncclRecv on the context stream and no host
// synchronisation: the migration keeps every count on the device.  Each
// migration buffer has a fixed capacity (a fraction of a boundary plane's
// share of the store) and carries its count in-band in its first 32-byte
// slot; holes left by emigrants are refilled from the store's tail by
// device-side lists; the store's count lives on the device (Species::dn)
// until a host caller needs it.  So the whole step — pushes, fold, field
// updates, the exchanges — is one capturable stream of work (a CUDA graph).
//
// The transport is NCCL itself (dlopen'ed: the copy torch has loaded, else
// the system's libnccl.so.2), including at world 1, where every message is
// a send / receive to self.  Order of the matching: each pair of ranks
// issues its messages as (send down, send up; receive from up, receive from
// down), so with world 1 or 2 (one neighbour on both sides) the k-th send
// meets the k-th receive correctly.
//
// The host-sequenced Python path (paper_2102_13133_b200/domain.py) keeps the
// walled decks (LPI) and deterministic mode; this is the fast periodic step.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "pic_device.cuh"
#include "pic_internal.hpp"

namespace picb {

void step_graphed_dd(struct DD& d, unsigned flags);

namespace {

// ---- NCCL through dlopen ---------------------------------------------------------
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  std::string from;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.send) return api;
  // prefer the NCCL already in the process (torch's: the Python wrapper
  // imports torch first), else the system's, loaded locally (a second
  // libnccl.so.2 in the global namespace would capture torch's symbols)
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  api.from = "loaded libnccl.so.2";
  if (!h) {
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    api.from = "libnccl.so.2";
  }
  if (!h) throw UsageError(std::string("decomposed step: NCCL not found (") + dlerror() + ")");
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) throw UsageError(std::string("decomposed step: NCCL lacks ") + n);
    return p;
  };
  api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
  api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
  api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
  api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
  api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
  api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
  api.errorString = reinterpret_cast<decltype(api.errorString)>(sym("ncclGetErrorString"));
  api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
  return api;
}

void NCCL_OK(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().errorString(r));
}

// ---- migration kernels (device-side counts) -------------------------------------
// Migration buffer: slot 0 = {count, 0, 0, 0} (32 B), then cap records of
// (pos, mom).  An emigrant's voxel id moves into the receiver's frame (equal
// slabs: a low-face emigrant lands in the receiver's ix = nx, a high-face
// one in ix = 1) and its slot in the store becomes a hole (voxel -1).
__global__ void dd_pack_kernel(GridC g, const unsigned* __restrict__ idx, const unsigned* __restrict__ cnt,
                               unsigned lcap, float4* __restrict__ pos, const float4* __restrict__ mom,
                               float4* __restrict__ low, float4* __restrict__ high, unsigned bcap,
                               int* __restrict__ err, unsigned* __restrict__ vcnt) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * lcap) return;
  const int side = t >= lcap ? 1 : 0;
  const unsigned k = t - (unsigned)side * lcap;
  const unsigned n = min(cnt[side], lcap);
  float4* buf = side ? high : low;
  if (k == 0) {
    if (cnt[side] > bcap) atomicOr(err, kErrMigCap);
    buf[0] = make_float4(__uint_as_float(min(n, bcap)), 0.f, 0.f, 0.f);
  }
  if (k >= n || k >= bcap) return;
  const unsigned i = idx[(size_t)side * lcap + k];
  float4 p = pos[i];
  const int v = __float_as_int(p.w);
  const unsigned rest = fast_div((unsigned)v, g.mag_pnx);
  const int ix = v - (int)rest * g.pnx;
  p.w = __int_as_float(v - ix + (ix == 0 ? g.nx : 1));
  if (vcnt) atomicAdd(vcnt + v, 0xffffffffu);  // it was counted in its ghost voxel: it leaves
  buf[2 + 2 * (size_t)k] = p;
  buf[3 + 2 * (size_t)k] = mom[i];
  pos[i].w = __int_as_float(-1);  // a hole
}

// holes = emigrant slots below the new count n' = n - E; fillers = the
// non-hole slots of the tail [n', n); both listed (any order: fast mode)
__global__ void dd_lists_kernel(const unsigned* __restrict__ idx, const unsigned* __restrict__ cnt, unsigned lcap,
                                const unsigned long long* __restrict__ dn, const float4* __restrict__ pos,
                                unsigned* __restrict__ holes, unsigned* __restrict__ fillers,
                                unsigned* __restrict__ nlist) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * lcap) return;
  const unsigned c0 = min(cnt[0], lcap), c1 = min(cnt[1], lcap), E = c0 + c1;
  const unsigned long long n = *dn, n1 = n - E;
  if (t < E) {  // the t-th emigrant
    const unsigned i = t < c0 ? idx[t] : idx[(size_t)lcap + (t - c0)];
    if (i < n1) holes[atomicAdd(nlist, 1u)] = i;
    const unsigned long long j = n1 + t;  // the t-th tail slot
    if (__float_as_int(pos[j].w) >= 0) fillers[atomicAdd(nlist + 1, 1u)] = (unsigned)j;
  }
}

__global__ void dd_fill_kernel(const unsigned* __restrict__ holes, const unsigned* __restrict__ fillers,
                               const unsigned* __restrict__ nlist, unsigned lim, float4* __restrict__ pos,
                               float4* __restrict__ mom) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= lim || t >= nlist[0]) return;
  const unsigned h = holes[t], f = fillers[t];
  pos[h] = pos[f];
  mom[h] = mom[f];
}

// immigrants appended at n' (from the low neighbour first, then the high)
__global__ void dd_append_kernel(const unsigned* __restrict__ cnt, unsigned lcap,
                                 const unsigned long long* __restrict__ dn, const float4* __restrict__ from_low,
                                 const float4* __restrict__ from_high, unsigned bcap, unsigned long long cap,
                                 float4* __restrict__ pos, float4* __restrict__ mom, int* __restrict__ err,
                                 unsigned* __restrict__ vcnt) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * bcap) return;
  const unsigned E = min(cnt[0], lcap) + min(cnt[1], lcap);
  const unsigned long long base = *dn - E;
  const unsigned nl = __float_as_uint(from_low[0].x), nh = __float_as_uint(from_high[0].x);
  const unsigned long long total = base + nl + nh;
  if (t == 0 && total > cap) atomicOr(err, kErrMigCap);
  unsigned long long dst;
  const float4* src;
  if (t < nl) {
    dst = base + t;
    src = from_low + 2 + 2 * (size_t)t;
  } else if (t < nl + nh) {
    dst = base + t;
    src = from_high + 2 + 2 * (size_t)(t - nl);
  } else {
    return;
  }
  if (dst >= cap) return;
  const float4 p = src[0];
  pos[dst] = p;
  mom[dst] = src[1];
  if (vcnt) atomicAdd(vcnt + __float_as_int(p.w), 1u);  // counted in the voxel it arrives in
}

// the new count; emigrant counters and list counters cleared
__global__ void dd_count_kernel(unsigned* __restrict__ cnt, unsigned lcap, unsigned long long* __restrict__ dn,
                                const float4* __restrict__ from_low, const float4* __restrict__ from_high,
                                unsigned long long cap, unsigned* __restrict__ nlist) {
  const unsigned E = min(cnt[0], lcap) + min(cnt[1], lcap);
  const unsigned long long total = *dn - E + __float_as_uint(from_low[0].x) + __float_as_uint(from_high[0].x);
  *dn = total < cap ? total : cap;
  cnt[0] = cnt[1] = 0u;
  nlist[0] = nlist[1] = 0u;
}

__global__ void dd_set_count_kernel(unsigned long long* dn, unsigned long long n) { *dn = n; }

}  // namespace

// ---- the decomposed step --------------------------------------------------------------
struct DD {
  Context* c = nullptr;
  int rank = 0, world = 1, low = 0, high = 0;
  ncclComm_t comm = nullptr;
  double mig_frac = 0.125;
  // plane buffers: accumulator (4) and E / B (4): send down / up, receive from up / down
  void* acc[4] = {};
  void* fld[4] = {};
  struct Mig {
    float4* buf[4] = {};  // send down, send up, receive from up, receive from down
    unsigned cap = 0;     // records per buffer
    unsigned* lists = nullptr;  // holes [2 lcap], fillers [2 lcap], counters [2]
    // physical voxel order: pushes since the last reordering one; vcur
    // ready (the previous step counted); this step's push counted
    unsigned since = 0;
    bool counts_ready = false, counted = false;
  };
  std::vector<Mig> mig;
  // CUDA graphs of the step (NCCL calls included), one per host state;
  // replay re-applies the state the capture produced
  struct Graph {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec = nullptr;
    std::vector<Context::SpeciesState> post;
    std::vector<Mig> mig_post;
  };
  std::vector<Graph> graphs;
  std::vector<std::vector<uint64_t>> seen;
  bool use_graphs = true;
  bool order = true;  // physical voxel order (PIC_VOXEL_ORDER=0: in-place pushes + the radix sort)

  void exchange(void* const* b, size_t bytes) {
    NcclApi& n = nccl();
    NCCL_OK(n.groupStart(), "ncclGroupStart");
    NCCL_OK(n.send(b[0], bytes, ncclUint8, low, comm, c->stream), "ncclSend");
    NCCL_OK(n.send(b[1], bytes, ncclUint8, high, comm, c->stream), "ncclSend");
    NCCL_OK(n.recv(b[2], bytes, ncclUint8, high, comm, c->stream), "ncclRecv");
    NCCL_OK(n.recv(b[3], bytes, ncclUint8, low, comm, c->stream), "ncclRecv");
    NCCL_OK(n.groupEnd(), "ncclGroupEnd");
  }

  // planes: send_ix[0] down / send_ix[1] up (-1: none), unpack into recv_ix
  // (a message from up lands in recv_ix[0], from down in recv_ix[1])
  void planes(int kind, int sd, int su, int rd, int ru, bool zero_after, bool accumulate) {
    void** b = kind == 0 ? acc : fld;
    const size_t bytes = halo_plane_bytes(*c, kind);
    if (sd >= 0) halo_pack(*c, kind, sd, b[0], zero_after);
    if (su >= 0) halo_pack(*c, kind, su, b[1], zero_after);
    exchange(b, bytes);
    if (sd >= 0) halo_unpack(*c, kind, rd, b[2], accumulate);
    if (su >= 0) halo_unpack(*c, kind, ru, b[3], accumulate);
  }

  void ensure_species() {
    Context& x = *c;
    if (mig.size() == x.species.size()) return;
    mig.resize(x.species.size());
    for (size_t i = 0; i < x.species.size(); ++i) {
      Species& s = x.species[i];
      ensure_mig_lists(x, s);
      ensure_count_buffers(x, s);
      if (!s.dn) CUDA_OK(cudaMalloc(&s.dn, sizeof(unsigned long long)));
      Mig& m = mig[i];
      if (m.cap) continue;
      const size_t per_plane = std::max<size_t>(1, s.cap) / (size_t)std::max(1, x.gc.nx);
      m.cap = (unsigned)std::min<size_t>(s.mig_cap, std::max<size_t>(4096, (size_t)(mig_frac * per_plane)));
      for (auto& p : m.buf) CUDA_OK(cudaMalloc(&p, (size_t)(m.cap + 1) * 32));
      CUDA_OK(cudaMalloc(&m.lists, ((size_t)4 * s.mig_cap + 2) * sizeof(unsigned)));
      CUDA_OK(cudaMemsetAsync(m.lists + 4 * (size_t)s.mig_cap, 0, 2 * sizeof(unsigned), x.stream));
    }
  }

  void migrate() {
    Context& x = *c;
    for (size_t i = 0; i < x.species.size(); ++i) {
      Species& s = x.species[i];
      Mig& m = mig[i];
      const unsigned lcap = s.mig_cap;
      unsigned* holes = m.lists;
      unsigned* fillers = m.lists + 2 * (size_t)lcap;
      unsigned* nlist = m.lists + 4 * (size_t)lcap;
      const unsigned b2 = (2 * lcap + 255) / 256;
      unsigned* vc = m.counted ? s.vcnt : nullptr;  // keep this step's counts true through the migration
      dd_pack_kernel<<<b2, 256, 0, x.stream>>>(x.gc, s.mig_idx, s.mig_count, lcap, s.pos, s.mom, m.buf[0],
                                              m.buf[1], m.cap, x.d_err, vc);
      dd_lists_kernel<<<b2, 256, 0, x.stream>>>(s.mig_idx, s.mig_count, lcap, s.dn, s.pos, holes, fillers, nlist);
      dd_fill_kernel<<<b2, 256, 0, x.stream>>>(holes, fillers, nlist, 2 * lcap, s.pos, s.mom);
      x.count_launch(3);
      void* b[4] = {m.buf[0], m.buf[1], m.buf[2], m.buf[3]};
      exchange(b, (size_t)(m.cap + 1) * 32);
      dd_append_kernel<<<(2 * m.cap + 255) / 256, 256, 0, x.stream>>>(s.mig_count, lcap, s.dn, m.buf[3], m.buf[2],
                                                                       m.cap, s.cap, s.pos, s.mom, x.d_err, vc);
      dd_count_kernel<<<1, 1, 0, x.stream>>>(s.mig_count, lcap, s.dn, m.buf[3], m.buf[2], s.cap, nlist);
      x.count_launch(2);
      if (m.counted) scan_voxel_counts(x, s);  // chunk starts for the next reordering push
      m.counts_ready = m.counted;
    }
  }

  // SimState::step (proj/src/sim.cpp:143-183) over the slab; the order of
  // paper_2102_13133_b200/domain.py DecomposedSim.step
  void step(unsigned flags) {
    Context& x = *c;
    const bool exact = (flags & PIC_EXACT_GYRATION) != 0;
    x.phase_begin(Context::kPhScatter);
    launch_clear_accumulator(x);
    launch_clear_currents(x);
    x.phase_end();
    x.phase_begin(Context::kPhInterp);
    launch_load_interpolators(x);
    x.phase_end();
    x.phase_begin(Context::kPhPush);
    // physical voxel order: every reorder_interval-th push (and the one
    // after a blocked sort) writes the store in voxel chunks, the one before
    // it counts the new voxels; the counts follow the migration
    const unsigned mi = (unsigned)std::max(1, x.reorder_interval);
    for (size_t i = 0; i < x.species.size(); ++i) {
      Species& s = x.species[i];
      Mig& m = mig[i];
      bool reorder = order && (s.resort_pending || m.since + 1 >= mi);
      bool count = order && !reorder && m.since + 2 >= mi;
      if (reorder && !m.counts_ready) {  // the stored voxels' counts, fresh
        count_stored_voxels(x, s);
        scan_voxel_counts(x, s);
      }
      const bool rcount = reorder && mi == 1;  // the next push reorders too
      if (!launch_advance_p_dd(x, s, exact, reorder ? (rcount ? 3 : 2) : (count ? 1 : 0)))
        reorder = count = false;
      m.counted = (reorder && rcount) || count;
      if (reorder) {
        m.since = 0;
        s.resort_pending = false;
      } else {
        ++m.since;
      }
      m.counts_ready = false;
    }
    x.phase_end();
    const int nx = x.gc.nx;
    x.phase_begin(Context::kPhScatter);
    planes(0, 0, nx + 1, nx, 1, true, true);  // ghost planes folded into the neighbours
    launch_ghost_fold(x);                     // the y, z passes
    planes(0, -1, nx, 0, 0, false, false);    // folded plane nx -> the high neighbour's ghost 0
    x.phase_end();
    x.phase_begin(Context::kPhField);
    auto sync = [&] {
      launch_ghost_sync(x);  // y, z
      planes(1, 1, nx, nx + 1, 0, false, false);
    };
    launch_advance_b(x, 0.5f);
    sync();
    launch_unload_advance_e(x, true, true);
    sync();
    launch_advance_b(x, 0.5f);
    sync();
    x.phase_end();
    x.phase_begin(Context::kPhScatter);  // the exchanges' phase (the push phase is the pushes)
    migrate();
    x.phase_end();
    ++x.steps_done;
  }
};

static std::vector<uint64_t> dd_key(const DD& d, unsigned flags) {
  std::vector<uint64_t> k{flags, (uint64_t)(uintptr_t)d.c->stream};
  for (size_t i = 0; i < d.c->species.size(); ++i) {
    const Species& s = d.c->species[i];
    k.push_back((uint64_t)(uintptr_t)s.pos);
    k.push_back((uint64_t)(uintptr_t)s.mom);
    k.push_back((s.perm_pending ? 1u : 0u) | (s.resort_pending ? 2u : 0u));
    if (i < d.mig.size())
      k.push_back(((uint64_t)d.mig[i].since << 8) | (d.mig[i].counts_ready ? 1u : 0u));
  }
  return k;
}

static void dd_save(const DD& d, std::vector<Context::SpeciesState>& ss, std::vector<DD::Mig>& ms) {
  ss.clear();
  for (const auto& s : d.c->species)
    ss.push_back({s.pos, s.mom, s.pos_alt, s.mom_alt, s.lidx, s.lidx_alt, s.perm_pending, s.ordered,
                  s.resort_pending, s.counts_ready, s.since_reorder});
  ms = d.mig;
}

static void dd_restore(DD& d, const std::vector<Context::SpeciesState>& ss, const std::vector<DD::Mig>& ms) {
  for (size_t i = 0; i < ss.size() && i < d.c->species.size(); ++i) {
    Species& s = d.c->species[i];
    s.pos = ss[i].pos;
    s.mom = ss[i].mom;
    s.pos_alt = ss[i].pos_alt;
    s.mom_alt = ss[i].mom_alt;
    s.resort_pending = ss[i].relabel_pending;  // (the slot carries resort_pending here)
  }
  d.mig = ms;
}

static const DD::Graph& dd_capture(DD& d, unsigned flags, const std::vector<uint64_t>& key);

void step_graphed_dd(DD& d, unsigned flags) {
  Context& c = *d.c;
  if (c.gc.ywall || c.gc.zwall || has_walls(c))
    throw UsageError("decomposed step: periodic boxes only (walled decks: the host-sequenced path)");
  if (flags & PIC_DETERMINISTIC)
    throw UsageError("decomposed step: fast mode only (deterministic: the host-sequenced path)");
  d.ensure_species();
  for (auto& s : c.species) {
    materialize(c, s);  // the in-place push: logical order (a deferred sort is applied first)
    if (!s.n_on_device) {
      dd_set_count_kernel<<<1, 1, 0, c.stream>>>(s.dn, (unsigned long long)s.n);
      s.n_on_device = true;
    }
  }
  const bool graphs = d.use_graphs && !c.phase_timing;
  const auto key = dd_key(d, flags);
  if (graphs)
    for (auto& g : d.graphs)
      if (g.key == key) {
        CUDA_OK(cudaGraphLaunch(g.exec, c.stream));
        dd_restore(d, g.post, g.mig_post);
        ++c.steps_done;
        return;
      }
  if (!graphs || std::find(d.seen.begin(), d.seen.end(), key) == d.seen.end()) {
    // plain the first time a state comes up (allocations, attributes)
    if (graphs) {
      d.seen.push_back(key);
      if (d.seen.size() > 64) d.seen.erase(d.seen.begin());
    }
    d.step(flags);
    return;
  }
  CUDA_OK(cudaGraphLaunch(dd_capture(d, flags, key).exec, c.stream));
  ++c.steps_done;
}

// Records one decomposed step (its NCCL exchanges included) into a new
// cached graph without running it; the host state advances as the step's.
static const DD::Graph& dd_capture(DD& d, unsigned flags, const std::vector<uint64_t>& key) {
  Context& c = *d.c;
  const uint64_t l0 = c.launches;
  cudaGraph_t graph = nullptr;
  CUDA_OK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  try {
    d.step(flags);
  } catch (...) {
    cudaStreamEndCapture(c.stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  CUDA_OK(cudaStreamEndCapture(c.stream, &graph));
  DD::Graph g;
  g.key = key;
  CUDA_OK(cudaGraphInstantiate(&g.exec, graph, 0));
  CUDA_OK(cudaGraphDestroy(graph));
  dd_save(d, g.post, g.mig_post);
  --c.steps_done;
  c.launches = l0;
  if (d.graphs.size() >= 32) {
    cudaGraphExecDestroy(d.graphs.front().exec);
    d.graphs.erase(d.graphs.begin());
  }
  d.graphs.push_back(std::move(g));
  return d.graphs.back();
}

// pic_prepare_step_graphs for the decomposed step: the graphs of the next
// `steps` steps (a blocked sort of every species after each step whose
// count steps_taken + k is a multiple of sort_interval: host-only here, the
// next push reorders) captured ahead without running; host state restored.
// Every rank walks the same state machine, so the captured exchanges match.
static int dd_prepare(DD& d, unsigned flags, int steps, int sort_interval, long long taken) {
  Context& c = *d.c;
  if (!d.use_graphs || c.phase_timing || steps <= 0 || d.mig.size() != c.species.size()) return 0;
  for (auto& s : c.species)
    if (!s.n_on_device || s.perm_pending || s.ordered) return 0;
  std::vector<Context::SpeciesState> ss0;
  std::vector<DD::Mig> ms0;
  dd_save(d, ss0, ms0);
  const long long sd = c.steps_done;
  const uint64_t l0 = c.launches;
  int made = 0;
  try {
    for (int k = 1; k <= steps; ++k) {
      const auto key = dd_key(d, flags);
      const DD::Graph* hit = nullptr;
      for (const auto& g : d.graphs)
        if (g.key == key) hit = &g;
      if (!hit) {
        if (d.graphs.size() >= 31) break;
        hit = &dd_capture(d, flags, key);
        ++made;
      }
      dd_restore(d, hit->post, hit->mig_post);
      if (sort_interval > 0 && (taken + k) % sort_interval == 0)
        for (auto& s : c.species) sort_species(c, s, PIC_SORT_BLOCKED);  // physical order: host-only
    }
  } catch (...) {
    dd_restore(d, ss0, ms0);
    c.steps_done = sd;
    c.launches = l0;
    throw;
  }
  dd_restore(d, ss0, ms0);
  c.steps_done = sd;
  c.launches = l0;
  return made;
}

}  // namespace picb

using namespace picb;

struct pic_dd {
  DD d;
};

extern "C" {

int pic_dd_unique_id(void* out128) {
  return capi_guard([&] {
    if (!out128) throw UsageError("pic_dd_unique_id: null");
    ncclUniqueId id;
    NCCL_OK(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof id);
  });
}

int pic_dd_create(pic_context* ctx, int rank, int world, const void* unique_id128, double mig_frac, pic_dd** out) {
  return capi_guard([&] {
    if (!ctx || !ctx->c || !unique_id128 || !out) throw UsageError("pic_dd_create: null argument");
    if (world < 1 || rank < 0 || rank >= world) throw UsageError("pic_dd_create: bad rank / world");
    Context& c = *ctx->c;
    CUDA_OK(cudaSetDevice(c.device));
    if (!c.gc.xopen) throw UsageError("pic_dd_create: the context must be x-open (pic_set_x_open)");
    auto* p = new pic_dd;
    p->d.c = &c;
    p->d.rank = rank;
    p->d.world = world;
    p->d.low = (rank + world - 1) % world;
    p->d.high = (rank + 1) % world;
    if (mig_frac > 0) p->d.mig_frac = mig_frac;
    if (const char* v = std::getenv("PIC_DD_GRAPHS")) p->d.use_graphs = std::atoi(v) != 0;
    p->d.order = c.voxel_order;
    c.physical_order = p->d.order;
    ncclUniqueId id;
    std::memcpy(&id, unique_id128, sizeof id);
    try {
      NCCL_OK(nccl().commInitRank(&p->d.comm, world, id, rank), "ncclCommInitRank");
      const size_t ab = halo_plane_bytes(c, 0), fb = halo_plane_bytes(c, 1);
      for (auto& b : p->d.acc) CUDA_OK(cudaMalloc(&b, ab));
      for (auto& b : p->d.fld) CUDA_OK(cudaMalloc(&b, fb));
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

int pic_dd_step(pic_dd* dd, unsigned flags) {
  return capi_guard([&] {
    if (!dd) throw UsageError("pic_dd_step: null");
    CUDA_OK(cudaSetDevice(dd->d.c->device));
    step_graphed_dd(dd->d, flags);
    CUDA_OK(cudaGetLastError());
  });
}

int pic_dd_prepare_graphs(pic_dd* dd, unsigned flags, int steps, int sort_interval, long long steps_taken,
                          int* captured) {
  return capi_guard([&] {
    if (!dd) throw UsageError("pic_dd_prepare_graphs: null");
    CUDA_OK(cudaSetDevice(dd->d.c->device));
    const int made = dd_prepare(dd->d, flags, steps, sort_interval, steps_taken);
    if (captured) *captured = made;
    CUDA_OK(cudaGetLastError());
  });
}

int pic_dd_destroy(pic_dd* dd) {
  if (!dd) return PIC_OK;
  return capi_guard([&] {
    DD& d = dd->d;
    cudaSetDevice(d.c->device);
    cudaStreamSynchronize(d.c->stream);
    for (auto& g : d.graphs) cudaGraphExecDestroy(g.exec);
    d.c->physical_order = false;
    for (auto& b : d.acc) cudaFree(b);
    for (auto& b : d.fld) cudaFree(b);
    for (auto& m : d.mig) {
      for (auto& p : m.buf) cudaFree(p);
      cudaFree(m.lists);
    }
    if (d.comm) nccl().commDestroy(d.comm);
    delete dd;
  });
}

}  // extern "C"
