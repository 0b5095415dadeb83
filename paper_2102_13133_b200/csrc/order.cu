// Voxel order of the fast push's store: kept physically near sorted and
// logically in the reference's order (sm_100a).
//
// The reference sorts a species by voxel every sort_interval steps
// (sort_particles, proj/src/particles.cpp:412-458; run loop
// proj/src/sim.cpp:217-222) and otherwise pushes the store in place, so a
// store's locality decays between sorts (the push falls from
// 8.2 to 4.5e10 pushes/s over a 20-step cycle on the thermal deck).  Here
// every reorder_interval-th push writes its output in voxel chunks — an
// unstable counting sort fused into the push — and the reference's order is
// kept logically:
//
//   * lidx[i]  - the logical (reference-order) index of physical record i,
//                moved with the record by every reordering push;
//   * vcnt[v]  - records per voxel, counted by the push before a reordering
//                one (or by voxel_histogram_kernel), scanned into
//   * vcur[v]  - chunk cursors: the reordering push gives every record a
//                slot in the chunk of the voxel it starts the step in (one
//                atomic per equal-voxel group of 32 records).
//
// A blocked sort_particles only marks the species (relabel_pending) and
// makes the next push a reordering one: that push groups the store by
// exactly the voxels the sort keys on, and relabel_kernel renumbers lidx in
// (voxel, old logical index) order — the stable counting sort's permutation
// — without moving a record.  Any consumer that observes the order
// (downloads, deterministic mode, walls, migration, other sorts) first
// scatters the records into logical order (leave_voxel_order), so callers
// always see the reference's order.
#include "pic_device.cuh"
#include "pic_internal.hpp"

namespace picb {

namespace {

constexpr int kScanThreads = 256, kScanItems = 16, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned lane_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan of cnt[0, n) into cur, clearing cnt, in two fully
// parallel passes over 4096-entry tiles: the tile sums, then every tile adds
// the sums of the tiles before it (at most a few thousand, read from L2) to
// its own block scan.  No inter-CTA waiting: a look-back chain measured
// 167 us for 17 M voxels.
__device__ __forceinline__ unsigned block_sum(unsigned x, unsigned* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  __syncthreads();
  if (lane == 0) s_warp[warp] = x;
  __syncthreads();
  unsigned t = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) t += s_warp[w];
  return t;
}

__global__ void __launch_bounds__(kScanThreads)
vtile_sum_kernel(const unsigned* __restrict__ cnt, long long n, unsigned* __restrict__ tsum) {
  __shared__ unsigned s_warp[kScanThreads / 32];
  const long long base = (long long)blockIdx.x * kScanTile;
  unsigned sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long i = base + (long long)k * kScanThreads + threadIdx.x;  // coalesced
    sum += i < n ? cnt[i] : 0u;
  }
  const unsigned t = block_sum(sum, s_warp);
  if (threadIdx.x == 0) tsum[blockIdx.x] = t;
}

__device__ __forceinline__ int scan_pad(int e) { return e + (e >> 5); }  // conflict-free blocked reads

__global__ void __launch_bounds__(kScanThreads)
vscan_kernel(unsigned* __restrict__ cnt, unsigned* __restrict__ cur, long long n,
             const unsigned* __restrict__ tsum) {
  __shared__ unsigned s_warp[kScanThreads / 32];
  __shared__ unsigned s_data[kScanTile + kScanTile / 32];
  const unsigned t = blockIdx.x;
  const long long base = (long long)t * kScanTile;
  // coalesced (striped) in, cleared behind
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int e = k * kScanThreads + threadIdx.x;
    const long long i = base + e;
    s_data[scan_pad(e)] = i < n ? cnt[i] : 0u;
    if (i < n) cnt[i] = 0u;
  }
  // the exclusive prefix of this tile: the sums of tiles [0, t)
  unsigned pre = 0;
  for (unsigned k = threadIdx.x; k < t; k += kScanThreads) pre += tsum[k];
  pre = block_sum(pre, s_warp);  // (its barriers also publish s_data)
  // each thread scans 16 consecutive entries
  unsigned v[kScanItems];
  unsigned sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = s_data[scan_pad(threadIdx.x * kScanItems + k)];
    sum += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  unsigned woff = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) woff += w < warp ? s_warp[w] : 0u;
  unsigned run = pre + woff + incl - sum;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const unsigned x = v[k];
    v[k] = run;
    run += x;
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) s_data[scan_pad(threadIdx.x * kScanItems + k)] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int e = k * kScanThreads + threadIdx.x;
    const long long i = base + e;
    if (i < n) cur[i] = s_data[scan_pad(e)];
  }
}

// Particles per stored voxel (the first chunk sizes of a store entering the
// continuous order): equal voxels of a warp share one atomic.
__global__ void __launch_bounds__(256)
voxel_histogram_kernel(const float4* __restrict__ pos, long long n, unsigned* __restrict__ cnt,
                       const unsigned long long* __restrict__ ndev = nullptr) {
  if (ndev) n = (long long)*ndev;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int key = i < n ? __float_as_int(__ldcs(pos + i).w) : -1;
  const unsigned peers = __match_any_sync(kFull, key);
  if (key >= 0 && (peers & lane_lt()) == 0) atomicAdd(cnt + key, (unsigned)__popc(peers));
}

// lidx[i] = i (physical == logical), or from a deferred sort permutation:
// the record perm[j] belongs at logical position j.
__global__ void lidx_init_kernel(unsigned* __restrict__ lidx, const unsigned* __restrict__ perm, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (perm)
    lidx[perm[i]] = (unsigned)i;
  else
    lidx[i] = (unsigned)i;
}

// Stable counting sort by voxel as a relabelling: the store is grouped in
// chunks by the voxels the sort keys on (chunk v = [ends[v-1], ends[v])),
// and within a chunk the new logical order is the old logical order.  One
// warp per chunk: each record's rank = the number of smaller old indices
// in its chunk (indices are unique).
__global__ void __launch_bounds__(256)
relabel_kernel(const unsigned* __restrict__ ends, long long V, const unsigned* __restrict__ lin,
               unsigned* __restrict__ lout) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long v = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < V; v += nwarps) {
    const unsigned b = v ? ends[v - 1] : 0u, e = ends[v];
    for (unsigned t0 = b; t0 < e; t0 += 32) {
      const unsigned i = t0 + lane;
      const unsigned my = i < e ? lin[i] : 0xffffffffu;
      unsigned rank = 0;
      for (unsigned u0 = b; u0 < e; u0 += 32) {
        const unsigned o = u0 + lane < e ? lin[u0 + lane] : 0xffffffffu;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) rank += __shfl_sync(kFull, o, k) < my ? 1u : 0u;
      }
      if (i < e) lout[i] = b + rank;
    }
  }
}

// Records into logical order: out[lidx[i]] = record i.
__global__ void __launch_bounds__(256)
to_logical_kernel(const unsigned* __restrict__ lidx, long long n, const float4* __restrict__ pos,
                  const float4* __restrict__ mom, float4* __restrict__ pos_out, float4* __restrict__ mom_out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned d = __ldcs(lidx + i);
  st_stream(pos_out + d, ld_stream(pos + i));
  st_stream(mom_out + d, ld_stream(mom + i));
}

inline unsigned blocks_of(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

bool voxel_order_usable(const Context& c) {
  // periodic boxes only (the order is kept where particles wrap, not leave)
  return c.voxel_order && !c.gc.xopen && !c.gc.ywall && !c.gc.zwall && !has_walls(c);
}

void ensure_count_buffers(Context& c, Species& s) {
  const size_t V = (size_t)c.gc.V;
  if (!s.vcnt) {
    const size_t tiles = (V + kScanTile - 1) / kScanTile;
    CUDA_OK(cudaMalloc(&s.vcnt, V * sizeof(unsigned)));
    CUDA_OK(cudaMalloc(&s.vcur, V * sizeof(unsigned)));
    CUDA_OK(cudaMalloc(&s.vscan, (tiles + 1) * sizeof(unsigned)));
    CUDA_OK(cudaMemsetAsync(s.vcnt, 0, V * sizeof(unsigned), c.stream));
  }
  if (!s.pos_alt) {
    const size_t cap = s.cap ? s.cap : 1;
    CUDA_OK(cudaMalloc(&s.pos_alt, cap * sizeof(float4)));
    CUDA_OK(cudaMalloc(&s.mom_alt, cap * sizeof(float4)));
  }
}

// records per stored voxel into vcnt (the count may live on the device)
void count_stored_voxels(Context& c, Species& s) {
  const long long nl = s.n_on_device ? (long long)s.cap : (long long)s.n;
  if (nl > 0) {
    voxel_histogram_kernel<<<blocks_of(nl), 256, 0, c.stream>>>(s.pos, (long long)s.n, s.vcnt,
                                                                 s.n_on_device ? s.dn : nullptr);
    c.count_launch();
  }
}

static void ensure_order_buffers(Context& c, Species& s) {
  const size_t V = (size_t)c.gc.V;
  const size_t cap = s.cap ? s.cap : 1;
  if (!s.pos_alt) {
    CUDA_OK(cudaMalloc(&s.pos_alt, cap * sizeof(float4)));
    CUDA_OK(cudaMalloc(&s.mom_alt, cap * sizeof(float4)));
  }
  if (!s.lidx) {
    CUDA_OK(cudaMalloc(&s.lidx, cap * sizeof(unsigned)));
    CUDA_OK(cudaMalloc(&s.lidx_alt, cap * sizeof(unsigned)));
  }
  if (!s.vcnt) {
    const size_t tiles = (V + kScanTile - 1) / kScanTile;
    CUDA_OK(cudaMalloc(&s.vcnt, V * sizeof(unsigned)));
    CUDA_OK(cudaMalloc(&s.vcur, V * sizeof(unsigned)));
    CUDA_OK(cudaMalloc(&s.vscan, (tiles + 1) * sizeof(unsigned)));
    CUDA_OK(cudaMemsetAsync(s.vcnt, 0, V * sizeof(unsigned), c.stream));
  }
}

// vcnt -> vcur (exclusive prefix), vcnt cleared.
void scan_voxel_counts(Context& c, Species& s) {
  const long long V = c.gc.V;
  const unsigned tiles = (unsigned)((V + kScanTile - 1) / kScanTile);
  vtile_sum_kernel<<<tiles, kScanThreads, 0, c.stream>>>(s.vcnt, V, s.vscan);
  vscan_kernel<<<tiles, kScanThreads, 0, c.stream>>>(s.vcnt, s.vcur, V, s.vscan);
  c.count_launch(2);
}

void enter_voxel_order(Context& c, Species& s) {
  if (s.ordered) return;
  ensure_order_buffers(c, s);
  const long long n = (long long)s.n;
  if (n > 0) {
    lidx_init_kernel<<<blocks_of(n), 256, 0, c.stream>>>(s.lidx, s.perm_pending ? s.perm : nullptr, n);
    c.count_launch();
  }
  s.perm_pending = false;  // the deferred sort permutation now lives in lidx
  s.ordered = true;
  s.relabel_pending = false;
  s.counts_ready = false;
  // a store entering the order is sorted (load, sort) or about to be
  // reordered: the in-place pushes come first
  s.since_reorder = 0;
}

void prepare_reorder(Context& c, Species& s) {
  if (!s.counts_ready) {  // the previous push did not count the stored voxels
    const long long n = (long long)s.n;
    if (n > 0) {
      voxel_histogram_kernel<<<blocks_of(n), 256, 0, c.stream>>>(s.pos, n, s.vcnt);
      c.count_launch();
    }
    scan_voxel_counts(c, s);
    s.counts_ready = true;
  }
}

void after_ordered_push(Context& c, Species& s, bool reordered, bool counted) {
  if (reordered) {
    std::swap(s.pos, s.pos_alt);
    std::swap(s.mom, s.mom_alt);
    std::swap(s.lidx, s.lidx_alt);
    if (s.relabel_pending) {
      // the push grouped its output by the voxels the owed sort keys on;
      // vcur now holds every chunk's end
      const long long V = c.gc.V;
      const unsigned blocks = (unsigned)std::min<long long>((V + 7) / 8, (long long)c.num_sms * 16);
      relabel_kernel<<<blocks, 256, 0, c.stream>>>(s.vcur, V, s.lidx, s.lidx_alt);
      c.count_launch();
      std::swap(s.lidx, s.lidx_alt);
      s.relabel_pending = false;
    }
    s.since_reorder = 0;
  } else {
    ++s.since_reorder;
  }
  // a reordering or counting push counted its new voxels: chunk cursors
  // ready for the next reordering push
  if (reordered || counted) scan_voxel_counts(c, s);
  s.counts_ready = reordered || counted;
}

void leave_voxel_order(Context& c, Species& s) {
  if (!s.ordered) return;
  s.ordered = false;
  s.counts_ready = false;
  const long long n = (long long)s.n;
  if (n > 0) {
    to_logical_kernel<<<blocks_of(n), 256, 0, c.stream>>>(s.lidx, n, s.pos, s.mom, s.pos_alt, s.mom_alt);
    c.count_launch();
    std::swap(s.pos, s.pos_alt);
    std::swap(s.mom, s.mom_alt);
  }
  if (s.relabel_pending) {
    s.relabel_pending = false;
    sort_species(c, s, PIC_SORT_BLOCKED);
  }
}

}  // namespace picb
