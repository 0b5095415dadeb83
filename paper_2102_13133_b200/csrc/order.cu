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

// The same relabelling over a block of kRelVB voxels per CTA: the chunks'
// ends and their logical indices are staged in shared memory with coalesced
// loads, then a warp per chunk ranks its records against the staged copy
// (broadcast reads).  relabel_kernel, one warp per chunk straight from
// global memory, measured 8.1 ms per 2^29 records (dependent ends -> lin
// loads per 32 records, latency bound).  Blocks whose records exceed the
// staging buffer rank from global memory.
constexpr int kRelThreads = 256, kRelCap = 8192;
constexpr unsigned kBig = 0x7fffffffu;  // never smaller than a logical index (< 2^31 - 1)

// [x < my] as the sign bit of x - my (both < 2^31): a compare-and-add is two
// instructions (IADD + LEA.HI)
__device__ __forceinline__ unsigned lt_bit(unsigned x, unsigned my) { return (x - my) >> 31; }

// rank[r] += #{ j in [lo, hi) : s[j] < my[r] } for R records per lane, with
// 128-bit broadcast reads over the 4-aligned cover [a0, a1) of the chunk;
// the cover's words outside it (neighbouring chunks, or past the staged
// range) are masked in the first and last vectors only
template <int R>
__device__ __forceinline__ void rank_cover(const unsigned* __restrict__ s, unsigned lo, unsigned hi,
                                           const unsigned (&my)[R], unsigned (&rank)[R]) {
  const unsigned a0 = lo & ~3u, a1 = (hi + 3u) & ~3u;
  auto add = [&](uint4 x) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      rank[r] += lt_bit(x.x, my[r]) + lt_bit(x.y, my[r]) + lt_bit(x.z, my[r]) + lt_bit(x.w, my[r]);
  };
  auto masked = [&](unsigned q) {
    uint4 x = *reinterpret_cast<const uint4*>(s + q);
    x.x = q + 0u >= lo && q + 0u < hi ? x.x : kBig;
    x.y = q + 1u >= lo && q + 1u < hi ? x.y : kBig;
    x.z = q + 2u >= lo && q + 2u < hi ? x.z : kBig;
    x.w = q + 3u >= lo && q + 3u < hi ? x.w : kBig;
    return x;
  };
  add(masked(a0));
  if (a1 - a0 > 4u) {
#pragma unroll 4
    for (unsigned q = a0 + 4u; q < a1 - 4u; q += 4) add(*reinterpret_cast<const uint4*>(s + q));
    add(masked(a1 - 4u));
  }
}

// Ranks of up to 32 (R = 1) or 64 (R = 2) distinct keys held one (two) per
// lane, lanes past the chunk holding kBig: a bitonic sort across the warp
// (15 / 21 compare-exchange stages, a shuffle and a min/max each), then
// every key's rank as its lower bound in the sorted keys (5 / 6 shuffle
// probes).  ~80 / ~170 instructions per chunk against c^2/16 for the
// all-pairs count.
template <int R>
__device__ __forceinline__ void warp_ranks(const unsigned (&key)[R], unsigned (&rank)[R], int lane) {
  unsigned a[R];
#pragma unroll
  for (int r = 0; r < R; ++r) a[r] = key[r];
  constexpr int kN = 32 * R;
#pragma unroll
  for (int k = 2; k <= kN; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j == 32) {  // R == 2: the partner is the lane's other key
        const unsigned lo_ = min(a[0], a[1]), hi_ = max(a[0], a[1]);
        a[0] = lo_;  // k == 64: ascending everywhere
        a[1] = hi_;
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const unsigned p = __shfl_xor_sync(kFull, a[r], j);
          const unsigned i = (unsigned)(r * 32 + lane);
          const bool up = (i & (unsigned)k) == 0u, lower = (lane & j) == 0;
          a[r] = (up == lower) ? min(a[r], p) : max(a[r], p);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    unsigned pos = 0;
#pragma unroll
    for (int st = kN / 2; st >= 1; st >>= 1) {
      const unsigned idx = pos + (unsigned)st - 1u;
      unsigned y = __shfl_sync(kFull, a[0], (int)(idx & 31u));
      if (R == 2) {
        const unsigned y1 = __shfl_sync(kFull, a[R - 1], (int)(idx & 31u));
        y = idx >= 32u ? y1 : y;
      }
      pos += y < key[r] ? (unsigned)st : 0u;
    }
    rank[r] = pos;
  }
}

__global__ void __launch_bounds__(kRelThreads)
relabel_tiled_kernel(const unsigned* __restrict__ ends, long long V, int vb_per_cta,
                     const unsigned* __restrict__ lin, unsigned* __restrict__ lout) {
  __shared__ __align__(16) unsigned s_lin[kRelCap + 4];
  extern __shared__ unsigned s_ends[];  // vb_per_cta + 1
  const long long v0 = (long long)blockIdx.x * vb_per_cta;
  const int nv = (int)(V - v0 < vb_per_cta ? V - v0 : vb_per_cta);
  for (int t = threadIdx.x; t <= nv; t += kRelThreads) {
    const long long v = v0 - 1 + t;
    s_ends[t] = v >= 0 ? ends[v] : 0u;
  }
  __syncthreads();
  const unsigned rb = s_ends[0], re = s_ends[nv];
  const bool staged = re - rb <= (unsigned)kRelCap;
  if (staged)
    for (unsigned i = rb + threadIdx.x; i < re; i += kRelThreads) s_lin[i - rb] = __ldcs(lin + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (!staged) {  // a crowded block: rank from global memory
    for (int t = warp; t < nv; t += kRelThreads / 32) {
      const unsigned b = s_ends[t], e = s_ends[t + 1];
      for (unsigned g = b; g < e; g += 32) {
        const unsigned i = g + lane;
        const unsigned my = i < e ? __ldg(lin + i) : 0u;
        unsigned rank = 0;
        for (unsigned j = b; j < e; ++j) rank += lt_bit(__ldg(lin + j), my);
        if (i < e) __stcs(lout + i, b + rank);
      }
    }
    return;
  }
  for (int t = warp; t < nv; t += kRelThreads / 32) {
    const unsigned b = s_ends[t], e = s_ends[t + 1];
    const unsigned lo = b - rb, hi = e - rb;
    if (hi == lo) continue;
    if (hi - lo <= 32u) {  // one record per lane (the common chunk)
      const unsigned i = lo + lane;
      const unsigned my[1] = {i < hi ? s_lin[i] : kBig};
      unsigned rank[1];
      warp_ranks<1>(my, rank, lane);
      if (i < hi) __stcs(lout + rb + i, b + rank[0]);
    } else if (hi - lo <= 64u) {  // two per lane
      const unsigned i0 = lo + lane, i1 = lo + 32u + lane;
      const unsigned my[2] = {s_lin[i0], i1 < hi ? s_lin[i1] : kBig};
      unsigned rank[2];
      warp_ranks<2>(my, rank, lane);
      __stcs(lout + rb + i0, b + rank[0]);
      if (i1 < hi) __stcs(lout + rb + i1, b + rank[1]);
    } else {  // all-pairs counts, one pass over the chunk per 64 records
      for (unsigned g = lo; g < hi; g += 64) {
        const unsigned i0 = g + lane, i1 = g + 32u + lane;
        const unsigned my[2] = {i0 < hi ? s_lin[i0] : 0u, i1 < hi ? s_lin[i1] : 0u};
        unsigned rank[2] = {0u, 0u};
        rank_cover<2>(s_lin, lo, hi, my, rank);
        if (i0 < hi) __stcs(lout + rb + i0, b + rank[0]);
        if (i1 < hi) __stcs(lout + rb + i1, b + rank[1]);
      }
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

// lout = the stable counting sort's logical indices of a store grouped in
// voxel chunks (chunk v ends at ends[v]; n records in all).
void relabel_chunks(Context& c, const unsigned* ends, long long n, const unsigned* lin, unsigned* lout) {
  const long long V = c.gc.V;
  if (c.relabel_variant == 1 || n >= (1ll << 31) - 1) {  // one warp per chunk (ablation; any n)
    const unsigned blocks = (unsigned)std::min<long long>((V + 7) / 8, (long long)c.num_sms * 16);
    relabel_kernel<<<blocks, 256, 0, c.stream>>>(ends, V, lin, lout);
  } else {
    // about 2048 records per CTA (a quarter of the staging buffer)
    const long long per_voxel = std::max<long long>(1, n / std::max<long long>(V, 1));
    const int vb = (int)std::min<long long>(1024, std::max<long long>(8, 2048 / per_voxel));
    const unsigned blocks = (unsigned)((V + vb - 1) / vb);
    relabel_tiled_kernel<<<blocks, kRelThreads, (vb + 1) * sizeof(unsigned), c.stream>>>(ends, V, vb, lin, lout);
  }
  c.count_launch();
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
      relabel_chunks(c, s.vcur, (long long)s.n, s.lidx, s.lidx_alt);
      std::swap(s.lidx, s.lidx_alt);
      s.relabel_pending = false;
    }
    s.since_reorder = 0;
  } else {
    ++s.since_reorder;
  }
  // a counting push counted its new voxels: chunk cursors ready for the
  // next reordering push
  if (counted) scan_voxel_counts(c, s);
  s.counts_ready = counted;
}

// The records of a voxel-ordered species in logical order into device
// buffers without leaving the order (the store, its chunks and logical
// indices stay as they are): false when that is not possible (not ordered,
// a relabel owed, a count on the device).
bool copy_logical(Context& c, Species& s, float4* pos, float4* mom) {
  if (!s.ordered || s.relabel_pending || s.perm_pending || s.n_on_device) return false;
  const long long n = (long long)s.n;
  if (n > 0) {
    to_logical_kernel<<<blocks_of(n), 256, 0, c.stream>>>(s.lidx, n, s.pos, s.mom, pos, mom);
    c.count_launch();
  }
  return true;
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
