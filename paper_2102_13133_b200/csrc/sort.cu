// sort_p for sm_100a: stable device sorts that reproduce the reference's
// counting-sort permutations exactly.
//
// Reference: sort_particles (proj/src/particles.cpp:412-458).
//   blocked     = stable counting sort by voxel id;
//   interleaved = then a stable counting sort of that sequence by the
//                 particle's rank within its voxel run.
// Both are stable sorts by an integer key, so a stable LSD radix sort over
// (key, original index) pairs yields the identical permutation.  Each pass is
// the classic reduce-then-scan split: per-tile digit histograms, one
// device-wide exclusive scan over the digit-major (digit, tile) table, and a
// scatter in which every tile ranks its keys stably (warp match_any +
// cross-warp prefix in shared memory) and writes them at
// offset[digit][tile] + local rank.  The 32-byte particle records are then
// permuted once with a gather.
#include <algorithm>

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "pic_device.cuh"
#include "pic_internal.hpp"

namespace picb {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 keys per tile
constexpr int kRadixBits = 9;  // largest digit width the kernels support (Context::sort_radix_bits picks)
constexpr int kDigits = 1 << kRadixBits;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- exclusive scan (uint32), reduce-then-scan --------------------------------
__global__ void __launch_bounds__(kThreads) scan_reduce_kernel(const unsigned* __restrict__ in, size_t n,
                                                               unsigned* __restrict__ partial) {
  __shared__ unsigned s[kWarps];
  const size_t base = (size_t)blockIdx.x * kTile;
  unsigned sum = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const size_t i = base + (size_t)r * kThreads + threadIdx.x;
    if (i < n) sum += in[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < kWarps; ++w) t += s[w];
    partial[blockIdx.x] = t;
  }
}

// Exclusive scan of one tile (blocked per thread: thread t owns items
// [t*kItems, (t+1)*kItems)), plus a per-tile carry-in.
__global__ void __launch_bounds__(kThreads) scan_tile_kernel(const unsigned* __restrict__ in, size_t n,
                                                             const unsigned* __restrict__ carry,
                                                             unsigned* __restrict__ out) {
  __shared__ unsigned s[kWarps];
  const size_t base = (size_t)blockIdx.x * kTile + (size_t)threadIdx.x * kItems;
  unsigned x[kItems];
  unsigned tsum = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const size_t i = base + k;
    x[k] = i < n ? in[i] : 0u;
    tsum += x[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s[warp] = incl;
  __syncthreads();
  unsigned wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += s[w];
  unsigned run = (carry ? carry[blockIdx.x] : 0u) + wpre + incl - tsum;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const size_t i = base + k;
    if (i < n) out[i] = run;
    run += x[k];
  }
}

// ---- radix passes -------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
radix_hist_kernel(const unsigned* __restrict__ keys, size_t n, int shift, unsigned mask,
                  size_t ntiles, unsigned* __restrict__ table) {
  __shared__ unsigned h[kDigits];
  const int ndig = (int)mask + 1;  // digits of this pass (<= kDigits)
  for (int d = threadIdx.x; d < ndig; d += kThreads) h[d] = 0;
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * kTile;
  const int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int r = 0; r < kItems; ++r) {
    const size_t i = base + (size_t)r * kThreads + threadIdx.x;
    const int d = i < n ? (int)((keys[i] >> shift) & mask) : -1;
    const unsigned peers = __match_any_sync(kFull, d);
    if (d >= 0 && (peers & lanemask_lt()) == 0) atomicAdd(&h[d], (unsigned)__popc(peers));
    (void)lane;
  }
  __syncthreads();
  for (int d = threadIdx.x; d <= (int)mask; d += kThreads) table[(size_t)d * ntiles + blockIdx.x] = h[d];
}

__global__ void __launch_bounds__(kThreads)
radix_scatter_kernel(const unsigned* __restrict__ keys, const unsigned* __restrict__ vals, size_t n,
                     int shift, unsigned mask, size_t ntiles, const unsigned* __restrict__ offsets,
                     unsigned* __restrict__ keys_out, unsigned* __restrict__ vals_out) {
  __shared__ unsigned cnt[kWarps][kDigits];
  __shared__ unsigned base_d[kDigits];
  __shared__ unsigned goff[kDigits];
  const int ndig = (int)mask + 1;  // digits of this pass (<= kDigits)
  for (int d = threadIdx.x; d < ndig; d += kThreads) {
    base_d[d] = 0;
    goff[d] = offsets[(size_t)d * ntiles + blockIdx.x];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t tbase = (size_t)blockIdx.x * kTile;
  for (int r = 0; r < kItems; ++r) {
    for (int d = threadIdx.x; d < ndig; d += kThreads)
#pragma unroll
      for (int w = 0; w < kWarps; ++w) cnt[w][d] = 0;
    __syncthreads();
    const size_t i = tbase + (size_t)r * kThreads + threadIdx.x;
    const bool valid = i < n;
    const unsigned key = valid ? keys[i] : 0u;
    const unsigned val = valid ? (vals ? vals[i] : (unsigned)i) : 0u;
    const int d = valid ? (int)((key >> shift) & mask) : -1;
    const unsigned peers = __match_any_sync(kFull, d);
    const unsigned rank = __popc(peers & lanemask_lt());
    if (valid && rank == 0) cnt[warp][d] = __popc(peers);
    __syncthreads();
    for (int dd = threadIdx.x; dd < ndig; dd += kThreads) {
      unsigned run = base_d[dd];
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const unsigned t = cnt[w][dd];
        cnt[w][dd] = run;
        run += t;
      }
      base_d[dd] = run;
    }
    __syncthreads();
    if (valid) {
      const unsigned p = goff[d] + cnt[warp][d] + rank;
      keys_out[p] = key;
      vals_out[p] = val;
    }
    __syncthreads();
  }
  (void)lane;
}

// ---- particle sort helpers ----------------------------------------------------
__global__ void extract_keys_kernel(const float4* __restrict__ pos, size_t n, unsigned* __restrict__ keys) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = (unsigned)__float_as_int(pos[i].w);
}
__global__ void count_keys_kernel(const unsigned* __restrict__ keys, size_t n, unsigned* __restrict__ count) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int k = i < n ? (int)keys[i] : -1;
  const unsigned peers = __match_any_sync(kFull, k);
  if (k >= 0 && (peers & lanemask_lt()) == 0) atomicAdd(&count[k], (unsigned)__popc(peers));
}
// rank within the voxel run of the blocked order: within[j] = j - start[key[j]]
__global__ void within_kernel(const unsigned* __restrict__ skeys, size_t n, const unsigned* __restrict__ start,
                              unsigned* __restrict__ within) {
  const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) within[j] = (unsigned)j - start[skeys[j]];
}
__global__ void max_kernel(const unsigned* __restrict__ x, size_t n, unsigned* __restrict__ out) {
  unsigned m = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = max(m, x[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
__global__ void permute_kernel(const unsigned* __restrict__ perm, size_t n, const float4* __restrict__ pos,
                               const float4* __restrict__ mom, float4* __restrict__ pos_out,
                               float4* __restrict__ mom_out) {
  const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const unsigned p = perm[j];
  st_stream(pos_out + j, pos[p]);
  st_stream(mom_out + j, mom[p]);
}

inline unsigned blocks_for(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// ---- tiled stable counting sort (blocked order) ---------------------------------
// The stable counting sort of sort_particles (particles.cpp:419-433) split in
// tiles of kCT consecutive particles: (A) each tile sorts its keys stably in
// shared memory and run-length encodes them into (voxel, count) runs; (B-D)
// the runs of all tiles — about one per (tile, voxel) on a sorted-ish store,
// ~1/30 of the particles — are sorted stably by voxel and scanned, giving
// every run its global offset (tile order within a voxel = original order);
// (E) each tile scatters its records to offset + rank in run.  Bit-identical
// permutation to the reference, with ~90 B of traffic per particle instead
// of the ~140 B of the LSD radix sort over (key, index) pairs — but the
// in-tile block sort is compute-bound and the run count grows with the
// store's staleness, so it only wins on freshly sorted stores (measured on
// B200: 16.9 vs 22.3 ms fresh, 28-29 vs 22.7 ms 20 steps after a sort, per
// 2^29 particles).  Kept as sort variant 1 (ablation).
constexpr int kCThreads = 256, kCItems = 16, kCT = kCThreads * kCItems;  // 4096 particles per tile

__global__ void __launch_bounds__(kCThreads)
tile_runs_kernel(const float4* __restrict__ pos, size_t n, int key_bits, unsigned* __restrict__ meta,
                 unsigned* __restrict__ run_key, unsigned* __restrict__ run_cs, unsigned* __restrict__ nruns) {
  using BRS = cub::BlockRadixSort<unsigned, kCThreads, kCItems, unsigned short>;
  using BScan = cub::BlockScan<unsigned, kCThreads>;
  __shared__ union {
    typename BRS::TempStorage sort;
    typename BScan::TempStorage scan;
  } tmp;
  __shared__ unsigned last_key[kCThreads];
  const size_t tbase = (size_t)blockIdx.x * kCT;
  const int t = threadIdx.x;
  unsigned key[kCItems];
  unsigned short idx[kCItems];
#pragma unroll
  for (int k = 0; k < kCItems; ++k) {
    const int li = t * kCItems + k;  // blocked: rank order = original order
    const size_t gi = tbase + li;
    key[k] = gi < n ? (unsigned)__float_as_int(pos[gi].w) : 0xffffffffu;
    idx[k] = (unsigned short)li;
  }
  BRS(tmp.sort).Sort(key, idx, 0, key_bits < 32 ? key_bits + 1 : 32);  // +1 bit: padding keys sort last
  __syncthreads();
  last_key[t] = key[kCItems - 1];
  __syncthreads();
  unsigned prev = t > 0 ? last_key[t - 1] : 0xfffffffeu;
  unsigned flags = 0, nflag = 0;
#pragma unroll
  for (int k = 0; k < kCItems; ++k) {
    const bool f = key[k] != prev && key[k] != 0xffffffffu;
    flags |= (f ? 1u : 0u) << k;
    nflag += f;
    prev = key[k];
  }
  unsigned run0 = 0, total = 0;
  BScan(tmp.scan).ExclusiveSum(nflag, run0, total);
  // run id of each item (the run containing it = last flag at or before it)
  int run = (int)run0 - 1;
  const int tpos = t * kCItems;
#pragma unroll
  for (int k = 0; k < kCItems; ++k) {
    const bool f = (flags >> k) & 1u;
    if (f) {
      ++run;
      run_key[tbase + run] = key[k];
      run_cs[tbase + run] = (unsigned)(tpos + k);  // start position; count added below
    }
    if (key[k] != 0xffffffffu) meta[tbase + tpos + k] = ((unsigned)idx[k] << 12) | (unsigned)run;
  }
  if (t == 0) nruns[blockIdx.x] = total;
  __syncthreads();
  // counts: next run's start (or the tile's valid length) minus this start
  const size_t valid = n - tbase < (size_t)kCT ? n - tbase : (size_t)kCT;
  for (unsigned r = t; r < total; r += kCThreads) {
    const unsigned st = run_cs[tbase + r] & 4095u;
    const unsigned en = r + 1 < total ? (run_cs[tbase + r + 1] & 4095u) : (unsigned)valid;
    run_cs[tbase + r] = ((en - st) << 12) | st;
  }
}

__global__ void compact_runs_kernel(const unsigned* __restrict__ run_key, const unsigned* __restrict__ run_cs,
                                    const unsigned* __restrict__ nruns, const unsigned* __restrict__ runoff,
                                    unsigned* __restrict__ dkey, unsigned* __restrict__ did) {
  const size_t tile = blockIdx.x;
  const unsigned nr = nruns[tile], o = runoff[tile];
  for (unsigned r = threadIdx.x; r < nr; r += blockDim.x) {
    dkey[o + r] = run_key[tile * kCT + r];
    did[o + r] = o + r;
  }
  (void)run_cs;
}

// dense run id -> (tile, local run) is recovered from runoff by binary search
__device__ __forceinline__ unsigned tile_of_run(const unsigned* __restrict__ runoff, unsigned ntiles, unsigned id) {
  unsigned lo = 0, hi = ntiles;  // largest tile with runoff[tile] <= id
  while (hi - lo > 1) {
    const unsigned mid = (lo + hi) >> 1;
    if (runoff[mid] <= id) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void run_counts_sorted_kernel(const unsigned* __restrict__ sid, size_t R,
                                         const unsigned* __restrict__ runoff, unsigned ntiles,
                                         const unsigned* __restrict__ run_cs, unsigned* __restrict__ cnt_sorted) {
  const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= R) return;
  const unsigned id = sid[j];
  const unsigned tile = tile_of_run(runoff, ntiles, id);
  cnt_sorted[j] = run_cs[(size_t)tile * kCT + (id - runoff[tile])] >> 12;
}

__global__ void scatter_offsets_kernel(const unsigned* __restrict__ sid, size_t R,
                                       const unsigned* __restrict__ off_sorted, unsigned* __restrict__ off_by_run) {
  const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < R) off_by_run[sid[j]] = off_sorted[j];
}

__global__ void __launch_bounds__(kCThreads)
tile_scatter_kernel(const unsigned* __restrict__ meta, size_t n, const unsigned* __restrict__ run_cs,
                    const unsigned* __restrict__ runoff, const unsigned* __restrict__ off_by_run,
                    const float4* __restrict__ pos, const float4* __restrict__ mom, float4* __restrict__ pos_out,
                    float4* __restrict__ mom_out) {
  const size_t tbase = (size_t)blockIdx.x * kCT;
  const unsigned o = runoff[blockIdx.x];
  for (int i = threadIdx.x; i < kCT; i += kCThreads) {
    const size_t gi = tbase + i;
    if (gi >= n) break;
    const unsigned m = meta[gi];
    const unsigned run = m & 4095u, src = m >> 12;
    const unsigned st = run_cs[tbase + run] & 4095u;
    const size_t dst = (size_t)off_by_run[o + run] + (unsigned)i - st;
    st_stream(pos_out + dst, ld_stream(pos + tbase + src));
    st_stream(mom_out + dst, ld_stream(mom + tbase + src));
  }
}

}  // namespace

// Stable blocked sort of species s by voxel id into (pos_alt, mom_alt).
static void tiled_counting_sort(Context& c, Species& s) {
  const size_t n = s.n;
  const size_t ntiles = (n + kCT - 1) / kCT;
  const int kb = key_bits_for(c.gc.V);
  unsigned* meta = static_cast<unsigned*>(c.scratch_bytes(Context::kScrKeyA, ntiles * kCT * 4));
  unsigned* run_key = static_cast<unsigned*>(c.scratch_bytes(Context::kScrValA, ntiles * kCT * 4));
  unsigned* run_cs = static_cast<unsigned*>(c.scratch_bytes(Context::kScrKeyB, ntiles * kCT * 4));
  unsigned* nruns = static_cast<unsigned*>(c.scratch_bytes(Context::kScrHist, (ntiles + 1) * 4 * 2));
  unsigned* runoff = nruns + ntiles + 1;
  tile_runs_kernel<<<(unsigned)ntiles, kCThreads, 0, c.stream>>>(s.pos, n, kb, meta, run_key, run_cs, nruns);
  CUDA_OK(cudaMemsetAsync(nruns + ntiles, 0, 4, c.stream));
  exclusive_scan_u32(c, nruns, runoff, ntiles + 1);
  unsigned R = 0;
  CUDA_OK(cudaMemcpyAsync(&R, runoff + ntiles, 4, cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
  // dense runs -> stable sort by voxel -> offsets
  unsigned* dense = static_cast<unsigned*>(c.scratch_bytes(Context::kScrValB, (size_t)R * 4 * 6 + 64));
  unsigned *dkey = dense, *did = dense + R, *skey = dense + 2 * (size_t)R, *sid = dense + 3 * (size_t)R;
  unsigned *cnt = dense + 4 * (size_t)R, *off = dense + 5 * (size_t)R;
  compact_runs_kernel<<<(unsigned)ntiles, 256, 0, c.stream>>>(run_key, run_cs, nruns, runoff, dkey, did);
  size_t tb = 0;
  CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dkey, skey, did, sid, (int)R, 0, kb, c.stream));
  size_t tb2 = 0;
  CUDA_OK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt, off, (int)R, c.stream));
  void* tmp = c.scratch_bytes(Context::kScrWithin, std::max(tb, tb2) + 256);
  tb = std::max(tb, tb2);
  size_t t1 = tb;
  CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp, t1, dkey, skey, did, sid, (int)R, 0, kb, c.stream));
  run_counts_sorted_kernel<<<blocks_for(R), 256, 0, c.stream>>>(sid, R, runoff, (unsigned)ntiles, run_cs, cnt);
  t1 = tb;
  CUDA_OK(cub::DeviceScan::ExclusiveSum(tmp, t1, cnt, off, (int)R, c.stream));
  // off_by_run reuses dkey (free after the sort)
  scatter_offsets_kernel<<<blocks_for(R), 256, 0, c.stream>>>(sid, R, off, dkey);
  tile_scatter_kernel<<<(unsigned)ntiles, kCThreads, 0, c.stream>>>(meta, n, run_cs, runoff, dkey, s.pos, s.mom,
                                                                     s.pos_alt, s.mom_alt);
  c.count_launch(8);
}


int key_bits_for(long long max_key_exclusive) {
  int b = 1;
  while (b < 32 && (1LL << b) < max_key_exclusive) ++b;
  return b;
}

static void scan_level(Context& c, const unsigned* in, unsigned* out, size_t n, unsigned* partial) {
  const size_t tiles = (n + kTile - 1) / kTile;
  if (tiles == 1) {
    scan_tile_kernel<<<1, kThreads, 0, c.stream>>>(in, n, nullptr, out);
    c.count_launch();
    return;
  }
  scan_reduce_kernel<<<(unsigned)tiles, kThreads, 0, c.stream>>>(in, n, partial);
  c.count_launch();
  scan_level(c, partial, partial, tiles, partial + tiles);  // next level after this one
  scan_tile_kernel<<<(unsigned)tiles, kThreads, 0, c.stream>>>(in, n, partial, out);
  c.count_launch();
}

void exclusive_scan_u32(Context& c, const unsigned* in, unsigned* out, size_t n) {
  if (n == 0) return;
  // partial sums of every level live back to back in one grow-only slot
  size_t need = 0;
  for (size_t t = (n + kTile - 1) / kTile; t > 1; t = (t + kTile - 1) / kTile) need += t;
  unsigned* partial = static_cast<unsigned*>(c.scratch_bytes(Context::kScrScan, (need + 1) * sizeof(unsigned)));
  scan_level(c, in, out, n, partial);
}

void radix_sort_pairs(Context& c, const unsigned* keys, const unsigned* vals, size_t n, int key_bits,
                      unsigned** keys_out, unsigned** vals_out) {
  unsigned* ka = static_cast<unsigned*>(c.scratch_bytes(Context::kScrKeyA, n * 4));
  unsigned* va = static_cast<unsigned*>(c.scratch_bytes(Context::kScrValA, n * 4));
  unsigned* kb = static_cast<unsigned*>(c.scratch_bytes(Context::kScrKeyB, n * 4));
  unsigned* vb = static_cast<unsigned*>(c.scratch_bytes(Context::kScrValB, n * 4));
  const size_t ntiles = (n + kTile - 1) / kTile;
  unsigned* table = static_cast<unsigned*>(c.scratch_bytes(Context::kScrHist, ntiles * kDigits * 4));
  const unsigned* kin = keys;
  const unsigned* vin = vals;
  unsigned* kout = ka;
  unsigned* vout = va;
  // digit width: c.sort_radix_bits (<= kRadixBits), evened out over the passes
  const int maxb = std::min(std::max(c.sort_radix_bits, 1), kRadixBits);
  const int passes = (key_bits + maxb - 1) / maxb;
  const int step = (key_bits + passes - 1) / passes;
  for (int shift = 0; shift < key_bits; shift += step) {
    const int bits = key_bits - shift < step ? key_bits - shift : step;
    const unsigned mask = (1u << bits) - 1u;
    const size_t entries = ntiles * ((size_t)mask + 1);
    radix_hist_kernel<<<(unsigned)ntiles, kThreads, 0, c.stream>>>(kin, n, shift, mask, ntiles, table);
    exclusive_scan_u32(c, table, table, entries);
    radix_scatter_kernel<<<(unsigned)ntiles, kThreads, 0, c.stream>>>(kin, vin, n, shift, mask, ntiles, table,
                                                                      kout, vout);
    c.count_launch(2);
    kin = kout;
    vin = vout;
    kout = (kout == ka) ? kb : ka;
    vout = (vout == va) ? vb : va;
  }
  *keys_out = const_cast<unsigned*>(kin);
  *vals_out = const_cast<unsigned*>(vin);
}

// sort_particles (particles.cpp:412-458).
void sort_species(Context& c, Species& s, int order) {
  const size_t n = s.n;
  if (n == 0) return;
  if (!s.pos_alt) {
    CUDA_OK(cudaMalloc(&s.pos_alt, s.cap * sizeof(float4)));
    CUDA_OK(cudaMalloc(&s.mom_alt, s.cap * sizeof(float4)));
  }
  if (order == PIC_SORT_BLOCKED && c.sort_variant == 1) {
    tiled_counting_sort(c, s);
    std::swap(s.pos, s.pos_alt);
    std::swap(s.mom, s.mom_alt);
    return;
  }
  unsigned* keys = static_cast<unsigned*>(c.scratch_bytes(Context::kScrCount, n * 4));
  extract_keys_kernel<<<blocks_for(n), 256, 0, c.stream>>>(s.pos, n, keys);
  c.count_launch();
  unsigned *skey = nullptr, *perm = nullptr;
  radix_sort_pairs(c, keys, nullptr, n, key_bits_for(c.gc.V), &skey, &perm);
  if (order == PIC_SORT_INTERLEAVED) {
    // within-voxel rank of every slot of the blocked order
    const size_t V = (size_t)c.gc.V;
    unsigned* cnt = static_cast<unsigned*>(c.scratch_bytes(Context::kScrStart, (V + 1) * 4));
    CUDA_OK(cudaMemsetAsync(cnt, 0, (V + 1) * 4, c.stream));
    count_keys_kernel<<<blocks_for(n), 256, 0, c.stream>>>(skey, n, cnt);
    exclusive_scan_u32(c, cnt, cnt, V + 1);
    // skey / perm live in the radix scratch; move them aside before the
    // second sort reuses it.
    unsigned* within = static_cast<unsigned*>(c.scratch_bytes(Context::kScrWithin, n * 4));
    within_kernel<<<blocks_for(n), 256, 0, c.stream>>>(skey, n, cnt, within);
    unsigned* perm1 = static_cast<unsigned*>(c.scratch_bytes(Context::kScrCount, n * 4));
    CUDA_OK(cudaMemcpyAsync(perm1, perm, n * 4, cudaMemcpyDeviceToDevice, c.stream));
    unsigned* dmax = static_cast<unsigned*>(c.scratch_bytes(Context::kScrSmall, 64));
    CUDA_OK(cudaMemsetAsync(dmax, 0, 4, c.stream));
    max_kernel<<<592, 256, 0, c.stream>>>(within, n, dmax);
    c.count_launch(3);
    unsigned hmax = 0;
    CUDA_OK(cudaMemcpyAsync(&hmax, dmax, 4, cudaMemcpyDeviceToHost, c.stream));
    CUDA_OK(cudaStreamSynchronize(c.stream));
    unsigned* skey2 = nullptr;
    radix_sort_pairs(c, within, perm1, n, key_bits_for((long long)hmax + 1), &skey2, &perm);
  }
  permute_kernel<<<blocks_for(n), 256, 0, c.stream>>>(perm, n, s.pos, s.mom, s.pos_alt, s.mom_alt);
  c.count_launch();
  std::swap(s.pos, s.pos_alt);
  std::swap(s.mom, s.mom_alt);
}

}  // namespace picb
