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
// scatter in which every tile ranks its keys stably in registers (match.any
// digit groups + running per-warp counters + cross-warp prefix), stages them
// digit-sorted in shared memory and writes contiguous runs per digit at
// offset[digit][tile].  The first pass's histogram is taken while the keys
// are extracted from the records, and the last pass gathers the 32-byte
// particle records itself instead of writing a permutation.
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
// Tile = 4096 consecutive keys; warp w of the CTA owns keys [512w, 512w+512)
// and visits them in 16 coalesced rounds of 32, so (warp, round, lane) is the
// keys' original order and a running per-warp digit counter ranks them
// stably.  Lanes holding the same digit are grouped with match.any (a ballot
// per digit bit is the ablation: 23.0 vs 17.6 ms per 2^29-particle sort).
constexpr int kRankWarps = kThreads / 32;
constexpr int kRounds = kTile / kThreads;  // 16

template <int BITS>
__device__ __forceinline__ unsigned peers_of(unsigned d, unsigned valid_mask) {
  unsigned peers = valid_mask;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const unsigned bal = __ballot_sync(kFull, (d >> b) & 1u);
    peers &= ((d >> b) & 1u) ? bal : ~bal;
  }
  return peers;
}

// Per-tile digit counts of one pass, table[d * ntiles + tile].  No ranking
// is needed here, so each thread takes 16 consecutive keys (vector loads),
// merges runs of equal digits in registers (the input is always grouped by
// key to some degree: voxel runs of the sorted-then-aged store, or the
// previous pass's output) and adds one shared-memory atomic per run.
// FROM_POS: the keys are the voxel ids in pos[i].w (first pass), which are
// also written out as the key array the later passes read.
template <int BITS, bool FROM_POS>
__global__ void __launch_bounds__(kThreads)
radix_hist_kernel(const unsigned* __restrict__ keys, const float4* __restrict__ pos, size_t n, int shift,
                  size_t ntiles, unsigned* __restrict__ table, unsigned* __restrict__ keys_out) {
  constexpr int D = 1 << BITS;
  constexpr int kPer = kTile / kThreads;  // 16
  __shared__ unsigned h[D];
  for (int d = threadIdx.x; d < D; d += kThreads) h[d] = 0;
  const size_t tbase = (size_t)blockIdx.x * kTile;
  const size_t i0 = tbase + (size_t)threadIdx.x * kPer;
  unsigned key[kPer];
  const bool full = i0 + kPer <= n;
  if (FROM_POS) {
    // records read coalesced (a thread's 16 consecutive records would be 16
    // loads 256 B apart per warp instruction), keys written coalesced, then
    // transposed through shared memory into the per-thread runs
    __shared__ uint4 skeys[kTile / 4];
    unsigned* sk = reinterpret_cast<unsigned*>(skeys);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int j = k * kThreads + threadIdx.x;
      const size_t i = tbase + j;
      const unsigned kv = i < n ? (unsigned)__float_as_int(ld_stream(pos + i).w) : 0u;
      sk[j] = kv;
      if (i < n) keys_out[i] = kv;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer / 4; ++k) {
      const uint4 v = skeys[threadIdx.x * (kPer / 4) + k];
      key[4 * k] = v.x;
      key[4 * k + 1] = v.y;
      key[4 * k + 2] = v.z;
      key[4 * k + 3] = v.w;
    }
  } else if (full) {
    const uint4* in = reinterpret_cast<const uint4*>(keys + i0);
#pragma unroll
    for (int k = 0; k < kPer / 4; ++k) {
      const uint4 v = in[k];
      key[4 * k] = v.x;
      key[4 * k + 1] = v.y;
      key[4 * k + 2] = v.z;
      key[4 * k + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kPer; ++k) key[k] = i0 + k < n ? keys[i0 + k] : 0u;
  }
  __syncthreads();
  const int nv = full ? kPer : (i0 < n ? (int)(n - i0) : 0);
  unsigned cur = (key[0] >> shift) & (D - 1), run = nv > 0 ? 1u : 0u;
#pragma unroll
  for (int k = 1; k < kPer; ++k) {
    if (k < nv) {
      const unsigned d = (key[k] >> shift) & (D - 1);
      if (d != cur) {
        atomicAdd(&h[cur], run);
        cur = d;
        run = 0;
      }
      ++run;
    }
  }
  if (run) atomicAdd(&h[cur], run);
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += kThreads) table[(size_t)d * ntiles + blockIdx.x] = h[d];
}

// One stable scatter pass.  offsets[d * ntiles + tile] = where the tile's
// first key with digit d goes.  Keys are ranked in registers, placed in a
// digit-sorted shared copy of the tile and written out in contiguous runs per
// digit.  VALS: 0 = the value is the key's index (first pass), 1 = load vals.
// GATHER: instead of (key, value) pairs write the 32-byte particle record
// the value indexes (the permute fused into the last pass).
// The first pass (values = indices) runs 4 CTAs per SM at 64 registers (a
// few spilled words): its loads are latency-bound, 3.20 vs 3.76 ms per 2^29
// keys; the later passes gain nothing from it (2.77 vs 2.82 ms) and keep 3.
template <int BITS, int VALS, bool GATHER, bool MATCH>
__global__ void __launch_bounds__(kThreads, VALS == 0 ? 4 : 3)
radix_scatter_kernel(const unsigned* __restrict__ keys, const unsigned* __restrict__ vals, size_t n, int shift,
                     size_t ntiles, const unsigned* __restrict__ offsets, unsigned* __restrict__ keys_out,
                     unsigned* __restrict__ vals_out, const float4* __restrict__ pos,
                     const float4* __restrict__ mom, float4* __restrict__ pos_out, float4* __restrict__ mom_out) {
  constexpr int D = 1 << BITS;
  __shared__ union {
    unsigned cnt[kRankWarps][D];
    struct {
      unsigned key[kTile];
      unsigned val[kTile];
    } s;
  } sm;
  __shared__ unsigned dstart[D];
  __shared__ unsigned goff[D];
  __shared__ unsigned wsum[kRankWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < D; d += kThreads) {
#pragma unroll
    for (int w = 0; w < kRankWarps; ++w) sm.cnt[w][d] = 0;
    goff[d] = offsets[(size_t)d * ntiles + blockIdx.x];
  }
  __syncthreads();
  const size_t tbase = (size_t)blockIdx.x * kTile;
  const int valid = n - tbase < (size_t)kTile ? (int)(n - tbase) : kTile;
  const int wbase = warp * (kTile / kRankWarps);
  unsigned key[kRounds], val[kRounds], rank[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int i = wbase + r * 32 + lane;
    key[r] = i < valid ? keys[tbase + i] : 0u;
    if (VALS == 0) val[r] = (unsigned)(tbase + i);
    else val[r] = i < valid ? vals[tbase + i] : 0u;
  }
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int i = wbase + r * 32 + lane;
    const unsigned vm = __ballot_sync(kFull, i < valid);
    const unsigned d = (key[r] >> shift) & (D - 1);
    const unsigned peers = MATCH ? (__match_any_sync(kFull, d) & vm) : peers_of<BITS>(d, vm);
    const int leader = __ffs(peers) - 1;
    unsigned old = 0;
    if (i < valid && lane == leader) {
      old = sm.cnt[warp][d];
      sm.cnt[warp][d] = old + __popc(peers);
    }
    old = __shfl_sync(kFull, old, leader < 0 ? 0 : leader);
    rank[r] = old + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over warps (in place) and the tile total,
  // then the tile-local digit starts (exclusive scan over digits; thread t
  // owns the D/kThreads consecutive digits from t*D/kThreads)
  constexpr int DPT = D / kThreads > 0 ? D / kThreads : 1;
  unsigned tot[DPT];
  unsigned tsum = 0;
#pragma unroll
  for (int k = 0; k < DPT; ++k) {
    const int d = threadIdx.x * DPT + k;
    unsigned run = 0;
    if (d < D) {
#pragma unroll
      for (int w = 0; w < kRankWarps; ++w) {
        const unsigned t = sm.cnt[w][d];
        sm.cnt[w][d] = run;
        run += t;
      }
    }
    tot[k] = run;
    tsum += run;
  }
  unsigned incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  unsigned pre = incl - tsum;
  for (int w = 0; w < warp; ++w) pre += wsum[w];
#pragma unroll
  for (int k = 0; k < DPT; ++k) {
    const int d = threadIdx.x * DPT + k;
    if (d < D) {
      dstart[d] = pre;
      goff[d] -= pre;  // from here on: global position = goff[d] + tile-sorted index
    }
    pre += tot[k];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const unsigned d = (key[r] >> shift) & (D - 1);
    rank[r] += dstart[d] + sm.cnt[warp][d];
  }
  __syncthreads();  // cnt is overwritten by the sorted copy below
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int i = wbase + r * 32 + lane;
    if (i < valid) {
      sm.s.key[rank[r]] = key[r];
      sm.s.val[rank[r]] = val[r];
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < valid; j += kThreads) {
    const unsigned k = sm.s.key[j];
    const unsigned d = (k >> shift) & (D - 1);
    const size_t p = (size_t)(goff[d] + (unsigned)j);
    const unsigned v = sm.s.val[j];
    if (GATHER) {
      st_stream(pos_out + p, pos[v]);
      st_stream(mom_out + p, mom[v]);
    } else {
      if (keys_out) keys_out[p] = k;
      vals_out[p] = v;
    }
  }
}

// ---- particle sort helpers ----------------------------------------------------
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

#ifdef PIC_ABLATIONS
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

#endif  // PIC_ABLATIONS
}  // namespace
#ifdef PIC_ABLATIONS

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


#endif  // PIC_ABLATIONS

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

// start[v] = first position of key v in a sorted key array (start[V] = n).
void key_run_starts(Context& c, const unsigned* skey, size_t n, size_t V, unsigned* start) {
  CUDA_OK(cudaMemsetAsync(start, 0, (V + 1) * 4, c.stream));
  if (n) {
    count_keys_kernel<<<blocks_for(n), 256, 0, c.stream>>>(skey, n, start);
    c.count_launch();
  }
  exclusive_scan_u32(c, start, start, V + 1);
}

void exclusive_scan_u32(Context& c, const unsigned* in, unsigned* out, size_t n) {
  if (n == 0) return;
  // partial sums of every level live back to back in one grow-only slot
  size_t need = 0;
  for (size_t t = (n + kTile - 1) / kTile; t > 1; t = (t + kTile - 1) / kTile) need += t;
  unsigned* partial = static_cast<unsigned*>(c.scratch_bytes(Context::kScrScan, (need + 1) * sizeof(unsigned)));
  scan_level(c, in, out, n, partial);
}

// One LSD pass: per-tile histogram (or the one the key extraction made),
// scan, ranked scatter.  kout == nullptr: only the values are written (the
// last pass of a species sort needs just the permutation).
template <int BITS>
static void radix_pass(Context& c, const unsigned* kin, const unsigned* vin, size_t n, int shift, size_t ntiles,
                       unsigned* table, bool hist_done, unsigned* kout, unsigned* vout) {
  if (!hist_done)
    radix_hist_kernel<BITS, false><<<(unsigned)ntiles, kThreads, 0, c.stream>>>(kin, nullptr, n, shift, ntiles,
                                                                                table, nullptr);
  exclusive_scan_u32(c, table, table, ntiles << BITS);
  const bool m = c.sort_match != 0;
#define PIC_SCATTER(V, M)                                                                                        \
  radix_scatter_kernel<BITS, V, false, M><<<(unsigned)ntiles, kThreads, 0, c.stream>>>(                         \
      kin, vin, n, shift, ntiles, table, kout, vout, nullptr, nullptr, nullptr, nullptr)
  if (vin) {
    if (m) PIC_SCATTER(1, true); else PIC_SCATTER(1, false);
  } else {
    if (m) PIC_SCATTER(0, true); else PIC_SCATTER(0, false);
  }
#undef PIC_SCATTER
  c.count_launch(hist_done ? 1 : 2);
}

// digit widths of the passes: at most c.sort_radix_bits (8 or 9), evened out
static int pass_bits(const Context& c, int key_bits, int* passes) {
  const int maxb = std::min(std::max(c.sort_radix_bits, 1), kRadixBits);
  *passes = std::max(1, (key_bits + maxb - 1) / maxb);
  return (key_bits + *passes - 1) / *passes;
}

static void radix_pass_bits(Context& c, int bits, const unsigned* kin, const unsigned* vin, size_t n, int shift,
                            size_t ntiles, unsigned* table, bool hist_done, unsigned* kout, unsigned* vout) {
  switch (bits) {
    case 9: radix_pass<9>(c, kin, vin, n, shift, ntiles, table, hist_done, kout, vout); break;
    case 8: radix_pass<8>(c, kin, vin, n, shift, ntiles, table, hist_done, kout, vout); break;
    case 7: radix_pass<7>(c, kin, vin, n, shift, ntiles, table, hist_done, kout, vout); break;
    case 6: radix_pass<6>(c, kin, vin, n, shift, ntiles, table, hist_done, kout, vout); break;
    case 5: radix_pass<5>(c, kin, vin, n, shift, ntiles, table, hist_done, kout, vout); break;
    case 4: radix_pass<4>(c, kin, vin, n, shift, ntiles, table, hist_done, kout, vout); break;
    case 3: radix_pass<3>(c, kin, vin, n, shift, ntiles, table, hist_done, kout, vout); break;
    case 2: radix_pass<2>(c, kin, vin, n, shift, ntiles, table, hist_done, kout, vout); break;
    default: radix_pass<1>(c, kin, vin, n, shift, ntiles, table, hist_done, kout, vout); break;
  }
}

// Stable LSD radix sort of (key, value) pairs; vals == nullptr means value =
// index.  first_hist: the first pass's per-tile histogram is already in the
// table.  keys_out == nullptr: the sorted keys are not wanted.
static void radix_sort_impl(Context& c, const unsigned* keys, const unsigned* vals, size_t n, int key_bits,
                            bool first_hist, unsigned** keys_out, unsigned** vals_out,
                            unsigned* last_vals = nullptr) {
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
  int passes = 0;
  const int step = pass_bits(c, key_bits, &passes);
  for (int p = 0, shift = 0; p < passes; ++p, shift += step) {
    const int bits = std::min(step, key_bits - shift);
    const bool last = p + 1 == passes;
    if (last && last_vals) vout = last_vals;  // the permutation straight into its own buffer
    radix_pass_bits(c, bits, kin, vin, n, shift, ntiles, table, p == 0 && first_hist,
                    (last && !keys_out) ? nullptr : kout, vout);
    kin = kout;
    vin = vout;
    kout = (kout == ka) ? kb : ka;
    vout = (vout == va) ? vb : va;
  }
  if (keys_out) *keys_out = const_cast<unsigned*>(kin);
  if (vals_out) *vals_out = const_cast<unsigned*>(vin);
}

void radix_sort_pairs(Context& c, const unsigned* keys, const unsigned* vals, size_t n, int key_bits,
                      unsigned** keys_out, unsigned** vals_out) {
  radix_sort_impl(c, keys, vals, n, key_bits, false, keys_out, vals_out);
}

void materialize(Context& c, Species& s) {
  leave_voxel_order(c, s);  // continuous voxel order -> logical order (+ an owed sort)
  if (!s.perm_pending) return;
  s.perm_pending = false;
  if (s.n == 0) return;
  permute_kernel<<<blocks_for(s.n), 256, 0, c.stream>>>(s.perm, s.n, s.pos, s.mom, s.pos_alt, s.mom_alt);
  c.count_launch();
  std::swap(s.pos, s.pos_alt);
  std::swap(s.mom, s.mom_alt);
}

void materialize_all(Context& c) {
  for (auto& s : c.species) {
    settle_count(c, s);
    materialize(c, s);
  }
}
// Order-free reads (charge deposit, energy sums): a species in continuous
// voxel order is read where it lies (its n records are all valid); only a
// deferred sort permutation is applied.
void materialize_for_sums(Context& c) {
  for (auto& s : c.species) {
    settle_count(c, s);
    if (!s.ordered) materialize(c, s);
  }
}

// sort_particles (particles.cpp:412-458).
void sort_species(Context& c, Species& s, int order) {
  if (c.physical_order && !s.ordered && order == PIC_SORT_BLOCKED) {
    // the decomposed fast path (dd.cu): the next push reorders the store by voxel
    s.resort_pending = true;
    return;
  }
  if (s.ordered && order == PIC_SORT_BLOCKED) {
    // owed to the next push, a reordering one: it groups the store by
    // exactly these voxels, so the stable counting sort becomes a
    // relabelling of the logical indices (order.cu)
    s.relabel_pending = true;
    return;
  }
  materialize(c, s);
  const size_t n = s.n;
  if (n == 0) return;
  if (!s.pos_alt) {
    CUDA_OK(cudaMalloc(&s.pos_alt, s.cap * sizeof(float4)));
    CUDA_OK(cudaMalloc(&s.mom_alt, s.cap * sizeof(float4)));
  }
#ifdef PIC_ABLATIONS
  if (order == PIC_SORT_BLOCKED && c.sort_variant == 1) {
    tiled_counting_sort(c, s);
    std::swap(s.pos, s.pos_alt);
    std::swap(s.mom, s.mom_alt);
    return;
  }
#endif
  const int kbits = key_bits_for(c.gc.V);
  // keys out of the records, fused with the first pass's tile histogram
  unsigned* keys = static_cast<unsigned*>(c.scratch_bytes(Context::kScrCount, n * 4));
  const size_t ntiles = (n + kTile - 1) / kTile;
  unsigned* table = static_cast<unsigned*>(c.scratch_bytes(Context::kScrHist, ntiles * kDigits * 4));
  int passes = 0;
  const int b0 = std::min(pass_bits(c, kbits, &passes), kbits);
  switch (b0) {
#define PIC_EXTRACT_HIST(B)                                                                                     \
  case B:                                                                                                       \
    radix_hist_kernel<B, true><<<(unsigned)ntiles, kThreads, 0, c.stream>>>(nullptr, s.pos, n, 0, ntiles, table, \
                                                                           keys);                               \
    break;
    PIC_EXTRACT_HIST(9)
    PIC_EXTRACT_HIST(8)
    PIC_EXTRACT_HIST(7)
    PIC_EXTRACT_HIST(6)
    PIC_EXTRACT_HIST(5)
    PIC_EXTRACT_HIST(4)
    PIC_EXTRACT_HIST(3)
    PIC_EXTRACT_HIST(2)
    default: PIC_EXTRACT_HIST(1)
#undef PIC_EXTRACT_HIST
  }
  c.count_launch();
  unsigned* perm = nullptr;
  if (order != PIC_SORT_INTERLEAVED && c.sort_defer) {
    // blocked order, deferred: the next push gathers through the permutation
    // (a separate gather pass reads and writes every record once more)
    if (!s.perm) CUDA_OK(cudaMalloc(&s.perm, s.cap * sizeof(unsigned)));
    radix_sort_impl(c, keys, nullptr, n, kbits, true, nullptr, nullptr, s.perm);
    s.perm_pending = true;
    return;
  }
  if (order != PIC_SORT_INTERLEAVED) {
    radix_sort_impl(c, keys, nullptr, n, kbits, true, nullptr, &perm);
  } else {
    unsigned* skey = nullptr;
    radix_sort_impl(c, keys, nullptr, n, kbits, true, &skey, &perm);
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
    radix_sort_impl(c, within, perm1, n, key_bits_for((long long)hmax + 1), false, nullptr, &perm);
  }
  // one gather of the 32-byte records in output order (coalesced on a
  // nearly sorted store; a gather fused into the last pass reads them in
  // that pass's order and measured 8.6 vs 5.9 ms per 2^29 particles)
  permute_kernel<<<blocks_for(n), 256, 0, c.stream>>>(perm, n, s.pos, s.mom, s.pos_alt, s.mom_alt);
  c.count_launch();
  std::swap(s.pos, s.pos_alt);
  std::swap(s.mom, s.mom_alt);
}

}  // namespace picb
