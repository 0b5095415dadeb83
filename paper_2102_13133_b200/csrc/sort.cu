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
#include "pic_device.cuh"
#include "pic_internal.hpp"

namespace picb {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 keys per tile
constexpr int kRadixBits = 8;
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
  for (int d = threadIdx.x; d < kDigits; d += kThreads) h[d] = 0;
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
  for (int d = threadIdx.x; d < kDigits; d += kThreads) {
    base_d[d] = 0;
    goff[d] = d <= (int)mask ? offsets[(size_t)d * ntiles + blockIdx.x] : 0u;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t tbase = (size_t)blockIdx.x * kTile;
  for (int r = 0; r < kItems; ++r) {
    for (int d = threadIdx.x; d < kDigits; d += kThreads)
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
    for (int dd = threadIdx.x; dd < kDigits; dd += kThreads) {
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

}  // namespace

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
  for (int shift = 0; shift < key_bits; shift += kRadixBits) {
    const int bits = key_bits - shift < kRadixBits ? key_bits - shift : kRadixBits;
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
