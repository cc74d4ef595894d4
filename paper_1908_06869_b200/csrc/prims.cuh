// Device-wide primitives written for this path: exclusive scan and a stable
// LSD radix sort of (u64 key, u32 value) pairs with digit skipping.
// Used for the rare-path reorderings (explicit-parent kernels, orphan and
// ambiguity lists, a10 name grouping) and for stage (b) sort_timeline.
#pragma once

#include "xsp_common.cuh"

namespace xsp {

// ---------------------------------------------------------------------------
// Small transfers (counts, flags, group descriptors) between device memory and
// pinned host memory, which is device-addressable under unified virtual
// addressing: one warp moves the words, so the transfer never waits on a copy
// engine behind bulk copies that other streams have queued (csrc/pipeline.cu
// streams the next chunk's columns while the current chunk computes).
static __global__ void k_xfer_words(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
// launches of k_xfer_words by this host thread (added to the API call's count)
inline thread_local uint64_t g_xfer_launches = 0;
// bytes: a multiple of 4, both pointers 4-byte aligned
inline void xfer_small(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  ++g_xfer_launches;
  const uint32_t n = static_cast<uint32_t>(bytes / 4);
  const uint32_t threads = n <= 32 ? 32 : 256;
  uint32_t blocks = (n + threads - 1) / threads;
  if (blocks > 64) blocks = 64;
  if (blocks == 0) blocks = 1;
  k_xfer_words<<<blocks, threads, 0, st>>>(static_cast<uint32_t*>(dst), static_cast<const uint32_t*>(src), n);
}

// ---------------------------------------------------------------------------
// Exclusive scan, reduce-then-scan (3 launches per level, recursive on the
// block sums). `total` (optional, device) receives the sum of all inputs.

constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem_warp, T* total) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < (blockDim.x >> 5) ? smem_warp[lane] : T(0);
    T s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= (uint32_t)o) s += y;
    }
    if (lane < (blockDim.x >> 5)) smem_warp[lane] = s - w;
    if (lane == (blockDim.x >> 5) - 1) smem_warp[32] = s;
  }
  __syncthreads();
  T res = smem_warp[warp] + x - v;
  if (total) *total = smem_warp[32];
  __syncthreads();
  return res;
}

template <typename Tin, typename T>
__global__ void k_scan_reduce(const Tin* __restrict__ in, uint64_t n, T* __restrict__ block_sums) {
  __shared__ T sm[33];
  uint64_t base = (uint64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  T s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j)
    if (base + j < n) s += (T)in[base + j];
  T tot;
  block_exclusive_scan<T>(s, sm, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

template <typename Tin, typename T>
__global__ void k_scan_down(const Tin* __restrict__ in, uint64_t n, const T* __restrict__ block_prefix,
                            T* __restrict__ out, T* __restrict__ total, uint64_t total_index) {
  __shared__ T sm[33];
  uint64_t base = (uint64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  T vals[kScanItems];
  T s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    vals[j] = (base + j < n) ? (T)in[base + j] : T(0);
    s += vals[j];
  }
  T tot;
  T run = block_exclusive_scan<T>(s, sm, &tot) + (block_prefix ? block_prefix[blockIdx.x] : T(0));
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (base + j < n) out[base + j] = run;
    run += vals[j];
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) total[total_index] = run;
}

// Scratch needed by exclusive_scan for n items (in elements of T).
inline uint64_t scan_scratch_elems(uint64_t n) {
  uint64_t s = 0;
  while (n > (uint64_t)kScanTile) {
    n = (n + kScanTile - 1) / kScanTile;
    s += n + 1;
  }
  return s + 1;
}

// out[i] = sum(in[0..i)); if total != nullptr, total[0] = sum(in). in may alias out.
template <typename Tin, typename T>
void exclusive_scan(const Tin* in, T* out, uint64_t n, T* scratch, T* total, cudaStream_t st,
                    uint64_t* launches) {
  if (n == 0) {
    if (total) cudaMemsetAsync(total, 0, sizeof(T), st);
    return;
  }
  unsigned nb = ceil_div(n, kScanTile);
  if (nb == 1) {
    k_scan_down<Tin, T><<<1, kScanBlock, 0, st>>>(in, n, nullptr, out, total, 0);
    ++*launches;
    return;
  }
  T* sums = scratch;
  k_scan_reduce<Tin, T><<<nb, kScanBlock, 0, st>>>(in, n, sums);
  ++*launches;
  exclusive_scan<T, T>(sums, sums, nb, scratch + nb + 1, (T*)nullptr, st, launches);
  k_scan_down<Tin, T><<<nb, kScanBlock, 0, st>>>(in, n, sums, out, total, 0);
  ++*launches;
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort of (u64 key, u32 value), 8-bit digits.

constexpr int kRsBlock = 256;
constexpr int kRsItems = 16;
constexpr int kRsTile = kRsBlock * kRsItems;

static __global__ void k_rs_bits(const uint64_t* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ and_or) {
  unsigned long long a = ~0ull, o = 0ull;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long k = keys[i];
    a &= k;
    o |= k;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    a &= __shfl_xor_sync(0xffffffffu, a, s);
    o |= __shfl_xor_sync(0xffffffffu, o, s);
  }
  if ((threadIdx.x & 31u) == 0) {
    atomicAnd(&and_or[0], a);
    atomicOr(&and_or[1], o);
  }
}

static __global__ void k_rs_hist(const uint64_t* __restrict__ keys, uint64_t n, int shift,
                          uint32_t* __restrict__ counts, uint32_t ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  uint64_t base = (uint64_t)blockIdx.x * kRsTile;
#pragma unroll 4
  for (int r = 0; r < kRsItems; ++r) {
    uint64_t i = base + (uint64_t)r * kRsBlock + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  counts[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

static __global__ void k_rs_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                             uint64_t* __restrict__ kout, uint32_t* __restrict__ vout, uint64_t n,
                             int shift, const uint32_t* __restrict__ offsets, uint32_t ntiles) {
  __shared__ uint32_t base[256];
  __shared__ uint32_t wcnt[kRsBlock / 32][256];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  base[tid] = offsets[(uint64_t)tid * ntiles + blockIdx.x];
#pragma unroll
  for (int w = 0; w < kRsBlock / 32; ++w) wcnt[w][tid] = 0;
  __syncthreads();
  uint64_t tbase = (uint64_t)blockIdx.x * kRsTile;
  for (int r = 0; r < kRsItems; ++r) {
    uint64_t i = tbase + (uint64_t)r * kRsBlock + tid;
    bool valid = i < n;
    uint64_t key = valid ? kin[i] : 0;
    uint32_t val = valid ? vin[i] : 0;
    uint32_t d = valid ? (uint32_t)((key >> shift) & 255u) : 0u;
    uint32_t mask = match8(d, __ballot_sync(0xffffffffu, valid));
    uint32_t rank = __popc(mask & lanemask_lt());
    uint32_t leader = __ffs(mask) - 1;
    if (valid && lane == leader) wcnt[warp][d] = __popc(mask);
    __syncthreads();
    if (valid) {
      uint32_t pos = base[d] + rank;
      for (uint32_t w = 0; w < warp; ++w) pos += wcnt[w][d];
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kRsBlock / 32; ++w) {
      tot += wcnt[w][tid];
      wcnt[w][tid] = 0;
    }
    base[tid] += tot;
    __syncthreads();
  }
}

struct RadixScratch {
  uint64_t* keys_alt;
  uint32_t* vals_alt;
  uint32_t* counts;      // 256 * ntiles
  uint32_t* scan_tmp;    // scan_scratch_elems(256*ntiles)
  unsigned long long* and_or;  // 2 (device)
  unsigned long long* and_or_host;  // 2 (pinned host)
};

inline uint64_t radix_counts_elems(uint64_t n) { return 256ull * ceil_div(n ? n : 1, kRsTile); }

// Sorts keys/vals in place (result ends in keys/vals). Bits outside [lo_bit, hi_bit)
// are ignored; digits that are constant over all keys are skipped (one
// synchronous 16-byte read-back decides which).
inline void radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t n, int lo_bit, int hi_bit,
                             const RadixScratch& s, cudaStream_t st, uint64_t* launches) {
  if (n <= 1) return;
  s.and_or_host[0] = ~0ull;
  s.and_or_host[1] = 0ull;
  xfer_small(s.and_or, s.and_or_host, 16, st);
  unsigned g = ceil_div(n, 256);
  if (g > 1184) g = 1184;
  k_rs_bits<<<g, 256, 0, st>>>(keys, n, s.and_or);
  ++*launches;
  xfer_small(s.and_or_host, s.and_or, 16, st);
  cudaStreamSynchronize(st);
  const uint64_t varying = s.and_or_host[0] ^ s.and_or_host[1];
  const uint32_t ntiles = ceil_div(n, kRsTile);
  uint64_t* kin = keys;
  uint32_t* vin = vals;
  uint64_t* kout = s.keys_alt;
  uint32_t* vout = s.vals_alt;
  for (int shift = lo_bit; shift < hi_bit; shift += 8) {
    uint64_t dmask = (shift + 8 >= 64) ? (~0ull << shift) : (((1ull << 8) - 1) << shift);
    if (!(varying & dmask)) continue;
    k_rs_hist<<<ntiles, kRsBlock, 0, st>>>(kin, n, shift, s.counts, ntiles);
    exclusive_scan<uint32_t, uint32_t>(s.counts, s.counts, 256ull * ntiles, s.scan_tmp,
                                       (uint32_t*)nullptr, st, launches);
    k_rs_scatter<<<ntiles, kRsBlock, 0, st>>>(kin, vin, kout, vout, n, shift, s.counts, ntiles);
    launches[0] += 2;
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  if (kin != keys) {
    cudaMemcpyAsync(keys, kin, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(vals, vin, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
  }
}


// trimmed_mean (analysis.cpp:28-39) of any number of samples without storing
// them: the distinct values are visited in ascending order by repeated minimum
// selection (each(fn) calls fn(x) for every sample, in any order), and the ranks
// [drop, n - drop) are summed left to right exactly as the reference sums its
// sorted vector. O(n * distinct) loads: the path for groups with more runs than
// the register sorting networks hold (kept warp-uniform when `each` is).
template <typename Each>
__device__ __forceinline__ double trimmed_mean_select(Each each, uint32_t n, double f) {
  const uint32_t drop = (uint32_t)floor(f * (double)n);
  double s = 0.0, cur = 0.0;
  bool first = true;
  uint32_t pos = 0;
  while (pos < n) {
    double v = 0.0;
    bool found = false;
    each([&](double x) {
      if ((first || x > cur) && (!found || x < v)) {
        v = x;
        found = true;
      }
    });
    if (!found) break;  // unordered samples (NaN): nothing left to rank
    uint32_t c = 0;
    each([&](double x) { c += x == v; });
    for (uint32_t k = pos; k < pos + c; ++k)
      if (k >= drop && k < n - drop) s = __dadd_rn(s, v);
    cur = v;
    first = false;
    pos += c;
  }
  return s / (double)(n - 2 * drop);
}

}  // namespace xsp
