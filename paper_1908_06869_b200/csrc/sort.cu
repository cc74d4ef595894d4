// Stage (b): sort_timeline (span.cpp:112-127) on the device — a stable sort of
// every trace's spans by (begin_ns, rank(level), span_id).
//
// Presorted input (the TraceBundle invariant) is detected first (k_sort_check)
// and returns the identity without sorting. Otherwise every trace of up to
// kSegCap spans is sorted by ONE CTA in shared memory (k_sort_merge): the
// trace's begin / span_id ranges are reduced, each span gets a unique packed
// 64-bit key (begin - min, rank, span_id - min, local index), the thread-local
// runs are sorted in registers and merged by merge path in shared memory.
// Three size classes (4 K / 8 K / 16 K spans) keep 6 / 3 / 1 CTAs per SM
// (256 / 512 / 1024 threads, 16 keys per thread).
// HBM traffic is one read of begin/span_id/flags and one perm write (21 B/span).
// Traces that are longer, or whose begin range alone needs more than 47 bits,
// fall back to one global LSD radix sort over the composite key (trace,
// begin_ns, rank, span_id): four stable passes from the least significant
// field, each skipping the 8-bit digits that are constant over the batch.

#include "ctx.h"
#include "prims.cuh"

namespace xsp {

namespace {

// Timeline-order check fused with the identity permutation. Every block owns a
// contiguous run of 1024-span chunks; per chunk it marks the trace heads in a
// shared bitmap (walking the trace offsets forward from the previous chunk, so
// no per-span trace lookup), then checks every pair (i-1, i) that is not a
// head: begin must not decrease, and equal begins are ordered by (rank,
// span_id). One barrier per chunk: the begin / flags / offset loads and the
// disorder flag are issued together, and the bitmaps and trace cursors are
// triple-buffered (chunk q clears the buffers of chunk q + 2, which chunk q + 1's
// barrier orders before their use). Once disorder has been found the remaining
// chunks are skipped.
constexpr int kCheckItems = 4;
constexpr uint32_t kCheckChunk = 256 * kCheckItems;
__global__ void __launch_bounds__(256) k_sort_check(const uint64_t* __restrict__ begin,
                                                    const uint8_t* __restrict__ flags,
                                                    const uint64_t* __restrict__ sid,
                                                    const uint64_t* __restrict__ off, uint32_t T, uint64_t n,
                                                    uint32_t* __restrict__ perm, uint32_t* __restrict__ unsorted) {
  __shared__ uint32_t s_head[3][kCheckChunk / 32];
  __shared__ uint32_t s_tn[3];  // last trace starting <= the chunk end
  __shared__ uint32_t s_t0;
  const uint32_t tid = threadIdx.x;
  const uint64_t nchunks = (n + kCheckChunk - 1) / kCheckChunk;
  const uint64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const uint64_t q0 = (uint64_t)blockIdx.x * per, q1 = min(nchunks, q0 + per);
  if (q0 >= q1) return;
  if (tid < 3 * kCheckChunk / 32) (&s_head[0][0])[tid] = 0;
  if (tid < 3) s_tn[tid] = 0;
  if (tid == 0) s_t0 = trace_of(off, 0, T, q0 * kCheckChunk);  // last trace starting <= the run start
  __syncthreads();
  uint32_t tcur = s_t0;
  for (uint64_t q = q0; q < q1; ++q) {
    const uint32_t buf = (uint32_t)(q % 3);
    uint32_t* head = s_head[buf];
    const uint64_t c0 = q * kCheckChunk, c1 = min(n, c0 + kCheckChunk);
    uint64_t b0[kCheckItems], b1[kCheckItems];
    uint32_t f01[kCheckItems];
#pragma unroll
    for (int k = 0; k < kCheckItems; ++k) {
      const uint64_t i = c0 + k * 256 + tid;
      const bool v = i > 0 && i < c1;
      b0[k] = v ? begin[i - 1] : 0;
      b1[k] = v ? begin[i] : 1;
      f01[k] = v ? (uint32_t)flags[i - 1] << 8 | flags[i] : 0;
      if (i < c1) perm[i] = (uint32_t)i;
    }
    const bool stop = tid == 0 && __ldcg(unsorted) != 0;
    // heads: traces starting in [c0, c1)
    uint64_t tb = tcur;
    bool more;
    for (;;) {
      const uint64_t tt = tb + tid;
      const uint64_t o = tt <= T ? off[tt] : ~0ull;
      if (o >= c0 && o < c1) atomicOr(&head[(uint32_t)(o - c0) >> 5], 1u << ((uint32_t)(o - c0) & 31u));
      if (o <= c1) atomicMax(&s_tn[buf], (uint32_t)tt);
      more = tid == 255 && o <= c1;
      if (__syncthreads_or(more || stop) == 0) break;
      if (__syncthreads_or(stop)) return;
      tb += 256;
    }
    tcur = max(tcur, s_tn[buf]);
    if (tid < kCheckChunk / 32) s_head[(q + 2) % 3][tid] = 0;
    if (tid == 0) s_tn[(q + 2) % 3] = 0;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < kCheckItems; ++k) {
      const uint32_t j = k * 256 + tid;
      const uint64_t i = c0 + j;
      if (b0[k] < b1[k] || ((head[j >> 5] >> (j & 31u)) & 1u)) continue;
      if (b0[k] > b1[k]) {
        bad = true;
        continue;
      }
      const uint32_t l0 = f_level((uint8_t)(f01[k] >> 8)), l1 = f_level((uint8_t)f01[k]);
      const uint32_t r0 = l0 >= 2 ? 3 : l0 + 1, r1 = l1 >= 2 ? 3 : l1 + 1;
      bad |= r0 > r1 || (r0 == r1 && sid[i - 1] > sid[i]);
    }
    if (bad) *unsorted = 1;
  }
}

__global__ void k_iota_u32(uint32_t* v, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}

// key[j] = field of the span currently at position j
__global__ void k_sort_key(int field, const uint32_t* __restrict__ val, const uint64_t* __restrict__ begin,
                           const uint8_t* __restrict__ flags, const uint64_t* __restrict__ sid,
                           const uint64_t* __restrict__ off, uint32_t T, uint64_t n, uint64_t* __restrict__ key) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t i = val[j];
  uint64_t k;
  switch (field) {
    case 0: k = sid[i]; break;
    case 1: {
      const uint32_t l = f_level(flags[i]);
      k = l >= 2 ? 3 : l + 1;
      break;
    }
    case 2: k = begin[i]; break;
    default: k = trace_of(off, 0, T, i); break;
  }
  key[j] = k;
}

constexpr uint32_t kSegCap = 16384;  // spans per CTA-sorted trace (large class)
constexpr uint32_t kSegCapSmall = 4096;  // small class: 4 CTAs per SM
constexpr uint32_t kSegCapMid = 8192;    // middle class: 2 CTAs per SM

__device__ __forceinline__ uint32_t bit_width64(uint64_t v) { return v ? 64 - __clzll(v) : 0; }

// ---- per-trace merge sort ----------------------------------------------------
// Keys are unique u64s: (begin - min) | rank | (span_id - min) | local index j
// (14 bits) when that fits 63 bits ("full" keys), else (begin - min) | rank | j
// and runs of equal (begin, rank) are ordered by span_id afterwards (stable:
// j ascends inside a run). Every thread sorts ITEMS keys in registers (Batcher's
// odd-even merge network), then log2(THREADS) merge-path rounds double the
// sorted runs in shared memory: a thread binary-searches where its ITEMS
// outputs start on the two runs' cross diagonal and merges them serially into
// registers. Only the keys of the trace (rounded up to ITEMS) take part, so
// the work follows the trace length, not the class capacity. The shared-memory
// layout pads one word per 16 so that a thread's ITEMS consecutive keys are
// stored and loaded without bank conflicts.
__device__ __forceinline__ uint32_t mpad(uint32_t p) { return p + (p >> 4); }

// Bitonic sorting network over a thread's registers (N a power of two; fixed
// loop bounds so that it unrolls completely and the array stays in registers).
template <int N>
__device__ __forceinline__ void sort_network(uint64_t (&a)[N]) {
#pragma unroll
  for (int k = 2; k <= N; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int l = i ^ j;
        if (l <= i) continue;
        const bool up = (i & k) == 0;
        const uint64_t x = a[i], y = a[l];
        const bool sw = up ? x > y : x < y;
        a[i] = sw ? y : x;
        a[l] = sw ? x : y;
      }
}

template <int THREADS, int ITEMS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_sort_merge(const uint64_t* __restrict__ begin,
                                                        const uint8_t* __restrict__ flags,
                                                        const uint64_t* __restrict__ sid,
                                                        const uint64_t* __restrict__ off, uint32_t min_len,
                                                        uint32_t* __restrict__ perm,
                                                        uint32_t* __restrict__ fallback) {
  constexpr uint32_t CAP = (uint32_t)THREADS * ITEMS;
  constexpr int kWarps = THREADS / 32;
  static_assert(CAP <= 16384, "local indices are packed in 14 bits");
  extern __shared__ __align__(16) unsigned long long mkeys[];  // [mpad(CAP)]
  __shared__ unsigned long long red[4][kWarps];
  __shared__ uint32_t s_mode, s_sh_r, s_sh_b;
  const uint32_t t = blockIdx.x, tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint64_t lo = off[t], hi = off[t + 1];
  const uint32_t len = (uint32_t)(hi - lo);
  if (len < min_len) return;  // a smaller class sorts it
  if (len <= 1) {
    if (len == 1 && tid == 0) perm[lo] = (uint32_t)lo;
    return;
  }
  if (len > CAP) {
    if (CAP < kSegCap) return;  // a larger class sorts it
    if (tid == 0) atomicOr(fallback, 1u);
    return;
  }
  // ranges of begin and span_id; begin is staged in the key buffer (the loads
  // of a thread's ITEMS spans are independent and issued together)
  uint64_t bmin = ~0ull, bmax = 0, smin = ~0ull, smax = 0;
#pragma unroll 8
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t j = tid + k * THREADS;
    if (j < len) {
      const uint64_t b = begin[lo + j], s = sid[lo + j];
      mkeys[mpad(j)] = b;
      bmin = min(bmin, b); bmax = max(bmax, b);
      smin = min(smin, s); smax = max(smax, s);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bmin = min(bmin, __shfl_xor_sync(0xffffffffu, bmin, o));
    bmax = max(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    smin = min(smin, __shfl_xor_sync(0xffffffffu, smin, o));
    smax = max(smax, __shfl_xor_sync(0xffffffffu, smax, o));
  }
  if (lane == 0) {
    red[0][warp] = bmin; red[1][warp] = bmax; red[2][warp] = smin; red[3][warp] = smax;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kWarps; ++w) {
      red[0][0] = min(red[0][0], red[0][w]); red[1][0] = max(red[1][0], red[1][w]);
      red[2][0] = min(red[2][0], red[2][w]); red[3][0] = max(red[3][0], red[3][w]);
    }
    const uint32_t sb = bit_width64(red[3][0] - red[2][0]);
    const uint32_t bb = bit_width64(red[1][0] - red[0][0]);
    // mode 0: full keys; 1: (begin, rank, j) + span_id fix-up of equal runs; 2: too wide
    s_mode = bb + 2 + sb + 14 <= 63 ? 0u : (bb + 2 + 14 <= 63 ? 1u : 2u);
    s_sh_r = (s_mode == 0 ? sb : 0) + 14;
    s_sh_b = s_sh_r + 2;
    if (s_mode == 2) atomicOr(fallback, 1u);
  }
  __syncthreads();
  const uint32_t mode = s_mode;
  if (mode == 2) return;
  bmin = red[0][0];
  smin = red[2][0];
  const uint32_t sh_r = s_sh_r, sh_b = s_sh_b;
  const uint32_t n_act = (len + ITEMS - 1) / ITEMS * ITEMS;  // keys taking part (sentinel-padded)
#pragma unroll 8
  for (int q = 0; q < ITEMS; ++q) {
    const uint32_t j = tid + q * THREADS;
    if (j >= n_act) continue;
    uint64_t k = ~0ull;
    if (j < len) {
      const uint32_t l = f_level(flags[lo + j]);
      const uint64_t r = l >= XSP_LEVEL_KERNEL ? 3 : l + 1;  // rank (span.hpp:51-59)
      k = ((mkeys[mpad(j)] - bmin) << sh_b) | (r << sh_r) | j;
      if (mode == 0) k |= (sid[lo + j] - smin) << 14;
    }
    mkeys[mpad(j)] = k;
  }
  __syncthreads();
  const uint32_t my0 = tid * ITEMS;
  const bool active = my0 < n_act;
  uint64_t v[ITEMS];
  if (active) {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) v[k] = mkeys[mpad(my0 + k)];
    sort_network(v);
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) mkeys[mpad(my0 + k)] = v[k];
  }
  for (uint32_t w = ITEMS; w < n_act; w <<= 1) {
    __syncthreads();
    if (active) {
      const uint32_t g0 = my0 / (2 * w) * (2 * w);
      const uint32_t a0 = g0, a1 = min(g0 + w, n_act), b1 = min(g0 + 2 * w, n_act);
      const uint32_t na = a1 - a0, nb = b1 - a1, d = my0 - g0;
      // merge path: i keys of A and d - i of B precede this thread's outputs
      uint32_t l = d > nb ? d - nb : 0, h = min(d, na);
      while (l < h) {
        const uint32_t m = (l + h) >> 1;
        if (mkeys[mpad(a0 + m)] < mkeys[mpad(a1 + d - 1 - m)]) l = m + 1; else h = m;
      }
      uint32_t ia = a0 + l, ib = a1 + (d - l);
      uint64_t xa = ia < a1 ? mkeys[mpad(ia)] : ~0ull, xb = ib < b1 ? mkeys[mpad(ib)] : ~0ull;
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        // branch-free step: one load from the side that advanced
        const bool ta = xa < xb;
        v[k] = ta ? xa : xb;
        ia += ta;
        ib += !ta;
        const uint32_t nx = ta ? ia : ib;
        const bool in = ta ? ia < a1 : ib < b1;
        const uint64_t y = in ? mkeys[mpad(nx)] : ~0ull;
        xa = ta ? y : xa;
        xb = ta ? xb : y;
      }
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) mkeys[mpad(my0 + k)] = v[k];
    }
  }
  __syncthreads();
  if (mode == 1) {
    // runs of equal (begin, rank): order by span_id, stably (j ascends in a run).
    // Phase 1 (read-only) records each run's length at its start in the perm
    // slots of the trace (scratch until the final write); phase 2 sorts every
    // run by its own thread, touching only that run's keys.
    for (uint32_t p = tid; p < len; p += THREADS) {
      const uint64_t kp = mkeys[mpad(p)] >> 14;
      uint32_t run = 0;
      if (p == 0 || (mkeys[mpad(p - 1)] >> 14) != kp) {
        uint32_t e = p + 1;
        while (e < len && (mkeys[mpad(e)] >> 14) == kp) ++e;
        run = e - p;
      }
      perm[lo + p] = run;
    }
    __syncthreads();
    for (uint32_t p = tid; p < len; p += THREADS) {
      const uint32_t run = perm[lo + p];
      if (run < 2) continue;
      if (run > 1024) {  // pathological tie run: the global sort handles the batch
        atomicOr(fallback, 1u);
        continue;
      }
      const uint32_t e = p + run;
      for (uint32_t q = p + 1; q < e; ++q) {  // insertion by span_id
        const uint64_t kq = mkeys[mpad(q)];
        const uint64_t sq = sid[lo + (kq & 0x3FFFu)];
        uint32_t r = q;
        while (r > p && sid[lo + (mkeys[mpad(r - 1)] & 0x3FFFu)] > sq) {
          mkeys[mpad(r)] = mkeys[mpad(r - 1)];
          --r;
        }
        mkeys[mpad(r)] = kq;
      }
    }
    __syncthreads();
  }
  for (uint32_t j = tid; j < len; j += THREADS) perm[lo + j] = (uint32_t)(lo + (mkeys[mpad(j)] & 0x3FFFu));
}

}  // namespace

void run_sort_timeline(xsp_ctx* ctx, uint64_t n, const uint64_t* begin, const uint8_t* flags, const uint64_t* sid,
                       uint32_t T, const uint64_t* off, uint32_t* perm, uint32_t* was_sorted, cudaStream_t st) {
  uint32_t* flag = ctx->d<uint32_t>("s.flag", 1);
  XSP_CUDA(cudaMemsetAsync(flag, 0, 4, st));
  auto blocks = [](uint64_t m) { return ceil_div(m ? m : 1, 256); };
  k_sort_check<<<(unsigned)std::min<uint64_t>(ceil_div(n ? n : 1, kCheckChunk), 148 * 8), 256, 0, st>>>(
      begin, flags, sid, off, T, n, perm, flag);
  ++ctx->launches;
  uint32_t* h = ctx->h<uint32_t>("s.flag_h", 1);
  XSP_CUDA(cudaMemcpyAsync(h, flag, 4, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  *was_sorted = h[0] == 0;
  if (*was_sorted || n <= 1) return;
  // per-trace CTA sort; the global radix sort only if some trace does not fit
  XSP_CUDA(cudaMemsetAsync(flag, 0, 4, st));
  ctx->stage_begin("sort", st);
  // register budgets sized for 6 / 3 / 1 resident CTAs per SM (a few spilled
  // registers cost less than the lost occupancy)
  auto* k_small = k_sort_merge<256, 16, 6>;
  auto* k_mid = k_sort_merge<512, 16, 3>;
  auto* k_large = k_sort_merge<1024, 16, 1>;
  auto smem = [](uint32_t cap) { return (size_t)(cap + cap / 16) * 8; };
  XSP_CUDA(cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(kSegCapSmall)));
  XSP_CUDA(cudaFuncSetAttribute(k_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(kSegCapMid)));
  XSP_CUDA(cudaFuncSetAttribute(k_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(kSegCap)));
  for (const void* f : {(const void*)k_small, (const void*)k_mid, (const void*)k_large})
    XSP_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  k_small<<<T, 256, smem(kSegCapSmall), st>>>(begin, flags, sid, off, 0, perm, flag);
  k_mid<<<T, 512, smem(kSegCapMid), st>>>(begin, flags, sid, off, kSegCapSmall + 1, perm, flag);
  k_large<<<T, 1024, smem(kSegCap), st>>>(begin, flags, sid, off, kSegCapMid + 1, perm, flag);
  ctx->stage_end("sort", st);
  ctx->launches += 3;
  XSP_CUDA(cudaMemcpyAsync(h, flag, 4, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  if (!h[0] && !getenv("XSP_SORT_GLOBAL")) return;
  k_iota_u32<<<blocks(n), 256, 0, st>>>(perm, n);
  ++ctx->launches;
  uint64_t* key = ctx->d<uint64_t>("s.key", n);
  RadixScratch rs;
  rs.keys_alt = ctx->d<uint64_t>("rs.keys_alt", n);
  rs.vals_alt = ctx->d<uint32_t>("rs.vals_alt", n);
  const uint64_t ce = radix_counts_elems(n);
  rs.counts = ctx->d<uint32_t>("rs.counts", ce);
  rs.scan_tmp = ctx->d<uint32_t>("rs.scan", scan_scratch_elems(ce));
  rs.and_or = ctx->d<unsigned long long>("rs.andor", 2);
  rs.and_or_host = ctx->h<unsigned long long>("rs.andor_h", 2);
  const int bits[4] = {64, 8, 64, 32};
  for (int field = 0; field < 4; ++field) {
    k_sort_key<<<blocks(n), 256, 0, st>>>(field, perm, begin, flags, sid, off, T, n, key);
    ++ctx->launches;
    radix_sort_pairs(key, perm, n, 0, bits[field], rs, st, &ctx->launches);
  }
}

}  // namespace xsp
