// Stage (b): sort_timeline (span.cpp:112-127) on the device — a stable sort of
// every trace's spans by (begin_ns, rank(level), span_id).
//
// Presorted input (the TraceBundle invariant) is detected first and returns the
// identity without sorting. Otherwise every trace of up to kSegCap spans is
// sorted by ONE CTA in shared memory: the trace's begin / span_id ranges are
// reduced, each span gets a packed 64-bit key
//   (begin - min_begin) | rank | (span_id - min_span_id)
// and a stable LSD radix sort of the 16-bit index permutation (warp-level
// histograms, a digit-major scan, ballot-ranked scatter) orders it.
// HBM traffic is one read of begin/span_id/flags and one perm write (21 B/span).
// Traces that are longer or whose packed key needs more than 64 bits fall back
// to one global LSD radix sort over the composite key (trace, begin_ns, rank,
// span_id): four stable passes from the least significant field, each skipping
// the 8-bit digits that are constant over the batch.

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

// Lanes of `valid` holding the same 8-bit digit as this lane: one ballot per
// digit bit (warp-level multisplit) instead of __match_any_sync; bits that are
// constant over the trace (clear in `vary`) need no ballot.
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, uint32_t valid, uint32_t vary) {
  uint32_t m = valid;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (!((vary >> b) & 1u)) continue;
    const uint32_t bit = (d >> b) & 1u;
    const uint32_t v = __ballot_sync(0xffffffffu, bit);
    m &= bit ? v : ~v;
  }
  return m;
}

// Shared memory of k_sort_seg: the packed keys stay in place; the LSD passes
// permute 16-bit indices between two buffers (the trace's keys plus both index
// buffers fit one SM: 128 + 64 KB).
template <uint32_t CAP, int WARPS>
struct SegSmem {
  unsigned long long key[CAP];
  uint16_t idx[2][CAP];
  uint16_t wcnt[WARPS][258];  // per-warp digit counts, then per-warp digit offsets (rows padded
                              // by one word: the digit scan reads them conflict-free)
};

// One CTA per trace: key = (begin - min) | rank | (span_id - min), packed into
// 64 bits when the trace's ranges allow (else the trace falls back), then a
// stable LSD radix sort (8-bit digits, constant digits skipped) of the index
// permutation: per pass every warp histograms its contiguous segment of the
// current order, a scan gives each (digit, warp) its output offset, and the
// warp re-walks its segment placing indices with ballot (multisplit) ranks.
// Size classes: traces of at most kSegCapSmall spans run as 256-thread CTAs with
// 52 KB of shared memory (4 per SM), up to kSegCapMid as 512-thread CTAs with
// 104 KB (2 per SM), longer ones as 1024-thread CTAs with 210 KB.
// Every launch covers all traces; a CTA leaves traces of the other class.
template <uint32_t CAP, int THREADS>
__global__ void __launch_bounds__(THREADS) k_sort_seg(const uint64_t* __restrict__ begin,
                                                      const uint8_t* __restrict__ flags,
                                                      const uint64_t* __restrict__ sid,
                                                      const uint64_t* __restrict__ off, uint32_t min_len,
                                                      uint32_t* __restrict__ perm, uint32_t* __restrict__ fallback) {
  constexpr int kSegWarps = THREADS / 32;
  constexpr uint32_t cap = CAP;
  // iterations of 32 spans per warp segment (a segment holds <= CAP / kSegWarps)
  constexpr int kIters = (int)(CAP / (kSegWarps * 32));
  static_assert(CAP <= 16384, "indices are packed in 14 bits");
  extern __shared__ __align__(16) unsigned char seg_dyn[];
  SegSmem<CAP, kSegWarps>& sm = *reinterpret_cast<SegSmem<CAP, kSegWarps>*>(seg_dyn);
  __shared__ unsigned long long red[4][kSegWarps];
  __shared__ uint32_t s_shift[2];
  __shared__ int s_ok;
  __shared__ unsigned long long s_and, s_or;
  __shared__ uint32_t s_tot[256];
  const uint32_t t = blockIdx.x, tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint64_t lo = off[t], hi = off[t + 1];
  const uint32_t len = (uint32_t)(hi - lo);
  if (len < min_len) return;  // the small class sorts it
  if (len <= 1) {
    if (len == 1 && tid == 0) perm[lo] = (uint32_t)lo;
    return;
  }
  if (len > cap) {
    if (CAP < kSegCap) return;  // the large class sorts it
    if (tid == 0) atomicOr(fallback, 1u);
    return;
  }
  // ranges of begin and span_id
  uint64_t bmin = ~0ull, bmax = 0, smin = ~0ull, smax = 0;
  for (uint32_t j = tid; j < len; j += blockDim.x) {
    const uint64_t b = begin[lo + j], s = sid[lo + j];
    bmin = min(bmin, b); bmax = max(bmax, b);
    smin = min(smin, s); smax = max(smax, s);
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
    for (uint32_t w = 1; w < kSegWarps; ++w) {
      red[0][0] = min(red[0][0], red[0][w]); red[1][0] = max(red[1][0], red[1][w]);
      red[2][0] = min(red[2][0], red[2][w]); red[3][0] = max(red[3][0], red[3][w]);
    }
    const uint32_t sb = bit_width64(red[3][0] - red[2][0]);
    const uint32_t bb = bit_width64(red[1][0] - red[0][0]);
    s_ok = sb + 2 + bb <= 64;
    s_shift[0] = sb;      // rank field
    s_shift[1] = sb + 2;  // begin field
    s_and = ~0ull;
    s_or = 0;
    if (!s_ok) atomicOr(fallback, 1u);
  }
  __syncthreads();
  if (!s_ok) return;
  bmin = red[0][0];
  smin = red[2][0];
  const uint32_t sh_r = s_shift[0], sh_b = s_shift[1];
  unsigned long long kand = ~0ull, kor = 0;
  for (uint32_t j = tid; j < len; j += blockDim.x) {
    const uint32_t l = f_level(flags[lo + j]);
    const uint64_t r = l >= XSP_LEVEL_KERNEL ? 3 : l + 1;  // rank (span.hpp:51-59)
    const unsigned long long k = ((begin[lo + j] - bmin) << sh_b) | (r << sh_r) | (sid[lo + j] - smin);
    sm.key[j] = k;
    sm.idx[0][j] = (uint16_t)j;
    kand &= k;
    kor |= k;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kand &= __shfl_xor_sync(0xffffffffu, kand, o);
    kor |= __shfl_xor_sync(0xffffffffu, kor, o);
  }
  if (lane == 0) {
    atomicAnd(&s_and, kand);
    atomicOr(&s_or, kor);
  }
  __syncthreads();
  const unsigned long long varying = s_and ^ s_or;
  // warp w owns positions [w * seg, (w + 1) * seg) of the current order
  const uint32_t seg = ((len + kSegWarps - 1) / kSegWarps + 31) & ~31u;
  const uint32_t p0 = min(len, warp * seg), p1 = min(len, p0 + seg);
  int cur = 0;
  for (int shift = 0; shift < 64; shift += 8) {
    if (!((varying >> shift) & 0xFFull)) continue;
    const uint16_t* src = sm.idx[cur];
    uint16_t* dst = sm.idx[cur ^ 1];
    for (uint32_t d = lane; d < 256; d += 32) sm.wcnt[warp][d] = 0;
    __syncwarp();
    // histogram of the warp's segment; every lane keeps, per iteration, its
    // index, digit, rank among equal digits and whether it is the last of them
    // (packed: x | d << 14 | below << 22 | last << 27 | valid << 28), so the
    // scatter needs neither the keys nor the ballots again
    const uint32_t vary = (uint32_t)(varying >> shift) & 0xFFu;
    uint32_t pk[kIters];
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      pk[it] = 0;
      const uint32_t base = p0 + 32u * it;
      if (base >= p1) continue;  // warp-uniform
      const uint32_t i = base + lane;
      const bool v = i < p1;
      const uint32_t valid = __ballot_sync(0xffffffffu, v);
      const uint32_t x = v ? src[i] : 0u;
      const uint32_t d = v ? (uint32_t)(sm.key[x] >> shift) & 0xFFu : 0u;
      const uint32_t peers = digit_peers(d, valid, vary);
      const uint32_t below = __popc(peers & lanemask_lt());
      const bool last = (peers >> lane) <= 1u;  // no equal digit in a higher lane
      if (v && last) sm.wcnt[warp][d] += (uint16_t)(below + 1);
      __syncwarp();
      if (v) pk[it] = x | d << 14 | below << 22 | (uint32_t)last << 27 | 1u << 28;
    }
    __syncthreads();
    // per digit: totals and the exclusive offsets of the warps (digit-major);
    // kDP consecutive threads share a digit, each scanning kSegWarps / kDP warps
    {
      constexpr int kDP = THREADS >= 256 ? THREADS / 256 : 1;
      constexpr int kWPT = kSegWarps / kDP;
      static_assert(kSegWarps % kDP == 0, "warps per digit thread");
      const uint32_t d = tid / kDP, q = tid % kDP;
      if (d < 256) {
        uint32_t c[kWPT], sum = 0;
#pragma unroll
        for (int w = 0; w < kWPT; ++w) {
          c[w] = sm.wcnt[q * kWPT + w][d];
          sum += c[w];
        }
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < kDP; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o, kDP);
          if (q >= (uint32_t)o) inc += y;
        }
        uint32_t run = inc - sum;
#pragma unroll
        for (int w = 0; w < kWPT; ++w) {
          sm.wcnt[q * kWPT + w][d] = (uint16_t)run;
          run += c[w];
        }
        if (q == kDP - 1) s_tot[d] = inc;
      }
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 256 digit totals (8 per lane)
      uint32_t v[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[q] = s_tot[lane * 8 + q];
        sum += v[q];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      uint32_t run = incl - sum;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        s_tot[lane * 8 + q] = run;
        run += v[q];
      }
    }
    __syncthreads();
    // stable scatter: digit start + earlier warps + running rank in this warp
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      if (p0 + 32u * it >= p1) continue;  // warp-uniform
      const uint32_t u = pk[it];
      const bool v = (u >> 28) & 1u;
      const uint32_t x = u & 0x3FFFu, d = (u >> 14) & 0xFFu, below = (u >> 22) & 31u;
      const uint32_t r0 = v ? sm.wcnt[warp][d] : 0u;
      __syncwarp();
      if (v) {
        dst[s_tot[d] + r0 + below] = (uint16_t)x;
        if ((u >> 27) & 1u) sm.wcnt[warp][d] = (uint16_t)(r0 + below + 1);
      }
      __syncwarp();
    }
    __syncthreads();
    cur ^= 1;
  }
  for (uint32_t j = tid; j < len; j += blockDim.x) perm[lo + j] = (uint32_t)(lo + sm.idx[cur][j]);
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
  auto* k_small = k_sort_seg<kSegCapSmall, 256>;
  auto* k_mid = k_sort_seg<kSegCapMid, 512>;
  auto* k_large = k_sort_seg<kSegCap, 1024>;
  constexpr size_t smem_small = sizeof(SegSmem<kSegCapSmall, 8>), smem_mid = sizeof(SegSmem<kSegCapMid, 16>),
                   smem_large = sizeof(SegSmem<kSegCap, 32>);
  XSP_CUDA(cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_small));
  XSP_CUDA(cudaFuncSetAttribute(k_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_mid));
  XSP_CUDA(cudaFuncSetAttribute(k_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_large));
  ctx->stage_begin("sort", st);
  k_small<<<T, 256, smem_small, st>>>(begin, flags, sid, off, 0, perm, flag);
  k_mid<<<T, 512, smem_mid, st>>>(begin, flags, sid, off, kSegCapSmall + 1, perm, flag);
  k_large<<<T, 1024, smem_large, st>>>(begin, flags, sid, off, kSegCapMid + 1, perm, flag);
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
