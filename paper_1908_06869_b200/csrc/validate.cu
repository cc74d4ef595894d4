// Stage (a) invariants: validate_bundle (span.cpp:129-192) for every trace of a
// batch on the device.
//
// The reference walks each bundle once with an unordered_set of span ids and
// reports, per span and in this order: negative duration; correlation_id
// missing (launch/exec) / present on a sync span; duplicate span_id (every
// occurrence after the first); trace_id mismatch; out of order (timeline key of
// the predecessor greater); negative int64 metric tag (flop_count_sp,
// dram_read_bytes, dram_write_bytes, in that order); occupancy double outside
// [0,1]. Then per bundle: model span missing / multiple model spans, and model
// level disabled.
//
// Here the per-span rules are one streaming pass over the columns (8
// consecutive spans per thread). Duplicate ids use a device hash table keyed by
// (trace, span_id) whose slot keeps the smallest row of the key (atomicMin), so
// a span is a duplicate iff its key's minimum row is not its own. Issues are
// appended as (trace, local row, rule) keys, radix-sorted into the reference's
// report order, and delimited per trace by a scan of per-trace counts.

#include "ctx.h"
#include "prims.cuh"

namespace xsp {

namespace {

constexpr int kValThreads = 256;
constexpr int kValItems = 8;
constexpr int kValTile = kValThreads * kValItems;
constexpr uint64_t kLocalBundle = (1ull << 36) - 1;  // bundle-level issues sort last

__device__ __forceinline__ uint32_t span_trace(const uint64_t* __restrict__ off, uint32_t T, uint64_t i) {
  return trace_of(off, 0, T, i);
}

__device__ __forceinline__ uint64_t hash_key(uint32_t t, uint64_t sid) {
  uint64_t h = sid * 0x9E3779B97F4A7C15ull ^ ((uint64_t)t * 0xC2B2AE3D27D4EB4Full);
  h ^= h >> 31;
  h *= 0xBF58476D1CE4E5B9ull;
  return h ^ (h >> 29);
}

// Table entry: trace << 32 | (row + 1); 0 = empty. Equal keys share one slot
// (the first inserted), which keeps the minimum row.
__global__ void k_val_insert(const uint64_t* __restrict__ sid, const uint64_t* __restrict__ off, uint32_t T,
                             uint64_t n, unsigned long long* __restrict__ table, uint64_t mask,
                             const uint32_t* __restrict__ t_big) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t t = span_trace(off, T, i);
  if (!t_big[t]) return;  // checked on chip (k_val_dup_local)
  const uint64_t s = sid[i];
  const unsigned long long mine = ((unsigned long long)t << 32) | (uint32_t)(i + 1);
  for (uint64_t slot = hash_key(t, s) & mask;; slot = (slot + 1) & mask) {
    unsigned long long cur = atomicCAS(table + slot, 0ull, mine);
    if (cur == 0ull) return;
    if ((uint32_t)(cur >> 32) == t && sid[(uint32_t)cur - 1] == s) {
      atomicMin(table + slot, mine);
      return;
    }
  }
}

__device__ __forceinline__ bool is_duplicate(const uint64_t* __restrict__ sid, uint32_t t, uint64_t i,
                                             const unsigned long long* __restrict__ table, uint64_t mask) {
  const uint64_t s = sid[i];
  for (uint64_t slot = hash_key(t, s) & mask;; slot = (slot + 1) & mask) {
    const unsigned long long cur = table[slot];
    if ((uint32_t)(cur >> 32) == t && sid[(uint32_t)cur - 1] == s) return (uint32_t)cur != (uint32_t)(i + 1);
  }
}

// Traces of at most kDupCap spans find their duplicate span ids on chip: one
// CTA per trace stages the trace's span ids in shared memory and inserts them
// into a shared open-addressing table (slot = local row + 1, the minimum row
// of a key kept by atomicMin), so the check never touches a global table.
// Longer traces are flagged for the global table (k_val_insert).
constexpr uint32_t kDupCap = 12288;
constexpr uint32_t kDupSlots = 32768;  // power-of-two table >= 2 x the trace, at most this
constexpr size_t kDupSmem = kDupCap * 8 + kDupSlots * 4;
constexpr int kDupThreads = 1024;

__global__ void __launch_bounds__(kDupThreads) k_val_dup_local(const uint64_t* __restrict__ sid,
                                                               const uint64_t* __restrict__ off, uint32_t T,
                                                               uint8_t* __restrict__ dup, uint32_t* __restrict__ t_big,
                                                               uint32_t* __restrict__ any_big) {
  extern __shared__ __align__(16) unsigned char dup_dyn[];
  uint64_t* s_sid = reinterpret_cast<uint64_t*>(dup_dyn);
  uint32_t* s_tab = reinterpret_cast<uint32_t*>(s_sid + kDupCap);
  const uint32_t t = blockIdx.x;
  const uint64_t lo = off[t], m = off[t + 1] - lo;
  if (m > kDupCap) {
    if (threadIdx.x == 0) {
      t_big[t] = 1;
      *any_big = 1;
    }
    return;
  }
  if (threadIdx.x == 0) t_big[t] = 0;
  uint32_t slots = 16;
  while (slots < 2 * m) slots <<= 1;
  const uint32_t mask = slots - 1;
  for (uint32_t r = threadIdx.x; r < m; r += kDupThreads) s_sid[r] = sid[lo + r];
  for (uint32_t q = threadIdx.x; q < slots; q += kDupThreads) s_tab[q] = 0;
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < m; r += kDupThreads) {
    const uint64_t s = s_sid[r];
    for (uint32_t slot = (uint32_t)hash_key(0, s) & mask;; slot = (slot + 1) & mask) {
      const uint32_t cur = atomicCAS(s_tab + slot, 0u, r + 1);
      if (cur == 0u) break;
      if (s_sid[cur - 1] == s) {
        atomicMin(s_tab + slot, r + 1);
        break;
      }
    }
  }
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < m; r += kDupThreads) {
    const uint64_t s = s_sid[r];
    uint8_t d = 0;
    for (uint32_t slot = (uint32_t)hash_key(0, s) & mask;; slot = (slot + 1) & mask) {
      const uint32_t cur = s_tab[slot];
      if (s_sid[cur - 1] == s) {
        d = cur != r + 1;
        break;
      }
    }
    dup[lo + r] = d;
  }
}

struct ValArgs {
  const uint64_t* span_id;
  const uint64_t* begin;
  const uint64_t* end;
  const uint8_t* flags;
  const double* occupancy;
  const uint64_t* trace_id;       // optional
  const uint64_t* meta_trace_id;  // optional (with trace_id)
  const uint8_t* tag_bits;        // optional
  const uint64_t* off;
  const uint32_t* levels;
  uint32_t T;
  uint64_t n;
  const uint32_t* metric_base;  // [blocks] metric rows before each block
  const uint8_t* dup;           // duplicate flags of the on-chip traces
  const uint32_t* t_big;        // traces checked through the global table
  const unsigned long long* table;
  uint64_t mask;
  uint32_t* model_count;  // [T]
  uint32_t* trace_count;  // [T] issues per trace
  uint64_t* keys;         // issue keys
  uint32_t* n_keys;
  uint64_t cap;
};

__device__ __forceinline__ void emit_issue(const ValArgs& a, uint32_t t, uint64_t local, uint32_t rule) {
  const uint32_t s = atomicAdd(a.n_keys, 1u);
  if (s < a.cap) a.keys[s] = ((uint64_t)t << 40) | (local << 4) | rule;
  atomicAdd(a.trace_count + t, 1u);
}

__device__ __forceinline__ uint32_t tl_rank(uint8_t f) {
  const uint32_t l = f_level(f);
  return l >= XSP_LEVEL_KERNEL ? 3 : l + 1;  // rank(): Model 1, Layer 2, Kernel = Api 3 (span.hpp:51-59)
}

// metric rows per block of kValTile spans
__global__ void __launch_bounds__(kValThreads) k_val_mcount(const uint8_t* __restrict__ flags, uint64_t n,
                                                            uint32_t* __restrict__ counts) {
  const uint64_t base = (uint64_t)blockIdx.x * kValTile + threadIdx.x * kValItems;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kValItems; ++k)
    if (base + k < n) c += (flags[base + k] & XSP_F_METRICS) != 0;
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t w[kValThreads / 32];
  if (lane_id() == 0) w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int k = 0; k < kValThreads / 32; ++k) s += w[k];
    counts[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kValThreads) k_val_spans(ValArgs a) {
  __shared__ uint32_t sm[33];
  const uint64_t base = (uint64_t)blockIdx.x * kValTile + threadIdx.x * kValItems;
  uint8_t fl[kValItems];
  uint32_t mine = 0;
#pragma unroll
  for (int k = 0; k < kValItems; ++k) {
    fl[k] = base + k < a.n ? a.flags[base + k] : 0;
    mine += base + k < a.n && (fl[k] & XSP_F_METRICS);
  }
  uint32_t mrow = a.metric_base[blockIdx.x] + block_exclusive_scan<uint32_t>(mine, sm, nullptr);
  if (base >= a.n) return;
  uint32_t t = span_trace(a.off, a.T, base);
  uint64_t t_lo = a.off[t], t_hi = a.off[t + 1];
  for (int k = 0; k < kValItems; ++k) {
    const uint64_t i = base + k;
    if (i >= a.n) break;
    while (i >= t_hi) {
      ++t;
      t_lo = t_hi;
      t_hi = a.off[t + 1];
    }
    const uint8_t f = fl[k];
    const uint64_t local = i - t_lo;
    const uint64_t b = a.begin[i], e = a.end[i];
    if (e < b) emit_issue(a, t, local, XSP_V_NEG_DURATION);
    const uint32_t kind = f_kind(f);
    const bool needs_cid = kind == XSP_KIND_LAUNCH || kind == XSP_KIND_EXEC;
    const bool has_cid = (f & XSP_F_CID) != 0;
    if (needs_cid && !has_cid) emit_issue(a, t, local, XSP_V_CID_MISSING);
    if (!needs_cid && has_cid) emit_issue(a, t, local, XSP_V_CID_ON_SYNC);
    if (a.t_big[t] ? is_duplicate(a.span_id, t, i, a.table, a.mask) : a.dup[i] != 0)
      emit_issue(a, t, local, XSP_V_DUP_SPAN_ID);
    if (a.trace_id && a.trace_id[i] != a.meta_trace_id[t]) emit_issue(a, t, local, XSP_V_TRACE_ID);
    if (is_model_span(f)) atomicAdd(a.model_count + t, 1u);
    if (local > 0) {
      const uint64_t pb = a.begin[i - 1];
      const uint8_t pf = a.flags[i - 1];
      bool bad = pb > b;
      if (pb == b) {
        const uint32_t r0 = tl_rank(pf), r1 = tl_rank(f);
        bad = r0 > r1 || (r0 == r1 && a.span_id[i - 1] > a.span_id[i]);
      }
      if (bad) emit_issue(a, t, local, XSP_V_OUT_OF_ORDER);
    }
    const uint8_t tb = a.tag_bits ? a.tag_bits[i] : 0;
    if (tb & XSP_TAG_NEG_FLOPS) emit_issue(a, t, local, XSP_V_NEG_FLOPS);
    if (tb & XSP_TAG_NEG_READ) emit_issue(a, t, local, XSP_V_NEG_READ);
    if (tb & XSP_TAG_NEG_WRITE) emit_issue(a, t, local, XSP_V_NEG_WRITE);
    if (f & XSP_F_METRICS) {
      if (tb & XSP_TAG_OCC_DOUBLE) {
        const double o = a.occupancy[mrow];
        if (o < 0.0 || o > 1.0) emit_issue(a, t, local, XSP_V_OCC_RANGE);
      }
      ++mrow;
    }
  }
}

// bundle-level rules (span.cpp:183-190); one thread per trace
__global__ void k_val_traces(ValArgs a) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.T) return;
  const uint32_t m = a.model_count[t];
  if (m == 0) emit_issue(a, t, kLocalBundle, XSP_V_NO_MODEL);
  else if (m > 1) emit_issue(a, t, kLocalBundle, XSP_V_MULTI_MODEL);
  if (!(a.levels[t] & (1u << XSP_LEVEL_MODEL))) emit_issue(a, t, kLocalBundle, XSP_V_MODEL_LEVEL);
}

__global__ void k_val_out(const uint64_t* __restrict__ keys, uint32_t nk, const uint64_t* __restrict__ off,
                          uint32_t* __restrict__ row, uint8_t* __restrict__ rule) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nk) return;
  const uint64_t k = keys[j];
  const uint32_t t = (uint32_t)(k >> 40);
  const uint64_t local = (k >> 4) & kLocalBundle;
  row[j] = local == kLocalBundle ? 0xFFFFFFFFu : (uint32_t)(off[t] + local);
  rule[j] = (uint8_t)(k & 15u);
}

}  // namespace

void run_validate(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_traces* tr, const xsp_validate_in* vin,
                  xsp_validation_out* out, cudaStream_t st) {
  const uint64_t n = c->n_spans;
  const uint32_t T = tr->n_traces;
  if (n >= 0xFFFFFFF0ull) throw std::invalid_argument("more than 2^32-16 spans in one call");
  if (T >= (1u << 24)) throw std::invalid_argument("more than 2^24 traces in one validation call");
  const unsigned nb = ceil_div(n ? n : 1, kValTile);
  uint32_t* mcount = ctx->d<uint32_t>("v.mcount", nb + 1);
  uint32_t* counters = ctx->d<uint32_t>("v.counters", 4);
  uint32_t* model_count = ctx->d<uint32_t>("v.model_count", T + 1);
  uint32_t* trace_count = ctx->d<uint32_t>("v.trace_count", T + 1);
  // duplicate span ids: on chip per trace; traces beyond kDupCap spans through a
  // global (trace, span_id) table sized for their spans only
  uint8_t* dupf = ctx->d<uint8_t>("v.dup", n + 1);
  uint32_t* t_big = ctx->d<uint32_t>("v.t_big", T + 1);
  uint32_t* any_big = ctx->d<uint32_t>("v.any_big", 1);
  XSP_CUDA(cudaMemsetAsync(any_big, 0, 4, st));
  if (T) {
    XSP_CUDA(cudaFuncSetAttribute(k_val_dup_local, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDupSmem));
    k_val_dup_local<<<T, kDupThreads, kDupSmem, st>>>(c->span_id, tr->span_off, T, dupf, t_big, any_big);
    ++ctx->launches;
  }
  uint32_t* hb = ctx->h<uint32_t>("v.any_big_h", 1);
  xfer_small(hb, any_big, 4, st);
  XSP_CUDA(cudaStreamSynchronize(st));
  uint64_t cap = 16;
  if (hb[0])
    while (cap < 2 * n) cap <<= 1;
  auto* table = ctx->d<unsigned long long>("v.table", cap);
  if (hb[0]) XSP_CUDA(cudaMemsetAsync(table, 0, cap * 8, st));
  ValArgs a;
  a.span_id = c->span_id;
  a.begin = c->begin_ns;
  a.end = c->end_ns;
  a.flags = c->flags;
  a.occupancy = c->occupancy;
  a.trace_id = vin ? vin->trace_id : nullptr;
  a.meta_trace_id = vin ? vin->meta_trace_id : nullptr;
  a.tag_bits = vin ? vin->tag_bits : nullptr;
  if (a.trace_id && !a.meta_trace_id) throw std::invalid_argument("trace_id given without meta_trace_id");
  a.off = tr->span_off;
  a.levels = tr->levels;
  a.T = T;
  a.n = n;
  a.metric_base = mcount;
  a.dup = dupf;
  a.t_big = t_big;
  a.table = table;
  a.mask = cap - 1;
  a.model_count = model_count;
  a.trace_count = trace_count;
  a.n_keys = counters;
  if (n) {
    k_val_mcount<<<nb, kValThreads, 0, st>>>(c->flags, n, mcount);
    uint32_t* scr = ctx->d<uint32_t>("v.scan", scan_scratch_elems(nb));
    exclusive_scan<uint32_t, uint32_t>(mcount, mcount, nb, scr, (uint32_t*)nullptr, st, &ctx->launches);
    ctx->launches += 1;
    if (hb[0]) {
      k_val_insert<<<ceil_div(n, 256), 256, 0, st>>>(c->span_id, tr->span_off, T, n, table, cap - 1, t_big);
      ++ctx->launches;
    }
  }
  // issue keys: sized for a mostly clean batch; rerun once with the exact count on overflow
  uint32_t* h = ctx->h<uint32_t>("v.count_h", 1);
  uint64_t kcap = n / 8 + 3ull * T + 1024;
  uint32_t nk = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    XSP_CUDA(cudaMemsetAsync(counters, 0, 16, st));
    XSP_CUDA(cudaMemsetAsync(model_count, 0, (T + 1) * 4ull, st));
    XSP_CUDA(cudaMemsetAsync(trace_count, 0, (T + 1) * 4ull, st));
    a.keys = ctx->d<uint64_t>("v.keys", kcap);
    a.cap = kcap;
    ctx->stage_begin("validate", st);
    if (n) k_val_spans<<<nb, kValThreads, 0, st>>>(a);
    if (T) k_val_traces<<<ceil_div(T, 256), 256, 0, st>>>(a);
    ctx->stage_end("validate", st);
    ctx->launches += 2;
    xfer_small(h, counters, 4, st);
    XSP_CUDA(cudaStreamSynchronize(st));
    nk = h[0];
    if (nk <= kcap) break;
    kcap = nk;
  }
  uint64_t* keys = a.keys;
  // per-trace offsets
  uint32_t* toff = ctx->d<uint32_t>("v.trace_off", T + 2);
  uint32_t* scr2 = ctx->d<uint32_t>("v.scan2", scan_scratch_elems(T + 1));
  exclusive_scan<uint32_t, uint32_t>(trace_count, toff, (uint64_t)T + 1, scr2, (uint32_t*)nullptr, st,
                                     &ctx->launches);
  uint32_t* vals = ctx->d<uint32_t>("v.vals", nk + 1);
  uint32_t* row = ctx->d<uint32_t>("v.row", nk + 1);
  uint8_t* rule = ctx->d<uint8_t>("v.rule", nk + 1);
  if (nk > 1) {
    RadixScratch rs;
    rs.keys_alt = ctx->d<uint64_t>("v.rs.keys_alt", nk);
    rs.vals_alt = ctx->d<uint32_t>("v.rs.vals_alt", nk);
    const uint64_t ce = radix_counts_elems(nk);
    rs.counts = ctx->d<uint32_t>("v.rs.counts", ce);
    rs.scan_tmp = ctx->d<uint32_t>("v.rs.scan", scan_scratch_elems(ce));
    rs.and_or = ctx->d<unsigned long long>("v.rs.andor", 2);
    rs.and_or_host = ctx->h<unsigned long long>("v.rs.andor_h", 2);
    XSP_CUDA(cudaMemsetAsync(vals, 0, (uint64_t)nk * 4, st));
    radix_sort_pairs(keys, vals, nk, 0, 64, rs, st, &ctx->launches);
  }
  if (nk) {
    k_val_out<<<ceil_div(nk, 256), 256, 0, st>>>(keys, nk, tr->span_off, row, rule);
    ++ctx->launches;
  }
  out->n_issues = nk;
  out->trace_issue_off = toff;
  out->issue_row = row;
  out->issue_rule = rule;
}

}  // namespace xsp
