// Stages (c) + (d): parent assignment by interval containment and the
// correlation-id launch->exec join, for every trace of a batch at once.
//
// Reference semantics: assign_parents (correlator.cpp:141-282) and
// correlate_async (correlator.cpp:287-364). The reference walks an interval
// tree per child span; here the whole batch is ONE reduce-then-scan
// over the timeline-ordered span columns (pass 1):
//   * layers are placed by a per-span compare against their trace's model span
//     and numbered by a global placed-layer count (layer_index = count - trace base);
//   * because the input is sorted by (begin, rank, span_id), the containment
//     candidates of a child are exactly the preceding placed layers of its trace
//     with end >= child.end. The scan carries, for the last preceding placed
//     layer j, end_j and M_j = max end over the layers before j, which decides
//     0 / 1 / >=2 candidates exactly except when end_j < e <= M_j (nested or
//     overlapping layers), which goes to an exact rare path;
//   * kernel launches (+ synchronous kernels) and execs are compacted into
//     timeline-ordered 16-byte entries.
// The cid join (stage d) is a sort-merge join on presorted input: per trace,
// the r-th cid-bearing launch meets the r-th exec when both streams carry the
// same strictly increasing cids (checked in one streaming pass); traces that
// fail the check use a per-trace open-addressing table.
// Orphans, ambiguities and explicit-parent kernels are rare: they are appended
// to exception lists and put into the reference's output order by radix sort.

#include <cuda.h>
#include <cudaTypedefs.h>

#include "ctx.h"
#include "prims.cuh"

namespace xsp {

constexpr uint32_t PAR_ORPHAN = 0xFFFFFFFFu;
constexpr uint32_t PAR_AMBIG = 0xFFFFFFFEu;
constexpr uint32_t PAR_PENDING = 0xFFFFFFFDu;
constexpr uint32_t PAR_MAXROW = 0xFFFFFFF0u;

// Orphan categories = the reference's emission phases, in output order.
enum : uint32_t {
  CAT_LAYER = 0,      // layer pass, timeline order            (correlator.cpp:168-204)
  CAT_KERNEL = 1,     // kernel pass, timeline order           (:226-259)
  CAT_EXEC_NOCID = 2, // exec without cid, timeline order      (:289-295)
  CAT_LAUNCH = 3,     // launch fusion failures, tree order    (:321-346)
  CAT_LEFTOVER = 4    // unconsumed execs, by span_id          (:355-363)
};

// Kernel-list entry: a kernel launch (Kernel/Api level) or a synchronous kernel.
struct __align__(16) KlEnt {
  uint32_t row;     // span row
  uint32_t parent;  // placed layer row, or PAR_*
  uint64_t cid;     // correlation id (0 if absent)
};
// Execution-list entry: an exec span carrying a correlation id.
// Its correlation id is read back from the cid column by row when needed; the
// duration is computed by pass 1 from the staged tile, so the gather does not
// re-read begin_ns / end_ns at the (strided) exec rows.
struct __align__(16) ExEnt {
  uint32_t row;   // span row
  uint32_t mrow;  // metric-table row, kNone if none
  uint64_t dur;   // clamped end - begin of the exec span
};

struct Orphans {
  uint64_t* tc;   // trace << 3 | category
  uint64_t* key;  // order key within the category
  uint32_t* row;
  uint8_t* reason;
  uint32_t* count;
  uint32_t cap;   // entries beyond cap are counted, not written (the host retries larger)
};

__device__ __forceinline__ void emit_orphan(const Orphans& o, uint32_t t, uint32_t cat,
                                            uint64_t key, uint32_t row, uint8_t reason) {
  uint32_t s = atomicAdd(o.count, 1u);
  if (s >= o.cap) return;
  o.tc[s] = ((uint64_t)t << 3) | cat;
  o.key[s] = key;
  o.row[s] = row;
  o.reason[s] = reason;
}

__device__ __forceinline__ uint32_t trace_of32(const uint32_t* __restrict__ off, uint32_t T, uint32_t i) {
  uint32_t lo = 0, hi = T;  // off[lo] <= i < off[hi]
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// Trace of item i for a warp processing consecutive items: one binary search
// per warp, then a short per-lane walk (items of a trace are contiguous).
__device__ __forceinline__ uint32_t warp_trace_of(const uint32_t* __restrict__ off, uint32_t T,
                                                  uint32_t i, uint32_t first_i) {
  uint32_t t0 = 0;
  if (lane_id() == 0) t0 = trace_of32(off, T, first_i);
  uint32_t t = __shfl_sync(0xffffffffu, t0, 0);
  while (t + 1 < T && __ldg(off + t + 1) <= i) ++t;
  return t;
}

// ---------------------------------------------------------------------------
// K0: per trace, the model span = first MODEL/SYNC span (TraceBundle::model_span,
// span.cpp:298-303). One warp per trace; the model span is normally row 0.

__global__ void k_trace_prep(const uint8_t* __restrict__ flags, const uint64_t* __restrict__ begin,
                             const uint64_t* __restrict__ end, const uint64_t* __restrict__ sid,
                             const uint64_t* __restrict__ off, uint32_t T,
                             uint32_t* __restrict__ model_row, uint64_t* __restrict__ mb,
                             uint64_t* __restrict__ me, uint64_t* __restrict__ msid,
                             unsigned long long* __restrict__ err_key, uint64_t n, uint32_t tile_spans,
                             uint32_t* __restrict__ tile_lo, uint32_t* __restrict__ tile_hi) {
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  if (t >= T) return;
  const uint64_t lo = off[t], hi = off[t + 1];
  if (tile_lo && lo < hi) {
    // pass-1 tiles whose first / last span lies in this trace (trace_of semantics:
    // the containing non-empty trace); batches of long traces use k_tile_traces
    for (uint64_t b = (lo + tile_spans - 1) / tile_spans + lane; b * tile_spans < hi; b += 32) tile_lo[b] = t;
    for (uint64_t b = lo / tile_spans + lane; b * tile_spans < hi; b += 32) {
      const uint64_t last = min((b + 1) * tile_spans, n) - 1;
      if (last >= lo && last < hi) tile_hi[b] = t;
    }
  }
  uint64_t found = ~0ull;
  for (uint64_t base = lo; base < hi; base += 32) {
    uint64_t i = base + lane;
    bool m = i < hi && is_model_span(flags[i]);
    uint32_t bal = __ballot_sync(0xffffffffu, m);
    if (bal) {
      found = base + (__ffs(bal) - 1);
      break;
    }
  }
  if (lane == 0) {
    err_key[t] = ~0ull;
    if (found != ~0ull) {
      model_row[t] = (uint32_t)found;
      mb[t] = begin[found];
      me[t] = end[found];
      msid[t] = sid[found];
    } else {
      model_row[t] = kNone;
      mb[t] = 1;
      me[t] = 0;  // contains nothing
      msid[t] = 0;
    }
  }
}

// Pass-1 tiles: the (non-empty) trace holding each tile's first / last span, by
// binary search over the trace offsets — one thread per tile, so a long trace
// costs no serial walk over its tiles.
__global__ void k_tile_traces(const uint64_t* __restrict__ off, uint32_t T, uint64_t n, uint32_t tile_spans,
                              uint32_t ntiles, uint32_t* __restrict__ tile_lo, uint32_t* __restrict__ tile_hi) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= ntiles) return;
  // the last trace t < T with off[t] <= i (empty traces share their offset with
  // the next trace, so the last one is the non-empty trace that holds i)
  auto trace_at = [&](uint64_t i) {
    uint32_t lo = 0, hi = T;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(off + mid) <= i) lo = mid; else hi = mid;
    }
    return lo;
  };
  const uint64_t first = (uint64_t)b * tile_spans;
  tile_lo[b] = trace_at(first);
  tile_hi[b] = trace_at(min(first + tile_spans, n) - 1);
}

// ---------------------------------------------------------------------------
// Pass-1 scan state (the scan payload of a tile / warp / thread). Ends are stored as
// end+1 so that 0 means "no layer".
struct Full {
  uint64_t last_end1;  // end+1 of the last placed layer of the current trace segment
  uint64_t last_M1;    // max end+1 over placed layers before it in the segment
  uint64_t run_M1;     // max end+1 over all placed layers of the segment
  uint32_t c;          // placed layers (global count)
  uint32_t head;       // the range contains the first span of a trace
  uint32_t c_metric, c_lay, c_kl, c_ex;
};
static_assert(sizeof(Full) == 48, "Full layout");

__device__ __forceinline__ uint64_t max64(uint64_t a, uint64_t b) { return a > b ? a : b; }

__device__ __forceinline__ Full full_combine(const Full& a, const Full& b) {
  Full r;
  r.c = a.c + b.c;
  r.head = a.head | b.head;
  r.c_metric = a.c_metric + b.c_metric;
  r.c_lay = a.c_lay + b.c_lay;
  r.c_kl = a.c_kl + b.c_kl;
  r.c_ex = a.c_ex + b.c_ex;
  if (b.head) {
    r.last_end1 = b.last_end1;
    r.last_M1 = b.last_M1;
    r.run_M1 = b.run_M1;
  } else if (b.last_end1) {
    r.last_end1 = b.last_end1;
    r.last_M1 = max64(a.run_M1, b.last_M1);
    r.run_M1 = max64(a.run_M1, b.run_M1);
  } else {
    r.last_end1 = a.last_end1;
    r.last_M1 = a.last_M1;
    r.run_M1 = a.run_M1;
  }
  return r;
}

__device__ __forceinline__ Full full_identity() {
  Full f;
  f.last_end1 = f.last_M1 = f.run_M1 = 0;
  f.c = f.head = f.c_metric = f.c_lay = f.c_kl = f.c_ex = 0;
  return f;
}

__device__ __forceinline__ Full shfl_full(const Full& v, int src) {
  Full u;
  const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
  uint32_t* d = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
  for (int w = 0; w < 12; ++w) d[w] = __shfl_sync(0xffffffffu, s[w], src);
  return u;
}

// Pass-1 work decomposition: a tile of P1_TILE timeline-consecutive spans per
// CTA, 8 consecutive spans per thread. Pass 1 is reduce-then-scan (no
// decoupled look-back: a look-back makes every tile wait for the slowest of its
// recent predecessors, which measured a third of the kernel's time):
//   k_p1_reduce  per tile, each thread folds its 8 spans serially into a Full;
//                a warp scan + block combine gives the tile aggregate (reads
//                flags, begin, end, parent_id);
//   k_p1_scan    one CTA: exclusive scan over groups of 32 tile aggregates;
//   k_pass1      per tile, the tile is staged into shared memory by TMA, the
//                thread folds are recomputed, and every thread re-walks its
//                spans from its exclusive prefix emitting outputs with plain
//                counters.
// Code size matters: the fully unrolled 8-span walks put k_pass1 at ~5.7 K SASS
// instructions and ncu attributed 30% of its warp samples to stall_no_inst
// (instruction fetch). The rarely taken general fold and the emit walk are
// unrolled by pairs only.
#ifndef XSP_P1_SLOW_UNROLL
#define XSP_P1_SLOW_UNROLL 1
#endif
#ifndef XSP_P1_EMIT_UNROLL
#define XSP_P1_EMIT_UNROLL 1
#endif
constexpr int kP1SlowUnroll = XSP_P1_SLOW_UNROLL;
constexpr int kP1EmitUnroll = XSP_P1_EMIT_UNROLL;
#ifndef XSP_P1_WARPS
#define XSP_P1_WARPS 8
#endif
constexpr int P1_WARPS = XSP_P1_WARPS;
constexpr int P1_THREADS = P1_WARPS * 32;
constexpr int P1_ITEMS = 8;
constexpr int P1_SUB = P1_ITEMS * 32;  // spans per warp
constexpr int P1_TILE = P1_WARPS * P1_SUB;
constexpr int P1_ROWS = P1_TILE / 16;  // 128-byte rows of 16 u64 per column
static_assert(P1_TILE % 128 == 0, "swizzled columns need 1024-byte aligned bases");
static_assert(P1_ROWS <= 256, "TMA box rows");
constexpr int P1_TCACHE = 32;          // traces of a tile cached in shared memory
constexpr int P1_SCAN_THREADS = 1024;

struct P1Args {
  int bulk;     // full tiles staged by TMA tensor copies (columns 16-byte aligned)
  int parents_only;
  const uint64_t* span_id;
  const uint8_t* flags;
  const uint64_t* begin;
  const uint64_t* end;
  const uint64_t* parent;
  const uint64_t* cid;
  uint64_t n;
  const uint64_t* off;
  uint32_t T;
  const uint32_t* levels;
  const uint32_t* model_row;
  const uint64_t* mb;
  const uint64_t* me;
  const uint64_t* msid;
  const uint32_t* tile_lo;  // trace of each tile's first span (k_trace_prep / k_tile_traces)
  const uint32_t* tile_hi;  // trace of each tile's last span
  uint32_t ntiles;
  Full* tile_agg;           // [ntiles] (k_p1_reduce)
  Full* group_sum;          // [ngroups] totals of 32-tile groups (k_p1_reduce)
  uint32_t* group_done;     // [ngroups] finished tiles per group (zeroed per call)
  Full* tile_prefix;        // [ngroups + 1] exclusive prefixes of 32-tile groups + total (k_p1_scan)
  Full* tile_excl;          // [ntiles] exclusive prefix of every tile (k_p1_tile_prefix)
  Full* warp_excl;          // [ntiles * P1_WARPS] exclusive prefix of every warp within its tile
  uint8_t* placed8;         // [n / 8] bit k of byte q: span 8q + k is a placed layer (k_p1_reduce)
  uint32_t* unsorted;
  unsigned long long* err_key;
  uint32_t* layer_row;
  uint64_t* layer_dur;
  uint32_t* layer_attr_row;
  KlEnt* kl;
  uint32_t* kl_mrow;  // synchronous kernels only
  ExEnt* ex;
  uint32_t* t_layer_off;
  uint32_t* t_kl_off;
  uint32_t* t_ex_off;
  Orphans orph;
  uint32_t* amb_kl;
  uint32_t* amb_gx;
  uint32_t* amb_count;
  uint32_t* pend_kl;
  uint32_t* pend_count;
  uint32_t amb_cap, pend_cap;  // list capacities (counts beyond them trigger a retry)
  // direct mode (k_pass1<true>, a clean-batch guess): pass 1 writes the kernel
  // table itself — launch r of a trace at its kernel-list position, exec r at its
  // exec-list position, which coincide when every trace is merge-aligned — and
  // records per trace the min / max of (cid - list position) over its launches
  // and execs (equal <=> the cids are one dense run shared by both lists)
  uint32_t *k_launch, *k_exec, *k_mrow, *k_name, *l_koff;
  uint64_t* k_dur;
  double* k_occ;
  const uint32_t* name;
  const double* occ;
  unsigned long long *t_dmin, *t_dmax;
  uint32_t* direct_fail;  // a kernel-list entry that is not a launch with a cid
};

// TMA descriptors of the four u64 columns, each viewed as a 2-D tensor of
// [n/16 rows][16 spans] and copied as 128-row boxes with the 128-byte swizzle.
struct P1Maps {
  CUtensorMap begin, end, cid, parent;
};

struct TraceCache {
  uint64_t off[P1_TCACHE + 1];
  uint64_t mb[P1_TCACHE], me[P1_TCACHE], msid[P1_TCACHE];
  uint32_t model_row[P1_TCACHE], levels[P1_TCACHE];
};

// Tile staging buffer (dynamic shared memory, 1024-byte aligned). The u64
// columns are stored in the TMA SWIZZLE_128B pattern: span j lives in row j/16,
// 16-byte chunk ((j/2) % 8) ^ (row % 8). A thread's 8 consecutive spans are four
// 16-byte chunks whose swizzled addresses fall in distinct banks across every
// quarter-warp, so the per-thread serial walk reads shared memory conflict-free.
struct TileSmem {
  uint64_t begin[P1_TILE];
  uint64_t end[P1_TILE];
  uint64_t cid[P1_TILE];
  uint8_t flags[P1_TILE];
};
constexpr size_t P1_SMEM = sizeof(TileSmem) + 1024;  // + alignment slack
// resident CTAs per SM the register budget is sized for (shared memory bound)
constexpr int P1_MINB = (int)((220u * 1024u) / (P1_SMEM + 2048u)) < 8 ? (int)((220u * 1024u) / (P1_SMEM + 2048u)) : 8;

__host__ __device__ __forceinline__ uint32_t sw128(uint32_t j) {
  return (j & ~15u) | (((((j >> 1) & 7u) ^ ((j >> 4) & 7u))) << 1) | (j & 1u);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_g2s_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// two consecutive spans (j even) of a swizzled column
__device__ __forceinline__ void ld_pair(const uint64_t* col, uint32_t j, uint64_t& v0, uint64_t& v1) {
  const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(col + sw128(j));
  v0 = p.x;
  v1 = p.y;
}
__device__ __forceinline__ ulonglong2 ldg_nc_v2(const uint64_t* p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

// Per-trace attributes a thread needs while walking its spans.
struct TraceAttrs {
  uint64_t cur, next;  // offsets of the current trace and the one after it
  uint64_t mb, me, msid;
  uint32_t model, levels;
};

// The tile's traces [tlo, thi): attributes of the first P1_TCACHE of them are
// cached in shared memory; the rest are read from global memory.
struct TileTraces {
  const P1Args& a;
  const TraceCache& tc;
  uint32_t tlo;
  bool cached;
  __device__ __forceinline__ uint64_t off(uint32_t r) const { return cached ? tc.off[r] : __ldg(a.off + tlo + r); }
  __device__ __forceinline__ void load(uint32_t r, TraceAttrs& ta) const {
    ta.cur = off(r);
    ta.next = off(r + 1);
    if (cached) {
      ta.mb = tc.mb[r];
      ta.me = tc.me[r];
      ta.msid = tc.msid[r];
      ta.model = tc.model_row[r];
      ta.levels = tc.levels[r];
    } else {
      const uint32_t t = tlo + r;
      ta.mb = __ldg(a.mb + t);
      ta.me = __ldg(a.me + t);
      ta.msid = __ldg(a.msid + t);
      ta.model = __ldg(a.model_row + t);
      ta.levels = __ldg(a.levels + t);
    }
  }
  // trace (relative to tlo) of span i of the tile
  __device__ __forceinline__ uint32_t find(uint64_t i, uint32_t thi) const {
    uint32_t lo = 0, hi = thi - tlo;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (off(mid) <= i) lo = mid; else hi = mid;
    }
    return lo;
  }
};

__device__ __forceinline__ void fill_trace_cache(const P1Args& a, TraceCache& tc, uint32_t tlo, uint32_t thi) {
  const uint32_t ncache = min(thi - tlo, (uint32_t)P1_TCACHE);
  if (threadIdx.x <= ncache) tc.off[threadIdx.x] = a.off[tlo + threadIdx.x];
  if (threadIdx.x < ncache) {
    const uint32_t t = tlo + threadIdx.x;
    tc.mb[threadIdx.x] = a.mb[t];
    tc.me[threadIdx.x] = a.me[t];
    tc.msid[threadIdx.x] = a.msid[t];
    tc.model_row[threadIdx.x] = a.model_row[t];
    tc.levels[threadIdx.x] = a.levels[t];
  }
}

// layer placement under the model span (correlator.cpp:169-194)
__device__ __forceinline__ bool placed_in(const TraceAttrs& ta, uint8_t f, uint64_t b, uint64_t e, uint64_t par) {
  if (ta.model == kNone) return false;
  if (f & XSP_F_PARENT) return par == ta.msid;
  return ta.mb <= b && e <= ta.me;
}

// Phase 1: the Full aggregate of a thread's P1_ITEMS consecutive spans starting
// at global row i0 (local index j0 of a tile of tile_n spans). ld(p, b[2], e[2],
// par[2], f0, f1) yields spans 2p and 2p+1; parent_id is only needed (and only
// read) for spans with XSP_F_PARENT.
// Byte-parallel (SWAR) role masks of 8 flags bytes: bit k = predicate of span k.
__device__ __forceinline__ uint32_t byte_mask_eq(uint64_t fl8, uint32_t and_mask, uint32_t value) {
  const uint32_t lo = __vcmpeq4((uint32_t)fl8 & and_mask, value);
  const uint32_t hi = __vcmpeq4((uint32_t)(fl8 >> 32) & and_mask, value);
  const uint64_t m = ((uint64_t)hi << 32 | lo) & 0x0101010101010101ull;
  return (uint32_t)((m * 0x0102040810204080ull) >> 56);  // gather bit 0 of every byte
}
struct RoleMasks {
  uint32_t layer, layer_sync, metric, kl, ex_cid;
};
// Roles (xsp_common.cuh): layer = level 1; layer_sync = layer + kind Sync;
// kl = is_kernel_launch (kind Launch, level >= Kernel) or is_sync_kernel
// (kind Sync, level Kernel); ex_cid = is_exec with a correlation id.
__device__ __forceinline__ RoleMasks role_masks(uint64_t fl8) {
  RoleMasks m;
  m.layer = byte_mask_eq(fl8, 0x03030303u, 0x01010101u);
  m.layer_sync = byte_mask_eq(fl8, 0x0F0F0F0Fu, 0x01010101u);
  m.metric = byte_mask_eq(fl8, 0x40404040u, 0x40404040u);
  m.kl = byte_mask_eq(fl8, 0x0E0E0E0Eu, 0x06060606u) | byte_mask_eq(fl8, 0x0F0F0F0Fu, 0x02020202u);
  m.ex_cid = byte_mask_eq(fl8, 0x2C2C2C2Cu, 0x28282828u);
  return m;
}

// kHaveMask: the placement of the thread's layer spans is given by pmask (bit k
// = span k is a placed layer, computed by k_p1_reduce), so parent_id is not
// needed; otherwise placement is computed and recorded in pmask.
template <bool kHaveMask, typename Load>
__device__ __forceinline__ Full fold_thread(const TileTraces& tt, uint32_t r0, uint64_t i0, uint32_t j0,
                                            uint32_t tile_n, uint64_t fl8, uint32_t& pmask, Load ld) {
  Full th = full_identity();
  TraceAttrs ta;
  uint32_t r = r0;
  tt.load(r, ta);
  if (j0 + P1_ITEMS <= tile_n && ta.cur < i0 && ta.next >= i0 + P1_ITEMS) {
    // fast path: 8 spans inside one trace, no trace head among them. Counts
    // from the flag bytes; only layer/sync spans touch the containment state.
    const RoleMasks m = role_masks(fl8);
    th.c_lay = __popc(m.layer);
    th.c_metric = __popc(m.metric);
    th.c_kl = __popc(m.kl);
    th.c_ex = __popc(m.ex_cid);
    if (m.layer_sync) {
#pragma unroll
      for (int p = 0; p < P1_ITEMS / 2; ++p) {
        if (!((m.layer_sync >> (2 * p)) & 3u)) continue;
        uint64_t bb[2], ee[2], pp[2];
        ld(p, bb, ee, pp, (uint8_t)(fl8 >> (16 * p)), (uint8_t)(fl8 >> (16 * p + 8)));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = 2 * p + h;
          const uint8_t f = (uint8_t)(fl8 >> (8 * k));
          bool placed;
          if constexpr (kHaveMask) {
            placed = (pmask >> k) & 1u;
          } else {
            placed = ((m.layer_sync >> k) & 1u) && placed_in(ta, f, bb[h], ee[h], pp[h]);
            pmask |= (uint32_t)placed << k;
          }
          if (placed) {
            const uint64_t e = ee[h];
            const uint64_t w = e == ~0ull ? e : e + 1;
            th.last_M1 = th.run_M1;
            th.last_end1 = w;
            th.run_M1 = max64(th.run_M1, w);
            ++th.c;
          }
        }
      }
    }
    return th;
  }
#pragma unroll kP1SlowUnroll
  for (int p = 0; p < P1_ITEMS / 2; ++p) {
    uint64_t bb[2], ee[2], pp[2];
    ld(p, bb, ee, pp, (uint8_t)(fl8 >> (16 * p)), (uint8_t)(fl8 >> (16 * p + 8)));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 2 * p + h;
      const uint64_t i = i0 + k;
      if (j0 + k >= tile_n) continue;
      const uint8_t f = (uint8_t)(fl8 >> (8 * k));
      if (i >= ta.next) {
        do { ++r; } while (tt.off(r + 1) <= i);
        tt.load(r, ta);
      }
      if (ta.cur == i) {  // trace head: new segment
        th.head = 1;
        th.last_end1 = th.last_M1 = th.run_M1 = 0;
      }
      const bool is_layer = f_level(f) == XSP_LEVEL_LAYER;
      const uint64_t e = ee[h];
      bool placed;
      if constexpr (kHaveMask) {
        placed = (pmask >> k) & 1u;
      } else {
        placed = is_layer && f_kind(f) == XSP_KIND_SYNC && placed_in(ta, f, bb[h], e, pp[h]);
        pmask |= (uint32_t)placed << k;
      }
      if (placed) {
        const uint64_t w = e == ~0ull ? e : e + 1;
        th.last_M1 = th.run_M1;
        th.last_end1 = w;
        th.run_M1 = max64(th.run_M1, w);
        ++th.c;
      }
      th.c_lay += is_layer;
      th.c_metric += (f & XSP_F_METRICS) != 0;
      th.c_kl += is_kernel_launch(f) || is_sync_kernel(f);
      th.c_ex += is_exec(f) && (f & XSP_F_CID);
    }
  }
  return th;
}

__device__ __forceinline__ Full warp_inclusive(const Full& th, uint32_t lane) {
  Full inc = th;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Full u;
    const uint32_t* s = reinterpret_cast<const uint32_t*>(&inc);
    uint32_t* d = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int w = 0; w < 12; ++w) d[w] = __shfl_up_sync(0xffffffffu, s[w], o);
    if (lane >= (uint32_t)o) inc = full_combine(u, inc);
  }
  return inc;
}

// The same inclusive scan for thread folds of one warp (lane = sequence order,
// every count < 2^16), built from ballots instead of 5 rounds of 12-word
// shuffles + full_combine. Lane l's inclusive prefix over lanes [0, l]:
//   s = last lane <= l whose fold holds a trace head (the segment start),
//   j = last lane in [s, l] whose fold placed a layer;
//   last_end1 = fold_j.last_end1, last_M1 = max(fold_j.last_M1, run over [s, j)),
//   run_M1 = run over [s, l] (a segmented max-scan), counts = add-scans.
// This is exactly the left fold of full_combine over the lanes.
__device__ __forceinline__ Full warp_inclusive_fold(const Full& th, uint32_t lane) {
  const uint32_t le = 0xffffffffu >> (31u - lane);
  const uint32_t H = __ballot_sync(0xffffffffu, th.head != 0) & le;
  const uint32_t L = __ballot_sync(0xffffffffu, th.last_end1 != 0) & le;
  const int s = H ? 31 - __clz(H) : -1;
  const int s0 = s < 0 ? 0 : s;
  uint32_t p0 = th.c | (th.c_metric << 16), p1 = th.c_lay | (th.c_kl << 16), p2 = th.c_ex;
  uint64_t R = th.run_M1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u0 = __shfl_up_sync(0xffffffffu, p0, o);
    const uint32_t u1 = __shfl_up_sync(0xffffffffu, p1, o);
    const uint32_t u2 = __shfl_up_sync(0xffffffffu, p2, o);
    const uint64_t uR = __shfl_up_sync(0xffffffffu, R, o);
    if (lane >= (uint32_t)o) {
      p0 += u0;
      p1 += u1;
      p2 += u2;
      if ((int)lane - o >= s0) R = max64(R, uR);
    }
  }
  const uint32_t Ls = s > 0 ? (L & ~((1u << s) - 1u)) : L;  // layer lanes in [s, l]
  const int j = Ls ? 31 - __clz(Ls) : -1;
  const uint64_t le_j = __shfl_sync(0xffffffffu, th.last_end1, j >= 0 ? j : 0);
  const uint64_t lm_j = __shfl_sync(0xffffffffu, th.last_M1, j >= 0 ? j : 0);
  const uint64_t r_j1 = __shfl_sync(0xffffffffu, R, j >= 1 ? j - 1 : 0);
  Full r;
  r.c = p0 & 0xFFFFu;
  r.c_metric = p0 >> 16;
  r.c_lay = p1 & 0xFFFFu;
  r.c_kl = p1 >> 16;
  r.c_ex = p2;
  r.head = s >= 0;
  r.run_M1 = R;
  r.last_end1 = j >= 0 ? le_j : 0;
  r.last_M1 = j >= 0 ? max64(lm_j, j - 1 >= s0 ? r_j1 : 0) : 0;
  return r;
}

// Tile header shared by the reduce and emit kernels.
struct TileHdr {
  uint64_t tile_base;
  uint32_t tile_n, tlo, thi;
};
__device__ __forceinline__ TileHdr tile_hdr(const P1Args& a, uint32_t tile) {
  TileHdr h;
  h.tile_base = (uint64_t)tile * P1_TILE;
  h.tile_n = (uint32_t)min((uint64_t)P1_TILE, a.n - h.tile_base);
  h.tlo = __ldg(a.tile_lo + tile);
  h.thi = __ldg(a.tile_hi + tile) + 1;
  return h;
}

__device__ __forceinline__ Full warp_reduce_ordered(Full v, uint32_t lane) {
  // result in lane 0; lane order = sequence order
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Full u;
    const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
    uint32_t* d = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int w = 0; w < 12; ++w) d[w] = __shfl_down_sync(0xffffffffu, s[w], o);
    if ((lane & (2 * o - 1)) == 0) v = full_combine(v, u);
  }
  return v;
}

// L2 load of a Full written by another CTA of this grid (bypasses L1)
__device__ __forceinline__ Full ld_full_cg(const Full* p) {
  Full v;
  const uint4* s = reinterpret_cast<const uint4*>(p);
  uint32_t* d = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const uint4 w = __ldcg(s + q);
    d[4 * q] = w.x; d[4 * q + 1] = w.y; d[4 * q + 2] = w.z; d[4 * q + 3] = w.w;
  }
  return v;
}

// ---- k_p1_reduce: tile aggregates (tile staged by TMA) ---------------
// Reduce staging buffer: the three u64 columns the fold reads (TMA, 128-byte
// swizzle as in TileSmem) and the flag bytes.
struct RedSmem {
  uint64_t begin[P1_TILE];
  uint64_t end[P1_TILE];
  uint64_t parent[P1_TILE];
  uint8_t flags[P1_TILE];
};
constexpr size_t P1_RED_SMEM = sizeof(RedSmem) + 1024;

__global__ void __launch_bounds__(P1_THREADS) k_p1_reduce(P1Args a, const __grid_constant__ P1Maps maps) {
  extern __shared__ unsigned char red_dyn[];
  RedSmem& sm = *reinterpret_cast<RedSmem*>(red_dyn + ((1024u - (smem_u32(red_dyn) & 1023u)) & 1023u));
  __shared__ TraceCache tc;
  __shared__ Full s_wagg[P1_WARPS];
  __shared__ __align__(8) uint64_t s_bar;
  const uint32_t tile = blockIdx.x, warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t j0 = threadIdx.x * P1_ITEMS;
  const uint64_t tile_base = (uint64_t)tile * P1_TILE;
  const uint32_t tile_n = (uint32_t)min((uint64_t)P1_TILE, a.n - tile_base);
  const uint64_t i0 = tile_base + j0;
  const bool bulk = a.bulk && tile_n == P1_TILE;
  if (threadIdx.x == 0 && bulk) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&s_bar, P1_TILE * (3 * 8 + 1));
    const int y = (int)(tile_base / 16);
    tma_g2s_2d(sm.begin, &maps.begin, 0, y, &s_bar);
    tma_g2s_2d(sm.end, &maps.end, 0, y, &s_bar);
    tma_g2s_2d(sm.parent, &maps.parent, 0, y, &s_bar);
    bulk_g2s(sm.flags, a.flags + tile_base, P1_TILE, &s_bar);
  }
  if (!bulk) {
    for (uint32_t j = threadIdx.x; j < P1_TILE; j += P1_THREADS) {
      const bool v = j < tile_n;
      const uint64_t i = tile_base + j;
      const uint32_t sw = sw128(j);
      sm.flags[j] = v ? a.flags[i] : (uint8_t)0xFF;
      sm.begin[sw] = v ? a.begin[i] : 0;
      sm.end[sw] = v ? a.end[i] : 0;
      sm.parent[sw] = v ? a.parent[i] : 0;
    }
  }
  const uint32_t tlo = __ldg(a.tile_lo + tile), thi = __ldg(a.tile_hi + tile) + 1;
  fill_trace_cache(a, tc, tlo, thi);
  __syncthreads();
  if (bulk) mbar_wait(&s_bar, 0);
  const TileTraces tt{a, tc, tlo, thi - tlo <= (uint32_t)P1_TCACHE};
  Full th = full_identity();
  if (j0 < tile_n) {
    const uint32_t r0 = tt.find(i0, thi);
    const uint64_t fl8 = *reinterpret_cast<const uint64_t*>(sm.flags + j0);
    uint32_t pmask = 0;
    th = fold_thread<false>(tt, r0, i0, j0, tile_n, fl8, pmask,
                     [&](int p, uint64_t (&bb)[2], uint64_t (&ee)[2], uint64_t (&pp)[2], uint8_t, uint8_t) {
                       ld_pair(sm.begin, j0 + 2 * p, bb[0], bb[1]);
                       ld_pair(sm.end, j0 + 2 * p, ee[0], ee[1]);
                       ld_pair(sm.parent, j0 + 2 * p, pp[0], pp[1]);
                     });
    a.placed8[i0 >> 3] = (uint8_t)pmask;
  }
  const Full inc = warp_inclusive_fold(th, lane);
  if (lane == 31) s_wagg[warp] = inc;
  __syncthreads();
  if (warp != 0) return;
  uint32_t last = 0;
  if (lane < P1_WARPS) {
    // exclusive prefix of every warp within the tile: k_pass1's warps start
    // from it without waiting for each other
    Full ex = full_identity();
    for (uint32_t w = 0; w < lane; ++w) ex = full_combine(ex, s_wagg[w]);
    a.warp_excl[(uint64_t)tile * P1_WARPS + lane] = ex;
  }
  if (lane == 0) {
    Full agg = s_wagg[0];
    for (int w = 1; w < P1_WARPS; ++w) agg = full_combine(agg, s_wagg[w]);
    a.tile_agg[tile] = agg;
    // the last tile of a 32-tile group to finish reduces the group
    __threadfence();
    const uint32_t g = tile >> 5, gsize = min(32u, a.ntiles - (g << 5));
    last = atomicAdd(a.group_done + g, 1u) == gsize - 1;
  }
  if (__shfl_sync(0xffffffffu, last, 0)) {
    __threadfence();
    const uint32_t g = tile >> 5, k = (g << 5) + lane;
    const Full v = warp_reduce_ordered(k < a.ntiles ? ld_full_cg(a.tile_agg + k) : full_identity(), lane);
    if (lane == 0) a.group_sum[g] = v;
  }
}

// ---- k_p1_scan: exclusive prefixes of the 32-tile group totals -------------
// One CTA. The group totals come from k_p1_reduce (the last tile of each group
// to finish reduces the group); a block scan gives gprefix[g] (exclusive) and
// gprefix[ngroups] = the grand total. k_pass1 finishes a tile's prefix with one
// warp reduction over the <= 31 preceding tiles of its group.
__global__ void __launch_bounds__(P1_SCAN_THREADS) k_p1_scan(const Full* __restrict__ gsum, uint32_t ngroups,
                                                             Full* __restrict__ gprefix) {
  __shared__ Full s_w[P1_SCAN_THREADS / 32];
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t per = (ngroups + P1_SCAN_THREADS - 1) / P1_SCAN_THREADS;
  const uint32_t lo = min(ngroups, threadIdx.x * per), hi = min(ngroups, lo + per);
  Full th = full_identity();
  for (uint32_t k = lo; k < hi; ++k) th = full_combine(th, gsum[k]);
  const Full inc = warp_inclusive(th, lane);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) s_w[lane] = warp_inclusive(s_w[lane], lane);  // inclusive over warps
  __syncthreads();
  Full run = warp > 0 ? s_w[warp - 1] : full_identity();
  {
    Full ex;
    const uint32_t* s = reinterpret_cast<const uint32_t*>(&inc);
    uint32_t* d = reinterpret_cast<uint32_t*>(&ex);
#pragma unroll
    for (int w = 0; w < 12; ++w) d[w] = __shfl_up_sync(0xffffffffu, s[w], 1);
    if (lane > 0) run = full_combine(run, ex);
  }
  for (uint32_t k = lo; k < hi; ++k) {
    gprefix[k] = run;
    run = full_combine(run, gsum[k]);
  }
  if (threadIdx.x == P1_SCAN_THREADS - 1) gprefix[ngroups] = s_w[31];
}

// ---- k_p1_tile_prefix: exclusive prefix of every tile (one warp per tile) ---
// group prefix + ordered reduction over the preceding tiles of the group.
__global__ void k_p1_tile_prefix(const Full* __restrict__ agg, const Full* __restrict__ gprefix, uint32_t ntiles,
                                 Full* __restrict__ excl) {
  const uint32_t tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = lane_id();
  if (tile >= ntiles) return;
  const uint32_t gbase = tile & ~31u;
  const Full v = warp_reduce_ordered(gbase + lane < tile ? agg[gbase + lane] : full_identity(), lane);
  if (lane == 0) excl[tile] = full_combine(gprefix[tile >> 5], v);
}

// ---- k_pass1: per-span outputs ----------------------------------------------
// Per-trace min / max with atomics, warp-aggregated when every lane holding a
// value (t != kNone) has the same trace (one atomic pair per warp), else per lane.
__device__ __forceinline__ void minmax_atomic_warp(uint32_t t, uint64_t mn, uint64_t mx,
                                                   unsigned long long* __restrict__ dmin,
                                                   unsigned long long* __restrict__ dmax) {
  const uint32_t act = __activemask();
  if (act == 0xffffffffu) {
    const uint32_t has = __ballot_sync(act, t != kNone);
    if (!has) return;
    const uint32_t t0 = __shfl_sync(act, t, __ffs(has) - 1);
    if (__ballot_sync(act, t == t0 || t == kNone) == act) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t b0 = __shfl_xor_sync(act, mn, o), b1 = __shfl_xor_sync(act, mx, o);
        mn = b0 < mn ? b0 : mn;
        mx = b1 > mx ? b1 : mx;
      }
      if (lane_id() == 0) {  // skip atomics that cannot change the value (one hot word per long trace)
        if (mn < *((volatile unsigned long long*)(dmin + t0))) atomicMin(dmin + t0, (unsigned long long)mn);
        if (mx > *((volatile unsigned long long*)(dmax + t0))) atomicMax(dmax + t0, (unsigned long long)mx);
      }
      return;
    }
  }
  if (t != kNone) {
    if (mn < *((volatile unsigned long long*)(dmin + t))) atomicMin(dmin + t, (unsigned long long)mn);
    if (mx > *((volatile unsigned long long*)(dmax + t))) atomicMax(dmax + t, (unsigned long long)mx);
  }
}

// Per-trace min / max of (cid - list position) in direct mode: a thread keeps
// the run of its current trace and flushes it with atomics; the final runs of a
// warp whose lanes share one trace are reduced first (one atomic pair per warp).
struct DirectAcc {
  uint64_t mn = ~0ull, mx = 0;
  uint32_t t = kNone;
  __device__ __forceinline__ void flush(const P1Args& a) {
    if (t != kNone) {
      atomicMin(a.t_dmin + t, (unsigned long long)mn);
      atomicMax(a.t_dmax + t, (unsigned long long)mx);
    }
    mn = ~0ull;
    mx = 0;
    t = kNone;
  }
  __device__ __forceinline__ void add(const P1Args& a, uint32_t tr, uint64_t d) {
    if (tr != t) {
      flush(a);
      t = tr;
    }
    mn = d < mn ? d : mn;
    mx = d > mx ? d : mx;
  }
  __device__ __forceinline__ void finish(const P1Args& a) { minmax_atomic_warp(t, mn, mx, a.t_dmin, a.t_dmax); }
};

template <bool kDirect>
__global__ void __launch_bounds__(P1_THREADS, P1_MINB) k_pass1(P1Args a, const __grid_constant__ P1Maps maps) {
  extern __shared__ unsigned char p1_dyn[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(p1_dyn + ((1024u - (smem_u32(p1_dyn) & 1023u)) & 1023u));
  __shared__ TraceCache tc;
  __shared__ __align__(8) uint64_t s_bar;

  const uint32_t tile = blockIdx.x, warp = threadIdx.x >> 5, lane = lane_id();
  const TileHdr hd = tile_hdr(a, tile);
  const uint64_t tile_base = hd.tile_base;
  const uint32_t tile_n = hd.tile_n, tlo = hd.tlo, thi = hd.thi;
  const bool bulk = a.bulk && tile_n == P1_TILE;
  if (threadIdx.x == 0 && bulk) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&s_bar, P1_TILE * (3 * 8 + 1));
    const int y = (int)(tile_base / 16);
    tma_g2s_2d(sm.begin, &maps.begin, 0, y, &s_bar);
    tma_g2s_2d(sm.end, &maps.end, 0, y, &s_bar);
    tma_g2s_2d(sm.cid, &maps.cid, 0, y, &s_bar);
    bulk_g2s(sm.flags, a.flags + tile_base, P1_TILE, &s_bar);
  }
  fill_trace_cache(a, tc, tlo, thi);
  const Full tile_pre = a.tile_excl[tile];
  const Full warp_pre = a.warp_excl[(uint64_t)tile * P1_WARPS + warp];
  if (!bulk) {
    for (uint32_t j = threadIdx.x; j < P1_TILE; j += P1_THREADS) {
      const bool v = j < tile_n;
      const uint64_t i = tile_base + j;
      const uint32_t s = sw128(j);
      sm.flags[j] = v ? a.flags[i] : (uint8_t)0xFF;
      sm.begin[s] = v ? a.begin[i] : 0;
      sm.end[s] = v ? a.end[i] : 0;
      sm.cid[s] = v ? a.cid[i] : 0;
    }
  }
  __syncthreads();
  if (bulk) mbar_wait(&s_bar, 0);
  const TileTraces tt{a, tc, tlo, thi - tlo <= (uint32_t)P1_TCACHE};
  const uint32_t j0 = threadIdx.x * P1_ITEMS;  // thread's first local index
  const uint64_t i0 = tile_base + j0;
  uint32_t r0 = 0;
  if (j0 < tile_n) r0 = tt.find(i0, thi);
  const uint64_t fl8 = *reinterpret_cast<const uint64_t*>(sm.flags + j0);
  uint32_t pmask = j0 < tile_n ? a.placed8[i0 >> 3] : 0u;

  // ---- phase 1 (recomputed from shared memory): thread fold + warp scan
  Full lane_ex;  // exclusive prefix of the thread within its warp
  {
    const Full th = j0 < tile_n ? fold_thread<true>(tt, r0, i0, j0, tile_n, fl8, pmask,
                                                    [&](int p, uint64_t (&bb)[2], uint64_t (&ee)[2],
                                                        uint64_t (&pp)[2], uint8_t, uint8_t) {
                                                      ld_pair(sm.begin, j0 + 2 * p, bb[0], bb[1]);
                                                      ld_pair(sm.end, j0 + 2 * p, ee[0], ee[1]);
                                                      pp[0] = pp[1] = 0;
                                                    })
                                : full_identity();
    const Full inc = warp_inclusive_fold(th, lane);
    const uint32_t* s = reinterpret_cast<const uint32_t*>(&inc);
    uint32_t* d = reinterpret_cast<uint32_t*>(&lane_ex);
#pragma unroll
    for (int w = 0; w < 12; ++w) d[w] = __shfl_up_sync(0xffffffffu, s[w], 1);
    if (lane == 0) lane_ex = full_identity();
  }
  // tile prefix + the warps before this one (k_p1_reduce): no CTA barrier
  Full carry = full_combine(full_combine(tile_pre, warp_pre), lane_ex);

  // ---- phase 3: per-span outputs (serial over the thread's 8 spans) ----------
  if (j0 >= tile_n) return;
  TraceAttrs ta;
  uint32_t r = r0;
  tt.load(r, ta);
  uint32_t g = carry.c, c_metric = carry.c_metric, c_lay = carry.c_lay, c_kl = carry.c_kl, c_ex = carry.c_ex;
  uint64_t lastE = carry.last_end1, lastM = carry.last_M1, runM = carry.run_M1;
  // predecessor of the first span, for the timeline-order check
  uint64_t pb = 0;
  uint8_t pf = 0;
  if (i0 > 0) {
    pb = j0 > 0 ? sm.begin[sw128(j0 - 1)] : __ldg(a.begin + i0 - 1);
    pf = j0 > 0 ? sm.flags[j0 - 1] : __ldg(a.flags + i0 - 1);
  }
  DirectAcc dacc;
  // Fast emit: the 8 spans lie inside one trace with no trace head, no model
  // span, and the trace profiles the layer level. The roles come from the flag
  // bytes as bit masks and each output list is filled by walking its mask in
  // span order (the same entries, positions and counters as the general walk).
  if (j0 + P1_ITEMS <= tile_n && ta.cur < i0 && ta.next >= i0 + P1_ITEMS &&
      (ta.levels & (1u << XSP_LEVEL_LAYER)) && !byte_mask_eq(fl8, 0x0F0F0F0Fu, 0u)) {
    const uint32_t t = tlo + r;
    // timeline order (begin_ns, rank, span_id) within the trace (span.hpp:161-163)
    bool bad = false;
#pragma unroll
    for (int k = 0; k < P1_ITEMS; ++k) {
      const uint64_t b = sm.begin[sw128(j0 + k)];
      const uint8_t f = (uint8_t)(fl8 >> (8 * k));
      if (pb >= b) {
        bool bk = pb > b;
        if (!bk) {
          const uint32_t l0 = f_level(pf), l1 = f_level(f);
          const uint32_t r0_ = l0 >= 2 ? 3 : l0 + 1, r1_ = l1 >= 2 ? 3 : l1 + 1;
          bk = r0_ > r1_ || (r0_ == r1_ && __ldg(a.span_id + i0 + k - 1) > __ldg(a.span_id + i0 + k));
        }
        bad |= bk;
      }
      pb = b;
      pf = f;
    }
    if (bad) atomicOr(a.unsorted, 1u);
    const RoleMasks m = role_masks(fl8);
    const uint32_t exec_m = byte_mask_eq(fl8, 0x0C0C0C0Cu, 0x08080808u);
    const uint32_t sync_k = byte_mask_eq(fl8, 0x0F0F0F0Fu, 0x02020202u);
    const uint32_t placed = pmask & m.layer_sync;
    // placed layers (in order, with the containment state) and kernel-list entries
    for (uint32_t ev = placed | m.kl; ev; ev &= ev - 1) {
      const int k = __ffs(ev) - 1;
      const uint32_t below = (1u << k) - 1u;
      const uint64_t i = i0 + k;
      const uint64_t e = sm.end[sw128(j0 + k)];
      if ((placed >> k) & 1u) {
        a.layer_row[g] = (uint32_t)i;
        a.layer_dur[g] = clamp_dur(sm.begin[sw128(j0 + k)], e);
        a.layer_attr_row[g] = c_lay + __popc(m.layer & below);
        if constexpr (kDirect) a.l_koff[g] = c_kl;  // kernels before it = the layer's first kernel
        ++g;
        const uint64_t w = e == ~0ull ? e : e + 1;
        lastM = runM;
        lastE = w;
        runM = max64(runM, w);
        continue;
      }
      const uint8_t f = (uint8_t)(fl8 >> (8 * k));
      const uint32_t k_ex = c_kl++;
      uint32_t par;
      if (f & XSP_F_PARENT) {
        par = PAR_PENDING;
        const uint32_t s = atomicAdd(a.pend_count, 1u);
        if (s < a.pend_cap) a.pend_kl[s] = k_ex;
      } else {
        const bool in_j = lastE > e;  // end_j >= e (ends stored +1)
        const bool in_m = lastM > e;  // an earlier layer has end >= e
        // e == UINT64_MAX: the saturated +1 encoding cannot tell end_j == e from
        // end_j == e - 1, so the exact rare path decides
        if (in_j && !in_m) {
          par = g - 1;
        } else if (!in_j && !in_m && e != ~0ull) {
          par = PAR_ORPHAN;
          emit_orphan(a.orph, t, CAT_KERNEL, i, (uint32_t)i, XSP_O_KERNEL_NO_LAYER);
        } else {
          par = PAR_AMBIG;
          const uint32_t s = atomicAdd(a.amb_count, 1u);
          if (s < a.amb_cap) {
            a.amb_kl[s] = k_ex;
            a.amb_gx[s] = g;
          }
        }
      }
      if constexpr (kDirect) {
        a.k_launch[k_ex] = (uint32_t)i;
        if (f_kind(f) == XSP_KIND_LAUNCH && (f & XSP_F_CID))
          dacc.add(a, t, sm.cid[sw128(j0 + k)] - k_ex);
        else
          *a.direct_fail = 1;
        (void)par;
      } else {
        KlEnt ent;
        ent.row = (uint32_t)i;
        ent.parent = par;
        ent.cid = (f & XSP_F_CID) ? sm.cid[sw128(j0 + k)] : 0;
        a.kl[k_ex] = ent;
        if ((sync_k >> k) & 1u) a.kl_mrow[k_ex] = ((m.metric >> k) & 1u) ? c_metric + __popc(m.metric & below) : kNone;
      }
    }
    // layers that are not placed (correlator.cpp:169-194)
    for (uint32_t lo = m.layer & ~placed; lo; lo &= lo - 1) {
      const int k = __ffs(lo) - 1;
      const uint8_t f = (uint8_t)(fl8 >> (8 * k));
      emit_orphan(a.orph, t, CAT_LAYER, i0 + k, (uint32_t)(i0 + k),
                  !((m.layer_sync >> k) & 1u)
                      ? XSP_O_LAYER_NON_SYNC
                      : ((f & XSP_F_PARENT) ? XSP_O_LAYER_BAD_PARENT : XSP_O_LAYER_OUTSIDE_MODEL));
    }
    // executions: with a cid into the exec list, without one an orphan
    for (uint32_t ex = exec_m; ex; ex &= ex - 1) {
      const int k = __ffs(ex) - 1;
      if ((m.ex_cid >> k) & 1u) {
        const uint32_t mr = ((m.metric >> k) & 1u) ? c_metric + __popc(m.metric & ((1u << k) - 1u)) : kNone;
        const uint64_t dur = clamp_dur(sm.begin[sw128(j0 + k)], sm.end[sw128(j0 + k)]);
        if constexpr (kDirect) {
          const uint32_t x = c_ex++;
          a.k_exec[x] = (uint32_t)(i0 + k);
          a.k_mrow[x] = mr;
          a.k_dur[x] = dur;
          a.k_name[x] = __ldg(a.name + i0 + k);
          a.k_occ[x] = mr != kNone ? __ldg(a.occ + mr) : 0.0;
          dacc.add(a, t, sm.cid[sw128(j0 + k)] - x);
        } else {
          ExEnt ent;
          ent.row = (uint32_t)(i0 + k);
          ent.mrow = mr;
          ent.dur = dur;
          a.ex[c_ex++] = ent;
        }
      } else if (!a.parents_only) {
        emit_orphan(a.orph, t, CAT_EXEC_NOCID, i0 + k, (uint32_t)(i0 + k), XSP_O_EXEC_NO_CID);
      }
    }
    if constexpr (kDirect) dacc.finish(a);
    return;
  }
#pragma unroll kP1EmitUnroll
  for (int p = 0; p < P1_ITEMS / 2; ++p) {
    uint64_t bb[2], ee[2], cc[2];
    ld_pair(sm.begin, j0 + 2 * p, bb[0], bb[1]);
    ld_pair(sm.end, j0 + 2 * p, ee[0], ee[1]);
    ld_pair(sm.cid, j0 + 2 * p, cc[0], cc[1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 2 * p + h;
      const uint64_t i = i0 + k;
      if (j0 + k >= tile_n) break;
      const uint8_t f = (uint8_t)(fl8 >> (8 * k));
      const uint64_t b = bb[h], e = ee[h];
      if (i >= ta.next) {
        do { ++r; } while (tt.off(r + 1) <= i);
        tt.load(r, ta);
      }
      const uint32_t t = tlo + r;
      const bool head = ta.cur == i;
      if (head) {
        lastE = lastM = runM = 0;
        int64_t tx = t;
        do {
          a.t_layer_off[tx] = g;
          a.t_kl_off[tx] = c_kl;
          a.t_ex_off[tx] = c_ex;
          --tx;
        } while (tx >= 0 && __ldg(a.off + tx) == i);
      } else if (i > 0 && pb >= b) {
        // timeline order (begin_ns, rank, span_id) within the trace (span.hpp:161-163)
        bool bad = pb > b;
        if (!bad) {
          const uint32_t l0 = f_level(pf), l1 = f_level(f);
          const uint32_t r0_ = l0 >= 2 ? 3 : l0 + 1, r1_ = l1 >= 2 ? 3 : l1 + 1;
          bad = r0_ > r1_ || (r0_ == r1_ && __ldg(a.span_id + i - 1) > __ldg(a.span_id + i));
        }
        if (bad) atomicOr(a.unsorted, 1u);
      }
      pb = b;
      pf = f;

      // trace errors raised while walking the bundle (correlator.cpp:146-158)
      // (the reference compares span ids: a second model span sharing the
      // model's span_id is not an error)
      if (is_model_span(f) && (uint32_t)i != ta.model && __ldg(a.span_id + i) != ta.msid)
        atomicMin(a.err_key + t, ((unsigned long long)i << 8) | XSP_T_MULTI_MODEL);
      if (f_level(f) >= XSP_LEVEL_KERNEL && !(ta.levels & (1u << XSP_LEVEL_LAYER)))
        atomicMin(a.err_key + t, ((unsigned long long)i << 8) | XSP_T_SKIP_LEVEL);

      const bool met = (f & XSP_F_METRICS) != 0;
      const uint32_t mrow = met ? c_metric : kNone;
      c_metric += met;
      if (f_level(f) == XSP_LEVEL_LAYER) {
        const bool layer_sync = f_kind(f) == XSP_KIND_SYNC;
        if (layer_sync && ((pmask >> k) & 1u)) {
          a.layer_row[g] = (uint32_t)i;
          a.layer_dur[g] = clamp_dur(b, e);
          a.layer_attr_row[g] = c_lay;
          if constexpr (kDirect) a.l_koff[g] = c_kl;
          ++g;
          const uint64_t w = e == ~0ull ? e : e + 1;
          lastM = runM;
          lastE = w;
          runM = max64(runM, w);
        } else {
          emit_orphan(a.orph, t, CAT_LAYER, i, (uint32_t)i,
                      !layer_sync ? XSP_O_LAYER_NON_SYNC
                                  : ((f & XSP_F_PARENT) ? XSP_O_LAYER_BAD_PARENT : XSP_O_LAYER_OUTSIDE_MODEL));
        }
        ++c_lay;
      }
      const bool sync = is_sync_kernel(f);
      const bool has_cid = (f & XSP_F_CID) != 0;
      if (is_kernel_launch(f) || sync) {
        const uint32_t k_ex = c_kl++;
        uint32_t par;
        if (f & XSP_F_PARENT) {
          par = PAR_PENDING;
          const uint32_t s = atomicAdd(a.pend_count, 1u);
          if (s < a.pend_cap) a.pend_kl[s] = k_ex;
        } else {
          const bool in_j = lastE > e;  // end_j >= e (ends stored +1)
          const bool in_m = lastM > e;  // an earlier layer has end >= e
          if (in_j && !in_m) {
            par = g - 1;
          } else if (!in_j && !in_m && e != ~0ull) {  // e == UINT64_MAX: exact rare path
            par = PAR_ORPHAN;
            emit_orphan(a.orph, t, CAT_KERNEL, i, (uint32_t)i, XSP_O_KERNEL_NO_LAYER);
          } else {
            // >= 2 candidates, or an earlier layer outlives j: exact rare path
            par = PAR_AMBIG;
            const uint32_t s = atomicAdd(a.amb_count, 1u);
            if (s < a.amb_cap) {
              a.amb_kl[s] = k_ex;
              a.amb_gx[s] = g;
            }
          }
        }
        if constexpr (kDirect) {
          a.k_launch[k_ex] = (uint32_t)i;
          if (f_kind(f) == XSP_KIND_LAUNCH && has_cid)
            dacc.add(a, t, cc[h] - k_ex);
          else
            *a.direct_fail = 1;
          (void)par;
        } else {
          KlEnt ent;
          ent.row = (uint32_t)i;
          ent.parent = par;
          ent.cid = has_cid ? cc[h] : 0;
          a.kl[k_ex] = ent;
          if (sync) a.kl_mrow[k_ex] = mrow;
        }
      }
      if (is_exec(f)) {
        if (has_cid) {
          if constexpr (kDirect) {
            const uint32_t x = c_ex++;
            a.k_exec[x] = (uint32_t)i;
            a.k_mrow[x] = mrow;
            a.k_dur[x] = clamp_dur(b, e);
            a.k_name[x] = __ldg(a.name + i);
            a.k_occ[x] = mrow != kNone ? __ldg(a.occ + mrow) : 0.0;
            dacc.add(a, t, cc[h] - x);
          } else {
            ExEnt ent;
            ent.row = (uint32_t)i;
            ent.mrow = mrow;
            ent.dur = clamp_dur(b, e);
            a.ex[c_ex++] = ent;
          }
        } else if (!a.parents_only) {
          emit_orphan(a.orph, t, CAT_EXEC_NOCID, i, (uint32_t)i, XSP_O_EXEC_NO_CID);
        }
      }
    }
  }
  if constexpr (kDirect) dacc.finish(a);
}

// Offsets of traces that start at or after the end of the span table (empty
// trailing traces) and the [T] sentinel.
__global__ void k_pass1_tail(const uint64_t* __restrict__ off, uint32_t T, uint64_t n,
                             const Full* __restrict__ tile_prefix, uint32_t ntiles,
                             uint32_t* t_layer_off, uint32_t* t_kl_off, uint32_t* t_ex_off,
                             uint32_t* totals) {
  const Full tot = ntiles ? tile_prefix[(ntiles + 31) / 32] : full_identity();
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= T; t += gridDim.x * blockDim.x) {
    if (off[t] >= n) {
      t_layer_off[t] = tot.c;
      t_kl_off[t] = tot.c_kl;
      t_ex_off[t] = tot.c_ex;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    totals[0] = tot.c;
    totals[1] = tot.c_kl;
    totals[2] = tot.c_ex;
    totals[3] = tot.c_metric;
    totals[4] = tot.c_lay;
  }
}

// Direct mode, everything after pass 1 in one launch: the trailing empty
// traces' offsets and the totals (k_pass1_tail), the merge-alignment check
// (a trace is merge-aligned iff it has as many
// execs with a cid as kernel-list entries and all of them share one (cid -
// position) value: then launch r and exec r carry the same cid, the cids
// increase strictly and none repeats — what the reference's hash join
// produces, correlator.cpp:287-364), the layer CSR sentinel, per-trace kernel offsets
// (k_trace_kernel_off) and trace status (k_status without duplicate cids: a
// merge-aligned batch has none). The values the host decides on — totals,
// counters, per-trace layer / kernel offsets — are stored straight into pinned
// host memory (device-addressable under UVA); the last block to finish copies
// the counters once every block's flags are in.
struct FinishArgs {
  const uint64_t* off;
  uint32_t T;
  uint64_t n;
  const Full* tile_prefix;
  uint32_t ntiles;
  uint32_t *t_layer_off, *t_kl_off, *t_ex_off;
  uint32_t* totals;
  const unsigned long long *dmin, *dmax;
  uint32_t* l_koff;
  uint32_t* t_koff;
  const uint32_t* model_row;
  const unsigned long long* err_key;
  int32_t* status;
  uint32_t* err_row;
  uint32_t* counters;  // [0..7] as in run_correlate_once, [8] finished blocks
  uint32_t* h_totals;  // pinned: [0..4] totals, [8..15] counters
  uint32_t *h_loff, *h_koff;  // pinned: [T + 1] each
};
__global__ void k_direct_finish(FinishArgs a) {
  const Full tot = a.ntiles ? a.tile_prefix[(a.ntiles + 31) / 32] : full_identity();
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= a.T) {
    const bool tail = a.off[t] >= a.n;
    const uint32_t lc = tail ? tot.c : a.t_layer_off[t];
    const uint32_t kc = tail ? tot.c_kl : a.t_kl_off[t];
    if (tail) {
      a.t_layer_off[t] = tot.c;
      a.t_kl_off[t] = tot.c_kl;
      a.t_ex_off[t] = tot.c_ex;
    }
    const uint32_t koff = lc == tot.c ? tot.c_kl : a.l_koff[lc];
    a.t_koff[t] = koff;
    a.h_loff[t] = lc;
    a.h_koff[t] = koff;
    if (t < a.T) {
      const bool ntail = a.off[t + 1] >= a.n;
      const uint32_t kn = ntail ? tot.c_kl : a.t_kl_off[t + 1];
      const uint32_t xc = tail ? tot.c_ex : a.t_ex_off[t];
      const uint32_t xn = ntail ? tot.c_ex : a.t_ex_off[t + 1];
      if (kn - kc != xn - xc || (kn != kc && a.dmin[t] != a.dmax[t])) atomicOr(a.counters + 7, 1u);
      int32_t st = XSP_T_OK;
      uint32_t ra = kNone;
      if (a.model_row[t] == kNone) {
        st = XSP_T_NO_MODEL;
      } else if (a.err_key[t] != ~0ull) {
        st = (int32_t)(a.err_key[t] & 0xFF);
        ra = (uint32_t)(a.err_key[t] >> 8);
      }
      a.status[t] = st;
      a.err_row[2 * t] = ra;
      a.err_row[2 * t + 1] = kNone;
      if (st != XSP_T_OK) atomicAdd(a.counters + 4, 1u);
    }
  }
  if (t == 0) {
    a.l_koff[tot.c] = tot.c_kl;
    a.totals[0] = a.h_totals[0] = tot.c;
    a.totals[1] = a.h_totals[1] = tot.c_kl;
    a.totals[2] = a.h_totals[2] = tot.c_ex;
    a.totals[3] = a.h_totals[3] = tot.c_metric;
    a.totals[4] = a.h_totals[4] = tot.c_lay;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.counters + 8, 1u) == gridDim.x - 1) {
      __threadfence();
      for (int q = 0; q < 8; ++q) a.h_totals[8 + q] = __ldcg(a.counters + q);
      __threadfence_system();
    }
  }
}

// ---------------------------------------------------------------------------
// Explicit-parent kernels (correlator.cpp:232-240): the parent must be a
// placed layer of the same trace; layer_by_span_id keeps the LAST layer (in
// layer_index order) with a given span_id (map assignment, :217-219).

// per trace: are placed-layer span_ids non-decreasing in layer order?
__global__ void k_layer_ids_sorted(const uint32_t* __restrict__ layer_row, const uint64_t* __restrict__ sid,
                                   const uint32_t* __restrict__ t_layer_off, uint32_t T, uint32_t nl,
                                   uint32_t* __restrict__ t_unsorted) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g + 1 >= nl) return;
  uint32_t t = trace_of32(t_layer_off, T, g);
  if (t_layer_off[t + 1] <= g + 1) return;  // g is the trace's last layer
  if (sid[layer_row[g]] > sid[layer_row[g + 1]]) t_unsorted[t] = 1;
}

__global__ void k_resolve_explicit(const uint32_t* __restrict__ pend_kl, const uint32_t* __restrict__ pend_count,
                                   KlEnt* __restrict__ kl, const uint64_t* __restrict__ parent,
                                   const uint64_t* __restrict__ sid, const uint32_t* __restrict__ layer_row,
                                   const uint32_t* __restrict__ t_layer_off, const uint32_t* __restrict__ t_kl_off,
                                   uint32_t T, const uint32_t* __restrict__ t_unsorted, Orphans orph) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= *pend_count) return;
  uint32_t k = pend_kl[p];
  uint32_t i = kl[k].row;
  uint32_t t = trace_of32(t_kl_off, T, k);
  uint64_t want = parent[i];
  uint32_t lo = t_layer_off[t], hi = t_layer_off[t + 1];
  uint32_t found = kNone;
  if (!t_unsorted[t]) {
    // last g in [lo, hi) with sid <= want, then check equality
    uint32_t l = lo, h = hi;
    while (l < h) {
      uint32_t mid = (l + h) >> 1;
      if (sid[layer_row[mid]] <= want) l = mid + 1; else h = mid;
    }
    if (l > lo && sid[layer_row[l - 1]] == want) found = l - 1;
  } else {
    for (uint32_t g = lo; g < hi; ++g)
      if (sid[layer_row[g]] == want) found = g;
  }
  if (found == kNone) {
    kl[k].parent = PAR_ORPHAN;
    emit_orphan(orph, t, CAT_KERNEL, i, i, XSP_O_KERNEL_BAD_PARENT);
  } else {
    kl[k].parent = found;
  }
}

// ---------------------------------------------------------------------------
// Ambiguities (correlator.cpp:242-257): all placed layers of the trace that
// precede the child in timeline order (g < gx) with end >= child end.

// The candidates are found through a 32-ary max tree over the placed layers'
// ends (level 0 = end[layer_row[g]], level L+1 = max of 32 level-L nodes):
// walking back from the child, a node whose max end is below the child's end is
// skipped whole, so each candidate costs O(32 * levels) loads however far back
// it lies (the reference's IntervalTree prunes on subtree max end the same way,
// correlator.cpp:79-109). Scanning layer by layer was O(layers of the trace) per
// child: quadratic on one long trace with concurrent layer groups (C4).
constexpr int kMtLevels = 7;  // 32^6 > 2^30 leaves under the top level
struct MaxTree {
  const uint64_t* lv[kMtLevels];  // lv[0] unused (leaves are read through layer_row)
  uint32_t n[kMtLevels];
  int levels;  // number of levels in use (>= 1); the top one has <= 32 nodes
  const uint32_t* layer_row;
  const uint64_t* end;
};

__device__ __forceinline__ uint64_t mt_val(const MaxTree& m, int L, uint32_t i) {
  return L == 0 ? __ldg(m.end + __ldg(m.layer_row + i)) : __ldg(m.lv[L] + i);
}

// Largest layer index g' in [lo, g) with end >= e, or kNone.
__device__ uint32_t mt_prev(const MaxTree& m, uint32_t g, uint32_t lo, uint64_t e) {
  if (g <= lo) return kNone;
  int L = 0;
  uint32_t i = g;  // exclusive bound at level L
  uint32_t j = kNone;
  for (;;) {  // ascend until a node of the bound's 32-group (and >= lo) holds an end >= e
    const uint32_t lo_l = lo >> (5 * L);
    const uint32_t grp = (i - 1) & ~31u;
    const uint32_t stop = grp > lo_l ? grp : lo_l;
    for (uint32_t x = i; x > stop;) {
      --x;
      if (mt_val(m, L, x) >= e) {
        j = x;
        break;
      }
    }
    if (j != kNone) break;
    if (grp <= lo_l || L + 1 >= m.levels) return kNone;
    i = grp >> 5;
    ++L;
  }
  while (L > 0) {  // descend into the rightmost child holding an end >= e
    --L;
    const uint32_t lo_l = lo >> (5 * L);
    const uint32_t c0 = j << 5, c1 = min(c0 + 32u, m.n[L]);
    const uint32_t stop = c0 > lo_l ? c0 : lo_l;
    uint32_t k = kNone;
    for (uint32_t x = c1; x > stop;) {
      --x;
      if (mt_val(m, L, x) >= e) {
        k = x;
        break;
      }
    }
    if (k == kNone) return kNone;  // only the node straddling lo: its max came from below lo
    j = k;
  }
  return j;
}

__global__ void k_mt_level(const uint64_t* __restrict__ in, const uint32_t* __restrict__ layer_row,
                           const uint64_t* __restrict__ end, uint32_t n_in, uint64_t* __restrict__ out) {
  const uint32_t o = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = lane_id();
  const uint32_t x = o * 32u + lane;
  if (o * 32u >= n_in) return;
  uint64_t v = 0;
  if (x < n_in) v = in ? in[x] : end[layer_row[x]];
#pragma unroll
  for (int s = 16; s; s >>= 1) v = max64(v, __shfl_xor_sync(0xffffffffu, v, s));
  if (lane == 0) out[o] = v;
}

// Children flagged in pass 1 with >= 2 candidates, or whose last preceding
// layer does not contain them while an earlier one might: count exactly.
__global__ void k_amb_resolve(uint32_t n_raw, const uint32_t* __restrict__ amb_kl,
                              const uint32_t* __restrict__ amb_gx, KlEnt* __restrict__ kl,
                              const uint64_t* __restrict__ end, const uint32_t* __restrict__ t_kl_off,
                              const uint32_t* __restrict__ t_layer_off, uint32_t T,
                              const __grid_constant__ MaxTree mt, uint32_t* __restrict__ keep, Orphans orph) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_raw) return;
  const uint32_t k = amb_kl[p];
  const uint32_t t = trace_of32(t_kl_off, T, k);
  const uint32_t row = kl[k].row;
  const uint64_t e = end[row];
  const uint32_t lo = t_layer_off[t];
  const uint32_t g1 = mt_prev(mt, amb_gx[p], lo, e);
  const uint32_t g2 = g1 == kNone ? kNone : mt_prev(mt, g1, lo, e);
  if (g1 != kNone && g2 == kNone) {
    kl[k].parent = g1;
    keep[p] = 0;
  } else if (g1 == kNone) {  // only for a child ending at UINT64_MAX (see k_pass1)
    kl[k].parent = PAR_ORPHAN;
    keep[p] = 0;
    emit_orphan(orph, t, CAT_KERNEL, row, row, XSP_O_KERNEL_NO_LAYER);
  } else {
    keep[p] = 1;
  }
}

__global__ void k_amb_compact(uint32_t n_raw, const uint32_t* __restrict__ keep, const uint32_t* __restrict__ pos,
                              const uint32_t* __restrict__ kl, const uint32_t* __restrict__ gx,
                              uint32_t* __restrict__ kl2, uint32_t* __restrict__ gx2) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_raw || !keep[p]) return;
  kl2[pos[p]] = kl[p];
  gx2[pos[p]] = gx[p];
}

__global__ void k_amb_keys(const uint32_t* __restrict__ amb_kl, uint32_t n_amb, const KlEnt* __restrict__ kl,
                           const uint64_t* __restrict__ sid, const uint32_t* __restrict__ t_kl_off, uint32_t T,
                           uint64_t* __restrict__ key_sid, uint64_t* __restrict__ key_trace,
                           uint32_t* __restrict__ idx) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_amb) return;
  uint32_t k = amb_kl[p];
  key_sid[p] = sid[kl[k].row];
  key_trace[p] = trace_of32(t_kl_off, T, k);
  idx[p] = p;
}

__global__ void k_amb_count(const uint32_t* __restrict__ order, uint32_t n_amb,
                            const uint32_t* __restrict__ amb_kl, const uint32_t* __restrict__ amb_gx,
                            const KlEnt* __restrict__ kl, const uint64_t* __restrict__ end,
                            const uint32_t* __restrict__ t_kl_off, const uint32_t* __restrict__ t_layer_off,
                            uint32_t T, const __grid_constant__ MaxTree mt, uint32_t* __restrict__ cnt) {
  uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_amb) return;
  uint32_t p = order[q];
  uint32_t k = amb_kl[p];
  uint32_t t = trace_of32(t_kl_off, T, k);
  uint64_t e = end[kl[k].row];
  const uint32_t lo = t_layer_off[t];
  uint32_t c = 0;
  for (uint32_t g = mt_prev(mt, amb_gx[p], lo, e); g != kNone; g = mt_prev(mt, g, lo, e)) ++c;
  cnt[q] = c;
}

__global__ void k_amb_fill(const uint32_t* __restrict__ order, uint32_t n_amb,
                           const uint32_t* __restrict__ amb_kl, const uint32_t* __restrict__ amb_gx,
                           const KlEnt* __restrict__ kl, const uint64_t* __restrict__ end,
                           const uint64_t* __restrict__ sid, const uint32_t* __restrict__ t_kl_off,
                           const uint32_t* __restrict__ t_layer_off, uint32_t T, const __grid_constant__ MaxTree mt,
                           const uint32_t* __restrict__ cand_off, uint32_t* __restrict__ amb_row,
                           uint32_t* __restrict__ cand_row) {
  uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_amb) return;
  uint32_t p = order[q];
  uint32_t k = amb_kl[p];
  uint32_t t = trace_of32(t_kl_off, T, k);
  uint64_t e = end[kl[k].row];
  amb_row[q] = kl[k].row;
  const uint32_t lo = t_layer_off[t];
  uint32_t o = cand_off[q], n = 0;
  for (uint32_t g = mt_prev(mt, amb_gx[p], lo, e); g != kNone; g = mt_prev(mt, g, lo, e)) {
    uint32_t r = mt.layer_row[g];
    // insertion by span_id (IntervalTree::containing sorts by span_id, :115-117)
    uint64_t s = sid[r];
    uint32_t j = n;
    while (j > 0 && sid[cand_row[o + j - 1]] > s) {
      cand_row[o + j] = cand_row[o + j - 1];
      --j;
    }
    cand_row[o + j] = r;
    ++n;
  }
}

// ---------------------------------------------------------------------------
// (d) cid join.
//
// Fast path (sort-merge on presorted streams): trace t is "merge-aligned" when
// it has as many cid-bearing exec entries as kernel-list entries, every entry is
// a launch with a cid, and launch r and exec r carry the same cid with cids
// strictly increasing in r. Then the r-th launch fuses with the r-th exec, every
// exec is consumed and no cid repeats — exactly what the reference's hash maps
// produce. Other traces use the per-trace open-addressing table below.

__global__ void k_join_counts(const uint32_t* __restrict__ t_kl_off, const uint32_t* __restrict__ t_ex_off,
                              uint32_t T, uint32_t* __restrict__ t_slow, uint32_t* __restrict__ any_slow) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const bool mismatch = (t_kl_off[t + 1] - t_kl_off[t]) != (t_ex_off[t + 1] - t_ex_off[t]);
  t_slow[t] = mismatch;
  if (mismatch) *any_slow = 1;
}

// t_slow[t] = 1 when some kernel-list entry of t is not a cid launch, its cid
// does not exceed the previous entry's, or launch r and exec r disagree on the
// cid (not merge-aligned); t_lmin / t_lmax = the launch cid range of every
// trace (the direct-address join needs it). A warp covers 32 x JC_ITEMS
// consecutive entries (lane-strided, coalesced) and keeps running min / max per
// lane, so a long trace issues one atomic pair per warp, not per 32 entries.
constexpr uint32_t JC_ITEMS = 8;
__global__ void k_join_check(uint32_t nkl, const KlEnt* __restrict__ kl, const ExEnt* __restrict__ ex,
                             const uint64_t* __restrict__ cid,
                             const uint8_t* __restrict__ flags, const uint32_t* __restrict__ t_kl_off,
                             const uint32_t* __restrict__ t_ex_off, uint32_t T, uint32_t* __restrict__ t_slow,
                             uint32_t* __restrict__ any_slow, unsigned long long* __restrict__ t_lmin,
                             unsigned long long* __restrict__ t_lmax, uint32_t* __restrict__ t_nonmono) {
  const uint32_t lane = lane_id();
  const uint64_t wbase64 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32ull * JC_ITEMS;
  if (wbase64 >= nkl) return;
  const uint32_t wbase = (uint32_t)wbase64;
  uint32_t t0 = 0;
  if (lane == 0) t0 = trace_of32(t_kl_off, T, wbase);
  uint32_t t = __shfl_sync(0xffffffffu, t0, 0);
  uint32_t tl = kNone;
  uint64_t mn = ~0ull, mx = 0;
  // a trace already known to be slow needs no alignment check (one L2 read per
  // trace change, not per entry). A stale 0 only costs the check, so the read
  // of the warp's first trace is a plain L2 load issued with the entry loads
  // (a volatile read there held 37% of the kernel's stall samples on C4).
  uint32_t tslow = t, tnm = kNone;
  bool slow = __ldcg(t_slow + t) != 0;
  // all of the lane's entries and their flag bytes are loaded up front (the
  // loads of an entry no longer wait for the previous entry's checks)
  KlEnt e[JC_ITEMS];
  uint8_t fb[JC_ITEMS];
#pragma unroll
  for (uint32_t i = 0; i < JC_ITEMS; ++i) {
    const uint32_t k = wbase + i * 32 + lane;
    if (k < nkl) e[i] = kl[k];
    else e[i] = KlEnt{0, 0, 0};
  }
#pragma unroll
  for (uint32_t i = 0; i < JC_ITEMS; ++i) {
    const uint32_t k = wbase + i * 32 + lane;
    fb[i] = k < nkl ? flags[e[i].row] : (uint8_t)0;
  }
  uint64_t prev_last = (wbase > 0 && lane == 0) ? kl[wbase - 1].cid : 0;  // entry before the warp's first
#pragma unroll
  for (uint32_t i = 0; i < JC_ITEMS; ++i) {
    const uint32_t k = wbase + i * 32 + lane;
    // the previous entry's cid: the lane below, or lane 31 of the previous item
    uint64_t pc = __shfl_up_sync(0xffffffffu, e[i].cid, 1);
    const uint64_t last = __shfl_sync(0xffffffffu, i == 0 ? prev_last : e[i - (i > 0)].cid, i == 0 ? 0 : 31);
    if (lane == 0) pc = last;
    if (k >= nkl) continue;
    while (t + 1 < T && __ldg(t_kl_off + t + 1) <= k) ++t;
    if (t != tslow) {
      tslow = t;
      slow = __ldcg(t_slow + t) != 0;
    }
    const uint32_t r = k - t_kl_off[t];
    const KlEnt ent = e[i];
    const uint8_t f = fb[i];
    const bool launch = f_kind(f) == XSP_KIND_LAUNCH && (f & XSP_F_CID);
    const bool mono = launch && (r == 0 || pc < ent.cid);
    if (launch) {
      if (tl != t) {
        if (tl != kNone) {
          atomicMin(t_lmin + tl, (unsigned long long)mn);
          atomicMax(t_lmax + tl, (unsigned long long)mx);
        }
        tl = t;
        mn = ~0ull;
        mx = 0;
      }
      mn = ent.cid < mn ? ent.cid : mn;
      mx = ent.cid > mx ? ent.cid : mx;
    }
    // only the first mismatch of a trace stores (a reordered long trace would
    // otherwise have every launch store to the same two words)
    if (!mono && t != tnm) {  // once per trace per thread
      t_nonmono[t] = 1;
      tnm = t;
    }
    if (!slow && !(mono && cid[ex[t_ex_off[t] + r].row] == ent.cid)) {
      t_slow[t] = 1;
      *any_slow = 1;
      slow = true;
    }
  }
  __syncwarp();
  minmax_atomic_warp(tl, mn, mx, t_lmin, t_lmax);
}

// Direct-address join for slow traces whose launch cids span a dense range
// (in any order: executions reordered across streams, concurrent layers'
// interleaved launches): the slot of a cid is cid - lmin, with no hashing or
// probing. t_lmin[t] = the least launch cid (k_join_check), or ~0 when t uses
// the hash table.
__global__ void k_join_direct(const uint32_t* __restrict__ t_kl_off, const uint32_t* __restrict__ t_slow,
                              uint32_t T, uint64_t* __restrict__ t_lmin, uint64_t* __restrict__ t_lmax) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint32_t k0 = t_kl_off[t], k1 = t_kl_off[t + 1];
  const uint64_t a = t_lmin[t], b = t_lmax[t];
  if (!(t_slow[t] && a != ~0ull && b - a < 4ull * (k1 - k0) + 64)) {
    t_lmin[t] = ~0ull;
    t_lmax[t] = 0;
  }
}

// An exec whose cid lies outside its direct trace's launch range matches no
// launch but may still duplicate another exec: that trace uses the hash table.
__global__ void k_join_far(uint32_t nex, const ExEnt* __restrict__ ex, const uint64_t* __restrict__ cid,
                           const uint32_t* __restrict__ t_ex_off,
                           uint32_t T, uint64_t* __restrict__ t_lmin, const uint64_t* __restrict__ t_lmax) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t first = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  if (first >= nex) return;
  const uint32_t t = warp_trace_of(t_ex_off, T, x < nex ? x : nex - 1, first);
  if (x >= nex) return;
  const uint64_t lmin = t_lmin[t];
  if (lmin == ~0ull) return;
  const uint64_t c = cid[ex[x].row];
  if (c < lmin || c > t_lmax[t]) t_lmin[t] = ~0ull;
}

__device__ __forceinline__ uint32_t mix32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return (uint32_t)x;
}

// A direct-address trace is "dense" when its kernel-list entries are all cid
// launches with strictly increasing cids covering the range without gaps: the
// r-th launch owns slot r, so launches need no insert, no duplicate check and
// no leftover pass (every in-range execution has its launch).
__global__ void k_region_size(const uint32_t* __restrict__ t_kl_off, const uint32_t* __restrict__ t_ex_off,
                              const uint32_t* __restrict__ t_slow, const uint64_t* __restrict__ t_lmin,
                              const uint64_t* __restrict__ t_lmax, uint32_t T, uint64_t* __restrict__ rsize,
                              const uint32_t* __restrict__ t_nonmono, uint32_t* __restrict__ t_dense) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  t_dense[t] = 0;
  if (t_lmin[t] != ~0ull) {  // direct-address region: one slot per cid of the launch range
    rsize[t] = t_lmax[t] - t_lmin[t] + 1;
    t_dense[t] = !t_nonmono[t] && rsize[t] == (uint64_t)(t_kl_off[t + 1] - t_kl_off[t]);
    return;
  }
  uint64_t items = (uint64_t)(t_kl_off[t + 1] - t_kl_off[t]) + (t_ex_off[t + 1] - t_ex_off[t]);
  uint64_t s = 16;
  while (s < items * 2) s <<= 1;
  rsize[t] = (items && t_slow[t]) ? s : 0;
}

struct JoinArgs {
  const ExEnt* ex;
  const uint64_t* cid;  // span cid column (exec cids by row)
  const KlEnt* kl;
  const uint8_t* flags;
  const uint32_t* t_ex_off;
  const uint32_t* t_kl_off;
  const uint32_t* t_slow;
  const uint64_t* t_lmin;  // direct-address traces: first launch cid, else ~0
  uint32_t T;
  uint32_t n_ex, n_kl;
  const uint64_t* roff;  // region offsets [T+1]
  uint32_t* owner;       // 0 empty, else item + 1
  uint32_t* sl_exec;     // min exec item
  uint32_t* sl_launch;   // min klist item
  uint32_t* ex_slot;
  uint32_t* kl_slot;
  uint32_t* t_dup;       // bit0 exec dup, bit1 launch dup
  uint32_t* any_dup;     // some trace has a duplicate (zeroed per call)
  const uint32_t* t_dense;  // dense direct-address traces (k_region_size)
};

// Items 0..n_ex-1 are execs, n_ex..n_ex+n_kl-1 kernel-list entries (launches
// with a cid). Only items of slow traces take part.
__global__ void k_join_insert(JoinArgs a) {
  uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= a.n_ex + a.n_kl) return;
  const bool is_ex = it < a.n_ex;
  uint32_t t;
  uint64_t cid;
  if (is_ex) {
    t = trace_of32(a.t_ex_off, a.T, it);
    if (!a.t_slow[t]) return;
    cid = a.cid[a.ex[it].row];
  } else {
    uint32_t k = it - a.n_ex;
    t = trace_of32(a.t_kl_off, a.T, k);
    if (!a.t_slow[t] || a.t_dense[t]) return;  // dense: launch r owns slot r (no insert)
    const uint8_t f = a.flags[a.kl[k].row];
    if (!is_kernel_launch(f) || !(f & XSP_F_CID)) return;
    cid = a.kl[k].cid;
  }
  const uint64_t base = a.roff[t];
  const uint64_t lmin = a.t_lmin[t];
  const uint32_t mask = (uint32_t)(a.roff[t + 1] - base - 1);
  uint32_t h = lmin != ~0ull ? (uint32_t)(cid - lmin) : mix32(cid) & mask;
  for (; lmin == ~0ull;) {
    uint32_t* slot = a.owner + base + h;
    uint32_t o = *((volatile uint32_t*)slot);
    if (o == 0) {
      o = atomicCAS(slot, 0u, it + 1);
      if (o == 0) break;
    }
    uint32_t oi = o - 1;
    uint64_t ocid = oi < a.n_ex ? a.cid[a.ex[oi].row] : a.kl[oi - a.n_ex].cid;
    if (ocid == cid) break;
    h = (h + 1) & mask;
  }
  const uint32_t s = (uint32_t)(base + h);
  if (is_ex) {
    a.ex_slot[it] = s;
    if (atomicMin(a.sl_exec + s, it) != kNone) {
      atomicOr(a.t_dup + t, 1u);
      *a.any_dup = 1;
    }
  } else {
    uint32_t k = it - a.n_ex;
    a.kl_slot[k] = s;
    if (atomicMin(a.sl_launch + s, k) != kNone) {
      atomicOr(a.t_dup + t, 2u);
      *a.any_dup = 1;
    }
  }
}

// Exact duplicate report: the first item in timeline order whose cid was seen
// before, and that earlier (first) item (correlator.cpp:296-316). Grid-stride;
// a batch without duplicates (the common case) exits on one flag read.
__global__ void k_join_dups(JoinArgs a, unsigned long long* __restrict__ dup_ex,
                            unsigned long long* __restrict__ dup_kl) {
  if (!*((volatile uint32_t*)a.any_dup)) return;
  const uint32_t n = a.n_ex + a.n_kl;
  for (uint32_t it = blockIdx.x * blockDim.x + threadIdx.x; it < n; it += gridDim.x * blockDim.x) {
    if (it < a.n_ex) {
      uint32_t t = trace_of32(a.t_ex_off, a.T, it);
      if (!(a.t_dup[t] & 1u)) continue;
      uint32_t first = a.sl_exec[a.ex_slot[it]];
      if (first != it) atomicMin(dup_ex + t, ((unsigned long long)it << 32) | first);
    } else {
      uint32_t k = it - a.n_ex;
      uint32_t t = trace_of32(a.t_kl_off, a.T, k);
      if (!(a.t_dup[t] & 2u)) continue;
      const uint8_t f = a.flags[a.kl[k].row];
      if (!is_kernel_launch(f) || !(f & XSP_F_CID)) continue;
      uint32_t first = a.sl_launch[a.kl_slot[k]];
      if (first != k) atomicMin(dup_kl + t, ((unsigned long long)k << 32) | first);
    }
  }
}

// ---------------------------------------------------------------------------
// Kernel fusion (correlator.cpp:321-346) + kept flags; leftover execs (:348-363).

struct FuseArgs {
  uint32_t n_kl, n_ex, T;
  const KlEnt* kl;
  const ExEnt* ex;
  const uint8_t* flags;
  const uint32_t* t_slow;
  const uint32_t* kl_slot;
  const uint32_t* sl_exec;
  const uint32_t* sl_launch;
  const uint32_t* ex_slot;
  const uint64_t* sid;
  const uint32_t* t_kl_off;
  const uint32_t* t_ex_off;
  uint32_t* kept;     // [n_kl] 0/1
  uint32_t* kl_exec;  // matched exec item
  Orphans orph;
  bool any_slow;
  bool parents_only;  // assign_parents without correlate_async
  const uint32_t* t_dense;  // dense direct-address traces: slot of launch k = roff[t] + (k - t_kl_off[t])
  const uint64_t* roff;
  uint32_t* drop;     // [0] entries not kept, [1] kept parents not in timeline order
};

__global__ void k_fuse(FuseArgs a) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t first = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  if (first >= a.n_kl) return;
  const uint32_t t = warp_trace_of(a.t_kl_off, a.T, k < a.n_kl ? k : a.n_kl - 1, first);
  if (k >= a.n_kl) return;
  const KlEnt ent = a.kl[k];
  uint32_t keep = 0, x = kNone;
  if (ent.parent < PAR_MAXROW) {
    const uint8_t f = a.flags[ent.row];
    if (is_sync_kernel(f) || a.parents_only) {
      keep = 1;
      x = is_sync_kernel(f) ? kNone : kNone - 1;  // kNone-1: launch left unfused
    } else if (!(f & XSP_F_CID)) {
      emit_orphan(a.orph, t, CAT_LAUNCH, ((uint64_t)ent.parent << 32) | k, ent.row, XSP_O_LAUNCH_NO_CID);
    } else {
      if (a.any_slow && a.t_slow[t])
        x = a.sl_exec[a.t_dense[t] ? (uint32_t)(a.roff[t] + (k - a.t_kl_off[t])) : a.kl_slot[k]];
      else
        x = a.t_ex_off[t] + (k - a.t_kl_off[t]);
      if (x != kNone) {
        keep = 1;
      } else {
        emit_orphan(a.orph, t, CAT_LAUNCH, ((uint64_t)ent.parent << 32) | k, ent.row, XSP_O_LAUNCH_NO_EXEC);
      }
    }
  }
  a.kept[k] = keep;
  a.kl_exec[k] = x;
  if (!keep) atomicAdd(a.drop, 1u);
  else if (k > 0 && a.kl[k - 1].parent > ent.parent) atomicOr(a.drop + 1, 1u);
}

__global__ void k_leftover(FuseArgs a) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= a.n_ex) return;
  const uint32_t t = trace_of32(a.t_ex_off, a.T, x);
  if (!a.t_slow[t] || a.t_dense[t]) return;  // merge-aligned / dense traces consume every exec
  if (a.sl_launch[a.ex_slot[x]] == kNone) {
    const uint32_t r = a.ex[x].row;
    emit_orphan(a.orph, t, CAT_LEFTOVER, a.sid[r], r, XSP_O_EXEC_NO_LAUNCH);
  }
}

// Compact kept kernels (timeline order) with their parent layer as the sort key.
__global__ void k_compact_kernels(uint32_t n_kl, const uint32_t* __restrict__ kept,
                                  const uint32_t* __restrict__ pos, const KlEnt* __restrict__ kl,
                                  uint64_t* __restrict__ key, uint32_t* __restrict__ val,
                                  uint32_t* __restrict__ nonmono) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_kl || !kept[k]) return;
  const uint32_t j = pos[k];
  const uint32_t par = kl[k].parent;
  key[j] = par;
  val[j] = k;
  // tree order == list order unless a kept entry's parent is below the previous
  // kept entry's (key[j] < key[j - 1]). Only the first kept entry after a run of
  // dropped ones walks it (e.g. the ambiguous launches of a concurrent layer
  // group); a run longer than 4096 sets the flag conservatively (the stable
  // sort is then a no-op)
  if (j > 0) {
    uint32_t q = k - 1;
    for (int step = 0; !kept[q] && step < 4096; ++step) --q;
    if (!kept[q] || kl[q].parent > par) *nonmono = 1;
  }
}

__global__ void k_gather_kernels(uint32_t nk, const uint32_t* __restrict__ val, const KlEnt* __restrict__ kl,
                                 const uint32_t* __restrict__ kl_mrow, const uint32_t* __restrict__ kl_exec,
                                 const ExEnt* __restrict__ ex, const uint8_t* __restrict__ flags,
                                 const uint64_t* __restrict__ begin, const uint64_t* __restrict__ end,
                                 const uint32_t* __restrict__ name, const double* __restrict__ occ,
                                 uint32_t* __restrict__ k_launch, uint32_t* __restrict__ k_exec,
                                 uint32_t* __restrict__ k_mrow, uint64_t* __restrict__ k_dur,
                                 uint32_t* __restrict__ k_name, double* __restrict__ k_occ) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nk) return;
  const uint32_t k = val ? val[j] : j;  // no val: every entry kept, in order
  const uint32_t r = kl[k].row;
  const uint32_t x = kl_exec[k];
  uint32_t er, mr;
  if (x == kNone) {  // synchronous kernel: launch and exec are the same record
    er = r;
    mr = kl_mrow[k];
  } else if (x == kNone - 1) {  // assign_parents only: launch without its exec
    k_launch[j] = r;
    k_exec[j] = kNone;
    k_mrow[j] = kNone;
    k_dur[j] = 0;
    k_name[j] = name[r];
    k_occ[j] = 0.0;
    return;
  } else {
    const ExEnt e = ex[x];
    k_launch[j] = r;
    k_exec[j] = e.row;
    k_mrow[j] = e.mrow;
    k_dur[j] = e.dur;
    k_name[j] = name[e.row];
    k_occ[j] = e.mrow != kNone ? occ[e.mrow] : 0.0;
    return;
  }
  k_launch[j] = r;
  k_exec[j] = er;
  k_mrow[j] = mr;
  k_dur[j] = clamp_dur(begin[er], end[er]);
  k_name[j] = name[er];
  k_occ[j] = mr != kNone ? occ[mr] : 0.0;
}

// Clean batches (no orphan, ambiguity or explicit parent): optimistic fusion.
// Every kernel-list entry is kept in tree order and entry r of trace t fuses
// with exec r of trace t, PROVIDED the trace is merge-aligned (same count of
// launches and execs, every entry a launch with a cid, equal cids at equal
// rank, strictly increasing). The same pass verifies that; any failure sets
// *fail and the caller reruns the general join.
__device__ __forceinline__ void gather_fast_one(uint32_t j, uint32_t first, uint32_t nl, uint32_t nk, uint32_t nex, const KlEnt* __restrict__ kl,
                              const ExEnt* __restrict__ ex, const uint8_t* __restrict__ flags,
                              const uint32_t* __restrict__ t_kl_off, const uint32_t* __restrict__ t_ex_off,
                              uint32_t T, const uint64_t* __restrict__ cid,
                              const uint32_t* __restrict__ name, const double* __restrict__ occ,
                              uint32_t* __restrict__ k_launch, uint32_t* __restrict__ k_exec,
                              uint32_t* __restrict__ k_mrow, uint64_t* __restrict__ k_dur,
                              uint32_t* __restrict__ k_name, double* __restrict__ k_occ,
                              uint32_t* __restrict__ l_koff, uint32_t* __restrict__ fail) {
  if (first > nk) return;
  uint32_t t = 0;
  if (nk) t = warp_trace_of(t_kl_off, T, j < nk ? j : nk - 1, first < nk ? first : nk - 1);
  if (j > nk) return;
  // layer CSR boundaries (keys = parents, non-decreasing); a pending / orphan /
  // ambiguous parent means the batch is not clean (the general path redoes it)
  const uint32_t pp = j > 0 ? kl[j - 1].parent : 0u;
  const uint32_t pc = j < nk ? kl[j].parent : nl;
  if ((j > 0 && pp >= PAR_MAXROW) || pc >= PAR_MAXROW) {
    *fail = 1;
    return;
  }
  const int64_t prev = j > 0 ? (int64_t)pp : -1;
  const int64_t cur = (int64_t)pc;
  for (int64_t g = prev + 1; g <= cur; ++g) l_koff[g] = j;
  if (j == nk) {
    if (nex != nk) *fail = 1;  // some trace has execs but no launches
    return;
  }
  const KlEnt ent = kl[j];
  const uint32_t kb = t_kl_off[t], xb = t_ex_off[t];
  const uint32_t r = j - kb;
  const uint8_t f = flags[ent.row];
  bool ok = (t_kl_off[t + 1] - kb) == (t_ex_off[t + 1] - xb) && f_kind(f) == XSP_KIND_LAUNCH && (f & XSP_F_CID);
  ExEnt e;
  e.row = ent.row;
  e.mrow = kNone;
  e.dur = 0;
  if (ok) {
    e = ex[xb + r];
    ok = cid[e.row] == ent.cid && (r == 0 || kl[j - 1].cid < ent.cid);
  }
  if (!ok) {
    *fail = 1;
    return;
  }
  k_launch[j] = ent.row;
  k_exec[j] = e.row;
  k_mrow[j] = e.mrow;
  k_dur[j] = e.dur;
  k_name[j] = name[e.row];
  k_occ[j] = e.mrow != kNone ? occ[e.mrow] : 0.0;
}

// Sizes come from pass 1's totals on the device and the grid strides over them,
// so the clean path needs no host round trip before it runs.
__global__ void __launch_bounds__(256) k_gather_fast(const uint32_t* __restrict__ totals,
                              const KlEnt* __restrict__ kl,
                              const ExEnt* __restrict__ ex, const uint8_t* __restrict__ flags,
                              const uint32_t* __restrict__ t_kl_off, const uint32_t* __restrict__ t_ex_off,
                              uint32_t T, const uint64_t* __restrict__ cid,
                              const uint32_t* __restrict__ name, const double* __restrict__ occ,
                              uint32_t* __restrict__ k_launch, uint32_t* __restrict__ k_exec,
                              uint32_t* __restrict__ k_mrow, uint64_t* __restrict__ k_dur,
                              uint32_t* __restrict__ k_name, double* __restrict__ k_occ,
                              uint32_t* __restrict__ l_koff, uint32_t* __restrict__ fail) {
  const uint32_t nl = totals[0], nk = totals[1], nex = totals[2];
  // a batch found not clean is redone by the general path: stop early (the
  // flag is polled every 16 strides so the clean case pays almost nothing)
  uint32_t it = 0;
  for (uint32_t base = blockIdx.x * blockDim.x; base <= nk; base += gridDim.x * blockDim.x, ++it) {
    if ((it & 15u) == 15u && __ldcg(fail)) return;
    gather_fast_one(base + threadIdx.x, base + (threadIdx.x & ~31u), nl, nk, nex, kl, ex, flags, t_kl_off,
                    t_ex_off, T, cid, name, occ, k_launch, k_exec, k_mrow, k_dur, k_name, k_occ, l_koff,
                    fail);
  }
}

// layer_kernel_off[g] = first kernel j whose parent >= g (keys sorted): each
// boundary between consecutive keys fills the layers in between.
__global__ void k_layer_kernel_off(uint32_t nl, uint32_t nk, const uint64_t* __restrict__ key,
                                   uint32_t* __restrict__ off) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > nk) return;
  const int64_t prev = j > 0 ? (int64_t)key[j - 1] : -1;
  const int64_t cur = j < nk ? (int64_t)key[j] : (int64_t)nl;
  for (int64_t g = prev + 1; g <= cur; ++g) off[g] = j;
}
// the same with every kernel-list entry kept, in order: keys are the parents
__global__ void k_layer_kernel_off_kl(uint32_t nl, uint32_t nk, const KlEnt* __restrict__ kl,
                                      uint32_t* __restrict__ off) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > nk) return;
  const int64_t prev = j > 0 ? (int64_t)kl[j - 1].parent : -1;
  const int64_t cur = j < nk ? (int64_t)kl[j].parent : (int64_t)nl;
  for (int64_t g = prev + 1; g <= cur; ++g) off[g] = j;
}

__global__ void k_trace_kernel_off(uint32_t T, const uint32_t* __restrict__ t_layer_off,
                                   const uint32_t* __restrict__ l_koff, uint32_t* __restrict__ t_koff) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > T) return;
  t_koff[t] = l_koff[t_layer_off[t]];
}

// ---------------------------------------------------------------------------
// Orphans in reference order: sort by (trace, category, key).

__global__ void k_iota(uint32_t* v, uint32_t n) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}
__global__ void k_gather_u64(const uint64_t* __restrict__ src, const uint32_t* __restrict__ idx,
                             uint64_t* __restrict__ dst, uint32_t n) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_orphan_out(uint32_t n, const uint32_t* __restrict__ order, const uint32_t* __restrict__ row,
                             const uint8_t* __restrict__ reason, uint32_t* __restrict__ out_row,
                             uint8_t* __restrict__ out_reason) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out_row[i] = row[order[i]];
  out_reason[i] = reason[order[i]];
}
// CSR over traces from keys sorted by trace (key >> shift).
__global__ void k_csr_by_trace(uint32_t T, uint32_t n, const uint64_t* __restrict__ keys, int shift,
                               uint32_t* __restrict__ off) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > T) return;
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if ((keys[mid] >> shift) < t) lo = mid + 1; else hi = mid;
  }
  off[t] = lo;
}

// Final per-trace status (assign_parents faults first, then correlate_async).
__global__ void k_status(uint32_t T, const uint32_t* __restrict__ model_row,
                         const unsigned long long* __restrict__ err_key,
                         const unsigned long long* __restrict__ dup_ex,
                         const unsigned long long* __restrict__ dup_kl, const ExEnt* __restrict__ ex,
                         const KlEnt* __restrict__ kl, int32_t* __restrict__ status,
                         uint32_t* __restrict__ err_row, uint32_t* __restrict__ n_failed) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  int32_t st = XSP_T_OK;
  uint32_t ra = kNone, rb = kNone;
  if (model_row[t] == kNone) {
    st = XSP_T_NO_MODEL;
  } else if (err_key[t] != ~0ull) {
    st = (int32_t)(err_key[t] & 0xFF);
    ra = (uint32_t)(err_key[t] >> 8);
  } else if (dup_ex[t] != ~0ull) {
    st = XSP_T_DUP_EXEC_CID;
    ra = ex[(uint32_t)dup_ex[t]].row;          // first occurrence
    rb = ex[(uint32_t)(dup_ex[t] >> 32)].row;  // the duplicate
  } else if (dup_kl[t] != ~0ull) {
    st = XSP_T_DUP_LAUNCH_CID;
    ra = kl[(uint32_t)dup_kl[t]].row;
    rb = kl[(uint32_t)(dup_kl[t] >> 32)].row;
  }
  status[t] = st;
  err_row[2 * t] = ra;
  err_row[2 * t + 1] = rb;
  if (st != XSP_T_OK) atomicAdd(n_failed, 1u);
}

// ---------------------------------------------------------------------------
// Orchestration

namespace {

template <typename K, typename... Args>
void launch(xsp_ctx* ctx, K kernel, uint64_t n, cudaStream_t st, Args... args) {
  if (n == 0) return;
  unsigned blocks = ceil_div(n, 256);
  kernel<<<blocks, 256, 0, st>>>(args...);
  ++ctx->launches;
}

RadixScratch radix_scratch(xsp_ctx* ctx, uint64_t n) {
  RadixScratch s;
  s.keys_alt = ctx->d<uint64_t>("rs.keys_alt", n);
  s.vals_alt = ctx->d<uint32_t>("rs.vals_alt", n);
  uint64_t ce = radix_counts_elems(n);
  s.counts = ctx->d<uint32_t>("rs.counts", ce);
  s.scan_tmp = ctx->d<uint32_t>("rs.scan", scan_scratch_elems(ce));
  s.and_or = ctx->d<unsigned long long>("rs.andor", 2);
  s.and_or_host = ctx->h<unsigned long long>("rs.andor_h", 2);
  return s;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    XSP_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// A u64 span column as a [n/16][16] tensor, 128-row boxes, 128-byte swizzle.
void col_tmap(CUtensorMap* m, const uint64_t* col, uint64_t n) {
  cuuint64_t dims[2] = {16, n / 16};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {16, (cuuint32_t)P1_ROWS};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = tmap_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint64_t*>(col), dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

// Enqueue the host copies of the per-trace offsets (read with the final sync).
void cache_offsets_begin(xsp_ctx* ctx, const uint32_t* t_loff, const uint32_t* t_koff, uint32_t T,
                         cudaStream_t st) {
  ctx->hc_layer_key = ctx->hc_kernel_key = nullptr;
  xfer_small(ctx->h<uint32_t>("c.hc_loff", T + 1), t_loff, (T + 1) * 4ull, st);
  xfer_small(ctx->h<uint32_t>("c.hc_koff", T + 1), t_koff, (T + 1) * 4ull, st);
}
void cache_offsets_end(xsp_ctx* ctx, const uint32_t* t_loff, const uint32_t* t_koff, uint32_t T) {
  ctx->hc_layer_key = t_loff;
  ctx->hc_kernel_key = t_koff;
  ctx->hc_T = T;
}

uint32_t read_u32(xsp_ctx* ctx, const uint32_t* dptr, cudaStream_t st) {
  uint32_t* h = ctx->h<uint32_t>("readback.u32", 1);
  xfer_small(h, dptr, 4, st);
  XSP_CUDA(cudaStreamSynchronize(st));
  return *h;
}

}  // namespace

struct ListOverflow {};

void run_correlate_once(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_traces* tr, int mode,
                        xsp_corr_out* out, cudaStream_t st);

void run_correlate(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_traces* tr, int mode,
                   xsp_corr_out* out, cudaStream_t st) {
  for (int attempt = 0;; ++attempt) {
    try {
      run_correlate_once(ctx, c, tr, mode, out, st);
      return;
    } catch (const ListOverflow&) {
      if (attempt >= 2) throw std::runtime_error("correlate: exception lists kept overflowing");
    }
  }
}

void run_correlate_once(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_traces* tr, int mode,
                        xsp_corr_out* out, cudaStream_t st) {
  const int sort_if_needed = mode & 1;
  const bool parents_only = (mode & XSP_CORR_PARENTS_ONLY) != 0;
  const uint64_t n = c->n_spans;
  const uint32_t T = tr->n_traces;
  if (n >= 0xFFFFFFF0ull) throw std::invalid_argument("more than 2^32-16 spans in one call");
  const uint64_t* off = tr->span_off;

  // ---- per-trace state
  uint32_t* model_row = ctx->d<uint32_t>("c.model_row", T);
  uint64_t* mb = ctx->d<uint64_t>("c.mb", T);
  uint64_t* me = ctx->d<uint64_t>("c.me", T);
  uint64_t* msid = ctx->d<uint64_t>("c.msid", T);
  auto* err_key = ctx->d<unsigned long long>("c.err_key", T);
  const uint32_t ntiles = ceil_div(n, P1_TILE);
  uint32_t* tile_lo = ctx->d<uint32_t>("c.tile_lo", ntiles + 1);
  uint32_t* tile_hi = ctx->d<uint32_t>("c.tile_hi", ntiles + 1);
  if (T) {
    ctx->stage_begin("trace_prep", st);
    unsigned blocks = ceil_div((uint64_t)T * 32, 256);
    // tile -> trace: per trace by its warp when traces are short on average (one
    // launch), per tile by binary search when they are long (a trace's warp
    // would walk all of its tiles serially)
    const bool per_tile = ntiles && n / T > 64ull * P1_TILE;
    k_trace_prep<<<blocks, 256, 0, st>>>(c->flags, c->begin_ns, c->end_ns, c->span_id, off, T, model_row, mb, me,
                                         msid, err_key, n, (uint32_t)P1_TILE, per_tile ? nullptr : tile_lo,
                                         tile_hi);
    if (per_tile)
      k_tile_traces<<<ceil_div((uint64_t)ntiles, 256), 256, 0, st>>>(off, T, n, (uint32_t)P1_TILE, ntiles, tile_lo,
                                                                     tile_hi);
    ctx->stage_end("trace_prep", st);
    ctx->launches += 1 + per_tile;
  }

  // ---- pass 1
  // counters: [0] orphans [1] ambiguities [2] pending [3] nonmono [4] n_failed
  //           [5] unsorted [6] ambiguities after resolution [7] any slow trace
  uint32_t* counters = ctx->d<uint32_t>("c.counters", 16);
  XSP_CUDA(cudaMemsetAsync(counters, 0, 16 * 4, st));
  P1Args a;
  a.span_id = c->span_id;
  a.flags = c->flags;
  a.begin = c->begin_ns;
  a.end = c->end_ns;
  a.parent = c->parent_id;
  a.cid = c->cid;
  a.n = n;
  a.off = off;
  a.T = T;
  a.levels = tr->levels;
  a.model_row = model_row;
  a.mb = mb;
  a.me = me;
  a.msid = msid;
  a.tile_lo = tile_lo;
  a.tile_hi = tile_hi;
  a.tile_agg = ctx->d<Full>("c.tile_agg", ntiles + 1);
  a.tile_prefix = ctx->d<Full>("c.tile_prefix", ntiles / 32 + 2);
  a.ntiles = ntiles;
  a.tile_excl = ctx->d<Full>("c.tile_excl", ntiles + 1);
  a.warp_excl = ctx->d<Full>("c.warp_excl", (uint64_t)ntiles * P1_WARPS + 1);
  a.placed8 = ctx->d<uint8_t>("c.placed8", n / 8 + 16);
  a.group_sum = ctx->d<Full>("c.tile_gsum", ntiles / 32 + 2);
  a.group_done = ctx->d<uint32_t>("c.group_done", ntiles / 32 + 2);
  XSP_CUDA(cudaMemsetAsync(a.group_done, 0, (ntiles / 32 + 2) * 4, st));
  a.unsorted = counters + 5;
  a.err_key = err_key;
  a.layer_row = ctx->d<uint32_t>("o.layer_row", n);
  a.layer_dur = ctx->d<uint64_t>("o.layer_dur", n);
  a.layer_attr_row = ctx->d<uint32_t>("o.layer_attr_row", n);
  a.kl = ctx->d<KlEnt>("c.kl", n);
  a.kl_mrow = ctx->d<uint32_t>("c.kl_mrow", n);
  a.ex = ctx->d<ExEnt>("c.ex", n);
  a.t_layer_off = ctx->d<uint32_t>("o.t_layer_off", T + 1);
  a.t_kl_off = ctx->d<uint32_t>("c.t_kl_off", T + 1);
  a.t_ex_off = ctx->d<uint32_t>("c.t_ex_off", T + 1);
  Orphans orph;
  // Orphan / ambiguity / explicit-parent lists are rare: sized for a fraction
  // of the spans (or the size a previous call needed); overflow is detected at
  // the read-backs and the call is redone with room for every entry.
  auto list_cap = [&](uint64_t hint) {
    const uint64_t lo = std::min<uint64_t>(2 * n + 32, n / 16 + 4096);
    return (uint32_t)std::min<uint64_t>(std::max<uint64_t>(hint, lo), 0xFFFFFFF0ull);
  };
  const uint32_t orph_cap = list_cap(ctx->cap_orph);
  orph.tc = ctx->d<uint64_t>("c.o_tc", orph_cap);
  orph.key = ctx->d<uint64_t>("c.o_key", orph_cap);
  orph.row = ctx->d<uint32_t>("c.o_row", orph_cap);
  orph.reason = ctx->d<uint8_t>("c.o_reason", orph_cap);
  orph.cap = orph_cap;
  orph.count = counters + 0;
  a.orph = orph;
  a.parents_only = parents_only;
  a.amb_cap = list_cap(ctx->cap_amb);
  a.pend_cap = list_cap(ctx->cap_pend);
  a.amb_kl = ctx->d<uint32_t>("c.amb_kl", a.amb_cap);
  a.amb_gx = ctx->d<uint32_t>("c.amb_gx", a.amb_cap);
  a.amb_count = counters + 1;
  a.pend_kl = ctx->d<uint32_t>("c.pend_kl", a.pend_cap);
  a.pend_count = counters + 2;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  a.bulk = n >= (uint64_t)P1_TILE && al16(c->begin_ns) && al16(c->end_ns) && al16(c->cid) &&
           al16(c->parent_id) && al16(c->flags);
  P1Maps maps;
  memset(&maps, 0, sizeof(maps));
  if (a.bulk) {
    col_tmap(&maps.begin, c->begin_ns, n);
    col_tmap(&maps.end, c->end_ns, n);
    col_tmap(&maps.cid, c->cid, n);
    col_tmap(&maps.parent, c->parent_id, n);
  }
  // hints from the previous call on this ctx: a clean batch goes straight to the
  // direct kernel-table emit; after a batch with exceptions or reordered
  // executions the optimistic clean gather is skipped (a wrong hint costs time,
  // never correctness: both paths verify)
  const bool try_clean = !parents_only && !ctx->unclean_hint;
  const bool direct = try_clean && ctx->direct_hint;
  if (try_clean) {
    out->kernel_launch_row = ctx->d<uint32_t>("o.k_launch", n);
    out->kernel_exec_row = ctx->d<uint32_t>("o.k_exec", n);
    out->kernel_metric_row = ctx->d<uint32_t>("o.k_mrow", n);
    out->kernel_dur = ctx->d<uint64_t>("o.k_dur", n);
    out->kernel_name = ctx->d<uint32_t>("o.k_name", n);
    out->kernel_occ = ctx->d<double>("o.k_occ", n);
    out->layer_kernel_off = ctx->d<uint32_t>("o.l_koff", n + 1);
  }
  if (direct) {
    a.k_launch = out->kernel_launch_row;
    a.k_exec = out->kernel_exec_row;
    a.k_mrow = out->kernel_metric_row;
    a.k_dur = out->kernel_dur;
    a.k_name = out->kernel_name;
    a.k_occ = out->kernel_occ;
    a.l_koff = out->layer_kernel_off;
    a.name = c->name_id;
    a.occ = c->occupancy;
    a.t_dmin = ctx->d<unsigned long long>("c.t_dmin", T + 1);
    a.t_dmax = ctx->d<unsigned long long>("c.t_dmax", T + 1);
    a.direct_fail = counters + 7;
    XSP_CUDA(cudaMemsetAsync(a.t_dmin, 0xFF, (T + 1) * 8ull, st));
    XSP_CUDA(cudaMemsetAsync(a.t_dmax, 0, (T + 1) * 8ull, st));
  }
  if (ntiles) {
    XSP_CUDA(cudaFuncSetAttribute(k_pass1<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P1_SMEM));
    XSP_CUDA(cudaFuncSetAttribute(k_pass1<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P1_SMEM));
    ctx->stage_begin("pass1_reduce", st);
    XSP_CUDA(cudaFuncSetAttribute(k_p1_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P1_RED_SMEM));
    k_p1_reduce<<<ntiles, P1_THREADS, P1_RED_SMEM, st>>>(a, maps);
    ctx->stage_end("pass1_reduce", st);
    ctx->stage_begin("pass1_scan", st);
    k_p1_scan<<<1, P1_SCAN_THREADS, 0, st>>>(a.group_sum, (ntiles + 31) / 32, a.tile_prefix);
    k_p1_tile_prefix<<<ceil_div((uint64_t)ntiles * 32, 256), 256, 0, st>>>(a.tile_agg, a.tile_prefix, ntiles,
                                                                           a.tile_excl);
    ctx->stage_end("pass1_scan", st);
    ctx->stage_begin("pass1", st);
    if (direct)
      k_pass1<true><<<ntiles, P1_THREADS, P1_SMEM, st>>>(a, maps);
    else
      k_pass1<false><<<ntiles, P1_THREADS, P1_SMEM, st>>>(a, maps);
    ctx->stage_end("pass1", st);
    ctx->launches += 4;
  }
  uint32_t* totals = ctx->d<uint32_t>("c.totals", 8);
  uint32_t* htot = ctx->h<uint32_t>("c.totals_h", 16);
  if (direct) {
    out->trace_kernel_off = ctx->d<uint32_t>("o.t_koff", T + 1);
    out->trace_status = ctx->d<int32_t>("o.t_status", T);
    out->trace_err_row = ctx->d<uint32_t>("o.t_err_row", 2ull * T);
    FinishArgs fa;
    fa.off = off;
    fa.T = T;
    fa.n = n;
    fa.tile_prefix = a.tile_prefix;
    fa.ntiles = ntiles;
    fa.t_layer_off = a.t_layer_off;
    fa.t_kl_off = a.t_kl_off;
    fa.t_ex_off = a.t_ex_off;
    fa.totals = totals;
    fa.dmin = a.t_dmin;
    fa.dmax = a.t_dmax;
    fa.l_koff = out->layer_kernel_off;
    fa.t_koff = out->trace_kernel_off;
    fa.model_row = model_row;
    fa.err_key = err_key;
    fa.status = out->trace_status;
    fa.err_row = out->trace_err_row;
    fa.counters = counters;
    fa.h_totals = htot;
    ctx->hc_layer_key = ctx->hc_kernel_key = nullptr;
    fa.h_loff = ctx->h<uint32_t>("c.hc_loff", T + 1);
    fa.h_koff = ctx->h<uint32_t>("c.hc_koff", T + 1);
    ctx->stage_begin("gather", st);
    k_direct_finish<<<ceil_div((uint64_t)T + 1, 256), 256, 0, st>>>(fa);
    ctx->stage_end("gather", st);
    ++ctx->launches;
  } else {
    k_pass1_tail<<<ceil_div((uint64_t)T + 1, 256), 256, 0, st>>>(off, T, n, a.tile_prefix, ntiles, a.t_layer_off,
                                                                 a.t_kl_off, a.t_ex_off, totals);
    ++ctx->launches;
  }
  // ---- optimistic clean path, launched before any host round trip: a batch
  // with no orphan, ambiguity or explicit-parent kernel whose traces are all
  // merge-aligned fuses launch r with exec r (k_gather_fast verifies it). Buffers
  // are sized by the span count; the device totals gate the kernels. ONE
  // read-back then decides: done, unsorted, or the general path below.
  auto* no_dup = ctx->d<unsigned long long>("c.no_dup", T);
  if (try_clean && !direct) {
    ctx->stage_begin("gather", st);
    {
      const unsigned gb = std::min<uint64_t>(ceil_div((uint64_t)n + 1, 256), 148u * 8u);
      k_gather_fast<<<gb, 256, 0, st>>>(totals, a.kl, a.ex, c->flags, a.t_kl_off, a.t_ex_off, T, c->cid,
                                        c->name_id, c->occupancy, out->kernel_launch_row,
                                        out->kernel_exec_row, out->kernel_metric_row, out->kernel_dur,
                                        out->kernel_name, out->kernel_occ, out->layer_kernel_off, counters + 7);
    }
    ++ctx->launches;
    out->trace_kernel_off = ctx->d<uint32_t>("o.t_koff", T + 1);
    launch(ctx, k_trace_kernel_off, (uint64_t)T + 1, st, T, a.t_layer_off, out->layer_kernel_off,
           out->trace_kernel_off);
    XSP_CUDA(cudaMemsetAsync(no_dup, 0xFF, T * 8ull, st));
    out->trace_status = ctx->d<int32_t>("o.t_status", T);
    out->trace_err_row = ctx->d<uint32_t>("o.t_err_row", 2ull * T);
    launch(ctx, k_status, T, st, T, model_row, err_key, no_dup, no_dup, a.ex, a.kl, out->trace_status,
           out->trace_err_row, counters + 4);
    cache_offsets_begin(ctx, a.t_layer_off, out->trace_kernel_off, T, st);
    ctx->stage_end("gather", st);
  }
  if (!direct) {
    xfer_small(htot, totals, 5 * 4, st);
    xfer_small(htot + 8, counters, 8 * 4, st);
  }
  XSP_CUDA(cudaStreamSynchronize(st));
  const uint32_t nl = htot[0], nkl = htot[1], nex = htot[2];
  const uint32_t n_amb_raw = htot[9], n_pend = htot[10];
  if (htot[8] > orph_cap || n_amb_raw > a.amb_cap || n_pend > a.pend_cap) {
    ctx->cap_orph = std::max<uint64_t>(ctx->cap_orph, htot[8] + htot[8] / 4 + 1024);
    ctx->cap_amb = std::max<uint64_t>(ctx->cap_amb, n_amb_raw + n_amb_raw / 4 + 1024);
    ctx->cap_pend = std::max<uint64_t>(ctx->cap_pend, n_pend + n_pend / 4 + 1024);
    throw ListOverflow{};
  }
  if (htot[13]) {
    // not in timeline order (span.hpp:161-163)
    (void)sort_if_needed;
    throw std::runtime_error("UNSORTED");
  }
  const bool clean = try_clean && htot[8] == 0 && n_pend == 0 && n_amb_raw == 0 && htot[15] == 0;
  if (try_clean) {
    ctx->direct_hint = clean;
    ctx->unclean_hint = !clean && (htot[8] || n_pend || n_amb_raw || htot[15]);
  }
  if (clean) {
    cache_offsets_end(ctx, a.t_layer_off, out->trace_kernel_off, T);
    out->n_traces = T;
    out->n_failed = htot[12];
    out->trace_model_row = model_row;
    out->n_kernels = nkl;
    out->n_layers = nl;
    out->layer_row = a.layer_row;
    out->layer_dur = a.layer_dur;
    out->layer_attr_row = a.layer_attr_row;
    out->trace_layer_off = a.t_layer_off;
    out->n_orphans = 0;
    out->orphan_row = ctx->d<uint32_t>("o.orphan_row", 1);
    out->orphan_reason = ctx->d<uint8_t>("o.orphan_reason", 1);
    out->trace_orphan_off = ctx->d<uint32_t>("o.t_orph_off", T + 1);
    XSP_CUDA(cudaMemsetAsync(out->trace_orphan_off, 0, (T + 1) * 4ull, st));
    out->n_ambiguities = 0;
    out->n_candidates = 0;
    out->trace_amb_off = ctx->d<uint32_t>("o.t_amb_off", T + 1);
    out->amb_row = ctx->d<uint32_t>("o.amb_row", 1);
    out->amb_cand_off = ctx->d<uint32_t>("o.amb_cand_off", 1);
    out->amb_cand_row = ctx->d<uint32_t>("o.amb_cand_row", 1);
    XSP_CUDA(cudaMemsetAsync(out->trace_amb_off, 0, (T + 1) * 4ull, st));
    XSP_CUDA(cudaMemsetAsync(out->amb_cand_off, 0, 4, st));
    return;
  }
  if (try_clean) XSP_CUDA(cudaMemsetAsync(counters + 4, 0, 4 * 4, st));  // general path: reset n_failed, flags
  if (direct) {
    // the guess was wrong: pass 1 again, writing the kernel-list / exec entries
    // the general join needs (same outputs otherwise; the rare-entry lists are
    // refilled, so their counters restart)
    XSP_CUDA(cudaMemsetAsync(counters, 0, 3 * 4, st));
    if (ntiles) {
      ctx->stage_begin("pass1", st);
      k_pass1<false><<<ntiles, P1_THREADS, P1_SMEM, st>>>(a, maps);
      ctx->stage_end("pass1", st);
      ++ctx->launches;
    }
  }

  // ---- explicit parents
  if (n_pend) {
    uint32_t* t_uns = ctx->d<uint32_t>("c.t_uns", T);
    XSP_CUDA(cudaMemsetAsync(t_uns, 0, T * 4ull, st));
    launch(ctx, k_layer_ids_sorted, nl, st, a.layer_row, c->span_id, a.t_layer_off, T, nl, t_uns);
    launch(ctx, k_resolve_explicit, n_pend, st, a.pend_kl, a.pend_count, a.kl, c->parent_id, c->span_id,
           a.layer_row, a.t_layer_off, a.t_kl_off, T, t_uns, orph);
  }

  // ---- rare containment cases: exact candidate count by scanning back
  uint32_t n_amb = 0;
  MaxTree mt;
  memset(&mt, 0, sizeof(mt));
  if (n_amb_raw) {  // the layers' max tree for the exact candidate walks
    mt.layer_row = a.layer_row;
    mt.end = c->end_ns;
    mt.n[0] = nl;
    mt.levels = 1;
    const uint64_t* prev = nullptr;
    while (mt.n[mt.levels - 1] > 32 && mt.levels < kMtLevels) {
      const int L = mt.levels;
      const uint32_t nin = mt.n[L - 1];
      mt.n[L] = (nin + 31) / 32;
      uint64_t* lv = ctx->d<uint64_t>(L == 1 ? "c.mt1" : L == 2 ? "c.mt2" : L == 3 ? "c.mt3" : L == 4 ? "c.mt4"
                                                                    : L == 5 ? "c.mt5" : "c.mt6", mt.n[L]);
      k_mt_level<<<ceil_div((uint64_t)mt.n[L], 8), 256, 0, st>>>(prev, a.layer_row, c->end_ns, nin, lv);
      ++ctx->launches;
      mt.lv[L] = lv;
      prev = lv;
      ++mt.levels;
    }
    uint32_t* keep = ctx->d<uint32_t>("c.amb_keep", n_amb_raw + 1);
    uint32_t* pos = ctx->d<uint32_t>("c.amb_pos", n_amb_raw + 1);
    launch(ctx, k_amb_resolve, n_amb_raw, st, n_amb_raw, a.amb_kl, a.amb_gx, a.kl, c->end_ns, a.t_kl_off,
           a.t_layer_off, T, mt, keep, orph);
    uint32_t* scan_tmp = ctx->d<uint32_t>("c.scan_tmp", scan_scratch_elems(n + 16));
    exclusive_scan<uint32_t, uint32_t>(keep, pos, n_amb_raw, scan_tmp, counters + 6, st, &ctx->launches);
    uint32_t* kl2 = ctx->d<uint32_t>("c.amb_kl2", n_amb_raw);
    uint32_t* gx2 = ctx->d<uint32_t>("c.amb_gx2", n_amb_raw);
    launch(ctx, k_amb_compact, n_amb_raw, st, n_amb_raw, keep, pos, a.amb_kl, a.amb_gx, kl2, gx2);
    n_amb = read_u32(ctx, counters + 6, st);
    a.amb_kl = kl2;
    a.amb_gx = gx2;
  }

  // ---- ambiguities, ordered by (trace, span_id)
  out->n_ambiguities = n_amb;
  out->trace_amb_off = ctx->d<uint32_t>("o.t_amb_off", T + 1);
  out->amb_row = ctx->d<uint32_t>("o.amb_row", n_amb);
  out->amb_cand_off = ctx->d<uint32_t>("o.amb_cand_off", n_amb + 1);
  out->n_candidates = 0;
  if (n_amb) {
    RadixScratch rs = radix_scratch(ctx, n_amb);
    uint64_t* ksid = ctx->d<uint64_t>("c.amb_ksid", n_amb);
    uint64_t* ktr = ctx->d<uint64_t>("c.amb_ktr", n_amb);
    uint64_t* ktr2 = ctx->d<uint64_t>("c.amb_ktr2", n_amb);
    uint32_t* idx = ctx->d<uint32_t>("c.amb_idx", n_amb);
    launch(ctx, k_amb_keys, n_amb, st, a.amb_kl, n_amb, a.kl, c->span_id, a.t_kl_off, T, ksid, ktr, idx);
    radix_sort_pairs(ksid, idx, n_amb, 0, 64, rs, st, &ctx->launches);
    launch(ctx, k_gather_u64, n_amb, st, ktr, idx, ktr2, n_amb);
    radix_sort_pairs(ktr2, idx, n_amb, 0, 32, rs, st, &ctx->launches);
    uint32_t* cnt = ctx->d<uint32_t>("c.amb_cnt", n_amb + 1);
    launch(ctx, k_amb_count, n_amb, st, idx, n_amb, a.amb_kl, a.amb_gx, a.kl, c->end_ns, a.t_kl_off,
           a.t_layer_off, T, mt, cnt);
    uint32_t* scan_tmp = ctx->d<uint32_t>("c.scan_tmp", scan_scratch_elems(n + 16));
    uint32_t* tot = ctx->d<uint32_t>("c.amb_tot", 1);
    exclusive_scan<uint32_t, uint32_t>(cnt, out->amb_cand_off, n_amb, scan_tmp, tot, st, &ctx->launches);
    XSP_CUDA(cudaMemcpyAsync(out->amb_cand_off + n_amb, tot, 4, cudaMemcpyDeviceToDevice, st));
    uint32_t ncand = read_u32(ctx, tot, st);
    out->n_candidates = ncand;
    out->amb_cand_row = ctx->d<uint32_t>("o.amb_cand_row", ncand);
    launch(ctx, k_amb_fill, n_amb, st, idx, n_amb, a.amb_kl, a.amb_gx, a.kl, c->end_ns, c->span_id, a.t_kl_off,
           a.t_layer_off, T, mt, out->amb_cand_off, out->amb_row, out->amb_cand_row);
    launch(ctx, k_csr_by_trace, (uint64_t)T + 1, st, T, n_amb, ktr2, 0, out->trace_amb_off);
  } else {
    out->amb_cand_row = ctx->d<uint32_t>("o.amb_cand_row", 1);
    XSP_CUDA(cudaMemsetAsync(out->trace_amb_off, 0, (T + 1) * 4ull, st));
    XSP_CUDA(cudaMemsetAsync(out->amb_cand_off, 0, 4, st));
  }

  // ---- cid join: merge-aligned check, hash table for the other traces
  ctx->stage_begin("join", st);
  JoinArgs j;
  j.ex = a.ex;
  j.cid = c->cid;
  j.kl = a.kl;
  j.flags = c->flags;
  j.t_ex_off = a.t_ex_off;
  j.t_kl_off = a.t_kl_off;
  uint32_t* t_slow = ctx->d<uint32_t>("c.t_slow", T + 1);
  uint32_t* t_nonmono = ctx->d<uint32_t>("c.t_nonmono", T + 1);
  uint32_t* t_dense = ctx->d<uint32_t>("c.t_dense", T + 1);
  uint64_t* t_lmin = ctx->d<uint64_t>("c.t_lmin", T + 1);
  uint64_t* t_lmax = ctx->d<uint64_t>("c.t_lmax", T + 1);
  j.t_slow = t_slow;
  j.T = T;
  j.n_ex = nex;
  j.n_kl = nkl;
  uint32_t any_slow = 0;
  if (!parents_only) {
    XSP_CUDA(cudaMemsetAsync(t_lmin, 0xFF, (T + 1) * 8ull, st));
    XSP_CUDA(cudaMemsetAsync(t_lmax, 0, (T + 1) * 8ull, st));
    XSP_CUDA(cudaMemsetAsync(t_nonmono, 0, (T + 1) * 4ull, st));
    launch(ctx, k_join_counts, T, st, a.t_kl_off, a.t_ex_off, T, t_slow, counters + 7);
    launch(ctx, k_join_check, ceil_div((uint64_t)nkl, JC_ITEMS), st, nkl, a.kl, a.ex, c->cid, c->flags,
           a.t_kl_off, a.t_ex_off, T, t_slow, counters + 7, reinterpret_cast<unsigned long long*>(t_lmin),
           reinterpret_cast<unsigned long long*>(t_lmax), t_nonmono);
    any_slow = read_u32(ctx, counters + 7, st);
  }
  auto* dup_ex = ctx->d<unsigned long long>("c.dup_ex", T);
  auto* dup_kl = ctx->d<unsigned long long>("c.dup_kl", T);
  XSP_CUDA(cudaMemsetAsync(dup_ex, 0xFF, T * 8ull, st));
  XSP_CUDA(cudaMemsetAsync(dup_kl, 0xFF, T * 8ull, st));
  j.ex_slot = ctx->d<uint32_t>("c.ex_slot", nex + 1);
  j.kl_slot = ctx->d<uint32_t>("c.kl_slot", nkl + 1);
  uint64_t* roff = nullptr;
  if (any_slow) {
    uint64_t* rsize = ctx->d<uint64_t>("c.rsize", T + 1);
    roff = ctx->d<uint64_t>("c.roff", T + 1);
    if (getenv("XSP_JOIN_HASH")) {
      XSP_CUDA(cudaMemsetAsync(t_lmin, 0xFF, (T + 1) * 8ull, st));
    } else {
      launch(ctx, k_join_direct, T, st, a.t_kl_off, t_slow, T, t_lmin, t_lmax);
      launch(ctx, k_join_far, nex, st, nex, a.ex, c->cid, a.t_ex_off, T, t_lmin, t_lmax);
    }
    j.t_lmin = t_lmin;
    launch(ctx, k_region_size, T, st, a.t_kl_off, a.t_ex_off, t_slow, t_lmin, t_lmax, T, rsize, t_nonmono,
           t_dense);
    uint64_t* scan64 = ctx->d<uint64_t>("c.scan64", scan_scratch_elems(T + 1));
    exclusive_scan<uint64_t, uint64_t>(rsize, roff, T, scan64, roff + T, st, &ctx->launches);
    uint64_t* hroff = ctx->h<uint64_t>("c.roff_h", 1);
    xfer_small(hroff, roff + T, 8, st);
    XSP_CUDA(cudaStreamSynchronize(st));
    const uint64_t nslots = *hroff;
    j.roff = roff;
    j.owner = ctx->d<uint32_t>("c.owner", nslots);
    j.sl_exec = ctx->d<uint32_t>("c.sl_exec", nslots);
    j.sl_launch = ctx->d<uint32_t>("c.sl_launch", nslots);
    j.t_dup = ctx->d<uint32_t>("c.t_dup", T);
    j.t_dense = t_dense;
    XSP_CUDA(cudaMemsetAsync(j.owner, 0, nslots * 4, st));
    XSP_CUDA(cudaMemsetAsync(j.sl_exec, 0xFF, nslots * 4, st));
    XSP_CUDA(cudaMemsetAsync(j.sl_launch, 0xFF, nslots * 4, st));
    XSP_CUDA(cudaMemsetAsync(j.t_dup, 0, T * 4ull, st));
    j.any_dup = ctx->d<uint32_t>("c.any_dup", 1);
    XSP_CUDA(cudaMemsetAsync(j.any_dup, 0, 4, st));
    launch(ctx, k_join_insert, (uint64_t)nex + nkl, st, j);
    k_join_dups<<<(unsigned)std::min<uint64_t>(ceil_div((uint64_t)nex + nkl, 256), 148u * 8u), 256, 0, st>>>(
        j, dup_ex, dup_kl);
    ++ctx->launches;
  } else {
    j.sl_exec = j.sl_launch = nullptr;
  }
  ctx->stage_end("join", st);

  // ---- fusion, kept kernels, leftover execs
  ctx->stage_begin("fuse", st);
  FuseArgs fa;
  fa.n_kl = nkl;
  fa.n_ex = nex;
  fa.T = T;
  fa.kl = a.kl;
  fa.ex = a.ex;
  fa.flags = c->flags;
  fa.t_slow = t_slow;
  fa.t_dense = t_dense;
  fa.roff = roff;
  fa.kl_slot = j.kl_slot;
  fa.sl_exec = j.sl_exec;
  fa.sl_launch = j.sl_launch;
  fa.ex_slot = j.ex_slot;
  fa.sid = c->span_id;
  fa.t_kl_off = a.t_kl_off;
  fa.t_ex_off = a.t_ex_off;
  fa.kept = ctx->d<uint32_t>("c.kept", nkl + 1);
  fa.kl_exec = ctx->d<uint32_t>("c.kl_exec", nkl + 1);
  fa.orph = orph;
  fa.any_slow = any_slow != 0;
  fa.parents_only = parents_only;
  fa.drop = ctx->d<uint32_t>("c.fuse_drop", 2);
  XSP_CUDA(cudaMemsetAsync(fa.drop, 0, 8, st));
  launch(ctx, k_fuse, nkl, st, fa);
  if (any_slow) launch(ctx, k_leftover, nex, st, fa);
  // every entry kept and in timeline order (the common case, e.g. executions
  // reordered across streams): no compaction, the kernel list is the order
  xfer_small(htot, fa.drop, 8, st);
  XSP_CUDA(cudaStreamSynchronize(st));
  const bool all_kept = htot[0] == 0 && htot[1] == 0;
  uint64_t* kkey = nullptr;
  uint32_t* kval = nullptr;
  uint32_t nk = nkl;
  htot[1] = 0;
  if (!all_kept) {
    uint32_t* kpos = ctx->d<uint32_t>("c.kpos", nkl + 1);
    uint32_t* scan_tmp = ctx->d<uint32_t>("c.scan_tmp", scan_scratch_elems(n + 16));
    uint32_t* nk_d = ctx->d<uint32_t>("c.nk", 1);
    exclusive_scan<uint32_t, uint32_t>(fa.kept, kpos, nkl, scan_tmp, nk_d, st, &ctx->launches);
    kkey = ctx->d<uint64_t>("c.kkey", nkl + 1);
    kval = ctx->d<uint32_t>("c.kval", nkl + 1);
    launch(ctx, k_compact_kernels, nkl, st, nkl, fa.kept, kpos, a.kl, kkey, kval, counters + 3);
    xfer_small(htot, nk_d, 4, st);
    xfer_small(htot + 1, counters + 3, 4, st);
    XSP_CUDA(cudaStreamSynchronize(st));
    nk = htot[0];
  }
  ctx->stage_end("fuse", st);
  if (htot[1]) {
    // explicit parents broke the timeline order of layers: stable sort by layer
    RadixScratch rs = radix_scratch(ctx, nk);
    radix_sort_pairs(kkey, kval, nk, 0, 32, rs, st, &ctx->launches);
  }
  ctx->stage_begin("gather", st);
  out->n_kernels = nk;
  out->kernel_launch_row = ctx->d<uint32_t>("o.k_launch", nk);
  out->kernel_exec_row = ctx->d<uint32_t>("o.k_exec", nk);
  out->kernel_metric_row = ctx->d<uint32_t>("o.k_mrow", nk);
  out->kernel_dur = ctx->d<uint64_t>("o.k_dur", nk);
  out->kernel_name = ctx->d<uint32_t>("o.k_name", nk);
  out->kernel_occ = ctx->d<double>("o.k_occ", nk);
  launch(ctx, k_gather_kernels, nk, st, nk, kval, a.kl, a.kl_mrow, fa.kl_exec, a.ex, c->flags, c->begin_ns,
         c->end_ns, c->name_id, c->occupancy, out->kernel_launch_row, out->kernel_exec_row,
         out->kernel_metric_row, out->kernel_dur, out->kernel_name, out->kernel_occ);
  out->n_layers = nl;
  out->layer_row = a.layer_row;
  out->layer_dur = a.layer_dur;
  out->layer_attr_row = a.layer_attr_row;
  out->layer_kernel_off = ctx->d<uint32_t>("o.l_koff", nl + 1);
  if (all_kept)
    launch(ctx, k_layer_kernel_off_kl, (uint64_t)nk + 1, st, nl, nk, a.kl, out->layer_kernel_off);
  else
    launch(ctx, k_layer_kernel_off, (uint64_t)nk + 1, st, nl, nk, kkey, out->layer_kernel_off);
  out->trace_layer_off = a.t_layer_off;
  out->trace_kernel_off = ctx->d<uint32_t>("o.t_koff", T + 1);
  launch(ctx, k_trace_kernel_off, (uint64_t)T + 1, st, T, a.t_layer_off, out->layer_kernel_off,
         out->trace_kernel_off);
  ctx->stage_end("gather", st);

  // ---- orphans in reference order
  const uint32_t no = read_u32(ctx, orph.count, st);
  if (no > orph_cap) {  // the fusion phases added more than the room left
    ctx->cap_orph = std::max<uint64_t>(ctx->cap_orph, no + no / 4 + 1024);
    throw ListOverflow{};
  }
  out->n_orphans = no;
  out->orphan_row = ctx->d<uint32_t>("o.orphan_row", no);
  out->orphan_reason = ctx->d<uint8_t>("o.orphan_reason", no);
  out->trace_orphan_off = ctx->d<uint32_t>("o.t_orph_off", T + 1);
  if (no) {
    RadixScratch rs = radix_scratch(ctx, no);
    uint32_t* idx = ctx->d<uint32_t>("c.o_idx", no);
    uint64_t* k1 = ctx->d<uint64_t>("c.o_k1", no);
    uint64_t* k2 = ctx->d<uint64_t>("c.o_k2", no);
    launch(ctx, k_iota, no, st, idx, no);
    XSP_CUDA(cudaMemcpyAsync(k1, orph.key, no * 8ull, cudaMemcpyDeviceToDevice, st));
    radix_sort_pairs(k1, idx, no, 0, 64, rs, st, &ctx->launches);
    launch(ctx, k_gather_u64, no, st, orph.tc, idx, k2, no);
    radix_sort_pairs(k2, idx, no, 0, 40, rs, st, &ctx->launches);
    launch(ctx, k_orphan_out, no, st, no, idx, orph.row, orph.reason, out->orphan_row, out->orphan_reason);
    launch(ctx, k_csr_by_trace, (uint64_t)T + 1, st, T, no, k2, 3, out->trace_orphan_off);
  } else {
    XSP_CUDA(cudaMemsetAsync(out->trace_orphan_off, 0, (T + 1) * 4ull, st));
  }

  // ---- status
  out->n_traces = T;
  out->trace_status = ctx->d<int32_t>("o.t_status", T);
  out->trace_err_row = ctx->d<uint32_t>("o.t_err_row", 2ull * T);
  out->trace_model_row = model_row;
  launch(ctx, k_status, T, st, T, model_row, err_key, dup_ex, dup_kl, a.ex, a.kl, out->trace_status,
         out->trace_err_row, counters + 4);
  uint32_t* hf = ctx->h<uint32_t>("c.failed_h", 1);
  xfer_small(hf, counters + 4, 4, st);
  cache_offsets_begin(ctx, out->trace_layer_off, out->trace_kernel_off, T, st);
  XSP_CUDA(cudaStreamSynchronize(st));
  out->n_failed = *hf;
  cache_offsets_end(ctx, out->trace_layer_off, out->trace_kernel_off, T);
  if (!parents_only) {
    const bool was_clean = no == 0 && n_pend == 0 && n_amb_raw == 0 && any_slow == 0;
    ctx->unclean_hint = !was_clean;
    ctx->direct_hint = was_clean;
  }
}

}  // namespace xsp
