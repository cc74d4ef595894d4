// resolve_with_serialized (correlator.cpp:379-456) for a batch of trace pairs:
// trace t of the original (concurrent) batch is resolved against trace t of the
// serialized batch.
//
// The reference identifies an event across the two runs by (level, kind, name,
// occurrence index in timeline order), takes each ambiguous kernel's parent from
// the serialized run's tree, maps that parent back to the original run by its
// event key, sets it as the kernel's explicit parent_id and correlates again.
// Here:
//   1. the serialized batch is correlated (assign_parents) on the device and its
//      parent relation becomes a per-row array (layer -> model, launch -> layer);
//   2. the original batch is correlated (assign_parents) for its ambiguities;
//   3. event keys (trace, level, kind, name_id) of both batches are radix-sorted
//      (stably, so timeline order survives); a span's occurrence is its distance
//      to the first equal key, and an event (key, occurrence) is found by one
//      binary search;
//   4. one thread per ambiguity walks original -> serialized twin -> its parent ->
//      the parent's original twin and patches a copy of parent_id / flags;
//   5. the patched batch is correlated in full.
// Both batches must intern names with one string table (name_id equality is
// name equality). A trace whose serialized twin is itself ambiguous or fails
// gets XSP_T_SER_AMBIGUOUS / XSP_T_SER_FAILED.

#include "ctx.h"
#include "prims.cuh"

namespace xsp {

namespace {

constexpr uint32_t kNo = 0xFFFFFFFFu;

__global__ void k_fill(uint32_t* __restrict__ p, uint64_t n, uint32_t v) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// serialized parent relation: layer -> model span, kernel launch -> layer
__global__ void k_ser_parents(uint32_t nl, const uint32_t* __restrict__ layer_row,
                              const uint32_t* __restrict__ layer_koff, const uint32_t* __restrict__ launch_row,
                              const uint32_t* __restrict__ t_layer_off, const uint32_t* __restrict__ model_row,
                              uint32_t T, uint32_t* __restrict__ par) {
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nl) return;
  uint32_t lo = 0, hi = T;  // trace of layer l: t_layer_off[t] <= l < t_layer_off[t + 1]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (t_layer_off[mid] <= l) lo = mid; else hi = mid;
  }
  const uint32_t lr = layer_row[l];
  par[lr] = model_row[lo];
  for (uint32_t k = layer_koff[l]; k < layer_koff[l + 1]; ++k) par[launch_row[k]] = lr;
}

// event key without the occurrence: trace | level | kind | name_id
__global__ void k_event_keys(uint64_t n, const uint8_t* __restrict__ flags, const uint32_t* __restrict__ name,
                             const uint64_t* __restrict__ off, uint32_t T, uint64_t* __restrict__ key,
                             uint32_t* __restrict__ val, uint32_t* __restrict__ bad) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t t = trace_of(off, 0, T, i);
  const uint32_t nm = name[i];
  if (nm >= (1u << 26)) *bad = 1;
  const uint8_t f = flags[i];
  key[i] = ((uint64_t)t << 30) | ((uint64_t)f_level(f) << 28) | ((uint64_t)f_kind(f) << 26) | nm;
  val[i] = (uint32_t)i;
}

__device__ __forceinline__ uint64_t lower_bound64(const uint64_t* __restrict__ a, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// per row: its key and occurrence (distance to the first equal sorted key)
__global__ void k_event_occ(uint64_t n, const uint64_t* __restrict__ skey, const uint32_t* __restrict__ srow,
                            uint64_t* __restrict__ row_key, uint32_t* __restrict__ row_occ) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint64_t k = skey[p];
  const uint64_t first = (p > 0 && skey[p - 1] == k) ? lower_bound64(skey, p, k) : p;
  const uint32_t r = srow[p];
  row_key[r] = k;
  row_occ[r] = (uint32_t)(p - first);
}

struct EventIndex {
  uint64_t n;
  const uint64_t* skey;  // sorted keys
  const uint32_t* srow;  // rows in sorted order
  const uint64_t* row_key;
  const uint32_t* row_occ;
};

__device__ __forceinline__ uint32_t find_event(const EventIndex& x, uint64_t key, uint32_t occ) {
  const uint64_t p = lower_bound64(x.skey, x.n, key) + occ;
  return (p < x.n && x.skey[p] == key) ? x.srow[p] : kNo;
}

__global__ void k_resolve_patch(uint32_t na, const uint32_t* __restrict__ amb_row, EventIndex orig, EventIndex ser,
                                const uint32_t* __restrict__ ser_par, const uint64_t* __restrict__ span_id,
                                uint64_t* __restrict__ parent, uint8_t* __restrict__ flags) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= na) return;
  const uint32_t a = amb_row[i];
  const uint32_t twin = find_event(ser, orig.row_key[a], orig.row_occ[a]);
  if (twin == kNo) return;  // stays ambiguous
  const uint32_t pr = ser_par[twin];
  if (pr == kNo) return;
  const uint32_t op = find_event(orig, ser.row_key[pr], ser.row_occ[pr]);
  if (op == kNo) return;
  parent[a] = span_id[op];
  flags[a] = (uint8_t)(flags[a] | XSP_F_PARENT);
}

// traces whose serialized twin could not be used
__global__ void k_resolve_status(uint32_t T, const int32_t* __restrict__ ser_status,
                                 const uint32_t* __restrict__ ser_err_row, const uint32_t* __restrict__ ser_amb_off,
                                 int32_t* __restrict__ status, uint32_t* __restrict__ err_row,
                                 uint32_t* __restrict__ n_failed) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  int32_t st = status[t];
  if (ser_status[t] != XSP_T_OK) {
    st = XSP_T_SER_FAILED;
    err_row[2 * t] = ser_err_row[2 * t];
    err_row[2 * t + 1] = ser_err_row[2 * t + 1];
  } else if (ser_amb_off[t + 1] > ser_amb_off[t]) {
    st = XSP_T_SER_AMBIGUOUS;
    err_row[2 * t] = ser_amb_off[t + 1] - ser_amb_off[t];  // ambiguity count (the message quotes it)
    err_row[2 * t + 1] = kNo;
  }
  status[t] = st;
  if (st != XSP_T_OK) atomicAdd(n_failed, 1u);
}

EventIndex build_index(xsp_ctx* ctx, const char* tag, const xsp_span_cols* c, const xsp_traces* tr,
                       uint32_t* bad, cudaStream_t st) {
  const uint64_t n = c->n_spans;
  const std::string p = std::string("r.") + tag;
  uint64_t* key = ctx->d<uint64_t>(p + ".key", n + 1);
  uint32_t* val = ctx->d<uint32_t>(p + ".val", n + 1);
  uint64_t* row_key = ctx->d<uint64_t>(p + ".row_key", n + 1);
  uint32_t* row_occ = ctx->d<uint32_t>(p + ".row_occ", n + 1);
  if (n) {
    k_event_keys<<<ceil_div(n, 256), 256, 0, st>>>(n, c->flags, c->name_id, tr->span_off, tr->n_traces, key, val,
                                                   bad);
    RadixScratch rs;
    rs.keys_alt = ctx->d<uint64_t>("r.rs.keys_alt", n);
    rs.vals_alt = ctx->d<uint32_t>("r.rs.vals_alt", n);
    const uint64_t ce = radix_counts_elems(n);
    rs.counts = ctx->d<uint32_t>("r.rs.counts", ce);
    rs.scan_tmp = ctx->d<uint32_t>("r.rs.scan", scan_scratch_elems(ce));
    rs.and_or = ctx->d<unsigned long long>("r.rs.andor", 2);
    rs.and_or_host = ctx->h<unsigned long long>("r.rs.andor_h", 2);
    radix_sort_pairs(key, val, n, 0, 64, rs, st, &ctx->launches);
    k_event_occ<<<ceil_div(n, 256), 256, 0, st>>>(n, key, val, row_key, row_occ);
    ctx->launches += 2;
  }
  return EventIndex{n, key, val, row_key, row_occ};
}

}  // namespace

void run_resolve(xsp_ctx* ctx, const xsp_span_cols* oc, const xsp_traces* ot, const xsp_span_cols* sc,
                 const xsp_traces* stt, xsp_corr_out* out, cudaStream_t st) {
  const uint32_t T = ot->n_traces;
  if (stt->n_traces != T) throw std::invalid_argument("original and serialized batches hold different trace counts");
  if (T >= (1u << 30)) throw std::invalid_argument("too many traces for resolve_with_serialized");
  const uint64_t no = oc->n_spans, ns = sc->n_spans;
  // 1. serialized run: parent relation, ambiguity counts, statuses
  xsp_corr_out s;
  std::memset(&s, 0, sizeof(s));
  run_correlate(ctx, sc, stt, XSP_CORR_PARENTS_ONLY, &s, st);
  uint32_t* ser_par = ctx->d<uint32_t>("r.ser_par", ns + 1);
  k_fill<<<std::min<uint64_t>(ceil_div(ns + 1, 256), 4096), 256, 0, st>>>(ser_par, ns + 1, kNo);
  if (s.n_layers)
    k_ser_parents<<<ceil_div(s.n_layers, 256), 256, 0, st>>>((uint32_t)s.n_layers, s.layer_row, s.layer_kernel_off,
                                                            s.kernel_launch_row, s.trace_layer_off,
                                                            s.trace_model_row, T, ser_par);
  uint32_t* ser_amb_off = ctx->d<uint32_t>("r.ser_amb_off", T + 1);
  int32_t* ser_status = ctx->d<int32_t>("r.ser_status", T + 1);
  uint32_t* ser_err = ctx->d<uint32_t>("r.ser_err", 2ull * T + 2);
  XSP_CUDA(cudaMemcpyAsync(ser_amb_off, s.trace_amb_off, (T + 1) * 4ull, cudaMemcpyDeviceToDevice, st));
  if (T) {
    XSP_CUDA(cudaMemcpyAsync(ser_status, s.trace_status, T * 4ull, cudaMemcpyDeviceToDevice, st));
    XSP_CUDA(cudaMemcpyAsync(ser_err, s.trace_err_row, 2ull * T * 4, cudaMemcpyDeviceToDevice, st));
  }
  ctx->launches += 2;
  // 2. original run: its ambiguities
  xsp_corr_out o;
  std::memset(&o, 0, sizeof(o));
  run_correlate(ctx, oc, ot, XSP_CORR_PARENTS_ONLY, &o, st);
  const uint32_t na = (uint32_t)o.n_ambiguities;
  uint32_t* amb = ctx->d<uint32_t>("r.amb_row", na + 1);
  if (na) XSP_CUDA(cudaMemcpyAsync(amb, o.amb_row, na * 4ull, cudaMemcpyDeviceToDevice, st));
  // 3. event indexes, 4. patched parent_id / flags
  uint64_t* parent = ctx->d<uint64_t>("r.parent", no + 1);
  uint8_t* flags = ctx->d<uint8_t>("r.flags", no + 1);
  if (no) {
    XSP_CUDA(cudaMemcpyAsync(parent, oc->parent_id, no * 8, cudaMemcpyDeviceToDevice, st));
    XSP_CUDA(cudaMemcpyAsync(flags, oc->flags, no, cudaMemcpyDeviceToDevice, st));
  }
  if (na) {
    uint32_t* bad = ctx->d<uint32_t>("r.bad", 1);
    XSP_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    const EventIndex io = build_index(ctx, "o", oc, ot, bad, st);
    const EventIndex is = build_index(ctx, "s", sc, stt, bad, st);
    k_resolve_patch<<<ceil_div(na, 256), 256, 0, st>>>(na, amb, io, is, ser_par, oc->span_id, parent, flags);
    ++ctx->launches;
    uint32_t* hb = ctx->h<uint32_t>("r.bad_h", 1);
    xfer_small(hb, bad, 4, st);
    XSP_CUDA(cudaStreamSynchronize(st));
    if (*hb) throw std::invalid_argument("resolve_with_serialized: name ids must be below 2^26");
  }
  // 5. the patched run, in full
  xsp_span_cols patched = *oc;
  patched.parent_id = parent;
  patched.flags = flags;
  run_correlate(ctx, &patched, ot, 0, out, st);
  // traces whose serialized twin was ambiguous or failed
  uint32_t* nf = ctx->d<uint32_t>("r.n_failed", 1);
  XSP_CUDA(cudaMemsetAsync(nf, 0, 4, st));
  if (T)
    k_resolve_status<<<ceil_div(T, 256), 256, 0, st>>>(T, ser_status, ser_err, ser_amb_off, out->trace_status,
                                                      out->trace_err_row, nf);
  ++ctx->launches;
  uint32_t* hn = ctx->h<uint32_t>("r.n_failed_h", 1);
  xfer_small(hn, nf, 4, st);
  XSP_CUDA(cudaStreamSynchronize(st));
  out->n_failed = *hn;
}

}  // namespace xsp
