// Chunked, overlapped host pipeline behind xsp_run_host (include/xsp.h).
//
// A host-resident batch is cut at analysis-group boundaries into chunks of
// ~XSP_CHUNK_SPANS spans (traces and groups are independent units, so every
// chunk is a complete sub-problem). While chunk c is correlated and analysed
// on the work stream, chunk c+1's columns stream in on a second (copy) stream
// into the other of two device slots, and chunk c's results stream out into
// the host result columns at their global positions. Row indices and CSR
// offsets of a chunk are re-based on the device before the copy, so the host
// result is byte-identical to a single-shot run. The H2D and D2H copy engines
// run concurrently, so the call costs ~max(H2D, D2H) + one chunk of compute
// instead of their sum.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstddef>
#include <cstdlib>
#include <vector>

#include "ctx.h"
#include "xsp_common.cuh"

namespace xsp {
namespace {

__global__ void k_rebase(uint32_t* __restrict__ p, uint64_t n, uint32_t base) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = p[i];
    if (v != kNone) p[i] = v + base;
  }
}

// what a column counts / what its values index
enum Count : uint8_t { N_T, N_2T, N_L, N_K, N_O, N_A, N_AC, N_G, N_TL, N_TK, N_TN, N_TLK, N_TY, N_COUNTS };
enum Base : uint8_t { B_NONE, B_SPAN, B_METRIC, B_LAYER, B_L, B_K, B_O, B_A, B_AC, B_TL, B_TK, B_TN, B_TY, B_BASES };

struct Field {
  size_t off;   // offsetof the pointer member
  uint32_t esz;
  Count cnt;
  bool csr;     // [count + 1] offsets: the last chunk also writes the sentinel
  Base base;
  const char* name;
  bool lookup = false;  // a span / metric column lookup (skipped under XSP_HOST_OUT_ROWS)
};

#define CF(m, T, c, csr, b) Field{offsetof(xsp_corr_out, m), sizeof(T), c, csr, b, "pc." #m}
#define CFL(m, T, c) Field{offsetof(xsp_corr_out, m), sizeof(T), c, false, B_NONE, "pc." #m, true}
const Field kCorrFields[] = {
    CF(trace_status, int32_t, N_T, false, B_NONE),    CF(trace_err_row, uint32_t, N_2T, false, B_SPAN),
    CF(trace_model_row, uint32_t, N_T, false, B_SPAN), CF(trace_layer_off, uint32_t, N_T, true, B_L),
    CF(trace_kernel_off, uint32_t, N_T, true, B_K),    CF(trace_orphan_off, uint32_t, N_T, true, B_O),
    CF(trace_amb_off, uint32_t, N_T, true, B_A),       CF(layer_row, uint32_t, N_L, false, B_SPAN),
    CF(layer_kernel_off, uint32_t, N_L, true, B_K),    CFL(layer_dur, uint64_t, N_L),
    CF(layer_attr_row, uint32_t, N_L, false, B_LAYER), CF(kernel_launch_row, uint32_t, N_K, false, B_SPAN),
    CF(kernel_exec_row, uint32_t, N_K, false, B_SPAN), CF(kernel_metric_row, uint32_t, N_K, false, B_METRIC),
    CFL(kernel_dur, uint64_t, N_K),      CFL(kernel_name, uint32_t, N_K),
    CFL(kernel_occ, double, N_K),        CF(orphan_row, uint32_t, N_O, false, B_SPAN),
    CF(orphan_reason, uint8_t, N_O, false, B_NONE),    CF(amb_row, uint32_t, N_A, false, B_SPAN),
    CF(amb_cand_off, uint32_t, N_A, true, B_AC),       CF(amb_cand_row, uint32_t, N_AC, false, B_SPAN),
};
#undef CF
#undef CFL

#define TF(m, T, c) Field{offsetof(xsp_tables_out, m), sizeof(T), c, false, B_NONE, "pt." #m}
#define TFB(m, T, c, csr, b) Field{offsetof(xsp_tables_out, m), sizeof(T), c, csr, b, "pt." #m}
const Field kTableFields[] = {
    TF(group_status, int32_t, N_G), TF(group_err_arg, uint32_t, N_G),
    TFB(group_layer_off, uint32_t, N_G, true, B_TL), TFB(group_kernel_off, uint32_t, N_G, true, B_TK),
    TFB(group_name_off, uint32_t, N_G, true, B_TN),
    TF(k_name, uint32_t, N_TK), TF(k_layer, uint32_t, N_TK), TF(k_lat, double, N_TK), TF(k_flops, uint64_t, N_TK),
    TF(k_read, uint64_t, N_TK), TF(k_write, uint64_t, N_TK), TF(k_occ, double, N_TK), TF(k_ai, double, N_TK),
    TF(k_tput, double, N_TK), TF(k_bound, int8_t, N_TK), TF(k_roofline_in, uint8_t, N_TK),
    TF(l_index, uint32_t, N_TL), TFB(l_row, uint32_t, N_TL, false, B_SPAN), TF(l_layer_lat, double, N_TL),
    TF(l_kern_lat, double, N_TL), TF(l_flops, uint64_t, N_TL), TF(l_read, uint64_t, N_TL),
    TF(l_write, uint64_t, N_TL), TF(l_occ, double, N_TL), TF(l_count, uint64_t, N_TL), TF(l_ai, double, N_TL),
    TF(l_tput, double, N_TL), TF(l_bound, int8_t, N_TL), TF(l_nongpu, double, N_TL),
    TF(l_gpu_share, double, N_TL), TF(l_nongpu_share, double, N_TL), TF(l_flagged, uint8_t, N_TL),
    TF(l_roofline_in, uint8_t, N_TL), TF(l_topk, uint32_t, N_TLK),
    TF(n_name, uint32_t, N_TN), TF(n_count, uint64_t, N_TN), TF(n_lat, double, N_TN), TF(n_pct, double, N_TN),
    TF(n_flops, uint64_t, N_TN), TF(n_read, uint64_t, N_TN), TF(n_write, uint64_t, N_TN), TF(n_occ, double, N_TN),
    TF(n_ai, double, N_TN), TF(n_tput, double, N_TN), TF(n_bound, int8_t, N_TN),
    TF(m_lat, double, N_G), TF(m_kern_lat, double, N_G), TF(m_flops, uint64_t, N_G), TF(m_read, uint64_t, N_G),
    TF(m_write, uint64_t, N_G), TF(m_occ, double, N_G), TF(m_count, uint64_t, N_G), TF(m_ai, double, N_G),
    TF(m_tput, double, N_G), TF(m_bound, int8_t, N_G), TF(m_gpu, double, N_G), TF(m_gpu_pct, double, N_G),
    TF(m_throughput, double, N_G), TF(m_roofline_in, uint8_t, N_G),
    TFB(group_type_off, uint32_t, N_G, true, B_TY),
    TF(y_type, uint32_t, N_TY), TF(y_count, uint64_t, N_TY), TF(y_lat, double, N_TY), TF(y_alloc, int64_t, N_TY),
};
#undef TF
#undef TFB

void*& member(void* s, size_t off) { return *reinterpret_cast<void**>(static_cast<char*>(s) + off); }

struct Chunk {
  uint32_t t0, t1, g0, g1;
  uint64_t s0, s1, m0, m1, l0, l1;
};

// Per-chunk counts and global write positions, indexed by Count / Base.
struct Pos {
  uint64_t n[N_COUNTS] = {};   // element counts of this chunk
  uint64_t at[N_COUNTS] = {};  // global element position of its first element
  uint64_t base[B_BASES] = {}; // value to add (Base)
};

__attribute__((target("popcnt"))) void count_rows(const uint8_t* f, uint64_t n, uint64_t& metric, uint64_t& layer,
                                                  uint64_t& child_parent) {
  // eight flags per step: metric bit -> popcount; level == Layer -> bytes whose
  // low two bits equal XSP_LEVEL_LAYER; child_parent = non-layer spans with an
  // explicit parent_id (they take the explicit-parent path, which reads the
  // span_id column densely)
  constexpr uint64_t kOnes = 0x0101010101010101ull;
  uint64_t m = 0, l = 0, cp = 0, i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, f + i, 8);
    m += __builtin_popcountll(w & (kOnes * XSP_F_METRICS));
    const uint64_t x = (w ^ (kOnes * XSP_LEVEL_LAYER)) & (kOnes * 3u);
    const uint64_t not_layer = (x | (x >> 1)) & kOnes;
    l += 8 - __builtin_popcountll(not_layer);
    cp += __builtin_popcountll(not_layer & (w >> 4));  // XSP_F_PARENT = bit 4
  }
  for (; i < n; ++i) {
    m += (f[i] & XSP_F_METRICS) != 0;
    l += (f[i] & 3u) == XSP_LEVEL_LAYER;
    cp += (f[i] & 3u) != XSP_LEVEL_LAYER && (f[i] & XSP_F_PARENT);
  }
  metric = m;
  layer = l;
  child_parent = cp;
}

// Device alias of a page-locked host column (zero-copy reads over PCIe), or
// nullptr when the memory is pageable or not mapped.
const uint64_t* mapped_alias(const uint64_t* host) {
  if (!host || std::getenv("XSP_NO_ZERO_COPY")) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
  return static_cast<const uint64_t*>(at.devicePointer);
}

// Large copies go out in pieces so that the small transfers of the compute
// stream (count read-backs, group arrays) interleave instead of queueing behind
// a whole column on the same copy engine.
constexpr uint64_t kPiece = 1ull << 40;
void copy_pieces(void* dst, const void* src, uint64_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
  for (uint64_t o = 0; o < bytes; o += kPiece)
    XSP_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                             std::min(kPiece, bytes - o), kind, st));
}

}  // namespace

// Returns false (nothing done) when the batch is too small or the groups are
// not an ordered partition of trace ranges; the caller then runs single-shot.
uint64_t stage_packed(xsp_ctx* ctx, const xsp_packed_cols* pk, uint64_t s0, uint64_t s1, uint8_t* flags,
                      uint32_t* name_id, uint64_t* begin, uint64_t* end, uint64_t* cid, uint64_t* parent,
                      const std::string& tag, cudaStream_t st, void* deferred);
void launch_unpack(xsp_ctx* ctx, const void* args, cudaStream_t st);
uint64_t stage_tables_packed(xsp_ctx* ctx, const xsp_packed_cols* pk, const xsp_span_cols* hc, uint64_t s0,
                             uint64_t s1, uint64_t m0, uint64_t m1, uint64_t l0, uint64_t l1, uint32_t* name_id,
                             uint64_t* flops, uint64_t* rd, uint64_t* wr, double* occ, int64_t* alloc,
                             uint32_t* type_id, const std::string& tag, cudaStream_t st, void* deferred);
void launch_unpack_tables(xsp_ctx* ctx, const void* args, cudaStream_t st);
size_t unpack_tables_args_bytes();
size_t unpack_args_bytes();

bool run_host_chunked(xsp_ctx* ctx, const xsp_span_cols* hc, const xsp_traces* ht, const xsp_groups* groups,
                      const xsp_system_spec* spec, const xsp_analysis_opts* opts, xsp_corr_out* corr_host,
                      xsp_tables_out* tab_host, const xsp_packed_cols* pk) {
  uint64_t target = 12000000;
  if (const char* e = std::getenv("XSP_CHUNK_SPANS")) target = std::strtoull(e, nullptr, 10);
  const uint64_t n = hc->n_spans;
  const uint32_t T = ht->n_traces, G = groups->n_groups;
  if (target == 0 || n < 2 * target || G < 2) return false;
  for (uint32_t g = 0; g + 1 < G; ++g)
    if ((uint64_t)groups->first_trace[g] + groups->n_runs[g] > groups->first_trace[g + 1]) return false;
  if ((uint64_t)groups->first_trace[G - 1] + groups->n_runs[G - 1] > T) return false;
  const uint64_t* off = ht->span_off;

  // ---- plan: cut after the group that brings a chunk to >= target spans
  std::vector<Chunk> ch;
  {
    Chunk c{};
    c.t0 = 0;
    c.g0 = 0;
    for (uint32_t g = 0; g < G; ++g) {
      const uint64_t end_t = (uint64_t)groups->first_trace[g] + groups->n_runs[g];
      if (g + 1 < G && off[end_t] - off[c.t0] >= target) {
        c.t1 = groups->first_trace[g + 1];
        c.g1 = g + 1;
        ch.push_back(c);
        c = Chunk{};
        c.t0 = groups->first_trace[g + 1];
        c.g0 = g + 1;
      }
    }
    c.t1 = T;
    c.g1 = G;
    // the compute + D2H of the final chunk is the only part not hidden behind
    // the input stream, but every chunk also has ~1 ms of fixed cost (launches,
    // read-backs): measured on C3 (12 M-span chunks), no tail split beat
    // geometric tails down to 1 M / 3 M / 6 M spans by 0.2-0.6 ms. XSP_TAIL_SPANS
    // cuts the tail ~2/3 : 1/3 at group boundaries until it is below that size.
    uint64_t tail_min = target;
    if (const char* e = std::getenv("XSP_TAIL_SPANS")) tail_min = std::strtoull(e, nullptr, 10);
    for (;;) {
      const uint64_t rem = off[T] - off[c.t0];
      if (rem <= tail_min) break;
      bool cut = false;
      for (uint32_t g = c.g0; g + 1 < G; ++g) {
        const uint64_t end_t = (uint64_t)groups->first_trace[g] + groups->n_runs[g];
        if (3 * (off[end_t] - off[c.t0]) >= 2 * rem) {
          Chunk a = c;
          a.t1 = groups->first_trace[g + 1];
          a.g1 = g + 1;
          ch.push_back(a);
          c.t0 = a.t1;
          c.g0 = g + 1;
          cut = true;
          break;
        }
      }
      if (!cut) break;
    }
    ch.push_back(c);
  }
  if (ch.size() < 2) return false;
  if (unpack_args_bytes() > 1024) throw std::logic_error("UnpackArgs outgrew its slot");
  if (unpack_tables_args_bytes() > 1024) throw std::logic_error("TabUnpackArgs outgrew its slot");
  uint64_t max_n = 0;
  uint32_t max_t = 0;
  for (auto& c : ch) {
    c.s0 = off[c.t0];
    c.s1 = off[c.t1];
    max_n = std::max(max_n, c.s1 - c.s0);
    max_t = std::max(max_t, c.t1 - c.t0);
  }

  cudaStream_t cs = ctx->stream_copy(), ws = ctx->stream_work(), os = ctx->stream_out();
  // make sure nothing from an earlier (failed) call is still in flight
  XSP_CUDA(cudaStreamSynchronize(cs));
  XSP_CUDA(cudaStreamSynchronize(ws));
  XSP_CUDA(cudaStreamSynchronize(os));
  struct Drain {  // on any exit (including exceptions) leave no copy in flight
    xsp_ctx* ctx;
    cudaStream_t a, b, c;
    ~Drain() {
      cudaStreamSynchronize(a);
      cudaStreamSynchronize(b);
      cudaStreamSynchronize(c);
      ctx->tag.clear();
    }
  } drain{ctx, cs, ws, os};

  // ---- device slots (sized up front: no reallocation while copies fly)
  struct Slot {
    xsp_span_cols cols;
    xsp_traces tr;
    uint64_t* h_off;  // pinned staging of the re-based trace offsets
    uint64_t* sid_buf;  // device span_id column (unused while span_id is read zero-copy)
    alignas(16) unsigned char unpack[1024];  // deferred k_unpack (+ delta-list decode) arguments
    alignas(16) unsigned char tab_unpack[1024];  // deferred k_unpack_tables arguments
    cudaEvent_t in_ready, free;
    cudaEvent_t computed, out_done;  // this parity's ctx buffers: results ready / copied out
  } slot[2];
  for (int s = 0; s < 2; ++s) {
    const std::string p = "pl" + std::to_string(s) + ".";
    Slot& S = slot[s];
    S.sid_buf = ctx->d<uint64_t>(p + "sid", max_n);
    S.cols.span_id = S.sid_buf;
    S.cols.parent_id = ctx->d<uint64_t>(p + "par", max_n);
    S.cols.begin_ns = ctx->d<uint64_t>(p + "beg", max_n);
    S.cols.end_ns = ctx->d<uint64_t>(p + "end", max_n);
    S.cols.cid = ctx->d<uint64_t>(p + "cid", max_n);
    S.cols.flags = ctx->d<uint8_t>(p + "flg", max_n);
    S.cols.name_id = ctx->d<uint32_t>(p + "nam", max_n);
    S.cols.flops = ctx->d<uint64_t>(p + "flops", max_n);
    S.cols.dram_read = ctx->d<uint64_t>(p + "rd", max_n);
    S.cols.dram_write = ctx->d<uint64_t>(p + "wr", max_n);
    S.cols.occupancy = ctx->d<double>(p + "occ", max_n);
    S.cols.alloc_bytes = ctx->d<int64_t>(p + "alloc", max_n);
    S.cols.type_id = ctx->d<uint32_t>(p + "type", max_n);
    S.tr.span_off = ctx->d<uint64_t>(p + "off", (uint64_t)max_t + 1);
    S.tr.levels = ctx->d<uint32_t>(p + "lvl", max_t);
    S.h_off = ctx->h<uint64_t>("plh" + std::to_string(s) + ".off", (uint64_t)max_t + 1);
    S.in_ready = ctx->take_event();
    S.free = ctx->take_event();
    S.computed = ctx->take_event();
    S.out_done = ctx->take_event();
  }
  struct EventBack {
    xsp_ctx* ctx;
    Slot* s;
    ~EventBack() {
      for (int i = 0; i < 2; ++i) {
        ctx->event_pool.push_back(s[i].in_ready);
        ctx->event_pool.push_back(s[i].free);
        ctx->event_pool.push_back(s[i].computed);
        ctx->event_pool.push_back(s[i].out_done);
      }
    }
  } evback{ctx, slot};

  const uint64_t* sid_alias = mapped_alias(hc->span_id);
  auto h2d = [&](void* dst, const void* src, uint64_t bytes) {
    if (!bytes) return;
    copy_pieces(dst, src, bytes, cudaMemcpyHostToDevice, cs);
    ctx->h2d_bytes += bytes;
  };
  uint64_t m_run = 0, l_run = 0;  // metric / layer table rows before the next chunk to stage
  auto stage = [&](size_t c) {
    Chunk& C = ch[c];
    Slot& S = slot[c & 1];
    if (c >= 2) XSP_CUDA(cudaStreamWaitEvent(cs, S.free, 0));
    const uint64_t s0 = C.s0, ns = C.s1 - C.s0;
    // span columns first: they do not depend on the table-row counts below
    if (pk) {  // packed wire form: unpacked on the copy stream into the slot's columns
      ctx->h2d_bytes += stage_packed(ctx, pk, s0, C.s1, const_cast<uint8_t*>(S.cols.flags),
                                     const_cast<uint32_t*>(S.cols.name_id), const_cast<uint64_t*>(S.cols.begin_ns),
                                     const_cast<uint64_t*>(S.cols.end_ns), const_cast<uint64_t*>(S.cols.cid),
                                     const_cast<uint64_t*>(S.cols.parent_id), "plk" + std::to_string(c & 1) + ".",
                                     cs, S.unpack);
    } else {
      h2d(const_cast<uint8_t*>(S.cols.flags), hc->flags + s0, ns);
      h2d(const_cast<uint64_t*>(S.cols.begin_ns), hc->begin_ns + s0, ns * 8);
      h2d(const_cast<uint64_t*>(S.cols.end_ns), hc->end_ns + s0, ns * 8);
      h2d(const_cast<uint64_t*>(S.cols.cid), hc->cid + s0, ns * 8);
      h2d(const_cast<uint64_t*>(S.cols.parent_id), hc->parent_id + s0, ns * 8);
      h2d(const_cast<uint32_t*>(S.cols.name_id), hc->name_id + s0, ns * 4);
    }
    uint64_t mc, lc, cp;
    if (pk && pk->blk_met0 && pk->blk_lay0 && pk->blk_cpar0) {
      // packed input: per-block prefix counts + the partial blocks at the chunk's edges
      auto before = [&](uint64_t s, uint64_t& m, uint64_t& l, uint64_t& p) {
        const uint64_t b = s / XSP_PACK_BLOCK;
        uint64_t pm, pl, pp;
        count_rows(pk->flags + b * XSP_PACK_BLOCK, s - b * XSP_PACK_BLOCK, pm, pl, pp);
        m = pk->blk_met0[b] + pm;
        l = pk->blk_lay0[b] + pl;
        p = pk->blk_cpar0[b] + pp;
      };
      uint64_t m0, l0, p0, m1, l1, p1;
      before(s0, m0, l0, p0);
      before(C.s1, m1, l1, p1);
      mc = m1 - m0;
      lc = l1 - l0;
      cp = p1 - p0;
    } else {
      count_rows((pk ? pk->flags : hc->flags) + s0, ns, mc, lc, cp);
    }
    // span_id is read sparsely (model spans, timeline ties, orphans,
    // ambiguities) unless kernels carry explicit parents: read it in place
    // from page-locked host memory when possible instead of copying it
    if (sid_alias && cp == 0) {
      S.cols.span_id = sid_alias + s0;
    } else {
      S.cols.span_id = S.sid_buf;
      h2d(S.sid_buf, hc->span_id + s0, ns * 8);
    }
    C.m0 = m_run;
    C.m1 = m_run + mc;
    C.l0 = l_run;
    C.l1 = l_run + lc;
    if (C.m1 > hc->n_metric_rows || C.l1 > hc->n_layer_rows)
      throw std::invalid_argument("metric/layer table shorter than the span flags imply");
    m_run = C.m1;
    l_run = C.l1;
    if (pk) {  // coded name_id / tables: decoded on the work stream with the span columns
      ctx->h2d_bytes += stage_tables_packed(
          ctx, pk, hc, s0, C.s1, C.m0, C.m1, C.l0, C.l1, const_cast<uint32_t*>(S.cols.name_id),
          const_cast<uint64_t*>(S.cols.flops), const_cast<uint64_t*>(S.cols.dram_read),
          const_cast<uint64_t*>(S.cols.dram_write), const_cast<double*>(S.cols.occupancy),
          const_cast<int64_t*>(S.cols.alloc_bytes), const_cast<uint32_t*>(S.cols.type_id),
          "plt" + std::to_string(c & 1) + ".", cs, S.tab_unpack);
    } else {
      h2d(const_cast<uint64_t*>(S.cols.flops), hc->flops + C.m0, mc * 8);
      h2d(const_cast<uint64_t*>(S.cols.dram_read), hc->dram_read + C.m0, mc * 8);
      h2d(const_cast<uint64_t*>(S.cols.dram_write), hc->dram_write + C.m0, mc * 8);
      h2d(const_cast<double*>(S.cols.occupancy), hc->occupancy + C.m0, mc * 8);
      h2d(const_cast<int64_t*>(S.cols.alloc_bytes), hc->alloc_bytes + C.l0, lc * 8);
      h2d(const_cast<uint32_t*>(S.cols.type_id), hc->type_id + C.l0, lc * 4);
    }
    const uint32_t nt = C.t1 - C.t0;
    for (uint32_t t = 0; t <= nt; ++t) S.h_off[t] = off[C.t0 + t] - s0;
    h2d(const_cast<uint64_t*>(S.tr.span_off), S.h_off, ((uint64_t)nt + 1) * 8);
    h2d(const_cast<uint32_t*>(S.tr.levels), ht->levels + C.t0, (uint64_t)nt * 4);
    S.cols.n_spans = ns;
    S.cols.n_metric_rows = mc;
    S.cols.n_layer_rows = lc;
    S.tr.n_traces = nt;
    XSP_CUDA(cudaEventRecord(S.in_ready, cs));
  };

  // ---- outputs: totals so far, per Count kind
  uint64_t tot[N_COUNTS] = {};
  std::memset(corr_host, 0, sizeof(*corr_host));
  std::memset(tab_host, 0, sizeof(*tab_host));
  const uint64_t tk = opts->top_k ? opts->top_k : 1;
  auto d2h_fields = [&](const Field* F, size_t nf, void* dev_struct, void* host_struct, const Pos& P, bool last) {
    // grow host columns first (rare: sync so that no copy targets a moved buffer)
    bool synced = false;
    const bool rows_only = ctx->host_out == XSP_HOST_OUT_ROWS;
    for (size_t f = 0; f < nf; ++f) {
      if (rows_only && F[f].lookup) continue;
      const uint64_t cnt = P.n[F[f].cnt] + (F[f].csr && last ? 1 : 0);
      const uint64_t need = (P.at[F[f].cnt] + cnt) * F[f].esz;
      if (ctx->hcap(F[f].name) < need || !ctx->host[F[f].name].ptr) {
        if (!synced) {
          XSP_CUDA(cudaStreamSynchronize(os));
          synced = true;
        }
        ctx->hbuf_keep(F[f].name, need, P.at[F[f].cnt] * F[f].esz);
      }
    }
    for (size_t f = 0; f < nf; ++f) {
      const Field& fd = F[f];
      if (rows_only && fd.lookup) {
        member(host_struct, fd.off) = nullptr;
        continue;
      }
      const uint64_t cnt = P.n[fd.cnt] + (fd.csr && last ? 1 : 0);
      void* dsrc = member(dev_struct, fd.off);
      char* hdst = static_cast<char*>(ctx->host[fd.name].ptr);
      member(host_struct, fd.off) = hdst;
      if (!cnt) continue;
      const uint64_t bv = P.base[fd.base];
      if (fd.base != B_NONE && bv) {
        const unsigned blocks = (unsigned)std::min<uint64_t>((cnt + 255) / 256, 148ull * 8);
        k_rebase<<<blocks, 256, 0, os>>>(static_cast<uint32_t*>(dsrc), cnt, (uint32_t)bv);
        ++ctx->launches;
      }
      copy_pieces(hdst + P.at[fd.cnt] * fd.esz, dsrc, cnt * fd.esz, cudaMemcpyDeviceToHost, os);
      ctx->d2h_bytes += cnt * fd.esz;
    }
  };

  const bool trace = std::getenv("XSP_PIPE_TRACE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto now_ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(); };
  stage(0);
  for (size_t c = 0; c < ch.size(); ++c) {
    const double h0 = now_ms();
    if (c + 1 < ch.size()) stage(c + 1);  // the next chunk streams in during this one
    const double h1 = now_ms();
    Chunk& C = ch[c];
    Slot& S = slot[c & 1];
    XSP_CUDA(cudaStreamWaitEvent(ws, S.in_ready, 0));
    // this parity's ctx buffers are free once chunk c-2's results are copied out
    if (c >= 2) XSP_CUDA(cudaStreamWaitEvent(ws, S.out_done, 0));
    if (pk) {  // packed input: rebuild the span columns and tables first
      launch_unpack(ctx, S.unpack, ws);
      launch_unpack_tables(ctx, S.tab_unpack, ws);
    }
    ctx->tag = (c & 1) ? "#p1" : "#p0";
    xsp_corr_out dcorr;
    std::memset(&dcorr, 0, sizeof(dcorr));
    run_correlate(ctx, &S.cols, &S.tr, 0, &dcorr, ws);
    const double h2 = now_ms();
    std::vector<uint32_t> gf(C.g1 - C.g0), gr(C.g1 - C.g0), gb(C.g1 - C.g0);
    for (uint32_t g = C.g0; g < C.g1; ++g) {
      gf[g - C.g0] = groups->first_trace[g] - C.t0;
      gr[g - C.g0] = groups->n_runs[g];
      gb[g - C.g0] = groups->batch_size[g];
    }
    xsp_groups cg{C.g1 - C.g0, gf.data(), gr.data(), gb.data()};
    xsp_tables_out dtab;
    std::memset(&dtab, 0, sizeof(dtab));
    run_analyze(ctx, &S.cols, &dcorr, &cg, spec, opts, &dtab, ws);
    XSP_CUDA(cudaEventRecord(S.free, ws));  // the slot's inputs are no longer read
    XSP_CUDA(cudaEventRecord(S.computed, ws));
    XSP_CUDA(cudaStreamWaitEvent(os, S.computed, 0));
    const double h3 = now_ms();

    const bool last = c + 1 == ch.size();
    Pos P;
    P.n[N_T] = C.t1 - C.t0;
    P.n[N_2T] = 2ull * (C.t1 - C.t0);
    P.n[N_L] = dcorr.n_layers;
    P.n[N_K] = dcorr.n_kernels;
    P.n[N_O] = dcorr.n_orphans;
    P.n[N_A] = dcorr.n_ambiguities;
    P.n[N_AC] = dcorr.n_candidates;
    P.n[N_G] = C.g1 - C.g0;
    P.n[N_TL] = dtab.n_layers;
    P.n[N_TK] = dtab.n_kernels;
    P.n[N_TN] = dtab.n_names;
    P.n[N_TLK] = dtab.n_layers * tk;
    P.n[N_TY] = dtab.n_type_rows;
    for (int k = 0; k < N_COUNTS; ++k) P.at[k] = tot[k];
    P.base[B_SPAN] = C.s0;
    P.base[B_METRIC] = C.m0;
    P.base[B_LAYER] = C.l0;
    P.base[B_L] = tot[N_L];
    P.base[B_K] = tot[N_K];
    P.base[B_O] = tot[N_O];
    P.base[B_A] = tot[N_A];
    P.base[B_AC] = tot[N_AC];
    P.base[B_TL] = tot[N_TL];
    P.base[B_TK] = tot[N_TK];
    P.base[B_TN] = tot[N_TN];
    P.base[B_TY] = tot[N_TY];
    d2h_fields(kCorrFields, sizeof(kCorrFields) / sizeof(Field), &dcorr, corr_host, P, last);
    d2h_fields(kTableFields, sizeof(kTableFields) / sizeof(Field), &dtab, tab_host, P, last);
    XSP_CUDA(cudaEventRecord(S.out_done, os));
    for (int k = 0; k < N_COUNTS; ++k) tot[k] += P.n[k];
    corr_host->n_failed += dcorr.n_failed;
    if (trace)
      std::fprintf(stderr, "chunk %zu spans %lu: stage %.2f  correlate-done %.2f  analyze-done %.2f  d2h-issued %.2f ms\n",
                   c, (unsigned long)(C.s1 - C.s0), h1 - h0, h2, h3, now_ms());
  }
  XSP_CUDA(cudaStreamSynchronize(ws));
  XSP_CUDA(cudaStreamSynchronize(os));
  ctx->tag.clear();
  if (trace) std::fprintf(stderr, "done %.2f ms\n", now_ms());
  corr_host->n_traces = T;
  corr_host->n_layers = tot[N_L];
  corr_host->n_kernels = tot[N_K];
  corr_host->n_orphans = tot[N_O];
  corr_host->n_ambiguities = tot[N_A];
  corr_host->n_candidates = tot[N_AC];
  tab_host->n_groups = G;
  tab_host->n_layers = tot[N_TL];
  tab_host->n_kernels = tot[N_TK];
  tab_host->n_names = tot[N_TN];
  tab_host->n_type_rows = tot[N_TY];
  return true;
}

}  // namespace xsp
