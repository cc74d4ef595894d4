// Report emission: the CSV files of the reference's report
// module (report.cpp:42-147 to_csv, :166-330 to_table converters) written on
// the GPU straight from the analysis tables in HBM, byte for byte.
//
// One table of one analysis group per call. A table is its header line, its
// data rows and its note lines ("# ..."); every row (and note) is a virtual
// row v of the launch. Two passes over the virtual rows with the same
// formatter: the size pass counts each row's bytes (formatter with a null
// buffer), an exclusive scan places the rows, the write pass formats each row
// at its offset. Doubles go through fmt_double (Ryu shortest digits laid out
// like std::to_chars, csrc/fmt.cuh), integers through fmt_u64 (std::to_string);
// cells holding ',', '"', CR or LF are quoted as csv_quote does (report.cpp:49-58).
// Optional cells (intensity, throughput, memory_bound) are empty when absent.
#include <cstring>
#include <stdexcept>
#include <string>

#include "ctx.h"
#include "fmt.cuh"
#include "prims.cuh"
#include "xsp_common.cuh"

namespace xsp {

namespace {

struct StrTab {
  const char* bytes;
  const uint64_t* off;  // [n + 1]
  uint32_t n;
};

struct RepArgs {
  int table;
  // group ranges (group-local rows [0, nk), [0, nl), [0, nn))
  uint32_t k0, nk, l0, nl, n0, nn;
  uint32_t gl_trace_layer0;  // the canonical run's first layer in the correlation
  // a8 / a9
  const uint32_t* k_name;
  const uint32_t* k_layer;
  const double* k_lat;
  const uint64_t* k_flops;
  const uint64_t* k_read;
  const uint64_t* k_write;
  const double* k_occ;
  const double* k_ai;
  const double* k_tput;
  const int8_t* k_bound;
  const uint8_t* k_in;
  // a10
  const uint32_t* n_name;
  const uint64_t* n_count;
  const double* n_lat;
  const double* n_pct;
  const uint64_t* n_flops;
  const uint64_t* n_read;
  const uint64_t* n_write;
  const double* n_occ;
  const double* n_ai;
  const double* n_tput;
  const int8_t* n_bound;
  // a11 - a14
  const uint32_t* l_index;
  const uint32_t* l_row;
  const double* l_layer_lat;
  const double* l_kern_lat;
  const uint64_t* l_flops;
  const uint64_t* l_read;
  const uint64_t* l_write;
  const double* l_occ;
  const uint64_t* l_count;
  const double* l_ai;
  const double* l_tput;
  const int8_t* l_bound;
  const double* l_nongpu;
  const double* l_gpu_share;
  const double* l_nongpu_share;
  const uint8_t* l_flagged;
  const uint8_t* l_in;
  // model scalars of the group (notes)
  double m_lat, m_gpu, m_gpu_pct;
  // strings
  const uint32_t* span_name;   // name_id column (layer names by l_row)
  const uint32_t* attr_row;    // correlation layer -> layer-table row
  const uint32_t* type_id;     // layer-table type column
  StrTab names, types;
  uint64_t base;               // header bytes before the first row
};

__device__ __forceinline__ bool csv_special(char c) { return c == ',' || c == '"' || c == '\n' || c == '\r'; }

// csv_quote(prefix + s): quoted when any byte is special; '"' doubled
__device__ int put_cell_str(char* p, const char* pre, int npre, const char* s, int n) {
  bool q = false;
  int dq = 0;
  for (int i = 0; i < npre; ++i) {
    q |= csv_special(pre[i]);
    dq += pre[i] == '"';
  }
  for (int i = 0; i < n; ++i) {
    q |= csv_special(s[i]);
    dq += s[i] == '"';
  }
  if (!q) {
    if (p) {
      for (int i = 0; i < npre; ++i) p[i] = pre[i];
      for (int i = 0; i < n; ++i) p[npre + i] = s[i];
    }
    return npre + n;
  }
  if (!p) return npre + n + dq + 2;
  int w = 0;
  p[w++] = '"';
  for (int i = 0; i < npre; ++i) {
    if (pre[i] == '"') p[w++] = '"';
    p[w++] = pre[i];
  }
  for (int i = 0; i < n; ++i) {
    if (s[i] == '"') p[w++] = '"';
    p[w++] = s[i];
  }
  p[w++] = '"';
  return w;
}

__device__ __forceinline__ int cstrlen(const char* s) {
  int n = 0;
  while (s[n]) ++n;
  return n;
}

struct W {  // cursor: p == nullptr counts only
  char* p;
  uint64_t n = 0;
  __device__ char* at() { return p ? p + n : nullptr; }
  __device__ void ch(char c) {
    if (p) p[n] = c;
    ++n;
  }
  __device__ void raw(const char* s, int len) { n += fmt_str(at(), s, len); }
  __device__ void lit(const char* s) { raw(s, cstrlen(s)); }
  __device__ void u64(uint64_t v) { n += fmt_u64(at(), v); }
  __device__ void dbl(double v) { n += fmt_double(at(), v); }
  __device__ void boolean(bool v) { v ? lit("true") : lit("false"); }
  __device__ void str(const StrTab& t, uint32_t id, const char* pre = "", int npre = 0) {
    const char* s = t.bytes + t.off[id];
    const int len = (int)(t.off[id + 1] - t.off[id]);
    n += put_cell_str(at(), pre, npre, s, len);
  }
  // optional roofline cells: intensity iff bound >= 0 (bytes > 0), throughput iff
  // latency > 0, memory_bound iff intensity (analysis.cpp:196-211 / :356-368)
  __device__ void opt_roof(double ai, double tput, int8_t bound, double lat) {
    ch(',');
    if (bound >= 0) dbl(ai);
    ch(',');
    if (lat > 0.0) dbl(tput);
    ch(',');
    if (bound >= 0) boolean(bound != 0);
  }
};

// number of decimal digits of v, into buf (for "kernel N: " prefixes)
__device__ int u64_prefix(char* buf, const char* head, int nh, uint64_t v) {
  int w = 0;
  for (int i = 0; i < nh; ++i) buf[w++] = head[i];
  w += fmt_u64(buf + w, v);
  buf[w++] = ':';
  buf[w++] = ' ';
  return w;
}


// formats virtual row v; returns its bytes
__device__ uint64_t format_row(const RepArgs& a, uint64_t v, char* p) {
  W w{p};
  switch (a.table) {
    case 8: {  // a8 kernel info (report.cpp:230-252)
      const uint32_t q = a.k0 + (uint32_t)v;
      w.str(a.names, a.k_name[q]);
      w.ch(',');
      w.u64(a.k_layer[q]);
      w.ch(',');
      w.dbl(a.k_lat[q]);
      w.ch(',');
      w.u64(a.k_flops[q]);
      w.ch(',');
      w.u64(a.k_read[q]);
      w.ch(',');
      w.u64(a.k_write[q]);
      w.ch(',');
      w.dbl(a.k_occ[q]);
      w.opt_roof(a.k_ai[q], a.k_tput[q], a.k_bound[q], a.k_lat[q]);
      w.ch('\n');
      break;
    }
    case 9:
    case 14: {  // roofline reports (report.cpp:254-262): subject rows, excluded as notes
      const bool kern = a.table == 9;
      const uint64_t cnt = kern ? a.nk : a.nl;
      const bool note = v >= cnt;
      const uint32_t r = (uint32_t)(note ? v - cnt : v);
      const uint32_t q = (kern ? a.k0 : a.l0) + r;
      const bool in = kern ? a.k_in[q] != 0 : a.l_in[q] != 0;
      if (note == in) break;  // classified rows / excluded notes only
      char pre[40];
      const int np = kern ? u64_prefix(pre, "kernel ", 7, r) : u64_prefix(pre, "layer ", 6, a.l_index[q]);
      const StrTab& t = a.names;
      const uint32_t id = kern ? a.k_name[q] : a.span_name[a.l_row[q]];
      if (note) {
        w.lit("# excluded (undefined intensity or zero latency): ");
        w.raw(pre, np);
        w.raw(t.bytes + t.off[id], (int)(t.off[id + 1] - t.off[id]));
        w.ch('\n');
        break;
      }
      w.str(t, id, pre, np);
      w.ch(',');
      w.dbl(kern ? a.k_ai[q] : a.l_ai[q]);
      w.ch(',');
      w.dbl(kern ? a.k_tput[q] : a.l_tput[q]);
      w.ch(',');
      w.boolean((kern ? a.k_bound[q] : a.l_bound[q]) != 0);
      w.ch('\n');
      break;
    }
    case 10: {  // a10 by name (report.cpp:264-287)
      if (v == a.nn) {
        w.lit("# model_latency_ns=");
        w.dbl(a.m_lat);
        w.ch('\n');
        break;
      }
      const uint32_t q = a.n0 + (uint32_t)v;
      w.str(a.names, a.n_name[q]);
      w.ch(',');
      w.u64(a.n_count[q]);
      w.ch(',');
      w.dbl(a.n_lat[q]);
      w.ch(',');
      w.dbl(a.n_pct[q]);
      w.ch(',');
      w.u64(a.n_flops[q]);
      w.ch(',');
      w.u64(a.n_read[q]);
      w.ch(',');
      w.u64(a.n_write[q]);
      w.ch(',');
      w.dbl(a.n_occ[q]);
      w.opt_roof(a.n_ai[q], a.n_tput[q], a.n_bound[q], a.n_lat[q]);
      w.ch('\n');
      break;
    }
    case 11: {  // a11 by layer (report.cpp:289-313)
      const uint32_t q = a.l0 + (uint32_t)v;
      w.u64(a.l_index[q]);
      w.ch(',');
      w.str(a.names, a.span_name[a.l_row[q]]);
      w.ch(',');
      w.str(a.types, a.type_id[a.attr_row[a.gl_trace_layer0 + a.l_index[q]]]);
      w.ch(',');
      w.dbl(a.l_layer_lat[q]);
      w.ch(',');
      w.dbl(a.l_kern_lat[q]);
      w.ch(',');
      w.u64(a.l_flops[q]);
      w.ch(',');
      w.u64(a.l_read[q]);
      w.ch(',');
      w.u64(a.l_write[q]);
      w.ch(',');
      w.dbl(a.l_occ[q]);
      w.ch(',');
      w.u64(a.l_count[q]);
      w.opt_roof(a.l_ai[q], a.l_tput[q], a.l_bound[q], a.l_kern_lat[q]);
      w.ch('\n');
      break;
    }
    case 12: {  // a12 metrics per layer (report.cpp:315-326)
      const uint32_t q = a.l0 + (uint32_t)v;
      w.u64(v);
      w.ch(',');
      w.u64(a.l_flops[q]);
      w.ch(',');
      w.u64(a.l_read[q]);
      w.ch(',');
      w.u64(a.l_write[q]);
      w.ch('\n');
      break;
    }
    case 13: {  // a13 GPU vs non-GPU (report.cpp:328-345)
      if (v == a.nl) {
        w.lit("# model_latency_ns=");
        w.dbl(a.m_lat);
        w.lit("\n# model_gpu_latency_ns=");
        w.dbl(a.m_gpu);
        w.lit("\n# model_gpu_percent=");
        w.dbl(a.m_gpu_pct);
        w.ch('\n');
        break;
      }
      const uint32_t q = a.l0 + (uint32_t)v;
      w.u64(a.l_index[q]);
      w.ch(',');
      w.dbl(a.l_kern_lat[q]);
      w.ch(',');
      w.dbl(a.l_nongpu[q]);
      w.ch(',');
      w.dbl(a.l_gpu_share[q]);
      w.ch(',');
      w.dbl(a.l_nongpu_share[q]);
      w.ch(',');
      w.boolean(a.l_flagged[q] != 0);
      w.ch('\n');
      break;
    }
  }
  return w.n;
}

__global__ void k_rep_size(RepArgs a, uint64_t n, uint64_t* __restrict__ len) {
  const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) len[v] = format_row(a, v, nullptr);
}

__global__ void k_rep_write(RepArgs a, uint64_t n, const uint64_t* __restrict__ off, char* __restrict__ out) {
  const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) format_row(a, v, out + a.base + off[v]);
}

const char* header(int table) {
  switch (table) {
    case 8:
      return "name,layer_index,latency_ns,flops,dram_read_bytes,dram_write_bytes,achieved_occupancy,"
             "arithmetic_intensity,arithmetic_throughput,memory_bound\n";
    case 9:
    case 14: return "subject,arithmetic_intensity,arithmetic_throughput,memory_bound\n";
    case 10:
      return "name,count,total_latency_ns,latency_percent,total_flops,total_dram_read_bytes,"
             "total_dram_write_bytes,weighted_achieved_occupancy,arithmetic_intensity,"
             "arithmetic_throughput,memory_bound\n";
    case 11:
      return "layer_index,name,type,layer_latency_ns,kernel_latency_ns,total_flops,total_dram_read_bytes,"
             "total_dram_write_bytes,weighted_achieved_occupancy,kernel_count,arithmetic_intensity,"
             "arithmetic_throughput,memory_bound\n";
    case 12: return "layer_index,total_flops,total_dram_read_bytes,total_dram_write_bytes\n";
    case 13: return "layer_index,gpu_latency_ns,non_gpu_latency_ns,gpu_share,non_gpu_share,flagged\n";
    default: throw std::invalid_argument("report table must be one of 8..14");
  }
}

StrTab upload_strings(xsp_ctx* ctx, const xsp_string_table* s, const std::string& tag, cudaStream_t st) {
  StrTab t{nullptr, nullptr, 0};
  if (!s) return t;
  const uint64_t nb = s->off[s->n];
  char* b = ctx->d<char>(tag + ".bytes", nb + 1);
  uint64_t* o = ctx->d<uint64_t>(tag + ".off", s->n + 1ull);
  if (nb) XSP_CUDA(cudaMemcpyAsync(b, s->bytes, nb, cudaMemcpyHostToDevice, st));
  XSP_CUDA(cudaMemcpyAsync(o, s->off, (s->n + 1ull) * 8, cudaMemcpyHostToDevice, st));
  t.bytes = b;
  t.off = o;
  t.n = s->n;
  return t;
}

template <typename T>
T read1(const T* d, cudaStream_t st) {
  T v;
  XSP_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  return v;
}

}  // namespace

void run_report_csv(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr, const xsp_groups* groups,
                    const xsp_tables_out* t, const xsp_string_table* names, const xsp_string_table* types,
                    uint32_t group, int table, char** text, uint64_t* len, int to_host, cudaStream_t st) {
  if (group >= t->n_groups) throw std::invalid_argument("group out of range");
  const char* head = header(table);
  if (!names) throw std::invalid_argument("the name table is required");
  if (table == 11 && !types) throw std::invalid_argument("a11 needs the layer type table");
  if (read1(t->group_status + group, st) != XSP_G_OK)
    throw std::invalid_argument("the group's analysis failed (group_status)");
  RepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.table = table;
  uint32_t go[2];
  XSP_CUDA(cudaMemcpyAsync(go, t->group_kernel_off + group, 8, cudaMemcpyDeviceToHost, st));
  uint32_t gl[2];
  XSP_CUDA(cudaMemcpyAsync(gl, t->group_layer_off + group, 8, cudaMemcpyDeviceToHost, st));
  uint32_t gn[2];
  XSP_CUDA(cudaMemcpyAsync(gn, t->group_name_off + group, 8, cudaMemcpyDeviceToHost, st));
  double ms[3];
  XSP_CUDA(cudaMemcpyAsync(ms, t->m_lat + group, 8, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaMemcpyAsync(ms + 1, t->m_gpu + group, 8, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaMemcpyAsync(ms + 2, t->m_gpu_pct + group, 8, cudaMemcpyDeviceToHost, st));
  uint32_t tl0 = 0;
  if (table == 11) XSP_CUDA(cudaMemcpyAsync(&tl0, corr->trace_layer_off + groups->first_trace[group], 4,
                                            cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  a.k0 = go[0];
  a.nk = go[1] - go[0];
  a.l0 = gl[0];
  a.nl = gl[1] - gl[0];
  a.n0 = gn[0];
  a.nn = gn[1] - gn[0];
  a.m_lat = ms[0];
  a.m_gpu = ms[1];
  a.m_gpu_pct = ms[2];
  a.gl_trace_layer0 = tl0;
  a.k_name = t->k_name; a.k_layer = t->k_layer; a.k_lat = t->k_lat; a.k_flops = t->k_flops;
  a.k_read = t->k_read; a.k_write = t->k_write; a.k_occ = t->k_occ; a.k_ai = t->k_ai; a.k_tput = t->k_tput;
  a.k_bound = t->k_bound; a.k_in = t->k_roofline_in;
  a.n_name = t->n_name; a.n_count = t->n_count; a.n_lat = t->n_lat; a.n_pct = t->n_pct;
  a.n_flops = t->n_flops; a.n_read = t->n_read; a.n_write = t->n_write; a.n_occ = t->n_occ;
  a.n_ai = t->n_ai; a.n_tput = t->n_tput; a.n_bound = t->n_bound;
  a.l_index = t->l_index; a.l_row = t->l_row; a.l_layer_lat = t->l_layer_lat; a.l_kern_lat = t->l_kern_lat;
  a.l_flops = t->l_flops; a.l_read = t->l_read; a.l_write = t->l_write; a.l_occ = t->l_occ;
  a.l_count = t->l_count; a.l_ai = t->l_ai; a.l_tput = t->l_tput; a.l_bound = t->l_bound;
  a.l_nongpu = t->l_nongpu; a.l_gpu_share = t->l_gpu_share; a.l_nongpu_share = t->l_nongpu_share;
  a.l_flagged = t->l_flagged; a.l_in = t->l_roofline_in;
  a.span_name = cols->name_id;
  a.attr_row = corr ? corr->layer_attr_row : nullptr;
  a.type_id = cols->type_id;
  a.names = upload_strings(ctx, names, "r.names", st);
  a.types = upload_strings(ctx, types, "r.types", st);
  const uint64_t hl = std::strlen(head);
  a.base = hl;
  uint64_t n = 0;
  switch (table) {
    case 8: n = a.nk; break;
    case 9: n = 2ull * a.nk; break;
    case 10: n = a.nn + 1ull; break;
    case 11: case 12: n = a.nl; break;
    case 13: n = a.nl + 1ull; break;
    case 14: n = 2ull * a.nl; break;
  }
  uint64_t* rl = ctx->d<uint64_t>("r.len", n + 1);
  uint64_t* ro = ctx->d<uint64_t>("r.off", n + 1);
  uint64_t* scratch = ctx->d<uint64_t>("r.scan", scan_scratch_elems(n + 1));
  if (n) {
    k_rep_size<<<ceil_div(n, 128), 128, 0, st>>>(a, n, rl);
    ++ctx->launches;
  }
  exclusive_scan<uint64_t, uint64_t>(rl, ro, n, scratch, ro + n, st, &ctx->launches);
  const uint64_t body = read1(ro + n, st);
  const uint64_t total = hl + body;
  char* out = ctx->d<char>("r.text", total + 1);
  XSP_CUDA(cudaMemcpyAsync(out, head, hl, cudaMemcpyHostToDevice, st));
  if (n) {
    k_rep_write<<<ceil_div(n, 128), 128, 0, st>>>(a, n, ro, out);
    ++ctx->launches;
  }
  if (to_host) {
    char* h = ctx->h<char>("r.text_h", total + 1);
    XSP_CUDA(cudaMemcpyAsync(h, out, total, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaStreamSynchronize(st));
    h[total] = 0;
    *text = h;
  } else {
    *text = out;
  }
  *len = total;
}

}  // namespace xsp
