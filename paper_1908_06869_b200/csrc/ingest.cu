// JSONL wire-format ingest on the GPU: the reference's
// ingest() (collector.cpp:219-266) of many JSONL streams — one TraceBundle each
// — straight into the SoA span columns the correlate/analyze path reads.
//
//   1. H2D of the text; newline positions (a per-chunk count, a scan, a write);
//   2. one thread per line parses a span record in the reference writer's
//      canonical layout (encode_span_record: keys in order, no whitespace):
//      exact u64 fields, kind / level names, the name and layer_type strings as
//      byte ranges, the metric tags (integers exact; decimal doubles by the
//      exact Clinger fast path: <= 2^53 significand, |exp10| <= 22, one
//      correctly rounded multiply / divide), and the raw-tag facts validation
//      needs; it also hashes the name (FNV-1a 64);
//   3. names and layer types are interned in lexicographic order: the hashes
//      are radix-sorted, every span is checked byte for byte against its run's
//      representative (a hash collision sends the batch to the host), the few
//      distinct strings are ordered on the host and their ranks scattered back;
//   4. sort_timeline (stage (b)) and validate_bundle (stage (a)) on the device.
//
// Meta records are parsed on the host (one short line per stream, canonical
// layout). Anything the fast path does not cover exactly — escapes or non-ASCII
// bytes in strings, other layouts or whitespace, numbers outside the exact
// cases, unknown record kinds, a missing or repeated meta record, a trace_id
// mismatch, validation issues — is reported as XSP_INGEST_HOST with the first
// such stream: the caller runs the reference-exact host parser (the C++
// drop-in's strata::ingest) for the error text or the result.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "ctx.h"
#include "prims.cuh"
#include "xsp_common.cuh"

namespace xsp {

void run_sort_timeline(xsp_ctx* ctx, uint64_t n, const uint64_t* begin, const uint8_t* flags, const uint64_t* sid,
                       uint32_t T, const uint64_t* off, uint32_t* perm, uint32_t* was_sorted, cudaStream_t st);
void run_validate(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_traces* tr, const xsp_validate_in* vin,
                  xsp_validation_out* out, cudaStream_t st);

namespace {

constexpr uint32_t LK_BLANK = 0, LK_SPAN = 1, LK_META = 2, LK_HOST = 3;

struct LineOut {
  uint8_t* kind;       // LK_*
  uint64_t* span_id;
  uint64_t* parent;
  uint64_t* begin;
  uint64_t* end;
  uint64_t* cid;
  uint64_t* trace_id;
  uint8_t* flags;
  uint64_t* name_hash;
  uint64_t* name_off;  // byte range of the name in the text
  uint32_t* name_len;
  uint64_t* type_hash;
  uint64_t* type_off;
  uint32_t* type_len;  // layer_type string (layers; "" when absent)
  uint64_t* flops;
  uint64_t* dread;
  uint64_t* dwrite;
  double* occ;
  int64_t* alloc;
  uint8_t* tag_bits;
};

__device__ __forceinline__ uint64_t fnv_step(uint64_t h, uint8_t c) { return (h ^ c) * 0x100000001b3ull; }
constexpr uint64_t kFnv0 = 0xcbf29ce484222325ull;

struct Cur {
  const char* p;
  const char* e;
  __device__ bool lit(const char* s) {
    const char* q = p;
    for (; *s; ++s, ++q)
      if (q >= e || *q != *s) return false;
    p = q;
    return true;
  }
  __device__ bool u64(uint64_t& v) {
    if (p >= e || *p < '0' || *p > '9') return false;
    if (*p == '0') {
      ++p;
      v = 0;
      return p >= e || *p < '0' || *p > '9';
    }
    uint64_t x = 0;
    while (p < e && *p >= '0' && *p <= '9') {
      const uint64_t d = (uint64_t)(*p - '0');
      if (x > (~0ull - d) / 10) return false;  // beyond u64: a double in JSON terms
      x = x * 10 + d;
      ++p;
    }
    v = x;
    return true;
  }
  __device__ bool u64_or_null(uint64_t& v, bool& has) {
    if (lit("null")) {
      has = false;
      v = 0;
      return true;
    }
    has = true;
    return u64(v);
  }
  // a plain string (no escapes, printable ASCII): its byte range and FNV-1a hash
  __device__ bool str(const char* base, uint64_t& off, uint32_t& len, uint64_t& h) {
    if (p >= e || *p != '"') return false;
    ++p;
    const char* s = p;
    uint64_t x = kFnv0;
    while (p < e && *p != '"') {
      const unsigned char c = (unsigned char)*p;
      if (c < 0x20 || c >= 0x80 || c == '\\') return false;
      x = fnv_step(x, c);
      ++p;
    }
    if (p >= e) return false;
    off = (uint64_t)(s - base);
    len = (uint32_t)(p - s);
    h = x;
    ++p;
    return true;
  }
  __device__ bool key(const char*& ks, int& kn) {
    if (p >= e || *p != '"') return false;
    ++p;
    ks = p;
    while (p < e && *p != '"') {
      const unsigned char c = (unsigned char)*p;
      if (c < 0x20 || c >= 0x80 || c == '\\') return false;
      ++p;
    }
    if (p >= e) return false;
    kn = (int)(p - ks);
    ++p;
    return p < e && *p++ == ':';
  }
};

__device__ __forceinline__ bool key_is(const char* ks, int kn, const char* s) {
  int i = 0;
  for (; s[i]; ++i)
    if (i >= kn || ks[i] != s[i]) return false;
  return i == kn;
}

// a JSON tag value: t = 1 integer (i), 2 double (d), 3 string, 4 bool (i = 0/1);
// false when outside the exactly handled cases (the host decides)
__device__ bool tag_value(Cur& c, int& t, int64_t& i, double& d, const char* base, uint64_t& soff, uint32_t& slen,
                          uint64_t& sh) {
  if (c.p >= c.e) return false;
  const char ch = *c.p;
  if (ch == '"') {
    t = 3;
    return c.str(base, soff, slen, sh);
  }
  if (c.lit("true")) {
    t = 4;
    i = 1;
    return true;
  }
  if (c.lit("false")) {
    t = 4;
    i = 0;
    return true;
  }
  // number: -?(0|[1-9][0-9]*)(.[0-9]+)?([eE][+-]?[0-9]+)?
  bool neg = false;
  if (*c.p == '-') {
    neg = true;
    ++c.p;
  }
  if (c.p >= c.e || *c.p < '0' || *c.p > '9') return false;
  uint64_t m = 0;
  int nd = 0, e10 = 0;
  bool big = false;
  if (*c.p == '0') {
    ++c.p;
    if (c.p < c.e && *c.p >= '0' && *c.p <= '9') return false;
  } else {
    while (c.p < c.e && *c.p >= '0' && *c.p <= '9') {
      if (nd < 19) {
        m = m * 10 + (uint64_t)(*c.p - '0');
        if (m) ++nd;
      } else {
        big = true;
      }
      ++c.p;
    }
  }
  bool frac = false;
  if (c.p < c.e && *c.p == '.') {
    frac = true;
    ++c.p;
    if (c.p >= c.e || *c.p < '0' || *c.p > '9') return false;
    while (c.p < c.e && *c.p >= '0' && *c.p <= '9') {
      if (nd < 19) {
        m = m * 10 + (uint64_t)(*c.p - '0');
        if (m) ++nd;
        --e10;
      } else {
        big = true;
      }
      ++c.p;
    }
  }
  if (c.p < c.e && (*c.p == 'e' || *c.p == 'E')) {
    frac = true;
    ++c.p;
    bool eneg = false;
    if (c.p < c.e && (*c.p == '+' || *c.p == '-')) eneg = *c.p++ == '-';
    if (c.p >= c.e || *c.p < '0' || *c.p > '9') return false;
    int x = 0;
    while (c.p < c.e && *c.p >= '0' && *c.p <= '9') {
      if (x < 100000) x = x * 10 + (*c.p - '0');
      ++c.p;
    }
    e10 += eneg ? -x : x;
  }
  if (big) return false;
  if (!frac) {  // JSON integer: u64 when non-negative, i64 when negative (a tag keeps it as i64)
    if (neg) {
      if (m > (1ull << 63)) return false;
      t = 1;
      i = (int64_t)(0 - m);
      return true;
    }
    t = 1;
    i = (int64_t)m;  // u64 beyond i64 wraps, as get<int64_t>() of an unsigned does
    return true;
  }
  // Clinger's exact case: m and 10^|e10| are exact doubles, one rounding
  if (m > (1ull << 53) || e10 < -22 || e10 > 22) return false;
  constexpr double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                              1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
  double v = (double)m;
  v = e10 >= 0 ? __dmul_rn(v, p10[e10]) : __ddiv_rn(v, p10[-e10]);
  t = 2;
  d = neg ? -v : v;
  return true;
}


__device__ uint32_t parse_span(const char* base, const char* s, const char* e, uint64_t li, const LineOut& o) {
  Cur c{s, e};
  uint64_t begin, end, cid, parent, sid, tid;
  bool has_cid, has_par;
  uint64_t noff, th = 0, toff = 0, nh;
  uint32_t nlen, tlen = 0;
  if (!c.lit("{\"begin_ns\":") || !c.u64(begin)) return LK_HOST;
  if (!c.lit(",\"correlation_id\":") || !c.u64_or_null(cid, has_cid)) return LK_HOST;
  if (!c.lit(",\"end_ns\":") || !c.u64(end)) return LK_HOST;
  uint32_t kind, level;
  if (!c.lit(",\"kind\":\"")) return LK_HOST;
  if (c.lit("sync\"")) kind = XSP_KIND_SYNC;
  else if (c.lit("launch\"")) kind = XSP_KIND_LAUNCH;
  else if (c.lit("exec\"")) kind = XSP_KIND_EXEC;
  else return LK_HOST;
  if (!c.lit(",\"level\":\"")) return LK_HOST;
  if (c.lit("model\"")) level = XSP_LEVEL_MODEL;
  else if (c.lit("layer\"")) level = XSP_LEVEL_LAYER;
  else if (c.lit("kernel\"")) level = XSP_LEVEL_KERNEL;
  else if (c.lit("api\"")) level = XSP_LEVEL_API;
  else return LK_HOST;
  if (!c.lit(",\"name\":") || !c.str(base, noff, nlen, nh)) return LK_HOST;
  if (!c.lit(",\"parent_id\":") || !c.u64_or_null(parent, has_par)) return LK_HOST;
  if (!c.lit(",\"rec\":\"span\",\"span_id\":") || !c.u64(sid)) return LK_HOST;
  if (!c.lit(",\"tags\":{")) return LK_HOST;
  // tags (metrics_from_tags / tag_int / tag_string semantics, span.cpp / correlator.cpp)
  bool hf = false, hr = false, hw = false, ho = false, ht = false, ha = false;
  int64_t vf = 0, vr = 0, vw = 0, va = 0;
  double vo = 0.0;
  uint8_t tb = 0;
  if (!c.lit("}")) {
    for (;;) {
      const char* ks;
      int kn;
      if (!c.key(ks, kn)) return LK_HOST;
      int t;
      int64_t iv = 0;
      double dv = 0.0;
      uint64_t so = 0, sh = 0;
      uint32_t sl = 0;
      if (!tag_value(c, t, iv, dv, base, so, sl, sh)) return LK_HOST;
      const bool num = t == 1 || t == 2 || t == 4;
      // integer value of a number tag: an int, or a double truncated toward zero
      auto as_int = [&](int64_t& out) -> bool {
        if (t == 2) {
          if (!(dv > -9.2233720368547758e18 && dv < 9.2233720368547758e18)) return false;
          out = (int64_t)dv;
        } else {
          out = iv;
        }
        return true;
      };
      if (key_is(ks, kn, "flop_count_sp")) {
        if (hf) return LK_HOST;
        if (num) {
          if (!as_int(vf)) return LK_HOST;
          hf = true;
          if (t == 1 && iv < 0) tb |= XSP_TAG_NEG_FLOPS;
        }
      } else if (key_is(ks, kn, "dram_read_bytes")) {
        if (hr) return LK_HOST;
        if (num) {
          if (!as_int(vr)) return LK_HOST;
          hr = true;
          if (t == 1 && iv < 0) tb |= XSP_TAG_NEG_READ;
        }
      } else if (key_is(ks, kn, "dram_write_bytes")) {
        if (hw) return LK_HOST;
        if (num) {
          if (!as_int(vw)) return LK_HOST;
          hw = true;
          if (t == 1 && iv < 0) tb |= XSP_TAG_NEG_WRITE;
        }
      } else if (key_is(ks, kn, "achieved_occupancy")) {
        if (ho) return LK_HOST;
        if (num) {
          ho = true;
          vo = t == 2 ? dv : (double)iv;
          if (t == 2) tb |= XSP_TAG_OCC_DOUBLE;
        }
      } else if (key_is(ks, kn, "alloc_bytes")) {
        if (ha) return LK_HOST;
        if (num) {
          if (!as_int(va)) return LK_HOST;
          ha = true;
        }
      } else if (key_is(ks, kn, "layer_type")) {
        if (ht) return LK_HOST;
        if (t == 3) {
          ht = true;
          toff = so;
          tlen = sl;
          th = sh;
        }
      }
      if (c.lit(",")) continue;
      if (c.lit("}")) break;
      return LK_HOST;
    }
  }
  if (!c.lit(",\"trace_id\":") || !c.u64(tid) || !c.lit("}") || c.p != e) return LK_HOST;
  const bool met = hf || hr || hw || ho;
  uint8_t f = (uint8_t)(level | (kind << 2));
  if (has_par) f |= XSP_F_PARENT;
  if (has_cid) f |= XSP_F_CID;
  if (met) f |= XSP_F_METRICS;
  o.span_id[li] = sid;
  o.parent[li] = has_par ? parent : 0;
  o.begin[li] = begin;
  o.end[li] = end;
  o.cid[li] = has_cid ? cid : 0;
  o.trace_id[li] = tid;
  o.flags[li] = f;
  o.name_hash[li] = nh;
  o.name_off[li] = noff;
  o.name_len[li] = nlen;
  if (!ht) {
    toff = 0;
    tlen = 0;
    th = kFnv0;
  }
  o.type_hash[li] = th;
  o.type_off[li] = toff;
  o.type_len[li] = tlen;
  o.flops[li] = hf && vf > 0 ? (uint64_t)vf : 0;
  o.dread[li] = hr && vr > 0 ? (uint64_t)vr : 0;
  o.dwrite[li] = hw && vw > 0 ? (uint64_t)vw : 0;
  o.occ[li] = ho ? vo : 0.0;
  o.alloc[li] = ha ? va : 0;
  o.tag_bits[li] = tb;
  return LK_SPAN;
}

// ---- line index
constexpr uint32_t kNlChunk = 64;

__global__ void k_nl_count(const char* __restrict__ t, uint64_t n, uint32_t* __restrict__ cnt) {
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t b = c * kNlChunk;
  if (b >= n) return;
  const uint64_t e = b + kNlChunk < n ? b + kNlChunk : n;
  uint32_t k = 0;
  for (uint64_t i = b; i < e; ++i) k += t[i] == '\n';
  cnt[c] = k;
}

__global__ void k_nl_write(const char* __restrict__ t, uint64_t n, const uint32_t* __restrict__ pos,
                           uint64_t* __restrict__ nl) {
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t b = c * kNlChunk;
  if (b >= n) return;
  const uint64_t e = b + kNlChunk < n ? b + kNlChunk : n;
  uint32_t k = pos[c];
  for (uint64_t i = b; i < e; ++i)
    if (t[i] == '\n') nl[k++] = i;
}

// Lines from the newline positions, on the device: stream s's lines are its
// newlines plus, when its last byte is not '\n', one unterminated tail line
// [last newline + 1, soff[s + 1]); a line never straddles two streams.
__device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t* __restrict__ v, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (v[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// nbefore[s] = newlines before soff[s] (s <= S); tail[s] = stream s ends in an unterminated line
__global__ void k_stream_lines(const uint64_t* __restrict__ nl, uint64_t hnl, const uint64_t* __restrict__ soff,
                               uint32_t S, uint64_t* __restrict__ nbefore, uint32_t* __restrict__ tail) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > S) return;
  nbefore[s] = lower_bound_u64(nl, hnl, soff[s]);
  if (s == S) return;
  const uint64_t nf = lower_bound_u64(nl, hnl, soff[s]), nla = lower_bound_u64(nl, hnl, soff[s + 1]);
  const uint64_t at = nla > nf ? nl[nla - 1] + 1 : soff[s];
  tail[s] = at < soff[s + 1] ? 1u : 0u;
}

// line of newline k: index k + (tail lines of earlier streams)
__global__ void k_lines_nl(const uint64_t* __restrict__ nl, uint64_t hnl, const uint64_t* __restrict__ soff,
                           uint32_t S, const uint32_t* __restrict__ tb, uint64_t* __restrict__ lstart,
                           uint64_t* __restrict__ lend, uint32_t* __restrict__ lstream) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= hnl) return;
  const uint64_t p = nl[k];
  uint32_t lo = 0, hi = S;  // the last stream with soff[s] <= p (empty streams before it hold no byte)
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (soff[mid] <= p) lo = mid; else hi = mid;
  }
  const uint64_t idx = k + tb[lo];
  lend[idx] = p;
  lstart[idx] = (k > 0 && nl[k - 1] >= soff[lo]) ? nl[k - 1] + 1 : soff[lo];
  lstream[idx] = lo;
}

__global__ void k_lines_tail(const uint64_t* __restrict__ nl, const uint64_t* __restrict__ nbefore,
                             const uint64_t* __restrict__ soff, uint32_t S, const uint32_t* __restrict__ tail,
                             const uint32_t* __restrict__ tb, uint64_t* __restrict__ lstart,
                             uint64_t* __restrict__ lend, uint32_t* __restrict__ lstream) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S || !tail[s]) return;
  const uint64_t nf = nbefore[s], nla = nbefore[s + 1];
  const uint64_t idx = nla + tb[s];
  lstart[idx] = nla > nf ? nl[nla - 1] + 1 : soff[s];
  lend[idx] = soff[s + 1];
  lstream[idx] = s;
}

// per stream: meta records (count, a line holding one), span lines; the first
// line the device parser left to the host
struct LineStats {
  uint32_t* nmeta;            // [S]
  uint32_t* nspan;            // [S]
  unsigned long long* mline;  // [S]
  unsigned long long* first_host;
};
__global__ void k_line_stats(const uint8_t* __restrict__ kind, const uint32_t* __restrict__ lstream, uint64_t L,
                             LineStats o) {
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const uint8_t k = kind[l];
  const uint32_t s = lstream[l];
  if (k == LK_HOST) {
    atomicMin(o.first_host, (unsigned long long)l);
  } else if (k == LK_META) {
    atomicAdd(o.nmeta + s, 1u);
    o.mline[s] = l;
  } else if (k == LK_SPAN) {
    atomicAdd(o.nspan + s, 1u);
  }
}

// byte range of each stream's meta line (the per-stream record of a clean batch)
__global__ void k_meta_ranges(const unsigned long long* __restrict__ mline, const uint32_t* __restrict__ nmeta,
                              uint32_t S, const uint64_t* __restrict__ lstart, const uint64_t* __restrict__ lend,
                              uint64_t* __restrict__ mrange) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const bool one = nmeta[s] == 1;
  mrange[2 * s] = one ? lstart[mline[s]] : 0;
  mrange[2 * s + 1] = one ? lend[mline[s]] : 0;
}

// line l = [start[l], end[l]) (end: its newline, or its stream's end)
__global__ void k_parse_lines(const char* __restrict__ t, uint64_t n, const uint64_t* __restrict__ start,
                              const uint64_t* __restrict__ nl, uint64_t nlines, LineOut o) {
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nlines) return;
  const uint64_t s = start[l];
  const uint64_t e = nl[l];
  // blank line: only ' ', '\t', '\r'
  bool blank = true;
  for (uint64_t i = s; i < e && blank; ++i) blank = t[i] == ' ' || t[i] == '\t' || t[i] == '\r';
  if (blank) {
    o.kind[l] = LK_BLANK;
    return;
  }
  const char* p = t + s;
  if (e - s >= 14 && p[0] == '{' && p[1] == '"' && p[2] == 'b' && p[3] == 'a') {  // {"batch_size": meta
    o.kind[l] = LK_META;
    return;
  }
  o.kind[l] = (uint8_t)parse_span(t, p, t + e, l, o);
}

// span index of every span line; the stream of every line
__global__ void k_span_flags(const uint8_t* __restrict__ kind, uint64_t nlines, uint32_t* __restrict__ isspan) {
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l < nlines) isspan[l] = kind[l] == LK_SPAN;
}

struct Gather {
  const uint32_t* isspan;
  const uint32_t* spos;
  const uint64_t* nl;
  uint64_t nlines;
  LineOut lo;
  // outputs in file order (span index)
  uint64_t *span_id, *parent, *begin, *end, *cid, *trace_id, *name_hash, *type_hash, *name_off, *type_off;
  uint32_t *name_len, *type_len, *line_of;
  uint8_t *flags, *tag_bits;
  uint64_t *flops, *dread, *dwrite;
  double* occ;
  int64_t* alloc;
};

__global__ void k_gather_spans(Gather g) {
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= g.nlines || !g.isspan[l]) return;
  const uint32_t j = g.spos[l];
  g.span_id[j] = g.lo.span_id[l];
  g.parent[j] = g.lo.parent[l];
  g.begin[j] = g.lo.begin[l];
  g.end[j] = g.lo.end[l];
  g.cid[j] = g.lo.cid[l];
  g.trace_id[j] = g.lo.trace_id[l];
  g.flags[j] = g.lo.flags[l];
  g.name_hash[j] = g.lo.name_hash[l];
  g.name_off[j] = g.lo.name_off[l];
  g.name_len[j] = g.lo.name_len[l];
  g.type_hash[j] = g.lo.type_hash[l];
  g.type_off[j] = g.lo.type_off[l];
  g.type_len[j] = g.lo.type_len[l];
  g.flops[j] = g.lo.flops[l];
  g.dread[j] = g.lo.dread[l];
  g.dwrite[j] = g.lo.dwrite[l];
  g.occ[j] = g.lo.occ[l];
  g.alloc[j] = g.lo.alloc[l];
  g.tag_bits[j] = g.lo.tag_bits[l];
  g.line_of[j] = (uint32_t)l;
}

__global__ void k_is_layer(const uint8_t* __restrict__ flags, uint64_t n, uint8_t* __restrict__ out) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = (flags[j] & 3u) == XSP_LEVEL_LAYER ? 1 : 0;
}

// ingest's trace_id check (collector.cpp:248-255): the first stream holding a
// span whose trace_id differs from its meta record's
__global__ void k_tid_check(const uint64_t* __restrict__ tid, const uint64_t* __restrict__ soff, uint32_t S,
                            const uint64_t* __restrict__ mtid, uint64_t n, uint32_t* __restrict__ bad) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  uint32_t lo = 0, hi = S;  // soff[lo] <= j < soff[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (soff[mid] <= j) lo = mid; else hi = mid;
  }
  if (tid[j] != mtid[lo]) atomicMin(bad, lo);
}

// ---- final columns in timeline order (perm = file index of timeline position)
struct Final {
  const uint32_t* perm;
  uint64_t n;
  const uint64_t *span_id, *parent, *begin, *end, *cid, *trace_id;
  const uint8_t *flags, *tag_bits;
  const uint32_t *name_id, *type_id;
  const uint64_t *flops, *dread, *dwrite;
  const double* occ;
  const int64_t* alloc;
  uint64_t *o_span_id, *o_parent, *o_begin, *o_end, *o_cid, *o_trace_id;
  uint8_t *o_flags, *o_tag_bits;
  uint32_t* o_name_id;
  uint32_t* met;  // metric / layer flags for the scans
  uint32_t* lay;
};

__global__ void k_final_spans(Final f) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  const uint32_t j = f.perm ? f.perm[i] : (uint32_t)i;
  f.o_span_id[i] = f.span_id[j];
  f.o_parent[i] = f.parent[j];
  f.o_begin[i] = f.begin[j];
  f.o_end[i] = f.end[j];
  f.o_cid[i] = f.cid[j];
  f.o_trace_id[i] = f.trace_id[j];
  const uint8_t fl = f.flags[j];
  f.o_flags[i] = fl;
  f.o_tag_bits[i] = f.tag_bits[j];
  f.o_name_id[i] = f.name_id[j];
  f.met[i] = (fl & XSP_F_METRICS) ? 1u : 0u;
  f.lay[i] = (fl & 3u) == XSP_LEVEL_LAYER ? 1u : 0u;
}

__global__ void k_final_tables(Final f, const uint32_t* __restrict__ mpos, const uint32_t* __restrict__ lpos,
                               uint64_t* __restrict__ flops, uint64_t* __restrict__ dread,
                               uint64_t* __restrict__ dwrite, double* __restrict__ occ,
                               int64_t* __restrict__ alloc, uint32_t* __restrict__ type_id) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  const uint32_t j = f.perm ? f.perm[i] : (uint32_t)i;
  if (f.met[i]) {
    const uint32_t m = mpos[i];
    flops[m] = f.flops[j];
    dread[m] = f.dread[j];
    dwrite[m] = f.dwrite[j];
    occ[m] = f.occ[j];
  }
  if (f.lay[i]) {
    const uint32_t q = lpos[i];
    alloc[q] = f.alloc[j];
    type_id[q] = f.type_id[j];
  }
}

// ---- interning by hash table (one insert pass; no sort of the span keys) ----
// Slot keys are the 64-bit string hashes of the parser (kHashEmpty = a free slot;
// a string hashing to it goes to the host interner); each slot keeps one member
// as its representative, every other member is byte-compared with it.
constexpr uint64_t kHashEmpty = ~0ull;
__global__ void k_mask_hash(uint64_t* __restrict__ h, uint64_t n, uint64_t mask) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) h[i] &= mask;
}

__global__ void k_hash_insert(const uint64_t* __restrict__ hash, const uint8_t* __restrict__ use, uint64_t n,
                              uint64_t mask, unsigned long long* __restrict__ tkey, uint32_t* __restrict__ trep,
                              uint32_t* __restrict__ slot_of, uint32_t* __restrict__ bad) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n || (use && !use[j])) return;
  const uint64_t h = hash[j];
  if (h == kHashEmpty) {
    *bad = 1;
    return;
  }
  uint64_t sl = (h ^ (h >> 29)) & mask;
  for (uint64_t probes = 0; probes <= mask; ++probes) {
    unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(tkey + sl);
    if (k == kHashEmpty) {
      k = atomicCAS(tkey + sl, kHashEmpty, (unsigned long long)h);
      if (k == kHashEmpty) {
        trep[sl] = (uint32_t)j;
        slot_of[j] = (uint32_t)sl;
        return;
      }
    }
    if (k == h) {
      slot_of[j] = (uint32_t)sl;
      return;
    }
    sl = (sl + 1) & mask;
  }
  *bad = 1;
}

// every member byte-equal to its slot's representative (else a hash collision)
__global__ void k_hash_verify(const char* __restrict__ t, const uint64_t* __restrict__ off,
                              const uint32_t* __restrict__ len, const uint32_t* __restrict__ slot_of,
                              const uint32_t* __restrict__ trep, const uint8_t* __restrict__ use, uint64_t n,
                              uint32_t* __restrict__ bad) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n || (use && !use[j])) return;
  const uint32_t r = *reinterpret_cast<const volatile uint32_t*>(trep + slot_of[j]);
  if (r == (uint32_t)j) return;
  if (len[r] != len[j]) {
    *bad = 1;
    return;
  }
  const char* a = t + off[j];
  const char* b = t + off[r];
  for (uint32_t k = 0; k < len[j]; ++k)
    if (a[k] != b[k]) {
      *bad = 1;
      return;
    }
}

__global__ void k_slot_used(const unsigned long long* __restrict__ tkey, uint64_t cap, uint32_t* __restrict__ used) {
  const uint64_t sl = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sl < cap) used[sl] = tkey[sl] != kHashEmpty;
}

// dense run number of each used slot; its representative's byte range
__global__ void k_slot_compact(const uint32_t* __restrict__ used, const uint32_t* __restrict__ pos,
                               const uint32_t* __restrict__ trep, const uint64_t* __restrict__ off,
                               const uint32_t* __restrict__ len, uint64_t cap, uint32_t* __restrict__ dense,
                               uint64_t* __restrict__ ro, uint32_t* __restrict__ rl, uint32_t* __restrict__ maxlen,
                               unsigned long long* __restrict__ total) {
  const uint64_t sl = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= cap || !used[sl]) return;
  const uint32_t u = pos[sl], r = trep[sl];
  dense[sl] = u;
  ro[u] = off[r];
  rl[u] = len[r];
  atomicMax(maxlen, len[r]);
  atomicAdd(total, (unsigned long long)len[r]);
}

__global__ void k_iota_u32(uint32_t* __restrict__ v, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}

// big-endian word w (bytes [8w, 8w + 8), zero padded) of distinct string ord[i]
__global__ void k_word_keys(const char* __restrict__ t, const uint64_t* __restrict__ ro,
                            const uint32_t* __restrict__ rl, const uint32_t* __restrict__ ord, uint64_t U, uint32_t w,
                            uint64_t* __restrict__ key) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= U) return;
  const uint32_t u = ord[i], l = rl[u];
  const unsigned char* a = reinterpret_cast<const unsigned char*>(t + ro[u]);
  uint64_t k = 0;
  for (uint32_t b = 0; b < 8; ++b) {
    const uint32_t at = 8 * w + b;
    k = k << 8 | (at < l ? a[at] : 0u);
  }
  key[i] = k;
}

// rank of each distinct string; the lengths in id order
__global__ void k_rank_lengths(const uint32_t* __restrict__ ord, const uint32_t* __restrict__ rl, uint64_t U,
                               uint32_t* __restrict__ rank, uint64_t* __restrict__ sl) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= U) return;
  rank[ord[k]] = (uint32_t)k;
  sl[k] = rl[ord[k]];
}

// string of id k to blob[so[k], so[k + 1])
__global__ void k_gather_sorted(const char* __restrict__ t, const uint64_t* __restrict__ ro,
                                const uint32_t* __restrict__ rl, const uint32_t* __restrict__ ord,
                                const uint64_t* __restrict__ so, uint64_t U, char* __restrict__ blob) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= U) return;
  const uint32_t u = ord[k];
  const char* a = t + ro[u];
  char* d = blob + so[k];
  for (uint32_t b = 0; b < rl[u]; ++b) d[b] = a[b];
}

__global__ void k_map_slots(const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ dense,
                            const uint32_t* __restrict__ rank, const uint8_t* __restrict__ use, uint64_t n,
                            uint32_t* __restrict__ ids) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) ids[j] = (use && !use[j]) ? 0u : rank[dense[slot_of[j]]];
}

unsigned blocks(uint64_t n) { return ceil_div(n ? n : 1, 256); }

// ---- canonical meta record on the host (encode_meta_record layout)
struct HostCur {
  const char* p;
  const char* e;
  bool lit(const char* s) {
    const size_t k = std::strlen(s);
    if ((size_t)(e - p) < k || std::memcmp(p, s, k) != 0) return false;
    p += k;
    return true;
  }
  bool u64(uint64_t& v) {
    if (p >= e || *p < '0' || *p > '9') return false;
    if (*p == '0') {
      ++p;
      v = 0;
      return p >= e || *p < '0' || *p > '9';
    }
    uint64_t x = 0;
    while (p < e && *p >= '0' && *p <= '9') {
      const uint64_t d = (uint64_t)(*p - '0');
      if (x > (~0ull - d) / 10) return false;
      x = x * 10 + d;
      ++p;
    }
    v = x;
    return true;
  }
  bool str(std::string& out) {
    if (p >= e || *p != '"') return false;
    const char* s = ++p;
    while (p < e && *p != '"') {
      const unsigned char c = (unsigned char)*p;
      if (c < 0x20 || c >= 0x80 || c == '\\') return false;
      ++p;
    }
    if (p >= e) return false;
    out.assign(s, p);
    ++p;
    return true;
  }
  bool number(double& d) {  // JSON number -> double (strtod: correctly rounded)
    const char* s = p;
    if (p < e && *p == '-') ++p;
    if (p >= e || *p < '0' || *p > '9') return false;
    if (*p == '0') {
      ++p;
      if (p < e && *p >= '0' && *p <= '9') return false;
    }
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p < e && *p == '.') {
      ++p;
      if (p >= e || *p < '0' || *p > '9') return false;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || *p < '0' || *p > '9') return false;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    const std::string t(s, p);
    d = std::strtod(t.c_str(), nullptr);
    return std::isfinite(d);
  }
};

struct Meta {
  uint64_t trace_id = 0, batch = 0, run = 0;
  uint32_t levels = 0;
  bool serialized = false;
  std::string sys_name;
  double peak = 0.0, bw = 0.0;
};

bool parse_meta(const char* s, const char* e, Meta& m) {
  HostCur c{s, e};
  if (!c.lit("{\"batch_size\":") || !c.u64(m.batch) || !c.lit(",\"levels\":[")) return false;
  if (!c.lit("]")) {
    for (;;) {
      std::string l;
      if (!c.str(l)) return false;
      int bit = l == "model" ? 0 : l == "layer" ? 1 : l == "kernel" ? 2 : l == "api" ? 3 : -1;
      if (bit < 0) return false;
      m.levels |= 1u << bit;
      if (c.lit(",")) continue;
      if (c.lit("]")) break;
      return false;
    }
  }
  if (!c.lit(",\"rec\":\"meta\",\"run_index\":") || !c.u64(m.run)) return false;
  if (!c.lit(",\"serialized\":")) return false;
  if (c.lit("true")) m.serialized = true;
  else if (!c.lit("false")) return false;
  if (!c.lit(",\"system\":{\"mem_bw\":") || !c.number(m.bw)) return false;
  if (!c.lit(",\"name\":") || !c.str(m.sys_name)) return false;
  if (!c.lit(",\"peak_flops\":") || !c.number(m.peak)) return false;
  if (!c.lit("},\"trace_id\":") || !c.u64(m.trace_id) || !c.lit("}")) return false;
  while (c.p < c.e && (*c.p == '\r' || *c.p == ' ' || *c.p == '\t')) ++c.p;
  return c.p == c.e && m.batch <= 0xFFFFFFFFull && m.run <= 0xFFFFFFFFull;
}

// interning: returns false on a hash collision; fills the string table (sorted)
// and ids[j] for the used entries
bool intern(xsp_ctx* ctx, const std::string& tag, const char* dtext, const char* htext, uint64_t n,
            const uint64_t* hash, const uint64_t* off, const uint32_t* len, const uint8_t* use, uint32_t* ids,
            std::string& tblob, std::vector<uint64_t>& toff, cudaStream_t st) {
  tblob.clear();
  toff.assign(1, 0);
  if (n == 0) return true;
  if (const char* e = std::getenv("XSP_INGEST_HASH_BITS")) {  // test hook: force hash collisions
    const int bits = std::atoi(e);
    if (bits > 0 && bits < 64)
      k_mask_hash<<<blocks(n), 256, 0, st>>>(const_cast<uint64_t*>(hash), n, (1ull << bits) - 1);
  }
  uint64_t cap = 1024;
  while (cap < 2 * n) cap <<= 1;
  auto* tkey = ctx->d<unsigned long long>(tag + ".tk", cap);
  uint32_t* trep = ctx->d<uint32_t>(tag + ".tr", cap);
  uint32_t* slot_of = ctx->d<uint32_t>(tag + ".so", n);
  uint32_t* used = ctx->d<uint32_t>(tag + ".us", cap + 1);
  uint32_t* pos = ctx->d<uint32_t>(tag + ".ps", cap + 1);
  uint32_t* dense = ctx->d<uint32_t>(tag + ".dn", cap);
  // [0] distinct strings [1] collision / probe overflow [2] longest [3] (pad) [4..5] total bytes
  uint32_t* cnt = ctx->d<uint32_t>(tag + ".cn", 6);
  XSP_CUDA(cudaMemsetAsync(tkey, 0xFF, cap * 8, st));
  XSP_CUDA(cudaMemsetAsync(cnt, 0, 24, st));
  k_hash_insert<<<blocks(n), 256, 0, st>>>(hash, use, n, cap - 1, tkey, trep, slot_of, cnt + 1);
  k_hash_verify<<<blocks(n), 256, 0, st>>>(dtext, off, len, slot_of, trep, use, n, cnt + 1);
  k_slot_used<<<blocks(cap), 256, 0, st>>>(tkey, cap, used);
  uint32_t* scr = ctx->d<uint32_t>(tag + ".sc", scan_scratch_elems(cap + 1));
  exclusive_scan<uint32_t, uint32_t>(used, pos, cap, scr, cnt, st, &ctx->launches);
  // the representatives' byte ranges (at most n of them), longest, total bytes
  uint64_t* d_ro = ctx->d<uint64_t>(tag + ".ro", n + 1);
  uint32_t* d_rl = ctx->d<uint32_t>(tag + ".rl", n + 1);
  k_slot_compact<<<blocks(cap), 256, 0, st>>>(used, pos, trep, off, len, cap, dense, d_ro, d_rl, cnt + 2,
                                               reinterpret_cast<unsigned long long*>(cnt + 4));
  uint32_t* h2 = ctx->h<uint32_t>(tag + ".h2", 6);
  XSP_CUDA(cudaMemcpyAsync(h2, cnt, 24, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  if (h2[1]) return false;
  const uint32_t U = h2[0], maxlen = h2[2];
  uint64_t nb;
  std::memcpy(&nb, h2 + 4, 8);
  if (U == 0) {  // nothing used (no layer spans): every id 0
    k_map_slots<<<blocks(n), 256, 0, st>>>(slot_of, dense, dense, use, n, ids);
    ++ctx->launches;
    return true;
  }
  // ids in lexicographic order of the strings (the reference interns sorted
  // names): an LSD radix sort of the distinct strings over their big-endian
  // 8-byte words on the device (zero padded: the strings hold no NUL), last
  // word first; strings longer than kDevSortMax are sorted on the host
  constexpr uint32_t kDevSortMax = 256;
  uint32_t* d_ord = ctx->d<uint32_t>(tag + ".ord", U + 1ull);
  if (maxlen <= kDevSortMax) {
    uint64_t* d_key = ctx->d<uint64_t>(tag + ".key", U + 1ull);
    RadixScratch rs;
    rs.keys_alt = ctx->d<uint64_t>(tag + ".rs.ka", U + 1ull);
    rs.vals_alt = ctx->d<uint32_t>(tag + ".rs.va", U + 1ull);
    const uint64_t ce = radix_counts_elems(U);
    rs.counts = ctx->d<uint32_t>(tag + ".rs.c", ce);
    rs.scan_tmp = ctx->d<uint32_t>(tag + ".rs.s", scan_scratch_elems(ce));
    rs.and_or = ctx->d<unsigned long long>(tag + ".rs.ao", 2);
    rs.and_or_host = ctx->h<unsigned long long>(tag + ".rs.aoh", 2);
    k_iota_u32<<<blocks(U), 256, 0, st>>>(d_ord, U);
    for (int w = (int)((maxlen + 7) / 8) - 1; w >= 0; --w) {
      k_word_keys<<<blocks(U), 256, 0, st>>>(dtext, d_ro, d_rl, d_ord, U, (uint32_t)w, d_key);
      radix_sort_pairs(d_key, d_ord, U, 0, 64, rs, st, &ctx->launches);
    }
  } else {
    uint64_t* roff = ctx->h<uint64_t>(tag + ".hro", U + 1ull);
    uint32_t* rlen = ctx->h<uint32_t>(tag + ".hrl", U + 1ull);
    XSP_CUDA(cudaMemcpyAsync(roff, d_ro, U * 8ull, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaMemcpyAsync(rlen, d_rl, U * 4ull, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaStreamSynchronize(st));
    uint32_t* order = ctx->h<uint32_t>(tag + ".hord", U + 1ull);
    for (uint32_t r = 0; r < U; ++r) order[r] = r;
    std::sort(order, order + U, [&](uint32_t a, uint32_t b) {
      return std::string_view(htext + roff[a], rlen[a]) < std::string_view(htext + roff[b], rlen[b]);
    });
    XSP_CUDA(cudaMemcpyAsync(d_ord, order, U * 4ull, cudaMemcpyHostToDevice, st));
  }
  // ranks, the strings in id order as one blob, the span ids
  uint32_t* d_rank = ctx->d<uint32_t>(tag + ".rank", U + 1ull);
  uint64_t* d_sl = ctx->d<uint64_t>(tag + ".sl", U + 1ull);
  uint64_t* d_so = ctx->d<uint64_t>(tag + ".so64", U + 1ull);
  uint64_t* scr64 = ctx->d<uint64_t>(tag + ".sc64", scan_scratch_elems(U + 1ull));
  char* d_blob = ctx->d<char>(tag + ".blob", nb + 1);
  k_rank_lengths<<<blocks(U), 256, 0, st>>>(d_ord, d_rl, U, d_rank, d_sl);
  exclusive_scan<uint64_t, uint64_t>(d_sl, d_so, U, scr64, d_so + U, st, &ctx->launches);
  k_gather_sorted<<<blocks(U), 256, 0, st>>>(dtext, d_ro, d_rl, d_ord, d_so, U, d_blob);
  k_map_slots<<<blocks(n), 256, 0, st>>>(slot_of, dense, d_rank, use, n, ids);
  char* hblob = ctx->h<char>(tag + ".hblob", nb + 1);
  uint64_t* hso = ctx->h<uint64_t>(tag + ".hso", U + 1ull);
  XSP_CUDA(cudaMemcpyAsync(hblob, d_blob, nb, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaMemcpyAsync(hso, d_so, (U + 1ull) * 8, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  tblob.assign(hblob, nb);
  toff.assign(hso, hso + U + 1);
  ctx->launches += 9;
  return true;
}

}  // namespace

// ctx-owned host storage of one ingest result
struct IngestHost {
  std::string blob_names, blob_types;  // interned strings in id order

  std::vector<uint64_t> off_names, off_types;
  std::vector<uint64_t> span_off, trace_id;
  std::vector<uint32_t> levels, batch, run;
  std::vector<uint8_t> serialized;
  std::string sys_name;
};

void run_ingest_jsonl(xsp_ctx* ctx, const char* htext, const uint64_t* soff, uint32_t S, xsp_ingest_out* out,
                      cudaStream_t st) {
  static thread_local IngestHost H;  // one result per thread (pointers valid until the next call)
  // XSP_INGEST_TRACE=1: host wall time at the phase boundaries (after syncs)
  const bool trace = std::getenv("XSP_INGEST_TRACE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    XSP_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr, "ingest %-10s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  };
  std::memset(out, 0, sizeof(*out));
  out->status = XSP_INGEST_HOST;
  out->bad_stream = 0;
  const uint64_t n_text = soff[S];
  // ---- text to the device; one line boundary per stream end so lines never straddle streams
  char* dtext = ctx->d<char>("ig.text", n_text + 1);
  XSP_CUDA(cudaMemcpyAsync(dtext, htext, n_text, cudaMemcpyHostToDevice, st));
  ctx->h2d_bytes = n_text;
  const uint64_t nch = ceil_div(n_text ? n_text : 1, kNlChunk);
  uint32_t* cnt = ctx->d<uint32_t>("ig.nlc", nch + 1);
  uint32_t* pos = ctx->d<uint32_t>("ig.nlp", nch + 1);
  uint32_t* tot = ctx->d<uint32_t>("ig.nlt", 1);
  mark("h2d");
  k_nl_count<<<blocks(nch), 256, 0, st>>>(dtext, n_text, cnt);
  uint32_t* scr = ctx->d<uint32_t>("ig.scan", scan_scratch_elems(nch + 1));
  exclusive_scan<uint32_t, uint32_t>(cnt, pos, nch, scr, tot, st, &ctx->launches);
  uint32_t hnl = 0;
  XSP_CUDA(cudaMemcpyAsync(&hnl, tot, 4, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  // newline positions, then the lines (device): newlines + unterminated stream tails
  uint64_t* nl = ctx->d<uint64_t>("ig.nl", hnl + 1ull);
  k_nl_write<<<blocks(nch), 256, 0, st>>>(dtext, n_text, pos, nl);
  uint64_t* d_tsoff = ctx->d<uint64_t>("ig.tsoff", S + 1ull);
  uint64_t* h_tsoff = ctx->h<uint64_t>("ig.htsoff", S + 1ull);
  std::memcpy(h_tsoff, soff, (S + 1ull) * 8);
  XSP_CUDA(cudaMemcpyAsync(d_tsoff, h_tsoff, (S + 1ull) * 8, cudaMemcpyHostToDevice, st));
  uint64_t* nbefore = ctx->d<uint64_t>("ig.nbef", S + 1ull);
  uint32_t* tail = ctx->d<uint32_t>("ig.tail", S + 1ull);
  uint32_t* tb = ctx->d<uint32_t>("ig.tb", S + 1ull);
  k_stream_lines<<<blocks(S + 1ull), 256, 0, st>>>(nl, hnl, d_tsoff, S, nbefore, tail);
  uint32_t* scr_s = ctx->d<uint32_t>("ig.scs", scan_scratch_elems(S + 1ull));
  exclusive_scan<uint32_t, uint32_t>(tail, tb, S, scr_s, tb + S, st, &ctx->launches);
  uint32_t* h_nt = ctx->h<uint32_t>("ig.hnt", 1);
  XSP_CUDA(cudaMemcpyAsync(h_nt, tb + S, 4, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  const uint64_t L = hnl + (uint64_t)*h_nt;
  uint64_t* lstart = ctx->d<uint64_t>("ig.ls", L + 1);
  uint64_t* lend = ctx->d<uint64_t>("ig.le", L + 1);
  uint32_t* lstream = ctx->d<uint32_t>("ig.lst", L + 1);
  if (hnl) k_lines_nl<<<blocks(hnl), 256, 0, st>>>(nl, hnl, d_tsoff, S, tb, lstart, lend, lstream);
  if (S) k_lines_tail<<<blocks(S), 256, 0, st>>>(nl, nbefore, d_tsoff, S, tail, tb, lstart, lend, lstream);
  ctx->launches += 4;
  // ---- parse every line
  LineOut lo;
  lo.kind = ctx->d<uint8_t>("ig.kind", L + 1);
  lo.span_id = ctx->d<uint64_t>("ig.l.sid", L);
  lo.parent = ctx->d<uint64_t>("ig.l.par", L);
  lo.begin = ctx->d<uint64_t>("ig.l.b", L);
  lo.end = ctx->d<uint64_t>("ig.l.e", L);
  lo.cid = ctx->d<uint64_t>("ig.l.cid", L);
  lo.trace_id = ctx->d<uint64_t>("ig.l.tid", L);
  lo.flags = ctx->d<uint8_t>("ig.l.f", L);
  lo.name_hash = ctx->d<uint64_t>("ig.l.nh", L);
  lo.name_off = ctx->d<uint64_t>("ig.l.no", L);
  lo.name_len = ctx->d<uint32_t>("ig.l.nl", L);
  lo.type_hash = ctx->d<uint64_t>("ig.l.th", L);
  lo.type_off = ctx->d<uint64_t>("ig.l.to", L);
  lo.type_len = ctx->d<uint32_t>("ig.l.tl", L);
  lo.flops = ctx->d<uint64_t>("ig.l.fl", L);
  lo.dread = ctx->d<uint64_t>("ig.l.dr", L);
  lo.dwrite = ctx->d<uint64_t>("ig.l.dw", L);
  lo.occ = ctx->d<double>("ig.l.oc", L);
  lo.alloc = ctx->d<int64_t>("ig.l.al", L);
  lo.tag_bits = ctx->d<uint8_t>("ig.l.tb", L);
  mark("lines");
  if (L) k_parse_lines<<<blocks(L), 256, 0, st>>>(dtext, n_text, lstart, lend, L, lo);
  mark("parse");
  // ---- per stream: exactly one meta record (parsed on the host), no line the
  // device parser left to the host; counted on the device, the host touches
  // only the S meta lines (the exact line-order walk runs only for a bad batch)
  LineStats ls;
  ls.nmeta = ctx->d<uint32_t>("ig.nmeta", 2ull * S + 1);
  ls.nspan = ls.nmeta + S;
  ls.mline = ctx->d<unsigned long long>("ig.mline", S + 1ull);
  ls.first_host = ls.mline + S;
  uint64_t* mrange = ctx->d<uint64_t>("ig.mrange", 2ull * S + 1);
  XSP_CUDA(cudaMemsetAsync(ls.nmeta, 0, (2ull * S + 1) * 4, st));
  XSP_CUDA(cudaMemsetAsync(ls.first_host, 0xFF, 8, st));
  if (L) k_line_stats<<<blocks(L), 256, 0, st>>>(lo.kind, lstream, L, ls);
  if (S) k_meta_ranges<<<blocks(S), 256, 0, st>>>(ls.mline, ls.nmeta, S, lstart, lend, mrange);
  uint32_t* h_cnt = ctx->h<uint32_t>("ig.hcnt", 2ull * S + 1);
  uint64_t* h_mr = ctx->h<uint64_t>("ig.hmr", 2ull * S + 2);
  XSP_CUDA(cudaMemcpyAsync(h_cnt, ls.nmeta, 2ull * S * 4, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaMemcpyAsync(h_mr, mrange, 2ull * S * 8, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaMemcpyAsync(h_mr + 2ull * S, ls.first_host, 8, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  ctx->launches += 6;
  std::vector<Meta> meta(S);
  std::vector<uint64_t> nspan(S, 0);
  bool clean = h_mr[2ull * S] == ~0ull;
  for (uint32_t s = 0; s < S && clean; ++s) clean = h_cnt[s] == 1;
  if (clean) {
    for (uint32_t s = 0; s < S; ++s) {
      if (!parse_meta(htext + h_mr[2 * s], htext + h_mr[2 * s + 1], meta[s])) {
        out->bad_stream = s;  // the first bad meta line in line order
        return;
      }
      nspan[s] = h_cnt[S + s];
    }
  } else {  // the first violation in line order, as the host ingest meets it
    std::vector<uint8_t> hkind(L);
    std::vector<uint32_t> hls(L);
    std::vector<uint64_t> hst(L), hen(L);
    XSP_CUDA(cudaMemcpyAsync(hkind.data(), lo.kind, L, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaMemcpyAsync(hls.data(), lstream, L * 4, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaMemcpyAsync(hst.data(), lstart, L * 8, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaMemcpyAsync(hen.data(), lend, L * 8, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaStreamSynchronize(st));
    std::vector<int> nmeta(S, 0);
    for (uint64_t l = 0; l < L; ++l) {
      const uint32_t s = hls[l];
      if (hkind[l] == LK_HOST) {
        out->bad_stream = s;
        return;
      }
      if (hkind[l] == LK_META) {
        if (++nmeta[s] > 1 || !parse_meta(htext + hst[l], htext + hen[l], meta[s])) {
          out->bad_stream = s;
          return;
        }
      }
    }
    for (uint32_t s = 0; s < S; ++s)
      if (nmeta[s] != 1) {
        out->bad_stream = s;
        return;
      }
    return;  // unreachable: a clean batch takes the branch above
  }
  uint64_t n = 0;
  H.span_off.assign(S + 1, 0);
  for (uint32_t s = 0; s < S; ++s) H.span_off[s + 1] = H.span_off[s] + nspan[s];
  n = H.span_off[S];
  if (n >= 0xFFFFFFF0ull) throw std::invalid_argument("more than 2^32-16 spans in one call");
  // ---- span lines -> spans (file order)
  uint32_t* isspan = ctx->d<uint32_t>("ig.iss", L + 1);
  uint32_t* spos = ctx->d<uint32_t>("ig.spos", L + 1);
  uint32_t* stot = ctx->d<uint32_t>("ig.stot", 1);
  k_span_flags<<<blocks(L), 256, 0, st>>>(lo.kind, L, isspan);
  uint32_t* scr2 = ctx->d<uint32_t>("ig.scan2", scan_scratch_elems(L + 1));
  exclusive_scan<uint32_t, uint32_t>(isspan, spos, L, scr2, stot, st, &ctx->launches);
  Gather g;
  g.isspan = isspan;
  g.spos = spos;
  g.nl = lend;
  g.nlines = L;
  g.lo = lo;
  g.span_id = ctx->d<uint64_t>("ig.s.sid", n + 1);
  g.parent = ctx->d<uint64_t>("ig.s.par", n + 1);
  g.begin = ctx->d<uint64_t>("ig.s.b", n + 1);
  g.end = ctx->d<uint64_t>("ig.s.e", n + 1);
  g.cid = ctx->d<uint64_t>("ig.s.cid", n + 1);
  g.trace_id = ctx->d<uint64_t>("ig.s.tid", n + 1);
  g.name_hash = ctx->d<uint64_t>("ig.s.nh", n + 1);
  g.type_hash = ctx->d<uint64_t>("ig.s.th", n + 1);
  g.name_off = ctx->d<uint64_t>("ig.s.no", n + 1);
  g.type_off = ctx->d<uint64_t>("ig.s.to", n + 1);
  g.name_len = ctx->d<uint32_t>("ig.s.nl", n + 1);
  g.type_len = ctx->d<uint32_t>("ig.s.tl", n + 1);
  g.line_of = ctx->d<uint32_t>("ig.s.line", n + 1);
  g.flags = ctx->d<uint8_t>("ig.s.f", n + 1);
  g.tag_bits = ctx->d<uint8_t>("ig.s.tb", n + 1);
  g.flops = ctx->d<uint64_t>("ig.s.fl", n + 1);
  g.dread = ctx->d<uint64_t>("ig.s.dr", n + 1);
  g.dwrite = ctx->d<uint64_t>("ig.s.dw", n + 1);
  g.occ = ctx->d<double>("ig.s.oc", n + 1);
  g.alloc = ctx->d<int64_t>("ig.s.al", n + 1);
  mark("meta");
  k_gather_spans<<<blocks(L), 256, 0, st>>>(g);
  mark("gather");
  ctx->launches += 2;
  // ---- intern names (every span) and layer types (layer spans only)
  uint32_t* name_fid = ctx->d<uint32_t>("ig.s.nid", n + 1);
  uint32_t* type_fid = ctx->d<uint32_t>("ig.s.tyid", n + 1);
  uint8_t* is_layer = ctx->d<uint8_t>("ig.s.isl", n + 1);
  if (n) k_is_layer<<<blocks(n), 256, 0, st>>>(g.flags, n, is_layer);
  if (!intern(ctx, "ig.in", dtext, htext, n, g.name_hash, g.name_off, g.name_len, nullptr, name_fid, H.blob_names,
              H.off_names, st)) {
    out->bad_stream = 0;  // a hash collision: the host interns
    return;
  }
  mark("names");
  if (!intern(ctx, "ig.it", dtext, htext, n, g.type_hash, g.type_off, g.type_len, is_layer, type_fid, H.blob_types,
              H.off_types, st)) {
    out->bad_stream = 0;
    return;
  }
  mark("types");
  // ---- trace arrays (host) and the trace_id check (ingest's own fault, collector.cpp:248-255)
  H.trace_id.resize(S);
  H.levels.resize(S);
  H.batch.resize(S);
  H.run.resize(S);
  H.serialized.resize(S);
  for (uint32_t s = 0; s < S; ++s) {
    H.trace_id[s] = meta[s].trace_id;
    H.levels[s] = meta[s].levels;
    H.batch[s] = (uint32_t)meta[s].batch;
    H.run[s] = (uint32_t)meta[s].run;
    H.serialized[s] = meta[s].serialized;
  }
  H.sys_name = S ? meta[0].sys_name : std::string();
  uint64_t* d_soff = ctx->d<uint64_t>("ig.soff", S + 1ull);
  XSP_CUDA(cudaMemcpyAsync(d_soff, H.span_off.data(), (S + 1ull) * 8, cudaMemcpyHostToDevice, st));
  uint64_t* d_mtid = ctx->d<uint64_t>("ig.mtid", S + 1ull);
  XSP_CUDA(cudaMemcpyAsync(d_mtid, H.trace_id.data(), S * 8ull, cudaMemcpyHostToDevice, st));
  uint32_t* d_lv = ctx->d<uint32_t>("ig.lv", S + 1ull);
  XSP_CUDA(cudaMemcpyAsync(d_lv, H.levels.data(), S * 4ull, cudaMemcpyHostToDevice, st));
  {
    uint32_t* bad = ctx->d<uint32_t>("ig.badtid", 1);
    XSP_CUDA(cudaMemsetAsync(bad, 0xFF, 4, st));
    if (n) k_tid_check<<<blocks(n), 256, 0, st>>>(g.trace_id, d_soff, S, d_mtid, n, bad);
    uint32_t hb = 0;
    XSP_CUDA(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaStreamSynchronize(st));
    if (hb != 0xFFFFFFFFu) {
      out->bad_stream = hb;
      return;
    }
  }
  // ---- sort_timeline per trace (stage (b)), then the final columns
  uint32_t* perm = ctx->d<uint32_t>("ig.perm", n + 1);
  uint32_t sorted = 1;
  mark("intern");
  if (n) run_sort_timeline(ctx, n, g.begin, g.flags, g.span_id, S, d_soff, perm, &sorted, st);
  mark("sort");
  Final f;
  f.perm = sorted ? nullptr : perm;
  f.n = n;
  f.span_id = g.span_id; f.parent = g.parent; f.begin = g.begin; f.end = g.end; f.cid = g.cid;
  f.trace_id = g.trace_id; f.flags = g.flags; f.tag_bits = g.tag_bits; f.name_id = name_fid;
  f.type_id = type_fid; f.flops = g.flops; f.dread = g.dread; f.dwrite = g.dwrite; f.occ = g.occ;
  f.alloc = g.alloc;
  xsp_span_cols& c = out->cols;
  c.n_spans = n;
  c.span_id = f.o_span_id = ctx->d<uint64_t>("ig.o.sid", n + 1);
  c.parent_id = f.o_parent = ctx->d<uint64_t>("ig.o.par", n + 1);
  c.begin_ns = f.o_begin = ctx->d<uint64_t>("ig.o.b", n + 1);
  c.end_ns = f.o_end = ctx->d<uint64_t>("ig.o.e", n + 1);
  c.cid = f.o_cid = ctx->d<uint64_t>("ig.o.cid", n + 1);
  f.o_trace_id = ctx->d<uint64_t>("ig.o.tid", n + 1);
  c.flags = f.o_flags = ctx->d<uint8_t>("ig.o.f", n + 1);
  f.o_tag_bits = ctx->d<uint8_t>("ig.o.tb", n + 1);
  c.name_id = f.o_name_id = ctx->d<uint32_t>("ig.o.nid", n + 1);
  f.met = ctx->d<uint32_t>("ig.o.met", n + 1);
  f.lay = ctx->d<uint32_t>("ig.o.lay", n + 1);
  if (n) k_final_spans<<<blocks(n), 256, 0, st>>>(f);
  uint32_t* mpos = ctx->d<uint32_t>("ig.mpos", n + 1);
  uint32_t* lpos = ctx->d<uint32_t>("ig.lpos", n + 1);
  uint32_t* mtot = ctx->d<uint32_t>("ig.mtot", 2);
  uint32_t* scr3 = ctx->d<uint32_t>("ig.scan3", scan_scratch_elems(n + 1));
  exclusive_scan<uint32_t, uint32_t>(f.met, mpos, n, scr3, mtot, st, &ctx->launches);
  exclusive_scan<uint32_t, uint32_t>(f.lay, lpos, n, scr3, mtot + 1, st, &ctx->launches);
  uint32_t ht[2] = {0, 0};
  XSP_CUDA(cudaMemcpyAsync(ht, mtot, 8, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  c.n_metric_rows = ht[0];
  c.n_layer_rows = ht[1];
  uint64_t* o_fl = ctx->d<uint64_t>("ig.o.fl", ht[0] + 1ull);
  uint64_t* o_dr = ctx->d<uint64_t>("ig.o.dr", ht[0] + 1ull);
  uint64_t* o_dw = ctx->d<uint64_t>("ig.o.dw", ht[0] + 1ull);
  double* o_oc = ctx->d<double>("ig.o.oc", ht[0] + 1ull);
  int64_t* o_al = ctx->d<int64_t>("ig.o.al", ht[1] + 1ull);
  uint32_t* o_ty = ctx->d<uint32_t>("ig.o.ty", ht[1] + 1ull);
  c.flops = o_fl;
  c.dram_read = o_dr;
  c.dram_write = o_dw;
  c.occupancy = o_oc;
  c.alloc_bytes = o_al;
  c.type_id = o_ty;
  if (n) k_final_tables<<<blocks(n), 256, 0, st>>>(f, mpos, lpos, o_fl, o_dr, o_dw, o_oc, o_al, o_ty);
  ctx->launches += 2;
  out->traces.n_traces = S;
  out->traces.span_off = d_soff;
  out->traces.levels = d_lv;
  // ---- validate_bundle (stage (a)); any issue: the host reproduces ingest's exact fault
  xsp_validate_in vin{f.o_trace_id, d_mtid, f.o_tag_bits};
  xsp_validation_out vout;
  std::memset(&vout, 0, sizeof(vout));
  mark("columns");
  run_validate(ctx, &c, &out->traces, &vin, &vout, st);
  mark("validate");
  if (vout.n_issues) {
    std::vector<uint32_t> toff(S + 1);
    XSP_CUDA(cudaMemcpyAsync(toff.data(), vout.trace_issue_off, (S + 1ull) * 4, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaStreamSynchronize(st));
    for (uint32_t s = 0; s < S; ++s)
      if (toff[s + 1] > toff[s]) {
        out->bad_stream = s;
        break;
      }
    return;
  }
  // ---- host side of the result
  out->names = {(uint32_t)(H.off_names.size() - 1), H.blob_names.data(), H.off_names.data()};
  out->types = {(uint32_t)(H.off_types.size() - 1), H.blob_types.data(), H.off_types.data()};
  out->trace_id = H.trace_id.data();
  out->trace_batch = H.batch.data();
  out->trace_run = H.run.data();
  out->trace_serialized = H.serialized.data();
  out->span_off_host = H.span_off.data();
  out->levels_host = H.levels.data();
  out->system_name = H.sys_name.c_str();
  out->peak_flops = S ? meta[0].peak : 0.0;
  out->mem_bw = S ? meta[0].bw : 0.0;
  out->status = XSP_INGEST_OK;
  XSP_CUDA(cudaStreamSynchronize(st));
}

}  // namespace xsp
