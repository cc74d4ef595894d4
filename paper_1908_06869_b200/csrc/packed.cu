// Packed host input for xsp_run_host_packed (include/xsp.h xsp_packed_cols).
//
// The end-to-end path is PCIe-bound: xsp_run_host moves ~52 B per span to the
// device, 37 of them in the five 8-byte span columns. Packed, the wire carries
// begin as a u32 delta, end as a u32 duration, cid as a u32 offset from its
// block base (cid spans only) and parent_id for explicit-parent spans only —
// ~34 B per span for C3 — and one CTA per 256-span block rebuilds the full
// columns in HBM (segmented scan of the begin deltas, in-block ranks of the
// sparse entries). Values that do not fit (trace and block starts, negative
// or >= 2^32 deltas, durations, cid offsets) travel raw in a sorted escape
// list.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <unordered_map>
#include <vector>

#include "ctx.h"
#include "xsp_common.cuh"

namespace xsp {

constexpr uint32_t kPB = XSP_PACK_BLOCK;

// ---- host packer -----------------------------------------------------------
// Byte-width code n values (xsp_bw_col): per block the bytes of its widest value.
// for_base: code value - (the block's least value), the least value in base[].
template <typename T>
void bw_encode(xsp_ctx* ctx, const std::string& tag, const T* v, uint64_t n, xsp_bw_col& out,
               bool for_base = false) {
  const uint64_t nb = (n + kPB - 1) / kPB;
  uint8_t* w = ctx->h<uint8_t>(tag + ".w", nb + 1);
  uint64_t* off = ctx->h<uint64_t>(tag + ".o", nb + 1);
  uint64_t* fb = for_base ? ctx->h<uint64_t>(tag + ".b", nb + 1) : nullptr;
  auto val = [&](uint64_t b, uint64_t i) { return (uint64_t)v[i] - (fb ? fb[b] : 0); };
  uint64_t total = 0;
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t r0 = b * kPB, r1 = std::min(n, r0 + kPB);
    if (fb) {
      uint64_t lo = ~0ull;
      for (uint64_t i = r0; i < r1; ++i) lo = std::min(lo, (uint64_t)v[i]);
      fb[b] = lo;
    }
    uint64_t m = 0;
    for (uint64_t i = r0; i < r1; ++i) m |= val(b, i);
    w[b] = m ? (uint8_t)((64 - __builtin_clzll(m) + 7) / 8) : 0;
    off[b] = total;
    total += w[b] * (r1 - r0);
  }
  off[nb] = total;
  uint8_t* d = ctx->h<uint8_t>(tag + ".d", total + 8);
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t r0 = b * kPB, r1 = std::min(n, r0 + kPB);
    uint8_t* p = d + off[b];
    const uint32_t wb = w[b];
    for (uint64_t i = r0; i < r1; ++i, p += wb) {
      const uint64_t x = val(b, i);
      std::memcpy(p, &x, wb);  // little-endian host
    }
  }
  out.width = w;
  out.boff = off;
  out.data = d;
  out.base = fb;
}

// Occupancy as u8 / u16 indexes into its distinct values (none if > 65536).
void occ_encode(xsp_ctx* ctx, const double* v, uint64_t n, xsp_packed_cols* out) {
  out->occ_dict_n = 0;
  out->occ_idx_bytes = 0;
  out->occ_dict = nullptr;
  out->occ_idx = nullptr;
  if (!n) return;
  std::unordered_map<uint64_t, uint32_t> ix;
  std::vector<double> dict;
  uint16_t* tmp = ctx->h<uint16_t>("pk.occ.t", n);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t bits;
    std::memcpy(&bits, v + i, 8);
    auto it = ix.find(bits);
    if (it == ix.end()) {
      if (dict.size() == 65536) return;
      it = ix.emplace(bits, (uint32_t)dict.size()).first;
      dict.push_back(v[i]);
    }
    tmp[i] = (uint16_t)it->second;
  }
  const uint32_t ib = dict.size() <= 256 ? 1 : 2;
  uint8_t* idx = ctx->h<uint8_t>("pk.occ.i", n * ib + 8);
  if (ib == 1)
    for (uint64_t i = 0; i < n; ++i) idx[i] = (uint8_t)tmp[i];
  else
    std::memcpy(idx, tmp, n * 2);
  double* d = ctx->h<double>("pk.occ.d", dict.size());
  std::memcpy(d, dict.data(), dict.size() * 8);
  out->occ_dict_n = (uint32_t)dict.size();
  out->occ_idx_bytes = ib;
  out->occ_dict = d;
  out->occ_idx = idx;
}

void pack_host(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_traces* tr, xsp_packed_cols* out) {
  const uint64_t n = c->n_spans;
  const uint64_t nb = (n + kPB - 1) / kPB;
  uint64_t ncid = 0, npar = 0;
  for (uint64_t i = 0; i < n; ++i) {
    ncid += (c->flags[i] & XSP_F_CID) != 0;
    npar += (c->flags[i] & XSP_F_PARENT) != 0;
  }
  uint32_t* dbeg = ctx->h<uint32_t>("pk.dbeg", n + 1);
  uint32_t* dur = ctx->h<uint32_t>("pk.dur", n + 1);
  uint32_t* dcid = ctx->h<uint32_t>("pk.dcid", ncid + 1);
  uint64_t* par = ctx->h<uint64_t>("pk.par", npar + 1);
  uint64_t* cbase = ctx->h<uint64_t>("pk.cbase", nb + 1);
  uint32_t* cid0 = ctx->h<uint32_t>("pk.cid0", nb + 1);
  uint32_t* par0 = ctx->h<uint32_t>("pk.par0", nb + 1);
  uint32_t* met0 = ctx->h<uint32_t>("pk.met0", nb + 1);
  uint32_t* lay0 = ctx->h<uint32_t>("pk.lay0", nb + 1);
  uint32_t* cpar0 = ctx->h<uint32_t>("pk.cpar0", nb + 1);
  {
    uint32_t m = 0, l = 0, cp = 0;
    for (uint64_t b = 0; b < nb; ++b) {
      met0[b] = m;
      lay0[b] = l;
      cpar0[b] = cp;
      for (uint64_t i = b * kPB, e = std::min(n, i + kPB); i < e; ++i) {
        const uint8_t f = c->flags[i];
        m += (f & XSP_F_METRICS) != 0;
        const bool lay = (f & 3u) == XSP_LEVEL_LAYER;
        l += lay;
        cp += !lay && (f & XSP_F_PARENT);
      }
    }
    met0[nb] = m;
    lay0[nb] = l;
    cpar0[nb] = cp;
  }
  std::vector<uint64_t> ekey, eval;
  ekey.reserve(nb + tr->n_traces + 1024);
  eval.reserve(nb + tr->n_traces + 1024);
  std::vector<uint8_t> head(n ? n : 1, 0);
  for (uint32_t t = 0; t < tr->n_traces; ++t)
    if (tr->span_off[t] < n) head[tr->span_off[t]] = 1;
  uint64_t ci = 0, pi = 0;
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t r0 = b * kPB, r1 = std::min(n, r0 + kPB);
    uint64_t base = ~0ull;
    for (uint64_t i = r0; i < r1; ++i)
      if (c->flags[i] & XSP_F_CID) base = std::min(base, c->cid[i]);
    cbase[b] = base == ~0ull ? 0 : base;
    cid0[b] = (uint32_t)ci;
    par0[b] = (uint32_t)pi;
    for (uint64_t i = r0; i < r1; ++i) {
      const uint64_t bg = c->begin_ns[i], en = c->end_ns[i];
      // begin: delta from the previous span (a reset at trace / block starts)
      const bool reset = i == r0 || head[i] || bg < c->begin_ns[i - 1] || bg - c->begin_ns[i - 1] >= XSP_PACK_ESC;
      if (reset) {
        dbeg[i] = XSP_PACK_ESC;
        ekey.push_back(i << 2 | 0);
        eval.push_back(bg);
      } else {
        dbeg[i] = (uint32_t)(bg - c->begin_ns[i - 1]);
      }
      if (en < bg || en - bg >= XSP_PACK_ESC) {
        dur[i] = XSP_PACK_ESC;
        ekey.push_back(i << 2 | 1);
        eval.push_back(en);
      } else {
        dur[i] = (uint32_t)(en - bg);
      }
      if (c->flags[i] & XSP_F_CID) {
        const uint64_t d = c->cid[i] - cbase[b];
        if (d >= XSP_PACK_ESC) {
          dcid[ci] = XSP_PACK_ESC;
          ekey.push_back(i << 2 | 2);
          eval.push_back(c->cid[i]);
        } else {
          dcid[ci] = (uint32_t)d;
        }
        ++ci;
      }
      if (c->flags[i] & XSP_F_PARENT) par[pi++] = c->parent_id[i];
    }
  }
  uint64_t* ek = ctx->h<uint64_t>("pk.ekey", ekey.size() + 1);
  uint64_t* ev = ctx->h<uint64_t>("pk.eval", eval.size() + 1);
  std::memcpy(ek, ekey.data(), ekey.size() * 8);
  std::memcpy(ev, eval.data(), eval.size() * 8);
  out->n_spans = n;
  out->flags = c->flags;
  out->name_id = c->name_id;
  out->dbegin = dbeg;
  out->dur = dur;
  out->n_cid = ncid;
  out->dcid = dcid;
  out->n_parent = npar;
  out->parent = par;
  out->n_blocks = nb;
  out->blk_cid_base = cbase;
  out->blk_cid0 = cid0;
  out->blk_par0 = par0;
  out->blk_met0 = met0;
  out->blk_lay0 = lay0;
  out->blk_cpar0 = cpar0;
  out->n_esc = ekey.size();
  out->esc_key = ek;
  out->esc_val = ev;
  xsp_bw_col none{nullptr, nullptr, nullptr, nullptr};
  out->name_bw = out->flops_bw = out->read_bw = out->write_bw = out->alloc_bw = out->type_bw = none;
  out->dbegin_bw = out->dur_bw = out->dcid_bw = out->parent_bw = none;
  out->occ_dict_n = out->occ_idx_bytes = 0;
  out->occ_dict = nullptr;
  out->occ_idx = nullptr;
  const char* e = std::getenv("XSP_PACK_TABLES");
  if (e && !std::strcmp(e, "0")) return;
  bw_encode(ctx, "pk.name", c->name_id, n, out->name_bw);
  {  // the delta lists + 1 (XSP_PACK_ESC wraps to 0)
    uint32_t* p1 = ctx->h<uint32_t>("pk.p1", std::max(n, ncid) + 1);
    for (uint64_t i = 0; i < n; ++i) p1[i] = dbeg[i] + 1u;
    bw_encode(ctx, "pk.xb", p1, n, out->dbegin_bw);
    for (uint64_t i = 0; i < n; ++i) p1[i] = dur[i] + 1u;
    bw_encode(ctx, "pk.xd", p1, n, out->dur_bw);
    for (uint64_t i = 0; i < ncid; ++i) p1[i] = dcid[i] + 1u;
    bw_encode(ctx, "pk.xc", p1, ncid, out->dcid_bw);
  }
  if (npar) bw_encode(ctx, "pk.xp", par, npar, out->parent_bw, true);
  if (c->n_metric_rows) {
    bw_encode(ctx, "pk.flops", c->flops, c->n_metric_rows, out->flops_bw);
    bw_encode(ctx, "pk.read", c->dram_read, c->n_metric_rows, out->read_bw);
    bw_encode(ctx, "pk.write", c->dram_write, c->n_metric_rows, out->write_bw);
    occ_encode(ctx, c->occupancy, c->n_metric_rows, out);
  }
  if (c->n_layer_rows) {
    bw_encode(ctx, "pk.alloc", c->alloc_bytes, c->n_layer_rows, out->alloc_bw);
    bw_encode(ctx, "pk.type", c->type_id, c->n_layer_rows, out->type_bw);
  }
}

// ---- device unpack -----------------------------------------------------------
__device__ uint64_t esc_lookup(const uint64_t* __restrict__ key, const uint64_t* __restrict__ val, uint32_t n,
                               uint64_t k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (key[mid] < k) lo = mid + 1; else hi = mid;
  }
  return val[lo < n ? lo : n - 1];
}

struct UnpackArgs {
  uint64_t s0, s1;             // the chunk's global rows
  uint64_t b0;                 // its first global block
  const uint8_t* flags;        // chunk-local (already on the device)
  const uint32_t* dbegin;      // chunk-local
  const uint32_t* dur;         // chunk-local
  const uint32_t* dcid;        // chunk-local list (entries from the chunk's first cid span)
  const uint64_t* parent;      // chunk-local list
  const uint64_t* cbase;       // blocks b0 ..
  const uint32_t* cid0;        // blocks b0 .. (global counts)
  const uint32_t* par0;
  uint64_t cid_first, par_first;  // global list index of the chunk's first entries
  const uint64_t* esc_key;     // the chunk's escapes
  const uint64_t* esc_val;
  uint32_t n_esc;
  uint64_t* begin;             // outputs, chunk-local rows
  uint64_t* end;
  uint64_t* cid;
  uint64_t* parent_out;
};

// one CTA (kPB threads) per global block overlapping the chunk
__global__ void __launch_bounds__(kPB) k_unpack(UnpackArgs a) {
  __shared__ uint64_t s_val[kPB / 32];
  __shared__ uint32_t s_rst[kPB / 32];
  __shared__ uint32_t s_cnt[2][kPB / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint64_t b = a.b0 + blockIdx.x;
  const uint64_t row = b * kPB + tid;
  const bool in = row >= a.s0 && row < a.s1;
  const uint64_t r = row - a.s0;
  const uint8_t f = in ? a.flags[r] : 0;
  // begin: segmented inclusive scan of (reset, value) within the block
  uint64_t v = 0;
  bool rst = true;
  if (in) {
    const uint32_t d = a.dbegin[r];
    rst = d == XSP_PACK_ESC;
    v = rst ? esc_lookup(a.esc_key, a.esc_val, a.n_esc, row << 2 | 0) : d;
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t pv = __shfl_up_sync(0xffffffffu, v, o);
    const uint32_t pr = __shfl_up_sync(0xffffffffu, (uint32_t)rst, o);
    if (lane >= (uint32_t)o && !rst) {
      v += pv;
      rst = pr;
    }
  }
  if (lane == 31) {
    s_val[warp] = v;
    s_rst[warp] = rst;
  }
  // sparse-entry ranks within the block
  const uint32_t hc = __ballot_sync(0xffffffffu, (f & XSP_F_CID) != 0);
  const uint32_t hp = __ballot_sync(0xffffffffu, (f & XSP_F_PARENT) != 0);
  if (lane == 0) {
    s_cnt[0][warp] = __popc(hc);
    s_cnt[1][warp] = __popc(hp);
  }
  __syncthreads();
  if (!in) return;
  // carry from the earlier warps of the block, up to the last reset
  if (!rst) {
    for (int w = (int)warp - 1; w >= 0; --w) {
      v += s_val[w];
      if (s_rst[w]) break;
    }
  }
  const uint64_t begin = v;
  a.begin[r] = begin;
  const uint32_t du = a.dur[r];
  a.end[r] = du == XSP_PACK_ESC ? esc_lookup(a.esc_key, a.esc_val, a.n_esc, row << 2 | 1) : begin + du;
  const uint32_t below = (1u << lane) - 1u;
  uint32_t pc = __popc(hc & below), pp = __popc(hp & below);
  for (uint32_t w = 0; w < warp; ++w) {
    pc += s_cnt[0][w];
    pp += s_cnt[1][w];
  }
  const uint64_t bi = b - a.b0;
  // list positions: entries of this chunk before the block (the chunk's first
  // block starts at s0, whose earlier rows are not part of the chunk)
  const uint64_t cbefore = bi == 0 ? 0 : a.cid0[bi] - a.cid_first;
  const uint64_t pbefore = bi == 0 ? 0 : a.par0[bi] - a.par_first;
  if (f & XSP_F_CID) {
    const uint64_t j = cbefore + pc;
    const uint32_t dc = a.dcid[j];
    a.cid[r] = dc == XSP_PACK_ESC ? esc_lookup(a.esc_key, a.esc_val, a.n_esc, row << 2 | 2) : a.cbase[bi] + dc;
  } else {
    a.cid[r] = 0;
  }
  a.parent_out[r] = (f & XSP_F_PARENT) ? a.parent[pbefore + pp] : 0;
}


// ---- coded name / table columns ----------------------------------------------
struct BwDev {
  const uint8_t* width;  // blocks b0 ..
  const uint64_t* boff;  // blocks b0 .. (global byte offsets)
  const uint8_t* data;   // the staged bytes from global offset `base`
  uint64_t base;
  uint64_t r0, n, b0;    // global first row, rows, first block
  const uint64_t* fbase;  // blocks b0 .. frame of reference, or null
  void* out;
  uint32_t osz;          // 4 or 8
  uint32_t sub1;         // decode to value - 1 (mod 2^32): the +1-coded delta lists
};
constexpr int kTabCols = 6;  // name_id + the metric / layer tables, or the four delta / sparse lists
struct TabUnpackArgs {
  BwDev c[kTabCols];
  uint32_t ncols;
  uint32_t idx_bytes;
  const double* dict;
  const uint8_t* idx;
  uint64_t n_occ;        // 0: no occupancy decode
  double* occ;
  uint64_t max_n;
};

// blockIdx.y < ncols: byte-width column y; == ncols: the occupancy dictionary
__global__ void k_unpack_tables(TabUnpackArgs a) {
  const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t y = blockIdx.y;
  if (y < a.ncols) {
    const BwDev& c = a.c[y];
    if (v >= c.n) return;
    const uint64_t row = c.r0 + v;
    const uint64_t b = row / kPB - c.b0;
    const uint32_t w = c.width[b];
    const uint8_t* p = c.data + (c.boff[b] - c.base) + (row % kPB) * w;
    uint64_t x = c.fbase ? c.fbase[b] : 0;
    uint64_t y = 0;
    for (uint32_t k = 0; k < w; ++k) y |= (uint64_t)p[k] << (8 * k);
    x += y;
    if (c.osz == 8)
      static_cast<uint64_t*>(c.out)[v] = x;
    else
      static_cast<uint32_t*>(c.out)[v] = (uint32_t)x - c.sub1;
  } else {
    if (v >= a.n_occ) return;
    const uint32_t k = a.idx_bytes == 1 ? a.idx[v] : (uint32_t)a.idx[2 * v] | (uint32_t)a.idx[2 * v + 1] << 8;
    a.occ[v] = a.dict[k];
  }
}

void launch_unpack_tables(xsp_ctx* ctx, const void* args, cudaStream_t st) {
  const TabUnpackArgs& a = *static_cast<const TabUnpackArgs*>(args);
  const uint32_t ny = a.ncols + (a.n_occ ? 1 : 0);
  if (!ny || !a.max_n) return;
  k_unpack_tables<<<dim3((unsigned)((a.max_n + 255) / 256), ny), 256, 0, st>>>(a);
  ++ctx->launches;
}

size_t unpack_tables_args_bytes() { return sizeof(TabUnpackArgs); }

// Stage rows [r0, r1) of a coded column (its covering blocks) and append its
// decode to `a`; a column without a width array goes raw (`raw`, esz bytes per row).
uint64_t stage_bw(xsp_ctx* ctx, TabUnpackArgs& a, const std::string& tag, const xsp_bw_col& bw, const void* raw,
                  uint32_t esz, uint64_t r0, uint64_t r1, void* out, cudaStream_t st, uint32_t sub1 = 0) {
  const uint64_t n = r1 - r0;
  if (!n) return 0;
  uint64_t bytes = 0;
  auto h2d = [&](void* d, const void* h, uint64_t nbytes) {
    if (!nbytes) return;
    XSP_CUDA(cudaMemcpyAsync(d, h, nbytes, cudaMemcpyHostToDevice, st));
    bytes += nbytes;
  };
  if (!bw.width) {
    h2d(out, static_cast<const char*>(raw) + r0 * esz, n * esz);
    return bytes;
  }
  if (a.ncols == (uint32_t)kTabCols) throw std::logic_error("TabUnpackArgs: too many coded columns");
  const uint64_t b0 = r0 / kPB, b1 = (r1 + kPB - 1) / kPB, nbk = b1 - b0;
  const uint64_t d0 = bw.boff[b0], d1 = bw.boff[b1];
  uint8_t* dw = ctx->d<uint8_t>(tag + ".w", nbk);
  uint64_t* doff = ctx->d<uint64_t>(tag + ".o", nbk);
  uint8_t* dd = ctx->d<uint8_t>(tag + ".d", d1 - d0 + 8);
  h2d(dw, bw.width + b0, nbk);
  h2d(doff, bw.boff + b0, nbk * 8);
  h2d(dd, bw.data + d0, d1 - d0);
  uint64_t* dfb = nullptr;
  if (bw.base) {
    dfb = ctx->d<uint64_t>(tag + ".b", nbk);
    h2d(dfb, bw.base + b0, nbk * 8);
  }
  BwDev& c = a.c[a.ncols++];
  c.fbase = dfb;
  c.width = dw;
  c.boff = doff;
  c.data = dd;
  c.base = d0;
  c.r0 = r0;
  c.n = n;
  c.b0 = b0;
  c.out = out;
  c.osz = esz;
  c.sub1 = sub1;
  a.max_n = std::max(a.max_n, n);
  return bytes;
}

void launch_unpack(xsp_ctx* ctx, const void* args, cudaStream_t st) {
  launch_unpack_tables(ctx, args, st);  // the coded delta lists first
  const UnpackArgs& a = *reinterpret_cast<const UnpackArgs*>(static_cast<const char*>(args) + sizeof(TabUnpackArgs));
  const uint64_t nbk = (a.s1 + kPB - 1) / kPB - a.b0;
  if (a.s1 > a.s0) {
    k_unpack<<<(unsigned)nbk, kPB, 0, st>>>(a);
    ++ctx->launches;
  }
}

size_t unpack_args_bytes() { return sizeof(TabUnpackArgs) + sizeof(UnpackArgs); }

// Stages rows [s0, s1) of a packed batch on stream st into the device columns
// of `dst` (begin / end / cid / parent_id rebuilt; flags and name_id copied),
// using `tag`-named staging buffers. Returns the H2D bytes issued. With
// `deferred` the unpack kernel is not launched: its arguments are stored there
// for launch_unpack on the stream that consumes the columns (so the copy
// stream carries copies only and never waits for SMs).
uint64_t stage_packed(xsp_ctx* ctx, const xsp_packed_cols* pk, uint64_t s0, uint64_t s1, uint8_t* flags,
                      uint32_t* name_id, uint64_t* begin, uint64_t* end, uint64_t* cid, uint64_t* parent,
                      const std::string& tag, cudaStream_t st, void* deferred) {
  const uint64_t ns = s1 - s0;
  if (!ns) return 0;
  uint64_t bytes = 0;
  auto h2d = [&](void* d, const void* h, uint64_t nbytes) {
    if (!nbytes) return;
    XSP_CUDA(cudaMemcpyAsync(d, h, nbytes, cudaMemcpyHostToDevice, st));
    bytes += nbytes;
  };
  const uint64_t b0 = s0 / kPB, b1 = (s1 + kPB - 1) / kPB, nbk = b1 - b0;
  // global list positions of the chunk's first / past-the-end sparse entries
  auto rank = [&](const uint32_t* blk0, uint8_t bit, uint64_t s) -> uint64_t {
    if (s >= pk->n_spans) return bit == XSP_F_CID ? pk->n_cid : pk->n_parent;
    const uint64_t b = s / kPB;
    uint64_t k = blk0[b];
    for (uint64_t i = b * kPB; i < s; ++i) k += (pk->flags[i] & bit) != 0;
    return k;
  };
  const uint64_t c0 = rank(pk->blk_cid0, XSP_F_CID, s0), c1 = rank(pk->blk_cid0, XSP_F_CID, s1);
  const uint64_t p0 = rank(pk->blk_par0, XSP_F_PARENT, s0), p1 = rank(pk->blk_par0, XSP_F_PARENT, s1);
  const uint64_t* e0 = std::lower_bound(pk->esc_key, pk->esc_key + pk->n_esc, s0 << 2);
  const uint64_t* e1 = std::lower_bound(pk->esc_key, pk->esc_key + pk->n_esc, s1 << 2);
  const uint64_t ne = e1 - e0;
  uint32_t* d_dbeg = ctx->d<uint32_t>(tag + "pk.dbeg", ns);
  uint32_t* d_dur = ctx->d<uint32_t>(tag + "pk.dur", ns);
  uint32_t* d_dcid = ctx->d<uint32_t>(tag + "pk.dcid", c1 - c0 + 1);
  uint64_t* d_par = ctx->d<uint64_t>(tag + "pk.par", p1 - p0 + 1);
  uint64_t* d_cb = ctx->d<uint64_t>(tag + "pk.cb", nbk + 1);
  uint32_t* d_c0 = ctx->d<uint32_t>(tag + "pk.c0", nbk + 1);
  uint32_t* d_p0 = ctx->d<uint32_t>(tag + "pk.p0", nbk + 1);
  uint64_t* d_ek = ctx->d<uint64_t>(tag + "pk.ek", ne + 1);
  uint64_t* d_ev = ctx->d<uint64_t>(tag + "pk.ev", ne + 1);
  h2d(flags, pk->flags + s0, ns);
  if (!pk->name_bw.width) h2d(name_id, pk->name_id + s0, ns * 4);  // else stage_tables_packed
  // the u32 delta lists, byte-width coded (+1) or raw; decoded by k_unpack_tables
  // into d_dbeg / d_dur / d_dcid before k_unpack reads them
  TabUnpackArgs pre;
  std::memset(&pre, 0, sizeof(pre));
  bytes += stage_bw(ctx, pre, tag + "pk.xb", pk->dbegin_bw, pk->dbegin, 4, s0, s1, d_dbeg, st, 1);
  bytes += stage_bw(ctx, pre, tag + "pk.xd", pk->dur_bw, pk->dur, 4, s0, s1, d_dur, st, 1);
  bytes += stage_bw(ctx, pre, tag + "pk.xc", pk->dcid_bw, pk->dcid, 4, c0, c1, d_dcid, st, 1);
  bytes += stage_bw(ctx, pre, tag + "pk.xp", pk->parent_bw, pk->parent, 8, p0, p1, d_par, st);
  h2d(d_cb, pk->blk_cid_base + b0, nbk * 8);
  h2d(d_c0, pk->blk_cid0 + b0, nbk * 4);
  h2d(d_p0, pk->blk_par0 + b0, nbk * 4);
  h2d(d_ek, e0, ne * 8);
  h2d(d_ev, pk->esc_val + (e0 - pk->esc_key), ne * 8);
  UnpackArgs a;
  a.s0 = s0;
  a.s1 = s1;
  a.b0 = b0;
  a.flags = flags;
  a.dbegin = d_dbeg;
  a.dur = d_dur;
  a.dcid = d_dcid;
  a.parent = d_par;
  a.cbase = d_cb;
  a.cid0 = d_c0;
  a.par0 = d_p0;
  a.cid_first = c0;
  a.par_first = p0;
  a.esc_key = d_ek;
  a.esc_val = d_ev;
  a.n_esc = (uint32_t)ne;
  a.begin = begin;
  a.end = end;
  a.cid = cid;
  a.parent_out = parent;
  if (deferred) {  // [TabUnpackArgs pre][UnpackArgs a]: launch_unpack runs both in order
    std::memcpy(deferred, &pre, sizeof(pre));
    std::memcpy(static_cast<char*>(deferred) + sizeof(pre), &a, sizeof(a));
  } else {
    launch_unpack_tables(ctx, &pre, st);
    k_unpack<<<(unsigned)nbk, kPB, 0, st>>>(a);
    ++ctx->launches;
  }
  return bytes;
}

// Stages name_id rows [s0, s1), metric rows [m0, m1) and layer rows [l0, l1)
// into dst's device columns: coded columns as their covering blocks (decoded
// by k_unpack_tables, deferred like k_unpack when `deferred` is given), the
// others raw. Returns the H2D bytes issued.
uint64_t stage_tables_packed(xsp_ctx* ctx, const xsp_packed_cols* pk, const xsp_span_cols* hc, uint64_t s0,
                             uint64_t s1, uint64_t m0, uint64_t m1, uint64_t l0, uint64_t l1, uint32_t* name_id,
                             uint64_t* flops, uint64_t* rd, uint64_t* wr, double* occ, int64_t* alloc,
                             uint32_t* type_id, const std::string& tag, cudaStream_t st, void* deferred) {
  uint64_t bytes = 0;
  auto h2d = [&](void* d, const void* h, uint64_t nbytes) {
    if (!nbytes) return;
    XSP_CUDA(cudaMemcpyAsync(d, h, nbytes, cudaMemcpyHostToDevice, st));
    bytes += nbytes;
  };
  TabUnpackArgs a;
  std::memset(&a, 0, sizeof(a));
  bytes += stage_bw(ctx, a, tag + "name", pk->name_bw, pk->name_id, 4, s0, s1, name_id, st);
  bytes += stage_bw(ctx, a, tag + "flops", pk->flops_bw, hc->flops, 8, m0, m1, flops, st);
  bytes += stage_bw(ctx, a, tag + "read", pk->read_bw, hc->dram_read, 8, m0, m1, rd, st);
  bytes += stage_bw(ctx, a, tag + "write", pk->write_bw, hc->dram_write, 8, m0, m1, wr, st);
  bytes += stage_bw(ctx, a, tag + "alloc", pk->alloc_bw, hc->alloc_bytes, 8, l0, l1, alloc, st);
  bytes += stage_bw(ctx, a, tag + "type", pk->type_bw, hc->type_id, 4, l0, l1, type_id, st);
  if (m1 > m0) {
    if (pk->occ_dict_n) {
      double* dd = ctx->d<double>(tag + "occ.d", pk->occ_dict_n);
      uint8_t* di = ctx->d<uint8_t>(tag + "occ.i", (m1 - m0) * pk->occ_idx_bytes + 8);
      h2d(dd, pk->occ_dict, pk->occ_dict_n * 8ull);
      h2d(di, pk->occ_idx + m0 * pk->occ_idx_bytes, (m1 - m0) * pk->occ_idx_bytes);
      a.dict = dd;
      a.idx = di;
      a.idx_bytes = pk->occ_idx_bytes;
      a.n_occ = m1 - m0;
      a.occ = occ;
      a.max_n = std::max(a.max_n, m1 - m0);
    } else {
      h2d(occ, hc->occupancy + m0, (m1 - m0) * 8);
    }
  }
  if (deferred)
    std::memcpy(deferred, &a, sizeof(a));
  else
    launch_unpack_tables(ctx, &a, st);
  return bytes;
}

}  // namespace xsp
