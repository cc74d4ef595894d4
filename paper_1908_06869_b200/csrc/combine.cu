// Multi-GPU table combine over NCCL (SURVEY §8(b) xsp_combine_nccl, §8(e)).
//
// Trace sharding: every rank correlates + analyses the analysis groups assigned
// to it (independent units, no data-path collective); the finished tables then
// travel once to rank 0, which lays them out in global group order — the
// tables an unsharded run produces. Per column family (per group: status and
// the a15 model row; per kernel: a8/a9; per layer: a11-a14 + top-k; per name:
// a10; per type: a5-a7) rank r ships its rows as one contiguous block:
//
//   1. ncclAllGather of every rank's five row counts (G, L, K, N, Y);
//   2. one NCCL group of ncclSend (rank r -> 0) / ncclRecv (rank 0 <- r) per
//      column and per metadata array (global group ids, the four CSR offset
//      arrays), into staging buffers on rank 0 laid out rank after rank;
//   3. on rank 0 the host builds, per global group, the source block (owner
//      rank's staging base + its local CSR offset) and the output offsets (an
//      exclusive scan of the block sizes), and one gather kernel per family
//      copies every output row from its source row, all columns of the family
//      at once.
//
// Bytes exchanged: exactly the tables (no padding): per rank r != 0,
// sum over columns of rows_r(family) * element size, plus 4 B per group and
// 16 B per group of CSR offsets. The layer tables' l_row (span rows) are
// rebased to global rows by the sender (l_row_map).
#include <dlfcn.h>

#include <cstddef>

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <nccl.h>

#include "ctx.h"
#include "prims.cuh"
#include "xsp_common.cuh"

namespace xsp {

namespace {

// NCCL is resolved at run time (the process may already hold torch's copy of
// libnccl.so.2, which dlopen then returns); libxsp.so has no link-time NCCL
// dependency.
struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static bool loaded = false;
  if (!loaded) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw std::runtime_error("libnccl.so.2 not found (needed for the NCCL table combine)");
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + s);
      return p;
    };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(n.init_rank)>(sym("ncclCommInitRank"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("ncclCommDestroy"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
    n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    loaded = true;
  }
  return n;
}

#define XSP_NCCL(call)                                                                          \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) throw std::runtime_error(std::string(#call) + ": " + nccl().error_string(r_)); \
  } while (0)

enum Fam { FG = 0, FL = 1, FK = 2, FN = 3, FY = 4, NFAM = 5 };

struct Col {
  const char* name;
  int fam;
  int es;  // element bytes (l_topk: 4 * top_k)
  size_t field;  // offsetof in xsp_tables_out
};

#define XSP_COL(n, f, e) {#n, f, e, offsetof(xsp_tables_out, n)}
std::vector<Col> columns(int top_k) {
  return {
      XSP_COL(group_status, FG, 4), XSP_COL(group_err_arg, FG, 4),
      XSP_COL(k_name, FK, 4), XSP_COL(k_layer, FK, 4), XSP_COL(k_lat, FK, 8), XSP_COL(k_flops, FK, 8),
      XSP_COL(k_read, FK, 8), XSP_COL(k_write, FK, 8), XSP_COL(k_occ, FK, 8), XSP_COL(k_ai, FK, 8),
      XSP_COL(k_tput, FK, 8), XSP_COL(k_bound, FK, 1), XSP_COL(k_roofline_in, FK, 1),
      XSP_COL(l_index, FL, 4), XSP_COL(l_row, FL, 4), XSP_COL(l_layer_lat, FL, 8), XSP_COL(l_kern_lat, FL, 8),
      XSP_COL(l_flops, FL, 8), XSP_COL(l_read, FL, 8), XSP_COL(l_write, FL, 8), XSP_COL(l_occ, FL, 8),
      XSP_COL(l_count, FL, 8), XSP_COL(l_ai, FL, 8), XSP_COL(l_tput, FL, 8), XSP_COL(l_bound, FL, 1),
      XSP_COL(l_nongpu, FL, 8), XSP_COL(l_gpu_share, FL, 8), XSP_COL(l_nongpu_share, FL, 8),
      XSP_COL(l_flagged, FL, 1), XSP_COL(l_roofline_in, FL, 1),
      {"l_topk", FL, 4 * (top_k ? top_k : 1), offsetof(xsp_tables_out, l_topk)},
      XSP_COL(n_name, FN, 4), XSP_COL(n_count, FN, 8), XSP_COL(n_lat, FN, 8), XSP_COL(n_pct, FN, 8),
      XSP_COL(n_flops, FN, 8), XSP_COL(n_read, FN, 8), XSP_COL(n_write, FN, 8), XSP_COL(n_occ, FN, 8),
      XSP_COL(n_ai, FN, 8), XSP_COL(n_tput, FN, 8), XSP_COL(n_bound, FN, 1),
      XSP_COL(m_lat, FG, 8), XSP_COL(m_kern_lat, FG, 8), XSP_COL(m_flops, FG, 8), XSP_COL(m_read, FG, 8),
      XSP_COL(m_write, FG, 8), XSP_COL(m_occ, FG, 8), XSP_COL(m_count, FG, 8), XSP_COL(m_ai, FG, 8),
      XSP_COL(m_tput, FG, 8), XSP_COL(m_bound, FG, 1), XSP_COL(m_gpu, FG, 8), XSP_COL(m_gpu_pct, FG, 8),
      XSP_COL(m_throughput, FG, 8), XSP_COL(m_roofline_in, FG, 1),
      XSP_COL(y_type, FY, 4), XSP_COL(y_count, FY, 8), XSP_COL(y_lat, FY, 8), XSP_COL(y_alloc, FY, 8),
  };
}
#undef XSP_COL

template <typename T>
T*& field(xsp_tables_out* t, size_t off) {
  return *reinterpret_cast<T**>(reinterpret_cast<char*>(t) + off);
}

// CSR offset arrays of the row families (G is one row per group)
uint32_t* const* csr_of(const xsp_tables_out* t, int fam) {
  switch (fam) {
    case FL: return &t->group_layer_off;
    case FK: return &t->group_kernel_off;
    case FN: return &t->group_name_off;
    case FY: return &t->group_type_off;
    default: return nullptr;
  }
}

struct GatherCol {
  const char* src;
  char* dst;
  int es;
};

// output row j of a family: its group g (binary search in dst_off), source row
// src_start[g] + (j - dst_off[g]); every column of the family copied
__global__ void k_combine_gather(uint64_t nrows, uint32_t G, const uint64_t* __restrict__ dst_off,
                                 const uint64_t* __restrict__ src_start, const GatherCol* __restrict__ cols,
                                 int ncols) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nrows) return;
  uint32_t lo = 0, hi = G;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (dst_off[mid] <= j) lo = mid; else hi = mid;
  }
  const uint64_t s = src_start[lo] + (j - dst_off[lo]);
  for (int c = 0; c < ncols; ++c) {
    const int es = cols[c].es;
    const char* src = cols[c].src + s * es;
    char* dst = cols[c].dst + j * es;
    if (es == 8) {
      *reinterpret_cast<uint64_t*>(dst) = *reinterpret_cast<const uint64_t*>(src);
    } else if (es == 4) {
      *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(src);
    } else {
      for (int b = 0; b < es; ++b) dst[b] = src[b];
    }
  }
}

__global__ void k_remap_rows(uint32_t* __restrict__ rows, uint64_t n, const uint32_t* __restrict__ map) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rows[i] = map[rows[i]];
}

__global__ void k_csr_from_sizes(const uint64_t* __restrict__ scan, uint32_t G, uint32_t* __restrict__ out) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g <= G) out[g] = (uint32_t)scan[g];
}

}  // namespace

void comm_unique_id(void* id) {
  ncclUniqueId u;
  XSP_NCCL(nccl().get_unique_id(&u));
  std::memcpy(id, &u, sizeof(u));
}

void comm_init(xsp_ctx* ctx, int world, int rank, const void* id) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad world / rank");
  if (ctx->nccl_comm) {
    nccl().destroy(static_cast<ncclComm_t>(ctx->nccl_comm));
    ctx->nccl_comm = nullptr;
  }
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  XSP_CUDA(cudaSetDevice(ctx->device));
  ncclComm_t c;
  XSP_NCCL(nccl().init_rank(&c, world, u, rank));
  ctx->nccl_comm = c;
  ctx->comm_world = world;
  ctx->comm_rank = rank;
  ctx->comm_destroy = [](void* p) { nccl().destroy(static_cast<ncclComm_t>(p)); };
}

void run_combine_tables(xsp_ctx* ctx, xsp_tables_out* local, const uint32_t* group_ids, uint32_t G_local,
                        uint32_t G_total, const uint32_t* l_row_map, int top_k, xsp_tables_out* out,
                        uint64_t* bytes_sent, cudaStream_t st) {
  if (!ctx->nccl_comm) throw std::invalid_argument("xsp_comm_init has not been called on this ctx");
  const Nccl& N = nccl();
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl_comm);
  const int W = ctx->comm_world, me = ctx->comm_rank;
  const std::vector<Col> cols = columns(top_k);
  // ---- local row counts (G, L, K, N, Y)
  uint64_t* hsz = ctx->h<uint64_t>("cb.sizes_h", 8ull * W);
  uint64_t* dsz = ctx->d<uint64_t>("cb.sizes", 8ull * W);
  uint32_t tot[4] = {0, 0, 0, 0};
  if (G_local) {
    XSP_CUDA(cudaMemcpyAsync(tot + 0, local->group_layer_off + G_local, 4, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaMemcpyAsync(tot + 1, local->group_kernel_off + G_local, 4, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaMemcpyAsync(tot + 2, local->group_name_off + G_local, 4, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaMemcpyAsync(tot + 3, local->group_type_off + G_local, 4, cudaMemcpyDeviceToHost, st));
    XSP_CUDA(cudaStreamSynchronize(st));
  }
  uint64_t mine[8] = {G_local, tot[0], tot[1], tot[2], tot[3], 0, 0, 0};
  // the sender rebases its layer rows to global span rows
  if (l_row_map && tot[0]) {
    k_remap_rows<<<ceil_div((uint64_t)tot[0], 256), 256, 0, st>>>(local->l_row, tot[0], l_row_map);
    ++ctx->launches;
  }
  XSP_CUDA(cudaMemcpyAsync(dsz + 8ull * me, mine, 64, cudaMemcpyHostToDevice, st));
  XSP_NCCL(N.all_gather(dsz + 8ull * me, dsz, 8, ncclUint64, comm, st));
  XSP_CUDA(cudaMemcpyAsync(hsz, dsz, 64ull * W, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  // rows per family per rank and the rank prefixes
  std::vector<uint64_t> rows(NFAM * W), pre(NFAM * (W + 1), 0);
  for (int r = 0; r < W; ++r) {
    rows[FG * W + r] = hsz[8 * r + 0];
    rows[FL * W + r] = hsz[8 * r + 1];
    rows[FK * W + r] = hsz[8 * r + 2];
    rows[FN * W + r] = hsz[8 * r + 3];
    rows[FY * W + r] = hsz[8 * r + 4];
  }
  for (int f = 0; f < NFAM; ++f)
    for (int r = 0; r < W; ++r) pre[f * (W + 1) + r + 1] = pre[f * (W + 1) + r] + rows[f * W + r];
  uint64_t sent = 0;
  // ---- staging on rank 0: metadata (group ids, 4 CSR arrays) + every column
  const bool root = me == 0;
  const uint64_t Gsum = pre[FG * (W + 1) + W];
  if (root && Gsum != G_total) throw std::invalid_argument("the ranks' groups do not add up to n_groups_total");
  uint32_t* st_gid = root ? ctx->d<uint32_t>("cb.st_gid", Gsum + 1) : nullptr;
  uint32_t* st_csr[NFAM] = {nullptr};
  for (int f = FL; f < NFAM; ++f)
    if (root) st_csr[f] = ctx->d<uint32_t>(std::string("cb.st_csr") + char('0' + f), Gsum + W + 1);
  std::vector<char*> st_col(cols.size(), nullptr);
  if (root)
    for (size_t c = 0; c < cols.size(); ++c)
      st_col[c] = ctx->d<char>(std::string("cb.st.") + cols[c].name,
                               pre[cols[c].fam * (W + 1) + W] * cols[c].es + 8);
  uint32_t* d_gid = ctx->d<uint32_t>("cb.gid", G_local + 1);
  if (G_local) XSP_CUDA(cudaMemcpyAsync(d_gid, group_ids, G_local * 4ull, cudaMemcpyHostToDevice, st));
  XSP_NCCL(N.group_start());
  for (int r = 0; r < W; ++r) {
    const uint64_t g_r = rows[FG * W + r];
    if (r == me || (!root && r != 0)) continue;
    // metadata
    if (root) {
      if (g_r) XSP_NCCL(N.recv(st_gid + pre[FG * (W + 1) + r], g_r, ncclUint32, r, comm, st));
      for (int f = FL; f < NFAM; ++f)
        XSP_NCCL(N.recv(st_csr[f] + pre[FG * (W + 1) + r] + r, g_r + 1, ncclUint32, r, comm, st));
      for (size_t c = 0; c < cols.size(); ++c) {
        const uint64_t nb = rows[cols[c].fam * W + r] * cols[c].es;
        if (nb) XSP_NCCL(N.recv(st_col[c] + pre[cols[c].fam * (W + 1) + r] * cols[c].es, nb, ncclUint8, r, comm, st));
      }
    }
  }
  if (!root && W > 1) {
    if (G_local) XSP_NCCL(N.send(d_gid, G_local, ncclUint32, 0, comm, st));
    for (int f = FL; f < NFAM; ++f) XSP_NCCL(N.send(*csr_of(local, f), G_local + 1ull, ncclUint32, 0, comm, st));
    sent += 4ull * G_local + 16ull * (G_local + 1);
    for (size_t c = 0; c < cols.size(); ++c) {
      const uint64_t nb = rows[cols[c].fam * W + me] * cols[c].es;
      if (nb) XSP_NCCL(N.send(field<char>(local, cols[c].field), nb, ncclUint8, 0, comm, st));
      sent += nb;
    }
  }
  XSP_NCCL(N.group_end());
  if (bytes_sent) *bytes_sent = sent;
  if (!root) {
    XSP_CUDA(cudaStreamSynchronize(st));
    std::memset(out, 0, sizeof(*out));
    return;
  }
  // rank 0's own block: device-to-device into its staging slot
  {
    const uint64_t g0 = rows[FG * W + 0];
    if (g0) XSP_CUDA(cudaMemcpyAsync(st_gid, d_gid, g0 * 4, cudaMemcpyDeviceToDevice, st));
    for (int f = FL; f < NFAM; ++f)
      XSP_CUDA(cudaMemcpyAsync(st_csr[f], *csr_of(local, f), (g0 + 1) * 4, cudaMemcpyDeviceToDevice, st));
    for (size_t c = 0; c < cols.size(); ++c) {
      const uint64_t nb = rows[cols[c].fam * W + 0] * cols[c].es;
      if (nb) XSP_CUDA(cudaMemcpyAsync(st_col[c], field<char>(local, cols[c].field), nb, cudaMemcpyDeviceToDevice, st));
    }
  }
  // ---- block table on the host (G_total groups: small)
  uint32_t* h_gid = ctx->h<uint32_t>("cb.gid_h", Gsum + 1);
  uint32_t* h_csr = ctx->h<uint32_t>("cb.csr_h", (NFAM - 1) * (Gsum + W + 1));
  if (Gsum) XSP_CUDA(cudaMemcpyAsync(h_gid, st_gid, Gsum * 4, cudaMemcpyDeviceToHost, st));
  for (int f = FL; f < NFAM; ++f)
    XSP_CUDA(cudaMemcpyAsync(h_csr + (f - 1) * (Gsum + W + 1), st_csr[f], (Gsum + W) * 4, cudaMemcpyDeviceToHost, st));
  XSP_CUDA(cudaStreamSynchronize(st));
  std::vector<int> owner(G_total, -1);
  std::vector<uint32_t> lidx(G_total, 0);
  for (int r = 0; r < W; ++r)
    for (uint64_t i = 0; i < rows[FG * W + r]; ++i) {
      const uint32_t g = h_gid[pre[FG * (W + 1) + r] + i];
      if (g >= G_total || owner[g] >= 0) throw std::invalid_argument("global group ids overlap or exceed n_groups_total");
      owner[g] = r;
      lidx[g] = (uint32_t)i;
    }
  for (uint32_t g = 0; g < G_total; ++g)
    if (owner[g] < 0) throw std::invalid_argument("a global group is held by no rank");
  // per family: src_start[g], dst_off[g] (G + 1)
  uint64_t* h_tab = ctx->h<uint64_t>("cb.tab_h", NFAM * 2ull * (G_total + 1));
  for (int f = 0; f < NFAM; ++f) {
    uint64_t* src = h_tab + f * 2ull * (G_total + 1);
    uint64_t* dst = src + G_total + 1;
    uint64_t run = 0;
    for (uint32_t g = 0; g < G_total; ++g) {
      const int r = owner[g];
      const uint32_t i = lidx[g];
      uint64_t b = i, n = 1;
      if (f != FG) {
        const uint32_t* o = h_csr + (f - 1) * (Gsum + W + 1) + pre[FG * (W + 1) + r] + r;
        b = o[i];
        n = o[i + 1] - o[i];
      }
      src[g] = pre[f * (W + 1) + r] + b;
      dst[g] = run;
      run += n;
    }
    dst[G_total] = run;
  }
  uint64_t* d_tab = ctx->d<uint64_t>("cb.tab", NFAM * 2ull * (G_total + 1));
  XSP_CUDA(cudaMemcpyAsync(d_tab, h_tab, NFAM * 2ull * (G_total + 1) * 8, cudaMemcpyHostToDevice, st));
  // ---- outputs on rank 0
  std::memset(out, 0, sizeof(*out));
  out->n_groups = G_total;
  uint64_t fam_rows[NFAM];
  for (int f = 0; f < NFAM; ++f) fam_rows[f] = h_tab[f * 2ull * (G_total + 1) + (G_total + 1) + G_total];
  out->n_layers = fam_rows[FL];
  out->n_kernels = fam_rows[FK];
  out->n_names = fam_rows[FN];
  out->n_type_rows = fam_rows[FY];
  std::vector<GatherCol> gc[NFAM];
  for (size_t c = 0; c < cols.size(); ++c) {
    const int f = cols[c].fam;
    char* dst = ctx->d<char>(std::string("cb.out.") + cols[c].name, fam_rows[f] * cols[c].es + 8);
    field<char>(out, cols[c].field) = dst;
    gc[f].push_back({st_col[c], dst, cols[c].es});
  }
  GatherCol* d_gc = ctx->d<GatherCol>("cb.gc", cols.size());
  GatherCol* h_gc = ctx->h<GatherCol>("cb.gc_h", cols.size());
  size_t k = 0;
  size_t base[NFAM];
  for (int f = 0; f < NFAM; ++f) {
    base[f] = k;
    for (const GatherCol& g : gc[f]) h_gc[k++] = g;
  }
  XSP_CUDA(cudaMemcpyAsync(d_gc, h_gc, k * sizeof(GatherCol), cudaMemcpyHostToDevice, st));
  for (int f = 0; f < NFAM; ++f) {
    const uint64_t n = fam_rows[f];
    if (!n || gc[f].empty()) continue;
    const uint64_t* src = d_tab + f * 2ull * (G_total + 1);
    k_combine_gather<<<ceil_div(n, 256), 256, 0, st>>>(n, G_total, src + G_total + 1, src, d_gc + base[f],
                                                       (int)gc[f].size());
    ++ctx->launches;
  }
  // the four CSR offset arrays
  uint32_t** offs[4] = {&out->group_layer_off, &out->group_kernel_off, &out->group_name_off, &out->group_type_off};
  const int fams[4] = {FL, FK, FN, FY};
  for (int q = 0; q < 4; ++q) {
    uint32_t* o = ctx->d<uint32_t>(std::string("cb.out.off") + char('0' + q), G_total + 1ull);
    k_csr_from_sizes<<<ceil_div((uint64_t)G_total + 1, 256), 256, 0, st>>>(
        d_tab + fams[q] * 2ull * (G_total + 1) + G_total + 1, G_total, o);
    ++ctx->launches;
    *offs[q] = o;
  }
  XSP_CUDA(cudaStreamSynchronize(st));
}

}  // namespace xsp
