// Stage (e): per-kernel, per-layer, per-name and per-model reductions with
// roofline classification and top-k, for every AnalysisInput of a batch.
//
// Reference semantics: combine() (analysis.cpp:102-170), Accumulator and
// attach_roofline (:173-211), a8/a9 (:342-397), a10 (:399-432), a11-a14
// (:437-525), a15/model_roofline (:532-586), a1 throughput (:236-263).
//
// Bit-exactness: this file is compiled with -fmad=false, and every fp64
// expression keeps the reference's operation sequence (flops / (lat / 1e9),
// a / b * 100, sums accumulated left to right in tree order). Integer counters
// are u64 sums (exact). Sequential fp64 chains (the Accumulator) are evaluated
// by one thread per subject in tree order, as the reference does.

#include <algorithm>
#include <functional>
#include <vector>

#include "ctx.h"
#include "prims.cuh"

namespace xsp {

constexpr int kMaxRuns = 64;

// trimmed_mean (analysis.cpp:28-39): sort, drop floor(f*n) each end, ordered sum.
__device__ double trimmed_mean_dev(double* v, uint32_t n, double f) {
  for (uint32_t i = 1; i < n; ++i) {
    double x = v[i];
    uint32_t j = i;
    while (j > 0 && v[j - 1] > x) {
      v[j] = v[j - 1];
      --j;
    }
    v[j] = x;
  }
  uint32_t drop = (uint32_t)floor(f * (double)n);
  double s = 0.0;
  for (uint32_t i = drop; i < n - drop; ++i) s = __dadd_rn(s, v[i]);
  return s / (double)(n - 2 * drop);
}

// Register-resident bitonic sorting networks (all indices compile-time after
// unrolling, so the values stay in registers).
template <int N, typename T>
__device__ __forceinline__ void bitonic_sort(T (&v)[N]) {
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const T a = v[i], b = v[l];
          const bool up = (i & k) == 0;
          const bool sw = up ? (b < a) : (a < b);
          v[i] = sw ? b : a;
          v[l] = sw ? a : b;
        }
      }
    }
  }
}

// trimmed_mean over n <= N doubles produced by load(r): the n values padded
// with +inf are sorted (skipped when they already are, e.g. all equal), then the
// kept middle is summed in ascending order as the reference does.
template <int N, typename Load>
__device__ __forceinline__ double trimmed_mean_net(Load load, uint32_t n, double f) {
  double v[N];
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = (uint32_t)i < n ? load((uint32_t)i) : __longlong_as_double(0x7ff0000000000000ll);
  bool sorted = true;
#pragma unroll
  for (int i = 1; i < N; ++i) sorted &= !(v[i] < v[i - 1]);
  if (!sorted) bitonic_sort<N>(v);
  const uint32_t drop = (uint32_t)floor(f * (double)n);
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if ((uint32_t)i >= drop && (uint32_t)i < n - drop) s = __dadd_rn(s, v[i]);
  return s / (double)(n - 2 * drop);
}

template <typename Load>
__device__ __forceinline__ double trimmed_mean_any(Load load, uint32_t n, double f) {
  if (n == 1) return load(0);  // one run: nothing is trimmed, the mean is the sample
  if (n <= 8) return trimmed_mean_net<8>(load, n, f);
  if (n <= 16) return trimmed_mean_net<16>(load, n, f);
  if (n <= 32) return trimmed_mean_net<32>(load, n, f);
  if (n > kMaxRuns)
    return trimmed_mean_select(
        [&](auto fn) {
          for (uint32_t r = 0; r < n; ++r) fn((double)load(r));
        },
        n, f);
  double v[kMaxRuns];
  for (uint32_t r = 0; r < n; ++r) v[r] = load(r);
  return trimmed_mean_dev(v, n, f);
}

// Integer samples (durations in ns): when every sample fits in 32 bits they are
// sorted as u32 and the kept middle is summed exactly in u64. The reference sums
// the same values as doubles in ascending order; every partial sum is an integer
// below 2^53, so each of its additions is exact and both give the same double.
template <int N, typename Load>
__device__ __forceinline__ bool trimmed_mean_u32(Load load, uint32_t n, double f, double& out) {
  uint32_t v[N];
  uint64_t hi = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const uint64_t x = (uint32_t)i < n ? load((uint32_t)i) : 0xFFFFFFFFull;
    hi |= x >> 32;
    v[i] = (uint32_t)x;
  }
  if (hi) return false;
  bitonic_sort<N>(v);
  const uint32_t drop = (uint32_t)floor(f * (double)n);
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if ((uint32_t)i >= drop && (uint32_t)i < n - drop) s += v[i];
  out = (double)s / (double)(n - 2 * drop);
  return true;
}

template <typename Load>  // load(r) -> uint64_t
__device__ __forceinline__ double trimmed_mean_int(Load load, uint32_t n, double f) {
  double out;
  if (n == 1) return (double)load(0);  // one run (long traces): the sample itself
  if (n <= 8 && trimmed_mean_u32<8>(load, n, f, out)) return out;
  if (n > 8 && n <= 16 && trimmed_mean_u32<16>(load, n, f, out)) return out;
  if (n > 16 && n <= 32 && trimmed_mean_u32<32>(load, n, f, out)) return out;
  return trimmed_mean_any([&](uint32_t r) { return (double)load(r); }, n, f);
}

struct Roof {
  double ai, tput;
  int8_t bound;
};

// arithmetic_intensity / arithmetic_throughput / ideal (analysis.cpp:41-57)
__device__ __forceinline__ Roof roofline(uint64_t flops, uint64_t r, uint64_t w, double lat,
                                         double peak, double bw) {
  Roof o;
  double bytes = __dadd_rn((double)r, (double)w);
  o.ai = bytes <= 0.0 ? nan("") : (double)flops / bytes;
  o.tput = lat > 0.0 ? (double)flops / (lat / 1e9) : nan("");
  o.bound = bytes <= 0.0 ? (int8_t)-1 : (int8_t)(o.ai < peak / bw ? 1 : 0);
  return o;
}

struct GroupArgs {
  uint32_t G;
  const uint32_t* ft;
  const uint32_t* nr;
  const uint32_t* batch;
  const int32_t* t_status;
  const uint32_t* t_layer_off;
  const uint32_t* t_kernel_off;
  const uint32_t* l_koff;
  uint32_t* gl;  // layers of run 0
  uint32_t* gk;  // kernels of run 0
  unsigned long long* gerr;
};

__global__ void k_group_prep(GroupArgs a) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.G) return;
  uint32_t t = a.ft[g];
  a.gerr[g] = ~0ull;
  if (a.nr[g] == 0) {
    a.gl[g] = a.gk[g] = 0;
    return;
  }
  a.gl[g] = a.t_layer_off[t + 1] - a.t_layer_off[t];
  a.gk[g] = a.t_kernel_off[t + 1] - a.t_kernel_off[t];
}

// Structure checks of combine() (analysis.cpp:103-118): first failing run, and
// within it the layer-count check before the per-layer kernel counts.
__global__ void k_group_check_runs(GroupArgs a, uint32_t total_runs, const uint32_t* __restrict__ run_off) {
  uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= total_runs) return;
  uint32_t lo = 0, hi = a.G;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (run_off[mid] <= q) lo = mid; else hi = mid;
  }
  uint32_t g = lo, r = q - run_off[g];
  uint32_t t = a.ft[g] + r;
  if (a.t_status[t] != XSP_T_OK) {
    atomicMin(a.gerr + g, 0ull);  // trace failure outranks everything
    return;
  }
  uint32_t L = a.t_layer_off[t + 1] - a.t_layer_off[t];
  if (L != a.gl[g]) atomicMin(a.gerr + g, ((unsigned long long)(r + 1) << 32) | 0ull);
}

// One thread per (canonical layer, repetition r >= 1): grid.y = r - 1, so the
// repetitions of a layer are checked in parallel instead of one dependent
// load chain per layer. The least (run, layer) mismatch wins (atomicMin), as
// the reference's loop order reports it (analysis.cpp:107-118).
__global__ void k_group_check_layers(GroupArgs a, uint32_t total_layers, const uint32_t* __restrict__ gl_off) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= total_layers) return;
  uint32_t lo = 0, hi = a.G;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (gl_off[mid] <= q) lo = mid; else hi = mid;
  }
  const uint32_t g = lo, li = q - gl_off[g];
  const uint32_t r = blockIdx.y + 1;
  if (r >= a.nr[g]) return;
  const uint32_t t0 = a.ft[g], t = t0 + r;
  if (a.t_status[t] != XSP_T_OK) return;
  const uint32_t L = a.t_layer_off[t + 1] - a.t_layer_off[t];
  if (L != a.gl[g]) return;
  const uint32_t gl0 = a.t_layer_off[t0] + li;
  const uint32_t k0 = a.l_koff[gl0 + 1] - a.l_koff[gl0];
  const uint32_t glr = a.t_layer_off[t] + li;
  const uint32_t kr = a.l_koff[glr + 1] - a.l_koff[glr];
  if (kr != k0) atomicMin(a.gerr + g, ((unsigned long long)(r + 1) << 32) | (li + 1));
}

__global__ void k_group_status(uint32_t G, const uint32_t* __restrict__ nr,
                               const unsigned long long* __restrict__ gerr, double trim,
                               int32_t* __restrict__ status, uint32_t* __restrict__ err_arg) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  int32_t s = XSP_G_OK;
  uint32_t arg = 0;
  unsigned long long e = gerr[g];
  if (nr[g] == 0) s = XSP_G_NO_RUNS;
  else if (e == 0ull) s = XSP_G_TRACE_FAILED;
  else if (e != ~0ull) {
    uint32_t li = (uint32_t)(e & 0xFFFFFFFFull);
    if (li == 0) s = XSP_G_LAYER_COUNT;
    else {
      s = XSP_G_KERNEL_COUNT;
      arg = li - 1;
    }
  } else if (!(trim >= 0.0 && trim < 0.5)) {
    s = XSP_G_BAD_TRIM;
  }
  status[g] = s;
  err_arg[g] = arg;
}

struct LayerArgs {
  uint32_t G, total_layers, top_k;
  const uint32_t* layer_attr_row;  // layer-table row of each layer (type_id, alloc_bytes)
  const uint32_t* type_id;
  const int64_t* alloc_bytes;
  uint32_t* l_type;    // canonical layer's type (a5 keys)
  uint64_t* l_alloc;   // canonical layer's alloc_bytes (two's complement, a7 sums)
  const uint32_t* gl_off;
  const uint32_t* gk_off;
  const uint32_t* ft;
  const uint32_t* nr;
  const int32_t* gstatus;
  const uint32_t* t_layer_off;
  const uint32_t* t_kernel_off;
  const uint32_t* l_koff;
  const uint64_t* layer_dur;
  const uint32_t* layer_row;
  const uint64_t* kernel_dur;
  const uint32_t* kernel_mrow;
  const uint32_t* kernel_name;
  const double* kernel_occ;
  const uint64_t* m_flops;
  const uint64_t* m_read;
  const uint64_t* m_write;
  const double* m_occ;
  double trim, noise, peak, bw;
  // out: kernels
  uint32_t* k_name;
  uint32_t* k_layer;
  double* k_lat;
  uint64_t* k_flops;
  uint64_t* k_read;
  uint64_t* k_write;
  double* k_occ;
  double* k_ai;
  double* k_tput;
  int8_t* k_bound;
  uint8_t* k_in;
  // out: layers
  uint32_t* l_index;
  uint32_t* l_row;
  double* l_layer_lat;
  double* l_kern_lat;
  uint64_t* l_flops;
  uint64_t* l_read;
  uint64_t* l_write;
  double* l_occ;
  uint64_t* l_count;
  double* l_ai;
  double* l_tput;
  int8_t* l_bound;
  double* l_nongpu;
  double* l_gpu_share;
  double* l_nongpu_share;
  uint8_t* l_flagged;
  uint8_t* l_in;
  uint32_t* l_topk;
  double* l_occw;  // optional (one-run long groups): the layer's raw sum(occ * lat) for the model fold
};

__device__ __forceinline__ uint32_t group_of(const uint32_t* __restrict__ off, uint32_t G, uint32_t q) {
  uint32_t lo = 0, hi = G;  // off[lo] <= q < off[hi]
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= q) lo = mid; else hi = mid;
  }
  return lo;
}

// Per (group, kernel ordinal): combine() over repetitions (analysis.cpp:146-167)
// and the a8 / a9 row (:342-397). One thread per kernel keeps R independent
// gathers in flight.
#ifndef XSP_KK_MINB
#define XSP_KK_MINB 3  // 80 registers, no spills: 3 CTAs of 256 per SM
#endif
__global__ void __launch_bounds__(256, XSP_KK_MINB) k_kernels(LayerArgs a, uint32_t total_kernels) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= total_kernels) return;
  const uint32_t g = group_of(a.gk_off, a.G, q);
  if (a.gstatus[g] != XSP_G_OK) return;
  const uint32_t ord = q - a.gk_off[g];
  const uint32_t R = a.nr[g], t0 = a.ft[g];
  const double klat =
      trimmed_mean_int([&](uint32_t r) { return a.kernel_dur[a.t_kernel_off[t0 + r] + ord]; }, R, a.trim);
  const double kocc = trimmed_mean_any([&](uint32_t r) { return a.kernel_occ[a.t_kernel_off[t0 + r] + ord]; }, R,
                                       a.trim);
  const uint32_t j = a.t_kernel_off[t0] + ord;
  const uint32_t mr0 = a.kernel_mrow[j];
  uint64_t f = 0, rd = 0, wr = 0;
  if (mr0 != kNone) {  // counters from the first repetition (:162-166)
    f = a.m_flops[mr0];
    rd = a.m_read[mr0];
    wr = a.m_write[mr0];
  }
  const Roof ro = roofline(f, rd, wr, klat, a.peak, a.bw);
  a.k_name[q] = a.kernel_name[j];
  a.k_lat[q] = klat;
  a.k_flops[q] = f;
  a.k_read[q] = rd;
  a.k_write[q] = wr;
  a.k_occ[q] = kocc;
  a.k_ai[q] = ro.ai;
  a.k_tput[q] = ro.tput;
  a.k_bound[q] = ro.bound;
  a.k_in[q] = (ro.bound >= 0 && klat > 0.0) ? 1 : 0;  // classify (analysis.cpp:59-71)
}

// Groups of one run each (a long single trace): kernel q's only sample is row
// j = t_kernel_off[ft[g]] + ord and its "trimmed mean" is that sample, so this
// variant carries none of the sorting-network code and its register budget
// (and resident warps) follows the loads alone.
__global__ void __launch_bounds__(256) k_kernels_r1(LayerArgs a, uint32_t total_kernels) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= total_kernels) return;
  const uint32_t g = group_of(a.gk_off, a.G, q);
  if (a.gstatus[g] != XSP_G_OK) return;
  const uint32_t j = a.t_kernel_off[a.ft[g]] + (q - a.gk_off[g]);
  const double klat = (double)a.kernel_dur[j];
  const double kocc = a.kernel_occ[j];
  const uint32_t mr0 = a.kernel_mrow[j];
  uint64_t f = 0, rd = 0, wr = 0;
  if (mr0 != kNone) {  // counters of the (only) repetition (:162-166)
    f = a.m_flops[mr0];
    rd = a.m_read[mr0];
    wr = a.m_write[mr0];
  }
  const Roof ro = roofline(f, rd, wr, klat, a.peak, a.bw);
  a.k_name[q] = a.kernel_name[j];
  a.k_lat[q] = klat;
  a.k_flops[q] = f;
  a.k_read[q] = rd;
  a.k_write[q] = wr;
  a.k_occ[q] = kocc;
  a.k_ai[q] = ro.ai;
  a.k_tput[q] = ro.tput;
  a.k_bound[q] = ro.bound;
  a.k_in[q] = (ro.bound >= 0 && klat > 0.0) ? 1 : 0;  // classify (analysis.cpp:59-71)
}

// a11-a14 row of layer q (group-local index li, correlation layer gl0) from its
// Accumulator (analysis.cpp:173-211, 458-494) and top-k
template <typename TopIdx>
__device__ __forceinline__ void layer_row_out(const LayerArgs& a, uint32_t q, uint32_t li, uint32_t gl0,
                                              double layer_lat, uint32_t nk, double acc_lat, double acc_occw,
                                              uint64_t acc_f, uint64_t acc_r, uint64_t acc_w,
                                              const TopIdx& top_idx, uint32_t ntop) {
  const uint32_t K = a.top_k;
  if (a.l_occw) a.l_occw[q] = acc_occw;
  const uint32_t lo_out = q;
  if (a.layer_attr_row && a.type_id && a.alloc_bytes) {
    const uint32_t ar = a.layer_attr_row[gl0];
    a.l_type[lo_out] = a.type_id[ar];
    a.l_alloc[lo_out] = (uint64_t)a.alloc_bytes[ar];
  } else {  // no layer table: every layer of type 0, no allocations
    a.l_type[lo_out] = 0;
    a.l_alloc[lo_out] = 0;
  }
  const Roof ro = roofline(acc_f, acc_r, acc_w, acc_lat, a.peak, a.bw);
  a.l_index[lo_out] = li;
  a.l_row[lo_out] = a.layer_row[gl0];
  a.l_layer_lat[lo_out] = layer_lat;
  a.l_kern_lat[lo_out] = acc_lat;
  a.l_flops[lo_out] = acc_f;
  a.l_read[lo_out] = acc_r;
  a.l_write[lo_out] = acc_w;
  a.l_occ[lo_out] = acc_lat > 0.0 ? acc_occw / acc_lat : 0.0;
  a.l_count[lo_out] = nk;
  a.l_ai[lo_out] = ro.ai;
  a.l_tput[lo_out] = ro.tput;
  a.l_bound[lo_out] = ro.bound;
  a.l_in[lo_out] = (ro.bound >= 0 && acc_lat > 0.0) ? 1 : 0;
  // a13 (analysis.cpp:484-494)
  const double nongpu = __dsub_rn(layer_lat, acc_lat);
  a.l_nongpu[lo_out] = nongpu;
  a.l_gpu_share[lo_out] = layer_lat > 0.0 ? acc_lat / layer_lat : 0.0;
  a.l_nongpu_share[lo_out] = layer_lat > 0.0 ? nongpu / layer_lat : 0.0;
  a.l_flagged[lo_out] = nongpu < -(__dmul_rn(a.noise, layer_lat)) ? 1 : 0;
  for (uint32_t s = 0; s < K; ++s) a.l_topk[(uint64_t)lo_out * K + s] = s < ntop ? top_idx[s] : kNone;
}

// top-k (K <= 4) in registers: the same insertion as topk_push (latency desc,
// ties in arrival order) without a dynamically indexed local array
struct TopK4 {
  double l0 = 0, l1 = 0, l2 = 0, l3 = 0;
  uint32_t i0 = 0, i1 = 0, i2 = 0, i3 = 0, n = 0;
  __device__ __forceinline__ void push(uint32_t K, double klat, uint32_t ord) {
    if (!K) return;
    const uint32_t pos = (n > 0 && l0 >= klat) + (n > 1 && l1 >= klat) + (n > 2 && l2 >= klat) +
                         (n > 3 && l3 >= klat);
    if (pos >= K) return;
    if (pos <= 2 && K > 3) { l3 = l2; i3 = i2; }
    if (pos <= 1 && K > 2) { l2 = l1; i2 = i1; }
    if (pos == 0 && K > 1) { l1 = l0; i1 = i0; }
    if (pos == 0) { l0 = klat; i0 = ord; }
    else if (pos == 1) { l1 = klat; i1 = ord; }
    else if (pos == 2) { l2 = klat; i2 = ord; }
    else { l3 = klat; i3 = ord; }
    if (n < K) ++n;
  }
  __device__ __forceinline__ uint32_t operator[](uint32_t s) const {
    return s == 0 ? i0 : s == 1 ? i1 : s == 2 ? i2 : i3;
  }
};

// top-k insertion: latency desc, ordinal asc
__device__ __forceinline__ void topk_push(uint32_t K, double klat, uint32_t ord, uint32_t* top_idx, double* top_lat,
                                          uint32_t& ntop) {
  if (!K) return;
  uint32_t pos = ntop;
  while (pos > 0 && top_lat[pos - 1] < klat) --pos;
  if (pos < K) {
    const uint32_t last = ntop < K ? ntop : K - 1;
    for (uint32_t s = last; s > pos; --s) {
      top_lat[s] = top_lat[s - 1];
      top_idx[s] = top_idx[s - 1];
    }
    top_lat[pos] = klat;
    top_idx[pos] = ord;
    if (ntop < K) ++ntop;
  }
}

// Per (group, layer): combine() layer latency (:135-144), the Accumulator over
// the layer's kernels in tree order (:173-211), a11-a14 rows and top-k.
// kOneRun: every group has one run (a long single trace), so the layer latency
// is its only sample and the trimmed-mean code is not instantiated.
template <bool kOneRun>
#ifndef XSP_LAYERS_R1_MINB
#define XSP_LAYERS_R1_MINB 4
#endif
__global__ void __launch_bounds__(256, kOneRun ? XSP_LAYERS_R1_MINB : 3) k_layers(LayerArgs a) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= a.total_layers) return;
  const uint32_t g = group_of(a.gl_off, a.G, q);
  const uint32_t li = q - a.gl_off[g];
  if (a.gstatus[g] != XSP_G_OK) return;
  const uint32_t R = a.nr[g], t0 = a.ft[g];
  double layer_lat;
  if constexpr (kOneRun)
    layer_lat = (double)a.layer_dur[a.t_layer_off[t0] + li];
  else
    layer_lat = trimmed_mean_int([&](uint32_t r) { return a.layer_dur[a.t_layer_off[t0 + r] + li]; }, R, a.trim);

  const uint32_t gl0 = a.t_layer_off[t0] + li;
  const uint32_t trace_kbase = a.t_kernel_off[t0];
  const uint32_t kb = a.gk_off[g] + (a.l_koff[gl0] - trace_kbase);
  const uint32_t ke = a.gk_off[g] + (a.l_koff[gl0 + 1] - trace_kbase);
  double acc_lat = 0.0, acc_occw = 0.0;
  uint64_t acc_f = 0, acc_r = 0, acc_w = 0;
  const uint32_t K = a.top_k;
  auto fold = [&](auto&& push) {
    for (uint32_t x = kb; x < ke; ++x) {
      const double klat = a.k_lat[x], kocc = a.k_occ[x];
      const uint64_t f = a.k_flops[x], rd = a.k_read[x], wr = a.k_write[x];
      a.k_layer[x] = li;
      acc_lat = __dadd_rn(acc_lat, klat);
      acc_f += f;
      acc_r += rd;
      acc_w += wr;
      acc_occw = __dadd_rn(acc_occw, __dmul_rn(kocc, klat));
      push(klat, x - a.gk_off[g]);
    }
  };
  if (K <= 4) {  // the usual top-3: registers only
    TopK4 t;
    fold([&](double l, uint32_t o) { t.push(K, l, o); });
    layer_row_out(a, q, li, gl0, layer_lat, ke - kb, acc_lat, acc_occw, acc_f, acc_r, acc_w, t, t.n);
  } else {
    uint32_t top_idx[8];
    double top_lat[8];
    uint32_t ntop = 0;
    fold([&](double l, uint32_t o) { topk_push(K, l, o, top_idx, top_lat, ntop); });
    layer_row_out(a, q, li, gl0, layer_lat, ke - kb, acc_lat, acc_occw, acc_f, acc_r, acc_w, top_idx, ntop);
  }
}

struct ModelArgs {
  uint32_t G;
  const uint32_t* gl_off;
  const uint32_t* gk_off;
  const uint32_t* ft;
  const uint32_t* nr;
  const uint32_t* batch;
  const int32_t* gstatus;
  const uint32_t* model_row;
  const uint64_t* begin;
  const uint64_t* end;
  const double* k_lat;
  const double* k_occ;
  const uint64_t* k_flops;
  const uint64_t* k_read;
  const uint64_t* k_write;
  const double* l_kern_lat;
  // long groups (> kBigGroup kernels or layers): chunk partials (k_big_chunks)
  const uint32_t* gkc_off;  // [G + 1] kernel chunks of each group (empty range: not chunked)
  const uint32_t* glc_off;  // [G + 1] layer chunks of each group
  bool layer_sums;          // one-run groups: the layer chunks carry the kernel sums
  const double* pk_lat;     // per kernel chunk: sum of latencies
  const double* pk_occw;    // per kernel chunk: sum of occ * lat
  const uint64_t* pk_cnt;   // per kernel chunk: sums of flops, read, write
  const double* pl_gpu;     // per layer chunk: sum of layer kernel latencies
  double trim, peak, bw;
  double* m_lat;
  double* m_kern_lat;
  uint64_t* m_flops;
  uint64_t* m_read;
  uint64_t* m_write;
  double* m_occ;
  uint64_t* m_count;
  double* m_ai;
  double* m_tput;
  int8_t* m_bound;
  double* m_gpu;
  double* m_gpu_pct;
  double* m_throughput;
  uint8_t* m_in;
};

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// model_aggregate_row (analysis.cpp:532-552), a13 totals (:495-499), a1 (:245-246).
// One 2-warp CTA per group. Warp 0 runs the kernel chains (latency and
// occupancy x latency) strictly left to right through register broadcast, with
// loads issued kModelPrefetch chunks of 32 rows ahead so the chain does not wait
// on memory; warp 1 sums the u64 counters (any order: exact), runs the layer
// chain (a13 GPU latency) and the model latency.
constexpr int kModelPrefetch = 4;

// strictly ordered fp64 fold of `v` over rows [b, e) (and of occ*v when kOcc)
template <bool kOcc>
__device__ __forceinline__ void chain_fold(const double* __restrict__ v, const double* __restrict__ occ,
                                           uint32_t b, uint32_t e, uint32_t lane, double& s, double& so) {
  double x[kModelPrefetch], o[kModelPrefetch];
#pragma unroll
  for (int d = 0; d < kModelPrefetch; ++d) {
    const uint32_t i = b + 32 * d + lane;
    x[d] = i < e ? v[i] : 0.0;
    o[d] = (kOcc && i < e) ? occ[i] : 0.0;
  }
  for (uint32_t base = b; base < e; base += 32 * kModelPrefetch) {
#pragma unroll
    for (int d = 0; d < kModelPrefetch; ++d) {
      const uint32_t cb = base + 32 * d;
      if (cb >= e) break;
      const double xv = x[d], pr = __dmul_rn(o[d], x[d]);
      const uint32_t i = cb + 32 * kModelPrefetch + lane;
      x[d] = i < e ? v[i] : 0.0;
      o[d] = (kOcc && i < e) ? occ[i] : 0.0;
      const uint32_t cnt = min(32u, e - cb);
      if (cnt == 32) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          s = __dadd_rn(s, __shfl_sync(0xffffffffu, xv, q));
          if (kOcc) so = __dadd_rn(so, __shfl_sync(0xffffffffu, pr, q));
        }
      } else {
        for (uint32_t q = 0; q < cnt; ++q) {
          s = __dadd_rn(s, __shfl_sync(0xffffffffu, xv, q));
          if (kOcc) so = __dadd_rn(so, __shfl_sync(0xffffffffu, pr, q));
        }
      }
    }
  }
}

// a15 model latency (trimmed mean over the runs' model spans, analysis.cpp:
// 154-157): one warp per group, launched before the per-kernel pass so the a10
// and a15 passes that divide by it can run concurrently. Lane r loads run r's
// model span; every lane then runs the same trimmed mean over the shuffled
// values (warp-uniform, no idle lanes).
__global__ void k_model_lat(ModelArgs a) {
  const uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
  if (g >= a.G) return;
  if (a.gstatus[g] != XSP_G_OK) {
    if (lane == 0) a.m_lat[g] = nan("");
    return;
  }
  const uint32_t R = a.nr[g], t0 = a.ft[g];
  uint64_t mdur = 0;
  if (lane < R) {
    const uint32_t m = a.model_row[t0 + lane];
    mdur = clamp_dur(a.begin[m], a.end[m]);
  }
  uint64_t mdur_hi = 0;  // runs 32..63
  if (R > 32 && lane + 32 < R) {
    const uint32_t m = a.model_row[t0 + 32 + lane];
    mdur_hi = clamp_dur(a.begin[m], a.end[m]);
  }
  const double mlat = trimmed_mean_int(
      [&](uint32_t r) {
        const uint64_t lo = __shfl_sync(0xffffffffu, mdur, r & 31u);
        const uint64_t hi = __shfl_sync(0xffffffffu, mdur_hi, r & 31u);
        if (r >= 64) {  // more than 64 runs: the rest straight from the model spans
          const uint32_t m = a.model_row[t0 + r];
          return clamp_dur(a.begin[m], a.end[m]);
        }
        return r < 32 ? lo : hi;
      },
      R, a.trim);
  if (lane == 0) a.m_lat[g] = mlat;
}

__global__ void __launch_bounds__(64) k_models(ModelArgs a) {
  __shared__ double s_gpu;
  __shared__ unsigned long long s_cnt[3];
  const uint32_t g = blockIdx.x;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  if (g >= a.G) return;
  if (a.gstatus[g] != XSP_G_OK) return;  // m_lat = NaN (k_model_lat)
  const uint32_t k0 = a.gk_off[g], k1 = a.gk_off[g + 1];
  const bool big_k = a.gkc_off && a.gkc_off[g + 1] > a.gkc_off[g];
  const bool big_l = a.glc_off && a.glc_off[g + 1] > a.glc_off[g];
  // kernel sums of a one-run long group come from its layer chunks (layer_sums)
  const uint32_t kc0 = a.layer_sums ? a.glc_off[g] : (big_k ? a.gkc_off[g] : 0);
  const uint32_t kc1 = a.layer_sums ? a.glc_off[g + 1] : (big_k ? a.gkc_off[g + 1] : 0);
  double lat = 0.0, occw = 0.0;
  if (warp == 1) {
    // u64 counters: any order is exact
    uint64_t f = 0, rd = 0, wr = 0;
    if (big_k) {
      for (uint32_t c = kc0 + lane; c < kc1; c += 32) {
        f += a.pk_cnt[3 * c];
        rd += a.pk_cnt[3 * c + 1];
        wr += a.pk_cnt[3 * c + 2];
      }
    } else {
#pragma unroll 8
      for (uint32_t x = k0 + lane; x < k1; x += 32) {
        f += a.k_flops[x];
        rd += a.k_read[x];
        wr += a.k_write[x];
      }
    }
    f = warp_sum_u64(f);
    rd = warp_sum_u64(rd);
    wr = warp_sum_u64(wr);
    // a13 model GPU latency: layer kernel latencies in layer order
    double gpu = 0.0, unused = 0.0;
    if (big_l) {
      if (lane == 0)
        for (uint32_t c = a.glc_off[g]; c < a.glc_off[g + 1]; ++c) gpu = __dadd_rn(gpu, a.pl_gpu[c]);
    } else {
      chain_fold<false>(a.l_kern_lat, nullptr, a.gl_off[g], a.gl_off[g + 1], lane, gpu, unused);
    }
    if (lane == 0) {
      s_gpu = gpu;
      s_cnt[0] = f;
      s_cnt[1] = rd;
      s_cnt[2] = wr;
    }
  } else {
    if (big_k) {
      // long group: the chunk partials in tree order (chunk sums of a one-run
      // group's integer latencies are exact, so lat is the reference's double;
      // sum(occ * lat) is re-associated at chunk boundaries)
      if (lane == 0)
        for (uint32_t c = kc0; c < kc1; ++c) {
          lat = __dadd_rn(lat, a.pk_lat[c]);
          occw = __dadd_rn(occw, a.pk_occw[c]);
        }
    } else {
      chain_fold<true>(a.k_lat, a.k_occ, k0, k1, lane, lat, occw);
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t f = s_cnt[0], rd = s_cnt[1], wr = s_cnt[2];
  const double gpu = s_gpu, mlat = a.m_lat[g];
  const uint64_t n = k1 - k0;
  Roof ro = roofline(f, rd, wr, lat, a.peak, a.bw);
  a.m_kern_lat[g] = lat;
  a.m_flops[g] = f;
  a.m_read[g] = rd;
  a.m_write[g] = wr;
  a.m_occ[g] = lat > 0.0 ? occw / lat : 0.0;
  a.m_count[g] = n;
  a.m_ai[g] = ro.ai;
  a.m_tput[g] = ro.tput;
  a.m_bound[g] = ro.bound;
  a.m_gpu[g] = gpu;
  a.m_gpu_pct[g] = gpu / mlat * 100.0;
  a.m_throughput[g] = (double)a.batch[g] / (mlat / 1e9);
  a.m_in[g] = (ro.bound >= 0 && lat > 0.0) ? 1 : 0;
}

// ---- long groups (one long trace: BASELINE config 4) -------------------------
// A group with more than kBigGroup kernels (or layers) would serialise one warp
// on a chain of millions of fp64 additions. Its kernels / layers are cut into
// chunks of kBigChunk; one warp per chunk folds the chunk in tree order, and the
// model / name rows fold the chunk partials in order.
constexpr uint32_t kBigGroup = 1u << 16;
constexpr uint32_t kBigChunk = 8192;

struct BigChunkArgs {
  const uint32_t* desc;  // [n] (begin, end, kind): kind 0 kernel range, 1 layer range
  uint32_t n;
  const double* k_lat;
  const double* k_occ;
  const double* l_kern_lat;
  const uint64_t* k_flops;
  const uint64_t* k_read;
  const uint64_t* k_write;
  double* p_lat;   // kernel chunks: sum lat; layer chunks: sum kern_lat
  double* p_occw;  // kernel chunks: sum occ * lat
  uint64_t* p_cnt; // kernel chunks: [3 c + 0..2] sums of flops, read, write
  // one-run groups: layer chunks also fold the layers' kernel sums (occ * lat,
  // flops, read, write) so the kernel chunks need not be read at all
  const double* l_occw;
  const uint64_t* l_flops;
  const uint64_t* l_read;
  const uint64_t* l_write;
  uint32_t c0;     // first chunk of this launch
};

// One CTA (kBigThreads) per chunk: thread-strided partial sums, then a fixed
// reduction order (xor-butterfly in each warp, warps in order) — the chunk sums
// are re-associated at chunk boundaries anyway (integer latencies stay exact).
constexpr int kBigThreads = 256;
__global__ void __launch_bounds__(kBigThreads) k_big_chunks(BigChunkArgs a) {
  __shared__ double s_s[kBigThreads / 32], s_so[kBigThreads / 32];
  __shared__ unsigned long long s_c[3][kBigThreads / 32];
  const uint32_t c = a.c0 + blockIdx.x, lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  if (c >= a.n) return;
  const uint32_t b = a.desc[3 * c], e = a.desc[3 * c + 1], kind = a.desc[3 * c + 2];
  const double* v = kind == 0 ? a.k_lat : a.l_kern_lat;
  double s = 0.0, so = 0.0;
  uint64_t f = 0, r = 0, w = 0;
  if (kind == 0) {
#pragma unroll 4
    for (uint32_t x = b + threadIdx.x; x < e; x += kBigThreads) {
      const double l = v[x];
      s = __dadd_rn(s, l);
      f += a.k_flops[x];
      r += a.k_read[x];
      w += a.k_write[x];
      so = __dadd_rn(so, __dmul_rn(a.k_occ[x], l));
    }
  } else if (a.l_occw) {
#pragma unroll 4
    for (uint32_t x = b + threadIdx.x; x < e; x += kBigThreads) {
      s = __dadd_rn(s, v[x]);
      so = __dadd_rn(so, a.l_occw[x]);
      f += a.l_flops[x];
      r += a.l_read[x];
      w += a.l_write[x];
    }
  } else {
#pragma unroll 4
    for (uint32_t x = b + threadIdx.x; x < e; x += kBigThreads) s = __dadd_rn(s, v[x]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
    so = __dadd_rn(so, __shfl_xor_sync(0xffffffffu, so, o));
  }
  f = warp_sum_u64(f);
  r = warp_sum_u64(r);
  w = warp_sum_u64(w);
  if (lane == 0) {
    s_s[warp] = s;
    s_so[warp] = so;
    s_c[0][warp] = f;
    s_c[1][warp] = r;
    s_c[2][warp] = w;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0.0, tso = 0.0;
    uint64_t tf = 0, tr = 0, tw = 0;
    for (int q = 0; q < kBigThreads / 32; ++q) {
      ts = __dadd_rn(ts, s_s[q]);
      tso = __dadd_rn(tso, s_so[q]);
      tf += s_c[0][q];
      tr += s_c[1][q];
      tw += s_c[2][q];
    }
    a.p_lat[c] = ts;
    a.p_occw[c] = tso;
    a.p_cnt[3 * c] = tf;
    a.p_cnt[3 * c + 1] = tr;
    a.p_cnt[3 * c + 2] = tw;
  }
}

// ---- a10 by name ------------------------------------------------------------
//
// Fast path: one CTA per group with a shared-memory table keyed by name_id
// (std::map<std::string, Accumulator> of analysis.cpp:402-407; ids are interned
// in string order, so sorting by id is sorting by name). u64 counters use shared
// atomics (order-free, exact); the two fp64 chains per name are applied by one
// thread per name strictly in tree order. Groups with more than NCAP distinct names fall back
// to the sort-based path below.

constexpr int NCAP = 128;
constexpr int NAME_WARPS = 4;
constexpr uint32_t NEMPTY = 0xFFFFFFFFu;

struct NameTable {
  uint32_t key[NCAP];
  double lat[NCAP], occw[NCAP];
  unsigned long long f[NCAP], r[NCAP], w[NCAP], cnt[NCAP];
  uint32_t used[NCAP];
  uint32_t start[NCAP];
  uint32_t nused;
};

struct NameFastArgs {
  uint32_t G;
  const uint32_t* gk_off;
  const uint32_t* gk_end;   // optional: group g = [gk_off[g], gk_end[g]) (chunk pseudo-groups)
  const uint32_t* big;      // optional: gkc_off; groups with chunks are left to k_names_big
  int raw;                  // chunk pseudo-groups: stage raw sums (s_lat, s_occ = sum occ*lat)
  const int32_t* gstatus;
  const uint32_t* k_name;
  const double* k_lat;
  const double* k_occ;
  const uint64_t* k_flops;
  const uint64_t* k_read;
  const uint64_t* k_write;
  const double* m_lat;
  double peak, bw;
  uint32_t* g_count;    // distinct names per group
  uint32_t* overflow;   // any group exceeded NCAP
  uint32_t* ks_slot;    // [TK] scratch: name slot of each kernel (groups above kNameSmemCap)
  uint32_t* ks_rank;    // [TK] scratch: rank of the kernel within its name
  uint32_t* perm;       // [TK] scratch: kernels grouped by name, tree order within
  // rows per group in final order, staged at [g * NCAP, g * NCAP + count)
  uint32_t* s_name;
  uint64_t* s_count;
  double* s_lat;
  double* s_pct;
  uint64_t* s_flops;
  uint64_t* s_read;
  uint64_t* s_write;
  double* s_occ;
  double* s_ai;
  double* s_tput;
  int8_t* s_bound;
};

// One CTA (NAME_WARPS warps) per group. Warp w hashes the w-th quarter of the
// group's kernels; stable ranks within a name combine the warp's running count
// with the counts of the earlier warps (tree order = warp order, then lane order).
// Groups of at most kNameSmemCap kernels keep the per-kernel slot (u8), rank
// and the by-name permutation (u16, group-local) in shared memory.
constexpr uint32_t kNameSmemCap = 8192;
constexpr size_t kNameSmem = kNameSmemCap * (1 + 2 + 2);

// Raw mode's per-warp accumulators (dynamic shared memory; raw launches ask for
// just this much, so more CTAs fit an SM than with the kNameSmem scratch).
struct RawAcc {
  double lat[NAME_WARPS][NCAP], occw[NAME_WARPS][NCAP];
  unsigned long long f[NAME_WARPS][NCAP], r[NAME_WARPS][NCAP], w[NAME_WARPS][NCAP];
  uint32_t cnt[NAME_WARPS][NCAP];
  double st_l[NAME_WARPS][32], st_o[NAME_WARPS][32];
  unsigned long long st_f[NAME_WARPS][32], st_r[NAME_WARPS][32], st_w[NAME_WARPS][32];
};
constexpr size_t kNameRawSmem = sizeof(RawAcc);

__global__ void __launch_bounds__(NAME_WARPS * 32) k_names_fast(NameFastArgs a) {
  extern __shared__ __align__(16) unsigned char nm_dyn[];
  uint8_t* s_slot = nm_dyn;
  uint16_t* s_rank = reinterpret_cast<uint16_t*>(nm_dyn + kNameSmemCap);
  uint16_t* s_perm = s_rank + kNameSmemCap;
  __shared__ NameTable T;
  __shared__ uint32_t wcnt[NAME_WARPS][NCAP];  // per-warp per-slot counts
  __shared__ uint32_t s_over;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u, tid = threadIdx.x;
  const uint32_t g = blockIdx.x;
  if (g >= a.G) return;
  if (a.big && a.big[g + 1] > a.big[g]) return;  // long group: k_names_big
  if (a.gstatus && a.gstatus[g] != XSP_G_OK) {
    if (tid == 0) a.g_count[g] = 0;
    return;
  }
  for (uint32_t s = tid; s < NCAP; s += blockDim.x) {
    T.key[s] = NEMPTY;
    T.lat[s] = T.occw[s] = 0.0;
    T.f[s] = T.r[s] = T.w[s] = T.cnt[s] = 0;
#pragma unroll
    for (int w = 0; w < NAME_WARPS; ++w) wcnt[w][s] = 0;
  }
  if (tid == 0) {
    T.nused = 0;
    s_over = 0;
  }
  __syncthreads();
  const uint32_t k0 = a.gk_off[g], k1 = a.gk_end ? a.gk_end[g] : a.gk_off[g + 1];
  const bool sm_ok = k1 - k0 <= kNameSmemCap;
  const uint32_t q = (k1 - k0 + NAME_WARPS * 32 - 1) / (NAME_WARPS * 32) * 32;  // warp quarter, 32-aligned
  const uint32_t w0 = min(k1, k0 + warp * q), w1 = min(k1, w0 + q);
  const uint32_t lt = lanemask_lt();
  bool over = false;
  if (a.raw) {
    // Raw mode (a chunk of a long group; its sums are re-associated at chunk
    // boundaries anyway): stream the warp's quarter in order with coalesced
    // loads. Per 32 kernels, each name's leader lane adds its peers' values in
    // lane order into the warp's table; the four warp tables are then added in
    // warp order. Deterministic, and no gathers through a name permutation.
    static_assert(sizeof(RawAcc) <= kNameSmem, "raw accumulators fit the scratch");
    RawAcc& R = *reinterpret_cast<RawAcc*>(nm_dyn);
    for (uint32_t s = lane; s < NCAP; s += 32) {
      R.lat[warp][s] = R.occw[warp][s] = 0.0;
      R.f[warp][s] = R.r[warp][s] = R.w[warp][s] = 0;
      R.cnt[warp][s] = 0;
    }
    __syncwarp();
    for (uint32_t base = w0; base < w1; base += 32) {
      const uint32_t x = base + lane;
      const bool v = x < w1;
      uint32_t slot = NCAP + lane;  // distinct dummy for idle lanes
      double l = 0.0, ow = 0.0;
      unsigned long long f = 0, rd = 0, wr = 0;
      if (v) {
        const uint32_t nm = a.k_name[x];
        l = a.k_lat[x];
        ow = __dmul_rn(a.k_occ ? a.k_occ[x] : 0.0, l);
        f = a.k_flops[x];
        if (a.k_read) rd = a.k_read[x];
        if (a.k_write) wr = a.k_write[x];
        uint32_t h = (nm * 2654435761u) & (NCAP - 1), probes = 0;
        for (;;) {
          uint32_t old = *reinterpret_cast<volatile uint32_t*>(&T.key[h]);
          if (old == NEMPTY) old = atomicCAS(&T.key[h], NEMPTY, nm);
          if (old == NEMPTY) {
            T.used[atomicAdd(&T.nused, 1u)] = h;
            break;
          }
          if (old == nm) break;
          h = (h + 1) & (NCAP - 1);
          if (++probes >= NCAP) {
            over = true;
            break;
          }
        }
        if (!over) slot = h;
      }
      if (__any_sync(0xffffffffu, over)) break;
      R.st_l[warp][lane] = l;
      R.st_o[warp][lane] = ow;
      R.st_f[warp][lane] = f;
      R.st_r[warp][lane] = rd;
      R.st_w[warp][lane] = wr;
      const uint32_t peers = match8(slot, 0xffffffffu);
      __syncwarp();
      if (v && (peers & lt) == 0) {  // leader: the name's kernels of this step, in lane order
        double sl = R.lat[warp][slot], so = R.occw[warp][slot];
        unsigned long long sf = R.f[warp][slot], sr = R.r[warp][slot], sw = R.w[warp][slot];
        for (uint32_t m = peers; m; m &= m - 1) {
          const uint32_t qq = __ffs(m) - 1;
          sl = __dadd_rn(sl, R.st_l[warp][qq]);
          so = __dadd_rn(so, R.st_o[warp][qq]);
          sf += R.st_f[warp][qq];
          sr += R.st_r[warp][qq];
          sw += R.st_w[warp][qq];
        }
        R.lat[warp][slot] = sl;
        R.occw[warp][slot] = so;
        R.f[warp][slot] = sf;
        R.r[warp][slot] = sr;
        R.w[warp][slot] = sw;
        R.cnt[warp][slot] += __popc(peers);
      }
      __syncwarp();
    }
    if (__any_sync(0xffffffffu, over) && lane == 0) s_over = 1;
    __syncthreads();
    if (s_over) {
      if (tid == 0) {
        a.g_count[g] = 0;
        atomicOr(a.overflow, 1u);
      }
      return;
    }
    const uint32_t nu = T.nused;
    for (uint32_t u = tid; u < nu; u += blockDim.x) {
      const uint32_t sl = T.used[u];
      double lat = 0.0, occw = 0.0;
      unsigned long long f = 0, rd = 0, wr = 0, cnt = 0;
#pragma unroll
      for (int w = 0; w < NAME_WARPS; ++w) {
        lat = __dadd_rn(lat, R.lat[w][sl]);
        occw = __dadd_rn(occw, R.occw[w][sl]);
        f += R.f[w][sl];
        rd += R.r[w][sl];
        wr += R.w[w][sl];
        cnt += R.cnt[w][sl];
      }
      const uint64_t o = (uint64_t)g * NCAP + u;
      a.s_name[o] = T.key[sl];
      a.s_count[o] = cnt;
      a.s_lat[o] = lat;
      a.s_occ[o] = occw;
      a.s_flops[o] = f;
      a.s_read[o] = rd;
      a.s_write[o] = wr;
    }
    if (tid == 0) a.g_count[g] = nu;
    return;
  }
  // pass A: slot per kernel and its rank within its name inside the warp's quarter
  uint32_t nm_next = w0 + lane < w1 ? a.k_name[w0 + lane] : 0;
  for (uint32_t base = w0; base < w1; base += 32) {
    const uint32_t x = base + lane;
    const bool v = x < w1;
    const uint32_t nm = nm_next;
    if (base + 32 + lane < w1) nm_next = a.k_name[base + 32 + lane];
    uint32_t slot = NCAP + lane;  // distinct dummy for idle lanes
    if (v) {
      uint32_t h = (nm * 2654435761u) & (NCAP - 1);
      uint32_t probes = 0;
      for (;;) {
        // plain read first: most kernels find their name already present, and
        // lanes of one name would otherwise serialise on the same CAS
        uint32_t old = *reinterpret_cast<volatile uint32_t*>(&T.key[h]);
        if (old == NEMPTY) old = atomicCAS(&T.key[h], NEMPTY, nm);
        if (old == NEMPTY) {
          T.used[atomicAdd(&T.nused, 1u)] = h;
          break;
        }
        if (old == nm) break;
        h = (h + 1) & (NCAP - 1);
        if (++probes >= NCAP) {
          over = true;
          break;
        }
      }
      if (!over) slot = h;
    }
    if (__any_sync(0xffffffffu, over)) break;
    const uint32_t peers = match8(slot, 0xffffffffu);  // idle lanes hold distinct dummies >= NCAP
    uint32_t rank = 0;
    if (v) rank = wcnt[warp][slot];
    __syncwarp();
    if (v && (peers & lt) == 0) wcnt[warp][slot] = rank + __popc(peers);
    if (v) {
      if (sm_ok) {
        s_slot[x - k0] = (uint8_t)slot;
        s_rank[x - k0] = (uint16_t)(rank + __popc(peers & lt));
      } else {
        a.ks_slot[x] = slot;
        a.ks_rank[x] = rank + __popc(peers & lt);
      }
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, over) && lane == 0) s_over = 1;
  __syncthreads();
  if (s_over) {
    if (tid == 0) {
      a.g_count[g] = 0;
      atomicOr(a.overflow, 1u);
    }
    return;
  }
  const uint32_t nu = T.nused;
  // pass B: per slot, counts of the earlier warps (wcnt becomes an exclusive
  // prefix) and the total; then the start of each name's run
  for (uint32_t s = tid; s < NCAP; s += blockDim.x) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < NAME_WARPS; ++w) {
      const uint32_t c = wcnt[w][s];
      wcnt[w][s] = run;
      run += c;
    }
    T.cnt[s] = run;
  }
  __syncthreads();
  if (warp == 0) {
    unsigned long long c4[NCAP / 32], sum = 0;
#pragma unroll
    for (int k = 0; k < NCAP / 32; ++k) {
      c4[k] = T.cnt[lane * (NCAP / 32) + k];
      sum += c4[k];
    }
    unsigned long long incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl += y;
    }
    unsigned long long run = incl - sum;
#pragma unroll
    for (int k = 0; k < NCAP / 32; ++k) {
      T.start[lane * (NCAP / 32) + k] = (uint32_t)run;
      run += c4[k];
    }
  }
  __syncthreads();
  // pass C: stable scatter of kernel ordinals by name
  for (uint32_t x = w0 + lane; x < w1; x += 32) {
    if (sm_ok) {
      const uint32_t s = s_slot[x - k0];
      s_perm[T.start[s] + wcnt[warp][s] + s_rank[x - k0]] = (uint16_t)(x - k0);
    } else {
      const uint32_t s = a.ks_slot[x];
      a.perm[k0 + T.start[s] + wcnt[warp][s] + a.ks_rank[x]] = x;
    }
  }
  __syncthreads();
  // pass D: one thread per name walks that name's kernels in tree order
  // (Accumulator::add, analysis.cpp:181-188); the u64 counters ride along (exact).
  // Raw mode (a chunk of a long group, whose sums are re-associated at chunk
  // boundaries anyway): one warp per name, lane-strided partial sums and a
  // fixed xor-butterfly, so a frequent name no longer serialises the chunk.
  if (a.raw) {
    for (uint32_t u = warp; u < nu; u += NAME_WARPS) {
      const uint32_t s = T.used[u];
      const uint32_t b = k0 + T.start[s], n = (uint32_t)T.cnt[s];
      double lat = 0.0, occw = 0.0;
      unsigned long long f = 0, rd = 0, wr = 0;
#pragma unroll 4
      for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t x = sm_ok ? k0 + s_perm[b - k0 + i] : a.perm[b + i];
        const double l = a.k_lat[x];
        lat = __dadd_rn(lat, l);
        occw = __dadd_rn(occw, __dmul_rn(a.k_occ ? a.k_occ[x] : 0.0, l));
        f += a.k_flops[x];
        if (a.k_read) rd += a.k_read[x];
        if (a.k_write) wr += a.k_write[x];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lat = __dadd_rn(lat, __shfl_xor_sync(0xffffffffu, lat, o));
        occw = __dadd_rn(occw, __shfl_xor_sync(0xffffffffu, occw, o));
        f += __shfl_xor_sync(0xffffffffu, f, o);
        rd += __shfl_xor_sync(0xffffffffu, rd, o);
        wr += __shfl_xor_sync(0xffffffffu, wr, o);
      }
      if (lane == 0) {
        T.lat[s] = lat;
        T.occw[s] = occw;
        T.f[s] = f;
        T.r[s] = rd;
        T.w[s] = wr;
      }
    }
  }
  for (uint32_t u = tid; u < (a.raw ? 0u : nu); u += blockDim.x) {
    const uint32_t s = T.used[u];
    const uint32_t b = k0 + T.start[s], n = (uint32_t)T.cnt[s];
    double lat = 0.0, occw = 0.0;
    unsigned long long f = 0, rd = 0, wr = 0;
    uint32_t i = 0;
    for (; i + 8 <= n; i += 8) {  // eight independent gathers in flight, then the ordered chain
      double l8[8], o8[8];
#pragma unroll
      for (int u2 = 0; u2 < 8; ++u2) {
        const uint32_t x = sm_ok ? k0 + s_perm[b - k0 + i + u2] : a.perm[b + i + u2];
        l8[u2] = a.k_lat[x];
        o8[u2] = a.k_occ ? a.k_occ[x] : 0.0;
        f += a.k_flops[x];
        if (a.k_read) rd += a.k_read[x];
        if (a.k_write) wr += a.k_write[x];
      }
#pragma unroll
      for (int u2 = 0; u2 < 8; ++u2) {
        lat = __dadd_rn(lat, l8[u2]);
        occw = __dadd_rn(occw, __dmul_rn(o8[u2], l8[u2]));
      }
    }
    for (; i < n; ++i) {
      const uint32_t x = sm_ok ? k0 + s_perm[b - k0 + i] : a.perm[b + i];
      const double l = a.k_lat[x];
      lat = __dadd_rn(lat, l);
      occw = __dadd_rn(occw, __dmul_rn(a.k_occ ? a.k_occ[x] : 0.0, l));
      f += a.k_flops[x];
      if (a.k_read) rd += a.k_read[x];
      if (a.k_write) wr += a.k_write[x];
    }
    T.lat[s] = lat;
    T.occw[s] = occw;
    T.f[s] = f;
    T.r[s] = rd;
    T.w[s] = wr;
  }
  __syncthreads();
  if (a.raw) {
    for (uint32_t u = tid; u < nu; u += blockDim.x) {
      const uint32_t s = T.used[u];
      const uint64_t o = (uint64_t)g * NCAP + u;
      a.s_name[o] = T.key[s];
      a.s_count[o] = T.cnt[s];
      a.s_lat[o] = T.lat[s];
      a.s_occ[o] = T.occw[s];
      a.s_flops[o] = T.f[s];
      a.s_read[o] = T.r[s];
      a.s_write[o] = T.w[s];
    }
    if (tid == 0) a.g_count[g] = nu;
    return;
  }
  const double mlat = a.m_lat[g];
  // rank = position under (total latency desc, name asc) (analysis.cpp:424-430)
  for (uint32_t u = tid; u < nu; u += blockDim.x) {
    const uint32_t s = T.used[u];
    const double l = T.lat[s];
    const uint32_t nm = T.key[s];
    uint32_t rank = 0;
    for (uint32_t v2 = 0; v2 < nu; ++v2) {
      const uint32_t s2 = T.used[v2];
      const double l2 = T.lat[s2];
      rank += (l2 > l) || (l2 == l && T.key[s2] < nm);
    }
    const uint64_t o = (uint64_t)g * NCAP + rank;
    const Roof ro = roofline(T.f[s], T.r[s], T.w[s], l, a.peak, a.bw);
    a.s_name[o] = nm;
    a.s_count[o] = T.cnt[s];
    a.s_lat[o] = l;
    a.s_pct[o] = l / mlat * 100.0;
    a.s_flops[o] = T.f[s];
    a.s_read[o] = T.r[s];
    a.s_write[o] = T.w[s];
    a.s_occ[o] = l > 0.0 ? T.occw[s] / l : 0.0;
    a.s_ai[o] = ro.ai;
    a.s_tput[o] = ro.tput;
    a.s_bound[o] = ro.bound;
  }
  if (tid == 0) a.g_count[g] = nu;
}

// a10 of a long group: the chunks' raw per-name sums (k_names_fast, raw mode)
// folded chunk by chunk in tree order. Within a chunk every name appears once,
// so lanes add distinct names concurrently; chunks are applied in order.
struct NameBigArgs {
  uint32_t G;
  const uint32_t* gkc_off;
  const int32_t* gstatus;
  const uint32_t* c_count;  // names per chunk
  const uint32_t* c_name;   // chunk rows [c * NCAP, + c_count[c])
  const uint64_t* c_cnt;
  const double* c_lat;
  const double* c_occw;
  const uint64_t* c_f;
  const uint64_t* c_r;
  const uint64_t* c_w;
  const double* m_lat;
  double peak, bw;
  uint32_t* g_count;
  uint32_t* overflow;
  uint32_t* s_name;
  uint64_t* s_count;
  double* s_lat;
  double* s_pct;
  uint64_t* s_flops;
  uint64_t* s_read;
  uint64_t* s_write;
  double* s_occ;
  double* s_ai;
  double* s_tput;
  int8_t* s_bound;
};

// Folds chunk tables [c0, c1) in order into T (one warp). Returns true when
// more than NCAP distinct names appear.
__device__ __forceinline__ bool fold_name_chunks(NameTable& T, const NameBigArgs& a, uint32_t c0, uint32_t c1,
                                                 uint32_t lane) {
  for (uint32_t s = lane; s < NCAP; s += 32) {
    T.key[s] = NEMPTY;
    T.lat[s] = T.occw[s] = 0.0;
    T.f[s] = T.r[s] = T.w[s] = T.cnt[s] = 0;
  }
  if (lane == 0) T.nused = 0;
  __syncwarp();
  bool over = false;
  for (uint32_t c = c0; c < c1; ++c) {
    const uint32_t nc = a.c_count[c];
    for (uint32_t e = lane; e < nc; e += 32) {
      const uint64_t o = (uint64_t)c * NCAP + e;
      const uint32_t nm = a.c_name[o];
      uint32_t h = (nm * 2654435761u) & (NCAP - 1), probes = 0;
      for (;;) {
        const uint32_t old = atomicCAS(&T.key[h], NEMPTY, nm);
        if (old == NEMPTY) {
          T.used[atomicAdd(&T.nused, 1u)] = h;
          break;
        }
        if (old == nm) break;
        h = (h + 1) & (NCAP - 1);
        if (++probes >= NCAP) {
          over = true;
          break;
        }
      }
      if (over) break;
      T.cnt[h] += a.c_cnt[o];
      T.lat[h] = __dadd_rn(T.lat[h], a.c_lat[o]);
      T.occw[h] = __dadd_rn(T.occw[h], a.c_occw[o]);
      T.f[h] += a.c_f[o];
      T.r[h] += a.c_r[o];
      T.w[h] += a.c_w[o];
    }
    if (__any_sync(0xffffffffu, over)) return true;
    __syncwarp();
  }
  __syncwarp();
  return false;
}

// First level of a long group's fold: partial p folds the chunk tables
// [pc0[p], pc1[p]) (consecutive chunks of one group) into one table of the
// chunk layout, so that k_names_big folds ~1/kNamePart as many tables
// serially. Integer latencies stay exact; the occupancy-weighted sums are
// re-associated (within 1e-12, as for the chunks themselves).
constexpr uint32_t kNamePart = 32;
struct NamePartOut {
  uint32_t* count;
  uint32_t* name;
  uint64_t* cnt;
  double* lat;
  double* occw;
  uint64_t* f;
  uint64_t* r;
  uint64_t* w;
};
__global__ void __launch_bounds__(32) k_names_partial(NameBigArgs a, const uint32_t* __restrict__ pc0,
                                                      const uint32_t* __restrict__ pc1, NamePartOut o) {
  __shared__ NameTable T;
  const uint32_t p = blockIdx.x, lane = threadIdx.x;
  if (fold_name_chunks(T, a, pc0[p], pc1[p], lane)) {
    if (lane == 0) {
      o.count[p] = 0;
      atomicOr(a.overflow, 1u);
    }
    return;
  }
  const uint32_t nu = T.nused;
  for (uint32_t u = lane; u < nu; u += 32) {
    const uint32_t sl = T.used[u];
    const uint64_t q = (uint64_t)p * NCAP + u;
    o.name[q] = T.key[sl];
    o.cnt[q] = T.cnt[sl];
    o.lat[q] = T.lat[sl];
    o.occw[q] = T.occw[sl];
    o.f[q] = T.f[sl];
    o.r[q] = T.r[sl];
    o.w[q] = T.w[sl];
  }
  if (lane == 0) o.count[p] = nu;
}

__global__ void __launch_bounds__(32) k_names_big(NameBigArgs a) {
  __shared__ NameTable T;
  const uint32_t g = blockIdx.x, lane = threadIdx.x;
  if (!(a.gkc_off[g + 1] > a.gkc_off[g])) return;
  if (a.gstatus[g] != XSP_G_OK) {
    if (lane == 0) a.g_count[g] = 0;
    return;
  }
  if (fold_name_chunks(T, a, a.gkc_off[g], a.gkc_off[g + 1], lane)) {
    if (lane == 0) {
      a.g_count[g] = 0;
      atomicOr(a.overflow, 1u);
    }
    return;
  }
  const uint32_t nu = T.nused;
  const double mlat = a.m_lat[g];
  for (uint32_t u = lane; u < nu; u += 32) {
    const uint32_t s = T.used[u];
    const double l = T.lat[s];
    const uint32_t nm = T.key[s];
    uint32_t rank = 0;
    for (uint32_t v2 = 0; v2 < nu; ++v2) {
      const uint32_t s2 = T.used[v2];
      const double l2 = T.lat[s2];
      rank += (l2 > l) || (l2 == l && T.key[s2] < nm);
    }
    const uint64_t o = (uint64_t)g * NCAP + rank;
    const Roof ro = roofline(T.f[s], T.r[s], T.w[s], l, a.peak, a.bw);
    a.s_name[o] = nm;
    a.s_count[o] = T.cnt[s];
    a.s_lat[o] = l;
    a.s_pct[o] = l / mlat * 100.0;
    a.s_flops[o] = T.f[s];
    a.s_read[o] = T.r[s];
    a.s_write[o] = T.w[s];
    a.s_occ[o] = l > 0.0 ? T.occw[s] / l : 0.0;
    a.s_ai[o] = ro.ai;
    a.s_tput[o] = ro.tput;
    a.s_bound[o] = ro.bound;
  }
  if (lane == 0) a.g_count[g] = nu;
}

// a5 / a6 / a7: one CTA per group. The group's canonical layers (at most
// kTypesCap) are staged in shared memory with their type slot (type_id mod 128;
// two types on one slot set *over and the 128-wide a10 machinery redoes the
// pass); then one thread per used slot walks the staged layers in order, so
// every type's fp64 latency sum runs in layer order (analysis.cpp:315-337).
// Long groups (layer chunks) are left to the chunked path.
constexpr uint32_t kTypesCap = 2048;
constexpr int kTypesThreads = 128;

__global__ void __launch_bounds__(kTypesThreads) k_types(uint32_t G, const uint32_t* __restrict__ gl_off,
                                                         const int32_t* __restrict__ gstatus,
                                                         const uint32_t* __restrict__ big,
                                                         const uint32_t* __restrict__ l_type,
                                                         const double* __restrict__ l_lat,
                                                         const uint64_t* __restrict__ l_alloc,
                                                         uint32_t* __restrict__ g_count, uint32_t* __restrict__ over,
                                                         uint32_t* __restrict__ s_key, uint64_t* __restrict__ s_count,
                                                         double* __restrict__ s_lat, uint64_t* __restrict__ s_sum) {
  __shared__ uint32_t key[NCAP];
  __shared__ double y_lat[NCAP];
  __shared__ uint8_t slot_of[kTypesCap];
  __shared__ double lat[kTypesCap];
  __shared__ uint64_t alloc[kTypesCap];
  __shared__ int s_bad;
  const uint32_t g = blockIdx.x, tid = threadIdx.x;
  if (g >= G) return;
  if (big && big[g + 1] > big[g]) return;  // long group: chunked path
  if (gstatus[g] != XSP_G_OK) {
    if (tid == 0) g_count[g] = 0;
    return;
  }
  const uint32_t l0 = gl_off[g], n = gl_off[g + 1] - l0;
  if (n > kTypesCap) {
    if (tid == 0) atomicOr(over, 1u);
    return;
  }
  for (uint32_t q = tid; q < NCAP; q += kTypesThreads) key[q] = NEMPTY;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (uint32_t i = tid; i < n; i += kTypesThreads) {
    const uint32_t t = l_type[l0 + i];
    const uint32_t sl = t & (NCAP - 1);
    const uint32_t old = atomicCAS(&key[sl], NEMPTY, t);
    if (old != NEMPTY && old != t) s_bad = 1;
    slot_of[i] = (uint8_t)sl;
    lat[i] = l_lat[l0 + i];
    alloc[i] = l_alloc[l0 + i];
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) atomicOr(over, 1u);
    return;
  }
  const uint32_t mykey = key[tid];
  double acc = 0.0;
  uint64_t cnt = 0, sum = 0;
  if (mykey != NEMPTY) {
    for (uint32_t i = 0; i < n; ++i)
      if (slot_of[i] == tid) {
        acc = __dadd_rn(acc, lat[i]);
        ++cnt;
        sum += alloc[i];
      }
  }
  y_lat[tid] = acc;
  const uint32_t nused = __syncthreads_count(mykey != NEMPTY);
  if (mykey != NEMPTY) {
    uint32_t rank = 0;
    for (uint32_t q = 0; q < NCAP; ++q) {
      const uint32_t kq = key[q];
      if (kq == NEMPTY) continue;
      const double lq = y_lat[q];
      rank += (lq > acc) || (lq == acc && kq < mykey);
    }
    const uint64_t o = (uint64_t)g * NCAP + rank;
    s_key[o] = mykey;
    s_count[o] = cnt;
    s_lat[o] = acc;
    s_sum[o] = sum;
  }
  if (tid == 0) g_count[g] = nused;
}

// a5 rows: type, count, total latency, total alloc_bytes of the staged rows
__global__ void k_types_place(uint32_t G, const uint32_t* __restrict__ off, const uint32_t* __restrict__ s_key,
                              const uint64_t* __restrict__ s_count, const double* __restrict__ s_lat,
                              const uint64_t* __restrict__ s_sum, uint32_t* __restrict__ y_type,
                              uint64_t* __restrict__ y_count, double* __restrict__ y_lat,
                              int64_t* __restrict__ y_alloc) {
  const uint32_t g = blockIdx.x;
  if (g >= G) return;
  const uint32_t b = off[g], n = off[g + 1] - b;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t s = (uint64_t)g * NCAP + i;
    y_type[b + i] = s_key[s];
    y_count[b + i] = s_count[s];
    y_lat[b + i] = s_lat[s];
    y_alloc[b + i] = (int64_t)s_sum[s];
  }
}

// every a10 column of the staged rows in one launch
struct NamePlaceArgs {
  uint32_t G;
  const uint32_t* off;
  const uint32_t* s_name; const uint64_t* s_count; const double* s_lat; const double* s_pct;
  const uint64_t* s_flops; const uint64_t* s_read; const uint64_t* s_write; const double* s_occ;
  const double* s_ai; const double* s_tput; const int8_t* s_bound;
  uint32_t* n_name; uint64_t* n_count; double* n_lat; double* n_pct;
  uint64_t* n_flops; uint64_t* n_read; uint64_t* n_write; double* n_occ;
  double* n_ai; double* n_tput; int8_t* n_bound;
};
__global__ void k_names_place_all(NamePlaceArgs a) {
  const uint32_t g = blockIdx.x;
  if (g >= a.G) return;
  const uint32_t b = a.off[g], n = a.off[g + 1] - b;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t s = (uint64_t)g * NCAP + i;
    a.n_name[b + i] = a.s_name[s];
    a.n_count[b + i] = a.s_count[s];
    a.n_lat[b + i] = a.s_lat[s];
    a.n_pct[b + i] = a.s_pct[s];
    a.n_flops[b + i] = a.s_flops[s];
    a.n_read[b + i] = a.s_read[s];
    a.n_write[b + i] = a.s_write[s];
    a.n_occ[b + i] = a.s_occ[s];
    a.n_ai[b + i] = a.s_ai[s];
    a.n_tput[b + i] = a.s_tput[s];
    a.n_bound[b + i] = a.s_bound[s];
  }
}


// Sort-based fallback (any number of names per group).

__global__ void k_name_keys(uint32_t total_k, const uint32_t* __restrict__ gk_off, uint32_t G,
                            const uint32_t* __restrict__ k_name, const int32_t* __restrict__ gstatus,
                            uint64_t* __restrict__ key, uint32_t* __restrict__ val) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= total_k) return;
  uint32_t lo = 0, hi = G;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (gk_off[mid] <= j) lo = mid; else hi = mid;
  }
  // failed groups sort to the end and are ignored
  key[j] = gstatus[lo] == XSP_G_OK ? (((uint64_t)lo << 32) | k_name[j]) : ~0ull;
  val[j] = j;
}

__global__ void k_seg_flags(uint32_t n, const uint64_t* __restrict__ key, uint32_t* __restrict__ flag) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  flag[j] = (key[j] != ~0ull && (j == 0 || key[j] != key[j - 1])) ? 1u : 0u;
}

struct NameArgs {
  uint32_t n;  // kernels in sorted array
  const uint64_t* key;
  const uint32_t* val;
  const uint32_t* seg_pos;  // exclusive scan of flags
  const uint32_t* flag;
  const double* k_lat;
  const double* k_occ;
  const uint64_t* k_flops;
  const uint64_t* k_read;
  const uint64_t* k_write;
  const double* m_lat;
  double peak, bw;
  uint32_t* s_group;
  uint32_t* s_name;
  uint64_t* s_count;
  double* s_lat;
  double* s_pct;
  uint64_t* s_flops;
  uint64_t* s_read;
  uint64_t* s_write;
  double* s_occ;
  double* s_ai;
  double* s_tput;
  int8_t* s_bound;
};

__global__ void k_name_rows(NameArgs a) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n || !a.flag[j]) return;
  const uint64_t k = a.key[j];
  const uint32_t s = a.seg_pos[j];
  double lat = 0.0, occw = 0.0;
  uint64_t f = 0, rd = 0, wr = 0, c = 0;
  for (uint32_t q = j; q < a.n && a.key[q] == k; ++q) {
    uint32_t x = a.val[q];
    double kl = a.k_lat[x];
    lat = __dadd_rn(lat, kl);
    f += a.k_flops[x];
    rd += a.k_read[x];
    wr += a.k_write[x];
    occw = __dadd_rn(occw, __dmul_rn(a.k_occ[x], kl));
    ++c;
  }
  const uint32_t g = (uint32_t)(k >> 32);
  Roof ro = roofline(f, rd, wr, lat, a.peak, a.bw);
  a.s_group[s] = g;
  a.s_name[s] = (uint32_t)k;
  a.s_count[s] = c;
  a.s_lat[s] = lat;
  a.s_pct[s] = lat / a.m_lat[g] * 100.0;
  a.s_flops[s] = f;
  a.s_read[s] = rd;
  a.s_write[s] = wr;
  a.s_occ[s] = lat > 0.0 ? occw / lat : 0.0;
  a.s_ai[s] = ro.ai;
  a.s_tput[s] = ro.tput;
  a.s_bound[s] = ro.bound;
}

// Per group: rows sorted by total latency desc, then name asc (analysis.cpp:424-430).
__global__ void k_name_order(uint32_t G, const uint32_t* __restrict__ g_name_off,
                             const double* __restrict__ s_lat, uint32_t* __restrict__ order) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  uint32_t b = g_name_off[g], e = g_name_off[g + 1];
  for (uint32_t i = b; i < e; ++i) {
    uint32_t x = i;
    uint32_t j = i;
    while (j > b && s_lat[order[j - 1]] < s_lat[x]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = x;
  }
}

template <typename T>
__global__ void k_permute(uint32_t n, const uint32_t* __restrict__ order, const T* __restrict__ src,
                          T* __restrict__ dst) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[order[i]];
}

__global__ void k_csr_groups(uint32_t G, uint32_t n, const uint32_t* __restrict__ s_group,
                             uint32_t* __restrict__ off) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > G) return;
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (s_group[mid] < g) lo = mid + 1; else hi = mid;
  }
  off[g] = lo;
}

// ---------------------------------------------------------------------------

namespace {
template <typename K, typename... Args>
void launch(xsp_ctx* ctx, K kernel, uint64_t n, cudaStream_t st, Args... args) {
  if (n == 0) return;
  kernel<<<ceil_div(n, 256), 256, 0, st>>>(args...);
  ++ctx->launches;
}
}  // namespace

void run_analyze(xsp_ctx* ctx, const xsp_span_cols* c, const xsp_corr_out* corr, const xsp_groups* gr,
                 const xsp_system_spec* spec, const xsp_analysis_opts* opts, xsp_tables_out* out,
                 cudaStream_t st) {
  const uint32_t G = gr->n_groups;
  if (opts->top_k > 8) throw std::invalid_argument("top_k must be <= 8");
  // group descriptors are host arrays
  uint32_t* hg = ctx->h<uint32_t>("a.groups_h", 4ull * G + 4);
  uint32_t total_runs = 0, max_runs = 0;
  bool all_one_run = G > 0;
  for (uint32_t g = 0; g < G; ++g) {
    all_one_run &= gr->n_runs[g] == 1;
    max_runs = std::max(max_runs, gr->n_runs[g]);
    hg[g] = gr->first_trace[g];
    hg[G + g] = gr->n_runs[g];
    hg[2 * G + g] = gr->batch_size[g];
    hg[3 * G + g] = total_runs;
    if ((uint64_t)gr->first_trace[g] + gr->n_runs[g] > corr->n_traces)
      throw std::invalid_argument("group references traces beyond the correlation result");
    total_runs += gr->n_runs[g];
  }
  hg[4 * G] = total_runs;
  uint32_t* dg = ctx->d<uint32_t>("a.groups", 4ull * G + 4);
  xfer_small(dg, hg, (4ull * G + 1) * 4, st);
  const uint32_t* ft = dg;
  const uint32_t* nr = dg + G;
  const uint32_t* batch = dg + 2 * G;
  const uint32_t* run_off = dg + 3 * G;

  GroupArgs ga;
  ga.G = G;
  ga.ft = ft;
  ga.nr = nr;
  ga.batch = batch;
  ga.t_status = corr->trace_status;
  ga.t_layer_off = corr->trace_layer_off;
  ga.t_kernel_off = corr->trace_kernel_off;
  ga.l_koff = corr->layer_kernel_off;
  ga.gl = ctx->d<uint32_t>("a.gl", G + 1);
  ga.gk = ctx->d<uint32_t>("a.gk", G + 1);
  ga.gerr = ctx->d<unsigned long long>("a.gerr", G);
  launch(ctx, k_group_prep, G, st, ga);
  out->n_groups = G;
  out->group_layer_off = ctx->d<uint32_t>("t.g_loff", G + 1);
  out->group_kernel_off = ctx->d<uint32_t>("t.g_koff", G + 1);
  uint32_t* scan_tmp = ctx->d<uint32_t>("a.scan", scan_scratch_elems(G + 16));
  uint32_t* htot = ctx->h<uint32_t>("a.tot_h", 8);
  uint32_t* hgl = ctx->h<uint32_t>("a.gl_h", G + 1);
  uint32_t* hgk = ctx->h<uint32_t>("a.gk_h", G + 1);
  if (ctx->hc_layer_key == corr->trace_layer_off && ctx->hc_kernel_key == corr->trace_kernel_off &&
      ctx->hc_T == corr->n_traces) {
    // the correlation's offsets are already on the host: group tables of the
    // canonical (first) runs without a device round trip
    const uint32_t* tl = ctx->h<uint32_t>("c.hc_loff", corr->n_traces + 1);
    const uint32_t* tk = ctx->h<uint32_t>("c.hc_koff", corr->n_traces + 1);
    uint32_t* hoff = ctx->h<uint32_t>("a.goff_h", 2ull * (G + 1));
    uint32_t sl = 0, sk = 0;
    for (uint32_t g = 0; g < G; ++g) {
      hgl[g] = hoff[g] = sl;
      hgk[g] = hoff[G + 1 + g] = sk;
      if (gr->n_runs[g]) {
        const uint32_t t = gr->first_trace[g];
        sl += tl[t + 1] - tl[t];
        sk += tk[t + 1] - tk[t];
      }
    }
    hgl[G] = hoff[G] = sl;
    hgk[G] = hoff[2 * G + 1] = sk;
    htot[0] = sl;
    htot[1] = sk;
    xfer_small(out->group_layer_off, hoff, (G + 1) * 4ull, st);
    xfer_small(out->group_kernel_off, hoff + G + 1, (G + 1) * 4ull, st);
  } else {
    exclusive_scan<uint32_t, uint32_t>(ga.gl, out->group_layer_off, G, scan_tmp, out->group_layer_off + G, st,
                                       &ctx->launches);
    exclusive_scan<uint32_t, uint32_t>(ga.gk, out->group_kernel_off, G, scan_tmp, out->group_kernel_off + G, st,
                                       &ctx->launches);
    xfer_small(htot, out->group_layer_off + G, 4, st);
    xfer_small(htot + 1, out->group_kernel_off + G, 4, st);
    // group offsets on the host too (same sync) when some group may be long
    xfer_small(hgl, out->group_layer_off, (G + 1) * 4ull, st);
    xfer_small(hgk, out->group_kernel_off, (G + 1) * 4ull, st);
    XSP_CUDA(cudaStreamSynchronize(st));
  }
  const uint32_t TL = htot[0], TK = htot[1];
  // long groups (one long trace): chunk descriptors for k_big_chunks
  std::vector<uint32_t> desc, gkc(G + 1, 0), glc(G + 1, 0);
  uint32_t nkc = 0;
  for (uint32_t g = 0; g < G; ++g) {
    gkc[g] = nkc;
    if (hgk[g + 1] - hgk[g] > kBigGroup || hgl[g + 1] - hgl[g] > kBigGroup)
      for (uint32_t b = hgk[g]; b < hgk[g + 1]; b += kBigChunk, ++nkc)
        desc.insert(desc.end(), {b, std::min(b + kBigChunk, hgk[g + 1]), 0u});
  }
  gkc[G] = nkc;
  uint32_t nlc = 0;
  for (uint32_t g = 0; g < G; ++g) {
    glc[g] = nkc + nlc;
    if (gkc[g + 1] > gkc[g])
      for (uint32_t b = hgl[g]; b < hgl[g + 1]; b += kBigChunk, ++nlc)
        desc.insert(desc.end(), {b, std::min(b + kBigChunk, hgl[g + 1]), 1u});
  }
  glc[G] = nkc + nlc;
  const uint32_t n_chunks = nkc + nlc;
  // partial folds of the chunk tables (k_names_partial): kNamePart consecutive
  // chunks of one group each; [pc0 | pc1] ranges and per-group partial offsets
  std::vector<uint32_t> pk_rng, pl_rng, pk_off(G + 1, 0), pl_off(G + 1, 0);
  for (uint32_t g = 0; g < G; ++g) {
    pk_off[g] = (uint32_t)(pk_rng.size() / 2);
    for (uint32_t c = gkc[g]; c < gkc[g + 1]; c += kNamePart)
      pk_rng.insert(pk_rng.end(), {c, std::min(c + kNamePart, gkc[g + 1])});
    pl_off[g] = (uint32_t)(pl_rng.size() / 2);
    for (uint32_t c = glc[g] - nkc; c < glc[g + 1] - nkc; c += kNamePart)
      pl_rng.insert(pl_rng.end(), {c, std::min(c + kNamePart, glc[g + 1] - nkc)});
  }
  const uint32_t npk = (uint32_t)(pk_rng.size() / 2), npl = (uint32_t)(pl_rng.size() / 2);
  pk_off[G] = npk;
  pl_off[G] = npl;
  uint32_t *d_desc = nullptr, *d_gkc = nullptr, *d_glc = nullptr, *d_kcb = nullptr, *d_kce = nullptr;
  uint32_t *d_lcb = nullptr, *d_lce = nullptr, *d_glc_rel = nullptr;
  uint32_t *d_pk = nullptr, *d_pk_off = nullptr, *d_pl = nullptr, *d_pl_off = nullptr;
  if (n_chunks) {
    const size_t words = desc.size() + 3ull * (G + 1) + 2ull * nkc + 2ull * nlc + 2ull * (npk + npl) + 2ull * (G + 1);
    uint32_t* hd = ctx->h<uint32_t>("a.big_h", words);
    std::memcpy(hd, desc.data(), desc.size() * 4);
    std::memcpy(hd + desc.size(), gkc.data(), (G + 1) * 4ull);
    std::memcpy(hd + desc.size() + G + 1, glc.data(), (G + 1) * 4ull);
    uint32_t* kcb = hd + desc.size() + 2ull * (G + 1);
    for (uint32_t c = 0; c < nkc; ++c) {
      kcb[c] = desc[3 * c];
      kcb[nkc + c] = desc[3 * c + 1];
    }
    uint32_t* lcb = kcb + 2ull * nkc;  // layer chunks (a5 of long groups)
    for (uint32_t c = 0; c < nlc; ++c) {
      lcb[c] = desc[3 * (nkc + c)];
      lcb[nlc + c] = desc[3 * (nkc + c) + 1];
    }
    uint32_t* grel = lcb + 2ull * nlc;
    for (uint32_t g = 0; g <= G; ++g) grel[g] = glc[g] - nkc;
    uint32_t* hp = grel + G + 1;  // [pk0 | pk1 | pk_off | pl0 | pl1 | pl_off]
    for (uint32_t q = 0; q < npk; ++q) {
      hp[q] = pk_rng[2 * q];
      hp[npk + q] = pk_rng[2 * q + 1];
    }
    std::memcpy(hp + 2ull * npk, pk_off.data(), (G + 1) * 4ull);
    uint32_t* hq = hp + 2ull * npk + G + 1;
    for (uint32_t q = 0; q < npl; ++q) {
      hq[q] = pl_rng[2 * q];
      hq[npl + q] = pl_rng[2 * q + 1];
    }
    std::memcpy(hq + 2ull * npl, pl_off.data(), (G + 1) * 4ull);
    uint32_t* dd = ctx->d<uint32_t>("a.big", words);
    XSP_CUDA(cudaMemcpyAsync(dd, hd, words * 4, cudaMemcpyHostToDevice, st));
    d_desc = dd;
    d_gkc = dd + desc.size();
    d_glc = d_gkc + G + 1;
    d_kcb = d_glc + G + 1;
    d_kce = d_kcb + nkc;
    d_lcb = d_kce + nkc;
    d_lce = d_lcb + nlc;
    d_glc_rel = d_lce + nlc;
    d_pk = d_glc_rel + G + 1;
    d_pk_off = d_pk + 2ull * npk;
    d_pl = d_pk_off + G + 1;
    d_pl_off = d_pl + 2ull * npl;
  }
  // a long group's chunk tables: partial folds (levels of kNamePart tables while
  // a group has more than kNamePart of them), then the ordered fold + ranking
  auto fold_big = [&](NameBigArgs nb, const uint32_t* d_rng, const uint32_t* d_poff, uint32_t np,
                      const std::vector<uint32_t>& h_poff, const std::string& tag, cudaStream_t st) {
    std::vector<uint32_t> poff = h_poff;  // group -> [first, last) table of the current level
    for (int level = 0; np; ++level) {
      const std::string lt = tag + (level ? std::to_string(level) : std::string());
      const uint64_t cap = (uint64_t)np * NCAP;
      NamePartOut po;
      po.count = ctx->d<uint32_t>(lt + ".count", np);
      po.name = ctx->d<uint32_t>(lt + ".name", cap);
      po.cnt = ctx->d<uint64_t>(lt + ".cnt", cap);
      po.lat = ctx->d<double>(lt + ".lat", cap);
      po.occw = ctx->d<double>(lt + ".occw", cap);
      po.f = ctx->d<uint64_t>(lt + ".f", cap);
      po.r = ctx->d<uint64_t>(lt + ".r", cap);
      po.w = ctx->d<uint64_t>(lt + ".w", cap);
      k_names_partial<<<np, 32, 0, st>>>(nb, d_rng, d_rng + np, po);
      ++ctx->launches;
      nb.gkc_off = d_poff;
      nb.c_count = po.count;
      nb.c_name = po.name;
      nb.c_cnt = po.cnt;
      nb.c_lat = po.lat;
      nb.c_occw = po.occw;
      nb.c_f = po.f;
      nb.c_r = po.r;
      nb.c_w = po.w;
      // next level: kNamePart consecutive partial tables of one group each
      uint32_t widest = 0;
      for (uint32_t g = 0; g < G; ++g) widest = std::max(widest, poff[g + 1] - poff[g]);
      if (widest <= kNamePart) break;
      std::vector<uint32_t> rng, noff(G + 1, 0);
      for (uint32_t g = 0; g < G; ++g) {
        noff[g] = (uint32_t)(rng.size() / 2);
        for (uint32_t q = poff[g]; q < poff[g + 1]; q += kNamePart)
          rng.insert(rng.end(), {q, std::min(q + kNamePart, poff[g + 1])});
      }
      np = (uint32_t)(rng.size() / 2);
      noff[G] = np;
      uint32_t* h = ctx->h<uint32_t>(lt + ".lvl_h", 2ull * np + G + 1);
      for (uint32_t q = 0; q < np; ++q) {
        h[q] = rng[2 * q];
        h[np + q] = rng[2 * q + 1];
      }
      std::memcpy(h + 2ull * np, noff.data(), (G + 1) * 4ull);
      uint32_t* d = ctx->d<uint32_t>(lt + ".lvl", 2ull * np + G + 1);
      xfer_small(d, h, (2ull * np + G + 1) * 4, st);
      d_rng = d;
      d_poff = d + 2ull * np;
      poff.swap(noff);
    }
    k_names_big<<<G, 32, 0, st>>>(nb);
    ++ctx->launches;
  };
  launch(ctx, k_group_check_runs, total_runs, st, ga, total_runs, run_off);
  if (TL && max_runs > 1) {
    k_group_check_layers<<<dim3(ceil_div((uint64_t)TL, 256), max_runs - 1), 256, 0, st>>>(ga, TL,
                                                                                         out->group_layer_off);
    ++ctx->launches;
  }
  out->group_status = ctx->d<int32_t>("t.g_status", G);
  out->group_err_arg = ctx->d<uint32_t>("t.g_arg", G);
  launch(ctx, k_group_status, G, st, G, nr, ga.gerr, opts->trim_fraction, out->group_status,
         out->group_err_arg);

  // ---- per layer + per kernel
  LayerArgs la;
  la.G = G;
  la.total_layers = TL;
  la.top_k = opts->top_k;
  la.gl_off = out->group_layer_off;
  la.gk_off = out->group_kernel_off;
  la.ft = ft;
  la.nr = nr;
  la.gstatus = out->group_status;
  la.t_layer_off = corr->trace_layer_off;
  la.t_kernel_off = corr->trace_kernel_off;
  la.l_koff = corr->layer_kernel_off;
  la.layer_dur = corr->layer_dur;
  la.layer_attr_row = corr->layer_attr_row;
  la.type_id = c->type_id;
  la.alloc_bytes = c->alloc_bytes;
  la.l_type = ctx->d<uint32_t>("a.l_type", TL);
  la.l_alloc = ctx->d<uint64_t>("a.l_alloc", TL);
  la.layer_row = corr->layer_row;
  la.kernel_dur = corr->kernel_dur;
  la.kernel_mrow = corr->kernel_metric_row;
  la.kernel_name = corr->kernel_name;
  la.kernel_occ = corr->kernel_occ;
  la.m_flops = c->flops;
  la.m_read = c->dram_read;
  la.m_write = c->dram_write;
  la.m_occ = c->occupancy;
  la.trim = opts->trim_fraction;
  la.noise = opts->noise_tolerance;
  la.peak = spec->peak_flops;
  la.bw = spec->memory_bandwidth_bytes_per_s;
  out->n_layers = TL;
  out->n_kernels = TK;
  out->k_name = la.k_name = ctx->d<uint32_t>("t.k_name", TK);
  out->k_layer = la.k_layer = ctx->d<uint32_t>("t.k_layer", TK);
  out->k_lat = la.k_lat = ctx->d<double>("t.k_lat", TK);
  out->k_flops = la.k_flops = ctx->d<uint64_t>("t.k_flops", TK);
  out->k_read = la.k_read = ctx->d<uint64_t>("t.k_read", TK);
  out->k_write = la.k_write = ctx->d<uint64_t>("t.k_write", TK);
  out->k_occ = la.k_occ = ctx->d<double>("t.k_occ", TK);
  out->k_ai = la.k_ai = ctx->d<double>("t.k_ai", TK);
  out->k_tput = la.k_tput = ctx->d<double>("t.k_tput", TK);
  out->k_bound = la.k_bound = ctx->d<int8_t>("t.k_bound", TK);
  out->k_roofline_in = la.k_in = ctx->d<uint8_t>("t.k_in", TK);
  out->l_index = la.l_index = ctx->d<uint32_t>("t.l_index", TL);
  out->l_row = la.l_row = ctx->d<uint32_t>("t.l_row", TL);
  out->l_layer_lat = la.l_layer_lat = ctx->d<double>("t.l_layer_lat", TL);
  out->l_kern_lat = la.l_kern_lat = ctx->d<double>("t.l_kern_lat", TL);
  out->l_flops = la.l_flops = ctx->d<uint64_t>("t.l_flops", TL);
  out->l_read = la.l_read = ctx->d<uint64_t>("t.l_read", TL);
  out->l_write = la.l_write = ctx->d<uint64_t>("t.l_write", TL);
  out->l_occ = la.l_occ = ctx->d<double>("t.l_occ", TL);
  out->l_count = la.l_count = ctx->d<uint64_t>("t.l_count", TL);
  out->l_ai = la.l_ai = ctx->d<double>("t.l_ai", TL);
  out->l_tput = la.l_tput = ctx->d<double>("t.l_tput", TL);
  out->l_bound = la.l_bound = ctx->d<int8_t>("t.l_bound", TL);
  out->l_nongpu = la.l_nongpu = ctx->d<double>("t.l_nongpu", TL);
  out->l_gpu_share = la.l_gpu_share = ctx->d<double>("t.l_gshare", TL);
  out->l_nongpu_share = la.l_nongpu_share = ctx->d<double>("t.l_ngshare", TL);
  out->l_flagged = la.l_flagged = ctx->d<uint8_t>("t.l_flagged", TL);
  out->l_roofline_in = la.l_in = ctx->d<uint8_t>("t.l_in", TL);
  out->l_topk = la.l_topk = ctx->d<uint32_t>("t.l_topk", (uint64_t)TL * (opts->top_k ? opts->top_k : 1));
  ctx->stage_begin("layers", st);
  la.l_occw = nullptr;
  if (all_one_run) {
    if (n_chunks) la.l_occw = ctx->d<double>("t.l_occw", TL);
    launch(ctx, k_kernels_r1, TK, st, la, TK);
    launch(ctx, k_layers<true>, TL, st, la);
  } else {
    launch(ctx, k_kernels, TK, st, la, TK);
    launch(ctx, k_layers<false>, TL, st, la);
  }
  ctx->stage_end("layers", st);

  // ---- per model
  ModelArgs ma;
  ma.G = G;
  ma.gl_off = out->group_layer_off;
  ma.gk_off = out->group_kernel_off;
  ma.ft = ft;
  ma.nr = nr;
  ma.batch = batch;
  ma.gstatus = out->group_status;
  ma.model_row = corr->trace_model_row;
  ma.begin = c->begin_ns;
  ma.end = c->end_ns;
  ma.k_lat = la.k_lat;
  ma.k_occ = la.k_occ;
  ma.k_flops = la.k_flops;
  ma.k_read = la.k_read;
  ma.k_write = la.k_write;
  ma.l_kern_lat = la.l_kern_lat;
  ma.trim = opts->trim_fraction;
  ma.peak = la.peak;
  ma.bw = la.bw;
  out->m_lat = ma.m_lat = ctx->d<double>("t.m_lat", G);
  out->m_kern_lat = ma.m_kern_lat = ctx->d<double>("t.m_kern_lat", G);
  out->m_flops = ma.m_flops = ctx->d<uint64_t>("t.m_flops", G);
  out->m_read = ma.m_read = ctx->d<uint64_t>("t.m_read", G);
  out->m_write = ma.m_write = ctx->d<uint64_t>("t.m_write", G);
  out->m_occ = ma.m_occ = ctx->d<double>("t.m_occ", G);
  out->m_count = ma.m_count = ctx->d<uint64_t>("t.m_count", G);
  out->m_ai = ma.m_ai = ctx->d<double>("t.m_ai", G);
  out->m_tput = ma.m_tput = ctx->d<double>("t.m_tput", G);
  out->m_bound = ma.m_bound = ctx->d<int8_t>("t.m_bound", G);
  out->m_gpu = ma.m_gpu = ctx->d<double>("t.m_gpu", G);
  out->m_gpu_pct = ma.m_gpu_pct = ctx->d<double>("t.m_gpu_pct", G);
  out->m_throughput = ma.m_throughput = ctx->d<double>("t.m_tp", G);
  out->m_roofline_in = ma.m_in = ctx->d<uint8_t>("t.m_in", G);
  ma.gkc_off = d_gkc;
  ma.glc_off = d_glc;
  ma.layer_sums = all_one_run && n_chunks;
  ma.pk_lat = ma.pk_occw = ma.pl_gpu = nullptr;
  ma.pk_cnt = nullptr;
  double *p_lat = nullptr, *p_occw = nullptr;
  ctx->stage_begin("models", st);
  if (n_chunks) {
    BigChunkArgs bc;
    bc.desc = d_desc;
    bc.n = n_chunks;
    bc.k_lat = la.k_lat;
    bc.k_occ = la.k_occ;
    bc.l_kern_lat = la.l_kern_lat;
    bc.p_lat = p_lat = ctx->d<double>("a.p_lat", n_chunks);
    bc.p_occw = p_occw = ctx->d<double>("a.p_occw", n_chunks);
    bc.k_flops = la.k_flops;
    bc.k_read = la.k_read;
    bc.k_write = la.k_write;
    bc.p_cnt = ctx->d<uint64_t>("a.p_cnt", 3ull * n_chunks);
    ma.pk_cnt = bc.p_cnt;
    bc.l_occw = la.l_occw;
    bc.l_flops = la.l_flops;
    bc.l_read = la.l_read;
    bc.l_write = la.l_write;
    // one-run: only the layer chunks are folded (they carry the kernel sums)
    bc.c0 = all_one_run ? nkc : 0;
    k_big_chunks<<<n_chunks - bc.c0, kBigThreads, 0, st>>>(bc);
    ++ctx->launches;
    ma.pk_lat = p_lat;
    ma.pk_occw = p_occw;
    ma.pl_gpu = p_lat;
  }
  if (G) {
    k_model_lat<<<ceil_div((uint64_t)G * 32, 256), 256, 0, st>>>(ma);
    ++ctx->launches;
  }
  // a15, a10 and a5 are independent once the kernel / layer rows and the model
  // latencies exist, and each is bound by its longest group's ordered fp64
  // chain, not by memory: they run concurrently on three streams
  const bool fork = G > 0 && TK > 0;
  cudaStream_t sn = st, sy = st;
  if (fork) {
    sn = ctx->side_stream(0);
    sy = ctx->side_stream(1);
    XSP_CUDA(cudaEventRecord(ctx->fork_event(), st));
    XSP_CUDA(cudaStreamWaitEvent(sn, ctx->fork_event(), 0));
    XSP_CUDA(cudaStreamWaitEvent(sy, ctx->fork_event(), 0));
  }
  if (G) {
    k_models<<<G, 64, 0, st>>>(ma);
    ++ctx->launches;
  }
  ctx->stage_end("models", st);

  // ---- a5 / a6 / a7 by layer type: the a10 machinery keyed by the canonical
  // layers' type ids (values: layer latency, alloc_bytes), launched before the
  // a10 read-back so both totals come back with one sync
  out->group_type_off = ctx->d<uint32_t>("t.g_yoff", G + 1);
  bool types_wide = false;
  std::function<void(cudaStream_t)> run_types;
  run_types = [&](cudaStream_t st) {
    if (!G) {
      htot[4] = htot[5] = 0;
      return;
    }
    NameFastArgs ty;
    std::memset(&ty, 0, sizeof(ty));
    ty.G = G;
    ty.gk_off = out->group_layer_off;
    ty.gk_end = nullptr;
    ty.big = d_glc_rel;
    ty.raw = 0;
    ty.gstatus = out->group_status;
    ty.k_name = la.l_type;
    ty.k_lat = la.l_layer_lat;
    ty.k_occ = nullptr;
    ty.k_flops = la.l_alloc;
    ty.k_read = ty.k_write = nullptr;
    ty.m_lat = ma.m_lat;
    ty.peak = la.peak;
    ty.bw = la.bw;
    ty.g_count = ctx->d<uint32_t>("a.y_gcount", G + 1);
    ty.overflow = ctx->d<uint32_t>("a.y_over", 1);
    ty.ks_slot = ctx->d<uint32_t>("a.y_ks_slot", TL + 1);
    ty.ks_rank = ctx->d<uint32_t>("a.y_ks_rank", TL + 1);
    ty.perm = ctx->d<uint32_t>("a.y_perm", TL + 1);
    const uint64_t cap = (uint64_t)G * NCAP;
    ty.s_name = ctx->d<uint32_t>("a.y_s_key", cap);
    ty.s_count = ctx->d<uint64_t>("a.y_s_count", cap);
    ty.s_lat = ctx->d<double>("a.y_s_lat", cap);
    ty.s_pct = ctx->d<double>("a.y_s_pct", cap);
    ty.s_flops = ctx->d<uint64_t>("a.y_s_sum", cap);
    ty.s_read = ctx->d<uint64_t>("a.y_s_r", cap);
    ty.s_write = ctx->d<uint64_t>("a.y_s_w", cap);
    ty.s_occ = ctx->d<double>("a.y_s_occ", cap);
    ty.s_ai = ctx->d<double>("a.y_s_ai", cap);
    ty.s_tput = ctx->d<double>("a.y_s_tput", cap);
    ty.s_bound = ctx->d<int8_t>("a.y_s_bound", cap);
    XSP_CUDA(cudaMemsetAsync(ty.overflow, 0, 4, st));
    if (!types_wide) {
      k_types<<<G, kTypesThreads, 0, st>>>(G, out->group_layer_off, out->group_status, d_glc_rel,
                                                            la.l_type, la.l_layer_lat, la.l_alloc, ty.g_count,
                                                            ty.overflow, ty.s_name, ty.s_count, ty.s_lat,
                                                            ty.s_flops);
    } else {  // a type-slot collision or a group above kTypesCap: the a10 machinery
      XSP_CUDA(cudaFuncSetAttribute(k_names_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kNameSmem));
      k_names_fast<<<G, NAME_WARPS * 32, kNameSmem, st>>>(ty);
    }
    ++ctx->launches;
    if (nlc) {
      NameFastArgs tc = ty;
      tc.G = nlc;
      tc.gk_off = d_lcb;
      tc.gk_end = d_lce;
      tc.big = nullptr;
      tc.gstatus = nullptr;
      tc.raw = 1;
      const uint64_t ccap = (uint64_t)nlc * NCAP;
      tc.g_count = ctx->d<uint32_t>("a.yc_count", nlc);
      tc.s_name = ctx->d<uint32_t>("a.yc_key", ccap);
      tc.s_count = ctx->d<uint64_t>("a.yc_cnt", ccap);
      tc.s_lat = ctx->d<double>("a.yc_lat", ccap);
      tc.s_occ = ctx->d<double>("a.yc_occw", ccap);
      tc.s_flops = ctx->d<uint64_t>("a.yc_sum", ccap);
      tc.s_read = ctx->d<uint64_t>("a.yc_r", ccap);
      tc.s_write = ctx->d<uint64_t>("a.yc_w", ccap);
      k_names_fast<<<nlc, NAME_WARPS * 32, kNameRawSmem, st>>>(tc);
      NameBigArgs yb;
      yb.G = G;
      yb.gkc_off = d_glc_rel;
      yb.gstatus = out->group_status;
      yb.c_count = tc.g_count;
      yb.c_name = tc.s_name;
      yb.c_cnt = tc.s_count;
      yb.c_lat = tc.s_lat;
      yb.c_occw = tc.s_occ;
      yb.c_f = tc.s_flops;
      yb.c_r = tc.s_read;
      yb.c_w = tc.s_write;
      yb.m_lat = ma.m_lat;
      yb.peak = la.peak;
      yb.bw = la.bw;
      yb.g_count = ty.g_count;
      yb.overflow = ty.overflow;
      yb.s_name = ty.s_name;
      yb.s_count = ty.s_count;
      yb.s_lat = ty.s_lat;
      yb.s_pct = ty.s_pct;
      yb.s_flops = ty.s_flops;
      yb.s_read = ty.s_read;
      yb.s_write = ty.s_write;
      yb.s_occ = ty.s_occ;
      yb.s_ai = ty.s_ai;
      yb.s_tput = ty.s_tput;
      yb.s_bound = ty.s_bound;
      fold_big(yb, d_pl, d_pl_off, npl, pl_off, "a.yp", st);
      ++ctx->launches;
    }
    exclusive_scan<uint32_t, uint32_t>(ty.g_count, out->group_type_off, G, ctx->d<uint32_t>("a.scan_y", scan_scratch_elems(G + 16)), out->group_type_off + G, st,
                                       &ctx->launches);
    xfer_small(htot + 4, out->group_type_off + G, 4, st);
    xfer_small(htot + 5, ty.overflow, 4, st);
    return;
  };
  auto place_types = [&]() {
    if (htot[5] && !types_wide) {  // more than 32 types somewhere: redo with 128-wide tables
      types_wide = true;
      run_types(st);
      XSP_CUDA(cudaStreamSynchronize(st));
    }
    if (htot[5]) throw std::invalid_argument("a5: more than 128 distinct layer types in one analysis group");
    const uint32_t NY = G ? htot[4] : 0;
    out->n_type_rows = NY;
    out->y_type = ctx->d<uint32_t>("t.y_type", NY);
    out->y_count = ctx->d<uint64_t>("t.y_count", NY);
    out->y_lat = ctx->d<double>("t.y_lat", NY);
    out->y_alloc = ctx->d<int64_t>("t.y_alloc", NY);
    if (!G) {
      XSP_CUDA(cudaMemsetAsync(out->group_type_off, 0, 4, st));
      return;
    }
    k_types_place<<<G, 128, 0, st>>>(G, out->group_type_off, ctx->d<uint32_t>("a.y_s_key", 1),
                                     ctx->d<uint64_t>("a.y_s_count", 1), ctx->d<double>("a.y_s_lat", 1),
                                     ctx->d<uint64_t>("a.y_s_sum", 1), out->y_type, out->y_count, out->y_lat,
                                     out->y_alloc);
    ++ctx->launches;
  };
  bool types_done = false;

  // ---- a10
  out->group_name_off = ctx->d<uint32_t>("t.g_noff", G + 1);
  uint32_t NN = 0;
  bool names_done = false;
  if (TK && G) {
    ctx->stage_begin("names", sn);
    NameFastArgs nf;
    nf.G = G;
    nf.gk_off = out->group_kernel_off;
    nf.gstatus = out->group_status;
    nf.k_name = la.k_name;
    nf.k_lat = la.k_lat;
    nf.k_occ = la.k_occ;
    nf.k_flops = la.k_flops;
    nf.k_read = la.k_read;
    nf.k_write = la.k_write;
    nf.m_lat = ma.m_lat;
    nf.peak = la.peak;
    nf.bw = la.bw;
    nf.g_count = ctx->d<uint32_t>("a.ng_count", G + 1);
    nf.overflow = ctx->d<uint32_t>("a.n_over", 1);
    nf.ks_slot = ctx->d<uint32_t>("a.ks_slot", TK);
    nf.ks_rank = ctx->d<uint32_t>("a.ks_rank", TK);
    nf.perm = ctx->d<uint32_t>("a.perm", TK);
    const uint64_t cap = (uint64_t)G * NCAP;
    nf.s_name = ctx->d<uint32_t>("a.s_name", cap);
    nf.s_count = ctx->d<uint64_t>("a.s_count", cap);
    nf.s_lat = ctx->d<double>("a.s_lat", cap);
    nf.s_pct = ctx->d<double>("a.s_pct", cap);
    nf.s_flops = ctx->d<uint64_t>("a.s_flops", cap);
    nf.s_read = ctx->d<uint64_t>("a.s_read", cap);
    nf.s_write = ctx->d<uint64_t>("a.s_write", cap);
    nf.s_occ = ctx->d<double>("a.s_occ", cap);
    nf.s_ai = ctx->d<double>("a.s_ai", cap);
    nf.s_tput = ctx->d<double>("a.s_tput", cap);
    nf.s_bound = ctx->d<int8_t>("a.s_bound", cap);
    nf.gk_end = nullptr;
    nf.big = d_gkc;
    nf.raw = 0;
    XSP_CUDA(cudaMemsetAsync(nf.overflow, 0, 4, sn));
    XSP_CUDA(cudaFuncSetAttribute(k_names_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kNameSmem));
    k_names_fast<<<G, NAME_WARPS * 32, kNameSmem, sn>>>(nf);
    ++ctx->launches;
    if (nkc) {
      // long groups: raw per-name sums per kernel chunk, then folded in order
      NameFastArgs nc = nf;
      nc.G = nkc;
      nc.gk_off = d_kcb;
      nc.gk_end = d_kce;
      nc.big = nullptr;
      nc.gstatus = nullptr;
      nc.raw = 1;
      const uint64_t ccap = (uint64_t)nkc * NCAP;
      nc.g_count = ctx->d<uint32_t>("a.c_count", nkc);
      nc.s_name = ctx->d<uint32_t>("a.c_name", ccap);
      nc.s_count = ctx->d<uint64_t>("a.c_cnt", ccap);
      nc.s_lat = ctx->d<double>("a.c_lat", ccap);
      nc.s_occ = ctx->d<double>("a.c_occw", ccap);
      nc.s_flops = ctx->d<uint64_t>("a.c_f", ccap);
      nc.s_read = ctx->d<uint64_t>("a.c_r", ccap);
      nc.s_write = ctx->d<uint64_t>("a.c_w", ccap);
      k_names_fast<<<nkc, NAME_WARPS * 32, kNameRawSmem, sn>>>(nc);
      NameBigArgs nb;
      nb.G = G;
      nb.gkc_off = d_gkc;
      nb.gstatus = out->group_status;
      nb.c_count = nc.g_count;
      nb.c_name = nc.s_name;
      nb.c_cnt = nc.s_count;
      nb.c_lat = nc.s_lat;
      nb.c_occw = nc.s_occ;
      nb.c_f = nc.s_flops;
      nb.c_r = nc.s_read;
      nb.c_w = nc.s_write;
      nb.m_lat = ma.m_lat;
      nb.peak = la.peak;
      nb.bw = la.bw;
      nb.g_count = nf.g_count;
      nb.overflow = nf.overflow;
      nb.s_name = nf.s_name;
      nb.s_count = nf.s_count;
      nb.s_lat = nf.s_lat;
      nb.s_pct = nf.s_pct;
      nb.s_flops = nf.s_flops;
      nb.s_read = nf.s_read;
      nb.s_write = nf.s_write;
      nb.s_occ = nf.s_occ;
      nb.s_ai = nf.s_ai;
      nb.s_tput = nf.s_tput;
      nb.s_bound = nf.s_bound;
      fold_big(nb, d_pk, d_pk_off, npk, pk_off, "a.np", sn);
      ++ctx->launches;
    }
    exclusive_scan<uint32_t, uint32_t>(nf.g_count, out->group_name_off, G, scan_tmp, out->group_name_off + G, sn,
                                       &ctx->launches);
    xfer_small(htot + 2, out->group_name_off + G, 4, sn);
    xfer_small(htot + 3, nf.overflow, 4, sn);
    run_types(sy);
    types_done = true;
    if (fork) {  // join the side streams
      XSP_CUDA(cudaEventRecord(ctx->join_event(0), sn));
      XSP_CUDA(cudaEventRecord(ctx->join_event(1), sy));
      XSP_CUDA(cudaStreamWaitEvent(st, ctx->join_event(0), 0));
      XSP_CUDA(cudaStreamWaitEvent(st, ctx->join_event(1), 0));
    }
    XSP_CUDA(cudaStreamSynchronize(st));
    place_types();
    if (!htot[3]) {
      NN = htot[2];
      out->n_name = ctx->d<uint32_t>("t.n_name", NN);
      out->n_count = ctx->d<uint64_t>("t.n_count", NN);
      out->n_lat = ctx->d<double>("t.n_lat", NN);
      out->n_pct = ctx->d<double>("t.n_pct", NN);
      out->n_flops = ctx->d<uint64_t>("t.n_flops", NN);
      out->n_read = ctx->d<uint64_t>("t.n_read", NN);
      out->n_write = ctx->d<uint64_t>("t.n_write", NN);
      out->n_occ = ctx->d<double>("t.n_occ", NN);
      out->n_ai = ctx->d<double>("t.n_ai", NN);
      out->n_tput = ctx->d<double>("t.n_tput", NN);
      out->n_bound = ctx->d<int8_t>("t.n_bound", NN);
      const uint32_t* o = out->group_name_off;
      NamePlaceArgs pa{G, o, nf.s_name, nf.s_count, nf.s_lat, nf.s_pct, nf.s_flops, nf.s_read, nf.s_write,
                       nf.s_occ, nf.s_ai, nf.s_tput, nf.s_bound, out->n_name, out->n_count, out->n_lat,
                       out->n_pct, out->n_flops, out->n_read, out->n_write, out->n_occ, out->n_ai,
                       out->n_tput, out->n_bound};
      k_names_place_all<<<G, 128, 0, st>>>(pa);
      ctx->launches += 1;
      names_done = true;
    }
    ctx->stage_end("names", st);
  }
  if (TK && !names_done) {
    ctx->stage_begin("names", st);
    uint64_t* key = ctx->d<uint64_t>("a.nkey", TK);
    uint32_t* val = ctx->d<uint32_t>("a.nval", TK);
    launch(ctx, k_name_keys, TK, st, TK, out->group_kernel_off, G, la.k_name, out->group_status, key, val);
    RadixScratch rs;
    rs.keys_alt = ctx->d<uint64_t>("rs.keys_alt", TK);
    rs.vals_alt = ctx->d<uint32_t>("rs.vals_alt", TK);
    uint64_t ce = radix_counts_elems(TK);
    rs.counts = ctx->d<uint32_t>("rs.counts", ce);
    rs.scan_tmp = ctx->d<uint32_t>("rs.scan", scan_scratch_elems(ce));
    rs.and_or = ctx->d<unsigned long long>("rs.andor", 2);
    rs.and_or_host = ctx->h<unsigned long long>("rs.andor_h", 2);
    radix_sort_pairs(key, val, TK, 0, 64, rs, st, &ctx->launches);
    uint32_t* flag = ctx->d<uint32_t>("a.nflag", TK);
    uint32_t* pos = ctx->d<uint32_t>("a.npos", TK + 1);
    launch(ctx, k_seg_flags, TK, st, TK, key, flag);
    uint32_t* scan2 = ctx->d<uint32_t>("a.scan2", scan_scratch_elems(TK + 16));
    exclusive_scan<uint32_t, uint32_t>(flag, pos, TK, scan2, pos + TK, st, &ctx->launches);
    xfer_small(htot + 2, pos + TK, 4, st);
    XSP_CUDA(cudaStreamSynchronize(st));
    NN = htot[2];
    NameArgs na;
    na.n = TK;
    na.key = key;
    na.val = val;
    na.seg_pos = pos;
    na.flag = flag;
    na.k_lat = la.k_lat;
    na.k_occ = la.k_occ;
    na.k_flops = la.k_flops;
    na.k_read = la.k_read;
    na.k_write = la.k_write;
    na.m_lat = ma.m_lat;
    na.peak = la.peak;
    na.bw = la.bw;
    na.s_group = ctx->d<uint32_t>("a.s_group", NN);
    na.s_name = ctx->d<uint32_t>("a.s_name", NN);
    na.s_count = ctx->d<uint64_t>("a.s_count", NN);
    na.s_lat = ctx->d<double>("a.s_lat", NN);
    na.s_pct = ctx->d<double>("a.s_pct", NN);
    na.s_flops = ctx->d<uint64_t>("a.s_flops", NN);
    na.s_read = ctx->d<uint64_t>("a.s_read", NN);
    na.s_write = ctx->d<uint64_t>("a.s_write", NN);
    na.s_occ = ctx->d<double>("a.s_occ", NN);
    na.s_ai = ctx->d<double>("a.s_ai", NN);
    na.s_tput = ctx->d<double>("a.s_tput", NN);
    na.s_bound = ctx->d<int8_t>("a.s_bound", NN);
    launch(ctx, k_name_rows, TK, st, na);
    launch(ctx, k_csr_groups, (uint64_t)G + 1, st, G, NN, na.s_group, out->group_name_off);
    uint32_t* order = ctx->d<uint32_t>("a.norder", NN);
    launch(ctx, k_name_order, G, st, G, out->group_name_off, na.s_lat, order);
    out->n_name = ctx->d<uint32_t>("t.n_name", NN);
    out->n_count = ctx->d<uint64_t>("t.n_count", NN);
    out->n_lat = ctx->d<double>("t.n_lat", NN);
    out->n_pct = ctx->d<double>("t.n_pct", NN);
    out->n_flops = ctx->d<uint64_t>("t.n_flops", NN);
    out->n_read = ctx->d<uint64_t>("t.n_read", NN);
    out->n_write = ctx->d<uint64_t>("t.n_write", NN);
    out->n_occ = ctx->d<double>("t.n_occ", NN);
    out->n_ai = ctx->d<double>("t.n_ai", NN);
    out->n_tput = ctx->d<double>("t.n_tput", NN);
    out->n_bound = ctx->d<int8_t>("t.n_bound", NN);
    launch(ctx, k_permute<uint32_t>, NN, st, NN, order, na.s_name, out->n_name);
    launch(ctx, k_permute<uint64_t>, NN, st, NN, order, na.s_count, out->n_count);
    launch(ctx, k_permute<double>, NN, st, NN, order, na.s_lat, out->n_lat);
    launch(ctx, k_permute<double>, NN, st, NN, order, na.s_pct, out->n_pct);
    launch(ctx, k_permute<uint64_t>, NN, st, NN, order, na.s_flops, out->n_flops);
    launch(ctx, k_permute<uint64_t>, NN, st, NN, order, na.s_read, out->n_read);
    launch(ctx, k_permute<uint64_t>, NN, st, NN, order, na.s_write, out->n_write);
    launch(ctx, k_permute<double>, NN, st, NN, order, na.s_occ, out->n_occ);
    launch(ctx, k_permute<double>, NN, st, NN, order, na.s_ai, out->n_ai);
    launch(ctx, k_permute<double>, NN, st, NN, order, na.s_tput, out->n_tput);
    launch(ctx, k_permute<int8_t>, NN, st, NN, order, na.s_bound, out->n_bound);
    ctx->stage_end("names", st);
  } else if (!names_done) {
    XSP_CUDA(cudaMemsetAsync(out->group_name_off, 0, (G + 1) * 4ull, st));
    out->n_name = ctx->d<uint32_t>("t.n_name", 1);
    out->n_count = ctx->d<uint64_t>("t.n_count", 1);
    out->n_lat = ctx->d<double>("t.n_lat", 1);
    out->n_pct = ctx->d<double>("t.n_pct", 1);
    out->n_flops = ctx->d<uint64_t>("t.n_flops", 1);
    out->n_read = ctx->d<uint64_t>("t.n_read", 1);
    out->n_write = ctx->d<uint64_t>("t.n_write", 1);
    out->n_occ = ctx->d<double>("t.n_occ", 1);
    out->n_ai = ctx->d<double>("t.n_ai", 1);
    out->n_tput = ctx->d<double>("t.n_tput", 1);
    out->n_bound = ctx->d<int8_t>("t.n_bound", 1);
  }
  out->n_names = NN;
  if (!types_done) {
    run_types(st);
    XSP_CUDA(cudaStreamSynchronize(st));
    place_types();
  }
}

}  // namespace xsp
