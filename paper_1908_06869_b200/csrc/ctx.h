// Host-side context: device arena, pinned staging, launch accounting.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "xsp.h"

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define XSP_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t err_ = (call);                                                          \
    if (err_ != cudaSuccess)                                                            \
      throw CudaError(std::string(#call) + ": " + cudaGetErrorString(err_));            \
  } while (0)

struct xsp_ctx {
  int device = 0;
  // NCCL communicator of the multi-GPU table combine (xsp_comm_init)
  void* nccl_comm = nullptr;
  int comm_world = 0, comm_rank = 0;
  void (*comm_destroy)(void*) = nullptr;
  std::string last_error;
  uint64_t launches = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;

  struct Buf {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> dev;
  std::map<std::string, Buf> host;  // pinned

  // ---- optional per-stage timing with CUDA events on the launching stream
  struct Stage {
    std::string name;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;  // pending (begin, end) pairs
    double ms = 0.0;
    uint64_t calls = 0;
  };
  bool profiling = false;
  uint32_t host_out = 0;  // XSP_HOST_OUT_* (xsp_set_host_outputs)
  std::vector<Stage> stages;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t take_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) throw CudaError("cudaEventCreate failed");
    return e;
  }
  Stage& stage(const std::string& name) {
    for (auto& s : stages)
      if (s.name == name) return s;
    stages.push_back(Stage{name, {}, 0.0, 0});
    return stages.back();
  }
  // begin/end of a named stage on stream st (no-ops unless profiling)
  void stage_begin(const std::string& name, cudaStream_t st) {
    if (!profiling) return;
    cudaEvent_t b = take_event();
    cudaEventRecord(b, st);
    stage(name).ev.push_back({b, nullptr});
  }
  void stage_end(const std::string& name, cudaStream_t st) {
    if (!profiling) return;
    cudaEvent_t e = take_event();
    cudaEventRecord(e, st);
    stage(name).ev.back().second = e;
  }
  // resolve pending events into milliseconds
  void stage_collect() {
    for (auto& s : stages) {
      for (auto& [b, e] : s.ev) {
        float ms = 0.f;
        if (e) {
          cudaEventSynchronize(e);
          cudaEventElapsedTime(&ms, b, e);
          event_pool.push_back(e);
        }
        event_pool.push_back(b);
        s.ms += ms;
        ++s.calls;
      }
      s.ev.clear();
    }
  }

  // Host copies of the last correlation's per-trace layer / kernel offsets,
  // fetched at its final read-back: xsp_analyze on that correlation sizes its
  // group tables on the host instead of with another device round trip.
  // capacities the rare-entry lists of correlate needed (grow-only hints)
  uint64_t cap_orph = 0, cap_amb = 0, cap_pend = 0;
  // correlate tries pass 1 in direct mode (kernel table written by pass 1) while
  // the previous call on this context was a clean batch (a guess: a wrong one
  // costs a second pass 1, never a different result)
  bool direct_hint = true;
  bool unclean_hint = false;

  const void* hc_layer_key = nullptr;
  const void* hc_kernel_key = nullptr;
  uint32_t hc_T = 0;

  // Suffix appended to every device buffer name while set: the chunked host
  // pipeline runs consecutive chunks on two disjoint buffer sets, so one
  // chunk's results can stream out while the next chunk computes.
  std::string tag;
  // Grow-only named device buffer with at least `bytes` bytes.
  void* dbuf(const std::string& name_, size_t bytes) {
    if (bytes == 0) bytes = 16;
    Buf& b = dev[tag.empty() ? name_ : name_ + tag];
    const std::string& name = name_;
    if (b.bytes < bytes) {
      if (b.ptr) cudaFree(b.ptr);
      b.ptr = nullptr;
      size_t want = bytes + bytes / 8;
      if (cudaMalloc(&b.ptr, want) != cudaSuccess) {
        b.bytes = 0;
        throw CudaError("cudaMalloc of " + std::to_string(want) + " bytes for '" + name + "' failed");
      }
      b.bytes = want;
    }
    return b.ptr;
  }
  template <typename T>
  T* d(const std::string& name, uint64_t count) {
    return static_cast<T*>(dbuf(name, count * sizeof(T)));
  }
  void* hbuf(const std::string& name, size_t bytes) {
    if (bytes == 0) bytes = 16;
    Buf& b = host[name];
    if (b.bytes < bytes) {
      if (b.ptr) cudaFreeHost(b.ptr);
      b.ptr = nullptr;
      size_t want = bytes + bytes / 8;
      if (cudaHostAlloc(&b.ptr, want, cudaHostAllocDefault) != cudaSuccess) {
        b.bytes = 0;
        throw CudaError("cudaHostAlloc of " + std::to_string(want) + " bytes failed");
      }
      b.bytes = want;
    }
    return b.ptr;
  }
  template <typename T>
  T* h(const std::string& name, uint64_t count) {
    return static_cast<T*>(hbuf(name, count * sizeof(T)));
  }
  // Pinned buffer with at least `bytes`, preserving its first `keep` bytes when
  // it has to grow (callers make sure no copy into it is in flight).
  void* hbuf_keep(const std::string& name, size_t bytes, size_t keep) {
    Buf& b = host[name];
    if (b.bytes >= bytes && b.ptr) return b.ptr;
    size_t want = bytes + bytes / 2 + 4096;
    void* p = nullptr;
    if (cudaHostAlloc(&p, want, cudaHostAllocDefault) != cudaSuccess)
      throw CudaError("cudaHostAlloc of " + std::to_string(want) + " bytes failed");
    if (b.ptr) {
      if (keep) std::memcpy(p, b.ptr, keep < b.bytes ? keep : b.bytes);
      cudaFreeHost(b.ptr);
    }
    b.ptr = p;
    b.bytes = want;
    return p;
  }
  size_t hcap(const std::string& name) {
    auto it = host.find(name);
    return it == host.end() ? 0 : it->second.bytes;
  }
  // ctx-owned non-blocking streams for the chunked host pipeline
  cudaStream_t copy_stream = nullptr, work_stream = nullptr, out_stream = nullptr;
  cudaStream_t stream_copy() {
    if (!copy_stream && cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking) != cudaSuccess)
      throw CudaError("cudaStreamCreate failed");
    return copy_stream;
  }
  cudaStream_t stream_out() {
    if (!out_stream && cudaStreamCreateWithFlags(&out_stream, cudaStreamNonBlocking) != cudaSuccess)
      throw CudaError("cudaStreamCreate failed");
    return out_stream;
  }
  cudaStream_t stream_work() {
    if (!work_stream && cudaStreamCreateWithFlags(&work_stream, cudaStreamNonBlocking) != cudaSuccess)
      throw CudaError("cudaStreamCreate failed");
    return work_stream;
  }
  // side streams + events for fork/join inside one API call (xsp_analyze runs
  // its a15 / a10 / a5 passes concurrently); ordered with the caller's stream
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
  cudaStream_t side_stream(int i) {
    if (!side[i] && cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking) != cudaSuccess)
      throw CudaError("cudaStreamCreate failed");
    return side[i];
  }
  static cudaEvent_t lazy_event(cudaEvent_t& e) {
    if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      throw CudaError("cudaEventCreate failed");
    return e;
  }
  cudaEvent_t fork_event() { return lazy_event(ev_fork); }
  cudaEvent_t join_event(int i) { return lazy_event(ev_join[i]); }
  ~xsp_ctx() {
    stage_collect();
    if (nccl_comm && comm_destroy) comm_destroy(nccl_comm);
    for (cudaStream_t& s : side)
      if (s) cudaStreamDestroy(s);
    if (ev_fork) cudaEventDestroy(ev_fork);
    for (cudaEvent_t& e : ev_join)
      if (e) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (work_stream) cudaStreamDestroy(work_stream);
    if (out_stream) cudaStreamDestroy(out_stream);
    for (cudaEvent_t e : event_pool) cudaEventDestroy(e);
    for (auto& [k, b] : dev)
      if (b.ptr) cudaFree(b.ptr);
    for (auto& [k, b] : host)
      if (b.ptr) cudaFreeHost(b.ptr);
  }
};

namespace xsp {
void run_correlate(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_traces* traces,
                   int sort_if_needed, xsp_corr_out* out, cudaStream_t st);
void run_analyze(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                 const xsp_groups* groups, const xsp_system_spec* spec,
                 const xsp_analysis_opts* opts, xsp_tables_out* out, cudaStream_t st);
void run_leveled(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr,
                 const xsp_level_sets* sets, const xsp_analysis_opts* opts, xsp_overhead_out* out,
                 cudaStream_t st);
void run_leveled_batch(xsp_ctx* ctx, const xsp_span_cols* cols, const xsp_corr_out* corr, uint32_t n_groups,
                       const xsp_level_sets* sets, const xsp_analysis_opts* opts, xsp_overhead_out* outs,
                       cudaStream_t st);
}  // namespace xsp
