// Host-side context: device arena, pinned staging, launch accounting.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>

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
  std::string last_error;
  uint64_t launches = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;

  struct Buf {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> dev;
  std::map<std::string, Buf> host;  // pinned

  // Grow-only named device buffer with at least `bytes` bytes.
  void* dbuf(const std::string& name, size_t bytes) {
    if (bytes == 0) bytes = 16;
    Buf& b = dev[name];
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
  ~xsp_ctx() {
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
}  // namespace xsp
