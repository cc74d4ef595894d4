// Shared device helpers for the xsp CUDA path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "xsp.h"

namespace xsp {

constexpr uint32_t kNone = 0xFFFFFFFFu;

// flags byte layout (include/xsp.h)
__host__ __device__ __forceinline__ uint32_t f_level(uint8_t f) { return f & 3u; }
__host__ __device__ __forceinline__ uint32_t f_kind(uint8_t f) { return (f >> 2) & 3u; }

// Span role predicates, each mirroring a reference helper.
// is_kernel_launch: correlator.cpp:32-35
__host__ __device__ __forceinline__ bool is_kernel_launch(uint8_t f) {
  return f_kind(f) == XSP_KIND_LAUNCH && f_level(f) >= XSP_LEVEL_KERNEL;
}
// is_exec: correlator.cpp:37 (any level)
__host__ __device__ __forceinline__ bool is_exec(uint8_t f) { return f_kind(f) == XSP_KIND_EXEC; }
// is_sync_kernel: correlator.cpp:40-42
__host__ __device__ __forceinline__ bool is_sync_kernel(uint8_t f) {
  return f_kind(f) == XSP_KIND_SYNC && f_level(f) == XSP_LEVEL_KERNEL;
}
// TraceBundle::model_span: span.cpp:298-303
__host__ __device__ __forceinline__ bool is_model_span(uint8_t f) {
  return f_kind(f) == XSP_KIND_SYNC && f_level(f) == XSP_LEVEL_MODEL;
}
// Span::duration_ns: span.hpp:93-95 (clamped)
__host__ __device__ __forceinline__ uint64_t clamp_dur(uint64_t b, uint64_t e) {
  return e >= b ? e - b : 0;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Last trace t with off[t] <= i, searching t in [lo, hi) (off has n_traces+1
// entries; empty traces are skipped because off[t] == off[t+1]).
// Lanes of `valid` holding the same 8-bit value as this lane: one ballot per
// bit (warp multisplit). Several times cheaper than __match_any_sync here.
__device__ __forceinline__ uint32_t match8(uint32_t d, uint32_t valid) {
  uint32_t m = valid;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t bit = (d >> b) & 1u;
    const uint32_t v = __ballot_sync(0xffffffffu, bit);
    m &= bit ? v : ~v;
  }
  return m;
}

__device__ __forceinline__ uint32_t trace_of(const uint64_t* __restrict__ off, uint32_t lo,
                                             uint32_t hi, uint64_t i) {
  // invariant: off[lo] <= i < off[hi]
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= i) lo = mid; else hi = mid;
  }
  return lo;
}

inline unsigned ceil_div(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

}  // namespace xsp
