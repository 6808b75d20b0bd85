// Shared helpers for the sm_100a sparse cross-encoder library.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/sparsecross_b200.h"

namespace sc {

// Thread-local last-error string behind sc_last_error().
void set_error(const char* fmt, ...);

#define SC_CHECK_ARG(cond, ...)                 \
  do {                                          \
    if (!(cond)) {                              \
      ::sc::set_error(__VA_ARGS__);             \
      return SC_ERR_INVALID;                    \
    }                                           \
  } while (0)

// Process-wide count of kernels this library launched (sc_kernel_launches()).
void count_launch();

#define SC_CHECK_LAUNCH(name)                                                      \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      ::sc::set_error("%s: CUDA launch failed: %s", name, cudaGetErrorString(_e)); \
      return SC_ERR_CUDA;                                                          \
    }                                                                              \
    ::sc::count_launch();                                                          \
  } while (0)

// Link encoding of the attention pattern (src x tgt), see sparsecross_b200.h.
struct Links {
  int32_t w[3][3];
};

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sequence lookup: largest j with cu[j] <= row (cu has nseq+1 entries).
__device__ __forceinline__ int find_seq(const int32_t* __restrict__ cu, int nseq, int row) {
  int lo = 0, hi = nseq - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(cu + mid) <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Group lengths of sequence j in the packed layout: cls = 1, query = qlen, doc = rest.
struct SeqGroups {
  int start;    // first token row of the sequence
  int len[3];   // group lengths (cls, query, doc)
  int off[3];   // group offsets relative to start
};

__device__ __forceinline__ SeqGroups seq_groups(const int32_t* __restrict__ cu,
                                                const int32_t* __restrict__ qlen, int j) {
  SeqGroups g;
  g.start = __ldg(cu + j);
  int s = __ldg(cu + j + 1) - g.start;
  int m = __ldg(qlen + j);
  g.len[0] = 1; g.len[1] = m; g.len[2] = s - 1 - m;
  g.off[0] = 0; g.off[1] = 1; g.off[2] = 1 + m;
  return g;
}

}  // namespace sc
