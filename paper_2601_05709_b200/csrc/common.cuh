// Shared device/host utilities for liblsgpu (sm_100a).
//
// Deterministic reductions: every reducing kernel writes one partial per CTA
// (warp-shuffle tree + fixed-order combine of the per-warp values), and the
// last CTA to finish (threadfence + atomic ticket) sums the partials in index
// order.  No floating-point atomics anywhere, so results are bitwise
// reproducible run to run -- the property the reference asserts for its
// serial vs threaded runs (test_driver.py:183-199, test_acceptance.py:467-483).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lsgpu.h"

namespace lsg {

void set_error(const char *fmt, ...);
int check_launch(const char *what);

constexpr int kWarp = 32;

// SM count of the current device (queried once per device): grids are sized in
// multiples of it, and a cooperative grid may not exceed it times the CTAs per SM.
int num_sms();
// L2 capacity of the current device in bytes (queried once per device).
int64_t l2_bytes();

// Programmatic dependent launch (PDL) for the PCG-iteration kernels: a kernel
// launched with launch_pdl may have its CTAs scheduled while its predecessor
// on the stream is still draining (hiding the launch and CTA-rasterisation
// latency of the kernel boundary); it calls pdl_wait() before it reads
// anything its predecessor wrote, which returns once that grid has completed
// and its memory is visible.  The predecessor triggers implicitly at exit, so
// a waiting CTA never holds an SM a predecessor CTA still needs.  Outside a
// programmatic dependency pdl_wait() is a no-op.  LSG_NO_PDL=1 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Asynchronous global -> shared copies (LDGSTS): staged prefetch that costs no
// registers; .cg (16 bytes) bypasses L1, so it is coherent with data written
// earlier in the same launch across a grid barrier.
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Reduce NV values over the CTA; slot v uses max when bit v of MAXMASK is set.
// Result is valid in thread 0.  `scratch` holds NV * (blockDim/32) doubles.
template <int NV, unsigned MAXMASK>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double *scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i] = ((MAXMASK >> i) & 1u) ? warp_max(v[i]) : warp_sum(v[i]);
    if (lane == 0) scratch[i * nw + warp] = v[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double acc = scratch[i * nw];
      for (int w = 1; w < nw; ++w)
        acc = ((MAXMASK >> i) & 1u) ? fmax(acc, scratch[i * nw + w]) : acc + scratch[i * nw + w];
      v[i] = acc;
    }
  }
  __syncthreads();
}

// Store this CTA's partial and, in the last CTA of the group, return the
// fixed-order total of all partials in `total` (valid in thread 0 of the
// last CTA only).  Returns true in every thread of the last CTA.
//   partials: nblk * NV doubles for this group; counter: one uint per group.
template <int NV, unsigned MAXMASK>
__device__ bool block_partial_and_total(double (&v)[NV], double *partials, uint32_t *counter,
                                        int blk, int nblk, double *scratch, double (&total)[NV]) {
  __shared__ bool am_last;
  block_reduce<NV, MAXMASK>(v, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) partials[(size_t)blk * NV + i] = v[i];
    __threadfence();
    unsigned ticket = atomicAdd(counter, 1u);
    am_last = (ticket == (unsigned)(nblk - 1));
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  // Fixed assignment: thread t sums blocks t, t+T, ... in order; then the
  // same fixed tree as block_reduce.
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = ((MAXMASK >> i) & 1u) ? -INFINITY : 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double x = __ldcg(partials + (size_t)b * NV + i);
      acc[i] = ((MAXMASK >> i) & 1u) ? fmax(acc[i], x) : acc[i] + x;
    }
  }
  block_reduce<NV, MAXMASK>(acc, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) total[i] = acc[i];
    *counter = 0u;  // re-arm for the next launch
  }
  return true;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace lsg
