// lg_common.cuh -- shared device/host helpers of liblapb200.
//
// Everything HBM-bound here follows one rule: stream each input once with
// coalesced loads, keep partial sums in registers, and finish reductions with
// a deterministic two-level tree (warp shuffles -> shared memory -> per-CTA
// partial in global memory -> the last CTA to arrive sums the partials in
// CTA order).  No floating-point atomics anywhere, so results are bitwise
// reproducible for a fixed grid.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/lapb200.h"

namespace lg {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define LG_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess)                                                   \
      return ::lg::fail(LG_ECUDA, std::string(#call) + ": " +                \
                                      cudaGetErrorString(_e));               \
  } while (0)

#define LG_LAUNCH_CHECK(name)                                                \
  do {                                                                       \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess)                                                   \
      return ::lg::fail(LG_ECUDA, std::string(name) + " launch: " +          \
                                      cudaGetErrorString(_e));               \
  } while (0)

// ------------------------------------------------------------ device info --
struct DevInfo {
  int sm_count = 148;
  int l2_bytes = 0;
  int major = 0, minor = 0;
};
const DevInfo& dev_info();

constexpr int kThreads = 256;                  // CTA size of vector kernels
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRedBlocks = 4096;            // upper bound on reducing CTAs
constexpr int kMaxRedVals = LG_MAXD + LG_MAXQ; // values reduced per launch

}  // namespace lg

// Reduction workspace: per-CTA partials + arrival ticket.  One per stream.
struct lg_ws {
  double* partial = nullptr;   // [kMaxRedBlocks * kMaxRedVals]
  unsigned* ticket = nullptr;  // [1]
  // SpMV long-row scratch (grown on demand to the largest matrix used)
  double* long_dots = nullptr;    // [long_cap * kMaxRedVals] epilogue dots
  unsigned* long_ticket = nullptr;  // [long_cap] arrival tickets (kept 0)
  int64_t long_cap = 0;           // capacity in long rows
  double* long_part = nullptr;    // [part_cap] partial sum of each part
  int64_t part_cap = 0;
  double* mm_part = nullptr;      // [mm_cap] long-row part partials of the SpMM
  int64_t mm_cap = 0;
};

namespace lg {

// --------------------------------------------------------- load helpers --
// Streaming loads (read once): keep them out of L1.
__device__ __forceinline__ double ld_stream(const double* p) {
  return __ldcs(p);
}
__device__ __forceinline__ int ld_stream(const int* p) { return __ldcs(p); }
// Coherent-at-L2 load (data written by other CTAs during this launch).
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Number of CTAs a grid-stride vector kernel uses for n rows: enough to fill
// the machine (4 CTAs of 256 threads per SM) but never more than the rows
// need.  Depends on n only, so the reduction tree is fixed per size.
inline int vec_grid(int64_t n) {
  // at least two elements per thread for small n; at most 4 CTAs per SM
  // (the grid-stride loop is unrolled with non-coherent loads, so a
  // thread keeps several elements in flight and the final cross-CTA
  // reduction stays short)
  int64_t want = (n + kThreads * 2 - 1) / (kThreads * 2);
  int64_t cap = (int64_t)dev_info().sm_count * 4;
  if (want < 1) want = 1;
  if (want > cap) want = cap;
  if (want > kMaxRedBlocks) want = kMaxRedBlocks;
  return (int)want;
}

// Deterministic grid reduction of `na` values held per thread in acc[].
// smem must hold kWarps * NA doubles.  The CTA that arrives last writes the
// totals to result[0:na] (summing per-CTA partials in CTA order) and then
// adds extra[e * stride_extra + d] for e < nextra (per-long-row slots of the
// SpMV) -- also in fixed order.  Returns true in the finishing CTA.
template <int NA>
__device__ __forceinline__ bool grid_reduce(double (&acc)[NA], int na,
                                            lg_ws ws, double* result,
                                            double* smem,
                                            const double* extra = nullptr,
                                            int64_t nextra = 0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int d = 0; d < NA; ++d) {
    if (d < na) {
      double v = warp_sum(acc[d]);
      if (lane == 0) smem[warp * NA + d] = v;
    }
  }
  __syncthreads();
  if (gridDim.x == 1 && nextra == 0) {
    // single CTA: the block sum is the result (same tree order as below)
    if ((int)threadIdx.x < na) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += smem[w * NA + threadIdx.x];
      // a one-element partial list summed lane-strided + butterfly equals s
      result[threadIdx.x] = s + 0.0;
    }
    return true;
  }
  if ((int)threadIdx.x < na) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += smem[w * NA + threadIdx.x];
    ws.partial[(int64_t)blockIdx.x * kMaxRedVals + threadIdx.x] = s;
  }
  __shared__ int am_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    // one acq_rel ticket instead of fence + atomic + fence: the release
    // publishes this CTA's partials (ordered before it by the barrier), the
    // acquire in the last CTA makes every partial visible to it
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(ws.ticket) : "memory");
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  const int nb = gridDim.x;
  for (int d = warp; d < na; d += nw) {
    // lane-strided partials, summed in increasing CTA order; the loads of
    // a batch are issued together (a dependent load-add chain would cost
    // one L2 round trip per 32 CTAs)
    double s = 0.0;
    for (int b0 = lane; b0 < nb; b0 += 32 * 16) {
      double v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int b = b0 + 32 * j;
        v[j] = b < nb ? ld_cg(ws.partial + (int64_t)b * kMaxRedVals + d) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (b0 + 32 * j < nb) s += v[j];
    }
    s = warp_sum(s);
    if (extra) {
      // long-row contributions, fixed order, lanes strided then tree
      double t = 0.0;
      for (int64_t e = lane; e < nextra; e += 32)
        t += ld_cg(extra + e * kMaxRedVals + d);
      s += warp_sum(t);
    }
    if (lane == 0) result[d] = s;
  }
  if (threadIdx.x == 0) *ws.ticket = 0u;
  return true;
}

}  // namespace lg
