// lg_build.cu -- Laplacian assembly on the device, bit-exact with
// graphs.py:250-263.
//
// The reference builds L = D - A from a canonical edge list (i < j, sorted by
// (i, j)) with np.add.at for the degrees and a COO lexsort for the CSR.  Row v
// of the result holds, in column order: the lower neighbours u < v (edges
// (u, v), ascending u), the diagonal, the upper neighbours w > v (edges
// (v, w), ascending w).  deg[v] is accumulated by np.add.at(deg, i, w)
// followed by np.add.at(deg, j, w), i.e. from 0.0 over the upper weights in
// ascending w and then the lower weights in ascending u -- the order used
// here, so degrees match bit for bit.
//
// Device plan (int32 node ids, int64 edge / nonzero offsets):
//   1. per-node counts of upper (as i) and lower (as j) incidences;
//   2. row lengths -> row_ptr (exclusive scan);
//   3. stable radix sort of edge ids by j gives every node's lower
//      neighbours in ascending u (the edge list is sorted by i);
//   4. scatter off-diagonals, then one thread per node sums its degree in the
//      reference order and writes the diagonal.
#include <cub/cub.cuh>
#include <vector>

#include "lg_common.cuh"

namespace lg {

__global__ void count_kernel(int64_t m, const int32_t* ei, const int32_t* ej,
                             int32_t* cnt_up, int32_t* cnt_lo) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    atomicAdd(cnt_up + ei[e], 1);
    atomicAdd(cnt_lo + ej[e], 1);
  }
}

__global__ void rowlen_kernel(int64_t n, const int32_t* cnt_up, const int32_t* cnt_lo,
                              int64_t* len, int64_t* up64, int64_t* lo64) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    len[v] = (int64_t)cnt_up[v] + cnt_lo[v] + 1;
    up64[v] = cnt_up[v];
    lo64[v] = cnt_lo[v];
  }
}

__global__ void scatter_upper_kernel(int64_t m, const int32_t* ei, const int32_t* ej,
                                     const double* w, const int64_t* rp,
                                     const int32_t* cnt_lo, const int64_t* ustart,
                                     int32_t* col, double* val) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    const int32_t v = ei[e];
    const int64_t p = rp[v] + cnt_lo[v] + 1 + (e - ustart[v]);
    col[p] = ej[e];
    val[p] = -w[e];
  }
}

__global__ void scatter_lower_kernel(int64_t m, const int32_t* sorted_j,
                                     const int64_t* perm, const int32_t* ei,
                                     const double* w, const int64_t* rp,
                                     const int64_t* lstart, int32_t* col, double* val) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
    const int32_t v = sorted_j[p];
    const int64_t e = perm[p];
    const int64_t q = rp[v] + (p - lstart[v]);
    col[q] = ei[e];
    val[q] = -w[e];
  }
}

// Degree of each node in the reference's order (graphs.py:253-254: np.add.at
// over the upper rows, then over the lower ones, from 0.0).  With integer
// weights every partial sum is an exact integer, so a row longer than
// kWideDeg may be summed by a whole warp (degree_wide_kernel) and still match
// bit for bit; otherwise every row is summed sequentially in that order.
constexpr int kWideDeg = 256;

__global__ void degree_kernel(int64_t n, const int64_t* ustart, const int32_t* cnt_up,
                              const int64_t* lstart, const int32_t* cnt_lo,
                              const int64_t* perm, const double* w, const int64_t* rp,
                              int32_t* col, double* val, int wide_ok) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    if (wide_ok && (int64_t)cnt_up[v] + cnt_lo[v] > kWideDeg) continue;
    double s = 0.0;
    const int64_t u0 = ustart[v], u1 = u0 + cnt_up[v];
    for (int64_t e = u0; e < u1; ++e) s += w[e];
    const int64_t l0 = lstart[v], l1 = l0 + cnt_lo[v];
    for (int64_t p = l0; p < l1; ++p) s += w[perm[p]];
    const int64_t q = rp[v] + cnt_lo[v];
    col[q] = (int32_t)v;
    val[q] = s;
  }
}

// long rows (integer weights only), cut into chunks of kDegChunk entries --
// one warp per (row, chunk): lane-strided partial sums and a butterfly, then
// one double atomicAdd per chunk into the row's (zeroed) diagonal slot.  Every
// partial and every sum is an integer below 2^53, so the result is exact and
// the same in any order (C4's 107,553-entry hub row no longer serialises on
// one warp).
constexpr int64_t kDegChunk = 2048;

__global__ void zero_diag_kernel(int64_t n, const int32_t* cnt_up, const int32_t* cnt_lo,
                                 const int64_t* rp, double* val) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    if ((int64_t)cnt_up[v] + cnt_lo[v] > kWideDeg) val[rp[v] + cnt_lo[v]] = 0.0;
}

__global__ void degree_wide_kernel(int64_t n, const int64_t* ustart, const int32_t* cnt_up,
                                   const int64_t* lstart, const int32_t* cnt_lo,
                                   const int64_t* perm, const double* w, const int64_t* rp,
                                   int32_t* col, double* val, const int64_t* crow,
                                   const int64_t* cfirst, int64_t nchunks) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nchunks; c += nw) {
    const int64_t v = crow[c];
    const int64_t k0 = (c - cfirst[c]) * kDegChunk;   // chunk's first entry in the row
    const int64_t nup = cnt_up[v], len = nup + cnt_lo[v];
    const int64_t k1 = min(len, k0 + kDegChunk);
    double s = 0.0;
    for (int64_t k = k0 + lane; k < k1; k += 32)
      s += k < nup ? w[ustart[v] + k] : w[perm[lstart[v] + (k - nup)]];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const int64_t q = rp[v] + cnt_lo[v];
      if (k0 == 0) col[q] = (int32_t)v;
      atomicAdd(val + q, s);
    }
  }
}

__global__ void iota_kernel(int64_t m, int64_t* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
    out[e] = e;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  ~DevBuf() { cudaFree(p); }
  bool alloc(size_t count) {
    return count == 0 || cudaMalloc(&p, sizeof(T) * count) == cudaSuccess;
  }
};

static inline int grid_for_n(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)dev_info().sm_count * 8;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

}  // namespace lg

using namespace lg;

extern "C" int lg_build_laplacian(int64_t n, int64_t m, const int64_t* i_h,
                                  const int64_t* j_h, const double* w_h,
                                  int64_t* rp_h, int64_t* col_h, double* val_h) {
  if (n < 1 || m < 0 || !rp_h || (m > 0 && (!i_h || !j_h || !w_h)) ||
      (n + 2 * m > 0 && (!col_h || !val_h)))
    return fail(LG_EINVAL, "lg_build_laplacian: bad argument");
  if (n >= ((int64_t)1 << 31)) return fail(LG_EINVAL, "lg_build_laplacian: n too large");
  std::vector<int32_t> hi32((size_t)m), hj32((size_t)m);
  for (int64_t e = 0; e < m; ++e) {
    if (i_h[e] < 0 || j_h[e] >= n || i_h[e] >= j_h[e])
      return fail(LG_EINVAL, "lg_build_laplacian: edges must satisfy 0 <= i < j < n");
    if (e > 0 && (i_h[e] < i_h[e - 1] || (i_h[e] == i_h[e - 1] && j_h[e] <= j_h[e - 1])))
      return fail(LG_EINVAL, "lg_build_laplacian: edges must be sorted and unique");
    hi32[(size_t)e] = (int32_t)i_h[e];
    hj32[(size_t)e] = (int32_t)j_h[e];
  }
  const int64_t nnz = n + 2 * m;
  DevBuf<int32_t> ei, ej, cnt_up, cnt_lo, sj, col;
  DevBuf<double> w, val;
  DevBuf<int64_t> len, up64, lo64, rp, ustart, lstart, perm_in, perm;
  bool ok = ei.alloc(m) && ej.alloc(m) && w.alloc(m) && cnt_up.alloc(n) &&
            cnt_lo.alloc(n) && sj.alloc(m) && col.alloc(nnz) && val.alloc(nnz) &&
            len.alloc(n) && up64.alloc(n) && lo64.alloc(n) && rp.alloc(n + 1) &&
            ustart.alloc(n) && lstart.alloc(n) && perm_in.alloc(m) && perm.alloc(m);
  if (!ok) return fail(LG_ENOMEM, "lg_build_laplacian: device allocation failed");
  cudaStream_t s = 0;
  if (m) {
    LG_CUDA(cudaMemcpy(ei.p, hi32.data(), 4 * (size_t)m, cudaMemcpyHostToDevice));
    LG_CUDA(cudaMemcpy(ej.p, hj32.data(), 4 * (size_t)m, cudaMemcpyHostToDevice));
    LG_CUDA(cudaMemcpy(w.p, w_h, 8 * (size_t)m, cudaMemcpyHostToDevice));
  }
  LG_CUDA(cudaMemset(cnt_up.p, 0, 4 * (size_t)n));
  LG_CUDA(cudaMemset(cnt_lo.p, 0, 4 * (size_t)n));
  if (m) count_kernel<<<grid_for_n(m), kThreads, 0, s>>>(m, ei.p, ej.p, cnt_up.p, cnt_lo.p);
  rowlen_kernel<<<grid_for_n(n), kThreads, 0, s>>>(n, cnt_up.p, cnt_lo.p, len.p, up64.p, lo64.p);
  LG_LAUNCH_CHECK("build counts");
  // scans: row_ptr (n+1 entries: rp[0] = 0), upper / lower starts
  LG_CUDA(cudaMemset(rp.p, 0, 8));
  size_t tmp_bytes = 0, t2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, len.p, rp.p + 1, (int)n, s);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, up64.p, ustart.p, (int)n, s);
  tmp_bytes = std::max(tmp_bytes, t2);
  if (m) {
    cub::DeviceRadixSort::SortPairs(nullptr, t2, ej.p, sj.p, perm_in.p, perm.p, (int)m, 0,
                                    32, s);
    tmp_bytes = std::max(tmp_bytes, t2);
  }
  DevBuf<unsigned char> tmp;
  if (!tmp.alloc(tmp_bytes)) return fail(LG_ENOMEM, "lg_build_laplacian: temp alloc failed");
  LG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tmp_bytes, len.p, rp.p + 1, (int)n, s));
  LG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, up64.p, ustart.p, (int)n, s));
  LG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, lo64.p, lstart.p, (int)n, s));
  if (m) {
    iota_kernel<<<grid_for_n(m), kThreads, 0, s>>>(m, perm_in.p);
    // stable LSD radix sort: ties keep edge order, i.e. ascending i
    LG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, ej.p, sj.p, perm_in.p,
                                            perm.p, (int)m, 0, 32, s));
    scatter_upper_kernel<<<grid_for_n(m), kThreads, 0, s>>>(m, ei.p, ej.p, w.p, rp.p,
                                                            cnt_lo.p, ustart.p, col.p,
                                                            val.p);
    scatter_lower_kernel<<<grid_for_n(m), kThreads, 0, s>>>(m, sj.p, perm.p, ei.p, w.p,
                                                            rp.p, lstart.p, col.p, val.p);
  }
  // integer weights (unit graphs, C4's counts): exact in any order, so hub
  // rows are summed by a warp each (C4's 107,553-entry row: 8 ms sequential)
  bool ints = true;
  double maxw = 0.0;
  for (int64_t e = 0; e < m && ints; ++e) {
    ints = w_h[e] == std::floor(w_h[e]);
    maxw = std::max(maxw, std::fabs(w_h[e]));
  }
  // every partial sum of a row is an integer of magnitude <= maxw * m < 2^53
  const int wide_ok = (ints && maxw * (double)m < 9.0e15) ? 1 : 0;
  degree_kernel<<<grid_for_n(n), kThreads, 0, s>>>(n, ustart.p, cnt_up.p, lstart.p,
                                                   cnt_lo.p, perm.p, w.p, rp.p, col.p,
                                                   val.p, wide_ok);
  if (wide_ok) {
    // chunk list of the long rows (host: the counts are small to copy)
    std::vector<int32_t> cu((size_t)n), cl((size_t)n);
    LG_CUDA(cudaMemcpy(cu.data(), cnt_up.p, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    LG_CUDA(cudaMemcpy(cl.data(), cnt_lo.p, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    std::vector<int64_t> crow, cfirst;
    std::vector<int64_t> qzero;
    for (int64_t v = 0; v < n; ++v) {
      const int64_t len = (int64_t)cu[(size_t)v] + cl[(size_t)v];
      if (len <= kWideDeg) continue;
      const int64_t first = (int64_t)crow.size();
      for (int64_t k = 0; k < len; k += kDegChunk) {
        crow.push_back(v);
        cfirst.push_back(first);
      }
    }
    if (!crow.empty()) {
      DevBuf<int64_t> dcrow, dcfirst;
      if (!dcrow.alloc(crow.size()) || !dcfirst.alloc(cfirst.size()))
        return fail(LG_ENOMEM, "lg_build_laplacian: chunk list alloc");
      LG_CUDA(cudaMemcpy(dcrow.p, crow.data(), 8 * crow.size(), cudaMemcpyHostToDevice));
      LG_CUDA(cudaMemcpy(dcfirst.p, cfirst.data(), 8 * cfirst.size(), cudaMemcpyHostToDevice));
      // the long rows' diagonal slots start from +0.0 (the chunks add into them)
      zero_diag_kernel<<<grid_for_n(n), kThreads, 0, s>>>(n, cnt_up.p, cnt_lo.p, rp.p, val.p);
      degree_wide_kernel<<<grid_for_n(32 * (int64_t)crow.size()), kThreads, 0, s>>>(
          n, ustart.p, cnt_up.p, lstart.p, cnt_lo.p, perm.p, w.p, rp.p, col.p, val.p, dcrow.p,
          dcfirst.p, (int64_t)crow.size());
      LG_CUDA(cudaDeviceSynchronize());
    }
  }
  LG_LAUNCH_CHECK("build scatter");
  LG_CUDA(cudaDeviceSynchronize());
  LG_CUDA(cudaMemcpy(rp_h, rp.p, 8 * (size_t)(n + 1), cudaMemcpyDeviceToHost));
  std::vector<int32_t> c32((size_t)nnz);
  LG_CUDA(cudaMemcpy(c32.data(), col.p, 4 * (size_t)nnz, cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < nnz; ++k) col_h[k] = c32[(size_t)k];
  LG_CUDA(cudaMemcpy(val_h, val.p, 8 * (size_t)nnz, cudaMemcpyDeviceToHost));
  return LG_OK;
}
