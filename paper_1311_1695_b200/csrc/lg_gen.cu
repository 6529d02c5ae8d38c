// lg_gen.cu -- device-side ingest for graphs too large for host numpy
// (BASELINE C5: R-MAT scale 26, edge factor 16, ~1.07e9 sampled edges).
//
// The reference cannot build C5 at all (its int64 CSR alone is
// ~33 GB and the Python IC(0) would take about a day), so this path has no
// bit-exactness target; it follows the same recipe as generators.rmat_graph
// (per-bit quadrant choice, symmetrise, drop self-loops and duplicates,
// keep the largest connected component, unit weights) with a counter-based
// RNG so it runs entirely on the device:
//
//   lg_rmat_device        edge sampling, one thread per edge, splitmix64 hash
//                         of (seed, edge, bit) -> uniform in [0, 1)
//   lg_canonical_device   (min, max) keys, radix sort, unique, self-loops out
//   lg_lcc_device         connected components by hooking + pointer jumping
//                         (Shiloach-Vishkin style), largest component kept,
//                         nodes renumbered in increasing order
//   lg_laplacian_device   L = D - A in the packed format directly on the
//                         device (unit weights: one table value, -1), plus
//                         the SpMV row-block schedule -> an lg_csr handle
#include <cub/cub.cuh>
#include <vector>

#include "lg_common.cuh"

namespace lg {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void rmat_kernel(int scale, int64_t m, double a, double b, double c, uint64_t seed,
                            uint64_t* key) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double ab = a + b, abc = a + b + c;
  const int64_t n = (int64_t)1 << scale;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    uint64_t row = 0, col = 0;
    for (int bit = 0; bit < scale; ++bit) {
      const uint64_t h = splitmix64(seed ^ ((uint64_t)e * 64u + (uint64_t)bit));
      const double r = (double)(h >> 11) * (1.0 / 9007199254740992.0);
      row |= (uint64_t)(r >= ab) << bit;
      col |= (uint64_t)(((r >= a) && (r < ab)) || (r >= abc)) << bit;
    }
    const uint64_t lo = row < col ? row : col, hi = row < col ? col : row;
    // self-loops map to the sentinel key n*n (sorted to the end, dropped)
    key[e] = (row == col) ? (uint64_t)n * (uint64_t)n : lo * (uint64_t)n + hi;
  }
}

__global__ void split_kernel(int64_t m, int64_t n, const uint64_t* key, int32_t* ei,
                             int32_t* ej) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    ei[e] = (int32_t)(key[e] / (uint64_t)n);
    ej[e] = (int32_t)(key[e] % (uint64_t)n);
  }
}

__global__ void iota32_kernel(int64_t n, int32_t* v) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    v[i] = (int32_t)i;
}

// hooking: the larger root label points to the smaller one
__global__ void hook_kernel(int64_t m, const int32_t* ei, const int32_t* ej, int32_t* label,
                            int* changed) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    int32_t lu = label[ei[e]], lv = label[ej[e]];
    if (lu == lv) continue;
    const int32_t hi = lu > lv ? lu : lv, lo = lu > lv ? lv : lu;
    if (label[hi] == hi) {
      atomicMin(label + hi, lo);
      *changed = 1;
    }
  }
}

__global__ void compress_kernel(int64_t n, int32_t* label) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    int32_t l = label[v];
    while (label[l] != l) l = label[l];
    label[v] = l;
  }
}

__global__ void count_labels_kernel(int64_t n, const int32_t* label, int32_t* cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    atomicAdd(cnt + label[v], 1);
}

__global__ void keep_kernel(int64_t n, const int32_t* label, int32_t keep, int32_t* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    flag[v] = label[v] == keep ? 1 : 0;
}

__global__ void relabel_kernel(int64_t m, const int32_t* ei, const int32_t* ej,
                               const int32_t* flag, const int32_t* newid, int32_t* oi,
                               int32_t* oj, const int64_t* pos) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    if (flag[ei[e]]) {
      const int64_t p = pos[e];
      oi[p] = newid[ei[e]];
      oj[p] = newid[ej[e]];
    }
  }
}

__global__ void edge_keep_kernel(int64_t m, const int32_t* ei, const int32_t* flag,
                                 int64_t* keepe) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
    keepe[e] = flag[ei[e]];
}

// degree counts of unit-weight canonical edges
__global__ void deg_kernel(int64_t m, const int32_t* ei, const int32_t* ej, int32_t* cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    atomicAdd(cnt + ei[e], 1);
    atomicAdd(cnt + ej[e], 1);
  }
}

static inline int gridn(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)dev_info().sm_count * 16;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

}  // namespace lg

using namespace lg;

extern "C" {

// Sample m = edge_factor * 2^scale R-MAT edges, canonicalise and dedupe on
// the device.  Outputs device arrays (cudaMalloc'ed, caller frees with
// lg_free): i < j sorted by (i, j).  *m_out = unique edges.
int lg_rmat_device(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                   int32_t** d_i, int32_t** d_j, int64_t* m_out) {
  if (scale < 1 || scale > 30 || edge_factor < 1 || !d_i || !d_j || !m_out)
    return fail(LG_EINVAL, "lg_rmat_device: bad argument");
  const int64_t n = (int64_t)1 << scale;
  const int64_t m = (int64_t)edge_factor * n;
  uint64_t *key = nullptr, *key2 = nullptr;
  int64_t* nuniq = nullptr;
  void* tmp = nullptr;
  size_t tb = 0, tb2 = 0;
  auto cleanup = [&]() {
    cudaFree(key);
    cudaFree(key2);
    cudaFree(nuniq);
    cudaFree(tmp);
  };
  if (cudaMalloc(&key, 8 * (size_t)m) != cudaSuccess ||
      cudaMalloc(&key2, 8 * (size_t)m) != cudaSuccess ||
      cudaMalloc(&nuniq, sizeof(int64_t)) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_rmat_device: key alloc");
  }
  rmat_kernel<<<gridn(m), kThreads>>>(scale, m, a, b, c, seed, key);
  const int bits = 2 * scale + 1;
  cub::DeviceRadixSort::SortKeys(nullptr, tb, key, key2, (int64_t)m, 0, bits);
  cub::DeviceSelect::Unique(nullptr, tb2, key2, key, nuniq, (int64_t)m);
  tb = std::max(tb, tb2);
  if (cudaMalloc(&tmp, tb) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_rmat_device: sort temp alloc");
  }
  cub::DeviceRadixSort::SortKeys(tmp, tb, key, key2, (int64_t)m, 0, bits);
  cub::DeviceSelect::Unique(tmp, tb, key2, key, nuniq, (int64_t)m);
  int64_t mu = 0;
  cudaMemcpy(&mu, nuniq, sizeof(int64_t), cudaMemcpyDeviceToHost);
  // the self-loop sentinel n*n sorts last: drop it if present
  uint64_t last = 0;
  if (mu > 0) cudaMemcpy(&last, key + mu - 1, 8, cudaMemcpyDeviceToHost);
  if (mu > 0 && last == (uint64_t)n * (uint64_t)n) --mu;
  int32_t *oi = nullptr, *oj = nullptr;
  if (cudaMalloc(&oi, 4 * (size_t)std::max<int64_t>(mu, 1)) != cudaSuccess ||
      cudaMalloc(&oj, 4 * (size_t)std::max<int64_t>(mu, 1)) != cudaSuccess) {
    cudaFree(oi);
    cleanup();
    return fail(LG_ENOMEM, "lg_rmat_device: edge alloc");
  }
  if (mu) split_kernel<<<gridn(mu), kThreads>>>(mu, n, key, oi, oj);
  cudaError_t e = cudaDeviceSynchronize();
  cleanup();
  if (e != cudaSuccess) {
    cudaFree(oi);
    cudaFree(oj);
    return fail(LG_ECUDA, std::string("lg_rmat_device: ") + cudaGetErrorString(e));
  }
  *d_i = oi;
  *d_j = oj;
  *m_out = mu;
  return LG_OK;
}

// Largest connected component of a canonical device edge list: renumbers
// the kept nodes 0..n_lcc-1 in increasing original order (the order of
// graphs.largest_component) and compacts the edges (order preserved, so
// they stay canonical).  Replaces *d_i / *d_j (old arrays freed).
int lg_lcc_device(int64_t n, int64_t m, int32_t** d_i, int32_t** d_j, int64_t* n_out,
                  int64_t* m_out) {
  if (n < 1 || m < 0 || !d_i || !d_j || !n_out || !m_out)
    return fail(LG_EINVAL, "lg_lcc_device: bad argument");
  int32_t *label = nullptr, *cnt = nullptr, *flag = nullptr, *newid = nullptr;
  int* changed = nullptr;
  int64_t *keepe = nullptr, *pos = nullptr;
  void* tmp = nullptr;
  auto cleanup = [&]() {
    cudaFree(label);
    cudaFree(cnt);
    cudaFree(flag);
    cudaFree(newid);
    cudaFree(changed);
    cudaFree(keepe);
    cudaFree(pos);
    cudaFree(tmp);
  };
  if (cudaMalloc(&label, 4 * (size_t)n) != cudaSuccess ||
      cudaMalloc(&cnt, 4 * (size_t)n) != cudaSuccess ||
      cudaMalloc(&flag, 4 * (size_t)n) != cudaSuccess ||
      cudaMalloc(&newid, 4 * (size_t)n) != cudaSuccess ||
      cudaMalloc(&changed, sizeof(int)) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_lcc_device: alloc");
  }
  iota32_kernel<<<gridn(n), kThreads>>>(n, label);
  for (int it = 0; it < 1000; ++it) {
    int h = 0;
    cudaMemsetAsync(changed, 0, sizeof(int));
    if (m) hook_kernel<<<gridn(m), kThreads>>>(m, *d_i, *d_j, label, changed);
    compress_kernel<<<gridn(n), kThreads>>>(n, label);
    cudaMemcpy(&h, changed, sizeof(int), cudaMemcpyDeviceToHost);
    if (!h) break;
  }
  cudaMemset(cnt, 0, 4 * (size_t)n);
  count_labels_kernel<<<gridn(n), kThreads>>>(n, label, cnt);
  // largest component; ties -> smallest label = smallest node
  std::vector<int32_t> hc((size_t)n);
  cudaMemcpy(hc.data(), cnt, 4 * (size_t)n, cudaMemcpyDeviceToHost);
  int32_t best = 0;
  for (int64_t v = 1; v < n; ++v)
    if (hc[(size_t)v] > hc[(size_t)best]) best = (int32_t)v;
  keep_kernel<<<gridn(n), kThreads>>>(n, label, best, flag);
  size_t tb = 0, tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, newid, (int64_t)n);
  if (cudaMalloc(&keepe, 8 * (size_t)std::max<int64_t>(m, 1)) != cudaSuccess ||
      cudaMalloc(&pos, 8 * (size_t)std::max<int64_t>(m, 1)) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_lcc_device: edge alloc");
  }
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, keepe, pos, (int64_t)std::max<int64_t>(m, 1));
  tb = std::max(tb, tb2);
  if (cudaMalloc(&tmp, tb) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_lcc_device: temp alloc");
  }
  cub::DeviceScan::ExclusiveSum(tmp, tb, flag, newid, (int64_t)n);
  const int64_t nl = hc[(size_t)best];
  int64_t ml = 0;
  int32_t *oi = nullptr, *oj = nullptr;
  if (m) {
    edge_keep_kernel<<<gridn(m), kThreads>>>(m, *d_i, flag, keepe);
    cub::DeviceScan::ExclusiveSum(tmp, tb, keepe, pos, (int64_t)m);
    int64_t lastpos = 0, lastkeep = 0;
    cudaMemcpy(&lastpos, pos + m - 1, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&lastkeep, keepe + m - 1, 8, cudaMemcpyDeviceToHost);
    ml = lastpos + lastkeep;
  }
  if (cudaMalloc(&oi, 4 * (size_t)std::max<int64_t>(ml, 1)) != cudaSuccess ||
      cudaMalloc(&oj, 4 * (size_t)std::max<int64_t>(ml, 1)) != cudaSuccess) {
    cudaFree(oi);
    cleanup();
    return fail(LG_ENOMEM, "lg_lcc_device: output alloc");
  }
  if (m) relabel_kernel<<<gridn(m), kThreads>>>(m, *d_i, *d_j, flag, newid, oi, oj, pos);
  cudaError_t e = cudaDeviceSynchronize();
  cleanup();
  if (e != cudaSuccess) {
    cudaFree(oi);
    cudaFree(oj);
    return fail(LG_ECUDA, std::string("lg_lcc_device: ") + cudaGetErrorString(e));
  }
  cudaFree(*d_i);
  cudaFree(*d_j);
  *d_i = oi;
  *d_j = oj;
  *n_out = nl;
  *m_out = ml;
  return LG_OK;
}

int lg_free(void* p) {
  cudaFree(p);
  return LG_OK;
}

}  // extern "C"
