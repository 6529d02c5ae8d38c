// Gather throughput on a real column stream (dev aid).  Reads int32 column
// indices (the off-diagonal stream of a Laplacian in CSR order) from a file
// and times sum_e x[col[e]] with 8 independent gathers per thread:
//   csr      the stream as stored
//   shuffled the same columns, randomly permuted (same multiset, no locality)
//   uniform  uniform random columns (same length)
//   hubsmem  csr, but columns of the top-K hubs read from a shared-memory
//            copy of their x values (remapped index | flag)
// each with x cold (L2 flushed by a 256 MB write before every rep) and warm.
// usage: gather_real cols.bin n [K]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

constexpr int kT = 256;

__global__ void gather(const int* __restrict__ col, const double* __restrict__ x, long m,
                       double* out) {
  double s = 0.0;
  const long stride = (long)gridDim.x * blockDim.x;
#pragma unroll 8
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
    s += __ldg(x + __ldcs(col + e));
  if (s == 12345.678) *out = s;
}

template <int K>
__global__ void gather_hub(const int* __restrict__ col, const double* __restrict__ x,
                           const double* __restrict__ xhub, long m, double* out) {
  extern __shared__ double hub[];
  for (int i = threadIdx.x; i < K; i += blockDim.x) hub[i] = xhub[i];
  __syncthreads();
  double s = 0.0;
  const long stride = (long)gridDim.x * blockDim.x;
#pragma unroll 8
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    const int c = __ldcs(col + e);
    s += c < 0 ? hub[c & 0x7fffffff] : __ldg(x + c);
  }
  if (s == 12345.678) *out = s;
}

int main(int argc, char** argv) {
  if (argc < 3) return 1;
  const long n = atol(argv[2]);
  FILE* f = fopen(argv[1], "rb");
  fseek(f, 0, SEEK_END);
  const long m = ftell(f) / 4;
  fseek(f, 0, SEEK_SET);
  std::vector<int> h(m);
  if (fread(h.data(), 4, m, f) != (size_t)m) return 2;
  fclose(f);
  std::mt19937_64 rng(1);
  std::vector<int> hs(h);
  std::shuffle(hs.begin(), hs.end(), rng);
  std::vector<int> hu(m);
  for (long e = 0; e < m; ++e) hu[e] = (int)(rng() % n);
  // hubs: top-K columns by count
  constexpr int K = 12288;
  std::vector<long> cnt(n, 0);
  for (int c : h) ++cnt[c];
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::partial_sort(order.begin(), order.begin() + K, order.end(),
                    [&](int a, int b) { return cnt[a] > cnt[b]; });
  std::vector<int> slot(n, -1);
  long hubhits = 0;
  for (int i = 0; i < K; ++i) { slot[order[i]] = i; hubhits += cnt[order[i]]; }
  std::vector<int> hh(h);
  for (auto& c : hh) if (slot[c] >= 0) c = slot[c] | 0x80000000;
  printf("m=%ld n=%ld top-%d hubs take %.1f%% of gathers\n", m, n, K, 100.0 * hubhits / m);

  int *col, *cols, *colu, *colh;
  double *x, *xh, *out;
  char* junk;
  cudaMalloc(&col, 4 * m); cudaMalloc(&cols, 4 * m); cudaMalloc(&colu, 4 * m); cudaMalloc(&colh, 4 * m);
  cudaMalloc(&x, 8 * n); cudaMalloc(&xh, 8 * K); cudaMalloc(&out, 8);
  cudaMalloc(&junk, 256 << 20);
  cudaMemcpy(col, h.data(), 4 * m, cudaMemcpyHostToDevice);
  cudaMemcpy(cols, hs.data(), 4 * m, cudaMemcpyHostToDevice);
  cudaMemcpy(colu, hu.data(), 4 * m, cudaMemcpyHostToDevice);
  cudaMemcpy(colh, hh.data(), 4 * m, cudaMemcpyHostToDevice);
  cudaMemset(x, 0, 8 * n);
  cudaMemset(xh, 0, 8 * K);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(gather_hub<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * K);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cold = 1; cold >= 0; --cold) {
    for (int bps : {4, 8}) {
      const int grid = sms * bps;
      auto run = [&](auto launch, const char* name) {
        float tot = 0.f;
        for (int r = 0; r < 23; ++r) {
          if (cold) cudaMemset(junk, r & 0xff, 256 << 20);
          cudaEventRecord(e0);
          launch();
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (r >= 3) tot += ms;
        }
        printf("%s grid %5d %-9s %7.1f us\n", cold ? "cold" : "warm", grid, name, tot * 1000 / 20);
      };
      run([&] { gather<<<grid, kT>>>(col, x, m, out); }, "csr");
      run([&] { gather<<<grid, kT>>>(cols, x, m, out); }, "shuffled");
      run([&] { gather<<<grid, kT>>>(colu, x, m, out); }, "uniform");
      if (bps == 4)
        run([&] { gather_hub<K><<<grid / 2, kT, 8 * K>>>(colh, x, xh, m, out); }, "hubsmem");
    }
  }
  return 0;
}
