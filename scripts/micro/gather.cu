// Pure gather throughput: stream int32 columns, gather f64 x, sum (dev aid).
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>

template <int MODE>
__global__ void gather(const int* __restrict__ col, const double* __restrict__ x, long m, double* out) {
  double s = 0.0;
  long stride = (long)gridDim.x * blockDim.x;
  #pragma unroll 8
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    int c = __ldcs(col + e);
    double v;
    if (MODE == 0) v = __ldg(x + c);
    else if (MODE == 1) v = __ldcg(x + c);
    else { asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(x + c)); }
    s += v;
  }
  if (s == 12345.678) *out = s;
}

__global__ void stream_only(const int* __restrict__ col, long m, double* out) {
  long s = 0; long stride = (long)gridDim.x * blockDim.x;
  #pragma unroll 8
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) s += __ldcs(col + e);
  if (s == 12345) *out = s;
}

int main() {
  const long n = 989777, m = 9917680;   // C4-like
  std::vector<int> h(m);
  std::mt19937_64 rng(1);
  for (long e = 0; e < m; ++e) h[e] = rng() % n;
  std::vector<int> hs(h);
  // per-1024 block sorted (locality inside warps)
  for (long b = 0; b < m; b += 1024) std::sort(hs.begin() + b, hs.begin() + std::min(m, b + 1024));
  int *col, *cols; double *x, *out;
  cudaMalloc(&col, 4 * m); cudaMalloc(&cols, 4 * m); cudaMalloc(&x, 8 * n); cudaMalloc(&out, 8);
  cudaMemcpy(col, h.data(), 4 * m, cudaMemcpyHostToDevice);
  cudaMemcpy(cols, hs.data(), 4 * m, cudaMemcpyHostToDevice);
  cudaMemset(x, 0, 8 * n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148;
  for (int blocksPerSm : {4, 8, 16}) for (int T : {256, 512}) {
    int grid = sms * blocksPerSm * 256 / T;
    float ms;
    auto run = [&](auto k, const int* c, const char* name) {
      for (int r = 0; r < 3; ++r) k<<<grid, T>>>(c, x, m, out);
      cudaEventRecord(e0); for (int r = 0; r < 20; ++r) k<<<grid, T>>>(c, x, m, out); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      printf("grid %5d T %3d %-22s %.1f us\n", grid, T, name, ms * 1000 / 20);
    };
    run(gather<0>, col, "ldg random");
    run(gather<1>, col, "ldcg random");
    run(gather<2>, col, "nc.no_allocate random");
    run(gather<0>, cols, "ldg block-sorted");
  }
  float ms;
  cudaEventRecord(e0); for (int r = 0; r < 20; ++r) stream_only<<<sms * 8, 256>>>(col, m, out); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("stream only %.1f us\n", ms * 1000 / 20);
  return 0;
}
