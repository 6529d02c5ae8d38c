// Gather throughput vs the footprint of the gathered x (dev aid): is an
// L1-resident (hub) region cheaper than L2 gathers, and what does a
// shared-memory hub table cost?  m = 9.9 M gathers (C4's off-diagonals).
#include <cstdio>
#include <random>
#include <vector>

__global__ void gather(const int* __restrict__ col, const double* __restrict__ x, long m,
                       double* out) {
  double s = 0.0;
  long stride = (long)gridDim.x * blockDim.x;
#pragma unroll 8
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
    s += __ldg(x + __ldcs(col + e));
  if (s == 12345.678) *out = s;
}

// hub indices (< H) read from a shared-memory copy, the rest from x
template <int H>
__global__ void gather_smem(const int* __restrict__ col, const double* __restrict__ x, long m,
                            double* out) {
  extern __shared__ double hub[];
  for (int i = threadIdx.x; i < H; i += blockDim.x) hub[i] = x[i];
  __syncthreads();
  double s = 0.0;
  long stride = (long)gridDim.x * blockDim.x;
#pragma unroll 8
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    int c = __ldcs(col + e);
    s += c < H ? hub[c] : __ldg(x + c);
  }
  if (s == 12345.678) *out = s;
}

int main() {
  const long n = 989777, m = 9917680;
  int *col;
  double *x, *out;
  cudaMalloc(&col, 4 * m);
  cudaMalloc(&x, 8 * n);
  cudaMalloc(&out, 8);
  cudaMemset(x, 0, 8 * n);
  std::vector<int> h(m);
  std::mt19937_64 rng(1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  auto timeit = [&](auto launch) {
    float ms;
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1000 / 20;
  };
  // uniform over a footprint of F doubles
  for (long F : {n, 1L << 17, 1L << 14, 1L << 12, 1L << 9, 1L << 5}) {
    for (long e = 0; e < m; ++e) h[e] = rng() % F;
    cudaMemcpy(col, h.data(), 4 * m, cudaMemcpyHostToDevice);
    float us = timeit([&] { gather<<<sms * 8, 256>>>(col, x, m, out); });
    printf("uniform footprint %8ld doubles (%7.1f KB): %6.1f us  %.2f gathers/SM/cycle\n", F,
           F * 8 / 1024.0, us, m / (us * 1e-6) / sms / 1.965e9);
  }
  // hub mixes: fraction p of gathers in [0, 16384), the rest uniform over n
  for (double p : {0.0, 0.25, 0.5, 0.75}) {
    for (long e = 0; e < m; ++e) {
      double u = (rng() >> 11) * (1.0 / 9007199254740992.0);
      h[e] = u < p ? (int)(rng() % 16384) : (int)(16384 + rng() % (n - 16384));
    }
    cudaMemcpy(col, h.data(), 4 * m, cudaMemcpyHostToDevice);
    float us = timeit([&] { gather<<<sms * 8, 256>>>(col, x, m, out); });
    cudaFuncSetAttribute(gather_smem<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    float us2 = timeit([&] { gather_smem<16384><<<sms, 1024, 131072>>>(col, x, m, out); });
    printf("hub fraction %.2f (16K hubs): L1/L2 gathers %6.1f us, smem hub table %6.1f us\n", p,
           us, us2);
  }
  return 0;
}
