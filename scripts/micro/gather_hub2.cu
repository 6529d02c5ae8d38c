// Gather throughput on a real column stream with the hottest columns' x
// values in shared memory, at FULL occupancy (dev aid; gather_real's hubsmem
// variant halved the resident warps, which confounded it).  One 1024-thread CTA
// per SM (32 warps, as the SpMV has), K hub values in dynamic shared memory;
// hub columns are remapped to slot | 0x80000000.  Also: the same stream with
// only half of each warp's lanes active per gather instruction (is a
// divergent LDG dearer per line than two narrower ones?).
// usage: gather_hub2 cols.bin n
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

constexpr int kT = 1024;

__global__ void __launch_bounds__(kT, 1) gather_plain(const int* __restrict__ col,
                                                       const double* __restrict__ x, long m,
                                                       double* out) {
  double s = 0.0;
  const long stride = (long)gridDim.x * blockDim.x;
#pragma unroll 8
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
    s += __ldg(x + __ldcs(col + e));
  if (s == 12345.678) *out = s;
}

__global__ void __launch_bounds__(kT, 1) gather_hub(const int* __restrict__ col,
                                                     const double* __restrict__ x,
                                                     const double* __restrict__ xhub, int K, long m,
                                                     double* out) {
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

// half of the lanes gather per instruction (even lanes, then odd lanes)
__global__ void __launch_bounds__(kT, 1) gather_half(const int* __restrict__ col,
                                                      const double* __restrict__ x, long m,
                                                      double* out) {
  double s = 0.0;
  const long stride = (long)gridDim.x * blockDim.x;
  const bool odd = threadIdx.x & 1;
#pragma unroll 8
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    const int c = __ldcs(col + e);
    double v = 0.0, w = 0.0;
    if (!odd) v = __ldg(x + c);
    if (odd) w = __ldg(x + c);
    s += v + w;
  }
  if (s == 12345.678) *out = s;
}

int main(int argc, char** argv) {
  if (argc < 3) return 1;
  const long n = atol(argv[2]);
  FILE* f = fopen(argv[1], "rb");
  if (!f) { printf("cannot open %s\n", argv[1]); return 2; }
  fseek(f, 0, SEEK_END);
  const long m = ftell(f) / 4;
  fseek(f, 0, SEEK_SET);
  std::vector<int> h(m);
  if (fread(h.data(), 4, m, f) != (size_t)m) return 2;
  fclose(f);
  std::vector<long> cnt(n, 0);
  for (int c : h) ++cnt[c];
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return cnt[a] > cnt[b]; });
  int *col, *colh;
  double *x, *xh, *out;
  char* junk;
  cudaMalloc(&col, 4 * m); cudaMalloc(&colh, 4 * m);
  cudaMalloc(&x, 8 * n); cudaMalloc(&xh, 8 * 28000); cudaMalloc(&out, 8);
  cudaMalloc(&junk, 256 << 20);
  cudaMemcpy(col, h.data(), 4 * m, cudaMemcpyHostToDevice);
  cudaMemset(x, 0, 8 * n); cudaMemset(xh, 0, 8 * 28000);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(gather_hub, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 28000);
  auto run = [&](auto launch, const char* name) {
    for (int cold = 1; cold >= 0; --cold) {
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
      printf("%s %-26s %7.1f us (%s)\n", cold ? "cold" : "warm", name, tot * 1000 / 20,
             cudaGetErrorString(cudaGetLastError()));
    }
  };
  run([&] { gather_plain<<<sms, kT>>>(col, x, m, out); }, "plain 1x1024");
  run([&] { gather_plain<<<2 * sms, kT>>>(col, x, m, out); }, "plain 2x1024");
  run([&] { gather_half<<<2 * sms, kT>>>(col, x, m, out); }, "half-warp LDGs 2x1024");
  for (int K : {4096, 12288, 20480, 27648}) {
    std::vector<int> slot(n, -1);
    long hits = 0;
    for (int i = 0; i < K; ++i) { slot[order[i]] = i; hits += cnt[order[i]]; }
    std::vector<int> hh(h);
    for (auto& c : hh) if (slot[c] >= 0) c = slot[c] | 0x80000000;
    cudaMemcpy(colh, hh.data(), 4 * m, cudaMemcpyHostToDevice);
    char name[64];
    snprintf(name, sizeof name, "hub K=%d (%.1f%% hits)", K, 100.0 * hits / m);
    run([&] { gather_hub<<<sms, kT, 8 * K>>>(colh, x, xh, K, m, out); }, name);
    if (8 * K <= 110 * 1024) {
      snprintf(name, sizeof name, "hub K=%d 2 CTAs/SM", K);
      run([&] { gather_hub<<<2 * sms, kT, 8 * K>>>(colh, x, xh, K, m, out); }, name);
    }
  }
  return 0;
}
