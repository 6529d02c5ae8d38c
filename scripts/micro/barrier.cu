// Microbenchmark: cost of grid-wide barriers on B200 (development aid).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_atomic(unsigned long long* bar, int nb, int sleepns) {
  __shared__ unsigned long long base;
  if (threadIdx.x == 0) base = ldr(bar) / ((unsigned long long)nb * gridDim.x) * ((unsigned long long)nb * gridDim.x);
  __syncthreads();
  for (int b = 1; b <= nb; ++b) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1ull);
      unsigned long long t = base + (unsigned long long)b * gridDim.x;
      while (ldr(bar) < t) if (sleepns) __nanosleep(sleepns);
      __threadfence();
    }
    __syncthreads();
  }
}

// red.release + ld.acquire flavour, no separate fences
__global__ void k_relacq(unsigned long long* bar, int nb) {
  __shared__ unsigned long long base;
  if (threadIdx.x == 0) base = ldr(bar) / ((unsigned long long)nb * gridDim.x) * ((unsigned long long)nb * gridDim.x);
  __syncthreads();
  for (int b = 1; b <= nb; ++b) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
      unsigned long long t = base + (unsigned long long)b * gridDim.x, v;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
      } while (v < t);
    }
    __syncthreads();
  }
}

__global__ void k_cg(int nb) {
  cg::grid_group g = cg::this_grid();
  for (int b = 0; b < nb; ++b) g.sync();
}

__global__ void k_block(int nb, int* out) {
  int acc = 0;
  for (int b = 0; b < nb; ++b) { __syncthreads(); acc += threadIdx.x; }
  if (acc == -1) *out = acc;
}

int main() {
  unsigned long long* bar;
  cudaMalloc(&bar, 8);
  cudaMemset(bar, 0, 8);
  int* out; cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int nb = 1000;
  int sms = 148;
  for (int G : {148, 296}) for (int T : {256, 512, 1024}) {
    if (G == 296 && T == 1024) continue;
    for (int sl : {0, 16, 64}) {
      void* args[] = {&bar, (void*)&nb, &sl};
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_atomic, G, T, args, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("atomic  G=%d T=%d sleep=%d: %.3f us/barrier (%s)\n", G, T, sl, ms * 1000 / nb, cudaGetErrorString(cudaGetLastError()));
    }
    {
      void* args[] = {&bar, (void*)&nb};
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_relacq, G, T, args, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("relacq  G=%d T=%d: %.3f us/barrier (%s)\n", G, T, ms * 1000 / nb, cudaGetErrorString(cudaGetLastError()));
    }
    {
      void* args[] = {(void*)&nb};
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_cg, G, T, args, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("cg      G=%d T=%d: %.3f us/barrier (%s)\n", G, T, ms * 1000 / nb, cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int T : {512, 1024}) {
    cudaEventRecord(e0);
    k_block<<<1, T>>>(nb * 10, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("block   T=%d: %.4f us/barrier\n", T, ms * 1000 / (nb * 10));
  }
  // empty cooperative launch latency
  for (int rep = 0; rep < 3; ++rep) {
    int z = 0; void* args[] = {(void*)&z};
    cudaEventRecord(e0);
    for (int i = 0; i < 100; ++i) cudaLaunchCooperativeKernel((void*)k_cg, 296, 512, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("empty coop launch: %.2f us\n", ms * 1000 / 100);
    cudaEventRecord(e0);
    for (int i = 0; i < 100; ++i) k_block<<<296, 512>>>(0, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("empty normal launch: %.2f us\n", ms * 1000 / 100);
  }
  return 0;
}
