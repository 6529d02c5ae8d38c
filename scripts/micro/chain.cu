// Microbenchmark: latency of one dependency hop between warps on different
// SMs -- the critical path of a level-scheduled triangular sweep.  Hop i is
// done by warp (i mod K) on CTA (i mod K): wait until flag[i-1] is set, read
// x[i-1] from L2, write x[i], publish flag[i].  Variants of the publish /
// observe pair (development aid).
#include <cstdio>

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// mode 0: threadfence + atomicAdd / relaxed poll + threadfence
// mode 1: red.release / ld.acquire poll
// mode 2: st.release flag / ld.acquire poll
// mode 3: data-as-flag: x written with st.relaxed (NaN sentinel), polled directly
// mode 4: red.release / ld.relaxed poll + fence.acq_rel
template <int MODE>
__global__ void chain(unsigned* flag, double* x, int hops, int sleepns) {
  const int K = gridDim.x;
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  for (int i = blockIdx.x + 1; i < hops; i += K) {
    double prev;
    if (MODE == 3) {
      do {
        prev = ld_relaxed64(x + i - 1);
        if (prev != prev && sleepns) __nanosleep(sleepns);
      } while (prev != prev);
    } else {
      if (MODE == 0) {
        while (ld_relaxed(flag + i - 1) == 0)
          if (sleepns) __nanosleep(sleepns);
        __threadfence();
      } else if (MODE == 4) {
        while (ld_relaxed(flag + i - 1) == 0)
          if (sleepns) __nanosleep(sleepns);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else {
        while (ld_acquire(flag + i - 1) == 0)
          if (sleepns) __nanosleep(sleepns);
      }
      prev = __ldcg(x + i - 1);
    }
    __syncwarp();
    if (lane == 0) {
      if (MODE == 3) {
        st_relaxed64(x + i, prev + 1.0);
      } else {
        x[i] = prev + 1.0;
        if (MODE == 0) {
          __threadfence();
          atomicAdd(flag + i, 1u);
        } else if (MODE == 2) {
          st_release(flag + i, 1u);
        } else {
          red_release(flag + i, 1u);
        }
      }
    }
    __syncwarp();
  }
}

template <int MODE>
static void run(int K, int hops, int sleepns) {
  unsigned* flag;
  double* x;
  cudaMalloc(&flag, 4 * (size_t)hops);
  cudaMalloc(&x, 8 * (size_t)hops);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaMemset(flag, 0, 4 * (size_t)hops);
    cudaMemset(x, 0xff, 8 * (size_t)hops);   // NaN
    double z = 0.0;
    cudaMemcpy(x, &z, 8, cudaMemcpyHostToDevice);
    cudaMemset(flag, 1, 4);
    cudaEventRecord(e0);
    chain<MODE><<<K, 32>>>(flag, x, hops, sleepns);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double last;
  cudaMemcpy(&last, x + hops - 1, 8, cudaMemcpyDeviceToHost);
  printf("mode %d K %d sleep %d: %.3f us/hop (check %s)\n", MODE, K, sleepns,
         best * 1e3 / hops, last == hops - 1 ? "ok" : "BAD");
  cudaFree(flag);
  cudaFree(x);
}

int main() {
  const int hops = 20000;
  for (int K : {2, 148}) {
    for (int s : {0, 32}) {
      run<0>(K, hops, s);
      run<1>(K, hops, s);
      run<2>(K, hops, s);
      run<3>(K, hops, s);
      run<4>(K, hops, s);
    }
  }
  return 0;
}
