// Microbenchmark: cluster barrier cost and a store->barrier->load chain.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void k_cluster(int nb, int mode, double* x, double* out) {
  double acc = 0.0;
  const unsigned rank = cg::this_cluster().block_rank();
  for (int b = 0; b < nb; ++b) {
    if (mode >= 1 && threadIdx.x == 0) x[(b * 16 + rank) & 1023] = acc + b;  // publish
    if (mode == 2) {
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (mode == 3) {
      asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    } else {
      cg::this_cluster().sync();
    }
    if (mode >= 1 && threadIdx.x == 0) acc += __ldcg(x + ((b * 16 + (rank + 1) % 16) & 1023));
  }
  if (acc == -1.0) *out = acc;
}

__global__ void k_block(int nb, double* x, double* out) {
  double acc = 0.0;
  for (int b = 0; b < nb; ++b) {
    if (threadIdx.x == 0) x[b & 1023] = acc + b;
    __syncthreads();
    if (threadIdx.x == 32) acc += x[b & 1023];
  }
  if (acc == -1.0) *out = acc;
}

__global__ void k_chain(int nb, double* x, double* out) {
  // single thread dependent L2 load chain (latency)
  double acc = 0.0;
  int idx = 0;
  for (int b = 0; b < nb; ++b) {
    acc += __ldcg(x + idx);
    idx = ((int)acc & 1) * 64 + (b * 97 & 1023);
  }
  if (acc == -1.0) *out = acc;
}

int main() {
  double *x, *out;
  cudaMalloc(&x, 8 * 4096);
  cudaMemset(x, 0, 8 * 4096);
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int nb = 2000;
  for (int cs : {2, 4, 8, 16}) for (int T : {128, 512}) for (int mode : {0, 1, 2, 3}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(T);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, k_cluster, nb, mode, x, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("cluster cs=%2d T=%3d mode=%d (%s): %.3f us/iter (%s)\n", cs, T, mode,
           mode == 0 ? "cg sync" : mode == 1 ? "cg sync + store/load" : mode == 2 ? "rel/acq + store/load" : "relaxed + store/load",
           ms * 1000 / nb, cudaGetErrorString(cudaGetLastError()));
  }
  float ms;
  for (int T : {128, 512, 1024}) {
    cudaEventRecord(e0); k_block<<<1, T>>>(nb, x, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("block T=%d store/sync/load: %.3f us/iter\n", T, ms * 1000 / nb);
  }
  cudaEventRecord(e0); k_chain<<<1, 32>>>(nb, x, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("L2 dependent load chain: %.3f us/load\n", ms * 1000 / nb);
  return 0;
}
