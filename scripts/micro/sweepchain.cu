// Microbenchmark: per-level cost of a level-synchronous triangular sweep run
// by ONE thread-block cluster (dev aid for the resident narrow-DAG sweep).
// Each level every thread gathers K entries of the previous level's x (written
// by any CTA of the cluster), reduces, divides, stores one entry of this
// level's x; levels are separated by a cluster barrier (release / acquire).
//   mode 0  x in global memory (st.relaxed.gpu / ld.relaxed.gpu, i.e. L2)
//   mode 1  x in distributed shared memory (st.shared local, ld.shared::cluster)
//   mode 2  as 0 but one CTA, __syncthreads, plain ld / st (L1 + L2)
//   mode 3  as 1 but one CTA (plain shared memory)
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

constexpr int K = 4;
constexpr int kXS = 8192;   // x slots per CTA (64 KB)

__device__ __forceinline__ double ldg_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void stg_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_dsmem(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

template <int MODE>
__global__ void k_sweep(int nb, int active, double* xg, double* out) {
  extern __shared__ double xs[];
  const unsigned cs = MODE <= 1 ? cg::this_cluster().num_blocks() : 1;
  const unsigned rank = MODE <= 1 ? cg::this_cluster().block_rank() : 0;
  const int T = blockDim.x, t = threadIdx.x;
  for (int i = t; i < kXS; i += T) xs[i] = 1.0;
  if (MODE == 0 || MODE == 2)
    for (int i = t; i < kXS; i += T) xg[rank * kXS + i] = 1.0;
  if (MODE <= 1) cg::this_cluster().sync(); else __syncthreads();
  const uint32_t xs_base = (uint32_t)__cvta_generic_to_shared(xs);
  double acc = 0.0;
  unsigned h = t * 2654435761u + rank * 40503u;
  for (int b = 0; b < nb; ++b) {
    if (t < active) {
      double s = 0.0;
      double xv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        h = h * 1664525u + 1013904223u;
        // an entry of the previous level: slot window (b-1), any CTA, any thread
        const unsigned src_cta = (h >> 8) % cs;
        const unsigned src_t = (h >> 16) % (unsigned)active;
        const unsigned slot = (((unsigned)(b + 7) & 7u) * 1024u + src_t) & (kXS - 1);
        if (MODE == 0) xv[k] = ldg_relaxed(xg + src_cta * kXS + slot);
        else if (MODE == 1) xv[k] = ld_dsmem(mapa(xs_base + 8u * slot, src_cta));
        else if (MODE == 2) xv[k] = xg[slot];
        else xv[k] = xs[slot];
      }
#pragma unroll
      for (int k = 0; k < K; ++k) s += 0.25 * xv[k];
      const double v = (1.0 + s) / (2.0 + 1e-9 * b);
      const unsigned my = (((unsigned)b & 7u) * 1024u + (unsigned)t) & (kXS - 1);
      if (MODE == 0) stg_relaxed(xg + rank * kXS + my, v);
      else if (MODE == 2) xg[my] = v;
      else xs[my] = v;
      acc += v;
    }
    if (MODE <= 1) {
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      __syncthreads();
    }
  }
  if (acc == -1.0) *out = acc;
}

template <int MODE>
static void run(int cs, int T, int active, int nb, double* xg, double* out) {
  cudaFuncSetAttribute(k_sweep<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_sweep<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kXS);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs); cfg.blockDim = dim3(T); cfg.dynamicSmemBytes = 8 * kXS;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k_sweep<MODE>, nb, active, xg, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const char* names[] = {"cluster, x in L2", "cluster, x in DSMEM", "1 CTA, x global (L1/L2)", "1 CTA, x in smem"};
  printf("mode %d (%-24s) cs=%2d T=%4d active=%4d: %.3f us/level (%s)\n", MODE, names[MODE], cs, T,
         active, ms * 1000 / nb, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *xg, *out;
  cudaMalloc(&xg, 8 * kXS * 16);
  cudaMalloc(&out, 8);
  const int nb = 4000;
  for (int T : {256, 512, 1024}) {
    for (int active : {32, T}) {
      run<3>(1, T, active, nb, xg, out);
      run<2>(1, T, active, nb, xg, out);
      for (int cs : {2, 4, 8, 16}) {
        run<1>(cs, T, active, nb, xg, out);
        run<0>(cs, T, active, nb, xg, out);
      }
    }
  }
  return 0;
}
