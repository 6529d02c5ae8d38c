// TMA tile::gather4 throughput vs LSU gathers (dev aid).
#include <cuda.h>
#include <cstdio>
#include <vector>
#include <random>
#include <cuda_runtime.h>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, int c0, int r0, int r1, int r2, int r3,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(smem_u32(dst)), "l"(tm), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)) : "memory");
}

constexpr int CH = 1024;           // entries per chunk
constexpr int OPS = CH / 4;        // gather4 ops per chunk
constexpr int T = 256;

// each CTA: chunks b = blockIdx.x, += gridDim.x; warp 0 issues TMA for the
// next chunk while all threads consume the current one
__global__ void __launch_bounds__(T) tma_kernel(const __grid_constant__ CUtensorMap tm, const int* col, long m,
                                                double* out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double* buf = (double*)smraw;                  // [2][CH][4] doubles = 2 * 32 KB
  __shared__ __align__(8) uint64_t bar[2];
  const long nch = m / CH;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto issue = [&](long c, int slot) {
    // warp 0: 32 lanes x 8 ops each
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) mbar_expect_tx(&bar[slot], CH * 32);
      __syncwarp();
      const int* cp = col + c * CH;
      for (int op = threadIdx.x; op < OPS; op += 32) {
        const int4 q = __ldcs((const int4*)cp + op);
        gather4(buf + (size_t)slot * CH * 4 + (size_t)op * 16, &tm, 0, q.x >> 2, q.y >> 2, q.z >> 2, q.w >> 2,
                &bar[slot]);
      }
    }
  };
  double s = 0.0;
  long c = blockIdx.x;
  int slot = 0, ph[2] = {0, 0};
  if (c < nch) issue(c, 0);
  for (; c < nch; c += gridDim.x) {
    const long cn = c + gridDim.x;
    if (cn < nch) issue(cn, slot ^ 1);
    mbar_wait(&bar[slot], ph[slot]);
    ph[slot] ^= 1;
    const int* cp = col + c * CH;
    const double* b = buf + (size_t)slot * CH * 4;
    for (int e = threadIdx.x; e < CH; e += T) {
      const int cc = __ldg(cp + e);
      s += b[e * 4 + (cc & 3)];
    }
    __syncthreads();   // buffer slot reused two chunks later
    slot ^= 1;
  }
  if (s == 12345.678) *out = s;
}

__global__ void lsu_kernel(const int* __restrict__ col, const double* __restrict__ x, long m, double* out) {
  double s = 0.0;
  long stride = (long)gridDim.x * blockDim.x;
#pragma unroll 8
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) s += __ldg(x + __ldcs(col + e));
  if (s == 12345.678) *out = s;
}

int main() {
  const long n = 989780, m = 9917440;   // C4-like, multiples of 4 / CH
  std::vector<int> h(m);
  std::mt19937_64 rng(1);
  for (long e = 0; e < m; ++e) h[e] = rng() % n;
  int* col; double *x, *out;
  cudaMalloc(&col, 4 * m); cudaMalloc(&x, 8 * n); cudaMalloc(&out, 8);
  cudaMemcpy(col, h.data(), 4 * m, cudaMemcpyHostToDevice);
  std::vector<double> hx(n);
  for (long i = 0; i < n; ++i) hx[i] = (double)i;
  cudaMemcpy(x, hx.data(), 8 * n, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (!fn) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  CUtensorMap tm;
  cuuint64_t dims[2] = {4, (cuuint64_t)(n / 4)};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * CH * 32);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int bpsm : {1, 2, 3}) {
    int grid = 148 * bpsm;
    for (int k = 0; k < 3; ++k) tma_kernel<<<grid, T, 2 * CH * 32>>>(tm, col, m, out);
    cudaError_t err = cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int k = 0; k < 20; ++k) tma_kernel<<<grid, T, 2 * CH * 32>>>(tm, col, m, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("tma gather4 grid %d: %.1f us (%s / %s)\n", grid, ms * 1000 / 20, cudaGetErrorString(err),
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int k = 0; k < 3; ++k) lsu_kernel<<<148 * 8, 256>>>(col, x, m, out);
  cudaEventRecord(e0);
  for (int k = 0; k < 20; ++k) lsu_kernel<<<148 * 8, 256>>>(col, x, m, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("lsu gather: %.1f us\n", ms * 1000 / 20);
  return 0;
}
