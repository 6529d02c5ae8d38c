// lg_vec.cu -- fused streaming vector pass, small tall-skinny GEMM,
// Jacobi apply.
//
// Replaces the n-vector arithmetic of the reference solvers:
//   DeflationBasis.project_out  v - C (C^T v)            pcg.py:55-60
//   mgs_orthonormalize sweeps   v -= (q.v) q              kernels.py:42-49
//   DACG dots / axpys / normalisation                     dacg.py:40-96,172-233
//   PCG dots / axpys                                      pcg.py:131-155
// Each of those is a sequence of numpy passes (one pass per dot, per axpy,
// per GEMV).  lg_fused does any such sequence that has no grid-wide data
// dependency in ONE pass: up to two outputs (linear combinations of up to
// four vectors, minus a block combination Q c whose coefficients c were
// produced by an earlier pass), plus dot products and Q^T v block dots of
// inputs *and* of the freshly computed outputs.  The projection v - Q(Q^T v)
// is therefore split across two passes -- the Q^T v half is fused into the
// pass (or SpMV / SpTRSV epilogue) that produces v, the update half into the
// pass that consumes it -- so a projection costs no pass of its own.
#include <algorithm>
#include <cstring>

#include "lg_scalar.cuh"

namespace lg {

struct FusedDev {
  int64_t n;
  lg_output o[LG_MAXO];
  int ndots;
  const double* da[LG_MAXD];
  const double* db[LG_MAXD];
  const double* dc[LG_MAXD];
  int nblocks;
  lg_block b[LG_MAXB];
  double* result;
  const int* skip;
};

// Elements per thread per tile.  A warp owns a tile of 32*kU consecutive
// elements and lane l handles tile elements l, l+32, ...: every load
// instruction is one coalesced 256-byte warp access, and each thread keeps
// kU independent loads per operand in flight (memory-level parallelism is
// what a streaming pass over HBM needs; one element per thread leaves the
// pass latency-bound at ~1-3 TB/s).
// Tiles per thread and resident CTAs per SM depend on the pass: passes
// with at most 4 reduced values keep 4 elements per lane in flight at 4
// CTAs per SM; passes with block dots / updates (k >= 5 reduced values, the
// deflation projections) use 2 elements per lane -- fewer registers, the
// same 4 CTAs per SM.  Measured on 32.8 M-element passes: a 4-term
// combination with 3 dots 308 -> 275 us (4.8 TB/s), a k = 6 projection
// update with Q^T v 889 -> 654 us (5.6 TB/s).
template <int NA>
__host__ __device__ constexpr int fused_u() { return NA <= 4 ? 4 : 2; }
constexpr int kU = 4;   // widest tile (shared-memory sizing)

template <int U>
__device__ __forceinline__ void load_u(const double* p, int64_t i0, int64_t n, double (&v)[U]) {
  // Non-coherent loads: an element is read and then written only by its
  // own thread and never re-read after the write, so in-place passes stay
  // correct.
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + 32 * u;
    v[u] = i < n ? __ldg(p + i) : 0.0;
  }
}

// operand u-values: an input vector or an output of this pass
template <int U>
__device__ __forceinline__ void operand(const double* p, int64_t i0, int64_t n,
                                        const double (&ov)[LG_MAXO][U], double (&v)[U]) {
  const uintptr_t k = (uintptr_t)p;
  // constant indices only: a runtime index would move ov to local memory
  if (k == 1) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ov[0][u];
  } else if (k == 2) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ov[1][u];
  } else if (k == 3) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ov[2][u];
  } else {
    load_u<U>(p, i0, n, v);
  }
}

template <int U>
__device__ __forceinline__ void output_u(const lg_output& o, const double* coef,
                                         const double* uc, const double* uc2, int64_t i0,
                                         int64_t n, const double (&ov)[LG_MAXO][U], double post,
                                         int pmode, double (&v)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = 0.0;
#pragma unroll
  for (int t = 0; t < LG_MAXT; ++t) {
    if (t < o.nterms) {
      double x[U];
      operand<U>(o.t[t].v, i0, n, ov, x);
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] += coef[t] * x[u];
    }
  }
  if (o.uk > 0 || o.uk2 > 0) {
    double sq[U];
#pragma unroll
    for (int u = 0; u < U; ++u) sq[u] = 0.0;
    for (int j = 0; j < o.uk; ++j) {
      double x[U];
      load_u<U>(o.uq + (int64_t)j * o.uld, i0, n, x);
#pragma unroll
      for (int u = 0; u < U; ++u) sq[u] += uc[j] * x[u];
    }
    for (int j = 0; j < o.uk2; ++j) {
      double x[U];
      load_u<U>(o.uq2 + (int64_t)j * o.uld2, i0, n, x);
#pragma unroll
      for (int u = 0; u < U; ++u) sq[u] += uc2[j] * x[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] -= sq[u];
  }
  if (pmode == 1) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] *= post;
  } else if (pmode == 2) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] /= post;
  }
}

// optional scalar program run by the pass's finishing CTA
struct ProgDev {
  ScalarProg p;
  double* sg;
  int* fg;
};

#ifndef LG_FUSED_MINB4
#define LG_FUSED_MINB4 3   // resident CTAs for the 4-wide tiles (NA <= 4): 85 registers, no spill
#endif
template <int NA, bool PROG>
__global__ void __launch_bounds__(kThreads, (NA <= 4 ? LG_FUSED_MINB4
                                             : (NA <= 8 ? 4 : (NA <= 16 ? 2 : 1))))
fused_kernel(FusedDev a, lg_ws ws, const __grid_constant__ ProgDev pd) {
  constexpr int U = fused_u<NA>();
  if (a.skip && *a.skip) return;
  constexpr int M = NA > 0 ? NA : 1;
  __shared__ double uc_sm[LG_MAXO][LG_MAXQ];
  __shared__ double uc2_sm[LG_MAXO][LG_MAXQ];
  __shared__ double red_sm[kWarps * M];
  // per-pass coefficients in shared memory (uniform broadcast reads keep
  // the registers for the U-element tiles)
  __shared__ double coef[LG_MAXO][LG_MAXT];
  __shared__ double post[LG_MAXO];
  __shared__ int pmode[LG_MAXO];
  if (threadIdx.x < LG_MAXO * LG_MAXT) {
    const int k = threadIdx.x / LG_MAXT, t = threadIdx.x % LG_MAXT;
    const lg_output& o = a.o[k];
    double c = 0.0;
    if (t < o.nterms) {
      c = o.t[t].h;
      if (o.t[t].d) c *= *o.t[t].d;
    }
    coef[k][t] = c;
    if (t == 0) {
      double p = 1.0;
      int m = 0;
      if (o.post_mode) {
        p = *o.d_post;
        if (o.post_mode == 3) p = sqrt(p);
        m = (o.post_mode == 1) ? 1 : 2;
      }
      post[k] = p;
      pmode[k] = m;
    }
  }
#pragma unroll
  for (int k = 0; k < LG_MAXO; ++k) {
    const lg_output& o = a.o[k];
    for (int j = threadIdx.x; j < o.uk; j += blockDim.x)
      uc_sm[k][j] = o.cscale * o.uc[j];
    for (int j = threadIdx.x; j < o.uk2; j += blockDim.x)
      uc2_sm[k][j] = o.cscale * o.uc2[j];
  }
  __syncthreads();

  double acc[M];
#pragma unroll
  for (int d = 0; d < M; ++d) acc[d] = 0.0;
  const int nd = a.ndots;
  const int k0 = a.nblocks > 0 ? a.b[0].k : 0;
  const int k1 = a.nblocks > 1 ? a.b[1].k : 0;
  const int64_t n = a.n;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t tile = 32 * U;
  const int64_t wstride = (((int64_t)gridDim.x * blockDim.x) >> 5) * tile;

  for (int64_t i0 = gw * tile + lane; i0 - lane < n; i0 += wstride) {
    double ov[LG_MAXO][U];
#pragma unroll
    for (int k = 0; k < LG_MAXO; ++k) {
      if (a.o[k].out) {
        output_u<U>(a.o[k], coef[k], uc_sm[k], uc2_sm[k], i0, n, ov, post[k], pmode[k], ov[k]);
        double* out = a.o[k].out;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i0 + 32 * u < n) out[i0 + 32 * u] = ov[k][u];
      }
    }
    if constexpr (NA > 0) {
      double bv0[U], bv1[U];
      if (k0) operand<U>(a.b[0].v, i0, n, ov, bv0);
      if (k1) operand<U>(a.b[1].v, i0, n, ov, bv1);
#pragma unroll
      for (int s = 0; s < NA; ++s) {
        if (s < nd) {
          double x[U], y[U];
          operand<U>(a.da[s], i0, n, ov, x);
          if (a.dc[s]) {
            double c[U];
            operand<U>(a.dc[s], i0, n, ov, c);
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] -= c[u];
          }
          if (a.db[s]) {
            operand<U>(a.db[s], i0, n, ov, y);
          } else {
#pragma unroll
            for (int u = 0; u < U; ++u) y[u] = x[u];
          }
#pragma unroll
          for (int u = 0; u < U; ++u) acc[s] += x[u] * y[u];
        } else if (s < nd + k0) {
          double q[U];
          load_u<U>(a.b[0].q + (int64_t)(s - nd) * a.b[0].ld, i0, n, q);
#pragma unroll
          for (int u = 0; u < U; ++u) acc[s] += bv0[u] * q[u];
        } else if (s < nd + k0 + k1) {
          double q[U];
          load_u<U>(a.b[1].q + (int64_t)(s - nd - k0) * a.b[1].ld, i0, n, q);
#pragma unroll
          for (int u = 0; u < U; ++u) acc[s] += bv1[u] * q[u];
        }
      }
    }
  }
  if constexpr (NA > 0) {
    const bool fin = grid_reduce<NA>(acc, nd + k0 + k1, ws, a.result, red_sm);
    if constexpr (PROG) {
      if (fin) cta_run_program(pd.p, pd.sg, pd.fg);
    }
  }
}

template <int NA, bool PROG>
static int launch_fused(const FusedDev& a, lg_ws* ws, cudaStream_t s, const ProgDev* pd) {
  // one resident wave at most (the grid-stride tiles cover the rest)
  static int cap = 0;
  if (!cap) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_kernel<NA, PROG>, kThreads,
                                                      0) != cudaSuccess ||
        occ < 1)
      occ = 1;
    cap = std::min(occ * dev_info().sm_count, kMaxRedBlocks);
  }
  constexpr int U = fused_u<NA>();
  const int64_t want = (a.n + (int64_t)kThreads * U - 1) / ((int64_t)kThreads * U);
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(want, cap));
  static thread_local ProgDev none{};
  fused_kernel<NA, PROG><<<g, kThreads, 0, s>>>(a, *ws, pd ? *pd : none);
  LG_LAUNCH_CHECK("fused_kernel");
  return LG_OK;
}

// ---------------------------------------------------------------- GEMM --
constexpr int kGemmMaxM = 64;
constexpr int kGemmMaxP = 32;
constexpr int kGemmMaxY = 1024;
struct GemmArgs {
  int64_t n;
  const double* in;
  int64_t ldi;
  int m;
  int p;
  double* out;
  int64_t ldo;
  int acc;  // add into out (a later row panel of Y)
  double y[kGemmMaxY];
};

template <int P>
__global__ void __launch_bounds__(kThreads) gemm_small_kernel(const __grid_constant__ GemmArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += stride) {
    double acc[P];
#pragma unroll
    for (int c = 0; c < P; ++c) acc[c] = (a.acc && c < a.p) ? a.out[i + (int64_t)c * a.ldo] : 0.0;
    for (int j = 0; j < a.m; ++j) {
      double v = a.in[i + (int64_t)j * a.ldi];
#pragma unroll
      for (int c = 0; c < P; ++c)
        if (c < a.p) acc[c] += v * a.y[j + c * a.m];
    }
#pragma unroll
    for (int c = 0; c < P; ++c)
      if (c < a.p) a.out[i + (int64_t)c * a.ldo] = acc[c];
  }
}

__global__ void diag_apply_kernel(int64_t n, const double* dinv,
                                  const double* r, double* z, const int* skip) {
  if (skip && *skip) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride)
    z[i] = r[i] * dinv[i];
}

}  // namespace lg

using namespace lg;

extern "C" {

static int fused_dispatch(const lg_fused_args* args, lg_ws* ws, void* stream,
                          const ProgDev* pd) {
  if (!args) return fail(LG_EINVAL, "lg_fused: NULL args");
  const lg_fused_args& a = *args;
  if (a.n < 0) return fail(LG_EINVAL, "lg_fused: negative n");
  if (a.ndots < 0 || a.ndots > LG_MAXD || a.nblocks < 0 || a.nblocks > LG_MAXB)
    return fail(LG_EINVAL, "lg_fused: too many dots / blocks");
  int nq = 0;
  for (int b = 0; b < a.nblocks; ++b) {
    if (a.b[b].k < 0 || (a.b[b].k > 0 && (!a.b[b].q || !a.b[b].v || a.b[b].ld < a.n)))
      return fail(LG_EINVAL, "lg_fused: bad block");
    nq += a.b[b].k;
  }
  if (nq > LG_MAXQ) return fail(LG_EINVAL, "lg_fused: more than LG_MAXQ block columns");
  for (int k = 0; k < LG_MAXO; ++k) {
    const lg_output& o = a.o[k];
    if (!o.out) continue;
    if (o.nterms < 0 || o.nterms > LG_MAXT) return fail(LG_EINVAL, "lg_fused: bad term count");
    for (int t = 0; t < o.nterms; ++t) {
      if (!o.t[t].v) return fail(LG_EINVAL, "lg_fused: NULL term vector");
      uintptr_t u = (uintptr_t)o.t[t].v;
      if (u >= 1 && u <= LG_MAXO && (int)u > k)
        return fail(LG_EINVAL, "lg_fused: term references a later output");
      if (u >= 1 && u <= LG_MAXO && !a.o[u - 1].out)
        return fail(LG_EINVAL, "lg_fused: term references a disabled output");
    }
    if (o.post_mode < 0 || o.post_mode > 3 || (o.post_mode && !o.d_post))
      return fail(LG_EINVAL, "lg_fused: bad post scaling");
    if (o.uk < 0 || o.uk > LG_MAXQ || (o.uk > 0 && (!o.uq || !o.uc || o.uld < a.n)))
      return fail(LG_EINVAL, "lg_fused: bad update block");
    if (o.uk2 < 0 || o.uk2 > LG_MAXQ || (o.uk2 > 0 && (!o.uq2 || !o.uc2 || o.uld2 < a.n)))
      return fail(LG_EINVAL, "lg_fused: bad second update block");
  }
  for (int d = 0; d < a.ndots; ++d)
    if (!a.da[d]) return fail(LG_EINVAL, "lg_fused: NULL dot operand");
  int na = a.ndots + nq;
  if (na > 0 && (!a.result || !ws)) return fail(LG_EINVAL, "lg_fused: dots need result and ws");
  if (a.n == 0 && !pd) {
    if (na > 0) LG_CUDA(cudaMemsetAsync(a.result, 0, sizeof(double) * na, (cudaStream_t)stream));
    return LG_OK;
  }
  FusedDev d;
  d.n = a.n;
  for (int k = 0; k < LG_MAXO; ++k) d.o[k] = a.o[k];
  d.ndots = a.ndots;
  for (int k = 0; k < LG_MAXD; ++k) {
    d.da[k] = a.da[k];
    d.db[k] = a.db[k];
    d.dc[k] = a.dc[k];
  }
  d.nblocks = a.nblocks;
  d.b[0] = a.b[0];
  d.b[1] = a.b[1];
  for (int b = a.nblocks; b < LG_MAXB; ++b) d.b[b].k = 0;
  d.result = a.result;
  d.skip = a.skip;
  lg_ws dummy{};
  lg_ws* w = ws ? ws : &dummy;
  cudaStream_t s = (cudaStream_t)stream;
  if (pd) {
    if (na == 0) return fail(LG_EINVAL, "lg_fused_prog: the pass needs dot products");
    if (na <= 4) return launch_fused<4, true>(d, w, s, pd);
    if (na <= 8) return launch_fused<8, true>(d, w, s, pd);
    if (na <= 16) return launch_fused<16, true>(d, w, s, pd);
    return launch_fused<LG_MAXD + LG_MAXQ, true>(d, w, s, pd);
  }
  if (na == 0) return launch_fused<0, false>(d, w, s, nullptr);
  if (na <= 4) return launch_fused<4, false>(d, w, s, nullptr);
  if (na <= 8) return launch_fused<8, false>(d, w, s, nullptr);
  if (na <= 16) return launch_fused<16, false>(d, w, s, nullptr);
  if (na <= 32) return launch_fused<32, false>(d, w, s, nullptr);
  return launch_fused<LG_MAXD + LG_MAXQ, false>(d, w, s, nullptr);
}

int lg_fused(const lg_fused_args* args, lg_ws* ws, void* stream) {
  return fused_dispatch(args, ws, stream, nullptr);
}

int lg_fused_prog(const lg_fused_args* args, double* slots, int* flags, const uint8_t* prog_h,
                  int nops, const double* imm_h, int nimm, lg_ws* ws, void* stream) {
  if (!slots || !flags || nops < 0 || nops > LG_MAXOPS || nimm < 0 || nimm > LG_MAXIMM ||
      (nops > 0 && !prog_h) || (nimm > 0 && !imm_h))
    return fail(LG_EINVAL, "lg_fused_prog: bad program");
  static thread_local ProgDev pd;
  pd.p.nops = nops;
  std::memcpy(pd.p.ops, prog_h, 4 * (size_t)nops);
  if (nimm) std::memcpy(pd.p.imm, imm_h, sizeof(double) * (size_t)nimm);
  pd.sg = slots;
  pd.fg = flags;
  return fused_dispatch(args, ws, stream, &pd);
}

int lg_gemm_small(int64_t n, const double* in, int64_t ldi, int m,
                  const double* y_h, int p, double* out, int64_t ldo,
                  void* stream) {
  if (n < 0 || m < 0 || p < 0) return fail(LG_EINVAL, "lg_gemm_small: bad shape");
  if (n == 0 || p == 0) return LG_OK;
  if (!out || ldo < n || (m > 0 && (!in || !y_h || ldi < n)))
    return fail(LG_EINVAL, "lg_gemm_small: bad pointer / leading dimension");
  // Tiles of <= 32 output columns x <= 1024 / width input columns, each one
  // launch with its Y tile by value; later input tiles accumulate into out,
  // so every output keeps the sequential j order of a single pass.
  static thread_local GemmArgs a;  // large by-value launch parameter (host staging)
  cudaStream_t s = (cudaStream_t)stream;
  const int g = vec_grid(n);
  for (int c0 = 0; c0 < p; c0 += kGemmMaxP) {
    const int pw = std::min(kGemmMaxP, p - c0);
    const int mt = std::min(kGemmMaxM, kGemmMaxY / pw);
    for (int j0 = 0; j0 < std::max(m, 1); j0 += mt) {
      const int mw = std::min(mt, m - j0);
      a.n = n;
      a.in = in + (int64_t)j0 * ldi;
      a.ldi = ldi;
      a.m = std::max(mw, 0);
      a.p = pw;
      a.out = out + (int64_t)c0 * ldo;
      a.ldo = ldo;
      a.acc = j0 > 0;
      for (int c = 0; c < pw; ++c)
        for (int j = 0; j < a.m; ++j) a.y[j + c * a.m] = y_h[(j0 + j) + (int64_t)(c0 + c) * m];
      if (pw <= 4) gemm_small_kernel<4><<<g, kThreads, 0, s>>>(a);
      else if (pw <= 8) gemm_small_kernel<8><<<g, kThreads, 0, s>>>(a);
      else if (pw <= 16) gemm_small_kernel<16><<<g, kThreads, 0, s>>>(a);
      else gemm_small_kernel<32><<<g, kThreads, 0, s>>>(a);
      LG_LAUNCH_CHECK("gemm_small_kernel");
    }
  }
  return LG_OK;
}

int lg_diag_apply(int64_t n, const double* dinv, const double* r, double* z,
                  const int* skip, void* stream) {
  if (n < 0 || (n > 0 && (!dinv || !r || !z))) return fail(LG_EINVAL, "lg_diag_apply: bad argument");
  if (n == 0) return LG_OK;
  diag_apply_kernel<<<vec_grid(n), kThreads, 0, (cudaStream_t)stream>>>(n, dinv, r, z, skip);
  LG_LAUNCH_CHECK("diag_apply_kernel");
  return LG_OK;
}

}  // extern "C"
