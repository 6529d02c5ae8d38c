// lg_spmv.cu -- CSR upload, nnz-balanced row-block schedule, fused SpMV.
//
// Replaces sparse.py:128-139 (y[nz] = add.reduceat(values * x[col_idx], ...)).
//
// Design (HBM-bound, arithmetic intensity 2 flops / 12 bytes):
//   * the matrix is cut at upload time into row blocks of at most kChunk
//     nonzeros (and kRowCap rows); a row longer than kChunk (power-law hubs:
//     107,553 nonzeros in C4's largest row) is split into parts of kChunk.
//     Every block therefore streams the same number of bytes, which is what
//     balances degree-skewed graphs.
//   * a persistent grid (CTAs = SMs x resident CTAs) walks the blocks
//     round-robin.  A normal block first streams its values / column indices
//     coalesced and stores val*x[col] into shared memory, then reduces rows
//     from shared memory with 1..32 lanes per row (chosen per block from its
//     mean row length at upload time).  A long-row part reduces in registers
//     and publishes one partial; the last part to arrive (atomic ticket) sums
//     the parts in part order.  Summation order is fixed, so y is bitwise
//     reproducible.
//   * the epilogue fuses the theta shift (JD's L - theta I, pcg.py:171-172)
//     and dot products of y with up to LG_MAXD vectors and a column block Q
//     (the Q^T y half of the next deflation projection, pcg.py:60).
//   * packed Laplacian format (default when it applies): a graph Laplacian's
//     off-diagonal values are -w for a handful of distinct weights (unit
//     graphs: one; C4's Geometric(0.5) counts: 30), so each off-diagonal
//     nonzero is one 32-bit word -- column in the low cbits, index into a
//     value table (shared memory) in the high bits -- and the diagonal is a
//     separate n-vector.  4 bytes per nonzero instead of 12 (f64 value +
//     int32 column): the SpMV streams 2.2x fewer bytes on C4 and the value
//     actually multiplied is bit-identical to the stored one.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "lg_common.cuh"

namespace lg {

// Warp-block schedule (built once per operator on the host, O(n + nnz/8)).
// A normal block is at most kWin stream positions of whole rows; its window
// starts at the 16-byte-aligned position at or below its first nonzero, so a
// lane's eight words are two aligned 128-bit loads.  A row longer than
// kLongPart (power-law hubs: 107,553 nonzeros in C4's largest row) is cut into
// parts of kLongPart from its first nonzero.  Every block therefore streams
// about the same bytes, which is what balances degree-skewed graphs.
constexpr int kWPer = 8;                 // stream words per lane
constexpr int kWin = 32 * kWPer;         // window of one warp block (positions)
constexpr int kLongPart = kWin - 4;      // part length of a long row
constexpr int kWRows = 256;              // rows per normal block (8-bit offsets)
constexpr int kWThreads = 256;           // CTA size of the SpMV (8 warps)
#ifndef LG_SPMV_MINB
#define LG_SPMV_MINB 4                   // resident CTAs per SM (register cap 64)
#endif
#ifndef LG_SPMV_PIPE
#define LG_SPMV_PIPE 1                   // next block's loads before this block's work
#endif
constexpr int kST = 128;                 // CTA size of the build kernels
// every stream array (pcol / col / val) is allocated with this many slack
// entries, so a lane's two 128-bit loads never leave the allocation
constexpr int64_t kStreamPad = 8;

enum : int32_t { kBlkLong = -1, kBlkSeg = 0, kBlkRows = 1 };

// -DLG_SPMV_CHECK: bounds-check every index the SpMV kernel uses (debug)
#ifdef LG_SPMV_CHECK
#define LG_CK(c, what)                                                                 \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      printf("lg_spmv check failed: %s (block %d thread %d)\n", what, blockIdx.x,      \
             threadIdx.x);                                                             \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define LG_CK(c, what) do { } while (0)
#endif

struct SpmvBlock {
  int64_t nz0, nz1;  // nonzero range
  int32_t row0;      // first row
  int32_t nrows;     // rows (normal) / long-row id (long)
  int32_t lshift;    // kind: kBlkLong part, kBlkSeg segmented, kBlkRows row-serial
  int32_t part;      // compact long-part slot (long)
  // kBlkSeg: per lane, bits 0-7 flag the window positions where a row starts,
  // bits 8-15 the row (relative to row0) of the lane's first valid position
  uint16_t meta[32];
};

}  // namespace lg

struct lg_csr {
  int64_t n = 0, nnz = 0;
  int64_t* row_ptr = nullptr;  // device [n+1]
  int32_t* col = nullptr;      // device [nnz]
  double* val = nullptr;       // device [nnz]
  lg::SpmvBlock* blocks = nullptr;
  int64_t nblocks = 0;
  int64_t nlong = 0;
  int64_t nparts = 0;              // total long-row parts
  // packed Laplacian format (see header)
  int packed = 0;
  int cbits = 0;
  int nvals = 0;
  int64_t noff = 0;                // off-diagonal nonzeros
  int64_t* prp = nullptr;          // off-diagonal row pointers [n+1]
  uint32_t* pcol = nullptr;        // col | vidx << cbits
  double* pdiag = nullptr;         // diagonal [n]
  double* table = nullptr;         // distinct off-diagonal values [nvals]
  int intw = 0;                    // table[i] == -(i + 1) for every i (integer weights)
  int32_t* long_nparts = nullptr;  // device [nlong]
  int64_t* long_first = nullptr;   // device [nlong] slot of part 0
  int32_t* long_row = nullptr;     // device [nlong] schedule row of each long row
  // row chunks of the schedule for the host-buffer path (lg_spmv_host):
  // blocks [chunk_b[c], chunk_b[c+1]) cover rows [chunk_row[c], chunk_row[c+1])
  int nchunks = 0;
  int64_t chunk_b[9] = {};
  int64_t chunk_row[9] = {};
  // column panels of a full operator (lg_csr_set_panels): when set, lg_spmv
  // runs y = P_0 x - theta x, y += P_k x instead of the one-pass product
  int npanels = 0;
  lg_csr* panel[16] = {};
  // rows absent from the schedule (SKIP_EMPTY, row blocks, split halves):
  // such an operator is not a full operator and cannot be panelled
  int is_block = 0;
  // compacted schedule (an operator whose rows with entries are scattered,
  // e.g. a column panel): schedule row i is matrix row rowmap[i]
  int32_t* rowmap = nullptr;       // device [rows with entries] or NULL
  int64_t nrows_sched = 0;         // rows the schedule writes (present rows)
  // columns a column panel reads (x[pf_c0:pf_c1] is what it prefetches)
  int64_t pf_c0 = 0, pf_c1 = 0;
};

namespace lg {

constexpr int kMaxTable = 2048;   // value-table entries kept in shared memory
// long-row parts from which the deferred finish (one more launch) beats a
// ticket per part: measured C5 13.6 -> 9.6 ms, C3 35.4 -> 33.8 us, C4 equal
constexpr int64_t kDeferParts = 1;

struct SpmvArgs {
  int64_t n;
  const int64_t* row_ptr;   // plain: row_ptr; packed: off-diagonal row ptr
  const int32_t* col;
  const double* val;
  const uint32_t* pcol;     // packed entries (NULL: plain format)
  const double* pdiag;
  const double* table;
  int nvals;
  int cbits;
  int intw;                 // value of index i is -(i + 1): computed, no table
  int64_t nzs;              // stream length (bounds the 128-bit loads)
  const SpmvBlock* blocks;
  int64_t nblocks;
  const int32_t* long_nparts;
  const int64_t* long_first;
  const int32_t* long_row;
  int defer_long;           // parts only publish; long_finish_kernel sums them
  const double* x;
  double* y;
  int accum;        // y += A x (the second half of a split row block)
  double theta_h;
  const double* theta_d;
  int theta_neg;
  const int* skip;
  const int32_t* rowmap;   // schedule row -> matrix row (NULL: identity)
  // L2 prefetch regions issued at kernel start (x, diagonal): the gathers of
  // a cold x then hit L2 instead of paying DRAM latency one sector at a time
  const void* pf[2];
  int64_t pf_bytes[2];
  int64_t nparts, nlong;    // bounds (LG_SPMV_CHECK builds)
  double* long_part;   // [nparts] partial of each long-row part
  unsigned* long_ticket;  // [nlong]
};

// One lane's eight stream positions [p, p + 8): two aligned 128-bit loads
// (the window may start up to 3 positions before the block and run past its
// end -- those positions are masked -- and the arrays carry kStreamPad slack
// entries, so the loads never leave the allocation).
template <bool PACKED>
struct WWords {
  uint32_t w[kWPer];
  double v[PACKED ? 1 : kWPer];
};

template <bool PACKED>
__device__ __forceinline__ void wload(const SpmvArgs& a, int64_t p, WWords<PACKED>& L) {
  LG_CK(p >= 0 && p + kWPer <= a.nzs + kStreamPad, "stream window");
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t q = p + 4 * h;
    uint4 u;
    if constexpr (PACKED) u = __ldcs(reinterpret_cast<const uint4*>(a.pcol + q));
    else u = __ldcs(reinterpret_cast<const uint4*>(a.col + q));
    L.w[4 * h] = u.x; L.w[4 * h + 1] = u.y; L.w[4 * h + 2] = u.z; L.w[4 * h + 3] = u.w;
    if constexpr (!PACKED) {
      const double2 v0 = __ldcs(reinterpret_cast<const double2*>(a.val + q));
      const double2 v1 = __ldcs(reinterpret_cast<const double2*>(a.val + q + 2));
      L.v[4 * h] = v0.x; L.v[4 * h + 1] = v0.y; L.v[4 * h + 2] = v1.x; L.v[4 * h + 3] = v1.y;
    }
  }
}

// products of the valid positions (vm bit j) of one lane's window; the eight
// gathers are issued before any multiply
template <bool PACKED>
__device__ __forceinline__ void wproducts(const SpmvArgs& a, const WWords<PACKED>& L,
                                          unsigned vm, const double* tab, uint32_t cmask,
                                          double (&p)[kWPer]) {
  double xv[kWPer];
#pragma unroll
  for (int j = 0; j < kWPer; ++j) {
    const uint32_t c = PACKED ? (L.w[j] & cmask) : L.w[j];
    if ((vm >> j) & 1u) LG_CK(c < (uint32_t)a.n, "gather column");
    xv[j] = ((vm >> j) & 1u) ? __ldg(a.x + c) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < kWPer; ++j) {
    if constexpr (PACKED)
      p[j] = a.intw ? -(xv[j] * __uint2double_rn((L.w[j] >> a.cbits) + 1u))
                    : xv[j] * tab[((vm >> j) & 1u) ? (L.w[j] >> a.cbits) : 0u];
    else p[j] = ((vm >> j) & 1u) ? L.v[j] * xv[j] : 0.0;
  }
}

template <bool PACKED>
__device__ __forceinline__ void finish_row(const SpmvArgs& a, int64_t r, double s,
                                           double theta) {
  if (a.rowmap) r = a.rowmap[r];
  LG_CK(r >= 0 && r < a.n, "row");
  if constexpr (PACKED) {
    if (a.pdiag) s += a.pdiag[r] * __ldg(a.x + r);  // NULL: accumulating column panel
  }
  if (theta != 0.0) s -= theta * __ldg(a.x + r);
  if (a.accum) s = a.y[r] + s;
  a.y[r] = s;
}

// y = A x - theta x (y += ... when accum).  Persistent grid; warp w of the
// grid takes blocks w, w + W, ... (W warps in the grid).  A segmented block:
// each lane multiplies its eight positions, folds them into row segments in
// registers (left to right), and the warp joins segments that cross lanes
// with a segmented inclusive scan over shuffles; the lane holding a row's
// last position writes it.  No shared memory, no barrier.  Summation order is
// fixed by the schedule, so y is bitwise reproducible.
//
// Software pipeline (the loop is latency-bound: descriptor -> stream words ->
// gathers -> row writes is a chain of dependent memory round trips): while a
// block's gathers are in flight the warp decodes the next block's descriptor,
// issues that block's stream loads, and loads the descriptor after it.  A
// descriptor is read with one coalesced 96-byte load (a word per lane) and
// decoded by shuffles.
struct WDesc {
  int64_t nz0, nz1;
  int32_t row0, nrows, kind, part;
  uint32_t meta;
};

__device__ __forceinline__ uint32_t desc_word(const SpmvArgs& a, int64_t b, int lane) {
  constexpr int kWords = (int)(sizeof(SpmvBlock) / 4);
  return (b < a.nblocks && lane < kWords)
             ? __ldcs(reinterpret_cast<const unsigned int*>(a.blocks + b) + lane)
             : 0u;
}

__device__ __forceinline__ WDesc desc_decode(uint32_t w, int lane) {
  WDesc d;
  const unsigned m = 0xffffffffu;
  d.nz0 = (int64_t)(((uint64_t)__shfl_sync(m, w, 1) << 32) | __shfl_sync(m, w, 0));
  d.nz1 = (int64_t)(((uint64_t)__shfl_sync(m, w, 3) << 32) | __shfl_sync(m, w, 2));
  d.row0 = (int32_t)__shfl_sync(m, w, 4);
  d.nrows = (int32_t)__shfl_sync(m, w, 5);
  d.kind = (int32_t)__shfl_sync(m, w, 6);
  d.part = (int32_t)__shfl_sync(m, w, 7);
  const uint32_t mw = __shfl_sync(m, w, 8 + (lane >> 1));
  d.meta = (lane & 1) ? (mw >> 16) : (mw & 0xffffu);
  return d;
}

__device__ __forceinline__ unsigned valid_mask(const WDesc& d, int lane) {
  if (d.kind == kBlkRows || d.nz1 <= d.nz0) return 0u;
  // the block's positions relative to its window: [lo, hi), lo <= 3, hi <= kWin
  const int lo = (int)(d.nz0 & 3) - kWPer * lane;
  const int hi = (int)(d.nz1 - (d.nz0 & ~(int64_t)3)) - kWPer * lane;
  const int a = min(max(lo, 0), kWPer), b = min(max(hi, 0), kWPer);
  return ((1u << b) - 1u) & ~((1u << a) - 1u);
}

// One block of the schedule, its products p already formed (any kind).
template <bool PACKED>
__device__ __forceinline__ void process_block(const SpmvArgs& a, const WDesc& d, unsigned vm,
                                              const double (&p)[kWPer], int lane, double theta,
                                              double* slot, const double* tab_sm,
                                              uint32_t cmask) {
  const int64_t row0 = d.row0;
  if (d.kind == kBlkRows) {
    // rows with no stored entry (or other irregular blocks): lane per row
    for (int i = lane; i < d.nrows; i += 32) {
      const int64_t r = row0 + i;
      double s = 0.0;
      for (int64_t k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) {
        if constexpr (PACKED) {
          const uint32_t w = a.pcol[k];
          s += tab_sm[w >> a.cbits] * __ldg(a.x + (w & cmask));
        } else {
          s += a.val[k] * __ldg(a.x + a.col[k]);
        }
      }
      finish_row<PACKED>(a, r, s, theta);
    }
  } else if (d.kind == kBlkLong) {
    // part of a long row: lane sums left to right, butterfly, ordered finish
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kWPer; ++j) s += p[j];
    s = warp_sum(s);
    unsigned last = 0u;
    const int lr = d.nrows;
    if (a.defer_long) {   // long_finish_kernel sums the parts after this launch
      if (lane == 0) a.long_part[d.part] = s;
    } else if (lane == 0) {
      LG_CK(d.part >= 0 && d.part < a.nparts && lr >= 0 && lr < a.nlong, "long part");
      a.long_part[d.part] = s;
      // release: the partial is visible before the ticket moves
      unsigned arrived;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;"
                   : "=r"(arrived) : "l"(a.long_ticket + lr) : "memory");
      last = arrived == (unsigned)a.long_nparts[lr] - 1u;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      // the last part to arrive sums every part lane-strided, then by
      // butterfly: fixed order whatever the arrival order
      __threadfence();
      const int64_t first = a.long_first[lr];
      const int np = a.long_nparts[lr];
      double t = 0.0;
      for (int q = lane; q < np; q += 32) t += ld_cg(a.long_part + first + q);
      t = warp_sum(t);
      if (lane == 0) {
        finish_row<PACKED>(a, row0, t, theta);
        a.long_ticket[lr] = 0u;
      }
    }
  } else {
    // ---- segmented block: each completed row's sum goes to the warp's slot
    // array (by row offset); one coalesced pass then finishes the rows
    // (diagonal, shift, accumulation, store).  Branch-free: running sums
    // c_j restart at every row start (flag F_j), the warp joins the lanes'
    // open tails with a segmented scan, and a row ends at position j when
    // j is valid and position j + 1 starts a row or ends the block.
    const unsigned F = d.meta & vm & 0xffu;
    // row ends: the next position (next lane's first for j = 7) starts a
    // row, or j is the block's last position
    const unsigned nf = __shfl_down_sync(0xffffffffu, F & 1u, 1);
    const int last = (int)(d.nz1 - 1 - (d.nz0 & ~(int64_t)3)) - kWPer * lane;
    unsigned E = vm & ((F >> 1) | ((lane < 31 ? nf : 0u) << (kWPer - 1)));
    if (last >= 0 && last < kWPer) E |= 1u << last;
    // positions before the lane's first row start continue a row from the
    // lanes before (the head row: its sum needs their carry)
    const unsigned before = F ? ((F & (0u - F)) - 1u) : 0xffu;
    const int rfirst = (int)(d.meta >> 8);
    const int fv = __ffs(vm) - 1;
    // row of position j: rfirst + (row starts in (fv, j])
    const unsigned fcount = F & ~(1u << (fv & 31));
    double run = 0.0, headv = 0.0;
    bool head_end = false;
#pragma unroll
    for (int j = 0; j < kWPer; ++j) {
      run = (((F >> j) & 1u) ? 0.0 : run) + p[j];
      if ((E >> j) & 1u) {
        if ((before >> j) & 1u) {
          headv = run;
          head_end = true;
        } else {
          const int r = rfirst + __popc(fcount & ((2u << j) - 1u));
          LG_CK(r >= 0 && r < d.nrows, "slot");
          slot[r] = run;
        }
      }
    }
    // segmented inclusive scan of the lanes' open tails
    double v = run;
    bool f = F != 0u;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const double vu = __shfl_up_sync(0xffffffffu, v, dd);
      const bool fu = __shfl_up_sync(0xffffffffu, (int)f, dd) != 0;
      if (lane >= dd && !f) {
        v = vu + v;
        f = fu;
      }
    }
    double cprev = __shfl_up_sync(0xffffffffu, v, 1);
    if (lane == 0) cprev = 0.0;
    if (head_end) slot[rfirst] = cprev + headv;
    __syncwarp();
    for (int i = lane; i < d.nrows; i += 32) finish_row<PACKED>(a, row0 + i, slot[i], theta);
    __syncwarp();
  }
}

template <bool PACKED>
__global__ void __launch_bounds__(kWThreads, PACKED ? LG_SPMV_MINB : 3) wspmv_kernel(SpmvArgs a) {
  if (a.skip && *a.skip) return;
  // each CTA prefetches its share of the prefetch regions into L2 (bulk
  // copy engine, 16-byte granules, one instruction per 32 KB piece)
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (a.pf_bytes[r] <= 0) continue;
    const int64_t g16 = (a.pf_bytes[r] + 15) >> 4;
    const int64_t per = (g16 + gridDim.x - 1) / gridDim.x;
    const int64_t lo = per * blockIdx.x, hi = g16 < lo + per ? g16 : lo + per;
    for (int64_t q = lo + (int64_t)threadIdx.x * 2048; q < hi; q += (int64_t)kWThreads * 2048) {
      const uint32_t bytes = (uint32_t)(16 * (hi - q < 2048 ? hi - q : (int64_t)2048));
      const char* src = static_cast<const char*>(a.pf[r]) + 16 * q;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
    }
  }
  extern __shared__ double tab_sm[];   // packed value table (max(nvals, 1) entries)
  if constexpr (PACKED) {
    // entry 0 always exists: masked positions read it (branch-free products)
    for (int i = threadIdx.x; i < max(a.nvals, 1); i += kWThreads)
      tab_sm[i] = i < a.nvals ? a.table[i] : 0.0;
    __syncthreads();
  }
  double theta = a.theta_h;
  if (a.theta_d) theta += a.theta_neg ? -*a.theta_d : *a.theta_d;
  const int lane = threadIdx.x & 31;
  const uint32_t cmask = PACKED ? ((a.cbits >= 32) ? 0xffffffffu : ((1u << a.cbits) - 1u)) : 0u;
  const int64_t nw = (int64_t)gridDim.x * (kWThreads / 32);
  int64_t b = (int64_t)blockIdx.x * (kWThreads / 32) + (threadIdx.x >> 5);
  __shared__ double rsum[kWThreads / 32][kWRows];   // per warp: row sums of a block
  double* slot = rsum[threadIdx.x >> 5];
  if (b >= a.nblocks) return;
  // pipeline prologue: current descriptor + words, next descriptor word
  WDesc d = desc_decode(desc_word(a, b, lane), lane);
  unsigned vm = valid_mask(d, lane);
  WWords<PACKED> W;
  if (vm) wload<PACKED>(a, (d.nz0 & ~(int64_t)3) + kWPer * lane, W);
  uint32_t wnext = desc_word(a, b + nw, lane);
  while (true) {
    // gathers of the current block
    double p[kWPer];
    wproducts<PACKED>(a, W, vm, tab_sm, cmask, p);
    // next block: decode, issue its stream words; load the descriptor after
    // (LG_SPMV_PIPE=0 builds issue them after this block instead)
    const int64_t bn = b + nw;
    WDesc dn;
    unsigned vmn = 0u;
    WWords<PACKED> Wn;
    auto next_loads = [&]() {
      dn = desc_decode(wnext, lane);
      vmn = bn < a.nblocks ? valid_mask(dn, lane) : 0u;
      if (vmn) wload<PACKED>(a, (dn.nz0 & ~(int64_t)3) + kWPer * lane, Wn);
      wnext = desc_word(a, bn + nw, lane);
    };
    if constexpr (LG_SPMV_PIPE) next_loads();
    process_block<PACKED>(a, d, vm, p, lane, theta, slot, tab_sm, cmask);
    if (bn >= a.nblocks) break;
    if constexpr (!LG_SPMV_PIPE) next_loads();
    b = bn;
    d = dn;
    vm = vmn;
    W = Wn;
  }
}

// Deferred long rows (SpmvArgs.defer_long): after the product kernel, one warp
// per long row sums its parts lane-strided then by butterfly -- the same
// order as the ticket finish, so the same bits -- and finishes the row.  One
// extra launch instead of an atomic ticket and a release per part (C5: ~7 M
// parts a product).
template <bool PACKED>
__global__ void __launch_bounds__(256) long_finish_kernel(SpmvArgs a) {
  if (a.skip && *a.skip) return;
  double theta = a.theta_h;
  if (a.theta_d) theta += a.theta_neg ? -*a.theta_d : *a.theta_d;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t lr = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; lr < a.nlong;
       lr += nw) {
    const int64_t first = a.long_first[lr];
    const int np = a.long_nparts[lr];
    double t = 0.0;
    for (int q = lane; q < np; q += 32) t += a.long_part[first + q];
    t = warp_sum(t);
    if (lane == 0) finish_row<PACKED>(a, a.long_row[lr], t, theta);
  }
}

// Measurement aid (lg_spmv_gather_probe): the x gathers of an operator's
// off-diagonal stream and nothing else -- no values, no row structure, no y --
// eight independent gathers in flight per thread.  Its time is the floor any
// SpMV on this stream pays for x[col] alone (bench.py reports the product
// against it next to the HBM roofline).
__global__ void __launch_bounds__(256) gather_probe_kernel(const uint32_t* __restrict__ words,
                                                            uint32_t cmask, int64_t m,
                                                            const double* __restrict__ x,
                                                            double* out) {
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#pragma unroll 8
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
    s += __ldg(x + (__ldcs(words + e) & cmask));
  // keep the loads alive without a store per thread
  if (s == 12345.678) *out = s;
}

// Build the warp-block schedule on the host.
// absent (optional): rows left out of the schedule altogether (y is not
// written there) -- the row block of one rank in the row-partitioned
// multi-GPU SpMV, embedded in the global index space.
static void build_schedule(int64_t n, const int64_t* rp, std::vector<SpmvBlock>& blocks,
                           std::vector<int32_t>& long_nparts,
                           std::vector<int64_t>& long_first,
                           std::vector<int32_t>& long_row,
                           const std::vector<char>* absent = nullptr) {
  int64_t r = 0, part_total = 0;
  blocks.reserve((size_t)(rp[n] / (kWin - 16) + n / kWRows + 16));
  while (r < n) {
    if (absent && (*absent)[(size_t)r]) {
      ++r;
      continue;
    }
    const int64_t len = rp[r + 1] - rp[r];
    if (len > kLongPart) {
      const int32_t np = (int32_t)((len + kLongPart - 1) / kLongPart);
      const int32_t lr = (int32_t)long_nparts.size();
      long_nparts.push_back(np);
      const int64_t slot0 = part_total;
      part_total += np;
      long_first.push_back(slot0);
      long_row.push_back((int32_t)r);
      for (int32_t q = 0; q < np; ++q) {
        SpmvBlock b{};
        b.nz0 = rp[r] + (int64_t)q * kLongPart;
        b.nz1 = std::min(rp[r] + (int64_t)(q + 1) * kLongPart, rp[r + 1]);
        b.row0 = (int32_t)r;
        b.nrows = lr;
        b.lshift = kBlkLong;
        b.part = (int32_t)(slot0 + q);
        blocks.push_back(b);
      }
      ++r;
      continue;
    }
    const int64_t r0 = r, nz0 = rp[r];
    const int64_t cap = kWin - (nz0 & 3);
    bool empty = false;
    while (r < n && r - r0 < kWRows) {
      if (absent && (*absent)[(size_t)r]) break;
      const int64_t l = rp[r + 1] - rp[r];
      if (l > kLongPart || rp[r + 1] - nz0 > cap) break;
      empty |= (l == 0);
      ++r;
    }
    SpmvBlock b{};
    b.nz0 = nz0;
    b.nz1 = rp[r];
    b.row0 = (int32_t)r0;
    b.nrows = (int32_t)(r - r0);
    b.lshift = empty ? kBlkRows : kBlkSeg;
    if (!empty) {
      const int64_t base = nz0 & ~(int64_t)3;
      for (int64_t i = 0; i < r - r0; ++i) {
        const int64_t s = rp[r0 + i] - base;
        b.meta[s >> 3] |= (uint16_t)(1u << (s & 7));
      }
      // row of each lane's first valid position
      int64_t row = 0;
      for (int l = 0; l < 32; ++l) {
        const int64_t fv = std::max<int64_t>(base + kWPer * l, nz0);
        if (fv >= b.nz1) break;
        while (rp[r0 + row + 1] <= fv) ++row;
        b.meta[l] |= (uint16_t)(row << 8);
      }
    }
    blocks.push_back(b);
  }
}

// Split the schedule into up to kHostChunks row chunks of about equal blocks
// (never inside a long row's parts) so the host-buffer path can copy y back
// chunk by chunk while the next chunk is computed.
constexpr int kHostChunks = 4;
static void set_chunks(lg_csr* a, const std::vector<SpmvBlock>& blocks) {
  const int64_t nb = (int64_t)blocks.size();
  a->nchunks = 0;
  if (nb == 0) return;
  int64_t prev = 0;
  a->chunk_b[0] = 0;
  a->chunk_row[0] = 0;
  int c = 0;
  for (int k = 1; k < kHostChunks; ++k) {
    int64_t b = k * nb / kHostChunks;
    while (b < nb && blocks[(size_t)b].lshift == kBlkLong && b > 0 &&
           blocks[(size_t)b - 1].lshift == kBlkLong &&
           blocks[(size_t)b - 1].nrows == blocks[(size_t)b].nrows)
      ++b;   // inside one long row's parts
    if (b <= prev || b >= nb) continue;
    a->chunk_b[++c] = b;
    a->chunk_row[c] = blocks[(size_t)b].row0;
    prev = b;
  }
  a->chunk_b[c + 1] = nb;
  a->chunk_row[c + 1] = a->n;
  a->nchunks = c + 1;
}

// Build the schedule of `a` from host row pointers and upload it (blocks,
// long-row part tables); sets nblocks / nlong / nparts / chunks.
static int attach_schedule(lg_csr* a, const int64_t* rp, const std::vector<char>* absent,
                           const char* who) {
  std::vector<SpmvBlock> blocks;
  std::vector<int32_t> lnp, lrow;
  std::vector<int64_t> lfirst;
  // Present rows in many separate runs (a column panel leaves every row
  // without an entry in its columns absent): schedule the present rows as one
  // compacted sequence and map each back through rowmap, so blocks are not
  // cut at every gap.  A few runs (a rank's row block) keep the plain form.
  std::vector<int32_t> map;
  std::vector<int64_t> crp;
  if (absent) {
    int64_t runs = 0;
    for (int64_t r = 0; r < a->n; ++r)
      runs += !(*absent)[(size_t)r] && (r == 0 || (*absent)[(size_t)r - 1]);
    if (runs > 64) {
      // absent rows hold no entries, so the present rows' entries stay one
      // contiguous stream: compacted row i starts where matrix row map[i] does
      for (int64_t r = 0; r < a->n; ++r) {
        if ((*absent)[(size_t)r]) continue;
        if (rp[r + 1] == rp[r] || (!map.empty() && rp[map.back() + 1] != rp[r])) {
          map.clear();   // an empty present row, or entries between present rows:
                         // keep the plain form
          crp.clear();
          break;
        }
        map.push_back((int32_t)r);
        crp.push_back(rp[r]);
      }
      if (!map.empty()) crp.push_back(rp[map.back() + 1]);
    }
  }
  a->nrows_sched = a->n;
  if (absent) {
    a->nrows_sched = 0;
    for (int64_t r = 0; r < a->n; ++r) a->nrows_sched += !(*absent)[(size_t)r];
  }
  if (!map.empty()) {
    const int64_t nc = (int64_t)map.size();
    build_schedule(nc, crp.data(), blocks, lnp, lfirst, lrow, nullptr);
    if (cudaMalloc(&a->rowmap, 4 * (size_t)nc) != cudaSuccess)
      return fail(LG_ENOMEM, std::string(who) + ": row map alloc");
    LG_CUDA(cudaMemcpy(a->rowmap, map.data(), 4 * (size_t)nc, cudaMemcpyHostToDevice));
  } else {
    build_schedule(a->n, rp, blocks, lnp, lfirst, lrow, absent);
  }
  a->nblocks = (int64_t)blocks.size();
  set_chunks(a, blocks);
  if (a->rowmap && a->nchunks > 1) {   // chunk rows are compacted indices: one chunk
    a->nchunks = 1;
    a->chunk_b[1] = a->nblocks;
    a->chunk_row[1] = a->n;
  }
  a->nlong = (int64_t)lnp.size();
  a->nparts = 0;
  for (int32_t v : lnp) a->nparts += v;
  if ((a->nblocks &&
       cudaMalloc(&a->blocks, sizeof(SpmvBlock) * (size_t)a->nblocks) != cudaSuccess) ||
      (a->nlong && (cudaMalloc(&a->long_nparts, 4 * (size_t)a->nlong) != cudaSuccess ||
                    cudaMalloc(&a->long_first, 8 * (size_t)a->nlong) != cudaSuccess ||
                    cudaMalloc(&a->long_row, 4 * (size_t)a->nlong) != cudaSuccess)))
    return fail(LG_ENOMEM, std::string(who) + ": schedule alloc");
  if (a->nblocks)
    LG_CUDA(cudaMemcpy(a->blocks, blocks.data(), sizeof(SpmvBlock) * blocks.size(),
                       cudaMemcpyHostToDevice));
  if (a->nlong) {
    LG_CUDA(cudaMemcpy(a->long_nparts, lnp.data(), 4 * lnp.size(), cudaMemcpyHostToDevice));
    LG_CUDA(cudaMemcpy(a->long_first, lfirst.data(), 8 * lfirst.size(), cudaMemcpyHostToDevice));
    LG_CUDA(cudaMemcpy(a->long_row, lrow.data(), 4 * lrow.size(), cudaMemcpyHostToDevice));
  }
  return LG_OK;
}

static int ensure_long_ws(lg_ws* ws, const lg_csr* a) {
  if (a->nlong > ws->long_cap) {
    cudaFree(ws->long_dots);
    cudaFree(ws->long_ticket);
    ws->long_dots = nullptr;
    ws->long_ticket = nullptr;
    ws->long_cap = 0;
    LG_CUDA(cudaMalloc(&ws->long_ticket, sizeof(unsigned) * (size_t)a->nlong));
    LG_CUDA(cudaMemset(ws->long_ticket, 0, sizeof(unsigned) * (size_t)a->nlong));
    LG_CUDA(cudaDeviceSynchronize());
    ws->long_cap = a->nlong;
  }
  if (a->nparts > ws->part_cap) {
    cudaFree(ws->long_part);
    ws->long_part = nullptr;
    ws->part_cap = 0;
    LG_CUDA(cudaMalloc(&ws->long_part, sizeof(double) * (size_t)a->nparts));
    ws->part_cap = a->nparts;
  }
  return LG_OK;
}

// Kernel arguments of a product with `m` (no theta, no accumulation).
static SpmvArgs spmv_args(const lg_csr* m, const double* x, double* y, lg_ws* ws) {
  SpmvArgs args{};
  args.n = m->n;
  args.row_ptr = m->packed ? m->prp : m->row_ptr;
  args.col = m->col;
  args.val = m->val;
  args.pcol = m->packed ? m->pcol : nullptr;
  args.pdiag = m->pdiag;
  args.table = m->table;
  args.nvals = m->nvals;
  args.cbits = m->cbits;
  args.intw = m->intw;
  args.nzs = m->packed ? m->noff : m->nnz;
  args.blocks = m->blocks;
  args.nblocks = m->nblocks;
  args.long_nparts = m->long_nparts;
  args.long_first = m->long_first;
  args.long_row = m->long_row;
  {
    static const int defer_env = [] {
      const char* e = getenv("LG_SPMV_DEFER");
      return e ? atoi(e) : -1;
    }();
    args.defer_long = defer_env >= 0 ? (defer_env != 0 && m->nlong > 0)
                                     : (m->nparts >= kDeferParts);
  }
  args.x = x;
  args.y = y;
  args.long_part = ws ? ws->long_part : nullptr;
  args.long_ticket = ws ? ws->long_ticket : nullptr;
  args.rowmap = m->rowmap;
  args.nparts = m->nparts;
  args.nlong = m->nlong;
  // x (and the diagonal) into L2 up front when both fit in a third of it;
  // a column panel prefetches its slice of x (why panels exist: C5)
  static const bool pf_on = [] {
    const char* e = getenv("LG_SPMV_PREFETCH");
    return !(e && atoi(e) == 0);
  }();
  const int64_t l2 = dev_info().l2_bytes > 0 ? dev_info().l2_bytes : (int64_t)126 << 20;
  if (pf_on && x && ((uintptr_t)x & 15) == 0) {
    const int64_t c0 = m->pf_c0 & ~(int64_t)1, c1 = m->pf_c1 > 0 ? m->pf_c1 : m->n;
    const int64_t xb = 8 * (c1 - c0);
    const int64_t db = (m->packed && m->pdiag) ? 8 * m->n : 0;
    if (xb + db <= l2 / 3) {
      args.pf[0] = x + c0;
      args.pf_bytes[0] = xb;
      if (db && ((uintptr_t)m->pdiag & 15) == 0) {
        args.pf[1] = m->pdiag;
        args.pf_bytes[1] = db;
      }
    } else if (xb <= l2 / 3) {
      args.pf[0] = x + c0;
      args.pf_bytes[0] = xb;
    }
  }
  return args;
}

template <bool PACKED>
static int launch_t(const SpmvArgs& args, cudaStream_t s) {
  static thread_local int occ = 0;
  if (!occ) {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, wspmv_kernel<PACKED>, kWThreads,
                                                      sizeof(double) * kMaxTable) !=
            cudaSuccess ||
        o < 1)
      o = 1;
    occ = o;
  }
  const int64_t warps = (int64_t)occ * dev_info().sm_count * (kWThreads / 32);
  const int64_t g = std::max<int64_t>(
      1, std::min<int64_t>((args.nblocks + kWThreads / 32 - 1) / (kWThreads / 32),
                           warps / (kWThreads / 32)));
  const size_t dyn = PACKED ? sizeof(double) * (size_t)std::max(args.nvals, 1) : 0;
  wspmv_kernel<PACKED><<<(unsigned)g, kWThreads, dyn, s>>>(args);
  LG_LAUNCH_CHECK("wspmv_kernel");
  if (args.defer_long && args.nlong > 0) {
    const int64_t gl = std::max<int64_t>(
        1, std::min<int64_t>((args.nlong + 7) / 8, (int64_t)dev_info().sm_count * 8));
    long_finish_kernel<PACKED><<<(unsigned)gl, 256, 0, s>>>(args);
    LG_LAUNCH_CHECK("long_finish_kernel");
  }
  return LG_OK;
}

static int launch(const SpmvArgs& args, cudaStream_t s, bool packed) {
  if (args.nblocks == 0) return LG_OK;
  if ((packed && ((uintptr_t)args.pcol & 15)) ||
      (!packed && (((uintptr_t)args.col & 15) || ((uintptr_t)args.val & 15))))
    return fail(LG_EINVAL, "lg_spmv: stream arrays must be 16-byte aligned");
  return packed ? launch_t<true>(args, s) : launch_t<false>(args, s);
}

// y = A x over the schedule blocks [b0, b1) only (a row chunk; no epilogue).
static int spmv_range(const lg_csr* a, const double* x, double* y, int64_t b0, int64_t b1,
                      lg_ws* ws, cudaStream_t s, int accum = 0) {
  if (b1 <= b0) return LG_OK;
  SpmvArgs args = spmv_args(a, x, y, ws);
  args.accum = accum;
  args.blocks = a->blocks + b0;
  args.nblocks = b1 - b0;
  args.defer_long = 0;   // a chunk finishes its own long rows (tickets)
  return launch(args, s, a->packed != 0);
}

// Packed Laplacian format eligibility: every row stores its diagonal, the
// distinct off-diagonal values fit the bits left above the column index and
// the shared-memory table.
static bool make_packed(int64_t n, const int64_t* rp, const int64_t* col, const double* val,
                        std::vector<int64_t>& prp, std::vector<uint32_t>& pcol,
                        std::vector<double>& diag, std::vector<double>& table, int& cbits) {
  if (n < 1) return false;
  cbits = 1;
  while (((int64_t)1 << cbits) < n) ++cbits;
  if (cbits > 31) return false;
  const int vbits = 32 - cbits;
  const int64_t maxvals = std::min<int64_t>((int64_t)1 << vbits, kMaxTable);
  std::vector<uint64_t> uniq;
  int64_t ndiag = 0;
  {
    std::vector<uint64_t> bitsv;
    bitsv.reserve(1024);
    // collect distinct values incrementally (stop early when too many)
    std::vector<uint64_t> tmp;
    for (int64_t r = 0; r < n; ++r) {
      bool has_diag = false;
      for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
        if (col[k] == r) {
          has_diag = true;
          ++ndiag;
          continue;
        }
        uint64_t bv;
        std::memcpy(&bv, val + k, 8);
        tmp.push_back(bv);
        if (tmp.size() >= 4096) {
          tmp.insert(tmp.end(), uniq.begin(), uniq.end());
          std::sort(tmp.begin(), tmp.end());
          tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
          uniq.swap(tmp);
          tmp.clear();
          if ((int64_t)uniq.size() > maxvals) return false;
        }
      }
      if (!has_diag && rp[r + 1] > rp[r]) return false;   // an empty row packs as 0
    }
    tmp.insert(tmp.end(), uniq.begin(), uniq.end());
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    uniq.swap(tmp);
    if ((int64_t)uniq.size() > maxvals) return false;
  }
  table.resize(uniq.size());
  for (size_t i = 0; i < uniq.size(); ++i) std::memcpy(&table[i], &uniq[i], 8);
  // integer weights (every off-diagonal value is -k for an integer k >= 1,
  // e.g. unit graphs or C4's Geometric counts): a dense table -1, -2, ...,
  // -kmax (unused entries included) so the value of index i is -(i + 1) and
  // the SpMV computes it instead of looking it up (lg_csr.intw)
  {
    bool ints = !uniq.empty();
    int64_t kmax = 0;
    for (double v : table) {
      const double k = -v;
      if (!(k >= 1.0 && k <= 2048.0 && k == (double)(int64_t)k)) {
        ints = false;
        break;
      }
      kmax = std::max<int64_t>(kmax, (int64_t)k);
    }
    if (ints && kmax <= maxvals) {
      std::vector<double> dense((size_t)kmax);
      for (int64_t i = 0; i < kmax; ++i) dense[(size_t)i] = -(double)(i + 1);
      table.swap(dense);
      uniq.resize((size_t)kmax);
      for (int64_t i = 0; i < kmax; ++i) std::memcpy(&uniq[(size_t)i], &table[(size_t)i], 8);
    }
  }
  prp.assign((size_t)n + 1, 0);
  diag.assign((size_t)n, 0.0);
  const int64_t noff = rp[n] - ndiag;
  pcol.resize((size_t)std::max<int64_t>(noff, 0));
  int64_t o = 0;
  for (int64_t r = 0; r < n; ++r) {
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      if (col[k] == r) {
        diag[(size_t)r] = val[k];
        continue;
      }
      uint64_t bv;
      std::memcpy(&bv, val + k, 8);
      const uint32_t idx =
          (uint32_t)(std::lower_bound(uniq.begin(), uniq.end(), bv) - uniq.begin());
      pcol[(size_t)o++] = (uint32_t)col[k] | (idx << cbits);
    }
    prp[(size_t)r + 1] = o;
  }
  return true;
}

}  // namespace lg

using namespace lg;

extern "C" {

int lg_csr_create(int64_t n, int64_t nnz, const int64_t* rp, const int64_t* col,
                  const double* val, int flags, lg_csr** out) {
  if (!out) return fail(LG_EINVAL, "lg_csr_create: out is NULL");
  if (n < 0 || nnz < 0) return fail(LG_EINVAL, "lg_csr_create: negative size");
  if (n >= ((int64_t)1 << 31))
    return fail(LG_EINVAL, "lg_csr_create: n >= 2^31 not supported (int32 columns)");
  if (!rp || (nnz > 0 && (!col || !val)))
    return fail(LG_EINVAL, "lg_csr_create: NULL array");
  if (rp[0] != 0 || rp[n] != nnz)
    return fail(LG_EINVAL, "lg_csr_create: row_ptr must start at 0 and end at nnz");
  for (int64_t r = 0; r < n; ++r)
    if (rp[r + 1] < rp[r])
      return fail(LG_EINVAL, "lg_csr_create: row_ptr must be nondecreasing");
  std::vector<int32_t> c32((size_t)nnz);
  for (int64_t k = 0; k < nnz; ++k) {
    if (col[k] < 0 || col[k] >= n)
      return fail(LG_EINVAL, "lg_csr_create: column index out of range");
    c32[(size_t)k] = (int32_t)col[k];
  }
  std::vector<int64_t> prp;
  std::vector<uint32_t> pcol;
  std::vector<double> pdiag, table;
  int cbits = 0;
  const bool packed = !(flags & 1) && make_packed(n, rp, col, val, prp, pcol, pdiag, table, cbits);
  std::vector<char> absent;
  if (flags & LG_CSR_SKIP_EMPTY) {
    absent.resize((size_t)n);
    for (int64_t r = 0; r < n; ++r) absent[(size_t)r] = rp[r + 1] == rp[r];
  }
  lg_csr* a = new lg_csr();
  a->n = n;
  a->nnz = nnz;
  a->packed = packed ? 1 : 0;
  a->cbits = cbits;
  a->nvals = (int)table.size();
  a->intw = packed && !table.empty() ? 1 : 0;
  for (size_t i = 0; i < table.size() && a->intw; ++i) a->intw = table[i] == -(double)(i + 1);
  a->noff = packed ? (int64_t)pcol.size() : 0;
  a->is_block = (flags & LG_CSR_SKIP_EMPTY) ? 1 : 0;
  auto cleanup = [&](const char* what) {
    lg_csr_destroy(a);
    return fail(LG_ENOMEM, std::string("lg_csr_create: ") + what);
  };
  if (cudaMalloc(&a->row_ptr, sizeof(int64_t) * (size_t)(n + 1)) != cudaSuccess)
    return cleanup("row_ptr alloc");
  if (nnz && cudaMalloc(&a->col, sizeof(int32_t) * (size_t)(nnz + kStreamPad)) != cudaSuccess)
    return cleanup("col alloc");
  if (nnz && cudaMalloc(&a->val, sizeof(double) * (size_t)(nnz + kStreamPad)) != cudaSuccess)
    return cleanup("val alloc");
  if (packed) {
    if (cudaMalloc(&a->prp, sizeof(int64_t) * (size_t)(n + 1)) != cudaSuccess ||
        (a->noff && cudaMalloc(&a->pcol, sizeof(uint32_t) * (size_t)(a->noff + kStreamPad)) != cudaSuccess) ||
        cudaMalloc(&a->pdiag, sizeof(double) * (size_t)n) != cudaSuccess ||
        (a->nvals && cudaMalloc(&a->table, sizeof(double) * (size_t)a->nvals) != cudaSuccess))
      return cleanup("packed alloc");
    cudaMemcpy(a->prp, prp.data(), sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice);
    if (a->noff)
      cudaMemcpy(a->pcol, pcol.data(), sizeof(uint32_t) * (size_t)a->noff,
                 cudaMemcpyHostToDevice);
    cudaMemcpy(a->pdiag, pdiag.data(), sizeof(double) * (size_t)n, cudaMemcpyHostToDevice);
    if (a->nvals)
      cudaMemcpy(a->table, table.data(), sizeof(double) * (size_t)a->nvals,
                 cudaMemcpyHostToDevice);
  }
  cudaMemcpy(a->row_ptr, rp, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice);
  if (nnz) {
    cudaMemcpy(a->col, c32.data(), sizeof(int32_t) * (size_t)nnz, cudaMemcpyHostToDevice);
    cudaMemcpy(a->val, val, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice);
  }
  {
    const int rc = attach_schedule(a, packed ? prp.data() : rp,
                                   (flags & LG_CSR_SKIP_EMPTY) ? &absent : nullptr,
                                   "lg_csr_create");
    if (rc) {
      lg_csr_destroy(a);
      return rc;
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    lg_csr_destroy(a);
    return fail(LG_ECUDA, std::string("lg_csr_create: ") + cudaGetErrorString(e));
  }
  *out = a;
  return LG_OK;
}

int lg_csr_destroy(lg_csr* a) {
  if (!a) return LG_OK;
  for (int k = 0; k < a->npanels; ++k) lg_csr_destroy(a->panel[k]);
  cudaFree(a->row_ptr);
  cudaFree(a->col);
  cudaFree(a->val);
  cudaFree(a->blocks);
  cudaFree(a->long_nparts);
  cudaFree(a->long_first);
  cudaFree(a->long_row);
  cudaFree(a->prp);
  cudaFree(a->pcol);
  cudaFree(a->pdiag);
  cudaFree(a->table);
  cudaFree(a->rowmap);
  delete a;
  return LG_OK;
}

int lg_csr_info(const lg_csr* a, int64_t* n, int64_t* nnz, int64_t* nblocks,
                int64_t* nlong, int* packed, int64_t* stream_bytes) {
  if (!a) return fail(LG_EINVAL, "lg_csr_info: NULL handle");
  if (n) *n = a->n;
  if (nnz) *nnz = a->nnz;
  if (nblocks) *nblocks = a->nblocks;
  if (nlong) *nlong = a->nlong;
  if (packed) *packed = a->packed;
  // bytes one SpMV streams: plain = f64 values + int32 columns + schedule
  // descriptors (row structure) + x read + y written; packed = 32-bit words
  // per off-diagonal + descriptors + diagonal + x + y
  if (stream_bytes) {
    const int64_t sched = (int64_t)sizeof(SpmvBlock) * a->nblocks;
    *stream_bytes = a->packed ? 4 * a->noff + sched + 8 * a->n + 16 * a->n
                              : 12 * a->nnz + sched + 16 * a->n;
    if (a->npanels > 1) {
      // panelled product: the (d - theta) x init pass, then per panel its
      // words and schedule, its slice of x, y read-modify-write and the row
      // map of the rows it writes
      int64_t b = 24 * a->n;
      for (int k = 0; k < a->npanels; ++k) {
        const lg_csr* m = a->panel[k];
        b += 4 * m->noff + (int64_t)sizeof(SpmvBlock) * m->nblocks +
             8 * (m->pf_c1 - m->pf_c0) + m->nrows_sched * (16 + (m->rowmap ? 4 : 0));
      }
      *stream_bytes = b;
    }
  }
  return LG_OK;
}

int lg_csr_download(const lg_csr* a, int64_t* rp, int64_t* col, double* val) {
  if (!a) return fail(LG_EINVAL, "lg_csr_download: NULL handle");
  if (!a->row_ptr) return fail(LG_EINVAL, "lg_csr_download: device-only matrix");
  if (rp)
    LG_CUDA(cudaMemcpy(rp, a->row_ptr, sizeof(int64_t) * (size_t)(a->n + 1),
                       cudaMemcpyDeviceToHost));
  if (col && a->nnz) {
    std::vector<int32_t> c32((size_t)a->nnz);
    LG_CUDA(cudaMemcpy(c32.data(), a->col, sizeof(int32_t) * (size_t)a->nnz,
                       cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < a->nnz; ++k) col[k] = c32[(size_t)k];
  }
  if (val && a->nnz)
    LG_CUDA(cudaMemcpy(val, a->val, sizeof(double) * (size_t)a->nnz,
                       cudaMemcpyDeviceToHost));
  return LG_OK;
}

int lg_spmv_panels_(const lg_csr* a, const double* x, double* y, double theta_h,
                    const double* theta_d, int theta_neg, const int* skip, lg_ws* ws,
                    void* stream);

int lg_spmv(const lg_csr* a, const double* x, double* y, double theta_h,
            const double* theta_d, int theta_neg, int ndots,
            const double* const* dvec, const double* q, int64_t ldq, int nq,
            double* out, lg_ws* ws, const int* skip, void* stream) {
  if (!a || !x || !y) return fail(LG_EINVAL, "lg_spmv: NULL argument");
  if (ndots < 0 || ndots > LG_MAXD || nq < 0 || nq > LG_MAXQ)
    return fail(LG_EINVAL, "lg_spmv: too many epilogue dots");
  if ((ndots + nq) > 0 && (!out || !ws))
    return fail(LG_EINVAL, "lg_spmv: epilogue dots need out and ws");
  if (nq > 0 && (!q || ldq < a->n))
    return fail(LG_EINVAL, "lg_spmv: bad Q block");
  if (a->n == 0) return LG_OK;
  lg_ws local{};
  if (!ws) ws = &local;
  if (a->nlong) {
    if (ws == &local) return fail(LG_EINVAL, "lg_spmv: matrix has long rows; pass a workspace");
    int rc = ensure_long_ws(ws, a);
    if (rc) return rc;
  }
  SpmvArgs args = spmv_args(a, x, y, ws);
  args.theta_h = theta_h;
  args.theta_d = theta_d;
  args.theta_neg = theta_neg;
  args.skip = skip;
  cudaStream_t s = (cudaStream_t)stream;
  if (a->npanels > 1 && ws == &local)
    return fail(LG_EINVAL, "lg_spmv: panelled matrix; pass a workspace");
  if (a->npanels > 1 && !a->pdiag)
    return fail(LG_EINVAL, "lg_spmv: panelled diagonal-free row block; apply it with lg_spmv_acc");
  int rc = a->npanels > 1
               ? lg_spmv_panels_(a, x, y, theta_h, theta_d, theta_neg, skip, ws, stream)
               : launch(args, s, a->packed != 0);
  if (rc || ndots + nq == 0) return rc;
  // The dots / Q^T y epilogue runs as one streaming pass over y right behind
  // the product (the gather loop wants every register for occupancy).
  // Result layout: dots, then Q^T y.
  lg_fused_args f{};
  f.n = a->n;
  f.ndots = ndots;
  for (int d = 0; d < ndots; ++d) {
    f.da[d] = y;
    f.db[d] = (dvec && dvec[d]) ? dvec[d] : nullptr;
  }
  if (nq) {
    f.nblocks = 1;
    f.b[0].q = q;
    f.b[0].ld = ldq;
    f.b[0].k = nq;
    f.b[0].v = y;
  }
  f.result = out;
  f.skip = skip;
  return lg_fused(&f, ws, stream);
}

int lg_spmv_gather_probe(const lg_csr* a, const double* x, double* out, void* stream) {
  if (!a || !x || !out) return fail(LG_EINVAL, "lg_spmv_gather_probe: NULL argument");
  if (a->n == 0) return LG_OK;
  const uint32_t* words = a->packed ? a->pcol : reinterpret_cast<const uint32_t*>(a->col);
  const int64_t m = a->packed ? a->noff : a->nnz;
  const uint32_t cmask =
      a->packed ? (a->cbits >= 32 ? 0xffffffffu : ((1u << a->cbits) - 1u)) : 0xffffffffu;
  if (!words || m <= 0) return LG_OK;
  gather_probe_kernel<<<dev_info().sm_count * 8, 256, 0, (cudaStream_t)stream>>>(words, cmask, m,
                                                                                  x, out);
  LG_LAUNCH_CHECK("gather_probe_kernel");
  return LG_OK;
}

}  // extern "C"

namespace {
// Pinned staging of the host-buffer SpMV (one pair per thread, grown on
// demand).  A pageable cudaMemcpy goes through the driver's bounce buffers at
// about half the PCIe rate and the D2H lands in pages the caller may never
// have touched; instead the caller's x is copied by a few host threads into
// pinned memory, moved by DMA, and y comes back the same way.
struct HostStaging {
  double* xin = nullptr;
  double* yout = nullptr;
  int64_t cap = 0;
  ~HostStaging() {
    if (xin) cudaFreeHost(xin);
    if (yout) cudaFreeHost(yout);
  }
  bool ensure(int64_t n) {
    if (n <= cap) return true;
    if (xin) cudaFreeHost(xin);
    if (yout) cudaFreeHost(yout);
    xin = yout = nullptr;
    cap = 0;
    if (cudaHostAlloc(&xin, 8 * (size_t)n, cudaHostAllocPortable) != cudaSuccess ||
        cudaHostAlloc(&yout, 8 * (size_t)n, cudaHostAllocPortable) != cudaSuccess)
      return false;
    cap = n;
    return true;
  }
};
thread_local HostStaging g_stage;
// workspace of the host-buffer path (long-row partials); the call is
// synchronous, so one per thread suffices
struct HostWs {
  lg_ws* ws = nullptr;
  cudaStream_t d2h = nullptr;           // device -> host copies of y chunks
  cudaEvent_t done[kHostChunks] = {};   // chunk product finished
  cudaEvent_t copied[kHostChunks] = {}; // chunk copied to pinned memory
  bool ok = false;
  int device = -1;
  bool ready() {
    int dv = 0;
    if (cudaGetDevice(&dv) != cudaSuccess) return false;
    if (ok && dv == device) return true;
    if (ok) {   // the thread moved to another device: new stream and events
      cudaStreamDestroy(d2h);
      for (int c = 0; c < kHostChunks; ++c) {
        cudaEventDestroy(done[c]);
        cudaEventDestroy(copied[c]);
      }
      if (ws) lg_ws_destroy(ws);
      ws = nullptr;
      ok = false;
    }
    device = dv;
    if (cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) != cudaSuccess) return false;
    for (int c = 0; c < kHostChunks; ++c)
      if (cudaEventCreateWithFlags(&done[c], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&copied[c], cudaEventDisableTiming) != cudaSuccess)
        return false;
    ok = true;
    return true;
  }
  ~HostWs() {
    if (ws) lg_ws_destroy(ws);
  }
};
thread_local HostWs g_host_ws;

void par_copy(double* dst, const double* src, int64_t n) {
  // OpenMP's persistent pool: spawning threads per call would cost more than
  // the copy (8 MB per vector at C4)
  const int64_t kChunkD = 1 << 16;   // doubles per task
  const int64_t nc = (n + kChunkD - 1) / kChunkD;
#pragma omp parallel for schedule(static) num_threads(8) if (nc > 1)
  for (int64_t c = 0; c < nc; ++c) {
    const int64_t lo = c * kChunkD, hi = std::min(n, lo + kChunkD);
    std::memcpy(dst + lo, src + lo, 8 * (size_t)(hi - lo));
  }
}
// cudaHostAlloc'ed / cudaHostRegister'ed memory (DMA-able as it is)
bool host_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}
}  // namespace

extern "C" {

int lg_spmv_host(const lg_csr* a, const double* x_h, double* y_h, double* xd,
                 double* yd, void* stream) {
  if (!a || !x_h || !y_h || !xd || !yd) return fail(LG_EINVAL, "lg_spmv_host: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = a->n;
  if (n == 0) return LG_OK;
  if (!g_stage.ensure(n)) return fail(LG_ENOMEM, "lg_spmv_host: pinned staging");
  if (!g_host_ws.ready()) return fail(LG_ECUDA, "lg_spmv_host: stream / event setup");
  if (!g_host_ws.ws) {
    int rc0 = lg_ws_create(&g_host_ws.ws);
    if (rc0) return rc0;
  }
  if (a->nlong) {
    int rc0 = ensure_long_ws(g_host_ws.ws, a);
    if (rc0) return rc0;
  }
  static const bool pipe = [] {
    const char* e = getenv("LG_HOST_PIPE");   // 0: one copy, one product, one D2H
    return !(e && atoi(e) == 0);
  }();
  // Page-locked caller buffers are DMA'd directly (no staging copy).
  const bool xpin = host_pinned(x_h), ypin = host_pinned(y_h);
  // x: host copy of chunk c+1 overlaps the DMA of chunk c
  if (xpin) {
    LG_CUDA(cudaMemcpyAsync(xd, x_h, 8 * (size_t)n, cudaMemcpyHostToDevice, s));
  } else {
    const int kx = pipe ? 4 : 1;
    const int64_t cx = (n + kx - 1) / kx;
    for (int c = 0; c < kx; ++c) {
      const int64_t lo = c * cx, hi = std::min(n, lo + cx);
      if (lo >= hi) break;
      par_copy(g_stage.xin + lo, x_h + lo, hi - lo);
      LG_CUDA(cudaMemcpyAsync(xd + lo, g_stage.xin + lo, 8 * (size_t)(hi - lo),
                              cudaMemcpyHostToDevice, s));
    }
  }
  // y: the product runs in row chunks; each chunk's D2H (second stream)
  // overlaps the next chunk's product, and the host copy of chunk c overlaps
  // the DMA of chunk c+1
  double* ydst = ypin ? y_h : g_stage.yout;
  const bool chunked = pipe && a->nchunks > 1;
  const int nc = chunked ? a->nchunks : 1;
  for (int c = 0; c < nc; ++c) {
    const int64_t b0 = chunked ? a->chunk_b[c] : 0;
    const int64_t b1 = chunked ? a->chunk_b[c + 1] : a->nblocks;
    const int64_t r0 = chunked ? a->chunk_row[c] : 0;
    const int64_t r1 = chunked ? a->chunk_row[c + 1] : n;
    int rc = spmv_range(a, xd, yd, b0, b1, g_host_ws.ws, s);
    if (rc) return rc;
    LG_CUDA(cudaEventRecord(g_host_ws.done[c], s));
    LG_CUDA(cudaStreamWaitEvent(g_host_ws.d2h, g_host_ws.done[c], 0));
    if (r1 > r0)
      LG_CUDA(cudaMemcpyAsync(ydst + r0, yd + r0, 8 * (size_t)(r1 - r0),
                              cudaMemcpyDeviceToHost, g_host_ws.d2h));
    LG_CUDA(cudaEventRecord(g_host_ws.copied[c], g_host_ws.d2h));
  }
  for (int c = 0; c < nc; ++c) {
    const int64_t r0 = chunked ? a->chunk_row[c] : 0;
    const int64_t r1 = chunked ? a->chunk_row[c + 1] : n;
    if (ypin && c < nc - 1) continue;   // the last event covers every chunk
    LG_CUDA(cudaEventSynchronize(g_host_ws.copied[c]));
    if (!ypin && r1 > r0) par_copy(y_h + r0, g_stage.yout + r0, r1 - r0);
  }
  // the caller's stream is ordered after the copies (xd / yd reuse)
  LG_CUDA(cudaStreamWaitEvent(s, g_host_ws.copied[nc - 1], 0));
  return LG_OK;
}

int lg_spmm(const lg_csr* a, const double* x, double* y, int k, void* stream) {
  if (!a || !x || !y || k < 0) return fail(LG_EINVAL, "lg_spmm: bad argument");
  if (!g_host_ws.ready()) return fail(LG_ECUDA, "lg_spmm: setup");
  if (!g_host_ws.ws) {
    int rc0 = lg_ws_create(&g_host_ws.ws);
    if (rc0) return rc0;
  }
  for (int j = 0; j < k; ++j) {
    int rc = lg_spmv(a, x + (int64_t)j * a->n, y + (int64_t)j * a->n, 0.0,
                     nullptr, 0, 0, nullptr, nullptr, 0, 0, nullptr, g_host_ws.ws,
                     nullptr, stream);
    if (rc) return rc;
  }
  return LG_OK;
}

}  // extern "C"

// ---- row-major SpMM: Y = A X for k <= 16 vectors at once --------------------
// With X stored row-major (n x k), the k values a nonzero needs are one
// contiguous k * 8-byte run: one gather serves all k products, where k
// separate SpMVs make k random gathers (the L1TEX line rate bounds the
// SpMV, section 3 of DESIGN.md).  Lanes form G = 32 / K groups of K (K = k
// rounded up to a power of two), lane j of a group owning column j.  A row
// of at most kMmGroupRow nonzeros is one group's (G rows per warp in
// flight); a longer row of a block is the whole warp's, group g taking
// nonzeros g, g + G, ..., the groups summed by a butterfly.  A long-row part (>= one block) is split over the
// CTA's warps and its K partials go through the long-row part slots and
// ticket, summed in part order by the last part to finish (deterministic).
// Packed format only (lg_spmm falls back to k SpMVs otherwise).
namespace {
constexpr int kMmThreads = 256;
constexpr int kMmGroupRow = 48;   // rows up to this long: one K-lane group each

template <int K>
__global__ void __launch_bounds__(kMmThreads) spmm_rm_kernel(
    const int64_t* prp, const uint32_t* pcol, const double* pdiag, const double* table, int nvals,
    int cbits, const SpmvBlock* blocks, int64_t nblocks, const int32_t* long_nparts,
    const int64_t* long_first, const double* x, double* y, int k, double* part_sum,
    unsigned* ticket) {
  constexpr int G = 32 / K;
  constexpr int W = kMmThreads / 32;
  __shared__ double tab[kMaxTable];
  __shared__ double red[W][K];
  extern __shared__ uint32_t scol[];   // one block's column words (kWin)
  __shared__ int fin;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / K, j = lane % K;
  const uint32_t cmask = (1u << cbits) - 1u;
  for (int i = threadIdx.x; i < nvals; i += kMmThreads) tab[i] = table[i];
  __syncthreads();
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
    const SpmvBlock blk = blocks[b];
    if (blk.lshift >= 0) {
      // the block's column words, coalesced into shared memory once; the
      // gathers below then depend on nothing but shared memory
      const int cnt = (int)(blk.nz1 - blk.nz0);
      for (int e = threadIdx.x; e < cnt; e += kMmThreads) scol[e] = pcol[blk.nz0 + e];
      __syncthreads();
      // short rows: one group of K lanes per row, W * G rows in flight per
      // CTA, the row's nonzeros walked four at a time
      for (int rr = warp * G + g; rr < blk.nrows; rr += W * G) {
        const int64_t r = blk.row0 + rr;
        const int e1 = (int)(prp[r + 1] - blk.nz0);
        int e = (int)(prp[r] - blk.nz0);
        if (e1 - e > kMmGroupRow) continue;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (j < k) {
          for (; e + 3 < e1; e += 4) {
            const uint32_t w0 = scol[e], w1 = scol[e + 1], w2 = scol[e + 2], w3 = scol[e + 3];
            a0 += tab[w0 >> cbits] * x[(int64_t)(w0 & cmask) * k + j];
            a1 += tab[w1 >> cbits] * x[(int64_t)(w1 & cmask) * k + j];
            a2 += tab[w2 >> cbits] * x[(int64_t)(w2 & cmask) * k + j];
            a3 += tab[w3 >> cbits] * x[(int64_t)(w3 & cmask) * k + j];
          }
          for (; e < e1; ++e) {
            const uint32_t w0 = scol[e];
            a0 += tab[w0 >> cbits] * x[(int64_t)(w0 & cmask) * k + j];
          }
          y[r * k + j] = ((a0 + a1) + (a2 + a3)) + pdiag[r] * x[r * k + j];
        }
      }
      // longer rows of the block: the whole warp, groups summed by butterfly
      for (int rr = warp; rr < blk.nrows; rr += W) {
        const int64_t r = blk.row0 + rr;
        const int e0 = (int)(prp[r] - blk.nz0), e1 = (int)(prp[r + 1] - blk.nz0);
        if (e1 - e0 <= kMmGroupRow) continue;
        double acc = 0.0;
        for (int e = e0 + g; e < e1; e += G) {
          const uint32_t w = scol[e];
          if (j < k) acc += tab[w >> cbits] * x[(int64_t)(w & cmask) * k + j];
        }
#pragma unroll
        for (int o = K; o < 32; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (g == 0 && j < k) y[r * k + j] = acc + pdiag[r] * x[r * k + j];
      }
      __syncthreads();   // scol reused by the next block
    } else {
      // part of a long row: the CTA's warps split the part, K partials
      const int cnt = (int)(blk.nz1 - blk.nz0);
      for (int e = threadIdx.x; e < cnt; e += kMmThreads) scol[e] = pcol[blk.nz0 + e];
      __syncthreads();
      double acc = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      if (j < k) {
        constexpr int S = W * G;
        int e = warp * G + g;
        for (; e + 3 * S < cnt; e += 4 * S) {
          const uint32_t w0 = scol[e], w1 = scol[e + S], w2 = scol[e + 2 * S],
                         w3 = scol[e + 3 * S];
          acc += tab[w0 >> cbits] * x[(int64_t)(w0 & cmask) * k + j];
          a1 += tab[w1 >> cbits] * x[(int64_t)(w1 & cmask) * k + j];
          a2 += tab[w2 >> cbits] * x[(int64_t)(w2 & cmask) * k + j];
          a3 += tab[w3 >> cbits] * x[(int64_t)(w3 & cmask) * k + j];
        }
        for (; e < cnt; e += S) {
          const uint32_t w0 = scol[e];
          acc += tab[w0 >> cbits] * x[(int64_t)(w0 & cmask) * k + j];
        }
        acc = (acc + a1) + (a2 + a3);
      }
#pragma unroll
      for (int o = K; o < 32; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (g == 0) red[warp][j] = acc;
      __syncthreads();
      if (threadIdx.x < K) {
        double t = 0.0;
        for (int w2 = 0; w2 < W; ++w2) t += red[w2][threadIdx.x];
        part_sum[(int64_t)blk.part * K + threadIdx.x] = t;
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned arrived = atomicAdd(ticket + blk.nrows, 1u);
        fin = arrived == (unsigned)long_nparts[blk.nrows] - 1u;
      }
      __syncthreads();
      if (fin && threadIdx.x < K) {
        __threadfence();
        const int lr = blk.nrows;
        const int64_t first = long_first[lr];
        const int np = long_nparts[lr];
        double t = 0.0;
        for (int p = 0; p < np; ++p) t += ld_cg(part_sum + (first + p) * K + threadIdx.x);
        const int64_t r = blk.row0;
        if ((int)threadIdx.x < k) y[r * k + threadIdx.x] = t + pdiag[r] * x[r * k + threadIdx.x];
        if (threadIdx.x == 0) ticket[lr] = 0u;
      }
      __syncthreads();
    }
  }
}
}  // namespace

extern "C" {

int lg_spmm_rowmajor(const lg_csr* a, const double* x, double* y, int k, lg_ws* ws,
                     void* stream) {
  if (!a || !x || !y || k < 1 || k > 16 || !ws)
    return fail(LG_EINVAL, "lg_spmm_rowmajor: bad argument (1 <= k <= 16, workspace)");
  if (!a->packed || !a->pdiag)
    return fail(LG_EINVAL, "lg_spmm_rowmajor: needs the packed format with its diagonal");
  if (a->n == 0 || a->nblocks == 0) return LG_OK;
  const int K = k <= 2 ? 2 : k <= 4 ? 4 : k <= 8 ? 8 : 16;
  if (a->nlong) {
    int rc = ensure_long_ws(ws, a);
    if (rc) return rc;
    if (ws->mm_cap < a->nparts * K) {
      cudaFree(ws->mm_part);
      ws->mm_part = nullptr;
      ws->mm_cap = 0;
      LG_CUDA(cudaMalloc(&ws->mm_part, 8 * (size_t)(a->nparts * K)));
      ws->mm_cap = a->nparts * K;
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = sizeof(uint32_t) * (size_t)kWin;
  static thread_local int occ = 0;
  if (!occ) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmm_rm_kernel<16>, kMmThreads,
                                                      sizeof(uint32_t) * kWin) !=
            cudaSuccess || occ < 1)
      occ = 1;
  }
  const unsigned g = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>(a->nblocks, (int64_t)occ * dev_info().sm_count));
#define LG_MM(KK)                                                                               \
  spmm_rm_kernel<KK><<<g, kMmThreads, smem, s>>>(a->prp, a->pcol, a->pdiag, a->table, a->nvals,  \
                                              a->cbits, a->blocks, a->nblocks,                 \
                                              a->long_nparts, a->long_first, x, y, k,          \
                                              ws->mm_part, ws->long_ticket)
  if (K == 2) LG_MM(2);
  else if (K == 4) LG_MM(4);
  else if (K == 8) LG_MM(8);
  else LG_MM(16);
#undef LG_MM
  LG_LAUNCH_CHECK("spmm_rm_kernel");
  return LG_OK;
}

// ---- device-built unit-weight Laplacian (C5 scale) -------------------------
namespace {

__global__ void dl_count(int64_t m, const int32_t* ei, const int32_t* ej, int32_t* up,
                         int32_t* lo) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    atomicAdd(up + ei[e], 1);
    atomicAdd(lo + ej[e], 1);
  }
}

__global__ void dl_len(int64_t n, const int32_t* up, const int32_t* lo, int64_t* len,
                       int64_t* up64, double* diag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    len[v] = (int64_t)up[v] + lo[v];
    up64[v] = up[v];
    diag[v] = (double)((int64_t)up[v] + lo[v]);   // unit weights: exact
  }
}

// row v: lower neighbours (ascending) then upper neighbours (ascending)
__global__ void dl_scatter_upper(int64_t m, const int32_t* ei, const int32_t* ej,
                                 const int64_t* rp, const int32_t* lo, const int64_t* ustart,
                                 uint32_t* pcol) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    const int32_t v = ei[e];
    pcol[rp[v] + lo[v] + (e - ustart[v])] = (uint32_t)ej[e];
  }
}

__global__ void dl_lower_pos(int64_t m, const int32_t* sj, const int64_t* lstart,
                             const int64_t* rp, const int32_t* si, uint32_t* pcol) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
    const int32_t v = sj[p];
    pcol[rp[v] + (p - lstart[v])] = (uint32_t)si[p];
  }
}

inline int gridm(int64_t n) {
  int64_t g = (n + kST - 1) / kST;
  int64_t cap = (int64_t)dev_info().sm_count * 32;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

}  // namespace

extern "C" int lg_csr_laplacian_device(int64_t n, int64_t m, const int32_t* d_i,
                                       const int32_t* d_j, lg_csr** out) {
  if (!out || n < 1 || m < 0 || (m > 0 && (!d_i || !d_j)))
    return fail(LG_EINVAL, "lg_csr_laplacian_device: bad argument");
  if (n >= ((int64_t)1 << 31)) return fail(LG_EINVAL, "lg_csr_laplacian_device: n too large");
  int cbits = 1;
  while (((int64_t)1 << cbits) < n) ++cbits;
  if (cbits > 31) return fail(LG_EINVAL, "lg_csr_laplacian_device: n too large for packing");
  lg_csr* a = new lg_csr();
  a->n = n;
  a->nnz = n + 2 * m;
  a->packed = 1;
  a->cbits = cbits;
  a->nvals = 1;
  a->intw = 1;   // table = {-1}
  a->noff = 2 * m;
  int32_t *up = nullptr, *lo = nullptr, *sj = nullptr, *si = nullptr;
  int64_t *len = nullptr, *up64 = nullptr, *lo64 = nullptr, *ustart = nullptr,
          *lstart = nullptr;
  void* tmp = nullptr;
  auto cleanup = [&]() {
    cudaFree(up);
    cudaFree(lo);
    cudaFree(sj);
    cudaFree(si);
    cudaFree(len);
    cudaFree(up64);
    cudaFree(lo64);
    cudaFree(ustart);
    cudaFree(lstart);
    cudaFree(tmp);
  };
  bool ok = cudaMalloc(&up, 4 * (size_t)n) == cudaSuccess &&
            cudaMalloc(&lo, 4 * (size_t)n) == cudaSuccess &&
            cudaMalloc(&len, 8 * (size_t)n) == cudaSuccess &&
            cudaMalloc(&up64, 8 * (size_t)n) == cudaSuccess &&
            cudaMalloc(&lo64, 8 * (size_t)n) == cudaSuccess &&
            cudaMalloc(&ustart, 8 * (size_t)n) == cudaSuccess &&
            cudaMalloc(&lstart, 8 * (size_t)n) == cudaSuccess &&
            cudaMalloc(&a->prp, 8 * (size_t)(n + 1)) == cudaSuccess &&
            cudaMalloc(&a->pdiag, 8 * (size_t)n) == cudaSuccess &&
            cudaMalloc(&a->table, 8) == cudaSuccess &&
            cudaMalloc(&a->pcol, 4 * (size_t)(2 * m + kStreamPad)) == cudaSuccess &&
            (m == 0 || (cudaMalloc(&sj, 4 * (size_t)m) == cudaSuccess &&
                        cudaMalloc(&si, 4 * (size_t)m) == cudaSuccess));
  if (!ok) {
    cleanup();
    lg_csr_destroy(a);
    return fail(LG_ENOMEM, "lg_csr_laplacian_device: allocation failed");
  }
  const double minus_one = -1.0;
  cudaMemcpy(a->table, &minus_one, 8, cudaMemcpyHostToDevice);
  cudaMemset(up, 0, 4 * (size_t)n);
  cudaMemset(lo, 0, 4 * (size_t)n);
  if (m) dl_count<<<gridm(m), kST>>>(m, d_i, d_j, up, lo);
  // lo64 = lo counts as int64 for the lower-run starts
  dl_len<<<gridm(n), kST>>>(n, up, lo, len, up64, a->pdiag);
  size_t tb = 0, t2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, len, a->prp + 1, (int64_t)n);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, up64, ustart, (int64_t)n);
  tb = std::max(tb, t2);
  if (m) {
    cub::DeviceRadixSort::SortPairs(nullptr, t2, d_j, sj, d_i, si, (int64_t)m, 0, cbits);
    tb = std::max(tb, t2);
  }
  if (cudaMalloc(&tmp, tb) != cudaSuccess) {
    cleanup();
    lg_csr_destroy(a);
    return fail(LG_ENOMEM, "lg_csr_laplacian_device: temp alloc");
  }
  cudaMemset(a->prp, 0, 8);
  cub::DeviceScan::InclusiveSum(tmp, tb, len, a->prp + 1, (int64_t)n);
  cub::DeviceScan::ExclusiveSum(tmp, tb, up64, ustart, (int64_t)n);
  if (m) {
    // stable radix sort by j keeps ascending i inside every key run
    cub::DeviceRadixSort::SortPairs(tmp, tb, d_j, sj, d_i, si, (int64_t)m, 0, cbits);
    // lower-run starts: exclusive scan of the lower counts
    dl_len<<<gridm(n), kST>>>(n, lo, up, len, lo64, a->pdiag);  // lo64 = lo
    cub::DeviceScan::ExclusiveSum(tmp, tb, lo64, lstart, (int64_t)n);
    dl_lower_pos<<<gridm(m), kST>>>(m, sj, lstart, a->prp, si, a->pcol);
    dl_scatter_upper<<<gridm(m), kST>>>(m, d_i, d_j, a->prp, lo, ustart, a->pcol);
  }
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    cleanup();
    lg_csr_destroy(a);
    return fail(LG_ECUDA, std::string("lg_csr_laplacian_device: ") + cudaGetErrorString(err));
  }
  cleanup();
  // row-block schedule from the off-diagonal row pointers (host, O(n))
  {
    std::vector<int64_t> prp((size_t)n + 1);
    cudaMemcpy(prp.data(), a->prp, 8 * (size_t)(n + 1), cudaMemcpyDeviceToHost);
    const int rc = attach_schedule(a, prp.data(), nullptr, "lg_csr_laplacian_device");
    if (rc) {
      lg_csr_destroy(a);
      return rc;
    }
  }
  // the plain arrays are not materialised (device-only matrix)
  *out = a;
  return LG_OK;
}

// Rows [r0, r1) of a plain-format matrix (e.g. a device-built FSAI factor)
// as an n x n plain matrix whose other rows are absent from the schedule.
static int plain_row_block(const lg_csr* a, int64_t r0, int64_t r1, lg_csr** out) {
  if (!a->row_ptr) return fail(LG_EINVAL, "lg_csr_row_block: matrix has no plain arrays");
  const int64_t n = a->n, nloc = r1 - r0;
  std::vector<int64_t> lrp((size_t)nloc + 1);
  LG_CUDA(cudaMemcpy(lrp.data(), a->row_ptr + r0, 8 * (size_t)(nloc + 1),
                     cudaMemcpyDeviceToHost));
  const int64_t off0 = lrp[0], m = lrp[(size_t)nloc] - off0;
  std::vector<int64_t> rp((size_t)n + 1, 0);
  for (int64_t i = 0; i < nloc; ++i) rp[(size_t)(r0 + i + 1)] = lrp[(size_t)i + 1] - off0;
  for (int64_t r = r1 + 1; r <= n; ++r) rp[(size_t)r] = m;
  std::vector<char> absent((size_t)n, 1);
  for (int64_t r = r0; r < r1; ++r) absent[(size_t)r] = 0;
  lg_csr* b = new lg_csr();
  b->n = n;
  b->nnz = m;
  b->is_block = 1;
  bool ok = cudaMalloc(&b->row_ptr, 8 * (size_t)(n + 1)) == cudaSuccess &&
            cudaMalloc(&b->col, 4 * (size_t)(m + kStreamPad)) == cudaSuccess &&
            cudaMalloc(&b->val, 8 * (size_t)(m + kStreamPad)) == cudaSuccess;
  if (!ok) {
    lg_csr_destroy(b);
    return fail(LG_ENOMEM, "lg_csr_row_block: allocation failed");
  }
  cudaMemcpy(b->row_ptr, rp.data(), 8 * (size_t)(n + 1), cudaMemcpyHostToDevice);
  if (m) {
    cudaMemcpy(b->col, a->col + off0, 4 * (size_t)m, cudaMemcpyDeviceToDevice);
    cudaMemcpy(b->val, a->val + off0, 8 * (size_t)m, cudaMemcpyDeviceToDevice);
  }
  int rc = attach_schedule(b, rp.data(), &absent, "lg_csr_row_block");
  cudaError_t err = cudaDeviceSynchronize();
  if (rc || err != cudaSuccess) {
    lg_csr_destroy(b);
    return rc ? rc : fail(LG_ECUDA, std::string("lg_csr_row_block: ") + cudaGetErrorString(err));
  }
  *out = b;
  return LG_OK;
}

// ---- one rank's row block (multi-GPU) --------------------------------------
// Rows [r0, r1) of a packed matrix as a packed n x n matrix whose other rows
// are absent from the schedule (lg_spmv leaves y there untouched): the
// operator one rank applies to the fully exchanged x in the row-partitioned
// SpMV.  Columns keep the global numbering, so every rank's slice of an
// n-vector is exchanged in place (no packing, no padding).
extern "C" int lg_csr_row_block(const lg_csr* a, int64_t r0, int64_t r1, lg_csr** out) {
  if (!a || !out || r0 < 0 || r1 < r0 || r1 > a->n)
    return fail(LG_EINVAL, "lg_csr_row_block: bad argument");
  if (!a->packed) return plain_row_block(a, r0, r1, out);
  const int64_t n = a->n, nloc = r1 - r0;
  std::vector<int64_t> lrp((size_t)nloc + 1);
  LG_CUDA(cudaMemcpy(lrp.data(), a->prp + r0, 8 * (size_t)(nloc + 1), cudaMemcpyDeviceToHost));
  const int64_t off0 = lrp[0], m = lrp[(size_t)nloc] - off0;
  std::vector<int64_t> prp((size_t)n + 1, 0);
  for (int64_t i = 0; i < nloc; ++i) prp[(size_t)(r0 + i + 1)] = lrp[(size_t)i + 1] - off0;
  for (int64_t r = r1 + 1; r <= n; ++r) prp[(size_t)r] = m;
  std::vector<char> absent((size_t)n, 1);
  for (int64_t r = r0; r < r1; ++r) absent[(size_t)r] = 0;
  lg_csr* b = new lg_csr();
  b->is_block = 1;
  b->n = n;
  b->nnz = m + nloc;
  b->packed = 1;
  b->cbits = a->cbits;
  b->nvals = a->nvals;
  b->intw = a->intw;
  b->noff = m;
  bool ok = cudaMalloc(&b->prp, 8 * (size_t)(n + 1)) == cudaSuccess &&
            (m == 0 || cudaMalloc(&b->pcol, 4 * (size_t)(m + kStreamPad)) == cudaSuccess) &&
            cudaMalloc(&b->pdiag, 8 * (size_t)n) == cudaSuccess &&
            (b->nvals == 0 || cudaMalloc(&b->table, 8 * (size_t)b->nvals) == cudaSuccess);
  if (!ok) {
    lg_csr_destroy(b);
    return fail(LG_ENOMEM, "lg_csr_row_block: allocation failed");
  }
  cudaMemcpy(b->prp, prp.data(), 8 * (size_t)(n + 1), cudaMemcpyHostToDevice);
  cudaMemset(b->pdiag, 0, 8 * (size_t)n);
  cudaMemcpy(b->pdiag + r0, a->pdiag + r0, 8 * (size_t)nloc, cudaMemcpyDeviceToDevice);
  if (b->nvals) cudaMemcpy(b->table, a->table, 8 * (size_t)b->nvals, cudaMemcpyDeviceToDevice);
  if (m) cudaMemcpy(b->pcol, a->pcol + off0, 4 * (size_t)m, cudaMemcpyDeviceToDevice);
  int rc = attach_schedule(b, prp.data(), &absent, "lg_csr_row_block");
  cudaError_t err = cudaDeviceSynchronize();
  if (rc || err != cudaSuccess) {
    lg_csr_destroy(b);
    return rc ? rc : fail(LG_ECUDA, std::string("lg_csr_row_block: ") + cudaGetErrorString(err));
  }
  *out = b;
  return LG_OK;
}

}  // extern "C"

// ---- interior / exterior split of a row block (overlapped exchange) -------
// Rank r's row block [r0, r1) splits by column into the interior part
// (columns in [r0, r1), with the diagonal: only the rank's own slice of x)
// and the exterior part (every other column, no diagonal).  The interior
// product runs while the slices of x are exchanged; the exterior product
// then accumulates into y (lg_spmv_acc).  Both stay in the packed format.
namespace {
__global__ void split_count(int64_t r0, int64_t r1, int64_t c0, int64_t c1, const int64_t* prp,
                            const uint32_t* pcol, uint32_t cmask, int64_t* cin, int64_t* cout) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1; r += st) {
    int64_t ni = 0;
    for (int64_t k = prp[r]; k < prp[r + 1]; ++k) {
      const int64_t c = pcol[k] & cmask;
      ni += (c >= c0 && c < c1);
    }
    cin[r - r0] = ni;
    if (cout) cout[r - r0] = (prp[r + 1] - prp[r]) - ni;
  }
}
__global__ void split_scatter(int64_t r0, int64_t r1, int64_t c0, int64_t c1, const int64_t* prp,
                              const uint32_t* pcol, uint32_t cmask, const int64_t* oin,
                              const int64_t* oout, uint32_t* win, uint32_t* wout) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1; r += st) {
    int64_t pi = oin[r - r0], po = wout ? oout[r - r0] : 0;
    for (int64_t k = prp[r]; k < prp[r + 1]; ++k) {
      const uint32_t w = pcol[k];
      const int64_t c = w & cmask;
      if (c >= c0 && c < c1) win[pi++] = w;
      else if (wout) wout[po++] = w;
    }
  }
}
}  // namespace

// one packed n x n operator holding rows [r0, r1) with the given per-row
// counts (host) and words (device, already placed)
static int make_part(const lg_csr* a, int64_t r0, int64_t r1, const std::vector<int64_t>& cnt,
                     uint32_t* words, int64_t m, bool with_diag, lg_csr** out) {
  const int64_t n = a->n, nloc = r1 - r0;
  std::vector<int64_t> prp((size_t)n + 1, 0);
  for (int64_t i = 0; i < nloc; ++i) prp[(size_t)(r0 + i + 1)] = prp[(size_t)(r0 + i)] + cnt[(size_t)i];
  for (int64_t r = r1 + 1; r <= n; ++r) prp[(size_t)r] = prp[(size_t)r1];
  std::vector<char> absent((size_t)n, 1);
  for (int64_t r = r0; r < r1; ++r) absent[(size_t)r] = 0;
  lg_csr* b = new lg_csr();
  b->n = n;
  b->nnz = m + (with_diag ? nloc : 0);
  b->packed = 1;
  b->cbits = a->cbits;
  b->nvals = a->nvals;
  b->intw = a->intw;
  b->noff = m;
  b->is_block = (r0 > 0 || r1 < n) ? 1 : 0;
  bool ok = cudaMalloc(&b->prp, 8 * (size_t)(n + 1)) == cudaSuccess &&
            (!with_diag || cudaMalloc(&b->pdiag, 8 * (size_t)n) == cudaSuccess) &&
            (b->nvals == 0 || cudaMalloc(&b->table, 8 * (size_t)b->nvals) == cudaSuccess);
  if (!ok) {
    lg_csr_destroy(b);  // words stay the caller's on failure
    return fail(LG_ENOMEM, "lg_csr_split_cols: allocation failed");
  }
  cudaMemcpy(b->prp, prp.data(), 8 * (size_t)(n + 1), cudaMemcpyHostToDevice);
  if (with_diag) {  // parts without the diagonal keep pdiag NULL (nothing to stream)
    cudaMemset(b->pdiag, 0, 8 * (size_t)n);
    cudaMemcpy(b->pdiag + r0, a->pdiag + r0, 8 * (size_t)nloc, cudaMemcpyDeviceToDevice);
  }
  if (b->nvals) cudaMemcpy(b->table, a->table, 8 * (size_t)b->nvals, cudaMemcpyDeviceToDevice);
  // an accumulating part (no diagonal) leaves its rows without entries alone
  if (!with_diag)
    for (int64_t r = r0; r < r1; ++r) absent[(size_t)r] = prp[(size_t)r + 1] == prp[(size_t)r];
  const int rc = attach_schedule(b, prp.data(), &absent, "lg_csr_split_cols");
  if (rc) {
    lg_csr_destroy(b);  // words stay the caller's on failure
    return rc;
  }
  b->pcol = words;    // owned by the part from here on
  *out = b;
  return LG_OK;
}

extern "C" int lg_csr_split_cols(const lg_csr* a, int64_t r0, int64_t r1, lg_csr** inner,
                                 lg_csr** outer) {
  if (!a || !inner || !outer || r0 < 0 || r1 < r0 || r1 > a->n)
    return fail(LG_EINVAL, "lg_csr_split_cols: bad argument");
  if (!a->packed) return fail(LG_EINVAL, "lg_csr_split_cols: only for packed matrices");
  const int64_t nloc = r1 - r0;
  const uint32_t cmask = (a->cbits >= 32) ? 0xffffffffu : ((1u << a->cbits) - 1u);
  int64_t *cin = nullptr, *cout = nullptr, *oin = nullptr, *oout = nullptr;
  void* tmp = nullptr;
  uint32_t *win = nullptr, *wout = nullptr;
  auto cleanup = [&]() {
    cudaFree(cin);
    cudaFree(cout);
    cudaFree(oin);
    cudaFree(oout);
    cudaFree(tmp);
  };
  const size_t nb = 8 * (size_t)std::max<int64_t>(nloc, 1);
  if (cudaMalloc(&cin, nb) != cudaSuccess || cudaMalloc(&cout, nb) != cudaSuccess ||
      cudaMalloc(&oin, nb) != cudaSuccess || cudaMalloc(&oout, nb) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_csr_split_cols: allocation failed");
  }
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((nloc + 255) / 256,
                                                             (int64_t)dev_info().sm_count * 16));
  if (nloc) split_count<<<g, 256>>>(r0, r1, r0, r1, a->prp, a->pcol, cmask, cin, cout);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cin, oin, std::max<int64_t>(nloc, 1));
  if (cudaMalloc(&tmp, std::max<size_t>(tb, 16)) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_csr_split_cols: scan scratch");
  }
  std::vector<int64_t> hin((size_t)nloc), hout((size_t)nloc);
  int64_t mi = 0, mo = 0;
  if (nloc) {
    cub::DeviceScan::ExclusiveSum(tmp, tb, cin, oin, nloc);
    cub::DeviceScan::ExclusiveSum(tmp, tb, cout, oout, nloc);
    cudaMemcpy(hin.data(), cin, 8 * (size_t)nloc, cudaMemcpyDeviceToHost);
    cudaMemcpy(hout.data(), cout, 8 * (size_t)nloc, cudaMemcpyDeviceToHost);
    for (int64_t i = 0; i < nloc; ++i) {
      mi += hin[(size_t)i];
      mo += hout[(size_t)i];
    }
  }
  if (cudaMalloc(&win, 4 * (size_t)(mi + kStreamPad)) != cudaSuccess ||
      cudaMalloc(&wout, 4 * (size_t)(mo + kStreamPad)) != cudaSuccess) {
    cudaFree(win);
    cleanup();
    return fail(LG_ENOMEM, "lg_csr_split_cols: allocation failed");
  }
  if (nloc) split_scatter<<<g, 256>>>(r0, r1, r0, r1, a->prp, a->pcol, cmask, oin, oout, win, wout);
  cudaError_t e = cudaDeviceSynchronize();
  cleanup();
  if (e != cudaSuccess) {
    cudaFree(win);
    cudaFree(wout);
    return fail(LG_ECUDA, std::string("lg_csr_split_cols: ") + cudaGetErrorString(e));
  }
  lg_csr *bi = nullptr, *bo = nullptr;
  int rc = make_part(a, r0, r1, hin, win, mi, true, &bi);
  if (rc) {
    cudaFree(win);
    cudaFree(wout);
    return rc;
  }
  rc = make_part(a, r0, r1, hout, wout, mo, false, &bo);
  if (rc) {
    lg_csr_destroy(bi);
    cudaFree(wout);
    return rc;
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    lg_csr_destroy(bi);
    lg_csr_destroy(bo);
    return fail(LG_ECUDA, std::string("lg_csr_split_cols: ") + cudaGetErrorString(e));
  }
  *inner = bi;
  *outer = bo;
  return LG_OK;
}

// Column panel [c0, c1) of the whole operator (every row, only the columns in
// the range; the diagonal when with_diag).  A product split into panels whose
// slice of x fits in L2 gathers x from L2 instead of DRAM: y = P_0 x, then
// y += P_k x (lg_spmv_acc) — for graphs whose x exceeds L2 (C5).
extern "C" int lg_csr_col_panel(const lg_csr* a, int64_t c0, int64_t c1, int with_diag,
                                lg_csr** out) {
  if (!a || !out || c0 < 0 || c1 < c0 || c1 > a->n)
    return fail(LG_EINVAL, "lg_csr_col_panel: bad argument");
  if (!a->packed) return fail(LG_EINVAL, "lg_csr_col_panel: only for packed matrices");
  const int64_t n = a->n;
  const uint32_t cmask = (a->cbits >= 32) ? 0xffffffffu : ((1u << a->cbits) - 1u);
  int64_t *cin = nullptr, *oin = nullptr;
  void* tmp = nullptr;
  uint32_t* win = nullptr;
  auto cleanup = [&]() {
    cudaFree(cin);
    cudaFree(oin);
    cudaFree(tmp);
  };
  const size_t nb = 8 * (size_t)std::max<int64_t>(n, 1);
  if (cudaMalloc(&cin, nb) != cudaSuccess || cudaMalloc(&oin, nb) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_csr_col_panel: allocation failed");
  }
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256,
                                                             (int64_t)dev_info().sm_count * 16));
  if (n) split_count<<<g, 256>>>(0, n, c0, c1, a->prp, a->pcol, cmask, cin, nullptr);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cin, oin, std::max<int64_t>(n, 1));
  if (cudaMalloc(&tmp, std::max<size_t>(tb, 16)) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_csr_col_panel: scan scratch");
  }
  std::vector<int64_t> hin((size_t)n);
  int64_t mi = 0;
  if (n) {
    cub::DeviceScan::ExclusiveSum(tmp, tb, cin, oin, n);
    cudaMemcpy(hin.data(), cin, nb, cudaMemcpyDeviceToHost);
    for (int64_t i = 0; i < n; ++i) mi += hin[(size_t)i];
  }
  if (cudaMalloc(&win, 4 * (size_t)(mi + kStreamPad)) != cudaSuccess) {
    cleanup();
    return fail(LG_ENOMEM, "lg_csr_col_panel: allocation failed");
  }
  if (n) split_scatter<<<g, 256>>>(0, n, c0, c1, a->prp, a->pcol, cmask, oin, nullptr, win, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  cleanup();
  if (e != cudaSuccess) {
    cudaFree(win);
    return fail(LG_ECUDA, std::string("lg_csr_col_panel: ") + cudaGetErrorString(e));
  }
  int rc = make_part(a, 0, n, hin, win, mi, with_diag != 0, out);
  if (rc) {
    cudaFree(win);
    return rc;
  }
  (*out)->pf_c0 = c0;
  (*out)->pf_c1 = c1;
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    lg_csr_destroy(*out);
    *out = nullptr;
    return fail(LG_ECUDA, std::string("lg_csr_col_panel: ") + cudaGetErrorString(e));
  }
  return LG_OK;
}

// Attach p equal-width column panels to a FULL operator (every row present;
// not a row block): lg_spmv then runs the panel chain.  p <= 1 detaches.
extern "C" int lg_csr_set_panels(lg_csr* a, int p) {
  if (!a || p < 0 || p > 16) return fail(LG_EINVAL, "lg_csr_set_panels: bad argument");
  if (p > 1 && !a->packed) return fail(LG_EINVAL, "lg_csr_set_panels: only for packed matrices");
  // a row block may be panelled only as an accumulating operator without a
  // diagonal (the exterior half of a split row block, applied by
  // lg_spmv_acc): its panels then hold only the block's rows; a full operator
  // gets the (d - theta) x init pass in lg_spmv
  if (p > 1 && a->is_block && a->pdiag)
    return fail(LG_EINVAL, "lg_csr_set_panels: only for full operators or the diagonal-free "
                           "exterior half of a row block (this one has absent rows)");
  cudaDeviceSynchronize();
  for (int k = 0; k < a->npanels; ++k) lg_csr_destroy(a->panel[k]);
  a->npanels = 0;
  if (p <= 1) return LG_OK;
  lg_csr* parts[16] = {};
  for (int k = 0; k < p; ++k) {
    int rc = lg_csr_col_panel(a, a->n * k / p, a->n * (k + 1) / p, 0, &parts[k]);
    if (rc) {
      for (int j = 0; j < k; ++j) lg_csr_destroy(parts[j]);
      return rc;
    }
  }
  for (int k = 0; k < p; ++k) a->panel[k] = parts[k];
  a->npanels = p;
  return LG_OK;
}

namespace {
// y = (d - theta) x elementwise, as (d x) - theta x: the diagonal and shift
// of a panelled product, before the panels accumulate their off-diagonals
__global__ void diag_init_kernel(int64_t n, const double* d, const double* x, double* y,
                                 double theta_h, const double* theta_d, int theta_neg,
                                 const int* skip) {
  if (skip && *skip) return;
  double theta = theta_h;
  if (theta_d) theta += theta_neg ? -*theta_d : *theta_d;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    const double xi = __ldcs(x + i);
    double s = 0.0 + __ldcs(d + i) * xi;
    if (theta != 0.0) s -= theta * xi;
    __stcs(y + i, s);
  }
}
}  // namespace

// The panel chain behind lg_spmv: y = (D - theta I) x, then every panel
// accumulates its off-diagonals (each panel's schedule holds only the rows
// with entries in its columns).  Same stream, same workspace, in order.
extern "C" int lg_spmv_panels_(const lg_csr* a, const double* x, double* y, double theta_h,
                               const double* theta_d, int theta_neg, const int* skip,
                               lg_ws* ws, void* stream) {
  {
    const int64_t g = std::max<int64_t>(
        1, std::min<int64_t>((a->n + 255) / 256, (int64_t)dev_info().sm_count * 8));
    diag_init_kernel<<<(unsigned)g, 256, 0, (cudaStream_t)stream>>>(
        a->n, a->pdiag, x, y, theta_h, theta_d, theta_neg, skip);
    LG_LAUNCH_CHECK("diag_init_kernel");
  }
  for (int k = 0; k < a->npanels; ++k) {
    const lg_csr* m = a->panel[k];
    if (m->nblocks == 0) continue;
    if (m->nlong) {
      int rc = ensure_long_ws(ws, m);
      if (rc) return rc;
    }
    SpmvArgs args = spmv_args(m, x, y, ws);
    args.accum = 1;
    args.pdiag = nullptr;
    args.skip = skip;
    int rc = launch(args, (cudaStream_t)stream, true);
    if (rc) return rc;
  }
  return LG_OK;
}

// y += A x (no epilogue): the exterior half of a split row block.
extern "C" int lg_spmv_acc(const lg_csr* a, const double* x, double* y, lg_ws* ws,
                           const int* skip, void* stream) {
  if (!a || !x || !y || !ws) return fail(LG_EINVAL, "lg_spmv_acc: NULL argument");
  if (a->n == 0 || a->nblocks == 0) return LG_OK;
  if (a->nlong) {
    int rc = ensure_long_ws(ws, a);
    if (rc) return rc;
  }
  if (a->npanels > 1) {   // accumulating panels (exterior half of a row block)
    for (int k = 0; k < a->npanels; ++k) {
      const lg_csr* m = a->panel[k];
      if (m->nblocks == 0) continue;
      if (m->nlong) {
        int rc = ensure_long_ws(ws, m);
        if (rc) return rc;
      }
      SpmvArgs args = spmv_args(m, x, y, ws);
      args.accum = 1;
      args.pdiag = nullptr;
      args.skip = skip;
      int rc = launch(args, (cudaStream_t)stream, true);
      if (rc) return rc;
    }
    return LG_OK;
  }
  SpmvArgs args = spmv_args(a, x, y, ws);
  args.accum = 1;
  args.skip = skip;
  return launch(args, (cudaStream_t)stream, a->packed != 0);
}

extern "C" {

// Stream row pointers of a matrix (packed: off-diagonal row pointers; plain:
// row_ptr) to the host, n + 1 entries -- what the nnz-balanced row
// partition of a device-only matrix is computed from.
// Host CSR of a packed matrix (also device-only ones, e.g. C5's device-built
// Laplacian): row pointers, columns and values with the diagonal in its
// sorted position -- what the host IC(0) factorization (ic0.py:48-116)
// consumes.  rp_h [n+1], col_h / val_h [noff + n] (every packed row stores
// its diagonal).
extern "C" int lg_csr_export_host(const lg_csr* a, int64_t* rp_h, int64_t* col_h,
                                  double* val_h) {
  if (!a || !rp_h || !col_h || !val_h) return fail(LG_EINVAL, "lg_csr_export_host: bad argument");
  if (!a->packed) return lg_csr_download(a, rp_h, col_h, val_h);
  const int64_t n = a->n;
  std::vector<int64_t> prp((size_t)n + 1);
  std::vector<uint32_t> pcol((size_t)a->noff);
  std::vector<double> diag((size_t)n), table((size_t)std::max(a->nvals, 1));
  LG_CUDA(cudaMemcpy(prp.data(), a->prp, 8 * (size_t)(n + 1), cudaMemcpyDeviceToHost));
  if (a->noff)
    LG_CUDA(cudaMemcpy(pcol.data(), a->pcol, 4 * (size_t)a->noff, cudaMemcpyDeviceToHost));
  LG_CUDA(cudaMemcpy(diag.data(), a->pdiag, 8 * (size_t)n, cudaMemcpyDeviceToHost));
  if (a->nvals)
    LG_CUDA(cudaMemcpy(table.data(), a->table, 8 * (size_t)a->nvals, cudaMemcpyDeviceToHost));
  const uint32_t cmask = (a->cbits >= 32) ? 0xffffffffu : ((1u << a->cbits) - 1u);
  int64_t o = 0;
  rp_h[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    bool placed = false;
    for (int64_t k = prp[(size_t)r]; k < prp[(size_t)r + 1]; ++k) {
      const uint32_t w = pcol[(size_t)k];
      const int64_t c = w & cmask;
      if (!placed && c > r) {
        col_h[o] = r;
        val_h[o++] = diag[(size_t)r];
        placed = true;
      }
      col_h[o] = c;
      val_h[o++] = table[(size_t)(w >> a->cbits)];
    }
    if (!placed) {
      col_h[o] = r;
      val_h[o++] = diag[(size_t)r];
    }
    rp_h[r + 1] = o;
  }
  return LG_OK;
}

extern "C" int lg_csr_row_ptr(const lg_csr* a, int64_t* host_out) {
  if (!a || !host_out) return fail(LG_EINVAL, "lg_csr_row_ptr: bad argument");
  LG_CUDA(cudaMemcpy(host_out, a->packed ? a->prp : a->row_ptr, 8 * (size_t)(a->n + 1),
                     cudaMemcpyDeviceToHost));
  return LG_OK;
}

// Device diagonal (degrees) of a packed matrix, for Jacobi preconditioning
// of device-only matrices.
extern "C" int lg_csr_diagonal(const lg_csr* a, double* d_out) {
  if (!a || !d_out) return fail(LG_EINVAL, "lg_csr_diagonal: bad argument");
  if (!a->packed) return fail(LG_EINVAL, "lg_csr_diagonal: only for packed matrices");
  if (!a->pdiag) {  // a part without the diagonal
    LG_CUDA(cudaMemset(d_out, 0, 8 * (size_t)a->n));
    return LG_OK;
  }
  LG_CUDA(cudaMemcpy(d_out, a->pdiag, 8 * (size_t)a->n, cudaMemcpyDeviceToDevice));
  return LG_OK;
}

}  // extern "C"

// ---- FSAI setup on the device (packed single-valued matrices) -------------
// The host setup (lg_fsai.cu) needs the matrix on the host; a device-only
// matrix (C5: 2.1e9 nonzeros built on the GPU) gets the same preconditioner
// built here, one warp per row:
//   P_i = the last kmax - 1 strictly lower columns of row i (with a single
//         off-diagonal value every |a_ij| ties, and the reference tie rule
//         of lg_fsai.cu keeps the larger columns) + {i};
//   M = A[P_i, P_i] in shared memory (adjacency by binary search in the rows
//       of P_i, diagonal from the stored diagonal), right-looking Cholesky
//       M = C C^T by the warp (lane r owns row r), C C^T g = e_last,
//   G[i, P_i] = g / sqrt(g_last).
// Then G^T by a stable radix sort of the entries on their column.  Both come
// back as plain-format matrices (the apply is lg_spmv on each).
namespace {
constexpr int kFsaiMax = 32;   // kmax limit of the device setup (one warp)

__global__ void fsai_count(int64_t n, const int64_t* prp, const uint32_t* pcol, uint32_t cmask,
                           int kmax, int64_t* cnt) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    int64_t lo = prp[i], hi = prp[i + 1];
    while (lo < hi) {   // first column >= i
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)(pcol[mid] & cmask) < i) lo = mid + 1;
      else hi = mid;
    }
    const int64_t low = lo - prp[i];
    cnt[i] = (low < kmax - 1 ? low : kmax - 1) + 1;
  }
}

__device__ __forceinline__ bool has_col(const int64_t* prp, const uint32_t* pcol, uint32_t cmask,
                                        int64_t r, int64_t c) {
  int64_t lo = prp[r], hi = prp[r + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int64_t v = pcol[mid] & cmask;
    if (v == c) return true;
    if (v < c) lo = mid + 1;
    else hi = mid;
  }
  return false;
}

constexpr int kFsaiWarps = 4;

__global__ void __launch_bounds__(32 * kFsaiWarps) fsai_rows(
    int64_t n, const int64_t* prp, const uint32_t* pcol, uint32_t cmask, const double* pdiag,
    double offv, const int64_t* g_rp, int32_t* g_col, double* g_val, int* bad) {
  __shared__ double M_sm[kFsaiWarps][kFsaiMax][kFsaiMax + 1];
  __shared__ int64_t P_sm[kFsaiWarps][kFsaiMax];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double (*M)[kFsaiMax + 1] = M_sm[w];
  int64_t* P = P_sm[w];
  const int64_t gw = (int64_t)blockIdx.x * kFsaiWarps + w;
  const int64_t nw = (int64_t)gridDim.x * kFsaiWarps;
  for (int64_t i = gw; i < n; i += nw) {
    const int64_t o = g_rp[i];
    const int m = (int)(g_rp[i + 1] - o);
    // pattern: the m - 1 lower columns just below the diagonal's position
    int64_t lo = prp[i], hi = prp[i + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)(pcol[mid] & cmask) < i) lo = mid + 1;
      else hi = mid;
    }
    if (lane < m - 1) P[lane] = pcol[lo - (m - 1) + lane] & cmask;
    if (lane == m - 1) P[lane] = i;
    __syncwarp();
    if (lane < m) {
      const int64_t pa = P[lane];
      for (int b = 0; b < lane; ++b) {
        const double v = has_col(prp, pcol, cmask, pa, P[b]) ? offv : 0.0;
        M[lane][b] = v;
        M[b][lane] = v;
      }
      M[lane][lane] = pdiag[pa];
    }
    __syncwarp();
    // right-looking Cholesky, lane r owns row r (lower part)
    bool ok = true;
    for (int j = 0; j < m; ++j) {
      const double d = M[j][j];
      if (!(d > 0.0)) ok = false;
      const double c = sqrt(d);
      __syncwarp();
      if (lane == j) M[j][j] = c;
      if (lane > j && lane < m) M[lane][j] /= c;
      __syncwarp();
      if (lane > j && lane < m) {
        const double lj = M[lane][j];
        for (int k = j + 1; k <= lane; ++k) M[lane][k] -= lj * M[k][j];
      }
      __syncwarp();
    }
    if (!ok) {
      if (lane == 0) atomicExch(bad, 1);
      continue;
    }
    // C C^T g = e_last: forward gives y = e_last / C[m-1][m-1]; backward
    // C^T g = y from the last row up, one warp reduction per row
    const double cl = M[m - 1][m - 1];
    double g_mine = (lane == m - 1) ? 1.0 / (cl * cl) : 0.0;
    for (int r = m - 2; r >= 0; --r) {
      double t = (lane > r && lane < m) ? M[lane][r] * g_mine : 0.0;
      t = warp_sum(t);
      if (lane == r) g_mine = -t / M[r][r];
    }
    // G row = g / sqrt(g_last), sqrt(g_last) = 1 / C[m-1][m-1]
    if (lane < m) {
      g_col[o + lane] = (int32_t)P[lane];
      g_val[o + lane] = g_mine * cl;
    }
    __syncwarp();
  }
}

__global__ void gather_rows_vals(int64_t nnz, const int64_t* idx, const int32_t* rows,
                                 const double* vals, int32_t* rows_out, double* vals_out) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += st) {
    rows_out[e] = rows[idx[e]];
    vals_out[e] = vals[idx[e]];
  }
}

__global__ void expand_rows(int64_t n, const int64_t* rp, int32_t* row_of) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) row_of[k] = (int32_t)i;
}

__global__ void iota64(int64_t m, int64_t* v) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += st) v[e] = e;
}

__global__ void count_cols(int64_t m, const int32_t* col, unsigned long long* cnt) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += st)
    atomicAdd(cnt + col[e] + 1, 1ull);
}

int grid_of(int64_t work, int per) {
  const int64_t g = (work + per - 1) / per;
  const int64_t cap = (int64_t)dev_info().sm_count * 32;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}
}  // namespace

// A plain-format n x n matrix over device arrays (taken over: freed with the
// handle); the schedule is built from the row pointers copied to the host.
static int plain_from_device(int64_t n, int64_t* rp, int32_t* col, double* val, int64_t nnz,
                             lg_csr** out) {
  std::vector<int64_t> hrp((size_t)n + 1);
  LG_CUDA(cudaMemcpy(hrp.data(), rp, 8 * (size_t)(n + 1), cudaMemcpyDeviceToHost));
  lg_csr* a = new lg_csr();
  a->n = n;
  a->nnz = nnz;
  a->row_ptr = rp;
  a->col = col;
  a->val = val;
  const int rc = attach_schedule(a, hrp.data(), nullptr, "fsai");
  if (rc) {
    lg_csr_destroy(a);
    return rc;
  }
  *out = a;
  return LG_OK;
}

extern "C" int lg_fsai_device(const lg_csr* a, int kmax, lg_csr** g_out, lg_csr** gt_out) {
  if (!a || !g_out || !gt_out || kmax < 1 || kmax > kFsaiMax)
    return fail(LG_EINVAL, "lg_fsai_device: bad argument (1 <= kmax <= 32)");
  if (!a->packed || a->nvals != 1 || !a->pdiag)
    return fail(LG_EINVAL, "lg_fsai_device: needs a packed matrix with one off-diagonal value "
                           "(use the host setup, lg_fsai_factorize, otherwise)");
  const int64_t n = a->n;
  const uint32_t cmask = (a->cbits >= 32) ? 0xffffffffu : ((1u << a->cbits) - 1u);
  double offv = 0.0;
  LG_CUDA(cudaMemcpy(&offv, a->table, 8, cudaMemcpyDeviceToHost));
  int64_t *cnt = nullptr, *grp = nullptr, *idx = nullptr, *idx2 = nullptr, *trp = nullptr;
  int32_t *gcol = nullptr, *grow = nullptr, *tcol_keys = nullptr, *trow = nullptr;
  double *gval = nullptr, *tval = nullptr;
  unsigned long long* ccount = nullptr;
  int* bad = nullptr;
  void* tmp = nullptr;
  auto cleanup = [&]() {
    cudaFree(cnt);
    cudaFree(idx);
    cudaFree(idx2);
    cudaFree(grow);
    cudaFree(tcol_keys);
    cudaFree(ccount);
    cudaFree(bad);
    cudaFree(tmp);
  };
  auto oom = [&](const char* what) {
    cleanup();
    cudaFree(grp);
    cudaFree(gcol);
    cudaFree(gval);
    cudaFree(trp);
    cudaFree(trow);
    cudaFree(tval);
    return fail(LG_ENOMEM, std::string("lg_fsai_device: ") + what);
  };
  if (cudaMalloc(&cnt, 8 * (size_t)n) != cudaSuccess ||
      cudaMalloc(&grp, 8 * (size_t)(n + 1)) != cudaSuccess ||
      cudaMalloc(&bad, sizeof(int)) != cudaSuccess)
    return oom("allocation");
  cudaMemset(bad, 0, sizeof(int));
  fsai_count<<<grid_of(n, 256), 256>>>(n, a->prp, a->pcol, cmask, kmax, cnt);
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, grp + 1, n);
  if (cudaMalloc(&tmp, std::max<size_t>(tb, 16)) != cudaSuccess) return oom("scan scratch");
  cudaMemset(grp, 0, 8);
  cub::DeviceScan::InclusiveSum(tmp, tb, cnt, grp + 1, n);
  cudaFree(tmp);
  tmp = nullptr;
  int64_t nnz = 0;
  LG_CUDA(cudaMemcpy(&nnz, grp + n, 8, cudaMemcpyDeviceToHost));
  if (cudaMalloc(&gcol, 4 * (size_t)(nnz + kStreamPad)) != cudaSuccess ||
      cudaMalloc(&gval, 8 * (size_t)(nnz + kStreamPad)) != cudaSuccess)
    return oom("G arrays");
  {
    const int64_t blocks = std::min<int64_t>((n + kFsaiWarps - 1) / kFsaiWarps,
                                             (int64_t)dev_info().sm_count * 64);
    fsai_rows<<<(unsigned)std::max<int64_t>(blocks, 1), 32 * kFsaiWarps>>>(
        n, a->prp, a->pcol, cmask, a->pdiag, offv, grp, gcol, gval, bad);
  }
  int hbad = 0;
  LG_CUDA(cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost));
  if (hbad) {
    cleanup();
    cudaFree(grp);
    cudaFree(gcol);
    cudaFree(gval);
    return fail(LG_EBREAKDOWN, "lg_fsai_device: a row's pattern submatrix is not positive "
                               "definite");
  }
  // G^T: entries sorted (stably) by column; row indices and values follow
  if (cudaMalloc(&grow, 4 * (size_t)nnz) != cudaSuccess ||
      cudaMalloc(&idx, 8 * (size_t)nnz) != cudaSuccess ||
      cudaMalloc(&idx2, 8 * (size_t)nnz) != cudaSuccess ||
      cudaMalloc(&tcol_keys, 4 * (size_t)nnz) != cudaSuccess ||
      cudaMalloc(&trow, 4 * (size_t)(nnz + kStreamPad)) != cudaSuccess ||
      cudaMalloc(&tval, 8 * (size_t)(nnz + kStreamPad)) != cudaSuccess ||
      cudaMalloc(&trp, 8 * (size_t)(n + 1)) != cudaSuccess ||
      cudaMalloc(&ccount, 8 * (size_t)(n + 1)) != cudaSuccess)
    return oom("G^T arrays");
  expand_rows<<<grid_of(n, 256), 256>>>(n, grp, grow);
  iota64<<<grid_of(nnz, 256), 256>>>(nnz, idx);
  int cbits = 1;
  while (((int64_t)1 << cbits) < n) ++cbits;
  tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, gcol, tcol_keys, idx, idx2, nnz, 0, cbits);
  if (cudaMalloc(&tmp, std::max<size_t>(tb, 16)) != cudaSuccess) return oom("sort scratch");
  cub::DeviceRadixSort::SortPairs(tmp, tb, gcol, tcol_keys, idx, idx2, nnz, 0, cbits);
  gather_rows_vals<<<grid_of(nnz, 256), 256>>>(nnz, idx2, grow, gval, trow, tval);
  cudaMemset(ccount, 0, 8 * (size_t)(n + 1));
  count_cols<<<grid_of(nnz, 256), 256>>>(nnz, gcol, ccount);
  cudaFree(tmp);
  tmp = nullptr;
  tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, ccount, (unsigned long long*)trp, n + 1);
  if (cudaMalloc(&tmp, std::max<size_t>(tb, 16)) != cudaSuccess) return oom("scan scratch");
  cub::DeviceScan::InclusiveSum(tmp, tb, ccount, (unsigned long long*)trp, n + 1);
  cudaError_t e = cudaDeviceSynchronize();
  cleanup();
  if (e != cudaSuccess) {
    cudaFree(grp);
    cudaFree(gcol);
    cudaFree(gval);
    cudaFree(trp);
    cudaFree(trow);
    cudaFree(tval);
    return fail(LG_ECUDA, std::string("lg_fsai_device: ") + cudaGetErrorString(e));
  }
  lg_csr *g = nullptr, *gt = nullptr;
  int rc = plain_from_device(n, grp, gcol, gval, nnz, &g);
  if (rc) return rc;
  rc = plain_from_device(n, trp, trow, tval, nnz, &gt);
  if (rc) {
    lg_csr_destroy(g);
    return rc;
  }
  *g_out = g;
  *gt_out = gt;
  return LG_OK;
}
