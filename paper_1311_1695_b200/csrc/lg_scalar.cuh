// lg_scalar.cuh -- the device scalar interpreter (see lg_scalar.cu), shared
// by the stand-alone program kernel and the fused vector pass, whose
// finishing CTA can run a program right after it has written its dot
// products (no launch of its own on the iteration's critical path).
#pragma once
#include "lg_common.cuh"

namespace lg {

enum : uint8_t {
  OP_NOP = 0,
  OP_MOV = 1,     // s[d] = s[a]
  OP_IMM = 2,     // s[d] = imm[a]
  OP_ADD = 3,     // s[d] = s[a] + s[b]
  OP_SUB = 4,
  OP_MUL = 5,
  OP_DIV = 6,
  OP_SQRT = 7,    // s[d] = sqrt(s[a])
  OP_NEG = 8,
  OP_HYPOT = 9,   // s[d] = hypot(s[a], s[b])
  OP_ABS = 10,
  OP_MAX = 11,
  OP_MIN = 12,
  OP_LE = 13,     // s[d] = s[a] <= s[b]
  OP_LT = 14,
  OP_EQ = 15,
  OP_SEL = 16,    // if (s[a] != 0) s[d] = s[b]
  OP_AND = 17,
  OP_OR = 18,
  OP_NOT = 19,
  OP_FLAG = 20,   // flags[d] = s[a] != 0
  OP_FLAGOR = 21, // flags[d] |= s[a] != 0
  OP_LDFLAG = 22, // s[d] = flags[a]
  OP_HALTIF = 23, // stop the program when s[a] != 0
  OP_DIVZ = 24,   // s[d] = s[b] != 0 ? s[a] / s[b] : 0
  OP_INC = 25,    // s[d] += 1
  OP_RECIP = 26,  // s[d] = 1 / s[a]
  OP_NE = 27,
  OP_GT = 28,
  OP_GE = 29,
};

struct ScalarProg {
  int nops;
  uint32_t ops[LG_MAXOPS];
  double imm[LG_MAXIMM];
};

// one thread; ops, slots and flags all in shared memory.  The operands are
// read before the dispatch and every arithmetic case is a single expression
// into r, so the switch compiles to a compact table of small cases (the
// interpreter sits on the iteration's critical path on small graphs).
__device__ __forceinline__ void run_program(const uint32_t* ops, int nops, const double* imm,
                                            double* s, int* flags) {
  for (int k = 0; k < nops; ++k) {
    const uint32_t w = ops[k];
    const uint32_t op = w & 0xff, d = (w >> 8) & 0xff, a = (w >> 16) & 0xff,
                   b = (w >> 24) & 0xff;
    const double va = s[a], vb = s[b];
    double r;
    switch (op) {
      case OP_MOV: r = va; break;
      case OP_IMM: r = imm[a]; break;
      case OP_ADD: r = va + vb; break;
      case OP_SUB: r = va - vb; break;
      case OP_MUL: r = va * vb; break;
      case OP_DIV: r = va / vb; break;
      case OP_SQRT: r = sqrt(va); break;
      case OP_NEG: r = -va; break;
      case OP_HYPOT: r = hypot(va, vb); break;
      case OP_ABS: r = fabs(va); break;
      case OP_MAX: r = fmax(va, vb); break;
      case OP_MIN: r = fmin(va, vb); break;
      case OP_LE: r = (va <= vb) ? 1.0 : 0.0; break;
      case OP_LT: r = (va < vb) ? 1.0 : 0.0; break;
      case OP_EQ: r = (va == vb) ? 1.0 : 0.0; break;
      case OP_NE: r = (va != vb) ? 1.0 : 0.0; break;
      case OP_GT: r = (va > vb) ? 1.0 : 0.0; break;
      case OP_GE: r = (va >= vb) ? 1.0 : 0.0; break;
      case OP_SEL: r = (va != 0.0) ? vb : s[d]; break;
      case OP_AND: r = (va != 0.0 && vb != 0.0) ? 1.0 : 0.0; break;
      case OP_OR: r = (va != 0.0 || vb != 0.0) ? 1.0 : 0.0; break;
      case OP_NOT: r = (va == 0.0) ? 1.0 : 0.0; break;
      case OP_LDFLAG: r = (double)flags[a & 31]; break;
      case OP_DIVZ: r = (vb != 0.0) ? va / vb : 0.0; break;
      case OP_INC: r = s[d] + 1.0; break;
      case OP_RECIP: r = 1.0 / va; break;
      case OP_NOP: continue;
      case OP_FLAG: flags[d & 31] = (va != 0.0) ? 1 : 0; continue;
      case OP_FLAGOR: if (va != 0.0) flags[d & 31] = 1; continue;
      case OP_HALTIF: if (va != 0.0) return; continue;
      default: return;
    }
    s[d] = r;
  }
}


// The whole CTA stages the program, the 256-slot window and the flags in
// shared memory, thread 0 interprets, the CTA writes slots and flags back.
// Call from every thread of one CTA (block-uniform); global writes the CTA
// made before the call are visible to it after the first barrier.
__device__ __forceinline__ void cta_run_program(const ScalarProg& p, double* sg, int* fg) {
  __shared__ double s[256];
  __shared__ uint32_t ops[LG_MAXOPS];
  __shared__ double imm[LG_MAXIMM];
  __shared__ int fl[32];
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = sg[i];
  for (int i = threadIdx.x; i < p.nops; i += blockDim.x) ops[i] = p.ops[i];
  for (int i = threadIdx.x; i < LG_MAXIMM; i += blockDim.x) imm[i] = p.imm[i];
  for (int i = threadIdx.x; i < 32; i += blockDim.x) fl[i] = fg[i];
  __syncthreads();
  if (threadIdx.x == 0) run_program(ops, p.nops, imm, s, fl);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sg[i] = s[i];
  for (int i = threadIdx.x; i < 32; i += blockDim.x) fg[i] = fl[i];
}

}  // namespace lg
