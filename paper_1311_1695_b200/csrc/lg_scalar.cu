// lg_scalar.cu -- device-side scalar programs.
//
// The solvers' scalar recurrences (Polak-Ribiere beta with its reset and
// clamp, dacg.py:188-195; the 2x2 plane pencil, dacg.py:55-96; the RQ
// monotonicity guard, dacg.py:221-225; PCG gamma / beta and the indefinite /
// converged tests, pcg.py:133-155) depend only on dot products that the
// vector passes leave in device memory.  Running them on the device keeps an
// iteration free of host round trips: one thread interprets a short program
// of 4-byte instructions {op, dst, a, b} over a 256-slot register file of
// doubles and writes predicate flags that later kernels of the same
// iteration test (their `skip` argument).  The programs are assembled by the
// Python layer (paper_1311_1695_b200/_scalar.py).
#include <cmath>
#include <cstring>

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

__device__ void run_program(const ScalarProg& p, double* s, int* flags);

__global__ void scalar_kernel(const __grid_constant__ ScalarProg p, double* sg,
                              int* flags, const int* skip) {
  if (skip && *skip) return;
  // the slot window lives in shared memory while the program runs: each
  // instruction reads what the previous one wrote, and a global-memory
  // round trip per instruction would cost ~0.3 us instead of ~30 cycles
  __shared__ double s[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = sg[i];
  __syncwarp();
  if (threadIdx.x == 0) run_program(p, s, flags);
  __syncwarp();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sg[i] = s[i];
}

__device__ void run_program(const ScalarProg& p, double* s, int* flags) {
  for (int k = 0; k < p.nops; ++k) {
    const uint32_t w = p.ops[k];
    const uint8_t op = w & 0xff, d = (w >> 8) & 0xff, a = (w >> 16) & 0xff,
                  b = (w >> 24) & 0xff;
    switch (op) {
      case OP_NOP: break;
      case OP_MOV: s[d] = s[a]; break;
      case OP_IMM: s[d] = p.imm[a]; break;
      case OP_ADD: s[d] = s[a] + s[b]; break;
      case OP_SUB: s[d] = s[a] - s[b]; break;
      case OP_MUL: s[d] = s[a] * s[b]; break;
      case OP_DIV: s[d] = s[a] / s[b]; break;
      case OP_SQRT: s[d] = sqrt(s[a]); break;
      case OP_NEG: s[d] = -s[a]; break;
      case OP_HYPOT: s[d] = hypot(s[a], s[b]); break;
      case OP_ABS: s[d] = fabs(s[a]); break;
      case OP_MAX: s[d] = fmax(s[a], s[b]); break;
      case OP_MIN: s[d] = fmin(s[a], s[b]); break;
      case OP_LE: s[d] = (s[a] <= s[b]) ? 1.0 : 0.0; break;
      case OP_LT: s[d] = (s[a] < s[b]) ? 1.0 : 0.0; break;
      case OP_EQ: s[d] = (s[a] == s[b]) ? 1.0 : 0.0; break;
      case OP_NE: s[d] = (s[a] != s[b]) ? 1.0 : 0.0; break;
      case OP_GT: s[d] = (s[a] > s[b]) ? 1.0 : 0.0; break;
      case OP_GE: s[d] = (s[a] >= s[b]) ? 1.0 : 0.0; break;
      case OP_SEL: if (s[a] != 0.0) s[d] = s[b]; break;
      case OP_AND: s[d] = (s[a] != 0.0 && s[b] != 0.0) ? 1.0 : 0.0; break;
      case OP_OR: s[d] = (s[a] != 0.0 || s[b] != 0.0) ? 1.0 : 0.0; break;
      case OP_NOT: s[d] = (s[a] == 0.0) ? 1.0 : 0.0; break;
      case OP_FLAG: flags[d] = (s[a] != 0.0) ? 1 : 0; break;
      case OP_FLAGOR: if (s[a] != 0.0) flags[d] = 1; break;
      case OP_LDFLAG: s[d] = (double)flags[a]; break;
      case OP_HALTIF: if (s[a] != 0.0) return; break;
      case OP_DIVZ: s[d] = (s[b] != 0.0) ? s[a] / s[b] : 0.0; break;
      case OP_INC: s[d] += 1.0; break;
      case OP_RECIP: s[d] = 1.0 / s[a]; break;
      default: return;
    }
  }
}

}  // namespace lg

using namespace lg;

extern "C" int lg_scalar_prog(double* s, int* flags, const uint8_t* prog_h,
                              int nops, const double* imm_h, int nimm,
                              const int* skip, void* stream) {
  if (!s || nops < 0 || nops > LG_MAXOPS || nimm < 0 || nimm > LG_MAXIMM ||
      (nops > 0 && !prog_h) || (nimm > 0 && !imm_h))
    return fail(LG_EINVAL, "lg_scalar_prog: bad program");
  static thread_local ScalarProg p;
  p.nops = nops;
  std::memcpy(p.ops, prog_h, 4 * (size_t)nops);
  if (nimm) std::memcpy(p.imm, imm_h, sizeof(double) * (size_t)nimm);
  scalar_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(p, s, flags, skip);
  LG_LAUNCH_CHECK("scalar_kernel");
  return LG_OK;
}
