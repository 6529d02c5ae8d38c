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

#include "lg_scalar.cuh"

namespace lg {

__global__ void scalar_kernel(const __grid_constant__ ScalarProg p, double* sg,
                              int* flags, const int* skip) {
  if (skip && *skip) return;
  cta_run_program(p, sg, flags);
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
