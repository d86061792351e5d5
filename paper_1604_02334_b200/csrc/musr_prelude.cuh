// musr_prelude.cuh -- device helpers available to the generated theory
// fragment (codegen.py).  Included before the fragment; musr_kernel.cuh after.
#ifndef MUSR_PRELUDE_CUH
#define MUSR_PRELUDE_CUH

#include "musr_math.cuh"

#ifndef MUSR_PT
#define MUSR_PT 8  // bins per consumer thread (musr_theory_vec works on one run)
#endif
#ifndef MUSR_EXP_DEG3
#define MUSR_EXP_DEG3 1  // anchored exp: degree-3 series for runs with every |d| < 2^-13
#endif

__device__ __forceinline__ double musr_sq(double x) { return __dmul_rn(x, x); }

// np.power with a bin-uniform exponent (numpy 2.x fast paths, measured).
__device__ __forceinline__ double musr_npy_pow_u(double x, double b) {
  if (b == 2.0) return __dmul_rn(x, x);
  if (b == 0.5) return __dsqrt_rn(x);
  if (b == -1.0) return __ddiv_rn(1.0, x);
  if (b == 1.0) return x;
  if (b == 0.0) return 1.0;
  return pow(x, b);
}

#endif  // MUSR_PRELUDE_CUH
