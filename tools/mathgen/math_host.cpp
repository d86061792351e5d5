/* Host build of the device math library (same source, IEEE fma from libm)
 * exposed to Python for validation: tests/test_device_math.py. */
#define MUSR_HOST_TEST 1
#include "../../paper_1604_02334_b200/csrc/musr_math.cuh"

extern "C" {

void v_exp(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = musr_exp(x[i]); }
void v_cos(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = musr_cos(x[i]); }
void v_sin(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = musr_sin(x[i]); }
void v_div_y(const double* a, const double* b, const double* yb, double* q, long n) {
  for (long i = 0; i < n; ++i) q[i] = musr_div_y(a[i], b[i], yb[i]);
}

}  // extern "C"
