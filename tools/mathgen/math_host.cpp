/* Host build of the device math library (same source, IEEE fma from libm)
 * exposed to Python for validation: tests/test_device_math.py. */
#define MUSR_HOST_TEST 1
#include "../../paper_1604_02334_b200/csrc/musr_math.cuh"

extern "C" {

void v_exp(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = musr_exp(x[i]); }
void v_cos(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = musr_cos(x[i]); }
void v_sin(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = musr_sin(x[i]); }
void v_exp_anchored(const double* x, const double* x0, double* y, long n) {
  for (long i = 0; i < n; ++i) {
    bool ok = true;
    const double e0 = musr_exp(x0[i]);
    y[i] = musr_exp_anchored(x[i], x0[i], e0, ok);
    if (!ok) y[i] = NAN;
  }
}
// exp(c * y) anchored on y (c = +-2^k): coefficients scaled as codegen.py emits them
void v_exp_anchored_k(const double* y, const double* y0, const double* c, double* out, long n) {
  for (long i = 0; i < n; ++i) {
    bool ok = true;
    const double k = c[i];
    const double e0 = musr_exp(k * y0[i]);
    int ex;
    frexp(fabs(k), &ex);
    const int hi = (1023 - 10 - (ex - 1)) << 20;
    out[i] = musr_exp_anchored_k(y[i], y0[i], e0, k * k * k * k * 0x1.5555555555555p-5,
                                 k * k * k * 0x1.5555555555555p-3, k * k * 0.5, k, hi, ok);
    if (!ok) out[i] = NAN;
  }
}
void v_pow_anchored(const double* x, const double* x0, const double* b, double* y, long n) {
  for (long i = 0; i < n; ++i) {
    bool ok = true;
    const MusrPowAnchor a = musr_pow_anchor(x0[i], pow(x0[i], b[i]), b[i]);
    y[i] = musr_pow_anchored(x[i], a, ok);
    if (!ok) y[i] = NAN;
  }
}
// rotated cos of a_j = a0 + D + e (codegen.py _rotated): c0*X - s0*Y
void v_cos_rotated(const double* a0, const double* D, const double* e, double* y, long n) {
  for (long i = 0; i < n; ++i) {
    const double c0 = musr_cos(a0[i]), s0 = musr_sin(a0[i]);
    const double cd = musr_cos(D[i]), sd = musr_sin(D[i]);
    const double X = fma(-sd, e[i], cd), Y = fma(cd, e[i], sd);
    y[i] = fma(c0, X, -(s0 * Y));
  }
}
void v_pow_fast(const double* x, const double* b, double* y, long n) {
  for (long i = 0; i < n; ++i) {
    bool ok = true;
    y[i] = musr_pow_fast(x[i], b[i], musr_log_t, ok);
    if (!ok) y[i] = NAN;
  }
}
void v_log_hl(const double* x, double* h, double* l, long n) {
  for (long i = 0; i < n; ++i) {
    bool ok = true;
    musr_log_hl(x[i], musr_log_t, &h[i], &l[i], ok);
  }
}
void v_rcp_approx(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) y[i] = musr_rcp_approx(x[i]);
}
void v_div_y(const double* a, const double* b, const double* yb, double* q, long n) {
  for (long i = 0; i < n; ++i) q[i] = musr_div_y(a[i], b[i], yb[i]);
}

void v_log(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) {
    bool ok = true;
    y[i] = musr_log_fast(x[i], musr_log_t, ok);
    if (!ok) y[i] = NAN;
  }
}
// the exponent-folded table log (MLH hot path), table built like the kernel's
void v_log_k(const double* x, double* y, long n) {
  static double2 t2[MUSR_LOGK_N];
  static double t1[MUSR_LOGK_N];
  for (int i = 0; i < MUSR_LOGK_N; ++i) musr_logk_entry(musr_log_t, i, &t2[i], &t1[i]);
  for (long i = 0; i < n; ++i) {
    bool ok = true;
    y[i] = musr_log_fast_k(x[i], t2, t1, ok);
    if (!ok) y[i] = NAN;
  }
}
void v_div_fast(const double* a, const double* b, double* q, long n) {
  for (long i = 0; i < n; ++i) {
    bool ok = true;
    q[i] = musr_div_fast(a[i], b[i], ok);
    if (!ok) q[i] = NAN;
  }
}

// chi2 error and reciprocal for integer counts k in [lo, hi) by the kernel's
// big-count path: err = max(1, musr_sqrt_fast(k)), rcp = musr_div_fast(1, err);
// returns the number of k where either differs from IEEE (sqrt, 1 / err) or ok dropped
long v_err_rcp_scan(long lo, long hi) {
  long bad = 0;
  for (long k = lo; k < hi; ++k) {
    bool ok = true;
    const double d = (double)k;
    const double s = musr_sqrt_fast(d, ok);
    const double err = s < 1.0 ? 1.0 : s;
    const double rcp = musr_div_fast(1.0, err, ok);
    const double e_ref = fmax(1.0, sqrt(d));
    if (!ok || err != e_ref || rcp != 1.0 / e_ref) ++bad;
  }
  return bad;
}
void v_sqrt_fast(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) {
    bool ok = true;
    y[i] = musr_sqrt_fast(x[i], ok);
    if (!ok) y[i] = NAN;
  }
}

}  // extern "C"
