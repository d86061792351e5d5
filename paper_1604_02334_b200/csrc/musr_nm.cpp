// musr_nm.cpp -- native Nelder-Mead loop around the GPU objective.
//
// A line-for-line restatement of the package's bounded Nelder-Mead
// (paper_1604_02334_b200/optimize.py, itself bitwise identical to the
// reference pkg/src/blk/optimize.py:41-146), so a fit no longer returns to
// Python between objective evaluations.  Every floating-point operation and
// comparison follows the numpy / Python semantics of that code:
//   * centroid: rows summed in order, then divided by n (np.mean(axis=0));
//   * clamp: np.minimum(np.maximum(x, lo), hi), NaN-propagating;
//   * ranking: np.argsort(kind="stable") with NaNs last;
//   * Python max()/min() of floats (first maximal / minimal element);
//   * np.argmin (first NaN if any, else the first minimum).
// The iterates are therefore bit-identical to the Python loop's for the same
// objective values (tests/test_host.py checks the core against optimize.py
// through musr_nm_run; tests/test_gpu.py the GPU fit against the Python loop).

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <vector>

#include "../../include/musr_b200.h"

namespace {

using Vec = std::vector<double>;

// Evaluate one point: status 0 = ok (value in *f), anything else aborts.
using EvalFn = std::function<int(const double* x, double* f)>;
// Evaluate k points (rows of xs, n each): values in fs; on a nonzero status
// *bad_row names the first failing row.
using EvalManyFn = std::function<int(const double* xs, int k, double* fs, int* bad_row)>;

double np_maximum(double a, double b) { return (std::isnan(a) || std::isnan(b)) ? NAN : (a >= b ? a : b); }
double np_minimum(double a, double b) { return (std::isnan(a) || std::isnan(b)) ? NAN : (a <= b ? a : b); }

// Python max(a, b, c) / min(a, b) on floats: keep the first unless a later one
// compares greater (less).
double py_max3(double a, double b, double c) {
  double m = a;
  if (b > m) m = b;
  if (c > m) m = c;
  return m;
}
double py_min2(double a, double b) { return b < a ? b : a; }

struct NmResult {
  int64_t iterations = 0, evaluations = 0;
  int converged = 0;
  double best_f = 0.0;
};

// The core.  `fail_x` receives the point whose evaluation reported a nonzero
// status (the caller re-raises there).  Returns that status or MUSR_OK.
// `speculate`: evaluate the reflection, expansion and both contraction points
// of an iteration as one batch before deciding (their coordinates depend only
// on the simplex), then take the values the sequential algorithm asks for.
// Every point's value equals its single evaluation bit for bit, and `calls`
// counts only the points the sequential loop evaluates, so iterates, counts
// and budget are unchanged; a failing batch (a speculative point the loop
// might never evaluate) falls back to the sequential evaluations, which fail
// exactly where the reference does.  Opt-in (MUSR_NM_SPECULATE=1): measured
// slower, because a batched evaluation takes the graph path (p upload, uniform
// table kernel, objective, D2H) -- C1 fit 6.4 -> 9.0 ms, C2 152 -> 356 ms
// (profiles/r2q_ab_nm_speculate.txt) -- while one point is a single direct launch.
int nm_core(int n, const double* x0, double f0, const double* step, const double* lo,
            const double* hi, double tol_f, int64_t budget, int restarts, const EvalFn& f1,
            const EvalManyFn& fmany, double* best_x_out, NmResult* res, double* fail_x,
            bool speculate = false) {
  const double alpha = 1.0, beta = 1.0 + 2.0 / n, gamma = 0.75 - 1.0 / (2.0 * n);
  const double delta = (n > 1) ? (1.0 - 1.0 / n) : 0.5;
  int64_t calls = 1;  // the initial point (evaluated by the caller)
  auto clamp = [&](Vec& x) {
    for (int j = 0; j < n; ++j) x[j] = np_minimum(np_maximum(x[j], lo[j]), hi[j]);
  };
  auto eval = [&](const Vec& x, double* f) -> int {
    ++calls;
    const int rc = f1(x.data(), f);
    if (rc != MUSR_OK) std::memcpy(fail_x, x.data(), sizeof(double) * n);
    return rc;
  };
  auto eval_many = [&](const std::vector<Vec>& xs, double* fs) -> int {
    const int k = (int)xs.size();
    if (k < 2) {
      for (int i = 0; i < k; ++i)
        if (const int rc = eval(xs[i], fs + i)) return rc;
      return MUSR_OK;
    }
    calls += k;
    Vec flat((size_t)k * n);
    for (int i = 0; i < k; ++i) std::memcpy(&flat[(size_t)i * n], xs[i].data(), sizeof(double) * n);
    int bad_row = 0;
    const int rc = fmany(flat.data(), k, fs, &bad_row);
    if (rc != MUSR_OK) std::memcpy(fail_x, &flat[(size_t)bad_row * n], sizeof(double) * n);
    return rc;
  };

  Vec best_x(x0, x0 + n);
  clamp(best_x);
  double best_f = f0;
  int64_t iterations = 0;
  int converged = 0;

  std::vector<Vec> simplex(n + 1, Vec(n));
  Vec values(n + 1);
  Vec spec;  // speculative points, 4 x n
  std::vector<int> rank(n + 1);
  for (int pass = 0; pass < restarts + 1; ++pass) {
    simplex[0] = best_x;
    std::vector<Vec> moved;
    for (int k = 0; k < n; ++k) {
      Vec m = best_x;
      m[k] += step[k];
      clamp(m);
      moved.push_back(m);
    }
    values[0] = best_f;
    if (const int rc = eval_many(moved, &values[1])) return rc;
    for (int k = 0; k < n; ++k) simplex[k + 1] = moved[k];

    while (calls < budget) {
      // np.argsort(values, kind="stable"): NaNs last, ties in index order
      std::iota(rank.begin(), rank.end(), 0);
      std::stable_sort(rank.begin(), rank.end(), [&](int a, int b) {
        const double va = values[a], vb = values[b];
        if (std::isnan(va)) return false;
        if (std::isnan(vb)) return true;
        return va < vb;
      });
      {
        std::vector<Vec> s2(n + 1);
        Vec v2(n + 1);
        for (int i = 0; i <= n; ++i) {
          s2[i] = simplex[rank[i]];
          v2[i] = values[rank[i]];
        }
        simplex.swap(s2);
        values.swap(v2);
      }
      const double lowest = values[0], highest = values[n];
      if (std::fabs(highest - lowest) <= tol_f * py_max3(std::fabs(lowest), std::fabs(highest), 1e-300)) {
        converged = 1;
        break;
      }
      ++iterations;
      const Vec worst = simplex[n];
      Vec c = simplex[0];
      for (int i = 1; i < n; ++i)
        for (int j = 0; j < n; ++j) c[j] = c[j] + simplex[i][j];
      for (int j = 0; j < n; ++j) c[j] = c[j] / (double)n;
      Vec xr(n);
      for (int j = 0; j < n; ++j) xr[j] = c[j] + alpha * (c[j] - worst[j]);
      clamp(xr);
      // speculative batch: [xr, xe, outside contraction, inside contraction]
      bool spec_ok = false;
      double sf[4];
      if (speculate) {
        spec.assign((size_t)4 * n, 0.0);
        for (int j = 0; j < n; ++j) {
          spec[j] = xr[j];
          spec[n + j] = c[j] + beta * (xr[j] - c[j]);
          spec[2 * n + j] = c[j] + gamma * (xr[j] - c[j]);
          spec[3 * n + j] = c[j] - gamma * (c[j] - worst[j]);
        }
        for (int r = 1; r < 4; ++r)
          for (int j = 0; j < n; ++j)
            spec[r * n + j] = np_minimum(np_maximum(spec[r * n + j], lo[j]), hi[j]);
        int bad_row = 0;
        spec_ok = fmany(spec.data(), 4, sf, &bad_row) == MUSR_OK;
      }
      // the value at x (speculative slot `slot`, or evaluated now)
      auto value_at = [&](int slot, const Vec& x, double* f) -> int {
        if (!spec_ok) return eval(x, f);
        ++calls;
        *f = sf[slot];
        return MUSR_OK;
      };
      double fr;
      if (const int rc = value_at(0, xr, &fr)) return rc;
      if (fr < values[0]) {
        Vec xe(n);
        for (int j = 0; j < n; ++j) xe[j] = c[j] + beta * (xr[j] - c[j]);
        clamp(xe);
        double fe;
        if (const int rc = value_at(1, xe, &fe)) return rc;
        if (fe < fr) {
          simplex[n] = xe;
          values[n] = fe;
        } else {
          simplex[n] = xr;
          values[n] = fr;
        }
        continue;
      }
      if (fr < values[n - 1]) {
        simplex[n] = xr;
        values[n] = fr;
        continue;
      }
      Vec xc(n);
      const bool outside = fr < values[n];
      if (outside) {
        for (int j = 0; j < n; ++j) xc[j] = c[j] + gamma * (xr[j] - c[j]);
      } else {
        for (int j = 0; j < n; ++j) xc[j] = c[j] - gamma * (c[j] - worst[j]);
      }
      clamp(xc);
      double fc;
      if (const int rc = value_at(outside ? 2 : 3, xc, &fc)) return rc;
      if (fc < py_min2(fr, values[n])) {
        simplex[n] = xc;
        values[n] = fc;
        continue;
      }
      std::vector<Vec> shrunk;
      for (int k = 1; k <= n; ++k) {  // shrink toward the best vertex
        Vec s(n);
        for (int j = 0; j < n; ++j) s[j] = simplex[0][j] + delta * (simplex[k][j] - simplex[0][j]);
        clamp(s);
        simplex[k] = s;
        shrunk.push_back(s);
      }
      if (const int rc = eval_many(shrunk, &values[1])) return rc;
    }
    // np.argmin: the first NaN if there is one, else the first minimum
    int ib = 0;
    for (int i = 0; i <= n; ++i) {
      if (std::isnan(values[i])) { ib = i; break; }
      if (values[i] < values[ib]) ib = i;
    }
    if (values[ib] < best_f) {
      best_f = values[ib];
      best_x = simplex[ib];
    }
    if (calls >= budget) break;
  }
  std::memcpy(best_x_out, best_x.data(), sizeof(double) * n);
  res->iterations = iterations;
  res->evaluations = calls;
  res->converged = converged;
  res->best_f = best_f;
  return MUSR_OK;
}

}  // namespace

extern "C" {

int musr_nm_run(int n, const double* x0, double f0, const double* step, const double* lo,
                const double* hi, double tol_f, int64_t budget, int restarts, musr_nm_eval_fn eval,
                void* user, double* best_x, double* best_f, int64_t* iterations,
                int64_t* evaluations, int* converged, double* fail_x) {
  if (n < 1 || !x0 || !step || !lo || !hi || !eval || !best_x || !fail_x) return MUSR_ERR_ARG;
  EvalFn f1 = [&](const double* x, double* f) { return eval(user, x, 1, n, f); };
  EvalManyFn fm = [&](const double* xs, int k, double* fs, int* bad_row) {
    int rc = MUSR_OK;  // a batch: one callback per point, in order (the callback's contract)
    for (int i = 0; i < k && rc == MUSR_OK; ++i)
      if ((rc = eval(user, xs + (size_t)i * n, 1, n, fs + i)) != MUSR_OK) *bad_row = i;
    return rc;
  };
  NmResult r;
  const char* sv = std::getenv("MUSR_NM_SPECULATE");  // tests: the speculative loop on the host
  const int rc = nm_core(n, x0, f0, step, lo, hi, tol_f, budget, restarts, f1, fm, best_x, &r,
                         fail_x, sv && std::atoi(sv) != 0);
  if (best_f) *best_f = r.best_f;
  if (iterations) *iterations = r.iterations;
  if (evaluations) *evaluations = r.evaluations;
  if (converged) *converged = r.converged;
  return rc;
}

int musr_minimize(musr_ctx* c, int kind, const double* p_full, int n_p, const int32_t* free_idx,
                  int n_free, const double* x0, double f0, const double* step, const double* lo,
                  const double* hi, double tol_f, int64_t budget, int restarts, double* best_x,
                  double* best_f, int64_t* iterations, int64_t* evaluations, int* converged,
                  double* fail_x) {
  if (!c || !p_full || !free_idx || n_free < 1 || n_p < 1) return MUSR_ERR_ARG;
  for (int i = 0; i < n_free; ++i)
    if (free_idx[i] < 0 || free_idx[i] >= n_p) return MUSR_ERR_ARG;
  int n_global = 0;
  if (const int rc = musr_n_datasets(c, &n_global)) return rc;
  std::vector<double> full(p_full, p_full + n_p);
  std::vector<int64_t> bad((size_t)n_global * 8);
  std::vector<double> pts;
  // an objective "raise" (an MLH non-positive model): a nonzero status; the
  // caller re-evaluates fail_x through the reference-semantics path
  constexpr int kRaised = 100;
  auto eval = [&](const double* xs, int k, double* fs, int* bad_row) -> int {
    if (k == 1) {
      for (int i = 0; i < n_free; ++i) full[free_idx[i]] = xs[i];
      if (const int rc = musr_eval(c, kind, full.data(), n_p, nullptr, bad.data(), fs)) return rc;
      for (int j = 0; j < n_global; ++j)
        if (bad[j] >= 0) return kRaised;
      return MUSR_OK;
    }
    pts.assign((size_t)k * n_p, 0.0);
    for (int r = 0; r < k; ++r) {
      std::memcpy(&pts[(size_t)r * n_p], p_full, sizeof(double) * n_p);
      for (int i = 0; i < n_free; ++i) pts[(size_t)r * n_p + free_idx[i]] = xs[(size_t)r * n_free + i];
    }
    if (bad.size() < (size_t)k * n_global) bad.resize((size_t)k * n_global);
    if (const int rc = musr_eval_batch(c, kind, pts.data(), k, n_p, nullptr, bad.data(), fs))
      return rc;
    for (int r = 0; r < k; ++r)
      for (int j = 0; j < n_global; ++j)
        if (bad[(size_t)r * n_global + j] >= 0) {
          *bad_row = r;
          return kRaised;
        }
    return MUSR_OK;
  };
  int unused = 0;
  EvalFn f1 = [&](const double* x, double* f) { return eval(x, 1, f, &unused); };
  EvalManyFn fm = [&](const double* xs, int k, double* fs, int* bad_row) { return eval(xs, k, fs, bad_row); };
  // speculative batches (see nm_core): opt-in, measured slower than single launches
  const char* sv = std::getenv("MUSR_NM_SPECULATE");
  const bool speculate = sv && std::atoi(sv) != 0;
  NmResult r;
  const int rc = nm_core(n_free, x0, f0, step, lo, hi, tol_f, budget, restarts, f1, fm, best_x, &r,
                         fail_x, speculate);
  if (best_f) *best_f = r.best_f;
  if (iterations) *iterations = r.iterations;
  if (evaluations) *evaluations = r.evaluations;
  if (converged) *converged = r.converged;
  return rc;
}

}  // extern "C"
