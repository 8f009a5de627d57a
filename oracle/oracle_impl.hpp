// oracle_impl.hpp — template bodies for oracle.hpp (TEST INFRASTRUCTURE).
#pragma once

#include <cmath>
#include <exception>
#include <mutex>
#include <thread>

namespace oracle {

// common.hpp:55-81: static block partition, first exception captured.
template <typename F>
void parallel_for(std::int64_t n, F&& body) {
  const int nt = thread_count();
  if (nt <= 1 || n < 2) {
    for (std::int64_t i = 0; i < n; ++i) body(i);
    return;
  }
  const int workers = (int)std::min<std::int64_t>(nt, n);
  std::vector<std::thread> pool;
  std::exception_ptr first;
  std::mutex mu;
  for (int t = 0; t < workers; ++t) {
    pool.emplace_back([&, t]() {
      const std::int64_t lo = n * t / workers, hi = n * (t + 1) / workers;
      try {
        for (std::int64_t i = lo; i < hi; ++i) body(i);
      } catch (...) {
        std::scoped_lock lk(mu);
        if (!first) first = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  if (first) std::rethrow_exception(first);
}

inline double dot(int n, const double* a, const double* b) {
  double s = 0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

// SPEC.md:431-439 (pcg) with the pins of SURVEY.md Appendix B.7:
//   x0 = 0; residuals[0] = |b|; true residual r = b - A x after the update at
//   every iteration k with k % 50 == 0; stop at the first k with |r| < rtol|b|;
//   <r, M r> <= 0 -> indefiniteness error; max_iter -> non-converged report.
template <typename A, typename M>
void pcg(int n, A&& aapply, M&& mapply, const double* b, double* x, double rtol, int max_iter,
         SolveReport& rep) {
  std::vector<double> r(b, b + n), z(n), p(n), q(n);
  for (int i = 0; i < n; ++i) x[i] = 0.0;
  rep = SolveReport{};
  const double bnorm = std::sqrt(dot(n, b, b));
  rep.residuals.push_back(bnorm);
  if (bnorm == 0.0) {
    rep.converged = true;
    return;
  }
  const double stop = rtol * bnorm;
  mapply(r.data(), z.data());
  double rz = dot(n, r.data(), z.data());
  if (!(rz > 0)) fail(ErrorCode::Internal, "pcg: preconditioner is not positive definite (<r,Mr> <= 0)");
  p = z;
  for (int k = 1; k <= max_iter; ++k) {
    aapply(p.data(), q.data());
    const double pq = dot(n, p.data(), q.data());
    if (!(pq > 0)) fail(ErrorCode::Internal, "pcg: operator is not positive definite (<p,Ap> <= 0)");
    const double alpha = rz / pq;
    for (int i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    if (k % 50 == 0) {
      aapply(x, q.data());
      for (int i = 0; i < n; ++i) r[i] = b[i] - q[i];
    }
    const double rn = std::sqrt(dot(n, r.data(), r.data()));
    rep.residuals.push_back(rn);
    rep.alpha.push_back(alpha);
    rep.iterations = k;
    if (rn < stop) {
      rep.converged = true;
      break;
    }
    mapply(r.data(), z.data());
    const double rz_new = dot(n, r.data(), z.data());
    if (!(rz_new > 0)) fail(ErrorCode::Internal, "pcg: preconditioner is not positive definite (<r,Mr> <= 0)");
    const double beta = rz_new / rz;
    rz = rz_new;
    rep.beta.push_back(beta);
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  if (rep.alpha.size() >= 2) {
    condition_estimate(rep.alpha, rep.beta, rep.lmin, rep.lmax);
    rep.cond = rep.lmax / rep.lmin;
  }
}

}  // namespace oracle
