// §3.3 plan selection, host C++.
//
// Independent of oracle/ (different language, different algorithms where the
// paper leaves freedom: GLL nodes by Newton on P'_{q-1}, 2-norms by Householder
// tridiagonalisation + Sturm bisection).  The free parameters the paper leaves
// unspecified (r grid, trapezoid resolution, boundary sampling, q range) are
// the documented readings R3-R5 of DESIGN.md, shared as *numbers* with the
// oracle so both choose the same (s, q).
#include "planner.h"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

namespace phiks {
namespace plan {

using cd = std::complex<double>;

namespace {

constexpr int kQmin = 2, kQmax = 12, kSmax = 60;   // reading R5 (Table 1 never exceeds q = 12)
constexpr double kWcap = 256.0;                    // reading R5
constexpr int kNside = 32;                         // reading R4
constexpr int kNr = 16;                            // reading R3: r ∈ geomspace(0.3, 6, 16)
constexpr int kGL = 256;                           // Gauss–Legendre points for k_q
constexpr double kExpMax = 709.782712893384;       // exp overflow threshold (fp64)
const double kSpectral = 1.0 + std::sqrt(2.0);     // (1+√2)-spectral set [CP17], l.908

// Legendre P_N(x) and P_{N-1}(x) by the three-term recurrence.
void legendre(int N, double x, double& pN, double& pNm1) {
  double p0 = 1.0, p1 = x;
  if (N == 0) {
    pN = 1.0;
    pNm1 = 0.0;
    return;
  }
  for (int k = 1; k < N; ++k) {
    const double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
    p0 = p1;
    p1 = p2;
  }
  pN = p1;
  pNm1 = p0;
}

// Gauss–Legendre nodes/weights on [0,1] (Newton on P_m, Chebyshev start).
const std::vector<std::pair<double, double>>& gauss_legendre01() {
  static std::vector<std::pair<double, double>> gl;
  static std::once_flag once;
  std::call_once(once, [] {
    const int m = kGL;
    gl.resize(m);
    for (int i = 0; i < m; ++i) {
      double x = std::cos(M_PI * (i + 0.75) / (m + 0.5));
      double pN = 0, pNm1 = 0, dp = 1;
      for (int it = 0; it < 100; ++it) {
        legendre(m, x, pN, pNm1);
        dp = m * (x * pN - pNm1) / (x * x - 1.0);
        const double dx = pN / dp;
        x -= dx;
        if (std::fabs(dx) < 1e-17) break;
      }
      legendre(m, x, pN, pNm1);
      dp = m * (x * pN - pNm1) / (x * x - 1.0);
      const double w = 2.0 / ((1.0 - x * x) * dp * dp);
      gl[m - 1 - i] = {(x + 1.0) / 2.0, w / 2.0};
    }
  });
  return gl;
}

double r_grid(int i) {  // geomspace(0.3, 6, kNr)
  if (i == kNr - 1) return 6.0;
  return 0.3 * std::pow(6.0 / 0.3, static_cast<double>(i) / (kNr - 1));
}

int n_zeta(double r, double wmax) {
  const double need = 2.0 * (wmax * (r + 1.0 / (16.0 * r) + 0.5) + 64.0);
  int n = 128;
  while (n < need && n < 4096) n *= 2;
  return n;
}

// k_q on the nz trapezoid points of Γ_r, memoised.
const std::vector<cd>& kq_on_ellipse(int q, int ri, int nz) {
  static std::map<std::tuple<int, int, int>, std::vector<cd>> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(q, ri, nz);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  std::vector<double> th, w;
  gll_rule(q, th, w);
  const auto& gl = gauss_legendre01();
  std::vector<double> pit(gl.size());
  for (size_t g = 0; g < gl.size(); ++g) {
    double v = 1.0;
    for (double t : th) v *= (gl[g].first - t);
    pit[g] = v * gl[g].second;
  }
  const double r = r_grid(ri);
  std::vector<cd> out(nz);
  for (int m = 0; m < nz; ++m) {
    const double zeta = 2.0 * M_PI * m / nz;
    const cd e(std::cos(zeta), std::sin(zeta));
    const cd z = r * e + 0.5 + 1.0 / (16.0 * r * e);
    cd num = 0.0;
    for (size_t g = 0; g < gl.size(); ++g) num += pit[g] / (z - gl[g].first);
    cd piz = 1.0;
    for (double t : th) piz *= (z - t);
    out[m] = num / piz;
  }
  return cache.emplace(key, std::move(out)).first->second;
}

// ---- symmetric eigen-extremes: Householder tridiagonalisation + bisection ----
void tridiagonalize(int n, std::vector<double>& A, std::vector<double>& d, std::vector<double>& e) {
  // A: n×n symmetric, column-major, destroyed.
  d.assign(n, 0.0);
  e.assign(n > 0 ? n - 1 : 0, 0.0);
  std::vector<double> v(n), pv(n), wv(n);
  for (int k = 0; k + 2 < n; ++k) {
    double nrm2 = 0.0;
    for (int i = k + 1; i < n; ++i) nrm2 += A[i + k * n] * A[i + k * n];
    const double nrm = std::sqrt(nrm2);
    const double x0 = A[(k + 1) + k * n];
    if (nrm == 0.0) {
      e[k] = 0.0;
      continue;
    }
    const double alpha = (x0 > 0) ? -nrm : nrm;
    for (int i = k + 1; i < n; ++i) v[i] = A[i + k * n];
    v[k + 1] -= alpha;
    double vn2 = 0.0;
    for (int i = k + 1; i < n; ++i) vn2 += v[i] * v[i];
    if (vn2 == 0.0) {
      e[k] = x0;
      continue;
    }
    const double vn = std::sqrt(vn2);
    for (int i = k + 1; i < n; ++i) v[i] /= vn;
    // p = A v (trailing block)
    for (int i = k + 1; i < n; ++i) pv[i] = 0.0;
    for (int j = k + 1; j < n; ++j) {
      const double vj = v[j];
      const double* col = &A[j * n];
      for (int i = k + 1; i < n; ++i) pv[i] += col[i] * vj;
    }
    double vp = 0.0;
    for (int i = k + 1; i < n; ++i) vp += v[i] * pv[i];
    for (int i = k + 1; i < n; ++i) wv[i] = 2.0 * pv[i] - 2.0 * vp * v[i];
    for (int j = k + 1; j < n; ++j) {
      double* col = &A[j * n];
      const double vj = v[j], wj = wv[j];
      for (int i = k + 1; i < n; ++i) col[i] -= v[i] * wj + wv[i] * vj;
    }
    e[k] = alpha;
    // column k / row k now (alpha at k+1, zeros below) — not needed further
  }
  for (int i = 0; i < n; ++i) d[i] = A[i + i * n];
  if (n >= 2) e[n - 2] = A[(n - 1) + (n - 2) * n];
}

int sturm_count(const std::vector<double>& d, const std::vector<double>& e, double x) {
  int cnt = 0;
  double qv = 1.0;
  const int n = static_cast<int>(d.size());
  for (int i = 0; i < n; ++i) {
    const double e2 = (i > 0) ? e[i - 1] * e[i - 1] : 0.0;
    qv = d[i] - x - ((i > 0) ? e2 / qv : 0.0);
    if (qv == 0.0) qv = -DBL_MIN * 1e3;
    if (qv < 0) ++cnt;
  }
  return cnt;
}

// returns max |λ| of the symmetric matrix given by its tridiagonal form
double tridiag_abs_max(const std::vector<double>& d, const std::vector<double>& e) {
  const int n = static_cast<int>(d.size());
  if (n == 0) return 0.0;
  double lo = d[0], hi = d[0];
  for (int i = 0; i < n; ++i) {
    const double r = ((i > 0) ? std::fabs(e[i - 1]) : 0.0) + ((i + 1 < n) ? std::fabs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
  }
  const double span = std::max(std::fabs(lo), std::fabs(hi));
  if (span == 0.0) return 0.0;
  auto bisect = [&](int k) {  // k-th smallest eigenvalue (0-based)
    double a = lo - 1e-300, b = hi;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (a + b);
      if (mid <= a || mid >= b) break;
      if (sturm_count(d, e, mid) > k) b = mid; else a = mid;
      if (b - a <= 4.0 * DBL_EPSILON * span) break;
    }
    return 0.5 * (a + b);
  };
  const double lmin = bisect(0), lmax = bisect(n - 1);
  return std::max(std::fabs(lmin), std::fabs(lmax));
}

}  // namespace

void gll_rule(int q, std::vector<double>& theta, std::vector<double>& w) {
  theta.assign(q, 0.0);
  w.assign(q, 0.0);
  const int N = q - 1;
  std::vector<double> x(q);
  x[0] = -1.0;
  x[q - 1] = 1.0;
  for (int i = 1; i < q - 1; ++i) {
    // interior nodes: roots of P'_N; Newton from Chebyshev–Gauss–Lobatto points
    double xi = -std::cos(M_PI * i / N);
    for (int it = 0; it < 100; ++it) {
      double pN, pNm1;
      legendre(N, xi, pN, pNm1);
      const double dp = N * (xi * pN - pNm1) / (xi * xi - 1.0);
      const double d2p = (2.0 * xi * dp - N * (N + 1.0) * pN) / (1.0 - xi * xi);
      const double dx = dp / d2p;
      xi -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    x[i] = xi;
  }
  for (int i = 0; i < q; ++i) {
    double pN, pNm1;
    legendre(N, x[i], pN, pNm1);
    const double wi = 2.0 / (N * (N + 1.0) * pN * pN);
    theta[i] = (x[i] + 1.0) / 2.0;
    w[i] = wi / 2.0;
  }
  theta[0] = 0.0;
  theta[q - 1] = 1.0;
}

FactorRange factor_range(int n, const double* A) {
  FactorRange fr{};
  double tr = 0.0;
  for (int i = 0; i < n; ++i) tr += A[i + i * n];
  fr.sigma = tr / n;
  std::vector<double> H(static_cast<size_t>(n) * n), S(static_cast<size_t>(n) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double bij = A[i + j * n] - (i == j ? fr.sigma : 0.0);
      const double bji = A[j + i * n] - (i == j ? fr.sigma : 0.0);
      H[i + j * n] = 0.5 * (bij + bji);
      S[i + j * n] = 0.5 * (bij - bji);
    }
  std::vector<double> d, e;
  tridiagonalize(n, H, d, e);
  fr.hnorm = tridiag_abs_max(d, e);
  // ||S||_2^2 = λ_max(S^T S), S^T S symmetric PSD
  std::vector<double> G(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const double skj = S[k + j * n];
      if (skj == 0.0) continue;
      for (int i = 0; i < n; ++i) G[i + j * n] += S[k + i * n] * skj;  // (S^T S)_{ij} = Σ_k S_ki S_kj
    }
  tridiagonalize(n, G, d, e);
  fr.snorm = std::sqrt(std::max(0.0, tridiag_abs_max(d, e)));
  return fr;
}

FactorRange factor_range_complex(int n, const double* Az) {
  FactorRange fr{};
  double tr_re = 0.0, tr_im = 0.0;
  for (int i = 0; i < n; ++i) {
    tr_re += Az[2 * (i + static_cast<size_t>(i) * n)];
    tr_im += Az[2 * (i + static_cast<size_t>(i) * n) + 1];
  }
  fr.sigma = tr_re / n;
  fr.sigma_im = tr_im / n;
  // B = A − σI; H = (B + B^H)/2 (Hermitian), S = (B − B^H)/2 (skew-Hermitian).
  // A Hermitian X = Xr + iXi has the real symmetric form [[Xr, −Xi], [Xi, Xr]]
  // with the same eigenvalues (each twice); ‖S‖₂ = ‖iS‖₂, iS = −Si + i·Sr.
  const size_t m = 2 * static_cast<size_t>(n);
  std::vector<double> RH(m * m), RS(m * m);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) {
      const size_t jk = j + static_cast<size_t>(k) * n, kj = k + static_cast<size_t>(j) * n;
      double br = Az[2 * jk], bi = Az[2 * jk + 1];
      double cr = Az[2 * kj], ci = Az[2 * kj + 1];  // B_kj
      if (j == k) {
        br -= fr.sigma;
        bi -= fr.sigma_im;
        cr -= fr.sigma;
        ci -= fr.sigma_im;
      }
      const double hr = 0.5 * (br + cr), hi = 0.5 * (bi - ci);  // H_jk = (B_jk + conj(B_kj))/2
      const double sr = 0.5 * (br - cr), si = 0.5 * (bi + ci);  // S_jk = (B_jk − conj(B_kj))/2
      const double xr = -si, xi = sr;                           // (iS)_jk
      RH[j + k * m] = hr;
      RH[(j + n) + (k + n) * m] = hr;
      RH[(j + n) + k * m] = hi;
      RH[j + (k + n) * m] = -hi;
      RS[j + k * m] = xr;
      RS[(j + n) + (k + n) * m] = xr;
      RS[(j + n) + k * m] = xi;
      RS[j + (k + n) * m] = -xi;
    }
  std::vector<double> d, e;
  tridiagonalize(static_cast<int>(m), RH, d, e);
  fr.hnorm = tridiag_abs_max(d, e);
  tridiagonalize(static_cast<int>(m), RS, d, e);
  fr.snorm = tridiag_abs_max(d, e);
  return fr;
}

int tucker_count(int mode, int s, int s_hat, int q, int p) {
  return mode == kSame ? (q + s * p + s_hat) : (q * p + s * p + s_hat);
}

namespace {

// bounds B[li] (ℓ = li+1) for one q at the scaled rectangle; min over r.
// The radii are independent: evaluated in parallel (OpenMP), reduced in order.
void bounds_for_q(const Rect& rect, int q, int p, const std::vector<cd>& wpts, double wmax,
                  std::vector<double>& B, std::vector<std::vector<cd>>& Ecache,
                  std::vector<int>& Enz, std::vector<char>& Einf) {
  B.assign(p, INFINITY);
  const int nb = static_cast<int>(wpts.size());
  for (int ri = 0; ri < kNr; ++ri) kq_on_ellipse(q, ri, n_zeta(r_grid(ri), wmax));  // memoise serially
  std::vector<std::vector<double>> Br(kNr, std::vector<double>(p, INFINITY));
#pragma omp parallel for schedule(dynamic, 1)
  for (int ri = 0; ri < kNr; ++ri) {
    std::vector<double>& Bri = Br[ri];
    const double r = r_grid(ri);
    const int nz = n_zeta(r, wmax);
    // E[m*nb + b] = exp((1 - z_m) w_b), cached per r across q
    if (Enz[ri] != nz) {
      Enz[ri] = nz;
      Ecache[ri].assign(static_cast<size_t>(nz) * nb, cd(0, 0));
      Einf[ri] = 0;
      for (int m = 0; m < nz && !Einf[ri]; ++m) {
        const double zeta = 2.0 * M_PI * m / nz;
        const cd e(std::cos(zeta), std::sin(zeta));
        const cd z = r * e + 0.5 + 1.0 / (16.0 * r * e);
        for (int b = 0; b < nb; ++b) {
          const cd x = (1.0 - z) * wpts[b];
          if (x.real() > kExpMax) {
            Einf[ri] = 1;
            break;
          }
          Ecache[ri][static_cast<size_t>(m) * nb + b] = std::exp(x);
        }
      }
    }
    if (Einf[ri]) continue;
    const std::vector<cd>& kq = kq_on_ellipse(q, ri, nz);
    const std::vector<cd>& E = Ecache[ri];
    std::vector<cd> acc(static_cast<size_t>(p) * nb, cd(0, 0));
    for (int m = 0; m < nz; ++m) {
      const double zeta = 2.0 * M_PI * m / nz;
      const cd e(std::cos(zeta), std::sin(zeta));
      const cd z = r * e + 0.5 + 1.0 / (16.0 * r * e);
      const cd dz = r * e - 1.0 / (16.0 * r * e);
      cd g = kq[m] * dz;  // ℓ = 1 coefficient; ℓ+1: g *= z/ℓ
      const cd* Em = &E[static_cast<size_t>(m) * nb];
      for (int li = 0; li < p; ++li) {
        if (li > 0) g *= z / static_cast<double>(li);
        cd* a = &acc[static_cast<size_t>(li) * nb];
        for (int b = 0; b < nb; ++b) a[b] += g * Em[b];
      }
    }
    for (int li = 0; li < p; ++li) {
      double mx = 0.0;
      bool fin = true;
      for (int b = 0; b < nb; ++b) {
        const double v = std::abs(acc[static_cast<size_t>(li) * nb + b]);
        if (!std::isfinite(v)) {
          fin = false;
          break;
        }
        mx = std::max(mx, v);
      }
      const double val = fin ? mx * kSpectral / nz : INFINITY;
      if (std::isfinite(val)) Bri[li] = val;
    }
  }
  for (int ri = 0; ri < kNr; ++ri)
    for (int li = 0; li < p; ++li) B[li] = std::min(B[li], Br[ri][li]);
}

// B for (scaled rectangle, q, p), memoised: the bound depends on neither the
// vector norms nor the tolerance, so a new right-hand side (a new time step of
// an integrator) re-plans with comparisons only.
struct BoundCache {
  std::mutex mu;
  std::map<std::vector<uint64_t>, std::vector<double>> map;
};
BoundCache& bound_cache() {
  static BoundCache* c = new BoundCache();
  return *c;
}
std::vector<uint64_t> bound_key(const Rect& rc, int q, int p) {
  auto bits = [](double x) {
    uint64_t u;
    std::memcpy(&u, &x, sizeof(u));
    return u;
  };
  return {bits(rc.center.real()), bits(rc.center.imag()), bits(rc.hr), bits(rc.hi), static_cast<uint64_t>(q),
          static_cast<uint64_t>(p)};
}

std::vector<cd> boundary(const Rect& rc) {
  std::vector<cd> pts;
  const double a = rc.hr, b = rc.hi;
  const cd corners[4] = {cd(-a, -b), cd(a, -b), cd(a, b), cd(-a, b)};
  for (int k = 0; k < 4; ++k) {
    const cd p0 = corners[k], p1 = corners[(k + 1) % 4];
    for (int i = 0; i < kNside; ++i) {
      const double s = static_cast<double>(i) / kNside;
      pts.push_back(rc.center + p0 + s * (p1 - p0));
    }
  }
  return pts;
}

}  // namespace

int q_for_s(int mode, const Rect& rect, int p, const std::vector<double>& norms, double delta, int s) {
  const double f = std::ldexp(1.0, -s);
  const Rect rc{rect.center * f, rect.hr * f, rect.hi * f};
  const std::vector<cd> w = boundary(rc);
  double wmax = 0.0;
  for (const cd& x : w) wmax = std::max(wmax, std::abs(x));
  if (wmax > kWcap) return 0;
  std::vector<std::vector<cd>> Ecache(kNr);
  std::vector<int> Enz(kNr, -1);
  std::vector<char> Einf(kNr, 0);
  std::vector<double> B;
  for (int q = kQmin; q <= kQmax; ++q) {
    const std::vector<uint64_t> key = bound_key(rc, q, p);
    bool have = false;
    {
      BoundCache& bc = bound_cache();
      std::lock_guard<std::mutex> lk(bc.mu);
      auto it = bc.map.find(key);
      if (it != bc.map.end()) {
        B = it->second;
        have = true;
      }
    }
    if (!have) {
      bounds_for_q(rc, q, p, w, wmax, B, Ecache, Enz, Einf);
      BoundCache& bc = bound_cache();
      std::lock_guard<std::mutex> lk(bc.mu);
      bc.map[key] = B;
    }
    bool ok = true;
    for (int ell = 1; ell <= p && ok; ++ell) {
      if (mode == kSame) {
        ok = B[ell - 1] * norms[0] <= delta * std::ldexp(1.0, ell * s);
      } else {
        double acc = 0.0;
        for (int k = 1; k <= ell; ++k) acc = acc + B[ell - k] * norms[p - k] / std::ldexp(1.0, (ell - k + 1) * s);
        ok = acc <= delta;
      }
    }
    if (ok) return q;
  }
  return 0;
}

Plan select_plan(int mode, const Rect& rect, int p, const std::vector<double>& norms, double delta,
                 int s_hat, int s_min) {
  Plan out;
  if (s_min < 0) s_min = 0;
  if (p == 0) {
    out.s = s_min;
    out.q = 0;
    out.T = tucker_count(mode, s_min, s_hat, 0, 0);
    out.ok = true;
    return out;
  }
  Plan prev;
  for (int s = s_min; s <= kSmax; ++s) {
    const int q = q_for_s(mode, rect, p, norms, delta, s);
    if (q == 0) continue;
    Plan cur;
    cur.s = s;
    cur.q = q;
    cur.T = tucker_count(mode, s, s_hat, q, p);
    cur.ok = true;
    if (prev.ok && cur.T > prev.T) return prev;
    prev = cur;
  }
  return prev;  // ok == false if nothing admissible
}

}  // namespace plan
}  // namespace phiks
