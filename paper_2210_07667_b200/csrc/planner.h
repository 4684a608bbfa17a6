// Host-side choice of the scaling s and the number q of Gauss–Lobatto–Legendre
// nodes (§3.3, l.779-960).  Pure C++, no device work.
#pragma once

#include <complex>
#include <vector>

namespace phiks {
namespace plan {

// q-point GLL rule on [0,1]: nodes 0 = θ_1 < … < θ_q = 1 and weights.
void gll_rule(int q, std::vector<double>& theta, std::vector<double>& w);

// Per-factor numerical-range data of a real n×n column-major matrix A
// (reading R1): σ = trace(A)/n, ||H||_2 and ||S||_2 of the Hermitian and
// skew-Hermitian parts of A − σI.
struct FactorRange {
  double sigma;   // trace shift tr(A)/n (real part)
  double hnorm;   // ||(B + B^H)/2||_2
  double snorm;   // ||(B − B^H)/2||_2
  double sigma_im = 0.0;  // imaginary part of the trace shift (complex A)
};
FactorRange factor_range(int n, const double* A);
// complex A (interleaved re, im, column-major): ‖H‖₂ and ‖S‖₂ through the real
// symmetric 2n×2n forms of the Hermitian matrices H and iS
FactorRange factor_range_complex(int n, const double* Az);

// Ξ = center + [−hr, hr] + i[−hi, hi]
struct Rect {
  std::complex<double> center;
  double hr, hi;
};

struct Plan {
  int s = 0, q = 0, T = 0;
  bool ok = false;
};

enum Mode { kSame = 0, kLincomb = 1 };

int tucker_count(int mode, int s, int s_hat, int q, int p);

// §3.3 search.  norms[k-1] = ||v_k|| (lincomb) or norms[0] = ||v|| (same).
Plan select_plan(int mode, const Rect& rect, int p, const std::vector<double>& norms, double delta,
                 int s_hat, int s_min);

// Exposed for tests: smallest admissible q at a given s (0 if none).
int q_for_s(int mode, const Rect& rect, int p, const std::vector<double>& norms, double delta, int s);

}  // namespace plan
}  // namespace phiks
