// basis.cpp -- Gauss-Lobatto (configs) and Gauss-Legendre (NEXT-3) nodes,
// weights and the weak-form derivative matrix Dhat = -M^-1 D^T M (
// reading R2: the transposed weight ratio of SPEC S:35, which preserves free
// streams), the edge values l_i(+-1) and lhat_i(+-1) = l_i(+-1) / w_i,
// computed in long double.
#include <cmath>
#include <vector>

namespace hbpdc {

// P_N(x), P_N'(x), P_N''(x) by recurrence (long double)
static void legendre(int N, long double x, long double& p, long double& dp, long double& ddp) {
  long double p0 = 1.0L, p1 = x;
  if (N == 0) { p = 1.0L; dp = 0.0L; ddp = 0.0L; return; }
  long double d0 = 0.0L, d1 = 1.0L;                 // derivatives
  for (int k = 2; k <= N; ++k) {
    long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    long double d2 = d0 + (2 * k - 1) * p1;           // P_k' = P_{k-2}' + (2k-1) P_{k-1}
    p0 = p1; p1 = p2; d0 = d1; d1 = d2;
  }
  p = p1; dp = d1;
  // Legendre ODE: (1-x^2) P'' - 2x P' + N(N+1) P = 0
  ddp = (1.0L - x * x) != 0.0L ? (2.0L * x * dp - N * (N + 1) * p) / (1.0L - x * x) : 0.0L;
}

struct Basis1D {
  int N;
  int gl;                             // 0: Gauss-Lobatto, 1: Gauss-Legendre
  std::vector<double> xi, w, Dhat;   // Dhat row-major (N+1)^2
  double lhp, lhm;                    // GLL: lhat_N(+1) = 1/w_N, lhat_0(-1) = 1/w_0
  std::vector<double> lp, lm;         // l_i(+1), l_i(-1)
  std::vector<double> lhpv, lhmv;     // lhat_i(+1), lhat_i(-1)
  std::vector<double> D;              // D_ij = l_j'(x_i), row-major
  std::vector<double> dlp, dlm;       // l_j'(+1), l_j'(-1)  (edge derivatives, BR2 on GL)
};

// barycentric weights, D_ij = l_j'(x_i), edge values and Dhat of a node set
static void finish_basis(Basis1D& b, const std::vector<long double>& x, const std::vector<long double>& w) {
  const int n = (int)x.size(), N = n - 1;
  std::vector<long double> lam(n, 1.0L), D(n * n, 0.0L), lp(n), lm(n);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      if (k != j) lam[j] /= (x[j] - x[k]);
  for (int i = 0; i < n; ++i) {
    long double s = 0.0L;
    for (int j = 0; j < n; ++j)
      if (i != j) { D[i * n + j] = (lam[j] / lam[i]) / (x[i] - x[j]); s += D[i * n + j]; }
    D[i * n + i] = -s;
  }
  for (int j = 0; j < n; ++j) {                       // l_j(+-1) = prod_{k != j} (+-1 - x_k) / (x_j - x_k)
    long double a = 1.0L, c = 1.0L;
    for (int k = 0; k < n; ++k)
      if (k != j) { a *= (1.0L - x[k]) / (x[j] - x[k]); c *= (-1.0L - x[k]) / (x[j] - x[k]); }
    lp[j] = a; lm[j] = c;
  }
  b.N = N;
  b.xi.resize(n); b.w.resize(n); b.Dhat.resize(n * n);
  b.lp.resize(n); b.lm.resize(n); b.lhpv.resize(n); b.lhmv.resize(n);
  for (int i = 0; i < n; ++i) {
    b.xi[i] = (double)x[i]; b.w[i] = (double)w[i];
    b.lp[i] = (double)lp[i]; b.lm[i] = (double)lm[i];
    b.lhpv[i] = (double)(lp[i] / w[i]); b.lhmv[i] = (double)(lm[i] / w[i]);
  }
  b.D.resize(n * n); b.dlp.resize(n); b.dlm.resize(n);
  for (int i = 0; i < n * n; ++i) b.D[i] = (double)D[i];
  for (int j = 0; j < n; ++j) {                       // l_j'(+-1) = sum_i l_i(+-1) D_ij (exact for degree N)
    long double a = 0.0L, c = 0.0L;
    for (int i = 0; i < n; ++i) { a += lp[i] * D[i * n + j]; c += lm[i] * D[i * n + j]; }
    b.dlp[j] = (double)a; b.dlm[j] = (double)c;
  }
  b.lhp = (double)(1.0L / w[N]);
  b.lhm = (double)(1.0L / w[0]);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) b.Dhat[i * n + j] = (double)(-(w[j] / w[i]) * D[j * n + i]);
    // enforce the free-stream row identity  sum_l Dhat_il = -lhat_i(1) + lhat_i(-1)
    long double target = -(long double)b.lhpv[i] + (long double)b.lhmv[i];
    long double off = 0.0L;
    for (int j = 0; j < n; ++j) if (j != i) off += b.Dhat[i * n + j];
    b.Dhat[i * n + i] = (double)(target - off);
  }
}

// Gauss-Legendre: roots of P_{N+1}, w_i = 2 / ((1 - x_i^2) P_{N+1}'(x_i)^2)
Basis1D gl_basis(int N) {
  const int n = N + 1;
  const long double PI = 3.141592653589793238462643383279502884L;
  std::vector<long double> x(n), w(n);
  for (int k = 0; k < n; ++k) {
    long double t = -cosl(PI * (k + 0.75L) / (n + 0.5L));
    for (int it = 0; it < 100; ++it) {
      long double p, dp, ddp;
      legendre(n, t, p, dp, ddp);
      long double dt = p / dp;
      t -= dt;
      if (fabsl(dt) < 1e-19L) break;
    }
    x[k] = t;
  }
  for (int i = 0; i < n; ++i) {
    long double p, dp, ddp;
    legendre(n, x[i], p, dp, ddp);
    w[i] = 2.0L / ((1.0L - x[i] * x[i]) * dp * dp);
  }
  Basis1D b;
  b.gl = 1;
  finish_basis(b, x, w);
  return b;
}

Basis1D gll_basis(int N) {
  const int n = N + 1;
  const long double PI = 3.141592653589793238462643383279502884L;
  std::vector<long double> x(n), w(n);
  x[0] = -1.0L; x[N] = 1.0L;
  for (int k = 1; k < N; ++k) {                       // interior: roots of P_N'
    long double t = -cosl(PI * k / N);
    for (int it = 0; it < 100; ++it) {
      long double p, dp, ddp;
      legendre(N, t, p, dp, ddp);
      long double dt = dp / ddp;
      t -= dt;
      if (fabsl(dt) < 1e-19L) break;
    }
    x[k] = t;
  }
  for (int i = 0; i < n; ++i) {
    long double p, dp, ddp;
    legendre(N, x[i], p, dp, ddp);
    w[i] = 2.0L / (N * (N + 1) * p * p);
  }
  Basis1D b;
  b.gl = 0;
  finish_basis(b, x, w);
  return b;
}

}  // namespace hbpdc
