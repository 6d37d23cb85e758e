// basis.cpp -- Gauss-Lobatto nodes, weights and the weak-form derivative matrix
// Dhat = -M^-1 D^T M (reading R2: the transposed weight ratio of
// SPEC S:35, which preserves free streams), computed in long double.
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
  std::vector<double> xi, w, Dhat;   // Dhat row-major (N+1)^2
  double lhp, lhm;                    // lhat_N(+1) = 1/w_N, lhat_0(-1) = 1/w_0
};

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
  // barycentric weights and D_ij = l_j'(x_i)
  std::vector<long double> lam(n, 1.0L), D(n * n, 0.0L);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      if (k != j) lam[j] /= (x[j] - x[k]);
  for (int i = 0; i < n; ++i) {
    long double s = 0.0L;
    for (int j = 0; j < n; ++j)
      if (i != j) { D[i * n + j] = (lam[j] / lam[i]) / (x[i] - x[j]); s += D[i * n + j]; }
    D[i * n + i] = -s;
  }
  Basis1D b;
  b.N = N;
  b.xi.resize(n); b.w.resize(n); b.Dhat.resize(n * n);
  for (int i = 0; i < n; ++i) { b.xi[i] = (double)x[i]; b.w[i] = (double)w[i]; }
  b.lhp = (double)(1.0L / w[N]);
  b.lhm = (double)(1.0L / w[0]);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) b.Dhat[i * n + j] = (double)(-(w[j] / w[i]) * D[j * n + i]);
    // enforce the free-stream row identity  sum_l Dhat_il = -lhat_i(1) + lhat_i(-1)
    long double target = (i == N ? -(long double)b.lhp : 0.0L) + (i == 0 ? (long double)b.lhm : 0.0L);
    long double off = 0.0L;
    for (int j = 0; j < n; ++j) if (j != i) off += b.Dhat[i * n + j];
    b.Dhat[i * n + i] = (double)(target - off);
  }
  return b;
}

}  // namespace hbpdc
