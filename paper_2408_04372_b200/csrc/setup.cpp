// Host-side discretisation primitives (see setup.hpp for the reference map).
#include "setup.hpp"

#include <algorithm>
#include <cmath>

namespace stmgb {

namespace {

// Legendre P_n(x) and P_n'(x) on [-1,1] by the three-term recurrence
void legendre(int n, double x, double& p, double& dp) {
  double p0 = 1.0, p1 = x;
  if (n == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  for (int j = 2; j <= n; ++j) {
    const double p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / j;
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  dp = n * (x * p1 - p0) / (x * x - 1.0);
}

template <typename F>
double newton(F&& f, double x) {
  for (int it = 0; it < 100; ++it) {
    double v, d;
    f(x, v, d);
    const double dx = v / d;
    x -= dx;
    if (std::abs(dx) < 1e-17) break;
  }
  return x;
}

Rule to_unit(std::vector<double> x, std::vector<double> w) {
  std::vector<int> idx(x.size());
  for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int>(i);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return x[a] < x[b]; });
  Rule r;
  for (int i : idx) {
    r.x.push_back(0.5 * (x[i] + 1.0));
    r.w.push_back(0.5 * w[i]);
  }
  return r;
}

}  // namespace

Rule gauss(int n) {
  if (n < 1) throw std::invalid_argument("gauss: n must be >= 1");
  if (n == 1) return {{0.5}, {1.0}};
  std::vector<double> x(n), w(n);
  for (int i = 0; i < n; ++i) {
    double xi = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    xi = newton([n](double t, double& v, double& d) { legendre(n, t, v, d); }, xi);
    double p, dp;
    legendre(n, xi, p, dp);
    x[i] = xi;
    w[i] = 2.0 / ((1.0 - xi * xi) * dp * dp);
  }
  return to_unit(x, w);
}

Rule gauss_lobatto(int n) {
  if (n < 2) throw std::invalid_argument("gauss_lobatto: n must be >= 2");
  const int m = n - 1;  // interior nodes are the roots of P_m'
  std::vector<double> x{-1.0, 1.0};
  for (int i = 1; i <= n - 2; ++i) {
    double xi = -std::cos(M_PI * i / m);
    xi = newton(
        [m](double t, double& v, double& d) {
          double p, dp;
          legendre(m, t, p, dp);
          v = dp;
          d = (2.0 * t * dp - m * (m + 1.0) * p) / (1.0 - t * t);
        },
        xi);
    x.push_back(xi);
  }
  std::vector<double> w;
  for (double xi : x) {
    double p, dp;
    if (std::abs(xi) == 1.0)
      p = (xi > 0 || m % 2 == 0) ? 1.0 : -1.0;
    else
      legendre(m, xi, p, dp);
    w.push_back(2.0 / (n * (n - 1.0) * p * p));
  }
  Rule r = to_unit(x, w);
  r.x.front() = 0.0;
  r.x.back() = 1.0;
  return r;
}

Rule gauss_radau_right(int n) {
  if (n < 1) throw std::invalid_argument("gauss_radau_right: n must be >= 1");
  if (n == 1) return {{1.0}, {1.0}};
  // left-sided rule: node -1 plus the roots of P_{n-1} + P_n; then reflect
  std::vector<double> x{-1.0}, w{2.0 / (static_cast<double>(n) * n)};
  for (int i = 1; i < n; ++i) {
    double xi = -std::cos(2.0 * M_PI * i / (2.0 * n - 1.0));
    xi = newton(
        [n](double t, double& v, double& d) {
          double pa, da, pb, db;
          legendre(n - 1, t, pa, da);
          legendre(n, t, pb, db);
          v = pa + pb;
          d = da + db;
        },
        xi);
    double p, dp;
    legendre(n - 1, xi, p, dp);
    x.push_back(xi);
    w.push_back((1.0 - xi) / (static_cast<double>(n) * n * p * p));
  }
  for (double& xi : x) xi = -xi;
  Rule r = to_unit(x, w);
  r.x.back() = 1.0;
  return r;
}

double lagrange_eval(const std::vector<double>& nodes, int i, double t) {
  double v = 1.0;
  for (std::size_t j = 0; j < nodes.size(); ++j)
    if (static_cast<int>(j) != i) v *= (t - nodes[j]) / (nodes[i] - nodes[j]);
  return v;
}

double lagrange_deriv(const std::vector<double>& nodes, int i, double t) {
  double sum = 0.0;
  const int n = static_cast<int>(nodes.size());
  for (int m = 0; m < n; ++m) {
    if (m == i) continue;
    double term = 1.0 / (nodes[i] - nodes[m]);
    for (int j = 0; j < n; ++j)
      if (j != i && j != m) term *= (t - nodes[j]) / (nodes[i] - nodes[j]);
    sum += term;
  }
  return sum;
}

double TemporalWeights::unknown_weight(int i, double t) const {
  return lagrange_eval(trial_nodes, scheme == TimeScheme::DG ? i : i + 1, t);
}
double TemporalWeights::left_weight(double t) const {
  return scheme == TimeScheme::DG ? 0.0 : lagrange_eval(trial_nodes, 0, t);
}

TemporalWeights dg_weights(int k) {
  if (k < 0) throw std::invalid_argument("dg_weights: k must be >= 0");
  TemporalWeights w;
  w.scheme = TimeScheme::DG;
  w.k = k;
  w.n_t = k + 1;
  w.trial_nodes = gauss_radau_right(k + 1).x;
  w.unknown_nodes = w.trial_nodes;
  const Rule q = gauss(k + 1);
  const int n = k + 1;
  w.m.assign(n * n, 0.0);
  w.a.assign(n * n, 0.0);
  w.alpha.assign(n, 0.0);
  w.beta.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      double m = 0.0, a = 0.0;
      for (std::size_t p = 0; p < q.x.size(); ++p) {
        m += q.w[p] * lagrange_eval(w.trial_nodes, j, q.x[p]) * lagrange_eval(w.trial_nodes, i, q.x[p]);
        a += q.w[p] * lagrange_deriv(w.trial_nodes, j, q.x[p]) * lagrange_eval(w.trial_nodes, i, q.x[p]);
      }
      a += lagrange_eval(w.trial_nodes, j, 0.0) * lagrange_eval(w.trial_nodes, i, 0.0);  // upwind jump
      w.m[i * n + j] = m;
      w.a[i * n + j] = a;
    }
    w.alpha[i] = lagrange_eval(w.trial_nodes, i, 0.0);
  }
  return w;
}

TemporalWeights cgp_weights(int k) {
  if (k < 1) throw std::invalid_argument("cgp_weights: k must be >= 1");
  TemporalWeights w;
  w.scheme = TimeScheme::CGP;
  w.k = k;
  w.n_t = k;
  w.trial_nodes = gauss_lobatto(k + 1).x;
  w.unknown_nodes.assign(w.trial_nodes.begin() + 1, w.trial_nodes.end());
  const std::vector<double> test(w.trial_nodes.begin() + 1, w.trial_nodes.end());
  const Rule q = gauss(k + 1);
  w.m.assign(k * k, 0.0);
  w.a.assign(k * k, 0.0);
  w.alpha.assign(k, 0.0);
  w.beta.assign(k, 0.0);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j <= k; ++j) {
      double m = 0.0, a = 0.0;
      for (std::size_t p = 0; p < q.x.size(); ++p) {
        m += q.w[p] * lagrange_eval(w.trial_nodes, j, q.x[p]) * lagrange_eval(test, i, q.x[p]);
        a += q.w[p] * lagrange_deriv(w.trial_nodes, j, q.x[p]) * lagrange_eval(test, i, q.x[p]);
      }
      if (j == 0) {
        w.beta[i] = m;
        w.alpha[i] = a;
      } else {
        w.m[i * k + j - 1] = m;
        w.a[i * k + j - 1] = a;
      }
    }
  return w;
}

std::vector<double> invert_small(const std::vector<double>& a_in, int n) {
  std::vector<double> a = a_in, inv(n * n, 0.0);
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::abs(a[r * n + c]) > std::abs(a[piv * n + c])) piv = r;
    if (a[piv * n + c] == 0.0) throw std::runtime_error("invert_small: singular matrix");
    for (int j = 0; j < n; ++j) {
      std::swap(a[c * n + j], a[piv * n + j]);
      std::swap(inv[c * n + j], inv[piv * n + j]);
    }
    const double d = a[c * n + c];
    for (int j = 0; j < n; ++j) {
      a[c * n + j] /= d;
      inv[c * n + j] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = a[r * n + c];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        a[r * n + j] -= f * a[c * n + j];
        inv[r * n + j] -= f * inv[c * n + j];
      }
    }
  }
  return inv;
}

std::vector<double> matmul_small(const std::vector<double>& a, const std::vector<double>& b, int n, int k, int m) {
  std::vector<double> c(n * m, 0.0);
  for (int i = 0; i < n; ++i)
    for (int l = 0; l < k; ++l)
      for (int j = 0; j < m; ++j) c[i * m + j] += a[i * k + l] * b[l * m + j];
  return c;
}

void block_coefficient_matrices(Equation eq, const TemporalWeights& w, double tau, int S, std::vector<double>& CM,
                                std::vector<double>& CA) {
  const int nt = w.n_t;
  const int F = S * nt;
  CM.assign(F * F, 0.0);
  CA.assign(F * F, 0.0);
  const bool cgp = w.scheme == TimeScheme::CGP;
  auto at = [F, nt](std::vector<double>& X, int s, int i, int j, int l) -> double& {
    return X[(s * nt + i) * F + (j * nt + l)];
  };
  const int last = nt - 1;
  if (eq == Equation::Heat) {
    for (int s = 0; s < S; ++s) {
      for (int i = 0; i < nt; ++i)
        for (int l = 0; l < nt; ++l) {
          at(CA, s, i, s, l) = tau * w.m[i * nt + l];
          at(CM, s, i, s, l) = w.a[i * nt + l];
        }
      if (s > 0)
        for (int i = 0; i < nt; ++i) {
          if (cgp) {
            at(CM, s, i, s - 1, last) = w.alpha[i];
            at(CA, s, i, s - 1, last) = tau * w.beta[i];
          } else {
            at(CM, s, i, s - 1, last) = -w.alpha[i];
          }
        }
    }
    return;
  }
  // wave, condensed displacement form: velocity eliminated block-locally
  const std::vector<double> minv = invert_small(w.m, nt);
  const std::vector<double> ama = matmul_small(matmul_small(w.a, minv, nt, nt, nt), w.a, nt, nt, nt);
  const std::vector<double> minv_a = matmul_small(minv, w.a, nt, nt, nt);
  const std::vector<double> minv_alpha = matmul_small(minv, w.alpha, nt, nt, 1);
  const std::vector<double> am_alpha = matmul_small(w.a, minv_alpha, nt, nt, 1);
  std::vector<double> alpha_a(nt, 0.0);
  double minv_beta_last = 0.0;
  if (cgp) {
    const std::vector<double> minv_beta = matmul_small(minv, w.beta, nt, nt, 1);
    const std::vector<double> a_minv_beta = matmul_small(w.a, minv_beta, nt, nt, 1);
    minv_beta_last = minv_beta[last];
    for (int i = 0; i < nt; ++i) alpha_a[i] = w.alpha[i] - a_minv_beta[i];
  }
  const double minv_alpha_last = minv_alpha[last];
  const double g = -minv_beta_last;
  const double z = minv_alpha_last / tau;
  for (int s = 0; s < S; ++s)
    for (int j = 0; j <= s; ++j)
      for (int i = 0; i < nt; ++i)
        for (int l = 0; l < nt; ++l) {
          double cm = 0.0, ca = 0.0;
          if (j == s) {
            ca = tau * w.m[i * nt + l];
            cm = ama[i * nt + l] / tau;
          } else if (!cgp) {
            if (j == s - 1)
              cm = -((l == last ? am_alpha[i] : 0.0) + w.alpha[i] * minv_a[last * nt + l]) / tau;
            else if (j == s - 2)
              cm = (l == last) ? minv_alpha_last / tau * w.alpha[i] : 0.0;
          } else {
            if (j == s - 1 && l == last) {
              cm += am_alpha[i] / tau;
              ca += tau * w.beta[i];
            }
            cm += std::pow(g, s - 1 - j) / tau * alpha_a[i] * minv_a[last * nt + l];
            if (j <= s - 2 && l == last) cm += std::pow(g, s - 2 - j) * z * alpha_a[i];
          }
          at(CM, s, i, j, l) = cm;
          at(CA, s, i, j, l) = ca;
        }
}

double cartesian_coord(const MeshLevel& m, int axis, Index i) {
  return m.lo[axis] + (m.hi[axis] - m.lo[axis]) * static_cast<double>(i) / static_cast<double>(m.cells[axis]);
}

namespace {
// corner positions of a cell (lexicographic corners, x fastest)
void cell_corners(const MeshLevel& m, Index cell, double X[8][3]) {
  const Index cx = cell % m.cells[0], cy = (cell / m.cells[0]) % m.cells[1], cz = cell / (m.cells[0] * m.cells[1]);
  const auto nv = m.n_verts_axis();
  const int corners = 1 << m.dim;
  for (int s = 0; s < corners; ++s) {
    const Index i = cx + (s & 1), j = cy + ((s >> 1) & 1), k = cz + ((s >> 2) & 1);
    for (int a = 0; a < 3; ++a) X[s][a] = 0.0;
    if (!m.vertices.empty()) {
      const Index v = (k * nv[1] + j) * nv[0] + i;
      for (int a = 0; a < m.dim; ++a) X[s][a] = m.vertices[static_cast<size_t>(3 * v + a)];
    } else {
      const Index idx[3] = {i, j, k};
      for (int a = 0; a < m.dim; ++a) X[s][a] = cartesian_coord(m, a, idx[a]);
    }
  }
}
}  // namespace

void locate_point(const MeshLevel& m, const double x[3], Index& cell_out, double xi_out[3]) {
  const int dim = m.dim, corners = 1 << dim;
  const double tol = 1e-10;
  for (Index cell = 0; cell < m.n_cells(); ++cell) {
    double X[8][3];
    cell_corners(m, cell, X);
    bool reject = false;
    for (int a = 0; a < dim && !reject; ++a) {
      double lo = X[0][a], hi = X[0][a];
      for (int s = 0; s < corners; ++s) {
        lo = std::min(lo, X[s][a]);
        hi = std::max(hi, X[s][a]);
      }
      const double pad = 0.25 * (hi - lo) + tol;
      if (x[a] < lo - pad || x[a] > hi + pad) reject = true;
    }
    if (reject) continue;
    double xi[3] = {0.5, 0.5, 0.5};
    bool converged = false;
    for (int it = 0; it < 50; ++it) {
      double g[3] = {0.0, 0.0, 0.0}, J[3][3] = {{0.0}};
      for (int s = 0; s < corners; ++s) {
        double w = 1.0;
        double dw[3];
        for (int a = 0; a < dim; ++a) w *= ((s >> a) & 1) ? xi[a] : 1.0 - xi[a];
        for (int bb = 0; bb < dim; ++bb) {
          double d = 1.0;
          for (int a = 0; a < dim; ++a)
            d *= a == bb ? (((s >> a) & 1) ? 1.0 : -1.0) : (((s >> a) & 1) ? xi[a] : 1.0 - xi[a]);
          dw[bb] = d;
        }
        for (int a = 0; a < dim; ++a) {
          g[a] += w * X[s][a];
          for (int bb = 0; bb < dim; ++bb) J[a][bb] += dw[bb] * X[s][a];
        }
      }
      double r[3], nr = 0.0;
      for (int a = 0; a < dim; ++a) {
        r[a] = g[a] - x[a];
        nr += r[a] * r[a];
      }
      if (std::sqrt(nr) < 1e-13) {
        converged = true;
        break;
      }
      // dxi = J^-1 r (Gaussian elimination with partial pivoting, dim <= 3)
      double A[3][4];
      for (int i = 0; i < dim; ++i) {
        for (int j = 0; j < dim; ++j) A[i][j] = J[i][j];
        A[i][dim] = r[i];
      }
      bool singular = false;
      for (int k = 0; k < dim; ++k) {
        int piv = k;
        for (int i = k + 1; i < dim; ++i)
          if (std::abs(A[i][k]) > std::abs(A[piv][k])) piv = i;
        if (A[piv][k] == 0.0) {
          singular = true;
          break;
        }
        for (int j = 0; j <= dim; ++j) std::swap(A[k][j], A[piv][j]);
        for (int i = k + 1; i < dim; ++i) {
          const double f = A[i][k] / A[k][k];
          for (int j = k; j <= dim; ++j) A[i][j] -= f * A[k][j];
        }
      }
      if (singular) break;
      double dxi[3] = {0.0, 0.0, 0.0};
      for (int i = dim - 1; i >= 0; --i) {
        double sum = A[i][dim];
        for (int j = i + 1; j < dim; ++j) sum -= A[i][j] * dxi[j];
        dxi[i] = sum / A[i][i];
      }
      for (int a = 0; a < dim; ++a) xi[a] -= dxi[a];
    }
    if (!converged) continue;
    bool inside = true;
    for (int a = 0; a < dim; ++a) {
      if (xi[a] < -tol || xi[a] > 1.0 + tol) inside = false;
      xi[a] = std::min(1.0, std::max(0.0, xi[a]));
    }
    if (inside) {
      cell_out = cell;
      for (int a = 0; a < 3; ++a) xi_out[a] = a < dim ? xi[a] : 0.0;
      return;
    }
  }
  throw std::runtime_error("locate_point: point outside mesh");
}

MeshHierarchy make_cartesian(int dim, std::array<double, 3> lo, std::array<double, 3> hi, Index base_cells,
                             int refinements) {
  return make_cartesian_box(dim, lo, hi, {base_cells, base_cells, base_cells}, refinements);
}

MeshHierarchy make_cartesian_box(int dim, std::array<double, 3> lo, std::array<double, 3> hi,
                                 std::array<Index, 3> base_cells, int refinements) {
  if (dim < 1 || dim > 3) throw std::invalid_argument("make_cartesian: dim must be 1, 2 or 3");
  if (refinements < 0) throw std::invalid_argument("make_cartesian: invalid sizes");
  for (int a = 0; a < dim; ++a)
    if (base_cells[a] < 1) throw std::invalid_argument("make_cartesian: invalid sizes");
  MeshHierarchy h;
  for (int l = 0; l <= refinements; ++l) {
    MeshLevel m;
    m.dim = dim;
    m.lo = lo;
    m.hi = hi;
    for (int a = 0; a < dim; ++a) m.cells[a] = base_cells[a] << l;
    h.levels.push_back(m);
  }
  return h;
}

void set_finest_vertices(MeshHierarchy& mesh, const double* xyz) {
  MeshLevel& fine = mesh.levels.back();
  fine.vertices.assign(xyz, xyz + 3 * fine.n_verts());
  const int fl = mesh.n_levels() - 1;
  const auto nf = fine.n_verts_axis();
  for (int l = 0; l < fl; ++l) {
    MeshLevel& m = mesh.levels[l];
    const Index stride = Index{1} << (fl - l);
    const auto nc = m.n_verts_axis();
    m.vertices.assign(3 * m.n_verts(), 0.0);
    for (Index kk = 0; kk < nc[2]; ++kk)
      for (Index j = 0; j < nc[1]; ++j)
        for (Index i = 0; i < nc[0]; ++i) {
          const Index src = ((m.dim > 2 ? kk * stride : 0) * nf[1] + (m.dim > 1 ? j * stride : 0)) * nf[0] + i * stride;
          const Index dst = (kk * nc[1] + j) * nc[0] + i;
          for (int a = 0; a < 3; ++a) m.vertices[3 * dst + a] = fine.vertices[3 * src + a];
        }
  }
}

std::vector<Coarsening> default_strategy(const LevelSpec& finest, TimeScheme scheme) {
  const int k_min = scheme == TimeScheme::DG ? 0 : 1;
  std::vector<Coarsening> s;
  for (int m = finest.mesh_level; m > 0; --m) s.push_back(Coarsening::SpaceH);
  for (int n = finest.n_steps; n > 1; n /= 2) s.push_back(Coarsening::TimeTau);
  for (int k = finest.k; k > k_min; --k) s.push_back(Coarsening::TimeK);
  return s;
}

std::vector<LevelSpec> build_level_plan(const LevelSpec& finest, TimeScheme scheme,
                                        const std::vector<Coarsening>& strategy) {
  const int k_min = scheme == TimeScheme::DG ? 0 : 1;
  auto valid = [k_min](const LevelSpec& c) { return c.mesh_level >= 0 && c.p >= 1 && c.k >= k_min && c.n_steps >= 1; };
  LevelSpec cur = finest;
  if (!valid(cur)) throw std::invalid_argument("build_level_plan: invalid finest level");
  std::vector<LevelSpec> plan{cur};
  for (Coarsening c : strategy) {
    switch (c) {
      case Coarsening::SpaceH: cur.mesh_level -= 1; break;
      case Coarsening::SpaceP:
        if (cur.p == 1) throw std::invalid_argument("build_level_plan: p already 1");
        cur.p = std::max(1, cur.p / 2);
        break;
      case Coarsening::TimeTau:
        if (cur.n_steps % 2 != 0) throw std::invalid_argument("build_level_plan: odd n_steps");
        cur.n_steps /= 2;
        cur.tau *= 2.0;
        break;
      case Coarsening::TimeK: cur.k -= 1; break;
    }
    if (!valid(cur)) throw std::invalid_argument("build_level_plan: invalid coarsening step");
    cur.from_finer = c;
    plan.push_back(cur);
  }
  return plan;
}

Xoshiro256pp::Xoshiro256pp(std::uint64_t seed) {
  std::uint64_t x = seed;
  for (auto& s : s_) {
    x += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    s = z ^ (z >> 31);
  }
}
std::uint64_t Xoshiro256pp::next() {
  auto rotl = [](std::uint64_t v, int k) { return (v << k) | (v >> (64 - k)); };
  const std::uint64_t result = rotl(s_[0] + s_[3], 23) + s_[0];
  const std::uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl(s_[3], 45);
  return result;
}
double Xoshiro256pp::uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
double Xoshiro256pp::normal() {
  if (have_cached_) {
    have_cached_ = false;
    return cached_;
  }
  double u1 = 0.0;
  while (u1 <= 1e-300) u1 = uniform();
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double th = 2.0 * M_PI * u2;
  cached_ = r * std::sin(th);
  have_cached_ = true;
  return r * std::cos(th);
}

}  // namespace stmgb

namespace stmgb {

std::vector<double> sym_eigen_jacobi(std::vector<double> A, int n, std::vector<double>& V) {
  V.assign(static_cast<size_t>(n * n), 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += A[i * n + j] * A[i * n + j];
    if (off < 1e-34) break;
    for (int pp = 0; pp < n; ++pp)
      for (int q = pp + 1; q < n; ++q) {
        const double apq = A[pp * n + q];
        if (std::abs(apq) < 1e-300) continue;
        const double theta = (A[q * n + q] - A[pp * n + pp]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k * n + pp], akq = A[k * n + q];
          A[k * n + pp] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[pp * n + k], aqk = A[q * n + k];
          A[pp * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[k * n + pp], vkq = V[k * n + q];
          V[k * n + pp] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  std::vector<double> w(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) w[i] = A[i * n + i];
  return w;
}

void fdm_axis_tables(int p, double h, double S[4][5][5], double lam[4][5]) {
  const int n = p + 1;
  const Rule q = gauss(n);
  const std::vector<double> gl = gauss_lobatto(n).x;
  std::vector<double> Me(n * n, 0.0), Ke(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (size_t k = 0; k < q.x.size(); ++k) {
        Me[i * n + j] += q.w[k] * lagrange_eval(gl, i, q.x[k]) * lagrange_eval(gl, j, q.x[k]) * h;
        Ke[i * n + j] += q.w[k] * lagrange_deriv(gl, i, q.x[k]) * lagrange_deriv(gl, j, q.x[k]) / h;
      }
  for (int type = 0; type < 4; ++type) {
    const bool first = type & 1, last = type & 2;
    std::vector<double> M = Me, K = Ke;
    if (!first) {  // left neighbour shares node 0
      M[0] += Me[(n - 1) * n + (n - 1)];
      K[0] += Ke[(n - 1) * n + (n - 1)];
    }
    if (!last) {  // right neighbour shares node p
      M[(n - 1) * n + (n - 1)] += Me[0];
      K[(n - 1) * n + (n - 1)] += Ke[0];
    }
    std::vector<int> keep;
    for (int i = 0; i < n; ++i)
      if (!((i == 0 && first) || (i == n - 1 && last))) keep.push_back(i);
    const int k = static_cast<int>(keep.size());
    for (int i = 0; i < 5; ++i) {
      lam[type][i] = 0.0;
      for (int j = 0; j < 5; ++j) S[type][i][j] = 0.0;
    }
    if (k == 0) continue;
    // Cholesky of the kept block of M, then C = L^-1 K L^-T
    std::vector<double> L(k * k, 0.0), Kk(k * k);
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) Kk[i * k + j] = K[keep[i] * n + keep[j]];
    for (int j = 0; j < k; ++j) {
      double d = M[keep[j] * n + keep[j]];
      for (int l = 0; l < j; ++l) d -= L[j * k + l] * L[j * k + l];
      L[j * k + j] = std::sqrt(d);
      for (int i = j + 1; i < k; ++i) {
        double s = M[keep[i] * n + keep[j]];
        for (int l = 0; l < j; ++l) s -= L[i * k + l] * L[j * k + l];
        L[i * k + j] = s / L[j * k + j];
      }
    }
    std::vector<double> Li(k * k, 0.0);  // L^-1
    for (int c = 0; c < k; ++c)
      for (int i = c; i < k; ++i) {
        double s = (i == c) ? 1.0 : 0.0;
        for (int l = c; l < i; ++l) s -= L[i * k + l] * Li[l * k + c];
        Li[i * k + c] = s / L[i * k + i];
      }
    std::vector<double> C(k * k, 0.0), T(k * k, 0.0);
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j)
        for (int l = 0; l < k; ++l) T[i * k + j] += Li[i * k + l] * Kk[l * k + j];
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j)
        for (int l = 0; l < k; ++l) C[i * k + j] += T[i * k + l] * Li[j * k + l];
    for (int i = 0; i < k; ++i)
      for (int j = i + 1; j < k; ++j) C[i * k + j] = C[j * k + i] = 0.5 * (C[i * k + j] + C[j * k + i]);
    std::vector<double> V;
    const std::vector<double> w = sym_eigen_jacobi(C, k, V);
    for (int e = 0; e < k; ++e) {
      lam[type][keep[e]] = w[e];
      for (int i = 0; i < k; ++i) {  // S = L^-T V
        double s = 0.0;
        for (int l = i; l < k; ++l) s += Li[l * k + i] * V[l * k + e];
        S[type][keep[i]][keep[e]] = s;
      }
    }
  }
}

}  // namespace stmgb
