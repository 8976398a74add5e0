// march(spec, probes) on the device (src/driver.cpp:95-262) and the mesh /
// coefficient construction it needs. See run.hpp.
#include "run.hpp"

#include <chrono>
#include <cmath>
#include <limits>
#include <memory>
#include <stdexcept>

#include "kernels.hpp"

namespace stmgb {

namespace {

double now_seconds() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Xoshiro256::direction (include/stmg/rng.hpp:63-77): dim normals, rejected
// while the norm vanishes, normalised
std::array<double, 3> random_direction(Xoshiro256pp& rng, int dim) {
  std::array<double, 3> v{0.0, 0.0, 0.0};
  double norm2 = 0.0;
  do {
    norm2 = 0.0;
    for (int a = 0; a < dim; ++a) {
      v[a] = rng.normal();
      norm2 += v[a] * v[a];
    }
  } while (norm2 < 1e-30);
  const double inv = 1.0 / std::sqrt(norm2);
  for (int a = 0; a < dim; ++a) v[a] *= inv;
  return v;
}

std::vector<double> level_vertices(const MeshLevel& m) {
  if (!m.vertices.empty()) return m.vertices;
  const auto n = m.n_verts_axis();
  std::vector<double> x(static_cast<size_t>(3 * m.n_verts()), 0.0);
  for (Index kk = 0; kk < n[2]; ++kk)
    for (Index j = 0; j < n[1]; ++j)
      for (Index i = 0; i < n[0]; ++i) {
        const Index vi = (kk * n[1] + j) * n[0] + i;
        const Index idx[3] = {i, j, kk};
        for (int a = 0; a < m.dim; ++a) x[static_cast<size_t>(3 * vi + a)] = cartesian_coord(m, a, idx[a]);
      }
  return x;
}

// min_adjacent_edge (src/mesh.cpp:42-57) on the unperturbed positions
double min_adjacent_edge(const std::vector<double>& x, const std::array<Index, 3>& n, int dim, Index i, Index j,
                         Index kk) {
  const Index idx[3] = {i, j, kk};
  const Index vi = (kk * n[1] + j) * n[0] + i;
  double best = std::numeric_limits<double>::max();
  for (int a = 0; a < dim; ++a)
    for (int dir : {-1, 1}) {
      Index nb[3] = {idx[0], idx[1], idx[2]};
      nb[a] += dir;
      if (nb[a] < 0 || nb[a] >= n[a]) continue;
      const Index wi = (nb[2] * n[1] + nb[1]) * n[0] + nb[0];
      double d2 = 0.0;
      for (int c = 0; c < dim; ++c) {
        const double d = x[static_cast<size_t>(3 * vi + c)] - x[static_cast<size_t>(3 * wi + c)];
        d2 += d * d;
      }
      best = std::min(best, std::sqrt(d2));
    }
  return best;
}

// Jacobian determinant of the d-linear map of the cell with corner vertex
// indices cv at reference point xi (src/mesh.cpp:59-90)
double jacobian_det(const std::vector<double>& x, int dim, const Index* cv, const double* xi) {
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int s = 0; s < (1 << dim); ++s)
    for (int c = 0; c < dim; ++c) {
      double g = 1.0;
      for (int a = 0; a < dim; ++a) {
        const int bit = (s >> a) & 1;
        g *= a == c ? (bit ? 1.0 : -1.0) : (bit ? xi[a] : 1.0 - xi[a]);
      }
      for (int r = 0; r < dim; ++r) J[r][c] += g * x[static_cast<size_t>(3 * cv[s] + r)];
    }
  if (dim == 1) return J[0][0];
  if (dim == 2) return J[0][0] * J[1][1] - J[0][1] * J[1][0];
  return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

// coefficient_shm (src/mesh.cpp:267-279)
double shm_base(int dim, const double* x) {
  if (dim >= 3) return x[1] < 0.2 ? 1.0 : (x[2] < 0.2 ? 9.0 : 16.0);
  return x[1] < 0.2 ? 1.0 : 9.0;
}

}  // namespace

void check_positive_jacobians(const MeshLevel& m) {
  if (m.vertices.empty()) return;  // exact Cartesian lattice
  static const double samples[5] = {0.0, 0.2113248654051871, 0.5, 0.7886751345948129, 1.0};
  const auto n = m.n_verts_axis();
  const int d = m.dim;
  const int total = d == 1 ? 5 : (d == 2 ? 25 : 125);
  for (Index c = 0; c < m.n_cells(); ++c) {
    const Index cx = c % m.cells[0], cy = (c / m.cells[0]) % m.cells[1], cz = c / (m.cells[0] * m.cells[1]);
    Index cv[8];
    for (int s = 0; s < (1 << d); ++s)
      cv[s] = ((cz + ((s >> 2) & 1)) * n[1] + (cy + ((s >> 1) & 1))) * n[0] + (cx + (s & 1));
    for (int t = 0; t < total; ++t) {
      const double xi[3] = {samples[t % 5], d > 1 ? samples[(t / 5) % 5] : 0.0, d > 2 ? samples[t / 25] : 0.0};
      if (jacobian_det(m.vertices, d, cv, xi) <= 0.0)
        throw std::runtime_error("perturb: inverted cell after perturbation");
    }
  }
}

void perturb_mesh(MeshHierarchy& mesh, double magnitude, std::uint64_t seed) {
  if (magnitude < 0.0 || magnitude >= 0.5) throw std::invalid_argument("perturb: magnitude must be in [0, 0.5)");
  if (magnitude == 0.0) return;
  const MeshLevel& fine = mesh.levels.back();
  const auto n = fine.n_verts_axis();
  const std::vector<double> x = level_vertices(fine);
  std::vector<double> moved = x;
  Xoshiro256pp rng(seed);
  for (Index kk = 0; kk < n[2]; ++kk)
    for (Index j = 0; j < n[1]; ++j)
      for (Index i = 0; i < n[0]; ++i) {
        const double len = magnitude * min_adjacent_edge(x, n, fine.dim, i, j, kk);
        const auto dir = random_direction(rng, fine.dim);
        const Index vi = (kk * n[1] + j) * n[0] + i;
        const Index idx[3] = {i, j, kk};
        for (int a = 0; a < fine.dim; ++a) {
          if (idx[a] == 0 || idx[a] == n[a] - 1) continue;  // tangential only on the boundary
          moved[static_cast<size_t>(3 * vi + a)] += len * dir[a];
        }
      }
  set_finest_vertices(mesh, moved.data());
  for (const MeshLevel& m : mesh.levels) check_positive_jacobians(m);
}

Coefficient problem_coefficient(const ProblemSpec& spec, const MeshHierarchy& mesh) {
  const MeshLevel& m0 = mesh.levels.front();
  const Index nc = m0.n_cells();
  Coefficient rho;
  if (spec.problem == ProblemKind::Shm) {
    if (spec.dim < 2) throw std::invalid_argument("shm problem: dim must be 2 or 3");
    // the jumps at y = 0.2 (and z = 0.2 in 3D) must be faces of the level-0
    // cells, so that the field is constant per level-0 cell
    if (spec.perturb > 0.0)
      throw std::invalid_argument("shm problem: the piecewise coefficient needs an unperturbed mesh on the device");
    for (int a = 1; a < spec.dim; ++a) {
      const double h0 = (spec.hi[a] - spec.lo[a]) / static_cast<double>(m0.cells[a]);
      const double pos = (0.2 - spec.lo[a]) / h0;
      if (pos > 0.0 && pos < static_cast<double>(m0.cells[a]) && std::abs(pos - std::round(pos)) > 1e-9)
        throw std::invalid_argument("shm problem: the coefficient jumps must lie on level-0 cell faces");
    }
    rho.coarse_cell_scale.resize(static_cast<size_t>(nc));
    for (Index c = 0; c < nc; ++c) {
      const Index idx[3] = {c % m0.cells[0], (c / m0.cells[0]) % m0.cells[1], c / (m0.cells[0] * m0.cells[1])};
      double x[3] = {0.0, 0.0, 0.0};
      for (int a = 0; a < spec.dim; ++a)
        x[a] = spec.lo[a] + (spec.hi[a] - spec.lo[a]) * (static_cast<double>(idx[a]) + 0.5) /
                                static_cast<double>(m0.cells[a]);
      rho.coarse_cell_scale[static_cast<size_t>(c)] = shm_base(spec.dim, x);
    }
  }
  if (spec.rho_random_hi > spec.rho_random_lo && spec.rho_random_lo > 0.0) {
    Xoshiro256pp rng(spec.seed);
    const bool had = !rho.coarse_cell_scale.empty();
    rho.coarse_cell_scale.resize(static_cast<size_t>(nc), 1.0);
    for (Index c = 0; c < nc; ++c) {
      const double scale = spec.rho_random_lo + (spec.rho_random_hi - spec.rho_random_lo) * rng.uniform();
      rho.coarse_cell_scale[static_cast<size_t>(c)] = had ? scale * rho.coarse_cell_scale[static_cast<size_t>(c)] : scale;
    }
  }
  return rho;
}

RunReport run_march(const ProblemSpec& spec, const std::vector<double>& probes, cudaStream_t s) {
  const double t_wall0 = now_seconds();
  if (spec.dim < 2 || spec.dim > 3) throw std::invalid_argument("march: dim must be 2 or 3 on the device");
  const int k_min = spec.scheme == TimeScheme::DG ? 0 : 1;
  if (spec.k < k_min || spec.p < 1) throw std::invalid_argument("march: invalid k or p");
  if (spec.refinements < 0 || spec.base_cells < 1 || spec.base_time_intervals < 1)
    throw std::invalid_argument("march: invalid mesh sizes");
  const int n_steps_total = spec.base_time_intervals << (spec.refinements + 1);
  if (spec.batch < 1 || n_steps_total % spec.batch != 0)
    throw std::invalid_argument("march: batch must divide the step count");
  if (probes.size() % 3 != 0) throw std::invalid_argument("march: probes need 3 coordinates each");
  const double tau = spec.t_final / n_steps_total;
  const bool wave = spec.equation == Equation::Wave;

  MeshHierarchy mesh = make_cartesian(spec.dim, spec.lo, spec.hi, spec.base_cells, spec.refinements);
  if (spec.perturb > 0.0) perturb_mesh(mesh, spec.perturb, spec.seed);
  const Coefficient rho = problem_coefficient(spec, mesh);
  const TemporalWeights weights = spec.scheme == TimeScheme::DG ? dg_weights(spec.k) : cgp_weights(spec.k);
  const int fine_level = spec.refinements;

  std::unique_ptr<SpaceTimeMultigrid> mg;
  std::unique_ptr<SpaceTimeOperator> own_op;
  if (spec.precondition) {
    LevelSpec finest{fine_level, spec.p, spec.k, spec.batch, tau, Coarsening::SpaceH};
    const std::vector<Coarsening> strategy =
        spec.strategy.empty() ? default_strategy(finest, spec.scheme) : spec.strategy;
    MultigridOptions mgo;
    mgo.n_smooth = spec.n_smooth;
    mgo.seed = spec.seed;
    mg = std::make_unique<SpaceTimeMultigrid>(spec.equation, spec.scheme, mesh, rho,
                                              build_level_plan(finest, spec.scheme, strategy), mgo);
    mg->enable_timers(spec.timers);
  } else {
    own_op = std::make_unique<SpaceTimeOperator>(spec.equation, weights, tau, spec.batch, mesh, fine_level, spec.p, rho);
  }
  const SpaceTimeOperator& op = mg ? mg->fine_operator() : *own_op;

  RunReport report;
  report.n_space_dofs = op.n_space();
  report.n_steps_total = n_steps_total;
  report.n_batches = n_steps_total / spec.batch;
  report.dofs_global = static_cast<Index>(n_steps_total) * weights.n_t * op.n_space();
  if (mg) report.hierarchy = mg->level_info();

  // initial state (driver.cpp:150-166): interpolated, boundary zeroed
  const Index nx = op.n_space();
  DeviceBuffer u(sizeof(double) * nx), v(sizeof(double) * nx);
  switch (spec.problem) {
    case ProblemKind::Manufactured:
      vec_fill(u.d(), 0.0, nx, s);
      if (wave) op.interpolate(4, spec.frequency, 0.0, nullptr, 1.0, true, v.d(), s);
      break;
    case ProblemKind::Shm:
      if (!wave) throw std::invalid_argument("config: shm problem requires equation=wave");
      op.interpolate(5, 0.0, 0.0, nullptr, spec.shm_s, true, u.d(), s);
      vec_fill(v.d(), 0.0, nx, s);
      break;
    case ProblemKind::Zero:
      vec_fill(u.d(), 0.0, nx, s);
      vec_fill(v.d(), 0.0, nx, s);
      break;
  }

  ProbeSpec ps;
  ps.xyz = probes;
  ps.samples_per_step = spec.probe_samples_per_step;
  SectionClock op_clock;
  MarchOptions mo;
  mo.n_batches = report.n_batches;
  mo.source_kind = spec.problem == ProblemKind::Manufactured ? 1 : 0;
  mo.frequency = spec.frequency;
  mo.gmres.abs_tol = spec.abs_tol;
  mo.gmres.rel_tol = spec.rel_tol;
  mo.gmres.max_iters = spec.max_iters;
  mo.gmres.restart = spec.restart;
  mo.errors_u = spec.problem == ProblemKind::Manufactured;
  mo.errors_v = wave && spec.problem == ProblemKind::Manufactured;
  mo.probes = probes.empty() ? nullptr : &ps;
  mo.op_clock = spec.timers ? &op_clock : nullptr;
  const MarchResult mr = march(op, mg.get(), u.d(), wave ? v.d() : nullptr, mo, s);

  report.converged = mr.converged;
  double iter_sum = 0.0;
  for (size_t b = 0; b < mr.iterations.size(); ++b) {
    report.batches.push_back({mr.iterations[b], mr.final_residuals[b], mr.batch_converged[b] != 0});
    report.work += static_cast<double>(spec.batch) * weights.n_t * static_cast<double>(nx) * mr.iterations[b];
    iter_sum += mr.iterations[b];
  }
  report.mean_iterations = report.batches.empty() ? 0.0 : iter_sum / static_cast<double>(report.batches.size());
  report.has_error_u = mo.errors_u;
  report.has_error_v = mo.errors_v;
  report.error_u = mr.error_u;
  report.error_v = mr.error_v;
  report.probe_times = mr.probe_times;
  report.probe_values = mr.probe_values;

  cuda_check(cudaStreamSynchronize(s), "run_march");
  SectionTimes& st = report.sections;
  st.total = now_seconds() - t_wall0;
  if (mg && spec.timers) {
    st.smoother = mg->seconds_smoother();
    st.gmg_wo_smoother = mg->seconds_total() - st.smoother;
  }
  st.operator_wo_gmg = spec.timers ? op_clock.seconds() : 0.0;
  st.other = st.total - st.smoother - st.gmg_wo_smoother - st.operator_wo_gmg;
  return report;
}

}  // namespace stmgb
