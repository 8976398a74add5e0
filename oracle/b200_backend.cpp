// The reference-side binding of INTEGRATION.md, compiled for real: the
// LinearMap adapter a maintainer adds to the reference (`stmg`, C++) so that
// its own gmres() (src/gmres.cpp:8-115) runs the B200 operator and V-cycle,
// exactly as march() plugs in its CPU ones (src/driver.cpp:193-203,
// include/stmg/gmres.hpp:9-10). Built by oracle/Makefile against the
// reference headers (read in place), the Eigen shim and
// paper_2408_04372_b200/libstmg_b200.so into oracle/_ref/libb200_backend.so.
//
// TEST INFRASTRUCTURE: the namespace-stmg part is the binding itself; the
// extern "C" b200_backend_gmres() below is the test harness that drives it
// (tests/test_gpu_ref_binding.py).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "stmg/gmres.hpp"
#include "stmg/mesh.hpp"
#include "stmg/space_time_operator.hpp"
#include "stmg/temporal_weights.hpp"
#include "stmg_b200.h"

namespace stmg {

struct B200Slab {
  stmg_mesh* mesh = nullptr;
  stmg_multigrid* mg = nullptr;
  const stmg_st_operator* op = nullptr;  // finest level of mg
  B200Slab() = default;
  B200Slab(const B200Slab&) = delete;
  B200Slab& operator=(const B200Slab&) = delete;
  ~B200Slab() {
    if (mg) stmg_multigrid_destroy(mg);
    if (mesh) stmg_mesh_destroy(mesh);
  }
};

inline void b200_check(int rc) {
  if (rc == -1) throw std::invalid_argument(stmg_last_error());
  if (rc != 0) throw std::runtime_error(stmg_last_error());
}

// built once per march() from the data the CPU path uses: the mesh hierarchy
// (perturbed finest vertices included), the coefficient's per-level-0-cell
// scale, the discretisation and the multigrid options
inline void make_b200_slab(B200Slab& b, const MeshHierarchy& mesh, const CoefficientField& rho, Equation eq,
                           TimeScheme scheme, int p, int k, int batch, double tau, int n_smooth,
                           std::uint64_t seed) {
  const MeshLevel& fine = mesh.finest();
  std::vector<double> xyz;
  if (fine.perturbed) {
    xyz.reserve(3 * fine.vertices.size());
    for (const Point& v : fine.vertices) xyz.insert(xyz.end(), v.begin(), v.end());
  }
  const MeshLevel& base = mesh.levels.front();
  const double lo[3] = {fine.lo[0], fine.lo[1], fine.lo[2]}, hi[3] = {fine.hi[0], fine.hi[1], fine.hi[2]};
  b200_check(stmg_mesh_create(fine.dim, lo, hi, base.cells[0], mesh.n_levels() - 1,
                              fine.perturbed ? xyz.data() : nullptr, &b.mesh));
  stmg_mg_options o;
  stmg_mg_options_default(&o);
  o.n_smooth = n_smooth;
  o.seed = seed;
  const double* scale = rho.coarse_cell_scale.empty() ? nullptr : rho.coarse_cell_scale.data();
  b200_check(stmg_multigrid_create(eq == Equation::Heat ? 0 : 1, scheme == TimeScheme::DG ? 0 : 1, b.mesh, scale,
                                   mesh.n_levels() - 1, p, k, batch, tau, -1, nullptr, &o, &b.mg));
  b.op = stmg_multigrid_operator_at(b.mg, 0);
}

// the two LinearMaps march() hands to gmres (driver.cpp:193-203)
inline LinearMap b200_operator(const B200Slab& b) {
  return [&b](const Eigen::VectorXd& u, Eigen::VectorXd& y) {
    y.resize(u.size());
    b200_check(stmg_st_operator_apply_host(b.op, u.data(), y.data()));
  };
}
inline LinearMap b200_vcycle(const B200Slab& b) {
  return [&b](const Eigen::VectorXd& r, Eigen::VectorXd& z) {
    z.resize(r.size());
    b200_check(stmg_multigrid_apply_host(b.mg, r.data(), z.data()));
  };
}

// or the whole slab solve on the device (one call per batch)
inline GmresResult b200_solve(const B200Slab& b, const Eigen::VectorXd& rhs, Eigen::VectorXd& x,
                              const GmresOptions& g) {
  stmg_gmres_options o{g.max_iters, g.restart, g.rel_tol, g.abs_tol};
  stmg_gmres_result r{};
  std::vector<double> hist(static_cast<size_t>(g.max_iters) + 2);
  x.resize(rhs.size());
  x.setZero();
  b200_check(stmg_solve_host(b.mg, 1, rhs.data(), x.data(), &o, &r, hist.data(), static_cast<int>(hist.size())));
  GmresResult out;
  out.converged = r.converged != 0;
  out.iterations = r.iterations;
  out.initial_residual = r.initial_residual;
  out.final_residual = r.final_residual;
  const int n = r.history_len < static_cast<int>(hist.size()) ? r.history_len : static_cast<int>(hist.size());
  out.residual_history.assign(hist.begin(), hist.begin() + n);
  return out;
}

}  // namespace stmg

// ------------------------------------------------------------ test harness
namespace {
thread_local std::string g_err;
}

extern "C" {

const char* b200_backend_last_error() { return g_err.c_str(); }

// The reference's gmres() on the slab system of a make_cartesian mesh
// (finest vertices injected when given, coefficient per level-0 cell), with
// the B200 LinearMaps (mode 0) or the device solve b200_solve (mode 1).
int b200_backend_gmres(int dim, int equation, int scheme, int p, int k, int batch, double tau, int base_cells,
                       int refinements, const double* vertices, const double* cell_scale, int n_smooth,
                       std::uint64_t seed, int mode, double rel_tol, double abs_tol, int restart, int max_iters,
                       const double* b, double* x, int* iterations, int* converged) {
  try {
    using namespace stmg;
    MeshHierarchy mesh = make_cartesian(dim, {0, 0, 0}, {1, 1, 1}, base_cells, refinements);
    if (vertices) {
      MeshLevel& fine = mesh.levels.back();
      for (size_t i = 0; i < fine.vertices.size(); ++i)
        fine.vertices[i] = {vertices[3 * i], vertices[3 * i + 1], vertices[3 * i + 2]};
      fine.perturbed = true;
    }
    CoefficientField rho = constant_coefficient(1.0);
    if (cell_scale)
      rho.coarse_cell_scale.assign(cell_scale, cell_scale + mesh.levels.front().n_cells());
    B200Slab slab;
    make_b200_slab(slab, mesh, rho, equation == 0 ? Equation::Heat : Equation::Wave,
                   scheme == 0 ? TimeScheme::DG : TimeScheme::CGP, p, k, batch, tau, n_smooth, seed);
    const long long n = stmg_st_operator_n_dofs(slab.op);
    Eigen::VectorXd rhs(n), sol(n);
    std::memcpy(rhs.data(), b, sizeof(double) * static_cast<size_t>(n));
    sol.setZero();
    GmresOptions o;
    o.rel_tol = rel_tol;
    o.abs_tol = abs_tol;
    o.restart = restart;
    o.max_iters = max_iters;
    const GmresResult r = mode == 0 ? gmres(b200_operator(slab), rhs, sol, o, b200_vcycle(slab))
                                    : b200_solve(slab, rhs, sol, o);
    std::memcpy(x, sol.data(), sizeof(double) * static_cast<size_t>(n));
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
