// C-ABI harness over the reference's own classes (compiled from
// /root/reference/proj/src against oracle/shim). Test infrastructure only: the
// checker for tests/ and the CPU baseline arm of bench.py. Each entry point
// names the reference interface it drives.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <json.hpp>

#include "stmg/asm_smoother.hpp"
#include "stmg/config.hpp"
#include "stmg/driver.hpp"
#include "stmg/gmres.hpp"
#include "stmg/multigrid.hpp"
#include "stmg/transfer.hpp"

using namespace stmg;

namespace {
thread_local std::string g_err;

struct RefDesc {
  int dim, equation, scheme, k, p, n_steps;
  double tau;
  int base_cells, refinements;
  double lo[3], hi[3];
  const double* vertices;     // finest level, n_verts*3, or null (Cartesian)
  const double* cell_scale;   // rho per level-0 cell, or null (rho = 1)
  double perturb_magnitude;   // >0: reference perturb() (mesh.cpp:191-240)
  std::uint64_t perturb_seed;
  int with_mg;                // build SpaceTimeMultigrid (multigrid.cpp:83-125)
  int n_strategy;             // <0: default_strategy
  const int* strategy;        // Coarsening codes (multigrid.hpp:14)
  int n_smooth;
  long direct_coarse_max;
  double coarse_rel_tol;
  int coarse_max_iters;
  int eig_iters;
  std::uint64_t mg_seed;
};

struct Ref {
  MeshHierarchy mesh;
  CoefficientField rho;
  TemporalWeights weights;
  std::unique_ptr<SpatialDofMap> dofmap;
  std::unique_ptr<SpatialOperator> mass, stiffness;
  std::unique_ptr<SpaceTimeOperator> op;
  std::unique_ptr<SpaceTimeMultigrid> mg;
  std::vector<std::unique_ptr<Transfer>> transfers;
  std::vector<LevelSpec> plan;
};

Eigen::VectorXd vec(const double* p, Index n) {
  Eigen::VectorXd v(n);
  if (n) std::memcpy(v.data(), p, sizeof(double) * static_cast<std::size_t>(n));
  return v;
}
void out(const Eigen::VectorXd& v, double* p) {
  if (v.size()) std::memcpy(p, v.data(), sizeof(double) * static_cast<std::size_t>(v.size()));
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_create(const RefDesc* d) {
  auto r = std::make_unique<Ref>();
  const int rc = guard([&] {
    r->mesh = make_cartesian(d->dim, {d->lo[0], d->lo[1], d->lo[2]}, {d->hi[0], d->hi[1], d->hi[2]},
                             d->base_cells, d->refinements);
    if (d->perturb_magnitude > 0.0) perturb(r->mesh, d->perturb_magnitude, d->perturb_seed);
    if (d->vertices) {
      // finest vertices injected; coarse levels take the shared positions
      // (same nesting convention as mesh.cpp:221-236)
      MeshLevel& fine = r->mesh.levels.back();
      for (std::size_t i = 0; i < fine.vertices.size(); ++i)
        fine.vertices[i] = {d->vertices[3 * i], d->vertices[3 * i + 1], d->vertices[3 * i + 2]};
      fine.perturbed = true;
      const int fl = r->mesh.n_levels() - 1;
      for (int l = 0; l < fl; ++l) {
        MeshLevel& m = r->mesh.levels[static_cast<std::size_t>(l)];
        const Index stride = Index{1} << (fl - l);
        const auto nc = m.n_verts_axis();
        for (Index kk = 0; kk < nc[2]; ++kk)
          for (Index j = 0; j < nc[1]; ++j)
            for (Index i = 0; i < nc[0]; ++i)
              m.vertices[static_cast<std::size_t>(m.vertex_index(i, j, kk))] =
                  fine.vertices[static_cast<std::size_t>(
                      fine.vertex_index(i * stride, m.dim > 1 ? j * stride : 0, m.dim > 2 ? kk * stride : 0))];
        m.perturbed = true;
      }
    }
    r->rho = constant_coefficient(1.0);
    if (d->cell_scale) {
      const Index nc = r->mesh.levels.front().n_cells();
      r->rho.coarse_cell_scale.assign(d->cell_scale, d->cell_scale + nc);
    }
    const TimeScheme scheme = d->scheme == 0 ? TimeScheme::DG : TimeScheme::CGP;
    const Equation eq = d->equation == 0 ? Equation::Heat : Equation::Wave;
    r->weights = scheme == TimeScheme::DG ? dg_weights(d->k) : cgp_weights(d->k);
    const int fine = d->refinements;
    r->dofmap = std::make_unique<SpatialDofMap>(r->mesh.levels[static_cast<std::size_t>(fine)], d->p);
    r->mass = std::make_unique<SpatialOperator>(SpatialOperator::Kind::Mass, r->mesh, fine, *r->dofmap);
    r->stiffness =
        std::make_unique<SpatialOperator>(SpatialOperator::Kind::Stiffness, r->mesh, fine, *r->dofmap, r->rho);
    r->op = std::make_unique<SpaceTimeOperator>(eq, r->weights, d->tau, d->n_steps, *r->mass, *r->stiffness);
    if (d->with_mg) {
      const LevelSpec finest{fine, d->p, d->k, d->n_steps, d->tau, Coarsening::SpaceH};
      std::vector<Coarsening> strategy;
      if (d->n_strategy < 0)
        strategy = default_strategy(finest, scheme);
      else
        for (int i = 0; i < d->n_strategy; ++i) strategy.push_back(static_cast<Coarsening>(d->strategy[i]));
      r->plan = build_level_plan(finest, scheme, strategy);
      MultigridOptions o;
      o.n_smooth = d->n_smooth;
      o.direct_coarse_max = d->direct_coarse_max;
      o.coarse_rel_tol = d->coarse_rel_tol;
      o.coarse_max_iters = d->coarse_max_iters;
      o.eig_iters = d->eig_iters;
      o.seed = d->mg_seed;
      r->mg = std::make_unique<SpaceTimeMultigrid>(eq, scheme, r->mesh, r->rho, r->plan, o);
      for (int l = 0; l + 1 < r->mg->n_levels(); ++l)
        r->transfers.push_back(std::make_unique<Transfer>(r->mg->operator_at(l), r->mg->operator_at(l + 1)));
    }
  });
  if (rc != 0) return nullptr;
  return r.release();
}

void ref_destroy(void* h) { delete static_cast<Ref*>(h); }

long ref_n_dofs(void* h) { return static_cast<long>(static_cast<Ref*>(h)->op->n_dofs()); }
long ref_n_space(void* h) { return static_cast<long>(static_cast<Ref*>(h)->op->n_space()); }

// SpaceTimeOperator::apply (space_time_operator.cpp:45-130)
int ref_apply(void* h, const double* u, double* y) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    Eigen::VectorXd yy;
    r->op->apply(vec(u, r->op->n_dofs()), yy);
    out(yy, y);
  });
}

// SpatialOperator::apply (spatial_operator.cpp:292-315); kind 0 mass, 1 stiffness
int ref_spatial_apply(void* h, int kind, const double* u, double* y) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    Eigen::VectorXd yy;
    const SpatialOperator& s = kind == 0 ? *r->mass : *r->stiffness;
    s.apply(vec(u, s.n_dofs()), yy);
    out(yy, y);
  });
}

int ref_mg_levels(void* h) {
  auto* r = static_cast<Ref*>(h);
  return r->mg ? r->mg->n_levels() : 0;
}

// SpaceTimeMultigrid::level_info (multigrid.cpp:236-247)
int ref_level_info(void* h, int l, int* ints /*mesh_level,p,k,n_steps,coarsening*/, long* n_dofs, double* omega) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    const auto info = r->mg->level_info();
    const LevelInfo& li = info.at(static_cast<std::size_t>(l));
    ints[0] = li.mesh_level;
    ints[1] = li.p;
    ints[2] = li.k;
    ints[3] = li.n_steps;
    ints[4] = l == 0 ? -1 : static_cast<int>(r->plan[static_cast<std::size_t>(l)].from_finer);
    *n_dofs = static_cast<long>(li.n_dofs);
    *omega = li.omega;
  });
}

double ref_level_tau(void* h, int l) { return static_cast<Ref*>(h)->plan.at(static_cast<std::size_t>(l)).tau; }

int ref_level_apply(void* h, int l, const double* u, double* y) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    const SpaceTimeOperator& op = r->mg->operator_at(l);
    Eigen::VectorXd yy;
    op.apply(vec(u, op.n_dofs()), yy);
    out(yy, y);
  });
}

// ASMSmoother::add_correction (asm_smoother.cpp:60-78): z accumulates
int ref_asm_add_correction(void* h, int l, const double* res, double* z) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    const SpaceTimeOperator& op = r->mg->operator_at(l);
    Eigen::VectorXd zz = vec(z, op.n_dofs());
    r->mg->smoother_at(l).add_correction(vec(res, op.n_dofs()), zz);
    out(zz, z);
  });
}

int ref_asm_overlap_counts(void* h, int l, double* counts) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] { out(r->mg->smoother_at(l).overlap_counts(), counts); });
}

// Transfer::prolong / restrict_ (transfer.cpp:118-190) between levels l, l+1
int ref_prolong(void* h, int l, const double* coarse, double* fine) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    Eigen::VectorXd f;
    r->transfers.at(static_cast<std::size_t>(l))->prolong(vec(coarse, r->mg->operator_at(l + 1).n_dofs()), f);
    out(f, fine);
  });
}
int ref_restrict(void* h, int l, const double* fine, double* coarse) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    Eigen::VectorXd c;
    r->transfers.at(static_cast<std::size_t>(l))->restrict_(vec(fine, r->mg->operator_at(l).n_dofs()), c);
    out(c, coarse);
  });
}

double ref_omega(void* h, int l) { return static_cast<Ref*>(h)->mg->omega_at(l); }
void ref_set_omega(void* h, int l, double w) { static_cast<Ref*>(h)->mg->set_omega(l, w); }

// SpaceTimeMultigrid::smooth / v_cycle / apply (multigrid.cpp:174-234)
int ref_smooth(void* h, int l, const double* f, double* u) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    const Index n = r->mg->operator_at(l).n_dofs();
    Eigen::VectorXd uu = vec(u, n);
    r->mg->smooth(l, vec(f, n), uu);
    out(uu, u);
  });
}
int ref_vcycle_apply(void* h, const double* res, double* z) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    Eigen::VectorXd zz;
    r->mg->apply(vec(res, r->op->n_dofs()), zz);
    out(zz, z);
  });
}

// gmres (gmres.cpp:8-115) with op = SpaceTimeOperator::apply and, if
// precond != 0, the V-cycle preconditioner, exactly as march() plugs them
// (driver.cpp:193-203)
int ref_gmres(void* h, const double* b, double* x, int max_iters, int restart, double rel_tol, double abs_tol,
              int precond, int* iterations, double* final_residual, double* initial_residual, double* history,
              int history_cap, int* history_len, int* converged) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    GmresOptions o;
    o.max_iters = max_iters;
    o.restart = restart;
    o.rel_tol = rel_tol;
    o.abs_tol = abs_tol;
    LinearMap op = [r](const Eigen::VectorXd& v, Eigen::VectorXd& y) { r->op->apply(v, y); };
    LinearMap pc;
    if (precond) pc = [r](const Eigen::VectorXd& v, Eigen::VectorXd& z) { r->mg->apply(v, z); };
    Eigen::VectorXd xx = vec(x, r->op->n_dofs());
    const GmresResult res = gmres(op, vec(b, r->op->n_dofs()), xx, o, pc);
    out(xx, x);
    *iterations = res.iterations;
    *final_residual = res.final_residual;
    *initial_residual = res.initial_residual;
    *converged = res.converged ? 1 : 0;
    const int n = std::min<int>(history_cap, static_cast<int>(res.residual_history.size()));
    for (int i = 0; i < n; ++i) history[i] = res.residual_history[static_cast<std::size_t>(i)];
    *history_len = static_cast<int>(res.residual_history.size());
  });
}

// SpaceTimeOperator::assemble_rhs (space_time_operator.cpp:138-221) with the
// manufactured source of driver.cpp:265-293 (source_kind 1, frequency f) or a
// zero source (source_kind 0); entering state u0 (and v0 for the wave)
int ref_assemble_rhs(void* h, int source_kind, double frequency, double t0, const double* u0, const double* v0,
                     double* rhs) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    ProblemSpec spec;
    spec.dim = r->mesh.finest().dim;
    spec.equation = r->op->equation();
    SpaceTimeFunction f = [](const Point&, double) { return 0.0; };
    if (source_kind == 1) {
      manufactured_problem(spec, frequency);
      f = spec.source;
    }
    BatchState st;
    st.u = vec(u0, r->op->n_space());
    if (r->op->equation() == Equation::Wave) st.v = vec(v0, r->op->n_space());
    out(r->op->assemble_rhs(f, t0, st), rhs);
  });
}

// error_norms (driver.cpp:83-92) of one batch solution u entering from u0
// against the manufactured solution of driver.cpp:265-293 (frequency f);
// out = {L2(L2), Linf(L2), Linf(Linf)}
int ref_error_norms(void* h, const double* u, const double* u0, double frequency, double t0, double* out3) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    ProblemSpec spec;
    spec.dim = r->mesh.finest().dim;
    spec.equation = r->op->equation();
    manufactured_problem(spec, frequency);
    BatchState st;
    st.u = vec(u0, r->op->n_space());
    const std::vector<Eigen::VectorXd> xs{vec(u, r->op->n_dofs())};
    const std::vector<BatchState> es{st};
    const ErrorRecord e = error_norms(*r->op, xs, es, spec.exact_u, t0);
    out3[0] = e.l2_l2;
    out3[1] = e.linf_l2;
    out3[2] = e.linf_linf;
  });
}

// value_at (space_time_operator.cpp:250-266) of a batch solution u entering
// from u0, then evaluate_fe at locate_point(x) on the finest mesh
// (spatial_operator.cpp:451-524): the probe sample march() records
int ref_probe_value(void* h, const double* u, const double* u0, int step, double t_ref, const double* x3, double* out) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    BatchState st;
    st.u = vec(u0, r->op->n_space());
    const Eigen::VectorXd val = r->op->value_at(vec(u, r->op->n_dofs()), st, step, t_ref);
    const Point x{x3[0], x3[1], x3[2]};
    const auto loc = locate_point(r->mesh.finest(), x);
    *out = evaluate_fe(*r->dofmap, val, loc.first, loc.second);
  });
}

// extract_final (space_time_operator.cpp:223-248)
int ref_extract_final(void* h, const double* u, const double* u0, const double* v0, double* uf, double* vf) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    BatchState st;
    st.u = vec(u0, r->op->n_space());
    if (r->op->equation() == Equation::Wave) st.v = vec(v0, r->op->n_space());
    const BatchState o = r->op->extract_final(vec(u, r->op->n_dofs()), st);
    out(o.u, uf);
    if (r->op->equation() == Equation::Wave) out(o.v, vf);
  });
}

// interpolate (spatial_operator.cpp:437-449) of a Gaussian pulse
// exp(-|x-c|^2/(2 w^2)) on the finest dofmap (C4 initial data)
int ref_interpolate_gaussian(void* h, const double* centre, double width, double* u) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    const int dim = r->mesh.finest().dim;
    const Point c{centre[0], centre[1], centre[2]};
    out(interpolate(*r->dofmap,
                    [&](const Point& x) {
                      double s = 0.0;
                      for (int a = 0; a < dim; ++a) s += (x[a] - c[a]) * (x[a] - c[a]);
                      return std::exp(-s / (2.0 * width * width));
                    }),
        u);
  });
}

// finest-level mesh vertices (after perturbation), n_verts*3
int ref_vertices(void* h, int level, double* xyz) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    const MeshLevel& m = r->mesh.levels.at(static_cast<std::size_t>(level));
    for (std::size_t i = 0; i < m.vertices.size(); ++i)
      for (int a = 0; a < 3; ++a) xyz[3 * i + a] = m.vertices[i][static_cast<std::size_t>(a)];
  });
}

// SpaceTimeOperator::block_coefficients (space_time_operator.cpp:269-317), n_t x n_t row-major
int ref_block_coefficients(void* h, int s, int j, double* cM, double* cA) {
  auto* r = static_cast<Ref*>(h);
  return guard([&] {
    Eigen::MatrixXd M, A;
    r->op->block_coefficients(s, j, M, A);
    for (Index a = 0; a < M.rows(); ++a)
      for (Index b = 0; b < M.cols(); ++b) {
        cM[a * M.cols() + b] = M(a, b);
        cA[a * M.cols() + b] = A(a, b);
      }
  });
}

// temporal weight tables (temporal_weights.cpp:29-106)
int ref_temporal_weights(int scheme, int k, double* m_tau, double* a_tau, double* alpha, double* beta, double* nodes) {
  return guard([&] {
    const TemporalWeights w = scheme == 0 ? dg_weights(k) : cgp_weights(k);
    for (int i = 0; i < w.n_t; ++i) {
      for (int j = 0; j < w.n_t; ++j) {
        m_tau[i * w.n_t + j] = w.m_tau(i, j);
        a_tau[i * w.n_t + j] = w.a_tau(i, j);
      }
      alpha[i] = w.alpha[i];
      beta[i] = w.beta[i];
      nodes[i] = w.unknown_nodes[static_cast<std::size_t>(i)];
    }
  });
}

// quadrature rules (quadrature.cpp:98-166); kind 0 gauss, 1 lobatto, 2 radau-right
int ref_quadrature(int kind, int n, double* pts, double* wts) {
  return guard([&] {
    const QuadratureRule q = kind == 0 ? gauss(n) : (kind == 1 ? gauss_lobatto(n) : gauss_radau_right(n));
    for (int i = 0; i < q.size(); ++i) {
      pts[i] = q.points[static_cast<std::size_t>(i)];
      wts[i] = q.weights[static_cast<std::size_t>(i)];
    }
  });
}

// ---- configured runs (src/config.cpp + march, src/driver.cpp:95-262): the
// run report in the key layout of the stmg tool's report_to_json
// (tools/stmg.cpp:30-62), plus the probe series, for parity of the device run
namespace {
nlohmann::json run_to_json(const RunReport& r) {
  using nlohmann::json;
  json batches = json::array();
  for (const BatchStats& b : r.batches)
    batches.push_back({{"iterations", b.iterations}, {"final_residual", b.final_residual}, {"converged", b.converged}});
  json hierarchy = json::array();
  for (const LevelInfo& l : r.hierarchy)
    hierarchy.push_back({{"coarsening", l.coarsening}, {"mesh_level", l.mesh_level}, {"p", l.p}, {"k", l.k},
                         {"n_steps", l.n_steps}, {"n_dofs", l.n_dofs}, {"omega", l.omega}});
  json out{{"converged", r.converged},       {"n_space_dofs", r.n_space_dofs}, {"n_steps_total", r.n_steps_total},
           {"n_batches", r.n_batches},       {"dofs_global", r.dofs_global},   {"mean_iterations", r.mean_iterations},
           {"work", r.work},                 {"batches", batches},             {"hierarchy", hierarchy},
           {"probe_times", r.probe_times},   {"probe_values", r.probe_values}};
  auto err = [](const ErrorRecord& e) {
    return json{{"l2_l2", e.l2_l2}, {"linf_l2", e.linf_l2}, {"linf_linf", e.linf_linf}};
  };
  if (r.error_u) out["error_u"] = err(*r.error_u);
  if (r.error_v) out["error_v"] = err(*r.error_v);
  return out;
}
int put(const std::string& s, char* out, long cap) {
  if (static_cast<long>(s.size()) + 1 > cap) {
    g_err = "output buffer too small (" + std::to_string(s.size() + 1) + " bytes needed)";
    return -2;
  }
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}
}  // namespace

// parse_config + make_problem + march(spec, resolve_probes) at refinement r
// (r < 0: config.refinements)
int ref_run_json(const char* config_json, int refinement, char* out, long cap) {
  std::string s;
  const int rc = guard([&] {
    const Config c = parse_config(config_json);
    const ProblemSpec spec = make_problem(c, refinement < 0 ? c.refinements : refinement);
    s = run_to_json(march(spec, resolve_probes(c))).dump();
  });
  return rc != 0 ? rc : put(s, out, cap);
}

// parse_config, the --set overrides (apply_override), config_to_json
// (src/config.cpp:87-160); returns -1 with the message on invalid input
int ref_config_json(const char* config_json, int n_overrides, const char* const* keys, const char* const* values,
                    char* out, long cap) {
  std::string s;
  const int rc = guard([&] {
    Config c = parse_config(config_json);
    for (int i = 0; i < n_overrides; ++i) apply_override(c, keys[i], values[i]);
    s = config_to_json(c).dump();
  });
  return rc != 0 ? rc : put(s, out, cap);
}

// make_cartesian + perturb (src/mesh.cpp:148-240): finest vertices
int ref_perturbed_vertices(int dim, const double* lo, const double* hi, int base_cells, int refinements,
                           double magnitude, std::uint64_t seed, double* xyz) {
  return guard([&] {
    MeshHierarchy m = make_cartesian(dim, {lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}, base_cells, refinements);
    perturb(m, magnitude, seed);
    const MeshLevel& f = m.levels.back();
    for (std::size_t v = 0; v < f.vertices.size(); ++v)
      for (int a = 0; a < 3; ++a) xyz[3 * v + a] = f.vertices[v][a];
  });
}

}  // extern "C"
