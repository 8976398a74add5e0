// C ABI over the host C++ layer (declarations: include/stmg_b200.h). No
// exception crosses this boundary; failures become negative return codes and
// stmg_last_error().
#include "../../include/stmg_b200.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "run.hpp"
#include "slab_mg.hpp"
#include "stmg.hpp"

using namespace stmgb;

struct stmg_mesh {
  MeshHierarchy h;
};
struct stmg_st_operator {
  std::unique_ptr<SpaceTimeOperator> owned;
  const SpaceTimeOperator* op = nullptr;  // owned.get() or a multigrid level
  TemporalWeights w;
  mutable DeviceBuffer hu, hy;  // staging for the host-buffer entry point
};
struct stmg_asm {
  std::unique_ptr<ASMSmoother> s;
};
struct stmg_transfer {
  std::unique_ptr<Transfer> t;
};
struct stmg_comm {
  std::unique_ptr<Comm> c;
};
struct stmg_slab_multigrid {
  std::unique_ptr<SlabMultigrid> mg;
};
struct stmg_multigrid {
  std::unique_ptr<SpaceTimeMultigrid> mg;
  std::vector<std::unique_ptr<stmg_st_operator>> views;  // non-owning wrappers for operator_at
  mutable GmresWorkspace ws;
  mutable DeviceBuffer hr, hz;  // staging for the host-buffer entry points
};

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      g_err = std::string("CUDA: ") + cudaGetErrorString(e);
      return -3;
    }
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}
// host-only entry points: no CUDA state is touched
template <typename F>
int guard_host(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}
cudaStream_t st(void* s) { return static_cast<cudaStream_t>(s); }
Coefficient coeff(const MeshHierarchy& h, const double* scale) {
  Coefficient c;
  if (scale) c.coarse_cell_scale.assign(scale, scale + h.levels.front().n_cells());
  return c;
}
}  // namespace

extern "C" {

const char* stmg_last_error(void) { return g_err.c_str(); }
const char* stmg_version(void) { return "stmg-b200 0.1 (sm_100a)"; }
long long stmg_kernel_launches(void) { return kernel_launches(); }

int stmg_quadrature(int kind, int n, double* points, double* weights) {
  return guard_host([&] {
    const Rule r = kind == 0 ? gauss(n) : (kind == 1 ? gauss_lobatto(n) : gauss_radau_right(n));
    for (size_t i = 0; i < r.x.size(); ++i) {
      points[i] = r.x[i];
      weights[i] = r.w[i];
    }
  });
}
int stmg_temporal_weights(int scheme, int k, double* m_tau, double* a_tau, double* alpha, double* beta,
                          double* unknown_nodes) {
  return guard_host([&] {
    const TemporalWeights w = scheme == STMG_DG ? dg_weights(k) : cgp_weights(k);
    std::copy(w.m.begin(), w.m.end(), m_tau);
    std::copy(w.a.begin(), w.a.end(), a_tau);
    std::copy(w.alpha.begin(), w.alpha.end(), alpha);
    std::copy(w.beta.begin(), w.beta.end(), beta);
    std::copy(w.unknown_nodes.begin(), w.unknown_nodes.end(), unknown_nodes);
  });
}
int stmg_block_coefficients(int equation, int scheme, int k, double tau, int n_steps, double* CM, double* CA) {
  return guard_host([&] {
    const TemporalWeights w = scheme == STMG_DG ? dg_weights(k) : cgp_weights(k);
    std::vector<double> cm, ca;
    block_coefficient_matrices(static_cast<Equation>(equation), w, tau, n_steps, cm, ca);
    std::copy(cm.begin(), cm.end(), CM);
    std::copy(ca.begin(), ca.end(), CA);
  });
}

int stmg_mesh_create(int dim, const double lo[3], const double hi[3], long long base_cells, int refinements,
                     const double* finest_vertices, stmg_mesh** out) {
  return guard_host([&] {
    if (!out) throw std::invalid_argument("stmg_mesh_create: null out");
    auto m = std::make_unique<stmg_mesh>();
    m->h = make_cartesian(dim, {lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}, base_cells, refinements);
    if (finest_vertices) set_finest_vertices(m->h, finest_vertices);
    *out = m.release();
  });
}
int stmg_mesh_create_box(int dim, const double lo[3], const double hi[3], const long long base_cells[3],
                         int refinements, const double* finest_vertices, stmg_mesh** out) {
  return guard_host([&] {
    if (!out || !base_cells) throw std::invalid_argument("stmg_mesh_create_box: null argument");
    auto m = std::make_unique<stmg_mesh>();
    m->h = make_cartesian_box(dim, {lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]},
                              {base_cells[0], base_cells[1], base_cells[2]}, refinements);
    if (finest_vertices) set_finest_vertices(m->h, finest_vertices);
    *out = m.release();
  });
}
void stmg_mesh_destroy(stmg_mesh* mesh) { delete mesh; }

int stmg_st_operator_create(const stmg_mesh* mesh, int mesh_level, int p, int equation, int scheme, int k, double tau,
                            int n_steps, const double* coarse_cell_scale, stmg_st_operator** out) {
  return guard([&] {
    if (!mesh || !out) throw std::invalid_argument("stmg_st_operator_create: null argument");
    auto o = std::make_unique<stmg_st_operator>();
    o->w = scheme == STMG_DG ? dg_weights(k) : cgp_weights(k);
    o->owned = std::make_unique<SpaceTimeOperator>(static_cast<Equation>(equation), o->w, tau, n_steps, mesh->h,
                                                   mesh_level, p, coeff(mesh->h, coarse_cell_scale));
    o->op = o->owned.get();
    *out = o.release();
  });
}
void stmg_st_operator_destroy(stmg_st_operator* op) { delete op; }
long long stmg_st_operator_n_dofs(const stmg_st_operator* op) { return op ? op->op->n_dofs() : -1; }
long long stmg_st_operator_n_space(const stmg_st_operator* op) { return op ? op->op->n_space() : -1; }
int stmg_st_operator_n_t(const stmg_st_operator* op) { return op ? op->op->n_t() : -1; }

int stmg_st_operator_apply(const stmg_st_operator* op, const double* d_u, double* d_y, void* stream) {
  return guard([&] {
    if (!op || !d_u || !d_y) throw std::invalid_argument("stmg_st_operator_apply: null argument");
    op->op->apply(d_u, d_y, st(stream));
  });
}

int stmg_st_operator_apply_host(const stmg_st_operator* op, const double* h_u, double* h_y) {
  return guard([&] {
    if (!op || !h_u || !h_y) throw std::invalid_argument("stmg_st_operator_apply_host: null argument");
    const size_t bytes = sizeof(double) * op->op->n_dofs();
    if (op->hu.bytes() != bytes) {
      op->hu.allocate(bytes);
      op->hy.allocate(bytes);
    }
    copy_to_device(op->hu.d(), h_u, bytes, nullptr);
    op->op->apply(op->hu.d(), op->hy.d(), nullptr);
    copy_to_host(h_y, op->hy.d(), bytes, nullptr);
  });
}

int stmg_spatial_apply(const stmg_st_operator* op, int kind, const double* d_u, double* d_y, void* stream) {
  return guard([&] {
    if (!op || !d_u || !d_y || (kind != 0 && kind != 1)) throw std::invalid_argument("stmg_spatial_apply: bad argument");
    op->op->spatial_apply(kind, d_u, d_y, st(stream));
  });
}

int stmg_st_operator_residual(const stmg_st_operator* op, const double* d_f, const double* d_u, double* d_r,
                              void* stream) {
  return guard([&] {
    if (!op || !d_f || !d_u || !d_r) throw std::invalid_argument("stmg_st_operator_residual: null argument");
    op->op->residual(d_f, d_u, d_r, st(stream));
  });
}

int stmg_st_operator_interpolate(const stmg_st_operator* op, int kind, double frequency, double t,
                                 const double centre[3], double width, int zero_boundary, double* d_out,
                                 void* stream) {
  return guard([&] {
    if (!op || !d_out || kind < 0 || kind > 5) throw std::invalid_argument("stmg_st_operator_interpolate: bad argument");
    op->op->interpolate(kind, frequency, t, centre, width, zero_boundary != 0, d_out, st(stream));
  });
}

int stmg_st_operator_assemble_rhs(const stmg_st_operator* op, int source_kind, double frequency, double t0,
                                  const double* d_u0, const double* d_v0, double* d_rhs, void* stream) {
  return guard([&] {
    if (!op || !d_u0 || !d_rhs) throw std::invalid_argument("stmg_st_operator_assemble_rhs: null argument");
    op->op->assemble_rhs(source_kind, frequency, t0, d_u0, d_v0, d_rhs, st(stream));
  });
}

int stmg_st_operator_extract_final(const stmg_st_operator* op, const double* d_u, const double* d_u0,
                                   const double* d_v0, double* d_uf, double* d_vf, void* stream) {
  return guard([&] {
    if (!op || !d_u || !d_u0 || !d_uf) throw std::invalid_argument("stmg_st_operator_extract_final: null argument");
    op->op->extract_final(d_u, d_u0, d_v0, d_uf, d_vf, st(stream));
  });
}

int stmg_asm_create(const stmg_st_operator* op, stmg_asm** out) {
  return guard([&] {
    if (!op || !out) throw std::invalid_argument("stmg_asm_create: null argument");
    auto a = std::make_unique<stmg_asm>();
    a->s = std::make_unique<ASMSmoother>(*op->op);
    *out = a.release();
  });
}
void stmg_asm_destroy(stmg_asm* a) { delete a; }
int stmg_asm_add_correction(const stmg_asm* a, const double* d_r, double* d_z, void* stream) {
  return guard([&] {
    if (!a || !d_r || !d_z) throw std::invalid_argument("stmg_asm_add_correction: null argument");
    a->s->add_correction(d_r, d_z, st(stream));
  });
}

int stmg_transfer_create(const stmg_st_operator* fine, const stmg_st_operator* coarse, stmg_transfer** out) {
  return guard([&] {
    if (!fine || !coarse || !out) throw std::invalid_argument("stmg_transfer_create: null argument");
    auto t = std::make_unique<stmg_transfer>();
    t->t = std::make_unique<Transfer>(*fine->op, *coarse->op);
    *out = t.release();
  });
}
void stmg_transfer_destroy(stmg_transfer* t) { delete t; }
int stmg_transfer_prolong(const stmg_transfer* t, const double* d_c, double* d_f, void* stream) {
  return guard([&] {
    if (!t || !d_c || !d_f) throw std::invalid_argument("stmg_transfer_prolong: null argument");
    t->t->prolong(d_c, d_f, st(stream));
  });
}
int stmg_transfer_restrict(const stmg_transfer* t, const double* d_f, double* d_c, void* stream) {
  return guard([&] {
    if (!t || !d_f || !d_c) throw std::invalid_argument("stmg_transfer_restrict: null argument");
    t->t->restrict_(d_f, d_c, st(stream));
  });
}

void stmg_mg_options_default(stmg_mg_options* o) {
  const MultigridOptions d;
  o->n_smooth = d.n_smooth;
  o->direct_coarse_max = d.direct_coarse_max;
  o->coarse_rel_tol = d.coarse_rel_tol;
  o->coarse_max_iters = d.coarse_max_iters;
  o->eig_iters = d.eig_iters;
  o->seed = d.seed;
}

namespace {
MultigridOptions mg_opts(const stmg_mg_options* options) {
  MultigridOptions mo;
  if (options) {
    mo.n_smooth = options->n_smooth;
    mo.direct_coarse_max = options->direct_coarse_max;
    mo.coarse_rel_tol = options->coarse_rel_tol;
    mo.coarse_max_iters = options->coarse_max_iters;
    mo.eig_iters = options->eig_iters;
    mo.seed = options->seed;
  }
  return mo;
}
std::vector<LevelSpec> mg_plan(int scheme, int fine_mesh_level, int p, int k, int n_steps, double tau, int n_strategy,
                               const int* strategy) {
  const TimeScheme sch = static_cast<TimeScheme>(scheme);
  LevelSpec finest{fine_mesh_level, p, k, n_steps, tau, Coarsening::SpaceH};
  std::vector<Coarsening> strat;
  if (n_strategy < 0)
    strat = default_strategy(finest, sch);
  else
    for (int i = 0; i < n_strategy; ++i) strat.push_back(static_cast<Coarsening>(strategy[i]));
  return build_level_plan(finest, sch, strat);
}
}  // namespace

int stmg_multigrid_create(int equation, int scheme, const stmg_mesh* mesh, const double* coarse_cell_scale,
                          int fine_mesh_level, int p, int k, int n_steps, double tau, int n_strategy,
                          const int* strategy, const stmg_mg_options* options, stmg_multigrid** out) {
  return guard([&] {
    if (!mesh || !out) throw std::invalid_argument("stmg_multigrid_create: null argument");
    const TimeScheme sch = static_cast<TimeScheme>(scheme);
    LevelSpec finest{fine_mesh_level, p, k, n_steps, tau, Coarsening::SpaceH};
    std::vector<Coarsening> strat;
    if (n_strategy < 0)
      strat = default_strategy(finest, sch);
    else
      for (int i = 0; i < n_strategy; ++i) strat.push_back(static_cast<Coarsening>(strategy[i]));
    MultigridOptions mo;
    if (options) {
      mo.n_smooth = options->n_smooth;
      mo.direct_coarse_max = options->direct_coarse_max;
      mo.coarse_rel_tol = options->coarse_rel_tol;
      mo.coarse_max_iters = options->coarse_max_iters;
      mo.eig_iters = options->eig_iters;
      mo.seed = options->seed;
    }
    auto m = std::make_unique<stmg_multigrid>();
    m->mg = std::make_unique<SpaceTimeMultigrid>(static_cast<Equation>(equation), sch, mesh->h,
                                                 coeff(mesh->h, coarse_cell_scale),
                                                 build_level_plan(finest, sch, strat), mo);
    *out = m.release();
  });
}
void stmg_multigrid_destroy(stmg_multigrid* mg) { delete mg; }
int stmg_multigrid_n_levels(const stmg_multigrid* mg) { return mg ? mg->mg->n_levels() : -1; }
long long stmg_multigrid_smoother_bytes(const stmg_multigrid* mg, int level) {
  if (!mg || level < 0 || level + 1 >= mg->mg->n_levels()) return -1;
  return static_cast<long long>(mg->mg->smoother_at(level).bytes());
}
int stmg_multigrid_smoother_kind(const stmg_multigrid* mg, int level) {
  if (!mg || level < 0 || level + 1 >= mg->mg->n_levels()) return -1;
  return mg->mg->smoother_at(level).kind();
}

int stmg_multigrid_level_info(const stmg_multigrid* mg, int level, int ints[5], long long* n_dofs, double* omega) {
  return guard([&] {
    if (!mg || level < 0 || level >= mg->mg->n_levels()) throw std::invalid_argument("level_info: bad level");
    const LevelInfo li = mg->mg->level_info()[static_cast<size_t>(level)];
    ints[0] = li.mesh_level;
    ints[1] = li.p;
    ints[2] = li.k;
    ints[3] = li.n_steps;
    int c = -1;
    if (li.coarsening == "space-h") c = 0;
    if (li.coarsening == "space-p") c = 1;
    if (li.coarsening == "time-tau") c = 2;
    if (li.coarsening == "time-k") c = 3;
    ints[4] = c;
    *n_dofs = li.n_dofs;
    *omega = li.omega;
  });
}
int stmg_multigrid_set_omega(stmg_multigrid* mg, int level, double omega) {
  return guard([&] {
    if (!mg || level < 0 || level >= mg->mg->n_levels()) throw std::invalid_argument("set_omega: bad level");
    mg->mg->set_omega(level, omega);
  });
}
const stmg_st_operator* stmg_multigrid_operator_at(const stmg_multigrid* mg, int level) {
  if (!mg || level < 0 || level >= mg->mg->n_levels()) return nullptr;
  // wrapper objects that alias the multigrid's operators (never deleted by callers)
  auto* self = const_cast<stmg_multigrid*>(mg);
  if (self->views.empty()) {
    for (int l = 0; l < mg->mg->n_levels(); ++l) {
      auto v = std::make_unique<stmg_st_operator>();
      v->op = &mg->mg->operator_at(l);
      self->views.push_back(std::move(v));
    }
  }
  return self->views[static_cast<size_t>(level)].get();
}
int stmg_multigrid_apply(const stmg_multigrid* mg, const double* d_r, double* d_z, void* stream) {
  return guard([&] {
    if (!mg || !d_r || !d_z) throw std::invalid_argument("stmg_multigrid_apply: null argument");
    mg->mg->apply(d_r, d_z, st(stream));
  });
}
int stmg_multigrid_apply_host(const stmg_multigrid* mg, const double* h_r, double* h_z) {
  return guard([&] {
    if (!mg || !h_r || !h_z) throw std::invalid_argument("stmg_multigrid_apply_host: null argument");
    const size_t bytes = sizeof(double) * mg->mg->fine_operator().n_dofs();
    if (mg->hr.bytes() != bytes) {
      mg->hr.allocate(bytes);
      mg->hz.allocate(bytes);
    }
    copy_to_device(mg->hr.d(), h_r, bytes, nullptr);
    mg->mg->apply(mg->hr.d(), mg->hz.d(), nullptr);
    copy_to_host(h_z, mg->hz.d(), bytes, nullptr);
  });
}
int stmg_multigrid_smooth(const stmg_multigrid* mg, int level, const double* d_f, double* d_u, void* stream) {
  return guard([&] {
    if (!mg || level < 0 || level + 1 >= mg->mg->n_levels() + (mg->mg->n_levels() == 1 ? 1 : 0))
      throw std::invalid_argument("stmg_multigrid_smooth: bad level");
    mg->mg->smooth(level, d_f, d_u, st(stream));
  });
}
int stmg_multigrid_asm_add_correction(const stmg_multigrid* mg, int level, const double* d_r, double* d_z,
                                      void* stream) {
  return guard([&] {
    if (!mg || level < 0 || level >= mg->mg->n_levels()) throw std::invalid_argument("asm_add_correction: bad level");
    mg->mg->smoother_at(level).add_correction(d_r, d_z, st(stream));
  });
}
int stmg_multigrid_prolong(const stmg_multigrid* mg, int level, const double* d_c, double* d_f, void* stream) {
  return guard([&] {
    if (!mg || level < 0 || level + 1 >= mg->mg->n_levels()) throw std::invalid_argument("prolong: bad level");
    mg->mg->transfer_at(level).prolong(d_c, d_f, st(stream));
  });
}
int stmg_multigrid_restrict(const stmg_multigrid* mg, int level, const double* d_f, double* d_c, void* stream) {
  return guard([&] {
    if (!mg || level < 0 || level + 1 >= mg->mg->n_levels()) throw std::invalid_argument("restrict: bad level");
    mg->mg->transfer_at(level).restrict_(d_f, d_c, st(stream));
  });
}
long long stmg_multigrid_device_bytes(const stmg_multigrid* mg) {
  return mg ? static_cast<long long>(mg->mg->device_bytes()) : -1;
}

void stmg_gmres_options_default(stmg_gmres_options* o) {
  const GmresOptions d;
  o->max_iters = d.max_iters;
  o->restart = d.restart;
  o->rel_tol = d.rel_tol;
  o->abs_tol = d.abs_tol;
}

namespace {
GmresOptions gopts(const stmg_gmres_options* o) {
  GmresOptions g;
  if (o) {
    g.max_iters = o->max_iters;
    g.restart = o->restart;
    g.rel_tol = o->rel_tol;
    g.abs_tol = o->abs_tol;
  }
  return g;
}
void fill_result(const GmresResult& r, stmg_gmres_result* out, double* history, int cap) {
  if (out) {
    out->converged = r.converged ? 1 : 0;
    out->iterations = r.iterations;
    out->initial_residual = r.initial_residual;
    out->final_residual = r.final_residual;
    out->history_len = static_cast<int>(r.residual_history.size());
  }
  if (history)
    for (int i = 0; i < cap && i < static_cast<int>(r.residual_history.size()); ++i)
      history[i] = r.residual_history[static_cast<size_t>(i)];
}
thread_local GmresWorkspace g_ws;
}  // namespace

int stmg_gmres(long long n, stmg_linear_map op, void* op_ctx, stmg_linear_map precond, void* precond_ctx,
               const double* d_b, double* d_x, const stmg_gmres_options* options, stmg_gmres_result* result,
               double* history, int history_cap, void* stream) {
  return guard([&] {
    if (!op || !d_b || !d_x || n <= 0) throw std::invalid_argument("stmg_gmres: bad argument");
    DeviceMap A = [op, op_ctx](const double* in, double* out, cudaStream_t s) {
      if (op(op_ctx, in, out, s) != 0) throw std::runtime_error("stmg_gmres: operator callback failed");
    };
    DeviceMap M;
    if (precond)
      M = [precond, precond_ctx](const double* in, double* out, cudaStream_t s) {
        if (precond(precond_ctx, in, out, s) != 0) throw std::runtime_error("stmg_gmres: preconditioner failed");
      };
    const GmresResult r = gmres(A, d_b, d_x, n, gopts(options), M, g_ws, st(stream));
    fill_result(r, result, history, history_cap);
  });
}

int stmg_solve(const stmg_multigrid* mg, int precondition, const double* d_b, double* d_x,
               const stmg_gmres_options* options, stmg_gmres_result* result, double* history, int history_cap,
               void* stream) {
  return guard([&] {
    if (!mg || !d_b || !d_x) throw std::invalid_argument("stmg_solve: null argument");
    const SpaceTimeOperator& op = mg->mg->fine_operator();
    const SpaceTimeMultigrid* m = mg->mg.get();
    DeviceMap A = [&op](const double* in, double* out, cudaStream_t s) { op.apply(in, out, s); };
    DeviceMap M;
    if (precondition) M = [m](const double* in, double* out, cudaStream_t s) { m->apply(in, out, s); };
    const GmresResult r = gmres(A, d_b, d_x, op.n_dofs(), gopts(options), M, mg->ws, st(stream));
    fill_result(r, result, history, history_cap);
  });
}

int stmg_solve_host(const stmg_multigrid* mg, int precondition, const double* h_b, double* h_x,
                    const stmg_gmres_options* options, stmg_gmres_result* result, double* history, int history_cap) {
  return guard([&] {
    if (!mg || !h_b || !h_x) throw std::invalid_argument("stmg_solve_host: null argument");
    const size_t bytes = sizeof(double) * mg->mg->fine_operator().n_dofs();
    DeviceBuffer b(bytes), x(bytes);
    copy_to_device(b.d(), h_b, bytes, nullptr);
    copy_to_device(x.d(), h_x, bytes, nullptr);
    const int rc = stmg_solve(mg, precondition, b.d(), x.d(), options, result, history, history_cap, nullptr);
    if (rc != 0) throw std::runtime_error(g_err);
    copy_to_host(h_x, x.d(), bytes, nullptr);
  });
}

}  // extern "C"

extern "C" {

int stmg_st_operator_error_norms(const stmg_st_operator* op, const double* d_x, const double* d_u0, double frequency,
                                 double t0, double out[3]) {
  return guard([&] {
    if (!op || !d_x || !d_u0 || !out) throw std::invalid_argument("stmg_st_operator_error_norms: null argument");
    ErrorRecord acc;
    accumulate_errors(*op->op, d_x, d_u0, frequency, t0, acc, nullptr);
    out[0] = std::sqrt(acc.l2_l2);
    out[1] = acc.linf_l2;
    out[2] = acc.linf_linf;
  });
}

int stmg_march(const stmg_multigrid* mg, int n_batches, int source_kind, double frequency, double* d_u, double* d_v,
               const stmg_gmres_options* options, int* iterations, double errors[3], void* stream) {
  bool converged = true;
  const int rc = guard([&] {
    if (!mg || !d_u || !iterations) throw std::invalid_argument("stmg_march: null argument");
    const MarchResult r = march(*mg->mg, n_batches, source_kind, frequency, d_u, d_v, gopts(options),
                                errors != nullptr, st(stream));
    for (int b = 0; b < n_batches; ++b)
      iterations[b] = b < static_cast<int>(r.iterations.size()) ? r.iterations[static_cast<size_t>(b)] : 0;
    if (errors) {
      errors[0] = r.error_u.l2_l2;
      errors[1] = r.error_u.linf_l2;
      errors[2] = r.error_u.linf_linf;
    }
    converged = r.converged;
  });
  if (rc == 0 && !converged) {
    g_err = "stmg_march: a batch did not converge";
    return -2;
  }
  return rc;
}

int stmg_march_probes(const stmg_multigrid* mg, int n_batches, int source_kind, double frequency, double* d_u,
                      double* d_v, const stmg_gmres_options* options, int* iterations, double errors[3], int n_probes,
                      const double* probe_xyz, int samples_per_step, double* times, double* values, void* stream) {
  bool converged = true;
  const int rc = guard([&] {
    if (!mg || !d_u || !iterations) throw std::invalid_argument("stmg_march_probes: null argument");
    if (n_probes < 0 || (n_probes > 0 && (!probe_xyz || !times || !values)) || samples_per_step < 1)
      throw std::invalid_argument("stmg_march_probes: bad probe arguments");
    ProbeSpec ps;
    ps.xyz.assign(probe_xyz, probe_xyz + 3 * n_probes);
    ps.samples_per_step = samples_per_step;
    const MarchResult r = march(*mg->mg, n_batches, source_kind, frequency, d_u, d_v, gopts(options),
                                errors != nullptr, st(stream), n_probes > 0 ? &ps : nullptr);
    for (int b = 0; b < n_batches; ++b)
      iterations[b] = b < static_cast<int>(r.iterations.size()) ? r.iterations[static_cast<size_t>(b)] : 0;
    if (errors) {
      errors[0] = r.error_u.l2_l2;
      errors[1] = r.error_u.linf_l2;
      errors[2] = r.error_u.linf_linf;
    }
    const size_t ns = r.probe_times.size();
    for (size_t i = 0; i < ns; ++i) times[i] = r.probe_times[i];
    for (int p = 0; p < n_probes; ++p)
      for (size_t i = 0; i < ns; ++i) values[static_cast<size_t>(p) * ns + i] = r.probe_values[static_cast<size_t>(p)][i];
    converged = r.converged;
  });
  if (rc == 0 && !converged) {
    g_err = "stmg_march_probes: a batch did not converge";
    return -2;
  }
  return rc;
}

namespace {
ProblemSpec problem_spec(const stmg_problem* p) {
  if (!p) throw std::invalid_argument("stmg_problem: null argument");
  if (p->equation < 0 || p->equation > 1 || p->scheme < 0 || p->scheme > 1 || p->problem < 0 || p->problem > 2)
    throw std::invalid_argument("stmg_problem: bad equation, scheme or problem");
  if (p->n_strategy < 0 || p->n_strategy > 32) throw std::invalid_argument("stmg_problem: bad strategy length");
  ProblemSpec s;
  s.equation = static_cast<Equation>(p->equation);
  s.scheme = static_cast<TimeScheme>(p->scheme);
  s.problem = static_cast<ProblemKind>(p->problem);
  s.k = p->k;
  s.p = p->p;
  s.dim = p->dim;
  for (int a = 0; a < 3; ++a) {
    s.lo[a] = p->lo[a];
    s.hi[a] = p->hi[a];
  }
  s.t_final = p->t_final;
  s.refinements = p->refinements;
  s.base_cells = p->base_cells;
  s.base_time_intervals = p->base_time_intervals;
  s.batch = p->batch;
  s.frequency = p->frequency;
  s.shm_s = p->shm_s;
  s.perturb = p->perturb;
  s.seed = p->seed;
  s.rho_random_lo = p->rho_random_lo;
  s.rho_random_hi = p->rho_random_hi;
  s.abs_tol = p->abs_tol;
  s.rel_tol = p->rel_tol;
  s.max_iters = p->max_iters;
  s.restart = p->restart;
  s.n_smooth = p->n_smooth;
  s.precondition = p->precondition != 0;
  s.probe_samples_per_step = p->probe_samples_per_step;
  for (int i = 0; i < p->n_strategy; ++i) {
    if (p->strategy[i] < 0 || p->strategy[i] > 3) throw std::invalid_argument("stmg_problem: unknown coarsening");
    s.strategy.push_back(static_cast<Coarsening>(p->strategy[i]));
  }
  s.timers = p->timers != 0;
  return s;
}
int coarsening_code(const std::string& name) {
  if (name == "space-h") return 0;
  if (name == "space-p") return 1;
  if (name == "time-tau") return 2;
  if (name == "time-k") return 3;
  return -1;  // "finest"
}
}  // namespace

int stmg_problem_sizes(const stmg_problem* spec, int* n_steps_total, int* n_batches, long long* n_probe_samples) {
  return guard_host([&] {
    const ProblemSpec s = problem_spec(spec);
    if (s.refinements < 0 || s.refinements > 24 || s.base_time_intervals < 1)
      throw std::invalid_argument("stmg_problem_sizes: bad refinements or time intervals");
    const int nst = s.base_time_intervals << (s.refinements + 1);
    if (s.batch < 1 || nst % s.batch != 0) throw std::invalid_argument("march: batch must divide the step count");
    if (n_steps_total) *n_steps_total = nst;
    if (n_batches) *n_batches = nst / s.batch;
    if (n_probe_samples) *n_probe_samples = 1 + static_cast<long long>(nst) * std::max(0, s.probe_samples_per_step);
  });
}

int stmg_run(const stmg_problem* spec, int n_probes, const double* probe_xyz, stmg_run_report* report, int batch_cap,
             int* batch_iterations, double* batch_residuals, int* batch_converged, int level_cap, int* level_ints,
             long long* level_dofs, double* level_omega, long long probe_cap, double* probe_times,
             double* probe_values) {
  return guard([&] {
    if (!report) throw std::invalid_argument("stmg_run: null report");
    if (n_probes < 0 || (n_probes > 0 && (!probe_xyz || !probe_times || !probe_values)))
      throw std::invalid_argument("stmg_run: bad probe arguments");
    const ProblemSpec s = problem_spec(spec);
    if (n_probes > 0 && s.probe_samples_per_step < 1)
      throw std::invalid_argument("stmg_run: probe_samples_per_step must be >= 1");
    const std::vector<double> probes(probe_xyz, probe_xyz + 3 * n_probes);
    const RunReport r = run_march(s, probes, nullptr);
    std::memset(report, 0, sizeof(*report));
    report->converged = r.converged ? 1 : 0;
    report->n_space_dofs = r.n_space_dofs;
    report->n_steps_total = r.n_steps_total;
    report->n_batches = r.n_batches;
    report->dofs_global = r.dofs_global;
    report->n_batches_run = static_cast<int>(r.batches.size());
    report->mean_iterations = r.mean_iterations;
    report->work = r.work;
    report->has_error_u = r.has_error_u ? 1 : 0;
    report->has_error_v = r.has_error_v ? 1 : 0;
    const ErrorRecord* er[2] = {&r.error_u, &r.error_v};
    double* eo[2] = {report->error_u, report->error_v};
    for (int i = 0; i < 2; ++i) {
      eo[i][0] = er[i]->l2_l2;
      eo[i][1] = er[i]->linf_l2;
      eo[i][2] = er[i]->linf_linf;
    }
    report->n_levels = static_cast<int>(r.hierarchy.size());
    report->sections[0] = r.sections.total;
    report->sections[1] = r.sections.smoother;
    report->sections[2] = r.sections.gmg_wo_smoother;
    report->sections[3] = r.sections.operator_wo_gmg;
    report->sections[4] = r.sections.other;
    report->n_probe_samples = static_cast<long long>(r.probe_times.size());
    for (int b = 0; b < std::min(batch_cap, report->n_batches_run); ++b) {
      const BatchStats& bs = r.batches[static_cast<size_t>(b)];
      if (batch_iterations) batch_iterations[b] = bs.iterations;
      if (batch_residuals) batch_residuals[b] = bs.final_residual;
      if (batch_converged) batch_converged[b] = bs.converged ? 1 : 0;
    }
    for (int l = 0; l < std::min(level_cap, report->n_levels); ++l) {
      const LevelInfo& li = r.hierarchy[static_cast<size_t>(l)];
      if (level_ints) {
        int* o = level_ints + 5 * l;
        o[0] = coarsening_code(li.coarsening);
        o[1] = li.mesh_level;
        o[2] = li.p;
        o[3] = li.k;
        o[4] = li.n_steps;
      }
      if (level_dofs) level_dofs[l] = li.n_dofs;
      if (level_omega) level_omega[l] = li.omega;
    }
    const long long ns = std::min<long long>(probe_cap, report->n_probe_samples);
    for (long long i = 0; i < ns && n_probes > 0; ++i) probe_times[i] = r.probe_times[static_cast<size_t>(i)];
    for (int p = 0; p < n_probes; ++p)
      for (long long i = 0; i < ns; ++i)
        probe_values[static_cast<long long>(p) * probe_cap + i] =
            r.probe_values[static_cast<size_t>(p)][static_cast<size_t>(i)];
  });
}

int stmg_level_plan(int scheme, int fine_mesh_level, int p, int k, int n_steps, double tau, int n_strategy,
                    const int* strategy, int cap, int* n_levels, int* ints, double* taus) {
  return guard_host([&] {
    if (!n_levels || (n_strategy > 0 && !strategy)) throw std::invalid_argument("stmg_level_plan: null argument");
    if (scheme < 0 || scheme > 1) throw std::invalid_argument("stmg_level_plan: bad scheme");
    for (int i = 0; i < n_strategy; ++i)
      if (strategy[i] < 0 || strategy[i] > 3) throw std::invalid_argument("stmg_level_plan: unknown coarsening");
    const auto plan = mg_plan(scheme, fine_mesh_level, p, k, n_steps, tau, n_strategy, strategy);
    *n_levels = static_cast<int>(plan.size());
    for (int l = 0; l < std::min(cap, *n_levels); ++l) {
      const LevelSpec& ls = plan[static_cast<size_t>(l)];
      if (ints) {
        int* o = ints + 5 * l;
        o[0] = l == 0 ? -1 : static_cast<int>(ls.from_finer);
        o[1] = ls.mesh_level;
        o[2] = ls.p;
        o[3] = ls.k;
        o[4] = ls.n_steps;
      }
      if (taus) taus[l] = ls.tau;
    }
  });
}

int stmg_perturbed_vertices(int dim, const double lo[3], const double hi[3], int base_cells, int refinements,
                            double magnitude, unsigned long long seed, double* xyz) {
  return guard_host([&] {
    if (!lo || !hi || !xyz) throw std::invalid_argument("stmg_perturbed_vertices: null argument");
    MeshHierarchy m = make_cartesian(dim, {lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}, base_cells, refinements);
    const MeshLevel& f = m.levels.back();
    perturb_mesh(m, magnitude, seed);
    if (f.vertices.empty()) {
      // magnitude 0: the Cartesian lattice
      const auto n = f.n_verts_axis();
      for (Index kk = 0; kk < n[2]; ++kk)
        for (Index j = 0; j < n[1]; ++j)
          for (Index i = 0; i < n[0]; ++i) {
            const Index vi = (kk * n[1] + j) * n[0] + i, idx[3] = {i, j, kk};
            for (int a = 0; a < 3; ++a) xyz[3 * vi + a] = a < dim ? cartesian_coord(f, a, idx[a]) : 0.0;
          }
    } else {
      std::copy(f.vertices.begin(), f.vertices.end(), xyz);
    }
  });
}

int stmg_nccl_unique_id(char id[128]) {
  return guard_host([&] {
    if (!id) throw std::invalid_argument("stmg_nccl_unique_id: null argument");
    const std::string u = NcclComm::unique_id();
    std::memcpy(id, u.data(), 128);
  });
}
int stmg_comm_create(int world, int rank, const char id[128], stmg_comm** out) {
  return guard([&] {
    if (!id || !out) throw std::invalid_argument("stmg_comm_create: null argument");
    auto c = std::make_unique<stmg_comm>();
    c->c = std::make_unique<NcclComm>(world, rank, std::string(id, 128));
    *out = c.release();
  });
}
void stmg_comm_destroy(stmg_comm* c) { delete c; }
int stmg_comm_create_host(int world, int rank, const stmg_host_transport* transport, stmg_comm** out) {
  return guard_host([&] {
    if (!transport || !out) throw std::invalid_argument("stmg_comm_create_host: null argument");
    HostTransport t;
    t.ctx = transport->ctx;
    t.allreduce_sum = transport->allreduce_sum;
    t.sendrecv = transport->sendrecv;
    auto c = std::make_unique<stmg_comm>();
    c->c = std::make_unique<HostComm>(world, rank, t);
    *out = c.release();
  });
}

int stmg_slab_plan(int scheme, int fine_mesh_level, int p, int k, int n_steps, long long cells_z, int n_parts,
                   int* dist_levels, int* n_levels) {
  return guard_host([&] {
    if (!dist_levels || !n_levels) throw std::invalid_argument("stmg_slab_plan: null argument");
    const auto plan = mg_plan(scheme, fine_mesh_level, p, k, n_steps, 1.0, -1, nullptr);
    const SlabPlan sp = make_slab_plan(plan, cells_z, fine_mesh_level, n_parts);
    *dist_levels = sp.dist_levels;
    *n_levels = static_cast<int>(plan.size());
  });
}

int stmg_slab_multigrid_create(int equation, int scheme, const stmg_mesh* mesh, const double* coarse_cell_scale,
                               int fine_mesh_level, int p, int k, int n_steps, double tau, int n_strategy,
                               const int* strategy, const stmg_mg_options* options, int n_parts, int first_part,
                               int local_parts, const stmg_comm* comm, stmg_slab_multigrid** out) {
  return guard([&] {
    if (!mesh || !out) throw std::invalid_argument("stmg_slab_multigrid_create: null argument");
    auto m = std::make_unique<stmg_slab_multigrid>();
    m->mg = std::make_unique<SlabMultigrid>(
        static_cast<Equation>(equation), static_cast<TimeScheme>(scheme), mesh->h, coeff(mesh->h, coarse_cell_scale),
        mg_plan(scheme, fine_mesh_level, p, k, n_steps, tau, n_strategy, strategy), mg_opts(options), n_parts,
        first_part, local_parts, comm ? comm->c.get() : nullptr);
    *out = m.release();
  });
}
void stmg_slab_multigrid_destroy(stmg_slab_multigrid* mg) { delete mg; }
long long stmg_slab_multigrid_local_dofs(const stmg_slab_multigrid* mg) { return mg ? mg->mg->local_dofs() : -1; }
int stmg_slab_multigrid_info(const stmg_slab_multigrid* mg, int info[2]) {
  return guard_host([&] {
    if (!mg || !info) throw std::invalid_argument("stmg_slab_multigrid_info: null argument");
    info[0] = mg->mg->dist_levels();
    info[1] = mg->mg->n_levels();
  });
}
int stmg_slab_multigrid_part(const stmg_slab_multigrid* mg, int i, long long* offset, long long* n_dofs,
                             long long* plane0) {
  return guard_host([&] {
    if (!mg || !offset || !n_dofs || !plane0) throw std::invalid_argument("stmg_slab_multigrid_part: null argument");
    if (i < 0 || i >= mg->mg->local_parts()) throw std::invalid_argument("stmg_slab_multigrid_part: bad part");
    *offset = mg->mg->part_offset(i);
    *n_dofs = mg->mg->part_dofs(i);
    *plane0 = mg->mg->part_plane0(i);
  });
}
double stmg_slab_multigrid_omega(const stmg_slab_multigrid* mg, int level) {
  try {
    return mg ? mg->mg->omega_at(level) : -1.0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}
int stmg_slab_multigrid_set_omega(stmg_slab_multigrid* mg, int level, double omega) {
  return guard_host([&] {
    if (!mg) throw std::invalid_argument("stmg_slab_multigrid_set_omega: null argument");
    mg->mg->set_omega(level, omega);
  });
}
int stmg_slab_multigrid_apply(const stmg_slab_multigrid* mg, const double* d_u, double* d_y, void* stream) {
  return guard([&] {
    if (!mg || !d_u || !d_y) throw std::invalid_argument("stmg_slab_multigrid_apply: null argument");
    mg->mg->apply(d_u, d_y, st(stream));
  });
}
int stmg_slab_multigrid_vcycle(const stmg_slab_multigrid* mg, const double* d_r, double* d_z, void* stream) {
  return guard([&] {
    if (!mg || !d_r || !d_z) throw std::invalid_argument("stmg_slab_multigrid_vcycle: null argument");
    mg->mg->vcycle(d_r, d_z, st(stream));
  });
}
int stmg_slab_multigrid_asm_add_correction(const stmg_slab_multigrid* mg, const double* d_r, double* d_z,
                                           void* stream) {
  return guard([&] {
    if (!mg || !d_r || !d_z) throw std::invalid_argument("stmg_slab_multigrid_asm_add_correction: null argument");
    mg->mg->asm_add_correction(d_r, d_z, st(stream));
  });
}
int stmg_slab_multigrid_solve(const stmg_slab_multigrid* mg, const double* d_b, double* d_x,
                              const stmg_gmres_options* options, stmg_gmres_result* result, void* stream) {
  return guard([&] {
    if (!mg || !d_b || !d_x) throw std::invalid_argument("stmg_slab_multigrid_solve: null argument");
    const GmresResult r = mg->mg->solve(d_b, d_x, gopts(options), st(stream));
    if (result) fill_result(r, result, nullptr, 0);
  });
}
int stmg_slab_multigrid_dot(const stmg_slab_multigrid* mg, const double* d_a, const double* d_b, double* out) {
  return guard([&] {
    if (!mg || !d_a || !d_b || !out) throw std::invalid_argument("stmg_slab_multigrid_dot: null argument");
    *out = mg->mg->dot(d_a, d_b, nullptr);
  });
}
int stmg_slab_multigrid_scatter(const stmg_slab_multigrid* mg, const double* d_full, double* d_local, void* stream) {
  return guard([&] {
    if (!mg || !d_full || !d_local) throw std::invalid_argument("stmg_slab_multigrid_scatter: null argument");
    mg->mg->scatter(d_full, d_local, st(stream));
  });
}
int stmg_slab_multigrid_gather(const stmg_slab_multigrid* mg, const double* d_local, double* d_full, void* stream) {
  return guard([&] {
    if (!mg || !d_local || !d_full) throw std::invalid_argument("stmg_slab_multigrid_gather: null argument");
    mg->mg->gather(d_local, d_full, st(stream));
  });
}

}  // extern "C"
