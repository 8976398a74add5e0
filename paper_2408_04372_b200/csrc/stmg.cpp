// Host C++ layer of the B200 STMG path (see stmg.hpp for the interface map).
#include "stmg.hpp"

#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

namespace stmgb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {
void solver_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS) throw std::runtime_error(std::string(what) + ": cusolver status " + std::to_string(s));
}
template <typename T>
DeviceBuffer upload(const std::vector<T>& v) {
  DeviceBuffer b(sizeof(T) * std::max<size_t>(v.size(), 1));
  if (!v.empty()) cuda_check(cudaMemcpy(b.raw(), v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice), "upload");
  return b;
}
double host_dot(const double* a, const double* b, Index n, cudaStream_t s, DeviceBuffer& ptrs, DeviceBuffer& scratch,
                DeviceBuffer& out) {
  const double* hp[1] = {a};
  cuda_check(cudaMemcpyAsync(ptrs.raw(), hp, sizeof(hp), cudaMemcpyHostToDevice, s), "dot ptrs");
  vec_multidot(static_cast<const double* const*>(ptrs.raw()), 1, b, n, out.d(), scratch.d(), s);
  double r = 0.0;
  cuda_check(cudaMemcpyAsync(&r, out.d(), sizeof(double), cudaMemcpyDeviceToHost, s), "dot result");
  cuda_check(cudaStreamSynchronize(s), "dot sync");
  return r;
}
}  // namespace

// ------------------------------------------------------------------ buffers
DeviceBuffer::DeviceBuffer(size_t bytes) { allocate(bytes); }
DeviceBuffer::~DeviceBuffer() { release(); }
DeviceBuffer::DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), bytes_(o.bytes_) {
  o.p_ = nullptr;
  o.bytes_ = 0;
}
DeviceBuffer& DeviceBuffer::operator=(DeviceBuffer&& o) noexcept {
  if (this != &o) {
    release();
    p_ = o.p_;
    bytes_ = o.bytes_;
    o.p_ = nullptr;
    o.bytes_ = 0;
  }
  return *this;
}
void DeviceBuffer::allocate(size_t bytes) {
  release();
  if (bytes == 0) bytes = 8;
  cuda_check(cudaMalloc(&p_, bytes), "cudaMalloc");
  bytes_ = bytes;
}
void DeviceBuffer::release() {
  if (p_) cudaFree(p_);
  p_ = nullptr;
  bytes_ = 0;
}

// ------------------------------------------------------ SpaceTimeOperator
SpaceTimeOperator::SpaceTimeOperator(Equation equation, const TemporalWeights& weights, double tau, int n_steps,
                                     const MeshHierarchy& mesh, int mesh_level, int p, const Coefficient& rho)
    : equation_(equation), weights_(weights), tau_(tau), n_steps_(n_steps), mesh_level_(mesh_level), p_(p) {
  if (tau <= 0.0 || n_steps < 1) throw std::invalid_argument("SpaceTimeOperator: bad tau or n_steps");
  if (mesh_level < 0 || mesh_level >= mesh.n_levels()) throw std::invalid_argument("SpaceTimeOperator: bad level");
  if (p < 1 || p + 1 > kMaxN) throw std::invalid_argument("SpaceTimeOperator: p must be in [1, 4]");
  const int F = n_steps * weights.n_t;
  if (F > kMaxWideF) throw std::invalid_argument("SpaceTimeOperator: n_steps * n_t must be <= 64");
  wide_ = F > kMaxF;
  const MeshLevel& m = mesh.levels[static_cast<size_t>(mesh_level)];
  mesh_level_ptr_ = &m;
  if (m.dim < 2 || m.dim > 3) throw std::invalid_argument("SpaceTimeOperator: dim must be 2 or 3");
  DevLevel& d = desc_;
  d.dim = m.dim;
  d.p = p;
  d.n = p + 1;
  d.S = n_steps;
  d.nt = weights.n_t;
  d.F = F;
  d.n_space = 1;
  for (int a = 0; a < 3; ++a) {
    d.cells[a] = a < m.dim ? m.cells[a] : 1;
    d.dofs[a] = a < m.dim ? m.cells[a] * p + 1 : 1;
    d.n_space *= d.dofs[a];
    d.h[a] = a < m.dim ? (m.hi[a] - m.lo[a]) / static_cast<double>(m.cells[a]) : 1.0;
    d.lo[a] = m.lo[a];
  }
  d.n_dofs = d.n_space * F;
  d.zbc = m.dim == 3 ? m.zbc : 3;
  d.cz0 = m.dim == 3 ? m.cz0 : 0;
  if (!m.vertices.empty()) {
    verts_ = upload(m.vertices);
    d.verts = verts_.d();
  } else {
    d.verts = nullptr;
  }
  if (!rho.coarse_cell_scale.empty()) {
    const MeshLevel& m0 = mesh.levels.front();
    std::array<Index, 3> c0 = m0.cells;
    if (mesh.global_cells0[0] > 0) c0 = mesh.global_cells0;
    if (static_cast<Index>(rho.coarse_cell_scale.size()) != c0[0] * c0[1] * c0[2])
      throw std::invalid_argument("SpaceTimeOperator: coefficient needs one value per level-0 cell");
    for (double v : rho.coarse_cell_scale)
      if (!(v > 0.0)) throw std::runtime_error("CoefficientField: non-positive value");
    rho0_ = upload(rho.coarse_cell_scale);
    d.rho0 = rho0_.d();
    d.rho_shift = mesh_level;
    for (int a = 0; a < 3; ++a) d.cells0[a] = a < m.dim ? c0[a] : 1;
    d.rho_zonly = 1;
    const Index layer = c0[0] * c0[1];
    for (size_t i = 0; i < rho.coarse_cell_scale.size(); ++i)
      if (rho.coarse_cell_scale[i] != rho.coarse_cell_scale[(i / layer) * layer]) d.rho_zonly = 0;
  } else {
    d.rho0 = nullptr;
    d.rho_zonly = 1;
  }
  const Rule q = gauss(d.n);
  const Rule gl = gauss_lobatto(d.n);
  for (int i = 0; i < kMaxN; ++i)
    for (int j = 0; j < kMaxN; ++j) {
      d.B[i][j] = (i < d.n && j < d.n) ? lagrange_eval(gl.x, j, q.x[i]) : 0.0;
      d.Dq[i][j] = (i < d.n && j < d.n) ? lagrange_deriv(q.x, j, q.x[i]) : 0.0;
      d.D[i][j] = (i < d.n && j < d.n) ? lagrange_deriv(gl.x, j, q.x[i]) : 0.0;
    }
  for (int i = 0; i < kMaxN; ++i) {
    d.w[i] = i < d.n ? q.w[i] : 0.0;
    d.xq[i] = i < d.n ? q.x[i] : 0.0;
    d.gl[i] = i < d.n ? gl.x[i] : 0.0;
  }
  for (int i = 0; i < kMaxN; ++i)
    for (int j = 0; j < kMaxN; ++j) {
      double mr = 0.0, kr = 0.0;
      for (int k = 0; k < d.n; ++k) {
        mr += d.w[k] * d.B[k][i] * d.B[k][j];
        kr += d.w[k] * d.D[k][i] * d.D[k][j];
      }
      d.Mr[i][j] = mr;
      d.Kr[i][j] = kr;
    }
  for (int a = 0; a < 3; ++a) d.hinv2[a] = 1.0 / (d.h[a] * d.h[a]);
  std::memset(d.MrE, 0, sizeof(d.MrE));
  std::memset(d.MrO, 0, sizeof(d.MrO));
  std::memset(d.KrE, 0, sizeof(d.KrE));
  std::memset(d.KrO, 0, sizeof(d.KrO));
  {
    const int n = d.n, H = n / 2, HE = (n + 1) / 2;
    for (int i = 0; i < HE; ++i)
      for (int k = 0; k < HE; ++k) {
        const bool mid = (n % 2 == 1) && k == H;
        d.MrE[i][k] = mid ? d.Mr[i][k] : 0.5 * (d.Mr[i][k] + d.Mr[i][n - 1 - k]);
        d.KrE[i][k] = mid ? d.Kr[i][k] : 0.5 * (d.Kr[i][k] + d.Kr[i][n - 1 - k]);
      }
    for (int i = 0; i < H; ++i)
      for (int k = 0; k < H; ++k) {
        d.MrO[i][k] = 0.5 * (d.Mr[i][k] - d.Mr[i][n - 1 - k]);
        d.KrO[i][k] = 0.5 * (d.Kr[i][k] - d.Kr[i][n - 1 - k]);
      }
  }
  std::vector<double> CM, CA;
  block_coefficient_matrices(equation, weights, tau, n_steps, CM, CA);
  std::memset(d.CM, 0, sizeof(d.CM));
  std::memset(d.CA, 0, sizeof(d.CA));
  if (!wide_) {
    std::copy(CM.begin(), CM.end(), d.CM);
    std::copy(CA.begin(), CA.end(), d.CA);
    // G = CA^-1 CM when CA is well conditioned (Gauss-Jordan with partial
    // pivoting; the ratio of the extreme pivots bounds the conditioning)
    d.g_ok = 0;
    std::memset(d.G, 0, sizeof(d.G));
    {
      std::vector<double> a(CA), g(CM);
      double pmax = 0.0, pmin = 1e300;
      bool ok = true;
      for (int k = 0; k < F && ok; ++k) {
        int piv = k;
        for (int i = k + 1; i < F; ++i)
          if (std::abs(a[static_cast<size_t>(i * F + k)]) > std::abs(a[static_cast<size_t>(piv * F + k)])) piv = i;
        const double pv = a[static_cast<size_t>(piv * F + k)];
        if (pv == 0.0) {
          ok = false;
          break;
        }
        pmax = std::max(pmax, std::abs(pv));
        pmin = std::min(pmin, std::abs(pv));
        for (int j = 0; j < F; ++j) {
          std::swap(a[static_cast<size_t>(k * F + j)], a[static_cast<size_t>(piv * F + j)]);
          std::swap(g[static_cast<size_t>(k * F + j)], g[static_cast<size_t>(piv * F + j)]);
        }
        for (int i = 0; i < F; ++i) {
          if (i == k) continue;
          const double m = a[static_cast<size_t>(i * F + k)] / a[static_cast<size_t>(k * F + k)];
          if (m == 0.0) continue;
          for (int j = 0; j < F; ++j) {
            a[static_cast<size_t>(i * F + j)] -= m * a[static_cast<size_t>(k * F + j)];
            g[static_cast<size_t>(i * F + j)] -= m * g[static_cast<size_t>(k * F + j)];
          }
        }
      }
      if (ok && pmax / pmin < 1e6) {
        for (int i = 0; i < F; ++i)
          for (int j = 0; j < F; ++j) d.G[i * F + j] = g[static_cast<size_t>(i * F + j)] / a[static_cast<size_t>(i * F + i)];
        d.g_ok = 1;
      }
    }
  } else {
    // the fused kernels hold at most kMaxF fields: wide batches compose 2F
    // single-field applications (st_apply_wide) with the full tables
    wide_cm_ = upload(CM);
    wide_ca_ = upload(CA);
    wide_mu_.allocate(sizeof(double) * static_cast<size_t>(d.n_dofs));
    wide_au_.allocate(sizeof(double) * static_cast<size_t>(d.n_dofs));
  }
  cm_ = CM;
  ca_ = CA;
  // single-field spatial mass / stiffness (SpatialOperator::apply)
  mass_desc_ = desc_;
  mass_desc_.S = mass_desc_.nt = mass_desc_.F = 1;
  mass_desc_.n_dofs = d.n_space;
  std::memset(mass_desc_.CM, 0, sizeof(mass_desc_.CM));
  std::memset(mass_desc_.CA, 0, sizeof(mass_desc_.CA));
  mass_desc_.g_ok = 0;  // single-field tables: the direct CM / CA coupling
  std::memset(mass_desc_.G, 0, sizeof(mass_desc_.G));
  stiff_desc_ = mass_desc_;
  mass_desc_.CM[0] = 1.0;
  stiff_desc_.CA[0] = 1.0;
}

void SpaceTimeOperator::apply(const double* u, double* y, cudaStream_t stream) const {
  ++apply_count_;
  if (wide_)
    st_apply_wide(desc_, mass_desc_, stiff_desc_, wide_cm_.d(), wide_ca_.d(), nullptr, u, y, wide_mu_.d(),
                  wide_au_.d(), stream);
  else
    st_apply(desc_, u, y, stream);
}

void SpaceTimeOperator::residual(const double* f, const double* u, double* r, cudaStream_t stream) const {
  ++apply_count_;
  if (wide_)
    st_apply_wide(desc_, mass_desc_, stiff_desc_, wide_cm_.d(), wide_ca_.d(), f, u, r, wide_mu_.d(), wide_au_.d(),
                  stream);
  else
    st_residual(desc_, f, u, r, stream);
}

void SpaceTimeOperator::spatial_apply(int kind, const double* u, double* y, cudaStream_t stream) const {
  st_apply(kind == 0 ? mass_desc_ : stiff_desc_, u, y, stream);
}

// --------------------------------------------- slab RHS and state transfer
namespace {
struct WaveHelpers {
  std::vector<double> am_alpha, alpha_a, minv_a_last;
  double minv_alpha_last = 0.0, minv_beta_last = 0.0;
};
// the velocity-elimination helpers of space_time_operator.cpp:22-33
WaveHelpers wave_helpers(const TemporalWeights& w) {
  const int nt = w.n_t;
  WaveHelpers h;
  const std::vector<double> minv = invert_small(w.m, nt);
  const std::vector<double> minv_a = matmul_small(minv, w.a, nt, nt, nt);
  const std::vector<double> minv_alpha = matmul_small(minv, w.alpha, nt, nt, 1);
  h.am_alpha = matmul_small(w.a, minv_alpha, nt, nt, 1);
  h.minv_a_last.assign(minv_a.begin() + (nt - 1) * nt, minv_a.begin() + nt * nt);
  h.minv_alpha_last = minv_alpha[nt - 1];
  h.alpha_a.assign(nt, 0.0);
  if (w.scheme == TimeScheme::CGP) {
    const std::vector<double> minv_beta = matmul_small(minv, w.beta, nt, nt, 1);
    const std::vector<double> a_minv_beta = matmul_small(w.a, minv_beta, nt, nt, 1);
    h.minv_beta_last = minv_beta[nt - 1];
    for (int i = 0; i < nt; ++i) h.alpha_a[i] = w.alpha[i] - a_minv_beta[i];
  }
  return h;
}
}  // namespace

void SpaceTimeOperator::interpolate(int kind, double frequency, double t, const double* centre, double width,
                                    bool zero_boundary, double* out, cudaStream_t s) const {
  interpolate_nodes(desc_, kind, 2.0 * M_PI * frequency, t, centre, width, zero_boundary, out, s);
}

void SpaceTimeOperator::assemble_rhs(int source_kind, double frequency, double t0, const double* u0,
                                     const double* v0, double* rhs, cudaStream_t s) const {
  const int S = n_steps_, nt = weights_.n_t;
  const Index nx = n_space();
  const bool cgp = weights_.scheme == TimeScheme::CGP;
  const bool wave = equation_ == Equation::Wave;
  const TemporalWeights& w = weights_;
  if (wave && !v0) throw std::invalid_argument("assemble_rhs: the wave equation needs the entering velocity");
  vec_fill(rhs, 0.0, n_dofs(), s);
  DeviceBuffer fi(sizeof(double) * nx), Fl(sizeof(double) * nx), Ft(sizeof(double) * nx * nt);
  auto seg = [&](int step, int i) { return rhs + block_offset(step, i); };
  // source collocated at the temporal unknown nodes (space_time_operator.cpp:148-173)
  if (source_kind != 0) {
    const int kind = wave ? 1 : 0;
    auto mass_of = [&](double t, double* out) {
      interpolate(kind, frequency, t, nullptr, 0.0, /*zero_boundary=*/true, fi.d(), s);
      spatial_apply(0, fi.d(), out, s);
    };
    for (int st = 0; st < S; ++st) {
      const double t_left = t0 + st * tau_;
      for (int j = 0; j < nt; ++j) mass_of(t_left + w.unknown_nodes[j] * tau_, Ft.d() + j * nx);
      if (cgp) mass_of(t_left, Fl.d());
      for (int i = 0; i < nt; ++i) {
        for (int j = 0; j < nt; ++j) vec_axpy(seg(st, i), tau_ * w.m[i * nt + j], Ft.d() + j * nx, nx, s);
        if (cgp) vec_axpy(seg(st, i), tau_ * w.beta[i], Fl.d(), nx, s);
      }
    }
  }
  // coupling to the entering state (space_time_operator.cpp:175-218)
  DeviceBuffer uz(sizeof(double) * nx), Mu(sizeof(double) * nx), Au(sizeof(double) * nx), mvk(sizeof(double) * nx),
      tmp(sizeof(double) * nx);
  vec_copy(uz.d(), u0, nx, s);
  zero_boundary_field(uz.d(), s);
  spatial_apply(0, uz.d(), Mu.d(), s);
  spatial_apply(1, uz.d(), Au.d(), s);
  WaveHelpers h;
  if (wave) {
    h = wave_helpers(w);
    vec_copy(tmp.d(), v0, nx, s);
    zero_boundary_field(tmp.d(), s);
    spatial_apply(0, tmp.d(), mvk.d(), s);
  }
  const double z = wave ? h.minv_alpha_last / tau_ : 0.0;
  const double g = -h.minv_beta_last;
  for (int st = 0; st < S; ++st) {
    for (int i = 0; i < nt; ++i) {
      double* sg = seg(st, i);
      if (!wave) {
        if (st == 0) {
          if (cgp) {
            vec_axpy(sg, -w.alpha[i], Mu.d(), nx, s);
            vec_axpy(sg, -tau_ * w.beta[i], Au.d(), nx, s);
          } else {
            vec_axpy(sg, w.alpha[i], Mu.d(), nx, s);
          }
        }
      } else if (st == 0) {
        if (cgp) {
          vec_axpy(sg, -h.am_alpha[i] / tau_, Mu.d(), nx, s);
          vec_axpy(sg, -tau_ * w.beta[i], Au.d(), nx, s);
          vec_axpy(sg, -h.alpha_a[i], mvk.d(), nx, s);
        } else {
          vec_axpy(sg, h.am_alpha[i] / tau_, Mu.d(), nx, s);
          vec_axpy(sg, w.alpha[i], mvk.d(), nx, s);
        }
      } else {
        if (cgp)
          vec_axpy(sg, -h.alpha_a[i], mvk.d(), nx, s);
        else
          vec_axpy(sg, w.alpha[i], mvk.d(), nx, s);
      }
    }
    if (wave) {
      if (st == 0) {
        if (cgp)
          vec_axpby(mvk.d(), z, Mu.d(), g, nx, s);  // mvk = z Mu + g mvk
        else
          vec_scale_into(mvk.d(), -z, Mu.d(), nx, s);
      } else {
        if (cgp)
          vec_scale_into(mvk.d(), g, mvk.d(), nx, s);
        else
          vec_fill(mvk.d(), 0.0, nx, s);
      }
    }
  }
  for (int st = 0; st < S; ++st)
    for (int i = 0; i < nt; ++i) zero_boundary_field(seg(st, i), s);
  cuda_check(cudaStreamSynchronize(s), "assemble_rhs");
}

void SpaceTimeOperator::extract_final(const double* u, const double* u0, const double* v0, double* uf, double* vf,
                                      cudaStream_t s) const {
  const int S = n_steps_, nt = weights_.n_t;
  const Index nx = n_space();
  vec_copy(uf, u + block_offset(S - 1, nt - 1), nx, s);
  if (equation_ == Equation::Heat) return;
  if (!v0 || !vf) throw std::invalid_argument("extract_final: the wave equation needs velocities");
  const bool cgp = weights_.scheme == TimeScheme::CGP;
  const WaveHelpers h = wave_helpers(weights_);
  DeviceBuffer vl(sizeof(double) * nx), vs(sizeof(double) * nx);
  vec_copy(vl.d(), v0, nx, s);
  const double* prev_last = u0;
  for (int st = 0; st < S; ++st) {
    vec_fill(vs.d(), 0.0, nx, s);
    for (int j = 0; j < nt; ++j) vec_axpy(vs.d(), h.minv_a_last[j] / tau_, u + block_offset(st, j), nx, s);
    if (cgp) {
      vec_axpy(vs.d(), h.minv_alpha_last / tau_, prev_last, nx, s);
      vec_axpy(vs.d(), -h.minv_beta_last, vl.d(), nx, s);
    } else {
      vec_axpy(vs.d(), -h.minv_alpha_last / tau_, prev_last, nx, s);
    }
    vec_copy(vl.d(), vs.d(), nx, s);
    prev_last = u + block_offset(st, nt - 1);
  }
  vec_copy(vf, vl.d(), nx, s);
  cuda_check(cudaStreamSynchronize(s), "extract_final");
}

void SpaceTimeOperator::velocity_trajectory(const double* u, const double* u0, const double* v0, double* vout,
                                            cudaStream_t s) const {
  if (equation_ != Equation::Wave) throw std::invalid_argument("velocity_trajectory: wave equation only");
  if (!u || !u0 || !v0 || !vout) throw std::invalid_argument("velocity_trajectory: null argument");
  const int S = n_steps_, nt = weights_.n_t;
  const Index nx = n_space();
  const bool cgp = weights_.scheme == TimeScheme::CGP;
  const std::vector<double> minv = invert_small(weights_.m, nt);
  const std::vector<double> minv_a = matmul_small(minv, weights_.a, nt, nt, nt);
  const std::vector<double> minv_alpha = matmul_small(minv, weights_.alpha, nt, nt, 1);
  const std::vector<double> minv_beta =
      cgp ? matmul_small(minv, weights_.beta, nt, nt, 1) : std::vector<double>(static_cast<size_t>(nt), 0.0);
  // v_{s,i} = sum_j (M^-1 A)_ij / tau u_{s,j} + history of the previous step
  const double* prev_last = u0;
  const double* v_prev_last = v0;
  for (int st = 0; st < S; ++st) {
    for (int i = 0; i < nt; ++i) {
      double* vi = vout + block_offset(st, i);
      vec_fill(vi, 0.0, nx, s);
      for (int j = 0; j < nt; ++j) vec_axpy(vi, minv_a[i * nt + j] / tau_, u + block_offset(st, j), nx, s);
      if (cgp) {
        vec_axpy(vi, minv_alpha[i] / tau_, prev_last, nx, s);
        vec_axpy(vi, -minv_beta[i], v_prev_last, nx, s);
      } else {
        vec_axpy(vi, -minv_alpha[i] / tau_, prev_last, nx, s);
      }
    }
    prev_last = u + block_offset(st, nt - 1);
    v_prev_last = vout + block_offset(st, nt - 1);
  }
}

void SpaceTimeOperator::value_at(const double* u, const double* u0, int step, double t_ref, double* out,
                                 cudaStream_t s) const {
  if (step < 0 || step >= n_steps_) throw std::invalid_argument("value_at: bad step");
  const int nt = weights_.n_t;
  const Index nx = n_space();
  vec_fill(out, 0.0, nx, s);
  for (int i = 0; i < nt; ++i) vec_axpy(out, weights_.unknown_weight(i, t_ref), u + block_offset(step, i), nx, s);
  const double lw = weights_.left_weight(t_ref);
  if (lw != 0.0) vec_axpy(out, lw, step == 0 ? u0 : u + block_offset(step - 1, nt - 1), nx, s);
}

std::pair<double, double> SpaceTimeOperator::spatial_error(const double* field, int kind, double frequency, double t,
                                                           cudaStream_t s) const {
  const Rule q = gauss(p_ + 2);
  DeviceBuffer acc(2 * sizeof(double));
  cuda_check(cudaMemsetAsync(acc.raw(), 0, 2 * sizeof(double), s), "error acc");
  ::stmgb::spatial_error(desc_, field, p_ + 2, q.x.data(), q.w.data(), kind, 2.0 * M_PI * frequency, t, acc.d(), s);
  double h[2];
  cuda_check(cudaMemcpyAsync(h, acc.raw(), sizeof(h), cudaMemcpyDeviceToHost, s), "error result");
  cuda_check(cudaStreamSynchronize(s), "error sync");
  return {h[0], h[1]};
}

void SpaceTimeOperator::zero_boundary_field(double* v, cudaStream_t s) const {
  // Dirichlet entries of one spatial field set to zero: the identity rows of
  // the boundary pass applied to (f = v, u = v) give v_b - v_b = 0
  DevLevel one = desc_;
  one.F = 1;
  one.n_dofs = one.n_space;
  st_zero_boundary(one, v, s);
}

// ------------------------------------------------------------ ASMSmoother
namespace {
// inverse of a small dense n x n matrix (Gauss-Jordan, partial pivoting);
// false when singular
bool invert_small(std::vector<double> a, int n, std::vector<double>& inv) {
  inv.assign(static_cast<size_t>(n * n), 0.0);
  for (int i = 0; i < n; ++i) inv[static_cast<size_t>(i * n + i)] = 1.0;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a[static_cast<size_t>(i * n + k)]) > std::abs(a[static_cast<size_t>(piv * n + k)])) piv = i;
    if (a[static_cast<size_t>(piv * n + k)] == 0.0) return false;
    for (int j = 0; j < n; ++j) {
      std::swap(a[static_cast<size_t>(k * n + j)], a[static_cast<size_t>(piv * n + j)]);
      std::swap(inv[static_cast<size_t>(k * n + j)], inv[static_cast<size_t>(piv * n + j)]);
    }
    const double d = 1.0 / a[static_cast<size_t>(k * n + k)];
    for (int j = 0; j < n; ++j) {
      a[static_cast<size_t>(k * n + j)] *= d;
      inv[static_cast<size_t>(k * n + j)] *= d;
    }
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = a[static_cast<size_t>(i * n + k)];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        a[static_cast<size_t>(i * n + j)] -= f * a[static_cast<size_t>(k * n + j)];
        inv[static_cast<size_t>(i * n + j)] -= f * inv[static_cast<size_t>(k * n + j)];
      }
    }
  }
  return true;
}

// null vector of (G - sigma I), G real n x n, sigma complex: complete-pivoting
// elimination, the last pivot is the (numerically) zero one
std::vector<std::complex<double>> eigvec_small(const std::vector<double>& G, int n, std::complex<double> sigma) {
  using C = std::complex<double>;
  std::vector<C> a(static_cast<size_t>(n * n));
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) a[static_cast<size_t>(i * n + j)] = G[static_cast<size_t>(i * n + j)] - (i == j ? sigma : 0.0);
  std::vector<int> colp(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) colp[static_cast<size_t>(j)] = j;
  auto A = [&](int i, int j) -> C& { return a[static_cast<size_t>(i * n + j)]; };
  for (int k = 0; k < n - 1; ++k) {
    int pi = k, pj = k;
    for (int i = k; i < n; ++i)
      for (int j = k; j < n; ++j)
        if (std::abs(A(i, j)) > std::abs(A(pi, pj))) {
          pi = i;
          pj = j;
        }
    for (int j = 0; j < n; ++j) std::swap(A(k, j), A(pi, j));
    for (int i = 0; i < n; ++i) std::swap(A(i, k), A(i, pj));
    std::swap(colp[static_cast<size_t>(k)], colp[static_cast<size_t>(pj)]);
    for (int i = k + 1; i < n; ++i) {
      const C f = A(i, k) / A(k, k);
      for (int j = k; j < n; ++j) A(i, j) -= f * A(k, j);
    }
  }
  // U y = 0 with y_{n-1} = 1 (permuted unknowns)
  std::vector<C> y(static_cast<size_t>(n));
  y[static_cast<size_t>(n - 1)] = 1.0;
  for (int i = n - 2; i >= 0; --i) {
    C s = 0.0;
    for (int j = i + 1; j < n; ++j) s += A(i, j) * y[static_cast<size_t>(j)];
    y[static_cast<size_t>(i)] = -s / A(i, i);
  }
  std::vector<C> v(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) v[static_cast<size_t>(colp[static_cast<size_t>(j)])] = y[static_cast<size_t>(j)];
  // scale so the largest component is 1 (a real eigenvalue gives a real vector)
  size_t im = 0;
  for (size_t i = 1; i < v.size(); ++i)
    if (std::abs(v[i]) > std::abs(v[im])) im = i;
  const C s = v[im];
  for (auto& x : v) x /= s;
  return v;
}
}  // namespace

struct TBlk {
  int size;
  double a, b;
};

// G = T_A^-1 T_M = Q B Q^-1 with B real block diagonal (1x1 eigenvalues, 2x2
// [[a, b], [-b, a]] blocks for conjugate pairs, pairs first); Pm = Q^-1 T_A^-1.
// false when T_A is singular, G has a repeated eigenvalue, or Q is
// ill-conditioned (the callers keep the pivoted solves then).
bool temporal_fd(const double* TMp, const double* TAp, int n, std::vector<double>& Pm, std::vector<double>& Qm,
                 std::vector<TBlk>& blocks) {
  if (n < 1 || n > 4) return false;
  std::vector<double> TM(TMp, TMp + n * n), TA(TAp, TAp + n * n), TAi, G(static_cast<size_t>(n * n), 0.0);
  if (!invert_small(TA, n, TAi)) return false;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) G[static_cast<size_t>(i * n + j)] += TAi[static_cast<size_t>(i * n + k)] * TM[static_cast<size_t>(k * n + j)];
  std::vector<std::pair<double, double>> ev;
  try {
    ev = eigenvalues_small(G, n);
  } catch (const std::exception&) {
    return false;
  }
  double gmax = 0.0;
  for (auto& e : ev) gmax = std::max(gmax, std::hypot(e.first, e.second));
  for (size_t a = 0; a < ev.size(); ++a)
    for (size_t b = a + 1; b < ev.size(); ++b)
      if (std::hypot(ev[a].first - ev[b].first, ev[a].second - ev[b].second) < 1e-8 * gmax) return false;
  // blocks in Q column order: complex pairs first (they need aligned slot pairs)
  blocks.clear();
  Qm.assign(static_cast<size_t>(n * n), 0.0);
  int col = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (auto& e : ev) {
      const bool cplx = std::abs(e.second) > 1e-12 * gmax;
      if (pass == 0 && !(cplx && e.second > 0)) continue;
      if (pass == 1 && cplx) continue;
      const auto v = eigvec_small(G, n, {e.first, cplx ? e.second : 0.0});
      for (int i = 0; i < n; ++i) {
        Qm[static_cast<size_t>(i * n + col)] = v[static_cast<size_t>(i)].real();
        if (cplx) Qm[static_cast<size_t>(i * n + col + 1)] = v[static_cast<size_t>(i)].imag();
      }
      blocks.push_back({cplx ? 2 : 1, e.first, cplx ? e.second : 0.0});
      col += cplx ? 2 : 1;
    }
  if (col != n) return false;
  std::vector<double> Qi;
  if (!invert_small(Qm, n, Qi)) return false;
  // conditioning and reconstruction checks: Q B Q^-1 == G
  double nq = 0.0, nqi = 0.0;
  for (int i = 0; i < n; ++i) {
    double r1 = 0.0, r2 = 0.0;
    for (int j = 0; j < n; ++j) {
      r1 += std::abs(Qm[static_cast<size_t>(i * n + j)]);
      r2 += std::abs(Qi[static_cast<size_t>(i * n + j)]);
    }
    nq = std::max(nq, r1);
    nqi = std::max(nqi, r2);
  }
  if (nq * nqi > 1e6) return false;
  std::vector<double> B(static_cast<size_t>(n * n), 0.0);
  {
    int c = 0;
    for (auto& b : blocks) {
      B[static_cast<size_t>(c * n + c)] = b.a;
      if (b.size == 2) {
        B[static_cast<size_t>(c * n + c + 1)] = b.b;
        B[static_cast<size_t>((c + 1) * n + c)] = -b.b;
        B[static_cast<size_t>((c + 1) * n + c + 1)] = b.a;
      }
      c += b.size;
    }
  }
  double err = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < n; ++k)
        for (int l = 0; l < n; ++l)
          s += Qm[static_cast<size_t>(i * n + k)] * B[static_cast<size_t>(k * n + l)] * Qi[static_cast<size_t>(l * n + j)];
      err = std::max(err, std::abs(s - G[static_cast<size_t>(i * n + j)]));
    }
  if (err > 1e-10 * std::max(gmax, 1e-300)) return false;
  // Pm = Q^-1 T_A^-1
  Pm.assign(static_cast<size_t>(n * n), 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) Pm[static_cast<size_t>(i * n + j)] += Qi[static_cast<size_t>(i * n + k)] * TAi[static_cast<size_t>(k * n + j)];
  return true;
}

// Real block diagonalisation of the temporal solves of the cell blocks:
// T_M + lam T_A = T_A (G + lam I), G = T_A^-1 T_M = Q B Q^-1 with B 1x1 real
// eigenvalues and 2x2 [[a, b], [-b, a]] blocks for conjugate pairs a +- ib, so
// (T_M + lam T_A)^-1 = Q (B + lam)^-1 (Q^-1 T_A^-1). Fills A.P/Q/kind/s0/s1
// over the S*n_t slab columns and sets A.tdiag; leaves it 0 (the pivoted
// per-eigenvalue solve is used) when G has a repeated eigenvalue or Q is
// ill-conditioned.
void temporal_block_diagonalise(DevASM& A) {
  A.tdiag = 0;
  const int n = A.nt, S = A.S, ncol = n * S;
  if (ncol > 8 || n < 1) return;
  std::vector<double> Pm, Qm;
  std::vector<TBlk> blocks;
  if (!temporal_fd(A.TM, A.TA, n, Pm, Qm, blocks)) return;
  // slots: complex blocks of every step on aligned pairs, then the reals
  std::vector<int> slot(static_cast<size_t>(S * n), -1);  // (step, transformed component) -> slot
  int next_pair = 0;
  for (int s = 0; s < S; ++s) {
    int c = 0;
    for (auto& b : blocks) {
      if (b.size == 2) {
        slot[static_cast<size_t>(s * n + c)] = 2 * next_pair;
        slot[static_cast<size_t>(s * n + c + 1)] = 2 * next_pair + 1;
        ++next_pair;
      }
      c += b.size;
    }
  }
  int next_slot = 2 * next_pair;
  for (int s = 0; s < S; ++s) {
    int c = 0;
    for (auto& b : blocks) {
      if (b.size == 1) slot[static_cast<size_t>(s * n + c)] = next_slot++;
      c += b.size;
    }
  }
  if (next_slot > 8) return;
  std::memset(A.P, 0, sizeof(A.P));
  std::memset(A.Q, 0, sizeof(A.Q));
  for (int j = 0; j < 4; ++j) {
    A.kind[j] = 0;
    A.s0[j] = A.s1[j] = 1.0;  // unused slots: any nonzero value
  }
  for (int s = 0; s < S; ++s) {
    int c = 0;
    for (auto& b : blocks) {
      const int k0 = slot[static_cast<size_t>(s * n + c)];
      if (b.size == 2) {
        A.kind[k0 / 2] = 1;
        A.s0[k0 / 2] = b.a;
        A.s1[k0 / 2] = b.b;
      } else if (k0 % 2 == 0) {
        A.s0[k0 / 2] = b.a;
      } else {
        A.s1[k0 / 2] = b.a;
      }
      c += b.size;
    }
    for (int comp = 0; comp < n; ++comp) {
      const int k = slot[static_cast<size_t>(s * n + comp)];
      for (int i = 0; i < n; ++i) {
        A.P[k][s * n + i] = Pm[static_cast<size_t>(comp * n + i)];
        A.Q[s * n + i][k] = Qm[static_cast<size_t>(i * n + comp)];
      }
    }
  }
  A.tdiag = 1;
}

// Reorders the interior-class 1D eigenpairs of every axis: eigenvectors
// symmetric about the cell centre first, antisymmetric after (the even-odd
// FDM transforms, asm_fdm.cu fdm_fwd / fdm_bwd). The interior 1D matrices
// are centro-symmetric, so with distinct eigenvalues every eigenvector has a
// parity; false (tables untouched) if one does not or the counts differ.
bool fdm_order_interior_by_parity(DevFDM& F, int dim) {
  const int n = F.n, H = n / 2, HE = (n + 1) / 2;
  double S[3][kMaxN][kMaxN], L[3][kMaxN];
  for (int a = 0; a < dim; ++a) {
    std::vector<int> sym, anti;
    for (int e = 0; e < n; ++e) {
      double scale = 0.0, ds = 0.0, da = 0.0;
      for (int k = 0; k < n; ++k) {
        scale = std::max(scale, std::abs(F.S1[a][0][k][e]));
        ds = std::max(ds, std::abs(F.S1[a][0][k][e] - F.S1[a][0][n - 1 - k][e]));
        da = std::max(da, std::abs(F.S1[a][0][k][e] + F.S1[a][0][n - 1 - k][e]));
      }
      if (ds <= 1e-12 * scale)
        sym.push_back(e);
      else if (da <= 1e-12 * scale)
        anti.push_back(e);
      else
        return false;
    }
    if (static_cast<int>(sym.size()) != HE || static_cast<int>(anti.size()) != H) return false;
    std::vector<int> order(sym);
    order.insert(order.end(), anti.begin(), anti.end());
    for (int e = 0; e < n; ++e) {
      L[a][e] = F.L1[a][0][order[static_cast<size_t>(e)]];
      for (int k = 0; k < n; ++k) S[a][k][e] = F.S1[a][0][k][order[static_cast<size_t>(e)]];
    }
  }
  for (int a = 0; a < dim; ++a)
    for (int e = 0; e < n; ++e) {
      F.L1[a][0][e] = L[a][e];
      for (int k = 0; k < n; ++k) F.S1[a][0][k][e] = S[a][k][e];
    }
  return true;
}

ASMSmoother::ASMSmoother(const SpaceTimeOperator& op, const SpaceTimeOperator* probe_op, int probe_zcells)
    : op_(&op) {
  const DevLevel& d = op.desc();
  DevASM& A = asm_;
  A.zbc = d.zbc;
  A.cz0 = d.cz0;
  A.dim = d.dim;
  A.p = d.p;
  A.n = d.n;
  A.m = d.dim == 2 ? d.n * d.n : d.n * d.n * d.n;
  A.S = d.S;
  A.nt = d.nt;
  if (A.nt > 4) throw std::invalid_argument("ASMSmoother: n_t must be <= 4");
  for (int a = 0; a < 3; ++a) {
    A.cells[a] = d.cells[a];
    A.dofs[a] = d.dofs[a];
  }
  A.n_space = d.n_space;
  for (int i = 0; i < 16; ++i) A.TM[i] = A.TA[i] = 0.0;
  const int F = d.F;
  for (int i = 0; i < A.nt; ++i)
    for (int j = 0; j < A.nt; ++j) {
      A.TM[i * A.nt + j] = op.block_cm()[static_cast<size_t>(i * F + j)];
      A.TA[i * A.nt + j] = op.block_ca()[static_cast<size_t>(i * F + j)];
    }
  const Index n_cells = d.cells[0] * d.cells[1] * d.cells[2];
  const bool cartesian = d.verts == nullptr;
  std::vector<long long> exact_cells;
  if (cartesian) {
    // tensor-product FDM for every cell whose coefficient neighbourhood is
    // uniform (exact there); the others get the exact per-cell eigenbasis
    use_fdm_ = true;
    DevFDM& Fd = fdm_;
    Fd.dim = d.dim;
    Fd.p = d.p;
    Fd.n = d.n;
    Fd.S = d.S;
    Fd.nt = d.nt;
    for (int a = 0; a < 3; ++a) {
      Fd.cells[a] = d.cells[a];
      Fd.dofs[a] = d.dofs[a];
      Fd.cells0[a] = d.cells0[a];
    }
    Fd.n_space = d.n_space;
    std::memcpy(Fd.TM, A.TM, sizeof(A.TM));
    std::memcpy(Fd.TA, A.TA, sizeof(A.TA));
    // temporal fast diagonalisation of the per-eigen-index n_t x n_t solves
    // (STMG_NO_TDIAG keeps the pivoted elimination, for testing)
    Fd.tdiag = 0;
    {
      std::vector<double> Pm, Qm;
      std::vector<TBlk> blocks;
      if (!std::getenv("STMG_NO_TDIAG") && temporal_fd(A.TM, A.TA, A.nt, Pm, Qm, blocks)) {
        const int n = A.nt;
        for (int i = 0; i < 16; ++i) Fd.tP[i] = Fd.tQ[i] = 0.0;
        for (int i = 0; i < n * n; ++i) {
          Fd.tP[i] = Pm[static_cast<size_t>(i)];
          Fd.tQ[i] = Qm[static_cast<size_t>(i)];
        }
        for (int i = 0; i < 4; ++i) {
          Fd.tkind[i] = 0;
          Fd.ta[i] = 1.0;
          Fd.tb[i] = 0.0;
        }
        int c = 0;
        for (const TBlk& b : blocks) {
          Fd.tkind[c] = b.size == 2 ? 1 : 0;
          Fd.ta[c] = b.a;
          Fd.tb[c] = b.b;
          if (b.size == 2) {
            Fd.tkind[c + 1] = 2;
            Fd.ta[c + 1] = b.a;
            Fd.tb[c + 1] = b.b;
          }
          c += b.size;
        }
        Fd.tdiag = 1;
      }
    }
    Fd.rho0 = d.rho0;
    Fd.rho_shift = d.rho_shift;
    Fd.skip = nullptr;
    Fd.zbc = d.zbc;
    Fd.cz0 = d.cz0;
    std::memset(Fd.S1, 0, sizeof(Fd.S1));
    std::memset(Fd.L1, 0, sizeof(Fd.L1));
    for (int a = 0; a < d.dim; ++a) {
      double S[4][5][5], L[4][5];
      fdm_axis_tables(d.p, d.h[a], S, L);
      for (int t = 0; t < 4; ++t)
        for (int i = 0; i < kMaxN; ++i) {
          Fd.L1[a][t][i] = L[t][i];
          for (int j = 0; j < kMaxN; ++j) Fd.S1[a][t][i][j] = S[t][i][j];
        }
    }
    // STMG_FDM_GENERIC keeps the unordered tables, i.e. the generic line-owner
    // kernel on every cell (the path taken when the interior eigenvectors
    // cannot be ordered by parity), for testing the strip kernel against it
    Fd.eo = !std::getenv("STMG_FDM_GENERIC") && fdm_order_interior_by_parity(Fd, d.dim) ? 1 : 0;
    Fd.left = nullptr;
    Fd.n_left = 0;
    // cells the strip kernel leaves to the line-owner kernel (asm_fdm.cu)
    auto list_left_out = [&](const unsigned char* skip_host) {
      if (!Fd.eo || d.dim != 3) return;
      const std::vector<long long> left = fdm_left_out_cells(Fd, skip_host);
      left_ = upload(left);
      Fd.left = static_cast<const long long*>(left_.raw());
      Fd.n_left = static_cast<long long>(left.size());
    };
    if (!d.rho0) list_left_out(nullptr);
    if (d.rho0) {
      // host copy of the level-0 coefficient table
      const Index n0 = d.cells0[0] * d.cells0[1] * d.cells0[2];
      std::vector<double> rho0(static_cast<size_t>(n0));
      cuda_check(cudaMemcpy(rho0.data(), d.rho0, sizeof(double) * n0, cudaMemcpyDeviceToHost), "rho0");
      auto rho_of = [&](long long cx, long long cy, long long cz) {
        return rho0[static_cast<size_t>(((cz >> d.rho_shift) * d.cells0[1] + (cy >> d.rho_shift)) * d.cells0[0] +
                                        (cx >> d.rho_shift))];
      };
      std::vector<unsigned char> skip(static_cast<size_t>(n_cells), 0);
      // neighbourhoods in global cell coordinates (a slab's interface cells
      // see the neighbouring slab's coefficient)
      const long long nz_global = d.dim == 3 ? (d.cells0[2] << d.rho_shift) : 1;
      for (Index c = 0; c < n_cells; ++c) {
        const long long cx = c % d.cells[0], cy = (c / d.cells[0]) % d.cells[1];
        const long long cz = c / (d.cells[0] * d.cells[1]) + d.cz0;
        const double r0 = rho_of(cx, cy, cz);
        bool uniform = true;
        for (int dz = (d.dim == 3 ? -1 : 0); dz <= (d.dim == 3 ? 1 : 0) && uniform; ++dz)
          for (int dy = -1; dy <= 1 && uniform; ++dy)
            for (int dxx = -1; dxx <= 1 && uniform; ++dxx) {
              const long long nx = cx + dxx, ny = cy + dy, nz = cz + dz;
              if (nx < 0 || ny < 0 || nz < 0 || nx >= d.cells[0] || ny >= d.cells[1] || nz >= nz_global) continue;
              if (rho_of(nx, ny, nz) != r0) uniform = false;
            }
        if (!uniform) exact_cells.push_back(c);
      }
      if (!exact_cells.empty()) {
        if (A.m > 128) {
          exact_cells.clear();  // no exact kernel beyond 128 dofs: FDM with the cell's own rho
          exact_ = false;
        } else {
          for (long long c : exact_cells) skip[static_cast<size_t>(c)] = 1;
          skip_ = upload(skip);
          Fd.skip = static_cast<const unsigned char*>(skip_.raw());
        }
      }
      list_left_out(Fd.skip ? skip.data() : nullptr);
    }
    if (exact_cells.empty()) {
      A.n_list = 0;
      A.list = nullptr;
      return;
    }
    list_ = upload(exact_cells);
    A.list = static_cast<const long long*>(list_.raw());
    A.n_list = static_cast<long long>(exact_cells.size());
  } else {
    if (A.m > 128)
      throw std::invalid_argument("ASMSmoother: exact cell blocks on deformed meshes need (p+1)^dim <= 128");
    A.list = nullptr;
    A.n_list = n_cells;
  }
  build_exact(op, probe_op, probe_zcells);
}

void ASMSmoother::build_exact(const SpaceTimeOperator& op, const SpaceTimeOperator* probe_op, int probe_zcells) {
  const DevLevel& d = op.desc();
  DevASM& A = asm_;
  // the restricted global matrices are probed on `probe_op`: the operator
  // itself, or for a z-slab with interfaces a copy extended by one halo cell
  // layer across each interface (probe_zcells layers below), so the interface
  // entries include the neighbouring slab's cells
  const SpaceTimeOperator& pop = probe_op ? *probe_op : op;
  const DevLevel& pd = pop.desc();
  if (!probe_op) probe_zcells = 0;
  const Index n_pos = A.n_list;
  const size_t mat_bytes = sizeof(double) * static_cast<size_t>(n_pos) * A.m * A.m;
  cudaStream_t s = nullptr;
  DeviceBuffer cellM(mat_bytes), cellA(mat_bytes), probe(sizeof(double) * pd.n_space), ind(sizeof(double) * pd.n_space);
  cuda_check(cudaMemsetAsync(cellM.raw(), 0, mat_bytes, s), "memset");
  cuda_check(cudaMemsetAsync(cellA.raw(), 0, mat_bytes, s), "memset");
  // restricted global matrices by probing the matrix-free operators with
  // colour classes of period 2p+1 (no two same-colour dofs share a cell
  // neighbourhood, so every probe entry is a single matrix entry)
  const int P = 2 * d.p + 1;
  const int cz_max = d.dim == 3 ? P : 1;
  for (int cz = 0; cz < cz_max; ++cz)
    for (int cy = 0; cy < P; ++cy)
      for (int cx = 0; cx < P; ++cx) {
        vec_colour_indicator(ind.d(), pd.dofs, pd.dim, P, cx, cy, cz, (pd.cz0) * pd.p, s);
        pop.spatial_apply(0, ind.d(), probe.d(), s);
        asm_extract_probe(A, cx, cy, cz, P, probe.d(), probe_zcells, cellM.d(), s);
        pop.spatial_apply(1, ind.d(), probe.d(), s);
        asm_extract_probe(A, cx, cy, cz, P, probe.d(), probe_zcells, cellA.d(), s);
      }
  if (A.m > 64) {
    build_exact_large(cellM, cellA, s);
    return;
  }
  // standard form C = L^-1 A L^-T (into cellA), L^-1 (into cellM)
  asm_reduce_standard(A, cellM.d(), cellA.d(), s);
  cuda_check(cudaGetLastError(), "asm setup kernels");
  // batched symmetric eigensolver
  lam_.allocate(sizeof(double) * static_cast<size_t>(n_pos) * A.m);
  cusolverDnHandle_t h = nullptr;
  cusolverDnParams_t prm = nullptr;
  solver_check(cusolverDnCreate(&h), "cusolverDnCreate");
  solver_check(cusolverDnCreateParams(&prm), "cusolverDnCreateParams");
  solver_check(cusolverDnSetStream(h, s), "cusolverDnSetStream");
  // the batched solver rejects very large batches: shrink until accepted
  Index chunk = std::min<Index>(n_pos, 1 << 15);
  size_t dws = 0, hws = 0;
  for (;;) {
    const cusolverStatus_t st = cusolverDnXsyevBatched_bufferSize(
        h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, A.m, CUDA_R_64F, cellA.raw(), A.m, CUDA_R_64F,
        lam_.raw(), CUDA_R_64F, &dws, &hws, chunk);
    if (st == CUSOLVER_STATUS_SUCCESS) break;
    if (st != CUSOLVER_STATUS_INVALID_VALUE || chunk <= 64) solver_check(st, "syevBatched_bufferSize");
    chunk /= 4;
  }
  DeviceBuffer dwork(std::max<size_t>(dws, 8)), info(sizeof(int) * static_cast<size_t>(chunk));
  std::vector<char> hwork(std::max<size_t>(hws, 8));
  std::vector<int> hinfo(static_cast<size_t>(chunk));
  for (Index c0 = 0; c0 < n_pos; c0 += chunk) {
    const Index nb = std::min<Index>(chunk, n_pos - c0);
    solver_check(cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, A.m, CUDA_R_64F,
                                        cellA.d() + c0 * A.m * A.m, A.m, CUDA_R_64F, lam_.d() + c0 * A.m, CUDA_R_64F,
                                        dwork.raw(), dws, hwork.data(), hws, static_cast<int*>(info.raw()), nb),
                 "syevBatched");
    cuda_check(cudaMemcpy(hinfo.data(), info.raw(), sizeof(int) * nb, cudaMemcpyDeviceToHost), "info");
    for (Index i = 0; i < nb; ++i)
      if (hinfo[static_cast<size_t>(i)] != 0)
        throw std::runtime_error("ASMSmoother: singular block (eigensolver info " +
                                 std::to_string(hinfo[static_cast<size_t>(i)]) + ")");
  }
  cusolverDnDestroyParams(prm);
  cusolverDnDestroy(h);
  // m = 64: one TMA record per cell, X (swizzled) followed by its eigenvalues
  // (FP64 tensor-core kernel); 25/27 dofs: tensor cores on pitch-28 rows
  // (layout 2); smaller blocks: contiguous rows (DFMA warp kernel)
  A.x_layout = (A.m > 24 && A.m <= 28) ? 2 : 0;
  A.xs = asm_record_stride(A.m, A.x_layout);
  X_.allocate(sizeof(double) * static_cast<size_t>(n_pos) * A.xs);
  // pitch-28 rows leave padding columns m..27 unwritten: zero them once so the
  // bulk copies stream defined data
  cuda_check(cudaMemsetAsync(X_.raw(), 0, sizeof(double) * static_cast<size_t>(n_pos) * A.xs, s), "records");
  asm_back_transform(A.m, A.xs, A.x_layout, n_pos, cellM.d(), cellA.d(), X_.d(), s);
  if (A.m == 64) {
    cuda_check(cudaMemcpy2DAsync(X_.d() + 64 * 64, sizeof(double) * kRec64, lam_.d(), sizeof(double) * 64,
                                 sizeof(double) * 64, static_cast<size_t>(n_pos), cudaMemcpyDeviceToDevice, s),
               "asm records");
    // per position: lattice offset of local dof 0 and Dirichlet face mask
    std::vector<long long> meta(static_cast<size_t>(2 * n_pos));
    std::vector<long long> cells_h;
    if (A.list) {
      cells_h.resize(static_cast<size_t>(n_pos));
      cuda_check(cudaMemcpy(cells_h.data(), A.list, sizeof(long long) * n_pos, cudaMemcpyDeviceToHost), "list");
    }
    for (Index q = 0; q < n_pos; ++q) {
      const long long c = A.list ? cells_h[static_cast<size_t>(q)] : q;
      const long long cx = c % A.cells[0], cy = (c / A.cells[0]) % A.cells[1], cz = c / (A.cells[0] * A.cells[1]);
      meta[static_cast<size_t>(2 * q)] = (cz * A.p * A.dofs[1] + cy * A.p) * A.dofs[0] + cx * A.p;
      long long mask = 0;
      if (cx == 0) mask |= 1;
      if (cx == A.cells[0] - 1) mask |= 2;
      if (cy == 0) mask |= 4;
      if (cy == A.cells[1] - 1) mask |= 8;
      if (cz == 0 && (A.zbc & 1)) mask |= 16;
      if (cz == A.cells[2] - 1 && (A.zbc & 2)) mask |= 32;
      meta[static_cast<size_t>(2 * q + 1)] = mask;
    }
    meta_ = upload(meta);
    A.meta = static_cast<const long long*>(meta_.raw());
    // STMG_NO_TDIAG: keep the pivoted per-eigenvalue solves (the fallback
    // kernel for non-diagonalisable temporal blocks), for testing
    if (!std::getenv("STMG_NO_TDIAG")) temporal_block_diagonalise(A);
  } else if (!std::getenv("STMG_NO_TDIAG")) {
    // the padded tensor-core kernels (m = 25, 27) use it as well
    temporal_block_diagonalise(A);
  }
  cuda_check(cudaStreamSynchronize(s), "asm setup");
  A.X = X_.d();
  A.lam = lam_.d();
  if (A.S * A.nt > 8) {
    // wide batches: sweep groups of 8 / n_t steps (see add_correction)
    const bool td = !std::getenv("STMG_NO_TDIAG");
    chunk_ = A;
    chunk_.S = 8 / A.nt;
    chunk_.tdiag = 0;
    if (td) temporal_block_diagonalise(chunk_);
    tail_ = A;
    tail_.S = A.S % chunk_.S;
    tail_.tdiag = 0;
    if (td && tail_.S > 0) temporal_block_diagonalise(tail_);
  }
}

// Large cell blocks (m > 64): the same fast diagonalisation with library
// factorisations on the probed matrices -- batched Cholesky M = L L^T,
// C = L^-1 A L^-T by two batched triangular solves, batched syev, and the
// back transform X = L^-T V by a third -- in chunks that bound the
// eigensolver workspace.
void ASMSmoother::build_exact_large(DeviceBuffer& cellM, DeviceBuffer& cellA, cudaStream_t s) {
  DevASM& A = asm_;
  const Index n_pos = A.n_list;
  const int m = A.m;
  const long long mm = static_cast<long long>(m) * m;
  asm_dirichlet_rows(A, cellM.d(), cellA.d(), s);
  lam_.allocate(sizeof(double) * static_cast<size_t>(n_pos) * m);
  A.xs = mm;
  X_.allocate(sizeof(double) * static_cast<size_t>(n_pos) * mm);
  cusolverDnHandle_t h = nullptr;
  cusolverDnParams_t prm = nullptr;
  cublasHandle_t bh = nullptr;
  solver_check(cusolverDnCreate(&h), "cusolverDnCreate");
  solver_check(cusolverDnCreateParams(&prm), "cusolverDnCreateParams");
  solver_check(cusolverDnSetStream(h, s), "cusolverDnSetStream");
  if (cublasCreate(&bh) != CUBLAS_STATUS_SUCCESS) throw std::runtime_error("cublasCreate failed");
  cublasSetStream(bh, s);
  auto blas = [](cublasStatus_t st, const char* what) {
    if (st != CUBLAS_STATUS_SUCCESS) throw std::runtime_error(std::string("cuBLAS ") + what + " failed");
  };
  // chunk so the batched eigensolver workspace stays below ~2 GB
  size_t dws1 = 0, hws = 0;
  solver_check(cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m,
                                                 CUDA_R_64F, cellA.raw(), m, CUDA_R_64F, lam_.raw(), CUDA_R_64F, &dws1,
                                                 &hws, 1),
               "syevBatched_bufferSize");
  const Index chunk = std::max<Index>(1, std::min<Index>(n_pos, static_cast<Index>((size_t{2} << 30) / std::max<size_t>(dws1, 1))));
  size_t dws = 0;
  solver_check(cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m,
                                                 CUDA_R_64F, cellA.raw(), m, CUDA_R_64F, lam_.raw(), CUDA_R_64F, &dws,
                                                 &hws, chunk),
               "syevBatched_bufferSize");
  DeviceBuffer dwork(std::max<size_t>(dws, 8)), info(sizeof(int) * static_cast<size_t>(chunk)),
      pm(sizeof(double*) * static_cast<size_t>(chunk)), pa(sizeof(double*) * static_cast<size_t>(chunk));
  std::vector<char> hwork(std::max<size_t>(hws, 8));
  std::vector<int> hinfo(static_cast<size_t>(chunk));
  std::vector<double*> hm(static_cast<size_t>(chunk)), ha(static_cast<size_t>(chunk));
  const double one = 1.0;
  for (Index c0 = 0; c0 < n_pos; c0 += chunk) {
    const Index nb = std::min<Index>(chunk, n_pos - c0);
    for (Index i = 0; i < nb; ++i) {
      hm[static_cast<size_t>(i)] = cellM.d() + (c0 + i) * mm;
      ha[static_cast<size_t>(i)] = cellA.d() + (c0 + i) * mm;
    }
    cuda_check(cudaMemcpyAsync(pm.raw(), hm.data(), sizeof(double*) * nb, cudaMemcpyHostToDevice, s), "ptrs");
    cuda_check(cudaMemcpyAsync(pa.raw(), ha.data(), sizeof(double*) * nb, cudaMemcpyHostToDevice, s), "ptrs");
    double** Mp = static_cast<double**>(pm.raw());
    double** Ap = static_cast<double**>(pa.raw());
    solver_check(cusolverDnDpotrfBatched(h, CUBLAS_FILL_MODE_LOWER, m, Mp, m, static_cast<int*>(info.raw()),
                                         static_cast<int>(nb)),
                 "potrfBatched");
    cuda_check(cudaMemcpyAsync(hinfo.data(), info.raw(), sizeof(int) * nb, cudaMemcpyDeviceToHost, s), "info");
    cuda_check(cudaStreamSynchronize(s), "potrf");
    for (Index i = 0; i < nb; ++i)
      if (hinfo[static_cast<size_t>(i)] != 0) throw std::runtime_error("ASMSmoother: cell mass matrix not SPD");
    blas(cublasDtrsmBatched(bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, m,
                            &one, Mp, m, Ap, m, static_cast<int>(nb)),
         "trsm L^-1 A");
    blas(cublasDtrsmBatched(bh, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, m, m,
                            &one, Mp, m, Ap, m, static_cast<int>(nb)),
         "trsm A L^-T");
    solver_check(cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F,
                                        cellA.d() + c0 * mm, m, CUDA_R_64F, lam_.d() + c0 * m, CUDA_R_64F,
                                        dwork.raw(), dws, hwork.data(), hws, static_cast<int*>(info.raw()), nb),
                 "syevBatched");
    cuda_check(cudaMemcpyAsync(hinfo.data(), info.raw(), sizeof(int) * nb, cudaMemcpyDeviceToHost, s), "info");
    cuda_check(cudaStreamSynchronize(s), "syev");
    for (Index i = 0; i < nb; ++i)
      if (hinfo[static_cast<size_t>(i)] != 0)
        throw std::runtime_error("ASMSmoother: singular block (eigensolver info " +
                                 std::to_string(hinfo[static_cast<size_t>(i)]) + ")");
    // X = L^-T V (V column-major in cellA)
    blas(cublasDtrsmBatched(bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, m, m,
                            &one, Mp, m, Ap, m, static_cast<int>(nb)),
         "trsm L^-T V");
    asm_transpose_cells(m, nb, mm, cellA.d() + c0 * mm, X_.d() + c0 * mm, s);
  }
  cuda_check(cudaStreamSynchronize(s), "asm large setup");
  cublasDestroy(bh);
  cusolverDnDestroyParams(prm);
  cusolverDnDestroy(h);
  A.X = X_.d();
  A.lam = lam_.d();
  // temporal fast diagonalisation for the tensor-core 125-dof kernel
  A.tdiag = 0;
  if (!std::getenv("STMG_NO_TDIAG")) temporal_block_diagonalise(A);
}

void ASMSmoother::add_correction(const double* residual, double* correction, cudaStream_t stream,
                                 double scale) const {
  ++sweep_count_;
  if (use_fdm_) fdm_add_correction(fdm_, residual, correction, scale, stream);
  if (asm_.n_list == 0) return;
  if (asm_.S * asm_.nt <= 8) {
    asm_add_correction(asm_, residual, correction, scale, stream);
    return;
  }
  // wide batches: the blocks are per (step, cell) (asm_smoother.cpp:24-28),
  // so groups of whole steps are independent sweeps of <= 8 columns
  const long long step = static_cast<long long>(asm_.nt) * asm_.n_space;
  for (int s0 = 0; s0 < asm_.S; s0 += chunk_.S) {
    const DevASM& A = asm_.S - s0 >= chunk_.S ? chunk_ : tail_;
    asm_add_correction(A, residual + s0 * step, correction + s0 * step, scale, stream);
  }
}

// --------------------------------------------------------------- Transfer
namespace {
// dense 1D prolongation matrix, nf x nc (transfer.cpp:32-54)
std::vector<double> axis_prolongation(Index fine_cells, int pf, Index coarse_cells, int pc) {
  const Index nf = fine_cells * pf + 1, nc = coarse_cells * pc + 1;
  const bool h = coarse_cells != fine_cells;
  const std::vector<double> fn = gauss_lobatto(pf + 1).x, cn = gauss_lobatto(pc + 1).x;
  std::vector<double> P(static_cast<size_t>(nf * nc), 0.0);
  for (Index cf = 0; cf < fine_cells; ++cf)
    for (int m = 0; m <= pf; ++m) {
      const Index row = cf * pf + m;
      Index cc = cf;
      double tc = fn[m];
      if (h) {
        cc = cf / 2;
        tc = 0.5 * static_cast<double>(cf % 2) + 0.5 * fn[m];
      }
      for (int j = 0; j <= pc; ++j) P[static_cast<size_t>(row * nc + cc * pc + j)] = lagrange_eval(cn, j, tc);
    }
  return P;
}
}  // namespace

Transfer::Transfer(const SpaceTimeOperator& fine, const SpaceTimeOperator& coarse) : fine_(&fine), coarse_(&coarse) {
  spatial_ = fine.mesh_level() != coarse.mesh_level() || fine.p() != coarse.p();
  Ff_ = fine.desc().F;
  Fc_ = coarse.desc().F;
  if (spatial_) {
    if (fine.n_steps() != coarse.n_steps() || fine.weights().k != coarse.weights().k ||
        fine.weights().scheme != coarse.weights().scheme)
      throw std::invalid_argument("Transfer: more than one attribute changed");
    const bool h = fine.mesh_level() != coarse.mesh_level();
    for (int a = 0; a < fine.dim(); ++a) {
      const Index cf = fine.desc().cells[a], cc = coarse.desc().cells[a];
      if (h && cc * 2 != cf) throw std::invalid_argument("Transfer: meshes are not nested");
      const int pf = fine.p(), pc = coarse.p();
      const std::vector<double> P = axis_prolongation(cf, pf, cc, pc);
      const Index nf = cf * pf + 1, nc = cc * pc + 1;
      // CSR of P (rows: fine index) and of P^T (rows: coarse index)
      std::vector<int> rptr(static_cast<size_t>(nf + 1), 0), ridx, cptr(static_cast<size_t>(nc + 1), 0), cidx;
      std::vector<double> rw, cw;
      for (Index i = 0; i < nf; ++i) {
        for (Index j = 0; j < nc; ++j) {
          const double v = P[static_cast<size_t>(i * nc + j)];
          if (v != 0.0) {
            ridx.push_back(static_cast<int>(j));
            rw.push_back(v);
          }
        }
        rptr[static_cast<size_t>(i + 1)] = static_cast<int>(ridx.size());
      }
      for (Index j = 0; j < nc; ++j) {
        for (Index i = 0; i < nf; ++i) {
          const double v = P[static_cast<size_t>(i * nc + j)];
          if (v != 0.0) {
            cidx.push_back(static_cast<int>(i));
            cw.push_back(v);
          }
        }
        cptr[static_cast<size_t>(j + 1)] = static_cast<int>(cidx.size());
      }
      bufs_.push_back(upload(rptr));
      ax_[a].row_ptr = static_cast<const int*>(bufs_.back().raw());
      bufs_.push_back(upload(ridx));
      ax_[a].row_idx = static_cast<const int*>(bufs_.back().raw());
      bufs_.push_back(upload(rw));
      ax_[a].row_w = bufs_.back().d();
      bufs_.push_back(upload(cptr));
      ax_[a].col_ptr = static_cast<const int*>(bufs_.back().raw());
      bufs_.push_back(upload(cidx));
      ax_[a].col_idx = static_cast<const int*>(bufs_.back().raw());
      bufs_.push_back(upload(cw));
      ax_[a].col_w = bufs_.back().d();
      ax_[a].nf = nf;
      ax_[a].nc = nc;
      // structured h weights: the rows of P for the fine nodes of coarse cell 0
      ax_[a].hp = 0;
      if (h && pf == pc) {
        ax_[a].hp = pf;
        for (int r = 0; r <= 2 * pf; ++r)
          for (int j = 0; j < kMaxN; ++j)
            ax_[a].hw[r][j] = j <= pc ? P[static_cast<size_t>(r * nc + j)] : 0.0;
      }
    }
    const long long* df = fine.desc().dofs;
    const long long* dc = coarse.desc().dofs;
    const long long F = fine.desc().F;
    const long long t1 = F * std::max(df[0] * dc[1] * dc[2], dc[0] * df[1] * df[2]);
    const long long t2 = F * std::max(df[0] * df[1] * dc[2], dc[0] * dc[1] * df[2]);
    t1_.allocate(sizeof(double) * t1);
    t2_.allocate(sizeof(double) * t2);
  } else {
    const TemporalWeights& wf = fine.weights();
    const TemporalWeights& wc = coarse.weights();
    const int Sf = fine.n_steps(), Sc = coarse.n_steps();
    const bool tau_c = Sf != Sc;
    if (tau_c && (Sf != 2 * Sc || wf.k != wc.k)) throw std::invalid_argument("Transfer: invalid tau coarsening");
    if (!tau_c && wf.k != wc.k + 1) throw std::invalid_argument("Transfer: invalid k coarsening");
    // evaluation matrix of the coarse trajectory at the fine unknown nodes,
    // CGP left value folded in (transfer.cpp:75-105)
    std::vector<double> T(static_cast<size_t>(Ff_ * Fc_), 0.0);
    for (int sf = 0; sf < Sf; ++sf)
      for (int i = 0; i < wf.n_t; ++i) {
        const int row = sf * wf.n_t + i;
        const double tf = wf.unknown_nodes[static_cast<size_t>(i)];
        int sc = sf;
        double tc = tf;
        if (tau_c) {
          sc = sf / 2;
          tc = 0.5 * static_cast<double>(sf % 2) + 0.5 * tf;
        }
        for (int j = 0; j < wc.n_t; ++j) T[static_cast<size_t>(row * Fc_ + sc * wc.n_t + j)] += wc.unknown_weight(j, tc);
        const double lw = wc.left_weight(tc);
        if (lw != 0.0 && sc > 0) T[static_cast<size_t>(row * Fc_ + sc * wc.n_t - 1)] += lw;
      }
    time_p_ = upload(T);
  }
}

void Transfer::prolong(const double* coarse, double* fine, cudaStream_t stream, bool accumulate,
                       long long coarse_fstride) const {
  const DevLevel& df = fine_->desc();
  const DevLevel& dc = coarse_->desc();
  TransferSlab sl;
  sl.zbc = df.zbc;
  sl.accumulate = accumulate;
  sl.coarse_fstride = coarse_fstride;
  if (spatial_)
    spatial_prolong(ax_, df.dim, df.F, dc.dofs, df.dofs, coarse, fine, t1_.d(), t2_.d(), sl, stream);
  else
    temporal_prolong(time_p_.d(), Ff_, Fc_, df.n_space, df.dofs, df.dim, coarse, fine, sl, stream);
}

void Transfer::restrict_(const double* fine, double* coarse, cudaStream_t stream, bool accumulate,
                         long long coarse_fstride) const {
  const DevLevel& df = fine_->desc();
  const DevLevel& dc = coarse_->desc();
  TransferSlab sl;
  sl.zbc = df.zbc;
  sl.skip_lo_in = df.dim == 3 && !(df.zbc & 1);
  sl.accumulate = accumulate;
  sl.coarse_fstride = coarse_fstride;
  if (spatial_)
    spatial_restrict(ax_, df.dim, df.F, dc.dofs, df.dofs, fine, coarse, t1_.d(), t2_.d(), sl, stream);
  else
    temporal_restrict(time_p_.d(), Ff_, Fc_, df.n_space, df.dofs, df.dim, fine, coarse, sl, stream);
}

// ------------------------------------------------------------------ GMRES
void GmresWorkspace::ensure(Index n, int vectors) {
  if (n != n_) {
    basis_.clear();
    n_ = n;
    r_.allocate(sizeof(double) * n);
    w_.allocate(sizeof(double) * n);
    z_.allocate(sizeof(double) * n);
    ptrs_.allocate(sizeof(double*) * 1030);
    scratch_.allocate(sizeof(double) * kDotBlocks * 1030);
    small_.allocate(sizeof(double) * 4 * 1030);
  }
  if (static_cast<int>(basis_.size()) < vectors) {
    if (vectors > 1024) throw std::invalid_argument("gmres: restart must be <= 1023");
    const size_t old = basis_.size();
    while (static_cast<int>(basis_.size()) < vectors) basis_.emplace_back(sizeof(double) * n);
    std::vector<const double*> hp(basis_.size());
    for (size_t i = 0; i < basis_.size(); ++i) hp[i] = basis_[i].d();
    cuda_check(cudaMemcpy(static_cast<const double**>(ptrs_.raw()) + old, hp.data() + old,
                          sizeof(double*) * (hp.size() - old), cudaMemcpyHostToDevice),
               "gmres ptrs");
  }
}

GmresResult gmres(const DeviceMap& op, const double* b, double* x, Index n, const GmresOptions& options,
                  const DeviceMap& precond, GmresWorkspace& ws, cudaStream_t s, const DotPolicy* dots) {
  if (!op) throw std::invalid_argument("gmres: missing operator");
  const int m = std::max(1, options.restart);
  ws.ensure(n, 1);
  // k inner products <V_i, w> into the device buffer out (owned entries and a
  // sum over ranks for a distributed vector)
  auto multidot = [&](const double* const* V, int k, const double* w, double* out) {
    if (!dots) {
      vec_multidot(V, k, w, n, out, ws.scratch(), s);
      return;
    }
    vec_multidot_seg(V, k, w, dots->seg, out, ws.scratch(), s);
    if (dots->allreduce) dots->allreduce(out, k, s);
  };
  // extra pointer slot after the basis for norms of w / r
  DeviceBuffer one_ptr(sizeof(double*));
  auto norm_of = [&](const double* v) {
    const double* hp[1] = {v};
    cuda_check(cudaMemcpyAsync(one_ptr.raw(), hp, sizeof(hp), cudaMemcpyHostToDevice, s), "ptr");
    multidot(static_cast<const double* const*>(one_ptr.raw()), 1, v, ws.small());
    double r = 0.0;
    cuda_check(cudaMemcpyAsync(&r, ws.small(), sizeof(double), cudaMemcpyDeviceToHost, s), "nrm");
    cuda_check(cudaStreamSynchronize(s), "nrm sync");
    return std::sqrt(r);
  };
  GmresResult result;
  op(x, ws.r(), s);
  vec_sub_into(ws.r(), b, ws.r(), n, s);
  double beta = norm_of(ws.r());
  result.initial_residual = beta;
  result.residual_history.push_back(beta);
  const double tol = std::max(options.abs_tol, options.rel_tol * std::max(beta, 1e-300));
  if (!std::isfinite(beta)) throw std::runtime_error("gmres: non-finite initial residual");
  if (beta <= tol) {
    result.converged = true;
    result.final_residual = beta;
    return result;
  }
  std::vector<double> H(static_cast<size_t>((m + 1) * m), 0.0), cs(m), sn(m), g(m + 1);
  auto Hs = [&H, m](int i, int j) -> double& { return H[static_cast<size_t>(i * m + j)]; };
  std::vector<double> hbuf(static_cast<size_t>(2 * (m + 1) + 1));
  while (result.iterations < options.max_iters) {
    ws.ensure(n, 1);
    vec_scale_into(ws.vec(0), 1.0 / beta, ws.r(), n, s);
    std::fill(g.begin(), g.end(), 0.0);
    std::fill(H.begin(), H.end(), 0.0);
    g[0] = beta;
    int k = 0;
    for (; k < m && result.iterations < options.max_iters; ++k) {
      ++result.iterations;
      ws.ensure(n, k + 2);
      if (precond) {
        precond(ws.vec(k), ws.z(), s);
        op(ws.z(), ws.w(), s);
      } else {
        op(ws.vec(k), ws.w(), s);
      }
      // classical Gram-Schmidt, two passes (h1 + h2 = the reference's two MGS passes)
      double* h1 = ws.small();
      double* h2 = ws.small() + (m + 1);
      multidot(ws.dev_ptrs(), k + 1, ws.w(), h1);
      vec_multi_axpy(ws.w(), ws.dev_ptrs(), k + 1, h1, -1.0, n, s);
      multidot(ws.dev_ptrs(), k + 1, ws.w(), h2);
      vec_multi_axpy(ws.w(), ws.dev_ptrs(), k + 1, h2, -1.0, n, s);
      cuda_check(cudaMemcpyAsync(hbuf.data(), ws.small(), sizeof(double) * 2 * (m + 1), cudaMemcpyDeviceToHost, s),
                 "h");
      const double hn = norm_of(ws.w());  // synchronises
      for (int i = 0; i <= k; ++i) Hs(i, k) = hbuf[static_cast<size_t>(i)] + hbuf[static_cast<size_t>(m + 1 + i)];
      Hs(k + 1, k) = hn;
      if (!std::isfinite(hn)) throw std::runtime_error("gmres: non-finite Arnoldi coefficient");
      const bool breakdown = !(hn > 0.0);
      if (!breakdown) vec_scale_into(ws.vec(k + 1), 1.0 / hn, ws.w(), n, s);
      for (int i = 0; i < k; ++i) {
        const double t = cs[i] * Hs(i, k) + sn[i] * Hs(i + 1, k);
        Hs(i + 1, k) = -sn[i] * Hs(i, k) + cs[i] * Hs(i + 1, k);
        Hs(i, k) = t;
      }
      const double denom = std::hypot(Hs(k, k), Hs(k + 1, k));
      if (denom == 0.0) {
        cs[k] = 1.0;
        sn[k] = 0.0;
      } else {
        cs[k] = Hs(k, k) / denom;
        sn[k] = Hs(k + 1, k) / denom;
      }
      Hs(k, k) = denom;
      Hs(k + 1, k) = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      const double res = std::abs(g[k + 1]);
      result.residual_history.push_back(res);
      if (res <= tol || breakdown) {
        ++k;
        break;
      }
    }
    // y = H(0:k,0:k)^-1 g(0:k), then x += M^-1 (V y)
    std::vector<double> y(static_cast<size_t>(k));
    for (int i = k - 1; i >= 0; --i) {
      double sum = g[i];
      for (int j = i + 1; j < k; ++j) sum -= Hs(i, j) * y[static_cast<size_t>(j)];
      y[static_cast<size_t>(i)] = sum / Hs(i, i);
    }
    cuda_check(cudaMemcpyAsync(ws.small(), y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s), "y");
    vec_fill(ws.w(), 0.0, n, s);
    vec_multi_axpy(ws.w(), ws.dev_ptrs(), k, ws.small(), 1.0, n, s);
    if (precond) {
      precond(ws.w(), ws.z(), s);
      vec_axpy(x, 1.0, ws.z(), n, s);
    } else {
      vec_axpy(x, 1.0, ws.w(), n, s);
    }
    op(x, ws.r(), s);
    vec_sub_into(ws.r(), b, ws.r(), n, s);
    beta = norm_of(ws.r());
    result.final_residual = beta;
    if (beta <= tol) {
      result.converged = true;
      return result;
    }
    if (beta == 0.0) break;
  }
  result.final_residual = beta;
  result.converged = beta <= tol;
  return result;
}

// ---------------------------------------------------------------- eigen
std::vector<std::pair<double, double>> eigenvalues_small(std::vector<double> a, int n) {
  // Householder reduction to upper Hessenberg form
  auto A = [&a, n](int i, int j) -> double& { return a[static_cast<size_t>(i * n + j)]; };
  std::vector<double> v(static_cast<size_t>(n));
  for (int k = 0; k < n - 2; ++k) {
    double alpha = 0.0;
    for (int i = k + 1; i < n; ++i) alpha += A(i, k) * A(i, k);
    alpha = std::sqrt(alpha);
    if (alpha == 0.0) continue;
    if (A(k + 1, k) > 0) alpha = -alpha;
    std::fill(v.begin(), v.end(), 0.0);
    v[k + 1] = A(k + 1, k) - alpha;
    for (int i = k + 2; i < n; ++i) v[i] = A(i, k);
    double vn = 0.0;
    for (int i = k + 1; i < n; ++i) vn += v[i] * v[i];
    if (vn == 0.0) continue;
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int i = k + 1; i < n; ++i) s += v[i] * A(i, j);
      s *= 2.0 / vn;
      for (int i = k + 1; i < n; ++i) A(i, j) -= s * v[i];
    }
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = k + 1; j < n; ++j) s += A(i, j) * v[j];
      s *= 2.0 / vn;
      for (int j = k + 1; j < n; ++j) A(i, j) -= s * v[j];
    }
  }
  // Francis double-shift QR on the Hessenberg matrix (active window [lo, hi])
  std::vector<std::pair<double, double>> ev(static_cast<size_t>(n));
  double norm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = std::max(i - 1, 0); j < n; ++j) norm += std::abs(A(i, j));
  int hi = n - 1;
  double shift_acc = 0.0;
  int iter = 0;
  while (hi >= 0) {
    int l = hi;
    for (; l > 0; --l) {
      double s = std::abs(A(l - 1, l - 1)) + std::abs(A(l, l));
      if (s == 0.0) s = norm;
      if (std::abs(A(l, l - 1)) < 1e-16 * s) {
        A(l, l - 1) = 0.0;
        break;
      }
    }
    const double x = A(hi, hi);
    if (l == hi) {  // one real root
      ev[static_cast<size_t>(hi)] = {x + shift_acc, 0.0};
      --hi;
      iter = 0;
      continue;
    }
    const double yv = A(hi - 1, hi - 1), w = A(hi, hi - 1) * A(hi - 1, hi);
    if (l == hi - 1) {  // 2x2 block
      const double p = 0.5 * (yv - x), q = p * p + w, zz = std::sqrt(std::abs(q));
      const double xs = x + shift_acc;
      if (q >= 0.0) {
        const double z = p + (p >= 0 ? zz : -zz);
        ev[static_cast<size_t>(hi - 1)] = {xs + z, 0.0};
        ev[static_cast<size_t>(hi)] = {z != 0.0 ? xs - w / z : xs + z, 0.0};
      } else {
        ev[static_cast<size_t>(hi - 1)] = {xs + p, zz};
        ev[static_cast<size_t>(hi)] = {xs + p, -zz};
      }
      hi -= 2;
      iter = 0;
      continue;
    }
    if (++iter > 200) throw std::runtime_error("eigenvalues_small: QR iteration did not converge");
    double sx = x, sy = yv, sw = w;
    if (iter == 10 || iter == 20) {  // exceptional shift
      shift_acc += x;
      for (int i = 0; i <= hi; ++i) A(i, i) -= x;
      const double s = std::abs(A(hi, hi - 1)) + std::abs(A(hi - 1, hi - 2));
      sx = sy = 0.75 * s;
      sw = -0.4375 * s * s;
    }
    // find the start row of the bulge
    int mrow = hi - 2;
    double p = 0, q = 0, r = 0;
    for (; mrow >= l; --mrow) {
      const double z = A(mrow, mrow);
      const double rr = sx - z, ss = sy - z;
      p = (rr * ss - sw) / A(mrow + 1, mrow) + A(mrow, mrow + 1);
      q = A(mrow + 1, mrow + 1) - z - rr - ss;
      r = A(mrow + 2, mrow + 1);
      const double s = std::abs(p) + std::abs(q) + std::abs(r);
      p /= s;
      q /= s;
      r /= s;
      if (mrow == l) break;
      const double u = std::abs(A(mrow, mrow - 1)) * (std::abs(q) + std::abs(r));
      const double vv = std::abs(p) * (std::abs(A(mrow - 1, mrow - 1)) + std::abs(z) + std::abs(A(mrow + 1, mrow + 1)));
      if (u < 1e-16 * vv) break;
    }
    for (int i = mrow + 2; i <= hi; ++i) {
      A(i, i - 2) = 0.0;
      if (i != mrow + 2) A(i, i - 3) = 0.0;
    }
    for (int k = mrow; k <= hi - 1; ++k) {
      double xk = 0.0;
      if (k != mrow) {
        p = A(k, k - 1);
        q = A(k + 1, k - 1);
        r = (k != hi - 1) ? A(k + 2, k - 1) : 0.0;
        xk = std::abs(p) + std::abs(q) + std::abs(r);
        if (xk != 0.0) {
          p /= xk;
          q /= xk;
          r /= xk;
        }
      }
      double s = std::sqrt(p * p + q * q + r * r);
      if (p < 0) s = -s;
      if (s == 0.0) continue;
      if (k == mrow) {
        if (l != mrow) A(k, k - 1) = -A(k, k - 1);
      } else {
        A(k, k - 1) = -s * xk;
      }
      p += s;
      const double xx = p / s, yy = q / s, zz = r / s;
      q /= p;
      r /= p;
      for (int j = k; j <= hi; ++j) {
        double t = A(k, j) + q * A(k + 1, j);
        if (k != hi - 1) {
          t += r * A(k + 2, j);
          A(k + 2, j) -= t * zz;
        }
        A(k + 1, j) -= t * yy;
        A(k, j) -= t * xx;
      }
      const int mmin = std::min(hi, k + 3);
      for (int i = l; i <= mmin; ++i) {
        double t = xx * A(i, k) + yy * A(i, k + 1);
        if (k != hi - 1) {
          t += zz * A(i, k + 2);
          A(i, k + 2) -= t * r;
        }
        A(i, k + 1) -= t * q;
        A(i, k) -= t;
      }
    }
  }
  return ev;
}

// ------------------------------------------------------- march / errors
void accumulate_errors(const SpaceTimeOperator& op, const double* x, const double* u0, double frequency, double t0,
                       ErrorRecord& acc, cudaStream_t s, int kind) {
  if (kind != 3 && kind != 4) throw std::invalid_argument("accumulate_errors: kind must be 3 (u) or 4 (v)");
  const Rule tq = gauss(op.weights().k + 2);
  DeviceBuffer uval(sizeof(double) * op.n_space());
  for (int st = 0; st < op.n_steps(); ++st)
    for (size_t q = 0; q < tq.x.size(); ++q) {
      const double t = t0 + (st + tq.x[q]) * op.tau();
      op.value_at(x, u0, st, tq.x[q], uval.d(), s);
      const auto e = op.spatial_error(uval.d(), kind, frequency, t, s);
      acc.l2_l2 += tq.w[q] * op.tau() * e.first;
      acc.linf_l2 = std::max(acc.linf_l2, std::sqrt(e.first));
      acc.linf_linf = std::max(acc.linf_linf, e.second);
    }
}

// ------------------------------------------------------------ SectionClock
SectionClock::~SectionClock() {
  for (cudaEvent_t e : ev_) cudaEventDestroy(e);
}

void SectionClock::begin(cudaStream_t s) {
  if (used_ % 2 != 0) throw std::logic_error("SectionClock: begin inside an open section");
  if (used_ >= 1024) fold();
  while (ev_.size() < used_ + 2) {
    cudaEvent_t e = nullptr;
    cuda_check(cudaEventCreate(&e), "section event");
    ev_.push_back(e);
  }
  cuda_check(cudaEventRecord(ev_[used_++], s), "section begin");
}

void SectionClock::end(cudaStream_t s) {
  if (used_ % 2 != 1) throw std::logic_error("SectionClock: end without begin");
  cuda_check(cudaEventRecord(ev_[used_++], s), "section end");
}

void SectionClock::fold() {
  if (used_ == 0) return;
  cuda_check(cudaEventSynchronize(ev_[used_ - 1]), "section sync");
  for (size_t i = 0; i + 1 < used_; i += 2) {
    float ms = 0.0f;
    cuda_check(cudaEventElapsedTime(&ms, ev_[i], ev_[i + 1]), "section elapsed");
    total_ += 1e-3 * static_cast<double>(ms);
  }
  used_ = 0;
}

double SectionClock::seconds() {
  fold();
  return total_;
}

void SectionClock::reset() {
  if (used_ > 0) cuda_check(cudaEventSynchronize(ev_[used_ - 1]), "section sync");
  used_ = 0;
  total_ = 0.0;
}

MarchResult march(const SpaceTimeMultigrid& mg, int n_batches, int source_kind, double frequency, double* u, double* v,
                  const GmresOptions& options, bool errors, cudaStream_t s, const ProbeSpec* probes) {
  MarchOptions o;
  o.n_batches = n_batches;
  o.source_kind = source_kind;
  o.frequency = frequency;
  o.gmres = options;
  o.errors_u = errors;
  o.probes = probes;
  return march(mg.fine_operator(), &mg, u, v, o, s);
}

MarchResult march(const SpaceTimeOperator& op, const SpaceTimeMultigrid* mg, double* u, double* v,
                  const MarchOptions& mo, cudaStream_t s) {
  const int n_batches = mo.n_batches, source_kind = mo.source_kind;
  const double frequency = mo.frequency;
  const GmresOptions& options = mo.gmres;
  const ProbeSpec* probes = mo.probes;
  const bool wave = op.equation() == Equation::Wave;
  if (n_batches < 1) throw std::invalid_argument("march: n_batches must be >= 1");
  if (wave && !v) throw std::invalid_argument("march: the wave equation needs the initial velocity");
  const Index nx = op.n_space(), n = op.n_dofs();
  // homogeneous Dirichlet convention of the entering state (driver.cpp:158-166)
  op.zero_boundary_field(u, s);
  if (wave) op.zero_boundary_field(v, s);
  if (mo.errors_v && !wave) throw std::invalid_argument("march: velocity errors need the wave equation");
  DeviceBuffer rhs(sizeof(double) * n), x(sizeof(double) * n), uf(sizeof(double) * nx), vf(sizeof(double) * nx);
  DeviceBuffer vtraj;
  if (mo.errors_v) vtraj.allocate(sizeof(double) * n);
  GmresWorkspace ws;
  MarchResult res;
  ErrorRecord acc, acc_v;
  SectionClock* clk = mo.op_clock;
  const DeviceMap apply_op = [&op, clk](const double* in, double* out, cudaStream_t st) {
    if (clk) clk->begin(st);
    op.apply(in, out, st);
    if (clk) clk->end(st);
  };
  DeviceMap precond;
  if (mg) precond = [mg](const double* in, double* out, cudaStream_t st) { mg->apply(in, out, st); };
  // probes: located once on the finest mesh (locate_point), evaluated as
  // evaluate_fe of every temporal field and combined with the trial basis
  // weights at the sample times (value_at is linear)
  const int np = probes ? static_cast<int>(probes->xyz.size() / 3) : 0;
  const int F = op.desc().F, nt = op.n_t();
  DeviceBuffer pcells, pxi, pout;
  std::vector<double> hv(static_cast<size_t>(np) * (F + 1));
  auto probe = [&](const double* fields, int nf, long long fstride) {
    probe_fields(op.desc(), fields, nf, fstride, np, static_cast<const long long*>(pcells.raw()), pxi.d(), pout.d(), s);
    cuda_check(cudaMemcpyAsync(hv.data(), pout.raw(), sizeof(double) * np * nf, cudaMemcpyDeviceToHost, s), "probe");
    cuda_check(cudaStreamSynchronize(s), "probe");
  };
  if (np > 0) {
    std::vector<long long> cells(static_cast<size_t>(np));
    std::vector<double> xi(static_cast<size_t>(3 * np));
    for (int pi = 0; pi < np; ++pi) {
      Index cell = 0;
      locate_point(op.mesh(), probes->xyz.data() + 3 * pi, cell, xi.data() + 3 * pi);
      cells[static_cast<size_t>(pi)] = cell;
    }
    pcells = upload(cells);
    pxi = upload(xi);
    pout.allocate(sizeof(double) * static_cast<size_t>(np) * (F + 1));
    res.probe_values.assign(static_cast<size_t>(np), {});
    res.probe_times.push_back(0.0);
  }
  for (int b = 0; b < n_batches; ++b) {
    const double t0 = static_cast<double>(b) * op.n_steps() * op.tau();
    op.assemble_rhs(source_kind, frequency, t0, u, v, rhs.d(), s);
    vec_fill(x.d(), 0.0, n, s);
    const GmresResult r = gmres(apply_op, rhs.d(), x.d(), n, options, precond, ws, s);
    res.iterations.push_back(r.iterations);
    res.final_residuals.push_back(r.final_residual);
    res.batch_converged.push_back(r.converged ? 1 : 0);
    if (!r.converged) {
      res.converged = false;
      break;
    }
    if (mo.errors_u) accumulate_errors(op, x.d(), u, frequency, t0, acc, s, 3);
    if (mo.errors_v) {
      // the velocity trajectory entering from v, measured like u
      // (driver.cpp:213-223)
      op.velocity_trajectory(x.d(), u, v, vtraj.d(), s);
      accumulate_errors(op, vtraj.d(), v, frequency, t0, acc_v, s, 4);
    }
    if (np > 0) {
      // entering state, then the F fields of the batch
      probe(u, 1, nx);
      std::vector<double> u0v(static_cast<size_t>(np));
      for (int pi = 0; pi < np; ++pi) u0v[static_cast<size_t>(pi)] = hv[static_cast<size_t>(pi)];
      if (b == 0)
        for (int pi = 0; pi < np; ++pi) res.probe_values[static_cast<size_t>(pi)].push_back(u0v[static_cast<size_t>(pi)]);
      probe(x.d(), F, nx);
      const int ns = probes->samples_per_step;
      for (int st = 0; st < op.n_steps(); ++st)
        for (int j = 1; j <= ns; ++j) {
          const double tr = static_cast<double>(j) / ns;
          const double lw = op.weights().left_weight(tr);
          for (int pi = 0; pi < np; ++pi) {
            const double* fv = hv.data() + static_cast<size_t>(pi) * F;
            double val = 0.0;
            for (int i = 0; i < nt; ++i) val += op.weights().unknown_weight(i, tr) * fv[st * nt + i];
            if (lw != 0.0) val += lw * (st == 0 ? u0v[static_cast<size_t>(pi)] : fv[(st - 1) * nt + nt - 1]);
            res.probe_values[static_cast<size_t>(pi)].push_back(val);
          }
          res.probe_times.push_back(t0 + (st + tr) * op.tau());
        }
    }
    op.extract_final(x.d(), u, v, uf.d(), wave ? vf.d() : nullptr, s);
    vec_copy(u, uf.d(), nx, s);
    if (wave) vec_copy(v, vf.d(), nx, s);
  }
  cuda_check(cudaStreamSynchronize(s), "march");
  res.error_u = acc;
  res.error_u.l2_l2 = std::sqrt(acc.l2_l2);
  res.error_v = acc_v;
  res.error_v.l2_l2 = std::sqrt(acc_v.l2_l2);
  return res;
}

// ---------------------------------------------------- SpaceTimeMultigrid
namespace {
std::string coarsening_name(Coarsening c) {
  switch (c) {
    case Coarsening::SpaceH: return "space-h";
    case Coarsening::SpaceP: return "space-p";
    case Coarsening::TimeTau: return "time-tau";
    case Coarsening::TimeK: return "time-k";
  }
  return "?";
}
}  // namespace

SpaceTimeMultigrid::SpaceTimeMultigrid(Equation equation, TimeScheme scheme, const MeshHierarchy& mesh,
                                       const Coefficient& rho, const std::vector<LevelSpec>& plan,
                                       const MultigridOptions& options)
    : options_(options) {
  if (plan.empty()) throw std::invalid_argument("SpaceTimeMultigrid: empty plan");
  levels_.resize(plan.size());
  for (size_t l = 0; l < plan.size(); ++l) {
    Level& lv = levels_[l];
    lv.spec = plan[l];
    lv.weights = scheme == TimeScheme::DG ? dg_weights(lv.spec.k) : cgp_weights(lv.spec.k);
    lv.op = std::make_unique<SpaceTimeOperator>(equation, lv.weights, lv.spec.tau, lv.spec.n_steps, mesh,
                                                lv.spec.mesh_level, lv.spec.p, rho);
    const Index n = lv.op->n_dofs();
    lv.r.allocate(sizeof(double) * n);
    const bool coarsest = l + 1 == plan.size();
    if (!coarsest || levels_.size() == 1) {
      lv.smoother = std::make_unique<ASMSmoother>(*lv.op);
      lv.omega = estimate_relaxation(lv, options_.seed + l);
    }
    if (coarsest && n <= options_.direct_coarse_max) build_coarse_inverse(lv);
  }
  for (size_t l = 0; l + 1 < levels_.size(); ++l) {
    levels_[l].to_coarser = std::make_unique<Transfer>(*levels_[l].op, *levels_[l + 1].op);
    const Index nc = levels_[l + 1].op->n_dofs();
    levels_[l].rc.allocate(sizeof(double) * nc);
    levels_[l].ec.allocate(sizeof(double) * nc);
  }
}

double SpaceTimeMultigrid::estimate_relaxation(const Level& lv, std::uint64_t seed) const {
  // extremal Ritz values of P^-1 S from a short seeded Arnoldi run
  // (multigrid.cpp:127-172), modified Gram-Schmidt in the reference order
  const Index n = lv.op->n_dofs();
  const int m = static_cast<int>(std::min<Index>(options_.eig_iters, n));
  if (m <= 0) return 1.0;  // no Arnoldi steps: the unestimated relaxation factor
  Xoshiro256pp rng(seed);
  std::vector<double> hv(static_cast<size_t>(n));
  double nrm2 = 0.0;
  for (Index i = 0; i < n; ++i) {
    hv[static_cast<size_t>(i)] = rng.normal();
    nrm2 += hv[static_cast<size_t>(i)] * hv[static_cast<size_t>(i)];
  }
  if (nrm2 == 0.0) return 1.0;
  const double inv = 1.0 / std::sqrt(nrm2);
  for (double& x : hv) x *= inv;
  cudaStream_t s = nullptr;
  std::vector<DeviceBuffer> V;
  V.emplace_back(sizeof(double) * n);
  cuda_check(cudaMemcpy(V[0].raw(), hv.data(), sizeof(double) * n, cudaMemcpyHostToDevice), "arnoldi v0");
  DeviceBuffer w(sizeof(double) * n), z(sizeof(double) * n), ptrs(sizeof(double*)),
      scratch(sizeof(double) * kDotBlocks), out(sizeof(double));
  std::vector<double> H(static_cast<size_t>((m + 1) * m), 0.0);
  int kdim = 0;
  for (int j = 0; j < m; ++j) {
    lv.op->apply(V[j].d(), w.d(), s);
    vec_fill(z.d(), 0.0, n, s);
    lv.smoother->add_correction(w.d(), z.d(), s);
    for (int i = 0; i <= j; ++i) {
      const double h = host_dot(V[i].d(), z.d(), n, s, ptrs, scratch, out);
      H[static_cast<size_t>(i * m + j)] = h;
      vec_axpy(z.d(), -h, V[i].d(), n, s);
    }
    const double hn = std::sqrt(host_dot(z.d(), z.d(), n, s, ptrs, scratch, out));
    H[static_cast<size_t>((j + 1) * m + j)] = hn;
    kdim = j + 1;
    if (hn < 1e-13) break;
    V.emplace_back(sizeof(double) * n);
    vec_scale_into(V.back().d(), 1.0 / hn, z.d(), n, s);
  }
  if (kdim == 0) return 1.0;
  std::vector<double> Hk(static_cast<size_t>(kdim * kdim));
  for (int i = 0; i < kdim; ++i)
    for (int j = 0; j < kdim; ++j) Hk[static_cast<size_t>(i * kdim + j)] = H[static_cast<size_t>(i * m + j)];
  std::vector<std::pair<double, double>> ev;
  try {
    ev = eigenvalues_small(Hk, kdim);
  } catch (const std::exception&) {
    return 1.0;
  }
  double lmax = -1e300, lmin = 1e300;
  for (const auto& e : ev) {
    lmax = std::max(lmax, e.first);
    lmin = std::min(lmin, e.first);
  }
  lmin = std::max(0.0, lmin);
  const double omega = 2.0 / (lmax + lmin);
  if (!std::isfinite(omega) || omega <= 0.0) return 1.0;
  return std::min(omega, 1.0);
}

void SpaceTimeMultigrid::build_coarse_inverse(Level& lv) {
  // dense coarse matrix = matrix-free operator applied to the unit vectors,
  // inverted once with cuSOLVER (multigrid.cpp:112-120 uses SparseLU)
  const Index n = lv.op->n_dofs();
  cudaStream_t s = nullptr;
  DeviceBuffer Acm(sizeof(double) * n * n), e(sizeof(double) * n);
  vec_fill(e.d(), 0.0, n, s);
  for (Index j = 0; j < n; ++j) {
    vec_set_element(e.d(), j, 1.0, s);
    lv.op->apply(e.d(), Acm.d() + j * n, s);
    vec_set_element(e.d(), j, 0.0, s);
  }
  lv.coarse_inv.allocate(sizeof(double) * n * n);
  vec_fill(lv.coarse_inv.d(), 0.0, n * n, s);
  {
    // identity right-hand side
    std::vector<double> eye(static_cast<size_t>(n * n), 0.0);
    for (Index i = 0; i < n; ++i) eye[static_cast<size_t>(i * n + i)] = 1.0;
    cuda_check(cudaMemcpy(lv.coarse_inv.raw(), eye.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice), "eye");
  }
  cusolverDnHandle_t h = nullptr;
  solver_check(cusolverDnCreate(&h), "cusolverDnCreate");
  int lwork = 0;
  solver_check(cusolverDnDgetrf_bufferSize(h, static_cast<int>(n), static_cast<int>(n), Acm.d(), static_cast<int>(n),
                                           &lwork),
               "getrf_bufferSize");
  DeviceBuffer work(sizeof(double) * std::max(lwork, 1)), piv(sizeof(int) * n), info(sizeof(int));
  solver_check(cusolverDnDgetrf(h, static_cast<int>(n), static_cast<int>(n), Acm.d(), static_cast<int>(n), work.d(),
                                static_cast<int*>(piv.raw()), static_cast<int*>(info.raw())),
               "getrf");
  int hinfo = 0;
  cuda_check(cudaMemcpy(&hinfo, info.raw(), sizeof(int), cudaMemcpyDeviceToHost), "getrf info");
  if (hinfo != 0) throw std::runtime_error("SpaceTimeMultigrid: coarse factorization failed");
  // A^T X = I gives X = A^-T (column-major) = A^-1 read row-major
  solver_check(cusolverDnDgetrs(h, CUBLAS_OP_T, static_cast<int>(n), static_cast<int>(n), Acm.d(), static_cast<int>(n),
                                static_cast<int*>(piv.raw()), lv.coarse_inv.d(), static_cast<int>(n),
                                static_cast<int*>(info.raw())),
               "getrs");
  cuda_check(cudaDeviceSynchronize(), "coarse inverse");
  cusolverDnDestroy(h);
}

void SpaceTimeMultigrid::coarse_solve(const double* f, double* u, cudaStream_t s) const {
  const Level& lv = levels_.back();
  const Index n = lv.op->n_dofs();
  if (lv.coarse_inv.raw()) {
    dense_matvec(lv.coarse_inv.d(), f, u, static_cast<int>(n), s);
    return;
  }
  GmresOptions o;
  o.rel_tol = options_.coarse_rel_tol;
  o.abs_tol = 0.0;
  o.max_iters = options_.coarse_max_iters;
  vec_fill(u, 0.0, n, s);
  gmres([&lv](const double* x, double* y, cudaStream_t st) { lv.op->apply(x, y, st); }, f, u, n, o, DeviceMap{},
        coarse_ws_, s);
}

void SpaceTimeMultigrid::smooth(int l, const double* f, double* u, cudaStream_t s) const {
  // u += omega * ASM(f - S u) (multigrid.cpp:174-185): fused residual, and the
  // smoother scatters omega * W * (block solves) straight into u
  const Level& lv = levels_[static_cast<size_t>(l)];
  if (timers_) clock_smoother_.begin(s);
  lv.op->residual(f, u, lv.r.d(), s);
  lv.smoother->add_correction(lv.r.d(), u, s, lv.omega);
  if (timers_) clock_smoother_.end(s);
}

void SpaceTimeMultigrid::v_cycle(int l, const double* f, double* u, cudaStream_t s) const {
  // u enters as zero (multigrid.cpp:219,231), so the first residual is f
  const Level& lv = levels_[static_cast<size_t>(l)];
  if (l + 1 == n_levels()) {
    coarse_solve(f, u, s);
    return;
  }
  for (int i = 0; i < options_.n_smooth; ++i) {
    if (i == 0) {
      if (timers_) clock_smoother_.begin(s);
      lv.smoother->add_correction(f, u, s, lv.omega);  // S 0 = 0 exactly
      if (timers_) clock_smoother_.end(s);
    } else {
      smooth(l, f, u, s);
    }
  }
  lv.op->residual(f, u, lv.r.d(), s);
  lv.to_coarser->restrict_(lv.r.d(), lv.rc.d(), s);
  if (l == 0) {
    coarse_cycle(s);
  } else {
    const Index nc = levels_[static_cast<size_t>(l) + 1].op->n_dofs();
    vec_fill(lv.ec.d(), 0.0, nc, s);
    v_cycle(l + 1, lv.rc.d(), lv.ec.d(), s);
  }
  lv.to_coarser->prolong(lv.ec.d(), u, s, /*accumulate=*/true);
  for (int i = 0; i < options_.n_smooth; ++i) smooth(l, f, u, s);
}

SpaceTimeMultigrid::~SpaceTimeMultigrid() { reset_graph(); }

void SpaceTimeMultigrid::reset_graph() const {
  if (coarse_exec_) cudaGraphExecDestroy(coarse_exec_);
  coarse_exec_ = nullptr;
  coarse_nodes_ = 0;
}

void SpaceTimeMultigrid::coarse_cycle(cudaStream_t s) const {
  const Level& lv = levels_[0];
  const Index nc = levels_[1].op->n_dofs();
  auto direct = [&](cudaStream_t st) {
    vec_fill(lv.ec.d(), 0.0, nc, st);
    v_cycle(1, lv.rc.d(), lv.ec.d(), st);
  };
  static const bool disabled = std::getenv("STMG_NO_GRAPH") != nullptr;
  if (disabled || graph_failed_ || timers_) {
    direct(s);
    return;
  }
  if (!coarse_exec_) {
    // capture on a private stream; nothing executes during capture
    cudaStream_t cs = nullptr;
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess;
    const long long before = kernel_launches();
    if (ok) ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      try {
        direct(cs);
      } catch (...) {
        ok = false;
      }
      const cudaError_t e = cudaStreamEndCapture(cs, &g);
      ok = ok && e == cudaSuccess && g != nullptr;
    }
    coarse_nodes_ = kernel_launches() - before;
    count_launch(-coarse_nodes_);  // captured, not launched
    if (ok) ok = cudaGraphInstantiate(&coarse_exec_, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (cs) cudaStreamDestroy(cs);
    cudaGetLastError();  // a failed capture leaves a sticky-free error behind
    if (!ok) {
      coarse_exec_ = nullptr;
      graph_failed_ = true;
      direct(s);
      return;
    }
  }
  cuda_check(cudaGraphLaunch(coarse_exec_, s), "coarse cycle graph");
  count_launch(coarse_nodes_);
}

void SpaceTimeMultigrid::apply(const double* r, double* z, cudaStream_t s) const {
  if (timers_) clock_total_.begin(s);
  vec_fill(z, 0.0, fine_operator().n_dofs(), s);
  v_cycle(0, r, z, s);
  if (timers_) clock_total_.end(s);
}

void SpaceTimeMultigrid::enable_timers(bool on) {
  timers_ = on;
  reset_timers();
}

std::vector<LevelInfo> SpaceTimeMultigrid::level_info() const {
  std::vector<LevelInfo> info;
  for (size_t l = 0; l < levels_.size(); ++l) {
    const Level& lv = levels_[l];
    info.push_back({l == 0 ? std::string("finest") : coarsening_name(lv.spec.from_finer), lv.spec.mesh_level,
                    lv.spec.p, lv.spec.k, lv.spec.n_steps, lv.op->n_dofs(), lv.omega});
  }
  return info;
}

size_t SpaceTimeMultigrid::device_bytes() const {
  size_t b = 0;
  for (const Level& lv : levels_) {
    b += lv.r.bytes() + lv.rc.bytes() + lv.ec.bytes() + lv.coarse_inv.bytes();
    if (lv.smoother) b += lv.smoother->bytes();
  }
  return b;
}

}  // namespace stmgb
