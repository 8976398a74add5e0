// Host C++ layer of the B200 STMG path. The classes mirror the reference's
// operator / smoother / transfer / multigrid / GMRES interfaces (same names,
// argument meaning, overwrite-vs-accumulate semantics and exceptions), but
// operate on device-resident vectors and launch the sm_100a kernels:
//   SpaceTimeOperator   include/stmg/space_time_operator.hpp:34-105
//   ASMSmoother         include/stmg/asm_smoother.hpp:16-45
//   Transfer            include/stmg/transfer.hpp:22-40
//   SpaceTimeMultigrid  include/stmg/multigrid.hpp:61-113
//   gmres               include/stmg/gmres.hpp:9-33
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "device.cuh"
#include "kernels.hpp"
#include "setup.hpp"

namespace stmgb {

void cuda_check(cudaError_t e, const char* what);
// host <-> device copies of the host-buffer entry points (host_xfer.cpp):
// pinned-chunk pipeline with parallel host copies; synchronous on return
void copy_to_device(double* d_dst, const double* h_src, size_t bytes, cudaStream_t s);
void copy_to_host(double* h_dst, const double* d_src, size_t bytes, cudaStream_t s);

// owning device buffer of doubles (or raw bytes)
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes);
  ~DeviceBuffer();
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept;
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept;
  void allocate(size_t bytes);
  void release();
  double* d() const { return static_cast<double*>(p_); }
  void* raw() const { return p_; }
  size_t bytes() const { return bytes_; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

// cell-wise positive coefficient: rho(cell) = coarse_cell_scale[ancestor on
// mesh level 0] (include/stmg/mesh.hpp:76-83 with base == 1)
struct Coefficient {
  std::vector<double> coarse_cell_scale;  // empty = 1
};

class SpaceTimeOperator {
 public:
  SpaceTimeOperator(Equation equation, const TemporalWeights& weights, double tau, int n_steps,
                    const MeshHierarchy& mesh, int mesh_level, int p, const Coefficient& rho);

  Equation equation() const { return equation_; }
  const TemporalWeights& weights() const { return weights_; }
  double tau() const { return tau_; }
  int n_steps() const { return n_steps_; }
  int n_t() const { return weights_.n_t; }
  int p() const { return p_; }
  int dim() const { return desc_.dim; }
  int mesh_level() const { return mesh_level_; }
  Index n_space() const { return desc_.n_space; }
  Index n_dofs() const { return desc_.n_dofs; }
  Index block_offset(int step, int node) const { return (static_cast<Index>(step) * weights_.n_t + node) * n_space(); }
  const DevLevel& desc() const { return desc_; }
  const MeshLevel& mesh() const { return *mesh_level_ptr_; }

  // y = S u (overwrite), device pointers (space_time_operator.cpp:45-130)
  void apply(const double* u, double* y, cudaStream_t stream = nullptr) const;
  // SpatialOperator::apply of the constrained mass (kind 0) or stiffness (1)
  void spatial_apply(int kind, const double* u, double* y, cudaStream_t stream = nullptr) const;
  // r = f - S u (overwrite), one fused pass
  void residual(const double* f, const double* u, double* r, cudaStream_t stream = nullptr) const;
  // nodal interpolant of a known function on this level's Q_p lattice
  // (interpolate, spatial_operator.cpp:437-449); kinds as interpolate_nodes
  void interpolate(int kind, double frequency, double t, const double* centre, double width, bool zero_boundary,
                   double* out, cudaStream_t stream = nullptr) const;
  // assemble_rhs (space_time_operator.cpp:138-221): source_kind 0 zero,
  // 1 manufactured (driver.cpp:265-293, frequency f); entering state u0 (v0)
  void assemble_rhs(int source_kind, double frequency, double t0, const double* u0, const double* v0, double* rhs,
                    cudaStream_t stream = nullptr) const;
  // extract_final (space_time_operator.cpp:223-248)
  void extract_final(const double* u, const double* u0, const double* v0, double* uf, double* vf,
                     cudaStream_t stream = nullptr) const;
  // velocity_trajectory (driver.cpp:47-82, wave only): the velocity node
  // values of every (step, temporal node) of a batch solution u entering
  // from (u0, v0), in the layout of u (overwrite vout, n_dofs)
  void velocity_trajectory(const double* u, const double* u0, const double* v0, double* vout,
                           cudaStream_t stream = nullptr) const;
  void zero_boundary_field(double* v, cudaStream_t stream = nullptr) const;
  // value_at (space_time_operator.cpp:250-266): the discrete trajectory of
  // step `step` at reference time t_ref, entering state u0 (n_space)
  void value_at(const double* u, const double* u0, int step, double t_ref, double* out,
                cudaStream_t stream = nullptr) const;
  // sample_spatial_error (spatial_operator.cpp:526-557) of a nodal field
  // against the manufactured solution (kind 3: u, 4: v) at time t with the
  // (p+2)^d Gauss rule: {sum w |J| e^2, max |e|}
  std::pair<double, double> spatial_error(const double* field, int kind, double frequency, double t,
                                          cudaStream_t stream = nullptr) const;
  long applications() const { return apply_count_; }
  // the F x F block coefficient tables CM, CA (row-major, F = S n_t)
  const std::vector<double>& block_cm() const { return cm_; }
  const std::vector<double>& block_ca() const { return ca_; }
  bool wide() const { return wide_; }

 private:
  Equation equation_;
  TemporalWeights weights_;
  double tau_;
  int n_steps_;
  int mesh_level_;
  int p_;
  const MeshLevel* mesh_level_ptr_;
  DevLevel desc_{};
  DevLevel mass_desc_{}, stiff_desc_{};
  DeviceBuffer verts_, rho0_;
  mutable long apply_count_ = 0;
  // S * n_t > kMaxF ("wide" batches): composed application, see st_apply_wide
  bool wide_ = false;
  std::vector<double> cm_, ca_;  // full F x F block coefficients
  DeviceBuffer wide_cm_, wide_ca_;
  mutable DeviceBuffer wide_mu_, wide_au_;
};

class ASMSmoother {
 public:
  // probe_op: for a z-slab with interfaces, the slab extended by one halo
  // cell layer across each interface (probe_zcells of them below), used only
  // to extract the restricted global block matrices at setup
  explicit ASMSmoother(const SpaceTimeOperator& op, const SpaceTimeOperator* probe_op = nullptr,
                       int probe_zcells = 0);
  // correction += W sum_T R_T^T B_T^-1 R_T residual (accumulate; the
  // relaxation factor is applied by the caller) -- asm_smoother.cpp:60-78
  void add_correction(const double* residual, double* correction, cudaStream_t stream = nullptr,
                      double scale = 1.0) const;
  int block_size() const { return op_->n_t() * asm_.m; }
  Index n_blocks() const { return static_cast<Index>(op_->n_steps()) * op_->mesh().n_cells(); }
  long sweeps() const { return sweep_count_; }
  size_t bytes() const { return X_.bytes() + lam_.bytes() + list_.bytes() + skip_.bytes() + meta_.bytes() + left_.bytes(); }
  // cells solved by tensor FDM / by the per-cell eigenbasis; exact() is false
  // when some block is only approximated (non-uniform coefficient around a
  // (p+1)^3 > 64 cell)
  bool uses_fdm() const { return use_fdm_; }
  Index n_exact_cells() const { return asm_.n_list; }
  bool exact() const { return exact_; }
  // bit 0: tensor FDM cells, bit 1: per-cell eigenbasis cells, bit 2: the
  // eigenbasis kernel also fast-diagonalises the temporal solves
  int kind() const { return (use_fdm_ ? 1 : 0) | (asm_.n_list > 0 ? 2 : 0) | (asm_.n_list > 0 && asm_.tdiag && asm_.meta ? 4 : 0); }

 private:
  void build_exact(const SpaceTimeOperator& op, const SpaceTimeOperator* probe_op, int probe_zcells);
  void build_exact_large(DeviceBuffer& cellM, DeviceBuffer& cellA, cudaStream_t s);
  const SpaceTimeOperator* op_;
  DevASM asm_{};
  DevASM chunk_{}, tail_{};  // S * n_t > 8: step groups of chunk_.S steps (tail_: the rest)
  DevFDM fdm_{};
  bool use_fdm_ = false;
  bool exact_ = true;
  DeviceBuffer X_, lam_, list_, skip_, meta_, left_;
  mutable long sweep_count_ = 0;
};

class Transfer {
 public:
  Transfer(const SpaceTimeOperator& fine, const SpaceTimeOperator& coarse);
  // overwrite (accumulate = false, the reference semantics) or fine += P coarse;
  // coarse_fstride > 0: the coarse vector is a slab view inside a longer one
  // (field stride coarse_fstride). On a z-slab whose low plane is an interface
  // owned by the slab below, restriction skips that fine plane so the
  // interface sum over both slabs counts it once.
  void prolong(const double* coarse, double* fine, cudaStream_t stream = nullptr, bool accumulate = false,
               long long coarse_fstride = 0) const;
  void restrict_(const double* fine, double* coarse, cudaStream_t stream = nullptr, bool accumulate = false,
                 long long coarse_fstride = 0) const;
  bool spatial() const { return spatial_; }

 private:
  const SpaceTimeOperator* fine_;
  const SpaceTimeOperator* coarse_;
  bool spatial_ = true;
  DevAxisTransfer ax_[3]{};
  std::vector<DeviceBuffer> bufs_;
  mutable DeviceBuffer t1_, t2_;  // separable-pass work buffers
  DeviceBuffer time_p_;
  int Ff_ = 0, Fc_ = 0;
};

struct MultigridOptions {
  int n_smooth = 1;
  Index direct_coarse_max = 20000;
  double coarse_rel_tol = 1e-3;
  int coarse_max_iters = 2000;
  int eig_iters = 20;
  std::uint64_t seed = 42;
};

struct LevelInfo {
  std::string coarsening;
  int mesh_level, p, k, n_steps;
  Index n_dofs;
  double omega;
};

struct GmresOptions {
  int max_iters = 1000;
  int restart = 100;
  double rel_tol = 1e-12;
  double abs_tol = 1e-12;
};
struct GmresResult {
  bool converged = false;
  int iterations = 0;
  double initial_residual = 0.0;
  double final_residual = 0.0;
  std::vector<double> residual_history;
};
// device-vector linear map y = A x (overwrite)
using DeviceMap = std::function<void(const double*, double*, cudaStream_t)>;

// Krylov workspace reused across solves (basis vectors allocated lazily)
class GmresWorkspace {
 public:
  void ensure(Index n, int vectors);
  double* vec(int i) const { return basis_[static_cast<size_t>(i)].d(); }
  const double* const* dev_ptrs() const { return static_cast<const double* const*>(ptrs_.raw()); }
  double* scratch() const { return scratch_.d(); }
  double* small() const { return small_.d(); }
  double* r() const { return r_.d(); }
  double* w() const { return w_.d(); }
  double* z() const { return z_.d(); }
  Index n() const { return n_; }

 private:
  Index n_ = 0;
  std::vector<DeviceBuffer> basis_;
  DeviceBuffer ptrs_, scratch_, small_, r_, w_, z_;
};

// Inner products of a distributed vector (z-slab partition): only the owned
// entries (segments) count locally, then the k partial sums are summed over
// the ranks in place on the device (allreduce; empty = single process)
struct DotPolicy {
  DotSegments seg{};
  std::function<void(double* d_vals, int k, cudaStream_t)> allreduce;
};

// Restarted right-preconditioned GMRES (gmres.cpp:8-115) on device vectors.
GmresResult gmres(const DeviceMap& op, const double* b, double* x, Index n, const GmresOptions& options,
                  const DeviceMap& precond, GmresWorkspace& ws, cudaStream_t stream = nullptr,
                  const DotPolicy* dots = nullptr);

// error norms over time slabs (driver.hpp:49-52, driver.cpp:18-43):
// accumulate with accumulate_errors, then l2_l2 = sqrt(sum)
struct ErrorRecord {
  double l2_l2 = 0.0, linf_l2 = 0.0, linf_linf = 0.0;
};
// accumulate_errors (driver.cpp:27-43): temporal Gauss (k+2) x spatial Gauss
// (p+2) sample of one batch solution x entering from u0 against the
// manufactured solution of frequency f; acc.l2_l2 holds the squared sum
// (kind 3: u = sin(om t) prod sin(om x_a); kind 4: its velocity)
void accumulate_errors(const SpaceTimeOperator& op, const double* x, const double* u0, double frequency, double t0,
                       ErrorRecord& acc, cudaStream_t stream = nullptr, int kind = 3);

// Device time of one profile section: the reference's wall-clock section
// accounting (multigrid.hpp:85-88, driver.cpp:186-196) restated with CUDA
// event pairs recorded on the launching stream and folded into the total
// when read (or when the pool fills)
class SectionClock {
 public:
  SectionClock() = default;
  SectionClock(const SectionClock&) = delete;
  SectionClock& operator=(const SectionClock&) = delete;
  ~SectionClock();
  void begin(cudaStream_t stream);
  void end(cudaStream_t stream);
  double seconds();  // waits for the recorded events
  void reset();

 private:
  void fold();
  std::vector<cudaEvent_t> ev_;
  size_t used_ = 0;
  double total_ = 0.0;
};

class SpaceTimeMultigrid;
// march (driver.cpp:95-260) with every slab on the device: per batch
// assemble_rhs -> STMG-preconditioned GMRES -> (errors) -> extract_final.
// u (and v for the wave equation) hold the entering state on input (device,
// n_space each; Dirichlet entries are zeroed first) and the final state on
// output.
struct MarchResult {
  std::vector<int> iterations;  // per batch run (the last one may not have converged)
  std::vector<double> final_residuals;
  std::vector<char> batch_converged;
  bool converged = true;
  ErrorRecord error_u;  // finished (l2_l2 = sqrt of the sum)
  ErrorRecord error_v;  // velocity errors (wave, errors_v)
  // probe time series (driver.cpp:146-186, 226-236): times, and per probe
  // the value at t = 0 and at samples_per_step points of every step
  std::vector<double> probe_times;
  std::vector<std::vector<double>> probe_values;
};
struct ProbeSpec {
  std::vector<double> xyz;  // 3 per point
  int samples_per_step = 16;
};
MarchResult march(const SpaceTimeMultigrid& mg, int n_batches, int source_kind, double frequency, double* u, double* v,
                  const GmresOptions& options, bool errors, cudaStream_t stream = nullptr,
                  const ProbeSpec* probes = nullptr);
// the general form: op with an optional preconditioner (spec.precondition,
// driver.cpp:121-137, 197-201), velocity errors against the manufactured
// velocity (driver.cpp:213-223), and op_clock timing every operator
// application inside GMRES (the "Operator w/o GMG" section, driver.cpp:193-196)
struct MarchOptions {
  int n_batches = 1;
  int source_kind = 1;
  double frequency = 0.5;
  GmresOptions gmres;
  bool errors_u = false;
  bool errors_v = false;
  const ProbeSpec* probes = nullptr;
  SectionClock* op_clock = nullptr;
};
MarchResult march(const SpaceTimeOperator& op, const SpaceTimeMultigrid* mg, double* u, double* v,
                  const MarchOptions& options, cudaStream_t stream = nullptr);

class SpaceTimeMultigrid {
 public:
  SpaceTimeMultigrid(Equation equation, TimeScheme scheme, const MeshHierarchy& mesh, const Coefficient& rho,
                     const std::vector<LevelSpec>& plan, const MultigridOptions& options = {});
  int n_levels() const { return static_cast<int>(levels_.size()); }
  const SpaceTimeOperator& fine_operator() const { return *levels_[0].op; }
  const SpaceTimeOperator& operator_at(int l) const { return *levels_[l].op; }
  const ASMSmoother& smoother_at(int l) const { return *levels_[l].smoother; }
  const Transfer& transfer_at(int l) const { return *levels_[l].to_coarser; }
  double omega_at(int l) const { return levels_[l].omega; }
  void set_omega(int l, double w) {
    levels_[l].omega = w;
    reset_graph();  // omega is baked into the captured launches
  }
  ~SpaceTimeMultigrid();
  SpaceTimeMultigrid(const SpaceTimeMultigrid&) = delete;
  SpaceTimeMultigrid& operator=(const SpaceTimeMultigrid&) = delete;
  std::vector<LevelInfo> level_info() const;
  // one V-cycle from the finest level, zero initial guess (overwrite z)
  void apply(const double* r, double* z, cudaStream_t stream = nullptr) const;
  void v_cycle(int l, const double* f, double* u, cudaStream_t stream) const;
  void smooth(int l, const double* f, double* u, cudaStream_t stream) const;
  size_t device_bytes() const;
  // profile sections (multigrid.hpp:85-88): device seconds inside apply() and
  // inside the smoothing steps; while enabled the coarse cycle runs as plain
  // launches so every smoothing step is bracketed by its own events
  void enable_timers(bool on);
  double seconds_total() const { return clock_total_.seconds(); }
  double seconds_smoother() const { return clock_smoother_.seconds(); }
  void reset_timers() const {
    clock_total_.reset();
    clock_smoother_.reset();
  }

 private:
  struct Level {
    LevelSpec spec;
    TemporalWeights weights;
    std::unique_ptr<SpaceTimeOperator> op;
    std::unique_ptr<ASMSmoother> smoother;
    std::unique_ptr<Transfer> to_coarser;
    double omega = 1.0;
    DeviceBuffer coarse_inv;  // dense inverse of the coarsest operator
    mutable DeviceBuffer r, rc, ec;  // work vectors: residual, restricted residual, coarse correction
  };
  double estimate_relaxation(const Level& lv, std::uint64_t seed) const;
  void coarse_solve(const double* f, double* u, cudaStream_t stream) const;
  void build_coarse_inverse(Level& lv);
  // the sub-cycle below the finest level (fixed internal buffers) replayed as
  // one CUDA graph; captured on first use, plain launches if capture fails
  void coarse_cycle(cudaStream_t stream) const;
  void reset_graph() const;
  mutable cudaGraphExec_t coarse_exec_ = nullptr;
  mutable long long coarse_nodes_ = 0;
  mutable bool graph_failed_ = false;
  bool timers_ = false;
  mutable SectionClock clock_total_, clock_smoother_;

  MultigridOptions options_;
  std::vector<Level> levels_;
  mutable GmresWorkspace coarse_ws_;
};

// eigenvalues (real, imag) of a small dense real matrix (row-major n x n):
// Hessenberg reduction + shifted QR, as needed for the Ritz values of the
// relaxation estimate (multigrid.cpp:156-171)
std::vector<std::pair<double, double>> eigenvalues_small(std::vector<double> a, int n);
void temporal_block_diagonalise(DevASM& A);

}  // namespace stmgb
