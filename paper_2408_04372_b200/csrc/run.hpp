// One configured run on the device: the reference's ProblemSpec / RunReport
// and march(spec, probes) (include/stmg/driver.hpp:14-91, src/driver.cpp:95-262)
// with the mesh perturbation and coefficient fields it builds on
// (src/mesh.cpp:42-57, 59-111, 190-240, 254-298). Every batch stays on the
// device; the section times are device times of the same sections.
#pragma once

#include <cstdint>
#include <vector>

#include "stmg.hpp"

namespace stmgb {

// problem families of make_problem (src/config.cpp:175-211)
enum class ProblemKind : int { Manufactured = 0, Shm = 1, Zero = 2 };

struct ProblemSpec {
  Equation equation = Equation::Heat;
  TimeScheme scheme = TimeScheme::DG;
  ProblemKind problem = ProblemKind::Manufactured;
  int k = 1, p = 1, dim = 2;
  std::array<double, 3> lo{0.0, 0.0, 0.0}, hi{1.0, 1.0, 1.0};
  double t_final = 1.0;
  int refinements = 2, base_cells = 2, base_time_intervals = 1, batch = 1;
  double frequency = 2.0;  // manufactured: om = 2 pi frequency
  double shm_s = 0.3;      // shm: pulse radius
  double perturb = 0.0;
  std::uint64_t seed = 42;
  double rho_random_lo = 0.0, rho_random_hi = 0.0;  // per level-0 cell scaling when hi > lo > 0
  double abs_tol = 1e-12, rel_tol = 1e-12;
  int max_iters = 1000, restart = 100, n_smooth = 1;
  bool precondition = true;
  int probe_samples_per_step = 16;
  std::vector<Coarsening> strategy;  // empty = default_strategy
  bool timers = true;                // record the profile sections
};

struct BatchStats {
  int iterations = 0;
  double final_residual = 0.0;
  bool converged = false;
};

struct SectionTimes {
  double total = 0.0, smoother = 0.0, gmg_wo_smoother = 0.0, operator_wo_gmg = 0.0, other = 0.0;
};

struct RunReport {
  bool converged = false;
  Index n_space_dofs = 0;
  int n_steps_total = 0, n_batches = 0;
  Index dofs_global = 0;
  std::vector<BatchStats> batches;
  double mean_iterations = 0.0;
  double work = 0.0;  // sum over batches of (batch * n_t) * n_space * iterations
  bool has_error_u = false, has_error_v = false;
  ErrorRecord error_u, error_v;
  std::vector<LevelInfo> hierarchy;
  SectionTimes sections;
  std::vector<double> probe_times;
  std::vector<std::vector<double>> probe_values;
};

// perturb (src/mesh.cpp:190-240): every finest vertex moves by
// magnitude * (shortest adjacent edge) along a xoshiro256++ direction,
// boundary vertices only tangentially; coarse levels copy the shared
// vertices; throws when a cell inverts (check_positive_jacobians)
void perturb_mesh(MeshHierarchy& mesh, double magnitude, std::uint64_t seed);
// check_positive_jacobians (src/mesh.cpp:92-111): 5 samples per axis
void check_positive_jacobians(const MeshLevel& m);
// the problem's coefficient as a per level-0 cell field (the only form the
// device operator takes): 1 (manufactured, zero) or coefficient_shm
// (src/mesh.cpp:267-279) when its jumps lie on level-0 cell faces, times
// randomize_coefficient (src/mesh.cpp:281-298) when enabled
Coefficient problem_coefficient(const ProblemSpec& spec, const MeshHierarchy& mesh);
// march(spec, probes) (src/driver.cpp:95-262); probes: 3 coordinates each
RunReport run_march(const ProblemSpec& spec, const std::vector<double>& probes, cudaStream_t stream = nullptr);

}  // namespace stmgb
