// Host-side discretisation primitives for the B200 STMG path: quadrature,
// Lagrange bases, temporal weight tables, the space-time block coefficients,
// mesh hierarchies and multigrid level plans. Written from the published
// formulas; each function cites the reference routine whose results it must
// reproduce (paths relative to /root/reference/proj).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace stmgb {

using Index = std::int64_t;

enum class Equation : int { Heat = 0, Wave = 1 };
enum class TimeScheme : int { DG = 0, CGP = 1 };
enum class Coarsening : int { SpaceH = 0, SpaceP = 1, TimeTau = 2, TimeK = 3 };

struct Rule {
  std::vector<double> x, w;  // on [0,1], weights sum to 1
};

// src/quadrature.cpp:98-166
Rule gauss(int n);
Rule gauss_lobatto(int n);
Rule gauss_radau_right(int n);

// src/lagrange.cpp:20-42 (cardinal polynomials on strictly increasing nodes)
double lagrange_eval(const std::vector<double>& nodes, int i, double t);
double lagrange_deriv(const std::vector<double>& nodes, int i, double t);

// include/stmg/temporal_weights.hpp:11-51, src/temporal_weights.cpp:29-106.
// Matrices are n_t x n_t, row-major.
struct TemporalWeights {
  TimeScheme scheme = TimeScheme::DG;
  int k = 0;
  int n_t = 1;
  std::vector<double> m, a, alpha, beta;
  std::vector<double> trial_nodes;    // DG: Radau nodes; CGP: Lobatto incl. left node
  std::vector<double> unknown_nodes;  // reference times of the n_t unknowns
  double unknown_weight(int i, double t) const;
  double left_weight(double t) const;
};
TemporalWeights dg_weights(int k);
TemporalWeights cgp_weights(int k);

// Space-time block coefficients: the (S*n_t)^2 matrices CM, CA such that the
// batched operator is  S = CM (x) M_h + CA (x) A_h  with Dirichlet identity
// rows (src/space_time_operator.cpp:269-317, 319-352). Row-major, row index
// s*n_t+i, column index j*n_t+l.
void block_coefficient_matrices(Equation eq, const TemporalWeights& w, double tau, int n_steps,
                                std::vector<double>& CM, std::vector<double>& CA);

// Mesh hierarchy (include/stmg/mesh.hpp:17-60, src/mesh.cpp:148-187, 221-236):
// lexicographic vertices, x fastest; levels[0] coarsest.
struct MeshLevel {
  int dim = 1;
  std::array<Index, 3> cells{1, 1, 1};
  std::array<double, 3> lo{0, 0, 0}, hi{1, 1, 1};
  std::vector<double> vertices;  // n_verts*3; empty = exact Cartesian lattice
  // z-slab of a partitioned mesh: first cell layer in the global
  // level, and which z faces are physical boundaries (bit 0 low, bit 1 high)
  Index cz0 = 0;
  int zbc = 3;
  std::array<Index, 3> n_verts_axis() const {
    return {cells[0] + 1, dim > 1 ? cells[1] + 1 : 1, dim > 2 ? cells[2] + 1 : 1};
  }
  Index n_cells() const { return cells[0] * cells[1] * cells[2]; }
  Index n_verts() const {
    auto n = n_verts_axis();
    return n[0] * n[1] * n[2];
  }
};
struct MeshHierarchy {
  std::vector<MeshLevel> levels;
  // level-0 cells of the global mesh when the levels are slabs (coefficient
  // lookup); zero = levels.front().cells
  std::array<Index, 3> global_cells0{0, 0, 0};
  int n_levels() const { return static_cast<int>(levels.size()); }
};
MeshHierarchy make_cartesian(int dim, std::array<double, 3> lo, std::array<double, 3> hi, Index base_cells,
                             int refinements);
// per-axis base cell counts (box meshes of the weak-scaling study; the
// reference's make_cartesian is the cube case)
MeshHierarchy make_cartesian_box(int dim, std::array<double, 3> lo, std::array<double, 3> hi,
                                 std::array<Index, 3> base_cells, int refinements);
// Inject finest-level vertex positions; coarser levels take the positions of
// the vertices they share with the finest level (src/mesh.cpp:221-236).
void set_finest_vertices(MeshHierarchy& mesh, const double* xyz);
// Cartesian vertex coordinate along an axis (src/mesh.cpp:171-184)
double cartesian_coord(const MeshLevel& m, int axis, Index i);
// locate_point (spatial_operator.cpp:475-524): the first cell (lexicographic)
// whose d-linear map reaches x by Newton iteration from the cell centre,
// with its reference coordinates; throws when x is outside the mesh
void locate_point(const MeshLevel& m, const double x[3], Index& cell, double xi[3]);

// Level plans (include/stmg/multigrid.hpp:18-38, src/multigrid.cpp:34-81)
struct LevelSpec {
  int mesh_level = 0;
  int p = 1;
  int k = 0;
  int n_steps = 1;
  double tau = 1.0;
  Coarsening from_finer = Coarsening::SpaceH;
};
std::vector<Coarsening> default_strategy(const LevelSpec& finest, TimeScheme scheme);
std::vector<LevelSpec> build_level_plan(const LevelSpec& finest, TimeScheme scheme,
                                        const std::vector<Coarsening>& strategy);

// xoshiro256++ with splitmix64 seeding and Box-Muller normals: the published
// generator the reference uses for its Arnoldi start vectors
// (include/stmg/rng.hpp:11-82)
class Xoshiro256pp {
 public:
  explicit Xoshiro256pp(std::uint64_t seed);
  std::uint64_t next();
  double uniform();
  double normal();

 private:
  std::uint64_t s_[4];
  double cached_ = 0.0;
  bool have_cached_ = false;
};

// small dense helpers (row-major)
std::vector<double> invert_small(const std::vector<double>& a, int n);
std::vector<double> matmul_small(const std::vector<double>& a, const std::vector<double>& b, int n, int k, int m);

}  // namespace stmgb

namespace stmgb {
// Tensor-product FDM tables for one lattice axis of a Cartesian level with
// spacing h and degree p: for the four position classes of a cell along the
// axis (0 interior, 1 first, 2 last, 3 single) the generalised eigenpairs
// K_r S = M_r S Lambda (S^T M_r S = I) of the restricted global 1D stiffness
// K_r and mass M_r on the cell's p+1 nodes; Dirichlet end nodes are removed
// (their rows/columns of S are zero, Lambda = 0). S is row-major [node][eig].
void fdm_axis_tables(int p, double h, double S[4][5][5], double lam[4][5]);
// symmetric eigen-decomposition by cyclic Jacobi rotations (small n):
// A = V diag(w) V^T, V row-major [i][eig]
std::vector<double> sym_eigen_jacobi(std::vector<double> A, int n, std::vector<double>& V);
}  // namespace stmgb
