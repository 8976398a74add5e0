/*
 * stmg_b200.h -- C ABI of the B200-native space-time multigrid (STMG) solve
 * path (arXiv 2408.04372). Plain pointers and sizes only; every compute entry
 * point takes DEVICE pointers plus a cudaStream_t passed as void* (NULL = the
 * legacy default stream), except the *_host variants, which take host buffers
 * and do the host<->device copies themselves. All vectors use the reference's
 * layout: index (s*n_t + i)*n_space + g, spatial lattice x fastest
 * (include/stmg/space_time_operator.hpp:23-29,43-45 of the reference).
 *
 * Every function returns 0 on success and a negative code on failure; the
 * message is available from stmg_last_error() (the reference throws
 * std::invalid_argument / std::runtime_error instead).
 * Codes: -1 invalid argument, -2 runtime/numerical failure, -3 CUDA error.
 *
 * Each entry point names the reference interface it replaces; paths are
 * relative to /root/reference/proj.
 */
#ifndef STMG_B200_H
#define STMG_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct stmg_mesh stmg_mesh;
typedef struct stmg_st_operator stmg_st_operator;
typedef struct stmg_asm stmg_asm;
typedef struct stmg_transfer stmg_transfer;
typedef struct stmg_multigrid stmg_multigrid;

enum { STMG_HEAT = 0, STMG_WAVE = 1 };                 /* Equation, space_time_operator.hpp:12 */
enum { STMG_DG = 0, STMG_CGP = 1 };                    /* TimeScheme, temporal_weights.hpp:9 */
enum { STMG_SPACE_H = 0, STMG_SPACE_P = 1, STMG_TIME_TAU = 2, STMG_TIME_K = 3 }; /* Coarsening, multigrid.hpp:14 */

const char* stmg_last_error(void);
const char* stmg_version(void);
/* number of sm_100a kernels this library has launched since it was loaded */
long long stmg_kernel_launches(void);

/* Host-side discretisation tables (no GPU needed), for parity checks:
 * quadrature rules on [0,1] (src/quadrature.cpp:98-166; kind 0 Gauss,
 * 1 Gauss-Lobatto, 2 right Gauss-Radau), temporal weights
 * (src/temporal_weights.cpp:29-106; n_t x n_t row-major) and the slab block
 * coefficients CM, CA ((S n_t)^2 row-major, src/space_time_operator.cpp:269-317). */
int stmg_quadrature(int kind, int n, double* points, double* weights);
int stmg_temporal_weights(int scheme, int k, double* m_tau, double* a_tau, double* alpha, double* beta,
                          double* unknown_nodes);
int stmg_block_coefficients(int equation, int scheme, int k, double tau, int n_steps, double* CM, double* CA);

/* MeshHierarchy: make_cartesian (src/mesh.cpp:148-187). finest_vertices
 * (n_verts*3 doubles, x fastest) may be NULL for the exact Cartesian lattice;
 * otherwise they replace the finest level's vertices and coarser levels take
 * the shared positions (src/mesh.cpp:221-236). */
int stmg_mesh_create(int dim, const double lo[3], const double hi[3], long long base_cells, int refinements,
                     const double* finest_vertices, stmg_mesh** out);
/* box mesh with per-axis base cell counts (no reference counterpart: the
 * weak-scaling study's 128^2 x 256 ... 256^3 meshes; the cube case is
 * stmg_mesh_create) */
int stmg_mesh_create_box(int dim, const double lo[3], const double hi[3], const long long base_cells[3],
                         int refinements, const double* finest_vertices, stmg_mesh** out);
void stmg_mesh_destroy(stmg_mesh* mesh);

/* SpaceTimeOperator ctor (include/stmg/space_time_operator.hpp:34-36) with its
 * SpatialOperator pair built on mesh level `mesh_level` with degree p; the
 * coefficient is coarse_cell_scale[level-0 ancestor] (CoefficientField,
 * include/stmg/mesh.hpp:76-83), NULL = 1. */
int stmg_st_operator_create(const stmg_mesh* mesh, int mesh_level, int p, int equation, int scheme, int k, double tau,
                            int n_steps, const double* coarse_cell_scale, stmg_st_operator** out);
void stmg_st_operator_destroy(stmg_st_operator* op);
long long stmg_st_operator_n_dofs(const stmg_st_operator* op);  /* n_dofs(), space_time_operator.hpp:42 */
long long stmg_st_operator_n_space(const stmg_st_operator* op); /* n_space(), :41 */
int stmg_st_operator_n_t(const stmg_st_operator* op);           /* n_t(), :40 */
/* SpaceTimeOperator::apply (space_time_operator.cpp:45-130): y = S u, overwrite */
int stmg_st_operator_apply(const stmg_st_operator* op, const double* d_u, double* d_y, void* stream);
int stmg_st_operator_apply_host(const stmg_st_operator* op, const double* h_u, double* h_y);
/* SpatialOperator::apply (spatial_operator.cpp:292-315), kind 0 mass / 1 stiffness */
int stmg_spatial_apply(const stmg_st_operator* op, int kind, const double* d_u, double* d_y, void* stream);
/* r = f - S u in one fused pass (the residual of multigrid.cpp:181,215) */
int stmg_st_operator_residual(const stmg_st_operator* op, const double* d_f, const double* d_u, double* d_r,
                              void* stream);
/* interpolate (spatial_operator.cpp:437-449) of a known function at the Q_p
 * support points into d_out (n_space): kind 0 manufactured heat source,
 * 1 manufactured wave source, 2 Gaussian exp(-|x-centre|^2/(2 width^2)),
 * 3 manufactured solution, 4 manufactured velocity (driver.cpp:265-293,
 * omega = 2 pi frequency), 5 the shm pulse exp(-r^2)(1-r^2), r = |x|/width < 1
 * (driver.cpp:295-316); zero_boundary sets the Dirichlet entries to 0 */
int stmg_st_operator_interpolate(const stmg_st_operator* op, int kind, double frequency, double t,
                                 const double centre[3], double width, int zero_boundary, double* d_out,
                                 void* stream);
/* assemble_rhs (space_time_operator.cpp:138-221): source_kind 0 zero source,
 * 1 manufactured source; entering state d_u0 (and d_v0 for the wave) */
int stmg_st_operator_assemble_rhs(const stmg_st_operator* op, int source_kind, double frequency, double t0,
                                  const double* d_u0, const double* d_v0, double* d_rhs, void* stream);
/* extract_final (space_time_operator.cpp:223-248): state after the slab */
int stmg_st_operator_extract_final(const stmg_st_operator* op, const double* d_u, const double* d_u0,
                                   const double* d_v0, double* d_uf, double* d_vf, void* stream);

/* ASMSmoother (include/stmg/asm_smoother.hpp:16-30) */
int stmg_asm_create(const stmg_st_operator* op, stmg_asm** out);
void stmg_asm_destroy(stmg_asm* a);
/* add_correction (asm_smoother.cpp:60-78): d_z += W sum_T R_T^T B_T^-1 R_T d_r (accumulate) */
int stmg_asm_add_correction(const stmg_asm* a, const double* d_r, double* d_z, void* stream);

/* Transfer (include/stmg/transfer.hpp:22-24) between two operators that
 * differ in exactly one attribute */
int stmg_transfer_create(const stmg_st_operator* fine, const stmg_st_operator* coarse, stmg_transfer** out);
void stmg_transfer_destroy(stmg_transfer* t);
int stmg_transfer_prolong(const stmg_transfer* t, const double* d_coarse, double* d_fine, void* stream);
int stmg_transfer_restrict(const stmg_transfer* t, const double* d_fine, double* d_coarse, void* stream);

/* MultigridOptions (include/stmg/multigrid.hpp:39-46) */
typedef struct {
  int n_smooth;
  long long direct_coarse_max;
  double coarse_rel_tol;
  int coarse_max_iters;
  int eig_iters;
  unsigned long long seed;
} stmg_mg_options;
void stmg_mg_options_default(stmg_mg_options* o);

/* SpaceTimeMultigrid ctor (multigrid.cpp:83-125) for the plan
 * build_level_plan(finest, scheme, strategy) (multigrid.cpp:34-81);
 * n_strategy < 0 selects default_strategy. */
int stmg_multigrid_create(int equation, int scheme, const stmg_mesh* mesh, const double* coarse_cell_scale,
                          int fine_mesh_level, int p, int k, int n_steps, double tau, int n_strategy,
                          const int* strategy, const stmg_mg_options* options, stmg_multigrid** out);
void stmg_multigrid_destroy(stmg_multigrid* mg);
int stmg_multigrid_n_levels(const stmg_multigrid* mg);
/* level_info (multigrid.cpp:236-247): ints = {mesh_level, p, k, n_steps, coarsening(-1 finest)} */
int stmg_multigrid_level_info(const stmg_multigrid* mg, int level, int ints[5], long long* n_dofs, double* omega);
int stmg_multigrid_set_omega(stmg_multigrid* mg, int level, double omega);
/* which cell-solve kernels the level-l smoother runs (no reference counterpart;
   diagnostics): bit 0 tensor FDM, bit 1 per-cell eigenbasis, bit 2 temporal
   fast diagonalisation in the eigenbasis kernel; -1 on the coarsest level */
int stmg_multigrid_smoother_kind(const stmg_multigrid* mg, int level);
/* device bytes of the level-l smoother's per-cell data (eigenbases,
 * eigenvalues, metadata), streamed once per sweep; -1 on the coarsest level */
long long stmg_multigrid_smoother_bytes(const stmg_multigrid* mg, int level);
const stmg_st_operator* stmg_multigrid_operator_at(const stmg_multigrid* mg, int level);
/* apply (multigrid.cpp:228-234): one V-cycle, zero initial guess, overwrite d_z */
int stmg_multigrid_apply(const stmg_multigrid* mg, const double* d_r, double* d_z, void* stream);
int stmg_multigrid_apply_host(const stmg_multigrid* mg, const double* h_r, double* h_z);
/* smooth (multigrid.cpp:174-185): d_u += omega_l ASM_l(d_f - S_l d_u) */
int stmg_multigrid_smooth(const stmg_multigrid* mg, int level, const double* d_f, double* d_u, void* stream);
/* the level-l smoother and the level-l -> l+1 transfer of the hierarchy */
int stmg_multigrid_asm_add_correction(const stmg_multigrid* mg, int level, const double* d_r, double* d_z, void* stream);
int stmg_multigrid_prolong(const stmg_multigrid* mg, int level, const double* d_coarse, double* d_fine, void* stream);
int stmg_multigrid_restrict(const stmg_multigrid* mg, int level, const double* d_fine, double* d_coarse, void* stream);
long long stmg_multigrid_device_bytes(const stmg_multigrid* mg);

/* GmresOptions / GmresResult (include/stmg/gmres.hpp:12-25) */
typedef struct {
  int max_iters;
  int restart;
  double rel_tol;
  double abs_tol;
} stmg_gmres_options;
typedef struct {
  int converged;
  int iterations;
  double initial_residual;
  double final_residual;
  int history_len;
} stmg_gmres_result;
void stmg_gmres_options_default(stmg_gmres_options* o);

/* LinearMap (include/stmg/gmres.hpp:9-10) on device vectors: out = A in */
typedef int (*stmg_linear_map)(void* ctx, const double* d_in, double* d_out, void* stream);

/* gmres (gmres.cpp:8-115): restarted right-preconditioned GMRES on device
 * vectors; precond may be NULL (identity). history (may be NULL) receives up
 * to history_cap residual norms including the initial one. */
int stmg_gmres(long long n, stmg_linear_map op, void* op_ctx, stmg_linear_map precond, void* precond_ctx,
               const double* d_b, double* d_x, const stmg_gmres_options* options, stmg_gmres_result* result,
               double* history, int history_cap, void* stream);
/* The slab solve as march() plugs it (driver.cpp:193-203): op = the finest
 * SpaceTimeOperator of mg, precond = one V-cycle (precondition != 0). */
int stmg_solve(const stmg_multigrid* mg, int precondition, const double* d_b, double* d_x,
               const stmg_gmres_options* options, stmg_gmres_result* result, double* history, int history_cap,
               void* stream);
/* same with host buffers (b in, x in/out): copies inside */
int stmg_solve_host(const stmg_multigrid* mg, int precondition, const double* h_b, double* h_x,
                    const stmg_gmres_options* options, stmg_gmres_result* result, double* history, int history_cap);

/* error_norms (driver.cpp:83-92) of one batch solution d_x entering from
 * d_u0 against the manufactured solution of driver.cpp:265-293 (frequency):
 * out = {L2(L2), Linf(L2), Linf(Linf)} with the reference's temporal Gauss
 * (k+2) x spatial Gauss (p+2) sampling (driver.cpp:27-43) */
int stmg_st_operator_error_norms(const stmg_st_operator* op, const double* d_x, const double* d_u0, double frequency,
                                 double t0, double out[3]);
/* march (driver.cpp:95-260) with every slab on the device: n_batches slabs of
 * mg's finest operator, each assemble_rhs (source_kind 0 zero, 1 manufactured)
 * -> STMG-preconditioned GMRES -> extract_final. d_u (and d_v for the wave)
 * hold the entering state on input and the final state on output;
 * iterations[n_batches] receives the GMRES iterations (0 after a
 * non-converged batch); errors (may be NULL) the manufactured-solution error
 * norms of u over the run. Returns -2 if a batch did not converge. */
int stmg_march(const stmg_multigrid* mg, int n_batches, int source_kind, double frequency, double* d_u, double* d_v,
               const stmg_gmres_options* options, int* iterations, double errors[3], void* stream);

/* march with probes (driver.cpp:146-186, 226-236): n_probes points
 * (probe_xyz, 3 each, located on the finest mesh by locate_point,
 * spatial_operator.cpp:475-524) sampled samples_per_step times per step;
 * times receives 1 + n_batches * n_steps * samples_per_step sample times and
 * values the series of each probe (probe-major, same length) */
int stmg_march_probes(const stmg_multigrid* mg, int n_batches, int source_kind, double frequency, double* d_u,
                      double* d_v, const stmg_gmres_options* options, int* iterations, double errors[3], int n_probes,
                      const double* probe_xyz, int samples_per_step, double* times, double* values, void* stream);

/* ---- configured runs: the reference's ProblemSpec -> march(spec, probes)
 * -> RunReport (include/stmg/driver.hpp:14-91, src/driver.cpp:95-262), with
 * the mesh perturbation (src/mesh.cpp:190-240), coefficient fields
 * (src/mesh.cpp:254-298) and problem families (src/driver.cpp:265-320) it
 * builds on. The config front end (src/config.cpp) and the report writer
 * (tools/stmg.cpp) sit above this, in paper_2408_04372_b200/config.py,
 * report.py and cli.py. */
typedef struct {
  int equation, scheme;
  int problem; /* 0 manufactured, 1 shm, 2 zero */
  int k, p, dim;
  double lo[3], hi[3];
  double t_final;
  int refinements, base_cells, base_time_intervals, batch;
  double frequency, shm_s, perturb;
  unsigned long long seed;
  double rho_random_lo, rho_random_hi;
  double abs_tol, rel_tol;
  int max_iters, restart, n_smooth, precondition, probe_samples_per_step;
  int n_strategy; /* 0 = default ordering */
  int strategy[32];
  int timers; /* record the profile sections */
} stmg_problem;
typedef struct {
  int converged;
  long long n_space_dofs;
  int n_steps_total, n_batches;
  long long dofs_global;
  int n_batches_run; /* entries written to the batch arrays */
  double mean_iterations, work;
  int has_error_u, has_error_v;
  double error_u[3], error_v[3]; /* l2_l2, linf_l2, linf_linf */
  int n_levels;
  /* total, smoother, gmg_wo_smoother, operator_wo_gmg, other (seconds) */
  double sections[5];
  long long n_probe_samples; /* per probe, t = 0 included */
} stmg_run_report;
/* the step and batch counts of a problem (no device work): n_steps_total =
 * base_time_intervals * 2^(refinements+1), n_batches = n_steps_total / batch */
int stmg_problem_sizes(const stmg_problem* spec, int* n_steps_total, int* n_batches, long long* n_probe_samples);
/* one run. Batch arrays hold batch_cap entries, level arrays level_cap
 * (level_ints: coarsening 0..3 or -1 for the finest, mesh_level, p, k,
 * n_steps per level), probe arrays probe_cap samples per probe (probe-major).
 * Returns 0 also when a batch did not converge (report->converged == 0). */
int stmg_run(const stmg_problem* spec, int n_probes, const double* probe_xyz, stmg_run_report* report, int batch_cap,
             int* batch_iterations, double* batch_residuals, int* batch_converged, int level_cap, int* level_ints,
             long long* level_dofs, double* level_omega, long long probe_cap, double* probe_times,
             double* probe_values);
/* host-only: the level plan build_level_plan(finest, scheme, strategy)
 * (multigrid.cpp:34-81) of (fine_mesh_level, p, k, n_steps, tau);
 * n_strategy < 0 = default_strategy. ints: 5 per level as stmg_run. */
int stmg_level_plan(int scheme, int fine_mesh_level, int p, int k, int n_steps, double tau, int n_strategy,
                    const int* strategy, int cap, int* n_levels, int* ints, double* taus);
/* host-only: the finest-level vertices of make_cartesian + perturb
 * (src/mesh.cpp:148-240), 3 per vertex, x fastest */
int stmg_perturbed_vertices(int dim, const double lo[3], const double hi[3], int base_cells, int refinements,
                            double magnitude, unsigned long long seed, double* xyz);

/* ---- z-slab partitioned solve over several GPUs (no
 * reference counterpart: the reference is single-process). The finest mesh
 * is cut into n_parts slabs of cell layers along z; a process holds
 * local_parts consecutive slabs starting at first_part, and the processes
 * talk over NCCL (interface-plane exchanges and dot-product allreduces). One
 * process holding every part runs the same partitioned algorithm on one GPU.
 * Vectors of the partitioned finest level are the concatenation of the local
 * parts' slab vectors (each in the reference layout of its slab lattice,
 * interface planes included on both sides). */
typedef struct stmg_comm stmg_comm;
typedef struct stmg_slab_multigrid stmg_slab_multigrid;
/* NCCL unique id (128 bytes) for stmg_comm_create, on the root rank
 * (the NCCL communicator: NVLink / NVSwitch between the GPUs of one box) */
int stmg_nccl_unique_id(char id[128]);
int stmg_comm_create(int world, int rank, const char id[128], stmg_comm** out);
void stmg_comm_destroy(stmg_comm* c);
/* Host-staged transport (no reference counterpart): the partition's
 * interface exchanges and allreduces go through page-locked host buffers
 * and these callbacks (e.g. torch.distributed over gloo). allreduce_sum sums
 * n doubles in place over all ranks; sendrecv sends n doubles to rank peer
 * and receives n doubles from it. Both return 0 on success. */
typedef struct {
  void* ctx;
  int (*allreduce_sum)(void* ctx, double* h, long long n);
  int (*sendrecv)(void* ctx, int peer, const double* h_send, double* h_recv, long long n);
} stmg_host_transport;
int stmg_comm_create_host(int world, int rank, const stmg_host_transport* transport, stmg_comm** out);
/* host-only: how many levels of the default plan of (fine_mesh_level, p, k,
 * n_steps) stay partitioned for n_parts slabs of cells_z finest layers */
int stmg_slab_plan(int scheme, int fine_mesh_level, int p, int k, int n_steps, long long cells_z, int n_parts,
                   int* dist_levels, int* n_levels);
/* SpaceTimeMultigrid over the partition (options/strategy as
 * stmg_multigrid_create); comm may be NULL for a single process */
int stmg_slab_multigrid_create(int equation, int scheme, const stmg_mesh* mesh, const double* coarse_cell_scale,
                               int fine_mesh_level, int p, int k, int n_steps, double tau, int n_strategy,
                               const int* strategy, const stmg_mg_options* options, int n_parts, int first_part,
                               int local_parts, const stmg_comm* comm, stmg_slab_multigrid** out);
void stmg_slab_multigrid_destroy(stmg_slab_multigrid* mg);
long long stmg_slab_multigrid_local_dofs(const stmg_slab_multigrid* mg);
/* info[0] partitioned levels, info[1] total levels */
int stmg_slab_multigrid_info(const stmg_slab_multigrid* mg, int info[2]);
/* local part i: offset and length in the local vector, first global lattice plane */
int stmg_slab_multigrid_part(const stmg_slab_multigrid* mg, int i, long long* offset, long long* n_dofs,
                             long long* plane0);
double stmg_slab_multigrid_omega(const stmg_slab_multigrid* mg, int level);
int stmg_slab_multigrid_set_omega(stmg_slab_multigrid* mg, int level, double omega);
/* SpaceTimeOperator::apply on the partition (interface-summed), overwrite */
int stmg_slab_multigrid_apply(const stmg_slab_multigrid* mg, const double* d_u, double* d_y, void* stream);
/* one V-cycle, zero initial guess, overwrite */
int stmg_slab_multigrid_vcycle(const stmg_slab_multigrid* mg, const double* d_r, double* d_z, void* stream);
/* finest-level smoother, accumulate (ASMSmoother::add_correction) */
int stmg_slab_multigrid_asm_add_correction(const stmg_slab_multigrid* mg, const double* d_r, double* d_z,
                                           void* stream);
/* STMG-preconditioned GMRES on the partition */
int stmg_slab_multigrid_solve(const stmg_slab_multigrid* mg, const double* d_b, double* d_x,
                              const stmg_gmres_options* options, stmg_gmres_result* result, void* stream);
/* owned-entry inner product summed over the ranks */
int stmg_slab_multigrid_dot(const stmg_slab_multigrid* mg, const double* d_a, const double* d_b, double* out);
/* full-length finest vector <-> local parts (device); gather writes the
 * owned planes of the local parts only */
int stmg_slab_multigrid_scatter(const stmg_slab_multigrid* mg, const double* d_full, double* d_local, void* stream);
int stmg_slab_multigrid_gather(const stmg_slab_multigrid* mg, const double* d_local, double* d_full, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STMG_B200_H */
