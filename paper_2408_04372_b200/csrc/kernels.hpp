// Launch entry points of the sm_100a kernels (host-callable).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "device.cuh"

namespace stmgb {

// y = S u (overwrite), fused space-time operator -- st_operator.cu
void st_apply(const DevLevel& L, const double* u, double* y, cudaStream_t stream);
// owner-computes Cartesian form (st_brick.cu): y = S u (f == nullptr) or
// y = f - S u, Dirichlet rows included, every dof written once
bool st_brick_supported(const DevLevel& L);
void st_brick(const DevLevel& L, const double* f, const double* u, double* y, cudaStream_t stream);
// Dirichlet entries of every field of v set to zero
void st_zero_boundary(const DevLevel& L, double* v, cudaStream_t stream);
// r = f - S u (overwrite), fused residual (no separate subtraction pass)
void st_residual(const DevLevel& L, const double* f, const double* u, double* r, cudaStream_t stream);
// S * n_t > kMaxF: 2F single-field applications of the constrained mass and
// stiffness (descriptors mass / stiff) into mu / au (F * n_space each), then
// the temporal combination with the full F x F CM / CA (device, row-major);
// f != nullptr gives the residual f - S u
void st_apply_wide(const DevLevel& L, const DevLevel& mass, const DevLevel& stiff, const double* cm, const double* ca,
                   const double* f, const double* u, double* y, double* mu, double* au, cudaStream_t stream);

// nodal interpolant at the Q_p support points (rhs.cu); kind: 0 heat source,
// 1 wave source, 2 Gaussian(centre, width), 3 manufactured u, 4 manufactured v
void interpolate_nodes(const DevLevel& L, int kind, double omega, double t, const double* centre, double width,
                       bool zero_boundary, double* out, cudaStream_t s);

// error sample against the manufactured solution (rhs.cu; kind 3 u, 4 v) at
// the n_q^d Gauss points (qx, qw on [0,1], n_q <= 8) of every cell:
// out[0] += sum w |J| (u_h - u)^2, out[1] = max(out[1], max |u_h - u|)
void spatial_error(const DevLevel& L, const double* u, int n_q, const double* qx, const double* qw, int kind,
                   double omega, double t, double* out, cudaStream_t s);

// evaluate_fe at located points (rhs.cu): out[p * n_fields + f] for n_fields
// nodal fields u + f * fstride; cells / xi (3 per point) on the device
void probe_fields(const DevLevel& L, const double* u, int n_fields, long long fstride, int n_probes,
                  const long long* d_cells, const double* d_xi, double* d_out, cudaStream_t s);

// ---- z-slab partition helpers (slab.cu)
// v[f * fstride + plane * plane_len + i] = val for every field f < F, i < plane_len
void plane_fill(double* v, int F, long long fstride, long long plane, long long plane_len, double val, cudaStream_t s);
// interface sum of two slabs held by this process: a_plane = b_plane = a_plane + b_plane
void plane_pair_sum(double* a, long long a_plane, double* b, long long b_plane, int F, long long a_fstride,
                    long long b_fstride, long long plane_len, cudaStream_t s);
// buf[f][i] = v[f * fstride + plane * plane_len + i]
void plane_pack(const double* v, int F, long long fstride, long long plane, long long plane_len, double* buf,
                cudaStream_t s);
// v[f * fstride + plane * plane_len + i] += buf[f][i]
void plane_unpack_add(double* v, int F, long long fstride, long long plane, long long plane_len, const double* buf,
                      cudaStream_t s);
// owned-entry segments of a distributed vector (GMRES dots)
constexpr int kMaxSeg = 64;
struct DotSegments {
  int n;
  long long begin[kMaxSeg], end[kMaxSeg];
};
// out[i] = sum over the segments of V_i . w (i < k); scratch as vec_multidot
void vec_multidot_seg(const double* const* V, int k, const double* w, const DotSegments& seg, double* out,
                      double* scratch, cudaStream_t s);

// ---- vector kernels (vector_ops.cu)
void vec_copy(double* y, const double* x, long long n, cudaStream_t s);
void vec_axpy(double* y, double a, const double* x, long long n, cudaStream_t s);         // y += a x
void vec_axpby(double* y, double a, const double* x, double b, long long n, cudaStream_t s);  // y = a x + b y
void vec_scale_into(double* y, double a, const double* x, long long n, cudaStream_t s);   // y = a x
void vec_sub_into(double* r, const double* f, const double* y, long long n, cudaStream_t s);  // r = f - y
// out[i] = <V_i, w>, i < k; V = device array of k vector pointers; out is a
// device buffer of k doubles; scratch holds kDotBlocks * k doubles
void vec_multidot(const double* const* V, int k, const double* w, long long n, double* out, double* scratch,
                  cudaStream_t s);
// w += sign * sum_i h_i V_i (h on device)
void vec_multi_axpy(double* w, const double* const* V, int k, const double* h, double sign, long long n,
                    cudaStream_t s);
constexpr int kDotBlocks = 592;
void vec_fill(double* y, double v, long long n, cudaStream_t s);
void vec_set_element(double* y, long long i, double v, cudaStream_t s);
// y[g] = 1 where every lattice coordinate of g is congruent to colour (mod period)
void vec_colour_indicator(double* y, const long long* dofs, int dim, int period, int cx, int cy, int cz,
                          long long z_offset, cudaStream_t s);  // z_offset: global lattice z of plane 0
// dense matvec y = A x, A row-major n x n (coarse-grid inverse)
void dense_matvec(const double* A, const double* x, double* y, int n, cudaStream_t s);

// ---- grid transfers (transfer.cu)
struct DevAxisTransfer {
  // CSR of the 1D embedding P (rows = fine index, transfer.cpp:32-54) and of
  // P^T (rows = coarse index)
  const int* row_ptr;
  const int* row_idx;
  const double* row_w;
  const int* col_ptr;
  const int* col_idx;
  const double* col_w;
  long long nf, nc;
  // pure h-coarsening with equal p (hp = p > 0): P[2p c + r][c p + j] =
  // hw[r][j], r = 0..2p, the coarse basis at the fine nodes of one coarse
  // cell -- applied without the CSR arrays
  int hp;
  double hw[9][kMaxN];
};
// slab options of a transfer: physical z faces, skip the input's low z plane
// (an interface owned by the slab below), accumulate into the output, and the
// coarse side's field stride (0 = compact; > 0: coarse data inside a longer
// vector, e.g. the full coarse level under a slab)
struct TransferSlab {
  int zbc = 3;
  bool skip_lo_in = false;
  bool accumulate = false;
  long long coarse_fstride = 0;
};
// separable per-axis passes; t1/t2 are work buffers of Transfer-chosen size
void spatial_prolong(const DevAxisTransfer* ax, int dim, int F, const long long* dofs_c, const long long* dofs_f,
                     const double* coarse, double* fine, double* t1, double* t2, const TransferSlab& sl,
                     cudaStream_t s);
void spatial_restrict(const DevAxisTransfer* ax, int dim, int F, const long long* dofs_c, const long long* dofs_f,
                      const double* fine, double* coarse, double* t1, double* t2, const TransferSlab& sl,
                      cudaStream_t s);
// temporal: fine block r = sum_c T[r][c] coarse block c (T row-major Ff x Fc)
void temporal_prolong(const double* T_dev, int Ff, int Fc, long long n_space, const long long* dofs, int dim,
                      const double* coarse, double* fine, const TransferSlab& sl, cudaStream_t s);
void temporal_restrict(const double* T_dev, int Ff, int Fc, long long n_space, const long long* dofs, int dim,
                       const double* fine, double* coarse, const TransferSlab& sl, cudaStream_t s);

// ---- additive Schwarz (asm_smoother.cu)
struct DevASM {
  int dim, p, n, m;       // m = n^dim local dofs per cell
  int S, nt;
  long long cells[3], dofs[3], n_space;
  const double* X;        // per cell m x m (row-major [a][e]), M_T-orthonormal eigenvectors,
                          // cell stride xs = m*m rounded up to even (16-byte TMA alignment)
  long long xs;
  const double* lam;      // per cell m eigenvalues (0 on Dirichlet dofs)
  double TM[16], TA[16];  // diagonal (s,s) temporal blocks, n_t x n_t
  const long long* list;  // cells handled (X/lam stored per list entry); nullptr = all cells
  long long n_list;       // number of handled cells
  // z-slab partition (as DevLevel::zbc / cz0)
  int zbc;
  long long cz0;
  // m = 64 records: X (swizzled, 4096 doubles) followed by the 64 eigenvalues,
  // xs = kRec64; meta[pos] = {lattice offset of local dof 0, Dirichlet face
  // mask (bit 2a: low face of axis a, 2a+1: high face)}
  const long long* meta;
  // temporal fast diagonalisation (T_M + lam T_A)^-1 = Q (B + lam)^-1 P of the
  // n_t x n_t solves, expanded over the S steps into 8 MMA columns ("slots"):
  // slot k <- sum_c P[k][c] col c; col c <- sum_k Q[c][k] slot k; slot pair
  // (2j, 2j+1) is two real eigenvalues s0/s1 (kind 0) or one conjugate pair
  // s0 +- i s1 (kind 1)
  int tdiag;
  // record layout: 0 contiguous rows (m = 64: swizzled for the FP64 tensor
  // cores), 2 pitch-28 rows (25 / 27 dofs); see asm_record_stride
  int x_layout;
  int kind[4];
  double s0[4], s1[4];
  double P[8][8], Q[8][8];
};
constexpr int kRec64 = 64 * 64 + 64;
constexpr int kMma32Pitch = 28;  // row pitch of the 25 / 27-dof records (layout 2)
// doubles per cell record of the exact smoother, by block size and layout;
// the single definition setup (stmg.cpp) and the kernels (asm_smoother.cu) use
inline long long asm_record_stride(int m, int layout) {
  if (m == 64) return kRec64;
  if (layout == 2) return static_cast<long long>(m) * kMma32Pitch;
  return (static_cast<long long>(m) * m + 1) & ~1LL;
}
// z += scale * W sum_T R_T^T B_T^-1 R_T r
void asm_add_correction(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s);

// tensor-product FDM cell solves on Cartesian levels (asm_fdm.cu)
struct DevFDM {
  int dim, p, n, S, nt;
  long long cells[3], dofs[3], n_space;
  double S1[3][4][kMaxN][kMaxN];  // per axis and position class: 1D eigenvectors [node][eig]
  double L1[3][4][kMaxN];         // matching eigenvalues
  double TM[16], TA[16];
  const double* rho0;             // coefficient per level-0 cell (nullptr: 1)
  int rho_shift;
  long long cells0[3];
  const unsigned char* skip;      // per cell: 1 = solved by the exact per-cell kernel
  int zbc;                        // z-slab partition (as DevLevel::zbc / cz0)
  long long cz0;
  // temporal fast diagonalisation of the n_t x n_t solves (tdiag = 1):
  // (T_M + mu T_A)^-1 = Q (B + mu)^-1 P, row-major n_t x n_t tP / tQ; B is
  // block diagonal: tkind[i] = 0 real eigenvalue ta[i]; 1 first column of a
  // conjugate pair [[ta, tb], [-tb, ta]] (2 its second column)
  int tdiag;
  // interior position class (S1[a][0]) ordered symmetric-then-antisymmetric
  // eigenvectors on every axis: the even-odd transforms apply
  int eo;
  int tkind[4];
  double ta[4], tb[4];
  double tP[16], tQ[16];
  // eo = 1, 3D: the cells the strip kernel leaves to the line-owner kernel
  // (boundary strips, strips holding a skipped cell), from fdm_left_out_cells
  const long long* left;
  long long n_left;
};
// fields a strip-kernel CTA works on: n_t times the largest of 1, 2, 4 that
// divides S and keeps the product <= 4 (consecutive steps are independent
// smoother blocks)
inline int fdm_fields_per_cta(int nt, int S) {
  int sg = 1;
  for (int d = 2; d <= 4 && nt * d <= 4; d *= 2)
    if (S % d == 0) sg = d;
  return nt * sg;
}
// host: the left-out cell list of F (skip_host: host copy of F.skip or nullptr)
std::vector<long long> fdm_left_out_cells(const DevFDM& F, const unsigned char* skip_host);
void fdm_add_correction(const DevFDM& F, const double* r, double* z, double scale, cudaStream_t s);
// probing-based extraction of restricted cell matrices (setup)
// colours are classes of GLOBAL lattice coordinates; the probe lattice may
// carry probe_zcells extra cell layers below the slab (halo for the setup)
void asm_extract_probe(const DevASM& A, int colour_x, int colour_y, int colour_z, int period, const double* probe,
                       int probe_zcells, double* cellmat, cudaStream_t s);
void asm_reduce_standard(const DevASM& A, double* Mt, double* At, cudaStream_t s);  // At <- L^-1 At L^-T, Mt <- L^-1
void asm_back_transform(int m, long long xs, int layout, long long n_cells, const double* Linv, const double* V,
                        double* X, cudaStream_t s);
// large blocks (m > 64): Dirichlet rows/cols of the cell matrices (M identity,
// A zero) and column-major -> row-major X records
void asm_dirichlet_rows(const DevASM& A, double* Mt, double* At, cudaStream_t s);
void asm_transpose_cells(int m, long long n_cells, long long xs, const double* colmajor, double* X, cudaStream_t s);

}  // namespace stmgb

namespace stmgb {
// number of kernels launched by this library since load (the bench's
// gpu_launches evidence); incremented at every launch site
void count_launch(long long n = 1);
long long kernel_launches();
}  // namespace stmgb
