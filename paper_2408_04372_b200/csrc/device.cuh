// Device-side level descriptor shared by the sm_100a kernels. One descriptor
// describes one multigrid level: the spatial Q_p lattice, its geometry
// (exact Cartesian lattice or d-linear cells from vertex coordinates), the
// coefficient, the 1D shape tables at the Gauss points, and the space-time
// block coefficients CM/CA of the batched slab system.
//
// HBM layout of every space-time vector (identical to the reference's,
// include/stmg/space_time_operator.hpp:23-29,43-45): index
// (s*n_t + i)*n_space + g with the spatial lattice index
// g = ix + dofs_x*(iy + dofs_y*iz), ix = cx*p + local (spatial_operator.cpp:70-114).
#pragma once

#include <cstdint>

namespace stmgb {

constexpr int kMaxN = 5;   // p <= 4
constexpr int kMaxF = 8;   // S * n_t <= 8 in the fused kernels
constexpr int kMaxWideF = 64;  // composed (wide-batch) application

struct DevLevel {
  int dim;
  int p;
  int n;           // p + 1 (= number of Gauss points per axis)
  int S, nt, F;    // steps, temporal unknowns per step, F = S*nt fields
  long long cells[3];
  long long dofs[3];  // per axis: cells*p + 1 (1 for unused axes)
  long long n_space;  // prod dofs
  long long n_dofs;   // F * n_space
  // geometry: verts == nullptr -> Cartesian lattice with spacing h
  const double* verts;  // (cells+1)^dim * 3 doubles, x fastest
  double h[3];
  double lo[3];             // domain origin (Cartesian node positions)
  // z-slab partition: the lattice is the slab's, its low / high z
  // faces are Dirichlet boundaries only if zbc bit 0 / bit 1 is set (an
  // interface plane shared with the neighbouring slab otherwise); cz0 is the
  // slab's first cell layer in the global mesh (coefficient lookup).
  // Unpartitioned: zbc = 3, cz0 = 0.
  int zbc;
  long long cz0;
  // coefficient: rho(cell) = rho0[ancestor on level 0] (1 if rho0 == nullptr)
  const double* rho0;
  int rho_shift;          // refinement levels between this level and level 0
  long long cells0[3];
  // rho is constant on every z layer of level-0 cells (or rho0 == nullptr):
  // the owner-computes Cartesian kernel (st_brick.cu) applies
  int rho_zonly;
  // 1D tables at the q = n Gauss points of [0,1]
  double B[kMaxN][kMaxN];   // B[q][j] = phi_j(x_q)      (spatial_operator.cpp:141-147)
  double Dq[kMaxN][kMaxN];  // collocation derivative at the Gauss points
  double D[kMaxN][kMaxN];   // D[q][j] = phi_j'(x_q), nodal derivative at the Gauss points (= Dq B)
  double w[kMaxN];          // Gauss weights
  double xq[kMaxN];         // Gauss points on [0,1]
  double gl[kMaxN];         // Gauss-Lobatto support nodes on [0,1]
  // 1D element matrices of [0,1] (Cartesian fast path, st_cart.cuh):
  // Mr = B^T W B, Kr = D^T W D; hinv2[a] = 1 / h[a]^2
  double Mr[kMaxN][kMaxN];
  double Kr[kMaxN][kMaxN];
  double hinv2[3];
  // even-odd halves of Mr / Kr (both centro-symmetric: A[i][j] =
  // A[n-1-i][n-1-j]): E[i][k] = (A[i][k] + A[i][n-1-k]) / 2 (k < n/2),
  // E[i][n/2] = A[i][n/2] (odd n); O[i][k] = (A[i][k] - A[i][n-1-k]) / 2
  double MrE[3][3], MrO[2][2], KrE[3][3], KrO[2][2];
  // space-time block coefficients, row-major F x F (space_time_operator.cpp:269-317)
  double CM[kMaxF * kMaxF];
  double CA[kMaxF * kMaxF];
  // G = CA^-1 CM (row-major F x F), g_ok = 1 when CA is safely invertible:
  // S = (CA (x) I)(G (x) M + I (x) A), the form st_brick.cu applies (the
  // temporal coupling of the z stage becomes one F x F product per point,
  // CA is applied once per output plane)
  double G[kMaxF * kMaxF];
  int g_ok;
};

}  // namespace stmgb
