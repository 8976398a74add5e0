// Cell-wise space-time additive Schwarz smoother (reference: ASMSmoother,
// asm_smoother.cpp:7-78). The reference extracts, per (step, cell) block T,
// the restriction B_T = R_T S R_T^T of the assembled slab matrix and LU-solves
// it. Every such block has the Kronecker form
//     B_T = T_M (x) M_T + T_A (x) A_T           (interior dofs; identity on
//                                                 Dirichlet dofs)
// with the n_t x n_t diagonal temporal blocks T_M, T_A of the slab operator
// (space_time_operator.cpp:269-317) and the restricted GLOBAL spatial mass and
// stiffness matrices M_T, A_T. With the generalised eigen-decomposition
// A_T X = M_T X Lambda, X^T M_T X = I (fast diagonalisation of the block),
//     B_T^-1 = (I (x) X) (T_M (x) I + T_A (x) Lambda)^-1 (I (x) X^T),
// i.e. two m x m products per temporal field and one n_t x n_t solve per
// eigenvalue -- exact (to rounding) for every cell, including perturbed
// cells and heterogeneous coefficients, where a 1D tensor-product
// diagonalisation would only approximate B_T. X is stored per cell (m^2
// doubles), shared by all S steps of the slab.
//
// Setup (restricted matrices by probing the matrix-free operator, Cholesky
// reduction to standard form, batched symmetric eigensolver, back transform)
// lives here too; the eigensolver itself is cuSOLVER's batched syev.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.hpp"

namespace stmgb {

namespace {

__device__ __forceinline__ void cell_coords(long long cell, const long long* cells, long long& cx, long long& cy,
                                            long long& cz) {
  cx = cell % cells[0];
  cy = (cell / cells[0]) % cells[1];
  cz = cell / (cells[0] * cells[1]);
}

// local dof l of a cell -> global lattice index, boundary flag, multiplicity
struct LocalDof {
  long long g;
  bool bdry;
  double mult;
};
__device__ __forceinline__ LocalDof local_dof(const DevASM& A, long long cx, long long cy, long long cz, int l) {
  const int n = A.n;
  const int lx = l % n, ly = (l / n) % n, lz = A.dim == 3 ? l / (n * n) : 0;
  const long long gx = cx * A.p + lx, gy = cy * A.p + ly, gz = cz * A.p + lz;
  LocalDof d;
  d.g = (gz * A.dofs[1] + gy) * A.dofs[0] + gx;
  d.bdry = gx == 0 || gx == A.dofs[0] - 1 || (A.dim > 1 && (gy == 0 || gy == A.dofs[1] - 1)) ||
           (A.dim > 2 && (gz == 0 || gz == A.dofs[2] - 1));
  // number of cells containing the dof (asm_smoother.cpp:45-49)
  double m = 1.0;
  if (gx % A.p == 0 && gx > 0 && gx < A.dofs[0] - 1) m *= 2.0;
  if (A.dim > 1 && gy % A.p == 0 && gy > 0 && gy < A.dofs[1] - 1) m *= 2.0;
  if (A.dim > 2 && gz % A.p == 0 && gz > 0 && gz < A.dofs[2] - 1) m *= 2.0;
  d.mult = m;
  return d;
}

// solve (TM + lam TA) x = b for n_t <= 4, partial pivoting, in registers
__device__ __forceinline__ void small_solve(const double* TM, const double* TA, double lam, int nt, double* b) {
  double a[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) a[i][j] = (i < nt && j < nt) ? fma(lam, TA[i * nt + j], TM[i * nt + j]) : 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= nt) break;
    int piv = k;
#pragma unroll
    for (int i = k + 1; i < 4; ++i)
      if (i < nt && fabs(a[i][k]) > fabs(a[piv][k])) piv = i;
    if (piv != k) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double t = a[k][j];
        a[k][j] = a[piv][j];
        a[piv][j] = t;
      }
      const double t = b[k];
      b[k] = b[piv];
      b[piv] = t;
    }
    const double inv = 1.0 / a[k][k];
#pragma unroll
    for (int i = k + 1; i < 4; ++i) {
      if (i >= nt) break;
      const double f = a[i][k] * inv;
#pragma unroll
      for (int j = k; j < 4; ++j) a[i][j] = fma(-f, a[k][j], a[i][j]);
      b[i] = fma(-f, b[k], b[i]);
    }
  }
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    if (i >= nt) continue;
    double s = b[i];
#pragma unroll
    for (int j = i + 1; j < 4; ++j)
      if (j < nt) s = fma(-a[i][j], b[j], s);
    b[i] = s / a[i][i];
  }
}

// one CTA per cell; blockDim >= m; handles all S steps of the slab
__global__ void asm_apply_kernel(const __grid_constant__ DevASM A, const double* __restrict__ r, double* __restrict__ z) {
  extern __shared__ double sm[];
  const int m = A.m, ld = m + 1, nt = A.nt;
  double* Xs = sm;               // [m][m+1]
  double* rs = Xs + m * ld;      // [nt][m]
  double* hs = rs + nt * m;      // [nt][m]
  const long long cell = blockIdx.x;
  const double* Xg = A.X + cell * static_cast<long long>(m) * m;
  for (int i = threadIdx.x; i < m * m; i += blockDim.x) Xs[(i / m) * ld + (i % m)] = Xg[i];
  long long cx, cy, cz;
  cell_coords(cell, A.cells, cx, cy, cz);
  const int t = threadIdx.x;
  LocalDof d{};
  double lam = 0.0;
  if (t < m) {
    d = local_dof(A, cx, cy, cz, t);
    lam = A.lam[cell * m + t];
  }
  for (int s = 0; s < A.S; ++s) {
    __syncthreads();
    if (t < m)
      for (int i = 0; i < nt; ++i) rs[i * m + t] = r[(static_cast<long long>(s) * nt + i) * A.n_space + d.g];
    __syncthreads();
    // hat r[.,e] = X^T r, thread e
    if (t < m) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int a = 0; a < m; ++a) {
        const double x = Xs[a * ld + t];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < nt) acc[i] = fma(x, rs[i * m + a], acc[i]);
      }
      small_solve(A.TM, A.TA, lam, nt, acc);
      for (int i = 0; i < nt; ++i) hs[i * m + t] = acc[i];
    }
    __syncthreads();
    // z_loc[., a] = X hat z, thread a; boundary rows are identity
    if (t < m) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int e = 0; e < m; ++e) {
        const double x = Xs[t * ld + e];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < nt) acc[i] = fma(x, hs[i * m + e], acc[i]);
      }
      const double w = 1.0 / d.mult;
      for (int i = 0; i < nt; ++i) {
        const double v = d.bdry ? rs[i * m + t] : acc[i];
        atomicAdd(z + (static_cast<long long>(s) * nt + i) * A.n_space + d.g, v * w);
      }
    }
  }
}

// column b of every cell matrix from one probe of colour (cx,cy,cz) mod period
__global__ void extract_probe_kernel(const __grid_constant__ DevASM A, int colx, int coly, int colz, int period,
                                     const double* __restrict__ probe, double* __restrict__ cellmat) {
  const long long n_cells = A.cells[0] * A.cells[1] * A.cells[2];
  const int m = A.m, n = A.n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_cells * m;
       t += (long long)gridDim.x * blockDim.x) {
    const long long cell = t / m;
    const int a = static_cast<int>(t - cell * m);
    long long cx, cy, cz;
    cell_coords(cell, A.cells, cx, cy, cz);
    // local index per axis whose lattice coordinate has the probe colour
    int lb[3] = {0, 0, 0};
    bool found = true;
    const long long c3[3] = {cx, cy, cz};
    const int col[3] = {colx, coly, colz};
    for (int ax = 0; ax < A.dim; ++ax) {
      int hit = -1;
      for (int l = 0; l < n; ++l)
        if ((c3[ax] * A.p + l) % period == col[ax]) hit = l;
      if (hit < 0) found = false;
      lb[ax] = hit;
    }
    if (!found) continue;
    const int b = lb[0] + n * (lb[1] + (A.dim == 3 ? n * lb[2] : 0));
    const LocalDof da = local_dof(A, cx, cy, cz, a);
    cellmat[cell * static_cast<long long>(m) * m + static_cast<long long>(a) * m + b] = probe[da.g];
  }
}

// per cell: M = L L^T (Dirichlet dofs: M=1, A=0 decoupled); At <- L^-1 A L^-T,
// Mt <- L^-1. One CTA per cell, blockDim >= m.
__global__ void reduce_standard_kernel(const __grid_constant__ DevASM A, double* __restrict__ Mt,
                                       double* __restrict__ At) {
  extern __shared__ double sm[];
  const int m = A.m, ld = m + 1;
  double* L = sm;            // [m][ld]
  double* As = L + m * ld;   // [m][ld]
  double* T = As + m * ld;   // [m][ld]
  const long long cell = blockIdx.x;
  double* Mg = Mt + cell * static_cast<long long>(m) * m;
  double* Ag = At + cell * static_cast<long long>(m) * m;
  long long cx, cy, cz;
  cell_coords(cell, A.cells, cx, cy, cz);
  for (int i = threadIdx.x; i < m * m; i += blockDim.x) {
    const int r = i / m, c = i % m;
    L[r * ld + c] = Mg[i];
    As[r * ld + c] = Ag[i];
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < m) {
    const LocalDof d = local_dof(A, cx, cy, cz, t);
    if (d.bdry) {
      for (int j = 0; j < m; ++j) {
        L[t * ld + j] = (j == t) ? 1.0 : 0.0;
        As[t * ld + j] = 0.0;
      }
    }
  }
  __syncthreads();
  if (t < m) {
    const LocalDof d = local_dof(A, cx, cy, cz, t);
    if (d.bdry)
      for (int j = 0; j < m; ++j) {
        L[j * ld + t] = (j == t) ? 1.0 : 0.0;
        As[j * ld + t] = 0.0;
      }
  }
  __syncthreads();
  // right-looking Cholesky, lower triangle
  for (int k = 0; k < m; ++k) {
    if (t == 0) L[k * ld + k] = sqrt(L[k * ld + k]);
    __syncthreads();
    if (t > k && t < m) L[t * ld + k] /= L[k * ld + k];
    __syncthreads();
    if (t > k && t < m) {
      const double lik = L[t * ld + k];
      for (int j = k + 1; j <= t; ++j) L[t * ld + j] = fma(-lik, L[j * ld + k], L[t * ld + j]);
    }
    __syncthreads();
  }
  // T = L^-1 (column t by forward substitution), stored in T
  if (t < m) {
    for (int i = 0; i < m; ++i) {
      double s = (i == t) ? 1.0 : 0.0;
      if (i < t) {
        T[i * ld + t] = 0.0;
        continue;
      }
      for (int k = t; k < i; ++k) s = fma(-L[i * ld + k], T[k * ld + t], s);
      T[i * ld + t] = s / L[i * ld + i];
    }
  }
  __syncthreads();
  // L <- T A (row t), then At = (T A) T^T (row t)
  if (t < m) {
    for (int j = 0; j < m; ++j) {
      double s = 0.0;
      for (int k = 0; k <= t; ++k) s = fma(T[t * ld + k], As[k * ld + j], s);
      L[t * ld + j] = s;
    }
  }
  __syncthreads();
  if (t < m) {
    for (int j = 0; j < m; ++j) {
      double s = 0.0;
      for (int k = 0; k <= j; ++k) s = fma(L[t * ld + k], T[j * ld + k], s);
      Ag[static_cast<long long>(t) * m + j] = s;
    }
    for (int j = 0; j < m; ++j) Mg[static_cast<long long>(t) * m + j] = T[t * ld + j];
  }
}

// X[a][e] = sum_k Linv[k][a] V[k][e]; V column-major from syev (V[e*m+k])
__global__ void back_transform_kernel(int m, const double* __restrict__ Linv, const double* __restrict__ V,
                                      double* __restrict__ X) {
  const long long cell = blockIdx.x;
  const double* Lc = Linv + cell * static_cast<long long>(m) * m;
  const double* Vc = V + cell * static_cast<long long>(m) * m;
  double* Xc = X + cell * static_cast<long long>(m) * m;
  for (int i = threadIdx.x; i < m * m; i += blockDim.x) {
    const int a = i / m, e = i % m;
    double s = 0.0;
    for (int k = a; k < m; ++k) s = fma(Lc[static_cast<long long>(k) * m + a], Vc[static_cast<long long>(e) * m + k], s);
    Xc[i] = s;
  }
}

}  // namespace

void asm_add_correction(const DevASM& A, const double* r, double* z, cudaStream_t s) {
  const long long n_cells = A.cells[0] * A.cells[1] * A.cells[2];
  const int threads = ((A.m + 31) / 32) * 32;
  const size_t smem = sizeof(double) * (static_cast<size_t>(A.m) * (A.m + 1) + 2 * A.nt * A.m);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(asm_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  count_launch();
  asm_apply_kernel<<<static_cast<unsigned>(n_cells), threads, smem, s>>>(A, r, z);
}

void asm_extract_probe(const DevASM& A, int cx, int cy, int cz, int period, const double* probe, double* cellmat,
                       cudaStream_t s) {
  const long long total = A.cells[0] * A.cells[1] * A.cells[2] * A.m;
  const unsigned grid = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 148LL * 64)));
  count_launch();
  extract_probe_kernel<<<grid, 256, 0, s>>>(A, cx, cy, cz, period, probe, cellmat);
}

void asm_reduce_standard(const DevASM& A, double* Mt, double* At, cudaStream_t s) {
  const long long n_cells = A.cells[0] * A.cells[1] * A.cells[2];
  const int threads = ((A.m + 31) / 32) * 32;
  const size_t smem = sizeof(double) * 3 * static_cast<size_t>(A.m) * (A.m + 1);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(reduce_standard_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  count_launch();
  reduce_standard_kernel<<<static_cast<unsigned>(n_cells), threads, smem, s>>>(A, Mt, At);
}

void asm_back_transform(int m, long long n_cells, const double* Linv, const double* V, double* X, cudaStream_t s) {
  count_launch();
  back_transform_kernel<<<static_cast<unsigned>(n_cells), 128, 0, s>>>(m, Linv, V, X);
}

}  // namespace stmgb
