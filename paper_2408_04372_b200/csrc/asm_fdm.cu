// Tensor-product fast-diagonalisation (FDM) cell solves for the space-time
// additive Schwarz smoother on Cartesian levels (reference: ASMSmoother,
// asm_smoother.cpp:7-78, which LU-factors every (step, cell) block).
//
// On a Cartesian cell whose neighbourhood has one coefficient value rho, the
// restricted global matrices are Kronecker products of restricted 1D
// matrices, M_T = M_z (x) M_y (x) M_x and
// A_T = rho (K_z(x)M_y(x)M_x + M_z(x)K_y(x)M_x + M_z(x)M_y(x)K_x), so with the
// 1D generalised eigenpairs K_a S_a = M_a S_a Lambda_a (S_a^T M_a S_a = I),
//   B_T^-1 = (I(x)S)(T_M(x)I + T_A(x)rho(Lz(+)Ly(+)Lx))^-1 (I(x)S^T),
//   S = S_z (x) S_y (x) S_x,
// i.e. d sum-factorised sweeps each way and one n_t x n_t solve per
// eigen-index; no per-cell data is stored. The 1D tables depend only on the
// cell's position class along each axis (interior / first / last / single,
// Dirichlet nodes removed). Cells flagged in `skip` are solved exactly by the
// per-cell eigenbasis kernel instead (asm_smoother.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <stdexcept>

#include "kernels.hpp"
#include "st_cart_layout.h"

namespace stmgb {

namespace {

constexpr int kT = 256;

template <int DIM, int N>
struct FCfg {
  static constexpr int ND = DIM == 2 ? N * N : N * N * N;
  static constexpr int LINES = DIM == 2 ? N : N * N;
  static constexpr int NC = (kT / ND) > 0 ? (kT / ND) : 1;
};

__device__ __forceinline__ void solve_small(const double* TM, const double* TA, double lam, int nt, double* b) {
  double a[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) a[i][j] = (i < nt && j < nt) ? fma(lam, TA[i * nt + j], TM[i * nt + j]) : (i == j);
  // Gaussian elimination with partial pivoting, fully unrolled (no local memory)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int i = k + 1; i < 4; ++i) {
      if (fabs(a[i][k]) > fabs(a[k][k])) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double t = a[k][j];
          a[k][j] = a[i][j];
          a[i][j] = t;
        }
        const double t = b[k];
        b[k] = b[i];
        b[i] = t;
      }
    }
    const double inv = 1.0 / a[k][k];
#pragma unroll
    for (int i = k + 1; i < 4; ++i) {
      const double f = a[i][k] * inv;
#pragma unroll
      for (int j = k; j < 4; ++j) a[i][j] = fma(-f, a[k][j], a[i][j]);
      b[i] = fma(-f, b[k], b[i]);
    }
  }
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    double s = b[i];
#pragma unroll
    for (int j = i + 1; j < 4; ++j) s = fma(-a[i][j], b[j], s);
    b[i] = s / a[i][i];
  }
}

// (T_M + mu T_A)^-1 b for every eigen-index: pivoted elimination, or, when
// the host block-diagonalised T_A^-1 T_M = Q B Q^-1 (P.tdiag),
// Q (B + mu)^-1 P b with P = Q^-1 T_A^-1 -- two n_t x n_t products and one
// reciprocal per 1x1 / 2x2 block, no pivoting
template <int NT, bool TD>
__device__ __forceinline__ void temporal_solve(const DevFDM& P, double mu, double (&b)[4]) {
  if constexpr (!TD) {
    solve_small(P.TM, P.TA, mu, NT, b);
    return;
  }
  double w[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NT; ++j) s = fma(P.tP[i * NT + j], b[j], s);
    w[i] = s;
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    if (P.tkind[i] == 0) {
      w[i] = w[i] / (P.ta[i] + mu);
    } else if (P.tkind[i] == 1 && i + 1 < NT) {
      const double al = P.ta[i] + mu, be = P.tb[i];
      const double inv = 1.0 / fma(al, al, be * be);
      const double w0 = w[i], w1 = w[i + 1];
      w[i] = (al * w0 - be * w1) * inv;
      w[i + 1] = (be * w0 + al * w1) * inv;
    }
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NT; ++j) s = fma(P.tQ[i * NT + j], w[j], s);
    b[i] = s;
  }
}

template <int N, bool TRANS>
__device__ __forceinline__ void sweep(double* arr, int base, int stride, const double (&S)[kMaxN][kMaxN]) {
  double in[N];
#pragma unroll
  for (int k = 0; k < N; ++k) in[k] = arr[base + k * stride];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(TRANS ? S[k][i] : S[i][k], in[k], s);
    arr[base + i * stride] = s;
  }
}

template <int N, int A>
__device__ __forceinline__ int lbase(int line) {
  constexpr int st = A == 0 ? 1 : (A == 1 ? N : N * N);
  return (line % st) + (line / st) * st * N;
}

template <int DIM, int N, int NT>
__global__ void __launch_bounds__(kT) asm_fdm_kernel(const __grid_constant__ DevFDM P, const double* __restrict__ r,
                                                      double* __restrict__ z, double scale) {
  using C = FCfg<DIM, N>;
  constexpr int ND = C::ND, LINES = C::LINES, NC = C::NC;
  extern __shared__ __align__(16) double sm[];
  double* W = sm;                    // [NC][NT][ND] working
  double* R = W + NC * NT * ND;      // [NC][NT][ND] residual (Dirichlet rows)
  double* rho_s = R + NC * NT * ND;  // [NC]
  long long* base_s = reinterpret_cast<long long*>(rho_s + NC);
  int* info_s = reinterpret_cast<int*>(base_s + NC);  // mask | type_x<<8 | type_y<<10 | type_z<<12
  const long long n_cells = P.cells[0] * P.cells[1] * P.cells[2];
  const long long cell0 = static_cast<long long>(blockIdx.x) * NC;
  const int tid = threadIdx.x;
  const long long dx = P.dofs[0], dxy = P.dofs[0] * P.dofs[1];
  const int p = N - 1;
  if (tid < NC) {
    const long long cell = cell0 + tid;
    long long base = -1;
    int info = 0;
    if (cell < n_cells && !(P.skip && P.skip[cell])) {
      const unsigned ci = static_cast<unsigned>(cell);
      const unsigned nx = static_cast<unsigned>(P.cells[0]), ny = static_cast<unsigned>(P.cells[1]),
                     nz = static_cast<unsigned>(P.cells[2]);
      const unsigned cx = ci % nx, cy = (ci / nx) % ny, cz = ci / (nx * ny);
      base = static_cast<long long>(cz) * p * dxy + static_cast<long long>(cy) * p * dx + static_cast<long long>(cx) * p;
      const int tx = (cx == 0 ? 1 : 0) | (cx == nx - 1 ? 2 : 0);
      const int ty = (cy == 0 ? 1 : 0) | (cy == ny - 1 ? 2 : 0);
      const int tz = DIM == 3 ? ((cz == 0 && (P.zbc & 1) ? 1 : 0) | (cz == nz - 1 && (P.zbc & 2) ? 2 : 0)) : 0;
      info = tx | (ty << 2) | (tz << 4) | (tx << 8) | (ty << 10) | (tz << 12);
      double rho = 1.0;
      if (P.rho0) {
        const long long ax = cx >> P.rho_shift, ay = cy >> P.rho_shift, az = (cz + P.cz0) >> P.rho_shift;
        rho = P.rho0[(az * P.cells0[1] + ay) * P.cells0[0] + ax];
      }
      rho_s[tid] = rho;
    }
    base_s[tid] = base;
    info_s[tid] = info;
  }
  __syncthreads();
  for (int s = 0; s < P.S; ++s) {
    // gather the block residual of step s
    for (int idx = tid; idx < NC * NT * ND; idx += kT) {
      const int c = idx / (NT * ND);
      const int rem = idx - c * (NT * ND);
      const int i = rem / ND;
      const int l = rem - i * ND;
      const long long base = base_s[c];
      double v = 0.0;
      if (base >= 0) {
        const int lx = l % N, ly = (l / N) % N, lz = DIM == 3 ? l / (N * N) : 0;
        v = r[(static_cast<long long>(s) * NT + i) * P.n_space + base + lz * dxy + ly * dx + lx];
      }
      R[idx] = v;
      W[idx] = v;
    }
    __syncthreads();
    // hat r = S^T r (axis by axis); Dirichlet rows of S are zero
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      for (int ln = tid; ln < NC * NT * LINES; ln += kT) {
        const int ci = ln / LINES, line = ln - ci * LINES;
        const int c = ci / NT;
        if (base_s[c] < 0) continue;
        const int info = info_s[c];
        const int t = (info >> (8 + 2 * a)) & 3;
        if (a == 0) sweep<N, true>(W + ci * ND, lbase<N, 0>(line), 1, P.S1[0][t]);
        if (a == 1) sweep<N, true>(W + ci * ND, lbase<N, 1>(line), N, P.S1[1][t]);
        if (a == 2) sweep<N, true>(W + ci * ND, lbase<N, 2>(line), N * N, P.S1[2][t]);
      }
      __syncthreads();
    }
    // per eigen-index n_t x n_t solves
    for (int idx = tid; idx < NC * ND; idx += kT) {
      const int c = idx / ND, e = idx - (idx / ND) * ND;
      if (base_s[c] < 0) continue;
      const int info = info_s[c];
      const int ex = e % N, ey = (e / N) % N, ez = DIM == 3 ? e / (N * N) : 0;
      double lam = P.L1[0][info >> 8 & 3][ex] + P.L1[1][info >> 10 & 3][ey];
      if (DIM == 3) lam += P.L1[2][info >> 12 & 3][ez];
      lam *= rho_s[c];
      double b[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < NT; ++i) b[i] = W[(c * NT + i) * ND + e];
      if (P.tdiag)
        temporal_solve<NT, true>(P, lam, b);
      else
        temporal_solve<NT, false>(P, lam, b);
#pragma unroll
      for (int i = 0; i < NT; ++i) W[(c * NT + i) * ND + e] = b[i];
    }
    __syncthreads();
    // z_T = S hat z
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      for (int ln = tid; ln < NC * NT * LINES; ln += kT) {
        const int ci = ln / LINES, line = ln - ci * LINES;
        const int c = ci / NT;
        if (base_s[c] < 0) continue;
        const int info = info_s[c];
        const int t = (info >> (8 + 2 * a)) & 3;
        if (a == 0) sweep<N, false>(W + ci * ND, lbase<N, 0>(line), 1, P.S1[0][t]);
        if (a == 1) sweep<N, false>(W + ci * ND, lbase<N, 1>(line), N, P.S1[1][t]);
        if (a == 2) sweep<N, false>(W + ci * ND, lbase<N, 2>(line), N * N, P.S1[2][t]);
      }
      __syncthreads();
    }
    // weighted scatter-add; Dirichlet rows are identity (correction = r)
    for (int idx = tid; idx < NC * NT * ND; idx += kT) {
      const int c = idx / (NT * ND);
      const int rem = idx - c * (NT * ND);
      const int i = rem / ND;
      const int l = rem - i * ND;
      const long long base = base_s[c];
      if (base < 0) continue;
      const int lx = l % N, ly = (l / N) % N, lz = DIM == 3 ? l / (N * N) : 0;
      const int m = info_s[c];
      bool bd = ((m & 1) && lx == 0) || ((m & 2) && lx == N - 1) || ((m & 4) && ly == 0) || ((m & 8) && ly == N - 1);
      if (DIM == 3) bd = bd || ((m & 16) && lz == 0) || ((m & 32) && lz == N - 1);
      const long long g = base + lz * dxy + ly * dx + lx;
      // multiplicity: cells sharing the dof (asm_smoother.cpp:45-49)
      double mult = 1.0;
      if ((lx == 0 && !(m & 1)) || (lx == N - 1 && !(m & 2))) mult *= 2.0;
      if ((ly == 0 && !(m & 4)) || (ly == N - 1 && !(m & 8))) mult *= 2.0;
      if (DIM == 3 && ((lz == 0 && !(m & 16)) || (lz == N - 1 && !(m & 32)))) mult *= 2.0;
      const double v = bd ? R[idx] : W[idx];
      atomicAdd(z + (static_cast<long long>(s) * NT + i) * P.n_space + g, scale * v / mult);
    }
    __syncthreads();
  }
}

// 1D eigenbasis line transforms. Generic: out[e] = sum_k S[k][e] in[k]
// (forward, S^T) / out[k] = sum_e S[k][e] in[e] (backward, S). EO: the
// interior position class, whose host-reordered eigenvectors are symmetric
// (columns 0 .. HE-1) then antisymmetric (HE .. N-1) about the cell centre,
// so both transforms split into even / odd halves (N = 5: 13 FMAs instead
// of 25) and read the table at compile-time indices.
template <int N, bool EO>
__device__ __forceinline__ void fdm_fwd(const double (&S)[kMaxN][kMaxN], const double (&in)[N], double (&out)[N]) {
  if constexpr (EO) {
    constexpr int H = N / 2, HE = (N + 1) / 2;
    double ev[HE], ov[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
      ev[k] = in[k] + in[N - 1 - k];
      ov[k] = in[k] - in[N - 1 - k];
    }
    if constexpr (N % 2 == 1) ev[H] = in[H];
#pragma unroll
    for (int e = 0; e < HE; ++e) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < HE; ++k) acc = fma(S[k][e], ev[k], acc);
      out[e] = acc;
    }
#pragma unroll
    for (int e = 0; e < H; ++e) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < H; ++k) acc = fma(S[k][HE + e], ov[k], acc);
      out[HE + e] = acc;
    }
  } else {
#pragma unroll
    for (int e = 0; e < N; ++e) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) acc = fma(S[k][e], in[k], acc);
      out[e] = acc;
    }
  }
}
template <int N, bool EO>
__device__ __forceinline__ void fdm_bwd(const double (&S)[kMaxN][kMaxN], const double (&in)[N], double (&out)[N]) {
  if constexpr (EO) {
    constexpr int H = N / 2, HE = (N + 1) / 2;
#pragma unroll
    for (int k = 0; k < HE; ++k) {
      double A = 0.0, B = 0.0;
#pragma unroll
      for (int e = 0; e < HE; ++e) A = fma(S[k][e], in[e], A);
      if (k < H) {
#pragma unroll
        for (int e = 0; e < H; ++e) B = fma(S[k][HE + e], in[HE + e], B);
        out[k] = A + B;
        out[N - 1 - k] = A - B;
      } else {
        out[k] = A;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) acc = fma(S[k][e], in[e], acc);
      out[k] = acc;
    }
  }
}

// the five stages of one cell batch; EO: every cell of the CTA is interior
// along all three axes (position class 0, even-odd transforms)
template <int N, int NT, bool TD, bool EO>
__device__ __forceinline__ void fdm_stages(const DevFDM& P, const double* __restrict__ r, double* __restrict__ z,
                                           double scale, double* W, bool valid, long long base, int mask, int tx,
                                           int ty, int tz, double rho, int a, int b, int oy, int ox, int oz) {
  using Y = stc::FdmLayout<N, NT>;
  constexpr int SD = Y::SD, RY = Y::RY, PZ = Y::PZ;
  constexpr int p = N - 1;
  const long long dx = P.dofs[0], dxy = P.dofs[0] * P.dofs[1];
  auto bdry = [&](int lx, int ly, int lz) {
    return ((mask & 1) && lx == 0) || ((mask & 2) && lx == p) || ((mask & 4) && ly == 0) || ((mask & 8) && ly == p) ||
           ((mask & 16) && lz == 0) || ((mask & 32) && lz == p);
  };
  const double(&Sx)[kMaxN][kMaxN] = P.S1[0][EO ? 0 : tx];
  const double(&Sy)[kMaxN][kMaxN] = P.S1[1][EO ? 0 : ty];
  const double(&Sz)[kMaxN][kMaxN] = P.S1[2][EO ? 0 : tz];
  {  // one step per CTA row (blockIdx.y): no loop-invariant table hoisting
    const long long st = blockIdx.y;
    const double* rs = r + st * NT * P.n_space;
    double* zs = z + st * NT * P.n_space;
    // A: y-owner (x = a, z = b): gather, S_y^T
    if (valid) {
#pragma unroll
      for (int f = 0; f < NT; ++f) {
        double in[N], out[N];
#pragma unroll
        for (int k = 0; k < N; ++k) in[k] = __ldg(rs + f * P.n_space + base + b * dxy + k * dx + a);
        fdm_fwd<N, EO>(Sy, in, out);
#pragma unroll
        for (int e = 0; e < N; ++e) W[oy + f * SD + e * RY] = out[e];
      }
    }
    __syncthreads();
    // B: x-owner (y = a, z = b): S_x^T
    if (valid) {
#pragma unroll
      for (int f = 0; f < NT; ++f) {
        double in[N], out[N];
#pragma unroll
        for (int k = 0; k < N; ++k) in[k] = W[ox + f * SD + k];
        fdm_fwd<N, EO>(Sx, in, out);
#pragma unroll
        for (int e = 0; e < N; ++e) W[ox + f * SD + e] = out[e];
      }
    }
    __syncthreads();
    // C: z-owner (eigen-indices ex = a, ey = b): S_z^T, solves, S_z
    if (valid) {
      double v[NT][N];
#pragma unroll
      for (int f = 0; f < NT; ++f) {
        double in[N];
#pragma unroll
        for (int k = 0; k < N; ++k) in[k] = W[oz + f * SD + k * PZ];
        fdm_fwd<N, EO>(Sz, in, v[f]);
      }
      const double lxy = P.L1[0][EO ? 0 : tx][a] + P.L1[1][EO ? 0 : ty][b];
#pragma unroll
      for (int e = 0; e < N; ++e) {
        double bb[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int f = 0; f < NT; ++f) bb[f] = v[f][e];
        temporal_solve<NT, TD>(P, rho * (lxy + P.L1[2][EO ? 0 : tz][e]), bb);
#pragma unroll
        for (int f = 0; f < NT; ++f) v[f][e] = bb[f];
      }
#pragma unroll
      for (int f = 0; f < NT; ++f) {
        double out[N];
        fdm_bwd<N, EO>(Sz, v[f], out);
#pragma unroll
        for (int k = 0; k < N; ++k) W[oz + f * SD + k * PZ] = out[k];
      }
    }
    __syncthreads();
    // D: x-owner: S_x
    if (valid) {
#pragma unroll
      for (int f = 0; f < NT; ++f) {
        double in[N], out[N];
#pragma unroll
        for (int e = 0; e < N; ++e) in[e] = W[ox + f * SD + e];
        fdm_bwd<N, EO>(Sx, in, out);
#pragma unroll
        for (int k = 0; k < N; ++k) W[ox + f * SD + k] = out[k];
      }
    }
    __syncthreads();
    // E: y-owner: S_y, weighted scatter (asm_smoother.cpp:45-49, 75)
    if (valid) {
      const double wxz = ((a == 0 && !(mask & 1)) || (a == p && !(mask & 2)) ? 0.5 : 1.0) *
                         ((b == 0 && !(mask & 16)) || (b == p && !(mask & 32)) ? 0.5 : 1.0);
#pragma unroll
      for (int f = 0; f < NT; ++f) {
        double in[N], out[N];
#pragma unroll
        for (int e = 0; e < N; ++e) in[e] = W[oy + f * SD + e * RY];
        fdm_bwd<N, EO>(Sy, in, out);
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const long long g = base + b * dxy + k * dx + a;
          const double val = bdry(a, k, b) ? __ldg(rs + f * P.n_space + g) : out[k];
          const double wy = (k == 0 && !(mask & 4)) || (k == p && !(mask & 8)) ? 0.5 : 1.0;
          atomicAdd(zs + f * P.n_space + g, scale * wxz * wy * val);
        }
      }
    }
  }
}

// 3D line-owner FDM solve (the st_lines.cuh pattern): a 128-thread CTA owns
// NC cells, thread (c, a, b) owns lattice line (a, b) of cell c along the
// axis the stage sweeps, for the n_t fields of the step blockIdx.y, in
// registers. y-owner gathers r and applies S_y^T, x-owner S_x^T,
// z-owner S_z^T + the n_t x n_t solves at its N eigen-points + S_z, x-owner
// S_x, y-owner S_y and the weighted scatter (Dirichlet rows: w r, re-read).
// MODE 0: every CTA, generic transforms; 1: only CTAs whose cells are all
// interior, even-odd transforms; 2: only the other CTAs, generic. Modes 1 and
// 2 are two launches over the same grid (CTAs of the other kind return at
// once), so each kernel's code stays small enough for the instruction cache.
template <int N, int NT, bool TD, int MODE>
__global__ void __launch_bounds__(128, 4) fdm_lines_kernel(const __grid_constant__ DevFDM P,
                                                        const double* __restrict__ r, double* __restrict__ z,
                                                        double scale) {
  using Y = stc::FdmLayout<N, NT>;  // bank-conflict-modelled (scripts/gen_cart_layout.py)
  constexpr int NL = N * N, NC = 128 / NL, RY = Y::RY, PZ = Y::PZ;
  __shared__ double W[NC * Y::CS];
  const int t = threadIdx.x;
  const int c = t / NL, l = t - (t / NL) * NL;
  const int a = l % N, b = l / N;
  const long long n_cells = P.cells[0] * P.cells[1] * P.cells[2];
  const long long cell = static_cast<long long>(blockIdx.x) * NC + c;
  const bool valid = c < NC && cell < n_cells && !(P.skip && P.skip[cell]);
  const long long dx = P.dofs[0], dxy = P.dofs[0] * P.dofs[1];
  constexpr int p = N - 1;
  long long base = 0;
  int mask = 0, tx = 0, ty = 0, tz = 0;
  double rho = 1.0;
  if (valid) {
    const unsigned ci = static_cast<unsigned>(cell);
    const unsigned nx = static_cast<unsigned>(P.cells[0]), ny = static_cast<unsigned>(P.cells[1]),
                   nz = static_cast<unsigned>(P.cells[2]);
    const unsigned cx = ci % nx, cy = (ci / nx) % ny, cz = ci / (nx * ny);
    base = static_cast<long long>(cz) * p * dxy + static_cast<long long>(cy) * p * dx + static_cast<long long>(cx) * p;
    tx = (cx == 0 ? 1 : 0) | (cx == nx - 1 ? 2 : 0);
    ty = (cy == 0 ? 1 : 0) | (cy == ny - 1 ? 2 : 0);
    tz = (cz == 0 && (P.zbc & 1) ? 1 : 0) | (cz == nz - 1 && (P.zbc & 2) ? 2 : 0);
    mask = tx | (ty << 2) | (tz << 4);
    if (P.rho0) {
      const long long ax = cx >> P.rho_shift, ay = cy >> P.rho_shift, az = (cz + P.cz0) >> P.rho_shift;
      rho = P.rho0[(az * P.cells0[1] + ay) * P.cells0[0] + ax];
    }
  }
  const int cb = c * Y::CS;
  const int oy = cb + a + PZ * b, oz = cb + a + RY * b;
  const int ox = cb + RY * (Y::SWAP ? b : a) + PZ * (Y::SWAP ? a : b);
  // CTAs whose cells are all interior take the even-odd transforms (P.eo = 0
  // when the host could not order the interior eigenvectors by parity: one
  // MODE 0 launch)
  if constexpr (MODE != 0) {
    const bool all_interior = __syncthreads_and(!valid || mask == 0);
    if (all_interior != (MODE == 1)) return;
  }
  fdm_stages<N, NT, TD, MODE == 1>(P, r, z, scale, W, valid, base, mask, tx, ty, tz, rho, a, b, oy, ox, oz);
}

// ---------------------------------------------------------------------------
// Owner-computes FDM sweep (3D): the same cell solves as fdm_lines_kernel, but
// the weighted sum over the overlapping cells (asm_smoother.cpp:45-49, 75) is
// formed in shared memory instead of by fp64 atomics into z. A CTA owns a
// tile of TX x TY cells in x-y and marches a chunk of cell layers along z:
//   stage: the residual on the layer's (TX p + 1) x (TY p + 1) x (p + 1)
//     node box (cp.async, issued one layer ahead)
//   Fy: thread = (x node of the box, plane, field): S_y^T of every y cell of
//     the tile along its column (node columns on cell faces serve both cells)
//   Fx: thread = (y cell, y eigen-index, plane, field): S_x^T per x cell
//   Z:  thread = (cell, x and y eigen-indices): S_z^T, the n_t x n_t solves
//     at the p + 1 z eigen-indices, S_z
//   Bx: S_x per x cell, summed at shared x nodes (assembled along x)
//   By: S_y per y cell, summed at shared y nodes, times the inverse
//     multiplicity of the node, then z += scale * (.) -- a plain
//     read-modify-write for nodes only this CTA's cells touch; fp64 atomics
//     only on the tile's edge nodes and on the chunk's first / last plane.
//     The layer's top plane is carried in shared memory to the next layer.
// Dirichlet nodes receive scale * r once (the identity rows summed over the
// cells divided by the multiplicity), from the CTA owning the node.
namespace ft {
constexpr int kT = 512, TX = 4, TY = 4;
template <int N, int NT>
struct Cfg {
  static constexpr int P = N - 1;
  static constexpr int NX = TX * P + 1, NY = TY * P + 1;
  // residual box rows [f][b][y], each one 16-byte aligned bulk copy of the
  // 16-byte aligned span covering the row's NX doubles (x at [s + x], s the
  // row's start parity): pitch RP doubles
  static constexpr int RW = ((NX + 1 + 1) / 2) * 2;  // doubles per row copy (NX + 1 rounded to even)
  static constexpr int RP = RW;
  static constexpr int ROWS = NT * N * NY;
  static constexpr int RB = ROWS * RP;
  // x-assembled / y-transformed data W1[cy][ey][f][b][x]
  static constexpr int W1 = TY * N * NT * N * NX;
  // per-cell coefficients W2[cx][ex][cy][ey] x 21-padded (b, f)
  static constexpr int W2S = N * NT + 1;
  static constexpr int W2 = TX * N * TY * N * W2S;
  static constexpr int CY = 2 * NT * NY * NX;  // carried top plane [parity][f][y][x]
  static constexpr size_t smem_bytes() { return sizeof(double) * static_cast<size_t>(RB + W1 + W2 + CY) + 16; }
  static constexpr int IFY = NX * N * NT, IFX = TY * N * N * NT, IZ = TX * TY * N * N;
  static_assert(IFX <= kT && IZ <= kT, "one Fx / Z item per thread");
};

__device__ __forceinline__ int axis_class(long long c, long long n, bool lo_phys, bool hi_phys) {
  return (c == 0 && lo_phys ? 1 : 0) | (c == n - 1 && hi_phys ? 2 : 0);
}

// share of a Dirichlet node's identity row handled here: the cells around it
// that are not solved by the exact per-cell kernel (skip), over all its cells
__device__ double dirichlet_share(const DevFDM& P, long long gx, long long gy, long long gz) {
  if (!P.skip) return 1.0;
  const int p = P.p;
  int all = 0, mine = 0;
  const long long g[3] = {gx, gy, gz};
  long long lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    const long long c = g[a] / p;
    lo[a] = (g[a] % p == 0) ? c - 1 : c;
    hi[a] = c;
    if (lo[a] < 0) lo[a] = 0;
    if (hi[a] > P.cells[a] - 1) hi[a] = P.cells[a] - 1;
  }
  for (long long cz = lo[2]; cz <= hi[2]; ++cz)
    for (long long cy = lo[1]; cy <= hi[1]; ++cy)
      for (long long cx = lo[0]; cx <= hi[0]; ++cx) {
        ++all;
        if (!P.skip[(cz * P.cells[1] + cy) * P.cells[0] + cx]) ++mine;
      }
  return all > 0 ? static_cast<double>(mine) / all : 0.0;
}

__device__ __forceinline__ void bulk_g2s_fdm(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes), "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
               : "memory");
}

template <int N, int NT, bool TD>
__global__ void __launch_bounds__(kT, 1) fdm_tile_kernel(const __grid_constant__ DevFDM P, const double* __restrict__ r,
                                                         double* __restrict__ z, double scale, int ntx, int zc) {
  using C = Cfg<N, NT>;
  constexpr int p = C::P, NX = C::NX, NY = C::NY;
  extern __shared__ __align__(16) double sm[];
  double* Rb = sm;
  double* W1 = Rb + C::RB;
  double* W2 = W1 + C::W1;
  double* Cy = W2 + C::W2;
  const int t = threadIdx.x;
  const long long dx = P.dofs[0], dy = P.dofs[1], dz = P.dofs[2], dxy = dx * dy, ns = P.n_space;
  const long long ncx = P.cells[0], ncy = P.cells[1];
  const int ncz = static_cast<int>(P.cells[2]);
  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  const long long cx0 = static_cast<long long>(tx) * TX, cy0 = static_cast<long long>(ty) * TY;
  const long long X0 = cx0 * p, Y0 = cy0 * p;
  const int L0 = static_cast<int>(blockIdx.y) * zc, L1 = L0 + zc < ncz ? L0 + zc : ncz;
  const bool lo_phys = (P.zbc & 1) != 0, hi_phys = (P.zbc & 2) != 0;
  const long long st = blockIdx.z;  // step: fields st*NT .. st*NT + NT - 1
  const double* rs = r + st * NT * ns;
  double* zs = z + st * NT * ns;

  unsigned long long* bar = reinterpret_cast<unsigned long long*>(Cy + C::CY);
  const long long total = static_cast<long long>(P.S) * NT * ns;
  // ---- stage the residual box of layer e: thread t < ROWS issues row t as
  // one bulk copy (rows beyond the lattice are zero-filled, the array's last
  // row avoids reading past the end)
  auto stage = [&](int e) {
    if (t < C::ROWS) {
      const int y = t % NY, fb = t / NY;
      const int b = fb % N, f = fb / N;
      const long long gy = Y0 + y;
      double* dst = Rb + t * C::RP;
      if (gy < dy) {
        const long long g = (st * NT + f) * ns + (static_cast<long long>(e) * p + b) * dxy + gy * dx + X0;
        const long long g0 = g & ~1LL;
        if (g0 + C::RW <= total) {
          bulk_g2s_fdm(dst, r + g0, sizeof(double) * C::RW, bar);
        } else {
          const int n16 = static_cast<int>(((total - g0) / 2) * 2);
          if (n16 > 0) bulk_g2s_fdm(dst, r + g0, sizeof(double) * n16, bar);
          for (int k = n16; k < C::RW; ++k) dst[k] = g0 + k < total ? r[g0 + k] : 0.0;
          if (n16 < C::RW) asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(
                                          static_cast<unsigned>(__cvta_generic_to_shared(bar))),
                                      "r"(static_cast<unsigned>(sizeof(double) * (C::RW - n16)))
                                      : "memory");
        }
      } else {
        for (int k = 0; k < C::RW; ++k) dst[k] = 0.0;
        asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(
                         static_cast<unsigned>(__cvta_generic_to_shared(bar))),
                     "r"(static_cast<unsigned>(sizeof(double) * C::RW))
                     : "memory");
      }
    }
  };
  auto stage_arm = [&]() {
    if (t == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(bar))),
                   "r"(static_cast<unsigned>(sizeof(double) * C::RW * C::ROWS))
                   : "memory");
  };
  // start parity of box row (f, b, y): x = 0 of the row sits at [s + 0]
  auto row_shift = [&](int f, int b, int y, int e) -> int {
    const long long g = (st * NT + f) * ns + (static_cast<long long>(e) * p + b) * dxy + (Y0 + y) * dx + X0;
    return static_cast<int>(g & 1);
  };

  // per-item identities
  // Fy / By: items i = x + NX (b + N f) (x node, plane b, field f), looped
  // Fx / Bx: (cy, ey, f, b) -- t = b + N (f + NT (ey + N cy))
  const int fx_b = t % N, fx_f = (t / N) % NT, fx_ey = (t / (N * NT)) % N, fx_cy = t / (N * NT * N);
  // Z: (ey, cy, ex, cx) -- t = ey + N (cy + TY (ex + N cx))
  const int z_ey = t % N, z_cy = (t / N) % TY, z_ex = (t / (N * TY)) % N, z_cx = t / (N * TY * N);
  auto w1 = [&](int cy, int ey, int f, int b, int x) { return W1 + (((cy * N + ey) * NT + f) * N + b) * NX + x; };
  auto w2 = [&](int cx, int ex, int cy, int ey) { return W2 + ((ey + N * cy) + TY * N * (ex + N * cx)) * C::W2S; };

  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
                 "r"(1u)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  stage_arm();
  stage(L0);
  unsigned phase = 0;
  for (int e = L0; e < L1; ++e) {
    {
      unsigned ok = 0;
      for (long long spin = 0; !ok; ++spin) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))), "r"(phase)
            : "memory");
        if (spin > (1LL << 28)) __trap();
      }
      phase ^= 1;
    }
    __syncthreads();
    const int tz = axis_class(e, ncz, lo_phys, hi_phys);
    // ---- Fy: S_y^T of each y cell along the node column
    for (int it = t; it < C::IFY; it += kT) {
      const int fy_x = it % NX, fy_b = (it / NX) % N, fy_f = it / (NX * N);
      const double* col = Rb + (fy_f * N + fy_b) * NY * C::RP + fy_x;
      const int s0 = row_shift(fy_f, fy_b, 0, e);
#pragma unroll
      for (int cy = 0; cy < TY; ++cy) {
        double in[N], out[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const int yy = cy * p + k;
          in[k] = col[yy * C::RP + (s0 ^ (yy & static_cast<int>(dx & 1)))];
        }
        const int cls = axis_class(cy0 + cy, ncy, true, true);
        if (cls == 0 && P.eo)
          fdm_fwd<N, true>(P.S1[1][0], in, out);
        else
          fdm_fwd<N, false>(P.S1[1][cls], in, out);
#pragma unroll
        for (int k = 0; k < N; ++k) *w1(cy, k, fy_f, fy_b, fy_x) = out[k];
      }
    }
    __syncthreads();
    if (e + 1 < L1) {  // the box is consumed: stage the next layer
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      stage_arm();
      stage(e + 1);
    }
    // ---- Fx: S_x^T per x cell
    if (t < C::IFX) {
      const double* row = w1(fx_cy, fx_ey, fx_f, fx_b, 0);
#pragma unroll
      for (int cx = 0; cx < TX; ++cx) {
        double in[N], out[N];
#pragma unroll
        for (int k = 0; k < N; ++k) in[k] = row[cx * p + k];
        const int cls = axis_class(cx0 + cx, ncx, true, true);
        if (cls == 0 && P.eo)
          fdm_fwd<N, true>(P.S1[0][0], in, out);
        else
          fdm_fwd<N, false>(P.S1[0][cls], in, out);
#pragma unroll
        for (int k = 0; k < N; ++k) w2(cx, k, fx_cy, fx_ey)[fx_b + N * fx_f] = out[k];
      }
    }
    __syncthreads();
    // ---- Z: S_z^T, temporal solves, S_z for one (cell, ex, ey)
    if (t < C::IZ) {
      double* v = w2(z_cx, z_ex, z_cy, z_ey);
      const long long gcx = cx0 + z_cx, gcy = cy0 + z_cy;
      const bool valid = gcx < ncx && gcy < ncy &&
                         !(P.skip && P.skip[(static_cast<long long>(e) * ncy + gcy) * ncx + gcx]);
      double a[NT][N];
      if (valid) {
        const int cxs = axis_class(gcx, ncx, true, true), cys = axis_class(gcy, ncy, true, true);
        double rho = 1.0;
        if (P.rho0) {
          const long long ax = gcx >> P.rho_shift, ay = gcy >> P.rho_shift, az = (e + P.cz0) >> P.rho_shift;
          rho = __ldg(P.rho0 + (az * P.cells0[1] + ay) * P.cells0[0] + ax);
        }
#pragma unroll
        for (int f = 0; f < NT; ++f) {
          double in[N];
#pragma unroll
          for (int k = 0; k < N; ++k) in[k] = v[k + N * f];
          if (tz == 0 && P.eo)
            fdm_fwd<N, true>(P.S1[2][0], in, a[f]);
          else
            fdm_fwd<N, false>(P.S1[2][tz], in, a[f]);
        }
        const double lxy = P.L1[0][cxs][z_ex] + P.L1[1][cys][z_ey];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double bb[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int f = 0; f < NT; ++f) bb[f] = a[f][k];
          temporal_solve<NT, TD>(P, rho * (lxy + P.L1[2][tz][k]), bb);
#pragma unroll
          for (int f = 0; f < NT; ++f) a[f][k] = bb[f];
        }
#pragma unroll
        for (int f = 0; f < NT; ++f) {
          double out[N];
          if (tz == 0 && P.eo)
            fdm_bwd<N, true>(P.S1[2][0], a[f], out);
          else
            fdm_bwd<N, false>(P.S1[2][tz], a[f], out);
#pragma unroll
          for (int k = 0; k < N; ++k) v[k + N * f] = out[k];
        }
      } else {
#pragma unroll
        for (int f = 0; f < NT; ++f)
#pragma unroll
          for (int k = 0; k < N; ++k) v[k + N * f] = 0.0;
      }
    }
    __syncthreads();
    // ---- Bx: S_x per x cell, assembled along x
    if (t < C::IFX) {
      double* row = w1(fx_cy, fx_ey, fx_f, fx_b, 0);
      double carry = 0.0;
#pragma unroll
      for (int cx = 0; cx < TX; ++cx) {
        double in[N], out[N];
#pragma unroll
        for (int k = 0; k < N; ++k) in[k] = w2(cx, k, fx_cy, fx_ey)[fx_b + N * fx_f];
        const int cls = axis_class(cx0 + cx, ncx, true, true);
        if (cls == 0 && P.eo)
          fdm_bwd<N, true>(P.S1[0][0], in, out);
        else
          fdm_bwd<N, false>(P.S1[0][cls], in, out);
        row[cx * p] = carry + out[0];
#pragma unroll
        for (int k = 1; k < p; ++k) row[cx * p + k] = out[k];
        carry = out[p];
      }
      row[TX * p] = carry;
    }
    __syncthreads();
    // ---- By: S_y per y cell, assembled along y; weights; write
    for (int it = t; it < C::IFY; it += kT) {
      const int x = it % NX, b = (it / NX) % N, f = it / (NX * N);
      double col[NY];
      {
        double carry = 0.0;
#pragma unroll
        for (int cy = 0; cy < TY; ++cy) {
          double in[N], out[N];
#pragma unroll
          for (int k = 0; k < N; ++k) in[k] = *w1(cy, k, f, b, x);
          const int cls = axis_class(cy0 + cy, ncy, true, true);
          if (cls == 0 && P.eo)
            fdm_bwd<N, true>(P.S1[1][0], in, out);
          else
            fdm_bwd<N, false>(P.S1[1][cls], in, out);
          col[cy * p] = carry + out[0];
#pragma unroll
          for (int k = 1; k < p; ++k) col[cy * p + k] = out[k];
          carry = out[p];
        }
        col[TY * p] = carry;
      }
      const long long gz = static_cast<long long>(e) * p + b;
      const long long gx = X0 + x;
      // the layer's bottom plane: add the previous layer's top plane (carry
      // buffers alternate with the layer parity)
      if (b == 0 && e > L0) {
        const double* cin = Cy + ((((e - 1) & 1) * NT + f) * NY) * NX + x;
#pragma unroll
        for (int y = 0; y < NY; ++y) col[y] += cin[y * NX];
      }
      const bool last_layer = e == L1 - 1;
      if (b == p && !last_layer) {
        double* cout = Cy + (((e & 1) * NT + f) * NY) * NX + x;
#pragma unroll
        for (int y = 0; y < NY; ++y) cout[y * NX] = col[y];
      } else if (gx < dx) {
        // plane gz is final here, or (chunk-boundary planes) a partial sum
        const bool zshared = (b == 0 && e == L0 && L0 > 0) || (b == p && L1 < ncz);
        const bool zdir = (gz == 0 && lo_phys) || (gz == dz - 1 && hi_phys);
        const bool z_owner = b < p || L1 == ncz;  // Dirichlet r added once
        const bool xdir = gx == 0 || gx == dx - 1;
        const bool xedge = (x == 0 && tx > 0) || (x == NX - 1 && gx != dx - 1);
        const bool xown = x < NX - 1 || gx == dx - 1;
        const double wz = (gz % p == 0 && !zdir) ? 0.5 : 1.0;
        // a slab's interface plane: the other slab holds the other half of
        // the node's cells (the interface sum adds its share)
        const double ziface = ((gz == 0 && !lo_phys) || (gz == dz - 1 && !hi_phys)) ? 0.5 : 1.0;
        const double wx = (gx % p == 0 && !xdir) ? 0.5 : 1.0;
        double* zp = zs + f * ns + gz * dxy + gx;
        const double* rp = rs + f * ns + gz * dxy + gx;
        // plain read-modify-write nodes: all old values requested first
        double old[NY];
        bool plain[NY];
#pragma unroll
        for (int y = 0; y < NY; ++y) {
          const long long gy = Y0 + y;
          const bool in = gy < dy;
          const bool ydir = gy == 0 || gy == dy - 1;
          const bool yedge = (y == 0 && ty > 0) || (y == NY - 1 && gy != dy - 1);
          plain[y] = in && !(zdir || xdir || ydir) && !(zshared || xedge || yedge);
          old[y] = plain[y] ? zp[gy * dx] : 0.0;
        }
#pragma unroll
        for (int y = 0; y < NY; ++y) {
          const long long gy = Y0 + y;
          if (gy >= dy) break;
          const bool ydir = gy == 0 || gy == dy - 1;
          const bool yown = y < NY - 1 || gy == dy - 1;
          if (zdir || xdir || ydir) {
            if (z_owner && xown && yown)
              zp[gy * dx] += scale * ziface * dirichlet_share(P, gx, gy, gz) * __ldg(rp + gy * dx);
            continue;
          }
          const double wy = (gy % p == 0) ? 0.5 : 1.0;
          const double val = scale * wx * wy * wz * col[y];
          if (plain[y])
            zp[gy * dx] = old[y] + val;
          else
            atomicAdd(zp + gy * dx, val);
        }
      }
    }
  }
}
}  // namespace ft

template <int N, int NT>
void launch_tile(const DevFDM& P, const double* r, double* z, double scale, cudaStream_t s) {
  using C = ft::Cfg<N, NT>;
  const long long ntx = (P.cells[0] + ft::TX - 1) / ft::TX, nty = (P.cells[1] + ft::TY - 1) / ft::TY;
  const long long tiles = ntx * nty, ncz = P.cells[2];
  long long nch = std::max<long long>(1, (148LL * 12 + tiles * P.S - 1) / (tiles * P.S));
  nch = std::min<long long>(nch, std::max<long long>(1, ncz / 2));
  const long long zc = (ncz + nch - 1) / nch;
  nch = (ncz + zc - 1) / zc;
  const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(nch), static_cast<unsigned>(P.S));
  count_launch();
  auto go = [&](auto kern) {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::smem_bytes()));
      configured = true;
    }
    kern<<<grid, ft::kT, C::smem_bytes(), s>>>(P, r, z, scale, static_cast<int>(ntx), static_cast<int>(zc));
  };
  if (P.tdiag)
    go(ft::fdm_tile_kernel<N, NT, true>);
  else
    go(ft::fdm_tile_kernel<N, NT, false>);
}

template <int N, int NT>
void launch_lines(const DevFDM& P, const double* r, double* z, double scale, cudaStream_t s) {
  constexpr int NC = 128 / (N * N);
  const long long n_cells = P.cells[0] * P.cells[1] * P.cells[2];
  count_launch();
  const dim3 grid(static_cast<unsigned>((n_cells + NC - 1) / NC), static_cast<unsigned>(P.S));
  auto go = [&](auto td) {
    constexpr bool TD = decltype(td)::value;
    if (P.eo) {
      count_launch();  // the second launch of the pair
      fdm_lines_kernel<N, NT, TD, 1><<<grid, 128, 0, s>>>(P, r, z, scale);
      fdm_lines_kernel<N, NT, TD, 2><<<grid, 128, 0, s>>>(P, r, z, scale);
    } else {
      fdm_lines_kernel<N, NT, TD, 0><<<grid, 128, 0, s>>>(P, r, z, scale);
    }
  };
  if (P.tdiag)
    go(std::true_type{});
  else
    go(std::false_type{});
}

template <int DIM, int N, int NT>
void launch(const DevFDM& P, const double* r, double* z, double scale, cudaStream_t s) {
  if (DIM == 3) {
    // owner-computes tiles where one layer of TX x TY cells fits a CTA
    if constexpr (ft::Cfg<N, NT>::IFX <= ft::kT && ft::Cfg<N, NT>::IZ <= ft::kT) {
      launch_tile<N, NT>(P, r, z, scale, s);
      return;
    }
    launch_lines<N, NT>(P, r, z, scale, s);
    return;
  }
  using C = FCfg<DIM, N>;
  const size_t smem = sizeof(double) * (2 * C::NC * NT * C::ND + C::NC) + sizeof(long long) * C::NC + sizeof(int) * C::NC;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(asm_fdm_kernel<DIM, N, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  const long long n_cells = P.cells[0] * P.cells[1] * P.cells[2];
  count_launch();
  asm_fdm_kernel<DIM, N, NT><<<static_cast<unsigned>((n_cells + C::NC - 1) / C::NC), kT, smem, s>>>(P, r, z, scale);
}

template <int DIM, int N>
void launch_nt(const DevFDM& P, const double* r, double* z, double scale, cudaStream_t s) {
  switch (P.nt) {
    case 1: launch<DIM, N, 1>(P, r, z, scale, s); break;
    case 2: launch<DIM, N, 2>(P, r, z, scale, s); break;
    case 3: launch<DIM, N, 3>(P, r, z, scale, s); break;
    case 4: launch<DIM, N, 4>(P, r, z, scale, s); break;
    default: throw std::invalid_argument("FDM smoother: n_t must be in [1, 4]");
  }
}

}  // namespace

void fdm_add_correction(const DevFDM& P, const double* r, double* z, double scale, cudaStream_t s) {
  const int key = P.dim * 10 + P.n;
  switch (key) {
    case 22: launch_nt<2, 2>(P, r, z, scale, s); break;
    case 23: launch_nt<2, 3>(P, r, z, scale, s); break;
    case 24: launch_nt<2, 4>(P, r, z, scale, s); break;
    case 25: launch_nt<2, 5>(P, r, z, scale, s); break;
    case 32: launch_nt<3, 2>(P, r, z, scale, s); break;
    case 33: launch_nt<3, 3>(P, r, z, scale, s); break;
    case 34: launch_nt<3, 4>(P, r, z, scale, s); break;
    case 35: launch_nt<3, 5>(P, r, z, scale, s); break;
    default: throw std::invalid_argument("FDM smoother: unsupported dim/p");
  }
}

}  // namespace stmgb
