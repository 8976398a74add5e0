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
#include <vector>

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
// reciprocal by the hardware seed (rcp.approx.ftz.f64, >= 20 bits) and two
// Newton steps: full double accuracy for the normal, well-scaled pivots of
// the temporal blocks, without the special-case path of the IEEE division
__device__ __forceinline__ double rcp_newton(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
}

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
      w[i] = w[i] * rcp_newton(P.ta[i] + mu);
    } else if (P.tkind[i] == 1 && i + 1 < NT) {
      const double al = P.ta[i] + mu, be = P.tb[i];
      const double inv = rcp_newton(fma(al, al, be * be));
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

// the N temporal solves of one eigen-line at once (tdiag form): every entry of
// P / Q is loaded once and applied to all N right-hand sides
template <int N, int NT>
__device__ __forceinline__ void temporal_solve_line(const DevFDM& P, const double (&mu)[N], double (&v)[NT][N]) {
  double w[NT][N];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
#pragma unroll
    for (int e = 0; e < N; ++e) w[i][e] = 0.0;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const double c = P.tP[i * NT + j];
#pragma unroll
      for (int e = 0; e < N; ++e) w[i][e] = fma(c, v[j][e], w[i][e]);
    }
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    if (P.tkind[i] == 0) {
      const double ta = P.ta[i];
#pragma unroll
      for (int e = 0; e < N; ++e) w[i][e] *= rcp_newton(ta + mu[e]);
    } else if (P.tkind[i] == 1 && i + 1 < NT) {
      const double ta = P.ta[i], be = P.tb[i];
#pragma unroll
      for (int e = 0; e < N; ++e) {
        const double al = ta + mu[e];
        const double inv = rcp_newton(fma(al, al, be * be));
        const double w0 = w[i][e], w1 = w[i + 1 < NT ? i + 1 : i][e];
        w[i][e] = (al * w0 - be * w1) * inv;
        w[i + 1 < NT ? i + 1 : i][e] = (be * w0 + al * w1) * inv;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
#pragma unroll
    for (int e = 0; e < N; ++e) v[i][e] = 0.0;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const double c = P.tQ[i * NT + j];
#pragma unroll
      for (int e = 0; e < N; ++e) v[i][e] = fma(c, w[j][e], v[i][e]);
    }
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
// MODE 3: generic transforms, only the cells the strip kernel below leaves
// out (strips touching the boundary or holding an exactly-solved cell).
template <int N, int NT>
struct SCfg;
template <int N, int NT, bool TD, int MODE>
__device__ __forceinline__ void fdm_lines_group(const DevFDM& P, const double* __restrict__ r, double* __restrict__ z,
                                                double scale, double* W, long long group) {
  using Y = stc::FdmLayout<N, NT>;  // bank-conflict-modelled (scripts/gen_cart_layout.py)
  constexpr int NL = N * N, NC = 128 / NL, RY = Y::RY, PZ = Y::PZ;
  const int t = threadIdx.x;
  const int c = t / NL, l = t - (t / NL) * NL;
  const int a = l % N, b = l / N;
  const long long n_cells = P.cells[0] * P.cells[1] * P.cells[2];
  long long cell = group * NC + c;
  bool valid;
  if constexpr (MODE == 3) {
    valid = c < NC && cell < P.n_left;
    if (valid) cell = P.left[cell];
  } else {
    valid = c < NC && cell < n_cells && !(P.skip && P.skip[cell]);
  }
  const long long dx = P.dofs[0], dxy = P.dofs[0] * P.dofs[1];
  constexpr int p = N - 1;
  long long base = 0;
  int mask = 0, tx = 0, ty = 0, tz = 0;
  double rho = 1.0;
  unsigned cx = 0, cy = 0, cz = 0;
  if (valid) {
    const unsigned ci = static_cast<unsigned>(cell);
    const unsigned nx = static_cast<unsigned>(P.cells[0]), ny = static_cast<unsigned>(P.cells[1]),
                   nz = static_cast<unsigned>(P.cells[2]);
    cx = ci % nx, cy = (ci / nx) % ny, cz = ci / (nx * ny);
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
  if constexpr (MODE != 0 && MODE != 3) {
    const bool all_interior = __syncthreads_and(!valid || mask == 0);
    if (all_interior != (MODE == 1)) return;
  }
  (void)cx, (void)cy, (void)cz;
  fdm_stages<N, NT, TD, MODE == 1>(P, r, z, scale, W, valid, base, mask, tx, ty, tz, rho, a, b, oy, ox, oz);
}

template <int N, int NT, bool TD, int MODE>
__global__ void __launch_bounds__(128, 4) fdm_lines_kernel(const __grid_constant__ DevFDM P,
                                                        const double* __restrict__ r, double* __restrict__ z,
                                                        double scale) {
  using Y = stc::FdmLayout<N, NT>;
  constexpr int NC = 128 / (N * N);
  __shared__ double W[NC * Y::CS];
  // MODE 3: blockIdx.x counts groups of the left-out cell list
  fdm_lines_group<N, NT, TD, MODE>(P, r, z, scale, W, blockIdx.x);
}

// ---------------------------------------------------------------------------
// Strip form of the interior cells (even-odd transforms). A 128-thread CTA
// owns NCX cells consecutive in x of one (cy, cz) row and one step; one
// shared buffer, per cell [field][z][y][x], is used in place throughout:
//   load : one coalesced row of the strip's residual block per warp
//          instruction (cp.async), written straight into the cells' layout
//          (x-face nodes to both cells)
//   P1   : thread = (cell, field, z plane): S_x^T and S_y^T of the 5 x 5
//          plane in registers
//   P2   : thread = (cell, e_y, e_x): S_z^T, the n_t x n_t solves at its N
//          eigen-points, S_z for all fields
//   P3   : thread = (cell, field, z plane): S_y, S_x, multiplicity weights
//   scatter : one coalesced row of reductions into z per warp instruction,
//          x-face nodes summed over their two cells
//          (asm_smoother.cpp:45-49, 75).
// Against the line-owner kernel: 3 stages instead of 5 through shared memory
// (2 / 5 of its shared-memory traffic), row-contiguous global accesses instead
// of 5-double segments, N * NCX fewer reductions on the shared x faces.
template <int N, int NT>
struct SCfg {
  static constexpr int T = 128;
  static constexpr int NL = N * N;   // P2 threads per cell
  static constexpr int NP = NT * N;  // P1 / P3 threads per cell
  static constexpr int P = N - 1;
  static constexpr int min3(int a, int b, int c) { return a < b ? (a < c ? a : c) : (b < c ? b : c); }
  static constexpr int NCX = min3(T / NL, T / NP, 31 / P);  // cells per strip (one row <= 32 nodes)
  static constexpr int RX = P * NCX + 1;      // nodes of the strip along x
  static constexpr int ROWS = NT * N * N;     // (field, z, y) rows of the block
  static constexpr int BLK = ROWS * RX;
  static constexpr int ND = N * N * N;
  // one buffer, per cell [field][z][y][x], used in place by every stage. Cell
  // stride = N^2 NP (mod 16): the plane owners t = plane + NP * cell then
  // address word N^2 t (mod 16), conflict-free for odd N
  static constexpr int CS = NT * ND + (((NL * NP - NT * ND) % 16) + 16) % 16;
  static constexpr size_t smem_bytes() { return sizeof(double) * NCX * CS; }
  static_assert(RX <= 32, "one warp instruction per row");
};

// strips are the whole groups of NCX cells starting at cell 1 of every row
// that stay clear of the row's last cell: the cells left out along x are
// cell 0 and the tail of fewer than NCX + 1 cells
template <int N, int NT>
__host__ __device__ __forceinline__ unsigned strips_per_row(long long nx) {
  return nx >= 2 ? static_cast<unsigned>((nx - 2) / SCfg<N, NT>::NCX) : 0u;
}
template <int N, int NT>
__host__ __device__ __forceinline__ bool strip_left_out(const DevFDM& P, const unsigned char* skip, unsigned cx,
                                                        unsigned cy, unsigned cz) {
  constexpr unsigned NCX = SCfg<N, NT>::NCX;
  const unsigned nx = static_cast<unsigned>(P.cells[0]), ny = static_cast<unsigned>(P.cells[1]),
                 nz = static_cast<unsigned>(P.cells[2]);
  if (cx == 0 || (cx - 1) / NCX >= strips_per_row<N, NT>(nx) || cy == 0 || cy == ny - 1) return true;
  if ((cz == 0 && (P.zbc & 1)) || (cz == nz - 1 && (P.zbc & 2))) return true;
  (void)skip;  // exactly-solved cells inside a strip are masked by the strip kernel
  return false;
}

// 8-byte cp.async / fp64 reduction at base + 8 * off: the address is one
// mad.wide.u32 (lattice offsets inside a field fit 32 bits)
__device__ __forceinline__ void cp8_off(unsigned dst, const double* base, unsigned off) {
  asm volatile(
      "{\n"
      ".reg .u64 a;\n"
      "mad.wide.u32 a, %2, 8, %1;\n"
      "cp.async.ca.shared.global [%0], [a], 8;\n"
      "}\n" ::"r"(dst),
      "l"(base), "r"(off)
      : "memory");
}
__device__ __forceinline__ void red_off(double* base, unsigned off, double v) {
  asm volatile(
      "{\n"
      ".reg .u64 a;\n"
      "mad.wide.u32 a, %1, 8, %0;\n"
      "red.global.add.f64 [a], %2;\n"
      "}\n" ::"l"(base),
      "r"(off), "d"(v)
      : "memory");
}

// NT = n_t fields of a step; SG consecutive steps (independent blocks,
// asm_smoother.cpp:24-28) share the CTA so that NTF = NT * SG fields keep the
// plane owners busy (n_t = 2: 50 of 128 threads otherwise)
template <int N, int NT, int SG, bool TD>
__global__ void __launch_bounds__(SCfg<N, NT * SG>::T, 6) fdm_strip_kernel(const __grid_constant__ DevFDM P,
                                                                            const double* __restrict__ r,
                                                                            double* __restrict__ z, double scale) {
  constexpr int NTF = NT * SG;
  using C = SCfg<N, NTF>;
  constexpr int p = C::P, NCX = C::NCX, RX = C::RX, ROWS = C::ROWS, CS = C::CS, ND = C::ND;
  extern __shared__ __align__(16) double W[];  // per cell [field][z][y][x]
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const unsigned nx = static_cast<unsigned>(P.cells[0]), ny = static_cast<unsigned>(P.cells[1]);
  const unsigned sxn = strips_per_row<N, NTF>(nx);
  const unsigned sid = blockIdx.x;
  const unsigned sx = sid % sxn, cy = (sid / sxn) % ny, cz = sid / (sxn * ny);
  const unsigned cx0 = 1 + sx * NCX;
  if (strip_left_out<N, NTF>(P, P.skip, cx0, cy, cz)) return;  // CTA-uniform
  const int ncell = NCX;  // interior strips are whole
  const long long dx = P.dofs[0], dxy = P.dofs[0] * P.dofs[1];
  const long long base = static_cast<long long>(cz) * p * dxy + static_cast<long long>(cy) * p * dx +
                         static_cast<long long>(cx0) * p;
  const long long st = blockIdx.y;
  const double* rs = r + st * NTF * P.n_space + base;
  double* zs = z + st * NTF * P.n_space + base;
  // coefficient and "solved exactly elsewhere" flag of cell c of the strip
  // (the coefficient is uniform over an FDM cell's neighbourhood, not over the strip)
  auto rho_of = [&](int c) {
    if (!P.rho0) return 1.0;
    const long long ax = (cx0 + c) >> P.rho_shift, ay = cy >> P.rho_shift, az = (cz + P.cz0) >> P.rho_shift;
    return __ldg(P.rho0 + (az * P.cells0[1] + ay) * P.cells0[0] + ax);
  };
  const unsigned char* skip_row = P.skip ? P.skip + (static_cast<size_t>(cz) * ny + cy) * nx + cx0 : nullptr;
  auto skipped = [&](int c) { return skip_row && skip_row[c] != 0; };
  if (skip_row) {  // nothing to do when the exact kernel solves every cell of the strip (CTA-uniform)
    bool any = false;
    for (int c = 0; c < ncell; ++c) any = any || skip_row[c] == 0;
    if (!any) return;
  }
  // ---- load: row (f, lz, ly) of the block per warp instruction; a warp
  // takes (field, z) pairs, the N rows of a pair are unrolled. Lane = node x
  // of the strip: local node x % p of cell x / p, and, on a shared face,
  // node p of the cell before
  const int lc = lane / p, lj = lane - lc * p;
  const bool own = lane < RX && lc < ncell;
  const int o_own = lc * CS + lj;
  // x faces, compact: lane = (row ly, face fc = 1 .. ncell); the face is node
  // p of cell fc - 1 and, but for the last one, node 0 of cell fc
  constexpr int NF = NCX, FIT = (N * NF + 31) / 32;  // face items per lane
  const unsigned dxu = static_cast<unsigned>(dx);
  const unsigned w_u32 = static_cast<unsigned>(__cvta_generic_to_shared(W));
  // per-lane invariants: shared-memory byte offset and lattice offset of the
  // lane's own node (row ly = 0) and of its face item(s)
  const unsigned own_sm = 8u * o_own;
  unsigned face_sm[FIT], face_gl[FIT], face_to[FIT];
  bool face_ok[FIT], face_in[FIT];
#pragma unroll
  for (int k = 0; k < FIT; ++k) {
    const int l = lane + 32 * k, fy = l / NF, fc = 1 + l - fy * NF;
    face_ok[k] = l < N * NF;
    face_in[k] = face_ok[k] && fc < ncell;
    face_sm[k] = 8u * ((fc - 1) * CS + fy * N + p);  // node p of cell fc - 1
    face_to[k] = 8u * (fc * CS + fy * N);            // node 0 of cell fc
    face_gl[k] = fy * dxu + fc * p;
  }
  for (int pr = warp; pr < NTF * N; pr += C::T / 32) {
    const int f = pr / N, lz = pr - f * N;
    const double* src = rs + f * P.n_space + lz * dxy;
    const unsigned d0 = w_u32 + 8u * (pr * N * N);
    if (own) {
#pragma unroll
      for (int ly = 0; ly < N; ++ly) cp8_off(d0 + own_sm + 8u * (ly * N), src, ly * dxu + lane);
    }
#pragma unroll
    for (int k = 0; k < FIT; ++k)
      if (face_ok[k]) cp8_off(d0 + face_sm[k], src, face_gl[k]);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  const double(&Sx)[kMaxN][kMaxN] = P.S1[0][0];
  const double(&Sy)[kMaxN][kMaxN] = P.S1[1][0];
  const double(&Sz)[kMaxN][kMaxN] = P.S1[2][0];
  // ---- P1: plane owner, S_x^T then S_y^T in registers
  const int pc = t / C::NP, pf = (t % C::NP) / N, pz = t % N;
  const bool pact = pc < ncell;
  double* wpl = W + pc * CS + pf * ND + pz * N * N;  // this thread's plane
  if (pact) {
    double a[N][N];
#pragma unroll
    for (int y = 0; y < N; ++y) {
      double v[N];
#pragma unroll
      for (int x = 0; x < N; ++x) v[x] = wpl[y * N + x];
      fdm_fwd<N, true>(Sx, v, a[y]);
    }
#pragma unroll
    for (int ex = 0; ex < N; ++ex) {
      double v[N], o[N];
#pragma unroll
      for (int y = 0; y < N; ++y) v[y] = a[y][ex];
      fdm_fwd<N, true>(Sy, v, o);
#pragma unroll
      for (int ey = 0; ey < N; ++ey) wpl[ey * N + ex] = o[ey];
    }
  }
  __syncthreads();
  // ---- P2: eigen-line owner along z
  {
    const int c = t / C::NL, e = t % C::NL;
    if (c < ncell && !skipped(c)) {
      const int ey = e / N, ex = e % N;
      const double rho = rho_of(c);
      const double lxy = P.L1[0][0][ex] + P.L1[1][0][ey];
#pragma unroll
      for (int g = 0; g < SG; ++g) {
        double* wl = W + c * CS + g * NT * ND + e;  // the NT fields of step slot g
        double v[NT][N];
#pragma unroll
        for (int f = 0; f < NT; ++f) {
          double in[N];
#pragma unroll
          for (int k = 0; k < N; ++k) in[k] = wl[f * ND + k * N * N];
          fdm_fwd<N, true>(Sz, in, v[f]);
        }
        if constexpr (TD) {
          double mu[N];
#pragma unroll
          for (int ez = 0; ez < N; ++ez) mu[ez] = rho * (lxy + P.L1[2][0][ez]);
          temporal_solve_line<N, NT>(P, mu, v);
        } else {
#pragma unroll
          for (int ez = 0; ez < N; ++ez) {
            double bb[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int f = 0; f < NT; ++f) bb[f] = v[f][ez];
            temporal_solve<NT, TD>(P, rho * (lxy + P.L1[2][0][ez]), bb);
#pragma unroll
            for (int f = 0; f < NT; ++f) v[f][ez] = bb[f];
          }
        }
#pragma unroll
        for (int f = 0; f < NT; ++f) {
          double out[N];
          fdm_bwd<N, true>(Sz, v[f], out);
#pragma unroll
          for (int k = 0; k < N; ++k) wl[f * ND + k * N * N] = out[k];
        }
      }
    }
  }
  __syncthreads();
  // ---- P3: plane owner, S_y then S_x, weights; block assembly
  if (pact) {
    double a[N][N];
#pragma unroll
    for (int ex = 0; ex < N; ++ex) {
      double v[N], o[N];
#pragma unroll
      for (int ey = 0; ey < N; ++ey) v[ey] = wpl[ey * N + ex];
      fdm_bwd<N, true>(Sy, v, o);
#pragma unroll
      for (int y = 0; y < N; ++y) a[y][ex] = o[y];
    }
    // a cell solved by the exact kernel contributes nothing here
    const double wz = skipped(pc) ? 0.0 : scale * (pz == 0 || pz == p ? 0.5 : 1.0);
#pragma unroll
    for (int y = 0; y < N; ++y) {
      double o[N];
      fdm_bwd<N, true>(Sx, a[y], o);
      const double wzy = wz * (y == 0 || y == p ? 0.5 : 1.0);
#pragma unroll
      for (int x = 0; x < N; ++x) wpl[y * N + x] = (x == 0 || x == p ? 0.5 : 1.0) * wzy * o[x];
    }
  }
  __syncthreads();
  // ---- scatter: the faces first take the contribution of the cell before
  // (same warp, same (field, z) pair), then one row (f, lz, ly) of the strip
  // per warp instruction
  const bool last = lane == p * ncell;  // the strip's last node: node p of the last cell
  const unsigned row_sm = last ? 8u * ((ncell - 1) * CS + p) : own_sm;
  for (int pr = warp; pr < NTF * N; pr += C::T / 32) {
    const int f = pr / N, lz = pr - f * N;
    char* w0 = reinterpret_cast<char*>(W + pr * N * N);
#pragma unroll
    for (int k = 0; k < FIT; ++k)
      if (face_in[k])
        *reinterpret_cast<double*>(w0 + face_to[k]) += *reinterpret_cast<const double*>(w0 + face_sm[k]);
    __syncwarp();
    if (own || last) {
      double* dst = zs + f * P.n_space + lz * dxy;
#pragma unroll
      for (int ly = 0; ly < N; ++ly)
        red_off(dst, ly * dxu + lane, *reinterpret_cast<const double*>(w0 + row_sm + 8u * (ly * N)));
    }
  }
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
      // steps per CTA: the largest divisor of S with n_t * SG <= 4 fields
      auto strips = [&](auto sgc) {
        constexpr int SG = decltype(sgc)::value;
        using SC = SCfg<N, NT * SG>;
        static bool configured = false;
        if (!configured) {
          cudaFuncSetAttribute(fdm_strip_kernel<N, NT, SG, TD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(SC::smem_bytes()));
          configured = true;
        }
        const long long sxn = strips_per_row<N, NT * SG>(P.cells[0]);
        const dim3 sgrid(static_cast<unsigned>(sxn * P.cells[1] * P.cells[2]), static_cast<unsigned>(P.S / SG));
        if (sxn > 0) fdm_strip_kernel<N, NT, SG, TD><<<sgrid, SC::T, SC::smem_bytes(), s>>>(P, r, z, scale);
      };
      const int sg = fdm_fields_per_cta(NT, P.S) / NT;
      if constexpr (NT == 1) {
        if (sg == 4) strips(std::integral_constant<int, 4>{});
        else if (sg == 2) strips(std::integral_constant<int, 2>{});
        else strips(std::integral_constant<int, 1>{});
      } else if constexpr (NT == 2) {
        if (sg == 2) strips(std::integral_constant<int, 2>{});
        else strips(std::integral_constant<int, 1>{});
      } else {
        strips(std::integral_constant<int, 1>{});
      }
      const dim3 lgrid(static_cast<unsigned>((P.n_left + NC - 1) / NC), grid.y);
      if (P.n_left > 0) fdm_lines_kernel<N, NT, TD, 3><<<lgrid, 128, 0, s>>>(P, r, z, scale);
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

namespace {
template <int N, int NT>
std::vector<long long> left_out_cells(const DevFDM& P, const unsigned char* skip) {
  std::vector<long long> out;
  const unsigned nx = static_cast<unsigned>(P.cells[0]), ny = static_cast<unsigned>(P.cells[1]),
                 nz = static_cast<unsigned>(P.cells[2]);
  for (unsigned cz = 0; cz < nz; ++cz)
    for (unsigned cy = 0; cy < ny; ++cy)
      for (unsigned cx = 0; cx < nx; ++cx) {
        const long long cell = (static_cast<long long>(cz) * ny + cy) * nx + cx;
        if (skip && skip[cell]) continue;
        if (strip_left_out<N, NT>(P, skip, cx, cy, cz)) out.push_back(cell);
      }
  return out;
}
template <int N>
std::vector<long long> left_out_cells_nt(const DevFDM& P, const unsigned char* skip) {
  switch (fdm_fields_per_cta(P.nt, P.S)) {  // the strip geometry follows the fields per CTA
    case 1: return left_out_cells<N, 1>(P, skip);
    case 2: return left_out_cells<N, 2>(P, skip);
    case 3: return left_out_cells<N, 3>(P, skip);
    case 4: return left_out_cells<N, 4>(P, skip);
    default: throw std::invalid_argument("FDM smoother: n_t must be in [1, 4]");
  }
}
}  // namespace

std::vector<long long> fdm_left_out_cells(const DevFDM& P, const unsigned char* skip_host) {
  if (P.dim != 3) return {};
  switch (P.n) {
    case 2: return left_out_cells_nt<2>(P, skip_host);
    case 3: return left_out_cells_nt<3>(P, skip_host);
    case 4: return left_out_cells_nt<4>(P, skip_host);
    case 5: return left_out_cells_nt<5>(P, skip_host);
    default: throw std::invalid_argument("FDM smoother: unsupported p");
  }
}

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
