// 3D fused space-time operator, line-owner formulation (reference:
// SpaceTimeOperator::apply, space_time_operator.cpp:45-130, over
// SpatialOperator::apply_cells, spatial_operator.cpp:187-315).
//
// A CTA of 128 threads owns NC cells; thread (c, a, b) owns lattice line
// (a, b) of cell c along whichever axis the current stage sweeps, for ALL F
// temporal fields, with the line held in registers. Sweeps along the owned
// axis are register-only; the axis changes through shared memory. Sweep
// order (B = nodal->Gauss interpolation, D = nodal derivative at the Gauss
// points, both q x n; every forward sweep reads a nodal or partially
// interpolated line once and produces all outputs that need it):
//   A  y-owner: gather u along y (Dirichlet inputs zeroed), T = B_y u,
//               T' = D_y u
//   B  x-owner: U = B_x T, Ux = D_x T, Uy = B_x T', then the temporal block
//               coupling (CM, CA; space_time_operator.cpp:269-317) mixes the
//               fields: UM_i = sum_j CM_ij U_j, UA/UAx/UAy_i = sum_j CA_ij (.)_j
//               -- it commutes with the remaining z sweep, so stage C is
//               field-local
//   C  z-owner: V = B_z UM, Gx = B_z UAx, Gy = B_z UAy, Gz = D_z UA at the q
//               points of its z-line; V' = w|J| V, G' = rho w |J| J^-1 J^-T G
//               with J from the cell's d-linear map (spatial_operator.cpp:
//               152-183), cached per z-line and reused by every field; back:
//               P1 = B_z^T V' + D_z^T Gz', P2 = B_z^T Gx', P3 = B_z^T Gy'
//   D  x-owner: R1 = B_x^T P1 + D_x^T P2, R3 = B_x^T P3
//   E  y-owner: Y = B_y^T R1 + D_y^T R3, scatter-add (Dirichlet rows skipped;
//               the boundary pass writes them, space_time_operator.cpp:125-129)
// Four CTA barriers per batch, about 20 shared-memory accesses per point and
// field (the one-thread-per-line-per-sweep form needs ~37), and no index
// decoding inside the stages: every thread's line offsets are computed once.
#pragma once

#include <cuda_runtime.h>

#include "device.cuh"

namespace stmgb {
namespace stl {

constexpr int kT = 128;

// padded cell array layout x + RY y + PZ z (bank-conflict search over the
// three line orientations, 64-bit accesses, cells packed NL lines apart)
template <int N>
struct Lay;
template <>
struct Lay<2> {
  static constexpr int RY = 2, PZ = 5, SD = 10;
};
template <>
struct Lay<3> {
  static constexpr int RY = 3, PZ = 10, SD = 30;
};
template <>
struct Lay<4> {
  static constexpr int RY = 4, PZ = 19, SD = 74;
};
template <>
struct Lay<5> {
  static constexpr int RY = 5, PZ = 26, SD = 130;
};

template <int N, int F>
struct Cfg {
  static constexpr int NL = N * N;
  static constexpr int NC = (kT / NL) > 0 ? (kT / NL) : 1;
  static constexpr int SD = Lay<N>::SD;
  static constexpr int ARR = NC * F * SD;  // doubles per array
  static constexpr size_t smem_bytes() {
    return sizeof(double) * (4 * static_cast<size_t>(ARR) + NC * 25);
  }
};

// the kernel fits when the stage-C registers (4N line inputs, 3N
// accumulators, 7N metric cache) stay below ~160 and 4 arrays fit in smem
template <int N, int F>
constexpr bool fits() {
  return N * F <= 16 && Cfg<N, F>::smem_bytes() <= 100 * 1024;
}

template <int N>
constexpr int lines_min_blocks() {
  return N <= 3 ? 4 : 3;
}
template <int N, int F, bool CART>
__global__ void __launch_bounds__(kT, lines_min_blocks<N>()) st_lines_kernel(const __grid_constant__ DevLevel L,
                                                         const double* __restrict__ u, double* __restrict__ y,
                                                         double sign) {
  using C = Cfg<N, F>;
  constexpr int NL = C::NL, NC = C::NC, SD = C::SD, ARR = C::ARR;
  constexpr int RY = Lay<N>::RY, PZ = Lay<N>::PZ;
  extern __shared__ __align__(16) double smem[];
  double* A0 = smem;
  double* A1 = A0 + ARR;
  double* A2 = A1 + ARR;
  double* A3 = A2 + ARR;
  double* vtx = A3 + ARR;      // [NC][8][3] cell vertices
  double* rho_s = vtx + NC * 24;  // [NC]

  const int t = threadIdx.x;
  const int c = t / NL, l = t - (t / NL) * NL;
  const int a = l % N, b = l / N;
  const bool active = c < NC;
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long cell = static_cast<long long>(blockIdx.x) * NC + c;
  const bool valid = active && cell < n_cells;
  const long long dx = L.dofs[0], dxy = L.dofs[0] * L.dofs[1];
  const int p = N - 1;
  long long base = 0;
  int mask = 0;
  double gin[F][N];  // this thread's y-line of every field, requested first
  if (valid) {
    const unsigned ci = static_cast<unsigned>(cell);
    const unsigned nx = static_cast<unsigned>(L.cells[0]), ny = static_cast<unsigned>(L.cells[1]);
    const unsigned cx = ci % nx, cy = (ci / nx) % ny, cz = ci / (nx * ny);
    base = static_cast<long long>(cz) * p * dxy + static_cast<long long>(cy) * p * dx + static_cast<long long>(cx) * p;
    mask = (cx == 0 ? 1 : 0) | (cx == nx - 1 ? 2 : 0) | (cy == 0 ? 4 : 0) | (cy == ny - 1 ? 8 : 0) |
           (cz == 0 && (L.zbc & 1) ? 16 : 0) | (cz == L.cells[2] - 1 && (L.zbc & 2) ? 32 : 0);
    // the gather is issued before the vertex / coefficient loads and their
    // shared-memory stores, so the two DRAM round trips overlap
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const bool dir = ((mask & 1) && a == 0) || ((mask & 2) && a == p) || ((mask & 4) && k == 0) ||
                         ((mask & 8) && k == p) || ((mask & 16) && b == 0) || ((mask & 32) && b == p);
        gin[f][k] = dir ? 0.0 : __ldg(u + f * L.n_space + base + b * dxy + k * dx + a);
      }
    if (L.verts) {
      const long long vx = L.cells[0] + 1, vy = L.cells[1] + 1;
      for (int s = l; s < 8; s += NL) {
        const long long i = cx + (s & 1), j = cy + ((s >> 1) & 1), k = cz + ((s >> 2) & 1);
        const double* v = L.verts + 3 * ((k * vy + j) * vx + i);
#pragma unroll
        for (int d = 0; d < 3; ++d) vtx[(c * 8 + s) * 3 + d] = v[d];
      }
    }
    if (l == 0) {
      double rho = 1.0;
      if (L.rho0) {
        const long long ax = cx >> L.rho_shift, ay = cy >> L.rho_shift, az = (cz + L.cz0) >> L.rho_shift;
        rho = L.rho0[(az * L.cells0[1] + ay) * L.cells0[0] + ax];
      }
      rho_s[c] = rho;
    }
  }
  // Dirichlet faces of lattice coordinate (lx, ly, lz) of this cell
  auto dirichlet = [&](int lx, int ly, int lz) {
    return ((mask & 1) && lx == 0) || ((mask & 2) && lx == p) || ((mask & 4) && ly == 0) ||
           ((mask & 8) && ly == p) || ((mask & 16) && lz == 0) || ((mask & 32) && lz == p);
  };
  const int cbase = c * F * SD;
  // smem offsets of the lines this thread owns (element i at + i * stride)
  const int oy = cbase + a + PZ * b;       // y-line (x = a, z = b), stride RY
  const int ox = cbase + RY * a + PZ * b;  // x-line (y = a, z = b), stride 1
  const int oz = cbase + a + RY * b;       // z-line (x = a, y = b), stride PZ

  // ---- A: y-owner gather, T = B_y u, T' = D_y u
  if (valid) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
#pragma unroll
      for (int q = 0; q < N; ++q) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          s0 = fma(L.B[q][k], gin[f][k], s0);
          s1 = fma(L.D[q][k], gin[f][k], s1);
        }
        A0[oy + f * SD + q * RY] = s0;
        A1[oy + f * SD + q * RY] = s1;
      }
    }
  }
  __syncthreads();

  // ---- B: x-owner, U = B_x T, Ux = D_x T, Uy = B_x T', temporal coupling
  if (valid) {
    double U[F][N], Ux[F][N], Uy[F][N];
#pragma unroll
    for (int f = 0; f < F; ++f) {
      double tt[N], tp[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        tt[k] = A0[ox + f * SD + k];
        tp[k] = A1[ox + f * SD + k];
      }
#pragma unroll
      for (int q = 0; q < N; ++q) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          s0 = fma(L.B[q][k], tt[k], s0);
          s1 = fma(L.D[q][k], tt[k], s1);
          s2 = fma(L.B[q][k], tp[k], s2);
        }
        U[f][q] = s0;
        Ux[f][q] = s1;
        Uy[f][q] = s2;
      }
    }
#pragma unroll
    for (int i = 0; i < F; ++i) {
#pragma unroll
      for (int q = 0; q < N; ++q) {
        double m = 0.0, ua = 0.0, ux = 0.0, uy = 0.0;
#pragma unroll
        for (int j = 0; j < F; ++j) {
          const double cm = L.CM[i * F + j], ca = L.CA[i * F + j];
          m = fma(cm, U[j][q], m);
          ua = fma(ca, U[j][q], ua);
          ux = fma(ca, Ux[j][q], ux);
          uy = fma(ca, Uy[j][q], uy);
        }
        A0[ox + i * SD + q] = m;
        A1[ox + i * SD + q] = ua;
        A2[ox + i * SD + q] = ux;
        A3[ox + i * SD + q] = uy;
      }
    }
  }
  __syncthreads();

  // ---- C: z-owner, quadrature-point work, back along z
  if (valid) {
    // metric at the N q-points (a, b, qz) of this z-line
    // metric at the N q-points of this z-line: Cartesian cells need only
    // three constants (diagonal J), d-linear cells a cached mf / K per point
    double mf[CART ? 1 : N], K[CART ? 1 : N][6];
    const double wxy = L.w[a] * L.w[b];
    const double rho = rho_s[c];
    const double detc = L.h[0] * L.h[1] * L.h[2];
    const double cm = wxy * detc, ck0 = rho * cm / (L.h[0] * L.h[0]), ck1 = rho * cm / (L.h[1] * L.h[1]),
                 ck2 = rho * cm / (L.h[2] * L.h[2]);
    if constexpr (!CART) {
      const double* X = vtx + c * 24;
      const double xx = L.xq[a], xy = L.xq[b];
      // J(:, 0) = A0 + xz B0, J(:, 1) = A1 + xz B1, J(:, 2) = const (d-linear map)
      double Ja0[3], Jb0[3], Ja1[3], Jb1[3], J2[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double x0 = X[0 * 3 + d], x1 = X[1 * 3 + d], x2 = X[2 * 3 + d], x3 = X[3 * 3 + d];
        const double x4 = X[4 * 3 + d], x5 = X[5 * 3 + d], x6 = X[6 * 3 + d], x7 = X[7 * 3 + d];
        const double c1 = x1 - x0, c2 = x2 - x0, c4 = x4 - x0;
        const double c3 = x3 - x2 - x1 + x0, c5 = x5 - x4 - x1 + x0, c6 = x6 - x4 - x2 + x0;
        const double c7 = x7 - x6 - x5 + x4 - x3 + x2 + x1 - x0;
        Ja0[d] = fma(c3, xy, c1);
        Jb0[d] = fma(c7, xy, c5);
        Ja1[d] = fma(c3, xx, c2);
        Jb1[d] = fma(c7, xx, c6);
        J2[d] = fma(xy, fma(c7, xx, c6), fma(c5, xx, c4));
      }
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const double xz = L.xq[q];
        double J[3][3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          J[d][0] = fma(xz, Jb0[d], Ja0[d]);
          J[d][1] = fma(xz, Jb1[d], Ja1[d]);
          J[d][2] = J2[d];
        }
        const double R00 = J[1][1] * J[2][2] - J[2][1] * J[1][2];
        const double R01 = J[2][1] * J[0][2] - J[0][1] * J[2][2];
        const double R02 = J[0][1] * J[1][2] - J[1][1] * J[0][2];
        const double R10 = J[1][2] * J[2][0] - J[2][2] * J[1][0];
        const double R11 = J[2][2] * J[0][0] - J[0][2] * J[2][0];
        const double R12 = J[0][2] * J[1][0] - J[1][2] * J[0][0];
        const double R20 = J[1][0] * J[2][1] - J[2][0] * J[1][1];
        const double R21 = J[2][0] * J[0][1] - J[0][0] * J[2][1];
        const double R22 = J[0][0] * J[1][1] - J[1][0] * J[0][1];
        const double det = J[0][0] * R00 + J[1][0] * R01 + J[2][0] * R02;
        const double wq = wxy * L.w[q];
        const double s = rho * wq / det;
        mf[q] = wq * det;
        K[q][0] = s * (R00 * R00 + R01 * R01 + R02 * R02);
        K[q][1] = s * (R00 * R10 + R01 * R11 + R02 * R12);
        K[q][2] = s * (R00 * R20 + R01 * R21 + R02 * R22);
        K[q][3] = s * (R10 * R10 + R11 * R11 + R12 * R12);
        K[q][4] = s * (R10 * R20 + R11 * R21 + R12 * R22);
        K[q][5] = s * (R20 * R20 + R21 * R21 + R22 * R22);
      }
    }
#pragma unroll
    for (int f = 0; f < F; ++f) {
      double um[N], ua[N], ux[N], uy[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        um[k] = A0[oz + f * SD + k * PZ];
        ua[k] = A1[oz + f * SD + k * PZ];
        ux[k] = A2[oz + f * SD + k * PZ];
        uy[k] = A3[oz + f * SD + k * PZ];
      }
      double P1[N], P2[N], P3[N];
#pragma unroll
      for (int k = 0; k < N; ++k) P1[k] = P2[k] = P3[k] = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        double v = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          v = fma(L.B[q][k], um[k], v);
          gx = fma(L.B[q][k], ux[k], gx);
          gy = fma(L.B[q][k], uy[k], gy);
          gz = fma(L.D[q][k], ua[k], gz);
        }
        double vo, ox_, oy_, oz_;
        if constexpr (CART) {
          const double wq = L.w[q];
          vo = cm * wq * v;
          ox_ = ck0 * wq * gx;
          oy_ = ck1 * wq * gy;
          oz_ = ck2 * wq * gz;
        } else {
          vo = mf[q] * v;
          ox_ = fma(K[q][0], gx, fma(K[q][1], gy, K[q][2] * gz));
          oy_ = fma(K[q][1], gx, fma(K[q][3], gy, K[q][4] * gz));
          oz_ = fma(K[q][2], gx, fma(K[q][4], gy, K[q][5] * gz));
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          P1[k] = fma(L.B[q][k], vo, fma(L.D[q][k], oz_, P1[k]));
          P2[k] = fma(L.B[q][k], ox_, P2[k]);
          P3[k] = fma(L.B[q][k], oy_, P3[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        A0[oz + f * SD + k * PZ] = P1[k];
        A1[oz + f * SD + k * PZ] = P2[k];
        A2[oz + f * SD + k * PZ] = P3[k];
      }
    }
  }
  __syncthreads();

  // ---- D: x-owner, R1 = B_x^T P1 + D_x^T P2, R3 = B_x^T P3
  if (valid) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      double p1[N], p2[N], p3[N];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        p1[q] = A0[ox + f * SD + q];
        p2[q] = A1[ox + f * SD + q];
        p3[q] = A2[ox + f * SD + q];
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double r1 = 0.0, r3 = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          r1 = fma(L.B[q][k], p1[q], fma(L.D[q][k], p2[q], r1));
          r3 = fma(L.B[q][k], p3[q], r3);
        }
        A0[ox + f * SD + k] = r1;
        A1[ox + f * SD + k] = r3;
      }
    }
  }
  __syncthreads();

  // ---- E: y-owner, Y = B_y^T R1 + D_y^T R3, scatter-add
  if (valid) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      double r1[N], r3[N];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        r1[q] = A0[oy + f * SD + q * RY];
        r3[q] = A1[oy + f * SD + q * RY];
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) s = fma(L.B[q][k], r1[q], fma(L.D[q][k], r3[q], s));
        if (!dirichlet(a, k, b)) atomicAdd(y + f * L.n_space + base + b * dxy + k * dx + a, sign * s);
      }
    }
  }
}

// Variant for N * F > 16 (C4: Q4 with 8 fields, C5: Q4 with 4): the temporal
// block coupling is applied to the NODAL lines in stage A (it commutes with
// every sweep), which makes stages B-E field-local, so the fields run in
// groups of G through a G-field shared-memory footprint:
//   A  y-owner: all F input lines in registers; per output field i of the
//      group uM_i = sum_j CM_ij u_j, uA_i = sum_j CA_ij u_j; T = B_y uM,
//      TA = B_y uA, TA' = D_y uA
//   B  x-owner: UM = B_x T, UA = B_x TA, UAx = D_x TA, UAy = B_x TA'
//   C, D, E as in st_lines_kernel (metric at the q-points, back sweeps,
//      scatter)
template <int N>
constexpr int mix_group() {
  return N >= 5 ? 2 : 4;
}
template <int N, int F>
struct MixCfg {
  static constexpr int NL = N * N;
  static constexpr int NC = (kT / NL) > 0 ? (kT / NL) : 1;
  static constexpr int G = mix_group<N>() < F ? mix_group<N>() : F;
  static constexpr int SD = Lay<N>::SD;
  static constexpr int ARR = NC * G * SD;
  static constexpr size_t smem_bytes() { return sizeof(double) * (4 * static_cast<size_t>(ARR) + NC * 25); }
};

template <int N, int F, bool CART>
__global__ void __launch_bounds__(kT, 3) st_mix_kernel(const __grid_constant__ DevLevel L,
                                                       const double* __restrict__ u, double* __restrict__ y,
                                                       double sign) {
  using C = MixCfg<N, F>;
  constexpr int NL = C::NL, NC = C::NC, SD = C::SD, ARR = C::ARR, G = C::G;
  constexpr int RY = Lay<N>::RY, PZ = Lay<N>::PZ;
  extern __shared__ __align__(16) double smem[];
  double* A0 = smem;
  double* A1 = A0 + ARR;
  double* A2 = A1 + ARR;
  double* A3 = A2 + ARR;
  double* vtx = A3 + ARR;
  double* rho_s = vtx + NC * 24;
  const int t = threadIdx.x;
  const int c = t / NL, l = t - (t / NL) * NL;
  const int a = l % N, b = l / N;
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long cell = static_cast<long long>(blockIdx.x) * NC + c;
  const bool valid = c < NC && cell < n_cells;
  const long long dx = L.dofs[0], dxy = L.dofs[0] * L.dofs[1];
  const int p = N - 1;
  long long base = 0;
  int mask = 0;
  if (valid) {
    const unsigned ci = static_cast<unsigned>(cell);
    const unsigned nx = static_cast<unsigned>(L.cells[0]), ny = static_cast<unsigned>(L.cells[1]);
    const unsigned cx = ci % nx, cy = (ci / nx) % ny, cz = ci / (nx * ny);
    base = static_cast<long long>(cz) * p * dxy + static_cast<long long>(cy) * p * dx + static_cast<long long>(cx) * p;
    mask = (cx == 0 ? 1 : 0) | (cx == nx - 1 ? 2 : 0) | (cy == 0 ? 4 : 0) | (cy == ny - 1 ? 8 : 0) |
           (cz == 0 && (L.zbc & 1) ? 16 : 0) | (cz == L.cells[2] - 1 && (L.zbc & 2) ? 32 : 0);
    if (L.verts) {
      const long long vx = L.cells[0] + 1, vy = L.cells[1] + 1;
      for (int sv = l; sv < 8; sv += NL) {
        const long long i = cx + (sv & 1), j = cy + ((sv >> 1) & 1), k = cz + ((sv >> 2) & 1);
        const double* v = L.verts + 3 * ((k * vy + j) * vx + i);
#pragma unroll
        for (int d = 0; d < 3; ++d) vtx[(c * 8 + sv) * 3 + d] = v[d];
      }
    }
    if (l == 0) {
      double rho = 1.0;
      if (L.rho0) {
        const long long ax = cx >> L.rho_shift, ay = cy >> L.rho_shift, az = (cz + L.cz0) >> L.rho_shift;
        rho = L.rho0[(az * L.cells0[1] + ay) * L.cells0[0] + ax];
      }
      rho_s[c] = rho;
    }
  }
  auto dirichlet = [&](int lx, int ly, int lz) {
    return ((mask & 1) && lx == 0) || ((mask & 2) && lx == p) || ((mask & 4) && ly == 0) ||
           ((mask & 8) && ly == p) || ((mask & 16) && lz == 0) || ((mask & 32) && lz == p);
  };
  const int cbase = c * G * SD;
  const int oy = cbase + a + PZ * b, ox = cbase + RY * a + PZ * b, oz = cbase + a + RY * b;

#pragma unroll 1
  for (int i0 = 0; i0 < F; i0 += G) {
    // ---- A: y-owner, nodal temporal coupling, T = B_y uM, TA = B_y uA, TA' = D_y uA
    if (valid) {
      double in[F][N];
#pragma unroll
      for (int j = 0; j < F; ++j)
#pragma unroll
        for (int k = 0; k < N; ++k)
          in[j][k] = dirichlet(a, k, b) ? 0.0 : __ldg(u + j * L.n_space + base + b * dxy + k * dx + a);
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        const int i = i0 + gi;
        if (i >= F) break;
        double um[N], ua[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double m = 0.0, aa = 0.0;
#pragma unroll
          for (int j = 0; j < F; ++j) {
            m = fma(L.CM[i * F + j], in[j][k], m);
            aa = fma(L.CA[i * F + j], in[j][k], aa);
          }
          um[k] = m;
          ua[k] = aa;
        }
#pragma unroll
        for (int q = 0; q < N; ++q) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            s0 = fma(L.B[q][k], um[k], s0);
            s1 = fma(L.B[q][k], ua[k], s1);
            s2 = fma(L.D[q][k], ua[k], s2);
          }
          A0[oy + gi * SD + q * RY] = s0;
          A1[oy + gi * SD + q * RY] = s1;
          A2[oy + gi * SD + q * RY] = s2;
        }
      }
    }
    __syncthreads();
    // ---- B: x-owner, UM = B_x T, UA = B_x TA, UAx = D_x TA, UAy = B_x TA'
    if (valid) {
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        if (i0 + gi >= F) break;
        double tm[N], ta[N], tp[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          tm[k] = A0[ox + gi * SD + k];
          ta[k] = A1[ox + gi * SD + k];
          tp[k] = A2[ox + gi * SD + k];
        }
#pragma unroll
        for (int q = 0; q < N; ++q) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            s0 = fma(L.B[q][k], tm[k], s0);
            s1 = fma(L.B[q][k], ta[k], s1);
            s2 = fma(L.D[q][k], ta[k], s2);
            s3 = fma(L.B[q][k], tp[k], s3);
          }
          A0[ox + gi * SD + q] = s0;
          A1[ox + gi * SD + q] = s1;
          A2[ox + gi * SD + q] = s2;
          A3[ox + gi * SD + q] = s3;
        }
      }
    }
    __syncthreads();
    // ---- C: z-owner, q-point metric (per z-line), field-local q-point work
    if (valid) {
      double mf[CART ? 1 : N], K[CART ? 1 : N][6];
      const double wxy = L.w[a] * L.w[b];
      const double rho = rho_s[c];
      const double detc = L.h[0] * L.h[1] * L.h[2];
      const double cm = wxy * detc, ck0 = rho * cm / (L.h[0] * L.h[0]), ck1 = rho * cm / (L.h[1] * L.h[1]),
                   ck2 = rho * cm / (L.h[2] * L.h[2]);
      if constexpr (!CART) {
        const double* X = vtx + c * 24;
        const double xx = L.xq[a], xy = L.xq[b];
        double Ja0[3], Jb0[3], Ja1[3], Jb1[3], J2[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double x0 = X[0 * 3 + d], x1 = X[1 * 3 + d], x2 = X[2 * 3 + d], x3 = X[3 * 3 + d];
          const double x4 = X[4 * 3 + d], x5 = X[5 * 3 + d], x6 = X[6 * 3 + d], x7 = X[7 * 3 + d];
          const double c1 = x1 - x0, c2 = x2 - x0, c4 = x4 - x0;
          const double c3 = x3 - x2 - x1 + x0, c5 = x5 - x4 - x1 + x0, c6 = x6 - x4 - x2 + x0;
          const double c7 = x7 - x6 - x5 + x4 - x3 + x2 + x1 - x0;
          Ja0[d] = fma(c3, xy, c1);
          Jb0[d] = fma(c7, xy, c5);
          Ja1[d] = fma(c3, xx, c2);
          Jb1[d] = fma(c7, xx, c6);
          J2[d] = fma(xy, fma(c7, xx, c6), fma(c5, xx, c4));
        }
#pragma unroll
        for (int q = 0; q < N; ++q) {
          const double xz = L.xq[q];
          double J[3][3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            J[d][0] = fma(xz, Jb0[d], Ja0[d]);
            J[d][1] = fma(xz, Jb1[d], Ja1[d]);
            J[d][2] = J2[d];
          }
          const double R00 = J[1][1] * J[2][2] - J[2][1] * J[1][2];
          const double R01 = J[2][1] * J[0][2] - J[0][1] * J[2][2];
          const double R02 = J[0][1] * J[1][2] - J[1][1] * J[0][2];
          const double R10 = J[1][2] * J[2][0] - J[2][2] * J[1][0];
          const double R11 = J[2][2] * J[0][0] - J[0][2] * J[2][0];
          const double R12 = J[0][2] * J[1][0] - J[1][2] * J[0][0];
          const double R20 = J[1][0] * J[2][1] - J[2][0] * J[1][1];
          const double R21 = J[2][0] * J[0][1] - J[0][0] * J[2][1];
          const double R22 = J[0][0] * J[1][1] - J[1][0] * J[0][1];
          const double det = J[0][0] * R00 + J[1][0] * R01 + J[2][0] * R02;
          const double wq = wxy * L.w[q];
          const double s = rho * wq / det;
          mf[q] = wq * det;
          K[q][0] = s * (R00 * R00 + R01 * R01 + R02 * R02);
          K[q][1] = s * (R00 * R10 + R01 * R11 + R02 * R12);
          K[q][2] = s * (R00 * R20 + R01 * R21 + R02 * R22);
          K[q][3] = s * (R10 * R10 + R11 * R11 + R12 * R12);
          K[q][4] = s * (R10 * R20 + R11 * R21 + R12 * R22);
          K[q][5] = s * (R20 * R20 + R21 * R21 + R22 * R22);
        }
      }
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        if (i0 + gi >= F) break;
        double um[N], ua[N], ux[N], uy[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          um[k] = A0[oz + gi * SD + k * PZ];
          ua[k] = A1[oz + gi * SD + k * PZ];
          ux[k] = A2[oz + gi * SD + k * PZ];
          uy[k] = A3[oz + gi * SD + k * PZ];
        }
        double P1[N], P2[N], P3[N];
#pragma unroll
        for (int k = 0; k < N; ++k) P1[k] = P2[k] = P3[k] = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          double v = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            v = fma(L.B[q][k], um[k], v);
            gx = fma(L.B[q][k], ux[k], gx);
            gy = fma(L.B[q][k], uy[k], gy);
            gz = fma(L.D[q][k], ua[k], gz);
          }
          double vo, ox_, oy_, oz_;
          if constexpr (CART) {
            const double wq = L.w[q];
            vo = cm * wq * v;
            ox_ = ck0 * wq * gx;
            oy_ = ck1 * wq * gy;
            oz_ = ck2 * wq * gz;
          } else {
            vo = mf[q] * v;
            ox_ = fma(K[q][0], gx, fma(K[q][1], gy, K[q][2] * gz));
            oy_ = fma(K[q][1], gx, fma(K[q][3], gy, K[q][4] * gz));
            oz_ = fma(K[q][2], gx, fma(K[q][4], gy, K[q][5] * gz));
          }
#pragma unroll
          for (int k = 0; k < N; ++k) {
            P1[k] = fma(L.B[q][k], vo, fma(L.D[q][k], oz_, P1[k]));
            P2[k] = fma(L.B[q][k], ox_, P2[k]);
            P3[k] = fma(L.B[q][k], oy_, P3[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          A0[oz + gi * SD + k * PZ] = P1[k];
          A1[oz + gi * SD + k * PZ] = P2[k];
          A2[oz + gi * SD + k * PZ] = P3[k];
        }
      }
    }
    __syncthreads();
    // ---- D: x-owner, R1 = B_x^T P1 + D_x^T P2, R3 = B_x^T P3
    if (valid) {
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        if (i0 + gi >= F) break;
        double p1[N], p2[N], p3[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
          p1[q] = A0[ox + gi * SD + q];
          p2[q] = A1[ox + gi * SD + q];
          p3[q] = A2[ox + gi * SD + q];
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double r1 = 0.0, r3 = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) {
            r1 = fma(L.B[q][k], p1[q], fma(L.D[q][k], p2[q], r1));
            r3 = fma(L.B[q][k], p3[q], r3);
          }
          A0[ox + gi * SD + k] = r1;
          A1[ox + gi * SD + k] = r3;
        }
      }
    }
    __syncthreads();
    // ---- E: y-owner, Y = B_y^T R1 + D_y^T R3, scatter-add
    if (valid) {
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        const int i = i0 + gi;
        if (i >= F) break;
        double r1[N], r3[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
          r1[q] = A0[oy + gi * SD + q * RY];
          r3[q] = A1[oy + gi * SD + q * RY];
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double sacc = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) sacc = fma(L.B[q][k], r1[q], fma(L.D[q][k], r3[q], sacc));
          if (!dirichlet(a, k, b)) atomicAdd(y + i * L.n_space + base + b * dxy + k * dx + a, sign * sacc);
        }
      }
    }
  }
}

template <int N, int F, bool CART>
void launch_mix_c(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t stream) {
  using C = MixCfg<N, F>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(st_mix_kernel<N, F, CART>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(C::smem_bytes()));
    cudaFuncSetAttribute(st_mix_kernel<N, F, CART>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    configured = true;
  }
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long blocks = (n_cells + C::NC - 1) / C::NC;
  st_mix_kernel<N, F, CART><<<static_cast<unsigned>(blocks), kT, C::smem_bytes(), stream>>>(L, u, y, sign);
}
template <int N, int F>
void launch_mix(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t stream) {
  if (L.verts)
    launch_mix_c<N, F, false>(L, u, y, sign, stream);
  else
    launch_mix_c<N, F, true>(L, u, y, sign, stream);
}

template <int N, int F, bool CART>
void launch_c(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t stream) {
  using C = Cfg<N, F>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(st_lines_kernel<N, F, CART>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(C::smem_bytes()));
    cudaFuncSetAttribute(st_lines_kernel<N, F, CART>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    configured = true;
  }
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long blocks = (n_cells + C::NC - 1) / C::NC;
  st_lines_kernel<N, F, CART><<<static_cast<unsigned>(blocks), kT, C::smem_bytes(), stream>>>(L, u, y, sign);
}
template <int N, int F>
void launch(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t stream) {
  if (L.verts)
    launch_c<N, F, false>(L, u, y, sign, stream);
  else
    launch_c<N, F, true>(L, u, y, sign, stream);
}

}  // namespace stl
}  // namespace stmgb
