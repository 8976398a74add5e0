// 3D fused space-time operator on Cartesian levels (axis-aligned cells of
// one size h, the lattice every level of C3/C4/C5 lives on): the same
// y = sum_j CM_ij M u_j + CA_ij A u_j as st_lines.cuh (reference:
// SpaceTimeOperator::apply, space_time_operator.cpp:45-130, over
// SpatialOperator::apply_cells, spatial_operator.cpp:187-315), but applied
// with the 1D ELEMENT matrices instead of through the quadrature points.
//
// On an affine box cell the reference's Gauss quadrature (q = p + 1 points,
// exact for the degree-2p integrands) of the cell mass and stiffness factors
// into Kronecker products of the [0,1] interval matrices
//   Mr = B^T W B,  Kr = D^T W D     ((p+1) x (p+1), symmetric),
//   M_e = V Mr(x)Mr(x)Mr,  A_e = rho V (Kr/hx^2 (x) Mr (x) Mr + Mr (x) Kr/hy^2 (x) Mr
//                                      + Mr (x) Mr (x) Kr/hz^2),  V = hx hy hz,
// so a cell needs 7 line sweeps per field (the quadrature form needs 18):
//   A  y-owner: gather u along y (Dirichlet inputs zeroed), a = Mr_y u,
//               b = Kr_y u
//   B  x-owner: c = Mr_x a, pre = Kr_x a / hx^2 + Mr_x b / hy^2
//   C  z-owner: temporal block coupling of the z-lines of every field,
//               Zm_i = V sum_j (CM_ij c_j + CA_ij rho pre_j),
//               Zk_i = rho V / hz^2 sum_j CA_ij c_j,
//               y_i = Mr_z Zm_i + Kr_z Zk_i, scatter-add (Dirichlet rows
//               skipped; the boundary pass writes them,
//               space_time_operator.cpp:125-129)
// Two shared arrays. Their padded layouts come from a bank-conflict model of
// the three line orientations (scripts/gen_cart_layout.py ->
// st_cart_layout.h): where one layout cannot serve all three, stage B reads
// layout 1 and, after a third barrier, writes layout 2. Wide field counts
// (N * F > 20) split each line's fields over two thread groups in stages A
// and B; in stage C each group produces half of the output fields.
#pragma once

#include <cuda_runtime.h>

#include "device.cuh"
#include "st_cart_layout.h"

namespace stmgb {
namespace stc {

// Even-odd (centro-symmetric) line products: v -> (e, o) with
// e[k] = v[k] + v[n-1-k], o[k] = v[k] - v[n-1-k] (k < n/2), e[n/2] = v[n/2]
// for odd n; then A v = (E e + O o, mirrored: (E e - O o) on the upper half).
// N = 5: 13 FMAs per product instead of 25, and 26 distinct table values
// (both matrices) that stay in uniform registers.
template <int N>
struct EO {
  static constexpr int H = N / 2, HE = (N + 1) / 2;
};
template <int N>
__device__ __forceinline__ void eo_split(const double (&v)[N], double (&e)[EO<N>::HE], double (&o)[EO<N>::H]) {
#pragma unroll
  for (int k = 0; k < EO<N>::H; ++k) {
    e[k] = v[k] + v[N - 1 - k];
    o[k] = v[k] - v[N - 1 - k];
  }
  if constexpr (N % 2 == 1) e[EO<N>::H] = v[EO<N>::H];
}
// E-part / O-part of one matrix applied to a split vector
template <int N>
__device__ __forceinline__ void eo_even(const double (&E)[3][3], const double (&e)[EO<N>::HE], double (&se)[EO<N>::HE]) {
#pragma unroll
  for (int i = 0; i < EO<N>::HE; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < EO<N>::HE; ++k) s = fma(E[i][k], e[k], s);
    se[i] = s;
  }
}
template <int N>
__device__ __forceinline__ void eo_odd(const double (&O)[2][2], const double (&o)[EO<N>::H], double (&so)[EO<N>::H > 0 ? EO<N>::H : 1]) {
#pragma unroll
  for (int i = 0; i < EO<N>::H; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < EO<N>::H; ++k) s = fma(O[i][k], o[k], s);
    so[i] = s;
  }
}
template <int N>
__device__ __forceinline__ void eo_merge(const double (&se)[EO<N>::HE], const double (&so)[EO<N>::H], double (&out)[N]) {
#pragma unroll
  for (int i = 0; i < EO<N>::H; ++i) {
    out[i] = se[i] + so[i];
    out[N - 1 - i] = se[i] - so[i];
  }
  if constexpr (N % 2 == 1) out[EO<N>::H] = se[EO<N>::H];
}

template <int N, int F>
struct Cfg {
  static constexpr int NL = N * N;
  static constexpr int FG = (N * F > 20) ? 2 : 1;  // thread groups per line
  static constexpr int FPG = (F + FG - 1) / FG;    // fields per group
  static constexpr int NC = (128 / NL) > 0 ? (128 / NL) : 1;
  static constexpr int T = ((NC * NL * FG + 31) / 32) * 32;
  static constexpr int MINB = FG == 1 ? 4 : 2;
  using Lay = Layout<N, F>;
  // one buffer per array, holding layout 1 (stage A -> B) and then layout 2
  // (stage B -> C)
  static constexpr int ARR = NC * (Lay::CS1 > Lay::CS2 ? Lay::CS1 : Lay::CS2);
  static constexpr size_t smem_bytes() { return sizeof(double) * 2 * static_cast<size_t>(ARR); }
};

template <int N, int F>
__global__ void __launch_bounds__(Cfg<N, F>::T, Cfg<N, F>::MINB)
    st_cart_kernel(const __grid_constant__ DevLevel L, const double* __restrict__ u, double* __restrict__ y,
                   double sign) {
  using C = Cfg<N, F>;
  using Y = typename C::Lay;
  constexpr int NL = C::NL, NC = C::NC, ARR = C::ARR, FPG = C::FPG;
  extern __shared__ __align__(16) double smem[];
  double* A0 = smem;
  double* A1 = A0 + ARR;

  const int t = threadIdx.x;
  const int g = t / (NC * NL);
  const int r = t - g * (NC * NL);
  const int c = r / NL, l = r - (r / NL) * NL;
  const int a = l % N, b = l / N;
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long cell = static_cast<long long>(blockIdx.x) * NC + c;
  const bool valid = g < C::FG && cell < n_cells;
  const int j0 = g * FPG;  // first field of this thread's group
  const long long dx = L.dofs[0], dxy = L.dofs[0] * L.dofs[1], ns = L.n_space;
  const int p = N - 1;
  long long base = 0;
  int mask = 0;
  unsigned cx = 0, cy = 0, cz = 0;
  double gin[FPG][N];
  if (valid) {
    const unsigned ci = static_cast<unsigned>(cell);
    const unsigned nx = static_cast<unsigned>(L.cells[0]), ny = static_cast<unsigned>(L.cells[1]);
    cx = ci % nx;
    cy = (ci / nx) % ny;
    cz = ci / (nx * ny);
    base = static_cast<long long>(cz) * p * dxy + static_cast<long long>(cy) * p * dx + static_cast<long long>(cx) * p;
    mask = (cx == 0 ? 1 : 0) | (cx == nx - 1 ? 2 : 0) | (cy == 0 ? 4 : 0) | (cy == ny - 1 ? 8 : 0) |
           (cz == 0 && (L.zbc & 1) ? 16 : 0) | (cz == L.cells[2] - 1 && (L.zbc & 2) ? 32 : 0);
#pragma unroll
    for (int jj = 0; jj < FPG; ++jj)
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const bool dir = ((mask & 1) && a == 0) || ((mask & 2) && a == p) || ((mask & 4) && k == 0) ||
                         ((mask & 8) && k == p) || ((mask & 16) && b == 0) || ((mask & 32) && b == p);
        gin[jj][k] = (dir || j0 + jj >= F) ? 0.0 : __ldg(u + (j0 + jj) * ns + base + b * dxy + k * dx + a);
      }
  }
  // stage A: y-line (x = a, z = b) of layout 1; stage B: x-line (y, z) =
  // (a, b), or (b, a) when the layout swaps, read from layout 1 and written to
  // layout 2; stage C: z-line (x = a, y = b) of layout 2
  const int oy = c * Y::CS1 + a + Y::PZ1 * b;
  const int by = Y::SWAP ? b : a, bz = Y::SWAP ? a : b;
  const int ox1 = c * Y::CS1 + Y::RY1 * by + Y::PZ1 * bz;
  const int ox2 = c * Y::CS2 + Y::RY2 * by + Y::PZ2 * bz;
  const int oz = c * Y::CS2 + a + Y::RY2 * b;

  // ---- A: y-owner, a = Mr_y u, b = Kr_y u
  if (valid) {
#pragma unroll
    for (int jj = 0; jj < FPG; ++jj) {
      if (j0 + jj >= F) break;
      const int o = oy + (j0 + jj) * Y::SD1;
      double e[EO<N>::HE], od[EO<N>::H], se[EO<N>::HE], so[EO<N>::H], ra[N], rb[N];
      eo_split<N>(gin[jj], e, od);
      eo_even<N>(L.MrE, e, se);
      eo_odd<N>(L.MrO, od, so);
      eo_merge<N>(se, so, ra);
      eo_even<N>(L.KrE, e, se);
      eo_odd<N>(L.KrO, od, so);
      eo_merge<N>(se, so, rb);
#pragma unroll
      for (int q = 0; q < N; ++q) {
        A0[o + q * Y::RY1] = ra[q];
        A1[o + q * Y::RY1] = rb[q];
      }
    }
  }
  __syncthreads();

  // ---- B: x-owner, c = Mr_x a, pre = Kr_x a / hx^2 + Mr_x b / hy^2
  {
    double vc[FPG][N], vp[FPG][N];
    if (valid) {
      const double sx = L.hinv2[0], sy = L.hinv2[1];
#pragma unroll
      for (int jj = 0; jj < FPG; ++jj) {
        if (j0 + jj >= F) break;
        const int o = ox1 + (j0 + jj) * Y::SD1;
        double va[N], vb[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          va[k] = A0[o + k];
          vb[k] = A1[o + k];
        }
        double ea[EO<N>::HE], oa[EO<N>::H], eb[EO<N>::HE], ob[EO<N>::H];
        eo_split<N>(va, ea, oa);
        eo_split<N>(vb, eb, ob);
        double se[EO<N>::HE], so[EO<N>::H], te[EO<N>::HE], to[EO<N>::H];
        eo_even<N>(L.MrE, ea, se);
        eo_odd<N>(L.MrO, oa, so);
        eo_merge<N>(se, so, vc[jj]);
        eo_even<N>(L.KrE, ea, se);
        eo_odd<N>(L.KrO, oa, so);
        eo_even<N>(L.MrE, eb, te);
        eo_odd<N>(L.MrO, ob, to);
#pragma unroll
        for (int i = 0; i < EO<N>::HE; ++i) se[i] = fma(sx, se[i], sy * te[i]);
#pragma unroll
        for (int i = 0; i < EO<N>::H; ++i) so[i] = fma(sx, so[i], sy * to[i]);
        eo_merge<N>(se, so, vp[jj]);
        if constexpr (!Y::SPLIT) {  // in place: this thread owns the line
#pragma unroll
          for (int q = 0; q < N; ++q) {
            A0[o + q] = vc[jj][q];
            A1[o + q] = vp[jj][q];
          }
        }
      }
    }
    if constexpr (Y::SPLIT) {
      __syncthreads();
      if (valid) {
#pragma unroll
        for (int jj = 0; jj < FPG; ++jj) {
          if (j0 + jj >= F) break;
          const int o = ox2 + (j0 + jj) * Y::SD2;
#pragma unroll
          for (int q = 0; q < N; ++q) {
            A0[o + q] = vc[jj][q];
            A1[o + q] = vp[jj][q];
          }
        }
      }
    }
  }
  __syncthreads();

  // ---- C: z-owner, temporal coupling, Mr_z / Kr_z, scatter-add
  if (valid) {
    const double V = L.h[0] * L.h[1] * L.h[2];
    double rho = 1.0;
    if (L.rho0) {
      const long long ax = cx >> L.rho_shift, ay = cy >> L.rho_shift, az = (cz + L.cz0) >> L.rho_shift;
      rho = __ldg(L.rho0 + (az * L.cells0[1] + ay) * L.cells0[0] + ax);
    }
    const double rvz = rho * V * L.hinv2[2];
    double Zm[FPG][N], Zk[FPG][N];
#pragma unroll
    for (int ii = 0; ii < FPG; ++ii)
#pragma unroll
      for (int k = 0; k < N; ++k) Zm[ii][k] = Zk[ii][k] = 0.0;
    if constexpr (F >= 6) {
      // wide slabs: raw table coefficients in the j loop (rho folded into
      // pre once per value, V and rho V / hz^2 applied after the sums), so
      // no per-cell coefficient products stay live in registers (F = 8
      // spilled otherwise)
#pragma unroll
      for (int j = 0; j < F; ++j) {
        double vc[N], vp[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          vc[k] = A0[oz + j * Y::SD2 + k * Y::PZ2];
          vp[k] = rho * A1[oz + j * Y::SD2 + k * Y::PZ2];
        }
#pragma unroll
        for (int ii = 0; ii < FPG; ++ii) {
          const int i = j0 + ii;
          if (i >= F) break;
          const double cm = L.CM[i * F + j], ca = L.CA[i * F + j];
          if (cm == 0.0 && ca == 0.0) continue;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            Zm[ii][k] = fma(cm, vc[k], fma(ca, vp[k], Zm[ii][k]));
            Zk[ii][k] = fma(ca, vc[k], Zk[ii][k]);
          }
        }
      }
#pragma unroll
      for (int ii = 0; ii < FPG; ++ii)
#pragma unroll
        for (int k = 0; k < N; ++k) {
          Zm[ii][k] *= V;
          Zk[ii][k] *= rvz;
        }
    } else {
      const double rv = rho * V;
#pragma unroll
      for (int j = 0; j < F; ++j) {
        double vc[N], vp[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          vc[k] = A0[oz + j * Y::SD2 + k * Y::PZ2];
          vp[k] = A1[oz + j * Y::SD2 + k * Y::PZ2];
        }
#pragma unroll
        for (int ii = 0; ii < FPG; ++ii) {
          const int i = j0 + ii;
          if (i >= F) break;
          const double cmv = L.CM[i * F + j], cav = L.CA[i * F + j];
          if (cmv == 0.0 && cav == 0.0) continue;
          const double cm = V * cmv, ca = rv * cav, ck = rvz * cav;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            Zm[ii][k] = fma(cm, vc[k], fma(ca, vp[k], Zm[ii][k]));
            Zk[ii][k] = fma(ck, vc[k], Zk[ii][k]);
          }
        }
      }
    }
    auto dirichlet = [&](int lx, int ly, int lz) {
      return ((mask & 1) && lx == 0) || ((mask & 2) && lx == p) || ((mask & 4) && ly == 0) ||
             ((mask & 8) && ly == p) || ((mask & 16) && lz == 0) || ((mask & 32) && lz == p);
    };
#pragma unroll
    for (int ii = 0; ii < FPG; ++ii) {
      const int i = j0 + ii;
      if (i >= F) break;
      double em[EO<N>::HE], om[EO<N>::H], ek[EO<N>::HE], ok[EO<N>::H];
      eo_split<N>(Zm[ii], em, om);
      eo_split<N>(Zk[ii], ek, ok);
      double se[EO<N>::HE], so[EO<N>::H], te[EO<N>::HE], to[EO<N>::H], out[N];
      eo_even<N>(L.MrE, em, se);
      eo_odd<N>(L.MrO, om, so);
      eo_even<N>(L.KrE, ek, te);
      eo_odd<N>(L.KrO, ok, to);
#pragma unroll
      for (int q = 0; q < EO<N>::HE; ++q) se[q] += te[q];
#pragma unroll
      for (int q = 0; q < EO<N>::H; ++q) so[q] += to[q];
      eo_merge<N>(se, so, out);
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (!dirichlet(a, b, k)) atomicAdd(y + i * ns + base + k * dxy + b * dx + a, sign * out[k]);
    }
  }
}

template <int N, int F>
void launch(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t stream) {
  using C = Cfg<N, F>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(st_cart_kernel<N, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(C::smem_bytes()));
    cudaFuncSetAttribute(st_cart_kernel<N, F>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    configured = true;
  }
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long blocks = (n_cells + C::NC - 1) / C::NC;
  st_cart_kernel<N, F><<<static_cast<unsigned>(blocks), C::T, C::smem_bytes(), stream>>>(L, u, y, sign);
}

}  // namespace stc
}  // namespace stmgb
