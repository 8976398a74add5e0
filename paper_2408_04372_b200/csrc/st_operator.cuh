// Fused matrix-free space-time operator y = S u for one slab system on one
// level (reference: SpaceTimeOperator::apply, space_time_operator.cpp:45-130,
// which calls SpatialOperator::apply 2*S*n_t times, spatial_operator.cpp:187-315).
//
// One CTA owns NC consecutive cells and ALL F = S*n_t temporal fields of
// each cell, so u and y cross HBM once per application:
//   1. gather the cells' nodal values of every field into shared memory
//      (Dirichlet inputs zeroed, spatial_operator.cpp:304-307),
//   2. sum-factorised interpolation to the q = p+1 Gauss points per axis
//      (B sweeps) and collocation derivatives (Dq sweeps), one thread per
//      (cell, field, lattice line),
//   3. at every quadrature point: the temporal block coupling of the whole
//      slab (CM/CA, space_time_operator.cpp:269-317) and the metric terms
//      w|J| and rho w |J| J^-1 J^-T computed on the fly from the cell's
//      d-linear map (spatial_operator.cpp:152-183) -- no cached metric is
//      streamed from HBM,
//   4. transposed sweeps back to the nodes and one atomic scatter-add into y;
//      Dirichlet rows of y are set to u by a separate boundary pass
//      (space_time_operator.cpp:125-129).
// All shapes (dim, p+1, F) are compile-time: index arithmetic is shifts and
// constant multiplies; the only 64-bit math is one base offset per cell.
#pragma once

#include <cuda_runtime.h>

#include "device.cuh"

namespace stmgb {
namespace stk {

constexpr int kThreads = 256;

template <int DIM, int N, int F>
struct Cfg {
  static constexpr int ND = DIM == 2 ? N * N : N * N * N;
  static constexpr int LINES = DIM == 2 ? N : N * N;
  // padded shared-memory layout x + N y + PZ z of a cell array: for p = 3 the
  // plane pitch 19 makes the x- and z-line sweeps bank-conflict free and the
  // y-line sweep at most 2-way (the natural pitch 16 gives 4-way on x lines)
  static constexpr int PZ = (DIM == 3 && N == 4) ? 19 : N * N;
  static constexpr int SD = DIM == 2 ? N * N : N * PZ;  // array stride in doubles
  static constexpr int NC = (kThreads / ND) > 0 ? (kThreads / ND) : 1;  // cells per CTA
  static constexpr int NCF = NC * F;
  static constexpr int GEO = DIM == 2 ? 6 : 21;  // d-linear map coefficients per cell
  static constexpr size_t smem_bytes() {
    return sizeof(double) * (static_cast<size_t>(NCF) * SD * (1 + DIM) + static_cast<size_t>(NC) * (GEO + 1)) +
           sizeof(long long) * NC + sizeof(int) * NC;
  }
};

template <int N, bool T>
__device__ __forceinline__ void sweep_inplace(double* arr, int base, int stride, const double (&M)[kMaxN][kMaxN]) {
  double in[N];
#pragma unroll
  for (int k = 0; k < N; ++k) in[k] = arr[base + k * stride];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(T ? M[k][i] : M[i][k], in[k], s);
    arr[base + i * stride] = s;
  }
}

template <int N>
__device__ __forceinline__ void sweep_copy(const double* src, double* dst, int base, int stride,
                                           const double (&M)[kMaxN][kMaxN]) {
  double in[N];
#pragma unroll
  for (int k = 0; k < N; ++k) in[k] = src[base + k * stride];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(M[i][k], in[k], s);
    dst[base + i * stride] = s;
  }
}

template <int N>
__device__ __forceinline__ void sweep_addT(const double* src, double* dst, int base, int stride,
                                           const double (&M)[kMaxN][kMaxN]) {
  double in[N];
#pragma unroll
  for (int k = 0; k < N; ++k) in[k] = src[base + k * stride];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = dst[base + i * stride];
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(M[k][i], in[k], s);
    dst[base + i * stride] = s;
  }
}

template <int N, int A>
__device__ __forceinline__ constexpr int pw() {
  return A == 0 ? 1 : (A == 1 ? N : N * N);
}

// natural local index l (x fastest) -> padded position x + N y + PZ z
template <int N, int PZ>
__device__ __forceinline__ int pidx(int l) {
  return (l % N) + N * ((l / N) % N) + PZ * (l / (N * N));
}

// base position of lattice line `line` along axis A in the padded layout
// (lines enumerate the other two axes, lower axis fastest)
template <int N, int PZ, int A>
__device__ __forceinline__ int line_base(int line) {
  const int a = line % N, b = line / N;
  if (A == 0) return N * a + PZ * b;  // (y, z)
  if (A == 1) return a + PZ * b;      // (x, z)
  return a + N * b;                   // (x, y)
}

template <int DIM, int N, int F>
__global__ void __launch_bounds__(kThreads, 2) st_apply_kernel(const __grid_constant__ DevLevel L,
                                                               const double* __restrict__ u, double* __restrict__ y,
                                                               double sign) {
  using C = Cfg<DIM, N, F>;
  constexpr int ND = C::ND, LINES = C::LINES, NC = C::NC, NCF = C::NCF, GEO = C::GEO;
  constexpr int PZ = C::PZ, SD = C::SD;
  constexpr int T = kThreads;
  extern __shared__ __align__(16) double smem[];
  double* V = smem;                    // [NCF][SD]
  double* G = V + NCF * SD;            // [DIM][NCF][SD]
  double* geo = G + DIM * NCF * SD;    // [NC][GEO] map coefficients
  double* rho_s = geo + NC * GEO;      // [NC]
  long long* base_s = reinterpret_cast<long long*>(rho_s + NC);  // [NC] lattice offset of local dof 0
  int* mask_s = reinterpret_cast<int*>(base_s + NC);             // [NC] Dirichlet face mask (bit 2a: low, 2a+1: high)

  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long cell0 = static_cast<long long>(blockIdx.x) * NC;
  const int tid = threadIdx.x;
  const long long dx = L.dofs[0], dxy = L.dofs[0] * L.dofs[1];
  const int p = N - 1;

  // ---- per-cell data: offsets, boundary faces, d-linear map, coefficient
  if (tid < NC) {
    const int c = tid;
    const long long cell = cell0 + c;
    long long base = -1;
    int mask = 0;
    if (cell < n_cells) {
      const unsigned ci = static_cast<unsigned>(cell);
      const unsigned nx = static_cast<unsigned>(L.cells[0]), ny = static_cast<unsigned>(L.cells[1]);
      const unsigned cx = ci % nx, cy = (ci / nx) % ny, cz = ci / (nx * ny);
      base = static_cast<long long>(cz) * p * dxy + static_cast<long long>(cy) * p * dx + static_cast<long long>(cx) * p;
      if (cx == 0) mask |= 1;
      if (cx == nx - 1) mask |= 2;
      if (cy == 0) mask |= 4;
      if (cy == ny - 1) mask |= 8;
      if (DIM == 3) {
        if (cz == 0 && (L.zbc & 1)) mask |= 16;
        if (cz == L.cells[2] - 1 && (L.zbc & 2)) mask |= 32;
      }
      double* gc = geo + c * GEO;
      if (L.verts) {
        const long long vx = L.cells[0] + 1, vy = L.cells[1] + 1;
        double X[8][3];
#pragma unroll
        for (int s = 0; s < (1 << DIM); ++s) {
          const long long i = cx + (s & 1), j = cy + ((s >> 1) & 1), k = DIM == 3 ? cz + ((s >> 2) & 1) : 0;
          const double* v = L.verts + 3 * ((k * vy + j) * vx + i);
#pragma unroll
          for (int a = 0; a < 3; ++a) X[s][a] = v[a];
        }
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
          if (DIM == 2) {
            gc[0 * 2 + a] = X[1][a] - X[0][a];                        // c1
            gc[1 * 2 + a] = X[2][a] - X[0][a];                        // c2
            gc[2 * 2 + a] = X[3][a] - X[2][a] - X[1][a] + X[0][a];    // c3
          } else {
            gc[0 * 3 + a] = X[1][a] - X[0][a];                                                      // c1
            gc[1 * 3 + a] = X[2][a] - X[0][a];                                                      // c2
            gc[2 * 3 + a] = X[4][a] - X[0][a];                                                      // c4
            gc[3 * 3 + a] = X[3][a] - X[2][a] - X[1][a] + X[0][a];                                  // c3
            gc[4 * 3 + a] = X[5][a] - X[4][a] - X[1][a] + X[0][a];                                  // c5
            gc[5 * 3 + a] = X[6][a] - X[4][a] - X[2][a] + X[0][a];                                  // c6
            gc[6 * 3 + a] = X[7][a] - X[6][a] - X[5][a] + X[4][a] - X[3][a] + X[2][a] + X[1][a] - X[0][a];  // c7
          }
        }
      }
      double rho = 1.0;
      if (L.rho0) {
        const long long ax = cx >> L.rho_shift, ay = cy >> L.rho_shift, az = (cz + L.cz0) >> L.rho_shift;
        rho = L.rho0[(az * L.cells0[1] + ay) * L.cells0[0] + ax];
      }
      rho_s[c] = rho;
    }
    base_s[c] = base;
    mask_s[c] = mask;
  }
  __syncthreads();

  // ---- 1. gather (Dirichlet inputs zeroed)
#pragma unroll 4
  for (int idx = tid; idx < NCF * ND; idx += T) {
    const int c = idx / (F * ND);
    const int rem = idx - c * (F * ND);
    const int f = rem / ND;
    const int l = rem - f * ND;
    const long long base = base_s[c];
    double v = 0.0;
    if (base >= 0) {
      const int lx = l % N, ly = (l / N) % N, lz = DIM == 3 ? l / (N * N) : 0;
      const int m = mask_s[c];
      bool bd = ((m & 1) && lx == 0) || ((m & 2) && lx == N - 1) || ((m & 4) && ly == 0) || ((m & 8) && ly == N - 1);
      if (DIM == 3) bd = bd || ((m & 16) && lz == 0) || ((m & 32) && lz == N - 1);
      if (!bd) v = __ldg(u + f * L.n_space + base + lz * dxy + ly * dx + lx);
    }
    V[(c * F + f) * SD + pidx<N, PZ>(l)] = v;
  }
  __syncthreads();

  // ---- 2. values and reference gradients at the Gauss points
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    for (int ln = tid; ln < NCF * LINES; ln += T) {
      const int cf = ln / LINES, line = ln - cf * LINES;
      if (a == 0) sweep_inplace<N, false>(V + cf * SD, line_base<N, PZ, 0>(line), 1, L.B);
      if (a == 1) sweep_inplace<N, false>(V + cf * SD, line_base<N, PZ, 1>(line), N, L.B);
      if (a == 2) sweep_inplace<N, false>(V + cf * SD, line_base<N, PZ, 2>(line), PZ, L.B);
    }
    __syncthreads();
  }
  for (int ln = tid; ln < NCF * LINES; ln += T) {
    const int cf = ln / LINES, line = ln - cf * LINES;
    sweep_copy<N>(V + cf * SD, G + (0 * NCF + cf) * SD, line_base<N, PZ, 0>(line), 1, L.Dq);
    sweep_copy<N>(V + cf * SD, G + (1 * NCF + cf) * SD, line_base<N, PZ, 1>(line), N, L.Dq);
    if (DIM == 3) sweep_copy<N>(V + cf * SD, G + (2 * NCF + cf) * SD, line_base<N, PZ, 2>(line), PZ, L.Dq);
  }
  __syncthreads();

  // ---- 3. quadrature-point work
  for (int idx = tid; idx < NC * ND; idx += T) {
    const int c = idx / ND;
    const int q = idx - c * ND;
    const int qp = pidx<N, PZ>(q);
    if (base_s[c] < 0) continue;
    const int qx = q % N, qy = (q / N) % N, qz = DIM == 3 ? q / (N * N) : 0;
    double wq = L.w[qx] * L.w[qy];
    if (DIM == 3) wq *= L.w[qz];
    const double rho = rho_s[c];
    double K00, K01, K02 = 0.0, K11, K12 = 0.0, K22 = 0.0, mass_fac;
    if (!L.verts) {
      const double det = DIM == 3 ? L.h[0] * L.h[1] * L.h[2] : L.h[0] * L.h[1];
      mass_fac = wq * det;
      const double s = rho * wq * det;
      K00 = s / (L.h[0] * L.h[0]);
      K11 = s / (L.h[1] * L.h[1]);
      if (DIM == 3) K22 = s / (L.h[2] * L.h[2]);
      K01 = 0.0;
    } else {
      const double* gc = geo + c * GEO;
      const double xx = L.xq[qx], xy = L.xq[qy];
      if (DIM == 2) {
        // columns of J: d/dxi_x = c1 + c3 xi_y, d/dxi_y = c2 + c3 xi_x
        const double J00 = fma(gc[4], xy, gc[0]), J10 = fma(gc[5], xy, gc[1]);
        const double J01 = fma(gc[4], xx, gc[2]), J11 = fma(gc[5], xx, gc[3]);
        const double det = J00 * J11 - J01 * J10;
        const double s = rho * wq / det;
        K00 = s * (J11 * J11 + J01 * J01);
        K01 = -s * (J11 * J10 + J01 * J00);
        K11 = s * (J10 * J10 + J00 * J00);
        mass_fac = wq * det;
      } else {
        const double xz = L.xq[qz];
        double J[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double c1 = gc[0 * 3 + a], c2 = gc[1 * 3 + a], c4 = gc[2 * 3 + a];
          const double c3 = gc[3 * 3 + a], c5 = gc[4 * 3 + a], c6 = gc[5 * 3 + a], c7 = gc[6 * 3 + a];
          J[a][0] = fma(xz, fma(c7, xy, c5), fma(c3, xy, c1));
          J[a][1] = fma(xz, fma(c7, xx, c6), fma(c3, xx, c2));
          J[a][2] = fma(xy, fma(c7, xx, c6), fma(c5, xx, c4));
        }
        // rows of adj(J) (cofactors), det = J col 0 . adj row 0
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
        const double s = rho * wq / det;
        K00 = s * (R00 * R00 + R01 * R01 + R02 * R02);
        K01 = s * (R00 * R10 + R01 * R11 + R02 * R12);
        K02 = s * (R00 * R20 + R01 * R21 + R02 * R22);
        K11 = s * (R10 * R10 + R11 * R11 + R12 * R12);
        K12 = s * (R10 * R20 + R11 * R21 + R12 * R22);
        K22 = s * (R20 * R20 + R21 * R21 + R22 * R22);
        mass_fac = wq * det;
      }
    }
    double vin[F], gin[F][DIM];
#pragma unroll
    for (int j = 0; j < F; ++j) {
      vin[j] = V[(c * F + j) * SD + qp];
#pragma unroll
      for (int a = 0; a < DIM; ++a) gin[j][a] = G[(a * NCF + c * F + j) * SD + qp];
    }
#pragma unroll
    for (int i = 0; i < F; ++i) {
      double vo = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
#pragma unroll
      for (int j = 0; j < F; ++j) {
        vo = fma(L.CM[i * F + j], vin[j], vo);
        const double ca = L.CA[i * F + j];
        g0 = fma(ca, gin[j][0], g0);
        g1 = fma(ca, gin[j][1], g1);
        if (DIM == 3) g2 = fma(ca, gin[j][DIM - 1], g2);
      }
      V[(c * F + i) * SD + qp] = mass_fac * vo;
      if (DIM == 2) {
        G[(0 * NCF + c * F + i) * SD + qp] = fma(K00, g0, K01 * g1);
        G[(1 * NCF + c * F + i) * SD + qp] = fma(K01, g0, K11 * g1);
      } else {
        G[(0 * NCF + c * F + i) * SD + qp] = fma(K00, g0, fma(K01, g1, K02 * g2));
        G[(1 * NCF + c * F + i) * SD + qp] = fma(K01, g0, fma(K11, g1, K12 * g2));
        G[((DIM - 1) * NCF + c * F + i) * SD + qp] = fma(K02, g0, fma(K12, g1, K22 * g2));
      }
    }
  }
  __syncthreads();

  // ---- 4. back to the nodes: V += sum_a Dq_a^T G_a, then B^T sweeps
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    for (int ln = tid; ln < NCF * LINES; ln += T) {
      const int cf = ln / LINES, line = ln - cf * LINES;
      if (a == 0) sweep_addT<N>(G + (0 * NCF + cf) * SD, V + cf * SD, line_base<N, PZ, 0>(line), 1, L.Dq);
      if (a == 1) sweep_addT<N>(G + (1 * NCF + cf) * SD, V + cf * SD, line_base<N, PZ, 1>(line), N, L.Dq);
      if (a == 2) sweep_addT<N>(G + (2 * NCF + cf) * SD, V + cf * SD, line_base<N, PZ, 2>(line), PZ, L.Dq);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    for (int ln = tid; ln < NCF * LINES; ln += T) {
      const int cf = ln / LINES, line = ln - cf * LINES;
      if (a == 0) sweep_inplace<N, true>(V + cf * SD, line_base<N, PZ, 0>(line), 1, L.B);
      if (a == 1) sweep_inplace<N, true>(V + cf * SD, line_base<N, PZ, 1>(line), N, L.B);
      if (a == 2) sweep_inplace<N, true>(V + cf * SD, line_base<N, PZ, 2>(line), PZ, L.B);
    }
    __syncthreads();
  }

  // ---- 5. scatter-add (Dirichlet rows are written by the boundary pass)
#pragma unroll 4
  for (int idx = tid; idx < NCF * ND; idx += T) {
    const int c = idx / (F * ND);
    const int rem = idx - c * (F * ND);
    const int f = rem / ND;
    const int l = rem - f * ND;
    const long long base = base_s[c];
    if (base < 0) continue;
    const int lx = l % N, ly = (l / N) % N, lz = DIM == 3 ? l / (N * N) : 0;
    const int m = mask_s[c];
    bool bd = ((m & 1) && lx == 0) || ((m & 2) && lx == N - 1) || ((m & 4) && ly == 0) || ((m & 8) && ly == N - 1);
    if (DIM == 3) bd = bd || ((m & 16) && lz == 0) || ((m & 32) && lz == N - 1);
    if (!bd) atomicAdd(y + f * L.n_space + base + lz * dxy + ly * dx + lx, sign * V[(c * F + f) * SD + pidx<N, PZ>(l)]);
  }
}

template <int DIM, int N, int F>
void launch(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t stream) {
  using C = Cfg<DIM, N, F>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(st_apply_kernel<DIM, N, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(C::smem_bytes()));
    configured = true;
  }
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long blocks = (n_cells + C::NC - 1) / C::NC;
  st_apply_kernel<DIM, N, F><<<static_cast<unsigned>(blocks), kThreads, C::smem_bytes(), stream>>>(L, u, y, sign);
}

template <int DIM, int N>
void launch_f(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t s) {
  switch (L.F) {
    case 1: launch<DIM, N, 1>(L, u, y, sign, s); break;
    case 2: launch<DIM, N, 2>(L, u, y, sign, s); break;
    case 3: launch<DIM, N, 3>(L, u, y, sign, s); break;
    case 4: launch<DIM, N, 4>(L, u, y, sign, s); break;
    case 5: launch<DIM, N, 5>(L, u, y, sign, s); break;
    case 6: launch<DIM, N, 6>(L, u, y, sign, s); break;
    case 7: launch<DIM, N, 7>(L, u, y, sign, s); break;
    case 8: launch<DIM, N, 8>(L, u, y, sign, s); break;
  }
}

}  // namespace stk

// y += sign * (cell contributions of S u), Dirichlet rows untouched
void st_apply_2d(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t s);
void st_apply_3d(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t s);

}  // namespace stmgb
