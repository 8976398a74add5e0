// Fused matrix-free space-time operator y = S u for one slab system on one
// level (reference: SpaceTimeOperator::apply, space_time_operator.cpp:45-130,
// which calls SpatialOperator::apply 2*S*n_t times, spatial_operator.cpp:187-315).
//
// One CTA processes NC consecutive cells and ALL F = S*n_t temporal fields of
// each cell in one pass, so u and y cross HBM once per application:
//   1. gather the cells' nodal values of every field into shared memory
//      (Dirichlet inputs zeroed, spatial_operator.cpp:304-307),
//   2. sum-factorised interpolation to the q = p+1 Gauss points per axis
//      (B sweeps) and collocation derivatives (Dq sweeps), one thread per
//      (cell, field, lattice line),
//   3. at every quadrature point: the temporal block coupling of the whole
//      slab (CM/CA, space_time_operator.cpp:269-317) and the metric terms
//      w|J| and rho w |J| J^-1 J^-T, computed on the fly from the cell's
//      corner vertices (spatial_operator.cpp:152-183) -- no cached metric is
//      streamed from HBM,
//   4. transposed sweeps back to the nodes and one atomic scatter-add into y,
//   5. Dirichlet rows of y set to u (space_time_operator.cpp:125-129).
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "device.cuh"
#include "kernels.hpp"

namespace stmgb {

namespace {

template <int DIM, int N>
struct Shape {
  static constexpr int ND = DIM == 2 ? N * N : N * N * N;
  static constexpr int LINES = DIM == 2 ? N : N * N;
};

__device__ __forceinline__ int ipow(int n, int a) { return a == 0 ? 1 : (a == 1 ? n : n * n); }

// in-place y_line = M x_line (transpose=false) or M^T x_line along `axis`
template <int N, bool TRANSPOSE>
__device__ __forceinline__ void sweep_inplace(double* arr, int base, int stride, const double (&M)[kMaxN][kMaxN]) {
  double in[N];
#pragma unroll
  for (int k = 0; k < N; ++k) in[k] = arr[base + k * stride];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(TRANSPOSE ? M[k][i] : M[i][k], in[k], s);
    arr[base + i * stride] = s;
  }
}

// dst_line = M src_line
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

// dst_line += M^T src_line
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

__device__ __forceinline__ double det3(const double J[3][3]) {
  return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

template <int DIM, int N>
__global__ void __launch_bounds__(512) st_apply_kernel(const __grid_constant__ DevLevel L, const double* __restrict__ u,
                                                       double* __restrict__ y, int NC) {
  using Sh = Shape<DIM, N>;
  constexpr int ND = Sh::ND;
  constexpr int LINES = Sh::LINES;
  constexpr int NCORN = 1 << DIM;
  extern __shared__ double smem[];
  const int F = L.F;
  const int NCF = NC * F;
  double* V = smem;                          // [NCF][ND] values
  double* G = V + NCF * ND;                  // [DIM][NCF][ND] gradients
  double* geo = G + DIM * NCF * ND;          // [NC][NCORN*3 + 1] corners, rho
  constexpr int GEO = NCORN * 3 + 1;

  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long cell0 = static_cast<long long>(blockIdx.x) * NC;
  const int tid = threadIdx.x;
  const int nth = blockDim.x;
  const long long dx = L.dofs[0], dy = L.dofs[1], dz = L.dofs[2];

  // ---- 1. gather (Dirichlet inputs zeroed) + per-cell geometry
  for (int idx = tid; idx < NCF * ND; idx += nth) {
    const int c = idx / (F * ND);
    const int rem = idx - c * F * ND;
    const int f = rem / ND;
    const int l = rem - f * ND;
    const long long cell = cell0 + c;
    double v = 0.0;
    if (cell < n_cells) {
      const long long cx = cell % L.cells[0];
      const long long cy = (cell / L.cells[0]) % L.cells[1];
      const long long cz = cell / (L.cells[0] * L.cells[1]);
      const int lx = l % N, ly = (l / N) % N, lz = DIM == 3 ? l / (N * N) : 0;
      const long long gx = cx * L.p + lx, gy = cy * L.p + ly, gz = cz * L.p + lz;
      bool bdry = gx == 0 || gx == dx - 1 || gy == 0 || gy == dy - 1;
      if (DIM == 3) bdry = bdry || gz == 0 || gz == dz - 1;
      if (!bdry) v = __ldg(u + f * L.n_space + (gz * dy + gy) * dx + gx);
    }
    V[(c * F + f) * ND + l] = v;
  }
  for (int c = tid; c < NC; c += nth) {
    const long long cell = cell0 + c;
    double* gc = geo + c * GEO;
    if (cell < n_cells) {
      const long long cx = cell % L.cells[0];
      const long long cy = (cell / L.cells[0]) % L.cells[1];
      const long long cz = cell / (L.cells[0] * L.cells[1]);
      if (L.verts) {
        const long long vx = L.cells[0] + 1, vy = L.cells[1] + 1;
        for (int s = 0; s < NCORN; ++s) {
          const long long i = cx + (s & 1), j = cy + ((s >> 1) & 1), k = DIM == 3 ? cz + ((s >> 2) & 1) : 0;
          const long long vi = (k * vy + j) * vx + i;
          for (int a = 0; a < 3; ++a) gc[3 * s + a] = L.verts[3 * vi + a];
        }
      }
      double rho = 1.0;
      if (L.rho0) {
        const long long ax = cx >> L.rho_shift, ay = cy >> L.rho_shift, az = cz >> L.rho_shift;
        rho = L.rho0[(az * L.cells0[1] + ay) * L.cells0[0] + ax];
      }
      gc[GEO - 1] = rho;
    }
  }
  __syncthreads();

  const int cf = tid / LINES;  // (cell, field) pair of this thread's line
  const int line = tid - cf * LINES;
  const bool sweeper = cf < NCF;

  // ---- 2. values and reference gradients at the Gauss points
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const int stride = ipow(N, a);
    if (sweeper) sweep_inplace<N, false>(V + cf * ND, (line % stride) + (line / stride) * stride * N, stride, L.B);
    __syncthreads();
  }
  if (sweeper) {
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const int stride = ipow(N, a);
      sweep_copy<N>(V + cf * ND, G + (a * NCF + cf) * ND, (line % stride) + (line / stride) * stride * N, stride,
                    L.Dq);
    }
  }
  __syncthreads();

  // ---- 3. quadrature-point work: temporal coupling + metric
  for (int idx = tid; idx < NC * ND; idx += nth) {
    const int c = idx / ND;
    const int q = idx - c * ND;
    if (cell0 + c >= n_cells) continue;
    const double* gc = geo + c * GEO;
    const int qx = q % N, qy = (q / N) % N, qz = DIM == 3 ? q / (N * N) : 0;
    double wq = L.w[qx] * L.w[qy];
    if (DIM == 3) wq *= L.w[qz];
    const double rho = gc[GEO - 1];
    double Kq[3][3];
    double mass_fac;
    if (!L.verts) {
      double det = L.h[0] * L.h[1];
      if (DIM == 3) det *= L.h[2];
      mass_fac = wq * det;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) Kq[a][b] = (a == b && a < DIM) ? rho * wq * det / (L.h[a] * L.h[a]) : 0.0;
    } else {
      double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
      const double xq[3] = {L.xq[qx], L.xq[qy], DIM == 3 ? L.xq[qz] : 0.0};
#pragma unroll
      for (int s = 0; s < NCORN; ++s) {
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
          double dw = 1.0;
#pragma unroll
          for (int a = 0; a < DIM; ++a) {
            const int bit = (s >> a) & 1;
            dw *= (a == b) ? (bit ? 1.0 : -1.0) : (bit ? xq[a] : 1.0 - xq[a]);
          }
#pragma unroll
          for (int a = 0; a < DIM; ++a) J[a][b] = fma(dw, gc[3 * s + a], J[a][b]);
        }
      }
      if (DIM == 2) {
        const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const double s = rho * wq / det;
        // adj rows: (J11, -J01), (-J10, J00); K = s * adj adj^T
        const double r0[2] = {J[1][1], -J[0][1]}, r1[2] = {-J[1][0], J[0][0]};
        Kq[0][0] = s * (r0[0] * r0[0] + r0[1] * r0[1]);
        Kq[0][1] = Kq[1][0] = s * (r0[0] * r1[0] + r0[1] * r1[1]);
        Kq[1][1] = s * (r1[0] * r1[0] + r1[1] * r1[1]);
        Kq[0][2] = Kq[1][2] = Kq[2][0] = Kq[2][1] = Kq[2][2] = 0.0;
        mass_fac = wq * det;
      } else {
        const double det = det3(J);
        // rows of adj(J): cross products of the Jacobian columns
        double R[3][3];
        R[0][0] = J[1][1] * J[2][2] - J[2][1] * J[1][2];
        R[0][1] = J[2][1] * J[0][2] - J[0][1] * J[2][2];
        R[0][2] = J[0][1] * J[1][2] - J[1][1] * J[0][2];
        R[1][0] = J[1][2] * J[2][0] - J[2][2] * J[1][0];
        R[1][1] = J[2][2] * J[0][0] - J[0][2] * J[2][0];
        R[1][2] = J[0][2] * J[1][0] - J[1][2] * J[0][0];
        R[2][0] = J[1][0] * J[2][1] - J[2][0] * J[1][1];
        R[2][1] = J[2][0] * J[0][1] - J[0][0] * J[2][1];
        R[2][2] = J[0][0] * J[1][1] - J[1][0] * J[0][1];
        const double s = rho * wq / det;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = a; b < 3; ++b) {
            const double v = s * (R[a][0] * R[b][0] + R[a][1] * R[b][1] + R[a][2] * R[b][2]);
            Kq[a][b] = v;
            Kq[b][a] = v;
          }
        mass_fac = wq * det;
      }
    }
    // inputs of all fields at this point
    double vin[kMaxF], gin[kMaxF][3];
#pragma unroll
    for (int j = 0; j < kMaxF; ++j) {
      if (j < F) {
        vin[j] = V[(c * F + j) * ND + q];
#pragma unroll
        for (int a = 0; a < DIM; ++a) gin[j][a] = G[(a * NCF + c * F + j) * ND + q];
      }
    }
#pragma unroll
    for (int i = 0; i < kMaxF; ++i) {
      if (i < F) {
        double vo = 0.0, gt[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < kMaxF; ++j) {
          if (j < F) {
            const double cm = L.CM[i * F + j], ca = L.CA[i * F + j];
            vo = fma(cm, vin[j], vo);
#pragma unroll
            for (int a = 0; a < DIM; ++a) gt[a] = fma(ca, gin[j][a], gt[a]);
          }
        }
        V[(c * F + i) * ND + q] = mass_fac * vo;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < DIM; ++b) s = fma(Kq[a][b], gt[b], s);
          G[(a * NCF + c * F + i) * ND + q] = s;
        }
      }
    }
  }
  __syncthreads();

  // ---- 4. back to the nodes: V += sum_a Dq_a^T G_a, then B^T sweeps
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const int stride = ipow(N, a);
    if (sweeper)
      sweep_addT<N>(G + (a * NCF + cf) * ND, V + cf * ND, (line % stride) + (line / stride) * stride * N, stride,
                    L.Dq);
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const int stride = ipow(N, a);
    if (sweeper) sweep_inplace<N, true>(V + cf * ND, (line % stride) + (line / stride) * stride * N, stride, L.B);
    __syncthreads();
  }

  // ---- 5. scatter-add (Dirichlet rows are written by the boundary pass)
  for (int idx = tid; idx < NCF * ND; idx += nth) {
    const int c = idx / (F * ND);
    const int rem = idx - c * F * ND;
    const int f = rem / ND;
    const int l = rem - f * ND;
    const long long cell = cell0 + c;
    if (cell >= n_cells) continue;
    const long long cx = cell % L.cells[0];
    const long long cy = (cell / L.cells[0]) % L.cells[1];
    const long long cz = cell / (L.cells[0] * L.cells[1]);
    const int lx = l % N, ly = (l / N) % N, lz = DIM == 3 ? l / (N * N) : 0;
    const long long gx = cx * L.p + lx, gy = cy * L.p + ly, gz = cz * L.p + lz;
    bool bdry = gx == 0 || gx == dx - 1 || gy == 0 || gy == dy - 1;
    if (DIM == 3) bdry = bdry || gz == 0 || gz == dz - 1;
    if (!bdry) atomicAdd(y + f * L.n_space + (gz * dy + gy) * dx + gx, V[(c * F + f) * ND + l]);
  }
}

// y_b = u_b on every Dirichlet dof of every field
__global__ void boundary_identity_kernel(long long n_space, long long dx, long long dy, long long dz, int dim, int F,
                                         const double* __restrict__ u, double* __restrict__ y) {
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < n_space;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long ix = g % dx, iy = (g / dx) % dy, iz = g / (dx * dy);
    bool b = ix == 0 || ix == dx - 1;
    if (dim > 1) b = b || iy == 0 || iy == dy - 1;
    if (dim > 2) b = b || iz == 0 || iz == dz - 1;
    if (b)
      for (int f = 0; f < F; ++f) y[f * n_space + g] = u[f * n_space + g];
  }
}

template <int DIM, int N>
void launch_st(const DevLevel& L, const double* u, double* y, cudaStream_t stream) {
  using Sh = Shape<DIM, N>;
  const int tpc = L.F * Sh::LINES;  // threads per cell
  int NC = std::max(1, 256 / tpc);
  auto smem_bytes = [&](int nc) {
    return static_cast<size_t>(nc) * (L.F * Sh::ND * (1 + DIM) + ((1 << DIM) * 3 + 1)) * sizeof(double);
  };
  while (NC > 1 && smem_bytes(NC) > 200 * 1024) --NC;
  const int threads = std::max(NC * tpc, 32);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(st_apply_kernel<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long blocks = (n_cells + NC - 1) / NC;
  count_launch();
  st_apply_kernel<DIM, N><<<static_cast<unsigned>(blocks), threads, smem_bytes(NC), stream>>>(L, u, y, NC);
}

}  // namespace

void st_apply(const DevLevel& L, const double* u, double* y, cudaStream_t stream) {
  cudaMemsetAsync(y, 0, sizeof(double) * L.n_dofs, stream);
  const int key = L.dim * 10 + L.n;
  switch (key) {
    case 22: launch_st<2, 2>(L, u, y, stream); break;
    case 23: launch_st<2, 3>(L, u, y, stream); break;
    case 24: launch_st<2, 4>(L, u, y, stream); break;
    case 25: launch_st<2, 5>(L, u, y, stream); break;
    case 32: launch_st<3, 2>(L, u, y, stream); break;
    case 33: launch_st<3, 3>(L, u, y, stream); break;
    case 34: launch_st<3, 4>(L, u, y, stream); break;
    case 35: launch_st<3, 5>(L, u, y, stream); break;
    default: throw std::invalid_argument("st_apply: unsupported dim/p (dim 2-3, p 1-4)");
  }
  const int bthreads = 256;
  const long long bblocks = std::min<long long>((L.n_space + bthreads - 1) / bthreads, 148LL * 16);
  count_launch();
  boundary_identity_kernel<<<static_cast<unsigned>(bblocks), bthreads, 0, stream>>>(
      L.n_space, L.dofs[0], L.dofs[1], L.dofs[2], L.dim, L.F, u, y);
}

}  // namespace stmgb
