// Grid transfers between consecutive multigrid levels (reference: Transfer,
// transfer.cpp:58-190). Spatial h/p transfers are tensor products of the
// per-axis embedding matrices P (fine x coarse); here each fine dof gathers
// the (p_c+1)^d coarse values of its parent cell with the per-axis weights
// (local parent-cell stencil instead of the reference's dense O(n_f*n_c) 1D
// contraction), and restriction (= P^T) gathers along the CSR columns of P.
// Temporal tau/k transfers apply the small (S_f n_tf) x (S_c n_tc) evaluation
// matrix blockwise over the spatial dofs. Dirichlet entries are zeroed on both
// sides, as transfer.cpp:108-116.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.hpp"

namespace stmgb {

namespace {

struct Axes {
  DevAxisTransfer a[3];
};

__device__ __forceinline__ bool on_bdry(long long i, long long n) { return i == 0 || i == n - 1; }

__global__ void spatial_prolong_kernel(Axes ax, int dim, int F, long long dcx, long long dcy, long long dcz,
                                       long long dfx, long long dfy, long long dfz, const double* __restrict__ c,
                                       double* __restrict__ f) {
  const long long nfs = dfx * dfy * dfz, ncs = dcx * dcy * dcz;
  const long long total = nfs * F;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int fld = static_cast<int>(t / nfs);
    const long long g = t - fld * nfs;
    const long long ix = g % dfx, iy = (g / dfx) % dfy, iz = g / (dfx * dfy);
    bool bd = on_bdry(ix, dfx) || (dim > 1 && on_bdry(iy, dfy)) || (dim > 2 && on_bdry(iz, dfz));
    double s = 0.0;
    if (!bd) {
      const double* cf = c + fld * ncs;
      const int nx = ax.a[0].row_nnz;
      const int ny = dim > 1 ? ax.a[1].row_nnz : 1;
      const int nz = dim > 2 ? ax.a[2].row_nnz : 1;
      const long long sx = ax.a[0].row_start[ix];
      const long long sy = dim > 1 ? ax.a[1].row_start[iy] : 0;
      const long long sz = dim > 2 ? ax.a[2].row_start[iz] : 0;
      for (int kz = 0; kz < nz; ++kz) {
        const long long jz = sz + kz;
        if (dim > 2 && on_bdry(jz, dcz)) continue;
        const double wz = dim > 2 ? ax.a[2].row_w[iz * nz + kz] : 1.0;
        if (wz == 0.0) continue;
        for (int ky = 0; ky < ny; ++ky) {
          const long long jy = sy + ky;
          if (dim > 1 && on_bdry(jy, dcy)) continue;
          const double wyz = wz * (dim > 1 ? ax.a[1].row_w[iy * ny + ky] : 1.0);
          if (wyz == 0.0) continue;
          double sxs = 0.0;
          for (int kx = 0; kx < nx; ++kx) {
            const long long jx = sx + kx;
            if (on_bdry(jx, dcx)) continue;
            sxs = fma(ax.a[0].row_w[ix * nx + kx], cf[(jz * dcy + jy) * dcx + jx], sxs);
          }
          s = fma(wyz, sxs, s);
        }
      }
    }
    f[t] = s;
  }
}

__global__ void spatial_restrict_kernel(Axes ax, int dim, int F, long long dcx, long long dcy, long long dcz,
                                        long long dfx, long long dfy, long long dfz, const double* __restrict__ f,
                                        double* __restrict__ c) {
  const long long nfs = dfx * dfy * dfz, ncs = dcx * dcy * dcz;
  const long long total = ncs * F;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int fld = static_cast<int>(t / ncs);
    const long long g = t - fld * ncs;
    const long long jx = g % dcx, jy = (g / dcx) % dcy, jz = g / (dcx * dcy);
    bool bd = on_bdry(jx, dcx) || (dim > 1 && on_bdry(jy, dcy)) || (dim > 2 && on_bdry(jz, dcz));
    double s = 0.0;
    if (!bd) {
      const double* ff = f + fld * nfs;
      const int bz0 = dim > 2 ? ax.a[2].col_ptr[jz] : 0, bz1 = dim > 2 ? ax.a[2].col_ptr[jz + 1] : 1;
      const int by0 = dim > 1 ? ax.a[1].col_ptr[jy] : 0, by1 = dim > 1 ? ax.a[1].col_ptr[jy + 1] : 1;
      const int bx0 = ax.a[0].col_ptr[jx], bx1 = ax.a[0].col_ptr[jx + 1];
      for (int kz = bz0; kz < bz1; ++kz) {
        const long long iz = dim > 2 ? ax.a[2].col_idx[kz] : 0;
        if (dim > 2 && on_bdry(iz, dfz)) continue;
        const double wz = dim > 2 ? ax.a[2].col_w[kz] : 1.0;
        for (int ky = by0; ky < by1; ++ky) {
          const long long iy = dim > 1 ? ax.a[1].col_idx[ky] : 0;
          if (dim > 1 && on_bdry(iy, dfy)) continue;
          const double wyz = wz * (dim > 1 ? ax.a[1].col_w[ky] : 1.0);
          double sxs = 0.0;
          for (int kx = bx0; kx < bx1; ++kx) {
            const long long ix = ax.a[0].col_idx[kx];
            if (on_bdry(ix, dfx)) continue;
            sxs = fma(ax.a[0].col_w[kx], ff[(iz * dfy + iy) * dfx + ix], sxs);
          }
          s = fma(wyz, sxs, s);
        }
      }
    }
    c[t] = s;
  }
}

__global__ void temporal_kernel(const double* __restrict__ T, int Ff, int Fc, bool transpose, long long n_space,
                                long long dx, long long dy, long long dz, int dim, const double* __restrict__ in,
                                double* __restrict__ out) {
  // prolong: out (Ff blocks) = T in (Fc blocks); restrict: out (Fc) = T^T in (Ff)
  const int Fin = transpose ? Ff : Fc, Fout = transpose ? Fc : Ff;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n_space; g += (long long)gridDim.x * blockDim.x) {
    const long long ix = g % dx, iy = (g / dx) % dy, iz = g / (dx * dy);
    const bool bd = on_bdry(ix, dx) || (dim > 1 && on_bdry(iy, dy)) || (dim > 2 && on_bdry(iz, dz));
    double x[kMaxF];
#pragma unroll
    for (int c = 0; c < kMaxF; ++c) x[c] = (c < Fin && !bd) ? in[c * n_space + g] : 0.0;
#pragma unroll
    for (int r = 0; r < kMaxF; ++r) {
      if (r >= Fout) break;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < kMaxF; ++c)
        if (c < Fin) s = fma(transpose ? T[c * Fc + r] : T[r * Fc + c], x[c], s);
      out[r * n_space + g] = s;
    }
  }
}

inline unsigned grid_for(long long n) {
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 64)));
}

}  // namespace

void spatial_prolong(const DevAxisTransfer* ax, int dim, int F, const long long* dc, const long long* df,
                     const double* coarse, double* fine, cudaStream_t s) {
  Axes a{};
  for (int i = 0; i < dim; ++i) a.a[i] = ax[i];
  const long long total = df[0] * df[1] * df[2] * F;
  count_launch();
  spatial_prolong_kernel<<<grid_for(total), 256, 0, s>>>(a, dim, F, dc[0], dc[1], dc[2], df[0], df[1], df[2], coarse,
                                                          fine);
}
void spatial_restrict(const DevAxisTransfer* ax, int dim, int F, const long long* dc, const long long* df,
                      const double* fine, double* coarse, cudaStream_t s) {
  Axes a{};
  for (int i = 0; i < dim; ++i) a.a[i] = ax[i];
  const long long total = dc[0] * dc[1] * dc[2] * F;
  count_launch();
  spatial_restrict_kernel<<<grid_for(total), 256, 0, s>>>(a, dim, F, dc[0], dc[1], dc[2], df[0], df[1], df[2], fine,
                                                           coarse);
}
void temporal_prolong(const double* T, int Ff, int Fc, long long n_space, const long long* d, int dim,
                      const double* coarse, double* fine, cudaStream_t s) {
  count_launch();
  temporal_kernel<<<grid_for(n_space), 256, 0, s>>>(T, Ff, Fc, false, n_space, d[0], d[1], d[2], dim, coarse, fine);
}
void temporal_restrict(const double* T, int Ff, int Fc, long long n_space, const long long* d, int dim,
                       const double* fine, double* coarse, cudaStream_t s) {
  count_launch();
  temporal_kernel<<<grid_for(n_space), 256, 0, s>>>(T, Ff, Fc, true, n_space, d[0], d[1], d[2], dim, fine, coarse);
}

}  // namespace stmgb
