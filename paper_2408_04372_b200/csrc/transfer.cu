// Grid transfers between consecutive multigrid levels (reference: Transfer,
// transfer.cpp:58-190). Spatial h/p transfers are tensor products of the
// per-axis embedding matrices P (n_f x n_c, transfer.cpp:32-54); they are
// applied here as separable passes, one lattice axis at a time, each output
// entry gathering the few nonzeros of its CSR row of P (prolongation) or of
// P^T (restriction) -- O((p+1) d) work per entry instead of the reference's
// dense O(n_f n_c) line contraction. Temporal tau/k transfers apply the small
// (S_f n_tf) x (S_c n_tc) evaluation matrix blockwise over the spatial dofs.
// Dirichlet entries are zeroed on the input and output sides
// (transfer.cpp:108-116).
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.hpp"

namespace stmgb {

namespace {

__device__ __forceinline__ bool on_bdry(long long i, long long n) { return i == 0 || i == n - 1; }

// out[f][z][y][x] (dims o[]) = sum_k w_k in[f][..src..] along `axis`;
// input dims i[] equal o[] except along axis.
template <int AXIS>
__global__ void axis_pass_kernel(int F, long long ix, long long iy, long long iz, long long ox, long long oy,
                                 long long oz, const int* __restrict__ ptr, const int* __restrict__ idx,
                                 const double* __restrict__ w, bool mask_in, bool mask_out, bool accumulate,
                                 const double* __restrict__ in, double* __restrict__ out) {
  const long long on = ox * oy * oz, in_n = ix * iy * iz;
  const long long total = on * F;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long f = t / on;
    const long long g = t - f * on;
    const long long x = g % ox, y = (g / ox) % oy, z = g / (ox * oy);
    double s = 0.0;
    const bool zero_out = mask_out && (on_bdry(x, ox) || (oy > 1 && on_bdry(y, oy)) || (oz > 1 && on_bdry(z, oz)));
    if (!zero_out) {
      const long long o = AXIS == 0 ? x : (AXIS == 1 ? y : z);
      const int k0 = ptr[o], k1 = ptr[o + 1];
      const double* src = in + f * in_n;
      bool other_bd = false;
      if (mask_in) {
        if (AXIS != 0) other_bd = other_bd || on_bdry(x, ix);
        if (AXIS != 1 && iy > 1) other_bd = other_bd || on_bdry(y, iy);
        if (AXIS != 2 && iz > 1) other_bd = other_bd || on_bdry(z, iz);
      }
      if (!other_bd) {
        const long long n_ax = AXIS == 0 ? ix : (AXIS == 1 ? iy : iz);
        for (int k = k0; k < k1; ++k) {
          const long long j = idx[k];
          if (mask_in && on_bdry(j, n_ax)) continue;
          const long long sidx = AXIS == 0 ? (z * iy + y) * ix + j : (AXIS == 1 ? (z * iy + j) * ix + x : (j * iy + y) * ix + x);
          s = fma(w[k], src[sidx], s);
        }
      }
    }
    if (accumulate)
      out[t] += s;
    else
      out[t] = s;
  }
}

__global__ void temporal_kernel(const double* __restrict__ T, int Ff, int Fc, bool transpose, bool accumulate,
                                long long n_space, long long dx, long long dy, long long dz, int dim,
                                const double* __restrict__ in, double* __restrict__ out) {
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
      if (accumulate)
        out[r * n_space + g] += s;
      else
        out[r * n_space + g] = s;
    }
  }
}

inline unsigned grid_for(long long n) {
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 64)));
}

template <int AXIS>
void pass(int F, const long long* in_d, const long long* out_d, const int* ptr, const int* idx, const double* w,
          bool mask_in, bool mask_out, bool accumulate, const double* in, double* out, cudaStream_t s) {
  const long long total = out_d[0] * out_d[1] * out_d[2] * F;
  count_launch();
  axis_pass_kernel<AXIS><<<grid_for(total), 256, 0, s>>>(F, in_d[0], in_d[1], in_d[2], out_d[0], out_d[1], out_d[2],
                                                         ptr, idx, w, mask_in, mask_out, accumulate, in, out);
}

// apply the per-axis CSR maps x, then y, then z (2D: x, y)
void separable(const DevAxisTransfer* ax, bool prolong, int dim, int F, const long long* src_d, const long long* dst_d,
               const double* in, double* out, double* t1, double* t2, bool accumulate, cudaStream_t s) {
  auto P = [&](int a, const int*& ptr, const int*& idx, const double*& w) {
    if (prolong) {
      ptr = ax[a].row_ptr;
      idx = ax[a].row_idx;
      w = ax[a].row_w;
    } else {
      ptr = ax[a].col_ptr;
      idx = ax[a].col_idx;
      w = ax[a].col_w;
    }
  };
  const int *ptr, *idx;
  const double* w;
  long long d1[3] = {dst_d[0], src_d[1], src_d[2]};
  P(0, ptr, idx, w);
  pass<0>(F, src_d, d1, ptr, idx, w, true, false, false, in, t1, s);
  if (dim == 2) {
    P(1, ptr, idx, w);
    pass<1>(F, d1, dst_d, ptr, idx, w, false, true, accumulate, t1, out, s);
    return;
  }
  long long d2[3] = {dst_d[0], dst_d[1], src_d[2]};
  P(1, ptr, idx, w);
  pass<1>(F, d1, d2, ptr, idx, w, false, false, false, t1, t2, s);
  P(2, ptr, idx, w);
  pass<2>(F, d2, dst_d, ptr, idx, w, false, true, accumulate, t2, out, s);
}

}  // namespace

void spatial_prolong(const DevAxisTransfer* ax, int dim, int F, const long long* dc, const long long* df,
                     const double* coarse, double* fine, double* t1, double* t2, bool accumulate, cudaStream_t s) {
  separable(ax, true, dim, F, dc, df, coarse, fine, t1, t2, accumulate, s);
}
void spatial_restrict(const DevAxisTransfer* ax, int dim, int F, const long long* dc, const long long* df,
                      const double* fine, double* coarse, double* t1, double* t2, cudaStream_t s) {
  separable(ax, false, dim, F, df, dc, fine, coarse, t1, t2, false, s);
}
void temporal_prolong(const double* T, int Ff, int Fc, long long n_space, const long long* d, int dim,
                      const double* coarse, double* fine, bool accumulate, cudaStream_t s) {
  count_launch();
  temporal_kernel<<<grid_for(n_space), 256, 0, s>>>(T, Ff, Fc, false, accumulate, n_space, d[0], d[1], d[2], dim,
                                                     coarse, fine);
}
void temporal_restrict(const double* T, int Ff, int Fc, long long n_space, const long long* d, int dim,
                       const double* fine, double* coarse, cudaStream_t s) {
  count_launch();
  temporal_kernel<<<grid_for(n_space), 256, 0, s>>>(T, Ff, Fc, true, false, n_space, d[0], d[1], d[2], dim, fine,
                                                     coarse);
}

}  // namespace stmgb
