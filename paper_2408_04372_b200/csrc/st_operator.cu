// Space-time operator dispatch: zero y, fused cell kernel (st_operator.cuh,
// instantiated per dimension in st_operator_{2d,3d}.cu), Dirichlet identity
// rows (space_time_operator.cpp:125-129).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>

#include "kernels.hpp"
#include "st_operator.cuh"

namespace stmgb {

namespace {

// y_b = u_b on every Dirichlet dof of every field: enumerate the boundary
// faces of the lattice directly (edges/corners written more than once with
// the same value)
__global__ void boundary_identity_kernel(int dim, int zbc, long long dx, long long dy, long long dz, long long n_space,
                                         int F, const double* __restrict__ f, const double* __restrict__ u,
                                         double* __restrict__ y) {
  // faces: x=0, x=dx-1 (dy*dz each), y=0, y=dy-1 (dx*dz), z=0, z=dz-1 (dx*dy);
  // a slab's z faces only where they are physical (zbc), never on interfaces
  const long long fx = dy * dz, fy = dx * dz, fz = dim == 3 ? dx * dy : 0;
  const long long total = 2 * (fx + fy + fz);
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long g;
    long long r = t;
    // face-local indices fit 32 bits (a face has < 2^32 entries): 32-bit
    // division instead of the 64-bit software sequence
    const unsigned udx = static_cast<unsigned>(dx), udy = static_cast<unsigned>(dy);
    // the low plane of a slab whose low face is an interface is owned by the
    // slab below: its Dirichlet rows are written there only
    if (r < 2 * fx) {
      const long long side = r >= fx;
      const unsigned k = static_cast<unsigned>(r - side * fx), kz = k / udy, ky = k - kz * udy;
      if (dim == 3 && !(zbc & 1) && kz == 0) continue;
      g = static_cast<long long>(kz) * dx * dy + static_cast<long long>(ky) * dx + (side ? dx - 1 : 0);
    } else if ((r -= 2 * fx) < 2 * fy) {
      const long long side = r >= fy;
      const unsigned k = static_cast<unsigned>(r - side * fy), kz = k / udx, kx = k - kz * udx;
      if (dim == 3 && !(zbc & 1) && kz == 0) continue;
      g = static_cast<long long>(kz) * dx * dy + (side ? dy - 1 : 0) * dx + kx;
    } else {
      r -= 2 * fy;
      const long long side = r >= fz, k = r - side * fz;
      if (!(zbc & (side ? 2 : 1))) continue;
      g = (side ? dz - 1 : 0) * dx * dy + k;
    }
    // apply: y_b = u_b; residual: y_b = f_b - u_b
    for (int k = 0; k < F; ++k) y[k * n_space + g] = f ? f[k * n_space + g] - u[k * n_space + g] : u[k * n_space + g];
  }
}

}  // namespace

namespace {
void run(const DevLevel& L, const double* f, const double* u, double* y, cudaStream_t stream) {
  if (st_brick_supported(L)) {
    st_brick(L, f, u, y, stream);
    return;
  }
  if (f) {
    vec_copy(y, f, L.n_dofs, stream);
    // slab whose low z plane is an interface owned by the slab below: its f
    // entries are counted there, so the partial residual starts from 0
    if (L.dim == 3 && !(L.zbc & 1)) plane_fill(y, L.F, L.n_space, 0, L.dofs[0] * L.dofs[1], 0.0, stream);
  } else {
    cudaMemsetAsync(y, 0, sizeof(double) * L.n_dofs, stream);
  }
  const double sign = f ? -1.0 : 1.0;
  count_launch();
  if (L.dim == 2)
    st_apply_2d(L, u, y, sign, stream);
  else if (L.dim == 3)
    st_apply_3d(L, u, y, sign, stream);
  else
    throw std::invalid_argument("st_apply: dim must be 2 or 3");
  const long long faces = 2 * (L.dofs[1] * L.dofs[2] + L.dofs[0] * L.dofs[2] + (L.dim == 3 ? L.dofs[0] * L.dofs[1] : 0));
  const unsigned blocks = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((faces + 255) / 256, 148LL * 8)));
  count_launch();
  boundary_identity_kernel<<<blocks, 256, 0, stream>>>(L.dim, L.dim == 3 ? L.zbc : 3, L.dofs[0], L.dofs[1], L.dofs[2], L.n_space, L.F, f, u, y);
}
}  // namespace

void st_apply(const DevLevel& L, const double* u, double* y, cudaStream_t stream) { run(L, nullptr, u, y, stream); }

namespace {
// y_f += sign * sum_g CM[f][g] (M u_g) + CA[f][g] (A u_g): the temporal
// combination of the reference's apply (space_time_operator.cpp:59-89);
// zero coefficients are skipped (uniform branch)
__global__ void wide_combine_kernel(int F, long long n_space, double sign, const double* __restrict__ cm,
                                    const double* __restrict__ ca, const double* __restrict__ mu,
                                    const double* __restrict__ au, double* __restrict__ y) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n_space;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    for (int f = 0; f < F; ++f) {
      double s = 0.0;
      for (int g = 0; g < F; ++g) {
        const double a = __ldg(cm + f * F + g), b = __ldg(ca + f * F + g);
        if (a != 0.0) s = fma(a, __ldg(mu + g * n_space + i), s);
        if (b != 0.0) s = fma(b, __ldg(au + g * n_space + i), s);
      }
      y[f * n_space + i] += sign * s;
    }
}
}  // namespace

void st_apply_wide(const DevLevel& L, const DevLevel& mass, const DevLevel& stiff, const double* cm, const double* ca,
                   const double* f, const double* u, double* y, double* mu, double* au, cudaStream_t stream) {
  const long long ns = L.n_space;
  for (int g = 0; g < L.F; ++g) {
    run(mass, nullptr, u + g * ns, mu + g * ns, stream);
    run(stiff, nullptr, u + g * ns, au + g * ns, stream);
  }
  if (f) {
    vec_copy(y, f, L.n_dofs, stream);
    if (L.dim == 3 && !(L.zbc & 1)) plane_fill(y, L.F, L.n_space, 0, L.dofs[0] * L.dofs[1], 0.0, stream);
  } else {
    cudaMemsetAsync(y, 0, sizeof(double) * L.n_dofs, stream);
  }
  const unsigned grid = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((ns + 255) / 256, 148LL * 8)));
  count_launch();
  wide_combine_kernel<<<grid, 256, 0, stream>>>(L.F, ns, f ? -1.0 : 1.0, cm, ca, mu, au, y);
  const long long faces = 2 * (L.dofs[1] * L.dofs[2] + L.dofs[0] * L.dofs[2] + (L.dim == 3 ? L.dofs[0] * L.dofs[1] : 0));
  const unsigned blocks = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((faces + 255) / 256, 148LL * 8)));
  count_launch();
  boundary_identity_kernel<<<blocks, 256, 0, stream>>>(L.dim, L.dim == 3 ? L.zbc : 3, L.dofs[0], L.dofs[1], L.dofs[2],
                                                       L.n_space, L.F, f, u, y);
}
void st_zero_boundary(const DevLevel& L, double* v, cudaStream_t stream) {
  const long long faces = 2 * (L.dofs[1] * L.dofs[2] + L.dofs[0] * L.dofs[2] + (L.dim == 3 ? L.dofs[0] * L.dofs[1] : 0));
  const unsigned blocks = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((faces + 255) / 256, 148LL * 8)));
  count_launch();
  boundary_identity_kernel<<<blocks, 256, 0, stream>>>(L.dim, L.dim == 3 ? L.zbc : 3, L.dofs[0], L.dofs[1], L.dofs[2], L.n_space, L.F, v, v, v);
}
void st_residual(const DevLevel& L, const double* f, const double* u, double* r, cudaStream_t stream) {
  run(L, f, u, r, stream);
}

}  // namespace stmgb
