// Slab right-hand side and state transfer support on the device
// (reference: SpaceTimeOperator::assemble_rhs / extract_final,
// space_time_operator.cpp:138-248; interpolate, spatial_operator.cpp:437-449).
// The nodal interpolant of the known source / initial data is evaluated at
// the Q_p support points (Gauss-Lobatto nodes of the d-linear cell map);
// everything else is mass/stiffness applications and vector updates issued by
// the host layer (stmg.cpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "kernels.hpp"

namespace stmgb {

namespace {

// physical position of lattice node g (any cell containing it gives the same
// point: the d-linear maps of neighbouring cells agree on shared faces)
__device__ void node_position(const DevLevel& L, const double* gl, long long g, double x[3]) {
  const long long dx = L.dofs[0], dy = L.dofs[1];
  const long long i[3] = {g % dx, (g / dx) % dy, g / (dx * dy)};
  long long c[3];
  double xi[3];
  for (int a = 0; a < 3; ++a) {
    if (a < L.dim) {
      c[a] = min(i[a] / L.p, L.cells[a] - 1);
      xi[a] = gl[i[a] - c[a] * L.p];
    } else {
      c[a] = 0;
      xi[a] = 0.0;
    }
  }
  x[0] = x[1] = x[2] = 0.0;
  if (!L.verts) {
    for (int a = 0; a < L.dim; ++a) x[a] = L.lo[a] + (static_cast<double>(c[a]) + xi[a]) * L.h[a];
    return;
  }
  const long long vx = L.cells[0] + 1, vy = L.cells[1] + 1;
  const int corners = 1 << L.dim;
  for (int s = 0; s < corners; ++s) {
    double w = 1.0;
    for (int a = 0; a < L.dim; ++a) w *= ((s >> a) & 1) ? xi[a] : 1.0 - xi[a];
    const long long vi =
        ((L.dim > 2 ? c[2] + ((s >> 2) & 1) : 0) * vy + (c[1] + ((s >> 1) & 1))) * vx + (c[0] + (s & 1));
    for (int a = 0; a < L.dim; ++a) x[a] += w * L.verts[3 * vi + a];
  }
}

// kind 0: manufactured heat source  (om cos(om t) + d om^2 sin(om t)) prod sin(om x_a)
// kind 1: manufactured wave source  (d-1) om^2 sin(om t) prod sin(om x_a)
// kind 2: Gaussian pulse exp(-|x-c|^2 / (2 w^2))
// kind 3: manufactured solution     sin(om t) prod sin(om x_a)
// kind 4: manufactured velocity     om cos(om t) prod sin(om x_a)
// (driver.cpp:265-293 with om = 2 pi frequency)
__global__ void interpolate_kernel(const __grid_constant__ DevLevel L, int kind, double om, double t, double cx,
                                   double cy, double cz, double width, bool zero_bdry, double* __restrict__ out) {
  const long long n = L.n_space;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < n;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    double x[3];
    node_position(L, L.gl, g, x);
    double v;
    if (kind == 2) {
      const double r2 = (x[0] - cx) * (x[0] - cx) + (L.dim > 1 ? (x[1] - cy) * (x[1] - cy) : 0.0) +
                        (L.dim > 2 ? (x[2] - cz) * (x[2] - cz) : 0.0);
      v = exp(-r2 / (2.0 * width * width));
    } else {
      double sp = 1.0;
      for (int a = 0; a < L.dim; ++a) sp *= sin(om * x[a]);
      if (kind == 0)
        v = (om * cos(om * t) + L.dim * om * om * sin(om * t)) * sp;
      else if (kind == 1)
        v = (L.dim - 1) * om * om * sin(om * t) * sp;
      else if (kind == 3)
        v = sin(om * t) * sp;
      else
        v = om * cos(om * t) * sp;
    }
    if (zero_bdry) {
      const long long dx = L.dofs[0], dy = L.dofs[1], dz = L.dofs[2];
      const long long ix = g % dx, iy = (g / dx) % dy, iz = g / (dx * dy);
      bool b = ix == 0 || ix == dx - 1 || iy == 0 || iy == dy - 1;
      if (L.dim > 2) b = b || (iz == 0 && (L.zbc & 1)) || (iz == dz - 1 && (L.zbc & 2));
      if (b) v = 0.0;
    }
    out[g] = v;
  }
}

}  // namespace

void interpolate_nodes(const DevLevel& L, int kind, double omega, double t, const double* centre, double width,
                       bool zero_boundary, double* out, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((L.n_space + 255) / 256, 148LL * 32)));
  count_launch();
  interpolate_kernel<<<grid, 256, 0, s>>>(L, kind, omega, t, centre ? centre[0] : 0.0, centre ? centre[1] : 0.0,
                                          centre ? centre[2] : 0.0, width, zero_boundary, out);
}

}  // namespace stmgb
