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
// kind 5: the compact pulse of shm_problem (driver.cpp:295-316), r = |x| / width:
//         exp(-r^2) (1 - r^2) for r < 1, else 0
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
    } else if (kind == 5) {
      double r2 = 0.0;
      for (int a = 0; a < L.dim; ++a) r2 += (x[a] / width) * (x[a] / width);
      v = r2 >= 1.0 ? 0.0 : exp(-r2) * (1.0 - r2);
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

// Error sample of a nodal field against the manufactured solution at the
// n_q^d Gauss points of every cell (sample_spatial_error,
// spatial_operator.cpp:526-557): out[0] += sum w |J| (u_h - u)^2,
// out[1] = max |u_h - u|. kind 3: u = sin(om t) prod sin(om x_a),
// kind 4: om cos(om t) prod sin(om x_a).
struct GaussRule {
  int n;
  double x[8], w[8];
};

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(__double_as_longlong(v)));
}

__global__ void error_kernel(const __grid_constant__ DevLevel L, const GaussRule Q, const double* __restrict__ u,
                             int kind, double om, double t, double* __restrict__ out) {
  const int dim = L.dim, n = L.n, p = L.p, nq = Q.n;
  const int nqd = dim == 3 ? nq * nq * nq : nq * nq;
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long total = n_cells * nqd;
  double l2 = 0.0, linf = 0.0;
  for (long long tt = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; tt < total;
       tt += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long cell = tt / nqd;
    const int q = static_cast<int>(tt - cell * nqd);
    const long long c[3] = {cell % L.cells[0], (cell / L.cells[0]) % L.cells[1], cell / (L.cells[0] * L.cells[1])};
    const int qi[3] = {q % nq, (q / nq) % nq, q / (nq * nq)};
    double xi[3] = {0.0, 0.0, 0.0}, wq = 1.0;
    for (int a = 0; a < dim; ++a) {
      xi[a] = Q.x[qi[a]];
      wq *= Q.w[qi[a]];
    }
    // Gauss-Lobatto Lagrange basis at xi
    double phi[3][kMaxN];
    for (int a = 0; a < 3; ++a)
      for (int j = 0; j < kMaxN; ++j) {
        double v = 1.0;
        if (a < dim && j < n) {
          for (int m = 0; m < n; ++m)
            if (m != j) v *= (xi[a] - L.gl[m]) / (L.gl[j] - L.gl[m]);
        }
        phi[a][j] = v;
      }
    const long long dx = L.dofs[0], dxy = L.dofs[0] * L.dofs[1];
    const long long base = (dim == 3 ? c[2] * p * dxy : 0) + c[1] * p * dx + c[0] * p;
    double uh = 0.0;
    const int nz = dim == 3 ? n : 1;
    for (int lz = 0; lz < nz; ++lz)
      for (int ly = 0; ly < n; ++ly)
        for (int lx = 0; lx < n; ++lx)
          uh += u[base + lz * dxy + ly * dx + lx] * phi[0][lx] * phi[1][ly] * (dim == 3 ? phi[2][lz] : 1.0);
    // position and Jacobian of the d-linear map
    double x[3] = {0.0, 0.0, 0.0}, J[3][3] = {{0.0}};
    if (!L.verts) {
      for (int a = 0; a < dim; ++a) {
        x[a] = L.lo[a] + (static_cast<double>(c[a]) + xi[a]) * L.h[a];
        J[a][a] = L.h[a];
      }
    } else {
      const long long vx = L.cells[0] + 1, vy = L.cells[1] + 1;
      const int corners = 1 << dim;
      for (int sidx = 0; sidx < corners; ++sidx) {
        const long long vi =
            ((dim > 2 ? c[2] + ((sidx >> 2) & 1) : 0) * vy + (c[1] + ((sidx >> 1) & 1))) * vx + (c[0] + (sidx & 1));
        double w = 1.0, dw[3];
        for (int a = 0; a < dim; ++a) w *= ((sidx >> a) & 1) ? xi[a] : 1.0 - xi[a];
        for (int b = 0; b < dim; ++b) {
          double d = 1.0;
          for (int a = 0; a < dim; ++a) d *= a == b ? (((sidx >> a) & 1) ? 1.0 : -1.0) : (((sidx >> a) & 1) ? xi[a] : 1.0 - xi[a]);
          dw[b] = d;
        }
        for (int a = 0; a < dim; ++a) {
          const double X = L.verts[3 * vi + a];
          x[a] += w * X;
          for (int b = 0; b < dim; ++b) J[a][b] += dw[b] * X;
        }
      }
    }
    double det;
    if (dim == 2)
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    else
      det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    double sp = 1.0;
    for (int a = 0; a < dim; ++a) sp *= sin(om * x[a]);
    const double ex = kind == 3 ? sin(om * t) * sp : om * cos(om * t) * sp;
    const double d = uh - ex;
    l2 += wq * det * d * d;
    linf = fmax(linf, fabs(d));
  }
  for (int o = 16; o > 0; o >>= 1) {
    l2 += __shfl_down_sync(0xffffffffu, l2, o);
    linf = fmax(linf, __shfl_down_sync(0xffffffffu, linf, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, l2);
    atomic_max_nonneg(out + 1, linf);
  }
}

// evaluate_fe (spatial_operator.cpp:451-473) of n_fields nodal fields
// (field stride fstride) at located points: out[p * n_fields + f]
__global__ void probe_kernel(const __grid_constant__ DevLevel L, const double* __restrict__ u, int n_fields,
                             long long fstride, int n_probes, const long long* __restrict__ cells,
                             const double* __restrict__ xis, double* __restrict__ out) {
  const int tt = blockIdx.x * blockDim.x + threadIdx.x;
  if (tt >= n_probes * n_fields) return;
  const int pr = tt / n_fields, f = tt - pr * n_fields;
  const int dim = L.dim, n = L.n, p = L.p;
  const long long cell = cells[pr];
  const long long c[3] = {cell % L.cells[0], (cell / L.cells[0]) % L.cells[1], cell / (L.cells[0] * L.cells[1])};
  double phi[3][kMaxN];
  for (int a = 0; a < 3; ++a)
    for (int j = 0; j < kMaxN; ++j) {
      double v = 1.0;
      if (a < dim && j < n)
        for (int m = 0; m < n; ++m)
          if (m != j) v *= (xis[3 * pr + a] - L.gl[m]) / (L.gl[j] - L.gl[m]);
      phi[a][j] = v;
    }
  const long long dx = L.dofs[0], dxy = L.dofs[0] * L.dofs[1];
  const long long base = f * fstride + (dim == 3 ? c[2] * p * dxy : 0) + c[1] * p * dx + c[0] * p;
  double s = 0.0;
  const int nz = dim == 3 ? n : 1;
  for (int lz = 0; lz < nz; ++lz)
    for (int ly = 0; ly < n; ++ly)
      for (int lx = 0; lx < n; ++lx)
        s += u[base + lz * dxy + ly * dx + lx] * phi[0][lx] * phi[1][ly] * (dim == 3 ? phi[2][lz] : 1.0);
  out[tt] = s;
}

}  // namespace

void probe_fields(const DevLevel& L, const double* u, int n_fields, long long fstride, int n_probes,
                  const long long* d_cells, const double* d_xi, double* d_out, cudaStream_t s) {
  const int total = n_probes * n_fields;
  if (total == 0) return;
  count_launch();
  probe_kernel<<<(total + 127) / 128, 128, 0, s>>>(L, u, n_fields, fstride, n_probes, d_cells, d_xi, d_out);
}

void spatial_error(const DevLevel& L, const double* u, int n_q, const double* qx, const double* qw, int kind,
                   double omega, double t, double* out, cudaStream_t s) {
  GaussRule Q{};
  Q.n = n_q;
  for (int i = 0; i < n_q && i < 8; ++i) {
    Q.x[i] = qx[i];
    Q.w[i] = qw[i];
  }
  const long long n_cells = L.cells[0] * L.cells[1] * L.cells[2];
  const long long total = n_cells * (L.dim == 3 ? n_q * n_q * n_q : n_q * n_q);
  const unsigned grid = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 148LL * 16)));
  count_launch();
  error_kernel<<<grid, 256, 0, s>>>(L, Q, u, kind, omega, t, out);
}

void interpolate_nodes(const DevLevel& L, int kind, double omega, double t, const double* centre, double width,
                       bool zero_boundary, double* out, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((L.n_space + 255) / 256, 148LL * 32)));
  count_launch();
  interpolate_kernel<<<grid, 256, 0, s>>>(L, kind, omega, t, centre ? centre[0] : 0.0, centre ? centre[1] : 0.0,
                                          centre ? centre[2] : 0.0, width, zero_boundary, out);
}

}  // namespace stmgb
