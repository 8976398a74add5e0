// Cell-wise space-time additive Schwarz smoother (reference: ASMSmoother,
// asm_smoother.cpp:7-78). The reference extracts, per (step, cell) block T,
// the restriction B_T = R_T S R_T^T of the assembled slab matrix and LU-solves
// it. Every such block has the Kronecker form
//     B_T = T_M (x) M_T + T_A (x) A_T           (interior dofs; identity on
//                                                 Dirichlet dofs)
// with the n_t x n_t diagonal temporal blocks T_M, T_A of the slab operator
// (space_time_operator.cpp:269-317) and the restricted GLOBAL spatial mass and
// stiffness matrices M_T, A_T. With the generalised eigen-decomposition
// A_T X = M_T X Lambda, X^T M_T X = I (fast diagonalisation of the block),
//     B_T^-1 = (I (x) X) (T_M (x) I + T_A (x) Lambda)^-1 (I (x) X^T),
// i.e. two m x m products per temporal field and one n_t x n_t solve per
// eigenvalue -- exact (to rounding) for every cell, including perturbed
// cells and heterogeneous coefficients, where a 1D tensor-product
// diagonalisation would only approximate B_T. X is stored per cell (m^2
// doubles), shared by all S steps of the slab.
//
// Setup (restricted matrices by probing the matrix-free operator, Cholesky
// reduction to standard form, batched symmetric eigensolver, back transform)
// lives here too; the eigensolver itself is cuSOLVER's batched syev.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace stmgb {

namespace {

__device__ __forceinline__ void cell_coords(long long cell, const long long* cells, long long& cx, long long& cy,
                                            long long& cz) {
  cx = cell % cells[0];
  cy = (cell / cells[0]) % cells[1];
  cz = cell / (cells[0] * cells[1]);
}

// local dof l of a cell -> global lattice index, boundary flag, multiplicity
struct LocalDof {
  long long g;
  bool bdry;
  double mult;
};
__device__ __forceinline__ LocalDof local_dof(const DevASM& A, long long cx, long long cy, long long cz, int l) {
  const int n = A.n;
  const int lx = l % n, ly = (l / n) % n, lz = A.dim == 3 ? l / (n * n) : 0;
  const long long gx = cx * A.p + lx, gy = cy * A.p + ly, gz = cz * A.p + lz;
  LocalDof d;
  d.g = (gz * A.dofs[1] + gy) * A.dofs[0] + gx;
  // slab z faces are Dirichlet only where physical (A.zbc); interface planes
  // are shared with the neighbouring slab's cells
  const bool zlo = gz == 0 && (A.zbc & 1), zhi = gz == A.dofs[2] - 1 && (A.zbc & 2);
  d.bdry = gx == 0 || gx == A.dofs[0] - 1 || (A.dim > 1 && (gy == 0 || gy == A.dofs[1] - 1)) ||
           (A.dim > 2 && (zlo || zhi));
  // number of cells containing the dof (asm_smoother.cpp:45-49)
  // (gx % p == 0 exactly when the local index is a cell vertex: no 64-bit
  // modulo on the hot path)
  double m = 1.0;
  if ((lx == 0 || lx == A.p) && gx > 0 && gx < A.dofs[0] - 1) m *= 2.0;
  if (A.dim > 1 && (ly == 0 || ly == A.p) && gy > 0 && gy < A.dofs[1] - 1) m *= 2.0;
  if (A.dim > 2 && (lz == 0 || lz == A.p) && !zlo && !zhi) m *= 2.0;
  d.mult = m;
  return d;
}

// solve (TM + lam TA) x = b for n_t <= 4, partial pivoting, fully unrolled so
// everything stays in registers (padded to 4 with an identity block)
__device__ __forceinline__ void small_solve(const double* TM, const double* TA, double lam, int nt, double* b) {
  double a[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) a[i][j] = (i < nt && j < nt) ? fma(lam, TA[i * nt + j], TM[i * nt + j]) : (i == j);
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

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
// bounded wait: a copy that never lands traps instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  for (long long spin = 0; !mbar_try_wait(bar, phase); ++spin)
    if (spin > (1LL << 28)) __trap();
}
// 1D TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Small cell blocks (m <= 32: 2D Q1-Q4, 3D Q1-Q2): one WARP per cell, no
// CTA barriers. Lane a < m owns local dof a. Per warp, shared memory holds
// the cell's X (row-major, odd row stride, so row and column reads are both
// conflict-free) and the residual / eigen-coefficient rows, read back as
// warp-wide broadcasts:
//   hat r = X^T r  (lane e: X row reads)
//   hat z_e = (T_M + lam_e T_A)^-1 hat r_e per step (pivoted n_t x n_t solve)
//   z = X hat z    (lane a: X column reads)
// then the weighted scatter-add (Dirichlet rows: w r).
// X block rounded up to 32 bytes so the row buffers (read as double4) and
// every warp's slice stay 32-byte aligned
template <int M>
constexpr int warp_x_doubles() {
  return (M * (M | 1) + 3) & ~3;
}
template <int M>
constexpr int warp_smem_doubles() {
  return warp_x_doubles<M>() + 16 * M;
}

template <int M, int NT>
__global__ void __launch_bounds__(256, 3) asm_apply_warp_kernel(const __grid_constant__ DevASM A,
                                                             const double* __restrict__ r, double* __restrict__ z,
                                                             double scale) {
  static_assert(M <= 32, "one lane per local dof");
  constexpr int LD = M | 1, WS = warp_smem_doubles<M>();
  extern __shared__ __align__(16) double wsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* X = wsm + warp * WS;
  double* rb = X + warp_x_doubles<M>();  // [M][8]
  double* hb = rb + 8 * M;  // [M][8]
  const int ncol = A.S * NT;
  const bool hi = ncol > 4;
  const unsigned cxn = static_cast<unsigned>(A.cells[0]), cyn = static_cast<unsigned>(A.cells[1]);
  const long long stride = static_cast<long long>(gridDim.x) * 8;
  for (long long pos = static_cast<long long>(blockIdx.x) * 8 + warp; pos < A.n_list; pos += stride) {
    const unsigned ci = static_cast<unsigned>(A.list ? A.list[pos] : pos);
    LocalDof d{};
    double rr[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) rr[c] = 0.0;
    const double* Xg = A.X + pos * A.xs;
    {
      // all of the lane's record loads in flight before any shared store
      constexpr int NX = (M * M + 31) / 32;
      double xv[NX];
#pragma unroll
      for (int k = 0; k < NX; ++k) {
        const int i = lane + 32 * k;
        xv[k] = i < M * M ? __ldg(Xg + i) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < NX; ++k) {
        const int i = lane + 32 * k;
        if (i < M * M) X[(i / M) * LD + (i % M)] = xv[k];
      }
    }
    if (lane < M) {
      d = local_dof(A, ci % cxn, (ci / cxn) % cyn, ci / (cxn * cyn), lane);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < ncol) rr[c] = __ldg(r + static_cast<long long>(c) * A.n_space + d.g);
#pragma unroll
      for (int c = 0; c < 8; c += 2) *reinterpret_cast<double2*>(rb + lane * 8 + c) = make_double2(rr[c], rr[c + 1]);
    }
    const double lam = lane < M ? __ldg(A.lam + pos * M + lane) : 0.0;
    __syncwarp();
    if (lane < M) {
      // hat r (lane e)
      double h[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) h[c] = 0.0;
      if (hi) {
#pragma unroll 3
        for (int a = 0; a < M; ++a) {
          const double x = X[a * LD + lane];
          const double4 r0 = *reinterpret_cast<const double4*>(rb + a * 8);
          const double4 r1 = *reinterpret_cast<const double4*>(rb + a * 8 + 4);
          h[0] = fma(x, r0.x, h[0]);
          h[1] = fma(x, r0.y, h[1]);
          h[2] = fma(x, r0.z, h[2]);
          h[3] = fma(x, r0.w, h[3]);
          h[4] = fma(x, r1.x, h[4]);
          h[5] = fma(x, r1.y, h[5]);
          h[6] = fma(x, r1.z, h[6]);
          h[7] = fma(x, r1.w, h[7]);
        }
      } else {
        // <= 4 columns: even / odd rows into separate accumulators (two
        // independent FMA chains per column), folded after the loop
#pragma unroll 3
        for (int a = 0; a < M - 1; a += 2) {
          const double x0 = X[a * LD + lane], x1 = X[(a + 1) * LD + lane];
          const double4 r0 = *reinterpret_cast<const double4*>(rb + a * 8);
          const double4 r1 = *reinterpret_cast<const double4*>(rb + (a + 1) * 8);
          h[0] = fma(x0, r0.x, h[0]);
          h[1] = fma(x0, r0.y, h[1]);
          h[2] = fma(x0, r0.z, h[2]);
          h[3] = fma(x0, r0.w, h[3]);
          h[4] = fma(x1, r1.x, h[4]);
          h[5] = fma(x1, r1.y, h[5]);
          h[6] = fma(x1, r1.z, h[6]);
          h[7] = fma(x1, r1.w, h[7]);
        }
        if (M % 2 == 1) {
          const double x = X[(M - 1) * LD + lane];
          const double4 r0 = *reinterpret_cast<const double4*>(rb + (M - 1) * 8);
          h[0] = fma(x, r0.x, h[0]);
          h[1] = fma(x, r0.y, h[1]);
          h[2] = fma(x, r0.z, h[2]);
          h[3] = fma(x, r0.w, h[3]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          h[c] += h[c + 4];
          h[c + 4] = 0.0;
        }
      }
#pragma unroll
      for (int st = 0; st < 8 / NT; ++st) {
        if (st >= A.S) break;
        double b4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < NT; ++i) b4[i] = h[st * NT + i];
        small_solve(A.TM, A.TA, lam, NT, b4);
#pragma unroll
        for (int i = 0; i < NT; ++i) h[st * NT + i] = b4[i];
      }
#pragma unroll
      for (int c = 0; c < 8; c += 2) *reinterpret_cast<double2*>(hb + lane * 8 + c) = make_double2(h[c], h[c + 1]);
    }
    __syncwarp();
    if (lane < M) {
      // z (lane a)
      double o[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) o[c] = 0.0;
      if (hi) {
#pragma unroll 3
        for (int e = 0; e < M; ++e) {
          const double x = X[lane * LD + e];
          const double4 h0 = *reinterpret_cast<const double4*>(hb + e * 8);
          const double4 h1 = *reinterpret_cast<const double4*>(hb + e * 8 + 4);
          o[0] = fma(x, h0.x, o[0]);
          o[1] = fma(x, h0.y, o[1]);
          o[2] = fma(x, h0.z, o[2]);
          o[3] = fma(x, h0.w, o[3]);
          o[4] = fma(x, h1.x, o[4]);
          o[5] = fma(x, h1.y, o[5]);
          o[6] = fma(x, h1.z, o[6]);
          o[7] = fma(x, h1.w, o[7]);
        }
      } else {
#pragma unroll 3
        for (int e = 0; e < M - 1; e += 2) {
          const double x0 = X[lane * LD + e], x1 = X[lane * LD + e + 1];
          const double4 h0 = *reinterpret_cast<const double4*>(hb + e * 8);
          const double4 h1 = *reinterpret_cast<const double4*>(hb + (e + 1) * 8);
          o[0] = fma(x0, h0.x, o[0]);
          o[1] = fma(x0, h0.y, o[1]);
          o[2] = fma(x0, h0.z, o[2]);
          o[3] = fma(x0, h0.w, o[3]);
          o[4] = fma(x1, h1.x, o[4]);
          o[5] = fma(x1, h1.y, o[5]);
          o[6] = fma(x1, h1.z, o[6]);
          o[7] = fma(x1, h1.w, o[7]);
        }
        if (M % 2 == 1) {
          const double x = X[lane * LD + M - 1];
          const double4 h0 = *reinterpret_cast<const double4*>(hb + (M - 1) * 8);
          o[0] = fma(x, h0.x, o[0]);
          o[1] = fma(x, h0.y, o[1]);
          o[2] = fma(x, h0.z, o[2]);
          o[3] = fma(x, h0.w, o[3]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          o[c] += o[c + 4];
          o[c + 4] = 0.0;
        }
      }
      const double w = scale / d.mult;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < ncol) atomicAdd(z + static_cast<long long>(c) * A.n_space + d.g, (d.bdry ? rr[c] : o[c]) * w);
    }
    __syncwarp();
  }
}

// Tensor-core variant for m = 64 (3D Q3 cells): both block products run on
// the FP64 tensor cores (mma.sync.m8n8k4.f64), all S*n_t step columns of the
// slab batched into the 8 MMA columns. X is stored XOR-swizzled per cell
// (swz64) so the A-fragment loads of both X^T r and X z are bank-conflict
// free. 8 warps: warp w owns rows [8w, 8w+8) of each product; the k loop is
// split into two independent accumulator chains.
__host__ __device__ __forceinline__ int swz64(int a, int e) { return a * 64 + (e ^ ((a & 7) << 2)); }
// record layout of 64-dof cells for the DFMA kernel: column XOR (row & 15),
// conflict-free row and column reads of 64-bit words

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(256) asm_apply_mma_kernel(const __grid_constant__ DevASM A,
                                                            const double* __restrict__ r, double* __restrict__ z,
                                                            double scale) {
  constexpr int M = 64, XS = M * M;
  extern __shared__ __align__(128) double sm[];
  double* Xb0 = sm;
  double* Xb1 = sm + XS;
  double* rs = Xb1 + XS;  // [M][8] block residual, columns s*NT+i
  double* hs = rs + 8 * M;  // [M][8] hat r / hat z
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(hs + 8 * M);
  const long long n_pos = A.n_list;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ncol = A.S * NT;  // <= 8
  constexpr unsigned XBYTES = static_cast<unsigned>(XS * sizeof(double));
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long pos = blockIdx.x;
  if (t == 0 && pos < n_pos) {
    mbar_expect_tx(&bar[0], XBYTES);
    bulk_g2s(Xb0, A.X + pos * A.xs, XBYTES, &bar[0]);
  }
  unsigned ph0 = 0, ph1 = 0;
  int buf = 0;
  const unsigned cxn = static_cast<unsigned>(A.cells[0]), cyn = static_cast<unsigned>(A.cells[1]);
  struct Col8 {
    double v[8];
  };
  // block residual of list position q for local dof t (columns s*NT + i)
  auto gather = [&](long long q) {
    Col8 o;
#pragma unroll
    for (int c = 0; c < 8; ++c) o.v[c] = 0.0;
    if (t < M) {
      const unsigned ci = static_cast<unsigned>(A.list ? A.list[q] : q);
      const LocalDof d = local_dof(A, ci % cxn, (ci / cxn) % cyn, ci / (cxn * cyn), t);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < ncol) o.v[c] = __ldg(r + static_cast<long long>(c) * A.n_space + d.g);
    }
    return o;
  };
  Col8 rnext;
  for (; pos < n_pos; pos += gridDim.x) {
    const long long next = pos + gridDim.x;
    if (t == 0 && next < n_pos) {
      fence_proxy_async();
      unsigned long long* b = &bar[buf ^ 1];
      mbar_expect_tx(b, XBYTES);
      bulk_g2s(buf ? Xb0 : Xb1, A.X + next * A.xs, XBYTES, b);
    }
    const unsigned cidx = static_cast<unsigned>(A.list ? A.list[pos] : pos);
    const long long cx = cidx % cxn, cy = (cidx / cxn) % cyn, cz = cidx / (cxn * cyn);
    // the block residual of this cell was prefetched into registers during
    // the previous iteration (first cell: load now); stage it, then prefetch
    // the next cell's so its gather latency hides behind this cell's MMAs
    if (pos == blockIdx.x) rnext = gather(pos);
    if (t < M) {
#pragma unroll
      for (int c = 0; c < 8; ++c) rs[t * 8 + c] = c < ncol ? rnext.v[c] : 0.0;
    }
    if (next < n_pos) rnext = gather(next);
    if (buf == 0) {
      mbar_wait(&bar[0], ph0);
      ph0 ^= 1;
    } else {
      mbar_wait(&bar[1], ph1);
      ph1 ^= 1;
    }
    __syncthreads();
    const double* Xs = buf ? Xb1 : Xb0;
    const int row = warp * 8 + (lane >> 2), col = (lane & 3) * 2;
    {
      // hat r (e x 8) = X^T r: A[row=e][k=a] = X[a][e]
      double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
      for (int kt = 0; kt < M / 4; kt += 2) {
        const int a0 = kt * 4 + (lane & 3), a1 = a0 + 4;
        dmma(d00, d01, Xs[swz64(a0, row)], rs[a0 * 8 + (lane >> 2)]);
        dmma(d10, d11, Xs[swz64(a1, row)], rs[a1 * 8 + (lane >> 2)]);
      }
      // (T_M + lam_e T_A)^-1 per eigen-index e = row and step, solved in
      // registers: the 4 lanes holding row e exchange its 8 columns
      double v[8];
      const double c0 = d00 + d10, c1 = d01 + d11;
      const int grp = lane & ~3;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[2 * j] = __shfl_sync(0xffffffffu, c0, grp | j);
        v[2 * j + 1] = __shfl_sync(0xffffffffu, c1, grp | j);
      }
      const double lam = A.lam[pos * M + row];
      double out0 = 0.0, out1 = 0.0;
#pragma unroll
      for (int s = 0; s < 8 / NT; ++s) {
        if (s >= A.S) break;
        double b4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < NT; ++i) b4[i] = v[s * NT + i];
        small_solve(A.TM, A.TA, lam, NT, b4);
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          if (s * NT + i == col) out0 = b4[i];
          if (s * NT + i == col + 1) out1 = b4[i];
        }
      }
      *reinterpret_cast<double2*>(hs + row * 8 + col) = make_double2(out0, out1);
    }
    __syncthreads();
    {
      // z_T (a x 8) = X hat z: A[row=a][k=e] = X[a][e]
      double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
      for (int kt = 0; kt < M / 4; kt += 2) {
        const int e0 = kt * 4 + (lane & 3), e1 = e0 + 4;
        dmma(d00, d01, Xs[swz64(row, e0)], hs[e0 * 8 + (lane >> 2)]);
        dmma(d10, d11, Xs[swz64(row, e1)], hs[e1 * 8 + (lane >> 2)]);
      }
      const LocalDof d = local_dof(A, cx, cy, cz, row);
      const double w = scale / d.mult;
      const double v0 = d.bdry ? rs[row * 8 + col] : d00 + d10;
      const double v1 = d.bdry ? rs[row * 8 + col + 1] : d01 + d11;
      if (col < ncol) atomicAdd(z + static_cast<long long>(col) * A.n_space + d.g, v0 * w);
      if (col + 1 < ncol) atomicAdd(z + static_cast<long long>(col + 1) * A.n_space + d.g, v1 * w);
    }
    __syncthreads();
    buf ^= 1;
  }
}

// Tensor-core variant for 24 < m <= 32 (3D Q2 cells, m = 27: the exact cells
// of a Cartesian level, e.g. coefficient-jump neighbourhoods; 2D Q4, m = 25).
// One WARP per cell, as in the DFMA warp kernel above, but both block
// products run as mma.sync.m8n8k4.f64 over the block padded to 32 rows (four
// 8-row tiles, k in steps of 4 up to 28; entries past m predicated to zero),
// and the per-row work happens in the lane-per-dof layout between them:
//   stage   lane a: gather r_a (local dof a), P-mix into slots (A.tdiag)
//   MMA 1   hat r = X^T r            (D fragments -> shared, transposed)
//   row     lane e: (B + lam_e)^-1 on the slot pairs, then Q back to the
//           time columns (Q commutes with X); pivoted solves without tdiag
//   MMA 2   z_T = X hat z            (D fragments -> shared, transposed)
//   scatter lane a: weighted atomics with its own local dof
// X arrives by one TMA bulk copy per cell into the warp's double buffer; 4
// independent warps per CTA, no CTA barriers in the loop.
// With A.tdiag (the temporal blocks are real-block-diagonalisable, see
// temporal_block_diagonalise) the padded kernels replace the per-lane pivoted
// solves by the m = 64 kernel's scheme: P mixes the residual columns at the
// staging, the lane holding slot pair (2j, 2j+1) of eigen-row e applies the
// 1x1 / 2x2 (B + lam_e)^-1, and Q mixes the slots of each output row after a
// 4-lane shuffle; Dirichlet rows add w r straight from the staging threads.
__device__ __forceinline__ void tdiag_scale(const DevASM& A, int j, double lam, double v0, double v1, double& o0,
                                            double& o1) {
  const int kd = A.kind[j];
  const double a0 = A.s0[j], a1 = A.s1[j];
  const double p0 = a0 + lam, p1 = a1 + lam;
  const double m00 = kd ? p0 : p1, m11 = p0, m01 = kd ? -a1 : 0.0, m10 = kd ? a1 : 0.0;
  const double inv = 1.0 / (kd ? fma(p0, p0, a1 * a1) : p0 * p1);
  o0 = fma(m00, v0, m01 * v1) * inv;
  o1 = fma(m10, v0, m11 * v1) * inv;
}
// Ps / Qs: A.P / A.Q copied to shared memory (param-space tables read inside a
// persistent loop get hoisted into registers and spill)
__device__ __forceinline__ void tdiag_qmix(const double* Qs, int lane, double v0, double v1, double& o0, double& o1) {
  double v[8];
  const int grp = lane & ~3, c0 = 2 * (lane & 3);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __shfl_sync(0xffffffffu, v0, grp | i);
    v[2 * i + 1] = __shfl_sync(0xffffffffu, v1, grp | i);
  }
  o0 = 0.0;
  o1 = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    o0 = fma(Qs[c0 * 8 + k], v[k], o0);
    o1 = fma(Qs[(c0 + 1) * 8 + k], v[k], o1);
  }
}
// residual row of one local dof, P-transformed when A.tdiag (slots), raw
// otherwise; a Dirichlet row under tdiag adds w r to z here
__device__ __forceinline__ void stage_row(const DevASM& A, const double* Ps, const double* rn, long long g, bool bdry,
                                          double mult, double scale, int ncol, double* z, double* dst, int sw = 0) {
  double tr[8];
  if (A.tdiag) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) s = fma(Ps[k * 8 + c], rn[c], s);
      tr[k] = s;
    }
    if (bdry) {
      const double w = scale / mult;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < ncol) atomicAdd(z + static_cast<long long>(c) * A.n_space + g, rn[c] * w);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) tr[k] = rn[k];
  }
#pragma unroll
  for (int c = 0; c < 8; c += 2) *reinterpret_cast<double2*>(dst + (c ^ sw)) = make_double2(tr[c], tr[c + 1]);
}

// records of the 25/27-dof tensor-core kernel are stored with row pitch 28
// (DevASM::x_layout == 2): the A-fragment loads X[a][e] (4 k-rows x 4 m-rows
// per half-warp) then fall in 16 distinct 64-bit banks in both products; the
// contiguous pitch 27 was 2-way conflicted (ncu: 117 M conflicts per C3 sweep)
template <int M>
constexpr int mma32_xbuf() {
  static_assert(M <= kMma32Pitch && (M * kMma32Pitch) % 2 == 0, "16-byte bulk copies");
  return M * kMma32Pitch;  // = DevASM::xs under x_layout 2
}
// rs / hs rows of 8 doubles with the columns XOR-swizzled by row bits 1-2
// (wmma_sw, even so 16-byte pairs stay whole): the B-fragment loads (4 rows x
// 4 columns per half-warp), the 16-byte row accesses of 8 lanes and the
// accumulator-pair stores are conflict-free, the per-lane scatter reads 2-way
// (pitch 12 unswizzled: 2-way / 4-way on the last two)
constexpr int kWmmaWarps = 4, kWmmaPitch = 8;
__device__ __forceinline__ int wmma_sw(int row) { return 4 * ((row >> 1) & 1) + 2 * ((row >> 2) & 1); }
template <int M>
constexpr int wmma_warp_doubles() {
  return 2 * mma32_xbuf<M>() + 2 * 32 * kWmmaPitch;
}
template <int M>
constexpr size_t mma32_smem() {
  return sizeof(double) * (128 + static_cast<size_t>(kWmmaWarps) * wmma_warp_doubles<M>()) +
         2 * kWmmaWarps * sizeof(unsigned long long);
}

template <int M, int NT>
__global__ void __launch_bounds__(32 * kWmmaWarps, 3) asm_apply_mma32_kernel(const __grid_constant__ DevASM A,
                                                                             const double* __restrict__ r,
                                                                             double* __restrict__ z, double scale) {
  static_assert(M > 24 && M <= 32, "four 8-row MMA tiles");
  constexpr int XB = mma32_xbuf<M>(), KT = (M + 3) / 4, RS = kWmmaPitch, W = kWmmaWarps;
  constexpr unsigned XBYTES = static_cast<unsigned>(XB * sizeof(double));
  static_assert(XBYTES % 16 == 0, "bulk copy size");
  extern __shared__ __align__(128) double sm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double* PQ = sm;  // A.P, A.Q
  double* X0 = sm + 128 + warp * wmma_warp_doubles<M>();
  double* X1 = X0 + XB;
  double* rs = X1 + XB;       // [32][RS] staged residual (slots)
  double* hs = rs + 32 * RS;  // [32][RS] product outputs, transposed
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + 128 + W * wmma_warp_doubles<M>()) + 2 * warp;
  PQ[t] = t < 64 ? A.P[t >> 3][t & 7] : A.Q[(t - 64) >> 3][t & 7];
  for (int i = lane; i < 2 * 32 * RS; i += 32) rs[i] = 0.0;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long n_pos = A.n_list, nsp = A.n_space;
  const long long stride = static_cast<long long>(gridDim.x) * W;
  const int ncol = A.S * NT;
  const int kl = lane & 3, n8 = lane >> 2;
  const bool own = lane < M;
  const unsigned cxn = static_cast<unsigned>(A.cells[0]), cyn = static_cast<unsigned>(A.cells[1]);
  long long pos = static_cast<long long>(blockIdx.x) * W + warp;
  if (lane == 0 && pos < n_pos) {
    mbar_expect_tx(&bar[0], XBYTES);
    bulk_g2s(X0, A.X + pos * A.xs, XBYTES, &bar[0]);
  }
  unsigned ph0 = 0, ph1 = 0;
  int buf = 0;
  // lane a's local dof, residual row and eigenvalue of list position q, loaded
  // one cell ahead so the gather latency hides behind the current cell
  LocalDof dn{0, false, 1.0};
  double rnn[8], lamn = 0.0;
  auto gather = [&](long long q) {
#pragma unroll
    for (int c = 0; c < 8; ++c) rnn[c] = 0.0;
    if (own) {
      const unsigned ci = static_cast<unsigned>(A.list ? A.list[q] : q);
      dn = local_dof(A, ci % cxn, (ci / cxn) % cyn, ci / (cxn * cyn), lane);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < ncol) rnn[c] = __ldg(r + static_cast<long long>(c) * nsp + dn.g);
      lamn = __ldg(A.lam + q * M + lane);
    }
  };
  if (pos < n_pos) gather(pos);
  for (; pos < n_pos; pos += stride) {
    const long long next = pos + stride;
    if (lane == 0 && next < n_pos) {
      fence_proxy_async();
      unsigned long long* b = &bar[buf ^ 1];
      mbar_expect_tx(b, XBYTES);
      bulk_g2s(buf ? X0 : X1, A.X + next * A.xs, XBYTES, b);
    }
    // ---- stage: lane a's residual row (gathered during the previous cell)
    const LocalDof d = dn;
    const double lam = lamn;
    double rn[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) rn[c] = rnn[c];
    if (own) stage_row(A, PQ, rn, d.g, d.bdry, d.mult, scale, ncol, z, rs + lane * RS, wmma_sw(lane));
    if (next < n_pos) gather(next);
    if (buf == 0) {
      mbar_wait(&bar[0], ph0);
      ph0 ^= 1;
    } else {
      mbar_wait(&bar[1], ph1);
      ph1 ^= 1;
    }
    __syncwarp();
    const double* Xs = buf ? X1 : X0;
    double acc[4][2];
    // ---- MMA 1: hat r (e x 8) = X^T r, A[row=e][k=a] = X[a][e]
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const int a = kt * 4 + kl;
      const double b = rs[a * RS + (n8 ^ wmma_sw(a))];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = i * 8 + n8;
        const double xa = (a < M && e < M) ? Xs[a * kMma32Pitch + e] : 0.0;
        dmma(acc[i][0], acc[i][1], xa, b);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<double2*>(hs + (i * 8 + n8) * RS + ((2 * kl) ^ wmma_sw(i * 8 + n8))) = make_double2(acc[i][0], acc[i][1]);
    __syncwarp();
    // ---- row work: lane e solves its eigen-row (slots -> time columns)
    if (own) {
      double v[8];
#pragma unroll
      for (int c = 0; c < 8; c += 2) {
        const double2 q = *reinterpret_cast<const double2*>(hs + lane * RS + (c ^ wmma_sw(lane)));
        v[c] = q.x;
        v[c + 1] = q.y;
      }
      double o[8];
      if (A.tdiag) {
        double sl[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) tdiag_scale(A, j, lam, v[2 * j], v[2 * j + 1], sl[2 * j], sl[2 * j + 1]);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          double s = 0.0;
          if (c < ncol) {
#pragma unroll
            for (int k = 0; k < 8; ++k) s = fma(PQ[64 + c * 8 + k], sl[k], s);
          }
          o[c] = s;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) o[c] = v[c];
#pragma unroll
        for (int st = 0; st < 8 / NT; ++st) {
          if (st >= A.S) break;
          double b4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int i = 0; i < NT; ++i) b4[i] = o[st * NT + i];
          small_solve(A.TM, A.TA, lam, NT, b4);
#pragma unroll
          for (int i = 0; i < NT; ++i) o[st * NT + i] = b4[i];
        }
      }
#pragma unroll
      for (int c = 0; c < 8; c += 2) *reinterpret_cast<double2*>(hs + lane * RS + (c ^ wmma_sw(lane))) = make_double2(o[c], o[c + 1]);
    }
    __syncwarp();
    // ---- MMA 2: z_T (a x 8) = X hat z, A[row=a][k=e] = X[a][e]
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const int e = kt * 4 + kl;
      const double b = hs[e * RS + (n8 ^ wmma_sw(e))];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int a = i * 8 + n8;
        const double xa = (a < M && e < M) ? Xs[a * kMma32Pitch + e] : 0.0;
        dmma(acc[i][0], acc[i][1], xa, b);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<double2*>(hs + (i * 8 + n8) * RS + ((2 * kl) ^ wmma_sw(i * 8 + n8))) = make_double2(acc[i][0], acc[i][1]);
    __syncwarp();
    // ---- scatter: lane a, weighted (Dirichlet rows: w r; under tdiag added at the staging)
    if (own) {
      const double w = scale / d.mult;
      if (!d.bdry) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < ncol) atomicAdd(z + static_cast<long long>(c) * nsp + d.g, hs[lane * RS + (c ^ wmma_sw(lane))] * w);
      } else if (!A.tdiag) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < ncol) atomicAdd(z + static_cast<long long>(c) * nsp + d.g, rn[c] * w);
      }
    }
    __syncwarp();
    buf ^= 1;
  }
}

// m = 64 smoother with the temporal solves fast-diagonalised as well
// (A.tdiag): per cell and eigen-index e the n_t x n_t solve
// (T_M + lam_e T_A)^-1 = Q (B + lam_e)^-1 P, B block-diagonal. P mixes the
// temporal columns of every residual row before the first product, the
// 1x1/2x2 scalings (B + lam_e)^-1 act on the MMA accumulator pair each lane
// already holds, and Q mixes the columns of the second product's rows (one
// 4-lane shuffle exchange) -- no pivoted small solves, no redundant lanes.
// One TMA bulk copy per cell brings X (swizzled) and its eigenvalues; the
// cell's lattice offset and Dirichlet faces come from a 16-byte meta entry,
// and the multiplicity weight of an interior dof depends only on its local
// index, so no per-dof division or index decoding is left in the loop.
// Dirichlet dofs of a block (identity rows, asm_smoother.cpp:29-33 with the
// global identity) contribute w * r directly from the gather threads.
// NBUF record buffers per CTA: the record of cell i + NBUF - 1 is requested
// while cell i is solved (prefetch distance NBUF - 1)
template <int NBUF>
constexpr size_t fd64_smem() {
  return sizeof(double) * (NBUF * static_cast<size_t>(kRec64) + 16 * 64) + 4 * sizeof(long long) +
         NBUF * sizeof(unsigned long long);
}

template <int NT, int S, int NBUF>
__global__ void __launch_bounds__(256, NBUF == 2 ? 3 : 2) asm_apply_fd64_kernel(const __grid_constant__ DevASM A,
                                                                               const double* __restrict__ r,
                                                                               double* __restrict__ z, double scale) {
  constexpr int M = 64, NCOL = NT * S, NPAIR = (NCOL + 1) / 2;
  constexpr unsigned RBYTES = static_cast<unsigned>(kRec64 * sizeof(double));
  static_assert(RBYTES % 16 == 0, "record must be a multiple of 16 bytes");
  extern __shared__ __align__(128) double sm[];
  double* rs = sm + NBUF * kRec64;  // [64][8] P-transformed residual, pair-swizzled rows
  double* hs = rs + 8 * M;          // [64][8] scaled eigen-coefficients
  long long* cinfo = reinterpret_cast<long long*>(hs + 8 * M);       // [2][2] {g0, mask} per parity
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(cinfo + 4);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const long long n_pos = A.n_list, nsp = A.n_space;
  const long long dx = A.dofs[0], dxy = A.dofs[0] * A.dofs[1];
  auto local_off = [&](int a, int& fb) {
    const int lx = a & 3, ly = (a >> 2) & 3, lz = a >> 4;
    fb = (lx == 0 ? 1 : 0) | (lx == 3 ? 2 : 0) | (ly == 0 ? 4 : 0) | (ly == 3 ? 8 : 0) | (lz == 0 ? 16 : 0) |
         (lz == 3 ? 32 : 0);
    return lz * dxy + ly * dx + lx;
  };
  // gather role (t < 64: local dof t), epilogue role (row a of the 2nd product)
  int fb_g = 0, fb_e = 0;
  const long long off_g = local_off(t & 63, fb_g);
  const int j = lane & 3, n8 = lane >> 2;
  const int row = warp * 8 + n8;  // eigen-index of product 1 / local dof of product 2
  const long long off_e = local_off(row, fb_e);
  const double w_e = scale * ldexp(1.0, -__popc(fb_e));
  // constant smem offsets of the fragment loads (see swz64 and the rs swizzle)
  const int x1e = j * 64 + (row ^ (4 * j)), x1o = j * 64 + (row ^ (16 + 4 * j));
  // B operands are loaded per half-warp (16 lanes x 8 B): rows 4kt + j and
  // 4kt + j + 2 must land in different 8-double bank halves, hence the XOR of
  // bit 2 by row bit 1 (rs: also bit 1 by row bit 2, for the gather's 16-byte
  // stores from consecutive rows)
  const int swj = ((j >> 1) & 1) << 2;
  const int r1e = j * 8 + (n8 ^ swj), r1o = j * 8 + (n8 ^ (swj | 2));
  const int h2 = j * 8 + (n8 ^ swj);
  const int hst = row * 8 + ((2 * j) ^ (((row >> 1) & 1) << 2));
  const int sw2 = row & 7;
  const int xrow = row * 64 + j;
  const int kd = A.kind[j];
  const double a0 = A.s0[j], a1 = A.s1[j];

  if (t == 0) {
#pragma unroll
    for (int b = 0; b < NBUF; ++b) mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long pos = blockIdx.x;
  if (t == 0) {
#pragma unroll
    for (int b = 0; b + 1 < NBUF; ++b) {
      const long long q = pos + static_cast<long long>(b) * gridDim.x;
      if (q < n_pos) {
        mbar_expect_tx(&bar[b], RBYTES);
        bulk_g2s(sm + b * kRec64, A.X + q * kRec64, RBYTES, &bar[b]);
      }
    }
  }
  double rn[NCOL];
  long long g0n = 0, maskn = 0;
  auto fetch = [&](long long q) {
    if (t < M) {
      const longlong2 mt = *reinterpret_cast<const longlong2*>(A.meta + 2 * q);
      g0n = mt.x;
      maskn = mt.y;
#pragma unroll
      for (int c = 0; c < NCOL; ++c) rn[c] = __ldg(r + c * nsp + g0n + off_g);
    }
  };
  if (pos < n_pos) fetch(pos);
  unsigned phase_bits = 0;  // parity of each buffer's barrier
  int buf = 0;
  for (int it = 0; pos < n_pos; pos += gridDim.x, ++it) {
    const int par = it & 1;
    const long long next = pos + gridDim.x;
    // ---- stage the residual of this cell (prefetched last iteration)
    if (t < M) {
      double tr[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double s = 0.0;
        if (k < NCOL) {
#pragma unroll
          for (int c = 0; c < NCOL; ++c) s = fma(A.P[k][c], rn[c], s);
        }
        tr[k] = s;
      }
      const int swr = (((t >> 1) & 1) << 2) | (((t >> 2) & 1) << 1);
#pragma unroll
      for (int p = 0; p < 4; ++p)
        *reinterpret_cast<double2*>(rs + t * 8 + ((2 * p) ^ swr)) = make_double2(tr[2 * p], tr[2 * p + 1]);
      if (maskn & fb_g) {
        const double w = scale * ldexp(1.0, -__popc(fb_g & ~static_cast<int>(maskn)));
#pragma unroll
        for (int c = 0; c < NCOL; ++c) atomicAdd(z + c * nsp + g0n + off_g, w * rn[c]);
      }
      if (t == 0) {
        cinfo[2 * par] = g0n;
        cinfo[2 * par + 1] = maskn;
      }
      if (next < n_pos) fetch(next);
    }
    mbar_wait(&bar[buf], (phase_bits >> buf) & 1u);
    phase_bits ^= 1u << buf;
    __syncthreads();
    // every warp is past cell it-1, so its buffer takes cell it + NBUF - 1
    {
      const int fb = buf == 0 ? NBUF - 1 : buf - 1;
      const long long q = pos + static_cast<long long>(NBUF - 1) * gridDim.x;
      if (t == 0 && q < n_pos) {
        fence_proxy_async();
        mbar_expect_tx(&bar[fb], RBYTES);
        bulk_g2s(sm + fb * kRec64, A.X + q * kRec64, RBYTES, &bar[fb]);
      }
    }
    const double* Xs = sm + buf * kRec64;
    {
      // product 1: hat r (e x slots) = X^T rs
      double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
      for (int kt = 0; kt < 16; kt += 2) {
        dmma(d00, d01, Xs[kt * 256 + x1e], rs[kt * 32 + r1e]);
        dmma(d10, d11, Xs[(kt + 1) * 256 + x1o], rs[(kt + 1) * 32 + r1o]);
      }
      const double v0 = d00 + d10, v1 = d01 + d11;
      // (B + lam_e)^-1 on slots (2j, 2j+1): two reals or one conjugate pair
      const double lam = Xs[4096 + row];
      const double p0 = a0 + lam, p1 = a1 + lam;
      const double m00 = kd ? p0 : p1, m11 = p0, m01 = kd ? -a1 : 0.0, m10 = kd ? a1 : 0.0;
      const double den = kd ? fma(p0, p0, a1 * a1) : p0 * p1;
      const double inv = 1.0 / den;
      *reinterpret_cast<double2*>(hs + hst) =
          make_double2(fma(m00, v0, m01 * v1) * inv, fma(m10, v0, m11 * v1) * inv);
    }
    __syncthreads();
    {
      // product 2: z_T (a x slots) = X hat z, then Q mixes the slots of row a
      double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
      for (int kt = 0; kt < 16; kt += 2) {
        dmma(d00, d01, Xs[xrow + 4 * (kt ^ sw2)], hs[kt * 32 + h2]);
        dmma(d10, d11, Xs[xrow + 4 * ((kt + 1) ^ sw2)], hs[(kt + 1) * 32 + h2]);
      }
      const double v0 = d00 + d10, v1 = d01 + d11;
      double v[2 * NPAIR];
      const int grp = lane & ~3;
#pragma unroll
      for (int i = 0; i < NPAIR; ++i) {
        v[2 * i] = __shfl_sync(0xffffffffu, v0, grp | i);
        v[2 * i + 1] = __shfl_sync(0xffffffffu, v1, grp | i);
      }
      const long long g0 = cinfo[2 * par];
      const int mask = static_cast<int>(cinfo[2 * par + 1]);
      if (j < NPAIR && !(mask & fb_e)) {
        const int c0 = 2 * j, c1 = 2 * j + 1;
        double o0 = 0.0, o1 = 0.0;
#pragma unroll
        for (int k = 0; k < NCOL; ++k) {
          o0 = fma(A.Q[c0][k], v[k], o0);
          if (c1 < NCOL) o1 = fma(A.Q[c1][k], v[k], o1);
        }
        double* zp = z + g0 + off_e;
        atomicAdd(zp + c0 * nsp, o0 * w_e);
        if (c1 < NCOL) atomicAdd(zp + c1 * nsp, o1 * w_e);
      }
    }
    buf = buf + 1 == NBUF ? 0 : buf + 1;
  }
}

// Tensor-core variant for 3D Q4 exact cells (m = 125, padded to 128 rows):
// one CTA of 16 warps per cell (persistent), warp w owns rows [8w, 8w+8) of
// both products, mma.sync.m8n8k4.f64 over k in 32 steps of 4 (entries past m
// predicated to zero). The A fragments come straight from global memory --
// product 1 reads X[a][e] as 4 row segments of 64 bytes per warp and k step
// (HBM stream, all 32 loads of a warp in flight before the first MMA),
// product 2 reads X[a][e] along rows, 32-byte sectors, from L2 where the first
// product just left the record. r / hat z are shared-memory B fragments; the
// n_t x n_t solves are the pivoted small_solve, the next cell's residual is
// gathered into registers while this cell is solved.
constexpr int kLargeMmaPitch = 12;
template <int M, int NT>
__global__ void __launch_bounds__(((M + 7) / 8) * 32, 1) asm_apply_large_mma_kernel(const __grid_constant__ DevASM A,
                                                                                   const double* __restrict__ r,
                                                                                   double* __restrict__ z,
                                                                                   double scale) {
  constexpr int NW = (M + 7) / 8, MP = NW * 8, KT = (M + 3) / 4, KH = (KT + 1) / 2;
  // row pitch 12: the B-fragment rows 4kt + kl of a half-warp fall in distinct banks
  constexpr int RS = kLargeMmaPitch;
  static_assert(KT * 4 <= MP, "k rows inside the padded block");
  extern __shared__ __align__(16) double lsm[];
  double* rs = lsm;            // [MP][RS] block residual (rows >= M stay zero)
  double* hs = rs + RS * MP;  // [MP][RS] hat z
  double* PQ = hs + RS * MP;  // A.P, A.Q
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ncol = A.S * NT;
  for (int i = t; i < 2 * RS * MP; i += NW * 32) lsm[i] = 0.0;
  if (t < 128) PQ[t] = t < 64 ? A.P[t >> 3][t & 7] : A.Q[(t - 64) >> 3][t & 7];
  const unsigned cxn = static_cast<unsigned>(A.cells[0]), cyn = static_cast<unsigned>(A.cells[1]);
  const int row = warp * 8 + (lane >> 2), col = (lane & 3) * 2, kl = lane & 3, n8 = lane >> 2;
  const bool row_ok = row < M;
  double rn[8];
  LocalDof dn{0, false, 1.0};
  auto gather = [&](long long q) {
#pragma unroll
    for (int c = 0; c < 8; ++c) rn[c] = 0.0;
    if (t < M) {
      const unsigned ci = static_cast<unsigned>(A.list ? A.list[q] : q);
      dn = local_dof(A, ci % cxn, (ci / cxn) % cyn, ci / (cxn * cyn), t);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < ncol) rn[c] = __ldg(r + static_cast<long long>(c) * A.n_space + dn.g);
    }
  };
  if (blockIdx.x < A.n_list) gather(blockIdx.x);
  __syncthreads();
  for (long long pos = blockIdx.x; pos < A.n_list; pos += gridDim.x) {
    const unsigned ci = static_cast<unsigned>(A.list ? A.list[pos] : pos);
    const long long cx = ci % cxn, cy = (ci / cxn) % cyn, cz = ci / (cxn * cyn);
    const double* X = A.X + pos * A.xs;
    // stage this cell's residual, put the next cell's gather in flight, then
    // the 32 A-fragment loads of product 1
    if (t < M) stage_row(A, PQ, rn, dn.g, dn.bdry, dn.mult, scale, ncol, z, rs + t * RS);
    if (pos + gridDim.x < A.n_list) gather(pos + gridDim.x);
    // (two halves of KH loads each: all 32 in flight spill at 128 registers)
    double xa[KH];
#pragma unroll
    for (int kt = 0; kt < KH; ++kt) {
      const int a = kt * 4 + kl;
      xa[kt] = (row_ok && a < M) ? __ldg(X + a * M + row) : 0.0;
    }
    const double lam = row_ok ? __ldg(A.lam + pos * M + row) : 0.0;
    __syncthreads();
    {
      // hat r (e x 8) = X^T r: A[row=e][k=a] = X[a][e]
      double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
      for (int kt = 0; kt < KH; ++kt) {
        const double rb = rs[(kt * 4 + kl) * RS + n8];
        const int a = (kt + KH) * 4 + kl;
        const double xn = (kt + KH < KT && row_ok && a < M) ? __ldg(X + a * M + row) : 0.0;
        if (kt & 1)
          dmma(d10, d11, xa[kt], rb);
        else
          dmma(d00, d01, xa[kt], rb);
        xa[kt] = xn;
      }
#pragma unroll
      for (int kt = KH; kt < KT; ++kt) {
        const double rb = rs[(kt * 4 + kl) * RS + n8];
        if (kt & 1)
          dmma(d10, d11, xa[kt - KH], rb);
        else
          dmma(d00, d01, xa[kt - KH], rb);
      }
      const double c0 = d00 + d10, c1 = d01 + d11;
      double out0 = 0.0, out1 = 0.0;
      if (A.tdiag) {
        if (row_ok) tdiag_scale(A, kl, lam, c0, c1, out0, out1);
      } else {
      double v[8];
      const int grp = lane & ~3;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[2 * j] = __shfl_sync(0xffffffffu, c0, grp | j);
        v[2 * j + 1] = __shfl_sync(0xffffffffu, c1, grp | j);
      }
      if (row_ok) {
#pragma unroll
        for (int s = 0; s < 8 / NT; ++s) {
          if (s >= A.S) break;
          double b4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int i = 0; i < NT; ++i) b4[i] = v[s * NT + i];
          small_solve(A.TM, A.TA, lam, NT, b4);
#pragma unroll
          for (int i = 0; i < NT; ++i) {
            if (s * NT + i == col) out0 = b4[i];
            if (s * NT + i == col + 1) out1 = b4[i];
          }
        }
      }
      }
      *reinterpret_cast<double2*>(hs + row * RS + col) = make_double2(out0, out1);
    }
    // second product's A fragments: X[row][e], e = 4 kt + kl (L2)
#pragma unroll
    for (int kt = 0; kt < KH; ++kt) {
      const int e = kt * 4 + kl;
      xa[kt] = (row_ok && e < M) ? __ldg(X + row * M + e) : 0.0;
    }
    __syncthreads();
    {
      double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
      for (int kt = 0; kt < KH; ++kt) {
        const double hb = hs[(kt * 4 + kl) * RS + n8];
        const int e = (kt + KH) * 4 + kl;
        const double xn = (kt + KH < KT && row_ok && e < M) ? __ldg(X + row * M + e) : 0.0;
        if (kt & 1)
          dmma(d10, d11, xa[kt], hb);
        else
          dmma(d00, d01, xa[kt], hb);
        xa[kt] = xn;
      }
#pragma unroll
      for (int kt = KH; kt < KT; ++kt) {
        const double hb = hs[(kt * 4 + kl) * RS + n8];
        if (kt & 1)
          dmma(d10, d11, xa[kt - KH], hb);
        else
          dmma(d00, d01, xa[kt - KH], hb);
      }
      double v0 = d00 + d10, v1 = d01 + d11;
      if (A.tdiag) tdiag_qmix(PQ + 64, lane, d00 + d10, d01 + d11, v0, v1);
      if (row_ok) {
        const LocalDof d = local_dof(A, cx, cy, cz, row);
        const double w = scale / d.mult;
        if (!(A.tdiag && d.bdry)) {
          if (d.bdry) {
            v0 = rs[row * RS + col];
            v1 = rs[row * RS + col + 1];
          }
          if (col < ncol) atomicAdd(z + static_cast<long long>(col) * A.n_space + d.g, v0 * w);
          if (col + 1 < ncol) atomicAdd(z + static_cast<long long>(col + 1) * A.n_space + d.g, v1 * w);
        }
      }
    }
    __syncthreads();
  }
}

// Dirichlet dofs of every cell matrix pair: M rows/cols -> identity, A -> 0
// (the decoupled identity rows of asm_smoother.cpp:29-33 in the eigenbasis)
__global__ void dirichlet_rows_kernel(const __grid_constant__ DevASM A, double* __restrict__ Mt,
                                      double* __restrict__ At) {
  const int m = A.m;
  const long long total = A.n_list * m;
  for (long long tt = blockIdx.x * (long long)blockDim.x + threadIdx.x; tt < total;
       tt += (long long)gridDim.x * blockDim.x) {
    const long long pos = tt / m;
    const int a = static_cast<int>(tt - pos * m);
    const long long cell = A.list ? A.list[pos] : pos;
    long long cx, cy, cz;
    cell_coords(cell, A.cells, cx, cy, cz);
    if (!local_dof(A, cx, cy, cz, a).bdry) continue;
    double* Mc = Mt + pos * static_cast<long long>(m) * m;
    double* Ac = At + pos * static_cast<long long>(m) * m;
    for (int j = 0; j < m; ++j) {
      Mc[static_cast<long long>(a) * m + j] = (j == a) ? 1.0 : 0.0;
      Mc[static_cast<long long>(j) * m + a] = (j == a) ? 1.0 : 0.0;
      Ac[static_cast<long long>(a) * m + j] = 0.0;
      Ac[static_cast<long long>(j) * m + a] = 0.0;
    }
  }
}

// column-major X (cuSOLVER / cuBLAS) -> row-major records
__global__ void transpose_cells_kernel(int m, long long n_cells, long long xs, const double* __restrict__ colmajor,
                                       double* __restrict__ X) {
  const long long total = n_cells * m * m;
  for (long long tt = blockIdx.x * (long long)blockDim.x + threadIdx.x; tt < total;
       tt += (long long)gridDim.x * blockDim.x) {
    const long long cell = tt / (static_cast<long long>(m) * m);
    const long long r = tt - cell * m * m;
    const int a = static_cast<int>(r / m), e = static_cast<int>(r % m);
    X[cell * xs + r] = colmajor[cell * static_cast<long long>(m) * m + static_cast<long long>(e) * m + a];
  }
}

// column b of every cell matrix from one probe of colour (cx,cy,cz) mod period
__global__ void extract_probe_kernel(const __grid_constant__ DevASM A, int colx, int coly, int colz, int period,
                                     const double* __restrict__ probe, int probe_zcells,
                                     double* __restrict__ cellmat) {
  const long long n_pos = A.n_list;
  const int m = A.m, n = A.n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_pos * m;
       t += (long long)gridDim.x * blockDim.x) {
    const long long pos = t / m;
    const int a = static_cast<int>(t - pos * m);
    const long long cell = A.list ? A.list[pos] : pos;
    long long cx, cy, cz;
    cell_coords(cell, A.cells, cx, cy, cz);
    // local index per axis whose lattice coordinate has the probe colour
    int lb[3] = {0, 0, 0};
    bool found = true;
    const long long c3[3] = {cx, cy, cz + A.cz0};  // colours: global lattice coordinates
    const int col[3] = {colx, coly, colz};
    for (int ax = 0; ax < A.dim; ++ax) {
      int hit = -1;
      for (int l = 0; l < n; ++l)
        if ((c3[ax] * A.p + l) % period == col[ax]) hit = l;
      if (hit < 0) found = false;
      lb[ax] = hit;
    }
    if (!found) continue;
    const int b = lb[0] + n * (lb[1] + (A.dim == 3 ? n * lb[2] : 0));
    const LocalDof da = local_dof(A, cx, cy, cz, a);
    const long long gp = da.g + static_cast<long long>(probe_zcells) * A.p * A.dofs[0] * A.dofs[1];
    cellmat[pos * static_cast<long long>(m) * m + static_cast<long long>(a) * m + b] = probe[gp];
  }
}

// per cell: M = L L^T (Dirichlet dofs: M=1, A=0 decoupled); At <- L^-1 A L^-T,
// Mt <- L^-1. One CTA per cell, blockDim >= m.
__global__ void reduce_standard_kernel(const __grid_constant__ DevASM A, double* __restrict__ Mt,
                                       double* __restrict__ At) {
  extern __shared__ double sm[];
  const int m = A.m, ld = m + 1;
  double* L = sm;            // [m][ld]
  double* As = L + m * ld;   // [m][ld]
  double* T = As + m * ld;   // [m][ld]
  const long long pos = blockIdx.x;
  const long long cell = A.list ? A.list[pos] : pos;
  double* Mg = Mt + pos * static_cast<long long>(m) * m;
  double* Ag = At + pos * static_cast<long long>(m) * m;
  long long cx, cy, cz;
  cell_coords(cell, A.cells, cx, cy, cz);
  for (int i = threadIdx.x; i < m * m; i += blockDim.x) {
    const int r = i / m, c = i % m;
    L[r * ld + c] = Mg[i];
    As[r * ld + c] = Ag[i];
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < m) {
    const LocalDof d = local_dof(A, cx, cy, cz, t);
    if (d.bdry) {
      for (int j = 0; j < m; ++j) {
        L[t * ld + j] = (j == t) ? 1.0 : 0.0;
        As[t * ld + j] = 0.0;
      }
    }
  }
  __syncthreads();
  if (t < m) {
    const LocalDof d = local_dof(A, cx, cy, cz, t);
    if (d.bdry)
      for (int j = 0; j < m; ++j) {
        L[j * ld + t] = (j == t) ? 1.0 : 0.0;
        As[j * ld + t] = 0.0;
      }
  }
  __syncthreads();
  // right-looking Cholesky, lower triangle
  for (int k = 0; k < m; ++k) {
    if (t == 0) L[k * ld + k] = sqrt(L[k * ld + k]);
    __syncthreads();
    if (t > k && t < m) L[t * ld + k] /= L[k * ld + k];
    __syncthreads();
    if (t > k && t < m) {
      const double lik = L[t * ld + k];
      for (int j = k + 1; j <= t; ++j) L[t * ld + j] = fma(-lik, L[j * ld + k], L[t * ld + j]);
    }
    __syncthreads();
  }
  // T = L^-1 (column t by forward substitution), stored in T
  if (t < m) {
    for (int i = 0; i < m; ++i) {
      double s = (i == t) ? 1.0 : 0.0;
      if (i < t) {
        T[i * ld + t] = 0.0;
        continue;
      }
      for (int k = t; k < i; ++k) s = fma(-L[i * ld + k], T[k * ld + t], s);
      T[i * ld + t] = s / L[i * ld + i];
    }
  }
  __syncthreads();
  // L <- T A (row t), then At = (T A) T^T (row t)
  if (t < m) {
    for (int j = 0; j < m; ++j) {
      double s = 0.0;
      for (int k = 0; k <= t; ++k) s = fma(T[t * ld + k], As[k * ld + j], s);
      L[t * ld + j] = s;
    }
  }
  __syncthreads();
  if (t < m) {
    for (int j = 0; j < m; ++j) {
      double s = 0.0;
      for (int k = 0; k <= j; ++k) s = fma(L[t * ld + k], T[j * ld + k], s);
      Ag[static_cast<long long>(t) * m + j] = s;
    }
    for (int j = 0; j < m; ++j) Mg[static_cast<long long>(t) * m + j] = T[t * ld + j];
  }
}

// X[a][e] = sum_k Linv[k][a] V[k][e]; V column-major from syev (V[e*m+k])
__global__ void back_transform_kernel(int m, long long xs, int layout, const double* __restrict__ Linv,
                                      const double* __restrict__ V, double* __restrict__ X) {
  const long long cell = blockIdx.x;
  const double* Lc = Linv + cell * static_cast<long long>(m) * m;
  const double* Vc = V + cell * static_cast<long long>(m) * m;
  double* Xc = X + cell * xs;
  for (int i = threadIdx.x; i < m * m; i += blockDim.x) {
    const int a = i / m, e = i % m;
    double s = 0.0;
    for (int k = a; k < m; ++k) s = fma(Lc[static_cast<long long>(k) * m + a], Vc[static_cast<long long>(e) * m + k], s);
    Xc[m == 64 ? swz64(a, e) : (layout == 2 ? a * kMma32Pitch + e : i)] = s;
  }
}

}  // namespace

namespace {
template <int M, int NT>
void launch_asm(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  if (A.n_list == 0) return;
  if (A.S * NT > 8) throw std::invalid_argument("ASMSmoother: S * n_t must be <= 8");
  constexpr size_t smem = sizeof(double) * 8 * warp_smem_doubles<M>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(asm_apply_warp_kernel<M, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    configured = true;
  }
  int per_sm = 0, dev = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, asm_apply_warp_kernel<M, NT>, 256, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long warps = (A.n_list + 7) / 8;
  const long long grid = std::max<long long>(1, std::min<long long>(warps, static_cast<long long>(std::max(per_sm, 1)) * sms));
  count_launch();
  asm_apply_warp_kernel<M, NT><<<static_cast<unsigned>(grid), 256, smem, s>>>(A, r, z, scale);
}
template <int M, int NT>
void launch_mma32(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  if (A.xs != mma32_xbuf<M>()) throw std::invalid_argument("ASMSmoother: unexpected record stride");
  constexpr size_t smem = mma32_smem<M>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(asm_apply_mma32_kernel<M, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaFuncSetAttribute(asm_apply_mma32_kernel<M, NT>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    configured = true;
  }
  int per_sm = 0, dev = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, asm_apply_mma32_kernel<M, NT>, 128, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long warps = (A.n_list + kWmmaWarps - 1) / kWmmaWarps;
  const long long grid =
      std::max<long long>(1, std::min<long long>(warps, static_cast<long long>(std::max(per_sm, 1)) * sms));
  count_launch();
  asm_apply_mma32_kernel<M, NT><<<static_cast<unsigned>(grid), 128, smem, s>>>(A, r, z, scale);
}
// m = 25 / 27 run on the tensor cores (C3 fine sweep 1.79 -> 1.51 ms against
// the DFMA warp-per-cell kernel, which serves the smaller blocks)
template <int M, int NT>
void launch_small(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  if constexpr (M > 24) {
    // the record layout chosen at setup (stmg.cpp) selects the kernel
    if (A.x_layout == 2) {
      if (A.n_list == 0) return;
      if (A.S * NT > 8) throw std::invalid_argument("ASMSmoother: S * n_t must be <= 8");
      launch_mma32<M, NT>(A, r, z, scale, s);
      return;
    }
  }
  launch_asm<M, NT>(A, r, z, scale, s);
}
template <int M>
void launch_asm_nt(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  switch (A.nt) {
    case 1: launch_small<M, 1>(A, r, z, scale, s); break;
    case 2: launch_small<M, 2>(A, r, z, scale, s); break;
    case 3: launch_small<M, 3>(A, r, z, scale, s); break;
    case 4: launch_small<M, 4>(A, r, z, scale, s); break;
    default: throw std::invalid_argument("ASMSmoother: n_t must be in [1, 4]");
  }
}
}  // namespace

namespace {
template <int NT>
void launch_mma(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  const size_t smem = sizeof(double) * (2 * 64 * 64 + 16 * 64) + 2 * sizeof(unsigned long long);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(asm_apply_mma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(asm_apply_mma_kernel<NT>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    configured = true;
  }
  int per_sm = 0, dev = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, asm_apply_mma_kernel<NT>, 256, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (A.n_list == 0) return;
  const long long grid = std::max<long long>(1, std::min<long long>(A.n_list, static_cast<long long>(std::max(per_sm, 1)) * sms));
  count_launch();
  asm_apply_mma_kernel<NT><<<static_cast<unsigned>(grid), 256, smem, s>>>(A, r, z, scale);
}
void launch_asm_mma(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  if (A.S * A.nt > 8) throw std::invalid_argument("ASMSmoother: S * n_t must be <= 8");
  switch (A.nt) {
    case 1: launch_mma<1>(A, r, z, scale, s); break;
    case 2: launch_mma<2>(A, r, z, scale, s); break;
    case 3: launch_mma<3>(A, r, z, scale, s); break;
    case 4: launch_mma<4>(A, r, z, scale, s); break;
    default: throw std::invalid_argument("ASMSmoother: n_t must be in [1, 4]");
  }
}
template <int NT, int S, int NBUF>
void launch_fd64_nbuf(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  constexpr size_t smem = fd64_smem<NBUF>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(asm_apply_fd64_kernel<NT, S, NBUF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaFuncSetAttribute(asm_apply_fd64_kernel<NT, S, NBUF>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    configured = true;
  }
  int per_sm = 0, dev = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, asm_apply_fd64_kernel<NT, S, NBUF>, 256, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (A.n_list == 0) return;
  const long long grid =
      std::max<long long>(1, std::min<long long>(A.n_list, static_cast<long long>(std::max(per_sm, 1)) * sms));
  count_launch();
  asm_apply_fd64_kernel<NT, S, NBUF><<<static_cast<unsigned>(grid), 256, smem, s>>>(A, r, z, scale);
}
// one record in flight per CTA at 3 CTAs / SM (1.61 ms per C2 sweep against
// 1.91 ms for three buffers at 2 CTAs / SM: the per-cell solve, not the bytes
// in flight, limits the sweep)
template <int NT, int S>
void launch_fd64(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  launch_fd64_nbuf<NT, S, 2>(A, r, z, scale, s);
}
void launch_asm_fd64(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  switch (A.nt * 10 + A.S) {
    case 11: launch_fd64<1, 1>(A, r, z, scale, s); break;
    case 12: launch_fd64<1, 2>(A, r, z, scale, s); break;
    case 13: launch_fd64<1, 3>(A, r, z, scale, s); break;
    case 14: launch_fd64<1, 4>(A, r, z, scale, s); break;
    case 15: launch_fd64<1, 5>(A, r, z, scale, s); break;
    case 16: launch_fd64<1, 6>(A, r, z, scale, s); break;
    case 17: launch_fd64<1, 7>(A, r, z, scale, s); break;
    case 18: launch_fd64<1, 8>(A, r, z, scale, s); break;
    case 21: launch_fd64<2, 1>(A, r, z, scale, s); break;
    case 22: launch_fd64<2, 2>(A, r, z, scale, s); break;
    case 23: launch_fd64<2, 3>(A, r, z, scale, s); break;
    case 24: launch_fd64<2, 4>(A, r, z, scale, s); break;
    case 31: launch_fd64<3, 1>(A, r, z, scale, s); break;
    case 32: launch_fd64<3, 2>(A, r, z, scale, s); break;
    case 41: launch_fd64<4, 1>(A, r, z, scale, s); break;
    case 42: launch_fd64<4, 2>(A, r, z, scale, s); break;
    default: launch_asm_mma(A, r, z, scale, s);
  }
}

template <int M, int NT>
void launch_large_mma(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  constexpr int NTH = ((M + 7) / 8) * 32;
  constexpr size_t smem = sizeof(double) * (2 * kLargeMmaPitch * ((M + 7) / 8) * 8 + 128);
  int per_sm = 0, dev = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, asm_apply_large_mma_kernel<M, NT>, NTH, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long grid =
      std::max<long long>(1, std::min<long long>(A.n_list, static_cast<long long>(std::max(per_sm, 1)) * sms));
  count_launch();
  asm_apply_large_mma_kernel<M, NT><<<static_cast<unsigned>(grid), NTH, smem, s>>>(A, r, z, scale);
}
// m = 125 (3D Q4): the tensor-core kernel (the CTA-per-cell DFMA form it
// replaced ran 2.8 vs 2.2 ms per C4 fine sweep)
template <int NT>
void launch_large(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  if (A.n_list == 0) return;
  if (A.m != 125) throw std::invalid_argument("ASMSmoother: exact blocks above 64 dofs need m = 125 (3D Q4)");
  launch_large_mma<125, NT>(A, r, z, scale, s);
}
void launch_asm_large(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  if (A.m > 128) throw std::invalid_argument("ASMSmoother: cell blocks larger than 128 dofs are not supported");
  if (A.S * A.nt > 8) throw std::invalid_argument("ASMSmoother: S * n_t must be <= 8");
  switch (A.nt) {
    case 1: launch_large<1>(A, r, z, scale, s); break;
    case 2: launch_large<2>(A, r, z, scale, s); break;
    case 3: launch_large<3>(A, r, z, scale, s); break;
    case 4: launch_large<4>(A, r, z, scale, s); break;
    default: throw std::invalid_argument("ASMSmoother: n_t must be in [1, 4]");
  }
}
}  // namespace

void asm_add_correction(const DevASM& A, const double* r, double* z, double scale, cudaStream_t s) {
  if (A.m == 64 && A.tdiag && A.meta) {
    launch_asm_fd64(A, r, z, scale, s);
    return;
  }
  if (A.m > 64) {
    launch_asm_large(A, r, z, scale, s);
    return;
  }
  switch (A.m) {
    case 4: launch_asm_nt<4>(A, r, z, scale, s); break;
    case 8: launch_asm_nt<8>(A, r, z, scale, s); break;
    case 9: launch_asm_nt<9>(A, r, z, scale, s); break;
    case 16: launch_asm_nt<16>(A, r, z, scale, s); break;
    case 25: launch_asm_nt<25>(A, r, z, scale, s); break;
    case 27: launch_asm_nt<27>(A, r, z, scale, s); break;
    case 64: launch_asm_mma(A, r, z, scale, s); break;
    default: throw std::invalid_argument("ASMSmoother: unsupported cell block size");
  }
}

void asm_extract_probe(const DevASM& A, int cx, int cy, int cz, int period, const double* probe, int probe_zcells,
                       double* cellmat, cudaStream_t s) {
  const long long total = A.n_list * A.m;
  if (total == 0) return;
  const unsigned grid = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 148LL * 64)));
  count_launch();
  extract_probe_kernel<<<grid, 256, 0, s>>>(A, cx, cy, cz, period, probe, probe_zcells, cellmat);
}

void asm_reduce_standard(const DevASM& A, double* Mt, double* At, cudaStream_t s) {
  const long long n_cells = A.n_list;
  if (n_cells == 0) return;
  const int threads = ((A.m + 31) / 32) * 32;
  const size_t smem = sizeof(double) * 3 * static_cast<size_t>(A.m) * (A.m + 1);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(reduce_standard_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  count_launch();
  reduce_standard_kernel<<<static_cast<unsigned>(n_cells), threads, smem, s>>>(A, Mt, At);
}

void asm_dirichlet_rows(const DevASM& A, double* Mt, double* At, cudaStream_t s) {
  const long long total = A.n_list * A.m;
  if (total == 0) return;
  count_launch();
  dirichlet_rows_kernel<<<static_cast<unsigned>(std::max<long long>(1, std::min<long long>((total + 127) / 128, 148LL * 32))),
                          128, 0, s>>>(A, Mt, At);
}

void asm_transpose_cells(int m, long long n_cells, long long xs, const double* colmajor, double* X, cudaStream_t s) {
  const long long total = n_cells * m * m;
  if (total == 0) return;
  count_launch();
  transpose_cells_kernel<<<static_cast<unsigned>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 148LL * 64))),
                           256, 0, s>>>(m, n_cells, xs, colmajor, X);
}

void asm_back_transform(int m, long long xs, int layout, long long n_cells, const double* Linv, const double* V,
                        double* X, cudaStream_t s) {
  count_launch();
  back_transform_kernel<<<static_cast<unsigned>(n_cells), 128, 0, s>>>(m, xs, layout, Linv, V, X);
}

}  // namespace stmgb
