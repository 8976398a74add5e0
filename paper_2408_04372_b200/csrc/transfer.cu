// Grid transfers between consecutive multigrid levels (reference: Transfer,
// transfer.cpp:58-190). Spatial h/p transfers are tensor products of the
// per-axis embedding matrices P (n_f x n_c, transfer.cpp:32-54); they are
// applied here as separable passes, one lattice axis at a time. Pure
// h-coarsening with equal p uses the structured weights of one coarse cell
// (no index arrays); other spatial transfers gather the few nonzeros of a CSR
// row of P (prolongation) or P^T (restriction) -- O((p+1) d) work per entry
// instead of the reference's dense O(n_f n_c) line contraction. Temporal
// tau/k transfers apply the small (S_f n_tf) x (S_c n_tc) evaluation matrix
// blockwise over the spatial dofs. Dirichlet entries are zeroed on the input
// and output sides (transfer.cpp:108-116).
//
// z-slab partition: z faces are Dirichlet only where physical
// (zbc), the input's low z plane can be skipped (an interface plane owned by
// the slab below, so a restriction's interface contributions are counted
// once), and each side has its own field stride so a slab's coarse data can
// live inside a full-length coarse vector.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.hpp"

namespace stmgb {

namespace {

struct PassArgs {
  long long i[3], o[3];    // input / output lattice dims
  long long fs_in, fs_out;  // field strides
  int zbc;                  // physical low (bit 0) / high (bit 1) z faces
  bool mask_in, mask_out, skip_lo_in, accumulate;
};

__device__ __forceinline__ bool on_bdry(long long i, long long n) { return i == 0 || i == n - 1; }
__device__ __forceinline__ bool on_bdry_z(long long i, long long n, int zbc) {
  return (i == 0 && (zbc & 1)) || (i == n - 1 && (zbc & 2));
}

// boundary status of output entry (x, y, z) and of the input row it reads
template <int AXIS>
__device__ __forceinline__ bool skip_entry(const PassArgs& A, long long x, long long y, long long z) {
  const long long ox = A.o[0], oy = A.o[1], oz = A.o[2];
  if (A.mask_out && (on_bdry(x, ox) || (oy > 1 && on_bdry(y, oy)) || (oz > 1 && on_bdry_z(z, oz, A.zbc)))) return true;
  if (A.mask_in) {
    if (AXIS != 0 && on_bdry(x, A.i[0])) return true;
    if (AXIS != 1 && A.i[1] > 1 && on_bdry(y, A.i[1])) return true;
    if (AXIS != 2 && A.i[2] > 1 && on_bdry_z(z, A.i[2], A.zbc)) return true;
  }
  if (A.skip_lo_in && AXIS != 2 && z == 0) return true;
  return false;
}

__device__ __forceinline__ bool skip_input_along(const PassArgs& A, int axis, long long j, long long n_ax) {
  if (A.mask_in && (axis == 2 ? on_bdry_z(j, n_ax, A.zbc) : on_bdry(j, n_ax))) return true;
  return A.skip_lo_in && axis == 2 && j == 0;
}

// out[f][z][y][x] = sum_k w_k in[f][..src..] along AXIS (CSR weights). One
// thread per output entry of a 32 x 4 (x, y) tile: grid (x tiles, y tiles,
// z * F), so no per-entry index decoding; reads along y/z are coalesced across
// the x-consecutive threads.
template <int AXIS>
__global__ void __launch_bounds__(128) axis_pass_kernel(const PassArgs A, const int* __restrict__ ptr,
                                                        const int* __restrict__ idx, const double* __restrict__ w,
                                                        const double* __restrict__ in, double* __restrict__ out) {
  const long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long y = static_cast<long long>(blockIdx.y) * blockDim.y + threadIdx.y;
  if (x >= A.o[0] || y >= A.o[1]) return;
  const long long z = blockIdx.z % A.o[2], f = blockIdx.z / A.o[2];
  const long long oidx = f * A.fs_out + (z * A.o[1] + y) * A.o[0] + x;
  double s = 0.0;
  if (!skip_entry<AXIS>(A, x, y, z)) {
    const long long o = AXIS == 0 ? x : (AXIS == 1 ? y : z);
    const int k0 = __ldg(ptr + o), k1 = __ldg(ptr + o + 1);
    const long long n_ax = A.i[AXIS];
    const double* src = in + f * A.fs_in;
    const long long ix = A.i[0], iy = A.i[1];
    const long long base = AXIS == 0 ? (z * iy + y) * ix : (AXIS == 1 ? z * iy * ix + x : y * ix + x);
    const long long stride = AXIS == 0 ? 1 : (AXIS == 1 ? ix : ix * iy);
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
      const long long j = __ldg(idx + k);
      if (skip_input_along(A, AXIS, j, n_ax)) continue;
      s = fma(__ldg(w + k), __ldg(src + base + j * stride), s);
    }
  }
  if (A.accumulate)
    out[oidx] += s;
  else
    out[oidx] = s;
}

// Cell-blocked h-transfer pass (equal p): one thread per coarse cell of a
// lattice row along AXIS reads the row's inputs of that cell once and writes
// all outputs the cell owns -- prolongation: the 2p fine nodes 2pc .. 2pc+2p-1
// from the p+1 coarse nodes (the last cell also the final fine node);
// restriction: coarse nodes cp .. cp+p-1 from the cell's 2p+1 fine nodes plus
// the left cell's 2p (vertex node), the last cell also the final coarse node.
// Boundary masks are evaluated only on the row's first / last cell.
template <int AXIS, int P, bool PROLONG>
__global__ void __launch_bounds__(128) axis_cell_kernel(const PassArgs A, const DevAxisTransfer T,
                                                        const double* __restrict__ in, double* __restrict__ out) {
  const long long n_in = A.i[AXIS], n_out = A.o[AXIS];
  const long long ncc = PROLONG ? (n_in - 1) / P : (n_out - 1) / P;
  long long x, y, z, f, c;
  if (AXIS == 0) {
    c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    y = static_cast<long long>(blockIdx.y) * blockDim.y + threadIdx.y;
    z = blockIdx.z % A.o[2];
    f = blockIdx.z / A.o[2];
    x = 0;
    if (c >= ncc || y >= A.o[1]) return;
  } else if (AXIS == 1) {
    x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    c = static_cast<long long>(blockIdx.y) * blockDim.y + threadIdx.y;
    z = blockIdx.z % A.o[2];
    f = blockIdx.z / A.o[2];
    y = 0;
    if (x >= A.o[0] || c >= ncc) return;
  } else {
    x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    y = static_cast<long long>(blockIdx.y) * blockDim.y + threadIdx.y;
    c = blockIdx.z % ncc;
    f = blockIdx.z / ncc;
    z = 0;
    if (x >= A.o[0] || y >= A.o[1]) return;
  }
  // rows: input / output base offsets and the stride along AXIS
  const long long ix = A.i[0], iy = A.i[1], ox = A.o[0], oy = A.o[1];
  const long long ibase = f * A.fs_in + (AXIS == 0 ? (z * iy + y) * ix : (AXIS == 1 ? z * iy * ix + x : y * ix + x));
  const long long obase = f * A.fs_out + (AXIS == 0 ? (z * oy + y) * ox : (AXIS == 1 ? z * oy * ox + x : y * ox + x));
  const long long istr = AXIS == 0 ? 1 : (AXIS == 1 ? ix : ix * iy);
  const long long ostr = AXIS == 0 ? 1 : (AXIS == 1 ? ox : ox * oy);
  // the row itself masked out (other coordinates on a boundary)?
  bool row_in0 = false, row_out0 = false;
  if (A.mask_in) {
    if (AXIS != 0 && on_bdry(x, ix)) row_in0 = true;
    if (AXIS != 1 && A.i[1] > 1 && on_bdry(y, iy)) row_in0 = true;
    if (AXIS != 2 && A.i[2] > 1 && on_bdry_z(z, A.i[2], A.zbc)) row_in0 = true;
  }
  if (A.skip_lo_in && AXIS != 2 && z == 0) row_in0 = true;
  if (A.mask_out) {
    if (AXIS != 0 && on_bdry(x, ox)) row_out0 = true;
    if (AXIS != 1 && oy > 1 && on_bdry(y, oy)) row_out0 = true;
    if (AXIS != 2 && A.o[2] > 1 && on_bdry_z(z, A.o[2], A.zbc)) row_out0 = true;
  }
  // only the first / last cells (and the left neighbour of cell 1) touch
  // boundary nodes
  const bool edge = c <= 1 || c == ncc - 1;
  auto ld = [&](long long j) -> double {
    if (row_in0) return 0.0;
    if (edge && skip_input_along(A, AXIS, j, n_in)) return 0.0;
    return __ldg(in + ibase + j * istr);
  };
  auto st = [&](long long j, double v) {
    if (row_out0 || (edge && A.mask_out && (AXIS == 2 ? on_bdry_z(j, n_out, A.zbc) : on_bdry(j, n_out)))) v = 0.0;
    double* o = out + obase + j * ostr;
    if (A.accumulate)
      *o += v;
    else
      *o = v;
  };
  if (PROLONG) {
    double cv[P + 1];
#pragma unroll
    for (int j = 0; j <= P; ++j) cv[j] = ld(c * P + j);
    const int rmax = c == ncc - 1 ? 2 * P : 2 * P - 1;
#pragma unroll
    for (int r = 0; r <= 2 * P; ++r) {
      if (r > rmax) break;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j <= P; ++j) s = fma(T.hw[r][j], cv[j], s);
      st(2 * P * c + r, s);
    }
  } else {
    double fv[2 * P + 1], lv[2 * P];
#pragma unroll
    for (int r = 0; r <= 2 * P; ++r) fv[r] = ld(2 * P * c + r);
#pragma unroll
    for (int r = 0; r < 2 * P; ++r) lv[r] = c > 0 ? ld(2 * P * (c - 1) + r) : 0.0;
#pragma unroll
    for (int jj = 0; jj < P; ++jj) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r <= 2 * P; ++r) s = fma(T.hw[r][jj], fv[r], s);
      if (jj == 0) {
#pragma unroll
        for (int r = 0; r < 2 * P; ++r) s = fma(T.hw[r][P], lv[r], s);
      }
      st(c * P + jj, s);
    }
    if (c == ncc - 1) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r <= 2 * P; ++r) s = fma(T.hw[r][P], fv[r], s);
      st(c * P + P, s);
    }
  }
}

__global__ void temporal_kernel(const double* __restrict__ T, int Ff, int Fc, bool transpose, bool accumulate,
                                long long n_space, long long dx, long long dy, long long dz, int dim, int zbc,
                                bool skip_lo_in, long long fs_in, long long fs_out, const double* __restrict__ in,
                                double* __restrict__ out) {
  // prolong: out (Ff blocks) = T in (Fc blocks); restrict: out (Fc) = T^T in (Ff)
  const int Fin = transpose ? Ff : Fc, Fout = transpose ? Fc : Ff;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n_space; g += (long long)gridDim.x * blockDim.x) {
    const long long ix = g % dx, iy = (g / dx) % dy, iz = g / (dx * dy);
    const bool bd = on_bdry(ix, dx) || (dim > 1 && on_bdry(iy, dy)) ||
                    (dim > 2 && (on_bdry_z(iz, dz, zbc) || (skip_lo_in && iz == 0)));
    if (Fin > kMaxF || Fout > kMaxF) {
      // wide batches: straight from memory
      for (int r = 0; r < Fout; ++r) {
        double s = 0.0;
        if (!bd)
          for (int c = 0; c < Fin; ++c) s = fma(transpose ? T[c * Fc + r] : T[r * Fc + c], in[c * fs_in + g], s);
        if (accumulate)
          out[r * fs_out + g] += s;
        else
          out[r * fs_out + g] = s;
      }
      continue;
    }
    double x[kMaxF];
#pragma unroll
    for (int c = 0; c < kMaxF; ++c) x[c] = (c < Fin && !bd) ? in[c * fs_in + g] : 0.0;
#pragma unroll
    for (int r = 0; r < kMaxF; ++r) {
      if (r >= Fout) break;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < kMaxF; ++c)
        if (c < Fin) s = fma(transpose ? T[c * Fc + r] : T[r * Fc + c], x[c], s);
      if (accumulate)
        out[r * fs_out + g] += s;
      else
        out[r * fs_out + g] = s;
    }
  }
}

inline unsigned grid_for(long long n) {
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 64)));
}

template <int AXIS, int P, bool PROLONG>
void launch_h(int F, const PassArgs& A, const DevAxisTransfer& T, const double* in, double* out, cudaStream_t s) {
  // one thread per coarse cell of a lattice row along AXIS
  const long long ncc = PROLONG ? (A.i[AXIS] - 1) / P : (A.o[AXIS] - 1) / P;
  const dim3 block(32, 4);
  dim3 grid;
  if (AXIS == 0)
    grid = dim3(static_cast<unsigned>((ncc + 31) / 32), static_cast<unsigned>((A.o[1] + 3) / 4),
                static_cast<unsigned>(A.o[2] * F));
  else if (AXIS == 1)
    grid = dim3(static_cast<unsigned>((A.o[0] + 31) / 32), static_cast<unsigned>((ncc + 3) / 4),
                static_cast<unsigned>(A.o[2] * F));
  else
    grid = dim3(static_cast<unsigned>((A.o[0] + 31) / 32), static_cast<unsigned>((A.o[1] + 3) / 4),
                static_cast<unsigned>(ncc * F));
  axis_cell_kernel<AXIS, P, PROLONG><<<grid, block, 0, s>>>(A, T, in, out);
}

template <int AXIS>
void pass(int F, const PassArgs& A, const DevAxisTransfer& T, bool prolong, const double* in, double* out,
          cudaStream_t s) {
  const dim3 block(32, 4);
  const dim3 grid(static_cast<unsigned>((A.o[0] + 31) / 32), static_cast<unsigned>((A.o[1] + 3) / 4),
                  static_cast<unsigned>(A.o[2] * F));
  count_launch();
  if (T.hp > 0) {
#define STMG_H(PP)                                            \
  case PP:                                                    \
    if (prolong)                                              \
      launch_h<AXIS, PP, true>(F, A, T, in, out, s);          \
    else                                                      \
      launch_h<AXIS, PP, false>(F, A, T, in, out, s);         \
    return;
    switch (T.hp) {
      STMG_H(1)
      STMG_H(2)
      STMG_H(3)
      STMG_H(4)
      default: break;
    }
#undef STMG_H
  }
  const int* ptr = prolong ? T.row_ptr : T.col_ptr;
  const int* idx = prolong ? T.row_idx : T.col_idx;
  const double* w = prolong ? T.row_w : T.col_w;
  axis_pass_kernel<AXIS><<<grid, block, 0, s>>>(A, ptr, idx, w, in, out);
}

// Fused x-y h-transfer (equal p, 3D): one CTA per tile of TCX x TCY coarse
// cells of one (z plane, field) stages the tile's input plane region in
// shared memory (coalesced rows), applies the x pass into a second shared
// array and the y pass straight to global memory -- the x-pass intermediate
// never touches HBM. Restriction (first of two passes, z follows): input
// masks as the separable first pass; prolongation (last pass, after the z
// pass): output masks and accumulation as the separable last pass. The
// per-cell rules are those of axis_cell_kernel.
constexpr int kXyTCX = 16, kXyTCY = 4, kXyThreads = 256;

template <int P, bool PROLONG>
struct XyCfg {
  // restriction: fine region of the tile's cells plus the left neighbour
  // cell; prolongation: the tile's coarse nodes
  static constexpr int LX = PROLONG ? kXyTCX * P + 1 : 2 * P * (kXyTCX + 1) + 1;
  static constexpr int LY = PROLONG ? kXyTCY * P + 1 : 2 * P * (kXyTCY + 1) + 1;
  // x-pass output columns: restriction coarse x nodes, prolongation fine x nodes
  static constexpr int MX = PROLONG ? 2 * P * kXyTCX + 1 : kXyTCX * P + 1;
  static constexpr size_t smem_bytes() { return sizeof(double) * (static_cast<size_t>(LX) * LY + static_cast<size_t>(MX) * LY); }
};

template <int P, bool PROLONG>
__global__ void __launch_bounds__(kXyThreads) xy_cell_kernel(const PassArgs A, const DevAxisTransfer Tx,
                                                             const DevAxisTransfer Ty, const double* __restrict__ in,
                                                             double* __restrict__ out) {
  using C = XyCfg<P, PROLONG>;
  extern __shared__ __align__(16) double sm[];
  double* R0 = sm;                 // [LY][LX] input region
  double* R1 = sm + C::LX * C::LY;  // [LY][MX] after the x pass
  const long long ix = A.i[0], iy = A.i[1], ox = A.o[0], oy = A.o[1];
  const long long z = blockIdx.z % A.o[2], f = blockIdx.z / A.o[2];
  // coarse cells along x / y (coarse side: output of a restriction, input of a prolongation)
  const long long ncx = PROLONG ? (ix - 1) / P : (ox - 1) / P, ncy = PROLONG ? (iy - 1) / P : (oy - 1) / P;
  const long long cx0 = static_cast<long long>(blockIdx.x) * kXyTCX, cy0 = static_cast<long long>(blockIdx.y) * kXyTCY;
  const int t = threadIdx.x;
  // ---- load the input region (masked as the first / an inner pass)
  const long long gx0 = PROLONG ? cx0 * P : 2 * P * (cx0 - 1), gy0 = PROLONG ? cy0 * P : 2 * P * (cy0 - 1);
  bool plane0 = false;
  if (!PROLONG && A.mask_in && A.i[2] > 1 && on_bdry_z(z, A.i[2], A.zbc)) plane0 = true;
  if (!PROLONG && A.skip_lo_in && z == 0) plane0 = true;
  const double* src = in + f * A.fs_in + z * iy * ix;
  // all of a thread's loads are issued before any shared store (the loop is
  // latency-bound otherwise)
  constexpr int NLD = (C::LX * C::LY + kXyThreads - 1) / kXyThreads;
  double v[NLD];
#pragma unroll
  for (int i = 0; i < NLD; ++i) {
    const int e = t + i * kXyThreads;
    const int ly = e / C::LX, lx = e - ly * C::LX;
    const long long gx = gx0 + lx, gy = gy0 + ly;
    v[i] = 0.0;
    if (e < C::LX * C::LY && !plane0 && gx >= 0 && gx < ix && gy >= 0 && gy < iy) {
      const bool masked = !PROLONG && A.mask_in && (on_bdry(gx, ix) || on_bdry(gy, iy));
      if (!masked) v[i] = __ldg(src + gy * ix + gx);
    }
  }
#pragma unroll
  for (int i = 0; i < NLD; ++i) {
    const int e = t + i * kXyThreads;
    if (e < C::LX * C::LY) R0[e] = v[i];
  }
  __syncthreads();
  if (!PROLONG) {
    // ---- x pass: (fine row ly, local coarse cell lc) -> coarse x nodes lc*P + jj;
    // lanes run over rows (odd row pitch: conflict-free)
    for (int e = t; e < C::LY * kXyTCX; e += kXyThreads) {
      const int lc = e / C::LY, ly = e - lc * C::LY;
      const long long c = cx0 + lc;
      if (c >= ncx) continue;
      const double* row = R0 + ly * C::LX;
      double fv[2 * P + 1], lv[2 * P];
#pragma unroll
      for (int r = 0; r <= 2 * P; ++r) fv[r] = row[2 * P * (lc + 1) + r];
#pragma unroll
      for (int r = 0; r < 2 * P; ++r) lv[r] = row[2 * P * lc + r];
#pragma unroll
      for (int jj = 0; jj < P; ++jj) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r <= 2 * P; ++r) s = fma(Tx.hw[r][jj], fv[r], s);
        if (jj == 0) {
#pragma unroll
          for (int r = 0; r < 2 * P; ++r) s = fma(Tx.hw[r][P], lv[r], s);
        }
        R1[ly * C::MX + lc * P + jj] = s;
      }
      if (c == ncx - 1) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r <= 2 * P; ++r) s = fma(Tx.hw[r][P], fv[r], s);
        R1[ly * C::MX + lc * P + P] = s;
      }
    }
    __syncthreads();
    // ---- y pass: (coarse x node lx, local coarse y cell lc) -> coarse y nodes
    double* dst = out + f * A.fs_out + z * oy * ox;
    for (int e = t; e < C::MX * kXyTCY; e += kXyThreads) {
      const int lc = e / C::MX, lx = e - lc * C::MX;
      const long long c = cy0 + lc, gx = cx0 * P + lx;
      if (c >= ncy || gx >= ox) continue;
      if (lx == kXyTCX * P && gx != ox - 1) continue;  // the next tile's first node
      double fv[2 * P + 1], lv[2 * P];
#pragma unroll
      for (int r = 0; r <= 2 * P; ++r) fv[r] = R1[(2 * P * (lc + 1) + r) * C::MX + lx];
#pragma unroll
      for (int r = 0; r < 2 * P; ++r) lv[r] = R1[(2 * P * lc + r) * C::MX + lx];
#pragma unroll
      for (int jj = 0; jj < P; ++jj) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r <= 2 * P; ++r) s = fma(Ty.hw[r][jj], fv[r], s);
        if (jj == 0) {
#pragma unroll
          for (int r = 0; r < 2 * P; ++r) s = fma(Ty.hw[r][P], lv[r], s);
        }
        double* o = dst + (c * P + jj) * ox + gx;
        if (A.accumulate) *o += s; else *o = s;
      }
      if (c == ncy - 1) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r <= 2 * P; ++r) s = fma(Ty.hw[r][P], fv[r], s);
        double* o = dst + (c * P + P) * ox + gx;
        if (A.accumulate) *o += s; else *o = s;
      }
    }
  } else {
    // ---- x pass: (coarse row ly, local coarse cell lc) -> fine x nodes 2P lc + r;
    // lanes run over rows (odd row pitch: conflict-free)
    for (int e = t; e < C::LY * kXyTCX; e += kXyThreads) {
      const int lc = e / C::LY, ly = e - lc * C::LY;
      const long long c = cx0 + lc;
      if (c >= ncx) continue;
      const double* row = R0 + ly * C::LX;
      double cv[P + 1];
#pragma unroll
      for (int j = 0; j <= P; ++j) cv[j] = row[lc * P + j];
      const int rmax = c == ncx - 1 ? 2 * P : 2 * P - 1;
#pragma unroll
      for (int r = 0; r <= 2 * P; ++r) {
        if (r > rmax) break;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j <= P; ++j) s = fma(Tx.hw[r][j], cv[j], s);
        R1[ly * C::MX + 2 * P * lc + r] = s;
      }
    }
    __syncthreads();
    // ---- y pass: (fine x column lx, local coarse y cell lc) -> fine y rows, masked store
    const bool plane_out0 = A.mask_out && A.o[2] > 1 && on_bdry_z(z, A.o[2], A.zbc);
    double* dst = out + f * A.fs_out + z * oy * ox;
    for (int e = t; e < C::MX * kXyTCY; e += kXyThreads) {
      const int lc = e / C::MX, lx = e - lc * C::MX;
      const long long c = cy0 + lc, gx = 2 * P * cx0 + lx;
      if (c >= ncy || gx >= ox) continue;
      if (lx == 2 * P * kXyTCX && gx != ox - 1) continue;
      double cv[P + 1];
#pragma unroll
      for (int j = 0; j <= P; ++j) cv[j] = R1[(lc * P + j) * C::MX + lx];
      const bool col0 = plane_out0 || (A.mask_out && on_bdry(gx, ox));
      const int rmax = c == ncy - 1 ? 2 * P : 2 * P - 1;
      // accumulation: every old value is requested before the first store
      double old[2 * P + 1];
#pragma unroll
      for (int r = 0; r <= 2 * P; ++r) old[r] = (A.accumulate && r <= rmax) ? dst[(2 * P * c + r) * ox + gx] : 0.0;
#pragma unroll
      for (int r = 0; r <= 2 * P; ++r) {
        if (r > rmax) break;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j <= P; ++j) s = fma(Ty.hw[r][j], cv[j], s);
        const long long gy = 2 * P * c + r;
        if (col0 || (A.mask_out && on_bdry(gy, oy))) s = 0.0;
        dst[gy * ox + gx] = old[r] + s;
      }
    }
  }
}

template <int P, bool PROLONG>
void launch_xy(int F, const PassArgs& A, const DevAxisTransfer& Tx, const DevAxisTransfer& Ty, const double* in,
               double* out, cudaStream_t s) {
  using C = XyCfg<P, PROLONG>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(xy_cell_kernel<P, PROLONG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(C::smem_bytes()));
    configured = true;
  }
  const long long ncx = PROLONG ? (A.i[0] - 1) / P : (A.o[0] - 1) / P;
  const long long ncy = PROLONG ? (A.i[1] - 1) / P : (A.o[1] - 1) / P;
  const dim3 grid(static_cast<unsigned>((ncx + kXyTCX - 1) / kXyTCX), static_cast<unsigned>((ncy + kXyTCY - 1) / kXyTCY),
                  static_cast<unsigned>(A.o[2] * F));
  count_launch();
  xy_cell_kernel<P, PROLONG><<<grid, kXyThreads, C::smem_bytes(), s>>>(A, Tx, Ty, in, out);
}

void xy_pass(int F, const PassArgs& A, const DevAxisTransfer& Tx, const DevAxisTransfer& Ty, bool prolong,
             const double* in, double* out, cudaStream_t s) {
  switch (Tx.hp) {
#define STMG_XY(PP)                                     \
  case PP:                                              \
    if (prolong)                                        \
      launch_xy<PP, true>(F, A, Tx, Ty, in, out, s);    \
    else                                                \
      launch_xy<PP, false>(F, A, Tx, Ty, in, out, s);   \
    return;
    STMG_XY(1)
    STMG_XY(2)
    STMG_XY(3)
    STMG_XY(4)
#undef STMG_XY
    default: break;
  }
}

// ---------------------------------------------------------------------------
// Fused 3D h-transfers (equal p on all three axes): one kernel per transfer,
// no HBM intermediate. A CTA owns a tile of TCX x TCY coarse cells and
// marches a chunk of coarse cell layers along z, one fine plane at a time:
//   restriction: the fine plane tile (plus the left neighbour cell in x and
//     y) is staged by cp.async one plane ahead, the x and y passes run in
//     shared memory (as xy_cell_kernel), and each y-pass thread accumulates
//     its coarse (x, y) nodes into a z window of the p + 1 coarse planes of
//     the open coarse layer held in registers; when the layer closes its p
//     lower planes are final and stored. The chunk starts one coarse layer
//     early (its contribution to the chunk's first coarse plane).
//   prolongation: the p + 1 coarse planes of the open coarse layer are
//     staged; every fine plane is the z combination of them, then the x and
//     y passes, added into the fine vector.
// Masks, slab options and field strides are those of the separable passes
// (input masked as the first pass, output as the last).
constexpr int kZT = 256, kZCX = 8, kZCY = 8;

__device__ __forceinline__ void cp8(double* dst, const double* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(ok ? src : nullptr), "r"(ok ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <int P>
struct ZCfg {
  static constexpr int LX = 2 * P * (kZCX + 1) + 1, LY = 2 * P * (kZCY + 1) + 1;  // fine tile + left cells
  static constexpr int LXP = LX | 1;                 // odd row pitch
  static constexpr int MX = kZCX * P + 1;            // coarse x nodes of the tile (+ right edge)
  static constexpr int MXP = MX | 1;
  static constexpr int YI = kZCX * P * kZCY;         // y-pass items: (coarse x node, coarse y cell)
  static constexpr size_t r_smem() { return sizeof(double) * (2 * static_cast<size_t>(LY) * LXP + LY * MXP); }
  // prolongation: coarse tile (P + 1 planes), z-combined plane, x-pass output
  static constexpr int CX = kZCX * P + 1, CY = kZCY * P + 1, CXP = CX | 1;
  static constexpr int FX = 2 * P * kZCX + 1, FXP = FX | 1;  // fine x nodes of the tile (+ right edge)
  static constexpr size_t p_smem() {
    return sizeof(double) * (static_cast<size_t>(P + 1) * CY * CXP + CY * CXP + static_cast<size_t>(CY) * FXP);
  }
};

template <int P>
__global__ void __launch_bounds__(kZT, 2) xyz_restrict_kernel(const PassArgs A, const DevAxisTransfer Tx,
                                                           const DevAxisTransfer Ty, const DevAxisTransfer Tz,
                                                           const double* __restrict__ in, double* __restrict__ out,
                                                           int ntx, int nch, int zc) {
  using C = ZCfg<P>;
  extern __shared__ __align__(16) double sm[];
  constexpr int R0S = C::LY * C::LXP;  // one staged fine plane (two buffers at sm)
  double* R1 = sm + 2 * C::LY * C::LXP;
  const long long ix = A.i[0], iy = A.i[1], iz = A.i[2], ox = A.o[0], oy = A.o[1];
  const int ncx = static_cast<int>((ox - 1) / P), ncy = static_cast<int>((oy - 1) / P),
            ncz = static_cast<int>((A.o[2] - 1) / P);
  const int tile = blockIdx.x, f = blockIdx.y / nch, ch = blockIdx.y - (blockIdx.y / nch) * nch;
  const int cx0 = (tile % ntx) * kZCX, cy0 = (tile / ntx) * kZCY;
  const int C0 = ch * zc, C1 = C0 + zc < ncz ? C0 + zc : ncz;
  const int zf0 = 2 * P * (C0 > 0 ? C0 - 1 : 0), zf1 = 2 * P * C1 - 1;  // + the top plane if C1 == ncz
  const int zf_end = C1 == ncz ? zf1 + 1 : zf1;
  const int t = threadIdx.x;
  const long long gx0 = 2LL * P * (cx0 - 1), gy0 = 2LL * P * (cy0 - 1);
  const double* src_f = in + f * A.fs_in;
  // stage fine plane zf of the tile region (input masks; left-of-domain zero).
  // The rows / columns of the region that lie inside the lattice and off its
  // masked faces are the tile-coordinate ranges [ly_lo, ly_hi) x [lx_lo, lx_hi)
  const int mk = A.mask_in ? 1 : 0;
  const int lx_lo = static_cast<int>(std::max<long long>(0, mk - gx0));
  const int lx_hi = static_cast<int>(std::min<long long>(C::LX, ix - mk - gx0));
  const int ly_lo = static_cast<int>(std::max<long long>(0, mk - gy0));
  const int ly_hi = static_cast<int>(std::min<long long>(C::LY, iy - mk - gy0));
  const bool tile_in = lx_lo == 0 && lx_hi == C::LX && ly_lo == 0 && ly_hi == C::LY;
  auto stage = [&](int zf, double* dst) {
    // warp w stages rows w, w + 8, ...; lanes run along x (one row base per row)
    const bool plane0 = (A.mask_in && on_bdry_z(zf, iz, A.zbc)) || (A.skip_lo_in && zf == 0);
    const double* src = src_f + static_cast<long long>(zf) * iy * ix + gy0 * ix + gx0;
    const int lane = t & 31, w = t >> 5;
    if (tile_in && !plane0) {
      // interior tile: plain copies, no per-element tests
      for (int ly = w; ly < C::LY; ly += kZT / 32) {
        const double* rs = src + static_cast<long long>(ly) * ix;
        const unsigned rd = static_cast<unsigned>(__cvta_generic_to_shared(dst + ly * C::LXP));
#pragma unroll
        for (int k = 0; k < (C::LX + 31) / 32; ++k) {
          const int lx = lane + 32 * k;
          if (lx < C::LX)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(rd + 8u * lx), "l"(rs + lx) : "memory");
        }
      }
    } else {
      for (int ly = w; ly < C::LY; ly += kZT / 32) {
        const bool rok = !plane0 && ly >= ly_lo && ly < ly_hi;
        const double* rs = src + static_cast<long long>(ly) * ix;
        double* rd = dst + ly * C::LXP;
#pragma unroll
        for (int k = 0; k < (C::LX + 31) / 32; ++k) {
          const int lx = lane + 32 * k;
          if (lx < C::LX) cp8(rd + lx, rs + lx, rok && lx >= lx_lo && lx < lx_hi);
        }
      }
    }
    cp_commit();
  };
  // y-pass identity: coarse x node lxn of the tile, coarse y cell lcy
  const int lxn = t % (kZCX * P), lcy = t / (kZCX * P);
  const bool yitem = t < C::YI;
  const long long gxc = static_cast<long long>(cx0) * P + lxn;
  const bool xin = gxc < ox - 1;  // the last coarse x node is a boundary node (zero)
  const int cyg = cy0 + lcy;
  const bool yin = cyg < ncy;
  double win[P][P + 1];
#pragma unroll
  for (int a = 0; a < P; ++a)
#pragma unroll
    for (int j = 0; j <= P; ++j) win[a][j] = 0.0;
  double* dst_f = out + f * A.fs_out;
  auto store_layer = [&](int cz, int nj) {  // coarse planes cz*P + j, j < nj
    if (yitem && xin && yin) {
#pragma unroll
      for (int j = 0; j <= P; ++j) {
        if (j >= nj) break;
        const long long zc_ = static_cast<long long>(cz) * P + j;
        const bool pz = A.mask_out && on_bdry_z(zc_, A.o[2], A.zbc);
#pragma unroll
        for (int a = 0; a < P; ++a) {
          const long long gy = static_cast<long long>(cyg) * P + a;
          double v = win[a][j];
          if (pz || (A.mask_out && (gy == 0 || gxc == 0))) v = 0.0;
          double* o = dst_f + (zc_ * oy + gy) * ox + gxc;
          if (A.accumulate) *o += v; else *o = v;
        }
      }
    }
    // the last coarse x column / y row of the lattice (boundary nodes): zero
    if (!A.accumulate) {
      const bool last_x = cx0 + kZCX >= ncx, last_y = cy0 + kZCY >= ncy;
      for (int j = 0; j < nj; ++j) {
        const long long zc_ = static_cast<long long>(cz) * P + j;
        double* pl = dst_f + zc_ * oy * ox;
        if (last_x && t < kZCY * P + 1) {
          const long long gy = static_cast<long long>(cy0) * P + t;
          if (gy < oy) pl[gy * ox + ox - 1] = 0.0;
        }
        if (last_y && t < kZCX * P + 1) {
          const long long gx = static_cast<long long>(cx0) * P + t;
          if (gx < ox) pl[(oy - 1) * ox + gx] = 0.0;
        }
      }
    }
  };
  stage(zf0, sm);
  for (int zf = zf0; zf <= zf_end; ++zf) {
    const int buf = (zf - zf0) & 1;
    cp_wait_all();
    __syncthreads();  // plane zf staged; the previous plane's R1 readers are done
    if (zf + 1 <= zf_end) stage(zf + 1, sm + (buf ^ 1) * R0S);
    const double* R = sm + buf * R0S;
    // ---- x pass: (fine row ly, coarse cell lc) -> coarse x nodes lc*P + jj
    for (int e = t; e < C::LY * kZCX; e += kZT) {
      const int lc = e / C::LY, ly = e - lc * C::LY;
      const double* row = R + ly * C::LXP;
      double fv[2 * P + 1], lv[2 * P];
#pragma unroll
      for (int r = 0; r <= 2 * P; ++r) fv[r] = row[2 * P * (lc + 1) + r];
#pragma unroll
      for (int r = 0; r < 2 * P; ++r) lv[r] = row[2 * P * lc + r];
#pragma unroll
      for (int jj = 0; jj < P; ++jj) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r <= 2 * P; ++r) s = fma(Tx.hw[r][jj], fv[r], s);
        if (jj == 0) {
#pragma unroll
          for (int r = 0; r < 2 * P; ++r) s = fma(Tx.hw[r][P], lv[r], s);
        }
        R1[ly * C::MXP + lc * P + jj] = s;
      }
    }
    __syncthreads();
    // ---- y pass + z window
    const bool top = zf == 2 * P * ncz;  // the lattice's top fine plane: r = 2P of the last layer
    const int cz = top ? ncz - 1 : zf / (2 * P), r = top ? 2 * P : zf - 2 * P * (zf / (2 * P));
    if (r == 0 && zf > zf0) {
      // fine vertex plane: coarse layer cz - 1 closes
      if (cz - 1 >= C0) store_layer(cz - 1, P);
#pragma unroll
      for (int a = 0; a < P; ++a) {
        win[a][0] = win[a][P];
#pragma unroll
        for (int j = 1; j <= P; ++j) win[a][j] = 0.0;
      }
    }
    if (yitem) {
      double fv[2 * P + 1], lv[2 * P];
#pragma unroll
      for (int rr = 0; rr <= 2 * P; ++rr) fv[rr] = R1[(2 * P * (lcy + 1) + rr) * C::MXP + lxn];
#pragma unroll
      for (int rr = 0; rr < 2 * P; ++rr) lv[rr] = R1[(2 * P * lcy + rr) * C::MXP + lxn];
      double wz[P + 1];
#pragma unroll
      for (int j = 0; j <= P; ++j) wz[j] = Tz.hw[r][j];
#pragma unroll
      for (int a = 0; a < P; ++a) {
        double s = 0.0;
#pragma unroll
        for (int rr = 0; rr <= 2 * P; ++rr) s = fma(Ty.hw[rr][a], fv[rr], s);
        if (a == 0) {
#pragma unroll
          for (int rr = 0; rr < 2 * P; ++rr) s = fma(Ty.hw[rr][P], lv[rr], s);
        }
#pragma unroll
        for (int j = 0; j <= P; ++j) win[a][j] = fma(wz[j], s, win[a][j]);
      }
    }
  }
  // close the chunk's last layer; the top coarse plane too on the last chunk
  store_layer(C1 - 1, C1 == ncz ? P + 1 : P);
}

template <int P>
__global__ void __launch_bounds__(kZT, 2) xyz_prolong_kernel(const PassArgs A, const DevAxisTransfer Tx,
                                                          const DevAxisTransfer Ty, const DevAxisTransfer Tz,
                                                          const double* __restrict__ in, double* __restrict__ out,
                                                          int ntx, int nch, int zc) {
  using C = ZCfg<P>;
  extern __shared__ __align__(16) double sm[];
  double* Cb = sm;                                   // [P+1][CY][CXP] coarse planes of the open layer
  double* Zp = Cb + (P + 1) * C::CY * C::CXP;        // [CY][CXP] z-combined plane
  double* R1 = Zp + C::CY * C::CXP;                  // [CY][FXP] after the x pass
  const long long ix = A.i[0], iy = A.i[1], iz = A.i[2], ox = A.o[0], oy = A.o[1], oz = A.o[2];
  const int ncx = static_cast<int>((ix - 1) / P), ncy = static_cast<int>((iy - 1) / P),
            ncz = static_cast<int>((iz - 1) / P);
  const int tile = blockIdx.x, f = blockIdx.y / nch, ch = blockIdx.y - (blockIdx.y / nch) * nch;
  const int cx0 = (tile % ntx) * kZCX, cy0 = (tile / ntx) * kZCY;
  const int C0 = ch * zc, C1 = C0 + zc < ncz ? C0 + zc : ncz;
  const int t = threadIdx.x;
  const double* src_f = in + f * A.fs_in;
  double* dst_f = out + f * A.fs_out;
  const long long cgx0 = static_cast<long long>(cx0) * P, cgy0 = static_cast<long long>(cy0) * P;
  auto stage_layer = [&](int cz) {
    for (int e = t; e < (P + 1) * C::CY * C::CX; e += kZT) {
      const int j = e / (C::CY * C::CX), rem = e - j * (C::CY * C::CX);
      const int ly = rem / C::CX, lx = rem - ly * C::CX;
      const long long gx = cgx0 + lx, gy = cgy0 + ly, gz = static_cast<long long>(cz) * P + j;
      const bool ok = gx < ix && gy < iy &&
                      !(A.mask_in && (on_bdry(gx, ix) || on_bdry(gy, iy) || on_bdry_z(gz, iz, A.zbc))) &&
                      !(A.skip_lo_in && gz == 0);
      cp8(Cb + (j * C::CY + ly) * C::CXP + lx, src_f + (gz * iy + gy) * ix + gx, ok);
    }
    cp_commit();
  };
  const int zf_last = C1 == ncz ? 2 * P * C1 : 2 * P * C1 - 1;
  int open = -1;
  for (int zf = 2 * P * C0; zf <= zf_last; ++zf) {
    const bool top = zf == 2 * P * ncz;
    const int cz = top ? ncz - 1 : zf / (2 * P), r = top ? 2 * P : zf - 2 * P * (zf / (2 * P));
    if (cz != open) {
      __syncthreads();  // the previous layer's readers are done
      stage_layer(cz);
      cp_wait_all();
      open = cz;
    }
    __syncthreads();
    // ---- z combination of the layer's coarse planes at fine z index r
    for (int e = t; e < C::CY * C::CX; e += kZT) {
      const int ly = e / C::CX, lx = e - ly * C::CX;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j <= P; ++j) s = fma(Tz.hw[r][j], Cb[(j * C::CY + ly) * C::CXP + lx], s);
      Zp[ly * C::CXP + lx] = s;
    }
    __syncthreads();
    // ---- x pass: (coarse row ly, coarse cell lc) -> fine x nodes 2P lc + rr
    for (int e = t; e < C::CY * kZCX; e += kZT) {
      const int lc = e / C::CY, ly = e - lc * C::CY;
      if (cx0 + lc >= ncx) continue;
      const double* row = Zp + ly * C::CXP + lc * P;
      double cv[P + 1];
#pragma unroll
      for (int j = 0; j <= P; ++j) cv[j] = row[j];
#pragma unroll
      for (int rr = 0; rr <= 2 * P; ++rr) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j <= P; ++j) s = fma(Tx.hw[rr][j], cv[j], s);
        R1[ly * C::FXP + 2 * P * lc + rr] = s;  // rr = 2P: the next cell's rr = 0 (same value)
      }
    }
    __syncthreads();
    // ---- y pass: (fine x column lx, coarse y cell lc) -> fine rows, masked add
    const bool plane_out0 = A.mask_out && on_bdry_z(zf, oz, A.zbc);
    double* dst = dst_f + static_cast<long long>(zf) * oy * ox;
    auto y_item = [&](int lc, int lx) {
      const long long c = cy0 + lc, gx = 2LL * P * cx0 + lx;
      if (c >= ncy || gx >= ox) return;
      double cv[P + 1];
#pragma unroll
      for (int j = 0; j <= P; ++j) cv[j] = R1[(lc * P + j) * C::FXP + lx];
      const bool col0 = plane_out0 || (A.mask_out && on_bdry(gx, ox));
      const int rmax = c == ncy - 1 ? 2 * P : 2 * P - 1;
      double old[2 * P + 1];
#pragma unroll
      for (int rr = 0; rr <= 2 * P; ++rr) old[rr] = (A.accumulate && rr <= rmax) ? dst[(2 * P * c + rr) * ox + gx] : 0.0;
#pragma unroll
      for (int rr = 0; rr <= 2 * P; ++rr) {
        if (rr > rmax) break;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j <= P; ++j) s = fma(Ty.hw[rr][j], cv[j], s);
        const long long gy = 2 * P * c + rr;
        if (col0 || (A.mask_out && on_bdry(gy, oy))) s = 0.0;
        dst[gy * ox + gx] = old[rr] + s;
      }
    };
    // the tile's own 2P kZCX columns: whole passes of the CTA; column 2P kZCX
    // is the next tile's first one, except on the lattice's last column
    constexpr int FXO = 2 * P * kZCX;
    for (int e = t; e < FXO * kZCY; e += kZT) y_item(e / FXO, e % FXO);
    if (2LL * P * cx0 + FXO == ox - 1 && t < kZCY) y_item(t, FXO);
  }
}

template <int P>
void launch_xyz(int F, const PassArgs& A, const DevAxisTransfer* ax, bool prolong, const double* in, double* out,
                cudaStream_t s) {
  using C = ZCfg<P>;
  const long long ncx = prolong ? (A.i[0] - 1) / P : (A.o[0] - 1) / P;
  const long long ncy = prolong ? (A.i[1] - 1) / P : (A.o[1] - 1) / P;
  const long long ncz = prolong ? (A.i[2] - 1) / P : (A.o[2] - 1) / P;
  const long long ntx = (ncx + kZCX - 1) / kZCX, nty = (ncy + kZCY - 1) / kZCY;
  const long long tiles = ntx * nty;
  // prolongation: ~8 CTAs per SM-slot. Restriction: every chunk repeats one
  // halo coarse layer (2p fine planes); 4 chunks measured best at C5-64 and
  // C5-128 (4: 1.71 ms, 14: 1.86 ms)
  long long nch = std::max<long long>(1, (148LL * 3 * 8 + tiles * F - 1) / (tiles * F));
  nch = std::min<long long>(nch, std::max<long long>(1, prolong ? ncz : std::min<long long>(4, ncz / 4)));
  const long long zc = (ncz + nch - 1) / nch;
  nch = (ncz + zc - 1) / zc;
  const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(F * nch));
  count_launch();
  if (prolong) {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(xyz_prolong_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(C::p_smem()));
      configured = true;
    }
    xyz_prolong_kernel<P><<<grid, kZT, C::p_smem(), s>>>(A, ax[0], ax[1], ax[2], in, out, static_cast<int>(ntx),
                                                          static_cast<int>(nch), static_cast<int>(zc));
  } else {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(xyz_restrict_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(C::r_smem()));
      configured = true;
    }
    xyz_restrict_kernel<P><<<grid, kZT, C::r_smem(), s>>>(A, ax[0], ax[1], ax[2], in, out, static_cast<int>(ntx),
                                                           static_cast<int>(nch), static_cast<int>(zc));
  }
}

bool xyz_pass(int F, const PassArgs& A, const DevAxisTransfer* ax, bool prolong, const double* in, double* out,
              cudaStream_t s) {
  const int p = ax[0].hp;
  if (p < 1 || p > 4 || ax[1].hp != p || ax[2].hp != p) return false;
  // the z march is sequential per CTA: small levels (few planes of work per
  // CTA, latency-bound) keep the plane-parallel separable passes
  const long long fine_planes = prolong ? A.o[2] : A.i[2];
  const long long fine_plane = prolong ? A.o[0] * A.o[1] : A.i[0] * A.i[1];
  if (fine_plane < (1LL << 16) || fine_planes < 64) return false;
  switch (p) {
    case 1: launch_xyz<1>(F, A, ax, prolong, in, out, s); break;
    case 2: launch_xyz<2>(F, A, ax, prolong, in, out, s); break;
    case 3: launch_xyz<3>(F, A, ax, prolong, in, out, s); break;
    case 4: launch_xyz<4>(F, A, ax, prolong, in, out, s); break;
    default: return false;
  }
  return true;
}

// apply the per-axis maps x, then y, then z (2D: x, y); the intermediates are
// compact, the source / destination use the given field strides
void separable(const DevAxisTransfer* ax, bool prolong, int dim, int F, const long long* src_d, const long long* dst_d,
               const double* in, double* out, double* t1, double* t2, const TransferSlab& sl, cudaStream_t s) {
  auto args = [&](const long long* i, const long long* o, long long fs_in, long long fs_out, bool first, bool last) {
    PassArgs A{};
    for (int a = 0; a < 3; ++a) {
      A.i[a] = i[a];
      A.o[a] = o[a];
    }
    A.fs_in = fs_in > 0 ? fs_in : i[0] * i[1] * i[2];
    A.fs_out = fs_out > 0 ? fs_out : o[0] * o[1] * o[2];
    A.zbc = dim == 3 ? sl.zbc : 3;
    A.mask_in = first;
    A.mask_out = last;
    A.skip_lo_in = first && sl.skip_lo_in;
    A.accumulate = last && sl.accumulate;
    return A;
  };
  const long long fs_src = prolong ? sl.coarse_fstride : 0, fs_dst = prolong ? 0 : sl.coarse_fstride;
  long long d1[3] = {dst_d[0], src_d[1], src_d[2]};
  if (dim == 2) {
    pass<0>(F, args(src_d, d1, fs_src, 0, true, false), ax[0], prolong, in, t1, s);
    pass<1>(F, args(d1, dst_d, 0, fs_dst, false, true), ax[1], prolong, t1, out, s);
    return;
  }
  long long d2[3] = {dst_d[0], dst_d[1], src_d[2]};
  // equal-p h-coarsening on all three axes: one fused z-marching kernel
  if (xyz_pass(F, args(src_d, dst_d, fs_src, fs_dst, true, true), ax, prolong, in, out, s)) return;
  static const bool no_fused = std::getenv("STMG_XFER_SEPARABLE") != nullptr;
  if (!no_fused && ax[0].hp > 0 && ax[0].hp == ax[1].hp && ax[0].hp <= 4) {
    // equal-p h-coarsening in x and y: one fused x-y pass plus the z pass --
    // restriction x-y first, prolongation z first (the passes commute), so
    // the single HBM intermediate is the (coarse x, coarse y, fine z) lattice
    if (prolong) {
      long long dz[3] = {src_d[0], src_d[1], dst_d[2]};
      pass<2>(F, args(src_d, dz, fs_src, 0, true, false), ax[2], true, in, t2, s);
      xy_pass(F, args(dz, dst_d, 0, fs_dst, false, true), ax[0], ax[1], true, t2, out, s);
    } else {
      xy_pass(F, args(src_d, d2, fs_src, 0, true, false), ax[0], ax[1], false, in, t2, s);
      pass<2>(F, args(d2, dst_d, 0, fs_dst, false, true), ax[2], false, t2, out, s);
    }
    return;
  }
  pass<0>(F, args(src_d, d1, fs_src, 0, true, false), ax[0], prolong, in, t1, s);
  pass<1>(F, args(d1, d2, 0, 0, false, false), ax[1], prolong, t1, t2, s);
  pass<2>(F, args(d2, dst_d, 0, fs_dst, false, true), ax[2], prolong, t2, out, s);
}

}  // namespace

void spatial_prolong(const DevAxisTransfer* ax, int dim, int F, const long long* dc, const long long* df,
                     const double* coarse, double* fine, double* t1, double* t2, const TransferSlab& sl,
                     cudaStream_t s) {
  separable(ax, true, dim, F, dc, df, coarse, fine, t1, t2, sl, s);
}
void spatial_restrict(const DevAxisTransfer* ax, int dim, int F, const long long* dc, const long long* df,
                      const double* fine, double* coarse, double* t1, double* t2, const TransferSlab& sl,
                      cudaStream_t s) {
  separable(ax, false, dim, F, df, dc, fine, coarse, t1, t2, sl, s);
}
void temporal_prolong(const double* T, int Ff, int Fc, long long n_space, const long long* d, int dim,
                      const double* coarse, double* fine, const TransferSlab& sl, cudaStream_t s) {
  count_launch();
  temporal_kernel<<<grid_for(n_space), 256, 0, s>>>(T, Ff, Fc, false, sl.accumulate, n_space, d[0], d[1], d[2], dim,
                                                     dim == 3 ? sl.zbc : 3, false,
                                                     sl.coarse_fstride > 0 ? sl.coarse_fstride : n_space, n_space,
                                                     coarse, fine);
}
void temporal_restrict(const double* T, int Ff, int Fc, long long n_space, const long long* d, int dim,
                       const double* fine, double* coarse, const TransferSlab& sl, cudaStream_t s) {
  count_launch();
  temporal_kernel<<<grid_for(n_space), 256, 0, s>>>(T, Ff, Fc, true, sl.accumulate, n_space, d[0], d[1], d[2], dim,
                                                     dim == 3 ? sl.zbc : 3, dim == 3 && sl.skip_lo_in, n_space,
                                                     sl.coarse_fstride > 0 ? sl.coarse_fstride : n_space, fine,
                                                     coarse);
}

}  // namespace stmgb
