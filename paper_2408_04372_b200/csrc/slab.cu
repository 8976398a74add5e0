// z-slab partition helpers: interface-plane fills, in-process
// interface sums, pack / unpack of the planes exchanged with a neighbouring
// rank, and the owned-segment dot products of a distributed vector.
//
// A slab's local lattice holds its interface planes on both sides; after a
// cell loop each side holds a partial sum there, and the interface sum makes
// both copies the full value (the reference's assembled operator,
// spatial_operator.cpp:287-288, summed over the cells of both slabs).
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.hpp"

namespace stmgb {

namespace {

constexpr int kT = 256;

inline unsigned grid_for(long long n) {
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + kT - 1) / kT, 148LL * 16)));
}

__global__ void plane_fill_kernel(double* __restrict__ v, int F, long long fstride, long long off, long long len,
                                  double val) {
  const long long n = static_cast<long long>(F) * len;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long f = t / len, i = t - f * len;
    v[f * fstride + off + i] = val;
  }
}

__global__ void plane_pair_sum_kernel(double* __restrict__ a, long long aoff, long long afs, double* __restrict__ b,
                                      long long boff, long long bfs, int F, long long len) {
  const long long n = static_cast<long long>(F) * len;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long f = t / len, i = t - f * len;
    double* pa = a + f * afs + aoff + i;
    double* pb = b + f * bfs + boff + i;
    const double s = *pa + *pb;
    *pa = s;
    *pb = s;
  }
}

__global__ void plane_pack_kernel(const double* __restrict__ v, long long fstride, long long off, int F, long long len,
                                  double* __restrict__ buf) {
  const long long n = static_cast<long long>(F) * len;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long f = t / len, i = t - f * len;
    buf[t] = v[f * fstride + off + i];
  }
}

__global__ void plane_unpack_add_kernel(double* __restrict__ v, long long fstride, long long off, int F, long long len,
                                        const double* __restrict__ buf) {
  const long long n = static_cast<long long>(F) * len;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long f = t / len, i = t - f * len;
    v[f * fstride + off + i] += buf[t];
  }
}

// partial dots over the owned segments, up to 8 basis vectors per group,
// fixed grid and fixed-order second stage (reproducible)
constexpr int kDotGrid = 592;
template <int G>
__global__ void multidot_seg_kernel(const double* const* __restrict__ V, int i0, int k, const double* __restrict__ w,
                                    const DotSegments seg, double* __restrict__ partial) {
  const double* vp[G];
#pragma unroll
  for (int g = 0; g < G; ++g) vp[g] = (i0 + g < k) ? V[i0 + g] : w;
  double acc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g] = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int sg = 0; sg < seg.n; ++sg) {
    for (long long j = seg.begin[sg] + blockIdx.x * (long long)blockDim.x + threadIdx.x; j < seg.end[sg]; j += stride) {
      const double wj = __ldg(w + j);
#pragma unroll
      for (int g = 0; g < G; ++g) acc[g] = fma(__ldg(vp[g] + j), wj, acc[g]);
    }
  }
  __shared__ double red[G][kT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    double v = acc[g];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[g][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < G && i0 + threadIdx.x < k) {
    double s = 0.0;
    for (int i = 0; i < kT / 32; ++i) s += red[threadIdx.x][i];
    partial[static_cast<long long>(i0 + threadIdx.x) * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void reduce_seg_partials_kernel(const double* __restrict__ partial, int nblocks, int k,
                                           double* __restrict__ out) {
  const int i = blockIdx.x;
  if (i >= k) return;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 32) s += partial[static_cast<long long>(i) * nblocks + b];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) out[i] = s;
}

}  // namespace

void plane_fill(double* v, int F, long long fstride, long long plane, long long plane_len, double val, cudaStream_t s) {
  count_launch();
  plane_fill_kernel<<<grid_for(F * plane_len), kT, 0, s>>>(v, F, fstride, plane * plane_len, plane_len, val);
}

void plane_pair_sum(double* a, long long a_plane, double* b, long long b_plane, int F, long long a_fstride,
                    long long b_fstride, long long plane_len, cudaStream_t s) {
  count_launch();
  plane_pair_sum_kernel<<<grid_for(F * plane_len), kT, 0, s>>>(a, a_plane * plane_len, a_fstride, b,
                                                                b_plane * plane_len, b_fstride, F, plane_len);
}

void plane_pack(const double* v, int F, long long fstride, long long plane, long long plane_len, double* buf,
                cudaStream_t s) {
  count_launch();
  plane_pack_kernel<<<grid_for(F * plane_len), kT, 0, s>>>(v, fstride, plane * plane_len, F, plane_len, buf);
}

void plane_unpack_add(double* v, int F, long long fstride, long long plane, long long plane_len, const double* buf,
                      cudaStream_t s) {
  count_launch();
  plane_unpack_add_kernel<<<grid_for(F * plane_len), kT, 0, s>>>(v, fstride, plane * plane_len, F, plane_len, buf);
}

void vec_multidot_seg(const double* const* V, int k, const double* w, const DotSegments& seg, double* out,
                      double* scratch, cudaStream_t s) {
  // scratch: kDotBlocks * k doubles (kDotGrid == kDotBlocks)
  static_assert(kDotGrid == kDotBlocks, "dot grid");
  // as vec_multidot: the last group takes the smallest kernel that holds it
  for (int i0 = 0; i0 < k;) {
    const int rem = k - i0;
    count_launch();
    if (rem > 4) {
      multidot_seg_kernel<8><<<kDotGrid, kT, 0, s>>>(V, i0, k, w, seg, scratch);
      i0 += 8;
    } else if (rem > 2) {
      multidot_seg_kernel<4><<<kDotGrid, kT, 0, s>>>(V, i0, k, w, seg, scratch);
      i0 += 4;
    } else if (rem > 1) {
      multidot_seg_kernel<2><<<kDotGrid, kT, 0, s>>>(V, i0, k, w, seg, scratch);
      i0 += 2;
    } else {
      multidot_seg_kernel<1><<<kDotGrid, kT, 0, s>>>(V, i0, k, w, seg, scratch);
      i0 += 1;
    }
  }
  count_launch();
  reduce_seg_partials_kernel<<<k, 32, 0, s>>>(scratch, kDotGrid, k, out);
}

}  // namespace stmgb
