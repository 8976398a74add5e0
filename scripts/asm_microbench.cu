// Microbenchmark of cell-block smoother apply variants at C2 size
// (262,144 cells, m = 64 local dofs, n_t = 3): z_T += X (D^-1 (X^T r_T)).
// Variants: 0 TMA streaming only (lower bound), 1 scalar FMA (one output per
// thread), 2 FP64 tensor-core mma.sync.m8n8k4 on an XOR-swizzled X layout.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o asm_mb asm_microbench.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

constexpr int M = 64, NT = 3;
constexpr int XS = M * M;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(b) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* bar, unsigned ph) {
  unsigned ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok)
               : "r"(smem_u32(bar)), "r"(ph)
               : "memory");
  return ok;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned ph) {
  for (long long i = 0; !mbar_try(bar, ph); ++i)
    if (i > (1LL << 28)) __trap();
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// swizzled position of X[a][e] inside a cell block
__host__ __device__ __forceinline__ int swz(int a, int e) { return a * M + (e ^ ((a & 7) << 2)); }

// simple per-eigen diagonal "solve": hat z = hat r / (1 + lam)
template <int VAR, int NTH>
__global__ void __launch_bounds__(NTH) apply_kernel(long long n_cells, const double* __restrict__ X,
                                                    const double* __restrict__ lam, const double* __restrict__ r,
                                                    double* __restrict__ z) {
  extern __shared__ __align__(128) double sm[];
  double* Xb[2] = {sm, sm + XS};
  double* rs = sm + 2 * XS;    // [M][8]
  double* hs = rs + 8 * M;     // [M][8]
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(hs + 8 * M);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long cell = blockIdx.x;
  if (t == 0 && cell < n_cells) {
    mbar_expect_tx(&bar[0], XS * 8);
    bulk(Xb[0], X + cell * XS, XS * 8, &bar[0]);
  }
  unsigned ph[2] = {0, 0};
  int buf = 0;
  for (; cell < n_cells; cell += gridDim.x) {
    const long long next = cell + gridDim.x;
    if (VAR != 6 && t == 0 && next < n_cells) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bar[buf ^ 1], XS * 8);
      bulk(Xb[buf ^ 1], X + next * XS, XS * 8, &bar[buf ^ 1]);
    }
    // residual of the block: synthetic gather (contiguous per cell)
    if (t < M) {
      for (int i = 0; i < 8; ++i) rs[t * 8 + i] = i < NT ? r[(cell * M + t) * NT + i] : 0.0;
    }
    if (VAR != 6 || cell == blockIdx.x) {
      mbar_wait(&bar[buf], ph[buf]);
      ph[buf] ^= 1;
    }
    __syncthreads();
    const double* Xs = VAR == 6 ? Xb[0] : Xb[buf];
    if (VAR == 0) {
      if (t < M) z[(cell * M + t) * NT] += Xs[t * M + t];
    } else if (VAR == 1) {
      // scalar: threads 0..63 own eigen-index e / local dof a
      if (t < M) {
        double acc[NT] = {0, 0, 0};
#pragma unroll 16
        for (int a = 0; a < M; ++a) {
          const double x = Xs[a * M + t];
#pragma unroll
          for (int i = 0; i < NT; ++i) acc[i] = fma(x, rs[a * 8 + i], acc[i]);
        }
        const double d = 1.0 / (1.0 + lam[cell * M + t]);
#pragma unroll
        for (int i = 0; i < NT; ++i) hs[t * 8 + i] = acc[i] * d;
      }
      __syncthreads();
      if (t < M) {
        double acc[NT] = {0, 0, 0};
        int e = t;
#pragma unroll 16
        for (int j = 0; j < M; ++j) {
          const double x = Xs[t * M + e];
#pragma unroll
          for (int i = 0; i < NT; ++i) acc[i] = fma(x, hs[e * 8 + i], acc[i]);
          e = (e + 1) & (M - 1);
        }
#pragma unroll
        for (int i = 0; i < NT; ++i) atomicAdd(z + (cell * M + t) * NT + i, acc[i]);
      }
    } else if (VAR == 7) {
      if (t < M) {
        for (int i = 0; i < NT; ++i) atomicAdd(z + (cell * M + t) * NT + i, Xs[t * M + i]);
      }
    } else if (VAR == 3 || VAR == 4 || VAR == 5 || VAR == 6) {
      // tensor cores, independent accumulator chains:
      // VAR 3: 8 warps, one 8-row tile each, k split into 2 chains
      // VAR 4: 4 warps, two 8-row tiles each interleaved, k split into 2 chains
      constexpr int TPW = VAR == 4 ? 2 : 1;
      double d[TPW][2][2];
#pragma unroll
      for (int q = 0; q < TPW; ++q) d[q][0][0] = d[q][0][1] = d[q][1][0] = d[q][1][1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < M / 4; ++kt) {
        const int a = kt * 4 + (lane & 3);
        const double bv = rs[a * 8 + (lane >> 2)];
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
          const int e = (warp * TPW + q) * 8 + (lane >> 2);
          const double av = Xs[swz(a, e)];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(d[q][kt & 1][0]), "+d"(d[q][kt & 1][1])
                       : "d"(av), "d"(bv));
        }
      }
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        const int e = (warp * TPW + q) * 8 + (lane >> 2);
        const int col = (lane & 3) * 2;
        const double dd = 1.0 / (1.0 + lam[cell * M + e]);
        hs[e * 8 + col] = (d[q][0][0] + d[q][1][0]) * dd;
        hs[e * 8 + col + 1] = (d[q][0][1] + d[q][1][1]) * dd;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < TPW; ++q) d[q][0][0] = d[q][0][1] = d[q][1][0] = d[q][1][1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < M / 4; ++kt) {
        const int e = kt * 4 + (lane & 3);
        const double bv = hs[e * 8 + (lane >> 2)];
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
          const int a = (warp * TPW + q) * 8 + (lane >> 2);
          const double av = Xs[swz(a, e)];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(d[q][kt & 1][0]), "+d"(d[q][kt & 1][1])
                       : "d"(av), "d"(bv));
        }
      }
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        const int a = (warp * TPW + q) * 8 + (lane >> 2);
        const int col = (lane & 3) * 2;
        if (VAR == 5) {
          if (col < NT) z[(cell * M + a) * NT + col] = d[q][0][0] + d[q][1][0];
          if (col + 1 < NT) z[(cell * M + a) * NT + col + 1] = d[q][0][1] + d[q][1][1];
        } else {
          if (col < NT) atomicAdd(z + (cell * M + a) * NT + col, d[q][0][0] + d[q][1][0]);
          if (col + 1 < NT) atomicAdd(z + (cell * M + a) * NT + col + 1, d[q][0][1] + d[q][1][1]);
        }
      }
    } else {
      // tensor cores: 4 warps x 2 row tiles of 8; X swizzled (swz)
      // product 1: hat r (e x 8) = X^T (e x a) * r (a x 8)
      for (int mt = warp * 2; mt < warp * 2 + 2; ++mt) {
        double d0 = 0.0, d1 = 0.0;
        const int e = mt * 8 + (lane >> 2);
#pragma unroll
        for (int kt = 0; kt < M / 4; ++kt) {
          const int a = kt * 4 + (lane & 3);
          const double av = Xs[swz(a, e)];                       // A[row=e][col=a]
          const double bv = rs[(kt * 4 + (lane & 3)) * 8 + (lane >> 2)];  // B[row=a][col]
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(d0), "+d"(d1)
                       : "d"(av), "d"(bv));
        }
        const int col = (lane & 3) * 2;
        const double dd = 1.0 / (1.0 + lam[cell * M + e]);
        hs[e * 8 + col] = d0 * dd;
        hs[e * 8 + col + 1] = d1 * dd;
      }
      __syncthreads();
      // product 2: z (a x 8) = X (a x e) * hat z (e x 8)
      for (int mt = warp * 2; mt < warp * 2 + 2; ++mt) {
        double d0 = 0.0, d1 = 0.0;
        const int a = mt * 8 + (lane >> 2);
#pragma unroll
        for (int kt = 0; kt < M / 4; ++kt) {
          const int e = kt * 4 + (lane & 3);
          const double av = Xs[swz(a, e)];                        // A[row=a][col=e]
          const double bv = hs[(kt * 4 + (lane & 3)) * 8 + (lane >> 2)];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(d0), "+d"(d1)
                       : "d"(av), "d"(bv));
        }
        const int col = (lane & 3) * 2;
        if (col < NT) atomicAdd(z + (cell * M + a) * NT + col, d0);
        if (col + 1 < NT) atomicAdd(z + (cell * M + a) * NT + col + 1, d1);
      }
    }
    __syncthreads();
    buf ^= 1;
  }
}

int main(int argc, char** argv) {
  const long long n_cells = argc > 1 ? atoll(argv[1]) : 262144;
  const size_t xb = sizeof(double) * XS * n_cells;
  double *X, *Xsw, *lam, *r, *z;
  CK(cudaMalloc(&X, xb));
  CK(cudaMalloc(&Xsw, xb));
  CK(cudaMalloc(&lam, sizeof(double) * M * n_cells));
  CK(cudaMalloc(&r, sizeof(double) * M * NT * n_cells));
  CK(cudaMalloc(&z, sizeof(double) * M * NT * n_cells));
  {
    // deterministic fill on host for a small prefix, device memset pattern for the rest
    std::vector<double> h(XS);
    for (int i = 0; i < XS; ++i) h[i] = std::sin(0.37 * i + 1.0) / 8.0;
    std::vector<double> hs(XS);
    for (int a = 0; a < M; ++a)
      for (int e = 0; e < M; ++e) hs[swz(a, e)] = h[a * M + e];
    for (long long c = 0; c < n_cells; c += 1) {
      CK(cudaMemcpyAsync(X + c * XS, h.data(), sizeof(double) * XS, cudaMemcpyHostToDevice));
      CK(cudaMemcpyAsync(Xsw + c * XS, hs.data(), sizeof(double) * XS, cudaMemcpyHostToDevice));
      if (c > 64) break;
    }
    std::vector<double> hl(M * n_cells), hr(M * NT * n_cells);
    for (size_t i = 0; i < hl.size(); ++i) hl[i] = 0.5 + (i % 7) * 0.1;
    for (size_t i = 0; i < hr.size(); ++i) hr[i] = std::cos(0.11 * i);
    CK(cudaMemcpy(lam, hl.data(), sizeof(double) * hl.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(r, hr.data(), sizeof(double) * hr.size(), cudaMemcpyHostToDevice));
  }
  const size_t smem = sizeof(double) * (2 * XS + 16 * M) + 16;
  auto run = [&](int var, const double* Xp, int reps) {
    void (*k)(long long, const double*, const double*, const double*, double*) = nullptr;
    switch (var) {
      case 0: k = apply_kernel<0, 128>; break;
      case 1: k = apply_kernel<1, 128>; break;
      case 2: k = apply_kernel<2, 128>; break;
      case 3: k = apply_kernel<3, 256>; break;
      case 4: k = apply_kernel<4, 128>; break;
      case 5: k = apply_kernel<5, 256>; break;
      case 6: k = apply_kernel<6, 256>; break;
      default: k = apply_kernel<7, 256>; break;
    }
    const int nth = (var == 3 || var >= 5) ? 256 : 128;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, nth, smem));
    const long long grid = std::min<long long>(n_cells, 148LL * per_sm);
    CK(cudaMemset(z, 0, sizeof(double) * M * NT * n_cells));
    k<<<grid, nth, smem>>>(n_cells, Xp, lam, r, z);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) k<<<grid, nth, smem>>>(n_cells, Xp, lam, r, z);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("variant %d: %.3f ms  (%.0f GB/s of X stream, %d CTAs/SM)\n", var, ms, xb / (ms * 1e-3) / 1e9, per_sm);
    return ms;
  };
  run(0, X, 5);
  run(1, X, 5);
  run(2, Xsw, 5);
  run(3, Xsw, 5);
  run(4, Xsw, 5);
  run(5, Xsw, 5);
  run(6, Xsw, 5);
  run(7, Xsw, 5);
  // correctness: compare variant 1 vs 2 on cell 0..15 outputs (one launch each)
  std::vector<double> z1(M * NT * 16), z2(M * NT * 16);
  CK(cudaMemset(z, 0, sizeof(double) * M * NT * n_cells));
  {
    auto k = apply_kernel<1, 128>;
    k<<<148, 128, smem>>>(16, X, lam, r, z);
    CK(cudaMemcpy(z1.data(), z, sizeof(double) * z1.size(), cudaMemcpyDeviceToHost));
  }
  CK(cudaMemset(z, 0, sizeof(double) * M * NT * n_cells));
  {
    auto k = apply_kernel<3, 256>;
    k<<<148, 256, smem>>>(16, Xsw, lam, r, z);
    CK(cudaMemcpy(z2.data(), z, sizeof(double) * z2.size(), cudaMemcpyDeviceToHost));
  }
  double err = 0, nrm = 0;
  for (size_t i = 0; i < z1.size(); ++i) {
    err += (z1[i] - z2[i]) * (z1[i] - z2[i]);
    nrm += z1[i] * z1[i];
  }
  printf("mma vs scalar rel diff %.3e (norm %.3e)\n", std::sqrt(err / nrm), std::sqrt(nrm));
  return 0;
}
