// Owner-computes space-time operator on Cartesian levels whose coefficient
// is constant on every z layer of cells (every level of C4 and C5):
//   y = S u          (SpaceTimeOperator::apply, space_time_operator.cpp:45-130)
//   r = f - S u      (the residual f - S u of multigrid.cpp:174-185)
// with the Dirichlet identity rows (space_time_operator.cpp:125-129) written
// in the same pass -- no memset of y, no copy of f, no boundary kernel and
// no atomics: every output dof is written exactly once, by the CTA owning it.
//
// Why this is exact. On a uniform axis-aligned lattice the reference's cell
// matrices (Gauss rule with q = p + 1 points, spatial_operator.cpp:129-185)
// are Kronecker products of the [0,1] element matrices Mr = B^T W B and
// Kr = D^T W D, and with rho depending on z only the assembled spatial
// operators factor into ASSEMBLED 1D operators along x and y:
//   M = Mz (x) My (x) Mx,
//   A = sum_ez rho_ez [Mz^e (x) (Ky/hy^2 (x) Mx + My (x) Kx/hx^2) + Kz^e/hz^2 (x) My (x) Mx]
// so a CTA owning a tile of x-y lattice nodes needs u only on the tile plus
// p nodes of halo on the low side and 1 node on the high side, and each
// assembled 1D product costs one even-odd element product per element plus
// one add per shared vertex -- half the arithmetic of the per-cell form
// (st_cart.cuh), whose 125 cell dofs cover 64 owned ones for p = 4.
//
// Schedule. Grid = (x-y tiles) x (z chunks). A CTA marches its chunk plane by
// plane, PB planes per batch:
//   Y: thread = (x column of the input box, field, plane): loads the column
//      of u from HBM (Dirichlet and out-of-domain inputs zeroed,
//      spatial_operator.cpp:304-307), a = My u, b = Ky u on the owned rows
//      -> shared memory
//   X: thread = (owned row, field, plane): c = Mx a, pre = Kx a / hx^2 +
//      Mx b / hy^2 on the owned columns -> shared memory
//   Z: thread = owned (x, y) point (and field group): temporal block
//      coupling of all F fields (space_time_operator.cpp:59-89 through the
//      block coefficients CM / CA, :269-317), then the z element products of
//      the plane's layer(s) accumulated into the per-thread z window held in
//      registers; when a layer closes, its p planes are final and are stored
//      (residual: f - S u read and written in the same step).
// The z chunk additionally processes the layer below it (halo) so the
// chunk's first plane receives both layers' contributions.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <type_traits>

#include "kernels.hpp"
#include "st_cart.cuh"

namespace stmgb {
namespace stb {

using stc::EO;

constexpr int kThreads = 256;

template <int N, int F>
struct Cfg {
  static constexpr int P = N - 1;
  static constexpr int FG = F > 4 ? 2 : 1;          // field groups in stage Z
  static constexpr int FPG = (F + FG - 1) / FG;      // fields per group
  static constexpr int OX = 16;                      // owned nodes per tile (x)
  static constexpr int OY = FG == 1 ? 16 : 8;        // owned nodes per tile (y)
  static constexpr int TX = OX / P, TY = OY / P;     // cells per tile
  static constexpr int WX = OX + P + 1, WY = OY + P + 1;  // input box
#ifndef STB_PB4
#define STB_PB4 2
#endif
#ifndef STB_MINB
#define STB_MINB 2
#endif
  static constexpr int PB = F > 4 ? 1 : (F > 2 ? STB_PB4 : 2);  // planes per batch
  static constexpr int XP = WX;                      // AB row pitch (odd: conflict-free rows)
  static constexpr int CPP = OX + 1;                 // CP row pitch
  // block strides padded to WX (mod 16): the stage-Y threads t = x + WX * block
  // then address word t (mod 16) -- conflict-free 64-bit shared accesses
  static constexpr int pad16(int base, int want) { return base + (((want - base) % 16) + 16) % 16; }
  static constexpr int AB_F = pad16(OY * XP, WX);    // one (field, plane) of a / b
  static constexpr int CP_F = OY * CPP;              // one (field, plane) of c / pre
  static constexpr int AB = PB * F * AB_F;
  static constexpr int CP = PB * F * CP_F;
  static constexpr int UB_F = pad16(WY * WX, WX);     // one (field, plane) of the staged u box
  static constexpr int UB = PB * F * UB_F;
  static constexpr int XH = 2;                        // stage-X items per row (halves)
  static constexpr size_t smem_bytes() { return sizeof(double) * (2 * static_cast<size_t>(AB + CP) + UB); }
  static_assert(OX % P == 0 && OY % P == 0, "tile must hold whole cells");
  static_assert(OX * OY * FG == kThreads, "one stage-Z item per thread");
  static_assert(WX * F * PB <= kThreads && XH * OY * F * PB <= kThreads, "stage Y / X items per thread");
  static_assert((OX / P) % XH == 0, "stage-X halves hold whole cells");
};

// se/so of one element (the even / odd halves of E and O applied to the
// element's split input)
template <int N>
struct Split {
  double e[EO<N>::HE];
  double o[EO<N>::H > 0 ? EO<N>::H : 1];
};
template <int N>
__device__ __forceinline__ Split<N> split_at(const double* v) {
  Split<N> s;
#pragma unroll
  for (int k = 0; k < EO<N>::H; ++k) {
    s.e[k] = v[k] + v[N - 1 - k];
    s.o[k] = v[k] - v[N - 1 - k];
  }
  if constexpr (N % 2 == 1) s.e[EO<N>::H] = v[EO<N>::H];
  return s;
}
// out[j] (j = 0..N-1) of the element product with (E, O)
template <int N>
__device__ __forceinline__ void elem(const double (&E)[3][3], const double (&O)[2][2], const Split<N>& s,
                                     double (&out)[N]) {
  double se[EO<N>::HE], so[EO<N>::H > 0 ? EO<N>::H : 1];
#pragma unroll
  for (int i = 0; i < EO<N>::HE; ++i) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < EO<N>::HE; ++k) t = fma(E[i][k], s.e[k], t);
    se[i] = t;
  }
#pragma unroll
  for (int i = 0; i < EO<N>::H; ++i) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < EO<N>::H; ++k) t = fma(O[i][k], s.o[k], t);
    so[i] = t;
  }
#pragma unroll
  for (int i = 0; i < EO<N>::H; ++i) {
    out[i] = se[i] + so[i];
    out[N - 1 - i] = se[i] - so[i];
  }
  if constexpr (N % 2 == 1) out[EO<N>::H] = se[EO<N>::H];
}
// last entry (j = N-1) of the element product only (halo element)
template <int N>
__device__ __forceinline__ double elem_last(const double (&E)[3][3], const double (&O)[2][2], const Split<N>& s) {
  double se = 0.0, so = 0.0;
#pragma unroll
  for (int k = 0; k < EO<N>::HE; ++k) se = fma(E[0][k], s.e[k], se);
#pragma unroll
  for (int k = 0; k < EO<N>::H; ++k) so = fma(O[0][k], s.o[k], so);
  return se - so;
}

// 8-byte asynchronous global -> shared copy; bytes = 0 fills zeros
__device__ __forceinline__ void cp_async8(double* dst, const double* src, int bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <int N, int F, bool RES>
__global__ void __launch_bounds__(kThreads, STB_MINB)
    st_brick_kernel(const __grid_constant__ DevLevel L, const double* __restrict__ u, const double* __restrict__ fvec,
                    double* __restrict__ y, int ntx, int zc) {
  using C = Cfg<N, F>;
  constexpr int P = C::P, OX = C::OX, OY = C::OY, WX = C::WX, WY = C::WY, PB = C::PB, FPG = C::FPG;
  extern __shared__ __align__(16) double smem[];
  double* Aa = smem;
  double* Ab = Aa + C::AB;
  double* Cc = Ab + C::AB;
  double* Cp = Cc + C::CP;
  double* Ub = Cp + C::CP;

  const int t = threadIdx.x;
  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  const long long X0 = static_cast<long long>(tx) * OX, Y0 = static_cast<long long>(ty) * OY;
  const long long dx = L.dofs[0], dy = L.dofs[1], dz = L.dofs[2];
  const long long dxy = dx * dy, ns = L.n_space;
  const int ncz = static_cast<int>(L.cells[2]);
  const int L0 = static_cast<int>(blockIdx.y) * zc;
  const int L1 = L0 + zc < ncz ? L0 + zc : ncz;
  const int Ls = L0 > 0 ? L0 - 1 : 0;  // first layer processed (halo)
  const int z_first = Ls * P, z_last = L1 * P;
  const bool lo_dir = (L.zbc & 1) != 0, hi_dir = (L.zbc & 2) != 0;
  const double V = L.h[0] * L.h[1] * L.h[2];
  const double sx = L.hinv2[0], sy = L.hinv2[1], sz = L.hinv2[2];
  auto rho_of = [&](int e) -> double {
    if (!L.rho0) return 1.0;
    const long long az = (e + L.cz0) >> L.rho_shift;
    return __ldg(L.rho0 + az * L.cells0[1] * L.cells0[0]);
  };

  // stage-Z identity of this thread
  const int g = t / (OX * OY);                 // field group
  const int pt = t - g * (OX * OY);
  const int zx = pt % OX, zy = pt / OX;
  const long long gx = X0 + zx, gy = Y0 + zy;
  const int f0 = g * FPG;
  // the point is written by this CTA if it lies on the lattice; x / y end
  // planes (always Dirichlet) are written by the tile containing them, or by
  // the last tile's border threads when the tile ends exactly on them
  const bool on_lat = gx < dx && gy < dy;
  const long long pbase = gy * dx + gx;
  const bool xend_extra = (zx == OX - 1) && (X0 + OX == dx - 1);
  const bool yend_extra = (zy == OY - 1) && (Y0 + OY == dy - 1);

  double win[FPG][N];  // z window of the open layer, per own field
#pragma unroll
  for (int i = 0; i < FPG; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) win[i][j] = 0.0;

  // store one output plane zz of the own fields (value v[i] per field)
  // Dirichlet row: u (residual f - u); on a slab's low interface plane the
  // row belongs to the slab below, this copy holds 0 (the interface sum adds it)
  auto store_dir = [&](long long x, long long yy, long long zz) {
    const bool other = zz == 0 && !lo_dir;
#pragma unroll
    for (int i = 0; i < FPG; ++i) {
      const int f = f0 + i;
      if (f >= F) break;
      const long long idx = f * ns + zz * dxy + yy * dx + x;
      if (other) {
        y[idx] = 0.0;
      } else {
        const double uv = __ldg(u + idx);
        y[idx] = RES ? __ldg(fvec + idx) - uv : uv;
      }
    }
  };
  // residual: pull the f entries of layer e's owned planes towards L2 when
  // the layer opens; they are read when it closes, p planes later
  auto prefetch_layer = [&](int e) {
    if (!RES || !on_lat || e < L0) return;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const long long base = f0 * ns + static_cast<long long>(e * P + q) * dxy + pbase;
#pragma unroll
      for (int i = 0; i < FPG; ++i) {
        if (f0 + i >= F) break;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(fvec + base + i * ns));
      }
    }
  };
  auto store_plane = [&](long long zz, int jw) {
    const bool zdir = (zz == 0 && lo_dir) || (zz == dz - 1 && hi_dir);
    if (on_lat) {
      const bool dir = zdir || gx == 0 || gy == 0 || gx == dx - 1 || gy == dy - 1;
      if (dir) {
        store_dir(gx, gy, zz);
      } else {
        const bool no_f = (zz == 0 && !lo_dir);  // low interface plane: f counted by the slab below
        const long long base = f0 * ns + zz * dxy + pbase;
        double out[FPG];
        if (C::FG == 1 && L.g_ok) {
#pragma unroll
          for (int i = 0; i < FPG; ++i) {
            double v = 0.0;
#pragma unroll
            for (int h = 0; h < F; ++h) v = fma(L.CA[i * F + h], win[h][jw], v);
            out[i] = v;
          }
        } else {
#pragma unroll
          for (int i = 0; i < FPG; ++i) out[i] = win[i][jw];
        }
#pragma unroll
        for (int i = 0; i < FPG; ++i) {
          if (f0 + i >= F) break;
          const long long idx = base + i * ns;
          if (RES)
            y[idx] = no_f ? -out[i] : __ldg(fvec + idx) - out[i];
          else
            y[idx] = out[i];
        }
      }
    }
    if (xend_extra && gy < dy) store_dir(dx - 1, gy, zz);
    if (yend_extra && gx < dx) store_dir(gx, dy - 1, zz);
    if (xend_extra && yend_extra) store_dir(dx - 1, dy - 1, zz);
  };

  // stage-Y identity: one column (x, field, plane slot) of the input box;
  // the thread stages its own column of u into Ub (cp.async, Dirichlet and
  // out-of-domain entries zero-filled) and later reads it back, so no
  // barrier orders the staging
  const bool ycol = t < WX * F * PB;
  const int yx = t % WX, yf = (t / WX) % F, yb = t / (WX * F);
  int rlo = 0, rhi = 0;  // rows [rlo, rhi) of the column lie inside the lattice, off its Dirichlet faces
  const double* ybase = u;
  {
    const long long gxx = X0 - P + yx;
    if (gxx > 0 && gxx < dx - 1) {
      rlo = static_cast<int>(Y0 - P) < 1 ? static_cast<int>(1 - (Y0 - P)) : 0;
      const long long rmax = dy - 1 - (Y0 - P);  // first row at or beyond the high face
      rhi = rmax < WY ? static_cast<int>(rmax) : WY;
      ybase = u + yf * ns + (Y0 - P + rlo) * dx + gxx;
    }
  }
  double* ycolbuf = Ub + (yb * F + yf) * C::UB_F + yx;
  auto stage_u = [&](int zb, int nb) {
    if (!ycol || yb >= nb) return;
    const int z = zb + yb;
    const bool zd = (z == 0 && lo_dir) || (z == dz - 1 && hi_dir);
    const double* src = ybase + z * dxy;
    if (!zd && rlo == 0 && rhi == WY) {
#pragma unroll
      for (int r = 0; r < WY; ++r) cp_async8(ycolbuf + r * WX, src + r * dx, 8);
    } else {
#pragma unroll
      for (int r = 0; r < WY; ++r) {
        const bool ok = !zd && r >= rlo && r < rhi;
        cp_async8(ycolbuf + r * WX, ok ? src + (r - rlo) * dx : u, ok ? 8 : 0);
      }
    }
    cp_async_commit();
  };
  stage_u(z_first, z_last - z_first + 1 < PB ? z_last - z_first + 1 : PB);
  prefetch_layer(Ls);

  for (int zb = z_first; zb <= z_last; zb += PB) {
    const int nb = z_last - zb + 1 < PB ? z_last - zb + 1 : PB;
    // ---- Y: columns of u along y on the input box
    if (ycol && yb < nb) {
      const int x = yx, f = yf, b = yb;
      {
        cp_async_wait_all();
        // this thread's column is consumed element by element below; the next
        // batch's column is staged once the last element has been read
        double* oa = Aa + (b * F + f) * C::AB_F + x;
        double* ob = Ab + (b * F + f) * C::AB_F + x;
        // element 0 is the halo cell: it reaches owned row 0 only
        double v[N];
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = ycolbuf[k * WX];
        double ca, cb;
        {
          const Split<N> s = split_at<N>(v);
          ca = elem_last<N>(L.MrE, L.MrO, s);
          cb = elem_last<N>(L.KrE, L.KrO, s);
        }
#pragma unroll
        for (int e = 1; e <= OY / P; ++e) {
          v[0] = v[P];
#pragma unroll
          for (int k = 1; k < N; ++k) v[k] = ycolbuf[(e * P + k) * WX];
          if (e == OY / P && zb + PB <= z_last)
            stage_u(zb + PB, z_last - zb - PB + 1 < PB ? z_last - zb - PB + 1 : PB);
          const Split<N> s = split_at<N>(v);
          double ea[N], eb[N];
          elem<N>(L.MrE, L.MrO, s, ea);
          elem<N>(L.KrE, L.KrO, s, eb);
          const int r0 = (e - 1) * P;
          oa[r0 * C::XP] = ca + ea[0];
          ob[r0 * C::XP] = cb + eb[0];
#pragma unroll
          for (int j = 1; j < P; ++j) {
            oa[(r0 + j) * C::XP] = ea[j];
            ob[(r0 + j) * C::XP] = eb[j];
          }
          ca = ea[P];
          cb = eb[P];
        }
      }
    }
    __syncthreads();
    // ---- X: half rows of a / b along x -> c, pre on the owned columns
    if (t < C::XH * OY * F * PB) {
      constexpr int HX = OX / C::XH;  // owned columns per half
      const int h = t % C::XH, rfb = t / C::XH;
      const int r = rfb % OY, fb = rfb / OY;
      const int f = fb % F, b = fb / F;
      if (b < nb) {
        const double* ia = Aa + (b * F + f) * C::AB_F + r * C::XP + h * HX;
        const double* ib = Ab + (b * F + f) * C::AB_F + r * C::XP + h * HX;
        double* oc = Cc + (b * F + f) * C::CP_F + r * C::CPP + h * HX;
        double* op = Cp + (b * F + f) * C::CP_F + r * C::CPP + h * HX;
        double va[N], vb[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          va[k] = ia[k];
          vb[k] = ib[k];
        }
        double cc, cp;
        {
          const Split<N> sa = split_at<N>(va), sb = split_at<N>(vb);
          cc = elem_last<N>(L.MrE, L.MrO, sa);
          cp = fma(sx, elem_last<N>(L.KrE, L.KrO, sa), sy * elem_last<N>(L.MrE, L.MrO, sb));
        }
#pragma unroll
        for (int e = 1; e <= HX / P; ++e) {
          va[0] = va[P];
          vb[0] = vb[P];
#pragma unroll
          for (int k = 1; k < N; ++k) {
            va[k] = ia[e * P + k];
            vb[k] = ib[e * P + k];
          }
          const Split<N> sa = split_at<N>(va), sb = split_at<N>(vb);
          double ec[N], ek[N], em[N];
          elem<N>(L.MrE, L.MrO, sa, ec);
          elem<N>(L.KrE, L.KrO, sa, ek);
          elem<N>(L.MrE, L.MrO, sb, em);
          const int r0 = (e - 1) * P;
          oc[r0] = cc + ec[0];
          op[r0] = cp + fma(sx, ek[0], sy * em[0]);
#pragma unroll
          for (int j = 1; j < P; ++j) {
            oc[r0 + j] = ec[j];
            op[r0 + j] = fma(sx, ek[j], sy * em[j]);
          }
          cc = ec[P];
          cp = fma(sx, ek[P], sy * em[P]);
        }
      }
    }
    __syncthreads();
    // ---- Z: temporal coupling and the z element products
    for (int b = 0; b < nb; ++b) {
      const int z = zb + b;
      const int e_of = z / P, j = z - e_of * P;
      double cmc[FPG], cap[FPG], cac[FPG];
#pragma unroll
      for (int i = 0; i < FPG; ++i) cmc[i] = cap[i] = cac[i] = 0.0;
      const double* ic = Cc + b * F * C::CP_F + zy * C::CPP + zx;
      const double* ip = Cp + b * F * C::CP_F + zy * C::CPP + zx;
      if (C::FG == 1 && L.g_ok) {
        // (CA (x) I)(G (x) M + I (x) A): G c on the point, CA at the store
#pragma unroll
        for (int gg = 0; gg < F; ++gg) {
          const double vc = ic[gg * C::CP_F];
          cap[gg] = ip[gg * C::CP_F];
          cac[gg] = vc;
#pragma unroll
          for (int i = 0; i < F; ++i) cmc[i] = fma(L.G[i * F + gg], vc, cmc[i]);
        }
      } else {
#pragma unroll
        for (int gg = 0; gg < F; ++gg) {
          const double vc = ic[gg * C::CP_F], vp = ip[gg * C::CP_F];
#pragma unroll
          for (int i = 0; i < FPG; ++i) {
            const int f = (C::FG == 1 ? 0 : f0) + i;
            if (f >= F) break;
            const double cm = L.CM[f * F + gg], ca = L.CA[f * F + gg];
            cmc[i] = fma(cm, vc, cmc[i]);
            cap[i] = fma(ca, vp, cap[i]);
            cac[i] = fma(ca, vc, cac[i]);
          }
        }
      }
      // contribution of this plane to layer e at local index jl
      auto add_layer = [&](int e, int jl) {
        const double rho = rho_of(e);
        const double rv = rho * V * sz;
        double mc[N], kc[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
          mc[q] = L.Mr[q][jl];
          kc[q] = L.Kr[q][jl];
        }
#pragma unroll
        for (int i = 0; i < FPG; ++i) {
          const double zm = V * fma(rho, cap[i], cmc[i]);
          const double zk = rv * cac[i];
#pragma unroll
          for (int q = 0; q < N; ++q) win[i][q] = fma(mc[q], zm, fma(kc[q], zk, win[i][q]));
        }
      };
      if (j == 0 && z > z_first) {
        // vertex plane: close layer e - 1; its p lower planes are final
        const int e = e_of - 1;
        add_layer(e, P);
        if (e >= L0) {
#pragma unroll
          for (int q = 0; q < P; ++q) store_plane(e * P + q, q);
        }
#pragma unroll
        for (int i = 0; i < FPG; ++i) {
          win[i][0] = win[i][P];
#pragma unroll
          for (int q = 1; q < N; ++q) win[i][q] = 0.0;
        }
        if (z < z_last) prefetch_layer(e_of);
      }
      if (z < z_last) add_layer(e_of, j);
    }
  }
  // the slab's top plane: Dirichlet, or an interface partial sum
  if (L1 == ncz) store_plane(z_last, 0);
}


// ---------------------------------------------------------------------------
// Warp-specialised form of the same schedule (F <= 4). The stages run as
// groups of warps on different planes at the same time, coupled by
// shared-memory rings and mbarriers instead of CTA-wide barriers:
//   loader warp: stages the (WY x WX) input box of every field of a plane
//            with 8-byte cp.async (Dirichlet and out-of-domain inputs
//            zero-filled, spatial_operator.cpp:304-307), NSU planes ahead;
//            completion is counted on the ring's mbarrier
//   Y warps: column (x, field) of the box: a = My u, b = Ky u -> ring AB
//   X warps: half row (row, field): c = Mx a, pre = Kx a / hx^2 + Mx b / hy^2
//            -> ring CP
//   Z warps: owned point: temporal coupling, z window in registers, stores
// so no warp idles while another stage runs (the barrier after stage Y held
// 18 % of the stall samples of st_brick_kernel: 168 of 256 threads have a
// stage-Y item), and each group keeps only its own tables in registers.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// the executing thread's earlier cp.async copies arrive on the barrier when they land
__device__ __forceinline__ void cp_async_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
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
// bounded wait: a ring that never advances traps instead of hanging the GPU
// (back-off sleeps of 50 - 400 ns between polls measured the same as none)
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  for (unsigned spin = 0; !mbar_try_wait(bar, phase); ++spin)
    if (spin > (1u << 24)) __trap();
}
__device__ __forceinline__ void cp_async8_s(unsigned dst, const double* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}

#ifndef STB_NSU
#define STB_NSU 4
#endif
#ifndef STB_NSA
#define STB_NSA 3
#endif
#ifndef STB_NSC
#define STB_NSC 3
#endif

template <int N, int F>
struct WsCfg {
  using C = Cfg<N, F>;
  static_assert(C::FG == 1, "warp-specialised form: all fields in one stage-Z thread");
  static constexpr int YI = C::WX * F;            // stage-Y items per plane
  static constexpr int XI = C::XH * C::OY * F;    // stage-X items per plane
  static constexpr int ZI = C::OX * C::OY;        // stage-Z items per plane
  static constexpr int YW = (YI + 31) / 32, XW = (XI + 31) / 32, ZW = ZI / 32;
  static constexpr int THREADS = 32 * (1 + YW + XW + ZW);
  static constexpr int BOX = C::WX * C::WY;       // entries of one field's input box
  static constexpr int NI = (BOX + 31) / 32;      // loader copies per lane and field
  static constexpr int NSU = STB_NSU, NSA = STB_NSA, NSC = STB_NSC;  // ring depths (planes)
  static constexpr int U_S = F * C::UB_F;          // one plane of the staged u boxes
  static constexpr int AB_S = 2 * F * C::AB_F;     // one plane of a and b
  static constexpr int CP_S = 2 * F * C::CP_F;     // one plane of c and pre
  static constexpr int NBAR = 2 * (NSU + NSA + NSC);
  static constexpr size_t smem_bytes() {
    return sizeof(double) * (static_cast<size_t>(NSU) * U_S + NSA * AB_S + NSC * CP_S) + 8 * NBAR;
  }
};

template <int K>
using IntC = std::integral_constant<int, K>;

template <int N, int F, bool RES>
__global__ void __launch_bounds__(WsCfg<N, F>::THREADS, 1)
    st_brick_ws_kernel(const __grid_constant__ DevLevel L, const double* __restrict__ u,
                       const double* __restrict__ fvec, double* __restrict__ y, int ntx, int zc) {
  using C = Cfg<N, F>;
  using W = WsCfg<N, F>;
  constexpr int P = C::P, OX = C::OX, OY = C::OY, WX = C::WX;
  constexpr int NSU = W::NSU, NSA = W::NSA, NSC = W::NSC;
  extern __shared__ __align__(16) double smem[];
  double* Ub = smem;
  double* ABr = Ub + NSU * W::U_S;
  double* CPr = ABr + NSA * W::AB_S;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(CPr + NSC * W::CP_S);
  unsigned long long* u_full = bars;
  unsigned long long* u_empty = u_full + NSU;
  unsigned long long* ab_full = u_empty + NSU;
  unsigned long long* ab_empty = ab_full + NSA;
  unsigned long long* cp_full = ab_empty + NSA;
  unsigned long long* cp_empty = cp_full + NSC;

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    for (int i = 0; i < NSU; ++i) {
      mbar_init(u_full + i, 32);
      mbar_init(u_empty + i, W::YW);
    }
    for (int i = 0; i < NSA; ++i) {
      mbar_init(ab_full + i, W::YW);
      mbar_init(ab_empty + i, W::XW);
    }
    for (int i = 0; i < NSC; ++i) {
      mbar_init(cp_full + i, W::XW);
      mbar_init(cp_empty + i, W::ZW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  const long long X0 = static_cast<long long>(tx) * OX, Y0 = static_cast<long long>(ty) * OY;
  const long long dx = L.dofs[0], dy = L.dofs[1], dz = L.dofs[2];
  const long long dxy = dx * dy, ns = L.n_space;
  const int ncz = static_cast<int>(L.cells[2]);
  const int L0 = static_cast<int>(blockIdx.y) * zc;
  const int L1 = L0 + zc < ncz ? L0 + zc : ncz;
  const int Ls = L0 > 0 ? L0 - 1 : 0;  // first layer processed (halo)
  const int z_first = Ls * P, z_last = L1 * P;
  const bool lo_dir = (L.zbc & 1) != 0, hi_dir = (L.zbc & 2) != 0;

  if (warp == 0) {
    // ================= loader =================
    // entry idx = lane + 32 i of the box is (row idx / WX, column idx % WX);
    // its shared-memory offset inside the field's box is idx itself
    int off[W::NI];
    unsigned vmask = 0;  // entries inside the lattice, off its x / y Dirichlet faces
#pragma unroll
    for (int i = 0; i < W::NI; ++i) {
      const int idx = lane + 32 * i;
      const int r = idx / WX, x = idx - r * WX;
      const long long gxx = X0 - P + x, gyy = Y0 - P + r;
      const bool ok = idx < W::BOX && gxx > 0 && gxx < dx - 1 && gyy > 0 && gyy < dy - 1;
      off[i] = ok ? static_cast<int>(gyy * dx + gxx) : 0;
      if (ok) vmask |= 1u << i;
    }
    const bool last_in = lane + 32 * (W::NI - 1) < W::BOX;
    const unsigned want = last_in ? (1u << W::NI) - 1u : (1u << (W::NI - 1)) - 1u;
    const bool interior = __all_sync(0xffffffffu, vmask == want);
    const unsigned dst0 = smem_u32(Ub) + 8u * lane;
    int su = 0;
    unsigned pu = 1;  // fresh barrier: the first pass over the ring does not wait
    for (int z = z_first; z <= z_last; ++z) {
      mbar_wait(u_empty + su, pu);
      const bool zd = (z == 0 && lo_dir) || (z == dz - 1 && hi_dir);
      const double* pz = u + z * dxy;
      const unsigned d = dst0 + 8u * (su * W::U_S);
      if (interior && !zd) {
#pragma unroll
        for (int f = 0; f < F; ++f)
#pragma unroll
          for (int i = 0; i < W::NI; ++i)
            if (i + 1 < W::NI || last_in) cp_async8_s(d + 8u * (f * C::UB_F + 32 * i), pz + f * ns + off[i], 8);
      } else {
#pragma unroll
        for (int f = 0; f < F; ++f)
#pragma unroll
          for (int i = 0; i < W::NI; ++i)
            if (i + 1 < W::NI || last_in) {
              const bool ok = !zd && ((vmask >> i) & 1u);
              cp_async8_s(d + 8u * (f * C::UB_F + 32 * i), ok ? pz + f * ns + off[i] : u, ok ? 8 : 0);
            }
      }
      cp_async_arrive(u_full + su);
      if (++su == NSU) {
        su = 0;
        pu ^= 1;
      }
    }
    cp_async_wait_all();
  } else if (warp < 1 + W::YW) {
    // ================= stage Y =================
    const int i = t - 32;
    const bool act = i < W::YI;
    const int yx = i % WX, yf = act ? i / WX : 0;
    const int uoff = yf * C::UB_F + yx, aoff = yf * C::AB_F + yx;
    int su = 0, sa = 0;
    unsigned pu = 0, pa = 1;
    for (int z = z_first; z <= z_last; ++z) {
      mbar_wait(u_full + su, pu);
      mbar_wait(ab_empty + sa, pa);
      if (act) {
        const double* ycolbuf = Ub + su * W::U_S + uoff;
        // (a, b) of one node are one 16-byte entry: one store here, one load in stage X
        double2* oab = reinterpret_cast<double2*>(ABr + sa * W::AB_S) + aoff;
        // element 0 is the halo cell: it reaches owned row 0 only
        double v[N];
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = ycolbuf[k * WX];
        double ca, cb;
        {
          const Split<N> s = split_at<N>(v);
          ca = elem_last<N>(L.MrE, L.MrO, s);
          cb = elem_last<N>(L.KrE, L.KrO, s);
        }
#pragma unroll
        for (int e = 1; e <= OY / P; ++e) {
          v[0] = v[P];
#pragma unroll
          for (int k = 1; k < N; ++k) v[k] = ycolbuf[(e * P + k) * WX];
          const Split<N> s = split_at<N>(v);
          double ea[N], eb[N];
          elem<N>(L.MrE, L.MrO, s, ea);
          elem<N>(L.KrE, L.KrO, s, eb);
          const int r0 = (e - 1) * P;
          oab[r0 * C::XP] = make_double2(ca + ea[0], cb + eb[0]);
#pragma unroll
          for (int j = 1; j < P; ++j) oab[(r0 + j) * C::XP] = make_double2(ea[j], eb[j]);
          ca = ea[P];
          cb = eb[P];
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(u_empty + su);
        mbar_arrive(ab_full + sa);
      }
      if (++su == NSU) {
        su = 0;
        pu ^= 1;
      }
      if (++sa == NSA) {
        sa = 0;
        pa ^= 1;
      }
    }
  } else if (warp < 1 + W::YW + W::XW) {
    // ================= stage X =================
    constexpr int HX = OX / C::XH;  // owned columns per half
    const int i = t - 32 * (1 + W::YW);
    const bool act = i < W::XI;
    // rows fastest: 8 consecutive lanes touch 16-byte entries a row pitch
    // apart (odd pitches: distinct banks)
    const int r = i % OY, hf = i / OY;
    const int h = hf % C::XH, f = act ? hf / C::XH : 0;
    const double sx = L.hinv2[0], sy = L.hinv2[1];
    const int ioff = f * C::AB_F + r * C::XP + h * HX;
    const int ooff = f * C::CP_F + r * C::CPP + h * HX;
    int sa = 0, sc = 0;
    unsigned pa = 0, pc = 1;
    for (int z = z_first; z <= z_last; ++z) {
      mbar_wait(ab_full + sa, pa);
      mbar_wait(cp_empty + sc, pc);
      if (act) {
        const double2* iab = reinterpret_cast<const double2*>(ABr + sa * W::AB_S) + ioff;
        double2* ocp = reinterpret_cast<double2*>(CPr + sc * W::CP_S) + ooff;
        double va[N], vb[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double2 ab = iab[k];
          va[k] = ab.x;
          vb[k] = ab.y;
        }
        double cc, cp;
        {
          const Split<N> sa_ = split_at<N>(va), sb_ = split_at<N>(vb);
          cc = elem_last<N>(L.MrE, L.MrO, sa_);
          cp = fma(sx, elem_last<N>(L.KrE, L.KrO, sa_), sy * elem_last<N>(L.MrE, L.MrO, sb_));
        }
#pragma unroll
        for (int e = 1; e <= HX / P; ++e) {
          va[0] = va[P];
          vb[0] = vb[P];
#pragma unroll
          for (int k = 1; k < N; ++k) {
            const double2 ab = iab[e * P + k];
            va[k] = ab.x;
            vb[k] = ab.y;
          }
          const Split<N> sa_ = split_at<N>(va), sb_ = split_at<N>(vb);
          double ec[N], ek[N], em[N];
          elem<N>(L.MrE, L.MrO, sa_, ec);
          elem<N>(L.KrE, L.KrO, sa_, ek);
          elem<N>(L.MrE, L.MrO, sb_, em);
          const int r0 = (e - 1) * P;
          ocp[r0] = make_double2(cc + ec[0], cp + fma(sx, ek[0], sy * em[0]));
#pragma unroll
          for (int j = 1; j < P; ++j) ocp[r0 + j] = make_double2(ec[j], fma(sx, ek[j], sy * em[j]));
          cc = ec[P];
          cp = fma(sx, ek[P], sy * em[P]);
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(ab_empty + sa);
        mbar_arrive(cp_full + sc);
      }
      if (++sa == NSA) {
        sa = 0;
        pa ^= 1;
      }
      if (++sc == NSC) {
        sc = 0;
        pc ^= 1;
      }
    }
  } else {
    // ================= stage Z =================
    const int pt = t - 32 * (1 + W::YW + W::XW);
    const int zx = pt % OX, zy = pt / OX;
    const long long gx = X0 + zx, gy = Y0 + zy;
    const double V = L.h[0] * L.h[1] * L.h[2];
    const double Vsz = V * L.hinv2[2];
    auto rho_of = [&](int e) -> double {
      if (!L.rho0) return 1.0;
      const long long az = (e + L.cz0) >> L.rho_shift;
      return __ldg(L.rho0 + az * L.cells0[1] * L.cells0[0]);
    };
    // the point is written by this CTA if it lies on the lattice; x / y end
    // planes (always Dirichlet) are written by the tile containing them, or by
    // the last tile's border threads when the tile ends exactly on them
    const bool on_lat = gx < dx && gy < dy;
    const long long pbase = gy * dx + gx;
    const bool xend_extra = (zx == OX - 1) && (X0 + OX == dx - 1);
    const bool yend_extra = (zy == OY - 1) && (Y0 + OY == dy - 1);
    const bool xy_dir = gx == 0 || gy == 0 || gx == dx - 1 || gy == dy - 1;
    // CTA-uniform: every point of the tile is an interior lattice node in x and y
    const bool tile_int = tx > 0 && ty > 0 && X0 + OX < dx - 1 && Y0 + OY < dy - 1;

    double win[F][N];  // z window of the open layer
#pragma unroll
    for (int i = 0; i < F; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) win[i][j] = 0.0;

    // Dirichlet row: u (residual f - u); on a slab's low interface plane the
    // row belongs to the slab below, this copy holds 0 (the interface sum adds it)
    auto store_dir = [&](long long x, long long yy, long long zz) {
      const bool other = zz == 0 && !lo_dir;
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const long long idx = f * ns + zz * dxy + yy * dx + x;
        if (other) {
          y[idx] = 0.0;
        } else {
          const double uv = __ldg(u + idx);
          y[idx] = RES ? __ldg(fvec + idx) - uv : uv;
        }
      }
    };
    // residual: pull the f entries of layer e's owned planes towards L2 when
    // the layer opens; they are read when it closes, p planes later
    auto prefetch_layer = [&](int e) {
      if (!RES || !on_lat || e < L0) return;
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const double* base = fvec + static_cast<long long>(e * P + q) * dxy + pbase;
#pragma unroll
        for (int f = 0; f < F; ++f) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + f * ns));
      }
    };
    auto combine = [&](int jw, double (&out)[F]) {
      if (L.g_ok) {
#pragma unroll
        for (int i = 0; i < F; ++i) {
          double v = 0.0;
#pragma unroll
          for (int h = 0; h < F; ++h) v = fma(L.CA[i * F + h], win[h][jw], v);
          out[i] = v;
        }
      } else {
#pragma unroll
        for (int i = 0; i < F; ++i) out[i] = win[i][jw];
      }
    };
    auto store_plane = [&](long long zz, int jw) {
      const bool zedge = zz == 0 || zz == dz - 1;
      if (tile_int && !zedge) {
        // interior tile, interior plane: plain rows of the operator
        const long long base = zz * dxy + pbase;
        double out[F];
        combine(jw, out);
#pragma unroll
        for (int i = 0; i < F; ++i) {
          const long long idx = base + i * ns;
          y[idx] = RES ? __ldg(fvec + idx) - out[i] : out[i];
        }
        return;
      }
      const bool zdir = (zz == 0 && lo_dir) || (zz == dz - 1 && hi_dir);
      if (on_lat) {
        if (zdir || xy_dir) {
          store_dir(gx, gy, zz);
        } else {
          const bool no_f = (zz == 0 && !lo_dir);  // low interface plane: f counted by the slab below
          const long long base = zz * dxy + pbase;
          double out[F];
          combine(jw, out);
#pragma unroll
          for (int i = 0; i < F; ++i) {
            const long long idx = base + i * ns;
            if (RES)
              y[idx] = no_f ? -out[i] : __ldg(fvec + idx) - out[i];
            else
              y[idx] = out[i];
          }
        }
      }
      if (xend_extra && gy < dy) store_dir(dx - 1, gy, zz);
      if (yend_extra && gx < dx) store_dir(gx, dy - 1, zz);
      if (xend_extra && yend_extra) store_dir(dx - 1, dy - 1, zz);
    };

    const int coff = zy * C::CPP + zx;
    int sc = 0;
    unsigned pc = 0;
    double cmc[F], cap[F], cac[F];
    // next plane of the CP ring -> the three coupled inputs of the z products
    auto next_plane = [&]() {
      mbar_wait(cp_full + sc, pc);
      double vc[F];
      {
        const double2* icp = reinterpret_cast<const double2*>(CPr + sc * W::CP_S) + coff;
#pragma unroll
        for (int gg = 0; gg < F; ++gg) {
          const double2 cpv = icp[gg * C::CP_F];
          vc[gg] = cpv.x;
          cap[gg] = cpv.y;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(cp_empty + sc);
      if (++sc == NSC) {
        sc = 0;
        pc ^= 1;
      }
      if (L.g_ok) {
        // (CA (x) I)(G (x) M + I (x) A): G c on the point, CA at the store
#pragma unroll
        for (int i = 0; i < F; ++i) {
          double s = 0.0;
#pragma unroll
          for (int gg = 0; gg < F; ++gg) s = fma(L.G[i * F + gg], vc[gg], s);
          cmc[i] = s;
          cac[i] = vc[i];
        }
      } else {
        double vp[F];
#pragma unroll
        for (int i = 0; i < F; ++i) vp[i] = cap[i];
#pragma unroll
        for (int i = 0; i < F; ++i) {
          double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
          for (int gg = 0; gg < F; ++gg) {
            const double cm = L.CM[i * F + gg], ca = L.CA[i * F + gg];
            a = fma(cm, vc[gg], a);
            b = fma(ca, vp[gg], b);
            c = fma(ca, vc[gg], c);
          }
          cmc[i] = a;
          cap[i] = b;
          cac[i] = c;
        }
      }
    };
    // contribution of the current plane to a layer with coefficient rho at
    // the layer's local index JL (compile time: the table entries are immediates)
    auto add_layer = [&](auto jc, double rho) {
      constexpr int JL = decltype(jc)::value;
      const double rv = rho * Vsz;
#pragma unroll
      for (int i = 0; i < F; ++i) {
        const double zm = V * fma(rho, cap[i], cmc[i]);
        const double zk = rv * cac[i];
#pragma unroll
        for (int q = 0; q < N; ++q) win[i][q] = fma(L.Mr[q][JL], zm, fma(L.Kr[q][JL], zk, win[i][q]));
      }
    };
    // vertex plane above layer e: the layer's p lower planes are final
    auto close_layer = [&](int e, double rho) {
      add_layer(IntC<P>{}, rho);
      if (e >= L0) {
#pragma unroll
        for (int q = 0; q < P; ++q) store_plane(static_cast<long long>(e) * P + q, q);
      }
#pragma unroll
      for (int i = 0; i < F; ++i) {
        win[i][0] = win[i][P];
#pragma unroll
        for (int q = 1; q < N; ++q) win[i][q] = 0.0;
      }
    };

    prefetch_layer(Ls);
    double rho_prev = 1.0;
    for (int e = Ls; e < L1; ++e) {
      const double rho = rho_of(e);
      next_plane();
      if (e > Ls) {
        close_layer(e - 1, rho_prev);
        prefetch_layer(e);
      }
      add_layer(IntC<0>{}, rho);
      if constexpr (P > 1) {
        next_plane();
        add_layer(IntC<1>{}, rho);
      }
      if constexpr (P > 2) {
        next_plane();
        add_layer(IntC<2>{}, rho);
      }
      if constexpr (P > 3) {
        next_plane();
        add_layer(IntC<3>{}, rho);
      }
      rho_prev = rho;
    }
    next_plane();
    close_layer(L1 - 1, rho_prev);
    // the slab's top plane: Dirichlet, or an interface partial sum
    if (L1 == ncz) store_plane(z_last, 0);
  }
}

template <int N, int F>
void launch_ws(const DevLevel& L, const double* u, const double* f, double* y, cudaStream_t s) {
  using C = Cfg<N, F>;
  using W = WsCfg<N, F>;
  static bool configured = false;
  if (!configured) {
    for (auto k : {st_brick_ws_kernel<N, F, false>, st_brick_ws_kernel<N, F, true>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(W::smem_bytes()));
    configured = true;
  }
  const long long ntx = std::max<long long>(1, (L.dofs[0] - 1 + C::OX - 1) / C::OX);
  const long long nty = std::max<long long>(1, (L.dofs[1] - 1 + C::OY - 1) / C::OY);
  const long long tiles = ntx * nty;
  const long long ncz = L.cells[2];
  // one CTA per SM. Measured at C5 16^3 .. 128^3 (z chunks 1 .. 12): ~24 CTAs
  // per SM over the launch, chunks of >= 12 layers (halo layer + pipeline
  // fill) unless that leaves fewer than 2 CTAs per SM, never below 2 layers
  long long nch = (148LL * 24 + tiles - 1) / tiles;
  nch = std::min(nch, std::max(ncz / 12, (148LL * 2 + tiles - 1) / tiles));
  nch = std::max<long long>(1, std::min(nch, ncz / 2));
  const long long zc = (ncz + nch - 1) / nch;
  nch = (ncz + zc - 1) / zc;
  const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(nch));
  count_launch();
  if (f)
    st_brick_ws_kernel<N, F, true><<<grid, W::THREADS, W::smem_bytes(), s>>>(L, u, f, y, static_cast<int>(ntx),
                                                                             static_cast<int>(zc));
  else
    st_brick_ws_kernel<N, F, false><<<grid, W::THREADS, W::smem_bytes(), s>>>(L, u, nullptr, y, static_cast<int>(ntx),
                                                                              static_cast<int>(zc));
}

#ifndef STB_WS
#define STB_WS 1
#endif

template <int N, int F>
void launch(const DevLevel& L, const double* u, const double* f, double* y, cudaStream_t s) {
  using C = Cfg<N, F>;
  if constexpr (STB_WS && C::FG == 1) {
    launch_ws<N, F>(L, u, f, y, s);
    return;
  }

  using C = Cfg<N, F>;
  static bool configured = false;
  if (!configured) {
    for (auto k : {st_brick_kernel<N, F, false>, st_brick_kernel<N, F, true>}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::smem_bytes()));
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    configured = true;
  }
  const long long ntx = std::max<long long>(1, (L.dofs[0] - 1 + C::OX - 1) / C::OX);
  const long long nty = std::max<long long>(1, (L.dofs[1] - 1 + C::OY - 1) / C::OY);
  const long long tiles = ntx * nty;
  const long long ncz = L.cells[2];
  // the rule of launch_ws for 2 CTAs per SM (C4: 3 / 6 / 12 chunks measured 7.04 / 6.79 / 6.94 ms)
  long long nch = (148LL * 2 * 20 + tiles - 1) / tiles;
  nch = std::min(nch, std::max(ncz / 12, (148LL * 2 * 2 + tiles - 1) / tiles));
  nch = std::max<long long>(1, std::min(nch, ncz / 2));
  const long long zc = (ncz + nch - 1) / nch;
  nch = (ncz + zc - 1) / zc;
  const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(nch));
  count_launch();
  if (f)
    st_brick_kernel<N, F, true><<<grid, kThreads, C::smem_bytes(), s>>>(L, u, f, y, static_cast<int>(ntx),
                                                                        static_cast<int>(zc));
  else
    st_brick_kernel<N, F, false><<<grid, kThreads, C::smem_bytes(), s>>>(L, u, nullptr, y, static_cast<int>(ntx),
                                                                         static_cast<int>(zc));
}

template <int N>
void launch_n(const DevLevel& L, const double* u, const double* f, double* y, cudaStream_t s) {
  switch (L.F) {
    case 1: launch<N, 1>(L, u, f, y, s); break;
    case 2: launch<N, 2>(L, u, f, y, s); break;
    case 3: launch<N, 3>(L, u, f, y, s); break;
    case 4: launch<N, 4>(L, u, f, y, s); break;
    case 5: launch<N, 5>(L, u, f, y, s); break;
    case 6: launch<N, 6>(L, u, f, y, s); break;
    case 7: launch<N, 7>(L, u, f, y, s); break;
    case 8: launch<N, 8>(L, u, f, y, s); break;
    default: throw std::invalid_argument("st_brick: S * n_t must be in [1, 8]");
  }
}

}  // namespace stb

bool st_brick_supported(const DevLevel& L) {
  return L.dim == 3 && L.verts == nullptr && L.rho_zonly && (L.n == 2 || L.n == 3 || L.n == 5) && L.F >= 1 &&
         L.F <= kMaxF;
}

void st_brick(const DevLevel& L, const double* f, const double* u, double* y, cudaStream_t s) {
  switch (L.n) {
    case 2: stb::launch_n<2>(L, u, f, y, s); break;
    case 3: stb::launch_n<3>(L, u, f, y, s); break;
    case 5: stb::launch_n<5>(L, u, f, y, s); break;
    default: throw std::invalid_argument("st_brick: p must be 1, 2 or 4");
  }
}

}  // namespace stmgb
