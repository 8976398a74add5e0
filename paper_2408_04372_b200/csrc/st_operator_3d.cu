// 3D instantiations of the fused space-time operator: the line-owner kernel
// (st_lines.cuh) wherever its registers and shared memory fit (N * F <= 16),
// its nodal-coupling, field-grouped variant (st_mix_kernel) otherwise;
// Cartesian levels take the element-matrix kernel (st_cart.cuh) unless
// STMG_VMULT=quad asks for the quadrature form.
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "st_cart.cuh"
#include "st_lines.cuh"
#include "st_operator.cuh"

namespace stmgb {
namespace {
template <int N, int F>
void launch_nf(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t s) {
  static const bool quad = [] {
    const char* e = std::getenv("STMG_VMULT");
    return e != nullptr && std::strcmp(e, "quad") == 0;
  }();
  if (!L.verts && !quad) {
    stc::launch<N, F>(L, u, y, sign, s);
    return;
  }
  if constexpr (stl::fits<N, F>())
    stl::launch<N, F>(L, u, y, sign, s);
  else
    stl::launch_mix<N, F>(L, u, y, sign, s);
}
template <int N>
void launch_n(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t s) {
  switch (L.F) {
    case 1: launch_nf<N, 1>(L, u, y, sign, s); break;
    case 2: launch_nf<N, 2>(L, u, y, sign, s); break;
    case 3: launch_nf<N, 3>(L, u, y, sign, s); break;
    case 4: launch_nf<N, 4>(L, u, y, sign, s); break;
    case 5: launch_nf<N, 5>(L, u, y, sign, s); break;
    case 6: launch_nf<N, 6>(L, u, y, sign, s); break;
    case 7: launch_nf<N, 7>(L, u, y, sign, s); break;
    case 8: launch_nf<N, 8>(L, u, y, sign, s); break;
    default: throw std::invalid_argument("st_apply: S * n_t must be in [1, 8]");
  }
}
}  // namespace

void st_apply_3d(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t s) {
  switch (L.n) {
    case 2: launch_n<2>(L, u, y, sign, s); break;
    case 3: launch_n<3>(L, u, y, sign, s); break;
    case 4: launch_n<4>(L, u, y, sign, s); break;
    case 5: launch_n<5>(L, u, y, sign, s); break;
    default: throw std::invalid_argument("st_apply: p must be in [1, 4]");
  }
}
}  // namespace stmgb
