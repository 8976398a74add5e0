// 2D instantiations of the fused space-time operator (st_operator.cuh)
#include <stdexcept>

#include "st_operator.cuh"

namespace stmgb {
void st_apply_2d(const DevLevel& L, const double* u, double* y, double sign, cudaStream_t s) {
  switch (L.n) {
    case 2: stk::launch_f<2, 2>(L, u, y, sign, s); break;
    case 3: stk::launch_f<2, 3>(L, u, y, sign, s); break;
    case 4: stk::launch_f<2, 4>(L, u, y, sign, s); break;
    case 5: stk::launch_f<2, 5>(L, u, y, sign, s); break;
    default: throw std::invalid_argument("st_apply: p must be in [1, 4]");
  }
}
}  // namespace stmgb
