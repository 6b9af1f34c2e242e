// libpac: k_agg_lean instances for key spec KS = 2, mode P (private copies) (agg_lean.cuh)
#include "agg_lean.cuh"

namespace pac {
typedef void (*LeanKernel)(AggPlan, int, int);
template <int KS, int OWN> LeanKernel lean_kernel(int ni, int nf);
template <>
LeanKernel lean_kernel<2, 0>(int ni, int nf) {
  switch (ni * 3 + nf) {
    case 0: return k_agg_lean<0, 0, 2, 0>;
    case 1: return k_agg_lean<0, 1, 2, 0>;
    case 2: return k_agg_lean<0, 2, 2, 0>;
    case 3: return k_agg_lean<1, 0, 2, 0>;
    case 4: return k_agg_lean<1, 1, 2, 0>;
    case 5: return k_agg_lean<1, 2, 2, 0>;
    case 6: return k_agg_lean<2, 0, 2, 0>;
    case 7: return k_agg_lean<2, 1, 2, 0>;
    default: return nullptr;
  }
}
}  // namespace pac
