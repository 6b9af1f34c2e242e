// Explicit instantiations of the warp-specialized kernel k_agg_ws (agg_ws.cuh) for NI = 2 int64
// SUM columns (one unit per NI so the instances compile in parallel; build.py).
#include "agg_ws.cuh"

namespace pac {
template cudaError_t launch_ws<2, 0, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
template cudaError_t launch_ws<2, 1, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
template cudaError_t launch_ws<2, 2, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
}  // namespace pac
