// Explicit instantiations of the k_agg_tiles family for NI = 1 int64 SUM and NF = 1 f64 SUM/AVG
// columns (one unit per (NI, NF) so the instances compile in parallel; build.py).
#include "agg_tiles.cuh"
#include "agg_tm.cuh"

namespace pac {
template cudaError_t launch_smem<1, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<1, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<1, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<1, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<1, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<1, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<1, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<1, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
}  // namespace pac
