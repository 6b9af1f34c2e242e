// Explicit instantiations of the k_agg_tiles family for NI = 0 int64 SUM and NF = 0 f64 SUM/AVG
// columns (one unit per (NI, NF) so the instances compile in parallel; build.py).
#include "agg_tiles.cuh"
#include "agg_tm.cuh"

namespace pac {
template cudaError_t launch_smem<0, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<0, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<0, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<0, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<0, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<0, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<0, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<0, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
}  // namespace pac
