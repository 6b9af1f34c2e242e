// Explicit instantiations of the k_agg_tiles family for NI = 2 int64 SUM columns.
#include "agg_tiles.cuh"
#include "agg_tm.cuh"

namespace pac {
template cudaError_t launch_smem<2, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 2, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 2, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 2, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_smem<2, 2, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 2, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 2, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 2, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
template cudaError_t launch_tm<2, 2, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
}  // namespace pac
