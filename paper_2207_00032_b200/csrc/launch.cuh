// cudaLaunchKernelEx with the optional cluster shape and programmatic dependent launch.
#pragma once

#include <cuda_runtime.h>

#include "common.h"

namespace dsinf {

template <class K, class P>
void launch_pdl(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, const P& params,
                dim3 cluster = dim3(1, 1, 1)) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (cluster.x * cluster.y * cluster.z > 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = cluster.x;
    attrs[na].val.clusterDim.y = cluster.y;
    attrs[na].val.clusterDim.z = cluster.z;
    ++na;
  }
  if (pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  DSINF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, params));
}

}  // namespace dsinf
