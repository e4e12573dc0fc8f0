// Instantiation unit for the fused hot-path kernel, T = double (split per type to
// keep nvcc compile units small and parallel).
#include "gcpb_fused.cuh"

namespace gcpb {
template cudaError_t launch_fused<double>(const FusedArgs<double>&, int64_t, bool, cudaStream_t, int,
                                                 bool*, int);
}  // namespace gcpb
