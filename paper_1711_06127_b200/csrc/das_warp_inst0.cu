// das_warp_inst0.cu -- explicit instantiations of the warp-split DAS kernel, mode 0.
#include "das_warp_kernel.cuh"

namespace supra {
template cudaError_t launch_w<32, false, 0>(const CUtensorMap&, const DasArgs&, cudaStream_t);
template cudaError_t launch_w<64, false, 0>(const CUtensorMap&, const DasArgs&, cudaStream_t);
template cudaError_t launch_w<32, true, 0>(const CUtensorMap&, const DasArgs&, cudaStream_t);
template cudaError_t launch_w<64, true, 0>(const CUtensorMap&, const DasArgs&, cudaStream_t);
}  // namespace supra
