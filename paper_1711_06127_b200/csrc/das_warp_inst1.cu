// das_warp_inst1.cu -- explicit instantiations of the warp-split DAS kernel, mode 1.
#include "das_warp_kernel.cuh"

namespace supra {
template cudaError_t launch_w<32, false, 1>(const CUtensorMap&, const DasArgs&, cudaStream_t);
template cudaError_t launch_w<64, false, 1>(const CUtensorMap&, const DasArgs&, cudaStream_t);
template cudaError_t launch_w<32, true, 1>(const CUtensorMap&, const DasArgs&, cudaStream_t);
template cudaError_t launch_w<64, true, 1>(const CUtensorMap&, const DasArgs&, cudaStream_t);
}  // namespace supra
