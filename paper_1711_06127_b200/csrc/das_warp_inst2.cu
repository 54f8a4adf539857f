// das_warp_inst2.cu -- explicit instantiations of the warp-split DAS kernel, mode 2.
#include "das_warp_kernel.cuh"

namespace supra {
template cudaError_t launch_w<32, false, 2>(const CUtensorMap&, const DasArgs&, cudaStream_t);
template cudaError_t launch_w<64, false, 2>(const CUtensorMap&, const DasArgs&, cudaStream_t);
template cudaError_t launch_w<32, true, 2>(const CUtensorMap&, const DasArgs&, cudaStream_t);
template cudaError_t launch_w<64, true, 2>(const CUtensorMap&, const DasArgs&, cudaStream_t);
}  // namespace supra
