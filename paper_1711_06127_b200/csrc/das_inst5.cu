// das_inst5.cu -- explicit instantiations of the DAS batch kernel (das_kernel.cuh).
#include "das_kernel.cuh"

namespace supra {
template cudaError_t launch_k<8, 4, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
template cudaError_t launch_k<4, 16, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
template cudaError_t launch_k<1, 16, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
template cudaError_t launch_k<2, 4, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
}  // namespace supra
