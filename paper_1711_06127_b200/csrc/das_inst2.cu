// das_inst2.cu -- explicit instantiations of the DAS batch kernel (das_kernel.cuh).
#include "das_kernel.cuh"

namespace supra {
template cudaError_t launch_k<8, 8, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
template cudaError_t launch_k<4, 8, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
template cudaError_t launch_k<2, 8, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
template cudaError_t launch_k<1, 8, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
}  // namespace supra
