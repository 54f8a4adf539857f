// das_inst6.cu -- explicit instantiations of the DAS batch kernel (das_kernel.cuh),
// mirror-line variants (MIR lines per CTA share one delay set).
#include "das_kernel.cuh"

namespace supra {
template cudaError_t launch_k<1, 8, false, 2>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
template cudaError_t launch_k<1, 16, false, 2>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
template cudaError_t launch_k<2, 8, false, 2>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
}  // namespace supra
