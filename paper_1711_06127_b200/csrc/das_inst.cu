// das_inst.cu -- explicit instantiations of the DAS batch kernel
// (das_kernel.cuh), ONE per translation unit: build.py compiles this file
// once per row of kDasInst with -DDAS_INST=<row>.  One kernel per unit keeps
// the front end's inlining decisions (and so register allocation) those of
// the kernel alone -- grouped, several variants spilled a few registers
// into the tap loop -- and the units compile in parallel.  The rows must
// match the extern declarations in das.cu.
#include "das_kernel.cuh"

namespace supra {
// {frames per CTA, tiles per pass, t0 != 0, mirror lines per CTA}
constexpr int kDasInst[][4] = {
    {16, 4, 0, 1},  // 0
    {4, 4, 1, 1},  // 1
    {2, 16, 0, 1},  // 2
    {1, 4, 1, 1},  // 3
    {16, 4, 1, 1},  // 4
    {4, 4, 0, 1},  // 5
    {2, 16, 1, 1},  // 6
    {1, 4, 0, 1},  // 7
    {8, 8, 0, 1},  // 8
    {4, 8, 1, 1},  // 9
    {2, 8, 0, 1},  // 10
    {1, 8, 1, 1},  // 11
    {8, 8, 1, 1},  // 12
    {4, 8, 0, 1},  // 13
    {2, 8, 1, 1},  // 14
    {1, 8, 0, 1},  // 15
    {8, 4, 0, 1},  // 16
    {4, 16, 1, 1},  // 17
    {1, 16, 0, 1},  // 18
    {2, 4, 1, 1},  // 19
    {8, 4, 1, 1},  // 20
    {4, 16, 0, 1},  // 21
    {1, 16, 1, 1},  // 22
    {2, 4, 0, 1},  // 23
    {1, 8, 0, 2},  // 24
    {1, 16, 0, 2},  // 25
    {2, 8, 0, 2},  // 26
    {2, 16, 0, 2},  // 27
    {8, 4, 0, 2},  // 28
    {1, 8, 0, 4},  // 29
    {1, 16, 0, 4},  // 30
    {2, 4, 0, 4},  // 31
    {2, 8, 0, 4},  // 32
    {4, 4, 0, 4},  // 33
    {1, 4, 0, 4},  // 34
};
#ifdef DAS_INST
template cudaError_t launch_k<kDasInst[DAS_INST][0], kDasInst[DAS_INST][1], kDasInst[DAS_INST][2] != 0,
                              kDasInst[DAS_INST][3]>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
#endif
}  // namespace supra
