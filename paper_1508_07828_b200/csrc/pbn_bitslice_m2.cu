// pbn_bitslice_m2.cu -- K1b kernels of MODE 2 (VECTOR with the geometric-skip stream); see pbn_bitslice_kernel.cuh.
#include "pbn_bitslice_kernel.cuh"

namespace pbn {

const void* pick_bitslice_kernel_mode2(int L, int img, int cmax, int threads)
{
    return pick_mode<2>(L, img, cmax, threads);
}

}  // namespace pbn
