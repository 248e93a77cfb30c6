// pbn_bitslice_m0.cu -- K1b kernels of MODE 0 (VECTOR); see pbn_bitslice_kernel.cuh.
#include "pbn_bitslice_kernel.cuh"

namespace pbn {

const void* pick_bitslice_kernel_mode0(int L, int img, int cmax, int threads)
{
    return pick_mode<0>(L, img, cmax, threads);
}

}  // namespace pbn
