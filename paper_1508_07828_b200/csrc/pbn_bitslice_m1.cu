// pbn_bitslice_m1.cu -- K1b kernels of MODE 1 (PER_NODE); see pbn_bitslice_kernel.cuh.
#include "pbn_bitslice_kernel.cuh"

namespace pbn {

const void* pick_bitslice_kernel_mode1(int L, int img, int cmax, int threads)
{
    return pick_mode<1>(L, img, cmax, threads);
}

}  // namespace pbn
