// pbn_bitslice_m0.cu -- K1b kernels of MODE 0 (VECTOR); see pbn_bitslice_kernel.cuh.
#include "pbn_bitslice_kernel.cuh"

namespace pbn {

const void* pick_bitslice_kernel_mode0(int L, bool smem_image, int cmax) { return pick_mode<0>(L, smem_image, cmax); }

}  // namespace pbn
