// pbn_bitslice.cu -- K1b dispatch: the kernel of (semantics, largest ell,
// image placement, largest task class); kernels in pbn_bitslice_m{0,1,2}.cu.
#include "pbn_internal.h"

namespace pbn {

const void* pick_bitslice_kernel_mode0(int L, bool smem_image, int cmax);
const void* pick_bitslice_kernel_mode1(int L, bool smem_image, int cmax);
const void* pick_bitslice_kernel_mode2(int L, bool smem_image, int cmax);

const void* pick_bitslice_kernel(int mode, int L, bool smem_image, int cmax)
{
    return mode == 1   ? pick_bitslice_kernel_mode1(L, smem_image, cmax)
           : mode == 2 ? pick_bitslice_kernel_mode2(L, smem_image, cmax)
                       : pick_bitslice_kernel_mode0(L, smem_image, cmax);
}

}  // namespace pbn
