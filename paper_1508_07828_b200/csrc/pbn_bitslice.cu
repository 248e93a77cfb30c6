// pbn_bitslice.cu -- K1b dispatch: the kernel of (semantics, largest ell,
// image placement, largest task class); kernels in pbn_bitslice_m{0,1,2}.cu.
#include "pbn_internal.h"

namespace pbn {

const void* pick_bitslice_kernel_mode0(int L, int img, int cmax);
const void* pick_bitslice_kernel_mode1(int L, int img, int cmax);
const void* pick_bitslice_kernel_mode2(int L, int img, int cmax);

const void* pick_bitslice_kernel(int mode, int L, int img, int cmax)
{
    return mode == 1   ? pick_bitslice_kernel_mode1(L, img, cmax)
           : mode == 2 ? pick_bitslice_kernel_mode2(L, img, cmax)
                       : pick_bitslice_kernel_mode0(L, img, cmax);
}

}  // namespace pbn
