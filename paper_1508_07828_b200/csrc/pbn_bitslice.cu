// pbn_bitslice.cu -- K1b dispatch: the kernel of (semantics, largest ell,
// image placement, largest task class); kernels in pbn_bitslice_m{0,1,2}.cu.
#include "pbn_internal.h"

namespace pbn {

const void* pick_bitslice_kernel_mode0(int L, int img, int cmax, int threads);
const void* pick_bitslice_kernel_mode1(int L, int img, int cmax, int threads);
const void* pick_bitslice_kernel_mode2(int L, int img, int cmax, int threads);

const void* pick_bitslice_kernel(int mode, int L, int img, int cmax, int threads)
{
    return mode == 1   ? pick_bitslice_kernel_mode1(L, img, cmax, threads)
           : mode == 2 ? pick_bitslice_kernel_mode2(L, img, cmax, threads)
                       : pick_bitslice_kernel_mode0(L, img, cmax, threads);
}

}  // namespace pbn
