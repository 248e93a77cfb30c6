// pbn_traj_m0.cu -- K1 kernels of MODE 0 (VECTOR); see pbn_traj_kernel.cuh.
#include "pbn_traj_kernel.cuh"

namespace pbn {

const void* pick_traj_kernel_mode0(bool smem, int FT, bool slow)
{
    return smem ? pick_ft<true, 0>(FT, slow) : pick_ft<false, 0>(FT, slow);
}

}  // namespace pbn
