// pbn_traj_m1.cu -- K1 kernels of MODE 1 (PER_NODE); see pbn_traj_kernel.cuh.
#include "pbn_traj_kernel.cuh"

namespace pbn {

const void* pick_traj_kernel_mode1(bool smem, int FT, bool slow)
{
    return smem ? pick_ft<true, 1>(FT, slow) : pick_ft<false, 1>(FT, slow);
}

}  // namespace pbn
