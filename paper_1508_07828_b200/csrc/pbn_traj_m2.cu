// pbn_traj_m2.cu -- K1 kernels of MODE 2 (GEOMETRIC (VECTOR semantics)); see pbn_traj_kernel.cuh.
#include "pbn_traj_kernel.cuh"

namespace pbn {

const void* pick_traj_kernel_mode2(bool smem, int FT, bool slow)
{
    return smem ? pick_ft<true, 2>(FT, slow) : pick_ft<false, 2>(FT, slow);
}

}  // namespace pbn
