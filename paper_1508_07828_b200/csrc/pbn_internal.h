// pbn_internal.h -- internal layout shared by the host API (pbn_api.cpp) and
// the kernels (pbn_traj.cu, pbn_recount.cu).  Not part of the C ABI.
//
// Device image of a PBN (built once by pbn_load).  One
// contiguous blob, 16-byte aligned sections, staged whole into each CTA's
// shared memory with one bulk async copy when it fits:
//
//   nrec [n]    uint4 per node i:
//                 .x .y .z  selection thresholds E_1..E_3 of node i, where
//                           function j (0-based) is chosen iff
//                           j = #{k : u > E_k} (E_k = D_k - 1, reading Q3);
//                           unused entries are 0xFFFFFFFF
//                 .w        fn_base (bits 0-19) | theta_max of the node
//                           (bits 20-24) | ell-1 (bits 25-31)
//   fdesc[nf]   uint2 per function f:
//                 .x        truth table word 0 (theta <= 5: the whole table)
//                 .y        theta (bits 0-4) | aux offset in u32 (bits 5-31)
//   aux  []     per function: ceil(theta/2) u32 holding theta u16 parent
//               byte offsets (node * 4) in REVERSED order -- half-word m is
//               parents[theta-1-m], i.e. the parent whose bit is index bit m
//               (parents[0] is the MSB, reading Q5); then, for theta >= 6,
//               the 2^theta/32 table words.
//   xthr [nf]   only when some ell(i) > 4: xthr[fn_base + k - 1] = E_k
//
// The thresholds are the product's own computation of reading Q3
// (pbn_api.cpp build_image); nothing here is shared with oracle/.
#pragma once
#include <cstdint>

namespace pbn {

constexpr int kMaxPred = 16;
constexpr int kMaxWarpsPerCta = 32;

struct ImageLayout {
    uint32_t off_nrec = 0, off_fdesc = 0, off_aux = 0, off_xthr = 0;
    uint32_t bytes = 0;
    int32_t n = 0, nf = 0;
    int32_t aux_words = 0;
    int32_t has_xthr = 0;
    int32_t max_theta = 0, max_ell = 0;
};

struct TrajParams {
    const uint8_t* image;      // device image (global)
    ImageLayout L;
    uint32_t Tp;
    int32_t per_node;          // PBN_PERTURB_PER_NODE semantics
    int32_t n;
    int32_t nquads;            // ceil(n/4)
    int32_t n_pad;             // n rounded up to a multiple of 4 (u32 words per buffer)
    int32_t state_words;       // ceil(n/32): row stride of the chain-major state
    int32_t groups_per_cta;
    int32_t warps_per_group;
    int32_t group_stride;      // u32 words of shared memory per chain group
    uint32_t image_smem_bytes; // 0 when the image is read from global memory
    uint64_t seed;
    int64_t n_chains, chain_base, step0, burn_in, steps, batch;
    int32_t init, emit_bits;
    int32_t pred_k;
    uint16_t pred_node[kMaxPred];
    uint8_t pred_val[kMaxPred];
    int64_t batch_row;         // ceil(steps/batch) (0 if no batches)
    int64_t bits_row;          // row stride of bits in u32
    int64_t bits_offset;       // window element w -> row bit bits_offset + w
    // outputs
    uint32_t* state;
    uint32_t* c1;
    uint32_t* n01;
    uint32_t* n10;
    uint8_t* first_last;
    uint32_t* batch_sums;
    uint32_t* bits;
    unsigned long long* totals;
};

struct LaunchPlan {
    int groups_per_cta;
    int warps_per_group;
    int ctas;
    int threads;
    size_t smem_bytes;
    bool image_in_smem;
};

// Implemented in pbn_traj.cu.  Returns 0 on success, else a cudaError_t value;
// *usage_error set (and nonzero returned) when the sizes cannot be served.
int plan_traj_launch(const TrajParams& P, int device, int want_groups, int want_warps,
                     LaunchPlan* plan, const char** why);
int launch_traj(TrajParams P, const LaunchPlan& plan, void* stream);

struct RecountParams {
    const uint32_t* bits;
    int64_t n_chains, row_words, start, length, batch, batch_row;
    uint32_t* c1;
    uint32_t* n01;
    uint32_t* n10;
    uint8_t* first_last;
    uint32_t* batch_sums;
    unsigned long long* totals;
};
int launch_recount(const RecountParams& R, void* stream);

}  // namespace pbn
