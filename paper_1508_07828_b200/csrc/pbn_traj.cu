// pbn_traj.cu -- K1: launch planning and launch of the fused PBN trajectory
// kernel (the kernel template: pbn_traj_kernel.cuh, instantiated per mode in
// pbn_traj_m{0,1,2}.cu).
//
// Hot path of PAPER.md §2.2 with the per-chain statistics of
// Algorithms 3-5 fused:
//
//   layout     one warp lane = one chain; 32 chains form a "group" whose state
//              is BIT-SLICED in shared memory: word[i] holds node i of the
//              group's 32 chains (bit l = lane l), double-buffered (A7).  A
//              group's nodes are split over W warps (4-node quads, the Philox
//              granularity); a named barrier per group closes each step.
//   per node   the warp walks its nodes in lock-step, so network metadata reads
//              are broadcasts (<= 4 distinct addresses); per lane: one 32-bit
//              Philox word u (A3), perturbation u < T_p (A4), function
//              j = #{k : u > E_k} (A5), then the node's theta_max parents are
//              gathered MSB-first -- every function of a node is padded to the
//              node's theta_max (pbn_internal.h), so the gather count is
//              warp-uniform and branch-free: per parent one LDS of the parent
//              word, a rotate that brings bit `lane` to bit 31 and a funnel
//              shift that appends it to the index (A6); the padded 64-bit table
//              gives the bit and one __ballot_sync commits the 32 chains' new
//              bits as one word (A7).
//   VECTOR each step also stores gamma words; after the
//              step barrier every warp patches its own nodes for the chains
//              with any gamma: new = (f & ~M) | ((old ^ gamma) & M).
//   stats      warp 0 of each group evaluates the property on the new words
//              (A8: AND over (node, value) pairs, bit-sliced) and keeps per
//              lane (= chain) counters in registers: c1, n01, n10, first/last,
//              batch sums, packed bits (A9); the epilogue writes them and adds
//              the six u64 totals with integer atomics (A10, order-independent).
//   image      staged into shared memory once per CTA by cp.async.bulk (TMA
//              bulk copy, mbarrier completion) when it fits; otherwise read
//              through the read-only global path (ld.global.nc).
//
// Randomness: Philox4x32-10 with counter (i/4, chain, t lo, t hi) and key
// (seed lo, seed hi) -- reading Q2; the round keys are precomputed on the
// host and read from the constant bank.  Every output depends only on
// (model, seed, chain id, absolute step), never on the launch shape.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "pbn_internal.h"

namespace pbn {

const void* pick_traj_kernel_mode0(bool smem, int FT, bool slow);
const void* pick_traj_kernel_mode1(bool smem, int FT, bool slow);
const void* pick_traj_kernel_mode2(bool smem, int FT, bool slow);

namespace {

// Thread budget of the global-image kernels (see pbn_traj_kernel.cuh)
#ifndef PBN_GLOBAL_THREADS
#define PBN_GLOBAL_THREADS 896
#endif
constexpr int kGlobalImageThreads = PBN_GLOBAL_THREADS < PBN_MAX_THREADS ? PBN_GLOBAL_THREADS : PBN_MAX_THREADS;

int sm_count(int device)
{
    return cached_device_attr(cudaDevAttrMultiProcessorCount, device);
}

const void* pick_kernel(bool smem, int mode, int FT, bool slow)
{
    return mode == 1 ? pick_traj_kernel_mode1(smem, FT, slow)
                     : mode == 2 ? pick_traj_kernel_mode2(smem, FT, slow) : pick_traj_kernel_mode0(smem, FT, slow);
}

// Warps per 32-chain group.  Every warp waits at the per-step barrier for the
// one with the most quads, so the count is chosen among multiples of 4 (whole
// warps per SM sub-partition) in [20, 32] to minimise that imbalance, the
// smallest on ties (measured on C4, 500 quads: 20 warps x 25 quads
// 5.28e11 > 24: 5.26 > 28: 5.25 > 32 (15.6 quads): 5.19e11 node-updates/s).
int default_warps(int nquads)
{
    if (nquads <= 20) return std::max(1, nquads);
    int best = 20;
    double best_imb = 1e30;
    for (int W = 20; W <= std::min(kMaxWarpsPerCta, 32); W += 4) {
        if (W > nquads) break;
        const double imb = (double)((nquads + W - 1) / W) * W / nquads;
        if (imb < best_imb - 1e-12) {
            best_imb = imb;
            best = W;
        }
    }
    return best;
}

}  // namespace

int default_group_warps(int nquads) { return default_warps(nquads); }

int plan_traj_launch(const TrajParams& P, int device, int want_warps, LaunchPlan* plan, const char** why)
{
    const int smem_optin = cached_device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (smem_optin <= 0) return (int)cudaErrorInvalidDevice;
    const size_t static_smem = 64;  // mbarrier + slack
    const size_t limit = (size_t)smem_optin - static_smem;
    const size_t group_bytes = (size_t)P.group_words * 4;
    // PBN_FORCE_GLOBAL_IMAGE=1 (test knob): read the image through L1/L2 even
    // when it fits shared memory, so small models exercise that kernel too
    const char* fg = std::getenv("PBN_FORCE_GLOBAL_IMAGE");
    const bool force_global = fg && fg[0] == '1';
    const bool in_smem = !force_global && (size_t)P.L.bytes + group_bytes <= limit;
    const size_t img = in_smem ? P.L.bytes : 0;
    if (img + group_bytes > limit) {
        *why = "network too large: one 32-chain group's state does not fit in shared memory";
        return -1;
    }
    // every property needs a statistics warp: warps [0, n_props), shared with
    // the node work (dedicated statistics warps after the node warps measured
    // 0.5 % slower on C4: the layout keeps node_warps / stats_warp0 general)
    // (image through L1/L2: as many warps as possible, to cover the L2 latency)
    int Wp = want_warps > 0 ? want_warps
                           : in_smem ? default_warps(P.nquads)
                                     : std::max(1, std::min(kGlobalImageThreads / 32, P.nquads));
    Wp = std::max(Wp, P.n_props);
    if (Wp > kMaxWarpsPerCta || Wp > std::max(P.nquads, P.n_props)) {
        *why = "warps_per_group must be <= the CTA warp budget and <= max(ceil(n/4), properties)";
        return -1;
    }
    plan->node_warps = Wp;
    plan->stats_warp0 = 0;
    plan->warps_per_group = Wp;
    plan->ctas = (int)((P.n_chains + 31) / 32);
    plan->threads = Wp * 32;
    plan->smem_bytes = img + group_bytes;
    plan->image_in_smem = in_smem;
    return 0;
}

size_t traj_workspace_bytes(const TrajParams& P)
{
    const int64_t G = (P.n_chains + 31) / 32;
    const int64_t stride = P.n_pad + 8 * 32 * (int64_t)std::max(P.n_props, 1);
    const size_t ctl_bytes = ((8 + (size_t)G * 4) + 15) & ~(size_t)15;
    return ctl_bytes + (size_t)G * (size_t)stride * 4 + 16;
}

int launch_traj(TrajParams P, const LaunchPlan& plan, int device, int schedule, int64_t chunk_steps, void* workspace,
                size_t workspace_bytes, void* stream)
{
    P.warps_per_group = plan.warps_per_group;
    P.node_warps = plan.node_warps;
    P.stats_warp0 = plan.stats_warp0;
    P.image_smem_bytes = plan.image_in_smem ? P.L.bytes : 0u;
    const int mode = P.per_node ? 1 : P.geometric ? 2 : 0;
    const void* fn = pick_kernel(plan.image_in_smem, mode, P.L.fast_theta, P.L.slow_nodes > 0);
    return launch_group_units(P, fn, &P, plan, device, schedule, chunk_steps, workspace, workspace_bytes, stream);
}

int launch_group_units(TrajParams& P, const void* fn, void* kparams, const LaunchPlan& plan, int device, int schedule,
                       int64_t chunk_steps, void* workspace, size_t workspace_bytes, void* stream)
{
    cudaError_t e = ensure_func_smem(fn, plan.smem_bytes, false);
    if (e != cudaSuccess) return (int)e;
    cudaStream_t s = (cudaStream_t)stream;

    // Persistent scheduling when one-CTA-per-group would leave the last wave
    // partly empty (e.g. 512 groups on 148 SMs: 3.46 waves -> 86% busy).
    const int64_t G = (P.n_chains + 31) / 32;
    const int64_t total = P.burn_in + P.steps;
    int per_sm = 0;
    e = cached_blocks_per_sm(fn, plan.threads, plan.smem_bytes, &per_sm);
    if (e != cudaSuccess) return (int)e;
    const int64_t resident = (int64_t)sm_count(device) * std::max(per_sm, 1);
    bool persistent = false;
    if (schedule == 2) {
        persistent = total > 0;
    } else if (schedule == 0 && G > resident && total >= 128) {
        const int64_t waves = (G + resident - 1) / resident;
        persistent = (double)G / (double)(waves * resident) < 0.97;
    }
    P.persistent = persistent ? 1 : 0;
    int ctas = plan.ctas;
    uint8_t* ws = nullptr;
    bool owned = false;
    if (persistent) {
        // ~128 units per CTA keeps the last round's imbalance below 1%; a unit
        // switch costs one group state save/restore (~10 KB through L2)
        int64_t K = chunk_steps > 0 ? chunk_steps
                                    : std::max<int64_t>(32, (total * G + resident * 128 - 1) / (resident * 128));
        K = std::min(K, total);
        P.n_groups = G;
        P.chunk_steps = K;
        P.total_units = G * ((total + K - 1) / K);
        P.scratch_stride = P.n_pad + 8 * 32 * (int64_t)std::max(P.n_props, 1);
        const size_t need = traj_workspace_bytes(P);
        const size_t ctl_bytes = 8 + (size_t)G * 4;
        if (workspace) {
            // caller-owned scratch (pbn_simulate_workspace_size): no allocation
            if (workspace_bytes < need) return -2;
            ws = reinterpret_cast<uint8_t*>(workspace);
        } else {
            // no workspace passed: one stream-ordered allocation for this call
            e = cudaMallocAsync(reinterpret_cast<void**>(&ws), need, s);
            if (e != cudaSuccess) return (int)e;
            owned = true;
        }
        P.work_ctr = reinterpret_cast<unsigned long long*>(ws);
        P.done = reinterpret_cast<uint32_t*>(ws + 8);
        P.scratch = reinterpret_cast<uint32_t*>(ws + ((ctl_bytes + 15) & ~(size_t)15));
        e = cudaMemsetAsync(ws, 0, ctl_bytes, s);
        if (e != cudaSuccess) return (int)e;
        ctas = (int)std::min<int64_t>(resident, P.total_units);
    }
    void* args[] = {kparams};
    e = cudaLaunchKernel(fn, dim3(ctas), dim3(plan.threads), args, plan.smem_bytes, s);
    if (owned) {
        const cudaError_t e2 = cudaFreeAsync(ws, s);
        if (e == cudaSuccess) e = e2;
    }
    return (int)e;
}

}  // namespace pbn
