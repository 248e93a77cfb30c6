// pbn_internal.h -- internal layout shared by the host API (pbn_api.cpp) and
// the kernels (pbn_traj.cu, pbn_recount.cu).  Not part of the C ABI.
//
// Device image of a PBN (built once by pbn_load): one
// contiguous blob addressed by BYTE OFFSETS from its start, every record
// 16-byte aligned, staged whole into each CTA's shared memory with a bulk
// async copy when it fits (else read through the read-only global path).
//
//   nrec[i] (uint4, node i)       {E1, E2, E3, w}
//       E_k  selection thresholds of reading Q3 as E_k = D_k - 1: the
//            selected function is j = #{k : u > E_k}; unused = 0xFFFFFFFF
//       w    FAST node (ell <= 4, theta_max <= 8): offset of the node's first
//            fast descriptor (16-aligned, low 4 bits 0)
//            SLOW node (anything else): offset of its slow record | 7
//   fast descriptor (desc_bytes(FT) bytes, per function of a fast node,
//            consecutive): u32 words {t0, [t1 if FT == 6], a[0..FT-1]} for
//            FT <= 6; {a[0..7], 2^FT/32 table words} for FT = 7, 8 (the first
//            FT-5 parents select the table word, loaded after the gather)
//       every fast function is PADDED to the model-wide fast width FT (the
//       largest theta over fast nodes, 3 <= FT <= 8): its parent list is
//       extended with dummy parents that the table ignores
//       (table'[idx'] = table[idx' >> (FT - theta)]), so every lane of a warp
//       gathers exactly FT parents whatever function it chose -- straight-line
//       code with a compile-time trip count.
//       t0,t1  the padded 2^FT-entry table, entries 0-31 in t0 and 32-63 in t1,
//              each word BIT-REVERSED (entry e at bit 31 - (e & 31)) so the
//              kernel reads an entry as the sign bit of (word << (e & 31))
//       a[m]   state_off(parent m), MSB first (parents[0] first, reading Q5);
//              the pad entries read node 0
//   slow record (uint4, per slow node)  {thr, ell, gdesc, theta_max}
//       thr    offset of ell-1 u32 thresholds E_1..E_{ell-1}
//       gdesc  offset of ell generic descriptors
//   generic descriptor (uint4)          {toff, theta, poff, 0}
//       toff   offset of the ceil(2^theta/32) table words; poff: u32 list of
//              state_off(parent), parents[0] first (MSB, reading Q5)
//   PACKED form (pbn_nodepar.cu, lanes over nodes): the same records; a
//       fast descriptor holds the parents as u16 NODE IDS (the state is
//       bit-packed, node i = bit i & 31 of word i >> 5; not relocated):
//       {t0, a[0..FT-1]} (FT <= 5, 16 bytes), {t0, t1, a[0..5]} (FT = 6),
//       {a[0..7], table words} (FT = 7, 8) -- desc_bytes_packed(FT); a
//       generic descriptor's poff list holds u32 node ids
//   relocation list (u32, stored after the image in device memory, not staged)
//       byte offsets of every image-offset-valued word above (nrec.w, thr,
//       gdesc, toff, poff) and, flagged with kRelocState, of every fast
//       parent offset a[m].  After staging, each CTA adds its shared-memory
//       image base (resp. its group-state base) to those words, so the hot
//       loop uses absolute shared addresses: a parent's state word is one
//       LDS [a[m] + 16 b].  (Global-image launches add the state base per load.)
//
// Group state in shared memory (one 32-chain group per CTA): BIT-SLICED,
// word (node i, buffer b) holds node i of the 32 chains (bit l = lane l) at
//     state base + state_off(i) + 16 b,   state_off(i) = 32 (i >> 2) + 4 (i & 3)
// i.e. the two buffers are interleaved at 4-node-quad granularity: a quad's
// four words are contiguous in each buffer (one 16-byte commit) and the
// buffer is an immediate offset on every state load.
//
// The thresholds are the product's own computation of reading Q3
// (pbn_api.cpp build_image); nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/pbnsim.h"

namespace pbn {

constexpr int kMaxPred = 16;
constexpr int kMaxProps = 8;   // properties per launch (multi-property reuse)
// threads per CTA the trajectory kernel is compiled for (register budget
// 65536 / threads per thread); one 32-chain group's nodes are split over
// these warps
// 896 = 28 warps at 72 registers: C4 (20 warps x 25 quads) 5.33e11 vs 5.28e11
// node-updates/s with the 64 registers of a 1024-thread budget
#ifndef PBN_MAX_THREADS
#define PBN_MAX_THREADS 896
#endif
constexpr int kMaxWarpsPerCta = PBN_MAX_THREADS / 32;
constexpr uint32_t kSlowNode = 7;   // nrec.w low bits marking a slow node
constexpr uint32_t kRelocState = 0x80000000u;  // relocation entry: add the state base
// fast descriptor stride for fast width FT: t0 (+t1 when FT == 6) + FT offsets,
// rounded up to 16 bytes
__host__ __device__ constexpr uint32_t desc_bytes(int FT) { return FT == 3 ? 16u : FT <= 6 ? 32u : FT == 7 ? 48u : 64u; }
// the same for the PACKED image (lanes over nodes): u16 parent ids --
// {t0, a[0..FT-1]} in one 16-byte chunk for FT <= 5, {t0, t1, a[0..5]} for
// FT = 6, {a[0..7], 2^FT / 32 table words} for FT = 7, 8
__host__ __device__ constexpr uint32_t desc_bytes_packed(int FT) { return FT <= 5 ? 16u : FT <= 7 ? 32u : 48u; }
// byte offset of node i's word in buffer 0 of the group state
// (qs = bytes between quads: 32 for two interleaved buffers, 48 for three)
__host__ __device__ constexpr uint32_t state_off(uint32_t i, uint32_t qs = 32) { return qs * (i >> 2) + 4u * (i & 3u); }
constexpr int kFastMaxTheta = 8;
constexpr int kFastMinTheta = 3;
constexpr int kFastMaxEll = 4;

struct ImageLayout {
    uint32_t bytes = 0;        // image bytes (staged to shared memory)
    uint32_t reloc_off = 0;    // byte offset of the relocation list after the image
    int32_t reloc_count = 0;
    int32_t n = 0, nf = 0;
    int32_t max_theta = 0, max_ell = 0;
    int32_t slow_nodes = 0;
    int32_t fast_theta = kFastMinTheta;  // FT
};

struct TrajParams {
    const uint8_t* image;      // device image (global); relocation list at image + L.reloc_off
    ImageLayout L;
    uint32_t rk[20];           // Philox round keys (k0 + r W0, k1 + r W1), r = 0..9
    uint32_t Tp;               // perturbation threshold of the node words (0 in geometric mode)
    int32_t per_node;          // PBN_PERTURB_PER_NODE semantics
    int32_t n;
    int32_t nquads;            // ceil(n/4)
    int32_t n_pad;             // n rounded up to a multiple of 4 (u32 words per buffer)
    int32_t state_words;       // ceil(n/32): row stride of the chain-major state
    int32_t warps_per_group;   // one 32-chain group per CTA
    int32_t node_warps;        // warps [0, node_warps) own quads
    int32_t stats_warp0;       // warp stats_warp0 + p keeps property p's statistics
    int32_t group_words;       // u32 words of shared memory for the group's state
    uint32_t image_smem_bytes; // 0 when the image is read from global memory
    int64_t n_chains, chain_base, step0, burn_in, steps, batch;
    int32_t init, emit_bits;
    // properties: warp p < n_props evaluates property p and keeps its
    // per-chain statistics (outputs property-major, stride n_chains)
    int32_t n_props;
    int32_t pred_k[kMaxProps];
    uint16_t pred_node[kMaxProps][kMaxPred];
    uint8_t pred_val[kMaxProps][kMaxPred];
    // persistent scheduling (grid = resident CTAs; units = (group, step chunk))
    int32_t persistent;
    int64_t n_groups;          // ceil(n_chains / 32)
    int64_t chunk_steps;       // steps per unit
    int64_t total_units;       // n_groups * ceil(total steps / chunk_steps)
    unsigned long long* work_ctr;  // unit queue head (zeroed per launch)
    uint32_t* done;            // [n_groups] chunks completed per group (zeroed per launch)
    uint32_t* scratch;         // [n_groups x scratch_stride] suspended group state
    int64_t scratch_stride;    // n_pad + 8 * 32 * n_props words
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
    unsigned long long* totals;  // [6 x n_props]
    // geometric-skip stream (PBN_PERTURB_GEOMETRIC, reading Q18); kept at the
    // end of the struct: inserting them earlier changed the global-image K1's
    // register allocation (more spills, C5 -4 %)
    int32_t geometric;         // gamma(t) from the skip stream
    float geo_inv_lnq;         // 1 / ln(1 - p): start of the skip search (the table decides)
    uint32_t geo_off;          // byte offset of the table Cg[0..n-1] (u32) in the image
};

// Cluster launch (pbn_cluster.cu): one 32-chain group per cluster of K CTAs,
// CTA rank r owns quads [q_lo[r], q_lo[r+1]) and stages sub-image r.
constexpr int kMaxCluster = 16;
struct ClusterParams {
    TrajParams T;               // T.image = base of the K concatenated sub-images
    int32_t K;
    uint32_t img_off[kMaxCluster];    // byte offset of sub-image r from T.image
    uint32_t img_bytes[kMaxCluster];  // staged bytes of sub-image r
    uint32_t reloc_off[kMaxCluster];  // relocation list of r, from its sub-image start
    int32_t reloc_count[kMaxCluster];
    int32_t q_lo[kMaxCluster + 1];
};
size_t cluster_smem_bytes(const TrajParams& P, uint32_t max_sub_image);
int launch_traj_cluster(const ClusterParams& C, int warps, size_t smem_bytes, void* stream);
int max_active_clusters(const ClusterParams& C, int warps, size_t smem_bytes, int* out);

// Lanes-over-nodes launch (pbn_nodepar.cu): G chains per cluster of K CTAs,
// CTA rank r owns the packed state words [w_lo[r], w_lo[r+1]) (nodes
// 32 w_lo[r] ..) and stages sub-image r, built in the packed form.
struct NodeParParams {
    TrajParams T;               // T.image = base of the K concatenated packed sub-images
    int32_t K;
    int32_t G;                  // chains per cluster (1..32; cluster c runs chains c G ..)
    int32_t n_words;            // ceil(n/32)
    uint32_t img_off[kMaxCluster];
    uint32_t img_bytes[kMaxCluster];
    uint32_t reloc_off[kMaxCluster];
    int32_t reloc_count[kMaxCluster];
    int32_t w_lo[kMaxCluster + 1];
    const uint32_t* geo_table;  // geometric mode: Cg[0..n-1] in global memory (the full image's copy)
    uint32_t geo_last;          // Cg[n-1]: gamma(t) != 0 iff the first skip word is below it
    int32_t share;              // kernel variant: Philox calls shared by shuffles (>= 2 items per warp)
};
size_t nodepar_smem_bytes(int n_words, int G, uint32_t max_sub_image);
int launch_traj_nodepar(const NodeParParams& C, int threads, size_t smem_bytes, void* stream);
int max_active_nodepar_clusters(const NodeParParams& C, int threads, size_t smem_bytes, int* out);

// Bit-sliced evaluation launch (pbn_bitslice.cu, K1b): one 32-chain group
// per CTA with K1's bit-sliced state words (THREE interleaved buffers, quads
// 48 bytes apart: state_off(i, 48) + 16 b), the node step split in two phases:
//   A  lane = chain: Philox words, and per node the bits of the selected
//      function's index j = #{m : u > E_m} as ballots -- b_0 (bit 0: the
//      parity of the compares) and, for L >= 3, b_1 (bit 1: [u > E_2]) --
//      and gamma = ballot(u < T_p) for the ~1 % of quads where some chain drew
//      one; stored per quad as PV = NP + 1 16-byte vectors (b_0, [b_1], gamma
//      of its 4 nodes; NP = 0, 1, 2 for L = 1, 2, >= 3); each warp zeroes its
//      quads' words of the step's state buffer
//   B  lane = (node, function) task: the function is evaluated for all 32
//      chains at once on the parents' bit-sliced words (a multiplexer tree
//      over its truth table), masked by the chains whose index bits equal
//      its j and OR-ed into the node's new word (the chains' selections are
//      disjoint, so the OR of all tasks of a node is the new word)
// Phase A needs no state, so A of step t+1 runs in the same interval as B of
// step t (planes and any words double-buffered by step parity, state
// triple-buffered): one barrier per step.
// BITSLICE image (staged whole into shared memory when it fits with the
// group state, else read through the read-only global path; byte offsets
// from its start):
//   erec   [nquads][L-1] uint4: E_{m+1} of the quad's 4 nodes (0xFFFFFFFF
//          when m + 1 >= ell or the node is padding: the compare is false)
//   tasks  per class c = max(theta, 1) = 1..8, padded to whole rounds of 32
//          (dummy tasks: table 0, node 0, j 1), each record the 2^c-entry
//          table in T = max(1, 2^c / 32) words (entry e at bit e & 31 of word
//          e >> 5), then the u16 list [state_off(i, 48) | j, p_0 .. p_{c-1}]; stride 16
//          bytes (c <= 5), 32 (c = 6, 7), 64 (c = 8).  idx = sum_m x(p_m)
//          2^(c-1-m) (parents[0] the MSB, reading Q5); i = node, j = function
//          index within the node, p_m = state_off(parent m, 48) (theta = 0
//          pads one ignored parent)
//   rounds [n_rounds] uint2 {byte offset of the round's first task, c},
//          most expensive class first (warps take them in snake order)
constexpr int kBitsliceMaxTheta = 8;
constexpr int kBitsliceMaxEll = 4;
constexpr int kBitsliceMaxNodes = 5460;  // u16 state offsets 48 (i >> 2) + 4 (i & 3) and node ids << 2
constexpr uint32_t kBitsliceQs = 48;     // bytes between quads: three interleaved state buffers
// thread budget of the bitslice kernel (its register budget is 65536 / threads):
// 768 = 24 warps at 80 registers, no spills (896 x 72 spilled ~60 bytes: per-
// step and per-round local loads that tripled the launch's DRAM traffic,
// 253 MB vs 99.9 MB on C4; C4 6.79e11 either way, C3 5.92e11 -> 6.14e11)
#ifndef PBN_BS_THREADS
#define PBN_BS_THREADS 768
#endif
constexpr int kBitsliceMaxWarps = PBN_BS_THREADS / 32;
// the staged-image kernels' second build: 640 threads = 20 warps at ~94
// registers (C4 7.97e11 -> 8.08e11, C3 7.03e11 -> 7.28e11 node-updates/s; warp
// counts that are not a multiple of the 4 schedulers lose 8 %); the default
// when the image is staged.  The global-image kernel keeps 24 warps (C5
// 5.87e11 vs 5.77e11 at 20)
constexpr int kBitsliceSmallThreads = 640;
constexpr int kBitsliceSmallWarps = kBitsliceSmallThreads / 32;
struct BitsliceParams {
    TrajParams T;              // T.image = the bitslice image
    uint32_t erec_off;         // image offsets
    uint32_t rounds_off;
    int32_t n_rounds;
    int32_t sel_off;           // from the group state base: planes[2][nquads][PV] uint4
    int32_t sel_bytes;         // bytes of one plane buffer (16 PV nquads)
    int32_t any_off;           // from the group state base: any[2][32] words
    int32_t pq_off;            // from the group state base: [nquads + 1] uint4 per-quad Philox values (below)
    int32_t rl_off;            // from the group state base: the warps' phase-B round lists (below)
    int32_t rl_stride;         // words per warp: ceil(rounds / warps) + 9
    const uint32_t* geo_table; // geometric mode: Cg[0..n-1] (the main image's copy, global memory)
    // cluster launch (IMG = 2): K CTAs per group, rank r's sub-image at
    // T.image + c_img_off[r] (c_img_bytes[r] bytes, its erec / rounds at the
    // given offsets), owning quads [c_qlo[r], c_qlo[r+1])
    int32_t K;
    uint32_t c_img_off[kMaxCluster], c_img_bytes[kMaxCluster], c_erec_off[kMaxCluster], c_rounds_off[kMaxCluster];
    int32_t c_rounds[kMaxCluster];
    int32_t c_qlo[kMaxCluster + 1];
};
// plane vectors per quad for the model's largest ell L
inline int32_t bitslice_pv(int32_t L) { return (L >= 3 ? 2 : L == 2 ? 1 : 0) + 1; }
// group shared memory of the bitslice kernel (u32 words): 3 state buffers,
// 2 x 32 any words + 4 spare, 2 plane buffers of 4 PV words per quad, the
// per-quad Philox table (4 words per quad: the lane-uniform part of rounds
// 1-3 for the current step, rewritten by the quad's warp every step), the
// warps' phase-B round lists
// (nq_local: the quads of one CTA -- all of them, or a cluster CTA's share;
// the any region: any[2][32], the cluster ranks' any words [2][16], a dummy)
constexpr int32_t kBitsliceAnyWords = 100;
// the warps' phase-B round lists: per warp its rounds' task offsets in class
// order, one sentinel after each class (built once per CTA): at most
// rounds + 10 warps words, rounds <= 16 nq / 32 + 8 (four functions per node,
// one partial round per class)
// (a multiple of 4 words: the staged image after the group state is 16-byte aligned)
inline int32_t bitslice_round_list_words(int32_t nq_local)
{
    return (nq_local / 2 + 8 + 10 * (PBN_BS_THREADS / 32) + 3) & ~3;
}
inline int32_t bitslice_group_words(int32_t n_pad, int32_t L, int32_t nq_local = -1)
{
    if (nq_local < 0) nq_local = n_pad / 4;
    return 3 * n_pad + kBitsliceAnyWords + 2 * bitslice_pv(L) * 4 * nq_local + 4 * nq_local + 4 +
           bitslice_round_list_words(nq_local);
}
// img: 0 image through L1/L2, 1 staged, 2 staged sub-image of a cluster (K1bc)
// threads: the launch's block size (staged images: a 640-thread build for <= 20 warps)
const void* pick_bitslice_kernel(int mode, int L, int img, int cmax, int threads);
// K1's default warps per group for ceil(n/4) quads (pbn_traj.cu)
int default_group_warps(int nquads);

struct LaunchPlan {
    int warps_per_group;
    int node_warps;
    int stats_warp0;
    int ctas;
    int threads;
    size_t smem_bytes;
    bool image_in_smem;
};

// Host-side launch caches (pbn_api.cpp; thread-safe): the per-kernel
// dynamic shared-memory limit is raised once (never lowered), occupancy
// answers and device attributes are computed once per key -- pbn_simulate
// repeats none of these driver calls on its hot path.
cudaError_t ensure_func_smem(const void* fn, size_t bytes, bool nonportable_cluster);
cudaError_t cached_blocks_per_sm(const void* fn, int threads, size_t smem, int* out);
int cached_device_attr(cudaDeviceAttr attr, int device);

// Implemented in pbn_traj.cu.  Returns 0 on success, a cudaError_t value on a
// CUDA failure, or -1 (with *why set) when the sizes cannot be served.
int plan_traj_launch(const TrajParams& P, int device, int want_warps, LaunchPlan* plan, const char** why);
// schedule: 0 auto, 1 one CTA per 32-chain group, 2 persistent (chunk_steps 0 = auto).
// workspace: caller-owned scratch of >= traj_workspace_bytes(P) bytes for the
// persistent schedule, or NULL (one stream-ordered allocation per call).
// Returns 0, a cudaError_t value, or -2 when the workspace is too small.
size_t traj_workspace_bytes(const TrajParams& P);
int launch_traj(TrajParams P, const LaunchPlan& plan, int device, int schedule, int64_t chunk_steps, void* workspace,
                size_t workspace_bytes, void* stream);
// The (group, step-chunk) unit schedule of launch_traj for any kernel whose
// parameter struct embeds P (`kparams` is the kernel's single argument; the
// persistent fields are filled in P, which must live inside *kparams).
int launch_group_units(TrajParams& P, const void* fn, void* kparams, const LaunchPlan& plan, int device, int schedule,
                       int64_t chunk_steps, void* workspace, size_t workspace_bytes, void* stream);

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

// Pooled samples of omega chains for the Skart state machine (pbn_skart.cpp):
// the count of ones among the first `len` samples of every chain, and the
// chain-major sums of `per` consecutive kappa-batches of every chain from the
// sample start ([omega x per], all chains -- gathered across shards).
struct SkartSource {
    virtual ~SkartSource() = default;
    virtual pbn_status ones(int64_t len, uint64_t* S1) = 0;
    virtual pbn_status batch_sums(int64_t kappa, int64_t per, std::vector<uint32_t>& out) = 0;
};
// Algorithm 5 lines 3-21 over the first `avail` samples per chain: PBN_OK
// (res complete) or PBN_E_NOT_CONVERGED with res->need_per_chain > avail
// (extend and call again; need_per_chain = 0: an iteration cap was hit).
pbn_status skart_machine(SkartSource& src, int64_t omega, int64_t avail, double h_star, double alpha_conf,
                         pbn_skart_result* res);

}  // namespace pbn
