// pbn_cluster.cu -- K1c: the trajectory kernel for one 32-chain group per
// THREAD-BLOCK CLUSTER of K CTAs (K = 2..16), for networks whose image does
// not fit one CTA's shared memory (C5: 5000 nodes) and for the few-chain
// regime (1..1024 chains: too few groups to fill 148 SMs).
//
// Same method and same per-node step as K1 (pbn_traj.cu, pbn_node.cuh):
// PAPER.md §2.2 with the fused statistics of Alg 3-5 (SURVEY
// §8(a) A1-A10).  What changes is the split of the work:
//   nodes      CTA rank r of the cluster owns quads [q_lo[r], q_lo[r+1]) and
//              stages only ITS sub-image (records and descriptors of its
//              nodes, pbn_api.cpp build_image(node range, qs = 48)).
//   state      every CTA keeps the WHOLE bit-sliced state of the group,
//              triple-buffered (word (i, b) at 48 (i/4) + 4 (i%4) + 16 b):
//              each new quad word is stored locally and into every peer CTA's
//              copy through distributed shared memory (st.shared::cluster),
//              then one cluster barrier per step (release/acquire) publishes
//              the step.
//   VECTOR     each CTA's any-gamma words and its (rare) nonzero gamma words
//              are also pushed to every peer, so after the barrier every CTA
//              applies s XOR gamma to its own full copy -- no
//              second cluster barrier.  Triple-buffered state and
//              step-parity-buffered gamma / any words make that safe: a peer
//              can be at most one step ahead, and the buffers it then writes
//              are not the ones this CTA is still reading.
//   stats      rank 0's warps p < n_props evaluate the properties and keep
//              the per-chain statistics exactly as K1 does.
// Randomness: the same Philox4x32-10 stream keyed by (seed, chain, t, node)
// (reading Q2), so the outputs are bit-identical to K1's for any K.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "pbn_internal.h"
#include "pbn_node.cuh"

namespace pbn {

namespace {

constexpr uint32_t QS3 = 48;  // bytes between quads of the triple-buffered state

__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cta address -> the same offset in CTA `peer`'s shared memory (shared::cluster)
__device__ __forceinline__ uint32_t map_peer(uint32_t a, uint32_t peer)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(peer));
    return r;
}

__device__ __forceinline__ void st_cluster128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w)
{
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w)
                 : "memory");
}

__device__ __forceinline__ void st_cluster32(uint32_t a, uint32_t v)
{
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <bool PER_NODE, int FT, bool SLOW>
__global__ void __launch_bounds__(PBN_MAX_THREADS, 1) traj_cluster_kernel(const __grid_constant__ ClusterParams C)
{
    const TrajParams& P = C.T;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t mbar;

    const int tid = threadIdx.x;
    const int wg = tid >> 5;
    const int lane = tid & 31;
    const int W = P.warps_per_group;
    const int n = P.n;
    const uint32_t rank = cluster_rank();
    const uint32_t K = (uint32_t)C.K;
    const int64_t group = blockIdx.x / K;

    // dynamic shared memory: [state 3 buffers | gamma x2 | any x2 | sub-image]
    const uint32_t gbase = smem_u32(smem);
    const uint32_t gam0 = gbase + QS3 * (uint32_t)P.nquads;            // gamma words, parity 0 / 1
    const uint32_t anyb = gam0 + 8u * (uint32_t)P.n_pad;               // [2][16][32] any words
    const uint32_t sbase = anyb + 2u * 16u * 32u * 4u;                 // sub-image
    const uint32_t img_bytes = C.img_bytes[rank];
    const uint8_t* gimg = P.image + C.img_off[rank];

    // ---- A1: stage this rank's sub-image (bulk async copy) and relocate ----
    Img<true> img;
    img.gbase = gimg;
    {
        const uint32_t bar = smem_u32(&mbar);
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(img_bytes)
                         : "memory");
            for (uint32_t off = 0; off < img_bytes; off += 32768u) {
                const uint32_t sz = min(32768u, img_bytes - off);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sbase + off),
                    "l"(gimg + off), "r"(sz), "r"(bar)
                    : "memory");
            }
        }
        __syncthreads();
        asm volatile(
            "{\n.reg .pred p;\nWAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
            "@!p bra WAIT_%=;\n}\n" ::"r"(bar)
            : "memory");
        const uint32_t* rel = reinterpret_cast<const uint32_t*>(gimg + C.reloc_off[rank]);
        for (int k = tid; k < C.reloc_count[rank]; k += blockDim.x) {
            const uint32_t e = __ldg(rel + k);
            const uint32_t a = sbase + (e & ~kRelocState);
            sts32(a, lds32(a) + ((e & kRelocState) ? gbase : sbase));
        }
        // gamma and any words start all-zero (the fix-up keeps gamma zero)
        for (uint32_t i = tid; i < 2u * (uint32_t)P.n_pad + 2u * 16u * 32u; i += blockDim.x) sts32(gam0 + 4u * i, 0u);
    }

    const bool leader = lane == 0;
    const uint32_t lead = leader ? FULL : 0u;
    const uint32_t rot = 31u - (uint32_t)lane;
    const uint32_t lmask = 1u << lane;

    // this CTA's quads, split over its warps
    const int rq0 = C.q_lo[rank], rq1 = C.q_lo[rank + 1];
    const int q0 = rq0 + (int)((int64_t)wg * (rq1 - rq0) / W);
    const int q1 = rq0 + (int)((int64_t)(wg + 1) * (rq1 - rq0) / W);
    const uint32_t node_lo = 4u * (uint32_t)rq0;  // first node of the sub-image
    const bool full_quads = (n & 3) == 0 || q1 < P.nquads;
    const int nsw = P.state_words;

    const int64_t chain_local = group * 32 + lane;
    const bool valid = chain_local < P.n_chains;
    const uint32_t chain = (uint32_t)(P.chain_base + chain_local);
    const uint32_t vmask = __ballot_sync(FULL, valid);  // lanes holding real chains
    const int prop = wg;
    const bool stats = rank == 0 && prop < P.n_props;
    const int64_t pofs = (int64_t)prop * P.n_chains;
    const int64_t total = P.burn_in + P.steps;
    const uint32_t Tp = P.Tp;

    // ---- A2: the whole initial state in buffer 0 (every CTA the same) ----
    if (P.init) {
        for (int q = wg; q < P.nquads; q += W) {
            const uint4 r = philox4x32_10((uint32_t)q, chain, 0u, 0u, P.rk);
            const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * q + k;
                if (i < n) {
                    const uint32_t wv = __ballot_sync(FULL, (rr[k] >> 31) != 0u);
                    if (leader) sts32(gbase + state_off(i, QS3), wv);
                }
            }
        }
    } else {
        for (int b = wg; b < nsw; b += W) {
            const uint32_t v = valid ? P.state[chain_local * nsw + b] : 0u;
            for (int k = 0; k < 32; ++k) {
                const int i = 32 * b + k;
                if (i >= n) break;
                const uint32_t wv = __ballot_sync(FULL, (v >> k) & 1u);
                if (leader) sts32(gbase + state_off(i, QS3), wv);
            }
        }
    }
    // every CTA of the cluster is staged and initialised before any remote store
    __syncthreads();
    cluster_sync_all();

    ChainStats cs;  // statistics of property `prop` (rank 0's statistics warps)

    auto step = [&](const int64_t r, auto ob_c) {
        constexpr uint32_t OB = decltype(ob_c)::value;
        constexpr uint32_t NB = OB == 32u ? 0u : OB + 16u;
        const uint32_t par = (uint32_t)(r & 1);
        const uint32_t gam = gam0 + 4u * (uint32_t)P.n_pad * par;
        const uint32_t anyw = anyb + 2048u * par;  // [16][32] words of this parity
        const uint64_t t = (uint64_t)(P.step0 + r);
        const uint32_t t_lo = (uint32_t)t, t_hi = (uint32_t)(t >> 32);
        uint32_t any = 0;
        const PhiloxStep ps = philox_step(chain, t_lo, t_hi, P.rk);
        const int qf = (full_quads || q1 == q0) ? q1 : q1 - 1;
        auto quad = [&](const int q, const uint4 rw, const Recs& rc, auto&& between) {
            const uint32_t i0 = 4u * (uint32_t)q;
            uint32_t g0, g1, g2, g3;
            const uint32_t w0 =
                node_word<true, PER_NODE, FT, SLOW, OB, QS3>(img, rc.r[0], i0, rw.x, Tp, gbase, lmask, rot, g0);
            const uint32_t w1 =
                node_word<true, PER_NODE, FT, SLOW, OB, QS3>(img, rc.r[1], i0 + 1, rw.y, Tp, gbase, lmask, rot, g1);
            const uint32_t w2 =
                node_word<true, PER_NODE, FT, SLOW, OB, QS3>(img, rc.r[2], i0 + 2, rw.z, Tp, gbase, lmask, rot, g2);
            const uint32_t w3 =
                node_word<true, PER_NODE, FT, SLOW, OB, QS3>(img, rc.r[3], i0 + 3, rw.w, Tp, gbase, lmask, rot, g3);
            between();
            // lane p < K pushes the quad's words into CTA p's copy: one store
            // instruction per quad for all the peers (the words are warp-uniform)
            if (lane < (int)K) st_cluster128(map_peer(gbase + QS3 * (uint32_t)q + NB, (uint32_t)lane), w0, w1, w2, w3);
            if (!PER_NODE) {
                const uint32_t g = g0 | g1 | g2 | g3;
                any |= g;
                if (g && lane < (int)K) st_cluster128(map_peer(gam + 4u * i0, (uint32_t)lane), g0, g1, g2, g3);
            }
        };
        uint4 rw = philox_quad((uint32_t)q0, ps, P.rk);
        for (int q = q0; q < qf; ++q) {
            uint4 rn;
            quad(q, rw, load_recs(img, sbase + 16u * (4u * (uint32_t)q - node_lo)),
                 [&] { rn = philox_quad((uint32_t)(q + 1), ps, P.rk); });
            rw = rn;
        }
        if (qf < q1) {  // ragged last quad (n % 4 != 0), node by node
            const uint32_t i0 = 4u * (uint32_t)qf;
            const uint32_t rr[4] = {rw.x, rw.y, rw.z, rw.w};
            for (uint32_t k = 0; k < 4 && (int)(i0 + k) < n; ++k) {
                uint32_t gk;
                const uint32_t wk = node_word<true, PER_NODE, FT, SLOW, OB, QS3>(
                    img, img.ld128(sbase + 16u * (i0 + k - node_lo)), i0 + k, rr[k], Tp, gbase, lmask, rot, gk);
                if (lane < (int)K) st_cluster32(map_peer(gbase + state_off(i0 + k, QS3) + NB, (uint32_t)lane), wk);
                if (!PER_NODE) {
                    any |= gk;
                    if (gk && lane < (int)K) st_cluster32(map_peer(gam + 4u * (i0 + k), (uint32_t)lane), gk);
                }
            }
        }
        if (!PER_NODE && lane < (int)K) st_cluster32(map_peer(anyw + 4u * (32u * rank + (uint32_t)wg), (uint32_t)lane), any);
        // publish the step to the cluster (release) and see every peer's (acquire)
        cluster_sync_all();
        if (!PER_NODE) {
            // VECTOR on this CTA's full copy: chains with any gamma
            // anywhere take s XOR gamma instead of f(s)
            uint32_t m = 0;
            for (uint32_t k = (uint32_t)lane; k < 32u * K; k += 32u) m |= lds32(anyw + 4u * k);
            // (lanes past the last chain are never written out: no fix-up for them)
            const uint32_t M = __reduce_or_sync(FULL, m) & vmask;
            if (M) {
                for (int i = tid; i < n; i += blockDim.x) {
                    const uint32_t gmm = lds32(gam + 4u * (uint32_t)i);
                    if (gmm) sts32(gam + 4u * (uint32_t)i, 0u);  // keep this parity's gamma words zero
                    const uint32_t a = gbase + state_off((uint32_t)i, QS3);
                    const uint32_t f = lds32(a + NB), o = lds32(a + OB);
                    sts32(a + NB, (f & ~M) | ((o ^ gmm) & M));
                }
            }
            // this parity's any words are rewritten by every warp before they
            // are read again (two steps later)
            __syncthreads();
        }
        if (stats && r > P.burn_in) {
            const uint32_t b =
                ChainStats::indicator(P, prop, lane, [&](uint32_t i) { return gbase + state_off(i, QS3) + NB; });
            cs.record(P, b, r - P.burn_in - 1, valid, pofs + chain_local);
        }
    };
    for (int64_t r = 1; r <= total; r += 3) {
        step(r, std::integral_constant<uint32_t, 0u>());
        if (r + 1 <= total) step(r + 1, std::integral_constant<uint32_t, 16u>());
        if (r + 2 <= total) step(r + 2, std::integral_constant<uint32_t, 32u>());
    }
    const uint32_t cur = 16u * (uint32_t)(total % 3);  // buffer of the newest state
    __syncthreads();

    // ---- epilogue (rank 0): final state back to chain-major rows, statistics ----
    if (rank == 0) {
        for (int b = wg; b < nsw; b += W) {
            uint32_t v = 0;
            for (int k = 0; k < 32; ++k) {
                const int i = 32 * b + k;
                if (i >= n) break;
                v |= ((lds32(gbase + state_off(i, QS3) + cur) >> lane) & 1u) << k;
            }
            if (valid) P.state[chain_local * nsw + b] = v;
        }
    }
    if (stats) cs.finish(P, prop, valid, pofs + chain_local, leader);
    // no CTA may exit while a peer can still read or write its shared memory
    cluster_sync_all();
}

template <bool PER_NODE, int FT, bool SLOW>
const void* ckptr()
{
    return reinterpret_cast<const void*>(&traj_cluster_kernel<PER_NODE, FT, SLOW>);
}

template <bool PER_NODE>
const void* cpick_ft(int FT, bool slow)
{
    switch (FT) {
        case 3: return slow ? ckptr<PER_NODE, 3, true>() : ckptr<PER_NODE, 3, false>();
        case 4: return slow ? ckptr<PER_NODE, 4, true>() : ckptr<PER_NODE, 4, false>();
        case 5: return slow ? ckptr<PER_NODE, 5, true>() : ckptr<PER_NODE, 5, false>();
        case 6: return slow ? ckptr<PER_NODE, 6, true>() : ckptr<PER_NODE, 6, false>();
        case 7: return slow ? ckptr<PER_NODE, 7, true>() : ckptr<PER_NODE, 7, false>();
        default: return slow ? ckptr<PER_NODE, 8, true>() : ckptr<PER_NODE, 8, false>();
    }
}

}  // namespace

size_t cluster_smem_bytes(const TrajParams& P, uint32_t max_sub_image)
{
    return (size_t)QS3 * P.nquads + 8u * (size_t)P.n_pad + 2u * 16u * 32u * 4u + max_sub_image;
}

int launch_traj_cluster(const ClusterParams& C, int warps, size_t smem_bytes, void* stream)
{
    const void* fn = C.T.per_node ? cpick_ft<true>(C.T.L.fast_theta, C.T.L.slow_nodes > 0)
                                  : cpick_ft<false>(C.T.L.fast_theta, C.T.L.slow_nodes > 0);
    cudaError_t e = ensure_func_smem(fn, smem_bytes, C.K > 8);
    if (e != cudaSuccess) return (int)e;
    const int64_t groups = (C.T.n_chains + 31) / 32;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(groups * C.K));
    cfg.blockDim = dim3((unsigned)(warps * 32));
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C.K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {const_cast<ClusterParams*>(&C)};
    e = cudaLaunchKernelExC(&cfg, fn, args);
    return (int)e;
}

int max_active_clusters(const ClusterParams& C, int warps, size_t smem_bytes, int* out)
{
    const void* fn = C.T.per_node ? cpick_ft<true>(C.T.L.fast_theta, C.T.L.slow_nodes > 0)
                                  : cpick_ft<false>(C.T.L.fast_theta, C.T.L.slow_nodes > 0);
    cudaError_t e = ensure_func_smem(fn, smem_bytes, C.K > 8);
    if (e != cudaSuccess) return (int)e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)C.K);
    cfg.blockDim = dim3((unsigned)(warps * 32));
    cfg.dynamicSmemBytes = smem_bytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C.K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaOccupancyMaxActiveClusters(out, fn, &cfg);
    return (int)e;
}

}  // namespace pbn
