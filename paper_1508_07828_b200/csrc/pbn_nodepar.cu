// pbn_nodepar.cu -- K1n: the trajectory kernel with LANES OVER NODES for the
// few-chain regime (BASELINE north_star: "one warp per chain with lanes over
// nodes for large n"; the node-parallel synchronous update of P:156-157).
//
// K1 / K1c put 32 chains on the 32 lanes of a warp (bit-sliced state), which
// leaves 31 of 32 lanes idle when a run has one chain.  Here G chains (G >= 1)
// run on a thread-block cluster of K CTAs (K = 1..16); a warp computes one
// 32-node word of one chain, its lane = a node (the quad's four lanes compute
// the same Philox call, whose 4 words cover nodes 4q..4q+3):
//   image      CTA rank r stages the records and descriptors of its nodes
//              [32 w_lo[r], 32 w_lo[r+1]) (whole packed state words), built
//              by pbn_load in the PACKED form: a parent entry is the parent's
//              node id (pbn_api.cpp build_image(..., packed = true)).
//   state      every CTA keeps the whole chain state bit-packed (node i = bit
//              i & 31 of word i >> 5, the API's row layout), double-buffered
//              by step parity; a parent bit is one LDS + one funnel shift.
//   exchange   a warp ballots its 32 nodes' new bits f and perturbation
//              bits gamma into one word each, lane 0 stores them locally and
//              lane p < K into peer p's exchange slot with st.async, whose
//              complete_tx lands on the peer's per-parity mbarrier -- no
//              cluster-wide barrier per step: a CTA waits only until the
//              bytes of this step from all its peers have arrived.  Two
//              slots per parity are enough: a peer cannot start step t+2
//              before it has this CTA's step t+1 words, which are sent after
//              this CTA has consumed step t.
//   commit     after the wait, every CTA forms s_t for the WHOLE chain from
//              the packed words: VECTOR s_t = any gamma ?
//              s_{t-1} XOR gamma : f (any gamma over all words of all CTAs);
//              PER_NODE s_t = f (the flip was applied per node).
//   stats      rank 0's warps p < n_props evaluate property p on s_t and keep
//              chain g's statistics in lane g (ChainStats, as K1).
// Randomness: the same Philox4x32-10 stream keyed by (seed, chain, t, node)
// (reading Q2): outputs are bit-identical to K1 / K1c for any K.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

#include "pbn_internal.h"
#include "pbn_node.cuh"

namespace pbn {

namespace {

__device__ __forceinline__ uint32_t np_cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t np_map_peer(uint32_t a, uint32_t peer)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(peer));
    return r;
}

__device__ __forceinline__ void np_cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 8 bytes {f, gamma} into a peer's shared memory; the transaction bytes
// complete on the peer's mbarrier (both shared::cluster addresses)
__device__ __forceinline__ void st_async_v2(uint32_t a, uint32_t x, uint32_t y, uint32_t mbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(a),
                 "r"(x), "r"(y), "r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void mbar_arm(uint32_t bar, uint32_t tx)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}

// wait for the phase with parity `phase`: the st.async bytes counted by
// complete_tx are visible to the waiting CTA once the phase completes (the
// transaction-count mechanism of TMA / st.async), so the default .acquire.cta
// semantics suffice (PBN_NP_ACQ_CLUSTER: cluster scope, for A/B only)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase)
{
#ifdef PBN_NP_ACQ_CLUSTER
#define PBN_NP_WAIT "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
#else
#define PBN_NP_WAIT "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
#endif
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n" PBN_NP_WAIT
        "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(phase)
        : "memory");
#undef PBN_NP_WAIT
}

// bit of node p in the packed state at S (shared address of word 0)
__device__ __forceinline__ uint32_t pbit(uint32_t S, uint32_t p)
{
    const uint32_t w = lds32_state(S + ((p >> 5) << 2));
    return __funnelshift_r(w, w, p) & 1u;  // wrap mode: rotate right by p mod 32
}

// A6 for one fast function of the packed image (desc_bytes_packed layout,
// u16 parent node ids, MSB first, reading Q5): returns the new bit
__device__ __forceinline__ uint32_t u16of(const uint32_t* pairs, int m)
{
    return (m & 1) ? pairs[m >> 1] >> 16 : pairs[m >> 1] & 0xFFFFu;
}
template <int FT>
__device__ __forceinline__ uint32_t fast_bit_packed(uint32_t dp, uint32_t S)
{
    uint32_t tw, idx = 0;
    const uint4 d0 = lds128_ro(dp);
    if constexpr (FT >= 7) {
        // {a[0..7] as u16, table words}: the first FT-5 parents pick the table word
        const uint32_t pr[4] = {d0.x, d0.y, d0.z, d0.w};
        uint32_t widx = 0;
#pragma unroll
        for (int m = 0; m < FT - 5; ++m) widx = 2u * widx + pbit(S, u16of(pr, m));
#pragma unroll
        for (int m = FT - 5; m < FT; ++m) idx = 2u * idx + pbit(S, u16of(pr, m));
        tw = lds32_ro(dp + 16u + 4u * widx);
    } else if constexpr (FT == 6) {
        // {t0, t1, a[0..5] as u16}
        const uint32_t pr[3] = {d0.z, d0.w, lds32_ro(dp + 16u)};
        tw = pbit(S, u16of(pr, 0)) ? d0.y : d0.x;
#pragma unroll
        for (int m = 1; m < 6; ++m) idx = 2u * idx + pbit(S, u16of(pr, m));
    } else {
        // {t0, a[0..FT-1] as u16}
        const uint32_t pr[3] = {d0.y, d0.z, d0.w};
        tw = d0.x;
#pragma unroll
        for (int m = 0; m < FT; ++m) idx = 2u * idx + pbit(S, u16of(pr, m));
    }
    // table words are stored bit-reversed: the entry is the sign bit of tw << idx
    return (uint32_t)((int32_t)(tw << idx) < 0);
}

// generic node (ell > 4 or theta_max > 8): slow record {thr, ell, gdesc,
// theta_max}, generic descriptors {toff, theta, poff, 0}, poff = parent node
// ids; binary-search selection (ascending thresholds), as slow_node_bit
__device__ __noinline__ uint32_t slow_bit_packed(uint32_t w, uint32_t u, uint32_t S)
{
    const uint4 sr = lds128_ro(w & ~15u);
    const uint32_t m1 = sr.y - 1u;
    uint32_t j = 0;
    for (uint32_t step = m1 ? 1u << (31 - __clz(m1)) : 0u; step; step >>= 1)
        if (j + step <= m1 && u > lds32_ro(sr.x + 4u * (j + step - 1u))) j += step;  // lane-divergent anyway
    const uint4 gd = lds128_ro(sr.z + 16u * j);
    uint32_t idx = 0;
    for (uint32_t m = 0; m < gd.y; ++m) idx = 2u * idx + pbit(S, lds32_ro(gd.z + 4u * m));
    const uint32_t tw = lds32_ro(gd.x + 4u * (idx >> 5));
    return (tw >> (idx & 31u)) & 1u;
}

// MODE: 0 VECTOR, 1 PER_NODE, 2 VECTOR with the geometric-skip stream
// (reading Q18): one warp per chain draws gamma(t) at the start of the step
// (any flip <=> the first skip word is below Cg[n-1]; the flip positions by
// skips over the image's table in global memory) into flip words Gm; a chain
// with gamma != 0 takes s XOR gamma, so its node evaluation is skipped.
// SHARE: a warp has >= 2 items per step, so quads' Philox calls are shared
// through shuffles (batches of up to 4 items); else one call per lane (the
// shuffles would only lengthen the latency chain of a lone item)
template <int MODE, int FT, bool SLOW, bool SHARE>
__global__ void __launch_bounds__(1024, 1) traj_nodepar_kernel(const __grid_constant__ NodeParParams C)
{
    constexpr bool PER_NODE = MODE == 1;
    constexpr bool GEO = MODE == 2;
    const TrajParams& P = C.T;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t mbar_img;
    __shared__ __align__(8) uint64_t mbar_x[2];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int wg = tid >> 5;
    const int T = blockDim.x;
    const int NWARP = T >> 5;
    const int n = P.n;
    const uint32_t rank = np_cluster_rank();
    const uint32_t K = (uint32_t)C.K;
    // G chains per cluster (the last cluster may hold fewer: every CTA of a
    // cluster agrees on Ge, so the exchange byte counts match)
    const int64_t cluster = blockIdx.x / K;
    const int64_t chain0 = cluster * C.G;
    const int Ge = (int)(P.n_chains - chain0 < (int64_t)C.G ? P.n_chains - chain0 : (int64_t)C.G);
    const int NW = C.n_words;
    const int NWp = (NW + 3) & ~3;

    // dynamic shared memory: S[2][G][NWp] packed state per step parity and
    // chain, X[2][G][NWp] {f, gamma} exchange words, Gm[2][G][NWp] geometric
    // flip words and Gf[2][G4] flags per step parity, then the sub-image
    const int G4 = (C.G + 3) & ~3;
    const uint32_t Sb = smem_u32(smem);
    const uint32_t Xb = Sb + 8u * (uint32_t)(C.G * NWp);
    const uint32_t Gmb = Xb + 16u * (uint32_t)(C.G * NWp);
    const uint32_t Gfb = Gmb + 8u * (uint32_t)(C.G * NWp);
    const uint32_t ibase = Gfb + 8u * (uint32_t)G4;
    auto Gmp = [&](uint32_t par, int g) { return Gmb + 4u * (uint32_t)((2 * g + (int)par) * NWp); };
    auto Gfp = [&](uint32_t par, int g) { return Gfb + 4u * (uint32_t)((int)par * G4 + g); };
    auto Sp = [&](uint32_t par, int g) { return Sb + 4u * (uint32_t)((2 * g + (int)par) * NWp); };
    auto Xp = [&](uint32_t par, int g) { return Xb + 8u * (uint32_t)((2 * g + (int)par) * NWp); };

    const int w_lo = C.w_lo[rank], w_hi = C.w_lo[rank + 1];  // own packed words (32 nodes each)
    const int OW = w_hi - w_lo;
    const uint32_t node_lo = 32u * (uint32_t)w_lo;
    const uint32_t tx_bytes = 8u * (uint32_t)Ge * (uint32_t)(NW - OW);  // bytes from the peers per step
    const uint32_t bx0 = smem_u32(&mbar_x[0]), bx1 = smem_u32(&mbar_x[1]);

    // ---- A1: stage this rank's sub-image; exchange barriers ----
    const uint8_t* gimg = P.image + C.img_off[rank];
    const uint32_t img_bytes = C.img_bytes[rank];
    {
        const uint32_t bar = smem_u32(&mbar_img);
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bx0));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bx1));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            // the exchange barriers of steps 1 and 2
            mbar_arm(bx1, tx_bytes);
            mbar_arm(bx0, tx_bytes);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(img_bytes)
                         : "memory");
            for (uint32_t off = 0; off < img_bytes; off += 32768u) {
                const uint32_t sz = min(32768u, img_bytes - off);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        ibase + off),
                    "l"(gimg + off), "r"(sz), "r"(bar)
                    : "memory");
            }
        }
        __syncthreads();
        mbar_wait(bar, 0);
        const uint32_t* rel = reinterpret_cast<const uint32_t*>(gimg + C.reloc_off[rank]);
        for (int k = tid; k < C.reloc_count[rank]; k += T) {
            const uint32_t a = ibase + __ldg(rel + k);
            sts32(a, lds32(a) + ibase);
        }
    }

    // ---- A2: every chain's whole initial state s_0 in S[0] (every CTA the same) ----
    for (int it = wg; it < Ge * NW; it += NWARP) {
        const int g = it / NW, j = it % NW;
        const uint32_t chain = (uint32_t)(P.chain_base + chain0 + g);
        uint32_t v;
        if (P.init) {
            const uint32_t i = 32u * (uint32_t)j + (uint32_t)lane;
            const uint4 r = philox4x32_10(i >> 2, chain, 0u, 0u, P.rk);
            const uint32_t u = (i & 2u) ? ((i & 1u) ? r.w : r.z) : ((i & 1u) ? r.y : r.x);
            v = __ballot_sync(FULL, (int)i < n && (u >> 31) != 0u);
        } else {
            v = P.state[(chain0 + g) * NW + j];
        }
        if (lane == 0) sts32(Sp(0, g) + 4u * (uint32_t)j, v);
    }
    // A4 of the geometric stream (reading Q18) for chain g at step t into the
    // parity `par` buffers: gamma(t) != 0 iff the first skip word is below
    // Cg[n-1]; then the flip positions by skips over the table (global
    // memory, L1-cached).  Every CTA draws the whole gamma(t) of its chains
    // (the commit applies it locally), one step AHEAD, so that a chain-step
    // with gamma != 0 skips its node evaluation and the draw is off the
    // step's critical path.
    auto geo_draw = [&](int g, uint64_t tt, uint32_t par) {
        const uint32_t Gm = Gmp(par, g), Gf = Gfp(par, g);
        if (lds32(Gf))  // the flips of two steps ago: clear their words
            for (int j = lane; j < NW; j += 32) sts32(Gm + 4u * (uint32_t)j, 0u);
        __syncwarp();
        if (lane == 0) {
            const uint32_t chain = (uint32_t)(P.chain_base + chain0 + g);
            uint32_t any = 0;
            uint4 v = philox4x32_10(0x80000000u, chain, (uint32_t)tt, (uint32_t)(tt >> 32), P.rk);
            if (v.x < C.geo_last) {
                any = 1;
                int k = -1;
                for (uint32_t m = 0;; ++m) {
                    if (m > 0 && (m & 3u) == 0)
                        v = philox4x32_10(0x80000000u + (m >> 2), chain, (uint32_t)tt, (uint32_t)(tt >> 32), P.rk);
                    const uint32_t w = (m & 3u) == 0 ? v.x : (m & 3u) == 1 ? v.y : (m & 3u) == 2 ? v.z : v.w;
                    k += 1 + geometric_skip(w, n, P.geo_inv_lnq, [&](int gg) { return __ldg(C.geo_table + gg); });
                    if (k >= n) break;
                    const uint32_t a = Gm + 4u * (uint32_t)(k >> 5);
                    sts32(a, lds32(a) | (1u << (k & 31)));
                }
            }
            sts32(Gf, any);
        }
        __syncwarp();
    };
    if (GEO) {
        for (int i = tid; i < 2 * C.G * NWp + 2 * G4; i += T) sts32(Gmb + 4u * i, 0u);  // flips start zero
        __syncthreads();
        for (int g = wg; g < Ge; g += NWARP) geo_draw(g, (uint64_t)(P.step0 + 1), 1u);  // step 1's gamma
    }
    __syncthreads();
    // every CTA is staged and its barriers armed before any peer stores
    np_cluster_sync();

    // statistics: rank 0's warp p < n_props keeps property p of the cluster's
    // chains in lanes 0..Ge-1 (ChainStats, as K1)
    const int prop = wg;
    const bool stats = rank == 0 && prop < P.n_props;
    const bool valid = lane < Ge;
    const int64_t row = (int64_t)prop * P.n_chains + chain0 + lane;
    ChainStats cs;
    const int64_t total = P.burn_in + P.steps;
    const uint32_t Tp = P.Tp;

    for (int64_t r = 1; r <= total; ++r) {
        const uint32_t par = (uint32_t)(r & 1);
        const uint32_t bar = par ? bx1 : bx0;
        const uint64_t t = (uint64_t)(P.step0 + r);
        // the geometric stream's gamma(t+1): drawn first by the last warps, so
        // that its latency overlaps this step's node work and exchange
        if (GEO && r < total)
            for (int g = NWARP - 1 - wg; g >= 0 && g < Ge; g += NWARP) geo_draw(g, t + 1, par ^ 1u);
        // ---- A3-A6: warp = (chain g, own word j), lane = node 32 j + lane ----
        // Items it = g OW + (j - w_lo), strided by the warp count and walked
        // without integer division.
        // one (chain g, word j) item with the 4 words of this lane's quad
        auto item = [&](int g, int j, uint32_t ux, uint32_t uy, uint32_t uz, uint32_t uw) {
            const uint32_t a = Xp(par, g) + 8u * (uint32_t)j;
            if (GEO && lds32(Gfp(par, g))) {
                // gamma(t) != 0: s_t = s_{t-1} XOR gamma, applied by
                // every CTA from its own draw at the commit; nothing to evaluate
                if (lane == 0) asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(0u), "r"(0u) : "memory");
                if (lane < (int)K && lane != (int)rank)
                    st_async_v2(np_map_peer(a, (uint32_t)lane), 0u, 0u, np_map_peer(bar, (uint32_t)lane));
                return;
            }
            const uint32_t So = Sp(par ^ 1u, g);
            const uint32_t i = 32u * (uint32_t)j + (uint32_t)lane;
            const bool live = (int)i < n;
            const uint32_t ic = live ? i : node_lo;  // lanes past the last node read a valid record
            const uint32_t u = (i & 2u) ? ((i & 1u) ? uw : uz) : ((i & 1u) ? uy : ux);
            const uint4 rec = lds128_ro(ibase + 16u * (ic - node_lo));
            const uint32_t gm = u < Tp ? 1u : 0u;  // gamma_i(t) (A4)
            uint32_t bit;
            if (!SLOW || (rec.w & 7u) != kSlowNode) {
                // A5: function j = #{k : u > E_k}
                uint32_t dp = rec.w;
                constexpr uint32_t DS = desc_bytes_packed(FT);
                if (u > rec.x) dp += DS;
                if (u > rec.y) dp += DS;
                if (u > rec.z) dp += DS;
                bit = fast_bit_packed<FT>(dp, So);
            } else {
                bit = slow_bit_packed(rec.w, u, So);
            }
            if (PER_NODE && gm) bit = pbit(So, ic) ^ 1u;  // node flips (reading Q1)
            // A7: the word of 32 nodes, f and gamma
            const uint32_t vf = __ballot_sync(FULL, live && bit);
            const uint32_t vg = __ballot_sync(FULL, live && gm);
            // lane 0 keeps it, lane p < K pushes it to peer p (one instruction for all peers)
            if (lane == 0) asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(vf), "r"(vg) : "memory");
            if (lane < (int)K && lane != (int)rank)
                st_async_v2(np_map_peer(a, (uint32_t)lane), vf, vg, np_map_peer(bar, (uint32_t)lane));
        };
        int g = wg / OW, jj = wg % OW;
        if constexpr (!SHARE) {
            // one item per warp and step: each lane computes its quad's call
            for (int it = wg; it < Ge * OW; it += NWARP, jj += NWARP) {
                while (jj >= OW) {
                    jj -= OW;
                    ++g;
                }
                const int j = w_lo + jj;
                const uint32_t i = 32u * (uint32_t)j + (uint32_t)lane;
                const uint32_t q = min(i >> 2, (uint32_t)P.nquads - 1u);
                const uint4 rw = philox4x32_10(q, (uint32_t)(P.chain_base + chain0 + g), (uint32_t)t,
                                               (uint32_t)(t >> 32), P.rk);
                item(g, j, rw.x, rw.y, rw.z, rw.w);
            }
        } else {
            // batches of up to 4 items: lane l computes the call of quad l & 7
            // of item l >> 3 (32 distinct calls), node lanes take their words
            // by shuffles -- one call per quad instead of one per node
            const int BATCH = min(4, (Ge * OW + NWARP - 1) / NWARP);
            for (int it0 = wg; it0 < Ge * OW; it0 += BATCH * NWARP) {
                int gk[4], jk[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (k > 0 && k < BATCH) jj += NWARP;
                    while (jj >= OW) {
                        jj -= OW;
                        ++g;
                    }
                    gk[k] = g;
                    jk[k] = w_lo + jj;
                }
                jj += NWARP;  // the next batch starts one stride after its last item
                const int nk = min(BATCH, (Ge * OW - it0 + NWARP - 1) / NWARP);  // items in this batch
                uint4 rw;
                {
                    const int k = lane >> 3;
                    const int gg = k == 0 ? gk[0] : k == 1 ? gk[1] : k == 2 ? gk[2] : gk[3];
                    const int jq = k == 0 ? jk[0] : k == 1 ? jk[1] : k == 2 ? jk[2] : jk[3];
                    const uint32_t q = min(8u * (uint32_t)jq + (uint32_t)(lane & 7), (uint32_t)P.nquads - 1u);
                    rw = philox4x32_10(q, (uint32_t)(P.chain_base + chain0 + gg), (uint32_t)t, (uint32_t)(t >> 32),
                                       P.rk);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (k >= nk) break;
                    const int src = 8 * k + (lane >> 2);  // the quad's call: lane 8 k + quad-in-word
                    const uint32_t ux = __shfl_sync(FULL, rw.x, src), uy = __shfl_sync(FULL, rw.y, src);
                    const uint32_t uz = __shfl_sync(FULL, rw.z, src), uw = __shfl_sync(FULL, rw.w, src);
                    item(gk[k], jk[k], ux, uy, uz, uw);
                }
            }
        }
        // ---- wait for every peer's words of this step: one warp spins on the
        // mbarrier, the others wait in the CTA barrier (spinning warps would
        // steal issue slots from the warps still computing) ----
        if (wg == 0) mbar_wait(bar, (uint32_t)((r - 1) >> 1) & 1u);
        __syncthreads();  // this CTA's own words too
        // ---- A7 commit of every chain (VECTOR: any gamma -> s XOR gamma), warp per chain ----
        for (int g = wg; g < Ge; g += NWARP) {
            const uint32_t So = Sp(par ^ 1u, g), Sn = Sp(par, g), X = Xp(par, g);
            uint32_t anyg = 0;
            if (!PER_NODE && !GEO)
                for (int j = lane; j < NW; j += 32) anyg |= lds32(X + 8u * (uint32_t)j + 4u);
            const bool any = PER_NODE ? false : GEO ? lds32(Gfp(par, g)) != 0u : __any_sync(FULL, anyg != 0u);
            // gamma words: exchanged (VECTOR) or this CTA's own draw (GEO)
            const uint32_t Gw = GEO ? Gmp(par, g) : X + 4u;
            const uint32_t Gs = GEO ? 4u : 8u;
            for (int j = lane; j < NW; j += 32) {
                uint32_t v = lds32(X + 8u * (uint32_t)j);
                if (!PER_NODE && any) v = lds32(So + 4u * (uint32_t)j) ^ lds32(Gw + Gs * (uint32_t)j);
                sts32(Sn + 4u * (uint32_t)j, v);
            }
        }
        // the exchange barrier of step r + 2 (same parity)
        if (tid == 0) mbar_arm(bar, tx_bytes);
        __syncthreads();
        // ---- A8 + A9 (rank 0): lane g = chain g ----
        if (stats && r > P.burn_in) {
            uint32_t b = 0;
            if (valid) {
                const uint32_t Sn = Sp(par, lane);
                b = 1;
                for (int k = 0; k < P.pred_k[prop]; ++k)
                    b &= pbit(Sn, P.pred_node[prop][k]) ^ (P.pred_val[prop][k] ^ 1u);
            }
            cs.record(P, b, r - P.burn_in - 1, valid, row);
        }
    }

    // ---- epilogue (rank 0): final state rows, statistics ----
    if (rank == 0)
        for (int it = tid; it < Ge * NW; it += T) {
            const int g = it / NW, j = it % NW;
            P.state[(chain0 + g) * NW + j] = lds32(Sp((uint32_t)(total & 1), g) + 4u * (uint32_t)j);
        }
    if (stats) cs.finish(P, prop, valid, row, lane == 0);
    // no CTA may exit while a peer can still write into its shared memory
    np_cluster_sync();
}

template <int MODE, int FT, bool SLOW>
const void* nkptr(bool share)
{
    return share ? reinterpret_cast<const void*>(&traj_nodepar_kernel<MODE, FT, SLOW, true>)
                 : reinterpret_cast<const void*>(&traj_nodepar_kernel<MODE, FT, SLOW, false>);
}

template <int MODE>
const void* npick_ft(int FT, bool slow, bool share)
{
    switch (FT) {
        case 3: return slow ? nkptr<MODE, 3, true>(share) : nkptr<MODE, 3, false>(share);
        case 4: return slow ? nkptr<MODE, 4, true>(share) : nkptr<MODE, 4, false>(share);
        case 5: return slow ? nkptr<MODE, 5, true>(share) : nkptr<MODE, 5, false>(share);
        case 6: return slow ? nkptr<MODE, 6, true>(share) : nkptr<MODE, 6, false>(share);
        case 7: return slow ? nkptr<MODE, 7, true>(share) : nkptr<MODE, 7, false>(share);
        default: return slow ? nkptr<MODE, 8, true>(share) : nkptr<MODE, 8, false>(share);
    }
}

const void* npick(const NodeParParams& C)
{
    const int FT = C.T.L.fast_theta;
    const bool slow = C.T.L.slow_nodes > 0;
    return C.T.per_node ? npick_ft<1>(FT, slow, C.share)
                        : C.T.geometric ? npick_ft<2>(FT, slow, C.share) : npick_ft<0>(FT, slow, C.share);
}

cudaLaunchConfig_t ncfg(const NodeParParams& C, int threads, size_t smem, unsigned grid, cudaLaunchAttribute* attr)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C.K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

cudaError_t nprepare(const void* fn, const NodeParParams& C, size_t smem)
{
    return ensure_func_smem(fn, smem, C.K > 8);
}

}  // namespace

size_t nodepar_smem_bytes(int n_words, int G, uint32_t max_sub_image)
{
    const size_t NWp = ((size_t)n_words + 3) & ~(size_t)3;
    return (8u + 16u + 8u) * NWp * (size_t)G + 8u * (((size_t)G + 3) & ~(size_t)3) + max_sub_image;
}

int launch_traj_nodepar(const NodeParParams& C, int threads, size_t smem_bytes, void* stream)
{
    const void* fn = npick(C);
    cudaError_t e = nprepare(fn, C, smem_bytes);
    if (e != cudaSuccess) return (int)e;
    cudaLaunchAttribute attr[1];
    const int64_t clusters = (C.T.n_chains + C.G - 1) / C.G;
    cudaLaunchConfig_t cfg = ncfg(C, threads, smem_bytes, (unsigned)(clusters * C.K), attr);
    cfg.stream = (cudaStream_t)stream;
    void* args[] = {const_cast<NodeParParams*>(&C)};
    return (int)cudaLaunchKernelExC(&cfg, fn, args);
}

int max_active_nodepar_clusters(const NodeParParams& C, int threads, size_t smem_bytes, int* out)
{
    const void* fn = npick(C);
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
    const auto key = std::make_tuple(fn, (int)C.K, threads, smem_bytes);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *out = it->second;
            return 0;
        }
    }
    cudaError_t e = nprepare(fn, C, smem_bytes);
    if (e != cudaSuccess) return (int)e;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = ncfg(C, threads, smem_bytes, (unsigned)C.K, attr);
    const cudaError_t r = cudaOccupancyMaxActiveClusters(out, fn, &cfg);
    if (r == cudaSuccess) {
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = *out;
    }
    return (int)r;
}

}  // namespace pbn
