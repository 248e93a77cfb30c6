// pbn_bitslice_kernel.cuh -- K1b: the fused PBN trajectory kernel with
// BIT-SLICED function evaluation (sm_100a); the kernel template, instantiated
// per MODE in pbn_bitslice_m{0,1,2}.cu (parallel build), dispatched by
// pick_bitslice_kernel (pbn_bitslice.cu).
//
// The same hot path as K1 (§2.2) on
// the same group layout -- one 32-chain group per CTA, its state bit-sliced
// in shared memory (word i = node i of the 32 chains, bit l = chain of lane
// l; here THREE interleaved buffers, pbn_internal.h) -- but the node step is
// split in two phases so that the truth-table work is done once per 32
// chains instead of once per chain:
//
//   phase A (lane = chain; every warp its quads of nodes, as K1):
//     one Philox4x32-10 call per quad (A3, reading Q2), finished from a per-
//     (quad, step) table entry that one lane per quad computes once per step
//     (rounds 1-2 and the lane-uniform M0 product of round 3; pbn_node.cuh:
//     philox_quad_step_consts / philox_quad_ps); per node the bits of the
//     selected index j = #{m : u > E_m} as ballots (A5: b_0 = the parity of
//     the compares, b_1 = [u > E_2]; phase B takes the chains whose index
//     bits equal a function's j); one vote per quad flags the ~1 % of quads
//     where some chain drew u < T_p, whose gamma words (A4) are formed after
//     the quad loop; per quad the plane vectors are stored by every lane
//     (warp-uniform values, no predicate), the gamma and next-state zero
//     vectors for 32 quads at once before the loop.
//   phase B (lane = task = one predictor function of one node):
//     the parents' bit-sliced words are gathered (A6: one LDS per parent for
//     all 32 chains), the function's truth table is evaluated on them as a
//     multiplexer tree (entry masks at the leaves, one LOP3 per inner node:
//     bit l of the result is table[idx of chain l]), masked by the
//     function's selection plane and OR-ed into the node's new word (A7:
//     the chains' selections are disjoint, so the OR over a node's tasks is
//     f(s)); the task of function 0 also adds the perturbation term --
//     VECTOR: chains with any gamma (M) take s XOR gamma;
//     PER_NODE: chains with gamma_i take NOT s_i.
//   statistics (A8-A10): as K1, on the committed words.
//
// Phase A reads no state, so phase A of step t+1 shares an interval with
// phase B of step t (half of each scheduler's warps A first, the others B
// first, so the pipes see both instruction mixes at once): one CTA barrier per step; the planes and
// any words are double-buffered by step parity and the state triple-buffered
// (B(t) reads S_{t-1}, ORs into S_t; A(t+1) zeroes S_{t+1}'s buffer; the
// statistics warp reads S_t in the next interval).
//
// The quads are split over the warps by each warp's phase-B round cost (all
// warps meet at the one barrier per step), and phase B walks a per-warp list
// of its rounds class by class (the class a compile-time constant).
//
// Per node-update the work is one quarter of a Philox call, L-1 compare +
// ballot pairs and ~1/32 of the task's gather and tree instead
// of K1's per-chain gather of FT padded parents and per-chain descriptor
// reads.  Every output is bit-identical to K1's (the same stream,
// thresholds, tables and statistics).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "pbn_internal.h"
#include "pbn_node.cuh"

namespace pbn {
namespace {

// 16-byte shared load ordered with the barriers (the per-quad Philox table
// is rewritten every step)
__device__ __forceinline__ uint4 lds128_state(uint32_t a)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

#if defined(PBN_BS_PRED_STORES)
__device__ __forceinline__ void sts128_all(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w)
{
    sts128_if(a, x, y, z, w, (threadIdx.x & 31) == 0 ? FULL : 0u);
}
#else
// 16-byte store of a warp-uniform vector by every lane (same address, same value)
__device__ __forceinline__ void sts128_all(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w)
{
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
#endif

// multiplexer tree: the sub-table of entries [B, B + 2^(C-K)) evaluated on
// the parent words x[K..C-1] (x[0] = parents[0] = the index MSB, reading Q5):
// x[K] = 0 selects the lower half, 1 the upper -- bit l of the result is the
// entry at chain l's index; table word w holds entries 32 w .. 32 w + 31
template <int K, int C, int B>
__device__ __forceinline__ uint32_t mux_tree(const uint32_t (&t)[8], const uint32_t (&x)[C])
{
    if constexpr (K == C) {
        return (uint32_t)((int32_t)(t[B >> 5] << (31 - (B & 31))) >> 31);  // entry B as a word mask
    } else {
        constexpr int H = 1 << (C - K - 1);
        const uint32_t lo = mux_tree<K + 1, C, B>(t, x);
        const uint32_t hi = mux_tree<K + 1, C, B + H>(t, x);
        return (x[K] & hi) | (~x[K] & lo);
    }
}

// The bitslice image, staged in shared memory (SMEM) or read through the
// read-only global path (large models, e.g. C5: tasks are read coalesced,
// a round's 32 records consecutive; thresholds and round records are warp-
// uniform broadcasts).  Offsets are bytes from the image start.
template <bool SMEM>
struct BImg {
    const uint8_t* g;  // global image
    uint32_t s;        // shared address of the staged image
    __device__ __forceinline__ uint4 ld128(uint32_t off) const
    {
        if (SMEM) return lds128_ro(s + off);
        return __ldg(reinterpret_cast<const uint4*>(g + off));
    }
    __device__ __forceinline__ uint2 ld64(uint32_t off) const
    {
        if (SMEM) return lds64_ro(s + off);
        return __ldg(reinterpret_cast<const uint2*>(g + off));
    }
};

// record stride of task class c (table words, then the u16 list
// [state_off(i) | j, p_0 .. p_{c-1}]; pbn_internal.h)
__host__ __device__ constexpr uint32_t bs_stride(int c) { return c <= 5 ? 16u : c <= 7 ? 32u : 64u; }

// plane vectors per quad: NP selection-index planes (b0 = bit 0 of j, b1 =
// bit 1) and the gamma vector
template <int L>
struct Planes {
    static constexpr int NP = L >= 3 ? 2 : L == 2 ? 1 : 0;
    static constexpr int PV = NP + 1;
};

// one round of 32 tasks of class C (theta = C parents), lane = task.  gob / gnb
// are the shared addresses of the old / new state buffer (uniform); the node's
// plane words are at pl + 16 m (m < NP: b_m; m = NP: gamma).
template <int C, int MODE, int L, bool SMEM>
__device__ __forceinline__ void bs_round(const BImg<SMEM>& img, uint32_t ta, uint32_t gob, uint32_t gnb, uint32_t selq,
                                         uint32_t M)
{
    constexpr int T = C <= 5 ? 1 : (1 << C) / 32;      // table words
    constexpr int NV = (4 * T + 2 * (C + 1) + 15) / 16;  // 16-byte vectors of the record
    constexpr int NP = Planes<L>::NP, PV = Planes<L>::PV;
    uint32_t w[4 * NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const uint4 r = img.ld128(ta + 16u * v);
        w[4 * v] = r.x;
        w[4 * v + 1] = r.y;
        w[4 * v + 2] = r.z;
        w[4 * v + 3] = r.w;
    }
    uint32_t t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) t[k] = k < T ? w[k] : 0u;
    // u16 k of the list (0: state_off(i) | j; 1 + m: parent m)
    auto u16 = [&](int k) -> uint32_t {
        const uint32_t x = w[T + (k >> 1)];
        return (k & 1) ? x >> 16 : x & 0xFFFFu;
    };
    uint32_t x[C];
#pragma unroll
    for (int m = 0; m < C; ++m) x[m] = lds32_state(gob + u16(1 + m));
    const uint32_t F = mux_tree<0, C, 0>(t, x);
    // u16 0 = the node's state offset 48 (i >> 2) + 4 (i & 3) with j in its two
    // low bits; with three plane vectors per quad it is also the offset of the
    // node's plane words (selq = the plane buffer less the CTA's first quad)
    const uint32_t h0 = u16(0);
    const uint32_t so = h0 & 0xFFFCu, j = h0 & 3u;
    uint32_t pl;
    if constexpr (PV == 3)
        pl = selq + so;
    else
        pl = selq + 16u * (uint32_t)PV * ((so * 43691u) >> 21) + (so & 12u);  // (so / 48: exact below 2^16)
    // selection plane of function j: the chains whose index bits equal j's
    const uint32_t b0 = NP >= 1 ? lds32_state(pl) : 0u;
    const uint32_t b1 = NP >= 2 ? lds32_state(pl + 16u) : 0u;
    const uint32_t gam = lds32_state(pl + 16u * NP);
    const uint32_t m0 = (j & 1u) - 1u, m1 = ((j >> 1) & 1u) - 1u;  // all ones where the bit of j is 0
    const uint32_t sj = (b0 ^ m0) & (NP >= 2 ? (b1 ^ m1) : m1);
    const uint32_t out = so;
    const uint32_t old = lds32_state(gob + out);
    const uint32_t first = j == 0 ? FULL : 0u;  // function 0 carries the perturbation term
    uint32_t c;
    if (MODE == 1) {  // PER_NODE: chains with gamma_i take NOT s_i
        c = (F & sj & ~gam) | (~old & gam & first);
    } else {          // VECTOR: chains with any gamma take s XOR gamma
        c = (F & sj & ~M) | ((old ^ gam) & M & first);
    }
    // (unconditional: a zero word is rare, and the predicated form costs a branch)
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(gnb + out), "r"(c) : "memory");
}

// MODE: 0 VECTOR, 1 PER_NODE, 2 geometric; L = the model's largest ell;
// IMG: 0 image through L1/L2, 1 image staged, 2 CLUSTER -- one group per
// cluster of K CTAs, CTA rank r owns quads [qlo, qhi) (its sub-image: their
// thresholds and their nodes' tasks), keeps the whole state and, after each
// step's barrier, pushes its nodes' new words (and its any word) into every
// peer through distributed shared memory before one cluster barrier;
// CMAX: the largest task class (6 or 8)
// TB: the thread budget (768 = 24 warps x 80 registers, or 640 = 20 warps x
// ~94 registers: the staged-image kernels run faster with the latter, the
// global-image kernel needs the warps to cover its L1/L2 reads)
template <int MODE, int L, int IMG, int CMAX, int TB>
__global__ void __launch_bounds__(TB, 1) bitslice_kernel(const __grid_constant__ BitsliceParams B)
{
    constexpr bool SMEM = IMG != 0;
    constexpr bool CLU = IMG == 2;
    const TrajParams& P = B.T;
    constexpr bool PER_NODE = MODE == 1;
    constexpr bool GEO = MODE == 2;  // VECTOR with the geometric-skip stream (reading Q18)
    constexpr uint32_t QS = kBitsliceQs;
    constexpr int NP = Planes<L>::NP, PV = Planes<L>::PV;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t mbar;

    const int tid = threadIdx.x;
    const int wg = (int)__reduce_max_sync(FULL, (uint32_t)(tid >> 5));  // (warp-uniform for ptxas: no divergence guards on the votes)
    const int lane = tid & 31;
    const int W = P.warps_per_group;
    const int n = P.n;
    const uint32_t gbase = smem_u32(smem);
    const uint32_t sbase = gbase + 4u * (uint32_t)P.group_words;  // staged image base
    uint32_t rank = 0;
    if (CLU) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int KC = CLU ? B.K : 1;  // CTAs per cluster
    const uint8_t* const gimg = P.image + (CLU ? B.c_img_off[rank] : 0u);
    const uint32_t img_bytes = CLU ? B.c_img_bytes[rank] : P.image_smem_bytes;

    // ---- A1: stage the image into shared memory (bulk async copy) ----
    if (SMEM) {
        const uint32_t bar = smem_u32(&mbar);
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(img_bytes)
                         : "memory");
            const uint32_t chunk = 32768;
            for (uint32_t off = 0; off < img_bytes; off += chunk) {
                const uint32_t sz = min(chunk, img_bytes - off);
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
    }
    BImg<SMEM> img;
    img.g = P.image;
    img.s = sbase;

    const bool leader = lane == 0;
    const uint32_t lead = leader ? FULL : 0u;
    const uint32_t lmask = 1u << lane;
    const uint32_t anyw0 = gbase + (uint32_t)B.any_off;  // any[2][32]
    const uint32_t sel0 = gbase + (uint32_t)B.sel_off;   // planes[2]
    const uint32_t pqt = gbase + (uint32_t)B.pq_off;     // per-quad Philox table
    const uint32_t erec = CLU ? B.c_erec_off[rank] : B.erec_off;
    const uint32_t rounds = CLU ? B.c_rounds_off[rank] : B.rounds_off;
    const int R = CLU ? B.c_rounds[rank] : B.n_rounds;
    // this CTA's quads [qlo, qhi) (all of them outside a cluster); erec, the
    // planes and the Philox table are indexed by the local quad q - qlo
    const int qlo = CLU ? B.c_qlo[rank] : 0, qhi = CLU ? B.c_qlo[rank + 1] : P.nquads;
    const uint32_t cany = anyw0 + 256u;  // cluster: any words of the ranks [2][16], then a dummy word

    const int NW = P.node_warps;
#if defined(PBN_BS_NO_BALANCE)
    const int q0 = wg < NW ? qlo + (int)((int64_t)wg * (qhi - qlo) / NW) : qhi;
    const int q1 = wg < NW ? qlo + (int)((int64_t)(wg + 1) * (qhi - qlo) / NW) : qhi;
#else
    // Quads over the node warps so that every warp's step costs the same: the
    // snake order gives the warps phase-B rounds of different classes (one
    // class-6 round is worth ~4 quads of phase A), and all of them meet at
    // one barrier per step.  Lane l works out warp l's share (instruction
    // counts of the SASS bodies, per round / per quad); every warp computes
    // the same split.  Outputs do not depend on it.
    int q0, q1;
    {
        constexpr int kRoundCost[9] = {0, 37, 48, 62, 90, 145, 270, 525, 1035};
        constexpr int kQuadCost = L >= 4 ? 68 : L == 3 ? 62 : L == 2 ? 52 : 42;
        int cb = 0;
        if (lane < W)
            for (int m = 0; m * W < R; ++m) {
                const int rr_i = (m & 1) ? (m + 1) * W - 1 - lane : m * W + lane;
                if (rr_i < R) cb += kRoundCost[min(img.ld64(rounds + 8u * (uint32_t)rr_i).y, 8u)];
            }
        const int nq = qhi - qlo;
        const int tot = (int)__reduce_add_sync(FULL, lane < NW ? (uint32_t)cb : 0u) + kQuadCost * nq;
        // warp l's phase-A share x_l = T - cb_l (>= 0), T = tot / NW
        int x = lane < NW ? max(tot / NW - cb, 0) : 0;
        int sx = x;  // inclusive scan
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(FULL, sx, d);
            if (lane >= d) sx += y;
        }
        const int st = __shfl_sync(FULL, sx, 31);
        // cumulative rounding: warp l ends at round(nq S_l / S_tot), the last at nq
        const int e1 = st > 0 ? (int)(((int64_t)sx * nq + st / 2) / st) : (int)((int64_t)(min(lane, NW - 1) + 1) * nq / NW);
        const int e0 = __shfl_up_sync(FULL, e1, 1);
        const int w_ = min(wg, 31);
        const int a1 = __shfl_sync(FULL, e1, w_), a0 = wg == 0 ? 0 : __shfl_sync(FULL, e0, w_);
        q0 = wg < NW ? qlo + a0 : qhi;
        q1 = wg < NW ? qlo + a1 : qhi;
    }
#endif
    // This warp's phase-B rounds (the snake order over the round list, which
    // is sorted by class, most expensive first) as a list of task offsets in
    // shared memory, one sentinel after each class from CMAX down to 1: phase
    // B walks it class by class with the class a compile-time constant (no
    // per-round index arithmetic, round record, stride select or switch).
    constexpr uint32_t kListEnd = 0xFFFFFFFFu;
    const uint32_t rl = gbase + (uint32_t)B.rl_off + 4u * (uint32_t)(wg * B.rl_stride);
    if (leader) {
        uint32_t p = rl;
        int c = CMAX;
        for (int m = 0; m * W < R; ++m) {
            const int rr_i = (m & 1) ? (m + 1) * W - 1 - wg : m * W + wg;
            if (rr_i >= R) continue;
            const uint2 rr = img.ld64(rounds + 8u * (uint32_t)rr_i);
            for (; c > (int)rr.y; --c, p += 4u) sts32(p, kListEnd);
            sts32(p, rr.x);
            p += 4u;
        }
        for (; c >= 1; --c, p += 4u) sts32(p, kListEnd);
    }
    __syncwarp();
    // all quads over the warps (the initial state: every CTA forms all of it)
    const int qi0 = (int)((int64_t)wg * P.nquads / W), qi1 = (int)((int64_t)(wg + 1) * P.nquads / W);
    const int nsw = P.state_words;
    const int b0 = (int)((int64_t)wg * nsw / W), b1 = (int)((int64_t)(wg + 1) * nsw / W);
    const int64_t total = P.burn_in + P.steps;
    const uint32_t Tp = P.Tp;
    const bool full_quads = (n & 3) == 0 || q1 < P.nquads;
    // half of the warps run A(t+1) then B(t), the others B(t) then A(t+1),
    // alternating among the warps of one scheduler (warp w issues on scheduler
    // w % 4), so every scheduler sees both instruction mixes at once (by warp
    // parity instead -- the same order on all of a scheduler's warps -- C5
    // loses 2-3 %, C4 / C3 0.4 %; all warps A first: C4 -1 %)
    const bool a_first = ((wg >> 2) & 1) == 0;
    __shared__ unsigned long long s_unit;

    for (int64_t it = 0;; ++it) {
        int64_t group, chunk, r_begin, r_end;
        if (!P.persistent) {
            if (it > 0) break;
            group = CLU ? blockIdx.x / KC : blockIdx.x;
            chunk = 0;
            r_begin = 1;
            r_end = total;
        } else {
            __syncthreads();
            if (tid == 0) s_unit = atomicAdd(P.work_ctr, 1ull);
            __syncthreads();
            const unsigned long long u = __reduce_max_sync(FULL, (uint32_t)s_unit);
            if (u >= (unsigned long long)P.total_units) break;
            group = (int64_t)(u % (unsigned long long)P.n_groups);
            chunk = (int64_t)(u / (unsigned long long)P.n_groups);
            r_begin = chunk * P.chunk_steps + 1;
            r_end = min(total, (chunk + 1) * P.chunk_steps);
            if (chunk > 0 && tid == 0) {
                for (;;) {
                    unsigned int d;
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(P.done + group) : "memory");
                    if ((int64_t)d >= chunk) break;
                    __nanosleep(256);
                }
            }
        }
        const bool first_chunk = chunk == 0;
        const bool last_chunk = r_end >= total;
        const uint32_t chain_local = (uint32_t)group * 32u + (uint32_t)lane;
        const bool valid = (int64_t)chain_local < P.n_chains;
        const uint32_t chain = (uint32_t)(P.chain_base + chain_local);
        const uint32_t vmask = __ballot_sync(FULL, valid);
        auto scr = [&]() { return P.scratch + group * (int64_t)P.scratch_stride; };
        const int prop = wg - P.stats_warp0;
        const bool stats = prop >= 0 && prop < P.n_props && rank == 0;  // (cluster: rank 0 keeps them)
        auto orow = [&]() { return (int64_t)prop * P.n_chains + chain_local; };
        ChainStats cs;

        // S_0 of the unit into state buffer 0
        if (!first_chunk) {
            __syncthreads();
            for (int i = tid; i < n; i += blockDim.x) sts32(gbase + state_off(i, QS), __ldcg(scr() + i));
            if (stats) {
                const uint32_t* st = scr() + P.n_pad + 8 * 32 * prop + 8 * lane;
                cs.c1 = __ldcg(st + 0);
                cs.n01 = __ldcg(st + 1);
                cs.n10 = __ldcg(st + 2);
                cs.first = __ldcg(st + 3);
                cs.prev = __ldcg(st + 4);
                cs.bacc = __ldcg(st + 5);
                cs.bitw = __ldcg(st + 6);
                cs.bcount = __ldcg(st + 7);
            }
        } else if (P.init) {
            // A2: s_0[i] = u(chain, 0, i) >> 31
            for (int q = qi0; q < qi1; ++q) {
                const uint4 r = philox4x32_10((uint32_t)q, chain, 0u, 0u, P.rk);
                const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = 4 * q + k;
                    if (i < n) {
                        const uint32_t wv = __ballot_sync(FULL, (rr[k] >> 31) != 0u);
                        if (leader) sts32(gbase + state_off(i, QS), wv);
                    }
                }
            }
        } else {
            for (int b = b0; b < b1; ++b) {
                const uint32_t v = valid ? P.state[(int64_t)chain_local * nsw + b] : 0u;
                for (int k = 0; k < 32; ++k) {
                    const int i = 32 * b + k;
                    if (i >= n) break;
                    const uint32_t wv = __ballot_sync(FULL, (v >> k) & 1u);
                    if (leader) sts32(gbase + state_off(i, QS), wv);
                }
            }
        }

        // unit step k = 1..K is step r = r_begin - 1 + k; S_k in buffer k % 3
        const int64_t K = r_end - r_begin + 1;

        // ---- phase A of unit step k: planes -> planes[k & 1], zero S_k's buffer (byte offset zb) ----
        auto phaseA = [&](const int64_t k, const uint32_t zb) {
            const uint64_t t = (uint64_t)(P.step0 + r_begin - 1 + k);
            const uint32_t t_lo = (uint32_t)t, t_hi = (uint32_t)(t >> 32);
            const uint32_t sel = sel0 + (uint32_t)(k & 1) * (uint32_t)B.sel_bytes;
            const uint32_t gzb = gbase + zb;
            uint32_t any = 0;
            const PhiloxStep ps = philox_step(chain, t_lo, t_hi, P.rk);
            const int qf = (full_quads || q1 == q0) ? q1 : q1 - 1;
            // quad q's record: PV vectors of 16 bytes at sel + 16 PV q -- the
            // selection-index planes b_0 (b_1) of its 4 nodes, then their gamma
            // words: chain l picks function j = #{m : u_l > E_m}, b_0 = bit 0 of j
            // (the parity of the compares, the thresholds ascending), b_1 = bit 1
            // (= [u > E_2])
            auto thresholds = [&](const int q, uint4 (&e)[3]) {
                const uint32_t ea = erec + 16u * (uint32_t)(L - 1) * (uint32_t)(q - qlo);
#pragma unroll
                for (int m = 0; m < L - 1; ++m) e[m] = img.ld128(ea + 16u * m);
            };
            auto planes = [&](const int q, const uint4 rw, const uint4 (&e)[3]) {
                const uint32_t pa = sel + 16u * (uint32_t)PV * (uint32_t)(q - qlo);
                const uint32_t u[4] = {rw.x, rw.y, rw.z, rw.w};
                uint32_t pb0[4], pb1[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t E1 = k == 0 ? e[0].x : k == 1 ? e[0].y : k == 2 ? e[0].z : e[0].w;
                    const uint32_t E2 = k == 0 ? e[1].x : k == 1 ? e[1].y : k == 2 ? e[1].z : e[1].w;
                    const uint32_t E3 = k == 0 ? e[2].x : k == 1 ? e[2].y : k == 2 ? e[2].z : e[2].w;
                    if (L == 2) {
                        pb0[k] = __ballot_sync(FULL, u[k] > E1);
                    } else if (L == 3) {
                        // (the compare of E_2 shared by both planes: setp with
                        // a predicate operand, 2 ISETP + 2 VOTE per node)
                        asm volatile("{\n\t.reg .pred p2, p0;\n\t"
                            "setp.gt.u32 p2, %2, %4;\n\t"
                            "setp.gt.xor.u32 p0, %2, %3, p2;\n\t"
                            "vote.sync.ballot.b32 %0, p0, 0xffffffff;\n\t"
                            "vote.sync.ballot.b32 %1, p2, 0xffffffff;\n\t}"
                            : "=r"(pb0[k]), "=r"(pb1[k])
                            : "r"(u[k]), "r"(E1), "r"(E2));
                    } else if (L == 4) {
                        // (3 ISETP + 2 VOTE per node; ptxas recomputes the E_2
                        // compare when this is written with bools: 4 ISETP)
                        asm volatile("{\n\t.reg .pred p2, p0;\n\t"
                            "setp.gt.u32 p2, %2, %4;\n\t"
                            "setp.gt.xor.u32 p0, %2, %3, p2;\n\t"
                            "setp.gt.xor.u32 p0, %2, %5, p0;\n\t"
                            "vote.sync.ballot.b32 %0, p0, 0xffffffff;\n\t"
                            "vote.sync.ballot.b32 %1, p2, 0xffffffff;\n\t}"
                            : "=r"(pb0[k]), "=r"(pb1[k])
                            : "r"(u[k]), "r"(E1), "r"(E2), "r"(E3));
                    }
                }
                // (the ballots are warp-uniform: every lane stores the same
                // vector to the same address, no predicate)
                if (NP >= 1) sts128_all(pa, pb0[0], pb0[1], pb0[2], pb0[3]);
                if (NP >= 2) sts128_all(pa + 16u, pb1[0], pb1[1], pb1[2], pb1[3]);
            };
            auto gammas = [&](const int q, const uint4 rq) {
                const uint32_t g0 = __ballot_sync(FULL, rq.x < Tp), g1 = __ballot_sync(FULL, rq.y < Tp);
                const uint32_t g2 = __ballot_sync(FULL, rq.z < Tp), g3 = __ballot_sync(FULL, rq.w < Tp);
                any |= g0 | g1 | g2 | g3;
                sts128_if(sel + 16u * (uint32_t)PV * (uint32_t)(q - qlo) + 16u * NP, g0, g1, g2, g3, lead);
            };
            // the per-(quad, step) Philox entries of this warp's quads (and of
            // the quad after them, which the last iteration prefetches): one
            // lane per quad; only this warp reads them (the neighbour warp
            // writes the same value into the shared boundary entry)
            // (uniform trip count and a predicated store: the warp stays
            // provably converged for the ballots below)
            // The same lanes zero their quad's gamma vector (flagged quads
            // fill it below) and its words of S_k's buffer (OR-ed in phase B):
            // one store per 32 quads instead of one per quad.
            for (int qb = q0; qb <= q1 && q0 < q1; qb += 32) {
                const int qe = qb + lane;
                const uint4 c = philox_quad_step_consts((uint32_t)qe, ps, P.rk);
                sts128_if(pqt + 16u * (uint32_t)(qe - qlo), c.x, c.y, c.z, c.w, qe <= q1 ? FULL : 0u);
                const uint32_t own = qe < q1 ? FULL : 0u;
                if (!GEO) sts128_if(sel + 16u * (uint32_t)PV * (uint32_t)(qe - qlo) + 16u * NP, 0u, 0u, 0u, 0u, own);
                sts128_if(gzb + QS * (uint32_t)qe, 0u, 0u, 0u, 0u, own);
            }
            __syncwarp();
            uint4 rw = philox_quad_ps(lds128_state(pqt + 16u * (uint32_t)(q0 - qlo)), ps, P.rk);
            uint4 e[3];
            for (int qc = q0; qc < qf; qc += 32) {
                const int qe = min(qf, qc + 32);
                uint32_t gpend = 0;  // flags of the chunk's quads, newest = bit 0
                // one quad: the flag vote first -- the quad's thresholds, the
                // next quad's Philox call and the plane ballots follow it in
                // one basic block, so the scheduler overlaps the loads' latency
                // and the Philox chain with the ballots
                auto quad = [&](const int q, const uint4& cur, uint4& next) {
                    // (geometric stream: T_p = 0, no node word draws a perturbation)
                    uint32_t vq = 0u;
                    if (!GEO)
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %1, %2;\n\tvote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}"
                            : "=r"(vq)
                            : "r"(min(min(cur.x, cur.y), min(cur.z, cur.w))), "r"(Tp));
                    thresholds(q, e);
#if defined(PBN_BS_SKIP_PHILOX)
                    next = make_uint4(cur.y * 3u + (uint32_t)q, cur.z ^ cur.x, cur.w + cur.y, cur.x * 5u);
#else
                    next = philox_quad_ps(lds128_state(pqt + 16u * (uint32_t)(q + 1 - qlo)), ps, P.rk);
#endif
                    planes(q, cur, e);
                    if (!GEO)
                        asm("{\n\t.reg .u32 f;\n\tmin.u32 f, %1, 1;\n\tmad.lo.u32 %0, %0, 2, f;\n\t}" : "+r"(gpend) : "r"(vq));
                };
                // two quads per iteration with the Philox words alternating
                // between rw and rn: no register rotation moves
                int q = qc;
                uint4 rn;
                for (; q + 1 < qe; q += 2) {
                    quad(q, rw, rn);
                    quad(q + 1, rn, rw);
                }
                if (q < qe) {
                    quad(q, rw, rn);
                    rw = rn;
                }
                // flagged quads: their gamma words (A4)
                while (gpend) {
                    const int jb = __ffs((int)gpend) - 1;
                    gpend &= gpend - 1;
                    const int qq = qe - 1 - jb;
                    gammas(qq, philox_quad_ps(lds128_state(pqt + 16u * (uint32_t)(qq - qlo)), ps, P.rk));
                }
            }
            if (qf < q1) {  // ragged last quad: padding nodes draw no perturbation
                const int q = qf;
                const uint32_t nv = (uint32_t)(n - 4 * q);  // 1..3 real nodes
                const uint4 rq = make_uint4(rw.x, nv > 1 ? rw.y : FULL, nv > 2 ? rw.z : FULL, FULL);
                thresholds(q, e);
                planes(q, rq, e);
                if (!GEO) gammas(q, rq);
            }
            if (GEO && wg == W - 1) {
                // the geometric-skip stream (reading Q18): this warp clears the
                // buffer's gamma vectors, then every lane draws its chain's
                // gamma(t) by skips over Cg and ORs its bit into the gamma
                // words (node k's at sel + 16 PV (k >> 2) + 16 NP + 4 (k & 3))
                for (int q = lane; q < qhi - qlo; q += 32)
                    sts128_if(sel + 16u * (uint32_t)PV * (uint32_t)q + 16u * NP, 0u, 0u, 0u, 0u, FULL);
                __syncwarp();
                Img<false> gi;
                gi.gbase = reinterpret_cast<const uint8_t*>(B.geo_table);
                any = geometric_gamma_at(
                    gi, 0u, n, P.geo_inv_lnq, chain, t_lo, t_hi, P.rk,
                    [&](uint32_t kk) {
                        // (cluster: another rank's node -> the dummy word)
                        const int kq = (int)(kk >> 2);
                        return (kq >= qlo && kq < qhi)
                                   ? sel + 16u * (uint32_t)PV * (uint32_t)(kq - qlo) + 16u * NP + 4u * (kk & 3u)
                                   : cany + 128u;
                    },
                    lmask, valid);
            }
            if (!PER_NODE && leader) sts32(anyw0 + 128u * (uint32_t)(k & 1) + 4u * wg, any);
        };

        // ---- phase B of unit step k: S_k (buffer nb) from S_{k-1} (ob) and planes[k & 1] ----
        auto phaseB = [&](const int64_t k, const uint32_t ob, const uint32_t nb) {
            const uint32_t selq = sel0 + (uint32_t)(k & 1) * (uint32_t)B.sel_bytes - 16u * (uint32_t)PV * (uint32_t)qlo;
            const uint32_t gob = gbase + ob, gnb = gbase + nb;
            uint32_t M = 0;
            if (!PER_NODE) {
                if (CLU)  // the ranks' any words (exchanged before this interval)
                    M = __reduce_or_sync(FULL, lane < KC ? lds32(cany + 64u * (uint32_t)(k & 1) + 4u * lane) : 0u) & vmask;
                else
                    M = __reduce_or_sync(FULL, lane < W ? lds32(anyw0 + 128u * (uint32_t)(k & 1) + 4u * lane) : 0u) &
                        vmask;
            }
            uint32_t p = rl;
            auto run_class = [&](auto cc) {
                constexpr int C = decltype(cc)::value;
                for (;;) {
                    const uint32_t tb = lds32(p);
                    p += 4u;
                    if (tb == kListEnd) break;
                    bs_round<C, MODE, L, SMEM>(img, tb + (uint32_t)lane * bs_stride(C), gob, gnb, selq, M);
                }
            };
            // classes 7 and 8 only in the CMAX = 8 kernels: their trees'
            // registers would otherwise spill the theta <= 6 kernels
            if constexpr (CMAX >= 8) run_class(std::integral_constant<int, 8>{});
            if constexpr (CMAX >= 7) run_class(std::integral_constant<int, 7>{});
            run_class(std::integral_constant<int, 6>{});
            run_class(std::integral_constant<int, 5>{});
            run_class(std::integral_constant<int, 4>{});
            run_class(std::integral_constant<int, 3>{});
            run_class(std::integral_constant<int, 2>{});
            run_class(std::integral_constant<int, 1>{});
        };

        // statistics of unit step k (S_k in the buffer at byte offset buf), statistics warps
        auto record = [&](const int64_t k, const uint32_t buf) {
            const int64_t r = r_begin - 1 + k;
            if (stats && r > P.burn_in) {
                const uint32_t b = ChainStats::indicator(
                    P, prop, lane, [&](uint32_t i) { return gbase + state_off(i, QS) + buf; });
                cs.record(P, b, r - P.burn_in - 1, valid, orow());
            }
        };

        // (PBN_BS_SKIP_A / PBN_BS_SKIP_B: timing-only builds that drop one
        // phase -- wrong outputs, used to split the step time between them)
#if defined(PBN_BS_SKIP_A)
        constexpr bool kA = false;
#else
        constexpr bool kA = true;
#endif
#if defined(PBN_BS_SKIP_B)
        constexpr bool kB = false;
#else
        constexpr bool kB = true;
#endif
        // cluster: this CTA's words of S_k (buffer nb) and its any word of step
        // k + 1 into every peer (DSMEM), then one cluster barrier (release /
        // acquire): the next interval reads a complete S_k and M everywhere
        auto exchange = [&](const int64_t k, const uint32_t nb) {
            if constexpr (CLU) {
                const uint32_t nq_own = (uint32_t)(qhi - qlo);
                for (uint32_t x = tid; x < nq_own * (uint32_t)KC; x += blockDim.x) {
                    const uint32_t peer = x / nq_own, q = (uint32_t)qlo + x % nq_own;
                    if (peer == rank) continue;
                    const uint32_t a = gbase + QS * q + nb;
                    const uint4 v = lds128_state(a);
                    uint32_t ra;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(peer));
                    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(ra), "r"(v.x), "r"(v.y),
                                 "r"(v.z), "r"(v.w)
                                 : "memory");
                }
                if (!PER_NODE && wg == 0 && k + 1 <= K) {
                    const uint32_t ca =
                        __reduce_or_sync(FULL, lane < W ? lds32(anyw0 + 128u * (uint32_t)((k + 1) & 1) + 4u * lane) : 0u);
                    if (lane < KC) {
                        uint32_t ra;
                        const uint32_t a = cany + 64u * (uint32_t)((k + 1) & 1) + 4u * rank;
                        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(lane));
                        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(ca) : "memory");
                    }
                }
                asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                                 "memory");
            }
        };
        __syncthreads();  // the unit's S_0 is complete; the previous unit is done with the buffers
        if (K >= 1) phaseA(1, 16u);
        __syncthreads();
        exchange(0, 0u);  // (S_0 is complete in every CTA; this carries any(1))
        // one interval per step k: statistics of k-1, phase B of k and phase A
        // of k+1; buffers ob = S_{k-1}, nb = S_k, zb = S_{k+1} rotate (uniform)
        uint32_t ob = 0u, nb = 16u, zb = 32u;
        for (int64_t k = 1; k <= K; ++k) {
            if (k > 1) record(k - 1, ob);
            if (a_first) {
                if (kA && k < K) phaseA(k + 1, zb);
                if (kB) phaseB(k, ob, nb);
            } else {
                if (kB) phaseB(k, ob, nb);
                if (kA && k < K) phaseA(k + 1, zb);
            }
            __syncthreads();
            exchange(k, nb);
            const uint32_t t3 = ob;
            ob = nb;
            nb = zb;
            zb = t3;
        }
        const uint32_t cur = ob;  // S_K's buffer (K >= 1), buffer 0 for K = 0
        if (K >= 1) record(K, cur);

        if (!last_chunk) {
            __syncthreads();
            for (int i = tid; i < n; i += blockDim.x) __stcg(scr() + i, lds32(gbase + state_off(i, QS) + cur));
            if (stats) {
                uint32_t* st = scr() + P.n_pad + 8 * 32 * prop + 8 * lane;
                __stcg(st + 0, cs.c1);
                __stcg(st + 1, cs.n01);
                __stcg(st + 2, cs.n10);
                __stcg(st + 3, cs.first);
                __stcg(st + 4, cs.prev);
                __stcg(st + 5, cs.bacc);
                __stcg(st + 6, cs.bitw);
                __stcg(st + 7, cs.bcount);
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.done + group), "r"((uint32_t)(chunk + 1))
                             : "memory");
            }
            continue;
        }
        for (int b = b0; b < b1; ++b) {
            uint32_t v = 0;
            for (int k = 0; k < 32; ++k) {
                const int i = 32 * b + k;
                if (i >= n) break;
                v |= ((lds32(gbase + state_off(i, QS) + cur) >> lane) & 1u) << k;
            }
            if (valid && rank == 0) P.state[(int64_t)chain_local * nsw + b] = v;
        }
        if (stats) cs.finish(P, prop, valid, orow(), leader);
    }
}

template <int MODE, int IMG, int CMAX, int TB>
const void* pick_L(int L)
{
    switch (L) {
        case 1: return reinterpret_cast<const void*>(&bitslice_kernel<MODE, 1, IMG, CMAX, TB>);
        case 2: return reinterpret_cast<const void*>(&bitslice_kernel<MODE, 2, IMG, CMAX, TB>);
        case 3: return reinterpret_cast<const void*>(&bitslice_kernel<MODE, 3, IMG, CMAX, TB>);
        default: return reinterpret_cast<const void*>(&bitslice_kernel<MODE, 4, IMG, CMAX, TB>);
    }
}

// img: 0 global image, 1 staged, 2 staged sub-image of a cluster; threads: the
// launch's block size (the staged kernels have a 640-thread build)
template <int MODE>
const void* pick_mode(int L, int img, int cmax, int threads)
{
    if (img != 0 && threads <= kBitsliceSmallThreads) {
        if (img == 2) return cmax <= 6 ? pick_L<MODE, 2, 6, kBitsliceSmallThreads>(L) : pick_L<MODE, 2, 8, kBitsliceSmallThreads>(L);
        return cmax <= 6 ? pick_L<MODE, 1, 6, kBitsliceSmallThreads>(L) : pick_L<MODE, 1, 8, kBitsliceSmallThreads>(L);
    }
    if (img == 2) return cmax <= 6 ? pick_L<MODE, 2, 6, PBN_BS_THREADS>(L) : pick_L<MODE, 2, 8, PBN_BS_THREADS>(L);
    if (img == 1) return cmax <= 6 ? pick_L<MODE, 1, 6, PBN_BS_THREADS>(L) : pick_L<MODE, 1, 8, PBN_BS_THREADS>(L);
    return cmax <= 6 ? pick_L<MODE, 0, 6, PBN_BS_THREADS>(L) : pick_L<MODE, 0, 8, PBN_BS_THREADS>(L);
}

}  // namespace
}  // namespace pbn
