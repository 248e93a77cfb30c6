// pbn_bitslice.cu -- K1b: the fused PBN trajectory kernel with BIT-SLICED
// function evaluation (sm_100a).
//
// The same hot path as K1 (§2.2) on
// the same group layout -- one 32-chain group per CTA, its state bit-sliced
// in shared memory (word i = node i of the 32 chains, bit l = chain of lane
// l; here THREE interleaved buffers, pbn_internal.h) -- but the node step is
// split in two phases so that the truth-table work is done once per 32
// chains instead of once per chain:
//
//   phase A (lane = chain; every warp its quads of nodes, as K1):
//     one Philox4x32-10 call per quad (A3, reading Q2); per node the
//     selection planes s_m = ballot(u > E_m), m = 1..L-1 (A5: chain l picks
//     function j = #{m : u_l > E_m}, so bit l of s_j & ~s_{j+1} is set iff
//     chain l picks j); one vote per quad flags the ~1 % of quads where some
//     chain drew u < T_p, whose gamma words (A4) are formed after the quad
//     loop; per quad the planes and gamma words go to L 16-byte vectors, and
//     the warp zeroes its quads' words of the step's state buffer.
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
// phase B of step t (even warps A first, odd warps B first, so the pipes see
// both instruction mixes at once): one CTA barrier per step; the planes and
// any words are double-buffered by step parity and the state triple-buffered
// (B(t) reads S_{t-1}, ORs into S_t; A(t+1) zeroes S_{t+1}'s buffer; the
// statistics warp reads S_t in the next interval).
//
// Per node-update the work is one quarter of a Philox call, L-1 compare +
// ballot pairs and ~1/32 of the task's gather and tree instead
// of K1's per-chain gather of FT padded parents and per-chain descriptor
// reads.  Every output is bit-identical to K1's (the same stream,
// thresholds, tables and statistics).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "pbn_internal.h"
#include "pbn_node.cuh"

namespace pbn {
namespace {

// 16-byte shared load ordered with the barriers (the per-quad Philox table
// is refilled when t_hi changes)
__device__ __forceinline__ uint4 lds128_state(uint32_t a)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// table entry E as a word mask (all ones iff the entry is 1)
template <int E>
__device__ __forceinline__ uint32_t entry_mask(uint32_t t0, uint32_t t1)
{
    const uint32_t w = E < 32 ? t0 : t1;
    return (uint32_t)((int32_t)(w << (31 - (E & 31))) >> 31);
}

// multiplexer tree: the sub-table of entries [B, B + 2^(C-K)) evaluated on
// the parent words x[K..C-1] (x[0] = parents[0] = the index MSB, reading Q5):
// x[K] = 0 selects the lower half, 1 the upper -- bit l of the result is the
// entry at chain l's index
template <int K, int C, int B>
__device__ __forceinline__ uint32_t mux_tree(uint32_t t0, uint32_t t1, const uint32_t (&x)[C])
{
    if constexpr (K == C) {
        return entry_mask<B>(t0, t1);
    } else {
        constexpr int H = 1 << (C - K - 1);
        const uint32_t lo = mux_tree<K + 1, C, B>(t0, t1, x);
        const uint32_t hi = mux_tree<K + 1, C, B + H>(t0, t1, x);
        return (x[K] & hi) | (~x[K] & lo);
    }
}

// one round of 32 tasks of class C (theta = C parents), lane = task.  The
// node's plane words are at pl + 16 m (m = 0..L-2: s_{m+1}; m = L-1:
// gamma); `cw` holds the constant words FULL (cw) and ZERO (cw + 4) that
// stand in for s_0 and s_L, so every load is unconditional.
template <int C, int MODE, int L, uint32_t OB, uint32_t NB>
__device__ __forceinline__ void bs_round(uint32_t ta, uint32_t gbase, uint32_t sel, uint32_t cw, uint32_t M)
{
    uint32_t t0, t1 = 0, w0, w1, w2, w3 = 0;
    if constexpr (C <= 5) {
        const uint4 r = lds128_ro(ta);
        t0 = r.x;
        w0 = r.y;
        w1 = r.z;
        w2 = r.w;
    } else {
        const uint4 r = lds128_ro(ta);
        const uint2 r2 = lds64_ro(ta + 16u);
        t0 = r.x;
        t1 = r.y;
        w0 = r.z;
        w1 = r.w;
        w2 = r2.x;
        w3 = r2.y;
    }
    const uint32_t pw[6] = {w0 >> 16, w1 & 0xFFFFu, w1 >> 16, w2 & 0xFFFFu, w2 >> 16, w3 & 0xFFFFu};
    uint32_t x[C];
#pragma unroll
    for (int m = 0; m < C; ++m) x[m] = lds32_state(gbase + pw[m] + OB);
    const uint32_t F = mux_tree<0, C, 0>(t0, t1, x);
    const uint32_t i = (w0 & 0xFFFFu) >> 2, j = w0 & 3u;
    const uint32_t pl = sel + 16u * (uint32_t)L * (i >> 2) + 4u * (i & 3u);
    // selection plane of function j: s_j & ~s_{j+1} (s_0 = all chains, s_L = none)
    const uint32_t s_lo = lds32_state(j == 0 ? cw : pl + 16u * (j - 1u));
    const uint32_t s_hi = lds32_state(j == (uint32_t)(L - 1) ? cw + 4u : pl + 16u * j);
    const uint32_t gam = lds32_state(pl + 16u * (uint32_t)(L - 1));
    const uint32_t out = gbase + state_off(i, kBitsliceQs);
    const uint32_t old = lds32_state(out + OB);
    const uint32_t first = j == 0 ? FULL : 0u;  // function 0 carries the perturbation term
    uint32_t c;
    if (MODE == 1) {  // PER_NODE: chains with gamma_i take NOT s_i
        c = (F & s_lo & ~s_hi & ~gam) | (~old & gam & first);
    } else {          // VECTOR: chains with any gamma take s XOR gamma
        c = (F & s_lo & ~s_hi & ~M) | ((old ^ gam) & M & first);
    }
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p red.shared.or.b32 [%0], %1;\n\t}" ::"r"(out + NB),
                 "r"(c)
                 : "memory");
}

// MODE: 0 VECTOR, 1 PER_NODE; L = the model's largest ell (planes s_1..s_{L-1})
template <int MODE, int L>
__global__ void __launch_bounds__(PBN_BS_THREADS, 1) bitslice_kernel(const __grid_constant__ BitsliceParams B)
{
    const TrajParams& P = B.T;
    constexpr bool PER_NODE = MODE == 1;
    constexpr uint32_t QS = kBitsliceQs;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t mbar;

    const int tid = threadIdx.x;
    const int wg = tid >> 5;
    const int lane = tid & 31;
    const int W = P.warps_per_group;
    const int n = P.n;
    const uint32_t gbase = smem_u32(smem);
    const uint32_t sbase = gbase + 4u * (uint32_t)P.group_words;  // image base

    // ---- A1: stage the image into shared memory (bulk async copy) ----
    {
        const uint32_t bar = smem_u32(&mbar);
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(P.image_smem_bytes)
                         : "memory");
            const uint32_t chunk = 32768;
            for (uint32_t off = 0; off < P.image_smem_bytes; off += chunk) {
                const uint32_t sz = min(chunk, P.image_smem_bytes - off);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sbase + off),
                    "l"(P.image + off), "r"(sz), "r"(bar)
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

    const bool leader = lane == 0;
    const uint32_t lead = leader ? FULL : 0u;
    const uint32_t anyw0 = gbase + (uint32_t)B.any_off;  // any[2][32]
    const uint32_t cw = anyw0 + 256u;                    // constant words FULL, ZERO
    const uint32_t sel0 = gbase + (uint32_t)B.sel_off;   // planes[2]
    const uint32_t pqt = gbase + (uint32_t)B.pq_off;     // per-quad Philox table
    const uint32_t erec = sbase + B.erec_off;
    const uint32_t rounds = sbase + B.rounds_off;
    const int R = B.n_rounds;
    if (tid == 0) {
        sts32(cw, FULL);
        sts32(cw + 4u, 0u);
    }

    const int NW = P.node_warps;
    const int q0 = wg < NW ? (int)((int64_t)wg * P.nquads / NW) : P.nquads;
    const int q1 = wg < NW ? (int)((int64_t)(wg + 1) * P.nquads / NW) : P.nquads;
    const int nsw = P.state_words;
    const int b0 = (int)((int64_t)wg * nsw / W), b1 = (int)((int64_t)(wg + 1) * nsw / W);
    const int64_t total = P.burn_in + P.steps;
    const uint32_t Tp = P.Tp;
    const bool full_quads = (n & 3) == 0 || q1 < P.nquads;
    const bool a_first = (wg & 1) == 0;  // even warps: A(t+1) then B(t); odd: B(t) then A(t+1)
    __shared__ unsigned long long s_unit;

    for (int64_t it = 0;; ++it) {
        int64_t group, chunk, r_begin, r_end;
        if (!P.persistent) {
            if (it > 0) break;
            group = blockIdx.x;
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
        const bool stats = prop >= 0 && prop < P.n_props;
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
            for (int q = q0; q < q1; ++q) {
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

        // ---- phase A of unit step k: planes -> planes[k & 1], zero S_k's buffer ZB ----
        auto phaseA = [&](const int64_t k, auto zb_c) {
            constexpr uint32_t ZB = decltype(zb_c)::value;
            const uint64_t t = (uint64_t)(P.step0 + r_begin - 1 + k);
            const uint32_t t_lo = (uint32_t)t, t_hi = (uint32_t)(t >> 32);
            const uint32_t sel = sel0 + (uint32_t)(k & 1) * (uint32_t)B.sel_bytes;
            uint32_t any = 0;
            const PhiloxStep ps = philox_step(chain, t_lo, t_hi, P.rk);
            const int qf = (full_quads || q1 == q0) ? q1 : q1 - 1;
            // quad q's record: L vectors of 16 bytes at sel + 16 L q -- the planes
            // s_1..s_{L-1} of its 4 nodes, then their gamma words
            auto thresholds = [&](const int q, uint4 (&e)[3]) {
                const uint32_t ea = erec + 16u * (uint32_t)(L - 1) * (uint32_t)q;
#pragma unroll
                for (int m = 0; m < L - 1; ++m) e[m] = lds128_ro(ea + 16u * m);
            };
            auto planes = [&](const int q, const uint4 rw, const uint4 (&e)[3]) {
                const uint32_t pa = sel + 16u * (uint32_t)L * (uint32_t)q;
                uint4 s[3];
#pragma unroll
                for (int m = 0; m < L - 1; ++m)
#if defined(PBN_BS_SKIP_PLANES)
                    s[m] = make_uint4(rw.x ^ e[m].x, rw.y ^ e[m].y, rw.z ^ e[m].z, rw.w ^ e[m].w);
#else
                    s[m] = make_uint4(__ballot_sync(FULL, rw.x > e[m].x), __ballot_sync(FULL, rw.y > e[m].y),
                                      __ballot_sync(FULL, rw.z > e[m].z), __ballot_sync(FULL, rw.w > e[m].w));
#endif
#pragma unroll
                for (int m = 0; m < L - 1; ++m) sts128_if(pa + 16u * m, s[m].x, s[m].y, s[m].z, s[m].w, lead);
                sts128_if(pa + 16u * (L - 1), 0u, 0u, 0u, 0u, lead);              // gamma (flagged quads: below)
                sts128_if(gbase + QS * (uint32_t)q + ZB, 0u, 0u, 0u, 0u, lead);  // S_k's words, OR-ed in phase B
            };
            auto gammas = [&](const int q, const uint4 rq) {
                const uint32_t g0 = __ballot_sync(FULL, rq.x < Tp), g1 = __ballot_sync(FULL, rq.y < Tp);
                const uint32_t g2 = __ballot_sync(FULL, rq.z < Tp), g3 = __ballot_sync(FULL, rq.w < Tp);
                any |= g0 | g1 | g2 | g3;
                sts128_if(sel + 16u * (uint32_t)L * (uint32_t)q + 16u * (L - 1), g0, g1, g2, g3, lead);
            };
            uint4 rw = philox_quad_pc(lds128_state(pqt + 16u * (uint32_t)q0), ps, P.rk);
            uint4 e[3];
            for (int qc = q0; qc < qf; qc += 32) {
                const int qe = min(qf, qc + 32);
                uint32_t gpend = 0;  // flags of the chunk's quads, newest = bit 0
                // one quad: the flag vote first -- the quad's thresholds, the
                // next quad's Philox call and the plane ballots follow it in
                // one basic block, so the scheduler overlaps the loads' latency
                // and the Philox chain with the ballots
                auto quad = [&](const int q, const uint4& cur, uint4& next) {
                    const uint32_t vq = __ballot_sync(FULL, min(min(cur.x, cur.y), min(cur.z, cur.w)) < Tp);
                    thresholds(q, e);
#if defined(PBN_BS_SKIP_PHILOX)
                    next = make_uint4(cur.y * 3u + (uint32_t)q, cur.z ^ cur.x, cur.w + cur.y, cur.x * 5u);
#else
                    next = philox_quad_pc(lds128_state(pqt + 16u * (uint32_t)(q + 1)), ps, P.rk);
#endif
                    planes(q, cur, e);
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
                    gammas(qq, philox_quad_pc(lds128_state(pqt + 16u * (uint32_t)qq), ps, P.rk));
                }
            }
            if (qf < q1) {  // ragged last quad: padding nodes draw no perturbation
                const int q = qf;
                const uint32_t nv = (uint32_t)(n - 4 * q);  // 1..3 real nodes
                const uint4 rq = make_uint4(rw.x, nv > 1 ? rw.y : FULL, nv > 2 ? rw.z : FULL, FULL);
                thresholds(q, e);
                planes(q, rq, e);
                gammas(q, rq);
            }
            if (!PER_NODE && leader) sts32(anyw0 + 128u * (uint32_t)(k & 1) + 4u * wg, any);
        };

        // ---- phase B of unit step k: S_k (buffer NB) from S_{k-1} (OB) and planes[k & 1] ----
        auto phaseB = [&](const int64_t k, auto ob_c, auto nb_c) {
            constexpr uint32_t OB = decltype(ob_c)::value;
            constexpr uint32_t NB = decltype(nb_c)::value;
            const uint32_t sel = sel0 + (uint32_t)(k & 1) * (uint32_t)B.sel_bytes;
            uint32_t M = 0;
            if (!PER_NODE)
                M = __reduce_or_sync(FULL, lane < W ? lds32(anyw0 + 128u * (uint32_t)(k & 1) + 4u * lane) : 0u) & vmask;
            for (int m = 0; m * W < R; ++m) {
                const int rr_i = (m & 1) ? (m + 1) * W - 1 - wg : m * W + wg;
                if (rr_i >= R) continue;
                const uint2 rr = lds64_ro(rounds + 8u * (uint32_t)rr_i);
                const uint32_t ta = sbase + rr.x + (uint32_t)lane * (rr.y == 6u ? 32u : 16u);
                switch (rr.y) {
                    case 1: bs_round<1, MODE, L, OB, NB>(ta, gbase, sel, cw, M); break;
                    case 2: bs_round<2, MODE, L, OB, NB>(ta, gbase, sel, cw, M); break;
                    case 3: bs_round<3, MODE, L, OB, NB>(ta, gbase, sel, cw, M); break;
                    case 4: bs_round<4, MODE, L, OB, NB>(ta, gbase, sel, cw, M); break;
                    case 5: bs_round<5, MODE, L, OB, NB>(ta, gbase, sel, cw, M); break;
                    default: bs_round<6, MODE, L, OB, NB>(ta, gbase, sel, cw, M); break;
                }
            }
        };

        // statistics of unit step k (S_k in buffer BUF), statistics warps
        auto record = [&](const int64_t k, const uint32_t buf) {
            const int64_t r = r_begin - 1 + k;
            if (stats && r > P.burn_in) {
                const uint32_t b = ChainStats::indicator(
                    P, prop, lane, [&](uint32_t i) { return gbase + state_off(i, QS) + buf; });
                cs.record(P, b, r - P.burn_in - 1, valid, orow());
            }
        };

        // one interval: statistics of k-1, phase B of k and phase A of k+1
        // the per-quad Philox table for t_hi of unit step k (all threads;
        // the caller brackets it with barriers)
        uint32_t table_thi = 0;
        auto fill_table = [&](const int64_t k) {
            table_thi = (uint32_t)((uint64_t)(P.step0 + r_begin - 1 + k) >> 32);
            for (int q = tid; q <= P.nquads; q += blockDim.x) {
                const uint4 c = philox_quad_consts((uint32_t)q, table_thi, P.rk);
                sts128_if(pqt + 16u * (uint32_t)q, c.x, c.y, c.z, c.w, FULL);
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
        auto interval = [&](const int64_t k, auto ob_c, auto nb_c, auto zb_c) {
            // t_hi of step k + 1 changed (every 2^32 steps): refill the table
            // first (uniform over the CTA; nobody reads it until phase A)
            if (k < K && (uint32_t)((uint64_t)(P.step0 + r_begin + k) >> 32) != table_thi) {
                fill_table(k + 1);
                __syncthreads();
            }
            if (k > 1) record(k - 1, decltype(ob_c)::value);
            if (a_first) {
                if (kA && k < K) phaseA(k + 1, zb_c);
                if (kB) phaseB(k, ob_c, nb_c);
            } else {
                if (kB) phaseB(k, ob_c, nb_c);
                if (kA && k < K) phaseA(k + 1, zb_c);
            }
            __syncthreads();
        };
        using C0 = std::integral_constant<uint32_t, 0u>;
        using C1 = std::integral_constant<uint32_t, 16u>;
        using C2 = std::integral_constant<uint32_t, 32u>;
        __syncthreads();  // the previous unit's phase A is done with the table
        fill_table(1);
        __syncthreads();
        if (K >= 1) phaseA(1, C1());
        __syncthreads();
        for (int64_t k = 1; k <= K; k += 3) {
            interval(k, C0(), C1(), C2());
            if (k + 1 <= K) interval(k + 1, C1(), C2(), C0());
            if (k + 2 <= K) interval(k + 2, C2(), C0(), C1());
        }
        const uint32_t cur = 16u * (uint32_t)(K % 3);  // S_K's buffer
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
            if (valid) P.state[(int64_t)chain_local * nsw + b] = v;
        }
        if (stats) cs.finish(P, prop, valid, orow(), leader);
    }
}

template <int MODE>
const void* pick_L(int L)
{
    switch (L) {
        case 1: return reinterpret_cast<const void*>(&bitslice_kernel<MODE, 1>);
        case 2: return reinterpret_cast<const void*>(&bitslice_kernel<MODE, 2>);
        case 3: return reinterpret_cast<const void*>(&bitslice_kernel<MODE, 3>);
        default: return reinterpret_cast<const void*>(&bitslice_kernel<MODE, 4>);
    }
}

}  // namespace

const void* pick_bitslice_kernel(int mode, int L) { return mode == 1 ? pick_L<1>(L) : pick_L<0>(L); }

}  // namespace pbn
