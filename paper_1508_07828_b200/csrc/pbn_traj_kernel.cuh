// pbn_traj_kernel.cuh -- K1: fused PBN trajectory kernel for sm_100a (the
// kernel template; instantiated per MODE in pbn_traj_m{0,1,2}.cu so the
// three semantics compile in parallel, launched from pbn_traj.cu).
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

#pragma once
#include "pbn_internal.h"
#include "pbn_node.cuh"

namespace pbn {
namespace {

// Thread budget of the global-image kernels (image through L1/L2, 64-bit
// image addresses): 896 threads = 28 warps at 72 registers, no spills in the
// quad loop (C5, 16384 chains: 3.13e11 vs 2.88e11 node-updates/s with 32 warps
// at 64 registers and local-memory reloads in the loop; 24 warps: 2.90e11)
#ifndef PBN_GLOBAL_THREADS
#define PBN_GLOBAL_THREADS 896
#endif
constexpr int kGlobalImageThreads = PBN_GLOBAL_THREADS < PBN_MAX_THREADS ? PBN_GLOBAL_THREADS : PBN_MAX_THREADS;

// MODE: 0 VECTOR, 1 PER_NODE, 2 VECTOR with the geometric-skip stream (a
// template parameter: the draw code in the step loop cost the other modes
// 0.5 % on C4 as a runtime branch)
template <bool SMEM, int MODE, int FT, bool SLOW>
__global__ void __launch_bounds__(SMEM ? PBN_MAX_THREADS : kGlobalImageThreads, 1)
    traj_kernel(const __grid_constant__ TrajParams P)
{
    constexpr bool PER_NODE = MODE == 1;
    constexpr bool GEO = MODE == 2;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t mbar;

    const int tid = threadIdx.x;
    const int wg = tid >> 5;  // warp within the (single) group of this CTA
    const int lane = tid & 31;
    const int W = P.warps_per_group;
    const int n = P.n;
    // dynamic shared memory: [group state | gamma words | any words] then the
    // staged image (16-aligned) -- the state sits at the window's dynamic base
    // state base; the global-image kernels add it to every parent offset, so
    // it is made a uniform value (redux: UR) and the adds fold into the LDS
    // address ([R + UR]) -- from the symbol, ptxas rematerialises it per use
    const uint32_t gbase = SMEM ? smem_u32(smem) : __reduce_or_sync(FULL, smem_u32(smem));
    const uint32_t sbase = gbase + 4u * (uint32_t)P.group_words;  // image base

    // ---- A1: stage the model image into shared memory (bulk async copy) ----
    Img<SMEM> img;
    img.gbase = P.image;
    if (SMEM) {
        const uint32_t bar = smem_u32(&mbar);
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                         "r"(P.image_smem_bytes)
                         : "memory");
            const uint32_t chunk = 32768;
            for (uint32_t off = 0; off < P.image_smem_bytes; off += chunk) {
                const uint32_t sz = min(chunk, P.image_smem_bytes - off);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
                    "[%3];" ::"r"(sbase + off),
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
        // relocate: offsets -> absolute shared addresses of this CTA's copy
        const uint32_t* rel = reinterpret_cast<const uint32_t*>(P.image + P.L.reloc_off);
        const uint32_t state_base = gbase;
        for (int k = tid; k < P.L.reloc_count; k += blockDim.x) {
            const uint32_t e = __ldg(rel + k);
            const uint32_t a = sbase + (e & ~kRelocState);
            sts32(a, lds32(a) + ((e & kRelocState) ? state_base : sbase));
        }
        __syncthreads();
    }

    const bool leader = lane == 0;
    const uint32_t lead = leader ? FULL : 0u;        // store predicate as a word
    const uint32_t rot = 31u - (uint32_t)lane;       // rotate-left amount: bit `lane` -> bit 31
    const uint32_t lmask = 1u << lane;               // this chain's bit in a state word

    const uint32_t gam = gbase + 8u * P.n_pad;   // VECTOR: gamma words
    const uint32_t anyw = gbase + 4u * (PER_NODE ? 2 : 3) * P.n_pad;  // [W]
    const uint32_t nrec = SMEM ? sbase : 0u;     // node records start the image

    const int NW = P.node_warps;  // warps >= NW own no quads (statistics only)
    const int q0 = wg < NW ? (int)((int64_t)wg * P.nquads / NW) : P.nquads;
    const int q1 = wg < NW ? (int)((int64_t)(wg + 1) * P.nquads / NW) : P.nquads;
    const int nsw = P.state_words;
    const int b0 = (int)((int64_t)wg * nsw / W), b1 = (int)((int64_t)(wg + 1) * nsw / W);

    if (!PER_NODE)  // the gamma buffer is all-zero between steps (the fixup clears it)
        for (int i = tid; i < P.n_pad; i += blockDim.x) sts32(gam + 4u * i, 0u);

    const int64_t total = P.burn_in + P.steps;
    const uint32_t Tp = P.Tp;
    const bool full_quads = (n & 3) == 0 || q1 < P.nquads;  // this warp never sees a ragged quad
    __shared__ unsigned long long s_unit;

    // ---- work units: (group, chunk of steps).  Non-persistent launches run one
    // unit per CTA (its group, all steps); persistent launches pull units from a
    // queue, chunk c of group g after chunk c-1 (flag done[g]), and carry the
    // group's bit-sliced state and per-lane counters across chunks in scratch.
    for (int64_t it = 0;; ++it) {
        int64_t group, chunk, r_begin, r_end;
        if (!P.persistent) {
            if (it > 0) break;
            group = blockIdx.x;
            chunk = 0;
            r_begin = 1;
            r_end = total;
        } else {
            __syncthreads();  // s_unit free for reuse
            if (tid == 0) s_unit = atomicAdd(P.work_ctr, 1ull);
            __syncthreads();
            // redux makes the unit index a uniform value (UR), so the loop stays
            // warp-uniform and the buffer bases stay in uniform registers
            const unsigned long long u = __reduce_max_sync(FULL, (uint32_t)s_unit);
            if (u >= (unsigned long long)P.total_units) break;
            group = (int64_t)(u % (unsigned long long)P.n_groups);
            chunk = (int64_t)(u / (unsigned long long)P.n_groups);
            r_begin = chunk * P.chunk_steps + 1;
            r_end = min(total, (chunk + 1) * P.chunk_steps);
            if (chunk > 0 && tid == 0) {
                // wait for chunk c-1 of this group (acquire)
                for (;;) {
                    unsigned int d;
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(P.done + group) : "memory");
                    if ((int64_t)d >= chunk) break;
                    __nanosleep(256);
                }
            }
        }
#if defined(PBN_GZ_START)
        // a previous unit of this CTA (e.g. a ragged group, whose lanes
        // without a chain may draw perturbations that never trigger the
        // fix-up) can leave gamma bits behind: clear them per unit
        if (!PER_NODE && P.persistent && it > 0)
            for (int i = tid; i < P.n_pad; i += blockDim.x) sts32(gam + 4u * i, 0u);
#endif
        const bool first_chunk = chunk == 0;
        const bool last_chunk = r_end >= total;
        // (kept in 32 bits: few live registers across the step loop -- the
        // global-image kernel spilled with 64-bit row indices)
        const uint32_t chain_local = (uint32_t)group * 32u + (uint32_t)lane;
        const bool valid = (int64_t)chain_local < P.n_chains;
        const uint32_t chain = (uint32_t)(P.chain_base + chain_local);
        const uint32_t vmask = __ballot_sync(FULL, valid);  // lanes holding real chains
        // state buffers: word (i, b) at gbase + state_off(i) + 16 b; every
        // chunk starts from buffer 0, `cur` tracks the newest buffer
        uint32_t cur = 0;
        auto scr = [&]() { return P.scratch + group * (int64_t)P.scratch_stride; };  // persistent only
        // statistics warp: warp p < n_props owns property p (A8-A10)
        const int prop = wg - P.stats_warp0;
        const bool stats = prop >= 0 && prop < P.n_props;
        // property-major output row of this lane's chain
        auto orow = [&]() { return (int64_t)prop * P.n_chains + chain_local; };

        // ---- per-lane statistics (statistics warps) ----
        ChainStats cs;

        if (!first_chunk) {
            // resume: bit-sliced state words and warp-0 counters from scratch
            __syncthreads();
            for (int i = tid; i < n; i += blockDim.x) sts32(gbase + state_off(i), __ldcg(scr() + i));
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
            // ---- A2: initial state s_0[i] = u(chain, 0, i) >> 31 ----
            for (int q = q0; q < q1; ++q) {
                const uint4 r = philox4x32_10((uint32_t)q, chain, 0u, 0u, P.rk);
                const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = 4 * q + k;
                    if (i < n) {
                        const uint32_t wv = __ballot_sync(FULL, (rr[k] >> 31) != 0u);
                        if (leader) sts32(gbase + state_off(i), wv);
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
                    if (leader) sts32(gbase + state_off(i), wv);
                }
            }
        }
        __syncthreads();

    // one synchronous step s_{t-1} (buffer OB) -> s_t (buffer NB = 16 - OB);
    // the step loop below is unrolled by two with the buffer roles fixed in
    // each half, so every state access is [R + UR + imm]
    auto step = [&](const int64_t r, auto ob_c) {
        constexpr uint32_t OB = decltype(ob_c)::value;
        constexpr uint32_t NB = 16u - OB;
        const uint64_t t = (uint64_t)(P.step0 + r);
        const uint32_t t_lo = (uint32_t)t, t_hi = (uint32_t)(t >> 32);
        uint32_t any = 0;
        const PhiloxStep ps = philox_step(chain, t_lo, t_hi, P.rk);
        // geometric-skip stream (reading Q18): warp 0 draws every lane's
        // gamma(t) and marks it in the gamma words; the VECTOR fix-up after
        // the step barrier applies it (the node words carry no perturbation)
        if (GEO && wg == 0)
            any |= geometric_gamma(img, (SMEM ? sbase : 0u) + P.geo_off, n, P.geo_inv_lnq, chain, t_lo, t_hi, P.rk,
                                   gam, lmask, valid);
        const int qf = (full_quads || q1 == q0) ? q1 : q1 - 1;  // full quads [q0, qf), ragged after
        // one full quad: four independent nodes, then one 16-byte store commits
        // them (and their gamma words if any)
        // VECTOR gamma words: with the image in shared memory, quads are flagged
        // by one vote and their ballots formed after the loop (lazy, C4 +2 %);
        // with the image read through L1/L2 the per-node ballots are kept
        // (eager: the flag vote's dependence on the Philox words costs there)
        constexpr bool LAZY = SMEM && !PER_NODE;
        constexpr bool GWQ = !LAZY;
        uint32_t gpend = 0;  // VECTOR: flags of the current chunk's quads, bit qe-1-q
        int qc = q0;
        auto quad = [&](const int q, const uint4 rw, const Recs& rc, auto&& between) {
            const uint32_t i0 = 4u * (uint32_t)q;
            // (the quad's perturbation flag is voted first: one convergence
            // point for all the ballots below)
            const uint32_t vq = LAZY ? __ballot_sync(FULL, min(min(rw.x, rw.y), min(rw.z, rw.w)) < Tp) : 0u;
            // the quad's four nodes are independent: compute all, then one
            // 16-byte store commits them (and their gamma words if any)
            uint32_t g0, g1, g2, g3;
            const uint32_t w0 =
                node_word<SMEM, PER_NODE, FT, SLOW, OB, 32, GWQ>(img, rc.r[0], i0, rw.x, Tp, gbase, lmask, rot, g0);
            const uint32_t w1 =
                node_word<SMEM, PER_NODE, FT, SLOW, OB, 32, GWQ>(img, rc.r[1], i0 + 1, rw.y, Tp, gbase, lmask, rot, g1);
            const uint32_t w2 =
                node_word<SMEM, PER_NODE, FT, SLOW, OB, 32, GWQ>(img, rc.r[2], i0 + 2, rw.z, Tp, gbase, lmask, rot, g2);
            const uint32_t w3 =
                node_word<SMEM, PER_NODE, FT, SLOW, OB, 32, GWQ>(img, rc.r[3], i0 + 3, rw.w, Tp, gbase, lmask, rot, g3);
            // the next quad's Philox words: after the votes, in the same basic
            // block as (and interleaved by the scheduler into) this quad's gathers
            between();
            sts128_if(gbase + 32u * (uint32_t)q + NB, w0, w1, w2, w3, lead);
            if (PER_NODE) return;
            if (!LAZY) {
                const uint32_t g = g0 | g1 | g2 | g3;
                any |= g;
                // gamma words only when nonzero (rare); the fixup clears them
                sts128_if(gam + 4u * i0, g0, g1, g2, g3, g & lead);
                return;
            }
            // VECTOR needs the gamma words only of quads where some chain drew a
            // perturbation (p = 1e-4: ~1 % of quads): flag the quad with one
            // vote on the lanes' minimum word; the flagged quads' gamma ballots
            // are formed after the loop (gpend, below)
            gpend = gpend * 2u + min(vq, 1u);  // shift in the quad's flag (newest quad = bit 0)
        };
        // software pipeline: the next quad's Philox words are computed while
        // this quad's nodes gather (independent instruction streams); the
        // quads run in chunks of <= 32 so each chunk's flags fit one word
        uint4 rw = philox_quad((uint32_t)q0, ps, P.rk);
        // (eager kernels: one chunk spanning all the warp's quads)
        for (qc = q0; qc < qf; qc += LAZY ? 32 : qf) {
            const int qe = LAZY ? min(qf, qc + 32) : qf;
            gpend = 0;
            for (int q = qc; q < qe; ++q) {
                uint4 rn;
                quad(q, rw, load_recs(img, nrec + 64u * (uint32_t)q),
                     [&] { rn = philox_quad((uint32_t)(q + 1), ps, P.rk); });
                rw = rn;
            }
            // flagged quads: recompute their words, form and store the gamma ballots
            while (LAZY && gpend) {
                const int j = __ffs((int)gpend) - 1;
                gpend &= gpend - 1;
                const uint32_t q = (uint32_t)(qe - 1 - j);
                const uint4 rq = philox_quad(q, ps, P.rk);
                const uint32_t g0 = __ballot_sync(FULL, rq.x < Tp), g1 = __ballot_sync(FULL, rq.y < Tp);
                const uint32_t g2 = __ballot_sync(FULL, rq.z < Tp), g3 = __ballot_sync(FULL, rq.w < Tp);
                any |= g0 | g1 | g2 | g3;
                sts128_if(gam + 16u * q, g0, g1, g2, g3, lead);
            }
        }
        if (qf < q1) {  // ragged last quad (n % 4 != 0), node by node
            const int q = qf;
            const uint32_t i0 = 4u * (uint32_t)q;
            const uint32_t ra = nrec + 16u * i0;
            const uint32_t rr[4] = {rw.x, rw.y, rw.z, rw.w};
            for (uint32_t k = 0; k < 4 && (int)(i0 + k) < n; ++k) {
                uint32_t gk;
                const uint32_t wk = node_word<SMEM, PER_NODE, FT, SLOW, OB>(img, img.ld128(ra + 16u * k), i0 + k, rr[k], Tp,
                                                                            gbase, lmask, rot, gk);
                sts32_if(gbase + 32u * (uint32_t)q + NB + 4u * k, wk, lead);
                if (!PER_NODE) {
                    any |= gk;
                    sts32_if(gam + 4u * (i0 + k), gk, gk & lead);
                }
            }
        }
        if (!PER_NODE && leader) sts32(anyw + 4u * wg, any);
        __syncthreads();
        if (!PER_NODE) {
            // VECTOR: chains with any gamma take s XOR gamma instead of f(s)
            // (lanes past the last chain are never written out: their chains
            // need no fix-up, which skips it on most steps of a ragged group)
            const uint32_t M = __reduce_or_sync(FULL, lane < W ? lds32(anyw + 4u * lane) : 0u) & vmask;
            if (M) {
                const int lo = 4 * q0, hi = min(4 * q1, n);
                for (int i = lo + lane; i < hi; i += 32) {
                    const uint32_t gmm = lds32(gam + 4u * (uint32_t)i);
                    if (gmm) sts32(gam + 4u * (uint32_t)i, 0u);  // keep the gamma buffer all-zero
                    const uint32_t a = gbase + state_off((uint32_t)i);
                    const uint32_t f = lds32(a + NB), o = lds32(a + OB);
                    sts32(a + NB, (f & ~M) | ((o ^ gmm) & M));
                }
            }
            __syncthreads();
        }
        if (stats && r > P.burn_in) {
            // A8 + A9 for this property, bit-sliced over the group's chains
            const uint32_t b = ChainStats::indicator(P, prop, lane, [&](uint32_t i) { return gbase + state_off(i) + NB; });
            cs.record(P, b, r - P.burn_in - 1, valid, orow());
        }
    };
    for (int64_t r = r_begin; r <= r_end; r += 2) {
        step(r, std::integral_constant<uint32_t, 0u>());
        if (r + 1 <= r_end) step(r + 1, std::integral_constant<uint32_t, 16u>());
    }
    if (r_end >= r_begin && ((r_end - r_begin + 1) & 1)) cur = 16u;  // odd step count: newest in buffer 1

    if (!last_chunk) {
        // suspend: bit-sliced state and warp-0 counters to scratch, then
        // release chunk c+1 of this group
        for (int i = tid; i < n; i += blockDim.x) __stcg(scr() + i, lds32(gbase + state_off(i) + cur));
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
#if !defined(PBN_GZ_START) && !defined(PBN_GZ_NONE)
        if (!PER_NODE && vmask != FULL)  // see the end of the unit below
            for (int i = tid; i < P.n_pad; i += blockDim.x) sts32(gam + 4u * i, 0u);
#endif
        continue;
    }

    // ---- epilogue: final state back to chain-major rows ----
    {
        for (int b = b0; b < b1; ++b) {
            uint32_t v = 0;
            for (int k = 0; k < 32; ++k) {
                const int i = 32 * b + k;
                if (i >= n) break;
                v |= ((lds32(gbase + state_off(i) + cur) >> lane) & 1u) << k;
            }
            if (valid) P.state[(int64_t)chain_local * nsw + b] = v;
        }
    }
    if (stats) cs.finish(P, prop, valid, orow(), leader);
#if !defined(PBN_GZ_START) && !defined(PBN_GZ_NONE)
    // a ragged group's chain-less lanes may draw perturbations that never
    // trigger the fix-up (M masks them): their gamma bits must not reach the
    // next unit of this CTA, where those lanes hold chains
    if (!PER_NODE && P.persistent && vmask != FULL)
        for (int i = tid; i < P.n_pad; i += blockDim.x) sts32(gam + 4u * i, 0u);
#endif
    }  // work units
}

// kernel table: [SMEM][MODE][FT-3][SLOW]
template <bool SMEM, int MODE, int FT, bool SLOW>
const void* kptr()
{
    return reinterpret_cast<const void*>(&traj_kernel<SMEM, MODE, FT, SLOW>);
}

template <bool SMEM, int MODE>
const void* pick_ft(int FT, bool slow)
{
    switch (FT) {
        case 3: return slow ? kptr<SMEM, MODE, 3, true>() : kptr<SMEM, MODE, 3, false>();
        case 4: return slow ? kptr<SMEM, MODE, 4, true>() : kptr<SMEM, MODE, 4, false>();
        case 5: return slow ? kptr<SMEM, MODE, 5, true>() : kptr<SMEM, MODE, 5, false>();
        case 6: return slow ? kptr<SMEM, MODE, 6, true>() : kptr<SMEM, MODE, 6, false>();
        case 7: return slow ? kptr<SMEM, MODE, 7, true>() : kptr<SMEM, MODE, 7, false>();
        default: return slow ? kptr<SMEM, MODE, 8, true>() : kptr<SMEM, MODE, 8, false>();
    }
}

}  // namespace
}  // namespace pbn
