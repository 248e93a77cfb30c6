// pbn_traj.cu -- K1: fused PBN trajectory kernel for sm_100a.
//
// Hot path of PAPER.md §2.2 with the per-chain statistics of
// Algorithms 3-5 fused:
//
//   layout     one warp lane = one chain; 32 chains form a "group" whose state
//              is BIT-SLICED in shared memory: word[i] holds node i of the
//              group's 32 chains (bit l = lane l), double-buffered (A7).  A
//              group's nodes are split over W warps (4-node quads, the Philox
//              granularity); a named barrier per group closes each step.
//   per node   the warp walks its nodes in lock-step, so all network metadata
//              reads are broadcasts; per lane: one 32-bit Philox word u (A3),
//              perturbation u < T_p (A4), function j = #{k : u > E_k} (A5),
//              parent bits gathered from the old buffer with a rotate so bit
//              `lane` lands at index position m (A6), table lookup, and one
//              __ballot_sync commits the 32 chains' new bits as one word (A7).
//   VECTOR each step also stores gamma words; after the
//              step barrier every warp patches its own nodes for the chains
//              with any gamma: new = (f & ~M) | ((old ^ gamma) & M).
//   stats      warp 0 of each group evaluates the property on the new words
//              (A8: AND over (node, value) pairs, bit-sliced) and keeps per
//              lane (= chain) counters in registers: c1, n01, n10, first/last,
//              batch sums, packed bits (A9); epilogue writes them and adds the
//              six u64 totals with integer atomics (A10, order-independent).
//   image      the model image is staged into shared memory once per CTA with
//              one cp.async.bulk (TMA bulk copy, mbarrier completion) when it
//              fits; otherwise it is read through the read-only L1 path.
//
// Randomness: Philox4x32-10 with counter (i/4, chain, t lo, t hi) and key
// (seed lo, seed hi) -- reading Q2.  Every output depends only on (model,
// seed, chain id, absolute step), never on the launch shape.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "pbn_internal.h"

namespace pbn {

namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;

// Philox4x32-10 (Salmon et al., SC'11), product implementation.
__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ void group_barrier(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Image accessors: shared memory (SMEM=true) or read-only global path.
template <bool SMEM>
struct Img {
    const uint4* nrec;
    const uint2* fdesc;
    const uint32_t* aux;
    const uint32_t* xthr;
    __device__ __forceinline__ uint4 rec(int i) const { return SMEM ? nrec[i] : __ldg(nrec + i); }
    __device__ __forceinline__ uint2 desc(uint32_t f) const { return SMEM ? fdesc[f] : __ldg(fdesc + f); }
    __device__ __forceinline__ uint32_t a32(uint32_t w) const { return SMEM ? aux[w] : __ldg(aux + w); }
    __device__ __forceinline__ uint32_t a16(uint32_t h) const
    {
        const uint16_t* p = reinterpret_cast<const uint16_t*>(aux) + h;
        return SMEM ? (uint32_t)*p : (uint32_t)__ldg(p);
    }
    __device__ __forceinline__ uint32_t xt(uint32_t f) const { return SMEM ? xthr[f] : __ldg(xthr + f); }
};

// One node of one step for the warp's 32 chains (A4-A7).
template <bool SMEM, bool PER_NODE>
__device__ __forceinline__ void step_node(const Img<SMEM>& img, int i, uint32_t u, uint32_t Tp,
                                          const uint32_t* __restrict__ old, uint32_t* __restrict__ nw,
                                          uint32_t* __restrict__ gam, uint32_t& any, int lane)
{
    const uint4 rec = img.rec(i);
    const bool flip = u < Tp;                                   // gamma_i(t) = 1 (A4)
    const uint32_t gw = __ballot_sync(FULL, flip);
    const uint32_t fn_base = rec.w & 0xFFFFFu;
    const uint32_t thmax = (rec.w >> 20) & 31u;
    const uint32_t ellm1 = rec.w >> 25;
    // function selection by the same word (A5): j = #{k : u > E_k}
    uint32_t j = (uint32_t)(u > rec.x) + (uint32_t)(u > rec.y) + (uint32_t)(u > rec.z);
    if (ellm1 > 3u) {
        for (uint32_t k = 3; k < ellm1; ++k) j += (uint32_t)(u > img.xt(fn_base + k));
    }
    const uint2 d = img.desc(fn_base + j);
    const uint32_t theta = d.y & 31u;
    const uint32_t auxo = d.y >> 5;
    // parent gather (A6): parent m's bit for this lane lands at index bit m
    uint32_t idx = 0;
    for (uint32_t m = 0; m < thmax; ++m) {
        if (m < theta) {
            const uint32_t off = img.a16(2u * auxo + m);
            const uint32_t w = *reinterpret_cast<const uint32_t*>(
                reinterpret_cast<const uint8_t*>(old) + off);
            idx |= __funnelshift_r(w, w, (uint32_t)lane - m) & (1u << m);
        }
    }
    uint32_t tw;
    if (theta <= 5u) {
        tw = d.x;
    } else {
        tw = img.a32(auxo + ((theta + 1u) >> 1) + (idx >> 5));
    }
    const bool bit = (tw >> (idx & 31u)) & 1u;
    uint32_t nb = __ballot_sync(FULL, bit);                     // commit (A7)
    if (PER_NODE) {
        const uint32_t ow = old[i];
        nb = (nb & ~gw) | (~ow & gw);
    } else {
        any |= gw;
    }
    if (lane == 0) {
        nw[i] = nb;
        if (!PER_NODE) gam[i] = gw;
    }
}

template <bool SMEM, bool PER_NODE>
__global__ void __launch_bounds__(1024, 1) traj_kernel(const __grid_constant__ TrajParams P)
{
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t mbar;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int W = P.warps_per_group;
    const int g = warp / W;
    const int wg = warp - g * W;
    const int n = P.n;

    // ---- A1: stage the model image into shared memory (one bulk copy) ----
    Img<SMEM> img;
    {
        const uint8_t* base = SMEM ? smem : P.image;
        img.nrec = reinterpret_cast<const uint4*>(base + P.L.off_nrec);
        img.fdesc = reinterpret_cast<const uint2*>(base + P.L.off_fdesc);
        img.aux = reinterpret_cast<const uint32_t*>(base + P.L.off_aux);
        img.xthr = reinterpret_cast<const uint32_t*>(base + P.L.off_xthr);
    }
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
                    "[%3];" ::"r"(smem_u32(smem + off)),
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

    const int64_t group = (int64_t)blockIdx.x * P.groups_per_cta + g;
    if (g >= P.groups_per_cta || group * 32 >= P.n_chains) return;
    const int64_t chain_local = group * 32 + lane;
    const bool valid = chain_local < P.n_chains;
    const uint32_t chain = (uint32_t)(P.chain_base + chain_local);

    uint32_t* gbase = reinterpret_cast<uint32_t*>(smem + P.image_smem_bytes) + (size_t)g * P.group_stride;
    uint32_t* bufA = gbase;                 // bufA: current state, bufB: next
    uint32_t* bufB = gbase + P.n_pad;
    uint32_t* gam = gbase + 2 * P.n_pad;                        // VECTOR only
    uint32_t* anyw = gbase + (PER_NODE ? 2 : 3) * P.n_pad;      // [W]
    const int bar_id = 1 + g;
    const int bar_n = W * 32;

    const int q0 = (int)((int64_t)wg * P.nquads / W);
    const int q1 = (int)((int64_t)(wg + 1) * P.nquads / W);
    const uint32_t k0 = (uint32_t)P.seed, k1 = (uint32_t)(P.seed >> 32);

    // ---- A2: initial state ----
    if (P.init) {
        for (int q = q0; q < q1; ++q) {
            const uint4 r = philox4x32_10((uint32_t)q, chain, 0u, 0u, k0, k1);
            const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * q + k;
                if (i < n) {
                    const uint32_t wv = __ballot_sync(FULL, (rr[k] >> 31) != 0u);
                    if (lane == 0) bufA[i] = wv;
                }
            }
        }
    } else {
        const int nb = P.state_words;
        const int b0 = (int)((int64_t)wg * nb / W), b1 = (int)((int64_t)(wg + 1) * nb / W);
        for (int b = b0; b < b1; ++b) {
            const uint32_t v = valid ? P.state[chain_local * nb + b] : 0u;
            for (int k = 0; k < 32; ++k) {
                const int i = 32 * b + k;
                if (i >= n) break;
                const uint32_t wv = __ballot_sync(FULL, (v >> k) & 1u);
                if (lane == 0) bufA[i] = wv;
            }
        }
    }
    group_barrier(bar_id, bar_n);

    // ---- per-lane statistics (warp 0 of the group) ----
    uint32_t c1 = 0, n01 = 0, n10 = 0, first = 0, prev = 0, bacc = 0, bitw = 0;
    int64_t bcount = 0;  // elements in the current batch
    const int64_t total = P.burn_in + P.steps;
    const uint32_t Tp = P.Tp;

    for (int64_t r = 1; r <= total; ++r) {
        const uint64_t t = (uint64_t)(P.step0 + r);
        const uint32_t t_lo = (uint32_t)t, t_hi = (uint32_t)(t >> 32);
        const uint32_t* old = bufA;
        uint32_t* nw = bufB;
        uint32_t any = 0;
        for (int q = q0; q < q1; ++q) {
            const uint4 rw = philox4x32_10((uint32_t)q, chain, t_lo, t_hi, k0, k1);
            const int i0 = 4 * q;
            if (i0 + 3 < n) {
                step_node<SMEM, PER_NODE>(img, i0 + 0, rw.x, Tp, old, nw, gam, any, lane);
                step_node<SMEM, PER_NODE>(img, i0 + 1, rw.y, Tp, old, nw, gam, any, lane);
                step_node<SMEM, PER_NODE>(img, i0 + 2, rw.z, Tp, old, nw, gam, any, lane);
                step_node<SMEM, PER_NODE>(img, i0 + 3, rw.w, Tp, old, nw, gam, any, lane);
            } else {
                const uint32_t rr[4] = {rw.x, rw.y, rw.z, rw.w};
                for (int k = 0; k < 4 && i0 + k < n; ++k)
                    step_node<SMEM, PER_NODE>(img, i0 + k, rr[k], Tp, old, nw, gam, any, lane);
            }
        }
        if (!PER_NODE && lane == 0) anyw[wg] = any;
        group_barrier(bar_id, bar_n);
        if (!PER_NODE) {
            // VECTOR: chains with any gamma take s XOR gamma instead of f(s)
            uint32_t M = 0;
            for (int w = 0; w < W; ++w) M |= anyw[w];
            if (M) {
                const int lo = 4 * q0, hi = min(4 * q1, n);
                for (int i = lo + lane; i < hi; i += 32) nw[i] = (nw[i] & ~M) | ((old[i] ^ gam[i]) & M);
            }
            group_barrier(bar_id, bar_n);
        }
        if (wg == 0 && r > P.burn_in) {
            // A8: property indicator, bit-sliced over the group's chains
            uint32_t Iw = FULL;
            for (int k = 0; k < P.pred_k; ++k) {
                const uint32_t w = nw[P.pred_node[k]];
                Iw &= P.pred_val[k] ? w : ~w;
            }
            const uint32_t b = (Iw >> lane) & 1u;
            const int64_t wpos = r - P.burn_in - 1;
            // A9: fused per-chain statistics
            if (wpos == 0) {
                first = b;
            } else {
                n01 += (~prev & b) & 1u;
                n10 += (prev & ~b) & 1u;
            }
            prev = b;
            c1 += b;
            if (P.batch > 0) {
                bacc += b;
                if (++bcount == P.batch || wpos + 1 == P.steps) {
                    if (valid) P.batch_sums[chain_local * P.batch_row + wpos / P.batch] = bacc;
                    bacc = 0;
                    bcount = 0;
                }
            }
            if (P.emit_bits) {
                const int64_t bpos = P.bits_offset + wpos;
                bitw |= b << (bpos & 31);
                const bool word_end = (bpos & 31) == 31;
                if (word_end || wpos + 1 == P.steps) {
                    if (valid) {
                        uint32_t* dst = P.bits + chain_local * P.bits_row + (bpos >> 5);
                        // the word holding bit bits_offset keeps its lower (earlier)
                        // bits: OR-merge; every other word is overwritten
                        const bool own = (bpos & ~(int64_t)31) >= P.bits_offset;
                        if (own) *dst = bitw;
                        else atomicOr(dst, bitw);
                    }
                    bitw = 0;
                }
            }
        }
        { uint32_t* tmp = bufA; bufA = bufB; bufB = tmp; }  // bufA holds the newest state
    }

    // ---- epilogue: final state back to chain-major rows ----
    {
        const uint32_t* fin = bufA;
        const int nb = P.state_words;
        const int b0 = (int)((int64_t)wg * nb / W), b1 = (int)((int64_t)(wg + 1) * nb / W);
        for (int b = b0; b < b1; ++b) {
            uint32_t v = 0;
            for (int k = 0; k < 32; ++k) {
                const int i = 32 * b + k;
                if (i >= n) break;
                v |= ((fin[i] >> lane) & 1u) << k;
            }
            if (valid) P.state[chain_local * nb + b] = v;
        }
    }
    if (wg == 0) {
        const uint32_t last = prev;
        const int64_t Wn = P.steps;
        uint32_t n0from = 0, n1from = 0;
        if (Wn > 0) {
            n1from = c1 - last;
            n0from = (uint32_t)(Wn - c1) - (1u - last);
        }
        if (valid) {
            if (P.c1) P.c1[chain_local] = c1;
            if (P.n01) P.n01[chain_local] = n01;
            if (P.n10) P.n10[chain_local] = n10;
            if (P.first_last) P.first_last[chain_local] = (uint8_t)((Wn > 0) ? (first | (last << 1)) : 0);
        }
        if (P.totals) {
            unsigned long long v[6];
            v[0] = valid ? c1 : 0;
            v[1] = valid ? (unsigned long long)c1 * c1 : 0;
            v[2] = valid ? n01 : 0;
            v[3] = valid ? n10 : 0;
            v[4] = valid ? n0from : 0;
            v[5] = valid ? n1from : 0;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(FULL, v[k], o);
            }
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < 6; ++k)
                    if (v[k]) atomicAdd(P.totals + k, v[k]);
            }
        }
    }
}

template <bool SMEM, bool PER_NODE>
const void* kernel_ptr()
{
    return reinterpret_cast<const void*>(&traj_kernel<SMEM, PER_NODE>);
}

int sm_count(int device)
{
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v;
}

}  // namespace

int plan_traj_launch(const TrajParams& P, int device, int want_groups, int want_warps,
                     LaunchPlan* plan, const char** why)
{
    int smem_optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return (int)e;
    const size_t static_smem = 64;  // mbarrier + slack
    const size_t limit = (size_t)smem_optin - static_smem;
    const size_t group_bytes = (size_t)P.group_stride * 4;
    const int64_t total_groups = (P.n_chains + 31) / 32;
    const int sms = sm_count(device);

    bool in_smem = (size_t)P.L.bytes + group_bytes <= limit;
    const size_t img = in_smem ? P.L.bytes : 0;
    if (img + group_bytes > limit) {
        *why = "network too large: one 32-chain group's state does not fit in shared memory";
        return -1;
    }
    const int g_fit = (int)((limit - img) / group_bytes);
    int G;
    if (want_groups > 0) {
        G = want_groups;
        if (G > g_fit) {
            *why = "groups_per_cta exceeds what fits in shared memory";
            return -1;
        }
    } else {
        // spread groups so that every SM gets work before stacking groups
        int64_t per_sm = (total_groups + sms - 1) / sms;
        G = (int)std::min<int64_t>(std::max<int64_t>(per_sm, 1), g_fit);
        G = std::min(G, kMaxWarpsPerCta);
    }
    int Wp;
    if (want_warps > 0) {
        Wp = want_warps;
    } else {
        Wp = kMaxWarpsPerCta / G;
        Wp = std::max(1, std::min(Wp, P.nquads));
    }
    if (G * Wp > kMaxWarpsPerCta || Wp > P.nquads) {
        *why = "groups_per_cta * warps_per_group must be <= 32 and warps_per_group <= ceil(n/4)";
        return -1;
    }
    if (G + 1 > 16) {
        *why = "at most 15 groups per CTA (named barriers)";
        return -1;
    }
    plan->groups_per_cta = G;
    plan->warps_per_group = Wp;
    plan->ctas = (int)((total_groups + G - 1) / G);
    plan->threads = G * Wp * 32;
    plan->smem_bytes = img + (size_t)G * group_bytes;
    plan->image_in_smem = in_smem;
    return 0;
}

int launch_traj(TrajParams P, const LaunchPlan& plan, void* stream)
{
    P.groups_per_cta = plan.groups_per_cta;
    P.warps_per_group = plan.warps_per_group;
    P.image_smem_bytes = plan.image_in_smem ? P.L.bytes : 0u;
    const void* fn;
    if (plan.image_in_smem)
        fn = P.per_node ? kernel_ptr<true, true>() : kernel_ptr<true, false>();
    else
        fn = P.per_node ? kernel_ptr<false, true>() : kernel_ptr<false, false>();
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)plan.smem_bytes);
    if (e != cudaSuccess) return (int)e;
    void* args[] = {&P};
    e = cudaLaunchKernel(fn, dim3(plan.ctas), dim3(plan.threads), args, plan.smem_bytes,
                         (cudaStream_t)stream);
    return (int)e;
}

}  // namespace pbn
