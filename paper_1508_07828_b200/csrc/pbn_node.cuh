// pbn_node.cuh -- device building blocks shared by the trajectory kernels
// (pbn_traj.cu: one 32-chain group per CTA; pbn_cluster.cu: one group per
// thread-block cluster).  Philox4x32-10 (reading Q2), shared-memory access
// helpers, the device image accessors and the per-node step (A4-A7).
// Internal; included only by the .cu files of libpbnsim.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pbn_internal.h"

namespace pbn {
namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;

__device__ __forceinline__ void mulhilo(uint32_t a, uint32_t m, uint32_t& lo, uint32_t& hi)
{
    asm("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "r"(a), "r"(m));
}

// Philox4x32-10 (Salmon et al., SC'11) with precomputed round keys.
__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               const uint32_t* __restrict__ rk)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0, hi0, lo1, hi1;
        mulhilo(c0, 0xD2511F53u, lo0, hi0);
        mulhilo(c2, 0xCD9E8D57u, lo1, hi1);
        const uint32_t n0 = hi1 ^ c1 ^ rk[2 * r];
        const uint32_t n2 = hi0 ^ c3 ^ rk[2 * r + 1];
        c1 = lo1;
        c3 = lo0;
        c0 = n0;
        c2 = n2;
    }
    return make_uint4(c0, c1, c2, c3);
}

// The same generator split for the step loop.  With counter (q, chain, t_lo,
// t_hi), the parts of rounds 1-2 that depend only on (chain, t) are computed
// once per step (PhiloxStep); philox_quad finishes the 10 rounds for quad q.
struct PhiloxStep {
    uint32_t c0r1;   // round-1 output word 0: hi(M1 t_lo) ^ chain ^ k0
    uint32_t c1r1;   // round-1 output word 1: lo(M1 t_lo)
    uint32_t hi0r2;  // round-2 hi(M0 c0r1)
    uint32_t lo0r2;  // round-2 lo(M0 c0r1) = round-2 output word 3
    uint32_t t_hi;
};

__device__ __forceinline__ PhiloxStep philox_step(uint32_t chain, uint32_t t_lo, uint32_t t_hi,
                                                  const uint32_t* __restrict__ rk)
{
    PhiloxStep s;
    uint32_t lo1, hi1;
    mulhilo(t_lo, 0xCD9E8D57u, lo1, hi1);
    s.c0r1 = hi1 ^ chain ^ rk[0];
    s.c1r1 = lo1;
    mulhilo(s.c0r1, 0xD2511F53u, s.lo0r2, s.hi0r2);
    s.t_hi = t_hi;
    return s;
}

__device__ __forceinline__ uint4 philox_quad(uint32_t q, const PhiloxStep& s, const uint32_t* __restrict__ rk)
{
    // round 1 (quad part): (hi0, lo0) = M0 q
    uint32_t lo0, hi0;
    mulhilo(q, 0xD2511F53u, lo0, hi0);
    const uint32_t c2r1 = hi0 ^ s.t_hi ^ rk[1];
    const uint32_t c3r1 = lo0;
    // round 2: M0 * c0r1 is per step; M1 * c2r1 per quad
    uint32_t lo1, hi1;
    mulhilo(c2r1, 0xCD9E8D57u, lo1, hi1);
    uint32_t c0 = hi1 ^ s.c1r1 ^ rk[2];
    uint32_t c1 = lo1;
    uint32_t c2 = s.hi0r2 ^ c3r1 ^ rk[3];
    uint32_t c3 = s.lo0r2;
#pragma unroll
    for (int r = 2; r < 10; ++r) {
        uint32_t a0, b0, a1, b1;
        mulhilo(c0, 0xD2511F53u, a0, b0);
        mulhilo(c2, 0xCD9E8D57u, a1, b1);
        const uint32_t n0 = b1 ^ c1 ^ rk[2 * r];
        const uint32_t n2 = b0 ^ c3 ^ rk[2 * r + 1];
        c1 = a1;
        c3 = a0;
        c0 = n0;
        c2 = n2;
    }
    return make_uint4(c0, c1, c2, c3);
}

// The lane-uniform part of rounds 1-3 of philox_quad for quad q at one step:
// entering round 3, word 0 (hi(M1 c2r1) ^ lo(M1 t_lo) ^ k[2]) depends only on
// (q, key, t), so its product with M0 is the same for every chain.  One lane
// computes it per (quad, step) -- {lo(M0 c0) ^ k[7], hi(M0 c0) ^ k[5],
// lo(M1 c2r1) ^ k[4], lo(M0 q) ^ k[3]}, the round keys of the words they are
// XOR-ed into folded in -- and philox_quad_ps finishes the call with 15
// instead of 16 64-bit multiplies (philox_quad: 18, philox4x32_10: 20).
__device__ __forceinline__ uint4 philox_quad_step_consts(uint32_t q, const PhiloxStep& s,
                                                         const uint32_t* __restrict__ rk)
{
    uint32_t lo0, hi0, lo1, hi1, a0, b0;
    mulhilo(q, 0xD2511F53u, lo0, hi0);
    mulhilo(hi0 ^ s.t_hi ^ rk[1], 0xCD9E8D57u, lo1, hi1);
    mulhilo(hi1 ^ s.c1r1 ^ rk[2], 0xD2511F53u, a0, b0);
    return make_uint4(a0 ^ rk[7], b0 ^ rk[5], lo1 ^ rk[4], lo0 ^ rk[3]);
}

// philox_quad from the per-(quad, step) entry e: bit-identical output
__device__ __forceinline__ uint4 philox_quad_ps(const uint4 e, const PhiloxStep& s, const uint32_t* __restrict__ rk)
{
    uint32_t a0, b0, a1, b1;
    // round 3: the M0 product is e's; c2 = hi0r2 ^ lo(M0 q) ^ k[3]
    mulhilo(s.hi0r2 ^ e.w, 0xCD9E8D57u, a1, b1);
    uint32_t c0 = b1 ^ e.z;
    uint32_t c2 = e.y ^ s.lo0r2;
    uint32_t c1 = a1;
    // round 4 (word 3 = lo(M0 c0) of round 3, with k[7] folded in)
    mulhilo(c0, 0xD2511F53u, a0, b0);
    mulhilo(c2, 0xCD9E8D57u, a1, b1);
    c0 = b1 ^ c1 ^ rk[6];
    c2 = b0 ^ e.x;
    c1 = a1;
    uint32_t c3 = a0;
#pragma unroll
    for (int r = 4; r < 10; ++r) {
        mulhilo(c0, 0xD2511F53u, a0, b0);
        mulhilo(c2, 0xCD9E8D57u, a1, b1);
        const uint32_t n0 = b1 ^ c1 ^ rk[2 * r];
        const uint32_t n2 = b0 ^ c3 ^ rk[2 * r + 1];
        c1 = a1;
        c3 = a0;
        c0 = n0;
        c2 = n2;
    }
    return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

// shared-memory accessors on 32-bit shared addresses.  State words change
// every step (volatile: never cached across barriers); image words are
// immutable (plain asm: the compiler may schedule and CSE them freely).
__device__ __forceinline__ uint32_t lds32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds32_ro(uint32_t a)
{
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds16_ro(uint32_t a)
{
    uint16_t v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return (uint32_t)v;
}
__device__ __forceinline__ uint2 lds64_ro(uint32_t a)
{
    uint2 v;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds128_ro(uint32_t a)
{
    uint4 v;
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v)
{
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// State words of the current buffer.  `asm volatile` keeps them on the right
// side of the step barriers at the compiler level; the plain ld.shared lets
// ptxas interleave the loads of different nodes freely.
__device__ __forceinline__ uint32_t lds32_state(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void fence_state(uint32_t&, uint32_t&) {}
// 16-byte store of four consecutive words by one lane when pred != 0
__device__ __forceinline__ void sts128_if(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w, uint32_t pred)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t@p st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"r"(a),
        "r"(x), "r"(y), "r"(z), "r"(w), "r"(pred)
        : "memory");
}
__device__ __forceinline__ void sts32_if(uint32_t a, uint32_t v, uint32_t pred)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u32 [%0], %1;\n\t}" ::"r"(a), "r"(v),
                 "r"(pred)
                 : "memory");
}


// Image accessors.  SMEM: the staged image was relocated, so every stored
// offset is already an absolute shared address.  Global: offsets are
// relative to the image pointer (read-only path).
template <bool SMEM>
struct Img {
    const uint8_t* gbase;  // global address of the image (!SMEM)
    __device__ __forceinline__ uint4 ld128(uint32_t a) const
    {
        if (SMEM) return lds128_ro(a);
        return __ldg(reinterpret_cast<const uint4*>(gbase + a));
    }
    __device__ __forceinline__ uint2 ld64(uint32_t a) const
    {
        if (SMEM) return lds64_ro(a);
        return __ldg(reinterpret_cast<const uint2*>(gbase + a));
    }
    __device__ __forceinline__ uint32_t ld32(uint32_t a) const
    {
        if (SMEM) return lds32_ro(a);
        return __ldg(reinterpret_cast<const uint32_t*>(gbase + a));
    }
    __device__ __forceinline__ uint32_t ld16(uint32_t a) const
    {
        if (SMEM) return lds16_ro(a);
        return (uint32_t)__ldg(reinterpret_cast<const uint16_t*>(gbase + a));
    }
    // a + OFF with OFF a compile-time byte offset: the global path forms the
    // 64-bit address of a once and folds OFF into the load's immediate (a
    // 32-bit a + OFF first would cost an add and a 64-bit extension per load)
    template <uint32_t OFF>
    __device__ __forceinline__ uint4 ld128(uint32_t a) const
    {
        if (SMEM) return lds128_ro(a + OFF);
        return __ldg(reinterpret_cast<const uint4*>(gbase + a + OFF));
    }
    template <uint32_t OFF>
    __device__ __forceinline__ uint2 ld64(uint32_t a) const
    {
        if (SMEM) return lds64_ro(a + OFF);
        return __ldg(reinterpret_cast<const uint2*>(gbase + a + OFF));
    }
    template <uint32_t OFF>
    __device__ __forceinline__ uint32_t ld32(uint32_t a) const
    {
        if (SMEM) return lds32_ro(a + OFF);
        return __ldg(reinterpret_cast<const uint32_t*>(gbase + a + OFF));
    }
};

// Generic path for nodes outside the fast shape (ell > 4 or theta_max > 8:
// the dense class of P:605-609, NEXT-3).  `old` = address of buffer-0 word
// of node 0 plus the old buffer's offset.  Every loop has a warp-uniform
// trip count (the lanes' chains select different functions):
//   A5  j = #{k : u > E_k}: the node's thresholds are the same for every
//       lane, so they are read as warp-uniform 16-byte vectors (broadcast,
//       independent loads) and counted four at a time; beyond 64 functions
//       a binary search over the ascending thresholds (ceil(log2 ell) steps)
//   A6  theta_max(node) gather steps, predicated on m < theta of the
//       selected function
// inlined: C6 (all nodes generic) 5.23e10 -> 5.51e10 node-updates/s and
// fewer spills than the out-of-line call (PBN_SLOW_NOINLINE for A/B)
#ifdef PBN_SLOW_NOINLINE
#define PBN_SLOW_ATTR __noinline__
#else
#define PBN_SLOW_ATTR __forceinline__
#endif
template <bool SMEM>
__device__ PBN_SLOW_ATTR uint32_t slow_node_bit(const Img<SMEM>& img, uint32_t w, uint32_t u, uint32_t old,
                                                uint32_t rot)
{
    const uint4 sr = img.ld128(w & ~15u);  // {thr, ell, gdesc, theta_max}
    const uint32_t m1 = sr.y - 1u;         // thresholds E_1..E_{ell-1}
    uint32_t j = 0;
#ifndef PBN_DENSE_BSEARCH
    if (m1 <= 64u) {
        for (uint32_t k = 0; k < m1; k += 4u) {
            const uint4 e = img.ld128(sr.x + 4u * k);  // padded with 0xFFFFFFFF
            j += (uint32_t)(u > e.x) + (uint32_t)(u > e.y) + (uint32_t)(u > e.z) + (uint32_t)(u > e.w);
        }
    } else
#endif
    for (uint32_t step = m1 ? 1u << (31 - __clz(m1)) : 0u; step; step >>= 1)
        if (j + step <= m1 && u > img.ld32(sr.x + 4u * (j + step - 1u))) j += step;
    const uint4 gd = img.ld128(sr.z + 16u * j);  // {toff, theta, poff, 0}
    uint32_t idx = 0;
    // the parent offsets four at a time (poff 16-aligned, padded to whole
    // vectors): one dependent image read per four parents, not per parent
    for (uint32_t m = 0; m < sr.w; m += 4u) {
        const uint4 o = img.ld128(gd.z + 4u * m);
        const uint32_t oo[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
        for (uint32_t k = 0; k < 4u; ++k) {
            if (m + k < gd.y) {
                const uint32_t wv = lds32(old + oo[k]);
                idx = __funnelshift_l(__funnelshift_l(wv, wv, rot), idx, 1);
            }
        }
    }
    const uint32_t tw = img.ld32(gd.x + 4u * (idx >> 5));
    return (tw >> (idx & 31u)) & 1u;
}

// idx += B when this lane's bit of the parent word is set: one LOP3 producing a
// predicate (ALU pipe) and one predicated add.
template <uint32_t B>
__device__ __forceinline__ void add_if_bit(uint32_t& idx, uint32_t wv, uint32_t lmask)
{
    if (B == 0) return;
    asm("{\n\t.reg .pred p;\n\t.reg .u32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t"
        "@p add.u32 %0, %0, %3;\n\t}"
        : "+r"(idx)
        : "r"(wv), "r"(lmask), "n"(B));
}

// A6 for one fast function: dp = its descriptor; returns the lane's new bit.
template <bool SMEM, int FT, uint32_t OB>
__device__ __forceinline__ uint32_t fast_bit(const Img<SMEM>& img, const uint32_t dp, uint32_t sb, uint32_t lmask)
{
    // parent state word: absolute (relocated) address in shared-image
    // launches, state-relative otherwise
#define SB(x) (SMEM ? (x) : sb + (x))
    uint32_t tw, idx = 0;
    if constexpr (FT >= 7) {
        // descriptor words {a[0..7], table words}: the first FT-5 parents
        // pick one of the 2^(FT-5) table words (a dependent load), the other
        // five index within it
        const uint4 d0 = img.ld128(dp);
        const uint4 d1 = img.template ld128<16u>(dp);
        const uint32_t a[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
        constexpr int S = FT >= 7 ? FT - 5 : 2;
        uint32_t widx = 0;
        add_if_bit<(1u << (S - 1)) * 4u>(widx, lds32_state(SB(a[0]) + OB), lmask);
        add_if_bit<(S > 1 ? 1u << (S - 2) : 0u) * 4u>(widx, lds32_state(SB(a[1]) + OB), lmask);
        if (S > 2) add_if_bit<4u>(widx, lds32_state(SB(a[2 % FT]) + OB), lmask);
        add_if_bit<16u>(idx, lds32_state(SB(a[S % 8]) + OB), lmask);
        add_if_bit<8u>(idx, lds32_state(SB(a[(S + 1) % 8]) + OB), lmask);
        add_if_bit<4u>(idx, lds32_state(SB(a[(S + 2) % 8]) + OB), lmask);
        add_if_bit<2u>(idx, lds32_state(SB(a[(S + 3) % 8]) + OB), lmask);
        add_if_bit<1u>(idx, lds32_state(SB(a[(S + 4) % 8]) + OB), lmask);
        tw = img.template ld32<32u>(dp + widx);
    } else {
    // descriptor words {t0, [t1], a[0..FT-1]}: table word(s), then the FT
    // padded parents' state offsets, MSB first
    uint32_t tw0, tw1 = 0, a[6];
    {
        const uint4 d0 = img.ld128(dp);
        if (FT == 6) {
            const uint4 d1 = img.template ld128<16u>(dp);
            tw0 = d0.x; tw1 = d0.y; a[0] = d0.z; a[1] = d0.w;
            a[2] = d1.x; a[3] = d1.y; a[4] = d1.z; a[5] = d1.w;
        } else if (FT == 5) {
            const uint2 d1 = img.template ld64<16u>(dp);
            tw0 = d0.x; a[0] = d0.y; a[1] = d0.z; a[2] = d0.w; a[3] = d1.x; a[4] = d1.y; a[5] = 0;
        } else if (FT == 4) {
            const uint32_t d1 = img.template ld32<16u>(dp);
            tw0 = d0.x; a[0] = d0.y; a[1] = d0.z; a[2] = d0.w; a[3] = d1; a[4] = a[5] = 0;
        } else {
            tw0 = d0.x; a[0] = d0.y; a[1] = d0.z; a[2] = d0.w; a[3] = a[4] = a[5] = 0;
        }
    }
    // A6: gather: parent k contributes bit (FT-1-k) of the table index when
    // bit `lane` of its state word is set (LOP3 -> predicate, predicated add)
    // FT = 6: the first (most significant) parent picks the table word
    // (entries 32-63 in t1), the other five index within it
    tw = tw0;
    if (FT == 6) tw = (lds32_state(SB(a[0]) + OB) & lmask) ? tw1 : tw0;
    constexpr int S = FT == 6 ? 1 : 0;  // first parent handled above
    constexpr int R = FT - S;          // parents indexing within the word
    if (R > 0) add_if_bit<1u << (R > 0 ? R - 1 : 0)>(idx, lds32_state(SB(a[S + 0]) + OB), lmask);
    if (R > 1) add_if_bit<1u << (R > 1 ? R - 2 : 0)>(idx, lds32_state(SB(a[S + 1]) + OB), lmask);
    if (R > 2) add_if_bit<1u << (R > 2 ? R - 3 : 0)>(idx, lds32_state(SB(a[(S + 2) % 6]) + OB), lmask);
    if (R > 3) add_if_bit<1u << (R > 3 ? R - 4 : 0)>(idx, lds32_state(SB(a[(S + 3) % 6]) + OB), lmask);
    if (R > 4) add_if_bit<1u << (R > 4 ? R - 5 : 0)>(idx, lds32_state(SB(a[(S + 4) % 6]) + OB), lmask);
    }
    // the table words are stored bit-REVERSED (entry e at bit 31 - (e & 31)),
    // so the entry is the sign bit of the word shifted left by idx
    return (uint32_t)((int32_t)(tw << idx) < 0);
#undef SB
}

// One node of one step for the warp's 32 chains (A4-A7): returns the node's
// new state word (bit l = chain of lane l) and its gamma word in *gw_out.
//   sb   state base (shared address of buffer-0 word of node 0; uniform)
//   OB   byte offset of the OLD buffer (0 or 16, compile time)
template <bool SMEM, bool PER_NODE, int FT, bool SLOW, uint32_t OB, uint32_t QS = 32, bool GW = true>
__device__ __forceinline__ uint32_t node_word(const Img<SMEM>& img, const uint4 rec, uint32_t i, uint32_t u,
                                              uint32_t Tp, uint32_t sb, uint32_t lmask, uint32_t rot,
                                              uint32_t& gw_out)
{
    constexpr uint32_t DS = desc_bytes(FT);
    // gamma_i(t) = 1 (A4); callers that form it elsewhere (K1's VECTOR path) skip the vote
    const uint32_t gw = (GW || PER_NODE) ? __ballot_sync(FULL, u < Tp) : 0u;
    uint32_t bit;
    if (!SLOW || (rec.w & 7u) != kSlowNode) {
        // A5: descriptor of function j = #{k : u > E_k}
        uint32_t dp = rec.w;
        if (u > rec.x) dp += DS;
        if (u > rec.y) dp += DS;
        if (u > rec.z) dp += DS;
        bit = fast_bit<SMEM, FT, OB>(img, dp, sb, lmask);
    } else {
        bit = slow_node_bit<SMEM>(img, rec.w, u, sb + OB, rot);
    }
    uint32_t nb = __ballot_sync(FULL, bit != 0u);  // commit (A7)
    if (PER_NODE) {
        const uint32_t ow = lds32_state(sb + QS * (i >> 2) + 4u * (i & 3u) + OB);
        nb = (nb & ~gw) | (~ow & gw);
    }
    gw_out = gw;
    return nb;
}

// Geometric-skip perturbation stream (PBN_PERTURB_GEOMETRIC, reading Q18),
// one lane = one chain: gamma(t) = ones at k_1 = G(v_0), k_{j+1} = k_j + 1 +
// G(v_j) while k < n, G(v) = #{g < n : Cg[g] <= v} (geometric_skip over the
// image's table at `geo`), skip words v(chain, t, m) =
// Philox((2^31 + m/4, chain, t)).  Each flip ORs this lane's bit into the
// gamma word of its node (gam = buffer base, word i at gam + 4 i).  Returns
// the ballot of lanes with gamma(t) != 0.  The first word decides "any
// flip" with one compare (G(v_0) < n iff v_0 < Cg[n-1]).
template <bool SMEM, typename GamAddr>
__device__ __forceinline__ uint32_t geometric_gamma_at(const Img<SMEM>& img, uint32_t geo, int n, float inv_lnq,
                                                       uint32_t chain, uint32_t t_lo, uint32_t t_hi,
                                                       const uint32_t* __restrict__ rk, GamAddr gam_of, uint32_t lmask,
                                                       bool valid);
template <bool SMEM>
__device__ __forceinline__ uint32_t geometric_gamma(const Img<SMEM>& img, uint32_t geo, int n, float inv_lnq,
                                                    uint32_t chain, uint32_t t_lo, uint32_t t_hi,
                                                    const uint32_t* __restrict__ rk, uint32_t gam, uint32_t lmask,
                                                    bool valid)
{
    return geometric_gamma_at(img, geo, n, inv_lnq, chain, t_lo, t_hi, rk,
                              [gam](uint32_t k) { return gam + 4u * k; }, lmask, valid);
}
// the same with node k's gamma word at gam_of(k) (K1b: inside the plane vectors)
template <bool SMEM, typename GamAddr>
__device__ __forceinline__ uint32_t geometric_gamma_at(const Img<SMEM>& img, uint32_t geo, int n, float inv_lnq,
                                                       uint32_t chain, uint32_t t_lo, uint32_t t_hi,
                                                       const uint32_t* __restrict__ rk, GamAddr gam_of, uint32_t lmask,
                                                       bool valid)
{
    uint32_t has = 0;
    if (valid) {
        uint4 v = philox4x32_10(0x80000000u, chain, t_lo, t_hi, rk);
        if (v.x < img.ld32(geo + 4u * (uint32_t)(n - 1))) {
            has = 1;
            int k = -1;
            for (uint32_t m = 0;; ++m) {
                if (m > 0 && (m & 3u) == 0) v = philox4x32_10(0x80000000u + (m >> 2), chain, t_lo, t_hi, rk);
                const uint32_t w = (m & 3u) == 0 ? v.x : (m & 3u) == 1 ? v.y : (m & 3u) == 2 ? v.z : v.w;
                k += 1 + geometric_skip(w, n, inv_lnq, [&](int g) { return img.ld32(geo + 4u * (uint32_t)g); });
                if (k >= n) break;
                asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(gam_of((uint32_t)k)), "r"(lmask) : "memory");
            }
        }
    }
    return __ballot_sync(FULL, has != 0u);
}

// G(w) = #{g < n : Cg[g] <= w} (Cg non-decreasing): an estimate from the
// geometric law, g0 ~ ln(1 - w 2^-32) / ln(1 - p) (inv_lnq = 1 / ln(1 - p)),
// corrected against the table until exact -- the result depends on the table
// only, the estimate only sets where the (usually 0-2 step) search starts
template <typename Load>
__device__ __forceinline__ int geometric_skip(uint32_t w, int n, float inv_lnq, Load cg)
{
    const float x = (float)w * 2.3283064365386963e-10f;  // w 2^-32
    float e = log1pf(-x) * inv_lnq;
    e = fminf(fmaxf(e, 0.0f), (float)n);
    int g = (int)e;
    while (g < n && cg(g) <= w) ++g;
    while (g > 0 && cg(g - 1) > w) --g;
    return g;
}

// node records {E1, E2, E3, w} of one quad
struct Recs {
    uint4 r[4];
};
template <bool SMEM>
__device__ __forceinline__ Recs load_recs(const Img<SMEM>& img, uint32_t a)
{
    Recs x;
#pragma unroll
    for (int k = 0; k < 4; ++k) x.r[k] = img.ld128(a + 16u * k);
    return x;
}


// Per-chain statistics of one property over the recorded window (SURVEY
// §8(a) A8-A10), kept in the registers of the property's statistics warp
// (lane = chain) and written once at the end of the launch.
struct ChainStats {
    uint32_t c1 = 0, n01 = 0, n10 = 0, first = 0, prev = 0, bacc = 0, bitw = 0, bcount = 0;

    // A8: I_t of the lane's chain = AND of (node, value) pairs over the
    // bit-sliced new state (word address of node i: word(i))
    template <typename WordAddr>
    __device__ __forceinline__ static uint32_t indicator(const TrajParams& P, int prop, int lane, WordAddr word)
    {
        uint32_t Iw = FULL;
        for (int k = 0; k < P.pred_k[prop]; ++k) {
            const uint32_t w = lds32(word(P.pred_node[prop][k]));
            Iw &= P.pred_val[prop][k] ? w : ~w;
        }
        return (Iw >> lane) & 1u;
    }

    // A9: window element wpos = b; `row` = the chain's property-major row
    __device__ __forceinline__ void record(const TrajParams& P, uint32_t b, int64_t wpos, bool valid, int64_t row)
    {
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
                if (valid) P.batch_sums[row * P.batch_row + wpos / P.batch] = bacc;
                bacc = 0;
                bcount = 0;
            }
        }
        if (P.emit_bits) {
            const int64_t bpos = P.bits_offset + wpos;
            bitw |= b << (bpos & 31);
            if ((bpos & 31) == 31 || wpos + 1 == P.steps) {
                if (valid) {
                    uint32_t* dst = P.bits + row * P.bits_row + (bpos >> 5);
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

    // end of the launch: counters, first/last and (A10) the six u64 totals
    // with integer atomics (order-independent, exact)
    __device__ __forceinline__ void finish(const TrajParams& P, int prop, bool valid, int64_t row, bool leader) const
    {
        const uint32_t last = prev;
        const int64_t Wn = P.steps;
        uint32_t n0from = 0, n1from = 0;
        if (Wn > 0) {
            n1from = c1 - last;
            n0from = (uint32_t)(Wn - c1) - (1u - last);
        }
        if (valid) {
            if (P.c1) P.c1[row] = c1;
            if (P.n01) P.n01[row] = n01;
            if (P.n10) P.n10[row] = n10;
            if (P.first_last) P.first_last[row] = (uint8_t)((Wn > 0) ? (first | (last << 1)) : 0);
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
            if (leader) {
#pragma unroll
                for (int k = 0; k < 6; ++k)
                    if (v[k]) atomicAdd(P.totals + 6 * prop + k, v[k]);
            }
        }
    }
};

}  // namespace
}  // namespace pbn
