// pbn_recount.cu -- K2: window statistics of a sub-window of a stored
// indicator bitstream, without re-simulation.
//
// Used by the Algorithm 4 burn-in re-check ("additional M - psi elements
// will be discarded in the beginning of each chain") and by
// Skart re-batching.  One warp per chain; lanes stride over
// 32-element chunks of the sub-window (coalesced row reads); counts are
// popcounts, transitions are popcounts of (x, x >> 1) masks with the
// successor bit of the next chunk spliced in.  Totals as in K1 (A10).
#include <cuda_runtime.h>
#include <cstdint>

#include "pbn_internal.h"

namespace pbn {

namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;

// window bit w (0-based) of the sub-window = row bit (start + w)
__device__ __forceinline__ uint32_t row_bit(const uint32_t* row, int64_t pos)
{
    return (row[pos >> 5] >> (pos & 31)) & 1u;
}

// 32 window bits starting at window position 32*c (zero beyond length)
__device__ __forceinline__ uint32_t chunk(const uint32_t* row, int64_t start, int64_t length, int64_t c)
{
    const int64_t pos = start + 32 * c;
    const int64_t w = pos >> 5;
    const uint32_t sh = (uint32_t)(pos & 31);
    const int64_t row_end_word = (start + length - 1) >> 5;
    const uint32_t lo = row[w];
    const uint32_t hi = (w + 1 <= row_end_word) ? row[w + 1] : 0u;
    uint32_t x = __funnelshift_r(lo, hi, sh);
    const int64_t left = length - 32 * c;
    if (left < 32) x &= (left <= 0) ? 0u : ((1u << left) - 1u);
    return x;
}

__global__ void recount_kernel(const RecountParams R)
{
    const int64_t chain = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (chain >= R.n_chains) return;
    const uint32_t* row = R.bits + chain * R.row_words;
    const int64_t L = R.length;
    const int64_t nchunks = (L + 31) / 32;
    uint32_t c1 = 0, n01 = 0, n10 = 0;
    for (int64_t c = lane; c < nchunks; c += 32) {
        const uint32_t x = chunk(row, R.start, L, c);
        c1 += __popc(x);
        // successor of element k is element k+1; element 32 is next chunk's 0
        const int64_t nxt_pos = 32 * (c + 1);
        const uint32_t nb = (nxt_pos < L) ? row_bit(row, R.start + nxt_pos) : 0u;
        const uint32_t succ = (x >> 1) | (nb << 31);
        const int64_t pairs = min((int64_t)32, L - 1 - 32 * c);  // elements with a successor
        const uint32_t pm = pairs >= 32 ? FULL : (pairs <= 0 ? 0u : ((1u << pairs) - 1u));
        n01 += __popc(~x & succ & pm);
        n10 += __popc(x & ~succ & pm);
    }
    for (int o = 16; o > 0; o >>= 1) {
        c1 += __shfl_xor_sync(FULL, c1, o);
        n01 += __shfl_xor_sync(FULL, n01, o);
        n10 += __shfl_xor_sync(FULL, n10, o);
    }
    const uint32_t first = L > 0 ? row_bit(row, R.start) : 0u;
    const uint32_t last = L > 0 ? row_bit(row, R.start + L - 1) : 0u;
    if (R.batch > 0 && R.batch_sums) {
        const int64_t nb = R.batch_row;
        for (int64_t b = lane; b < nb; b += 32) {
            const int64_t lo = b * R.batch, hi = min(L, lo + R.batch);
            uint32_t s = 0;
            int64_t w = lo;
            while (w < hi) {
                const int64_t pos = R.start + w;
                const uint32_t sh = (uint32_t)(pos & 31);
                const int64_t take = min((int64_t)(32 - sh), hi - w);
                uint32_t v = row[pos >> 5] >> sh;
                if (take < 32) v &= (1u << take) - 1u;
                s += __popc(v);
                w += take;
            }
            R.batch_sums[chain * nb + b] = s;
        }
    }
    if (lane == 0) {
        if (R.c1) R.c1[chain] = c1;
        if (R.n01) R.n01[chain] = n01;
        if (R.n10) R.n10[chain] = n10;
        if (R.first_last) R.first_last[chain] = (uint8_t)(L > 0 ? (first | (last << 1)) : 0);
        if (R.totals) {
            const uint32_t n1from = L > 0 ? c1 - last : 0u;
            const uint32_t n0from = L > 0 ? (uint32_t)(L - c1) - (1u - last) : 0u;
            atomicAdd(R.totals + 0, (unsigned long long)c1);
            atomicAdd(R.totals + 1, (unsigned long long)c1 * c1);
            atomicAdd(R.totals + 2, (unsigned long long)n01);
            atomicAdd(R.totals + 3, (unsigned long long)n10);
            atomicAdd(R.totals + 4, (unsigned long long)n0from);
            atomicAdd(R.totals + 5, (unsigned long long)n1from);
        }
    }
}

}  // namespace

int launch_recount(const RecountParams& R, void* stream)
{
    if (R.n_chains <= 0) return 0;
    const int threads = 256;
    const int64_t blocks = (R.n_chains * 32 + threads - 1) / threads;
    recount_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(R);
    return (int)cudaGetLastError();
}

}  // namespace pbn
