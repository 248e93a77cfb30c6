// mix.cu -- co-issue of the integer pipes on B200 (sm_100a) for the Philox
// multiply: how many warp-instructions per SM-clock each instruction mix
// sustains (K1b phase A is bound by its Philox rounds: 2 mul.wide + 2
// three-input XOR per round).  2 CTAs x 1024 threads on every SM, 8
// independent register chains per thread, CUDA-event timing of the grid,
// rate = warp-instructions / (elapsed x SM clock x SMs) with the SM clock
// given on the command line (the pool runs at 1965 MHz; bench.py samples it).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix mix.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define ITERS 16384

__device__ uint32_t g_sink[1 << 20];

template <int OP>
__global__ void __launch_bounds__(1024, 2) kmix(uint32_t seed)
{
    uint32_t r[8], s[8];
    const uint32_t tid = threadIdx.x;
    const uint32_t lmask = 1u << (tid & 31);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        r[k] = seed * (tid + 1) + k * 77u;
        s[k] = (k + 1) * 0x9E3779B9u | 1u;
    }
#pragma unroll 1
    for (int it = 0; it < ITERS; it += 16) {
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            const int k = kk & 7;
            if (OP == 0) {  // IMAD.WIDE alone: (r, s) <- (hi, lo)(r * C)
                asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, 0xD2511F53; mov.b64 {%1, %0}, t;}"
                             : "+r"(r[k]), "+r"(s[k]));
            } else if (OP == 1) {  // Philox round shape: IMAD.WIDE then LOP3 on its hi word
                asm volatile(
                    "{.reg .u64 t; .reg .u32 h, l; mul.wide.u32 t, %0, 0xD2511F53; mov.b64 {l, h}, t;"
                    " lop3.b32 %0, h, %1, %2, 0x96; mov.u32 %1, l;}"
                    : "+r"(r[k]), "+r"(s[k])
                    : "r"(lmask));
            } else if (OP == 2) {  // mul.hi alone
                asm volatile("mul.hi.u32 %0, %0, 0xD2511F53;" : "+r"(r[k]));
            } else if (OP == 3) {  // mul.hi + mul.lo (the 64-bit product as two 32-bit ops) + LOP3
                asm volatile(
                    "{.reg .u32 h, l; mul.hi.u32 h, %0, 0xD2511F53; mul.lo.u32 l, %0, 0xD2511F53;"
                    " lop3.b32 %0, h, %1, %2, 0x96; mov.u32 %1, l;}"
                    : "+r"(r[k]), "+r"(s[k])
                    : "r"(lmask));
            } else if (OP == 4) {  // ISETP + VOTE (a selection plane) alone
                asm volatile("{.reg .pred p; setp.gt.u32 p, %0, %1; vote.sync.ballot.b32 %0, p, 0xffffffff;}"
                             : "+r"(r[k])
                             : "r"(s[k]));
            } else if (OP == 5) {  // plane (ISETP + VOTE) interleaved with one IMAD.WIDE
                if (kk & 1)
                    asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, 0xD2511F53; mov.b64 {%1, %0}, t;}"
                                 : "+r"(r[k]), "+r"(s[k]));
                else
                    asm volatile("{.reg .pred p; setp.gt.u32 p, %0, %1; vote.sync.ballot.b32 %0, p, 0xffffffff;}"
                                 : "+r"(r[k])
                                 : "r"(s[k]));
            } else if (OP == 6) {  // LOP3 alone (reference)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[k]) : "r"(s[k]), "r"(lmask));
            } else if (OP == 8) {  // 1 ISETP + 4 VOTE (the vote's own rate)
                asm volatile(
                    "{.reg .pred p; .reg .u32 a, b, c; setp.ne.u32 p, %0, 0; vote.sync.ballot.b32 a, p, 0xffffffff;"
                    " vote.sync.ballot.b32 b, !p, 0xffffffff; vote.sync.ballot.b32 c, p, 0xffffffff;"
                    " vote.sync.ballot.b32 %0, !p, 0xffffffff; add.u32 %1, a, b; add.u32 %1, %1, c;}"
                    : "+r"(r[k]), "+r"(s[k]));
            } else if (OP == 9) {  // ISETP + VOTE + 2 LOP3 (do the votes co-issue with the ALU pipe?)
                asm volatile(
                    "{.reg .pred p; setp.gt.u32 p, %0, %1; vote.sync.ballot.b32 %0, p, 0xffffffff;"
                    " lop3.b32 %1, %1, %2, %1, 0x96; lop3.b32 %1, %1, %2, %0, 0x96;}"
                    : "+r"(r[k]), "+r"(s[k])
                    : "r"(lmask));
            } else if (OP == 10) {  // ISETP + VOTE + 2 IMAD.WIDE + 2 LOP3 (phase A's mix)
                asm volatile(
                    "{.reg .pred p; .reg .u64 t; .reg .u32 h, l; setp.gt.u32 p, %0, %1; vote.sync.ballot.b32 h, p, 0xffffffff;"
                    " mul.wide.u32 t, %0, 0xD2511F53; mov.b64 {l, %0}, t; lop3.b32 %0, %0, h, %2, 0x96;"
                    " mul.wide.u32 t, %1, 0xCD9E8D57; mov.b64 {%1, h}, t; lop3.b32 %1, %1, h, l, 0x96;}"
                    : "+r"(r[k]), "+r"(s[k])
                    : "r"(lmask));
            } else if (OP == 11) {  // phase A's ratio per node: 4 IMAD.WIDE, 5 LOP3, 3 ISETP, 2 VOTE (14 instr)
                asm volatile(
                    "{.reg .pred p, q; .reg .u64 t; .reg .u32 h, l, g;"
                    " mul.wide.u32 t, %0, 0xD2511F53; mov.b64 {l, h}, t; lop3.b32 %0, h, %1, %2, 0x96;"
                    " mul.wide.u32 t, %1, 0xCD9E8D57; mov.b64 {g, h}, t; lop3.b32 %1, h, l, %2, 0x96;"
                    " mul.wide.u32 t, %0, 0xD2511F53; mov.b64 {l, h}, t; lop3.b32 %0, h, g, %2, 0x96;"
                    " mul.wide.u32 t, %1, 0xCD9E8D57; mov.b64 {g, h}, t; lop3.b32 %1, h, l, %2, 0x96;"
                    " setp.gt.u32 q, %0, g; setp.gt.xor.u32 p, %0, l, q; setp.gt.xor.u32 p, %0, h, p;"
                    " vote.sync.ballot.b32 l, p, 0xffffffff; vote.sync.ballot.b32 h, q, 0xffffffff;"
                    " lop3.b32 %1, %1, l, h, 0x96;}"
                    : "+r"(r[k]), "+r"(s[k])
                    : "r"(lmask));
            } else if (OP == 7) {  // LOP3 + IMAD (lo) 1:1 (reference: both pipes)
                if (kk & 1)
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[k]) : "r"(s[k]), "r"(lmask));
                else
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[k]) : "r"(s[k]), "r"(lmask));
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= r[k] ^ s[k];
    g_sink[(blockIdx.x * blockDim.x + tid) & ((1 << 20) - 1)] = acc;
}

// SASS instructions per (kk) step of each OP, from cuobjdump of this file
// (checked when run: the counts below are the ones the rate is divided by)
static const double kInstPerStep[12] = {1.0, 2.0, 1.0, 3.0, 2.0, 1.5, 1.0, 1.0, 4.0625, 4.0, 6.0, 14.0};
static const char* kName[12] = {"IMAD.WIDE",
                               "IMAD.WIDE + LOP3 (Philox round shape)",
                               "IMAD.HI",
                               "IMAD.HI + IMAD + LOP3",
                               "ISETP + VOTE",
                               "ISETP + VOTE + IMAD.WIDE (per 2 steps: 3 instr)",
                               "LOP3",
                               "LOP3 + IMAD 1:1",
                               "ISETP + 4 VOTE + 2 IADD (7 instr)",
                               "ISETP + VOTE + 2 LOP3 (4 instr)",
                               "ISETP + VOTE + 2 IMAD.WIDE + 2 LOP3 (6 instr)",
                               "phase-A ratio: 4 IMAD.WIDE + 5 LOP3 + 3 ISETP + 2 VOTE (14 instr)"};

template <int OP>
void run(int sms, double mhz)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kmix<OP><<<2 * sms, 1024>>>(1);
    cudaEventRecord(a);
    kmix<OP><<<2 * sms, 1024>>>(2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double warps = 2.0 * sms * 1024 / 32;
    const double inst = warps * ITERS * kInstPerStep[OP];
    const double rate = inst / (ms * 1e-3 * mhz * 1e6 * sms);
    printf("{\"op\": \"%s\", \"warp_instr_per_clk_per_sm\": %.4f, \"ms\": %.3f}\n", kName[OP], rate, ms);
}

int main(int argc, char** argv)
{
    const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>(sms, mhz);
    run<1>(sms, mhz);
    run<2>(sms, mhz);
    run<3>(sms, mhz);
    run<4>(sms, mhz);
    run<5>(sms, mhz);
    run<6>(sms, mhz);
    run<7>(sms, mhz);
    run<8>(sms, mhz);
    run<9>(sms, mhz);
    run<10>(sms, mhz);
    run<11>(sms, mhz);
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
