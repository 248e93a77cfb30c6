// peaks.cu -- measured integer-pipe / shared-memory throughputs on B200 (sm_100a).
//
// Roofline inputs for the PBN trajectory kernel: each kernel
// runs a long unrolled loop of ONE instruction type over 8 independent
// register chains per thread, 1024 threads per CTA, 2 CTAs per SM, and
// reports warp-instructions per clock per SM (SM clock from clock64, all
// SMs busy).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define ITERS 4096
#define CHECK(x)                                                                   \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

__device__ unsigned long long g_cycles[4096];
__device__ uint32_t g_sink[1 << 20];

// ---- one instruction type per kernel; 8 independent chains ----
#define BODY8(STMT) STMT(0) STMT(1) STMT(2) STMT(3) STMT(4) STMT(5) STMT(6) STMT(7)

template <int OP>
__global__ void __launch_bounds__(1024, 2) kbench(uint32_t seed)
{
    __shared__ uint32_t sm[2048];
    uint32_t r[8], s[8];
    const uint32_t tid = threadIdx.x;
    for (int i = tid; i < 2048; i += blockDim.x) sm[i] = i * 2654435761u;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        r[k] = seed * (tid + 1) + k * 77u;
        s[k] = (k + 1) * 0x9E3779B9u;
    }
    const uint32_t lmask = 1u << (tid & 31);
    __syncthreads();
    const unsigned long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; it += 8) {
#pragma unroll
        for (int kk = 0; kk < 64; ++kk) {
            const int k = kk & 7;
            if (OP == 0) {  // LOP3 (3-input XOR)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[k]) : "r"(s[k]), "r"(lmask));
            } else if (OP == 1) {  // IADD (add.u32 -> IADD3 / VIADD)
                asm volatile("add.u32 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
            } else if (OP == 2) {  // IMAD (mad.lo)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[k]) : "r"(s[k]), "r"(lmask));
            } else if (OP == 3) {  // IMAD.WIDE (mul.wide.u32)
                asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, %1; mov.b64 {%0, %2}, t;}"
                             : "+r"(r[k]), "+r"(s[k])
                             : "r"(0xD2511F53u));
            } else if (OP == 4) {  // SHF (funnel rotate)
                asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
            } else if (OP == 5) {  // LOP3 -> predicate + predicated add
                asm volatile("{.reg .pred p; .reg .u32 t; and.b32 t, %1, %2; setp.ne.u32 p, t, 0; @p add.u32 %0, %0, 3;}"
                             : "+r"(r[k])
                             : "r"(s[k] ^ r[(k + 1) & 7]), "r"(lmask));
            } else if (OP == 6) {  // ISETP + SELP
                asm volatile("{.reg .pred p; setp.gt.u32 p, %0, %1; selp.u32 %0, %1, %0, p;}" : "+r"(r[k]) : "r"(s[k]));
            } else if (OP == 7) {  // VOTE.ballot
                asm volatile("{.reg .pred p; setp.ne.u32 p, %0, 0; vote.sync.ballot.b32 %0, p, 0xffffffff;}"
                             : "+r"(r[k]));
            } else if (OP == 8) {  // LDS broadcast (all lanes same address)
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(&sm[(r[k] & 1023)])));
                r[k] = v + k;
            } else if (OP == 9) {  // LDS.128 broadcast
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"((uint32_t)__cvta_generic_to_shared(&sm[(r[k] & 255) * 4])));
                r[k] = v.x ^ v.w;
            } else if (OP == 10) {  // LDS, 4 distinct addresses per warp (lane & 3)
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];"
                             : "=r"(v)
                             : "r"((uint32_t)__cvta_generic_to_shared(&sm[((r[k] & 255) * 8 + (tid & 3) * 37) & 2047])));
                r[k] = v + k;
            } else if (OP == 11) {  // LDS.64, 4 distinct addresses
                uint2 v;
                asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];"
                             : "=r"(v.x), "=r"(v.y)
                             : "r"((uint32_t)__cvta_generic_to_shared(&sm[(((r[k] & 127) * 8 + (tid & 3) * 38) & 2046)])));
                r[k] = v.x ^ v.y;
            } else if (OP == 12) {  // SEL only
                asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; selp.u32 %0, %1, %0, p;}" : "+r"(r[k]) : "r"(s[k]), "r"(lmask & 1));
            }
        }
    }
    const unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= r[k] ^ s[k];
    g_sink[(blockIdx.x * blockDim.x + tid) & ((1 << 20) - 1)] = acc;
    if (tid == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// Philox4x32-10 calls per clock per SM (the RNG cost of one node-quad)
__global__ void __launch_bounds__(1024, 2) kphilox(uint32_t seed)
{
    uint32_t c0 = threadIdx.x, c1 = blockIdx.x, c2 = seed, c3 = 0, acc = 0;
    const unsigned long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS / 8; ++it) {
        uint32_t a = c0 + it, b = c1, c = c2, d = c3;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            uint32_t lo0, hi0, lo1, hi1;
            asm("{.reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t;}" : "=r"(lo0), "=r"(hi0) : "r"(a), "r"(0xD2511F53u));
            asm("{.reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t;}" : "=r"(lo1), "=r"(hi1) : "r"(c), "r"(0xCD9E8D57u));
            const uint32_t na = hi1 ^ b ^ (seed + r * 0x9E3779B9u);
            const uint32_t nc = hi0 ^ d ^ (seed + r * 0xBB67AE85u);
            a = na; b = lo1; c = nc; d = lo0;
        }
        acc ^= a ^ b ^ c ^ d;
    }
    const unsigned long long t1 = clock64();
    g_sink[(blockIdx.x * blockDim.x + threadIdx.x) & ((1 << 20) - 1)] = acc;
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

static const char* NAMES[] = {"LOP3",  "IADD(add.u32)", "IMAD",     "IMAD.WIDE",  "SHF.rot",     "LOP3.P+@P add",
                              "ISETP+SEL", "VOTE.ballot", "LDS bcast", "LDS.128 bcast", "LDS 4-addr", "LDS.64 4-addr",
                              "SEL"};

template <int OP>
void run(int sms, double* out_per_sm_clk)
{
    const int blocks = sms * 2, threads = 1024;
    kbench<OP><<<blocks, threads>>>(12345);
    CHECK(cudaDeviceSynchronize());
    kbench<OP><<<blocks, threads>>>(777);
    CHECK(cudaDeviceSynchronize());
    unsigned long long cyc[4096];
    CHECK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * blocks));
    double mean = 0;
    for (int b = 0; b < blocks; ++b) mean += (double)cyc[b];
    mean /= blocks;
    // per SM: 2 CTAs x 32 warps x ITERS x 8 warp-instructions in `mean` cycles
    const double warp_instr = 2.0 * 32 * ITERS * 8;
    *out_per_sm_clk = warp_instr / mean;
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    CHECK(cudaGetDevice(&dev));
    CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CHECK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    double v[13];
    run<0>(sms, &v[0]);
    run<1>(sms, &v[1]);
    run<2>(sms, &v[2]);
    run<3>(sms, &v[3]);
    run<4>(sms, &v[4]);
    run<5>(sms, &v[5]);
    run<6>(sms, &v[6]);
    run<7>(sms, &v[7]);
    run<8>(sms, &v[8]);
    run<9>(sms, &v[9]);
    run<10>(sms, &v[10]);
    run<11>(sms, &v[11]);
    run<12>(sms, &v[12]);
    // Philox
    kphilox<<<sms * 2, 1024>>>(1);
    CHECK(cudaDeviceSynchronize());
    kphilox<<<sms * 2, 1024>>>(2);
    CHECK(cudaDeviceSynchronize());
    unsigned long long cyc[4096];
    CHECK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sms * 2));
    double mean = 0;
    for (int b = 0; b < sms * 2; ++b) mean += (double)cyc[b];
    mean /= sms * 2;
    const double philox_per_sm_clk = 2.0 * 1024 * (ITERS / 8) / mean;  // thread-calls per clock per SM
    printf("{\"sms\": %d, \"clock_rate_khz\": %d, \"warp_instr_per_clk_per_sm\": {", sms, clk);
    for (int i = 0; i < 13; ++i) printf("%s\"%s\": %.4f", i ? ", " : "", NAMES[i], v[i]);
    printf("}, \"philox_calls_per_clk_per_sm\": %.4f}\n", philox_per_sm_clk);
    return 0;
}
