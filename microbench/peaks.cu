// peaks.cu -- measured roofline inputs for the PBN trajectory kernel on B200
// (sm_100a): integer ALU / FMA pipe issue rates, total issue rate, shared-
// memory wavefront rate and L2 read bandwidth ("All P are
// measured ... at the SM clock observed during the run").
//
// Method (round 2; round 1's per-thread clock64 window was not bracketed by a
// barrier and over-reported): every kernel runs 2 CTAs x 1024
// threads on every SM; each CTA brackets its timed loop with __syncthreads()
// and records clock64() and %globaltimer at both ends (thread 0), so
//   rate   = warp-instructions issued by the SM's CTAs / the SM's cycle count
//            over the union of their barrier-bracketed windows (clock64 is
//            the SM's own counter)
//   clock  = cycles / globaltimer ns of the same window (the SM clock under
//            this load, MHz)
// and the whole grid is also timed with CUDA events (elapsed_ms).  One
// instruction type per kernel, 8 independent register chains per thread,
// 64 instructions per loop iteration (loop overhead < 5 %).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#define ITERS 32768
#define CHECK(x)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__device__ unsigned long long g_c0[4096], g_c1[4096];  // clock64 at the window ends (per-SM counter)
__device__ unsigned long long g_n0[4096], g_n1[4096];  // %globaltimer at the window ends
__device__ uint32_t g_smid[4096];
__device__ uint32_t g_sink[1 << 20];

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid()
{
    uint32_t s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}

template <int OP>
__global__ void __launch_bounds__(1024, 2) kbench(uint32_t seed)
{
    __shared__ uint32_t sm[4096];
    uint32_t r[8], s[8];
    const uint32_t tid = threadIdx.x;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    // pointer-chase tables: word i -> address of word i + 32 (same bank) for
    // OP 6/7; 16-byte slot j -> slot j + 8 (same 4 banks) for OP 8
    for (int i = tid; i < 4096; i += blockDim.x)
        sm[i] = (OP == 8) ? sbase + 16u * ((((uint32_t)i >> 2) + 8u) & 1023u) : sbase + 4u * ((i + 32u) & 4095u);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        r[k] = seed * (tid + 1) + k * 77u;
        s[k] = (k + 1) * 0x9E3779B9u | 1u;
        if (OP == 6) r[k] = sbase + 4u * ((32u * (8u * k + (seed & 7u)) + (tid & 31u)) & 4095u);
        if (OP == 7) r[k] = sbase + 4u * ((32u * (8u * k + (seed & 7u)) + ((tid >> 5) & 31u)) & 4095u);
        if (OP == 8) r[k] = sbase + 16u * ((8u * (8u * k + (seed & 7u)) + 2u * (tid & 3u)) & 1023u);
    }
    const uint32_t lmask = 1u << (tid & 31);
    __syncthreads();
    unsigned long long t0 = 0, n0 = 0;
    if (tid == 0) {
        t0 = clock64();
        n0 = gtimer();
    }
#pragma unroll 1
    for (int it = 0; it < ITERS; it += 64) {
#pragma unroll
        for (int kk = 0; kk < 64; ++kk) {
            const int k = kk & 7;
            if (OP == 0) {  // LOP3 (3-input XOR): ALU pipe
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[k]) : "r"(s[k]), "r"(lmask));
            } else if (OP == 1) {  // IMAD.WIDE (mul.wide.u32): FMA (heavy) pipe; (r, s) <- (hi, lo)(r s)
                asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, %1; mov.b64 {%1, %0}, t;}"
                             : "+r"(r[k]), "+r"(s[k]));
            } else if (OP == 2) {  // IMAD (mad.lo): FMA pipe
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[k]) : "r"(s[k]), "r"(lmask));
            } else if (OP == 3) {  // LOP3 and IMAD alternating: total issue (both pipes)
                if (kk & 1)
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[k]) : "r"(s[k]), "r"(lmask));
                else
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[k]) : "r"(s[k]), "r"(lmask));
            } else if (OP == 4) {  // IADD (add.u32), chained across the 8 registers (not foldable)
                asm volatile("add.u32 %0, %0, %1;" : "+r"(r[k]) : "r"(r[(k + 3) & 7]));
            } else if (OP == 5) {  // ISETP + SELP (selection compare; ptxas fuses it into VIMNMX)
                asm volatile("{.reg .pred p; setp.gt.u32 p, %0, %1; selp.u32 %0, %1, %0, p;}" : "+r"(r[k]) : "r"(r[(k + 5) & 7]));
            } else if (OP == 6 || OP == 7 || OP == 8) {
                // pointer chase: every word holds the shared address of the
                // next word of its chain (no address arithmetic in the loop)
                // 6: LDS.32, lane l stays in bank l (32 distinct banks: 1 wavefront)
                // 7: LDS.32 broadcast (every lane the same address)
                // 8: LDS.128, 4 distinct 16-byte addresses (lane & 3) in distinct banks
                if (OP == 8) {
                    uint4 v;
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                 : "r"(r[k]));
                    r[k] = v.x;
                } else {
                    asm volatile("ld.shared.u32 %0, [%0];" : "+r"(r[k]));
                }
            } else if (OP == 9) {  // VOTE.ballot
                asm volatile("{.reg .pred p; setp.ne.u32 p, %0, 0; vote.sync.ballot.b32 %0, p, 0xffffffff;}"
                             : "+r"(r[k]));
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        g_c0[blockIdx.x] = t0;
        g_c1[blockIdx.x] = clock64();
        g_n0[blockIdx.x] = n0;
        g_n1[blockIdx.x] = gtimer();
        g_smid[blockIdx.x] = smid();
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= r[k] ^ s[k];
    g_sink[(blockIdx.x * blockDim.x + tid) & ((1 << 20) - 1)] = acc;
}

// L2 read bandwidth: every CTA streams a buffer that fits the L2 (64 MiB),
// 16-byte ld.global.cg (L1 bypass), several passes.
__global__ void __launch_bounds__(1024, 2) kl2(const uint4* __restrict__ buf, size_t n16, int passes)
{
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
            uint4 v;
            asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "l"(buf + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    g_sink[(blockIdx.x * blockDim.x + threadIdx.x) & ((1 << 20) - 1)] = acc;
}

struct Res {
    double warp_instr_per_clk_per_sm, sm_mhz, elapsed_ms;
};

template <int OP>
Res run(int sms)
{
    const int blocks = sms * 2, threads = 1024;
    kbench<OP><<<blocks, threads>>>(12345);  // warm-up (clocks ramp)
    CHECK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    CHECK(cudaEventCreate(&a));
    CHECK(cudaEventCreate(&b));
    CHECK(cudaEventRecord(a));
    kbench<OP><<<blocks, threads>>>(777);
    CHECK(cudaEventRecord(b));
    CHECK(cudaDeviceSynchronize());
    float ms = 0;
    CHECK(cudaEventElapsedTime(&ms, a, b));
    std::vector<unsigned long long> c0(blocks), c1(blocks), n0(blocks), n1(blocks);
    std::vector<uint32_t> sid(blocks);
    CHECK(cudaMemcpyFromSymbol(c0.data(), g_c0, sizeof(unsigned long long) * blocks));
    CHECK(cudaMemcpyFromSymbol(c1.data(), g_c1, sizeof(unsigned long long) * blocks));
    CHECK(cudaMemcpyFromSymbol(n0.data(), g_n0, sizeof(unsigned long long) * blocks));
    CHECK(cudaMemcpyFromSymbol(n1.data(), g_n1, sizeof(unsigned long long) * blocks));
    CHECK(cudaMemcpyFromSymbol(sid.data(), g_smid, sizeof(uint32_t) * blocks));
    // per SM: the UNION of the windows of the CTAs it ran (clock64 is the
    // SM's own cycle counter, so the windows of co-resident CTAs compare)
    std::vector<unsigned long long> lo(4096, ~0ull), hi(4096, 0), nlo(4096, ~0ull), nhi(4096, 0);
    std::vector<int> cnt(4096, 0);
    for (int i = 0; i < blocks; ++i) {
        const uint32_t s = sid[i] & 4095u;
        lo[s] = std::min(lo[s], c0[i]);
        hi[s] = std::max(hi[s], c1[i]);
        nlo[s] = std::min(nlo[s], n0[i]);
        nhi[s] = std::max(nhi[s], n1[i]);
        cnt[s]++;
    }
    double rate = 0, mhz = 0;
    int used = 0;
    for (int s = 0; s < 4096; ++s)
        if (cnt[s]) {
            rate += (double)cnt[s] * 32.0 * ITERS / (double)(hi[s] - lo[s]);
            mhz += (double)(hi[s] - lo[s]) / (double)(nhi[s] - nlo[s]) * 1e3;
            used++;
        }
    Res r;
    r.warp_instr_per_clk_per_sm = rate / used;
    r.sm_mhz = mhz / used;
    r.elapsed_ms = ms;
    return r;
}

int main()
{
    int dev = 0, sms = 0;
    CHECK(cudaGetDevice(&dev));
    CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const char* names[] = {"LOP3 (alu)",        "IMAD.WIDE (fma heavy)", "IMAD (fma)",    "LOP3+IMAD (issue)",
                           "IADD (add.u32)",    "ISETP+SEL (VIMNMX)",             "LDS.32 32 banks (1 wf)", "LDS.32 broadcast",
                           "LDS.128 4 addresses", "VOTE.ballot (+ISETP)"};
    Res v[10];
    v[0] = run<0>(sms);
    v[1] = run<1>(sms);
    v[2] = run<2>(sms);
    v[3] = run<3>(sms);
    v[4] = run<4>(sms);
    v[5] = run<5>(sms);
    v[6] = run<6>(sms);
    v[7] = run<7>(sms);
    v[8] = run<8>(sms);
    v[9] = run<9>(sms);
    // L2 read bandwidth
    const size_t bytes = 64ull << 20;
    uint4* buf = nullptr;
    CHECK(cudaMalloc(&buf, bytes));
    CHECK(cudaMemset(buf, 1, bytes));
    const int passes = 20;
    kl2<<<sms * 2, 1024>>>(buf, bytes / 16, 2);
    CHECK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    CHECK(cudaEventCreate(&a));
    CHECK(cudaEventCreate(&b));
    CHECK(cudaEventRecord(a));
    kl2<<<sms * 2, 1024>>>(buf, bytes / 16, passes);
    CHECK(cudaEventRecord(b));
    CHECK(cudaDeviceSynchronize());
    float ms = 0;
    CHECK(cudaEventElapsedTime(&ms, a, b));
    const double l2_gbs = (double)bytes * passes / (ms * 1e-3) / 1e9;
    printf("{\"sms\": %d, \"iters\": %d, \"tests\": {", sms, ITERS);
    for (int i = 0; i < 10; ++i)
        printf("%s\"%s\": {\"warp_instr_per_clk_per_sm\": %.4f, \"sm_mhz\": %.1f, \"elapsed_ms\": %.3f}", i ? ", " : "",
               names[i], v[i].warp_instr_per_clk_per_sm, v[i].sm_mhz, v[i].elapsed_ms);
    printf("}, \"l2_read_gbs\": %.1f, \"l2_buffer_mib\": %d}\n", l2_gbs, (int)(bytes >> 20));
    return 0;
}
