// lds_patterns.cu -- shared-memory wavefronts of the access patterns the
// trajectory kernels issue (B200, sm_100a), read with ncu:
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum ./lds_patterns
// One kernel per pattern; each thread does ITERS loads of the pattern (the
// address comes from the previous load's value, so nothing is hoisted).
// Patterns (lane l, iteration value v = a data-dependent 0..3 "function"):
//   0 LDS.128, every lane the same address (K1's node record)
//   1 LDS.128, 4 addresses 32 B apart, lane l -> l & 3
//   2 LDS.128, 4 addresses 32 B apart, lane l -> (l * 7 + v) & 3 (data dependent, like
//     K1's descriptor of the selected function)
//   3 LDS.128, 4 addresses 32 B apart, quarter-warp uniform (l >> 3)
//   4 LDS.128, 2 addresses (l & 1), 32 B apart
//   5 LDS.32, every lane the same address
//   6 LDS.32, 4 addresses in 4 distinct banks, lane -> (l*7+v)&3
//   7 LDS.64, 4 addresses 32 B apart, lane -> (l*7+v)&3
//   8 LDS.128, 4 addresses 64 B apart, lane -> (l*7+v)&3
//   9 LDS.128, 4 addresses 16 B apart (one 64 B block), lane -> (l*7+v)&3
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define ITERS 4096

__device__ uint32_t g_sink[1 << 16];

template <int PAT>
__global__ void __launch_bounds__(512) kpat(uint32_t seed)
{
    __shared__ __align__(16) uint32_t sm[4096];
    const uint32_t tid = threadIdx.x, l = tid & 31;
    // every word holds a small pseudo-random value 0..3 (the "selected function")
    for (uint32_t i = tid; i < 4096; i += blockDim.x) sm[i] = (i * 2654435761u >> 13) & 3u;
    __syncthreads();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    uint32_t v = seed & 3u, acc = 0, blk = (tid >> 5) * 64u;
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
        // warp-uniform 256-byte-aligned block, different every iteration
        const uint32_t b = base + 4u * (((uint32_t)it * 64u + blk) & 4095u);
        uint32_t sel, a;
        if (PAT == 0 || PAT == 5) a = b;
        else if (PAT == 1) a = b + 32u * (l & 3u);
        else if (PAT == 3) a = b + 32u * (l >> 3);
        else if (PAT == 4) a = b + 32u * (l & 1u);
        else {
            sel = (l * 7u + v) & 3u;
            a = b + (PAT == 8 ? 64u : PAT == 9 ? 16u : 32u) * sel;
        }
        if (PAT == 5 || PAT == 6) {
            uint32_t x;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(PAT == 6 ? b + 4u * ((l * 7u + v) & 3u) : a));
            v = x & 3u;
            acc ^= x;
        } else if (PAT == 7) {
            uint2 x;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x.x), "=r"(x.y) : "r"(a));
            v = x.x & 3u;
            acc ^= x.y;
        } else {
            uint4 x;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "r"(a));
            v = x.x & 3u;
            acc ^= x.y ^ x.z ^ x.w;
        }
    }
    g_sink[(blockIdx.x * blockDim.x + tid) & 0xFFFF] = acc ^ v;
}

int main()
{
    kpat<0><<<148, 512>>>(1);
    kpat<1><<<148, 512>>>(1);
    kpat<2><<<148, 512>>>(1);
    kpat<3><<<148, 512>>>(1);
    kpat<4><<<148, 512>>>(1);
    kpat<5><<<148, 512>>>(1);
    kpat<6><<<148, 512>>>(1);
    kpat<7><<<148, 512>>>(1);
    kpat<8><<<148, 512>>>(1);
    kpat<9><<<148, 512>>>(1);
    cudaDeviceSynchronize();
    printf("ok %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
