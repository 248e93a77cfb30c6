// Pin for the oracle's Philox4x32-10: cuRAND's own header implementation,
// compiled for the HOST (the header has an NV_IS_HOST path for mulhilo32).
// Test helper only; never linked into the product or the oracle.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>

extern "C" void curand_philox_host(const unsigned* ctr, const unsigned* key, unsigned* out, int count)
{
    for (int i = 0; i < count; ++i) {
        uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
        uint2 k = make_uint2(key[2 * i], key[2 * i + 1]);
        uint4 r = curand_Philox4x32_10(c, k);
        out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
    }
}
