// pbn_api.cpp -- host side of libpbnsim: validation, device-image builder,
// launch wrappers, fp64 statistics and the Algorithm 3/4/5 driver.
//
// C ABI declared in include/pbnsim.h.  Nothing here is shared with oracle/.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pbnsim.h"
#include "pbn_internal.h"

#include <map>
#include <mutex>
#include <tuple>

namespace pbn {

namespace {
std::mutex g_cache_mu;
std::map<const void*, std::pair<size_t, bool>> g_func_smem;
std::map<std::tuple<const void*, int, size_t>, int> g_occ;
std::map<std::pair<int, int>, int> g_dev_attr;
}  // namespace

cudaError_t ensure_func_smem(const void* fn, size_t bytes, bool nonportable_cluster)
{
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto& e = g_func_smem[fn];
    if (bytes > e.first) {
        const cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (r != cudaSuccess) return r;
        e.first = bytes;
    }
    if (nonportable_cluster && !e.second) {
        const cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (r != cudaSuccess) return r;
        e.second = true;
    }
    return cudaSuccess;
}

cudaError_t cached_blocks_per_sm(const void* fn, int threads, size_t smem, int* out)
{
    std::lock_guard<std::mutex> lk(g_cache_mu);
    const auto key = std::make_tuple(fn, threads, smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) {
        *out = it->second;
        return cudaSuccess;
    }
    const cudaError_t r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, threads, smem);
    if (r == cudaSuccess) g_occ[key] = *out;
    return r;
}

int cached_device_attr(cudaDeviceAttr attr, int device)
{
    std::lock_guard<std::mutex> lk(g_cache_mu);
    const auto key = std::make_pair((int)attr, device);
    auto it = g_dev_attr.find(key);
    if (it != g_dev_attr.end()) return it->second;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, attr, device) != cudaSuccess) return 0;
    g_dev_attr[key] = v;
    return v;
}

}  // namespace pbn

// Sub-images of one cluster size K (pbn_cluster.cu), concatenated on the device.
struct ClusterImages {
    int K = 0;
    uint8_t* d_buf = nullptr;
    uint32_t off[pbn::kMaxCluster] = {}, bytes[pbn::kMaxCluster] = {}, reloc_off[pbn::kMaxCluster] = {};
    int32_t reloc_count[pbn::kMaxCluster] = {};
    int32_t q_lo[pbn::kMaxCluster + 1] = {};
    uint32_t max_bytes = 0;
};

// Packed sub-images of one cluster size K for the lanes-over-nodes kernel
// (pbn_nodepar.cu): rank r owns packed state words [w_lo[r], w_lo[r+1]).
struct NodeParImages {
    int K = 0;
    uint8_t* d_buf = nullptr;
    uint32_t off[pbn::kMaxCluster] = {}, bytes[pbn::kMaxCluster] = {}, reloc_off[pbn::kMaxCluster] = {};
    int32_t reloc_count[pbn::kMaxCluster] = {};
    int32_t w_lo[pbn::kMaxCluster + 1] = {};
    uint32_t max_bytes = 0;
};

struct pbn_model_s {
    int device = 0;
    pbn::ImageLayout L;
    uint8_t* d_image = nullptr;
    uint32_t Tp = 0;
    uint32_t flags = 0;
    int64_t n_parents = 0;
    std::vector<ClusterImages> clusters;  // K = 2, 4, 8, 16 (K <= quads)
    std::vector<NodeParImages> nodepar;   // K = 1, 2, 4, 8, 16 (K <= packed words)
    // bit-sliced evaluation image (K1b), when every function has <= 6 parents
    // and every node <= 4 functions (pbn_internal.h)
    uint8_t* d_bs = nullptr;
    uint32_t bs_bytes = 0, bs_erec_off = 0, bs_rounds_off = 0;
    int32_t bs_rounds = 0, bs_L = 0, bs_cmax = 0;
    // its sub-images for cluster launches (K1bc): K = 2, 4, 8, 16
    struct BsCluster {
        int K = 0;
        uint8_t* d_buf = nullptr;
        uint32_t off[pbn::kMaxCluster] = {}, bytes[pbn::kMaxCluster] = {}, erec_off[pbn::kMaxCluster] = {},
                 rounds_off[pbn::kMaxCluster] = {};
        int32_t rounds[pbn::kMaxCluster] = {};
        int32_t qlo[pbn::kMaxCluster + 1] = {};
        uint32_t max_bytes = 0;
        int32_t max_lq = 0;
    };
    std::vector<BsCluster> bs_clusters;
    uint32_t geo_last = 0;                // geometric mode: Cg[n-1]
    uint32_t geo_off = 0;                 // geometric mode: byte offset of Cg in the image
    double p = 0.0;
};

namespace {

void set_err(char* err, size_t errlen, const char* fmt, ...)
{
    if (!err || errlen == 0) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
}

constexpr uint64_t kTwo32 = 1ull << 32;

// pbn_last_kernel(): the kernel of this thread's last successful launch
thread_local const char* g_last_kernel = "";

uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

// ---------------------------------------------------------------------
// Reading Q3: the 32-bit word scheme.  T_p = floor(p 2^32); for the j-th
// cumulative selection probability C_j (left-to-right fp64 sum) of a node,
// Q_j = min(floor(C_j 2^32), 2^32) and D_j = T_p + floor(Q_j (2^32 - T_p) / 2^32).
// Function j (0-based) is chosen iff D_j <= u < D_{j+1}; the kernel uses
// E_j = D_j - 1 and counts j = #{k : u > E_k}.
// ---------------------------------------------------------------------
uint32_t quantise_p(double p) { return (uint32_t)std::floor(std::ldexp(p, 32)); }

uint32_t boundary_E(double cum, uint32_t Tp)
{
    double q = std::floor(std::ldexp(cum, 32));
    uint64_t Q = q >= (double)kTwo32 ? kTwo32 : (uint64_t)q;
    const unsigned __int128 prod = (unsigned __int128)Q * (unsigned __int128)(kTwo32 - Tp);
    const uint64_t D = (uint64_t)Tp + (uint64_t)(prod >> 32);  // 1 <= D <= 2^32
    return (uint32_t)(D - 1);
}

pbn_status validate(const pbn_model_desc* d, char* err, size_t errlen)
{
    if (!d) {
        set_err(err, errlen, "null model description");
        return PBN_E_INVALID;
    }
    if (d->n < 1) {
        set_err(err, errlen, "n must be >= 1 (got %d)", d->n);
        return PBN_E_INVALID;
    }
    if (!d->fn_off || !d->par_off || !d->tbl_off || !d->tables || !d->sel_prob) {
        set_err(err, errlen, "null array in model description");
        return PBN_E_INVALID;
    }
    if (!(d->p >= std::ldexp(1.0, -32) && d->p < 1.0)) {
        set_err(err, errlen, "perturbation p must satisfy 2^-32 <= p < 1 (got %.17g)", d->p);
        return PBN_E_INVALID;
    }
    if (d->flags > PBN_PERTURB_GEOMETRIC) {
        set_err(err, errlen, "unknown flags %u (VECTOR, PER_NODE or GEOMETRIC)", d->flags);
        return PBN_E_INVALID;
    }
    if (d->fn_off[0] != 0) {
        set_err(err, errlen, "fn_off[0] must be 0");
        return PBN_E_INVALID;
    }
    for (int32_t i = 0; i < d->n; ++i) {
        const int32_t f0 = d->fn_off[i], f1 = d->fn_off[i + 1];
        if (f1 <= f0) {
            set_err(err, errlen, "node %d: needs at least one predictor function (ell >= 1)", i);
            return PBN_E_INVALID;
        }
        double sum = 0.0;
        for (int32_t f = f0; f < f1; ++f) {
            const double c = d->sel_prob[f];
            if (!(c > 0.0 && c <= 1.0)) {
                set_err(err, errlen, "node %d: selection probability of function %d must be in (0,1] (got %.17g)",
                        i, f - f0, c);
                return PBN_E_INVALID;
            }
            sum += c;
            const int32_t p0 = d->par_off[f], p1 = d->par_off[f + 1];
            if (p1 < p0) {
                set_err(err, errlen, "node %d: function %d has negative parent count", i, f - f0);
                return PBN_E_INVALID;
            }
            const int32_t theta = p1 - p0;
            if (theta > 0 && !d->parents) {
                set_err(err, errlen, "null parents array");
                return PBN_E_INVALID;
            }
            for (int32_t a = p0; a < p1; ++a) {
                if ((int32_t)d->parents[a] >= d->n) {
                    set_err(err, errlen, "node %d: function %d parent %u out of range (n=%d)", i, f - f0,
                            (unsigned)d->parents[a], d->n);
                    return PBN_E_INVALID;
                }
                for (int32_t b = p0; b < a; ++b)
                    if (d->parents[a] == d->parents[b]) {
                        set_err(err, errlen, "node %d: function %d repeats parent %u", i, f - f0,
                                (unsigned)d->parents[a]);
                        return PBN_E_INVALID;
                    }
            }
            if (theta > 30) {
                set_err(err, errlen, "node %d: function %d has %d parents (> 30)", i, f - f0, theta);
                return PBN_E_INVALID;
            }
            const int64_t words = ((int64_t)1 << theta) <= 32 ? 1 : ((int64_t)1 << theta) / 32;
            if ((int64_t)d->tbl_off[f + 1] - d->tbl_off[f] != words) {
                set_err(err, errlen, "node %d: function %d table has %d words, expected %lld for %d parents", i,
                        f - f0, d->tbl_off[f + 1] - d->tbl_off[f], (long long)words, theta);
                return PBN_E_INVALID;
            }
        }
        if (std::fabs(sum - 1.0) > 1e-9) {
            set_err(err, errlen, "node %d: selection probabilities sum to %.17g, not 1 (+-1e-9)", i, sum);
            return PBN_E_INVALID;
        }
    }
    return PBN_OK;
}

// Limits of the device kernels (beyond model validity).
pbn_status check_device_limits(const pbn_model_desc* d, char* err, size_t errlen)
{
    if (d->n > PBN_MAX_NODES) {
        set_err(err, errlen, "n=%d exceeds PBN_MAX_NODES=%d of this build", d->n, PBN_MAX_NODES);
        return PBN_E_USAGE;
    }
    const int32_t nf = d->fn_off[d->n];
    if (nf >= (1 << 20)) {
        set_err(err, errlen, "%d predictor functions exceed 2^20-1", nf);
        return PBN_E_USAGE;
    }
    for (int32_t i = 0; i < d->n; ++i) {
        const int32_t ell = d->fn_off[i + 1] - d->fn_off[i];
        if (ell > PBN_MAX_ELL) {
            set_err(err, errlen, "node %d: %d functions exceed PBN_MAX_ELL=%d", i, ell, PBN_MAX_ELL);
            return PBN_E_USAGE;
        }
        for (int32_t f = d->fn_off[i]; f < d->fn_off[i + 1]; ++f)
            if (d->par_off[f + 1] - d->par_off[f] > PBN_MAX_THETA) {
                set_err(err, errlen, "node %d: function with %d parents exceeds PBN_MAX_THETA=%d", i,
                        d->par_off[f + 1] - d->par_off[f], PBN_MAX_THETA);
                return PBN_E_USAGE;
            }
    }
    return PBN_OK;
}

// Device image (layout: pbn_internal.h).
struct ImageBuilder {
    std::vector<uint8_t> buf;
    uint32_t alloc(size_t bytes, size_t align = 16)
    {
        size_t off = (buf.size() + align - 1) & ~(align - 1);
        buf.resize(off + bytes, 0);
        return (uint32_t)off;
    }
    uint32_t* u32(uint32_t off) { return reinterpret_cast<uint32_t*>(buf.data() + off); }
    uint16_t* u16(uint32_t off) { return reinterpret_cast<uint16_t*>(buf.data() + off); }
};

inline uint32_t reverse_bits(uint32_t x)
{
    uint32_t r = 0;
    for (int b = 0; b < 32; ++b) r |= ((x >> b) & 1u) << (31 - b);
    return r;
}

// Table entry idx of function f (parents[0] is the MSB of idx, reading Q5).
inline uint32_t table_bit(const pbn_model_desc* d, int32_t f, uint32_t idx)
{
    return (d->tables[d->tbl_off[f] + (int32_t)(idx >> 5)] >> (idx & 31u)) & 1u;
}

// Image of the nodes [node_lo, node_hi) (records at local index i - node_lo)
// for a group state whose quads are qs bytes apart (32: two buffers, pbn_traj;
// 48: three buffers, pbn_cluster).  The fast width FT and the slow-node
// count are model-wide, so every sub-image of a cluster uses one kernel.
std::vector<uint8_t> build_image(const pbn_model_desc* d, uint32_t Tp, pbn::ImageLayout* L, int32_t node_lo = 0,
                                 int32_t node_hi = -1, uint32_t qs = 32, bool packed = false, bool geo = false,
                                 double geo_p = 0.0, uint32_t* geo_off = nullptr)
{
    const int32_t n = d->n, nf = d->fn_off[n];
    if (node_hi < 0) node_hi = n;
    ImageBuilder B;
    std::vector<uint32_t> reloc;  // byte offsets of offset-valued words
    const uint32_t off_nrec = B.alloc(16u * (size_t)std::max(node_hi - node_lo, 1));
    std::vector<int32_t> thmax(n, 0);
    std::vector<char> fast(n, 0);
    int32_t max_ell = 0, max_theta = 0, slow = 0, FT = pbn::kFastMinTheta;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t ell = d->fn_off[i + 1] - d->fn_off[i];
        max_ell = std::max(max_ell, ell);
        for (int32_t f = d->fn_off[i]; f < d->fn_off[i + 1]; ++f)
            thmax[i] = std::max(thmax[i], d->par_off[f + 1] - d->par_off[f]);
        max_theta = std::max(max_theta, thmax[i]);
        fast[i] = ell <= pbn::kFastMaxEll && thmax[i] <= pbn::kFastMaxTheta;
        slow += !fast[i];
        if (fast[i]) FT = std::max(FT, thmax[i]);
    }
    L->n = n;
    L->nf = nf;
    L->max_theta = max_theta;
    L->max_ell = max_ell;
    L->slow_nodes = slow;
    L->fast_theta = FT;

    for (int32_t i = node_lo; i < node_hi; ++i) {
        const int32_t f0 = d->fn_off[i], f1 = d->fn_off[i + 1], ell = f1 - f0;
        // selection thresholds E_1..E_{ell-1} (reading Q3)
        std::vector<uint32_t> E;
        double cum = 0.0;
        for (int32_t j = 0; j + 1 < ell; ++j) {
            cum += d->sel_prob[f0 + j];
            E.push_back(boundary_E(cum, Tp));
        }
        uint32_t w3 = 0;  // nrec[i].w, written last (B.alloc may move the buffer)
        if (fast[i]) {
            const int32_t tm = FT;  // every fast function is padded to the model-wide FT
            const uint32_t ds = packed ? pbn::desc_bytes_packed(tm) : pbn::desc_bytes(tm);
            const uint32_t off_desc = B.alloc((size_t)ds * ell, 16);
            for (int32_t j = 0; j < ell; ++j) {
                const int32_t f = f0 + j;
                const int32_t theta = d->par_off[f + 1] - d->par_off[f];
                // table padded to FT index bits: dummy parents are the low bits
                const uint32_t entries = 1u << tm;
                std::vector<uint32_t> T((entries + 31) / 32, 0u);
                for (uint32_t idx = 0; idx < entries; ++idx)
                    T[idx >> 5] |= table_bit(d, f, idx >> (tm - theta)) << (idx & 31u);
                uint32_t* w = B.u32(off_desc + ds * (uint32_t)j);
                const uint32_t wbase = off_desc + ds * (uint32_t)j;
                if (packed) {
                    // lanes over nodes: parents as u16 node ids (the K1n state is
                    // bit-packed), so a descriptor is one 16-byte chunk (FT <= 5)
                    // plus table words -- half the lane-divergent shared-memory
                    // wavefronts of the u32 layout; pad parents read node 0
                    auto pid = [&](int32_t m) -> uint32_t {
                        return m < theta ? (uint32_t)d->parents[d->par_off[f] + m] : 0u;
                    };
                    const int32_t na = tm >= 7 ? 8 : tm;  // u16 parent slots
                    const int32_t a0 = tm >= 7 ? 0 : (tm == 6 ? 2 : 1);  // first word of the u16 pairs
                    for (int32_t m = 0; m < na; ++m) w[a0 + m / 2] |= pid(m) << (16 * (m & 1));
                    if (tm >= 7) {
                        for (size_t q = 0; q < T.size(); ++q) w[4 + q] = reverse_bits(T[q]);
                    } else {
                        w[0] = reverse_bits(T[0]);
                        if (tm == 6) w[1] = reverse_bits(T[1]);
                    }
                    continue;
                }
                auto par = [&](int32_t m) {
                    const uint32_t node = m < theta ? d->parents[d->par_off[f] + m] : 0u;
                    return packed ? node : pbn::state_off(node, qs);
                };
                if (tm >= 7) {
                    // {a[0..7] (a[7] padding when FT = 7), table words}
                    for (int32_t m = 0; m < 8; ++m) {
                        if (!packed) reloc.push_back((wbase + 4u * (uint32_t)m) | pbn::kRelocState);
                        w[m] = par(m < tm ? m : tm);
                    }
                    // stored bit-reversed per word: entry e at bit 31 - (e & 31)
                    for (size_t q = 0; q < T.size(); ++q) w[8 + q] = reverse_bits(T[q]);
                } else {
                    int k = 0;
                    w[k++] = reverse_bits(T[0]);
                    if (tm == 6) w[k++] = reverse_bits(T[1]);
                    // padded parent list, MSB first, relocated by the state base
                    for (int32_t m = 0; m < tm; ++m) {
                        if (!packed) reloc.push_back((wbase + 4u * (uint32_t)k) | pbn::kRelocState);
                        w[k++] = par(m);
                    }
                }
            }
            w3 = off_desc;
        } else {
            const uint32_t off_slow = B.alloc(16);
            // thresholds padded with 0xFFFFFFFF to whole 16-byte vectors (the
            // generic path scans them four at a time; u > 0xFFFFFFFF never holds)
            const size_t nthr = (std::max<size_t>(E.size(), 1) + 3) & ~(size_t)3;
            const uint32_t off_thr = B.alloc(4u * nthr, 16);
            for (size_t k = 0; k < nthr; ++k) B.u32(off_thr)[k] = k < E.size() ? E[k] : 0xFFFFFFFFu;
            const uint32_t off_gd = B.alloc(16u * ell);
            for (int32_t j = 0; j < ell; ++j) {
                const int32_t f = f0 + j;
                const int32_t theta = d->par_off[f + 1] - d->par_off[f];
                const int32_t words = d->tbl_off[f + 1] - d->tbl_off[f];
                const uint32_t off_t = B.alloc(4u * words, 4);
                for (int32_t w = 0; w < words; ++w) B.u32(off_t)[w] = d->tables[d->tbl_off[f] + w];
                // parent offsets 16-aligned and padded to whole 16-byte vectors
                // (the generic path reads them four at a time)
                const uint32_t off_p = B.alloc(16u * (size_t)((std::max(theta, 1) + 3) / 4), 16);
                for (int32_t m = 0; m < theta; ++m) {
                    const uint32_t node = d->parents[d->par_off[f] + m];
                    B.u32(off_p)[m] = packed ? node : pbn::state_off(node, qs);
                }
                uint32_t* gd = B.u32(off_gd + 16u * j);
                gd[0] = off_t;
                gd[1] = (uint32_t)theta;
                gd[2] = off_p;
                gd[3] = 0;
                reloc.push_back(off_gd + 16u * j);
                reloc.push_back(off_gd + 16u * j + 8u);
            }
            uint32_t* sr = B.u32(off_slow);
            sr[0] = off_thr;
            sr[1] = (uint32_t)ell;
            sr[2] = off_gd;
            sr[3] = (uint32_t)thmax[i];  // warp-uniform gather trip count
            reloc.push_back(off_slow);
            reloc.push_back(off_slow + 8u);
            w3 = off_slow | pbn::kSlowNode;
        }
        uint32_t* rec = B.u32(off_nrec + 16u * (uint32_t)(i - node_lo));
        for (int k = 0; k < 3; ++k) rec[k] = k < (int)E.size() ? E[k] : 0xFFFFFFFFu;
        rec[3] = w3;
        reloc.push_back(off_nrec + 16u * (uint32_t)(i - node_lo) + 12u);
    }
    if (geo) {
        // geometric-skip table Cg[g] = floor((1 - q^(g+1)) 2^32), q^(g+1) by
        // repeated fp64 multiplication (reading Q18)
        const uint32_t go = B.alloc(4u * (size_t)n, 16);
        if (geo_off) *geo_off = go;
        double q = 1.0 - geo_p, r = 1.0;
        for (int32_t g = 0; g < n; ++g) {
            r *= q;
            B.u32(go)[g] = (uint32_t)std::floor(std::ldexp(1.0 - r, 32));
        }
    }
    B.alloc(16);  // tail slack
    L->bytes = (uint32_t)B.buf.size();
    // relocation list after the image (not staged to shared memory)
    L->reloc_off = B.alloc(4u * std::max<size_t>(reloc.size(), 1), 16);
    L->reloc_count = (int32_t)reloc.size();
    std::memcpy(B.buf.data() + L->reloc_off, reloc.data(), 4u * reloc.size());
    B.alloc(16);
    return B.buf;
}

// BITSLICE image (layout: pbn_internal.h): per-quad selection thresholds,
// function tasks grouped by class c = max(theta, 1) in whole rounds of 32,
// and the round list (most expensive class first).  Returns false when the
// model is outside the bit-sliced kernel's shape (theta > 6, ell > 4, too
// many nodes for u16 offsets).
// (q_lo, q_hi: the quads of a cluster CTA's sub-image -- erec indexed by the
// local quad, tasks of its nodes only; -1 = all)
bool build_bitslice_image(const pbn_model_desc* d, uint32_t Tp, std::vector<uint8_t>& out, uint32_t* erec_off,
                          uint32_t* rounds_off, int32_t* n_rounds, int32_t* L_out, int32_t* cmax_out,
                          int32_t q_lo = -1, int32_t q_hi = -1)
{
    const int32_t n = d->n;
    if (n > pbn::kBitsliceMaxNodes) return false;
    int32_t L = 1;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t ell = d->fn_off[i + 1] - d->fn_off[i];
        if (ell > pbn::kBitsliceMaxEll) return false;
        L = std::max(L, ell);
        for (int32_t f = d->fn_off[i]; f < d->fn_off[i + 1]; ++f)
            if (d->par_off[f + 1] - d->par_off[f] > pbn::kBitsliceMaxTheta) return false;
    }
    const int32_t nq_all = (n + 3) / 4;
    if (q_lo < 0) {
        q_lo = 0;
        q_hi = nq_all;
    }
    const int32_t nq = q_hi - q_lo;
    // model-wide largest class (one kernel for every sub-image of a cluster)
    int32_t cmax = 1;
    for (int32_t f = 0; f < d->fn_off[n]; ++f) cmax = std::max(cmax, d->par_off[f + 1] - d->par_off[f]);
    ImageBuilder B;
    // thresholds E_1..E_{L-1} per quad, plane-major: [q][m] = {E_{m+1} of nodes 4q..4q+3}
    const uint32_t eo = B.alloc(16u * (size_t)std::max(nq * (L - 1), 1));
    for (int32_t i = 4 * q_lo; i < 4 * q_hi; ++i) {
        std::vector<uint32_t> E;
        if (i < n) {
            const int32_t f0 = d->fn_off[i], ell = d->fn_off[i + 1] - f0;
            double cum = 0.0;
            for (int32_t j = 0; j + 1 < ell; ++j) {
                cum += d->sel_prob[f0 + j];
                E.push_back(boundary_E(cum, Tp));
            }
        }
        for (int32_t m = 0; m + 1 < L; ++m)
            B.u32(eo + 16u * (uint32_t)(((i >> 2) - q_lo) * (L - 1) + m))[i & 3] =
                m < (int32_t)E.size() ? E[m] : 0xFFFFFFFFu;
    }
    // tasks by class
    std::vector<std::pair<int32_t, int32_t>> cls[pbn::kBitsliceMaxTheta + 1];  // (node, j)
    for (int32_t i = 4 * q_lo; i < std::min(n, 4 * q_hi); ++i)
        for (int32_t f = d->fn_off[i]; f < d->fn_off[i + 1]; ++f)
            cls[std::max(d->par_off[f + 1] - d->par_off[f], 1)].push_back({i, f - d->fn_off[i]});
    std::vector<std::pair<uint32_t, uint32_t>> rounds;  // (task offset, class)
    for (int32_t c = pbn::kBitsliceMaxTheta; c >= 1; --c) {
        if (cls[c].empty()) continue;
        const uint32_t T = c <= 5 ? 1u : (1u << c) / 32u;                 // table words
        const uint32_t stride = c <= 5 ? 16u : c <= 7 ? 32u : 64u;      // kernel: bs_stride
        const size_t cnt = (cls[c].size() + 31) & ~(size_t)31;
        const uint32_t to = B.alloc(stride * cnt, 16);
        for (size_t k = 0; k < cnt; ++k) {
            uint32_t* w = B.u32(to + stride * (uint32_t)k);
            uint16_t* h = B.u16(to + stride * (uint32_t)k + 4u * T);  // [state_off(i) | j, p_0 .. p_{c-1}]
            if (k >= cls[c].size()) {  // dummy task: table 0 contributes nothing
                h[0] = (uint16_t)(pbn::state_off((uint32_t)(4 * q_lo), pbn::kBitsliceQs) | 1u);  // the first own node, function 1
                continue;
            }
            const int32_t i = cls[c][k].first, j = cls[c][k].second, f = d->fn_off[i] + j;
            const int32_t theta = d->par_off[f + 1] - d->par_off[f];
            // table padded to c index bits: padding parents are the low bits
            for (uint32_t e = 0; e < (1u << c); ++e)
                w[e >> 5] |= table_bit(d, f, e >> (c - theta)) << (e & 31u);
            h[0] = (uint16_t)(pbn::state_off((uint32_t)i, pbn::kBitsliceQs) | (uint32_t)j);
            for (int32_t m = 0; m < c; ++m)
                h[1 + m] = (uint16_t)pbn::state_off(m < theta ? d->parents[d->par_off[f] + m] : 0u, pbn::kBitsliceQs);
        }
        for (size_t k = 0; k < cnt; k += 32) rounds.push_back({to + stride * (uint32_t)k, (uint32_t)c});
    }
    const uint32_t ro = B.alloc(8u * std::max<size_t>(rounds.size(), 1), 16);
    for (size_t r = 0; r < rounds.size(); ++r) {
        B.u32(ro)[2 * r] = rounds[r].first;
        B.u32(ro)[2 * r + 1] = rounds[r].second;
    }
    B.alloc(16);
    B.buf.resize((B.buf.size() + 15) & ~(size_t)15);
    out.swap(B.buf);
    *erec_off = eo;
    *rounds_off = ro;
    *n_rounds = (int32_t)rounds.size();
    *L_out = L;
    *cmax_out = cmax;
    return true;
}

pbn_status cuda_status(cudaError_t e, char* err, size_t errlen, const char* what)
{
    if (e == cudaSuccess) return PBN_OK;
    set_err(err, errlen, "%s: %s", what, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? PBN_E_NOMEM : PBN_E_CUDA;
}

// Declared Skart constants (reading Q11).
constexpr double kSkartClamp = 0.999999;

}  // namespace

// =====================================================================
// C ABI
// =====================================================================
extern "C" {

const char* pbn_version(void) { return "libpbnsim 0.1 sm_100a"; }

const char* pbn_last_kernel(void) { return g_last_kernel; }

pbn_status pbn_validate(const pbn_model_desc* desc, char* err, size_t errlen)
{
    return validate(desc, err, errlen);
}

pbn_status pbn_load(const pbn_model_desc* desc, int device, pbn_model* out, char* err, size_t errlen)
{
    if (!out) {
        set_err(err, errlen, "null output handle");
        return PBN_E_USAGE;
    }
    *out = nullptr;
    pbn_status st = validate(desc, err, errlen);
    if (st != PBN_OK) return st;
    st = check_device_limits(desc, err, errlen);
    if (st != PBN_OK) return st;
    if (device < 0) {
        cudaError_t e = cudaGetDevice(&device);
        if (e != cudaSuccess) return cuda_status(e, err, errlen, "cudaGetDevice");
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, err, errlen, "cudaSetDevice");
    auto* m = new pbn_model_s();
    m->device = device;
    m->flags = desc->flags;
    m->Tp = quantise_p(desc->p);
    m->p = desc->p;
    m->n_parents = desc->par_off[desc->fn_off[desc->n]];
    const bool geo = desc->flags == PBN_PERTURB_GEOMETRIC;
    // geometric mode: no per-node perturbation share in the thresholds (T_p = 0)
    const uint32_t Tsel = geo ? 0u : m->Tp;
    std::vector<uint8_t> img = build_image(desc, Tsel, &m->L, 0, -1, 32u, false, geo, desc->p, &m->geo_off);
    if (geo) std::memcpy(&m->geo_last, img.data() + m->geo_off + 4u * (uint32_t)(desc->n - 1), 4);
    e = cudaMalloc(&m->d_image, img.size());
    if (e != cudaSuccess) {
        delete m;
        return cuda_status(e, err, errlen, "cudaMalloc(image)");
    }
    e = cudaMemcpy(m->d_image, img.data(), img.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(m->d_image);
        delete m;
        return cuda_status(e, err, errlen, "cudaMemcpy(image)");
    }
    // bit-sliced evaluation image (K1b; every semantics -- geometric: the
    // thresholds without the T_p share, gamma from the skip stream)
    {
        std::vector<uint8_t> bs;
        if (build_bitslice_image(desc, Tsel, bs, &m->bs_erec_off, &m->bs_rounds_off, &m->bs_rounds, &m->bs_L,
                                 &m->bs_cmax)) {
            if (cudaMalloc(&m->d_bs, bs.size()) != cudaSuccess ||
                cudaMemcpy(m->d_bs, bs.data(), bs.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
                if (m->d_bs) cudaFree(m->d_bs);
                cudaFree(m->d_image);
                delete m;
                set_err(err, errlen, "bitslice image upload failed");
                return PBN_E_CUDA;
            }
            m->bs_bytes = (uint32_t)bs.size();
            const int32_t nq = (desc->n + 3) / 4;
            for (int K = 2; K <= pbn::kMaxCluster && K <= nq; K *= 2) {
                pbn_model_s::BsCluster bc;
                bc.K = K;
                std::vector<uint8_t> all;
                for (int r = 0; r <= K; ++r) bc.qlo[r] = (int32_t)((int64_t)nq * r / K);
                bool ok = true;
                for (int r = 0; r < K && ok; ++r) {
                    std::vector<uint8_t> sub;
                    int32_t L2 = 0, cm2 = 0;
                    ok = build_bitslice_image(desc, Tsel, sub, &bc.erec_off[r], &bc.rounds_off[r], &bc.rounds[r], &L2, &cm2,
                                              bc.qlo[r], bc.qlo[r + 1]);
                    const size_t off = (all.size() + 15) & ~(size_t)15;
                    all.resize(off + sub.size(), 0);
                    std::memcpy(all.data() + off, sub.data(), sub.size());
                    bc.off[r] = (uint32_t)off;
                    bc.bytes[r] = (uint32_t)sub.size();
                    bc.max_bytes = std::max(bc.max_bytes, bc.bytes[r]);
                    bc.max_lq = std::max(bc.max_lq, bc.qlo[r + 1] - bc.qlo[r]);
                }
                if (!ok) break;
                if (cudaMalloc(&bc.d_buf, all.size()) != cudaSuccess ||
                    cudaMemcpy(bc.d_buf, all.data(), all.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
                    if (bc.d_buf) cudaFree(bc.d_buf);
                    for (auto& c : m->bs_clusters) cudaFree(c.d_buf);
                    cudaFree(m->d_bs);
                    cudaFree(m->d_image);
                    delete m;
                    set_err(err, errlen, "bitslice cluster sub-image upload failed");
                    return PBN_E_CUDA;
                }
                m->bs_clusters.push_back(bc);
            }
        }
    }
    // sub-images for the cluster kernel: CTA r of a K-cluster owns quads
    // [Q r / K, Q (r+1) / K) and its nodes' records and descriptors
    const int32_t nq = (desc->n + 3) / 4;
    // the geometric-skip stream runs in K1 (the cluster and lanes-over-nodes
    // kernels draw gamma per node): no sub-images for it
    for (int K = 2; !geo && K <= pbn::kMaxCluster && K <= nq; K *= 2) {
        ClusterImages ci;
        ci.K = K;
        std::vector<uint8_t> all;
        for (int r = 0; r <= K; ++r) ci.q_lo[r] = (int32_t)((int64_t)nq * r / K);
        for (int r = 0; r < K; ++r) {
            pbn::ImageLayout Lr;
            const int32_t lo = 4 * ci.q_lo[r], hi = std::min(desc->n, 4 * ci.q_lo[r + 1]);
            std::vector<uint8_t> sub = build_image(desc, m->Tp, &Lr, lo, hi, 48u);
            const size_t off = (all.size() + 15) & ~(size_t)15;
            all.resize(off + sub.size(), 0);
            std::memcpy(all.data() + off, sub.data(), sub.size());
            ci.off[r] = (uint32_t)off;
            ci.bytes[r] = Lr.bytes;
            ci.reloc_off[r] = Lr.reloc_off;
            ci.reloc_count[r] = Lr.reloc_count;
            ci.max_bytes = std::max(ci.max_bytes, Lr.bytes);
        }
        if (cudaMalloc(&ci.d_buf, all.size()) != cudaSuccess ||
            cudaMemcpy(ci.d_buf, all.data(), all.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            if (ci.d_buf) cudaFree(ci.d_buf);
            for (auto& c : m->clusters) cudaFree(c.d_buf);
            if (m->d_bs) cudaFree(m->d_bs);
            for (auto& c : m->bs_clusters) cudaFree(c.d_buf);
            cudaFree(m->d_image);
            delete m;
            set_err(err, errlen, "cluster sub-image upload failed");
            return PBN_E_CUDA;
        }
        m->clusters.push_back(ci);
    }
    // packed sub-images for the lanes-over-nodes kernel: CTA r of a K-cluster
    // owns packed state words [W r / K, W (r+1) / K)
    const int32_t nw = (desc->n + 31) / 32;
    for (int K = 1; K <= pbn::kMaxCluster && K <= nw; K *= 2) {
        NodeParImages ni;
        ni.K = K;
        std::vector<uint8_t> all;
        for (int r = 0; r <= K; ++r) ni.w_lo[r] = (int32_t)((int64_t)nw * r / K);
        for (int r = 0; r < K; ++r) {
            pbn::ImageLayout Lr;
            const int32_t lo = 32 * ni.w_lo[r], hi = std::min(desc->n, 32 * ni.w_lo[r + 1]);
            std::vector<uint8_t> sub = build_image(desc, Tsel, &Lr, lo, hi, 32u, true);
            const size_t off = (all.size() + 15) & ~(size_t)15;
            all.resize(off + sub.size(), 0);
            std::memcpy(all.data() + off, sub.data(), sub.size());
            ni.off[r] = (uint32_t)off;
            ni.bytes[r] = Lr.bytes;
            ni.reloc_off[r] = Lr.reloc_off;
            ni.reloc_count[r] = Lr.reloc_count;
            ni.max_bytes = std::max(ni.max_bytes, Lr.bytes);
        }
        if (cudaMalloc(&ni.d_buf, all.size()) != cudaSuccess ||
            cudaMemcpy(ni.d_buf, all.data(), all.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            if (ni.d_buf) cudaFree(ni.d_buf);
            for (auto& c : m->nodepar) cudaFree(c.d_buf);
            for (auto& c : m->clusters) cudaFree(c.d_buf);
            if (m->d_bs) cudaFree(m->d_bs);
            for (auto& c : m->bs_clusters) cudaFree(c.d_buf);
            cudaFree(m->d_image);
            delete m;
            set_err(err, errlen, "node-parallel sub-image upload failed");
            return PBN_E_CUDA;
        }
        m->nodepar.push_back(ni);
    }
    *out = m;
    return PBN_OK;
}

void pbn_free(pbn_model model)
{
    if (!model) return;
    if (model->d_image) cudaFree(model->d_image);
    if (model->d_bs) cudaFree(model->d_bs);
    for (auto& c : model->bs_clusters) cudaFree(c.d_buf);
    for (auto& c : model->clusters) cudaFree(c.d_buf);
    for (auto& c : model->nodepar) cudaFree(c.d_buf);
    delete model;
}

pbn_status pbn_get_model_info(pbn_model m, pbn_model_info* info)
{
    if (!m || !info) return PBN_E_USAGE;
    info->n = m->L.n;
    info->nf = m->L.nf;
    info->n_parents = m->n_parents;
    info->density = (double)m->n_parents / (double)m->L.n;
    info->T_p = m->Tp;
    info->flags = m->flags;
    info->max_ell = m->L.max_ell;
    info->max_theta = m->L.max_theta;
    info->image_bytes = m->L.bytes;
    return PBN_OK;
}

static pbn_status fill_traj_params(pbn_model m, const pbn_sim_args* a, const pbn_sim_out* o,
                                   pbn::TrajParams* P)
{
    if (!m || !a || !o || !o->state) return PBN_E_USAGE;
    if (a->n_chains < 0 || a->chain_base < 0 || a->step0 < 0 || a->burn_in < 0 || a->steps < 0 ||
        a->batch < 0)
        return PBN_E_USAGE;
    if (a->chain_base + a->n_chains > (int64_t)kTwo32) return PBN_E_USAGE;
    if (a->steps >= (int64_t)kTwo32) return PBN_E_USAGE;  // u32 counters
    if (a->init && a->step0 != 0) return PBN_E_USAGE;
    if (a->n_props < 0 || a->n_props > PBN_MAX_PROPS || (a->n_props > 0 && !a->props)) return PBN_E_USAGE;
    const int nprops = a->n_props > 0 ? a->n_props : 1;
    const pbn_predicate* props = a->n_props > 0 ? a->props : &a->pred;
    for (int p = 0; p < nprops; ++p) {
        if (props[p].k < 0 || props[p].k > PBN_MAX_PRED) return PBN_E_USAGE;
        if (props[p].k > 0 && (!props[p].node || !props[p].value)) return PBN_E_USAGE;
    }
    if (a->steps > 0 && a->batch > 0 && !o->batch_sums) return PBN_E_USAGE;
    if (a->steps > 0 && a->emit_bits && !o->bits) return PBN_E_USAGE;
    if (a->bits_offset < 0 || a->bits_row_words < 0) return PBN_E_USAGE;
    if (a->groups_per_cta > 1) return PBN_E_USAGE;  // one 32-chain group per CTA
    std::memset(P, 0, sizeof(*P));
    P->image = m->d_image;
    P->L = m->L;
    P->per_node = m->flags == PBN_PERTURB_PER_NODE;
    P->geometric = m->flags == PBN_PERTURB_GEOMETRIC ? 1 : 0;
    // geometric mode: gamma comes from the skip stream, never from u < T_p
    P->Tp = P->geometric ? 0u : m->Tp;
    P->geo_inv_lnq = P->geometric ? (float)(1.0 / std::log1p(-m->p)) : 0.0f;
    P->geo_off = m->geo_off;
    P->n = m->L.n;
    P->nquads = (m->L.n + 3) / 4;
    P->n_pad = (m->L.n + 3) & ~3;
    P->state_words = (m->L.n + 31) / 32;
    // group state (2 interleaved buffers) + gamma words + [32] any words, 16-aligned
    P->group_words = ((P->per_node ? 2 : 3) * P->n_pad + 32 + 3) & ~3;
    // Philox4x32-10 key schedule: round r uses (k0 + r W0, k1 + r W1), key = seed
    for (uint32_t r = 0; r < 10; ++r) {
        P->rk[2 * r + 0] = (uint32_t)a->seed + r * 0x9E3779B9u;
        P->rk[2 * r + 1] = (uint32_t)(a->seed >> 32) + r * 0xBB67AE85u;
    }
    P->n_chains = a->n_chains;
    P->chain_base = a->chain_base;
    P->step0 = a->step0;
    P->burn_in = a->burn_in;
    P->steps = a->steps;
    P->batch = a->batch;
    P->init = a->init ? 1 : 0;
    P->emit_bits = a->emit_bits ? 1 : 0;
    P->n_props = nprops;
    for (int p = 0; p < nprops; ++p) {
        P->pred_k[p] = props[p].k;
        for (int k = 0; k < props[p].k; ++k) {
            if ((int32_t)props[p].node[k] >= m->L.n || props[p].value[k] > 1) return PBN_E_INVALID;
            P->pred_node[p][k] = props[p].node[k];
            P->pred_val[p][k] = props[p].value[k];
        }
    }
    P->batch_row = a->batch > 0 ? (a->steps + a->batch - 1) / a->batch : 0;
    const int64_t need_words = (a->bits_offset + a->steps + 31) / 32;
    P->bits_row = a->bits_row_words > 0 ? a->bits_row_words : (a->steps + 31) / 32;
    if (a->emit_bits && a->steps > 0 && P->bits_row < need_words) return PBN_E_USAGE;
    P->bits_offset = a->bits_offset;
    P->state = o->state;
    P->c1 = o->c1;
    P->n01 = o->n01;
    P->n10 = o->n10;
    P->first_last = o->first_last;
    P->batch_sums = o->batch_sums;
    P->bits = o->bits;
    P->totals = reinterpret_cast<unsigned long long*>(o->totals);
    return PBN_OK;
}

// K1b launch: one 32-chain group per CTA (persistent schedule as K1), the
// bitslice image staged into shared memory or read through L1/L2.
// PBN_E_USAGE when the model has no bitslice image (theta > 8, ell > 4,
// n > 5460) or its group state does not fit.
static pbn_status simulate_bitslice(pbn_model m, const pbn::TrajParams& P, const pbn_sim_args* a, void* stream,
                                    int smem_optin)
{
    if (!m->d_bs) return PBN_E_USAGE;
    pbn::BitsliceParams Bp;
    std::memset(&Bp, 0, sizeof(Bp));
    Bp.T = P;
    Bp.T.image = m->d_bs;
    Bp.T.group_words = pbn::bitslice_group_words(P.n_pad, m->bs_L);
    const size_t group_bytes = (size_t)Bp.T.group_words * 4;
    if (group_bytes + 64 > (size_t)smem_optin) return PBN_E_USAGE;
    // the image in shared memory when it fits beside the group state, else
    // through the read-only global path (L1/L2; PBN_FORCE_GLOBAL_IMAGE=1 forces it)
    const char* fg = std::getenv("PBN_FORCE_GLOBAL_IMAGE");
    const bool smem_image = !(fg && fg[0] == '1') && group_bytes + m->bs_bytes + 64 <= (size_t)smem_optin;
    Bp.T.image_smem_bytes = smem_image ? m->bs_bytes : 0u;
    Bp.erec_off = m->bs_erec_off;
    Bp.rounds_off = m->bs_rounds_off;
    Bp.n_rounds = m->bs_rounds;
    Bp.any_off = 12 * P.n_pad;
    Bp.sel_off = 12 * P.n_pad + 4 * pbn::kBitsliceAnyWords;
    Bp.sel_bytes = 4 * pbn::bitslice_pv(m->bs_L) * P.n_pad;
    Bp.pq_off = Bp.sel_off + 2 * Bp.sel_bytes;
    // 20 warps on the staged image, all 24 of the budget on the global image
    int W = a->warps_per_group > 0
                ? a->warps_per_group
                : std::min(smem_image ? pbn::kBitsliceSmallWarps : pbn::kBitsliceMaxWarps, std::max(P.nquads, 1));
    W = std::max(W, P.n_props);
    if (W > pbn::kBitsliceMaxWarps || W > std::max(P.nquads, P.n_props)) return PBN_E_USAGE;
    pbn::LaunchPlan plan;
    plan.warps_per_group = W;
    plan.node_warps = std::min(W, P.nquads);
    plan.stats_warp0 = 0;
    plan.ctas = (int)((P.n_chains + 31) / 32);
    Bp.rl_off = Bp.pq_off + 16 * (P.n_pad / 4 + 1);
    Bp.rl_stride = (m->bs_rounds + W - 1) / W + 9;
    plan.threads = 32 * W;
    plan.smem_bytes = group_bytes + (smem_image ? m->bs_bytes : 0u);
    plan.image_in_smem = smem_image;
    Bp.T.warps_per_group = W;
    Bp.T.node_warps = plan.node_warps;
    Bp.T.stats_warp0 = 0;
    if (a->schedule < 0 || a->schedule > 2 || a->chunk_steps < 0 || a->workspace_bytes < 0) return PBN_E_USAGE;
    if (P.geometric) Bp.geo_table = reinterpret_cast<const uint32_t*>(m->d_image + m->geo_off);
    const void* fn = pbn::pick_bitslice_kernel(P.per_node ? 1 : P.geometric ? 2 : 0, m->bs_L, smem_image ? 1 : 0,
                                               m->bs_cmax, plan.threads);
    const int rc = pbn::launch_group_units(Bp.T, fn, &Bp, plan, m->device, a->schedule, a->chunk_steps, a->workspace,
                                           (size_t)a->workspace_bytes, stream);
    if (rc == -2) return PBN_E_USAGE;
    if (rc == 0) g_last_kernel = smem_image ? "K1b" : "K1b-global";
    return rc == 0 ? PBN_OK : PBN_E_CUDA;
}

// K1bc launch: one 32-chain group per cluster of K CTAs (K1b's kernel with
// IMG = 2), each CTA staging its sub-image; K = cluster_size, or (0) the
// largest whose clusters all fit one wave on the SMs.  Returns PBN_E_USAGE
// when no K fits (the caller may fall back), `*launched` false.
static pbn_status simulate_bitslice_cluster(pbn_model m, const pbn::TrajParams& P, const pbn_sim_args* a, void* stream,
                                            int smem_optin, int sms, bool* launched)
{
    *launched = false;
    if (!m->d_bs || m->bs_clusters.empty()) return PBN_E_USAGE;
    const int64_t groups = (P.n_chains + 31) / 32;
    const pbn_model_s::BsCluster* use = nullptr;
    auto smem_of = [&](const pbn_model_s::BsCluster& c) {
        return (size_t)pbn::bitslice_group_words(P.n_pad, m->bs_L, c.max_lq) * 4 + c.max_bytes;
    };
    for (const auto& c : m->bs_clusters) {
        if (smem_of(c) + 64 > (size_t)smem_optin) continue;
        if (a->cluster_size >= 2) {
            if (c.K == a->cluster_size) use = &c;
        } else if (c.K <= 8 && c.max_lq >= 32 && groups * c.K <= sms) {
            // auto: the largest K <= 8 whose clusters fit one wave while every
            // CTA keeps >= 32 quads (measured, profiles/k1bc_r3w.txt: C5 / C4
            // 1024 chains K = 4 3.8e11 / 3.8e11 vs K1c 1.6e11 / 3.0e11; C3 2048
            // chains K = 2 4.3e11 vs 3.4e11; 256 chains K = 8 beats K1n by 7-16 %
            // and K = 16 loses; C2 (6 quads per CTA at K = 4) stays on K1c)
            use = &c;
        }
    }
    if (!use) return PBN_E_USAGE;
    pbn::BitsliceParams Bp;
    std::memset(&Bp, 0, sizeof(Bp));
    Bp.T = P;
    Bp.T.image = use->d_buf;
    Bp.T.group_words = pbn::bitslice_group_words(P.n_pad, m->bs_L, use->max_lq);
    Bp.T.image_smem_bytes = use->max_bytes;
    Bp.any_off = 12 * P.n_pad;
    Bp.sel_off = 12 * P.n_pad + 4 * pbn::kBitsliceAnyWords;
    Bp.sel_bytes = 16 * pbn::bitslice_pv(m->bs_L) * use->max_lq;
    Bp.pq_off = Bp.sel_off + 2 * Bp.sel_bytes;
    Bp.K = use->K;
    for (int r = 0; r < use->K; ++r) {
        Bp.c_img_off[r] = use->off[r];
        Bp.c_img_bytes[r] = use->bytes[r];
        Bp.c_erec_off[r] = use->erec_off[r];
        Bp.c_rounds_off[r] = use->rounds_off[r];
        Bp.c_rounds[r] = use->rounds[r];
    }
    for (int r = 0; r <= use->K; ++r) Bp.c_qlo[r] = use->qlo[r];
    if (P.geometric) Bp.geo_table = reinterpret_cast<const uint32_t*>(m->d_image + m->geo_off);
    int W = a->warps_per_group > 0 ? a->warps_per_group
                                   : std::min(pbn::kBitsliceSmallWarps, std::max(use->max_lq, 1));
    W = std::max(W, P.n_props);
    if (W > pbn::kBitsliceMaxWarps) return PBN_E_USAGE;
    Bp.T.warps_per_group = W;
    Bp.T.node_warps = std::min(W, std::max(use->max_lq, 1));
    Bp.T.stats_warp0 = 0;
    Bp.T.persistent = 0;
    {
        int32_t max_rounds = 0;
        for (int r = 0; r < use->K; ++r) max_rounds = std::max(max_rounds, use->rounds[r]);
        Bp.rl_off = Bp.pq_off + 16 * (use->max_lq + 1);
        Bp.rl_stride = (max_rounds + W - 1) / W + 9;
    }
    const size_t smem = smem_of(*use);
    const void* fn = pbn::pick_bitslice_kernel(P.per_node ? 1 : P.geometric ? 2 : 0, m->bs_L, 2, m->bs_cmax, 32 * W);
    cudaError_t e = pbn::ensure_func_smem(fn, smem, use->K > 8);
    if (e != cudaSuccess) return PBN_E_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(groups * use->K));
    cfg.blockDim = dim3((unsigned)(32 * W));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)use->K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int active = 0;
    {
        cudaLaunchConfig_t one = cfg;
        one.gridDim = dim3((unsigned)use->K);
        if (cudaOccupancyMaxActiveClusters(&active, fn, &one) != cudaSuccess || active < 1) {
            cudaGetLastError();
            return PBN_E_USAGE;
        }
    }
    void* args[] = {&Bp};
    e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return PBN_E_CUDA;
    *launched = true;
    g_last_kernel = "K1bc";
    return PBN_OK;
}

pbn_status pbn_simulate(pbn_model m, const pbn_sim_args* a, const pbn_sim_out* o, void* stream)
{
    pbn::TrajParams P;
    pbn_status st = fill_traj_params(m, a, o, &P);
    if (st != PBN_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (o->totals) {
        if (cudaMemsetAsync(o->totals, 0, 6 * sizeof(uint64_t) * (size_t)P.n_props, s) != cudaSuccess)
            return PBN_E_CUDA;
    }
    if (a->n_chains == 0) return PBN_OK;
    if (a->cluster_size < 0 || a->cluster_size > pbn::kMaxCluster) return PBN_E_USAGE;
    // ---- one CTA per group (K1) or a cluster of K CTAs per group (K1c) ----
    const int smem_optin = pbn::cached_device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, m->device);
    const int sms = pbn::cached_device_attr(cudaDevAttrMultiProcessorCount, m->device);
    if (smem_optin <= 0 || sms <= 0) return PBN_E_CUDA;
    const size_t limit = (size_t)smem_optin - 64;
    const int64_t groups = (a->n_chains + 31) / 32;
    if (a->layout < PBN_LAYOUT_AUTO || a->layout > PBN_LAYOUT_BITSLICE) return PBN_E_USAGE;
    if (a->layout == PBN_LAYOUT_BITSLICE) {
        if (a->chains_per_cluster != 0) return PBN_E_USAGE;
        if (a->cluster_size >= 2) {
            bool launched = false;
            return simulate_bitslice_cluster(m, P, a, stream, smem_optin, sms, &launched);
        }
        return simulate_bitslice(m, P, a, stream, smem_optin);
    }
    // auto: the bit-sliced kernel wherever the one-CTA-per-group kernel would
    // run (enough groups to fill the GPU) and the model has a bitslice image
    // that fits (C3 4.15e11 -> 5.9e11, C4 5.32e11 -> 6.4e11 node-updates/s);
    // cluster_size = 1 keeps asking for K1 itself
    if (a->layout == PBN_LAYOUT_AUTO && a->cluster_size == 0 && m->d_bs && 2 * groups > sms &&
        (size_t)pbn::bitslice_group_words(P.n_pad, m->bs_L) * 4 <= limit) {
        const char* nb = std::getenv("PBN_NO_BITSLICE");  // A/B knob: auto without K1b
        if (!(nb && nb[0] == '1')) return simulate_bitslice(m, P, a, stream, smem_optin);
    }
    // ---- lanes over nodes (K1n): G chains per cluster of K CTAs ----
    const int32_t nw = (P.n + 31) / 32;
    if (a->chains_per_cluster < 0 || a->chains_per_cluster > 32) return PBN_E_USAGE;
    auto np_fits = [&](const NodeParImages& ni, int G) {
        return pbn::nodepar_smem_bytes(nw, G, ni.max_bytes) <= limit;
    };
    // chains per cluster: enough to put one CTA on every SM (a wave of
    // clusters), at most 32 and what the shared memory holds
    auto np_G = [&](const NodeParImages& ni) {
        int G = a->chains_per_cluster;
        if (G == 0) G = (int)std::min<int64_t>(32, std::max<int64_t>(1, (a->n_chains * ni.K + sms - 1) / sms));
        while (G > 1 && !np_fits(ni, G)) --G;
        return G;
    };
    // auto cluster size: the smallest K whose sub-image fits, raised while
    // the clusters still fit one wave on the SMs and every CTA keeps >= 4
    // packed words (128 nodes) -- measured (profiles/nodelanes_r2.jsonl):
    // 1 chain of C3-C5 is fastest at K = 8-16, 64 chains at K = 2 (C5: the
    // fitting 4), 256 chains at the smallest fitting K with G = 2
    auto np_auto = [&]() -> const NodeParImages* {
        const NodeParImages* use = nullptr;
        for (const auto& ni : m->nodepar) {
            if (!np_fits(ni, 1)) continue;
            if (!use || (a->n_chains * ni.K <= sms && nw >= 4 * ni.K)) use = &ni;
        }
        return use;
    };
    // auto layout (cluster_size 0): lanes over nodes for few chains --
    // measured faster than the chain-lanes kernels up to 256 chains
    // (profiles/nodelanes_auto_r2.jsonl; at 1024 chains K1c / K1 win)
    // (<= 128 chains when K1bc applies: at 256 chains it beats K1n, at 64 K1n
    // wins by 2.3x -- profiles/k1bc_r3w.txt)
    bool bc_applies = false;
    for (const auto& c : m->bs_clusters)
        bc_applies |= c.K <= 8 && c.max_lq >= 32 && groups * c.K <= sms &&
                      (size_t)pbn::bitslice_group_words(P.n_pad, m->bs_L, c.max_lq) * 4 + c.max_bytes <= limit;
    const bool node_lanes = a->layout == PBN_LAYOUT_NODE_LANES ||
                            (a->layout == PBN_LAYOUT_AUTO && a->cluster_size == 0 &&
                             a->n_chains <= (bc_applies ? 128 : 256));
    const NodeParImages* np_use = nullptr;
    if (node_lanes) {
        if (a->cluster_size >= 1) {
            for (const auto& ni : m->nodepar)
                if (ni.K == a->cluster_size) np_use = &ni;
            if (!np_use || !np_fits(*np_use, 1)) return PBN_E_USAGE;
        } else {
            np_use = np_auto();
            if (!np_use && a->layout == PBN_LAYOUT_NODE_LANES) return PBN_E_USAGE;
        }
    }
    if (np_use) {
        pbn::NodeParParams C;
        std::memset(&C, 0, sizeof(C));
        C.T = P;
        C.T.image = np_use->d_buf;
        C.K = np_use->K;
        C.G = np_G(*np_use);
        if (P.geometric) {
            C.geo_table = reinterpret_cast<const uint32_t*>(m->d_image + m->geo_off);
            C.geo_last = m->geo_last;
        }
        if (a->chains_per_cluster > 0 && C.G != a->chains_per_cluster) return PBN_E_USAGE;
        C.n_words = nw;
        int ow = 0;
        for (int r = 0; r < np_use->K; ++r) {
            C.img_off[r] = np_use->off[r];
            C.img_bytes[r] = np_use->bytes[r];
            C.reloc_off[r] = np_use->reloc_off[r];
            C.reloc_count[r] = np_use->reloc_count[r];
            ow = std::max(ow, np_use->w_lo[r + 1] - np_use->w_lo[r]);
        }
        for (int r = 0; r <= np_use->K; ++r) C.w_lo[r] = np_use->w_lo[r];
        // one warp per (chain, own word) -- up to 32 warps, which then loop;
        // the geometric stream adds a warp that only draws gamma(t+1)
        auto threads_for = [&](int G) {
            int t = std::min(1024, 32 * (G * ow + (P.geometric ? 1 : 0)));
            if (a->warps_per_group > 0) t = std::min(1024, 32 * a->warps_per_group);
            return std::max(t, 32 * P.n_props);
        };
        if (a->chains_per_cluster == 0) {
            // auto G: the smallest G (from one CTA per SM upward) whose
            // clusters all fit one wave -- clusters pack per GPC, so e.g. at
            // most 32 clusters of 4 are resident on 148 SMs (C5, 256 chains:
            // G = 7 -> 37 clusters, two waves, 6.3e10; G = 8 -> 1.12e11)
                for (int G = C.G; G <= 32 && np_fits(*np_use, G); ++G) {
                C.G = G;
                C.share = (int)(G * ow > threads_for(G) / 32);
                int active = 0;
                const int64_t clusters = (a->n_chains + G - 1) / G;
                if (pbn::max_active_nodepar_clusters(C, threads_for(G), pbn::nodepar_smem_bytes(nw, G, np_use->max_bytes),
                                                     &active) != 0) {
                    cudaGetLastError();
                    break;
                }
                if (clusters <= active) break;
            }
        }
        const int threads = threads_for(C.G);
        // warps with >= 2 (chain, word) items per step share Philox calls
        C.share = (int)(C.G * ow > threads / 32);
        const size_t smem = pbn::nodepar_smem_bytes(nw, C.G, np_use->max_bytes);
        const int rc = pbn::launch_traj_nodepar(C, threads, smem, stream);
        if (rc == 0) g_last_kernel = "K1n";
        return rc == 0 ? PBN_OK : PBN_E_CUDA;
    }
    auto fits = [&](const ClusterImages& ci) { return pbn::cluster_smem_bytes(P, ci.max_bytes) <= limit; };
    const ClusterImages* use = nullptr;
    if (a->cluster_size >= 2) {
        for (const auto& ci : m->clusters)
            if (ci.K == a->cluster_size) use = &ci;
        if (!use || !fits(*use)) return PBN_E_USAGE;
    } else if (a->cluster_size == 0 && 2 * groups <= sms) {
        // few groups: the bit-sliced kernel over a cluster per group when it
        // applies (K1bc), else K1c below
        if (a->layout == PBN_LAYOUT_AUTO) {
            const char* nb = std::getenv("PBN_NO_BITSLICE");
            if (!(nb && nb[0] == '1')) {
                bool launched = false;
                const pbn_status sb = simulate_bitslice_cluster(m, P, a, stream, smem_optin, sms, &launched);
                if (launched || sb == PBN_E_CUDA) return sb;
            }
        }
        // few-chain regime: one CTA per group would leave at least half the
        // SMs idle, so split each group's nodes over a cluster (measured: C3,
        // 64 groups: K = 2 1.6x the single-CTA kernel; 128 groups: single-CTA
        // 1.24x K = 2; with a full wave the single-CTA kernel wins even when
        // its image is read through L1/L2, profiles/sweep_c5_r1.jsonl)
        // the largest fitting K whose groups x K CTAs still fit one wave on
        // the SMs; if even the smallest fitting K does not, that smallest K
        // (each CTA keeps >= 3 quads: below that the per-step cluster barrier
        // dominates -- C2, 25 quads: K = 8 beats K = 16 by 20 %)
        const ClusterImages* smallest = nullptr;
        for (const auto& ci : m->clusters) {
            if (!fits(ci) || 3 * ci.K > (P.n + 3) / 4) continue;
            if (!smallest) smallest = &ci;
            if (groups * ci.K <= sms) use = &ci;
        }
        if (!use) use = smallest;
    }
    if (use) {
        pbn::ClusterParams C;
        std::memset(&C, 0, sizeof(C));
        C.T = P;
        C.T.image = use->d_buf;
        C.K = use->K;
        for (int r = 0; r < use->K; ++r) {
            C.img_off[r] = use->off[r];
            C.img_bytes[r] = use->bytes[r];
            C.reloc_off[r] = use->reloc_off[r];
            C.reloc_count[r] = use->reloc_count[r];
        }
        for (int r = 0; r <= use->K; ++r) C.q_lo[r] = use->q_lo[r];
        int qmax = 0;
        for (int r = 0; r < use->K; ++r) qmax = std::max(qmax, use->q_lo[r + 1] - use->q_lo[r]);
        int W = a->warps_per_group > 0 ? a->warps_per_group : std::min(pbn::kMaxWarpsPerCta, std::max(qmax, 1));
        W = std::max(W, P.n_props);
        if (W > pbn::kMaxWarpsPerCta) return PBN_E_USAGE;
        C.T.warps_per_group = W;
        const size_t smem = pbn::cluster_smem_bytes(P, use->max_bytes);
        int active = 0;
        if (pbn::max_active_clusters(C, W, smem, &active) != 0 || active < 1) {
            // a forced cluster size must run as asked; in auto mode fall
            // through to the one-CTA-per-group kernel (its image in shared
            // memory or, when it does not fit, read through L1/L2)
            cudaGetLastError();
            if (a->cluster_size >= 2) return PBN_E_USAGE;
        } else {
            const int rc = pbn::launch_traj_cluster(C, W, smem, stream);
            if (rc == 0) g_last_kernel = "K1c";
            return rc == 0 ? PBN_OK : PBN_E_CUDA;
        }
    }
    pbn::LaunchPlan plan;
    const char* why = nullptr;
    int rc = pbn::plan_traj_launch(P, m->device, a->warps_per_group, &plan, &why);
    if (rc < 0) return PBN_E_USAGE;
    if (rc > 0) return PBN_E_CUDA;
    if (a->schedule < 0 || a->schedule > 2 || a->chunk_steps < 0) return PBN_E_USAGE;
    if (a->workspace_bytes < 0) return PBN_E_USAGE;
    rc = pbn::launch_traj(P, plan, m->device, a->schedule, a->chunk_steps, a->workspace, (size_t)a->workspace_bytes,
                          stream);
    if (rc == -2) return PBN_E_USAGE;
    if (rc == 0) g_last_kernel = plan.image_in_smem ? "K1" : "K1-global";
    return rc == 0 ? PBN_OK : PBN_E_CUDA;
}

pbn_status pbn_simulate_workspace_size(pbn_model m, const pbn_sim_args* a, int64_t* bytes)
{
    if (!bytes) return PBN_E_USAGE;
    *bytes = 0;
    if (!m || !a || a->n_chains < 0 || a->n_props < 0 || a->n_props > PBN_MAX_PROPS) return PBN_E_USAGE;
    pbn::TrajParams P;
    std::memset(&P, 0, sizeof(P));
    P.n_chains = a->n_chains;
    P.n_pad = (m->L.n + 3) & ~3;
    P.n_props = a->n_props > 0 ? a->n_props : 1;
    *bytes = a->n_chains > 0 ? (int64_t)pbn::traj_workspace_bytes(P) : 0;
    return PBN_OK;
}

pbn_status pbn_recount(const uint32_t* bits, int64_t n_chains, int64_t row_words, int64_t start,
                       int64_t length, int64_t batch, uint32_t* c1, uint32_t* n01, uint32_t* n10,
                       uint8_t* first_last, uint32_t* batch_sums, uint64_t* totals, void* stream)
{
    if (!bits || n_chains < 0 || row_words <= 0 || start < 0 || length < 0 || batch < 0)
        return PBN_E_USAGE;
    if ((start + length + 31) / 32 > row_words) return PBN_E_USAGE;
    if (batch > 0 && !batch_sums) return PBN_E_USAGE;
    cudaStream_t s = (cudaStream_t)stream;
    if (totals && cudaMemsetAsync(totals, 0, 6 * sizeof(uint64_t), s) != cudaSuccess) return PBN_E_CUDA;
    pbn::RecountParams R;
    R.bits = bits;
    R.n_chains = n_chains;
    R.row_words = row_words;
    R.start = start;
    R.length = length;
    R.batch = batch;
    R.batch_row = batch > 0 ? (length + batch - 1) / batch : 0;
    R.c1 = c1;
    R.n01 = n01;
    R.n10 = n10;
    R.first_last = first_last;
    R.batch_sums = batch_sums;
    R.totals = reinterpret_cast<unsigned long long*>(totals);
    return pbn::launch_recount(R, stream) == 0 ? PBN_OK : PBN_E_CUDA;
}

// ---------------------------------------------------------------------
// Gelman & Rubin (Alg 3) from exact integer sums:
//   B = (omega S2 - S1^2) / (omega psi (omega-1))
//   W = (psi S1 - S2) / (omega psi (psi-1))
// both numerators formed exactly in 128-bit integers.
// ---------------------------------------------------------------------
pbn_status pbn_gelman_rubin(uint64_t S1, uint64_t S2, int64_t omega, int64_t psi, double* rhat,
                            double* B, double* W, double* sigma2)
{
    if (omega < 2 || psi < 2) return PBN_E_USAGE;
    const unsigned __int128 om = (unsigned __int128)omega, ps = (unsigned __int128)psi;
    const unsigned __int128 s1 = S1, s2 = S2;
    const unsigned __int128 bn_a = om * s2, bn_b = s1 * s1;
    const unsigned __int128 wn_a = ps * s1;
    if (bn_a < bn_b || wn_a < s2) return PBN_E_USAGE;  // inconsistent sums
    const double Bv = (double)(bn_a - bn_b) / ((double)omega * (double)psi * (double)(omega - 1));
    const double Wv = (double)(wn_a - s2) / ((double)omega * (double)psi * (double)(psi - 1));
    const double s2v = (1.0 - 1.0 / (double)psi) * Wv + Bv / (double)psi;
    if (B) *B = Bv;
    if (W) *W = Wv;
    if (sigma2) *sigma2 = s2v;
    if (Wv == 0.0) {
        if (rhat) *rhat = NAN;
        return PBN_E_DEGENERATE;
    }
    if (rhat) *rhat = std::sqrt(s2v / Wv);
    return PBN_OK;
}

// ---------------------------------------------------------------------
// Phi^-1: Abramowitz & Stegun 26.2.23 start, then Halley steps on erfc.
// ---------------------------------------------------------------------
double pbn_inv_norm_cdf(double q)
{
    if (!(q > 0.0 && q < 1.0)) return NAN;
    if (q > 0.5) return -pbn_inv_norm_cdf(1.0 - q);
    const double t = std::sqrt(-2.0 * std::log(q));
    double x = -(t - (2.515517 + 0.802853 * t + 0.010328 * t * t) /
                         (1.0 + 1.432788 * t + 0.189269 * t * t + 0.001308 * t * t * t));
    const double rt2pi = 2.5066282746310002;  // sqrt(2 pi)
    for (int it = 0; it < 4; ++it) {
        const double e = 0.5 * std::erfc(-x / 1.4142135623730951) - q;
        const double u = e * rt2pi * std::exp(0.5 * x * x);
        x = x - u / (1.0 + 0.5 * x * u);
    }
    return x;
}

// Regularised incomplete beta I_x(a,b) by the modified Lentz continued fraction.
static double betacf(double a, double b, double x)
{
    const double tiny = 1e-300, eps = 1e-16;
    double qab = a + b, qap = a + 1.0, qam = a - 1.0;
    double c = 1.0, d = 1.0 - qab * x / qap;
    if (std::fabs(d) < tiny) d = tiny;
    d = 1.0 / d;
    double h = d;
    for (int m = 1; m <= 10000; ++m) {
        const int m2 = 2 * m;
        double aa = m * (b - m) * x / ((qam + m2) * (a + m2));
        d = 1.0 + aa * d;
        if (std::fabs(d) < tiny) d = tiny;
        c = 1.0 + aa / c;
        if (std::fabs(c) < tiny) c = tiny;
        d = 1.0 / d;
        h *= d * c;
        aa = -(a + m) * (qab + m) * x / ((a + m2) * (qap + m2));
        d = 1.0 + aa * d;
        if (std::fabs(d) < tiny) d = tiny;
        c = 1.0 + aa / c;
        if (std::fabs(c) < tiny) c = tiny;
        d = 1.0 / d;
        const double del = d * c;
        h *= del;
        if (std::fabs(del - 1.0) < eps) break;
    }
    return h;
}

// Stirling remainder lgamma(z) - [(z-1/2) ln z - z + ln(2 pi)/2], z >= 10.
static double stirling_delta(double z)
{
    const double r = 1.0 / z, r2 = r * r;
    return r * (1.0 / 12.0 - r2 * (1.0 / 360.0 - r2 * (1.0 / 1260.0 - r2 * (1.0 / 1680.0))));
}

// lgamma(a+b) - lgamma(a) - lgamma(b) without cancellation when a is large.
static double log_inv_beta(double a, double b)
{
    if (a < 10.0) return std::lgamma(a + b) - std::lgamma(a) - std::lgamma(b);
    return (a - 0.5) * std::log1p(b / a) + b * std::log(a + b) - b + stirling_delta(a + b) -
           stirling_delta(a) - std::lgamma(b);
}

// I_x(a,b) given both x and y = 1 - x (each computed without cancellation).
static double inc_beta(double a, double b, double x, double y)
{
    if (x <= 0.0) return 0.0;
    if (y <= 0.0) return 1.0;
    const double big = std::max(a, b), small = std::min(a, b);
    const double lbt = log_inv_beta(big, small) + a * std::log(x) + b * std::log(y);
    const double bt = std::exp(lbt);
    if (x < (a + 1.0) / (a + b + 2.0)) return bt * betacf(a, b, x) / a;
    return 1.0 - bt * betacf(b, a, y) / b;
}

// Student-t lower tail probability P(T <= t) for t <= 0:
// 0.5 I_{df/(df+t^2)}(df/2, 1/2).
static double t_lower_tail(double t, double df)
{
    const double den = df + t * t;
    return 0.5 * inc_beta(0.5 * df, 0.5, df / den, (t * t) / den);
}

double pbn_t_quantile(double q, double df)
{
    if (!(q > 0.0 && q < 1.0) || !(df >= 1.0)) return NAN;
    if (q > 0.5) return -pbn_t_quantile(1.0 - q, df);
    if (q == 0.5) return 0.0;
    if (df == 1.0) return std::tan(M_PI * (q - 0.5));
    // Newton on the lower tail from the normal quantile, safeguarded by bisection
    double x = pbn_inv_norm_cdf(q);
    double lo = -1e300, hi = 0.0;
    const double lgc = std::lgamma(0.5 * (df + 1.0)) - std::lgamma(0.5 * df) - 0.5 * std::log(df * M_PI);
    for (int it = 0; it < 200; ++it) {
        const double F = t_lower_tail(x, df);
        const double f = F - q;
        if (f > 0.0) hi = std::min(hi, x);
        else lo = std::max(lo, x);
        const double pdf = std::exp(lgc - 0.5 * (df + 1.0) * std::log1p(x * x / df));
        double nx = x - f / pdf;
        if (!(nx > lo && nx < hi)) nx = (lo > -1e299) ? 0.5 * (lo + hi) : 2.0 * x - 1.0;
        if (std::fabs(nx - x) <= 1e-15 * std::max(1.0, std::fabs(x))) {
            x = nx;
            break;
        }
        x = nx;
    }
    return x;
}

pbn_status pbn_two_state(uint64_t n01, uint64_t n0from, uint64_t n10, uint64_t n1from, double r,
                         double s, double eps, pbn_two_state_result* res)
{
    if (!res || !(r > 0.0) || !(s > 0.0 && s < 1.0) || !(eps > 0.0)) return PBN_E_USAGE;
    res->alpha = res->beta = res->M_raw = res->N_raw = NAN;
    res->M = res->N = 0;
    if (n0from == 0 || n1from == 0) return PBN_E_DEGENERATE;
    const double a = (double)n01 / (double)n0from;
    const double b = (double)n10 / (double)n1from;
    res->alpha = a;
    res->beta = b;
    const double apb = a + b;
    if (apb == 0.0 || apb == 2.0) return PBN_E_DEGENERATE;
    const double lam = std::fabs(1.0 - apb);
    const double M_raw = lam == 0.0 ? 1.0 : std::log(eps * apb / std::max(a, b)) / std::log(lam);
    const double z = pbn_inv_norm_cdf(0.5 * (1.0 + s));
    const double N_raw = (a * b * (2.0 - apb) / (apb * apb * apb)) * (z * z / (r * r));
    res->M_raw = M_raw;
    res->N_raw = N_raw;
    res->M = (int64_t)std::ceil(M_raw);
    res->N = (int64_t)std::ceil(N_raw);
    return PBN_OK;
}

// ---------------------------------------------------------------------
// Skart CI (readings Q11/Q12) over chain-major batch means.
// ---------------------------------------------------------------------
pbn_status pbn_skart_ci_from_batches(const uint32_t* bs, int64_t omega, int64_t per_chain, int64_t kappa,
                                     double alpha_conf, pbn_skart_ci* res)
{
    if (!bs || !res || omega < 1 || per_chain < 1 || kappa < 1 || !(alpha_conf > 0.0 && alpha_conf < 1.0))
        return PBN_E_USAGE;
    const int64_t P = omega * per_chain;
    if (P < 3) return PBN_E_USAGE;
    // batch means and their moments (mean, variance with divisor P-1)
    long double sum = 0.0L;
    for (int64_t j = 0; j < P; ++j) sum += (long double)bs[j];
    const double mu = (double)(sum / (long double)P) / (double)kappa;
    double m2 = 0.0, m3 = 0.0, lag = 0.0;
    for (int64_t j = 0; j < P; ++j) {
        const double y = (double)bs[j] / (double)kappa - mu;
        m2 += y * y;
        m3 += y * y * y;
    }
    for (int64_t c = 0; c < omega; ++c)
        for (int64_t k = 0; k + 1 < per_chain; ++k) {  // no cross-chain pairs (Q12)
            const int64_t j = c * per_chain + k;
            lag += ((double)bs[j] / (double)kappa - mu) * ((double)bs[j + 1] / (double)kappa - mu);
        }
    res->batches = P;
    res->mu = mu;
    if (m2 == 0.0) {
        res->var = 0.0;
        res->phi = 0.0;
        res->skew = NAN;
        res->ci_lo = res->ci_hi = mu;
        res->H = 0.0;
        return PBN_E_DEGENERATE;
    }
    const double var = m2 / (double)(P - 1);
    double phi = lag / m2;
    phi = std::max(-kSkartClamp, std::min(kSkartClamp, phi));
    const double skew = (m3 / (double)P) / std::pow(m2 / (double)P, 1.5);
    const double A = (1.0 + phi) / (1.0 - phi);
    const double bhat = skew / (6.0 * std::sqrt((double)P));
    auto G = [bhat](double t) {
        if (bhat == 0.0) return t;
        return (std::cbrt(1.0 + 6.0 * bhat * (t - bhat)) - 1.0) / (2.0 * bhat);
    };
    const double df = (double)(P - 1);
    const double tl = pbn_t_quantile(0.5 * alpha_conf, df);
    const double tu = pbn_t_quantile(1.0 - 0.5 * alpha_conf, df);
    const double sc = std::sqrt(A * var / (double)P);
    res->var = var;
    res->phi = phi;
    res->skew = skew;
    res->ci_lo = mu + G(tl) * sc;
    res->ci_hi = mu + G(tu) * sc;
    res->H = std::max(mu - res->ci_lo, res->ci_hi - mu);
    return PBN_OK;
}

}  // extern "C"
