// pbn_skart.cpp -- the Skart sample-size state machine of Algorithm 5
// (parallelised Skart; Skart itself, Alg 2) over the
// pooled 0/1 indicator samples of omega chains, written once and used by
//   - pbn_skart (C ABI): over device bitstreams the caller owns, and
//   - the host driver (pbn_driver.cpp): over the driver's own bitstreams,
//     with the per-chain batch sums all-gathered across shards.
//
// The machine is a pure function of the sample prefix it reads: it replays
// Alg 5 lines 3-21 from the start over the first `avail` samples of every
// chain and stops at the first point that needs more (returning that
// per-chain length).  The caller extends the chains and calls again; since
// earlier decisions only read the unchanged prefix, the replay retakes them
// and the sequence of extensions equals a single pass's.
//
// Declared Skart constants (reading Q11 -- the paper defers
// Skart's internals to [AJE08]): skewness limit 4 (kappa 1, else 16;
// undefined skewness -> 16), von Neumann randomness test at level 0.20
// two-sided on spaced batch means, kappa <- ceil(sqrt(2) kappa) and spacer
// d <- d + 1 on failure, batch-count ceiling 1024 in the CI loop, exit when
// H <= H*.  Reading Q12: p is rounded up to a multiple of omega so batches
// never straddle chains (Fig. 2b); batch means are chain-major;
// lag-1 / successive differences never pair batches of different chains.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/pbnsim.h"
#include "pbn_internal.h"

namespace pbn {

pbn_status skart_machine(SkartSource& src, int64_t omega, int64_t avail, double h_star, double alpha_conf,
                         pbn_skart_result* res)
{
    std::memset(res, 0, sizeof(*res));
    res->estimate = res->ci_lo = res->ci_hi = res->H = res->skew = NAN;
    if (omega < 1 || avail < 0 || !(h_star > 0.0) || !(alpha_conf > 0.0 && alpha_conf < 1.0)) return PBN_E_USAGE;
    auto round_up = [omega](int64_t v) { return (v + omega - 1) / omega * omega; };
    auto need = [&](int64_t per_chain) {
        if (per_chain <= avail) return false;
        res->need_per_chain = per_chain;
        return true;
    };
    const double z_pass = pbn_inv_norm_cdf(1.0 - 0.20 / 2.0);
    int64_t eta = round_up(1280);  // Alg 5 line 3
    if (need(eta / omega)) return PBN_E_NOT_CONVERGED;
    // skewness of all eta samples (line 5): for 0/1 data (1 - 2m) / sqrt(m (1 - m))
    uint64_t ones = 0;
    pbn_status st = src.ones(eta / omega, &ones);
    if (st != PBN_OK) return st;
    const double m1 = (double)ones / (double)eta;
    const bool skew_defined = m1 > 0.0 && m1 < 1.0;
    res->skew = skew_defined ? (1.0 - 2.0 * m1) / std::sqrt(m1 * (1.0 - m1)) : NAN;
    int64_t kappa = (skew_defined && std::fabs(res->skew) <= 4.0) ? 1 : 16;
    int64_t p = round_up(eta);  // line 6
    eta = kappa * p;
    int64_t d = 0;
    std::vector<uint32_t> hbs;
    // lines 7-12: randomness (independence) test on spaced batch means
    for (int iter = 0;; ++iter) {
        if (iter >= 64) return PBN_E_NOT_CONVERGED;
        if (need(eta / omega)) return PBN_E_NOT_CONVERGED;
        const int64_t per = p / omega;
        if ((st = src.batch_sums(kappa, per, hbs)) != PBN_OK) return st;
        res->randomness_tests++;
        // spaced batch means: every (d+1)-th batch of each chain
        const int64_t kept = (per + d) / (d + 1);
        const int64_t pairs = omega * (kept - 1);
        bool pass = true;
        if (pairs >= 2) {
            const int64_t P = omega * kept;
            long double sum = 0.0L;
            for (int64_t ch = 0; ch < omega; ++ch)
                for (int64_t k = 0; k < kept; ++k) sum += hbs[(size_t)(ch * per + k * (d + 1))];
            const double mu = (double)(sum / (long double)P) / (double)kappa;
            double ss = 0.0, sd = 0.0;
            for (int64_t ch = 0; ch < omega; ++ch)
                for (int64_t k = 0; k < kept; ++k) {
                    const double y = (double)hbs[(size_t)(ch * per + k * (d + 1))] / (double)kappa;
                    ss += (y - mu) * (y - mu);
                    if (k > 0) {
                        const double yp = (double)hbs[(size_t)(ch * per + (k - 1) * (d + 1))] / (double)kappa;
                        sd += (y - yp) * (y - yp);
                    }
                }
            if (ss == 0.0) {
                pass = false;  // constant spaced means: no evidence of independence
            } else {
                const double Cst = (sd / (double)pairs) / (2.0 * ss / (double)(P - 1));
                const double mm = (double)(pairs + 1);
                const double z = (1.0 - Cst) * std::sqrt((mm * mm - 1.0) / (mm - 2.0));
                pass = std::fabs(z) <= z_pass;
            }
        }
        if (pass) break;
        kappa = (int64_t)std::ceil(std::sqrt(2.0) * (double)kappa);
        d += 1;
        p = round_up(p);
        eta = kappa * p;
    }
    // lines 13-21: CI loop on non-spaced batch means (no further discarding)
    for (int iter = 0;; ++iter) {
        if (iter >= 64) return PBN_E_NOT_CONVERGED;
        if (need(eta / omega)) return PBN_E_NOT_CONVERGED;
        const int64_t per = p / omega;
        if ((st = src.batch_sums(kappa, per, hbs)) != PBN_OK) return st;
        pbn_skart_ci ci;
        st = pbn_skart_ci_from_batches(hbs.data(), omega, per, kappa, alpha_conf, &ci);
        if (st != PBN_OK && st != PBN_E_DEGENERATE) return st;
        if (ci.H <= h_star) {
            res->estimate = ci.mu;
            res->ci_lo = ci.ci_lo;
            res->ci_hi = ci.ci_hi;
            res->H = ci.H;
            res->kappa = kappa;
            res->batches = p;
            res->spacer = d;
            res->eta = eta;
            res->need_per_chain = 0;
            return PBN_OK;
        }
        const double g = (ci.H / h_star) * (ci.H / h_star);
        const int64_t new_eta = (int64_t)std::ceil(g * (double)eta);
        if (p < 1024) p = std::min<int64_t>(1024, (int64_t)std::ceil(g * (double)p));
        p = round_up(p);
        kappa = std::max(kappa, (new_eta + p - 1) / p);
        eta = kappa * p;
    }
}

}  // namespace pbn

namespace {

// Sample source over caller-owned device bitstreams (one GPU).
struct DeviceBitsSource : pbn::SkartSource {
    const uint32_t* bits;
    int64_t omega, row_words, start;
    cudaStream_t s;
    uint32_t* d_batch = nullptr;
    int64_t cap = 0;
    uint64_t* d_tot = nullptr;
    ~DeviceBitsSource()
    {
        cudaFree(d_batch);
        cudaFree(d_tot);
    }
    pbn_status ones(int64_t len, uint64_t* S1) override
    {
        if (!d_tot && cudaMalloc(&d_tot, 6 * sizeof(uint64_t)) != cudaSuccess) return PBN_E_NOMEM;
        pbn_status st = pbn_recount(bits, omega, row_words, start, len, 0, nullptr, nullptr, nullptr, nullptr,
                                    nullptr, d_tot, s);
        if (st != PBN_OK) return st;
        uint64_t t[6];
        if (cudaMemcpyAsync(t, d_tot, sizeof(t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return PBN_E_CUDA;
        *S1 = t[0];
        return PBN_OK;
    }
    pbn_status batch_sums(int64_t kappa, int64_t per, std::vector<uint32_t>& out) override
    {
        const int64_t n = omega * per;
        if (n > cap) {
            cudaFree(d_batch);
            d_batch = nullptr;
            cap = 0;
            if (cudaMalloc(&d_batch, sizeof(uint32_t) * (size_t)n) != cudaSuccess) return PBN_E_NOMEM;
            cap = n;
        }
        pbn_status st = pbn_recount(bits, omega, row_words, start, kappa * per, kappa, nullptr, nullptr, nullptr,
                                    nullptr, d_batch, nullptr, s);
        if (st != PBN_OK) return st;
        out.resize((size_t)n);
        if (cudaMemcpyAsync(out.data(), d_batch, sizeof(uint32_t) * (size_t)n, cudaMemcpyDeviceToHost, s) !=
                cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return PBN_E_CUDA;
        return PBN_OK;
    }
};

}  // namespace

extern "C" pbn_status pbn_skart(const uint32_t* bits, int64_t omega, int64_t row_words, int64_t start,
                                int64_t available, double h_star, double alpha_conf, pbn_skart_result* res,
                                void* stream)
{
    if (!bits || !res || omega < 1 || row_words < 1 || start < 0 || available < 0) return PBN_E_USAGE;
    if ((start + available + 31) / 32 > row_words) return PBN_E_USAGE;
    DeviceBitsSource src;
    src.bits = bits;
    src.omega = omega;
    src.row_words = row_words;
    src.start = start;
    src.s = (cudaStream_t)stream;
    return pbn::skart_machine(src, omega, available, h_star, alpha_conf, res);
}
