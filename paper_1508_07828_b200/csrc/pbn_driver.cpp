// pbn_driver.cpp -- host driver: Algorithm 3 (Gelman & Rubin),
// then Algorithm 4 (parallelised two-state) or Algorithm 5
// (parallelised Skart), over the device trajectory engine.
//
// All decisions are taken on exact integer counters read back from the
// device (48 bytes of totals + omega first/last bytes per extension); the
// indicator bitstream of every chain stays on the device and is recounted
// by K2 when Algorithm 4 discards a burn-in prefix.  Readings Q7-Q12 of
// DESIGN.md fix the garbled details (extend_by sign, "M not larger than
// psi", boundary pairs, batch rounding).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/pbnsim.h"
#include "pbn_internal.h"

namespace {

void set_err(char* err, size_t errlen, const char* fmt, ...)
{
    if (!err || errlen == 0) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
}

struct Counts {
    uint64_t S1 = 0, S2 = 0, n01 = 0, n10 = 0, n0from = 0, n1from = 0;
};

// Device workspace of one driver run.
struct Workspace {
    cudaStream_t s = nullptr;
    int64_t omega = 0, state_words = 0;
    uint32_t *state = nullptr, *c1 = nullptr, *n01 = nullptr, *n10 = nullptr;
    uint8_t* fl = nullptr;
    uint64_t* totals = nullptr;
    uint32_t* bits = nullptr;
    int64_t row_words = 0;
    uint32_t* batch = nullptr;
    int64_t batch_cap = 0;

    ~Workspace()
    {
        cudaFree(state);
        cudaFree(c1);
        cudaFree(n01);
        cudaFree(n10);
        cudaFree(fl);
        cudaFree(totals);
        cudaFree(bits);
        cudaFree(batch);
    }
    bool init(int64_t w, int64_t sw, int64_t rw)
    {
        omega = w;
        state_words = sw;
        row_words = rw;
        return cudaMalloc(&state, sizeof(uint32_t) * w * sw) == cudaSuccess &&
               cudaMalloc(&c1, sizeof(uint32_t) * w) == cudaSuccess &&
               cudaMalloc(&n01, sizeof(uint32_t) * w) == cudaSuccess &&
               cudaMalloc(&n10, sizeof(uint32_t) * w) == cudaSuccess &&
               cudaMalloc(&fl, w) == cudaSuccess && cudaMalloc(&totals, 6 * sizeof(uint64_t)) == cudaSuccess &&
               cudaMalloc(&bits, sizeof(uint32_t) * w * rw) == cudaSuccess &&
               cudaMemsetAsync(bits, 0, sizeof(uint32_t) * w * rw, s) == cudaSuccess;
    }
    // make every row hold at least `need_words` words (copying the old rows)
    bool ensure_rows(int64_t need_words)
    {
        if (need_words <= row_words) return true;
        int64_t nw = std::max(need_words, 2 * row_words);
        uint32_t* nb = nullptr;
        if (cudaMalloc(&nb, sizeof(uint32_t) * omega * nw) != cudaSuccess) return false;
        if (cudaMemsetAsync(nb, 0, sizeof(uint32_t) * omega * nw, s) != cudaSuccess) return false;
        if (cudaMemcpy2DAsync(nb, nw * 4, bits, row_words * 4, row_words * 4, omega, cudaMemcpyDeviceToDevice,
                              s) != cudaSuccess)
            return false;
        if (cudaStreamSynchronize(s) != cudaSuccess) return false;
        cudaFree(bits);
        bits = nb;
        row_words = nw;
        return true;
    }
    bool ensure_batch(int64_t n)
    {
        if (n <= batch_cap) return true;
        cudaFree(batch);
        batch = nullptr;
        batch_cap = 0;
        if (cudaMalloc(&batch, sizeof(uint32_t) * n) != cudaSuccess) return false;
        batch_cap = n;
        return true;
    }
};

pbn_status read_counts(Workspace& ws, Counts* c, std::vector<uint8_t>* fl)
{
    uint64_t t[6];
    if (cudaMemcpyAsync(t, ws.totals, sizeof(t), cudaMemcpyDeviceToHost, ws.s) != cudaSuccess) return PBN_E_CUDA;
    if (fl) {
        fl->resize(ws.omega);
        if (cudaMemcpyAsync(fl->data(), ws.fl, ws.omega, cudaMemcpyDeviceToHost, ws.s) != cudaSuccess)
            return PBN_E_CUDA;
    }
    if (cudaStreamSynchronize(ws.s) != cudaSuccess) return PBN_E_CUDA;
    c->S1 = t[0];
    c->S2 = t[1];
    c->n01 = t[2];
    c->n10 = t[3];
    c->n0from = t[4];
    c->n1from = t[5];
    return PBN_OK;
}

}  // namespace

// One driver for one GPU (pbn_run) and for a shard of the chains on each of
// several GPUs (pbn_run_sharded): this process simulates chains
// [chain_base, chain_base + ol) of omega; every decision is taken on counts
// pooled by `allreduce` (the only exchange of the method), so
// all shards take the same branches and issue the same collectives.
static pbn_status run_impl(pbn_model m, const pbn_run_args* a, int64_t chain_base, int64_t ol,
                           pbn_allreduce_u64_fn allreduce, void* ctx, pbn_run_result* res, void* stream, char* err,
                           size_t errlen)
{
    if (!m || !a || !res) {
        set_err(err, errlen, "null argument");
        return PBN_E_USAGE;
    }
    if (a->omega < 2 || a->psi0 < 2 || !(a->rhat_threshold > 1.0) || a->max_steps < 4 * a->psi0) {
        set_err(err, errlen, "need omega >= 2, psi0 >= 2, rhat_threshold > 1, max_steps >= 4 psi0");
        return PBN_E_USAGE;
    }
    if (a->method != PBN_METHOD_TWO_STATE && a->method != PBN_METHOD_SKART) {
        set_err(err, errlen, "unknown method %d", a->method);
        return PBN_E_USAGE;
    }
    std::memset(res, 0, sizeof(*res));
    pbn_model_info info;
    pbn_get_model_info(m, &info);
    Workspace ws;
    ws.s = (cudaStream_t)stream;
    const int64_t omega = a->omega;  // all chains (every formula); this shard simulates ol of them
    if (ol < 1 || chain_base < 0 || chain_base + ol > omega) {
        set_err(err, errlen, "shard [%lld, %lld) outside the %lld chains", (long long)chain_base,
                (long long)(chain_base + ol), (long long)omega);
        return PBN_E_USAGE;
    }
    if (allreduce && a->method != PBN_METHOD_TWO_STATE) {
        set_err(err, errlen, "sharded runs support the two-state method (Skart needs every batch mean)");
        return PBN_E_USAGE;
    }
    // pooled counts of all shards (identity on one GPU)
    auto pool = [&](const Counts& loc, Counts* out) -> pbn_status {
        *out = loc;
        if (!allreduce) return PBN_OK;
        uint64_t v[6] = {loc.S1, loc.S2, loc.n01, loc.n10, loc.n0from, loc.n1from};
        if (allreduce(v, 6, ctx) != 0) return PBN_E_CUDA;
        out->S1 = v[0];
        out->S2 = v[1];
        out->n01 = v[2];
        out->n10 = v[3];
        out->n0from = v[4];
        out->n1from = v[5];
        return PBN_OK;
    };
    if (!ws.init(ol, (info.n + 31) / 32, std::max<int64_t>(2 * a->psi0 / 32 + 2, 64))) {
        set_err(err, errlen, "workspace allocation failed");
        return PBN_E_NOMEM;
    }

    int64_t len = 0;  // transitions simulated per chain
    auto launch = [&](int init, int64_t burn_in, int64_t steps, int64_t bits_offset, int64_t batch,
                      uint32_t* batch_out) -> pbn_status {
        if (!ws.ensure_rows((bits_offset + steps + 31) / 32 + 1)) return PBN_E_NOMEM;
        pbn_sim_args sa;
        std::memset(&sa, 0, sizeof(sa));
        sa.n_chains = ol;
        sa.chain_base = chain_base;
        sa.step0 = len;
        sa.burn_in = burn_in;
        sa.steps = steps;
        sa.batch = batch;
        sa.seed = a->seed;
        sa.pred = a->pred;
        sa.init = init;
        sa.emit_bits = 1;
        sa.bits_offset = bits_offset;
        sa.bits_row_words = ws.row_words;
        pbn_sim_out so;
        so.state = ws.state;
        so.c1 = ws.c1;
        so.n01 = ws.n01;
        so.n10 = ws.n10;
        so.first_last = ws.fl;
        so.batch_sums = batch_out;
        so.bits = ws.bits;
        so.totals = ws.totals;
        pbn_status st = pbn_simulate(m, &sa, &so, ws.s);
        if (st == PBN_OK) len += burn_in + steps;
        return st;
    };

    // ------------------------- Algorithm 3 --------------------------------
    int64_t psi = a->psi0;
    Counts c;
    std::vector<uint8_t> fl;
    pbn_status st = launch(1, psi, psi, 0, 0, nullptr);  // 2 psi0 steps, window = last psi0
    if (st != PBN_OK) {
        set_err(err, errlen, "simulate failed (%d)", (int)st);
        return st;
    }
    double rhat = NAN;
    for (;;) {
        if ((st = read_counts(ws, &c, &fl)) != PBN_OK) return st;
        res->gr_iterations++;
        Counts cp;
        if ((st = pool(c, &cp)) != PBN_OK) return st;
        pbn_status g = pbn_gelman_rubin(cp.S1, cp.S2, omega, psi, &rhat, nullptr, nullptr, nullptr);
        if (g == PBN_OK && rhat < a->rhat_threshold) break;
        if (4 * psi > a->max_steps) {
            res->rhat = rhat;
            res->psi = psi;
            res->steps_per_chain = len;
            set_err(err, errlen, "Gelman-Rubin did not converge within %lld steps", (long long)a->max_steps);
            return PBN_E_NOT_CONVERGED;
        }
        psi *= 2;  // extend all chains to 2 psi: the new window is the new segment
        if ((st = launch(0, 0, psi, 0, 0, nullptr)) != PBN_OK) return st;
    }
    res->rhat = rhat;

    // The merged sample: per chain the row bits [disc, ns), ns = psi initially.
    int64_t ns = psi, disc = 0;
    std::vector<uint8_t> first(ol), last(ol);  // this shard's chains
    for (int64_t k = 0; k < ol; ++k) {
        first[k] = fl[k] & 1;
        last[k] = (fl[k] >> 1) & 1;
    }
    const int64_t psi_gr = psi;
    (void)psi_gr;

    if (a->method == PBN_METHOD_TWO_STATE) {
        // --------------------- Algorithm 4 (reading Q9) --------------------
        pbn_two_state_result ts;
        std::memset(&ts, 0, sizeof(ts));
        for (;;) {
            for (;;) {
                const int64_t L = ns - disc;
                Counts cp;
                if ((st = pool(c, &cp)) != PBN_OK) return st;
                pbn_status t2 = (L >= 2) ? pbn_two_state(cp.n01, cp.n0from, cp.n10, cp.n1from, a->r, a->s, a->eps, &ts)
                                         : PBN_E_DEGENERATE;
                int64_t ext;
                if (t2 == PBN_OK) {
                    if (ts.N <= omega * L) break;
                    ext = (ts.N - omega * L + omega - 1) / omega;  // ceil((N - omega n)/omega)
                } else {
                    ext = std::max<int64_t>(L, psi);  // degenerate abstraction: double the sample
                }
                if (len + ext > a->max_steps) {
                    res->steps_per_chain = len;
                    set_err(err, errlen, "two-state sample exceeds the step cap");
                    return PBN_E_NOT_CONVERGED;
                }
                if ((st = launch(0, 0, ext, ns, 0, nullptr)) != PBN_OK) return st;
                Counts d;
                std::vector<uint8_t> fl2;
                if ((st = read_counts(ws, &d, &fl2)) != PBN_OK) return st;
                // pooled counts + the boundary pair (last of old, first of new) per chain (Q7)
                for (int64_t k = 0; k < ol; ++k) {
                    const int a0 = (L > 0) ? last[k] : -1, b0 = fl2[k] & 1;
                    if (a0 == 0) {
                        c.n0from++;
                        c.n01 += (b0 == 1);
                    } else if (a0 == 1) {
                        c.n1from++;
                        c.n10 += (b0 == 0);
                    }
                    if (L == 0) first[k] = fl2[k] & 1;
                    last[k] = (fl2[k] >> 1) & 1;
                }
                c.S1 += d.S1;
                c.n01 += d.n01;
                c.n10 += d.n10;
                c.n0from += d.n0from;
                c.n1from += d.n1from;
                ns += ext;
                res->extensions++;
            }
            // burn-in re-check: M must not be larger than psi
            if (ts.M > psi) {
                disc += ts.M - psi;
                psi = ts.M;
                const int64_t L = std::max<int64_t>(ns - disc, 0);
                if (disc > ns) disc = ns;
                st = pbn_recount(ws.bits, ol, ws.row_words, disc, L, 0, nullptr, nullptr, nullptr, ws.fl,
                                 nullptr, ws.totals, ws.s);
                if (st != PBN_OK) return st;
                if ((st = read_counts(ws, &c, &fl)) != PBN_OK) return st;
                for (int64_t k = 0; k < ol; ++k) {
                    first[k] = fl[k] & 1;
                    last[k] = (fl[k] >> 1) & 1;
                }
                continue;
            }
            break;
        }
        res->M = ts.M;
        res->N = ts.N;
        res->alpha = ts.alpha;
        res->beta = ts.beta;
        res->psi = psi;
        res->sample_size = omega * (ns - disc);
        res->steps_per_chain = len;
        Counts cp;
        if ((st = pool(c, &cp)) != PBN_OK) return st;
        res->estimate = (double)cp.S1 / (double)res->sample_size;
        res->ci_lo = res->ci_hi = NAN;
        return PBN_OK;
    }

    // ------------------- Algorithm 5 (readings Q11/Q12) ----------------------
    // Declared Skart constants: skewness limit 4 (kappa 1 or 16),
    // von Neumann randomness test at level 0.20 two-sided, kappa <- ceil(sqrt2
    // kappa) and spacer d <- d + 1 on failure, batch-count ceiling 1024 in the
    // CI loop.  Batches never straddle chains: p is a multiple of omega.
    const double z_pass = pbn_inv_norm_cdf(1.0 - 0.20 / 2.0);
    auto round_up = [omega](int64_t v) { return (v + omega - 1) / omega * omega; };
    auto ensure = [&](int64_t per_chain_len) -> pbn_status {
        const int64_t need = per_chain_len - ns;
        if (need <= 0) return PBN_OK;
        if (len + need > a->max_steps) return PBN_E_NOT_CONVERGED;
        pbn_status s2 = launch(0, 0, need, ns, 0, nullptr);
        if (s2 == PBN_OK) ns += need;
        return s2;
    };
    std::vector<uint32_t> hbs;
    // per-chain sums of `per` consecutive kappa-batches from the sample start
    auto batches = [&](int64_t kappa, int64_t per) -> pbn_status {
        if (!ws.ensure_batch(omega * per)) return PBN_E_NOMEM;
        pbn_status s2 = pbn_recount(ws.bits, omega, ws.row_words, 0, kappa * per, kappa, nullptr, nullptr, nullptr,
                                    nullptr, ws.batch, nullptr, ws.s);
        if (s2 != PBN_OK) return s2;
        hbs.resize((size_t)(omega * per));
        if (cudaMemcpyAsync(hbs.data(), ws.batch, sizeof(uint32_t) * hbs.size(), cudaMemcpyDeviceToHost, ws.s) !=
                cudaSuccess ||
            cudaStreamSynchronize(ws.s) != cudaSuccess)
            return PBN_E_CUDA;
        return PBN_OK;
    };
    auto fail = [&](pbn_status s2, const char* what) {
        res->steps_per_chain = len;
        set_err(err, errlen, "%s", what);
        return s2;
    };

    int64_t eta = round_up(1280);  // Alg 5 line 3
    if ((st = ensure(eta / omega)) != PBN_OK) return fail(st, "Skart: initial sample exceeds the step cap");
    // skewness of all eta samples (line 5): for 0/1 data (1 - 2m) / sqrt(m (1 - m))
    if ((st = pbn_recount(ws.bits, omega, ws.row_words, 0, eta / omega, 0, nullptr, nullptr, nullptr, nullptr,
                          nullptr, ws.totals, ws.s)) != PBN_OK)
        return st;
    if ((st = read_counts(ws, &c, nullptr)) != PBN_OK) return st;
    const double m1 = (double)c.S1 / (double)eta;
    const bool skew_defined = m1 > 0.0 && m1 < 1.0;
    const double skew = skew_defined ? (1.0 - 2.0 * m1) / std::sqrt(m1 * (1.0 - m1)) : NAN;
    int64_t kappa = (skew_defined && std::fabs(skew) <= 4.0) ? 1 : 16;
    int64_t p = round_up(eta);  // line 6
    eta = kappa * p;
    int64_t d = 0;
    // lines 7-12: randomness (independence) test on spaced batch means
    for (int iter = 0;; ++iter) {
        if (iter >= 64) return fail(PBN_E_NOT_CONVERGED, "Skart: randomness test iteration cap");
        if ((st = ensure(eta / omega)) != PBN_OK) return fail(st, "Skart: sample exceeds the step cap");
        const int64_t per = p / omega;
        if ((st = batches(kappa, per)) != PBN_OK) return st;
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
                pass = false;
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
        if (iter >= 64) return fail(PBN_E_NOT_CONVERGED, "Skart: precision iteration cap");
        if ((st = ensure(eta / omega)) != PBN_OK) return fail(st, "Skart: sample exceeds the step cap");
        const int64_t per = p / omega;
        if ((st = batches(kappa, per)) != PBN_OK) return st;
        pbn_skart_ci ci;
        st = pbn_skart_ci_from_batches(hbs.data(), omega, per, kappa, a->alpha_conf, &ci);
        if (st != PBN_OK && st != PBN_E_DEGENERATE) return st;
        if (ci.H <= a->h_star) {
            res->estimate = ci.mu;
            res->ci_lo = ci.ci_lo;
            res->ci_hi = ci.ci_hi;
            res->psi = psi;
            res->sample_size = eta;
            res->steps_per_chain = len;
            res->M = kappa;  // report the final batch size and count in M / N
            res->N = p;
            return PBN_OK;
        }
        const double g = (ci.H / a->h_star) * (ci.H / a->h_star);
        const int64_t new_eta = (int64_t)std::ceil(g * (double)eta);
        if (p < 1024) p = std::min<int64_t>(1024, (int64_t)std::ceil(g * (double)p));
        p = round_up(p);
        kappa = std::max(kappa, (new_eta + p - 1) / p);
        eta = kappa * p;
    }
}


extern "C" pbn_status pbn_run(pbn_model m, const pbn_run_args* a, pbn_run_result* res, void* stream, char* err,
                              size_t errlen)
{
    return run_impl(m, a, 0, a ? a->omega : 0, nullptr, nullptr, res, stream, err, errlen);
}

extern "C" pbn_status pbn_run_sharded(pbn_model m, const pbn_run_args* a, int64_t chain_base, int64_t omega_local,
                                      pbn_allreduce_u64_fn allreduce, void* ctx, pbn_run_result* res, void* stream,
                                      char* err, size_t errlen)
{
    if (!allreduce) {
        set_err(err, errlen, "null all-reduce");
        return PBN_E_USAGE;
    }
    return run_impl(m, a, chain_base, omega_local, allreduce, ctx, res, stream, err, errlen);
}
