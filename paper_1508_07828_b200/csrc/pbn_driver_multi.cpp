// pbn_driver_multi.cpp -- host driver for several properties at once:
// Algorithm 3 then Algorithm 4 with the multi-property reuse of samples
// (§4.2; reading Q13 in DESIGN.md).
//
// One set of omega trajectories is abstracted into q meta-state sequences in
// the same kernel launch (pbn_simulate with n_props = q); the statistics of
// every property come from its own counters and indicator bitstream.
//   - Gelman & Rubin: the chains are converged when every property whose
//     windows are not all constant has R-hat below the threshold (Q8); the
//     largest R-hat is reported.
//   - Extension: per property N_p from its pooled alpha, beta;
//     "the next extension length is determined by the minimal value of all
//     the calculated Ns": the pooled sample grows to the smallest N_p
//     that is not yet met, then every N_p is re-evaluated; it stops "when all
//     the calculated Ns are smaller than the current sample size".
//     Properties whose two-state statistics are degenerate (alpha+beta in
//     {0, 2}, an unvisited meta state) are reported as such and do not drive
//     the extension ("reported individually").
//   - Burn-in re-check (reading Q9): with M = the largest M_p, if
//     M > psi the first M - psi elements of every chain are discarded for all
//     properties (K2 recount of each bitstream), psi := M, re-enter.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/pbnsim.h"

namespace {

void set_err(char* err, size_t errlen, const char* fmt, ...)
{
    if (!err || errlen == 0) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
}

struct PropCounts {
    uint64_t S1 = 0, S2 = 0, n01 = 0, n10 = 0, n0from = 0, n1from = 0;
};

// Device buffers of one run: q property-major blocks of omega rows.
struct MultiWorkspace {
    cudaStream_t s = nullptr;
    int64_t omega = 0, q = 0, row_words = 0;
    uint32_t *state = nullptr, *c1 = nullptr, *n01 = nullptr, *n10 = nullptr, *bits = nullptr;
    uint8_t* fl = nullptr;
    uint64_t* totals = nullptr;

    ~MultiWorkspace()
    {
        cudaFree(state);
        cudaFree(c1);
        cudaFree(n01);
        cudaFree(n10);
        cudaFree(bits);
        cudaFree(fl);
        cudaFree(totals);
    }
    bool init(int64_t w, int64_t nq, int64_t state_words, int64_t rw)
    {
        omega = w;
        q = nq;
        row_words = rw;
        const size_t rows = (size_t)(w * nq);
        return cudaMalloc(&state, sizeof(uint32_t) * w * state_words) == cudaSuccess &&
               cudaMalloc(&c1, sizeof(uint32_t) * rows) == cudaSuccess &&
               cudaMalloc(&n01, sizeof(uint32_t) * rows) == cudaSuccess &&
               cudaMalloc(&n10, sizeof(uint32_t) * rows) == cudaSuccess && cudaMalloc(&fl, rows) == cudaSuccess &&
               cudaMalloc(&totals, sizeof(uint64_t) * 6 * nq) == cudaSuccess &&
               cudaMalloc(&bits, sizeof(uint32_t) * rows * rw) == cudaSuccess &&
               cudaMemsetAsync(bits, 0, sizeof(uint32_t) * rows * rw, s) == cudaSuccess;
    }
    bool ensure_rows(int64_t need_words)
    {
        if (need_words <= row_words) return true;
        const int64_t nw = std::max(need_words, 2 * row_words);
        const size_t rows = (size_t)(omega * q);
        uint32_t* nb = nullptr;
        if (cudaMalloc(&nb, sizeof(uint32_t) * rows * nw) != cudaSuccess) return false;
        if (cudaMemsetAsync(nb, 0, sizeof(uint32_t) * rows * nw, s) != cudaSuccess ||
            cudaMemcpy2DAsync(nb, nw * 4, bits, row_words * 4, row_words * 4, rows, cudaMemcpyDeviceToDevice, s) !=
                cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            cudaFree(nb);
            return false;
        }
        cudaFree(bits);
        bits = nb;
        row_words = nw;
        return true;
    }
    // q x 6 totals and q x omega first/last bytes
    pbn_status read(std::vector<PropCounts>* c, std::vector<uint8_t>* flh)
    {
        std::vector<uint64_t> t((size_t)(6 * q));
        flh->resize((size_t)(omega * q));
        if (cudaMemcpyAsync(t.data(), totals, sizeof(uint64_t) * t.size(), cudaMemcpyDeviceToHost, s) !=
                cudaSuccess ||
            cudaMemcpyAsync(flh->data(), fl, flh->size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return PBN_E_CUDA;
        c->assign((size_t)q, PropCounts());
        for (int64_t p = 0; p < q; ++p) {
            PropCounts& x = (*c)[(size_t)p];
            x.S1 = t[6 * p + 0];
            x.S2 = t[6 * p + 1];
            x.n01 = t[6 * p + 2];
            x.n10 = t[6 * p + 3];
            x.n0from = t[6 * p + 4];
            x.n1from = t[6 * p + 5];
        }
        return PBN_OK;
    }
};

}  // namespace

extern "C" pbn_status pbn_run_multi(pbn_model m, const pbn_run_args* a, const pbn_predicate* props, int32_t n_props,
                                    pbn_run_result* res, pbn_prop_result* per_prop, void* stream, char* err,
                                    size_t errlen)
{
    if (!m || !a || !res || !per_prop || !props) {
        set_err(err, errlen, "null argument");
        return PBN_E_USAGE;
    }
    if (n_props < 1 || n_props > PBN_MAX_PROPS) {
        set_err(err, errlen, "n_props must be in 1..%d", PBN_MAX_PROPS);
        return PBN_E_USAGE;
    }
    if (a->method != PBN_METHOD_TWO_STATE) {
        set_err(err, errlen, "multi-property reuse is defined for the two-state method (P:507-526)");
        return PBN_E_USAGE;
    }
    if (a->omega < 2 || a->psi0 < 2 || !(a->rhat_threshold > 1.0) || a->max_steps < 4 * a->psi0) {
        set_err(err, errlen, "need omega >= 2, psi0 >= 2, rhat_threshold > 1, max_steps >= 4 psi0");
        return PBN_E_USAGE;
    }
    std::memset(res, 0, sizeof(*res));
    std::memset(per_prop, 0, sizeof(*per_prop) * (size_t)n_props);
    pbn_model_info info;
    pbn_status st = pbn_get_model_info(m, &info);
    if (st != PBN_OK) return st;
    const int64_t omega = a->omega, q = n_props;
    MultiWorkspace ws;
    ws.s = (cudaStream_t)stream;
    if (!ws.init(omega, q, (info.n + 31) / 32, std::max<int64_t>(2 * a->psi0 / 32 + 2, 64))) {
        set_err(err, errlen, "workspace allocation failed");
        return PBN_E_NOMEM;
    }

    int64_t len = 0;  // transitions simulated per chain
    auto launch = [&](int init, int64_t burn_in, int64_t steps, int64_t bits_offset) -> pbn_status {
        if (!ws.ensure_rows((bits_offset + steps + 31) / 32 + 1)) return PBN_E_NOMEM;
        pbn_sim_args sa;
        std::memset(&sa, 0, sizeof(sa));
        sa.n_chains = omega;
        sa.step0 = len;
        sa.burn_in = burn_in;
        sa.steps = steps;
        sa.seed = a->seed;
        sa.init = init;
        sa.emit_bits = 1;
        sa.bits_offset = bits_offset;
        sa.bits_row_words = ws.row_words;
        sa.n_props = n_props;
        sa.props = props;
        pbn_sim_out so;
        std::memset(&so, 0, sizeof(so));
        so.state = ws.state;
        so.c1 = ws.c1;
        so.n01 = ws.n01;
        so.n10 = ws.n10;
        so.first_last = ws.fl;
        so.bits = ws.bits;
        so.totals = ws.totals;
        pbn_status s2 = pbn_simulate(m, &sa, &so, ws.s);
        if (s2 == PBN_OK) len += burn_in + steps;
        return s2;
    };

    // ------------------------- Algorithm 3 --------------------------------
    int64_t psi = a->psi0;
    std::vector<PropCounts> c;
    std::vector<uint8_t> fl;
    if ((st = launch(1, psi, psi, 0)) != PBN_OK) {
        set_err(err, errlen, "simulate failed (%d)", (int)st);
        return st;
    }
    double rhat_max = NAN;
    for (;;) {
        if ((st = ws.read(&c, &fl)) != PBN_OK) return st;
        res->gr_iterations++;
        bool any = false, ok = true;
        rhat_max = NAN;
        for (int64_t p = 0; p < q; ++p) {
            double rh = NAN;
            const pbn_status g = pbn_gelman_rubin(c[p].S1, c[p].S2, omega, psi, &rh, nullptr, nullptr, nullptr);
            per_prop[p].rhat = rh;
            if (g != PBN_OK) continue;  // all windows constant: R-hat undefined (Q8)
            any = true;
            if (!(rh < a->rhat_threshold)) ok = false;
            if (std::isnan(rhat_max) || rh > rhat_max) rhat_max = rh;
        }
        if (any && ok) break;
        if (4 * psi > a->max_steps) {
            res->rhat = rhat_max;
            res->psi = psi;
            res->steps_per_chain = len;
            set_err(err, errlen, "Gelman-Rubin did not converge within %lld steps", (long long)a->max_steps);
            return PBN_E_NOT_CONVERGED;
        }
        psi *= 2;  // extend all chains to 2 psi: the new window is the new segment
        if ((st = launch(0, 0, psi, 0)) != PBN_OK) return st;
    }
    res->rhat = rhat_max;

    // merged sample per chain: row bits [disc, ns) of every property's stream
    int64_t ns = psi, disc = 0;
    std::vector<uint8_t> first((size_t)(q * omega)), last((size_t)(q * omega));
    auto take_fl = [&](const std::vector<uint8_t>& f) {
        for (size_t i = 0; i < f.size(); ++i) {
            first[i] = f[i] & 1;
            last[i] = (f[i] >> 1) & 1;
        }
    };
    take_fl(fl);
    std::vector<pbn_two_state_result> ts((size_t)q);
    std::vector<pbn_status> tst((size_t)q, PBN_E_DEGENERATE);
    for (;;) {
        for (;;) {
            const int64_t L = ns - disc;
            int64_t target = -1;  // smallest unmet N_p
            bool any_ok = false;
            for (int64_t p = 0; p < q; ++p) {
                std::memset(&ts[p], 0, sizeof(ts[p]));
                tst[p] = (L >= 2) ? pbn_two_state(c[p].n01, c[p].n0from, c[p].n10, c[p].n1from, a->r, a->s, a->eps,
                                                  &ts[p])
                                  : PBN_E_DEGENERATE;
                if (tst[p] != PBN_OK) continue;
                any_ok = true;
                if (ts[p].N > omega * L && (target < 0 || ts[p].N < target)) target = ts[p].N;
            }
            int64_t ext;
            if (any_ok) {
                if (target < 0) break;  // every N_p is met by the pooled sample
                ext = (target - omega * L + omega - 1) / omega;
            } else {
                ext = std::max<int64_t>(L, psi);  // no property has usable statistics yet: double
            }
            if (len + ext > a->max_steps) {
                res->steps_per_chain = len;
                set_err(err, errlen, "two-state sample exceeds the step cap");
                return PBN_E_NOT_CONVERGED;
            }
            if ((st = launch(0, 0, ext, ns)) != PBN_OK) return st;
            std::vector<PropCounts> d;
            std::vector<uint8_t> fl2;
            if ((st = ws.read(&d, &fl2)) != PBN_OK) return st;
            // pooled counts + the boundary pair (last of old, first of new) per chain (Q7)
            for (int64_t p = 0; p < q; ++p) {
                for (int64_t k = 0; k < omega; ++k) {
                    const size_t i = (size_t)(p * omega + k);
                    const int a0 = (L > 0) ? last[i] : -1, b0 = fl2[i] & 1;
                    if (a0 == 0) {
                        c[p].n0from++;
                        c[p].n01 += (b0 == 1);
                    } else if (a0 == 1) {
                        c[p].n1from++;
                        c[p].n10 += (b0 == 0);
                    }
                    if (L == 0) first[i] = fl2[i] & 1;
                    last[i] = (fl2[i] >> 1) & 1;
                }
                c[p].S1 += d[p].S1;
                c[p].n01 += d[p].n01;
                c[p].n10 += d[p].n10;
                c[p].n0from += d[p].n0from;
                c[p].n1from += d[p].n1from;
            }
            ns += ext;
            res->extensions++;
        }
        // burn-in re-check with the largest M_p
        int64_t Mmax = 0;
        for (int64_t p = 0; p < q; ++p)
            if (tst[p] == PBN_OK) Mmax = std::max<int64_t>(Mmax, ts[p].M);
        if (Mmax > psi) {
            disc += Mmax - psi;
            psi = Mmax;
            if (disc > ns) disc = ns;
            const int64_t L = ns - disc;
            for (int64_t p = 0; p < q; ++p) {
                st = pbn_recount(ws.bits + (size_t)(p * omega) * (size_t)ws.row_words, omega, ws.row_words, disc, L,
                                 0, nullptr, nullptr, nullptr, ws.fl + p * omega, nullptr, ws.totals + 6 * p, ws.s);
                if (st != PBN_OK) return st;
            }
            if ((st = ws.read(&c, &fl)) != PBN_OK) return st;
            take_fl(fl);
            continue;
        }
        break;
    }
    const int64_t L = ns - disc;
    res->psi = psi;
    res->sample_size = omega * L;
    res->steps_per_chain = len;
    for (int64_t p = 0; p < q; ++p) {
        per_prop[p].status = tst[p];
        per_prop[p].estimate = L > 0 ? (double)c[p].S1 / (double)(omega * L) : NAN;
        per_prop[p].M = ts[p].M;
        per_prop[p].N = ts[p].N;
        per_prop[p].alpha = ts[p].alpha;
        per_prop[p].beta = ts[p].beta;
    }
    // the first property's numbers also fill the single-property fields
    res->estimate = per_prop[0].estimate;
    res->M = per_prop[0].M;
    res->N = per_prop[0].N;
    res->alpha = per_prop[0].alpha;
    res->beta = per_prop[0].beta;
    res->ci_lo = res->ci_hi = NAN;
    return PBN_OK;
}
