// pbn_driver.cpp -- host driver: Algorithm 3 (Gelman & Rubin),
// then Algorithm 4 (parallelised two-state, with the
// multi-property reuse of samples) or Algorithm 5 (parallelised
// Skart), over the device trajectory engine.
//
// One driver serves pbn_run (one property, one GPU), pbn_run_multi (q
// properties abstracted from the same trajectories in the same launches) and
// pbn_run_sharded (this process simulates a contiguous block of the omega
// chains; every pooled number goes through the caller's all-reduce).
//
// All decisions are taken on exact integer counters read back from the
// device (6 u64 totals + omega first/last bytes per property and extension);
// the indicator bitstream of every chain stays on the device and is recounted
// by K2 when Algorithm 4 discards a burn-in prefix or Skart re-batches.
// Readings Q7-Q13 of DESIGN.md fix the garbled details (extend_by sign, "M not
// larger than psi", boundary pairs, batch rounding, the min-N rule).
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

// S1, S2, n01, n10, n0from, n1from of one property (A10)
struct Counts {
    uint64_t S1 = 0, S2 = 0, n01 = 0, n10 = 0, n0from = 0, n1from = 0;
};

// Device buffers of one run: q property-major blocks of ol rows (this
// process's chains); the chain state is shared by the properties.
struct Workspace {
    cudaStream_t s = nullptr;
    int64_t ol = 0, q = 0, row_words = 0;
    uint32_t *state = nullptr, *c1 = nullptr, *n01 = nullptr, *n10 = nullptr, *bits = nullptr;
    uint8_t* fl = nullptr;
    uint64_t* totals = nullptr;
    uint32_t* batch = nullptr;
    int64_t batch_cap = 0;
    void* sim_ws = nullptr;  // pbn_simulate scratch (pbn_simulate_workspace_size)
    int64_t sim_ws_bytes = 0;

    ~Workspace()
    {
        cudaFree(state);
        cudaFree(c1);
        cudaFree(n01);
        cudaFree(n10);
        cudaFree(bits);
        cudaFree(fl);
        cudaFree(totals);
        cudaFree(batch);
        cudaFree(sim_ws);
    }
    bool init(pbn_model m, int64_t rows, int64_t nq, int64_t state_words, int64_t rw)
    {
        ol = rows;
        q = nq;
        row_words = rw;
        const size_t r = (size_t)(rows * nq);
        pbn_sim_args sa;
        std::memset(&sa, 0, sizeof(sa));
        sa.n_chains = rows;
        sa.n_props = (int32_t)nq;
        if (pbn_simulate_workspace_size(m, &sa, &sim_ws_bytes) != PBN_OK) return false;
        return cudaMalloc(&state, sizeof(uint32_t) * rows * state_words) == cudaSuccess &&
               cudaMalloc(&c1, sizeof(uint32_t) * r) == cudaSuccess &&
               cudaMalloc(&n01, sizeof(uint32_t) * r) == cudaSuccess &&
               cudaMalloc(&n10, sizeof(uint32_t) * r) == cudaSuccess && cudaMalloc(&fl, r) == cudaSuccess &&
               cudaMalloc(&totals, sizeof(uint64_t) * 6 * nq) == cudaSuccess &&
               cudaMalloc(&bits, sizeof(uint32_t) * r * rw) == cudaSuccess &&
               cudaMemsetAsync(bits, 0, sizeof(uint32_t) * r * rw, s) == cudaSuccess &&
               (sim_ws_bytes == 0 || cudaMalloc(&sim_ws, (size_t)sim_ws_bytes) == cudaSuccess);
    }
    uint32_t* bits_of(int64_t p) const { return bits + (size_t)(p * ol) * (size_t)row_words; }
    // make every row hold at least `need_words` words (copying the old rows)
    bool ensure_rows(int64_t need_words)
    {
        if (need_words <= row_words) return true;
        const int64_t nw = std::max(need_words, 2 * row_words);
        const size_t rows = (size_t)(ol * q);
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
    // q x 6 totals and (optionally) q x ol first/last bytes
    pbn_status read(std::vector<Counts>* c, std::vector<uint8_t>* flh)
    {
        std::vector<uint64_t> t((size_t)(6 * q));
        if (cudaMemcpyAsync(t.data(), totals, sizeof(uint64_t) * t.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return PBN_E_CUDA;
        if (flh) {
            flh->resize((size_t)(ol * q));
            if (cudaMemcpyAsync(flh->data(), fl, flh->size(), cudaMemcpyDeviceToHost, s) != cudaSuccess)
                return PBN_E_CUDA;
        }
        if (cudaStreamSynchronize(s) != cudaSuccess) return PBN_E_CUDA;
        c->assign((size_t)q, Counts());
        for (int64_t p = 0; p < q; ++p) {
            Counts& x = (*c)[(size_t)p];
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

// The one driver.  This process simulates chains [chain_base, chain_base + ol)
// of omega (the whole set when allreduce is NULL); every decision is taken on
// counts pooled by `allreduce` -- the only exchange of the method (SURVEY
// §8(e)) -- so all shards take the same branches and issue the same
// collectives.  Every collective carries a leading error flag, so a shard
// that fails locally reports it at its next collective and every shard
// returns (no shard is left blocked in a collective the others never reach).
static pbn_status run_impl(pbn_model m, const pbn_run_args* a, const pbn_predicate* props, int32_t n_props,
                           int64_t chain_base, int64_t ol, pbn_allreduce_u64_fn allreduce, void* ctx,
                           pbn_run_result* res, pbn_prop_result* per_prop, void* stream, char* err, size_t errlen)
{
    if (!m || !a || !res || !props) {
        set_err(err, errlen, "null argument");
        return PBN_E_USAGE;
    }
    if (n_props < 1 || n_props > PBN_MAX_PROPS) {
        set_err(err, errlen, "n_props must be in 1..%d", PBN_MAX_PROPS);
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
    if (a->method == PBN_METHOD_SKART && n_props != 1) {
        set_err(err, errlen, "multi-property reuse is defined for the two-state method (P:507-526)");
        return PBN_E_USAGE;
    }
    const int64_t omega = a->omega;  // all chains (every formula); this process simulates ol of them
    if (ol < 1 || chain_base < 0 || chain_base + ol > omega) {
        set_err(err, errlen, "shard [%lld, %lld) outside the %lld chains (every shard needs >= 1 chain)",
                (long long)chain_base, (long long)(chain_base + ol), (long long)omega);
        return PBN_E_USAGE;
    }
    std::memset(res, 0, sizeof(*res));
    if (per_prop) std::memset(per_prop, 0, sizeof(*per_prop) * (size_t)n_props);
    pbn_model_info info;
    pbn_status st = pbn_get_model_info(m, &info);
    if (st != PBN_OK) return st;
    const int64_t q = n_props;
    Workspace ws;
    ws.s = (cudaStream_t)stream;
    pbn_status local = PBN_OK;  // first local failure, reported at the next collective
    if (!ws.init(m, ol, q, (info.n + 31) / 32, std::max<int64_t>(2 * a->psi0 / 32 + 2, 64))) local = PBN_E_NOMEM;

    // ---- collectives (identity on one GPU): slot 0 = error flag ----
    auto collective = [&](std::vector<uint64_t>& v) -> pbn_status {
        v[0] = local != PBN_OK ? 1u : 0u;
        if (allreduce && allreduce(v.data(), (int32_t)v.size(), ctx) != 0) {
            set_err(err, errlen, "all-reduce failed");
            return PBN_E_CUDA;
        }
        if (local != PBN_OK) {
            set_err(err, errlen, "local failure (%d)", (int)local);
            return local;
        }
        if (v[0] != 0) {
            set_err(err, errlen, "another shard failed");
            return PBN_E_CUDA;
        }
        return PBN_OK;
    };
    auto pool = [&](const std::vector<Counts>& loc, std::vector<Counts>* out) -> pbn_status {
        std::vector<uint64_t> v(1 + 6 * q, 0);
        for (int64_t p = 0; p < q && local == PBN_OK; ++p) {
            const Counts& x = loc[(size_t)p];
            uint64_t* d = v.data() + 1 + 6 * p;
            d[0] = x.S1, d[1] = x.S2, d[2] = x.n01, d[3] = x.n10, d[4] = x.n0from, d[5] = x.n1from;
        }
        pbn_status s2 = collective(v);
        if (s2 != PBN_OK) return s2;
        out->assign((size_t)q, Counts());
        for (int64_t p = 0; p < q; ++p) {
            const uint64_t* d = v.data() + 1 + 6 * p;
            Counts& x = (*out)[(size_t)p];
            x.S1 = d[0], x.S2 = d[1], x.n01 = d[2], x.n10 = d[3], x.n0from = d[4], x.n1from = d[5];
        }
        return PBN_OK;
    };

    int64_t len = 0;  // transitions simulated per chain
    auto launch = [&](int init, int64_t burn_in, int64_t steps, int64_t bits_offset) -> pbn_status {
        if (!ws.ensure_rows((bits_offset + steps + 31) / 32 + 1)) return PBN_E_NOMEM;
        pbn_sim_args sa;
        std::memset(&sa, 0, sizeof(sa));
        sa.n_chains = ol;
        sa.chain_base = chain_base;
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
        sa.workspace = ws.sim_ws;
        sa.workspace_bytes = ws.sim_ws_bytes;
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
    // window [start, start + length) of every property's bitstream -> totals (+ first/last)
    auto recount = [&](int64_t start, int64_t length) -> pbn_status {
        for (int64_t p = 0; p < q; ++p) {
            pbn_status s2 = pbn_recount(ws.bits_of(p), ol, ws.row_words, start, length, 0, nullptr, nullptr, nullptr,
                                        ws.fl + p * ol, nullptr, ws.totals + 6 * p, ws.s);
            if (s2 != PBN_OK) return s2;
        }
        return PBN_OK;
    };

    // ------------------------- Algorithm 3 --------------------------------
    int64_t psi = a->psi0;
    std::vector<Counts> c, cp;
    std::vector<uint8_t> fl;
    if (local == PBN_OK) local = launch(1, psi, psi, 0);  // 2 psi0 steps, window = last psi0
    double rhat_max = NAN;
    for (;;) {
        if (local == PBN_OK) local = ws.read(&c, &fl);
        if ((st = pool(c, &cp)) != PBN_OK) return st;
        res->gr_iterations++;
        // converged when every property whose windows are not all constant
        // has R-hat < threshold (Q8, Q13); one property: R-hat defined and < threshold
        bool any = false, ok = true;
        rhat_max = NAN;
        for (int64_t p = 0; p < q; ++p) {
            double rh = NAN;
            const pbn_status g = pbn_gelman_rubin(cp[p].S1, cp[p].S2, omega, psi, &rh, nullptr, nullptr, nullptr);
            if (per_prop) per_prop[p].rhat = rh;
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
        if (local == PBN_OK) local = launch(0, 0, psi, 0);
    }
    res->rhat = rhat_max;

    // The merged sample of every property: per chain the row bits [disc, ns)
    // (ns = psi after Algorithm 3: the Gelman-Rubin window is the first
    // sample).  disc may exceed ns: then the sample is empty and
    // the discard continues into the next extension.
    int64_t ns = psi, disc = 0;
    std::vector<uint8_t> last((size_t)(q * ol));  // this shard's chains, per property
    auto take_last = [&](const std::vector<uint8_t>& f) {
        for (size_t i = 0; i < f.size() && i < last.size(); ++i) last[i] = (f[i] >> 1) & 1;
    };
    take_last(fl);

    if (a->method == PBN_METHOD_TWO_STATE) {
        // ------------- Algorithm 4 (readings Q9, Q13) ----------------------
        std::vector<pbn_two_state_result> ts((size_t)q);
        std::vector<pbn_status> tst((size_t)q, PBN_E_DEGENERATE);
        for (;;) {
            for (;;) {
                const int64_t L = std::max<int64_t>(ns - disc, 0);
                if ((st = pool(c, &cp)) != PBN_OK) return st;
                // per property N_p; extend to the smallest unmet
                // N_p until every N_p is met
                int64_t target = -1;
                bool any_ok = false;
                for (int64_t p = 0; p < q; ++p) {
                    std::memset(&ts[p], 0, sizeof(ts[p]));
                    tst[p] = (L >= 2) ? pbn_two_state(cp[p].n01, cp[p].n0from, cp[p].n10, cp[p].n1from, a->r, a->s,
                                                      a->eps, &ts[p])
                                      : PBN_E_DEGENERATE;
                    if (tst[p] != PBN_OK) continue;
                    any_ok = true;
                    if (ts[p].N > omega * L && (target < 0 || ts[p].N < target)) target = ts[p].N;
                }
                int64_t ext;
                if (any_ok) {
                    if (target < 0) break;
                    ext = (target - omega * L + omega - 1) / omega;  // ceil((N - omega n)/omega)
                } else {
                    ext = std::max<int64_t>(L, psi);  // no usable abstraction yet: double the sample
                }
                if (len + ext > a->max_steps) {
                    res->steps_per_chain = len;
                    set_err(err, errlen, "two-state sample exceeds the step cap");
                    return PBN_E_NOT_CONVERGED;
                }
                const int64_t ns_old = ns;
                if (local == PBN_OK) local = launch(0, 0, ext, ns);
                ns += ext;
                res->extensions++;
                if (local != PBN_OK) continue;  // reported at the next pool
                if (disc >= ns_old) {
                    // the sample starts inside the new segment (a burn-in
                    // discard longer than the old sample): recount
                    // the window [disc, ns) of the stored bits
                    if (disc < ns) {
                        local = recount(disc, ns - disc);
                        if (local == PBN_OK) local = ws.read(&c, &fl);
                        if (local == PBN_OK) take_last(fl);
                    } else {
                        c.assign((size_t)q, Counts());  // still inside the discarded prefix
                    }
                    continue;
                }
                std::vector<Counts> d;
                std::vector<uint8_t> fl2;
                if ((local = ws.read(&d, &fl2)) != PBN_OK) continue;
                // pooled counts + the boundary pair (last of old, first of new) per chain (Q7)
                for (int64_t p = 0; p < q; ++p) {
                    Counts& x = c[(size_t)p];
                    for (int64_t k = 0; k < ol; ++k) {
                        const size_t i = (size_t)(p * ol + k);
                        const int b0 = fl2[i] & 1;
                        if (last[i] == 0) {
                            x.n0from++;
                            x.n01 += (b0 == 1);
                        } else {
                            x.n1from++;
                            x.n10 += (b0 == 0);
                        }
                    }
                    x.S1 += d[(size_t)p].S1;
                    x.n01 += d[(size_t)p].n01;
                    x.n10 += d[(size_t)p].n10;
                    x.n0from += d[(size_t)p].n0from;
                    x.n1from += d[(size_t)p].n1from;
                }
                take_last(fl2);
            }
            // burn-in re-check with the largest M_p: M must not be larger
            // than psi; otherwise discard M - psi more elements at
            // the front of every chain's sample, psi := M, and re-enter
            int64_t Mmax = 0;
            for (int64_t p = 0; p < q; ++p)
                if (tst[p] == PBN_OK) Mmax = std::max<int64_t>(Mmax, ts[p].M);
            if (Mmax > psi) {
                disc += Mmax - psi;
                psi = Mmax;
                if (local == PBN_OK) {
                    if (disc < ns) {
                        local = recount(disc, ns - disc);
                        if (local == PBN_OK) local = ws.read(&c, &fl);
                        if (local == PBN_OK) take_last(fl);
                    } else {
                        c.assign((size_t)q, Counts());  // empty sample until the next extension
                    }
                }
                continue;
            }
            break;
        }
        const int64_t L = ns - disc;
        if ((st = pool(c, &cp)) != PBN_OK) return st;
        res->psi = psi;
        res->sample_size = omega * L;
        res->steps_per_chain = len;
        for (int64_t p = 0; p < q; ++p) {
            const double est = L > 0 ? (double)cp[p].S1 / (double)(omega * L) : NAN;
            if (per_prop) {
                per_prop[p].status = tst[p];
                per_prop[p].estimate = est;
                per_prop[p].M = ts[p].M;
                per_prop[p].N = ts[p].N;
                per_prop[p].alpha = ts[p].alpha;
                per_prop[p].beta = ts[p].beta;
            }
            if (p == 0) {
                res->estimate = est;
                res->M = ts[0].M;
                res->N = ts[0].N;
                res->alpha = ts[0].alpha;
                res->beta = ts[0].beta;
            }
        }
        res->ci_lo = res->ci_hi = NAN;
        return PBN_OK;
    }

    // ------------------- Algorithm 5 (readings Q11/Q12) ----------------------
    // The Skart state machine (pbn_skart.cpp) over this run's bitstreams:
    // batches never straddle chains (Fig. 2b), so the pooled
    // batch means of a sharded run are an all-gather of every shard's
    // per-chain batch sums (chain-major), done as a sum of disjoint blocks.
    struct Source : pbn::SkartSource {
        decltype(collective)* coll;
        decltype(pool)* pl;
        Workspace* ws;
        pbn_status* local;
        int64_t omega, ol, chain_base;
        pbn_status ones(int64_t len, uint64_t* S1) override
        {
            std::vector<Counts> c1(1), cp1;
            if (*local == PBN_OK)
                *local = pbn_recount(ws->bits, ol, ws->row_words, 0, len, 0, nullptr, nullptr, nullptr, nullptr,
                                     nullptr, ws->totals, ws->s);
            if (*local == PBN_OK) *local = ws->read(&c1, nullptr);
            pbn_status s2 = (*pl)(c1, &cp1);
            if (s2 != PBN_OK) return s2;
            *S1 = cp1[0].S1;
            return PBN_OK;
        }
        pbn_status batch_sums(int64_t kappa, int64_t per, std::vector<uint32_t>& out) override
        {
            std::vector<uint64_t> v(1 + (size_t)(omega * per), 0);
            if (*local == PBN_OK && !ws->ensure_batch(ol * per)) *local = PBN_E_NOMEM;
            if (*local == PBN_OK)
                *local = pbn_recount(ws->bits, ol, ws->row_words, 0, kappa * per, kappa, nullptr, nullptr, nullptr,
                                     nullptr, ws->batch, nullptr, ws->s);
            std::vector<uint32_t> mine;
            if (*local == PBN_OK) {
                mine.resize((size_t)(ol * per));
                if (cudaMemcpyAsync(mine.data(), ws->batch, sizeof(uint32_t) * mine.size(), cudaMemcpyDeviceToHost,
                                    ws->s) != cudaSuccess ||
                    cudaStreamSynchronize(ws->s) != cudaSuccess)
                    *local = PBN_E_CUDA;
            }
            if (*local == PBN_OK)
                for (size_t j = 0; j < mine.size(); ++j) v[1 + (size_t)(chain_base * per) + j] = mine[j];
            pbn_status s2 = (*coll)(v);
            if (s2 != PBN_OK) return s2;
            out.resize((size_t)(omega * per));
            for (size_t j = 0; j < out.size(); ++j) out[j] = (uint32_t)v[1 + j];
            return PBN_OK;
        }
    } src;
    src.coll = &collective;
    src.pl = &pool;
    src.ws = &ws;
    src.local = &local;
    src.omega = omega;
    src.ol = ol;
    src.chain_base = chain_base;
    for (;;) {
        pbn_skart_result sk;
        st = pbn::skart_machine(src, omega, ns, a->h_star, a->alpha_conf, &sk);
        if (st == PBN_OK) {
            res->estimate = sk.estimate;
            res->ci_lo = sk.ci_lo;
            res->ci_hi = sk.ci_hi;
            res->psi = psi;
            res->sample_size = sk.eta;
            res->steps_per_chain = len;
            res->M = sk.kappa;  // report the final batch size and count in M / N
            res->N = sk.batches;
            res->extensions = sk.spacer;  // Skart: the final spacer d
            return PBN_OK;
        }
        if (st != PBN_E_NOT_CONVERGED) return st;
        if (sk.need_per_chain <= ns) {
            res->steps_per_chain = len;
            set_err(err, errlen, "Skart: iteration cap");
            return PBN_E_NOT_CONVERGED;
        }
        const int64_t need = sk.need_per_chain - ns;
        if (len + need > a->max_steps) {
            res->steps_per_chain = len;
            set_err(err, errlen, "Skart: sample exceeds the step cap");
            return PBN_E_NOT_CONVERGED;
        }
        if (local == PBN_OK) local = launch(0, 0, need, ns);
        ns += need;
    }
}

extern "C" pbn_status pbn_run(pbn_model m, const pbn_run_args* a, pbn_run_result* res, void* stream, char* err,
                              size_t errlen)
{
    return run_impl(m, a, a ? &a->pred : nullptr, 1, 0, a ? a->omega : 0, nullptr, nullptr, res, nullptr, stream, err,
                    errlen);
}

extern "C" pbn_status pbn_run_multi(pbn_model m, const pbn_run_args* a, const pbn_predicate* props, int32_t n_props,
                                    pbn_run_result* res, pbn_prop_result* per_prop, void* stream, char* err,
                                    size_t errlen)
{
    if (!per_prop) {
        set_err(err, errlen, "null per_prop");
        return PBN_E_USAGE;
    }
    if (a && a->method != PBN_METHOD_TWO_STATE) {
        set_err(err, errlen, "multi-property reuse is defined for the two-state method (P:507-526)");
        return PBN_E_USAGE;
    }
    return run_impl(m, a, props, n_props, 0, a ? a->omega : 0, nullptr, nullptr, res, per_prop, stream, err, errlen);
}

extern "C" pbn_status pbn_run_sharded(pbn_model m, const pbn_run_args* a, int64_t chain_base, int64_t omega_local,
                                      pbn_allreduce_u64_fn allreduce, void* ctx, pbn_run_result* res, void* stream,
                                      char* err, size_t errlen)
{
    if (!allreduce) {
        set_err(err, errlen, "null all-reduce");
        return PBN_E_USAGE;
    }
    return run_impl(m, a, a ? &a->pred : nullptr, 1, chain_base, omega_local, allreduce, ctx, res, nullptr, stream,
                    err, errlen);
}
