/*
 * pbn_oracle.c -- plain, slow, obviously-correct CPU oracle for the PBN
 * trajectory hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * product path (paper_1508_07828_b200/csrc), and includes nothing from it.
 *
 * What it computes, in the paper's order (§2.2):
 *   - state s(t) in {0,1}^n held UNPACKED, one byte per node;
 *   - per step t and node i one 32-bit uniform word u(chain,t,i) from
 *     Philox4x32-10 (reading Q2/Q3 of DESIGN.md);
 *   - perturbation gamma_i(t) = [u < T_p] ~ Bernoulli(p);
 *   - VECTOR semantics (default): if any gamma_i(t) = 1 then
 *     s(t+1) = s(t) XOR gamma(t); otherwise every node applies its selected
 *     predictor function synchronously, s(t+1) = f(t)(s(t));
 *     PER_NODE semantics (load-time flag, reading Q1): node i flips iff
 *     gamma_i(t) = 1, otherwise applies its function;
 *   - selection of function j for node i with probability c_j^(i)
 *      by comparing the same word against cumulative
 *     thresholds (reading Q3);
 *   - truth-table lookup with parents[0] as the most significant index
 *     bit (reading Q5);
 *   - the property indicator I_t = AND_k [s_t[node_k] = v_k];
 *   - optionally (NEXT-2, reading Q18) gamma(t) drawn by geometric skips
 *     from a separate word stream, VECTOR semantics.
 *
 * Statistics (counts, transitions, batches, R-hat, two-state, Skart) are
 * computed in Python by definition from the stored I sequence
 * (oracle/stats.py); nothing here accumulates them.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: */
/* as easy as 1, 2, 3", SC'11): 10 rounds of                            */
/*   (hi0,lo0) = M0 * c0 ; (hi1,lo1) = M1 * c2                          */
/*   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)                      */
/* with the key bumped by the Weyl constants (W0,W1) between rounds.    */
/* ------------------------------------------------------------------ */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += PHILOX_W0;
            k1 += PHILOX_W1;
        }
        uint64_t prod0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Stream definition (reading Q2):
 *   key     = (seed mod 2^32, seed >> 32)
 *   counter = (floor(i/4), chain, t mod 2^32, t >> 32)
 *   u(chain, t, i) = philox(counter, key)[i mod 4]
 * t = 0 is reserved for the initial state, transition t (s_{t-1} -> s_t)
 * uses t >= 1. */
uint32_t oracle_word(uint64_t seed, uint32_t chain, uint64_t t, uint32_t i)
{
    uint32_t ctr[4] = {i / 4u, chain, (uint32_t)(t & 0xFFFFFFFFu), (uint32_t)(t >> 32)};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    uint32_t out[4];
    oracle_philox4x32_10(ctr, key, out);
    return out[i % 4u];
}

/* ------------------------------------------------------------------ */
/* Thresholds (reading Q3): p and c are quantised to 2^-32.  */
/*   T_p     = floor(p * 2^32)                                         */
/*   C_{i,j} = c_1 + ... + c_j   (left-to-right fp64 sum)              */
/*   Q_{i,j} = min(floor(C_{i,j} * 2^32), 2^32)                        */
/*   D_{i,j} = T_p + floor(Q_{i,j} * (2^32 - T_p) / 2^32)   (in u64)   */
/* for j = 1 .. ell(i)-1.  A word u < T_p is a perturbation; otherwise */
/* node i selects function j = min{ j : u < D_{i,j} }, else the last.  */
/* D is written per function: D[f] for f the j-th function of node i   */
/* (j < ell(i)); the last function of each node gets D = 2^32.         */
/* ------------------------------------------------------------------ */
uint32_t oracle_perturbation_threshold(double p)
{
    return (uint32_t)floor(ldexp(p, 32));
}

void oracle_selection_thresholds(int32_t n, const int32_t* fn_off, const double* sel_prob,
                                 double p, uint64_t* D)
{
    uint64_t Tp = oracle_perturbation_threshold(p);
    uint64_t span = (((uint64_t)1) << 32) - Tp;
    for (int32_t i = 0; i < n; ++i) {
        double C = 0.0;
        for (int32_t f = fn_off[i]; f < fn_off[i + 1]; ++f) {
            C += sel_prob[f];
            if (f == fn_off[i + 1] - 1) {
                D[f] = ((uint64_t)1) << 32;
            } else {
                uint64_t Q = (uint64_t)floor(ldexp(C, 32));
                if (Q > (((uint64_t)1) << 32))
                    Q = ((uint64_t)1) << 32; /* cumulative sum rounded above 1 */
                /* Q * span < 2^33 * 2^32: use 128-bit to stay exact */
                unsigned __int128 prod = (unsigned __int128)Q * (unsigned __int128)span;
                D[f] = Tp + (uint64_t)(prod >> 32);
            }
        }
    }
}

/* ------------------------------------------------------------------ */
/* Geometric-skip perturbation stream (SPEC S:177's optional mode,      */
/* SURVEY NEXT-2; reading Q18), VECTOR semantics.             */
/* The perturbation vector gamma(t) in {0,1}^n with i.i.d. Bernoulli(p) */
/* components is drawn as the positions of its ones:        */
/*   k_1 = G(v_0),  k_{j+1} = k_j + 1 + G(v_j),  stop at the first k>=n */
/* where G(v) = #{g in [0,n) : Cg[g] <= v} is a geometric skip drawn    */
/* from one 32-bit word v by inverting the cumulative table             */
/*   Cg[g] = floor((1 - q^(g+1)) * 2^32),  q = 1 - p,                   */
/* with q^(g+1) formed by repeated fp64 multiplication (q, q*q, ...).   */
/* The skip words are a separate Philox counter space:                  */
/*   v(chain, t, m) = philox((2^31 + m/4, chain, t lo, t hi), key)[m%4] */
/* When gamma(t) = 0 every node selects function j = min{j : u < Q_j}   */
/* with its node word u(chain, t, i) (reading Q3 with T_p = 0).         */
/* ------------------------------------------------------------------ */
void oracle_geometric_table(int32_t n, double p, uint32_t* Cg)
{
    double q = 1.0 - p, r = 1.0;
    for (int32_t g = 0; g < n; ++g) {
        r = r * q; /* q^(g+1) */
        Cg[g] = (uint32_t)floor(ldexp(1.0 - r, 32));
    }
}

uint32_t oracle_skip_word(uint64_t seed, uint32_t chain, uint64_t t, uint32_t m)
{
    uint32_t ctr[4] = {0x80000000u + m / 4u, chain, (uint32_t)(t & 0xFFFFFFFFu), (uint32_t)(t >> 32)};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    uint32_t out[4];
    oracle_philox4x32_10(ctr, key, out);
    return out[m % 4u];
}

/* G(v): the number of table entries <= v, by a plain linear count */
int32_t oracle_skip(const uint32_t* Cg, int32_t n, uint32_t v)
{
    int32_t G = 0;
    for (int32_t g = 0; g < n; ++g)
        if (Cg[g] <= v)
            G++;
    return G;
}

/* gamma(t) of one chain-step into gam[0..n-1]; returns the number of ones */
static int32_t geometric_gamma(const uint32_t* Cg, int32_t n, uint64_t seed, uint32_t chain, uint64_t t,
                               uint8_t* gam)
{
    memset(gam, 0, (size_t)n);
    int32_t ones = 0;
    int64_t k = -1;
    for (uint32_t m = 0;; ++m) {
        k = k + 1 + oracle_skip(Cg, n, oracle_skip_word(seed, chain, t, m));
        if (k >= n)
            break;
        gam[k] = 1;
        ones++;
    }
    return ones;
}

/* ------------------------------------------------------------------ */
/* One synchronous step with given words u[0..n-1].        */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t n;
    const int32_t* fn_off;
    const int32_t* par_off;
    const uint16_t* parents;
    const int32_t* tbl_off;
    const uint32_t* tables;
    const double* sel_prob;
    double p;
    int32_t per_node; /* 0 = VECTOR, 1 = PER_NODE */
} oracle_model;

static int apply_function(const oracle_model* m, int32_t f, const uint8_t* s)
{
    /* index formed from the parents' values, parents[0] most significant */
    uint32_t idx = 0;
    for (int32_t k = m->par_off[f]; k < m->par_off[f + 1]; ++k)
        idx = idx * 2u + (uint32_t)s[m->parents[k]];
    uint32_t word = m->tables[m->tbl_off[f] + (int32_t)(idx / 32u)];
    return (int)((word >> (idx % 32u)) & 1u);
}

static int32_t select_function(const oracle_model* m, const uint64_t* D, int32_t i, uint32_t u)
{
    for (int32_t f = m->fn_off[i]; f < m->fn_off[i + 1]; ++f)
        if ((uint64_t)u < D[f])
            return f;
    return m->fn_off[i + 1] - 1; /* unreachable: the last D is 2^32 */
}

static void step_with_words(const oracle_model* m, uint32_t Tp, const uint64_t* D,
                            const uint8_t* s, const uint32_t* u, uint8_t* s_next)
{
    int32_t n = m->n;
    int any_gamma = 0;
    for (int32_t i = 0; i < n; ++i)
        if (u[i] < Tp)
            any_gamma = 1;
    if (!m->per_node && any_gamma) {
        /* s(t+1) = s(t) XOR gamma(t) */
        for (int32_t i = 0; i < n; ++i)
            s_next[i] = (uint8_t)(s[i] ^ (u[i] < Tp ? 1 : 0));
        return;
    }
    for (int32_t i = 0; i < n; ++i) {
        if (m->per_node && u[i] < Tp) {
            s_next[i] = (uint8_t)(1 - s[i]);
        } else {
            int32_t f = select_function(m, D, i, u[i]);
            s_next[i] = (uint8_t)apply_function(m, f, s);
        }
    }
}

/* Exported single step with injected words (used by the step pins). */
int oracle_step(int32_t n, const int32_t* fn_off, const int32_t* par_off, const uint16_t* parents,
                const int32_t* tbl_off, const uint32_t* tables, const double* sel_prob, double p,
                int32_t per_node, const uint8_t* s, const uint32_t* u, uint8_t* s_next)
{
    oracle_model m = {n, fn_off, par_off, parents, tbl_off, tables, sel_prob, p, per_node};
    uint64_t* D = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(fn_off[n] > 0 ? fn_off[n] : 1));
    if (!D)
        return 1;
    oracle_selection_thresholds(n, fn_off, sel_prob, p, D);
    step_with_words(&m, oracle_perturbation_threshold(p), D, s, u, s_next);
    free(D);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Trajectories of a list of chains.                                   */
/*   state   [nchains x n] bytes, in: s_{step0} (ignored if init),     */
/*           out: s_{step0 + burn_in + steps}                          */
/*   init    if 1 (requires step0 == 0): s_0[i] = u(chain,0,i) >> 31   */
/*   I_out   [nchains x steps] bytes: I_t for the recorded window      */
/*           t = step0+burn_in+1 .. step0+burn_in+steps (reading Q6)   */
/* ------------------------------------------------------------------ */
int oracle_simulate(int32_t n, const int32_t* fn_off, const int32_t* par_off,
                    const uint16_t* parents, const int32_t* tbl_off, const uint32_t* tables,
                    const double* sel_prob, double p, int32_t per_node, uint64_t seed,
                    const uint32_t* chain_ids, int64_t nchains, int64_t step0, int64_t burn_in,
                    int64_t steps, int32_t init, int32_t k, const uint16_t* pred_node,
                    const uint8_t* pred_value, uint8_t* state, uint8_t* I_out)
{
    if (init && step0 != 0)
        return 2;
    /* per_node: 0 VECTOR, 1 PER_NODE, 2 VECTOR with the geometric-skip stream */
    const int geometric = per_node == 2;
    oracle_model m = {n, fn_off, par_off, parents, tbl_off, tables, sel_prob, p, geometric ? 0 : per_node};
    uint64_t* D = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(fn_off[n] > 0 ? fn_off[n] : 1));
    uint32_t* u = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    uint8_t* s_next = (uint8_t*)malloc((size_t)n);
    uint32_t* Cg = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    uint8_t* gam = (uint8_t*)malloc((size_t)n);
    if (!D || !u || !s_next || !Cg || !gam) {
        free(D); free(u); free(s_next); free(Cg); free(gam);
        return 1;
    }
    /* geometric mode: selection thresholds with no perturbation share (T_p = 0) */
    oracle_selection_thresholds(n, fn_off, sel_prob, geometric ? 0.0 : p, D);
    uint32_t Tp = oracle_perturbation_threshold(p);
    if (geometric)
        oracle_geometric_table(n, p, Cg);

    for (int64_t c = 0; c < nchains; ++c) {
        uint32_t chain = chain_ids[c];
        uint8_t* s = state + c * (int64_t)n;
        if (init)
            for (int32_t i = 0; i < n; ++i)
                s[i] = (uint8_t)(oracle_word(seed, chain, 0, (uint32_t)i) >> 31);
        for (int64_t r = 1; r <= burn_in + steps; ++r) {
            uint64_t t = (uint64_t)(step0 + r);
            for (int32_t i = 0; i < n; ++i)
                u[i] = oracle_word(seed, chain, t, (uint32_t)i);
            if (geometric) {
                if (geometric_gamma(Cg, n, seed, chain, t, gam) > 0) {
                    for (int32_t i = 0; i < n; ++i) /* s(t+1) = s(t) XOR gamma(t) */
                        s_next[i] = (uint8_t)(s[i] ^ gam[i]);
                } else {
                    step_with_words(&m, 0u, D, s, u, s_next); /* no perturbation: f(t)(s(t)) */
                }
            } else {
                step_with_words(&m, Tp, D, s, u, s_next);
            }
            memcpy(s, s_next, (size_t)n);
            if (r > burn_in) {
                int I = 1;
                for (int32_t q = 0; q < k; ++q)
                    if (s[pred_node[q]] != pred_value[q])
                        I = 0;
                I_out[c * steps + (r - burn_in - 1)] = (uint8_t)I;
            }
        }
    }
    free(D); free(u); free(s_next); free(Cg); free(gam);
    return 0;
}
