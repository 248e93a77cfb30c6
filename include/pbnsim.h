/*
 * pbnsim.h -- C ABI of libpbnsim, the B200 (sm_100a) PBN trajectory engine.
 *
 * The hot path of Mizera, Pang & Yuan, "Parallel Approximate Steady-state
 * Analysis of Large Probabilistic Boolean Networks" (arXiv 1508.07828):
 * synchronous simulation of many independent PBN trajectories with fused
 * per-chain statistics, plus the host statistics and driver that consume
 * them.  Citations: P:n = line n of the paper's PAPER.md; readings Qn are
 * listed in DESIGN.md.
 *
 * Conventions (all calls)
 *   - No exceptions cross the ABI; every call returns a pbn_status.
 *   - Host pointers are read during the call only; the caller keeps
 *     ownership.  Device pointers are caller-allocated device memory (e.g.
 *     torch tensors' data_ptr()) and are written asynchronously on the
 *     caller's stream.
 *   - A pbn_model owns only its device image; it is immutable after
 *     pbn_load and may be used from several streams concurrently.
 *   - Error text (when err != NULL) is NUL-terminated and truncated to errlen.
 */
#ifndef PBNSIM_H
#define PBNSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PBN_OK = 0,
    PBN_E_INVALID = 1,       /* model or predicate violates an invariant */
    PBN_E_USAGE = 2,         /* bad arguments / unsupported size for this build   */
    PBN_E_DEGENERATE = 3,    /* statistic undefined: W=0, alpha+beta in {0,2}, ... */
    PBN_E_NOT_CONVERGED = 4, /* driver hit its step cap                            */
    PBN_E_IO = 5,
    PBN_E_CUDA = 6,          /* a CUDA runtime call failed                         */
    PBN_E_NOMEM = 7
} pbn_status;

/* Perturbation semantics (reading Q1), chosen at load time. */
enum {
    PBN_PERTURB_VECTOR = 0,   /* any gamma_i(t)=1  =>  s(t+1) = s(t) XOR gamma(t) */
    PBN_PERTURB_PER_NODE = 1, /* node i flips iff gamma_i(t)=1, else applies f     */
    /* VECTOR semantics with gamma(t) drawn by geometric skips from its own word
     * stream (SPEC S:177's optional mode, reading Q18):
     *   k_1 = G(v_0), k_{j+1} = k_j + 1 + G(v_j) until k >= n, gamma_k = 1,
     *   G(v) = #{g < n : Cg[g] <= v}, Cg[g] = floor((1 - q^(g+1)) 2^32),
     *   q = 1 - p (q^(g+1) by repeated fp64 multiplication),
     *   v(chain,t,m) = Philox4x32-10((2^31 + m/4, chain, t mod 2^32, t >> 32), key)[m mod 4];
     * with gamma(t) = 0 node i selects with its word u(chain,t,i) against the
     * unperturbed thresholds Q_j (T_p = 0).  A different random stream from
     * VECTOR's (same law up to the 2^-32 quantisation). */
    PBN_PERTURB_GEOMETRIC = 2
};

/* -------------------------------------------------------------------- */
/* Model                                                     */
/* -------------------------------------------------------------------- */
typedef struct pbn_model_s* pbn_model;

/* CSR description of a PBN G(V, F).  All arrays host memory.
 *   n         1 <= n <= PBN_MAX_NODES
 *   fn_off    [n+1]  node i owns functions fn_off[i] .. fn_off[i+1]-1;
 *                    ell(i) = fn_off[i+1] - fn_off[i] >= 1
 *   par_off   [nf+1] function f reads parents[par_off[f] .. par_off[f+1]-1]
 *   parents   node ids < n, pairwise distinct per function; the FIRST
 *             parent is the most significant bit of the table index (Q5)
 *   tbl_off   [nf+1] in uint32 words; function f has ceil(2^theta/32) words
 *   tables    entry idx of function f is bit (idx & 31) of word
 *             tables[tbl_off[f] + (idx >> 5)]; bit 0 of word 0 = all parents 0
 *   sel_prob  [nf]   c_j^(i) in (0,1]; per node the sum is within 1e-9 of 1
 *   p         perturbation probability, 2^-32 <= p < 1
 *   flags     PBN_PERTURB_* */
typedef struct {
    int32_t n;
    const int32_t* fn_off;
    const int32_t* par_off;
    const uint16_t* parents;
    const int32_t* tbl_off;
    const uint32_t* tables;
    const double* sel_prob;
    double p;
    uint32_t flags;
} pbn_model_desc;

#define PBN_MAX_NODES 16383   /* one group's state must fit in shared memory   */
#define PBN_MAX_THETA 16      /* parents per predictor function                */
#define PBN_MAX_ELL   128     /* predictor functions per node                  */
#define PBN_MAX_PRED  16      /* (node, value) pairs in a property             */
#define PBN_MAX_PROPS 8       /* properties evaluated by one pbn_simulate call */

/* Host-only validation: returns PBN_OK or PBN_E_INVALID with a
 * message naming the node and the violated rule.  Needs no GPU. */
pbn_status pbn_validate(const pbn_model_desc* desc, char* err, size_t errlen);

/* Validate, quantise p and c to 2^-32 (reading Q3), build the device image
 * and upload it to `device` (the current device if device < 0).
 * *out receives an opaque handle; release it with pbn_free. */
pbn_status pbn_load(const pbn_model_desc* desc, int device, pbn_model* out, char* err,
                    size_t errlen);
void pbn_free(pbn_model model);

typedef struct {
    int32_t n;
    int32_t nf;             /* total predictor functions                        */
    int64_t n_parents;      /* sum of theta over all functions                  */
    double density;         /* D(G) = (1/n) sum_f theta(f)        */
    uint32_t T_p;           /* floor(p 2^32)                                    */
    uint32_t flags;
    int32_t max_ell;
    int32_t max_theta;
    int64_t image_bytes;    /* device image size                                */
} pbn_model_info;

pbn_status pbn_get_model_info(pbn_model model, pbn_model_info* info);

/* -------------------------------------------------------------------- */
/* Trajectories with fused statistics              */
/* -------------------------------------------------------------------- */

/* Property = conjunction of k <= 16 (node, value) pairs.
 * k = 0 means every state is in meta state 1.  Host pointers. */
typedef struct {
    int32_t k;
    const uint16_t* node;
    const uint8_t* value;
} pbn_predicate;

/* One call continues chains chain_base .. chain_base+n_chains-1 (global ids,
 * < 2^32) from s_{step0} and performs burn_in + steps synchronous
 * transitions.  Transition t (s_{t-1} -> s_t) uses the words
 *     u(chain, t, i) = Philox4x32-10(counter = (i/4, chain, t mod 2^32, t >> 32),
 *                                    key = (seed mod 2^32, seed >> 32))[i mod 4]
 * (reading Q2), so outputs are independent of launch shape and of how
 * chains and steps are split into calls (A12).  The recorded window is
 * s_{step0+burn_in+1} .. s_{step0+burn_in+steps} (reading Q6).
 *   init         1: ignore the input state and set s_0[i] = u(chain,0,i) >> 31
 *                (requires step0 == 0; reading Q4)
 *   batch        kappa >= 1 for batch sums of consecutive kappa-blocks of the
 *                window (Fig. 2); 0 = none
 *   emit_bits    1: write the window's indicator bits
 *   bits_offset  window element w goes to bit (bits_offset + w) of its row,
 *                so successive calls can append to one bitstream; the word
 *                holding bit bits_offset is OR-merged (its bits below
 *                bits_offset are kept, bits above must be 0), every other
 *                touched word is overwritten
 *   bits_row_words  row stride of `bits` in u32 (0 = ceil(steps/32))
 *   groups_per_cta  0 or 1 (one 32-chain group per CTA in this build)
 *   warps_per_group warps sharing one group's nodes (0 = auto; <= 28 in this build,
 *                <= 24 for the bit-sliced kernels, whose auto is 20 on a
 *                staged image and 24 on a global one)
 *   schedule     0 auto; 1 one CTA per group; 2 persistent CTAs pulling
 *                (group, chunk of chunk_steps steps) units, state carried
 *                between chunks in `workspace`
 *   chunk_steps  persistent chunk length (0 = auto)
 *   workspace    caller-owned device scratch (see pbn_simulate_workspace_size)
 *   layout       PBN_LAYOUT_*: AUTO picks, per call: the bit-sliced kernel
 *                (K1b, one group per CTA) when the groups fill the GPU and the
 *                model has theta <= 8, ell <= 4, n <= 5460; for few groups its
 *                cluster form (K1bc) or K1c; for <= 128 (256) chains K1n;
 *                K1 otherwise.  CHAIN_LANES forces K1 / K1c, NODE_LANES K1n,
 *                BITSLICE K1b (cluster_size >= 2: K1bc); pbn_last_kernel()
 *                names the kernel a call ran
 *   chains_per_cluster  K1n: chains sharing one cluster (0 = auto)
 *   cluster_size 0: chosen per call -- one CTA per 32-chain group when there
 *                are enough groups to fill the GPU, else a thread-block
 *                cluster of K CTAs per group (each stages 1/K of the image and
 *                computes 1/K of the nodes, the state is mirrored through
 *                distributed shared memory); 1 / K force it
 *   n_props, props  several properties from the same trajectories (the
 *                multi-property reuse of P:507-526): every statistic below is
 *                produced per property, property-major (property p's block
 *                follows property p-1's; block sizes as for one property)
 * The launch-shape fields never change any output. */
typedef struct {
    int64_t n_chains;
    int64_t chain_base;
    int64_t step0;
    int64_t burn_in;
    int64_t steps;
    int64_t batch;
    uint64_t seed;
    pbn_predicate pred;
    int32_t init;
    int32_t emit_bits;
    int64_t bits_offset;
    int64_t bits_row_words;
    int32_t groups_per_cta;
    int32_t warps_per_group;
    int32_t schedule;
    int64_t chunk_steps;
    int32_t n_props;                /* 0: one property, `pred`; 1..PBN_MAX_PROPS:  */
    const pbn_predicate* props;     /*    props[0..n_props-1] (pred ignored)       */
    int32_t cluster_size;           /* 0 auto; 1 one CTA per group; 2,4,8,16: a    */
                                    /* cluster of that many CTAs per group         */
    void* workspace;                /* caller-owned DEVICE scratch of at least     */
    int64_t workspace_bytes;        /* pbn_simulate_workspace_size() bytes, or NULL */
    int32_t layout;                 /* PBN_LAYOUT_*: which lanes a warp spreads    */
    int32_t chains_per_cluster;     /* NODE_LANES: chains per cluster, 1..32 (0 = auto) */
} pbn_sim_args;

/* Kernel layouts (pbn_sim_args.layout).  Outputs never depend on it. */
enum {
    PBN_LAYOUT_AUTO = 0,        /* chosen per call from the chain count and image size  */
    PBN_LAYOUT_CHAIN_LANES = 1, /* 32 chains per warp, bit-sliced state (K1, K1c)       */
    PBN_LAYOUT_NODE_LANES = 2,  /* one chain per cluster of cluster_size CTAs (0 = auto), */
                                /* threads over node quads, bit-packed state (K1n)     */
    PBN_LAYOUT_BITSLICE = 3     /* K1's group layout, functions evaluated bit-sliced    */
                                /* over the 32 chains (K1b; cluster_size >= 2: K1bc);   */
                                /* models with theta <= 8, ell <= 4, n <= 5460; every   */
                                /* semantics; PBN_E_USAGE outside that shape            */
};

/* Caller-owned DEVICE buffers, chain-major (row c = chain chain_base + c).
 *   state       [n_chains x ceil(n/32)] u32, in/out; node i of chain c is
 *               bit (i & 31) of word state[c*ceil(n/32) + (i >> 5)]
 *   c1          [n_chains] number of window states in meta state 1
 *   n01, n10    [n_chains] 0->1 / 1->0 transitions between consecutive
 *               window elements (pairs inside the window only, Q7)
 *   first_last  [n_chains] bit 0 = I of the first window element, bit 1 = last
 *   batch_sums  [n_chains x ceil(steps/batch)] or NULL (last batch may be short)
 *   bits        [n_chains x bits_row_words] or NULL; element w of the window
 *               is bit (b & 31) of word b >> 5 of its row, b = bits_offset + w
 *   totals      [6] u64, overwritten: S1 = sum c1, S2 = sum c1^2, sum n01,
 *               sum n10, sum n0from, sum n1from, where n0from / n1from count
 *               window elements with a successor that are 0 / 1 (A10).
 * Any pointer except state may be NULL if not wanted (totals NULL skips A10).
 * With n_props = q > 1 every array except state holds q property-major
 * blocks: c1[p*n_chains + c], bits[(p*n_chains + c)*bits_row_words + w],
 * batch_sums[(p*n_chains + c)*ceil(steps/batch) + b], totals[6*p + k]. */
typedef struct {
    uint32_t* state;
    uint32_t* c1;
    uint32_t* n01;
    uint32_t* n10;
    uint8_t* first_last;
    uint32_t* batch_sums;
    uint32_t* bits;
    uint64_t* totals;
} pbn_sim_out;

/* Enqueue the trajectory kernel on `cuda_stream` (a cudaStream_t; NULL =
 * legacy default stream).  Asynchronous: the caller synchronises.  Errors:
 * PBN_E_USAGE (bad sizes, init with step0 != 0, > 2^32 chains, model too
 * large for shared memory), PBN_E_CUDA (launch failure). */
pbn_status pbn_simulate(pbn_model model, const pbn_sim_args* args, const pbn_sim_out* out,
                        void* cuda_stream);

/* Device scratch a pbn_simulate call with these args may need (the
 * persistent schedule suspends each 32-chain group's bit-sliced state and
 * counters between step chunks): *bytes = 0 when none can be needed.  Only
 * n_chains and n_props of `args` are read.  Passing a buffer of at least this
 * size as args->workspace makes pbn_simulate allocation-free; with
 * workspace = NULL a persistent launch makes one stream-ordered
 * cudaMallocAsync/cudaFreeAsync pair.  A workspace is used by one call at a
 * time (calls on one stream may share it).  PBN_E_USAGE for bad arguments. */
pbn_status pbn_simulate_workspace_size(pbn_model model, const pbn_sim_args* args, int64_t* bytes);

/* Recount (K2) window statistics of a sub-window [start, start+length) of a
 * stored indicator bitstream (device) without re-simulation: used by the
 * Algorithm 4 burn-in re-check and by Skart re-batching
 * (P:368).  bits has row stride `row_words` u32 per chain.  Outputs
 * as in pbn_sim_out (device, any may be NULL). */
pbn_status pbn_recount(const uint32_t* bits, int64_t n_chains, int64_t row_words, int64_t start,
                       int64_t length, int64_t batch, uint32_t* c1, uint32_t* n01, uint32_t* n10,
                       uint8_t* first_last, uint32_t* batch_sums, uint64_t* totals,
                       void* cuda_stream);

/* -------------------------------------------------------------------- */
/* Host statistics, fp64                              */
/* -------------------------------------------------------------------- */

/* Gelman & Rubin potential scale reduction factor (Alg 3) of
 * omega >= 2 windows of length psi >= 2 over the 0/1 indicator, from
 * S1 = sum_i c_i and S2 = sum_i c_i^2 (exact integers):
 *   B = psi/(omega-1) sum (mu_i - mu)^2,  W = (1/omega) sum s_i^2 (divisor psi-1),
 *   sigma2 = (1 - 1/psi) W + B/psi,       rhat = sqrt(sigma2 / W).
 * PBN_E_DEGENERATE when W = 0 (all windows constant); outputs may be NULL. */
pbn_status pbn_gelman_rubin(uint64_t S1, uint64_t S2, int64_t omega, int64_t psi, double* rhat,
                            double* B, double* W, double* sigma2);

/* Two-state Markov chain rule (Alg 1 line 8) from pooled counts:
 * alpha = n01/n0from, beta = n10/n1from, then
 *   M = ceil( log(eps (alpha+beta)/max(alpha,beta)) / log|1-alpha-beta| )
 *   N = ceil( alpha beta (2-alpha-beta)/(alpha+beta)^3 * Phi^-1((1+s)/2)^2 / r^2 ).
 * alpha+beta = 1 gives M = 1 (reading Q10).  PBN_E_DEGENERATE when n0from
 * or n1from is 0 or alpha+beta is 0 or 2.  M_raw / N_raw are the values
 * before ceil. */
typedef struct {
    double alpha, beta, M_raw, N_raw;
    int64_t M, N;
} pbn_two_state_result;

pbn_status pbn_two_state(uint64_t n01, uint64_t n0from, uint64_t n10, uint64_t n1from, double r,
                         double s, double eps, pbn_two_state_result* res);

/* Standard normal quantile Phi^-1(q), 0 < q < 1 (|error| < 1e-15 relative). */
double pbn_inv_norm_cdf(double q);
/* Student-t quantile with df >= 1 degrees of freedom. */
double pbn_t_quantile(double q, double df);

/* Skart CI step (Alg 2 lines 10-14 / Alg 5 lines 13-16, P:372-382,
 * P:564-575) over batch means of omega chains laid out chain-major
 * (batches never straddle chains, Fig. 2b): given per-chain batch sums
 * [omega x per_chain] of batch size kappa, returns the grand mean mu, the
 * skewness- and autoregression-adjusted CI and H = max(mu-lo, hi-mu).
 * Declared Skart constants per SPEC S:375 (reading Q11/Q12). */
typedef struct {
    double mu, var, phi, skew, ci_lo, ci_hi, H;
    int64_t batches;
} pbn_skart_ci;

pbn_status pbn_skart_ci_from_batches(const uint32_t* batch_sums, int64_t omega, int64_t per_chain,
                                     int64_t kappa, double alpha_conf, pbn_skart_ci* res);

/* Skart sample sizing (Alg 5 lines 3-21; Alg 2) over
 * the pooled 0/1 indicator samples of omega converged chains held as DEVICE
 * bitstreams: chain c's sample element w is bit (start + w) of row c of
 * `bits` (row stride row_words u32, layout of pbn_sim_out.bits), the first
 * `available` elements of every row are valid.  Batches never straddle
 * chains (p is rounded up to a multiple of omega, Fig. 2b); batch
 * sums come from K2 recounts of the bits.  Declared Skart constants per SPEC
 * S:375 (reading Q11), chain-major batch means without cross-chain pairs
 * (Q12).  Returns
 *   PBN_OK               the CI meets H <= h_star: res complete;
 *   PBN_E_NOT_CONVERGED  res->need_per_chain > available: extend every chain
 *                        to that many samples and call again (the machine
 *                        replays its decisions on the unchanged prefix, so
 *                        repeated calls take the decisions of one pass);
 *                        need_per_chain = 0: an iteration cap (64) was hit;
 *   PBN_E_USAGE / PBN_E_CUDA / PBN_E_NOMEM.
 * Synchronises `cuda_stream` (batch sums are read back to the host). */
typedef struct {
    double estimate;         /* grand mean of the batch means mu              */
    double ci_lo, ci_hi;     /* skewness- and autoregression-adjusted CI      */
    double H;                /* max(mu - ci_lo, ci_hi - mu) <= h_star         */
    double skew;             /* skewness of the first 1280 samples (line 5)   */
    int64_t kappa;           /* final batch size                              */
    int64_t batches;         /* final batch count p (multiple of omega)       */
    int64_t spacer;          /* final spacer d (randomness-test failures)     */
    int64_t eta;             /* kappa * p samples used                        */
    int64_t need_per_chain;  /* PBN_E_NOT_CONVERGED: samples per chain needed */
    int32_t randomness_tests;
} pbn_skart_result;

pbn_status pbn_skart(const uint32_t* bits, int64_t omega, int64_t row_words, int64_t start,
                     int64_t available, double h_star, double alpha_conf, pbn_skart_result* res,
                     void* cuda_stream);

/* -------------------------------------------------------------------- */
/* Host driver: Algorithm 3 then Algorithm 4 or 5           */
/* -------------------------------------------------------------------- */
enum { PBN_METHOD_TWO_STATE = 0, PBN_METHOD_SKART = 1 };

typedef struct {
    int32_t method;          /* PBN_METHOD_*                                     */
    int64_t omega;           /* chains >= 2                                      */
    int64_t psi0;            /* initial Gelman-Rubin half length (Alg 3)         */
    double rhat_threshold;   /* "close to 1": stop when rhat < threshold (Q8)    */
    double r, s, eps;        /* two-state precision, confidence, epsilon         */
    double h_star, alpha_conf; /* Skart precision and confidence parameter       */
    uint64_t seed;
    pbn_predicate pred;
    int64_t max_steps;       /* per-chain step cap (PBN_E_NOT_CONVERGED)         */
} pbn_run_args;

typedef struct {
    double estimate;         /* steady-state probability of the property         */
    double ci_lo, ci_hi;     /* Skart only                                       */
    double rhat;             /* last R-hat (the one that passed)                 */
    int64_t psi;             /* burn-in psi returned by Alg 3 (after Alg 4 re-check) */
    int64_t sample_size;     /* pooled elements used by the estimate             */
    int64_t steps_per_chain; /* total transitions simulated per chain            */
    int64_t gr_iterations;
    int64_t extensions;      /* two-state: Alg 4 extensions; Skart: final spacer d */
    int64_t M, N;            /* two-state: last burn-in M / sample size N;       */
                             /* Skart: final batch size kappa / batch count p    */
    double alpha, beta;
} pbn_run_result;

pbn_status pbn_run(pbn_model model, const pbn_run_args* args, pbn_run_result* res,
                   void* cuda_stream, char* err, size_t errlen);

/* The same driver over chains spread across several GPUs:
 * this process simulates chains [chain_base, chain_base + omega_local) of
 * args->omega (global chain ids: the random stream, hence every chain, is the
 * one of a single-GPU run; omega_local >= 1 on every shard) and calls
 * allreduce(values, count, ctx) -- an in-place element-wise sum over all
 * shards of `count` u64 values, returning 0 on success -- whenever a decision
 * needs pooled numbers.  values[0] is an error flag (a shard that failed
 * locally sends 1 and returns; every other shard then returns PBN_E_CUDA
 * instead of waiting in a collective the failed shard never reaches); the
 * rest are, for the two-state method and the Gelman & Rubin loop, the six
 * counts (S1, S2, n01, n10, n0from, n1from) (Alg 3 line 9; Alg 4
 * lines 8-10), and for Skart the all-gather of the per-chain
 * batch sums [omega x per_chain] (chain-major; each shard fills its own rows,
 * the others are 0; batches never straddle chains, Fig. 2b).  All
 * shards take the same decisions and call allreduce the same number of times
 * with the same counts.  The result is identical to pbn_run over all omega
 * chains. */
typedef int (*pbn_allreduce_u64_fn)(uint64_t* values, int32_t count, void* ctx);

pbn_status pbn_run_sharded(pbn_model model, const pbn_run_args* args, int64_t chain_base,
                           int64_t omega_local, pbn_allreduce_u64_fn allreduce, void* ctx,
                           pbn_run_result* res, void* cuda_stream, char* err, size_t errlen);

/* Several properties from one set of trajectories: Algorithm 3, then
 * Algorithm 4 with the multi-property reuse of samples (reading
 * Q13).  The omega chains are abstracted into n_props meta-state sequences
 * in the same kernel launches (pbn_simulate with n_props).  Gelman & Rubin
 * converges when every property with non-constant windows has R-hat below
 * the threshold; the pooled sample then grows to the smallest per-property
 * N that is not yet met until every N is met; the burn-in
 * re-check uses the largest M.  args->method must be PBN_METHOD_TWO_STATE;
 * args->pred is ignored.  per_prop[n_props] receives each property's
 * estimate, M, N, alpha, beta, R-hat and status (PBN_E_DEGENERATE for a
 * property whose two-state statistics are undefined: it is reported, not
 * fatal, and does not drive the extension).  res receives the shared
 * numbers (psi, pooled sample size, steps per chain, iterations, largest
 * R-hat; estimate/M/N/alpha/beta of property 0). */
typedef struct {
    double estimate;
    double rhat;
    double alpha, beta;
    int64_t M, N;
    int32_t status;          /* pbn_status of this property's two-state step  */
} pbn_prop_result;

pbn_status pbn_run_multi(pbn_model model, const pbn_run_args* args, const pbn_predicate* props,
                         int32_t n_props, pbn_run_result* res, pbn_prop_result* per_prop,
                         void* cuda_stream, char* err, size_t errlen);

/* Version string of the build, e.g. "libpbnsim 0.1 sm_100a". */
const char* pbn_version(void);

/* Name of the trajectory kernel the calling thread's most recent successful
 * pbn_simulate launched: "K1b" (bit-sliced evaluation), "K1" (chain lanes,
 * image in shared memory), "K1-global" (image through L1/L2), "K1c"
 * (cluster), "K1n" (lanes over nodes); "" before the first launch.  A static
 * string; thread-local state, no device call. */
const char* pbn_last_kernel(void);

#ifdef __cplusplus
}
#endif

#endif /* PBNSIM_H */
