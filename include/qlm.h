/*
 * qlm.h -- C ABI of the B200 bulk RWT-scoring library (libqlm.so).
 *
 * The library evaluates QLM's Request Waiting Time (RWT) estimator
 * (Sec. 6, Eqs. 1-5) in bulk over candidate orderings of
 * request groups into virtual queues, scores each ordering with the global
 * scheduler's objective (Sec. 7, Eqs. 6-11 + objective, L665-767) and picks
 * the best one.  "P:Lx" cites /root/reference/PAPER.md line x, "S:Lx"
 * SPEC.md line x; R-numbers are the readings listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Return an int status (qlm_status); 0 = QLM_OK.  No exception or abort
 *    crosses the ABI.  On error, qlm_last_error() returns a thread-local
 *    message naming the offending field and index.
 *  - Host arrays passed to qlm_create / qlm_update_groups are deep-copied;
 *    the caller may free them on return.
 *  - Device arrays (candidate rows, outputs) are caller-owned device memory
 *    (e.g. torch tensors' data_ptr) on the context's device, 16-byte
 *    aligned where stated.  The context owns its tables and scratch.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Bulk calls
 *    are asynchronous on it; calls on one context must be stream-ordered
 *    (a context is not thread-safe).
 *  - No CPU fallback: if the device is not an sm_100 part, qlm_create fails
 *    with QLM_ECUDA.
 */
#ifndef QLM_H
#define QLM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QLM_ABI_VERSION 4

#if defined(__GNUC__)
#define QLM_API __attribute__((visibility("default")))
#else
#define QLM_API
#endif

typedef enum {
    QLM_OK = 0,
    QLM_EINVAL = 1,     /* invalid argument; qlm_last_error names it           */
    QLM_ENOMEM = 2,     /* device allocation failed                             */
    QLM_ECUDA = 3,      /* CUDA runtime error / unsupported device              */
    QLM_ENCCL = 4,      /* NCCL missing or a communicator call failed           */
    QLM_EBADORDER = 5,  /* a row is not a permutation of 0..T-1 (Eq. 6)         */
    QLM_ERANGE = 6      /* T > 32768, ENUM index >= T!, index overflow          */
} qlm_status;

typedef struct qlm_ctx qlm_ctx;

/* A request group (Def. P:L443-447): homogeneous in model and SLO.        */
typedef struct {
    int32_t model;     /* [0, M): model served (m_i of Eq. 7)          */
    int32_t n_req;     /* >= 1 requests in the group (<= 65536 if dist_id >= 0)     */
    double slo_s;      /* > 0, finite: TTFT deadline in seconds (Def. 2) */
    double mu_out;     /* > 0: mean output tokens per request (Eq. 3)        */
    double var_out;    /* >= 0: variance of output tokens per request (Eq. 3)        */
    int32_t dist_id;   /* MC length table of the group, or -1 (Gaussian only)        */
    int32_t reserved;  /* must be 0                                                   */
} qlm_group;           /* 40 bytes */

/* A virtual queue = one serving instance (Def. P:L449-453, Def. 3). */
typedef struct {
    int32_t device;          /* [0, D): row of the per-device profile tables        */
    int32_t resident_model;  /* [0, M): model loaded at t = 0 (m_{g,-1}, R4)        */
    double backlog_mean_s;   /* >= 0: expected in-flight work pinned ahead (R12)     */
    double backlog_var_s2;   /* >= 0: its variance                                    */
} qlm_queue;                 /* 24 bytes */

/* Offline-profiled constants per (device type, model).
 * Row-major [D][M] unless stated.  The library derives, per (d, m):
 *   tail = prefill + max_out * eps * decode   (C - W, Eq. 1 + Eq. 4, R3)    */
typedef struct {
    int32_t D, M;            /* >= 1 device types, >= 1 models                     */
    const double *theta;     /* > 0 output tokens/s (Theta, Eq. 2)         */
    const double *prefill_s; /* >= 0 prefill time P (Eq. 1)             */
    const double *eps;       /* > 0 inefficiency factor epsilon (Eq. 4)             */
    const double *decode_s;  /* >= 0 decode time per token d (Eq. 4)                */
    const double *max_out;   /* >= 0 max output tokens O_q (Eq. 4)          */
    const double *swap_s;    /* [D][M][M] >= 0 swap time from->to, diagonal 0 (S)   */
} qlm_profile;

/* Output-length quantile tables for the Monte-Carlo mode (R13).           */
typedef struct {
    int32_t K;               /* power of two in [2, 65536]                          */
    int32_t n_tables;        /* >= 1                                                */
    const uint16_t *len;     /* [n_tables][K] output lengths in tokens              */
} qlm_len_tables;

typedef struct {
    double z_clamp;          /* > 0, default 8: v := 0/1 beyond +-z_clamp (R9)      */
    double alpha;            /* [0, 1), default 0.01 (p99): n_over = #{v > alpha} */
    int32_t device;          /* CUDA ordinal                                         */
    int32_t reserved;        /* must be 0                                            */
} qlm_options;

/* Candidate orderings (encoding of Eq. 6, R10): a row of T = G+Q-1 tokens,
 * a permutation of 0..T-1; token < G is a request group, token >= G a
 * queue separator.  Queue q holds the groups between the q-th and the
 * (q+1)-th separator, in order (position j of Eq. 6).                       */
enum { QLM_CAND_EXPLICIT = 0, QLM_CAND_RANDOM = 1, QLM_CAND_ENUM = 2, QLM_CAND_NEIGHBOR = 3 };
#define QLM_MAX_MOVES 8

/* Best-candidate record, device-resident (16 bytes).  key orders
 * candidates lexicographically by (fp32 S1, fp32 S2) (R11); ties go to the
 * lowest index (R14).  key = UINT64_MAX / index = -1 means "none".          */
typedef struct {
    uint64_t key;    /* fp32bits(S1) << 32 | ord32(fp32 S2)                        */
    int64_t index;   /* global candidate index                                      */
} qlm_record;

/* Candidate kinds (R10, R18):
 *   EXPLICIT  rows given by the caller;
 *   RANDOM    candidate c = forward Fisher-Yates permutation from Philox(seed, c)
 *             (R10: 16-bit swap draws, 8 per Philox block, for T <= 256;
 *             32-bit draws, 4 per block, above);
 *   ENUM      candidate c = the c-th permutation in lexicographic order (T <= 20);
 *   NEIGHBOR  candidate c = the base row `rows` (one row of T tokens) with
 *             `moves` Philox(seed, c)-drawn transpositions (R18; SURVEY 8(f) N1,
 *             the neighbourhood of an incumbent ordering for local search).   */
typedef struct {
    int32_t kind;          /* QLM_CAND_*                                             */
    int32_t token_bytes;   /* EXPLICIT / NEIGHBOR: 1 (needs T <= 256) or 2            */
    const void *rows;      /* EXPLICIT: device [count][stride] bytes, 16-B aligned;
                              NEIGHBOR: device base row, T tokens, 16-B aligned       */
    int64_t stride;        /* EXPLICIT: bytes per row, multiple of 16, >= T*token_bytes */
    uint64_t seed;         /* RANDOM / NEIGHBOR: Philox key                           */
    int64_t first;         /* global index of the first candidate (RANDOM/ENUM/NEIGHBOR) */
    int64_t count;         /* number of candidates, >= 0                              */
    const qlm_record *first_from; /* optional device record: if non-NULL, count must be
                              1 and the candidate index is read on the device from
                              first_from->index at kernel time (no host sync); an
                              index < 0 makes the call a no-op on the device.        */
    int32_t moves;         /* NEIGHBOR: transpositions per candidate, 0..QLM_MAX_MOVES */
    int32_t reserved;      /* must be 0                                               */
} qlm_candidates;

typedef struct {
    int64_t index;         /* winner's global candidate index (-1 if count == 0)     */
    float s1, s2;          /* its objective (R11)                                    */
    int32_t n_over;        /* #{groups with v > alpha}                               */
    int32_t reserved;
} qlm_best;

/* ---- lifetime --------------------------------------------------------- */

/* Validate, deep-copy and upload the problem, build the derived tables on
 * the device (per-(d,g) W = n*mu/Theta and n*var/Theta^2, per-(d,m) tail),
 * and synchronise.  `tabs` may be NULL (then every dist_id must be -1);
 * `opt` may be NULL (defaults).  Errors: QLM_EINVAL (named field), QLM_ERANGE
 * (T = G+Q-1 > 32768), QLM_ECUDA (no sm_100 device), QLM_ENOMEM.             */
QLM_API int qlm_create(const qlm_group *groups, int32_t G, const qlm_queue *queues, int32_t Q,
               const qlm_profile *prof, const qlm_len_tables *tabs, const qlm_options *opt,
               qlm_ctx **out);
QLM_API void qlm_destroy(qlm_ctx *ctx);
QLM_API const char *qlm_last_error(void);

/* Replace all G group records (same G) from host memory: validated on the
 * host, deep-copied into a context-owned pinned buffer (the caller may reuse
 * or free the array on return; the device reads the validated snapshot),
 * copied H2D on `stream` and the derived tables rebuilt there (asynchronous).
 * Back-to-back calls wait for the previous call's copy to leave the staging
 * buffer.  A new request arriving in a group is this call.     */
QLM_API int qlm_update_groups(qlm_ctx *ctx, const qlm_group *groups, void *stream);

/* ---- the hot path -------------------------------------------------------- */

/* Per-candidate scores (Gaussian): s1[k], s2[k] (device fp32 [count]) and
 * optionally n_over[k] (device int32 [count], nullable) for candidate
 * first + k.                                                                */
QLM_API int qlm_score_orderings(qlm_ctx *ctx, const qlm_candidates *cand, float *s1, float *s2,
                        int32_t *n_over, void *stream);

/* Argmin over the candidates on this device: writes one qlm_record to
 * `rec` (device memory).  Asynchronous; no host sync.                       */
QLM_API int qlm_best_ordering_async(qlm_ctx *ctx, const qlm_candidates *cand, qlm_record *rec,
                            void *stream);

/* Lexicographic min over n device records (e.g. all-gathered from every
 * rank) -> *out (device).  Asynchronous.                                    */
QLM_API int qlm_reduce_records(qlm_ctx *ctx, const qlm_record *recs, int32_t n, qlm_record *out,
                       void *stream);

/* Synchronous convenience: argmin + decode of the winner into host arrays
 * queue_of_group[G] / pos_of_group[G] (both nullable).                      */
QLM_API int qlm_best_ordering(qlm_ctx *ctx, const qlm_candidates *cand, qlm_best *out,
                      int32_t *queue_of_group, int32_t *pos_of_group, void *stream);

/* The result of a step, read into host memory without a host sync: the
 * candidate named by a device record (`one`: count 1, first_from = the record,
 * a RANDOM / ENUM / NEIGHBOR description) is scored and decoded on `stream`,
 * then out->{index, s1, s2, n_over} and queue_of_group[G] / pos_of_group[G]
 * (nullable) reach the caller's host buffers: pinned (page-locked, mapped)
 * buffers are written by the device directly with one kernel, pageable ones
 * get one copy per field.  Asynchronous: the host values are valid once
 * `stream` reaches this point.  Typical use: the winner record of
 * qlm_score_estimate / qlm_best_ordering_async (global once a communicator is
 * attached).  Errors: QLM_EINVAL (count != 1, no first_from, EXPLICIT).     */
QLM_API int qlm_winner(qlm_ctx *ctx, const qlm_candidates *one, qlm_best *out, int32_t *queue_of_group,
                       int32_t *pos_of_group, void *stream);

/* Request-level violating fractions (R19), asynchronous:
 * request r of group i waits wt_i + r*mu_i/Theta (variance V_i +
 * r*var_i/Theta^2); frac[g][k] = the fraction of group g's requests whose
 * SLO is violated in candidate first + k (mean of the per-request R8/R9
 * probabilities), device fp32 [G][count]; s1_req[k] = sum n_i f_i / sum n_i,
 * device fp32 [count].  Both nullable.  One warp per candidate, O(sum n_i)
 * work per candidate: meant for evaluating winners and short lists.
 * QLM_ERANGE when one candidate's per-group state does not fit in shared
 * memory (G above about 11000).                                            */
QLM_API int qlm_request_violations(qlm_ctx *ctx, const qlm_candidates *cand, float *frac,
                           float *s1_req, void *stream);

/* Two-tier (warm / cold) model swapping (R20):
 * every model goes storage -> CPU memory -> GPU memory; "models present
 * later in the virtual queue are warm and placed in the CPU memory until all
 * the CPU memory is exhausted", the rest are cold.  Per queue on device d,
 * the swap targets in order of their first transition (Eq. 9, m_{-1} =
 * resident) are warm while the sizes taken so far plus model_mem[m] fit in
 * cpu_cap[d]; from the first target that does not fit, CPU memory is
 * exhausted and every new target is cold.  A cold transition adds
 * load_s[d][m] to the swap: trans = tail + (swap + load) (R1/R2).        */
typedef struct {
    const int32_t *model_mem; /* host [M] >= 1: model size (integer units, e.g. GB) */
    const int32_t *cpu_cap;   /* host [D] >= 0: CPU memory of a device-d instance    */
    const double *load_s;     /* host [D][M] >= 0: storage -> CPU load time (s)      */
} qlm_tiers;

/* Set (deep copy, synchronous: drains the context's device first, so no
 * tiered kernel on any stream reads half-updated tables) or clear (tiers =
 * NULL) the context's tier tables.  Errors: QLM_EINVAL (M > 32, a NULL array, a size < 1, a negative
 * cap, a negative or non-finite load; the message names it), QLM_ERANGE
 * (sum of model_mem > 2^24).                                               */
QLM_API int qlm_set_tiers(qlm_ctx *ctx, const qlm_tiers *tiers);

/* qlm_score_estimate under two-tier swapping (R20): bulk estimates
 * (group-major fp32 [G][count]), per-candidate s1 / s2 / n_over ([count])
 * and the argmin record, every output nullable.  Asynchronous.  One thread
 * per candidate; wt / V follow the oracle's operation order.  Errors:
 * QLM_EINVAL if qlm_set_tiers has not been called, else as
 * qlm_score_estimate.                                                      */
QLM_API int qlm_tiered_score_estimate(qlm_ctx *ctx, const qlm_candidates *cand, float *wt_mean,
                              float *wt_std, float *viol, float *s1, float *s2, int32_t *n_over,
                              qlm_record *rec, void *stream);

/* ---- request-group formation (R21; Alg. 1) ---- */

/* Requests in arrival order, all arrays device memory.                     */
typedef struct {
    int32_t n;                 /* 1 <= n < 2^28                                           */
    int32_t dims;              /* feature dimensions, 1..4                                */
    const int32_t *model;      /* [n] in [0, M): a hard partition (Def. P:L443-447)       */
    const double *slo_s;       /* [n] > 0: the group's SLO is its members' minimum        */
    const int32_t *out_tokens; /* [n] in [0, 65535]: output tokens from the history */
    const int32_t *feat;       /* [n][dims] in [0, 65535]: quantised features (SLO, input /
                                  output token distribution, Def. P:L443-447)             */
} qlm_requests;

/* Alg. 1 under reading R21, on the device: per model m, k-means with
 * k_per_model[m] centres (deterministic farthest-point start, Lloyd
 * iterations in fp64 until no label changes or max_iter), then every
 * cluster larger than `limit` (= delta x average batch) is split
 * in half by arrival order, recursively (splitHalf).  Outputs: label_of[n]
 * (device, cluster of each request), group_of[n] (device, group id;
 * groups are numbered cluster by cluster, halves left to right) and the
 * first min(n_groups, group_cap) records of groups[] (device qlm_group:
 * model, n_req, slo_s = min member SLO, mu_out / var_out = mean /
 * population variance of the members' out_tokens, dist_id = -1) ready for
 * qlm_create.  *n_groups (host) = the number of groups, *iters (host,
 * nullable) = Lloyd iterations run.  Synchronises `stream`; device scratch
 * is stream-ordered (cudaMallocAsync).  `device` = CUDA ordinal.
 * Errors: QLM_EINVAL (bad sizes: k_per_model[m] in [1, 1024] with sum <=
 * 1024, limit in [1, 32768], max_iter in [1, 1000]; a request with a model,
 * SLO, output length or feature out of range -- checked on the device),
 * QLM_ERANGE (n_groups > group_cap; *n_groups is still set).               */
QLM_API int qlm_form_groups(const qlm_requests *req, int32_t M, const int32_t *k_per_model,
                            int32_t limit, int32_t max_iter, int32_t *label_of, int32_t *group_of,
                            qlm_group *groups, int32_t group_cap, int32_t *n_groups, int32_t *iters,
                            int32_t device, void *stream);

/* qlm_mc_count under two-tier swapping (R13 + R20): counts[k][g] with the
 * warm/cold transition costs of qlm_set_tiers.  Same contract as
 * qlm_mc_count; QLM_EINVAL if no tier tables are set.                      */
QLM_API int qlm_tiered_mc_count(qlm_ctx *ctx, const qlm_candidates *cand, int64_t trial_count,
                                uint32_t *counts, void *stream);

/* Local-search step (R18), asynchronous on `stream`:
 * if *rec (e.g. from qlm_best_ordering_async over NEIGHBOR candidates of
 * base row cand->rows) has index >= 0 and a key strictly below
 * incumbent->key, the winning candidate's row is materialised into
 * cand->rows (in place, it becomes the new base row) and *incumbent = *rec;
 * otherwise nothing changes.  cand must be NEIGHBOR; rec and incumbent are
 * device records; the decision is taken on the device (no host sync).      */
QLM_API int qlm_adopt_best(qlm_ctx *ctx, const qlm_candidates *cand, const qlm_record *rec,
                   qlm_record *incumbent, void *stream);

/* Iterated best-of-N local search (R18), entirely asynchronous on `stream`:
 * scores the device row `row` (T tokens of token_bytes each, 16-B aligned)
 * into *incumbent, then for it = 0..iters-1 scores NEIGHBOR candidates
 * [it*per_iter, (it+1)*per_iter) of the current row (seed, moves) and adopts
 * the argmin if it improves the key (qlm_adopt_best).  On completion `row`
 * holds the best ordering found and *incumbent its key (index = the
 * candidate index it was adopted from, -1 if the start row was kept).
 * Unless the stream is already capturing, the 2*iters + 2
 * launches are captured into a CUDA graph kept in the context (updated in
 * place by later calls) and launched as one unit (the
 * scheduler must stay off the critical path).  Errors: QLM_EINVAL (moves
 * outside 1..QLM_MAX_MOVES, per_iter < 1, iters < 0, NULL pointers,
 * misaligned row).                                                         */
QLM_API int qlm_local_search(qlm_ctx *ctx, void *row, int32_t token_bytes, int32_t moves,
                     int64_t per_iter, int32_t iters, uint64_t seed, qlm_record *incumbent,
                     void *stream);

/* Bulk per-group estimates for every candidate (Eq. 2/3/10), group-major:
 * device fp32 [G][count] arrays, element [g][k] = group g in candidate
 * first + k, each nullable:  wt_mean = expected waiting time (s), wt_std =
 * sqrt(variance), viol = SLO-violation probability (R8, R9).  Outputs that
 * are 16-B aligned with count % 4 == 0 leave through bulk async copies.    */
QLM_API int qlm_rwt_estimate(qlm_ctx *ctx, const qlm_candidates *cand, float *wt_mean, float *wt_std,
                     float *viol, void *stream);

/* The whole Gaussian hot path in ONE pass over the candidates: the bulk
 * estimates of qlm_rwt_estimate, the per-candidate scores of
 * qlm_score_orderings and the argmin record of qlm_best_ordering_async,
 * every output nullable.  Asynchronous.                                    */
QLM_API int qlm_score_estimate(qlm_ctx *ctx, const qlm_candidates *cand, float *wt_mean,
                       float *wt_std, float *viol, float *s1, float *s2, int32_t *n_over,
                       qlm_record *rec, void *stream);

/* Monte-Carlo estimate (R13): samples trials [trial_first, trial_first +
 * trial_count) of every group's total output tokens with Philox (key =
 * mc_seed), walks each candidate's queues with the sampled work and writes
 * counts[k][g] = #{trials with W_g > slo_g} (device uint32 [count][G],
 * overwritten).  Needs length tables.  trial_first + trial_count <= 2^32.
 * Equivalent to qlm_mc_sample followed by qlm_mc_count on `stream`.        */
QLM_API int qlm_mc_estimate(qlm_ctx *ctx, const qlm_candidates *cand, uint64_t mc_seed,
                    int64_t trial_first, int64_t trial_count, uint32_t *counts, void *stream);

/* The candidate-independent half of the MC mode: per (group, trial) the
 * sampled total output tokens X and the work X / Theta[d][m_g] for every
 * device row d, kept in the context.  It touches no state the scan calls
 * use, so it may run on another stream concurrently with them.             */
QLM_API int qlm_mc_sample(qlm_ctx *ctx, uint64_t mc_seed, int64_t trial_first,
                          int64_t trial_count, void *stream);

/* The candidate-dependent half: counts for `cand` from the samples of the
 * last qlm_mc_sample (which must be complete on `stream`, e.g. via an
 * event); trial_count must match it.                                        */
QLM_API int qlm_mc_count(qlm_ctx *ctx, const qlm_candidates *cand, int64_t trial_count,
                         uint32_t *counts, void *stream);

/* Decode candidates into per-group queue index and position (x_{g,i,j} of
 * Eq. 6): device int32 [count][G] each (nullable).                         */
QLM_API int qlm_decode(qlm_ctx *ctx, const qlm_candidates *cand, int32_t *queue_of_group,
               int32_t *pos_of_group, void *stream);

/* Materialise candidate rows as uint16 tokens: device [count][T].          */
QLM_API int qlm_rows(qlm_ctx *ctx, const qlm_candidates *cand, uint16_t *rows_out, void *stream);

/* Validate EXPLICIT rows (Eq. 6 bijection); synchronous.  *n_bad = number
 * of rows that are not permutations of 0..T-1.                              */
QLM_API int qlm_check_rows(qlm_ctx *ctx, const qlm_candidates *cand, int64_t *n_bad, void *stream);

/* ---- multi-GPU: one NCCL communicator per context ----------
 * The scheduler makes ONE global choice of plan (objective
 * P:L761-767) while candidates (and MC trials) are sharded over the GPUs of a
 * box, one process and one context per GPU, each rank passing its own
 * candidate range (and trial range).  Once a communicator is attached, every
 * call that produces an argmin record returns the GLOBAL record -- the
 * lexicographic (S1, S2, index) min over all ranks (R11/R14), the same on
 * every rank -- and every MC count is the sum over ranks:
 *   qlm_best_ordering_async, qlm_score_estimate (rec), qlm_tiered_score_estimate
 *   (rec): one 16-B NCCL all-gather + qlm_reduce_records on `stream`, no host
 *   synchronisation;
 *   qlm_best_ordering: the global record, scored and decoded by the rank
 *   whose range holds it and shared with one NCCL max all-reduce (so EXPLICIT
 *   rows never leave their rank);
 *   qlm_mc_count, qlm_mc_estimate, qlm_tiered_mc_count: counts summed with one
 *   NCCL all-reduce on `stream`;
 *   qlm_local_search: iteration it's candidates [it*per_iter, (it+1)*per_iter)
 *   are split into contiguous rank shards; the global winner is adopted on
 *   every rank, so the incumbent stays identical everywhere.
 * These calls are then collective: every rank must make the same sequence of
 * them.  NCCL is loaded at run time (the copy torch already loaded, else
 * libnccl.so.2 or $QLM_NCCL_PATH); without it the comm calls return
 * QLM_ENCCL and everything else works as before.                            */
#define QLM_COMM_ID_BYTES 128

/* A fresh NCCL unique id (rank 0 calls it and broadcasts the 128 bytes to
 * the other ranks, e.g. with torch.distributed).  Host memory, caller-owned. */
QLM_API int qlm_comm_unique_id(uint8_t id[QLM_COMM_ID_BYTES]);

/* Collective over `world` ranks: create this context's communicator (rank
 * `rank`, on the context's device) from the broadcast id and attach it.
 * Each rank's context must be on a different GPU.  Errors: QLM_EINVAL (rank
 * not in [0, world), world < 1, already attached), QLM_ENCCL, QLM_ENOMEM.  */
QLM_API int qlm_comm_attach(qlm_ctx *ctx, const uint8_t id[QLM_COMM_ID_BYTES], int32_t rank,
                            int32_t world);

/* Destroy and detach the communicator (qlm_destroy also does it).  Calls
 * return to per-device results.  Synchronises the context's device.          */
QLM_API int qlm_comm_detach(qlm_ctx *ctx);

/* *rank, *world of the attached communicator (0, 1 when none is attached);
 * *nccl_version = NCCL's version code (0 when NCCL is not loaded).          */
QLM_API int qlm_comm_info(const qlm_ctx *ctx, int32_t *rank, int32_t *world, int32_t *nccl_version);

/* ---- introspection --------------------------------------------------------- */
QLM_API int qlm_dims(const qlm_ctx *ctx, int32_t *G, int32_t *Q, int32_t *T, int32_t *D, int32_t *M);
QLM_API int64_t qlm_kernel_launches(void);   /* kernels launched by this process so far */

/* Testing: restrict the kernel selection process-wide so tests can compare
 * the kernels that implement one call (they must agree bit for bit, R22).
 * flags: QLM_OVERRIDE_* bits (0 = the measured default choice); ilv_cap > 0
 * limits the candidates per chunk of the large-T two-phase path (0 = the
 * default).  Errors: QLM_EINVAL on unknown bits or ilv_cap < 0.             */
#define QLM_OVERRIDE_NO_WS 1u          /* no warp-specialised kernels (qlm_ws.cu, qlm_ws2.cu) */
#define QLM_OVERRIDE_NO_WS2 2u         /* no D = 1 warp-specialised kernel (qlm_ws2.cu)       */
#define QLM_OVERRIDE_NO_TWO_PHASE 4u   /* no two-phase large-T RANDOM path                    */
#define QLM_OVERRIDE_NO_WIDE 8u        /* no warp-per-candidate large-G bulk kernel           */
#define QLM_OVERRIDE_NO_TIER_WARP 16u  /* no lane-per-queue tiered kernel                     */
#define QLM_OVERRIDE_NO_GRAPH 32u      /* qlm_local_search launches directly (no CUDA graph)   */
#define QLM_OVERRIDE_NO_LARGE 64u      /* no D = 1 thread-per-candidate large-T scorer (qlm_large.cu) */
#define QLM_OVERRIDE_ALL 127u
QLM_API int qlm_set_kernel_overrides(uint32_t flags, int64_t ilv_cap);
QLM_API int qlm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QLM_H */
