// qlm_api.cu -- the C ABI (include/qlm.h): validation, context, device memory,
// argument marshalling to the kernels in qlm_kernels.cu.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "qlm_comm.h"
#include "qlm_launch.h"

using namespace qlm;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(QLM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool is_fin(double x) { return std::isfinite(x); }

}  // namespace

struct qlm_ctx {
    int device = 0;
    Dims dm{};
    double z_clamp = 8.0, zc2 = 64.0;
    float alpha = 0.01f;
    bool has_tables = false;
    // raw uploads (one allocation)
    void *d_raw = nullptr;
    qlm_group *d_groups = nullptr;
    qlm_queue *d_queues = nullptr;
    double *d_theta = nullptr, *d_prefill = nullptr, *d_eps = nullptr, *d_dec = nullptr,
           *d_maxo = nullptr, *d_swap = nullptr;
    // derived tables (one allocation)
    void *d_tab = nullptr;
    Tables tb{};
    // scratch
    qlm_record *d_block_recs = nullptr;
    unsigned int *d_counter = nullptr;
    qlm_record *d_rec = nullptr;           // sync best_ordering
    qlm_record *d_ls_rec = nullptr;        // local search: per-iteration winner
    int32_t *d_dec_out = nullptr;          // [2][G] sync decode
    unsigned long long *d_bad = nullptr;
    int max_blocks = 0;
    uint32_t *d_ilv = nullptr;         // large-T RANDOM: interleaved row chunk
    int64_t ilv_cap = 0;               // candidates per chunk
    qlm_record *d_chunk_recs = nullptr;
    double *d_X = nullptr;             // MC: (X / Theta)[D][G][trials]
    int64_t mc_trials = -1;            // trials of the last qlm_mc_sample
    size_t X_cap = 0;
    void *d_tier = nullptr;            // two-tier swapping (R20): mem [M] | cap [D] | load [D][M]
    bool has_tiers = false;
    // multi-GPU (qlm_comm_attach): the communicator and its scratch
    Comm *comm = nullptr;
    cudaGraphExec_t ls_exec = nullptr;     // qlm_local_search's captured launches
    cudaStream_t aux = nullptr;            // blocking stream standing in for the legacy default stream
    std::vector<int64_t> ls_sig;           // arguments the captured search was built from
    qlm_record *d_comm_recs = nullptr;     // [world] gathered records
    int32_t *d_comm_buf = nullptr;         // [2G + 5] winner decode / scores (max all-reduce)
    std::vector<qlm_group> groups;
    int slo_hi_only = 0;                   // every groups[i].slo_s has a zero low word
    qlm_group *h_stage = nullptr;          // pinned staging of qlm_update_groups (deep copy)
    cudaEvent_t ev_stage = nullptr;        // the staging's last H2D copy
    std::vector<qlm_queue> queues;
    std::vector<double> prof;              // theta|prefill|eps|dec|maxo [D*M] each, swap [D*M*M]
};

namespace {

size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

int validate_groups(const qlm_group *g, int G, int M, int n_tables) {
    for (int i = 0; i < G; ++i) {
        const qlm_group &x = g[i];
        if (x.model < 0 || x.model >= M)
            return fail(QLM_EINVAL, "groups[%d].model=%d not in [0,M=%d)", i, x.model, M);
        if (x.n_req < 1) return fail(QLM_EINVAL, "groups[%d].n_req=%d must be >= 1", i, x.n_req);
        if (!(x.slo_s > 0.0) || !is_fin(x.slo_s))
            return fail(QLM_EINVAL, "groups[%d].slo_s=%g must be > 0 and finite", i, x.slo_s);
        if (!(x.mu_out > 0.0) || !is_fin(x.mu_out))
            return fail(QLM_EINVAL, "groups[%d].mu_out=%g must be > 0 and finite", i, x.mu_out);
        if (!(x.var_out >= 0.0) || !is_fin(x.var_out))
            return fail(QLM_EINVAL, "groups[%d].var_out=%g must be >= 0 and finite", i, x.var_out);
        if (x.dist_id < -1 || x.dist_id >= n_tables)
            return fail(QLM_EINVAL, "groups[%d].dist_id=%d not in [-1,n_tables=%d)", i, x.dist_id,
                        n_tables);
        if (x.dist_id >= 0 && x.n_req > 65536)
            return fail(QLM_EINVAL, "groups[%d].n_req=%d > 65536 with a length table", i, x.n_req);
        if (x.reserved != 0) return fail(QLM_EINVAL, "groups[%d].reserved must be 0", i);
    }
    // S1's numerator over clamped slots is a sum of n_i kept in fp32 by every
    // kernel: exact while the total request count is below 2^24 (R11)
    int64_t total = 0;
    for (int i = 0; i < G; ++i) total += g[i].n_req;
    if (total >= ((int64_t)1 << 24))
        return fail(QLM_ERANGE, "sum of groups[].n_req = %lld >= 2^24 (S1 is exact below 2^24 requests)",
                    (long long)total);
    return QLM_OK;
}

// The warp-specialised D = 1 kernel keeps only the high word of each slo_s
// (qlm_ws2.cu); exact when every low word is zero (20 s, 60 s, 3600 s, 0.5 s ...).
int slo_hi_only(const std::vector<qlm_group> &g) {
    for (const qlm_group &x : g) {
        uint64_t u;
        memcpy(&u, &x.slo_s, 8);
        if ((uint32_t)u != 0u) return 0;
    }
    return 1;
}

// Every entry point leaves the caller's current device as it found it: the
// context's device is made current for the call and restored on return.
struct DevGuard {
    int prev = -1;
    DevGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
    }
    ~DevGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DevGuard(const DevGuard &) = delete;
    DevGuard &operator=(const DevGuard &) = delete;
};

// NVTX range over an entry point (free when no tool is attached): nsys / ncu
// timelines show every library call with its kernels and collectives.
struct NvtxRange {
    explicit NvtxRange(const char *name) {
        nvtxRangePushA(name);
        qlog(2, "%s", name);
    }
    ~NvtxRange() { nvtxRangePop(); }
};

int check_dev(qlm_ctx *ctx) {
    cudaError_t e = cudaSetDevice(ctx->device);
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "cudaSetDevice");
}

// a8 when a communicator is attached: the global min-loc of every rank's
// record -- one 16-B all-gather and the (key, index) reduction, both on `st`.
int global_record(qlm_ctx *ctx, qlm_record *rec, cudaStream_t st) {
    if (!ctx->comm) return QLM_OK;
    std::string err;
    if (!comm_allgather_bytes(ctx->comm, rec, ctx->d_comm_recs, sizeof(qlm_record), st, err))
        return fail(QLM_ENCCL, "%s", err.c_str());
    cudaError_t e = launch_reduce_records(ctx->d_comm_recs, comm_world(ctx->comm), rec, st);
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "reduce_records (global)");
}

// a12 when a communicator is attached: counts summed over the ranks on `st`.
int global_counts(qlm_ctx *ctx, uint32_t *counts, size_t n, cudaStream_t st) {
    if (!ctx->comm || n == 0) return QLM_OK;
    std::string err;
    if (!comm_allreduce_sum_u32(ctx->comm, counts, n, st, err)) return fail(QLM_ENCCL, "%s", err.c_str());
    return QLM_OK;
}

// Rank r's contiguous shard [first, first + count) of n items.
void shard(int64_t n, int r, int w, int64_t &first, int64_t &count) {
    const int64_t base = n / w, extra = n % w;
    first = r * base + (r < extra ? r : extra);
    count = base + (r < extra ? 1 : 0);
}

int check_cand(const qlm_ctx *ctx, const qlm_candidates *c) {
    if (!c) return fail(QLM_EINVAL, "cand is NULL");
    const int T = ctx->dm.T;
    if (c->count < 0) return fail(QLM_EINVAL, "cand.count=%lld < 0", (long long)c->count);
    if (c->first_from && c->count != 1)
        return fail(QLM_EINVAL, "cand.first_from requires cand.count == 1");
    switch (c->kind) {
    case QLM_CAND_EXPLICIT:
        if (c->token_bytes != 1 && c->token_bytes != 2)
            return fail(QLM_EINVAL, "cand.token_bytes=%d must be 1 or 2", c->token_bytes);
        if (c->token_bytes == 1 && T > 256)
            return fail(QLM_EINVAL, "cand.token_bytes=1 needs T=%d <= 256", T);
        if (c->count > 0 && !c->rows) return fail(QLM_EINVAL, "cand.rows is NULL");
        if (((uintptr_t)c->rows & 15) != 0) return fail(QLM_EINVAL, "cand.rows not 16-B aligned");
        if (c->stride % 16 != 0 || c->stride < (int64_t)T * c->token_bytes)
            return fail(QLM_EINVAL, "cand.stride=%lld must be a multiple of 16 and >= T*token_bytes=%d",
                        (long long)c->stride, T * c->token_bytes);
        if (c->first_from) return fail(QLM_EINVAL, "cand.first_from not supported for EXPLICIT");
        break;
    case QLM_CAND_RANDOM:
        if (c->first < 0) return fail(QLM_EINVAL, "cand.first=%lld < 0", (long long)c->first);
        if (c->count > 0 && c->first > INT64_MAX - c->count)
            return fail(QLM_ERANGE, "cand.first + cand.count overflows");
        break;
    case QLM_CAND_NEIGHBOR:
        if (c->token_bytes != 1 && c->token_bytes != 2)
            return fail(QLM_EINVAL, "cand.token_bytes=%d must be 1 or 2", c->token_bytes);
        if (c->token_bytes == 1 && T > 256)
            return fail(QLM_EINVAL, "cand.token_bytes=1 needs T=%d <= 256", T);
        if (!c->rows) return fail(QLM_EINVAL, "cand.rows (NEIGHBOR base row) is NULL");
        if (((uintptr_t)c->rows & 15) != 0) return fail(QLM_EINVAL, "cand.rows not 16-B aligned");
        if (c->moves < 0 || c->moves > QLM_MAX_MOVES)
            return fail(QLM_EINVAL, "cand.moves=%d must lie in [0, %d]", c->moves, QLM_MAX_MOVES);
        if (c->first < 0) return fail(QLM_EINVAL, "cand.first=%lld < 0", (long long)c->first);
        if (c->count > 0 && c->first > INT64_MAX - c->count)
            return fail(QLM_ERANGE, "cand.first + cand.count overflows");
        break;
    case QLM_CAND_ENUM: {
        if (T > 20) return fail(QLM_ERANGE, "ENUM needs T=%d <= 20", T);
        uint64_t f = 1;
        for (int k = 2; k <= T; ++k) f *= (uint64_t)k;
        if (c->first < 0) return fail(QLM_EINVAL, "cand.first=%lld < 0", (long long)c->first);
        if (!c->first_from && (uint64_t)c->first + (uint64_t)c->count > f)
            return fail(QLM_ERANGE, "ENUM range [%lld, %lld) exceeds T!=%llu", (long long)c->first,
                        (long long)(c->first + c->count), (unsigned long long)f);
        break;
    }
    default:
        return fail(QLM_EINVAL, "cand.kind=%d unknown", c->kind);
    }
    return QLM_OK;
}

Cand to_cand(const qlm_candidates *c) {
    Cand d;
    d.kind = c->kind;
    d.tb = c->token_bytes;
    d.rows = static_cast<const uint8_t *>(c->rows);
    d.stride = c->stride;
    d.seed = c->seed;
    d.first = c->first;
    d.count = c->count;
    d.first_from = c->first_from;
    d.moves = c->kind == QLM_CAND_NEIGHBOR ? c->moves : 0;
    return d;
}

ScanParams base_params(const qlm_ctx *ctx, const qlm_candidates *c) {
    ScanParams p;
    memset(&p, 0, sizeof p);
    p.dm = ctx->dm;
    p.tb = ctx->tb;
    p.cd = to_cand(c);
    p.block_recs = ctx->d_block_recs;
    p.counter = ctx->d_counter;
    p.max_blocks = ctx->max_blocks;
    p.zc2 = ctx->zc2;
    p.zc = (float)ctx->z_clamp;
    p.alpha = ctx->alpha;
    p.slo_hi_only = ctx->slo_hi_only;
    return p;
}

// Large-T RANDOM scoring runs in chunks through an interleaved row scratch
// (launch_two_phase); allocated on first use, at most 1 GB (enough candidates
// per chunk to fill every SM with scan warps).
void attach_ilv(qlm_ctx *ctx, ScanParams &p) {
    if (p.cd.kind != QLM_CAND_RANDOM || ctx->dm.T <= 256 || p.cd.first_from || p.cd.count < 4096)
        return;
    if (override_on(QLM_OVERRIDE_NO_TWO_PHASE)) return;   // tests: force the fused fallback
    if (!ctx->d_ilv) {
        const size_t row_bytes = (size_t)((ctx->dm.T + 1) / 2) * 4;
        int64_t cap = (int64_t)(((size_t)1 << 30) / row_bytes);
        cap = cap > 262144 ? 262144 : cap;
        const int64_t ec = g_override_ilv_cap.load();      // tests: small chunks
        if (ec > 0 && ec < cap) cap = ec;
        cap &= ~int64_t(31);
        if (cap < 32) return;
        if (cudaMalloc(&ctx->d_ilv, (size_t)cap * row_bytes) != cudaSuccess) {
            cudaGetLastError();
            ctx->d_ilv = nullptr;
            return;
        }
        if (cudaMalloc(&ctx->d_chunk_recs, 2 * sizeof(qlm_record)) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(ctx->d_ilv);
            ctx->d_ilv = nullptr;
            return;
        }
        ctx->ilv_cap = cap;
    }
    p.ilv = ctx->d_ilv;
    p.ilv_cap = ctx->ilv_cap;
    p.chunk_recs = ctx->d_chunk_recs;
}

int rebuild(qlm_ctx *ctx, cudaStream_t st) {
    cudaError_t e = launch_build(ctx->dm, ctx->d_groups, ctx->d_queues, ctx->d_theta,
                                 ctx->d_prefill, ctx->d_eps, ctx->d_dec, ctx->d_maxo, ctx->d_swap,
                                 ctx->tb, st);
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "build_tables");
}

// The local search's launches (start-row score, then per iteration: the
// neighbourhood argmin, the global exchange when a communicator is attached,
// the adoption), in stream order on `st`.
int enqueue_search(qlm_ctx *ctx, void *row, int32_t token_bytes, int32_t moves, int64_t per_iter,
                   int32_t iters, uint64_t seed, qlm_record *incumbent, cudaStream_t st) {
    const int T = ctx->dm.T;
    int rc;
    // score the start row (EXPLICIT, one candidate) into the incumbent record
    qlm_candidates ex;
    memset(&ex, 0, sizeof ex);
    ex.kind = QLM_CAND_EXPLICIT;
    ex.token_bytes = token_bytes;
    ex.rows = row;
    ex.stride = (((int64_t)T * token_bytes) + 15) / 16 * 16;
    ex.count = 1;
    if ((rc = check_cand(ctx, &ex))) return rc;
    ScanParams p0 = base_params(ctx, &ex);
    p0.out_rec = incumbent;
    cudaError_t e = launch_any_scan(p0, st);
    if (e == cudaSuccess)             // index -1: the start row is the incumbent
        e = cudaMemsetAsync(&incumbent->index, 0xFF, sizeof(int64_t), st);
    if (e != cudaSuccess) return cuda_fail(e, "local search: start row");
    qlm_candidates nb = ex;
    nb.kind = QLM_CAND_NEIGHBOR;
    nb.stride = 0;
    nb.seed = seed;
    nb.moves = moves;
    nb.count = per_iter;
    // with a communicator, rank r scores its contiguous shard of every
    // iteration and the global winner is adopted everywhere
    int64_t sh_first = 0, sh_count = per_iter;
    if (ctx->comm) shard(per_iter, comm_rank(ctx->comm), comm_world(ctx->comm), sh_first, sh_count);
    for (int32_t it = 0; it < iters; ++it) {
        nb.first = (int64_t)it * per_iter + sh_first;
        nb.count = sh_count;
        if ((rc = check_cand(ctx, &nb))) return rc;
        if (sh_count > 0) {
            ScanParams p = base_params(ctx, &nb);
            p.out_rec = ctx->d_ls_rec;
            if ((e = launch_any_scan(p, st)) != cudaSuccess) return cuda_fail(e, "local search: scores");
        } else if ((e = cudaMemsetAsync(ctx->d_ls_rec, 0xFF, sizeof(qlm_record), st)) != cudaSuccess) {
            return cuda_fail(e, "local search: empty shard");
        }
        if ((rc = global_record(ctx, ctx->d_ls_rec, st))) return rc;
        if ((e = launch_adopt(ctx->dm, to_cand(&nb), ctx->d_ls_rec, incumbent, st)) != cudaSuccess)
            return cuda_fail(e, "local search: adopt");
    }
    return QLM_OK;
}

}  // namespace

extern "C" {

int qlm_abi_version(void) { return QLM_ABI_VERSION; }

const char *qlm_last_error(void) { return g_err.c_str(); }

int64_t qlm_kernel_launches(void) { return g_launches.load(); }

int qlm_set_kernel_overrides(uint32_t flags, int64_t ilv_cap) {
    if (flags & ~(uint32_t)QLM_OVERRIDE_ALL) return fail(QLM_EINVAL, "flags=0x%x has unknown bits", flags);
    if (ilv_cap < 0) return fail(QLM_EINVAL, "ilv_cap=%lld < 0", (long long)ilv_cap);
    g_override_flags.store(flags);
    g_override_ilv_cap.store(ilv_cap);
    return QLM_OK;
}

int qlm_dims(const qlm_ctx *ctx, int32_t *G, int32_t *Q, int32_t *T, int32_t *D, int32_t *M) {
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    if (G) *G = ctx->dm.G;
    if (Q) *Q = ctx->dm.Q;
    if (T) *T = ctx->dm.T;
    if (D) *D = ctx->dm.D;
    if (M) *M = ctx->dm.M;
    return QLM_OK;
}

int qlm_create(const qlm_group *groups, int32_t G, const qlm_queue *queues, int32_t Q,
               const qlm_profile *prof, const qlm_len_tables *tabs, const qlm_options *opt,
               qlm_ctx **out) {
    DevGuard dg_;
    NvtxRange nv_("qlm_create");
    if (!out) return fail(QLM_EINVAL, "out is NULL");
    *out = nullptr;
    if (!groups || G < 1) return fail(QLM_EINVAL, "G=%d must be >= 1 with non-NULL groups", G);
    if (!queues || Q < 1) return fail(QLM_EINVAL, "Q=%d must be >= 1 with non-NULL queues", Q);
    // T <= 32768: every scoring path keeps a candidate's row (4T bytes with its
    // swap targets) in one warp's shared memory (qlm_big.cu)
    if ((int64_t)G + Q - 1 > 32768) return fail(QLM_ERANGE, "T=G+Q-1=%lld > 32768", (long long)G + Q - 1);
    if (!prof) return fail(QLM_EINVAL, "prof is NULL");
    const int D = prof->D, M = prof->M;
    if (D < 1 || M < 1 || D > 64 || M > 64)
        return fail(QLM_EINVAL, "profile D=%d, M=%d must be in [1,64]", D, M);
    const double *arr[6] = {prof->theta, prof->prefill_s, prof->eps, prof->decode_s, prof->max_out,
                            prof->swap_s};
    const char *names[6] = {"theta", "prefill_s", "eps", "decode_s", "max_out", "swap_s"};
    for (int a = 0; a < 6; ++a)
        if (!arr[a]) return fail(QLM_EINVAL, "prof.%s is NULL", names[a]);
    for (int k = 0; k < D * M; ++k) {
        const int d = k / M, m = k % M;
        if (!(prof->theta[k] > 0.0) || !is_fin(prof->theta[k]))
            return fail(QLM_EINVAL, "prof.theta[%d][%d]=%g must be > 0 and finite", d, m, prof->theta[k]);
        if (!(prof->prefill_s[k] >= 0.0) || !is_fin(prof->prefill_s[k]))
            return fail(QLM_EINVAL, "prof.prefill_s[%d][%d]=%g must be >= 0", d, m, prof->prefill_s[k]);
        if (!(prof->eps[k] > 0.0) || !is_fin(prof->eps[k]))
            return fail(QLM_EINVAL, "prof.eps[%d][%d]=%g must be > 0", d, m, prof->eps[k]);
        if (!(prof->decode_s[k] >= 0.0) || !is_fin(prof->decode_s[k]))
            return fail(QLM_EINVAL, "prof.decode_s[%d][%d]=%g must be >= 0", d, m, prof->decode_s[k]);
        if (!(prof->max_out[k] >= 0.0) || !is_fin(prof->max_out[k]))
            return fail(QLM_EINVAL, "prof.max_out[%d][%d]=%g must be >= 0", d, m, prof->max_out[k]);
    }
    for (int k = 0; k < D * M * M; ++k) {
        const int d = k / (M * M), a = (k / M) % M, b = k % M;
        const double s = prof->swap_s[k];
        if (!(s >= 0.0) || !is_fin(s))
            return fail(QLM_EINVAL, "prof.swap_s[%d][%d][%d]=%g must be >= 0 and finite", d, a, b, s);
        if (a == b && s != 0.0)
            return fail(QLM_EINVAL, "prof.swap_s[%d][%d][%d]=%g: diagonal must be 0", d, a, b, s);
    }
    int n_tables = 0, K = 0;
    if (tabs) {
        K = tabs->K;
        n_tables = tabs->n_tables;
        if (K < 2 || K > 65536 || (K & (K - 1)))
            return fail(QLM_EINVAL, "tabs.K=%d must be a power of two in [2,65536]", K);
        if (n_tables < 1 || !tabs->len)
            return fail(QLM_EINVAL, "tabs.n_tables=%d must be >= 1 with non-NULL len", n_tables);
    }
    int rc = validate_groups(groups, G, M, n_tables);
    if (rc) return rc;
    for (int q = 0; q < Q; ++q) {
        const qlm_queue &u = queues[q];
        if (u.device < 0 || u.device >= D)
            return fail(QLM_EINVAL, "queues[%d].device=%d not in [0,D=%d)", q, u.device, D);
        if (u.resident_model < 0 || u.resident_model >= M)
            return fail(QLM_EINVAL, "queues[%d].resident_model=%d not in [0,M=%d)", q,
                        u.resident_model, M);
        if (!(u.backlog_mean_s >= 0.0) || !is_fin(u.backlog_mean_s))
            return fail(QLM_EINVAL, "queues[%d].backlog_mean_s=%g must be >= 0", q, u.backlog_mean_s);
        if (!(u.backlog_var_s2 >= 0.0) || !is_fin(u.backlog_var_s2))
            return fail(QLM_EINVAL, "queues[%d].backlog_var_s2=%g must be >= 0", q, u.backlog_var_s2);
    }
    double z_clamp = 8.0, alpha = 0.01;
    int device = 0;
    if (opt) {
        z_clamp = opt->z_clamp;
        alpha = opt->alpha;
        device = opt->device;
        if (!(z_clamp > 0.0) || !is_fin(z_clamp))
            return fail(QLM_EINVAL, "opt.z_clamp=%g must be > 0", z_clamp);
        if (!(alpha >= 0.0 && alpha < 1.0)) return fail(QLM_EINVAL, "opt.alpha=%g not in [0,1)", alpha);
        if (opt->reserved != 0) return fail(QLM_EINVAL, "opt.reserved must be 0");
    }
    // device: must be sm_100 (no CPU fallback, no other arch path)
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) return fail(QLM_ECUDA, "no CUDA device (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(QLM_EINVAL, "opt.device=%d not in [0,%d)", device, ndev);
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(QLM_ECUDA, "device %d is sm_%d%d; libqlm is built for sm_100a only", device,
                    prop.major, prop.minor);
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");

    qlm_ctx *ctx = new qlm_ctx();
    ctx->device = device;
    ctx->dm.G = G; ctx->dm.Q = Q; ctx->dm.D = D; ctx->dm.M = M; ctx->dm.T = G + Q - 1;
    ctx->dm.K = K; ctx->dm.n_tables = n_tables;
    int lg = 0;
    while ((1 << lg) < K) ++lg;
    ctx->dm.shift = 32 - lg;
    ctx->z_clamp = z_clamp;
    ctx->zc2 = z_clamp * z_clamp;
    ctx->alpha = (float)alpha;
    ctx->has_tables = tabs != nullptr;
    ctx->groups.assign(groups, groups + G);
    ctx->slo_hi_only = slo_hi_only(ctx->groups);
    ctx->queues.assign(queues, queues + Q);
    const size_t DM = (size_t)D * M;
    ctx->prof.resize(5 * DM + DM * M);
    for (int a = 0; a < 5; ++a) memcpy(&ctx->prof[a * DM], arr[a], DM * sizeof(double));
    memcpy(&ctx->prof[5 * DM], prof->swap_s, DM * M * sizeof(double));

    // raw region
    const size_t o_g = 0, o_q = a16(o_g + G * sizeof(qlm_group)),
                 o_p = a16(o_q + Q * sizeof(qlm_queue)),
                 raw_bytes = a16(o_p + ctx->prof.size() * sizeof(double));
    // table region
    const size_t t_grec = 0, t_ab = a16(t_grec + G * sizeof(GRec)),
                 t_q = a16(t_ab + (size_t)D * G * sizeof(double2)),
                 t_tail = a16(t_q + Q * sizeof(QRec)), t_swap = a16(t_tail + DM * 8),
                 t_theta = a16(t_swap + DM * M * 8), t_dist = a16(t_theta + DM * 8),
                 t_den = a16(t_dist + G * 4), t_len = a16(t_den + 8),
                 tab_bytes = a16(t_len + (size_t)n_tables * K * 2);
    ctx->max_blocks = sm_count() * 32;
    if (cudaMalloc(&ctx->d_raw, raw_bytes) != cudaSuccess ||
        cudaMalloc(&ctx->d_tab, tab_bytes) != cudaSuccess ||
        cudaMalloc(&ctx->d_block_recs, ctx->max_blocks * sizeof(qlm_record)) != cudaSuccess ||
        cudaMalloc(&ctx->d_counter, 64) != cudaSuccess ||
        cudaMalloc(&ctx->d_rec, 64) != cudaSuccess ||
        cudaMalloc(&ctx->d_ls_rec, 64) != cudaSuccess ||
        cudaMalloc(&ctx->d_dec_out, 2 * (size_t)G * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&ctx->d_bad, 64) != cudaSuccess) {
        qlm_destroy(ctx);
        return fail(QLM_ENOMEM, "device allocation failed");
    }
    uint8_t *raw = static_cast<uint8_t *>(ctx->d_raw);
    ctx->d_groups = reinterpret_cast<qlm_group *>(raw + o_g);
    ctx->d_queues = reinterpret_cast<qlm_queue *>(raw + o_q);
    double *pp = reinterpret_cast<double *>(raw + o_p);
    ctx->d_theta = pp; ctx->d_prefill = pp + DM; ctx->d_eps = pp + 2 * DM; ctx->d_dec = pp + 3 * DM;
    ctx->d_maxo = pp + 4 * DM; ctx->d_swap = pp + 5 * DM;
    uint8_t *tab = static_cast<uint8_t *>(ctx->d_tab);
    ctx->tb.grec = reinterpret_cast<GRec *>(tab + t_grec);
    ctx->tb.ab = reinterpret_cast<double2 *>(tab + t_ab);
    ctx->tb.qrec = reinterpret_cast<QRec *>(tab + t_q);
    ctx->tb.tail = reinterpret_cast<double *>(tab + t_tail);
    ctx->tb.swap = reinterpret_cast<double *>(tab + t_swap);
    ctx->tb.theta = reinterpret_cast<double *>(tab + t_theta);
    ctx->tb.dist = reinterpret_cast<int32_t *>(tab + t_dist);
    ctx->tb.den = reinterpret_cast<double *>(tab + t_den);
    ctx->tb.len = reinterpret_cast<uint16_t *>(tab + t_len);

    if ((e = cudaMemcpy(ctx->d_groups, groups, G * sizeof(qlm_group), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(ctx->d_queues, queues, Q * sizeof(qlm_queue), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(pp, ctx->prof.data(), ctx->prof.size() * sizeof(double), cudaMemcpyHostToDevice)) ||
        (e = cudaMemset(ctx->d_counter, 0, 64))) {
        qlm_destroy(ctx);
        return cuda_fail(e, "upload");
    }
    if (tabs && (e = cudaMemcpy(ctx->tb.len, tabs->len, (size_t)n_tables * K * 2, cudaMemcpyHostToDevice))) {
        qlm_destroy(ctx);
        return cuda_fail(e, "upload length tables");
    }
    rc = rebuild(ctx, nullptr);
    if (!rc && (e = cudaDeviceSynchronize()) != cudaSuccess) rc = cuda_fail(e, "build_tables");
    if (rc) {
        qlm_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return QLM_OK;
}

void qlm_destroy(qlm_ctx *ctx) {
    DevGuard dg_;
    NvtxRange nv_("qlm_destroy");
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->comm) qlm_comm_detach(ctx);
    void *ptrs[] = {ctx->d_raw, ctx->d_tab, ctx->d_block_recs, ctx->d_counter, ctx->d_rec,
                    ctx->d_dec_out, ctx->d_bad, ctx->d_X, ctx->d_ilv, ctx->d_chunk_recs,
                    ctx->d_ls_rec, ctx->d_tier};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    if (ctx->ls_exec) cudaGraphExecDestroy(ctx->ls_exec);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    if (ctx->ev_stage) cudaEventDestroy(ctx->ev_stage);
    delete ctx;
}

int qlm_update_groups(qlm_ctx *ctx, const qlm_group *groups, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_update_groups");
    if (!ctx || !groups) return fail(QLM_EINVAL, "ctx or groups is NULL");
    int rc = validate_groups(groups, ctx->dm.G, ctx->dm.M, ctx->dm.n_tables);
    if (rc || (rc = check_dev(ctx))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t bytes = ctx->dm.G * sizeof(qlm_group);
    cudaError_t e;
    if (!ctx->h_stage) {
        if ((e = cudaMallocHost(&ctx->h_stage, bytes)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&ctx->ev_stage, cudaEventDisableTiming)) != cudaSuccess) {
            ctx->h_stage = nullptr;
            return cuda_fail(e, "update_groups staging");
        }
    } else if ((e = cudaEventSynchronize(ctx->ev_stage)) != cudaSuccess) {   // previous copy has read it
        return cuda_fail(e, "update_groups staging");
    }
    // deep copy: the device reads the validated snapshot, never the caller's buffer
    memcpy(ctx->h_stage, groups, bytes);
    if ((e = cudaMemcpyAsync(ctx->d_groups, ctx->h_stage, bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaEventRecord(ctx->ev_stage, st)) != cudaSuccess)
        return cuda_fail(e, "update_groups copy");
    ctx->groups.assign(groups, groups + ctx->dm.G);
    ctx->slo_hi_only = slo_hi_only(ctx->groups);
    return rebuild(ctx, st);
}

int qlm_score_orderings(qlm_ctx *ctx, const qlm_candidates *cand, float *s1, float *s2,
                        int32_t *n_over, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_score_orderings");
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    if (cand->count > 0 && (!s1 || !s2)) return fail(QLM_EINVAL, "s1/s2 outputs are NULL");
    if (cand->count == 0) return QLM_OK;
    ScanParams p = base_params(ctx, cand);
    p.s1 = s1; p.s2 = s2; p.n_over = n_over;
    attach_ilv(ctx, p);
    cudaError_t e = launch_any_scan(p, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "score kernel");
}

int qlm_best_ordering_async(qlm_ctx *ctx, const qlm_candidates *cand, qlm_record *rec,
                            void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_best_ordering_async");
    if (!ctx || !rec) return fail(QLM_EINVAL, "ctx or rec is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cand->count == 0) {                                  // the "none" record
        cudaError_t e = cudaMemsetAsync(rec, 0xFF, sizeof(qlm_record), st);
        if (e != cudaSuccess) return cuda_fail(e, "empty record");
        return global_record(ctx, rec, st);
    }
    ScanParams p = base_params(ctx, cand);
    p.out_rec = rec;
    attach_ilv(ctx, p);
    cudaError_t e = launch_any_scan(p, st);
    if (e != cudaSuccess) return cuda_fail(e, "score/argmin kernel");
    return global_record(ctx, rec, st);
}

int qlm_reduce_records(qlm_ctx *ctx, const qlm_record *recs, int32_t n, qlm_record *out,
                       void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_reduce_records");
    if (!ctx || !recs || !out || n < 1) return fail(QLM_EINVAL, "reduce_records: bad arguments");
    int rc = check_dev(ctx);
    if (rc) return rc;
    cudaError_t e = launch_reduce_records(recs, n, out, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "reduce_records");
}

int qlm_decode(qlm_ctx *ctx, const qlm_candidates *cand, int32_t *queue_of_group,
               int32_t *pos_of_group, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_decode");
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    if (cand->count == 0) return QLM_OK;
    ScanParams p = base_params(ctx, cand);
    cudaError_t e = launch_rows(p, nullptr, queue_of_group, pos_of_group,
                                static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "decode kernel");
}

// The device address of a pinned host buffer (page-locked and mapped, as
// cudaHostAlloc / cudaHostRegister memory is under unified addressing), or
// nullptr for pageable memory.
static void *mapped_host(void *h) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

int qlm_winner(qlm_ctx *ctx, const qlm_candidates *one, qlm_best *out, int32_t *queue_of_group,
               int32_t *pos_of_group, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_winner");
    if (!ctx || !one || !out) return fail(QLM_EINVAL, "ctx, one or out is NULL");
    if (one->count != 1 || !one->first_from)
        return fail(QLM_EINVAL, "qlm_winner needs cand.count == 1 and cand.first_from = the device record");
    int rc = check_cand(ctx, one);
    if (rc || (rc = check_dev(ctx))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int G = ctx->dm.G;
    // the record's candidate scored and decoded on the device (no host sync),
    // then one D2H copy per result field into the caller's host buffers
    float *d_s = reinterpret_cast<float *>(ctx->d_rec + 1);
    int32_t *d_no = reinterpret_cast<int32_t *>(ctx->d_rec + 2);
    if ((rc = qlm_score_orderings(ctx, one, d_s, d_s + 1, d_no, stream))) return rc;
    if ((rc = qlm_decode(ctx, one, ctx->d_dec_out, ctx->d_dec_out + G, stream))) return rc;
    cudaError_t e;
    // pinned (device-mapped) host buffers: the device writes the result fields
    // straight into them with one small kernel; otherwise one copy per field
    void *m_out = mapped_host(out), *m_qo = queue_of_group ? mapped_host(queue_of_group) : nullptr,
         *m_po = pos_of_group ? mapped_host(pos_of_group) : nullptr;
    if (m_out && (m_qo || !queue_of_group) && (m_po || !pos_of_group)) {
        e = launch_winner_out(one->first_from, d_s, d_no, ctx->d_dec_out, G, static_cast<qlm_best *>(m_out),
                              static_cast<int32_t *>(m_qo), static_cast<int32_t *>(m_po), st);
        return e == cudaSuccess ? QLM_OK : cuda_fail(e, "winner readback");
    }
    if ((e = cudaMemcpyAsync(&out->index, &one->first_from->index, sizeof(int64_t), cudaMemcpyDeviceToHost, st)) ||
        (e = cudaMemcpyAsync(&out->s1, d_s, 2 * sizeof(float), cudaMemcpyDeviceToHost, st)) ||
        (e = cudaMemcpyAsync(&out->n_over, d_no, sizeof(int32_t), cudaMemcpyDeviceToHost, st)) ||
        (queue_of_group && (e = cudaMemcpyAsync(queue_of_group, ctx->d_dec_out, G * sizeof(int32_t),
                                                cudaMemcpyDeviceToHost, st))) ||
        (pos_of_group && (e = cudaMemcpyAsync(pos_of_group, ctx->d_dec_out + G, G * sizeof(int32_t),
                                              cudaMemcpyDeviceToHost, st))))
        return cuda_fail(e, "winner readback");
    return QLM_OK;
}

int qlm_rows(qlm_ctx *ctx, const qlm_candidates *cand, uint16_t *rows_out, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_rows");
    if (!ctx || !rows_out) return fail(QLM_EINVAL, "ctx or rows_out is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    if (cand->count == 0) return QLM_OK;
    ScanParams p = base_params(ctx, cand);
    cudaError_t e = launch_rows(p, rows_out, nullptr, nullptr, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "rows kernel");
}

int qlm_best_ordering(qlm_ctx *ctx, const qlm_candidates *cand, qlm_best *out,
                      int32_t *queue_of_group, int32_t *pos_of_group, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_best_ordering");
    if (!ctx || !out) return fail(QLM_EINVAL, "ctx or out is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    memset(out, 0, sizeof *out);
    out->index = -1;
    if (cand->count == 0 && !ctx->comm) return QLM_OK;
    if ((rc = qlm_best_ordering_async(ctx, cand, ctx->d_rec, stream))) return rc;   // global when attached
    qlm_record h;
    cudaError_t e = cudaMemcpyAsync(&h, ctx->d_rec, sizeof h, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "best_ordering");
    out->index = h.index;
    if (h.index < 0) return QLM_OK;
    // re-score and decode the winner on the device -- on the rank whose range
    // holds it (EXPLICIT rows live there), shared by a max all-reduce
    const int G = ctx->dm.G;
    const bool owner = h.index >= cand->first && h.index < cand->first + cand->count;
    int32_t sc[5] = {-1, -1, -1, -1, -1};                   // s1 hi/lo, s2 hi/lo (16-bit halves), n_over
    if (owner) {
        qlm_candidates one = *cand;
        one.first = h.index;
        one.count = 1;
        one.first_from = nullptr;
        if (cand->kind == QLM_CAND_EXPLICIT)
            one.rows = static_cast<const uint8_t *>(cand->rows) + (h.index - cand->first) * cand->stride;
        float *d_s = reinterpret_cast<float *>(ctx->d_rec + 1);
        int32_t *d_no = reinterpret_cast<int32_t *>(ctx->d_rec + 2);
        if ((rc = qlm_score_orderings(ctx, &one, d_s, d_s + 1, d_no, stream))) return rc;
        if ((rc = qlm_decode(ctx, &one, ctx->d_dec_out, ctx->d_dec_out + G, stream))) return rc;
        float sv[2];
        int32_t no = 0;
        if ((e = cudaMemcpyAsync(sv, d_s, sizeof sv, cudaMemcpyDeviceToHost, st)) ||
            (e = cudaMemcpyAsync(&no, d_no, sizeof no, cudaMemcpyDeviceToHost, st)) ||
            (e = cudaStreamSynchronize(st)))
            return cuda_fail(e, "best_ordering scores");
        uint32_t b1, b2;
        memcpy(&b1, &sv[0], 4);
        memcpy(&b2, &sv[1], 4);
        sc[0] = (int32_t)(b1 >> 16); sc[1] = (int32_t)(b1 & 0xFFFFu);
        sc[2] = (int32_t)(b2 >> 16); sc[3] = (int32_t)(b2 & 0xFFFFu);
        sc[4] = no;
    }
    const int32_t *dec = ctx->d_dec_out;
    if (ctx->comm) {
        int32_t *buf = ctx->d_comm_buf;                     // non-owners contribute -1 everywhere
        std::string err;
        if ((e = owner ? cudaMemcpyAsync(buf, ctx->d_dec_out, 2 * (size_t)G * 4, cudaMemcpyDeviceToDevice, st)
                       : cudaMemsetAsync(buf, 0xFF, 2 * (size_t)G * 4, st)) ||
            (e = cudaMemcpyAsync(buf + 2 * G, sc, sizeof sc, cudaMemcpyHostToDevice, st)))
            return cuda_fail(e, "best_ordering share");
        if (!comm_allreduce_max_i32(ctx->comm, buf, 2 * (size_t)G + 5, st, err))
            return fail(QLM_ENCCL, "%s", err.c_str());
        if ((e = cudaMemcpyAsync(sc, buf + 2 * G, sizeof sc, cudaMemcpyDeviceToHost, st))) return cuda_fail(e, "share");
        dec = buf;
    }
    if ((queue_of_group && (e = cudaMemcpyAsync(queue_of_group, dec, G * sizeof(int32_t),
                                                cudaMemcpyDeviceToHost, st))) ||
        (pos_of_group && (e = cudaMemcpyAsync(pos_of_group, dec + G, G * sizeof(int32_t),
                                              cudaMemcpyDeviceToHost, st))) ||
        (e = cudaStreamSynchronize(st)))
        return cuda_fail(e, "best_ordering readback");
    const uint32_t b1 = ((uint32_t)sc[0] << 16) | (uint32_t)sc[1], b2 = ((uint32_t)sc[2] << 16) | (uint32_t)sc[3];
    memcpy(&out->s1, &b1, 4);
    memcpy(&out->s2, &b2, 4);
    out->n_over = sc[4];
    return QLM_OK;
}

int qlm_rwt_estimate(qlm_ctx *ctx, const qlm_candidates *cand, float *wt_mean, float *wt_std,
                     float *viol, void *stream) {
    return qlm_score_estimate(ctx, cand, wt_mean, wt_std, viol, nullptr, nullptr, nullptr, nullptr,
                              stream);
}

int qlm_score_estimate(qlm_ctx *ctx, const qlm_candidates *cand, float *wt_mean, float *wt_std,
                       float *viol, float *s1, float *s2, int32_t *n_over, qlm_record *rec,
                       void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_score_estimate");
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cand->count == 0) {
        if (!rec) return QLM_OK;
        cudaError_t e = cudaMemsetAsync(rec, 0xFF, sizeof(qlm_record), st);   // the "none" record
        if (e != cudaSuccess) return cuda_fail(e, "empty record");
        return global_record(ctx, rec, st);
    }
    if (!wt_mean && !wt_std && !viol && !s1 && !s2 && !n_over && !rec) return QLM_OK;
    ScanParams p = base_params(ctx, cand);
    p.wt = wt_mean; p.sd = wt_std; p.vo = viol;
    p.s1 = s1; p.s2 = s2; p.n_over = n_over; p.out_rec = rec;
    attach_ilv(ctx, p);
    cudaError_t e = launch_any_scan(p, st);
    if (e != cudaSuccess) return cuda_fail(e, "scan kernel");
    return rec ? global_record(ctx, rec, st) : QLM_OK;
}

int qlm_mc_sample(qlm_ctx *ctx, uint64_t mc_seed, int64_t trial_first, int64_t trial_count,
                  void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_mc_sample");
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    int rc = check_dev(ctx);
    if (rc) return rc;
    if (!ctx->has_tables) return fail(QLM_EINVAL, "MC mode needs length tables at qlm_create");
    for (int i = 0; i < ctx->dm.G; ++i)
        if (ctx->groups[i].dist_id < 0)
            return fail(QLM_EINVAL, "groups[%d].dist_id=-1: MC mode needs a length table", i);
    if (trial_first < 0 || trial_count < 0 || trial_first + trial_count > (int64_t)1 << 32)
        return fail(QLM_ERANGE, "trials [%lld, +%lld) must lie in [0, 2^32)", (long long)trial_first,
                    (long long)trial_count);
    if ((uint64_t)trial_count * (uint64_t)ctx->dm.G >= ((uint64_t)1 << 32))
        return fail(QLM_ERANGE, "trial_count * G = %lld must be < 2^32", (long long)(trial_count * ctx->dm.G));
    ctx->mc_trials = trial_count;
    if (trial_count == 0) return QLM_OK;
    const size_t needX = (size_t)trial_count * ctx->dm.G * ctx->dm.D * sizeof(double);
    if (needX > ctx->X_cap) {
        if (ctx->d_X) cudaFree(ctx->d_X);
        ctx->d_X = nullptr;
        ctx->X_cap = 0;
        if (cudaMalloc(&ctx->d_X, needX) != cudaSuccess) return fail(QLM_ENOMEM, "MC scratch %zu B", needX);
        ctx->X_cap = needX;
    }
    cudaError_t e = launch_mc_sample(ctx->dm, ctx->tb, mc_seed, trial_first, trial_count, ctx->d_X,
                                     static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "MC sample kernel");
}

int qlm_mc_count(qlm_ctx *ctx, const qlm_candidates *cand, int64_t trial_count, uint32_t *counts,
                 void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_mc_count");
    if (!ctx || !counts) return fail(QLM_EINVAL, "ctx or counts is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    if (trial_count != ctx->mc_trials)
        return fail(QLM_EINVAL, "trial_count=%lld differs from the last qlm_mc_sample (%lld)",
                    (long long)trial_count, (long long)ctx->mc_trials);
    if (cand->count > 65535) return fail(QLM_ERANGE, "MC: cand.count=%lld > 65535", (long long)cand->count);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cand->count == 0) return QLM_OK;
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)cand->count * ctx->dm.G * 4, st);
    if (e != cudaSuccess) return cuda_fail(e, "counts memset");
    if (trial_count == 0) return global_counts(ctx, counts, (size_t)cand->count * ctx->dm.G, st);
    if ((e = launch_mc_count(ctx->dm, ctx->tb, to_cand(cand), ctx->d_X, trial_count, counts, st)) !=
        cudaSuccess)
        return cuda_fail(e, "MC count kernel");
    return global_counts(ctx, counts, (size_t)cand->count * ctx->dm.G, st);
}

int qlm_mc_estimate(qlm_ctx *ctx, const qlm_candidates *cand, uint64_t mc_seed,
                    int64_t trial_first, int64_t trial_count, uint32_t *counts, void *stream) {
    if (!ctx || !counts) return fail(QLM_EINVAL, "ctx or counts is NULL");
    int rc = check_cand(ctx, cand);
    if (rc) return rc;
    if ((rc = qlm_mc_sample(ctx, mc_seed, trial_first, trial_count, stream))) return rc;
    return qlm_mc_count(ctx, cand, trial_count, counts, stream);
}

int qlm_check_rows(qlm_ctx *ctx, const qlm_candidates *cand, int64_t *n_bad, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_check_rows");
    if (!ctx || !n_bad) return fail(QLM_EINVAL, "ctx or n_bad is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    if (cand->kind != QLM_CAND_EXPLICIT) { *n_bad = 0; return QLM_OK; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(ctx->d_bad, 0, 8, st);
    if (e == cudaSuccess) e = launch_check_rows(to_cand(cand), ctx->dm.T, ctx->d_bad, st);
    unsigned long long h = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, ctx->d_bad, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "check_rows");
    *n_bad = (int64_t)h;
    return QLM_OK;
}

int qlm_adopt_best(qlm_ctx *ctx, const qlm_candidates *cand, const qlm_record *rec,
                   qlm_record *incumbent, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_adopt_best");
    if (!ctx || !rec || !incumbent) return fail(QLM_EINVAL, "ctx, rec or incumbent is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    if (cand->kind != QLM_CAND_NEIGHBOR) return fail(QLM_EINVAL, "qlm_adopt_best needs NEIGHBOR candidates");
    cudaError_t e = launch_adopt(ctx->dm, to_cand(cand), rec, incumbent, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "adopt kernel");
}

int qlm_local_search(qlm_ctx *ctx, void *row, int32_t token_bytes, int32_t moves, int64_t per_iter,
                     int32_t iters, uint64_t seed, qlm_record *incumbent, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_local_search");
    if (!ctx || !row || !incumbent) return fail(QLM_EINVAL, "ctx, row or incumbent is NULL");
    if (moves < 1 || moves > QLM_MAX_MOVES)
        return fail(QLM_EINVAL, "moves=%d must lie in [1, %d]", moves, QLM_MAX_MOVES);
    if (per_iter < 1) return fail(QLM_EINVAL, "per_iter=%lld < 1", (long long)per_iter);
    if (iters < 0) return fail(QLM_EINVAL, "iters=%d < 0", iters);
    if (iters > 0 && per_iter > INT64_MAX / iters) return fail(QLM_ERANGE, "iters * per_iter overflows");
    int rc = check_dev(ctx);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the search is 2 * iters + 2 short launches: they are captured once into
    // a CUDA graph (updated in place on later calls of the same shape) and
    // launched as one unit, so the launches do not pace it.  The legacy
    // default stream cannot capture: a blocking context stream stands in for
    // it (ordered with the legacy stream both ways)
    if (!st && iters >= 2 && !override_on(QLM_OVERRIDE_NO_GRAPH) && !ctx->aux &&
        cudaStreamCreateWithFlags(&ctx->aux, cudaStreamDefault) != cudaSuccess) {
        cudaGetLastError();
        ctx->aux = nullptr;
    }
    cudaStream_t cst = st ? st : ctx->aux;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cst && cudaStreamIsCapturing(cst, &cs) != cudaSuccess) {
        cudaGetLastError();
        cs = cudaStreamCaptureStatusActive;                   // unknown: do not nest
    }
    const bool graph = cst && iters >= 2 && cs == cudaStreamCaptureStatusNone &&
                       !override_on(QLM_OVERRIDE_NO_GRAPH);
    if (!graph) return enqueue_search(ctx, row, token_bytes, moves, per_iter, iters, seed, incumbent, st);
    // the same call again (same row buffer, record, shape, seed and stream):
    // replay the instantiated graph without capturing
    const std::vector<int64_t> sig = {(int64_t)(uintptr_t)row, token_bytes, moves, per_iter, iters,
                                      (int64_t)seed, (int64_t)(uintptr_t)incumbent, (int64_t)(uintptr_t)cst,
                                      (int64_t)ctx->dm.G, (int64_t)(uintptr_t)ctx->comm};
    cudaError_t e;
    if (ctx->ls_exec && sig == ctx->ls_sig) {
        e = cudaGraphLaunch(ctx->ls_exec, cst);
        return e == cudaSuccess ? QLM_OK : cuda_fail(e, "local search: graph launch");
    }
    e = cudaStreamBeginCapture(cst, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_fail(e, "local search: begin capture");
    rc = enqueue_search(ctx, row, token_bytes, moves, per_iter, iters, seed, incumbent, cst);
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(cst, &g);
    if (rc || e != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        return rc ? rc : cuda_fail(e, "local search: end capture");
    }
    if (ctx->ls_exec) {
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(ctx->ls_exec, g, &info) != cudaSuccess) {   // another shape: rebuild
            cudaGetLastError();
            cudaGraphExecDestroy(ctx->ls_exec);
            ctx->ls_exec = nullptr;
        }
    }
    if (!ctx->ls_exec && (e = cudaGraphInstantiate(&ctx->ls_exec, g, 0)) != cudaSuccess) {
        ctx->ls_exec = nullptr;
        cudaGraphDestroy(g);
        return cuda_fail(e, "local search: instantiate");
    }
    cudaGraphDestroy(g);
    ctx->ls_sig = sig;
    qlog(1, "local search: CUDA graph of %d iterations x %lld candidates", iters, (long long)per_iter);
    e = cudaGraphLaunch(ctx->ls_exec, cst);
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "local search: graph launch");
}

int qlm_request_violations(qlm_ctx *ctx, const qlm_candidates *cand, float *frac, float *s1_req,
                           void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_request_violations");
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    if (cand->count == 0 || (!frac && !s1_req)) return QLM_OK;
    ScanParams p = base_params(ctx, cand);
    cudaError_t e = launch_req(p, ctx->d_groups, frac, s1_req, static_cast<cudaStream_t>(stream));
    if (e == cudaErrorInvalidConfiguration) {
        cudaGetLastError();
        return fail(QLM_ERANGE, "request violations keep 20 B per group and 4 B per token of one "
                    "candidate in shared memory: G=%d is too large (about 11000 at most)", ctx->dm.G);
    }
    return e == cudaSuccess ? QLM_OK : cuda_fail(e, "request-violations kernel");
}

int qlm_set_tiers(qlm_ctx *ctx, const qlm_tiers *tiers) {
    DevGuard dg_;
    NvtxRange nv_("qlm_set_tiers");
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    int rc = check_dev(ctx);
    if (rc) return rc;
    if (!tiers) {
        ctx->has_tiers = false;
        return QLM_OK;
    }
    const int D = ctx->dm.D, M = ctx->dm.M;
    if (M > 32) return fail(QLM_EINVAL, "two-tier swapping needs M=%d <= 32", M);
    if (!tiers->model_mem || !tiers->cpu_cap || !tiers->load_s)
        return fail(QLM_EINVAL, "tiers.model_mem / cpu_cap / load_s must be non-NULL");
    int64_t total = 0;
    for (int m = 0; m < M; ++m) {
        if (tiers->model_mem[m] < 1)
            return fail(QLM_EINVAL, "tiers.model_mem[%d]=%d must be >= 1", m, tiers->model_mem[m]);
        total += tiers->model_mem[m];
    }
    if (total > (1 << 24)) return fail(QLM_ERANGE, "sum of tiers.model_mem=%lld > 2^24", (long long)total);
    for (int d = 0; d < D; ++d)
        if (tiers->cpu_cap[d] < 0)
            return fail(QLM_EINVAL, "tiers.cpu_cap[%d]=%d must be >= 0", d, tiers->cpu_cap[d]);
    for (int k = 0; k < D * M; ++k)
        if (!(tiers->load_s[k] >= 0.0) || !is_fin(tiers->load_s[k]))
            return fail(QLM_EINVAL, "tiers.load_s[%d][%d]=%g must be >= 0 and finite", k / M, k % M,
                        tiers->load_s[k]);
    const size_t o_cap = a16((size_t)M * 4), o_load = a16(o_cap + (size_t)D * 4);
    const size_t bytes = o_load + (size_t)D * M * 8;
    if (!ctx->d_tier) {
        cudaError_t e = cudaMalloc(&ctx->d_tier, bytes);
        if (e != cudaSuccess) {
            ctx->d_tier = nullptr;
            return fail(QLM_ENOMEM, "tier tables: %s", cudaGetErrorString(e));
        }
    }
    std::vector<uint8_t> h(bytes, 0);
    memcpy(h.data(), tiers->model_mem, (size_t)M * 4);
    memcpy(h.data() + o_cap, tiers->cpu_cap, (size_t)D * 4);
    memcpy(h.data() + o_load, tiers->load_s, (size_t)D * M * 8);
    // tiered kernels may still read the old tables on any stream: drain the
    // device before overwriting them (this call is synchronous by contract)
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "set_tiers: device sync");
    e = cudaMemcpy(ctx->d_tier, h.data(), bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "upload tier tables");
    ctx->has_tiers = true;
    return QLM_OK;
}

int qlm_tiered_score_estimate(qlm_ctx *ctx, const qlm_candidates *cand, float *wt_mean,
                              float *wt_std, float *viol, float *s1, float *s2, int32_t *n_over,
                              qlm_record *rec, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_tiered_score_estimate");
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    if (!ctx->has_tiers) return fail(QLM_EINVAL, "no tier tables: call qlm_set_tiers first");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cand->count == 0) {
        if (!rec) return QLM_OK;
        cudaError_t e = cudaMemsetAsync(rec, 0xFF, sizeof(qlm_record), st);   // the "none" record
        if (e != cudaSuccess) return cuda_fail(e, "empty record");
        return global_record(ctx, rec, st);
    }
    if (!wt_mean && !wt_std && !viol && !s1 && !s2 && !n_over && !rec) return QLM_OK;
    ScanParams p = base_params(ctx, cand);
    p.wt = wt_mean; p.sd = wt_std; p.vo = viol;
    p.s1 = s1; p.s2 = s2; p.n_over = n_over; p.out_rec = rec;
    const int M = ctx->dm.M, D = ctx->dm.D;
    const size_t o_cap = a16((size_t)M * 4), o_load = a16(o_cap + (size_t)D * 4);
    uint8_t *t = static_cast<uint8_t *>(ctx->d_tier);
    p.t_mem = reinterpret_cast<const int32_t *>(t);
    p.t_cap = reinterpret_cast<const int32_t *>(t + o_cap);
    p.t_load = reinterpret_cast<const double *>(t + o_load);
    attach_ilv(ctx, p);                                  // large-T RANDOM: two-phase row chunks
    cudaError_t e = launch_tier(p, st);
    if (e != cudaSuccess) return cuda_fail(e, "tier kernel");
    return rec ? global_record(ctx, rec, st) : QLM_OK;
}

int qlm_form_groups(const qlm_requests *req, int32_t M, const int32_t *k_per_model, int32_t limit,
                    int32_t max_iter, int32_t *label_of, int32_t *group_of, qlm_group *groups,
                    int32_t group_cap, int32_t *n_groups, int32_t *iters, int32_t device, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_form_groups");
    if (!req || !k_per_model || !n_groups)
        return fail(QLM_EINVAL, "req, k_per_model and n_groups must be non-NULL");
    if (req->n < 1 || req->n >= (1 << 28)) return fail(QLM_EINVAL, "req.n=%d not in [1, 2^28)", req->n);
    if (req->dims < 1 || req->dims > 4) return fail(QLM_EINVAL, "req.dims=%d not in [1, 4]", req->dims);
    if (!req->model || !req->slo_s || !req->out_tokens || !req->feat)
        return fail(QLM_EINVAL, "req.model / slo_s / out_tokens / feat must be non-NULL");
    if (M < 1 || M > 64) return fail(QLM_EINVAL, "M=%d not in [1, 64]", M);
    int K = 0;
    for (int m = 0; m < M; ++m) {
        if (k_per_model[m] < 1 || k_per_model[m] > 1024)
            return fail(QLM_EINVAL, "k_per_model[%d]=%d not in [1, 1024]", m, k_per_model[m]);
        K += k_per_model[m];
    }
    if (K > 1024) return fail(QLM_EINVAL, "sum of k_per_model=%d > 1024", K);
    if (limit < 1 || limit > 32768) return fail(QLM_EINVAL, "limit=%d not in [1, 32768]", limit);
    if (max_iter < 1 || max_iter > 1000) return fail(QLM_EINVAL, "max_iter=%d not in [1, 1000]", max_iter);
    if (!label_of || !group_of) return fail(QLM_EINVAL, "label_of and group_of must be non-NULL");
    if (group_cap < 0 || (group_cap > 0 && !groups)) return fail(QLM_EINVAL, "groups is NULL with group_cap > 0");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    int32_t bad = 0, it = 0, G = 0;
    e = launch_form_groups(req->n, req->dims, M, k_per_model, limit, max_iter, req->model, req->slo_s,
                           req->out_tokens, req->feat, label_of, group_of, groups, group_cap, &G, &it,
                           &bad, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "group formation");
    if (bad) return fail(QLM_EINVAL, "req: %d requests with a model, SLO, output length or feature out of range", bad);
    *n_groups = G;
    if (iters) *iters = it;
    if (G > group_cap) return fail(QLM_ERANGE, "%d groups > group_cap=%d (n_groups is set)", G, group_cap);
    return QLM_OK;
}

int qlm_tiered_mc_count(qlm_ctx *ctx, const qlm_candidates *cand, int64_t trial_count,
                        uint32_t *counts, void *stream) {
    DevGuard dg_;
    NvtxRange nv_("qlm_tiered_mc_count");
    if (!ctx || !counts) return fail(QLM_EINVAL, "ctx or counts is NULL");
    if (!ctx->has_tiers) return fail(QLM_EINVAL, "no tier tables: call qlm_set_tiers first");
    int rc = check_cand(ctx, cand);
    if (rc || (rc = check_dev(ctx))) return rc;
    if (trial_count != ctx->mc_trials)
        return fail(QLM_EINVAL, "trial_count=%lld differs from the last qlm_mc_sample (%lld)",
                    (long long)trial_count, (long long)ctx->mc_trials);
    if (cand->count > 65535) return fail(QLM_ERANGE, "MC: cand.count=%lld > 65535", (long long)cand->count);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cand->count == 0) return QLM_OK;
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)cand->count * ctx->dm.G * 4, st);
    if (e != cudaSuccess) return cuda_fail(e, "counts memset");
    if (trial_count == 0) return global_counts(ctx, counts, (size_t)cand->count * ctx->dm.G, st);
    const int M = ctx->dm.M, D = ctx->dm.D;
    const size_t o_cap = a16((size_t)M * 4), o_load = a16(o_cap + (size_t)D * 4);
    uint8_t *t = static_cast<uint8_t *>(ctx->d_tier);
    if ((e = launch_mc_count(ctx->dm, ctx->tb, to_cand(cand), ctx->d_X, trial_count, counts, st,
                             reinterpret_cast<const int32_t *>(t), reinterpret_cast<const int32_t *>(t + o_cap),
                             reinterpret_cast<const double *>(t + o_load))) != cudaSuccess)
        return cuda_fail(e, "MC count kernel");
    return global_counts(ctx, counts, (size_t)cand->count * ctx->dm.G, st);
}

int qlm_comm_unique_id(uint8_t id[QLM_COMM_ID_BYTES]) {
    if (!id) return fail(QLM_EINVAL, "id is NULL");
    std::string err;
    if (!comm_unique_id(id, err)) return fail(QLM_ENCCL, "%s", err.c_str());
    return QLM_OK;
}

int qlm_comm_attach(qlm_ctx *ctx, const uint8_t id[QLM_COMM_ID_BYTES], int32_t rank, int32_t world) {
    DevGuard dg_;
    NvtxRange nv_("qlm_comm_attach");
    if (!ctx || !id) return fail(QLM_EINVAL, "ctx or id is NULL");
    if (world < 1 || rank < 0 || rank >= world)
        return fail(QLM_EINVAL, "rank=%d, world=%d: need 0 <= rank < world", rank, world);
    if (ctx->comm) return fail(QLM_EINVAL, "a communicator is already attached");
    int rc = check_dev(ctx);
    if (rc) return rc;
    if (cudaMalloc(&ctx->d_comm_recs, (size_t)world * sizeof(qlm_record)) != cudaSuccess ||
        cudaMalloc(&ctx->d_comm_buf, (2 * (size_t)ctx->dm.G + 5) * sizeof(int32_t)) != cudaSuccess) {
        cudaFree(ctx->d_comm_recs);
        ctx->d_comm_recs = nullptr;
        return fail(QLM_ENOMEM, "communicator scratch");
    }
    std::string err;
    ctx->comm = comm_init(id, rank, world, err);
    if (!ctx->comm) {
        cudaFree(ctx->d_comm_recs);
        cudaFree(ctx->d_comm_buf);
        ctx->d_comm_recs = nullptr;
        ctx->d_comm_buf = nullptr;
        return fail(QLM_ENCCL, "%s", err.c_str());
    }
    return QLM_OK;
}

int qlm_comm_detach(qlm_ctx *ctx) {
    DevGuard dg_;
    NvtxRange nv_("qlm_comm_detach");
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    if (!ctx->comm) return QLM_OK;
    int rc = check_dev(ctx);
    if (rc) return rc;
    cudaDeviceSynchronize();
    if (ctx->ls_exec) {                       // a captured search may hold the communicator's calls
        cudaGraphExecDestroy(ctx->ls_exec);
        ctx->ls_exec = nullptr;
        ctx->ls_sig.clear();
    }
    comm_destroy(ctx->comm);
    ctx->comm = nullptr;
    cudaFree(ctx->d_comm_recs);
    cudaFree(ctx->d_comm_buf);
    ctx->d_comm_recs = nullptr;
    ctx->d_comm_buf = nullptr;
    return QLM_OK;
}

int qlm_comm_info(const qlm_ctx *ctx, int32_t *rank, int32_t *world, int32_t *nccl_version) {
    if (!ctx) return fail(QLM_EINVAL, "ctx is NULL");
    if (rank) *rank = ctx->comm ? comm_rank(ctx->comm) : 0;
    if (world) *world = ctx->comm ? comm_world(ctx->comm) : 1;
    if (nccl_version) *nccl_version = comm_nccl_version();
    return QLM_OK;
}

}  // extern "C"
