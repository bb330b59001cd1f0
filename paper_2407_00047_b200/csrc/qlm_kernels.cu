// qlm_kernels.cu -- sm_100a kernels of the bulk RWT-scoring path and their
// launchers.  See DESIGN.md "Kernels" for the roofline of each.
//
//   build_tables_kernel  a0: derived tables (Eq. 2/3 per-group work, Eq. 1/4 tails)
//   scan_kernel<SCORE>   a1-a5, a7: fused candidate generation + Eq. 10 scan +
//                        violation probability + S1/S2 + block/grid argmin
//   scan_kernel<BULK>    a1-a4, a6: per-(candidate, group) wt / sd / v, staged in
//                        shared memory and written with bulk async (TMA) copies
//   reduce_records       a8: min-loc over device records (all-gathered ranks)
//   row_kernel           a9: winner decode / row materialisation
//   mc_sample_kernel     a10: Philox sampling of per-group output tokens
//   mc_count_kernel      a11: per-trial Eq. 10 walk + violation counts
#include <atomic>
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "qlm_device.cuh"
#include "qlm_launch.h"

namespace qlm {

std::atomic<int64_t> g_launches{0};

// =============================================================================
// a0: table build (one block; runs once per qlm_create / qlm_update_groups)
// =============================================================================
__global__ void build_tables_kernel(Dims dm, const qlm_group *__restrict__ grp,
                                    const qlm_queue *__restrict__ que,
                                    const double *__restrict__ theta,
                                    const double *__restrict__ prefill,
                                    const double *__restrict__ eps,
                                    const double *__restrict__ dec,
                                    const double *__restrict__ maxo,
                                    const double *__restrict__ swp, Tables tb) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int G = dm.G, D = dm.D, M = dm.M;
    unsigned long long nsum = 0;
    for (int i = tid; i < G; i += nt) {
        const qlm_group g = grp[i];
        GRec r;
        r.slo = g.slo_s; r.n = g.n_req; r.model = g.model;
        tb.grec[i] = r;
        tb.dist[i] = g.dist_id;
        nsum += (unsigned long long)g.n_req;
    }
    for (int k = tid; k < D * G; k += nt) {
        const int d = k / G, i = k - d * G;
        const qlm_group g = grp[i];
        const double th = theta[d * M + g.model];
        const double n = (double)g.n_req;
        // Eq. 2: W = n mu / Theta;  Eq. 3: var of W = n sigma^2 / Theta^2  (R6/R7)
        tb.ab[k] = make_double2(__ddiv_rn(__dmul_rn(n, g.mu_out), th),
                                __ddiv_rn(__dmul_rn(n, g.var_out), __dmul_rn(th, th)));
    }
    for (int q = tid; q < dm.Q; q += nt) {
        const qlm_queue u = que[q];
        QRec r;
        r.bmean = u.backlog_mean_s; r.bvar = u.backlog_var_s2;
        r.d = u.device; r.r = u.resident_model; r.backlog = u.backlog_mean_s > 0.0; r.pad = 0;
        tb.qrec[q] = r;
    }
    for (int k = tid; k < D * M; k += nt) {
        // Eq. 1 + Eq. 4 with O_q := max output: C - W = P + max_out eps d (R3)
        tb.tail[k] = __dadd_rn(prefill[k], __dmul_rn(__dmul_rn(maxo[k], eps[k]), dec[k]));
        tb.theta[k] = theta[k];
    }
    for (int k = tid; k < D * M * M; k += nt) tb.swap[k] = swp[k];
    // sum_i n_i (exact integer)
    __shared__ unsigned long long red[32];
    for (int o = 16; o; o >>= 1) nsum += __shfl_xor_sync(0xFFFFFFFFu, nsum, o);
    if ((tid & 31) == 0) red[tid >> 5] = nsum;
    __syncthreads();
    if (tid == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < (nt + 31) / 32; ++w) s += red[w];
        *tb.den = (double)s;
    }
}

// =============================================================================
// a1-a7: the scan kernel
// =============================================================================
template <int KIND, typename TOK, typename F>
__device__ __forceinline__ void for_tokens(const ScanParams &p, uint8_t *scratch, int64_t loc,
                                           int64_t c, F &&f) {
    if constexpr (KIND == QLM_CAND_RANDOM)
        tokens_random<TOK>(scratch, p.blk, threadIdx.x, p.dm.T, p.cd.seed, (uint64_t)c, f);
    else if constexpr (KIND == QLM_CAND_EXPLICIT)
        tokens_explicit<TOK>(p.cd.rows + loc * p.cd.stride, p.dm.T, f);
    else
        tokens_enum((uint64_t)c, p.dm.T, f);
}

template <int REP>
__device__ __forceinline__ Walker<REP> stage_tables(const ScanParams &p, uint8_t *smem) {
    const int tid = threadIdx.x, blk = blockDim.x;
    const Dims dm = p.dm;
    GRec *sgrec = reinterpret_cast<GRec *>(smem + p.off_grec);
    for (int i = tid; i < dm.G * REP; i += blk) sgrec[i] = p.tb.grec[i / REP];
    double2 *sab = reinterpret_cast<double2 *>(smem + p.off_ab);
    for (int i = tid; i < dm.D * dm.G * REP; i += blk) sab[i] = p.tb.ab[i / REP];
    QRec *sq = reinterpret_cast<QRec *>(smem + p.off_q);
    for (int i = tid; i < dm.Q; i += blk) sq[i] = p.tb.qrec[i];
    double *stail = reinterpret_cast<double *>(smem + p.off_tail);
    for (int i = tid; i < dm.D * dm.M; i += blk) stail[i] = p.tb.tail[i];
    double *sswap = reinterpret_cast<double *>(smem + p.off_swap);
    for (int i = tid; i < dm.D * dm.M * dm.M; i += blk) sswap[i] = p.tb.swap[i];
    Walker<REP> w;
    w.sgrec = sgrec; w.sab = sab; w.sq = sq; w.stail = stail; w.sswap = sswap;
    w.G = dm.G; w.Q = dm.Q; w.M = dm.M; w.lrep = tid & (REP - 1);
    return w;
}

template <int KIND, typename TOK, int REP>
__global__ void __launch_bounds__(256) score_kernel(const ScanParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, blk = p.blk;
    Walker<REP> w = stage_tables<REP>(p, smem);
    uint8_t *scratch = smem + p.off_scratch;
    __syncthreads();

    int64_t first = p.cd.first;
    if (p.cd.first_from) {
        first = p.cd.first_from->index;
        if (first < 0) {
            if (blockIdx.x == 0 && tid == 0 && p.out_rec) {
                p.out_rec->key = ~0ull; p.out_rec->index = -1;
            }
            return;
        }
    }
    const double den = *p.tb.den;
    const int64_t count = p.cd.count;
    uint64_t bkey = ~0ull;
    int64_t bidx = -1;
    for (int64_t loc = (int64_t)blockIdx.x * blk + tid; loc < count;
         loc += (int64_t)gridDim.x * blk) {
        const int64_t c = first + loc;
        w.start_queue(0);
        double S2 = 0.0, frac = 0.0;
        int cnt = 0, over = 0;
        for_tokens<KIND, TOK>(p, scratch, loc, c, [&](int tok) {
            double wt, V;
            GRec g;
            if (!w.step(tok, wt, V, g)) return;
            const double slack = __dsub_rn(g.slo, wt);   // -p_i (Eq. 11)
            S2 = __dsub_rn(S2, slack);                   // objective sum p
            const float v = violation(slack, V, p.zc2);
            if (v == 1.0f) cnt += g.n;
            else if (v != 0.0f) frac = __dadd_rn(frac, __dmul_rn((double)g.n, (double)v));
            over += v > p.alpha;
        });
        const float s1 = (float)(__dadd_rn((double)cnt, frac) / den);   // R11
        const float s2 = (float)S2;
        if (p.s1) p.s1[loc] = s1;
        if (p.s2) p.s2[loc] = s2;
        if (p.n_over) p.n_over[loc] = over;
        const uint64_t key = make_key(s1, s2);
        if (better(key, c, bkey, bidx)) { bkey = key; bidx = c; }
    }
    if (!p.out_rec) return;

    // ---- argmin: warp -> block -> grid (last block reduces block records) ----
    __shared__ uint64_t rk[32];
    __shared__ int64_t ri[32];
    __shared__ int is_last;
    const int lane = tid & 31, wid = tid >> 5, nwarp = blk >> 5;
    warp_argmin(bkey, bidx);
    if (lane == 0) { rk[wid] = bkey; ri[wid] = bidx; }
    __syncthreads();
    if (wid == 0) {
        uint64_t k = lane < nwarp ? rk[lane] : ~0ull;
        int64_t i = lane < nwarp ? ri[lane] : -1;
        warp_argmin(k, i);
        if (lane == 0) {
            p.block_recs[blockIdx.x].key = k;
            p.block_recs[blockIdx.x].index = i;
            __threadfence();
            const unsigned ticket = atomicAdd(p.counter, 1u);
            is_last = ticket == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    uint64_t k = ~0ull;
    int64_t i = -1;
    for (int j = tid; j < (int)gridDim.x; j += blk) {
        const uint64_t kk = __ldcg(reinterpret_cast<const unsigned long long *>(&p.block_recs[j].key));
        const int64_t ii = __ldcg(reinterpret_cast<const long long *>(&p.block_recs[j].index));
        if (better(kk, ii, k, i)) { k = kk; i = ii; }
    }
    warp_argmin(k, i);
    __syncthreads();
    if (lane == 0) { rk[wid] = k; ri[wid] = i; }
    __syncthreads();
    if (wid == 0) {
        k = lane < nwarp ? rk[lane] : ~0ull;
        i = lane < nwarp ? ri[lane] : -1;
        warp_argmin(k, i);
        if (lane == 0) {
            p.out_rec->key = k;
            p.out_rec->index = i;
            *p.counter = 0u;
        }
    }
}

template <int KIND, typename TOK, int REP, bool STAGE>
__global__ void __launch_bounds__(256) bulk_kernel(const ScanParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, blk = p.blk;
    const int G = p.dm.G;
    Walker<REP> w = stage_tables<REP>(p, smem);
    uint8_t *scratch = smem + p.off_scratch;
    __syncthreads();

    int64_t first = p.cd.first;
    if (p.cd.first_from) {
        first = p.cd.first_from->index;
        if (first < 0) return;
    }
    float *stw = p.off_stage_w >= 0 ? reinterpret_cast<float *>(smem + p.off_stage_w) : nullptr;
    float *sts = p.off_stage_s >= 0 ? reinterpret_cast<float *>(smem + p.off_stage_s) : nullptr;
    float *stv = p.off_stage_v >= 0 ? reinterpret_cast<float *>(smem + p.off_stage_v) : nullptr;
    const int64_t count = p.cd.count;
    const int64_t ntiles = (count + blk - 1) / blk;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t loc0 = tile * blk;
        const int nvalid = (int)min((int64_t)blk, count - loc0);
        const int64_t loc = loc0 + tid;
        if (STAGE && p.use_tma && tile != blockIdx.x) {
            if (tid == 0) bulk_wait_read0();          // staging buffer free again
            __syncthreads();
        }
        if (tid < nvalid) {
            float *pw = p.wt ? (STAGE ? stw + tid * G : p.wt + loc * G) : nullptr;
            float *ps = p.sd ? (STAGE ? sts + tid * G : p.sd + loc * G) : nullptr;
            float *pv = p.vo ? (STAGE ? stv + tid * G : p.vo + loc * G) : nullptr;
            w.start_queue(0);
            for_tokens<KIND, TOK>(p, scratch, loc, first + loc, [&](int tok) {
                double wt, V;
                GRec g;
                if (!w.step(tok, wt, V, g)) return;
                if (pw) pw[tok] = (float)wt;
                if (ps) ps[tok] = sqrtf((float)V);
                if (pv) pv[tok] = violation(__dsub_rn(g.slo, wt), V, p.zc2);
            });
        }
        if constexpr (STAGE) {
            const uint32_t bytes = (uint32_t)nvalid * (uint32_t)G * 4u;
            if (p.use_tma) {
                fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0) {
                    if (stw) bulk_s2g(p.wt + loc0 * G, stw, bytes);
                    if (sts) bulk_s2g(p.sd + loc0 * G, sts, bytes);
                    if (stv) bulk_s2g(p.vo + loc0 * G, stv, bytes);
                    bulk_commit();
                }
            } else {
                __syncthreads();
                const int nw = nvalid * G;
                for (int i = tid; i < nw; i += blk) {
                    if (stw) p.wt[loc0 * G + i] = stw[i];
                    if (sts) p.sd[loc0 * G + i] = sts[i];
                    if (stv) p.vo[loc0 * G + i] = stv[i];
                }
                __syncthreads();
            }
        }
    }
    if constexpr (STAGE) {
        if (p.use_tma && tid == 0) bulk_wait0();
    }
}

// =============================================================================
// a8: min-loc over records (e.g. one per rank after an all-gather)
// =============================================================================
__global__ void reduce_records_kernel(const qlm_record *recs, int n, qlm_record *out) {
    __shared__ uint64_t rk[32];
    __shared__ int64_t ri[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
    uint64_t k = ~0ull;
    int64_t i = -1;
    for (int j = tid; j < n; j += blockDim.x)
        if (better(recs[j].key, recs[j].index, k, i)) { k = recs[j].key; i = recs[j].index; }
    warp_argmin(k, i);
    if (lane == 0) { rk[wid] = k; ri[wid] = i; }
    __syncthreads();
    if (wid == 0) {
        k = lane < nwarp ? rk[lane] : ~0ull;
        i = lane < nwarp ? ri[lane] : -1;
        warp_argmin(k, i);
        if (lane == 0) { out->key = k; out->index = i; }
    }
}

// =============================================================================
// a9: rows / decode (thread per candidate, same generators as the scan)
// =============================================================================
template <int KIND, typename TOK>
__global__ void __launch_bounds__(64) row_kernel(const ScanParams p, uint16_t *rows_out,
                                                 int32_t *queue_of, int32_t *pos_of) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t *scratch = smem;
    int64_t first = p.cd.first;
    if (p.cd.first_from) {
        first = p.cd.first_from->index;
        if (first < 0) return;
    }
    const int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (loc >= p.cd.count) return;
    const int T = p.dm.T, G = p.dm.G, Q = p.dm.Q;
    int s = 0, q = 0, pos = 0;
    for_tokens<KIND, TOK>(p, scratch, loc, first + loc, [&](int tok) {
        if (rows_out) rows_out[loc * T + s] = (uint16_t)tok;
        ++s;
        if (tok >= G) {
            q = q + 1 < Q ? q + 1 : Q - 1;
            pos = 0;
            return;
        }
        if (queue_of) queue_of[loc * G + tok] = q;
        if (pos_of) pos_of[loc * G + tok] = pos;
        ++pos;
    });
}

// Eq. 6 bijection check, one block per row.
__global__ void check_rows_kernel(const Cand cd, int T, unsigned long long *n_bad) {
    extern __shared__ uint32_t bits[];
    const int nwords = (T + 31) / 32;
    for (int k = threadIdx.x; k < nwords; k += blockDim.x) bits[k] = 0u;
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    const uint8_t *row = cd.rows + (int64_t)blockIdx.x * cd.stride;
    int mybad = 0;
    for (int s = threadIdx.x; s < T; s += blockDim.x) {
        const int tok = cd.tb == 1 ? row[s] : reinterpret_cast<const uint16_t *>(row)[s];
        if (tok >= T) { mybad = 1; continue; }
        const uint32_t m = 1u << (tok & 31);
        if (atomicOr(&bits[tok >> 5], m) & m) mybad = 1;
    }
    if (mybad) atomicOr(&bad, 1);
    __syncthreads();
    if (threadIdx.x == 0 && bad) atomicAdd(n_bad, 1ull);
}

// =============================================================================
// a10-a11: Monte-Carlo
// =============================================================================
// X[k][t] = sum_{r < n_k} len[dist_k][word(t, k, r) >> shift]   (R13)
__global__ void __launch_bounds__(256) mc_sample_kernel(Dims dm, Tables tb, uint64_t seed,
                                                        int64_t t0, int64_t nt, uint32_t *X,
                                                        int tabs_in_smem) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint16_t *len = tb.len;
    if (tabs_in_smem) {
        uint4 *s4 = reinterpret_cast<uint4 *>(smem);
        const uint4 *g4 = reinterpret_cast<const uint4 *>(tb.len);
        const int n4 = dm.n_tables * dm.K * 2 / 16;
        for (int i = threadIdx.x; i < n4; i += blockDim.x) s4[i] = g4[i];
        __syncthreads();
        len = reinterpret_cast<const uint16_t *>(smem);
    }
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const int64_t total = (int64_t)dm.G * nt;
    const int shift = dm.shift;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx / nt);
        const int64_t tl = idx - (int64_t)k * nt;
        const uint32_t t = (uint32_t)(t0 + tl);
        const int n = tb.grec[k].n;
        const uint16_t *tab = len + (int64_t)tb.dist[k] * dm.K;
        uint32_t sum = 0;
        for (int r0 = 0; r0 < n; r0 += 4) {
            const uint4 wd = philox10(make_uint4((uint32_t)(r0 >> 2), (uint32_t)k, t, kMcTag), key);
            sum += tab[wd.x >> shift];
            if (r0 + 1 < n) sum += tab[wd.y >> shift];
            if (r0 + 2 < n) sum += tab[wd.z >> shift];
            if (r0 + 3 < n) sum += tab[wd.w >> shift];
        }
        X[(int64_t)k * nt + tl] = sum;
    }
}

// One block per (candidate, chunk of trials); every thread is one trial and
// walks the shared row; counts via warp ballots into shared counters.
__global__ void __launch_bounds__(256) mc_count_kernel(Dims dm, Tables tb, const uint16_t *rows,
                                                       const qlm_record *first_from,
                                                       const uint32_t *X, int64_t nt,
                                                       uint32_t *counts) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (first_from && first_from->index < 0) return;
    const int T = dm.T, G = dm.G, M = dm.M;
    uint16_t *srow = reinterpret_cast<uint16_t *>(smem);
    uint32_t *scnt = reinterpret_cast<uint32_t *>(smem + ((T * 2 + 15) & ~15));
    const int64_t c = blockIdx.y;
    for (int s = threadIdx.x; s < T; s += blockDim.x) srow[s] = rows[c * T + s];
    for (int g = threadIdx.x; g < G; g += blockDim.x) scnt[g] = 0u;
    __syncthreads();
    const int64_t tl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = tl < nt;
    const int lane = threadIdx.x & 31;
    int q = 0;
    QRec qr = tb.qrec[0];
    double A = qr.bmean;
    int d = qr.d, prev = qr.r, first = 1, backlog = qr.backlog;
    for (int s = 0; s < T; ++s) {
        const int tok = srow[s];
        if (tok >= G) {
            q = q + 1 < dm.Q ? q + 1 : dm.Q - 1;
            qr = tb.qrec[q];
            A = qr.bmean; d = qr.d; prev = qr.r; first = 1; backlog = qr.backlog;
            continue;
        }
        const GRec g = tb.grec[tok];
        const int m = g.model;
        if (m != prev) {
            const double t = (first && !backlog) ? 0.0 : tb.tail[d * M + prev];
            A = __dadd_rn(A, t);
            A = __dadd_rn(A, tb.swap[(d * M + prev) * M + m]);
        }
        const unsigned b = __ballot_sync(0xFFFFFFFFu, act && A > g.slo);
        if (lane == 0 && b) atomicAdd(&scnt[tok], (unsigned)__popc(b));
        const double x = act ? (double)X[(int64_t)tok * nt + tl] : 0.0;
        A = __dadd_rn(A, __ddiv_rn(x, tb.theta[d * M + m]));   // Eq. 2 with realised O
        prev = m; first = 0;
    }
    __syncthreads();
    for (int g = threadIdx.x; g < G; g += blockDim.x)
        if (scnt[g]) atomicAdd(&counts[c * G + g], scnt[g]);
}

// =============================================================================
// launchers
// =============================================================================
static int g_sm_count = 0;

int sm_count() {
    if (!g_sm_count) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    }
    return g_sm_count;
}

static size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Shared-memory plan of the scan kernels.
static size_t plan_smem(ScanParams &p, int rep, int kind, int tok_bytes, int blk, int nstage,
                        bool stage) {
    const Dims &dm = p.dm;
    size_t off = 0;
    p.off_grec = (int)off; off = align16(off + (size_t)dm.G * rep * sizeof(GRec));
    p.off_ab = (int)off;   off = align16(off + (size_t)dm.D * dm.G * rep * sizeof(double2));
    p.off_q = (int)off;    off = align16(off + (size_t)dm.Q * sizeof(QRec));
    p.off_tail = (int)off; off = align16(off + (size_t)dm.D * dm.M * sizeof(double));
    p.off_swap = (int)off; off = align16(off + (size_t)dm.D * dm.M * dm.M * sizeof(double));
    p.off_scratch = (int)off;
    if (kind == QLM_CAND_RANDOM) {
        const int epw = 4 / tok_bytes;
        off = align16(off + (size_t)((dm.T + epw - 1) / epw) * 4 * blk);
    }
    p.off_stage_w = p.off_stage_s = p.off_stage_v = -1;
    if (stage) {
        const size_t arr = (size_t)blk * dm.G * 4;
        if (p.wt) { p.off_stage_w = (int)off; off = align16(off + arr); }
        if (p.sd) { p.off_stage_s = (int)off; off = align16(off + arr); }
        if (p.vo) { p.off_stage_v = (int)off; off = align16(off + arr); }
    }
    (void)nstage;
    return off;
}

static const size_t kMaxSmem = 227 * 1024;

// Largest dynamic shared memory a launch of `kern` may use (opt-in limit
// minus the kernel's static shared memory); opts the kernel into it once.
template <typename K>
static size_t max_dyn(K kern) {
    static std::mutex mu;
    static std::unordered_map<const void *, size_t> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(reinterpret_cast<const void *>(kern));
    if (it != cache.end()) return it->second;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) { cudaGetLastError(); return 0; }
    size_t m = optin > (int)fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
    if (m > kMaxSmem) m = kMaxSmem;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cache[reinterpret_cast<const void *>(kern)] = m;
    return m;
}

template <typename K>
static cudaError_t prep(K kern, size_t smem) {
    return smem <= max_dyn(kern) ? cudaSuccess : cudaErrorInvalidValue;
}

template <typename K>
static int occupancy(K kern, int blk, size_t smem) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, blk, smem) != cudaSuccess) return 0;
    return nb;
}

static int choose_rep(const Dims &dm) {
    const size_t rec = (size_t)dm.G * (1 + dm.D) * 16;
    return rec * 8 <= 40 * 1024 ? 8 : 1;
}

// ---- score ----
template <int KIND, typename TOK, int REP>
static cudaError_t launch_score_t(ScanParams p, cudaStream_t st) {
    auto kern = score_kernel<KIND, TOK, REP>;
    const size_t lim = max_dyn(kern);
    int blk = 128;
    size_t smem = 0;
    for (; blk >= 32; blk >>= 1) {
        smem = plan_smem(p, REP, KIND, sizeof(TOK), blk, 0, false);
        if (smem <= lim) break;
    }
    if (blk < 32) return cudaErrorInvalidConfiguration;
    p.blk = blk;
    cudaError_t e = prep(kern, smem);
    if (e != cudaSuccess) return e;
    const int nb = occupancy(kern, blk, smem);
    int64_t grid = (p.cd.count + blk - 1) / blk;
    const int64_t maxg = (int64_t)sm_count() * (nb > 0 ? nb : 1);
    if (grid > maxg) grid = maxg;
    if (grid > p.max_blocks) grid = p.max_blocks;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, blk, smem, st>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

template <int KIND, typename TOK>
static cudaError_t launch_score_k(const ScanParams &p, cudaStream_t st) {
    return choose_rep(p.dm) == 8 ? launch_score_t<KIND, TOK, 8>(p, st)
                                 : launch_score_t<KIND, TOK, 1>(p, st);
}

cudaError_t launch_score(const ScanParams &p, cudaStream_t st) {
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM:
        return p.dm.T <= 256 ? launch_score_k<QLM_CAND_RANDOM, uint8_t>(p, st)
                             : launch_score_k<QLM_CAND_RANDOM, uint16_t>(p, st);
    case QLM_CAND_EXPLICIT:
        return p.cd.tb == 1 ? launch_score_k<QLM_CAND_EXPLICIT, uint8_t>(p, st)
                            : launch_score_k<QLM_CAND_EXPLICIT, uint16_t>(p, st);
    default:
        return launch_score_k<QLM_CAND_ENUM, uint8_t>(p, st);
    }
}

// ---- bulk ----
template <int KIND, typename TOK, int REP>
static cudaError_t launch_bulk_t(ScanParams p, cudaStream_t st) {
    const int nout = (p.wt != nullptr) + (p.sd != nullptr) + (p.vo != nullptr);
    // pick the block size maximising resident candidates per SM with staging
    int best_blk = 0, best_thr = 0;
    size_t best_smem = 0;
    for (int blk = 128; blk >= 32; blk >>= 1) {
        ScanParams q = p;
        const size_t smem = plan_smem(q, REP, KIND, sizeof(TOK), blk, nout, true);
        auto kern = bulk_kernel<KIND, TOK, REP, true>;
        if (smem > max_dyn(kern)) continue;
        if (prep(kern, smem) != cudaSuccess) continue;
        const int thr = occupancy(kern, blk, smem) * blk;
        if (thr > best_thr) { best_thr = thr; best_blk = blk; best_smem = smem; }
    }
    const bool aligned = (p.dm.G % 4 == 0) &&
                         (!p.wt || ((uintptr_t)p.wt & 15) == 0) &&
                         (!p.sd || ((uintptr_t)p.sd & 15) == 0) &&
                         (!p.vo || ((uintptr_t)p.vo & 15) == 0);
    if (best_blk && nout > 0) {
        p.blk = best_blk;
        plan_smem(p, REP, KIND, sizeof(TOK), best_blk, nout, true);
        p.use_tma = aligned ? 1 : 0;
        auto kern = bulk_kernel<KIND, TOK, REP, true>;
        int64_t grid = (p.cd.count + best_blk - 1) / best_blk;
        const int64_t maxg = (int64_t)sm_count() * (best_thr / best_blk);
        if (grid > maxg) grid = maxg;
        if (grid < 1) grid = 1;
        kern<<<(unsigned)grid, best_blk, best_smem, st>>>(p);
        ++g_launches;
        return cudaGetLastError();
    }
    // no staging: direct stores
    const size_t lim = max_dyn(bulk_kernel<KIND, TOK, REP, false>);
    int blk = 128;
    size_t smem = 0;
    for (; blk >= 32; blk >>= 1) {
        smem = plan_smem(p, REP, KIND, sizeof(TOK), blk, 0, false);
        if (smem <= lim) break;
    }
    if (blk < 32) return cudaErrorInvalidConfiguration;
    p.blk = blk;
    p.use_tma = 0;
    auto kern = bulk_kernel<KIND, TOK, REP, false>;
    cudaError_t e = prep(kern, smem);
    if (e != cudaSuccess) return e;
    const int nb = occupancy(kern, blk, smem);
    int64_t grid = (p.cd.count + blk - 1) / blk;
    const int64_t maxg = (int64_t)sm_count() * (nb > 0 ? nb : 1);
    if (grid > maxg) grid = maxg;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, blk, smem, st>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

template <int KIND, typename TOK>
static cudaError_t launch_bulk_k(const ScanParams &p, cudaStream_t st) {
    return choose_rep(p.dm) == 8 ? launch_bulk_t<KIND, TOK, 8>(p, st)
                                 : launch_bulk_t<KIND, TOK, 1>(p, st);
}

cudaError_t launch_bulk(const ScanParams &p, cudaStream_t st) {
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM:
        return p.dm.T <= 256 ? launch_bulk_k<QLM_CAND_RANDOM, uint8_t>(p, st)
                             : launch_bulk_k<QLM_CAND_RANDOM, uint16_t>(p, st);
    case QLM_CAND_EXPLICIT:
        return p.cd.tb == 1 ? launch_bulk_k<QLM_CAND_EXPLICIT, uint8_t>(p, st)
                            : launch_bulk_k<QLM_CAND_EXPLICIT, uint16_t>(p, st);
    default:
        return launch_bulk_k<QLM_CAND_ENUM, uint8_t>(p, st);
    }
}

// ---- rows / decode ----
template <int KIND, typename TOK>
static cudaError_t launch_rows_t(ScanParams p, uint16_t *rows, int32_t *qo, int32_t *po,
                                 cudaStream_t st) {
    auto kern = row_kernel<KIND, TOK>;
    const size_t lim = max_dyn(kern);
    int blk = 64;
    size_t smem = 0;
    for (; blk >= 1; blk >>= 1) {
        smem = 0;
        if (KIND == QLM_CAND_RANDOM) {
            const int epw = 4 / (int)sizeof(TOK);
            smem = align16((size_t)((p.dm.T + epw - 1) / epw) * 4 * blk);
        }
        if (smem <= lim) break;
    }
    p.blk = blk;
    cudaError_t e = prep(kern, smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (p.cd.count + blk - 1) / blk;
    if (grid < 1) return cudaSuccess;
    kern<<<(unsigned)grid, blk, smem, st>>>(p, rows, qo, po);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_rows(const ScanParams &p, uint16_t *rows, int32_t *qo, int32_t *po,
                        cudaStream_t st) {
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM:
        return p.dm.T <= 256 ? launch_rows_t<QLM_CAND_RANDOM, uint8_t>(p, rows, qo, po, st)
                             : launch_rows_t<QLM_CAND_RANDOM, uint16_t>(p, rows, qo, po, st);
    case QLM_CAND_EXPLICIT:
        return p.cd.tb == 1 ? launch_rows_t<QLM_CAND_EXPLICIT, uint8_t>(p, rows, qo, po, st)
                            : launch_rows_t<QLM_CAND_EXPLICIT, uint16_t>(p, rows, qo, po, st);
    default:
        return launch_rows_t<QLM_CAND_ENUM, uint8_t>(p, rows, qo, po, st);
    }
}

cudaError_t launch_reduce_records(const qlm_record *recs, int n, qlm_record *out,
                                  cudaStream_t st) {
    reduce_records_kernel<<<1, 256, 0, st>>>(recs, n, out);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_check_rows(const Cand &cd, int T, unsigned long long *n_bad, cudaStream_t st) {
    if (cd.count <= 0) return cudaSuccess;
    const size_t smem = (size_t)((T + 31) / 32) * 4;
    check_rows_kernel<<<(unsigned)cd.count, 128, smem, st>>>(cd, T, n_bad);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_build(const Dims &dm, const qlm_group *g, const qlm_queue *q,
                         const double *theta, const double *prefill, const double *eps,
                         const double *dec, const double *maxo, const double *swp,
                         const Tables &tb, cudaStream_t st) {
    build_tables_kernel<<<1, 256, 0, st>>>(dm, g, q, theta, prefill, eps, dec, maxo, swp, tb);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_mc_sample(const Dims &dm, const Tables &tb, uint64_t seed, int64_t t0,
                             int64_t nt, uint32_t *X, cudaStream_t st) {
    const size_t tab_bytes = (size_t)dm.n_tables * dm.K * 2;
    const int in_smem = tab_bytes <= 160 * 1024 && (tab_bytes % 16) == 0;
    const size_t smem = in_smem ? tab_bytes : 0;
    cudaError_t e = prep(mc_sample_kernel, smem);
    if (e != cudaSuccess) return e;
    const int nb = occupancy(mc_sample_kernel, 256, smem);
    int64_t grid = ((int64_t)dm.G * nt + 255) / 256;
    const int64_t maxg = (int64_t)sm_count() * (nb > 0 ? nb : 1) * 4;
    if (grid > maxg) grid = maxg;
    if (grid < 1) grid = 1;
    mc_sample_kernel<<<(unsigned)grid, 256, smem, st>>>(dm, tb, seed, t0, nt, X, in_smem);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_mc_count(const Dims &dm, const Tables &tb, const uint16_t *rows,
                            const qlm_record *first_from, int64_t count, const uint32_t *X,
                            int64_t nt, uint32_t *counts, cudaStream_t st) {
    const size_t smem = align16((size_t)dm.T * 2) + (size_t)dm.G * 4;
    cudaError_t e = prep(mc_count_kernel, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((nt + 255) / 256), (unsigned)count);
    mc_count_kernel<<<grid, 256, smem, st>>>(dm, tb, rows, first_from, X, nt, counts);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace qlm
