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
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>

#include "qlm_device.cuh"
#include "qlm_launch.h"

namespace qlm {

std::atomic<int64_t> g_launches{0};
std::atomic<uint32_t> g_override_flags{0};
std::atomic<int64_t> g_override_ilv_cap{0};

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
// a1-a7: the fused scan kernel
// =============================================================================
// One thread = one candidate.  Per tile of blockDim consecutive candidates:
// generate the row (RANDOM: Philox + forward Fisher-Yates in per-thread smem
// scratch; EXPLICIT: 16-B row loads; ENUM: Lehmer unranking), walk it once
// (Eq. 2/3/10), and in the same pass
//   OUT_STAGED: stage wt / sd / v group-major in smem ([g][tid]: bank = lane,
//               conflict-free) and write each group's row segment with one
//               bulk async copy (TMA engine) -> out[g][c0 .. c0+n)
//   OUT_DIRECT: store them straight to out[g][c] (large G, no room to stage)
//   SCORE:      S1 / S2 / n_over per candidate and the running argmin.
enum { OUT_NONE = 0, OUT_STAGED = 1, OUT_DIRECT = 2 };

template <int KIND, typename TOK, typename F>
__device__ __forceinline__ void for_tokens(const Cand &cd, int T, uint8_t *scratch, int blk,
                                           int64_t loc, int64_t c, F &&f) {
    if constexpr (KIND == QLM_CAND_RANDOM) {
        fy_materialise<TOK>(scratch, blk, threadIdx.x, T, cd.seed, (uint64_t)c);
        tokens_scratch<TOK>(scratch, blk, threadIdx.x, T, f);
    } else if constexpr (KIND == QLM_CAND_EXPLICIT) {
        tokens_explicit<TOK>(cd.rows + loc * cd.stride, T, f);
    } else if constexpr (KIND == QLM_CAND_NEIGHBOR) {
        tokens_neighbor<TOK>(cd, T, (uint64_t)c, f);
    } else if constexpr (KIND == KIND_ILV) {
        // word-interleaved rows: consecutive candidates read consecutive words
        constexpr int EPW = 4 / (int)sizeof(TOK);
        const uint32_t *w32 = reinterpret_cast<const uint32_t *>(cd.rows) + loc;
        const int nw = (T + EPW - 1) / EPW;
        uint32_t nxt = __ldcs(w32);
        for (int w = 0; w < nw; ++w) {
            const uint32_t cur = nxt;
            if (w + 1 < nw) nxt = __ldcs(w32 + (size_t)(w + 1) * cd.stride);   // prefetch
#pragma unroll
            for (int k = 0; k < EPW; ++k) {
                const int s = w * EPW + k;
                if (s >= T) break;
                f(EPW == 2 ? (int)((cur >> (16 * k)) & 0xFFFFu) : (int)((cur >> (8 * k)) & 0xFFu));
            }
        }
    } else {
        tokens_enum((uint64_t)c, T, f);
    }
}

__device__ __forceinline__ SlotTables stage_tables(const ScanParams &p, uint8_t *smem) {
    const int tid = threadIdx.x, blk = blockDim.x;
    const Dims dm = p.dm;
    const int rs = p.rep_shift;
    GRec *sg = reinterpret_cast<GRec *>(smem + p.off_grec);
    for (int i = tid; i < (dm.G << rs); i += blk) sg[i] = p.tb.grec[i >> rs];
    double2 *sab = reinterpret_cast<double2 *>(smem + p.off_ab);
    for (int i = tid; i < ((dm.D * dm.G) << rs); i += blk) sab[i] = p.tb.ab[i >> rs];
    QRec *sq = reinterpret_cast<QRec *>(smem + p.off_q);
    for (int i = tid; i < dm.Q; i += blk) sq[i] = p.tb.qrec[i];
    double *str = reinterpret_cast<double *>(smem + p.off_tr);
    const int M = dm.M;
    const int trs = p.tr_shift;
    for (int i = tid; i < (dm.D * 2 * M * M) << trs; i += blk) {
        const int e = i >> trs;
        const int m = e % M, pp = (e / M) % (2 * M), d = e / (2 * M * M);
        const int from = pp < M ? pp : pp - M;
        const double sw = p.tb.swap[(d * M + from) * M + m];
        const double tl = (pp < M && m != pp) ? p.tb.tail[d * M + pp] : 0.0;
        str[i] = __dadd_rn(tl, sw);                       // one transition term (R2/R3)
    }
    SlotTables t;
    t.sg = sg; t.sab = sab; t.str = str; t.sq = sq;
    t.G = dm.G; t.Q = dm.Q; t.M = dm.M; t.rs = rs; t.rl = tid & ((1 << rs) - 1);
    t.trs = trs; t.trl = tid & ((1 << trs) - 1);
    return t;
}

template <int KIND, typename TOK, int OUT, bool SCORE>
__global__ void __launch_bounds__(256) scan_kernel(const ScanParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, blk = blockDim.x;
    const SlotTables tab = stage_tables(p, smem);
    uint8_t *scratch = smem + p.off_scratch;
    __syncthreads();

    const Cand cd = p.cd;
    int64_t first = cd.first;
    if (cd.first_from) {
        first = cd.first_from->index;
        if (first < 0) {
            if (SCORE && p.out_rec && blockIdx.x == 0 && tid == 0) {
                p.out_rec->key = ~0ull; p.out_rec->index = -1;
            }
            return;
        }
    }
    const int G = p.dm.G, Q = p.dm.Q, T = p.dm.T;
    const float zc = p.zc;
    const float alpha = p.alpha;
    const int64_t count = cd.count;
    const int64_t ldo = p.ld_out ? p.ld_out : count;     // bulk leading dimension
    float *const gout[3] = {p.wt, p.sd, p.vo};
    float *st0 = nullptr, *st1 = nullptr, *st2 = nullptr;   // staged tile [3][G][blk]
    if constexpr (OUT == OUT_STAGED) {
        st0 = reinterpret_cast<float *>(smem + p.off_stage);
        st1 = st0 + (size_t)G * blk;
        st2 = st1 + (size_t)G * blk;
    }
    const double den = SCORE ? *p.tb.den : 1.0;
    uint64_t bkey = ~0ull;
    int64_t bidx = -1;
    const int64_t ntiles = (count + blk - 1) / blk;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t c0 = tile * blk;
        const int nvalid = (int)min((int64_t)blk, count - c0);
        const int64_t loc = c0 + tid;
        if constexpr (OUT == OUT_STAGED) {
            if (tile != blockIdx.x) {                 // staging free again?
                if (p.use_tma) bulk_wait_read0();
                __syncthreads();
            }
        }
        if (tid < nvalid) {
            ScanState s;
            start_queue(tab, s, 0);
            double S2 = 0.0, acc2 = 0.0;          // sum n_i v_i: clamped (fp32, exact integers) /
            float acc1 = 0.0f;                    // unclamped (fp64) slots, row order (R11)
            int over = 0;
            for_tokens<KIND, TOK>(cd, T, scratch, blk, loc, first + loc, [&](int tok) {
                if (tok >= G) {                          // queue separator
                    start_queue(tab, s, s.q + 1 < Q ? s.q + 1 : Q - 1);
                    return;
                }
                double wt;
                float V;
                GRec g;
                group_slot(tab, s, tok, wt, V, g);
                const double slack = __dsub_rn(g.slo, wt);        // -p_i (Eq. 11)
                const float sd = slot_sd(V);
                bool clamped;
                const float v = slot_v(slack, sd, zc, clamped);
                if constexpr (SCORE) {
                    S2 = __dsub_rn(S2, slack);                    // sum_i p_i
                    if (clamped) acc1 = fmaf((float)g.n, v, acc1);
                    else acc2 = __fma_rn((double)g.n, (double)v, acc2);
                    over += v > alpha;
                }
                if constexpr (OUT == OUT_STAGED) {
                    const int o = tok * blk + tid;
                    st0[o] = (float)wt;
                    st1[o] = sd;
                    st2[o] = v;
                } else if constexpr (OUT == OUT_DIRECT) {
                    const int64_t o = (int64_t)tok * ldo + loc;
                    if (gout[0]) gout[0][o] = (float)wt;
                    if (gout[1]) gout[1][o] = sd;
                    if (gout[2]) gout[2][o] = v;
                }
            });
            if constexpr (SCORE) {
                const float s1 = (float)(((double)acc1 + acc2) / den);   // R11
                const float s2 = (float)S2;
                if (p.s1) p.s1[loc] = s1;
                if (p.s2) p.s2[loc] = s2;
                if (p.n_over) p.n_over[loc] = over;
                const uint64_t key = make_key(s1, s2);
                const int64_t c = first + loc;
                if (better(key, c, bkey, bidx)) { bkey = key; bidx = c; }
            }
        }
        if constexpr (OUT == OUT_STAGED) {
            float *const sts[3] = {st0, st1, st2};
            if (p.use_tma) {
                fence_proxy_async_smem();
                __syncthreads();
                for (int r = tid; r < 3 * G; r += blk) {
                    const int a = r / G, g = r - a * G;
                    if (gout[a])
                        bulk_s2g(gout[a] + (int64_t)g * ldo + c0, sts[a] + (size_t)g * blk,
                                 (uint32_t)nvalid * 4u);
                }
                bulk_commit();
            } else {
                __syncthreads();
                if (tid < nvalid)
                    for (int a = 0; a < 3; ++a)
                        if (gout[a])
                            for (int g = 0; g < G; ++g)
                                gout[a][(int64_t)g * ldo + loc] = sts[a][g * blk + tid];
            }
        }
    }
    if constexpr (OUT == OUT_STAGED) {
        if (p.use_tma) bulk_wait0();
    }
    if constexpr (!SCORE) return;
    if (!p.out_rec) return;

    // ---- argmin: warp -> block -> grid (the last block reduces block records) ----
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
// a1 for large T: RANDOM rows materialised word-interleaved (two-phase path)
// =============================================================================
// One lane per candidate; the lane's row lives in its column of a [T][32] u16
// shared-memory tile (address = base + 64 j).  Forward Fisher-Yates (R10),
// software-pipelined two steps deep: step i issues the loads of position i+2
// and of row[j_{i+1}] before its own store, and the consumers forward the
// values of the (at most two) stores issued after a load that may alias it.
// So the store chain waits on a load issued two steps earlier.  Finals are
// packed two per word and leave as coalesced 128-B warp stores.
// Large T only (the two-phase path runs for T > 256): 32-bit draws (R10).
__global__ void __launch_bounds__(32) fy_rows_kernel(Cand cd, int T, uint32_t *out, int64_t ld) {
    extern __shared__ __align__(16) uint16_t srow16[];
    const int lane = threadIdx.x;
    const int64_t loc = (int64_t)blockIdx.x * 32 + lane;
    const bool act = loc < cd.count;
    const uint64_t c = (uint64_t)(cd.first + loc);
    for (int i = 0; i < T; ++i) srow16[i * 32 + lane] = (uint16_t)i;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(srow16) + 2u * lane;
    auto ld16 = [&](int i) {
        uint16_t v;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(base + ((uint32_t)i << 6)) : "memory");
        return (uint32_t)v;
    };
    auto st16 = [&](int i, uint32_t v) {
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(base + ((uint32_t)i << 6)), "h"((uint16_t)v) : "memory");
    };
    const uint2 key = make_uint2((uint32_t)cd.seed, (uint32_t)(cd.seed >> 32));
    const uint32_t clo = (uint32_t)c, chi = (uint32_t)(c >> 32);
    uint32_t *o = out + loc;
    auto jof = [&](uint4 wd, int k, int i) { return i + (int)__umulhi(pick4(wd, k), (uint32_t)(T - i)); };
    if (T == 1) {
        if (act) __stcs(o, 0u);
        return;
    }
    // pipeline state: t0 = value at position i, t1m = value step i-1 stored,
    // jm = j_{i-1}; raw1 = mem[i+1] loaded before store i-1 (pending forwards
    // from steps i-1 and i); rj = mem[j_i] loaded before store i-1 (forward
    // from step i-1)
    uint4 wd = philox10(make_uint4(0u, clo, chi, kRowTag), key);
    int j = jof(wd, 0, 0);
    uint32_t t0 = 0, t1m = 0xFFFFFFFFu;
    int jm = -1;
    uint32_t raw1 = ld16(1), rj = ld16(j);
    uint32_t fin = 0;
    uint32_t *op = o;                                  // word (i >> 1) of this lane's row
    // one step i: forward the pending values, store row[j_i] = row[i], pack the
    // final row[i] and advance the two-deep pipeline (jn = j_{i+1}, raw2 =
    // mem[i+2] and rjn = mem[j_{i+1}] were loaded before this step's store)
    auto step = [&](int i, int jn, uint32_t raw2, uint32_t rjn) {
        const uint32_t tj = (jm == j) ? t1m : rj;              // value at j_i before step i
        st16(j, t0);                                           // row[j_i] = row[i]
        if (i & 1) {
            fin |= tj << 16;
            if (act) __stcs(op, fin);
            op += ld;
        } else {
            fin = tj;
        }
        // value at position i+1 before step i+1 (raw1 misses stores i-1 and i)
        const uint32_t t1 = (j == i + 1) ? t0 : ((jm == i + 1) ? t1m : raw1);
        t1m = t0; jm = j;
        t0 = t1; j = jn;
        raw1 = raw2; rj = rjn;
    };
    int i0 = 0;
    // main body: whole Philox blocks whose steps all have i + 2 < T (no bounds
    // checks); the next block is independent of this one's steps: issue it first
    for (; i0 + 4 <= T - 3; i0 += 4) {
        const uint4 wn = philox10(make_uint4((uint32_t)((i0 >> 2) + 1), clo, chi, kRowTag), key);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k;
            const int jn = k < 3 ? jof(wd, k + 1, i + 1) : jof(wn, 0, i + 1);
            step(i, jn, ld16(i + 2), ld16(jn));
        }
        wd = wn;
    }
    // tail: the last steps, with bounds
    for (; i0 < T - 1; i0 += 4) {
        const uint4 wn = i0 + 4 < T - 1 ? philox10(make_uint4((uint32_t)((i0 >> 2) + 1), clo, chi, kRowTag), key)
                                        : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k;
            if (i >= T - 1) break;
            const int jn = i + 1 < T - 1 ? (k < 3 ? jof(wd, k + 1, i + 1) : jof(wn, 0, i + 1)) : 0;
            const uint32_t raw2 = i + 2 < T ? ld16(i + 2) : 0u;   // mem[i+2]: misses stores i, i+1
            step(i, jn, raw2, ld16(jn));                           // mem[j_{i+1}]: misses store i
        }
        wd = wn;
    }
    if ((T - 1) & 1) fin |= t0 << 16;             // position T-1 holds the carried value
    else fin = t0;
    if (act) __stcs(op, fin);
}

// qlm_winner's result, written by the device straight into the caller's
// pinned (device-mapped) host buffers: one launch instead of five D2H copies.
__global__ void __launch_bounds__(256) winner_out_kernel(const qlm_record *rec, const float *s12,
                                                         const int32_t *n_over, const int32_t *dec, int G,
                                                         qlm_best *out, int32_t *qo, int32_t *po) {
    if (threadIdx.x == 0) {
        qlm_best b;
        b.index = rec->index;
        b.s1 = s12[0];
        b.s2 = s12[1];
        b.n_over = *n_over;
        b.reserved = 0;
        *out = b;
    }
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        if (qo) qo[g] = dec[g];
        if (po) po[g] = dec[G + g];
    }
}

cudaError_t launch_winner_out(const qlm_record *rec, const float *s12, const int32_t *n_over,
                              const int32_t *dec, int G, qlm_best *out, int32_t *qo, int32_t *po,
                              cudaStream_t st) {
    winner_out_kernel<<<1, 256, 0, st>>>(rec, s12, n_over, dec, G, out, qo, po);
    ++g_launches;
    return cudaGetLastError();
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
    for_tokens<KIND, TOK>(p.cd, T, scratch, blockDim.x, loc, first + loc, [&](int tok) {
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

// One candidate row generated by a whole warp (small counts: winner decode,
// MC).  RANDOM: the lanes compute the row's Philox blocks in parallel, then
// lane 0 runs the Fisher-Yates swaps from shared memory (same permutation as
// fy_materialise).  Returns with srow[0..T) valid for all lanes.
// Rows / decode with one warp per candidate (small counts).
__global__ void __launch_bounds__(32) row_warp_kernel(const ScanParams p, uint16_t *rows_out,
                                                      int32_t *queue_of, int32_t *pos_of) {
    extern __shared__ __align__(16) uint8_t smem[];
    int64_t first = p.cd.first;
    if (p.cd.first_from) {
        first = p.cd.first_from->index;
        if (first < 0) return;
    }
    const int64_t loc = blockIdx.x;
    const int T = p.dm.T, G = p.dm.G, Q = p.dm.Q;
    uint16_t *srow = reinterpret_cast<uint16_t *>(smem);
    uint16_t *sJ = srow + ((T + 7) & ~7);
    warp_gen_row(p.cd, T, (uint64_t)(first + loc), loc, srow, sJ);
    const int lane = threadIdx.x;
    if (rows_out)
        for (int s = lane; s < T; s += 32) rows_out[loc * T + s] = srow[s];
    if (queue_of || pos_of)
        warp_slots(srow, T, G, Q, [&](int tok, int q, int pos, int) {
            if (queue_of) queue_of[loc * G + tok] = q;
            if (pos_of) pos_of[loc * G + tok] = pos;
        });
}

// Local-search step (R18): adopt the winning NEIGHBOR candidate if its key
// beats the incumbent's.  One block; the base row is rewritten in place.
__global__ void __launch_bounds__(256) adopt_kernel(Dims dm, Cand cd, const qlm_record *rec,
                                                    qlm_record *inc) {
    extern __shared__ __align__(16) uint16_t arow[];
    const qlm_record r = *rec, cur = *inc;
    if (r.index < 0 || r.key >= cur.key) return;                 // uniform: keep the incumbent
    const int T = dm.T;
    for (int s = threadIdx.x; s < T; s += blockDim.x)
        arow[s] = cd.tb == 1 ? (uint16_t)base_token<uint8_t>(cd, s) : (uint16_t)base_token<uint16_t>(cd, s);
    __syncthreads();
    if (threadIdx.x == 0) {
        int mi[QLM_MAX_MOVES], mj[QLM_MAX_MOVES];
        nbr_moves(cd, T, (uint64_t)r.index, mi, mj);
        for (int m = 0; m < cd.moves; ++m) {
            const uint16_t t = arow[mi[m]];
            arow[mi[m]] = arow[mj[m]];
            arow[mj[m]] = t;
        }
    }
    __syncthreads();
    uint8_t *rows = const_cast<uint8_t *>(cd.rows);
    for (int s = threadIdx.x; s < T; s += blockDim.x) {
        if (cd.tb == 1) rows[s] = (uint8_t)arow[s];
        else reinterpret_cast<uint16_t *>(rows)[s] = arow[s];
    }
    if (threadIdx.x == 0) *inc = r;
}

// =============================================================================
// a10-a11: Monte-Carlo
// =============================================================================
// X[k][t] = sum_{r < n_k} len[dist_k][u16(t, k, r) >> (16 - log2 K)]   (R13).
// One block per item (group k, 32 consecutive trials), persistent over items:
// lane = trial, so every lane walks the same n_k requests; the 8 warps split
// the request blocks (warp w takes Philox blocks b = w, w+8, ...; block b holds
// requests 8b..8b+7, two 16-bit halves per word) and reduce through shared
// memory, so a 1000-request group costs the block ~16 blocks per warp instead
// of one warp 127. Tables are staged in shared memory once per block when they
// fit; a lookup is SHF/LOP3 + LEA + LDS. Sums are exact integers, order-free.
template <bool SMEM>
__device__ __forceinline__ uint32_t mc_lookup(const uint16_t *tab, uint32_t tab_s, uint32_t idx) {
    if constexpr (SMEM) {
        uint16_t v;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(tab_s + (idx << 1)));
        return v;
    } else {
        return __ldg(tab + idx);
    }
}

template <bool SMEM>
__device__ __forceinline__ uint32_t mc_block8(const uint16_t *tab, uint32_t tab_s, uint4 wd,
                                              int s, uint32_t km) {
    const uint32_t w[4] = {wd.x, wd.y, wd.z, wd.w};
    uint32_t a = 0;
#pragma unroll
    for (int h = 0; h < 4; ++h)       // (w >> s) & (K-1) == (w & 0xFFFF) >> s since s + log2 K = 16
        a += mc_lookup<SMEM>(tab, tab_s, (w[h] >> s) & km) + mc_lookup<SMEM>(tab, tab_s, w[h] >> (16 + s));
    return a;
}

template <bool SMEM>
__global__ void __launch_bounds__(256) mc_sample_kernel(Dims dm, Tables tb, uint64_t seed,
                                                        int64_t t0, int64_t nt, double *Y) {
    extern __shared__ __align__(16) uint8_t smem[];
    if constexpr (SMEM) {
        uint4 *s4 = reinterpret_cast<uint4 *>(smem);
        const uint4 *g4 = reinterpret_cast<const uint4 *>(tb.len);
        const int n4 = dm.n_tables * dm.K * 2 / 16;
        for (int i = threadIdx.x; i < n4; i += blockDim.x) s4[i] = g4[i];
        __syncthreads();
    }
    __shared__ uint32_t red[8][32];
    const uint32_t smem_s = (uint32_t)__cvta_generic_to_shared(smem);
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const uint32_t ntu = (uint32_t)nt;                   // trials < 2^32 (validated)
    const uint32_t ntw = (ntu + 31) >> 5;                // items per group
    const uint32_t total = (uint32_t)dm.G * ntw;
    const int s = dm.shift - 16;                         // 16 - log2 K
    const uint32_t km = (uint32_t)dm.K - 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t item = blockIdx.x; item < total; item += gridDim.x) {
        const uint32_t k = item / ntw;
        const uint32_t tl = (item - k * ntw) * 32 + lane;
        const uint32_t t = (uint32_t)t0 + tl;
        const int n = tb.grec[k].n;
        const uint32_t toff = (uint32_t)tb.dist[k] * (uint32_t)dm.K;
        const uint16_t *tab = tb.len + toff;
        const uint32_t tab_s = smem_s + 2 * toff;
        const uint32_t nfull = (uint32_t)n >> 3;
        uint32_t sum = 0, sum2 = 0;
        uint32_t b = warp;
        for (; b + 8 < nfull; b += 16) {                 // two independent Philox chains
            const uint4 w0 = philox10(make_uint4(b, k, t, kMcTag), key);
            const uint4 w1 = philox10(make_uint4(b + 8, k, t, kMcTag), key);
            sum += mc_block8<SMEM>(tab, tab_s, w0, s, km);
            sum2 += mc_block8<SMEM>(tab, tab_s, w1, s, km);
        }
        if (b < nfull) {
            sum += mc_block8<SMEM>(tab, tab_s, philox10(make_uint4(b, k, t, kMcTag), key), s, km);
            b += 8;
        }
        const int rem = n & 7;                            // the partial last block (uniform)
        if (rem && b == nfull) {
            const uint4 wd = philox10(make_uint4(b, k, t, kMcTag), key);
            const uint32_t w[4] = {wd.x, wd.y, wd.z, wd.w};
#pragma unroll
            for (int h = 0; h < 7; ++h)
                if (h < rem) sum2 += mc_lookup<SMEM>(tab, tab_s, (h & 1) ? (w[h >> 1] >> (16 + s)) : ((w[h >> 1] >> s) & km));
        }
        red[warp][lane] = sum + sum2;
        __syncthreads();
        // y[d][k][t] = X / Theta[d][m_k]: Eq. 2 with the realised token count, per device row
        if (warp == 0 && tl < ntu) {
            uint32_t x = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) x += red[w][lane];
            const int m = tb.grec[k].model;
            for (int d = 0; d < dm.D; ++d)
                Y[((size_t)d * dm.G + k) * ntu + tl] = __ddiv_rn((double)x, tb.theta[d * dm.M + m]);
        }
        __syncthreads();
    }
}

// One block per (candidate, 32 trials); every lane is one trial, and the
// block's warps split the candidate's queues (queues are independent in Eq.
// 10, so each warp walks whole queues in row order: the oracle's operation
// order).  Warp 0 materialises the row and precomputes per group slot (in
// row order, all trial-independent): the deterministic addend of the walk at
// a model change (tail + swap, R2/R3/R4/R12), the SLO, the start value of the
// queue (backlog mean) and the row of Y to read.  The walk itself is then
// A = start?; A += tail + swap; count A > slo; A += y  -- branch-free
// (+0.0 where no model change: A >= 0, so A + 0.0 == A bit for bit).
constexpr int kMcWarps = 8;
__global__ void __launch_bounds__(32 * kMcWarps) mc_count_kernel(Dims dm, Tables tb, Cand cd,
                                                                 const double *Y, int64_t nt,
                                                                 uint32_t *counts, const int32_t *t_mem,
                                                                 const int32_t *t_cap, const double *t_load) {
    extern __shared__ __align__(16) uint8_t smem[];
    int64_t first = cd.first;
    if (cd.first_from) {
        first = cd.first_from->index;
        if (first < 0) return;
    }
    const int T = dm.T, G = dm.G, M = dm.M, Q = dm.Q;
    double *st = reinterpret_cast<double *>(smem);     // [G] transition addend
    double *sslo = st + G;                              // [G] SLO
    double *sa0 = sslo + G;                             // [G] queue start (backlog mean) or -1
    int32_t *yrow = reinterpret_cast<int32_t *>(sa0 + G);   // [G] d * G + token
    int32_t *qs = yrow + G;                             // [Q + 1] first slot of each queue
    uint16_t *stok = reinterpret_cast<uint16_t *>(qs + ((Q + 1 + 3) & ~3));  // [G]
    uint16_t *sq = stok + G;                            // [G]
    uint16_t *srow = sq + G;                            // [T]
    uint16_t *sJ = srow + ((T + 7) & ~7);               // [T]
    uint8_t *scold = reinterpret_cast<uint8_t *>(sJ + ((T + 7) & ~7));   // [G] two-tier: cold target (R20)
    const int64_t loc = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (warp == 0) {
        warp_gen_row(cd, T, (uint64_t)(first + loc), loc, srow, sJ);
        warp_slots(srow, T, G, Q, [&](int tok, int q, int, int i) {
            stok[i] = (uint16_t)tok;
            sq[i] = (uint16_t)q;
        });
        __syncwarp();
        if (t_mem && lane == 0) {                        // R20 tier state: sequential per queue
            uint32_t seen = 0u, warm = 0u;
            int cum = 0;
            bool exh = false;
            for (int i = 0; i < G; ++i) {
                const int q = sq[i];
                const bool firsts = i == 0 || sq[i - 1] != q;
                if (firsts) { seen = 0u; warm = 0u; cum = 0; exh = false; }
                const int prev = firsts ? tb.qrec[q].r : tb.grec[stok[i - 1]].model;
                const int m = tb.grec[stok[i]].model, d = tb.qrec[q].d;
                bool cold = false;
                if (m != prev) {
                    const uint32_t bit = 1u << m;
                    if (!(seen & bit)) {
                        seen |= bit;
                        if (!exh && cum + t_mem[m] <= t_cap[d]) { warm |= bit; cum += t_mem[m]; }
                        else exh = true;
                    }
                    cold = !(warm & bit);
                }
                scold[i] = cold ? 1 : 0;
            }
        }
        __syncwarp();
        for (int i = lane; i < G; i += 32) {
            const int tok = stok[i], q = sq[i];
            const QRec qr = tb.qrec[q];
            const GRec g = tb.grec[tok];
            const bool firsts = i == 0 || sq[i - 1] != q;
            const int prev = firsts ? qr.r : tb.grec[stok[i - 1]].model;
            const int d = qr.d, m = g.model;
            double c = 0.0;                              // transition term (R2/R3; R20 cold load)
            if (m != prev) {
                const double t = (firsts && !qr.backlog) ? 0.0 : tb.tail[d * M + prev];
                double sw = tb.swap[(d * M + prev) * M + m];
                if (t_mem && scold[i]) sw = __dadd_rn(sw, t_load[d * M + m]);
                c = __dadd_rn(t, sw);
            }
            st[i] = c;
            sslo[i] = g.slo;
            sa0[i] = firsts ? qr.bmean : -1.0;
            yrow[i] = d * G + tok;
        }
        for (int q = lane; q <= Q; q += 32) {            // qs[q] = #slots in queues < q
            int lo = 0, hi = G;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sq[mid] < q) lo = mid + 1; else hi = mid;
            }
            qs[q] = lo;
        }
    }
    __syncthreads();
    const int64_t tl = (int64_t)blockIdx.x * 32 + lane;
    const bool act = tl < nt;
    uint32_t *cnt = counts + loc * G;
    constexpr int PF = 8;
    for (int q = warp; q < Q; q += nw) {
        const int i0 = qs[q], i1 = qs[q + 1];
        double A = 0.0;
        for (int b = i0; b < i1; b += PF) {
            double y[PF];
#pragma unroll
            for (int k = 0; k < PF; ++k) {               // loads first: independent of A
                const int i = b + k < i1 ? b + k : i1 - 1;
                y[k] = act ? __ldg(&Y[(int64_t)yrow[i] * nt + tl]) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < PF; ++k) {
                const int i = b + k;
                if (i >= i1) break;
                const double a0 = sa0[i];
                A = a0 >= 0.0 ? a0 : A;
                A = __dadd_rn(A, st[i]);
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, act && A > sslo[i]);
                if (lane == 0 && bal) atomicAdd(&cnt[stok[i]], (unsigned)__popc(bal));
                A = __dadd_rn(A, y[k]);
            }
        }
    }
}

// =============================================================================
// launchers
// =============================================================================
// Per-device caches: a process may hold contexts on several ordinals, and the
// SM count and the dynamic shared-memory opt-in are properties of a device.
int sm_count() {
    static std::mutex mu;
    static std::unordered_map<int, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n;
    return n;
}

// Environment overrides (tests and tuning only) are read once per process.
int env_cached(const char *name, int dflt) {
    static std::mutex mu;
    static std::unordered_map<std::string, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    const std::string key = std::string(name) + "#" + std::to_string(dflt);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    const char *v = getenv(name);
    const int r = v && *v ? atoi(v) : dflt;
    cache[key] = r;
    return r;
}

int log_level() {
    static const int lvl = env_cached("QLM_LOG", 0);
    return lvl;
}

void qlog(int level, const char *fmt, ...) {
    if (log_level() < level) return;
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    fprintf(stderr, "[qlm] %s\n", buf);
}

static size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

static int env_int(const char *name, int dflt) { return env_cached(name, dflt); }

static const size_t kMaxSmem = 227 * 1024;

// Largest dynamic shared memory a launch of `kern` may use (opt-in limit
// minus the kernel's static shared memory); opts the kernel into it once.
template <typename K>
static size_t max_dyn(K kern) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, size_t> cache;   // (kernel, device)
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(reinterpret_cast<const void *>(kern), dev);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) { cudaGetLastError(); return 0; }
    size_t m = optin > (int)fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
    if (m > kMaxSmem) m = kMaxSmem;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cache[key] = m;
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

// Shared-memory plan of the scan kernel for a block of `blk` threads.
static size_t plan_smem(ScanParams &p, int rep_shift, int kind, int tok_bytes, int blk, int out) {
    const Dims &dm = p.dm;
    size_t off = 0;
    p.rep_shift = rep_shift;
    p.off_grec = (int)off; off = align16(off + ((size_t)dm.G << rep_shift) * sizeof(GRec));
    p.off_ab = (int)off;   off = align16(off + ((size_t)dm.D * dm.G << rep_shift) * sizeof(double2));
    p.off_q = (int)off;    off = align16(off + (size_t)dm.Q * sizeof(QRec));
    // transition entries (8 B) may be replicated (QLM_TR_SHIFT) for conflict-free 64-bit loads
    p.tr_shift = env_int("QLM_TR_SHIFT", 0);   // measured: no gain in the thread-per-candidate scan
    p.off_tr = (int)off;   off = align16(off + ((size_t)dm.D * 2 * dm.M * dm.M << p.tr_shift) * sizeof(double));
    p.off_scratch = (int)off;
    if (kind == QLM_CAND_RANDOM) {
        const int epw = 4 / tok_bytes;
        off = align16(off + (size_t)((dm.T + epw - 1) / epw) * 4 * blk);
    }
    p.off_stage = (int)off;
    if (out == OUT_STAGED) off = align16(off + (size_t)3 * blk * dm.G * 4);
    return off;
}

static int default_rep_shift(const Dims &dm) {
    const size_t rec = (size_t)dm.G * (1 + dm.D) * 16;
    return rec * 8 <= 24 * 1024 ? 3 : 0;
}

template <int KIND, typename TOK, int OUT, bool SCORE>
static cudaError_t launch_scan_t(ScanParams p, cudaStream_t st) {
    auto kern = scan_kernel<KIND, TOK, OUT, SCORE>;
    const size_t lim = max_dyn(kern);
    if (!lim) return cudaErrorInvalidConfiguration;
    // choose (block size, replication) maximising resident candidates per SM;
    // QLM_BLK / QLM_REP_SHIFT override (tuning sweeps)
    int best_blk = 0, best_rs = 0, best_thr = 0;
    size_t best_smem = 0;
    const int rs0 = default_rep_shift(p.dm);
    const int env_blk = env_int("QLM_BLK", 0), env_rs = env_int("QLM_REP_SHIFT", -1);
    const int blks[] = {128, 96, 64, 32};
    for (int rs : {rs0, rs0 > 2 ? 2 : 0, 0}) {
        if (env_rs >= 0 && rs != env_rs) continue;
        for (int blk : blks) {
            if (env_blk && blk != env_blk) continue;
            ScanParams q = p;
            const size_t smem = plan_smem(q, rs, KIND, sizeof(TOK), blk, OUT);
            if (smem > lim) continue;
            const int thr = occupancy(kern, blk, smem) * blk;
            if (thr > best_thr) { best_thr = thr; best_blk = blk; best_rs = rs; best_smem = smem; }
        }
        if (best_thr >= 192 || (OUT != OUT_STAGED && best_thr)) break;
    }
    if (!best_blk) return cudaErrorInvalidConfiguration;
    p.blk = best_blk;
    plan_smem(p, best_rs, KIND, sizeof(TOK), best_blk, OUT);
    int64_t grid = (p.cd.count + best_blk - 1) / best_blk;
    const int64_t maxg = (int64_t)sm_count() * (best_thr / best_blk);
    if (grid > maxg) grid = maxg;
    if (grid > p.max_blocks) grid = p.max_blocks;
    if (grid < 1) grid = 1;
    qlog(1, "scan_kernel<kind=%d,tok=%zu,out=%d,score=%d> count=%lld grid=%lld block=%d smem=%zu",
         KIND, sizeof(TOK), OUT, (int)SCORE, (long long)p.cd.count, (long long)grid, best_blk, best_smem);
    kern<<<(unsigned)grid, best_blk, best_smem, st>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

template <int KIND, typename TOK>
static cudaError_t launch_scan_k(ScanParams &p, cudaStream_t st) {
    const bool score = p.s1 || p.s2 || p.n_over || p.out_rec;
    p.n_out = (p.wt != nullptr) + (p.sd != nullptr) + (p.vo != nullptr);
    if (p.n_out == 0) return launch_scan_t<KIND, TOK, OUT_NONE, true>(p, st);
    // staged (group-major smem tile + bulk copies) when one fits, else direct stores
    const size_t stage_bytes = (size_t)3 * 32 * p.dm.G * 4;
    const bool fits = stage_bytes + 64 * 1024 <= kMaxSmem;
    p.use_tma = ((p.ld_out ? p.ld_out : p.cd.count) % 4 == 0) && (!p.wt || ((uintptr_t)p.wt & 15) == 0) &&
                (!p.sd || ((uintptr_t)p.sd & 15) == 0) && (!p.vo || ((uintptr_t)p.vo & 15) == 0);
    if (fits) {
        cudaError_t e = score ? launch_scan_t<KIND, TOK, OUT_STAGED, true>(p, st)
                              : launch_scan_t<KIND, TOK, OUT_STAGED, false>(p, st);
        if (e != cudaErrorInvalidConfiguration) return e;
        cudaGetLastError();
    }
    return score ? launch_scan_t<KIND, TOK, OUT_DIRECT, true>(p, st)
                 : launch_scan_t<KIND, TOK, OUT_DIRECT, false>(p, st);
}

// The warp-per-candidate kernel (qlm_wide.cu) takes bulk outputs whose
// [G][32] staging tile does not fit (G > ~420): thread-per-candidate direct
// stores would scatter 4-B writes across partial sectors.
static bool wide_first(const ScanParams &p) {
    const bool bulk = p.wt || p.sd || p.vo;
    if (env_int("QLM_WIDE_SCORE", 0)) return true;         // experiments: score-only too
    const size_t stage_bytes = (size_t)3 * 32 * p.dm.G * 4;
    return bulk && stage_bytes + 64 * 1024 > kMaxSmem;
}

// Large-T RANDOM (T > 256, outside the warp-specialised kernel's range): the
// per-thread Fisher-Yates scratch (2T bytes) would cap the fused scan at a few
// warps per SM, so rows are generated per chunk into an interleaved scratch by
// fy_rows_kernel (cheap, latency-bound) and scored by the scan kernel reading
// them with coalesced loads at full occupancy.  Argmin is carried across
// chunks in chunk_recs[0].
cudaError_t launch_fy_rows(const Cand &g, int T, uint32_t *out, int64_t n, cudaStream_t st) {
    const size_t fy_smem = (size_t)T * 32 * 2;
    cudaError_t e = prep(fy_rows_kernel, fy_smem);
    if (e != cudaSuccess) return e;
    qlog(1, "fy_rows_kernel T=%d rows=%lld", T, (long long)n);
    fy_rows_kernel<<<(unsigned)((n + 31) / 32), 32, fy_smem, st>>>(g, T, out, n);
    ++g_launches;
    return cudaGetLastError();
}

static cudaError_t launch_two_phase(const ScanParams &p0, cudaStream_t st) {
    const int64_t count = p0.cd.count, cap = p0.ilv_cap;
    cudaError_t e;
    for (int64_t c0 = 0; c0 < count; c0 += cap) {
        const int64_t n = count - c0 < cap ? count - c0 : cap;
        Cand g = p0.cd;
        g.first = p0.cd.first + c0;
        g.count = n;
        if ((e = launch_fy_rows(g, p0.dm.T, p0.ilv, n, st)) != cudaSuccess) return e;
        ScanParams p = p0;
        p.cd.kind = KIND_ILV;
        p.cd.tb = 2;
        p.cd.rows = reinterpret_cast<const uint8_t *>(p0.ilv);
        p.cd.stride = n;
        p.cd.first = g.first;
        p.cd.count = n;
        p.ld_out = count;
        if (p.s1) p.s1 += c0;
        if (p.s2) p.s2 += c0;
        if (p.n_over) p.n_over += c0;
        if (p.wt) p.wt += c0;
        if (p.sd) p.sd += c0;
        if (p.vo) p.vo += c0;
        if (p0.out_rec) p.out_rec = p0.chunk_recs + (c0 ? 1 : 0);
        e = wide_first(p) ? launch_wide(p, st) : launch_large(p, st);
        if (e == cudaErrorNotSupported) {
            cudaGetLastError();
            e = launch_scan_k<KIND_ILV, uint16_t>(p, st);
        }
        if (e != cudaSuccess) return e;
        if (p0.out_rec && c0) {
            reduce_records_kernel<<<1, 64, 0, st>>>(p0.chunk_recs, 2, p0.chunk_recs);
            ++g_launches;
        }
    }
    if (p0.out_rec) {
        reduce_records_kernel<<<1, 32, 0, st>>>(p0.chunk_recs, 1, p0.out_rec);
        ++g_launches;
    }
    return cudaGetLastError();
}

cudaError_t launch_any_scan(const ScanParams &p, cudaStream_t st) {
    cudaError_t e = launch_ws(p, st);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
    if ((p.cd.kind == QLM_CAND_EXPLICIT || p.cd.kind == QLM_CAND_NEIGHBOR) && p.cd.tb == 2 &&
        wide_first(p)) {
        e = launch_wide(p, st);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    if (p.cd.kind == QLM_CAND_RANDOM && p.dm.T > 256 && p.ilv && p.ilv_cap >= 32 &&
        p.chunk_recs && !p.cd.first_from && p.cd.count >= 4096) {
        e = launch_two_phase(p, st);
    } else {
        e = launch_scan(p, st);
    }
    if (e == cudaErrorInvalidValue || e == cudaErrorInvalidConfiguration || e == cudaErrorNotSupported) {
        // no shared-memory plan of the scan kernels fits (very large G): the
        // warp-per-candidate path with global tables rewrites every output
        cudaGetLastError();
        return launch_big(p, st);
    }
    return e;
}

cudaError_t launch_scan(ScanParams p, cudaStream_t st) {
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM:
        return p.dm.T <= 256 ? launch_scan_k<QLM_CAND_RANDOM, uint8_t>(p, st)
                             : launch_scan_k<QLM_CAND_RANDOM, uint16_t>(p, st);
    case QLM_CAND_EXPLICIT:
        return p.cd.tb == 1 ? launch_scan_k<QLM_CAND_EXPLICIT, uint8_t>(p, st)
                            : launch_scan_k<QLM_CAND_EXPLICIT, uint16_t>(p, st);
    case QLM_CAND_NEIGHBOR:
        return p.cd.tb == 1 ? launch_scan_k<QLM_CAND_NEIGHBOR, uint8_t>(p, st)
                            : launch_scan_k<QLM_CAND_NEIGHBOR, uint16_t>(p, st);
    default:
        return launch_scan_k<QLM_CAND_ENUM, uint8_t>(p, st);
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
    if (p.cd.count <= 1024) {
        const size_t smem = (size_t)4 * ((p.dm.T + 7) & ~7);
        cudaError_t e = prep(row_warp_kernel, smem);
        if (e != cudaSuccess) return e;
        row_warp_kernel<<<(unsigned)p.cd.count, 32, smem, st>>>(p, rows, qo, po);
        ++g_launches;
        return cudaGetLastError();
    }
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM:
        return p.dm.T <= 256 ? launch_rows_t<QLM_CAND_RANDOM, uint8_t>(p, rows, qo, po, st)
                             : launch_rows_t<QLM_CAND_RANDOM, uint16_t>(p, rows, qo, po, st);
    case QLM_CAND_EXPLICIT:
        return p.cd.tb == 1 ? launch_rows_t<QLM_CAND_EXPLICIT, uint8_t>(p, rows, qo, po, st)
                            : launch_rows_t<QLM_CAND_EXPLICIT, uint16_t>(p, rows, qo, po, st);
    case QLM_CAND_NEIGHBOR:
        return p.cd.tb == 1 ? launch_rows_t<QLM_CAND_NEIGHBOR, uint8_t>(p, rows, qo, po, st)
                            : launch_rows_t<QLM_CAND_NEIGHBOR, uint16_t>(p, rows, qo, po, st);
    default:
        return launch_rows_t<QLM_CAND_ENUM, uint8_t>(p, rows, qo, po, st);
    }
}

cudaError_t launch_adopt(const Dims &dm, const Cand &cd, const qlm_record *rec, qlm_record *inc,
                         cudaStream_t st) {
    const size_t smem = (size_t)((dm.T + 7) & ~7) * 2;
    cudaError_t e = prep(adopt_kernel, smem);
    if (e != cudaSuccess) return e;
    adopt_kernel<<<1, 256, smem, st>>>(dm, cd, rec, inc);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_reduce_records(const qlm_record *recs, int n, qlm_record *out,
                                  cudaStream_t st) {
    reduce_records_kernel<<<1, 256, 0, st>>>(recs, n, out);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_check_rows(const Cand &cd, int T, unsigned long long *n_bad, cudaStream_t st) {
    if (cd.count <= 0) return cudaSuccess;
    if (cd.count > INT32_MAX) return cudaErrorInvalidValue;        // one block per row
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
                             int64_t nt, double *X, cudaStream_t st) {
    const size_t tab_bytes = (size_t)dm.n_tables * dm.K * 2;
    const bool in_smem = tab_bytes <= 100 * 1024 && (tab_bytes % 16) == 0;
    const size_t smem = in_smem ? tab_bytes : 0;
    auto kern = in_smem ? mc_sample_kernel<true> : mc_sample_kernel<false>;
    cudaError_t e = prep(kern, smem);
    if (e != cudaSuccess) return e;
    const int nb = occupancy(kern, 256, smem);
    const int64_t items = (int64_t)dm.G * ((nt + 31) / 32);   // one block each
    int64_t grid = items;
    const int64_t maxg = (int64_t)sm_count() * (nb > 0 ? nb : 1);
    if (grid > maxg) grid = maxg;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 256, smem, st>>>(dm, tb, seed, t0, nt, X);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_mc_count(const Dims &dm, const Tables &tb, const Cand &cd, const double *X,
                            int64_t nt, uint32_t *counts, cudaStream_t st, const int32_t *t_mem,
                            const int32_t *t_cap, const double *t_load) {
    const size_t smem = (size_t)32 * dm.G + (size_t)4 * ((dm.Q + 1 + 3) & ~3) +
                        (size_t)4 * ((dm.T + 7) & ~7) + (size_t)((dm.G + 15) & ~15);
    cudaError_t e = prep(mc_count_kernel, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((nt + 31) / 32), (unsigned)cd.count);
    const int warps = dm.Q < kMcWarps ? dm.Q : kMcWarps;   // warps split the queues
    mc_count_kernel<<<grid, 32 * warps, smem, st>>>(dm, tb, cd, X, nt, counts, t_mem, t_cap, t_load);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace qlm
