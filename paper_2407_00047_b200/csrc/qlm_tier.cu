// qlm_tier.cu -- two-tier (warm / cold) model swapping in the Eq. 10 scan
// (DESIGN R20).
//
// Models later in a virtual queue are warm in the instance's CPU memory
// until it is exhausted; the rest are cold in the registry and pay a
// storage -> CPU load before their CPU -> GPU swap.  Per queue, the swap
// targets in order of their first transition take CPU memory while it lasts
// (strict prefix); a model keeps its tier for every later transition into it.
//
// One thread per candidate, like the general scan kernel: the row streams
// through the candidate generators of qlm_device.cuh, the thread walks it
// once, carrying the queue's tier state in four registers (seen / warm model
// bit masks, CPU memory taken, exhausted flag).  Each transition adds ONE
// precomputed fp64 term -- tail + swap (warm) or tail + (swap + load)
// (cold) -- in the oracle's operation order, so wt / V are bit-identical to
// or_estimate_row_tiered; with every target warm the kernel reproduces the
// untiered scan kernel bit for bit (same S1 accumulators, same order).
// Bulk outputs are staged per block ([3][G][blk] fp32) and leave as
// coalesced 128-B warp stores, or go straight to HBM when no tile fits.
#include <cuda_runtime.h>

#include <cstdlib>

#include "qlm_device.cuh"
#include "qlm_launch.h"
#include "qlm_argmin.cuh"

namespace qlm {

struct TierSmem {
    int off_g, off_ab, off_q, off_trw, off_trc, off_mem, off_cap, off_scratch, off_stage;
    int blk, stage;
};

template <int KIND, typename TOK, typename F>
__device__ __forceinline__ void tier_tokens(const Cand &cd, int T, uint8_t *scratch, int blk,
                                            int64_t loc, int64_t c, F &&f) {
    if constexpr (KIND == QLM_CAND_RANDOM) {
        fy_materialise<TOK>(scratch, blk, threadIdx.x, T, cd.seed, (uint64_t)c);
        tokens_scratch<TOK>(scratch, blk, threadIdx.x, T, f);
    } else if constexpr (KIND == QLM_CAND_EXPLICIT) {
        tokens_explicit<TOK>(cd.rows + loc * cd.stride, T, f);
    } else if constexpr (KIND == QLM_CAND_NEIGHBOR) {
        tokens_neighbor<TOK>(cd, T, (uint64_t)c, f);
    } else {
        tokens_enum((uint64_t)c, T, f);
    }
}

template <int KIND, typename TOK>
__global__ void __launch_bounds__(128) tier_kernel(const ScanParams p, const TierSmem L) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, blk = blockDim.x;
    const Dims dm = p.dm;
    const int G = dm.G, Q = dm.Q, T = dm.T, M = dm.M, D = dm.D;

    // ---- tables -> shared memory ----
    GRec *sg = reinterpret_cast<GRec *>(smem + L.off_g);
    for (int i = tid; i < G; i += blk) sg[i] = p.tb.grec[i];
    double2 *sab = reinterpret_cast<double2 *>(smem + L.off_ab);
    for (int i = tid; i < D * G; i += blk) sab[i] = p.tb.ab[i];
    QRec *sq = reinterpret_cast<QRec *>(smem + L.off_q);
    for (int i = tid; i < Q; i += blk) sq[i] = p.tb.qrec[i];
    // transition terms, rows p' < M: previous model p'; p' >= M: nothing ran
    // yet on resident p' - M (R4).  warm: tail + swap; cold: tail + (swap + load)
    double *trw = reinterpret_cast<double *>(smem + L.off_trw);
    double *trc = reinterpret_cast<double *>(smem + L.off_trc);
    for (int i = tid; i < D * 2 * M * M; i += blk) {
        const int m = i % M, pp = (i / M) % (2 * M), d = i / (2 * M * M);
        const int from = pp < M ? pp : pp - M;
        const double sw = p.tb.swap[(d * M + from) * M + m];
        const double tl = (pp < M && m != pp) ? p.tb.tail[d * M + pp] : 0.0;
        const double ld = m != from ? p.t_load[d * M + m] : 0.0;
        trw[i] = __dadd_rn(tl, sw);
        trc[i] = __dadd_rn(tl, __dadd_rn(sw, ld));
    }
    int *smem_m = reinterpret_cast<int *>(smem + L.off_mem);
    for (int i = tid; i < M; i += blk) smem_m[i] = p.t_mem[i];
    int *scap = reinterpret_cast<int *>(smem + L.off_cap);
    for (int i = tid; i < D; i += blk) scap[i] = p.t_cap[i];
    uint8_t *scratch = smem + L.off_scratch;
    __syncthreads();

    const Cand cd = p.cd;
    int64_t first = cd.first;
    bool none = false;
    if (cd.first_from) {
        first = cd.first_from->index;
        none = first < 0;
    }
    const float zc = p.zc;
    const float alpha = p.alpha;
    const int64_t count = none ? 0 : cd.count;
    float *const gout[3] = {p.wt, p.sd, p.vo};
    float *st[3] = {nullptr, nullptr, nullptr};
    if (L.stage) {
        st[0] = reinterpret_cast<float *>(smem + L.off_stage);
        st[1] = st[0] + (size_t)G * blk;
        st[2] = st[1] + (size_t)G * blk;
    }
    const bool bulk = p.wt || p.sd || p.vo;
    const double den = *p.tb.den;
    uint64_t bkey = ~0ull;
    int64_t bidx = -1;
    const int64_t ntiles = (count + blk - 1) / blk;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t c0 = tile * blk, loc = c0 + tid;
        const int nvalid = (int)min((int64_t)blk, count - c0);
        if (tid < nvalid) {
            // queue state (R4/R12) and tier state (R20)
            int q = 0, d = sq[0].d, prow = sq[0].backlog ? sq[0].r : M + sq[0].r;
            double A = sq[0].bmean, S2 = 0.0, acc2 = 0.0;
            float B = (float)sq[0].bvar;                      // fp32 (R22)
            uint32_t seen = 0u, warm = 0u;
            int cum = 0;
            bool exh = false;
            float acc1 = 0.0f;
            int over = 0;
            tier_tokens<KIND, TOK>(cd, T, scratch, blk, loc, first + loc, [&](int tok) {
                if (tok >= G) {                              // separator: next queue, fresh CPU memory
                    q = q + 1 < Q ? q + 1 : Q - 1;
                    const QRec r = sq[q];
                    d = r.d; prow = r.backlog ? r.r : M + r.r;
                    A = r.bmean; B = (float)r.bvar;
                    seen = 0u; warm = 0u; cum = 0; exh = false;
                    return;
                }
                const GRec g = sg[tok];
                const int m = g.model;
                const int pm = prow < M ? prow : prow - M;
                bool cold = false;
                if (m != pm) {                               // a transition (Eq. 9)
                    const uint32_t bit = 1u << m;
                    if (!(seen & bit)) {                     // first transition into m
                        seen |= bit;
                        if (!exh && cum + smem_m[m] <= scap[d]) { warm |= bit; cum += smem_m[m]; }
                        else exh = true;
                    }
                    cold = !(warm & bit);
                }
                const int ti = (d * 2 * M + prow) * M + m;
                A = __dadd_rn(A, cold ? trc[ti] : trw[ti]);
                const double wt = A;                         // exclusive (R5)
                const float V = B;
                const double2 ab = sab[d * G + tok];
                A = __dadd_rn(A, ab.x);
                B = __fadd_rn(B, (float)ab.y);
                prow = m;
                const double slack = __dsub_rn(g.slo, wt);
                const float sd = slot_sd(V);
                bool clamped;
                const float v = slot_v(slack, sd, zc, clamped);
                S2 = __dsub_rn(S2, slack);
                if (clamped) acc1 = fmaf((float)g.n, v, acc1);
                else acc2 = __fma_rn((double)g.n, (double)v, acc2);
                over += v > alpha;
                if (bulk) {
                    const float o3[3] = {(float)wt, sd, v};
                    if (L.stage) {
#pragma unroll
                        for (int a = 0; a < 3; ++a) st[a][tok * blk + tid] = o3[a];
                    } else {
#pragma unroll
                        for (int a = 0; a < 3; ++a)
                            if (gout[a]) gout[a][(int64_t)tok * count + loc] = o3[a];
                    }
                }
            });
            const float s1 = (float)(((double)acc1 + acc2) / den);   // R11
            const float s2 = (float)S2;
            if (p.s1) p.s1[loc] = s1;
            if (p.s2) p.s2[loc] = s2;
            if (p.n_over) p.n_over[loc] = over;
            const uint64_t key = make_key(s1, s2);
            if (better(key, first + loc, bkey, bidx)) { bkey = key; bidx = first + loc; }
        }
        if (bulk && L.stage) {                               // coalesced copy-out of the tile
            __syncthreads();
            if (tid < nvalid)
                for (int a = 0; a < 3; ++a)
                    if (gout[a])
                        for (int g = 0; g < G; ++g) gout[a][(int64_t)g * count + loc] = st[a][g * blk + tid];
            __syncthreads();
        }
    }
    if (p.out_rec) {
        if (none) {
            if (blockIdx.x == 0 && tid == 0) { p.out_rec->key = ~0ull; p.out_rec->index = -1; }
            return;
        }
        block_grid_argmin(p, bkey, bidx);
    }
}

template <int KIND, typename TOK>
static cudaError_t launch_tier_t(const ScanParams &p, cudaStream_t st) {
    auto kern = tier_kernel<KIND, TOK>;
    const Dims &dm = p.dm;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const bool bulk = p.wt || p.sd || p.vo;
    auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };
    TierSmem L{};
    size_t total = 0;
    for (int blk = 128; blk >= 32; blk >>= 1) {
        for (int stage = bulk ? 1 : 0; stage >= 0; --stage) {
            size_t o = 0;
            L.off_g = (int)o;   o = a16(o + (size_t)dm.G * sizeof(GRec));
            L.off_ab = (int)o;  o = a16(o + (size_t)dm.D * dm.G * sizeof(double2));
            L.off_q = (int)o;   o = a16(o + (size_t)dm.Q * sizeof(QRec));
            L.off_trw = (int)o; o = a16(o + (size_t)dm.D * 2 * dm.M * dm.M * 8);
            L.off_trc = (int)o; o = a16(o + (size_t)dm.D * 2 * dm.M * dm.M * 8);
            L.off_mem = (int)o; o = a16(o + (size_t)dm.M * 4);
            L.off_cap = (int)o; o = a16(o + (size_t)dm.D * 4);
            L.off_scratch = (int)o;
            if (KIND == QLM_CAND_RANDOM) o = a16(o + (size_t)((dm.T * sizeof(TOK) + 3) / 4) * 4 * blk);
            L.off_stage = (int)o;
            if (stage) o += (size_t)3 * dm.G * blk * 4;
            L.blk = blk;
            L.stage = stage;
            total = o;
            if (o <= (size_t)optin && (!stage || o <= 110 * 1024)) break;
            total = 0;
        }
        if (total) break;
    }
    if (!total) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)total);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L.blk, total);
    if (per_sm < 1) per_sm = 1;
    const int64_t ntiles = (p.cd.count + L.blk - 1) / L.blk;
    int64_t grid = (int64_t)sm_count() * per_sm;
    if (grid > ntiles) grid = ntiles;
    if (grid > p.max_blocks) grid = p.max_blocks;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, L.blk, total, st>>>(p, L);
    ++g_launches;
    return cudaGetLastError();
}

// ---- large G: one warp per candidate, one lane per queue -------------------
// The tier state (R20) is per queue, so a lane that walks one whole queue in
// row order carries it exactly (and in the oracle's operation order).  Eight
// warps score eight consecutive candidates; their bulk outputs are staged in
// a [3][G][9] tile and leave as full 32-B rows of the group-major arrays.
constexpr int kTwWarps = 8;
constexpr int kTwPad = kTwWarps + 1;
constexpr int kTwPf = 24;           // prefetched row words per lane (interleaved rows, T <= 1536)

struct TierWarpSmem {
    int off_g, off_ab, off_q, off_trw, off_trc, off_mem, off_cap, off_tile, off_rows, off_qbeg;
    int ldr;
};

__global__ void __launch_bounds__(256, 1) tier_warp_kernel(const ScanParams p, const TierWarpSmem L) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Dims dm = p.dm;
    const int G = dm.G, Q = dm.Q, T = dm.T, M = dm.M, D = dm.D;
    GRec *sg = reinterpret_cast<GRec *>(smem + L.off_g);
    for (int i = tid; i < G; i += 256) sg[i] = p.tb.grec[i];
    double2 *sab = reinterpret_cast<double2 *>(smem + L.off_ab);
    for (int i = tid; i < D * G; i += 256) sab[i] = p.tb.ab[i];
    QRec *sq = reinterpret_cast<QRec *>(smem + L.off_q);
    for (int i = tid; i < Q; i += 256) sq[i] = p.tb.qrec[i];
    double *trw = reinterpret_cast<double *>(smem + L.off_trw);
    double *trc = reinterpret_cast<double *>(smem + L.off_trc);
    for (int i = tid; i < D * 2 * M * M; i += 256) {
        const int m = i % M, pp = (i / M) % (2 * M), d = i / (2 * M * M);
        const int from = pp < M ? pp : pp - M;
        const double sw = p.tb.swap[(d * M + from) * M + m];
        const double tl = (pp < M && m != pp) ? p.tb.tail[d * M + pp] : 0.0;
        const double ld = m != from ? p.t_load[d * M + m] : 0.0;
        trw[i] = __dadd_rn(tl, sw);
        trc[i] = __dadd_rn(tl, __dadd_rn(sw, ld));
    }
    int *smemsz = reinterpret_cast<int *>(smem + L.off_mem);
    for (int i = tid; i < M; i += 256) smemsz[i] = p.t_mem[i];
    int *scap = reinterpret_cast<int *>(smem + L.off_cap);
    for (int i = tid; i < D; i += 256) scap[i] = p.t_cap[i];
    float *tile = reinterpret_cast<float *>(smem + L.off_tile);          // [3][G][kTwPad]
    uint16_t *srow = reinterpret_cast<uint16_t *>(smem + L.off_rows) + (size_t)warp * 2 * L.ldr;
    uint16_t *sJ = srow + L.ldr;
    int *qbeg = reinterpret_cast<int *>(smem + L.off_qbeg) + (size_t)warp * (Q + 1);
    __syncthreads();

    const Cand cd = p.cd;
    int64_t first = cd.first;
    bool none = false;
    if (cd.first_from) {
        first = cd.first_from->index;
        none = first < 0;
    }
    const int64_t count = none ? 0 : cd.count;
    const float zc = p.zc;
    const float alpha = p.alpha;
    const double den = *p.tb.den;
    float *const gout[3] = {p.wt, p.sd, p.vo};
    const int64_t ldo = p.ld_out ? p.ld_out : count;           // chunked launches write into the full range
    const bool bulk = p.wt || p.sd || p.vo;
    uint64_t bkey = ~0ull;
    int64_t bidx = -1;
    const int64_t nbatch = (count + kTwWarps - 1) / kTwWarps;
    // interleaved rows (two-phase): the warp's next row is loaded into
    // registers (kTwPf words per lane) before the current one is walked, so
    // the strided global loads overlap the walk
    const int nw = (T + 1) >> 1;
    const bool pf = cd.kind == KIND_ILV && nw <= 32 * kTwPf;
    const uint32_t *r32 = reinterpret_cast<const uint32_t *>(cd.rows);
    uint32_t pfv[kTwPf];
    auto pf_load = [&](int64_t l) {
#pragma unroll
        for (int u = 0; u < kTwPf; ++u) {
            const int w = lane + 32 * u;
            pfv[u] = (w < nw && l < count) ? __ldg(r32 + (size_t)w * cd.stride + l) : 0u;
        }
    };
    if (pf) pf_load((int64_t)blockIdx.x * kTwWarps + warp);
    for (int64_t bt = blockIdx.x; bt < nbatch; bt += gridDim.x) {
        const int64_t c0 = bt * kTwWarps, loc = c0 + warp;
        if (pf) {
            uint32_t *s32 = reinterpret_cast<uint32_t *>(srow);   // srow is 4-B aligned (ldr even)
#pragma unroll
            for (int u = 0; u < kTwPf; ++u) {
                const int w = lane + 32 * u;
                if (w < nw) s32[w] = pfv[u];
            }
            __syncwarp();
            pf_load((bt + gridDim.x) * kTwWarps + warp);
        }
        if (loc < count) {                                    // warp-uniform
            if (!pf) warp_gen_row(cd, T, (uint64_t)(first + loc), loc, srow, sJ);
            // queue q covers row positions [qbeg[q], qbeg[q + 1] - 1)
            if (lane == 0) qbeg[0] = 0;
            int nsep = 0;
            for (int s0 = 0; s0 < T; s0 += 32) {
                const int s = s0 + lane;
                const bool sep = s < T && srow[s] >= G;
                const uint32_t bs = __ballot_sync(0xFFFFFFFFu, sep);
                if (sep) {
                    const int k = nsep + __popc(bs & ((1u << lane) - 1u));
                    if (k + 1 <= Q - 1) qbeg[k + 1] = s + 1;
                }
                nsep += __popc(bs);
            }
            if (lane == 0) qbeg[Q] = T + 1;
            __syncwarp();
            double S2 = 0.0, num = 0.0;
            int over = 0;
            for (int q = lane; q < Q; q += 32) {
                const QRec r = sq[q];
                const int d = r.d;
                int prow = r.backlog ? r.r : M + r.r;         // R4 / R12
                double A = r.bmean;
                float B = (float)r.bvar;                      // fp32 (R22)
                uint32_t seen = 0u, warm = 0u;
                int cum = 0;
                bool exh = false;
                const int s1 = qbeg[q + 1] - 1;
                for (int s = qbeg[q]; s < s1; ++s) {
                    const int tok = srow[s];
                    const GRec g = sg[tok];
                    const int m = g.model;
                    const int pm = prow < M ? prow : prow - M;
                    bool cold = false;
                    if (m != pm) {                            // transition (Eq. 9), tier (R20)
                        const uint32_t bit = 1u << m;
                        if (!(seen & bit)) {
                            seen |= bit;
                            if (!exh && cum + smemsz[m] <= scap[d]) { warm |= bit; cum += smemsz[m]; }
                            else exh = true;
                        }
                        cold = !(warm & bit);
                    }
                    const int ti = (d * 2 * M + prow) * M + m;
                    A = __dadd_rn(A, cold ? trc[ti] : trw[ti]);
                    const double wt = A;
                    const float V = B;
                    const double2 ab = sab[d * G + tok];
                    A = __dadd_rn(A, ab.x);
                    B = __fadd_rn(B, (float)ab.y);
                    prow = m;
                    const double slack = __dsub_rn(g.slo, wt);
                    const float sd = slot_sd(V);
                    bool clamped;
                    const float v = slot_v(slack, sd, zc, clamped);
                    S2 = __dsub_rn(S2, slack);
                    num = __dadd_rn(num, (double)g.n * (double)v);
                    over += v > alpha;
                    if (bulk) {
                        float *o = tile + (size_t)tok * kTwPad + warp;
                        o[0] = (float)wt;
                        o[(size_t)G * kTwPad] = sd;
                        o[(size_t)2 * G * kTwPad] = v;
                    }
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                S2 += __shfl_xor_sync(0xFFFFFFFFu, S2, o);
                num += __shfl_xor_sync(0xFFFFFFFFu, num, o);
                over += __shfl_xor_sync(0xFFFFFFFFu, over, o);
            }
            const float s1v = (float)(num / den), s2v = (float)S2;   // R11
            if (lane == 0) {
                if (p.s1) p.s1[loc] = s1v;
                if (p.s2) p.s2[loc] = s2v;
                if (p.n_over) p.n_over[loc] = over;
            }
            const uint64_t key = make_key(s1v, s2v);
            if (lane == 0 && better(key, first + loc, bkey, bidx)) { bkey = key; bidx = first + loc; }
        }
        if (bulk) {                                           // full 32-B rows of the outputs
            __syncthreads();
            const int nv = (int)min((int64_t)kTwWarps, count - c0);
            // 8 consecutive lanes write one row's 8 floats: each store instruction
            // covers 4 whole 32-B sectors (no partial-sector writes); thread t
            // takes column t mod 8 of rows t/8, t/8 + 32, ... (no divisions)
            const int k = tid & 7;
            if (k < nv) {
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    float *const base = gout[a];
                    if (!base) continue;
                    float *dst = base + c0 + k + (int64_t)(tid >> 3) * ldo;
                    const float *src = tile + (size_t)a * G * kTwPad + k + (tid >> 3) * kTwPad;
                    const int64_t dstep = 32 * ldo;
                    for (int g = tid >> 3; g < G; g += 32, dst += dstep, src += 32 * kTwPad) __stcs(dst, *src);
                }
            }
            __syncthreads();
        }
    }
    if (p.out_rec) {
        if (none) {
            if (blockIdx.x == 0 && tid == 0) { p.out_rec->key = ~0ull; p.out_rec->index = -1; }
            return;
        }
        block_grid_argmin(p, bkey, bidx);
    }
}

static cudaError_t launch_tier_warp(const ScanParams &p, cudaStream_t st) {
    const Dims &dm = p.dm;
    auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };
    TierWarpSmem L{};
    L.ldr = (dm.T + 7) & ~7;
    size_t o = 0;
    L.off_g = (int)o;    o = a16(o + (size_t)dm.G * sizeof(GRec));
    L.off_ab = (int)o;   o = a16(o + (size_t)dm.D * dm.G * sizeof(double2));
    L.off_q = (int)o;    o = a16(o + (size_t)dm.Q * sizeof(QRec));
    L.off_trw = (int)o;  o = a16(o + (size_t)dm.D * 2 * dm.M * dm.M * 8);
    L.off_trc = (int)o;  o = a16(o + (size_t)dm.D * 2 * dm.M * dm.M * 8);
    L.off_mem = (int)o;  o = a16(o + (size_t)dm.M * 4);
    L.off_cap = (int)o;  o = a16(o + (size_t)dm.D * 4);
    L.off_tile = (int)o; o = a16(o + ((p.wt || p.sd || p.vo) ? (size_t)3 * dm.G * kTwPad * 4 : 0));
    L.off_rows = (int)o; o = a16(o + (size_t)kTwWarps * 2 * L.ldr * 2);
    L.off_qbeg = (int)o; o = a16(o + (size_t)kTwWarps * (dm.Q + 1) * 4);
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, tier_warp_kernel);
    if (e != cudaSuccess) return e;
    if (o + fa.sharedSizeBytes > (size_t)optin) return cudaErrorNotSupported;
    if ((e = cudaFuncSetAttribute(tier_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)o)))
        return e;
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tier_warp_kernel, 256, o);
    if (nb < 1) return cudaErrorNotSupported;
    int64_t grid = (p.cd.count + kTwWarps - 1) / kTwWarps;
    if (grid > (int64_t)sm_count() * nb) grid = (int64_t)sm_count() * nb;
    if (grid > p.max_blocks) grid = p.max_blocks;
    if (grid < 1) grid = 1;
    tier_warp_kernel<<<(unsigned)grid, 256, o, st>>>(p, L);
    ++g_launches;
    return cudaGetLastError();
}

// Large-T RANDOM under tiers: rows generated per chunk by fy_rows_kernel (one
// lane per row, 32 rows per warp) instead of one lane of the scoring warp, then
// scored by the lane-per-queue kernel reading them; argmin carried across
// chunks like launch_two_phase.
static cudaError_t launch_tier_two_phase(const ScanParams &p0, cudaStream_t st) {
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
        if ((e = launch_tier_warp(p, st)) != cudaSuccess) return e;
        if (p0.out_rec && c0) {
            if ((e = launch_reduce_records(p0.chunk_recs, 2, p0.chunk_recs, st)) != cudaSuccess) return e;
        }
    }
    return p0.out_rec ? launch_reduce_records(p0.chunk_recs, 1, p0.out_rec, st) : cudaSuccess;
}

cudaError_t launch_tier(const ScanParams &p, cudaStream_t st) {
    const cudaError_t ws = launch_ws_tier(p, st);            // warp-specialised fast path
    if (ws != cudaErrorNotSupported) return ws;
    if (p.dm.G > 256 && p.cd.kind == QLM_CAND_RANDOM && p.dm.T > 256 && p.ilv && p.ilv_cap >= 32 &&
        p.chunk_recs && !p.cd.first_from && p.cd.count >= 4096 && !override_on(QLM_OVERRIDE_NO_TIER_WARP) &&
        !override_on(QLM_OVERRIDE_NO_TWO_PHASE)) {
        const cudaError_t w = launch_tier_two_phase(p, st);
        if (w != cudaErrorNotSupported) return w;
        cudaGetLastError();
    }
    if (p.dm.G > 256 && !override_on(QLM_OVERRIDE_NO_TIER_WARP)) {   // large G: lane per queue
        const cudaError_t w = launch_tier_warp(p, st);
        if (w != cudaErrorNotSupported) return w;
        cudaGetLastError();
        return launch_big_tier(p, st);                        // tables too large for shared memory
    }
    const bool u8 = p.dm.T <= 256;
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM:
        return u8 ? launch_tier_t<QLM_CAND_RANDOM, uint8_t>(p, st) : launch_tier_t<QLM_CAND_RANDOM, uint16_t>(p, st);
    case QLM_CAND_EXPLICIT:
        return p.cd.tb == 1 ? launch_tier_t<QLM_CAND_EXPLICIT, uint8_t>(p, st)
                            : launch_tier_t<QLM_CAND_EXPLICIT, uint16_t>(p, st);
    case QLM_CAND_NEIGHBOR:
        return p.cd.tb == 1 ? launch_tier_t<QLM_CAND_NEIGHBOR, uint8_t>(p, st)
                            : launch_tier_t<QLM_CAND_NEIGHBOR, uint16_t>(p, st);
    default:
        return launch_tier_t<QLM_CAND_ENUM, uint8_t>(p, st);
    }
}

}  // namespace qlm
