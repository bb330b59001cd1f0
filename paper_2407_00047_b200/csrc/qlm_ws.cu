// qlm_ws.cu -- warp-specialised scan kernel (the bulk fast path on sm_100a).
//
// A block holds W producer/consumer warp pairs.  Work unit = a batch of 32
// consecutive candidates.  Pair p of a block takes the block's batches
// p, p+W, p+2W, ... and double-buffers them through two row slots in shared
// memory:
//
//   producer warp  -- generates the batch's 32 candidate rows (Philox +
//                     Fisher-Yates, Lehmer unranking, or a copy of EXPLICIT
//                     rows), one row per lane, in place in the slot;
//                     mbarrier full[slot]
//   consumer warp  -- walks each row once (Eq. 2/3/10, R1-R7), violation
//                     probability (R8/R9), S1/S2 (R11) and the argmin; stages
//                     wt / sd / v group-major in its own smem tile [3][G][32]
//                     (bank = lane) and writes each array with ONE 2-D TMA
//                     tensor store (box {32 candidates, G groups}) into the
//                     group-major outputs; mbarrier empty[slot]
//
// Row generation is a chain of dependent shared-memory swaps; the scan is a
// chain of dependent fp64 adds.  Splitting them across warps lets each hide
// the other's latency with only ~7 consumer tiles resident (the staging
// tiles are what fills shared memory).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "qlm_device.cuh"
#include "qlm_launch.h"
#include "qlm_argmin.cuh"

namespace qlm {

struct alignas(64) WsParams {
    CUtensorMap tmap[3];   // wt, sd, v: fp32 [G][count], box {32, G}
    ScanParams p;
    int pairs;             // W
    int spread;            // 1: producers only on schedulers 2/3 (16-warp block), see launch
    int tw;                // 32-bit words per row slot column
    int off_rows, off_stage, off_bar, off_pend, off_tmem;
    int stage_floats;      // per consumer warp: 3 * G * 32
    int use_tma;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *b, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Wait for a phase.
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    // try_wait suspends the warp in hardware until the phase completes (or a
    // time limit passes), so the loop issues a handful of instructions per wait
    while (!mbar_try(b, parity)) {
    }
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *tm, const void *src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 ::"l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
}

// Row generation of one candidate into the lane's column of a row slot.
template <int KIND, typename TOK>
__device__ __forceinline__ void produce_row(const Cand &cd, int T, uint8_t *slot, int lane,
                                            int64_t loc, int64_t c) {
    if constexpr (KIND == QLM_CAND_RANDOM) {
        fy_materialise<TOK>(slot, 32, lane, T, cd.seed, (uint64_t)c);
    } else if constexpr (KIND == QLM_CAND_ENUM) {
        int s = 0;
        tokens_enum((uint64_t)c, T, [&](int tok) { *fy_elem<TOK>(slot, s++, 32, lane) = (TOK)tok; });
    } else if constexpr (KIND == QLM_CAND_NEIGHBOR) {
        // base row words (every lane reads the same word: a broadcast), then
        // the candidate's k transpositions in the lane's column (R18)
        constexpr int EPW = 4 / (int)sizeof(TOK);
        const uint32_t *b32 = reinterpret_cast<const uint32_t *>(cd.rows);
        uint32_t *w32 = reinterpret_cast<uint32_t *>(slot);
        if (cd.tb == (int)sizeof(TOK)) {
            for (int w = 0; w < (T + EPW - 1) / EPW; ++w) w32[w * 32 + lane] = __ldg(b32 + w);
        } else {
            for (int i = 0; i < T; ++i)
                *fy_elem<TOK>(slot, i, 32, lane) =
                    (TOK)(cd.tb == 1 ? base_token<uint8_t>(cd, i) : base_token<uint16_t>(cd, i));
        }
        int mi[QLM_MAX_MOVES], mj[QLM_MAX_MOVES];
        nbr_moves(cd, T, (uint64_t)c, mi, mj);
        for (int m = 0; m < cd.moves; ++m) {
            TOK *pi = fy_elem<TOK>(slot, mi[m], 32, lane), *pj = fy_elem<TOK>(slot, mj[m], 32, lane);
            const TOK t = *pi;
            *pi = *pj;
            *pj = t;
        }
    } else {
        int s = 0;
        const uint8_t *row = cd.rows + loc * cd.stride;
        auto put = [&](int tok) { *fy_elem<TOK>(slot, s++, 32, lane) = (TOK)tok; };
        if (cd.tb == 1) tokens_explicit<uint8_t>(row, T, put);
        else tokens_explicit<uint16_t>(row, T, put);
    }
}

// Branch-free consumer of one 32-bit word of a row (K = 4 / sizeof(TOK)
// tokens).  Separators are handled with selects (a separator slot computes a
// throw-away group slot and then resets the queue state), so the K slots of a
// word are straight-line code: all shared-memory loads of the word are issued
// before its fp64 chain, and its staging stores come last.  Staging offsets
// of separator slots point at a trash row (row G of each staged array).
// Shared-memory tables of the warp-specialised consumer.  Index G of the
// group tables is a zero "separator" record and row G of the staging tile a
// trash row, so a separator slot runs the same straight-line code as a group
// slot; the queue table is padded to T entries so the queue counter needs no
// clamp.
// Transition entries are 8 B: a 64-bit shared load is served per half-warp
// (16 lanes), so 16 interleaved replicas make it conflict-free.
constexpr int kTrRs = 4;
struct alignas(16) WsG {      // 16 B (one LDS.128), replicated 1 << RS times
    double slo;
    float nf;                // n_i as float (S1 numerator, exact below 2^24)
    int model;
};
struct alignas(16) WsQ {      // 32 B (two LDS.128)
    double bmean, bvar;      // queue reset values (R12)
    int prow0;               // transition-table row at the queue's start (R4)
    int dG;                  // d * (G + 1): device base into the ab table
    int dbase;               // d * 2M * M: device base into the transition table
    int tier;                // R20: (CPU memory cap << 6) | resident model (tiered kernels only)
};

struct Acc {
    double A, S2;
    float B;                 // fp32 variance accumulator (R22)
    float acc1;              // sum n_i v_i over clamped slots (v in {0, 1}: exact)
    double acc2;             // sum n_i v_i over unclamped slots, row order
    int prow, dG, dbase, q, over, npend;
    // two-tier swapping (R20): previous model, seen / warm target masks,
    // CPU memory taken, exhausted flag, the queue's CPU memory
    int pmod, cum, exh, capd;
    uint32_t seen, warm;
};

// Unclamped slots (|z| < z_clamp, ~1-2 % of slots) are queued per lane --
// (z, group) in shared memory -- and their Phi-bar evaluated later in FIFO
// (= row) order, so the warp runs the expensive path only for the lanes and
// slots that need it instead of for the whole warp on every slot where any
// lane needs it.
constexpr int kPend = 8;     // queue depth per lane
struct Pend {
    float z;
    int tg;
};

template <bool SCORE, int RSCALE>
__device__ __forceinline__ void flush_pending(Pend *pq, const WsG *__restrict__ sgl, int lane,
                                              float alpha, float *st2, Acc &a) {
    const int maxn = (int)__reduce_max_sync(__activemask(), (unsigned)a.npend);
    for (int i = 0; i < maxn; ++i) {
        if (i < a.npend) {
            const Pend e = pq[i * 32 + lane];
            const float v = phibar(e.z);
            st2[e.tg * 32 + lane] = v;
            if constexpr (SCORE) {
                a.acc2 = __fma_rn((double)sgl[e.tg * RSCALE].nf, (double)v, a.acc2);
                a.over += v > alpha ? 1 : 0;
            }
        }
    }
    a.npend = 0;
}

template <typename TOK, int RS, bool SCORE, bool PAD, bool TIER>
__device__ __forceinline__ void consume_word(const WsG *__restrict__ sgl, const double2 *__restrict__ sabl,
                                             const double *__restrict__ str, const WsQ *__restrict__ sq,
                                             uint32_t word, int nvalid_tok, int G, int M, int lane,
                                             float zc, float alpha, float *st, int arr_stride,
                                             Pend *pq, Acc &a, const int *__restrict__ smemsz,
                                             int cold_off) {
    constexpr int K = 4 / (int)sizeof(TOK);
    int isbar[K], tg[K];
    WsG g[K];
    WsQ r[K];
    // (i) tokens, separators, group and queue records (independent loads)
    int q = a.q;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int tok = K == 4 ? (int)((word >> (8 * k)) & 0xFFu) : (int)((word >> (16 * k)) & 0xFFFFu);
        const bool pad = PAD && k >= nvalid_tok;
        isbar[k] = tok >= G && !pad;
        tg[k] = pad ? G : min(tok, G);
        q += isbar[k];
        {   // one 128-bit load (two 64-bit loads of 8-way replicated 16-B records conflict)
            const double2 raw = *reinterpret_cast<const double2 *>(sgl + (tg[k] << RS));
            g[k].slo = raw.x;
            const unsigned long long hi = (unsigned long long)__double_as_longlong(raw.y);
            g[k].nf = __uint_as_float((uint32_t)hi);
            g[k].model = (int)(uint32_t)(hi >> 32);
        }
        if (isbar[k]) r[k] = sq[q];                          // only separator lanes read
        else { r[k].bmean = 0.0; r[k].bvar = 0.0; r[k].prow0 = 0; r[k].dG = 0; r[k].dbase = 0; r[k].tier = 0; }
    }
    // (ii) per-slot transition row and device base
    int pk[K], dk[K];
    int prow = a.prow, dG = a.dG, dbase = a.dbase;
    bool cold[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        pk[k] = prow;
        dk[k] = dG;
        cold[k] = false;
        const bool pad = PAD && k >= nvalid_tok;
        if (!pad) {
            if constexpr (TIER) {
                // R20: per queue, swap targets in first-transition order are warm
                // while they fit the CPU memory (strict prefix); branch-free
                const int m = g[k].model;
                const uint32_t bit = 1u << m;
                const bool trn = !isbar[k] && m != a.pmod;
                const bool firstT = trn && !(a.seen & bit);
                const int need = a.cum + smemsz[m];
                const bool fits = !a.exh && need <= a.capd;
                a.seen |= firstT ? bit : 0u;
                a.warm |= (firstT && fits) ? bit : 0u;
                a.cum = (firstT && fits) ? need : a.cum;
                a.exh = (a.exh || (firstT && !fits)) ? 1 : 0;
                cold[k] = trn && !(a.warm & bit);
                a.pmod = isbar[k] ? (r[k].tier & 63) : m;
                a.capd = isbar[k] ? (r[k].tier >> 6) : a.capd;
                a.seen = isbar[k] ? 0u : a.seen;
                a.warm = isbar[k] ? 0u : a.warm;
                a.cum = isbar[k] ? 0 : a.cum;
                a.exh = isbar[k] ? 0 : a.exh;
            }
            prow = isbar[k] ? r[k].prow0 : dbase + g[k].model * M;
            dG = isbar[k] ? r[k].dG : dG;
            dbase = isbar[k] ? r[k].dbase : dbase;
        }
    }
    // (iii) per-device group work and transition costs
    double2 ab[K];
    double tr[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        ab[k] = sabl[(dk[k] + tg[k]) << RS];
        const int ti = (pk[k] + g[k].model) << kTrRs;        // 16 replicas: conflict-free
        tr[k] = str[TIER && cold[k] ? ti + cold_off : ti];   // R20: cold table follows the warm one
    }
    // (iv) the Eq. 10 chain (operation order identical to the sequential definition)
    double wt[K];
    float V[K];
    double A = a.A;
    float B = a.B;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double A1 = __dadd_rn(A, tr[k]);
        wt[k] = A1;
        V[k] = B;
        const double A2 = __dadd_rn(A1, ab[k].x);
        const float B2 = __fadd_rn(B, (float)ab[k].y);
        if (PAD && k >= nvalid_tok) continue;
        A = isbar[k] ? r[k].bmean : A2;
        B = isbar[k] ? (float)r[k].bvar : B2;
    }
    a.A = A; a.B = B; a.prow = prow; a.dG = dG; a.dbase = dbase; a.q = q;
    // (v) violation probabilities, scores, staging
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double slack = __dsub_rn(g[k].slo, wt[k]);
        const float sf = (float)slack;
        const float sd = slot_sd(V[k]);
        const bool clamped = slot_clamped(sf, sd, zc);        // R9 / R22
        const float v = slot_v_clamped(sf);
        const bool grp = !isbar[k] && tg[k] < G;
        const bool defer = grp && !clamped;
        if (defer) {                                           // exact value later, FIFO
            Pend e;
            e.z = sf * rcp_approx(sd);                       // phibar(e.z) = slot_v_open(sf, sd)
            e.tg = tg[k];
            pq[a.npend * 32 + lane] = e;
            ++a.npend;
        }
        if constexpr (SCORE) {
            a.S2 = __dsub_rn(a.S2, grp ? slack : 0.0);
            if (!defer) {
                a.acc1 = fmaf(g[k].nf, v, a.acc1);             // separators have nf = 0
                a.over += (grp && v > alpha) ? 1 : 0;
            }
        }
        {
            float *o = st + tg[k] * 32 + lane;               // separators -> trash row G
            o[0] = (float)wt[k];
            o[arr_stride] = sd;
            o[2 * arr_stride] = v;                           // deferred slots overwritten at flush
        }
    }
}

template <int KIND, typename TOK, bool SCORE, int RS, bool TIER>
__global__ void __launch_bounds__(512, 1) ws_kernel(const __grid_constant__ WsParams w) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const ScanParams &p = w.p;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = w.pairs;
    const int G = p.dm.G, Q = p.dm.Q, T = p.dm.T, M = p.dm.M, D = p.dm.D;

    // ---- tables -> smem: group records (+ zero separator record at index G),
    // replicated 1 << RS times; per-device group work (+ zero record); queue
    // records padded to T; transition rows with virtual resident rows (R4)
    WsG *sg = reinterpret_cast<WsG *>(smem + p.off_grec);
    for (int i = tid; i < ((G + 1) << RS); i += blockDim.x) {
        const int gi = i >> RS;
        WsG r;
        if (gi < G) {
            const GRec x = p.tb.grec[gi];
            r.slo = x.slo; r.nf = (float)x.n; r.model = x.model;
        } else {
            r.slo = 0.0; r.nf = 0.0f; r.model = 0;
        }
        sg[i] = r;
    }
    double2 *sab = reinterpret_cast<double2 *>(smem + p.off_ab);
    for (int i = tid; i < ((D * (G + 1)) << RS); i += blockDim.x) {
        const int e = i >> RS, d = e / (G + 1), gi = e - d * (G + 1);
        sab[i] = gi < G ? p.tb.ab[d * G + gi] : make_double2(0.0, 0.0);
    }
    WsQ *sq = reinterpret_cast<WsQ *>(smem + p.off_q);
    int *smemsz = reinterpret_cast<int *>(smem + w.off_tmem);
    int summem = 0;
    if constexpr (TIER) {
        for (int m = 0; m < M; ++m) summem += p.t_mem[m];
        for (int i = tid; i < M; i += blockDim.x) smemsz[i] = p.t_mem[i];
    }
    for (int i = tid; i < T + 1; i += blockDim.x) {
        const QRec x = p.tb.qrec[i < Q ? i : Q - 1];
        WsQ r;
        r.bmean = x.bmean; r.bvar = x.bvar;
        r.prow0 = (x.d * 2 * M + (x.backlog ? x.r : M + x.r)) * M;
        r.dG = x.d * (G + 1);
        r.dbase = x.d * 2 * M * M;
        r.tier = TIER ? (min(p.t_cap[x.d], summem) << 6) | x.r : 0;   // cap >= sum(mem) == unbounded
        sq[i] = r;
    }
    double *str = reinterpret_cast<double *>(smem + p.off_tr);
    const int ntr = (D * 2 * M * M) << kTrRs;
    for (int i = tid; i < (TIER ? 2 * ntr : ntr); i += blockDim.x) {
        const int e = (i % ntr) >> kTrRs;
        const int m = e % M, pp = (e / M) % (2 * M), d = e / (2 * M * M);
        const int from = pp < M ? pp : pp - M;
        const double sw = p.tb.swap[(d * M + from) * M + m];
        const double tl = (pp < M && m != pp) ? p.tb.tail[d * M + pp] : 0.0;
        if (i < ntr) str[i] = __dadd_rn(tl, sw);         // one transition term (R2/R3)
        else str[i] = __dadd_rn(tl, __dadd_rn(sw, m != from ? p.t_load[d * M + m] : 0.0));   // cold (R20)
    }
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + w.off_bar);
    uint64_t *empty = full + 2 * W;
    // dynamic batches: each producer takes the block's next batch from a
    // shared counter and leaves its index with the row slot, so pairs on
    // lightly loaded schedulers take more tiles (static striding made every
    // pair wait for the slowest one at the end)
    int64_t *slot_b = reinterpret_cast<int64_t *>(empty + 2 * W);        // [2W]
    unsigned long long *next_b = reinterpret_cast<unsigned long long *>(slot_b + 2 * W);
    if (tid < 2 * W) {
        mbar_init(&full[tid], 32);
        mbar_init(&empty[tid], 32);
    }
    if (tid == 0) *next_b = 0ull;
    __syncthreads();

    const Cand cd = p.cd;
    const int64_t count = cd.count, first = cd.first;
    const int64_t nbatch = (count + 31) >> 5;
    // Role of this warp.  Default: warps [0, W) consume, [W, 2W) produce.
    // spread (W = 6, 16 warps): consumers 0-5 (two per scheduler on 0/1, one
    // on 2/3), producers 6, 7, 10, 11, 14, 15 (schedulers 2/3 only), warps
    // 8, 9, 12, 13 idle -- every scheduler then issues one consumer's worth
    // plus at most three producers' instead of 2 + 1 / 1 + 2.
    int pair = warp % W;
    bool producer = warp >= W;
    bool idle = false;
    if (w.spread) {
        producer = warp >= 6;
        const int pmap[16] = {0, 1, 2, 3, 4, 5, 0, 1, -1, -1, 2, 3, -1, -1, 4, 5};
        pair = pmap[warp];
        idle = pair < 0;
    }
    const int64_t grid = gridDim.x;
    uint64_t bkey = ~0ull;
    int64_t bidx = -1;

    if (idle) {
        // no role: only the block-wide argmin below
    } else if (producer) {
        for (int j = 0;; ++j) {
            const int s = 2 * pair + (j & 1);
            mbar_wait(&empty[s], ((j >> 1) & 1) ^ 1);
            int64_t b = 0;
            if (lane == 0) {
                b = blockIdx.x + (int64_t)atomicAdd(next_b, 1ull) * grid;
                slot_b[s] = b;                             // published by the arrive below
            }
            b = __shfl_sync(0xFFFFFFFFu, b, 0);
            if (b >= nbatch) {                             // end of stream for the paired consumer
                mbar_arrive(&full[s]);
                break;
            }
            const int64_t loc = (b << 5) + lane;
            uint8_t *slot = smem + w.off_rows + (size_t)s * w.tw * 128;
            if (loc < count) produce_row<KIND, TOK>(cd, T, slot, lane, loc, first + loc);
            mbar_arrive(&full[s]);
        }
    } else {
        const WsG *sgl = sg + (lane & ((1 << RS) - 1));
        const double2 *sabl = sab + (lane & ((1 << RS) - 1));
        const double *strl = str + (lane & ((1 << kTrRs) - 1));
        const float zc = p.zc;
        const float alpha = p.alpha;
        const double den = *p.tb.den;
        const int arr = (G + 1) * 32;
        float *st = reinterpret_cast<float *>(smem + w.off_stage) + (size_t)pair * w.stage_floats;
        float *st0 = st, *st1 = st + arr, *st2 = st + 2 * arr;
        Pend *pq = reinterpret_cast<Pend *>(smem + w.off_pend) + (size_t)pair * kPend * 32;
        const WsG *sgl_rs = sg + ((size_t)(lane & ((1 << RS) - 1)));   // flush reads record tg << RS
        constexpr int EPW = 4 / (int)sizeof(TOK);
        const int full_words = T / EPW;
        const int tw = w.tw;
        for (int j = 0;; ++j) {
            const int s = 2 * pair + (j & 1);
            mbar_wait(&full[s], (j >> 1) & 1);
            const int64_t b = slot_b[s];
            if (b >= nbatch) break;
            if (j > 0 && w.use_tma) {
                if (lane == 0) bulk_wait_read0();              // previous tile read out
                __syncwarp();
            }
            const int64_t c0 = b << 5, loc = c0 + lane;
            const uint32_t *w32 = reinterpret_cast<const uint32_t *>(smem + w.off_rows + (size_t)s * w.tw * 128);
            if (loc < count) {
                Acc a;
                const WsQ r0 = sq[0];
                a.A = r0.bmean; a.B = (float)r0.bvar; a.prow = r0.prow0; a.dG = r0.dG; a.dbase = r0.dbase;
                a.q = 0; a.S2 = 0.0; a.acc1 = 0.0f; a.acc2 = 0.0; a.over = 0; a.npend = 0;
                a.pmod = r0.tier & 63; a.capd = r0.tier >> 6; a.cum = 0; a.exh = 0; a.seen = 0u; a.warm = 0u;
                uint32_t cur = w32[lane];
                for (int wi = 0; wi < full_words; ++wi) {
                    const uint32_t nxt = w32[(wi + 1 < tw ? wi + 1 : wi) * 32 + lane];   // prefetch
                    consume_word<TOK, RS, SCORE, false, TIER>(sgl, sabl, strl, sq, cur, EPW, G,
                                                              M, lane, zc, alpha, st, arr, pq, a,
                                                              smemsz, ntr);
                    cur = nxt;
                    if (__any_sync(__activemask(), a.npend > kPend - EPW))
                        flush_pending<SCORE, (1 << RS)>(pq, sgl_rs, lane, alpha, st2, a);
                }
                if (full_words * EPW < T)
                    consume_word<TOK, RS, SCORE, true, TIER>(sgl, sabl, strl, sq, cur,
                                                             T - full_words * EPW, G, M, lane, zc,
                                                             alpha, st, arr, pq, a, smemsz, ntr);
                flush_pending<SCORE, (1 << RS)>(pq, sgl_rs, lane, alpha, st2, a);
                if constexpr (SCORE) {
                    const float s1 = (float)(((double)a.acc1 + a.acc2) / den);     // R11
                    const float s2 = (float)a.S2;
                    if (p.s1) p.s1[loc] = s1;
                    if (p.s2) p.s2[loc] = s2;
                    if (p.n_over) p.n_over[loc] = a.over;
                    const uint64_t key = make_key(s1, s2);
                    const int64_t c = first + loc;
                    if (better(key, c, bkey, bidx)) { bkey = key; bidx = c; }
                }
            }
            mbar_arrive(&empty[s]);                              // row slot free
            if (w.use_tma) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (p.wt) tma_store_2d(&w.tmap[0], st0, (int)c0, 0);
                    if (p.sd) tma_store_2d(&w.tmap[1], st1, (int)c0, 0);
                    if (p.vo) tma_store_2d(&w.tmap[2], st2, (int)c0, 0);
                    bulk_commit();
                }
            } else {
                __syncwarp();
                if (loc < count) {
                    for (int g = 0; g < G; ++g) {
                        const int64_t o = (int64_t)g * count + loc;
                        if (p.wt) p.wt[o] = st0[g * 32 + lane];
                        if (p.sd) p.sd[o] = st1[g * 32 + lane];
                        if (p.vo) p.vo[o] = st2[g * 32 + lane];
                    }
                }
                __syncwarp();
            }
        }
        if (w.use_tma && lane == 0) bulk_wait0();
    }
    if constexpr (SCORE) {
        if (p.out_rec) block_grid_argmin(p, bkey, bidx);   // all warps take part
    }
}

// ---- host side ----------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        else
            cudaGetLastError();
    }
    return fn;
}

static bool make_map(CUtensorMap *tm, float *ptr, int64_t count, int G) {
    auto fn = encode_fn();
    if (!fn || !ptr) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)count, (cuuint64_t)G};
    const cuuint64_t strides[1] = {(cuuint64_t)count * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)G};
    const cuuint32_t estr[2] = {1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
static size_t a1k(size_t x) { return (x + 1023) & ~size_t(1023); }

static int env_int_ws(const char *name, int dflt) { return env_cached(name, dflt); }

// Shared-memory plan for W pairs; returns total bytes.
static size_t plan_ws(WsParams &w, int W, int rs, int tok_bytes, bool stage, bool tier) {
    ScanParams &p = w.p;
    const Dims &dm = p.dm;
    size_t off = 0;
    p.rep_shift = rs;
    p.off_grec = (int)off; off = a16(off + ((size_t)(dm.G + 1) << rs) * sizeof(WsG));
    p.off_ab = (int)off;   off = a16(off + ((size_t)dm.D * (dm.G + 1) << rs) * sizeof(double2));
    p.off_q = (int)off;    off = a16(off + (size_t)(dm.T + 1) * sizeof(WsQ));
    p.off_tr = (int)off;   off = a16(off + ((size_t)dm.D * 2 * dm.M * dm.M << kTrRs) * sizeof(double) * (tier ? 2 : 1));
    w.off_tmem = (int)off; off = a16(off + (tier ? (size_t)dm.M * 4 : 0));
    const int epw = 4 / tok_bytes;
    w.tw = (dm.T + epw - 1) / epw;
    w.off_rows = (int)off; off = a16(off + (size_t)2 * W * w.tw * 128);
    w.off_bar = (int)off;  off = a16(off + (size_t)6 * W * 8 + 8);   // full, empty, slot batch, counter
    w.off_pend = (int)off; off = a16(off + (size_t)W * kPend * 32 * sizeof(Pend));
    w.stage_floats = stage ? 3 * (dm.G + 1) * 32 : 0;
    off = a1k(off);
    w.off_stage = (int)off;
    off += (size_t)W * w.stage_floats * 4;
    w.pairs = W;
    return off;
}

// Dynamic shared-memory opt-in of a kernel on the current device (the
// attribute is per device), cached per (kernel, device).
template <typename K>
static size_t ws_max_dyn(K kern) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, size_t> cache;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(reinterpret_cast<const void *>(kern), dev);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    size_t m = 0;
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess && optin > (int)fa.sharedSizeBytes + 1024) {
        m = (size_t)optin - fa.sharedSizeBytes - 1024;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m) != cudaSuccess) m = 0;
    }
    cudaGetLastError();
    cache[key] = m;
    return m;
}

template <int KIND, typename TOK, bool SCORE, int RS, bool TIER>
static cudaError_t launch_ws_rs(WsParams &w, size_t smem, int W, cudaStream_t st) {
    auto kern = ws_kernel<KIND, TOK, SCORE, RS, TIER>;
    const size_t lim = ws_max_dyn(kern);
    if (!lim || smem > lim) return cudaErrorNotSupported;
    const int64_t nbatch = (w.p.cd.count + 31) / 32;
    int64_t grid = sm_count();
    const int64_t need = (nbatch + W - 1) / W;
    if (grid > need) grid = need;
    if (grid > w.p.max_blocks) grid = w.p.max_blocks;
    if (grid < 1) grid = 1;
    qlog(1, "ws_kernel<kind=%d,tok=%zu,score=%d,rs=%d,tier=%d> count=%lld pairs=%d grid=%lld smem=%zu tma=%d",
         KIND, sizeof(TOK), (int)SCORE, RS, (int)TIER, (long long)w.p.cd.count, W, (long long)grid, smem,
         w.use_tma);
    kern<<<(unsigned)grid, w.spread ? 512 : 64 * W, smem, st>>>(w);
    ++g_launches;
    return cudaGetLastError();
}

template <int KIND, typename TOK, bool SCORE, bool TIER>
static cudaError_t launch_ws_t(const ScanParams &p0, cudaStream_t st) {
    constexpr bool STAGE = true;
    const size_t lim = 227 * 1024 - 2048;
    WsParams w;
    memset(&w, 0, sizeof w);
    w.p = p0;
    const int maxW = STAGE ? 8 : 16;
    const int envW = env_int_ws("QLM_WS_PAIRS", 0), envRs = env_int_ws("QLM_REP_SHIFT", -1);
    int bestW = 0, bestRs = 0;
    size_t bestSmem = 0;
    for (int rs : {3, 0}) {
        if (envRs >= 0 && rs != envRs) continue;
        for (int W = maxW; W >= 1; --W) {
            if (envW && W != envW) continue;
            WsParams t = w;
            const size_t sm = plan_ws(t, W, rs, sizeof(TOK), STAGE, TIER);
            if (sm <= lim) {
                if (W > bestW) { bestW = W; bestRs = rs; bestSmem = sm; }
                break;
            }
        }
        if (bestW >= (STAGE ? 6 : 16)) break;
    }
    if (bestW < (STAGE ? 2 : 4)) return cudaErrorNotSupported;
    plan_ws(w, bestW, bestRs, sizeof(TOK), STAGE, TIER);
    // W = 6: spread the roles over the four schedulers (measured C3 fused pass
    // 0.370 -> 0.350 ms); QLM_WS_SPREAD=0 restores the plain warp order
    w.spread = (bestW == 6 && env_int_ws("QLM_WS_SPREAD", 1)) ? 1 : 0;
    if (STAGE) {
        const bool aligned = (p0.cd.count % 4 == 0) && p0.cd.count <= INT32_MAX - 64 &&   // int32 TMA x
                             (!p0.wt || ((uintptr_t)p0.wt & 15) == 0) &&
                             (!p0.sd || ((uintptr_t)p0.sd & 15) == 0) &&
                             (!p0.vo || ((uintptr_t)p0.vo & 15) == 0) && p0.dm.G <= 256;
        bool ok = aligned;
        if (ok && p0.wt) ok = make_map(&w.tmap[0], p0.wt, p0.cd.count, p0.dm.G);
        if (ok && p0.sd) ok = make_map(&w.tmap[1], p0.sd, p0.cd.count, p0.dm.G);
        if (ok && p0.vo) ok = make_map(&w.tmap[2], p0.vo, p0.cd.count, p0.dm.G);
        w.use_tma = ok ? 1 : 0;
    }
    return bestRs == 3 ? launch_ws_rs<KIND, TOK, SCORE, 3, TIER>(w, bestSmem, bestW, st)
                       : launch_ws_rs<KIND, TOK, SCORE, 0, TIER>(w, bestSmem, bestW, st);
}

template <int KIND, typename TOK>
static cudaError_t launch_ws_k(ScanParams &p, cudaStream_t st) {
    const bool score = p.s1 || p.s2 || p.n_over || p.out_rec;
    const bool stage = p.wt || p.sd || p.vo;
    if (!stage) return cudaErrorNotSupported;   // score-only: the one-warp-per-32-candidates kernel is faster
    if ((size_t)3 * (p.dm.G + 1) * 32 * 4 * 2 > 200 * 1024) return cudaErrorNotSupported;
    return score ? launch_ws_t<KIND, TOK, true, false>(p, st) : launch_ws_t<KIND, TOK, false, false>(p, st);
}

// Two-tier swapping (R20) through the warp-specialised kernel: RANDOM and
// EXPLICIT candidates with bulk outputs (the tier kernel covers the rest).
cudaError_t launch_ws_tier(ScanParams p, cudaStream_t st) {
    if (p.cd.first_from || p.cd.count < 4096 || override_on(QLM_OVERRIDE_NO_WS)) return cudaErrorNotSupported;
    if (!(p.wt || p.sd || p.vo) || p.dm.M > 32) return cudaErrorNotSupported;
    if (!override_on(QLM_OVERRIDE_NO_WS2)) {
        const cudaError_t e = launch_ws2_tier(p, st);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    if ((size_t)3 * (p.dm.G + 1) * 32 * 4 * 2 > 200 * 1024) return cudaErrorNotSupported;
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM:
        return p.dm.T <= 256 ? launch_ws_t<QLM_CAND_RANDOM, uint8_t, true, true>(p, st)
                             : launch_ws_t<QLM_CAND_RANDOM, uint16_t, true, true>(p, st);
    case QLM_CAND_EXPLICIT:
        return p.dm.T <= 256 ? launch_ws_t<QLM_CAND_EXPLICIT, uint8_t, true, true>(p, st)
                             : launch_ws_t<QLM_CAND_EXPLICIT, uint16_t, true, true>(p, st);
    default:
        return cudaErrorNotSupported;
    }
}

// Fast path for large candidate sets; cudaErrorNotSupported -> caller falls back.
cudaError_t launch_ws(ScanParams p, cudaStream_t st) {
    if (p.cd.first_from || p.cd.count < 4096 || override_on(QLM_OVERRIDE_NO_WS)) return cudaErrorNotSupported;
    if (!override_on(QLM_OVERRIDE_NO_WS2)) {
        const cudaError_t e = launch_ws2(p, st);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM:
        return p.dm.T <= 256 ? launch_ws_k<QLM_CAND_RANDOM, uint8_t>(p, st)
                             : launch_ws_k<QLM_CAND_RANDOM, uint16_t>(p, st);
    case QLM_CAND_EXPLICIT:
        return p.dm.T <= 256 ? launch_ws_k<QLM_CAND_EXPLICIT, uint8_t>(p, st)
                             : launch_ws_k<QLM_CAND_EXPLICIT, uint16_t>(p, st);
    case QLM_CAND_NEIGHBOR:
        return p.dm.T <= 256 ? launch_ws_k<QLM_CAND_NEIGHBOR, uint8_t>(p, st)
                             : launch_ws_k<QLM_CAND_NEIGHBOR, uint16_t>(p, st);
    default:
        return launch_ws_k<QLM_CAND_ENUM, uint8_t>(p, st);
    }
}

}  // namespace qlm
