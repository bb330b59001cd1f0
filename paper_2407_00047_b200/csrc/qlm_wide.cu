// qlm_wide.cu -- warp-per-candidate scan for large G (the bulk path when no
// [G][32] staging tile fits in shared memory).
//
// A block holds 8 warps; warp w scores candidate c0 + w of a batch of 8
// consecutive candidates, so the block's outputs for one group are 8
// consecutive floats = one 32-B sector of the group-major [G][count] arrays.
// They are staged in a [3][G][9] shared tile (row padded to 9 floats: the
// warp's lanes write different groups of one column without bank conflicts)
// and leave as full 32-B rows, so no sector is ever written partially
// (partial 4-B scatters were the 8x write amplification of the DIRECT path).
//
// Within a candidate the row is split into 32 contiguous chunks, one per
// lane.  Queues (R9) make Eq. 10 a *segmented* scan: every separator resets
// (A, B) to the queue's backlog (R12), so
//   pass 1: each lane walks its chunk from a zero state (or from the reset
//           state if a separator precedes it) and reports (reset seen?,
//           A, B) at the chunk end;
//   scan:   a 5-step segmented Kogge-Stone scan over the lanes gives every
//           lane the exact-state-or-sum it starts from;
//   pass 2: each lane walks its chunk again with that start state and emits
//           wt, sd, v for its groups (Eq. 2/3/10, R1-R9).
// The per-chunk state at entry (queue, device, previous model, first slot?)
// is read from the row itself (the token before the chunk, and the number of
// separators before it), so only (A, B) need the scan.  Slots after a
// separator inside a chunk are computed exactly in the oracle's order; slots
// of a chunk's first queue segment start from a scanned sum whose rounding
// differs from the sequential one in the last bits (|rel| ~ 1e-15, DESIGN R15).
#include <cuda_runtime.h>

#include "qlm_argmin.cuh"
#include "qlm_device.cuh"
#include "qlm_launch.h"

namespace qlm {

constexpr int kWideCands = 8;                 // candidates per block (= warps)
constexpr int kWidePad = kWideCands + 1;      // staged row stride (floats)

// The batch's 8 rows are staged in shared memory (u16 tokens, [8][T rounded
// up to 8]) with coalesced loads: for word-interleaved rows, 8 consecutive
// threads read one 32-B sector (word w of the 8 candidates).
template <int KIND>
__device__ __forceinline__ void wide_stage_rows(const Cand &cd, int T, int64_t c0, int nv,
                                                uint16_t *srow, int ldr) {
    const int nw = (T + 1) >> 1;
    uint32_t *s32 = reinterpret_cast<uint32_t *>(srow);
    const int ldw = ldr >> 1;
    if constexpr (KIND == KIND_ILV) {
        // 8 loads in flight per thread before the shared stores
        const uint32_t *r32 = reinterpret_cast<const uint32_t *>(cd.rows);
        const int n = nw * kWideCands, step = blockDim.x;
        for (int i0 = threadIdx.x; i0 < n; i0 += 8 * step) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * step, w = i >> 3, k = i & 7;
                v[u] = (i < n && k < nv) ? __ldcs(r32 + (size_t)w * cd.stride + c0 + k) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * step, w = i >> 3, k = i & 7;
                if (i < n) s32[k * ldw + w] = v[u];
            }
        }
    } else if constexpr (KIND == QLM_CAND_NEIGHBOR) {    // base row (u16) + k swaps per row
        const uint32_t *b32 = reinterpret_cast<const uint32_t *>(cd.rows);
        for (int i = threadIdx.x; i < nw * kWideCands; i += blockDim.x) {
            const int k = i / nw, w = i - k * nw;
            s32[k * ldw + w] = __ldg(b32 + w);
        }
        __syncthreads();
        if (threadIdx.x < nv) {
            uint16_t *r = srow + threadIdx.x * ldr;
            int mi[QLM_MAX_MOVES], mj[QLM_MAX_MOVES];
            nbr_moves(cd, T, (uint64_t)(cd.first + c0 + threadIdx.x), mi, mj);
            for (int m = 0; m < cd.moves; ++m) {
                const uint16_t t = r[mi[m]];
                r[mi[m]] = r[mj[m]];
                r[mj[m]] = t;
            }
        }
    } else {                                   // EXPLICIT u16: row-major, 4-B words
        for (int i = threadIdx.x; i < nw * kWideCands; i += blockDim.x) {
            const int k = i / nw, w = i - k * nw;
            if (k < nv) {
                const uint16_t *row = reinterpret_cast<const uint16_t *>(cd.rows + (c0 + k) * cd.stride);
                const uint32_t lo = __ldg(row + 2 * w);
                const uint32_t hi = 2 * w + 1 < T ? __ldg(row + 2 * w + 1) : 0u;
                s32[k * ldw + w] = lo | (hi << 16);
            }
        }
    }
}

// Word-interleaved rows, software-pipelined: the next batch's words are
// loaded into registers (kWidePf per thread) before the current batch is
// scored and stored to shared memory after it, so the global-load latency
// hides behind the passes (the synchronous staging left the warps waiting on
// it: long-scoreboard stalls were the largest share).
constexpr int kWidePf = 24;                   // words per thread in flight (8 * nw <= 256 * kWidePf)

__device__ __forceinline__ void wide_pf_load(const Cand &cd, int nw, int64_t c0, int nv, uint32_t (&v)[kWidePf]) {
    const uint32_t *r32 = reinterpret_cast<const uint32_t *>(cd.rows);
    const int n = nw * kWideCands;
#pragma unroll
    for (int u = 0; u < kWidePf; ++u) {
        const int i = threadIdx.x + u * 256, w = i >> 3, k = i & 7;
        v[u] = (i < n && k < nv) ? __ldcs(r32 + (size_t)w * cd.stride + c0 + k) : 0u;
    }
}

__device__ __forceinline__ void wide_pf_store(int nw, const uint32_t (&v)[kWidePf], uint16_t *srow, int ldr) {
    uint32_t *s32 = reinterpret_cast<uint32_t *>(srow);
    const int ldw = ldr >> 1, n = nw * kWideCands;
#pragma unroll
    for (int u = 0; u < kWidePf; ++u) {
        const int i = threadIdx.x + u * 256, w = i >> 3, k = i & 7;
        if (i < n) s32[k * ldw + w] = v[u];
    }
}

template <int KIND, bool SCORE>
__global__ void __launch_bounds__(256, 2) wide_kernel(const ScanParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Dims dm = p.dm;
    const int G = dm.G, Q = dm.Q, T = dm.T, M = dm.M;
    // tables (no replication): group records, per-device work, transitions, queues
    // group records and per-device work replicated 1 << rs times (lane l reads
    // copy l mod 2^rs: fewer bank conflicts on the random per-lane lookups);
    // transitions replicated 16 times
    const int rs = p.rep_shift;
    GRec *sg = reinterpret_cast<GRec *>(smem + p.off_grec);
    for (int i = tid; i < (G << rs); i += 256) sg[i] = p.tb.grec[i >> rs];
    double2 *sab = reinterpret_cast<double2 *>(smem + p.off_ab);
    for (int i = tid; i < ((dm.D * G) << rs); i += 256) sab[i] = p.tb.ab[i >> rs];
    QRec *sq = reinterpret_cast<QRec *>(smem + p.off_q);
    for (int i = tid; i < Q; i += 256) sq[i] = p.tb.qrec[i];
    double *str = reinterpret_cast<double *>(smem + p.off_tr);
    for (int i = tid; i < (dm.D * 2 * M * M) << 4; i += 256) {
        const int e = i >> 4;
        const int m = e % M, pp = (e / M) % (2 * M), d = e / (2 * M * M);
        const int from = pp < M ? pp : pp - M;
        const double sw = p.tb.swap[(d * M + from) * M + m];
        const double tl = (pp < M && m != pp) ? p.tb.tail[d * M + pp] : 0.0;
        str[i] = __dadd_rn(tl, sw);                       // one transition term (R2/R3)
    }
    float *tile = reinterpret_cast<float *>(smem + p.off_stage);   // [3][G][kWidePad]
    const int ldr = (T + 7) & ~7;
    uint16_t *srows = reinterpret_cast<uint16_t *>(smem + p.off_scratch);   // [8][ldr]
    __syncthreads();
    SlotTables tab;
    tab.sg = sg; tab.sab = sab; tab.str = str; tab.sq = sq;
    tab.G = G; tab.Q = Q; tab.M = M; tab.rs = rs; tab.rl = lane & ((1 << rs) - 1); tab.trs = 4; tab.trl = lane & 15;

    const Cand cd = p.cd;
    const int64_t count = cd.count;
    const int64_t ldo = p.ld_out ? p.ld_out : count;
    const bool any_out = p.wt || p.sd || p.vo;
    const float zc = p.zc;
    const float alpha = p.alpha;
    const double den = SCORE ? *p.tb.den : 1.0;
    const int S = (T + 31) >> 5;                          // chunk length
    const int p0 = lane * S, p1 = min(p0 + S, T);
    uint64_t bkey = ~0ull;
    int64_t bidx = -1;
    const int64_t nbatch = (count + kWideCands - 1) / kWideCands;
    const int nw = (T + 1) >> 1;
    constexpr bool kIlv = KIND == KIND_ILV;
    const bool pf = kIlv && nw * kWideCands <= 256 * kWidePf;
    uint32_t pfv[kWidePf];
    if (kIlv && pf && blockIdx.x < nbatch)
        wide_pf_load(cd, nw, (int64_t)blockIdx.x * kWideCands,
                     (int)min((int64_t)kWideCands, count - (int64_t)blockIdx.x * kWideCands), pfv);
    for (int64_t bt = blockIdx.x; bt < nbatch; bt += gridDim.x) {
        const int64_t c0 = bt * kWideCands;
        const int64_t loc = c0 + warp;
        if (kIlv && pf) {
            wide_pf_store(nw, pfv, srows, ldr);
            __syncthreads();
            const int64_t bn = bt + gridDim.x;                 // next batch: loads in flight now
            if (bn < nbatch)
                wide_pf_load(cd, nw, bn * kWideCands, (int)min((int64_t)kWideCands, count - bn * kWideCands), pfv);
        } else {
            wide_stage_rows<KIND>(cd, T, c0, (int)min((int64_t)kWideCands, count - c0), srows, ldr);
            __syncthreads();
        }
        const uint16_t *row = srows + warp * ldr;
        if (loc < count) {
            // ---- entry state of this lane's chunk (from the row itself)
            int nsep = 0;
            for (int s = p0; s < p1; ++s) nsep += row[s] >= G;
            int before = nsep;                                 // inclusive -> exclusive scan
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xFFFFFFFFu, before, o);
                if (lane >= o) before += v;
            }
            before -= nsep;
            const int q0 = min(before, Q - 1);
            bool fresh = true;                                 // chunk starts a queue
            int prev_model = 0;
            if (p0 > 0 && p0 < T) {
                const int tb_ = row[p0 - 1];
                if (tb_ < G) { fresh = false; prev_model = sg[tb_ << rs].model; }
            }
            auto enter = [&](ScanState &s) {
                if (fresh) {
                    start_queue(tab, s, q0);
                } else {
                    s.q = q0; s.d = sq[q0].d; s.prev = prev_model;   // mid-queue: previous slot's model
                }
            };
            // ---- pass 1: chunk aggregate from a zero (or reset) state
            ScanState s;
            enter(s);
            if (!fresh) { s.A = 0.0; s.B = 0.0f; }
            bool reset = fresh;
            for (int pos = p0; pos < p1; ++pos) {
                const int tok = row[pos];
                if (tok >= G) {
                    start_queue(tab, s, s.q + 1 < Q ? s.q + 1 : Q - 1);
                    reset = true;
                    continue;
                }
                double wt;
                float V;
                GRec g;
                group_slot(tab, s, tok, wt, V, g);
            }
            // ---- segmented inclusive scan of (reset, A, B) over the lanes
            bool f = reset || p0 >= T;
            double a = p0 >= T ? 0.0 : s.A;
            float b = p0 >= T ? 0.0f : s.B;
            if (p0 >= T) f = false;                            // empty chunk: identity
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int f2 = __shfl_up_sync(0xFFFFFFFFu, (int)f, o);
                const double a2 = __shfl_up_sync(0xFFFFFFFFu, a, o);
                const float b2 = __shfl_up_sync(0xFFFFFFFFu, b, o);
                if (lane >= o && !f) { a = __dadd_rn(a2, a); b = __fadd_rn(b2, b); f = f2 != 0; }
            }
            const double ain = __shfl_up_sync(0xFFFFFFFFu, a, 1);   // exclusive: state at chunk start
            const float bin = __shfl_up_sync(0xFFFFFFFFu, b, 1);
            // ---- pass 2: emit the chunk's slots from the true start state
            enter(s);
            if (!fresh) { s.A = ain; s.B = bin; }
            double S2 = 0.0, num = 0.0;
            int over = 0;
            for (int pos = p0; pos < p1; ++pos) {
                const int tok = row[pos];
                if (tok >= G) {
                    start_queue(tab, s, s.q + 1 < Q ? s.q + 1 : Q - 1);
                    continue;
                }
                double wt;
                float V;
                GRec g;
                group_slot(tab, s, tok, wt, V, g);
                const double slack = __dsub_rn(g.slo, wt);
                const float sd = slot_sd(V);
                bool clamped;
                const float v = slot_v(slack, sd, zc, clamped);
                if constexpr (SCORE) {
                    S2 = __dsub_rn(S2, slack);
                    num = fma((double)g.n, (double)v, num);
                    over += v > alpha;
                }
                if (any_out) {
                    float *o = tile + (size_t)tok * kWidePad + warp;
                    o[0] = (float)wt;
                    o[(size_t)G * kWidePad] = sd;
                    o[(size_t)2 * G * kWidePad] = v;
                }
            }
            if constexpr (SCORE) {
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    S2 = __dadd_rn(S2, __shfl_xor_sync(0xFFFFFFFFu, S2, o));
                    num = __dadd_rn(num, __shfl_xor_sync(0xFFFFFFFFu, num, o));
                    over += __shfl_xor_sync(0xFFFFFFFFu, over, o);
                }
                const float s1 = (float)(num / den);
                const float s2 = (float)S2;
                if (lane == 0) {
                    if (p.s1) p.s1[loc] = s1;
                    if (p.s2) p.s2[loc] = s2;
                    if (p.n_over) p.n_over[loc] = over;
                }
                const uint64_t key = make_key(s1, s2);
                const int64_t c = cd.first + loc;
                if (better(key, c, bkey, bidx)) { bkey = key; bidx = c; }
            }
        }
        __syncthreads();                                       // tile complete, rows consumed
        if (any_out) {
            const int nv = (int)min((int64_t)kWideCands, count - c0);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                float *const base = a == 0 ? p.wt : (a == 1 ? p.sd : p.vo);
                if (!base) continue;
                for (int g = tid; g < G; g += 256) {
                    const float *src = tile + ((size_t)a * G + g) * kWidePad;
                    float *dst = base + (int64_t)g * ldo + c0;
                    if (nv == kWideCands && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
                        __stcs(reinterpret_cast<float4 *>(dst), make_float4(src[0], src[1], src[2], src[3]));
                        __stcs(reinterpret_cast<float4 *>(dst) + 1, make_float4(src[4], src[5], src[6], src[7]));
                    } else {
                        for (int k = 0; k < nv; ++k) dst[k] = src[k];
                    }
                }
            }
            __syncthreads();                                   // tile free for the next batch
        }
    }
    if constexpr (SCORE) {
        if (p.out_rec) block_grid_argmin(p, bkey, bidx);
    }
}

// ---- host -------------------------------------------------------------------
static size_t a16w(size_t x) { return (x + 15) & ~size_t(15); }

template <int KIND, bool SCORE>
static cudaError_t launch_wide_t(ScanParams p, cudaStream_t st) {
    const Dims &dm = p.dm;
    auto plan = [&](int rs) {
        size_t off = 0;
        p.rep_shift = rs;
        p.off_grec = (int)off; off = a16w(off + ((size_t)dm.G << rs) * sizeof(GRec));
        p.off_ab = (int)off;   off = a16w(off + ((size_t)dm.D * dm.G << rs) * sizeof(double2));
        p.off_q = (int)off;    off = a16w(off + (size_t)dm.Q * sizeof(QRec));
        p.off_tr = (int)off;   off = a16w(off + ((size_t)dm.D * 2 * dm.M * dm.M << 4) * sizeof(double));
        p.off_scratch = (int)off; off = a16w(off + (size_t)kWideCands * ((dm.T + 7) & ~7) * 2);
        p.off_stage = (int)off;
        if (p.wt || p.sd || p.vo) off += (size_t)3 * dm.G * kWidePad * 4;
        return off;
    };
    auto kern = wide_kernel<KIND, SCORE>;
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    // the most replication that fits (env QLM_WIDE_RS pins it for A/B timing)
    const int env_rs = env_cached("QLM_WIDE_RS", -1);
    size_t off = 0;
    int rs = env_rs >= 0 ? env_rs : 0;   // replication measured: no gain (latency-bound), so none by default
    for (; rs >= 0; --rs) {
        off = plan(rs);
        if (off + fa.sharedSizeBytes <= (size_t)optin || env_rs >= 0) break;
    }
    if (rs < 0) rs = 0, off = plan(0);
    if (off + fa.sharedSizeBytes > (size_t)optin) return cudaErrorNotSupported;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)off)) != cudaSuccess)
        return e;
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 256, off);
    if (nb < 1) return cudaErrorNotSupported;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = (p.cd.count + kWideCands - 1) / kWideCands;
    const int64_t maxg = (int64_t)sms * nb;
    if (grid > maxg) grid = maxg;
    if (grid > p.max_blocks) grid = p.max_blocks;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 256, off, st>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

// Warp-per-candidate path: rows word-interleaved (two-phase chunks) or
// EXPLICIT u16.  cudaErrorNotSupported when it does not apply.
cudaError_t launch_wide(const ScanParams &p, cudaStream_t st) {
    if (override_on(QLM_OVERRIDE_NO_WIDE)) return cudaErrorNotSupported;
    if (p.cd.first_from || p.cd.count < 1) return cudaErrorNotSupported;
    const bool ilv = p.cd.kind == KIND_ILV;
    const bool ex16 = p.cd.kind == QLM_CAND_EXPLICIT && p.cd.tb == 2;
    const bool nb16 = p.cd.kind == QLM_CAND_NEIGHBOR && p.cd.tb == 2;
    if (!ilv && !ex16 && !nb16) return cudaErrorNotSupported;
    const bool score = p.s1 || p.s2 || p.n_over || p.out_rec;
    if (ilv) return score ? launch_wide_t<KIND_ILV, true>(p, st) : launch_wide_t<KIND_ILV, false>(p, st);
    if (nb16)
        return score ? launch_wide_t<QLM_CAND_NEIGHBOR, true>(p, st) : launch_wide_t<QLM_CAND_NEIGHBOR, false>(p, st);
    return score ? launch_wide_t<QLM_CAND_EXPLICIT, true>(p, st) : launch_wide_t<QLM_CAND_EXPLICIT, false>(p, st);
}

}  // namespace qlm
