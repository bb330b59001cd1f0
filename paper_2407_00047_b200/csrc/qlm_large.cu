// qlm_large.cu -- score + argmin (a2-a5, a7) over 16-bit candidate rows that
// fy_rows_kernel materialised word-interleaved (the second phase of the
// large-T RANDOM path, T > 256: C5), for problems with one device type (D = 1).
//
// Thread per candidate, as qlm_ws2.cu's consumer and with its slot arithmetic
// (so scores and argmin are bit-identical to the other Gaussian kernels, R22):
//  * separators are relabelled in row order (the k-th becomes token G + k, the
//    start of queue k + 1) and are table entries like groups: {slo = 1e30, a =
//    the queue's backlog mean, b = its variance, transition state = the
//    queue's start state}; keep = 0 resets A' = fma(wt, 0, a) and B, so a slot
//    is straight-line code (no divergent separator branch);
//  * V accumulates in fp32; the rare unclamped slots (|z| < z_clamp) go to a
//    per-lane FIFO {slack, sd, n} whose Phi-bar terms are added in row order
//    at a flush (every two row words, when any lane's FIFO is half full);
//  * records live in shared memory with 2^r replicas (lane l reads copy
//    l mod 2^r) -- a 1000-group table cannot take the 8 / 16 replicas of the
//    small-G kernel, so some bank conflicts remain; the transition table has
//    16 replicas.
// Row words come straight from global memory (one coalesced 128-B load per
// warp per two slots), kPf = 8 words in flight per lane (the 128-B requests
// of a warp hit scattered DRAM pages: latency, not bandwidth, bounds them).
#include "qlm_argmin.cuh"
#include "qlm_device.cuh"
#include "qlm_launch.h"

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

namespace qlm {
namespace lg {

constexpr int kWPC = 2;                  // row words (2 slots each) per FIFO check
constexpr int kPend = 4 + 2 * kWPC;      // FIFO entries per lane (16 B each)
constexpr int kTrRep = 16;               // transition replicas (8-B entries)
#ifndef LG_PF
#define LG_PF 8
#endif
constexpr int kPf = LG_PF;               // row words in flight per lane

struct Params {
    ScanParams p;
    int r0s, r1s;                        // log2 replicas of the record halves
    int off_rec0, off_rec1, off_tr, off_pend;
    float oc;                            // 1 if a clamped late slot (v = 1) counts in n_over
};

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float2 lds64v(uint32_t a) {
    float2 v;
    asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds64f(uint32_t a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

struct Acc {
    double A, S2, acc2;      // running mean work (Eq. 10), S2 (R11), unclamped S1 terms
    float B;                 // running variance (R22: fp32)
    float acc1, over;        // clamped S1 terms (exact integers: sum n_i < 2^24), n_over
    uint32_t pq;             // next free FIFO entry (shared address)
};

struct Ctx {
    uint32_t rb0, rb1, tb;   // lane's record-half / transition bases
    uint32_t s0, s1;         // record strides (bytes per token)
    int G, R;                // groups, transition row stride (entries)
    float zc, oc;
    int T;                   // QLM_BOUNDS limits: record entries, transition table end,
    uint32_t tr_hi, pq_hi;   // end of the lane's FIFO
};

// One slot (R1-R9, R11, R22), token `tok` of the row in row order.
template <int SCORE>
__device__ __forceinline__ void slot(const Ctx &c, int tok, uint32_t &prow, int &gq, Acc &a) {
    int ix, kh;
    asm("{\n.reg .pred p;\nsetp.ge.s32 p, %3, %4;\nselp.b32 %0, %2, %3, p;\n"
        "selp.b32 %1, 0, 0x3FF00000, p;\n@p add.s32 %2, %2, 1;\n}\n"
        : "=r"(ix), "=r"(kh), "+r"(gq) : "r"(tok), "r"(c.G));
    QLM_CHECK(ix >= 0 && ix < c.T);
    const float4 r0 = lds128(c.rb0 + (uint32_t)ix * c.s0);      // {a, hi word of slo, n}
    const float2 r1 = lds64v(c.rb1 + (uint32_t)ix * c.s1);      // {b, 128 * state}
    const uint32_t xs = (uint32_t)__float_as_int(r1.y);
    QLM_CHECK(prow + xs + 8 <= c.tr_hi);
    const double tr = lds64f(prow + xs);                         // row of the state before
    prow = c.tb + xs * (uint32_t)c.R;
    const double aw = __hiloint2double(__float_as_int(r0.y), __float_as_int(r0.x));
    const double slo = __hiloint2double(__float_as_int(r0.z), 0);
    const double keep = __hiloint2double(kh, 0);
    // Eq. 10 in the oracle's order: wt = A + (tail + swap); A' = wt + a; a
    // separator (keep = 0) restarts A at its queue's backlog mean, B at its variance
    const double wt = __dadd_rn(a.A, tr);
    a.A = __fma_rn(wt, keep, aw);
    const float V = a.B;                                         // exclusive (R5)
    a.B = __fadd_rn(kh ? a.B : 0.0f, r1.x);
    // violation probability (R8/R9) and scores (R11)
    const double slack = __dsub_rn(slo, wt);
    const float sf = (float)slack;
    const float sd = sqrt_approx(V);
    const bool clamped = fabsf(sf) >= c.zc * sd;                 // R9: exact for V = 0
    const float v = sf < 0.0f ? 1.0f : 0.0f;
    if (clamped) {
        a.acc1 = fmaf(r0.w, v, a.acc1);                          // separators: n = 0
        if constexpr (SCORE > 1) a.over = fmaf(v, c.oc, a.over);
    }
    a.S2 = __fma_rn(slack, -keep, a.S2);                         // S2 += wt - slo (groups only)
    if (!clamped) {                                              // exact Phi-bar at the flush
        QLM_CHECK(a.pq < c.pq_hi);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a.pq), "f"(sf), "f"(sd), "f"(r0.w),
                     "f"(0.0f) : "memory");
        a.pq += 32 * 16;
    }
}

// Deferred slots in FIFO (row) order.
template <int SCORE>
__device__ __forceinline__ void flush(uint32_t pq0, float alpha, Acc &a) {
    const int n = (int)((a.pq - pq0) >> 9);
    const int maxn = (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)n);
    for (int i = 0; i < maxn; ++i) {
        if (i < n) {
            float sf, sd, nf, pad;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(sf), "=f"(sd), "=f"(nf), "=f"(pad) : "r"(pq0 + i * 512));
            const float v = phibar(sf * rcp_approx(sd));
            a.acc2 = __fma_rn((double)nf, (double)v, a.acc2);
            if constexpr (SCORE > 1) a.over += v > alpha ? 1.0f : 0.0f;
        }
    }
    a.pq = pq0;
}

template <int SCORE>
__global__ void __launch_bounds__(512, 1) large_kernel(const __grid_constant__ Params w) {
    extern __shared__ __align__(16) uint8_t smem[];
    const ScanParams &p = w.p;
    const int tid = threadIdx.x, lane = tid & 31;
    const int G = p.dm.G, T = p.dm.T, M = p.dm.M;

    // ---- tables -> smem: record halves per token value ix (groups 0..G-1,
    // G + k = separator k = start of queue k + 1), R0 / R1 replicas:
    //   half 0 (16 B): {a (f64), hi word of slo (its low word is 0), n (f32)}
    //   half 1 (8 B):  {b (f32), x = 128 * transition state}
    // states s < M: after a group of model s; M + r: queue start on resident r
    // with nothing running (R4); a declared backlog starts in the resident's
    // model state (R12)
    const int R0 = 1 << w.r0s, R1 = 1 << w.r1s;
    const int rms = w.r0s > w.r1s ? w.r0s : w.r1s;
    for (int i = tid; i < (T << rms); i += blockDim.x) {
        const int ix = i >> rms, r = i & ((1 << rms) - 1);
        double aw, slo;
        float b, nf;
        int st;
        if (ix < G) {
            const GRec g = p.tb.grec[ix];
            const double2 ab = p.tb.ab[ix];                      // device row 0 (D = 1)
            slo = g.slo; aw = ab.x; b = (float)ab.y; nf = (float)g.n; st = g.model;
        } else {
            const QRec q = p.tb.qrec[ix - G + 1];
            slo = 1e30; aw = q.bmean; b = (float)q.bvar; nf = 0.0f;
            st = q.backlog ? q.r : M + q.r;
        }
        if (r < R0)
            *reinterpret_cast<float4 *>(smem + w.off_rec0 + ((size_t)ix * R0 + r) * 16) =
                make_float4(__int_as_float(__double2loint(aw)), __int_as_float(__double2hiint(aw)),
                            __int_as_float(__double2hiint(slo)), nf);
        if (r < R1)
            *reinterpret_cast<float2 *>(smem + w.off_rec1 + ((size_t)ix * R1 + r) * 8) =
                make_float2(b, __int_as_float(st * kTrRep * 8));
    }
    // transitions [2M][M][16 replicas] f64 + M zero entries: row = state before
    // the slot, column = the slot's state, tail of the model ahead on a change
    // (R1) + swap (R2); a separator's column (>= M) reads the next row or the
    // padding -- finite values that keep = 0 discards
    const int ntr = M * (2 * M + 1) * kTrRep;
    for (int i = tid; i < ntr; i += blockDim.x) {
        const int e = i / kTrRep, col = e % M, row = e / M;
        double v = 0.0;
        if (row < 2 * M) {
            const int from = row < M ? row : row - M;
            const double sw = p.tb.swap[from * M + col];
            const double tl = (row < M && col != row) ? p.tb.tail[row] : 0.0;
            v = __dadd_rn(tl, sw);
        }
        reinterpret_cast<double *>(smem + w.off_tr)[i] = v;
    }
    __syncthreads();

    const Cand cd = p.cd;
    const int64_t count = cd.count, first = cd.first;
    Ctx c;
    c.rb0 = su32(smem + w.off_rec0) + (uint32_t)(lane & (R0 - 1)) * 16u;
    c.rb1 = su32(smem + w.off_rec1) + (uint32_t)(lane & (R1 - 1)) * 8u;
    c.tb = su32(smem + w.off_tr) + (uint32_t)(lane & (kTrRep - 1)) * 8u;
    c.s0 = 16u * R0;
    c.s1 = 8u * R1;
    c.G = G;
    c.R = M;
    c.zc = p.zc;
    c.oc = w.oc;
    c.T = T;
    c.tr_hi = su32(smem + w.off_tr) + (uint32_t)ntr * 8u;
    const float alpha = p.alpha;
    const double den = *p.tb.den;
    const QRec q0 = p.tb.qrec[0];
    const double q0mean = q0.bmean;
    const float q0var = (float)q0.bvar;
    const uint32_t prow0 = c.tb + (uint32_t)(q0.backlog ? q0.r : M + q0.r) * (kTrRep * 8u) * (uint32_t)M;
    const uint32_t pq0 = su32(smem + w.off_pend) + (uint32_t)(tid >> 5) * (kPend * 512u) + lane * 16u;
    const uint32_t pqlim = pq0 + (kPend - 2 * kWPC) * 512u;    // room until the next check
    c.pq_hi = pq0 + kPend * 512u;
    const int nw = (T + 1) >> 1, nfull = T >> 1;
    const int64_t ld = cd.stride;                                // words are [nw][stride] u32
    uint64_t bkey = ~0ull;
    int64_t bidx = -1;
    const int64_t nbatch = (count + 31) >> 5;
    const int64_t nwarp = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t bt = (int64_t)blockIdx.x * (blockDim.x >> 5) + (tid >> 5); bt < nbatch; bt += nwarp) {
        const int64_t loc = (bt << 5) + lane;
        // lanes past the end walk the last valid row (convergent loop; result dropped)
        const uint32_t *r32 = reinterpret_cast<const uint32_t *>(cd.rows) + (loc < count ? loc : count - 1);
        // ring of kPf row words per lane in registers: word wi + k sits in
        // ring[k] and is refilled with word wi + kPf + k as soon as it is used
        uint32_t ring[kPf];
#pragma unroll
        for (int k = 0; k < kPf; ++k) ring[k] = k < nw ? __ldcs(r32 + (int64_t)k * ld) : 0u;
        Acc a;
        a.A = q0mean; a.B = q0var;
        a.S2 = 0.0; a.acc2 = 0.0; a.acc1 = 0.0f; a.over = 0.0f; a.pq = pq0;
        uint32_t prow = prow0;
        int gq = G;
        int wi = 0;
        for (; wi + kPf <= nfull; wi += kPf) {
#pragma unroll
            for (int k = 0; k < kPf; ++k) {
                const uint32_t u = ring[k];
                ring[k] = wi + kPf + k < nw ? __ldcs(r32 + (int64_t)(wi + kPf + k) * ld) : 0u;
                slot<SCORE>(c, (int)(u & 0xFFFFu), prow, gq, a);
                slot<SCORE>(c, (int)(u >> 16), prow, gq, a);
                if (k & 1)
                    if (__any_sync(0xFFFFFFFFu, a.pq > pqlim)) flush<SCORE>(pq0, alpha, a);
            }
        }
#pragma unroll
        for (int k = 0; k < kPf; ++k) {                          // the remaining full words
            if (wi + k < nfull) {
                slot<SCORE>(c, (int)(ring[k] & 0xFFFFu), prow, gq, a);
                slot<SCORE>(c, (int)(ring[k] >> 16), prow, gq, a);
                if (k & 1)
                    if (__any_sync(0xFFFFFFFFu, a.pq > pqlim)) flush<SCORE>(pq0, alpha, a);
            } else if (wi + k == nfull && (T & 1)) {             // last slot; the pad half is not a token
                slot<SCORE>(c, (int)(ring[k] & 0xFFFFu), prow, gq, a);
            }
        }
        flush<SCORE>(pq0, alpha, a);
        if (loc < count) {
            const float s1 = (float)(((double)a.acc1 + a.acc2) / den);   // R11
            const float s2 = (float)a.S2;
            if (p.s1) p.s1[loc] = s1;
            if (p.s2) p.s2[loc] = s2;
            if (p.n_over) p.n_over[loc] = (int)a.over;
            const uint64_t key = make_key(s1, s2);
            const int64_t cc = first + loc;
            if (better(key, cc, bkey, bidx)) { bkey = key; bidx = cc; }
        }
    }
    if (p.out_rec) block_grid_argmin(p, bkey, bidx);            // all warps take part
}

static size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

static size_t plan(Params &w, int warps, int r0s, int r1s) {
    const Dims &dm = w.p.dm;
    size_t off = 0;
    w.r0s = r0s; w.r1s = r1s;
    w.off_tr = (int)off;   off = a16(off + (size_t)dm.M * (2 * dm.M + 1) * kTrRep * 8);
    w.off_rec0 = (int)off; off = a16(off + ((size_t)dm.T << r0s) * 16);
    w.off_rec1 = (int)off; off = a16(off + ((size_t)dm.T << r1s) * 8);
    w.off_pend = (int)off; off = a16(off + (size_t)warps * kPend * 512);
    return off;
}

template <typename K>
static size_t opt_in(K kern) {
    static std::mutex mu;
    static std::unordered_map<uint64_t, size_t> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t key = ((uint64_t)(uintptr_t)reinterpret_cast<const void *>(kern) << 8) ^ (uint64_t)dev;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    size_t m = 0;
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess && optin > (int)fa.sharedSizeBytes) {
        m = (size_t)optin - fa.sharedSizeBytes;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m) != cudaSuccess) m = 0;
    }
    cudaGetLastError();
    cache[key] = m;
    return m;
}

template <int SCORE>
static cudaError_t launch_t(const ScanParams &p0, cudaStream_t st) {
    auto kern = large_kernel<SCORE>;
    const size_t lim = opt_in(kern);
    if (!lim) return cudaErrorNotSupported;
    Params w;
    memset(&w, 0, sizeof w);
    w.p = p0;
    w.oc = 1.0f > p0.alpha ? 1.0f : 0.0f;
    // replicas of the record halves: the most that fit next to 16 warps'
    // FIFOs (QLM_LARGE_R0 / _R1 = log2 replicas, read once per process, pin
    // them for A/B timing; measured: 4 x 4 and 8 x 4 within 1 %)
    const int warps = 16;
    int r0 = env_cached("QLM_LARGE_R0", 3), r1 = env_cached("QLM_LARGE_R1", 4);
    size_t smem = plan(w, warps, r0, r1);
    while (smem > lim && (r0 > 0 || r1 > 0)) {
        if (r1 >= r0 && r1 > 0) --r1; else --r0;
        smem = plan(w, warps, r0, r1);
    }
    if (smem > lim) return cudaErrorNotSupported;
    const int64_t nbatch = (p0.cd.count + 31) / 32;
    int64_t grid = sm_count();
    const int64_t need = (nbatch + warps - 1) / warps;
    if (grid > need) grid = need;
    if (grid > p0.max_blocks) grid = p0.max_blocks;
    if (grid < 1) grid = 1;
    qlog(1, "large_kernel<score=%d> count=%lld grid=%lld replicas=%d,%d smem=%zu", SCORE,
         (long long)p0.cd.count, (long long)grid, 1 << w.r0s, 1 << w.r1s, smem);
    kern<<<(unsigned)grid, 32 * warps, smem, st>>>(w);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace lg

// Score-only pass over word-interleaved 16-bit rows (KIND_ILV) for D = 1;
// cudaErrorNotSupported -> the caller uses the general scan kernel.
cudaError_t launch_large(const ScanParams &p, cudaStream_t st) {
    if (p.cd.kind != KIND_ILV || p.cd.tb != 2 || p.dm.D != 1 || p.dm.M > 6 || !p.slo_hi_only ||
        p.cd.first_from || p.cd.count < 1 || p.wt || p.sd || p.vo || !(p.s1 || p.s2 || p.n_over || p.out_rec))
        return cudaErrorNotSupported;
    if (override_on(QLM_OVERRIDE_NO_LARGE)) return cudaErrorNotSupported;
    return p.n_over ? lg::launch_t<2>(p, st) : lg::launch_t<1>(p, st);
}

}  // namespace qlm
