// qlm_device.cuh -- device data layout and primitives of libqlm (sm_100a).
//
// Shares nothing with oracle/: this is the product path.  Citations:
// "P:Lx" = PAPER.md line x; R-numbers = readings in DESIGN.md.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "qlm.h"

// Debug bounds checks (build with -DQLM_BOUNDS, tools/gpu/s3_bounds.sh): a
// failed check prints its condition and traps, so the calling test fails.
#ifdef QLM_BOUNDS
#include <cstdio>
#define QLM_CHECK(c)                                                                          \
    do {                                                                                      \
        if (!(c)) {                                                                           \
            printf("QLM_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,     \
                   (int)blockIdx.x, (int)threadIdx.x, #c);                                   \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define QLM_CHECK(c) do { } while (0)
#endif

namespace qlm {

// ---- derived tables in HBM (built on the device by build_tables_kernel) ----
// Per group, device-independent: deadline, request count, model (16 B).
struct alignas(16) GRec {
    double slo;     // slo_i (Eq. 8)
    int32_t n;      // n_i
    int32_t model;  // m_i (Eq. 7)
};
// Per queue (32 B): backlog (R12), device row, resident model (R4).
struct alignas(16) QRec {
    double bmean, bvar;
    int32_t d, r, backlog, pad;
};

struct Dims {
    int G, Q, D, M, T;      // T = G + Q - 1 tokens per row
    int K, n_tables, shift; // MC tables; shift = 32 - log2(K)
};

struct Tables {             // device pointers, one allocation
    GRec *grec;             // [G]
    double2 *ab;            // [D][G]  {n mu / Theta, n var / Theta^2}  (Eq. 2/3)
    QRec *qrec;             // [Q]
    double *tail;           // [D][M]  P + max_out eps d  (Eq. 1/4, R3)
    double *swap;           // [D][M][M]
    double *theta;          // [D][M]
    int32_t *dist;          // [G]
    uint16_t *len;          // [n_tables][K]
    double *den;            // [1] sum_i n_i
};

// Internal candidate kind: rows materialised word-interleaved by fy_rows_kernel
// (word w of chunk-local candidate l at rows[(w * stride + l) * 4]).
constexpr int KIND_ILV = 7;

struct Cand {               // device view of qlm_candidates
    int kind, tb;
    const uint8_t *rows;
    int64_t stride;
    uint64_t seed;
    int64_t first, count;
    const qlm_record *first_from;
    int moves;              // NEIGHBOR: transpositions per candidate (R18)
};

// ---- Philox4x32-10 (Salmon et al. SC'11) ------------------------------------
__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

__device__ __forceinline__ uint32_t pick4(uint4 w, int k) {
    return k == 0 ? w.x : k == 1 ? w.y : k == 2 ? w.z : w.w;
}

// Candidate-row Philox stream (R10): key = seed, counter = (i/4, c_lo, c_hi, 'QLM\0').
constexpr uint32_t kRowTag = 0x514C4D00u;
// MC stream (R13): key = mc_seed, counter = (r/4, group, trial, 'MC\0\0').
constexpr uint32_t kMcTag = 0x4D430000u;
// NEIGHBOR stream (R18): key = seed, counter = (m/2, c_lo, c_hi, 'NBHR').
constexpr uint32_t kNbrTag = 0x4E424852u;

// ---- per-thread Fisher-Yates scratch in shared memory ----------------------
// Element i of thread `tid` lives in 32-bit word (i / EPW) * blk + tid, byte
// lane i % EPW: a warp touching any elements hits 32 distinct banks.
// Byte offset = 4 (w blk + tid) + (i mod EPW) sizeof(TOK) with w = i / EPW,
// written as i sizeof(TOK) + w (4 blk - 4) + 4 tid: one shift and one
// multiply-add per element (4 tid is loop-invariant).
template <typename TOK>
__device__ __forceinline__ TOK *fy_elem(uint8_t *base, int i, int blk, int tid) {
    constexpr int EPW = 4 / (int)sizeof(TOK);
    const unsigned u = (unsigned)i;
    return reinterpret_cast<TOK *>(base + 4u * (unsigned)tid +
                                   (u * (unsigned)sizeof(TOK) + (u / EPW) * (4u * (unsigned)blk - 4u)));
}

// Forward Fisher-Yates materialised in place: after the call, element s of
// the thread's scratch row holds token s.  Used by the two-phase scan (generate, then walk 4 tokens/load).
template <typename TOK>
__device__ __forceinline__ void fy_materialise(uint8_t *scratch, int blk, int tid, int T,
                                               uint64_t seed, uint64_t c) {
    constexpr int EPW = 4 / (int)sizeof(TOK);
    uint32_t *w32 = reinterpret_cast<uint32_t *>(scratch);
    const int nw = (T + EPW - 1) / EPW;
    for (int w = 0; w < nw; ++w)
        w32[w * blk + tid] = EPW == 4 ? 0x03020100u + 0x04040404u * (uint32_t)w
                                      : 0x00010000u + 0x00020002u * (uint32_t)w;
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const uint32_t clo = (uint32_t)c, chi = (uint32_t)(c >> 32);
    // Position i is final after step i and never read again (later steps touch
    // positions > i only), so finals are packed in a register and written one
    // 32-bit word at a time instead of one sub-word store per step.
    uint32_t fin = 0;
    auto step = [&](int i, int j) {
        TOK *pi = fy_elem<TOK>(scratch, i, blk, tid);
        TOK *pj = fy_elem<TOK>(scratch, j, blk, tid);
        const TOK ti = *pi, tj = *pj;
        *pj = ti;
        const int lanepos = i % EPW;
        fin |= (uint32_t)tj << (lanepos * 8 * sizeof(TOK));
        if (lanepos == EPW - 1) {
            w32[(i / EPW) * blk + tid] = fin;
            fin = 0;
        }
    };
    if (T <= 256) {                 // R10: two 16-bit draws per word, 8 per Philox block
        for (int i0 = 0; i0 < T - 1; i0 += 8) {
            const uint4 wd = philox10(make_uint4((uint32_t)(i0 >> 3), clo, chi, kRowTag), key);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = i0 + k;
                if (i >= T - 1) break;
                const uint32_t w = pick4(wd, k >> 1);
                const uint32_t u = (k & 1) ? (w >> 16) : (w & 0xFFFFu);
                step(i, i + (int)((u * (uint32_t)(T - i)) >> 16));
            }
        }
    } else {                        // 32-bit draws, 4 per Philox block
        for (int i0 = 0; i0 < T - 1; i0 += 4) {
            const uint4 wd = philox10(make_uint4((uint32_t)(i0 >> 2), clo, chi, kRowTag), key);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + k;
                if (i >= T - 1) break;
                step(i, i + (int)__umulhi(pick4(wd, k), (uint32_t)(T - i)));
            }
        }
    }
    // position T-1 is final (it holds whatever the last swap left there)
    {
        const int i = T - 1;
        const TOK last = *fy_elem<TOK>(scratch, i, blk, tid);
        fin |= (uint32_t)last << ((i % EPW) * 8 * sizeof(TOK));
        // keep the word's positions > T-1 as they were (padding is never read as tokens)
        w32[(i / EPW) * blk + tid] = fin;
    }
}

// Walk a materialised scratch row: one 32-bit load per EPW tokens.
template <typename TOK, typename F>
__device__ __forceinline__ void tokens_scratch(const uint8_t *scratch, int blk, int tid, int T,
                                               F &&f) {
    constexpr int EPW = 4 / (int)sizeof(TOK);
    const uint32_t *w32 = reinterpret_cast<const uint32_t *>(scratch);
    for (int s0 = 0; s0 < T; s0 += EPW) {
        const uint32_t w = w32[(s0 / EPW) * blk + tid];
#pragma unroll
        for (int k = 0; k < EPW; ++k) {
            if (s0 + k >= T) break;
            f(EPW == 4 ? (int)((w >> (8 * k)) & 0xFFu) : (int)((w >> (16 * k)) & 0xFFFFu));
        }
    }
}

// ---- NEIGHBOR rows (R18): base row with k Philox-drawn transpositions -------
// Move m of candidate c swaps positions (i_m, j_m) = (mulhi(u0, T), mulhi(u1, T)),
// (u0, u1) = words 2(m%2), 2(m%2)+1 of Philox(key = seed, ctr = (m/2, c, 'NBHR')).
__device__ __forceinline__ void nbr_moves(const Cand &cd, int T, uint64_t c, int *mi, int *mj) {
    const uint2 key = make_uint2((uint32_t)cd.seed, (uint32_t)(cd.seed >> 32));
    uint4 wd = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int m = 0; m < QLM_MAX_MOVES; ++m) {
        if (m >= cd.moves) break;
        if ((m & 1) == 0) wd = philox10(make_uint4((uint32_t)(m >> 1), (uint32_t)c, (uint32_t)(c >> 32), kNbrTag), key);
        mi[m] = (int)__umulhi((m & 1) ? wd.z : wd.x, (uint32_t)T);
        mj[m] = (int)__umulhi((m & 1) ? wd.w : wd.y, (uint32_t)T);
    }
}

template <typename TOK>
__device__ __forceinline__ int base_token(const Cand &cd, int p) {
    return (int)__ldg(reinterpret_cast<const TOK *>(cd.rows) + p);
}

// Streaming generator for one thread: the row differs from the base row in at
// most 2k positions; they are resolved once (apply the k swaps to the touched
// positions only) and sorted, then the row streams from the base row (all
// lanes read the same position: a broadcast) with the touched values spliced
// in.  No per-thread row scratch, so any T runs at full occupancy.
template <typename TOK, typename F>
__device__ __forceinline__ void tokens_neighbor(const Cand &cd, int T, uint64_t c, F &&f) {
    int mi[QLM_MAX_MOVES], mj[QLM_MAX_MOVES];
    nbr_moves(cd, T, c, mi, mj);
    int P[2 * QLM_MAX_MOVES], V[2 * QLM_MAX_MOVES];
    int n = 0;
    auto slot = [&](int pos) {
        for (int x = 0; x < n; ++x)
            if (P[x] == pos) return x;
        P[n] = pos;
        V[n] = base_token<TOK>(cd, pos);
        return n++;
    };
    for (int m = 0; m < cd.moves; ++m) {
        const int xi = slot(mi[m]), xj = slot(mj[m]);
        const int t = V[xi]; V[xi] = V[xj]; V[xj] = t;
    }
    for (int a = 1; a < n; ++a) {                       // insertion sort by position
        const int pa = P[a], va = V[a];
        int b = a - 1;
        while (b >= 0 && P[b] > pa) { P[b + 1] = P[b]; V[b + 1] = V[b]; --b; }
        P[b + 1] = pa; V[b + 1] = va;
    }
    int idx = 0, nextp = n > 0 ? P[0] : T;
    for (int pos = 0; pos < T; ++pos) {
        int tok = base_token<TOK>(cd, pos);
        if (pos == nextp) {
            tok = V[idx];
            ++idx;
            nextp = idx < n ? P[idx] : T;
        }
        f(tok);
    }
}

// EXPLICIT rows: 16-byte vector loads of the thread's own row.
template <typename TOK, typename F>
__device__ __forceinline__ void tokens_explicit(const uint8_t *row, int T, F &&f) {
    constexpr int PER = 16 / (int)sizeof(TOK);
    for (int s0 = 0; s0 < T; s0 += PER) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(row + (size_t)s0 * sizeof(TOK)));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            if (s0 + k >= T) break;
            const int tok = sizeof(TOK) == 1 ? (int)((w[k >> 2] >> ((k & 3) * 8)) & 0xFFu)
                                              : (int)((w[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu);
            f(tok);
        }
    }
}

// ENUM rows: Lehmer unranking in lexicographic order, T <= 20.
template <typename F>
__device__ __forceinline__ void tokens_enum(uint64_t c, int T, F &&f) {
    uint32_t avail = T >= 32 ? 0xFFFFFFFFu : ((1u << T) - 1u);
    uint64_t fact = 1;
    for (int k = 2; k < T; ++k) fact *= (uint64_t)k;   // (T-1)!
    for (int pos = 0; pos < T; ++pos) {
        const int rem = T - 1 - pos;
        const uint64_t k = c / fact;
        c -= k * fact;
        uint32_t a = avail;
        for (uint64_t s = 0; s < k; ++s) a &= a - 1u;   // drop the k lowest available
        const int tok = __ffs((int)a) - 1;
        avail &= ~(1u << tok);
        if (rem > 0) fact /= (uint64_t)rem;
        f(tok);
    }
}

// ---- one pass of the Eq. 2/3/10 recurrence over a row (R1-R7, R12) ---------
// Shared-memory tables of a scan block.  Group records are replicated
// (1 << rs) times and interleaved so that lane l reads copy l % (1 << rs):
// with 8 copies a warp's random 16-B reads are bank-conflict free.
//
// Transition table (Eq. 9/10, R1/R2/R4): rows p' in [0, 2M) per device:
//   p' <  M : the previous group ran model p'   -> (m != p' ? tail[d][p'] : 0) + swap[d][p'][m]
//   p' >= M : nothing has run yet on resident r = p' - M (no backlog)
//                                               -> 0 + swap[d][r][m]
// (one fp64 transition term, R2/R3), so every slot does A = A + c with no
// branch; c = 0 when the model does not change, and A + 0.0 == A keeps the
// arithmetic operation-for-operation identical to the sequential definition.
struct SlotTables {
    const GRec *sg;        // [G << rs]        {slo, n, model}
    const double2 *sab;    // [(D*G) << rs]    {n mu / Theta, n var / Theta^2}
    const double *str;     // [D * 2M * M]     tail part + swap part (one transition term)
    const QRec *sq;        // [Q]
    int G, Q, M, rs, rl;   // rl = lane & ((1 << rs) - 1)
    int trs, trl;          // transition table: 1 << trs replicas, trl = lane & ((1 << trs) - 1)
};

struct ScanState {
    double A;              // exclusive mean accumulator of the queue (fp64)
    float B;               // exclusive variance accumulator (fp32, R22)
    int q, d, prev;        // prev: transition-table row p'
};

__device__ __forceinline__ void start_queue(const SlotTables &t, ScanState &s, int q) {
    const QRec r = t.sq[q];
    s.A = r.bmean; s.B = (float)r.bvar; s.d = r.d;
    s.prev = r.backlog ? r.r : t.M + r.r;   // R4/R12: a tail only behind a pinned backlog
    s.q = q;
}

// One group slot: returns its (wt, V) and record.
__device__ __forceinline__ void group_slot(const SlotTables &t, ScanState &s, int tok,
                                           double &wt, float &V, GRec &g) {
    {   // one 128-bit load of the 16-B record (two 64-bit loads conflict across replicas)
        const double2 raw = *reinterpret_cast<const double2 *>(t.sg + (tok << t.rs) + t.rl);
        const unsigned long long hi = (unsigned long long)__double_as_longlong(raw.y);
        g.slo = raw.x;
        g.n = (int32_t)(uint32_t)hi;
        g.model = (int32_t)(uint32_t)(hi >> 32);
    }
    const double2 ab = t.sab[((s.d * t.G + tok) << t.rs) + t.rl];
    const int m = g.model;
    s.A = __dadd_rn(s.A, t.str[(((s.d * 2 * t.M + s.prev) * t.M + m) << t.trs) + t.trl]);   // C - W ahead + swap S
    wt = s.A;
    V = s.B;                                         // exclusive (R5)
    s.A = __dadd_rn(s.A, ab.x);
    s.B = __fadd_rn(s.B, (float)ab.y);
    s.prev = m;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Phi-bar(z) = 0.5 erfc(z / sqrt 2) for |z| < z_clamp, fp32, via Abramowitz &
// Stegun 7.1.26 (|erfc error| <= 1.5e-7, so |Phi-bar error| <= 7.5e-8 plus
// fp32 rounding, well inside the 1e-5 parity bar; R8).
__device__ __forceinline__ float phibar(float z) {
    const float x = fabsf(z) * 0.70710678118654752f;
    const float t = rcp_approx(fmaf(0.3275911f, x, 1.0f));
    float y = fmaf(1.061405429f, t, -1.453152027f);
    y = fmaf(y, t, 1.421413741f);
    y = fmaf(y, t, -0.284496736f);
    y = fmaf(y, t, 0.254829592f);
    const float h = 0.5f * y * t * ex2_approx(-1.4426950408889634f * x * x);
    return z >= 0.0f ? h : 1.0f - h;
}

// Violation probability of a slot (R8/R9): v = Phi-bar(slack / sqrt V), exactly
// 0 / 1 when |z| >= z_clamp, tested as slack^2 >= z_clamp^2 V in fp32 (exact
// for V = 0, where it reduces to the step [wt > slo]; near |z| = z_clamp the
// two forms can differ only where Phi-bar < 1e-15).  `clamped` reports the
// fast path.
__device__ __forceinline__ float violation(double slack, double V, double zc2, bool &clamped) {
    const float sf = (float)slack, Vf = (float)V;
    clamped = sf * sf >= (float)zc2 * Vf;
    float v = sf < 0.0f ? 1.0f : 0.0f;
    if (!clamped) v = phibar(sf * rsqrt_approx(fmaxf(Vf, 1e-30f)));
    return v;
}

// The slot arithmetic every Gaussian scan kernel shares (R8/R9/R22), so their
// outputs are bit-identical to each other:
//   V accumulates in fp32 (b rounded once to fp32 when the tables are built);
//   sd = sqrt.approx(V);  clamped <=> |slack| >= z_clamp * sd (exact for V = 0,
//   where it reduces to the step [wt > slo]; near |z| = z_clamp it can differ
//   from the exact test only where Phi-bar < 1e-15);  v = [slack < 0] when
//   clamped, else Phi-bar(slack / sd).
__device__ __forceinline__ float slot_sd(float V) { return sqrt_approx(V); }
__device__ __forceinline__ bool slot_clamped(float sf, float sd, float zc) { return fabsf(sf) >= zc * sd; }
__device__ __forceinline__ float slot_v_clamped(float sf) { return sf < 0.0f ? 1.0f : 0.0f; }
__device__ __forceinline__ float slot_v_open(float sf, float sd) { return phibar(sf * rcp_approx(sd)); }
__device__ __forceinline__ float slot_v(double slack, float sd, float zc, bool &clamped) {
    const float sf = (float)slack;
    clamped = slot_clamped(sf, sd, zc);
    return clamped ? slot_v_clamped(sf) : slot_v_open(sf, sd);
}

__device__ __forceinline__ uint64_t make_key(float s1, float s2) {
    s2 = s2 + 0.0f;                                       // -0 -> +0
    uint32_t b2 = __float_as_uint(s2);
    b2 = (b2 & 0x80000000u) ? ~b2 : (b2 | 0x80000000u);
    return ((uint64_t)__float_as_uint(s1) << 32) | b2;
}

__device__ __forceinline__ bool better(uint64_t k1, int64_t i1, uint64_t k2, int64_t i2) {
    return k1 < k2 || (k1 == k2 && (uint64_t)i1 < (uint64_t)i2);
}

__device__ __forceinline__ void warp_argmin(uint64_t &key, int64_t &idx) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const uint64_t k2 = __shfl_xor_sync(0xFFFFFFFFu, key, o);
        const int64_t i2 = __shfl_xor_sync(0xFFFFFFFFu, idx, o);
        if (better(k2, i2, key, idx)) { key = k2; idx = i2; }
    }
}

// ---- bulk async copies (TMA engine, no tensor map) ----------------------------
__device__ __forceinline__ void bulk_s2g(void *gdst, const void *ssrc, uint32_t bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gdst), "r"(s), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Materialise one candidate row into srow[0..T) with a warp (R9/R10).  For
// RANDOM, the lanes first compute every swap target j_i = i + mulhi(u_i, T-i)
// in parallel (they depend only on the Philox words, not on the row), then
// lane 0 runs the forward Fisher-Yates swaps with one shared-memory round trip
// per step: the value at position i+1 is loaded together with row[j_i] (the
// only store of step i that can touch position i+1 is row[j_i] = row[i]).
__device__ __forceinline__ void warp_gen_row(const Cand &cd, int T, uint64_t c, int64_t loc,
                                             uint16_t *srow, uint16_t *sJ) {
    const int lane = threadIdx.x & 31;
    if (cd.kind == QLM_CAND_RANDOM) {
        const bool d16 = T <= 256;                           // R10 draw width
        const int per = d16 ? 8 : 4;
        const int nb = (T - 1 + per - 1) / per;
        const uint2 key = make_uint2((uint32_t)cd.seed, (uint32_t)(cd.seed >> 32));
        for (int b = lane; b < nb; b += 32) {
            const uint4 wd = philox10(make_uint4((uint32_t)b, (uint32_t)c, (uint32_t)(c >> 32), kRowTag), key);
            if (d16) {
#pragma unroll
                for (int h = 0; h < 8; ++h) {
                    const int i = 8 * b + h;
                    const uint32_t w = pick4(wd, h >> 1);
                    const uint32_t u = (h & 1) ? (w >> 16) : (w & 0xFFFFu);
                    if (i + 1 < T) sJ[i] = (uint16_t)(i + (int)((u * (uint32_t)(T - i)) >> 16));
                }
            } else {
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int i = 4 * b + h;
                    if (i + 1 < T) sJ[i] = (uint16_t)(i + (int)__umulhi(pick4(wd, h), (uint32_t)(T - i)));
                }
            }
        }
        for (int s = lane; s < T; s += 32) srow[s] = (uint16_t)s;
        __syncwarp();
        if (lane == 0 && T > 1) {
            uint32_t ti = srow[0];
            int j = sJ[0];
            for (int i = 0; i + 1 < T; ++i) {
                const int jn = i + 2 < T ? sJ[i + 1] : 0;
                const uint32_t tj = srow[j];
                const uint32_t nx = srow[i + 1];
                srow[j] = (uint16_t)ti;
                srow[i] = (uint16_t)tj;
                ti = (j == i + 1) ? ti : nx;
                j = jn;
            }
        }
    } else if (cd.kind == KIND_ILV) {                     // rows made by fy_rows_kernel (u16 pairs)
        const uint32_t *r32 = reinterpret_cast<const uint32_t *>(cd.rows);
        for (int w = lane; w < (T + 1) / 2; w += 32) {
            const uint32_t v = __ldg(r32 + (size_t)w * cd.stride + loc);
            srow[2 * w] = (uint16_t)v;
            if (2 * w + 1 < T) srow[2 * w + 1] = (uint16_t)(v >> 16);
        }
    } else if (cd.kind == QLM_CAND_ENUM) {
        if (lane == 0) {
            int s = 0;
            tokens_enum(c, T, [&](int tok) { srow[s++] = (uint16_t)tok; });
        }
    } else if (cd.kind == QLM_CAND_NEIGHBOR) {
        for (int s = lane; s < T; s += 32)
            srow[s] = cd.tb == 1 ? (uint16_t)base_token<uint8_t>(cd, s) : (uint16_t)base_token<uint16_t>(cd, s);
        __syncwarp();
        if (lane == 0) {
            int mi[QLM_MAX_MOVES], mj[QLM_MAX_MOVES];
            nbr_moves(cd, T, c, mi, mj);
            for (int m = 0; m < cd.moves; ++m) {
                const uint16_t t = srow[mi[m]];
                srow[mi[m]] = srow[mj[m]];
                srow[mj[m]] = t;
            }
        }
    } else {
        const uint8_t *row = cd.rows + loc * cd.stride;
        for (int s = lane; s < T; s += 32)
            srow[s] = cd.tb == 1 ? row[s] : reinterpret_cast<const uint16_t *>(row)[s];
    }
    __syncwarp();
}

// Walk a materialised row in 32-token chunks with warp ballots: for each
// group token, its queue q (separators before it, capped at Q-1, R9), its
// position within the queue and its slot index (groups before it).
template <typename F>
__device__ __forceinline__ void warp_slots(const uint16_t *srow, int T, int G, int Q, F &&f) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    int nsep = 0, lastsep = -1;
    for (int s0 = 0; s0 < T; s0 += 32) {
        const int s = s0 + lane;
        const int tok = s < T ? srow[s] : 0;
        const bool sep = s < T && tok >= G;
        const uint32_t bs = __ballot_sync(0xFFFFFFFFu, sep);
        const uint32_t below = bs & lt;
        const int before = nsep + __popc(below);
        const int ls = below ? s0 + 31 - __clz(below) : lastsep;
        if (s < T && !sep) {
            const int q = before < Q - 1 ? before : Q - 1;
            f(tok, q, s - ls - 1, s - before);
        }
        nsep += __popc(bs);
        if (bs) lastsep = s0 + 31 - __clz(bs);
    }
}

}  // namespace qlm
