// qlm_ws2.cu -- the bulk fast path on sm_100a: one pass of a1-a7 for problems
// with one device type (D = 1) and byte rows (T <= 256).  This is the kernel of
// the C3 bench step (qlm_score_estimate / qlm_rwt_estimate).
//
// Same shape as qlm_ws.cu (producer/consumer warp pairs, row slots guarded by
// mbarriers, group-major [G][32] staging tiles leaving through 2-D TMA tensor
// stores, in-kernel argmin), with the consumer rebuilt around issue count --
// the scheduler issue load bounded the round-1 kernel at ~105 warp
// instructions per token step:
//
//  * one record per token value: groups 0..G-1 and the separators, which the
//    consumer relabels in row order (the k-th separator of a row becomes token
//    G + k, the start of queue k + 1), so a separator is a table entry like a
//    group -- {slo, a} | {b, n, next transition row, transition column} -- and
//    a slot is straight-line code with no queue table, no select chain and no
//    device bases (D = 1);
//  * the queue reset is arithmetic: A' = fma(A + tr, keep, a) with keep = 1 for
//    a group (exactly A + tr + a, the oracle's order) and 0 for a separator
//    (whose a is the queue's backlog mean and whose transition column is 0), so
//    wt stays bit-identical to the oracle;
//  * V accumulates in fp32 (R22): sd and z need fp32 only, and the variance
//    terms are positive, so the relative error of a queue's V is at most
//    (slots ahead) * 2^-24;
//  * separator slots are masked by one predicate (no trash row, no score
//    selects); scores, S1 and n_over use predicated adds;
//  * |z| >= z_clamp is tested as |slack| >= z_clamp * sd (sd = sqrt.approx V),
//    and the rare unclamped slots are deferred (slack, token) to a per-lane
//    FIFO whose entries find sd in the staging tile at flush time.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "qlm_argmin.cuh"
#include "qlm_device.cuh"
#include "qlm_launch.h"

namespace qlm {
namespace ws2 {

constexpr int kRep = 8;      // record replicas: lane l reads replica l & 7
constexpr int kTrRep = 16;   // transition replicas: lane l reads replica l & 15
// Two-tier swapping (R20) keeps two transition tables (warm, cold) in the same
// space with 8 replicas each, and a 16-byte second record half.
template <bool TIER> __host__ __device__ constexpr int tr_rep() { return TIER ? 8 : kTrRep; }
#ifndef WS2_PIPE
#define WS2_PIPE 0
#endif
#ifndef WS2_SPREAD
#define WS2_SPREAD 1
#endif
#ifndef WS2_SLEEP
#define WS2_SLEEP 0
#endif
#ifndef WS2_XNOSTORE
#define WS2_XNOSTORE 0
#endif
#ifndef WS2_XHALFREC
#define WS2_XHALFREC 0
#endif
#ifndef WS2_XNODEP
#define WS2_XNODEP 0
#endif
#ifndef WS2_XNOPROD
#define WS2_XNOPROD 0
#endif
#ifndef WS2_PRELABEL
#define WS2_PRELABEL 0    // 1: producers relabel separators in the final row words (measured +2 %, off)
#endif
#ifndef WS2_P6
#define WS2_P6 0          // 1: six producers feed seven consumers (balanced schedulers; measured +10 %, off)
#endif
#ifndef WS2_WMAX
#define WS2_WMAX 7
#endif
#ifndef WS2_XW5
#define WS2_XW5 0
#endif
#ifndef WS2_CHAIN1
#define WS2_CHAIN1 0
#endif
#ifndef WS2_PHXPIPE
#define WS2_PHXPIPE 1     // producer: Philox block b + 1 computed alongside block b's swaps
#endif
#ifndef WS2_LATEWAIT
#define WS2_LATEWAIT 1    // consumer: wait for the previous tile's TMA read after word 0's loads
#endif
constexpr int kWordsPerCheck = 2;
constexpr int kPend = 4 + 4 * kWordsPerCheck;   // deferred-slot FIFO depth per lane
constexpr int kRecStride = 2 * kRep * 16;   // bytes per token value: [2 halves][8 replicas][16 B]
// neutral records T .. T + nneu - 1 for the row padding (see load_word)
__host__ __device__ constexpr int neutral_count(int T) { return (-T) & 3; }

struct alignas(64) Params {
    CUtensorMap tmap[3];     // wt, sd, v: fp32 [G][count], box {32, G}
    ScanParams p;
    int pairs;               // W producer/consumer pairs (warps [0,W) consume, [W,2W) produce)
    int tw;                  // 32-bit words per row
    int off_rec, off_tr, off_rows, off_bar, off_pend, off_stage;
    int use_tma;
    float zc;                // z_clamp
    float oc;                // 1 if a clamped late slot (v = 1) counts in n_over (1 > alpha)
};

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
// Blocks in hardware until the phase with this parity has completed (the
// suspend-time hint keeps a waiting warp off the scheduler instead of spinning).
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n.reg .pred P1;\n"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(ok)
            : "r"(su32(b)), "r"(parity), "r"(0x100000u)
            : "memory");
    } while (!ok);
}
// One non-blocking probe of a phase.
__device__ __forceinline__ bool mbar_test(uint64_t *b, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Per-slot consumption counters of the six-producer hand-off: several
// producers fill one slot in turn, so the "slot free" signal is a count (an
// mbarrier parity wait would let a producer two uses ahead pass early).
__device__ __forceinline__ uint32_t ld_acquire_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t a, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap *tm, uint32_t src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 ::"l"(reinterpret_cast<uint64_t>(tm)), "r"(src), "r"(x), "r"(y)
                 : "memory");
}
// Loads of the read-only tables (records, transitions): not volatile and no
// memory clobber, so the scheduler may hoist a slot's table loads above the
// previous slots' staging stores (the tables are written once, before the
// block barrier, and their addresses depend on row words read after the
// slot's mbarrier wait).
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
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

// ---- producers: one candidate row per lane into the lane's column of a slot
// (token i of lane l in byte i mod 4 of word (i / 4) * 32 + l: any
// lane-parallel access hits 32 distinct banks) ----------------------------------

// Bytes of a row's last word past position T-1: 0xFF, a neutral token (>= G).
__device__ __forceinline__ uint32_t pad_mask(int T) {
    return (T & 3) ? 0xFFFFFFFFu << (8 * (T & 3)) : 0u;
}
__device__ __forceinline__ uint32_t ld_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void st_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// Separator relabelling in row order: the k-th token >= G of a row becomes
// G + k (the start of queue k + 1; padding bytes continue past T - 1 into the
// neutral records).  `gns` = G + separators seen so far.  With WS2_PRELABEL
// the producers apply it to every final row word, so the consumer reads labels.
__device__ __forceinline__ uint32_t relabel_word(uint32_t w, uint32_t G, uint32_t &gns) {
#if WS2_PRELABEL
    uint32_t out = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t t = __byte_perm(w, 0u, 0x4440u + k);
        const bool sep = t >= G;
        t = sep ? gns : t;
        gns += sep ? 1u : 0u;
        out |= t << (8 * k);
    }
    return out;
#else
    return w;
#endif
}

// RANDOM (R10, T <= 256: two 16-bit swap indices per Philox word, 8 per block):
// forward Fisher-Yates in the lane's column (shared address `cs` = slot + 4
// lane; byte of token i at cs + (i mod 4) + 128 (i / 4)).  Position i is final
// after step i (later steps touch positions > i), so finals are packed in a
// register and leave as whole words.
__device__ __forceinline__ void produce_random(uint32_t cs, int T, uint32_t G, uint64_t seed, uint64_t c) {
    const int tw = (T + 3) >> 2;
    uint32_t gns = G;
    for (int w = 0; w < tw; ++w) st_u32(cs + w * 128, 0x03020100u + 0x04040404u * (uint32_t)w);
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const uint32_t clo = (uint32_t)c, chi = (uint32_t)(c >> 32);
    const int nfull = (T - 1) >> 3;                     // Philox blocks with 8 live draws
    uint32_t fin = 0;
    // one swap: j = i + floor(u (T - i) / 2^16) (R10) = hi32((u << 16) (T - i));
    // byte address of j = cs + j + 124 (j / 4)
    auto step = [&](int i, uint32_t u16hi, uint32_t ai) {
        uint32_t jd;
        asm("{\n.reg .u64 t;\nmul.wide.u32 t, %1, %2;\nmov.b64 {_, %0}, t;\n}\n"
            : "=r"(jd) : "r"(u16hi), "r"((uint32_t)(T - i)));
        const uint32_t j = (uint32_t)i + jd;
        QLM_CHECK(j < (uint32_t)T && j >= (uint32_t)i);
        const uint32_t aj = (j >> 2) * 124u + (cs + j);
        const uint32_t ti = ld_u8(ai), tj = ld_u8(aj);
        st_u8(aj, ti);
        fin |= tj << ((i & 3) * 8);
    };
    int i0 = 0;
#if WS2_PHXPIPE
    // the Philox chain of block b + 1 is independent of block b's swaps: the
    // scheduler interleaves the two latency chains
    uint4 wn = philox10(make_uint4(0u, clo, chi, kRowTag), key);
#endif
    for (int b = 0; b < nfull; ++b, i0 += 8) {
#if WS2_PHXPIPE
        const uint4 wd = wn;
        wn = philox10(make_uint4((uint32_t)(b + 1), clo, chi, kRowTag), key);
#else
        const uint4 wd = philox10(make_uint4((uint32_t)b, clo, chi, kRowTag), key);
#endif
        const uint32_t pb = cs + (i0 << 5);             // word i0 / 4 of the lane's column
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t w = pick4(wd, k >> 1);
            step(i0 + k, (k & 1) ? (w & 0xFFFF0000u) : (w << 16), pb + ((k >> 2) << 7) + (k & 3));
            if ((k & 3) == 3) {
                st_u32(pb + ((k >> 2) << 7), relabel_word(fin, G, gns));
                fin = 0;
            }
        }
    }
    if (i0 < T - 1) {                                   // last partial block
#if WS2_PHXPIPE
        const uint4 wd = wn;
#else
        const uint4 wd = philox10(make_uint4((uint32_t)nfull, clo, chi, kRowTag), key);
#endif
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            const int i = i0 + k;
            if (i >= T - 1) break;
            const uint32_t w = pick4(wd, k >> 1);
            step(i, (k & 1) ? (w & 0xFFFF0000u) : (w << 16), cs + (i & 3) + ((i >> 2) << 7));
            if ((i & 3) == 3) {
                st_u32(cs + ((i >> 2) << 7), relabel_word(fin, G, gns));
                fin = 0;
            }
        }
    }
    {   // position T-1 holds whatever the last swap left there
        const int i = T - 1;
        fin |= ld_u8(cs + (i & 3) + ((i >> 2) << 7)) << ((i & 3) * 8);
        st_u32(cs + ((i >> 2) << 7), relabel_word(fin | pad_mask(T), G, gns));   // neutral padding past T-1
    }
}

// EXPLICIT byte rows: 16-byte loads of the lane's own row, word stores (the
// caller's padding bytes past T-1 are replaced by neutral tokens).
__device__ __forceinline__ void produce_explicit(uint32_t cs, int T, uint32_t G, int tw, const uint8_t *row) {
    const uint32_t pad = pad_mask(T);
    uint32_t gns = G;
    for (int w = 0; w < tw; w += 4) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(row + 4 * w));
        const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (w + k < tw) st_u32(cs + (w + k) * 128, relabel_word(w + k == tw - 1 ? x[k] | pad : x[k], G, gns));
    }
}

// NEIGHBOR over a byte base row (R18): base words (a broadcast load), the
// candidate's transpositions in the lane's column, then relabelling.
__device__ __forceinline__ void produce_neighbor(uint32_t cs, int T, uint32_t G, int tw, const Cand &cd, uint64_t c) {
    const uint32_t *b32 = reinterpret_cast<const uint32_t *>(cd.rows);
    for (int w = 0; w < tw; ++w) st_u32(cs + w * 128, __ldg(b32 + w) | (w == tw - 1 ? pad_mask(T) : 0u));
    int mi[QLM_MAX_MOVES], mj[QLM_MAX_MOVES];
    nbr_moves(cd, T, c, mi, mj);
    for (int m = 0; m < cd.moves; ++m) {
        const uint32_t ai = cs + (mi[m] & 3) + ((mi[m] >> 2) << 7);
        const uint32_t aj = cs + (mj[m] & 3) + ((mj[m] >> 2) << 7);
        const uint32_t t = ld_u8(ai);
        st_u8(ai, ld_u8(aj));
        st_u8(aj, t);
    }
#if WS2_PRELABEL
    uint32_t gns = G;
    for (int w = 0; w < tw; ++w) st_u32(cs + w * 128, relabel_word(ld_u32(cs + w * 128), G, gns));
#endif
}

// ENUM (Lehmer unranking, lexicographic).
__device__ __forceinline__ void produce_enum(uint32_t cs, int T, uint32_t G, uint64_t c) {
    int s = 0;
    uint32_t gns = G;
    uint32_t fin = 0;
    tokens_enum(c, T, [&](int tok) {
        fin |= (uint32_t)tok << ((s & 3) * 8);
        if ((s & 3) == 3 || s == T - 1) {
            st_u32(cs + (s >> 2) * 128, relabel_word(s == T - 1 ? fin | pad_mask(T) : fin, G, gns));
            fin = 0;
        }
        ++s;
    });
}

// ---- consumer -------------------------------------------------------------------

struct Acc {
    double A, S2, acc2;      // running mean work (Eq. 10), S2 (R11), unclamped S1 terms
    float B;                 // running variance (R22: fp32)
    float acc1, over;        // clamped S1 terms (exact integers: sum n_i < 2^24), n_over
    uint32_t pq;             // next free FIFO entry (shared address)
};

// One row word = 4 slots, in two halves so a software pipeline can issue the
// table loads of word w + 1 before the arithmetic of word w:
//   load:    token -> label -> record -> transition (integer + shared loads);
//   compute: the Eq. 10 fp64 chain, violation probabilities, scores, staging.
// Rows are padded to whole words with separator-like neutral tokens (>= G,
// relabelled past the last real separator to records T.. whose slo = 1e30,
// a = b = n = 0): they only touch the trash row, at the end of the row.
struct WordData {
    double slo[4], aw[4], tr[4];
    float b[4], nf[4];
    int ix[4], kh[4];
};

// R20 state of the queue being walked: bit of the model in memory, warm
// targets, the queue's CPU memory not yet taken by them (-1 once a target did
// not fit: later targets are cold, the warm set is a strict prefix)
struct TierState {
    uint32_t pbit, warm;
    int rem;
};

// Address limits for the QLM_BOUNDS build (unused otherwise).
struct Bounds {
    int ntok;                 // record entries (tokens + neutral padding)
    uint32_t tr_lo, tr_hi;    // transition table(s), shared addresses
    uint32_t pq_hi;           // end of the lane's FIFO
};

template <bool TIER>
__device__ __forceinline__ void load_word(uint32_t wd, int G, int R, uint32_t rb, uint32_t rb1, uint32_t tb,
                                          uint32_t cold_off, uint32_t &prow, int &gq, TierState &ts,
                                          WordData &d, const Bounds &bd) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int tok = (int)__byte_perm(wd, 0u, 0x4440u + k);
        // one predicate for everything a separator changes: its label (the k-th
        // separator -> G + k), keep (the A reset, the B reset and its staging
        // stores, which are predicated off) (gq is incremented last: the compiler
        // may give G and gq one register when their values coincide, so no
        // operand is read after the write)
#if WS2_PRELABEL
        (void)gq;                                        // the producer relabelled the row
        d.ix[k] = tok;
        d.kh[k] = tok >= G ? 0 : 0x3FF00000;
#else
        asm("{\n.reg .pred p;\nsetp.ge.s32 p, %3, %4;\nselp.b32 %0, %2, %3, p;\n"
            "selp.b32 %1, 0, 0x3FF00000, p;\n@p add.s32 %2, %2, 1;\n}\n"
            : "=r"(d.ix[k]), "=r"(d.kh[k]), "+r"(gq) : "r"(tok), "r"(G));
#endif
        QLM_CHECK(d.ix[k] >= 0 && d.ix[k] < bd.ntok);
        const uint32_t ra = (uint32_t)d.ix[k] * kRecStride;
        const float4 r0 = lds128(rb + ra);               // {a, slo hi, n}
        d.aw[k] = __hiloint2double(__float_as_int(r0.y), __float_as_int(r0.x));
        d.slo[k] = __hiloint2double(__float_as_int(r0.z), 0);
        d.nf[k] = r0.w;
        uint32_t xs;
        if constexpr (TIER) {
            // {b, transition state, CPU memory (group: its model's; separator:
            // its queue's), model bit (separator: the resident's)}
            const float4 r1 = lds128(rb1 + ra);
            d.b[k] = r1.x;
            xs = (uint32_t)__float_as_int(r1.y);
            const int mem = __float_as_int(r1.z);
            const uint32_t bit = (uint32_t)__float_as_int(r1.w);
            const bool sep = d.kh[k] == 0;
            // R20, in the order of qlm_ws.cu's tier walk: the first transition
            // into a model makes it warm while it fits the CPU memory.  No
            // "seen" set is needed: a model whose first transition did not fit
            // left the queue exhausted (capd = -1), so testing it again can
            // only fail again -- a transition is cold iff its model is not warm
            // after the test
            // `rem` = the queue's CPU memory minus what its warm models take
            // (the walk's cum + mem <= capd is mem <= rem), -1 once exhausted
            const bool trn = !sep && bit != ts.pbit;
            const bool test = trn && !(ts.warm & bit);   // first transition (or a failed one)
            const bool fits = mem <= ts.rem;
            ts.warm |= (test && fits) ? bit : 0u;
            ts.rem = (test && fits) ? ts.rem - mem : ts.rem;
            const bool cold = test && !fits;
            ts.rem = cold ? -1 : ts.rem;
            ts.pbit = bit;                                 // separator: its queue's resident
            ts.rem = sep ? mem : ts.rem;
            ts.warm = sep ? 0u : ts.warm;
            QLM_CHECK(prow + xs + (cold ? cold_off : 0u) >= bd.tr_lo && prow + xs + (cold ? cold_off : 0u) + 8 <= bd.tr_hi);
            d.tr[k] = lds64f(prow + xs + (cold ? cold_off : 0u));
        } else {
            const float2 r1 = lds64v(rb1 + ra);          // {b, 128 * state}
            d.b[k] = r1.x;
#if WS2_XNODEP
            xs = (uint32_t)(tok & 3) * 128u;             // timing experiment: no record dependency
#else
            xs = (uint32_t)__float_as_int(r1.y);
#endif
            QLM_CHECK(prow + xs >= bd.tr_lo && prow + xs + 8 <= bd.tr_hi);
            d.tr[k] = lds64f(prow + xs);                 // row of the state before
        }
        prow = tb + xs * R;                              // row of this slot's state
    }
}

template <int GS, int SCORE>
__device__ __forceinline__ void compute_word(const WordData &d, uint32_t sb, float zc, float oc, Acc &a,
                                             const Bounds &bd) {
    constexpr uint32_t ASTR = GS * 128;                  // staging array stride
    double wt[4];
    float V[4];
    // Eq. 10 in the oracle's order: wt = A + (tail + swap); A' = wt + a.  A
    // separator's column is 0 and keep = 0, so A' = its queue's backlog mean;
    // B (R22: fp32) restarts at the queue's backlog variance
    double A = a.A;
    float B = a.B;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        wt[k] = __dadd_rn(A, d.tr[k]);
#if WS2_CHAIN1
        A = __fma_rn(A, __hiloint2double(d.kh[k], 0), __dadd_rn(d.tr[k], d.aw[k]));
#else
        A = __fma_rn(wt[k], __hiloint2double(d.kh[k], 0), d.aw[k]);
#endif
        V[k] = B;                                        // exclusive (R5)
        float Bk;
        asm("{\n.reg .pred p;\nsetp.eq.s32 p, %2, 0;\nselp.f32 %0, 0f00000000, %1, p;\n}\n"
            : "=f"(Bk) : "f"(B), "r"(d.kh[k]));
        B = __fadd_rn(Bk, d.b[k]);
    }
    a.A = A;
    a.B = B;
    // violation probabilities (R8/R9), scores (R11), staging.  A separator's
    // slo is 1e30: its slack is huge, so it is clamped with v = 0 and adds
    // nothing to S1 / n_over; keep = 0 drops it from S2
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double slack = __dsub_rn(d.slo[k], wt[k]);
        const float sf = (float)slack;
        const float sd = sqrt_approx(V[k]);
        const bool clamped = fabsf(sf) >= zc * sd;       // R9: exact for V = 0
        const float v = sf < 0.0f ? 1.0f : 0.0f;
        if constexpr (SCORE > 0) {
            if (clamped) {
                a.acc1 = fmaf(d.nf[k], v, a.acc1);       // separators: n = 0
                if constexpr (SCORE > 1) a.over = fmaf(v, oc, a.over);
            }
            a.S2 = __fma_rn(slack, -__hiloint2double(d.kh[k], 0), a.S2);   // S2 += wt - slo (groups only)
        }
        if (!clamped) {                                  // |z| < z_clamp: exact value at flush
            // the token goes to the lane's byte FIFO, the slack to the v row
            QLM_CHECK(a.pq < bd.pq_hi);
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(a.pq), "r"(d.ix[k]) : "memory");
            a.pq += 32;
        }
        const uint32_t st = sb + (uint32_t)d.ix[k] * 128u;
        QLM_CHECK(d.kh[k] == 0 || d.ix[k] < GS);              // stores only for groups
        if (WS2_XNOSTORE) continue;
        // separators and padding (keep = 0) store nothing
        asm volatile("{\n.reg .pred p;\nsetp.ne.s32 p, %4, 0;\n@p st.shared.f32 [%0], %1;\n"
                     "@p st.shared.f32 [%0+%5], %2;\n@p st.shared.f32 [%0+%6], %3;\n}\n"
                     ::"r"(st), "f"((float)wt[k]), "f"(sd), "f"(clamped ? v : sf), "r"(d.kh[k]),
                     "n"(ASTR), "n"(2 * ASTR) : "memory");
    }
}

// Deferred slots: Phi-bar in FIFO (row) order; v overwrites the staged value.
template <int GS, int SCORE>
__device__ __forceinline__ void flush(uint32_t pq0, uint32_t rb, uint32_t sb, float alpha, Acc &a) {
    const int n = (int)((a.pq - pq0) >> 5);
    const int maxn = (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)n);
    for (int i = 0; i < maxn; ++i) {
        if (i < n) {
            const int ix = (int)ld_u8(pq0 + i * 32);
            QLM_CHECK(ix < GS);                                  // only groups are deferred
            const uint32_t s = sb + (uint32_t)ix * 128u;
            float sd, sf;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(sd) : "r"(s + GS * 128));
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(sf) : "r"(s + 2 * GS * 128));   // the slack
            const float v = phibar(sf * rcp_approx(sd));
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(s + 2 * GS * 128), "f"(v) : "memory");
            if constexpr (SCORE > 0) {
                float nf;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(nf) : "r"(rb + (uint32_t)ix * kRecStride + 12));
                a.acc2 = __fma_rn((double)nf, (double)v, a.acc2);
                a.over += v > alpha ? 1.0f : 0.0f;
            }
        }
    }
    a.pq = pq0;
}

template <int KIND, int GS, int SCORE, bool TIER>
__global__ void __launch_bounds__(512, 1) ws2_kernel(const __grid_constant__ Params w) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const ScanParams &p = w.p;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = w.pairs;
    const int G = p.dm.G, T = p.dm.T, M = p.dm.M;

    // ---- tables -> smem ------------------------------------------------------
    // Per token value ix (groups 0..G-1; G + k = separator k = start of queue
    // k + 1; T.. neutral padding) a 24-byte record in two halves:
    //   half 0, 8 replicas x 16 B: {a (f64), hi word of slo (its low word is
    //           0: the launcher checked), n (f32)}
    //   half 1, 16 replicas x 8 B: {b (f32), x = 128 * transition state}
    // Transition states s < M: after a group of model s; M + r: queue start on
    // resident r with nothing running (R4).  A group's state is its model, a
    // separator's the start state of its queue (a declared backlog starts in
    // the resident's model state, R12).
    constexpr int TRR = tr_rep<TIER>();
    int summem = 0;
    if constexpr (TIER)
        for (int m = 0; m < M; ++m) summem += p.t_mem[m];
    for (int i = tid; i < (T + neutral_count(T)) * kTrRep; i += blockDim.x) {
        const int ix = i / kTrRep, r = i % kTrRep;
        double aw, slo;
        float b, nf;
        int st, mem = 0;
        uint32_t bit = 0;
        if (ix < G) {
            const GRec g = p.tb.grec[ix];
            const double2 ab = p.tb.ab[ix];                       // device row 0 (D = 1)
            slo = g.slo; aw = ab.x; b = (float)ab.y; nf = (float)g.n; st = g.model;
            if constexpr (TIER) { mem = p.t_mem[g.model]; bit = 1u << g.model; }
        } else if (ix >= T) {                                    // neutral padding token
            slo = 1e30; aw = 0.0; b = 0.0f; nf = 0.0f; st = 0;
        } else {
            const QRec q = p.tb.qrec[ix - G + 1];
            slo = 1e30; aw = q.bmean; b = (float)q.bvar; nf = 0.0f;
            st = q.backlog ? q.r : M + q.r;
            if constexpr (TIER) { mem = min(p.t_cap[q.d], summem); bit = 1u << q.r; }
        }
        uint8_t *e = smem + w.off_rec + ix * kRecStride;
        if (r < kRep)
            *reinterpret_cast<float4 *>(e + r * 16) =
                make_float4(__int_as_float(__double2loint(aw)), __int_as_float(__double2hiint(aw)),
                            __int_as_float(__double2hiint(slo)), nf);
        if constexpr (TIER) {
            if (r < kRep)
                *reinterpret_cast<float4 *>(e + kRep * 16 + r * 16) =
                    make_float4(b, __int_as_float(st * TRR * 8), __int_as_float(mem), __int_as_float((int)bit));
        } else {
            *reinterpret_cast<float2 *>(e + kRep * 16 + r * 8) = make_float2(b, __int_as_float(st * TRR * 8));
        }
    }
    // transitions [2M][M][TRR replicas] f64 + M zero entries, row = state
    // before the slot, column = the slot's state: tail of the model ahead on a
    // change (R1) + swap, one fp64 term (R2).  A separator's column (its start
    // state, >= M) reads the next row's entries or the zero padding: finite
    // values that keep = 0 discards.  Tiered: a second (cold) table follows,
    // + the storage -> CPU load of a model that changes (R20)
    const int R = M;                                       // row stride in entries
    const int ntr = M * (2 * M + 1) * TRR;
    for (int i = tid; i < (TIER ? 2 : 1) * ntr; i += blockDim.x) {
        const int e = (i % ntr) / TRR, col = e % M, row = e / M;
        double v = 0.0;
        if (row < 2 * M) {
            const int from = row < M ? row : row - M;
            const double sw = p.tb.swap[from * M + col];
            const double tl = (row < M && col != row) ? p.tb.tail[row] : 0.0;
            v = i < ntr ? __dadd_rn(tl, sw) : __dadd_rn(tl, __dadd_rn(sw, col != from ? p.t_load[col] : 0.0));
        }
        reinterpret_cast<double *>(smem + w.off_tr)[i] = v;
    }
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + w.off_bar);
    uint64_t *empty = full + 2 * W;
    int64_t *slot_b = reinterpret_cast<int64_t *>(empty + 2 * W);
    unsigned long long *next_b = reinterpret_cast<unsigned long long *>(slot_b + 2 * W);
    // six producers for seven consumers (16-warp spread map): static task
    // rotation, "slot free" as a consumption count in empty[s]'s first word
    const bool p6 = WS2_P6 && WS2_SPREAD && W == 7;
    if (tid < 2 * W) {
        mbar_init(&full[tid], 32);
        if (p6) *reinterpret_cast<volatile uint32_t *>(&empty[tid]) = 0u;
        else mbar_init(&empty[tid], 32);
    }
    if (tid == 0) *next_b = 0ull;
    __syncthreads();

    const Cand cd = p.cd;
    const int64_t count = cd.count, first = cd.first;
    const int64_t nbatch = (count + 31) >> 5;
    const int64_t grid = gridDim.x;
    const int tw = w.tw;
    uint64_t bkey = ~0ull;
    int64_t bidx = -1;

    // roles: warps [0, W) consume, [W, 2W) produce; WS2_SPREAD (W = 6, 16
    // warps): producers on warps 6, 7, 10, 11, 14, 15 (schedulers 2/3), warps
    // 8, 9, 12, 13 idle
    int role_pair = warp < W ? warp : warp - W;
    bool is_prod = warp >= W, idle = false;
    if (WS2_SPREAD && W == 7) {
        // 16-warp block, warp w on scheduler w % 4: consumers 0-6 (schedulers
        // 0,1,2,3,0,1,2), producers 7-11, 14, 15, warps 12, 13 idle
        const int pmap[16] = {0, 1, 2, 3, 4, 5, 6, 0, 1, 2, 3, 4, -1, -1, 5, 6};
        // p6: producers 7-11, 15 (one on schedulers 0-2, three on 3)
        const int pmap6[16] = {0, 1, 2, 3, 4, 5, 6, 0, 1, 2, 3, 4, -1, -1, -1, 5};
        role_pair = p6 ? pmap6[warp] : pmap[warp];
        is_prod = warp >= 7;
        idle = role_pair < 0;
    } else if (WS2_SPREAD && W == 6) {
#if WS2_XW5   // timing experiment: pair 5 idle (five consumers, same placement)
        const int pmap[16] = {0, 1, 2, 3, 4, -1, 0, 1, -1, -1, 2, 3, -1, -1, 4, -1};
#else
        const int pmap[16] = {0, 1, 2, 3, 4, 5, 0, 1, -1, -1, 2, 3, -1, -1, 4, 5};
#endif
        role_pair = pmap[warp];
        is_prod = warp >= 6;
        idle = role_pair < 0;
    }
    if (idle) {
    } else if (is_prod) {   // ---------------- producer
        const int pair = role_pair;
        for (int j = 0;; ++j) {
            int s;
            int64_t b = 0;
            if (p6) {
                // task t = pair + 6 j of this block: batch blockIdx + t * grid,
                // row k = t / 7 of consumer t mod 7
                const int64_t t = pair + 6 * (int64_t)j;
                b = blockIdx.x + t * grid;
                if (b >= nbatch) break;
                const int kk = (int)(t / 7);
                s = 2 * (int)(t % 7) + (kk & 1);
                const uint32_t ca = su32(&empty[s]);
                if (lane == 0)
                    while (ld_acquire_u32(ca) < (uint32_t)(kk >> 1)) __nanosleep(32);
                __syncwarp();
                if (lane == 0) slot_b[s] = b;
            } else {
            s = 2 * pair + (j & 1);
#if WS2_SLEEP
            while (!mbar_test(&empty[s], ((j >> 1) & 1) ^ 1)) __nanosleep(WS2_SLEEP);
#else
            mbar_wait(&empty[s], ((j >> 1) & 1) ^ 1);
#endif
            if (lane == 0) {
                b = blockIdx.x + (int64_t)atomicAdd(next_b, 1ull) * grid;
                slot_b[s] = b;                                  // published by the arrive below
            }
            b = __shfl_sync(0xFFFFFFFFu, b, 0);
            if (b >= nbatch) {
                mbar_arrive(&full[s]);
                break;
            }
            }
            const int64_t loc = (b << 5) + lane;
            const uint32_t sl = su32(smem + w.off_rows) + (uint32_t)s * tw * 128;
            if (loc < count && !(WS2_XNOPROD && j >= 2)) {
                if constexpr (KIND == QLM_CAND_RANDOM) produce_random(sl + 4 * lane, T, G, cd.seed, (uint64_t)(first + loc));
                else if constexpr (KIND == QLM_CAND_EXPLICIT) produce_explicit(sl + 4 * lane, T, G, tw, cd.rows + loc * cd.stride);
                else if constexpr (KIND == QLM_CAND_NEIGHBOR) produce_neighbor(sl + 4 * lane, T, G, tw, cd, (uint64_t)(first + loc));
                else produce_enum(sl + 4 * lane, T, G, (uint64_t)(first + loc));
            } else {                                          // past the range: a valid row
                uint32_t gns = G;
                for (int wd = 0; wd < tw; ++wd)
                    st_u32(sl + 4 * lane + wd * 128,
                           relabel_word((0x03020100u + 0x04040404u * (uint32_t)wd) | (wd == tw - 1 ? pad_mask(T) : 0u), G, gns));
            }
            mbar_arrive(&full[s]);
        }
    } else {           // ---------------- consumer
        const int pair = role_pair;
        const uint32_t rb = su32(smem + w.off_rec) + (lane & (kRep - 1)) * 16;
        const uint32_t rb1 = su32(smem + w.off_rec) + kRep * 16 + (TIER ? (lane & 7) * 16 : (lane & 15) * 8);
        const uint32_t tb = su32(smem + w.off_tr) + (lane & (TRR - 1)) * 8;
        const uint32_t cold_off = (uint32_t)ntr * 8u;
        const uint32_t st0 = su32(smem + w.off_stage) + (uint32_t)pair * (3 * GS * 128);
        const uint32_t sb = st0 + lane * 4;
        const uint32_t pq0 = su32(smem + w.off_pend) + (uint32_t)pair * (kPend * 32) + lane;
        const uint32_t pqlim = pq0 + (kPend - 4 * kWordsPerCheck) * 32;    // room until the next check
        const float zc = w.zc, oc = w.oc, alpha = p.alpha;
        const double den = *p.tb.den;
        const QRec q0 = p.tb.qrec[0];                              // queue 0 start (R4 / R12)
        const double q0mean = q0.bmean;
        const float q0var = (float)q0.bvar;
        const int q0st = q0.backlog ? q0.r : M + q0.r;
        const uint32_t q0bit = 1u << q0.r;
        const int q0cap = TIER ? min(p.t_cap[q0.d], summem) : 0;
        const int nw = (T + 3) >> 2;                               // row words (padded)
        Bounds bd;
        bd.ntok = T + neutral_count(T);
        bd.tr_lo = su32(smem + w.off_tr);
        bd.tr_hi = bd.tr_lo + (uint32_t)(TIER ? 2 : 1) * (uint32_t)ntr * 8u;
        bd.pq_hi = pq0 + kPend * 32u;
        for (int j = 0;; ++j) {
            const int s = 2 * pair + (j & 1);
            int64_t b;
            if (p6) {
                b = blockIdx.x + (pair + 7 * (int64_t)j) * grid;   // task pair + 7 j
                if (b >= nbatch) break;
                mbar_wait(&full[s], (j >> 1) & 1);
            } else {
                mbar_wait(&full[s], (j >> 1) & 1);
                b = slot_b[s];
                if (b >= nbatch) break;
            }
            const bool tile_busy = j > 0 && w.use_tma;           // previous tile not yet read out
#if !WS2_LATEWAIT
            if (tile_busy) {
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
            }
#endif
            const int64_t c0 = b << 5, loc = c0 + lane;
            // row words; the slot has one spare word so the prefetch never leaves it
            uint32_t ra = su32(smem + w.off_rows) + (uint32_t)s * tw * 128 + 4 * lane;
            // every lane walks a row (lanes past the end of the range walk the
            // identity row the producer left them), so the loop stays convergent:
            // no reconvergence barriers and full-warp votes
            Acc a;
            a.A = q0mean; a.B = q0var;
            a.S2 = 0.0; a.acc2 = 0.0; a.acc1 = 0.0f; a.over = 0.0f; a.pq = pq0;
            uint32_t prow = tb + (uint32_t)q0st * (TRR * 8u) * R;   // queue 0 start row
            int gq = G;
            TierState ts;
            ts.pbit = q0bit; ts.warm = 0u; ts.rem = q0cap;
            uint32_t cur = ld_u32(ra);
            int wi = 0;
#if WS2_LATEWAIT
            {   // word 0 peeled: its table loads run before the wait for the TMA
                // engine to finish reading the previous tile out of the staging
                WordData d;
                load_word<TIER>(cur, G, R, rb, rb1, tb, cold_off, prow, gq, ts, d, bd);
                cur = ld_u32(ra + (nw > 1 ? 1 : 0) * 128);
                if (tile_busy) {
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
                }
                compute_word<GS, SCORE>(d, sb, zc, oc, a, bd);
                wi = 1;
            }
#endif
            for (; wi + 1 < nw; wi += 2) {
                const uint32_t nxt = ld_u32(ra + (wi + 1) * 128);
                WordData d;
                load_word<TIER>(cur, G, R, rb, rb1, tb, cold_off, prow, gq, ts, d, bd);
                compute_word<GS, SCORE>(d, sb, zc, oc, a, bd);
                cur = ld_u32(ra + (wi + 2 < nw ? wi + 2 : wi + 1) * 128);
                load_word<TIER>(nxt, G, R, rb, rb1, tb, cold_off, prow, gq, ts, d, bd);
                compute_word<GS, SCORE>(d, sb, zc, oc, a, bd);
                if (__any_sync(0xFFFFFFFFu, a.pq > pqlim)) flush<GS, SCORE>(pq0, rb, sb, alpha, a);
            }
            if (wi < nw) {
                WordData d;
                load_word<TIER>(cur, G, R, rb, rb1, tb, cold_off, prow, gq, ts, d, bd);
                compute_word<GS, SCORE>(d, sb, zc, oc, a, bd);
            }
            flush<GS, SCORE>(pq0, rb, sb, alpha, a);
            if (p6) {                                               // row slot free
                __syncwarp();
                if (lane == 0) st_release_u32(su32(&empty[s]), (uint32_t)((j >> 1) + 1));
            } else {
                mbar_arrive(&empty[s]);
            }
            if (w.use_tma) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (p.wt) tma_store_2d(&w.tmap[0], st0, (int)c0, 0);
                    if (p.sd) tma_store_2d(&w.tmap[1], st0 + GS * 128, (int)c0, 0);
                    if (p.vo) tma_store_2d(&w.tmap[2], st0 + 2 * GS * 128, (int)c0, 0);
                    bulk_commit();
                }
            } else {
                __syncwarp();
                if (loc < count) {
                    const float *stf = reinterpret_cast<const float *>(smem + w.off_stage) +
                                       (size_t)pair * 3 * GS * 32 + lane;
                    const int64_t ld = p.ld_out ? p.ld_out : count;
                    for (int g = 0; g < G; ++g) {
                        const int64_t o = (int64_t)g * ld + loc;
                        if (p.wt) p.wt[o] = stf[g * 32];
                        if (p.sd) p.sd[o] = stf[(GS + g) * 32];
                        if (p.vo) p.vo[o] = stf[(2 * GS + g) * 32];
                    }
                }
                __syncwarp();
            }
            // scores after the tile's TMA store is issued (they need no staging)
            if (loc < count) {
                if constexpr (SCORE > 0) {
                    const float s1 = (float)(((double)a.acc1 + a.acc2) / den);   // R11
                    const float s2 = (float)a.S2;
                    if (p.s1) p.s1[loc] = s1;
                    if (p.s2) p.s2[loc] = s2;
                    if (p.n_over) p.n_over[loc] = (int)a.over;
                    const uint64_t key = make_key(s1, s2);
                    const int64_t c = first + loc;
                    if (better(key, c, bkey, bidx)) { bkey = key; bidx = c; }
                }
            }
        }
        if (w.use_tma && lane == 0) bulk_wait0();
    }
    if constexpr (SCORE > 0) {
        if (p.out_rec) block_grid_argmin(p, bkey, bidx);           // all warps take part
    }
}

// ---- host side ------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        else
            cudaGetLastError();
    });
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

static size_t a128(size_t x) { return (x + 127) & ~size_t(127); }

static size_t plan(Params &w, int W, int GS, bool tier) {
    const Dims &dm = w.p.dm;
    (void)tier;                                            // tiered: 2 tables x 8 replicas, same bytes
    size_t off = 0;
    w.tw = (dm.T + 3) / 4;
    w.off_rows = (int)off;  off = a16(off + (size_t)2 * W * w.tw * 128);   // 1 KB aligned (the smem base)
    w.off_tr = (int)off;    off = a16(off + (size_t)dm.M * (2 * dm.M + 1) * kTrRep * 8);
    w.off_rec = (int)off;   off = a16(off + (size_t)(dm.T + neutral_count(dm.T)) * kRecStride);
    w.off_bar = (int)off;   off = a16(off + (size_t)6 * W * 8 + 8);
    w.off_pend = (int)off;  off = a16(off + (size_t)W * kPend * 32);
    off = a128(off);        // TMA source tiles: 128-byte aligned
    w.off_stage = (int)off; off += (size_t)W * 3 * GS * 128;
    w.pairs = W;
    return off;
}

// Dynamic shared-memory opt-in, per (device, kernel): the attribute is per device.
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
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess && optin > (int)fa.sharedSizeBytes + 1024) {
        m = (size_t)optin - fa.sharedSizeBytes - 1024;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m) != cudaSuccess) m = 0;
    }
    cudaGetLastError();
    cache[key] = m;
    return m;
}

template <int KIND, int GS, int SCORE, bool TIER>
static cudaError_t launch_t(const ScanParams &p0, cudaStream_t st) {
    auto kern = ws2_kernel<KIND, GS, SCORE, TIER>;
    const size_t lim = opt_in(kern);
    if (!lim) return cudaErrorNotSupported;
    Params w;
    memset(&w, 0, sizeof w);
    w.p = p0;
    int W = 0;
    size_t smem = 0;
    for (int cand = 8; cand >= 2; --cand) {
        Params t = w;
        const size_t sm = plan(t, cand, GS, TIER);
        if (sm <= lim) { W = cand; smem = sm; break; }
    }
    if (W < 2) return cudaErrorNotSupported;
    if (W > WS2_WMAX) W = WS2_WMAX;         // 7: 14 of 16 warps (the spread map)
    smem = plan(w, W, GS, TIER);
    const Dims &dm = p0.dm;
    w.zc = p0.zc;
    w.oc = 1.0f > p0.alpha ? 1.0f : 0.0f;
    w.use_tma = 0;
    const bool aligned = (p0.cd.count % 4 == 0) && !p0.ld_out &&
                         (!p0.wt || ((uintptr_t)p0.wt & 15) == 0) &&
                         (!p0.sd || ((uintptr_t)p0.sd & 15) == 0) &&
                         (!p0.vo || ((uintptr_t)p0.vo & 15) == 0);
    bool ok = aligned;
    if (ok && p0.wt) ok = make_map(&w.tmap[0], p0.wt, p0.cd.count, dm.G);
    if (ok && p0.sd) ok = make_map(&w.tmap[1], p0.sd, p0.cd.count, dm.G);
    if (ok && p0.vo) ok = make_map(&w.tmap[2], p0.vo, p0.cd.count, dm.G);
    w.use_tma = ok ? 1 : 0;
    const int64_t nbatch = (p0.cd.count + 31) / 32;
    int64_t grid = sm_count();
    const int64_t need = (nbatch + W - 1) / W;
    if (grid > need) grid = need;
    if (grid > p0.max_blocks) grid = p0.max_blocks;
    if (grid < 1) grid = 1;
    qlog(1, "ws2_kernel<kind=%d,GS=%d,score=%d,tier=%d> count=%lld pairs=%d grid=%lld smem=%zu tma=%d", KIND,
         GS, SCORE, (int)TIER, (long long)p0.cd.count, W, (long long)grid, smem, w.use_tma);
    kern<<<(unsigned)grid, (WS2_SPREAD && W >= 6) ? 512 : 64 * W, smem, st>>>(w);
    ++g_launches;
    return cudaGetLastError();
}

template <int KIND, int SCORE, bool TIER>
static cudaError_t launch_g(const ScanParams &p, cudaStream_t st) {
    const int G = p.dm.G;
    if (G <= 32) return launch_t<KIND, 32, SCORE, TIER>(p, st);
    if (G <= 64) return launch_t<KIND, 64, SCORE, TIER>(p, st);
    if (G <= 128) return launch_t<KIND, 128, SCORE, TIER>(p, st);
    return cudaErrorNotSupported;
}

template <int KIND, bool TIER = false>
static cudaError_t launch_k(const ScanParams &p, cudaStream_t st) {
    if (p.n_over) return launch_g<KIND, 2, TIER>(p, st);
    if (p.s1 || p.s2 || p.out_rec) return launch_g<KIND, 1, TIER>(p, st);
    return launch_g<KIND, 0, TIER>(p, st);
}

}  // namespace ws2

// Bulk fast path for D = 1 and byte rows; cudaErrorNotSupported -> the caller
// falls back to the general warp-specialised kernel (qlm_ws.cu).
cudaError_t launch_ws2(const ScanParams &p, cudaStream_t st) {
    if (p.dm.D != 1 || p.dm.T > 256 || p.dm.G > 128 || p.dm.M > 6 || !p.slo_hi_only || p.cd.first_from ||
        p.cd.count < 4096 ||
        p.cd.count > ((int64_t)1 << 31) - 64)
        return cudaErrorNotSupported;
    if (!(p.wt || p.sd || p.vo)) return cudaErrorNotSupported;   // score-only: the thread-per-candidate scan
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM: return ws2::launch_k<QLM_CAND_RANDOM>(p, st);
    case QLM_CAND_EXPLICIT: return p.cd.tb == 1 ? ws2::launch_k<QLM_CAND_EXPLICIT>(p, st) : cudaErrorNotSupported;
    case QLM_CAND_NEIGHBOR: return p.cd.tb == 1 ? ws2::launch_k<QLM_CAND_NEIGHBOR>(p, st) : cudaErrorNotSupported;
    case QLM_CAND_ENUM: return ws2::launch_k<QLM_CAND_ENUM>(p, st);
    default: return cudaErrorNotSupported;
    }
}

// The same kernel with two-tier swapping (R20): warm / cold transition tables
// and the per-queue tier walk in the consumer.  Model sizes and capacities
// travel as 32-bit ints in the records (set_tiers bounds them by 2^24).
cudaError_t launch_ws2_tier(const ScanParams &p, cudaStream_t st) {
    if (p.dm.D != 1 || p.dm.T > 256 || p.dm.G > 128 || p.dm.M > 6 || !p.slo_hi_only || p.cd.first_from ||
        p.cd.count < 4096 || p.cd.count > ((int64_t)1 << 31) - 64 || !p.t_mem || !p.t_cap || !p.t_load)
        return cudaErrorNotSupported;
    if (!(p.wt || p.sd || p.vo)) return cudaErrorNotSupported;
    switch (p.cd.kind) {
    case QLM_CAND_RANDOM: return ws2::launch_k<QLM_CAND_RANDOM, true>(p, st);
    case QLM_CAND_EXPLICIT: return p.cd.tb == 1 ? ws2::launch_k<QLM_CAND_EXPLICIT, true>(p, st) : cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
    }
}

}  // namespace qlm
