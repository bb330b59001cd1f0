// qlm_group.cu -- request-group formation on the GPU (DESIGN R21; SURVEY
// 8(f) N4; Algorithm 1).
//
// Alg. 1: groups <- kMeansClustering(requests); every group larger than
// avg_batch_size * delta is split in half.  Under R21 the pipeline is, all on
// the device and in stream order:
//
//   fp_first / fp_round / fp_pick   farthest-point initialisation per model
//                       (exact int64 squared distances; per-block max of a
//                       packed (distance, ~index) key, then one global atomicMax
//                       per model and block: lowest index wins ties)
//   lloyd_assign / lloyd_update     Lloyd iterations: nearest centre of the
//                       request's model in fp64 with the oracle's operation
//                       order (no FMA), per-block int64 sums in shared memory
//                       flushed with integer atomics (exact, order-free), a
//                       device-side convergence flag so the host can enqueue
//                       max_iter iterations without a sync
//   rank_block / rank_scan          stable rank of every request inside its
//                       cluster (arrival order): __match_any_sync per warp,
//                       warps in order through a shared running count, blocks
//                       through a column scan
//   group_leaves / group_assign / group_finalize   recursive splitHalf as a
//                       descent (leaf counts per size from two sizes per level),
//                       group ids, exact integer sums of output tokens, min SLO,
//                       and the qlm_group records the scheduler consumes
//
// Everything that decides an integer (a label, a farthest point, a group id)
// is computed in the oracle's precision and order, so labels and groups are
// bit-exact to or_form_groups.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "qlm_device.cuh"
#include "qlm_launch.h"

namespace qlm {

constexpr int kIdxBits = 28;                        // n < 2^28
constexpr uint64_t kIdxMask = (1ull << kIdxBits) - 1;

struct GroupScratch {
    int64_t *mind;          // [n] farthest-point min distance
    int32_t *first;         // [M] first request of each model
    unsigned long long *best;   // [M] packed (d2 << 28) | (mask - index)
    int32_t *k_req;         // [M] requested k
    int32_t *k_eff;         // [M]
    int32_t *active;        // [M]
    int32_t *off_req;       // [M] offsets of the requested k (init slots)
    int32_t *init_req;      // [Kmax] chosen requests
    int32_t *off;           // [M + 1] offsets of the effective centres
    double *C;              // [Kmax][4] centres
    unsigned long long *sums;   // [Kmax][5] int64 sums (coords, count)
    uint32_t *changed, *conv, *iters;
    int32_t *inrank;        // [n]
    int32_t *bcount;        // [nb][Kmax]
    int32_t *size;          // [Kmax]
    int32_t *base;          // [Kmax + 1] group id base per cluster; base[Kmax] = G
    unsigned long long *gacc;   // [n_groups_max][4]: S1, S2, min slo bits, n
    int32_t *gmodel;        // [n_groups_max]
    int32_t *bad;           // [1] invalid inputs
};

struct GroupArgs {
    int n, dims, M, Kmax, limit, nb, gmax;
    const int32_t *model, *out, *feat;
    const double *slo;
    int32_t *label, *group_of;
    qlm_group *groups;
    int group_cap;
};

__global__ void group_validate_kernel(GroupArgs a, GroupScratch s) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += gridDim.x * blockDim.x) {
        bool ok = a.model[r] >= 0 && a.model[r] < a.M && a.out[r] >= 0 && a.out[r] <= 65535 &&
                  a.slo[r] > 0.0;
        for (int f = 0; f < a.dims; ++f) ok = ok && a.feat[r * a.dims + f] >= 0 && a.feat[r * a.dims + f] <= 65535;
        if (!ok) atomicAdd(s.bad, 1);
    }
}

__global__ void fp_first_kernel(GroupArgs a, GroupScratch s) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += gridDim.x * blockDim.x) {
        atomicMin(&s.first[a.model[r]], r);
        s.mind[r] = INT64_MAX;
        a.label[r] = -1;
    }
}

// after fp_first: c_0 of every model = its first request (R21)
__global__ void fp_setup_kernel(GroupArgs a, GroupScratch s) {
    for (int m = threadIdx.x; m < a.M; m += blockDim.x) {
        const bool has = s.first[m] < a.n && s.k_req[m] >= 1;
        if (has) s.init_req[s.off_req[m]] = s.first[m];
        s.k_eff[m] = has ? 1 : 0;
        s.active[m] = has && s.k_req[m] > 1;
        s.best[m] = 0ull;
    }
}

// one farthest-point round: fold the newest centre of each active model into
// every request's min distance and take the per-model max (lowest index on ties)
__global__ void __launch_bounds__(256) fp_round_kernel(GroupArgs a, GroupScratch s) {
    __shared__ unsigned long long sb[64];
    for (int m = threadIdx.x; m < a.M; m += blockDim.x) sb[m] = 0ull;
    __syncthreads();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += gridDim.x * blockDim.x) {
        const int m = a.model[r];
        if (!s.active[m]) continue;
        const int c = s.init_req[s.off_req[m] + s.k_eff[m] - 1];
        int64_t d2 = 0;
        for (int f = 0; f < a.dims; ++f) {
            const int64_t t = (int64_t)a.feat[r * a.dims + f] - a.feat[c * a.dims + f];
            d2 += t * t;
        }
        s.mind[r] = min(s.mind[r], d2);
    }
    // per-model max of the packed key: warp REDUX on the two 32-bit halves (a
    // 64-bit shared-memory atomic is a CAS loop), then one atomic per warp
    __syncthreads();
    for (int r0 = blockIdx.x * blockDim.x; r0 < a.n; r0 += gridDim.x * blockDim.x) {
        const int r = r0 + threadIdx.x;
        const int m = r < a.n ? a.model[r] : -1;
        const bool act = m >= 0 && s.active[m];
        const unsigned long long key =
            act ? ((unsigned long long)s.mind[r] << kIdxBits) | (kIdxMask - (uint64_t)r) : 0ull;
        for (int mm = 0; mm < a.M; ++mm) {
            if (!__any_sync(0xFFFFFFFFu, act && m == mm)) continue;
            const unsigned hi = (act && m == mm) ? (unsigned)(key >> 32) : 0u;
            const unsigned hmax = __reduce_max_sync(0xFFFFFFFFu, hi);
            const unsigned lo = (act && m == mm && hi == hmax) ? (unsigned)key : 0u;
            const unsigned lmax = __reduce_max_sync(0xFFFFFFFFu, lo);
            if ((threadIdx.x & 31) == 0) atomicMax(&sb[mm], ((unsigned long long)hmax << 32) | lmax);
        }
    }
    __syncthreads();
    for (int m = threadIdx.x; m < a.M; m += blockDim.x)
        if (sb[m]) atomicMax(&s.best[m], sb[m]);
}

__global__ void fp_pick_kernel(GroupArgs a, GroupScratch s) {
    for (int m = threadIdx.x; m < a.M; m += blockDim.x) {
        if (!s.active[m]) continue;
        const unsigned long long key = s.best[m];
        s.best[m] = 0ull;
        if ((key >> kIdxBits) == 0ull) {           // no distinct point left
            s.active[m] = 0;
            continue;
        }
        s.init_req[s.off_req[m] + s.k_eff[m]] = (int)(kIdxMask - (key & kIdxMask));
        s.k_eff[m] += 1;
        s.active[m] = s.k_eff[m] < s.k_req[m];
    }
}

// compact the effective centres (model order) and load their coordinates
__global__ void fp_compact_kernel(GroupArgs a, GroupScratch s) {
    if (threadIdx.x == 0) {
        int K = 0;
        for (int m = 0; m < a.M; ++m) { s.off[m] = K; K += s.k_eff[m]; }
        s.off[a.M] = K;
    }
    __syncthreads();
    for (int m = 0; m < a.M; ++m)
        for (int j = threadIdx.x; j < s.k_eff[m]; j += blockDim.x) {
            const int r = s.init_req[s.off_req[m] + j], cj = s.off[m] + j;
            for (int f = 0; f < 4; ++f) s.C[cj * 4 + f] = f < a.dims ? (double)a.feat[r * a.dims + f] : 0.0;
        }
    for (int i = threadIdx.x; i < a.Kmax * 5; i += blockDim.x) s.sums[i] = 0ull;
    if (threadIdx.x == 0) { *s.changed = 0u; *s.conv = 0u; *s.iters = 0u; }
}

// Lloyd assignment step (R21): nearest centre of the request's model,
// d2 = sum_f ((double)x_f - c_f)^2 in f order, strict < (lowest index on ties)
__global__ void __launch_bounds__(256) lloyd_assign_kernel(GroupArgs a, GroupScratch s) {
    if (*s.conv) return;
    extern __shared__ __align__(16) uint8_t smem[];
    // per-block sums in 32-bit shared atomics (native; a block sees <= 32768
    // requests, so coordinate sums stay below 2^31), flushed as 64-bit adds
    double *sC = reinterpret_cast<double *>(smem);                                   // [Kmax][4]
    unsigned *ssum = reinterpret_cast<unsigned *>(sC + a.Kmax * 4);                  // [Kmax][5]
    int *soff = reinterpret_cast<int *>(ssum + a.Kmax * 5);                          // [M + 1]
    const int K = s.off[a.M];
    for (int i = threadIdx.x; i < K * 4; i += blockDim.x) sC[i] = s.C[i];
    for (int i = threadIdx.x; i < K * 5; i += blockDim.x) ssum[i] = 0u;
    for (int i = threadIdx.x; i <= a.M; i += blockDim.x) soff[i] = s.off[i];
    __syncthreads();
    unsigned nchg = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += gridDim.x * blockDim.x) {
        const int m = a.model[r];
        double x[4];
        for (int f = 0; f < 4; ++f) x[f] = f < a.dims ? (double)a.feat[r * a.dims + f] : 0.0;
        int arg = -1;
        double best = __longlong_as_double(0x7FF0000000000000ll);   // +inf
        for (int j = soff[m]; j < soff[m + 1]; ++j) {
            double d2 = 0.0;
            for (int f = 0; f < a.dims; ++f) {
                const double t = __dsub_rn(x[f], sC[j * 4 + f]);
                d2 = __dadd_rn(d2, __dmul_rn(t, t));
            }
            if (d2 < best) { best = d2; arg = j; }
        }
        if (arg != a.label[r]) { a.label[r] = arg; ++nchg; }
        if (arg >= 0) {
            for (int f = 0; f < a.dims; ++f) atomicAdd(&ssum[arg * 5 + f], (unsigned)a.feat[r * a.dims + f]);
            atomicAdd(&ssum[arg * 5 + 4], 1u);
        }
    }
    const unsigned wchg = __reduce_add_sync(0xFFFFFFFFu, nchg);
    if ((threadIdx.x & 31) == 0 && wchg) atomicAdd(s.changed, wchg);
    __syncthreads();
    for (int i = threadIdx.x; i < K * 5; i += blockDim.x)
        if (ssum[i]) atomicAdd(&s.sums[i], (unsigned long long)ssum[i]);
}

// Lloyd update step: stop when no label changed, else centres = exact integer
// sums / counts (an empty cluster keeps its centre); clears the accumulators
__global__ void lloyd_update_kernel(GroupArgs a, GroupScratch s) {
    __shared__ int stop;
    if (threadIdx.x == 0) {
        stop = *s.conv;
        if (!stop) {
            *s.iters += 1u;
            if (*s.changed == 0u) { *s.conv = 1u; stop = 1; }
        }
    }
    __syncthreads();
    const int K = s.off[a.M];
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
        const unsigned long long cnt = s.sums[j * 5 + 4];
        if (!stop && cnt > 0ull)
            for (int f = 0; f < a.dims; ++f)
                s.C[j * 4 + f] = __ddiv_rn((double)(long long)s.sums[j * 5 + f], (double)(long long)cnt);
        for (int f = 0; f < 5; ++f) s.sums[j * 5 + f] = 0ull;
    }
    __syncthreads();
    if (threadIdx.x == 0) *s.changed = 0u;
}

// Stable rank inside the cluster, block part: 1024 requests per block, warps
// in order through a shared running count per cluster.
__global__ void __launch_bounds__(1024) rank_block_kernel(GroupArgs a, GroupScratch s) {
    extern __shared__ int running[];                 // [Kmax]
    for (int i = threadIdx.x; i < a.Kmax; i += blockDim.x) running[i] = 0;
    const int r = blockIdx.x * 1024 + threadIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int lab = r < a.n ? a.label[r] : -1;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, lab);
    const int lrank = __popc(peers & ((1u << lane) - 1u));
    const bool leader = lrank == 0;
    const int cnt = __popc(peers);
    int rank = 0;
    for (int ww = 0; ww < 32; ++ww) {
        __syncthreads();
        if (w == ww && lab >= 0) {
            rank = running[lab] + lrank;
            __syncwarp(peers);
            if (leader) running[lab] += cnt;
        }
    }
    __syncthreads();
    if (r < a.n) s.inrank[r] = rank;
    for (int i = threadIdx.x; i < a.Kmax; i += blockDim.x) s.bcount[(size_t)blockIdx.x * a.Kmax + i] = running[i];
}

// number of groups splitHalf makes of a cluster of size x (R21): pieces at
// depth l have sizes floor(x / 2^l) or ceil(x / 2^l), so leaf counts are
// computed bottom-up for two sizes per level
__device__ int64_t split_leaves(int64_t x, int L) {
    if (x <= 0) return 0;
    if (x <= L) return 1;
    int D = 0;
    while (((x + (1ll << D) - 1) >> D) > L) ++D;
    int64_t lo = x >> D, hi = (x + (1ll << D) - 1) >> D;
    int64_t flo = lo > 0 ? 1 : 0, fhi = hi > 0 ? 1 : 0;
    for (int l = D - 1; l >= 0; --l) {
        const int64_t nlo = x >> l, nhi = (x + (1ll << l) - 1) >> l;
        auto f = [&](int64_t y) -> int64_t {
            if (y <= L) return y > 0 ? 1 : 0;
            const int64_t c = (y + 1) >> 1, fl = y >> 1;
            return (c == hi ? fhi : flo) + (fl == hi ? fhi : flo);
        };
        const int64_t a = f(nlo), b = f(nhi);
        lo = nlo; hi = nhi; flo = a; fhi = b;
    }
    return fhi;                                       // level 0: lo == hi == x
}

// column scan of the block counts (cluster offsets per block), cluster sizes,
// leaf counts and group bases (single block)
__global__ void rank_scan_kernel(GroupArgs a, GroupScratch s) {
    const int K = s.off[a.M];
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
        int acc = 0;
        for (int b = 0; b < a.nb; ++b) {
            int *p = &s.bcount[(size_t)b * a.Kmax + j];
            const int t = *p;
            *p = acc;
            acc += t;
        }
        s.size[j] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int g = 0;
        for (int j = 0; j < K; ++j) { s.base[j] = g; g += (int)split_leaves(s.size[j], a.limit); }
        s.base[a.Kmax] = g;
    }
}

__global__ void group_assign_kernel(GroupArgs a, GroupScratch s) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += gridDim.x * blockDim.x) {
        const int j = a.label[r];
        const int b = r >> 10;
        const int64_t rank = (int64_t)s.bcount[(size_t)b * a.Kmax + j] + s.inrank[r];
        int64_t lo = 0, x = s.size[j], leaf = 0;
        while (x > a.limit) {                        // splitHalf descent: first half = ceil
            const int64_t half = (x + 1) >> 1;
            if (rank - lo < half) x = half;
            else { leaf += split_leaves(half, a.limit); lo += half; x -= half; }
        }
        const int gid = s.base[j] + (int)leaf;
        a.group_of[r] = gid;
        const unsigned long long o = (unsigned long long)a.out[r];
        unsigned long long *g = s.gacc + (size_t)gid * 4;
        atomicAdd(&g[0], o);
        atomicAdd(&g[1], o * o);
        atomicMin(&g[2], (unsigned long long)__double_as_longlong(a.slo[r]));   // slo > 0: bits order
        atomicAdd(&g[3], 1ull);
        s.gmodel[gid] = a.model[r];
    }
}

__global__ void group_init_slo(unsigned long long *gacc, int gmax) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < gmax) gacc[(size_t)g * 4 + 2] = ~0ull;
}

__global__ void group_finalize_kernel(GroupArgs a, GroupScratch s) {
    const int G = s.base[a.Kmax];
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < G && g < a.group_cap; g += gridDim.x * blockDim.x) {
        const unsigned long long *x = s.gacc + (size_t)g * 4;
        const long long n = (long long)x[3], s1 = (long long)x[0], s2 = (long long)x[1];
        qlm_group q;
        q.model = s.gmodel[g];
        q.n_req = (int32_t)n;
        q.slo_s = __longlong_as_double((long long)x[2]);
        q.mu_out = __ddiv_rn((double)s1, (double)n);
        q.var_out = __ddiv_rn((double)(n * s2 - s1 * s1), __dmul_rn((double)n, (double)n));
        q.dist_id = -1;
        q.reserved = 0;
        a.groups[g] = q;
    }
}

static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

cudaError_t launch_form_groups(int n, int dims, int M, const int32_t *k_host, int limit, int max_iter,
                               const int32_t *model, const double *slo, const int32_t *out,
                               const int32_t *feat, int32_t *label, int32_t *group_of,
                               qlm_group *groups, int group_cap, int32_t *n_groups, int32_t *iters,
                               int32_t *n_bad, cudaStream_t st) {
    int Kmax = 0, kmax = 0;
    for (int m = 0; m < M; ++m) { Kmax += k_host[m]; kmax = k_host[m] > kmax ? k_host[m] : kmax; }
    const int nb = (n + 1023) / 1024;
    const int gmax = n;                              // every group holds >= 1 request
    // scratch: one allocation
    size_t o = 0;
    const size_t o_mind = o; o = a256(o + (size_t)n * 8);
    const size_t o_first = o; o = a256(o + (size_t)M * 4);
    const size_t o_best = o; o = a256(o + (size_t)M * 8);
    const size_t o_kreq = o; o = a256(o + (size_t)M * 4);
    const size_t o_keff = o; o = a256(o + (size_t)M * 4);
    const size_t o_act = o; o = a256(o + (size_t)M * 4);
    const size_t o_offr = o; o = a256(o + (size_t)M * 4);
    const size_t o_init = o; o = a256(o + (size_t)(Kmax + 1) * 4);
    const size_t o_off = o; o = a256(o + (size_t)(M + 1) * 4);
    const size_t o_C = o; o = a256(o + (size_t)(Kmax + 1) * 32);
    const size_t o_sums = o; o = a256(o + (size_t)(Kmax + 1) * 40);
    const size_t o_flags = o; o = a256(o + 16);
    const size_t o_inrank = o; o = a256(o + (size_t)n * 4);
    const size_t o_bcount = o; o = a256(o + (size_t)nb * (Kmax + 1) * 4);
    const size_t o_size = o; o = a256(o + (size_t)(Kmax + 1) * 4);
    const size_t o_base = o; o = a256(o + (size_t)(Kmax + 1) * 4);
    const size_t o_gacc = o; o = a256(o + (size_t)gmax * 32);
    const size_t o_gmodel = o; o = a256(o + (size_t)gmax * 4);
    // scratch: a per-device cache that only grows (a fresh stream-ordered
    // allocation per call costs a page-mapping round trip each time)
    static std::mutex mu;
    static void *cache[64] = {};
    static size_t cache_bytes[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaSuccess;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (cache_bytes[dev] < o) {
        if ((e = cudaStreamSynchronize(st))) return e;
        if (cache[dev]) cudaFree(cache[dev]);
        cache[dev] = nullptr;
        cache_bytes[dev] = 0;
        if ((e = cudaMalloc(&cache[dev], o))) return e;
        cache_bytes[dev] = o;
    }
    uint8_t *buf = static_cast<uint8_t *>(cache[dev]);
    GroupScratch s;
    s.mind = reinterpret_cast<int64_t *>(buf + o_mind);
    s.first = reinterpret_cast<int32_t *>(buf + o_first);
    s.best = reinterpret_cast<unsigned long long *>(buf + o_best);
    s.k_req = reinterpret_cast<int32_t *>(buf + o_kreq);
    s.k_eff = reinterpret_cast<int32_t *>(buf + o_keff);
    s.active = reinterpret_cast<int32_t *>(buf + o_act);
    s.off_req = reinterpret_cast<int32_t *>(buf + o_offr);
    s.init_req = reinterpret_cast<int32_t *>(buf + o_init);
    s.off = reinterpret_cast<int32_t *>(buf + o_off);
    s.C = reinterpret_cast<double *>(buf + o_C);
    s.sums = reinterpret_cast<unsigned long long *>(buf + o_sums);
    s.changed = reinterpret_cast<uint32_t *>(buf + o_flags);
    s.conv = s.changed + 1;
    s.iters = s.changed + 2;
    s.bad = reinterpret_cast<int32_t *>(s.changed + 3);
    s.inrank = reinterpret_cast<int32_t *>(buf + o_inrank);
    s.bcount = reinterpret_cast<int32_t *>(buf + o_bcount);
    s.size = reinterpret_cast<int32_t *>(buf + o_size);
    s.base = reinterpret_cast<int32_t *>(buf + o_base);
    s.gacc = reinterpret_cast<unsigned long long *>(buf + o_gacc);
    s.gmodel = reinterpret_cast<int32_t *>(buf + o_gmodel);
    // host-known per-model inputs: k and the init slot offsets
    int32_t hk[2 * 64];
    for (int m = 0, acc = 0; m < M; ++m) { hk[m] = k_host[m]; hk[64 + m] = acc; acc += k_host[m]; }
    GroupArgs a;
    a.n = n; a.dims = dims; a.M = M; a.Kmax = Kmax; a.limit = limit; a.nb = nb; a.gmax = gmax;
    a.model = model; a.out = out; a.feat = feat; a.slo = slo;
    a.label = label; a.group_of = group_of; a.groups = groups; a.group_cap = group_cap;
    const int sms = sm_count();
    int grid = (int)((n + 255) / 256 < (int64_t)sms * 8 ? (n + 255) / 256 : sms * 8);
    if (grid < (n + 32767) / 32768) grid = (n + 32767) / 32768;   // <= 32768 requests per block
    do {
        if ((e = cudaMemsetAsync(buf + o_flags, 0, 16, st))) break;
        if ((e = cudaMemsetAsync(s.first, 0x7F, (size_t)M * 4, st))) break;
        if ((e = cudaMemcpyAsync(s.k_req, hk, (size_t)M * 4, cudaMemcpyHostToDevice, st))) break;
        if ((e = cudaMemcpyAsync(s.off_req, hk + 64, (size_t)M * 4, cudaMemcpyHostToDevice, st))) break;
        group_validate_kernel<<<grid, 256, 0, st>>>(a, s);
        if ((e = cudaMemcpyAsync(n_bad, s.bad, 4, cudaMemcpyDeviceToHost, st))) break;
        if ((e = cudaStreamSynchronize(st))) break;
        g_launches += 1;
        if (*n_bad) break;
        if ((e = cudaMemsetAsync(s.gacc, 0, (size_t)gmax * 32, st))) break;
        fp_first_kernel<<<grid, 256, 0, st>>>(a, s);
        fp_setup_kernel<<<1, 64, 0, st>>>(a, s);
        for (int j = 1; j < kmax; ++j) {
            fp_round_kernel<<<grid, 256, 0, st>>>(a, s);
            fp_pick_kernel<<<1, 64, 0, st>>>(a, s);
        }
        fp_compact_kernel<<<1, 256, 0, st>>>(a, s);
        g_launches += 3 + 2 * (kmax > 1 ? kmax - 1 : 0);
        const size_t smem_assign = (size_t)Kmax * 52 + (size_t)(M + 1) * 4 + 16;
        if (smem_assign > 48 * 1024 &&
            (e = cudaFuncSetAttribute(lloyd_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem_assign)))
            break;
        // fewer, fuller blocks for the assignment: every block flushes K*5
        // global atomics per iteration, so the block count sets the contention
        int agrid = sms * 4;
        if (agrid > (n + 255) / 256) agrid = (n + 255) / 256;
        if (agrid < (n + 32767) / 32768) agrid = (n + 32767) / 32768;
        for (int it = 0; it < max_iter; ++it) {
            lloyd_assign_kernel<<<agrid, 256, smem_assign, st>>>(a, s);
            lloyd_update_kernel<<<1, 1024, 0, st>>>(a, s);
        }
        g_launches += 2 * max_iter;
        const size_t smem_rank = (size_t)(Kmax + 1) * 4;
        if (smem_rank > 48 * 1024 &&
            (e = cudaFuncSetAttribute(rank_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem_rank)))
            break;
        rank_block_kernel<<<nb, 1024, smem_rank, st>>>(a, s);
        rank_scan_kernel<<<1, 1024, 0, st>>>(a, s);
        group_init_slo<<<(gmax + 255) / 256, 256, 0, st>>>(s.gacc, gmax);   // min-SLO starts at max bits
        group_assign_kernel<<<grid, 256, 0, st>>>(a, s);
        group_finalize_kernel<<<(n + 255) / 256 < sms * 8 ? (n + 255) / 256 : sms * 8, 256, 0, st>>>(a, s);
        g_launches += 6;
        if ((e = cudaGetLastError())) break;
        if ((e = cudaMemcpyAsync(n_groups, s.base + Kmax, 4, cudaMemcpyDeviceToHost, st))) break;
        if ((e = cudaMemcpyAsync(iters, s.iters, 4, cudaMemcpyDeviceToHost, st))) break;
        e = cudaStreamSynchronize(st);
    } while (0);
    return e;
}

}  // namespace qlm
