// qlm_big.cu -- scoring path for very large G (the fallback when no
// shared-memory plan of the other scan kernels fits: G above ~2000).
//
// One warp per candidate, one lane per queue (DESIGN R1-R9 in the oracle's
// sequential order per queue, so wt / V are bit-identical to it).  Only the
// candidate's row lives in shared memory (warp_gen_row: 4T bytes per warp);
// the group, work, queue and transition tables are read from global memory
// through the read-only path (they stay L1/L2-resident).  Bulk outputs are
// stored straight to the group-major arrays: at this size every candidate
// writes thousands of groups, so the kernel is a correctness-first fallback
// rather than a bandwidth path.
#include <cuda_runtime.h>

#include "qlm_argmin.cuh"
#include "qlm_device.cuh"
#include "qlm_launch.h"

namespace qlm {

template <bool TIER>
__global__ void __launch_bounds__(256) big_kernel(const ScanParams p, int ldr) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
    const Dims dm = p.dm;
    const int G = dm.G, Q = dm.Q, T = dm.T, M = dm.M;
    const size_t per_warp = ((size_t)4 * ldr + 4 * (size_t)(Q + 1) + 15) & ~size_t(15);
    uint16_t *srow = reinterpret_cast<uint16_t *>(smem + (size_t)warp * per_warp);
    uint16_t *sJ = srow + ldr;
    int *qbeg = reinterpret_cast<int *>(sJ + ldr);
    const Cand cd = p.cd;
    int64_t first = cd.first;
    bool none = false;
    if (cd.first_from) {
        first = cd.first_from->index;
        none = first < 0;
    }
    const int64_t count = none ? 0 : cd.count;
    const int64_t ldo = p.ld_out ? p.ld_out : count;
    const float zc = p.zc;
    const float alpha = p.alpha;
    const double den = *p.tb.den;
    uint64_t bkey = ~0ull;
    int64_t bidx = -1;
    for (int64_t loc = (int64_t)blockIdx.x * W + warp; loc < count; loc += (int64_t)gridDim.x * W) {
        warp_gen_row(cd, T, (uint64_t)(first + loc), loc, srow, sJ);
        if (lane == 0) qbeg[0] = 0;                       // queue q: positions [qbeg[q], qbeg[q+1] - 1)
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
            const QRec qr = p.tb.qrec[q];
            const int d = qr.d;
            double A = qr.bmean;
            float B = (float)qr.bvar;                     // fp32 (R22)
            int prev = qr.r;
            bool firsts = true;
            uint32_t seen = 0u, warm = 0u;                // two-tier state (R20), per queue
            int cum = 0;
            bool exh = false;
            const int s1 = qbeg[q + 1] - 1;
            for (int s = qbeg[q]; s < s1; ++s) {
                const int g = srow[s];
                const GRec gr = p.tb.grec[g];
                const int m = gr.model;
                if (m != prev) {                          // one transition term (R1/R2/R4/R12)
                    double trans = __ldg(&p.tb.swap[(d * M + prev) * M + m]);
                    if constexpr (TIER) {                 // R20: cold targets pay the registry load
                        const uint32_t bit = 1u << m;
                        if (!(seen & bit)) {
                            seen |= bit;
                            const int need = cum + __ldg(&p.t_mem[m]);
                            if (!exh && need <= __ldg(&p.t_cap[d])) { warm |= bit; cum = need; }
                            else exh = true;
                        }
                        if (!(warm & bit)) trans = __dadd_rn(trans, __ldg(&p.t_load[d * M + m]));
                    }
                    if (!firsts || qr.backlog) trans = __dadd_rn(__ldg(&p.tb.tail[d * M + prev]), trans);
                    A = __dadd_rn(A, trans);
                }
                const double wt = A;                      // exclusive (R5)
                const float V = B;
                const double2 ab = p.tb.ab[d * G + g];
                A = __dadd_rn(A, ab.x);
                B = __fadd_rn(B, (float)ab.y);
                prev = m;
                firsts = false;
                const double slack = __dsub_rn(gr.slo, wt);
                const float sd = slot_sd(V);
                bool clamped;
                const float v = slot_v(slack, sd, zc, clamped);
                S2 = __dsub_rn(S2, slack);
                num = __dadd_rn(num, (double)gr.n * (double)v);
                over += v > alpha;
                const int64_t o = (int64_t)g * ldo + loc;
                if (p.wt) p.wt[o] = (float)wt;
                if (p.sd) p.sd[o] = sd;
                if (p.vo) p.vo[o] = v;
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
            const uint64_t key = make_key(s1v, s2v);
            if (better(key, first + loc, bkey, bidx)) { bkey = key; bidx = first + loc; }
        }
        __syncwarp();
    }
    if (p.out_rec) {
        if (none) {
            if (blockIdx.x == 0 && threadIdx.x == 0) { p.out_rec->key = ~0ull; p.out_rec->index = -1; }
            return;
        }
        block_grid_argmin(p, bkey, bidx);
    }
}

template <bool TIER>
static cudaError_t launch_big_t(const ScanParams &p, cudaStream_t st) {
    auto kern = big_kernel<TIER>;
    const Dims &dm = p.dm;
    const int ldr = (dm.T + 7) & ~7;
    const size_t per_warp = ((size_t)4 * ldr + 4 * (size_t)(dm.Q + 1) + 15) & ~size_t(15);
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    const size_t avail = (size_t)optin > fa.sharedSizeBytes + 1024 ? (size_t)optin - fa.sharedSizeBytes - 1024 : 0;
    int W = (int)(avail / per_warp);
    if (W > 8) W = 8;
    if (W < 1) return cudaErrorNotSupported;
    const size_t smem = per_warp * W;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
        return e;
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32 * W, smem);
    if (nb < 1) nb = 1;
    int64_t grid = (p.cd.count + W - 1) / W;
    if (grid > (int64_t)sm_count() * nb) grid = (int64_t)sm_count() * nb;
    if (grid > p.max_blocks) grid = p.max_blocks;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 32 * W, smem, st>>>(p, ldr);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_big(const ScanParams &p, cudaStream_t st) { return launch_big_t<false>(p, st); }
cudaError_t launch_big_tier(const ScanParams &p, cudaStream_t st) { return launch_big_t<true>(p, st); }

}  // namespace qlm
