// qlm_req.cu -- request-level violating fractions (DESIGN R19).
//
// Request r = 0..n_i-1 of group i waits wt_i + r mu_i/Theta with variance
// V_i + r sigma_i^2/Theta^2 (Eq. 2/3 with q over requests);
// f_i = (1/n_i) sum_r v_r (R8/R9) and S1_req = sum n_i f_i / sum n_i.
//
// One warp per candidate.  The warp materialises the row (any candidate
// kind), then lane q walks queue q in row order -- the oracle's operation
// order, so wt_i / V_i are bit-identical to it -- and finally all 32 lanes
// split each group's requests (lane l takes r = l, l+32, ...) and reduce.
#include <cuda_runtime.h>

#include "qlm_device.cuh"
#include "qlm_launch.h"

namespace qlm {

constexpr int kReqWarps = 8;

__global__ void __launch_bounds__(256) req_kernel(const ScanParams p, const qlm_group *groups,
                                                  float *frac, float *s1r, int warp_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Dims dm = p.dm;
    const int G = dm.G, Q = dm.Q, T = dm.T, M = dm.M;
    const Cand cd = p.cd;
    const int64_t loc = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (loc >= cd.count) return;                              // warp-uniform
    int64_t first = cd.first;
    if (cd.first_from) {
        first = cd.first_from->index;
        if (first < 0) return;
    }
    uint8_t *base = smem + (size_t)warp * warp_bytes;
    double *swt = reinterpret_cast<double *>(base);                 // [G]
    double *sV = swt + G;                                           // [G]
    int32_t *sdev = reinterpret_cast<int32_t *>(sV + G);            // [G]
    int32_t *qbeg = sdev + G;                                       // [Q + 1]
    uint16_t *srow = reinterpret_cast<uint16_t *>(qbeg + Q + 1);    // [T]
    uint16_t *sJ = srow + ((T + 7) & ~7);                           // [T]
    warp_gen_row(cd, T, (uint64_t)(first + loc), loc, srow, sJ);
    // queue boundaries: queue q covers positions [qbeg[q], qbeg[q+1] - 1)
    if (lane == 0) qbeg[0] = 0;
    int nsep = 0;
    for (int s0 = 0; s0 < T; s0 += 32) {
        const int s = s0 + lane;
        const bool sep = s < T && srow[s] >= G;
        const uint32_t bs = __ballot_sync(0xFFFFFFFFu, sep);
        if (sep) {
            const int k = nsep + __popc(bs & ((1u << lane) - 1u));   // k-th separator ends queue k
            if (k + 1 <= Q - 1) qbeg[k + 1] = s + 1;
        }
        nsep += __popc(bs);
    }
    if (lane == 0) qbeg[Q] = T + 1;
    __syncwarp();
    // Eq. 10 walk, one lane per queue, in the oracle's order (R1-R7, R12)
    for (int q = lane; q < Q; q += 32) {
        const QRec qr = p.tb.qrec[q];
        const int d = qr.d;
        double A = qr.bmean, B = qr.bvar;
        int prev = qr.r, firsts = 1;
        const int s1 = qbeg[q + 1] - 1;
        for (int s = qbeg[q]; s < s1; ++s) {
            const int g = srow[s];
            const int m = p.tb.grec[g].model;
            if (m != prev) {                                     // one transition term (R2)
                double trans = p.tb.swap[(d * M + prev) * M + m];
                if (!firsts || qr.backlog) trans = __dadd_rn(p.tb.tail[d * M + prev], trans);
                A = __dadd_rn(A, trans);
            }
            swt[g] = A;
            sV[g] = B;
            sdev[g] = d;
            const double2 ab = p.tb.ab[d * G + g];
            A = __dadd_rn(A, ab.x);
            B = __dadd_rn(B, ab.y);
            prev = m;
            firsts = 0;
        }
    }
    __syncwarp();
    // per-request violations: lanes split each group's requests
    const double zc2 = p.zc2;
    const int64_t count = cd.count;
    double num = 0.0, den = 0.0;
    for (int g = 0; g < G; ++g) {
        const GRec gr = p.tb.grec[g];
        const double th = p.tb.theta[sdev[g] * M + gr.model];
        const double a = __ddiv_rn(groups[g].mu_out, th);
        const double b = __ddiv_rn(groups[g].var_out, __dmul_rn(th, th));
        const double wt = swt[g], V = sV[g];
        double sum = 0.0;
        for (int r = lane; r < gr.n; r += 32) {
            const double mean = __dadd_rn(wt, __dmul_rn((double)r, a));
            const double var = __dadd_rn(V, __dmul_rn((double)r, b));
            bool clamped;
            sum += (double)violation(__dsub_rn(gr.slo, mean), var, zc2, clamped);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
        const double f = sum / (double)gr.n;
        if (lane == 0 && frac) frac[(int64_t)g * count + loc] = (float)f;
        num += (double)gr.n * f;
        den += (double)gr.n;
    }
    if (lane == 0 && s1r) s1r[loc] = (float)(num / den);
}

cudaError_t launch_req(const ScanParams &p, const qlm_group *groups, float *frac, float *s1r,
                       cudaStream_t st) {
    const Dims &dm = p.dm;
    const int warp_bytes = (int)(((size_t)16 * dm.G + 4 * (size_t)dm.G + 4 * (size_t)(dm.Q + 1) +
                                  4 * (size_t)((dm.T + 7) & ~7) + 15) & ~size_t(15));
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    int W = (int)(((size_t)optin - 1024) / (size_t)warp_bytes);   // up to 8 warps (one per candidate)
    if (W > kReqWarps) W = kReqWarps;
    if (W < 1) return cudaErrorInvalidConfiguration;
    const size_t smem = (size_t)warp_bytes * W;
    cudaError_t e = cudaFuncSetAttribute(req_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = (p.cd.count + W - 1) / W;
    req_kernel<<<(unsigned)grid, 32 * W, smem, st>>>(p, groups, frac, s1r, warp_bytes);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace qlm
