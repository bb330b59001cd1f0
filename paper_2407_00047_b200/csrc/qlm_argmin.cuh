// qlm_argmin.cuh -- in-kernel argmin over (key, index) records (R11/R14),
// shared by the warp-specialised and the warp-per-candidate kernels.
#pragma once
#include "qlm_device.cuh"
#include "qlm_launch.h"

namespace qlm {

// Warp -> block -> grid (last block) lexicographic argmin (R11/R14).
__device__ __forceinline__ void block_grid_argmin(const ScanParams &p, uint64_t bkey, int64_t bidx) {
    __shared__ uint64_t rk[32];
    __shared__ int64_t ri[32];
    __shared__ int is_last;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
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
            is_last = atomicAdd(p.counter, 1u) == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    uint64_t k = ~0ull;
    int64_t i = -1;
    for (int j = tid; j < (int)gridDim.x; j += blockDim.x) {
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

}  // namespace qlm
