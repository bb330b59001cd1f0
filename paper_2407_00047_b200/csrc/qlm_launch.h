// qlm_launch.h -- launchers shared by qlm_api.cu and qlm_kernels.cu (internal).
#pragma once

#include <atomic>

#include "qlm_device.cuh"

namespace qlm {

struct ScanParams {
    Dims dm;
    Tables tb;
    Cand cd;
    float *s1, *s2;            // score outputs [count] (nullable)
    int32_t *n_over;
    float *wt, *sd, *vo;       // bulk outputs, group-major [G][count] (nullable)
    qlm_record *block_recs;    // [max_blocks] argmin scratch
    unsigned int *counter;     // last-block ticket
    qlm_record *out_rec;       // argmin result (nullable = no argmin)
    int max_blocks;
    double zc2;                // z_clamp^2
    float zc;                  // z_clamp (fp32: the clamp test of R9/R22)
    float alpha;
    int blk;
    int use_tma;               // staged outputs leave through bulk async copies
    int n_out;                 // number of non-null bulk outputs
    int rep_shift;             // group tables replicated 1 << rep_shift times in smem
    int tr_shift;              // transition table replicated 1 << tr_shift times (scan kernel)
    int off_grec, off_ab, off_q, off_tr, off_scratch, off_stage;
    int64_t ld_out;            // leading dimension of the bulk outputs (0 = count)
    uint32_t *ilv;             // large-T RANDOM: word-interleaved row scratch [words][ilv_cap]
    int64_t ilv_cap;           // candidates per chunk that fit the scratch
    qlm_record *chunk_recs;    // [2] running argmin across chunks
    const int32_t *t_mem;      // two-tier swapping (R20): model sizes [M]
    const int32_t *t_cap;      // CPU memory per device row [D]
    const double *t_load;      // storage -> CPU load time [D][M]
    int slo_hi_only;           // every slo_s has a zero low 32-bit word (qlm_ws2.cu records)
};


extern std::atomic<int64_t> g_launches;
// qlm_set_kernel_overrides (tests: compare kernel paths on one process)
extern std::atomic<uint32_t> g_override_flags;
extern std::atomic<int64_t> g_override_ilv_cap;
inline bool override_on(uint32_t bit) { return (g_override_flags.load(std::memory_order_relaxed) & bit) != 0; }
int sm_count();                                 // of the current device (cached per device)
int env_cached(const char *name, int dflt);     // tuning/test overrides, read once per process
// Host logging (QLM_LOG=1: entry points and the kernel each call launches,
// with its grid and shared memory; QLM_LOG=2 adds per-launch argument detail),
// to stderr with a "[qlm]" prefix.  Off by default; read once per process.
int log_level();
void qlog(int level, const char *fmt, ...) __attribute__((format(printf, 2, 3)));

cudaError_t launch_build(const Dims &dm, const qlm_group *g, const qlm_queue *q,
                         const double *theta, const double *prefill, const double *eps,
                         const double *dec, const double *maxo, const double *swp,
                         const Tables &tb, cudaStream_t st);
cudaError_t launch_scan(ScanParams p, cudaStream_t st);
cudaError_t launch_ws(ScanParams p, cudaStream_t st);      // warp-specialised fast path
cudaError_t launch_ws2(const ScanParams &p, cudaStream_t st);  // same, D = 1 / byte rows (qlm_ws2.cu)
cudaError_t launch_ws_tier(ScanParams p, cudaStream_t st); // same, two-tier swapping (R20)
cudaError_t launch_ws2_tier(const ScanParams &p, cudaStream_t st);  // ws2 with R20 (D = 1 / byte rows)
cudaError_t launch_any_scan(const ScanParams &p, cudaStream_t st);   // ws, else scan
cudaError_t launch_wide(const ScanParams &p, cudaStream_t st);      // warp per candidate (large G)
cudaError_t launch_large(const ScanParams &p, cudaStream_t st);     // D = 1 score-only over 16-bit ILV rows
cudaError_t launch_big(const ScanParams &p, cudaStream_t st);       // very large G: global tables
cudaError_t launch_big_tier(const ScanParams &p, cudaStream_t st);  // same, two-tier swapping (R20)
cudaError_t launch_req(const ScanParams &p, const qlm_group *groups, float *frac, float *s1r,
                       cudaStream_t st);                            // request-level (R19)
cudaError_t launch_tier(const ScanParams &p, cudaStream_t st);     // two-tier swapping (R20)
// large-T RANDOM rows of candidates [g.first, g.first + n), word-interleaved
// into `out` (word w of candidate l at out[w * n + l]); fy_rows_kernel
cudaError_t launch_fy_rows(const Cand &g, int T, uint32_t *out, int64_t n, cudaStream_t st);
cudaError_t launch_form_groups(int n, int dims, int M, const int32_t *k_host, int limit, int max_iter,
                               const int32_t *model, const double *slo, const int32_t *out,
                               const int32_t *feat, int32_t *label, int32_t *group_of,
                               qlm_group *groups, int group_cap, int32_t *n_groups, int32_t *iters,
                               int32_t *n_bad, cudaStream_t st);  // Alg. 1 (R21)
cudaError_t launch_adopt(const Dims &dm, const Cand &cd, const qlm_record *rec, qlm_record *inc,
                         cudaStream_t st);                          // local-search step (R18)
// qlm_winner's fields into device-mapped host buffers (qo / po nullable)
cudaError_t launch_winner_out(const qlm_record *rec, const float *s12, const int32_t *n_over,
                              const int32_t *dec, int G, qlm_best *out, int32_t *qo, int32_t *po,
                              cudaStream_t st);
cudaError_t launch_rows(const ScanParams &p, uint16_t *rows, int32_t *qo, int32_t *po,
                        cudaStream_t st);
cudaError_t launch_reduce_records(const qlm_record *recs, int n, qlm_record *out,
                                  cudaStream_t st);
cudaError_t launch_check_rows(const Cand &cd, int T, unsigned long long *n_bad, cudaStream_t st);
cudaError_t launch_mc_sample(const Dims &dm, const Tables &tb, uint64_t seed, int64_t t0,
                             int64_t nt, double *Y, cudaStream_t st);
cudaError_t launch_mc_count(const Dims &dm, const Tables &tb, const Cand &cd, const double *Y,
                            int64_t nt, uint32_t *counts, cudaStream_t st,
                            const int32_t *t_mem = nullptr, const int32_t *t_cap = nullptr,
                            const double *t_load = nullptr);   // tier tables (R20) or none

}  // namespace qlm
