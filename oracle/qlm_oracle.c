/*
 * qlm_oracle.c -- plain, slow, fp64 CPU oracle of QLM's RWT estimator
 * evaluated over candidate queue orderings.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2407_00047_b200/csrc); neither side includes the other.
 *
 * Citations: "P:Lx" = /root/reference/PAPER.md line x, "S:Lx" = SPEC.md.
 * Every reading of a garbled or silent passage is listed in DESIGN.md
 * ("Readings of the paper", R1..R21) and referenced here by its R-number.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared -o liboracle.so qlm_oracle.c -lm
 * (-ffp-contract=off: no FMA contraction, so every + and * below is one IEEE
 * round-to-nearest operation in source order.)
 *
 * Pins (tests/test_oracle_pins.py) -- every function below is pinned:
 *   or_philox4x32_10   Random123 known-answer vectors.
 *   or_enum_row        itertools.permutations lexicographic order (T <= 7).
 *   or_random_row      permutation invariant + chi-square uniformity (T = 4).
 *   or_neighbor_row    permutation invariant, <= 2k displaced positions,
 *                      k = 0 identity, chi-square uniformity of (i, j);
 *                      local search built on it reaches the brute-force
 *                      optimum on small instances (tests/test_oracle_pins.py).
 *   or_estimate_row    SPEC worked examples S:L279/287/296/306/315, closed
 *                      form for identical groups (Eq. 2/3), Insight-3
 *                      transition arithmetic, textbook Phi-bar values.
 *   or_score_row       SPEC S:L375 (-105 tie), X-Y-X example, C1 golden,
 *                      SPT (min S2) and Moore-Hodgson (min S1) vs brute force.
 *   or_mc_sample       closed form for constant tables, CLT normality test.
 *   or_mc_count        deterministic-table special case == step function.
 *   or_estimate_row_tiered (R20, N3)  load = 0 and cap >= sum mem reduce to
 *                      or_estimate_row bit-exactly; cap = 0 equals
 *                      or_estimate_row with swap + load folded into the swap
 *                      table; hand-worked golden (prefix-not-first-fit,
 *                      re-entry keeps its tier); wt monotone in cap.
 *   or_form_groups (R21, N4)  SPEC S:L199-201 examples; Lloyd partition ==
 *                      scikit-learn KMeans(lloyd, tol=0) from the same start;
 *                      farthest-point start by brute force; fixed point; split
 *                      sizes; group stats == numpy mean / var / min.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- problem description (Table 3) ------------------ */
typedef struct {
    int32_t G, Q, D, M;
    const int32_t *model;      /* [G] model of group i (Eq. 7)   */
    const int32_t *n_req;      /* [G] requests in group i                    */
    const double *slo;         /* [G] TTFT deadline, s (Eq. 8)   */
    const double *mu;          /* [G] mean output tokens (Eq. 3)     */
    const double *var;         /* [G] output-token variance (Eq. 3)          */
    const int32_t *dist;       /* [G] MC length table id                     */
    const int32_t *q_device;   /* [Q] device-type row                        */
    const int32_t *q_resident; /* [Q] model loaded at t=0 (Def. 3)   */
    const double *q_bmean;     /* [Q] pinned in-flight work, s (R12)         */
    const double *q_bvar;      /* [Q]                                        */
    const double *theta;       /* [D][M] tokens/s (Eq. 2)            */
    const double *prefill;     /* [D][M] P (Eq. 1)               */
    const double *eps;         /* [D][M] epsilon (Eq. 4)         */
    const double *dtok;        /* [D][M] d (Eq. 4)                           */
    const double *max_out;     /* [D][M] max output tokens (Eq. 4 bound)     */
    const double *swap;        /* [D][M][M] swap time from->to (S)   */
    int32_t K, n_tables;       /* MC length tables                           */
    const uint16_t *len;       /* [n_tables][K]                              */
    double z_clamp;            /* R9: v := 0 / 1 beyond +-z_clamp            */
    double alpha;              /* n_over threshold                           */
} or_problem;

/* ---- Philox4x32-10 (Salmon et al., SC'11; Random123 reference) ---------- */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }   /* key bump */
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ---- candidate rows (encoding of Eq. 6; R10) ----------------
 * A candidate is a row of T = G+Q-1 tokens: a permutation of 0..T-1 where
 * token < G is a request group and token >= G separates virtual queues.    */

/* RANDOM(seed, c): forward Fisher-Yates driven by Philox words (R10).
 * T > 256: step i draws the 32-bit word i mod 4 of block i/4,
 *          j = i + floor(u * (T - i) / 2^32);
 * T <= 256: step i draws the 16-bit half (low for even i, high for odd i)
 *          of word (i/2) mod 4 of block i/8, j = i + floor(u * (T - i) / 2^16)
 *          (8 draws per Philox block; per-index bias <= (T - i) / 2^16).      */
void or_random_row(uint64_t seed, uint64_t c, int32_t T, int32_t *row)
{
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t words[4];
    int d16 = T <= 256;
    int per_block = d16 ? 8 : 4;
    for (int32_t k = 0; k < T; ++k) row[k] = k;
    for (int32_t i = 0; i + 1 < T; ++i) {
        if (i % per_block == 0) {    /* one Philox block per 4 (or 8 half-word) draws */
            uint32_t ctr[4] = { (uint32_t)(i / per_block), (uint32_t)c, (uint32_t)(c >> 32), 0x514C4D00u };
            or_philox4x32_10(ctr, key, words);
        }
        int32_t j;
        if (d16) {
            uint32_t w = words[(i / 2) % 4];
            uint32_t u = (i % 2 == 0) ? (w & 0xFFFFu) : (w >> 16);
            j = i + (int32_t)((u * (uint32_t)(T - i)) >> 16);
        } else {
            uint32_t u = words[i % 4];
            j = i + (int32_t)(((uint64_t)u * (uint64_t)(T - i)) >> 32);
        }
        int32_t t = row[i]; row[i] = row[j]; row[j] = t;
    }
}

/* NEIGHBOR(base, seed, c, k) (R18, neighbourhood search of
 * the incumbent ordering): the base row with k random transpositions.  Move
 * m swaps positions i = (u0 * T) >> 32 and j = (u1 * T) >> 32 (i == j leaves
 * the row as it is), with (u0, u1) = words 2(m mod 2), 2(m mod 2)+1 of
 * Philox4x32-10(key = seed, ctr = (m / 2, lo32 c, hi32 c, 0x4E424852)).     */
void or_neighbor_row(const int32_t *base, int32_t T, uint64_t seed, uint64_t c, int32_t k,
                     int32_t *row)
{
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t words[4];
    for (int32_t s = 0; s < T; ++s) row[s] = base[s];
    for (int32_t m = 0; m < k; ++m) {
        if (m % 2 == 0) {
            uint32_t ctr[4] = { (uint32_t)(m / 2), (uint32_t)c, (uint32_t)(c >> 32), 0x4E424852u };
            or_philox4x32_10(ctr, key, words);
        }
        uint32_t u0 = words[2 * (m % 2)], u1 = words[2 * (m % 2) + 1];
        int32_t i = (int32_t)(((uint64_t)u0 * (uint64_t)T) >> 32);
        int32_t j = (int32_t)(((uint64_t)u1 * (uint64_t)T) >> 32);
        int32_t t = row[i]; row[i] = row[j]; row[j] = t;
    }
}

/* ENUM(c): Lehmer unranking, lexicographic order, c < T! (T <= 20).       */
void or_enum_row(uint64_t c, int32_t T, int32_t *row)
{
    int32_t avail[64];
    uint64_t fact[21];
    fact[0] = 1;
    for (int k = 1; k <= 20; ++k) fact[k] = fact[k - 1] * (uint64_t)k;
    for (int32_t k = 0; k < T; ++k) avail[k] = k;
    int32_t left = T;
    for (int32_t pos = 0; pos < T; ++pos) {
        uint64_t f = fact[T - 1 - pos];
        int32_t k = (int32_t)(c / f);
        c = c % f;
        row[pos] = avail[k];
        for (int32_t m = k; m + 1 < left; ++m) avail[m] = avail[m + 1];
        --left;
    }
}

/* Row validity (Eq. 6): a permutation of 0..T-1.  Returns 1 if valid.     */
static int or_is_permutation(const int32_t *row, int32_t T)
{
    char *seen = (char *)calloc((size_t)(T > 0 ? T : 1), 1);
    int ok = 1;
    for (int32_t s = 0; s < T && ok; ++s) {
        if (row[s] < 0 || row[s] >= T || seen[row[s]]) ok = 0;
        else seen[row[s]] = 1;
    }
    free(seen);
    return ok;
}

/* ---- RWT estimator over one ordering ------------------------------------ */

/* C - W for a group of model m on device d: P + D with D = max_out*eps*d
 * (Eq. 1, Eq. 4 P:L632-648 with O_q := max output, Eq. 5 R3). */
static double tail_of(const or_problem *p, int32_t d, int32_t m)
{
    int32_t k = d * p->M + m;
    return p->prefill[k] + p->max_out[k] * p->eps[k] * p->dtok[k];
}

/* Per-group waiting time wt_i (mean, Eq. 2/10) and variance V_i (Eq. 3),
 * plus its queue index and position.  Reading of Eq. 10 (P:L741-746 and the
 * prose of P:L705): walking a queue in order, an exclusive accumulator A
 * holds the expected time until the slot can start, B its variance.
 *   - on a model change into the slot (Eq. 9, m_{-1} = resident model, R4):
 *       A += tail(previous model) + swap[prev][m]    (one transition term)
 *            tail: the group before the boundary contributes its completion
 *                  C = W + P + D (R1); skipped at the queue's first slot
 *                  unless a backlog is pinned (R4/R12)
 *            swap: Eq. 10 2nd term, incl. the slot's own switch (R2)
 *   - wt = A, V = B                 [exclusive: groups ahead only, R5]
 *   - A += n*mu/Theta, B += n*var/Theta^2   [Eq. 2/3, each group its own stats, R6/R7]
 * Returns 0, or -1 if the row is not a permutation of 0..T-1 (Eq. 6).     */
int or_estimate_row(const or_problem *p, const int32_t *row,
                    double *wt, double *V, int32_t *queue_of, int32_t *pos_of)
{
    int32_t T = p->G + p->Q - 1;
    if (!or_is_permutation(row, T)) return -1;
    int32_t q = 0;
    int32_t d = p->q_device[0], prev = p->q_resident[0], first = 1, pos = 0;
    double A = p->q_bmean[0], B = p->q_bvar[0];
    for (int32_t s = 0; s < T; ++s) {
        int32_t tok = row[s];
        if (tok >= p->G) {                       /* queue separator */
            ++q;
            d = p->q_device[q]; prev = p->q_resident[q]; first = 1; pos = 0;
            A = p->q_bmean[q]; B = p->q_bvar[q];
            continue;
        }
        int32_t i = tok, m = p->model[i];
        if (m != prev) {                                     /* t = 1, Eq. 9 */
            int backlog = p->q_bmean[q] > 0.0;
            double trans = p->swap[(d * p->M + prev) * p->M + m];
            if (!first || backlog) trans = tail_of(p, d, prev) + trans;
            A = A + trans;
        }
        wt[i] = A;
        V[i] = B;
        if (queue_of) queue_of[i] = q;
        if (pos_of) pos_of[i] = pos;
        double th = p->theta[d * p->M + m];
        A = A + ((double)p->n_req[i] * p->mu[i]) / th;
        B = B + ((double)p->n_req[i] * p->var[i]) / (th * th);
        prev = m; first = 0; ++pos;
    }
    return 0;
}

/* SLO-violation probability of one group: P(wt_true > slo) under the CLT
 * Normal N(wt, V) of Eq. 3, R8; V = 0 -> step, met iff
 * wt <= slo, R9; clamp beyond +-z_clamp, R9.                    */
double or_violation(double wt, double V, double slo, double z_clamp)
{
    if (V > 0.0) {
        double z = (slo - wt) / sqrt(V);
        if (z >= z_clamp) return 0.0;
        if (z <= -z_clamp) return 1.0;
        return 0.5 * erfc(z / sqrt(2.0));
    }
    return wt > slo ? 1.0 : 0.0;
}

/* Per-candidate objective (R11): S1 = sum n_i v_i / sum n_i (expected
 * fraction of violating requests, relaxation of p <= 0);
 * S2 = sum_i p_i with p_i = wt_i - slo_i (Eq. 11, objective
 * P:L761-767), both summed in row order; n_over = #{v_i > alpha}.          */
int or_score_row(const or_problem *p, const int32_t *row, double *s1, double *s2, int32_t *n_over)
{
    int32_t G = p->G, T = p->G + p->Q - 1;
    double *wt = (double *)malloc(sizeof(double) * (size_t)G);
    double *V = (double *)malloc(sizeof(double) * (size_t)G);
    int rc = or_estimate_row(p, row, wt, V, NULL, NULL);
    if (rc == 0) {
        double num = 0.0, den = 0.0, pen = 0.0;
        int32_t over = 0;
        for (int32_t s = 0; s < T; ++s) {
            int32_t i = row[s];
            if (i >= G) continue;
            double v = or_violation(wt[i], V[i], p->slo[i], p->z_clamp);
            num = num + (double)p->n_req[i] * v;
            den = den + (double)p->n_req[i];
            pen = pen + (wt[i] - p->slo[i]);
            if (v > p->alpha) ++over;
        }
        *s1 = num / den;
        *s2 = pen;
        if (n_over) *n_over = over;
    }
    free(wt); free(V);
    return rc;
}

/* ---- candidate ranges ---------------------------------------------------- */
enum { OR_EXPLICIT = 0, OR_RANDOM = 1, OR_ENUM = 2, OR_NEIGHBOR = 3 };

static void get_row(int kind, const void *rows, int32_t token_bytes, int64_t stride,
                    uint64_t seed, uint64_t c, int64_t local, int32_t T, int32_t *row)
{
    if (kind == OR_RANDOM) { or_random_row(seed, c, T, row); return; }
    if (kind == OR_ENUM) { or_enum_row(c, T, row); return; }
    if (kind == OR_NEIGHBOR) {       /* rows = the base row, stride = k (number of moves) */
        int32_t *b = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
        for (int32_t s = 0; s < T; ++s)
            b[s] = token_bytes == 1 ? ((const uint8_t *)rows)[s] : ((const uint16_t *)rows)[s];
        or_neighbor_row(b, T, seed, c, (int32_t)stride, row);
        free(b);
        return;
    }
    const uint8_t *base = (const uint8_t *)rows + local * stride;
    for (int32_t s = 0; s < T; ++s)
        row[s] = token_bytes == 1 ? base[s] : ((const uint16_t *)base)[s];
}

/* Scores of candidates first..first+count-1.  Returns #invalid rows.      */
int64_t or_score_range(const or_problem *p, int kind, const void *rows, int32_t token_bytes,
                       int64_t stride, uint64_t seed, uint64_t first, int64_t count,
                       double *s1, double *s2, int32_t *n_over)
{
    int32_t T = p->G + p->Q - 1;
    int32_t *row = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
    int64_t bad = 0;
    for (int64_t k = 0; k < count; ++k) {
        get_row(kind, rows, token_bytes, stride, seed, first + (uint64_t)k, k, T, row);
        if (or_score_row(p, row, &s1[k], &s2[k], n_over ? &n_over[k] : NULL) != 0) {
            s1[k] = NAN; s2[k] = NAN; ++bad;
        }
    }
    free(row);
    return bad;
}

/* Per-group estimates of candidates first..first+count-1, each [count][G]:
 * wt (mean), sd = sqrt(V), v.                                               */
int64_t or_estimate_range(const or_problem *p, int kind, const void *rows, int32_t token_bytes,
                          int64_t stride, uint64_t seed, uint64_t first, int64_t count,
                          double *wt, double *sd, double *v)
{
    int32_t G = p->G, T = p->G + p->Q - 1;
    int32_t *row = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
    double *V = (double *)malloc(sizeof(double) * (size_t)G);
    int64_t bad = 0;
    for (int64_t k = 0; k < count; ++k) {
        get_row(kind, rows, token_bytes, stride, seed, first + (uint64_t)k, k, T, row);
        double *w = wt + k * G;
        if (or_estimate_row(p, row, w, V, NULL, NULL) != 0) { ++bad; continue; }
        for (int32_t i = 0; i < G; ++i) {
            sd[k * G + i] = sqrt(V[i]);
            v[k * G + i] = or_violation(w[i], V[i], p->slo[i], p->z_clamp);
        }
    }
    free(row); free(V);
    return bad;
}

/* ---- request-level violations (R19) ----------------------
 * Request r = 0..n_i-1 of group i waits for the group's start plus the r
 * requests of the group ahead of it (Eq. 2 with q running over requests,
 * P:L616-619; Eq. 3 for the variance):
 *   mean_r = wt_i + r * (mu_i / Theta),   var_r = V_i + r * (var_i / Theta^2)
 * with Theta = Theta[d][m_i] of the group's queue device.  Its violation
 * probability follows R8/R9 (or_violation); the group's violating fraction
 * is f_i = (1/n_i) sum_r v_r and the candidate's S1_req = sum n_i f_i / sum n_i. */
int or_request_violations_row(const or_problem *p, const int32_t *row, double *frac, double *s1)
{
    int32_t G = p->G;
    double *wt = (double *)malloc(sizeof(double) * (size_t)G);
    double *V = (double *)malloc(sizeof(double) * (size_t)G);
    int32_t *q = (int32_t *)malloc(sizeof(int32_t) * (size_t)G);
    int rc = or_estimate_row(p, row, wt, V, q, NULL);
    if (rc == 0) {
        double num = 0.0, den = 0.0;
        for (int32_t i = 0; i < G; ++i) {
            int32_t d = p->q_device[q[i]];
            double th = p->theta[d * p->M + p->model[i]];
            double a = p->mu[i] / th, b = p->var[i] / (th * th);
            double sum = 0.0;
            for (int32_t r = 0; r < p->n_req[i]; ++r)
                sum = sum + or_violation(wt[i] + (double)r * a, V[i] + (double)r * b, p->slo[i], p->z_clamp);
            frac[i] = sum / (double)p->n_req[i];
            num = num + (double)p->n_req[i] * frac[i];
            den = den + (double)p->n_req[i];
        }
        *s1 = num / den;
    }
    free(wt); free(V); free(q);
    return rc;
}

/* ---- Monte-Carlo mode (R13) ----------------------------------------------
 * Output lengths are sampled per request: for trial t, group k, request r,
 *   w    = Philox4x32-10(key = mc_seed, ctr = (r/8, k, t, 0x4D430000))[(r/2) % 4]
 *   u16  = r even ? low 16 bits of w : high 16 bits of w
 *   O    = len[dist_k][u16 >> (16 - log2 K)]          (K divides 2^16: unbiased)
 * X[t][k] = sum_r O (exact integer), the group's total output tokens.      */
void or_mc_sample(const or_problem *p, uint64_t mc_seed, int64_t trial_first,
                  int64_t trial_count, uint32_t *X /* [trial_count][G] */)
{
    int32_t shift = 16;
    for (int32_t k = p->K; k > 1; k >>= 1) --shift;
    uint32_t key[2] = { (uint32_t)mc_seed, (uint32_t)(mc_seed >> 32) };
    uint32_t words[4];
    for (int64_t tt = 0; tt < trial_count; ++tt) {
        uint32_t t = (uint32_t)(trial_first + tt);
        for (int32_t k = 0; k < p->G; ++k) {
            const uint16_t *tab = p->len + (int64_t)p->dist[k] * p->K;
            uint32_t sum = 0;
            for (int32_t r = 0; r < p->n_req[k]; ++r) {
                if (r % 8 == 0) {       /* one Philox block yields 8 16-bit draws */
                    uint32_t ctr[4] = { (uint32_t)(r / 8), (uint32_t)k, t, 0x4D430000u };
                    or_philox4x32_10(ctr, key, words);
                }
                uint32_t w = words[(r / 2) % 4];
                uint32_t u16 = (r % 2 == 0) ? (w & 0xFFFFu) : (w >> 16);
                sum += tab[u16 >> shift];
            }
            X[tt * p->G + k] = sum;
        }
    }
}

/* For each candidate row and trial: the Eq. 10 walk of or_estimate_row with
 * the sampled X/Theta in place of n*mu/Theta (Eq. 2 with the realised token
 * count); counts[c][k] += (W_k > slo_k).  Returns #invalid rows.           */
int64_t or_mc_count(const or_problem *p, int kind, const void *rows, int32_t token_bytes,
                    int64_t stride, uint64_t seed, uint64_t first, int64_t count,
                    const uint32_t *X, int64_t trial_count, uint32_t *counts /* [count][G] */)
{
    int32_t G = p->G, T = p->G + p->Q - 1;
    int32_t *row = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
    int64_t bad = 0;
    for (int64_t c = 0; c < count; ++c) {
        get_row(kind, rows, token_bytes, stride, seed, first + (uint64_t)c, c, T, row);
        uint32_t *cnt = counts + c * G;
        for (int32_t i = 0; i < G; ++i) cnt[i] = 0;
        if (!or_is_permutation(row, T)) { ++bad; continue; }
        for (int64_t t = 0; t < trial_count; ++t) {
            const uint32_t *x = X + t * G;
            int32_t q = 0;
            int32_t d = p->q_device[0], prev = p->q_resident[0], first_slot = 1;
            double A = p->q_bmean[0];
            for (int32_t s = 0; s < T; ++s) {
                int32_t tok = row[s];
                if (tok >= G) {
                    ++q;
                    d = p->q_device[q]; prev = p->q_resident[q]; first_slot = 1;
                    A = p->q_bmean[q];
                    continue;
                }
                int32_t i = tok, m = p->model[i];
                if (m != prev) {
                    int backlog = p->q_bmean[q] > 0.0;
                    double trans = p->swap[(d * p->M + prev) * p->M + m];
                    if (!first_slot || backlog) trans = tail_of(p, d, prev) + trans;
                    A = A + trans;
                }
                if (A > p->slo[i]) cnt[i] += 1;
                A = A + (double)x[i] / p->theta[d * p->M + m];
                prev = m; first_slot = 0;
            }
        }
    }
    free(row);
    return bad;
}

/* Request-level violations of candidates first..first+count-1: frac
 * [count][G], s1 [count].  Returns #invalid rows.                           */
int64_t or_request_violations_range(const or_problem *p, int kind, const void *rows,
                                    int32_t token_bytes, int64_t stride, uint64_t seed,
                                    uint64_t first, int64_t count, double *frac, double *s1)
{
    int32_t T = p->G + p->Q - 1;
    int32_t *row = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
    int64_t bad = 0;
    for (int64_t k = 0; k < count; ++k) {
        get_row(kind, rows, token_bytes, stride, seed, first + (uint64_t)k, k, T, row);
        if (or_request_violations_row(p, row, frac + k * p->G, &s1[k]) != 0) { s1[k] = NAN; ++bad; }
    }
    free(row);
    return bad;
}

/* ---- two-tier (warm / cold) model swapping (R20) ---------
 * every model served from the registry goes storage -> CPU
 * memory -> GPU memory.  "Models present later in the virtual queue are
 * warm and placed in the CPU memory until all the CPU memory is exhausted.
 * The remaining models (cold models) are not swapped out from the LLM model
 * registry."  Reading R20, per queue q on device d:
 *   - the queue's swap targets, in order of their first transition (Eq. 9:
 *     slots with m != previous model, m_{-1} = resident, R4), are taken in
 *     turn; target m is warm while cum + mem[m] <= cap[d] (cum += mem[m]),
 *     and from the first target that does not fit on, CPU memory is
 *     exhausted: that target and every later new target are cold;
 *   - a model keeps its tier for every later transition into it;
 *   - the transition term of Eq. 10 (R1/R2) becomes
 *       trans = swap[d][prev][m]             (CPU -> GPU, warm)
 *       trans = swap[d][prev][m] + load[d][m] (storage -> CPU first, cold)
 *     then tail(prev) + trans as in or_estimate_row.
 * With load = 0, or cap >= sum of all mem, this is or_estimate_row exactly. */
typedef struct {
    const int32_t *mem;    /* [M] model size in integer units (e.g. GB), >= 1  */
    const int32_t *cap;    /* [D] CPU memory of a device-d instance, same units */
    const double *load;    /* [D][M] storage -> CPU load time of model m, s    */
} or_tiers;

int or_estimate_row_tiered(const or_problem *p, const or_tiers *t, const int32_t *row,
                           double *wt, double *V, int32_t *cold_of)
{
    int32_t T = p->G + p->Q - 1;
    char tier[64];                        /* tier: 0 = not a target yet, 1 warm, 2 cold */
    if (p->M > 64 || !or_is_permutation(row, T)) return -1;
    int32_t q = 0;
    int32_t d = p->q_device[0], prev = p->q_resident[0], first = 1;
    double A = p->q_bmean[0], B = p->q_bvar[0];
    int64_t cum = 0;
    int exhausted = 0;
    memset(tier, 0, sizeof tier);
    for (int32_t s = 0; s < T; ++s) {
        int32_t tok = row[s];
        if (tok >= p->G) {                       /* queue separator: new queue, new CPU memory */
            ++q;
            d = p->q_device[q]; prev = p->q_resident[q]; first = 1;
            A = p->q_bmean[q]; B = p->q_bvar[q];
            cum = 0; exhausted = 0;
            memset(tier, 0, sizeof tier);
            continue;
        }
        int32_t i = tok, m = p->model[i];
        int32_t cold = 0;
        if (m != prev) {                                     /* t = 1, Eq. 9 */
            if (tier[m] == 0) {                              /* first transition into m */
                if (!exhausted && cum + t->mem[m] <= t->cap[d]) { tier[m] = 1; cum += t->mem[m]; }
                else { tier[m] = 2; exhausted = 1; }
            }
            int backlog = p->q_bmean[q] > 0.0;
            double trans = p->swap[(d * p->M + prev) * p->M + m];
            if (tier[m] == 2) { trans = trans + t->load[d * p->M + m]; cold = 1; }
            if (!first || backlog) trans = tail_of(p, d, prev) + trans;
            A = A + trans;
        }
        wt[i] = A;
        V[i] = B;
        if (cold_of) cold_of[i] = cold;
        double th = p->theta[d * p->M + m];
        A = A + ((double)p->n_req[i] * p->mu[i]) / th;
        B = B + ((double)p->n_req[i] * p->var[i]) / (th * th);
        prev = m; first = 0;
    }
    return 0;
}

/* Scores (R11) and per-group estimates ([G] each, nullable) of one row
 * under R20; same sums and order as or_score_row.                          */
int or_score_row_tiered(const or_problem *p, const or_tiers *t, const int32_t *row,
                        double *s1, double *s2, int32_t *n_over, double *wt_out, double *V_out)
{
    int32_t G = p->G, T = p->G + p->Q - 1;
    double *wt = (double *)malloc(sizeof(double) * (size_t)G);
    double *V = (double *)malloc(sizeof(double) * (size_t)G);
    int rc = or_estimate_row_tiered(p, t, row, wt, V, NULL);
    if (rc == 0) {
        double num = 0.0, den = 0.0, pen = 0.0;
        int32_t over = 0;
        for (int32_t s = 0; s < T; ++s) {
            int32_t i = row[s];
            if (i >= G) continue;
            double v = or_violation(wt[i], V[i], p->slo[i], p->z_clamp);
            num = num + (double)p->n_req[i] * v;
            den = den + (double)p->n_req[i];
            pen = pen + (wt[i] - p->slo[i]);
            if (v > p->alpha) ++over;
        }
        *s1 = num / den;
        *s2 = pen;
        if (n_over) *n_over = over;
        for (int32_t i = 0; i < G; ++i) {
            if (wt_out) wt_out[i] = wt[i];
            if (V_out) V_out[i] = V[i];
        }
    }
    free(wt); free(V);
    return rc;
}

/* Range form: s1, s2 [count], n_over [count] and wt, V [count][G] (each
 * nullable except s1, s2).  Returns #invalid rows.                          */
int64_t or_tiered_range(const or_problem *p, const or_tiers *t, int kind, const void *rows,
                        int32_t token_bytes, int64_t stride, uint64_t seed, uint64_t first,
                        int64_t count, double *s1, double *s2, int32_t *n_over, double *wt,
                        double *V)
{
    int32_t G = p->G, T = p->G + p->Q - 1;
    int32_t *row = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
    int64_t bad = 0;
    for (int64_t k = 0; k < count; ++k) {
        get_row(kind, rows, token_bytes, stride, seed, first + (uint64_t)k, k, T, row);
        if (or_score_row_tiered(p, t, row, &s1[k], &s2[k], n_over ? &n_over[k] : NULL,
                                wt ? wt + k * G : NULL, V ? V + k * G : NULL) != 0) {
            s1[k] = NAN; s2[k] = NAN; ++bad;
        }
    }
    free(row);
    return bad;
}

/* ---- request-group formation (R21; Alg. 1) ----
 * Alg. 1: groups <- kMeansClustering(requests); every group larger than
 * avg_batch_size * delta is split in half (splitHalf), the halves appended.
 * Reading R21:
 *   - features: dims <= 4 integer coordinates per request in [0, 65535]
 *     (the caller's quantised model-independent features, e.g. log SLO,
 *     log input / output tokens: Def. P:L443-447 names them); the model is
 *     a hard partition: k_m clusters per model m, a request only joins a
 *     centroid of its own model;
 *   - initialisation, per model (deterministic farthest point): c_0 = the
 *     model's first request in arrival order; c_{j+1} = the request with the
 *     largest squared distance (exact int64) to its nearest chosen centre,
 *     lowest index on ties; stop early if that distance is 0 (fewer
 *     distinct points than k_m);
 *   - Lloyd iterations (at most max_iter): assign every request to the
 *     nearest centre of its model, d2 = sum_f ((double)x_f - c_f)^2 summed in
 *     f order, lowest centre index on ties; stop when no label changed;
 *     otherwise c = (double)(sum of member coords) / (double)count (sums in
 *     exact integers); an empty cluster keeps its centre;
 *   - splitHalf (Alg. 1 lines 3-5, applied until no group exceeds the
 *     limit): a cluster's members in arrival order [lo, hi) with hi - lo >
 *     limit become [lo, lo + ceil(n/2)) and [lo + ceil(n/2), hi), recursively;
 *   - groups are numbered cluster by cluster (model, then centre index),
 *     halves left to right; a group's model is its cluster's, slo = min
 *     member SLO, mu = S1 / n and var = (n S2 - S1^2) / n^2 with S1, S2 the
 *     exact integer sums of the members' output tokens and their squares
 *     ("fitted ... for the request group").
 * Returns the number of groups (written up to group_cap), -1 on bad input
 * (limit outside [1, 32768], a model, feature or output length out of range:
 * the bounds keep n S2 - S1^2 exact in int64).                             */
typedef struct {
    int32_t *g_model, *g_n;
    double *g_slo, *g_mu, *g_var;
} or_group_out;

static int32_t or_emit_halves(const int32_t *members, int32_t lo, int32_t hi, int32_t limit,
                              const int32_t *out_tok, const double *slo, int32_t model,
                              int32_t *group_of, const or_group_out *o, int32_t group_cap,
                              int32_t gid)
{
    int32_t n = hi - lo;
    if (n > limit) {
        int32_t half = (n + 1) / 2;
        gid = or_emit_halves(members, lo, lo + half, limit, out_tok, slo, model, group_of, o,
                             group_cap, gid);
        return or_emit_halves(members, lo + half, hi, limit, out_tok, slo, model, group_of, o,
                              group_cap, gid);
    }
    int64_t s1 = 0, s2 = 0;
    double mslo = INFINITY;
    for (int32_t i = lo; i < hi; ++i) {
        int32_t r = members[i];
        group_of[r] = gid;
        s1 += out_tok[r];
        s2 += (int64_t)out_tok[r] * out_tok[r];
        if (slo[r] < mslo) mslo = slo[r];
    }
    if (gid < group_cap) {
        o->g_model[gid] = model;
        o->g_n[gid] = n;
        o->g_slo[gid] = mslo;
        o->g_mu[gid] = (double)s1 / (double)n;
        o->g_var[gid] = (double)((int64_t)n * s2 - s1 * s1) / ((double)n * (double)n);
    }
    return gid + 1;
}

int32_t or_form_groups(int32_t n, int32_t dims, const int32_t *model, const double *slo,
                       const int32_t *out_tok, const int32_t *feat, int32_t M,
                       const int32_t *k_per_model, int32_t limit, int32_t max_iter,
                       int32_t *label_of, int32_t *group_of, int32_t *g_model, int32_t *g_n,
                       double *g_slo, double *g_mu, double *g_var, int32_t group_cap,
                       int32_t *iters_out, int32_t *k_eff_out, int32_t *init_out)
{
    if (n < 1 || dims < 1 || dims > 4 || M < 1 || limit < 1 || limit > 32768) return -1;
    for (int32_t r = 0; r < n; ++r) {
        if (model[r] < 0 || model[r] >= M || out_tok[r] < 0 || out_tok[r] > 65535) return -1;
        for (int32_t f = 0; f < dims; ++f)
            if (feat[r * dims + f] < 0 || feat[r * dims + f] > 65535) return -1;
    }
    /* farthest-point initialisation per model (exact integer distances) */
    int32_t *ctr_req = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);   /* chosen requests */
    int32_t *k_eff = (int32_t *)calloc((size_t)M, sizeof(int32_t));
    int32_t *off = (int32_t *)calloc((size_t)M + 1, sizeof(int32_t));
    int64_t *mind = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int32_t K = 0;
    for (int32_t m = 0; m < M; ++m) {
        off[m] = K;
        int32_t first = -1;
        for (int32_t r = 0; r < n; ++r) if (model[r] == m) { first = r; break; }
        if (first < 0 || k_per_model[m] < 1) continue;
        ctr_req[K + k_eff[m]++] = first;
        for (int32_t r = 0; r < n; ++r) mind[r] = INT64_MAX;
        while (k_eff[m] < k_per_model[m]) {
            int32_t c = ctr_req[K + k_eff[m] - 1];
            int64_t best = -1;
            int32_t arg = -1;
            for (int32_t r = 0; r < n; ++r) {
                if (model[r] != m) continue;
                int64_t d2 = 0;
                for (int32_t f = 0; f < dims; ++f) {
                    int64_t t = (int64_t)feat[r * dims + f] - feat[c * dims + f];
                    d2 += t * t;
                }
                if (d2 < mind[r]) mind[r] = d2;
                if (mind[r] > best) { best = mind[r]; arg = r; }
            }
            if (best <= 0) break;                  /* no distinct point left */
            ctr_req[K + k_eff[m]++] = arg;
        }
        K += k_eff[m];
    }
    off[M] = K;
    double *C = (double *)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1) * 4);
    for (int32_t j = 0; j < K; ++j)
        for (int32_t f = 0; f < dims; ++f) C[j * 4 + f] = (double)feat[ctr_req[j] * dims + f];
    /* Lloyd iterations */
    int64_t *sum = (int64_t *)malloc(sizeof(int64_t) * (size_t)(K > 0 ? K : 1) * 5);
    for (int32_t r = 0; r < n; ++r) label_of[r] = -1;
    int32_t it = 0;
    while (it < max_iter) {
        int changed = 0;
        for (int32_t r = 0; r < n; ++r) {
            int32_t m = model[r], arg = -1;
            double best = INFINITY;
            for (int32_t j = off[m]; j < off[m] + k_eff[m]; ++j) {
                double d2 = 0.0;
                for (int32_t f = 0; f < dims; ++f) {
                    double t = (double)feat[r * dims + f] - C[j * 4 + f];
                    d2 = d2 + t * t;
                }
                if (d2 < best) { best = d2; arg = j; }
            }
            if (arg != label_of[r]) { label_of[r] = arg; changed = 1; }
        }
        ++it;
        if (!changed) break;
        memset(sum, 0, sizeof(int64_t) * (size_t)(K > 0 ? K : 1) * 5);
        for (int32_t r = 0; r < n; ++r) {
            int32_t j = label_of[r];
            if (j < 0) continue;
            for (int32_t f = 0; f < dims; ++f) sum[j * 5 + f] += feat[r * dims + f];
            sum[j * 5 + 4] += 1;
        }
        for (int32_t j = 0; j < K; ++j)
            if (sum[j * 5 + 4] > 0)
                for (int32_t f = 0; f < dims; ++f)
                    C[j * 4 + f] = (double)sum[j * 5 + f] / (double)sum[j * 5 + 4];
    }
    if (iters_out) *iters_out = it;
    if (k_eff_out) for (int32_t m = 0; m < M; ++m) k_eff_out[m] = k_eff[m];
    if (init_out) for (int32_t j = 0; j < K; ++j) init_out[j] = ctr_req[j];   /* initial centres */
    /* splitHalf and group statistics, cluster by cluster */
    or_group_out o = { g_model, g_n, g_slo, g_mu, g_var };
    int32_t *members = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t gid = 0;
    for (int32_t j = 0; j < K; ++j) {
        int32_t cnt = 0, m = 0;
        for (int32_t r = 0; r < n; ++r) if (label_of[r] == j) { members[cnt++] = r; m = model[r]; }
        if (cnt > 0)
            gid = or_emit_halves(members, 0, cnt, limit, out_tok, slo, m, group_of, &o, group_cap, gid);
    }
    free(members); free(sum); free(C); free(mind); free(off); free(k_eff); free(ctr_req);
    return gid;
}

/* MC counts under two-tier swapping (R13 + R20): or_mc_count's walk with the
 * transition term of or_estimate_row_tiered (cold targets add load[d][m] to
 * the swap before the tail).  Returns #invalid rows.                        */
int64_t or_mc_count_tiered(const or_problem *p, const or_tiers *tt, int kind, const void *rows,
                           int32_t token_bytes, int64_t stride, uint64_t seed, uint64_t first,
                           int64_t count, const uint32_t *X, int64_t trial_count,
                           uint32_t *counts /* [count][G] */)
{
    int32_t G = p->G, T = p->G + p->Q - 1;
    int32_t *row = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
    int64_t bad = 0;
    if (p->M > 64) { free(row); return count; }
    for (int64_t c = 0; c < count; ++c) {
        get_row(kind, rows, token_bytes, stride, seed, first + (uint64_t)c, c, T, row);
        uint32_t *cnt = counts + c * G;
        for (int32_t i = 0; i < G; ++i) cnt[i] = 0;
        if (!or_is_permutation(row, T)) { ++bad; continue; }
        for (int64_t t = 0; t < trial_count; ++t) {
            const uint32_t *x = X + t * G;
            int32_t q = 0;
            int32_t d = p->q_device[0], prev = p->q_resident[0], first_slot = 1;
            double A = p->q_bmean[0];
            char tier[64];
            int64_t cum = 0;
            int exhausted = 0;
            memset(tier, 0, sizeof tier);
            for (int32_t s = 0; s < T; ++s) {
                int32_t tok = row[s];
                if (tok >= G) {
                    ++q;
                    d = p->q_device[q]; prev = p->q_resident[q]; first_slot = 1;
                    A = p->q_bmean[q];
                    cum = 0; exhausted = 0;
                    memset(tier, 0, sizeof tier);
                    continue;
                }
                int32_t i = tok, m = p->model[i];
                if (m != prev) {
                    if (tier[m] == 0) {
                        if (!exhausted && cum + tt->mem[m] <= tt->cap[d]) { tier[m] = 1; cum += tt->mem[m]; }
                        else { tier[m] = 2; exhausted = 1; }
                    }
                    int backlog = p->q_bmean[q] > 0.0;
                    double trans = p->swap[(d * p->M + prev) * p->M + m];
                    if (tier[m] == 2) trans = trans + tt->load[d * p->M + m];
                    if (!first_slot || backlog) trans = tail_of(p, d, prev) + trans;
                    A = A + trans;
                }
                if (A > p->slo[i]) cnt[i] += 1;
                A = A + (double)x[i] / p->theta[d * p->M + m];
                prev = m; first_slot = 0;
            }
        }
    }
    free(row);
    return bad;
}
