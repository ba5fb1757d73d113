/*
 * rgc_oracle.c -- CPU ORACLE for RedSync Residual Gradient Compression (RGC).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1808_04357_b200/) never links, imports or calls
 * it, and this file shares no code, header, table or constant generator with
 * the CUDA path.
 *
 * Plain, slow, single-threaded C99.  Every function follows one passage of
 * /root/reference/PAPER.md ("P:<line>") in the paper's order and notation, or
 * the reading of a silent/ambiguous passage listed in DESIGN.md ("R<n>").
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fno-fast-math -fPIC -shared
 * (no FMA contraction, no flush-to-zero; fmaf() is the correctly-rounded
 * C99 fused multiply-add).
 *
 * Parity status: every function is pinned by tests/test_oracle_pins.py to
 * something other than itself (closed forms, brute force, exact rational
 * arithmetic, hand-worked goldens in tests/golden/), including each reading of
 * a silent passage that changes results: R2's tile exponent and truncation
 * (mean_fx_bins.json), R3's double-precision thresholds and R18's
 * eps-termination rules (bs_hand_paths.json).  tests/test_oracle_mutations.py
 * checks that mutants of these readings fail the pins.  What stays unpinned is
 * only whether the authors' unpublished implementation made the same choices
 * (DESIGN.md section 2).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- result flags (numeric values documented in DESIGN.md §Flags) ---- */
#define RGCO_F_DEGENERATE   (1u << 0)  /* R10: max==0 or mean==max -> exact top-k */
#define RGCO_F_TRIM_ALL     (1u << 1)  /* Alg.2 reached ratio<=0 without nnz>=k */
#define RGCO_F_BS_BREAK     (1u << 2)  /* Alg.3 line "nnz > k and 2k > nnz" -> break */
#define RGCO_F_EPS_HIGH     (1u << 3)  /* eps-terminated, kept, nnz >= 2k */
#define RGCO_F_EPS_BEST     (1u << 4)  /* eps-terminated, last nnz<k, best nnz>=k used */
#define RGCO_F_EPS_EXACT    (1u << 5)  /* eps-terminated, no nnz>=k seen -> exact top-k */
#define RGCO_F_CAP_EXACT    (1u << 6)  /* R18: chosen count > max_count -> exact top-k */
#define RGCO_F_NONFINITE    (1u << 7)  /* residual holds Inf/NaN -> error */
#define RGCO_F_EPS_KEEP     (1u << 8)  /* eps-terminated, last nnz>=k kept */
#define RGCO_F_SAMPLED_REUSE (1u << 9) /* sampled BS: cached threshold reused */

#define RGCO_TILE 4096u            /* R2: mean_fx tile, layer-local */
#define RGCO_NBINS 277             /* exponents -149..127 */
#define RGCO_MAX_TRIM_LEVELS 16

/* per-layer state of the sampled threshold binary search */
typedef struct {
    uint64_t step;     /* compress calls so far */
    int32_t  valid;    /* a threshold is cached */
    float    t;        /* the cached threshold */
} rgco_sample_state_t;

typedef struct {
    uint32_t flags;
    uint32_t iters;          /* number of count_nonzero evaluations */
    uint32_t trim_level;     /* Alg.2: index j of the level used (== levels if TRIM_ALL) */
    uint32_t trim_levels;    /* number of ratio levels with ratio > 0 */
    uint64_t count;          /* size of the communication-set */
    float    threshold;      /* threshold whose strict ">" defined the set (0 if exact) */
    uint32_t maxkey;         /* bits(max|V|) */
    double   mean;           /* mean_fx |V| */
    uint64_t level_count[RGCO_MAX_TRIM_LEVELS]; /* Alg.2 nnz per level / Alg.3 nnz per step */
    float    level_thresh[RGCO_MAX_TRIM_LEVELS];
    uint64_t survivors;      /* Alg.2: elements left after trimming */
} rgco_info_t;

static uint32_t f2u(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static float u2f(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }

/* O1  k = ceil(D*n) clamped to [1,n]  (north_star "k = ceil(D·n)"; R1).
 * P:121 gives the compression ratio D; the paper never states the rounding. */
uint64_t rgco_k(uint64_t n, double D)
{
    double kd = ceil(D * (double)n);
    uint64_t k = (uint64_t)kd;
    if (k < 1) k = 1;
    if (k > n) k = n;
    return k;
}

/* O2  Residual accumulation with DGC momentum correction.
 * P:127 "V_j^k += G_j^k"; P:409-410 momentum correction (DGC), read as
 * u <- m*u + g ; V <- V + u  (R15).  m == 0 reduces to P:127 and leaves u
 * untouched (u may be NULL). */
void rgco_accumulate(uint64_t n, const float *g, float *u, float *V, float m)
{
    for (uint64_t i = 0; i < n; i++) {
        if (m == 0.0f) {
            V[i] = V[i] + g[i];
        } else {
            u[i] = fmaf(m, u[i], g[i]);
            V[i] = V[i] + u[i];
        }
    }
}

/* O3  mean(abs(X)) and max(abs(X))  (Alg.2 line 1 P:211, Alg.3 line 1 P:234).
 * max: the largest |V[i]|, returned as its bit pattern.
 * mean: the reproducible reading mean_fx (R2): per layer-local tile of 4096
 *   elements with tile maximum 2^E <= m_t < 2^(E+1), every |x| contributes
 *   floor(|x| * 2^(30-E)) to an integer bin B[E]; the mean is
 *   (sum_E ascending of B[E]*2^(E-30)) / n in double.
 * Returns 1 (and leaves mean undefined) if any element is Inf/NaN. */
int rgco_stats(uint64_t n, const float *V, uint32_t *maxkey_out, double *mean_out,
               uint64_t *bins_out /* [277] or NULL */)
{
    uint64_t B[RGCO_NBINS];
    memset(B, 0, sizeof B);
    uint32_t maxkey = 0;
    for (uint64_t i = 0; i < n; i++) {
        uint32_t key = f2u(V[i]) & 0x7FFFFFFFu;
        if (key > maxkey) maxkey = key;
    }
    *maxkey_out = maxkey;
    if (maxkey >= 0x7F800000u) return 1;

    for (uint64_t t0 = 0; t0 < n; t0 += RGCO_TILE) {
        uint64_t t1 = t0 + RGCO_TILE < n ? t0 + RGCO_TILE : n;
        double tmax = 0.0;
        for (uint64_t i = t0; i < t1; i++) {
            double a = fabs((double)V[i]);
            if (a > tmax) tmax = a;
        }
        if (tmax == 0.0) continue;
        int e;
        frexp(tmax, &e);             /* tmax = f * 2^e, f in [0.5,1) */
        int E = e - 1;               /* floor(log2(tmax)) */
        uint64_t S = 0;
        for (uint64_t i = t0; i < t1; i++)
            S += (uint64_t)floor(ldexp(fabs((double)V[i]), 30 - E));
        B[E + 149] += S;
    }
    double acc = 0.0;
    for (int b = 0; b < RGCO_NBINS; b++)
        acc += ldexp((double)B[b], (b - 149) - 30);
    *mean_out = acc / (double)n;
    if (bins_out) memcpy(bins_out, B, sizeof B);
    return 0;
}

/* count_nonzero(abs(X) > threshold) */
uint64_t rgco_count_above(uint64_t n, const float *X, float threshold)
{
    uint64_t c = 0;
    for (uint64_t i = 0; i < n; i++)
        if (fabsf(X[i]) > threshold) c++;
    return c;
}

/* nonzero_indices(abs(X) > threshold): ascending indices */
uint64_t rgco_nonzero_indices(uint64_t n, const float *X, float threshold, uint32_t *idx)
{
    uint64_t c = 0;
    for (uint64_t i = 0; i < n; i++)
        if (fabsf(X[i]) > threshold) idx[c++] = (uint32_t)i;
    return c;
}

typedef struct { float a; uint32_t i; } rgco_ai_t;

static int cmp_mag_desc_idx_asc(const void *pa, const void *pb)
{
    const rgco_ai_t *x = (const rgco_ai_t *)pa, *y = (const rgco_ai_t *)pb;
    if (x->a > y->a) return -1;
    if (x->a < y->a) return 1;
    return (x->i < y->i) ? -1 : (x->i > y->i);
}

static int cmp_u32(const void *pa, const void *pb)
{
    uint32_t x = *(const uint32_t *)pa, y = *(const uint32_t *)pb;
    return (x > y) - (x < y);
}

/* O7  exact top-k by |value| (the Quickselect/radixSelect result of P:165-169)
 * over the candidate index list cand[0..m) (or all of X when cand == NULL),
 * ties broken by lower index (R6); written to idx[0..k) in ascending order.
 * Plain definition: sort by (|x| desc, index asc), take the first k. */
void rgco_topk_of(const float *X, const uint32_t *cand, uint64_t m, uint64_t k, uint32_t *idx)
{
    rgco_ai_t *a = (rgco_ai_t *)malloc((m ? m : 1) * sizeof *a);
    for (uint64_t j = 0; j < m; j++) {
        uint32_t i = cand ? cand[j] : (uint32_t)j;
        a[j].a = fabsf(X[i]);
        a[j].i = i;
    }
    qsort(a, m, sizeof *a, cmp_mag_desc_idx_asc);
    for (uint64_t j = 0; j < k; j++) idx[j] = a[j].i;
    free(a);
    qsort(idx, k, sizeof *idx, cmp_u32);
}

void rgco_exact_topk(uint64_t n, const float *X, uint64_t k, uint32_t *idx)
{
    rgco_topk_of(X, NULL, n, k, idx);
}

static float thresh_at(double mean, double maxd, double ratio)
{
    /* P:215 / P:238: threshold <- mean + ratio * (max - mean); double, RN to f32 (R3) */
    double d = maxd - mean;
    double p = ratio * d;
    double t = mean + p;
    return (float)t;
}

/* Number of Alg.2 ratio levels with ratio > 0: ratio_0 = 1-eps, ratio_{j+1} = ratio_j - eps
 * (P:212).  Returns 0 if eps invalid or more than RGCO_MAX_TRIM_LEVELS levels. */
uint32_t rgco_trim_levels(double eps)
{
    if (!(eps > 0.0) || !(eps < 1.0)) return 0;
    uint32_t L = 0;
    for (double r = 1.0 - eps; r > 0.0; r = r - eps) {
        if (++L > RGCO_MAX_TRIM_LEVELS) return 0;
    }
    return L;
}

/* O5  Trimmed top-k selection (Algorithm 2).
 * Line 1 mean/max (given); line 2 eps, ratio = 1-eps; lines 3-8: lower the
 * threshold until nnz >= k (R4: the first threshold uses ratio 1-eps; R5: if no
 * level with ratio > 0 reaches k, all of X survive); then the exact top-k
 * (radixSelect) on the survivors with the lower-index tie rule.
 * Writes k ascending indices; returns k. */
uint64_t rgco_trimmed(uint64_t n, const float *X, uint64_t k, double mean, float maxf,
                      double eps, uint32_t *idx, rgco_info_t *info)
{
    uint32_t levels = rgco_trim_levels(eps);
    info->trim_levels = levels;
    double ratio = 1.0 - eps;
    uint32_t j;
    float threshold = 0.0f;
    uint64_t nnz = 0;
    for (j = 0; j < levels; j++) {
        threshold = thresh_at(mean, (double)maxf, ratio);
        nnz = rgco_count_above(n, X, threshold);
        info->level_count[j] = nnz;
        info->level_thresh[j] = threshold;
        info->iters++;
        if (nnz >= k) break;
        ratio = ratio - eps;
    }
    info->trim_level = j;
    if (j == levels) {
        info->flags |= RGCO_F_TRIM_ALL;
        info->survivors = n;
        rgco_topk_of(X, NULL, n, k, idx);
    } else {
        uint32_t *surv = (uint32_t *)malloc((nnz ? nnz : 1) * sizeof *surv);
        rgco_nonzero_indices(n, X, threshold, surv);
        info->survivors = nnz;
        rgco_topk_of(X, surv, nnz, k, idx);
        free(surv);
    }
    info->count = k;
    info->threshold = 0.0f;
    return k;
}

/* O6  Threshold binary search selection (Algorithm 3).
 * l = 0, r = 1; while r - l > eps: ratio = l + (r-l)/2,
 * threshold, nnz = count_nonzero; break if nnz > k and 2k > nnz
 * (strict, R9); otherwise move a border:
 *   branch 1 (PAPER_LITERAL): nnz < k/2 -> r = ratio, else l = ratio;
 *   branch 0 (MONOTONE, R7):  nnz <= k  -> r = ratio, else l = ratio.
 * After eps-termination (R7/R18): keep the last (threshold, nnz) if nnz >= k;
 * else the evaluated threshold with the smallest nnz >= k (the first evaluated
 * one on a tie: equal counts select the same set); else the exact top-k.
 * Finally, if the chosen count exceeds max_count, the exact top-k (R18).
 * Writes the selected ascending indices; returns their count. */
uint64_t rgco_bs(uint64_t n, const float *X, uint64_t k, double mean, float maxf,
                 double eps, int branch, uint64_t max_count, uint32_t *idx, rgco_info_t *info)
{
    double l = 0.0, r = 1.0;
    float threshold = 0.0f;
    uint64_t nnz = 0;
    int have_best = 0, broke = 0;
    float best_t = 0.0f;
    uint64_t best_c = 0;
    uint32_t it = 0;
    while (r - l > eps) {
        double ratio = l + (r - l) / 2;
        threshold = thresh_at(mean, (double)maxf, ratio);
        nnz = rgco_count_above(n, X, threshold);
        if (it < RGCO_MAX_TRIM_LEVELS) {
            info->level_count[it] = nnz;
            info->level_thresh[it] = threshold;
        }
        it++;
        if (nnz >= k && (!have_best || nnz < best_c)) {
            have_best = 1; best_t = threshold; best_c = nnz;
        }
        if (nnz > k && 2 * k > nnz) { broke = 1; break; }
        if (branch == 1) {
            if (2 * nnz < k) r = ratio; else l = ratio;
        } else {
            if (nnz <= k) r = ratio; else l = ratio;
        }
    }
    info->iters = it;
    int exact = 0;
    if (broke) {
        info->flags |= RGCO_F_BS_BREAK;
    } else if (it > 0 && nnz >= k) {
        info->flags |= RGCO_F_EPS_KEEP;
        if (nnz >= 2 * k) info->flags |= RGCO_F_EPS_HIGH;
    } else if (have_best) {
        info->flags |= RGCO_F_EPS_BEST;
        threshold = best_t; nnz = best_c;
    } else {
        info->flags |= RGCO_F_EPS_EXACT;
        exact = 1;
    }
    if (!exact && nnz > max_count) {
        info->flags |= RGCO_F_CAP_EXACT;
        exact = 1;
    }
    if (exact) {
        rgco_topk_of(X, NULL, n, k, idx);
        info->count = k;
        info->threshold = 0.0f;
        return k;
    }
    uint64_t c = rgco_nonzero_indices(n, X, threshold, idx);
    info->count = c;
    info->threshold = threshold;
    return c;
}

/* Sampled threshold binary search (NEXT-1): "after a threshold
 * binary search for this layer, the threshold element can be reused in the
 * next few iterations. The interval of search is empirically set to 5".
 * Reading (R20): on calls with step % interval != 0 and a cached
 * threshold, select {|x| > t_cached} in one count_nonzero + one compaction;
 * otherwise run Algorithm 3 and cache its threshold (or clear the cache when
 * it ended in an exact top-k).  The capacity rule R18 applies to both. */
uint64_t rgco_sampled_reuse(uint64_t n, const float *X, uint64_t k, uint64_t max_count,
                            const rgco_sample_state_t *st, uint32_t *idx, rgco_info_t *info)
{
    float t = st->t;
    uint64_t nnz = rgco_count_above(n, X, t);
    info->flags |= RGCO_F_SAMPLED_REUSE;
    info->iters = 1;
    info->level_count[0] = nnz;
    info->level_thresh[0] = t;
    if (nnz > max_count) {
        info->flags |= RGCO_F_CAP_EXACT;
        rgco_topk_of(X, NULL, n, k, idx);
        info->count = k;
        info->threshold = 0.0f;
        return k;
    }
    uint64_t c = rgco_nonzero_indices(n, X, t, idx);
    info->count = c;
    info->threshold = t;
    return c;
}

/* ASQ, Alternating Signs Quantization (R21).  "In two adjacent training
 * iterations, ASQ alternately quantizes the maximum 0.1% elements and the minimum
 * 0.1% elements as communication-set instead of quantifying the maximum 0.1%
 * elements with the largest absolute value", implemented "by slightly
 * modifying our parallel-friendly top-0.1% approaches".  Reading R21: the
 * selection algorithms run unchanged on the signed view
 *   phase 0 (POSITIVE, "the largest k elements (all positive numbers)"):
 *       X'[i] = X[i] if X[i] > 0 else 0
 *   phase 1 (NEGATIVE, "smallest k elements (all negative numbers)"):
 *       X'[i] = -X[i] if X[i] < 0 else 0
 * with the layer's mean/max of |X| as the threshold statistics, and the result is
 * restricted to X' > 0 (a layer with fewer than k elements of the phase's sign
 * sends all of them).  The phase alternates on every call. */
void rgco_asq_view(uint64_t n, const float *X, int phase, float *Xv)
{
    for (uint64_t i = 0; i < n; i++) {
        float x = phase == 0 ? X[i] : -X[i];
        Xv[i] = x > 0.0f ? x : 0.0f;
    }
}

/* quantize ("setting all value elements of the same sign to their
 * average ... transmitting only one average element"; R22): the mean of the c
 * selected values, all of one sign.  Reproducible reading: the exact sum of the
 * magnitudes is kept as integer significand sums per binary exponent,
 * B[e] = sum of the 24-bit significands s of the values whose biased exponent is
 * e (|v| = s * 2^(max(e,1)-150)); then acc = sum over e ascending of
 * (double)B[e] * 2^(max(e,1)-150), mean = acc / c in double, rounded once to f32,
 * with the values' sign.  c == 0 -> 0 (an empty message carries 0). */
float rgco_asq_mean(uint64_t c, const float *val)
{
    if (c == 0) return 0.0f;
    uint64_t B[255];
    memset(B, 0, sizeof B);
    for (uint64_t j = 0; j < c; j++) {
        uint32_t b = f2u(val[j]) & 0x7FFFFFFFu;
        uint32_t e = b >> 23;
        uint32_t s = (b & 0x7FFFFFu) | (e ? 0x800000u : 0u);
        B[e] += s;
    }
    double acc = 0.0;
    for (int e = 0; e < 255; e++)
        acc += ldexp((double)B[e], (e > 1 ? e : 1) - 150);
    double mean = acc / (double)c;
    float m = (float)mean;
    return (f2u(val[0]) >> 31) ? -m : m;
}

/* One layer of Algorithm 1's inner loop for one node:
 *   O2 accumulate; O3 stats; O4 degenerate check; O5/O6 select;
 *   O8 message <indices, values> with values = V[indices] before zeroing
 *   (P:129); O9 residual update V <- V (.) (1 - Masks) plus
 *   DGC momentum masking u <- u (.) (1 - Masks).
 * selector: 0 trimmed (Alg.2), 1 threshold binary search (Alg.3),
 *           2 sampled threshold binary search (state in *st, interval 0 -> 5).
 * max_count: 0 -> default (k for trimmed, 2k for BS).
 * quantize: ASQ (R21, R22) with the layer's phase in *phase (0 positive,
 *   1 negative; flipped by every call) and the message's single value in *qmean;
 *   val[] still receives the selected (pre-quantization) values.
 * idx/val must hold max(k, max_count) (2k for BS by default) entries.
 * Returns the message count, -1 on a non-finite residual, -2 for quantize with
 * sampled BS. */
int64_t rgco_compress_layer(uint64_t n, const float *g, float *u, float *V, float m,
                            double D, int selector, int bs_branch, double trim_eps,
                            double bs_eps, uint64_t max_count, uint32_t interval,
                            rgco_sample_state_t *st,
                            uint32_t *idx, float *val, rgco_info_t *info,
                            int quantize, uint32_t *phase, float *qmean)
{
    memset(info, 0, sizeof *info);
    if (quantize && selector == 2) return -2;   /* sampled BS "cannot be used with quantization" */
    uint64_t k = rgco_k(n, D);
    if (max_count == 0) max_count = (selector == 0) ? k : 2 * k;
    if (interval == 0) interval = 5;
    rgco_accumulate(n, g, u, V, m);
    uint32_t maxkey;
    double mean = 0.0;
    if (rgco_stats(n, V, &maxkey, &mean, NULL)) {
        info->flags |= RGCO_F_NONFINITE;
        info->maxkey = maxkey;
        if (selector == 2) { st->valid = 0; st->step++; }
        if (quantize) { *phase ^= 1u; *qmean = 0.0f; }
        return -1;
    }
    info->maxkey = maxkey;
    info->mean = mean;
    float maxf = u2f(maxkey);
    /* ASQ: select on the signed view of this call's phase (R21) */
    float *X = V;
    if (quantize) {
        X = (float *)malloc((n ? n : 1) * sizeof *X);
        rgco_asq_view(n, V, (int)*phase, X);
    }
    uint64_t c;
    if (selector == 2 && st->valid && st->step % interval != 0) {
        c = rgco_sampled_reuse(n, X, k, max_count, st, idx, info);
    } else if (maxkey == 0 || mean == (double)maxf) {
        info->flags |= RGCO_F_DEGENERATE;
        rgco_exact_topk(n, X, k, idx);
        c = k;
        info->count = k;
    } else if (selector == 0) {
        c = rgco_trimmed(n, X, k, mean, maxf, trim_eps, idx, info);
    } else {
        c = rgco_bs(n, X, k, mean, maxf, bs_eps, bs_branch, max_count, idx, info);
    }
    if (quantize) {
        /* only elements of the phase's sign (an exact top-k may have reached X' == 0) */
        uint64_t w = 0;
        for (uint64_t j = 0; j < c; j++)
            if (X[idx[j]] > 0.0f) idx[w++] = idx[j];
        c = w;
        info->count = c;
        free(X);
    }
    if (selector == 2) {
        if (!(info->flags & RGCO_F_SAMPLED_REUSE)) {
            /* a full search: cache its threshold, or clear the cache after an exact fallback */
            int has_t = !(info->flags & (RGCO_F_DEGENERATE | RGCO_F_EPS_EXACT | RGCO_F_CAP_EXACT));
            st->valid = has_t;
            st->t = has_t ? info->threshold : 0.0f;
        }
        st->step++;
    }
    for (uint64_t j = 0; j < c; j++) val[j] = V[idx[j]];
    if (quantize) {
        *qmean = rgco_asq_mean(c, val);   /* quantize(V (.) Masks), Alg.1 */
        *phase ^= 1u;
    }
    /* V <- V (.) (1 - Masks): Algorithm 1 zeroes the selected entries also
     * when the message carries their quantized mean */
    for (uint64_t j = 0; j < c; j++) {
        V[idx[j]] = 0.0f;
        if (u && m != 0.0f) u[idx[j]] = 0.0f;
    }
    return (int64_t)c;
}

/* O11  decompress: the dense averaged gradient from the p gathered
 * communication-sets, summed in rank order from +0 (R14) and
 * scaled by 1/p (R13):  acc = 0; for r: acc[idx] += val; out = acc * (1/p). */
void rgco_decompress(uint64_t n, int p, const uint64_t *counts,
                     const uint32_t *const *idx, const float *const *val, float *out)
{
    for (uint64_t i = 0; i < n; i++) out[i] = 0.0f;
    for (int r = 0; r < p; r++)
        for (uint64_t j = 0; j < counts[r]; j++)
            out[idx[r][j]] = out[idx[r][j]] + val[r][j];
    float s = 1.0f / (float)p;
    for (uint64_t i = 0; i < n; i++) out[i] = out[i] * s;
}
