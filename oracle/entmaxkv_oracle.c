/*
 * entmaxkv_oracle.c -- plain, slow, single-threaded CPU oracle for the EntmaxKV
 * sparse alpha-entmax decode step (arxiv 2605.21649).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2605_21649_b200/,
 * libentmaxkv.so) links, loads or calls this file.  Only tests/, bench.py's
 * cpu_baseline / --impl reference leg and __graft_entry__.smoke() may use it.
 * It shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:L" = /root/reference/PAPER.md line L (paper LaTeX source),
 * "S:L" = SPEC.md line L.  Readings of the paper where it is silent are listed in
 * DESIGN.md section "Readings" and referenced here as R<n>.
 *
 * Precision (the paper fixes none):
 *   - scores s_j, page bounds and Gaussian moments are fp32 with the canonical
 *     summation order of DESIGN.md R1 ("dot16x8"), because they decide integers
 *     (top-k membership, page selection) and both sides must take that decision
 *     in the same precision (the kernel's);
 *   - everything downstream of the scores (z = (alpha-1) s, tau, support, p, o,
 *     delta, rho, tau_hat, truncated Gaussian moments) is fp64.
 *
 * Parity status: every exported function is pinned by tests/test_oracle_pins.py
 * except where its comment says "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_D 128          /* head dim supported by the canonical order (R1) */

/* ------------------------------------------------------------------------- */
/* R1: canonical fp32 dot product over d = 128 ("dot16x8").                   */
/*   partial[c] = fma-chain over x[8c..8c+7]*y[8c..8c+7], c = 0..15, from +0   */
/*   then pairwise: level 1 c + (c+8) (c<8); level 2 c + (c+4) (c<4);          */
/*   level 3 c + (c+2) (c<2); level 4 c0 + c1.                                 */
/* This is one fixed evaluation order of  q^T k.       */
/* ------------------------------------------------------------------------- */
float orc_dot_canon(const float *x, const float *y)
{
    float part[16];
    for (int c = 0; c < 16; ++c) {
        float acc = 0.0f;
        for (int i = 8 * c; i < 8 * c + 8; ++i)
            acc = fmaf(x[i], y[i], acc);
        part[c] = acc;
    }
    for (int c = 0; c < 8; ++c) part[c] = part[c] + part[c + 8];
    for (int c = 0; c < 4; ++c) part[c] = part[c] + part[c + 4];
    for (int c = 0; c < 2; ++c) part[c] = part[c] + part[c + 2];
    return part[0] + part[1];
}

/* c_d = fl32(1/sqrt(d)); the score is fl32(dot * c_d) (R2: scale after the dot). */
static float scale_cd(void) { return (float)(1.0 / sqrt((double)ORC_D)); }

/* s_j = q^T k_j / sqrt(d) */
float orc_token_score(const float *q, const float *k)
{
    return orc_dot_canon(q, k) * scale_cd();
}

/* ------------------------------------------------------------------------- */
/* Page metadata (R5 clamp per S:175).                             */
/* keys: [c][d] the page's tokens in append order.                            */
/*   kmin/kmax: coordinate-wise min/max                           */
/*   ksum = sum_t k_t (fp32, t ascending), ksumsq = sum_t k_t*k_t (fma chain)  */
/*   kavg = ksum / c                                  */
/*   kvar = max(0, ksumsq/c - kavg*kavg) = k_std^2                */
/* ------------------------------------------------------------------------- */
void orc_page_stats(const float *keys, int c, int d, float *kmin, float *kmax,
                    float *ksum, float *ksumsq, float *kavg, float *kvar)
{
    for (int i = 0; i < d; ++i) {
        float mn = keys[i], mx = keys[i], s = 0.0f, ss = 0.0f;
        for (int t = 0; t < c; ++t) {
            float v = keys[(size_t)t * d + i];
            if (v < mn) mn = v;
            if (v > mx) mx = v;
            s = s + v;
            ss = fmaf(v, v, ss);
        }
        float cf = (float)c;
        float avg = s / cf;
        float m2 = ss / cf;
        float var = m2 - avg * avg;
        if (!(var > 0.0f)) var = 0.0f;
        kmin[i] = mn; kmax[i] = mx; ksum[i] = s; ksumsq[i] = ss;
        kavg[i] = avg; kvar[i] = var;
    }
}

/* Every valid page of a paged cache (composition of orc_page_stats, no new     */
/* arithmetic): K [n_phys][Hkv][P][d]; page_table [B][maxp]; seq_lens [B];      */
/* outputs [n_phys][Hkv][d].  The last page of a sequence holds c <= P tokens.  */
void orc_build_stats(const float *K, int Hkv, int P, int d, const int32_t *page_table,
                     const int32_t *seq_lens, int B, int maxp, float *kmin, float *kmax,
                     float *ksum, float *ksumsq, float *kavg, float *kvar)
{
    for (int b = 0; b < B; ++b) {
        int n = seq_lens[b], M = (n + P - 1) / P;
        for (int lp = 0; lp < M; ++lp) {
            int c = (lp == M - 1) ? n - lp * P : P;
            size_t ph = (size_t)page_table[(size_t)b * maxp + lp];
            for (int g = 0; g < Hkv; ++g) {
                size_t o = (ph * Hkv + g) * d;
                orc_page_stats(K + (ph * Hkv + g) * P * d, c, d, kmin + o, kmax + o,
                               ksum + o, ksumsq + o, kavg + o, kvar + o);
            }
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Compressed stored metadata (DESIGN R24).                   */
/* The box bound of Prop. B.1 needs only kmin_i <= k_{t,i} <=      */
/* kmax_i; any stored lower bound of kmin and upper bound of kmax keeps it an  */
/* upper bound of every token score.  Stored forms:                           */
/*   e4m3 (OCP fp8 "FN": 1 sign, 4 exponent bits with bias 7, 3 mantissa bits,*/
/*   no infinities, largest finite 448):                                       */
/*     kmin8 = largest e4m3 value <= kmin, kmax8 = smallest e4m3 value >= kmax */
/*   bf16 (kavg, kvar): the fp32 value rounded to nearest, ties to even.       */
/* The e4m3 set is written out from its definition (no bit tricks); rounding  */
/* is a plain search over it.                                                  */
/* ------------------------------------------------------------------------- */
static double e4m3_vals[256];
static int e4m3_n = 0;

static void e4m3_init(void)
{
    if (e4m3_n) return;
    double pos[127];
    int np = 0;
    for (int m = 0; m < 8; ++m) pos[np++] = ldexp((double)m / 8.0, -6);          /* e = 0: subnormals (and 0) */
    for (int e = 1; e <= 15; ++e)
        for (int m = 0; m < 8; ++m) {
            if (e == 15 && m == 7) continue;                                      /* NaN encoding */
            pos[np++] = ldexp(1.0 + (double)m / 8.0, e - 7);
        }
    /* ascending: the negatives (largest magnitude first), then 0, then the positives */
    int n = 0;
    for (int i = np - 1; i >= 1; --i) e4m3_vals[n++] = -pos[i];
    for (int i = 0; i < np; ++i) e4m3_vals[n++] = pos[i];
    e4m3_n = n;
}

/* largest e4m3 value <= x (x >= -448: the precondition of the stored form) */
float orc_e4m3_round_down(float x)
{
    e4m3_init();
    double best = e4m3_vals[0];
    for (int i = 0; i < e4m3_n; ++i)
        if (e4m3_vals[i] <= (double)x) best = e4m3_vals[i];
    return (float)best;
}

/* smallest e4m3 value >= x (x <= 448) */
float orc_e4m3_round_up(float x)
{
    e4m3_init();
    double best = e4m3_vals[e4m3_n - 1];
    for (int i = e4m3_n - 1; i >= 0; --i)
        if (e4m3_vals[i] >= (double)x) best = e4m3_vals[i];
    return (float)best;
}

/* fp32 -> nearest bf16 value (8 significant bits), ties to the even significand.
 * lo = x truncated to 8 significant bits, hi = the next bf16 value away from zero. */
float orc_bf16_round(float x)
{
    if (x == 0.0f || x != x) return x;
    uint32_t b;
    memcpy(&b, &x, 4);
    uint32_t lob = b & 0xffff0000u, hib = lob + 0x10000u;
    float lo, hi;
    memcpy(&lo, &lob, 4);
    memcpy(&hi, &hib, 4);
    double dlo = fabs((double)x - (double)lo), dhi = fabs((double)hi - (double)x);
    if (dlo < dhi) return lo;
    if (dhi < dlo) return hi;
    return ((lob >> 16) & 1u) ? hi : lo;                 /* tie: even last significand bit */
}

/* Replace freshly built fp32 metadata (orc_build_stats) by its stored form, in place.
 * bound: 0 = KV dtype (unchanged), 1 = e4m3 outward; stat: 0 = fp32, 1 = bf16.     */
void orc_store_meta(float *kmin, float *kmax, float *kavg, float *kvar, size_t n, int bound, int stat)
{
    for (size_t i = 0; i < n; ++i) {
        if (bound == 1) {
            kmin[i] = orc_e4m3_round_down(kmin[i]);
            kmax[i] = orc_e4m3_round_up(kmax[i]);
        }
        if (stat == 1) {
            kavg[i] = orc_bf16_round(kavg[i]);
            kvar[i] = orc_bf16_round(kvar[i]);
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Query-aware page scoring for ONE query head (kv head kvh) of one sequence. */
/*  box  = (1/sqrt d) sum_i max(q_i kmin_i, q_i kmax_i)  Eq. box-page-bound    */
/*         (P:321-333); evaluated as dot16x8(q, kext), kext_i = q_i>=0 ? kmax  */
/*         : kmin (the max of the two products, Prop. B.1 proof P:815).        */
/*  mu   = q^T kavg / sqrt d                     */
/*  sig2 = (1/d) sum_i q_i^2 kstd_i^2                     */
/* meta arrays: [n_phys][Hkv][d]; page_row: logical page -> physical page.    */
/* modes: bit0 box, bit1 gaussian.                                            */
/* ------------------------------------------------------------------------- */
void orc_score_pages(const float *q, int kvh, int Hkv, const float *kmin,
                     const float *kmax, const float *kavg, const float *kvar,
                     const int32_t *page_row, int M, int modes,
                     float *box, float *mu, float *sigma2)
{
    const int d = ORC_D;
    float kext[ORC_D], q2[ORC_D];
    for (int i = 0; i < d; ++i) q2[i] = q[i] * q[i];
    for (int p = 0; p < M; ++p) {
        size_t off = ((size_t)page_row[p] * Hkv + kvh) * d;
        if (modes & 1) {
            for (int i = 0; i < d; ++i)
                kext[i] = (q[i] >= 0.0f) ? kmax[off + i] : kmin[off + i];
            box[p] = orc_dot_canon(q, kext) * scale_cd();
        }
        if (modes & 2) {
            mu[p] = orc_dot_canon(q, kavg + off) * scale_cd();
            sigma2[p] = orc_dot_canon(q2, kvar + off) * (1.0f / (float)d);
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Top-k page selection: the min(k,M) pages with the largest box   */
/* score; tie -> lower page index (R3).  Output ascending page index.   */
/* ------------------------------------------------------------------------- */
typedef struct { double key; int32_t idx; } orc_kv;
static int cmp_desc_then_idx(const void *a, const void *b)
{
    const orc_kv *x = a, *y = b;
    if (x->key > y->key) return -1;
    if (x->key < y->key) return 1;
    return (x->idx < y->idx) ? -1 : (x->idx > y->idx);
}
static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x < y) ? -1 : (x > y);
}
int orc_topk(const float *score, int M, int k, int32_t *out)
{
    if (k > M) k = M;
    orc_kv *v = malloc(sizeof(orc_kv) * (size_t)(M > 0 ? M : 1));
    for (int p = 0; p < M; ++p) { v[p].key = (double)score[p]; v[p].idx = p; }
    qsort(v, (size_t)M, sizeof(orc_kv), cmp_desc_then_idx);
    for (int i = 0; i < k; ++i) out[i] = v[i].idx;
    qsort(out, (size_t)k, sizeof(int32_t), cmp_i32);
    free(v);
    return k;
}

/* ------------------------------------------------------------------------- */
/* alpha-entmax (Eq. entmax-def, support Eq. P:137-148, App. A).    */
/* z_i = (alpha-1) s_i is passed in.  beta = 1/(alpha-1).                      */
/* Support by the threshold-free criterion (R9): with F(x) = sum_i (z_i-x)_+^b */
/* strictly decreasing below max z and F(tau) = 1,  i in S  <=>  F(z_i) < 1.   */
/* Evaluated on z sorted descending: F(z_(k)) = sum_{i<k} (z_(i)-z_(k))^beta,   */
/* non-decreasing in k, so the support is the prefix before the first F >= 1.  */
/* tau: beta=1 (sparsemax) (S1-1)/k; beta=2 m - sqrt((1-ss)/k); otherwise      */
/* bisection on sum_{i in S}(z_i - tau)^beta = 1.  p_i = (z_i - tau)^beta.     */
/* ------------------------------------------------------------------------- */
static double powb(double x, double beta)
{
    if (beta == 1.0) return x;
    if (beta == 2.0) return x * x;
    if (beta == 3.0) return (x * x) * x;
    if (beta == 4.0) { double x2 = x * x; return x2 * x2; }
    return pow(x, beta);
}
static int cmp_desc_d(const void *a, const void *b)
{
    const orc_kv *x = a, *y = b;
    if (x->key > y->key) return -1;
    if (x->key < y->key) return 1;
    return (x->idx < y->idx) ? -1 : (x->idx > y->idx);
}

int orc_entmax(const double *z, int n, double alpha, double *p, double *tau_out)
{
    const double beta = 1.0 / (alpha - 1.0);
    if (n <= 0) { if (tau_out) *tau_out = NAN; return 0; }
    orc_kv *v = malloc(sizeof(orc_kv) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) { v[i].key = z[i]; v[i].idx = i; }
    qsort(v, (size_t)n, sizeof(orc_kv), cmp_desc_d);
    int k;
    for (k = 0; k < n; ++k) {
        double x = v[k].key, F = 0.0;
        for (int i = 0; i < k; ++i) F += powb(v[i].key - x, beta);
        if (!(F < 1.0)) break;
    }
    double tau;
    if (beta == 1.0) {
        double s1 = 0.0;
        for (int i = 0; i < k; ++i) s1 += v[i].key;
        tau = (s1 - 1.0) / (double)k;
    } else if (beta == 2.0) {
        double s1 = 0.0, ss = 0.0;
        for (int i = 0; i < k; ++i) s1 += v[i].key;
        double m = s1 / (double)k;
        for (int i = 0; i < k; ++i) ss += (v[i].key - m) * (v[i].key - m);
        tau = m - sqrt((1.0 - ss) / (double)k);
    } else {
        double hi = v[k - 1].key, lo = v[0].key - 1.0;
        for (int it = 0; it < 400; ++it) {
            double mid = 0.5 * (lo + hi);
            if (mid <= lo || mid >= hi) break;
            double G = 0.0;
            for (int i = 0; i < k; ++i) G += powb(v[i].key - mid, beta);
            if (G >= 1.0) lo = mid; else hi = mid;
        }
        tau = 0.5 * (lo + hi);
    }
    for (int i = 0; i < n; ++i) p[i] = 0.0;
    for (int i = 0; i < k; ++i) {
        double x = v[i].key - tau;
        p[v[i].idx] = x > 0.0 ? powb(x, beta) : 0.0;
    }
    free(v);
    if (tau_out) *tau_out = tau;
    return k;
}

/* ------------------------------------------------------------------------- */
/* Approximate tau, the paper's kernel recipe ("estimates the entmax   */
/* threshold tau using a histogram-based initialization followed by Halley     */
/* iterations"; DESIGN reading R23 fixes the unstated details):                */
/*  1. 64 bins over (z_max - 1, z_max]: z in bin b iff b = min(63,            */
/*     floor((z_max - z) * 64)), for z > z_max - 1 (tau >= z_max - 1);         */
/*  2. tau_0 = the largest edge e_k = z_max - k/64 whose certified lower bound  */
/*     LB_k = sum_{b<k} cnt_b ((k-1-b)/64)^beta reaches 1 (else z_max - 1);    */
/*  3. h Halley steps on f(t) = sum_{z>t} (z-t)^beta - 1:                      */
/*     t <- t - 2 f f' / (2 f'^2 - f f''), f' = -beta S_{beta-1},              */
/*     f'' = beta (beta-1) S_{beta-2}, S_m = sum_{z>t} (z-t)^m;                  */
/*  4. p_i = (z_i - tau)_+^beta (normalised by the caller, R12).               */
/* Returns |{z > tau}|.                                                         */
/* ------------------------------------------------------------------------- */
static int entmax_halley_from(const double *z, int n, double beta, double zmax, double t, int h, double *p,
                              double *tau_out);

int orc_entmax_approx(const double *z, int n, double alpha, int h, double *p, double *tau_out)
{
    const double beta = 1.0 / (alpha - 1.0);
    if (n <= 0) { if (tau_out) *tau_out = NAN; return 0; }
    double zmax = z[0];
    for (int i = 1; i < n; ++i) if (z[i] > zmax) zmax = z[i];
    double cnt[64] = {0};
    for (int i = 0; i < n; ++i) {
        if (!(z[i] > zmax - 1.0)) continue;
        double fb = floor((zmax - z[i]) * 64.0);
        int b = fb > 63.0 ? 63 : (int)fb;
        cnt[b] += 1.0;
    }
    double t = zmax - 1.0;
    for (int k = 1; k <= 64; ++k) {
        double lb = 0.0;
        for (int b = 0; b < k; ++b) lb += cnt[b] * powb((double)(k - 1 - b) / 64.0, beta);
        if (lb >= 1.0) { t = zmax - (double)k / 64.0; break; }
    }
    return entmax_halley_from(z, n, beta, zmax, t, h, p, tau_out);
}

/* ------------------------------------------------------------------------- */
/* The Gaussian variant's approximate tau ("The selected page indices  */
/* and estimated threshold are then passed to the decode kernel. Inside the   */
/* kernel, we perform one additional Halley refinement using the actual       */
/* selected scores"): start at the selector's tau_hat, then h Halley steps     */
/* (step 3 above).  DESIGN R25: tau_hat outside [z_max - 1, z_max) -- where    */
/* the exact tau always lies (F(z_max - 1) >= 1 > F(z_max) = 0) -- is replaced */
/* by z_max - 1.                                                              */
/* ------------------------------------------------------------------------- */
int orc_entmax_approx_init(const double *z, int n, double alpha, double tau0, int h, double *p, double *tau_out)
{
    const double beta = 1.0 / (alpha - 1.0);
    if (n <= 0) { if (tau_out) *tau_out = NAN; return 0; }
    double zmax = z[0];
    for (int i = 1; i < n; ++i) if (z[i] > zmax) zmax = z[i];
    double t = (tau0 >= zmax - 1.0 && tau0 < zmax) ? tau0 : zmax - 1.0;
    return entmax_halley_from(z, n, beta, zmax, t, h, p, tau_out);
}

/* h Halley steps from t (step 3); R25: an iterate below z_max - 1 (the exact tau's lower bound)
 * is raised to z_max - 1. */
static int entmax_halley_from(const double *z, int n, double beta, double zmax, double t, int h, double *p,
                              double *tau_out)
{
    for (int it = 0; it < h; ++it) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;   /* sum w^beta, w^(beta-1), w^(beta-2), w = z - t > 0 */
        for (int i = 0; i < n; ++i) {
            double w = z[i] - t;
            if (w > 0.0) {
                s0 += powb(w, beta);
                s1 += powb(w, beta - 1.0);
                s2 += (beta == 1.0) ? 0.0 : powb(w, beta - 2.0);
            }
        }
        double f = s0 - 1.0, fp = -beta * s1, fpp = beta * (beta - 1.0) * s2;
        double den = 2.0 * fp * fp - f * fpp;
        if (!(den != 0.0)) break;
        t -= 2.0 * f * fp / den;
        if (t < zmax - 1.0) t = zmax - 1.0;
    }
    int k = 0;
    for (int i = 0; i < n; ++i) {
        double w = z[i] - t;
        p[i] = w > 0.0 ? powb(w, beta) : 0.0;
        k += w > 0.0;
    }
    if (tau_out) *tau_out = t;
    return k;
}

/* softmax, fp64 with max subtraction. Returns log-normalizer. */
double orc_softmax(const double *s, int n, double *p)
{
    double mx = s[0], sum = 0.0;
    for (int i = 1; i < n; ++i) if (s[i] > mx) mx = s[i];
    for (int i = 0; i < n; ++i) { p[i] = exp(s[i] - mx); sum += p[i]; }
    for (int i = 0; i < n; ++i) p[i] /= sum;
    return mx + log(sum);
}

/* ------------------------------------------------------------------------- */
/* Attention over a page set for ONE query head of one sequence              */
/* (C_tok = union of the selected pages' tokens; p~ = transform of  */
/* {s_j : j in C_tok}; o~ = sum_j p~_j v_j; p~_j = 0 outside C_tok).           */
/* Kp, Vp: [n_phys][Hkv][P][d]; pages: logical page ids (any order, unique).   */
/* transform: 0 = alpha-entmax, 1 = softmax.                                   */
/* Outputs: o[dv] (fp64), *tau (entmax tau or softmax log-normalizer),         */
/* p_tok[seq_len] (optional; dense over the sequence, 0 outside C_tok),        */
/* s_tok[seq_len] (optional; fp32 scores of C_tok tokens, untouched elsewhere).*/
/* Returns the support size (entmax) or |C_tok| (softmax).                      */
/* ------------------------------------------------------------------------- */
int orc_attend(const float *q, const float *Kp, const float *Vp,
               const int32_t *page_row, int seq_len, int kvh, int Hkv, int P,
               int dv, const int32_t *pages, int n_pages, double alpha,
               int transform, double *o, double *tau, double *p_tok,
               float *s_tok, int approx_h, double tau0)
{
    const int d = ORC_D;
    int cap = n_pages * P;
    int32_t *tok = malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
    double *z = malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
    double *pr = malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
    int n = 0;
    for (int ip = 0; ip < n_pages; ++ip) {
        int lp = pages[ip];
        for (int t = 0; t < P; ++t) {
            int j = lp * P + t;
            if (j >= seq_len) break;
            size_t off = (((size_t)page_row[lp] * Hkv + kvh) * P + t) * d;
            float s = orc_token_score(q, Kp + off);
            if (s_tok) s_tok[j] = s;
            tok[n] = j;
            z[n] = (transform == 0) ? (alpha - 1.0) * (double)s : (double)s;
            ++n;
        }
    }
    int ret;
    if (n == 0) ret = 0, *tau = NAN;
    else if (transform == 0 && approx_h > 0 && tau0 == tau0)     /* tau0 given (not NaN): P:488 */
        ret = orc_entmax_approx_init(z, n, alpha, tau0, approx_h, pr, tau);
    else if (transform == 0 && approx_h > 0) ret = orc_entmax_approx(z, n, alpha, approx_h, pr, tau);
    else if (transform == 0) ret = orc_entmax(z, n, alpha, pr, tau);
    else { *tau = orc_softmax(z, n, pr); ret = n; }
    for (int i = 0; i < dv; ++i) o[i] = 0.0;
    if (p_tok) for (int j = 0; j < seq_len; ++j) p_tok[j] = 0.0;
    if (transform == 0 && approx_h > 0 && n > 0) {       /* R12: o = sum p v / sum p */
        double ps = 0.0;
        for (int m = 0; m < n; ++m) ps += pr[m];
        for (int m = 0; m < n; ++m) pr[m] /= ps;
    }
    for (int m = 0; m < n; ++m) {
        int j = tok[m];
        if (p_tok) p_tok[j] = pr[m];
        if (pr[m] == 0.0) continue;
        int lp = j / P, t = j % P;
        size_t off = (((size_t)page_row[lp] * Hkv + kvh) * P + t) * dv;
        for (int i = 0; i < dv; ++i) o[i] += pr[m] * (double)Vp[off + i];
    }
    free(tok); free(z); free(pr);
    return ret;
}

/* ------------------------------------------------------------------------- */
/* Metrics (P:165-171 delta, P:220-232 rho).  p_full over all n tokens,        */
/* in_keep[j] != 0 iff j in C_tok.  rho = 1 when the support is empty. */
/* ------------------------------------------------------------------------- */
void orc_metrics(const double *p_full, const uint8_t *in_keep, int n,
                 double *delta, double *rho, int32_t *recovered, int32_t *full_supp)
{
    double dl = 0.0; int rec = 0, sup = 0;
    for (int j = 0; j < n; ++j) {
        if (!in_keep[j]) dl += p_full[j];
        if (p_full[j] > 0.0) { ++sup; if (in_keep[j]) ++rec; }
    }
    *delta = dl;
    *rho = sup ? (double)rec / (double)sup : 1.0;
    *recovered = rec; *full_supp = sup;
}

/* ------------------------------------------------------------------------- */
/* Gaussian-aware selection (App. D).                   */
/* ------------------------------------------------------------------------- */
static double Phi(double t) { return 0.5 * erfc(-t / sqrt(2.0)); }
static double phi(double t) { return exp(-0.5 * t * t) / sqrt(2.0 * M_PI); }

/* E[(Y)_+^beta], Y ~ N(muY, sigY^2), t = muY/sigY.  Closed forms of App. D:   */
/*   beta=1: muY Phi + sigY phi               */
/*   beta=2: (muY^2+sigY^2) Phi + muY sigY phi               */
/*   beta=3: (muY^3+3muY sigY^2) Phi + (muY^2 sigY + 2 sigY^3) phi*/
/*   beta=4: not printed in the paper (R15): the same truncated-moment        */
/*           recursion M_k = muY M_{k-1} + (k-1) sigY^2 M_{k-2}, M_0 = Phi,     */
/*           M_1 = muY Phi + sigY phi, which reproduces the three above.       */
/*   sigY = 0: point mass [muY]_+^beta.                               */
double orc_trunc_moment(int beta, double muY, double sigY)
{
    if (!(sigY > 0.0)) {
        double x = muY > 0.0 ? muY : 0.0;
        double r = 1.0;
        for (int i = 0; i < beta; ++i) r *= x;
        return r;
    }
    double t = muY / sigY, Ph = Phi(t), ph = phi(t);
    switch (beta) {
    case 1: return muY * Ph + sigY * ph;
    case 2: return (muY * muY + sigY * sigY) * Ph + muY * sigY * ph;
    case 3: return (muY * muY * muY + 3.0 * muY * sigY * sigY) * Ph
                 + (muY * muY * sigY + 2.0 * sigY * sigY * sigY) * ph;
    default: {
        double m0 = Ph, m1 = muY * Ph + sigY * ph, m2 = 0.0;
        for (int k = 2; k <= beta; ++k) {
            m2 = muY * m1 + (double)(k - 1) * sigY * sigY * m0;
            m0 = m1; m1 = m2;
        }
        return m1;
    }
    }
}

/* E[(Y)_+^beta] for a real beta > 0 ("for generic alpha > 1  */
/* with non-integer beta ... the expectation can be evaluated numerically").          */
/* E = sigY^beta h(m), m = muY / sigY, h(m) = int_0^inf u^beta phi(u - m) du, by       */
/* tanh-sinh (double-exponential) quadrature on [L, U] = [max(0, m - 12),             */
/* max(m, 0) + 12] (phi(12) < 3e-32: the cut tails are below fp64 resolution), the    */
/* step halved from 1/8 until two successive sums agree to 1e-13 relative (the        */
/* double-exponential rule's error roughly squares per halving, so the finer sum is  */
/* then at fp64 resolution; at most 7 halvings).  The                                 */
/* substitution u = c + w tanh(pi/2 sinh t) clusters the nodes at the ends, which     */
/* absorbs the u^beta endpoint singularity at u = 0 (DESIGN R28).  sigY = 0: the     */
/* point mass [muY]_+^beta.                                                           */
double orc_trunc_moment_num(double beta, double muY, double sigY)
{
    if (!(sigY > 0.0)) return muY > 0.0 ? pow(muY, beta) : 0.0;
    double m = muY / sigY;
    double L = m - 12.0 > 0.0 ? m - 12.0 : 0.0;
    double U = (m > 0.0 ? m : 0.0) + 12.0;
    double hw = 0.5 * (U - L);
    double prev = NAN, s = 0.0;
    for (double h = 0.125; h > 0.0009; h *= 0.5) {
        s = 0.0;
        int K = (int)ceil(4.5 / h);
        for (int k = -K; k <= K; ++k) {
            double t = k * h;
            double y = 0.5 * M_PI * sinh(t);
            double e = exp(-2.0 * fabs(y));
            /* distance from the nearer end: w (1 - tanh|y|) = 2 w e / (1 + e) (no cancellation) */
            double dnear = 2.0 * hw * e / (1.0 + e);
            double u = (t < 0.0) ? L + dnear : U - dnear;
            double ch = cosh(y);
            double wgt = hw * 0.5 * M_PI * cosh(t) / (ch * ch);
            if (!(wgt > 0.0) || !(u > 0.0)) continue;
            s += wgt * pow(u, beta) * exp(-0.5 * (u - m) * (u - m));
        }
        s *= h / sqrt(2.0 * M_PI);
        if (fabs(s - prev) <= 1e-13 * fabs(s)) break;
        prev = s;
    }
    return pow(sigY, beta) * s;
}

/* Approximate normalization mass  sum_p |P_p| E[g_alpha(S^(p); tau)]          */
/* (Eq. gaussian-threshold-main), S^(p) ~ N(mu_p, sigma_p^2),        */
/* Y = a S - tau: muY = a mu - tau, sigY = a sigma.              */
double orc_gauss_mass(const float *mu, const float *sigma2, const int32_t *counts,
                      int M, double alpha, double tau)
{
    double a = alpha - 1.0;
    double bd = 1.0 / a;
    int beta = (int)lround(bd);
    /* integer beta: App. D's closed forms; any other beta > 0: the numerical expectation  */
    /* (orc_trunc_moment_num) -- never a rounded beta                   */
    int closed = fabs(bd - (double)beta) <= 1e-12 && beta >= 1;
    if (!(a > 0.0)) return NAN;
    double m = 0.0;
    for (int p = 0; p < M; ++p) {
        double s = sqrt((double)sigma2[p]);
        double muY = a * (double)mu[p] - tau, sigY = a * s;
        m += (double)counts[p] * (closed ? orc_trunc_moment(beta, muY, sigY)
                                         : orc_trunc_moment_num(bd, muY, sigY));
    }
    return m;
}

/* tau_hat: the root of mass(tau) = 1.  The mass is continuous,  */
/* non-increasing in tau and strictly decreasing where positive.       */
/* Plain bracketing + bisection to fp64 resolution (the paper's Newton/Halley */
/* is a faster route to the same root).  Returns 0 on success, -1 on a bracket */
/* failure, -2 for alpha <= 1.  Non-integer beta: the numerical expectation.    */
int orc_gauss_tau(const float *mu, const float *sigma2, const int32_t *counts,
                  int M, double alpha, double *tau_hat)
{
    double a = alpha - 1.0, top = -INFINITY;
    if (isnan(orc_gauss_mass(mu, sigma2, counts, 0, alpha, 0.0))) return -2;   /* alpha <= 1 */
    for (int p = 0; p < M; ++p) {
        double v = a * ((double)mu[p] + 8.0 * sqrt((double)sigma2[p]));
        if (v > top) top = v;
    }
    double hi = top, w = 1.0;
    int guard = 0;
    while (orc_gauss_mass(mu, sigma2, counts, M, alpha, hi) >= 1.0) {
        hi += w; w *= 2.0;
        if (++guard > 200) return -1;
    }
    double lo = hi - 1.0;
    w = 1.0; guard = 0;
    while (orc_gauss_mass(mu, sigma2, counts, M, alpha, lo) < 1.0) {
        lo -= w; w *= 2.0;
        if (++guard > 200) return -1;
    }
    for (int it = 0; it < 400; ++it) {
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (orc_gauss_mass(mu, sigma2, counts, M, alpha, mid) >= 1.0) lo = mid;
        else hi = mid;
    }
    *tau_hat = 0.5 * (lo + hi);
    return 0;
}

/* Phi^{-1}(u) by bisection on Phi (u in (0,1)); used for the page-max        */
/* quantile q_page^{1/|P_p|} of Eq. gaussian-page-bound-main.      */
double orc_norm_ppf(double u)
{
    /* symmetry Phi^{-1}(u) = -Phi^{-1}(1-u): bisect in the lower tail, where Phi */
    /* (via erfc) keeps full relative precision; 1-u is exact for u in [0.5, 1].  */
    if (u > 0.5) return -orc_norm_ppf(1.0 - u);
    double lo = -40.0, hi = 40.0;
    for (int it = 0; it < 400; ++it) {
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (Phi(mid) < u) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

/* Page rule (Eq. gaussian-selector-main):                          */
/*   keep p iff (alpha-1) * sbar_G(p) > tau_hat - Delta,                       */
/*   sbar_G = mu + sigma * zq[c_p],  zq[c] = Phi^{-1}(q_page^{1/c})*/
/* sbar_G is evaluated as fmaf(sqrtf(sigma2), (float)zq[c], mu) (R14) and the   */
/* comparison in fp64.  Empty selection -> argmax mu, lower index on ties (R6).*/
/* Output ascending.  Returns the count.                                       */
int orc_gauss_select(const float *mu, const float *sigma2, const int32_t *counts,
                     int M, double alpha, double tau_hat, double margin,
                     const double *zq /* [P+1], zq[c] */, int32_t *out)
{
    double a = alpha - 1.0;
    int n = 0;
    for (int p = 0; p < M; ++p) {
        float sg = fmaf(sqrtf(sigma2[p]), (float)zq[counts[p]], mu[p]);
        if (a * (double)sg > tau_hat - margin) out[n++] = p;
    }
    if (n == 0 && M > 0) {
        int best = 0;
        for (int p = 1; p < M; ++p) if (mu[p] > mu[best]) best = p;
        out[n++] = best;
    }
    return n;
}

/* Certified dropped-mass bound (R16): with z_j <= a*box_p     */
/* (Prop. B.1) and tau >= tau~ (sparse tau is a lower bound of the  */
/* full tau), delta <= sum_{p not selected} c_p [a*box_p - tau~]_+^beta.        */
double orc_delta_bar(const float *box, const int32_t *counts, const uint8_t *sel,
                     int M, double alpha, double tau_sparse)
{
    double a = alpha - 1.0, beta = 1.0 / a, s = 0.0;
    for (int p = 0; p < M; ++p) {
        if (sel[p]) continue;
        double x = a * (double)box[p] - tau_sparse;
        if (x > 0.0) s += (double)counts[p] * powb(x, beta);
    }
    return s;
}

/* Support-superset (certified conservative) page selection, SURVEY 8(f) N4 --   */
/* Prop. B.2 "No false negatives from deterministic page bounds":     */
/* C_page = {p : (alpha-1) * sbar_box(p) > tau_hat}, for any tau_hat <= tau.       */
/* The decision is taken in fp64 (R9's precision for z): (double)a * box[p].      */
/* Ascending page ids; returns |C_page|.  DESIGN R27: tau_hat is the exact         */
/* threshold of a first top-k pass (a lower bound of tau by R13).                  */
int orc_box_certified(const float *box, int M, double alpha, double tau_hat, int32_t *out)
{
    double a = alpha - 1.0;
    int n = 0;
    for (int p = 0; p < M; ++p)
        if (a * (double)box[p] > tau_hat) out[n++] = p;
    return n;
}
