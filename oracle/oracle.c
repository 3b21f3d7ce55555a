/*
 * oracle.c -- CPU restatement of the AdaFuse hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The shipped
 * path (paper_2603_11873_b200/) never links, imports or calls anything in oracle/.
 *
 * Every function restates one piece of the reference `lorafuse` package
 * (/root/reference/pkg/src/lorafuse, cited per function as file:line) in plain C.
 * Parity status: PINNED -- tests/test_oracle_golden.py checks these functions
 * against (a) the golden values the reference's own tests hold and (b) fixtures
 * produced by importing the unmodified Python reference (tests/golden/make_golden.py).
 *
 * Numerical contract restated here (verified against the
 * reference in "single" precision):
 *   - sgmm: per element, strict ascending-rank sequence of (multiply -> round to f32)
 *     then (add -> round to f32); no FMA.  Compile with -ffp-contract=off.
 *   - gate folding: down_cat block = (float)w * down, one f32 multiply; up_cat unscaled.
 *   - switch: down = [-prev.down_cat ; cur.down_cat], up = [prev.up_cat | cur.up_cat].
 *   - route: logits = W_g x ; stable descending order (ties -> lower index);
 *     softmax over the selected logits only, max-shifted, correctly rounded to f32.
 *
 * The one deliberate deviation: dot products (router logits, GEMVs) and the k-term softmax
 * accumulate in double and round once to f32.  The reference delegates those to numpy `@`
 * (OpenBLAS, linalg.py:252), whose summation order is unspecified; the correctly
 * rounded f32 dot product is inside OpenBLAS' own round-off band and is order
 * independent, which is what lets the GPU kernels match it bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EVALUE 1   /* ValueError    (bad k / sign)              */
#define ORC_EDIM 2     /* DimensionError                              */
#define ORC_EINDEX 3   /* IndexError    (expert id outside the bank)  */

/* ---------------------------------------------------------------- bf16 ---- */

/* Round-to-nearest-even f32 -> bf16 (the storage rounding of the B200 build). */
uint16_t orc_f32_to_bf16(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x0040u); /* NaN */
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

float orc_bf16_to_f32(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

void orc_round_to_bf16(const float* src, uint16_t* dst, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) dst[i] = orc_f32_to_bf16(src[i]);
}

void orc_widen_bf16(const uint16_t* src, float* dst, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) dst[i] = orc_bf16_to_f32(src[i]);
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* torchrun exports OMP_NUM_THREADS=1 to its workers; the timed baseline asks for the host's cores explicitly. */
void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* --------------------------------------------------------------- router --- */

/* routing.py:49-78 `route` (== `pre_gate`, routing.py:81-89).
 * wg: N x d row-major, x: d.  ids/weights: k outputs.  logits_out (optional): N.
 * Validation order follows routing.py:57-62 (k first; the shape check is the caller's
 * since x arrives as a bare pointer). */
int orc_route(const float* wg, int n_experts, int d, const float* x, int k,
              int32_t* ids, float* weights, float* logits_out) {
    if (k < 1 || k > n_experts) return ORC_EVALUE;
    float* logits = (float*)malloc(sizeof(float) * (size_t)n_experts);
    for (int e = 0; e < n_experts; ++e) {
        double acc = 0.0;
        const float* row = wg + (size_t)e * d;
        for (int j = 0; j < d; ++j) acc += (double)row[j] * (double)x[j];
        logits[e] = (float)acc;
    }
    if (logits_out) memcpy(logits_out, logits, sizeof(float) * (size_t)n_experts);
    /* routing.py:64-65: argsort(-logits, kind="stable")[:k].  Selection by repeated
     * strict-greater scan reproduces it: the first index holding the maximum wins, and
     * +0.0 / -0.0 compare equal so index order decides (Appendix A). */
    char* taken = (char*)calloc((size_t)n_experts, 1);
    for (int j = 0; j < k; ++j) {
        int best = -1;
        for (int e = 0; e < n_experts; ++e) {
            if (taken[e]) continue;
            if (best < 0 || logits[e] > logits[best]) best = e;
        }
        taken[best] = 1;
        ids[j] = best;
    }
    /* routing.py:66-68: softmax over the selected logits only, max-shifted.  Evaluated in
     * double (exp, left-to-right sum, division) and rounded once to f32: the correctly rounded
     * f32 softmax.  The reference evaluates it in f32 with numpy's exp; f32 exp
     * implementations (numpy SIMD, glibc, CUDA) differ among themselves by an ulp, so the
     * correctly rounded value is the one restatement every platform can reproduce bit for
     * bit; it is within 1 f32 ulp of the reference (pinned at 1e-5 in test_oracle_golden). */
    float mx = logits[ids[0]];
    double ex[64];
    double sum = 0.0;
    for (int j = 0; j < k; ++j) {
        ex[j & 63] = exp((double)logits[ids[j]] - (double)mx);
        sum += ex[j & 63];
    }
    if (k <= 64) {
        for (int j = 0; j < k; ++j) weights[j] = (float)(ex[j] / sum);
    } else { /* very wide k: recompute instead of buffering */
        for (int j = 0; j < k; ++j) weights[j] = (float)(exp((double)logits[ids[j]] - (double)mx) / sum);
    }
    free(taken);
    free(logits);
    return ORC_OK;
}

/* ------------------------------------------------------- adapter algebra --- */

/* adapters.py:188-211 `concat_gated` followed by adapters.py:214-233 `build_switch`,
 * for ONE adapted matrix.
 *   down_bank: [N][r][d_in]   (LoraExpert.down, adapters.py:53)
 *   up_bank  : [N][d_out][r]  (LoraExpert.up,   adapters.py:54)
 *   prev (kp ids/weights, kp may be 0 = ConcatAdapter.empty) and cur (kc >= 0).
 * Outputs: down_cat (s x d_in), up_cat (d_out x s), s = (kp + kc) * r.
 * Block order = prev blocks then cur blocks, each in its gate's expert order
 * (adapters.py:230-231); prev DOWN blocks are negated AFTER gate folding
 * (adapters.py:206 then :230). */
int orc_switch_factors(const float* down_bank, const float* up_bank, int n_experts, int r,
                       int d_out, int d_in, const int32_t* prev_ids, const float* prev_w, int kp,
                       const int32_t* cur_ids, const float* cur_w, int kc, float* down_cat,
                       float* up_cat) {
    int nb = kp + kc;
    int s = nb * r;
    for (int b = 0; b < nb; ++b) {
        int e = b < kp ? prev_ids[b] : cur_ids[b - kp];
        float w = b < kp ? prev_w[b] : cur_w[b - kp];
        if (e < 0 || e >= n_experts) return ORC_EINDEX; /* adapters.py:199-200 */
        const float* dn = down_bank + (size_t)e * r * d_in;
        const float* up = up_bank + (size_t)e * d_out * r;
        for (int q = 0; q < r; ++q) {
            float* dst = down_cat + (size_t)(b * r + q) * d_in;
            const float* src = dn + (size_t)q * d_in;
            for (int j = 0; j < d_in; ++j) {
                float v = w * src[j];       /* adapters.py:202: w * e.down.data (f32) */
                dst[j] = b < kp ? -v : v;   /* adapters.py:230: -prev.down_cat        */
            }
        }
        for (int i = 0; i < d_out; ++i)
            for (int q = 0; q < r; ++q)
                up_cat[(size_t)i * s + b * r + q] = up[(size_t)i * r + q];
    }
    return ORC_OK;
}

/* linalg.py:306-346 `sgmm`, one segment: target (d_out x d_in) += sign * up @ down as
 * the strict ascending-rank recurrence of linalg.py:338-343.  Tile extents do not
 * change bits (linalg.py:21-26), so the restatement walks whole rows. */
int orc_sgmm_segment(float* target, const float* up, const float* down, int d_out, int d_in,
                     int s, int sign) {
    if (sign != 1 && sign != -1) return ORC_EVALUE;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < d_out; ++i) {
        float* row = target + (size_t)i * d_in;
        const float* u = up + (size_t)i * s;
        for (int q = 0; q < s; ++q) {
            const float uq = u[q];
            const float* dn = down + (size_t)q * d_in;
            if (sign > 0) {
                for (int j = 0; j < d_in; ++j) {
                    float outer = uq * dn[j]; /* rounded product */
                    row[j] = row[j] + outer;  /* rounded add     */
                }
            } else {
                for (int j = 0; j < d_in; ++j) {
                    float outer = uq * dn[j];
                    row[j] = row[j] - outer;
                }
            }
        }
    }
    return ORC_OK;
}

/* linalg.py:262-290 `gemm_accumulate_inplace`: C += sign * (A @ B), product first
 * (double accumulate, one f32 rounding -- see header), then ONE add (linalg.py:280-284).
 * a: m x s, b: s x n, c: m x n. */
int orc_gemm_accumulate(float* c, const float* a, const float* b, int m, int n, int s, int sign) {
    if (sign != 1 && sign != -1) return ORC_EVALUE;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < m; ++i) {
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int q = 0; q < s; ++q) acc += (double)a[(size_t)i * s + q] * (double)b[(size_t)q * n + j];
            float prod = (float)acc;
            float* dst = c + (size_t)i * n + j;
            *dst = sign > 0 ? *dst + prod : *dst - prod;
        }
    }
    return ORC_OK;
}

/* The per-step parity oracle of the bf16 build (SURVEY.md section 7 hard part 2,
 * BASELINE.md section 4.4): the reference f32 switch applied to the upcast of the
 * live bf16 weights, result rounded RNE to bf16.  One adapted matrix, in place.
 * Factors are f32 arrays carrying bf16-representable bank values; the switch factors
 * are formed exactly as orc_switch_factors does, but streamed row by row so a
 * Llama-sized matrix needs no d_out x s / s x d_in temporaries beyond the slab. */
int orc_switch_segment_bf16(uint16_t* w, const uint16_t* down_bank, const uint16_t* up_bank,
                            int n_experts, int r, int d_out, int d_in, const int32_t* prev_ids,
                            const float* prev_w, int kp, const int32_t* cur_ids,
                            const float* cur_w, int kc) {
    int nb = kp + kc;
    int s = nb * r;
    for (int b = 0; b < nb; ++b) {
        int e = b < kp ? prev_ids[b] : cur_ids[b - kp];
        if (e < 0 || e >= n_experts) return ORC_EINDEX;
    }
    if (s == 0) return ORC_OK;
    /* gate-folded, sign-folded DOWN slab: s x d_in f32 (adapters.py:202, :230) */
    float* down_cat = (float*)malloc(sizeof(float) * (size_t)s * d_in);
    for (int b = 0; b < nb; ++b) {
        int e = b < kp ? prev_ids[b] : cur_ids[b - kp];
        float wgt = b < kp ? prev_w[b] : cur_w[b - kp];
        for (int q = 0; q < r; ++q) {
            const uint16_t* src = down_bank + ((size_t)e * r + q) * d_in;
            float* dst = down_cat + (size_t)(b * r + q) * d_in;
            for (int j = 0; j < d_in; ++j) {
                float v = wgt * orc_bf16_to_f32(src[j]);
                dst[j] = b < kp ? -v : v;
            }
        }
    }
#pragma omp parallel
    {
        float* row = (float*)malloc(sizeof(float) * (size_t)d_in);
#pragma omp for schedule(static)
        for (int i = 0; i < d_out; ++i) {
            uint16_t* wrow = w + (size_t)i * d_in;
            for (int j = 0; j < d_in; ++j) row[j] = orc_bf16_to_f32(wrow[j]);
            for (int b = 0; b < nb; ++b) {
                int e = b < kp ? prev_ids[b] : cur_ids[b - kp];
                const uint16_t* u = up_bank + ((size_t)e * d_out + i) * r;
                for (int q = 0; q < r; ++q) {
                    const float uq = orc_bf16_to_f32(u[q]);
                    const float* dn = down_cat + (size_t)(b * r + q) * d_in;
                    for (int j = 0; j < d_in; ++j) {
                        float outer = uq * dn[j];
                        row[j] = row[j] + outer; /* merge_all(sign=+1), model.py:357 */
                    }
                }
            }
            for (int j = 0; j < d_in; ++j) wrow[j] = orc_f32_to_bf16(row[j]);
        }
        free(row);
    }
    free(down_cat);
    return ORC_OK;
}

/* ------------------------------------------------------------- forward ---- */

/* linalg.py:246-259 `gemm` used as a bs=1 GEMV: y = W x (W: rows x cols row-major). */
void orc_gemv(const float* w, const float* x, float* y, int rows, int cols) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < rows; ++i) {
        double acc = 0.0;
        const float* row = w + (size_t)i * cols;
        for (int j = 0; j < cols; ++j) acc += (double)row[j] * (double)x[j];
        y[i] = (float)acc;
    }
}

/* Same GEMV over bf16-stored weights (the live merged backbone of the B200 build). */
void orc_gemv_bf16(const uint16_t* w, const float* x, float* y, int rows, int cols) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < rows; ++i) {
        double acc = 0.0;
        const uint16_t* row = w + (size_t)i * cols;
        for (int j = 0; j < cols; ++j) acc += (double)orc_bf16_to_f32(row[j]) * (double)x[j];
        y[i] = (float)acc;
    }
}

/* model.py:244-245 `_smooth_gelu` + the residual of model.py:305, f32:
 *   h = 0.5 * y * (1 + erf(y / sqrt(2)));  x <- x + h. */
void orc_gelu_residual(const float* y, float* x, int d) {
    const float inv_sqrt2 = (float)(1.0 / sqrt(2.0));
    for (int i = 0; i < d; ++i) {
        float h = 0.5f * y[i] * (1.0f + erff(y[i] * inv_sqrt2));
        x[i] = x[i] + h;
    }
}

/* model.py:261-263 `_unembed`: logits = x^T (1 x d) @ unembed (d x V). */
void orc_unembed(const float* unembed, const float* x, float* logits, int d, int vocab) {
#pragma omp parallel for schedule(static)
    for (int v = 0; v < vocab; ++v) {
        double acc = 0.0;
        for (int i = 0; i < d; ++i) acc += (double)x[i] * (double)unembed[(size_t)i * vocab + v];
        logits[v] = (float)acc;
    }
}

/* model.py:396 `np.argmax`: lowest index on ties. */
int orc_argmax(const float* v, int n) {
    int best = 0;
    for (int i = 1; i < n; ++i)
        if (v[i] > v[best]) best = i;
    return best;
}

/* model.py:231-236 `max_backbone_deviation` for one matrix pair (bf16 storage). */
float orc_max_abs_diff_bf16(const uint16_t* a, const uint16_t* b, int64_t n) {
    float worst = 0.0f;
#pragma omp parallel for reduction(max : worst) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        float dlt = fabsf(orc_bf16_to_f32(a[i]) - orc_bf16_to_f32(b[i]));
        if (dlt > worst) worst = dlt;
    }
    return worst;
}

/* Distance in bf16 ulps between two bf16 arrays (finite values): max over elements of
 * |ordinal(a) - ordinal(b)| where ordinal maps the sign-magnitude bit pattern onto a
 * monotone integer line.  Used by the "within 1 bf16 ulp" parity checks. */
int32_t orc_max_ulp_diff_bf16(const uint16_t* a, const uint16_t* b, int64_t n, int64_t* n_diff) {
    int32_t worst = 0;
    int64_t cnt = 0;
#pragma omp parallel for reduction(max : worst) reduction(+ : cnt) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        int32_t x = a[i] & 0x8000 ? -(int32_t)(a[i] & 0x7fff) : (int32_t)(a[i] & 0x7fff);
        int32_t y = b[i] & 0x8000 ? -(int32_t)(b[i] & 0x7fff) : (int32_t)(b[i] & 0x7fff);
        int32_t dlt = x > y ? x - y : y - x;
        if (dlt > worst) worst = dlt;
        if (dlt) cnt += 1;
    }
    if (n_diff) *n_diff = cnt;
    return worst;
}

/* One pass over a merged matrix for the parity report of tests/test_gpu_true_shapes.py (the numpy form of
 * oracle.strict_ulp_report takes seconds per 45M-element matrix; this takes tens of milliseconds):
 *   out[0] = elements that differ, out[1] = elements off by more than one ulp OF THE RESULT,
 *   out[2] = max |got - want| / ulp(max(|want|, |got|))            (the literal criterion)
 *   out[3] = max |got - want| / ulp(max(|want|, |ref_k|...))       (the operand-magnitude criterion)
 *   out[4] = over the strict violators, max |want| / max(|want|, |ref_k| ...)               (how deep they cancelled)
 * ulp(x) = 2^(floor(log2 x) - 7), with the smallest normal's spacing below it. */
static inline double orc_bf16_ulp(double mag) {
    if (mag < 1.1754943508222875e-38) mag = 1.1754943508222875e-38;
    int e;
    frexp(mag, &e);
    return ldexp(1.0, e - 1 - 7);
}
void orc_ulp_report_bf16(const uint16_t* got, const uint16_t* want, const uint16_t* const* refs, int n_refs, int64_t n, double* out) {
    int64_t n_diff = 0, n_viol = 0;
    double max_strict = 0.0, max_relaxed = 0.0, worst_ratio = 0.0;
#pragma omp parallel for reduction(+ : n_diff, n_viol) reduction(max : max_strict, max_relaxed, worst_ratio) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        if (got[i] == want[i]) continue;
        const double g = (double)orc_bf16_to_f32(got[i]), w = (double)orc_bf16_to_f32(want[i]);
        const double diff = fabs(g - w);
        if (diff == 0.0) continue; /* +0 against -0 */
        n_diff += 1;
        const double res = fmax(fabs(g), fabs(w));
        double mag = fabs(w);
        for (int k = 0; k < n_refs; ++k) mag = fmax(mag, fabs((double)orc_bf16_to_f32(refs[k][i])));
        const double strict = diff / orc_bf16_ulp(res), relaxed = diff / orc_bf16_ulp(mag);
        if (strict > max_strict) max_strict = strict;
        if (relaxed > max_relaxed) max_relaxed = relaxed;
        if (strict > 1.0) {
            n_viol += 1;
            const double ratio = mag > 0.0 ? fabs(w) / mag : 1.0;
            if (ratio > worst_ratio) worst_ratio = ratio;
        }
    }
    out[0] = (double)n_diff;
    out[1] = (double)n_viol;
    out[2] = max_strict;
    out[3] = max_relaxed;
    out[4] = worst_ratio;
}
