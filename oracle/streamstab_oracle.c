/*
 * streamstab_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference `streamstab` per-frame consistency step
 * (/root/reference/pkg/src/streamstab/{flow,consistency}.py).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker or the timed CPU baseline.
 * The product path (paper_2301_00750_b200) never links or calls it.
 *
 * Arithmetic follows numpy's float32 evaluation order exactly (compiled with
 * -ffp-contract=off, no -ffast-math): every array expression of the reference
 * is one rounding per elementwise op, left to right.  The only op that is not
 * bit-reproducible is exp (numpy's SIMD expf vs libm expf, <= 2 ulp); the
 * parity pins in tests/ state that tolerance.  Pinned against golden vectors
 * produced by the reference itself (tests/golden/make_golden.py).
 *
 * Layouts match the reference boundary (imgio.py:33-46, :154-192): frames are
 * float32 (H, W, C) interleaved, C in {1, 3}; flows are float32 (H, W, 2)
 * (u horizontal, v vertical) plus a uint8 (H, W) validity map.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_VALUE_ERROR 2
#define ORC_SOLVER_DIVERGENCE 3
#define ORC_NO_MEMORY 5

typedef struct orc_params {
    float k1, k2, alpha, lam, eta, kappa; /* already cast to float32 like np.float32(...) */
    int32_t iterations;
} orc_params;

/* ------------------------------------------------------------------------ */
/* flow.py:83-99  _bilinear_gather, one sample of a (h, w, c) plane stack.   */
/* ys/xs are the float32 sample coordinates before clamping.                 */
static inline void bilinear_sample(const float *planes, int h, int w, int c,
                                   float ys, float xs, float *out)
{
    /* np.clip(ys, 0.0, h - 1.0): float32 min/max (flow.py:89-90) */
    float hy = (float)(h - 1), wx = (float)(w - 1);
    ys = ys < 0.0f ? 0.0f : (ys > hy ? hy : ys);
    xs = xs < 0.0f ? 0.0f : (xs > wx ? wx : xs);
    /* np.clip propagates NaN; floor(NaN) cast to intp is undefined in numpy
     * as well -- flows are finite by construction (FlowField). */
    int y0 = (int)floorf(ys), x0 = (int)floorf(xs);        /* flow.py:91-92 */
    int y1 = y0 + 1 < h - 1 ? y0 + 1 : h - 1;               /* flow.py:93 */
    int x1 = x0 + 1 < w - 1 ? x0 + 1 : w - 1;               /* flow.py:94 */
    /* (ys - y0) is evaluated in float64 then cast (flow.py:95-96); it is
     * exact in float32 because y0 = floor(ys). */
    float fy = (float)((double)ys - (double)y0);
    float fx = (float)((double)xs - (double)x0);
    float gx = 1.0f - fx, gy = 1.0f - fy;
    const float *p00 = planes + ((size_t)y0 * w + x0) * c;
    const float *p01 = planes + ((size_t)y0 * w + x1) * c;
    const float *p10 = planes + ((size_t)y1 * w + x0) * c;
    const float *p11 = planes + ((size_t)y1 * w + x1) * c;
    for (int k = 0; k < c; ++k) {
        float top = p00[k] * gx + p01[k] * fx;   /* flow.py:97 */
        float bot = p10[k] * gx + p11[k] * fx;   /* flow.py:98 */
        out[k] = top * gy + bot * fy;            /* flow.py:99 */
    }
}

/* flow.py:102-127  backward_warp -> (warped, mask).  mask may be NULL. */
void orc_backward_warp(const float *img, int h, int w, int c, const float *uv,
                       const uint8_t *valid, float *out, float *mask)
{
    float hy = (float)(h - 1), wx = (float)(w - 1);
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            size_t i = (size_t)y * w + x;
            float ys = (float)y + uv[2 * i + 1];  /* flow.py:120 */
            float xs = (float)x + uv[2 * i + 0];  /* flow.py:121 */
            if (mask) {
                int inside = ys >= 0.0f && ys <= hy && xs >= 0.0f && xs <= wx; /* :122 */
                mask[i] = (inside && valid[i]) ? 1.0f : 0.0f;                  /* :123 */
            }
            bilinear_sample(img, h, w, c, ys, xs, out + i * c);
        }
    }
}

/* flow.py:130-153  forward-backward occlusion mask.  rint is round-half-even
 * (np.rint) == nearbyintf under the default rounding mode. */
void orc_occlusion_mask(const float *fuv, const uint8_t *fvalid, const float *buv,
                        const uint8_t *bvalid, int h, int w, float *out)
{
    float hy = (float)(h - 1), wx = (float)(w - 1);
    const float c001 = 0.01f, c05 = 0.5f; /* python floats -> float32 (NEP 50) */
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            size_t i = (size_t)y * w + x;
            float f0 = fuv[2 * i], f1 = fuv[2 * i + 1];
            float ys = (float)y + f1, xs = (float)x + f0;                   /* :142-143 */
            int inside = ys >= 0.0f && ys <= hy && xs >= 0.0f && xs <= wx; /* :144 */
            float back[2];
            bilinear_sample(buv, h, w, 2, ys, xs, back);                    /* :145 */
            float ry = nearbyintf(ys), rx = nearbyintf(xs);                 /* :147-148 */
            ry = ry < 0.0f ? 0.0f : (ry > hy ? hy : ry);
            rx = rx < 0.0f ? 0.0f : (rx > wx ? wx : rx);
            int bv = bvalid[(size_t)(int)ry * w + (int)rx];                 /* :146 */
            float s0 = f0 + back[0], s1 = f1 + back[1];
            float lhs = s0 * s0 + s1 * s1;                                  /* :150 */
            float ff = f0 * f0 + f1 * f1;
            float bb = back[0] * back[0] + back[1] * back[1];
            float rhs = c001 * (ff + bb) + c05;                             /* :151 */
            out[i] = (lhs < rhs && inside && fvalid[i] && bv) ? 1.0f : 0.0f; /* :152-153 */
        }
    }
}

/* consistency.py:125-130  sum_c (a - b)^2, channels summed left to right. */
static inline float sq_color_distance(const float *a, const float *b, int c)
{
    float d = a[0] - b[0];
    float s = d * d;
    for (int k = 1; k < c; ++k) {
        d = a[k] - b[k];
        s = s + d * d;
    }
    return s;
}

/* consistency.py:133-154  warp_weight (validity may be NULL). */
void orc_warp_weight(const float *ref, const float *warped, int h, int w, int c,
                     float alpha, float bound, const float *validity, float *out)
{
    float na = -alpha;
#pragma omp parallel for schedule(static)
    for (long i = 0; i < (long)h * w; ++i) {
        float e = expf(na * sq_color_distance(ref + i * c, warped + i * c, c));
        float v = bound < e ? bound : e;                 /* np.minimum(bound, exp) */
        if (validity) v = v * (validity[i] > 0.0f ? 1.0f : 0.0f);
        out[i] = v;
    }
}

/* consistency.py:157-171  (1 - (wp + wn)) * cur + wp * prev + wn * next. */
void orc_local_blend(const float *cur, const float *prev, const float *next,
                     const float *wp, const float *wn, int h, int w, int c, float *out)
{
#pragma omp parallel for schedule(static)
    for (long i = 0; i < (long)h * w; ++i) {
        float a = wp[i], b = wn[i];
        float one_m = 1.0f - (a + b);
        for (int k = 0; k < c; ++k) {
            size_t j = (size_t)i * c + k;
            out[j] = one_m * cur[j] + a * prev[j] + b * next[j];
        }
    }
}

/* consistency.py:190-195  wp * G + (1 - wp) * L. */
void orc_adaptive_blend(const float *g, const float *l, const float *wp, int h, int w,
                        int c, float *out)
{
#pragma omp parallel for schedule(static)
    for (long i = 0; i < (long)h * w; ++i) {
        float a = wp[i], om = 1.0f - a;
        for (int k = 0; k < c; ++k) {
            size_t j = (size_t)i * c + k;
            out[j] = a * g[j] + om * l[j];
        }
    }
}

/* consistency.py:198-208  lam * exp(-alpha * ||cur - blended||^2). */
void orc_consistency_weight(const float *cur, const float *blended, int h, int w, int c,
                            float alpha, float lam, float *out)
{
    float na = -alpha;
#pragma omp parallel for schedule(static)
    for (long i = 0; i < (long)h * w; ++i)
        out[i] = lam * expf(na * sq_color_distance(cur + i * c, blended + i * c, c));
}

/* consistency.py:211-221  _laplacian_into: (((-4c + N) + S) + W) + E with
 * replicate borders (the missing neighbour is the pixel itself). */
static inline float lap_at(const float *img, int h, int w, int c, int y, int x, int k)
{
    size_t row = (size_t)w * c;
    const float *p = img + (size_t)y * row + (size_t)x * c + k;
    float v = p[0] * -4.0f;
    v = v + (y > 0 ? p[-(ptrdiff_t)row] : p[0]);
    v = v + (y < h - 1 ? p[row] : p[0]);
    v = v + (x > 0 ? p[-c] : p[0]);
    v = v + (x < w - 1 ? p[c] : p[0]);
    return v;
}

void orc_laplacian(const float *img, int h, int w, int c, float *out)
{
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            for (int k = 0; k < c; ++k)
                out[((size_t)y * w + x) * c + k] = lap_at(img, h, w, c, y, x, k);
}

/* numpy float32 add.reduce over a contiguous array: pairwise summation with
 * 8-way unrolled leaves of <= 128 elements (numpy umath loops, the routine
 * behind np.sum at consistency.py:292).  Reproduced so that the divergence
 * iteration matches the reference exactly, including float32 overflow of the
 * sum of finite iterates. */
float orc_numpy_pairwise_sum(const float *a, ptrdiff_t n)
{
    if (n < 8) {
        float r = -0.0f;
        for (ptrdiff_t i = 0; i < n; ++i) r += a[i];
        return r;
    } else if (n <= 128) {
        float r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        ptrdiff_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    } else {
        ptrdiff_t n2 = n / 2;
        n2 -= n2 % 8;
        return orc_numpy_pairwise_sum(a, n2) + orc_numpy_pairwise_sum(a + n2, n - n2);
    }
}

/* consistency.py:253-295  solve_screened_poisson (SGD with momentum).
 * Returns ORC_SOLVER_DIVERGENCE with *div_iter = j + 1 (1-based) when the
 * pairwise sum of an updated iterate is non-finite (:292-293). */
int orc_solve_screened_poisson(const float *P, const float *A, const float *wc, int h,
                               int w, int c, const orc_params *prm, const float *init,
                               float *out, int *div_iter)
{
    size_t n = (size_t)h * w * c;
    float *lap_p = (float *)malloc(n * sizeof(float));
    float *cur = (float *)malloc(n * sizeof(float));
    float *prev = (float *)malloc(n * sizeof(float));
    float *upd = (float *)malloc(n * sizeof(float));
    if (!lap_p || !cur || !prev || !upd) {
        free(lap_p); free(cur); free(prev); free(upd);
        return ORC_NO_MEMORY;
    }
    orc_laplacian(P, h, w, c, lap_p);                    /* :269 */
    memcpy(cur, init, n * sizeof(float));                /* :272 */
    memcpy(prev, init, n * sizeof(float));               /* :273 */
    const float eta = prm->eta, kappa = prm->kappa;
    int status = ORC_OK;
    if (div_iter) *div_iter = 0;
    for (int j = 0; j < prm->iterations; ++j) {
#pragma omp parallel for schedule(static)
        for (int y = 0; y < h; ++y) {
            for (int x = 0; x < w; ++x) {
                size_t px = (size_t)y * w + x;
                float wcv = wc[px];
                for (int k = 0; k < c; ++k) {
                    size_t i = px * c + k;
                    float o = cur[i];
                    float g = lap_at(cur, h, w, c, y, x, k);   /* :282 */
                    g = g - lap_p[i];                          /* :283 */
                    float d = o - A[i];                        /* :284 */
                    d = d * wcv;                               /* :285 */
                    g = d - g;                                 /* :286 */
                    g = g * eta;                               /* :287 */
                    float m = o - prev[i];                     /* :288 */
                    m = m * kappa;                             /* :289 */
                    float u = o - g;                           /* :290 */
                    upd[i] = u + m;                            /* :291 */
                }
            }
        }
        if (!isfinite(orc_numpy_pairwise_sum(upd, (ptrdiff_t)n))) {   /* :292 */
            if (div_iter) *div_iter = j + 1;                          /* :293 */
            status = ORC_SOLVER_DIVERGENCE;
            break;
        }
        float *t = prev; prev = cur; cur = upd; upd = t;               /* :294 */
    }
    if (status == ORC_OK) {
        for (size_t i = 0; i < n; ++i) {                               /* :295 */
            float v = cur[i];
            out[i] = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
        }
    }
    free(lap_p); free(cur); free(prev); free(upd);
    return status;
}

/* consistency.py:368-413  _run_step after the two flow_between calls.
 * next_* may be NULL (stream_end_step: w_n = 0, next terms = current frame,
 * :395-398).  A_out / wc_out (optional) receive the solver inputs. */
int orc_run_step(int h, int w, int cin, int cp,
                 const float *I_prev, const float *P_prev,
                 const float *I_cur, const float *P_cur,
                 const float *I_next, const float *P_next,
                 const float *O_prev,
                 const float *fp_uv, const uint8_t *fp_valid,
                 const float *fn_uv, const uint8_t *fn_valid,
                 const orc_params *prm, float *out, float *A_out, float *wc_out,
                 int *div_iter)
{
    size_t np_ = (size_t)h * w;
    int with_next = I_next != NULL;
    float *wIp = malloc(np_ * cin * sizeof(float)), *wPp = malloc(np_ * cp * sizeof(float));
    float *wIn = malloc(np_ * cin * sizeof(float)), *wPn = malloc(np_ * cp * sizeof(float));
    float *mp = malloc(np_ * sizeof(float)), *mn = malloc(np_ * sizeof(float));
    float *wp = malloc(np_ * sizeof(float)), *wn = malloc(np_ * sizeof(float));
    float *L = malloc(np_ * cp * sizeof(float)), *G = malloc(np_ * cp * sizeof(float));
    float *A = malloc(np_ * cp * sizeof(float)), *AI = malloc(np_ * cin * sizeof(float));
    float *wc = malloc(np_ * sizeof(float));
    int status = ORC_NO_MEMORY;
    if (!wIp || !wPp || !wIn || !wPn || !mp || !mn || !wp || !wn || !L || !G || !A || !AI || !wc)
        goto done;
    orc_backward_warp(I_prev, h, w, cin, fp_uv, fp_valid, wIp, mp);           /* :387 */
    orc_backward_warp(P_prev, h, w, cp, fp_uv, fp_valid, wPp, NULL);          /* :388 */
    orc_warp_weight(I_cur, wIp, h, w, cin, prm->alpha, prm->k1, mp, wp);      /* :389 */
    const float *wIn_use, *wPn_use;
    if (with_next) {
        orc_backward_warp(I_next, h, w, cin, fn_uv, fn_valid, wIn, mn);       /* :392 */
        orc_backward_warp(P_next, h, w, cp, fn_uv, fn_valid, wPn, NULL);      /* :393 */
        orc_warp_weight(I_cur, wIn, h, w, cin, prm->alpha, prm->k2, mn, wn);  /* :394 */
        wIn_use = wIn; wPn_use = wPn;
    } else {
        wIn_use = I_cur; wPn_use = P_cur;                                     /* :396-397 */
        memset(wn, 0, np_ * sizeof(float));                                   /* :398 */
    }
    orc_local_blend(P_cur, wPp, wPn_use, wp, wn, h, w, cp, L);               /* :400 */
    orc_backward_warp(O_prev, h, w, cp, fp_uv, fp_valid, G, NULL);           /* :401 */
    orc_adaptive_blend(G, L, wp, h, w, cp, A);                               /* :402 */
    orc_local_blend(I_cur, wIp, wIn_use, wp, wn, h, w, cin, AI);             /* :403 */
    orc_consistency_weight(I_cur, AI, h, w, cin, prm->alpha, prm->lam, wc);   /* :404 */
    if (A_out) memcpy(A_out, A, np_ * cp * sizeof(float));
    if (wc_out) memcpy(wc_out, wc, np_ * sizeof(float));
    status = orc_solve_screened_poisson(P_cur, A, wc, h, w, cp, prm, A, out, div_iter); /* :407 */
done:
    free(wIp); free(wPp); free(wIn); free(wPn); free(mp); free(mn); free(wp); free(wn);
    free(L); free(G); free(A); free(AI); free(wc);
    return status;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
