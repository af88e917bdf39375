// Consistency-step kernels for sm_100a: bilinear backward warp, occlusion mask,
// warp/consistency weights, blends, Laplacian, and the fused pre-solve pass
// (K1) that replaces consistency.py:387-404 with one read of every input
// pixel and one write of every solver input.
//
// Compiled with -fmad=false; all float arithmetic goes through ss::fadd/fsub/
// fmul (round-to-nearest, never contracted), in the reference's op order, so
// warp, masks, blends and the Laplacian are bit-identical to numpy and the
// exp-derived weights differ only by expf ulps.
#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

// ---------------------------------------------------------------------------
// flow.py:102-127 backward_warp
template <int C>
__global__ void __launch_bounds__(256) k_backward_warp(const float *__restrict__ img, int h, int w,
                                                       const float *__restrict__ uv,
                                                       const uint8_t *__restrict__ valid,
                                                       float *__restrict__ out,
                                                       float *__restrict__ mask)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)h * w) return;
    const int y = (int)(i / w), x = (int)(i - (long)y * w);
    const float2 f = __ldg(reinterpret_cast<const float2 *>(uv) + i);
    const float ys = fadd((float)y, f.y), xs = fadd((float)x, f.x);
    if (mask) mask[i] = (inside(ys, xs, h, w) && (valid == nullptr || valid[i])) ? 1.0f : 0.0f;
    float v[C];
    gather<C>(img, make_taps(ys, xs, h, w), v);
#pragma unroll
    for (int k = 0; k < C; ++k) out[i * C + k] = v[k];
}

// flow.py:130-153 occlusion_mask
__global__ void __launch_bounds__(256) k_occlusion(const float *__restrict__ fuv,
                                                   const uint8_t *__restrict__ fvalid,
                                                   const float *__restrict__ buv,
                                                   const uint8_t *__restrict__ bvalid, int h,
                                                   int w, float *__restrict__ out)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)h * w) return;
    const int y = (int)(i / w), x = (int)(i - (long)y * w);
    const float2 f = __ldg(reinterpret_cast<const float2 *>(fuv) + i);
    const float ys = fadd((float)y, f.y), xs = fadd((float)x, f.x);
    const bool in = inside(ys, xs, h, w);
    float b[2];
    gather<2>(buv, make_taps(ys, xs, h, w), b);
    // np.clip(np.rint(ys), 0, h - 1) -> intp; rintf is round-half-even
    const float ry = fminf(fmaxf(rintf(ys), 0.0f), (float)(h - 1));
    const float rx = fminf(fmaxf(rintf(xs), 0.0f), (float)(w - 1));
    const bool bv = bvalid == nullptr || bvalid[(long)(int)ry * w + (int)rx];
    const float s0 = fadd(f.x, b[0]), s1 = fadd(f.y, b[1]);
    const float lhs = fadd(fmul(s0, s0), fmul(s1, s1));
    const float ff = fadd(fmul(f.x, f.x), fmul(f.y, f.y));
    const float bb = fadd(fmul(b[0], b[0]), fmul(b[1], b[1]));
    const float rhs = fadd(fmul(0.01f, fadd(ff, bb)), 0.5f);
    const bool fv = fvalid == nullptr || fvalid[i];
    out[i] = (lhs < rhs && in && fv && bv) ? 1.0f : 0.0f;
}

// consistency.py:133-154 warp_weight
template <int C>
__global__ void k_warp_weight(const float *__restrict__ ref, const float *__restrict__ warped,
                              long n, float alpha, float bound, const float *__restrict__ validity,
                              float *__restrict__ out)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float a[C], b[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        a[k] = ref[i * C + k];
        b[k] = warped[i * C + k];
    }
    float v = fminf(bound, expf(fmul(-alpha, sq_dist<C>(a, b))));
    if (validity) v = fmul(v, validity[i] > 0.0f ? 1.0f : 0.0f);
    out[i] = v;
}

// consistency.py:157-171 local_blend (also input_blend, :174-182)
template <int C>
__global__ void k_local_blend(const float *__restrict__ cur, const float *__restrict__ prev,
                              const float *__restrict__ next, const float *__restrict__ wp,
                              const float *__restrict__ wn, long n, float *__restrict__ out)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float a = wp[i], b = wn[i];
    const float om = fsub(1.0f, fadd(a, b));
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const long j = i * C + k;
        out[j] = fadd(fadd(fmul(om, cur[j]), fmul(a, prev[j])), fmul(b, next[j]));
    }
}

// consistency.py:190-195 adaptive_blend
template <int C>
__global__ void k_adaptive_blend(const float *__restrict__ g, const float *__restrict__ l,
                                 const float *__restrict__ wp, long n, float *__restrict__ out)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float a = wp[i], om = fsub(1.0f, a);
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const long j = i * C + k;
        out[j] = fadd(fmul(a, g[j]), fmul(om, l[j]));
    }
}

// consistency.py:198-208 consistency_weight
template <int C>
__global__ void k_consistency_weight(const float *__restrict__ cur,
                                     const float *__restrict__ blended, long n, float alpha,
                                     float lam, float *__restrict__ out)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float a[C], b[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        a[k] = cur[i * C + k];
        b[k] = blended[i * C + k];
    }
    out[i] = fmul(lam, expf(fmul(-alpha, sq_dist<C>(a, b))));
}

// consistency.py:211-221 Laplacian of an HWC image; writes HWC (planar=false)
// or channel planes (planar=true, the solver layout).
template <int C, bool PLANAR>
__global__ void k_laplacian(const float *__restrict__ img, int h, int w, float *__restrict__ out)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long hw = (long)h * w;
    if (i >= hw) return;
    const int y = (int)(i / w), x = (int)(i - (long)y * w);
    const long up = y > 0 ? i - w : i, dn = y < h - 1 ? i + w : i;
    const long lf = x > 0 ? i - 1 : i, rt = x < w - 1 ? i + 1 : i;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        float v = fmul(__ldg(img + i * C + k), -4.0f);
        v = fadd(v, __ldg(img + up * C + k));
        v = fadd(v, __ldg(img + dn * C + k));
        v = fadd(v, __ldg(img + lf * C + k));
        v = fadd(v, __ldg(img + rt * C + k));
        if (PLANAR)
            out[k * hw + i] = v;
        else
            out[i * C + k] = v;
    }
}

template <int C>
__global__ void k_hwc_to_planar(const float *__restrict__ src, long hw, float *__restrict__ dst)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
#pragma unroll
    for (int k = 0; k < C; ++k) dst[k * hw + i] = src[i * C + k];
}

// ---------------------------------------------------------------------------
// K1: fused pre-solve (consistency.py:387-404 in one pass).
// Per pixel: one flow read per direction, one tap set per direction shared by
// every warped image (I_{t-1}, P_{t-1}, O_{t-1} with f_prev; I_{t+1}, P_{t+1}
// with f_next), the two warp weights, local / adaptive / input blends, the
// consistency weight, and the Laplacian of P_t.  Writes the solver inputs in
// the solver's planar layout: A[c][y][x], lapP[c][y][x], wc[y][x].
// The per-pixel body: Ic / Pc are the pixel's I_t / P_t, fp / fn its flows,
// vp / vn their validity; returns A[CP], w_c and the Laplacian of P_t.
template <int CI, int CP, bool NEXT>
__device__ __forceinline__ void presolve_px(const PresolveArgs &a, long i, int y, int x, const float (&Ic)[CI],
                                            const float (&Pc)[CP], float2 fp, bool vp, float2 fn, bool vn,
                                            float (&Aout)[CP], float &wcv, float (&lap)[CP], float &wp_, float &wn_)
{
    const int h = a.h, w = a.w;
    // both directions' tap sets first, then every gather (prev: I, P, O; next:
    // I, P), then the math -- all the dependent loads are in flight together
    const float ysp = fadd((float)y, fp.y), xsp = fadd((float)x, fp.x);
    const bool mp = inside(ysp, xsp, h, w) && vp;
    const Taps tp = make_taps(ysp, xsp, h, w);
    bool mn = false;
    Taps tn = tp;
    if (NEXT) {
        const float ysn = fadd((float)y, fn.y), xsn = fadd((float)x, fn.x);
        mn = inside(ysn, xsn, h, w) && vn;
        tn = make_taps(ysn, xsn, h, w);
    }
    // ---- previous frame: consistency.py:387-389, :401
    float wIp[CI], wPp[CP], G[CP];
    gather<CI>(a.I_prev, tp, wIp);
    gather<CP>(a.P_prev, tp, wPp);
    gather<CP>(a.O_prev, tp, G);
    // ---- next frame: consistency.py:391-398
    float wIn[CI], wPn[CP], wn;
    if (NEXT) {
        gather<CI>(a.I_next, tn, wIn);
        gather<CP>(a.P_next, tn, wPn);
    }
    const float na = -a.p.alpha;
    float wp = fminf(a.p.k1, expf(fmul(na, sq_dist<CI>(Ic, wIp))));
    wp = fmul(wp, mp ? 1.0f : 0.0f);
    if (NEXT) {
        wn = fminf(a.p.k2, expf(fmul(na, sq_dist<CI>(Ic, wIn))));
        wn = fmul(wn, mn ? 1.0f : 0.0f);
    } else {
#pragma unroll
        for (int k = 0; k < CI; ++k) wIn[k] = Ic[k];
#pragma unroll
        for (int k = 0; k < CP; ++k) wPn[k] = Pc[k];
        wn = 0.0f;
    }

    // ---- blends: consistency.py:400, :402, :403 ; weight :404
    const float om = fsub(1.0f, fadd(wp, wn));
    const float omp = fsub(1.0f, wp);
#pragma unroll
    for (int k = 0; k < CP; ++k) {
        const float L = fadd(fadd(fmul(om, Pc[k]), fmul(wp, wPp[k])), fmul(wn, wPn[k]));
        Aout[k] = fadd(fmul(wp, G[k]), fmul(omp, L));
    }
    float AI[CI];
#pragma unroll
    for (int k = 0; k < CI; ++k)
        AI[k] = fadd(fadd(fmul(om, Ic[k]), fmul(wp, wIp[k])), fmul(wn, wIn[k]));
    wcv = fmul(a.p.lam, expf(fmul(na, sq_dist<CI>(Ic, AI))));

    // ---- Laplacian of P_t (consistency.py:269, :211-221)
    const long up = y > 0 ? i - w : i, dn = y < h - 1 ? i + w : i;
    const long lf = x > 0 ? i - 1 : i, rt = x < w - 1 ? i + 1 : i;
#pragma unroll
    for (int k = 0; k < CP; ++k) {
        float v = fmul(Pc[k], -4.0f);
        v = fadd(v, __ldg(a.P_cur + up * CP + k));
        v = fadd(v, __ldg(a.P_cur + dn * CP + k));
        v = fadd(v, __ldg(a.P_cur + lf * CP + k));
        v = fadd(v, __ldg(a.P_cur + rt * CP + k));
        lap[k] = v;
    }
    wp_ = wp;
    wn_ = wn;
}

template <int CI, int CP, bool NEXT>
__global__ void __launch_bounds__(256) k_presolve(PresolveArgs a)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int h = a.h, w = a.w;
    const long hw = (long)h * w;
    if (i >= hw) return;
    const int y = (int)(i / w), x = (int)(i - (long)y * w);
    float Ic[CI], Pc[CP];
#pragma unroll
    for (int k = 0; k < CI; ++k) Ic[k] = __ldg(a.I_cur + i * CI + k);
#pragma unroll
    for (int k = 0; k < CP; ++k) Pc[k] = __ldg(a.P_cur + i * CP + k);
    const float2 fp = __ldg(reinterpret_cast<const float2 *>(a.uv_prev) + i);
    const float2 fn = NEXT ? __ldg(reinterpret_cast<const float2 *>(a.uv_next) + i) : make_float2(0.f, 0.f);
    const bool vp = a.valid_prev == nullptr || a.valid_prev[i];
    const bool vn = !NEXT || a.valid_next == nullptr || a.valid_next[i];
    float A[CP], wcv, lap[CP], wp, wn;
    presolve_px<CI, CP, NEXT>(a, i, y, x, Ic, Pc, fp, vp, fn, vn, A, wcv, lap, wp, wn);
#pragma unroll
    for (int k = 0; k < CP; ++k) {
        a.A[k * hw + i] = A[k];
        a.lapP[k * hw + i] = lap[k];
    }
    a.wc[i] = wcv;
    if (a.wp_out) a.wp_out[i] = wp;
    if (a.wn_out) a.wn_out[i] = wn;
}

// ---------------------------------------------------------------------------
// host launchers
static const int kThreads = 256;

#define SS_DISPATCH_C(c, F, ...)                   \
    do {                                           \
        if ((c) == 1) {                            \
            F<1> __VA_ARGS__;                      \
        } else if ((c) == 2) {                     \
            F<2> __VA_ARGS__;                      \
        } else if ((c) == 3) {                     \
            F<3> __VA_ARGS__;                      \
        } else {                                   \
            set_error("channel count must be 1 or 3"); \
            return SS_VALUE_ERROR;                 \
        }                                          \
    } while (0)

int launch_backward_warp(const float *img, int h, int w, int c, const float *uv,
                         const uint8_t *valid, float *out, float *mask, cudaStream_t st)
{
    const long n = (long)h * w;
    if (n == 0) return SS_OK;
    SS_DISPATCH_C(c, k_backward_warp, <<<blocks_for(n, kThreads), kThreads, 0, st>>>(
                                          img, h, w, uv, valid, out, mask));
    SS_LAUNCH_CHECK("k_backward_warp");
    return SS_OK;
}

int launch_occlusion(const float *fuv, const uint8_t *fvalid, const float *buv,
                     const uint8_t *bvalid, int h, int w, float *out, cudaStream_t st)
{
    const long n = (long)h * w;
    if (n == 0) return SS_OK;
    k_occlusion<<<blocks_for(n, kThreads), kThreads, 0, st>>>(fuv, fvalid, buv, bvalid, h, w, out);
    SS_LAUNCH_CHECK("k_occlusion");
    return SS_OK;
}

int launch_warp_weight(const float *ref, const float *warped, long n, int c, float alpha,
                       float bound, const float *validity, float *out, cudaStream_t st)
{
    if (n == 0) return SS_OK;
    SS_DISPATCH_C(c, k_warp_weight, <<<blocks_for(n, kThreads), kThreads, 0, st>>>(
                                        ref, warped, n, alpha, bound, validity, out));
    SS_LAUNCH_CHECK("k_warp_weight");
    return SS_OK;
}

int launch_local_blend(const float *cur, const float *prev, const float *next, const float *wp,
                       const float *wn, long n, int c, float *out, cudaStream_t st)
{
    if (n == 0) return SS_OK;
    SS_DISPATCH_C(c, k_local_blend, <<<blocks_for(n, kThreads), kThreads, 0, st>>>(
                                        cur, prev, next, wp, wn, n, out));
    SS_LAUNCH_CHECK("k_local_blend");
    return SS_OK;
}

int launch_adaptive_blend(const float *g, const float *l, const float *wp, long n, int c,
                          float *out, cudaStream_t st)
{
    if (n == 0) return SS_OK;
    SS_DISPATCH_C(c, k_adaptive_blend,
                  <<<blocks_for(n, kThreads), kThreads, 0, st>>>(g, l, wp, n, out));
    SS_LAUNCH_CHECK("k_adaptive_blend");
    return SS_OK;
}

int launch_consistency_weight(const float *cur, const float *blended, long n, int c, float alpha,
                              float lam, float *out, cudaStream_t st)
{
    if (n == 0) return SS_OK;
    SS_DISPATCH_C(c, k_consistency_weight, <<<blocks_for(n, kThreads), kThreads, 0, st>>>(
                                               cur, blended, n, alpha, lam, out));
    SS_LAUNCH_CHECK("k_consistency_weight");
    return SS_OK;
}

int launch_laplacian(const float *img, int h, int w, int c, float *out, bool planar,
                     cudaStream_t st)
{
    const long n = (long)h * w;
    if (n == 0) return SS_OK;
    const unsigned nb = blocks_for(n, kThreads);
    if (c == 1)
        planar ? k_laplacian<1, true><<<nb, kThreads, 0, st>>>(img, h, w, out)
               : k_laplacian<1, false><<<nb, kThreads, 0, st>>>(img, h, w, out);
    else if (c == 3)
        planar ? k_laplacian<3, true><<<nb, kThreads, 0, st>>>(img, h, w, out)
               : k_laplacian<3, false><<<nb, kThreads, 0, st>>>(img, h, w, out);
    else {
        set_error("channel count must be 1 or 3");
        return SS_VALUE_ERROR;
    }
    SS_LAUNCH_CHECK("k_laplacian");
    return SS_OK;
}

int launch_hwc_to_planar(const float *src, int h, int w, int c, float *dst, cudaStream_t st)
{
    const long n = (long)h * w;
    if (n == 0) return SS_OK;
    SS_DISPATCH_C(c, k_hwc_to_planar, <<<blocks_for(n, kThreads), kThreads, 0, st>>>(src, n, dst));
    SS_LAUNCH_CHECK("k_hwc_to_planar");
    return SS_OK;
}

int launch_presolve(const PresolveArgs &a, int ci, int cp, bool with_next, cudaStream_t st)
{
    const long n = (long)a.h * a.w;
    const unsigned nb = blocks_for(n, kThreads);
#define SS_PRESOLVE(CI_, CP_)                                                         \
    if (ci == CI_ && cp == CP_) {                                                     \
        if (with_next)                                                                \
            k_presolve<CI_, CP_, true><<<nb, kThreads, 0, st>>>(a);                   \
        else                                                                          \
            k_presolve<CI_, CP_, false><<<nb, kThreads, 0, st>>>(a);                  \
        SS_LAUNCH_CHECK("k_presolve");                                                \
        return SS_OK;                                                                 \
    }
    SS_PRESOLVE(3, 3)
    SS_PRESOLVE(1, 3)
    SS_PRESOLVE(3, 1)
    SS_PRESOLVE(1, 1)
#undef SS_PRESOLVE
    set_error("channel counts must be 1 or 3");
    return SS_VALUE_ERROR;
}

}  // namespace ss
