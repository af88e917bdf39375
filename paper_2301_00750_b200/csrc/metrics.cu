// Evaluation metrics on B200: temporal warping error
// E_warp (metrics.py:107-128) and single-scale SSIM (metrics.py:75-104).
//
// E_warp fuses occlusion_mask (bit-exact, flow.py:130-153), backward_warp and
// its mask (flow.py:102-127) and the masked per-pixel channel-mean L1 into one
// pass; the two sums are accumulated in float64 like the reference
// (mask.sum(dtype=float64), (mask * per_pixel).sum(dtype=float64)).
// SSIM runs in float64 (the reference casts luma to float64): 11-tap Gaussian
// (sigma 1.5) separable blur with scipy "reflect" borders, SSIM map, mean over
// the valid-window crop.
#include <algorithm>
#include <cmath>

#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

__device__ __forceinline__ double block_sum(double v, double *sh)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    v = 0.0;
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    __syncthreads();
    return v;
}

template <int C>
__global__ void __launch_bounds__(256) k_warping_error(const float *__restrict__ fa,
                                                       const float *__restrict__ fb, int h, int w,
                                                       const float *__restrict__ fuv,
                                                       const uint8_t *__restrict__ fvalid,
                                                       const float *__restrict__ buv,
                                                       const uint8_t *__restrict__ bvalid,
                                                       double *__restrict__ sums)
{
    __shared__ double sh[32];
    double num = 0.0, den = 0.0;
    const long n = (long)h * w;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x) {
        const int y = (int)(i / w), x = (int)(i - (long)y * w);
        const float2 f = __ldg(reinterpret_cast<const float2 *>(fuv) + i);
        const float ys = fadd((float)y, f.y), xs = fadd((float)x, f.x);
        const bool in = inside(ys, xs, h, w);
        const Taps t = make_taps(ys, xs, h, w);
        // occlusion_mask(forward, backward) (flow.py:130-153)
        float b[2];
        gather<2>(buv, t, b);
        const float ry = fminf(fmaxf(rintf(ys), 0.0f), (float)(h - 1));
        const float rx = fminf(fmaxf(rintf(xs), 0.0f), (float)(w - 1));
        const bool bv = bvalid[(long)(int)ry * w + (int)rx];
        const float s0 = fadd(f.x, b[0]), s1 = fadd(f.y, b[1]);
        const float lhs = fadd(fmul(s0, s0), fmul(s1, s1));
        const float ff = fadd(fmul(f.x, f.x), fmul(f.y, f.y));
        const float bb = fadd(fmul(b[0], b[0]), fmul(b[1], b[1]));
        const float rhs = fadd(fmul(0.01f, fadd(ff, bb)), 0.5f);
        const bool fv = fvalid[i];
        const float occ = (lhs < rhs && in && fv && bv) ? 1.0f : 0.0f;
        // backward_warp(frame_b, forward) and its mask (same sample position)
        const float wmask = (in && fv) ? 1.0f : 0.0f;
        const float m = fmul(occ, wmask);
        float wb[C];
        gather<C>(fb, t, wb);
        // |a - warped| mean over channels: ((d0 + d1) + d2) / 3 in float32
        float s = fabsf(fsub(fa[i * C], wb[0]));
#pragma unroll
        for (int k = 1; k < C; ++k) s = fadd(s, fabsf(fsub(fa[i * C + k], wb[k])));
        const float per_pixel = C == 1 ? s : __fdiv_rn(s, (float)C);
        num += (double)fmul(m, per_pixel);
        den += (double)m;
    }
    num = block_sum(num, sh);
    den = block_sum(den, sh);
    if (threadIdx.x == 0) {
        atomicAdd(&sums[0], num);
        atomicAdd(&sums[1], den);
    }
}

int launch_warping_error(const float *fa, const float *fb, int h, int w, int c, const float *fuv,
                         const uint8_t *fvalid, const float *buv, const uint8_t *bvalid,
                         double *sums, cudaStream_t st)
{
    const long n = (long)h * w;
    const unsigned nb = (unsigned)std::min<long>(blocks_for(n, 256), 148L * 8);
    SS_CUDA_TRY(cudaMemsetAsync(sums, 0, 2 * sizeof(double), st));
    if (c == 3)
        k_warping_error<3><<<nb, 256, 0, st>>>(fa, fb, h, w, fuv, fvalid, buv, bvalid, sums);
    else if (c == 1)
        k_warping_error<1><<<nb, 256, 0, st>>>(fa, fb, h, w, fuv, fvalid, buv, bvalid, sums);
    else {
        set_error("frame must be (H, W, 1|3)");
        return SS_VALUE_ERROR;
    }
    SS_LAUNCH_CHECK("k_warping_error");
    return SS_OK;
}

// ---------------------------------------------------------------------------
// SSIM
__constant__ double c_gauss[11];

__device__ __forceinline__ int reflect(int i, int n)
{
    // scipy.ndimage "reflect": (d c b a | a b c d | d c b a)
    while (i < 0 || i >= n) i = i < 0 ? -i - 1 : 2 * n - i - 1;
    return i;
}

// luma = frame.astype(float32) @ LUMA_WEIGHTS (flow.py:45-51), which numpy
// hands to BLAS sgemv: fma(b, wb, fma(g, wg, r * wr)) in float32 (see dis.cu),
// then widened to float64 like ssim() does
template <int C>
__global__ void k_luma64(const float *__restrict__ img, long n, double *__restrict__ out)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (C == 1) {
        out[i] = (double)img[i];
    } else {
        const float l = __fmaf_rn(img[i * 3 + 2], 0.114f,
                                  __fmaf_rn(img[i * 3 + 1], 0.587f, __fmul_rn(img[i * 3], 0.299f)));
        out[i] = (double)l;
    }
}

// horizontal pass of the five moments x, y, x^2, y^2, xy
__global__ void k_ssim_h(const double *__restrict__ x, const double *__restrict__ y, int h, int w,
                         double *__restrict__ mom)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long n = (long)h * w;
    if (i >= n) return;
    const int r = (int)(i / w), c = (int)(i - (long)r * w);
    double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 11; ++j) {
        const long q = (long)r * w + reflect(c + j - 5, w);
        const double a = x[q], b = y[q], g = c_gauss[j];
        m[0] += g * a;
        m[1] += g * b;
        m[2] += g * (a * a);
        m[3] += g * (b * b);
        m[4] += g * (a * b);
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) mom[k * n + i] = m[k];
}

// vertical pass + SSIM map + sum over the cropped window
__global__ void k_ssim_v(const double *__restrict__ mom, int h, int w, double *__restrict__ sum)
{
    __shared__ double sh[32];
    const long n = (long)h * w;
    const int pad = 5;
    const long cw = w - 2 * pad, ch = h - 2 * pad;
    double acc = 0.0;
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < cw * ch;
         t += (long)gridDim.x * blockDim.x) {
        const int r = pad + (int)(t / cw), c = pad + (int)(t - (t / cw) * cw);
        double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 11; ++j) {
            const long q = (long)reflect(r + j - 5, h) * w + c;
            const double g = c_gauss[j];
#pragma unroll
            for (int k = 0; k < 5; ++k) m[k] += g * mom[k * n + q];
        }
        const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
        const double mx = m[0], my = m[1];
        const double sx = m[2] - mx * mx, sy = m[3] - my * my, sxy = m[4] - mx * my;
        acc += ((2 * mx * my + C1) * (2 * sxy + C2)) / ((mx * mx + my * my + C1) * (sx + sy + C2));
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) atomicAdd(sum, acc);
}

int launch_ssim(const float *a, const float *b, int h, int w, int c, double *scratch,
                double *sum, cudaStream_t st)
{
    static bool init = false;
    if (!init) {
        double g[11], s = 0.0;
        for (int j = 0; j < 11; ++j) {
            const double x = j - 5.0;
            g[j] = std::exp(-(x * x) / (2.0 * 1.5 * 1.5));
            s += g[j];
        }
        for (double &v : g) v /= s;
        SS_CUDA_TRY(cudaMemcpyToSymbol(c_gauss, g, sizeof g));
        init = true;
    }
    const long n = (long)h * w;
    double *x = scratch, *y = scratch + n, *mom = scratch + 2 * n;
    if (c == 3) {
        k_luma64<3><<<blocks_for(n, 256), 256, 0, st>>>(a, n, x);
        k_luma64<3><<<blocks_for(n, 256), 256, 0, st>>>(b, n, y);
    } else {
        k_luma64<1><<<blocks_for(n, 256), 256, 0, st>>>(a, n, x);
        k_luma64<1><<<blocks_for(n, 256), 256, 0, st>>>(b, n, y);
    }
    k_ssim_h<<<blocks_for(n, 256), 256, 0, st>>>(x, y, h, w, mom);
    SS_CUDA_TRY(cudaMemsetAsync(sum, 0, sizeof(double), st));
    const long m = (long)(h - 10) * (w - 10);
    const unsigned nb = (unsigned)std::min<long>(blocks_for(m, 256), 148L * 8);
    k_ssim_v<<<nb, 256, 0, st>>>(mom, h, w, sum);
    SS_LAUNCH_CHECK("ssim");
    return SS_OK;
}

}  // namespace ss
