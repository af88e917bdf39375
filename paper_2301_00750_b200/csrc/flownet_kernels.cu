// Lite flow network kernels (fp32 path), sm_100a.  Architecture:
// paper_2301_00750_b200/liteflownet.py.  NHWC activations, every channel count
// padded to a multiple of 4 (16-byte rows).  This TU uses FMA freely: the
// flow network has no reference bits to reproduce (parity is a tolerance vs.
// the CPU restatement).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <cstring>

#include "flownet.h"
#include "ss_common.cuh"

namespace ss {
namespace fn {

__device__ __forceinline__ float leaky(float v) { return v >= 0.f ? v : 0.1f * v; }

bool pdl_enabled()
{
    static const bool on = getenv("SS_FLOW_PDL") == nullptr || strcmp(getenv("SS_FLOW_PDL"), "0");
    return on;
}

int pdl_status(cudaError_t e, const char *what)
{
    if (e != cudaSuccess) return cuda_status(e, what);
    count_launches(1);
    return SS_OK;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool pred)
{
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int n = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------------------
// depthwise 3x3 (dilated), NHWC, zero padding, no bias / activation.
// A thread owns 4 channels x DW_PX horizontally adjacent pixels: its 9 weight
// float4 stay in registers, and all 9 x DW_PX input loads of a row are issued
// before the FMAs (memory-level parallelism; neighbours hit L1).
#ifndef DW_PX_OVERRIDE
constexpr int DW_PX = 4;
#else
constexpr int DW_PX = DW_PX_OVERRIDE;
#endif

__global__ void __launch_bounds__(256) k_depthwise(const float *__restrict__ in, int ld, int H, int W, int C,
                                                  const float *__restrict__ w, int dil, float *__restrict__ out,
                                                  int ld_out)
{
    pdl_wait();
    const int C4 = C / 4, WG = (W + DW_PX - 1) / DW_PX;
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)H * WG * C4) return;
    const int c = (int)(i % C4) * 4;
    const long g = i / C4;
    const int y = (int)(g / WG), x0 = (int)(g - (long)y * WG) * DW_PX;
    float4 k[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) k[t] = __ldg(reinterpret_cast<const float4 *>(w + t * C + c));
    float4 acc[DW_PX];
#pragma unroll
    for (int p = 0; p < DW_PX; ++p) acc[p] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int ky = 0; ky < 3; ++ky) {
        const int iy = y + (ky - 1) * dil;
        if (iy < 0 || iy >= H) continue;
        const float *row = in + (long)iy * W * ld + c;
        float4 v[3][DW_PX];
#pragma unroll
        for (int kx = 0; kx < 3; ++kx)
#pragma unroll
            for (int p = 0; p < DW_PX; ++p) {
                const int ix = x0 + p + (kx - 1) * dil;
                v[kx][p] = (ix >= 0 && ix < W) ? __ldg(reinterpret_cast<const float4 *>(row + (long)ix * ld))
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
            const float4 kk = k[ky * 3 + kx];
#pragma unroll
            for (int p = 0; p < DW_PX; ++p) {
                acc[p].x = fmaf(v[kx][p].x, kk.x, acc[p].x);
                acc[p].y = fmaf(v[kx][p].y, kk.y, acc[p].y);
                acc[p].z = fmaf(v[kx][p].z, kk.z, acc[p].z);
                acc[p].w = fmaf(v[kx][p].w, kk.w, acc[p].w);
            }
        }
    }
#pragma unroll
    for (int p = 0; p < DW_PX; ++p)
        if (x0 + p < W) *reinterpret_cast<float4 *>(out + ((long)y * W + x0 + p) * ld_out + c) = acc[p];
}

// Tap-sharing variant: a thread owns 4 channels x a 4 x 2 grid of pixels
// spaced by the dilation d (columns x, x+d, x+2d, x+3d; rows y, y+d), so its
// outputs' taps coincide: 6 distinct columns x 4 distinct rows = 24 float4
// loads for 32 outputs (the row-adjacent layout above loads 36 for 16 at
// d >= 4).  Per output the FMA order is the same (ky outer, kx inner).
constexpr int DWS_PX = 4, DWS_PY = 2;
__global__ void __launch_bounds__(256) k_depthwise_s(const float *__restrict__ in, int ld, int H, int W, int C,
                                                    const float *__restrict__ w, int dil, float *__restrict__ out,
                                                    int ld_out)
{
    pdl_wait();
    const int C4 = C / 4;
    // pixel groups: x = bx * 4d + r + k d (r < d, k < 4), y = by * 2d + q + j d (q < d, j < 2)
    const int gx = (W + DWS_PX * dil - 1) / (DWS_PX * dil), gy = (H + DWS_PY * dil - 1) / (DWS_PY * dil);
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long ng = (long)gx * gy * dil * dil;
    if (i >= ng * C4) return;
    const int c = (int)(i % C4) * 4;
    long g = i / C4;
    const int r = (int)(g % dil);
    g /= dil;
    const int q = (int)(g % dil);
    g /= dil;
    const int bx = (int)(g % gx), by = (int)(g / gx);
    const int x0 = bx * DWS_PX * dil + r, y0 = by * DWS_PY * dil + q;
    float4 k[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) k[t] = __ldg(reinterpret_cast<const float4 *>(w + t * C + c));
    float4 acc[DWS_PY][DWS_PX];
#pragma unroll
    for (int j = 0; j < DWS_PY; ++j)
#pragma unroll
        for (int p = 0; p < DWS_PX; ++p) acc[j][p] = make_float4(0.f, 0.f, 0.f, 0.f);
    // input rows y0 + (m - 1) d, m = 0 .. DWS_PY + 1; columns x0 + (n - 1) d, n = 0 .. DWS_PX + 1
#pragma unroll
    for (int m = 0; m < DWS_PY + 2; ++m) {
        const int iy = y0 + (m - 1) * dil;
        float4 v[DWS_PX + 2];
        const bool rok = iy >= 0 && iy < H;
        const float *row = in + (long)(rok ? iy : 0) * W * ld + c;
#pragma unroll
        for (int n = 0; n < DWS_PX + 2; ++n) {
            const int ix = x0 + (n - 1) * dil;
            v[n] = (rok && ix >= 0 && ix < W) ? __ldg(reinterpret_cast<const float4 *>(row + (long)ix * ld))
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        // this input row is tap row ky = m - j for output row j
#pragma unroll
        for (int j = 0; j < DWS_PY; ++j) {
            const int ky = m - j;
            if (ky < 0 || ky > 2) continue;
#pragma unroll
            for (int kx = 0; kx < 3; ++kx) {
                const float4 kk = k[ky * 3 + kx];
#pragma unroll
                for (int p = 0; p < DWS_PX; ++p) {
                    const float4 vv = v[p + kx];
                    acc[j][p].x = fmaf(vv.x, kk.x, acc[j][p].x);
                    acc[j][p].y = fmaf(vv.y, kk.y, acc[j][p].y);
                    acc[j][p].z = fmaf(vv.z, kk.z, acc[j][p].z);
                    acc[j][p].w = fmaf(vv.w, kk.w, acc[j][p].w);
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < DWS_PY; ++j) {
        const int y = y0 + j * dil;
        if (y >= H) continue;
#pragma unroll
        for (int p = 0; p < DWS_PX; ++p) {
            const int x = x0 + p * dil;
            if (x < W) *reinterpret_cast<float4 *>(out + ((long)y * W + x) * ld_out + c) = acc[j][p];
        }
    }
}

int launch_depthwise(const float *in, int ld, int H, int W, int C, const float *w, int dil,
                     float *out, int ld_out, cudaStream_t st)
{
    static const bool shared_taps = getenv("SS_DW") == nullptr || strcmp(getenv("SS_DW"), "rows");
    if (shared_taps) {
        const long gx = (W + DWS_PX * dil - 1) / (DWS_PX * dil), gy = (H + DWS_PY * dil - 1) / (DWS_PY * dil);
        const long n = gx * gy * dil * dil * (C / 4);
        return launch_pdl("k_depthwise_s", k_depthwise_s, dim3(blocks_for(n, 256)), dim3(256), 0, st, in, ld, H, W,
                          C, w, dil, out, ld_out);
    }
    const long n = (long)H * ((W + DW_PX - 1) / DW_PX) * (C / 4);
    return launch_pdl("k_depthwise", k_depthwise, dim3(blocks_for(n, 256)), dim3(256), 0, st, in, ld, H, W, C,
                      w, dil, out, ld_out);
}

// ---------------------------------------------------------------------------
// network input: (h, w, c) HWC in [0,1] -> (H64, W64, 8) NHWC, RGB - 0.5,
// replicate padding, zero channels 3..7; grey input is replicated to RGB
__global__ void k_prep(const float *__restrict__ img, int h, int w, int c, int H, int W,
                       float *__restrict__ out)
{
    pdl_wait();
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)H * W) return;
    const int y = (int)(i / W), x = (int)(i - (long)y * W);
    const long q = (long)min(y, h - 1) * w + min(x, w - 1);
    float r, g, b;
    if (c == 3) {
        r = img[q * 3];
        g = img[q * 3 + 1];
        b = img[q * 3 + 2];
    } else {
        r = g = b = img[q];
    }
    reinterpret_cast<float4 *>(out)[2 * i] = make_float4(r - 0.5f, g - 0.5f, b - 0.5f, 0.f);
    reinterpret_cast<float4 *>(out)[2 * i + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
}

int launch_prep(const float *img, int h, int w, int c, int H, int W, float *out, cudaStream_t st)
{
    return launch_pdl("k_prep", k_prep, dim3(blocks_for((long)H * W, 256)), dim3(256), 0, st, img, h, w, c, H, W,
                      out);
}

// ---------------------------------------------------------------------------
// Network input + first pyramid layer in one pass: pyr1a is a stride-2 3x3
// conv from the 3 live input channels (RGB - 0.5, replicate-padded to the
// 64-multiple size H0 x W0, zero conv padding outside it) to 16 channels +
// LeakyReLU.  One thread per level-1 pixel, fp32 FFMA over its 27 live taps,
// weights (rows of the 8-channel padded table: channels 0..2) in shared
// memory.  Replaces k_prep (an 8-channel padded copy of the frame) and a
// tensor-core launch that padded K from 27 to 72.
__global__ void __launch_bounds__(256) k_prep_pyr1a(const float *__restrict__ img, int h, int w, int c, int H0,
                                                   int W0, int H1, int W1, const float *__restrict__ wgt,
                                                   int cout_pad, const float *__restrict__ bias,
                                                   float *__restrict__ out)
{
    __shared__ __align__(16) float ws[27 * 16];
    __shared__ float bs[16];
    for (int i = threadIdx.x; i < 27 * 16; i += blockDim.x) {
        const int tc = i / 16, co = i - tc * 16, tap = tc / 3, ch = tc - tap * 3;
        ws[i] = wgt[(long)(tap * 8 + ch) * cout_pad + co];
    }
    if (threadIdx.x < 16) bs[threadIdx.x] = bias[threadIdx.x];
    pdl_wait();
    __syncthreads();
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)H1 * W1) return;
    const int oy = (int)(i / W1), ox = (int)(i - (long)oy * W1);
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.f;
#pragma unroll
    for (int ky = 0; ky < 3; ++ky) {
        const int iy = 2 * oy + ky - 1;
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
            const int ix = 2 * ox + kx - 1;
            if (iy < 0 || iy >= H0 || ix < 0 || ix >= W0) continue;  // conv zero padding
            const long q = (long)min(iy, h - 1) * w + min(ix, w - 1);  // replicate padding
            float v[3];
            if (c == 3) {
                v[0] = __ldg(img + q * 3) - 0.5f;
                v[1] = __ldg(img + q * 3 + 1) - 0.5f;
                v[2] = __ldg(img + q * 3 + 2) - 0.5f;
            } else {
                v[0] = v[1] = v[2] = __ldg(img + q) - 0.5f;
            }
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                const float4 *wr = reinterpret_cast<const float4 *>(ws + ((ky * 3 + kx) * 3 + ch) * 16);
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {
                    const float4 u = wr[k4];
                    acc[4 * k4] = fmaf(v[ch], u.x, acc[4 * k4]);
                    acc[4 * k4 + 1] = fmaf(v[ch], u.y, acc[4 * k4 + 1]);
                    acc[4 * k4 + 2] = fmaf(v[ch], u.z, acc[4 * k4 + 2]);
                    acc[4 * k4 + 3] = fmaf(v[ch], u.w, acc[4 * k4 + 3]);
                }
            }
        }
    }
    float4 *dst = reinterpret_cast<float4 *>(out + i * 16);
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4)
        dst[k4] = make_float4(leaky(acc[4 * k4] + bs[4 * k4]), leaky(acc[4 * k4 + 1] + bs[4 * k4 + 1]),
                              leaky(acc[4 * k4 + 2] + bs[4 * k4 + 2]), leaky(acc[4 * k4 + 3] + bs[4 * k4 + 3]));
}

int launch_prep_pyr1a(const float *img, int h, int w, int c, int H0, int W0, int H1, int W1, const float *wgt,
                      int cout_pad, const float *bias, float *out, cudaStream_t st)
{
    return launch_pdl("k_prep_pyr1a", k_prep_pyr1a, dim3(blocks_for((long)H1 * W1, 256)), dim3(256), 0, st, img, h,
                      w, c, H0, W0, H1, W1, wgt, cout_pad, bias, out);
}

// ---------------------------------------------------------------------------
// bilinear (align_corners=False) source coordinate with negative clamp
__device__ __forceinline__ void src_coord(int d, float inv_scale, int n, int &i0, int &i1, float &f)
{
    float s = fmaxf((d + 0.5f) * inv_scale - 0.5f, 0.f);
    i0 = (int)floorf(s);
    if (i0 > n - 1) i0 = n - 1;
    i1 = min(i0 + 1, n - 1);
    f = s - (float)i0;
}

// up = 2 * bilinear_x2(coarse flow) -> x[:, 88:90]; w2 = warp_zero(f2, up).
// One thread per (pixel, 16-channel group): the (cheap) upsampled flow is
// recomputed per group, and the 4 taps x 4 float4 of a group are all loaded
// before the FMAs.
__global__ void k_up2_warp(const float *__restrict__ coarse, int cld, int Hc, int Wc,
                           const float *__restrict__ f2, int C, int H, int W,
                           float *__restrict__ x, int xld, float *__restrict__ w2)
{
    pdl_wait();
    const int G = C / 16;
    const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= (long)H * W * G) return;
    const long i = j / G;
    const int g = (int)(j - i * G);
    const int y = (int)(i / W), xx = (int)(i - (long)y * W);
    int y0, y1, x0, x1;
    float fy, fx;
    src_coord(y, 0.5f, Hc, y0, y1, fy);
    src_coord(xx, 0.5f, Wc, x0, x1, fx);
    float up[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float a = __ldg(coarse + ((long)y0 * Wc + x0) * cld + k), b = __ldg(coarse + ((long)y0 * Wc + x1) * cld + k);
        const float c = __ldg(coarse + ((long)y1 * Wc + x0) * cld + k), d = __ldg(coarse + ((long)y1 * Wc + x1) * cld + k);
        const float top = a * (1.f - fx) + b * fx, bot = c * (1.f - fx) + d * fx;
        up[k] = 2.f * (top * (1.f - fy) + bot * fy);
    }
    if (g == 0) {
        x[i * xld + 88] = up[0];
        x[i * xld + 89] = up[1];
    }
    const float sx = (float)xx + up[0], sy = (float)y + up[1];
    const float gx0 = floorf(sx), gy0 = floorf(sy);
    const int ix = (int)gx0, iy = (int)gy0;
    const float ax = sx - gx0, ay = sy - gy0;
    const float wt[4] = {(1.f - ay) * (1.f - ax), (1.f - ay) * ax, ay * (1.f - ax), ay * ax};
    const int ty[4] = {iy, iy, iy + 1, iy + 1}, tx[4] = {ix, ix + 1, ix, ix + 1};
    float4 v[4][4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const bool ok = ty[t] >= 0 && ty[t] < H && tx[t] >= 0 && tx[t] < W;
        const float4 *src = reinterpret_cast<const float4 *>(f2 + ((long)(ok ? ty[t] : 0) * W + (ok ? tx[t] : 0)) * C + g * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) v[t][q] = ok ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float4 *dst = reinterpret_cast<float4 *>(w2 + i * C + g * 16);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            acc.x = fmaf(wt[t], v[t][q].x, acc.x);
            acc.y = fmaf(wt[t], v[t][q].y, acc.y);
            acc.z = fmaf(wt[t], v[t][q].z, acc.z);
            acc.w = fmaf(wt[t], v[t][q].w, acc.w);
        }
        dst[q] = acc;
    }
}

int launch_up2_warp(const float *coarse, int cld, int Hc, int Wc, const float *f2, int C, int H,
                    int W, float *x, int xld, float *w2, cudaStream_t st)
{
    if (C % 16 != 0) {
        set_error("feature warp needs C % 16 == 0");
        return SS_VALUE_ERROR;
    }
    const long n = (long)H * W * (C / 16);
    return launch_pdl("k_up2_warp", k_up2_warp, dim3(blocks_for(n, 128)), dim3(128), 0, st, coarse, cld, Hc,
                      Wc, f2, C, H, W, x, xld, w2);
}

// ---------------------------------------------------------------------------
// cost volume: x[:, d] = leaky(sum_c f1_c * w2_c(p + d) / C), d in [-4,4]^2;
// also copies f1 into x[:, 96:96+C] (l < 6).
//
// One CTA per (8 x 16 pixel tile, group of 3 dy rows): 64 threads, each owns
// 2 horizontally adjacent pixels x 3 dy x 9 dx = 54 accumulators in
// registers.  Channels stream through shared memory 16 at a time
// (cp.async, double-buffered, zero fill outside the image): the f1 tile and
// the w2 rows y + dy with a +-4 column halo.  Per float4 of channels a thread
// reads its 2 f1 vectors and 3 x 10 w2 vectors and does 216 FMAs.  Rows of
// the staged tiles are padded so the 8 threads of an LDS.128 phase (8
// consecutive tile rows) hit distinct bank groups.
constexpr int CR_TW = 16, CR_TH = 8, CR_CK = 16, CR_HALO = 4;
constexpr int CR_PX = CR_CK + 4;                          // floats per staged pixel
constexpr int CR_WW = CR_TW + 2 * CR_HALO;                // 24 w2 columns
constexpr int CR_WR = CR_TH + 2;                          // w2 rows per dy group (of 3)
constexpr int CR_W2P = CR_WW * CR_PX + 4;                 // w2 row pitch (odd # of 16 B)
constexpr int CR_F1P = CR_TW * CR_PX + 4;                 // f1 row pitch
constexpr int CR_W2F = CR_WR * CR_W2P, CR_F1F = CR_TH * CR_F1P;
#ifndef CR_CS_COARSE
#define CR_CS_COARSE 4
#endif
#ifndef CR_CS_FINE
#define CR_CS_FINE 2
#endif

// DY dy rows per CTA (grid z = 9 / DY): 3 for the fine level, 1 for the
// coarse ones (three times the CTAs where the image alone gives too few)
// CS channel groups of 64 threads: group g takes channels [g * 16 / CS,
// (g + 1) * 16 / CS) of every 16-channel chunk (CS x the warps for the same
// shared memory: the kernel is latency bound at 2 warps per CTA); the groups'
// partial sums are added in group order at the end (deterministic).
template <int DY, int CS>
__global__ void __launch_bounds__(64 * CS) k_corr(const float *__restrict__ f1, const float *__restrict__ w2,
                                                  int C, int H, int W, float *__restrict__ x, int xld,
                                                  int copy_f1)
{
    constexpr int WR = CR_TH + DY - 1;  // w2 rows staged
    constexpr int NT = 64 * CS, CPG = CR_CK / CS;  // threads, channels per group per chunk
    static_assert(CPG % 4 == 0, "channel groups are float4 multiples");
    pdl_wait();
    extern __shared__ __align__(16) float cr_smem[];
    float(*sw)[CR_W2F] = reinterpret_cast<float(*)[CR_W2F]>(cr_smem);
    float(*sf)[CR_F1F] = reinterpret_cast<float(*)[CR_F1F]>(cr_smem + 2 * CR_W2F);
    const int tid = threadIdx.x, grp = tid >> 6;
    const int t = tid & 63;
    const int ty = t & 7, cx = (t >> 3) * 2;  // tile row, first of 2 columns
    const int bx = blockIdx.x * CR_TW, by = blockIdx.y * CR_TH;
    const int dy0 = (int)blockIdx.z * DY - CR_HALO;  // dy rows dy0 .. dy0 + DY - 1

    auto load = [&](int buf, int c0) {
        // w2: WR rows x 24 columns x 4 float4
        for (int i = tid; i < WR * CR_WW * 4; i += NT) {
            const int q = i & 3, px = (i >> 2) % CR_WW, r = (i >> 2) / CR_WW;
            const int gy = by + r + dy0, gx = bx - CR_HALO + px;
            const bool ok = gy >= 0 && gy < H && gx >= 0 && gx < W;
            cp_async16(&sw[buf][r * CR_W2P + px * CR_PX + q * 4],
                       w2 + ((long)(ok ? gy : 0) * W + (ok ? gx : 0)) * C + c0 + q * 4, ok);
        }
        for (int i = tid; i < CR_TH * CR_TW * 4; i += NT) {
            const int q = i & 3, px = (i >> 2) % CR_TW, r = (i >> 2) / CR_TW;
            const int gy = by + r, gx = bx + px;
            const bool ok = gy < H && gx < W;
            cp_async16(&sf[buf][r * CR_F1P + px * CR_PX + q * 4],
                       f1 + ((long)(ok ? gy : 0) * W + (ok ? gx : 0)) * C + c0 + q * 4, ok);
        }
        cp_async_commit();
    };

    float acc[2][DY][9];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int j = 0; j < DY; ++j)
#pragma unroll
            for (int d = 0; d < 9; ++d) acc[p][j][d] = 0.f;

    const int nch = C / CR_CK;
    load(0, 0);
    for (int k = 0; k < nch; ++k) {
        const int buf = k & 1;
        if (k + 1 < nch) {
            load(buf ^ 1, (k + 1) * CR_CK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (copy_f1 && (int)blockIdx.z == 4 / DY) {  // f1 -> x[:, 96 + c], one dy group does it
            for (int i = tid; i < CR_TH * CR_TW * 4; i += NT) {
                const int q = i & 3, px = (i >> 2) % CR_TW, r = (i >> 2) / CR_TW;
                const int gy = by + r, gx = bx + px;
                if (gy < H && gx < W)
                    *reinterpret_cast<float4 *>(x + ((long)gy * W + gx) * xld + 96 + k * CR_CK + q * 4) =
                        *reinterpret_cast<const float4 *>(&sf[buf][r * CR_F1P + px * CR_PX + q * 4]);
            }
        }
        const float *w = &sw[buf][ty * CR_W2P + cx * CR_PX];
        const float *a = &sf[buf][ty * CR_F1P + cx * CR_PX];
#pragma unroll
        for (int c = grp * CPG; c < grp * CPG + CPG; c += 4) {
            const float4 a0 = *reinterpret_cast<const float4 *>(a + c);
            const float4 a1 = *reinterpret_cast<const float4 *>(a + CR_PX + c);
#pragma unroll
            for (int j = 0; j < DY; ++j) {
                float4 b[10];
#pragma unroll
                for (int d = 0; d < 10; ++d) b[d] = *reinterpret_cast<const float4 *>(w + j * CR_W2P + d * CR_PX + c);
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    acc[0][j][d] = fmaf(a0.x, b[d].x, fmaf(a0.y, b[d].y, fmaf(a0.z, b[d].z, fmaf(a0.w, b[d].w, acc[0][j][d]))));
                    acc[1][j][d] = fmaf(a1.x, b[d + 1].x, fmaf(a1.y, b[d + 1].y,
                                        fmaf(a1.z, b[d + 1].z, fmaf(a1.w, b[d + 1].w, acc[1][j][d]))));
                }
            }
        }
        __syncthreads();
    }
    if (CS > 1) {
        // groups 1.. hand their partial sums to group 0 through the (now
        // idle) staging buffers, which group 0 adds in group order
        float *red = cr_smem;
        constexpr int NV = 2 * DY * 9;
        static_assert((CS - 1) * NV * 64 <= 2 * (CR_W2F + CR_F1F), "reduction fits the staging buffers");
        if (grp > 0) {
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int j = 0; j < DY; ++j)
#pragma unroll
                    for (int d = 0; d < 9; ++d) red[((grp - 1) * NV + (p * DY + j) * 9 + d) * 64 + t] = acc[p][j][d];
        }
        __syncthreads();
        if (grp > 0) return;
#pragma unroll
        for (int g = 1; g < CS; ++g)
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int j = 0; j < DY; ++j)
#pragma unroll
                    for (int d = 0; d < 9; ++d) acc[p][j][d] += red[((g - 1) * NV + (p * DY + j) * 9 + d) * 64 + t];
    }
    const float inv = 1.f / (float)C;
    const int y = by + ty;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int xx = bx + cx + p;
        if (y >= H || xx >= W) continue;
        float *dst = x + ((long)y * W + xx) * xld + (dy0 + CR_HALO) * 9;
#pragma unroll
        for (int j = 0; j < DY; ++j)
#pragma unroll
            for (int d = 0; d < 9; ++d) dst[j * 9 + d] = leaky(acc[p][j][d] * inv);
    }
}

// Register-blocked variant (fine levels): a thread owns 8 horizontally adjacent
// pixels of one tile row and one dy, all 9 dx, so per float4 of channels it
// reads its 8 f1 vectors and streams the 16 w2 vectors of the row window once
// (24 LDS.128 for 288 FMAs; the 2-pixel layout above needs 32 for 216).
// Thread t of a channel group: row = t & 7, segment = (t >> 3) & 1, dy = t >> 4
// (8 consecutive threads read 8 rows: distinct bank groups).  Channel groups
// add their partial sums in group order at the end, like k_corr.
template <int DY, int CS>
__global__ void __launch_bounds__(16 * DY * CS) k_corr8(const float *__restrict__ f1, const float *__restrict__ w2,
                                                        int C, int H, int W, float *__restrict__ x, int xld,
                                                        int copy_f1)
{
    constexpr int WR = CR_TH + DY - 1;
    constexpr int NTG = 16 * DY, NT = NTG * CS, CPG = CR_CK / CS;
    static_assert(CPG % 4 == 0, "channel groups are float4 multiples");
    pdl_wait();
    extern __shared__ __align__(16) float cr_smem[];
    float(*sw)[CR_W2F] = reinterpret_cast<float(*)[CR_W2F]>(cr_smem);
    float(*sf)[CR_F1F] = reinterpret_cast<float(*)[CR_F1F]>(cr_smem + 2 * CR_W2F);
    const int tid = threadIdx.x, grp = tid / NTG;
    const int t = tid - grp * NTG;
    const int row = t & 7, seg = (t >> 3) & 1, j = t >> 4;
    const int bx = blockIdx.x * CR_TW, by = blockIdx.y * CR_TH;
    const int dy0 = (int)blockIdx.z * DY - CR_HALO;

    auto load = [&](int buf, int c0) {
        for (int i = tid; i < WR * CR_WW * 4; i += NT) {
            const int q = i & 3, px = (i >> 2) % CR_WW, r = (i >> 2) / CR_WW;
            const int gy = by + r + dy0, gx = bx - CR_HALO + px;
            const bool ok = gy >= 0 && gy < H && gx >= 0 && gx < W;
            cp_async16(&sw[buf][r * CR_W2P + px * CR_PX + q * 4],
                       w2 + ((long)(ok ? gy : 0) * W + (ok ? gx : 0)) * C + c0 + q * 4, ok);
        }
        for (int i = tid; i < CR_TH * CR_TW * 4; i += NT) {
            const int q = i & 3, px = (i >> 2) % CR_TW, r = (i >> 2) / CR_TW;
            const int gy = by + r, gx = bx + px;
            const bool ok = gy < H && gx < W;
            cp_async16(&sf[buf][r * CR_F1P + px * CR_PX + q * 4],
                       f1 + ((long)(ok ? gy : 0) * W + (ok ? gx : 0)) * C + c0 + q * 4, ok);
        }
        cp_async_commit();
    };

    float acc[8][9];
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int d = 0; d < 9; ++d) acc[p][d] = 0.f;

    const int nch = C / CR_CK;
    load(0, 0);
    for (int k = 0; k < nch; ++k) {
        const int buf = k & 1;
        if (k + 1 < nch) {
            load(buf ^ 1, (k + 1) * CR_CK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (copy_f1 && (int)blockIdx.z == 4 / DY) {  // f1 -> x[:, 96 + c], one dy group does it
            for (int i = tid; i < CR_TH * CR_TW * 4; i += NT) {
                const int q = i & 3, px = (i >> 2) % CR_TW, r = (i >> 2) / CR_TW;
                const int gy = by + r, gx = bx + px;
                if (gy < H && gx < W)
                    *reinterpret_cast<float4 *>(x + ((long)gy * W + gx) * xld + 96 + k * CR_CK + q * 4) =
                        *reinterpret_cast<const float4 *>(&sf[buf][r * CR_F1P + px * CR_PX + q * 4]);
            }
        }
        const float *a = &sf[buf][row * CR_F1P + seg * 8 * CR_PX];
        const float *w = &sw[buf][(row + j) * CR_W2P + seg * 8 * CR_PX];
#pragma unroll
        for (int c = grp * CPG; c < grp * CPG + CPG; c += 4) {
            float4 av[8];
#pragma unroll
            for (int p = 0; p < 8; ++p) av[p] = *reinterpret_cast<const float4 *>(a + p * CR_PX + c);
#pragma unroll
            for (int n = 0; n < 16; ++n) {
                const float4 b = *reinterpret_cast<const float4 *>(w + n * CR_PX + c);
#pragma unroll
                for (int p = 0; p < 8; ++p) {
                    const int d = n - p;
                    if (d < 0 || d > 8) continue;
                    acc[p][d] = fmaf(av[p].x, b.x, fmaf(av[p].y, b.y, fmaf(av[p].z, b.z, fmaf(av[p].w, b.w, acc[p][d]))));
                }
            }
        }
        __syncthreads();
    }
    if (CS > 1) {
        float *red = cr_smem;
        constexpr int NV = 72;
        static_assert((CS - 1) * NV * NTG <= 2 * (CR_W2F + CR_F1F), "reduction fits the staging buffers");
        if (grp > 0) {
#pragma unroll
            for (int p = 0; p < 8; ++p)
#pragma unroll
                for (int d = 0; d < 9; ++d) red[((grp - 1) * NV + p * 9 + d) * NTG + t] = acc[p][d];
        }
        __syncthreads();
        if (grp > 0) return;
#pragma unroll
        for (int g = 1; g < CS; ++g)
#pragma unroll
            for (int p = 0; p < 8; ++p)
#pragma unroll
                for (int d = 0; d < 9; ++d) acc[p][d] += red[((g - 1) * NV + p * 9 + d) * NTG + t];
    }
    const float inv = 1.f / (float)C;
    const int y = by + row;
    if (y >= H) return;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        const int xx = bx + seg * 8 + p;
        if (xx >= W) continue;
        float *dst = x + ((long)y * W + xx) * xld + (dy0 + CR_HALO + j) * 9;
#pragma unroll
        for (int d = 0; d < 9; ++d) dst[d] = leaky(acc[p][d] * inv);
    }
}

// one-time kernel attributes (call outside stream capture)
int prepare_flow_kernels()
{
    static bool done = false;
    if (done) return SS_OK;
    SS_CUDA_TRY(cudaFuncSetAttribute(k_corr<3, CR_CS_FINE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(2 * (CR_W2F + CR_F1F) * sizeof(float))));
    SS_CUDA_TRY(cudaFuncSetAttribute(k_corr<1, CR_CS_COARSE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(2 * (CR_W2F + CR_F1F) * sizeof(float))));
    SS_CUDA_TRY(cudaFuncSetAttribute(k_corr8<3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(2 * (CR_W2F + CR_F1F) * sizeof(float))));
    done = true;
    return SS_OK;
}

int launch_corr(const float *f1, const float *w2, int C, int H, int W, float *x, int xld,
                bool copy_f1, cudaStream_t st)
{
    if (C % CR_CK != 0) {
        set_error("correlation needs C % 16 == 0");
        return SS_VALUE_ERROR;
    }
    const size_t smem = 2 * (CR_W2F + CR_F1F) * sizeof(float);  // sized for DY = 3
    if (int rc = prepare_flow_kernels()) return rc;
    const int tiles = ((W + CR_TW - 1) / CR_TW) * ((H + CR_TH - 1) / CR_TH);
    static const int coarse_tiles = getenv("SS_CORR_COARSE_TILES") ? atoi(getenv("SS_CORR_COARSE_TILES")) : 64;
    if (tiles < coarse_tiles) {
        const dim3 grid((W + CR_TW - 1) / CR_TW, (H + CR_TH - 1) / CR_TH, 9);
        return launch_pdl("k_corr", k_corr<1, CR_CS_COARSE>, grid, dim3(64 * CR_CS_COARSE), smem, st, f1, w2, C, H,
                          W, x, xld, copy_f1 ? 1 : 0);
    }
    const dim3 grid((W + CR_TW - 1) / CR_TW, (H + CR_TH - 1) / CR_TH, 3);
    static const bool blocked = getenv("SS_CORR") == nullptr || strcmp(getenv("SS_CORR"), "pairs");
    if (blocked)
        return launch_pdl("k_corr8", k_corr8<3, 4>, grid, dim3(16 * 3 * 4), smem, st, f1, w2, C, H, W, x, xld,
                          copy_f1 ? 1 : 0);
    return launch_pdl("k_corr", k_corr<3, CR_CS_FINE>, grid, dim3(64 * CR_CS_FINE), smem, st, f1, w2, C, H, W, x,
                      xld, copy_f1 ? 1 : 0);
}

// ---------------------------------------------------------------------------
// full-resolution flow: 8 * bilinear_x8(flow3 + r), cropped; writes the
// session's (h, w, 2) flow slot and validity = 1
__global__ void k_flow_final(const float *__restrict__ f3, int ld3, const float *__restrict__ r,
                             int ldr, int Hc, int Wc, int h, int w, float *__restrict__ uv,
                             uint8_t *__restrict__ valid)
{
    pdl_wait();
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)h * w) return;
    const int y = (int)(i / w), x = (int)(i - (long)y * w);
    int y0, y1, x0, x1;
    float fy, fx;
    src_coord(y, 0.125f, Hc, y0, y1, fy);
    src_coord(x, 0.125f, Wc, x0, x1, fx);
    float o[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        auto at = [&](int yy, int xq) {
            const long q = (long)yy * Wc + xq;
            return f3[q * ld3 + k] + r[q * ldr + k];
        };
        const float top = at(y0, x0) * (1.f - fx) + at(y0, x1) * fx;
        const float bot = at(y1, x0) * (1.f - fx) + at(y1, x1) * fx;
        o[k] = 8.f * (top * (1.f - fy) + bot * fy);
    }
    reinterpret_cast<float2 *>(uv)[i] = make_float2(o[0], o[1]);
    if (valid) valid[i] = 1;
}

int launch_flow_final(const float *f3, int ld3, const float *r, int ldr, int Hc, int Wc, int h,
                      int w, float *uv, uint8_t *valid, cudaStream_t st)
{
    return launch_pdl("k_flow_final", k_flow_final, dim3(blocks_for((long)h * w, 256)), dim3(256), 0, st, f3, ld3,
                      r, ldr, Hc, Wc, h, w, uv, valid);
}

// ---------------------------------------------------------------------------
// provider-level downscale (FlowOptions.downscale, flow.py:34, :183-188): the
// network runs on box-downscaled frames and its flow is resized back

// box_downscale (flow.py:69-80) of an HWC frame by f (remainder cropped): per
// channel the f x f block, each row summed left to right, the row sums in
// order, then / f^2
__global__ void k_box_down_hwc(const float *__restrict__ in, int w, int c, int f, int ho, int wo,
                               float *__restrict__ out)
{
    pdl_wait();
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)ho * wo * c) return;
    const int ch = (int)(i % c);
    const long p = i / c;
    const int y = (int)(p / wo), x = (int)(p - (long)y * wo);
    float tot = 0.f;
    for (int dy = 0; dy < f; ++dy) {
        const float *row = in + ((long)(y * f + dy) * w + (long)x * f) * c + ch;
        float r = row[0];
        for (int dx = 1; dx < f; ++dx) r = __fadd_rn(r, row[dx * c]);
        tot = dy == 0 ? r : __fadd_rn(tot, r);
    }
    out[i] = __fdiv_rn(tot, (float)(f * f));
}

int launch_box_down_hwc(const float *in, int w, int c, int f, int ho, int wo, float *out, cudaStream_t st)
{
    return launch_pdl("k_box_down_hwc", k_box_down_hwc, dim3(blocks_for((long)ho * wo * c, 256)), dim3(256), 0, st,
                      in, w, c, f, ho, wo, out);
}

// resize_bilinear (flow.py:54-66: pixel centres, border clamp) of the
// network's (hi, wi, 2) flow to the frame's (ho, wo), times s; valid as a
// FlowField marks it (imgio.py: finite and |u|, |v| <= 1e9)
__global__ void k_upscale_flow(const float *__restrict__ in, int hi, int wi, int ho, int wo, float ry, float rx,
                               float s, float *__restrict__ uv, uint8_t *__restrict__ valid)
{
    pdl_wait();
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)ho * wo) return;
    const int y = (int)(i / wo), x = (int)(i - (long)y * wo);
    const float ys = fminf(fmaxf(((float)y + 0.5f) * ry - 0.5f, 0.f), (float)(hi - 1));
    const float xs = fminf(fmaxf(((float)x + 0.5f) * rx - 0.5f, 0.f), (float)(wi - 1));
    const int y0 = (int)floorf(ys), x0 = (int)floorf(xs);
    const int y1 = min(y0 + 1, hi - 1), x1 = min(x0 + 1, wi - 1);
    const float fy = ys - (float)y0, fx = xs - (float)x0;
    const float2 *f2 = reinterpret_cast<const float2 *>(in);
    const float2 a = f2[(long)y0 * wi + x0], b = f2[(long)y0 * wi + x1];
    const float2 c = f2[(long)y1 * wi + x0], d = f2[(long)y1 * wi + x1];
    const float u = ((a.x * (1.f - fx) + b.x * fx) * (1.f - fy) + (c.x * (1.f - fx) + d.x * fx) * fy) * s;
    const float v = ((a.y * (1.f - fx) + b.y * fx) * (1.f - fy) + (c.y * (1.f - fx) + d.y * fx) * fy) * s;
    reinterpret_cast<float2 *>(uv)[i] = make_float2(u, v);
    if (valid) valid[i] = fabsf(u) <= 1e9f && fabsf(v) <= 1e9f;
}

int launch_upscale_flow(const float *in, int hi, int wi, int ho, int wo, float s, float *uv, uint8_t *valid,
                        cudaStream_t st)
{
    return launch_pdl("k_upscale_flow", k_upscale_flow, dim3(blocks_for((long)ho * wo, 256)), dim3(256), 0, st, in,
                      hi, wi, ho, wo, (float)hi / (float)ho, (float)wi / (float)wo, s, uv, valid);
}

// ---------------------------------------------------------------------------
// split-K reduction of the conv kernels' partial sums (flownet_tma.cu)

// out[m, n] = act(sum_s ws[s, m, n] + bias[n])
// ws: [part][split][M][N]; output channel c of part c / N (N % 4 == 0, so a
// float4 group never straddles parts)
__global__ void k_splitk_reduce(const float *__restrict__ ws, int splits, int M, int N, int Cout,
                                const float *__restrict__ bias, int act, float *__restrict__ out,
                                int out_ld)
{
    pdl_wait();
    const int n4 = (Cout + 3) / 4;
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)M * n4) return;
    const int m = (int)(i / n4), n = (int)(i - (long)m * n4) * 4;
    const int part = n / N, nn = n - part * N;
    // partials are added in split order; their loads are issued eight at a
    // time (a serial load -> add chain would pay one L2 round trip per split)
    const float *src = ws + ((size_t)part * splits * M + m) * N + nn;
    const size_t stride = (size_t)M * N;
    float4 acc = *reinterpret_cast<const float4 *>(src);
    int s = 1;
    for (; s + 8 <= splits; s += 8) {
        float4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __ldcg(reinterpret_cast<const float4 *>(src + (s + j) * stride));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acc.x += v[j].x;
            acc.y += v[j].y;
            acc.z += v[j].z;
            acc.w += v[j].w;
        }
    }
    for (; s < splits; ++s) {
        const float4 v = __ldcg(reinterpret_cast<const float4 *>(src + s * stride));
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
    }
    float r[4] = {acc.x, acc.y, acc.z, acc.w};
    float *dst = out + (long)m * out_ld + n;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (n + j >= Cout) break;
        const float x = r[j] + bias[n + j];
        dst[j] = act ? leaky(x) : x;
    }
}

int launch_splitk_reduce(const float *ws, int splits, int M, int N, int Cout, const float *bias,
                         int act, float *out, int out_ld, cudaStream_t st, int parts)
{
    if (parts > 1 && N % 4 != 0) {
        set_error("split-K reduce: part width must be a multiple of 4");
        return SS_VALUE_ERROR;
    }
    const long n = (long)M * ((Cout + 3) / 4);
    return launch_pdl("k_splitk_reduce", k_splitk_reduce, dim3(blocks_for(n, 128)), dim3(128), 0, st, ws, splits,
                      M, N, Cout, bias, act, out, out_ld);
}

}  // namespace fn
}  // namespace ss
