// Shared helpers for the streamstab B200 kernels (sm_100a).
//
// Parity rule: every float op of the reference's numpy expression is one
// IEEE-rounded op here, in the same order.  The consistency/solver
// translation units are compiled with -fmad=false and additionally spell the
// ops with __f*_rn intrinsics (which are never contracted into FMA).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/streamstab_b200.h"

namespace ss {

// thread-local last error (ss_last_error)
void set_error(const std::string &msg);
int cuda_status(cudaError_t e, const char *what);

// process-wide count of kernels this library launched (ss_kernel_launches);
// launches recorded into a graph are counted when the graph is launched
void count_launches(long n);
void set_capturing(bool on);  // this thread is capturing a graph

#define SS_CUDA_TRY(expr)                                            \
    do {                                                             \
        cudaError_t _e = (expr);                                     \
        if (_e != cudaSuccess) return ::ss::cuda_status(_e, #expr);  \
    } while (0)

#define SS_LAUNCH_CHECK(what)                                        \
    do {                                                             \
        cudaError_t _e = cudaGetLastError();                         \
        if (_e != cudaSuccess) return ::ss::cuda_status(_e, what);   \
        ::ss::count_launches(1);                                     \
    } while (0)

__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }

// Packed FP32 (sm_100 FADD2 / FMUL2 / FFMA2): two independent IEEE
// round-to-nearest operations per instruction -- bit-identical per lane to the
// scalar __f*_rn forms.
__device__ __forceinline__ uint64_t f2u(float2 a) { return *reinterpret_cast<uint64_t *>(&a); }
__device__ __forceinline__ float2 u2f(uint64_t a) { return *reinterpret_cast<float2 *>(&a); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b)
{
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b)
{
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
// a * b + z with z = (-0, -0) supplied at RUN time: exactly round(a * b)
// (including the sign of zero).  ptxas contracts mul.rn.f32x2 -- and an fma
// with a literal -0 addend -- into a following add/sub as one FFMA2, which
// would skip the product's rounding; an addend it cannot see as zero keeps the
// product a separate instruction, as numpy's is.
__device__ __forceinline__ float2 fmul2(float2 a, float2 b, float2 z)
{
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(z)));
    return u2f(d);
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c)
{
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}

// Bilinear tap set of flow.py:83-99 for one sample position (ys, xs) before
// clamping: clamp to [0, h-1] x [0, w-1], floor, +1 neighbours clamped, and the
// fractional weights (exact in float32, flow.py:95-96).
struct Taps {
    int i00, i01, i10, i11;  // pixel indices
    float fx, fy, gx, gy;    // gx = 1 - fx, gy = 1 - fy
};

__device__ __forceinline__ Taps make_taps(float ys, float xs, int h, int w)
{
    const float hy = (float)(h - 1), wx = (float)(w - 1);
    ys = fminf(fmaxf(ys, 0.0f), hy);
    xs = fminf(fmaxf(xs, 0.0f), wx);
    const float fy0 = floorf(ys), fx0 = floorf(xs);
    const int y0 = (int)fy0, x0 = (int)fx0;
    const int y1 = min(y0 + 1, h - 1), x1 = min(x0 + 1, w - 1);
    Taps t;
    t.fy = fsub(ys, fy0);
    t.fx = fsub(xs, fx0);
    t.gy = fsub(1.0f, t.fy);
    t.gx = fsub(1.0f, t.fx);
    t.i00 = y0 * w + x0;
    t.i01 = y0 * w + x1;
    t.i10 = y1 * w + x0;
    t.i11 = y1 * w + x1;
    return t;
}

// top = p00*gx + p01*fx ; bot = p10*gx + p11*fx ; out = top*gy + bot*fy
__device__ __forceinline__ float bilerp(const Taps &t, float p00, float p01, float p10, float p11)
{
    const float top = fadd(fmul(p00, t.gx), fmul(p01, t.fx));
    const float bot = fadd(fmul(p10, t.gx), fmul(p11, t.fx));
    return fadd(fmul(top, t.gy), fmul(bot, t.fy));
}

template <int C>
__device__ __forceinline__ void gather(const float *__restrict__ img, const Taps &t, float *out)
{
#pragma unroll
    for (int k = 0; k < C; ++k)
        out[k] = bilerp(t, __ldg(img + (size_t)t.i00 * C + k), __ldg(img + (size_t)t.i01 * C + k),
                        __ldg(img + (size_t)t.i10 * C + k), __ldg(img + (size_t)t.i11 * C + k));
}

// inside test of flow.py:122 / :144 (float32 compares against h-1, w-1)
__device__ __forceinline__ bool inside(float ys, float xs, int h, int w)
{
    return ys >= 0.0f && ys <= (float)(h - 1) && xs >= 0.0f && xs <= (float)(w - 1);
}

// consistency.py:125-130: channels summed left to right
template <int C>
__device__ __forceinline__ float sq_dist(const float *a, const float *b)
{
    float d = fsub(a[0], b[0]);
    float s = fmul(d, d);
#pragma unroll
    for (int k = 1; k < C; ++k) {
        d = fsub(a[k], b[k]);
        s = fadd(s, fmul(d, d));
    }
    return s;
}

inline unsigned blocks_for(long n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace ss
