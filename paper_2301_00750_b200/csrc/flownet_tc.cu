// Implicit-GEMM convolution on the 5th-generation tensor cores (tcgen05 +
// TMEM), sm_100a.
//
//   D[m, n] = sum_k A[m, k] * W[k, n]   m = output pixel, n = output channel,
//   k = (ky, kx, cin) (Cin % 8 == 0, so a 16-byte chunk never straddles a tap)
//
// One CTA (4 warps) owns 128 output pixels x all N = pad16(Cout) channels,
// accumulating in TMEM (M = 128 lanes x N fp32 columns).  Each K stage is 128
// bytes of K per row: the 128 threads gather the im2col rows of the stage from
// the fp32 NHWC activations (one row = one pixel per thread), convert, and
// store them in the K-major core-matrix layout (tc_common.cuh); the weight
// stage is pre-arranged in the same layout at upload and arrives by cp.async.
// Thread 0 issues the MMAs; tcgen05.commit frees a stage.  The next stage's
// global loads are in flight while the tensor cores work on the current one.
//
// KIND 0 (bf16 path): kind::f16 with bf16 operands, 4 MMAs (K = 16) per stage.
// KIND 1 (fp32 path): kind::tf32 "3xTF32" -- a = a_hi + a_lo, w = w_hi + w_lo
//   with hi = tf32 truncation, and D += a_hi w_hi + a_hi w_lo + a_lo w_hi, which
//   keeps products to ~2^-21 relative error (fp32-class accuracy) at tensor-core
//   rate; 4 x 3 MMAs (K = 8) per stage.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "flownet.h"
#include "ss_common.cuh"
#include "tc_common.cuh"

namespace ss {
namespace fn {

using namespace tc;

constexpr int TC_THREADS = 128;
constexpr int TC_BM = 128;
constexpr uint32_t TC_TMEM_COLS = 256;
constexpr int A_TILE = TC_BM * 128;  // bytes of one A operand tile per stage

template <int KIND>
struct TcCfg {
    static constexpr int STAGES = KIND == 0 ? 3 : 2;
    static constexpr int CHUNK = KIND == 0 ? 8 : 4;           // K elements per 16 bytes
    static constexpr int BK = 8 * CHUNK;                       // K elements per stage
    static constexpr int A_BYTES = KIND == 0 ? A_TILE : 2 * A_TILE;  // (hi, lo)
    static constexpr int B_COPIES = KIND == 0 ? 1 : 2;
    static size_t smem(int N) { return (size_t)STAGES * (A_BYTES + B_COPIES * N * 128) + 1024 + 64; }
};

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *gmem)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ float lk(float v) { return v >= 0.f ? v : 0.1f * v; }

template <int KIND>
__global__ void __launch_bounds__(TC_THREADS, 1) k_conv_tc(ConvParams p)
{
    using C = TcCfg<KIND>;
    extern __shared__ __align__(1024) uint8_t tc_smem[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tc_smem) + 1023) & ~uintptr_t(1023));
    const int N = p.Cout_pad;
    const int B_BYTES = C::B_COPIES * N * 128;
    const int STAGE_BYTES = C::A_BYTES + B_BYTES;
    uint64_t *done = reinterpret_cast<uint64_t *>(base + C::STAGES * STAGE_BYTES);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + C::STAGES);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int M = p.Ho * p.Wo;
    const int m0 = blockIdx.x * TC_BM;
    const int Ktot = p.k * p.k * p.Cin;
    // split-K: this CTA owns K stages [kb, kb + nk) (blockIdx.y = split)
    const int nk_all = (Ktot + C::BK - 1) / C::BK;
    const int kb = blockIdx.y * p.k_per_split;
    const int nk = min(p.k_per_split, nk_all - kb);

    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&done[s], 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<TC_TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // this thread's im2col row
    const int pix = m0 + tid;
    const bool row_ok = pix < M;
    const int oy = row_ok ? pix / p.Wo : 0, ox = row_ok ? pix - oy * p.Wo : 0;
    // smem byte offset of (row = tid, chunk j): (tid/8)*1024 + j*128 + (tid%8)*16
    const uint32_t row_off = (uint32_t)(tid >> 3) * 1024u + (uint32_t)(tid & 7) * 16u;

    float4 ra[KIND == 0 ? 16 : 8];  // prefetched fp32 activations of one stage

    auto prefetch = [&](int kt) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int k = kt * C::BK + j * C::CHUNK;
            const int tap = k / p.Cin, ci = k - tap * p.Cin;
            const int ky = tap / p.k, kx = tap - ky * p.k;
            const int iy = oy * p.stride + ky * p.dil - p.pad;
            const int ix = ox * p.stride + kx * p.dil - p.pad;
            const bool ok = row_ok && k < Ktot && iy >= 0 && iy < p.H && ix >= 0 && ix < p.W;
            const float4 *src = reinterpret_cast<const float4 *>(
                p.in + ((long)(ok ? iy : 0) * p.W + (ok ? ix : 0)) * p.in_ld + (ok ? ci : 0));
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            if (KIND == 0) {
                ra[2 * j] = ok ? __ldg(src) : z;
                ra[2 * j + 1] = ok ? __ldg(src + 1) : z;
            } else {
                ra[j] = ok ? __ldg(src) : z;
            }
        }
    };

    auto store_a = [&](int s) {
        uint8_t *a = base + s * STAGE_BYTES;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (KIND == 0) {
                const float4 u = ra[2 * j], v = ra[2 * j + 1];
                __nv_bfloat162 b0 = __floats2bfloat162_rn(u.x, u.y), b1 = __floats2bfloat162_rn(u.z, u.w);
                __nv_bfloat162 b2 = __floats2bfloat162_rn(v.x, v.y), b3 = __floats2bfloat162_rn(v.z, v.w);
                uint4 q;
                q.x = *reinterpret_cast<uint32_t *>(&b0);
                q.y = *reinterpret_cast<uint32_t *>(&b1);
                q.z = *reinterpret_cast<uint32_t *>(&b2);
                q.w = *reinterpret_cast<uint32_t *>(&b3);
                *reinterpret_cast<uint4 *>(a + row_off + j * 128) = q;
            } else {
                const float4 u = ra[j];
                float4 hi, lo;
                hi.x = __uint_as_float(__float_as_uint(u.x) & 0xffffe000u);
                hi.y = __uint_as_float(__float_as_uint(u.y) & 0xffffe000u);
                hi.z = __uint_as_float(__float_as_uint(u.z) & 0xffffe000u);
                hi.w = __uint_as_float(__float_as_uint(u.w) & 0xffffe000u);
                lo.x = u.x - hi.x;
                lo.y = u.y - hi.y;
                lo.z = u.z - hi.z;
                lo.w = u.w - hi.w;
                *reinterpret_cast<float4 *>(a + row_off + j * 128) = hi;
                *reinterpret_cast<float4 *>(a + A_TILE + row_off + j * 128) = lo;
            }
        }
    };

    auto issue_b = [&](int kt, int s) {
        const uint8_t *src = reinterpret_cast<const uint8_t *>(p.wtc) + (size_t)kt * B_BYTES;
        const uint32_t dst = smem_u32(base + s * STAGE_BYTES + C::A_BYTES);
        for (int i = tid; i < B_BYTES / 16; i += TC_THREADS) cp_async16(dst + i * 16, src + i * 16);
        cp_commit();
    };

    const uint32_t id = idesc(KIND == 0 ? 1u : 2u, 128u, (uint32_t)N);

    prefetch(kb);
    issue_b(kb, 0);
    for (int kt = 0; kt < nk; ++kt) {  // kt: local stage index, kb + kt: global
        const int s = kt % C::STAGES;
        store_a(s);
        if (kt + 1 < nk) {
            const int s1 = (kt + 1) % C::STAGES;
            if (kt + 1 >= C::STAGES) mbar_wait(&done[s1], ((kt + 1 - C::STAGES) / C::STAGES) & 1);
            prefetch(kb + kt + 1);
            issue_b(kb + kt + 1, s1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t a0 = smem_u32(base + s * STAGE_BYTES);
            const uint32_t b0 = a0 + C::A_BYTES;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t acc = (kt > 0 || i > 0) ? 1u : 0u;
                if (KIND == 0) {
                    mma_bf16(tmem, sdesc(a0 + i * 256, 128, 1024), sdesc(b0 + i * 256, 128, 1024),
                             id, acc);
                } else {
                    const uint32_t alo = a0 + A_TILE, blo = b0 + N * 128;
                    mma_tf32(tmem, sdesc(a0 + i * 256, 128, 1024), sdesc(b0 + i * 256, 128, 1024),
                             id, acc);
                    mma_tf32(tmem, sdesc(a0 + i * 256, 128, 1024), sdesc(blo + i * 256, 128, 1024),
                             id, 1u);
                    mma_tf32(tmem, sdesc(alo + i * 256, 128, 1024), sdesc(b0 + i * 256, 128, 1024),
                             id, 1u);
                }
            }
            mma_commit(&done[s]);
        }
    }
    // all MMAs retired -> TMEM accumulator complete
    mbar_wait(&done[(nk - 1) % C::STAGES], ((nk - 1) / C::STAGES) & 1);
    tc_fence_after();

    const int row = m0 + warp * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tmem_ld16(trow + c0, v);
        if (p.ws) {  // split-K partial sums, reduced by k_splitk_reduce
            if (row < M) {
                float *dst = p.ws + ((size_t)blockIdx.y * M + row) * N + c0;
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    *reinterpret_cast<float4 *>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            }
        } else if (row < M && c0 < p.Cout) {
            float *dst = p.out + (long)row * p.out_ld + c0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                float x = v[i] + (c0 + i < p.Cout ? p.bias[c0 + i] : 0.f);
                v[i] = p.act ? lk(x) : x;
            }
            if (c0 + 16 <= p.Cout) {
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    *reinterpret_cast<float4 *>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (i < p.Cout - c0) dst[i] = v[i];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<TC_TMEM_COLS>(tmem);
}

// out[m, n] = act(sum_s ws[s, m, n] + bias[n])
__global__ void k_splitk_reduce(const float *__restrict__ ws, int splits, int M, int N, int Cout,
                                const float *__restrict__ bias, int act, float *__restrict__ out,
                                int out_ld)
{
    const int n4 = (Cout + 3) / 4;
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)M * n4) return;
    const int m = (int)(i / n4), n = (int)(i - (long)m * n4) * 4;
    float4 acc = *reinterpret_cast<const float4 *>(ws + (size_t)m * N + n);
    for (int s = 1; s < splits; ++s) {
        const float4 v = *reinterpret_cast<const float4 *>(ws + ((size_t)s * M + m) * N + n);
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
        dst[j] = act ? lk(x) : x;
    }
}

static int n_sm_ = 0;

// one-time kernel attributes (outside any stream capture): the largest layer
// has N = 192 output channels
int prepare_conv_tc()
{
    static bool done = false;
    if (done) return SS_OK;
    SS_CUDA_TRY(cudaFuncSetAttribute(k_conv_tc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)TcCfg<0>::smem(256)));
    SS_CUDA_TRY(cudaFuncSetAttribute(k_conv_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)TcCfg<1>::smem(192)));
    int dev = 0;
    SS_CUDA_TRY(cudaGetDevice(&dev));
    SS_CUDA_TRY(cudaDeviceGetAttribute(&n_sm_, cudaDevAttrMultiProcessorCount, dev));
    done = true;
    return SS_OK;
}

template <int KIND>
static int launch_tc(ConvParams p, cudaStream_t st)
{
    using C = TcCfg<KIND>;
    const size_t smem = C::smem(p.Cout_pad);
    if (int rc = prepare_conv_tc()) return rc;
    if ((KIND == 0 && p.Cout_pad > 256) || (KIND == 1 && p.Cout_pad > 192)) {
        set_error("conv_tc: too many output channels");
        return SS_VALUE_ERROR;
    }
    const int n_sm = n_sm_;
    const int M = p.Ho * p.Wo;
    const int ctas = (M + TC_BM - 1) / TC_BM;
    const int nk = (p.k * p.k * p.Cin + C::BK - 1) / C::BK;
    // split K when the pixel tiles alone leave SMs idle and K is long: each
    // split keeps >= 4 stages so the pipeline still overlaps loads and MMAs
    int splits = 1;
    if (p.ws && ctas < n_sm && nk >= 8) {
        splits = std::min((n_sm + ctas - 1) / ctas, nk / 4);
        const size_t need = (size_t)splits * M * p.Cout_pad;
        if (need > p.ws_floats) splits = (int)(p.ws_floats / ((size_t)M * p.Cout_pad));
        splits = std::max(splits, 1);
    }
    p.k_per_split = (nk + splits - 1) / splits;
    splits = (nk + p.k_per_split - 1) / p.k_per_split;
    float *ws = p.ws;
    if (splits == 1) p.ws = nullptr;
    k_conv_tc<KIND><<<dim3(ctas, splits), TC_THREADS, smem, st>>>(p);
    SS_LAUNCH_CHECK("k_conv_tc");
    if (splits > 1) {
        const long n = (long)M * ((p.Cout + 3) / 4);
        k_splitk_reduce<<<blocks_for(n, 256), 256, 0, st>>>(ws, splits, M, p.Cout_pad, p.Cout,
                                                              p.bias, p.act, p.out, p.out_ld);
        SS_LAUNCH_CHECK("k_splitk_reduce");
    }
    return SS_OK;
}

int launch_conv_tc(const ConvParams &p, int kind, cudaStream_t st)
{
    return kind == 0 ? launch_tc<0>(p, st) : launch_tc<1>(p, st);
}

}  // namespace fn
}  // namespace ss
