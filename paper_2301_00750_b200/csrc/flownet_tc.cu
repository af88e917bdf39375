// Implicit-GEMM convolution on the 5th-generation tensor cores (tcgen05 +
// TMEM), sm_100a.
//
//   D[m, n] = sum_k A[m, k] * W[k, n]   m = output pixel, n = output channel,
//   k = (ky, kx, cin) (Cin % 8 == 0, so a 16-byte chunk never straddles a tap)
//
// One CTA (8 warps) owns 128 output pixels x all N = pad16(Cout) channels,
// accumulating in TMEM (M = 128 lanes x N fp32 columns).  Each K stage is 128
// bytes of K per row.  Two threads share an im2col row (four 16-byte chunks
// each): they gather the chunks from the fp32 NHWC activations two stages
// ahead in registers, convert, and store them in the K-major core-matrix
// layout (tc_common.cuh); the weight stage is pre-arranged in the same layout
// at upload and arrives by cp.async two stages ahead.  Thread 0 issues the
// MMAs; tcgen05.commit frees a stage.  The epilogue reads TMEM with
// tcgen05.ld (warp w: lanes 32*(w%4).., column half w/4), adds bias and
// LeakyReLU and stores fp32 NHWC (or split-K partials).
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

constexpr int TC_THREADS = 256;
constexpr int TC_BM = 128;
constexpr int A_TILE = TC_BM * 128;  // bytes of one A operand tile per stage

template <int KIND>
struct TcCfg {
    static constexpr int STAGES = 3;
    static constexpr int CHUNK = KIND == 0 ? 8 : 4;                  // K elements per 16 bytes
    static constexpr int BK = 8 * CHUNK;                              // K elements per stage
    static constexpr int A_BYTES = KIND == 0 ? A_TILE : 2 * A_TILE;  // (hi, lo)
    static constexpr int B_COPIES = KIND == 0 ? 1 : 2;
    static constexpr int RA = KIND == 0 ? 8 : 4;                      // float4 per thread per stage
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
    pdl_wait();
    using C = TcCfg<KIND>;
    constexpr int S = C::STAGES;
    extern __shared__ __align__(1024) uint8_t tc_smem[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tc_smem) + 1023) & ~uintptr_t(1023));
    const int N = p.Cout_pad;
    const int B_BYTES = C::B_COPIES * N * 128;
    const int STAGE_BYTES = C::A_BYTES + B_BYTES;
    uint64_t *done = reinterpret_cast<uint64_t *>(base + S * STAGE_BYTES);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + S);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int M = p.Ho * p.Wo;
    const int n_tiles = (M + TC_BM - 1) / TC_BM;  // persistent over M tiles
    const int Ktot = p.k * p.k * p.Cin;
    // split-K: this CTA owns K stages [kb, kb + nk) (blockIdx.y = split)
    const int nk_all = (Ktot + C::BK - 1) / C::BK;
    const int kb = blockIdx.y * p.k_per_split;
    const int nk = min(p.k_per_split, nk_all - kb);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&done[s], 1);
        fence_barrier_init();
    }
    const uint32_t tcols = N <= 32 ? 32u : (N <= 64 ? 64u : (N <= 128 ? 128u : 256u));
    if (warp == 0) tmem_alloc_rt(tmem_slot, tcols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // this thread's im2col half-row: row r, chunks [4h, 4h + 4)
    const int r = tid & 127, hh = tid >> 7;
    bool row_ok = false;
    int oy = 0, ox = 0;
    // smem byte offset of (row r, chunk j): (r/8)*1024 + j*128 + (r%8)*16
    const uint32_t row_off = (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 16u;

    float4 ra[2][C::RA];  // two stages of prefetched fp32 activations

    auto prefetch = [&](int kt, float4(&dst)[C::RA]) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int k = kt * C::BK + (hh * 4 + jj) * C::CHUNK;
            const int tap = k / p.Cin, ci = k - tap * p.Cin;
            const int ky = tap / p.k, kx = tap - ky * p.k;
            const int iy = oy * p.stride + ky * p.dil - p.pad;
            const int ix = ox * p.stride + kx * p.dil - p.pad;
            const bool ok = row_ok && k < Ktot && iy >= 0 && iy < p.H && ix >= 0 && ix < p.W;
            const float4 *src = reinterpret_cast<const float4 *>(
                p.in + ((long)(ok ? iy : 0) * p.W + (ok ? ix : 0)) * p.in_ld + (ok ? ci : 0));
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            if (KIND == 0) {
                dst[2 * jj] = ok ? __ldg(src) : z;
                dst[2 * jj + 1] = ok ? __ldg(src + 1) : z;
            } else {
                dst[jj] = ok ? __ldg(src) : z;
            }
        }
    };

    auto store_a = [&](int s, const float4(&src)[C::RA]) {
        uint8_t *a = base + s * STAGE_BYTES;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int j = hh * 4 + jj;
            if (KIND == 0) {
                const float4 u = src[2 * jj], v = src[2 * jj + 1];
                __nv_bfloat162 b0 = __floats2bfloat162_rn(u.x, u.y), b1 = __floats2bfloat162_rn(u.z, u.w);
                __nv_bfloat162 b2 = __floats2bfloat162_rn(v.x, v.y), b3 = __floats2bfloat162_rn(v.z, v.w);
                uint4 q;
                q.x = *reinterpret_cast<uint32_t *>(&b0);
                q.y = *reinterpret_cast<uint32_t *>(&b1);
                q.z = *reinterpret_cast<uint32_t *>(&b2);
                q.w = *reinterpret_cast<uint32_t *>(&b3);
                *reinterpret_cast<uint4 *>(a + row_off + j * 128) = q;
            } else {
                const float4 u = src[jj];
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

    // weight stage kt: copy c (hi / lo) rows [n_off, n_off + N) of the layer's
    // n_full-row stage block
    auto issue_b = [&](int kt, int s) {
        const uint8_t *stage = reinterpret_cast<const uint8_t *>(p.wtc) +
                               (size_t)kt * C::B_COPIES * p.n_full * 128 + (size_t)p.n_off * 128;
        const uint32_t dst = smem_u32(base + s * STAGE_BYTES + C::A_BYTES);
        const int per_copy = N * 128 / 16;
        for (int i = tid; i < C::B_COPIES * per_copy; i += TC_THREADS) {
            const int c = i / per_copy, o = i - c * per_copy;
            cp_async16(dst + c * N * 128 + o * 16, stage + (size_t)c * p.n_full * 128 + o * 16);
        }
        cp_commit();
    };

    const uint32_t id = idesc(KIND == 0 ? 1u : 2u, 128u, (uint32_t)N);

    // stage bookkeeping runs across tiles: the g-th stage this CTA issues uses
    // slot g % S and completes done[g % S] with parity (g / S) & 1
    uint32_t gbase = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int m0 = tile * TC_BM;
    {
        const int pix = m0 + r;
        row_ok = pix < M;
        oy = row_ok ? pix / p.Wo : 0;
        ox = row_ok ? pix - oy * p.Wo : 0;
    }
    // prologue: A for stages 0, 1 in registers; B for stages 0, 1 in flight
    // (every slot is free: the previous tile's MMAs all retired)
    prefetch(kb, ra[0]);
    issue_b(kb, gbase % S);
    if (nk > 1) {
        prefetch(kb + 1, ra[1]);
        issue_b(kb + 1, (gbase + 1) % S);
    }
    for (int kt = 0; kt < nk; ++kt) {  // kt: local stage index, kb + kt: global K stage
        const int s = (gbase + kt) % S;
        // slot s was freed before B(kt) was issued into it
        if (kt & 1)
            store_a(s, ra[1]);
        else
            store_a(s, ra[0]);
        if (kt + 2 < nk) {
            if (kt & 1)
                prefetch(kb + kt + 2, ra[1]);
            else
                prefetch(kb + kt + 2, ra[0]);
            const int s2 = (gbase + kt + 2) % S;
            // slot s2 was last read by the MMAs of stage kt - 1 (of this tile)
            if (kt >= 1) mbar_wait(&done[s2], ((gbase + kt - 1) / S) & 1);
            issue_b(kb + kt + 2, s2);
            cp_wait<2>();  // B(kt) landed; B(kt+1), B(kt+2) may be in flight
        } else if (kt + 1 < nk) {
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
    mbar_wait(&done[(gbase + nk - 1) % S], ((gbase + nk - 1) / S) & 1);
    tc_fence_after();

    // epilogue: warp w reads TMEM lanes 32*(w%4).. (its lane quarter), columns
    // [w/4 * N/2, (w/4 + 1) * N/2) in 16-column groups (N = 16: warps 0-3 only)
    const int q = warp & 3, half = warp >> 2;
    const int row = m0 + q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int groups = N / 16;
    const int g0 = groups == 1 ? (half == 0 ? 0 : 1) : half * (groups / 2);
    const int g1 = groups == 1 ? (half == 0 ? 1 : 1) : (half == 0 ? groups / 2 : groups);
    for (int g = g0; g < g1; ++g) {
        const int c0 = g * 16;
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
    // TMEM reads done before the next tile's first MMA overwrites the accumulator
    tc_fence_before();
    __syncthreads();
    gbase += nk;
    }  // tile loop
    if (warp == 0) tmem_dealloc_rt(tmem, tcols);
}

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
        dst[j] = act ? lk(x) : x;
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
                                     (int)TcCfg<1>::smem(128)));
    int dev = 0;
    SS_CUDA_TRY(cudaGetDevice(&dev));
    SS_CUDA_TRY(cudaDeviceGetAttribute(&n_sm_, cudaDevAttrMultiProcessorCount, dev));
    done = true;
    return SS_OK;
}

template <int KIND>
static int launch_tc_part(ConvParams p, cudaStream_t st);

// N-split: 3 stages of (A, B) must fit in shared memory; 3xTF32 stages carry
// two copies of each operand, so layers wider than 128 channels run as
// several N parts over the same A (the im2col gather is repeated per part)
template <int KIND>
static int launch_tc(ConvParams p, cudaStream_t st)
{
    if (int rc = prepare_conv_tc()) return rc;
    const int nmax = KIND == 0 ? 256 : 128;
    const int parts = (p.Cout_pad + nmax - 1) / nmax;
    const int np = (p.Cout_pad / parts + 15) / 16 * 16;
    p.n_full = p.Cout_pad;
    const int cout = p.Cout;
    const float *bias = p.bias;
    float *out = p.out;
    for (int n0 = 0; n0 < p.n_full; n0 += np) {
        ConvParams q = p;
        q.n_off = n0;
        q.Cout_pad = std::min(np, p.n_full - n0);
        q.Cout = std::min(q.Cout_pad, cout - n0);
        q.bias = bias + n0;
        q.out = out + n0;
        if (q.Cout <= 0) break;
        if (int rc = launch_tc_part<KIND>(q, st)) return rc;
    }
    return SS_OK;
}

template <int KIND>
static int launch_tc_part(ConvParams p, cudaStream_t st)
{
    using C = TcCfg<KIND>;
    const size_t smem = C::smem(p.Cout_pad);
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
    // one M tile per CTA (measured faster than persistent CTAs here: the
    // hardware overlaps the per-tile prologues of co-resident CTAs); the
    // kernel's tile loop also supports a persistent grid
    if (int rc = launch_pdl("k_conv_tc", k_conv_tc<KIND>, dim3(ctas, splits), dim3(TC_THREADS), smem, st, p))
        return rc;
    if (splits > 1)
        return launch_splitk_reduce(ws, splits, M, p.Cout_pad, p.Cout, p.bias, p.act, p.out, p.out_ld, st);
    return SS_OK;
}

int launch_conv_tc(const ConvParams &p, int kind, cudaStream_t st)
{
    return kind == 0 ? launch_tc<0>(p, st) : launch_tc<1>(p, st);
}

}  // namespace fn
}  // namespace ss
