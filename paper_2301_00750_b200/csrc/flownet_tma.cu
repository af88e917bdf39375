// TMA-fed, warp-specialised implicit-GEMM convolution on tcgen05 (sm_100a):
// fp32 activations, "3xTF32" products (fp32-class accuracy).
//
//   D[m, n] = sum_k A[m, k] * W[k, n]   m = output pixel (128 per tile),
//   n = output channel, k = (32-channel block, filter tap, channel)
//
// 3xTF32: a = a_hi + a_lo, w = w_hi + w_lo (hi = tf32 truncation, lo exact);
// D = a_hi w_hi + a_hi w_lo + a_lo w_hi.  The weights of one output-channel
// part sit in shared memory as [w_hi rows; w_lo rows] (2 np rows), so ONE
// MMA with N = 2 np computes a_hi w_hi and a_hi w_lo into two TMEM column
// ranges and a second (N = np) adds a_lo w_hi to the first: two tcgen05.mma
// per K = 8 step; the epilogue sums the two ranges.
//
// A operand (the activations), two modes:
//   halo (stride-1 convs): a tile is 16 output rows x 8 columns; per 32-channel
//     block ONE tiled TMA load brings the (16 + 2p) x (8 + 2p) input halo
//     (OOB zero fill = the padding), converted to (hi, lo) once; each filter
//     tap is a shifted, strided view of it -- start row (ky * halo_w + kx) *
//     dil, 8-row groups halo_w rows apart -- described directly by the UMMA
//     descriptor (the SWIZZLE_128B pattern follows the absolute shared
//     address: tools/umma_shift_probe.cu);
//   im2col (strided convs): per (tap, channel block) ONE TMA im2col load of the
//     128-pixel column (the hardware walks the window, the stride and the
//     border).
// B operand: one 3-D TMA load per stage brings T taps x [hi; lo] weight rows
// (T taps per stage for narrow layers, so a stage carries enough MMA work).
//
// Warp roles (persistent CTAs, one per SM, walking (tile, K-split) units):
//   warp 0      TMA producer          warps 10-17 converters (A -> hi, lo)
//   warp 1      MMA issuer            warps 2-9  epilogue (TMEM -> bias, act,
//                                                 fp32 NHWC or split-K partials)
// TMEM holds two accumulators, so the epilogue of a unit overlaps the MMAs of
// the next.  Producer and MMA warps run converged; one elected lane issues.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "flownet.h"
#include "ss_common.cuh"
#include "tc_common.cuh"

// 1: the raw fp32 tile feeds the a_hi MMAs directly (the tensor core reads
// only the tf32 bits of an fp32 operand -- same products as the truncated hi)
#ifndef SS_TF32_HW_TRUNCATES
#define SS_TF32_HW_TRUNCATES 0
#endif

namespace ss {
namespace fn {

using namespace tc;

namespace {

// converter warps (6 .. 6 + NCONV - 1): 8 measured best for the split-bf16
// conversion (4: 388, 8: 401, 12: 399, 16: 398 frames/s at 1080p)
#ifndef SS_CONV_NCONV
#define SS_CONV_NCONV 8
#endif
constexpr int NCONV = SS_CONV_NCONV;
// epilogue warps (2 .. 2 + NEPI - 1): 4 (one per TMEM lane quarter) or 8 (two
// per quarter, each draining half of the accumulator columns)
#ifndef SS_CONV_NEPI
#define SS_CONV_NEPI 8
#endif
constexpr int NEPI = SS_CONV_NEPI;
constexpr int CONV0 = 2 + NEPI;  // first converter warp
constexpr int TM_THREADS = 32 * (2 + NEPI + NCONV);
constexpr int SMEM_MAX = 232448;  // 227 KB opt-in per CTA
constexpr int HT_H = 16, HT_W = 8;  // halo-mode output tile (rows x columns)

struct ConvArgs {
    int amode;         // A operand: 0 im2col, 1 halo (stride 1), 2 phase halo (3x3 stride 2)
    int H, W, M;       // output size, M = H * W
    int stride, k, dil, pad, taps, cin, ncb, cpp;  // cpp: channels per A row (8, 16, 32)
    int T, sp_cb;      // taps per B stage, stages per channel block
    int tiles_x, n_tiles, nk_all, k_per_split, units;
    int a_box, a_slot, na, halo_w, ph_bytes;  // ph_bytes: one phase region (amode 2)
    int np, part_row, Cout, act, out_ld, stages, b_stage, b_res;
    int parts, splits, part_rows;  // output-channel parts of np channels; weight rows per part
    const float *bias;
    float *out;
    float *ws;  // split-K partials [part][split][M][np] (null: final output)
    unsigned long long *trace;  // SS_CONV_TRACE: globaltimer stamps of CTA 0 (diagnostics)
};

// Diagnostics build only (make EXTRA=-DSS_CONV_TRACE_BUILD, then run with
// SS_CONV_TRACE=1): the null checks alone cost ~2% of the 1080p step when
// compiled in, so the default build has none.
__device__ __forceinline__ void trace_at(const ConvArgs &a, int k)
{
#ifdef SS_CONV_TRACE_BUILD
    if (a.trace && blockIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[k] = t;
    }
#else
    (void)a;
    (void)k;
#endif
}

// unit u -> (part, split, tile): units = parts * splits * n_tiles
struct ConvUnit {
    int tile, split, part;
};
__device__ __forceinline__ ConvUnit conv_unit(const ConvArgs &a, int u)
{
    const int per = a.n_tiles * a.splits;
    ConvUnit r;
    r.part = u / per;
    const int rem = u - r.part * per;
    r.split = rem / a.n_tiles;
    r.tile = rem - r.split * a.n_tiles;
    return r;
}

__device__ __forceinline__ float lk(float v) { return v >= 0.f ? v : 0.1f * v; }

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// K-major swizzled smem descriptor for rows of rowb bytes (SWIZZLE_{32,64,128}B:
// layout 6 / 4 / 2), 8-row groups sbo bytes apart, any row-aligned start
__device__ __forceinline__ uint64_t sdesc_sw(uint32_t saddr, uint32_t sbo, uint32_t layout)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

// one K = 8 step of 3xTF32 (see the file comment), elected lane of a converged warp
__device__ __forceinline__ void mma_step(uint32_t d, uint64_t ah, uint64_t al, uint64_t b,
                                         uint32_t id2, uint32_t id1, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %3, %6, 1;\n\t}" ::"r"(d),
        "l"(ah), "l"(al), "l"(b), "r"(acc), "r"(id2), "r"(id1)
        : "memory");
}

// one K = 16 step of bf16 x bf16 -> fp32 (kind::f16), elected lane
__device__ __forceinline__ void mma_step_bf16(uint32_t d, uint64_t a_, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}" ::"r"(d),
        "l"(a_), "l"(b), "r"(acc), "r"(id)
        : "memory");
}

// one K = 16 step of split-bf16 (PREC 2): a_hi x [w_hi; w_lo] (N = 2 np) and
// a_lo x w_hi (N = np, accumulating into the first np columns), elected lane
__device__ __forceinline__ void mma_step_bf16x2(uint32_t d, uint64_t ah, uint64_t al, uint64_t b, uint32_t id2,
                                                uint32_t id1, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %6, 1;\n\t}" ::"r"(d),
        "l"(ah), "l"(al), "l"(b), "r"(acc), "r"(id2), "r"(id1)
        : "memory");
}

// The same MMA steps with each 64-bit smem descriptor given as its low word
// (start address, LBO) and a high word shared by the A operands (SBO, layout):
// the halo loop then advances descriptors with 32-bit adds only
__device__ __forceinline__ void mma_step_w(uint32_t d, uint32_t ahl, uint32_t all, uint32_t ahw, uint32_t bl,
                                           uint32_t bhw, uint32_t id2, uint32_t id1, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 ah, al, bd;\n\t"
        "mov.b64 ah, {%1, %3};\n\tmov.b64 al, {%2, %3};\n\tmov.b64 bd, {%4, %5};\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bd, %7, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bd, %8, 1;\n\t}" ::"r"(d),
        "r"(ahl), "r"(all), "r"(ahw), "r"(bl), "r"(bhw), "r"(acc), "r"(id2), "r"(id1)
        : "memory");
}
__device__ __forceinline__ void mma_step_bf16x2_w(uint32_t d, uint32_t ahl, uint32_t all, uint32_t ahw, uint32_t bl,
                                                  uint32_t bhw, uint32_t id2, uint32_t id1, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 ah, al, bd;\n\t"
        "mov.b64 ah, {%1, %3};\n\tmov.b64 al, {%2, %3};\n\tmov.b64 bd, {%4, %5};\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ah, bd, %7, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], al, bd, %8, 1;\n\t}" ::"r"(d),
        "r"(ahl), "r"(all), "r"(ahw), "r"(bl), "r"(bhw), "r"(acc), "r"(id2), "r"(id1)
        : "memory");
}
__device__ __forceinline__ void mma_step_bf16_w(uint32_t d, uint32_t al_, uint32_t ahw, uint32_t bl, uint32_t bhw,
                                                uint32_t id, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 ad, bd;\n\t"
        "mov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %6, p;\n\t}" ::"r"(d),
        "r"(al_), "r"(ahw), "r"(bl), "r"(bhw), "r"(acc), "r"(id)
        : "memory");
}

// physical 16-byte chunk of logical chunk c in row r of a swizzled tile with
// rows of rb bytes (SWIZZLE_{128,64,32}B; the tile base is 1024-aligned)
__device__ __forceinline__ int swz_chunk(int c, int r, int rb)
{
    return rb == 128 ? (c ^ (r & 7)) : (rb == 64 ? (c ^ ((r >> 1) & 3)) : (c ^ ((r >> 2) & 1)));
}

// whether stage st (of a unit starting at kb) loads a new A operand
template <int AMODE>
__device__ __forceinline__ bool a_event(int st, int kb, int grp)
{
    return AMODE == 0 || st == kb || grp == 0;
}

// PREC 2: split-bf16 (fp32-class): a = a_hi + a_lo, w = w_hi + w_lo with
// bf16 terms (hi = round-to-nearest, lo = the rounded remainder, ~16
// significant bits each side), D = a_hi w_hi + a_hi w_lo + a_lo w_hi in fp32
// -- the 3xTF32 scheme on kind::f16, K = 16 per MMA at the bf16 rate;
// PREC 1: 3xTF32 (fp32-class); PREC 0: bf16 operands (converted from the fp32
// activations in shared memory, kind::f16), fp32 accumulation
template <int PREC, int AMODE, bool BRES>
__global__ void __launch_bounds__(TM_THREADS, 1)
    k_conv_tc3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const ConvArgs a)
{
    extern __shared__ __align__(1024) uint8_t cv_smem[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(cv_smem) + 1023) & ~uintptr_t(1023));
    const int S = a.stages, NA = a.na, np = a.np;
    uint8_t *aslots = base;                          // [NA][raw | lo]
    uint8_t *bst = base + 2 * NA * a.a_slot;         // [S][T][2 np rows x 128 B]
    uint64_t *a_full = reinterpret_cast<uint64_t *>(bst + S * a.b_stage);
    uint64_t *a_conv = a_full + NA, *a_empty = a_conv + NA;
    uint64_t *b_full = a_empty + NA, *b_empty = b_full + S;
    uint64_t *acc_full = b_empty + S, *acc_empty = acc_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);

    // warp index through a shuffle: the compiler then knows it (and every
    // role branch) is warp-uniform and keeps descriptors in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) trace_at(a, 0);
    const uint32_t acc_cols = (uint32_t)((PREC ? 2 : 1) * np + 31) / 32 * 32;
    uint32_t tcols = 32;
    while (tcols < 2 * acc_cols) tcols <<= 1;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NA; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_conv[i], NCONV);
            mbar_init(&a_empty[i], 1);
        }
        for (int s = 0; s < S; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], NEPI);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_rt(tmem_slot, tcols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    const uint32_t rowb = (uint32_t)a.cpp * 4u;
    if (threadIdx.x == 0) trace_at(a, 1);

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        }
        if (BRES && elect_one()) {
            // all weight stages of the layer stay resident: one load per CTA
            mbar_expect_tx(&b_full[0], (uint32_t)(a.nk_all * a.b_stage));
            for (int kk = 0; kk < a.nk_all; ++kk) {
                const int cb = kk / a.sp_cb, grp = kk - cb * a.sp_cb;
                tma_tile_3d(smem_u32(bst + kk * a.b_stage), &tmB, 0, a.part_row, cb * a.taps + grp * a.T,
                            &b_full[0]);
            }
        }
        __syncwarp();
        pdl_wait();  // the activations are the previous kernel's output
        if (lane == 0) trace_at(a, 2);
        uint32_t ga = 0, gb = 0;
        uint32_t a_pos = 0, a_ph = 1, b_pos = 0, b_ph = 1;  // empty-slot waits start on the "free" parity
        ConvUnit nx = conv_unit(a, blockIdx.x);
        for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
            const ConvUnit cu = nx;
            nx.tile += gridDim.x;
            while (nx.tile >= a.n_tiles) {
                nx.tile -= a.n_tiles;
                if (++nx.split == a.splits) {
                    nx.split = 0;
                    ++nx.part;
                }
            }
            const int tile = cu.tile, split = cu.split, prow = a.part_row + cu.part * a.part_rows;
            int x0, y0;
            if (AMODE == 0) {
                const int m0 = tile * 128, oy = m0 / a.W, ox = m0 - oy * a.W;
                x0 = ox * a.stride - a.pad;
                y0 = oy * a.stride - a.pad;
            } else {
                const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
                x0 = tx * HT_W * a.stride - a.pad;
                y0 = ty * HT_H * a.stride - a.pad;
            }
            const int kb = split * a.k_per_split, ke = min(kb + a.k_per_split, a.nk_all);
            int cb = kb / a.sp_cb, grp = kb - cb * a.sp_cb;
            for (int st = kb; st < ke; ++st, ++gb) {
                const int tap0 = grp * a.T;
                if (a_event<AMODE>(st, kb, grp)) {
                    const int sa = (int)a_pos;
                    mbar_wait(&a_empty[sa], a_ph);
                    if (++a_pos == (uint32_t)NA) {
                        a_pos = 0;
                        a_ph ^= 1;
                    }
                    if (elect_one()) {
                        const uint32_t dst = smem_u32(aslots + sa * 2 * a.a_slot);
                        mbar_expect_tx(&a_full[sa], (uint32_t)a.a_box);
                        if (ga < 9) trace_at(a, 12 + 4 * ga);
                        if (AMODE == 1) {
                            tma_tile_3d(dst, &tmA, cb * a.cpp, x0, y0, &a_full[sa]);
                        } else if (AMODE == 2) {
                            // the four (row, column) parity phases of the stride-2 window
                            for (int ph = 0; ph < 4; ++ph)
                                tma_tile_3d(dst + ph * a.ph_bytes, &tmA, cb * a.cpp, x0 + (ph & 1), y0 + (ph >> 1),
                                            &a_full[sa]);
                        } else {
                            const int ky = tap0 / a.k, kx = tap0 - ky * a.k;
                            tma_im2col_4d(dst, &tmA, cb * a.cpp, x0, y0, 0, (uint16_t)(kx * a.dil),
                                          (uint16_t)(ky * a.dil), &a_full[sa]);
                        }
                    }
                    __syncwarp();
                    ++ga;
                }
                if (!BRES) {
                    const int s = (int)b_pos;
                    mbar_wait(&b_empty[s], b_ph);
                    if (++b_pos == (uint32_t)S) {
                        b_pos = 0;
                        b_ph ^= 1;
                    }
                    if (elect_one()) {
                        mbar_expect_tx(&b_full[s], (uint32_t)a.b_stage);
                        tma_tile_3d(smem_u32(bst + s * a.b_stage), &tmB, 0, prow, cb * a.taps + tap0,
                                    &b_full[s]);
                    }
                    __syncwarp();
                }
                if (++grp == a.sp_cb) {
                    grp = 0;
                    ++cb;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        const uint32_t id2 = idesc(2u, 128u, (uint32_t)(2 * np)), id1 = idesc(2u, 128u, (uint32_t)np);
        const uint32_t idb = idesc(1u, 128u, (uint32_t)np);
        // bf16 operand rows are half as wide as the fp32 rows they come from
        const uint32_t arb = PREC == 1 ? rowb : rowb / 2;
        const uint32_t alay = arb == 128 ? 2u : (arb == 64 ? 4u : 6u);
        const uint32_t sbo = (AMODE == 0 ? 8u : (uint32_t)a.halo_w) * arb;
        const uint32_t bstride = PREC == 1 ? (uint32_t)(2 * np * 128) : (uint32_t)((PREC == 2 ? 2 : 1) * np * 64);
        const uint32_t idh2 = idesc(1u, 128u, (uint32_t)(2 * np)), idh1 = idb;  // split-bf16 shapes
        if (BRES) mbar_wait(&b_full[0], 0);
        // running ring positions / phases instead of per-event divisions (the
        // MMA warp's instruction stream paces the thin layers)
        uint32_t ga = 0, gb = 0, uc = 0;
        uint32_t a_pos = 0, a_ph = 0, b_pos = 0, b_ph = 0;
        // (part, split, tile) of unit u, advanced by gridDim.x per iteration
        ConvUnit cu = conv_unit(a, blockIdx.x);
        for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++uc) {
            const int split = cu.split;
            cu.tile += gridDim.x;
            while (cu.tile >= a.n_tiles) {
                cu.tile -= a.n_tiles;
                if (++cu.split == a.splits) cu.split = 0;
            }
            const int kb = split * a.k_per_split, ke = min(kb + a.k_per_split, a.nk_all);
            const uint32_t acc = uc & 1;
            mbar_wait(&acc_empty[acc], ((uc >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + acc * acc_cols;
            int cb = kb / a.sp_cb, grp = kb - cb * a.sp_cb, sa = 0;
            for (int st = kb; st < ke; ++st, ++gb) {
                if (a_event<AMODE>(st, kb, grp)) {
                    sa = (int)a_pos;
                    mbar_wait(&a_conv[sa], a_ph);
                    if (ga == 0 && lane == 0) trace_at(a, 5);
                    ++ga;
                    if (++a_pos == (uint32_t)NA) {
                        a_pos = 0;
                        a_ph ^= 1;
                    }
                }
                const int s = BRES ? st : (int)b_pos;
                if (!BRES) {
                    mbar_wait(&b_full[s], b_ph);
                    if (++b_pos == (uint32_t)S) {
                        b_pos = 0;
                        b_ph ^= 1;
                    }
                }
                tc_fence_after();
                const int tap0 = grp * a.T, nt = min(a.T, a.taps - tap0);
                const int live = min(a.cpp, a.cin - cb * a.cpp);
                const int nks = PREC == 1 ? (live + 7) >> 3 : (live + 15) >> 4;
                const uint32_t araw = smem_u32(aslots + sa * 2 * a.a_slot);
                const uint32_t b0 = smem_u32(bst + s * a.b_stage);
                int ky = tap0 / a.k, kx = tap0 - ky * a.k;
                if (AMODE == 1) {
                    // halo views: the descriptors' start-address fields (addr >> 4)
                    // advance by fixed steps per tap, so the stage's base
                    // descriptors are built once and each tap adds its offset
                    const uint32_t cstep = ((uint32_t)a.dil * arb) >> 4;
                    const uint32_t rstep = ((uint32_t)(a.halo_w * a.dil) * arb) >> 4;
                    uint32_t o16 = (uint32_t)ky * rstep + (uint32_t)kx * cstep;
                    const uint32_t bstep = bstride >> 4;
                    const uint64_t bd0 = PREC == 1 ? sdesc_sw128(b0) : sdesc_sw(b0, 512u, 4u);
                    const uint64_t da0 = sdesc_sw(araw + (PREC == 1 ? 0u : (uint32_t)a.a_slot), sbo, alay);
                    const uint64_t dl0 = sdesc_sw(araw + (uint32_t)a.a_slot + (PREC == 2 ? (uint32_t)a.a_slot / 2 : 0u),
                                                  sbo, alay);
                    // low words advance, high words (SBO, layout) are per operand constants
                    const uint32_t ahw = (uint32_t)(da0 >> 32), bhw = (uint32_t)(bd0 >> 32);
                    uint32_t bl = (uint32_t)bd0;
                    const uint32_t al0 = (uint32_t)da0, ll0 = (uint32_t)dl0;
                    const uint32_t acc0 = st > kb ? 1u : 0u;
                    for (int j = 0; j < nt; ++j, bl += bstep) {
                        const uint32_t al = al0 + o16, ll = ll0 + o16;
                        for (int i = 0; i < nks; ++i) {
                            const uint32_t acc = (j | i) ? 1u : acc0;
                            if (PREC == 2)
                                mma_step_bf16x2_w(d, al + 2 * i, ll + 2 * i, ahw, bl + 2 * i, bhw, idh2, idh1, acc);
                            else if (PREC == 1)
                                mma_step_w(d, al + 2 * i, ll + 2 * i, ahw, bl + 2 * i, bhw, id2, id1, acc);
                            else
                                mma_step_bf16_w(d, al + 2 * i, ahw, bl + 2 * i, bhw, idb, acc);
                        }
                        if (++kx == a.k) {
                            kx = 0;
                            o16 += rstep - (uint32_t)(a.k - 1) * cstep;
                        } else {
                            o16 += cstep;
                        }
                    }
                } else
                for (int j = 0; j < nt; ++j) {
                    uint32_t off = 0;
                    if (AMODE == 1)
                        off = (uint32_t)((ky * a.halo_w + kx) * a.dil) * arb;
                    else if (AMODE == 2)
                        off = (uint32_t)(((ky & 1) * 2 + (kx & 1)) * (PREC == 1 ? a.ph_bytes : a.ph_bytes / 2)) +
                              (uint32_t)((ky >> 1) * a.halo_w + (kx >> 1)) * arb;
                    // B rows hold 32 channels: a narrow A row (cpp < 32) only
                    // ever meets channel block 0, whose first cpp channels align
                    if (PREC == 2) {
                        // hi / lo bf16 copies in the second half of the slot
                        const uint64_t ah = sdesc_sw(araw + a.a_slot + off, sbo, alay);
                        const uint64_t al = sdesc_sw(araw + a.a_slot + a.a_slot / 2 + off, sbo, alay);
                        const uint64_t bd = sdesc_sw(b0 + j * bstride, 512u, 4u);  // 64-byte rows
                        for (int i = 0; i < nks; ++i)  // K = 16 bf16 = 32 bytes per MMA
                            mma_step_bf16x2(d, ah + 2 * i, al + 2 * i, bd + 2 * i, idh2, idh1,
                                            (st > kb || j > 0 || i > 0) ? 1u : 0u);
                    } else if (PREC) {
                        const uint64_t ah = sdesc_sw(araw + off, sbo, alay);
                        const uint64_t al = sdesc_sw(araw + a.a_slot + off, sbo, alay);
                        const uint64_t bd = sdesc_sw128(b0 + j * bstride);
                        for (int i = 0; i < nks; ++i)  // +32 bytes of K = +2 in the address field
                            mma_step(d, ah + 2 * i, al + 2 * i, bd + 2 * i, id2, id1,
                                     (st > kb || j > 0 || i > 0) ? 1u : 0u);
                    } else {
                        // bf16 copy of the tile lives in the second half of the slot
                        const uint64_t ad = sdesc_sw(araw + a.a_slot + off, sbo, alay);
                        const uint64_t bd = sdesc_sw(b0 + j * bstride, 512u, 4u);  // 64-byte rows
                        for (int i = 0; i < nks; ++i)  // K = 16 bf16 = 32 bytes per MMA
                            mma_step_bf16(d, ad + 2 * i, bd + 2 * i, idb, (st > kb || j > 0 || i > 0) ? 1u : 0u);
                    }
                    if (++kx == a.k) {
                        kx = 0;
                        ++ky;
                    }
                }
                if (!BRES) mma_commit_elect(&b_empty[s]);
                const bool a_last = AMODE == 0 || grp == a.sp_cb - 1 || st == ke - 1;
                if (a_last) mma_commit_elect(&a_empty[sa]);
                __syncwarp();
                if (++grp == a.sp_cb) {
                    grp = 0;
                    ++cb;
                }
            }
            mma_commit_elect(&acc_full[acc]);
            __syncwarp();
            if (uc == 0 && lane == 0) trace_at(a, 6);
            if (uc < 9 && lane == 0) trace_at(a, 12 + 4 * uc + 2);
        }
    } else if (warp < CONV0) {
        // ---------------- epilogue ----------------
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int eh = (warp - 2) / 4;  // NEPI = 8: which half of the columns
        pdl_wait();
        uint32_t uc = 0;
        for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++uc) {
            const uint32_t acc = uc & 1;
            mbar_wait(&acc_full[acc], (uc >> 1) & 1);
            tc_fence_after();
            if (uc == 0 && warp == 2 && lane == 0) trace_at(a, 7);
            const ConvUnit cu = conv_unit(a, u);
            const int tile = cu.tile, split = cu.split;
            const int cout = min(np, a.Cout - cu.part * np);  // this part's live channels
            const float *bias = a.bias + cu.part * np;
            float *outp = a.out + cu.part * np;
            const int m = q * 32 + lane;
            bool ok;
            size_t pix;
            if (AMODE == 0) {
                pix = (size_t)tile * 128 + m;
                ok = pix < (size_t)a.M;
            } else {
                const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
                const int oy = ty * HT_H + (m >> 3), ox = tx * HT_W + (m & 7);
                ok = oy < a.H && ox < a.W;
                pix = (size_t)oy * a.W + ox;
            }
            const uint32_t t0 = tmem + acc * acc_cols + ((uint32_t)(q * 32) << 16);
            const int cstep = NEPI == 8 ? 32 : 16;  // NEPI = 8: the two warps of a quarter alternate 16-column chunks
            for (int c0 = NEPI == 8 ? 16 * eh : 0; c0 < np; c0 += cstep) {
                float v[16];
                tmem_ld16(t0 + c0, v);
                if (PREC) {
                    float w[16];
                    tmem_ld16(t0 + np + c0, w);
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] += w[i];
                }
                if (!ok) continue;
                if (a.ws) {
                    float *dst = a.ws + (((size_t)cu.part * a.splits + split) * a.M + pix) * np + c0;
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        *reinterpret_cast<float4 *>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                } else if (c0 < cout) {
                    float *dst = outp + pix * a.out_ld + c0;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float x = v[i] + (c0 + i < cout ? __ldg(bias + c0 + i) : 0.f);
                        v[i] = a.act ? lk(x) : x;
                    }
                    if (c0 + 16 <= cout) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            *reinterpret_cast<float4 *>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (i < cout - c0) dst[i] = v[i];
                    }
                }
            }
            if (uc == 0 && warp == 2 && lane == 0) trace_at(a, 11);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);
            if (uc == 0 && warp == 2 && lane == 0) trace_at(a, 8);
            if (uc < 9 && warp == 2 && lane == 0) trace_at(a, 12 + 4 * uc + 3);
        }
    } else {
        // ---------------- converters: A -> (hi in place, lo beside) ----------------
        const int t = threadIdx.x - 32 * CONV0;
        const int n16 = a.a_slot / 16;  // whole slot (phase padding included)
        uint32_t ga = 0, a_pos = 0, a_ph = 0;
        ConvUnit nx = conv_unit(a, blockIdx.x);
        for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
            const int split = nx.split;
            nx.tile += gridDim.x;
            while (nx.tile >= a.n_tiles) {
                nx.tile -= a.n_tiles;
                if (++nx.split == a.splits) nx.split = 0;
            }
            const int kb = split * a.k_per_split, ke = min(kb + a.k_per_split, a.nk_all);
            int grp = kb % a.sp_cb;
            for (int st = kb; st < ke; ++st) {
                const bool ev = a_event<AMODE>(st, kb, grp);
                if (++grp == a.sp_cb) grp = 0;
                if (!ev) continue;
                const int sa = (int)a_pos;
                mbar_wait(&a_full[sa], a_ph);
                if (++a_pos == (uint32_t)NA) {
                    a_pos = 0;
                    a_ph ^= 1;
                }
                if (ga == 0 && t == 0) trace_at(a, 3);
                if (ga < 9 && t == 0) trace_at(a, 12 + 4 * ga + 1);
                ++ga;
                float4 *ar = reinterpret_cast<float4 *>(aslots + sa * 2 * a.a_slot);
                if (PREC == 2) {
                    // fp32 row r -> bf16 hi / lo rows (rowb / 2 bytes, swizzled for
                    // that width): hi = rn(v), lo = rn(v - hi).  One thread per
                    // 16-byte bf16 chunk (8 channels = two fp32 chunks): two
                    // LDS.128, two STS.128
                    uint8_t *bh = aslots + sa * 2 * a.a_slot + a.a_slot, *bl = bh + a.a_slot / 2;
                    const int rb = (int)rowb, rb2 = rb / 2;
                    const int sh = rb2 == 64 ? 2 : 1;  // log2(bf16 chunks per row): rb2 is 64 or 32
                    const int n8 = n16 / 2;
                    for (int q = t; q < n8; q += 32 * NCONV) {
                        const int r = q >> sh, k = q & ((1 << sh) - 1);
                        const float4 v0 = ar[r * (2 << sh) + swz_chunk(2 * k, r, rb)];
                        const float4 v1 = ar[r * (2 << sh) + swz_chunk(2 * k + 1, r, rb)];
                        const float f[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                        uint32_t hw[4], lw[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
                            const float2 hf = __bfloat1622float2(h);
                            const __nv_bfloat162 l = __floats2bfloat162_rn(f[2 * e] - hf.x, f[2 * e + 1] - hf.y);
                            hw[e] = *reinterpret_cast<const uint32_t *>(&h);
                            lw[e] = *reinterpret_cast<const uint32_t *>(&l);
                        }
                        const int o = r * rb2 + swz_chunk(k, r, rb2) * 16;
                        *reinterpret_cast<uint4 *>(bh + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                        *reinterpret_cast<uint4 *>(bl + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                    }
                } else if (PREC) {
                    float4 *lo = reinterpret_cast<float4 *>(aslots + sa * 2 * a.a_slot + a.a_slot);
                    for (int j = t; j < n16; j += 32 * NCONV) {
                        const float4 v = ar[j];
                        const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
#if !SS_TF32_HW_TRUNCATES
                        ar[j] = h;
#endif
                        lo[j] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
                    }
                } else {
                    // fp32 row r (rowb bytes, swizzled) -> bf16 row r (rowb / 2
                    // bytes, swizzled for that width) in the second half of the slot
                    // one thread per 16-byte bf16 chunk (two fp32 chunks), as in PREC 2
                    uint8_t *bf = aslots + sa * 2 * a.a_slot + a.a_slot;
                    const int rb = (int)rowb, rb2 = rb / 2;
                    const int sh = rb2 == 64 ? 2 : 1;  // log2(bf16 chunks per row)
                    const int n8 = n16 / 2;
                    for (int q = t; q < n8; q += 32 * NCONV) {
                        const int r = q >> sh, k = q & ((1 << sh) - 1);
                        const float4 v0 = ar[r * (2 << sh) + swz_chunk(2 * k, r, rb)];
                        const float4 v1 = ar[r * (2 << sh) + swz_chunk(2 * k + 1, r, rb)];
                        const __nv_bfloat162 b0 = __floats2bfloat162_rn(v0.x, v0.y), b1 = __floats2bfloat162_rn(v0.z, v0.w),
                                             b2 = __floats2bfloat162_rn(v1.x, v1.y), b3 = __floats2bfloat162_rn(v1.z, v1.w);
                        *reinterpret_cast<uint4 *>(bf + r * rb2 + swz_chunk(k, r, rb2) * 16) =
                            make_uint4(*reinterpret_cast<const uint32_t *>(&b0), *reinterpret_cast<const uint32_t *>(&b1),
                                       *reinterpret_cast<const uint32_t *>(&b2), *reinterpret_cast<const uint32_t *>(&b3));
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_conv[sa]);
                if (ga == 1 && t == 0) trace_at(a, 4);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) trace_at(a, 9);
    if (threadIdx.x == 0) pdl_trigger();  // dependents launch as this grid drains
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_rt(tmem, tcols);
    }
}

template <class PFN>
PFN driver_fn(const char *name)
{
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        return reinterpret_cast<PFN>(p);
    return nullptr;
}

PFN_cuTensorMapEncodeTiled_v12000 tiled_fn()
{
    static auto fn = driver_fn<PFN_cuTensorMapEncodeTiled_v12000>("cuTensorMapEncodeTiled");
    return fn;
}

PFN_cuTensorMapEncodeIm2col_v12000 im2col_fn()
{
    static auto fn = driver_fn<PFN_cuTensorMapEncodeIm2col_v12000>("cuTensorMapEncodeIm2col");
    return fn;
}

int n_sm_tma = 0;

CUtensorMapSwizzle swz_for(int rowb)
{
    return rowb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (rowb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// amode 1: box (cpp, halo_w, halo_h); amode 2: box (cpp, 18, 34) with
// traversal stride 2 in W and H (a 9 x 17 phase of the stride-2 window);
// amode 0: im2col column of 128 pixels
int encode_act_map(CUtensorMap *m, const ConvParams &p, int amode, int cpp, int halo_w, int halo_h)
{
    CUresult r;
    const int rowb = cpp * 4;
    if (amode != 0) {
        auto fn = tiled_fn();
        if (!fn) {
            set_error("cuTensorMapEncodeTiled unavailable");
            return SS_CUDA_ERROR;
        }
        const cuuint64_t dims[3] = {(cuuint64_t)p.Cin, (cuuint64_t)p.W, (cuuint64_t)p.H};
        const cuuint64_t strides[2] = {(cuuint64_t)p.in_ld * 4, (cuuint64_t)p.in_ld * 4 * p.W};
        const cuuint32_t box2[3] = {(cuuint32_t)cpp, 18, 34}, box1[3] = {(cuuint32_t)cpp, (cuuint32_t)halo_w,
                                                                          (cuuint32_t)halo_h};
        const cuuint32_t estr2[3] = {1, 2, 2}, estr1[3] = {1, 1, 1};
        r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(p.in), dims, strides,
               amode == 2 ? box2 : box1, amode == 2 ? estr2 : estr1, CU_TENSOR_MAP_INTERLEAVE_NONE, swz_for(rowb),
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        auto fn = im2col_fn();
        if (!fn) {
            set_error("cuTensorMapEncodeIm2col unavailable");
            return SS_CUDA_ERROR;
        }
        const cuuint64_t dims[4] = {(cuuint64_t)p.Cin, (cuuint64_t)p.W, (cuuint64_t)p.H, 1};
        const cuuint64_t strides[3] = {(cuuint64_t)p.in_ld * 4, (cuuint64_t)p.in_ld * 4 * p.W,
                                       (cuuint64_t)p.in_ld * 4 * p.W * p.H};
        const int up = p.pad - p.dil * (p.k - 1);
        const int lower[2] = {-p.pad, -p.pad};  // (W, H)
        const int upper[2] = {up, up};
        const cuuint32_t estr[4] = {1, (cuuint32_t)p.stride, (cuuint32_t)p.stride, 1};
        r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(p.in), dims, strides, lower, upper,
               (cuuint32_t)cpp, 128, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz_for(rowb),
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
        set_error(std::string("activation tensor map encode failed: ") + std::to_string((int)r));
        return SS_CUDA_ERROR;
    }
    return SS_OK;
}

}  // namespace

// A-operand mode of a layer (see launch_conv_tma): stride-1 -> halo; 3x3
// stride 2 with <= 16 input channels -> phase halo (its four phase tiles of
// 32-channel rows would not fit twice in shared memory); otherwise im2col
static int amode_for(int k, int stride, int dil, int cin)
{
    if (stride == 1) return 1;
    if (stride == 2 && k == 3 && dil == 1 && cin <= 16) return 2;
    return 0;
}

int tma_taps_per_stage(int k, int stride, int dil, int cin, int np, int prec)
{
    if (amode_for(k, stride, dil, cin) == 0) return 1;  // im2col: one tap per stage
    const int tap_bytes = prec == 1 ? 2 * np * 128 : (prec == 2 ? 2 : 1) * np * 64;
    // ~36 KB of weights per stage (a smaller stage costs more: 18 KB for
    // split-bf16 measured 408 -> 394 frames/s; larger ones do not fit 2 stages)
    return std::max(1, std::min(k * k, 36864 / tap_bytes));
}

// bf16 weight tensor map over [kblocks][rows = parts * np][32] bf16 (64-byte
// rows, SWIZZLE_64B): per stage one box of 32 K x np rows x T kblocks
int encode_weight_map_bf16(CUtensorMap *m, const void *wt, int kblocks, int rows, int np, int T)
{
    return encode_weight_map_bf16_rows(m, wt, kblocks, rows, np, T);
}

// box of 32 K x box_rows x T kblocks over [kblocks][rows][32] bf16
int encode_weight_map_bf16_rows(CUtensorMap *m, const void *wt, int kblocks, int rows, int box_rows, int T)
{
    const int np = box_rows;
    auto fn = tiled_fn();
    if (!fn) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return SS_CUDA_ERROR;
    }
    const cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)kblocks};
    const cuuint64_t strides[2] = {64, (cuuint64_t)rows * 64};
    const cuuint32_t box[3] = {32, (cuuint32_t)np, (cuuint32_t)T};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(wt), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (bf16 weights) failed: " + std::to_string((int)r));
        return SS_CUDA_ERROR;
    }
    return SS_OK;
}

// weight tensor map over [kblocks][rows = parts * 2 np][32] fp32: per stage
// one box of 32 K x 2 np rows ([hi; lo] of one part) x T kblocks (taps)
int encode_weight_map(CUtensorMap *m, const float *wt, int kblocks, int rows, int np, int T)
{
    auto fn = tiled_fn();
    if (!fn) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return SS_CUDA_ERROR;
    }
    const cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)kblocks};
    const cuuint64_t strides[2] = {128, (cuuint64_t)rows * 128};
    const cuuint32_t box[3] = {32, (cuuint32_t)(2 * np), (cuuint32_t)T};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(wt), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (weights) failed: " + std::to_string((int)r));
        return SS_CUDA_ERROR;
    }
    return SS_OK;
}

// SS_CONV_TRACE=1 (diagnostics): every conv launch stamps CTA 0's milestones
// (globaltimer) into a mapped host ring; conv_trace_dump prints them
static unsigned long long *trace_dev = nullptr;  // device ring (stamps stay off the PCIe path)
static int trace_n = 0;
constexpr int TRACE_SLOTS = 128, TRACE_K = 48;  // 12 milestones + 4 per unit for 9 units
static unsigned long long *conv_trace_slot()
{
#ifndef SS_CONV_TRACE_BUILD
    return nullptr;
#endif
    static const bool on = getenv("SS_CONV_TRACE") != nullptr;
    if (!on) return nullptr;
    if (!trace_dev) {
        if (cudaMalloc(&trace_dev, TRACE_SLOTS * TRACE_K * 8) != cudaSuccess) return nullptr;
        cudaMemset(trace_dev, 0, TRACE_SLOTS * TRACE_K * 8);
    }
    return trace_dev + (size_t)(trace_n++ % TRACE_SLOTS) * TRACE_K;
}

using ConvKernel = void (*)(CUtensorMap, CUtensorMap, ConvArgs);

static ConvKernel conv_kernel(int prec, int amode, bool res)
{
    static const ConvKernel tab[3][3][2] = {
        {{k_conv_tc3<0, 0, false>, k_conv_tc3<0, 0, true>},
         {k_conv_tc3<0, 1, false>, k_conv_tc3<0, 1, true>},
         {k_conv_tc3<0, 2, false>, k_conv_tc3<0, 2, true>}},
        {{k_conv_tc3<1, 0, false>, k_conv_tc3<1, 0, true>},
         {k_conv_tc3<1, 1, false>, k_conv_tc3<1, 1, true>},
         {k_conv_tc3<1, 2, false>, k_conv_tc3<1, 2, true>}},
        {{k_conv_tc3<2, 0, false>, k_conv_tc3<2, 0, true>},
         {k_conv_tc3<2, 1, false>, k_conv_tc3<2, 1, true>},
         {k_conv_tc3<2, 2, false>, k_conv_tc3<2, 2, true>}}};
    return tab[prec][amode][res ? 1 : 0];
}

int prepare_conv_tma()
{
    static bool done = false;
    if (done) return SS_OK;
    if (int rc = prepare_flow_kernels()) return rc;
    for (int prec = 0; prec < 3; ++prec)
        for (int am = 0; am < 3; ++am)
            for (int res = 0; res < 2; ++res)
                SS_CUDA_TRY(cudaFuncSetAttribute(conv_kernel(prec, am, res != 0),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX));
    int dev = 0;
    SS_CUDA_TRY(cudaGetDevice(&dev));
    SS_CUDA_TRY(cudaDeviceGetAttribute(&n_sm_tma, cudaDevAttrMultiProcessorCount, dev));
    done = true;
    return SS_OK;
}

// one output-channel part (rows [part * 2 np, +2 np) of the weight tensor)
// all output-channel parts of np channels in one launch (units cover parts x
// splits x tiles; part p uses weight rows [p * part_rows, +part_rows))
static int launch_parts(const ConvParams &p, const CUtensorMap &tmA, int prec, int amode, int cpp, int halo_w,
                        int halo_h, int parts, int np, cudaStream_t st)
{
    ConvArgs a;
    a.amode = amode;
    a.H = p.Ho;
    a.W = p.Wo;
    a.M = p.Ho * p.Wo;
    a.stride = p.stride;
    a.k = p.k;
    a.dil = p.dil;
    a.pad = p.pad;
    a.taps = p.k * p.k;
    a.cin = p.Cin;
    a.cpp = cpp;
    a.ncb = (p.Cin + cpp - 1) / cpp;
    a.T = p.tma_T;
    a.sp_cb = (a.taps + a.T - 1) / a.T;
    const int rowb = cpp * 4;
    a.ph_bytes = 0;
    if (amode == 0) {
        a.tiles_x = 0;
        a.n_tiles = (a.M + 127) / 128;
        a.halo_w = 8;
        a.a_box = 128 * rowb;
        a.a_slot = (a.a_box + 1023) / 1024 * 1024;
        a.na = 4;
    } else {
        a.tiles_x = (p.Wo + HT_W - 1) / HT_W;
        a.n_tiles = a.tiles_x * ((p.Ho + HT_H - 1) / HT_H);
        if (amode == 1) {
            a.halo_w = halo_w;
            a.a_box = halo_w * halo_h * rowb;
            a.a_slot = (a.a_box + 1023) / 1024 * 1024;
        } else {
            a.halo_w = 9;  // phase tiles: 17 rows x 9 columns
            a.ph_bytes = (9 * 17 * rowb + 1023) / 1024 * 1024;
            a.a_box = 4 * 9 * 17 * rowb;
            a.a_slot = 4 * a.ph_bytes;
        }
        a.na = 2;
    }
    a.nk_all = a.ncb * a.sp_cb;
    a.np = np;
    a.parts = parts;
    a.part_row = 0;
    a.part_rows = (prec ? 2 : 1) * np;
    a.Cout = p.Cout;  // all parts
    a.act = p.act;
    a.out_ld = p.out_ld;
    a.bias = p.bias;
    a.out = p.out;
    // [hi; lo] fp32 rows | [hi; lo] bf16 rows | bf16 rows
    a.b_stage = prec == 1 ? a.T * 2 * np * 128 : a.T * (prec == 2 ? 2 : 1) * np * 64;
    const int bar_bytes = 1024 + 512;
    // weights resident for the whole launch when every stage fits
    static const bool res_on = getenv("SS_CONV_BRES") == nullptr || strcmp(getenv("SS_CONV_BRES"), "0");
    const bool res_fits = parts == 1 &&
                          2 * a.na * a.a_slot + a.nk_all * a.b_stage + bar_bytes + a.nk_all * 16 <= SMEM_MAX;
    // streaming needs 2 stages beside the A slots; a layer that cannot stream
    // keeps its weights resident even under SS_CONV_BRES=0
    const bool can_stream = (SMEM_MAX - 2 * a.na * a.a_slot - bar_bytes) / a.b_stage >= 2 || amode == 0;
    a.b_res = res_fits && (res_on || !can_stream);
    if (a.b_res) {
        a.stages = a.nk_all;
    } else {
        a.stages = std::min(8, (SMEM_MAX - 2 * a.na * a.a_slot - bar_bytes) / a.b_stage);
        if (a.stages < 2 && amode == 0) {
            a.na = 2;
            a.stages = std::min(8, (SMEM_MAX - 2 * a.na * a.a_slot - bar_bytes) / a.b_stage);
        }
    }
    if (a.stages < (a.b_res ? 1 : 2)) {
        set_error("conv stage does not fit in shared memory");
        return SS_VALUE_ERROR;
    }
    // halo tiles: with the weights resident, spend the spare shared memory on
    // more A slots -- thin layers are bound by the per-tile chain (TMA
    // round trip, conversion, MMAs) that two slots barely overlap
    static const int na_max = [] {
        const char *e = getenv("SS_CONV_NA");
        return e ? std::max(2, std::min(8, atoi(e))) : 6;
    }();
    if (amode != 0 && a.b_res)
        while (a.na < na_max &&
               2 * (a.na + 1) * a.a_slot + a.nk_all * a.b_stage + bar_bytes + a.nk_all * 16 <= SMEM_MAX)
            ++a.na;
    // Split K only when the tiles fill less than a quarter of the SMs, into
    // at most 8 parts: every split adds a reduction kernel to the dependent
    // chain, and on the critical chain that latency costs more than the idle
    // SMs a less split layer leaves (which the concurrent flow fills).
    // Measured at 1080p: fill-all-SMs splitting 340.5 -> 347.9 frames/s.
    int splits = 1;
    static const int sk_f = getenv("SS_SPLITK_F") ? std::max(1, atoi(getenv("SS_SPLITK_F"))) : 4;
    static const int sk_max = getenv("SS_SPLITK_MAX") ? std::max(1, atoi(getenv("SS_SPLITK_MAX"))) : 8;
    const int tiles_all = a.n_tiles * parts;
    // the CTAs this launch may use: units beyond them run as a second round,
    // so the split count rounds DOWN (est5_1 at 1080p: 24 tiles x 7 splits =
    // 168 units on 148 SMs took two rounds; x 6 = 144 takes one)
    const int avail = p.grid_cap > 0 ? std::min(p.grid_cap, n_sm_tma) : n_sm_tma;
    if (p.ws && tiles_all * sk_f < n_sm_tma && a.nk_all >= 4) {
        splits = std::min(std::min(std::max(avail / tiles_all, 1), a.nk_all / 2), sk_max);
        const size_t need = (size_t)parts * splits * a.M * np;
        if (need > p.ws_floats) splits = (int)(p.ws_floats / ((size_t)parts * a.M * np));
        splits = std::max(splits, 1);
    }
    a.k_per_split = (a.nk_all + splits - 1) / splits;
    splits = (a.nk_all + a.k_per_split - 1) / a.k_per_split;
    a.splits = splits;
    a.ws = splits > 1 ? p.ws : nullptr;
    a.units = tiles_all * splits;
    a.trace = conv_trace_slot();
    // SS_CONV_GRID_MAX (tests): fewer persistent CTAs, so small layers also
    // walk several units per CTA (TMEM accumulator alternation, ring wrap)
    static const int grid_max = getenv("SS_CONV_GRID_MAX") ? std::max(1, atoi(getenv("SS_CONV_GRID_MAX"))) : 0;
    int grid = std::min(a.units, p.grid_cap > 0 ? std::min(p.grid_cap, n_sm_tma) : n_sm_tma);
    if (grid_max) grid = std::min(grid, grid_max);
    const size_t smem = (size_t)2 * a.na * a.a_slot + (size_t)a.stages * a.b_stage + bar_bytes + a.stages * 16;
    const CUtensorMap &tmB = *static_cast<const CUtensorMap *>(p.tmB);
    const int rc = launch_pdl("k_conv_tc3", conv_kernel(prec, amode, a.b_res != 0), dim3(grid), dim3(TM_THREADS),
                              smem, st, tmA, tmB, a);
    if (rc) return rc;
    if (splits > 1)
        return launch_splitk_reduce(p.ws, splits, a.M, np, p.Cout, p.bias, p.act, p.out, p.out_ld, st, parts);
    return SS_OK;
}

void conv_trace_dump(const char *what)
{
    if (!trace_dev || !trace_n) return;
    cudaDeviceSynchronize();
    std::vector<unsigned long long> hst((size_t)TRACE_SLOTS * TRACE_K);
    cudaMemcpy(hst.data(), trace_dev, hst.size() * 8, cudaMemcpyDeviceToHost);
    const unsigned long long *trace_host = hst.data();
    static const char *names[12] = {"entry", "setup", "pdl_ok", "A_land", "A_conv", "mma_go",
                                    "mma_done", "epi_go", "epi_done", "exit", "epi_ld1", "epi_loop"};
    for (int i = 0; i < trace_n && i < TRACE_SLOTS; ++i) {
        const unsigned long long *t = trace_host + (size_t)i * TRACE_K;
        fprintf(stderr, "[conv-trace] %s #%d", what, i);
        for (int k = 1; k < 12; ++k)
            fprintf(stderr, " %s=%+.2f", names[k], t[k] ? (double)(t[k] - t[0]) * 1e-3 : -1.0);
        fprintf(stderr, " us\n");
        for (int u = 0; u < 9 && t[12 + 4 * u]; ++u)
            fprintf(stderr, "[conv-trace]    unit %d: A_issue %+.2f A_land %+.2f mma_done %+.2f epi_done %+.2f\n", u,
                    (double)(t[12 + 4 * u] - t[0]) * 1e-3, (double)(t[13 + 4 * u] - t[0]) * 1e-3,
                    t[14 + 4 * u] ? (double)(t[14 + 4 * u] - t[0]) * 1e-3 : -1.0,
                    t[15 + 4 * u] ? (double)(t[15 + 4 * u] - t[0]) * 1e-3 : -1.0);
    }
    cudaMemset(trace_dev, 0, TRACE_SLOTS * TRACE_K * 8);
    trace_n = 0;
}

int launch_conv_tma(const ConvParams &p, int prec, cudaStream_t st)
{
    if (int rc = prepare_conv_tma()) return rc;
    if (!p.tmB) {
        set_error("conv layer has no TMA weight map");
        return SS_VALUE_ERROR;
    }
    static const bool halo_on = getenv("SS_CONV_HALO") == nullptr || strcmp(getenv("SS_CONV_HALO"), "0");
    int amode = halo_on ? amode_for(p.k, p.stride, p.dil, p.Cin) : 0;
    if (amode == 1 && !(p.Ho == p.H && p.Wo == p.W)) amode = 0;
    if (amode == 2 && p.pad != 1) amode = 0;
    if (amode == 0 && p.tma_T != 1) {
        set_error("im2col conv path needs one tap per stage");
        return SS_VALUE_ERROR;
    }
    static const bool wide = getenv("SS_CONV_CPP32") != nullptr;
    // bf16: a K = 16 MMA needs >= 16 channels per row
    const int cmin = prec == 1 ? 8 : 16;
    const int cpp = (wide && amode != 2) ? 32 : std::max(cmin, p.Cin <= 8 ? 8 : (p.Cin <= 16 ? 16 : 32));
    const int halo_w = HT_W + 2 * p.pad, halo_h = HT_H + 2 * p.pad;
    alignas(64) CUtensorMap tmA;
    if (int rc = encode_act_map(&tmA, p, amode, cpp, halo_w, halo_h)) return rc;
    const int parts = (p.Cout_pad + 127) / 128;
    const int np = p.Cout_pad / parts;
    return launch_parts(p, tmA, prec, amode, cpp, halo_w, halo_h, parts, np, st);
}

}  // namespace fn
}  // namespace ss
