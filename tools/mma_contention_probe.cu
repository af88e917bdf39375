// Probe: why do the thin conv layers' MMAs run ~4x slower in the real kernel
// (pyr1b: ~200 clk per kind::f16 MMA, N = 32 / 16) than back to back in
// tools/mma_rate_probe (~46 clk)?  One CTA issues the split-bf16 conv pattern
// (per K = 16 step: N = 2 np with A = a_hi, then N = np with A = a_lo, tap
// views of a halo tile) from one thread, while other warps of the CTA
// optionally generate the real kernel's side traffic:
//   mode bit 1: 8 "epilogue" warps loop tcgen05.ld over another TMEM range
//   mode bit 2: 8 "converter" warps stream LDS.128 / STS.128 over a separate
//               shared-memory buffer
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_contention_probe tools/mma_contention_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2301_00750_b200/csrc/tc_common.cuh"

using namespace ss::tc;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t sbo, uint32_t layout)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}

constexpr int NT = 18 * 32;  // 18 warps like the conv kernel

__global__ void __launch_bounds__(NT, 1) probe(int np, int reps, int mode, long long *out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *base = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t *ahi = base, *alo = base + 16 * 1024, *bs = base + 32 * 1024;  // A 16 KB each, B 9 x 4 KB
    uint8_t *side = base + 80 * 1024;                                         // 64 KB converter traffic
    __shared__ uint64_t mbar, ubar[2];
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (144 * 1024) / 4; i += NT) reinterpret_cast<float *>(base)[i] = 0.001f;
    if (tid == 0) {
        mbar_init(&mbar, 1);
        mbar_init(&ubar[0], 1);
        mbar_init(&ubar[1], 1);
        fence_barrier_init();
        stop = 0;
    }
    if (warp == 0) tmem_alloc_rt(&tslot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 1) {
        if ((tid & 31) == 0) {
            const uint32_t rowb = 32;  // 16 bf16 channels per row (pyr1b), SWIZZLE_32B
            const uint32_t lay = 6, sbo = 10 * rowb;
            const uint32_t id2 = idesc(1u, 128u, (uint32_t)(2 * np)), id1 = idesc(1u, 128u, (uint32_t)np);
            long long t0 = clock64();
            // mode bit 4: per "unit" of 9 K steps the conv kernel's bookkeeping --
            // a fresh accumulation (acc = 0) in the other TMEM accumulator and two
            // commits (slot free, accumulator full) to barriers nobody waits on
            const bool units = mode & 4;
            uint32_t d = tmem;
            for (int r = 0; r < reps; ++r) {
                const int tap = r % 9;
                if (units && tap == 0 && r > 0) {
                    mma_commit(&ubar[0]);
                    mma_commit(&ubar[1]);
                    d = d == tmem ? tmem + 128 : tmem;
                }
                const uint32_t off = (uint32_t)(((tap / 3) * 10 + tap % 3) * rowb);
                const uint64_t bd = desc(smem_u32(bs) + tap * 4096, 512, 4);
                mma_f16(d, desc(smem_u32(ahi) + off, sbo, lay), bd, id2, (units ? tap > 0 : r > 0) ? 1u : 0u);
                mma_f16(d, desc(smem_u32(alo) + off, sbo, lay), bd, id1, 1u);
            }
            mma_commit(&mbar);
            mbar_wait(&mbar, 0);
            out[0] = clock64() - t0;
            stop = 1;
        }
        __syncwarp();
    } else if (warp >= 2 && warp < 10 && (mode & 1)) {
        // epilogue-like TMEM reads of the other accumulator (columns 256..)
        const uint32_t t0 = tmem + 256 + ((uint32_t)((warp & 3) * 32) << 16);
        float v[16], acc = 0.f;
        while (!stop) {
            for (int c = 0; c < 64; c += 16) {
                tmem_ld16(t0 + c, v);
                for (int i = 0; i < 16; ++i) acc += v[i];
            }
        }
        if (acc == 12345.f) out[1] = 1;
    } else if (warp >= 10 && (mode & 2)) {
        // converter-like smem traffic on a separate buffer
        float4 *p = reinterpret_cast<float4 *>(side);
        const int t = tid - 320;
        float4 acc = make_float4(0, 0, 0, 0);
        while (!stop) {
            for (int j = t; j < 4096; j += 256) {
                const float4 x = p[j];
                acc.x += x.x;
                p[(j + 7) & 4095] = make_float4(x.y, x.z, x.w, acc.x);
            }
        }
        if (acc.x == 12345.f) out[1] = 2;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc_rt(tmem, 512);
}

int main()
{
    long long *d;
    cudaMalloc(&d, 2 * sizeof(long long));
    const size_t smem = 148 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 1800;
    const char *names[8] = {"alone", "+ TMEM loads", "+ smem traffic", "+ both",
                            "units", "units + TMEM", "units + smem", "units + both"};
    for (int np : {16, 32})
        for (int mode = 0; mode < 8; ++mode) {
            probe<<<1, NT, smem>>>(np, reps, mode, d);
            if (cudaDeviceSynchronize() != cudaSuccess) {
                printf("error np=%d mode=%d\n", np, mode);
                return 1;
            }
            long long c;
            cudaMemcpy(&c, d, sizeof c, cudaMemcpyDeviceToHost);
            printf("np=%3d %-15s: %6.1f clk per K=16 step (2 MMAs)\n", np, names[mode], (double)c / reps);
        }
    return 0;
}
