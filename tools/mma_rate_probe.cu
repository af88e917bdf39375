// Probe: cycles per tcgen05.mma kind::tf32 (cta_group::1) issued back to back
// by one elected thread, as a function of M, N and the A row width / swizzle
// mode -- is a thin MMA bound by a fixed per-instruction cost or by reading A
// from shared memory?  (Decides whether a 2-SM cta_group::2 tile can speed up
// the thin 3xTF32 conv layers.)  Operand contents are irrelevant here.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_rate_probe tools/mma_rate_probe.cu -lcuda
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2301_00750_b200/csrc/tc_common.cuh"

using namespace ss::tc;

// layout: 2 = SWIZZLE_128B, 4 = SWIZZLE_64B, 6 = SWIZZLE_32B; K-major rows of rowb bytes
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

__global__ void probe(int M, int N, int rowb, int reps, long long *out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *base = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t *as = base;              // 128 rows x rowb
    uint8_t *bs = base + 128 * 128;  // 256 rows x rowb
    __shared__ uint64_t mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (128 * 128 + 256 * 128) / 4; i += blockDim.x) reinterpret_cast<float *>(base)[i] = 0.001f;
    if (tid == 0) {
        mbar_init(&mbar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc_rt(&tslot, 256);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        const uint32_t lay = rowb == 128 ? 2 : (rowb == 64 ? 4 : 6);
        const uint64_t ad = desc(smem_u32(as), 8 * rowb, lay), bd = desc(smem_u32(bs), 8 * rowb, lay);
        const uint32_t id = idesc(2u, (uint32_t)M, (uint32_t)N);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) mma_tf32(tmem, ad, bd, id, r > 0 ? 1u : 0u);
        mma_commit(&mbar);
        mbar_wait(&mbar, 0);
        long long t1 = clock64();
        out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc_rt(tmem, 256);
}

// the conv kernel's pattern: per K step an N = 2 np MMA (A = a_hi) and an
// N = np MMA (A = a_lo, accumulating into the first np columns), with A / B
// descriptors that change every step (9 shifted halo views x 9 weight taps)
__global__ void probe_conv(int np, int rowb, int reps, int vary, int sep, long long *out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *base = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t *ahi = base, *alo = base + 16 * 1024, *bs = base + 32 * 1024;  // 16 KB each, B 9 x 4 KB
    __shared__ uint64_t mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (32 * 1024 + 9 * 4096) / 4; i += blockDim.x) reinterpret_cast<float *>(base)[i] = 0.001f;
    if (tid == 0) {
        mbar_init(&mbar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc_rt(&tslot, 256);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        const uint32_t lay = rowb == 128 ? 2 : (rowb == 64 ? 4 : 6);
        const uint32_t id2 = idesc(2u, 128u, (uint32_t)(2 * np)), id1 = idesc(2u, 128u, (uint32_t)np);
        long long t0 = clock64();
        if (sep == 2) {  // grouped: the 9 a_hi MMAs of a "stage", then its 9 a_lo MMAs
            for (int r0 = 0; r0 < reps; r0 += 9) {
                for (int q = 0; q < 9; ++q) {
                    const int tap = vary ? q : 0;
                    const uint32_t off = vary ? (uint32_t)(((tap / 3) * 10 + tap % 3) * rowb) : 0u;
                    mma_tf32(tmem, desc(smem_u32(ahi) + off, 10 * rowb, lay), desc(smem_u32(bs) + tap * 4096, 1024, 2),
                             id2, (r0 + q) > 0 ? 1u : 0u);
                }
                for (int q = 0; q < 9; ++q) {
                    const int tap = vary ? q : 0;
                    const uint32_t off = vary ? (uint32_t)(((tap / 3) * 10 + tap % 3) * rowb) : 0u;
                    mma_tf32(tmem, desc(smem_u32(alo) + off, 10 * rowb, lay), desc(smem_u32(bs) + tap * 4096, 1024, 2),
                             id1, 1u);
                }
            }
        } else
        for (int r = 0; r < reps; ++r) {
            const int tap = vary ? r % 9 : 0;
            const uint32_t off = vary ? (uint32_t)(((tap / 3) * 10 + tap % 3) * rowb) : 0u;  // halo_w = 10
            const uint64_t ah = desc(smem_u32(ahi) + off, 10 * rowb, lay), al = desc(smem_u32(alo) + off, 10 * rowb, lay);
            const uint64_t bd = desc(smem_u32(bs) + tap * 4096, 1024, 2);
            mma_tf32(tmem, ah, bd, id2, r > 0 ? 1u : 0u);
            // sep 1: the a_lo product into its own columns [2 np, 3 np) (summed later)
            // sep 3: same shape (N = 2 np) into the same columns; 4: same shape, own columns
            if (sep == 3)
                mma_tf32(tmem, al, bd, id2, 1u);
            else if (sep == 4)
                mma_tf32(tmem + 2 * np, al, bd, id2, r == 0 ? 0u : 1u);
            else
                mma_tf32(sep ? tmem + 2 * np : tmem, al, bd, id1, (sep && r == 0) ? 0u : 1u);
        }
        mma_commit(&mbar);
        mbar_wait(&mbar, 0);
        out[0] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc_rt(tmem, 256);
}

int main()
{
    long long *d;
    cudaMalloc(&d, sizeof(long long));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int reps = 999;
    printf("cycles per tcgen05.mma.cta_group::1.kind::tf32 (K = 8), %d back to back\n", reps);
    for (int rowb : {32, 64, 128})
        for (int M : {64, 128})
            for (int N : {16, 32, 48, 64, 128, 256}) {
                probe<<<1, 128, 64 * 1024>>>(M, N, rowb, reps, d);
                if (cudaDeviceSynchronize() != cudaSuccess) {
                    printf("error M=%d N=%d rowb=%d\n", M, N, rowb);
                    return 1;
                }
                long long c;
                cudaMemcpy(&c, d, sizeof c, cudaMemcpyDeviceToHost);
                printf("rowb=%3d M=%3d N=%3d : %6.1f clk/MMA  (%5.1f MAC/clk)\n", rowb, M, N, (double)c / reps,
                       (double)M * N * 8 * reps / (double)c);
            }
    cudaFuncSetAttribute(probe_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    printf("conv pattern: per K step MMA(N = 2 np, a_hi) + MMA(N = np, a_lo)\n");
    for (int rowb : {64})
    for (int np : {16, 32, 64})
        for (int sep : {0, 1, 2, 3, 4})
        for (int vary : {0, 1}) {
            probe_conv<<<1, 128, 80 * 1024>>>(np, rowb, reps, vary, sep, d);
            if (cudaDeviceSynchronize() != cudaSuccess) {
                printf("error conv np=%d\n", np);
                return 1;
            }
            long long c;
            cudaMemcpy(&c, d, sizeof c, cudaMemcpyDeviceToHost);
            printf("rowb=%3d np=%3d %s descriptors %s: %6.1f clk per K step (2 MMAs)\n", rowb, np,
                   sep == 2 ? "grouped     " : sep == 1 ? "separate acc" : sep == 3 ? "same shape  " : sep == 4 ? "same+sepacc " : "interleaved ", vary ? "varying" : "fixed  ", (double)c / reps);
        }
    return 0;
}
