// Probe: does a 2-SM tcgen05 MMA (cta_group::2, M = 256) cost the same cycles
// per instruction as a 1-SM one (cta_group::1, M = 128) at the thin N of the
// 3xTF32 pyramid convs?  If so, a CTA-pair conv tile halves the
// per-pixel instruction count of the MMA-instruction-bound thin layers.
// Back-to-back kind::tf32 MMAs (K = 8) issued by one thread; operand contents
// are irrelevant.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma2_rate_probe tools/mma2_rate_probe.cu
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

__device__ __forceinline__ uint32_t cta_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// PAIR = 1: cluster of 2, M = 256 (cta_group::2, leader issues); 0: M = 128
template <int PAIR>
__global__ void probe(int N, int rowb, int reps, long long *out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *base = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t *as = base;              // 128 rows x rowb
    uint8_t *bs = base + 128 * 128;  // 256 rows x rowb
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = PAIR ? cta_rank() : 0;
    for (int i = tid; i < (128 * 128 + 256 * 128) / 4; i += blockDim.x) reinterpret_cast<float *>(base)[i] = 0.001f;
    if (tid == 0) {
        mbar_init(&mbar, 1);
        fence_barrier_init();
    }
    if (warp == 0) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                         "r"(256)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            tmem_alloc_rt(&tslot, 256);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    if (PAIR)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0 && rank == 0) {
        const uint32_t lay = rowb == 128 ? 2 : (rowb == 64 ? 4 : 6);
        const uint64_t ad = desc(smem_u32(as), 8 * rowb, lay), bd = desc(smem_u32(bs), 8 * rowb, lay);
        const uint32_t id = idesc(2u, PAIR ? 256u : 128u, (uint32_t)N);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            const uint32_t acc = r > 0 ? 1u : 0u;
            if (PAIR)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(id), "r"(acc)
                    : "memory");
            else
                mma_tf32(tmem, ad, bd, id, acc);
        }
        if (PAIR)
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&mbar)),
                "h"((uint16_t)3)
                : "memory");
        else
            mma_commit(&mbar);
        mbar_wait(&mbar, 0);
        out[0] = clock64() - t0;
    }
    if (PAIR && tid == 0 && rank == 1) mbar_wait(&mbar, 0);  // the multicast commit reached the peer too
    tc_fence_before();
    if (PAIR)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else
        __syncthreads();
    if (warp == 0) {
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
        else
            tmem_dealloc_rt(tmem, 256);
    }
}

int main()
{
    long long *d;
    cudaMalloc(&d, sizeof(long long));
    const size_t smem = 64 * 1024;
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 999;
    printf("cycles per tcgen05.mma kind::tf32 (K = 8), %d back to back\n", reps);
    for (int rowb : {32, 64, 128})
        for (int N : {16, 32, 48, 64, 128, 256}) {
            double clk[2];
            for (int pair = 0; pair < 2; ++pair) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(pair ? 2 : 1);
                cfg.blockDim = dim3(128);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = pair ? 2 : 1;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaError_t e = pair ? cudaLaunchKernelEx(&cfg, probe<1>, N, rowb, reps, d)
                                     : cudaLaunchKernelEx(&cfg, probe<0>, N, rowb, reps, d);
                if (e == cudaSuccess) e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("error pair=%d N=%d rowb=%d: %s\n", pair, N, rowb, cudaGetErrorString(e));
                    return 1;
                }
                long long c;
                cudaMemcpy(&c, d, sizeof c, cudaMemcpyDeviceToHost);
                clk[pair] = (double)c / reps;
            }
            printf("rowb=%3d N=%3d : 1-SM M=128 %6.1f clk  | 2-SM M=256 %6.1f clk  -> per-SM rows/clk %.2f vs %.2f\n",
                   rowb, N, clk[0], clk[1], 128.0 / clk[0], 128.0 / clk[1]);
        }
    return 0;
}
