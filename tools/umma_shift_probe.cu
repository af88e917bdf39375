// Probe: does a tcgen05 SWIZZLE_128B K-major A descriptor whose start address
// is shifted by whole 128-byte rows (and whose SBO is not a multiple of
// 1024 B) read the rows TMA wrote?  Decides the shifted-view (halo tile)
// design of the conv kernel.  Standalone: nvcc -arch=sm_100a ... && ./probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2301_00750_b200/csrc/tc_common.cuh"

using namespace ss::tc;

// layout: 2 = SWIZZLE_128B, 4 = SWIZZLE_64B, 6 = SWIZZLE_32B
__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t sbo, uint32_t base_off, uint32_t layout)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(base_off & 7) << 49;
    d |= (uint64_t)layout << 61;
    return d;
}

__global__ void probe(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tw,
                      int shift, int sbo_rows, int base_mode, int rowb, float *out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *base = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t *xs = base;               // 256 rows x 128 B
    uint8_t *ws = base + 256 * 128;   // 32 rows x 128 B
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_init(&mbar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc_rt(&tslot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        mbar_expect_tx(&bar, 256 * rowb + 32 * 128);
        tma_tile_2d(smem_u32(xs), &tx, 0, 0, &bar);
        tma_tile_2d(smem_u32(ws), &tw, 0, 0, &bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (tid == 0) {
        const uint32_t a0 = smem_u32(xs) + shift * rowb;
        const uint32_t bo = base_mode ? ((a0 >> 7) & 7) : 0;
        const uint32_t id = idesc(2u, 128u, 32u);
        const uint32_t lay = rowb == 128 ? 2 : (rowb == 64 ? 4 : 6);
        const int ks = rowb / 32;  // K = 8 steps per row
        for (int i = 0; i < ks; ++i)
            mma_tf32(tmem, desc_sw(a0 + i * 32, sbo_rows * rowb, bo, lay),
                     desc_sw(smem_u32(ws) + i * 32, 1024, 0, 2), id, i > 0);
        mma_commit(&mbar);
    }
    mbar_wait(&mbar, 0);
    tc_fence_after();
    float v[16];
    const uint32_t t0 = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 32; c += 16) {
        tmem_ld16(t0 + c, v);
        for (int i = 0; i < 16; ++i) out[(warp * 32 + (tid & 31)) * 32 + c + i] = v[i];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc_rt(tmem, 32);
}

static PFN_cuTensorMapEncodeTiled_v12000 enc()
{
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

int main()
{
    const int R = 256;
    std::vector<float> X(R * 32), W(32 * 32, 0.f);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < 32; ++c) X[r * 32 + c] = r + 0.25f * c;
    for (int rowb : {128, 64, 32}) {
    const int cpp = rowb / 4;
    for (int n = 0; n < 32; ++n) W[n * 32 + n] = 1.f;  // B[n][k] = delta
    float *dx, *dw, *dout;
    cudaMalloc(&dx, X.size() * 4);
    cudaMalloc(&dw, W.size() * 4);
    cudaMalloc(&dout, 128 * 32 * 4);
    cudaMemcpy(dx, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap tx, tw;
    auto fn = enc();
    cuuint64_t dimx[2] = {32, (cuuint64_t)R}, strx[1] = {128};
    cuuint32_t boxx[2] = {(cuuint32_t)cpp, (cuuint32_t)R}, es[2] = {1, 1};
    fn(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dx, dimx, strx, boxx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       rowb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (rowb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t dimw[2] = {32, 32}, strw[1] = {128};
    cuuint32_t boxw[2] = {32, 32};
    fn(&tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dw, dimw, strw, boxw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    std::vector<float> out(128 * 32);
    const int shifts[] = {0, 1, 3, 8, 10, 17};
    const int sbos[] = {8, 9, 10, 17};
    for (int bm = 0; bm < 1; ++bm)
        for (int sbo : sbos)
            for (int sh : shifts) {
                probe<<<1, 128, 64 * 1024>>>(tx, tw, sh, sbo, bm, rowb, dout);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("err %s\n", cudaGetErrorString(e));
                    return 1;
                }
                cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
                int bad = 0;
                for (int m = 0; m < 128; ++m) {
                    const int row = sh + (m / 8) * sbo + m % 8;
                    for (int n = 0; n < cpp; ++n) {
                        const float want = row < R ? X[row * 32 + n] : 0.f;
                        if (row < R && out[m * 32 + n] != want) ++bad;
                    }
                }
                printf("rowb=%3d base_mode=%d sbo_rows=%2d shift=%2d : %s (%d bad)\n", rowb, bm, sbo, sh,
                       bad ? "MISMATCH" : "ok", bad);
            }
    }
    return 0;
}
