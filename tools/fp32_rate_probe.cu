// FP32 issue-rate probe (diagnostic): packed FADD2 / FFMA2 vs scalar FADD /
// FFMA throughput per SM on this B200, at 4 and 8 warps per SMSP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_rate_probe tools/fp32_rate_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;

template <int MODE>
__global__ void probe(float *out, int iters, float s)
{
    // 8 independent chains per thread
    float a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
    u64 p[8];
    for (int i = 0; i < 8; ++i) asm("mov.b64 %0, {%1, %2};" : "=l"(p[i]) : "f"(a[2 * i]), "f"(a[2 * i + 1]));
    u64 ss, zz;
    asm("mov.b64 %0, {%1, %1};" : "=l"(ss) : "f"(s));
    asm("mov.b64 %0, {%1, %1};" : "=l"(zz) : "f"(s * 0.0f));
    u64 q[8], r[8];
    for (int i = 0; i < 8; ++i) {
        asm("mov.b64 %0, {%1, %2};" : "=l"(q[i]) : "f"(a[i] + 1), "f"(a[i] + 2));
        asm("mov.b64 %0, {%1, %2};" : "=l"(r[i]) : "f"(a[i] + 3), "f"(a[i] + 4));
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (MODE == 0) {  // FADD2
#pragma unroll
                for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(ss));
            } else if (MODE == 1) {  // FFMA2
#pragma unroll
                for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[i]) : "l"(ss));
            } else if (MODE == 4) {  // FFMA2 with distinct pair operands (q, r per chain)
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(q[i]), "l"(r[(i + 3) & 7]));
            } else if (MODE == 5) {  // FADD2 with distinct pair operands
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(q[(i + 5) & 7]));
            } else if (MODE == 6) {  // solver-like: 13-op dependent chain per pair, 8 pairs
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    u64 g, d, m;
                    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(g) : "l"(p[i]), "l"(ss), "l"(q[(i + 1) & 7]));
                    asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(g) : "l"(q[(i + 2) & 7]));
                    asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(g) : "l"(p[(i + 1) & 7]));
                    asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(g) : "l"(p[(i + 7) & 7]));
                    asm volatile("sub.rn.f32x2 %0, %0, %1;" : "+l"(g) : "l"(r[i]));
                    asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(p[i]), "l"(r[(i + 1) & 7]));
                    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(d) : "l"(r[(i + 2) & 7]), "l"(zz));
                    asm volatile("sub.rn.f32x2 %0, %1, %0;" : "+l"(g) : "l"(d));
                    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(g) : "l"(ss), "l"(zz));
                    asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(p[i]), "l"(q[i]));
                    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(m) : "l"(ss), "l"(zz));
                    asm volatile("sub.rn.f32x2 %0, %1, %0;" : "+l"(g) : "l"(p[i]));
                    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(q[i]) : "l"(g), "l"(m));
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) { u64 t = p[i]; p[i] = q[i]; q[i] = t; }
            } else if (MODE == 7) {  // one dependent FADD2 chain (latency)
#pragma unroll
                for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[0]) : "l"(ss));
            } else if (MODE == 8) {  // one dependent FFMA2 chain (latency)
#pragma unroll
                for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[0]) : "l"(ss));
            } else if (MODE == 9) {  // one dependent scalar FADD chain (latency)
#pragma unroll
                for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[0]) : "f"(s));
            } else if (MODE == 2) {  // scalar FADD, 16 chains
#pragma unroll
                for (int i = 0; i < 16; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(s));
            } else {  // scalar FFMA
#pragma unroll
                for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(a[i]) : "f"(s));
            }
        }
    }
    float acc = 0;
    for (int i = 0; i < 8; ++i) {
        float l, h;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(l), "=f"(h) : "l"(p[i]));
        acc += l + h;
    }
    for (int i = 0; i < 16; ++i) acc += a[i];
    for (int i = 0; i < 8; ++i) {
        float l, h;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(l), "=f"(h) : "l"(q[i]));
        acc += l + h;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(l), "=f"(h) : "l"(r[i]));
        acc += l + h;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
static void run(const char *name, int threads)
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, (size_t)nsm * threads * 4 * sizeof(float));
    const int iters = 4000;
    probe<MODE><<<nsm, threads>>>(out, 10, 1.0f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<MODE><<<nsm, threads>>>(out, iters, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const bool packed = MODE <= 1 || (MODE >= 4 && MODE != 9);
    const double per = MODE == 6 ? 13.0 * 8 : (MODE >= 7 ? 8.0 : (packed ? 8.0 : 16.0));
    const double lanes_ops = (packed ? 2.0 : 1.0) * per * 8 * iters;       // fp32 results per thread
    const double warp_instr = per * 8 * iters;                             // per warp
    const double cycles = ms * 1e-3 * clk * 1e3;
    const int warps = threads / 32;
    printf("%-6s threads=%4d: %.3f ms, %.1f fp32 results/clk/SM, %.2f clk per warp-instr per SMSP\n",
           name, threads, ms, lanes_ops * threads / cycles, cycles / (warp_instr * warps / 4));
    cudaFree(out);
}

int main()
{
    run<7>("LAT-FADD2", 32);
    run<8>("LAT-FFMA2", 32);
    run<9>("LAT-FADD", 32);
    for (int t : {128, 256, 512}) {
        run<0>("FADD2", t);
        run<1>("FFMA2", t);
        run<2>("FADD", t);
        run<3>("FFMA", t);
        run<4>("FFMA2q", t);
        run<5>("FADD2q", t);
        run<6>("SGD", t);
    }
    return 0;
}
