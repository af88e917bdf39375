// Built-in DIS-style flow estimator on B200 (flow.py:168-325); see dis.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <tuple>
#include <utility>
#include <vector>

namespace ss {
namespace dis {

struct Options {  // FlowOptions (flow.py:27-42)
    int levels = 5, patch = 9, iters = 4, downscale = 1;
};

struct Estimator {
    int h = 0, w = 0;
    Options opts;
    std::vector<int> lh, lw;             // pyramid shapes (level 0 = finest working level)
    std::vector<float *> g1, g2;         // box pyramids of the two luma images
    float *ga = nullptr, *gb = nullptr, *tmp = nullptr;
    float *uvA = nullptr, *uvB = nullptr, *full = nullptr;
    float *du = nullptr, *dv = nullptr, *du2 = nullptr, *dv2 = nullptr;
    float *gu = nullptr, *gv = nullptr, *gu2 = nullptr, *gv2 = nullptr;
    float *lum1 = nullptr, *lum2 = nullptr;
    std::vector<void *> allocs;
    // one CUDA graph per (frames, outputs) pointer set: a flow is ~60 short
    // kernels whose eager launches would otherwise pace the GPU
    std::map<std::tuple<const float *, const float *, int, float *, uint8_t *>,
             std::pair<cudaGraphExec_t, long>>
        graphs;
    bool warmed = false;
    bool use_graphs = false;  // sessions only: their pointer sets are few and fixed
    ~Estimator();
    int init(int h, int w, const Options &o);
    // flow from frame a toward frame b ((h, w, c) float32 device) into
    // uv (h, w, 2) and valid (h, w) (may be null)
    int run(const float *fa, const float *fb, int c, float *uv, uint8_t *valid, cudaStream_t st);
    int run_impl(const float *fa, const float *fb, int c, float *uv, uint8_t *valid, cudaStream_t st);
};

}  // namespace dis
}  // namespace ss
