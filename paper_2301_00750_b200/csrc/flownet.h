// Lite flow network: kernel launchers and the native runner (see
// paper_2301_00750_b200/liteflownet.py for the architecture table).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <tuple>
#include <utility>
#include <vector>

namespace ss {
namespace fn {

// Programmatic dependent launch (PDL) for the network's kernel chain: every
// kernel is launched with programmatic stream serialization, triggers its
// dependents on entry and waits (griddepcontrol.wait) before its first
// global-memory access, so a kernel's launch and prologue (barrier init, TMEM
// allocation, tensor-map prefetch) overlap the tail of the previous one.
// SS_FLOW_PDL=0 launches them plainly.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif
bool pdl_enabled();
int pdl_status(cudaError_t e, const char *what);

template <typename... KArgs, typename... Args>
int launch_pdl(const char *name, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
               cudaStream_t st, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return pdl_status(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...), name);
}

struct ConvParams {
    const float *in;
    int in_ld, H, W, Cin;       // input NHWC slice (Cin % 4 == 0, 16-byte aligned)
    const float *wgt, *bias;    // wgt [k*k*Cin][Cout_pad], bias [Cout_pad]
    int Cout, Cout_pad;
    float *out;
    int out_ld, Ho, Wo;
    int k, stride, dil, pad, act;
    float *ws = nullptr;        // split-K workspace (tensor-core path), may be null
    size_t ws_floats = 0;
    int k_per_split = 0;        // set by the launcher
    int grid_cap = 0;           // > 0: at most this many CTAs (persistent kernels)
    int n_full = 0, n_off = 0;  // N-split (set by the launcher): weight rows [n_off, n_off + Cout_pad)
    const void *tmB = nullptr;  // TMA weight map (CUtensorMap, flownet_tma.cu), fp32 path
    int tma_T = 1;              // taps per weight stage of that map
};

enum ConvMode { CONV_TC_BF16 = 1, CONV_TC_TF32X3 = 2, CONV_TC_BF16X2 = 3 };

// kind 0: bf16 operands (kind::f16); kind 1: 3xTF32 (kind::tf32)
// TMA-fed warp-specialised 3xTF32 conv (flownet_tma.cu)
int launch_conv_tma(const ConvParams &p, int prec, cudaStream_t st);
void conv_trace_dump(const char *what);  // SS_CONV_TRACE diagnostics  // prec: 1 3xTF32, 0 bf16
int prepare_conv_tma();
int prepare_flow_kernels();
int encode_weight_map(CUtensorMap *m, const float *wt, int kblocks, int rows, int np, int T);
int tma_taps_per_stage(int k, int stride, int dil, int cin, int np, int prec);
int encode_weight_map_bf16(CUtensorMap *m, const void *wt, int kblocks, int rows, int np, int T);
int encode_weight_map_bf16_rows(CUtensorMap *m, const void *wt, int kblocks, int rows, int box_rows, int T);
int launch_splitk_reduce(const float *ws, int splits, int M, int N, int Cout, const float *bias,
                         int act, float *out, int out_ld, cudaStream_t st, int parts = 1);
int launch_depthwise(const float *in, int ld_in, int H, int W, int C, const float *w, int dil,
                     float *out, int ld_out, cudaStream_t st);
int launch_prep_pyr1a(const float *img, int h, int w, int c, int H0, int W0, int H1, int W1, const float *wgt,
                      int cout_pad, const float *bias, float *out, cudaStream_t st);  // k_prep + pyr1a fused
int launch_prep(const float *img, int h, int w, int c, int H, int W, float *out, cudaStream_t st);
int launch_up2_warp(const float *coarse, int cld, int Hc, int Wc, const float *f2, int C, int H,
                    int W, float *x, int xld, float *w2, cudaStream_t st);
int launch_corr(const float *f1, const float *w2, int C, int H, int W, float *x, int xld,
                bool copy_f1, cudaStream_t st);
int launch_flow_final(const float *f3, int ld3, const float *r, int ldr, int Hc, int Wc, int h,
                      int w, float *uv, uint8_t *valid, cudaStream_t st);
// provider downscale: box_downscale of an HWC frame by f; resize of the
// network's flow back to the frame size, times s (FlowOptions.downscale)
int launch_box_down_hwc(const float *in, int w, int c, int f, int ho, int wo, float *out, cudaStream_t st);
int launch_upscale_flow(const float *in, int hi, int wi, int ho, int wo, float s, float *uv, uint8_t *valid,
                        cudaStream_t st);

struct LayerDev {
    int cin, cout, cout_pad, k, stride, dil, act;
    bool dw;
    float *w = nullptr, *b = nullptr;
    // TMA path (flownet_tma.cu): [kblock = cb * k*k + tap][part][hi np rows;
    // lo np rows][32 channels] fp32, its tensor map, taps per stage
    const float *wt_tma = nullptr;
    int tma_T = 1;
    alignas(64) CUtensorMap tmB;
    // bf16 path: [kblock][part][np rows][32 channels] bf16, map, taps per stage
    const void *wt_bf = nullptr;
    int tma_T_bf = 1;
    alignas(64) CUtensorMap tmB_bf;
    // split-bf16 path: [kblock][part][hi np rows; lo np rows][32 channels] bf16
    const void *wt_bs = nullptr;
    int tma_T_bs = 1;
    alignas(64) CUtensorMap tmB_bs;
};

// Weights on one device, in liteflownet.layer_table() order.
struct Weights {
    std::vector<LayerDev> layers;
    float *block = nullptr;
    float *tma_block = nullptr;
    void *bf_block = nullptr;
    void *bs_block = nullptr;
    ~Weights();
    static int expected_params();
    int upload(const float *host, int64_t n);
    const LayerDev &L(int i) const { return layers[i]; }
};

// Resolution-specific buffers + a 3-slot pyramid cache (slots follow the
// session's frame ring: the pyramid of a frame is computed once and reused by
// the two steps that see it as a neighbour and the one that sees it as I_t).
struct Run {
    const Weights *wts = nullptr;
    int conv_mode = CONV_TC_TF32X3;
    // h, w: the network's frame; fh, fw: the caller's frame (fh / ds, fw / ds
    // = h, w with downscale ds: FlowOptions.downscale semantics)
    int h = 0, w = 0, H[7] = {0}, W[7] = {0};
    int fh = 0, fw = 0, ds = 1;
    float *small = nullptr, *uv_small = nullptr;
    float *prep = nullptr, *s0 = nullptr, *s1 = nullptr;
    struct Slot {
        int64_t key = -1;
        float *lvl[7] = {nullptr};
    } slots[3];
    // estimator / refinement buffers of the flow being computed (one set per
    // concurrently running flow; select_set points these at a set)
    float *x[7] = {nullptr}, *e1[7] = {nullptr}, *e2[7] = {nullptr}, *E[7] = {nullptr},
          *w2[7] = {nullptr};
    float *ra = nullptr, *rb = nullptr, *rr = nullptr;
    float *ws = nullptr;  // split-K partial sums
    size_t ws_floats = 0;
    struct EstBufs {
        float *x[7], *e1[7], *e2[7], *E[7], *w2[7];
        float *ra, *rb, *rr, *ws;
    } sets[2];
    int nsets = 1;
    std::vector<void *> allocs;
    // CUDA graphs (sessions: every buffer is fixed per ring slot, so the
    // ~60 launches of a pyramid / flow replay as one graph launch)
    bool use_graphs = false;
    // graph and its kernel-node count
    std::map<std::tuple<int, const void *, int>, std::pair<cudaGraphExec_t, long>> pyr_graphs;
    std::map<std::tuple<int, int, void *, void *, int>, std::pair<cudaGraphExec_t, long>> flow_graphs;
    ~Run();
    int init(const Weights *w, int h, int w_, int nsets = 1, int downscale = 1);
    // pyramid of img (h, w, c) into slot (skipped if key matches)
    int pyramid(int slot, int64_t key, const float *img, int c, cudaStream_t st);
    // flow from the frame in slot a toward the frame in slot b (both computed),
    // using estimator buffer set `set` (two flows may run concurrently on two
    // streams with different sets)
    int flow(int a, int b, float *uv, uint8_t *valid, cudaStream_t st, int set = 0);
    void select_set(int set);
    // average device time (CUDA events) of `reps` launches of the first
    // estimator conv at `level` on this run's buffers (roofline measurement)
    int time_est1(int level, int reps, cudaStream_t st, float *ms, double *flops);

  private:
    int pyramid_impl(int slot, const float *img, int c, cudaStream_t st);
    int flow_impl(int a, int b, float *uv, uint8_t *valid, cudaStream_t st);
};

}  // namespace fn
}  // namespace ss
