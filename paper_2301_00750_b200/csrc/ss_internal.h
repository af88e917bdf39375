// Internal (non-ABI) interfaces between the streamstab B200 translation units.
#pragma once

#include <functional>

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/streamstab_b200.h"

namespace ss {

struct PresolveArgs {
    int h, w;
    const float *I_prev, *P_prev, *I_cur, *P_cur, *I_next, *P_next, *O_prev;  // HWC
    const float *uv_prev, *uv_next;                                             // (H, W, 2)
    const uint8_t *valid_prev, *valid_next;                                     // may be null
    ss_params p;
    float *A, *lapP, *wc;   // planar solver inputs
    float *wp_out, *wn_out; // optional diagnostics (may be null)
};

int launch_backward_warp(const float *img, int h, int w, int c, const float *uv,
                         const uint8_t *valid, float *out, float *mask, cudaStream_t st);
int launch_occlusion(const float *fuv, const uint8_t *fvalid, const float *buv,
                     const uint8_t *bvalid, int h, int w, float *out, cudaStream_t st);
int launch_warp_weight(const float *ref, const float *warped, long n, int c, float alpha,
                       float bound, const float *validity, float *out, cudaStream_t st);
int launch_local_blend(const float *cur, const float *prev, const float *next, const float *wp,
                       const float *wn, long n, int c, float *out, cudaStream_t st);
int launch_adaptive_blend(const float *g, const float *l, const float *wp, long n, int c,
                          float *out, cudaStream_t st);
int launch_consistency_weight(const float *cur, const float *blended, long n, int c, float alpha,
                              float lam, float *out, cudaStream_t st);
int launch_laplacian(const float *img, int h, int w, int c, float *out, bool planar,
                     cudaStream_t st);
int launch_hwc_to_planar(const float *src, int h, int w, int c, float *dst, cudaStream_t st);
int launch_presolve(const PresolveArgs &a, int ci, int cp, bool with_next, cudaStream_t st);
// metrics.cu: sums[0] = sum(mask * per_pixel), sums[1] = sum(mask) (device, float64)
int launch_warping_error(const float *fa, const float *fb, int h, int w, int c, const float *fuv,
                         const uint8_t *fvalid, const float *buv, const uint8_t *bvalid,
                         double *sums, cudaStream_t st);
// scratch: 7 * h * w doubles; *sum (device) = sum of the cropped SSIM map
int launch_ssim(const float *a, const float *b, int h, int w, int c, double *scratch,
                double *sum, cudaStream_t st);

// numpy pairwise-sum tree for n elements (see solver.cu)
struct PairwisePlan {
    long n = 0;
    int C = 0;
    long hw = 0;
    int n_leaves = 0, n_nodes = 0;
    std::vector<int> group_off;  // internal-node groups by height
    int64_t *d_leaf_start = nullptr;
    int32_t *d_leaf_len = nullptr;
    int32_t *d_left = nullptr, *d_right = nullptr;
    float *d_vals = nullptr;
    ~PairwisePlan();
    void release();
    int build(long hw, int C);
};

// Device work buffers for the screened-Poisson solve of an (h, w, c) image.
struct SolverWork {
    int h = 0, w = 0, c = 0;
    float *O[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [set][cur/prev] planar
    unsigned *maxbits = nullptr;  // per-iteration max |x| bit pattern
    int maxiters = 0;
    float *sums = nullptr;        // exact pairwise sums (replay path)
    int *h_result = nullptr;      // pinned: [first_gray_iter, first_nonfinite_iter]
    unsigned *h_maxbits = nullptr;      // mapped pinned readback of the per-pass maxima
    unsigned *d_maxbits_map = nullptr;  // its device alias
    int *d_result = nullptr;
    PairwisePlan plan;
    int *mp_flags = nullptr;  // solver "mp": item counter + per-(pass, channel, tile row) counts
    size_t mp_flags_n = 0;
    ~SolverWork();
    int ensure(int h, int w, int c, int iterations);
};

// Run params->iterations SGD-momentum updates of consistency.py:281-294 from
// O = O_prev = A (init == target) or from init, on planar A / lapP / wc, then
// write clamp(O, 0, 1) as HWC into out.  Synchronises st.  Returns
// SS_SOLVER_DIVERGENCE with *div_iter set exactly as the reference would.
// after_enqueue (optional) runs once the solve is enqueued (done_ev recorded),
// before the host waits for it.
int solve_planar(SolverWork &wk, const float *A, const float *init_planar, const float *lapP,
                 const float *wc, const ss_params &p, float *out_hwc, int *div_iter,
                 cudaStream_t st, cudaEvent_t done_ev = nullptr,
                 const std::function<int()> &after_enqueue = {});

int solver_variant();  // 0 = streaming, 1 = temporally blocked (env SS_SOLVER)

}  // namespace ss
