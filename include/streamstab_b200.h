/*
 * streamstab_b200.h -- C ABI of the B200-native per-frame temporal-consistency
 * step (arXiv 2301.00750; reference package `streamstab`).
 *
 * The reference is pure Python/numpy and has no FFI; each entry point below
 * replaces one reference function (cited file:line under
 * /root/reference/pkg/src/streamstab/) and is what the reference's Python
 * layer binds through ctypes.  Plain pointers and sizes
 * only: no torch types.  All device work is ordered on the caller's
 * cudaStream_t (passed as void*; NULL = legacy default stream) or, for
 * sessions, on the session's stream.
 *
 * Layouts (reference boundary, imgio.py:33-46, :154-192):
 *   frame  float32 (H, W, C) interleaved, C in {1, 3}
 *   flow   float32 (H, W, 2) with u = horizontal, v = vertical, plus a
 *          uint8 (H, W) validity map (1 = valid)
 *   maps   float32 (H, W)  (weights, masks)
 *
 * Status codes map 1:1 onto the reference's exceptions:
 *   SS_RESOLUTION_MISMATCH -> flow.ResolutionMismatch   (flow.py:23)
 *   SS_VALUE_ERROR         -> ValueError
 *   SS_SOLVER_DIVERGENCE   -> consistency.SolverDivergence(iteration)
 */
#ifndef STREAMSTAB_B200_H
#define STREAMSTAB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 1

#if defined(__GNUC__)
#define SS_API __attribute__((visibility("default")))
#else
#define SS_API
#endif

enum ss_status {
    SS_OK = 0,
    SS_RESOLUTION_MISMATCH = 1,
    SS_VALUE_ERROR = 2,
    SS_SOLVER_DIVERGENCE = 3,
    SS_CUDA_ERROR = 4,
    SS_NO_MEMORY = 5,
};

/* One stream's device-resident state (see the session section below). */
typedef struct ss_session ss_session;

enum ss_where { SS_HOST = 0, SS_DEVICE = 1 };
enum ss_dtype { SS_F32 = 0, SS_U8 = 1 };

/* ConsistencyParams (consistency.py:37-51), cast to float32 exactly where the
 * reference casts with np.float32 (consistency.py:149, :207, :270-271). */
typedef struct ss_params {
    float k1, k2, alpha, lam, eta, kappa;
    int32_t iterations;
    int32_t flow_downscale;
} ss_params;

/* StepTiming (consistency.py:298-303) plus the fused pre-solve stage; device
 * time measured with CUDA events on the session stream. */
typedef struct ss_timing {
    float flow_ms;
    float warp_blend_ms;
    float solve_ms;
} ss_timing;

/* ---- library ------------------------------------------------------------ */
SS_API int ss_abi_version(void);
/* Number of GPU kernels this library has launched in this process (graph
 * replays count their kernels); a diagnostic for benchmarks. */
SS_API long long ss_kernel_launches(void);
SS_API const char *ss_status_string(int status);
/* Last error text of the calling thread (empty string if none). */
SS_API const char *ss_last_error(void);
/* Select the CUDA device for the calling thread; checks it is sm_100. */
SS_API int ss_init(int device);
/* ConsistencyParams.validate (consistency.py:53-69). */
SS_API int ss_params_validate(const ss_params *p);

/* ---- stateless ops on device pointers (stream-ordered) ------------------ */
/* backward_warp (flow.py:102-127).  mask may be NULL. */
SS_API int ss_backward_warp(const float *img, int h, int w, int c, const float *uv,
                     const uint8_t *valid, float *out, float *mask, void *stream);
/* occlusion_mask (flow.py:130-153); bit-exact with the reference. */
SS_API int ss_occlusion_mask(const float *fwd_uv, const uint8_t *fwd_valid, const float *bwd_uv,
                      const uint8_t *bwd_valid, int h, int w, float *out, void *stream);
/* warp_weight (consistency.py:133-154).  validity may be NULL. */
SS_API int ss_warp_weight(const float *ref, const float *warped, int h, int w, int c, float alpha,
                   float bound, const float *validity, float *out, void *stream);
/* local_blend / input_blend (consistency.py:157-182). */
SS_API int ss_local_blend(const float *cur, const float *prev, const float *next, const float *wp,
                   const float *wn, int h, int w, int c, float *out, void *stream);
/* adaptive_blend (consistency.py:190-195). */
SS_API int ss_adaptive_blend(const float *global_img, const float *local_img, const float *wp, int h,
                      int w, int c, float *out, void *stream);
/* consistency_weight (consistency.py:198-208). */
SS_API int ss_consistency_weight(const float *cur, const float *blended, int h, int w, int c,
                          float alpha, float lam, float *out, void *stream);
/* laplacian (consistency.py:211-227). */
SS_API int ss_laplacian(const float *img, int h, int w, int c, float *out, void *stream);
/* solve_screened_poisson (consistency.py:253-295).  init may equal target.
 * Synchronises the stream to report divergence; on SS_SOLVER_DIVERGENCE
 * *div_iter holds the 1-based iteration the reference would raise with. */
SS_API int ss_solve_screened_poisson(const float *processed, const float *target, const float *wc,
                              int h, int w, int c, const ss_params *p, const float *init,
                              float *out, int *div_iter, void *stream);

/* ---- built-in DIS flow (estimate_flow, flow.py:168-325) --- */
/* FlowOptions (flow.py:27-42): levels >= 1, odd patch >= 3, iterations per
 * level, downscale in {1, 2, 4}.  Flow from frame_a toward frame_b ((h, w, c)
 * float32 device pointers) into uv (h, w, 2) / valid (h, w) (may be NULL).
 * Scratch is per host thread; consecutive calls of one thread on different
 * streams are ordered (the later call waits for the earlier one's work). */
SS_API int ss_dis_flow(const float *frame_a, const float *frame_b, int h, int w, int c,
                       int levels, int patch, int iters, int downscale, float *uv,
                       uint8_t *valid, void *stream);
/* BuiltinFlow inside a session: flow slot `which` (0: t -> t-1, 1: t -> t+1). */
SS_API int ss_session_compute_dis_flow(ss_session *s, int which, int levels, int patch,
                                       int iters, int downscale);

/* ---- evaluation metrics -------------------------- */
/* warping_error_pair (metrics.py:107-128) on device frames / flows:
 * sums_host[0] = sum(mask * mean_c |a - warp(b)|), sums_host[1] = sum(mask),
 * mask = occlusion_mask(fwd, bwd) * backward_warp mask; float64 sums.
 * Synchronises the stream. */
SS_API int ss_warping_error_sums(const float *frame_a, const float *frame_b, int h, int w, int c,
                                 const float *fwd_uv, const uint8_t *fwd_valid,
                                 const float *bwd_uv, const uint8_t *bwd_valid,
                                 double *sums_host, void *stream);
/* ssim (metrics.py:75-104): luma, 11x11 Gaussian sigma 1.5, reflect borders,
 * valid-window mean, float64.  Synchronises the stream. */
SS_API int ss_ssim(const float *a, const float *b, int h, int w, int c, double *out_host,
                   void *stream);

/* ---- sessions: SessionState + stabilize_step (consistency.py:306-413) ---- */

/* One stream's device-resident state: the (t-1, t, t+1) ring of
 * (input, processed) pairs, O_{t-1}, flows and solver buffers.  stream may be
 * NULL (the session creates its own non-blocking stream). */
SS_API int ss_session_create(int h, int w, int c_in, int c_proc, void *stream, ss_session **out);
SS_API int ss_session_destroy(ss_session *s);
SS_API int ss_session_reset(ss_session *s);
/* SessionState.push_pair (consistency.py:321-340).  I has c_in channels, P
 * has c_proc; dtype SS_U8 frames are normalised by 1/255 (imgio.py:132). */
SS_API int ss_push_pair(ss_session *s, int64_t position, const void *I, const void *P, int dtype,
                 int where);
/* Position the next step will solve (solved_through + 1) and the state. */
/* Stage the next (I, P) pair: its host->device copy runs on a copy stream
 * while the session computes; a later ss_push_pair with the same position and
 * the same I / P pointers swaps the staged buffers into the ring instead of
 * copying.  float32 only; the host buffers must stay valid until that push. */
SS_API int ss_stage_pair(ss_session *s, int64_t position, const void *I, const void *P, int dtype,
                         int where);
SS_API int64_t ss_solved_through(const ss_session *s);
/* Assign SessionState.solved_through / prev_output (the reference's dataclass
 * fields, consistency.py:305-319, read by _snippet :342-345): resume a stream
 * from a known O_{t-1}.  mode SS_STATE_POSITION sets solved_through only;
 * SS_STATE_OUTPUT also uploads prev_output (H, W, c_proc; dtype / where as
 * ss_push_pair); SS_STATE_CLEAR sets prev_output = None (the next push pins
 * it to that pair's processed frame, :338-340). */
#define SS_STATE_POSITION 0
#define SS_STATE_OUTPUT 1
#define SS_STATE_CLEAR 2
SS_API int ss_session_set_state(ss_session *s, int mode, int64_t solved_through, const void *prev_output,
                                int dtype, int where);
SS_API int ss_pending(const ss_session *s, int64_t *t, int *has_prev, int *has_next);
/* Provide the flows for the pending step t: which = 0 -> flow t->t-1,
 * which = 1 -> flow t->t+1 (FlowProvider.flow_between, flow.py:353-358,
 * called at consistency.py:380, :384).  valid may be NULL (all valid). */
SS_API int ss_set_flow(ss_session *s, int which, const float *uv, const uint8_t *valid, int where);
/* Fill a flow slot with ConstantFlow(u, v) (flow.py:406-425) on device. */
SS_API int ss_set_constant_flow(ss_session *s, int which, double u, double v, int steps);
/* _snippet checks only (consistency.py:342-353): SS_OK if a step with
 * with_next could run now, else SS_VALUE_ERROR with the reference's message;
 * *t receives the position that would be solved. */
SS_API int ss_check_step(const ss_session *s, int with_next, int64_t *t);
/* stabilize_step (with_next = 1) / stream_end_step (with_next = 0)
 * (consistency.py:356-413).  On SS_SOLVER_DIVERGENCE the state is not
 * advanced and *div_iter is set. */
SS_API int ss_step(ss_session *s, int with_next, const ss_params *p, int *div_iter);
/* Copy O_{solved_through} (the last output, or P_1 after the first push). */
SS_API int ss_output(const ss_session *s, void *dst, int dtype, int where);
/* Device pointer of the current output (H, W, c_proc) float32; valid until
 * the next ss_step / ss_push_pair. */
/* Asynchronous output: enqueue the copy of O_t (as ss_output) on a copy
 * stream and return; it overlaps the next step (the next solver that would
 * overwrite O_t's buffer waits for it).  dst must stay valid until
 * ss_output_wait returns or the next ss_output_async call (which waits for
 * the previous copy first). */
SS_API int ss_output_async(ss_session *s, void *dst, int dtype, int where);
SS_API int ss_output_wait(ss_session *s);
SS_API const float *ss_output_device(const ss_session *s);
SS_API int ss_last_timing(const ss_session *s, ss_timing *t);
/* Copy the flows used by the last step (for feeding back into the
 * reference's FloDirFlow / FlowProvider seam). */
SS_API int ss_flows(const ss_session *s, int which, float *uv_dst, uint8_t *valid_dst, int where);

/* ---- lite flow network (north star (a); architecture in liteflownet.py) --- */
typedef struct ss_flownet ss_flownet;
/* Number of float32 parameters the network expects (liteflownet.n_params). */
SS_API int64_t ss_flownet_num_params(void);
/* Upload weights (host float32, liteflownet.flatten_weights layout) to the
 * current device.  precision: SS_FLOW_FP32 (fp32-class products on tcgen05
 * tensor cores: split-bf16 -- x = hi + lo in bf16, three products, fp32
 * accumulation -- on the 3x3 stride-1 layers, 3xTF32 on the others;
 * SS_FP32_IMPL=tf32x3 selects 3xTF32 everywhere) or SS_FLOW_BF16 (tcgen05,
 * bf16 operands, fp32 accumulation). */
enum ss_flow_precision { SS_FLOW_FP32 = 0, SS_FLOW_BF16 = 1 };
SS_API int ss_flownet_create(const float *weights, int64_t n, int precision, ss_flownet **out);
/* Provider downscale (replaces FlowOptions.downscale, flow.py:34, :183-188,
   for this provider): the network runs on box_downscale(frame, d) and its
   flow is resize_bilinear'd back to the frame size times d.  d in {1, 2, 4}
   (else SS_VALUE_ERROR, the reference's message); the fast preset's
   flow_downscale (consistency.py:101) is what callers pass. */
SS_API int ss_flownet_set_downscale(ss_flownet *net, int downscale);
SS_API int ss_flownet_destroy(ss_flownet *net);
/* Stateless: flow from frame_a toward frame_b ((h, w, c) HWC float32 device
 * pointers) into uv (h, w, 2) and valid (h, w) (may be NULL); stream-ordered.
 * Thread-safe: calls share one scratch set per frame size, serialised by a
 * mutex; a call on another stream waits for the previous user's work. */
SS_API int ss_flownet_flow(ss_flownet *net, const float *frame_a, const float *frame_b, int h,
                           int w, int c, float *uv, uint8_t *valid, void *stream);
/* Attach the network to a session: it computes the step's flows itself,
 * caching each ring frame's feature pyramid (FlowProvider.flow_between(t, I_t,
 * t-/+1, I_t-/+1), consistency.py:380, :384). */
SS_API int ss_session_attach_flownet(ss_session *s, ss_flownet *net);
/* Compute flow slot `which` (0: t -> t-1, 1: t -> t+1) for the pending step. */
SS_API int ss_session_compute_flow(ss_session *s, int which);
/* Roofline probe: average device time of `reps` launches of the session's
 * first estimator convolution at pyramid `level` (3..6) and its algorithmic
 * FLOPs (live channels only). */
SS_API int ss_session_time_conv(ss_session *s, int level, int reps, float *ms, double *flops);
SS_API void *ss_session_stream(const ss_session *s);
/* Make the session stream wait for the session's side-stream work (the flow
 * to the previous frame runs there) -- e.g. before recording an event that
 * must cover all of a step's work. */
SS_API int ss_session_join(ss_session *s);
/* Cross-stream ordering with a caller stream (NULL = legacy default stream).
 * ss_session_wait_stream: session work issued after this call starts only
 * once the caller's stream has finished what it had issued -- call it before
 * ss_push_pair / ss_set_flow / ss_stage_pair from device buffers the caller's
 * stream produced.  ss_session_signal_stream: the caller's stream waits for
 * the session work issued so far (e.g. those copies) -- call it before
 * freeing or reusing the source buffers on the caller's stream.  The
 * reference has no streams; these replace the implicit ordering of numpy
 * (consistency.py:321-340 keeps references to the caller's frames). */
SS_API int ss_session_wait_stream(ss_session *s, void *stream);
SS_API int ss_session_signal_stream(ss_session *s, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* STREAMSTAB_B200_H */
