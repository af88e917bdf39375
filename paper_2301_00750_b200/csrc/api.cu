// C ABI (include/streamstab_b200.h): stateless ops and the device-resident
// session that replaces SessionState + stabilize_step / stream_end_step
// (consistency.py:306-413).  The index logic (3-pair ring, consecutive
// positions, one-frame latency, error texts) follows consistency.py:321-353
// exactly; the per-frame math is K1 (k_presolve) + K2 (solve_planar).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>

#include "dis.h"
#include "flownet.h"
#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};
static thread_local bool g_capturing = false;

void count_launches(long n)
{
    if (!g_capturing) g_launches.fetch_add(n, std::memory_order_relaxed);
}

void set_capturing(bool on) { g_capturing = on; }

void set_error(const std::string &msg) { g_last_error = msg; }

int cuda_status(cudaError_t e, const char *what)
{
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? SS_NO_MEMORY : SS_CUDA_ERROR;
}

static int check_c(int c)
{
    if (c != 1 && c != 3) {
        set_error("frame must be (H, W, 1|3)");
        return SS_VALUE_ERROR;
    }
    return SS_OK;
}

static int check_hw(int h, int w)
{
    if (h <= 0 || w <= 0) {
        set_error("zero-sized frame");
        return SS_VALUE_ERROR;
    }
    return SS_OK;
}

// u8 -> f32 (x / 255) ingest, HWC
__global__ void k_u8_to_f32(const uint8_t *__restrict__ src, long n, float *__restrict__ dst)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = __fdiv_rn((float)src[i], 255.0f);
}

// rint(clip(x, 0, 1) * 255) -> u8 (service.py:101-102, imgio.py:132)
__global__ void k_f32_to_u8(const float *__restrict__ src, long n, uint8_t *__restrict__ dst)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (uint8_t)rintf(__fmul_rn(fminf(fmaxf(src[i], 0.0f), 1.0f), 255.0f));
}

// ConstantFlow (flow.py:406-425): FlowField(uv) marks a pixel invalid when
// max(|u|, |v|) > 1e9 or a component is NaN (imgio.py:172-174; NaN compares
// false, and 1e9 is exact in float32)
__global__ void k_fill_flow(float *__restrict__ uv, uint8_t *__restrict__ valid, long n, float u,
                            float v)
{
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        reinterpret_cast<float2 *>(uv)[i] = make_float2(u, v);
        valid[i] = fabsf(u) <= 1e9f && fabsf(v) <= 1e9f;
    }
}


// Host <-> device copies from / to PAGEABLE host memory (numpy arrays: the
// drop-in API) go through a small pinned bounce ring: the host-side memcpy of
// chunk i+1 (several threads) overlaps the DMA of chunk i, instead of the
// driver's single-threaded staging.  Pinned sources / destinations (cudaHostAlloc,
// torch pin_memory) are copied directly.
struct Bounce {
    static constexpr size_t CHUNK = 8u << 20;
    uint8_t *buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~Bounce()
    {
        for (int k = 0; k < 2; ++k) {
            if (ev[k]) {
                cudaEventSynchronize(ev[k]);
                cudaEventDestroy(ev[k]);
            }
            if (buf[k]) cudaFreeHost(buf[k]);
        }
    }
    int ensure()
    {
        for (int k = 0; k < 2; ++k) {
            if (!buf[k]) SS_CUDA_TRY(cudaHostAlloc(&buf[k], CHUNK, cudaHostAllocDefault));
            if (!ev[k]) SS_CUDA_TRY(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
        }
        return SS_OK;
    }
};

static bool host_pinned(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

static void par_memcpy(void *dst, const void *src, size_t n)
{
    constexpr size_t PIECE = 512u << 10;
    const long pieces = (long)((n + PIECE - 1) / PIECE);
#pragma omp parallel for schedule(static) num_threads(8) if (pieces > 1)
    for (long i = 0; i < pieces; ++i) {
        const size_t off = (size_t)i * PIECE;
        std::memcpy(static_cast<uint8_t *>(dst) + off, static_cast<const uint8_t *>(src) + off,
                    std::min(PIECE, n - off));
    }
}

// host -> device (returns once the host source may be reused; the DMA of the
// last chunks may still be in flight on `st`)
static int h2d(Bounce &b, void *dst, const void *src, size_t n, cudaStream_t st)
{
    if (n < (256u << 10) || host_pinned(src)) {
        SS_CUDA_TRY(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
        return SS_OK;
    }
    if (int rc = b.ensure()) return rc;
    for (size_t off = 0, i = 0; off < n; off += Bounce::CHUNK, ++i) {
        const int k = (int)(i & 1);
        const size_t c = std::min(Bounce::CHUNK, n - off);
        SS_CUDA_TRY(cudaEventSynchronize(b.ev[k]));  // the slot's previous DMA is done
        par_memcpy(b.buf[k], static_cast<const uint8_t *>(src) + off, c);
        SS_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t *>(dst) + off, b.buf[k], c,
                                    cudaMemcpyHostToDevice, st));
        SS_CUDA_TRY(cudaEventRecord(b.ev[k], st));
    }
    return SS_OK;
}

// device -> host, synchronous (the data is in dst on return)
static int d2h(Bounce &b, void *dst, const void *src, size_t n, cudaStream_t st)
{
    if (n < (256u << 10) || host_pinned(dst)) {
        SS_CUDA_TRY(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st));
        SS_CUDA_TRY(cudaStreamSynchronize(st));
        return SS_OK;
    }
    if (int rc = b.ensure()) return rc;
    size_t pend_off = 0, pend_n = 0;
    int pend_k = -1;
    for (size_t off = 0, i = 0; off < n; off += Bounce::CHUNK, ++i) {
        const int k = (int)(i & 1);
        const size_t c = std::min(Bounce::CHUNK, n - off);
        SS_CUDA_TRY(cudaEventSynchronize(b.ev[k]));
        SS_CUDA_TRY(cudaMemcpyAsync(b.buf[k], static_cast<const uint8_t *>(src) + off, c,
                                    cudaMemcpyDeviceToHost, st));
        SS_CUDA_TRY(cudaEventRecord(b.ev[k], st));
        if (pend_k >= 0) {  // drain the previous chunk while this one copies
            SS_CUDA_TRY(cudaEventSynchronize(b.ev[pend_k]));
            par_memcpy(static_cast<uint8_t *>(dst) + pend_off, b.buf[pend_k], pend_n);
        }
        pend_k = k;
        pend_off = off;
        pend_n = c;
    }
    if (pend_k >= 0) {
        SS_CUDA_TRY(cudaEventSynchronize(b.ev[pend_k]));
        par_memcpy(static_cast<uint8_t *>(dst) + pend_off, b.buf[pend_k], pend_n);
    }
    return SS_OK;
}

}  // namespace ss

using namespace ss;

// ---------------------------------------------------------------------------
struct ss_session {
    int h, w, ci, cp;
    cudaStream_t stream;
    bool own_stream;
    struct Slot {
        int64_t pos;
        float *I, *P;
    } slot[3];
    int order[3];  // slot indices in push order (oldest first)
    int n_pairs;
    float *O, *O_new;  // prev_output (HWC) and solver output
    bool has_output;
    int64_t solved_through;
    // flows for the pending step: [0] t -> t-1, [1] t -> t+1
    float *uv[2];
    uint8_t *valid[2];
    int64_t flow_for[2];  // step position the slot was provided for (-1 none)
    float *A, *lapP, *wc;  // planar solver inputs
    SolverWork solver;
    cudaEvent_t ev[3];
    ss_timing timing;
    // lite flow network (optional): pyramid slot i follows ring slot i
    ss_flownet *net = nullptr;
    std::unique_ptr<fn::Run> run;
    cudaEvent_t fev[2] = {nullptr, nullptr};
    bool flow_timed = false;
    // the flow to the previous frame runs on a side stream, concurrently with
    // the next frame's pyramid and the flow to it on the session stream
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaStream_t hi = nullptr;  // highest priority: pyramid + flow to the next frame
    cudaEvent_t hfork = nullptr, hjoin = nullptr;
    bool side_pending = false;
    int side_slots[2] = {-1, -1};  // ring slots whose pyramids the side flow reads
    // pre-launch: once a step's solver is enqueued (before the host waits for
    // it), the NEXT step's flow t+1 -> t -- both pyramids already cached -- is
    // launched on the side stream behind the solver, into spare buffers; the
    // next ss_session_compute_flow(0) claims it by swapping pointers.  The GPU
    // starts it the moment the solver ends instead of after the host's return
    // trip (and graph launch).  Spare buffers: a diverged step keeps its flows.
    float *uv_pre = nullptr;
    uint8_t *valid_pre = nullptr;
    cudaEvent_t pre_start = nullptr;
    int64_t pre_for = -1;  // step position the pre-launched flow is for
    int pre_slots[2] = {-1, -1};
    int pre_kind = 0;        // 1: lite CNN, 2: DIS (s->dis0)
    bool dis_used = false;   // this step's flow to t-1 came from ss_session_compute_dis_flow
    // asynchronous output (ss_output_async): device->host copy on its own
    // stream, overlapping the next step; the solver that would next overwrite
    // the copied buffer waits for it
    cudaStream_t copy = nullptr;
    cudaEvent_t out_src = nullptr, out_done = nullptr;
    bool out_pending = false;
    uint8_t *out_u8 = nullptr;
    // input staging (ss_stage_pair): the next pair's host->device copy runs on
    // the copy stream while the current step computes; ss_push_pair of that
    // pair then swaps the staged buffers into the ring (no copy)
    float *stI = nullptr, *stP = nullptr;
    const void *st_hostI = nullptr, *st_hostP = nullptr;
    int64_t staged_pos = -1;
    cudaEvent_t st_src = nullptr, st_done = nullptr;
    cudaStream_t up = nullptr;
    // the staging buffers have no reader left (their frame's last step
    // completed): an upload into them needs no ordering after the session
    bool stage_idle = true;
    cudaEvent_t xev = nullptr;  // ss_session_wait_stream / ss_session_signal_stream
    mutable Bounce bounce;      // pageable host <-> device copies
    std::unique_ptr<dis::Estimator> dis;   // built-in flow (BuiltinFlow)
    std::unique_ptr<dis::Estimator> dis0;  // its flow to t-1, on the side stream
};

// session-stream work that touches what the side-stream flow reads or writes
// waits for it (idempotent; the flag is cleared once a step consumed it)
static int join_side(const ss_session *s)
{
    if (s->side_pending) SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->join, 0));
    return SS_OK;
}

// Scratch reused by consecutive stateless calls: a call on another stream
// than the previous user of the same scratch first waits for that user's work
struct StreamOrder {
    cudaEvent_t done = nullptr;
    cudaStream_t last = nullptr;
    bool used = false;
    ~StreamOrder()
    {
        if (done) cudaEventDestroy(done);
    }
    int before(cudaStream_t st)
    {
        if (used && st != last) SS_CUDA_TRY(cudaStreamWaitEvent(st, done, 0));
        return SS_OK;
    }
    int after(cudaStream_t st)
    {
        if (!done) SS_CUDA_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        SS_CUDA_TRY(cudaEventRecord(done, st));
        last = st;
        used = true;
        return SS_OK;
    }
};

struct ss_flownet {
    int device;
    int precision;
    int downscale = 1;  // FlowOptions.downscale (flow.py:34): network on box-downscaled frames
    fn::Weights wts;
    // stateless calls (ss_flownet_flow): one scratch set per frame size,
    // shared by all callers -- host threads serialise on the mutex, streams
    // on the StreamOrder event
    std::mutex mu;
    std::map<std::pair<int, int>, std::pair<std::unique_ptr<fn::Run>, StreamOrder>> runs;
};

static int session_alloc(ss_session *s)
{
    const size_t px = (size_t)s->h * s->w;
    for (auto &sl : s->slot) {
        SS_CUDA_TRY(cudaMalloc(&sl.I, px * s->ci * sizeof(float)));
        SS_CUDA_TRY(cudaMalloc(&sl.P, px * s->cp * sizeof(float)));
        sl.pos = 0;
    }
    SS_CUDA_TRY(cudaMalloc(&s->O, px * s->cp * sizeof(float)));
    SS_CUDA_TRY(cudaMalloc(&s->O_new, px * s->cp * sizeof(float)));
    for (int k = 0; k < 2; ++k) {
        SS_CUDA_TRY(cudaMalloc(&s->uv[k], px * 2 * sizeof(float)));
        SS_CUDA_TRY(cudaMalloc(&s->valid[k], px));
    }
    // A, dP, w_c in one block (planar solver inputs)
    SS_CUDA_TRY(cudaMalloc(&s->A, px * (2 * s->cp + 1) * sizeof(float)));
    s->lapP = s->A + px * s->cp;
    s->wc = s->lapP + px * s->cp;
    for (auto &e : s->ev) SS_CUDA_TRY(cudaEventCreate(&e));
    for (auto &e : s->fev) SS_CUDA_TRY(cudaEventCreate(&e));
    return s->solver.ensure(s->h, s->w, s->cp, 150) == SS_OK ? SS_OK : SS_NO_MEMORY;
}

static void session_free(ss_session *s)
{
    for (auto &sl : s->slot) {
        cudaFree(sl.I);
        cudaFree(sl.P);
    }
    cudaFree(s->O);
    cudaFree(s->O_new);
    for (int k = 0; k < 2; ++k) {
        cudaFree(s->uv[k]);
        cudaFree(s->valid[k]);
    }
    cudaFree(s->A);  // also lapP, wc
    for (auto &e : s->ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : s->fev)
        if (e) cudaEventDestroy(e);
    if (s->side) {
        cudaStreamSynchronize(s->side);
        cudaStreamDestroy(s->side);
    }
    if (s->fork) cudaEventDestroy(s->fork);
    if (s->join) cudaEventDestroy(s->join);
    if (s->hi) {
        cudaStreamSynchronize(s->hi);
        cudaStreamDestroy(s->hi);
    }
    if (s->hfork) cudaEventDestroy(s->hfork);
    if (s->hjoin) cudaEventDestroy(s->hjoin);
    if (s->pre_start) cudaEventDestroy(s->pre_start);
    cudaFree(s->uv_pre);
    cudaFree(s->valid_pre);
    if (s->copy) {
        cudaStreamSynchronize(s->copy);
        cudaStreamDestroy(s->copy);
    }
    if (s->out_src) cudaEventDestroy(s->out_src);
    if (s->out_done) cudaEventDestroy(s->out_done);
    cudaFree(s->out_u8);
    if (s->up) {
        cudaStreamSynchronize(s->up);
        cudaStreamDestroy(s->up);
    }
    if (s->st_src) cudaEventDestroy(s->st_src);
    if (s->st_done) cudaEventDestroy(s->st_done);
    cudaFree(s->stI);
    cudaFree(s->stP);
    if (s->xev) cudaEventDestroy(s->xev);
    s->run.reset();
    s->dis.reset();
    s->dis0.reset();
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
}

static int copy_frame(ss_session *s, float *dst, const void *src, int c, int dtype, int where)
{
    const size_t n = (size_t)s->h * s->w * c;
    const cudaMemcpyKind kind = where == SS_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (dtype == SS_F32) {
        if (where == SS_HOST) return h2d(s->bounce, dst, src, n * sizeof(float), s->stream);
        SS_CUDA_TRY(cudaMemcpyAsync(dst, src, n * sizeof(float), kind, s->stream));
        return SS_OK;
    }
    if (dtype != SS_U8) {
        set_error("unsupported dtype");
        return SS_VALUE_ERROR;
    }
    // stage the u8 bytes in O_new (scratch between steps; an asynchronous
    // output copy may still be reading it -- it held the previous output)
    // and widen them into dst (x / 255, imgio.py:72)
    if (s->out_pending) SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->out_done, 0));
    uint8_t *stage = reinterpret_cast<uint8_t *>(s->O_new);
    if ((size_t)s->h * s->w * s->cp * sizeof(float) < n) {
        set_error("u8 staging buffer too small");
        return SS_VALUE_ERROR;
    }
    if (where == SS_HOST) {
        if (int rc = h2d(s->bounce, stage, src, n, s->stream)) return rc;
    } else {
        SS_CUDA_TRY(cudaMemcpyAsync(stage, src, n, kind, s->stream));
    }
    k_u8_to_f32<<<blocks_for((long)n, 256), 256, 0, s->stream>>>(stage, (long)n, dst);
    SS_LAUNCH_CHECK("k_u8_to_f32");
    return SS_OK;
}

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }

long long ss_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char *ss_status_string(int status)
{
    switch (status) {
    case SS_OK: return "ok";
    case SS_RESOLUTION_MISMATCH: return "resolution mismatch";
    case SS_VALUE_ERROR: return "value error";
    case SS_SOLVER_DIVERGENCE: return "solver divergence";
    case SS_CUDA_ERROR: return "cuda error";
    case SS_NO_MEMORY: return "out of device memory";
    default: return "unknown status";
    }
}

const char *ss_last_error(void) { return g_last_error.c_str(); }

int ss_init(int device)
{
    SS_CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    SS_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        set_error("streamstab_b200 targets sm_100 (B200); found sm_" + std::to_string(prop.major) +
                  std::to_string(prop.minor));
        return SS_CUDA_ERROR;
    }
    return SS_OK;
}

int ss_params_validate(const ss_params *p)
{
    // consistency.py:53-69, same order and messages
    if (!(0.0f <= p->k1 && p->k1 < 1.0f && 0.0f <= p->k2 && p->k2 < 1.0f)) {
        set_error("k1 and k2 must lie in [0, 1)");
        return SS_VALUE_ERROR;
    }
    if ((double)p->k1 + (double)p->k2 <= 0.0) {
        set_error("k1+k2 must be > 0");
        return SS_VALUE_ERROR;
    }
    if ((double)p->k1 + (double)p->k2 >= 1.0) {
        set_error("k1+k2 must be < 1");
        return SS_VALUE_ERROR;
    }
    if (p->lam < 0.0f) {
        set_error("lambda must be >= 0");
        return SS_VALUE_ERROR;
    }
    if (p->eta <= 0.0f) {
        set_error("eta must be > 0");
        return SS_VALUE_ERROR;
    }
    if (!(0.0f <= p->kappa && p->kappa < 1.0f)) {
        set_error("kappa must be in [0, 1)");
        return SS_VALUE_ERROR;
    }
    if (p->iterations < 1) {
        set_error("iterations must be >= 1");
        return SS_VALUE_ERROR;
    }
    if (p->flow_downscale != 1 && p->flow_downscale != 2 && p->flow_downscale != 4) {
        set_error("flow_downscale must be 1, 2 or 4");
        return SS_VALUE_ERROR;
    }
    return SS_OK;
}

// ---- stateless ops ----------------------------------------------------------
int ss_backward_warp(const float *img, int h, int w, int c, const float *uv, const uint8_t *valid,
                     float *out, float *mask, void *stream)
{
    if (int rc = check_hw(h, w)) return rc;
    return launch_backward_warp(img, h, w, c, uv, valid, out, mask, (cudaStream_t)stream);
}

int ss_occlusion_mask(const float *fwd_uv, const uint8_t *fwd_valid, const float *bwd_uv,
                      const uint8_t *bwd_valid, int h, int w, float *out, void *stream)
{
    if (int rc = check_hw(h, w)) return rc;
    return launch_occlusion(fwd_uv, fwd_valid, bwd_uv, bwd_valid, h, w, out, (cudaStream_t)stream);
}

int ss_warp_weight(const float *ref, const float *warped, int h, int w, int c, float alpha,
                   float bound, const float *validity, float *out, void *stream)
{
    if (!(0.0f <= bound && bound < 1.0f)) {
        set_error("bound must lie in [0, 1)");
        return SS_VALUE_ERROR;
    }
    return launch_warp_weight(ref, warped, (long)h * w, c, alpha, bound, validity, out,
                              (cudaStream_t)stream);
}

int ss_local_blend(const float *cur, const float *prev, const float *next, const float *wp,
                   const float *wn, int h, int w, int c, float *out, void *stream)
{
    return launch_local_blend(cur, prev, next, wp, wn, (long)h * w, c, out, (cudaStream_t)stream);
}

int ss_adaptive_blend(const float *g, const float *l, const float *wp, int h, int w, int c,
                      float *out, void *stream)
{
    return launch_adaptive_blend(g, l, wp, (long)h * w, c, out, (cudaStream_t)stream);
}

int ss_consistency_weight(const float *cur, const float *blended, int h, int w, int c,
                          float alpha, float lam, float *out, void *stream)
{
    if (lam < 0.0f) {
        set_error("lambda must be >= 0");
        return SS_VALUE_ERROR;
    }
    return launch_consistency_weight(cur, blended, (long)h * w, c, alpha, lam, out,
                                     (cudaStream_t)stream);
}

int ss_laplacian(const float *img, int h, int w, int c, float *out, void *stream)
{
    if (int rc = check_hw(h, w)) return rc;
    return launch_laplacian(img, h, w, c, out, false, (cudaStream_t)stream);
}

int ss_solve_screened_poisson(const float *processed, const float *target, const float *wc,
                              int h, int w, int c, const ss_params *p, const float *init,
                              float *out, int *div_iter, void *stream)
{
    if (int rc = check_hw(h, w)) return rc;
    if (int rc = check_c(c)) return rc;
    if (p->iterations < 1) {
        set_error("iterations must be >= 1");
        return SS_VALUE_ERROR;
    }
    cudaStream_t st = (cudaStream_t)stream;
    static thread_local SolverWork wk;
    const size_t n = (size_t)h * w * c;
    struct Tmp {
        float *p = nullptr;
        ~Tmp() { cudaFree(p); }
    } tA, tL, tI;
    SS_CUDA_TRY(cudaMalloc(&tA.p, n * sizeof(float)));
    SS_CUDA_TRY(cudaMalloc(&tL.p, n * sizeof(float)));
    if (init && init != target) SS_CUDA_TRY(cudaMalloc(&tI.p, n * sizeof(float)));
    if (int rc = wk.ensure(h, w, c, p->iterations)) return rc;
    if (int rc = launch_hwc_to_planar(target, h, w, c, tA.p, st)) return rc;
    if (int rc = launch_laplacian(processed, h, w, c, tL.p, true, st)) return rc;
    if (tI.p)
        if (int rc = launch_hwc_to_planar(init, h, w, c, tI.p, st)) return rc;
    const int rc = solve_planar(wk, tA.p, tI.p ? tI.p : tA.p, tL.p, wc, *p, out, div_iter, st);
    cudaStreamSynchronize(st);  // temporaries are freed on return
    return rc;
}

// ---- built-in DIS flow ------------------------------------------------------------
static dis::Options dis_options(int levels, int patch, int iters, int downscale)
{
    dis::Options o;
    o.levels = levels;
    o.patch = patch;
    o.iters = iters;
    o.downscale = downscale;
    return o;
}

static bool same_opts(const dis::Options &a, const dis::Options &b)
{
    return a.levels == b.levels && a.patch == b.patch && a.iters == b.iters &&
           a.downscale == b.downscale;
}

int ss_dis_flow(const float *frame_a, const float *frame_b, int h, int w, int c, int levels,
                int patch, int iters, int downscale, float *uv, uint8_t *valid, void *stream)
{
    if (int rc = check_hw(h, w)) return rc;
    if (int rc = check_c(c)) return rc;
    // per host thread; consecutive calls on different streams are ordered
    static thread_local std::unique_ptr<dis::Estimator> est;
    static thread_local StreamOrder order;
    const dis::Options o = dis_options(levels, patch, iters, downscale);
    cudaStream_t st = (cudaStream_t)stream;
    if (!est || est->h != h || est->w != w || !same_opts(est->opts, o)) {
        if (est && order.used) SS_CUDA_TRY(cudaEventSynchronize(order.done));  // freed below
        est.reset(new dis::Estimator());
        order.used = false;
        if (int rc = est->init(h, w, o)) {
            est.reset();
            return rc;
        }
    }
    if (int rc = order.before(st)) return rc;
    if (int rc = est->run(frame_a, frame_b, c, uv, valid, st)) return rc;
    return order.after(st);
}

// ---- metrics -------------------------------------------------------------------
namespace {
struct DevScratch {  // grow-only per-thread device scratch
    void *p = nullptr;
    size_t bytes = 0;
    ~DevScratch() { cudaFree(p); }
    int ensure(size_t b)
    {
        if (b <= bytes) return SS_OK;
        cudaFree(p);
        p = nullptr;
        bytes = 0;
        SS_CUDA_TRY(cudaMalloc(&p, b));
        bytes = b;
        return SS_OK;
    }
};
thread_local DevScratch metric_scratch;
}  // namespace

int ss_warping_error_sums(const float *frame_a, const float *frame_b, int h, int w, int c,
                          const float *fwd_uv, const uint8_t *fwd_valid, const float *bwd_uv,
                          const uint8_t *bwd_valid, double *sums_host, void *stream)
{
    if (int rc = check_hw(h, w)) return rc;
    if (int rc = check_c(c)) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (int rc = metric_scratch.ensure(2 * sizeof(double))) return rc;
    double *d = static_cast<double *>(metric_scratch.p);
    if (int rc = launch_warping_error(frame_a, frame_b, h, w, c, fwd_uv, fwd_valid, bwd_uv,
                                      bwd_valid, d, st))
        return rc;
    SS_CUDA_TRY(cudaMemcpyAsync(sums_host, d, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    SS_CUDA_TRY(cudaStreamSynchronize(st));
    return SS_OK;
}

int ss_ssim(const float *a, const float *b, int h, int w, int c, double *out_host, void *stream)
{
    if (int rc = check_hw(h, w)) return rc;
    if (int rc = check_c(c)) return rc;
    if (h < 11 || w < 11) {
        set_error("image " + std::to_string(w) + "x" + std::to_string(h) +
                  " smaller than the 11x11 window");
        return SS_VALUE_ERROR;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)h * w;
    if (int rc = metric_scratch.ensure((7 * n + 1) * sizeof(double))) return rc;
    double *scratch = static_cast<double *>(metric_scratch.p);
    double *sum = scratch + 7 * n;
    if (int rc = launch_ssim(a, b, h, w, c, scratch, sum, st)) return rc;
    double s = 0.0;
    SS_CUDA_TRY(cudaMemcpyAsync(&s, sum, sizeof(double), cudaMemcpyDeviceToHost, st));
    SS_CUDA_TRY(cudaStreamSynchronize(st));
    *out_host = s / ((double)(h - 10) * (double)(w - 10));
    return SS_OK;
}

// ---- sessions ----------------------------------------------------------------
int ss_session_create(int h, int w, int c_in, int c_proc, void *stream, ss_session **out)
{
    if (int rc = check_hw(h, w)) return rc;
    if (int rc = check_c(c_in)) return rc;
    if (int rc = check_c(c_proc)) return rc;
    ss_session *s = new (std::nothrow) ss_session();
    if (!s) return SS_NO_MEMORY;
    s->h = h;
    s->w = w;
    s->ci = c_in;
    s->cp = c_proc;
    s->n_pairs = 0;
    s->staged_pos = -1;
    s->has_output = false;
    s->solved_through = 0;
    s->flow_for[0] = s->flow_for[1] = -1;
    if (stream) {
        s->stream = (cudaStream_t)stream;
        s->own_stream = false;
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete s;
            return cuda_status(e, "cudaStreamCreate");
        }
        s->own_stream = true;
    }
    int rc = session_alloc(s);
    if (rc) {
        session_free(s);
        delete s;
        return rc;
    }
    *out = s;
    return SS_OK;
}

int ss_session_destroy(ss_session *s)
{
    if (!s) return SS_OK;
    cudaStreamSynchronize(s->stream);
    session_free(s);
    delete s;
    return SS_OK;
}

int ss_session_reset(ss_session *s)
{
    if (int rc = join_side(s)) return rc;
    s->side_pending = false;
    s->flow_timed = false;
    s->pre_for = -1;
    s->dis_used = false;
    s->n_pairs = 0;
    s->has_output = false;
    s->solved_through = 0;
    s->flow_for[0] = s->flow_for[1] = -1;
    s->timing = ss_timing{};
    return SS_OK;
}

void *ss_session_stream(const ss_session *s) { return (void *)s->stream; }

// cross-stream ordering with the caller's stream (e.g. torch's current
// stream, which may be the legacy default stream 0): device sources produced
// there are complete before the session reads them, and temporaries the
// caller frees afterwards are not reused before the session's copy ran
static int xev(ss_session *s)
{
    if (!s->xev) SS_CUDA_TRY(cudaEventCreateWithFlags(&s->xev, cudaEventDisableTiming));
    return SS_OK;
}

int ss_session_wait_stream(ss_session *s, void *stream)
{
    if ((cudaStream_t)stream == s->stream) return SS_OK;
    if (int rc = xev(s)) return rc;
    SS_CUDA_TRY(cudaEventRecord(s->xev, (cudaStream_t)stream));
    SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->xev, 0));
    return SS_OK;
}

int ss_session_signal_stream(ss_session *s, void *stream)
{
    if ((cudaStream_t)stream == s->stream) return SS_OK;
    if (int rc = xev(s)) return rc;
    SS_CUDA_TRY(cudaEventRecord(s->xev, s->stream));
    SS_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, s->xev, 0));
    return SS_OK;
}

int ss_session_join(ss_session *s)
{
    // everything the session has in flight on its internal streams (the side
    // flow, and the high-priority chain incl. a pre-launched pyramid)
    if (int rc = join_side(s)) return rc;
    if (s->hi) {
        SS_CUDA_TRY(cudaEventRecord(s->hjoin, s->hi));
        SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->hjoin, 0));
    }
    return SS_OK;
}

int ss_push_pair(ss_session *s, int64_t position, const void *I, const void *P, int dtype,
                 int where)
{
    // consistency.py:326-330
    if (s->n_pairs > 0) {
        const int64_t last = s->slot[s->order[s->n_pairs - 1]].pos;
        if (position != last + 1) {
            set_error("non-consecutive frame position " + std::to_string(position) + " after " +
                      std::to_string(last));
            return SS_VALUE_ERROR;
        }
    }
    // choose the slot: a free one, else the oldest (pop(0), :336-337)
    int idx;
    if (s->n_pairs < 3) {
        bool used[3] = {false, false, false};
        for (int i = 0; i < s->n_pairs; ++i) used[s->order[i]] = true;
        idx = !used[0] ? 0 : (!used[1] ? 1 : 2);
        s->order[s->n_pairs++] = idx;
    } else {
        idx = s->order[0];
        s->order[0] = s->order[1];
        s->order[1] = s->order[2];
        s->order[2] = idx;
    }
    auto &sl = s->slot[idx];
    // the evicted frame (position q) is read only by steps <= q + 1
    const bool evicted_idle = s->n_pairs == 3 && sl.pos + 1 <= s->solved_through;
    // the pending side flow reads the pyramids of two other ring slots; the
    // copy into this slot overlaps it unless it evicts one of them
    if (idx == s->side_slots[0] || idx == s->side_slots[1])
        if (int rc = join_side(s)) return rc;
    const bool staged = s->staged_pos == position && I == s->st_hostI && P == s->st_hostP && dtype == SS_F32;
    // the slot's cached pyramid is stale -- unless it is this staged pair's,
    // computed by ss_step from the staging buffers (keyed by its position)
    if (s->run && !(staged && s->run->slots[idx].key == position)) s->run->slots[idx].key = -1;
    if (staged) {
        // staged by ss_stage_pair: swap its buffers into the ring once copied
        SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->st_done, 0));
        std::swap(sl.I, s->stI);
        std::swap(sl.P, s->stP);
        s->staged_pos = -1;
        s->stage_idle = evicted_idle;  // the staging buffers now hold the evicted frame
    } else {
        if (int rc = copy_frame(s, sl.I, I, s->ci, dtype, where)) return rc;
        if (int rc = copy_frame(s, sl.P, P, s->cp, dtype, where)) return rc;
    }
    sl.pos = position;
    if (!s->has_output) {  // :338-340 (prev_output = first processed frame)
        SS_CUDA_TRY(cudaMemcpyAsync(s->O, sl.P, (size_t)s->h * s->w * s->cp * sizeof(float),
                                    cudaMemcpyDeviceToDevice, s->stream));
        s->has_output = true;
        s->solved_through = position;
    }
    return SS_OK;
}

int ss_stage_pair(ss_session *s, int64_t position, const void *I, const void *P, int dtype, int where)
{
    if (dtype != SS_F32) {
        set_error("ss_stage_pair stages float32 frames");
        return SS_VALUE_ERROR;
    }
    const size_t px = (size_t)s->h * s->w;
    if (!s->copy) {
        SS_CUDA_TRY(cudaStreamCreateWithFlags(&s->copy, cudaStreamNonBlocking));
        SS_CUDA_TRY(cudaEventCreateWithFlags(&s->out_src, cudaEventDisableTiming));
        SS_CUDA_TRY(cudaEventCreateWithFlags(&s->out_done, cudaEventDisableTiming));
    }
    if (!s->stI) {
        SS_CUDA_TRY(cudaMalloc(&s->stI, px * s->ci * sizeof(float)));
        SS_CUDA_TRY(cudaMalloc(&s->stP, px * s->cp * sizeof(float)));
        SS_CUDA_TRY(cudaEventCreateWithFlags(&s->st_src, cudaEventDisableTiming));
        SS_CUDA_TRY(cudaEventCreateWithFlags(&s->st_done, cudaEventDisableTiming));
    }
    if (s->staged_pos >= 0) SS_CUDA_TRY(cudaEventSynchronize(s->st_done));  // unconsumed: overwrite
    // a pyramid ss_step computed from an earlier staging of this position is stale
    if (s->run)
        for (int k = 0; k < 3; ++k)
            if (s->run->slots[k].key == position) s->run->slots[k].key = -1;
    // the staging buffers were the ring slot the last push evicted: unless
    // that frame's last step has completed (stage_idle), order the upload
    // after session work issued so far (it may still read them).  Uploads use
    // their own stream, so they never queue behind result downloads on the
    // copy stream.
    if (!s->up) SS_CUDA_TRY(cudaStreamCreateWithFlags(&s->up, cudaStreamNonBlocking));
    if (!s->stage_idle) {
        SS_CUDA_TRY(cudaEventRecord(s->st_src, s->stream));
        SS_CUDA_TRY(cudaStreamWaitEvent(s->up, s->st_src, 0));
    }
    const cudaMemcpyKind kind = where == SS_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    SS_CUDA_TRY(cudaMemcpyAsync(s->stI, I, px * s->ci * sizeof(float), kind, s->up));
    SS_CUDA_TRY(cudaMemcpyAsync(s->stP, P, px * s->cp * sizeof(float), kind, s->up));
    SS_CUDA_TRY(cudaEventRecord(s->st_done, s->up));
    s->staged_pos = position;
    s->st_hostI = I;
    s->st_hostP = P;
    return SS_OK;
}

int64_t ss_solved_through(const ss_session *s) { return s->solved_through; }

// SessionState.prev_output / solved_through assignment (the reference's
// dataclass fields, consistency.py:305-319; read at :342-345, written at
// :338-340 and :410-411): resume a stream from a known O_{t-1}
int ss_session_set_state(ss_session *s, int mode, int64_t solved_through, const void *prev_output, int dtype,
                         int where)
{
    if (mode < SS_STATE_POSITION || mode > SS_STATE_CLEAR) {
        set_error("mode must be SS_STATE_POSITION, SS_STATE_OUTPUT or SS_STATE_CLEAR");
        return SS_VALUE_ERROR;
    }
    if (mode == SS_STATE_OUTPUT && !prev_output) {
        set_error("prev_output is NULL");
        return SS_VALUE_ERROR;
    }
    // flows started for the old pending step no longer apply
    if (int rc = join_side(s)) return rc;
    s->side_pending = false;
    s->pre_for = -1;
    s->flow_for[0] = s->flow_for[1] = -1;
    if (mode == SS_STATE_OUTPUT) {
        if (int rc = copy_frame(s, s->O, prev_output, s->cp, dtype, where)) return rc;
        s->has_output = true;
    } else if (mode == SS_STATE_CLEAR) {
        s->has_output = false;  // prev_output = None: the next push pins it (:338-340)
    }
    s->solved_through = solved_through;
    return SS_OK;
}

static const ss_session::Slot *find_pos(const ss_session *s, int64_t pos)
{
    for (int i = 0; i < s->n_pairs; ++i)
        if (s->slot[s->order[i]].pos == pos) return &s->slot[s->order[i]];
    return nullptr;
}

int ss_pending(const ss_session *s, int64_t *t, int *has_prev, int *has_next)
{
    const int64_t tt = s->solved_through + 1;
    if (t) *t = tt;
    if (has_prev) *has_prev = find_pos(s, tt - 1) && find_pos(s, tt);
    if (has_next) *has_next = find_pos(s, tt + 1) != nullptr;
    return SS_OK;
}

int ss_set_flow(ss_session *s, int which, const float *uv, const uint8_t *valid, int where)
{
    if (which != 0 && which != 1) {
        set_error("which must be 0 (to previous) or 1 (to next)");
        return SS_VALUE_ERROR;
    }
    if (int rc = join_side(s)) return rc;
    if (which == 0) s->dis_used = false;
    const size_t px = (size_t)s->h * s->w;
    const cudaMemcpyKind kind = where == SS_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (where == SS_HOST) {
        if (int rc = h2d(s->bounce, s->uv[which], uv, px * 2 * sizeof(float), s->stream)) return rc;
        if (valid)
            if (int rc = h2d(s->bounce, s->valid[which], valid, px, s->stream)) return rc;
    } else {
        SS_CUDA_TRY(cudaMemcpyAsync(s->uv[which], uv, px * 2 * sizeof(float), kind, s->stream));
        if (valid) SS_CUDA_TRY(cudaMemcpyAsync(s->valid[which], valid, px, kind, s->stream));
    }
    if (!valid) SS_CUDA_TRY(cudaMemsetAsync(s->valid[which], 1, px, s->stream));
    s->flow_for[which] = s->solved_through + 1;
    return SS_OK;
}

int ss_set_constant_flow(ss_session *s, int which, double u, double v, int steps)
{
    if (which != 0 && which != 1) {
        set_error("which must be 0 (to previous) or 1 (to next)");
        return SS_VALUE_ERROR;
    }
    // ConstantFlow: uv = (u * steps, v * steps) in float64 then float32
    const float fu = (float)(u * steps), fv = (float)(v * steps);
    const long px = (long)s->h * s->w;
    if (int rc = join_side(s)) return rc;
    if (which == 0) s->dis_used = false;
    k_fill_flow<<<blocks_for(px, 256), 256, 0, s->stream>>>(s->uv[which], s->valid[which], px, fu, fv);
    SS_LAUNCH_CHECK("k_fill_flow");
    s->flow_for[which] = s->solved_through + 1;
    return SS_OK;
}

int ss_check_step(const ss_session *s, int with_next, int64_t *tp)
{
    // _snippet (consistency.py:342-353)
    if (!s->has_output) {
        set_error("no buffered frames");
        return SS_VALUE_ERROR;
    }
    const int64_t t = s->solved_through + 1;
    if (tp) *tp = t;
    if (!find_pos(s, t - 1) || !find_pos(s, t)) {
        set_error("missing buffered frames around position " + std::to_string(t));
        return SS_VALUE_ERROR;
    }
    const bool has_next = find_pos(s, t + 1) != nullptr;
    if (with_next && !has_next) {
        set_error("missing next frame " + std::to_string(t + 1) +
                  "; use stream_end_step at stream end");
        return SS_VALUE_ERROR;
    }
    if (!with_next && has_next) {
        set_error("next frame is available; use stabilize_step");
        return SS_VALUE_ERROR;
    }
    return SS_OK;
}

int ss_step(ss_session *s, int with_next, const ss_params *p, int *div_iter)
{
    if (div_iter) *div_iter = 0;
    int64_t t = 0;
    if (int rc = ss_check_step(s, with_next, &t)) return rc;
    const auto *prev = find_pos(s, t - 1), *cur = find_pos(s, t), *next = find_pos(s, t + 1);
    if (s->flow_for[0] != t || (with_next && s->flow_for[1] != t)) {
        set_error("flows for position " + std::to_string(t) + " were not provided");
        return SS_VALUE_ERROR;
    }
    if (p->iterations < 1) {
        set_error("iterations must be >= 1");
        return SS_VALUE_ERROR;
    }
    if (int rc = join_side(s)) return rc;
    s->side_pending = false;
    // an asynchronous output copy of O_new's buffer (two steps old) must finish
    // before this step's solver overwrites it
    if (s->out_pending) SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->out_done, 0));
    SS_CUDA_TRY(cudaEventRecord(s->ev[0], s->stream));
    PresolveArgs a;
    a.h = s->h;
    a.w = s->w;
    a.I_prev = prev->I;
    a.P_prev = prev->P;
    a.I_cur = cur->I;
    a.P_cur = cur->P;
    a.I_next = with_next ? next->I : nullptr;
    a.P_next = with_next ? next->P : nullptr;
    a.O_prev = s->O;
    a.uv_prev = s->uv[0];
    a.valid_prev = s->valid[0];
    a.uv_next = s->uv[1];
    a.valid_next = s->valid[1];
    a.p = *p;
    a.A = s->A;
    a.lapP = s->lapP;
    a.wc = s->wc;
    a.wp_out = a.wn_out = nullptr;
    if (int rc = launch_presolve(a, s->ci, s->cp, with_next != 0, s->stream)) return rc;
    SS_CUDA_TRY(cudaEventRecord(s->ev[1], s->stream));
    // the next step's pyramid(t+2) (if staged) and flow t+1 -> t, launched
    // once the solver is enqueued
    auto prelaunch = [&]() -> int {
        static const bool on = getenv("SS_FLOW_PRELAUNCH") == nullptr || strcmp(getenv("SS_FLOW_PRELAUNCH"), "0");
        if (!on || !with_next || !s->side) return SS_OK;
        const int64_t tn = t + 1;
        const int ia = (int)(next - s->slot), ib = (int)(cur - s->slot);
        const size_t npx = (size_t)s->h * s->w;
        if (!s->run) {
            // DIS provider: its flow t+1 -> t on the side estimator, behind the solver
            if (!s->dis_used || !s->dis0) return SS_OK;
            if (!s->uv_pre) {
                SS_CUDA_TRY(cudaMalloc(&s->uv_pre, npx * 2 * sizeof(float)));
                SS_CUDA_TRY(cudaMalloc(&s->valid_pre, npx));
                SS_CUDA_TRY(cudaEventCreate(&s->pre_start));
            }
            SS_CUDA_TRY(cudaStreamWaitEvent(s->side, s->ev[2], 0));
            SS_CUDA_TRY(cudaEventRecord(s->pre_start, s->side));
            if (int rc = s->dis0->run(next->I, cur->I, s->ci, s->uv_pre, s->valid_pre, s->side)) return rc;
            SS_CUDA_TRY(cudaEventRecord(s->join, s->side));
            s->side_pending = true;
            s->side_slots[0] = s->pre_slots[0] = ia;
            s->side_slots[1] = s->pre_slots[1] = ib;
            s->pre_for = tn;
            s->pre_kind = 2;
            return SS_OK;
        }
        if (s->run->slots[ia].key != tn || s->run->slots[ib].key != t) return SS_OK;  // pyramids not cached
        const size_t px = (size_t)s->h * s->w;
        if (!s->uv_pre) {
            SS_CUDA_TRY(cudaMalloc(&s->uv_pre, px * 2 * sizeof(float)));
            SS_CUDA_TRY(cudaMalloc(&s->valid_pre, px));
            SS_CUDA_TRY(cudaEventCreate(&s->pre_start));
        }
        // the caller staged frame t+2 (ss_stage_pair): its pyramid too, into
        // the pyramid slot ss_push_pair will give it -- that of the ring's
        // oldest frame (t-1), which neither upcoming flow reads -- so the
        // critical chain of the next step starts when the solver ends
        if (s->staged_pos == t + 2 && s->n_pairs == 3 && s->slot[s->order[0]].pos == t - 1) {
            const int idx = s->order[0];
            cudaStream_t ps = s->hi ? s->hi : s->stream;
            if (s->hi) SS_CUDA_TRY(cudaStreamWaitEvent(s->hi, s->ev[2], 0));
            SS_CUDA_TRY(cudaStreamWaitEvent(ps, s->st_done, 0));
            if (int rc = s->run->pyramid(idx, t + 2, s->stI, s->ci, ps)) return rc;
        }
        // (flow t+1 -> t gated on the pyramid instead of the solver: 341 -> 330
        // frames/s -- it then competes with the flow to t+2, the critical one)
        // behind the solver (ev[2] marks its end): the flow would only slow it
        SS_CUDA_TRY(cudaStreamWaitEvent(s->side, s->ev[2], 0));
        SS_CUDA_TRY(cudaEventRecord(s->pre_start, s->side));
        if (int rc = s->run->flow(ia, ib, s->uv_pre, s->valid_pre, s->side, 1)) return rc;
        SS_CUDA_TRY(cudaEventRecord(s->join, s->side));
        s->side_pending = true;
        s->side_slots[0] = s->pre_slots[0] = ia;
        s->side_slots[1] = s->pre_slots[1] = ib;
        s->pre_for = tn;
        s->pre_kind = 1;
        return SS_OK;
    };
    int rc = solve_planar(s->solver, s->A, s->A, s->lapP, s->wc, *p, s->O_new, div_iter, s->stream,
                          s->ev[2], prelaunch);
    if (rc) return rc;  // divergence: state not advanced (consistency.py:293, :410)
    SS_CUDA_TRY(cudaEventSynchronize(s->ev[2]));
    float t_blend = 0.f, t_solve = 0.f;
    cudaEventElapsedTime(&t_blend, s->ev[0], s->ev[1]);
    cudaEventElapsedTime(&t_solve, s->ev[1], s->ev[2]);
    s->timing.warp_blend_ms = t_blend;
    s->timing.solve_ms = t_solve;
    s->timing.flow_ms = 0.f;
    if (s->flow_timed) {  // device time of the flow network for this step
        cudaEventElapsedTime(&s->timing.flow_ms, s->fev[0], s->fev[1]);
        s->flow_timed = false;
    }
    float *tmp = s->O;  // commit (consistency.py:410-412)
    s->O = s->O_new;
    s->O_new = tmp;
    s->solved_through = t;
    s->flow_for[0] = s->flow_for[1] = -1;
    return SS_OK;
}

int ss_output(const ss_session *s, void *dst, int dtype, int where)
{
    if (!s->has_output) {
        set_error("no buffered frames");
        return SS_VALUE_ERROR;
    }
    const size_t n = (size_t)s->h * s->w * s->cp;
    const cudaMemcpyKind kind = where == SS_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const void *src = s->O;
    size_t bytes = n * sizeof(float);
    if (dtype == SS_U8) {
        // O_new is scratch between steps, but an asynchronous output copy
        // may still be reading it (it held the previous output)
        if (s->out_pending) SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->out_done, 0));
        uint8_t *tmp = reinterpret_cast<uint8_t *>(s->O_new);
        k_f32_to_u8<<<blocks_for((long)n, 256), 256, 0, s->stream>>>(s->O, (long)n, tmp);
        SS_LAUNCH_CHECK("k_f32_to_u8");
        src = tmp;
        bytes = n;
    } else if (dtype != SS_F32) {
        set_error("unsupported dtype");
        return SS_VALUE_ERROR;
    }
    if (where == SS_HOST) return d2h(s->bounce, dst, src, bytes, s->stream);
    SS_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, kind, s->stream));
    SS_CUDA_TRY(cudaStreamSynchronize(s->stream));
    return SS_OK;
}

int ss_output_async(ss_session *s, void *dst, int dtype, int where)
{
    if (!s->has_output) {
        set_error("no buffered frames");
        return SS_VALUE_ERROR;
    }
    if (dtype != SS_F32 && dtype != SS_U8) {
        set_error("unsupported dtype");
        return SS_VALUE_ERROR;
    }
    const size_t n = (size_t)s->h * s->w * s->cp;
    if (!s->copy) {
        SS_CUDA_TRY(cudaStreamCreateWithFlags(&s->copy, cudaStreamNonBlocking));
        SS_CUDA_TRY(cudaEventCreateWithFlags(&s->out_src, cudaEventDisableTiming));
        SS_CUDA_TRY(cudaEventCreateWithFlags(&s->out_done, cudaEventDisableTiming));
    }
    if (s->out_pending) SS_CUDA_TRY(cudaEventSynchronize(s->out_done));  // one copy in flight
    const cudaMemcpyKind kind = where == SS_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const void *src = s->O;
    if (dtype == SS_U8) {
        if (!s->out_u8) SS_CUDA_TRY(cudaMalloc(&s->out_u8, n));
        k_f32_to_u8<<<blocks_for((long)n, 256), 256, 0, s->stream>>>(s->O, (long)n, s->out_u8);
        SS_LAUNCH_CHECK("k_f32_to_u8");
        src = s->out_u8;
    }
    SS_CUDA_TRY(cudaEventRecord(s->out_src, s->stream));
    SS_CUDA_TRY(cudaStreamWaitEvent(s->copy, s->out_src, 0));
    SS_CUDA_TRY(cudaMemcpyAsync(dst, src, n * (dtype == SS_F32 ? sizeof(float) : 1), kind, s->copy));
    SS_CUDA_TRY(cudaEventRecord(s->out_done, s->copy));
    s->out_pending = true;
    return SS_OK;
}

int ss_output_wait(ss_session *s)
{
    if (s->out_pending) SS_CUDA_TRY(cudaEventSynchronize(s->out_done));
    return SS_OK;
}

const float *ss_output_device(const ss_session *s) { return s->has_output ? s->O : nullptr; }

int ss_last_timing(const ss_session *s, ss_timing *t)
{
    *t = s->timing;
    return SS_OK;
}

int ss_flows(const ss_session *s, int which, float *uv_dst, uint8_t *valid_dst, int where)
{
    if (which != 0 && which != 1) {
        set_error("which must be 0 (to previous) or 1 (to next)");
        return SS_VALUE_ERROR;
    }
    if (int rc = join_side(s)) return rc;
    const size_t px = (size_t)s->h * s->w;
    const cudaMemcpyKind kind = where == SS_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (uv_dst) SS_CUDA_TRY(cudaMemcpyAsync(uv_dst, s->uv[which], px * 2 * sizeof(float), kind, s->stream));
    if (valid_dst) SS_CUDA_TRY(cudaMemcpyAsync(valid_dst, s->valid[which], px, kind, s->stream));
    SS_CUDA_TRY(cudaStreamSynchronize(s->stream));
    return SS_OK;
}

// ---- lite flow network ----------------------------------------------------------
// fp32 -> 3xTF32 on tcgen05 (fp32-class accuracy); bf16 -> bf16 tcgen05
static int conv_mode_for(int precision)
{
    if (precision == SS_FLOW_BF16) return fn::CONV_TC_BF16;
    // the fp32-class path: split-bf16 on the 3x3 stride-1 layers, 3xTF32 on the
    // others (flownet.cu); SS_FP32_IMPL=tf32x3 runs every layer in 3xTF32
    static const bool tf32 = getenv("SS_FP32_IMPL") && !strcmp(getenv("SS_FP32_IMPL"), "tf32x3");
    return tf32 ? fn::CONV_TC_TF32X3 : fn::CONV_TC_BF16X2;
}

int64_t ss_flownet_num_params(void) { return fn::Weights::expected_params(); }

int ss_flownet_create(const float *weights, int64_t n, int precision, ss_flownet **out)
{
    if (precision != SS_FLOW_FP32 && precision != SS_FLOW_BF16) {
        set_error("precision must be SS_FLOW_FP32 or SS_FLOW_BF16");
        return SS_VALUE_ERROR;
    }
    std::unique_ptr<ss_flownet> net(new (std::nothrow) ss_flownet());
    if (!net) return SS_NO_MEMORY;
    SS_CUDA_TRY(cudaGetDevice(&net->device));
    net->precision = precision;
    if (int rc = net->wts.upload(weights, n)) return rc;
    *out = net.release();
    return SS_OK;
}

int ss_flownet_set_downscale(ss_flownet *net, int downscale)
{
    if (downscale != 1 && downscale != 2 && downscale != 4) {
        set_error("downscale must be 1, 2 or 4");
        return SS_VALUE_ERROR;
    }
    std::lock_guard<std::mutex> lock(net->mu);
    if (downscale != net->downscale) {
        cudaDeviceSynchronize();
        net->runs.clear();  // scratch sets are sized for the network's frame
        net->downscale = downscale;
    }
    return SS_OK;
}

int ss_flownet_destroy(ss_flownet *net)
{
    if (net) {
        cudaDeviceSynchronize();
        delete net;
    }
    return SS_OK;
}

int ss_flownet_flow(ss_flownet *net, const float *frame_a, const float *frame_b, int h, int w,
                    int c, float *uv, uint8_t *valid, void *stream)
{
    if (int rc = check_hw(h, w)) return rc;
    if (int rc = check_c(c)) return rc;
    std::lock_guard<std::mutex> lock(net->mu);
    auto &entry = net->runs[{h, w}];
    auto &run = entry.first;
    if (!run) {
        run.reset(new fn::Run());
        if (int rc = run->init(&net->wts, h, w, 1, net->downscale)) {
            run.reset();
            return rc;
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (int rc = entry.second.before(st)) return rc;
    run->conv_mode = conv_mode_for(net->precision);
    if (int rc = run->pyramid(0, -1, frame_a, c, st)) return rc;
    if (int rc = run->pyramid(1, -1, frame_b, c, st)) return rc;
    if (int rc = run->flow(0, 1, uv, valid, st)) return rc;
    return entry.second.after(st);
}

int ss_session_attach_flownet(ss_session *s, ss_flownet *net)
{
    if (s->net == net && s->run && s->run->ds == net->downscale) return SS_OK;
    if (int rc = join_side(s)) return rc;
    SS_CUDA_TRY(cudaStreamSynchronize(s->stream));
    s->side_pending = false;
    s->net = net;
    // SS_FLOW_CONCURRENT=0 runs both flows of a step on the session stream
    const char *cc = getenv("SS_FLOW_CONCURRENT");
    const bool concurrent = cc == nullptr || strcmp(cc, "0");
    s->run.reset(new fn::Run());
    if (int rc = s->run->init(&net->wts, s->h, s->w, concurrent ? 2 : 1, net->downscale)) {
        s->run.reset();
        s->net = nullptr;
        return rc;
    }
    s->run->conv_mode = conv_mode_for(net->precision);
    s->run->use_graphs = getenv("SS_FLOW_GRAPHS") == nullptr || strcmp(getenv("SS_FLOW_GRAPHS"), "0");
    if (concurrent && !s->side) {
        SS_CUDA_TRY(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
        SS_CUDA_TRY(cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming));
        SS_CUDA_TRY(cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming));
        // the critical chain (pyramid of the new frame -> flow to it) runs on
        // a highest-priority stream: the concurrent flow to the previous frame
        // (side stream, lowest priority) then fills the SMs it leaves idle
        // instead of holding them while the chain's small kernels queue
        static const bool prio = getenv("SS_FLOW_PRIO") == nullptr || strcmp(getenv("SS_FLOW_PRIO"), "0");
        if (prio) {
            int least = 0, greatest = 0;
            SS_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            SS_CUDA_TRY(cudaStreamCreateWithPriority(&s->hi, cudaStreamNonBlocking, greatest));
            SS_CUDA_TRY(cudaEventCreateWithFlags(&s->hfork, cudaEventDisableTiming));
            SS_CUDA_TRY(cudaEventCreateWithFlags(&s->hjoin, cudaEventDisableTiming));
        }
    }
    return fn::prepare_conv_tma();
}

int ss_session_compute_dis_flow(ss_session *s, int which, int levels, int patch, int iters,
                                int downscale)
{
    if (which != 0 && which != 1) {
        set_error("which must be 0 (to previous) or 1 (to next)");
        return SS_VALUE_ERROR;
    }
    const int64_t t = s->solved_through + 1, other = which == 0 ? t - 1 : t + 1;
    const auto *a = find_pos(s, t), *b = find_pos(s, other);
    if (!a || !b) {
        set_error("frames " + std::to_string(t) + " and " + std::to_string(other) +
                  " are not buffered");
        return SS_VALUE_ERROR;
    }
    // the flow to t-1 runs on the side stream with its own estimator,
    // concurrently with the flow to t+1 on the session stream
    // (SS_DIS_CONCURRENT=0: both on the session stream)
    static const bool conc = getenv("SS_DIS_CONCURRENT") == nullptr || strcmp(getenv("SS_DIS_CONCURRENT"), "0");
    const bool side = conc && which == 0;
    const dis::Options o0 = dis_options(levels, patch, iters, downscale);
    if (which == 0 && s->pre_for == t && s->pre_kind == 2 && s->pre_slots[0] == (int)(a - s->slot) &&
        s->pre_slots[1] == (int)(b - s->slot) && s->dis0 && same_opts(s->dis0->opts, o0)) {
        // pre-launched by the previous ss_step: claim it (side_pending stays set)
        std::swap(s->uv[0], s->uv_pre);
        std::swap(s->valid[0], s->valid_pre);
        std::swap(s->fev[0], s->pre_start);
        s->pre_for = -1;
        s->flow_timed = true;
        s->flow_for[0] = t;
        s->dis_used = true;
        return SS_OK;
    }
    if (which == 0) s->dis_used = side;
    if (which == 0 || !conc)
        if (int rc = join_side(s)) return rc;  // a pending side flow (its buffers / slots)
    if (which == 0) s->side_pending = false;
    const dis::Options o = dis_options(levels, patch, iters, downscale);
    std::unique_ptr<dis::Estimator> &est = side ? s->dis0 : s->dis;
    if (!est || !same_opts(est->opts, o)) {
        est.reset(new dis::Estimator());
        if (int rc = est->init(s->h, s->w, o)) {
            est.reset();
            return rc;
        }
        est->use_graphs = true;
    }
    if (which == 0 || !s->flow_timed) SS_CUDA_TRY(cudaEventRecord(s->fev[0], s->stream));
    if (side) {
        if (!s->side) {
            SS_CUDA_TRY(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
            SS_CUDA_TRY(cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming));
            SS_CUDA_TRY(cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming));
        }
        SS_CUDA_TRY(cudaEventRecord(s->fork, s->stream));
        SS_CUDA_TRY(cudaStreamWaitEvent(s->side, s->fork, 0));
        if (int rc = est->run(a->I, b->I, s->ci, s->uv[0], s->valid[0], s->side)) return rc;
        SS_CUDA_TRY(cudaEventRecord(s->join, s->side));
        SS_CUDA_TRY(cudaEventRecord(s->fev[1], s->side));
        s->side_pending = true;
        s->side_slots[0] = (int)(a - s->slot);
        s->side_slots[1] = (int)(b - s->slot);
    } else {
        // the flow to t+1 is on the critical chain: run it on a highest-priority
        // stream (forked from / joined to the session stream), ahead of the
        // side flow's kernels (SS_FLOW_PRIO=0: on the session stream)
        static const bool prio = getenv("SS_FLOW_PRIO") == nullptr || strcmp(getenv("SS_FLOW_PRIO"), "0");
        cudaStream_t ws = s->stream;
        if (prio && conc) {
            if (!s->hi) {
                int least = 0, greatest = 0;
                SS_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
                SS_CUDA_TRY(cudaStreamCreateWithPriority(&s->hi, cudaStreamNonBlocking, greatest));
                SS_CUDA_TRY(cudaEventCreateWithFlags(&s->hfork, cudaEventDisableTiming));
                SS_CUDA_TRY(cudaEventCreateWithFlags(&s->hjoin, cudaEventDisableTiming));
            }
            SS_CUDA_TRY(cudaEventRecord(s->hfork, s->stream));
            SS_CUDA_TRY(cudaStreamWaitEvent(s->hi, s->hfork, 0));
            ws = s->hi;
        }
        if (int rc = est->run(a->I, b->I, s->ci, s->uv[which], s->valid[which], ws)) return rc;
        if (ws != s->stream) {
            SS_CUDA_TRY(cudaEventRecord(s->hjoin, s->hi));
            SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->hjoin, 0));
        }
        if (int rc = join_side(s)) return rc;  // fev[1] marks the end of both flows
        SS_CUDA_TRY(cudaEventRecord(s->fev[1], s->stream));
    }
    s->flow_timed = true;
    s->flow_for[which] = t;
    return SS_OK;
}

int ss_session_time_conv(ss_session *s, int level, int reps, float *ms, double *flops)
{
    if (!s->run) {
        set_error("no flow network attached to the session");
        return SS_VALUE_ERROR;
    }
    if (int rc = join_side(s)) return rc;
    s->run->select_set(0);
    return s->run->time_est1(level, reps < 1 ? 1 : reps, s->stream, ms, flops);
}

int ss_session_compute_flow(ss_session *s, int which)
{
    if (which != 0 && which != 1) {
        set_error("which must be 0 (to previous) or 1 (to next)");
        return SS_VALUE_ERROR;
    }
    if (!s->run) {
        set_error("no flow network attached to the session");
        return SS_VALUE_ERROR;
    }
    const int64_t t = s->solved_through + 1, other = which == 0 ? t - 1 : t + 1;
    const auto *a = find_pos(s, t), *b = find_pos(s, other);
    if (!a || !b) {
        set_error("frames " + std::to_string(t) + " and " + std::to_string(other) +
                  " are not buffered");
        return SS_VALUE_ERROR;
    }
    const int ia = (int)(a - s->slot), ib = (int)(b - s->slot);
    if (which == 0 && s->pre_for == t && s->pre_kind == 1 && s->pre_slots[0] == ia && s->pre_slots[1] == ib &&
        s->run->slots[ia].key == t && s->run->slots[ib].key == other) {
        // pre-launched by the previous ss_step: claim it (it may still be
        // running on the side stream; side_pending stays set)
        std::swap(s->uv[0], s->uv_pre);
        std::swap(s->valid[0], s->valid_pre);
        std::swap(s->fev[0], s->pre_start);
        s->pre_for = -1;
        s->flow_timed = true;
        s->flow_for[0] = t;
        return SS_OK;
    }
    s->dis_used = false;
    if (which == 0 || !s->flow_timed) {
        if (which == 0 && s->side_pending) {  // a second flow to the previous frame
            if (int rc = join_side(s)) return rc;
            s->side_pending = false;
        }
        SS_CUDA_TRY(cudaEventRecord(s->fev[0], s->stream));
    }
    // pyramids always run on the session stream (they share scratch buffers);
    // recomputing one the pending side flow reads waits for it first
    for (int k = 0; k < 2; ++k) {
        const int sl = k == 0 ? ia : ib;
        const int64_t pos = k == 0 ? t : other;
        if (s->side_pending && (sl == s->side_slots[0] || sl == s->side_slots[1]) &&
            s->run->slots[sl].key != pos)
            if (int rc = join_side(s)) return rc;
    }
    // pyramids and the flow to the next frame: on the high-priority stream
    // (forked from and joined back to the session stream) when there is one
    cudaStream_t ws = s->stream;
    if (s->hi) {
        SS_CUDA_TRY(cudaEventRecord(s->hfork, s->stream));
        SS_CUDA_TRY(cudaStreamWaitEvent(s->hi, s->hfork, 0));
        ws = s->hi;
    }
    if (int rc = s->run->pyramid(ia, t, a->I, s->ci, ws)) return rc;
    if (int rc = s->run->pyramid(ib, other, b->I, s->ci, ws)) return rc;
    if (which == 0 && s->side) {
        // fork: the flow to t-1 (estimator buffer set 1) overlaps whatever the
        // session stream does next -- typically the pyramid of t+1 and the flow
        // to it (set 0); ss_step / any conflicting call joins it
        SS_CUDA_TRY(cudaEventRecord(s->fork, ws));
        SS_CUDA_TRY(cudaStreamWaitEvent(s->side, s->fork, 0));
        if (int rc = s->run->flow(ia, ib, s->uv[0], s->valid[0], s->side, 1)) return rc;
        SS_CUDA_TRY(cudaEventRecord(s->join, s->side));
        SS_CUDA_TRY(cudaEventRecord(s->fev[1], s->side));
        s->side_pending = true;
        s->side_slots[0] = ia;
        s->side_slots[1] = ib;
        if (s->hi) {
            SS_CUDA_TRY(cudaEventRecord(s->hjoin, s->hi));
            SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->hjoin, 0));
        }
    } else {
        if (int rc = s->run->flow(ia, ib, s->uv[which], s->valid[which], ws, 0)) return rc;
        if (s->hi) {
            SS_CUDA_TRY(cudaEventRecord(s->hjoin, s->hi));
            SS_CUDA_TRY(cudaStreamWaitEvent(s->stream, s->hjoin, 0));
        }
        if (int rc = join_side(s)) return rc;  // fev[1] marks the end of both flows
        SS_CUDA_TRY(cudaEventRecord(s->fev[1], s->stream));
    }
    s->flow_timed = true;
    s->flow_for[which] = t;
    return SS_OK;
}

}  // extern "C"
