// Native runner of the lite flow network: weight upload in the layout of
// liteflownet.layer_table(), per-resolution buffers, pyramid cache, and the
// estimator / refinement schedule (liteflownet.py docstring).
#include <cstring>
#include <string>
#include <vector>

#include "flownet.h"
#include "ss_common.cuh"

namespace ss {
namespace fn {

static const int PYR_CH[6] = {16, 32, 64, 96, 128, 192};
static inline int pad16(int c) { return (c + 15) / 16 * 16; }
static inline int est_in(int lvl) { return lvl == 6 ? 88 : 96 + PYR_CH[lvl - 1]; }
// estimator features: [flow 2 | 0 x6 | e5 32 | e4 64 | e3 96]
constexpr int E_LD = 200, E5_OFF = 8, E4_OFF = 40, E3_OFF = 104;

// layer indices (same order as liteflownet.layer_table())
static inline int pyr_idx(int lvl, int j) { return (lvl - 1) * 3 + j; }          // j: 0 a, 1 b, 2 c
static inline int est_idx(int lvl, int j) { return 18 + (6 - lvl) * 6 + (j - 1); }  // j: 1..6
static inline int ref_idx(int i, bool pw) { return 42 + (i - 1) * 2 + (pw ? 1 : 0); }  // i: 1..6
constexpr int REF7 = 54;

static std::vector<LayerDev> table()
{
    std::vector<LayerDev> L;
    auto conv = [&](int cin, int cout, int k, int stride, int dil, int act) {
        LayerDev d;
        d.cin = cin; d.cout = cout; d.cout_pad = pad16(cout); d.k = k; d.stride = stride;
        d.dil = dil; d.act = act; d.dw = false;
        L.push_back(d);
    };
    int cin = 8;
    for (int l = 1; l <= 6; ++l) {
        conv(cin, PYR_CH[l - 1], 3, 2, 1, 1);
        conv(PYR_CH[l - 1], PYR_CH[l - 1], 3, 1, 1, 1);
        conv(PYR_CH[l - 1], PYR_CH[l - 1], 3, 1, 1, 1);
        cin = PYR_CH[l - 1];
    }
    for (int lvl = 6; lvl >= 3; --lvl) {
        conv(est_in(lvl), 128, 3, 1, 1, 1);
        conv(128, 128, 3, 1, 1, 1);
        conv(128, 96, 3, 1, 1, 1);
        conv(96, 64, 3, 1, 1, 1);
        conv(64 + 96, 32, 3, 1, 1, 1);
        conv(32 + 64, 2, 3, 1, 1, 0);
    }
    const int sep[6][3] = {{104, 128, 1}, {128, 128, 2}, {128, 128, 4},
                           {128, 96, 8},  {96, 64, 16},  {64, 32, 1}};
    for (auto &s : sep) {
        LayerDev d;
        d.cin = s[0]; d.cout = s[0]; d.cout_pad = s[0]; d.k = 3; d.stride = 1; d.dil = s[2];
        d.act = 0; d.dw = true;
        L.push_back(d);
        conv(s[0], s[1], 1, 1, 1, 1);
    }
    conv(32, 2, 3, 1, 1, 0);
    return L;
}

Weights::~Weights()
{
    cudaFree(block);
    cudaFree(tma_block);
    cudaFree(bf_block);
    cudaFree(bs_block);
}

int Weights::expected_params()
{
    long n = 0;
    for (auto &l : table()) n += l.dw ? 9L * l.cin + l.cin : (long)l.k * l.k * l.cin * l.cout + l.cout;
    return (int)n;
}

int Weights::upload(const float *host, int64_t n)
{
    layers = table();
    if (n != expected_params()) {
        set_error("flow network expects " + std::to_string(expected_params()) +
                  " parameters, got " + std::to_string(n));
        return SS_VALUE_ERROR;
    }
    // device layout: conv W [k*k*cin][cout_pad] + b [cout_pad]; dw W [9][cin] + b [cin]
    size_t total = 0;
    for (auto &l : layers)
        total += l.dw ? (size_t)10 * l.cin : (size_t)(l.k * l.k * l.cin + 1) * l.cout_pad;
    std::vector<float> dev(total, 0.0f);
    size_t off = 0, src = 0;
    std::vector<size_t> woff(layers.size()), boff(layers.size());
    for (size_t i = 0; i < layers.size(); ++i) {
        auto &l = layers[i];
        if (l.dw) {
            woff[i] = off;
            std::memcpy(&dev[off], host + src, sizeof(float) * 9 * l.cin);
            off += 9 * l.cin;
            src += 9 * l.cin;
            boff[i] = off;
            std::memcpy(&dev[off], host + src, sizeof(float) * l.cin);
            off += l.cin;
            src += l.cin;
        } else {
            const int K = l.k * l.k * l.cin;
            woff[i] = off;
            for (int r = 0; r < K; ++r)
                std::memcpy(&dev[off + (size_t)r * l.cout_pad], host + src + (size_t)r * l.cout,
                            sizeof(float) * l.cout);
            off += (size_t)K * l.cout_pad;
            src += (size_t)K * l.cout;
            boff[i] = off;
            std::memcpy(&dev[off], host + src, sizeof(float) * l.cout);
            off += l.cout_pad;
            src += l.cout;
        }
    }
    cudaFree(block);
    block = nullptr;
    SS_CUDA_TRY(cudaMalloc(&block, total * sizeof(float)));
    SS_CUDA_TRY(cudaMemcpy(block, dev.data(), total * sizeof(float), cudaMemcpyHostToDevice));
    for (size_t i = 0; i < layers.size(); ++i) {
        layers[i].w = block + woff[i];
        layers[i].b = block + boff[i];
    }

    // TMA path (flownet_tma.cu): per layer [kblocks][parts][2 np][32] fp32 --
    // kblock = cb * k*k + tap (channel block outer, filter tap inner), per
    // output-channel part np tf32-hi rows then np lo rows, 32 input channels
    // cb * 32 + c' per row (zero past cin)
    std::vector<size_t> otm(layers.size(), 0);
    size_t tm_total = 0;
    for (size_t i = 0; i < layers.size(); ++i) {
        auto &l = layers[i];
        if (l.dw) continue;
        otm[i] = tm_total;
        tm_total += (size_t)l.k * l.k * ((l.cin + 31) / 32) * 2 * l.cout_pad * 32;
    }
    std::vector<float> tmh(tm_total, 0.0f);
    for (size_t i = 0; i < layers.size(); ++i) {
        auto &l = layers[i];
        if (l.dw) continue;
        const int taps = l.k * l.k, N = l.cout_pad;
        const int parts = (N + 127) / 128, np = N / parts;
        const float *wl = dev.data() + woff[i];  // [K][cout_pad]
        float *dst = tmh.data() + otm[i];
        for (int tap = 0; tap < taps; ++tap)
            for (int c = 0; c < l.cin; ++c) {
                const size_t kb = (size_t)(c / 32) * taps + tap;
                for (int n = 0; n < l.cout; ++n) {
                    const float f = wl[(size_t)(tap * l.cin + c) * N + n];
                    uint32_t u;
                    std::memcpy(&u, &f, 4);
                    const uint32_t hu = u & 0xffffe000u;
                    float hi;
                    std::memcpy(&hi, &hu, 4);
                    const int part = n / np, nn = n - part * np;
                    const size_t row = (size_t)part * 2 * np + nn;
                    dst[(kb * 2 * N + row) * 32 + c % 32] = hi;
                    dst[(kb * 2 * N + row + np) * 32 + c % 32] = f - hi;
                }
            }
    }
    cudaFree(tma_block);
    tma_block = nullptr;
    SS_CUDA_TRY(cudaMalloc(&tma_block, tm_total * sizeof(float)));
    SS_CUDA_TRY(cudaMemcpy(tma_block, tmh.data(), tm_total * sizeof(float), cudaMemcpyHostToDevice));
    for (size_t i = 0; i < layers.size(); ++i) {
        auto &l = layers[i];
        if (l.dw) continue;
        const int parts = (l.cout_pad + 127) / 128, np = l.cout_pad / parts;
        l.wt_tma = tma_block + otm[i];
        l.tma_T = tma_taps_per_stage(l.k, l.stride, l.dil, l.cin, np, 1);
        const int kblocks = l.k * l.k * ((l.cin + 31) / 32);
        if (int rc = encode_weight_map(&l.tmB, l.wt_tma, kblocks, 2 * l.cout_pad, np, l.tma_T)) return rc;
    }

    // bf16 TMA path: [kblocks][cout_pad rows][32] bf16 (round to nearest even),
    // same kblock order; rows of part p are [p * np, (p + 1) * np)
    std::vector<size_t> obt(layers.size(), 0);
    size_t bt_total = 0;
    for (size_t i = 0; i < layers.size(); ++i) {
        auto &l = layers[i];
        if (l.dw) continue;
        obt[i] = bt_total;
        bt_total += (size_t)l.k * l.k * ((l.cin + 31) / 32) * l.cout_pad * 32;
    }
    std::vector<uint16_t> bth(bt_total, 0);
    for (size_t i = 0; i < layers.size(); ++i) {
        auto &l = layers[i];
        if (l.dw) continue;
        const int taps = l.k * l.k, N = l.cout_pad;
        const float *wl = dev.data() + woff[i];
        uint16_t *dst = bth.data() + obt[i];
        for (int tap = 0; tap < taps; ++tap)
            for (int c = 0; c < l.cin; ++c) {
                const size_t kb = (size_t)(c / 32) * taps + tap;
                for (int n = 0; n < l.cout; ++n) {
                    const float f = wl[(size_t)(tap * l.cin + c) * N + n];
                    uint32_t u;
                    std::memcpy(&u, &f, 4);
                    dst[(kb * N + n) * 32 + c % 32] = (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
                }
            }
    }
    cudaFree(bf_block);
    bf_block = nullptr;
    SS_CUDA_TRY(cudaMalloc(&bf_block, bt_total * sizeof(uint16_t)));
    SS_CUDA_TRY(cudaMemcpy(bf_block, bth.data(), bt_total * sizeof(uint16_t), cudaMemcpyHostToDevice));
    for (size_t i = 0; i < layers.size(); ++i) {
        auto &l = layers[i];
        if (l.dw) continue;
        const int parts = (l.cout_pad + 127) / 128, np = l.cout_pad / parts;
        l.wt_bf = static_cast<uint16_t *>(bf_block) + obt[i];
        l.tma_T_bf = tma_taps_per_stage(l.k, l.stride, l.dil, l.cin, np, 0);
        const int kblocks = l.k * l.k * ((l.cin + 31) / 32);
        if (int rc = encode_weight_map_bf16(&l.tmB_bf, l.wt_bf, kblocks, l.cout_pad, np, l.tma_T_bf)) return rc;
    }

    // split-bf16 path: [kblocks][parts][hi np rows; lo np rows][32] bf16,
    // hi = rn(w), lo = rn(w - hi) (the fp32 path's [hi; lo] arrangement)
    auto bf16_rn = [](float f) {
        uint32_t u;
        std::memcpy(&u, &f, 4);
        return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
    };
    auto bf16_f = [](uint16_t b) {
        const uint32_t u = (uint32_t)b << 16;
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    };
    std::vector<uint16_t> bsh(bt_total * 2, 0);
    for (size_t i = 0; i < layers.size(); ++i) {
        auto &l = layers[i];
        if (l.dw) continue;
        const int taps = l.k * l.k, N = l.cout_pad;
        const int parts = (N + 127) / 128, np = N / parts;
        const float *wl = dev.data() + woff[i];
        uint16_t *dst = bsh.data() + 2 * obt[i];
        for (int tap = 0; tap < taps; ++tap)
            for (int c = 0; c < l.cin; ++c) {
                const size_t kb = (size_t)(c / 32) * taps + tap;
                for (int n = 0; n < l.cout; ++n) {
                    const float f = wl[(size_t)(tap * l.cin + c) * N + n];
                    const uint16_t hb = bf16_rn(f);
                    const int part = n / np, nn = n - part * np;
                    const size_t row = (size_t)part * 2 * np + nn;
                    dst[(kb * 2 * N + row) * 32 + c % 32] = hb;
                    dst[(kb * 2 * N + row + np) * 32 + c % 32] = bf16_rn(f - bf16_f(hb));
                }
            }
    }
    cudaFree(bs_block);
    bs_block = nullptr;
    SS_CUDA_TRY(cudaMalloc(&bs_block, bsh.size() * sizeof(uint16_t)));
    SS_CUDA_TRY(cudaMemcpy(bs_block, bsh.data(), bsh.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    for (size_t i = 0; i < layers.size(); ++i) {
        auto &l = layers[i];
        if (l.dw) continue;
        const int parts = (l.cout_pad + 127) / 128, np = l.cout_pad / parts;
        l.wt_bs = static_cast<uint16_t *>(bs_block) + 2 * obt[i];
        l.tma_T_bs = tma_taps_per_stage(l.k, l.stride, l.dil, l.cin, np, 2);
        const int kblocks = l.k * l.k * ((l.cin + 31) / 32);
        if (int rc = encode_weight_map_bf16_rows(&l.tmB_bs, l.wt_bs, kblocks, 2 * l.cout_pad, 2 * np, l.tma_T_bs))
            return rc;
    }
    return SS_OK;
}

Run::~Run()
{
    for (auto &g : pyr_graphs)
        if (g.second.first) cudaGraphExecDestroy(g.second.first);
    for (auto &g : flow_graphs)
        if (g.second.first) cudaGraphExecDestroy(g.second.first);
    for (void *p : allocs) cudaFree(p);
}

void Run::select_set(int set)
{
    const EstBufs &s = sets[set < nsets ? set : 0];
    for (int l = 0; l < 7; ++l) {
        x[l] = s.x[l];
        e1[l] = s.e1[l];
        e2[l] = s.e2[l];
        E[l] = s.E[l];
        w2[l] = s.w2[l];
    }
    ra = s.ra;
    rb = s.rb;
    rr = s.rr;
    ws = s.ws;
}

int Run::init(const Weights *wt, int h_, int w_, int nsets_, int downscale)
{
    nsets = nsets_ < 1 ? 1 : (nsets_ > 2 ? 2 : nsets_);
    wts = wt;
    if (downscale != 1 && downscale != 2 && downscale != 4) {
        set_error("downscale must be 1, 2 or 4");
        return SS_VALUE_ERROR;
    }
    fh = h_;
    fw = w_;
    ds = downscale;
    h = fh / ds;  // box_downscale crops the remainder (flow.py:74-75)
    w = fw / ds;
    if (h < 1 || w < 1) {
        set_error("frame smaller than the flow downscale factor");
        return SS_VALUE_ERROR;
    }
    H[0] = (h + 63) / 64 * 64;
    W[0] = (w + 63) / 64 * 64;
    for (int l = 1; l <= 6; ++l) {
        H[l] = H[l - 1] / 2;
        W[l] = W[l - 1] / 2;
    }
    auto alloc = [&](float **p, size_t floats) -> int {
        SS_CUDA_TRY(cudaMalloc(p, floats * sizeof(float)));
        SS_CUDA_TRY(cudaMemset(*p, 0, floats * sizeof(float)));
        allocs.push_back(*p);
        return SS_OK;
    };
    const size_t px1 = (size_t)H[1] * W[1];
    int rc;
    if ((rc = alloc(&prep, (size_t)H[0] * W[0] * 8))) return rc;
    if (ds > 1) {
        if ((rc = alloc(&small, (size_t)h * w * 3))) return rc;
        if ((rc = alloc(&uv_small, (size_t)h * w * 2))) return rc;
    }
    if ((rc = alloc(&s0, px1 * 16))) return rc;
    if ((rc = alloc(&s1, px1 * 16))) return rc;
    for (auto &sl : slots)
        for (int l = 3; l <= 6; ++l)
            if ((rc = alloc(&sl.lvl[l], (size_t)H[l] * W[l] * PYR_CH[l - 1]))) return rc;
    ws_floats = 6u << 20;  // 24 MB of split-K partials per set
    for (int s = 0; s < nsets; ++s) {
        EstBufs &b = sets[s];
        for (int l = 0; l < 7; ++l) b.x[l] = b.e1[l] = b.e2[l] = b.E[l] = b.w2[l] = nullptr;
        for (int l = 3; l <= 6; ++l) {
            const size_t px = (size_t)H[l] * W[l];
            if ((rc = alloc(&b.x[l], px * est_in(l)))) return rc;
            if ((rc = alloc(&b.e1[l], px * 128))) return rc;
            if ((rc = alloc(&b.e2[l], px * 128))) return rc;
            if ((rc = alloc(&b.E[l], px * E_LD))) return rc;
            if ((rc = alloc(&b.w2[l], px * PYR_CH[l - 1]))) return rc;
        }
        const size_t px3 = (size_t)H[3] * W[3];
        if ((rc = alloc(&b.ra, px3 * 128))) return rc;
        if ((rc = alloc(&b.rb, px3 * 128))) return rc;
        if ((rc = alloc(&b.rr, px3 * 4))) return rc;
        if ((rc = alloc(&b.ws, ws_floats))) return rc;
    }
    select_set(0);
    return SS_OK;
}

static thread_local int conv_mode_ = CONV_TC_TF32X3;  // set by the Run issuing the convs
// persistent conv grids of the concurrent flow (estimator set 1, the side
// stream) leave SS_SIDE_RESERVE SMs free, so the critical chain's small
// kernels (high-priority stream) find SMs instead of queueing behind them
static thread_local int grid_cap_ = 0;
static int side_grid_cap()
{
    static const int cap = [] {
        const char *e = getenv("SS_SIDE_RESERVE");
        const int r = e ? atoi(e) : 48;
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return r > 0 && r < n ? n - r : 0;
    }();
    return cap;
}
static thread_local float *ws_ = nullptr;
static thread_local size_t ws_floats_ = 0;

// SS_FLOW_PROFILE=1: per-launch device times of the network (CUDA events),
// printed to stderr after every pyramid / flow call (diagnostics only)
namespace {
struct Prof {
    bool on = getenv("SS_FLOW_PROFILE") != nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    void mark(const std::string &name, cudaStream_t st)
    {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        marks.emplace_back(name, e);
    }
    void dump(const char *what)
    {
        if (!on || marks.size() < 2) return;
        cudaEventSynchronize(marks.back().second);
        float total = 0.f;
        for (size_t i = 1; i < marks.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
            total += ms;
            fprintf(stderr, "[flow-prof] %s %-12s %8.1f us\n", what, marks[i].first.c_str(), ms * 1e3f);
        }
        fprintf(stderr, "[flow-prof] %s total %.3f ms\n", what, total);
        for (auto &m : marks) cudaEventDestroy(m.second);
        marks.clear();
    }
};
thread_local Prof prof;
}  // namespace

static int conv(const LayerDev &L, const float *in, int in_ld, int Hi, int Wi, float *out,
                int out_ld, cudaStream_t st);

static int convp(const char *name, const LayerDev &L, const float *in, int in_ld, int Hi, int Wi,
                 float *out, int out_ld, cudaStream_t st)
{
    const int rc = conv(L, in, in_ld, Hi, Wi, out, out_ld, st);
    prof.mark(name, st);
    return rc;
}

static int conv(const LayerDev &L, const float *in, int in_ld, int Hi, int Wi, float *out,
                int out_ld, cudaStream_t st)
{
    ConvParams p;
    p.ws = ws_;
    p.ws_floats = ws_floats_;
    p.in = in;
    p.in_ld = in_ld;
    p.H = Hi;
    p.W = Wi;
    p.Cin = L.cin;
    p.wgt = L.w;
    p.bias = L.b;
    p.Cout = L.cout;
    p.Cout_pad = L.cout_pad;
    p.out = out;
    p.out_ld = out_ld;
    p.k = L.k;
    p.stride = L.stride;
    p.dil = L.dil;
    p.pad = L.dil * (L.k / 2);
    p.Ho = (Hi + 2 * p.pad - L.dil * (L.k - 1) - 1) / L.stride + 1;
    p.Wo = (Wi + 2 * p.pad - L.dil * (L.k - 1) - 1) / L.stride + 1;
    p.act = L.act;
    // split-bf16 serves the 3x3 layers with halo tiles (stride 1, and the
    // stride-2 phase tiles of <= 16 input channels): K = 16 per MMA halves
    // their MMA count; the im2col stride-2 and the 1x1 layers keep 3xTF32,
    // whose in-place hi / lo conversion is cheaper there (1080p, 8 converter
    // warps: pyr3a 22.5 vs 30.5 us, ref*_pw ~21 vs ~25 us; pyr2a 33.0 vs 30.7)
    const bool split_ok = L.k == 3 && (L.stride == 1 || L.cin <= 16);
    const int prec = conv_mode_ == CONV_TC_BF16 ? 0 : (conv_mode_ == CONV_TC_BF16X2 && split_ok ? 2 : 1);
    p.tmB = prec == 0 ? &L.tmB_bf : (prec == 2 ? &L.tmB_bs : &L.tmB);
    p.grid_cap = grid_cap_;
    p.tma_T = prec == 0 ? L.tma_T_bf : (prec == 2 ? L.tma_T_bs : L.tma_T);
    return launch_conv_tma(p, prec, st);
}

// capture fn(st) into a graph (thread-local capture mode) and instantiate it
// capture fn(st) into a graph (thread-local capture mode) and instantiate it;
// *nodes = its kernel count (the launch counter counts them per replay)
template <class F>
static int capture(cudaStream_t st, cudaGraphExec_t *exec, long *nodes, F &&fn)
{
    SS_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    set_capturing(true);
    const int rc = fn();
    set_capturing(false);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return cuda_status(e, "cudaStreamEndCapture");
    size_t n = 0;
    cudaGraphGetNodes(g, nullptr, &n);
    *nodes = (long)n;
    const cudaError_t e2 = cudaGraphInstantiate(exec, g, 0);
    cudaGraphDestroy(g);
    if (e2 != cudaSuccess) return cuda_status(e2, "cudaGraphInstantiate");
    return SS_OK;
}

int Run::pyramid(int slot, int64_t key, const float *img, int c, cudaStream_t st)
{
    Slot &sl = slots[slot];
    if (key >= 0 && sl.key == key) return SS_OK;  // key < 0: never cached
    grid_cap_ = 0;  // pyramids run on the critical chain: the full grid
    sl.key = -1;
    int rc;
    if (use_graphs && !prof.on) {
        auto &g = pyr_graphs[std::make_tuple(slot, (const void *)img, c)];
        if (!g.first && (rc = capture(st, &g.first, &g.second, [&] { return pyramid_impl(slot, img, c, st); }))) {
            pyr_graphs.erase(std::make_tuple(slot, (const void *)img, c));
            return rc;
        }
        SS_CUDA_TRY(cudaGraphLaunch(g.first, st));
        count_launches(g.second);
    } else if ((rc = pyramid_impl(slot, img, c, st))) {
        return rc;
    }
    sl.key = key >= 0 ? key : -1;
    return SS_OK;
}

int Run::flow(int a, int b, float *uv, uint8_t *valid, cudaStream_t st, int set)
{
    set = set < nsets ? set : 0;
    select_set(set);
    grid_cap_ = set == 1 ? side_grid_cap() : 0;
    struct Reset {
        ~Reset() { grid_cap_ = 0; }
    } reset_cap;
    if (use_graphs && !prof.on) {
        const auto k = std::make_tuple(a, b, (void *)uv, (void *)valid, set);
        auto &g = flow_graphs[k];
        int rc;
        if (!g.first && (rc = capture(st, &g.first, &g.second, [&] { return flow_impl(a, b, uv, valid, st); }))) {
            flow_graphs.erase(k);
            return rc;
        }
        SS_CUDA_TRY(cudaGraphLaunch(g.first, st));
        count_launches(g.second);
        return SS_OK;
    }
    return flow_impl(a, b, uv, valid, st);
}

int Run::time_est1(int level, int reps, cudaStream_t st, float *ms, double *flops)
{
    if (level < 3 || level > 6) {
        set_error("level must be 3..6");
        return SS_VALUE_ERROR;
    }
    conv_mode_ = conv_mode;
    ws_ = ws;
    ws_floats_ = ws_floats;
    const LayerDev &L = wts->L(est_idx(level, 1));
    const int X = est_in(level), hh = H[level], ww = W[level];
    cudaEvent_t ev0, ev1;
    SS_CUDA_TRY(cudaEventCreate(&ev0));
    SS_CUDA_TRY(cudaEventCreate(&ev1));
    int rc = conv(L, x[level], X, hh, ww, e1[level], 128, st);  // warm-up
    SS_CUDA_TRY(cudaEventRecord(ev0, st));
    for (int i = 0; i < reps && !rc; ++i) rc = conv(L, x[level], X, hh, ww, e1[level], 128, st);
    SS_CUDA_TRY(cudaEventRecord(ev1, st));
    SS_CUDA_TRY(cudaEventSynchronize(ev1));
    float t = 0.f;
    cudaEventElapsedTime(&t, ev0, ev1);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    *ms = t / reps;
    // algorithmic MACs over the live (unpadded) input channels: 81 corr + 2 flow + C_l
    const int live = level == 6 ? 81 : 81 + 2 + PYR_CH[level - 1];
    *flops = 2.0 * hh * ww * 9.0 * live * L.cout;
    return rc;
}

int Run::pyramid_impl(int slot, const float *img, int c, cudaStream_t st)
{
    Slot &sl = slots[slot];
    conv_mode_ = conv_mode;
    ws_ = sets[0].ws;  // pyramids run on the session stream, as does the set-0 flow
    ws_floats_ = ws_floats;
    int rc;
    prof.mark("start", st);
    if (ds > 1) {  // the network sees the box-downscaled frame
        if ((rc = launch_box_down_hwc(img, fw, c, ds, h, w, small, st))) return rc;
        img = small;
        prof.mark("downscale", st);
    }
    // the frame -> level-1 "a" layer in one FFMA pass (SS_PYR1A_FUSED=0: the
    // 8-channel padded copy + tensor-core conv)
    static const bool fused = getenv("SS_PYR1A_FUSED") == nullptr || strcmp(getenv("SS_PYR1A_FUSED"), "0");
    if (fused) {
        const LayerDev &L1a = wts->L(pyr_idx(1, 0));
        if ((rc = launch_prep_pyr1a(img, h, w, c, H[0], W[0], H[1], W[1], L1a.w, L1a.cout_pad, L1a.b, s0, st)))
            return rc;
        prof.mark("prep+pyr1a", st);
    } else {
        if ((rc = launch_prep(img, h, w, c, H[0], W[0], prep, st))) return rc;
        prof.mark("prep", st);
    }
    const float *in = prep;
    int in_ld = 8;
    for (int l = 1; l <= 6; ++l) {
        const int C = PYR_CH[l - 1];
        const std::string tag = "pyr" + std::to_string(l);
        float *a = in == s0 ? s1 : s0;
        if (l == 1 && fused) {
            a = s0;  // written by k_prep_pyr1a
        } else if ((rc = convp((tag + "a").c_str(), wts->L(pyr_idx(l, 0)), in, in_ld, H[l - 1], W[l - 1], a, C,
                               st))) {
            return rc;
        }
        float *b = a == s0 ? s1 : s0;
        if ((rc = convp((tag + "b").c_str(), wts->L(pyr_idx(l, 1)), a, C, H[l], W[l], b, C, st))) return rc;
        float *c3 = l <= 2 ? a : sl.lvl[l];
        if ((rc = convp((tag + "c").c_str(), wts->L(pyr_idx(l, 2)), b, C, H[l], W[l], c3, C, st))) return rc;
        in = c3;
        in_ld = C;
    }
    prof.dump("pyramid");
    conv_trace_dump("pyramid");
    return SS_OK;
}

int Run::flow_impl(int a, int b, float *uv, uint8_t *valid, cudaStream_t st)
{
    conv_mode_ = conv_mode;
    ws_ = ws;
    ws_floats_ = ws_floats;
    int rc;
    prof.mark("start", st);
    for (int l = 6; l >= 3; --l) {
        const int C = PYR_CH[l - 1], X = est_in(l);
        const std::string tag = "est" + std::to_string(l) + "_";
        const float *f1 = slots[a].lvl[l], *f2 = slots[b].lvl[l];
        if (l == 6) {
            if ((rc = launch_corr(f1, f2, C, H[l], W[l], x[l], X, false, st))) return rc;
        } else {
            if ((rc = launch_up2_warp(E[l + 1], E_LD, H[l + 1], W[l + 1], f2, C, H[l], W[l], x[l], X,
                                      w2[l], st)))
                return rc;
            prof.mark(tag + "warp", st);
            if ((rc = launch_corr(f1, w2[l], C, H[l], W[l], x[l], X, true, st))) return rc;
        }
        prof.mark(tag + "corr", st);
        const int hh = H[l], ww = W[l];
        if ((rc = convp((tag + "1").c_str(), wts->L(est_idx(l, 1)), x[l], X, hh, ww, e1[l], 128, st))) return rc;
        if ((rc = convp((tag + "2").c_str(), wts->L(est_idx(l, 2)), e1[l], 128, hh, ww, e2[l], 128, st))) return rc;
        if ((rc = convp((tag + "3").c_str(), wts->L(est_idx(l, 3)), e2[l], 128, hh, ww, E[l] + E3_OFF, E_LD, st))) return rc;
        if ((rc = convp((tag + "4").c_str(), wts->L(est_idx(l, 4)), E[l] + E3_OFF, E_LD, hh, ww, E[l] + E4_OFF, E_LD, st))) return rc;
        if ((rc = convp((tag + "5").c_str(), wts->L(est_idx(l, 5)), E[l] + E4_OFF, E_LD, hh, ww, E[l] + E5_OFF, E_LD, st))) return rc;
        if ((rc = convp((tag + "6").c_str(), wts->L(est_idx(l, 6)), E[l] + E5_OFF, E_LD, hh, ww, E[l], E_LD, st))) return rc;
    }
    // separable refinement at level 3: r_in = E[3][0:104]
    const int hh = H[3], ww = W[3];
    const float *in = E[3];
    int in_ld = E_LD;
    const int cin[6] = {104, 128, 128, 128, 96, 64};
    for (int i = 1; i <= 6; ++i) {
        const LayerDev &dw = wts->L(ref_idx(i, false));
        if ((rc = launch_depthwise(in, in_ld, hh, ww, cin[i - 1], dw.w, dw.dil, ra, 128, st))) return rc;
        prof.mark("ref" + std::to_string(i) + "_dw", st);
        if ((rc = convp(("ref" + std::to_string(i) + "_pw").c_str(), wts->L(ref_idx(i, true)), ra, 128, hh, ww, rb, 128, st))) return rc;
        in = rb;
        in_ld = 128;
    }
    if ((rc = convp("ref7", wts->L(REF7), rb, 128, hh, ww, rr, 4, st))) return rc;
    if (ds > 1) {
        // resize_bilinear(flow, frame shape) * downscale (flow.py:187)
        if ((rc = launch_flow_final(E[3], E_LD, rr, 4, hh, ww, h, w, uv_small, nullptr, st))) return rc;
        rc = launch_upscale_flow(uv_small, h, w, fh, fw, (float)ds, uv, valid, st);
    } else {
        rc = launch_flow_final(E[3], E_LD, rr, 4, hh, ww, h, w, uv, valid, st);
    }
    prof.mark("final", st);
    prof.dump("flow");
    conv_trace_dump("flow");
    return rc;
}

}  // namespace fn
}  // namespace ss
