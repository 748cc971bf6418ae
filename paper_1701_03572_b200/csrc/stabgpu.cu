// stabgpu.cu — C ABI (include/stabgpu.h) and the Stage-I host driver.
//
// The driver re-expresses the reference's frame-sequential run_offline
// (pipeline.cpp:182-235) as a batched schedule that gives identical
// semantics: tracking state resets at every re-detect frame
// (flow.cpp:326-330), so the frames split into independent segments
// [sR, (s+1)R] that are tracked side by side; the selector scan and the
// trajectory are sequential recurrences over per-frame records and run on the
// device after all fits; composition is independent per frame.
//
// Schedule of one motion chunk (frames first .. first+count):
//   K1 pyramid levels (all frames, one launch per level)
//   K2-K4 corners on every segment's first frame (one launch each, batched)
//   R x { K5 LK forward+backward (all segments)  ->  ordered compaction }
//   K6 fit (+RANSAC) of every frame pair
// then K7 scan + smoothing and K8 compose over the sequence.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types only: the functions are resolved from libnccl.so.2 at run time

#include "common.cuh"
#include "kernels.cuh"

using namespace stabgpu;

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
};

// Stage timing: a Timer records an event pair (from a pool) on the context
// stream around a stage and queues it; nothing waits on it.  The queued pairs
// are read when the caller asks for the stats (stabgpu_get_stats), so timing
// never adds a host sync inside a call.  Slots: 0 pyramid, 1 detect, 2 track,
// 3 fit, 4 compose, 5 plan.
struct TimedSpan {
    int slot;
    cudaEvent_t a, b;
};

struct stabgpu_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t cin = nullptr, cout = nullptr;
    std::map<std::string, DevBuf> bufs;
    bool timing = false;
    stabgpu_stats stats{};
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<TimedSpan> spans;
    unsigned long long* iters_host = nullptr;  // pinned: LK counters of the last motion pass
    bool iters_pending = false;
    ncclComm_t comm = nullptr;  // multi-GPU sharding (stabgpu_comm_init)
    int nranks = 1, rank = 0;
};

namespace {
// NCCL is resolved at run time (dlopen), so the library loads without it and
// shares the process's libnccl.so.2 (e.g. the one torch.distributed loaded).
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};

const NcclApi& nccl_api() {
    static NcclApi a = [] {
        NcclApi r;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return r;
        r.get_unique_id = reinterpret_cast<decltype(r.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        r.comm_init_rank = reinterpret_cast<decltype(r.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        r.all_gather = reinterpret_cast<decltype(r.all_gather)>(dlsym(h, "ncclAllGather"));
        r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
        r.ok = r.get_unique_id && r.comm_init_rank && r.all_gather && r.comm_destroy && r.error_string;
        return r;
    }();
    return a;
}
}  // namespace

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
    char b[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(b, sizeof b, fmt, ap);
    va_end(ap);
    g_err = b;
    return code;
}

#define CUDA_TRY(x)                                                                   \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess)                                                        \
            return set_err(STABGPU_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                           __FILE__, __LINE__);                                       \
    } while (0)

#define TRY(x)              \
    do {                    \
        int r_ = (x);       \
        if (r_) return r_;  \
    } while (0)

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(STABGPU_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return STABGPU_OK;
}

template <typename T>
T* dbuf(stabgpu_ctx* ctx, const std::string& name, size_t count) {
    DevBuf& b = ctx->bufs[name];
    const size_t bytes = count * sizeof(T) + 256;
    if (b.n < bytes) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
        b.n = 0;
        if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        b.n = bytes;
    }
    return static_cast<T*>(b.p);
}

#define DBUF(T, var, name, count)                                                         \
    T* var = dbuf<T>(ctx, name, (count));                                                 \
    if (!var) return set_err(STABGPU_CUDA, "device allocation of %s (%zu x %zu B) failed", \
                             name, (size_t)(count), sizeof(T))

// ---- validation: the reference's validate() overloads --------------------
int validate_frame(int w, int h) {  // image_ops.cpp:9-16
    if (w < STABGPU_MIN_FRAME_DIM || h < STABGPU_MIN_FRAME_DIM)
        return set_err(STABGPU_INVALID_INPUT, "frame smaller than 16x16");
    if (w > 32767 || h > 32767) return set_err(STABGPU_INVALID_INPUT, "frame larger than 32767 px");
    return STABGPU_OK;
}

int validate_detect(const stabgpu_detect_cfg& c) {  // features.cpp:10-26
    if (c.max_corners < 8) return set_err(STABGPU_INVALID_CONFIG, "max_corners must be >= 8");
    if (!(c.quality_level > 0.0 && c.quality_level < 1.0))
        return set_err(STABGPU_INVALID_CONFIG, "quality_level must lie in (0, 1)");
    if (c.min_distance < 1.0) return set_err(STABGPU_INVALID_CONFIG, "min_distance must be >= 1");
    if (c.block_size < 3 || c.block_size % 2 == 0)
        return set_err(STABGPU_INVALID_CONFIG, "block_size must be odd and >= 3");
    if (!(c.roi_margin >= 0.0 && c.roi_margin < 0.4))
        return set_err(STABGPU_INVALID_CONFIG, "roi_margin must lie in [0, 0.4)");
    return STABGPU_OK;
}

int validate_flow(const stabgpu_flow_cfg& c) {  // flow.cpp:10-21
    if (c.window_radius < 1 || c.max_levels < 1 || c.max_iterations < 1 || c.epsilon <= 0.0 ||
        c.fb_threshold <= 0.0)
        return set_err(STABGPU_INVALID_CONFIG, "flow parameters must be positive");
    if (c.redetect_interval < 1) return set_err(STABGPU_INVALID_CONFIG, "redetect_interval must be >= 1");
    if (c.min_tracks < 4) return set_err(STABGPU_INVALID_CONFIG, "min_tracks must be >= 4");
    return STABGPU_OK;
}

int validate_transform(const stabgpu_transform& t) {  // transform.cpp:51-59
    if (!std::isfinite(t.tx) || !std::isfinite(t.ty) || !std::isfinite(t.theta) ||
        !std::isfinite(t.s) || t.s <= 0.0)
        return set_err(STABGPU_INVALID_TRANSFORM,
                       "similarity transform requires finite parameters and s > 0");
    if (t.kind == STABGPU_RIGID && t.s != 1.0)
        return set_err(STABGPU_INVALID_TRANSFORM, "rigid transform must have s == 1");
    return STABGPU_OK;
}

int validate_crop(double crop) {
    if (!(crop >= 0.0 && crop < 0.25))
        return set_err(STABGPU_INVALID_CONFIG, "crop_ratio must lie in [0, 0.25)");
    return STABGPU_OK;
}

int roi_of(int w, int h, double margin, stabgpu_roi* out) {  // features.cpp:28-36
    const int mx = (int)std::lround(margin * w), my = (int)std::lround(margin * h);
    *out = {mx, my, w - mx, h - my};
    if (out->x1 - out->x0 < 32 || out->y1 - out->y0 < 32)
        return set_err(STABGPU_INVALID_CONFIG, "detection ROI smaller than 32x32");
    return STABGPU_OK;
}

// build_pyramid level geometry (image_ops.cpp:62-77)
int level_dims(int w, int h, int max_levels, int* lw, int* lh) {
    int L = 1;
    lw[0] = w;
    lh[0] = h;
    while (L < max_levels && L < STABGPU_MAX_LEVELS) {
        if (lw[L - 1] / 2 < STABGPU_MIN_FRAME_DIM || lh[L - 1] / 2 < STABGPU_MIN_FRAME_DIM) break;
        lw[L] = lw[L - 1] / 2;
        lh[L] = lh[L - 1] / 2;
        ++L;
    }
    return L;
}

FramePlan host_plan(const stabgpu_transform& t) {
    // warp_similarity coefficients evaluated with the host libm, as the
    // reference does (image_ops.cpp:121-122)
    FramePlan p;
    p.tx = t.tx;
    p.ty = t.ty;
    p.theta = t.theta;
    p.s = t.s;
    p.c = std::cos(t.theta) / t.s;
    p.sn = std::sin(t.theta) / t.s;
    p.cf = p.snf = p.kxx = p.kyx = p.kxy = p.kyy = 0;
    return p;
}

cudaEvent_t pooled_event(stabgpu_ctx* ctx) {
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        ctx->ev_pool.push_back(e);
    }
    return ctx->ev_pool[ctx->ev_used++];
}

// A whole-sequence call starts its own stage times (spans queued by earlier
// calls and not read are dropped; their events are recycled).
void begin_timing(stabgpu_ctx* ctx) {
    if (!ctx->timing) return;
    ctx->spans.clear();
    ctx->ev_used = 0;
    ctx->iters_pending = false;
}

// Stage times = the spans queued since the previous read (waits for their end
// events); with none queued the stats keep their last values.
void harvest_timing(stabgpu_ctx* ctx) {
    if (!ctx->spans.empty()) {
        double ms_slot[6] = {0, 0, 0, 0, 0, 0};
        for (const TimedSpan& sp : ctx->spans) {
            float ms = 0.f;
            if (cudaEventSynchronize(sp.b) == cudaSuccess && cudaEventElapsedTime(&ms, sp.a, sp.b) == cudaSuccess)
                ms_slot[sp.slot] += ms;
        }
        ctx->spans.clear();
        ctx->ev_used = 0;
        stabgpu_stats& s = ctx->stats;
        s.ms_pyramid = ms_slot[0];
        s.ms_detect = ms_slot[1];
        s.ms_track = ms_slot[2];
        s.ms_fit = ms_slot[3];
        s.ms_compose = ms_slot[4];
        s.ms_plan = ms_slot[5];
        s.ms_total = s.ms_pyramid + s.ms_detect + s.ms_track + s.ms_fit + s.ms_compose + s.ms_plan;
    }
    stabgpu_stats& s = ctx->stats;
    if (ctx->iters_pending) {
        cudaStreamSynchronize(ctx->stream);
        s.lk_iterations = (long long)ctx->iters_host[0];
        s.lk_level_builds = (long long)ctx->iters_host[1];
        ctx->iters_pending = false;
    }
}

struct Timer {
    stabgpu_ctx* ctx;
    int slot;
    cudaEvent_t a = nullptr;
    Timer(stabgpu_ctx* c, int s) : ctx(c), slot(s) {
        if (ctx->timing && (a = pooled_event(ctx))) cudaEventRecord(a, ctx->stream);
    }
    ~Timer() {
        if (!a) return;
        cudaEvent_t b = pooled_event(ctx);
        if (!b) return;
        cudaEventRecord(b, ctx->stream);
        ctx->spans.push_back(TimedSpan{slot, a, b});
    }
};

// ---- K1 + K2-K4 + K5 + K6 over frames [first, first+count] ----------------
// y points at frame `first`; motion receives records for frames
// first+1 .. first+count at motion[first+1 ...] (and frame 0 when first == 0).
// n_streams > 1 (first == 0): the count+1 frames are n_streams independent
// sequences of equal length, stream-major; each is segmented from its own
// frame 0 and its first frame gets a FIRST record, exactly as if it were run
// alone.
int run_motion(stabgpu_ctx* ctx, const uint8_t* y, long long first, int count, int w, int h,
               const stabgpu_config& cfg, stabgpu_motion_record* motion, int n_streams = 1) {
    cudaStream_t st = ctx->stream;
    const int nF = count + 1;
    const int R = cfg.flow.redetect_interval;
    const int maxc = cfg.detect.max_corners;
    const int F = nF / n_streams;             // frames per stream
    const int nsps = (F - 1 + R - 1) / R;     // segments per stream
    const int nseg = n_streams * nsps;
    const bool uniform = n_streams == 1 || F % R == 0;  // seg_base(s) == s*R
    stabgpu_roi roi;
    TRY(roi_of(w, h, cfg.detect.roi_margin, &roi));
    static_assert(STABGPU_FRAME_FIRST == 0, "the FIRST record is all zero bytes");
    if (first == 0) CUDA_TRY(cudaMemsetAsync(motion, 0, sizeof(stabgpu_motion_record), st));
    if (count <= 0) return STABGPU_OK;
    // ---- K1: pyramid levels
    DevPyramid P;
    std::memset(&P, 0, sizeof P);
    P.levels = level_dims(w, h, cfg.flow.max_levels, P.w, P.h);
    P.lvl[0] = y;
    P.stride[0] = (size_t)w * h;
    {
        Timer tm(ctx, 0);
        for (int l = 1; l < P.levels; ++l) {
            P.stride[l] = (size_t)P.w[l] * P.h[l];
            DBUF(uint8_t, lv, ("pyr" + std::to_string(l)).c_str(), P.stride[l] * nF);
            P.lvl[l] = lv;
        }
        for (int l = 1; l < P.levels; ++l) {
            launch_pyramid_level(P.lvl[l - 1], P.stride[l - 1], P.w[l - 1], P.h[l - 1],
                                 const_cast<uint8_t*>(P.lvl[l]), P.stride[l], nF, st);
            ++ctx->stats.launches;
        }
        TRY(check_launch("pyramid"));
    }
    // ---- K2-K4: corners on each segment's first frame
    const size_t cap = (size_t)(roi.x1 - roi.x0) * (roi.y1 - roi.y0);
    // detection frames go in batches whose candidate scratch (24 B x ROI area
    // per frame, the worst case) stays under ~8 GB however long the sequence
    const int dbatch = (int)std::max<size_t>(1, std::min<size_t>((size_t)nseg, (8ull << 30) / (24 * cap)));
    DetectScratch ds;
    DBUF(unsigned long long, maxbits, "det_max", dbatch);
    DBUF(unsigned int, dcount, "det_count", dbatch);
    DBUF(unsigned long long, ckey, "det_ckey", cap * dbatch);
    DBUF(unsigned int, cidx, "det_cidx", cap * dbatch);
    DBUF(unsigned long long, skey, "det_skey", cap * dbatch);
    DBUF(unsigned int, sidx, "det_sidx", cap * dbatch);
    DBUF(unsigned int, dhist, "det_hist", (size_t)kRespBins * dbatch);
    DBUF(double, dlo, "det_lo", dbatch);
    DBUF(unsigned char, dflags, "det_flags", dbatch);
    DBUF(unsigned, dmlo, "det_mlo", dbatch);
    DBUF(unsigned, dbst, "det_bstart", (size_t)(kBuckets + 1) * dbatch);
    DBUF(unsigned, dbcur, "det_bcur", (size_t)kBuckets * dbatch);
    ds.maxbits = maxbits;
    ds.count = dcount;
    ds.hist = dhist;
    ds.cand_key = ckey;
    ds.cand_idx = cidx;
    ds.sort_key = skey;
    ds.sort_idx = sidx;
    ds.cap = cap;
    ds.lo = dlo;
    ds.flags = dflags;
    ds.mlo = dmlo;
    ds.bstart = dbst;
    ds.bcur = dbcur;
    DBUF(double2, ptsA, "seg_ptsA", (size_t)nseg * maxc);
    DBUF(double2, ptsB, "seg_ptsB", (size_t)nseg * maxc);
    DBUF(int, nA, "seg_nA", nseg);
    DBUF(int, nB, "seg_nB", nseg);
    DBUF(double, dscore, "seg_score", (size_t)nseg * maxc);
    {
        Timer tm(ctx, 1);
        // detection frames are R apart within a stream (and across streams
        // when F is a multiple of R): batches never straddle a gap
        const int run = uniform ? nseg : nsps;
        for (int s0 = 0; s0 < nseg; s0 += run) {
            for (int d0 = s0; d0 < s0 + run; d0 += dbatch) {
                const int nd = std::min(dbatch, s0 + run - d0);
                PlaneBatch fb{y + (size_t)seg_base(d0, R, F, nsps) * w * h, (size_t)R * w * h, w, h};
                launch_detect(fb, nd, cfg.detect, roi, ds, ptsA + (size_t)d0 * maxc,
                              dscore + (size_t)d0 * maxc, nA + d0, st);
                ctx->stats.launches += 7;
            }
        }
        TRY(check_launch("detect"));
    }
    // ---- K5: R tracking steps over all segments
    DBUF(double2, fwd, "lk_fwd", (size_t)nseg * maxc);
    DBUF(uint8_t, keep, "lk_keep", (size_t)nseg * maxc);
    DBUF(double2, trk_prev, "trk_prev", (size_t)count * maxc);
    DBUF(double2, trk_cur, "trk_cur", (size_t)count * maxc);
    DBUF(int, trk_n, "trk_n", count);
    DBUF(unsigned long long, iters, "lk_iters", 3);
    DBUF(unsigned, lk_work, "lk_work", 1);
    CUDA_TRY(cudaMemsetAsync(iters, 0, 3 * sizeof(unsigned long long), st));
    if (cfg.flow.window_radius <= 15) {
        // whole-segment chains in one launch, then one ordered compaction per step
        Timer tm(ctx, 2);
        const int steps = std::min(R, F - 1);
        DBUF(double2, pos, "lk_pos", (size_t)steps * nseg * maxc);
        DBUF(uint8_t, alive, "lk_alive", (size_t)steps * nseg * maxc);
        LkChain c;
        c.pyr = P;
        c.R = R;
        c.steps = steps;
        c.nseg = nseg;
        c.max_pts = maxc;
        c.nframes = nF;
        c.F = F;
        c.nsps = nsps;
        c.pts = ptsA;
        c.npts = nA;
        c.pos = pos;
        c.alive = alive;
        c.iter_count = iters;
        c.work = lk_work;
        launch_lk_chain(c, cfg.flow, st);
        ++ctx->stats.launches;
        const size_t plane = (size_t)nseg * maxc;
        for (int t = 1; t <= steps; ++t) {
            LkStep s;
            std::memset(&s, 0, sizeof s);
            s.frame0 = 0;
            s.seg_len = R;
            s.t = t;
            s.nseg = nseg;
            s.max_pts = maxc;
            s.pts = t == 1 ? ptsA : pos + (size_t)(t - 2) * plane;
            s.npts = nA;
            s.fwd = pos + (size_t)(t - 1) * plane;
            s.keep = alive + (size_t)(t - 1) * plane;
            s.nframes = nF;
            s.F = F;
            s.nsps = nsps;
            launch_compact(s, ptsB, nB, trk_prev, trk_cur, trk_n, 1, st);
            ++ctx->stats.launches;
        }
        TRY(check_launch("lk"));
    } else {
        Timer tm(ctx, 2);
        double2* cur_pts = ptsA;
        double2* nxt_pts = ptsB;
        int* cur_n = nA;
        int* nxt_n = nB;
        for (int t = 1; t <= R && t < F; ++t) {
            LkStep s;
            s.F = F;
            s.nsps = nsps;
            s.pyr = P;
            s.frame0 = 0;
            s.seg_len = R;
            s.t = t;
            s.nseg = nseg;
            s.max_pts = maxc;
            s.pts = cur_pts;
            s.npts = cur_n;
            s.fwd = fwd;
            s.keep = keep;
            s.iter_count = iters;
            s.nframes = nF;
            s.mode = 1;
            s.ref = nullptr;
            s.work = lk_work;
            launch_lk(s, cfg.flow, st);
            launch_compact(s, nxt_pts, nxt_n, trk_prev, trk_cur, trk_n, 1, st);
            ctx->stats.launches += 2;
            std::swap(cur_pts, nxt_pts);
            std::swap(cur_n, nxt_n);
        }
        TRY(check_launch("lk"));
    }
    // ---- K6: fits
    {
        Timer tm(ctx, 3);
        launch_fit(trk_prev, trk_cur, trk_n, maxc, count, first + 1, cfg, motion + first + 1, st,
                   n_streams > 1 ? F : 0);
        ++ctx->stats.launches;
        TRY(check_launch("fit"));
    }
    if (ctx->timing && ctx->iters_host) {  // LK counters, read at stabgpu_get_stats
        CUDA_TRY(cudaMemcpyAsync(ctx->iters_host, iters, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        ctx->iters_pending = true;
    }
    return STABGPU_OK;
}

// n states followed by n error words (for n == 1: the state, then its word)
int init_plan_state(stabgpu_ctx* ctx, const stabgpu_config& cfg, PlanState** out, int n = 1) {
    DBUF(PlanState, ps, "plan_state", 2 * (size_t)n);
    PlanState s;
    std::memset(&s, 0, sizeof s);
    s.current = cfg.selector.mode == STABGPU_FORCE_SIMILARITY ? STABGPU_SIMILARITY : STABGPU_RIGID;
    s.since = 0;
    s.pending = 1;
    std::vector<PlanState> z(2 * (size_t)n);
    std::memset(z.data(), 0, z.size() * sizeof(PlanState));
    for (int k = 0; k < n; ++k) z[k] = s;
    CUDA_TRY(cudaMemcpyAsync(ps, z.data(), z.size() * sizeof(PlanState), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    *out = ps;
    return STABGPU_OK;
}

int plan_error(stabgpu_ctx* ctx, PlanState* ps, int n = 1) {
    std::vector<int> err(n, 0);
    CUDA_TRY(cudaMemcpyAsync(err.data(), reinterpret_cast<int*>(ps + n), n * sizeof(int),
                             cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < n; ++k) {
        if (!err[k]) continue;
        const int code = err[k] & 0xf;
        const long long f = err[k] >> 4;
        const std::string where = n > 1 ? "stream " + std::to_string(k) + " " : std::string();
        return set_err(code, code == STABGPU_DEGENERATE_INPUT
                                 ? "%sframe %lld: degenerate point set (all source points coincide or non-positive scale)"
                                 : "%sframe %lld: estimation failed",
                       where.c_str(), f);
    }
    return STABGPU_OK;
}

int validate_all(const stabgpu_config& c) {
    TRY(validate_detect(c.detect));
    TRY(validate_flow(c.flow));
    if (c.smooth_radius < 1) return set_err(STABGPU_INVALID_CONFIG, "smoothing radius must be >= 1");
    if (c.selector.dwell < 1) return set_err(STABGPU_INVALID_CONFIG, "dwell must be >= 1");
    if (c.selector.margin < 0.0) return set_err(STABGPU_INVALID_CONFIG, "margin must be >= 0");
    TRY(validate_crop(c.crop_ratio));
    if (c.queue_capacity < 2 * (size_t)c.smooth_radius + 4)
        return set_err(STABGPU_INVALID_CONFIG, "queue_capacity must be >= 2*radius + 4");
    if (c.flow.window_radius > STABGPU_MAX_RADIUS)
        return set_err(STABGPU_INVALID_CONFIG, "window_radius above 31 is not supported");
    if (c.ransac.iterations < 0 || (c.ransac.iterations > 0 && !(c.ransac.threshold > 0.0)))
        return set_err(STABGPU_INVALID_CONFIG, "ransac needs iterations >= 0 and threshold > 0");
    // hypothesis indices stay in int with the scoring strides (h + 32 * stride)
    if (c.ransac.iterations > STABGPU_MAX_RANSAC_ITERATIONS)
        return set_err(STABGPU_INVALID_CONFIG, "ransac iterations above 2^24 are not supported");
    if (c.selector.mode < 0 || c.selector.mode > 2)
        return set_err(STABGPU_INVALID_CONFIG, "unknown selection mode");
    return STABGPU_OK;
}

int compose_range(stabgpu_ctx* ctx, const uint8_t* y, const uint8_t* cb, const uint8_t* cr,
                  long long first, long long count, int w, int h, int cw, int ch,
                  const FramePlan* plan, double crop, uint8_t* oy, uint8_t* ocb, uint8_t* ocr) {
    if (count <= 0) return STABGPU_OK;
    const size_t lo = (size_t)first * w * h, co = (size_t)first * cw * ch;
    PlaneBatch yb{y + lo, (size_t)w * h, w, h};
    PlaneBatch bb{cb ? cb + co : nullptr, (size_t)cw * ch, cw, ch};
    PlaneBatch rb{cr ? cr + co : nullptr, (size_t)cw * ch, cw, ch};
    launch_compose(yb, bb, rb, plan + first, (int)count, crop, oy + lo, ocb ? ocb + co : nullptr,
                   ocr ? ocr + co : nullptr, ctx->stream);
    ctx->stats.launches += (cb && cr) ? 2 : 1;
    return check_launch("compose");
}

}  // namespace

// =====================================================================
extern "C" {

const char* stabgpu_last_error(void) { return g_err.c_str(); }
const char* stabgpu_version(void) { return "stabgpu 0.1 (sm_100a)"; }

void stabgpu_default_config(stabgpu_config* c) {
    std::memset(c, 0, sizeof *c);
    c->detect = {50, 0.01, 10.0, 3, 0.1};
    c->flow = {10, 4, 30, 0.01, 0.5, 5, 8};
    c->smooth_radius = 10;
    c->selector = {20, 0.05, STABGPU_HYBRID};
    c->ransac = {0, 3.0, 0};
    c->crop_ratio = 0.04;
    c->queue_capacity = 64;
}

int stabgpu_validate_config(const stabgpu_config* c) { return validate_all(*c); }

int stabgpu_create(int device, stabgpu_ctx** out) {
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return set_err(STABGPU_CUDA, "no CUDA device available (stabgpu has no CPU fallback)");
    }
    if (device < 0 || device >= n) return set_err(STABGPU_CUDA, "device %d out of range", device);
    CUDA_TRY(cudaSetDevice(device));
    stabgpu_ctx* c = new stabgpu_ctx();
    c->device = device;
    CUDA_TRY(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->cin, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->cout, cudaStreamNonBlocking));
    c->stream = c->own;
    CUDA_TRY(cudaMallocHost((void**)&c->iters_host, 4 * sizeof(unsigned long long)));
    // Per-launch tables come from the stream-ordered allocator; keep freed
    // blocks mapped so repeated launches do not remap device memory.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    *out = c;
    return STABGPU_OK;
}

int stabgpu_destroy(stabgpu_ctx* c) {
    if (!c) return STABGPU_OK;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto& kv : c->bufs)
        if (kv.second.p) cudaFree(kv.second.p);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->iters_host) cudaFreeHost(c->iters_host);
    if (c->comm) nccl_api().comm_destroy(c->comm);
    cudaStreamDestroy(c->own);
    cudaStreamDestroy(c->cin);
    cudaStreamDestroy(c->cout);
    delete c;
    return STABGPU_OK;
}

int stabgpu_set_stream(stabgpu_ctx* c, void* s) {
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own;
    return STABGPU_OK;
}

int stabgpu_synchronize(stabgpu_ctx* c) {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return STABGPU_OK;
}

int stabgpu_enable_timing(stabgpu_ctx* c, int on) {
    c->timing = on != 0;
    return STABGPU_OK;
}

int stabgpu_get_stats(stabgpu_ctx* c, stabgpu_stats* out) {
    cudaSetDevice(c->device);
    harvest_timing(c);
    *out = c->stats;
    return STABGPU_OK;
}

int stabgpu_debug_read_scratch(stabgpu_ctx* c, const char* name, void* host, size_t bytes, size_t* have) {
    cudaSetDevice(c->device);
    auto it = c->bufs.find(name);
    if (it == c->bufs.end() || !it->second.p) {
        if (have) *have = 0;
        return set_err(STABGPU_INVALID_INPUT, "no scratch buffer named '%s'", name);
    }
    if (have) *have = it->second.n;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    const size_t nb = std::min(bytes, it->second.n);
    if (host && nb) CUDA_TRY(cudaMemcpy(host, it->second.p, nb, cudaMemcpyDeviceToHost));
    return STABGPU_OK;
}

size_t stabgpu_pyramid_bytes(int w, int h, int max_levels) {
    int lw[STABGPU_MAX_LEVELS], lh[STABGPU_MAX_LEVELS];
    if (w < 1 || h < 1 || max_levels < 1) return 0;
    const int L = level_dims(w, h, max_levels, lw, lh);
    size_t t = 0;
    for (int l = 0; l < L; ++l) t += (size_t)lw[l] * lh[l];
    return t;
}

// ---- per-stage ABI ----------------------------------------------------

int stabgpu_build_pyramid_batch(stabgpu_ctx* ctx, const uint8_t* src, int nframes, int w, int h,
                                int max_levels, uint8_t* out) {
    TRY(validate_frame(w, h));
    if (max_levels < 1) return set_err(STABGPU_INVALID_INPUT, "max_levels must be >= 1");
    if (nframes < 1) return set_err(STABGPU_INVALID_INPUT, "build_pyramid_batch needs at least 1 frame");
    cudaSetDevice(ctx->device);
    int lw[STABGPU_MAX_LEVELS], lh[STABGPU_MAX_LEVELS];
    const int L = level_dims(w, h, max_levels, lw, lh);
    const size_t per = stabgpu_pyramid_bytes(w, h, max_levels);
    cudaStream_t st = ctx->stream;
    // the Stage I layout: one [frames][h_l][w_l] array per level, one launch per level
    DBUF(uint8_t, d, "api_pyr_batch", per * nframes);
    CUDA_TRY(cudaMemcpyAsync(d, src, (size_t)w * h * nframes, cudaMemcpyHostToDevice, st));
    size_t lvl_off = 0, pk_off = 0;
    for (int l = 0; l < L; ++l) {
        const size_t stride = (size_t)lw[l] * lh[l];
        if (l > 0) {
            const size_t pstride = (size_t)lw[l - 1] * lh[l - 1];
            launch_pyramid_level(d + lvl_off - pstride * nframes, pstride, lw[l - 1], lh[l - 1], d + lvl_off, stride,
                                 nframes, st);
            ++ctx->stats.launches;
        }
        // frame f's level l goes to out + f * per + pk_off (stabgpu_pyramid packing)
        CUDA_TRY(cudaMemcpy2DAsync(out + pk_off, per, d + lvl_off, stride, stride, nframes, cudaMemcpyDeviceToHost, st));
        lvl_off += stride * nframes;
        pk_off += stride;
    }
    TRY(check_launch("pyramid"));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

int stabgpu_build_pyramid(stabgpu_ctx* ctx, const uint8_t* src, int w, int h, int max_levels,
                          stabgpu_pyramid* out) {
    TRY(validate_frame(w, h));
    if (max_levels < 1) return set_err(STABGPU_INVALID_INPUT, "max_levels must be >= 1");
    cudaSetDevice(ctx->device);
    int lw[STABGPU_MAX_LEVELS], lh[STABGPU_MAX_LEVELS];
    const int L = level_dims(w, h, max_levels, lw, lh);
    const size_t total = stabgpu_pyramid_bytes(w, h, max_levels);
    DBUF(uint8_t, d, "api_pyr", total);
    cudaStream_t st = ctx->stream;
    CUDA_TRY(cudaMemcpyAsync(d, src, (size_t)w * h, cudaMemcpyHostToDevice, st));
    size_t off = 0;
    out->levels = L;
    for (int l = 0; l < L; ++l) {
        out->width[l] = lw[l];
        out->height[l] = lh[l];
        out->offset[l] = off;
        if (l > 0) {
            launch_pyramid_level(d + out->offset[l - 1], 0, lw[l - 1], lh[l - 1], d + off, 0, 1, st);
            ++ctx->stats.launches;
        }
        off += (size_t)lw[l] * lh[l];
    }
    TRY(check_launch("pyramid"));
    CUDA_TRY(cudaMemcpyAsync(out->data, d, total, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

int stabgpu_gradients(stabgpu_ctx* ctx, const uint8_t* src, int w, int h, double* gx, double* gy) {
    TRY(validate_frame(w, h));
    cudaSetDevice(ctx->device);
    const size_t n = (size_t)w * h;
    DBUF(uint8_t, d, "api_img", n);
    DBUF(double, g, "api_grad", 2 * n);
    cudaStream_t st = ctx->stream;
    CUDA_TRY(cudaMemcpyAsync(d, src, n, cudaMemcpyHostToDevice, st));
    launch_gradients(d, w, h, g, g + n, st);
    ++ctx->stats.launches;
    TRY(check_launch("gradients"));
    CUDA_TRY(cudaMemcpyAsync(gx, g, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(gy, g + n, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

int stabgpu_min_eig_response(stabgpu_ctx* ctx, const uint8_t* src, int w, int h, int block,
                             double* out) {
    TRY(validate_frame(w, h));
    if (block < 3 || block % 2 == 0)
        return set_err(STABGPU_INVALID_CONFIG, "block_size must be odd and >= 3");
    cudaSetDevice(ctx->device);
    const size_t n = (size_t)w * h;
    DBUF(uint8_t, d, "api_img", n);
    DBUF(double, r, "api_resp", n);
    cudaStream_t st = ctx->stream;
    CUDA_TRY(cudaMemcpyAsync(d, src, n, cudaMemcpyHostToDevice, st));
    launch_min_eig(d, w, h, block, r, st);
    ++ctx->stats.launches;
    TRY(check_launch("min_eig"));
    CUDA_TRY(cudaMemcpyAsync(out, r, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

int stabgpu_detection_roi(int w, int h, double margin, stabgpu_roi* out) {
    return roi_of(w, h, margin, out);
}

int stabgpu_detect_corners(stabgpu_ctx* ctx, const uint8_t* src, int w, int h,
                           const stabgpu_detect_cfg* cfg, double* xy, double* score, int* n_out) {
    return stabgpu_detect_corners_batch(ctx, src, 1, w, h, cfg, xy, score, n_out);
}

int stabgpu_detect_corners_batch(stabgpu_ctx* ctx, const uint8_t* src, int nframes, int w, int h,
                                 const stabgpu_detect_cfg* cfg, double* xy, double* score, int* n_out) {
    for (int f = 0; f < nframes; ++f) n_out[f] = 0;
    TRY(validate_frame(w, h));
    TRY(validate_detect(*cfg));
    if (nframes < 1) return set_err(STABGPU_INVALID_INPUT, "detect_corners_batch needs at least 1 frame");
    stabgpu_roi roi;
    TRY(roi_of(w, h, cfg->roi_margin, &roi));
    cudaSetDevice(ctx->device);
    const size_t n = (size_t)w * h, cap = (size_t)(roi.x1 - roi.x0) * (roi.y1 - roi.y0);
    const int maxc = cfg->max_corners, nb = nframes;
    cudaStream_t st = ctx->stream;
    DBUF(uint8_t, d, "api_img", n * nb);
    DBUF(unsigned long long, maxbits, "det_max", nb);
    DBUF(unsigned int, dcount, "det_count", nb);
    DBUF(unsigned long long, ckey, "det_ckey", cap * nb);
    DBUF(unsigned int, cidx, "det_cidx", cap * nb);
    DBUF(unsigned long long, skey, "det_skey", cap * nb);
    DBUF(unsigned int, sidx, "det_sidx", cap * nb);
    DBUF(double2, pts, "api_pts", (size_t)maxc * nb);
    DBUF(double, sc, "api_score", (size_t)maxc * nb);
    DBUF(int, nn, "api_n", nb);
    CUDA_TRY(cudaMemcpyAsync(d, src, n * nb, cudaMemcpyHostToDevice, st));
    DBUF(unsigned int, dhist, "det_hist", (size_t)kRespBins * nb);
    DBUF(double, dlo, "det_lo", nb);
    DBUF(unsigned char, dflags, "det_flags", nb);
    DBUF(unsigned, dmlo, "det_mlo", nb);
    DetectScratch ds{maxbits, dcount, dhist, ckey, cidx, skey, sidx, cap, dlo, dflags, dmlo};
    PlaneBatch fb{d, n, w, h};
    launch_detect(fb, nb, *cfg, roi, ds, pts, sc, nn, st);
    ctx->stats.launches += 3;
    TRY(check_launch("detect"));
    std::vector<int> nc(nb);
    CUDA_TRY(cudaMemcpyAsync(nc.data(), nn, sizeof(int) * nb, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int f = 0; f < nb; ++f)
        if (nc[f] > 0) {
            CUDA_TRY(cudaMemcpyAsync(xy + (size_t)2 * maxc * f, pts + (size_t)maxc * f, sizeof(double2) * nc[f],
                                     cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(score + (size_t)maxc * f, sc + (size_t)maxc * f, sizeof(double) * nc[f],
                                     cudaMemcpyDeviceToHost, st));
        }
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int f = 0; f < nb; ++f) n_out[f] = nc[f];
    return STABGPU_OK;
}

namespace {
int check_pyramids(const stabgpu_pyramid* a, const stabgpu_pyramid* b) {  // flow.cpp:229-239
    if (a->levels < 1 || b->levels < 1 || a->levels != b->levels)
        return set_err(STABGPU_INVALID_INPUT, "pyramids must have matching level counts");
    for (int i = 0; i < a->levels; ++i)
        if (a->width[i] != b->width[i] || a->height[i] != b->height[i])
            return set_err(STABGPU_INVALID_INPUT, "pyramid levels differ in size");
    return STABGPU_OK;
}

// Uploads two host pyramids as a 2-frame batched DevPyramid.
int upload_pair(stabgpu_ctx* ctx, const stabgpu_pyramid* a, const stabgpu_pyramid* b, DevPyramid* P) {
    std::memset(P, 0, sizeof *P);
    P->levels = a->levels;
    cudaStream_t st = ctx->stream;
    for (int l = 0; l < a->levels; ++l) {
        P->w[l] = a->width[l];
        P->h[l] = a->height[l];
        P->stride[l] = (size_t)a->width[l] * a->height[l];
        DBUF(uint8_t, d, ("api_pair" + std::to_string(l)).c_str(), 2 * P->stride[l]);
        CUDA_TRY(cudaMemcpyAsync(d, a->data + a->offset[l], P->stride[l], cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(d + P->stride[l], b->data + b->offset[l], P->stride[l],
                                 cudaMemcpyHostToDevice, st));
        P->lvl[l] = d;
    }
    return STABGPU_OK;
}

int run_lk_api(stabgpu_ctx* ctx, const stabgpu_pyramid* prev, const stabgpu_pyramid* cur,
               const double* pts, const double* ref, int n, const stabgpu_flow_cfg* cfg, int mode,
               double* out_xy, uint8_t* ok) {
    TRY(validate_flow(*cfg));
    TRY(check_pyramids(prev, cur));
    if (cfg->window_radius > STABGPU_MAX_RADIUS)
        return set_err(STABGPU_INVALID_CONFIG, "window_radius above 31 is not supported");
    if (n <= 0) return STABGPU_OK;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    DevPyramid P;
    TRY(upload_pair(ctx, prev, cur, &P));
    DBUF(double2, dp, "api_lk_pts", n);
    DBUF(double2, dr, "api_lk_ref", n);
    DBUF(double2, df, "api_lk_fwd", n);
    DBUF(uint8_t, dk, "api_lk_keep", n);
    DBUF(int, dn, "api_lk_n", 1);
    DBUF(unsigned, lk_work, "lk_work", 1);
    CUDA_TRY(cudaMemcpyAsync(dp, pts, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    if (ref) CUDA_TRY(cudaMemcpyAsync(dr, ref, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dn, &n, sizeof n, cudaMemcpyHostToDevice, st));
    LkStep s;
    s.pyr = P;
    s.frame0 = 0;
    s.seg_len = 1;
    s.t = 1;
    s.nseg = 1;
    s.max_pts = n;
    s.pts = dp;
    s.npts = dn;
    s.fwd = df;
    s.keep = dk;
    s.iter_count = nullptr;
    s.nframes = 2;
    s.mode = mode;
    s.ref = dr;
    s.work = lk_work;
    launch_lk(s, *cfg, st);
    ++ctx->stats.launches;
    TRY(check_launch("track_lk"));
    if (out_xy) CUDA_TRY(cudaMemcpyAsync(out_xy, df, sizeof(double2) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(ok, dk, n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}
}  // namespace

int stabgpu_track_lk(stabgpu_ctx* ctx, const stabgpu_pyramid* prev, const stabgpu_pyramid* cur,
                     const double* xy, int n, const stabgpu_flow_cfg* cfg, double* out_xy,
                     uint8_t* ok) {
    const int rc = run_lk_api(ctx, prev, cur, xy, nullptr, n, cfg, 0, out_xy, ok);
    if (rc == STABGPU_OK)  // failed points keep their input position (flow.cpp:162-164)
        for (int i = 0; i < n; ++i)
            if (!ok[i]) {
                out_xy[2 * i] = xy[2 * i];
                out_xy[2 * i + 1] = xy[2 * i + 1];
            }
    return rc;
}

int stabgpu_weed_tracks(stabgpu_ctx* ctx, const stabgpu_pyramid* prev, const stabgpu_pyramid* cur,
                        const double* pxy, const double* cxy, int n, const stabgpu_flow_cfg* cfg,
                        double* kp, double* kc, int* n_out) {
    *n_out = 0;
    if (n == 0) return STABGPU_OK;  // weed_tracks returns before track_lk (flow.cpp:264-266)
    std::vector<uint8_t> keep(n);
    TRY(run_lk_api(ctx, prev, cur, cxy, pxy, n, cfg, 2, nullptr, keep.data()));
    int m = 0;
    for (int i = 0; i < n; ++i)
        if (keep[i]) {
            kp[2 * m] = pxy[2 * i];
            kp[2 * m + 1] = pxy[2 * i + 1];
            kc[2 * m] = cxy[2 * i];
            kc[2 * m + 1] = cxy[2 * i + 1];
            ++m;
        }
    *n_out = m;
    return STABGPU_OK;
}

namespace {
int fit_api(stabgpu_ctx* ctx, const double* p, const double* q, int n, int kind,
            const stabgpu_ransac_cfg* rc, int min_tracks, long long frame, stabgpu_transform* out,
            uint8_t* inliers, int* n_used) {
    if (n < 2) return set_err(STABGPU_DEGENERATE_INPUT, "estimation needs at least 2 point pairs");
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    DBUF(double2, dp, "api_fit_p", n);
    DBUF(double2, dq, "api_fit_q", n);
    DBUF(uint8_t, dm, "api_fit_m", n);
    DBUF(FitResult, dr, "api_fit_r", 1);
    CUDA_TRY(cudaMemcpyAsync(dp, p, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dq, q, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    stabgpu_ransac_cfg off{0, 0.0, 0};
    launch_fit_single(dp, dq, n, kind, rc ? *rc : off, min_tracks, frame, dr, dm, st);
    ++ctx->stats.launches;
    TRY(check_launch("fit"));
    FitResult r;
    CUDA_TRY(cudaMemcpyAsync(&r, dr, sizeof r, cudaMemcpyDeviceToHost, st));
    if (inliers) CUDA_TRY(cudaMemcpyAsync(inliers, dm, n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (r.status)
        return set_err(r.status, "estimation failed: degenerate point set (coincident points or non-positive scale)");
    out->tx = r.tx;
    out->ty = r.ty;
    out->theta = r.theta;
    out->s = r.s;
    out->kind = kind == STABGPU_RIGID ? STABGPU_RIGID : STABGPU_SIMILARITY;
    if (n_used) *n_used = r.used;
    return STABGPU_OK;
}
}  // namespace

int stabgpu_estimate(stabgpu_ctx* ctx, const double* p, const double* q, int n, int kind,
                     stabgpu_transform* out) {
    return fit_api(ctx, p, q, n, kind, nullptr, 0, 0, out, nullptr, nullptr);
}

int stabgpu_ransac_estimate(stabgpu_ctx* ctx, const double* p, const double* q, int n, int kind,
                            const stabgpu_ransac_cfg* rc, int min_tracks, int64_t frame,
                            stabgpu_transform* out, uint8_t* inliers, int* n_inliers) {
    if (rc && (rc->iterations < 0 || (rc->iterations > 0 && !(rc->threshold > 0.0))))
        return set_err(STABGPU_INVALID_CONFIG, "ransac needs iterations >= 0 and threshold > 0");
    return fit_api(ctx, p, q, n, kind, rc, min_tracks, frame, out, inliers, n_inliers);
}

int stabgpu_rms_residual(stabgpu_ctx* ctx, const double* p, const double* q, int n,
                         const stabgpu_transform* t, double* out) {
    if (n == 0) return set_err(STABGPU_DEGENERATE_INPUT, "rms_residual needs a non-empty track set");
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    DBUF(double2, dp, "api_fit_p", n);
    DBUF(double2, dq, "api_fit_q", n);
    DBUF(double, dr, "api_rms", 1);
    CUDA_TRY(cudaMemcpyAsync(dp, p, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dq, q, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    launch_rms_single(dp, dq, n, *t, dr, st);
    ++ctx->stats.launches;
    TRY(check_launch("rms"));
    CUDA_TRY(cudaMemcpyAsync(out, dr, sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

void stabgpu_extract_delta(const stabgpu_transform* t, stabgpu_delta* d) {  // motion.cpp:92-101
    d->dx = t->tx;
    d->dy = t->ty;
    d->da = t->theta;
    d->dls = t->kind == STABGPU_RIGID ? 0.0 : std::log(t->s);
    d->kind = t->kind;
    d->skipped = 0;
}

void stabgpu_delta_to_transform(double dx, double dy, double da, double dls, stabgpu_transform* t) {
    t->tx = dx;  // motion.cpp:103-111
    t->ty = dy;
    t->theta = da;
    t->s = std::exp(dls);
    t->kind = STABGPU_SIMILARITY;
}

int stabgpu_trajectory_corrections(stabgpu_ctx* ctx, const stabgpu_delta* deltas, int n, int radius,
                                   stabgpu_transform* out) {
    if (radius < 1) return set_err(STABGPU_INVALID_CONFIG, "smoothing radius must be >= 1");
    if (n <= 0) return STABGPU_OK;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    DBUF(stabgpu_delta, dd, "api_deltas", n);
    DBUF(double4, cum, "api_cum", n);
    DBUF(stabgpu_frame_record, rec, "api_rec", n);
    DBUF(FramePlan, plan, "api_plan", n);
    CUDA_TRY(cudaMemcpyAsync(dd, deltas, sizeof(stabgpu_delta) * n, cudaMemcpyHostToDevice, st));
    launch_prefix(dd, n, cum, st);
    launch_plan_smooth(cum, n, true, 0, n, radius, rec, plan, PlanGeom{16, 16, 0, 0, 0.0}, st);
    ctx->stats.launches += 2;
    TRY(check_launch("trajectory"));
    std::vector<stabgpu_frame_record> h(n);
    CUDA_TRY(cudaMemcpyAsync(h.data(), rec, sizeof(stabgpu_frame_record) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int i = 0; i < n; ++i) out[i] = h[i].correction;
    return STABGPU_OK;
}

int stabgpu_warp_similarity(stabgpu_ctx* ctx, const uint8_t* src, int w, int h,
                            const stabgpu_transform* t, uint8_t* out) {
    TRY(validate_frame(w, h));
    TRY(validate_transform(*t));
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const size_t n = (size_t)w * h;
    DBUF(uint8_t, d, "api_img", n);
    DBUF(uint8_t, o, "api_out", n);
    DBUF(FramePlan, plan, "api_plan1", 1);
    FramePlan p = host_plan(*t);
    finish_plan(p, w, h, 0, 0, 0.0);
    CUDA_TRY(cudaMemcpyAsync(d, src, n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(plan, &p, sizeof p, cudaMemcpyHostToDevice, st));
    launch_warp_only(d, w, h, plan, o, st);
    ++ctx->stats.launches;
    TRY(check_launch("warp"));
    CUDA_TRY(cudaMemcpyAsync(out, o, n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

int stabgpu_crop_resize(stabgpu_ctx* ctx, const uint8_t* src, int w, int h, double crop,
                        uint8_t* out) {
    TRY(validate_frame(w, h));
    TRY(validate_crop(crop));
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const size_t n = (size_t)w * h;
    DBUF(uint8_t, d, "api_img", n);
    DBUF(uint8_t, o, "api_out", n);
    CUDA_TRY(cudaMemcpyAsync(d, src, n, cudaMemcpyHostToDevice, st));
    launch_crop_only(d, w, h, crop, o, st);
    ++ctx->stats.launches;
    TRY(check_launch("crop"));
    CUDA_TRY(cudaMemcpyAsync(out, o, n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

int stabgpu_compose_stabilized(stabgpu_ctx* ctx, const uint8_t* y, const uint8_t* cb,
                               const uint8_t* cr, int w, int h, int cw, int ch,
                               const stabgpu_transform* t, double crop, uint8_t* oy, uint8_t* ocb,
                               uint8_t* ocr) {
    TRY(validate_frame(w, h));
    TRY(validate_transform(*t));
    TRY(validate_crop(crop));
    const bool chroma = cb && cr;
    if (chroma && (cw < 1 || ch < 1)) return set_err(STABGPU_INVALID_INPUT, "bad chroma geometry");
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const size_t n = (size_t)w * h, nc = chroma ? (size_t)cw * ch : 0;
    DBUF(uint8_t, d, "api_cmp_in", n + 2 * nc);
    DBUF(uint8_t, o, "api_cmp_out", n + 2 * nc);
    DBUF(FramePlan, plan, "api_plan1", 1);
    FramePlan p = host_plan(*t);
    finish_plan(p, w, h, chroma ? cw : 0, chroma ? ch : 0, crop);
    CUDA_TRY(cudaMemcpyAsync(plan, &p, sizeof p, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d, y, n, cudaMemcpyHostToDevice, st));
    if (chroma) {
        CUDA_TRY(cudaMemcpyAsync(d + n, cb, nc, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(d + n + nc, cr, nc, cudaMemcpyHostToDevice, st));
    }
    PlaneBatch yb{d, n, w, h};
    PlaneBatch bb{chroma ? d + n : nullptr, nc, cw, ch};
    PlaneBatch rb{chroma ? d + n + nc : nullptr, nc, cw, ch};
    launch_compose(yb, bb, rb, plan, 1, crop, o, chroma ? o + n : nullptr, chroma ? o + n + nc : nullptr, st);
    ctx->stats.launches += chroma ? 2 : 1;
    TRY(check_launch("compose"));
    CUDA_TRY(cudaMemcpyAsync(oy, o, n, cudaMemcpyDeviceToHost, st));
    if (chroma) {
        CUDA_TRY(cudaMemcpyAsync(ocb, o + n, nc, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(ocr, o + n + nc, nc, cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

// ---- Stage I ------------------------------------------------------------

int stabgpu_stabilize_sequence_device(stabgpu_ctx* ctx, const uint8_t* y, const uint8_t* cb,
                                      const uint8_t* cr, int n, int w, int h, int cw, int ch,
                                      const stabgpu_config* cfgp, uint8_t* oy, uint8_t* ocb,
                                      uint8_t* ocr, stabgpu_frame_record* records) {
    const stabgpu_config cfg = *cfgp;
    TRY(validate_all(cfg));
    TRY(validate_frame(w, h));
    if (n < 2) return set_err(STABGPU_INVALID_INPUT, "stabilization needs at least 2 frames");
    cudaSetDevice(ctx->device);
    begin_timing(ctx);
    cudaStream_t st = ctx->stream;
    DBUF(stabgpu_motion_record, motion, "seq_motion", n);
    DBUF(stabgpu_frame_record, rec, "seq_rec", n);
    DBUF(double4, cum, "seq_cum", n);
    DBUF(FramePlan, plan, "seq_plan", n);
    PlanState* ps;
    TRY(init_plan_state(ctx, cfg, &ps));
    TRY(run_motion(ctx, y, 0, n - 1, w, h, cfg, motion));
    {
        Timer tm(ctx, 5);
        launch_plan_scan(motion, 0, n, cfg, ps, rec, cum, st);
        launch_plan_smooth(cum, n, true, 0, n, cfg.smooth_radius, rec, plan,
                           PlanGeom{w, h, cb ? cw : 0, cb ? ch : 0, cfg.crop_ratio}, st);
    }
    ctx->stats.launches += 2;
    TRY(check_launch("plan"));
    {
        Timer tm(ctx, 4);
        TRY(compose_range(ctx, y, cb, cr, 0, n, w, h, cw, ch, plan, cfg.crop_ratio, oy, ocb, ocr));
    }
    TRY(plan_error(ctx, ps));
    if (records)
        CUDA_TRY(cudaMemcpyAsync(records, rec, sizeof(stabgpu_frame_record) * n,
                                 cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

// ---- multi-stream Stage I (BASELINE c5) -----------------------------------
// n_streams independent sequences of `frames` frames each, stream-major.
// Every stage runs once over all of them: one pyramid launch per level, the
// detections batched, one LK chain launch over every segment of every stream,
// one fit launch, one scan block per stream, one compose launch.  Each
// stream's output and records equal run_offline (pipeline.cpp:182-235) on
// that stream alone.
}  // extern "C"
namespace {
int validate_streams(const stabgpu_config& cfg, int n_streams, int frames, int w, int h) {
    TRY(validate_all(cfg));
    TRY(validate_frame(w, h));
    if (n_streams < 1) return set_err(STABGPU_INVALID_INPUT, "n_streams must be >= 1");
    if (frames < 2) return set_err(STABGPU_INVALID_INPUT, "stabilization needs at least 2 frames");
    if ((long long)n_streams * frames > INT32_MAX / 2)
        return set_err(STABGPU_INVALID_INPUT, "too many frames in one call");
    return STABGPU_OK;
}

// One group of streams on ctx->stream, queued without a host sync.  motion,
// rec, cum, plan point at the group's first frame; ps / err at its first
// stream's state and error word.
int streams_group(stabgpu_ctx* ctx, const uint8_t* y, const uint8_t* cb, const uint8_t* cr,
                  int S, int F, int w, int h, int cw, int ch, const stabgpu_config& cfg, uint8_t* oy,
                  uint8_t* ocb, uint8_t* ocr, stabgpu_motion_record* motion, stabgpu_frame_record* rec,
                  double4* cum, FramePlan* plan, PlanState* ps, int* err) {
    cudaStream_t st = ctx->stream;
    const long long n = (long long)S * F;
    TRY(run_motion(ctx, y, 0, (int)(n - 1), w, h, cfg, motion, S));
    {
        Timer tm(ctx, 5);
        launch_plan_scan(motion, 0, F, cfg, ps, rec, cum, st, S, F, err);
        launch_plan_smooth(cum, F, true, 0, n, cfg.smooth_radius, rec, plan,
                           PlanGeom{w, h, cb ? cw : 0, cb ? ch : 0, cfg.crop_ratio}, st, F);
    }
    ctx->stats.launches += 2;
    TRY(check_launch("plan"));
    {
        Timer tm(ctx, 4);
        TRY(compose_range(ctx, y, cb, cr, 0, n, w, h, cw, ch, plan, cfg.crop_ratio, oy, ocb, ocr));
    }
    return STABGPU_OK;
}

}  // namespace
extern "C" {

int stabgpu_stabilize_streams_device(stabgpu_ctx* ctx, const uint8_t* y, const uint8_t* cb,
                                     const uint8_t* cr, int n_streams, int frames, int w, int h,
                                     int cw, int ch, const stabgpu_config* cfgp, uint8_t* oy,
                                     uint8_t* ocb, uint8_t* ocr, stabgpu_frame_record* records) {
    const stabgpu_config cfg = *cfgp;
    TRY(validate_streams(cfg, n_streams, frames, w, h));
    const bool chroma = cb && cr && ocb && ocr;
    if (!chroma) cb = cr = nullptr;
    cudaSetDevice(ctx->device);
    begin_timing(ctx);
    cudaStream_t st = ctx->stream;
    const long long n = (long long)n_streams * frames;
    DBUF(stabgpu_motion_record, motion, "seq_motion", n);
    DBUF(stabgpu_frame_record, rec, "seq_rec", n);
    DBUF(double4, cum, "seq_cum", n);
    DBUF(FramePlan, plan, "seq_plan", n);
    PlanState* ps;
    TRY(init_plan_state(ctx, cfg, &ps, n_streams));
    TRY(streams_group(ctx, y, cb, cr, n_streams, frames, w, h, cw, ch, cfg, oy, ocb, ocr, motion, rec,
                      cum, plan, ps, reinterpret_cast<int*>(ps + n_streams)));
    TRY(plan_error(ctx, ps, n_streams));
    if (records)
        CUDA_TRY(cudaMemcpyAsync(records, rec, sizeof(stabgpu_frame_record) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

// Host buffers: groups of streams (about 2 GB of luma each) flow through two
// device slots, so the upload of group g+1 and the download of group g-1
// overlap the compute of group g.
int stabgpu_stabilize_streams(stabgpu_ctx* ctx, const uint8_t* hy, const uint8_t* hcb,
                              const uint8_t* hcr, int n_streams, int frames, int w, int h, int cw,
                              int ch, const stabgpu_config* cfgp, uint8_t* hoy, uint8_t* hocb,
                              uint8_t* hocr, stabgpu_frame_record* records) {
    const stabgpu_config cfg = *cfgp;
    TRY(validate_streams(cfg, n_streams, frames, w, h));
    cudaSetDevice(ctx->device);
    begin_timing(ctx);
    cudaStream_t st = ctx->stream;
    const bool chroma = hcb && hcr && hocb && hocr;
    const size_t fl = (size_t)w * h, fc = chroma ? (size_t)cw * ch : 0;
    const size_t sl = fl * frames, sc = fc * frames;  // bytes per stream and plane
    int G = (int)std::max<size_t>(1, std::min<size_t>((size_t)n_streams, (2ull << 30) / (sl + 2 * sc)));
    if (const char* e = std::getenv("STABGPU_STREAMS_PER_GROUP"))  // test knob: force small groups
        G = std::max(1, std::min(n_streams, std::atoi(e)));
    const int ngroups = (n_streams + G - 1) / G;
    const long long n = (long long)n_streams * frames;
    uint8_t *dy[2], *doy[2], *dcb[2] = {nullptr, nullptr}, *dcr[2] = {nullptr, nullptr},
            *docb[2] = {nullptr, nullptr}, *docr[2] = {nullptr, nullptr};
    for (int k = 0; k < 2; ++k) {
        const std::string t = std::to_string(k);
        dy[k] = dbuf<uint8_t>(ctx, ("ms_y" + t).c_str(), sl * G);
        doy[k] = dbuf<uint8_t>(ctx, ("ms_oy" + t).c_str(), sl * G);
        if (!dy[k] || !doy[k]) return set_err(STABGPU_CUDA, "device allocation of stream slots failed");
        if (chroma) {
            dcb[k] = dbuf<uint8_t>(ctx, ("ms_cb" + t).c_str(), sc * G);
            dcr[k] = dbuf<uint8_t>(ctx, ("ms_cr" + t).c_str(), sc * G);
            docb[k] = dbuf<uint8_t>(ctx, ("ms_ocb" + t).c_str(), sc * G);
            docr[k] = dbuf<uint8_t>(ctx, ("ms_ocr" + t).c_str(), sc * G);
            if (!dcb[k] || !dcr[k] || !docb[k] || !docr[k])
                return set_err(STABGPU_CUDA, "device allocation of stream slots failed");
        }
    }
    DBUF(stabgpu_motion_record, motion, "seq_motion", n);
    DBUF(stabgpu_frame_record, rec, "seq_rec", n);
    DBUF(double4, cum, "seq_cum", n);
    DBUF(FramePlan, plan, "seq_plan", n);
    PlanState* ps;
    TRY(init_plan_state(ctx, cfg, &ps, n_streams));
    int* err = reinterpret_cast<int*>(ps + n_streams);
    // in_ev[g]: group g uploaded; done_ev[g]: group g computed (its input slot
    // is free); out_ev[g]: group g downloaded (its output slot is free)
    std::vector<cudaEvent_t> in_ev(ngroups), done_ev(ngroups), out_ev(ngroups);
    for (int g = 0; g < ngroups; ++g) {
        CUDA_TRY(cudaEventCreateWithFlags(&in_ev[g], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&done_ev[g], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&out_ev[g], cudaEventDisableTiming));
    }
    auto upload = [&](int g) -> int {
        const int k = g & 1, s0 = g * G, ns = std::min(G, n_streams - s0);
        if (g >= 2) cudaStreamWaitEvent(ctx->cin, done_ev[g - 2], 0);
        if (cudaMemcpyAsync(dy[k], hy + s0 * sl, ns * sl, cudaMemcpyHostToDevice, ctx->cin) ||
            (chroma && (cudaMemcpyAsync(dcb[k], hcb + s0 * sc, ns * sc, cudaMemcpyHostToDevice, ctx->cin) ||
                        cudaMemcpyAsync(dcr[k], hcr + s0 * sc, ns * sc, cudaMemcpyHostToDevice, ctx->cin))))
            return set_err(STABGPU_CUDA, "upload failed: %s", cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(in_ev[g], ctx->cin);
        return STABGPU_OK;
    };
    int rc = upload(0);
    if (!rc && ngroups > 1) rc = upload(1);
    for (int g = 0; g < ngroups && !rc; ++g) {
        const int k = g & 1, s0 = g * G, ns = std::min(G, n_streams - s0);
        const long long f0 = (long long)s0 * frames;
        cudaStreamWaitEvent(st, in_ev[g], 0);
        if (g >= 2) cudaStreamWaitEvent(st, out_ev[g - 2], 0);
        rc = streams_group(ctx, dy[k], dcb[k], dcr[k], ns, frames, w, h, cw, ch, cfg, doy[k], docb[k],
                           docr[k], motion + f0, rec + f0, cum + f0, plan + f0, ps + s0, err + s0);
        if (rc) break;
        cudaEventRecord(done_ev[g], st);
        if (g + 2 < ngroups && (rc = upload(g + 2))) break;
        cudaStreamWaitEvent(ctx->cout, done_ev[g], 0);
        if (cudaMemcpyAsync(hoy + s0 * sl, doy[k], ns * sl, cudaMemcpyDeviceToHost, ctx->cout) ||
            (chroma && (cudaMemcpyAsync(hocb + s0 * sc, docb[k], ns * sc, cudaMemcpyDeviceToHost, ctx->cout) ||
                        cudaMemcpyAsync(hocr + s0 * sc, docr[k], ns * sc, cudaMemcpyDeviceToHost, ctx->cout))))
            rc = set_err(STABGPU_CUDA, "download failed: %s", cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(out_ev[g], ctx->cout);
    }
    cudaStreamSynchronize(ctx->cin);
    cudaStreamSynchronize(st);
    cudaStreamSynchronize(ctx->cout);
    for (int g = 0; g < ngroups; ++g) {
        cudaEventDestroy(in_ev[g]);
        cudaEventDestroy(done_ev[g]);
        cudaEventDestroy(out_ev[g]);
    }
    if (rc) return rc;
    TRY(plan_error(ctx, ps, n_streams));
    if (records)
        CUDA_TRY(cudaMemcpyAsync(records, rec, sizeof(stabgpu_frame_record) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

}  // extern "C"

namespace {

// Upload chunk boundaries 0 = b_0 < b_1 < ... < b_k = n: 60-frame chunks in
// the middle, ramped 10, 20, 40 frames at both ends when a 60-frame chunk is
// large (>= 256 MB: the copies bound the pipeline), so it fills (the first
// motion waits only for a 10-frame upload) and drains (the last compute
// releases the last chunk plus the smoothing tail, whose download is not
// overlapped) quickly.  Small frames keep flat chunks: there the per-chunk
// launches bound the pipeline (C1 e2e 42k flat vs 30k ramped).
std::vector<long long> chunk_bounds(long long n, size_t frame_bytes) {
    static const long long ramp[3] = {10, 20, 40};
    const bool flat = getenv("STABGPU_FLAT_CHUNKS") != nullptr || frame_bytes * 60 < (256ull << 20);
    std::vector<long long> sizes, tail;
    long long rem = n;
    if (flat) rem = 0;
    // flat chunks: each chunk's motion costs ~1 ms of launch- and latency-bound
    // work whatever its size (one select CTA per detection frame, one warp per
    // LK chain), so small frames take chunks of ~128 MB (at least 60 frames, at
    // most half the sequence so copies and compute still overlap): C1 runs as
    // 2 x 150 frames, C2 as 140-frame chunks
    long long cf = 60;
    if (flat) {
        if (const char* e = getenv("STABGPU_CHUNK_FRAMES")) cf = std::max(1, atoi(e));
        else {
            cf = (long long)((128ull << 20) / std::max<size_t>(frame_bytes, 1)) / 10 * 10;
            cf = std::max<long long>(60, std::min<long long>(cf, (n + 1) / 2));
        }
    }
    if (flat && n >= 3 * cf && cf >= 80 && !getenv("STABGPU_NO_FLAT_RAMP")) {
        // quarter and half chunks at both ends: the first motion starts and the
        // last download ends sooner
        const long long q = cf / 4 / 5 * 5, h2 = cf / 2 / 5 * 5;
        sizes.push_back(q);
        sizes.push_back(h2);
        long long mid = n - 2 * (q + h2);
        while (mid > 0) {
            const long long c = std::min(cf, mid);
            sizes.push_back(c);
            mid -= c;
        }
        sizes.push_back(h2);
        sizes.push_back(q);
    } else {
        for (long long f = 0; flat && f < n; f += cf) sizes.push_back(std::min<long long>(cf, n - f));
    }
    for (long long r : ramp)
        if (rem > r) {
            sizes.push_back(r);
            rem -= r;
        }
    for (long long r : ramp)
        if (rem > r + 60) {
            tail.push_back(r);
            rem -= r;
        }
    while (rem > 0) {
        const long long c = std::min<long long>(60, rem);
        sizes.push_back(c);
        rem -= c;
    }
    for (auto it = tail.rbegin(); it != tail.rend(); ++it) sizes.push_back(*it);
    std::vector<long long> b(1, 0);
    for (long long c : sizes) b.push_back(b.back() + c);
    return b;
}

// Host buffers: chunked upload -> motion -> incremental plan -> compose ->
// download, with the copies on two copy streams so upload, compute and
// download of different chunks overlap (PCIe is full duplex).
// RGB mode (hrgb / hout_rgb, interleaved 8-bit, 4:4:4): media_io's load /
// save conversions around run_offline.  Each uploaded chunk is converted
// (RGB -> Y/Cb/Cr) on the input copy stream as it lands — or, opt-in
// (STABGPU_RGB_ZEROCOPY), read and converted by the kernel itself straight
// from pinned host memory over PCIe — and K8 writes interleaved RGB
// (Y/Cb/Cr -> RGB fused into the compose store) when the geometry allows,
// else composes planes and converts.
int sequence_host(stabgpu_ctx* ctx, const uint8_t* hy, const uint8_t* hcb, const uint8_t* hcr, const uint8_t* hrgb,
                  int n, int w, int h, int cw, int ch, const stabgpu_config* cfgp, uint8_t* hoy, uint8_t* hocb,
                  uint8_t* hocr, uint8_t* hout_rgb, stabgpu_frame_record* records) {
    const stabgpu_config cfg = *cfgp;
    TRY(validate_all(cfg));
    TRY(validate_frame(w, h));
    if (n < 2) return set_err(STABGPU_INVALID_INPUT, "stabilization needs at least 2 frames");
    cudaSetDevice(ctx->device);
    begin_timing(ctx);
    cudaStream_t st = ctx->stream;
    const bool rgb = hrgb != nullptr;
    if (rgb) {
        cw = w;
        ch = h;
    }
    const bool chroma = rgb || (hcb && hcr && hocb && hocr);
    const size_t fl = (size_t)w * h, fc = chroma ? (size_t)cw * ch : 0;
    DBUF(uint8_t, dy, "io_y", fl * n);
    DBUF(uint8_t, doy, "io_oy", fl * n);
    // RGB: zero-copy upload when the host buffer is pinned (device-accessible)
    const uint8_t* zc_rgb = nullptr;
    uint8_t *drgb_in = nullptr, *drgb_out = nullptr;
    if (rgb) {
        cudaPointerAttributes pa;
        // Zero-copy is opt-in: alone it streams at 40-48 GB/s, but inside the
        // overlapped pipeline (downloads and compute running) it measured 4.1k
        // frames/s e2e at C3 against 6.7k for the copy-engine staging
        // (profiles/r2_rgb_probe.log), so the staged upload is the default.
        const bool zc_on = getenv("STABGPU_RGB_ZEROCOPY") != nullptr;
        if (zc_on && cudaPointerGetAttributes(&pa, hrgb) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer)
            zc_rgb = static_cast<const uint8_t*>(pa.devicePointer);
        cudaGetLastError();
        if (!zc_rgb) {
            DBUF(uint8_t, a, "io_rgb_in", 3 * fl * n);
            drgb_in = a;
        }
        DBUF(uint8_t, b, "io_rgb_out", 3 * fl * n);
        drgb_out = b;
    }
    uint8_t *dcb = nullptr, *dcr = nullptr, *docb = nullptr, *docr = nullptr;
    if (chroma) {
        DBUF(uint8_t, a, "io_cb", fc * n);
        DBUF(uint8_t, b, "io_cr", fc * n);
        DBUF(uint8_t, c, "io_ocb", fc * n);
        DBUF(uint8_t, d, "io_ocr", fc * n);
        dcb = a;
        dcr = b;
        docb = c;
        docr = d;
    }
    DBUF(stabgpu_motion_record, motion, "seq_motion", n);
    DBUF(stabgpu_frame_record, rec, "seq_rec", n);
    DBUF(double4, cum, "seq_cum", n);
    DBUF(FramePlan, plan, "seq_plan", n);
    PlanState* ps;
    TRY(init_plan_state(ctx, cfg, &ps));
    const int R = cfg.flow.redetect_interval;
    const std::vector<long long> cb = chunk_bounds(n, rgb ? 3 * fl : fl + 2 * fc);  // upload chunks
    const int nchunks = (int)cb.size() - 1;
    std::vector<cudaEvent_t> in_ev(nchunks), out_ev(nchunks + 1);
    for (auto& e : in_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : out_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    int rc = STABGPU_OK;
    // uploads, all queued up front on the input copy stream
    for (int k = 0; k < nchunks && !rc; ++k) {
        const size_t f0 = (size_t)cb[k], nf = (size_t)(cb[k + 1] - cb[k]);
        if (rgb) {
            const uint8_t* src = zc_rgb ? zc_rgb + 3 * f0 * fl : drgb_in + 3 * f0 * fl;
            if (!zc_rgb && cudaMemcpyAsync(drgb_in + 3 * f0 * fl, hrgb + 3 * f0 * fl, 3 * nf * fl,
                                           cudaMemcpyHostToDevice, ctx->cin))
                rc = set_err(STABGPU_CUDA, "upload failed: %s", cudaGetErrorString(cudaGetLastError()));
            launch_rgb_to_ycbcr(src, nf * fl, dy + f0 * fl, dcb + f0 * fl, dcr + f0 * fl, ctx->cin, zc_rgb != nullptr);
            ++ctx->stats.launches;
        } else if (cudaMemcpyAsync(dy + f0 * fl, hy + f0 * fl, nf * fl, cudaMemcpyHostToDevice, ctx->cin) ||
                   (chroma &&
                    (cudaMemcpyAsync(dcb + f0 * fc, hcb + f0 * fc, nf * fc, cudaMemcpyHostToDevice, ctx->cin) ||
                     cudaMemcpyAsync(dcr + f0 * fc, hcr + f0 * fc, nf * fc, cudaMemcpyHostToDevice, ctx->cin)))) {
            rc = set_err(STABGPU_CUDA, "upload failed: %s", cudaGetErrorString(cudaGetLastError()));
        }
        cudaEventRecord(in_ev[k], ctx->cin);
    }
    long long seg_done = 0;   // segments whose motion is computed
    long long known = 0;      // motion records known: frames [0, known)
    long long composed = 0;   // frames composed and queued for download
    const long long nseg_total = (n - 1 + R - 1) / R;
    const int r = cfg.smooth_radius;
    for (int k = 0; k < nchunks && !rc; ++k) {
        cudaStreamWaitEvent(st, in_ev[k], 0);
        const long long arrived = cb[k + 1];  // frames [0, arrived)
        // segments [s*R, min((s+1)R, n-1)] whose last frame has arrived
        long long seg_end = seg_done;
        while (seg_end < nseg_total && std::min<long long>((seg_end + 1) * R, n - 1) < arrived) ++seg_end;
        if (seg_end > seg_done) {
            const long long first = seg_done * R;
            const long long last = std::min<long long>(seg_end * R, n - 1);
            rc = run_motion(ctx, dy + first * fl, first, (int)(last - first), w, h, cfg, motion);
            if (rc) break;
            launch_plan_scan(motion, known, last + 1 - known, cfg, ps, rec, cum, st);
            ++ctx->stats.launches;
            known = last + 1;
            seg_done = seg_end;
        }
        const bool complete = known == n;
        const long long ready = complete ? n : std::max<long long>(0, known - r);
        if (ready > composed) {
            launch_plan_smooth(cum, known, complete, composed, ready - composed, r, rec, plan,
                               PlanGeom{w, h, chroma ? cw : 0, chroma ? ch : 0, cfg.crop_ratio}, st);
            ++ctx->stats.launches;
            const size_t f0 = composed, nf = ready - composed;
            if (rgb) {
                Timer tm(ctx, 4);
                PlaneBatch yb{dy + f0 * fl, fl, w, h}, bb{dcb + f0 * fl, fl, w, h}, cb2{dcr + f0 * fl, fl, w, h};
                if (!launch_compose_rgb(yb, bb, cb2, plan + f0, (int)nf, cfg.crop_ratio, drgb_out + 3 * f0 * fl, st)) {
                    // geometry without the fused store: planes, then the conversion
                    launch_compose(yb, bb, cb2, plan + f0, (int)nf, cfg.crop_ratio, doy + f0 * fl, docb + f0 * fl,
                                   docr + f0 * fl, st);
                    launch_ycbcr_to_rgb(doy + f0 * fl, docb + f0 * fl, docr + f0 * fl, nf * fl,
                                        drgb_out + 3 * f0 * fl, st);
                    ++ctx->stats.launches;
                }
                ++ctx->stats.launches;
                rc = check_launch("compose");
            } else {
                rc = compose_range(ctx, dy, dcb, dcr, composed, ready - composed, w, h, cw, ch, plan,
                                   cfg.crop_ratio, doy, docb, docr);
            }
            if (rc) break;
            cudaEventRecord(out_ev[k], st);
            cudaStreamWaitEvent(ctx->cout, out_ev[k], 0);
            if (rgb) {
                if (cudaMemcpyAsync(hout_rgb + 3 * f0 * fl, drgb_out + 3 * f0 * fl, 3 * nf * fl,
                                    cudaMemcpyDeviceToHost, ctx->cout))
                    rc = set_err(STABGPU_CUDA, "download failed: %s", cudaGetErrorString(cudaGetLastError()));
            } else if (cudaMemcpyAsync(hoy + f0 * fl, doy + f0 * fl, nf * fl, cudaMemcpyDeviceToHost, ctx->cout) ||
                       (chroma && (cudaMemcpyAsync(hocb + f0 * fc, docb + f0 * fc, nf * fc, cudaMemcpyDeviceToHost,
                                                   ctx->cout) ||
                                   cudaMemcpyAsync(hocr + f0 * fc, docr + f0 * fc, nf * fc, cudaMemcpyDeviceToHost,
                                                   ctx->cout)))) {
                rc = set_err(STABGPU_CUDA, "download failed: %s", cudaGetErrorString(cudaGetLastError()));
            }
            composed = ready;
        }
    }
    if (!rc && composed != n) rc = set_err(STABGPU_CUDA, "internal: %lld of %d frames composed", composed, n);
    cudaStreamSynchronize(ctx->cin);
    cudaStreamSynchronize(st);
    cudaStreamSynchronize(ctx->cout);
    for (auto& e : in_ev) cudaEventDestroy(e);
    for (auto& e : out_ev) cudaEventDestroy(e);
    if (rc) return rc;
    TRY(plan_error(ctx, ps));
    if (records)
        CUDA_TRY(cudaMemcpyAsync(records, rec, sizeof(stabgpu_frame_record) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return check_launch("stabilize_sequence");
}

}  // namespace

extern "C" {

int stabgpu_stabilize_sequence(stabgpu_ctx* ctx, const uint8_t* hy, const uint8_t* hcb,
                               const uint8_t* hcr, int n, int w, int h, int cw, int ch,
                               const stabgpu_config* cfgp, uint8_t* hoy, uint8_t* hocb,
                               uint8_t* hocr, stabgpu_frame_record* records) {
    return sequence_host(ctx, hy, hcb, hcr, nullptr, n, w, h, cw, ch, cfgp, hoy, hocb, hocr, nullptr, records);
}

// ---- multi-GPU split ------------------------------------------------------

int stabgpu_motion_chunk(stabgpu_ctx* ctx, const uint8_t* dev_y, int64_t first, int count, int w,
                         int h, const stabgpu_config* cfgp, stabgpu_motion_record* host_out) {
    const stabgpu_config cfg = *cfgp;
    TRY(validate_all(cfg));
    TRY(validate_frame(w, h));
    if (count < 0) return set_err(STABGPU_INVALID_INPUT, "negative frame count");
    if (first % cfg.flow.redetect_interval != 0)
        return set_err(STABGPU_SEQUENCING, "motion chunks must start on a re-detect frame");
    cudaSetDevice(ctx->device);
    DBUF(stabgpu_motion_record, motion, "chunk_motion", (size_t)count + 1);
    // records are written at motion[first + k]; shift the base so index
    // `first` lands on motion[0]
    stabgpu_motion_record* base = motion - first;
    if (first != 0) {
        stabgpu_motion_record none;
        std::memset(&none, 0, sizeof none);
        none.frame_kind = -1;
        CUDA_TRY(cudaMemcpyAsync(motion, &none, sizeof none, cudaMemcpyHostToDevice, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    }
    TRY(run_motion(ctx, dev_y, first, count, w, h, cfg, base));
    CUDA_TRY(cudaMemcpyAsync(host_out, motion, sizeof(stabgpu_motion_record) * ((size_t)count + 1),
                             cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return STABGPU_OK;
}

int stabgpu_plan_corrections(stabgpu_ctx* ctx, const stabgpu_motion_record* host_motion, int n,
                             const stabgpu_config* cfgp, stabgpu_frame_record* host_records) {
    const stabgpu_config cfg = *cfgp;
    TRY(validate_all(cfg));
    if (n < 1) return set_err(STABGPU_INVALID_INPUT, "no motion records");
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    DBUF(stabgpu_motion_record, motion, "seq_motion", n);
    DBUF(stabgpu_frame_record, rec, "seq_rec", n);
    DBUF(double4, cum, "seq_cum", n);
    DBUF(FramePlan, plan, "seq_plan", n);
    CUDA_TRY(cudaMemcpyAsync(motion, host_motion, sizeof(stabgpu_motion_record) * n,
                             cudaMemcpyHostToDevice, st));
    PlanState* ps;
    TRY(init_plan_state(ctx, cfg, &ps));
    {
        Timer tm(ctx, 5);
        launch_plan_scan(motion, 0, n, cfg, ps, rec, cum, st);
        launch_plan_smooth(cum, n, true, 0, n, cfg.smooth_radius, rec, plan, PlanGeom{16, 16, 0, 0, 0.0}, st);
    }
    ctx->stats.launches += 2;
    TRY(check_launch("plan"));
    TRY(plan_error(ctx, ps));
    CUDA_TRY(cudaMemcpyAsync(host_records, rec, sizeof(stabgpu_frame_record) * n,
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

int stabgpu_compose_frames(stabgpu_ctx* ctx, const uint8_t* y, const uint8_t* cb, const uint8_t* cr,
                           int count, int w, int h, int cw, int ch,
                           const stabgpu_transform* host_corr, double crop, uint8_t* oy,
                           uint8_t* ocb, uint8_t* ocr) {
    TRY(validate_frame(w, h));
    TRY(validate_crop(crop));
    if (count <= 0) return STABGPU_OK;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    DBUF(stabgpu_transform, corr, "cmp_corr", count);
    DBUF(FramePlan, plan, "cmp_plan", count);
    CUDA_TRY(cudaMemcpyAsync(corr, host_corr, sizeof(stabgpu_transform) * count,
                             cudaMemcpyHostToDevice, st));
    launch_plan_from_corrections(corr, count, plan, PlanGeom{w, h, (cb && cr) ? cw : 0, (cb && cr) ? ch : 0, crop}, st);
    ++ctx->stats.launches;
    {
        Timer tm(ctx, 4);
        TRY(compose_range(ctx, y, cb, cr, 0, count, w, h, cw, ch, plan, crop, oy, ocb, ocr));
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    return STABGPU_OK;
}

// ---- sharded Stage I ------------------------------------------
int stabgpu_nccl_unique_id(unsigned char* out) {
    const NcclApi& api = nccl_api();
    if (!api.ok) return set_err(STABGPU_CUDA, "libnccl.so.2 not found (needed for multi-GPU sharding)");
    ncclUniqueId id;
    const ncclResult_t r = api.get_unique_id(&id);
    if (r != ncclSuccess) return set_err(STABGPU_CUDA, "ncclGetUniqueId: %s", api.error_string(r));
    std::memcpy(out, id.internal, STABGPU_NCCL_ID_BYTES);
    return STABGPU_OK;
}

int stabgpu_comm_init(stabgpu_ctx* ctx, const unsigned char* id, int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_err(STABGPU_INVALID_INPUT, "bad rank %d of %d", rank, nranks);
    const NcclApi& api = nccl_api();
    if (!api.ok) return set_err(STABGPU_CUDA, "libnccl.so.2 not found (needed for multi-GPU sharding)");
    cudaSetDevice(ctx->device);
    if (ctx->comm) {
        api.comm_destroy(ctx->comm);
        ctx->comm = nullptr;
    }
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, STABGPU_NCCL_ID_BYTES);
    ncclComm_t c = nullptr;
    const ncclResult_t r = api.comm_init_rank(&c, nranks, uid, rank);
    if (r != ncclSuccess) return set_err(STABGPU_CUDA, "ncclCommInitRank: %s", api.error_string(r));
    ctx->comm = c;
    ctx->nranks = nranks;
    ctx->rank = rank;
    return STABGPU_OK;
}

}  // extern "C"
namespace {
// Shard geometry of every rank: the pipeline.shard_ranges partition.
struct ShardGeo {
    long long first;  // motion chunk frames first .. first+count (first: a re-detect frame)
    int count;        // 0: the rank idles (more ranks than segments)
    long long own_begin, own_end;
};

ShardGeo shard_geo(long long n, int R, int world, int g) {
    const long long nseg = (n - 1 + R - 1) / R;
    const long long s0 = nseg * g / world, s1 = nseg * (g + 1) / world;
    ShardGeo o;
    o.first = std::min(s0 * R, n - 1);
    const long long last = std::min(s1 * R, n - 1);
    o.own_begin = s0 == 0 ? 0 : o.first + 1;
    o.own_end = last + 1;
    o.count = (int)(last - o.first);
    if (s0 == s1) o.first = o.count = 0, o.own_begin = o.own_end = 0;
    return o;
}

// Uploads this rank's frames [first, first+count] into the context's resident
// shard buffers in chunks and estimates the motion of each segment as soon as
// its last frame has arrived (upload of chunk k+1 overlaps the motion of chunk
// k).  local_motion[0 .. count]: frame `first` (FIRST record on rank 0, else
// untouched), frames first+1 .. first+count.
int shard_motion(stabgpu_ctx* ctx, const uint8_t* hy, const uint8_t* hcb, const uint8_t* hcr, const ShardGeo& g,
                 int w, int h, int cw, int ch, const stabgpu_config& cfg, stabgpu_motion_record* local_motion) {
    cudaStream_t st = ctx->stream;
    const bool chroma = hcb && hcr;
    const size_t fl = (size_t)w * h, fc = chroma ? (size_t)cw * ch : 0;
    const long long nres = (long long)g.count + 1;
    DBUF(uint8_t, dy, "shard_y", fl * nres);
    if (chroma) {
        DBUF(uint8_t, a, "shard_cb", fc * nres);
        DBUF(uint8_t, b, "shard_cr", fc * nres);
        (void)a;
        (void)b;
    }
    uint8_t* dcb = chroma ? static_cast<uint8_t*>(ctx->bufs["shard_cb"].p) : nullptr;
    uint8_t* dcr = chroma ? static_cast<uint8_t*>(ctx->bufs["shard_cr"].p) : nullptr;
    stabgpu_motion_record* base = local_motion - g.first;  // motion[global frame]
    const int R = cfg.flow.redetect_interval;
    const std::vector<long long> cbd = chunk_bounds(nres, fl + 2 * fc);  // upload chunks
    const int nchunks = (int)cbd.size() - 1;
    std::vector<cudaEvent_t> in_ev(nchunks);
    for (auto& e : in_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    int rc = STABGPU_OK;
    for (int k = 0; k < nchunks && !rc; ++k) {
        const size_t f0 = (size_t)cbd[k], nf = (size_t)(cbd[k + 1] - cbd[k]);
        if (cudaMemcpyAsync(dy + f0 * fl, hy + f0 * fl, nf * fl, cudaMemcpyHostToDevice, ctx->cin) ||
            (chroma && (cudaMemcpyAsync(dcb + f0 * fc, hcb + f0 * fc, nf * fc, cudaMemcpyHostToDevice, ctx->cin) ||
                        cudaMemcpyAsync(dcr + f0 * fc, hcr + f0 * fc, nf * fc, cudaMemcpyHostToDevice, ctx->cin))))
            rc = set_err(STABGPU_CUDA, "upload failed: %s", cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(in_ev[k], ctx->cin);
    }
    // segments [first + s R, min(first + (s+1) R, first + count)] of the chunk
    const long long nseg = (g.count + R - 1) / R;
    long long seg_done = 0;
    for (int k = 0; k < nchunks && !rc; ++k) {
        cudaStreamWaitEvent(st, in_ev[k], 0);
        const long long arrived = cbd[k + 1];  // local frames [0, arrived)
        long long seg_end = seg_done;
        while (seg_end < nseg && std::min<long long>((seg_end + 1) * R, g.count) < arrived) ++seg_end;
        if (seg_end > seg_done) {
            const long long a = seg_done * R, b = std::min<long long>(seg_end * R, g.count);
            rc = run_motion(ctx, dy + a * fl, g.first + a, (int)(b - a), w, h, cfg, base);
            seg_done = seg_end;
        }
    }
    cudaStreamSynchronize(ctx->cin);
    for (auto& e : in_ev) cudaEventDestroy(e);
    return rc;
}

// Plans all n frames from the device motion records (the sequential scan,
// identical on every rank) and composes this rank's own frames.  vy/vcb/vcr
// and voy/vocb/vocr are frame-indexed device views (frame i at view + i *
// plane); with host outputs, each chunk of own frames is downloaded behind
// the compose of the next.
int shard_finish(stabgpu_ctx* ctx, const stabgpu_motion_record* motion_all, long long n, const ShardGeo& g, int w,
                 int h, int cw, int ch, bool chroma, const stabgpu_config& cfg, const uint8_t* vy,
                 const uint8_t* vcb, const uint8_t* vcr, uint8_t* voy, uint8_t* vocb, uint8_t* vocr, uint8_t* hoy,
                 uint8_t* hocb, uint8_t* hocr, stabgpu_frame_record* records) {
    cudaStream_t st = ctx->stream;
    const size_t fl = (size_t)w * h, fc = chroma ? (size_t)cw * ch : 0;
    DBUF(stabgpu_frame_record, rec, "seq_rec", n);
    DBUF(double4, cum, "seq_cum", n);
    DBUF(FramePlan, plan, "seq_plan", n);
    PlanState* ps;
    TRY(init_plan_state(ctx, cfg, &ps));
    {
        Timer tm(ctx, 5);
        launch_plan_scan(motion_all, 0, n, cfg, ps, rec, cum, st);
        // every frame's correction (the records cover all n frames; n threads)
        launch_plan_smooth(cum, n, true, 0, n, cfg.smooth_radius, rec, plan,
                           PlanGeom{w, h, chroma ? cw : 0, chroma ? ch : 0, cfg.crop_ratio}, st);
    }
    ctx->stats.launches += 2;
    TRY(check_launch("plan"));
    const long long own = g.own_end - g.own_begin;
    int rc = STABGPU_OK;
    if (own > 0) {
        const int C = hoy ? 60 : (int)own;  // host outputs: chunks downloaded behind the next compose
        const int nchunks = (int)((own + C - 1) / C);
        std::vector<cudaEvent_t> done(nchunks);
        for (auto& e : done) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (int k = 0; k < nchunks && !rc; ++k) {
            const long long f0 = g.own_begin + (long long)k * C, nf = std::min<long long>(C, g.own_end - f0);
            {
                Timer tm(ctx, 4);
                rc = compose_range(ctx, vy, vcb, vcr, f0, nf, w, h, cw, ch, plan, cfg.crop_ratio, voy, vocb, vocr);
            }
            if (rc) break;
            if (!hoy) continue;
            cudaEventRecord(done[k], st);
            cudaStreamWaitEvent(ctx->cout, done[k], 0);
            const size_t o = (size_t)(f0 - g.own_begin);
            if (cudaMemcpyAsync(hoy + o * fl, voy + f0 * fl, nf * fl, cudaMemcpyDeviceToHost, ctx->cout) ||
                (chroma && (cudaMemcpyAsync(hocb + o * fc, vocb + f0 * fc, nf * fc, cudaMemcpyDeviceToHost, ctx->cout) ||
                            cudaMemcpyAsync(hocr + o * fc, vocr + f0 * fc, nf * fc, cudaMemcpyDeviceToHost, ctx->cout))))
                rc = set_err(STABGPU_CUDA, "download failed: %s", cudaGetErrorString(cudaGetLastError()));
        }
        cudaStreamSynchronize(ctx->cout);
        for (auto& e : done) cudaEventDestroy(e);
    }
    if (rc) return rc;
    TRY(plan_error(ctx, ps));
    if (records)
        CUDA_TRY(cudaMemcpyAsync(records, rec, sizeof(stabgpu_frame_record) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return check_launch("stabilize_sharded");
}

// shard_finish on the context's resident shard buffers (host entry points)
int shard_finish_host(stabgpu_ctx* ctx, const stabgpu_motion_record* motion_all, long long n, const ShardGeo& g,
                      int w, int h, int cw, int ch, bool chroma, const stabgpu_config& cfg, uint8_t* hoy,
                      uint8_t* hocb, uint8_t* hocr, stabgpu_frame_record* records) {
    const size_t fl = (size_t)w * h, fc = chroma ? (size_t)cw * ch : 0;
    const long long own = std::max<long long>(g.own_end - g.own_begin, 1);
    uint8_t* dy = static_cast<uint8_t*>(ctx->bufs["shard_y"].p);
    uint8_t* dcb = chroma ? static_cast<uint8_t*>(ctx->bufs["shard_cb"].p) : nullptr;
    uint8_t* dcr = chroma ? static_cast<uint8_t*>(ctx->bufs["shard_cr"].p) : nullptr;
    DBUF(uint8_t, doy, "shard_oy", fl * own);
    uint8_t *docb = nullptr, *docr = nullptr;
    if (chroma) {
        DBUF(uint8_t, a, "shard_ocb", fc * own);
        DBUF(uint8_t, b, "shard_ocr", fc * own);
        docb = a;
        docr = b;
    }
    // frame-indexed views: frame i of the sequence at view + i * plane
    return shard_finish(ctx, motion_all, n, g, w, h, cw, ch, chroma, cfg, dy ? dy - g.first * fl : nullptr,
                        chroma ? dcb - g.first * fc : nullptr, chroma ? dcr - g.first * fc : nullptr,
                        doy - g.own_begin * fl, chroma ? docb - g.own_begin * fc : nullptr,
                        chroma ? docr - g.own_begin * fc : nullptr, hoy, hocb, hocr, records);
}

// The all-gather of every rank's count+1 records (send) and their scatter
// into the frame-indexed motion array ma (record 0 of rank 0 is frame 0).
int shard_exchange(stabgpu_ctx* ctx, long long n, int R, int world, const stabgpu_motion_record* send,
                   stabgpu_motion_record* recv, size_t blk, stabgpu_motion_record* ma) {
    cudaStream_t st = ctx->stream;
    const size_t bytes = blk * sizeof(stabgpu_motion_record);
    if (world > 1) {
        const ncclResult_t r = nccl_api().all_gather(send, recv, bytes, ncclUint8, ctx->comm, st);
        if (r != ncclSuccess) return set_err(STABGPU_CUDA, "ncclAllGather: %s", nccl_api().error_string(r));
    } else {
        CUDA_TRY(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
    }
    for (int k = 0; k < world; ++k) {
        const ShardGeo o = shard_geo(n, R, world, k);
        if (o.count == 0) continue;
        const stabgpu_motion_record* src = recv + (size_t)k * blk;
        if (o.first == 0) CUDA_TRY(cudaMemcpyAsync(ma, src, sizeof(stabgpu_motion_record), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(ma + o.first + 1, src + 1, sizeof(stabgpu_motion_record) * o.count,
                                 cudaMemcpyDeviceToDevice, st));
    }
    return STABGPU_OK;
}

int validate_shard(const stabgpu_config& cfg, long long n, int world, int rank, int w, int h) {
    TRY(validate_all(cfg));
    TRY(validate_frame(w, h));
    if (n < 2) return set_err(STABGPU_INVALID_INPUT, "stabilization needs at least 2 frames");
    if (world < 1 || rank < 0 || rank >= world) return set_err(STABGPU_INVALID_INPUT, "bad rank %d of %d", rank, world);
    return STABGPU_OK;
}
}  // namespace
extern "C" {

int stabgpu_shard_range(int64_t n, int redetect_interval, int world, int rank, int64_t* first, int* count,
                        int64_t* own_begin, int64_t* own_end) {
    if (n < 2 || redetect_interval < 1 || world < 1 || rank < 0 || rank >= world)
        return set_err(STABGPU_INVALID_INPUT, "bad shard request");
    const ShardGeo g = shard_geo(n, redetect_interval, world, rank);
    *first = g.first;
    *count = g.count;
    *own_begin = g.own_begin;
    *own_end = g.own_end;
    return STABGPU_OK;
}

int stabgpu_shard_motion(stabgpu_ctx* ctx, const uint8_t* hy, const uint8_t* hcb, const uint8_t* hcr, int64_t n,
                         int world, int rank, int w, int h, int cw, int ch, const stabgpu_config* cfgp,
                         stabgpu_motion_record* host_motion) {
    const stabgpu_config cfg = *cfgp;
    TRY(validate_shard(cfg, n, world, rank, w, h));
    cudaSetDevice(ctx->device);
    begin_timing(ctx);
    const ShardGeo g = shard_geo(n, cfg.flow.redetect_interval, world, rank);
    if (g.count == 0) return STABGPU_OK;
    DBUF(stabgpu_motion_record, lm, "shard_motion", (size_t)g.count + 1);
    TRY(shard_motion(ctx, hy, (hcb && hcr) ? hcb : nullptr, (hcb && hcr) ? hcr : nullptr, g, w, h, cw, ch, cfg, lm));
    CUDA_TRY(cudaMemcpyAsync(host_motion, lm, sizeof(stabgpu_motion_record) * ((size_t)g.count + 1),
                             cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return check_launch("shard_motion");
}

int stabgpu_shard_compose(stabgpu_ctx* ctx, const stabgpu_motion_record* host_all_motion, int64_t n, int world,
                          int rank, int w, int h, int cw, int ch, const stabgpu_config* cfgp, uint8_t* hoy,
                          uint8_t* hocb, uint8_t* hocr, stabgpu_frame_record* records) {
    const stabgpu_config cfg = *cfgp;
    TRY(validate_shard(cfg, n, world, rank, w, h));
    cudaSetDevice(ctx->device);
    const ShardGeo g = shard_geo(n, cfg.flow.redetect_interval, world, rank);
    const bool chroma = hocb && hocr && cw > 0 && ch > 0 && ctx->bufs.count("shard_cb");
    DBUF(stabgpu_motion_record, ma, "shard_motion_all", n);
    CUDA_TRY(cudaMemcpyAsync(ma, host_all_motion, sizeof(stabgpu_motion_record) * n, cudaMemcpyHostToDevice,
                             ctx->stream));
    return shard_finish_host(ctx, ma, n, g, w, h, cw, ch, chroma, cfg, hoy, hocb, hocr, records);
}

int stabgpu_stabilize_sharded(stabgpu_ctx* ctx, const uint8_t* hy, const uint8_t* hcb, const uint8_t* hcr, int64_t n,
                              int w, int h, int cw, int ch, const stabgpu_config* cfgp, uint8_t* hoy, uint8_t* hocb,
                              uint8_t* hocr, stabgpu_frame_record* records) {
    const stabgpu_config cfg = *cfgp;
    const int world = ctx->nranks, rank = ctx->rank;
    TRY(validate_shard(cfg, n, world, rank, w, h));
    if (world > 1 && !ctx->comm) return set_err(STABGPU_SEQUENCING, "stabilize_sharded needs stabgpu_comm_init first");
    cudaSetDevice(ctx->device);
    begin_timing(ctx);
    cudaStream_t st = ctx->stream;
    const int R = cfg.flow.redetect_interval;
    const bool chroma = hcb && hcr && hocb && hocr;
    const ShardGeo g = shard_geo(n, R, world, rank);
    int maxcount = 0;
    for (int k = 0; k < world; ++k) maxcount = std::max(maxcount, shard_geo(n, R, world, k).count);
    const size_t blk = (size_t)maxcount + 1;  // records per rank in the all-gather
    DBUF(stabgpu_motion_record, send, "shard_send", blk);
    DBUF(stabgpu_motion_record, recv, "shard_recv", blk * world);
    DBUF(stabgpu_motion_record, ma, "shard_motion_all", n);
    if (g.count > 0) TRY(shard_motion(ctx, hy, chroma ? hcb : nullptr, chroma ? hcr : nullptr, g, w, h, cw, ch, cfg, send));
    // ---- the one exchange: every rank's motion records, device to device
    TRY(shard_exchange(ctx, n, R, world, send, recv, blk, ma));
    return shard_finish_host(ctx, ma, n, g, w, h, cw, ch, chroma, cfg, hoy, hocb, hocr, records);
}

int stabgpu_stabilize_sharded_device(stabgpu_ctx* ctx, const uint8_t* dy, const uint8_t* dcb, const uint8_t* dcr,
                                     int64_t n, int w, int h, int cw, int ch, const stabgpu_config* cfgp,
                                     uint8_t* doy, uint8_t* docb, uint8_t* docr, stabgpu_frame_record* records) {
    const stabgpu_config cfg = *cfgp;
    const int world = ctx->nranks, rank = ctx->rank;
    TRY(validate_shard(cfg, n, world, rank, w, h));
    if (world > 1 && !ctx->comm) return set_err(STABGPU_SEQUENCING, "stabilize_sharded needs stabgpu_comm_init first");
    cudaSetDevice(ctx->device);
    begin_timing(ctx);
    const int R = cfg.flow.redetect_interval;
    const bool chroma = dcb && dcr && docb && docr;
    const ShardGeo g = shard_geo(n, R, world, rank);
    int maxcount = 0;
    for (int k = 0; k < world; ++k) maxcount = std::max(maxcount, shard_geo(n, R, world, k).count);
    const size_t blk = (size_t)maxcount + 1;
    DBUF(stabgpu_motion_record, send, "shard_send", blk);
    DBUF(stabgpu_motion_record, recv, "shard_recv", blk * world);
    DBUF(stabgpu_motion_record, ma, "shard_motion_all", n);
    if (g.count > 0) TRY(run_motion(ctx, dy, g.first, g.count, w, h, cfg, send - g.first));
    TRY(shard_exchange(ctx, n, R, world, send, recv, blk, ma));
    const size_t fl = (size_t)w * h, fc = chroma ? (size_t)cw * ch : 0;
    return shard_finish(ctx, ma, n, g, w, h, cw, ch, chroma, cfg, dy - g.first * fl,
                        chroma ? dcb - g.first * fc : nullptr, chroma ? dcr - g.first * fc : nullptr,
                        doy - g.own_begin * fl, chroma ? docb - g.own_begin * fc : nullptr,
                        chroma ? docr - g.own_begin * fc : nullptr, nullptr, nullptr, nullptr, records);
}

// ---- Stage II streaming ---------------------------------------------------
}  // extern "C"

// The streaming object owns its device memory (independent of the context's
// Stage I buffers).  Frame-indexed records grow geometrically; frames live in
// a ring of 2r + R + 2 slots (a frame is needed until its correction is
// released, at most 2r frames after it arrived).
struct stabgpu_stream {
    stabgpu_ctx* ctx = nullptr;
    stabgpu_config cfg{};
    int w = 0, h = 0, cw = 0, ch = 0;
    bool chroma = false, complete = false;
    int cap = 0, ocap = 0;       // input / output ring slots
    long long pushed = 0, next = 0;  // frames pushed, next frame to release
    std::vector<void*> allocs;
    // frames
    // input and output rings, frame-major: slot k holds Y | Cb | Cr at
    // ring_y/cb/cr + k * fs (plane offsets padded to 256 B), so a caller whose
    // frame is one contiguous planar buffer moves in one copy per direction
    uint8_t *ring_y = nullptr, *ring_cb = nullptr, *ring_cr = nullptr;
    uint8_t *out_y = nullptr, *out_cb = nullptr, *out_cr = nullptr;
    size_t fs = 0;         // bytes between two ring slots
    bool packed = false;   // no padding between the planes: Y, Cb, Cr of a slot are one contiguous run
    std::vector<long long> ready;    // released frame indices not yet popped (FIFO)
    size_t ready_head = 0;
    // motion state: two-frame pyramid (prev at 0, cur at 1)
    DevPyramid P{};
    stabgpu_roi roi{};
    DetectScratch ds{};
    double2 *pts = nullptr, *nxt = nullptr, *fwd = nullptr, *trk_prev = nullptr, *trk_cur = nullptr;
    int *npts = nullptr, *nnxt = nullptr, *trk_n = nullptr;
    // third point buffer: a re-detection (detect stream) writes it while the
    // frame's K5 step reads pts and its compaction writes nxt (motion stream)
    double2* det = nullptr;
    int* ndet = nullptr;
    int2* fit_pre = nullptr;  // per-CTA RANSAC results of the one-frame fit
    double* score = nullptr;
    uint8_t* keep = nullptr;
    unsigned* work = nullptr;
    // frame-indexed (grown on demand)
    long long fcap = 0;
    stabgpu_motion_record* motion = nullptr;
    stabgpu_frame_record* rec = nullptr;
    double4* cum = nullptr;
    FramePlan* plan = nullptr;
    PlanState* ps = nullptr;
    // copy/compute overlap: input slot k is free once the compose of its
    // frame ran (slot_free[k]); output slot k is downloadable once its frame
    // is composed (out_done[k]); pinned error word of the selector scan
    std::vector<cudaEvent_t> slot_free, out_done, in_done;
    int* err_host = nullptr;
    // three compute streams: the motion chain (context stream: K1, K5 step,
    // compaction, K6 fit, K7 scan), the release stream (smoothing + K8 compose
    // of the released frame, behind that frame's scan) and the detect stream
    // (the re-detection of frame kR beside its own K5 step; frame kR+1's K5
    // waits for it).  motion_done[k]: the motion chain that read input slot k
    // as its previous frame has run (the slot may be overwritten).
    cudaStream_t rst = nullptr, dst = nullptr, pst = nullptr;  // release chain, re-detection, pyramid
    cudaEvent_t ev_scan = nullptr, ev_rel = nullptr, ev_det = nullptr, ev_motion = nullptr, ev_grow = nullptr;
    cudaEvent_t last_in = nullptr;  // upload event of the last pushed frame (push_async / wait_inputs)
    cudaEvent_t ev_pyr = nullptr, ev_chain[2] = {nullptr, nullptr};  // K1 of the frame; end of the chain of frame f (slot f & 1)
    std::vector<cudaEvent_t> motion_done;
    bool det_wait = false, rel_any = false, grown = false, pops_pending = false;
    // pop_async: records land in a pinned ring (a download into pageable memory
    // would block the call) and reach the caller's pointers in wait_pops
    stabgpu_frame_record* rec_host = nullptr;
    std::vector<std::pair<stabgpu_frame_record*, int>> rec_owed;
    // per-frame CUDA graphs: each push's launch sequence (K1 levels, K5 step +
    // compaction + K6 fit or the detection, the K7 scan, and the smoothing +
    // K8 compose of the frame it releases) is stream-captured and launched as
    // one graph; the executable graph of each topology (first frame /
    // re-detect / tracking, 0 or 1 release) is instantiated once and updated
    // in place with the frame's parameters afterwards
    bool graphs = false;
    std::map<int, cudaGraphExec_t> execs;
    void* cscratch = nullptr;  // K8 tables of one frame (no allocation inside a graph)
    size_t cscratch_bytes = 0;
};

namespace {

template <typename T>
int salloc(stabgpu_stream* s, T** p, size_t count) {
    void* q = nullptr;
    if (cudaMalloc(&q, count * sizeof(T) + 256) != cudaSuccess) {
        cudaGetLastError();
        return set_err(STABGPU_CUDA, "stream: device allocation of %zu bytes failed", count * sizeof(T));
    }
    s->allocs.push_back(q);
    *p = static_cast<T*>(q);
    return STABGPU_OK;
}

// grows the frame-indexed arrays to hold frame index `need - 1`
int stream_grow(stabgpu_stream* s, long long need) {
    if (need <= s->fcap) return STABGPU_OK;
    long long nc = std::max<long long>(256, s->fcap);
    while (nc < need) nc *= 2;
    cudaStream_t st = s->ctx->stream;
    stabgpu_motion_record* m;
    stabgpu_frame_record* r;
    double4* c;
    FramePlan* pl;
    TRY(salloc(s, &m, nc));
    TRY(salloc(s, &r, nc));
    TRY(salloc(s, &c, nc));
    TRY(salloc(s, &pl, nc));
    if (s->fcap) {
        // the release stream's smoothing wrote records and plans into the old blocks
        if (s->rel_any) CUDA_TRY(cudaStreamWaitEvent(st, s->ev_rel, 0));
        CUDA_TRY(cudaMemcpyAsync(m, s->motion, sizeof(*m) * s->fcap, cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(r, s->rec, sizeof(*r) * s->fcap, cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(c, s->cum, sizeof(*c) * s->fcap, cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(pl, s->plan, sizeof(*pl) * s->fcap, cudaMemcpyDeviceToDevice, st));
        // pops of frames released earlier read their records from the new block
        CUDA_TRY(cudaEventRecord(s->ev_grow, st));
        s->grown = true;
    }
    s->motion = m;
    s->rec = r;
    s->cum = c;
    s->plan = pl;
    s->fcap = nc;  // the old blocks stay allocated until destroy (stream-ordered reuse is not needed)
    return STABGPU_OK;
}

bool graph_safe(const stabgpu_config& c) {
    return !detect_allocates(c.detect) && !fit_allocates(c.detect.max_corners);
}

// smoothing + K8 compose of released frame i into output slot i % ocap (release stream)
void stream_release_kernels(stabgpu_stream* s, long long i) {
    cudaStream_t st = s->rst;
    const int r = s->cfg.smooth_radius;
    launch_plan_smooth(s->cum, s->pushed, s->complete, i, 1, r, s->rec, s->plan,
                       PlanGeom{s->w, s->h, s->chroma ? s->cw : 0, s->chroma ? s->ch : 0, s->cfg.crop_ratio}, st);
    const size_t fl = (size_t)s->w * s->h, fc = (size_t)s->cw * s->ch;
    const size_t in = (size_t)(i % s->cap), o = (size_t)(i % s->ocap);
    PlaneBatch yb{s->ring_y + in * s->fs, fl, s->w, s->h};
    PlaneBatch bb{s->chroma ? s->ring_cb + in * s->fs : nullptr, fc, s->cw, s->ch};
    PlaneBatch rb{s->chroma ? s->ring_cr + in * s->fs : nullptr, fc, s->cw, s->ch};
    launch_compose(yb, bb, rb, s->plan + i, 1, s->cfg.crop_ratio, s->out_y + o * s->fs,
                   s->chroma ? s->out_cb + o * s->fs : nullptr, s->chroma ? s->out_cr + o * s->fs : nullptr, st,
                   s->cscratch, s->cscratch_bytes);
    s->ctx->stats.launches += 2;
}

// after frame i's release kernels were issued: its input slot is free and
// its output slot downloadable (events), and it is queued for pop
void stream_release_done(stabgpu_stream* s, long long i) {
    cudaStream_t st = s->rst;
    cudaEventRecord(s->slot_free[(size_t)(i % s->cap)], st);
    cudaEventRecord(s->out_done[(size_t)(i % s->ocap)], st);
    cudaEventRecord(s->ev_rel, st);
    s->rel_any = true;
    s->ready.push_back(i);
}

// CompensationPlanner::release (pipeline.cpp:137-150): the frames
// [s->next, s->next + count) are released now
int stream_release_count(const stabgpu_stream* s, long long* count) {
    *count = 0;
    const int r = s->cfg.smooth_radius;
    if (!s->complete && s->pushed < 2LL * r) return STABGPU_OK;
    long long n = s->next;
    while (n < s->pushed && (s->complete || n + r < s->pushed)) {
        if ((long long)(s->ready.size() - s->ready_head) + (n - s->next) >= s->ocap)
            return set_err(STABGPU_SEQUENCING, "stream: %d released frames not popped", s->ocap);
        ++n;
    }
    *count = n - s->next;
    return STABGPU_OK;
}

// launches a captured graph through the executable graph of its topology
int stream_launch_graph(stabgpu_stream* s, int key, cudaGraph_t g, cudaStream_t st) {
    auto it = s->execs.find(key);
    if (it != s->execs.end()) {
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(it->second, g, &info) != cudaSuccess) {
            cudaGetLastError();
            cudaGraphExecDestroy(it->second);
            s->execs.erase(it);
            it = s->execs.end();
        }
    }
    if (it == s->execs.end()) {
        cudaGraphExec_t ex = nullptr;
        CUDA_TRY(cudaGraphInstantiate(&ex, g, 0));
        it = s->execs.emplace(key, ex).first;
    }
    CUDA_TRY(cudaGraphLaunch(it->second, st));
    return STABGPU_OK;
}

// Runs `body` (kernel launches on st) as one CUDA graph keyed by its topology,
// or directly when graphs are off.
template <typename F>
int stream_run(stabgpu_stream* s, bool graph, int key, cudaStream_t st, const char* what, F body) {
    if (graph) CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    body();
    int rc = check_launch(what);
    if (graph) {
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(st, &g);
        if (rc == STABGPU_OK && e != cudaSuccess)
            rc = set_err(STABGPU_CUDA, "stream: graph capture failed: %s", cudaGetErrorString(e));
        if (rc == STABGPU_OK) rc = stream_launch_graph(s, key, g, st);
        if (g) cudaGraphDestroy(g);
        s->ctx->stats.launches += 1;
    }
    return rc;
}

// releases frames [s->next, s->next + n) on the release stream, behind the
// scan of the newest frame (ev_scan)
int stream_release(stabgpu_stream* s, long long n) {
    if (n <= 0) return STABGPU_OK;
    CUDA_TRY(cudaStreamWaitEvent(s->rst, s->ev_scan, 0));
    TRY(stream_run(s, s->graphs && n == 1, 0x300, s->rst, "stream compose", [&] {
        for (long long k = 0; k < n; ++k) stream_release_kernels(s, s->next + k);
    }));
    for (long long k = 0; k < n; ++k) stream_release_done(s, s->next + k);
    s->next += n;
    return STABGPU_OK;
}

}  // namespace

extern "C" {

int stabgpu_stream_create(stabgpu_ctx* ctx, const stabgpu_config* cfgp, int w, int h, int cw, int ch,
                          stabgpu_stream** out) {
    *out = nullptr;
    if (!ctx) return set_err(STABGPU_INVALID_INPUT, "stream: null context");
    const stabgpu_config cfg = *cfgp;
    TRY(validate_all(cfg));
    TRY(validate_frame(w, h));
    cudaSetDevice(ctx->device);
    auto* s = new stabgpu_stream();
    s->ctx = ctx;
    s->cfg = cfg;
    s->w = w;
    s->h = h;
    s->chroma = cw > 0 && ch > 0;
    s->cw = s->chroma ? cw : 0;
    s->ch = s->chroma ? ch : 0;
    const int r = cfg.smooth_radius, R = cfg.flow.redetect_interval, maxc = cfg.detect.max_corners;
    s->cap = 2 * r + R + 2;
    s->ocap = 2 * r + 2;
    int rc = STABGPU_OK;
    auto fail = [&](int code) {
        stabgpu_stream_destroy(s);
        return code;
    };
    const size_t fl = (size_t)w * h, fc = (size_t)s->cw * s->ch;
    {
        const size_t afl = (fl + 255) & ~(size_t)255, afc = s->chroma ? (fc + 255) & ~(size_t)255 : 0;
        s->fs = afl + 2 * afc;
        s->packed = afl == fl && afc == fc;
        if ((rc = salloc(s, &s->ring_y, s->fs * s->cap)) || (rc = salloc(s, &s->out_y, s->fs * s->ocap)))
            return fail(rc);
        if (s->chroma) {
            s->ring_cb = s->ring_y + afl;
            s->ring_cr = s->ring_cb + afc;
            s->out_cb = s->out_y + afl;
            s->out_cr = s->out_cb + afc;
        }
    }
    // three-frame pyramid for levels >= 1 (frame f in slot f % 3: frame f + 1's
    // levels are built on the pyramid stream while the motion chain still
    // tracks f - 1 -> f); level 0 is the input ring itself
    s->P.levels = level_dims(w, h, cfg.flow.max_levels, s->P.w, s->P.h);
    s->P.stride[0] = (size_t)w * h;
    for (int l = 1; l < s->P.levels; ++l) {
        uint8_t* lv;
        s->P.stride[l] = (size_t)s->P.w[l] * s->P.h[l];
        if ((rc = salloc(s, &lv, 3 * s->P.stride[l]))) return fail(rc);
        s->P.lvl[l] = lv;
    }
    // detection scratch (one frame)
    if ((rc = roi_of(w, h, cfg.detect.roi_margin, &s->roi))) return fail(rc);
    const size_t cap = (size_t)(s->roi.x1 - s->roi.x0) * (s->roi.y1 - s->roi.y0);
    DetectScratch& d = s->ds;
    d.cap = cap;
    if ((rc = salloc(s, &d.maxbits, 1)) || (rc = salloc(s, &d.count, 1)) || (rc = salloc(s, &d.hist, kRespBins)) ||
        (rc = salloc(s, &d.cand_key, cap)) || (rc = salloc(s, &d.cand_idx, cap)) ||
        (rc = salloc(s, &d.sort_key, cap)) || (rc = salloc(s, &d.sort_idx, cap)) || (rc = salloc(s, &d.lo, 1)) ||
        (rc = salloc(s, &d.flags, 1)) || (rc = salloc(s, &d.mlo, 1)) || (rc = salloc(s, &d.bstart, kBuckets + 1)) ||
        (rc = salloc(s, &d.bcur, kBuckets)))
        return fail(rc);
    if ((rc = salloc(s, &s->pts, maxc)) || (rc = salloc(s, &s->nxt, maxc)) || (rc = salloc(s, &s->fwd, maxc)) ||
        (rc = salloc(s, &s->trk_prev, maxc)) || (rc = salloc(s, &s->trk_cur, maxc)) ||
        (rc = salloc(s, &s->npts, 1)) || (rc = salloc(s, &s->nnxt, 1)) || (rc = salloc(s, &s->trk_n, 1)) ||
        (rc = salloc(s, &s->score, maxc)) || (rc = salloc(s, &s->keep, maxc)) || (rc = salloc(s, &s->work, 1)) ||
        (rc = salloc(s, &s->fit_pre, 2 * kFitPreCtas)) || (rc = salloc(s, &s->det, maxc)) ||
        (rc = salloc(s, &s->ndet, 1)))
        return fail(rc);
    if ((rc = stream_grow(s, 256))) return fail(rc);
    s->cscratch_bytes = compose_scratch_bytes(w, h, s->cw, s->ch, 1);
    if ((rc = salloc(s, reinterpret_cast<uint8_t**>(&s->cscratch), s->cscratch_bytes))) return fail(rc);
    // graphs need launch sequences without stream-ordered allocations: K4's
    // accepted list fits shared memory and K6's pairs fit its shared budget
    s->graphs = graph_safe(cfg);
    s->slot_free.resize(s->cap);
    s->in_done.resize(s->cap);
    s->motion_done.resize(s->cap);
    s->out_done.resize(s->ocap);
    for (auto* v : {&s->slot_free, &s->in_done, &s->out_done, &s->motion_done})
        for (auto& e : *v)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
                return fail(set_err(STABGPU_CUDA, "stream: event creation failed"));
    for (cudaEvent_t* e : {&s->ev_scan, &s->ev_rel, &s->ev_det, &s->ev_motion, &s->ev_grow, &s->ev_pyr, &s->ev_chain[0],
                           &s->ev_chain[1]})
        if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess)
            return fail(set_err(STABGPU_CUDA, "stream: event creation failed"));
    if (cudaStreamCreateWithFlags(&s->rst, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s->dst, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s->pst, cudaStreamNonBlocking) != cudaSuccess)
        return fail(set_err(STABGPU_CUDA, "stream: stream creation failed"));
    if (cudaMallocHost((void**)&s->err_host, sizeof(int)) != cudaSuccess ||
        cudaMallocHost((void**)&s->rec_host, sizeof(stabgpu_frame_record) * s->ocap) != cudaSuccess)
        return fail(set_err(STABGPU_CUDA, "stream: pinned allocation failed"));
    *s->err_host = 0;
    if ((rc = init_plan_state(ctx, cfg, &s->ps))) return fail(rc);
    // init_plan_state keeps its state in a context buffer: give the stream its own copy
    PlanState* own;
    if ((rc = salloc(s, &own, 2))) return fail(rc);
    if (cudaMemcpyAsync(own, s->ps, 2 * sizeof(PlanState), cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
        return fail(set_err(STABGPU_CUDA, "stream: state copy failed"));
    s->ps = own;
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return fail(set_err(STABGPU_CUDA, "stream: %s", cudaGetErrorString(cudaGetLastError())));
    *out = s;
    return STABGPU_OK;
}

}  // extern "C"
namespace {
int stream_push_impl(stabgpu_stream* s, const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int* n_ready,
                     bool wait_upload) {
    if (!s) return set_err(STABGPU_INVALID_INPUT, "stream: null handle");
    if (s->complete) return set_err(STABGPU_SEQUENCING, "stream: push after finish");
    if (!y || (s->chroma && (!cb || !cr))) return set_err(STABGPU_INVALID_INPUT, "stream: missing planes");
    stabgpu_ctx* ctx = s->ctx;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const stabgpu_config& cfg = s->cfg;
    const long long f = s->pushed;
    const int R = cfg.flow.redetect_interval, maxc = cfg.detect.max_corners;
    if (s->next + s->cap <= f)  // cannot happen with the release rule; guards the ring
        return set_err(STABGPU_SEQUENCING, "stream: input ring overrun");
    TRY(stream_grow(s, f + 1));
    const size_t fl = (size_t)s->w * s->h, fc = (size_t)s->cw * s->ch;
    const size_t slot = (size_t)(f % s->cap);
    uint8_t* fy = s->ring_y + slot * s->fs;
    // upload on the input copy stream once the slot's previous frame was
    // composed (and the motion chain that read it as its previous frame has
    // run); the motion stream waits for it.  The host buffers are read before
    // push returns (the upload is waited for at the end), while the previous
    // frames' compute and downloads keep running.
    if (f >= s->cap) {
        CUDA_TRY(cudaStreamWaitEvent(ctx->cin, s->slot_free[slot], 0));
        CUDA_TRY(cudaStreamWaitEvent(ctx->cin, s->motion_done[slot], 0));
    }
    if (s->chroma && s->packed && cb == y + fl && cr == cb + fc) {
        // the caller's frame is one planar buffer (Y | Cb | Cr): one copy
        // (frame-sized copies keep PCIe at its duplex rate; 2 MB ones do not)
        CUDA_TRY(cudaMemcpyAsync(fy, y, s->fs, cudaMemcpyDefault, ctx->cin));
    } else {
        CUDA_TRY(cudaMemcpyAsync(fy, y, fl, cudaMemcpyDefault, ctx->cin));
        if (s->chroma) {
            CUDA_TRY(cudaMemcpyAsync(s->ring_cb + slot * s->fs, cb, fc, cudaMemcpyDefault, ctx->cin));
            CUDA_TRY(cudaMemcpyAsync(s->ring_cr + slot * s->fs, cr, fc, cudaMemcpyDefault, ctx->cin));
        }
    }
    CUDA_TRY(cudaEventRecord(s->in_done[slot], ctx->cin));
    CUDA_TRY(cudaStreamWaitEvent(st, s->in_done[slot], 0));
    // the frames this push releases (CompensationPlanner::release)
    s->pushed = f + 1;
    long long nrel = 0;
    if (int rc = stream_release_count(s, &nrel)) {
        s->pushed = f;
        return rc;
    }
    const bool detect = f == 0 || f % R == 0;
    PlaneBatch cur{fy, fl, s->w, s->h};
    // detection of this frame (flow.cpp:303-308, 327-330) on the detect stream
    // as soon as the frame has landed: it reads the frame only, so with the
    // caller a few frames ahead it runs beside the K5 steps of the frames
    // before it instead of in front of the next one.  It writes the third
    // point buffer, last touched by the motion chain of the previous detection
    // frame (ev_motion: R frames ago).
    if (detect) {
        CUDA_TRY(cudaStreamWaitEvent(s->dst, s->in_done[slot], 0));
        if (f > 0) CUDA_TRY(cudaStreamWaitEvent(s->dst, s->ev_motion, 0));
        TRY(stream_run(s, s->graphs, 0x200, s->dst, "stream detect", [&] {
            launch_detect(cur, 1, cfg.detect, s->roi, s->ds, s->det, s->score, s->ndet, s->dst);
        }));
        CUDA_TRY(cudaEventRecord(s->ev_det, s->dst));
        ctx->stats.launches += 3;
    }
    // the previous frame's re-detection feeds this frame's K5 step
    if (s->det_wait) {
        CUDA_TRY(cudaStreamWaitEvent(st, s->ev_det, 0));
        s->det_wait = false;
    }
    // K1: the pyramid of the current frame, levels >= 1 into slot f % 3, on the
    // pyramid stream as soon as the frame has landed (off the motion chain: it
    // overlaps the previous frame's K5 step; the slot was last read by the
    // chain of frame f - 2).  No copies: level 0 stays in the ring, and the
    // tracker sees (previous, current) through a pyramid view whose frame
    // stride is the signed distance between the two slots
    DevPyramid& P = s->P;
    const int cs = (int)(f % 3), ps = (int)((f + 2) % 3);
    CUDA_TRY(cudaStreamWaitEvent(s->pst, s->in_done[slot], 0));
    if (f >= 2) CUDA_TRY(cudaStreamWaitEvent(s->pst, s->ev_chain[f & 1], 0));
    TRY(stream_run(s, false, 0x400, s->pst, "stream pyramid", [&] {  // three launches: cheaper direct than captured
        for (int l = 1; l < P.levels; ++l)
            launch_pyramid_level(l == 1 ? fy : P.lvl[l - 1] + cs * P.stride[l - 1], P.stride[l - 1], P.w[l - 1],
                                 P.h[l - 1], const_cast<uint8_t*>(P.lvl[l]) + cs * P.stride[l], P.stride[l], 1, s->pst);
    }));
    ctx->stats.launches += P.levels - 1;
    CUDA_TRY(cudaEventRecord(s->ev_pyr, s->pst));
    CUDA_TRY(cudaStreamWaitEvent(st, s->ev_pyr, 0));
    DevPyramid V = P;  // frame 0 = previous, frame 1 = current
    if (f > 0) {
        const uint8_t* py = s->ring_y + (size_t)((f - 1) % s->cap) * s->fs;
        V.lvl[0] = py;
        V.stride[0] = (size_t)(fy - py);  // two's complement: a wrapped ring gives a negative distance
        for (int l = 1; l < P.levels; ++l) {
            V.lvl[l] = P.lvl[l] + ps * P.stride[l];
            V.stride[l] = (size_t)((ptrdiff_t)(cs - ps) * (ptrdiff_t)P.stride[l]);
        }
    }
    TRY(stream_run(s, s->graphs, 0x100 | (f == 0 ? 1 : 0), st, "stream push", [&] {
        if (f == 0) {  // MotionStage first frame (pipeline.cpp:84-88)
            static_assert(STABGPU_FRAME_FIRST == 0, "the FIRST record is all zero bytes");
            cudaMemsetAsync(s->motion, 0, sizeof(stabgpu_motion_record), st);
        } else {  // Tracker::advance (flow.cpp:316-330): forward + weed, then fit
            LkStep k;
            std::memset(&k, 0, sizeof k);
            k.pyr = V;
            k.frame0 = 0;
            k.seg_len = R;
            k.t = 1;
            k.nseg = 1;
            k.max_pts = maxc;
            k.pts = s->pts;
            k.npts = s->npts;
            k.fwd = s->fwd;
            k.keep = s->keep;
            k.nframes = 2;
            k.mode = 1;
            k.work = s->work;
            launch_lk(k, cfg.flow, st);
            launch_compact(k, s->nxt, s->nnxt, s->trk_prev, s->trk_cur, s->trk_n, 1, st);
            launch_fit(s->trk_prev, s->trk_cur, s->trk_n, maxc, 1, f, cfg, s->motion + f, st, 0, s->fit_pre);
            ctx->stats.launches += 3;
        }
        // K7: selector + trajectory prefix for this frame
        launch_plan_scan(s->motion, f, 1, cfg, s->ps, s->rec, s->cum, st);
    }));
    CUDA_TRY(cudaEventRecord(s->ev_scan, st));
    if (detect) CUDA_TRY(cudaEventRecord(s->ev_motion, st));  // this chain's output buffer is the next detection's
    CUDA_TRY(cudaEventRecord(s->ev_chain[f & 1], st));
    if (f > 0) {  // this chain read the previous frame's slot
        CUDA_TRY(cudaEventRecord(s->motion_done[(size_t)((f - 1) % s->cap)], st));
        std::swap(s->pts, s->nxt);
        std::swap(s->npts, s->nnxt);
    }
    if (detect) {  // the fresh corners replace the carried points (flow.cpp:327-330)
        std::swap(s->pts, s->det);
        std::swap(s->npts, s->ndet);
        s->det_wait = true;
    }
    TRY(stream_release(s, nrel));
    s->last_in = s->in_done[slot];
    if (wait_upload) CUDA_TRY(cudaEventSynchronize(s->in_done[slot]));  // the caller's buffers are consumed
    if (n_ready) *n_ready = (int)(s->ready.size() - s->ready_head);
    return STABGPU_OK;
}
}  // namespace
extern "C" {

int stabgpu_stream_push(stabgpu_stream* s, const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int* n_ready) {
    return stream_push_impl(s, y, cb, cr, n_ready, true);
}

int stabgpu_stream_push_async(stabgpu_stream* s, const uint8_t* y, const uint8_t* cb, const uint8_t* cr,
                              int* n_ready) {
    return stream_push_impl(s, y, cb, cr, n_ready, false);
}

int stabgpu_stream_wait_inputs(stabgpu_stream* s) {
    if (!s) return set_err(STABGPU_INVALID_INPUT, "stream: null handle");
    if (s->last_in) {
        cudaSetDevice(s->ctx->device);
        CUDA_TRY(cudaEventSynchronize(s->last_in));  // uploads are in order on the input copy stream
    }
    return STABGPU_OK;
}

int stabgpu_stream_finish(stabgpu_stream* s, int* n_ready) {
    if (!s) return set_err(STABGPU_INVALID_INPUT, "stream: null handle");
    if (s->pushed < 2) return set_err(STABGPU_INVALID_INPUT, "stabilization needs at least 2 frames");
    cudaSetDevice(s->ctx->device);
    s->complete = true;
    long long n;
    TRY(stream_release_count(s, &n));
    TRY(stream_release(s, n));
    if (n_ready) *n_ready = (int)(s->ready.size() - s->ready_head);
    return STABGPU_OK;
}

int stabgpu_stream_pop_async(stabgpu_stream* s, int64_t* index, uint8_t* oy, uint8_t* ocb, uint8_t* ocr,
                             stabgpu_frame_record* record) {
    if (!s) return set_err(STABGPU_INVALID_INPUT, "stream: null handle");
    if (s->ready_head >= s->ready.size()) return set_err(STABGPU_SEQUENCING, "stream: no frame ready");
    cudaSetDevice(s->ctx->device);
    const long long i = s->ready[s->ready_head++];
    if (s->ready_head == s->ready.size()) {
        s->ready.clear();
        s->ready_head = 0;
    }
    // the download waits for this frame's compose only (frames pushed since
    // keep computing on the other streams)
    const size_t fl = (size_t)s->w * s->h, fc = (size_t)s->cw * s->ch, o = (size_t)(i % s->ocap);
    cudaStream_t co = s->ctx->cout;
    CUDA_TRY(cudaStreamWaitEvent(co, s->out_done[o], 0));
    if (s->grown) CUDA_TRY(cudaStreamWaitEvent(co, s->ev_grow, 0));  // the records may have moved
    if (s->chroma && s->packed && oy && ocb == oy + fl && ocr == ocb + fc) {
        CUDA_TRY(cudaMemcpyAsync(oy, s->out_y + o * s->fs, s->fs, cudaMemcpyDefault, co));  // one planar frame buffer
    } else {
        if (oy) CUDA_TRY(cudaMemcpyAsync(oy, s->out_y + o * s->fs, fl, cudaMemcpyDefault, co));
        if (s->chroma && ocb) CUDA_TRY(cudaMemcpyAsync(ocb, s->out_cb + o * s->fs, fc, cudaMemcpyDefault, co));
        if (s->chroma && ocr) CUDA_TRY(cudaMemcpyAsync(ocr, s->out_cr + o * s->fs, fc, cudaMemcpyDefault, co));
    }
    if (record) {
        // the records of the frames popped since the last wait are one
        // contiguous run of s->rec (frames pop in order): wait_pops fetches
        // them in one copy (a 96-byte copy per pop between the plane copies
        // stalls the copy queue)
        if (!s->rec_owed.empty() && i - s->rec_owed.front().second + 1 > s->ocap)  // the run must fit rec_host
            TRY(stabgpu_stream_wait_pops(s));
        s->rec_owed.emplace_back(record, (int)i);
    }
    s->pops_pending = true;  // wait_pops reads the selector scan's error word behind these copies
    if (index) *index = i;
    return STABGPU_OK;
}

int stabgpu_stream_wait_pops(stabgpu_stream* s) {
    if (!s) return set_err(STABGPU_INVALID_INPUT, "stream: null handle");
    if (!s->pops_pending) return STABGPU_OK;
    cudaSetDevice(s->ctx->device);
    s->pops_pending = false;
    // the selector scan's error word, once per wait (written before the popped
    // frames were released: the output copy stream has waited for their compose)
    CUDA_TRY(cudaMemcpyAsync(s->err_host, reinterpret_cast<int*>(s->ps + 1), sizeof(int), cudaMemcpyDeviceToHost,
                             s->ctx->cout));
    const long long i0 = s->rec_owed.empty() ? 0 : s->rec_owed.front().second;
    if (!s->rec_owed.empty()) {
        if (s->grown) CUDA_TRY(cudaStreamWaitEvent(s->ctx->cout, s->ev_grow, 0));  // the records may have moved
        const long long i1 = s->rec_owed.back().second;  // popped in order: [i0, i1] covers every owed record
        CUDA_TRY(cudaMemcpyAsync(s->rec_host, s->rec + i0, sizeof(stabgpu_frame_record) * (size_t)(i1 - i0 + 1),
                                 cudaMemcpyDeviceToHost, s->ctx->cout));
    }
    CUDA_TRY(cudaStreamSynchronize(s->ctx->cout));
    for (const auto& o : s->rec_owed) *o.first = s->rec_host[o.second - i0];
    s->rec_owed.clear();
    if (*s->err_host) TRY(plan_error(s->ctx, s->ps));
    return STABGPU_OK;
}

int stabgpu_stream_pop(stabgpu_stream* s, int64_t* index, uint8_t* oy, uint8_t* ocb, uint8_t* ocr,
                       stabgpu_frame_record* record) {
    TRY(stabgpu_stream_pop_async(s, index, oy, ocb, ocr, record));
    return stabgpu_stream_wait_pops(s);
}

int stabgpu_host_alloc(void** out, size_t bytes) {
    if (!out) return set_err(STABGPU_INVALID_INPUT, "host_alloc: null output pointer");
    *out = nullptr;
    if (cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return set_err(STABGPU_CUDA, "host_alloc: %zu page-locked bytes not available", bytes);
    }
    return STABGPU_OK;
}

int stabgpu_host_free(void* p) {
    if (p && cudaFreeHost(p) != cudaSuccess) {
        cudaGetLastError();
        return set_err(STABGPU_CUDA, "host_free: not a stabgpu_host_alloc pointer");
    }
    return STABGPU_OK;
}

int stabgpu_stream_set_graphs(stabgpu_stream* s, int on) {
    if (!s) return set_err(STABGPU_INVALID_INPUT, "stream: null handle");
    s->graphs = on != 0 && graph_safe(s->cfg);
    return STABGPU_OK;
}

int stabgpu_stream_destroy(stabgpu_stream* s) {
    if (!s) return STABGPU_OK;
    cudaSetDevice(s->ctx->device);
    cudaStreamSynchronize(s->ctx->stream);
    cudaStreamSynchronize(s->ctx->cin);
    cudaStreamSynchronize(s->ctx->cout);
    if (s->rst) cudaStreamSynchronize(s->rst);
    if (s->dst) cudaStreamSynchronize(s->dst);
    if (s->pst) cudaStreamSynchronize(s->pst);
    for (void* p : s->allocs) cudaFree(p);
    for (auto* v : {&s->slot_free, &s->in_done, &s->out_done, &s->motion_done})
        for (auto e : *v)
            if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {s->ev_scan, s->ev_rel, s->ev_det, s->ev_motion, s->ev_grow, s->ev_pyr, s->ev_chain[0], s->ev_chain[1]})
        if (e) cudaEventDestroy(e);
    if (s->rst) cudaStreamDestroy(s->rst);
    if (s->dst) cudaStreamDestroy(s->dst);
    if (s->pst) cudaStreamDestroy(s->pst);
    for (auto& kv : s->execs) cudaGraphExecDestroy(kv.second);
    if (s->err_host) cudaFreeHost(s->err_host);
    if (s->rec_host) cudaFreeHost(s->rec_host);
    delete s;
    return STABGPU_OK;
}


}  // extern "C"

// ---- device-resident Tracker (flow.hpp:56-82) -------------------------------
// Tracker::advance with its state on the device: the previous frame's
// pyramid (two slots, level 0 included), the carried points and the cadence
// counter.  One call uploads the new frame, builds its pyramid, tracks the
// points forward and weeds them backward (the Stage II LK step), compacts the
// TrackSet and re-detects every redetect_interval frames; only the TrackSet
// comes back.  The reference's frame-by-frame callers (MotionStage, the
// acceptance harness) keep their loop; the pyramids never cross PCIe.
struct stabgpu_tracker {
    stabgpu_ctx* ctx = nullptr;
    stabgpu_flow_cfg flow{};
    stabgpu_detect_cfg detect{};
    int w = 0, h = 0;
    long long last_index = -1, frames = 0;
    int since_detect = 0;
    long long detections = 0;
    std::vector<void*> allocs;
    uint8_t* frame[2] = {nullptr, nullptr};  // level 0 of slots 0 / 1
    DevPyramid P{};                          // levels >= 1 of both slots (slot stride = level size)
    stabgpu_roi roi{};
    DetectScratch ds{};
    double2 *pts = nullptr, *nxt = nullptr, *fwd = nullptr, *trk_prev = nullptr, *trk_cur = nullptr;
    int *npts = nullptr, *nnxt = nullptr, *trk_n = nullptr;
    double* score = nullptr;
    uint8_t* keep = nullptr;
    unsigned* work = nullptr;
    int* host_n = nullptr;  // pinned: TrackSet size, active points
};

namespace {
template <typename T>
int talloc(stabgpu_tracker* t, T** p, size_t count) {
    void* q = nullptr;
    if (cudaMalloc(&q, count * sizeof(T) + 256) != cudaSuccess) {
        cudaGetLastError();
        return set_err(STABGPU_CUDA, "tracker: device allocation of %zu bytes failed", count * sizeof(T));
    }
    t->allocs.push_back(q);
    *p = static_cast<T*>(q);
    return STABGPU_OK;
}
}  // namespace

extern "C" {

int stabgpu_tracker_create(stabgpu_ctx* ctx, const stabgpu_flow_cfg* flow, const stabgpu_detect_cfg* detect, int w,
                           int h, stabgpu_tracker** out) {
    *out = nullptr;
    if (!ctx) return set_err(STABGPU_INVALID_INPUT, "tracker: null context");
    TRY(validate_flow(*flow));
    TRY(validate_detect(*detect));
    TRY(validate_frame(w, h));
    if (flow->window_radius > STABGPU_MAX_RADIUS)
        return set_err(STABGPU_INVALID_CONFIG, "window_radius above 31 is not supported");
    cudaSetDevice(ctx->device);
    auto* t = new stabgpu_tracker();
    t->ctx = ctx;
    t->flow = *flow;
    t->detect = *detect;
    t->w = w;
    t->h = h;
    int rc = STABGPU_OK;
    auto fail = [&](int code) {
        stabgpu_tracker_destroy(t);
        return code;
    };
    const int maxc = detect->max_corners;
    const size_t fl = (size_t)w * h;
    if ((rc = talloc(t, &t->frame[0], 2 * fl))) return fail(rc);
    t->frame[1] = t->frame[0] + fl;
    t->P.levels = level_dims(w, h, flow->max_levels, t->P.w, t->P.h);
    t->P.stride[0] = fl;
    for (int l = 1; l < t->P.levels; ++l) {
        uint8_t* lv;
        t->P.stride[l] = (size_t)t->P.w[l] * t->P.h[l];
        if ((rc = talloc(t, &lv, 2 * t->P.stride[l]))) return fail(rc);
        t->P.lvl[l] = lv;
    }
    if ((rc = roi_of(w, h, detect->roi_margin, &t->roi))) return fail(rc);
    const size_t cap = (size_t)(t->roi.x1 - t->roi.x0) * (t->roi.y1 - t->roi.y0);
    DetectScratch& d = t->ds;
    d.cap = cap;
    if ((rc = talloc(t, &d.maxbits, 1)) || (rc = talloc(t, &d.count, 1)) || (rc = talloc(t, &d.hist, kRespBins)) ||
        (rc = talloc(t, &d.cand_key, cap)) || (rc = talloc(t, &d.cand_idx, cap)) ||
        (rc = talloc(t, &d.sort_key, cap)) || (rc = talloc(t, &d.sort_idx, cap)) || (rc = talloc(t, &d.lo, 1)) ||
        (rc = talloc(t, &d.flags, 1)) || (rc = talloc(t, &d.mlo, 1)) || (rc = talloc(t, &d.bstart, kBuckets + 1)) ||
        (rc = talloc(t, &d.bcur, kBuckets)))
        return fail(rc);
    if ((rc = talloc(t, &t->pts, maxc)) || (rc = talloc(t, &t->nxt, maxc)) || (rc = talloc(t, &t->fwd, maxc)) ||
        (rc = talloc(t, &t->trk_prev, maxc)) || (rc = talloc(t, &t->trk_cur, maxc)) || (rc = talloc(t, &t->npts, 1)) ||
        (rc = talloc(t, &t->nnxt, 1)) || (rc = talloc(t, &t->trk_n, 1)) || (rc = talloc(t, &t->score, maxc)) ||
        (rc = talloc(t, &t->keep, maxc)) || (rc = talloc(t, &t->work, 1)))
        return fail(rc);
    if (cudaMallocHost((void**)&t->host_n, 2 * sizeof(int)) != cudaSuccess)
        return fail(set_err(STABGPU_CUDA, "tracker: pinned allocation failed"));
    *out = t;
    return STABGPU_OK;
}

int stabgpu_tracker_advance(stabgpu_tracker* t, const uint8_t* host_frame, int64_t index, int* kind,
                            double* prev_xy, double* cur_xy, int* n_out, int* n_active) {
    if (!t) return set_err(STABGPU_INVALID_INPUT, "tracker: null handle");
    *n_out = 0;
    if (index <= t->last_index) return set_err(STABGPU_SEQUENCING, "frame index must be strictly increasing");
    stabgpu_ctx* ctx = t->ctx;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    t->last_index = index;
    const long long f = t->frames;
    const int cs = (int)(f & 1), ps = cs ^ 1;
    const size_t fl = (size_t)t->w * t->h;
    uint8_t* fy = t->frame[cs];
    CUDA_TRY(cudaMemcpyAsync(fy, host_frame, fl, cudaMemcpyHostToDevice, st));
    DevPyramid& P = t->P;
    for (int l = 1; l < P.levels; ++l)  // build_pyramid (image_ops.cpp:62-77) into slot cs
        launch_pyramid_level(l == 1 ? fy : P.lvl[l - 1] + cs * P.stride[l - 1], P.stride[l - 1], P.w[l - 1],
                             P.h[l - 1], const_cast<uint8_t*>(P.lvl[l]) + cs * P.stride[l], P.stride[l], 1, st);
    ctx->stats.launches += P.levels - 1;
    PlaneBatch cur{fy, fl, t->w, t->h};
    const int maxc = t->detect.max_corners;
    int n = 0;
    if (f == 0) {  // first frame: detect_fresh (flow.cpp:303-308)
        launch_detect(cur, 1, t->detect, t->roi, t->ds, t->pts, t->score, t->npts, st);
        t->since_detect = 0;
        ++t->detections;
        *kind = STABGPU_FRAME_FIRST;
    } else {  // track_lk forward + weed_tracks (flow.cpp:316-323) as one LK step
        DevPyramid V = P;  // frame 0 = previous slot, frame 1 = current slot
        V.lvl[0] = t->frame[ps];
        V.stride[0] = (size_t)(fy - t->frame[ps]);
        for (int l = 1; l < P.levels; ++l) {
            V.lvl[l] = P.lvl[l] + ps * P.stride[l];
            V.stride[l] = (size_t)((ptrdiff_t)(cs - ps) * (ptrdiff_t)P.stride[l]);
        }
        LkStep k;
        std::memset(&k, 0, sizeof k);
        k.pyr = V;
        k.frame0 = 0;
        k.seg_len = t->flow.redetect_interval;
        k.t = 1;
        k.nseg = 1;
        k.max_pts = maxc;
        k.pts = t->pts;
        k.npts = t->npts;
        k.fwd = t->fwd;
        k.keep = t->keep;
        k.nframes = 2;
        k.mode = 1;
        k.work = t->work;
        launch_lk(k, t->flow, st);
        launch_compact(k, t->nxt, t->nnxt, t->trk_prev, t->trk_cur, t->trk_n, 1, st);
        std::swap(t->pts, t->nxt);  // points_ = tracks.cur_points (flow.cpp:326)
        std::swap(t->npts, t->nnxt);
        ctx->stats.launches += 2;
        if (++t->since_detect >= t->flow.redetect_interval) {  // flow.cpp:327-330
            launch_detect(cur, 1, t->detect, t->roi, t->ds, t->pts, t->score, t->npts, st);
            t->since_detect = 0;
            ++t->detections;
        }
        // the whole point arrays come back with the counts (one round trip;
        // max_corners pairs are a few KB)
        CUDA_TRY(cudaMemcpyAsync(t->host_n, t->trk_n, sizeof(int), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(t->host_n + 1, t->npts, sizeof(int), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(prev_xy, t->trk_prev, sizeof(double2) * maxc, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(cur_xy, t->trk_cur, sizeof(double2) * maxc, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        n = t->host_n[0];
        *kind = n < t->flow.min_tracks ? STABGPU_FRAME_SKIPPED : STABGPU_FRAME_TRACKED;
    }
    if (f == 0) CUDA_TRY(cudaMemcpyAsync(t->host_n + 1, t->npts, sizeof(int), cudaMemcpyDeviceToHost, st));
    TRY(check_launch("tracker"));
    CUDA_TRY(cudaStreamSynchronize(st));
    t->frames = f + 1;
    *n_out = n;
    if (n_active) *n_active = t->host_n[1];
    return STABGPU_OK;
}

int stabgpu_tracker_points(stabgpu_tracker* t, int* n_out) {
    if (!t) return set_err(STABGPU_INVALID_INPUT, "tracker: null handle");
    cudaSetDevice(t->ctx->device);
    CUDA_TRY(cudaMemcpyAsync(t->host_n, t->npts, sizeof(int), cudaMemcpyDeviceToHost, t->ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(t->ctx->stream));
    *n_out = t->frames ? *t->host_n : 0;
    return STABGPU_OK;
}

int stabgpu_tracker_destroy(stabgpu_tracker* t) {
    if (!t) return STABGPU_OK;
    cudaSetDevice(t->ctx->device);
    cudaStreamSynchronize(t->ctx->stream);
    for (void* p : t->allocs) cudaFree(p);
    if (t->host_n) cudaFreeHost(t->host_n);
    delete t;
    return STABGPU_OK;
}

// ---- colour I/O + evaluation -----------------------------------------------
int stabgpu_rgb_to_ycbcr(stabgpu_ctx* ctx, const uint8_t* rgb, int n, int w, int h, uint8_t* y, uint8_t* cb,
                         uint8_t* cr) {
    TRY(validate_frame(w, h));
    if (n < 0) return set_err(STABGPU_INVALID_INPUT, "negative frame count");
    cudaSetDevice(ctx->device);
    launch_rgb_to_ycbcr(rgb, (size_t)n * w * h, y, cb, cr, ctx->stream);
    ++ctx->stats.launches;
    TRY(check_launch("rgb_to_ycbcr"));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return STABGPU_OK;
}

int stabgpu_ycbcr_to_rgb(stabgpu_ctx* ctx, const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int n, int w,
                         int h, uint8_t* rgb) {
    TRY(validate_frame(w, h));
    if (n < 0) return set_err(STABGPU_INVALID_INPUT, "negative frame count");
    cudaSetDevice(ctx->device);
    launch_ycbcr_to_rgb(y, cb, cr, (size_t)n * w * h, rgb, ctx->stream);
    ++ctx->stats.launches;
    TRY(check_launch("ycbcr_to_rgb"));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return STABGPU_OK;
}

int stabgpu_stabilize_sequence_rgb(stabgpu_ctx* ctx, const uint8_t* host_rgb, int n, int w, int h,
                                   const stabgpu_config* cfg, uint8_t* host_out_rgb,
                                   stabgpu_frame_record* records) {
    if (!host_rgb || !host_out_rgb) return set_err(STABGPU_INVALID_INPUT, "rgb: null buffer");
    return sequence_host(ctx, nullptr, nullptr, nullptr, host_rgb, n, w, h, w, h, cfg, nullptr, nullptr, nullptr,
                         host_out_rgb, records);
}

int stabgpu_interframe_sse(stabgpu_ctx* ctx, const uint8_t* y, int n, int w, int h, double crop,
                           uint64_t* host_sse, int64_t* host_count) {
    if (!(crop >= 0.0 && crop < 0.5)) return set_err(STABGPU_INVALID_CONFIG, "psnr crop_ratio must lie in [0, 0.5)");
    if (n < 2) return set_err(STABGPU_INVALID_INPUT, "inter-frame PSNR needs at least 2 frames");
    if (w < 1 || h < 1) return set_err(STABGPU_INVALID_INPUT, "empty frames");
    const int mx = (int)std::lround(crop * w), my = (int)std::lround(crop * h);
    const long long count = (long long)std::max(0, w - 2 * mx) * std::max(0, h - 2 * my);
    if (count == 0) return set_err(STABGPU_INVALID_INPUT, "PSNR crop region is empty");
    cudaSetDevice(ctx->device);
    DBUF(unsigned long long, sse, "eval_sse", (size_t)n - 1);
    launch_interframe_sse(y, n, w, h, mx, my, sse, ctx->stream);
    ++ctx->stats.launches;
    TRY(check_launch("interframe_sse"));
    CUDA_TRY(cudaMemcpyAsync(host_sse, sse, sizeof(uint64_t) * (n - 1), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (host_count) *host_count = count;
    return STABGPU_OK;
}

}  // extern "C"


// Profiling hook (tools/probe_pyramid.py), not part of the public ABI: one K1
// level over a frame batch on a caller stream, device pointers.
extern "C" __attribute__((visibility("default"))) void stabgpu_debug_pyramid_level(
    const uint8_t* src, size_t src_stride, int w, int h, uint8_t* dst, size_t dst_stride, int frames, void* stream) {
    stabgpu::launch_pyramid_level(src, src_stride, w, h, dst, dst_stride, frames, (cudaStream_t)stream);
}
