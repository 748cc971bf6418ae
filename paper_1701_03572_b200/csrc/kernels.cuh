// kernels.cuh — host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda.h>

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/stabgpu.h"

namespace stabgpu {

// Batched frame planes: frame f of a plane lives at base + f * stride.
struct PlaneBatch {
    const uint8_t* base;
    size_t stride;
    int w, h;
};

// Batched pyramid: level l of frame f at lvl[l] + f * stride[l].
struct DevPyramid {
    int levels;
    int w[STABGPU_MAX_LEVELS], h[STABGPU_MAX_LEVELS];
    const uint8_t* lvl[STABGPU_MAX_LEVELS];
    size_t stride[STABGPU_MAX_LEVELS];
};

// Per-frame plan output consumed by the compose kernels.
struct FramePlan {
    double tx, ty, theta, s;  // correction transform (delta_to_transform)
    double c, sn;             // cos(theta)/s, sin(theta)/s (warp_similarity, image_ops.cpp:121-122)
    // K8 fast-path steps in 16.48 fixed point: luma walk increments and the
    // chroma map's d/dx (kxx, kyx) and d/dy (kxy, kyy); filled by
    // finish_plan() for the frame geometry
    long long cf, snf, kxx, kyx, kxy, kyy;
};

// Fills the fixed-point members of a FramePlan (host or device).
__host__ __device__ inline void finish_plan(FramePlan& p, int w, int h, int cw, int ch, double crop) {
    const double FIXP = 281474976710656.0;  // 2^48
    p.cf = llrint(p.c * FIXP);
    p.snf = llrint(p.sn * FIXP);
    p.kxx = p.kyx = p.kxy = p.kyy = 0;
    if (cw > 0 && ch > 0) {
        const int mx = (int)llround(crop * w), my = (int)llround(crop * h);
        const double step_x = w > 1 ? (double)(w - 2 * mx - 1) / (w - 1) : 0.0;
        const double step_y = h > 1 ? (double)(h - 2 * my - 1) / (h - 1) : 0.0;
        const double fxl = (double)w / cw, fyl = (double)h / ch;
        const bool crop_on = mx != 0 || my != 0;
        const double lxs = crop_on ? fxl * step_x : fxl, lys = crop_on ? fyl * step_y : fyl;
        p.kxx = llrint(p.c * lxs / fxl * FIXP);
        p.kyx = llrint(-p.sn * lxs / fyl * FIXP);
        p.kxy = llrint(p.sn * lys / fxl * FIXP);
        p.kyy = llrint(p.c * lys / fyl * FIXP);
    }
}

// Device-resident motion records are the public stabgpu_motion_record.

// ---- K1 pyramid (k_pyramid.cu) ----
void launch_pyramid_level(const uint8_t* src, size_t src_stride, int w, int h, uint8_t* dst,
                          size_t dst_stride, int frames, cudaStream_t st);

// ---- K2-K4 detection (k_detect.cu) ----
struct DetectScratch {
    unsigned long long* maxbits;  // [nD]
    unsigned int* count;          // [nD]
    unsigned int* hist;           // [nD][kRespBins] response histogram (fast path), or null
    unsigned long long* cand_key; // [nD][cap]   score bits
    unsigned int* cand_idx;       // [nD][cap]   y*w + x
    unsigned long long* sort_key; // [nD][cap]
    unsigned int* sort_idx;       // [nD][cap]
    size_t cap;                   // candidates per detection frame (ROI area)
    double* lo;                   // [nD] candidate cut (fast path)
    unsigned char* flags;         // [nD] bit 1: redo with the full candidate list
    unsigned* mlo;                // [nD] fp32 bits of a lower bound of the max response
    // optional multi-CTA bucketing of the candidates (K4 phase A), or null:
    unsigned* bstart = nullptr;   // [nD][kBuckets + 1] bucket starts in sort order (counts first)
    unsigned* bcur = nullptr;     // [nD][kBuckets] scatter cursors
};
constexpr int kRespBins = 2048;
constexpr int kBuckets = 8192;
constexpr int kBucketShift = 13;
// Detects corners on nD frames at base + d*stride (d = 0..nD-1); writes up to
// max_corners points per frame (out_xy[d*max + k], out_score) and out_n[d].
void launch_detect(PlaneBatch frames, int nD, const stabgpu_detect_cfg& cfg, stabgpu_roi roi,
                   DetectScratch& s, double2* out_xy, double* out_score, int* out_n,
                   cudaStream_t st);
void launch_gradients(const uint8_t* src, int w, int h, double* gx, double* gy, cudaStream_t st);
void launch_min_eig(const uint8_t* src, int w, int h, int block, double* out, cudaStream_t st);

// ---- K5 LK (k_lk.cu) ----
struct LkStep {
    DevPyramid pyr;       // pyramids of all frames of the chunk
    int frame0;           // chunk-relative frame of segment 0's detection frame
    int seg_len;          // redetect_interval R
    int t;                // step within the segment (1..R): prev = frame0 + s*R + t-1
    int nseg;
    int max_pts;
    const double2* pts;   // [nseg][max_pts]
    const int* npts;      // [nseg]
    double2* fwd;         // [nseg][max_pts] forward result
    uint8_t* keep;        // [nseg][max_pts]
    unsigned long long* iter_count;  // optional LK iteration counter
    int nframes;          // frames in pyr; a segment is active while cur < nframes
    int mode;             // 0 track_lk, 1 forward + weed (sequence), 2 weed only
    const double2* ref;   // mode 2: prev points the backward track must return to
    unsigned* work;       // persistent-warp work counter (zeroed by launch_lk)
    // multi-stream map (seg_base/seg_end below); nsps == 0: one stream
    int F = 0, nsps = 0;
};
// Segment -> frame map of a chunk holding independent streams of F frames
// each (stream-major).  Stream k is cut into nsps segments of R steps from
// its own frame 0, so segment s starts at frame (s/nsps)*F + (s%nsps)*R and
// its chain may not step past (s/nsps)*F + F - 1.  One stream: F = all
// frames of the chunk, nsps = nseg.
__host__ __device__ inline int seg_base(int seg, int R, int F, int nsps) {
    return nsps ? (seg / nsps) * F + (seg % nsps) * R : seg * R;
}
__host__ __device__ inline int seg_end(int seg, int F, int nsps, int nframes) {
    return nsps ? (seg / nsps) * F + F : nframes;
}
void launch_lk(const LkStep& s, const stabgpu_flow_cfg& cfg, cudaStream_t st);
// Whole-segment tracking chains (r <= 15): every detected point of every
// segment through all R steps in one launch.  pos/alive are [R][nseg][max_pts]
// (step t at index t-1): the point after step t and whether step t kept it.
struct LkChain {
    DevPyramid pyr;
    int R, nseg, max_pts, nframes;
    int steps;           // planes of pos/alive: min(R, F - 1), the most steps any segment takes
    int F, nsps;         // segment map (seg_base / seg_end)
    const double2* pts;  // [nseg][max_pts] detected points (frame seg_base(seg))
    const int* npts;     // [nseg]
    double2* pos;
    uint8_t* alive;      // zeroed by launch_lk_chain
    unsigned long long* iter_count;
    unsigned* work;
};
void launch_lk_chain(const LkChain& c, const stabgpu_flow_cfg& cfg, cudaStream_t st);
// 3D uint8 tensor map (x, y, frame) with a box_w x box_h x 1 box (k_compose.cu)
bool encode_u8_3d(CUtensorMap* m, const uint8_t* base, int w, int h, int frames, size_t frame_stride, int box_w,
                  int box_h);
// Ordered compaction of kept pairs: TrackSet of frame (frame0 + s*R + t) and
// the next points of each segment.
void launch_compact(const LkStep& s, double2* next_pts, int* next_n, double2* trk_prev,
                    double2* trk_cur, int* trk_n, int trk_frame0, cudaStream_t st);

// ---- K6 fit + RANSAC (k_fit.cu) ----
// Fits frames [0, nframes) whose TrackSets are trk_*[f*max_pts ...], trk_n[f].
// pre_scratch (2 * kFitPreCtas int2): with nframes == 1, RANSAC's hypotheses are
// scored by kFitPreCtas CTAs first (Stage II), then the fit CTA merges them
constexpr int kFitPreCtas = 32;
void launch_fit(const double2* trk_prev, const double2* trk_cur, const int* trk_n, int max_pts,
                int nframes, long long frame_index0, const stabgpu_config& cfg,
                stabgpu_motion_record* out, cudaStream_t st, long long stream_frames = 0,
                int2* pre_scratch = nullptr);

// ---- K7 plan (k_plan.cu) ----
struct PlanState {  // carried across incremental calls (selector + prefix)
    int current, since, pending, pad;
    double cum[4];
    long long scanned;  // motion records consumed
};
// n_streams > 1: independent scans of streams k = 0..n_streams-1, whose
// records start at k*stream_stride, with states state[k] and error words
// err[k] (default: the word after state[0]).
void launch_plan_scan(const stabgpu_motion_record* motion, long long first, long long count,
                      const stabgpu_config& cfg, PlanState* state, stabgpu_frame_record* rec,
                      double4* cum, cudaStream_t st, int n_streams = 1, long long stream_stride = 0,
                      int* err = nullptr);
struct PlanGeom {  // frame geometry the compose constants depend on
    int w, h, cw, ch;
    double crop;
};
void launch_plan_smooth(const double4* cum, long long n_known, bool complete, long long first,
                        long long count, int radius, stabgpu_frame_record* rec, FramePlan* plan,
                        PlanGeom geo, cudaStream_t st, long long stream_frames = 0);

// launch sequences that allocate stream-ordered scratch (cannot be updated
// in place inside a CUDA graph): K4 with more corners than shared memory
// holds, K6 with more pairs than its shared budget
bool detect_allocates(const stabgpu_detect_cfg& cfg);
bool fit_allocates(int max_pts);

// ---- K8 compose (k_compose.cu) ----
// scratch: optional caller-owned table buffer of compose_scratch_bytes() bytes
// (no stream-ordered allocation inside: CUDA-graph friendly)
void launch_compose(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, const FramePlan* plan, int frames,
                    double crop_ratio, uint8_t* out_y, uint8_t* out_cb, uint8_t* out_cr,
                    cudaStream_t st, void* scratch = nullptr, size_t scratch_bytes = 0);
size_t compose_scratch_bytes(int w, int h, int cw, int ch, int frames);
// K8 with interleaved RGB output (the Y/Cb/Cr -> RGB conversion fused into
// the store; 4:4:4 chroma, crop margins >= 1 px, 16-byte aligned planes);
// false (nothing launched) when not applicable
bool launch_compose_rgb(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, const FramePlan* plan, int frames,
                        double crop_ratio, uint8_t* out_rgb, cudaStream_t st);
void launch_warp_only(const uint8_t* src, int w, int h, const FramePlan* plan, uint8_t* out,
                      cudaStream_t st);
void launch_crop_only(const uint8_t* src, int w, int h, double crop_ratio, uint8_t* out,
                      cudaStream_t st);

}  // namespace stabgpu

namespace stabgpu {
// ---- single-call helpers for the per-stage ABI ----
struct FitResult {
    double tx, ty, theta, s;
    int status, used;
};
void launch_fit_single(const double2* P, const double2* Q, int n, int kind,
                       const stabgpu_ransac_cfg& rc, int min_tracks, long long frame,
                       FitResult* out, uint8_t* mask, cudaStream_t st);
void launch_rms_single(const double2* P, const double2* Q, int n, stabgpu_transform t, double* out,
                       cudaStream_t st);
void launch_prefix(const stabgpu_delta* d, long long n, double4* cum, cudaStream_t st);
void launch_plan_from_corrections(const stabgpu_transform* corr, long long n, FramePlan* plan,
                                  PlanGeom geo, cudaStream_t st);
// ---- colour conversion + evaluation (k_eval.cu) ----
void launch_rgb_to_ycbcr(const uint8_t* rgb, size_t npx, uint8_t* y, uint8_t* cb, uint8_t* cr, cudaStream_t st,
                         bool zero_copy = false);
void launch_ycbcr_to_rgb(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, size_t npx, uint8_t* rgb,
                         cudaStream_t st);
void launch_interframe_sse(const uint8_t* frames, int n, int w, int h, int mx, int my, unsigned long long* sse,
                           cudaStream_t st);

}  // namespace stabgpu
