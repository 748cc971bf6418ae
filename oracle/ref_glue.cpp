// ref_glue.cpp — C entry points onto the UNMODIFIED reference stabilizer
// (test infrastructure + CPU baseline; never part of the product).
//
// Built by oracle/Makefile together with the reference's own sources, in
// place under /root/reference/proj/src, into oracle/_ref/libstabref.so.  Each
// ref_* function converts plain buffers into the reference value types
// (frame.hpp, flow.hpp, transform.hpp), calls the reference function named
// in its comment and maps exceptions onto stabgpu_status codes.
//
// Two pieces here are not reference code, because the reference has no
// counterpart: the RANSAC wrapper (SPEC.md:330 leaves room for one; this is
// an independent C++ restatement of the rule documented in stab_oracle.c,
// refitting with the reference estimate_*), and the multi-threaded driver
// used as the CPU baseline, which runs reference Trackers on independent
// re-detect segments on std::threads.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <deque>
#include <exception>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "../include/stabgpu.h"
#include "stab/features.hpp"
#include "stab/flow.hpp"
#include "stab/image_ops.hpp"
#include "stab/motion.hpp"
#include "stab/pipeline.hpp"
#include "stab/smoothing.hpp"
#include "stab/stream.hpp"
#include "stab/synth_eval.hpp"

namespace {

thread_local std::string g_err;

int map_exception() {
    try {
        throw;
    } catch (const stab::InvalidInputError& e) {
        g_err = e.what();
        return STABGPU_INVALID_INPUT;
    } catch (const stab::InvalidConfigError& e) {
        g_err = e.what();
        return STABGPU_INVALID_CONFIG;
    } catch (const stab::InvalidTransformError& e) {
        g_err = e.what();
        return STABGPU_INVALID_TRANSFORM;
    } catch (const stab::DegenerateInputError& e) {
        g_err = e.what();
        return STABGPU_DEGENERATE_INPUT;
    } catch (const stab::SequencingError& e) {
        g_err = e.what();
        return STABGPU_SEQUENCING;
    } catch (const stab::IoError& e) {
        g_err = e.what();
        return STABGPU_IO;
    } catch (const std::exception& e) {
        g_err = e.what();
        return STABGPU_INVALID_INPUT;
    }
}

#define GUARD_BEGIN try {
#define GUARD_END \
    }             \
    catch (...) { return map_exception(); } \
    return STABGPU_OK;

stab::GrayFrame frame_of(const uint8_t* px, int w, int h, std::int64_t index = 0) {
    stab::GrayFrame f(w, h, index);
    std::memcpy(f.pixels.data(), px, static_cast<std::size_t>(w) * h);
    return f;
}

stab::Pyramid pyramid_of(const stabgpu_pyramid* p) {
    stab::Pyramid pyr;
    for (int l = 0; l < p->levels; ++l)
        pyr.levels.push_back(frame_of(p->data + p->offset[l], p->width[l], p->height[l]));
    return pyr;
}

std::vector<stab::Point2> points_of(const double* xy, int n) {
    std::vector<stab::Point2> v(n);
    for (int i = 0; i < n; ++i) v[i] = {xy[2 * i], xy[2 * i + 1]};
    return v;
}

stab::SimilarityTransform transform_of(const stabgpu_transform* t) {
    stab::SimilarityTransform s;
    s.tx = t->tx;
    s.ty = t->ty;
    s.theta = t->theta;
    s.s = t->s;
    s.kind = t->kind == STABGPU_RIGID ? stab::ModelKind::Rigid : stab::ModelKind::Similarity;
    return s;
}

void put_transform(const stab::SimilarityTransform& s, stabgpu_transform* t) {
    t->tx = s.tx;
    t->ty = s.ty;
    t->theta = s.theta;
    t->s = s.s;
    t->kind = s.kind == stab::ModelKind::Rigid ? STABGPU_RIGID : STABGPU_SIMILARITY;
}

void put_delta(const stab::DeltaParams& d, stabgpu_delta* o) {
    o->dx = d.dx;
    o->dy = d.dy;
    o->da = d.da;
    o->dls = d.dls;
    o->kind = d.kind == stab::ModelKind::Rigid ? STABGPU_RIGID : STABGPU_SIMILARITY;
    o->skipped = d.skipped ? 1 : 0;
}

stab::StabConfig stab_config_of(const stabgpu_config* c) {
    stab::StabConfig s;
    s.detect.max_corners = c->detect.max_corners;
    s.detect.quality_level = c->detect.quality_level;
    s.detect.min_distance = c->detect.min_distance;
    s.detect.block_size = c->detect.block_size;
    s.detect.roi_margin = c->detect.roi_margin;
    s.flow.window_radius = c->flow.window_radius;
    s.flow.max_levels = c->flow.max_levels;
    s.flow.max_iterations = c->flow.max_iterations;
    s.flow.epsilon = c->flow.epsilon;
    s.flow.fb_threshold = c->flow.fb_threshold;
    s.flow.redetect_interval = c->flow.redetect_interval;
    s.flow.min_tracks = c->flow.min_tracks;
    s.smooth.radius = c->smooth_radius;
    s.selector.dwell = c->selector.dwell;
    s.selector.margin = c->selector.margin;
    s.selector.mode = c->selector.mode == STABGPU_FORCE_RIGID        ? stab::SelectionMode::ForceRigid
                      : c->selector.mode == STABGPU_FORCE_SIMILARITY ? stab::SelectionMode::ForceSimilarity
                                                                     : stab::SelectionMode::Hybrid;
    s.crop_ratio = c->crop_ratio;
    s.queue_capacity = c->queue_capacity;
    return s;
}

// ---- RANSAC (independent restatement of the rule in stab_oracle.c) ----
std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

struct Minimal {
    double a, b, tx, ty;
};

bool solve_pair(const stab::TrackSet& ts, std::size_t i, std::size_t j, bool rigid, Minimal& m) {
    const stab::Point2 pi = ts.prev_points[i], pj = ts.prev_points[j];
    const stab::Point2 qi = ts.cur_points[i], qj = ts.cur_points[j];
    const double mpx = 0.5 * (pi.x + pj.x), mpy = 0.5 * (pi.y + pj.y);
    const double mqx = 0.5 * (qi.x + qj.x), mqy = 0.5 * (qi.y + qj.y);
    const double ax = pj.x - pi.x, ay = pj.y - pi.y;
    const double bx = qj.x - qi.x, by = qj.y - qi.y;
    const double norm = ax * ax + ay * ay;
    if (norm == 0.0) return false;
    double a = (ax * bx + ay * by) / norm;
    double b = (ax * by - ay * bx) / norm;
    if (rigid) {
        const double r = std::sqrt(a * a + b * b);
        if (r == 0.0) return false;
        a = a / r;
        b = b / r;
    }
    m = {a, b, mqx - (a * mpx - b * mpy), mqy - (b * mpx + a * mpy)};
    return true;
}

bool is_inlier(const Minimal& m, stab::Point2 p, stab::Point2 q, double thr2) {
    const double ex = q.x - ((m.a * p.x - m.b * p.y) + m.tx);
    const double ey = q.y - ((m.b * p.x + m.a * p.y) + m.ty);
    return ex * ex + ey * ey <= thr2;
}

stab::SimilarityTransform fit_kind(const stab::TrackSet& ts, bool rigid) {
    return rigid ? stab::estimate_rigid(ts) : stab::estimate_similarity(ts);
}

// Robust estimate: returns the refit and the inlier count used.
stab::SimilarityTransform robust_fit(const stab::TrackSet& ts, bool rigid,
                                     const stabgpu_ransac_cfg& rc, int min_tracks,
                                     std::int64_t frame, int* n_used,
                                     std::vector<std::uint8_t>* mask = nullptr) {
    const std::size_t n = ts.size();
    if (n < 2) throw stab::DegenerateInputError("estimation needs at least 2 point pairs");
    int best_count = 0;
    bool have = false;
    Minimal best{};
    if (rc.iterations > 0) {
        const double thr2 = rc.threshold * rc.threshold;
        const std::uint64_t key = mix64(rc.seed ^ mix64(static_cast<std::uint64_t>(frame) +
                                                        0x9e3779b97f4a7c15ULL));
        for (int h = 0; h < rc.iterations; ++h) {
            const std::uint64_t u =
                mix64(key + static_cast<std::uint64_t>(h + 1) * 0x9e3779b97f4a7c15ULL);
            const std::size_t i = static_cast<std::uint32_t>(u >> 32) % static_cast<std::uint32_t>(n);
            std::size_t j = static_cast<std::uint32_t>(u) % static_cast<std::uint32_t>(n - 1);
            if (j >= i) ++j;
            Minimal m;
            if (!solve_pair(ts, i, j, rigid, m)) continue;
            int cnt = 0;
            for (std::size_t k = 0; k < n; ++k)
                cnt += is_inlier(m, ts.prev_points[k], ts.cur_points[k], thr2) ? 1 : 0;
            if (cnt > best_count) {
                best_count = cnt;
                best = m;
                have = true;
            }
        }
    }
    if (!have || best_count < min_tracks) {
        *n_used = static_cast<int>(n);
        if (mask) mask->assign(n, 1);
        return fit_kind(ts, rigid);
    }
    const double thr2 = rc.threshold * rc.threshold;
    stab::TrackSet in;
    in.frame_index = ts.frame_index;
    if (mask) mask->assign(n, 0);
    for (std::size_t k = 0; k < n; ++k) {
        if (is_inlier(best, ts.prev_points[k], ts.cur_points[k], thr2)) {
            in.prev_points.push_back(ts.prev_points[k]);
            in.cur_points.push_back(ts.cur_points[k]);
            if (mask) (*mask)[k] = 1;
        }
    }
    *n_used = static_cast<int>(in.size());
    return fit_kind(in, rigid);
}

// Per-frame motion result of one Tracker step (both fits in hybrid mode).
struct FrameMotion {
    int kind = STABGPU_FRAME_FIRST;
    int n_tracks = 0;
    stab::SimilarityTransform rigid, similarity;
    int n_rigid = 0, n_similarity = 0;
    double e_rigid = 0.0, e_similarity = 0.0;
};

// ModelSelector::select / note_skipped (motion.cpp:143-191) over
// precomputed fits; identical decisions because fits are pure functions of
// the TrackSet.
struct SelectorScan {
    stabgpu_selector_cfg cfg;
    int current;
    int since = 0;
    bool pending = true;
    explicit SelectorScan(const stabgpu_selector_cfg& c)
        : cfg(c), current(c.mode == STABGPU_FORCE_SIMILARITY ? STABGPU_SIMILARITY : STABGPU_RIGID) {}
    void advance() { since = (since + 1) % cfg.dwell; }
    void note_skipped() {
        if (since == 0) pending = true;
        advance();
    }
    // returns the chosen transform and decision flag
    const stab::SimilarityTransform& select(const FrameMotion& m, int* n_used, int* decision) {
        if (since == 0) pending = true;
        *decision = 0;
        const stab::SimilarityTransform* out = nullptr;
        if (cfg.mode == STABGPU_FORCE_RIGID || cfg.mode == STABGPU_FORCE_SIMILARITY) {
            const bool rigid = cfg.mode == STABGPU_FORCE_RIGID;
            out = rigid ? &m.rigid : &m.similarity;
            *n_used = rigid ? m.n_rigid : m.n_similarity;
            if (pending) {
                current = rigid ? STABGPU_RIGID : STABGPU_SIMILARITY;
                pending = false;
                *decision = 1;
            }
        } else if (pending) {
            if (m.e_rigid <= m.e_similarity * (1.0 + cfg.margin)) {
                current = STABGPU_RIGID;
                out = &m.rigid;
                *n_used = m.n_rigid;
            } else {
                current = STABGPU_SIMILARITY;
                out = &m.similarity;
                *n_used = m.n_similarity;
            }
            pending = false;
            *decision = 1;
        } else {
            out = current == STABGPU_RIGID ? &m.rigid : &m.similarity;
            *n_used = current == STABGPU_RIGID ? m.n_rigid : m.n_similarity;
        }
        advance();
        return *out;
    }
};

void motion_of(const stab::TrackSet& ts, const stabgpu_config& c, std::int64_t frame,
               FrameMotion& m) {
    m.n_tracks = static_cast<int>(ts.size());
    const bool need_rigid = c.selector.mode != STABGPU_FORCE_SIMILARITY;
    const bool need_sim = c.selector.mode != STABGPU_FORCE_RIGID;
    if (need_rigid) m.rigid = robust_fit(ts, true, c.ransac, c.flow.min_tracks, frame, &m.n_rigid);
    if (need_sim)
        m.similarity = robust_fit(ts, false, c.ransac, c.flow.min_tracks, frame, &m.n_similarity);
    if (need_rigid && need_sim) {
        m.e_rigid = stab::rms_residual(ts, m.rigid);
        m.e_similarity = stab::rms_residual(ts, m.similarity);
    }
}

// Runs reference Trackers over frames [first, last] (first is a re-detect
// frame) and fills motion[first+1 .. last] (and motion[0] when first == 0).
void track_range(const uint8_t* y, int w, int h, int first, int last, const stabgpu_config& c,
                 const stab::StabConfig& sc, std::vector<FrameMotion>& motion) {
    stab::Tracker tracker(sc.flow, sc.detect);
    for (int f = first; f <= last; ++f) {
        stab::GrayFrame fr = frame_of(y + static_cast<std::size_t>(f) * w * h, w, h, f);
        stab::Tracker::Advance adv = tracker.advance(fr);
        if (f == first) {
            if (f == 0) motion[0].kind = STABGPU_FRAME_FIRST;
            continue;
        }
        FrameMotion& m = motion[f];
        if (adv.kind == stab::Tracker::Advance::Kind::Skipped) {
            m.kind = STABGPU_FRAME_SKIPPED;
            m.n_tracks = 0;  // filled below if tracks exist
            continue;
        }
        m.kind = STABGPU_FRAME_TRACKED;
        motion_of(adv.tracks, c, f, m);
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

size_t ref_pyramid_bytes(int w, int h, int max_levels) {
    size_t total = 0;
    for (int l = 0; l < max_levels && l < STABGPU_MAX_LEVELS; ++l) {
        total += static_cast<size_t>(w) * h;
        if (w / 2 < stab::kMinFrameDim || h / 2 < stab::kMinFrameDim) break;
        w /= 2;
        h /= 2;
    }
    return total;
}

// build_pyramid, image_ops.cpp:62-77
int ref_build_pyramid(const uint8_t* src, int w, int h, int max_levels, stabgpu_pyramid* out) {
    GUARD_BEGIN
    stab::GrayFrame f(w, h);
    if (w > 0 && h > 0) std::memcpy(f.pixels.data(), src, static_cast<std::size_t>(w) * h);
    const stab::Pyramid p = stab::build_pyramid(f, max_levels);
    size_t off = 0;
    out->levels = p.level_count();
    for (int l = 0; l < p.level_count(); ++l) {
        out->width[l] = p.levels[l].width;
        out->height[l] = p.levels[l].height;
        out->offset[l] = off;
        std::memcpy(out->data + off, p.levels[l].pixels.data(), p.levels[l].pixels.size());
        off += p.levels[l].pixels.size();
    }
    GUARD_END
}

// gradients, image_ops.cpp:79-96
int ref_gradients(const uint8_t* src, int w, int h, double* gx, double* gy) {
    GUARD_BEGIN
    auto [a, b] = stab::gradients(frame_of(src, w, h));
    std::memcpy(gx, a.values.data(), a.values.size() * sizeof(double));
    std::memcpy(gy, b.values.data(), b.values.size() * sizeof(double));
    GUARD_END
}

// min_eig_response, features.cpp:78-87
int ref_min_eig_response(const uint8_t* src, int w, int h, int block, double* out) {
    GUARD_BEGIN
    const stab::ScalarMap m = stab::min_eig_response(frame_of(src, w, h), block);
    std::memcpy(out, m.values.data(), m.values.size() * sizeof(double));
    GUARD_END
}

// detection_roi, features.cpp:28-36
int ref_detection_roi(int w, int h, double margin, stabgpu_roi* out) {
    GUARD_BEGIN
    stab::GrayFrame f;
    f.width = w;
    f.height = h;
    const stab::RoiRect r = stab::detection_roi(f, margin);
    *out = {r.x0, r.y0, r.x1, r.y1};
    GUARD_END
}

// detect_corners, features.cpp:89-141
int ref_detect_corners(const uint8_t* src, int w, int h, const stabgpu_detect_cfg* c, double* xy,
                       double* score, int* n_out) {
    *n_out = 0;
    GUARD_BEGIN
    stab::DetectConfig dc;
    dc.max_corners = c->max_corners;
    dc.quality_level = c->quality_level;
    dc.min_distance = c->min_distance;
    dc.block_size = c->block_size;
    dc.roi_margin = c->roi_margin;
    const auto corners = stab::detect_corners(frame_of(src, w, h), dc);
    for (std::size_t i = 0; i < corners.size(); ++i) {
        xy[2 * i] = corners[i].position.x;
        xy[2 * i + 1] = corners[i].position.y;
        score[i] = corners[i].score;
    }
    *n_out = static_cast<int>(corners.size());
    GUARD_END
}

static stab::FlowConfig flow_of(const stabgpu_flow_cfg* c) {
    stab::FlowConfig f;
    f.window_radius = c->window_radius;
    f.max_levels = c->max_levels;
    f.max_iterations = c->max_iterations;
    f.epsilon = c->epsilon;
    f.fb_threshold = c->fb_threshold;
    f.redetect_interval = c->redetect_interval;
    f.min_tracks = c->min_tracks;
    return f;
}

// track_lk, flow.cpp:243-256
int ref_track_lk(const stabgpu_pyramid* prev, const stabgpu_pyramid* cur, const double* xy, int n,
                 const stabgpu_flow_cfg* c, double* out, uint8_t* ok) {
    GUARD_BEGIN
    const auto pts = points_of(xy, n);
    const auto res = stab::track_lk(pyramid_of(prev), pyramid_of(cur), pts, flow_of(c));
    for (int i = 0; i < n; ++i) {
        out[2 * i] = res[i].position.x;
        out[2 * i + 1] = res[i].position.y;
        ok[i] = res[i].ok ? 1 : 0;
    }
    GUARD_END
}

// weed_tracks, flow.cpp:258-280
int ref_weed_tracks(const stabgpu_pyramid* prev, const stabgpu_pyramid* cur, const double* pxy,
                    const double* cxy, int n, const stabgpu_flow_cfg* c, double* kp, double* kc,
                    int* n_out) {
    *n_out = 0;
    GUARD_BEGIN
    const auto pp = points_of(pxy, n), cp = points_of(cxy, n);
    const stab::TrackSet ts = stab::weed_tracks(pyramid_of(prev), pyramid_of(cur), pp, cp, flow_of(c));
    for (std::size_t i = 0; i < ts.size(); ++i) {
        kp[2 * i] = ts.prev_points[i].x;
        kp[2 * i + 1] = ts.prev_points[i].y;
        kc[2 * i] = ts.cur_points[i].x;
        kc[2 * i + 1] = ts.cur_points[i].y;
    }
    *n_out = static_cast<int>(ts.size());
    GUARD_END
}

static stab::TrackSet trackset_of(const double* p, const double* q, int n) {
    stab::TrackSet ts;
    ts.prev_points = points_of(p, n);
    ts.cur_points = points_of(q, n);
    return ts;
}

// estimate_rigid / estimate_similarity, motion.cpp:62-76
int ref_estimate(const double* p, const double* q, int n, int kind, stabgpu_transform* out) {
    GUARD_BEGIN
    put_transform(fit_kind(trackset_of(p, q, n), kind == STABGPU_RIGID), out);
    GUARD_END
}

// rms_residual, motion.cpp:78-90
int ref_rms_residual(const double* p, const double* q, int n, const stabgpu_transform* t,
                     double* out) {
    GUARD_BEGIN
    *out = stab::rms_residual(trackset_of(p, q, n), transform_of(t));
    GUARD_END
}

int ref_ransac_estimate(const double* p, const double* q, int n, int kind,
                        const stabgpu_ransac_cfg* rc, int min_tracks, int64_t frame,
                        stabgpu_transform* out, uint8_t* inliers, int* n_inliers) {
    GUARD_BEGIN
    std::vector<std::uint8_t> mask;
    stabgpu_ransac_cfg off{0, 0.0, 0};
    put_transform(robust_fit(trackset_of(p, q, n), kind == STABGPU_RIGID, rc ? *rc : off,
                             min_tracks, frame, n_inliers, &mask),
                  out);
    if (inliers) std::memcpy(inliers, mask.data(), mask.size());
    GUARD_END
}

// extract_delta / delta_to_transform, motion.cpp:92-111
void ref_extract_delta(const stabgpu_transform* t, stabgpu_delta* out) {
    put_delta(stab::extract_delta(transform_of(t)), out);
}

void ref_delta_to_transform(double dx, double dy, double da, double dls, stabgpu_transform* out) {
    put_transform(stab::delta_to_transform(dx, dy, da, dls), out);
}

// Trajectory append / mark_complete / correction, smoothing.cpp:16-57
int ref_trajectory_corrections(const stabgpu_delta* d, int n, int radius, stabgpu_transform* out) {
    GUARD_BEGIN
    stab::Trajectory traj;
    for (int i = 0; i < n; ++i) {
        stab::DeltaParams p;
        p.dx = d[i].dx;
        p.dy = d[i].dy;
        p.da = d[i].da;
        p.dls = d[i].dls;
        traj.append(p);
    }
    traj.mark_complete();
    stab::SmoothConfig sc;
    sc.radius = radius;
    for (int i = 0; i < n; ++i) put_transform(*traj.correction(i, sc), &out[i]);
    GUARD_END
}

// warp_similarity / crop_resize / compose_stabilized, image_ops.cpp:115-219
int ref_warp_similarity(const uint8_t* src, int w, int h, const stabgpu_transform* t, uint8_t* out) {
    GUARD_BEGIN
    const stab::GrayFrame r = stab::warp_similarity(frame_of(src, w, h), transform_of(t));
    std::memcpy(out, r.pixels.data(), r.pixels.size());
    GUARD_END
}

int ref_crop_resize(const uint8_t* src, int w, int h, double crop, uint8_t* out) {
    GUARD_BEGIN
    const stab::GrayFrame r = stab::crop_resize(frame_of(src, w, h), crop);
    std::memcpy(out, r.pixels.data(), r.pixels.size());
    GUARD_END
}

static stab::VideoFrame video_of(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int w,
                                 int h, int cw, int ch, std::int64_t index) {
    stab::VideoFrame v;
    v.luma = frame_of(y, w, h, index);
    if (cb && cr) {
        v.chroma_width = cw;
        v.chroma_height = ch;
        v.cb.assign(cb, cb + static_cast<std::size_t>(cw) * ch);
        v.cr.assign(cr, cr + static_cast<std::size_t>(cw) * ch);
    }
    return v;
}

int ref_compose_stabilized(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int w, int h,
                           int cw, int ch, const stabgpu_transform* t, double crop, uint8_t* oy,
                           uint8_t* ocb, uint8_t* ocr) {
    GUARD_BEGIN
    const stab::VideoFrame o =
        stab::compose_stabilized(video_of(y, cb, cr, w, h, cw, ch, 0), transform_of(t), crop);
    std::memcpy(oy, o.luma.pixels.data(), o.luma.pixels.size());
    if (o.has_chroma()) {
        std::memcpy(ocb, o.cb.data(), o.cb.size());
        std::memcpy(ocr, o.cr.data(), o.cr.size());
    }
    GUARD_END
}

// run_offline (pipeline.cpp:182-235) through the reference's own driver:
// in-memory FrameSource/FrameSink over the caller's planes.  Only valid with
// RANSAC off (the reference has no robust estimator).
namespace {
struct PlaneSource : stab::FrameSource {
    const uint8_t *y, *cb, *cr;
    int n, w, h, cw, ch, next_i = 0;
    std::optional<stab::VideoFrame> next() override {
        if (next_i >= n) return std::nullopt;
        const std::size_t lo = static_cast<std::size_t>(next_i) * w * h;
        const std::size_t co = static_cast<std::size_t>(next_i) * cw * ch;
        stab::VideoFrame v = video_of(y + lo, cb ? cb + co : nullptr, cr ? cr + co : nullptr, w, h,
                                      cw, ch, next_i);
        ++next_i;
        return v;
    }
};
struct PlaneSink : stab::FrameSink {
    uint8_t *y, *cb, *cr;
    int w, h, cw, ch, count = 0;
    void push(stab::VideoFrame f) override {
        if (y) std::memcpy(y + static_cast<std::size_t>(count) * w * h, f.luma.pixels.data(), f.luma.pixels.size());
        if (cb && f.has_chroma()) {
            std::memcpy(cb + static_cast<std::size_t>(count) * cw * ch, f.cb.data(), f.cb.size());
            std::memcpy(cr + static_cast<std::size_t>(count) * cw * ch, f.cr.data(), f.cr.size());
        }
        ++count;
    }
};
}  // namespace

int ref_run_offline(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int n, int w, int h,
                    int cw, int ch, const stabgpu_config* c, uint8_t* oy, uint8_t* ocb,
                    uint8_t* ocr, stabgpu_delta* deltas, stabgpu_transform* corrections,
                    double* wall_seconds) {
    GUARD_BEGIN
    PlaneSource src;
    src.y = y;
    src.cb = cb;
    src.cr = cr;
    src.n = n;
    src.w = w;
    src.h = h;
    src.cw = cw;
    src.ch = ch;
    PlaneSink sink;
    sink.y = oy;
    sink.cb = ocb;
    sink.cr = ocr;
    sink.w = w;
    sink.h = h;
    sink.cw = cw;
    sink.ch = ch;
    stab::Trajectory traj;
    const stab::StabConfig sc = stab_config_of(c);
    const stab::RunSummary s = stab::run_offline(src, sc, sink, &traj);
    if (wall_seconds) *wall_seconds = s.wall_seconds;
    for (std::size_t i = 0; i < traj.size(); ++i) {
        if (deltas) put_delta(traj.delta(i), &deltas[i]);
        if (corrections) put_transform(*traj.correction(i, sc.smooth), &corrections[i]);
    }
    GUARD_END
}

// Whole-sequence stabilization with reference stage functions on `threads`
// host threads: reference Trackers on independent re-detect segments
// (tracking state resets at every detection, flow.cpp:326-330), the
// selector scan and Trajectory sequentially, compose_stabilized per frame in
// parallel.  threads == 1 is the frame-sequential reference order.
int ref_stabilize_sequence(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int n, int w,
                           int h, int cw, int ch, const stabgpu_config* c, uint8_t* oy,
                           uint8_t* ocb, uint8_t* ocr, stabgpu_frame_record* rec, int threads) {
    GUARD_BEGIN
    const stab::StabConfig sc = stab_config_of(c);
    stab::validate(sc);
    if (c->ransac.iterations < 0 || (c->ransac.iterations > 0 && !(c->ransac.threshold > 0.0)))
        throw stab::InvalidConfigError("ransac needs iterations >= 0 and threshold > 0");
    if (n < 2) throw stab::InvalidInputError("stabilization needs at least 2 frames");
    const int R = c->flow.redetect_interval;
    const int nseg = (n - 1 + R - 1) / R;  // segments [sR, min((s+1)R, n-1)]
    std::vector<FrameMotion> motion(n);
    threads = std::max(1, std::min(threads, nseg));
    std::vector<std::exception_ptr> errs(threads);
    {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    const int s0 = static_cast<int>(static_cast<long long>(nseg) * t / threads);
                    const int s1 = static_cast<int>(static_cast<long long>(nseg) * (t + 1) / threads);
                    if (s0 < s1) track_range(y, w, h, s0 * R, std::min(s1 * R, n - 1), *c, sc, motion);
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        }
        for (auto& th : pool) th.join();
    }
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    // MotionStage::step + selector scan (pipeline.cpp:80-101).
    SelectorScan sel(c->selector);
    stab::Trajectory traj;
    std::vector<stabgpu_frame_record> recs(n);
    for (int f = 0; f < n; ++f) {
        const FrameMotion& m = motion[f];
        stab::DeltaParams d;
        stabgpu_frame_record& r = recs[f];
        std::memset(&r, 0, sizeof r);
        r.frame_kind = m.kind;
        r.n_tracks = m.n_tracks;
        if (m.kind != STABGPU_FRAME_TRACKED) {
            sel.note_skipped();
            d.kind = sel.current == STABGPU_RIGID ? stab::ModelKind::Rigid : stab::ModelKind::Similarity;
            d.skipped = m.kind == STABGPU_FRAME_SKIPPED;
        } else {
            int used = 0, dec = 0;
            d = stab::extract_delta(sel.select(m, &used, &dec));
            r.n_inliers = used;
            r.decision = dec;
        }
        put_delta(d, &r.delta);
        traj.append(d);
    }
    traj.mark_complete();
    std::vector<stab::SimilarityTransform> corr(n);
    for (int f = 0; f < n; ++f) {
        corr[f] = *traj.correction(f, sc.smooth);
        put_transform(corr[f], &recs[f].correction);
    }
    if (rec) std::memcpy(rec, recs.data(), sizeof(stabgpu_frame_record) * n);
    if (oy) {
        std::atomic<int> next{0};
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (int f = next++; f < n; f = next++) {
                        const std::size_t lo = static_cast<std::size_t>(f) * w * h;
                        const std::size_t co = static_cast<std::size_t>(f) * cw * ch;
                        const stab::VideoFrame o = stab::compose_stabilized(
                            video_of(y + lo, cb ? cb + co : nullptr, cr ? cr + co : nullptr, w, h,
                                     cw, ch, f),
                            corr[f], c->crop_ratio);
                        std::memcpy(oy + lo, o.luma.pixels.data(), o.luma.pixels.size());
                        if (ocb && o.has_chroma()) {
                            std::memcpy(ocb + co, o.cb.data(), o.cb.size());
                            std::memcpy(ocr + co, o.cr.data(), o.cr.size());
                        }
                    }
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        }
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    }
    GUARD_END
}

// Motion records of frames first+1 .. first+count from reference Trackers
// (the per-rank work of the sharded Stage I); out holds count+1 entries,
// entry 0 being frame `first` (FIRST on frame 0, frame_kind -1 otherwise).
int ref_motion_chunk(const uint8_t* y, long long first, int count, int w, int h,
                     const stabgpu_config* c, stabgpu_motion_record* out) {
    GUARD_BEGIN
    const stab::StabConfig sc = stab_config_of(c);
    stab::validate(sc);
    std::vector<FrameMotion> m(static_cast<std::size_t>(first) + count + 1);
    // track_range indexes absolute frames; offset the plane pointer so frame
    // `first` lands at index `first`.
    const uint8_t* base = y - static_cast<std::ptrdiff_t>(first) * w * h;
    track_range(base, w, h, static_cast<int>(first), static_cast<int>(first) + count, *c, sc, m);
    for (int k = 0; k <= count; ++k) {
        const FrameMotion& fm = m[first + k];
        stabgpu_motion_record& r = out[k];
        std::memset(&r, 0, sizeof r);
        r.frame_kind = k == 0 ? (first == 0 ? STABGPU_FRAME_FIRST : -1) : fm.kind;
        r.n_tracks = fm.n_tracks;
        put_delta(stab::extract_delta(fm.rigid), &r.rigid);
        put_delta(stab::extract_delta(fm.similarity), &r.similarity);
        r.e_rigid = fm.e_rigid;
        r.e_similarity = fm.e_similarity;
        r.n_inliers_rigid = fm.n_rigid;
        r.n_inliers_similarity = fm.n_similarity;
    }
    GUARD_END
}

// Selector scan + Trajectory over gathered motion records.
int ref_plan_corrections(const stabgpu_motion_record* motion, int n, const stabgpu_config* c,
                         stabgpu_frame_record* rec) {
    GUARD_BEGIN
    const stab::StabConfig sc = stab_config_of(c);
    SelectorScan sel(c->selector);
    stab::Trajectory traj;
    for (int f = 0; f < n; ++f) {
        const stabgpu_motion_record& m = motion[f];
        stabgpu_frame_record& r = rec[f];
        std::memset(&r, 0, sizeof r);
        r.frame_kind = m.frame_kind;
        r.n_tracks = m.n_tracks;
        stab::DeltaParams d;
        if (m.frame_kind != STABGPU_FRAME_TRACKED) {
            sel.note_skipped();
            d.kind = sel.current == STABGPU_RIGID ? stab::ModelKind::Rigid : stab::ModelKind::Similarity;
            d.skipped = m.frame_kind == STABGPU_FRAME_SKIPPED;
        } else {
            FrameMotion fm;
            fm.kind = m.frame_kind;
            fm.rigid = stab::delta_to_transform(m.rigid.dx, m.rigid.dy, m.rigid.da, 0.0);
            fm.rigid.kind = stab::ModelKind::Rigid;
            fm.similarity = stab::delta_to_transform(m.similarity.dx, m.similarity.dy,
                                                     m.similarity.da, m.similarity.dls);
            fm.n_rigid = m.n_inliers_rigid;
            fm.n_similarity = m.n_inliers_similarity;
            fm.e_rigid = m.e_rigid;
            fm.e_similarity = m.e_similarity;
            int used = 0, dec = 0;
            const stab::SimilarityTransform& t = sel.select(fm, &used, &dec);
            const bool rigid = &t == &fm.rigid;
            d.dx = rigid ? m.rigid.dx : m.similarity.dx;
            d.dy = rigid ? m.rigid.dy : m.similarity.dy;
            d.da = rigid ? m.rigid.da : m.similarity.da;
            d.dls = rigid ? 0.0 : m.similarity.dls;
            d.kind = rigid ? stab::ModelKind::Rigid : stab::ModelKind::Similarity;
            r.n_inliers = used;
            r.decision = dec;
        }
        put_delta(d, &r.delta);
        traj.append(d);
    }
    traj.mark_complete();
    for (int f = 0; f < n; ++f) put_transform(*traj.correction(f, sc.smooth), &rec[f].correction);
    GUARD_END
}


// ---- evaluation (synth_eval.cpp:214-349) ----------------------------------
static std::vector<stab::VideoFrame> frames_of(const uint8_t* y, int n, int w, int h) {
    std::vector<stab::VideoFrame> v(n);
    for (int i = 0; i < n; ++i) {
        v[i].luma = stab::GrayFrame(w, h, i);  // Tracker requires increasing frame indices
        std::memcpy(v[i].luma.pixels.data(), y + (size_t)i * w * h, (size_t)w * h);
    }
    return v;
}

int ref_psnr_pair(const uint8_t* a, const uint8_t* b, int w, int h, double crop, double* out) {
    GUARD_BEGIN
    stab::GrayFrame fa(w, h), fb(w, h);
    std::memcpy(fa.pixels.data(), a, (size_t)w * h);
    std::memcpy(fb.pixels.data(), b, (size_t)w * h);
    *out = stab::psnr_pair(fa, fb, crop);
    GUARD_END
}

int ref_reestimate_deltas(const uint8_t* y, int n, int w, int h, stabgpu_delta* out) {
    GUARD_BEGIN
    const std::vector<stab::DeltaParams> d = stab::reestimate_deltas(frames_of(y, n, w, h));
    for (size_t i = 0; i < d.size(); ++i) put_delta(d[i], &out[i]);
    GUARD_END
}

// out: psnr before, after; jitter before (dx dy da dls); jitter after; truth
// rmse (4); has_truth; frames_skipped
int ref_score(const uint8_t* orig, const uint8_t* stabilized, int n, int w, int h, const stabgpu_delta* truth,
              const stabgpu_delta* est, int nt, double crop, double* out) {
    GUARD_BEGIN
    auto deltas = [&](const stabgpu_delta* d) {
        std::vector<stab::DeltaParams> v;
        for (int i = 0; d && i < nt; ++i) {
            stab::DeltaParams p;
            p.dx = d[i].dx;
            p.dy = d[i].dy;
            p.da = d[i].da;
            p.dls = d[i].dls;
            p.kind = d[i].kind == STABGPU_RIGID ? stab::ModelKind::Rigid : stab::ModelKind::Similarity;
            p.skipped = d[i].skipped != 0;
            v.push_back(p);
        }
        return v;
    };
    const stab::EvalReport r = stab::score(frames_of(orig, n, w, h), frames_of(stabilized, n, w, h), deltas(truth),
                                           deltas(est), crop);
    const double vals[16] = {r.mean_psnr_before, r.mean_psnr_after, r.jitter_energy_before.dx,
                             r.jitter_energy_before.dy, r.jitter_energy_before.da, r.jitter_energy_before.dls,
                             r.jitter_energy_after.dx, r.jitter_energy_after.dy, r.jitter_energy_after.da,
                             r.jitter_energy_after.dls, r.truth_recovery_rmse.dx, r.truth_recovery_rmse.dy,
                             r.truth_recovery_rmse.da, r.truth_recovery_rmse.dls, r.has_truth ? 1.0 : 0.0,
                             (double)r.frames_skipped};
    std::memcpy(out, vals, sizeof vals);
    GUARD_END
}

}  // extern "C"
