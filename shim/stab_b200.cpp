// stab_b200.cpp — drop-in replacement for the reference's hot-path
// translation units (image_ops.cpp, features.cpp, flow.cpp, motion.cpp,
// smoothing.cpp): the `stab::` stage API, compiled against the reference's
// own headers (-I$REF/proj/include), executed on the B200 through the C ABI
// in include/stabgpu.h.  A maintainer links libstabcore_b200.so instead of
// those five sources; pipeline.cpp, synth_eval.cpp, media_io.cpp and the
// CLI are unchanged.
//
// Compute (pyramids, gradients, responses, corners, LK, weeding, fits,
// warps, composition) runs in libstabgpu.so.  What stays here is the
// reference API's host bookkeeping — argument validation, Tracker /
// ModelSelector / Trajectory state machines — restated against the same
// headers, because the reference classes keep that state in fixed private
// members (flow.hpp:74-82, motion.hpp:55-65, smoothing.hpp:50-52).
// Exceptions: every stabgpu_status is rethrown as the matching stab:: error.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../include/stabgpu.h"
#include "stab/features.hpp"
#include "stab/flow.hpp"
#include "stab/image_ops.hpp"
#include "stab/motion.hpp"
#include "stab/smoothing.hpp"

namespace {

[[noreturn]] void raise(int rc) {
    const std::string msg = stabgpu_last_error();
    switch (rc) {
        case STABGPU_INVALID_INPUT: throw stab::InvalidInputError(msg);
        case STABGPU_INVALID_CONFIG: throw stab::InvalidConfigError(msg);
        case STABGPU_INVALID_TRANSFORM: throw stab::InvalidTransformError(msg);
        case STABGPU_DEGENERATE_INPUT: throw stab::DegenerateInputError(msg);
        case STABGPU_SEQUENCING: throw stab::SequencingError(msg);
        case STABGPU_IO: throw stab::IoError(msg);
        default: throw stab::Error("stabgpu: " + msg);
    }
}

void check(int rc) {
    if (rc != STABGPU_OK) raise(rc);
}

// One device context per host thread (run_streaming calls stages from three
// threads; contexts own independent streams and scratch).
struct CtxHolder {
    stabgpu_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) stabgpu_destroy(ctx);
    }
};

stabgpu_ctx* ctx() {
    thread_local CtxHolder h;
    if (!h.ctx) check(stabgpu_create(0, &h.ctx));
    return h.ctx;
}

stabgpu_transform to_c(const stab::SimilarityTransform& t) {
    return {t.tx, t.ty, t.theta, t.s, t.kind == stab::ModelKind::Rigid ? STABGPU_RIGID : STABGPU_SIMILARITY};
}

stab::SimilarityTransform from_c(const stabgpu_transform& c) {
    stab::SimilarityTransform t;
    t.tx = c.tx;
    t.ty = c.ty;
    t.theta = c.theta;
    t.s = c.s;
    t.kind = c.kind == STABGPU_RIGID ? stab::ModelKind::Rigid : stab::ModelKind::Similarity;
    return t;
}

stabgpu_detect_cfg to_c(const stab::DetectConfig& d) {
    return {d.max_corners, d.quality_level, d.min_distance, d.block_size, d.roi_margin};
}

stabgpu_flow_cfg to_c(const stab::FlowConfig& f) {
    return {f.window_radius, f.max_levels, f.max_iterations, f.epsilon, f.fb_threshold,
            f.redetect_interval, f.min_tracks};
}

// Packed host view of a stab::Pyramid for the ABI.
struct PackedPyramid {
    std::vector<uint8_t> data;
    stabgpu_pyramid c{};
    explicit PackedPyramid(const stab::Pyramid& p) {
        std::memset(&c, 0, sizeof c);
        c.levels = std::min(p.level_count(), STABGPU_MAX_LEVELS);
        size_t total = 0;
        for (int l = 0; l < c.levels; ++l) total += p.levels[l].pixels.size();
        data.resize(std::max<size_t>(total, 1));
        size_t off = 0;
        for (int l = 0; l < c.levels; ++l) {
            c.width[l] = p.levels[l].width;
            c.height[l] = p.levels[l].height;
            c.offset[l] = off;
            std::memcpy(data.data() + off, p.levels[l].pixels.data(), p.levels[l].pixels.size());
            off += p.levels[l].pixels.size();
        }
        c.data = data.data();
    }
};

std::vector<double> flat(std::span<const stab::Point2> pts) {
    std::vector<double> v(2 * pts.size());
    for (size_t i = 0; i < pts.size(); ++i) {
        v[2 * i] = pts[i].x;
        v[2 * i + 1] = pts[i].y;
    }
    return v;
}

std::vector<double> flat(const std::vector<stab::Point2>& pts) {
    return flat(std::span<const stab::Point2>(pts.data(), pts.size()));
}

}  // namespace

namespace stab {

// ------------------------------------------------------------ image_ops
void validate(const GrayFrame& f) {  // image_ops.cpp:9-16
    if (f.width < kMinFrameDim || f.height < kMinFrameDim)
        throw InvalidInputError("frame smaller than 16x16");
    if (f.pixels.size() != static_cast<size_t>(f.width) * static_cast<size_t>(f.height))
        throw InvalidInputError("pixel buffer length does not match width*height");
}

Pyramid build_pyramid(const GrayFrame& frame, int max_levels) {
    validate(frame);
    if (max_levels < 1) throw InvalidInputError("max_levels must be >= 1");
    std::vector<uint8_t> buf(std::max<size_t>(stabgpu_pyramid_bytes(frame.width, frame.height, max_levels), 1));
    stabgpu_pyramid p{};
    p.data = buf.data();
    check(stabgpu_build_pyramid(ctx(), frame.pixels.data(), frame.width, frame.height, max_levels, &p));
    Pyramid out;
    for (int l = 0; l < p.levels; ++l) {
        GrayFrame g(p.width[l], p.height[l], frame.index);
        std::memcpy(g.pixels.data(), buf.data() + p.offset[l], g.pixels.size());
        out.levels.push_back(std::move(g));
    }
    return out;
}

std::pair<ScalarMap, ScalarMap> gradients(const GrayFrame& frame) {
    validate(frame);
    ScalarMap gx(frame.width, frame.height), gy(frame.width, frame.height);
    check(stabgpu_gradients(ctx(), frame.pixels.data(), frame.width, frame.height, gx.values.data(),
                            gy.values.data()));
    return {std::move(gx), std::move(gy)};
}

// Scalar utility (one point): evaluated here, it is not on the batched path.
double sample_bilinear(const GrayFrame& frame, Point2 p) {
    const double xmax = frame.width - 1.0, ymax = frame.height - 1.0;
    if (!(p.x >= 0.0 && p.y >= 0.0 && p.x <= xmax && p.y <= ymax)) return 0.0;
    const int x0 = static_cast<int>(p.x), y0 = static_cast<int>(p.y);
    const int x1 = std::min(x0 + 1, frame.width - 1), y1 = std::min(y0 + 1, frame.height - 1);
    const double fx = p.x - x0, fy = p.y - y0;
    const double a = frame.at(x0, y0), b = frame.at(x1, y0), c = frame.at(x0, y1), d = frame.at(x1, y1);
    const double top = a + fx * (b - a);
    const double bot = c + fx * (d - c);
    return top + fy * (bot - top);
}

GrayFrame warp_similarity(const GrayFrame& frame, const SimilarityTransform& t) {
    validate(frame);
    validate(t);
    GrayFrame out(frame.width, frame.height, frame.index);
    const stabgpu_transform c = to_c(t);
    check(stabgpu_warp_similarity(ctx(), frame.pixels.data(), frame.width, frame.height, &c,
                                  out.pixels.data()));
    return out;
}

GrayFrame crop_resize(const GrayFrame& frame, double crop_ratio) {
    validate(frame);
    GrayFrame out(frame.width, frame.height, frame.index);
    check(stabgpu_crop_resize(ctx(), frame.pixels.data(), frame.width, frame.height, crop_ratio,
                              out.pixels.data()));
    return out;
}

VideoFrame compose_stabilized(const VideoFrame& in, const SimilarityTransform& correction,
                              double crop_ratio) {
    validate(in.luma);
    VideoFrame out;
    out.luma = GrayFrame(in.luma.width, in.luma.height, in.luma.index);
    const stabgpu_transform c = to_c(correction);
    if (in.has_chroma()) {
        out.chroma_width = in.chroma_width;
        out.chroma_height = in.chroma_height;
        out.cb.resize(in.cb.size());
        out.cr.resize(in.cr.size());
        check(stabgpu_compose_stabilized(ctx(), in.luma.pixels.data(), in.cb.data(), in.cr.data(),
                                         in.luma.width, in.luma.height, in.chroma_width,
                                         in.chroma_height, &c, crop_ratio, out.luma.pixels.data(),
                                         out.cb.data(), out.cr.data()));
    } else {
        check(stabgpu_compose_stabilized(ctx(), in.luma.pixels.data(), nullptr, nullptr,
                                         in.luma.width, in.luma.height, 0, 0, &c, crop_ratio,
                                         out.luma.pixels.data(), nullptr, nullptr));
    }
    return out;
}

// ------------------------------------------------------------- features
void validate(const DetectConfig& cfg) {  // features.cpp:10-26
    if (cfg.max_corners < 8) throw InvalidConfigError("max_corners must be >= 8");
    if (!(cfg.quality_level > 0.0 && cfg.quality_level < 1.0))
        throw InvalidConfigError("quality_level must lie in (0, 1)");
    if (cfg.min_distance < 1.0) throw InvalidConfigError("min_distance must be >= 1");
    if (cfg.block_size < 3 || cfg.block_size % 2 == 0)
        throw InvalidConfigError("block_size must be odd and >= 3");
    if (!(cfg.roi_margin >= 0.0 && cfg.roi_margin < 0.4))
        throw InvalidConfigError("roi_margin must lie in [0, 0.4)");
}

RoiRect detection_roi(const GrayFrame& frame, double roi_margin) {
    stabgpu_roi r{};
    check(stabgpu_detection_roi(frame.width, frame.height, roi_margin, &r));
    return RoiRect{r.x0, r.y0, r.x1, r.y1};
}

ScalarMap min_eig_response(const GrayFrame& frame, int block_size) {
    validate(frame);
    ScalarMap out(frame.width, frame.height);
    check(stabgpu_min_eig_response(ctx(), frame.pixels.data(), frame.width, frame.height, block_size,
                                   out.values.data()));
    return out;
}

std::vector<Corner> detect_corners(const GrayFrame& frame, const DetectConfig& cfg) {
    validate(frame);
    validate(cfg);
    const stabgpu_detect_cfg c = to_c(cfg);
    std::vector<double> xy(2 * static_cast<size_t>(cfg.max_corners)), sc(cfg.max_corners);
    int n = 0;
    check(stabgpu_detect_corners(ctx(), frame.pixels.data(), frame.width, frame.height, &c, xy.data(),
                                 sc.data(), &n));
    std::vector<Corner> out(n);
    for (int i = 0; i < n; ++i) out[i] = Corner{Point2{xy[2 * i], xy[2 * i + 1]}, sc[i]};
    return out;
}

// ----------------------------------------------------------------- flow
void validate(const FlowConfig& cfg) {  // flow.cpp:10-21
    if (cfg.window_radius < 1 || cfg.max_levels < 1 || cfg.max_iterations < 1 || cfg.epsilon <= 0.0 ||
        cfg.fb_threshold <= 0.0)
        throw InvalidConfigError("flow parameters must be positive");
    if (cfg.redetect_interval < 1) throw InvalidConfigError("redetect_interval must be >= 1");
    if (cfg.min_tracks < 4) throw InvalidConfigError("min_tracks must be >= 4");
}

std::vector<TrackedPoint> track_lk(const Pyramid& prev, const Pyramid& cur,
                                   std::span<const Point2> points, const FlowConfig& cfg) {
    validate(cfg);
    const PackedPyramid a(prev), b(cur);
    const stabgpu_flow_cfg c = to_c(cfg);
    const std::vector<double> in = flat(points);
    std::vector<double> out(in.size());
    std::vector<uint8_t> ok(points.size());
    check(stabgpu_track_lk(ctx(), &a.c, &b.c, in.data(), static_cast<int>(points.size()), &c, out.data(),
                           ok.data()));
    std::vector<TrackedPoint> res(points.size());
    for (size_t i = 0; i < points.size(); ++i)
        res[i] = TrackedPoint{Point2{out[2 * i], out[2 * i + 1]}, ok[i] != 0};
    return res;
}

TrackSet weed_tracks(const Pyramid& prev, const Pyramid& cur, std::span<const Point2> prev_points,
                     std::span<const Point2> cur_points, const FlowConfig& cfg) {
    if (prev_points.size() != cur_points.size())
        throw InvalidInputError("prev/cur point lists must be index-aligned");
    TrackSet set;
    set.frame_index = cur.index();
    if (prev_points.empty()) return set;
    const PackedPyramid a(prev), b(cur);
    const stabgpu_flow_cfg c = to_c(cfg);
    const std::vector<double> p = flat(prev_points), q = flat(cur_points);
    std::vector<double> kp(p.size()), kc(q.size());
    int m = 0;
    check(stabgpu_weed_tracks(ctx(), &a.c, &b.c, p.data(), q.data(), static_cast<int>(prev_points.size()),
                              &c, kp.data(), kc.data(), &m));
    for (int i = 0; i < m; ++i) {
        set.prev_points.push_back(Point2{kp[2 * i], kp[2 * i + 1]});
        set.cur_points.push_back(Point2{kc[2 * i], kc[2 * i + 1]});
    }
    return set;
}

}  // namespace stab

namespace {
// Device state of each Tracker (flow.hpp:74-82 fixes its private members, so
// it lives beside them, keyed by the object's address): the previous
// pyramid and the carried points stay on the B200 between advance() calls
// (stabgpu_tracker_*); the private members keep the host bookkeeping
// (last_index_, since_detect_, detections_run_, the size of points_).
struct DevTracker {
    stabgpu_ctx* c = nullptr;  // its own context: outlives the creating thread's context
    stabgpu_tracker* t = nullptr;
    int w = 0, h = 0;
    ~DevTracker() {
        if (t) stabgpu_tracker_destroy(t);
        if (c) stabgpu_destroy(c);
    }
};
std::mutex g_trk_mu;
std::unordered_map<const stab::Tracker*, std::unique_ptr<DevTracker>>& trackers() {
    static auto* m = new std::unordered_map<const stab::Tracker*, std::unique_ptr<DevTracker>>();  // outlives statics
    return *m;
}
}  // namespace

namespace stab {

// Tracker: re-detect cadence and point carrying (flow.cpp:282-337 semantics),
// with the pyramids and points on the device.
Tracker::Tracker(FlowConfig flow_cfg, DetectConfig detect_cfg) : flow_(flow_cfg), detect_(detect_cfg) {
    validate(flow_);
    validate(detect_);
    if (flow_.window_radius > 31) throw InvalidConfigError("window_radius above 31 is not supported");
    std::lock_guard<std::mutex> g(g_trk_mu);
    trackers().erase(this);  // a new object at a recycled address starts fresh
}

void Tracker::detect_fresh(const GrayFrame& frame) {
    points_.clear();
    for (const Corner& c : detect_corners(frame, detect_)) points_.push_back(c.position);
    since_detect_ = 0;
    ++detections_run_;
}

Tracker::Advance Tracker::advance(const GrayFrame& cur) {
    validate(cur);
    if (cur.index <= last_index_) throw SequencingError("frame index must be strictly increasing");
    DevTracker* dt;
    {
        std::lock_guard<std::mutex> g(g_trk_mu);
        auto& slot = trackers()[this];
        if (!slot) {
            if (prev_) throw Error("stabgpu: a copied or moved Tracker cannot continue a sequence (device state stays with the original)");
            slot = std::make_unique<DevTracker>();
        }
        dt = slot.get();
    }
    if (!dt->t) {
        const stabgpu_flow_cfg fc = to_c(flow_);
        const stabgpu_detect_cfg dc = to_c(detect_);
        if (!dt->c) check(stabgpu_create(0, &dt->c));
        check(stabgpu_tracker_create(dt->c, &fc, &dc, cur.width, cur.height, &dt->t));
        dt->w = cur.width;
        dt->h = cur.height;
    } else if (cur.width != dt->w || cur.height != dt->h) {
        throw InvalidInputError("pyramid levels differ in size");  // check_pyramids (flow.cpp:229-239)
    }
    last_index_ = cur.index;
    std::vector<double> p(2 * static_cast<size_t>(detect_.max_corners)), q(p.size());
    int kind = 0, n = 0, active = 0;
    check(stabgpu_tracker_advance(dt->t, cur.pixels.data(), cur.index, &kind, p.data(), q.data(), &n, &active));
    const bool first = !prev_;
    if (first) {
        ++detections_run_;
        since_detect_ = 0;
        prev_ = Pyramid{};  // marks "a previous frame exists"; its levels live on the device
    } else if (++since_detect_ >= flow_.redetect_interval) {
        since_detect_ = 0;
        ++detections_run_;
    }
    points_.assign(static_cast<size_t>(active), Point2{});  // active_point_count(); positions on the device
    if (first) return {Advance::Kind::FirstFrame, {}};
    TrackSet tracks;
    tracks.frame_index = cur.index;
    tracks.prev_points.resize(n);
    tracks.cur_points.resize(n);
    for (int i = 0; i < n; ++i) {
        tracks.prev_points[i] = Point2{p[2 * i], p[2 * i + 1]};
        tracks.cur_points[i] = Point2{q[2 * i], q[2 * i + 1]};
    }
    if (kind == STABGPU_FRAME_SKIPPED) return {Advance::Kind::Skipped, {}};
    return {Advance::Kind::Tracked, std::move(tracks)};
}

// --------------------------------------------------------------- motion
namespace {
SimilarityTransform fit(const TrackSet& ts, int kind) {
    const std::vector<double> p = flat(ts.prev_points), q = flat(ts.cur_points);
    stabgpu_transform t{};
    check(stabgpu_estimate(ctx(), p.data(), q.data(), static_cast<int>(ts.size()), kind, &t));
    return from_c(t);
}
}  // namespace

SimilarityTransform estimate_similarity(const TrackSet& tracks) { return fit(tracks, STABGPU_SIMILARITY); }
SimilarityTransform estimate_rigid(const TrackSet& tracks) { return fit(tracks, STABGPU_RIGID); }

double rms_residual(const TrackSet& tracks, const SimilarityTransform& t) {
    if (tracks.empty()) throw DegenerateInputError("rms_residual needs a non-empty track set");
    const std::vector<double> p = flat(tracks.prev_points), q = flat(tracks.cur_points);
    const stabgpu_transform c = to_c(t);
    double out = 0.0;
    check(stabgpu_rms_residual(ctx(), p.data(), q.data(), static_cast<int>(tracks.size()), &c, &out));
    return out;
}

DeltaParams extract_delta(const SimilarityTransform& t) {
    const stabgpu_transform c = to_c(t);
    stabgpu_delta d{};
    stabgpu_extract_delta(&c, &d);
    DeltaParams out;
    out.dx = d.dx;
    out.dy = d.dy;
    out.da = d.da;
    out.dls = d.dls;
    out.kind = t.kind;
    out.skipped = false;
    return out;
}

SimilarityTransform delta_to_transform(double dx, double dy, double da, double dls) {
    stabgpu_transform t{};
    stabgpu_delta_to_transform(dx, dy, da, dls, &t);
    return from_c(t);
}

void validate(const SelectorConfig& cfg) {  // motion.cpp:113-120
    if (cfg.dwell < 1) throw InvalidConfigError("dwell must be >= 1");
    if (cfg.margin < 0.0) throw InvalidConfigError("margin must be >= 0");
}

ModelSelector::ModelSelector(SelectorConfig cfg) : cfg_(cfg) {
    validate(cfg_);
    if (cfg_.mode == SelectionMode::ForceSimilarity) current_ = ModelKind::Similarity;
}

void ModelSelector::advance_counter() { frames_since_decision_ = (frames_since_decision_ + 1) % cfg_.dwell; }

void ModelSelector::record_decision(ModelKind kind) {
    current_ = kind;
    (kind == ModelKind::Rigid ? rigid_decisions_ : similarity_decisions_) += 1;
    pending_decision_ = false;
}

// Decision frames fit both models and compare RMS with the margin; other
// frames fit the current model (motion.cpp:143-184 semantics).
SimilarityTransform ModelSelector::select(const TrackSet& tracks) {
    if (frames_since_decision_ == 0) pending_decision_ = true;
    SimilarityTransform out;
    if (cfg_.mode != SelectionMode::Hybrid) {
        const bool rigid = cfg_.mode == SelectionMode::ForceRigid;
        out = rigid ? estimate_rigid(tracks) : estimate_similarity(tracks);
        ++estimation_calls_;
        if (pending_decision_) record_decision(rigid ? ModelKind::Rigid : ModelKind::Similarity);
    } else if (pending_decision_) {
        const SimilarityTransform r = estimate_rigid(tracks), s = estimate_similarity(tracks);
        estimation_calls_ += 2;
        const bool rigid = rms_residual(tracks, r) <= rms_residual(tracks, s) * (1.0 + cfg_.margin);
        record_decision(rigid ? ModelKind::Rigid : ModelKind::Similarity);
        out = rigid ? r : s;
    } else {
        out = current_ == ModelKind::Rigid ? estimate_rigid(tracks) : estimate_similarity(tracks);
        ++estimation_calls_;
    }
    advance_counter();
    return out;
}

void ModelSelector::note_skipped() {
    if (frames_since_decision_ == 0) pending_decision_ = true;
    advance_counter();
}

// ------------------------------------------------------------ smoothing
void validate(const SmoothConfig& cfg) {
    if (cfg.radius < 1) throw InvalidConfigError("smoothing radius must be >= 1");
}

void Trajectory::append(const DeltaParams& d) {
    Params4 c = cumulative_.empty() ? Params4{} : cumulative_.back();
    c.x += d.dx;
    c.y += d.dy;
    c.a += d.da;
    c.ls += d.dls;
    deltas_.push_back(d);
    cumulative_.push_back(c);
}

std::optional<Params4> Trajectory::smooth_at(std::size_t i, const SmoothConfig& cfg) const {
    validate(cfg);
    if (i >= size()) throw InvalidInputError("smooth_at index past the trajectory");
    const std::size_t r = static_cast<std::size_t>(cfg.radius);
    if (!complete_ && i + r >= size()) return std::nullopt;
    const std::size_t lo = i >= r ? i - r : 0, hi = std::min(i + r, size() - 1);
    Params4 s;
    for (std::size_t j = lo; j <= hi; ++j) {
        s.x += cumulative_[j].x;
        s.y += cumulative_[j].y;
        s.a += cumulative_[j].a;
        s.ls += cumulative_[j].ls;
    }
    const double n = static_cast<double>(hi - lo + 1);
    return Params4{s.x / n, s.y / n, s.a / n, s.ls / n};
}

std::optional<SimilarityTransform> Trajectory::correction(std::size_t i, const SmoothConfig& cfg) const {
    const std::optional<Params4> sm = smooth_at(i, cfg);
    if (!sm) return std::nullopt;
    const Params4& c = cumulative_[i];
    return delta_to_transform(sm->x - c.x, sm->y - c.y, sm->a - c.a, sm->ls - c.ls);
}

}  // namespace stab
