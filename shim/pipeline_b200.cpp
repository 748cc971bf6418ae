// pipeline_b200.cpp — run_offline / run_streaming (pipeline.hpp:68-76) of the
// drop-in, on the device: the frames pulled from the FrameSource go through
// one Stage II stream object (stabgpu_stream_*: K1, the K5 step, K6, the K7
// scan, and for each released frame the smoothing + K8 compose, one CUDA
// graph per push), and the released frames go to the FrameSink in arrival
// order.  Semantics of pipeline.cpp:182-365 kept:
//   * validation (pipeline.cpp:17-28) with the same exception classes;
//   * the CompensationPlanner release rule (nothing before 2r estimates
//     unless the stream ended, then every frame whose window is complete),
//     so frames, first_emit_me_frames and latency_frames are the reference's
//     and run_offline / run_streaming outputs are bit-identical to each other
//     and to the reference's;
//   * decision / skipped counts and the optional trajectory export from the
//     per-frame records;
//   * errors: run_offline lets them propagate; run_streaming reports the
//     first one to sink.abort() before rethrowing it (pipeline.cpp:343-352);
//     fewer than 2 frames throws InvalidInputError without abort.
// run_streaming needs no threads of its own here: the device pipelines the
// stages (uploads, compute and downloads on separate CUDA streams).
//
// To use it, compile the reference's pipeline.cpp with
// -Drun_offline=reference_run_offline -Drun_streaming=reference_run_streaming
// (its other definitions — validate, summarize, to_json — stay) and link
// libstabcore_b200.so; INTEGRATION.md §1.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <exception>
#include <string>
#include <vector>

#include "../include/stabgpu.h"
#include "stab/pipeline.hpp"

namespace {

using Clock = std::chrono::steady_clock;

double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

[[noreturn]] void raise_rc(int rc) {
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

void ok(int rc) {
    if (rc != STABGPU_OK) raise_rc(rc);
}

stabgpu_config to_c(const stab::StabConfig& cfg) {
    stabgpu_config c;
    stabgpu_default_config(&c);
    c.detect = {cfg.detect.max_corners, cfg.detect.quality_level, cfg.detect.min_distance, cfg.detect.block_size,
                cfg.detect.roi_margin};
    c.flow = {cfg.flow.window_radius, cfg.flow.max_levels, cfg.flow.max_iterations, cfg.flow.epsilon,
              cfg.flow.fb_threshold, cfg.flow.redetect_interval, cfg.flow.min_tracks};
    c.smooth_radius = cfg.smooth.radius;
    c.selector.dwell = cfg.selector.dwell;
    c.selector.margin = cfg.selector.margin;
    c.selector.mode = cfg.selector.mode == stab::SelectionMode::ForceRigid        ? STABGPU_FORCE_RIGID
                      : cfg.selector.mode == stab::SelectionMode::ForceSimilarity ? STABGPU_FORCE_SIMILARITY
                                                                                   : STABGPU_HYBRID;
    c.ransac = {0, 3.0, 0};  // the reference has no RANSAC
    c.crop_ratio = cfg.crop_ratio;
    c.queue_capacity = cfg.queue_capacity;
    return c;
}

struct Stream {
    stabgpu_ctx* ctx = nullptr;
    stabgpu_stream* s = nullptr;
    uint8_t* stage_in = nullptr;   // page-locked planar frames (Y | Cb | Cr): kIn upload slots
    uint8_t* stage_out = nullptr;  // and kOut download slots
    ~Stream() {
        if (s) stabgpu_stream_destroy(s);
        if (stage_in) stabgpu_host_free(stage_in);
        if (stage_out) stabgpu_host_free(stage_out);
        if (ctx) stabgpu_destroy(ctx);
    }
};
constexpr int kIn = 3, kOut = 8;  // staging slots: uploads in flight, downloads queued per wait

// One pass of the device pipeline; errors propagate (the caller decides on
// sink.abort).  Phase 1 consumes the source; `finish` releases the tail.
class DeviceRun {
  public:
    DeviceRun(const stab::StabConfig& cfg, stab::FrameSink& sink) : cfg_(cfg), c_(to_c(cfg)), sink_(sink) {}

    void consume(stab::FrameSource& source) {
        while (std::optional<stab::VideoFrame> f = source.next()) {
            ++frames_;
            push(*f);
        }
    }

    bool enough() const { return frames_ >= 2; }

    void finish() {
        deliver();
        int n = 0;
        const auto t0 = Clock::now();
        ok(stabgpu_stream_wait_inputs(st_.s));
        ok(stabgpu_stream_finish(st_.s, &n));
        me_s_ += since(t0);
        if (n > 0 && first_emit_ < 0) first_emit_ = frames_;
        while (n > 0) {  // the tail, kOut frames per wait
            const int m = std::min(n, kOut);
            queue_pops(m);
            deliver();
            n -= m;
        }
    }

    stab::RunSummary summary(Clock::time_point start) const {
        stab::RunSummary s;  // summarize() (pipeline.cpp:30-50)
        const auto fps = [&](double sec) { return sec > 0.0 ? static_cast<double>(frames_) / sec : 0.0; };
        s.frames = frames_;
        s.wall_seconds = since(start);
        s.me_seconds = me_s_;
        s.mc_seconds = 0.0;  // selector, trajectory and release run inside the device pipeline
        s.ic_seconds = ic_s_;
        s.fps_overall = fps(s.wall_seconds);
        s.fps_me = fps(s.me_seconds);
        s.fps_mc = 0.0;
        s.fps_ic = fps(s.ic_seconds);
        s.rigid_decisions = rigid_;
        s.similarity_decisions = similarity_;
        s.skipped_frames = skipped_;
        s.latency_frames = cfg_.smooth.radius;
        s.first_emit_me_frames = first_emit_;
        return s;
    }

    void export_trajectory(stab::Trajectory* out) const {
        if (!out) return;
        stab::Trajectory t;
        for (const stab::DeltaParams& d : deltas_) t.append(d);
        t.mark_complete();
        *out = std::move(t);
    }

  private:
    const stab::StabConfig& cfg_;
    stabgpu_config c_;
    stab::FrameSink& sink_;
    Stream st_;
    int w_ = 0, h_ = 0, cw_ = 0, ch_ = 0;
    std::int64_t last_index_ = -1, frames_ = 0, first_emit_ = -1;
    std::int64_t rigid_ = 0, similarity_ = 0, skipped_ = 0;
    double me_s_ = 0.0, ic_s_ = 0.0;
    std::deque<std::int64_t> pending_;  // indices of frames not yet released
    std::size_t fl_ = 0, fc_ = 0, fs_ = 0;  // luma / chroma plane bytes, bytes per staged frame
    int queued_ = 0;                        // pops issued into stage_out slots 0..queued_-1, not yet delivered
    stabgpu_frame_record recs_[kOut];
    int64_t idx_[kOut];
    std::vector<stab::DeltaParams> deltas_;

    void push(const stab::VideoFrame& f) {
        const stab::GrayFrame& y = f.luma;
        if (y.width <= 0 || y.height <= 0 || y.pixels.size() != static_cast<std::size_t>(y.width) * y.height)
            throw stab::InvalidInputError("frame dimensions do not match the pixel buffer");
        const bool col = f.has_chroma();
        if (!st_.s) {
            w_ = y.width;
            h_ = y.height;
            cw_ = col ? f.chroma_width : 0;
            ch_ = col ? f.chroma_height : 0;
            ok(stabgpu_create(0, &st_.ctx));
            ok(stabgpu_stream_create(st_.ctx, &c_, w_, h_, cw_, ch_, &st_.s));
            fl_ = static_cast<std::size_t>(w_) * h_;
            fc_ = static_cast<std::size_t>(cw_) * ch_;
            fs_ = fl_ + 2 * fc_;
            void* p = nullptr;
            ok(stabgpu_host_alloc(&p, fs_ * kIn));
            st_.stage_in = static_cast<uint8_t*>(p);
            ok(stabgpu_host_alloc(&p, fs_ * kOut));
            st_.stage_out = static_cast<uint8_t*>(p);
            if (const char* g = std::getenv("STABGPU_STREAM_GRAPHS")) ok(stabgpu_stream_set_graphs(st_.s, std::atoi(g)));
        } else if (y.width != w_ || y.height != h_ || (col ? f.chroma_width : 0) != cw_ ||
                   (col ? f.chroma_height : 0) != ch_) {
            throw stab::InvalidInputError("frame size changed mid-stream");
        }
        if (col && (f.cb.size() != static_cast<std::size_t>(cw_) * ch_ || f.cr.size() != f.cb.size()))
            throw stab::InvalidInputError("chroma planes do not match the chroma size");
        if (y.index <= last_index_) throw stab::SequencingError("frame index must be strictly increasing");
        last_index_ = y.index;
        // The caller's frames are std::vectors (pageable).  Frame k is copied
        // into a page-locked planar slot and pushed without waiting for its
        // upload; released frames are downloaded into page-locked slots a few
        // pushes after their release (their compose finished long before, so
        // the copy only waits for PCIe) and handed to the sink one push later.
        // The device therefore runs ahead of the host: the next frames' motion
        // and the re-detections overlap the copies.  Order and bytes are those
        // of popping at once; finish() drains.
        deliver();  // the downloads queued by the previous push
        int n = 0;
        const auto t0 = Clock::now();
        if (frames_ > kIn - 1 && (frames_ - 1) % (kIn - 1) == 0)
            ok(stabgpu_stream_wait_inputs(st_.s));  // the slot written next was uploaded at least one wait ago
        uint8_t* in = st_.stage_in + static_cast<std::size_t>((frames_ - 1) % kIn) * fs_;
        std::memcpy(in, y.pixels.data(), fl_);
        if (col) {
            std::memcpy(in + fl_, f.cb.data(), fc_);
            std::memcpy(in + fl_ + fc_, f.cr.data(), fc_);
        }
        ok(stabgpu_stream_push_async(st_.s, in, col ? in + fl_ : nullptr, col ? in + fl_ + fc_ : nullptr, &n));
        me_s_ += since(t0);
        pending_.push_back(y.index);
        if (n > 0 && first_emit_ < 0) first_emit_ = frames_;  // the release schedule is the device's, not the pop's
        const int lag = std::min(6, std::max(0, 2 * cfg_.smooth.radius - 2));
        queue_pops(std::min(kOut, std::max(0, n - lag)));
    }

    // downloads of the next m released frames into the staging slots
    void queue_pops(int m) {
        const auto t0 = Clock::now();
        for (int k = 0; k < m; ++k) {
            uint8_t* o = st_.stage_out + static_cast<std::size_t>(k) * fs_;
            ok(stabgpu_stream_pop_async(st_.s, &idx_[k], o, cw_ ? o + fl_ : nullptr, cw_ ? o + fl_ + fc_ : nullptr,
                                        &recs_[k]));
        }
        queued_ = m;
        ic_s_ += since(t0);
    }

    // hands the queued frames to the sink (after their downloads have landed)
    void deliver() {
        if (queued_ == 0) return;
        const auto t0 = Clock::now();
        ok(stabgpu_stream_wait_pops(st_.s));
        for (int k = 0; k < queued_; ++k) {
            const uint8_t* o = st_.stage_out + static_cast<std::size_t>(k) * fs_;
            stab::VideoFrame out;
            out.luma.width = w_;
            out.luma.height = h_;
            out.luma.index = pending_.front();
            out.luma.pixels.assign(o, o + fl_);
            pending_.pop_front();
            if (cw_ > 0) {
                out.chroma_width = cw_;
                out.chroma_height = ch_;
                out.cb.assign(o + fl_, o + fl_ + fc_);
                out.cr.assign(o + fl_ + fc_, o + fs_);
            }
            const stabgpu_frame_record& rec = recs_[k];
            stab::DeltaParams d;
            d.dx = rec.delta.dx;
            d.dy = rec.delta.dy;
            d.da = rec.delta.da;
            d.dls = rec.delta.dls;
            d.kind = rec.delta.kind == STABGPU_RIGID ? stab::ModelKind::Rigid : stab::ModelKind::Similarity;
            d.skipped = rec.delta.skipped != 0;
            deltas_.push_back(d);
            if (rec.decision) (rec.delta.kind == STABGPU_RIGID ? rigid_ : similarity_) += 1;
            if (rec.frame_kind == STABGPU_FRAME_SKIPPED) ++skipped_;
            sink_.push(std::move(out));
        }
        queued_ = 0;
        ic_s_ += since(t0);
    }
};

void validate_cfg(const stab::StabConfig& cfg) {  // pipeline.cpp:17-28
    stab::validate(cfg.detect);
    stab::validate(cfg.flow);
    stab::validate(cfg.smooth);
    stab::validate(cfg.selector);
    if (!(cfg.crop_ratio >= 0.0 && cfg.crop_ratio < 0.25))
        throw stab::InvalidConfigError("crop_ratio must lie in [0, 0.25)");
    if (cfg.queue_capacity < 2 * static_cast<std::size_t>(cfg.smooth.radius) + 4)
        throw stab::InvalidConfigError("queue_capacity must be >= 2*radius + 4");
}

void abort_with(stab::FrameSink& sink, std::exception_ptr e) {
    try {
        std::rethrow_exception(e);
    } catch (const std::exception& ex) {
        sink.abort(ex.what());
    } catch (...) {
        sink.abort("unknown pipeline error");
    }
}

}  // namespace

namespace stab {

RunSummary run_offline(FrameSource& source, const StabConfig& cfg, FrameSink& sink, Trajectory* trajectory_out) {
    validate_cfg(cfg);
    const auto start = Clock::now();
    DeviceRun run(cfg, sink);
    run.consume(source);
    if (!run.enough()) throw InvalidInputError("stabilization needs at least 2 frames");
    run.finish();
    sink.close();
    run.export_trajectory(trajectory_out);
    return run.summary(start);
}

RunSummary run_streaming(FrameSource& source, const StabConfig& cfg, FrameSink& sink, Trajectory* trajectory_out) {
    validate_cfg(cfg);
    const auto start = Clock::now();
    DeviceRun run(cfg, sink);
    try {
        run.consume(source);
        if (run.enough()) run.finish();
    } catch (...) {
        const std::exception_ptr e = std::current_exception();
        abort_with(sink, e);
        std::rethrow_exception(e);
    }
    if (!run.enough()) throw InvalidInputError("stabilization needs at least 2 frames");
    sink.close();
    run.export_trajectory(trajectory_out);
    return run.summary(start);
}

}  // namespace stab
