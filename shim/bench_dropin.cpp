// bench_dropin.cpp — throughput of the drop-in's sequence API: stab::run_offline
// on the device (the shim's Stage II stream, pipeline_b200.cpp) against the
// reference's own run_offline loop (pipeline.cpp, renamed
// reference_run_offline) calling the shim's per-stage GPU functions frame by
// frame.  Frames come from the reference's synthetic generator (synth_eval)
// and are pre-rendered; outputs of the two runs are compared byte for byte.
//   bench_dropin [width height frames]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "stab/pipeline.hpp"
#include "stab/synth_eval.hpp"

namespace stab {
RunSummary reference_run_offline(FrameSource& source, const StabConfig& cfg, FrameSink& sink,
                                 Trajectory* trajectory_out);
}

namespace {
class VecSource : public stab::FrameSource {
  public:
    explicit VecSource(const std::vector<stab::VideoFrame>& f) : f_(f) {}
    std::optional<stab::VideoFrame> next() override {
        if (i_ >= f_.size()) return std::nullopt;
        return f_[i_++];
    }

  private:
    const std::vector<stab::VideoFrame>& f_;
    std::size_t i_ = 0;
};
class VecSink : public stab::FrameSink {
  public:
    void push(stab::VideoFrame f) override { frames.push_back(std::move(f)); }
    std::vector<stab::VideoFrame> frames;
};
}  // namespace

int main(int argc, char** argv) {
    const int w = argc > 1 ? std::atoi(argv[1]) : 640, h = argc > 2 ? std::atoi(argv[2]) : 480;
    const int n = argc > 3 ? std::atoi(argv[3]) : 300;
    stab::JitterSpec spec;
    spec.base = stab::make_textured_base(w + 64, h + 64, 99);
    spec.frames = n;
    spec.jitter_std = 3.0;
    spec.angle_std = 0.01;
    spec.seed = 909;
    const stab::SynthSequence seq = stab::generate(spec);
    std::vector<stab::VideoFrame> frames;
    for (int i = 0; i < n; ++i) {
        stab::VideoFrame f = seq.render(i);
        // crop to w x h (the generator renders the base size)
        stab::GrayFrame g(w, h, f.luma.index);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) g.at(x, y) = f.luma.at(x + 32, y + 32);
        stab::VideoFrame o;
        o.luma = std::move(g);
        frames.push_back(std::move(o));
    }
    stab::StabConfig cfg;
    const auto time = [&](auto fn, VecSink& sink) {
        VecSource src(frames);
        const auto t0 = std::chrono::steady_clock::now();
        fn(src, sink);
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    {  // warm-up (context creation, kernel loading)
        VecSink s;
        std::vector<stab::VideoFrame> few(frames.begin(), frames.begin() + std::min(n, 30));
        VecSource src(few);
        stab::run_offline(src, cfg, s);
    }
    VecSink dev, ref;
    stab::RunSummary sd;
    const double td = time([&](stab::FrameSource& s, stab::FrameSink& k) { sd = stab::run_offline(s, cfg, k); }, dev);
    const double tr =
        time([&](stab::FrameSource& s, stab::FrameSink& k) { stab::reference_run_offline(s, cfg, k, nullptr); }, ref);
    bool same = dev.frames.size() == ref.frames.size();
    for (std::size_t i = 0; same && i < dev.frames.size(); ++i) same = dev.frames[i].luma.pixels == ref.frames[i].luma.pixels;
    std::printf("%dx%d, %d frames: run_offline (device stream) %.1f frames/s; reference loop over GPU stages %.1f "
                "frames/s; outputs %s (device run: push %.3f s, pop %.3f s)\n",
                w, h, n, n / td, n / tr, same ? "bit-identical" : "DIFFER", sd.me_seconds, sd.ic_seconds);
    return same ? 0 : 1;
}
