// k_plan.cu — K7: model-selection scan, trajectory prefix and moving-average
// smoothing, on the device.
//
// Reference: ModelSelector::select / note_skipped (motion.cpp:143-191),
// MotionStage::step (pipeline.cpp:80-101), Trajectory::append (smoothing.cpp:
// 16-24), smooth_at (26-46), correction (48-57), delta_to_transform
// (motion.cpp:103-111).
//
// The selector and the running sum are sequential recurrences and are
// evaluated sequentially (one thread, reference order), which keeps the
// cumulative path bit-identical to the reference; the scan is incremental so
// a streaming caller can feed motion records chunk by chunk.  Each smoothed
// value is an independent window mean, one thread per frame, summed in the
// reference's ascending order.
#include "common.cuh"
#include "kernels.cuh"

namespace stabgpu {

namespace {

__global__ void plan_scan_kernel(const stabgpu_motion_record* __restrict__ motion, long long first,
                                 long long count, stabgpu_selector_cfg sel, PlanState* st,
                                 stabgpu_frame_record* __restrict__ rec, double4* __restrict__ cum,
                                 int* __restrict__ err, long long stride) {
    // The recurrence runs on lane 0; the whole warp stages the next 32 motion
    // records in shared memory first (one record per lane, loads in flight
    // together), so lane 0 never waits on a dependent global load per frame.
    constexpr int RW = sizeof(stabgpu_motion_record) / 8;  // 15 eight-byte words
    __shared__ unsigned long long buf[32][RW];
    __shared__ int finfo[32];
    __shared__ double4 fcum[32];
    const int lane = threadIdx.x & 31;
    // one block per independent stream
    motion += blockIdx.x * stride;
    rec += blockIdx.x * stride;
    cum += blockIdx.x * stride;
    st += blockIdx.x;
    err += blockIdx.x;
    PlanState s = *st;
    for (long long f0 = first; f0 < first + count; f0 += 32) {
        const long long nf = min(32LL, first + count - f0);
        if (lane < nf) {
            const unsigned long long* src = reinterpret_cast<const unsigned long long*>(motion + f0 + lane);
            unsigned long long v[RW];
#pragma unroll
            for (int k = 0; k < RW; ++k) v[k] = src[k];
#pragma unroll
            for (int k = 0; k < RW; ++k) buf[lane][k] = v[k];
        }
        __syncwarp();
        // lane 0: the recurrences only (selector state, trajectory prefix) in
        // reference order; the frame records are assembled by all lanes after
        if (lane == 0) {
            for (long long f = f0; f < f0 + nf; ++f) {
                const int j = (int)(f - f0);
                const stabgpu_motion_record& m = *reinterpret_cast<const stabgpu_motion_record*>(buf[j]);
                int info;  // bit 0: tracked, bit 1: rigid delta, bit 2: decision, bits 8+: kind of a zero delta
                double dx = 0.0, dy = 0.0, da = 0.0, dls = 0.0;
                if (m.frame_kind != STABGPU_FRAME_TRACKED) {
                    // note_skipped (motion.cpp:185-191)
                    if (s.since == 0) s.pending = 1;
                    s.since = s.since + 1 == sel.dwell ? 0 : s.since + 1;
                    info = s.current << 8;
                } else {
                    if (s.since == 0) s.pending = 1;
                    const int st_r = m.status & 0xff, st_s = (m.status >> 8) & 0xff;
                    int use_rigid, decision = 0;
                    if (sel.mode == STABGPU_FORCE_RIGID || sel.mode == STABGPU_FORCE_SIMILARITY) {
                        use_rigid = sel.mode == STABGPU_FORCE_RIGID;
                        if (s.pending) {
                            s.current = use_rigid ? STABGPU_RIGID : STABGPU_SIMILARITY;
                            s.pending = 0;
                            decision = 1;
                        }
                        const int e = use_rigid ? st_r : st_s;
                        if (e && *err == 0) *err = e | (int)(f << 4);
                    } else if (s.pending) {
                        if ((st_r || st_s) && *err == 0) *err = (st_r ? st_r : st_s) | (int)(f << 4);
                        use_rigid = m.e_rigid <= dmul(m.e_similarity, dadd(1.0, sel.margin));
                        s.current = use_rigid ? STABGPU_RIGID : STABGPU_SIMILARITY;
                        s.pending = 0;
                        decision = 1;
                    } else {
                        use_rigid = s.current == STABGPU_RIGID;
                        const int e = use_rigid ? st_r : st_s;
                        if (e && *err == 0) *err = e | (int)(f << 4);
                    }
                    s.since = s.since + 1 == sel.dwell ? 0 : s.since + 1;
                    const stabgpu_delta& d = use_rigid ? m.rigid : m.similarity;
                    dx = d.dx;
                    dy = d.dy;
                    da = d.da;
                    dls = d.dls;
                    info = 1 | (use_rigid << 1) | (decision << 2);
                }
                // Trajectory::append (smoothing.cpp:16-24)
                s.cum[0] = dadd(s.cum[0], dx);
                s.cum[1] = dadd(s.cum[1], dy);
                s.cum[2] = dadd(s.cum[2], da);
                s.cum[3] = dadd(s.cum[3], dls);
                finfo[j] = info;
                fcum[j] = make_double4(s.cum[0], s.cum[1], s.cum[2], s.cum[3]);
            }
        }
        __syncwarp();
        if (lane < nf) {  // frame record f0 + lane
            const stabgpu_motion_record& m = *reinterpret_cast<const stabgpu_motion_record*>(buf[lane]);
            const int info = finfo[lane];
            stabgpu_frame_record r;
            memset(&r, 0, sizeof r);
            r.frame_kind = m.frame_kind;
            r.n_tracks = m.n_tracks;
            if (info & 1) {
                const bool rigid = info & 2;
                r.delta = rigid ? m.rigid : m.similarity;
                r.delta.skipped = 0;
                r.n_inliers = rigid ? m.n_inliers_rigid : m.n_inliers_similarity;
                r.decision = (info >> 2) & 1;
            } else {
                r.delta = stabgpu_delta{0.0, 0.0, 0.0, 0.0, info >> 8, m.frame_kind == STABGPU_FRAME_SKIPPED};
            }
            rec[f0 + lane] = r;
            cum[f0 + lane] = fcum[lane];
        }
        __syncwarp();
    }
    if (lane == 0) {
        s.scanned = first + count;
        *st = s;
    }
}

__global__ void plan_smooth_kernel(const double4* __restrict__ cum, long long n_known,
                                   long long first, long long count, int radius,
                                   stabgpu_frame_record* __restrict__ rec, FramePlan* __restrict__ plan,
                                   PlanGeom geo, long long sf) {
    const long long i = first + blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= first + count) return;
    // window clipped to the frame's own stream (sf frames per stream, n_known each)
    const long long base = sf ? i - i % sf : 0;
    const long long lo = i - base >= radius ? i - radius : base;
    const long long hi = min(i + radius, base + n_known - 1);
    double sx = 0.0, sy = 0.0, sa = 0.0, sl = 0.0;
    for (long long j = lo; j <= hi; ++j) {
        const double4 c = cum[j];
        sx = dadd(sx, c.x);
        sy = dadd(sy, c.y);
        sa = dadd(sa, c.z);
        sl = dadd(sl, c.w);
    }
    const double n = (double)(hi - lo + 1);
    const double4 ci = cum[i];
    FramePlan p;
    p.tx = dsub(ddiv(sx, n), ci.x);
    p.ty = dsub(ddiv(sy, n), ci.y);
    p.theta = dsub(ddiv(sa, n), ci.z);
    p.s = exp(dsub(ddiv(sl, n), ci.w));
    // warp_similarity / apply_inverse coefficients (image_ops.cpp:121-122, transform.cpp:14-15)
    p.c = ddiv(cos(p.theta), p.s);
    p.sn = ddiv(sin(p.theta), p.s);
    finish_plan(p, geo.w, geo.h, geo.cw, geo.ch, geo.crop);
    plan[i] = p;
    stabgpu_transform t{p.tx, p.ty, p.theta, p.s, STABGPU_SIMILARITY};
    rec[i].correction = t;
}

}  // namespace

void launch_plan_scan(const stabgpu_motion_record* motion, long long first, long long count,
                      const stabgpu_config& cfg, PlanState* state, stabgpu_frame_record* rec,
                      double4* cum, cudaStream_t st, int n_streams, long long stream_stride, int* err) {
    if (count <= 0 || n_streams <= 0) return;
    // default error word: right after the state
    plan_scan_kernel<<<n_streams, 32, 0, st>>>(motion, first, count, cfg.selector, state, rec, cum,
                                               err ? err : reinterpret_cast<int*>(state + 1), stream_stride);
}

void launch_plan_smooth(const double4* cum, long long n_known, bool complete, long long first,
                        long long count, int radius, stabgpu_frame_record* rec, FramePlan* plan,
                        PlanGeom geo, cudaStream_t st, long long stream_frames) {
    (void)complete;
    if (count <= 0) return;
    const int tpb = 128;
    plan_smooth_kernel<<<(unsigned)((count + tpb - 1) / tpb), tpb, 0, st>>>(cum, n_known, first, count,
                                                                           radius, rec, plan, geo,
                                                                           stream_frames);
}

}  // namespace stabgpu

namespace stabgpu {
namespace {
__global__ void prefix_kernel(const stabgpu_delta* __restrict__ d, long long n, double4* __restrict__ cum) {
    if (threadIdx.x != 0) return;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    for (long long i = 0; i < n; ++i) {
        c0 = dadd(c0, d[i].dx);
        c1 = dadd(c1, d[i].dy);
        c2 = dadd(c2, d[i].da);
        c3 = dadd(c3, d[i].dls);
        cum[i] = make_double4(c0, c1, c2, c3);
    }
}

__global__ void plan_from_corr_kernel(const stabgpu_transform* __restrict__ t, long long n,
                                      FramePlan* __restrict__ plan, PlanGeom geo) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    FramePlan p;
    p.tx = t[i].tx;
    p.ty = t[i].ty;
    p.theta = t[i].theta;
    p.s = t[i].s;
    p.c = ddiv(cos(p.theta), p.s);
    p.sn = ddiv(sin(p.theta), p.s);
    finish_plan(p, geo.w, geo.h, geo.cw, geo.ch, geo.crop);
    plan[i] = p;
}
}  // namespace

void launch_prefix(const stabgpu_delta* d, long long n, double4* cum, cudaStream_t st) {
    if (n > 0) prefix_kernel<<<1, 32, 0, st>>>(d, n, cum);
}

void launch_plan_from_corrections(const stabgpu_transform* corr, long long n, FramePlan* plan,
                                  PlanGeom geo, cudaStream_t st) {
    if (n > 0) plan_from_corr_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(corr, n, plan, geo);
}
}  // namespace stabgpu
