// k_fit.cu — K6 (closed-form rigid/similarity fit) and K6b (RANSAC), one CTA
// per frame pair, batched over every frame of a chunk.
//
// Reference: accumulate/finish (motion.cpp:17-58), estimate_similarity /
// estimate_rigid (62-76), rms_residual (78-90), extract_delta (92-101).
// RANSAC has no reference counterpart; its rule is the one
// restated in oracle/stab_oracle.c (orc_ransac_estimate): counter-based pair
// sampling, a 2-point minimal model with only correctly rounded + - * / sqrt
// in a fixed order, inliers by residual^2 <= thr^2, most inliers wins with
// ties to the lowest hypothesis, fewer than min_tracks inliers falls back to
// all pairs, then the closed-form fit on the inliers.  Hypotheses are scored
// one per warp (lanes stride the pairs, popc-reduced counts), so inlier
// counts are bit-identical to the CPU rule; only the refit's sums are
// reduced in a different (fixed) order.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace stabgpu {

namespace {

constexpr int FIT_THREADS = 512;
constexpr int FIT_WARPS = FIT_THREADS / 32;
// dynamic shared memory above this goes to the in-place (global memory) path
constexpr size_t kFitSmemMax = 200 * 1024;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

struct Model {
    double a, b, tx, ty;
};

__device__ __forceinline__ bool minimal_model(const double2* P, const double2* Q, int i, int j,
                                              bool rigid, Model& m) {
    const double2 pi = P[i], pj = P[j], qi = Q[i], qj = Q[j];
    const double mpx = dmul(0.5, dadd(pi.x, pj.x)), mpy = dmul(0.5, dadd(pi.y, pj.y));
    const double mqx = dmul(0.5, dadd(qi.x, qj.x)), mqy = dmul(0.5, dadd(qi.y, qj.y));
    const double ax = dsub(pj.x, pi.x), ay = dsub(pj.y, pi.y);
    const double bx = dsub(qj.x, qi.x), by = dsub(qj.y, qi.y);
    const double norm = dadd(dmul(ax, ax), dmul(ay, ay));
    if (norm == 0.0) return false;
    double a = ddiv(dadd(dmul(ax, bx), dmul(ay, by)), norm);
    double b = ddiv(dsub(dmul(ax, by), dmul(ay, bx)), norm);
    if (rigid) {
        const double r = dsqrt(dadd(dmul(a, a), dmul(b, b)));
        if (r == 0.0) return false;
        a = ddiv(a, r);
        b = ddiv(b, r);
    }
    m.a = a;
    m.b = b;
    m.tx = dsub(mqx, dsub(dmul(a, mpx), dmul(b, mpy)));
    m.ty = dsub(mqy, dadd(dmul(b, mpx), dmul(a, mpy)));
    return true;
}

__device__ __forceinline__ bool inlier(const Model& m, double2 p, double2 q, double thr2) {
    const double ex = dsub(q.x, dadd(dsub(dmul(m.a, p.x), dmul(m.b, p.y)), m.tx));
    const double ey = dsub(q.y, dadd(dadd(dmul(m.b, p.x), dmul(m.a, p.y)), m.ty));
    return dadd(dmul(ex, ex), dmul(ey, ey)) <= thr2;
}

// Deterministic block sum (fixed tree: strided partials, butterfly, warps in order).
__device__ double block_dsum(double v, double* red) {
    v = warp_dsum(v);
    const int wid = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < FIT_WARPS; ++w) t = dadd(t, red[w]);
    return t;
}

struct FitOut {
    double tx, ty, theta, s;
    int status;
};

// accumulate + estimate_{rigid,similarity} over pairs with mask[k] != 0.
__device__ FitOut estimate(const double2* P, const double2* Q, const uint8_t* mask, int n, int used,
                           bool rigid, double* red) {
    FitOut o{0, 0, 0, 1, STABGPU_OK};
    if (used < 2) {
        o.status = STABGPU_DEGENERATE_INPUT;
        return o;
    }
    double sx = 0, sy = 0, dxs = 0, dys = 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x)
        if (!mask || mask[k]) {
            sx = dadd(sx, P[k].x);
            sy = dadd(sy, P[k].y);
            dxs = dadd(dxs, Q[k].x);
            dys = dadd(dys, Q[k].y);
        }
    const double dn = (double)used;
    const double scx = ddiv(block_dsum(sx, red), dn), scy = ddiv(block_dsum(sy, red), dn);
    const double dcx = ddiv(block_dsum(dxs, red), dn), dcy = ddiv(block_dsum(dys, red), dn);
    double dot = 0, cross = 0, norm = 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x)
        if (!mask || mask[k]) {
            const double x = dsub(P[k].x, scx), y = dsub(P[k].y, scy);
            const double xp = dsub(Q[k].x, dcx), yp = dsub(Q[k].y, dcy);
            dot = dadd(dot, dadd(dmul(x, xp), dmul(y, yp)));
            cross = dadd(cross, dsub(dmul(x, yp), dmul(y, xp)));
            norm = dadd(norm, dadd(dmul(x, x), dmul(y, y)));
        }
    dot = block_dsum(dot, red);
    cross = block_dsum(cross, red);
    norm = block_dsum(norm, red);
    if (norm == 0.0) {
        o.status = STABGPU_DEGENERATE_INPUT;
        return o;
    }
    const double theta = atan2(cross, dot);
    double scale = 1.0;
    if (!rigid) {
        scale = ddiv(dadd(dmul(cos(theta), dot), dmul(sin(theta), cross)), norm);
        if (!(scale > 0.0) || !isfinite(scale)) {
            o.status = STABGPU_DEGENERATE_INPUT;
            return o;
        }
    }
    const double c = dmul(scale, cos(theta)), sn = dmul(scale, sin(theta));
    o.theta = theta;
    o.s = scale;
    o.tx = dsub(dcx, dsub(dmul(c, scx), dmul(sn, scy)));
    o.ty = dsub(dcy, dadd(dmul(sn, scx), dmul(c, scy)));
    return o;
}

// rms_residual over all pairs (motion.cpp:78-90, apply = transform.cpp:7-11)
__device__ double rms(const double2* P, const double2* Q, int n, const FitOut& t, double* red) {
    const double c = dmul(t.s, cos(t.theta)), sn = dmul(t.s, sin(t.theta));
    double acc = 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const double mx = dadd(dsub(dmul(c, P[k].x), dmul(sn, P[k].y)), t.tx);
        const double my = dadd(dadd(dmul(sn, P[k].x), dmul(c, P[k].y)), t.ty);
        const double dx = dsub(Q[k].x, mx), dy = dsub(Q[k].y, my);
        acc = dadd(acc, dadd(dmul(dx, dx), dmul(dy, dy)));
    }
    return dsqrt(ddiv(block_dsum(acc, red), (double)n));
}

// RANSAC inlier selection; returns the pair count the refit uses and fills mask.
// Hypothesis h's minimal sample (counter-based: the same pair wherever h is scored)
__device__ __forceinline__ bool hypothesis(const double2* P, const double2* Q, int n, bool rigid, uint64_t key, int h,
                                           Model& m) {
    const uint64_t u = mix64(key + (uint64_t)(h + 1) * 0x9e3779b97f4a7c15ULL);
    const int i = (int)((uint32_t)(u >> 32) % (uint32_t)n);
    int j = (int)((uint32_t)u % (uint32_t)(n - 1));
    if (j >= i) ++j;
    return minimal_model(P, Q, i, j, rigid, m);
}

__device__ __forceinline__ uint64_t ransac_key(const stabgpu_ransac_cfg& rc, long long frame) {
    return mix64(rc.seed ^ mix64((uint64_t)frame + 0x9e3779b97f4a7c15ULL));
}

// Scores hypotheses h = first, first + stride, ... (ascending per warp) and
// returns the CTA's best (count, h): most inliers, ties to the lowest h;
// h = -1 when no hypothesis had a valid minimal model.
__device__ int2 ransac_score(const double2* P, const double2* Q, int n, bool rigid, const stabgpu_ransac_cfg& rc,
                             long long frame, int first, int stride, int* wbest_c, int* wbest_h) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double thr2 = dmul(rc.threshold, rc.threshold);
    const uint64_t key = ransac_key(rc, frame);
    int best_c = 0, best_h = -1;
    // the warp's hypotheses h = first + wid + k * stride, 32 at a time: lane l
    // builds the minimal model of k = kb + l (one model per lane instead of
    // every lane building every model), then the warp scores them in k order
    for (int h0 = first + wid; h0 < rc.iterations; h0 += 32 * stride) {
        const int hl = h0 + lane * stride;
        Model ml{0, 0, 0, 0};
        const bool vl = hl < rc.iterations && hypothesis(P, Q, n, rigid, key, hl, ml);
        const unsigned valid = __ballot_sync(0xffffffffu, vl);
        for (unsigned rem = valid; rem; rem &= rem - 1) {
            const int j = __ffs(rem) - 1;
            const Model m{__shfl_sync(0xffffffffu, ml.a, j), __shfl_sync(0xffffffffu, ml.b, j),
                          __shfl_sync(0xffffffffu, ml.tx, j), __shfl_sync(0xffffffffu, ml.ty, j)};
            int cnt = 0;
            for (int k = lane; k < n; k += 32) cnt += inlier(m, P[k], Q[k], thr2) ? 1 : 0;
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (cnt > best_c) {  // h ascends within a warp: strict > keeps the lowest h
                best_c = cnt;
                best_h = h0 + j * stride;
            }
        }
    }
    if (lane == 0) {
        wbest_c[wid] = best_c;
        wbest_h[wid] = best_h;
    }
    __syncthreads();
    int bc = 0, bh = -1;
    for (int w = 0; w < FIT_WARPS; ++w) {
        const int c = wbest_c[w], hh = wbest_h[w];
        if (hh < 0) continue;
        if (bh < 0 || c > bc || (c == bc && hh < bh)) {
            bc = c;
            bh = hh;
        }
    }
    __syncthreads();
    return make_int2(bc, bh);
}

// Given the winning (count, h): the inlier mask of its model (all pairs when
// no hypothesis won or it has fewer than min_tracks inliers); returns the
// number of pairs the refit uses.
__device__ int ransac_finish(const double2* P, const double2* Q, int n, bool rigid, const stabgpu_ransac_cfg& rc,
                             int min_tracks, long long frame, int2 best, uint8_t* mask) {
    const int bc = best.x, bh = best.y;
    if (bh < 0 || bc < min_tracks) {
        for (int k = threadIdx.x; k < n; k += blockDim.x) mask[k] = 1;
        __syncthreads();
        return n;
    }
    Model bm;
    hypothesis(P, Q, n, rigid, ransac_key(rc, frame), bh, bm);  // valid: it was scored
    const double thr2 = dmul(rc.threshold, rc.threshold);
    for (int k = threadIdx.x; k < n; k += blockDim.x) mask[k] = inlier(bm, P[k], Q[k], thr2) ? 1 : 0;
    __syncthreads();
    return bc;
}

__device__ int ransac_select(const double2* P, const double2* Q, int n, bool rigid,
                             const stabgpu_ransac_cfg& rc, int min_tracks, long long frame,
                             uint8_t* mask, int* wbest_c, int* wbest_h) {
    const int2 best = ransac_score(P, Q, n, rigid, rc, frame, 0, FIT_WARPS, wbest_c, wbest_h);
    return ransac_finish(P, Q, n, rigid, rc, min_tracks, frame, best, mask);
}

// Best of several scoring CTAs' results (most inliers, ties to the lowest h).
__device__ int2 merge_best(const int2* r, int k) {
    int bc = 0, bh = -1;
    for (int i = 0; i < k; ++i)
        if (r[i].y >= 0 && (bh < 0 || r[i].x > bc || (r[i].x == bc && r[i].y < bh))) {
            bc = r[i].x;
            bh = r[i].y;
        }
    return make_int2(bc, bh);
}

// Single frame (Stage II): the hypotheses of one fit spread over G CTAs.
// CTA g scores h = 16 g + w, 16 g + w + 16 G, ... (warp w); the fit CTA merges
// the G results, which is the same argmax (ties to the lowest h) as one CTA.
// best[g] (rigid pass) and best[G + g] (similarity pass).
__global__ void __launch_bounds__(FIT_THREADS) ransac_score_kernel(const double2* __restrict__ trk_prev,
                                                                   const double2* __restrict__ trk_cur,
                                                                   const int* __restrict__ trk_n, long long frame,
                                                                   stabgpu_config cfg, int2* __restrict__ best) {
    extern __shared__ __align__(16) unsigned char fsm[];
    __shared__ int wbest_c[FIT_WARPS], wbest_h[FIT_WARPS];
    const int n = trk_n[0];
    const int G = gridDim.x, g = blockIdx.x;
    if (n < cfg.flow.min_tracks) return;
    double2* P = reinterpret_cast<double2*>(fsm);
    double2* Q = P + n;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        P[k] = trk_prev[k];
        Q[k] = trk_cur[k];
    }
    __syncthreads();
    const int mode = cfg.selector.mode;
    for (int pass = 0; pass < 2; ++pass) {
        const bool rigid = pass == 0;
        if (rigid && mode == STABGPU_FORCE_SIMILARITY) continue;
        if (!rigid && mode == STABGPU_FORCE_RIGID) continue;
        const int2 r = ransac_score(P, Q, n, rigid, cfg.ransac, frame, FIT_WARPS * g, FIT_WARPS * G, wbest_c, wbest_h);
        if (threadIdx.x == 0) best[pass * G + g] = r;
    }
}

__global__ void __launch_bounds__(FIT_THREADS) fit_kernel(const double2* __restrict__ trk_prev,
                                                          const double2* __restrict__ trk_cur,
                                                          const int* __restrict__ trk_n, int max_pts,
                                                          long long frame_index0, stabgpu_config cfg,
                                                          stabgpu_motion_record* __restrict__ out,
                                                          long long stream_frames, const int2* __restrict__ pre,
                                                          int pre_ctas, uint8_t* __restrict__ gmask) {
    extern __shared__ __align__(16) unsigned char fsm[];
    __shared__ double red[FIT_WARPS];
    __shared__ int wbest_c[FIT_WARPS], wbest_h[FIT_WARPS];
    const int f = blockIdx.x;
    stabgpu_motion_record rec;
    memset(&rec, 0, sizeof rec);
    // multi-stream chunk: the frame's index within its own stream (the RANSAC
    // seed), and stream starts are first frames (MotionStage::step, pipeline.cpp:84-88)
    long long frame = frame_index0 + f;
    if (stream_frames > 0) {
        frame %= stream_frames;
        if (frame == 0) {
            if (threadIdx.x == 0) {
                rec.frame_kind = STABGPU_FRAME_FIRST;
                out[f] = rec;
            }
            return;
        }
    }
    const int n = trk_n[f];
    rec.n_tracks = n;
    rec.rigid.kind = STABGPU_RIGID;
    rec.similarity.kind = STABGPU_SIMILARITY;
    stabgpu_motion_record* o = out + f;
    if (n < cfg.flow.min_tracks) {
        if (threadIdx.x == 0) {
            rec.frame_kind = STABGPU_FRAME_SKIPPED;
            *o = rec;
        }
        return;
    }
    rec.frame_kind = STABGPU_FRAME_TRACKED;
    const double2* P;
    const double2* Q;
    uint8_t* mask;
    if (gmask) {  // TrackSets too large for shared memory: work in place in global memory
        P = trk_prev + (size_t)f * max_pts;
        Q = trk_cur + (size_t)f * max_pts;
        mask = gmask + (size_t)f * max_pts;
    } else {
        double2* sP = reinterpret_cast<double2*>(fsm);
        double2* sQ = sP + max_pts;
        mask = reinterpret_cast<uint8_t*>(sQ + max_pts);
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
            sP[k] = trk_prev[(size_t)f * max_pts + k];
            sQ[k] = trk_cur[(size_t)f * max_pts + k];
        }
        P = sP;
        Q = sQ;
    }
    __syncthreads();
    const int mode = cfg.selector.mode;
    FitOut fr{0, 0, 0, 1, STABGPU_OK}, fs{0, 0, 0, 1, STABGPU_OK};
    for (int pass = 0; pass < 2; ++pass) {
        const bool rigid = pass == 0;
        if (rigid && mode == STABGPU_FORCE_SIMILARITY) continue;
        if (!rigid && mode == STABGPU_FORCE_RIGID) continue;
        int used = n;
        const uint8_t* m = nullptr;
        if (cfg.ransac.iterations > 0) {
            if (pre)  // hypotheses scored by ransac_score_kernel (one frame)
                used = ransac_finish(P, Q, n, rigid, cfg.ransac, cfg.flow.min_tracks, frame,
                                     merge_best(pre + pass * pre_ctas, pre_ctas), mask);
            else
                used = ransac_select(P, Q, n, rigid, cfg.ransac, cfg.flow.min_tracks, frame, mask, wbest_c,
                                     wbest_h);
            m = used == n ? nullptr : mask;
        }
        const FitOut r = estimate(P, Q, m, n, used, rigid, red);
        if (rigid) {
            fr = r;
            rec.n_inliers_rigid = used;
        } else {
            fs = r;
            rec.n_inliers_similarity = used;
        }
        __syncthreads();
    }
    if (mode == STABGPU_HYBRID && fr.status == STABGPU_OK && fs.status == STABGPU_OK) {
        rec.e_rigid = rms(P, Q, n, fr, red);
        rec.e_similarity = rms(P, Q, n, fs, red);
    }
    if (threadIdx.x == 0) {
        // extract_delta (motion.cpp:92-101)
        rec.rigid.dx = fr.tx;
        rec.rigid.dy = fr.ty;
        rec.rigid.da = fr.theta;
        rec.rigid.dls = 0.0;
        rec.similarity.dx = fs.tx;
        rec.similarity.dy = fs.ty;
        rec.similarity.da = fs.theta;
        rec.similarity.dls = log(fs.s);
        rec.status = fr.status | (fs.status << 8);
        *o = rec;
    }
}

}  // namespace

bool fit_allocates(int max_pts) { return (size_t)max_pts * (2 * sizeof(double2) + 1) > kFitSmemMax; }

void launch_fit(const double2* trk_prev, const double2* trk_cur, const int* trk_n, int max_pts,
                int nframes, long long frame_index0, const stabgpu_config& cfg,
                stabgpu_motion_record* out, cudaStream_t st, long long stream_frames, int2* pre_scratch) {
    if (nframes <= 0) return;
    size_t smem = (size_t)max_pts * (2 * sizeof(double2) + 1);
    uint8_t* gmask = nullptr;
    if (smem > kFitSmemMax) {
        // more pairs than shared memory holds: the kernel reads the TrackSets in
        // place and keeps the inlier masks in stream-ordered global scratch (a
        // failed allocation stays in cudaGetLastError for check_launch)
        if (cudaMallocAsync((void**)&gmask, (size_t)nframes * max_pts, st) != cudaSuccess) return;
        smem = 0;
    }
    ensure_smem(fit_kernel, smem);
    const int2* pre = nullptr;
    int G = 0;
    if (!gmask && nframes == 1 && pre_scratch && cfg.ransac.iterations > 0 && stream_frames == 0) {
        // one frame: spread its hypotheses over G CTAs (one per warp), then fit
        G = std::min(kFitPreCtas, (cfg.ransac.iterations + FIT_WARPS - 1) / FIT_WARPS);
        const size_t ssm = (size_t)max_pts * 2 * sizeof(double2);
        ensure_smem(ransac_score_kernel, ssm);
        ransac_score_kernel<<<G, FIT_THREADS, ssm, st>>>(trk_prev, trk_cur, trk_n, frame_index0, cfg, pre_scratch);
        pre = pre_scratch;
    }
    fit_kernel<<<nframes, FIT_THREADS, smem, st>>>(trk_prev, trk_cur, trk_n, max_pts, frame_index0,
                                                   cfg, out, stream_frames, pre, G, gmask);
    if (gmask) cudaFreeAsync(gmask, st);
}

}  // namespace stabgpu

namespace stabgpu {
namespace {
__global__ void __launch_bounds__(FIT_THREADS) fit_single_kernel(const double2* __restrict__ gP,
                                                                 const double2* __restrict__ gQ,
                                                                 int n, int kind,
                                                                 stabgpu_ransac_cfg rc, int min_tracks,
                                                                 long long frame, FitResult* out,
                                                                 uint8_t* __restrict__ gmask, bool in_place) {
    extern __shared__ __align__(16) unsigned char fsm[];
    __shared__ double red[FIT_WARPS];
    __shared__ int wbest_c[FIT_WARPS], wbest_h[FIT_WARPS];
    const double2* P = gP;
    const double2* Q = gQ;
    uint8_t* mask = gmask;  // in_place: too many pairs for shared memory, work in global memory
    if (!in_place) {
        double2* sP = reinterpret_cast<double2*>(fsm);
        double2* sQ = sP + n;
        mask = reinterpret_cast<uint8_t*>(sQ + n);
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
            sP[k] = gP[k];
            sQ[k] = gQ[k];
        }
        P = sP;
        Q = sQ;
    }
    for (int k = threadIdx.x; k < n; k += blockDim.x) mask[k] = 1;
    __syncthreads();
    const bool rigid = kind == STABGPU_RIGID;
    int used = n;
    const uint8_t* m = nullptr;
    if (n >= 2 && rc.iterations > 0) {
        used = ransac_select(P, Q, n, rigid, rc, min_tracks, frame, mask, wbest_c, wbest_h);
        m = used == n ? nullptr : mask;
    }
    const FitOut r = estimate(P, Q, m, n, used, rigid, red);
    if (!in_place)
        for (int k = threadIdx.x; k < n; k += blockDim.x)
            if (gmask) gmask[k] = mask[k];
    if (threadIdx.x == 0) *out = FitResult{r.tx, r.ty, r.theta, r.s, r.status, used};
}

__global__ void __launch_bounds__(FIT_THREADS) rms_single_kernel(const double2* __restrict__ P,
                                                                 const double2* __restrict__ Q,
                                                                 int n, stabgpu_transform t,
                                                                 double* out) {
    __shared__ double red[FIT_WARPS];
    const FitOut f{t.tx, t.ty, t.theta, t.s, 0};
    const double v = rms(P, Q, n, f, red);
    if (threadIdx.x == 0) *out = v;
}
}  // namespace

void launch_fit_single(const double2* P, const double2* Q, int n, int kind,
                       const stabgpu_ransac_cfg& rc, int min_tracks, long long frame,
                       FitResult* out, uint8_t* mask, cudaStream_t st) {
    size_t smem = (size_t)n * (2 * sizeof(double2) + 1) + 16;
    const bool in_place = smem > kFitSmemMax && mask;
    if (in_place) smem = 0;
    ensure_smem(fit_single_kernel, smem);
    fit_single_kernel<<<1, FIT_THREADS, smem, st>>>(P, Q, n, kind, rc, min_tracks, frame, out, mask, in_place);
}

void launch_rms_single(const double2* P, const double2* Q, int n, stabgpu_transform t, double* out,
                       cudaStream_t st) {
    rms_single_kernel<<<1, FIT_THREADS, 0, st>>>(P, Q, n, t, out);
}
}  // namespace stabgpu
