// k_lk.cu — K5: pyramidal Lucas-Kanade, one warp per feature, forward then
// backward (forward-backward weeding) in the same warp.
//
// Reference: extract_patch (flow.cpp:28-59), build_level_patch (77-126),
// inside (128-130), track_one (132-227), track_lk (243-256), weed_tracks
// (258-280).  Every scalar step uses correctly rounded fp64 ops in the
// reference order; the only departure is the order of the window sums
// (G tensor and the b vector), which a warp reduces as 32 strided partials
// plus a butterfly.  That changes results by ~1e-13 px, far inside the 0.01 px
// tolerance, and every lane ends with identical bits, so the warp's control
// flow (convergence, divergence, status) stays uniform.
//
// Per warp, shared memory holds the extended (2r+3)^2 template patch and the
// template gradients over the valid window; the valid window is a rectangle
// (the reference's per-row / per-column clipping is separable), flattened so
// the 32 lanes stride it densely.  Segments (independent 5-frame tracking
// chains, grid.y) and features (grid.x) are both batched into one launch.
#include <algorithm>
#include <climits>

#include <cuda.h>

#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace stabgpu {

namespace {

struct Level {
    const uint8_t* px;
    int w, h;
    const CUtensorMap* map = nullptr;  // TMA map of the pyramid level (chain kernel), or none
    int frame = 0;                     // frame index of px inside that map
};

// Per-level TMA maps of the pyramid (3D: x, y, frame; box 64 x SM_ROWS x 1),
// passed to the chain kernel as one grid constant; bit l of mask: level l has one
struct LkMaps {
    CUtensorMap m[STABGPU_MAX_LEVELS];
    unsigned mask;
};

__device__ __forceinline__ bool inside(const Level& L, double x, double y) {
    return x >= 0.0 && y >= 0.0 && x <= (double)L.w - 1.0 && y <= (double)L.h - 1.0;
}

__device__ __forceinline__ double bilerp(const Level& L, int x0, int y0, int i, int j, double w00,
                                         double w10, double w01, double w11) {
    // flow.cpp:43-58: clamped indices, shared weights, left-to-right sum
    const int xa = clampi(x0 + i, 0, L.w - 1), xb = clampi(x0 + i + 1, 0, L.w - 1);
    const int ya = clampi(y0 + j, 0, L.h - 1), yb = clampi(y0 + j + 1, 0, L.h - 1);
    const uint8_t* ra = L.px + (size_t)ya * L.w;
    const uint8_t* rb = L.px + (size_t)yb * L.w;
    const double a = __ldg(ra + xa), b = __ldg(ra + xb), c = __ldg(rb + xa), d = __ldg(rb + xb);
    return dadd(dadd(dadd(dmul(w00, a), dmul(w10, b)), dmul(w01, c)), dmul(w11, d));
}

struct Weights {
    int x0, y0;
    double w00, w10, w01, w11;
};

__device__ __forceinline__ Weights weights_at(double cx, double cy) {
    Weights W;
    const double fx0 = floor(cx), fy0 = floor(cy);
    W.x0 = (int)fx0;
    W.y0 = (int)fy0;
    const double fx = dsub(cx, (double)W.x0), fy = dsub(cy, (double)W.y0);
    W.w00 = dmul(dsub(1.0, fx), dsub(1.0, fy));
    W.w10 = dmul(fx, dsub(1.0, fy));
    W.w01 = dmul(dsub(1.0, fx), fy);
    W.w11 = dmul(fx, fy);
    return W;
}

// track_one for one point; called by all 32 lanes of a warp (uniform flow).
__device__ bool track_warp(const DevPyramid& P, int fprev, int fcur, double px, double py,
                           const stabgpu_flow_cfg& cfg, double* ext, double* tgx, double* tgy,
                           double& ox, double& oy, unsigned& iters, unsigned& builds) {
    const int lane = threadIdx.x & 31;
    const int r = cfg.window_radius, side = 2 * r + 1;
    const int e = r + 1, es = 2 * e + 1;
    int start_level = 0;
    for (int l = P.levels - 1; l > 0; --l)
        if (min(P.w[l], P.h[l]) >= side) {
            start_level = l;
            break;
        }
    const int min_count = max(25, side * side / 4);
    const double r2 = (double)r * r, eps2 = dmul(cfg.epsilon, cfg.epsilon);
    double gfx = 0.0, gfy = 0.0;
    for (int level = start_level; level >= 0; --level) {
        const Level pi{P.lvl[level] + (size_t)fprev * P.stride[level], P.w[level], P.h[level]};
        const Level ci{P.lvl[level] + (size_t)fcur * P.stride[level], P.w[level], P.h[level]};
        const double scale = (double)(1u << level);
        const double plx = ddiv(px, scale), ply = ddiv(py, scale);
        if (!inside(pi, plx, ply)) return false;
        // ---- build_level_patch (flow.cpp:77-126)
        ++builds;
        const Weights T = weights_at(plx, ply);
        for (int k = lane; k < es * es; k += 32) {
            const int jj = k / es, ii = k - jj * es;
            ext[k] = bilerp(pi, T.x0 - e, T.y0 - e, ii, jj, T.w00, T.w10, T.w01, T.w11);
        }
        __syncwarp();
        // valid rows: 1 <= y0-r+j && y0-r+j+2 <= h-1 ; columns alike
        const int jv0 = max(0, 1 - T.y0 + r), jv1 = min(side - 1, pi.h - 3 - T.y0 + r);
        const int iv0 = max(0, 1 - T.x0 + r), iv1 = min(side - 1, pi.w - 3 - T.x0 + r);
        const int vh = jv1 - jv0 + 1, vw = iv1 - iv0 + 1;
        const int count = (vh > 0 && vw > 0) ? vh * vw : 0;
        if (count < min_count) {  // TooSmall (flow.cpp:116-118)
            if (level == 0) return false;
            gfx = dmul(gfx, 2.0);
            gfy = dmul(gfy, 2.0);
            continue;
        }
        const int di = 32 % vw, dj = 32 / vw;
        double gxx = 0.0, gxy = 0.0, gyy = 0.0;
        {
            int j = jv0 + lane / vw, i = iv0 + lane % vw;
            for (int k = lane; k < count; k += 32) {
                const double* mid = ext + (j + 1) * es + 1;
                const double dx = dmul(0.5, dsub(mid[i + 1], mid[i - 1]));
                const double dy = dmul(0.5, dsub(mid[i + es], mid[i - es]));
                tgx[k] = dx;
                tgy[k] = dy;
                gxx = dadd(gxx, dmul(dx, dx));
                gxy = dadd(gxy, dmul(dx, dy));
                gyy = dadd(gyy, dmul(dy, dy));
                i += di;
                j += dj;
                if (i > iv1) {
                    i -= vw;
                    ++j;
                }
            }
        }
        gxx = warp_dsum(gxx);
        gxy = warp_dsum(gxy);
        gyy = warp_dsum(gyy);
        __syncwarp();
        {
            const double ht = dmul(0.5, dadd(gxx, gyy)), hd = dmul(0.5, dsub(gxx, gyy));
            const double me = dsub(ht, dsqrt(dadd(dmul(hd, hd), dmul(gxy, gxy))));
            if (me < dmul(1e-4, (double)count)) return false;  // Unconditioned
        }
        const double det = dsub(dmul(gxx, gyy), dmul(gxy, gxy));
        double vx = 0.0, vy = 0.0;
        bool diverged = false;
        for (int it = 0; it < cfg.max_iterations; ++it) {
            const double qx = dadd(dadd(plx, gfx), vx), qy = dadd(dadd(ply, gfy), vy);
            if (!inside(ci, qx, qy)) {
                diverged = true;
                break;
            }
            ++iters;
            const Weights C = weights_at(qx, qy);
            double bx = 0.0, by = 0.0;
            int j = jv0 + lane / vw, i = iv0 + lane % vw;
            for (int k = lane; k < count; k += 32) {
                const double cur = bilerp(ci, C.x0 - r, C.y0 - r, i, j, C.w00, C.w10, C.w01, C.w11);
                const double d = dsub(ext[(j + 1) * es + i + 1], cur);
                bx = dadd(bx, dmul(d, tgx[k]));
                by = dadd(by, dmul(d, tgy[k]));
                i += di;
                j += dj;
                if (i > iv1) {
                    i -= vw;
                    ++j;
                }
            }
            bx = warp_dsum(bx);
            by = warp_dsum(by);
            const double dx = ddiv(dsub(dmul(gyy, bx), dmul(gxy, by)), det);
            const double dy = ddiv(dsub(dmul(gxx, by), dmul(gxy, bx)), det);
            vx = dadd(vx, dx);
            vy = dadd(vy, dy);
            if (dadd(dmul(vx, vx), dmul(vy, vy)) > r2) {
                diverged = true;
                break;
            }
            if (dadd(dmul(dx, dx), dmul(dy, dy)) < eps2) break;
        }
        __syncwarp();
        if (diverged && level == 0) return false;
        if (!diverged) {
            gfx = dadd(gfx, vx);
            gfy = dadd(gfy, vy);
        }
        if (level > 0) {
            gfx = dmul(gfx, 2.0);
            gfy = dmul(gfy, 2.0);
        }
    }
    const double rx = dadd(px, gfx), ry = dadd(py, gfy);
    const Level base{P.lvl[0] + (size_t)fcur * P.stride[0], P.w[0], P.h[0]};
    if (!inside(base, rx, ry)) return false;
    ox = rx;
    oy = ry;
    return true;
}


// ---------------------------------------------------------------------------
// Fast path for windows up to 31x31 (r <= 15): lanes are window columns, rows
// are rolled through registers, and the bilinear patch is evaluated in its
// separable form (horizontal lerp per image row, vertical lerp per window
// row), so each window entry costs one byte load, one shuffle and a handful
// of fp64 ops instead of four clamped 64-bit gathers.  Rounding differs from
// the reference's weighted form by ~1e-13 (tolerance-level, like the sums).

// horizontal lerp a + f*(b - a) of two bytes: b - a is taken exactly between
// the 2^52-magic doubles (one DADD saved), a = magic - 2^52 exactly
__device__ __forceinline__ double hlerp(uint32_t a, uint32_t b, double f) {
    const double ma = __hiloint2double(0x43300000, (int)a), mb = __hiloint2double(0x43300000, (int)b);
    return fma(f, mb - ma, ma - 4503599627370496.0);
}

__device__ __forceinline__ double u2d(uint32_t b) {  // exact u8 -> double, no I2F
    return __hiloint2double(0x43300000, (int)b) - 4503599627370496.0;
}

__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t px_at(const Level& L, int x, int y, bool interior) {
    if (!interior) {
        x = clampi(x, 0, L.w - 1);
        y = clampi(y, 0, L.h - 1);
    }
    return __ldg(L.px + (size_t)y * L.w + x);
}


// per-warp 2x2 system in shared memory, reloaded per use (volatile: keeps the
// six doubles out of the register file across the iteration loop)
__device__ __forceinline__ double ldsv(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}

// Current-frame window staging.  The iterations of one level read the
// (vh+1) x (vw+1) source block around the moving estimate; it is copied once
// into a per-warp shared tile with a margin of SM_MARGIN pixels (clamped at
// the image border exactly as the reference's clamped fetches), and re-copied
// only when the estimate leaves the staged region.  Every lane's byte loads
// are independent, so the global latency is paid once per staging instead of
// once per row.
constexpr int SM_MARGIN = 3;
constexpr int SM_PITCH = 64;  // bytes per staged row (>= 15 + 32 + 1 + 2 * margin + 3: the TMA box width)
constexpr int SM_ROWS = 40;   // >= 32 + 2 * margin (the TMA box height)
// Per-warp shared layout (doubles): the system record first (2x2 system,
// level origin, 1/det, S_uv, step count, level bounds, thresholds), then the
// staged window, then the template gradients.  With one warp per CTA (the
// chain kernel) every record address is a constant offset of the shared
// window: no address arithmetic in the iteration loop.
constexpr int SYS_D = 32;  // 256 B: the staged window after it is 128-byte aligned (TMA destination)
constexpr int STG_D = SM_ROWS * SM_PITCH / 8;
constexpr int SYS_TMA_PHASE = 23, SYS_TMA_BAR = 24;  // sys slots: TMA mbarrier parity (int) and the mbarrier
__host__ __device__ constexpr int lk_per_warp(int side) { return SYS_D + STG_D + 2 * (side * side + 1); }

// Copies image block [x0, x0+sw) x [y0, y0+sh) (clamped at the border) to a
// per-warp shared tile (row pitch SM_PITCH) and returns the tile column of
// image column x0.  Interior blocks of 4-byte-aligned rows go as aligned
// 32-bit words, several rows per warp instruction (lane -> (row, word)); the
// border case goes byte by byte with the reference's clamped indices.
__device__ __forceinline__ int stage_block(const Level& L, int x0, int y0, int sw, int sh, uint8_t* dst,
                                           double* sys = nullptr) {
    const int lane = threadIdx.x & 31;
    // interior block of a level with a TMA map: one bulk-tensor copy of the
    // 64 x SM_ROWS box at (x0 & ~15, y0) by lane 0, completion on the warp's
    // mbarrier (bytes past the image are zero-filled and never read)
    if (L.map && x0 >= 0 && y0 >= 0 && x0 + sw <= L.w && y0 + sh <= L.h && (x0 & 15) + sw <= SM_PITCH &&
        sh <= SM_ROWS) {
        const int xa = x0 & ~15;
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(sys + SYS_TMA_BAR);
        int* php = reinterpret_cast<int*>(sys + SYS_TMA_PHASE);
        const uint32_t ph = (uint32_t)*php;
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // this warp's reads of the old block
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(SM_PITCH * SM_ROWS)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                "[%5];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                "l"(L.map), "r"(xa), "r"(y0), "r"(L.frame), "r"(bar)
                : "memory");
        }
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}\n"
                : "=r"(done)
                : "r"(bar), "r"(ph)
                : "memory");
        __syncwarp();
        if (lane == 0) *php = (int)(ph ^ 1u);
        return x0 - xa;
    }
    const int xw = x0 & ~3;
    const int nw = ((x0 + sw - 1) >> 2) - (xw >> 2) + 1;  // words per row (<= SM_PITCH / 4)
    const bool words = ((L.w & 3) == 0) && ((reinterpret_cast<uintptr_t>(L.px) & 3) == 0) && x0 >= 0 &&
                       y0 >= 0 && xw + 4 * nw <= L.w && y0 + sh <= L.h;
    if (words) {
        // small quotients by reciprocal: floor((a + 0.5) / nw) == a / nw for
        // 0 <= a <= 32, nw <= 32, with a margin far above the RCP error
        const float rn = __fdividef(1.0f, (float)nw);
        const int rpp = (int)(32.5f * rn), lr = (int)(((float)lane + 0.5f) * rn), lw = lane - lr * nw;
        if (lr < rpp) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(L.px + (size_t)(y0 + lr) * L.w + xw) + lw;
            uint32_t* d = reinterpret_cast<uint32_t*>(dst + lr * SM_PITCH) + lw;
            const size_t sstep = (size_t)rpp * (L.w >> 2);
            const int dstep = rpp * (SM_PITCH / 4);
            // this lane's rows lr, lr + rpp, ...: passes of four predicated
            // loads, all issued before the first store (a 28-row window at
            // rpp = 4 is two passes, i.e. two global latencies)
            const int nr = (sh - lr + rpp - 1) / rpp;
            for (int base = 0; base < nr; base += 4) {
                uint32_t v0 = 0, v1 = 0, v2 = 0, v3 = 0;
                v0 = __ldg(src);
                if (base + 1 < nr) v1 = __ldg(src + sstep);
                if (base + 2 < nr) v2 = __ldg(src + 2 * sstep);
                if (base + 3 < nr) v3 = __ldg(src + 3 * sstep);
                d[0] = v0;
                if (base + 1 < nr) d[dstep] = v1;
                if (base + 2 < nr) d[2 * dstep] = v2;
                if (base + 3 < nr) d[3 * dstep] = v3;
                src += 4 * sstep;
                d += 4 * dstep;
            }
        }
        return x0 - xw;
    }
    for (int i = lane; i < sw * sh; i += 32) {
        const int r = i / sw, c = i - r * sw;
        dst[r * SM_PITCH + c] =
            __ldg(L.px + (size_t)clampi(y0 + r, 0, L.h - 1) * L.w + clampi(x0 + c, 0, L.w - 1));
    }
    return 0;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// Correlation sums of one integer window position.  With cur(j, i) the
// bilinear sample at (cy + j + fy, cx + i + fx) and P the staged pixels,
//   sum_{j,i} g(j,i) cur(j,i) = lerp_y(lerp_x(S00, S10), lerp_x(S01, S11))
// where S_uv = sum_{j,i} g(j,i) P(j+v, i+u) (lerp_x(a, b) = a + fx (b - a)).
// The S_uv depend on the integer position only, so an iteration that stays in
// the previous iteration's cell (about half of them) reuses them and costs a
// dozen fp64 ops instead of a window pass.  Lane C <-> gradient column C
// (0..vw-1; lanes past the window read the zero slot); per gradient row R:
// S00 += P(R,C) g(R,C), S10 += P(R,C+1) g(R,C), S01 += P(R+1,C) g(R,C),
// S11 += P(R+1,C+1) g(R,C).  Each lane loads its gradient once per row (one
// 16-byte LDS) and two pixel bytes; the pixel row R+1 carries over as row R.
// The same products as the bilinear form, summed in another order
// (tolerance-level, ~1e-13 px).
// Returns the eight lane partials in s[0..7] = {S00, S10, S01, S11} x {x, y}.
__device__ __forceinline__ void corr_pass(const uint8_t* src, int vh, const double2* ga, int sa, double* s) {
    // ga: column C of the gradients (or the zero slot, row step sa = 0)
    const int lane = threadIdx.x & 31;
    src += lane;
    double p0 = u2d(src[0]), q0 = u2d(src[1]);
    double a0x = 0.0, a0y = 0.0, b0x = 0.0, b0y = 0.0, a1x = 0.0, a1y = 0.0, b1x = 0.0, b1y = 0.0;
    // software-pipelined: row k+1's gradient and pixel bytes are loaded while
    // row k's products issue (the last prefetch reads one row past the
    // window: pixel row vh + 1 of the staging buffer, and — the gradient rows
    // being stored bottom-up, sa < 0 — the bytes in front of the gradient
    // array, i.e. the staging buffer's tail; both inside the warp's shared
    // area, both discarded)
    src += SM_PITCH;
    uint32_t pn = src[0], qn = src[1];
    double2 gn = ga[0];
#pragma unroll 3
    for (int k = 0; k < vh; ++k) {
        const double2 g = gn;
        const double p1 = u2d(pn), q1 = u2d(qn);
        ga += sa;
        src += SM_PITCH;
        gn = ga[0];
        pn = src[0];
        qn = src[1];
        a0x = fma(p0, g.x, a0x);
        a0y = fma(p0, g.y, a0y);
        b0x = fma(q0, g.x, b0x);
        b0y = fma(q0, g.y, b0y);
        a1x = fma(p1, g.x, a1x);
        a1y = fma(p1, g.y, a1y);
        b1x = fma(q1, g.x, b1x);
        b1y = fma(q1, g.y, b1y);
        p0 = p1;
        q0 = q1;
    }
    s[0] = a0x;
    s[1] = b0x;
    s[2] = a1x;
    s[3] = b1x;
    s[4] = a0y;
    s[5] = b0y;
    s[6] = a1y;
    s[7] = b1y;
}

// Halved warp totals of eight values by reduce-scatter (18 shuffles instead of 80):
// each xor step halves the set a lane carries.  Lane l ends with the total of
// value (l >> 2) & 7; lanes with l % 4 == 0 store it to out[(l >> 2) & 7].
__device__ __forceinline__ void warp_dsum8_store(const double* v, double* out) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
    double w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double send = h4 ? v[k] : v[k + 4], keep = h4 ? v[k + 4] : v[k];
        w[k] = keep + __shfl_xor_sync(FULL, send, 16);
    }
    double u[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double send = h3 ? w[k] : w[k + 2], keep = h3 ? w[k + 2] : w[k];
        u[k] = keep + __shfl_xor_sync(FULL, send, 8);
    }
    double z;
    {
        const double send = h2 ? u[0] : u[1], keep = h2 ? u[1] : u[0];
        z = keep + __shfl_xor_sync(FULL, send, 4);
    }
    z += __shfl_xor_sync(FULL, z, 2);
    z += __shfl_xor_sync(FULL, z, 1);
    if ((lane & 3) == 0) out[(lane >> 2) & 7] = 0.5 * z;  // gradients are stored doubled
}

// build_level_patch over the extended (es x es) patch: lane L <-> extended
// column L (XTRA: es == 33, lane 31 also owns column 32), image rows rolled
// through registers.  Writes the template gradients over the valid window
// (row stride vw) and accumulates G and T = sum(template value * gradient).
// Only the image rows the valid rows need are visited (jv0 .. jv1+3).  The
// central differences are stored and summed unscaled (right - left, not
// 0.5 * (right - left)); scaling by a power of two commutes with every
// rounding, so G * 1/4, T * 1/2 and the correlation sums * 1/2 are bitwise
// the scaled results.
template <bool XTRA>
__device__ __forceinline__ void template_pass(const uint8_t* src, double fx, double fy, int jv0, int jv1,
                                              int iv0, int iv1, uint32_t ga, uint32_t grow, double& gxx, double& gxy,
                                              double& gyy, double& tx, double& ty) {
    // src: staged image block of rows yb .. yb+es, columns xb .. xb+es+1
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const bool xtra = XTRA && lane == 31;
    const int ti = lane - 1;  // template column of this lane
    const bool tcol = ti >= iv0 && ti <= iv1;
    // rows are stored bottom-up (row j at [jv1 - j][.]): the correlation pass
    // walks them with a negative step, so its one-row-ahead prefetch past the
    // last row lands in front of the array (the tail of the staging buffer),
    // never past the end of the warp's shared memory
    ga += (uint32_t)((tcol ? ti - iv0 : 0) * 16) + (uint32_t)(jv1 - jv0) * grow;
    src += lane + jv0 * SM_PITCH;
    // extended rows jv0 (eA) and jv0 + 1 (eB) from image rows jv0 .. jv0+2
    double hp = hlerp(src[0], src[1], fx), hpx = 0.0;
    if (XTRA) hpx = hlerp(src[1], src[2], fx);
    double h = hlerp(src[SM_PITCH], src[SM_PITCH + 1], fx), hx = 0.0;
    if (XTRA) hx = hlerp(src[SM_PITCH + 1], src[SM_PITCH + 2], fx);
    double eA = fma(fy, h - hp, hp), eAx = 0.0;
    if (XTRA) eAx = fma(fy, hx - hpx, hpx);
    hp = h;
    hpx = hx;
    h = hlerp(src[2 * SM_PITCH], src[2 * SM_PITCH + 1], fx);
    if (XTRA) hx = hlerp(src[2 * SM_PITCH + 1], src[2 * SM_PITCH + 2], fx);
    double eB = fma(fy, h - hp, hp), eBx = 0.0;
    if (XTRA) eBx = fma(fy, hx - hpx, hpx);
    (void)eAx;
    hp = h;
    hpx = hx;
    src += 3 * SM_PITCH;
    // software-pipelined: image row j+3's bytes are loaded while row j's
    // template values are formed (the last prefetch reads one row past the
    // staged block, inside the warp's shared area, and is discarded)
    uint32_t n0 = src[0], n1 = src[1], n2 = XTRA ? src[2] : 0u;
#pragma unroll 3
    for (int j = jv0; j <= jv1; ++j) {  // template row j: extended rows j .. j+2
        const uint32_t c0 = n0, c1 = n1, c2 = n2;
        src += SM_PITCH;
        n0 = src[0];
        n1 = src[1];
        if (XTRA) n2 = src[2];
        h = hlerp(c0, c1, fx);
        if (XTRA) hx = hlerp(c1, c2, fx);
        const double ev = fma(fy, h - hp, hp);  // extended row j + 2
        double evx = 0.0;
        if (XTRA) evx = fma(fy, hx - hpx, hpx);
        double right = __shfl_down_sync(FULL, eB, 1);
        const double left = __shfl_up_sync(FULL, eB, 1);
        if (XTRA && xtra) right = eBx;
        // 2 * gradient; lanes outside the template columns accumulate finite
        // junk that is dropped after the loop (no per-row select)
        const double dx = right - left;
        const double dy = ev - eA;
        if (tcol)
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ga), "d"(dx), "d"(dy));
        ga -= grow;
        gxx = fma(dx, dx, gxx);
        gxy = fma(dx, dy, gxy);
        gyy = fma(dy, dy, gyy);
        tx = fma(eB, dx, tx);
        ty = fma(eB, dy, ty);
        eA = eB;
        eB = ev;
        if (XTRA) eBx = evx;
        hp = h;
        if (XTRA) hpx = hx;
    }
    if (!tcol) gxx = gxy = gyy = tx = ty = 0.0;
}

// a / b correctly rounded, given y = RN(1/b): q0 = RN(a*y) is within one ulp
// of a/b, r = a - q0*b is exact in one FMA, and RN(q0 + r*y) = RN(a/b)
// (Markstein's final correction step; b = det is a normal number bounded away
// from 0 by the Unconditioned test, and a/b is far from the underflow range).
// Three DP ops instead of the ~30-instruction IEEE division sequence; the
// bits equal __ddiv_rn(a, b).
__device__ __forceinline__ double div_rn_recip(double a, double b, double y) {
    const double q0 = dmul(a, y);
    const double r = fma(-q0, b, a);
    return fma(r, y, q0);
}

// Pyramidal track_one (flow.cpp:132-227) of up to two trackers that share one
// template: the patch around (px, py) in frame ft.  Tracker 0 follows the
// point into frame f0, tracker 1 (when f1 >= 0) into frame f1.  Both walk the
// levels coarse to fine with their own guesses; each level's template is
// built once (staged block -> gradients, G and T) and both trackers iterate on
// it.  Tracker j's success and result go to ok[j], o[j]; iteration counts to
// it[j].  A template failure (outside / TooSmall at level 0 / Unconditioned)
// fails both, exactly as it fails a lone track_one.
__device__ void track_dual(const DevPyramid& P, int ft, double px, double py, int f0, int f1,
                           const stabgpu_flow_cfg& cfg, double* tg, uint8_t* stg, double* sys, bool& ok0, bool& ok1,
                           double2& o0, double2& o1, unsigned& it0, unsigned& it1, unsigned& builds,
                           const LkMaps* maps = nullptr) {
    const int lane = threadIdx.x & 31;
    const int r = cfg.window_radius, side = 2 * r + 1;
    const int e = r + 1, es = 2 * e + 1;  // extended template patch (flow.cpp:79-81)
    int start_level = 0;
    for (int l = P.levels - 1; l > 0; --l)
        if (min(P.w[l], P.h[l]) >= side) {
            start_level = l;
            break;
        }
    const int min_count = max(25, side * side / 4);
    if (lane == 0) {  // per-call thresholds in the shared system record (sys[21..22])
        sys[21] = (double)r * r;
        sys[22] = dmul(cfg.epsilon, cfg.epsilon);
    }
    const int nt = f1 >= 0 ? 2 : 1;
    // per-tracker guesses in scalars (no local-memory arrays)
    double gx0 = 0.0, gy0 = 0.0, gx1 = 0.0, gy1 = 0.0;
    bool al0 = true, al1 = f1 >= 0;
    ok0 = ok1 = false;
    for (int level = start_level; level >= 0; --level) {
        const CUtensorMap* lmap = (maps && ((maps->mask >> level) & 1u)) ? &maps->m[level] : nullptr;
        const Level pi{P.lvl[level] + (size_t)ft * P.stride[level], P.w[level], P.h[level], lmap, ft};
        const double scale = (double)(1u << level);
        const double plx = ddiv(px, scale), ply = ddiv(py, scale);
        if (!inside(pi, plx, ply)) return;
        const int x0 = (int)floor(plx), y0 = (int)floor(ply);
        // valid window (flow.cpp:95-103): rows 1 <= y0-r+j <= h-3, columns alike
        const int jv0 = max(0, 1 - y0 + r), jv1 = min(side - 1, pi.h - 3 - y0 + r);
        const int iv0 = max(0, 1 - x0 + r), iv1 = min(side - 1, pi.w - 3 - x0 + r);
        const int vh = jv1 - jv0 + 1, vw = iv1 - iv0 + 1;
        const int count = (vh > 0 && vw > 0) ? vh * vw : 0;
        if (count < min_count) {  // TooSmall (flow.cpp:116-118) depends on the count only
            if (level == 0) return;
            gx0 = dmul(gx0, 2.0);
            gy0 = dmul(gy0, 2.0);
            gx1 = dmul(gx1, 2.0);
            gy1 = dmul(gy1, 2.0);
            continue;
        }
        ++builds;
        // ---- template (build_level_patch): lane L <-> extended column L.
        // Stored: gradients over the valid window; the template values enter
        // only through T = sum(tval * grad), accumulated here.
        const double fx = dsub(plx, (double)x0), fy = dsub(ply, (double)y0);
        const int xb = x0 - e, yb = y0 - e;  // image origin of the extended patch
        double gxx = 0.0, gxy = 0.0, gyy = 0.0, tx = 0.0, ty = 0.0;
        const uint32_t ga0 = (uint32_t)__cvta_generic_to_shared(tg);
        __syncwarp();
        const int toff = stage_block(pi, xb, yb, es + 2, es + 1, stg, sys);
        __syncwarp();
        const uint32_t grow = (uint32_t)vw * 16u;  // gradients: [vh][vw] {gx, gy}, then a zero slot
        if (es > 31) template_pass<true>(stg + toff, fx, fy, jv0, jv1, iv0, iv1, ga0, grow, gxx, gxy, gyy, tx, ty);
        else template_pass<false>(stg + toff, fx, fy, jv0, jv1, iv0, iv1, ga0, grow, gxx, gxy, gyy, tx, ty);
        if (lane == 0)
            asm volatile("st.shared.v2.f64 [%0], {%1, %1};" ::"r"(ga0 + (uint32_t)(vh * vw) * 16u), "d"(0.0));
        // the pass summed unscaled differences: exact power-of-two rescale
        gxx = 0.25 * warp_dsum(gxx);
        gxy = 0.25 * warp_dsum(gxy);
        gyy = 0.25 * warp_dsum(gyy);
        tx = 0.5 * warp_dsum(tx);
        ty = 0.5 * warp_dsum(ty);
        __syncwarp();
        {
            const double ht = dmul(0.5, dadd(gxx, gyy)), hd = dmul(0.5, dsub(gxx, gyy));
            const double me = dsub(ht, dsqrt(dadd(dmul(hd, hd), dmul(gxy, gxy))));
            if (me < dmul(1e-4, (double)count)) return;  // Unconditioned
        }
        {
            const double det = dsub(dmul(gxx, gyy), dmul(gxy, gxy));
            if (lane == 0) {
                sys[0] = gxx;
                sys[1] = gxy;
                sys[2] = gyy;
                sys[3] = tx;
                sys[4] = ty;
                sys[5] = det;
                sys[6] = plx;
                sys[7] = ply;
                sys[8] = ddiv(1.0, det);  // RN(1/det), for div_rn_recip
                sys[19] = (double)pi.w - 1.0;  // inside() bounds of the level (every frame has its dims)
                sys[20] = (double)pi.h - 1.0;
            }
            __syncwarp();
        }
        // lanes past the valid window read the zero slot (row step 0)
        // (gradient rows are stored bottom-up: row 0 is the last one, step -vw)
        const double2* gcol = reinterpret_cast<const double2*>(tg) + (lane < vw ? (vh - 1) * vw + lane : vh * vw);
        const int gstep = lane < vw ? -vw : 0;
        const int sw = vw + 1 + 2 * SM_MARGIN, sh = vh + 1 + 2 * SM_MARGIN;
#pragma unroll 1
        for (int j = 0; j < nt; ++j) {
            if (!(j ? al1 : al0)) continue;
            const int fc = j == 0 ? f0 : f1;
            const Level ci{P.lvl[level] + (size_t)fc * P.stride[level], P.w[level], P.h[level], lmap, fc};
            double gfx = j ? gx1 : gx0, gfy = j ? gy1 : gy0;
            unsigned nit = 0;
            // ---- iterations (flow.cpp:184-209): lane L <-> valid column iv0 + L
            double vx = 0.0, vy = 0.0;
            bool diverged = false;
            int sx0 = INT_MIN / 2, sy0 = INT_MIN / 2, soff = 0;  // staged region origin (none yet)
            int ccx = INT_MIN / 2, ccy = INT_MIN / 2;  // window cell whose S_uv are in sys[10..17]
            for (int k = 0; k < cfg.max_iterations; ++k) {
                const double qx = dadd(dadd(ldsv(sys + 6), gfx), vx), qy = dadd(dadd(ldsv(sys + 7), gfy), vy);
                if (!(qx >= 0.0 && qy >= 0.0 && qx <= ldsv(sys + 19) && qy <= ldsv(sys + 20))) {  // inside()
                    diverged = true;
                    break;
                }
                ++nit;
                const int qx0 = (int)floor(qx), qy0 = (int)floor(qy);
                const double cfx = dsub(qx, (double)qx0), cfy = dsub(qy, (double)qy0);
                const int cx = qx0 - r + iv0, cy = qy0 - r + jv0;  // image origin of the valid window
                if (cx != ccx || cy != ccy) {  // new cell: correlation sums S_uv
                    if (cx < sx0 || cy < sy0 || cx + vw + 1 > sx0 + sw || cy + vh + 1 > sy0 + sh) {
                        sx0 = cx - SM_MARGIN;
                        sy0 = cy - SM_MARGIN;
                        __syncwarp();
                        soff = stage_block(ci, sx0, sy0, sw, sh, stg, sys);
                        __syncwarp();
                    }
                    double sv[8];
                    corr_pass(stg + soff + (cy - sy0) * SM_PITCH + (cx - sx0), vh, gcol, gstep, sv);
                    warp_dsum8_store(sv, sys + 10);
                    __syncwarp();
                    ccx = cx;
                    ccy = cy;
                }
                // sum(cur * grad) from the cell's S_uv; b = T - that
                const double tx0 = fma(cfx, ldsv(sys + 11) - ldsv(sys + 10), ldsv(sys + 10));
                const double tx1 = fma(cfx, ldsv(sys + 13) - ldsv(sys + 12), ldsv(sys + 12));
                const double ty0 = fma(cfx, ldsv(sys + 15) - ldsv(sys + 14), ldsv(sys + 14));
                const double ty1 = fma(cfx, ldsv(sys + 17) - ldsv(sys + 16), ldsv(sys + 16));
                const double bx = ldsv(sys + 3) - fma(cfy, tx1 - tx0, tx0);
                const double by = ldsv(sys + 4) - fma(cfy, ty1 - ty0, ty0);
                const double sxx = ldsv(sys), sxy = ldsv(sys + 1), syy = ldsv(sys + 2), sdet = ldsv(sys + 5);
                const double rdet = ldsv(sys + 8);
                const double dx = div_rn_recip(dsub(dmul(syy, bx), dmul(sxy, by)), sdet, rdet);
                const double dy = div_rn_recip(dsub(dmul(sxx, by), dmul(sxy, bx)), sdet, rdet);
                vx = dadd(vx, dx);
                vy = dadd(vy, dy);
                if (dadd(dmul(vx, vx), dmul(vy, vy)) > ldsv(sys + 21)) {
                    diverged = true;
                    break;
                }
                if (dadd(dmul(dx, dx), dmul(dy, dy)) < ldsv(sys + 22)) break;
            }
            __syncwarp();
            if (j) it1 += nit;
            else it0 += nit;
            if (diverged && level == 0) {
                if (j) al1 = false;
                else al0 = false;
                continue;
            }
            if (!diverged) {
                gfx = dadd(gfx, vx);
                gfy = dadd(gfy, vy);
            }
            if (level > 0) {
                gfx = dmul(gfx, 2.0);
                gfy = dmul(gfy, 2.0);
            }
            if (j) {
                gx1 = gfx;
                gy1 = gfy;
            } else {
                gx0 = gfx;
                gy0 = gfy;
            }
        }
        if (!al0 && !al1) return;
    }
    const Level b0{P.lvl[0] + (size_t)f0 * P.stride[0], P.w[0], P.h[0]};
    if (al0) {
        const double rx = dadd(px, gx0), ry = dadd(py, gy0);
        if (inside(b0, rx, ry)) {
            ok0 = true;
            o0 = make_double2(rx, ry);
        }
    }
    if (al1) {
        const Level b1{P.lvl[0] + (size_t)f1 * P.stride[0], P.w[0], P.h[0]};
        const double rx = dadd(px, gx1), ry = dadd(py, gy1);
        if (inside(b1, rx, ry)) {
            ok1 = true;
            o1 = make_double2(rx, ry);
        }
    }
}

__device__ __forceinline__ bool track_warp_fast(const DevPyramid& P, int fprev, int fcur, double px, double py,
                                                const stabgpu_flow_cfg& cfg, double* tg, uint8_t* stg, double* sys,
                                                double& ox, double& oy, unsigned& iters, unsigned& builds) {
    bool ok0, ok1;
    double2 o0, o1;
    unsigned it0 = 0, it1 = 0;
    track_dual(P, fprev, px, py, fcur, -1, cfg, tg, stg, sys, ok0, ok1, o0, o1, it0, it1, builds);
    iters += it0;
    if (ok0) {
        ox = o0.x;
        oy = o0.y;
    }
    return ok0;
}

// Persistent warps: each warp pulls (segment, point) work items from a global
// counter, so early-exiting points never leave a warp slot idle.
__global__ void __launch_bounds__(128, 4) lk_fast_kernel(LkStep s, stabgpu_flow_cfg cfg,
                                                      unsigned* __restrict__ work, int smem_per_warp) {
    extern __shared__ __align__(16) double lsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* sys = lsm + (size_t)warp * smem_per_warp;
    uint8_t* stg = reinterpret_cast<uint8_t*>(sys + SYS_D);
    double* tg = sys + SYS_D + STG_D;
    const unsigned total = (unsigned)s.nseg * (unsigned)s.max_pts;
    while (true) {
        unsigned item = 0;
        if (lane == 0) item = atomicAdd(work, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= total) break;
        const int seg = (int)(item / (unsigned)s.max_pts), k = (int)(item % (unsigned)s.max_pts);
        const int fprev = s.frame0 + seg_base(seg, s.seg_len, s.F, s.nsps) + s.t - 1, fcur = fprev + 1;
        if (fcur >= s.frame0 + seg_end(seg, s.F, s.nsps, s.nframes - s.frame0) || k >= s.npts[seg]) continue;
        const size_t slot = (size_t)seg * s.max_pts + k;
        const double2 p = s.pts[slot];
        unsigned iters = 0, builds = 0;
        double fx = p.x, fy = p.y;
        // one call site (code size): mode 0 = forward, 1 = forward + backward,
        // 2 = backward from the current point against s.ref
        const int passes = s.mode == 1 ? 2 : 1;
        int fa = s.mode == 2 ? fcur : fprev, fb = s.mode == 2 ? fprev : fcur;
        double ax = p.x, ay = p.y, ox = 0.0, oy = 0.0;
        bool keep = true;
        for (int pass = 0; pass < passes && keep; ++pass) {
            keep = track_warp_fast(s.pyr, fa, fb, ax, ay, cfg, tg, stg, sys, ox, oy, iters, builds);
            if (keep && pass == 0 && s.mode != 2) {
                fx = ox;
                fy = oy;
            }
            const int t = fa;
            fa = fb;
            fb = t;
            ax = ox;
            ay = oy;
        }
        if (keep && s.mode != 0) {  // forward-backward test (flow.cpp weed_tracks)
            const double2 q = s.mode == 2 ? s.ref[slot] : p;
            const double ex = dsub(ox, q.x), ey = dsub(oy, q.y);
            keep = dadd(dmul(ex, ex), dmul(ey, ey)) <= dmul(cfg.fb_threshold, cfg.fb_threshold);
        }
        if (lane == 0) {
            s.fwd[slot] = make_double2(fx, fy);
            s.keep[slot] = keep ? 1 : 0;
            if (s.iter_count) {
                atomicAdd(s.iter_count, (unsigned long long)iters);
                atomicAdd(s.iter_count + 1, (unsigned long long)builds);
                atomicAdd(s.iter_count + 2, 1ull);
            }
        }
        __syncwarp();
    }
}

// Whole tracking chain of one detected point through its segment (all R
// steps of Tracker::advance, pipeline.cpp / flow.cpp:243-280) in one warp.
// Step t's backward track (weed_tracks: template in frame t around f_t) and
// step t+1's forward track (track_lk: the same template, since the kept
// point f_t is the next step's start) share one template build per level.
// The forward t+1 result is used only when step t keeps the point, and its
// iterations are counted only then, so the counters match a step-by-step run.
// MS: several streams per chunk (segment map; step count parked in shared
// memory).  The one-stream instance keeps the map in kernel parameters.
// One warp per CTA (20 per SM): the warp's shared region is the CTA's, so its
// address is uniform and cheap to rematerialise under the 96-register cap.
constexpr int CH_WPC = 1, CH_CTAS = 20;
template <bool MS>
__global__ void __launch_bounds__(32 * CH_WPC, CH_CTAS) lk_chain_kernel(LkChain c, stabgpu_flow_cfg cfg,
                                                                       unsigned* __restrict__ work, int smem_per_warp,
                                                                       const __grid_constant__ LkMaps maps) {
    extern __shared__ __align__(128) double lsm[];
    const int warp = CH_WPC == 1 ? 0 : threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* sys = lsm + (size_t)warp * smem_per_warp;
    uint8_t* stg = reinterpret_cast<uint8_t*>(sys + SYS_D);
    double* tg = sys + SYS_D + STG_D;
    int* nst_sh = reinterpret_cast<int*>(sys + 18);  // the segment's step count (MS)
    const unsigned total = (unsigned)c.nseg * (unsigned)c.max_pts;
    if (lane == 0) {  // the warp's TMA staging barrier
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(sys + SYS_TMA_BAR)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        *reinterpret_cast<int*>(sys + SYS_TMA_PHASE) = 0;
    }
    __syncwarp();
    const size_t plane = (size_t)c.nseg * c.max_pts;
    const double thr2 = dmul(cfg.fb_threshold, cfg.fb_threshold);
    while (true) {
        unsigned item = 0;
        if (lane == 0) item = atomicAdd(work, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= total) break;
        const int seg = (int)(item / (unsigned)c.max_pts), k = (int)(item % (unsigned)c.max_pts);
        int b0;  // detection frame of the segment (chunk-relative)
        if (MS) {
            b0 = seg_base(seg, c.R, c.F, c.nsps);
            // steps this segment may take, parked in shared memory (registers are full)
            const int nst = min(c.R, seg_end(seg, c.F, c.nsps, c.nframes) - 1 - b0);
            if (nst <= 0 || k >= c.npts[seg]) continue;
            if (lane == 0) *nst_sh = nst;
            __syncwarp();
        } else {
            b0 = seg * c.R;
            if (b0 + 1 >= c.nframes || k >= c.npts[seg]) continue;
        }
        const size_t slot = (size_t)seg * c.max_pts + k;
        double2 p = c.pts[slot], f = p;
        unsigned its = 0, blds = 0;
        bool ok0, ok1;
        double2 o0, o1;
        // round 0: step 1 forward (template in b0 at p, target b0+1).  Round
        // t >= 1: template in frame b0+t at f_t; tracker 0 = step t backward
        // into b0+t-1, tracker 1 = step t+1 forward into b0+t+1 (if any).
        // One call site keeps the kernel small (instruction cache).
        int t = 0, ft = b0, f0 = b0 + 1, f1 = -1;
        double2 q = p;
        while (true) {
            unsigned it0 = 0, it1 = 0;
            track_dual(c.pyr, ft, q.x, q.y, f0, f1, cfg, tg, stg, sys, ok0, ok1, o0, o1, it0, it1, blds,
                       maps.mask ? &maps : nullptr);
            its += it0;
            if (t == 0) {
                if (!ok0) break;
                f = o0;
            } else {
                bool keep = ok0;
                if (keep) {
                    const double ex = dsub(o0.x, p.x), ey = dsub(o0.y, p.y);
                    keep = dadd(dmul(ex, ex), dmul(ey, ey)) <= thr2;
                }
                if (!keep) break;
                if (lane == 0) c.alive[(size_t)(t - 1) * plane + slot] = 1;
                if (f1 < 0) break;
                its += it1;
                if (!ok1) break;
                p = f;
                f = o1;
            }
            ++t;  // also the count of forward tracks run
            if (lane == 0) c.pos[(size_t)(t - 1) * plane + slot] = f;
            if (MS)
                ++ft;  // b0 + t (b0 need not stay live)
            else
                ft = b0 + t;
            q = f;
            f0 = ft - 1;
            if (MS)
                f1 = t < *reinterpret_cast<volatile int*>(nst_sh) ? ft + 1 : -1;
            else
                f1 = (t < c.R && ft + 1 < c.nframes) ? ft + 1 : -1;
        }
        if (lane == 0 && c.iter_count) {
            atomicAdd(c.iter_count, (unsigned long long)its);
            atomicAdd(c.iter_count + 1, (unsigned long long)blds);
            atomicAdd(c.iter_count + 2, (unsigned long long)t);
        }
        __syncwarp();
    }
}

__global__ void lk_kernel(LkStep s, stabgpu_flow_cfg cfg, int warps_per_cta, int smem_per_warp) {
    extern __shared__ __align__(16) double lsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int seg = blockIdx.y;
    const int k = blockIdx.x * warps_per_cta + warp;
    const int fprev = s.frame0 + seg_base(seg, s.seg_len, s.F, s.nsps) + s.t - 1, fcur = fprev + 1;
    if (fcur >= s.frame0 + seg_end(seg, s.F, s.nsps, s.nframes - s.frame0)) return;
    if (k >= s.npts[seg]) return;
    const int r = cfg.window_radius, side = 2 * r + 1, es = 2 * r + 3;
    double* ext = lsm + (size_t)warp * smem_per_warp;
    double* tgx = ext + es * es;
    double* tgy = tgx + side * side;
    const size_t slot = (size_t)seg * s.max_pts + k;
    const double2 p = s.pts[slot];
    unsigned iters = 0, builds = 0;
    double fx = p.x, fy = p.y;
    bool keep;
    if (s.mode == 2) {  // weed only: p is the cur point, ref the prev point
        double bx, by;
        keep = track_warp(s.pyr, fcur, fprev, p.x, p.y, cfg, ext, tgx, tgy, bx, by, iters, builds);
        if (keep) {
            const double2 q = s.ref[slot];
            const double ex = dsub(bx, q.x), ey = dsub(by, q.y);
            keep = dadd(dmul(ex, ex), dmul(ey, ey)) <= dmul(cfg.fb_threshold, cfg.fb_threshold);
        }
    } else {
        keep = track_warp(s.pyr, fprev, fcur, p.x, p.y, cfg, ext, tgx, tgy, fx, fy, iters, builds);
        if (keep && s.mode == 1) {  // weed_tracks: backward re-track and fb test
            double bx, by;
            keep = track_warp(s.pyr, fcur, fprev, fx, fy, cfg, ext, tgx, tgy, bx, by, iters, builds);
            if (keep) {
                const double ex = dsub(bx, p.x), ey = dsub(by, p.y);
                keep = dadd(dmul(ex, ex), dmul(ey, ey)) <= dmul(cfg.fb_threshold, cfg.fb_threshold);
            }
        }
    }
    if (lane == 0) {
        s.fwd[slot] = make_double2(fx, fy);
        s.keep[slot] = keep ? 1 : 0;
        if (s.iter_count) {
            atomicAdd(s.iter_count, (unsigned long long)iters);
            atomicAdd(s.iter_count + 1, (unsigned long long)builds);
            atomicAdd(s.iter_count + 2, 1ull);
        }
    }
}

// Ordered compaction per segment (one CTA each).
__global__ void compact_kernel(LkStep s, double2* __restrict__ next_pts, int* __restrict__ next_n,
                               double2* __restrict__ trk_prev, double2* __restrict__ trk_cur,
                               int* __restrict__ trk_n, int trk_frame0) {
    __shared__ int warp_tot[32];
    __shared__ int base;
    const int seg = blockIdx.x;
    const int fcur = s.frame0 + seg_base(seg, s.seg_len, s.F, s.nsps) + s.t;
    if (fcur >= s.frame0 + seg_end(seg, s.F, s.nsps, s.nframes - s.frame0)) return;
    const int n = s.npts[seg];
    const int tf = fcur - trk_frame0;  // TrackSet slot of frame fcur
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
        const int k = c0 + threadIdx.x;
        const size_t slot = (size_t)seg * s.max_pts + k;
        const bool kp = k < n && s.keep[slot];
        const unsigned b = __ballot_sync(0xffffffffu, kp);
        if (lane == 0) warp_tot[wid] = __popc(b);
        __syncthreads();
        int off = base;
        for (int w2 = 0; w2 < wid; ++w2) off += warp_tot[w2];
        off += __popc(b & ((1u << lane) - 1));
        if (kp) {
            const double2 c = s.fwd[slot];
            const size_t o = (size_t)seg * s.max_pts + off;
            next_pts[o] = c;
            const size_t to = (size_t)tf * s.max_pts + off;
            trk_prev[to] = s.pts[slot];
            trk_cur[to] = c;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w2 = 0; w2 < nw; ++w2) t += warp_tot[w2];
            base += t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        next_n[seg] = base;
        trk_n[tf] = base;
    }
}

}  // namespace

void launch_lk(const LkStep& s, const stabgpu_flow_cfg& cfg, cudaStream_t st) {
    if (s.nseg <= 0 || s.max_pts <= 0) return;
    const int r = cfg.window_radius, side = 2 * r + 1, es = 2 * r + 3;
    if (r <= 15) {
        // doubles: template gradients {gx, gy}[side][32] + the staged window (bytes)
        const int per_warp = lk_per_warp(side);
        const int wpc = 4;
        const size_t smem = (size_t)wpc * per_warp * sizeof(double);
        ensure_smem(lk_fast_kernel, smem);
        const int sms = sm_count(), per_sm = blocks_per_sm(lk_fast_kernel, wpc * 32, smem);
        cudaMemsetAsync(s.work, 0, sizeof(unsigned), st);
        const long long items = (long long)s.nseg * s.max_pts;
        const long long want = (items + wpc - 1) / wpc;
        const int grid = (int)std::min<long long>(want, (long long)sms * std::max(per_sm, 1));
        lk_fast_kernel<<<grid, wpc * 32, smem, st>>>(s, cfg, s.work, per_warp);
        return;
    }
    const int per_warp = es * es + 2 * side * side;  // doubles
    int wpc = (int)((100 * 1024) / (per_warp * sizeof(double)));
    wpc = max(1, min(8, wpc));
    const size_t smem = (size_t)wpc * per_warp * sizeof(double);
    ensure_smem(lk_kernel, smem);
    dim3 grid((s.max_pts + wpc - 1) / wpc, s.nseg);
    lk_kernel<<<grid, wpc * 32, smem, st>>>(s, cfg, wpc, per_warp);
}

void launch_lk_chain(const LkChain& c, const stabgpu_flow_cfg& cfg, cudaStream_t st) {
    if (c.nseg <= 0 || c.max_pts <= 0) return;
    const int side = 2 * cfg.window_radius + 1;
    const int per_warp = lk_per_warp(side);  // doubles (even: 16 B aligned)
    const int wpc = CH_WPC;
    const size_t smem = (size_t)wpc * per_warp * sizeof(double);
    const bool multi = c.nsps != c.nseg;  // several streams in the chunk
    auto kern = multi ? lk_chain_kernel<true> : lk_chain_kernel<false>;
    ensure_smem(kern, smem);
    const int sms = sm_count(), per_sm = blocks_per_sm(kern, wpc * 32, smem);
    cudaMemsetAsync(c.work, 0, sizeof(unsigned), st);
    cudaMemsetAsync(c.alive, 0, (size_t)c.steps * c.nseg * c.max_pts, st);
    const long long items = (long long)c.nseg * c.max_pts;
    const long long want = (items + wpc - 1) / wpc;
    const int grid = (int)std::min<long long>(want, (long long)sms * std::max(per_sm, 1));
    // TMA maps of the levels whose frames are a regular 16-byte aligned 3D array
    LkMaps maps;
    memset(&maps, 0, sizeof maps);
    for (int l = 0; l < c.pyr.levels; ++l) {
        const size_t fs = (size_t)c.pyr.w[l] * c.pyr.h[l];
        if (c.pyr.stride[l] == fs && (c.pyr.w[l] % 16) == 0 &&
            encode_u8_3d(&maps.m[l], c.pyr.lvl[l], c.pyr.w[l], c.pyr.h[l], c.nframes, fs, SM_PITCH, SM_ROWS))
            maps.mask |= 1u << l;
    }
    kern<<<grid, wpc * 32, smem, st>>>(c, cfg, c.work, per_warp, maps);
}

void launch_compact(const LkStep& s, double2* next_pts, int* next_n, double2* trk_prev,
                    double2* trk_cur, int* trk_n, int trk_frame0, cudaStream_t st) {
    if (s.nseg <= 0) return;
    compact_kernel<<<s.nseg, 256, 0, st>>>(s, next_pts, next_n, trk_prev, trk_cur, trk_n, trk_frame0);
}

}  // namespace stabgpu
