// k_compose.cu — K8: fused inverse-similarity warp + crop/resize of every
// plane of a frame, batched over frames.  Bit-exact with the reference.
//
// Reference: sample_bilinear (image_ops.cpp:98-113), warp_similarity
// (115-134), crop_resize (136-159), compose_plane (165-202),
// compose_stabilized (206-219).
//
// One CTA owns a 64x32 output tile of one frame and all of its planes:
//   1. the tile's source footprint (inverse-mapped bounding box) of each
//      plane is staged in shared memory with coalesced 32-bit loads;
//   2. luma: the warped-and-rounded pixels W the crop stage reads (a <=66x34
//      tile) are recreated in shared memory, then crop-resampled (the
//      reference rounds twice, image_ops.cpp:209); chroma (4:4:4: same tile)
//      is one inverse map per pixel, both planes sharing coordinates;
//   3. the output tile is written with 16-byte streaming stores.
// So HBM sees one read and one write per plane byte.
//
// Exactness without fp64 per pixel.  Coordinates are carried in fixed point
// (16.48 in the per-frame tables, 32.32 in the TMA kernel's row loops), the
// bilinear blend in fp32.  Each decision the reference takes — integer part
// of a coordinate, in-bounds test, lround of the blended value — is taken on
// the fast path only when the fast value is provably on the same side of the
// decision boundary (coordinate error < 5e-9 px against a 2.4e-7 px guard;
// value error <= 6.4e-5 against a 7e-5 guard); away from the frame edges the
// coordinate guard is not needed at all (see the 32.32 section below).
// Per-row fixed-point starts (16.48) and the crop tables are
// computed once per frame / geometry by compose_prep_kernel, so a tile's
// setup is a handful of loads.  Otherwise the pixel is queued and recomputed
// with the reference's own fp64 arithmetic — for luma including the
// reference's sequential row walk (sx += c, image_ops.cpp:124-131), which
// fl_walk (walk.h) reproduces bit for bit in closed form.  About 0.05% of
// pixels take the exact path.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cstring>

#include "colour.cuh"
#include "common.cuh"
#include "kernels.cuh"
#include "walk.h"

namespace stabgpu {

namespace {

constexpr int TW = 64, TH = 32;          // output tile
constexpr int NT = 256;                  // threads per CTA
constexpr int NW = NT / 32;              // warps per CTA (row stride of the warp-per-row loops)
constexpr int WTW = 72, WTH = 36;        // warped-luma tile (<= 66 x 34 used)
constexpr int SRC_W = 128, SRC_H = 80;   // staged source capacity per plane
constexpr int QCAP = 1024;               // exact-path queue
constexpr uint32_t GUARD = 1024;         // coordinate guard, units of 2^-32 px
constexpr float VGUARD = 7.0e-5f;        // blended-value guard (the fast error is <= 6.35e-5)
constexpr double FIX48 = 281474976710656.0;  // 2^48

struct CropGeom {
    int mx, my;
    double step_x, step_y;
};

__host__ __device__ inline CropGeom crop_geom(int w, int h, double crop) {
    CropGeom g;
    g.mx = (int)llround(crop * w);
    g.my = (int)llround(crop * h);
    const int cw = w - 2 * g.mx, ch = h - 2 * g.my;
    g.step_x = w > 1 ? (double)(cw - 1) / (w - 1) : 0.0;
    g.step_y = h > 1 ? (double)(ch - 1) / (h - 1) : 0.0;
    return g;
}

// Per-launch tables (compose_prep_kernel).
struct Tables {
    long long *rxf, *ryf;  // [frames][h]  luma warp row starts at u = 0 (16.48)
    long long *pxf, *pyf;  // [frames][ch] chroma source coords of (0, y) (16.48)
    int *cx0, *cy0;        // crop_resize integer parts per column [w] / row [h]
    double *cfx, *cfy;     // and fractions
    int4* tiles;           // [frames][tiles] TMA tile parameters (TileParams), or null
    int h, ch;
};

// Per-tile parameters of the TMA kernel, precomputed one thread per tile:
// W region and the TMA box origins of the luma / chroma source footprints.
struct TileParams {
    int u0, v0, nu, nv;
    int lbx, lby, cbx, cby;
    int lfit, cfit, pad0, pad1;
};
static_assert(sizeof(TileParams) == 48, "TileParams is 3 x int4");

struct Smem {
    uint8_t src[3][SRC_H * SRC_W];
    uint8_t wt[WTH][WTW];
    uint8_t out[3][TH][TW];
    double cfx[TW], cfy[TH];
    float cfxf[TW], cfyf[TH];
    int cx0[TW], cy0[TH];
    long long sxf[WTH], syf[WTH];  // luma row starts of the W tile rows
    long long pxf[TH], pyf[TH];    // chroma rows of the tile
    int bbox[3][4];
    int staged[3];
    int qn;
    unsigned q[QCAP];
};

__device__ __forceinline__ bool near_int(uint32_t f) { return f < GUARD || f > 0xFFFFFFFFu - GUARD; }

// 0.32 fraction -> fp32 within 2^-24: top 23 bits, centred on the dropped
// bits ((1 + m 2^-23) - (1 - 2^-24) is exact).
__device__ __forceinline__ float frac_f(uint32_t f) {
    return __uint_as_float(0x3F800000u | (f >> 9)) - 0.99999994f;
}

// uint8 -> 256 + b as fp32 in one LEA (0x43800000 | b << 15), no I2F.
__device__ __forceinline__ float b256(uint32_t b) { return __uint_as_float(0x43800000u | (b << 15)); }

// fast bilinear (sample_bilinear's blend) in the 256-offset fp32 domain +
// lround; -1 when the rounding decision is within the error guard of a .5
// tie.  Error budget against the reference's fp64 value: in [256, 512)
// differences are exact (Sterbenz) and the three fma roundings contribute
// <= 2 * 2^-16 = 3.05e-5 to v (top and bot each <= 2^-16, weighted by 1-fy
// and fy, plus v's own); the fractions are within 2^-24 of the coordinate's
// (the crop's double table fractions within 2^-25), which is itself within
// 5e-9 px of the reference's, and |dv/dfx|, |dv/dfy| <= 255 — across an
// integer too, where the blend is continuous — so <= 2 * 255 * 6.46e-8 =
// 3.3e-5.  Total <= 6.35e-5 < VGUARD = 7e-5; |v - round(v)| is exact in fp32.
__device__ __forceinline__ int blend_round(uint32_t a, uint32_t b, uint32_t c, uint32_t d, float fx,
                                           float fy) {
    const float fa = b256(a), fc = b256(c);
    const float top = fmaf(fx, b256(b) - fa, fa);
    const float bot = fmaf(fx, b256(d) - fc, fc);
    const float v = fmaf(fy, bot - top, top);  // 256 + value
    const float m = v + 8388608.0f;             // nearest integer (ties are guarded below)
    const float dv = v - (m - 8388608.0f);      // in [-0.5, 0.5]
    if (fabsf(dv) > 0.5f - VGUARD) return -1;
    return __float_as_int(m) & 0xFF;            // (256 + k) mod 256 == k, k <= 255
}

// One fast-path sample of plane q (pitch, origin bx0/by0) at 16.48 (X, Y).
// Returns the byte, `out` outside [0, w-1] x [0, h-1] (lim = w-2 / h-2 on
// the integer part), or -1 when a decision is not certain.
template <typename P>
__device__ __forceinline__ int sample_fast(P q, int pitch, int bx0, int by0, unsigned limx,
                                           unsigned limy, long long X, long long Y, int out) {
    const uint32_t fxs = (uint32_t)(X >> 16), fys = (uint32_t)(Y >> 16);
    if (near_int(fxs) || near_int(fys)) return -1;
    const int ix = (int)(X >> 48), iy = (int)(Y >> 48);
    if ((unsigned)ix > limx || (unsigned)iy > limy) return out;
    const int o = (iy - by0) * pitch + (ix - bx0);
    return blend_round(q[o], q[o + 1], q[o + pitch], q[o + pitch + 1], frac_f(fxs), frac_f(fys));
}

// Two planes sharing one coordinate (chroma): packed result b | r << 16
template <typename P>
__device__ __forceinline__ int sample_fast2(P q1, P q2, int pitch, int bx0, int by0, unsigned limx,
                                            unsigned limy, long long X, long long Y, int out) {
    const uint32_t fxs = (uint32_t)(X >> 16), fys = (uint32_t)(Y >> 16);
    if (near_int(fxs) || near_int(fys)) return -1;
    const int ix = (int)(X >> 48), iy = (int)(Y >> 48);
    if ((unsigned)ix > limx || (unsigned)iy > limy) return out | (out << 16);
    const int o = (iy - by0) * pitch + (ix - bx0);
    const float fx = frac_f(fxs), fy = frac_f(fys);
    const int vb = blend_round(q1[o], q1[o + 1], q1[o + pitch], q1[o + pitch + 1], fx, fy);
    const int vr = blend_round(q2[o], q2[o + 1], q2[o + pitch], q2[o + pitch + 1], fx, fy);
    return (vb < 0 || vr < 0) ? -1 : (vb | (vr << 16));
}

// Stages rows [y0, y1] x cols [x0, x1] of a plane (already clipped): warp per
// row, lanes over 32-bit words.
__device__ void stage(const uint8_t* __restrict__ g, int w, int x0, int y0, int x1, int y1,
                      uint8_t* dst, int* bb, int* staged) {
    const int xa = x0 & ~3;
    const int nwords = ((x1 - xa) >> 2) + 1;
    const int rows = y1 - y0 + 1;
    const bool fits = nwords * 4 <= SRC_W && rows <= SRC_H && x1 >= x0 && y1 >= y0;
    if (threadIdx.x == 0) {
        bb[0] = xa;
        bb[1] = y0;
        *staged = fits;
    }
    if (!fits) return;
    const bool aligned = ((w & 3) == 0) && ((reinterpret_cast<uintptr_t>(g) & 3) == 0) &&
                         (xa + nwords * 4 <= w);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (aligned) {
        for (int r = warp; r < rows; r += NT / 32) {
            const uint32_t* grow = reinterpret_cast<const uint32_t*>(g + (size_t)(y0 + r) * w + xa);
            uint32_t* srow = reinterpret_cast<uint32_t*>(dst + r * SRC_W);
            for (int c = lane; c < nwords; c += 32) srow[c] = __ldg(grow + c);
        }
    } else {
        const int cols = nwords * 4;
        for (int r = warp; r < rows; r += NT / 32)
            for (int c = lane; c < cols; c += 32)
                dst[r * SRC_W + c] = __ldg(g + (size_t)(y0 + r) * w + min(xa + c, w - 1));
    }
}

__device__ __forceinline__ void push_q(int& qn, unsigned* q, unsigned item) {
    const int k = atomicAdd(&qn, 1);
    if (k < QCAP) q[k] = item;
}

__device__ __forceinline__ void push(Smem& S, unsigned item) {
    const int k = atomicAdd(&S.qn, 1);
    if (k < QCAP) S.q[k] = item;
}

// luma warp row start (image_ops.cpp:124-125), exact reference arithmetic
__device__ __forceinline__ void row_start(const FramePlan& p, int v, double& rx, double& ry) {
    rx = dadd(dmul(p.c, dsub(0.0, p.tx)), dmul(p.sn, dsub((double)v, p.ty)));
    ry = dadd(dmul(-p.sn, dsub(0.0, p.tx)), dmul(p.c, dsub((double)v, p.ty)));
}

struct ChromaMap {  // compose_plane constants (image_ops.cpp:167-177)
    double fxl, fyl;
    bool crop;
};

__device__ __forceinline__ ChromaMap chroma_map(int w, int h, int cw, int ch, const CropGeom& g) {
    return ChromaMap{(double)w / cw, (double)h / ch, g.mx != 0 || g.my != 0};
}

// compose_plane source coordinates of chroma pixel (x, y), reference order
__device__ __forceinline__ void chroma_coords(const FramePlan& p, const CropGeom& g,
                                              const ChromaMap& m, int x, int y, double& px,
                                              double& py) {
    double lx = dsub(dmul(dadd((double)x, 0.5), m.fxl), 0.5);
    double ly = dsub(dmul(dadd((double)y, 0.5), m.fyl), 0.5);
    if (m.crop) {
        lx = dadd((double)g.mx, dmul(lx, g.step_x));
        ly = dadd((double)g.my, dmul(ly, g.step_y));
    }
    const double dx = dsub(lx, p.tx), dy = dsub(ly, p.ty);
    const double qx = dadd(dmul(p.c, dx), dmul(p.sn, dy));
    const double qy = dadd(dmul(-p.sn, dx), dmul(p.c, dy));
    px = dsub(ddiv(dadd(qx, 0.5), m.fxl), 0.5);
    py = dsub(ddiv(dadd(qy, 0.5), m.fyl), 0.5);
}

// Exact luma W pixel.  Level 1: the direct fp64 coordinates rx + u*c differ
// from the reference's walked ones by <= (u+2) half-ulps, so unless a
// coordinate sits that close to an integer / the frame edge, or the fp64
// blend that close to a .5 tie, the direct result IS the reference result.
// Level 2 (about once per two 1080p frames): fl_walk, the exact walk.
// `fetch(x, y)` reads the source frame (global, or the staged TMA box).
template <typename F>
__device__ uint8_t w_exact_f(F fetch, int w, int h, const FramePlan& p, int u, int v) {
    double rx, ry;
    row_start(p, v, rx, ry);
    const double sx = dadd(rx, dmul((double)u, p.c)), sy = dsub(ry, dmul((double)u, p.sn));
    const double mag = fmax(fmax(fabs(sx), fabs(sy)), fmax(fabs(rx), fabs(ry))) + fabs((double)u) + 2.0;
    const double tol = ldexp(mag, -52) * ((double)u + 4.0);
    bool sure = true;
    const double fxx = sx - floor(sx), fyy = sy - floor(sy);
    if (fmin(fxx, 1.0 - fxx) <= tol || fabs(sx) <= tol || fabs(sx - ((double)w - 1.0)) <= tol) sure = false;
    if (fmin(fyy, 1.0 - fyy) <= tol || fabs(sy) <= tol || fabs(sy - ((double)h - 1.0)) <= tol) sure = false;
    if (sure) {
        const double val = bilinear_f(fetch, w, h, sx, sy);
        const double fr = val - floor(val);
        if (fabs(fr - 0.5) > 255.0 * 4.0 * tol + 1e-9) return round_u8(val);
    }
    return round_u8(bilinear_f(fetch, w, h, fl_walk(rx, p.c, u), fl_walk(ry, -p.sn, u)));
}

__device__ uint8_t w_exact(const uint8_t* __restrict__ g, int w, int h, const FramePlan& p, int u, int v) {
    return w_exact_f([=](int x, int y) { return (double)g[(size_t)y * w + x]; }, w, h, p, u, v);
}

__device__ __forceinline__ uint8_t crop_exact_t(const uint8_t (*wt)[WTW], const int* cx0,
                                                const int* cy0, const double* cfx,
                                                const double* cfy, int r, int c, int u0, int v0,
                                                int w, int h) {
    const int x0 = cx0[c], y0 = cy0[r];
    const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
    const double a = wt[y0 - v0][x0 - u0], b = wt[y0 - v0][x1 - u0];
    const double cc = wt[y1 - v0][x0 - u0], d = wt[y1 - v0][x1 - u0];
    const double top = dadd(a, dmul(cfx[c], dsub(b, a)));
    const double bot = dadd(cc, dmul(cfx[c], dsub(d, cc)));
    return round_u8(dadd(top, dmul(cfy[r], dsub(bot, top))));
}

__device__ __forceinline__ uint8_t crop_exact(const Smem& S, int r, int c, int u0, int v0, int w,
                                              int h) {
    const int x0 = S.cx0[c], y0 = S.cy0[r];
    const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
    const double a = S.wt[y0 - v0][x0 - u0], b = S.wt[y0 - v0][x1 - u0];
    const double cc = S.wt[y1 - v0][x0 - u0], d = S.wt[y1 - v0][x1 - u0];
    const double top = dadd(a, dmul(S.cfx[c], dsub(b, a)));
    const double bot = dadd(cc, dmul(S.cfx[c], dsub(d, cc)));
    return round_u8(dadd(top, dmul(S.cfy[r], dsub(bot, top))));
}

template <typename F1, typename F2>
__device__ __forceinline__ void chroma_exact_f(const FramePlan& p, const CropGeom& g, const ChromaMap& cm,
                                               F1 f1, F2 f2, int cw, int ch, int x, int y, uint8_t& ob,
                                               uint8_t& orr) {
    double px, py;
    chroma_coords(p, g, cm, x, y, px, py);
    ob = orr = 128;
    if (px >= 0.0 && py >= 0.0 && px <= (double)cw - 1.0 && py <= (double)ch - 1.0) {
        ob = round_u8(bilinear_f(f1, cw, ch, px, py));
        orr = round_u8(bilinear_f(f2, cw, ch, px, py));
    }
}

__device__ __forceinline__ void chroma_exact(const FramePlan& p, const CropGeom& g,
                                             const ChromaMap& cm, const uint8_t* gcb,
                                             const uint8_t* gcr, int cw, int ch, int x, int y,
                                             uint8_t& ob, uint8_t& orr) {
    chroma_exact_f(p, g, cm, [=](int xx, int yy) { return (double)gcb[(size_t)yy * cw + xx]; },
                   [=](int xx, int yy) { return (double)gcr[(size_t)yy * cw + xx]; }, cw, ch, x, y, ob, orr);
}

// Per-frame row tables + (frame 0) crop tables.
__global__ void compose_prep_kernel(const FramePlan* __restrict__ plan, int w, int h, int cw, int ch,
                                    CropGeom g, Tables T) {
    const int f = blockIdx.y;
    const FramePlan p = plan[f];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < h) {
        double rx, ry;
        row_start(p, i, rx, ry);
        T.rxf[(size_t)f * h + i] = __double2ll_rn(dmul(rx, FIX48));
        T.ryf[(size_t)f * h + i] = __double2ll_rn(dmul(ry, FIX48));
    }
    if (T.pxf && i < ch) {
        double px, py;
        chroma_coords(p, g, chroma_map(w, h, cw, ch, g), 0, i, px, py);
        T.pxf[(size_t)f * ch + i] = __double2ll_rn(dmul(px, FIX48));
        T.pyf[(size_t)f * ch + i] = __double2ll_rn(dmul(py, FIX48));
    }
    if (f == 0) {
        if (i < w) {  // crop_resize columns (image_ops.cpp:150-155)
            const double sx = dadd((double)g.mx, dmul((double)i, g.step_x));
            T.cx0[i] = (int)sx;
            T.cfx[i] = dsub(sx, (double)(int)sx);
        }
        if (i < h) {
            const double sy = dadd((double)g.my, dmul((double)i, g.step_y));
            T.cy0[i] = (int)sy;
            T.cfy[i] = dsub(sy, (double)(int)sy);
        }
    }
}

template <bool LUMA, bool CHROMA>
__global__ void __launch_bounds__(NT) compose_kernel(PlaneBatch Y, PlaneBatch CB, PlaneBatch CR,
                                                     const FramePlan* __restrict__ plan, CropGeom g,
                                                     Tables T, int tiles_x, uint8_t* __restrict__ oY,
                                                     uint8_t* __restrict__ oCB,
                                                     uint8_t* __restrict__ oCR) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int f = blockIdx.y;
    const FramePlan p = plan[f];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = LUMA ? Y.w : CB.w, H = LUMA ? Y.h : CB.h;
    const int X0 = (blockIdx.x % tiles_x) * TW, Y0 = (blockIdx.x / tiles_x) * TH;
    const int nx = min(TW, W - X0), ny = min(TH, H - Y0);
    const bool identity = g.mx == 0 && g.my == 0;
    const int w = Y.w, h = Y.h, cw = CB.w, ch = CB.h;
    const uint8_t* gy = LUMA ? Y.base + (size_t)f * Y.stride : nullptr;
    const uint8_t* gcb = CHROMA ? CB.base + (size_t)f * CB.stride : nullptr;
    const uint8_t* gcr = CHROMA ? CR.base + (size_t)f * CR.stride : nullptr;
    // ------------------------------------------------------------ setup (loads only)
    int u0 = X0, v0 = Y0, nu = nx, nv = ny;
    if (LUMA && !identity) {
        u0 = __ldg(T.cx0 + X0);
        v0 = __ldg(T.cy0 + Y0);
        nu = min(__ldg(T.cx0 + X0 + nx - 1) + 1, w - 1) - u0 + 1;
        nv = min(__ldg(T.cy0 + Y0 + ny - 1) + 1, h - 1) - v0 + 1;
    }
    if (tid == 0) S.qn = 0;
    if (LUMA) {
        if (!identity) {
            if (tid < nx) {
                S.cx0[tid] = __ldg(T.cx0 + X0 + tid);
                S.cfx[tid] = __ldg(T.cfx + X0 + tid);
                S.cfxf[tid] = (float)S.cfx[tid];
            } else if (tid >= 64 && tid < 64 + ny) {
                S.cy0[tid - 64] = __ldg(T.cy0 + Y0 + tid - 64);
                S.cfy[tid - 64] = __ldg(T.cfy + Y0 + tid - 64);
                S.cfyf[tid - 64] = (float)S.cfy[tid - 64];
            }
        }
        if (tid >= 128 && tid < 128 + nv) {
            S.sxf[tid - 128] = __ldg(T.rxf + (size_t)f * h + v0 + tid - 128);
            S.syf[tid - 128] = __ldg(T.ryf + (size_t)f * h + v0 + tid - 128);
        }
        if (warp == 7 && lane < 4) {  // luma footprint of the W tile: 4 corners
            const int u = u0 + ((lane & 1) ? nu - 1 : 0), v = v0 + ((lane & 2) ? nv - 1 : 0);
            const long long X = __ldg(T.rxf + (size_t)f * h + v) + (long long)u * p.cf;
            const long long Yv = __ldg(T.ryf + (size_t)f * h + v) - (long long)u * p.snf;
            int xmn = (int)(X >> 48), xmx = xmn, ymn = (int)(Yv >> 48), ymx = ymn;
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                xmn = min(xmn, __shfl_xor_sync(0xFu, xmn, o));
                xmx = max(xmx, __shfl_xor_sync(0xFu, xmx, o));
                ymn = min(ymn, __shfl_xor_sync(0xFu, ymn, o));
                ymx = max(ymx, __shfl_xor_sync(0xFu, ymx, o));
            }
            if (lane == 0) {
                S.bbox[0][0] = max(0, xmn - 1);
                S.bbox[0][1] = max(0, ymn - 1);
                S.bbox[0][2] = min(w - 1, xmx + 2);
                S.bbox[0][3] = min(h - 1, ymx + 2);
            }
        }
    }
    if (CHROMA) {
        if (tid >= 192 && tid < 192 + ny) {
            S.pxf[tid - 192] = __ldg(T.pxf + (size_t)f * ch + Y0 + tid - 192);
            S.pyf[tid - 192] = __ldg(T.pyf + (size_t)f * ch + Y0 + tid - 192);
        }
        if (warp == 7 && lane >= 4 && lane < 8) {  // chroma footprint: 4 corners
            const int k = lane - 4;
            const int x = X0 + ((k & 1) ? nx - 1 : 0), y = Y0 + ((k & 2) ? ny - 1 : 0);
            const long long X = __ldg(T.pxf + (size_t)f * ch + y) + (long long)x * p.kxx;
            const long long Yv = __ldg(T.pyf + (size_t)f * ch + y) + (long long)x * p.kyx;
            int xmn = (int)(X >> 48), xmx = xmn, ymn = (int)(Yv >> 48), ymx = ymn;
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                xmn = min(xmn, __shfl_xor_sync(0xF0u, xmn, o));
                xmx = max(xmx, __shfl_xor_sync(0xF0u, xmx, o));
                ymn = min(ymn, __shfl_xor_sync(0xF0u, ymn, o));
                ymx = max(ymx, __shfl_xor_sync(0xF0u, ymx, o));
            }
            if (k == 0) {
                S.bbox[1][0] = max(0, xmn - 1);
                S.bbox[1][1] = max(0, ymn - 1);
                S.bbox[1][2] = min(cw - 1, xmx + 2);
                S.bbox[1][3] = min(ch - 1, ymx + 2);
            }
        }
    }
    __syncthreads();
    // ------------------------------------------------------------ staging
    int bb0[4], bb1[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        bb0[j] = S.bbox[0][j];
        bb1[j] = S.bbox[1][j];
    }
    __syncthreads();
    if (LUMA) stage(gy, w, bb0[0], bb0[1], bb0[2], bb0[3], S.src[0], S.bbox[0], &S.staged[0]);
    if (CHROMA) {
        stage(gcb, cw, bb1[0], bb1[1], bb1[2], bb1[3], S.src[1], S.bbox[1], &S.staged[1]);
        stage(gcr, cw, bb1[0], bb1[1], bb1[2], bb1[3], S.src[2], S.bbox[2], &S.staged[2]);
    }
    __syncthreads();
    // ------------------------------------------------------------ luma W tile
    if (LUMA) {
        uint8_t* wdst = identity ? &S.out[0][0][0] : &S.wt[0][0];
        const int wp = identity ? TW : WTW;
        const unsigned limx = (unsigned)(w - 2), limy = (unsigned)(h - 2);
        const bool stg = S.staged[0];
        const int bx0 = S.bbox[0][0], by0 = S.bbox[0][1];
        const long long CF = p.cf, SNF = p.snf;
        // warp per row, 2 adjacent pixels per lane (64 columns), tail columns after
        for (int r = warp; r < nv; r += NT / 32) {
            const long long SXr = S.sxf[r], SYr = S.syf[r];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int c = 2 * lane + k;
                if (c >= nu) break;
                const long long u = u0 + c;
                const long long SX = SXr + u * CF, SY = SYr - u * SNF;
                const int val = stg ? sample_fast(&S.src[0][0], SRC_W, bx0, by0, limx, limy, SX, SY, 0)
                                    : sample_fast(gy, w, 0, 0, limx, limy, SX, SY, 0);
                if (val < 0) push(S, (unsigned)(r * nu + c));
                else wdst[r * wp + c] = (uint8_t)val;
            }
        }
        for (int i = tid; i < (nu - 64) * nv; i += NT) {  // columns 64.. (at most 2)
            const int r = i / (nu - 64), c = 64 + i - r * (nu - 64);
            const long long u = u0 + c;
            const long long SX = S.sxf[r] + u * CF, SY = S.syf[r] - u * SNF;
            const int val = stg ? sample_fast(&S.src[0][0], SRC_W, bx0, by0, limx, limy, SX, SY, 0)
                                : sample_fast(gy, w, 0, 0, limx, limy, SX, SY, 0);
            if (val < 0) push(S, (unsigned)(r * nu + c));
            else wdst[r * wp + c] = (uint8_t)val;
        }
        __syncthreads();
        const int nq = S.qn;
        if (nq <= QCAP) {
            for (int k = tid; k < nq; k += NT) {  // exact reference path
                const int i = (int)(S.q[k] & 0x3FFFFFFF), r = i / nu, c = i - r * nu;
                wdst[r * wp + c] = w_exact(gy, w, h, p, u0 + c, v0 + r);
            }
        } else {  // overflow: every pixel exactly (never seen in practice)
            for (int i = tid; i < nu * nv; i += NT) {
                const int r = i / nu, c = i - r * nu;
                wdst[r * wp + c] = w_exact(gy, w, h, p, u0 + c, v0 + r);
            }
        }
        __syncthreads();
        if (tid == 0) S.qn = 0;
        __syncthreads();
        // ---- crop_resize of the warped tile (image_ops.cpp:151-157)
        if (!identity) {
            int x0[2], x1[2];
            float fxv[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int c = min(2 * lane + k, nx - 1);
                x0[k] = S.cx0[c] - u0;
                x1[k] = min(S.cx0[c] + 1, w - 1) - u0;
                fxv[k] = S.cfxf[c];
            }
            for (int r = warp; r < ny; r += NT / 32) {
                const int y0 = S.cy0[r] - v0, y1 = min(S.cy0[r] + 1, h - 1) - v0;
                const float fy = S.cfyf[r];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int c = 2 * lane + k;
                    if (c >= nx) break;
                    const int val = blend_round(S.wt[y0][x0[k]], S.wt[y0][x1[k]], S.wt[y1][x0[k]],
                                                S.wt[y1][x1[k]], fxv[k], fy);
                    if (val < 0) push(S, (1u << 30) | (unsigned)(r * nx + c));
                    else S.out[0][r][c] = (uint8_t)val;
                }
            }
        }
    }
    // ------------------------------------------------------------ chroma
    const ChromaMap cm = chroma_map(w, h, cw, ch, g);
    if (CHROMA) {
        const unsigned limx = (unsigned)(cw - 2), limy = (unsigned)(ch - 2);
        const bool stg = S.staged[1] && S.staged[2];
        const int bx0 = S.bbox[1][0], by0 = S.bbox[1][1];
        const long long KX = p.kxx, KY = p.kyx;
        for (int r = warp; r < ny; r += NT / 32) {
            const long long PXr = S.pxf[r], PYr = S.pyf[r];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int c = 2 * lane + k;
                if (c >= nx) break;
                const long long x = X0 + c;
                const long long PX = PXr + x * KX, PY = PYr + x * KY;
                const int v = stg ? sample_fast2(&S.src[1][0], &S.src[2][0], SRC_W, bx0, by0, limx,
                                                 limy, PX, PY, 128)
                                  : sample_fast2(gcb, gcr, cw, 0, 0, limx, limy, PX, PY, 128);
                if (v < 0) {
                    push(S, (2u << 30) | (unsigned)(r * nx + c));
                } else {
                    S.out[1][r][c] = (uint8_t)(v & 0xFF);
                    S.out[2][r][c] = (uint8_t)(v >> 16);
                }
            }
        }
    }
    __syncthreads();
    {
        const int nq = S.qn;
        if (nq <= QCAP) {
            for (int k = tid; k < nq; k += NT) {
                const unsigned item = S.q[k];
                const int kind = item >> 30, i = (int)(item & 0x3FFFFFFF);
                const int r = i / nx, c = i - r * nx;
                if (LUMA && kind == 1) {
                    S.out[0][r][c] = crop_exact(S, r, c, u0, v0, w, h);
                } else if (CHROMA && kind == 2) {
                    chroma_exact(p, g, cm, gcb, gcr, cw, ch, X0 + c, Y0 + r, S.out[1][r][c],
                                 S.out[2][r][c]);
                }
            }
        } else {  // overflow: exact path for the whole tile
            for (int i = tid; i < nx * ny; i += NT) {
                const int r = i / nx, c = i - r * nx;
                if (LUMA && !identity) S.out[0][r][c] = crop_exact(S, r, c, u0, v0, w, h);
                if (CHROMA)
                    chroma_exact(p, g, cm, gcb, gcr, cw, ch, X0 + c, Y0 + r, S.out[1][r][c],
                                 S.out[2][r][c]);
            }
        }
    }
    __syncthreads();
    // ------------------------------------------------------------ store
    for (int k = (LUMA ? 0 : 1); k < (CHROMA ? 3 : 1); ++k) {
        uint8_t* base = k == 0 ? oY + (size_t)f * Y.stride
                               : (k == 1 ? oCB + (size_t)f * CB.stride : oCR + (size_t)f * CR.stride);
        const int pw = k == 0 ? w : cw;
        const bool vec = nx == TW && ((pw & 15) == 0) && ((reinterpret_cast<uintptr_t>(base) & 15) == 0);
        if (vec) {
            for (int i = tid; i < ny * (TW / 16); i += NT) {
                const int r = i >> 2, c = (i & 3) * 16;
                const uint4 v = *reinterpret_cast<const uint4*>(&S.out[k][r][c]);
                __stcs(reinterpret_cast<uint4*>(base + (size_t)(Y0 + r) * pw + X0 + c), v);
            }
        } else {
            for (int r = warp; r < ny; r += NT / 32)
                for (int c = lane; c < nx; c += 32) base[(size_t)(Y0 + r) * pw + X0 + c] = S.out[k][r][c];
        }
    }
}

__global__ void crop_kernel(const uint8_t* __restrict__ src, int w, int h, CropGeom g,
                            uint8_t* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w) return;
    if (g.mx == 0 && g.my == 0) {
        out[(size_t)y * w + x] = src[(size_t)y * w + x];
        return;
    }
    const double sy = dadd((double)g.my, dmul((double)y, g.step_y));
    const double sx = dadd((double)g.mx, dmul((double)x, g.step_x));
    out[(size_t)y * w + x] = round_u8(sample_bilinear(src, w, h, sx, sy));
}


// ===================================================================== TMA
// Persistent variant: each CTA walks tiles t = blockIdx.x + k*gridDim.x; the
// source footprints of tile t+1 are fetched by TMA (cp.async.bulk.tensor, one
// instruction per plane) into the other half of a double buffer while tile
// t is computed; an mbarrier per buffer carries the transaction bytes.
// TMA box per plane: the footprint of a 64x32 tile (up to ~10 degrees at
// scale ~1) plus 16 columns, because the box's x origin must be 16-byte
// aligned for uint8 tensors (an unaligned origin raises an illegal
// instruction on sm_100).
constexpr int BW = 96, BH = 144;
constexpr int TTH = 128;           // TMA path output tile: TW x TTH
static_assert((TTH + NW - 1) / NW <= 32, "the crop loop shuffles one row table entry per lane");
constexpr int TWTH = 132;          // its W tile rows (<= 130 used)
constexpr int QW = 64;  // per-warp exact-path queue

constexpr int PROWS = 18, PWP = 64;  // private W rows per warp (<= 17 used) and their pitch

struct SmemT {
    alignas(128) uint8_t box[2][3][BH * BW];  // TMA source footprints, double-buffered
    uint8_t wt[2][TWTH][WTW];  // warped luma of the tile (shared mode) or the warps' private W rows
    unsigned long long mbar[2];  // TMA transaction barrier of each buffer
    unsigned done[2];            // warps finished with the buffer's tile
    unsigned wq[NT / 32][QW];    // per-warp queues of pixels for the exact path
    alignas(16) TileParams tpw[NW][2];  // per-warp copies: the next tile's parameters arrive by cp.async
};
static_assert(NW * PROWS * PWP <= TWTH * WTW, "private W rows fit the tile buffer");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap* map, int x, int y, int f,
                                          uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(f), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
    }
}

// one thread per (frame, tile): W region + TMA box origins (integer math on the row tables)
__global__ void tile_prep_kernel(const FramePlan* __restrict__ plan, int frames, int tiles_x,
                                 int tiles_y, int W, int H, int w, int h, int cw, int ch,
                                 CropGeom g, Tables T, int luma, int chroma) {
    const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long tpf = (long long)tiles_x * tiles_y;
    if (id >= tpf * frames) return;
    const int f = (int)(id / tpf), t = (int)(id - f * tpf);
    const int X0 = (t % tiles_x) * TW, Y0 = (t / tiles_x) * TTH;
    const int nx = min(TW, W - X0), ny = min(TTH, H - Y0);
    const FramePlan p = plan[f];
    TileParams tp;
    memset(&tp, 0, sizeof tp);
    const bool identity = g.mx == 0 && g.my == 0;
    if (luma) {
        int u0 = X0, v0 = Y0, nu = nx, nv = ny;
        if (!identity) {
            u0 = T.cx0[X0];
            v0 = T.cy0[Y0];
            nu = min(T.cx0[X0 + nx - 1] + 1, w - 1) - u0 + 1;
            nv = min(T.cy0[Y0 + ny - 1] + 1, h - 1) - v0 + 1;
        }
        tp.u0 = u0;
        tp.v0 = v0;
        tp.nu = nu;
        tp.nv = nv;
        int xmn = INT_MAX, xmx = INT_MIN, ymn = INT_MAX, ymx = INT_MIN;
        for (int k = 0; k < 4; ++k) {
            const int u = u0 + ((k & 1) ? nu - 1 : 0), v = v0 + ((k & 2) ? nv - 1 : 0);
            const long long X = T.rxf[(size_t)f * h + v] + (long long)u * p.cf;
            const long long Yv = T.ryf[(size_t)f * h + v] - (long long)u * p.snf;
            xmn = min(xmn, (int)(X >> 48));
            xmx = max(xmx, (int)(X >> 48));
            ymn = min(ymn, (int)(Yv >> 48));
            ymx = max(ymx, (int)(Yv >> 48));
        }
        tp.lbx = (xmn - 1) & ~15;
        tp.lby = ymn - 1;
        tp.lfit = (xmx + 2) - tp.lbx < BW && (ymx + 2) - tp.lby < BH;
        // interior tile: every W sample's integer parts lie in [1, w-3] x [1, h-3]
        // (one pixel of slack for the 32.32 conversion), so the lean row loop
        // needs no per-pixel bounds or near-integer decisions (see inner32)
        if (tp.lfit && nu <= TW && xmn >= 2 && xmx <= w - 4 && ymn >= 2 && ymx <= h - 4) tp.pad0 |= 1;
        // private W rows (each warp computes the W rows its crop rows read, no
        // CTA barrier): interior tile whose crop taps are x0, x0 + 1 and whose
        // bottom row never clamps (crop_rows2)
        if ((tp.pad0 & 1) && !identity && g.my >= 1 && T.cx0[X0 + nx - 1] + 1 <= w - 1) tp.pad0 |= 4;
    }
    if (chroma) {
        int xmn = INT_MAX, xmx = INT_MIN, ymn = INT_MAX, ymx = INT_MIN;
        for (int k = 0; k < 4; ++k) {
            const int x = X0 + ((k & 1) ? nx - 1 : 0), y = Y0 + ((k & 2) ? ny - 1 : 0);
            const long long X = T.pxf[(size_t)f * ch + y] + (long long)x * p.kxx;
            const long long Yv = T.pyf[(size_t)f * ch + y] + (long long)x * p.kyx;
            xmn = min(xmn, (int)(X >> 48));
            xmx = max(xmx, (int)(X >> 48));
            ymn = min(ymn, (int)(Yv >> 48));
            ymx = max(ymx, (int)(Yv >> 48));
        }
        tp.cbx = (xmn - 1) & ~15;
        tp.cby = ymn - 1;
        tp.cfit = (xmx + 2) - tp.cbx < BW && (ymx + 2) - tp.cby < BH;
        if (tp.cfit && xmn >= 2 && xmx <= cw - 4 && ymn >= 2 && ymx <= ch - 4) tp.pad0 |= 2;
    }
    tp.pad1 = (X0 / TW) | (Y0 / TTH) << 16;  // tile coordinates (no division in the compose loop)
    int4* dst = T.tiles + 3 * id;
    const int4* src = reinterpret_cast<const int4*>(&tp);
    dst[0] = src[0];
    dst[1] = src[1];
    dst[2] = src[2];
}

__device__ __forceinline__ void sts_u8(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v));
}

__device__ __forceinline__ void stg_u8(uint8_t* p, uint32_t v) { __stcs(p, (uint8_t)v); }

// Per-warp queue push (warp-uniform count, no atomics).  All lanes call it.
__device__ __forceinline__ void wq_push(unsigned* q, int& qn, bool bad, unsigned item) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, bad);
    if (m) {
        const int pos = qn + __popc(m & ((1u << (threadIdx.x & 31)) - 1));
        if (bad && pos < QW) q[pos] = item;
        qn += __popc(m);
    }
}

// fast blend + lround of 4 bytes; sets bad when the rounding is not certain
__device__ __forceinline__ uint32_t blend_bad(uint32_t a, uint32_t b, uint32_t c, uint32_t d, float fx,
                                              float fy, bool& bad) {
    const float fa = b256(a), fc = b256(c);
    const float top = fmaf(fx, b256(b) - fa, fa);
    const float bot = fmaf(fx, b256(d) - fc, fc);
    const float v = fmaf(fy, bot - top, top);
    const float m = v + 8388608.0f;
    bad |= fabsf(v - (m - 8388608.0f)) > 0.5f - VGUARD;
    return (uint32_t)__float_as_int(m) & 0xFFu;
}

// Fast-path coordinate decode result (decode32 below): fractions, integer
// parts, in-bounds test.
struct Pt {
    float fx, fy;
    int ix, iy;
    bool inb;
};

// Two fast blends at once on the packed fp32x2 pipe (FFMA2/FADD2): the
// same arithmetic as blend_bad, lane-wise.  Returns rp | rq << 8.
struct Q4 {
    uint32_t a, b, c, d;
};

__device__ __forceinline__ float2 sub2(float2 x, float2 y) { return __fadd2_rn(x, make_float2(-y.x, -y.y)); }

__device__ __forceinline__ uint32_t blend2_bad(const Q4& p, const Q4& q, float2 fx, float2 fy, bool& badp,
                                               bool& badq) {
    const float2 fa = make_float2(b256(p.a), b256(q.a)), fb = make_float2(b256(p.b), b256(q.b));
    const float2 fc = make_float2(b256(p.c), b256(q.c)), fd = make_float2(b256(p.d), b256(q.d));
    const float2 top = __ffma2_rn(fx, sub2(fb, fa), fa);
    const float2 bot = __ffma2_rn(fx, sub2(fd, fc), fc);
    const float2 v = __ffma2_rn(fy, sub2(bot, top), top);
    const float2 m = __fadd2_rn(v, make_float2(8388608.0f, 8388608.0f));
    const float2 dv = sub2(v, __fadd2_rn(m, make_float2(-8388608.0f, -8388608.0f)));
    badp = fabsf(dv.x) > 0.5f - VGUARD;
    badq = fabsf(dv.y) > 0.5f - VGUARD;
    return (__float_as_uint(m.x) & 0xFFu) | ((__float_as_uint(m.y) & 0xFFu) << 8);
}

template <typename P>
__device__ __forceinline__ Q4 fetch4(P src, int pitch, int obase, const Pt& t) {
    const int o = t.inb ? t.iy * pitch + t.ix + obase : 0;
    return Q4{src[o], src[o + 1], src[o + pitch], src[o + pitch + 1]};
}

// ---- exact reference paths, out of line (taken by ~1% of warp rows) ----
__device__ __noinline__ uint32_t w_exact_tile(const FramePlan* __restrict__ plan, int f, const uint8_t* box,
                                              int lbx, int lby, int fit, const uint8_t* gy, int w, int h, int u,
                                              int v) {
    const FramePlan p = plan[f];
    if (fit) return w_exact_f([=](int x, int y) { return (double)box[(y - lby) * BW + x - lbx]; }, w, h, p, u, v);
    return w_exact(gy, w, h, p, u, v);
}

__device__ __noinline__ uint32_t chroma_exact_tile(const FramePlan* __restrict__ plan, int f, CropGeom g,
                                                   const uint8_t* b1, const uint8_t* b2, int cbx, int cby, int fit,
                                                   const uint8_t* gcb, const uint8_t* gcr, int w, int h, int cw,
                                                   int ch, int x, int y) {
    const FramePlan p = plan[f];
    const ChromaMap cm = chroma_map(w, h, cw, ch, g);
    uint8_t ob, orr;
    if (fit)
        chroma_exact_f(p, g, cm, [=](int xx, int yy) { return (double)b1[(yy - cby) * BW + xx - cbx]; },
                       [=](int xx, int yy) { return (double)b2[(yy - cby) * BW + xx - cbx]; }, cw, ch, x, y, ob,
                       orr);
    else
        chroma_exact(p, g, cm, gcb, gcr, cw, ch, x, y, ob, orr);
    return ob | ((uint32_t)orr << 8);
}

// crop_resize pixel (image_ops.cpp:151-157) of output (X, Y) from the W tile
// (wl: the W rows indexed by absolute row, row pitch wp)
__device__ __noinline__ uint32_t crop_exact_tile(const uint8_t* wl, int wp, const Tables T, int X, int Y, int u0,
                                                 int w, int h) {
    const int x0 = T.cx0[X], y0 = T.cy0[Y];
    const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
    const double a = wl[y0 * wp + x0 - u0], b = wl[y0 * wp + x1 - u0];
    const double cc = wl[y1 * wp + x0 - u0], d = wl[y1 * wp + x1 - u0];
    const double top = dadd(a, dmul(T.cfx[X], dsub(b, a)));
    const double bot = dadd(cc, dmul(T.cfx[X], dsub(d, cc)));
    return round_u8(dadd(top, dmul(T.cfy[Y], dsub(bot, top))));
}

// ---- 32.32 coordinates for the row loops --------------------------------
// The row loops carry coordinates as 32.32 fixed point with the integer part
// biased by -1 (hi word = ix - 1, lo word = the fraction), converted once per
// tile from the 16.48 tables: every step is one 64-bit add and the integer
// part / fraction are register halves.  Error against the reference
// coordinate: <= 2^-32 per conversion, <= 2^-32 per 8-row step (16 per
// tile), plus the tables' ~1e-13: < 5e-9 px.
//
// Interior fast path: when the biased integer part lies in [0, w-4] (ix in
// [1, w-3]) the reference's sample is in bounds with x1 = x0 + 1 whichever
// side of an integer the exact coordinate falls, and the bilinear blend is
// continuous across that integer (fraction ~0 with x0 = ix equals fraction
// ~1 with x0 = ix - 1 to within 255 * 5e-9), so no coordinate guard is
// needed: only the blended value's .5-tie guard (VGUARD) decides.  A warp row
// with any valid non-interior pixel takes the guarded decode (decode32).
constexpr long long ONE32 = 1LL << 32;

__device__ __forceinline__ long long to32(long long x48) { return (x48 >> 16) - ONE32; }

__device__ __forceinline__ int hi32(long long x) { return (int)(x >> 32); }

// Guarded decode of a biased 32.32 point (the rows with frame-edge pixels).
__device__ __forceinline__ Pt decode32(long long X, long long Y, unsigned limx, unsigned limy, bool valid,
                                       bool& bad) {
    Pt t;
    const uint32_t fxs = (uint32_t)X, fys = (uint32_t)Y;
    bad = valid && ((fxs + GUARD) < 2 * GUARD || (fys + GUARD) < 2 * GUARD);
    t.ix = hi32(X) + 1;
    t.iy = hi32(Y) + 1;
    t.inb = valid && (unsigned)t.ix <= limx && (unsigned)t.iy <= limy;
    t.fx = frac_f(fxs);
    t.fy = frac_f(fys);
    return t;
}

// interior test on the biased integer parts (limx = w - 2: biased <= w - 4)
__device__ __forceinline__ bool inner32(long long X, long long Y, unsigned limx, unsigned limy) {
    return ((unsigned)hi32(X) <= limx - 2) & ((unsigned)hi32(Y) <= limy - 2);
}

template <typename P>
__device__ __forceinline__ Q4 fetch4i(P src, int pitch, int ob1, long long X, long long Y, bool valid) {
    const int o = valid ? hi32(Y) * pitch + hi32(X) + ob1 : 0;  // ob1 = obase + pitch + 1
    return Q4{src[o], src[o + 1], src[o + pitch], src[o + pitch + 1]};
}

__device__ __forceinline__ float2 frac2(long long X0, long long X1) {
    return make_float2(frac_f((uint32_t)X0), frac_f((uint32_t)X1));
}

// Luma W rows of a tile (warp per row, lane per column) into the shared W
// tile; src is the staged TMA box (pitch BW, obase = -(lby*BW + lbx)) or the
// global frame (pitch w, obase 0).  Table and step inputs are 16.48.
// Returns the warp's queue length.
template <typename P>
__device__ __forceinline__ int w_rows_q(P src, int pitch, int obase, const long long* __restrict__ rxf,
                                        const long long* __restrict__ ryf, uint32_t wsm, int nu, int nv,
                                        long long uCF, long long uSN, long long CF32, long long SN32,
                                        long long RSX, long long RSY, unsigned limx, unsigned limy,
                                        unsigned* q) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool v0 = lane < nu, v1 = lane + 32 < nu, has2 = nu > 64;
    const int ob1 = obase + pitch + 1;
    int qn = 0;
    uint32_t row = wsm + warp * WTW + lane;
    // the warp's first row start from the table, then 8-row steps
    long long SX = to32(__ldg(rxf + min(warp, nv - 1)) + uCF), SY = to32(__ldg(ryf + min(warp, nv - 1)) - uSN);
    const long long cx = CF32 >> 16, cy = SN32 >> 16, rsx = RSX >> 16, rsy = RSY >> 16;
    for (int r = warp; r < nv; r += NW, row += NW * WTW, SX += rsx, SY += rsy) {
        const long long X1 = SX + cx, Y1 = SY - cy;
        bool b0, b1, b2 = false;
        if (__all_sync(0xFFFFFFFFu, (!v0 | inner32(SX, SY, limx, limy)) & (!v1 | inner32(X1, Y1, limx, limy)))) {
            const uint32_t pr = blend2_bad(fetch4i(src, pitch, ob1, SX, SY, v0), fetch4i(src, pitch, ob1, X1, Y1, v1),
                                           frac2(SX, X1), frac2(SY, Y1), b0, b1);
            b0 = b0 && v0;
            b1 = b1 && v1;
            if (v0) sts_u8(row, pr & 0xFF);
            if (v1) sts_u8(row + 32, pr >> 8);
        } else {
            bool e0, e1;
            const Pt t0 = decode32(SX, SY, limx, limy, v0, b0);
            const Pt t1 = decode32(X1, Y1, limx, limy, v1, b1);
            const uint32_t pr = blend2_bad(fetch4(src, pitch, obase, t0), fetch4(src, pitch, obase, t1),
                                           make_float2(t0.fx, t1.fx), make_float2(t0.fy, t1.fy), e0, e1);
            b0 = b0 || (t0.inb && e0);
            b1 = b1 || (t1.inb && e1);
            if (v0) sts_u8(row, t0.inb ? (pr & 0xFF) : 0u);
            if (v1) sts_u8(row + 32, t1.inb ? (pr >> 8) : 0u);
        }
        if (has2) {  // rare third half (nu = 65 .. 66)
            const bool v2 = lane + 64 < nu;
            const Pt t2 = decode32(SX + 2 * cx, SY - 2 * cy, limx, limy, v2, b2);
            const int o = t2.inb ? t2.iy * pitch + t2.ix + obase : 0;
            bool e2 = false;
            const uint32_t a2 = blend_bad(src[o], src[o + 1], src[o + pitch], src[o + pitch + 1], t2.fx, t2.fy, e2);
            b2 = b2 || (t2.inb && e2);
            if (v2) sts_u8(row + 64, t2.inb ? a2 : 0u);
        }
        if (__any_sync(0xFFFFFFFFu, b0 || b1 || b2)) {
            const unsigned it = ((unsigned)r << 8) | (unsigned)lane;
            wq_push(q, qn, b0, it);
            wq_push(q, qn, b1, it + 32);
            wq_push(q, qn, b2, it + 64);
        }
    }
    return qn;
}

// Chroma rows of a tile straight to the output planes (both planes share
// one coordinate per pixel).  Table and step inputs are 16.48.  Returns the
// warp's queue length.
template <typename P>
__device__ __forceinline__ int chroma_rows_q(P s1, P s2, int pitch, int obase, const long long* __restrict__ pxf,
                                             const long long* __restrict__ pyf, uint8_t* ob, uint8_t* orr, int op,
                                             int nx, int ny, long long xKX, long long xKY, long long KX32,
                                             long long KY32, long long RSX, long long RSY, unsigned limx,
                                             unsigned limy, unsigned* q) {
    // op: output row pitch
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool v0 = lane < nx, v1 = lane + 32 < nx;
    const int ob1 = obase + pitch + 1;
    int qn = 0;
    const size_t step = (size_t)NW * op;
    uint8_t* pb = ob + (size_t)warp * op + lane;
    uint8_t* pr = orr + (size_t)warp * op + lane;
    long long PX = to32(__ldg(pxf + min(warp, ny - 1)) + xKX), PY = to32(__ldg(pyf + min(warp, ny - 1)) + xKY);
    const long long kx = KX32 >> 16, ky = KY32 >> 16, rsx = RSX >> 16, rsy = RSY >> 16;
    for (int r = warp; r < ny; r += NW, pb += step, pr += step, PX += rsx, PY += rsy) {
        const long long X1 = PX + kx, Y1 = PY + ky;
        bool b0, b1, e0, e1, e2, e3;
        uint32_t a0, a1;
        if (__all_sync(0xFFFFFFFFu, (!v0 | inner32(PX, PY, limx, limy)) & (!v1 | inner32(X1, Y1, limx, limy)))) {
            const float fx0 = frac_f((uint32_t)PX), fy0 = frac_f((uint32_t)PY);
            const float fx1 = frac_f((uint32_t)X1), fy1 = frac_f((uint32_t)Y1);
            a0 = blend2_bad(fetch4i(s1, pitch, ob1, PX, PY, v0), fetch4i(s2, pitch, ob1, PX, PY, v0),
                            make_float2(fx0, fx0), make_float2(fy0, fy0), e0, e1);
            a1 = blend2_bad(fetch4i(s1, pitch, ob1, X1, Y1, v1), fetch4i(s2, pitch, ob1, X1, Y1, v1),
                            make_float2(fx1, fx1), make_float2(fy1, fy1), e2, e3);
            b0 = v0 && (e0 || e1);
            b1 = v1 && (e2 || e3);
        } else {
            const Pt t0 = decode32(PX, PY, limx, limy, v0, b0);
            const Pt t1 = decode32(X1, Y1, limx, limy, v1, b1);
            const uint32_t p0 = blend2_bad(fetch4(s1, pitch, obase, t0), fetch4(s2, pitch, obase, t0),
                                           make_float2(t0.fx, t0.fx), make_float2(t0.fy, t0.fy), e0, e1);
            const uint32_t p1 = blend2_bad(fetch4(s1, pitch, obase, t1), fetch4(s2, pitch, obase, t1),
                                           make_float2(t1.fx, t1.fx), make_float2(t1.fy, t1.fy), e2, e3);
            b0 = b0 || (t0.inb && (e0 || e1));
            b1 = b1 || (t1.inb && (e2 || e3));
            a0 = t0.inb ? p0 : 0x8080u;
            a1 = t1.inb ? p1 : 0x8080u;
        }
        if (v0) {
            stg_u8(pb, a0 & 0xFF);
            stg_u8(pr, a0 >> 8);
        }
        if (v1) {
            stg_u8(pb + 32, a1 & 0xFF);
            stg_u8(pr + 32, a1 >> 8);
        }
        if (__any_sync(0xFFFFFFFFu, b0 || b1)) {
            const unsigned it = ((unsigned)r << 8) | (unsigned)lane;
            wq_push(q, qn, b0, it);
            wq_push(q, qn, b1, it + 32);
        }
    }
    return qn;
}

__device__ __forceinline__ void sts_u16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "r"(v));
}

__device__ __forceinline__ void stg_u16(uint8_t* p, uint32_t v) {
    __stcs(reinterpret_cast<unsigned short*>(p), (unsigned short)v);
}

// ---- lean row loops, v2 (interior tiles) ----------------------------------
// Same exactness argument as w_rows_lean / chroma_rows_lean; fewer issued
// instructions per sample:
//  * the 32.32 coordinates are taken relative to the staged box origin once
//    per tile (hi word = tap column / row inside the box), so a tap address
//    is one IMAD and the four taps are immediate offsets;
//  * the lane's second column is its first plus one column step (one 64-bit
//    add; lanes past the tile width repeat their first column);
//  * both fractions of a coordinate pair come from one FADD2;
//  * the two rounded bytes are packed with one PRMT and stored unconditionally
//    (W-tile columns past nu are never read; output widths of the TMA path are
//    multiples of 16, so a lane's two columns are valid together);
//  * undecided pixels set one bit per row in a lane-local mask (<= 17 rows per
//    warp and tile) instead of a warp vote per row; the lane recomputes its
//    flagged rows with the exact reference path after the loop (divergent,
//    about one warp row in sixty).
// Coordinate error as before: <= 2^-32 per conversion / step, < 20 steps per
// tile: < 5e-9 px.
__device__ __forceinline__ float2 frac2p(uint32_t a, uint32_t b) {
    return __fadd2_rn(make_float2(__uint_as_float(0x3F800000u | (a >> 9)), __uint_as_float(0x3F800000u | (b >> 9))),
                      make_float2(-0.99999994f, -0.99999994f));
}

// blend2_bad with the two bytes packed by one PRMT (low 16 bits = p | q << 8)
__device__ __forceinline__ uint32_t blend2p(const Q4& p, const Q4& q, float2 fx, float2 fy, bool& bad) {
    const float2 fa = make_float2(b256(p.a), b256(q.a)), fb = make_float2(b256(p.b), b256(q.b));
    const float2 fc = make_float2(b256(p.c), b256(q.c)), fd = make_float2(b256(p.d), b256(q.d));
    const float2 top = __ffma2_rn(fx, sub2(fb, fa), fa);
    const float2 bot = __ffma2_rn(fx, sub2(fd, fc), fc);
    const float2 v = __ffma2_rn(fy, sub2(bot, top), top);
    const float2 m = __fadd2_rn(v, make_float2(8388608.0f, 8388608.0f));
    const float2 dv = sub2(v, __fadd2_rn(m, make_float2(-8388608.0f, -8388608.0f)));
    bad = fmaxf(fabsf(dv.x), fabsf(dv.y)) > 0.5f - VGUARD;
    return __byte_perm(__float_as_uint(m.x), __float_as_uint(m.y), 0x0040);
}

__device__ __forceinline__ Q4 taps(const uint8_t* p) { return Q4{p[0], p[1], p[BW], p[BW + 1]}; }

__device__ __forceinline__ const uint8_t* tap_ptr(const uint8_t* box, long long X, long long Y) {
    return box + hi32(Y) * BW + hi32(X);
}

// W rows r = rs, rs + RS, ... < re (tile rows, relative to v0) of an interior
// tile; the k-th row of the call goes to out + k * OP (lane: columns 2l, 2l+1)
template <int RS, int OP>
__device__ __forceinline__ void w_rows_lean2(const uint8_t* box, int lbx, int lby, const long long* __restrict__ rxf,
                                             const long long* __restrict__ ryf, uint8_t* out, int rs, int re, int nu,
                                             int u0, int v0, long long cf, long long snf,
                                             const FramePlan* __restrict__ plan, int f, int w, int h) {
    if (rs >= re) return;
    const int lane = threadIdx.x & 31;
    const int c0 = 2 * lane;
    const long long ua = (long long)(u0 + min(c0, nu - 1));
    long long XA = ((__ldg(rxf + rs) + ua * cf) >> 16) - ((long long)lbx << 32);
    long long YA = ((__ldg(ryf + rs) - ua * snf) >> 16) - ((long long)lby << 32);
    const bool vA = c0 < nu, vB = c0 + 1 < nu;
    const long long DX = vB ? (cf >> 16) : 0, DY = vB ? -(snf >> 16) : 0;
    const long long RX = ((long long)RS * snf) >> 16, RY = ((long long)RS * cf) >> 16;
    uint8_t* wr = out + c0;
    uint32_t bad = 0, bit = 1;
#pragma unroll 2
    for (int r = rs; r < re; r += RS, wr += OP, bit <<= 1, XA += RX, YA += RY) {
        const long long XB = XA + DX, YB = YA + DY;
        bool b;
        const uint32_t v = blend2p(taps(tap_ptr(box, XA, YA)), taps(tap_ptr(box, XB, YB)),
                                   frac2p((uint32_t)XA, (uint32_t)XB), frac2p((uint32_t)YA, (uint32_t)YB), b);
        *reinterpret_cast<uint16_t*>(wr) = (uint16_t)v;
        if (b) bad |= bit;
    }
    if (!vA) bad = 0;
    for (; bad; bad &= bad - 1) {  // this lane's undecided rows (both columns recomputed)
        const int k = __ffs(bad) - 1, r = rs + RS * k;
        out[k * OP + c0] = (uint8_t)w_exact_tile(plan, f, box, lbx, lby, 1, nullptr, w, h, u0 + c0, v0 + r);
        if (vB)
            out[k * OP + c0 + 1] =
                (uint8_t)w_exact_tile(plan, f, box, lbx, lby, 1, nullptr, w, h, u0 + c0 + 1, v0 + r);
    }
}

// 4:4:4 chroma rows of an interior tile straight to the output planes; the
// Cr box follows the Cb box (one immediate offset)
__device__ __forceinline__ void chroma_rows_lean2(const uint8_t* s1, int cbx, int cby, const long long* __restrict__ pxf,
                                                  const long long* __restrict__ pyf, uint8_t* ob, uint8_t* orr, int op,
                                                  int cw, int ch, int nx, int ny, int X0, int Y0, long long kxx,
                                                  long long kyx, long long kxy, long long kyy,
                                                  const FramePlan* __restrict__ plan, int f, CropGeom g, int w, int h) {
    // op: output row pitch
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = 2 * lane;
    const int r0 = min(warp, ny - 1);
    const long long xa = (long long)(X0 + min(c0, nx - 1));
    long long XA = ((__ldg(pxf + r0) + xa * kxx) >> 16) - ((long long)cbx << 32);
    long long YA = ((__ldg(pyf + r0) + xa * kyx) >> 16) - ((long long)cby << 32);
    const bool vA = c0 < nx, vB = c0 + 1 < nx;
    const long long DX = vB ? (kxx >> 16) : 0, DY = vB ? (kyx >> 16) : 0;
    const long long RX = ((long long)NW * kxy) >> 16, RY = ((long long)NW * kyy) >> 16;
    const size_t step = (size_t)NW * op;
    uint8_t* pb = ob + (size_t)warp * op + c0;
    const ptrdiff_t dr = orr - ob;
    uint32_t bad = 0, bit = 1;
#pragma unroll 2
    for (int r = warp; r < ny; r += NW, pb += step, bit <<= 1, XA += RX, YA += RY) {
        const long long XB = XA + DX, YB = YA + DY;
        const float2 fx = frac2p((uint32_t)XA, (uint32_t)XB), fy = frac2p((uint32_t)YA, (uint32_t)YB);
        const uint8_t* pa = tap_ptr(s1, XA, YA);
        const uint8_t* pq = tap_ptr(s1, XB, YB);
        bool e1, e2;
        const uint32_t vb = blend2p(taps(pa), taps(pq), fx, fy, e1);
        const uint32_t vr = blend2p(taps(pa + BH * BW), taps(pq + BH * BW), fx, fy, e2);
        if (vA) {
            stg_u16(pb, vb);
            stg_u16(pb + dr, vr);
        }
        if (e1 | e2) bad |= bit;
    }
    if (!vA) bad = 0;
    for (; bad; bad &= bad - 1) {
        const int r = warp + NW * (__ffs(bad) - 1);
        for (int j = 0; j < 2; ++j) {
            const int c = c0 + j;
            if (c >= nx) break;
            const uint32_t v = chroma_exact_tile(plan, f, g, s1, s1 + BH * BW, cbx, cby, 1, nullptr, nullptr, w, h, cw,
                                                 ch, X0 + c, Y0 + r);
            const size_t o = (size_t)r * op + c;
            stg_u8(ob + o, v & 0xFF);
            stg_u8(orr + o, v >> 8);
        }
    }
}

// two RGB pixels (6 bytes, 2-byte aligned) from two luma bytes yy (low 16
// bits) and the Cb / Cr pairs at c (chroma output tile, Cr TTH * TW later)
__device__ __forceinline__ void store_rgb2(uint8_t* p, uint32_t yy, const uint8_t* c) {
    const uint32_t cb = *reinterpret_cast<const uint16_t*>(c), cr = *reinterpret_cast<const uint16_t*>(c + TTH * TW);
    const uint32_t p0 = colour::ycc_to_rgb(yy & 0xFF, cb & 0xFF, cr & 0xFF);
    const uint32_t p1 = colour::ycc_to_rgb((yy >> 8) & 0xFF, cb >> 8, cr >> 8);
    stg_u16(p, p0);
    stg_u16(p + 2, (p0 >> 16) | (p1 << 8));
    stg_u16(p + 4, p1 >> 8);
}

// crop_resize rows of the W tile (image_ops.cpp:136-159) when every lane's two
// taps are x0, x0 + 1 and the bottom row never clamps (crop margins >= 1 px):
// each warp walks a contiguous run of output rows; cy0 advances by 0 or 1 per
// row (step < 1), so the new top lerp is the previous bottom one when it
// advances, and the bottom lerp is recomputed every row (the same value when
// cy0 stays) — no per-row branch.  Lane: output columns 2l, 2l+1.
// RGBO: the luma bytes are combined with the tile's Cb / Cr (csc: the chroma
// pass's output tile, pitch TW, Cr TTH * TW after Cb) and stored as
// interleaved RGB (yuv_to_rgb, colour.cuh) into the RGB frame oy (pitch 3w):
// Y/Cb/Cr -> RGB fused into the compose store.
// wl: the W rows indexed by absolute W row, row pitch WP; rows [rb, re) of
// the tile (crop_rows_of)
template <bool RGBO, int WP>
__device__ __forceinline__ void crop_rows2(const uint8_t* wl, const Tables& T, uint8_t* oy, int w, int h, int nx,
                                           int rb, int re, int X0, int Y0, int u0, const uint8_t* csc) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const int ny = re;  // rows past re are never read (myr clamps to re - 1)
    if (rb >= re) return;
    const int ca = X0 + min(2 * lane, nx - 1), cb = X0 + min(2 * lane + 1, nx - 1);
    const int xa = __ldg(T.cx0 + ca) - u0, xb = __ldg(T.cx0 + cb) - u0;
    const float2 fx2 = make_float2((float)__ldg(T.cfx + ca), (float)__ldg(T.cfx + cb));
    const bool vA = 2 * lane < nx, vB = 2 * lane + 1 < nx;
    auto hl2 = [&](int row) {
        const uint8_t* rp = wl + row * WP;
        const float2 fa = make_float2(b256(rp[xa]), b256(rp[xb])), fb = make_float2(b256(rp[xa + 1]), b256(rp[xb + 1]));
        return __ffma2_rn(fx2, sub2(fb, fa), fa);
    };
    const int myr = min(rb + lane, ny - 1);
    const int mycy = __ldg(T.cy0 + Y0 + myr);
    const float myfy = (float)__ldg(T.cfy + Y0 + myr);
    int trow = __shfl_sync(FULL, mycy, 0);
    float2 top = hl2(trow), bot = top;
    const int OP = RGBO ? 3 * w : w;  // output pitch
    uint8_t* py = oy + ((size_t)(Y0 + rb) * w + X0 + 2 * lane) * (RGBO ? 3 : 1);
    const uint8_t* pc = csc + rb * TW + 2 * lane;
    uint32_t bad = 0, bit = 1;
    for (int r = rb; r < re; ++r, py += OP, pc += TW, bit <<= 1) {
        const int cy = __shfl_sync(FULL, mycy, r - rb);
        const float fy = __shfl_sync(FULL, myfy, r - rb);
        if (r > rb) {
            const bool adv = cy != trow;
            top.x = adv ? bot.x : top.x;
            top.y = adv ? bot.y : top.y;
        }
        bot = hl2(cy + 1);
        trow = cy;
        const float2 v = __ffma2_rn(make_float2(fy, fy), sub2(bot, top), top);
        const float2 m = __fadd2_rn(v, make_float2(8388608.0f, 8388608.0f));
        const float2 dv = sub2(v, __fadd2_rn(m, make_float2(-8388608.0f, -8388608.0f)));
        const uint32_t yy = __byte_perm(__float_as_uint(m.x), __float_as_uint(m.y), 0x0040);
        if (RGBO) {
            if (vA) store_rgb2(py, yy, pc);
        } else if (vA) {
            stg_u16(py, yy);
        }
        if (fmaxf(fabsf(dv.x), fabsf(dv.y)) > 0.5f - VGUARD) bad |= bit;
    }
    if (!vA) bad = 0;
    for (; bad; bad &= bad - 1) {
        const int r = rb + __ffs(bad) - 1;
        const uint32_t y0 = crop_exact_tile(wl, WP, T, X0 + 2 * lane, Y0 + r, u0, w, h);
        const uint32_t y1 = vB ? crop_exact_tile(wl, WP, T, X0 + 2 * lane + 1, Y0 + r, u0, w, h) : 0u;
        if (RGBO) {
            store_rgb2(oy + ((size_t)(Y0 + r) * w + X0 + 2 * lane) * 3, y0 | y1 << 8, csc + r * TW + 2 * lane);
        } else {
            uint8_t* o = oy + (size_t)(Y0 + r) * w + X0 + 2 * lane;
            o[0] = (uint8_t)y0;
            if (vB) o[1] = (uint8_t)y1;
        }
    }
}

// Persistent TMA compose.  Per tile: every warp waits on the buffer's TMA
// mbarrier, computes the W rows (-> shared memory) and chroma rows (->
// global), then the crop_resize rows of W (-> global).  Two modes per tile:
//  * private (interior tiles, tile_prep pad0 bit 2): each warp computes the W
//    rows its own (contiguous) crop rows read into its private rows of wt[b]
//    (<= 17 rows; a row shared by two warps is computed by both), so the
//    crop follows after a __syncwarp — no CTA barrier;
//  * shared (edge tiles): W rows warp-strided into wt[b], one CTA barrier.
// Buffer reuse: each warp counts itself done with buffer b at the end of its
// tile; the last one issues the TMA of the tile two steps ahead into b (and
// resets the count), so a fast warp runs ahead into the next tile while slow
// ones finish.  Undecidable pixels take the exact reference path inline (the
// lane diverges for them only).
template <bool LUMA, bool CHROMA, bool RGBO>
__global__ void __launch_bounds__(NT, 2) compose_tma_kernel(
    PlaneBatch Y, PlaneBatch CB, PlaneBatch CR, const FramePlan* __restrict__ plan, CropGeom g,
    Tables T, int tiles_x, int tiles_y, int frames, const __grid_constant__ CUtensorMap mapY,
    const __grid_constant__ CUtensorMap mapCB, const __grid_constant__ CUtensorMap mapCR,
    uint8_t* __restrict__ oY, uint8_t* __restrict__ oCB, uint8_t* __restrict__ oCR, uint8_t* scr) {
    static_assert(!RGBO || (LUMA && CHROMA), "RGB output needs luma and 4:4:4 chroma");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SmemT& S = *reinterpret_cast<SmemT*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = LUMA ? Y.w : CB.w, H = LUMA ? Y.h : CB.h;
    const int w = Y.w, h = Y.h, cw = CB.w, ch = CB.h;
    const bool identity = g.mx == 0 && g.my == 0;
    const int tpf = tiles_x * tiles_y;
    const long long total = (long long)tpf * frames;
    const uint32_t bytes_l = LUMA ? BW * BH : 0, bytes_c = CHROMA ? 2 * BW * BH : 0;
    constexpr unsigned FULL = 0xFFFFFFFFu;

    auto issue = [&](long long t, int b) {  // one thread: TMA of tile t into buffer b
        const int4 p1 = __ldg(T.tiles + 3 * t + 1), p2 = __ldg(T.tiles + 3 * t + 2);  // lbx lby cbx cby | lfit cfit
        const int f = (int)(t / tpf);
        const uint32_t bar = smem_u32(&S.mbar[b]);
        const bool lfit = LUMA && p2.x, cfit = CHROMA && p2.y;
        const uint32_t bytes = (lfit ? bytes_l : 0) + (cfit ? bytes_c : 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the buffer
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        if (lfit) tma_load3(smem_u32(&S.box[b][0][0]), &mapY, p1.x, p1.y, f, bar);
        if (cfit) {
            tma_load3(smem_u32(&S.box[b][1][0]), &mapCB, p1.z, p1.w, f, bar);
            tma_load3(smem_u32(&S.box[b][2][0]), &mapCR, p1.z, p1.w, f, bar);
        }
    };
    long long t = blockIdx.x;
    const long long G = gridDim.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.mbar[1])));
        S.done[0] = S.done[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (t < total) issue(t, 0);
        if (t + G < total) issue(t + G, 1);
    }
    __syncthreads();
    // frame of t, advanced incrementally
    int f = (int)(t / tpf), ti = (int)(t - (long long)f * tpf);
    const int df = (int)(G / tpf), dti = (int)(G - (long long)df * tpf);
    // this warp's copy of tile t's parameters, then of tile t + G (lanes 0-2,
    // 16 bytes each), one tile ahead
    auto fetch_tp = [&](long long tt, int slot) {
        if (lane < 3 && tt < total) {
            const uint32_t dst = smem_u32(&S.tpw[warp][slot]) + 16 * lane;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(T.tiles + 3 * tt + lane)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    fetch_tp(t, 0);
    for (int k = 0; t < total; ++k, t += G) {
        const int b = k & 1;
        if (k) {
            f += df;
            ti += dti;
            if (ti >= tpf) {
                ti -= tpf;
                ++f;
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        const TileParams tp = S.tpw[warp][k & 1];
        __syncwarp();
        fetch_tp(t + G, (k + 1) & 1);
        const int X0 = (tp.pad1 & 0xFFFF) * TW, Y0 = (tp.pad1 >> 16) * TTH;
        const int nx = min(TW, W - X0), ny = min(TTH, H - Y0);
        const int u0 = tp.u0, v0 = tp.v0, nu = tp.nu, nv = tp.nv;
        const long long cf = plan[f].cf, snf = plan[f].snf, kxx = plan[f].kxx, kyx = plan[f].kyx;
        const long long kxy = plan[f].kxy, kyy = plan[f].kyy;
        const uint8_t* gy = LUMA ? Y.base + (size_t)f * Y.stride : nullptr;
        const uint8_t* gcb = CHROMA ? CB.base + (size_t)f * CB.stride : nullptr;
        const uint8_t* gcr = CHROMA ? CR.base + (size_t)f * CR.stride : nullptr;
        const uint8_t* wt = &S.wt[b][0][0];
        uint8_t* csc = RGBO ? scr + ((size_t)blockIdx.x * 2 + b) * (2 * TTH * TW) : nullptr;
        // private mode: this warp's crop rows [crb, cre) and the W rows they read
        const bool priv = LUMA && (tp.pad0 & 4);
        const int cper = (ny + NW - 1) / NW, crb = warp * cper, cre = min(crb + cper, ny);
        int pw0 = 0;  // first private W row (absolute)
        mbar_wait(smem_u32(&S.mbar[b]), (uint32_t)((k >> 1) & 1));
        // ------------------------------------------- W rows -> wt[b]
        if (LUMA) {
            const unsigned limx = (unsigned)(w - 2), limy = (unsigned)(h - 2);
            const long long uCF = (long long)(u0 + lane) * cf, uSN = (long long)(u0 + lane) * snf;
            const long long* rxf = T.rxf + (size_t)f * h + v0;
            const long long* ryf = T.ryf + (size_t)f * h + v0;
            const uint8_t* bx = &S.box[b][0][0];
            const uint32_t wsm = smem_u32(wt);
            int qn = 0;
            if (priv) {
                uint8_t* pr = &S.wt[b][0][0] + warp * PROWS * PWP;
                if (crb < cre) {
                    pw0 = __ldg(T.cy0 + Y0 + crb);
                    const int pw1 = __ldg(T.cy0 + Y0 + cre - 1) + 1;
                    w_rows_lean2<1, PWP>(bx, tp.lbx, tp.lby, rxf, ryf, pr, pw0 - v0, pw1 - v0 + 1, nu, u0, v0, cf,
                                         snf, plan, f, w, h);
                }
                __syncwarp();
            } else if (tp.pad0 & 1)
                w_rows_lean2<NW, NW * WTW>(bx, tp.lbx, tp.lby, rxf, ryf, &S.wt[b][0][0] + warp * WTW, warp, nv, nu,
                                           u0, v0, cf, snf, plan, f, w, h);
            else if (tp.lfit)
                qn = w_rows_q(bx, BW, -(tp.lby * BW + tp.lbx), rxf, ryf, wsm, nu, nv, uCF, uSN, 32 * cf, 32 * snf,
                              NW * snf, NW * cf, limx, limy, S.wq[warp]);
            else
                qn = w_rows_q(gy, w, 0, rxf, ryf, wsm, nu, nv, uCF, uSN, 32 * cf, 32 * snf, NW * snf, NW * cf, limx,
                              limy, S.wq[warp]);
            if (__any_sync(FULL, qn > 0)) {  // exact pixels of this warp's rows, lanes in parallel
                __syncwarp();
                const int nq = qn <= QW ? qn : ((nv - warp + NW - 1) / NW) * nu;
                for (int i = lane; i < nq; i += 32) {
                    int r, c;
                    if (qn <= QW) {
                        const unsigned it = S.wq[warp][i];
                        r = (int)(it >> 8);
                        c = (int)(it & 0xFF);
                    } else {  // queue overflow: every pixel of this warp's rows
                        r = warp + NW * (i / nu);
                        c = i % nu;
                    }
                    sts_u8(wsm + r * WTW + c, w_exact_tile(plan, f, bx, tp.lbx, tp.lby, tp.lfit, gy, w, h, u0 + c,
                                                           v0 + r));
                }
                __syncwarp();
            }
        }
        // ------------------------------------------- chroma rows -> global
        if (CHROMA) {
            const unsigned limx = (unsigned)(cw - 2), limy = (unsigned)(ch - 2);
            const long long xKX = (long long)(X0 + lane) * kxx, xKY = (long long)(X0 + lane) * kyx;
            const long long* pxf = T.pxf + (size_t)f * ch + Y0;
            const long long* pyf = T.pyf + (size_t)f * ch + Y0;
            const uint8_t* b1p = &S.box[b][1][0];
            const uint8_t* b2p = &S.box[b][2][0];
            uint8_t* ob = RGBO ? csc : oCB + (size_t)f * CB.stride + (size_t)Y0 * cw + X0;
            uint8_t* orr = RGBO ? csc + TTH * TW : oCR + (size_t)f * CR.stride + (size_t)Y0 * cw + X0;
            const int op = RGBO ? TW : cw;  // output row pitch
            int qn = 0;
            if (tp.pad0 & 2)
                chroma_rows_lean2(b1p, tp.cbx, tp.cby, pxf, pyf, ob, orr, op, cw, ch, nx, ny, X0, Y0, kxx, kyx, kxy,
                                  kyy, plan, f, g, w, h);
            else if (tp.cfit)
                qn = chroma_rows_q(b1p, b2p, BW, -(tp.cby * BW + tp.cbx), pxf, pyf, ob, orr, op, nx, ny, xKX, xKY,
                                   32 * kxx, 32 * kyx, NW * kxy, NW * kyy, limx, limy, S.wq[warp]);
            else
                qn = chroma_rows_q(gcb, gcr, cw, 0, pxf, pyf, ob, orr, op, nx, ny, xKX, xKY, 32 * kxx, 32 * kyx,
                                   NW * kxy, NW * kyy, limx, limy, S.wq[warp]);
            if (__any_sync(FULL, qn > 0)) {
                __syncwarp();
                const int nq = qn <= QW ? qn : ((ny - warp + NW - 1) / NW) * nx;
                for (int i = lane; i < nq; i += 32) {
                    int r, c;
                    if (qn <= QW) {
                        const unsigned it = S.wq[warp][i];
                        r = (int)(it >> 8);
                        c = (int)(it & 0xFF);
                    } else {
                        r = warp + NW * (i / nx);
                        c = i % nx;
                    }
                    const uint32_t v = chroma_exact_tile(plan, f, g, b1p, b2p, tp.cbx, tp.cby, tp.cfit, gcb, gcr, w,
                                                         h, cw, ch, X0 + c, Y0 + r);
                    const size_t o = (size_t)r * op + c;
                    stg_u8(ob + o, v & 0xFF);
                    stg_u8(orr + o, v >> 8);
                }
                __syncwarp();
            }
        }
        if (!priv) __syncthreads();  // shared mode: wt[b] complete (RGBO: the Cb / Cr tile too)
        // ------------------------------------------- crop_resize of W -> global
        if (priv) {
            const uint8_t* wl = &S.wt[b][0][0] + warp * PROWS * PWP - pw0 * PWP;
            if (RGBO) {
                // the Cb / Cr rows of this warp's crop rows come from other warps
                __syncthreads();
                crop_rows2<true, PWP>(wl, T, oY + (size_t)f * Y.stride * 3, w, h, nx, crb, cre, X0, Y0, u0, csc);
            } else {
                crop_rows2<false, PWP>(wl, T, oY + (size_t)f * Y.stride, w, h, nx, crb, cre, X0, Y0, u0, nullptr);
            }
        } else if (RGBO) {  // the host checked the crop_rows2 preconditions (margins >= 1 px)
            crop_rows2<true, WTW>(wt - v0 * WTW, T, oY + (size_t)f * Y.stride * 3, w, h, nx, crb, cre, X0, Y0, u0,
                                  csc);
        } else if (LUMA) {
            if (identity) {
                uint8_t* oy = oY + (size_t)f * Y.stride + (size_t)Y0 * w + X0 + lane;
                const bool c0 = lane < nx, c1 = lane + 32 < nx;
                for (int r = warp; r < ny; r += NT / 32) {
                    if (c0) stg_u8(oy + (size_t)r * w, wt[r * WTW + lane]);
                    if (c1) stg_u8(oy + (size_t)r * w + 32, wt[r * WTW + lane + 32]);
                }
            } else if (g.my >= 1 && __all_sync(FULL, __ldg(T.cx0 + X0 + min(2 * lane, nx - 1)) + 1 <= w - 1 &&
                                                         __ldg(T.cx0 + X0 + min(2 * lane + 1, nx - 1)) + 1 <= w - 1)) {
                crop_rows2<false, WTW>(wt - v0 * WTW, T, oY + (size_t)f * Y.stride, w, h, nx, crb, cre, X0, Y0, u0,
                                       nullptr);
            } else {
                // lane l owns output columns 2l and 2l+1 (one 16-bit store per row)
                uint8_t* oy = oY + (size_t)f * Y.stride + (size_t)Y0 * w + X0 + 2 * lane;
                const bool c0 = 2 * lane < nx, c1 = 2 * lane + 1 < nx;
                int x0[2], x1[2];
                float fxv[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int c = X0 + min(2 * lane + j, nx - 1);
                    const int cx = __ldg(T.cx0 + c);
                    x0[j] = cx - u0;
                    x1[j] = min(cx + 1, w - 1) - u0;
                    fxv[j] = (float)__ldg(T.cfx + c);
                }
                const bool xin = __all_sync(FULL, x1[0] == x0[0] + 1 && x1[1] == x0[1] + 1);
                const float2 fx2 = make_float2(fxv[0], fxv[1]);
                // horizontal lerps of W row `row` at the lane's two columns
                // (crop_resize's top / bot, image_ops.cpp:151-156)
                auto hl = [&](int row) {
                    const uint8_t* rp = wt + (row - v0) * WTW;
                    uint32_t a0, b0, a1, b1;
                    if (xin) {
                        a0 = rp[x0[0]];
                        b0 = rp[x0[0] + 1];
                        a1 = rp[x0[1]];
                        b1 = rp[x0[1] + 1];
                    } else {
                        a0 = rp[x0[0]];
                        b0 = rp[x1[0]];
                        a1 = rp[x0[1]];
                        b1 = rp[x1[1]];
                    }
                    const float2 fa = make_float2(b256(a0), b256(a1)), fb = make_float2(b256(b0), b256(b1));
                    return __ffma2_rn(fx2, sub2(fb, fa), fa);
                };
                // each warp walks a contiguous run of output rows (<= 32): cy0
                // advances by 0 or 1 per row (step < 1), so the new bottom lerp is
                // the only one computed per row; a row with the same cy0 keeps
                // both.  The run's cy0 / fy come from one load per lane + shuffles.
                int qn = 0;
                const int per = (ny + NW - 1) / NW;
                const int rb = warp * per, re = min(rb + per, ny);
                uint8_t* py = oy + (size_t)rb * w;
                const int myr = min(rb + lane, ny - 1);
                const int mycy = __ldg(T.cy0 + Y0 + myr);
                const float myfy = (float)__ldg(T.cfy + Y0 + myr);
                int trow = __shfl_sync(FULL, mycy, 0);
                float2 top = hl(trow), bot = hl(min(trow + 1, h - 1));
                for (int r = rb; r < re; ++r, py += w) {
                    const int cy = __shfl_sync(FULL, mycy, r - rb);
                    const float fy = __shfl_sync(FULL, myfy, r - rb);
                    if (cy != trow) {
                        if (cy == trow + 1) {  // the previous bottom row min(trow + 1, h - 1) = cy
                            top = bot;
                        } else {
                            top = hl(cy);
                        }
                        bot = hl(min(cy + 1, h - 1));
                        trow = cy;
                    }
                    const float2 v = __ffma2_rn(make_float2(fy, fy), sub2(bot, top), top);
                    const float2 m = __fadd2_rn(v, make_float2(8388608.0f, 8388608.0f));
                    const float2 dv = sub2(v, __fadd2_rn(m, make_float2(-8388608.0f, -8388608.0f)));
                    const uint32_t a0 = __float_as_uint(m.x) & 0xFFu, a1 = __float_as_uint(m.y) & 0xFFu;
                    if (c1) stg_u16(py, a0 | (a1 << 8));
                    else if (c0) stg_u8(py, a0);
                    const bool b0 = c0 & (fabsf(dv.x) > 0.5f - VGUARD);
                    const bool b1 = c1 & (fabsf(dv.y) > 0.5f - VGUARD);
                    if (__any_sync(FULL, b0 | b1)) {
                        const unsigned it = ((unsigned)r << 8) | (unsigned)(2 * lane);
                        wq_push(S.wq[warp], qn, b0, it);
                        wq_push(S.wq[warp], qn, b1, it + 1);
                    }
                }
                if (__any_sync(FULL, qn > 0)) {
                    __syncwarp();
                    const int nq = qn <= QW ? qn : (re - rb) * nx;
                    for (int i = lane; i < nq; i += 32) {
                        int r, c;
                        if (qn <= QW) {
                            const unsigned it = S.wq[warp][i];
                            r = (int)(it >> 8);
                            c = (int)(it & 0xFF);
                        } else {  // queue overflow: every pixel of this warp's rows
                            r = rb + i / nx;
                            c = i % nx;
                        }
                        stg_u8(oy + (size_t)r * w + c - 2 * lane,
                               crop_exact_tile(wt - v0 * WTW, WTW, T, X0 + c, Y0 + r, u0, w, h));
                    }
                    __syncwarp();
                }
            }
        }
        // ------------------------------------------- release buffer b
        // (the last warp done with it issues the tile two steps ahead)
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();  // this warp's reads of box[b] / wt[b] happen before the count
            if (atomicAdd(&S.done[b], 1u) == NW - 1) {
                __threadfence_block();
                atomicExch(&S.done[b], 0u);
                if (t + 2 * G < total) issue(t + 2 * G, b);
            }
        }
    }
}

// persistent grid of the TMA kernel (every instantiation has the same
// shared-memory and register footprint): SMs x resident CTAs
long long tma_grid() {
    static long long g = 0;
    if (!g) {
        ensure_smem(compose_tma_kernel<true, true, false>, sizeof(SmemT));
        g = (long long)sm_count() * std::max(blocks_per_sm(compose_tma_kernel<true, true, false>, NT, sizeof(SmemT)), 1);
    }
    return g;
}

typedef PFN_cuTensorMapEncodeTiled_v12000 EncodeFn;

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

bool make_map(CUtensorMap* m, const uint8_t* base, int w, int h, int frames) {
    EncodeFn enc = get_encode();
    if (!enc || !base) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)frames};
    const cuuint64_t strides[2] = {(cuuint64_t)w, (cuuint64_t)w * h};
    const cuuint32_t box[3] = {BW, BH, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// 3D uint8 tensor map (x, y, frame) with a box_w x box_h x 1 box; false when
// the driver entry point is missing or the layout is not TMA-eligible
bool encode_u8_3d(CUtensorMap* m, const uint8_t* base, int w, int h, int frames, size_t frame_stride, int box_w,
                  int box_h) {
    EncodeFn enc = get_encode();
    if (!enc || !base || (reinterpret_cast<uintptr_t>(base) & 15) || (w & 15) || (frame_stride & 15)) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)frames};
    const cuuint64_t strides[2] = {(cuuint64_t)w, (cuuint64_t)frame_stride};
    const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

// TMA eligibility: 16-byte aligned planes with 16-byte pitches
bool tma_ok(const PlaneBatch& p) {
    return p.base && (p.w % 16) == 0 && (reinterpret_cast<uintptr_t>(p.base) % 16) == 0 &&
           (p.stride % 16) == 0 && p.stride == (size_t)p.w * p.h;
}

template <bool L, bool C, bool RGBO = false>
bool launch_tma(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, const FramePlan* plan, int frames,
                CropGeom g, Tables T, uint8_t* oy, uint8_t* ocb, uint8_t* ocr, cudaStream_t st,
                uint8_t* scr = nullptr) {
    if ((L && !tma_ok(y)) || (C && (!tma_ok(cb) || !tma_ok(cr)))) return false;
    CUtensorMap my, mb, mr;
    memset(&my, 0, sizeof my);
    memset(&mb, 0, sizeof mb);
    memset(&mr, 0, sizeof mr);
    if (L && !make_map(&my, y.base, y.w, y.h, frames)) return false;
    if (C && (!make_map(&mb, cb.base, cb.w, cb.h, frames) || !make_map(&mr, cr.base, cr.w, cr.h, frames)))
        return false;
    const int W = L ? y.w : cb.w, H = L ? y.h : cb.h;
    const int tx = (W + TW - 1) / TW, ty = (H + TTH - 1) / TTH;
    const long long total = (long long)tx * ty * frames;
    tile_prep_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(plan, frames, tx, ty, W, H, y.w, y.h,
                                                                    cb.w, cb.h, g, T, L ? 1 : 0, C ? 1 : 0);
    const size_t smem = sizeof(SmemT);
    ensure_smem(compose_tma_kernel<L, C, RGBO>, smem);
    const long long grid = std::min<long long>(total, tma_grid());
    compose_tma_kernel<L, C, RGBO><<<(unsigned)grid, NT, smem, st>>>(y, cb, cr, plan, g, T, tx, ty, frames, my, mb,
                                                                     mr, oy, ocb, ocr, scr);
    return true;
}

template <bool L, bool C>
void launch_tiles(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, const FramePlan* plan, int frames,
                  CropGeom g, const Tables& T, uint8_t* oy, uint8_t* ocb, uint8_t* ocr,
                  cudaStream_t st) {
    const int W = L ? y.w : cb.w, H = L ? y.h : cb.h;
    const int tx = (W + TW - 1) / TW, ty = (H + TH - 1) / TH;
    const size_t smem = sizeof(Smem);
    ensure_smem(compose_kernel<L, C>, smem);
    for (int f0 = 0; f0 < frames; f0 += 65535) {
        const int nf = min(65535, frames - f0);
        PlaneBatch a = y, b = cb, c = cr;
        if (a.base) a.base += (size_t)f0 * a.stride;
        if (b.base) b.base += (size_t)f0 * b.stride;
        if (c.base) c.base += (size_t)f0 * c.stride;
        Tables t = T;
        t.rxf += (size_t)f0 * T.h;
        t.ryf += (size_t)f0 * T.h;
        if (t.pxf) {
            t.pxf += (size_t)f0 * T.ch;
            t.pyf += (size_t)f0 * T.ch;
        }
        dim3 grid(tx * ty, nf);
        compose_kernel<L, C><<<grid, NT, smem, st>>>(
            a, b, c, plan + f0, g, t, tx, oy ? oy + (size_t)f0 * y.stride : nullptr,
            ocb ? ocb + (size_t)f0 * cb.stride : nullptr, ocr ? ocr + (size_t)f0 * cr.stride : nullptr);
    }
}

// bytes of the per-launch tables (row starts, crop tables, tile parameters)
size_t table_bytes(int w, int h, int cw, int ch, int frames) {
    const bool sep = cw > 0 && !(cw == w && ch == h);
    const size_t nrow = (size_t)frames * h, ncrow = (size_t)frames * ch;
    const int tw_tiles = sep ? std::max((w + TW - 1) / TW, (cw + TW - 1) / TW) : (w + TW - 1) / TW;
    const int th_tiles = sep ? std::max((h + TH - 1) / TH, (ch + TH - 1) / TH) : (h + TH - 1) / TH;
    const size_t ntiles = (size_t)tw_tiles * th_tiles * frames;
    return sizeof(long long) * (2 * nrow + 2 * ncrow) + (sizeof(int) + sizeof(double)) * (w + h) +
           sizeof(TileParams) * ntiles + 512;
}

// RGB output (Y/Cb/Cr -> RGB fused into K8's store) is possible for 4:4:4
// chroma on the TMA path with crop margins of at least one pixel
bool rgb_ok(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, int frames, double crop_ratio) {
    const CropGeom g = crop_geom(y.w, y.h, crop_ratio);
    return frames <= 65535 && cb.w == y.w && cb.h == y.h && g.mx >= 1 && g.my >= 1 && tma_ok(y) && tma_ok(cb) &&
           tma_ok(cr);
}

void run_compose(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, const FramePlan* plan, int frames,
                 double crop_ratio, uint8_t* out_y, uint8_t* out_cb, uint8_t* out_cr, cudaStream_t st,
                 void* scratch = nullptr, size_t scratch_bytes = 0, uint8_t* out_rgb = nullptr) {
    if (frames <= 0) return;
    const CropGeom g = crop_geom(y.w, y.h, crop_ratio);
    const bool chroma = (cb.base && cr.base && out_cb && out_cr) || out_rgb;
    const int w = y.w, h = y.h, cw = chroma ? cb.w : 0, ch = chroma ? cb.h : 0;
    // per-launch tables: the caller's scratch, else a stream-ordered allocation
    const size_t nrow = (size_t)frames * h, ncrow = (size_t)frames * ch;
    const size_t tbytes = table_bytes(w, h, cw, ch, frames);
    // RGB output: + the per-CTA Cb / Cr tiles (2 buffers x 2 planes x TTH x TW)
    const size_t bytes = tbytes + (out_rgb ? (size_t)tma_grid() * 4 * TTH * TW + 256 : 0);
    char* buf = nullptr;
    const bool own = !(scratch && scratch_bytes >= bytes);
    if (!own) buf = static_cast<char*>(scratch);
    // a failed allocation stays in cudaGetLastError for the caller's check_launch
    else if (cudaMallocAsync((void**)&buf, bytes, st) != cudaSuccess) return;
    Tables T;
    long long* q = reinterpret_cast<long long*>(buf);
    T.rxf = q;
    T.ryf = q + nrow;
    T.pxf = chroma ? q + 2 * nrow : nullptr;
    T.pyf = chroma ? q + 2 * nrow + ncrow : nullptr;
    double* dd = reinterpret_cast<double*>(q + 2 * nrow + 2 * ncrow);
    T.cfx = dd;
    T.cfy = dd + w;
    int* ii = reinterpret_cast<int*>(dd + w + h);
    T.cx0 = ii;
    T.cy0 = ii + w;
    T.h = h;
    T.ch = ch;
    T.tiles = reinterpret_cast<int4*>(((uintptr_t)(ii + w + h) + 15) & ~uintptr_t(15));
    const int rows = max(max(h, ch), w);
    for (int f0 = 0; f0 < frames; f0 += 65535) {
        const int nf = min(65535, frames - f0);
        Tables t = T;
        t.rxf += (size_t)f0 * h;
        t.ryf += (size_t)f0 * h;
        if (t.pxf) {
            t.pxf += (size_t)f0 * ch;
            t.pyf += (size_t)f0 * ch;
        }
        dim3 grid((rows + 127) / 128, nf);
        compose_prep_kernel<<<grid, 128, 0, st>>>(plan + f0, w, h, cw, ch, g, t);
    }
    const bool frames_ok = frames <= 65535;
    if (out_rgb) {  // the caller checked rgb_ok
        uint8_t* scr = reinterpret_cast<uint8_t*>(((uintptr_t)(buf + tbytes) + 255) & ~uintptr_t(255));
        launch_tma<true, true, true>(y, cb, cr, plan, frames, g, T, out_rgb, nullptr, nullptr, st, scr);
    } else if (chroma && cb.w == y.w && cb.h == y.h) {
        if (!(frames_ok && launch_tma<true, true>(y, cb, cr, plan, frames, g, T, out_y, out_cb, out_cr, st)))
            launch_tiles<true, true>(y, cb, cr, plan, frames, g, T, out_y, out_cb, out_cr, st);
    } else {
        if (!(frames_ok && launch_tma<true, false>(y, cb, cr, plan, frames, g, T, out_y, nullptr, nullptr, st)))
            launch_tiles<true, false>(y, cb, cr, plan, frames, g, T, out_y, nullptr, nullptr, st);
        if (chroma &&
            !(frames_ok && launch_tma<false, true>(y, cb, cr, plan, frames, g, T, nullptr, out_cb, out_cr, st)))
            launch_tiles<false, true>(y, cb, cr, plan, frames, g, T, nullptr, out_cb, out_cr, st);
    }
    if (own) cudaFreeAsync(buf, st);
}

}  // namespace

void launch_compose(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, const FramePlan* plan, int frames,
                    double crop_ratio, uint8_t* out_y, uint8_t* out_cb, uint8_t* out_cr,
                    cudaStream_t st, void* scratch, size_t scratch_bytes) {
    run_compose(y, cb, cr, plan, frames, crop_ratio, out_y, out_cb, out_cr, st, scratch, scratch_bytes);
}

size_t compose_scratch_bytes(int w, int h, int cw, int ch, int frames) { return table_bytes(w, h, cw, ch, frames); }

bool launch_compose_rgb(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, const FramePlan* plan, int frames,
                        double crop_ratio, uint8_t* out_rgb, cudaStream_t st) {
    if (!rgb_ok(y, cb, cr, frames, crop_ratio)) return false;
    run_compose(y, cb, cr, plan, frames, crop_ratio, nullptr, nullptr, nullptr, st, nullptr, 0, out_rgb);
    return true;
}

void launch_warp_only(const uint8_t* src, int w, int h, const FramePlan* plan, uint8_t* out,
                      cudaStream_t st) {
    // warp_similarity == compose with crop_ratio 0 (crop_resize returns its input)
    PlaneBatch y{src, (size_t)w * h, w, h}, none{nullptr, 0, 0, 0};
    run_compose(y, none, none, plan, 1, 0.0, out, nullptr, nullptr, st);
}

void launch_crop_only(const uint8_t* src, int w, int h, double crop_ratio, uint8_t* out,
                      cudaStream_t st) {
    dim3 grid((w + 127) / 128, h);
    crop_kernel<<<grid, 128, 0, st>>>(src, w, h, crop_geom(w, h, crop_ratio), out);
}

}  // namespace stabgpu
