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
// Exactness without fp64 per pixel.  Coordinates are carried in 32.32 fixed
// point (int64 adds), the bilinear blend in fp32.  Each decision the
// reference takes — integer part of a coordinate, in-bounds test, lround of
// the blended value — is taken on the fast path only when the fast value is
// provably on the same side of the decision boundary (coordinate error
// <= ~40 units of 2^-32 px against a 1024-unit guard; value error <= 1.5e-4
// against a 2.5e-4 guard).  Otherwise the pixel is queued and recomputed
// with the reference's own fp64 arithmetic — for luma including the
// reference's sequential row walk (sx += c, image_ops.cpp:124-131), which
// fl_walk (walk.h) reproduces bit for bit in closed form.  About 0.05% of
// pixels take the exact path.
#include "common.cuh"
#include "kernels.cuh"
#include "walk.h"

namespace stabgpu {

namespace {

constexpr int TW = 64, TH = 32;          // output tile
constexpr int NT = 256;                  // threads per CTA
constexpr int WTW = 72, WTH = 36;        // warped-luma tile (<= 66 x 34 used)
constexpr int SRC_W = 128, SRC_H = 80;   // staged source capacity per plane
constexpr int QCAP = 1024;               // exact-path queue
constexpr long long GUARD = 1024;        // fixed-point guard (units of 2^-32 px)
constexpr float VGUARD = 2.5e-4f;        // blended-value guard (the fast error is <= 1.5e-4)
constexpr double FIX = 4294967296.0;     // 2^32

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

struct Src {  // a plane as seen by the kernel: staged tile or the global frame
    const uint8_t* p;
    int pitch, x0, y0;
};

struct Smem {
    uint8_t src[3][SRC_H * SRC_W];
    uint8_t wt[WTH][WTW];
    uint8_t out[3][TH][TW];
    double cfx[TW], cfy[TH];      // luma crop fractions per column / row
    float cfxf[TW], cfyf[TH];
    int cx0[TW], cy0[TH];
    long long sxf[WTH], syf[WTH]; // luma warp: fixed-point x/y of (u0, v) per W row
    double rxw[WTH], ryw[WTH];    // luma warp row starts (exact reference values)
    long long pxf[TH], pyf[TH];   // chroma: fixed-point source coords of (X0, y)
    int bbox[3][4];               // staged footprint per plane
    int staged[3];
    int qn;
    unsigned q[QCAP];
};

__device__ __forceinline__ bool near_int(uint32_t f) { return f < GUARD || f > 0xFFFFFFFFu - GUARD; }

__device__ __forceinline__ float frac_f(uint32_t f) {  // top 23 bits of a 0.32 fraction
    return __uint_as_float(0x3F800000u | (f >> 9)) - 1.0f;
}

// exact uint8 -> float without I2F (a quarter-rate pipe): 2^23 + b, minus 2^23
__device__ __forceinline__ float b2f(uint32_t b) { return __int_as_float(0x4B000000 | b) - 8388608.0f; }

// fast bilinear (sample_bilinear's blend in fp32) + lround; -1 when the
// rounding decision is within the error guard of a .5 tie
__device__ __forceinline__ int blend_round(uint32_t a, uint32_t b, uint32_t c, uint32_t d, float fx,
                                           float fy) {
    const float fa = b2f(a), fc = b2f(c);
    const float top = fmaf(fx, b2f(b) - fa, fa);
    const float bot = fmaf(fx, b2f(d) - fc, fc);
    const float t = fmaf(fy, bot - top, top) + 0.5f;  // lround(v) == floor(v + 0.5), v >= 0
    const float k = floorf(t);
    const float fr = t - k;
    if (fr < VGUARD || fr > 1.0f - VGUARD) return -1;
    return __float_as_int(k + 8388608.0f) & 0x3FF;
}



__device__ __forceinline__ uint8_t at(const Src& s, int x, int y) {
    return s.p[(y - s.y0) * s.pitch + (x - s.x0)];
}

// One fast-path sample of plane `q` (pitch, origin bx0/by0) at 32.32 fixed
// point (X, Y).  Returns the byte, `out` when the coordinate is outside
// [0, w-1] x [0, h-1] (lim = w-2 / h-2 on the integer part), or -1 when a
// decision is not certain.
template <typename P>
__device__ __forceinline__ int sample_fast(P q, int pitch, int bx0, int by0, unsigned limx,
                                           unsigned limy, long long X, long long Y, int out) {
    const uint32_t fxs = (uint32_t)X, fys = (uint32_t)Y;
    if (near_int(fxs) || near_int(fys)) return -1;
    const int ix = (int)(X >> 32), iy = (int)(Y >> 32);
    if ((unsigned)ix > limx || (unsigned)iy > limy) return out;
    const int o = (iy - by0) * pitch + (ix - bx0);
    return blend_round(q[o], q[o + 1], q[o + pitch], q[o + pitch + 1], frac_f(fxs), frac_f(fys));
}

// Two planes sharing one coordinate (4:4:4 chroma): packed result b | r << 16
template <typename P>
__device__ __forceinline__ int sample_fast2(P q1, P q2, int pitch, int bx0, int by0, unsigned limx,
                                            unsigned limy, long long X, long long Y, int out) {
    const uint32_t fxs = (uint32_t)X, fys = (uint32_t)Y;
    if (near_int(fxs) || near_int(fys)) return -1;
    const int ix = (int)(X >> 32), iy = (int)(Y >> 32);
    if ((unsigned)ix > limx || (unsigned)iy > limy) return out | (out << 16);
    const int o = (iy - by0) * pitch + (ix - bx0);
    const float fx = frac_f(fxs), fy = frac_f(fys);
    const int vb = blend_round(q1[o], q1[o + 1], q1[o + pitch], q1[o + pitch + 1], fx, fy);
    const int vr = blend_round(q2[o], q2[o + 1], q2[o + pitch], q2[o + pitch + 1], fx, fy);
    return (vb < 0 || vr < 0) ? -1 : (vb | (vr << 16));
}

// Stages rows [y0, y1] x cols [x0, x1] of a plane (clipped by the caller).
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

__device__ __forceinline__ void chroma_exact(const FramePlan& p, const CropGeom& g,
                                             const ChromaMap& cm, const uint8_t* gcb,
                                             const uint8_t* gcr, int cw, int ch, int x, int y,
                                             uint8_t& ob, uint8_t& orr) {
    double px, py;
    chroma_coords(p, g, cm, x, y, px, py);
    ob = orr = 128;
    if (px >= 0.0 && py >= 0.0 && px <= (double)cw - 1.0 && py <= (double)ch - 1.0) {
        ob = round_u8(sample_bilinear(gcb, cw, ch, px, py));
        orr = round_u8(sample_bilinear(gcr, cw, ch, px, py));
    }
}

// min/max of 4 corner coordinates held by 4 consecutive lanes -> staged bbox
__device__ __forceinline__ void corner_bbox(double x, double y, unsigned mask, int k, int w, int h,
                                            int* bb) {
    double xmn = x, xmx = x, ymn = y, ymx = y;
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
        xmn = fmin(xmn, __shfl_xor_sync(mask, xmn, o));
        xmx = fmax(xmx, __shfl_xor_sync(mask, xmx, o));
        ymn = fmin(ymn, __shfl_xor_sync(mask, ymn, o));
        ymx = fmax(ymx, __shfl_xor_sync(mask, ymx, o));
    }
    if (k == 0) {
        bb[0] = max(0, (int)floor(xmn) - 1);
        bb[1] = max(0, (int)floor(ymn) - 1);
        bb[2] = min(w - 1, (int)floor(xmx) + 2);
        bb[3] = min(h - 1, (int)floor(ymx) + 2);
    }
}

// Exact luma W pixel.  Level 1: the direct fp64 coordinates rx + u*c differ
// from the reference's walked ones by <= u*2^-43 px (|s| < 2^11; scaled
// bound below), so unless a coordinate sits that close to an integer / the
// frame edge, or the fp64 blend that close to a .5 tie, the direct result IS
// the reference result.  Level 2 (about once per two 1080p frames): fl_walk.
__device__ uint8_t w_exact(const uint8_t* __restrict__ g, int w, int h, const FramePlan& p,
                           double rx, double ry, int u) {
    const double sx = dadd(rx, dmul((double)u, p.c)), sy = dsub(ry, dmul((double)u, p.sn));
    // walk-vs-direct bound: u half-ulps of the largest |coordinate| + 2 ulps of rounding
    const double mag = fmax(fmax(fabs(sx), fabs(sy)), fmax(fabs(rx), fabs(ry))) + fabs((double)u) + 2.0;
    const double tol = ldexp(mag, -52) * ((double)u + 4.0);
    bool sure = true;
    const double bx[3] = {sx - floor(sx), sx, sx - ((double)w - 1.0)};
    const double by[3] = {sy - floor(sy), sy, sy - ((double)h - 1.0)};
    // near an integer (x0 / fx change) or near either domain edge
    if (fmin(bx[0], 1.0 - bx[0]) <= tol || fabs(bx[1]) <= tol || fabs(bx[2]) <= tol) sure = false;
    if (fmin(by[0], 1.0 - by[0]) <= tol || fabs(by[1]) <= tol || fabs(by[2]) <= tol) sure = false;
    if (sure) {
        const double v = sample_bilinear(g, w, h, sx, sy);
        const double fr = v - floor(v);
        if (fabs(fr - 0.5) > 255.0 * 4.0 * tol + 1e-9) return round_u8(v);
    }
    return round_u8(sample_bilinear(g, w, h, fl_walk(rx, p.c, u), fl_walk(ry, -p.sn, u)));
}

template <bool LUMA, bool CHROMA>
__global__ void __launch_bounds__(NT) compose_kernel(PlaneBatch Y, PlaneBatch CB, PlaneBatch CR,
                                                     const FramePlan* __restrict__ plan, CropGeom g,
                                                     int tiles_x, uint8_t* __restrict__ oY,
                                                     uint8_t* __restrict__ oCB,
                                                     uint8_t* __restrict__ oCR) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int f = blockIdx.y;
    const FramePlan p = plan[f];
    const int tid = threadIdx.x;
    // tile in the output plane (luma plane when LUMA, chroma plane otherwise)
    const int W = LUMA ? Y.w : CB.w, H = LUMA ? Y.h : CB.h;
    const int X0 = (blockIdx.x % tiles_x) * TW, Y0 = (blockIdx.x / tiles_x) * TH;
    const int nx = min(TW, W - X0), ny = min(TH, H - Y0);
    const bool identity = g.mx == 0 && g.my == 0;
    if (tid == 0) S.qn = 0;

    // ------------------------------------------------------------ setup
    const int w = Y.w, h = Y.h;
    const uint8_t* gy = LUMA ? Y.base + (size_t)f * Y.stride : nullptr;
    int u0 = 0, v0 = 0, nu = 0, nv = 0;
    const long long CF = p.cf, SNF = p.snf;
    if (LUMA) {
        if (identity) {
            u0 = X0;
            v0 = Y0;
            nu = nx;
            nv = ny;
        } else {
            u0 = (int)dadd((double)g.mx, dmul((double)X0, g.step_x));
            v0 = (int)dadd((double)g.my, dmul((double)Y0, g.step_y));
            nu = min((int)dadd((double)g.mx, dmul((double)(X0 + nx - 1), g.step_x)) + 1, w - 1) - u0 + 1;
            nv = min((int)dadd((double)g.my, dmul((double)(Y0 + ny - 1), g.step_y)) + 1, h - 1) - v0 + 1;
            if (tid < nx) {
                const double sx = dadd((double)g.mx, dmul((double)(X0 + tid), g.step_x));
                S.cx0[tid] = (int)sx;
                S.cfx[tid] = dsub(sx, (double)(int)sx);
                S.cfxf[tid] = (float)S.cfx[tid];
            }
            if (tid >= 64 && tid < 64 + ny) {
                const int r = tid - 64;
                const double sy = dadd((double)g.my, dmul((double)(Y0 + r), g.step_y));
                S.cy0[r] = (int)sy;
                S.cfy[r] = dsub(sy, (double)(int)sy);
                S.cfyf[r] = (float)S.cfy[r];
            }
        }
        if (tid >= 128 && tid < 128 + nv) {  // W rows: exact row starts + fixed point at u0
            const int r = tid - 128;
            double rx, ry;
            row_start(p, v0 + r, rx, ry);
            S.rxw[r] = rx;
            S.ryw[r] = ry;
            S.sxf[r] = __double2ll_rn(dmul(dadd(rx, dmul((double)u0, p.c)), FIX));
            S.syf[r] = __double2ll_rn(dmul(dsub(ry, dmul((double)u0, p.sn)), FIX));
        }
        if (tid >= 224 && tid < 228) {  // luma source footprint of the W tile: 4 corners
            const int k = tid - 224;
            const int u = u0 + ((k & 1) ? nu - 1 : 0), v = v0 + ((k & 2) ? nv - 1 : 0);
            double rx, ry;
            row_start(p, v, rx, ry);
            corner_bbox(rx + u * p.c, ry - u * p.sn, 0xFu << 0, k, w, h, S.bbox[0]);
        }
    }
    const int cw = CB.w, ch = CB.h;
    ChromaMap cm{0, 0, false};
    long long KXX = 0, KYX = 0;
    if (CHROMA) {
        cm.fxl = (double)w / cw;
        cm.fyl = (double)h / ch;
        cm.crop = g.mx != 0 || g.my != 0;
        KXX = p.kxx;
        KYX = p.kyx;
        if (tid >= 192 && tid < 192 + ny) {
            const int r = tid - 192;
            double px, py;
            chroma_coords(p, g, cm, X0, Y0 + r, px, py);
            S.pxf[r] = __double2ll_rn(dmul(px, FIX));
            S.pyf[r] = __double2ll_rn(dmul(py, FIX));
        }
        if (tid >= 228 && tid < 232) {  // chroma footprint: 4 corners
            const int k = tid - 228;
            double px, py;
            chroma_coords(p, g, cm, X0 + ((k & 1) ? nx - 1 : 0), Y0 + ((k & 2) ? ny - 1 : 0), px, py);
            corner_bbox(px, py, 0xFu << 4, k, cw, ch, S.bbox[1]);
            if (k == 0) {
                // bbox[2] mirrors bbox[1] (same geometry for both chroma planes)
            }
        }
    }
    __syncthreads();
    // ------------------------------------------------------------ staging
    const uint8_t* gcb = CHROMA ? CB.base + (size_t)f * CB.stride : nullptr;
    const uint8_t* gcr = CHROMA ? CR.base + (size_t)f * CR.stride : nullptr;
    int bb[3][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        bb[0][j] = S.bbox[0][j];
        bb[1][j] = bb[2][j] = S.bbox[1][j];
    }
    __syncthreads();
    if (LUMA) stage(gy, w, bb[0][0], bb[0][1], bb[0][2], bb[0][3], S.src[0], S.bbox[0], &S.staged[0]);
    if (CHROMA) {
        stage(gcb, cw, bb[1][0], bb[1][1], bb[1][2], bb[1][3], S.src[1], S.bbox[1], &S.staged[1]);
        stage(gcr, cw, bb[2][0], bb[2][1], bb[2][2], bb[2][3], S.src[2], S.bbox[2], &S.staged[2]);
    }
    __syncthreads();
    // ------------------------------------------------------------ luma W tile
    if (LUMA) {
        uint8_t* wdst = identity ? &S.out[0][0][0] : &S.wt[0][0];
        const int wp = identity ? TW : WTW;
        const unsigned limx = (unsigned)(w - 2), limy = (unsigned)(h - 2);
        const int lane = tid & 31, warp = tid >> 5;
        const bool stg = S.staged[0];
        const int bx0 = S.bbox[0][0], by0 = S.bbox[0][1];
        // warp per row, 2 adjacent pixels per lane (64 columns), tail columns after
        for (int r = warp; r < nv; r += NT / 32) {
            const long long SXr = S.sxf[r], SYr = S.syf[r];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int c = 2 * lane + k;
                if (c >= nu) break;
                const long long SX = SXr + (long long)c * CF, SY = SYr - (long long)c * SNF;
                const int val = stg ? sample_fast(&S.src[0][0], SRC_W, bx0, by0, limx, limy, SX, SY, 0)
                                    : sample_fast(gy, w, 0, 0, limx, limy, SX, SY, 0);
                if (val < 0) push(S, (unsigned)(r * nu + c));
                else wdst[r * wp + c] = (uint8_t)val;
            }
        }
        for (int i = tid; i < (nu - 64) * nv; i += NT) {  // columns 64.. (at most 2)
            const int r = i / (nu - 64), c = 64 + i - r * (nu - 64);
            const long long SX = S.sxf[r] + (long long)c * CF, SY = S.syf[r] - (long long)c * SNF;
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
                wdst[r * wp + c] = w_exact(gy, w, h, p, S.rxw[r], S.ryw[r], u0 + c);
            }
        } else {  // overflow: every pixel exactly (never seen in practice)
            for (int i = tid; i < nu * nv; i += NT) {
                const int r = i / nu, c = i - r * nu;
                wdst[r * wp + c] = w_exact(gy, w, h, p, S.rxw[r], S.ryw[r], u0 + c);
            }
        }
        __syncthreads();
        if (tid == 0) S.qn = 0;
        __syncthreads();
        // ---- crop_resize of the warped tile (image_ops.cpp:151-157)
        if (!identity) {
            const int lane = tid & 31, warp = tid >> 5;
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
    if (CHROMA) {
        const unsigned limx = (unsigned)(cw - 2), limy = (unsigned)(ch - 2);
        const int lane = tid & 31, warp = tid >> 5;
        const bool stg = S.staged[1] && S.staged[2];
        const int bx0 = S.bbox[1][0], by0 = S.bbox[1][1];
        for (int r = warp; r < ny; r += NT / 32) {
            const long long PXr = S.pxf[r], PYr = S.pyf[r];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int c = 2 * lane + k;
                if (c >= nx) break;
                const long long PX = PXr + (long long)c * KXX, PY = PYr + (long long)c * KYX;
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
                const int r = i / (TW / 16), c = (i % (TW / 16)) * 16;
                const uint4 v = *reinterpret_cast<const uint4*>(&S.out[k][r][c]);
                __stcs(reinterpret_cast<uint4*>(base + (size_t)(Y0 + r) * pw + X0 + c), v);
            }
        } else {
            for (int i = tid; i < nx * ny; i += NT) {
                const int r = i / nx, c = i - r * nx;
                base[(size_t)(Y0 + r) * pw + X0 + c] = S.out[k][r][c];
            }
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

template <bool L, bool C>
void launch_tiles(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, const FramePlan* plan, int frames,
                  CropGeom g, uint8_t* oy, uint8_t* ocb, uint8_t* ocr, cudaStream_t st) {
    const int W = L ? y.w : cb.w, H = L ? y.h : cb.h;
    const int tx = (W + TW - 1) / TW, ty = (H + TH - 1) / TH;
    const size_t smem = sizeof(Smem);
    cudaFuncSetAttribute(compose_kernel<L, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int f0 = 0; f0 < frames; f0 += 65535) {
        const int nf = min(65535, frames - f0);
        PlaneBatch a = y, b = cb, c = cr;
        if (a.base) a.base += (size_t)f0 * a.stride;
        if (b.base) b.base += (size_t)f0 * b.stride;
        if (c.base) c.base += (size_t)f0 * c.stride;
        dim3 grid(tx * ty, nf);
        compose_kernel<L, C><<<grid, NT, smem, st>>>(
            a, b, c, plan + f0, g, tx, oy ? oy + (size_t)f0 * y.stride : nullptr,
            ocb ? ocb + (size_t)f0 * cb.stride : nullptr, ocr ? ocr + (size_t)f0 * cr.stride : nullptr);
    }
}

}  // namespace

void launch_compose(PlaneBatch y, PlaneBatch cb, PlaneBatch cr, const FramePlan* plan, int frames,
                    double crop_ratio, uint8_t* out_y, uint8_t* out_cb, uint8_t* out_cr,
                    cudaStream_t st) {
    if (frames <= 0) return;
    const CropGeom g = crop_geom(y.w, y.h, crop_ratio);
    const bool chroma = cb.base && cr.base && out_cb && out_cr;
    if (chroma && cb.w == y.w && cb.h == y.h) {
        launch_tiles<true, true>(y, cb, cr, plan, frames, g, out_y, out_cb, out_cr, st);
    } else {
        launch_tiles<true, false>(y, cb, cr, plan, frames, g, out_y, nullptr, nullptr, st);
        if (chroma) launch_tiles<false, true>(y, cb, cr, plan, frames, g, nullptr, out_cb, out_cr, st);
    }
}

void launch_warp_only(const uint8_t* src, int w, int h, const FramePlan* plan, uint8_t* out,
                      cudaStream_t st) {
    // warp_similarity == compose with crop_ratio 0 (crop_resize returns its input)
    PlaneBatch y{src, (size_t)w * h, w, h}, none{nullptr, 0, 0, 0};
    launch_tiles<true, false>(y, none, none, plan, 1, crop_geom(w, h, 0.0), out, nullptr, nullptr, st);
}

void launch_crop_only(const uint8_t* src, int w, int h, double crop_ratio, uint8_t* out,
                      cudaStream_t st) {
    dim3 grid((w + 127) / 128, h);
    crop_kernel<<<grid, 128, 0, st>>>(src, w, h, crop_geom(w, h, crop_ratio), out);
}

}  // namespace stabgpu
