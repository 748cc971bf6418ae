// k_detect.cu — K2/K3/K4: Shi-Tomasi corners, batched over detection frames.
//
// Reference: gradients (image_ops.cpp:79-96), min_eig + response_in_rect
// (features.cpp:41-74) and detect_corners (features.cpp:89-141).
//
// Exactness argument.  A central difference of uint8 pixels is
// k/2 with |k| <= 255, so every product dx*dx, dx*dy, dy*dy in the reference
// is an exact multiple of 1/4 and the block sums are exact in any order.  The
// kernels therefore sum integer products and scale by 0.25 (exact), then
// evaluate min_eig with correctly rounded fp64 ops in the reference order:
// the response bits are identical to the reference, so the candidate set,
// the sort order and the greedy selection are identical too.
//
// K2 (resp_max_kernel): response over the ROI, block max, atomicMax of the
//     bit pattern (responses are >= 0, so bit order == value order).
// K3 (cand_kernel): recomputes the response (cheaper than writing an 8 B/px
//     map), keeps r >= quality*max && r > 0, warp-ballot compaction.
// K4 (select_kernel): one CTA per detection frame.  Candidates are bucketed
//     by a monotone 13-bit-truncated float key (histogram + scatter), then
//     consumed in score order in chunks of whole buckets: each chunk is
//     prefiltered against the corners accepted so far (a grid of cells >=
//     min_distance, or, when every candidate is listed, an exact exclusion
//     bitmap), the survivors are sorted by (score desc, y*w+x asc) — the
//     reference comparator, features.cpp:119-123 — and one warp runs the
//     greedy scan 32 candidates at a time with ballots, which reproduces the
//     sequential rank-order rule exactly, including the early stop at
//     max_corners.  A bucket larger than a chunk (large ties) is merge-sorted
//     in global memory first.
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace stabgpu {

namespace {

constexpr int RTW = 32, RTH = 16;  // response tile
constexpr int kHwMax = 256;        // K4: disc half-widths tabulated for row offsets 0 .. kHwMax-1

__device__ __forceinline__ double min_eig_q(int sxx4, int sxy4, int syy4) {
    // features.cpp:41-45 on the exact quarter-integer sums
    const double sxx = (double)sxx4 * 0.25, sxy = (double)sxy4 * 0.25, syy = (double)syy4 * 0.25;
    const double half_trace = dmul(0.5, dadd(sxx, syy));
    const double half_diff = dmul(0.5, dsub(sxx, syy));
    return dsub(half_trace, dsqrt(dadd(dmul(half_diff, half_diff), dmul(sxy, sxy))));
}

// Shared tile computation: integer structure-tensor sums for a RTW x RTH tile
// at (X0, Y0).  Products outside the frame are zero, which is exactly the
// reference's truncated window (features.cpp:55-60).
template <int H>
struct RespTile {
    static constexpr int PW = RTW + 2 * H, PH = RTH + 2 * H;
    static constexpr int IW = PW + 2, IH = PH + 2;
    uint8_t img[IH][IW];
    int pxx[PH][PW], pxy[PH][PW], pyy[PH][PW];

    __device__ void load(const uint8_t* __restrict__ f, int w, int h, int X0, int Y0) {
        for (int i = threadIdx.x; i < IH * IW; i += blockDim.x) {
            const int r = i / IW, c = i % IW;
            const int y = clampi(Y0 - H - 1 + r, 0, h - 1), x = clampi(X0 - H - 1 + c, 0, w - 1);
            img[r][c] = __ldg(f + (size_t)y * w + x);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < PH * PW; i += blockDim.x) {
            const int r = i / PW, c = i % PW;
            const int x = X0 - H + c, y = Y0 - H + r;
            int gx = 0, gy = 0;
            if (x >= 0 && x < w && y >= 0 && y < h) {
                gx = (int)img[r + 1][c + 2] - (int)img[r + 1][c];
                gy = (int)img[r + 2][c + 1] - (int)img[r][c + 1];
            }
            pxx[r][c] = gx * gx;
            pxy[r][c] = gx * gy;
            pyy[r][c] = gy * gy;
        }
        __syncthreads();
    }

    __device__ double response(int tx, int ty) const {
        int sxx = 0, sxy = 0, syy = 0;
#pragma unroll
        for (int dy = 0; dy <= 2 * H; ++dy)
#pragma unroll
            for (int dx = 0; dx <= 2 * H; ++dx) {
                sxx += pxx[ty + dy][tx + dx];
                sxy += pxy[ty + dy][tx + dx];
                syy += pyy[ty + dy][tx + dx];
            }
        return min_eig_q(sxx, sxy, syy);
    }
};

template <int H>
__global__ void __launch_bounds__(256) resp_max_kernel(PlaneBatch fr, stabgpu_roi roi,
                                                       unsigned long long* __restrict__ maxbits) {
    __shared__ RespTile<H> t;
    __shared__ unsigned long long wmax[8];
    const uint8_t* f = fr.base + (size_t)blockIdx.z * fr.stride;
    const int X0 = roi.x0 + blockIdx.x * RTW, Y0 = roi.y0 + blockIdx.y * RTH;
    t.load(f, fr.w, fr.h, X0, Y0);
    unsigned long long m = 0;
    for (int i = threadIdx.x; i < RTW * RTH; i += blockDim.x) {
        const int tx = i % RTW, ty = i / RTW;
        if (X0 + tx < roi.x1 && Y0 + ty < roi.y1) {
            const double r = t.response(tx, ty);
            if (r > 0.0) m = max(m, dbits(r));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < 8; ++i) m = max(m, wmax[i]);
        if (m) atomicMax(&maxbits[blockIdx.z], m);
    }
}

template <int H>
__global__ void __launch_bounds__(256) cand_kernel(PlaneBatch fr, stabgpu_roi roi, double quality,
                                                   const unsigned long long* __restrict__ maxbits,
                                                   unsigned int* __restrict__ count,
                                                   unsigned long long* __restrict__ cand_key,
                                                   unsigned int* __restrict__ cand_idx, size_t cap) {
    const unsigned long long mb = maxbits[blockIdx.z];
    if (mb == 0) return;  // max_response <= 0: no corners (features.cpp:103-105)
    __shared__ RespTile<H> t;
    const uint8_t* f = fr.base + (size_t)blockIdx.z * fr.stride;
    const int X0 = roi.x0 + blockIdx.x * RTW, Y0 = roi.y0 + blockIdx.y * RTH;
    t.load(f, fr.w, fr.h, X0, Y0);
    const double thr = dmul(quality, __longlong_as_double((long long)mb));
    const int lane = threadIdx.x & 31;
    for (int i0 = 0; i0 < RTW * RTH; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const int tx = i % RTW, ty = i / RTW;
        double r = 0.0;
        bool keep = false;
        if (X0 + tx < roi.x1 && Y0 + ty < roi.y1) {
            r = t.response(tx, ty);
            keep = r >= thr && r > 0.0;
        }
        const unsigned ball = __ballot_sync(0xffffffffu, keep);
        if (!ball) continue;
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(&count[blockIdx.z], (unsigned)__popc(ball));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
            const size_t pos = (size_t)blockIdx.z * cap + base + __popc(ball & ((1u << lane) - 1));
            cand_key[pos] = dbits(r);
            cand_idx[pos] = (unsigned)((Y0 + ty) * fr.w + X0 + tx);
        }
    }
}

// ---------------------------------------------------------------------------
// Streaming response (block_size 3): a warp owns 30 output columns (lanes
// 1..30; lanes 0 and 31 carry the box halo) and walks a band of rows.  Image
// values roll through registers (row r-1, r, r+1), horizontal neighbours come
// by shuffle, integer products are box-summed horizontally by shuffle and
// vertically over the last three rows.  min_eig is first evaluated in fp32
// with a rigorous bound |r32 - r| <= 2^-22 * half_trace (inputs are exact in
// fp32); only pixels the bound cannot decide take the exact
// fp64 reference arithmetic (min_eig_q).
constexpr int SW_COLS = 30;  // output columns per warp
constexpr int SW_BAND = 64;  // output rows per CTA
constexpr float SW_EPS = 7.62939453125e-06f;  // 2^-17: >= 8x the bound with sqrt.approx (rel. err. <= 2^-21)

__device__ __forceinline__ unsigned resp_bin(float r) { return min(__float_as_uint(r) >> 20, (unsigned)kRespBins - 1); }

__device__ __forceinline__ float sqrt_approx(float v) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

// The CTA's band (rows Y0-2 .. Y1+1, 256 columns from a 16-byte aligned xb)
// is staged in shared memory first — 16-byte loads for interior blocks, byte
// loads with the reference's clamped indices at the frame edges — so the row
// loop only reads shared memory; staged values outside the frame are the
// clamped pixels, which is exactly what the gradient clamps read.
constexpr int SB_W = 272;                 // staged columns (>= 15 + 8 * 30 + 2 + 1)
constexpr int SB_H = SW_BAND + 4;         // staged rows

// Appends a warp's buffered candidates to the frame's list (one atomic).
__device__ __forceinline__ int flush_cands(DetectScratch& s, int d, const unsigned long long* key,
                                           const unsigned* idx, int n) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(&s.count[d], (unsigned)n);
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    for (int k = lane; k < n; k += 32) {
        s.cand_key[(size_t)d * s.cap + base + k] = key[k];
        s.cand_idx[(size_t)d * s.cap + base + k] = idx[k];
    }
    __syncwarp();
    return 0;
}

// MODE 0: a proven lower bound of the per-frame max response + histogram of
//         fp32 responses, both over the output rows y = 8k only (any lower
//         bound of the max keeps the max pixel above the cut, and the
//         histogram only steers the cut), so only product rows 8k-1 .. 8k+1
//         are formed.
// MODE 1: candidates r >= lo[d] (or the threshold itself when redo) with r > 0.
template <int MODE>
__global__ void __launch_bounds__(256) resp_stream_kernel(PlaneBatch fr, stabgpu_roi roi, double quality,
                                                          DetectScratch s, int redo) {
    __shared__ unsigned sh[MODE == 0 ? kRespBins : 1];
    __shared__ __align__(16) uint8_t band[SB_H][SB_W];
    constexpr int WB = MODE == 1 ? 128 : 1;  // per-warp candidate buffer (flushed with one atomic)
    __shared__ unsigned long long wkey[8][WB];
    __shared__ unsigned widx[8][WB];
    const int d = blockIdx.z;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double lo = 0.0, hi_excl = 0.0;  // redo: the band [threshold, first cut) not yet listed
    if (MODE == 1) {
        if (redo) {
            if (!(s.flags[d] & 2)) return;
            lo = dmul(quality, __longlong_as_double((long long)s.maxbits[d]));
            hi_excl = s.lo[d];
        } else {
            lo = s.lo[d];
        }
    } else {
        for (int i = threadIdx.x; i < kRespBins; i += blockDim.x) sh[i] = 0;
    }
    const float lo32 = __double2float_rd(lo);
    const uint8_t* f = fr.base + (size_t)d * fr.stride;
    const int w = fr.w, h = fr.h;
    const int Y0 = roi.y0 + blockIdx.y * SW_BAND, Y1 = min(Y0 + SW_BAND, roi.y1);
    const int xs = roi.x0 + blockIdx.x * 8 * SW_COLS - 1;  // first column the CTA touches
    const int xb = xs & ~15;
    const int rows = (Y1 + 1) - (Y0 - 2) + 1;
    // ---- stage the band
    const bool inner = xb >= 0 && xb + SB_W <= w && Y0 - 2 >= 0 && Y1 + 1 <= h - 1 && (w & 15) == 0 &&
                       ((reinterpret_cast<uintptr_t>(f) & 15) == 0);
    if (inner) {
        for (int i = threadIdx.x; i < rows * (SB_W / 16); i += blockDim.x) {
            const int r = i / (SB_W / 16), c = i - r * (SB_W / 16);
            *reinterpret_cast<uint4*>(&band[r][16 * c]) =
                __ldg(reinterpret_cast<const uint4*>(f + (size_t)(Y0 - 2 + r) * w + xb) + c);
        }
    } else {
        for (int i = threadIdx.x; i < rows * SB_W; i += blockDim.x) {
            const int r = i / SB_W, c = i - r * SB_W;
            band[r][c] = __ldg(f + (size_t)clampi(Y0 - 2 + r, 0, h - 1) * w + clampi(xb + c, 0, w - 1));
        }
    }
    __syncthreads();
    // ---- rows
    const int x = xs + warp * SW_COLS + lane;  // lanes 0 and 31 carry the box halo
    const int c = x - xb;                      // 0 .. 256 (c + 1 <= 257 < SB_W)
    const bool out_col = lane >= 1 && lane <= SW_COLS && x < roi.x1;
    const bool in_x = x >= 0 && x < w;
    const uint8_t* bp = &band[0][0] + c;       // band row k at bp + k * SB_W
    int Im = bp[0], I0 = bp[SB_W];             // rows Y0-2, Y0-1
    int axx = 0, axy = 0, ayy = 0, bxx = 0, bxy = 0, byy = 0;  // box rows r-2, r-1
    unsigned long long best = 0;
    float best_low = -1.0f;
    int qn = 0;                     // MODE 1: warp buffer fill (warp-uniform)
    const uint8_t* rp = bp + SB_W;  // row r
#pragma unroll 3
    for (int r = Y0 - 1; r <= Y1; ++r, rp += SB_W) {
        if (MODE == 0 && ((r + 1) & 7) > 2) {  // product rows 8k+2 .. 8k+6: no sampled output row (8k) reads them
            Im = I0;
            I0 = rp[SB_W];
            continue;
        }
        const int L = rp[-1], R = rp[1], Ip = rp[SB_W];
        const bool inr = in_x && r >= 0 && r < h;  // products outside the frame are zero
        const int gx = inr ? R - L : 0, gy = inr ? Ip - Im : 0;
        int pxx = gx * gx, pxy = gx * gy, pyy = gy * gy;
        pxx += __shfl_up_sync(0xFFFFFFFFu, pxx, 1) + __shfl_down_sync(0xFFFFFFFFu, pxx, 1);
        pxy += __shfl_up_sync(0xFFFFFFFFu, pxy, 1) + __shfl_down_sync(0xFFFFFFFFu, pxy, 1);
        pyy += __shfl_up_sync(0xFFFFFFFFu, pyy, 1) + __shfl_down_sync(0xFFFFFFFFu, pyy, 1);
        const int y = r - 1;  // output row whose window is rows r-2 .. r
        bool keep = false;
        unsigned long long key = 0;
        if (y >= Y0 && out_col && (MODE == 1 || (y & 7) == 0)) {
            const int sxx = axx + bxx + pxx, sxy = axy + bxy + pxy, syy = ayy + byy + pyy;
            const float fxx = (float)sxx, fxy = (float)sxy, fyy = (float)syy;  // exact (< 2^24)
            // 4 * (half trace, half difference): the quarter scaling is folded in
            const float ht = 0.5f * (fxx + fyy), hd = 0.5f * (fxx - fyy);
            const float r32 = 0.25f * (ht - sqrt_approx(fmaf(hd, hd, fxy * fxy)));
            const float e = ht * SW_EPS + 1e-30f;
            if (MODE == 0) {  // rows y = 8k only: the histogram (x8) and a lower bound of the max
                if (r32 > 0.0f) {  // histogram steers the cut only
                    const unsigned bin = resp_bin(r32);
                    const unsigned peers = __match_any_sync(__activemask(), bin);
                    if (lane == __ffs(peers) - 1) atomicAdd(&sh[bin], 8u * __popc(peers));
                }
                best_low = fmaxf(best_low, r32 - e);  // max(r32 - e) over the sampled rows <= exact max
            } else if (r32 + e >= lo32) {
                const double rr = min_eig_q(sxx, sxy, syy);
                keep = rr >= lo && rr > 0.0 && (!redo || rr < hi_excl);
                key = dbits(rr);
                if (keep) best = max(best, key);  // exact max: the max pixel is always kept
            }
        }
        if (MODE == 1) {
            const unsigned ball = __ballot_sync(0xFFFFFFFFu, keep);
            if (ball) {
                if (qn + __popc(ball) > WB) {  // flush the warp's buffer (rare)
                    qn = flush_cands(s, d, wkey[warp], widx[warp], qn);
                }
                if (keep) {
                    const int k = qn + __popc(ball & ((1u << lane) - 1));
                    wkey[warp][k] = key;
                    widx[warp][k] = (unsigned)(y * w + x);
                }
                qn += __popc(ball);
            }
        }
        axx = bxx;
        axy = bxy;
        ayy = byy;
        bxx = pxx;
        bxy = pxy;
        byy = pyy;
        Im = I0;
        I0 = Ip;
    }
    if (MODE == 1) {
        if (qn) flush_cands(s, d, wkey[warp], widx[warp], qn);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
        if (lane == 0 && best) atomicMax(&s.maxbits[d], best);
    }
    if (MODE == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best_low = fmaxf(best_low, __shfl_xor_sync(0xFFFFFFFFu, best_low, o));
        if (lane == 0 && best_low > 0.0f) atomicMax(&s.mlo[d], __float_as_uint(best_low));
        __syncthreads();
        for (int i = threadIdx.x; i < kRespBins; i += blockDim.x)
            if (sh[i]) atomicAdd(&s.hist[(size_t)d * kRespBins + i], sh[i]);
    }
}

// Per frame: candidate cut lo such that about `keep` candidates lie above it
// (fp32 histogram), clamped to [quality * M, M] where M = s.mlo (a proven
// lower bound of the exact max response), so the max pixel is always kept and
// MODE 1 finds the exact max.  Exactness: the kept set {r >= lo} is a prefix
// of the reference's score order; select drops r < quality * max and falls
// back to the full list when lo > quality * max and the prefix runs out before
// max_corners.
__global__ void resp_cut_kernel(double quality, DetectScratch s, unsigned keep) {
    // one warp per frame: lane l sums bins [2047 - 64 l - 63, 2047 - 64 l]
    // (descending), a shuffle scan finds the segment where the running count
    // from the top reaches `keep`, and that lane walks it: the same bin b as
    // the serial scan from b = 2047 down to 1
    static_assert(kRespBins == 2048, "64 bins per lane");
    const int d = blockIdx.x, lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    const double m = (double)__uint_as_float(s.mlo[d]);
    double lo = 0.0;
    if (m > 0.0) {
        lo = dmul(quality, m);
        const unsigned* hs = s.hist + (size_t)d * kRespBins;
        const int top = kRespBins - 1 - 64 * lane;  // bins top .. top - 63 (bin 0 is never counted)
        unsigned seg = 0;
        for (int b = top; b > top - 64; --b) seg += b > 0 ? hs[b] : 0u;
        unsigned incl = seg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += v;
        }
        const unsigned reach = __ballot_sync(0xFFFFFFFFu, incl >= keep);
        if (reach) {
            const int l0 = __ffs(reach) - 1;
            if (lane == l0) {
                unsigned cum = incl - seg;
                for (int b = top; b > top - 64 && b > 0; --b) {
                    cum += hs[b];
                    if (cum >= keep) {
                        const double edge = (double)__uint_as_float((unsigned)b << 20);
                        lo = fmin(fmax(edge, lo), m);
                        break;
                    }
                }
            }
            lo = __shfl_sync(0xFFFFFFFFu, lo, l0);
        }
    }
    if (lane == 0) {
        s.lo[d] = lo;
        s.flags[d] = 0;
    }
}

// One launch clears a batch's per-frame detection state (max, candidate count,
// fp32 max bound, response histogram, bucket counts) instead of five memsets.
__global__ void detect_reset_kernel(DetectScratch s, int fast, int buckets) {
    const int d = blockIdx.x;
    if (threadIdx.x == 0) {
        s.maxbits[d] = 0ull;
        s.count[d] = 0u;
        if (fast) s.mlo[d] = 0u;
    }
    if (fast)
        for (int i = threadIdx.x; i < kRespBins; i += blockDim.x) s.hist[(size_t)d * kRespBins + i] = 0u;
    if (buckets)
        for (int i = threadIdx.x; i <= kBuckets; i += blockDim.x) s.bstart[(size_t)d * (kBuckets + 1) + i] = 0u;
}

// Generic block size (any odd >= 3): direct evaluation from global memory.
__global__ void resp_generic_kernel(PlaneBatch fr, stabgpu_roi roi, int half, int mode,
                                    double quality, unsigned long long* __restrict__ maxbits,
                                    unsigned int* __restrict__ count,
                                    unsigned long long* __restrict__ cand_key,
                                    unsigned int* __restrict__ cand_idx, size_t cap,
                                    double* __restrict__ resp_out) {
    const uint8_t* f = fr.base + (size_t)blockIdx.z * fr.stride;
    const int w = fr.w, h = fr.h;
    const int x = roi.x0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int y = roi.y0 + blockIdx.y;
    bool valid = x < roi.x1 && y < roi.y1;
    double r = 0.0;
    if (valid) {
        long long sxx = 0, sxy = 0, syy = 0;
        for (int wy = max(y - half, 0); wy <= min(y + half, h - 1); ++wy)
            for (int wx = max(x - half, 0); wx <= min(x + half, w - 1); ++wx) {
                const int gx = (int)f[(size_t)wy * w + min(wx + 1, w - 1)] - (int)f[(size_t)wy * w + max(wx - 1, 0)];
                const int gy = (int)f[(size_t)min(wy + 1, h - 1) * w + wx] - (int)f[(size_t)max(wy - 1, 0) * w + wx];
                sxx += gx * gx;
                sxy += gx * gy;
                syy += gy * gy;
            }
        const double dxx = (double)sxx * 0.25, dxy = (double)sxy * 0.25, dyy = (double)syy * 0.25;
        const double ht = dmul(0.5, dadd(dxx, dyy)), hd = dmul(0.5, dsub(dxx, dyy));
        r = dsub(ht, dsqrt(dadd(dmul(hd, hd), dmul(dxy, dxy))));
    }
    if (mode == 0) {  // max
        if (valid && r > 0.0) atomicMax(&maxbits[blockIdx.z], dbits(r));
    } else if (mode == 1) {  // candidates
        const unsigned long long mb = maxbits[blockIdx.z];
        if (mb == 0 || !valid) return;
        const double thr = dmul(quality, __longlong_as_double((long long)mb));
        if (r >= thr && r > 0.0) {
            const unsigned pos = atomicAdd(&count[blockIdx.z], 1u);
            cand_key[(size_t)blockIdx.z * cap + pos] = dbits(r);
            cand_idx[(size_t)blockIdx.z * cap + pos] = (unsigned)(y * w + x);
        }
    } else if (valid) {  // full response map (min_eig_response)
        resp_out[(size_t)y * w + x] = r;
    }
}

// ---------------------------------------------------------------- K4 ----

// Two shapes of the select CTA: 1024 threads, or 512 threads in <= 114 KB
// of shared memory, two frames per SM, so a batch with more frames than SMs
// runs its serial greedies (one warp per frame) two at a time on every SM.

__device__ __forceinline__ unsigned bucket_of(unsigned long long key, unsigned maxf_bits) {
    const float sf = __double2float_rn(__longlong_as_double((long long)key));
    const unsigned d = maxf_bits - __float_as_uint(sf);
    return min(d >> kBucketShift, (unsigned)(kBuckets - 1));
}

// (score desc, idx asc): a precedes b
__device__ __forceinline__ bool before(unsigned long long ka, unsigned ia, unsigned long long kb,
                                       unsigned ib) {
    return ka > kb || (ka == kb && ia < ib);
}

// Block-wide exclusive scan of one value per thread (up to 1024 threads).
__device__ unsigned block_excl_scan(unsigned v, unsigned* warp_tot, unsigned* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        unsigned t = lane < nw ? warp_tot[lane] : 0u;
        unsigned s = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_tot[lane] = s - t;
        if (lane == 31) *total = s;
    }
    __syncthreads();
    const unsigned r = warp_tot[wid] + x - v;
    __syncthreads();
    return r;
}

struct SelShared {
    unsigned bstart[kBuckets + 1];
    unsigned warp_tot[32];
    unsigned total;
    int nacc;
    int sflag;  // run_rank_sort: a bucket run longer than kMaxRun (fall back to the bitonic sort)
    short hw[kHwMax];  // disc half-width per row offset (-1: row outside the disc)
};

// bitonic sort of n (power of two) keys in shared memory, (score desc, idx asc)
__device__ void bitonic_sort(unsigned long long* key, unsigned* idx, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const bool up = (i & k) == 0;  // ascending in "before" order
                    const unsigned long long ka = key[i], kb = key[p];
                    const unsigned ia = idx[i], ib = idx[p];
                    const bool sw = up ? before(kb, ib, ka, ia) : before(ka, ia, kb, ib);
                    if (sw) {
                        key[i] = kb;
                        key[p] = ka;
                        idx[i] = ib;
                        idx[p] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// Exact order of n survivors that arrive in bucket order (the prefilter's
// compaction keeps the bucket-sorted order of the chunk): only the order
// inside each run of equal buckets is open, so every survivor counts the
// members of its run that precede it - (score desc, idx asc), a strict total
// order - and moves to run start + count.  Two barriers instead of the
// log^2(n) / 2 of a bitonic sort (78 at n = 4096).  Returns false (nothing
// moved) when a run is longer than kMaxRun.  Called by the whole CTA;
// S.sflag was cleared before the last barrier.
constexpr int kMaxRun = 96, kSortPer = 8;
__device__ bool run_rank_sort(unsigned long long* key, unsigned* idx, int n, unsigned maxf, int* sflag) {
    unsigned long long k[kSortPer];
    unsigned id[kSortPer];
    int pos[kSortPer];
    bool over = false;
#pragma unroll
    for (int q = 0; q < kSortPer; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        pos[q] = -1;
        if (i >= n) continue;
        k[q] = key[i];
        id[q] = idx[i];
        const unsigned b = bucket_of(k[q], maxf);
        int first = i, cnt = 0;
        for (int j = i - 1; j >= 0 && bucket_of(key[j], maxf) == b; --j) {
            if (i - j > kMaxRun) {
                over = true;
                break;
            }
            cnt += before(key[j], idx[j], k[q], id[q]) ? 1 : 0;
            first = j;
        }
        for (int j = i + 1; j < n && bucket_of(key[j], maxf) == b; ++j) {
            if (j - i > kMaxRun) {
                over = true;
                break;
            }
            cnt += before(key[j], idx[j], k[q], id[q]) ? 1 : 0;
        }
        pos[q] = first + cnt;
    }
    if (over) atomicOr(sflag, 1);
    __syncthreads();
    if (*reinterpret_cast<volatile int*>(sflag)) return false;
#pragma unroll
    for (int q = 0; q < kSortPer; ++q)
        if (pos[q] >= 0) {
            key[pos[q]] = k[q];
            idx[pos[q]] = id[q];
        }
    __syncthreads();
    return true;
}

// Exclusion bitmap of the accepted corners over the ROI (one bit per ROI
// pixel, rows of `wr` 32-bit words): a pixel's bit is set iff it lies closer
// than min_distance to an accepted corner, i.e. dx*dx + dy*dy < min_dist2 in
// the reference's double arithmetic (features.cpp:127-139; integer
// coordinates, so the disc is an exact set of offsets).  A candidate test is
// one shared (or L1-cached global) word; a new corner marks its disc.
__device__ __forceinline__ bool excluded(const uint32_t* bm, int wr, int x, int y) {
    return (bm[y * wr + (x >> 5)] >> (x & 31)) & 1u;
}

// largest R >= 0 with R*R < md2 (the disc's row reach), or -1 if none
__device__ __forceinline__ int disc_reach(double md2, int dy) {
    const double d2 = (double)((long long)dy * dy);
    if (!(d2 < md2)) return -1;
    int hw = (int)sqrt(fmax(md2 - d2, 0.0));
    while ((double)((long long)(hw + 1) * (hw + 1)) + d2 < md2) ++hw;
    while (hw > 0 && !((double)((long long)hw * hw) + d2 < md2)) --hw;
    return hw;
}

// Marks row dy of the disc of corner (ax, ay) (ROI coordinates).
__device__ __forceinline__ void mark_row(uint32_t* bm, int wr, int rw, int rh, int ax, int ay, int dy, double md2,
                                         const short* hwt) {
    const int yy = ay + dy;
    if (yy < 0 || yy >= rh) return;
    const int ady = abs(dy);
    const int hw = ady < kHwMax ? hwt[ady] : disc_reach(md2, dy);
    if (hw < 0) return;
    const int x0 = max(ax - hw, 0), x1 = min(ax + hw, rw - 1);
    uint32_t* row = bm + (size_t)yy * wr;
    for (int wd = x0 >> 5; wd <= (x1 >> 5); ++wd) {
        const int lo = max(x0 - 32 * wd, 0), hi = min(x1 - 32 * wd, 31);
        const uint32_t m = (hi == 31 ? 0xFFFFFFFFu : ((1u << (hi + 1)) - 1u)) & (0xFFFFFFFFu << lo);
        atomicOr(row + wd, m);
    }
}


// In-place stable-free merge sort of [0, m) by (score desc, idx asc) in
// global memory, ping-ponging with tmp (keys are unique, so rank-merging is
// exact).  Used only for buckets larger than the chunk capacity.
__device__ void global_merge_sort(unsigned long long* key, unsigned* idx, unsigned long long* tkey,
                                  unsigned* tidx, unsigned m) {
    unsigned long long *sk = key, *dk = tkey;
    unsigned *si = idx, *di = tidx;
    for (unsigned width = 1; width < m; width <<= 1) {
        for (unsigned i = threadIdx.x; i < m; i += blockDim.x) {
            const unsigned run = i / (2 * width) * (2 * width);
            const unsigned a0 = run, a1 = min(run + width, m), b0 = a1, b1 = min(run + 2 * width, m);
            const bool inA = i < a1;
            const unsigned long long k = sk[i];
            const unsigned id = si[i];
            // rank of (k,id) in the other run
            unsigned lo = inA ? b0 : a0, hi = inA ? b1 : a1;
            while (lo < hi) {
                const unsigned mid = (lo + hi) >> 1;
                if (before(sk[mid], si[mid], k, id)) lo = mid + 1;
                else hi = mid;
            }
            const unsigned pos = inA ? run + (i - a0) + (lo - b0) : run + (i - b0) + (lo - a0);
            dk[pos] = k;
            di[pos] = id;
        }
        __syncthreads();
        unsigned long long* t1 = sk;
        sk = dk;
        dk = t1;
        unsigned* t2 = si;
        si = di;
        di = t2;
    }
    if (sk != key) {
        for (unsigned i = threadIdx.x; i < m; i += blockDim.x) {
            key[i] = sk[i];
            idx[i] = si[i];
        }
    }
    __syncthreads();
}

// Warp bitonic sort of up to 32 (key, idx) pairs held one per lane, into
// the reference order (score desc, idx asc): lane 0 ends with the first.
// Empty lanes hold (0, ~0u), which sorts last (kept keys are > 0).
__device__ __forceinline__ void warp_sort32(unsigned long long& key, unsigned& idx) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, j);
            const unsigned oi = __shfl_xor_sync(0xffffffffu, idx, j);
            const bool lower = (lane & j) == 0, up = (lane & k) == 0;
            const bool ob = before(ok, oi, key, idx);
            if (lower == up ? ob : !ob) {
                key = ok;
                idx = oi;
            }
        }
}

// Does (x, y) lie closer than min_distance to an accepted corner?  Accepted
// corners are kept in a grid of cells >= min_distance (linked lists), so only
// the 3x3 neighbourhood can conflict (features.cpp:127-139).
constexpr int MAX_CELLS = 8192;
constexpr int SMEM_CORNERS = 8192;

// Grid geometry of the accepted corners: cell side (>= min_distance, so only
// the 3x3 neighbourhood can conflict), grid size, ROI origin, and the cell
// index of a ROI offset by a 32-bit reciprocal (offsets and cell < 2^16:
// v * (rcp * cell - 2^32) < 2^32, so umulhi(v, rcp) == v / cell exactly).
struct CellGrid {
    int gw, gh, cell, rx0, ry0;
    unsigned rcp;  // ceil(2^32 / cell); cell == 1 is handled apart (rcp would be 2^32)
    __device__ __forceinline__ int cell_of(int v) const { return cell == 1 ? v : (int)__umulhi((unsigned)v, rcp); }
};

__device__ __forceinline__ bool conflicts(int x, int y, const int* heads, const short2* axy, const int* anext,
                                          const CellGrid& g, unsigned imd2) {
    // imd2 = ceil(min_distance^2): for the integer d2 = dx*dx + dy*dy (coordinates
    // are 16-bit, so it fits 32 bits) d2 < md2 <=> d2 < imd2 — the reference's
    // double comparison on exact integers, without the conversions
    const int cx = g.cell_of(x - g.rx0), cy = g.cell_of(y - g.ry0);
    // the nine list heads first (independent loads; most cells are empty), then the lists
    int hd[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const int gx = cx + k % 3 - 1, gy = cy + k / 3 - 1;
        hd[k] = (gx >= 0 && gx < g.gw && gy >= 0 && gy < g.gh) ? heads[gy * g.gw + gx] : -1;
    }
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 9; ++k)
        for (int a = hd[k]; a >= 0; a = anext[a]) {
            const short2 p = axy[a];
            const int dx = x - p.x, dy = y - p.y;
            hit |= (unsigned)(dx * dx) + (unsigned)(dy * dy) < imd2;
        }
    return hit;
}

// K4 phase A over many CTAs per frame (when the scratch has bucket arrays):
// counts per bucket (shared histogram, then one global atomic per bin), an
// exclusive scan per frame, and a scatter in which each CTA reserves its range
// of every bucket once and fills it through shared-memory cursors.  The order inside a bucket is irrelevant (chunks are sorted
// exactly before the greedy), so the result is the phase the select CTA ran
// itself, with the candidate list read by ~16 CTAs per frame instead of one.
__device__ __forceinline__ bool bucket_frame(const DetectScratch& s, int d, int redo, unsigned& n,
                                             unsigned long long& thrb, unsigned& maxf, double quality) {
    if (redo && !(s.flags[d] & 2)) return false;
    n = s.count[d];
    const unsigned long long mb = s.maxbits[d];
    if (n == 0 || mb == 0) return false;
    thrb = dbits(dmul(quality, __longlong_as_double((long long)mb)));
    maxf = __float_as_uint(__double2float_rn(__longlong_as_double((long long)mb)));
    return true;
}

__global__ void __launch_bounds__(512) bucket_count_kernel(DetectScratch s, double quality, int redo) {
    const int d = blockIdx.y;
    unsigned n, maxf;
    unsigned long long thrb;
    if (!bucket_frame(s, d, redo, n, thrb, maxf, quality)) return;
    __shared__ unsigned hb[kBuckets];
    for (int b = threadIdx.x; b < kBuckets; b += blockDim.x) hb[b] = 0;
    __syncthreads();
    const unsigned long long* ck = s.cand_key + (size_t)d * s.cap;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = ck[i];
        if (k >= thrb) atomicAdd(&hb[bucket_of(k, maxf)], 1u);
    }
    __syncthreads();
    unsigned* cnt = s.bstart + (size_t)d * (kBuckets + 1);
    for (int b = threadIdx.x; b < kBuckets; b += blockDim.x)
        if (hb[b]) atomicAdd(&cnt[b], hb[b]);
}

__global__ void __launch_bounds__(1024) bucket_scan_kernel(DetectScratch s, double quality, int redo) {
    const int d = blockIdx.x;
    unsigned n, maxf;
    unsigned long long thrb;
    if (!bucket_frame(s, d, redo, n, thrb, maxf, quality)) return;
    __shared__ unsigned warp_tot[32], total;
    constexpr int PER = kBuckets / 1024;
    unsigned* st = s.bstart + (size_t)d * (kBuckets + 1);
    unsigned* cur = s.bcur + (size_t)d * kBuckets;
    unsigned v[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        v[k] = st[threadIdx.x * PER + k];
        sum += v[k];
    }
    unsigned off = block_excl_scan(sum, warp_tot, &total);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        st[threadIdx.x * PER + k] = off;
        cur[threadIdx.x * PER + k] = off;
        off += v[k];
    }
    if (threadIdx.x == 0) st[kBuckets] = total;
}

__global__ void __launch_bounds__(512) bucket_scatter_kernel(DetectScratch s, double quality, int redo) {
    // each CTA takes a contiguous slice: counts it per bucket in shared memory,
    // reserves its range of every non-empty bucket with one global atomic, then
    // scatters through shared cursors (no global atomic per candidate)
    const int d = blockIdx.y;
    unsigned n, maxf;
    unsigned long long thrb;
    if (!bucket_frame(s, d, redo, n, thrb, maxf, quality)) return;
    __shared__ unsigned hb[kBuckets];
    for (int b = threadIdx.x; b < kBuckets; b += blockDim.x) hb[b] = 0;
    __syncthreads();
    const unsigned per = (n + gridDim.x - 1) / gridDim.x;
    const unsigned lo = min(blockIdx.x * per, n), hi = min(lo + per, n);
    const unsigned long long* ck = s.cand_key + (size_t)d * s.cap;
    const unsigned* ci = s.cand_idx + (size_t)d * s.cap;
    for (unsigned i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const unsigned long long k = ck[i];
        if (k >= thrb) atomicAdd(&hb[bucket_of(k, maxf)], 1u);
    }
    __syncthreads();
    unsigned* cur = s.bcur + (size_t)d * kBuckets;
    for (int b = threadIdx.x; b < kBuckets; b += blockDim.x)
        if (hb[b]) hb[b] = atomicAdd(&cur[b], hb[b]);
    __syncthreads();
    unsigned long long* sk = s.sort_key + (size_t)d * s.cap;
    unsigned* si = s.sort_idx + (size_t)d * s.cap;
    for (unsigned i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const unsigned long long k = ck[i];
        if (k >= thrb) {
            const unsigned pos = atomicAdd(&hb[bucket_of(k, maxf)], 1u);
            sk[pos] = k;
            si[pos] = ci[i];
        }
    }
}

// y = id / w for candidate indices id = y * w + x < 2^24 (frames up to 16.7M
// pixels) by a 40-bit reciprocal: magic = ceil(2^40 / w) has error e = magic * w
// - 2^40 < w < 2^16, and id * e < 2^40, so floor(id * magic / 2^40) is exact;
// larger frames divide.
constexpr unsigned kTopFirst = 4096;  // select: candidates bucketed before the first greedy chunks

struct DivW {
    unsigned long long magic;
    unsigned w;
    bool fast;
    __device__ __forceinline__ void split(unsigned id, int& x, int& y) const {
        const unsigned q = fast ? (unsigned)((id * magic) >> 40) : id / w;
        y = (int)q;
        x = (int)(id - q * w);
    }
};

// K4: one CTA per detection frame.
//   A. the candidates >= quality * max are bucketed by a monotone 13-bit
//      truncated float key (histogram, scan, scatter) into sort_key/sort_idx,
//      so whole buckets come in score order;
//   B. the accepted-corner grid (and exclusion bitmap) are cleared, and on a
//      redo seeded with the first pass's corners;
//   C. chunks of whole buckets (<= ch candidates) in score order: every thread
//      prefilters its candidates against the corners accepted so far, the
//      survivors are compacted and sorted exactly (in registers when <= 32,
//      else a shared-memory bitonic sort), and one warp walks them 32 at a
//      time against the grid, resolving live lanes against each other in rank
//      order — the reference's sequential greedy (features.cpp:127-139),
//      including the early stop at max_corners.  A bucket larger than a chunk
//      (large ties) is merge-sorted in global memory first.
// The prefilter tests the grid, or — when every candidate is listed (no cut,
// e.g. C1: ~190k candidates for ~160 corners) and it fits in shared memory —
// an exclusion bitmap with one bit per ROI pixel (set iff closer than
// min_distance to an accepted corner: dx*dx + dy*dy < min_dist2 in the
// reference's double arithmetic on integer offsets, an exact set), which the
// whole CTA marks after each chunk's walk.
//
// Dynamic shared memory: chunk buffer (ch keys + ch indices, ch a power of
// two) | grid heads | accepted corners (when max_corners <= SMEM_CORNERS) |
// bitmap (use_bm); the bucket cursor of phase A aliases its start.
template <int SEL_THREADS>
__global__ void __launch_bounds__(SEL_THREADS, 1024 / SEL_THREADS)
    select_kernel(stabgpu_detect_cfg cfg, stabgpu_roi roi, int w, DetectScratch s,
                  double2* __restrict__ out_xy, double* __restrict__ out_score,
                  int* __restrict__ out_n, short2* __restrict__ g_axy, int* __restrict__ g_anext, int ch,
                  int use_bm, int redo) {
    static_assert(kBuckets % SEL_THREADS == 0, "per-thread strides");
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ SelShared S;
    if (redo && !(s.flags ? (s.flags[blockIdx.x] & 2) : 0)) return;
    unsigned char* p = smem;
    unsigned long long* ckey = reinterpret_cast<unsigned long long*>(p);
    p += sizeof(unsigned long long) * ch;
    unsigned* cidx = reinterpret_cast<unsigned*>(p);
    p += sizeof(unsigned) * ch;
    int* heads = reinterpret_cast<int*>(p);
    p += sizeof(int) * MAX_CELLS;
    unsigned* cursor = reinterpret_cast<unsigned*>(smem);  // aliases chunk buffer + grid during the scatter
    const int maxc = cfg.max_corners;
    const int d = blockIdx.x;
    short2* axy;
    int* anext;
    if (maxc <= SMEM_CORNERS) {
        axy = reinterpret_cast<short2*>(p);
        p += sizeof(short2) * maxc;
        anext = reinterpret_cast<int*>(p);
        p += sizeof(int) * maxc;
    } else {
        axy = g_axy + (size_t)d * maxc;
        anext = g_anext + (size_t)d * maxc;
    }
    const int rw = roi.x1 - roi.x0, rh = roi.y1 - roi.y0, wr = (rw + 31) >> 5;
    uint32_t* bm = reinterpret_cast<uint32_t*>(p);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned n = s.count[d];
    const unsigned long long mb = s.maxbits[d];
    // candidates below quality * max are not the reference's (the fast path's
    // cut may keep a few); a cut above the threshold is a prefix (may redo)
    const double thr = mb ? dmul(cfg.quality_level, __longlong_as_double((long long)mb)) : 0.0;
    const unsigned long long thrb = dbits(thr);
    const bool cut = s.flags && s.lo[d] > thr;
    if (n == 0 || mb == 0) {
        if (tid == 0 && !redo) {  // (redo: the first pass's corners stand)
            out_n[d] = 0;
            if (cut && mb != 0) {
                s.flags[d] |= 2;
                s.count[d] = 0;
            }
        }
        return;
    }
    const unsigned maxf = __float_as_uint(__double2float_rn(__longlong_as_double((long long)mb)));
    const unsigned long long* ck = s.cand_key + (size_t)d * s.cap;
    const unsigned* ci = s.cand_idx + (size_t)d * s.cap;
    unsigned long long* sk = s.sort_key + (size_t)d * s.cap;
    unsigned* si = s.sort_idx + (size_t)d * s.cap;

    int bc = kBuckets;  // round 0 takes the buckets [0, bc)
    // ---- A. histogram + exclusive scan + scatter into bucket order (or the
    // multi-CTA bucket kernels' result)
    if (s.bstart) {
        const unsigned* st = s.bstart + (size_t)d * (kBuckets + 1);
        for (int b = tid; b <= kBuckets; b += SEL_THREADS) S.bstart[b] = st[b];
        __syncthreads();
    } else {
    for (int b = tid; b < kBuckets; b += SEL_THREADS) cursor[b] = 0;
    __syncthreads();
    // (eight independent loads per thread and pass: one CTA walks up to a ROI's
    // worth of candidates, so the passes are bound by the load latency)
    for (unsigned i0 = tid; i0 < n; i0 += 8 * SEL_THREADS) {
        unsigned long long k[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const unsigned i = i0 + q * SEL_THREADS;
            k[q] = i < n ? ck[i] : 0ull;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (i0 + q * SEL_THREADS < n && k[q] >= thrb) atomicAdd(&cursor[bucket_of(k[q], maxf)], 1u);
    }
    __syncthreads();
    {
        constexpr int PER = kBuckets / SEL_THREADS;
        unsigned v[PER], sum = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            v[k] = cursor[tid * PER + k];
            sum += v[k];
        }
        unsigned off = block_excl_scan(sum, S.warp_tot, &S.total);
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            S.bstart[tid * PER + k] = off;
            cursor[tid * PER + k] = off;
            off += v[k];
        }
        if (tid == 0) S.bstart[kBuckets] = S.total;
    }
    __syncthreads();
    // Two rounds.  The scatter (two scattered global stores per candidate from
    // one SM) is what a long list costs, and the greedy usually needs only its
    // head: round 0 scatters the buckets [0, bc) holding the top ~kTopFirst
    // candidates; if they run out before max_corners, round 1 re-buckets the
    // rest, dropping every candidate that conflicts with a corner accepted so
    // far (exact: the greedy would reject it) — in the dense regime (C1) that is
    // nearly all of them.
    if (S.total > 2u * kTopFirst) {
        int lo = 1, hi = kBuckets;  // smallest b with bstart[b] >= kTopFirst
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (S.bstart[mid] >= kTopFirst) hi = mid;
            else lo = mid + 1;
        }
        bc = lo;
    }
    for (unsigned i0 = tid; i0 < n; i0 += 8 * SEL_THREADS) {
        unsigned long long k[8];
        unsigned id[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const unsigned i = i0 + q * SEL_THREADS;
            k[q] = i < n ? ck[i] : 0ull;
            id[q] = i < n ? ci[i] : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (i0 + q * SEL_THREADS >= n || k[q] < thrb) continue;
            const unsigned b = bucket_of(k[q], maxf);
            if ((int)b >= bc) continue;
            const unsigned pos = atomicAdd(&cursor[b], 1u);
            sk[pos] = k[q];
            si[pos] = id[q];
        }
    }
    __threadfence_block();
    __syncthreads();
    }
    // ---- B. grid (cells >= min_distance, <= MAX_CELLS) and bitmap, cleared
    int cell = max(1, (int)ceil(cfg.min_distance));
    while ((long long)((rw + cell - 1) / cell) * ((rh + cell - 1) / cell) > MAX_CELLS) ++cell;
    const int gw = (rw + cell - 1) / cell, gh = (rh + cell - 1) / cell;
    CellGrid cg;
    cg.gw = gw;
    cg.gh = gh;
    cg.cell = cell;
    cg.rx0 = roi.x0;
    cg.ry0 = roi.y0;
    cg.rcp = cell > 1 ? (unsigned)((0x100000000ull + (unsigned)cell - 1) / (unsigned)cell) : 0u;
    for (int c = tid; c < gw * gh; c += SEL_THREADS) heads[c] = -1;
    const double md2 = dmul(cfg.min_distance, cfg.min_distance);
    const unsigned imd2 = (unsigned)fmin(ceil(md2), 4294967295.0);
    int R = 0;  // largest row offset of a disc: R*R < md2
    if (use_bm) {
        for (size_t k = tid; k < (size_t)wr * rh; k += SEL_THREADS) bm[k] = 0u;
        R = (int)sqrt(md2);
        while ((double)((long long)(R + 1) * (R + 1)) < md2) ++R;
        while (R > 0 && !((double)((long long)R * R) < md2)) --R;
        for (int k = tid; k < kHwMax; k += SEL_THREADS) S.hw[k] = (short)min(disc_reach(md2, k), 32767);
    }
    __threadfence_block();
    __syncthreads();
    int nacc = 0;
    if (redo) {
        // continue after the first pass: its corners are the reference's first
        // out_n corners (the cut list was a prefix), so they seed the grid and
        // only the band below the first cut is scanned
        nacc = out_n[d];
        for (int k = tid; k < nacc; k += SEL_THREADS) {
            const double2 q = out_xy[(size_t)d * maxc + k];
            const int x = (int)q.x, y = (int)q.y;
            axy[k] = make_short2((short)x, (short)y);
            anext[k] = atomicExch(&heads[cg.cell_of(y - roi.y0) * gw + cg.cell_of(x - roi.x0)], k);
        }
        __threadfence_block();
        __syncthreads();
    }
    DivW dw;
    dw.w = (unsigned)w;
    dw.magic = ((1ull << 40) + (unsigned)w - 1) / (unsigned)w;
    dw.fast = s.cap <= (1u << 24) && (unsigned long long)w * (unsigned)(roi.y1 + 1) <= (1ull << 24) && w >= 16 && w < 65536;
    int marked = 0;  // corners [0, marked) are in the bitmap
    // ---- C. chunks of whole buckets in score order.  A chunk takes up to
    // `che` candidates; the survivors of its prefilter must fit the chunk buffer
    // (ch).  che adapts: once the accepted corners exclude nearly everything
    // (few survivors per chunk) it doubles, up to 32 candidates per thread, so
    // the tail of a long list costs a handful of passes instead of one
    // barrier-bound pass per ch candidates; a chunk whose survivors overflow
    // the buffer is retried with half the size (nothing was changed yet; at
    // che <= ch they always fit); many survivors halve it (down to 256), so
    // the early chunks mark their corners' discs before the neighbours of a
    // strong corner are sorted and walked.  Any chunking is exact: the prefilter only
    // drops candidates that conflict with corners accepted before the chunk.
    int b0 = 0;
    const unsigned che_min = min(256u, (unsigned)ch), che_max = 32u * SEL_THREADS;
    unsigned che = che_min;
    for (int round = 0; round < 2; ++round) {
    int b_end = bc;
    if (round == 1) {
        if (bc >= kBuckets || nacc >= maxc) break;
        // ---- round 1: the buckets [bc, kBuckets) minus the candidates excluded
        // by the corners accepted so far, re-bucketed from position 0 (counts,
        // then cursors, in S.bstart itself: the chunk buffer and the grid are live)
        if (use_bm && marked < nacc) {
            const int rows = 2 * R + 1;
            const long long items = (long long)(nacc - marked) * rows;
            for (long long i = tid; i < items; i += SEL_THREADS) {
                const int k = marked + (int)(i / rows), dy = (int)(i % rows) - R;
                const short2 q = axy[k];
                mark_row(bm, wr, rw, rh, q.x - roi.x0, q.y - roi.y0, dy, md2, S.hw);
            }
            marked = nacc;
        }
        for (int b = tid; b <= kBuckets; b += SEL_THREADS) S.bstart[b] = 0;
        __threadfence_block();
        __syncthreads();
        auto keeps = [&](unsigned long long k, unsigned id, unsigned& b) {
            if (k < thrb) return false;
            b = bucket_of(k, maxf);
            if ((int)b < bc) return false;
            int x, y;
            dw.split(id, x, y);
            return !(use_bm ? excluded(bm, wr, x - roi.x0, y - roi.y0)
                            : conflicts(x, y, heads, axy, anext, cg, imd2));
        };
        for (unsigned i0 = tid; i0 < n; i0 += 4 * SEL_THREADS) {
            unsigned long long k[4];
            unsigned id[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned i = i0 + q * SEL_THREADS;
                k[q] = i < n ? ck[i] : 0ull;
                id[q] = i < n ? ci[i] : 0u;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                unsigned b;
                if (i0 + q * SEL_THREADS < n && keeps(k[q], id[q], b)) atomicAdd(&S.bstart[b], 1u);
            }
        }
        __syncthreads();
        {
            constexpr int PER = kBuckets / SEL_THREADS;
            unsigned v[PER], sum = 0;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                v[k] = S.bstart[tid * PER + k];
                sum += v[k];
            }
            unsigned off = block_excl_scan(sum, S.warp_tot, &S.total);
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                S.bstart[tid * PER + k] = off;  // the bucket's cursor during the scatter
                off += v[k];
            }
        }
        __syncthreads();
        for (unsigned i0 = tid; i0 < n; i0 += 4 * SEL_THREADS) {
            unsigned long long k[4];
            unsigned id[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned i = i0 + q * SEL_THREADS;
                k[q] = i < n ? ck[i] : 0ull;
                id[q] = i < n ? ci[i] : 0u;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                unsigned b;
                if (i0 + q * SEL_THREADS >= n || !keeps(k[q], id[q], b)) continue;
                const unsigned pos = atomicAdd(&S.bstart[b], 1u);
                sk[pos] = k[q];
                si[pos] = id[q];
            }
        }
        __threadfence_block();
        __syncthreads();
        {
            // the cursors ended at the next bucket's start: shift them back by one
            constexpr int PER = kBuckets / SEL_THREADS;
            unsigned v[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int b = tid * PER + k;
                v[k] = b ? S.bstart[b - 1] : 0u;
            }
            const unsigned tot = S.bstart[kBuckets - 1];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < PER; ++k) S.bstart[tid * PER + k] = v[k];
            if (tid == 0) S.bstart[kBuckets] = tot;
            __syncthreads();
        }
        b0 = bc;
        b_end = kBuckets;
        che = min(che, (unsigned)ch / 2);
    }
    while (b0 < b_end && nacc < maxc) {
        if (use_bm && marked < nacc) {  // the CTA marks the new corners' discs: (corner, row) items
            const int rows = 2 * R + 1;
            const long long items = (long long)(nacc - marked) * rows;
            for (long long i = tid; i < items; i += SEL_THREADS) {
                const int k = marked + (int)(i / rows), dy = (int)(i % rows) - R;
                const short2 q = axy[k];
                mark_row(bm, wr, rw, rh, q.x - roi.x0, q.y - roi.y0, dy, md2, S.hw);
            }
            marked = nacc;
            __threadfence_block();
            __syncthreads();
        }
        int b1;  // largest run of whole buckets with <= che candidates (at least one)
        {
            const unsigned limit = S.bstart[b0] + che;
            int lo = b0 + 1, hi = b_end;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (S.bstart[mid] <= limit) lo = mid;
                else hi = mid - 1;
            }
            b1 = lo;
        }
        const unsigned c_lo = S.bstart[b0], c_hi = S.bstart[b1];
        const int b0_run = b0;
        b0 = b1;
        if (c_hi == c_lo) continue;
        const bool big = c_hi - c_lo > che;  // one tie-heavy bucket: exact order in global first
        if (big)
            global_merge_sort(sk + c_lo, si + c_lo, const_cast<unsigned long long*>(ck) + c_lo,
                              const_cast<unsigned*>(ci) + c_lo, c_hi - c_lo);
        bool rerun = false;
        unsigned c0 = c_lo;
        while (c0 < c_hi && nacc < maxc) {
            const unsigned m = min(che, c_hi - c0);
            // prefilter: thread t tests the contiguous run [t*per, (t+1)*per)
            const unsigned per = (m + SEL_THREADS - 1) / SEL_THREADS;
            const unsigned j0 = min(tid * per, m), j1 = min(j0 + per, m);
            unsigned alive = 0;  // bit q: candidate j0 + q survives (per <= 32: che <= 32 * threads)
            for (unsigned j = j0; j < j1; j += 8) {  // eight loads in flight per L2 latency
                unsigned id[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) id[q] = j + q < j1 ? si[c0 + j + q] : 0xffffffffu;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (j + q >= j1) break;
                    int x, y;
                    dw.split(id[q], x, y);
                    const bool ex = use_bm ? excluded(bm, wr, x - roi.x0, y - roi.y0)
                                           : conflicts(x, y, heads, axy, anext, cg, imd2);
                    if (!ex) alive |= 1u << (j + q - j0);
                }
            }
            unsigned o = block_excl_scan(__popc(alive), S.warp_tot, &S.total);
            const unsigned ns = S.total;
            if (ns > (unsigned)ch) {  // the survivors overflow the chunk buffer: half the chunk
                che = max(che_min, che >> 1);
                if (big) continue;  // the same slice start, shorter
                rerun = true;       // a shorter run of whole buckets
                break;
            }
            for (unsigned a = alive; a; a &= a - 1) {
                const unsigned j = j0 + __ffs(a) - 1;
                ckey[o] = sk[c0 + j];
                cidx[o] = si[c0 + j];
                ++o;
            }
            if (tid == 0) S.sflag = 0;
            __syncthreads();
            c0 += m;
            // the walk costs ~1.5 us per 32 survivors, a chunk ~6 us of barriers and
            // latencies: aim at 2-8 walk batches per chunk
            if (ns <= 16) che = min(che << 2, che_max);
            else if (ns <= 64) che = min(che << 1, che_max);
            else if (ns > 256) che = max(che_min, che >> 1);
            if (ns == 0) continue;
            // exact order of the survivors (a merge-sorted big bucket is in order already)
            if (!big) {
                if (ns <= 32) {
                    if (warp == 0) {
                        unsigned long long k = 0;
                        unsigned id = 0xffffffffu;
                        if ((unsigned)lane < ns) {
                            k = ckey[lane];
                            id = cidx[lane];
                        }
                        warp_sort32(k, id);
                        if ((unsigned)lane < ns) {
                            ckey[lane] = k;
                            cidx[lane] = id;
                        }
                    }
                } else if (ns > (unsigned)(kSortPer * SEL_THREADS) ||
                           !run_rank_sort(ckey, cidx, (int)ns, maxf, &S.sflag)) {
                    int np = 1;
                    while (np < (int)ns) np <<= 1;
                    for (int j = ns + tid; j < np; j += SEL_THREADS) {
                        ckey[j] = 0;
                        cidx[j] = 0xffffffffu;
                    }
                    __syncthreads();
                    bitonic_sort(ckey, cidx, np);
                }
            }
            // ---- the greedy walk over the sorted survivors, 32 at a time
            if (warp == 0) {
                for (unsigned w0 = 0; w0 < ns && nacc < maxc; w0 += 32) {
                    const unsigned j = w0 + lane;
                    int x = 0, y = 0;
                    bool ok = false;
                    if (j < ns) {
                        dw.split(cidx[j], x, y);
                        ok = !conflicts(x, y, heads, axy, anext, cg, imd2);
                    }
                    const unsigned live = __ballot_sync(0xffffffffu, ok);
                    if (!live) continue;
                    // earlier live lanes closer than min_distance: all 32 sources in an
                    // unrolled loop, so the shuffles issue back to back instead of as a
                    // dependent chain over the live set (one live lane needs none)
                    unsigned conf = 0;
                    if (live & (live - 1)) {
                        const unsigned xy = (unsigned)x | ((unsigned)y << 16);  // 16-bit coordinates: one shuffle per source
#pragma unroll
                        for (int src = 0; src < 32; ++src) {
                            const unsigned sxy = __shfl_sync(0xffffffffu, xy, src);
                            const int dx = x - (int)(sxy & 0xffffu), dy = y - (int)(sxy >> 16);
                            if (src < lane && ((live >> src) & 1u) && (unsigned)(dx * dx) + (unsigned)(dy * dy) < imd2)
                                conf |= 1u << src;
                        }
                    }
                    unsigned acc = live;  // no conflict inside the batch: every live lane is accepted
                    if (__ballot_sync(0xffffffffu, conf != 0)) {  // rank-order resolution
                        acc = 0;
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            const unsigned ck2 = __shfl_sync(0xffffffffu, conf, k);
                            if (((live >> k) & 1u) && !(ck2 & acc)) acc |= 1u << k;
                        }
                    }
                    const int room = maxc - nacc;
                    while (__popc(acc) > room) acc &= ~(1u << (31 - __clz(acc)));
                    if (acc & (1u << lane)) {
                        const int slot = nacc + __popc(acc & ((1u << lane) - 1));
                        axy[slot] = make_short2((short)x, (short)y);
                        const int cid = cg.cell_of(y - roi.y0) * gw + cg.cell_of(x - roi.x0);
                        anext[slot] = atomicExch(&heads[cid], slot);
                        out_xy[(size_t)d * maxc + slot] = make_double2((double)x, (double)y);
                        out_score[(size_t)d * maxc + slot] = __longlong_as_double((long long)ckey[j]);
                    }
                    nacc += __popc(acc);
                    __syncwarp();
                }
                if (lane == 0) S.nacc = nacc;
            }
            __syncthreads();
            nacc = S.nacc;
            if (use_bm && c0 < c_hi) {  // more slices of a big bucket follow: mark now
                const int rows = 2 * R + 1;
                const long long items = (long long)(nacc - marked) * rows;
                for (long long i = tid; i < items; i += SEL_THREADS) {
                    const int k = marked + (int)(i / rows), dy = (int)(i % rows) - R;
                    const short2 q = axy[k];
                    mark_row(bm, wr, rw, rh, q.x - roi.x0, q.y - roi.y0, dy, md2, S.hw);
                }
                marked = nacc;
                __threadfence_block();
                __syncthreads();
            }
        }
        if (rerun) b0 = b0_run;
    }
    }
    if (tid == 0) {
        out_n[d] = nacc;
        // the cut prefix ran out before max_corners: redo from the full list
        if (!redo && cut && nacc < maxc) {
            s.flags[d] |= 2;
            s.count[d] = 0;  // the redo pass lists the band below the cut from position 0
        }
    }
}

__global__ void gradients_kernel(const uint8_t* __restrict__ f, int w, int h, double* __restrict__ gx,
                                 double* __restrict__ gy) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w) return;
    const int xm = max(x - 1, 0), xp = min(x + 1, w - 1);
    const int ym = max(y - 1, 0), yp = min(y + 1, h - 1);
    gx[(size_t)y * w + x] = dmul(0.5, dsub((double)f[(size_t)y * w + xp], (double)f[(size_t)y * w + xm]));
    gy[(size_t)y * w + x] = dmul(0.5, dsub((double)f[(size_t)yp * w + x], (double)f[(size_t)ym * w + x]));
}

}  // namespace

size_t bitmap_words(stabgpu_roi roi) {
    return (size_t)((roi.x1 - roi.x0 + 31) >> 5) * (roi.y1 - roi.y0);
}


namespace {
void launch_buckets(const DetectScratch& s, int nD, double quality, int redo, cudaStream_t st) {
    if (!s.bstart || !s.bcur) return;  // (the bucket counts were cleared by detect_reset_kernel)
    const dim3 grid(16, nD);
    bucket_count_kernel<<<grid, 512, 0, st>>>(s, quality, redo);
    bucket_scan_kernel<<<nD, 1024, 0, st>>>(s, quality, redo);
    bucket_scatter_kernel<<<grid, 512, 0, st>>>(s, quality, redo);
}
}  // namespace

void launch_detect(PlaneBatch fr, int nD, const stabgpu_detect_cfg& cfg, stabgpu_roi roi,
                   DetectScratch& s, double2* out_xy, double* out_score, int* out_n,
                   cudaStream_t st) {
    if (nD <= 0) return;
    const int rw = roi.x1 - roi.x0, rh = roi.y1 - roi.y0;
    const int half = cfg.block_size / 2;
    const bool fast = half == 1 && s.hist && s.lo && s.flags && s.mlo;
    detect_reset_kernel<<<nD, 256, 0, st>>>(s, fast ? 1 : 0, (nD <= 32 && s.bstart && s.bcur) ? 1 : 0);
    if (fast) {
        dim3 grid((rw + 8 * SW_COLS - 1) / (8 * SW_COLS), (rh + SW_BAND - 1) / SW_BAND, nD);
        resp_stream_kernel<0><<<grid, 256, 0, st>>>(fr, roi, cfg.quality_level, s, 0);
        // the cut keeps ~16 candidates per corner.  When the corners' exclusion
        // discs would cover the ROI twice over (max_corners * pi * md^2 > 2 *
        // area, e.g. C1: 200 corners at 30 px in 512x384), the greedy scans
        // deep into the list, the prefix runs out and the redo costs more than
        // selecting from the full list once: no cut then (measured: C1 detect
        // 1.65 -> 1.49 ms per 60 frames; C2, ratio 1.1, is faster with the cut)
        const double cover = (double)cfg.max_corners * 3.141592653589793 * cfg.min_distance * cfg.min_distance;
        const unsigned keep =
            cover > 2.0 * rw * rh ? 0xFFFFFFFFu : (unsigned)std::max(4096, 16 * cfg.max_corners);
        resp_cut_kernel<<<nD, 32, 0, st>>>(cfg.quality_level, s, keep);
        resp_stream_kernel<1><<<grid, 256, 0, st>>>(fr, roi, cfg.quality_level, s, 0);
    } else if (half == 1) {
        dim3 grid((rw + RTW - 1) / RTW, (rh + RTH - 1) / RTH, nD);
        resp_max_kernel<1><<<grid, 256, 0, st>>>(fr, roi, s.maxbits);
        cand_kernel<1><<<grid, 256, 0, st>>>(fr, roi, cfg.quality_level, s.maxbits, s.count,
                                             s.cand_key, s.cand_idx, s.cap);
    } else if (half == 2) {
        dim3 grid((rw + RTW - 1) / RTW, (rh + RTH - 1) / RTH, nD);
        resp_max_kernel<2><<<grid, 256, 0, st>>>(fr, roi, s.maxbits);
        cand_kernel<2><<<grid, 256, 0, st>>>(fr, roi, cfg.quality_level, s.maxbits, s.count,
                                             s.cand_key, s.cand_idx, s.cap);
    } else {
        dim3 grid((rw + 127) / 128, rh, nD);
        resp_generic_kernel<<<grid, 128, 0, st>>>(fr, roi, half, 0, 0.0, s.maxbits, s.count,
                                                  s.cand_key, s.cand_idx, s.cap, nullptr);
        resp_generic_kernel<<<grid, 128, 0, st>>>(fr, roi, half, 1, cfg.quality_level, s.maxbits,
                                                  s.count, s.cand_key, s.cand_idx, s.cap, nullptr);
    }
    // shared memory per CTA: chunk buffer (12 B per candidate) + grid (32 KB) +
    // accepted corners (8 B each, when <= SMEM_CORNERS) [+ exclusion bitmap
    // when every candidate is listed (no cut) and it fits]; two 512-thread CTAs
    // per SM when the batch outnumbers the SMs and a 2048-candidate chunk fits
    // twice (static shared memory included)
    const bool no_cut = !fast || cfg.max_corners * 3.141592653589793 * cfg.min_distance * cfg.min_distance > 2.0 * rw * rh;
    const size_t bm_bytes = no_cut ? 4 * bitmap_words(roi) : 0;
    const size_t fixed = sizeof(int) * MAX_CELLS +
                         (cfg.max_corners <= SMEM_CORNERS ? (sizeof(short2) + sizeof(int)) * cfg.max_corners : 0);
    const size_t stat = sizeof(SelShared) + 1024;  // static shared + per-CTA reserve
    auto fit = [&](size_t budget, int cmin, int& ch, bool& bm) {  // largest chunk, bitmap if it fits
        for (int pass = 0; pass < 2; ++pass) {
            bm = pass == 0 && bm_bytes > 0;
            if (pass == 0 && !bm) continue;
            for (int c = 8192; c >= cmin; c >>= 1)
                if (stat + 12 * (size_t)c + fixed + (bm ? bm_bytes : 0) <= budget) {
                    ch = c;
                    return true;
                }
        }
        bm = false;
        return false;
    };
    int ch = 1024;
    bool use_bm = false;
    const bool pair = nD > sm_count() && fit(114 * 1024, 2048, ch, use_bm);
    if (!pair) fit(227 * 1024, 256, ch, use_bm);
    ch = std::min(ch, 2048);  // measured: larger chunks sort more survivors per walk (C1 1.04 ms at 2048, 1.09 at 4096)
    const size_t smem = std::max<size_t>(12 * (size_t)ch + fixed + (use_bm ? bm_bytes : 0), 4 * kBuckets);
    auto sel = pair ? select_kernel<512> : select_kernel<1024>;
    const int sel_threads = pair ? 512 : 1024;
    ensure_smem(sel, smem);
    short2* g_axy = nullptr;
    int* g_anext = nullptr;
    if (cfg.max_corners > SMEM_CORNERS) {
        // large budgets keep the accepted list in global scratch
        // (a failed allocation stays in cudaGetLastError for the caller's check_launch)
        if (cudaMallocAsync((void**)&g_axy, sizeof(short2) * (size_t)nD * cfg.max_corners, st) != cudaSuccess)
            return;
        if (cudaMallocAsync((void**)&g_anext, sizeof(int) * (size_t)nD * cfg.max_corners, st) != cudaSuccess) {
            cudaFreeAsync(g_axy, st);
            return;
        }
    }
    // phase A by the multi-CTA bucket kernels when the batch is too small to
    // fill the GPU with select CTAs (Stage II, single frames: C1 stream 3.6k ->
    // 4.3k frames/s); large batches keep it inside select (no gain measured)
    DetectScratch sf = s;
    if (!fast) sf.flags = nullptr;
    if (nD > 32) sf.bstart = sf.bcur = nullptr;
    launch_buckets(sf, nD, cfg.quality_level, 0, st);
    sel<<<nD, sel_threads, smem, st>>>(cfg, roi, fr.w, sf, out_xy, out_score, out_n, g_axy, g_anext, ch,
                                       use_bm ? 1 : 0, 0);
    if (fast) {  // frames whose cut prefix ran out: full candidate list (usually none)
        // (select cleared the candidate count of the frames it flagged; the redo
        // buckets inside select: usually no frame takes it, so two launches, not six)
        dim3 grid((rw + 8 * SW_COLS - 1) / (8 * SW_COLS), (rh + SW_BAND - 1) / SW_BAND, nD);
        resp_stream_kernel<1><<<grid, 256, 0, st>>>(fr, roi, cfg.quality_level, s, 1);
        DetectScratch sr = s;
        sr.bstart = sr.bcur = nullptr;
        sel<<<nD, sel_threads, smem, st>>>(cfg, roi, fr.w, sr, out_xy, out_score, out_n, g_axy, g_anext, ch,
                                           use_bm ? 1 : 0, 1);
    }
    if (g_axy) {
        cudaFreeAsync(g_axy, st);
        cudaFreeAsync(g_anext, st);
    }
}

bool detect_allocates(const stabgpu_detect_cfg& cfg) { return cfg.max_corners > SMEM_CORNERS; }

void launch_gradients(const uint8_t* src, int w, int h, double* gx, double* gy, cudaStream_t st) {
    dim3 grid((w + 127) / 128, h);
    gradients_kernel<<<grid, 128, 0, st>>>(src, w, h, gx, gy);
}

void launch_min_eig(const uint8_t* src, int w, int h, int block, double* out, cudaStream_t st) {
    PlaneBatch fr{src, (size_t)w * h, w, h};
    stabgpu_roi all{0, 0, w, h};
    dim3 grid((w + 127) / 128, h, 1);
    resp_generic_kernel<<<grid, 128, 0, st>>>(fr, all, block / 2, 2, 0.0, nullptr, nullptr, nullptr,
                                              nullptr, 0, out);
}

}  // namespace stabgpu
