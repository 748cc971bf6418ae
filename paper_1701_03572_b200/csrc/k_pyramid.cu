// k_pyramid.cu — K1: fused binomial blur + 2x decimation, batched over frames.
//
// Reference: downsample + build_pyramid, image_ops.cpp:25-77.  The reference
// filters every column horizontally into 16-bit, then filters even rows /
// even columns vertically and rounds with (acc + 128) >> 8, replicating
// borders.  All arithmetic is integer, so any evaluation order is exact; the
// kernel computes only the even columns the vertical pass consumes.
//
// Three kernels, chosen by alignment:
//  * pyramid_bulk_kernel (rows 16-byte aligned): persistent CTAs stream
//    (frame, band) items into shared memory with one cp.async.bulk each,
//    double-buffered behind mbarriers, and filter from shared memory;
//  * pyramid_stream_kernel (rows 8-byte aligned): register streaming, one
//    thread per 4 output columns walking a band of rows;
//  * pyramid_level_kernel (any width): a 64x16 output tile per CTA with its
//    (2*16+3) x (2*64+3) input window staged in shared memory.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace stabgpu {

namespace {

constexpr int TW = 64;  // output tile width
constexpr int TH = 16;  // output tile height
constexpr int IW = 2 * TW + 3;
constexpr int IH = 2 * TH + 3;
constexpr int IWP = 2 * TW + 8;  // padded smem row (word loads start 2 bytes early)

__global__ void __launch_bounds__(256) pyramid_level_kernel(const uint8_t* __restrict__ src,
                                                            size_t src_stride, int w, int h,
                                                            uint8_t* __restrict__ dst,
                                                            size_t dst_stride) {
    __shared__ __align__(16) uint8_t tile[IH][IWP];
    __shared__ uint16_t hrow[IH][TW];
    const int ow = w / 2, oh = h / 2;
    const int ox0 = blockIdx.x * TW, oy0 = blockIdx.y * TH;
    const uint8_t* f = src + (size_t)blockIdx.z * src_stride;
    const int ix0 = 2 * ox0 - 2, iy0 = 2 * oy0 - 2;
    const int tid = threadIdx.x;

    const bool interior = ix0 - 2 >= 0 && ix0 - 2 + IWP <= w && (w & 3) == 0 &&
                          ((reinterpret_cast<uintptr_t>(f) & 3) == 0);
    if (interior) {
        // words covering columns [ix0-2, ix0-2+IWP): tile col c <-> image col ix0-2+c
        constexpr int WPR = IWP / 4;
        for (int i = tid; i < IH * WPR; i += blockDim.x) {
            const int r = i / WPR, c = i % WPR;
            const int y = clampi(iy0 + r, 0, h - 1);
            const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(f + (size_t)y * w + ix0 - 2) + c);
            *reinterpret_cast<uint32_t*>(&tile[r][4 * c]) = v;
        }
    } else {
        for (int i = tid; i < IH * IW; i += blockDim.x) {
            const int r = i / IW, c = i % IW;
            const int y = clampi(iy0 + r, 0, h - 1);
            const int x = clampi(ix0 + c, 0, w - 1);
            tile[r][c + 2] = __ldg(f + (size_t)y * w + x);
        }
    }
    __syncthreads();
    // horizontal [1 4 6 4 1] at the even columns 2*ox (tile cols 2*j+2 .. 2*j+6)
    for (int i = tid; i < IH * TW; i += blockDim.x) {
        const int r = i / TW, j = i % TW;
        const uint8_t* t = &tile[r][2 * j + 2];
        hrow[r][j] = (uint16_t)(t[0] + 4 * t[1] + 6 * t[2] + 4 * t[3] + t[4]);
    }
    __syncthreads();
    // vertical on even rows, 4 consecutive outputs per thread
    const int j4 = (tid % (TW / 4)) * 4, r = tid / (TW / 4);  // 16 x 16 threads
    const int oy = oy0 + r;
    if (oy >= oh) return;
    uint8_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int j = j4 + k;
        const uint32_t acc = hrow[2 * r][j] + 4u * hrow[2 * r + 1][j] + 6u * hrow[2 * r + 2][j] +
                             4u * hrow[2 * r + 3][j] + hrow[2 * r + 4][j];
        o[k] = (uint8_t)((acc + 128) >> 8);
    }
    uint8_t* d = dst + (size_t)blockIdx.z * dst_stride + (size_t)oy * ow;
    const int ox = ox0 + j4;
    if (ox + 3 < ow && ((reinterpret_cast<uintptr_t>(d + ox) & 3) == 0)) {
        *reinterpret_cast<uchar4*>(d + ox) = make_uchar4(o[0], o[1], o[2], o[3]);
    } else {
        for (int k = 0; k < 4; ++k)
            if (ox + k < ow) d[ox + k] = o[k];
    }
}

// ---------------------------------------------------------------------------
// Register-streaming variant (rows 8-byte aligned, w % 8 == 0).  A thread owns
// 4 adjacent output columns (8 input columns) and walks a band of output rows
// top to bottom.  Each input row is read once: 8 bytes per thread, the halo
// words from the neighbour lanes.  The horizontal filter runs on packed
// 16-bit pairs (two outputs per register: sums stay below 2^16 — horizontal
// <= 16*255, vertical <= 256*255), the last five filtered rows stay in
// registers, and (acc + 128) >> 8 is byte 1 of each 16-bit lane.
constexpr int SPT = 128;   // threads per CTA: 512 output columns
constexpr int SBAND = 32;  // output rows per CTA

__device__ __forceinline__ uint32_t ev(uint32_t wd) { return wd & 0x00FF00FFu; }  // (b0, b2)
__device__ __forceinline__ uint32_t od(uint32_t wd) { return (wd >> 8) & 0x00FF00FFu; }  // (b1, b3)
__device__ __forceinline__ uint32_t fun16(uint32_t lo, uint32_t hi) { return __funnelshift_r(lo, hi, 16); }

// one input row: words L (cols -4..-1), X (0..3), Y (4..7), R (8..11) ->
// packed horizontal sums of outputs (0, 1) and (2, 3) (input cols 0, 2, 4, 6)
__device__ __forceinline__ void hrow(uint32_t L, uint32_t X, uint32_t Y, uint32_t R, uint32_t& a, uint32_t& b) {
    const uint32_t eL = ev(L), oL = od(L), eX = ev(X), oX = od(X), eY = ev(Y), oY = od(Y), eR = ev(R);
    const uint32_t m2a = fun16(eL, eX), m1a = fun16(oL, oX), p2a = fun16(eX, eY);  // (-2,0) (-1,1) (2,4)
    const uint32_t m1b = fun16(oX, oY), p2b = fun16(eY, eR);                        // (3,5) (6,8)
    a = (m2a + p2a) + 4u * (m1a + oX) + 6u * eX;
    b = (p2a + p2b) + 4u * (m1b + oY) + 6u * eY;
}


__device__ __forceinline__ void srow(const uint8_t* __restrict__ f, int w, int h, int y, int t, int lane, bool act,
                                     bool left_edge, bool right_edge, uint32_t& a, uint32_t& b) {
    y = min(max(y, 0), h - 1);
    const uint8_t* rp = f + (size_t)y * w + 8 * t;
    uint2 xy = make_uint2(0u, 0u);
    if (act) xy = __ldg(reinterpret_cast<const uint2*>(rp));
    uint32_t L = __shfl_up_sync(0xFFFFFFFFu, xy.y, 1);
    uint32_t R = __shfl_down_sync(0xFFFFFFFFu, xy.x, 1);
    if (lane == 0 && !left_edge && act) L = __ldg(reinterpret_cast<const uint32_t*>(rp - 4));
    if (lane == 31 && !right_edge && act) R = __ldg(reinterpret_cast<const uint32_t*>(rp + 8));
    if (left_edge) L = (xy.x & 0xFFu) * 0x01010101u;  // clamp: col 0
    if (right_edge) R = (xy.y >> 24) * 0x01010101u;    // clamp: col w-1 (= 8t+7)
    hrow(L, xy.x, xy.y, R, a, b);
}

__global__ void __launch_bounds__(SPT) pyramid_stream_kernel(const uint8_t* __restrict__ src, size_t src_stride,
                                                              int w, int h, uint8_t* __restrict__ dst,
                                                              size_t dst_stride) {
    const int ow = w / 2, oh = h / 2;
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * SPT + threadIdx.x;  // output columns 4t .. 4t+3
    const int oy0 = blockIdx.y * SBAND, oy1 = min(oy0 + SBAND, oh);
    const uint8_t* f = src + (size_t)blockIdx.z * src_stride;
    uint8_t* d = dst + (size_t)blockIdx.z * dst_stride;
    const bool act = 8 * t < w;
    const bool left_edge = t == 0, right_edge = 8 * t + 8 >= w;
#define ROW(Y, A, B) srow(f, w, h, (Y), t, lane, act, left_edge, right_edge, A, B)
    uint32_t a0, a1, a2, a3, a4, b0, b1, b2, b3, b4;  // filtered rows 2oy-2 .. 2oy+2
    ROW(2 * oy0 - 2, a0, b0);
    ROW(2 * oy0 - 1, a1, b1);
    ROW(2 * oy0, a2, b2);
    ROW(2 * oy0 + 1, a3, b3);
    ROW(2 * oy0 + 2, a4, b4);
    const bool vec = act && 4 * t + 3 < ow;
    for (int oy = oy0; oy < oy1; ++oy) {
        const uint32_t va = (a0 + a4) + 4u * (a1 + a3) + 6u * a2 + 0x00800080u;
        const uint32_t vb = (b0 + b4) + 4u * (b1 + b3) + 6u * b2 + 0x00800080u;
        const uint32_t o = __byte_perm(va, vb, 0x7531);  // byte 1 of each 16-bit lane
        uint8_t* op = d + (size_t)oy * ow + 4 * t;
        if (vec) {
            *reinterpret_cast<uint32_t*>(op) = o;
        } else if (act) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (4 * t + k < ow) op[k] = (uint8_t)(o >> (8 * k));
        }
        if (oy + 1 < oy1) {
            a0 = a2;
            b0 = b2;
            a1 = a3;
            b1 = b3;
            a2 = a4;
            b2 = b4;
            ROW(2 * oy + 3, a3, b3);
            ROW(2 * oy + 4, a4, b4);
        }
    }
}
#undef ROW

// ---------------------------------------------------------------------------
// Bulk-copy variant (rows 16-byte aligned, w % 16 == 0): a persistent CTA
// walks (frame, band) items.  A band's input rows are one contiguous range of
// the frame, so ONE cp.async.bulk per item moves them into shared memory,
// double-buffered behind an mbarrier: item k+1 streams in while item k is
// filtered from shared memory.  That keeps ~96 KB per SM in flight (two CTAs of two 48 KB buffers, or one of two 96 KB buffers for rows wider than ~3 KB), which the
// register-streaming kernel (a few 8-byte loads per thread) cannot.
// Threads = (column group of 4 outputs, row group); each row group walks its
// rows with the same packed 16-bit filter as the streaming kernel.
// Output rows [r0, r1) of one 4-column group from a staged band (cb = the
// group's first byte in the band's row lo; olast = offset of the band's last
// staged row).  Row pointers advance by 2w per output row; only the bottom
// row of the frame can clamp (one min).  EDGE: the warp holds the first or
// last column group (clamped neighbour words); interior warps load both
// neighbour words unconditionally.
template <bool EDGE>
__device__ __forceinline__ void band_rows(const uint8_t* cb, int w, int h, int lo, int olast, int r0, int r1,
                                          uint32_t* op, int ostep, bool hasL, bool hasR) {
    auto brow = [&](const uint8_t* rp, uint32_t& a, uint32_t& b) {
        const uint2 xy = *reinterpret_cast<const uint2*>(rp);
        uint32_t L, R;
        if (EDGE) {
            L = hasL ? *reinterpret_cast<const uint32_t*>(rp - 4) : (xy.x & 0xFFu) * 0x01010101u;
            R = hasR ? *reinterpret_cast<const uint32_t*>(rp + 8) : (xy.y >> 24) * 0x01010101u;
        } else {
            L = *reinterpret_cast<const uint32_t*>(rp - 4);
            R = *reinterpret_cast<const uint32_t*>(rp + 8);
        }
        hrow(L, xy.x, xy.y, R, a, b);
    };
    auto rowp = [&](int y) { return cb + (clampi(y, 0, h - 1) - lo) * w; };
    uint32_t a0, a1, a2, a3, a4, b0, b1, b2, b3, b4;
    brow(rowp(2 * r0 - 2), a0, b0);
    brow(rowp(2 * r0 - 1), a1, b1);
    brow(rowp(2 * r0), a2, b2);
    brow(rowp(2 * r0 + 1), a3, b3);
    brow(rowp(2 * r0 + 2), a4, b4);
    const uint8_t* last = cb + olast;
    const uint8_t* rp = cb + (2 * r0 + 3 - lo) * w;  // row 2oy+1 of the next output row
    for (int oy = r0;; rp += 2 * w, op += ostep) {
        const uint32_t va = (a0 + a4) + 4u * (a1 + a3) + 6u * a2 + 0x00800080u;
        const uint32_t vb = (b0 + b4) + 4u * (b1 + b3) + 6u * b2 + 0x00800080u;
        *op = __byte_perm(va, vb, 0x7531);
        if (++oy >= r1) break;
        a0 = a2;
        b0 = b2;
        a1 = a3;
        b1 = b3;
        a2 = a4;
        b2 = b4;
        brow(rp, a3, b3);
        const uint8_t* rq = rp + w;
        brow(rq < last ? rq : last, a4, b4);
    }
}

// BT threads per CTA, BBUF bytes per input buffer (two per CTA), MINB CTAs per SM

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void brow(const uint8_t* rp, int cg, int w, uint32_t& a, uint32_t& b) {
    const uint2 xy = *reinterpret_cast<const uint2*>(rp + 8 * cg);
    const uint32_t L = cg > 0 ? *reinterpret_cast<const uint32_t*>(rp + 8 * cg - 4) : (xy.x & 0xFFu) * 0x01010101u;
    const uint32_t R = 8 * cg + 8 < w ? *reinterpret_cast<const uint32_t*>(rp + 8 * cg + 8)
                                      : (xy.y >> 24) * 0x01010101u;
    hrow(L, xy.x, xy.y, R, a, b);
}

template <int BT, int BBUF, int MINB>
__global__ void __launch_bounds__(BT, MINB) pyramid_bulk_kernel(const uint8_t* __restrict__ src, size_t src_stride,
                                                              int w, int h, uint8_t* __restrict__ dst,
                                                              size_t dst_stride, int frames, int band, int rgroups) {
    extern __shared__ __align__(128) uint8_t pyr_smem[];
    __shared__ __align__(8) unsigned long long mbar[2];
    const int ow = w / 2, oh = h / 2;
    const int nb = (oh + band - 1) / band;
    const long long total = (long long)nb * frames;
    const int tid = threadIdx.x;
    const int ncg = ow / 4;
    auto issue = [&](long long item, int buf) {
        const int f = (int)(item / nb), b = (int)(item - (long long)f * nb);
        const int oy0 = b * band, oy1 = min(oy0 + band, oh);
        const int lo = max(0, 2 * oy0 - 2), hi = min(h - 1, 2 * oy1);
        const uint32_t bytes = (uint32_t)(hi - lo + 1) * (uint32_t)w;
        const uint32_t bar = su32(&mbar[buf]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(pyr_smem + buf * BBUF)),
            "l"(src + (size_t)f * src_stride + (size_t)lo * w), "r"(bytes), "r"(bar)
            : "memory");
    };
    long long item = blockIdx.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (item < total) issue(item, 0);
    }
    __syncthreads();
    const int per = (band + rgroups - 1) / rgroups;  // output rows per row group
    for (int k = 0; item < total; ++k, item += gridDim.x) {
        const int buf = k & 1;
        if (tid == 0 && item + gridDim.x < total) issue(item + gridDim.x, buf ^ 1);
        const int f = (int)(item / nb), b = (int)(item - (long long)f * nb);
        const int oy0 = b * band, oy1 = min(oy0 + band, oh);
        const int lo = max(0, 2 * oy0 - 2);
        {
            const uint32_t bar = su32(&mbar[buf]), phase = (uint32_t)((k >> 1) & 1);
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                    : "=r"(done)
                    : "r"(bar), "r"(phase)
                    : "memory");
        }
        const uint8_t* sb = pyr_smem + buf * BBUF;
        uint8_t* d = dst + (size_t)f * dst_stride;
        const int olast = (min(h - 1, 2 * oy1) - lo) * w;
        for (int u = tid; u < ncg * rgroups; u += BT) {
            const int cg = u % ncg, rg = u / ncg;
            const int r0 = oy0 + rg * per, r1 = min(r0 + per, oy1);
            const bool hasL = cg > 0, hasR = 8 * cg + 8 < w;
            const bool edge = __any_sync(__activemask(), !(hasL && hasR));
            if (r0 >= r1) continue;
            uint32_t* op = reinterpret_cast<uint32_t*>(d + (size_t)r0 * ow + 4 * cg);
            if (edge)
                band_rows<true>(sb + 8 * cg, w, h, lo, olast, r0, r1, op, ow / 4, hasL, hasR);
            else
                band_rows<false>(sb + 8 * cg, w, h, lo, olast, r0, r1, op, ow / 4, hasL, hasR);
        }
        __syncthreads();  // buffer `buf` is refilled by the issue of iteration k + 1
    }
}

// ---------------------------------------------------------------------------
// Carry variant (one column group per thread, i.e. >= BT/2 groups): each CTA
// takes a contiguous run of (frame, band) items, so consecutive items are
// usually consecutive bands of one frame.  The thread's five filtered rows
// then carry over from the previous band, and the next band's buffer holds
// only its new rows (2 oy0 + 1 .. 2 oy1): no 3-row prologue and no halo
// re-load per band.  A frame's first band (or a CTA's first item) starts with
// the 5-row prologue as in pyramid_bulk_kernel.
struct Rows5 {
    uint32_t a0, a1, a2, a3, a4, b0, b1, b2, b3, b4;
};

template <bool EDGE>
__device__ __forceinline__ void carry_band(Rows5& S, bool carry, const uint8_t* cb, int w, int h, int lo, int last,
                                           int oy0, int oy1, uint32_t* op, int ostep, bool hasL, bool hasR) {
    auto brow = [&](const uint8_t* rp, uint32_t& a, uint32_t& b) {
        const uint2 xy = *reinterpret_cast<const uint2*>(rp);
        uint32_t L, R;
        if (EDGE) {
            L = hasL ? *reinterpret_cast<const uint32_t*>(rp - 4) : (xy.x & 0xFFu) * 0x01010101u;
            R = hasR ? *reinterpret_cast<const uint32_t*>(rp + 8) : (xy.y >> 24) * 0x01010101u;
        } else {
            L = *reinterpret_cast<const uint32_t*>(rp - 4);
            R = *reinterpret_cast<const uint32_t*>(rp + 8);
        }
        hrow(L, xy.x, xy.y, R, a, b);
    };
    const uint8_t* lastp = cb + last;
    const uint8_t* rp = cb + (2 * oy0 + 1 - lo) * w;  // row 2 oy0 + 1
    if (carry) {  // the previous band left the rows of output oy0 - 1
        S.a0 = S.a2;
        S.b0 = S.b2;
        S.a1 = S.a3;
        S.b1 = S.b3;
        S.a2 = S.a4;
        S.b2 = S.b4;
        brow(rp, S.a3, S.b3);
        const uint8_t* rq = rp + w;
        brow(rq < lastp ? rq : lastp, S.a4, S.b4);
    } else {
        auto rowp = [&](int y) { return cb + (clampi(y, 0, h - 1) - lo) * w; };
        brow(rowp(2 * oy0 - 2), S.a0, S.b0);
        brow(rowp(2 * oy0 - 1), S.a1, S.b1);
        brow(rowp(2 * oy0), S.a2, S.b2);
        brow(rowp(2 * oy0 + 1), S.a3, S.b3);
        brow(rowp(2 * oy0 + 2), S.a4, S.b4);
    }
    rp += 2 * w;  // row 2 oy0 + 3
    for (int oy = oy0;; rp += 2 * w, op += ostep) {
        const uint32_t va = (S.a0 + S.a4) + 4u * (S.a1 + S.a3) + 6u * S.a2 + 0x00800080u;
        const uint32_t vb = (S.b0 + S.b4) + 4u * (S.b1 + S.b3) + 6u * S.b2 + 0x00800080u;
        *op = __byte_perm(va, vb, 0x7531);
        if (++oy >= oy1) break;
        S.a0 = S.a2;
        S.b0 = S.b2;
        S.a1 = S.a3;
        S.b1 = S.b3;
        S.a2 = S.a4;
        S.b2 = S.b4;
        brow(rp, S.a3, S.b3);
        const uint8_t* rq = rp + w;
        brow(rq < lastp ? rq : lastp, S.a4, S.b4);
    }
}

template <int BT, int BBUF, int MINB>
__global__ void __launch_bounds__(BT, MINB) pyramid_carry_kernel(const uint8_t* __restrict__ src, size_t src_stride,
                                                                  int w, int h, uint8_t* __restrict__ dst,
                                                                  size_t dst_stride, int frames, int band) {
    extern __shared__ __align__(128) uint8_t pyr_smem[];
    __shared__ __align__(8) unsigned long long mbar[2];
    const int ow = w / 2, oh = h / 2;
    const int nb = (oh + band - 1) / band;
    const long long total = (long long)nb * frames;
    const long long i0 = total * blockIdx.x / gridDim.x, i1 = total * (blockIdx.x + 1) / gridDim.x;
    const int tid = threadIdx.x;
    auto carry_of = [&](long long item) { return item > i0 && (item % nb) != 0; };
    auto region = [&](long long item, int& lo, int& hi) {
        const int b = (int)(item % nb), oy0 = b * band, oy1 = min(oy0 + band, oh);
        lo = carry_of(item) ? 2 * oy0 + 1 : max(0, 2 * oy0 - 2);
        hi = min(h - 1, 2 * oy1);
    };
    auto issue = [&](long long item, int buf) {
        const int f = (int)(item / nb);
        int lo, hi;
        region(item, lo, hi);
        const uint32_t bytes = (uint32_t)(hi - lo + 1) * (uint32_t)w;
        const uint32_t bar = su32(&mbar[buf]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(pyr_smem + buf * BBUF)),
            "l"(src + (size_t)f * src_stride + (size_t)lo * w), "r"(bytes), "r"(bar)
            : "memory");
    };
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (i0 < i1) issue(i0, 0);
    }
    __syncthreads();
    const int ncg = ow / 4, cg = tid;
    const bool act = cg < ncg, hasL = cg > 0, hasR = 8 * cg + 8 < w;
    const bool edge = __any_sync(0xFFFFFFFFu, act && !(hasL && hasR));
    Rows5 S{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    int k = 0;
    for (long long item = i0; item < i1; ++item, ++k) {
        const int buf = k & 1;
        if (tid == 0 && item + 1 < i1) issue(item + 1, buf ^ 1);
        {
            const uint32_t bar = su32(&mbar[buf]), phase = (uint32_t)((k >> 1) & 1);
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                    : "=r"(done)
                    : "r"(bar), "r"(phase)
                    : "memory");
        }
        if (act) {
            const int f = (int)(item / nb), b = (int)(item % nb);
            const int oy0 = b * band, oy1 = min(oy0 + band, oh);
            int lo, hi;
            region(item, lo, hi);
            const uint8_t* cb = pyr_smem + buf * BBUF + 8 * cg;
            uint32_t* op = reinterpret_cast<uint32_t*>(dst + (size_t)f * dst_stride + (size_t)oy0 * ow + 4 * cg);
            const bool carry = carry_of(item);
            if (edge)
                carry_band<true>(S, carry, cb, w, h, lo, (hi - lo) * w, oy0, oy1, op, ow / 4, hasL, hasR);
            else
                carry_band<false>(S, carry, cb, w, h, lo, (hi - lo) * w, oy0, oy1, op, ow / 4, hasL, hasR);
        }
        __syncthreads();  // buffer `buf` is refilled by the issue of iteration k + 1
    }
}

// output rows per band of the carry kernel with `bbuf`-byte buffers
inline int carry_band_rows(int bbuf, int w) { return (bbuf / w - 3) / 2; }

template <int BT, int BBUF, int MINB>
void launch_carry(const uint8_t* src, size_t src_stride, int w, int h, uint8_t* dst, size_t dst_stride, int frames,
                  cudaStream_t st) {
    const int oh = h / 2;
    // a CTA's first band (no carry) stages rows 2 oy0 - 2 .. 2 oy0 + 2 band:
    // 2 band + 3 rows must fit the buffer
    const int band = std::min(oh, carry_band_rows(BBUF, w));
    ensure_smem(pyramid_carry_kernel<BT, BBUF, MINB>, 2 * BBUF);
    const long long items = (long long)((oh + band - 1) / band) * frames;
    const int grid = (int)std::min<long long>(items, (long long)sm_count() * MINB);
    pyramid_carry_kernel<BT, BBUF, MINB><<<grid, BT, 2 * BBUF, st>>>(src, src_stride, w, h, dst, dst_stride, frames, band);
}

template <int BT, int BBUF, int MINB>
void launch_bulk(const uint8_t* src, size_t src_stride, int w, int h, uint8_t* dst, size_t dst_stride, int frames,
                 cudaStream_t st) {
    const int ow = w / 2, oh = h / 2;
    const int band = std::min(oh, (BBUF / w - 4) / 2);
    ensure_smem(pyramid_bulk_kernel<BT, BBUF, MINB>, 2 * BBUF);
    const int sms = sm_count();
    const int ncg = ow / 4;
    const int rgroups = std::max(1, std::min(band, BT / ncg));
    const long long items = (long long)((oh + band - 1) / band) * frames;
    const int grid = (int)std::min<long long>(items, (long long)sms * MINB);
    pyramid_bulk_kernel<BT, BBUF, MINB>
        <<<grid, BT, 2 * BBUF, st>>>(src, src_stride, w, h, dst, dst_stride, frames, band, rgroups);
}

}  // namespace

void launch_pyramid_level(const uint8_t* src, size_t src_stride, int w, int h, uint8_t* dst,
                          size_t dst_stride, int frames, cudaStream_t st) {
    const int ow = w / 2, oh = h / 2;
    if (frames <= 0 || ow <= 0 || oh <= 0) return;
    // bulk-copy kernel: 16-byte aligned rows and frames, 4-byte aligned output rows,
    // at least 16 input rows (2 * band + 4 with band >= 6) per buffer
    const int band = std::min(oh, (96 * 1024 / w - 4) / 2);  // the largest buffer below
    const bool bulk = (w % 16) == 0 && (ow % 4) == 0 && (reinterpret_cast<uintptr_t>(src) % 16) == 0 &&
                      (src_stride % 16) == 0 && (reinterpret_cast<uintptr_t>(dst) % 4) == 0 &&
                      (dst_stride % 4) == 0 && band >= 6;
    if (bulk) {
        // two 48 KB buffers per CTA, two CTAs per SM (one CTA's loads overlap the
        // other's filtering); rows wider than ~3 KB take two 96 KB buffers
        // carry kernel when one CTA row of threads covers the row (one column group per thread)
        const int ncg = ow / 4;
        if (ncg > 256 && ncg <= 512 && carry_band_rows(96 * 1024, w) >= 6)
            launch_carry<512, 96 * 1024, 1>(src, src_stride, w, h, dst, dst_stride, frames, st);
        else if (ncg > 128 && ncg <= 256 && carry_band_rows(48 * 1024, w) >= 6)
            launch_carry<256, 48 * 1024, 2>(src, src_stride, w, h, dst, dst_stride, frames, st);
        else if (ncg > 64 && ncg <= 128 && carry_band_rows(24 * 1024, w) >= 6)
            launch_carry<128, 24 * 1024, 4>(src, src_stride, w, h, dst, dst_stride, frames, st);
        else if ((48 * 1024 / w - 4) / 2 >= 6)
            launch_bulk<256, 48 * 1024, 2>(src, src_stride, w, h, dst, dst_stride, frames, st);
        else
            launch_bulk<512, 96 * 1024, 1>(src, src_stride, w, h, dst, dst_stride, frames, st);
        return;
    }
    // streaming kernel: 8-byte aligned rows and frames, 4-byte aligned output rows
    const bool stream = (w % 8) == 0 && (ow % 4) == 0 && (reinterpret_cast<uintptr_t>(src) % 8) == 0 &&
                        (src_stride % 8) == 0 && (reinterpret_cast<uintptr_t>(dst) % 4) == 0 &&
                        (dst_stride % 4) == 0;
    for (int f0 = 0; f0 < frames; f0 += 65535) {
        const int nf = min(65535, frames - f0);
        if (stream) {
            const int threads = (w / 8 + 31) / 32 * 32;
            dim3 grid((threads + SPT - 1) / SPT, (oh + SBAND - 1) / SBAND, nf);
            pyramid_stream_kernel<<<grid, SPT, 0, st>>>(src + (size_t)f0 * src_stride, src_stride, w, h,
                                                        dst + (size_t)f0 * dst_stride, dst_stride);
        } else {
            dim3 grid((ow + TW - 1) / TW, (oh + TH - 1) / TH, nf);
            pyramid_level_kernel<<<grid, 256, 0, st>>>(src + (size_t)f0 * src_stride, src_stride, w, h,
                                                       dst + (size_t)f0 * dst_stride, dst_stride);
        }
    }
}

}  // namespace stabgpu
