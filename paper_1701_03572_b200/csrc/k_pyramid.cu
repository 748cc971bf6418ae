// k_pyramid.cu — K1: fused binomial blur + 2x decimation, batched over frames.
//
// Reference: downsample + build_pyramid, image_ops.cpp:25-77.  The reference
// filters every column horizontally into 16-bit, then filters even rows /
// even columns vertically and rounds with (acc + 128) >> 8, replicating
// borders.  All arithmetic is integer, so any evaluation order is exact; the
// kernel computes only the even columns the vertical pass consumes.
//
// One CTA = a 64x16 tile of output pixels of one frame (grid.z = frame).
// The (2*16+3) x (2*64+3) input window is staged in shared memory with
// 32-bit loads when the tile is interior and rows are 4-byte aligned.
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

}  // namespace

void launch_pyramid_level(const uint8_t* src, size_t src_stride, int w, int h, uint8_t* dst,
                          size_t dst_stride, int frames, cudaStream_t st) {
    const int ow = w / 2, oh = h / 2;
    if (frames <= 0 || ow <= 0 || oh <= 0) return;
    for (int f0 = 0; f0 < frames; f0 += 65535) {
        const int nf = min(65535, frames - f0);
        dim3 grid((ow + TW - 1) / TW, (oh + TH - 1) / TH, nf);
        pyramid_level_kernel<<<grid, 256, 0, st>>>(src + (size_t)f0 * src_stride, src_stride, w, h,
                                                   dst + (size_t)f0 * dst_stride, dst_stride);
    }
}

}  // namespace stabgpu
