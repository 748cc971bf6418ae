// k_eval.cu — colour conversion and evaluation kernels around the hot path.
//
// Reference: media_io.cpp:75-89 (BT.601 full-range YCbCr <-> RGB), 568-570
// (luma_bt601), 339-344 (RGB -> Y/Cb/Cr at load); synth_eval.cpp:214-240
// (psnr_pair: squared differences over the cropped region).
//
// Conversions: colour.cuh (fixed point with the reference's fp64 sequence for
// the pixels near a rounding tie; bit-exact, proven over all 2^24 inputs).  The PSNR
// kernel accumulates exact integer squared differences; the host forms the
// reference's double mse and log10 from the exact sum.
#include "colour.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace stabgpu {

namespace {

// RGB -> Y/Cb/Cr, 16 pixels per thread: three 16-byte loads of interleaved
// RGB, one 16-byte store per plane.  `rgb` may be device memory or pinned
// host memory (zero-copy: the conversion runs on the PCIe read itself, the
// fused upload).  Exact: colour::rgb_to_ycc (colour.cuh).
__global__ void rgb_to_ycbcr_kernel(const uint8_t* __restrict__ rgb, size_t npx, uint8_t* __restrict__ y,
                                    uint8_t* __restrict__ cb, uint8_t* __restrict__ cr, bool vec) {
    const size_t n16 = vec ? npx / 16 : 0, stride = (size_t)gridDim.x * blockDim.x;
#pragma unroll 4
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
        const uint4* src = reinterpret_cast<const uint4*>(rgb + 48 * i);
        const uint4 a = src[0], b = src[1], c = src[2];
        const uint32_t wv[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
        uint32_t oy[4], ob[4], orr[4];
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            const int k = 3 * p;
            const uint32_t r = (wv[k >> 2] >> (8 * (k & 3))) & 0xFF;
            const uint32_t g = (wv[(k + 1) >> 2] >> (8 * ((k + 1) & 3))) & 0xFF;
            const uint32_t bl = (wv[(k + 2) >> 2] >> (8 * ((k + 2) & 3))) & 0xFF;
            const uint32_t v = colour::rgb_to_ycc(r, g, bl);
            const int j = p >> 2, sh = 8 * (p & 3);
            if (sh == 0) {
                oy[j] = v & 0xFF;
                ob[j] = (v >> 8) & 0xFF;
                orr[j] = v >> 16;
            } else {
                oy[j] |= (v & 0xFF) << sh;
                ob[j] |= ((v >> 8) & 0xFF) << sh;
                orr[j] |= (v >> 16) << sh;
            }
        }
        reinterpret_cast<uint4*>(y)[i] = make_uint4(oy[0], oy[1], oy[2], oy[3]);
        reinterpret_cast<uint4*>(cb)[i] = make_uint4(ob[0], ob[1], ob[2], ob[3]);
        reinterpret_cast<uint4*>(cr)[i] = make_uint4(orr[0], orr[1], orr[2], orr[3]);
    }
    for (size_t i = 16 * n16 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < npx; i += stride) {
        const uint32_t v = colour::rgb_to_ycc(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
        y[i] = (uint8_t)v;
        cb[i] = (uint8_t)(v >> 8);
        cr[i] = (uint8_t)(v >> 16);
    }
}

// Y/Cb/Cr -> RGB, 16 pixels per thread (one 16-byte load per plane, three
// 16-byte stores of interleaved RGB; `rgb` may be pinned host memory).
__global__ void ycbcr_to_rgb_kernel(const uint8_t* __restrict__ y, const uint8_t* __restrict__ cb,
                                    const uint8_t* __restrict__ cr, size_t npx, uint8_t* __restrict__ rgb,
                                    bool vec) {
    const size_t n16 = vec ? npx / 16 : 0, stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
        const uint4 a = reinterpret_cast<const uint4*>(y)[i], b = reinterpret_cast<const uint4*>(cb)[i],
                    c = reinterpret_cast<const uint4*>(cr)[i];
        const uint32_t ya[4] = {a.x, a.y, a.z, a.w}, ba[4] = {b.x, b.y, b.z, b.w}, ca[4] = {c.x, c.y, c.z, c.w};
        uint32_t o[12];
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // pixels 4j .. 4j+3 -> words 3j .. 3j+2
            uint32_t px[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                px[q] = colour::ycc_to_rgb((ya[j] >> (8 * q)) & 0xFF, (ba[j] >> (8 * q)) & 0xFF,
                                           (ca[j] >> (8 * q)) & 0xFF);
            o[3 * j] = px[0] | px[1] << 24;
            o[3 * j + 1] = px[1] >> 8 | px[2] << 16;
            o[3 * j + 2] = px[2] >> 16 | px[3] << 8;
        }
        uint4* dst = reinterpret_cast<uint4*>(rgb + 48 * i);
        dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
        dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
        dst[2] = make_uint4(o[8], o[9], o[10], o[11]);
    }
    for (size_t i = 16 * n16 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < npx; i += stride) {
        const uint32_t v = colour::ycc_to_rgb(y[i], cb[i], cr[i]);
        rgb[3 * i] = (uint8_t)v;
        rgb[3 * i + 1] = (uint8_t)(v >> 8);
        rgb[3 * i + 2] = (uint8_t)(v >> 16);
    }
}

// sum over rows [my, h-my) x cols [mx, w-mx) of (a - b)^2 for frame pairs
// (k-1, k), k = 1 .. n-1 (grid.y = pair)
__global__ void sse_kernel(const uint8_t* __restrict__ f, size_t stride, int w, int h, int mx, int my,
                           unsigned long long* __restrict__ sse) {
    const uint8_t* a = f + (size_t)blockIdx.y * stride;
    const uint8_t* b = a + stride;
    const int cw = w - 2 * mx;
    const long long total = (long long)cw * (h - 2 * my);
    unsigned long long acc = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int yy = my + (int)(i / cw), xx = mx + (int)(i % cw);
        const int d = (int)a[(size_t)yy * w + xx] - (int)b[(size_t)yy * w + xx];
        acc += (unsigned long long)(d * d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&sse[blockIdx.y], acc);
}

int grid_for(size_t npx) {  // 16 pixels per thread
    const size_t b = (npx / 16 + 255) / 256 + 1;
    return (int)(b < 148 * 8 ? b : 148 * 8);
}

}  // namespace

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

void launch_rgb_to_ycbcr(const uint8_t* rgb, size_t npx, uint8_t* y, uint8_t* cb, uint8_t* cr, cudaStream_t st,
                         bool zero_copy) {
    if (!npx) return;
    const bool vec = al16(rgb) && al16(y) && al16(cb) && al16(cr);
    // zero-copy (rgb in pinned host memory, read over PCIe): a small resident
    // footprint — 64 threads per SM with four 48-byte groups in flight each
    // (~1.8 MB outstanding, far above PCIe's bandwidth-delay product) — so
    // the kernel streams at the link rate for the whole upload while the
    // compute kernels of earlier chunks keep the SMs
    if (zero_copy) rgb_to_ycbcr_kernel<<<sm_count(), 64, 0, st>>>(rgb, npx, y, cb, cr, vec);
    else rgb_to_ycbcr_kernel<<<grid_for(npx), 256, 0, st>>>(rgb, npx, y, cb, cr, vec);
}

void launch_ycbcr_to_rgb(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, size_t npx, uint8_t* rgb,
                         cudaStream_t st) {
    if (npx)
        ycbcr_to_rgb_kernel<<<grid_for(npx), 256, 0, st>>>(y, cb, cr, npx, rgb,
                                                           al16(rgb) && al16(y) && al16(cb) && al16(cr));
}

void launch_interframe_sse(const uint8_t* frames, int n, int w, int h, int mx, int my, unsigned long long* sse,
                           cudaStream_t st) {
    if (n < 2) return;
    cudaMemsetAsync(sse, 0, sizeof(unsigned long long) * (n - 1), st);
    dim3 grid(64, n - 1);
    sse_kernel<<<grid, 256, 0, st>>>(frames, (size_t)w * h, w, h, mx, my, sse);
}

}  // namespace stabgpu
