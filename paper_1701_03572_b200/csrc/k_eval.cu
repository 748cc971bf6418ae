// k_eval.cu — colour conversion and evaluation kernels around the hot path.
//
// Reference: media_io.cpp:75-89 (BT.601 full-range YCbCr <-> RGB), 568-570
// (luma_bt601), 339-344 (RGB -> Y/Cb/Cr at load); synth_eval.cpp:214-240
// (psnr_pair: squared differences over the cropped region).
//
// Conversions are per pixel with the reference's own arithmetic: the integer
// luma formula, and fp64 products/sums in source order with lround + clamp
// for chroma and RGB (correctly rounded fp64 ops, so bit-exact).  The PSNR
// kernel accumulates exact integer squared differences; the host forms the
// reference's double mse and log10 from the exact sum.
#include "common.cuh"
#include "kernels.cuh"

namespace stabgpu {

namespace {

__device__ __forceinline__ uint8_t clamp_lround(double v) {  // clamp_u8(std::lround(v))
    const long long r = llround(v);
    return (uint8_t)(r < 0 ? 0 : (r > 255 ? 255 : r));
}

__global__ void rgb_to_ycbcr_kernel(const uint8_t* __restrict__ rgb, size_t npx, uint8_t* __restrict__ y,
                                    uint8_t* __restrict__ cb, uint8_t* __restrict__ cr) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < npx; i += (size_t)gridDim.x * blockDim.x) {
        const unsigned r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
        y[i] = (uint8_t)((299u * r + 587u * g + 114u * b + 500u) / 1000u);  // luma_bt601
        // chroma_cb: 128.0 - 0.168736*r - 0.331264*g + 0.5*b, left to right
        cb[i] = clamp_lround(dadd(dsub(dsub(128.0, dmul(0.168736, (double)r)), dmul(0.331264, (double)g)),
                                  dmul(0.5, (double)b)));
        // chroma_cr: 128.0 + 0.5*r - 0.418688*g - 0.081312*b
        cr[i] = clamp_lround(dsub(dsub(dadd(128.0, dmul(0.5, (double)r)), dmul(0.418688, (double)g)),
                                  dmul(0.081312, (double)b)));
    }
}

__global__ void ycbcr_to_rgb_kernel(const uint8_t* __restrict__ y, const uint8_t* __restrict__ cb,
                                    const uint8_t* __restrict__ cr, size_t npx, uint8_t* __restrict__ rgb) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < npx; i += (size_t)gridDim.x * blockDim.x) {
        const double yy = (double)y[i];
        const double du = dsub((double)cb[i], 128.0), dv = dsub((double)cr[i], 128.0);
        rgb[3 * i] = clamp_lround(dadd(yy, dmul(1.402, dv)));
        rgb[3 * i + 1] = clamp_lround(dsub(dsub(yy, dmul(0.344136, du)), dmul(0.714136, dv)));
        rgb[3 * i + 2] = clamp_lround(dadd(yy, dmul(1.772, du)));
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

int grid_for(size_t npx) {
    const size_t b = (npx + 255) / 256;
    return (int)(b < 148 * 32 ? b : 148 * 32);
}

}  // namespace

void launch_rgb_to_ycbcr(const uint8_t* rgb, size_t npx, uint8_t* y, uint8_t* cb, uint8_t* cr, cudaStream_t st) {
    if (npx) rgb_to_ycbcr_kernel<<<grid_for(npx), 256, 0, st>>>(rgb, npx, y, cb, cr);
}

void launch_ycbcr_to_rgb(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, size_t npx, uint8_t* rgb,
                         cudaStream_t st) {
    if (npx) ycbcr_to_rgb_kernel<<<grid_for(npx), 256, 0, st>>>(y, cb, cr, npx, rgb);
}

void launch_interframe_sse(const uint8_t* frames, int n, int w, int h, int mx, int my, unsigned long long* sse,
                           cudaStream_t st) {
    if (n < 2) return;
    cudaMemsetAsync(sse, 0, sizeof(unsigned long long) * (n - 1), st);
    dim3 grid(64, n - 1);
    sse_kernel<<<grid, 256, 0, st>>>(frames, (size_t)w * h, w, h, mx, my, sse);
}

}  // namespace stabgpu
