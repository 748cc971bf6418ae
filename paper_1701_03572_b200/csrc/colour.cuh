// colour.cuh — BT.601 full-range conversions of the reference
// (media_io.cpp:75-89 yuv_to_rgb / chroma_cb / chroma_cr, 568-570
// luma_bt601), bit-exact, for use inside other kernels (the RGB upload and
// K8's RGB store).
//
// The reference evaluates each channel in fp64 (products and sums in source
// order, then lround + clamp).  Here each channel is first evaluated in 10.22
// fixed point with 32-bit integer ops: every coefficient is rounded to a
// multiple of 2^-22 once, the channel value v + 1/2 is a sum of integer
// products, and the result is floor(.) + clamp.  The fixed-point sum differs
// from the exact real value by < 128 * 2^-23 per coefficient term, so the
// floor can differ from the reference's rounding only when the value lies
// within that distance of a .5 tie; such pixels (fraction within 256 units of
// the boundary: 0.4% of (r, g, b) triples for Cb / Cr, 0.8% of (y, cb, cr)
// for RGB — mostly exact real ties such as 1.772 * du = k + 1/2, where the
// reference's fp64 rounding decides) are recomputed with the reference's own
// fp64 sequence.
// tests/test_colour_fixed.py checks the rule against the reference formulas
// for every one of the 2^24 inputs of each conversion.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace stabgpu {

namespace colour {

constexpr int FB = 22;                     // fraction bits
constexpr int HALF = 1 << (FB - 1);
constexpr unsigned FMASK = (1u << FB) - 1u;
constexpr unsigned TIE = 256;              // fallback band around the rounding boundary
// round(c * 2^22) of the reference's coefficients
constexpr int K_R_V = 0x59ba5e;   // 1.402
constexpr int K_G_U = 0x160653;   // 0.344136
constexpr int K_G_V = 0x2db467;   // 0.714136
constexpr int K_B_U = 0x716873;   // 1.772
constexpr int K_CB_R = 0xacc92;   // 0.168736
constexpr int K_CB_G = 0x15336e;  // 0.331264
constexpr int K_CR_G = 0x1acbc9;  // 0.418688
constexpr int K_CR_B = 0x53437;   // 0.081312

__device__ __forceinline__ uint32_t clamp_lround_d(double v) {  // clamp_u8(std::lround(v))
    const long long r = llround(v);
    return (uint32_t)(r < 0 ? 0 : (r > 255 ? 255 : r));
}

// floor of a fixed-point value (v + 1/2 already added) clamped to [0, 255];
// near |= the value lies within TIE units of the boundary
__device__ __forceinline__ uint32_t fx_byte(int v, bool& near) {
    near |= ((unsigned)v + TIE & FMASK) <= 2 * TIE;
    return (uint32_t)min(max(v >> FB, 0), 255);
}

// yuv_to_rgb (media_io.cpp:75-81), packed r | g << 8 | b << 16
__device__ __forceinline__ uint32_t ycc_to_rgb(uint32_t y, uint32_t cb, uint32_t cr) {
    const int du = (int)cb - 128, dv = (int)cr - 128, yv = ((int)y << FB) + HALF;
    bool near = false;
    const uint32_t r = fx_byte(yv + dv * K_R_V, near);
    const uint32_t g = fx_byte(yv - du * K_G_U - dv * K_G_V, near);
    const uint32_t b = fx_byte(yv + du * K_B_U, near);
    if (!near) return r | g << 8 | b << 16;
    const double yy = (double)y, ddu = dsub((double)cb, 128.0), ddv = dsub((double)cr, 128.0);
    return clamp_lround_d(dadd(yy, dmul(1.402, ddv))) |
           clamp_lround_d(dsub(dsub(yy, dmul(0.344136, ddu)), dmul(0.714136, ddv))) << 8 |
           clamp_lround_d(dadd(yy, dmul(1.772, ddu))) << 16;
}

// luma_bt601 / chroma_cb / chroma_cr (media_io.cpp:83-89, 568-570), packed
// y | cb << 8 | cr << 16
__device__ __forceinline__ uint32_t rgb_to_ycc(uint32_t r, uint32_t g, uint32_t b) {
    const uint32_t y = (299u * r + 587u * g + 114u * b + 500u) / 1000u;
    const int base = (128 << FB) + HALF;
    bool near = false;
    const uint32_t cb = fx_byte(base - (int)r * K_CB_R - (int)g * K_CB_G + ((int)b << (FB - 1)), near);
    const uint32_t cr = fx_byte(base + ((int)r << (FB - 1)) - (int)g * K_CR_G - (int)b * K_CR_B, near);
    if (!near) return y | cb << 8 | cr << 16;
    const double rr = (double)r, gg = (double)g, bb = (double)b;
    return y | clamp_lround_d(dadd(dsub(dsub(128.0, dmul(0.168736, rr)), dmul(0.331264, gg)), dmul(0.5, bb))) << 8 |
           clamp_lround_d(dsub(dsub(dadd(128.0, dmul(0.5, rr)), dmul(0.418688, gg)), dmul(0.081312, bb))) << 16;
}

}  // namespace colour

}  // namespace stabgpu
