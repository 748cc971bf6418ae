// common.cuh — shared device helpers for the sm_100a stabilization kernels.
//
// Floating-point rule for every kernel: where the reference C++
// (/root/reference/proj/src) evaluates an expression, the device code uses
// the explicitly rounded intrinsics (__dadd_rn, __dmul_rn, ...) in the SAME
// order, so ptxas can never fuse a multiply-add the x86-64 reference did not
// fuse.  Only reductions whose order differs by construction (warp/block
// trees) are allowed to differ, and the tests bound that difference.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "../../include/stabgpu.h"

namespace stabgpu {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

// clamp_u8(std::lround(v)), image_ops.cpp:19-21 — lround rounds half away
// from zero, which __double2int_rn (half to even) does not.
__device__ __forceinline__ uint8_t round_u8(double v) {
    const long long r = llround(v);
    return (uint8_t)(r < 0 ? 0 : (r > 255 ? 255 : r));
}

// sample_bilinear, image_ops.cpp:98-113 (0 outside [0,w-1]x[0,h-1]), with
// the pixel fetch abstracted (global frame or a staged shared-memory copy).
template <typename F>
__device__ __forceinline__ double bilinear_f(F fetch, int w, int h, double px, double py) {
    const double xmax = (double)w - 1.0, ymax = (double)h - 1.0;
    if (!(px >= 0.0 && py >= 0.0 && px <= xmax && py <= ymax)) return 0.0;
    const int x0 = (int)px, y0 = (int)py;
    const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
    const double fx = dsub(px, (double)x0), fy = dsub(py, (double)y0);
    const double a = fetch(x0, y0), b = fetch(x1, y0);
    const double c = fetch(x0, y1), d = fetch(x1, y1);
    const double top = dadd(a, dmul(fx, dsub(b, a)));
    const double bot = dadd(c, dmul(fx, dsub(d, c)));
    return dadd(top, dmul(fy, dsub(bot, top)));
}

__device__ __forceinline__ double sample_bilinear(const uint8_t* __restrict__ f, int w, int h,
                                                  double px, double py) {
    return bilinear_f([=](int x, int y) { return (double)f[(size_t)y * w + x]; }, w, h, px, py);
}

// Positive doubles order like their bit patterns.
__device__ __forceinline__ unsigned long long dbits(double v) {
    return (unsigned long long)__double_as_longlong(v);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Butterfly sum of doubles: IEEE addition is commutative, so every lane ends
// with the same bits and control flow that depends on the sum stays uniform.
__device__ __forceinline__ double warp_dsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---- host: launch facts cached per (kernel, device) ------------------------
// The attribute and occupancy queries cost microseconds each; Stage II
// launches every kernel once per frame, so they are asked once.
struct LaunchCache {
    std::mutex m;
    std::map<std::tuple<const void*, int, int, size_t>, int> occ;  // (fn, dev, threads, smem) -> blocks/SM
    std::map<std::pair<const void*, int>, size_t> smem;             // (fn, dev) -> opted-in dynamic smem
    std::map<int, int> sms;
};

inline LaunchCache& launch_cache() {
    static LaunchCache c;
    return c;
}

inline int cur_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

inline int sm_count() {
    LaunchCache& c = launch_cache();
    const int d = cur_device();
    std::lock_guard<std::mutex> g(c.m);
    auto it = c.sms.find(d);
    if (it != c.sms.end()) return it->second;
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    c.sms[d] = n;
    return n;
}

// opt the kernel in to `bytes` of dynamic shared memory (only when it grows).
// The size is cached only when the attribute was accepted; a refused size
// leaves the error for the launch check (check_launch) to report.
template <typename K>
inline cudaError_t ensure_smem(K* fn, size_t bytes) {
    LaunchCache& c = launch_cache();
    const auto key = std::make_pair(reinterpret_cast<const void*>(fn), cur_device());
    std::lock_guard<std::mutex> g(c.m);
    auto it = c.smem.find(key);
    if (it != c.smem.end() && it->second >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) c.smem[key] = bytes;
    return e;
}

template <typename K>
inline int blocks_per_sm(K* fn, int threads, size_t bytes) {
    LaunchCache& c = launch_cache();
    const auto key = std::make_tuple(reinterpret_cast<const void*>(fn), cur_device(), threads, bytes);
    {
        std::lock_guard<std::mutex> g(c.m);
        auto it = c.occ.find(key);
        if (it != c.occ.end()) return it->second;
    }
    int per = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, bytes);
    per = per > 0 ? per : 1;
    std::lock_guard<std::mutex> g(c.m);
    c.occ[key] = per;
    return per;
}

}  // namespace stabgpu

#define STABGPU_HOST_DEVICE __host__ __device__
