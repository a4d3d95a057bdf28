// encode.cuh — byte encodings of a rendered pixel (image_io.cpp), shared by the fused raster
// epilogue (raster.cu) and the standalone encode kernel (encode.cu).
//
// Bit-exactness with the reference's writers:
//  * quantize8(clamp(v, 0, 1)) (image_io.cpp:43-45, :80-81, :92) is double arithmetic on the
//    float value: v*255.0 is exact IEEE on both sides and lround == llround (half away from 0).
//  * the sRGB path (linear_to_srgb, :19-22) goes through libm pow; the kernels never evaluate
//    it. The host precomputes, with the same transfer function, the 256 float thresholds at
//    which the 8-bit code steps (host.cu build_srgb_thresholds), and the device does an 8-step
//    binary search: for float inputs this equals quantize8(linear_to_srgb(v)) exactly.
//  * NaN: std::clamp keeps NaN and lround(NaN) is LONG_MIN on x86-64, clamped to 0 -> code 0.
//  * write_png_gray16 (:99-111): lround(double(v) * scale) clamped to [0, 65535], stored
//    big-endian. |x| >= 2^63 (or NaN) converts to LONG_MIN on x86-64 -> 0, emulated here.
#pragma once

#include <cstdint>

#include "../../include/gsim_gpu.h"

namespace gsim_gpu {

struct EncodeParams {
    uint8_t* dst;            // encoded blob (per camera blocks)
    const float* srgb_thr;   // [256] device thresholds (build_srgb_thresholds)
    double depth_scale;
    uint32_t flags;          // GSIM_ENCODE_*
    int32_t srgb;
};

// Bytes per pixel of the enabled parts.
__host__ __device__ inline uint32_t encoded_bpp(uint32_t flags) {
    return ((flags & GSIM_ENCODE_RGB8) ? 3u : 0u) + ((flags & GSIM_ENCODE_ALPHA8) ? 1u : 0u) +
           ((flags & GSIM_ENCODE_DEPTH16) ? 2u : 0u) + ((flags & GSIM_ENCODE_DEPTH_PFM) ? 4u : 0u);
}

__device__ __forceinline__ uint32_t quantize_unit(float v) {
    double d = double(v);
    if (!(d > 0.0)) return 0u;  // negatives, -0, NaN
    if (d > 1.0) d = 1.0;
    return uint32_t(llround(d * 255.0));
}

// Largest k with v >= thr[k]; thr[0] = -inf, thr monotone. NaN compares false -> 0.
__device__ __forceinline__ uint32_t quantize_srgb(float v, const float* thr) {
    uint32_t k = 0;
#pragma unroll
    for (uint32_t step = 128; step; step >>= 1)
        if (v >= thr[k + step]) k += step;
    return k;
}

__device__ __forceinline__ uint32_t quantize_depth16(float v, double scale) {
    const double x = double(v) * scale;
    if (!(fabs(x) < 9223372036854775808.0)) return 0u;  // NaN / out of long range -> LONG_MIN -> 0
    const long long r = llround(x);
    return r < 0 ? 0u : (r > 65535 ? 65535u : uint32_t(r));
}

// Write pixel (x, y) of a width x height camera whose block starts at `cam`.
__device__ __forceinline__ void encode_pixel(const EncodeParams& e, const float* thr, uint8_t* cam,
                                             uint32_t width, uint32_t height, uint32_t x,
                                             uint32_t y, float r, float g, float b, float depth,
                                             float alpha) {
    const size_t npx = size_t(width) * height;
    const size_t p = size_t(y) * width + x;
    uint8_t* part = cam;
    if (e.flags & GSIM_ENCODE_RGB8) {
        if (e.srgb) {
            part[3 * p + 0] = uint8_t(quantize_srgb(r, thr));
            part[3 * p + 1] = uint8_t(quantize_srgb(g, thr));
            part[3 * p + 2] = uint8_t(quantize_srgb(b, thr));
        } else {
            part[3 * p + 0] = uint8_t(quantize_unit(r));
            part[3 * p + 1] = uint8_t(quantize_unit(g));
            part[3 * p + 2] = uint8_t(quantize_unit(b));
        }
        part += 3 * npx;
    }
    if (e.flags & GSIM_ENCODE_ALPHA8) {
        part[p] = uint8_t(quantize_unit(alpha));
        part += npx;
    }
    if (e.flags & GSIM_ENCODE_DEPTH16) {
        const uint32_t q = quantize_depth16(depth, e.depth_scale);
        part[2 * p + 0] = uint8_t(q >> 8);  // PNG is big-endian (image_io.cpp:104)
        part[2 * p + 1] = uint8_t(q & 0xffu);
        part += 2 * npx;
    }
    if (e.flags & GSIM_ENCODE_DEPTH_PFM) {
        // rows bottom-up (image_io.cpp:171-177)
        uint8_t* q = part + 4 * (size_t(height - 1 - y) * width + x);
        if ((reinterpret_cast<uintptr_t>(q) & 3u) == 0) {
            *reinterpret_cast<float*>(q) = depth;
        } else {  // packed blocks of odd-sized cameras: little-endian bytes
            const uint32_t u = __float_as_uint(depth);
            q[0] = uint8_t(u);
            q[1] = uint8_t(u >> 8);
            q[2] = uint8_t(u >> 16);
            q[3] = uint8_t(u >> 24);
        }
    }
}

}  // namespace gsim_gpu
