// transfer.cu — SURVEY.md 8f row 3: the renderer's second caller, GS -> TSDF
// (/root/reference/proj/core/src/transfer.cpp).
//
//   field_bounds      transfer.cpp:27-34 over pose_primitive (trace.cpp:14-36): one thread per
//                     primitive computes the 3-sigma box, a block min/max, then one block
//                     reduces the per-block boxes (fmin / fmax are order independent, so the
//                     result equals the reference's serial Aabb::expand loop)
//   ring cameras      transfer.cpp:84-112 on the host (look_at, raster.cpp:25-42)
//   tsdf_fuse         transfer.cpp:143-172: one thread per voxel (x fastest, coalesced) keeps
//                     its tsdf and weight in registers and walks the views IN ORDER, so V
//                     views cost one read and one write of the volume instead of V of each;
//                     the per-view arithmetic is the reference's, in double, operation for
//                     operation (this file is compiled with -fmad=false), so the fused grid
//                     is bit-identical to V sequential reference calls on the same depth maps.
// render_depth_ring's depth masking (alpha < 0.5 -> 0, transfer.cpp:116-118) happens in the
// raster epilogue (RasterArgs::valid_alpha).
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "../../include/gsim_gpu.h"
#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {
constexpr int kBoundsThreads = 256;
constexpr double kBoundsSigma = 3.0;  // trace.hpp:25

__device__ __forceinline__ int trunc_int_x86(double x) {  // static_cast<int> as cvttsd2si
    if (!(x >= -2147483648.0 && x < 2147483648.0)) return INT32_MIN;
    return static_cast<int>(x);
}

// Block-wide fmin / fmax of 6 values (lo xyz, hi xyz) into out[0..5].
__device__ void block_minmax(double v[6], double* out) {
    __shared__ double s[6][kBoundsThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, x, o);
            x = k < 3 ? fmin(x, y) : fmax(x, y);
        }
        if (lane == 0) s[k][warp] = x;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        const int k = threadIdx.x;
        double x = s[k][0];
        for (int w = 1; w < kBoundsThreads / 32; ++w) x = k < 3 ? fmin(x, s[k][w]) : fmax(x, s[k][w]);
        out[k] = x;
    }
}
}  // namespace

__global__ void __launch_bounds__(kBoundsThreads) bounds_kernel(DevField f, double* partial) {
    double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < f.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        // pose_primitive(p, identity): the identity pose leaves mean and rotation bit-exact
        const dq rot = qmul(dq{1.0, 0.0, 0.0, 0.0}, dq{f.qw[i], f.qx[i], f.qy[i], f.qz[i]});
        const dm3 r = qmatrix(rot);
        const double sx = f.sx[i], sy = f.sy[i], sz = f.sz[i];
        const dm3 d{{sx * sx, 0, 0, 0, sy * sy, 0, 0, 0, sz * sz}};
        const dm3 cov = mmul(mmul(r, d), mtransposed(r));
        const double half[3] = {kBoundsSigma * sqrt(cov.m[0]), kBoundsSigma * sqrt(cov.m[4]),
                                kBoundsSigma * sqrt(cov.m[8])};
        const dv3 mean = add3(qrotate(dq{1.0, 0.0, 0.0, 0.0}, mk3(f.mx[i], f.my[i], f.mz[i])),
                              mk3(0.0, 0.0, 0.0));
        const double m[3] = {mean.x, mean.y, mean.z};
#pragma unroll
        for (int k = 0; k < 3; ++k) {  // bounds.expand(mean - half), bounds.expand(mean + half)
            const double a = m[k] - half[k], b = m[k] + half[k];
            double lo = fmin(INFINITY, a), hi = fmax(-INFINITY, a);
            lo = fmin(lo, b);
            hi = fmax(hi, b);
            v[k] = fmin(v[k], lo);
            v[3 + k] = fmax(v[3 + k], hi);
        }
    }
    block_minmax(v, partial + 6 * uint64_t(blockIdx.x));
}

__global__ void __launch_bounds__(kBoundsThreads) bounds_reduce_kernel(const double* partial,
                                                                       int n_blocks, double* out) {
    double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int b = threadIdx.x; b < n_blocks; b += blockDim.x)
#pragma unroll
        for (int k = 0; k < 6; ++k)
            v[k] = k < 3 ? fmin(v[k], partial[6 * b + k]) : fmax(v[k], partial[6 * b + k]);
    block_minmax(v, out);
}

__global__ void tsdf_reset_kernel(double* tsdf, double* weights, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        tsdf[i] = 1.0;
        weights[i] = 0.0;
    }
}

// One thread per voxel, views in order (tsdf_fuse, transfer.cpp:150-171, per view).
__global__ void __launch_bounds__(256) tsdf_fuse_kernel(TsdfArgs a) {
    extern __shared__ DevFuseView s_views[];
    for (uint32_t k = threadIdx.x; k < a.n_views; k += blockDim.x) s_views[k] = a.views[k];
    __syncthreads();
    const uint64_t nx = uint64_t(a.dims[0]), ny = uint64_t(a.dims[1]);
    const uint64_t n = nx * ny * uint64_t(a.dims[2]);
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < n;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const int x = int(idx % nx), y = int((idx / nx) % ny), z = int(idx / (nx * ny));
        // voxel_center, transfer.hpp:53-56
        const dv3 p = add3(mk3(a.origin[0], a.origin[1], a.origin[2]),
                           mk3((x + 0.5) * a.voxel_size, (y + 0.5) * a.voxel_size,
                               (z + 0.5) * a.voxel_size));
        double tsdf = a.tsdf[idx], w = a.weights[idx];
        bool touched = false;
        for (uint32_t k = 0; k < a.n_views; ++k) {
            const DevFuseView& v = s_views[k];
            const dv3 cp = add3(qrotate(dq{v.q[0], v.q[1], v.q[2], v.q[3]}, p),
                                mk3(v.t[0], v.t[1], v.t[2]));
            if (cp.z <= 0.0) continue;
            const int px = trunc_int_x86(floor(v.fx * cp.x / cp.z + v.cx));
            const int py = trunc_int_x86(floor(v.fy * cp.y / cp.z + v.cy));
            if (px < 0 || px >= v.width || py < 0 || py >= v.height) continue;
            const double measured = __ldg(a.depth + v.depth_offset + uint64_t(py) * v.width + px);
            if (measured <= 0.0) continue;  // invalid pixel
            const double sdf = measured - cp.z;
            if (sdf <= -a.truncation) continue;
            const double q = sdf / a.truncation;
            const double clamped = (q < -1.0) ? -1.0 : (1.0 < q) ? 1.0 : q;  // std::clamp
            tsdf = (tsdf * w + clamped) / (w + 1.0);
            w = w + 1.0;
            touched = true;
        }
        if (touched) {
            a.tsdf[idx] = tsdf;
            a.weights[idx] = w;
        }
    }
}

// ---- host side -------------------------------------------------------------------------------

void launch_bounds(const DevField& f, double* partial, int max_blocks, double* out,
                   cudaStream_t s) {
    const uint64_t want = (f.n + kBoundsThreads - 1) / kBoundsThreads;
    const int blocks = int(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(max_blocks))));
    bounds_kernel<<<blocks, kBoundsThreads, 0, s>>>(f, partial);
    bounds_reduce_kernel<<<1, kBoundsThreads, 0, s>>>(partial, blocks, out);
}

void launch_tsdf_reset(double* tsdf, double* weights, uint64_t n, int n_sms, cudaStream_t s) {
    if (!n) return;
    const uint64_t want = (n + 255) / 256;
    tsdf_reset_kernel<<<unsigned(std::min<uint64_t>(want, uint64_t(n_sms) * 8)), 256, 0, s>>>(
        tsdf, weights, n);
}

void launch_tsdf_fuse(const TsdfArgs& a, int n_sms, cudaStream_t s) {
    const uint64_t n = uint64_t(a.dims[0]) * a.dims[1] * a.dims[2];
    if (!n || !a.n_views) return;
    const size_t smem = sizeof(DevFuseView) * a.n_views;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(tsdf_fuse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const uint64_t want = (n + 255) / 256;
    tsdf_fuse_kernel<<<unsigned(std::min<uint64_t>(want, uint64_t(n_sms) * 16)), 256, smem, s>>>(a);
}

namespace {
dv3 normalized3(dv3 a) {  // math.hpp:39-42
    const double n = std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z);
    return n > 0.0 ? mk3(a.x / n, a.y / n, a.z / n) : mk3(0.0, 0.0, 0.0);
}

dq quat_from_matrix(const double* m) {  // Quat::from_matrix, math.hpp:158-187 (row-major)
    auto M = [&](int r, int c) { return m[r * 3 + c]; };
    dq q;
    const double tr = M(0, 0) + M(1, 1) + M(2, 2);
    if (tr > 0.0) {
        const double s = std::sqrt(tr + 1.0) * 2.0;
        q.w = 0.25 * s;
        q.x = (M(2, 1) - M(1, 2)) / s;
        q.y = (M(0, 2) - M(2, 0)) / s;
        q.z = (M(1, 0) - M(0, 1)) / s;
    } else if (M(0, 0) > M(1, 1) && M(0, 0) > M(2, 2)) {
        const double s = std::sqrt(1.0 + M(0, 0) - M(1, 1) - M(2, 2)) * 2.0;
        q.w = (M(2, 1) - M(1, 2)) / s;
        q.x = 0.25 * s;
        q.y = (M(0, 1) + M(1, 0)) / s;
        q.z = (M(0, 2) + M(2, 0)) / s;
    } else if (M(1, 1) > M(2, 2)) {
        const double s = std::sqrt(1.0 + M(1, 1) - M(0, 0) - M(2, 2)) * 2.0;
        q.w = (M(0, 2) - M(2, 0)) / s;
        q.x = (M(0, 1) + M(1, 0)) / s;
        q.y = 0.25 * s;
        q.z = (M(1, 2) + M(2, 1)) / s;
    } else {
        const double s = std::sqrt(1.0 + M(2, 2) - M(0, 0) - M(1, 1)) * 2.0;
        q.w = (M(1, 0) - M(0, 1)) / s;
        q.x = (M(0, 2) + M(2, 0)) / s;
        q.y = (M(1, 2) + M(2, 1)) / s;
        q.z = 0.25 * s;
    }
    return qnormalized(q);
}

// CameraModel::look_at (raster.cpp:25-42) with the default up = +z (camera.hpp:32).
gsim_camera look_at(dv3 eye, dv3 target, double fx, double fy, int width, int height) {
    gsim_camera cam{};
    cam.fx = fx;
    cam.fy = fy;
    cam.cx = width * 0.5;
    cam.cy = height * 0.5;
    cam.width = width;
    cam.height = height;
    cam.near_plane = 0.05;  // camera.hpp:20
    cam.far_plane = 100.0;
    const dv3 forward = normalized3(sub3(target, eye));
    dv3 right = normalized3(cross3(forward, mk3(0.0, 0.0, 1.0)));
    if (right.x * right.x + right.y * right.y + right.z * right.z < 1e-20)
        right = normalized3(cross3(forward, mk3(0.0, 1.0, 0.0)));
    const dv3 down = cross3(forward, right);
    const double w2c[9] = {right.x, right.y, right.z, down.x, down.y, down.z,
                           forward.x, forward.y, forward.z};
    const dq q = quat_from_matrix(w2c);
    const dv3 t = qrotate(q, eye);
    cam.pose.rotation[0] = q.w;
    cam.pose.rotation[1] = q.x;
    cam.pose.rotation[2] = q.y;
    cam.pose.rotation[3] = q.z;
    cam.pose.translation[0] = -t.x;
    cam.pose.translation[1] = -t.y;
    cam.pose.translation[2] = -t.z;
    return cam;
}
}  // namespace

// render_depth_ring's camera set-up (transfer.cpp:84-112). Returns a validation message or
// nullptr.
const char* depth_ring_cameras(const double lo[3], const double hi[3], int n_views, double radius,
                               int resolution, gsim_camera* cameras) {
    if (n_views < 8) return "render_depth_ring: n_views must be >= 8";
    if (!(radius > 0.0)) return "render_depth_ring: radius must be positive";
    const dv3 l = mk3(lo[0], lo[1], lo[2]), h = mk3(hi[0], hi[1], hi[2]);
    const dv3 extent = sub3(h, l);
    const double diag = std::sqrt(extent.x * extent.x + extent.y * extent.y + extent.z * extent.z);
    if (!(diag > 0.0)) return "render_depth_ring: degenerate field bounding box";
    const dv3 center = scale3(add3(l, h), 0.5);
    // focal length so the bounding sphere fits with margin
    const double tan_half = 0.65 * diag / radius;
    const double focal = 0.5 * resolution / tan_half;
    constexpr double kPi = 3.14159265358979323846;  // math.hpp:265-266
    constexpr double kTwoPi = 2.0 * kPi;
    const double elevations[3] = {-kPi / 6.0, 0.0, kPi / 6.0};  // transfer.cpp:21
    int v = 0;
    for (double elevation : elevations) {
        for (int k = 0; k < n_views; ++k, ++v) {
            const double azimuth = kTwoPi * k / n_views;
            const dv3 dir = mk3(std::cos(elevation) * std::cos(azimuth),
                                std::cos(elevation) * std::sin(azimuth), std::sin(elevation));
            const dv3 eye = add3(center, scale3(dir, radius));
            cameras[v] = look_at(eye, center, focal, focal, resolution, resolution);
            cameras[v].near_plane = std::max(1e-4, radius - diag);
            cameras[v].far_plane = radius + diag;
        }
    }
    return nullptr;
}

DevFuseView fuse_view(const gsim_camera& c, uint64_t depth_offset) {
    DevFuseView v{};
    for (int k = 0; k < 4; ++k) v.q[k] = c.pose.rotation[k];
    for (int k = 0; k < 3; ++k) v.t[k] = c.pose.translation[k];
    v.fx = c.fx;
    v.fy = c.fy;
    v.cx = c.cx;
    v.cy = c.cy;
    v.width = c.width;
    v.height = c.height;
    v.depth_offset = depth_offset;
    return v;
}

}  // namespace gsim_gpu
