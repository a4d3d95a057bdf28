// lidar.cu — SURVEY.md 8f row 4: LiDAR Gaussian ray tracing (/root/reference/proj/core/src/
// trace.cpp, bvh.hpp). Compiled with -fmad=false: every quantity that decides a hit is the
// reference's double arithmetic operation for operation.
//
// The reference poses the field, builds a SAH BVH and, per ray, gathers the primitives whose
// 3-sigma box the ray hits, sorts them by (peak t, index) and composites front to back. The BVH
// only accelerates: the candidate set is exactly {i : ray_aabb_hit(box_i)} (trace_linear is the
// contract). A spinning LiDAR's rays form a regular (channel, azimuth) grid around one origin,
// so instead of a tree we BIN primitives into that grid like tiles of an image:
//   lidar_pose_kernel     pose_primitive (trace.cpp:14-36) per primitive into SoA planes, plus the
//                         conservative (channel rank, azimuth step) rectangle of rays that can hit
//                         its box (box corners in the sensor frame -> azimuth / elevation ranges)
//   lidar_count_kernel    rays per rectangle row as +1/-1 row differences (global atomics)
//   lidar_rowscan_kernel  row prefix -> candidates per ray; a device-wide scan -> list offsets
//   lidar_scatter_kernel  every (ray, primitive) candidate at its ray's cursor (order free: the
//                         tracer orders by (t, index) itself)
//   lidar_trace_kernel    one warp per ray: exact ray_aabb_hit + ray_gaussian_peak per candidate,
//                         the survivors (response >= 1/255) compacted into a shared-memory pool,
//                         composited in (t, index) order by repeated warp arg-min over the pool
//                         (trace.cpp:65-85) until the transmittance cutoff; a ray with more
//                         survivors than the pool re-scans its list per step (same result)
//   lidar_emit_kernel     returns compacted in ray order: channel-major, azimuth ascending
// Sensor-frame ray directions are computed on the host with the reference's cos / sin (glibc,
// cached per channel set) and rotated on the device in the reference's double order, so the
// rays are bit-identical; only exp differs (CUDA's vs glibc's, <= 1 ulp).
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "../../include/gsim_gpu.h"
#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {
constexpr double kTraceScaleFloor = 1e-7;  // trace.hpp:24
constexpr double kBoundsSigmaL = 3.0;      // trace.hpp:25
constexpr double kTraceAlphaClamp = 0.99;  // trace.cpp:59-61
constexpr double kTraceAlphaSkip = 1.0 / 255.0;
constexpr double kTraceCutoff = 1e-4;
constexpr double kAngleMargin = 1e-7;      // radians added to every angular bound

__device__ __forceinline__ dv3 ldx3(const double* p, uint64_t i) {  // interleaved xyz
    return mk3(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
}

__device__ __forceinline__ dv3 matvec(const double* m, dv3 v) {  // Mat3 * Vec3, math.hpp:87-89
    return mk3(m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
               m[6] * v.x + m[7] * v.y + m[8] * v.z);
}

__device__ __forceinline__ double dot3(dv3 a, dv3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

__device__ __forceinline__ bool ray_aabb_hit(dv3 lo, dv3 hi, dv3 o, dv3 inv, double t_max) {
    // bvh.hpp:20-36, slab test over [0, t_max]
    double t0 = 0.0, t1 = t_max;
    const double tx0 = (lo.x - o.x) * inv.x, tx1 = (hi.x - o.x) * inv.x;
    t0 = fmax(t0, fmin(tx0, tx1));
    t1 = fmin(t1, fmax(tx0, tx1));
    const double ty0 = (lo.y - o.y) * inv.y, ty1 = (hi.y - o.y) * inv.y;
    t0 = fmax(t0, fmin(ty0, ty1));
    t1 = fmin(t1, fmax(ty0, ty1));
    const double tz0 = (lo.z - o.z) * inv.z, tz1 = (hi.z - o.z) * inv.z;
    t0 = fmax(t0, fmin(tz0, tz1));
    t1 = fmin(t1, fmax(tz0, tz1));
    return t0 <= t1;
}

// Peak of a primitive along the ray (trace.cpp:38-49) from its trace row; response 0 when
// d^T S^-1 d <= 0.
__device__ __forceinline__ void ray_peak_row(const double2* R, double opacity, dv3 o, dv3 d,
                                             double t_max, double& t, double& response) {
    const double2 r4 = __ldg(R + 4), r5 = __ldg(R + 5), r6 = __ldg(R + 6), r7 = __ldg(R + 7),
                  r8 = __ldg(R + 8), r9 = __ldg(R + 9);
    const dv3 mean = mk3(r4.x, r4.y, r5.x);
    const double ic[9] = {r5.y, r6.x, r6.y, r7.x, r7.y, r8.x, r8.y, r9.x, r9.y};
    const dv3 to_mean = sub3(mean, o);
    const dv3 si_d = matvec(ic, d);
    const double denom = dot3(d, si_d);
    t = 0.0;
    response = 0.0;
    if (!(denom > 0.0)) return;
    const double x = dot3(to_mean, si_d) / denom;
    t = (x < 0.0) ? 0.0 : (t_max < x) ? t_max : x;  // std::clamp
    const dv3 delta = sub3(add3(o, scale3(d, t)), mean);
    const double q = dot3(delta, matvec(ic, delta));
    response = opacity * exp(-0.5 * q);
}

__device__ __forceinline__ bool before(double ta, uint32_t ia, double tb, uint32_t ib) {
    return ta != tb ? ta < tb : ia < ib;  // trace.cpp:66-68
}

__device__ __forceinline__ int upper_seg(const DevSegment* segs, int n, uint64_t i) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (segs[mid].begin <= i) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ double wrap_pi(double x) {  // into (-pi, pi]
    constexpr double kTwoPi = 6.283185307179586;
    while (x > 3.141592653589793) x -= kTwoPi;
    while (x <= -3.141592653589793) x += kTwoPi;
    return x;
}
}  // namespace

// ---- pose + ray rectangle ----------------------------------------------------------------------
__global__ void __launch_bounds__(256) lidar_pose_kernel(LidarArgs a) {
    const DevField f = a.field;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < f.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const DevSegment& seg = a.segs[upper_seg(a.segs, a.n_segs, i)];
        const bool seen = seg.entry_count != 0;  // painted node visible to the sensor
        const dq nq{seg.q[0], seg.q[1], seg.q[2], seg.q[3]};
        const dv3 nt = mk3(seg.t[0], seg.t[1], seg.t[2]);
        // pose_primitive, trace.cpp:14-36
        const dv3 mean = add3(qrotate(nq, mk3(f.mx[i], f.my[i], f.mz[i])), nt);
        const dm3 r = qmatrix(qmul(nq, dq{f.qw[i], f.qx[i], f.qy[i], f.qz[i]}));
        const dm3 rt = mtransposed(r);
        const double sx0 = f.sx[i], sy0 = f.sy[i], sz0 = f.sz[i];
        const double sx = (sx0 < kTraceScaleFloor) ? kTraceScaleFloor : sx0;  // std::max
        const double sy = (sy0 < kTraceScaleFloor) ? kTraceScaleFloor : sy0;
        const double sz = (sz0 < kTraceScaleFloor) ? kTraceScaleFloor : sz0;
        const dm3 di{{1.0 / (sx * sx), 0, 0, 0, 1.0 / (sy * sy), 0, 0, 0, 1.0 / (sz * sz)}};
        const dm3 inv_cov = mmul(mmul(r, di), rt);
        const dm3 d{{sx0 * sx0, 0, 0, 0, sy0 * sy0, 0, 0, 0, sz0 * sz0}};
        const dm3 cov = mmul(mmul(r, d), rt);
        const double hx = kBoundsSigmaL * sqrt(cov.m[0]), hy = kBoundsSigmaL * sqrt(cov.m[4]),
                     hz = kBoundsSigmaL * sqrt(cov.m[8]);
        const dv3 pa = mk3(mean.x - hx, mean.y - hy, mean.z - hz);
        const dv3 pb = mk3(mean.x + hx, mean.y + hy, mean.z + hz);
        const dv3 lo = mk3(fmin(fmin(INFINITY, pa.x), pb.x), fmin(fmin(INFINITY, pa.y), pb.y),
                           fmin(fmin(INFINITY, pa.z), pb.z));
        const dv3 hi = mk3(fmax(fmax(-INFINITY, pa.x), pb.x), fmax(fmax(-INFINITY, pa.y), pb.y),
                           fmax(fmax(-INFINITY, pa.z), pb.z));
        const uint64_t n = f.n;
        double* P = a.posed;
        P[i] = mean.x; P[n + i] = mean.y; P[2 * n + i] = mean.z;
#pragma unroll
        for (int k = 0; k < 9; ++k) P[(3 + k) * n + i] = inv_cov.m[k];
        P[12 * n + i] = f.opacity[i];
        P[13 * n + i] = lo.x; P[14 * n + i] = lo.y; P[15 * n + i] = lo.z;
        P[16 * n + i] = hi.x; P[17 * n + i] = hi.y; P[18 * n + i] = hi.z;
        a.seen[i] = seen ? 1 : 0;
        {
            double2* R = reinterpret_cast<double2*>(a.trace_rec + 20 * uint64_t(i));
            R[0] = make_double2(lo.x, lo.y);
            R[1] = make_double2(lo.z, hi.x);
            R[2] = make_double2(hi.y, hi.z);
            R[3] = make_double2(f.opacity[i], seen ? 1.0 : 0.0);
            R[4] = make_double2(mean.x, mean.y);
            R[5] = make_double2(mean.z, inv_cov.m[0]);
            R[6] = make_double2(inv_cov.m[1], inv_cov.m[2]);
            R[7] = make_double2(inv_cov.m[3], inv_cov.m[4]);
            R[8] = make_double2(inv_cov.m[5], inv_cov.m[6]);
            R[9] = make_double2(inv_cov.m[7], inv_cov.m[8]);
        }
        if (!a.scan) continue;

        // Conservative ray rectangle: the box in the sensor frame (AABB of its 8 corners)
        // subtends an azimuth arc and an elevation band from the origin.
        LidarRect rc{0, 0, 0, 0, kRectNone};
        if (seen && lo.x <= hi.x && lo.y <= hi.y && lo.z <= hi.z) {
            const dq wq{a.w2s_q[0], a.w2s_q[1], a.w2s_q[2], a.w2s_q[3]};
            const dv3 wt = mk3(a.w2s_t[0], a.w2s_t[1], a.w2s_t[2]);
            dv3 slo = mk3(INFINITY, INFINITY, INFINITY), shi = mk3(-INFINITY, -INFINITY, -INFINITY);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const dv3 p = add3(qrotate(wq, mk3(c & 1 ? hi.x : lo.x, c & 2 ? hi.y : lo.y,
                                                    c & 4 ? hi.z : lo.z)), wt);
                slo = mk3(fmin(slo.x, p.x), fmin(slo.y, p.y), fmin(slo.z, p.z));
                shi = mk3(fmax(shi.x, p.x), fmax(shi.y, p.y), fmax(shi.z, p.z));
            }
            // widen by a relative margin so rounding of the corner transform can never shrink it
            const double m = 1e-9 * (fabs(slo.x) + fabs(slo.y) + fabs(slo.z) + fabs(shi.x) +
                                     fabs(shi.y) + fabs(shi.z)) + 1e-12;
            slo = mk3(slo.x - m, slo.y - m, slo.z - m);
            shi = mk3(shi.x + m, shi.y + m, shi.z + m);
            const double nx = fmax(fmax(slo.x, -shi.x), 0.0), ny = fmax(fmax(slo.y, -shi.y), 0.0),
                         nz = fmax(fmax(slo.z, -shi.z), 0.0);
            if (sqrt(nx * nx + ny * ny + nz * nz) > a.max_range * (1.0 + 1e-12)) {
                // beyond reach of every ray
            } else if (nx == 0.0 && ny == 0.0 && nz == 0.0) {
                rc.kind = kRectAll;  // the sensor sits in the box
            } else {
                const double dxy_min = sqrt(nx * nx + ny * ny);
                double dxy_max = 0.0, a_lo, a_hi;
                for (int c = 0; c < 4; ++c) {
                    const double x = c & 1 ? shi.x : slo.x, y = c & 2 ? shi.y : slo.y;
                    dxy_max = fmax(dxy_max, sqrt(x * x + y * y));
                }
                if (dxy_min == 0.0) {
                    a_lo = 0.0;  // the xy rectangle surrounds the axis: every azimuth
                    a_hi = a.two_pi;
                } else {
                    const double a0 = atan2(0.5 * (slo.y + shi.y), 0.5 * (slo.x + shi.x));
                    double dmin = 0.0, dmax = 0.0;
                    for (int c = 0; c < 4; ++c) {
                        const double x = c & 1 ? shi.x : slo.x, y = c & 2 ? shi.y : slo.y;
                        const double dd = wrap_pi(atan2(y, x) - a0);
                        dmin = fmin(dmin, dd);
                        dmax = fmax(dmax, dd);
                    }
                    a_lo = a0 + dmin - kAngleMargin;
                    a_hi = a0 + dmax + kAngleMargin;
                }
                const double e_hi = atan2(shi.z, shi.z > 0.0 ? dxy_min : dxy_max) + kAngleMargin;
                const double e_lo = atan2(slo.z, slo.z < 0.0 ? dxy_min : dxy_max) - kAngleMargin;
                // channel ranks with elevation in [e_lo, e_hi] (sorted regular channels)
                int r0 = 0, r1 = a.n_ranks - 1;
                while (r0 < a.n_ranks && a.rank_elev[r0] < e_lo) ++r0;
                while (r1 >= 0 && a.rank_elev[r1] > e_hi) --r1;
                // azimuth steps k with k * step in [a_lo, a_hi] (mod 2 pi)
                const int64_t k0 = int64_t(ceil(a_lo / a.step)), k1 = int64_t(floor(a_hi / a.step));
                if (r0 <= r1 && k0 <= k1) {
                    rc.r0 = uint16_t(r0);
                    rc.r1 = uint16_t(r1);
                    if (k1 - k0 + 1 >= int64_t(a.n_az)) {
                        rc.k0 = 0;
                        rc.k1 = a.n_az - 1;
                    } else {
                        rc.k0 = uint32_t(((k0 % int64_t(a.n_az)) + a.n_az) % a.n_az);
                        rc.k1 = uint32_t(((k1 % int64_t(a.n_az)) + a.n_az) % a.n_az);
                    }
                    rc.kind = kRectRange;
                }
            }
        }
        a.rects[i] = rc;
        if (rc.kind == kRectAll) a.all_list[atomicAdd(a.all_count, 1u)] = uint32_t(i);
    }
}

// Rays of a rectangle row: [k0, k1] or, wrapped, [k0, n_az) + [0, k1].
template <class F>
__device__ __forceinline__ void for_row_ranges(const LidarRect& rc, uint32_t n_az, F&& fn) {
    if (rc.k0 <= rc.k1) {
        fn(rc.k0, rc.k1);
    } else {
        fn(rc.k0, n_az - 1);
        fn(0u, rc.k1);
    }
}

__global__ void __launch_bounds__(256) lidar_count_kernel(LidarArgs a) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < a.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const LidarRect rc = a.rects[i];
        if (rc.kind != kRectRange) continue;
        for (uint32_t r = rc.r0; r <= rc.r1; ++r) {
            int* row = a.diff + uint64_t(a.rank_channel[r]) * (a.n_az + 1);
            for_row_ranges(rc, a.n_az, [&](uint32_t k0, uint32_t k1) {
                atomicAdd(row + k0, 1);
                atomicAdd(row + k1 + 1, -1);
            });
        }
    }
}

// One block per channel row: prefix of the row differences -> candidates per ray.
__global__ void __launch_bounds__(256) lidar_rowscan_kernel(LidarArgs a) {
    __shared__ int s_warp[8];
    __shared__ int s_carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int* row = a.diff + uint64_t(blockIdx.x) * (a.n_az + 1);
    uint32_t* cnt = a.ray_count + uint64_t(blockIdx.x) * a.n_az;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t k0 = 0; k0 < a.n_az; k0 += blockDim.x) {
        const uint32_t k = k0 + threadIdx.x;
        int v = k < a.n_az ? row[k] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane == 31) s_warp[warp] = v;
        __syncthreads();
        int pre = s_carry;
        for (int w = 0; w < warp; ++w) pre += s_warp[w];
        if (k < a.n_az) cnt[k] = uint32_t(v + pre);
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < int(blockDim.x >> 5); ++w) t += s_warp[w];
            s_carry += t;
        }
        __syncthreads();
    }
}

// Rays of a rectangle (both wrapped parts), enumerated by one thread.
__device__ __forceinline__ uint32_t rect_rays(const LidarRect& rc, uint32_t n_az) {
    const uint32_t w = rc.k0 <= rc.k1 ? rc.k1 - rc.k0 + 1 : (n_az - rc.k0) + rc.k1 + 1;
    return (uint32_t(rc.r1) - rc.r0 + 1) * w;
}

// Ray id of position p (row-major over the rectangle) of a rectangle.
__device__ __forceinline__ uint64_t rect_ray(const LidarArgs& a, const LidarRect& rc, uint32_t p) {
    const uint32_t w = rc.k0 <= rc.k1 ? rc.k1 - rc.k0 + 1 : (a.n_az - rc.k0) + rc.k1 + 1;
    const uint32_t r = rc.r0 + p / w;
    uint32_t k = rc.k0 + p % w;
    if (k >= a.n_az) k -= a.n_az;
    return uint64_t(a.rank_channel[r]) * a.n_az + k;
}

// Order within a ray's list is free (the tracer orders by (t, index)): every candidate takes
// its slot with one atomic on the ray's cursor. Small rectangles are walked by their thread;
// big ones (primitives close to the sensor cover thousands of rays) are queued and spread over
// whole warps by lidar_scatter_big_kernel, so no thread serialises thousands of atomics.
constexpr uint32_t kSmallRect = 64;

__global__ void __launch_bounds__(256) lidar_scatter_kernel(LidarArgs a) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < a.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const LidarRect rc = a.rects[i];
        if (rc.kind != kRectRange) continue;
        const uint32_t m = rect_rays(rc, a.n_az);
        if (m > kSmallRect) {
            a.big_list[atomicAdd(a.big_count, 1u)] = uint32_t(i);
            continue;
        }
        for (uint32_t p = 0; p < m; ++p) {
            const uint64_t ray = rect_ray(a, rc, p);
            a.list[a.ray_offset[ray] + atomicAdd(a.cursor + ray, 1u)] = uint32_t(i);
        }
    }
}

__global__ void __launch_bounds__(256) lidar_scatter_big_kernel(LidarArgs a) {
    const int lane = threadIdx.x & 31;
    const uint32_t n_big = *a.big_count;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_big;
         w += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t i = a.big_list[w];
        const LidarRect rc = a.rects[i];
        const uint32_t m = rect_rays(rc, a.n_az);
        for (uint32_t p = lane; p < m; p += 32) {
            const uint64_t ray = rect_ray(a, rc, p);
            a.list[a.ray_offset[ray] + atomicAdd(a.cursor + ray, 1u)] = i;
        }
    }
}

// ---- per-ray trace ----------------------------------------------------------------------------
namespace {
struct RayCands {
    const uint32_t* list;  // explicit candidates (nullptr: every primitive)
    uint32_t n_list;
    const uint32_t* extra;  // appended candidates (boxes around the sensor)
    uint32_t n_extra;
    __device__ __forceinline__ uint32_t count(uint64_t n_prims) const {
        return list ? n_list + n_extra : uint32_t(n_prims);
    }
    __device__ __forceinline__ uint32_t at(uint32_t j) const {
        return list ? (j < n_list ? list[j] : extra[j - n_list]) : j;
    }
};

// Candidate j of the ray as (t, response) if its box is hit and alpha >= 1/255 (else false).
__device__ __forceinline__ bool survivor(const LidarArgs& a, uint32_t i, dv3 o, dv3 d, dv3 inv,
                                         double t_max, double& t, double& resp) {
    // the primitive's 160-byte trace row: box first, the rest only for a box hit
    const double2* R = reinterpret_cast<const double2*>(a.trace_rec + 20 * uint64_t(i));
    const double2 r0 = __ldg(R), r1 = __ldg(R + 1), r2 = __ldg(R + 2), r3 = __ldg(R + 3);
    if (!(r3.y != 0.0)) return false;  // not seen
    const dv3 lo = mk3(r0.x, r0.y, r1.x);
    const dv3 hi = mk3(r1.y, r2.x, r2.y);
    if (!ray_aabb_hit(lo, hi, o, inv, t_max)) return false;
    ray_peak_row(R, r3.x, o, d, t_max, t, resp);
    // alpha = min(response, 0.99) is skipped below 1/255 (trace.cpp:73): composite-neutral
    return !(resp < kTraceAlphaSkip);
}
}  // namespace

// One warp per ray, composite in (t, index) order (trace.cpp:65-85) from a per-warp pool of
// at most kPool survivors (box hit, response >= 1/255) in shared memory, picked by warp arg-min.
//
// Scan rays (binned candidate lists): pass A computes every candidate's (t, response) once and
// stores it coalesced in the ray's scratch region (t = +inf marks a non-survivor). The rest
// works on that cache: the survivors after the last composited one are counted (with their t
// range); if more than the pool holds, a 64-bin histogram of t picks a window [lo, tau] that fits;
// the window is pooled and composited; the ray stops at the cutoff or moves to the next window.
// Rays that take every primitive (arbitrary rays, near-pole channels) recompute instead of
// caching, and re-scan per composite step when their survivors overflow the pool.
constexpr int kPool = 256;
constexpr int kTraceWarps = 8;
constexpr int kBins = 64;

namespace {
struct Composite {
    double depth_sum = 0.0, acc = 0.0, T = 1.0;
    double last_t = -INFINITY;
    uint32_t last_i = 0;
    bool first = true, done = false;
    __device__ __forceinline__ bool after(double t, uint32_t i) const {
        return first || before(last_t, last_i, t, i);
    }
    __device__ __forceinline__ void add(double t, double resp, uint32_t i) {
        const double alpha = resp < kTraceAlphaClamp ? resp : kTraceAlphaClamp;  // std::min
        const double w = alpha * T;
        depth_sum += t * w;
        acc += w;
        T *= 1.0 - alpha;
        last_t = t;
        last_i = i;
        first = false;
        if (T < kTraceCutoff) done = true;
    }
};

// Warp arg-min of (t, index) among the lanes' candidates.
__device__ __forceinline__ bool warp_argmin(double& bt, double& br, uint32_t& bi, bool have) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
        const double orr = __shfl_xor_sync(0xffffffffu, br, off);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
        const bool oh = __shfl_xor_sync(0xffffffffu, have, off);
        if (oh && (!have || before(ot, oi, bt, bi))) {
            bt = ot; br = orr; bi = oi; have = true;
        }
    }
    return have;
}

// Composite the pool (ns entries) in order until exhausted or saturated.
__device__ __forceinline__ void composite_pool(Composite& c, const double* pt, const double* pr,
                                               const uint32_t* pi, uint32_t ns) {
    const int lane = threadIdx.x & 31;
    while (!c.done) {
        double bt = INFINITY, br = 0.0;
        uint32_t bi = 0xFFFFFFFFu;
        bool have = false;
        for (uint32_t q = lane; q < ns; q += 32) {
            const double t = pt[q];
            const uint32_t i = pi[q];
            if (c.after(t, i) && (!have || before(t, i, bt, bi))) {
                bt = t; br = pr[q]; bi = i; have = true;
            }
        }
        if (!warp_argmin(bt, br, bi, have)) break;
        c.add(bt, br, bi);
    }
}
}  // namespace

__global__ void __launch_bounds__(32 * kTraceWarps) lidar_trace_kernel(LidarArgs a) {
    __shared__ double s_t[kTraceWarps][kPool];
    __shared__ double s_r[kTraceWarps][kPool];
    __shared__ uint32_t s_i[kTraceWarps][kPool];
    __shared__ uint32_t s_hist[kTraceWarps][kBins];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    double* pt = s_t[wib];
    double* pr = s_r[wib];
    uint32_t* pi = s_i[wib];
    uint32_t* hist = s_hist[wib];
    for (uint64_t ray = warp; ray < a.n_rays; ray += n_warps) {
        const dv3 o = a.scan ? mk3(a.origin[0], a.origin[1], a.origin[2]) : ldx3(a.ray_origin, ray);
        const dv3 d = ldx3(a.ray_dir, ray);
        const double t_max = a.scan ? a.max_range : a.ray_tmax[ray];
        const dv3 inv = mk3(1.0 / d.x, 1.0 / d.y, 1.0 / d.z);
        RayCands cs{};
        const bool brute = a.scan ? a.ray_all[ray / a.n_az] != 0 : a.ray_lists == 0;
        if (!brute) {
            // lists at ray_offset (exact sizes) or, single-pass BVH lists, at ray * list_stride
            const uint64_t b = a.list_stride ? ray * uint64_t(a.list_stride) : a.ray_offset[ray];
            cs.list = a.list + b;
            cs.n_list = a.list_stride ? a.list_count[ray] : uint32_t(a.ray_offset[ray + 1] - b);
            cs.extra = a.all_list;
            cs.n_extra = *a.all_count;
        }
        const uint32_t nc = cs.count(a.n);
        Composite c;
        if (!brute) {
            // pass A: (t, response) of every candidate, cached (t = inf: not a survivor)
            const uint64_t base = (a.list_stride ? ray * uint64_t(a.list_stride) : a.ray_offset[ray]) +
                                  ray * uint64_t(cs.n_extra);
            double* ct = a.cand_t + base;
            double* cr = a.cand_r + base;
            for (uint32_t j = lane; j < nc; j += 32) {
                double t = 0.0, resp = 0.0;
                const bool keep = survivor(a, cs.at(j), o, d, inv, t_max, t, resp);
                ct[j] = keep ? t : INFINITY;
                cr[j] = resp;
            }
            __syncwarp();
            // windows of at most kPool survivors, in t order
            double lo = -INFINITY;  // survivors with t > lo remain (all of t <= lo were pooled)
            while (!c.done) {
                uint32_t cnt = 0;
                double tmin = INFINITY, tmax = -INFINITY;
                for (uint32_t j = lane; j < nc; j += 32) {
                    const double t = ct[j];
                    if (t != INFINITY && t > lo) {
                        ++cnt;
                        tmin = fmin(tmin, t);
                        tmax = fmax(tmax, t);
                    }
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
                    tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, off));
                    tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
                }
                if (cnt == 0) break;
                if (cnt > uint32_t(kPool)) {
                    // 64-bin histogram of t over [tmin, tmax]; tau = upper edge of the last bin
                    // whose prefix fits the pool (bin 0 alone too big: selection on the cache)
                    for (int b = lane; b < kBins; b += 32) hist[b] = 0;
                    __syncwarp();
                    const double scale = double(kBins) / (tmax - tmin);
                    for (uint32_t j = lane; j < nc; j += 32) {
                        const double t = ct[j];
                        if (t != INFINITY && t > lo) {
                            int b = int((t - tmin) * scale);
                            b = b < 0 ? 0 : (b >= kBins ? kBins - 1 : b);
                            atomicAdd(&hist[b], 1u);
                        }
                    }
                    __syncwarp();
                    uint32_t run = 0;
                    int last_fit = -1;
                    for (int b = 0; b < kBins; ++b) {
                        run += hist[b];
                        if (run <= uint32_t(kPool)) last_fit = b;
                    }
                    __syncwarp();
                    if (last_fit < 0) {
                        // a tie cluster: pick survivors one by one straight from the cache
                        while (!c.done) {
                            double bt = INFINITY, br = 0.0;
                            uint32_t bi = 0xFFFFFFFFu;
                            bool have = false;
                            for (uint32_t j = lane; j < nc; j += 32) {
                                const double t = ct[j];
                                if (t == INFINITY || !(t > lo)) continue;
                                const uint32_t i = cs.at(j);
                                if (c.after(t, i) && (!have || before(t, i, bt, bi))) {
                                    bt = t; br = cr[j]; bi = i; have = true;
                                }
                            }
                            if (!warp_argmin(bt, br, bi, have)) break;
                            c.add(bt, br, bi);
                        }
                        break;
                    }
                    // a survivor is in the window iff its bin index (the same rounding as the
                    // histogram) is <= last_fit
                    uint32_t ns = 0;
                    double wmax = -INFINITY;
                    for (uint32_t j0 = 0; j0 < nc; j0 += 32) {
                        const uint32_t j = j0 + lane;
                        bool in = false;
                        double t = INFINITY;
                        if (j < nc) {
                            t = ct[j];
                            if (t != INFINITY && t > lo) {
                                int b = int((t - tmin) * scale);
                                b = b < 0 ? 0 : (b >= kBins ? kBins - 1 : b);
                                in = b <= last_fit;
                            }
                        }
                        const uint32_t bits = __ballot_sync(0xffffffffu, in);
                        if (in) {
                            const uint32_t slot = ns + __popc(bits & lanemask_lt());
                            pt[slot] = t;
                            pr[slot] = cr[j];
                            pi[slot] = cs.at(j);
                            wmax = fmax(wmax, t);
                        }
                        ns += __popc(bits);
                    }
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1)
                        wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
                    __syncwarp();
                    composite_pool(c, pt, pr, pi, ns);
                    __syncwarp();
                    // every survivor with t <= wmax was in the window (bins are monotone in t)
                    lo = wmax;
                    continue;
                }
                // everything left fits the pool
                uint32_t ns = 0;
                for (uint32_t j0 = 0; j0 < nc; j0 += 32) {
                    const uint32_t j = j0 + lane;
                    const double t = j < nc ? ct[j] : INFINITY;
                    const bool in = t != INFINITY && t > lo;
                    const uint32_t bits = __ballot_sync(0xffffffffu, in);
                    if (in) {
                        const uint32_t slot = ns + __popc(bits & lanemask_lt());
                        pt[slot] = t;
                        pr[slot] = cr[j];
                        pi[slot] = cs.at(j);
                    }
                    ns += __popc(bits);
                }
                __syncwarp();
                composite_pool(c, pt, pr, pi, ns);
                __syncwarp();
                break;
            }
        } else {
            // every primitive is a candidate: pool the survivors, or re-scan per step on overflow
            uint32_t ns = 0;
            bool overflow = false;
            for (uint32_t j0 = 0; j0 < nc; j0 += 32) {
                const uint32_t j = j0 + lane;
                double t = 0.0, resp = 0.0;
                uint32_t i = 0;
                bool keep = false;
                if (j < nc) {
                    i = cs.at(j);
                    keep = survivor(a, i, o, d, inv, t_max, t, resp);
                }
                const uint32_t bits = __ballot_sync(0xffffffffu, keep);
                if (ns + __popc(bits) > uint32_t(kPool)) {
                    overflow = true;
                    break;
                }
                if (keep) {
                    const uint32_t slot = ns + __popc(bits & lanemask_lt());
                    pt[slot] = t;
                    pr[slot] = resp;
                    pi[slot] = i;
                }
                ns += __popc(bits);
            }
            __syncwarp();
            if (!overflow) {
                composite_pool(c, pt, pr, pi, ns);
            } else {
                while (!c.done) {
                    double bt = INFINITY, br = 0.0;
                    uint32_t bi = 0xFFFFFFFFu;
                    bool have = false;
                    for (uint32_t j = lane; j < nc; j += 32) {
                        double t, resp;
                        const uint32_t i = cs.at(j);
                        if (survivor(a, i, o, d, inv, t_max, t, resp) && c.after(t, i) &&
                            (!have || before(t, i, bt, bi))) {
                            bt = t; br = resp; bi = i; have = true;
                        }
                    }
                    if (!warp_argmin(bt, br, bi, have)) break;
                    c.add(bt, br, bi);
                }
            }
            __syncwarp();
        }
        if (a.debug && lane == 0) {
            atomicAdd(a.debug, 1ull);
            atomicAdd(a.debug + 1, (unsigned long long)nc);
        }
        if (lane == 0) {
            const bool hit = c.acc >= a.alpha_threshold;
            a.out_hit[ray] = hit ? 1u : 0u;
            a.out_depth[ray] = hit ? c.depth_sum / c.acc : 0.0;
            a.out_acc[ray] = c.acc;
        }
        __syncwarp();  // the pool is reused by the warp's next ray
    }
}

// Returns in ray order (channel-major, azimuth ascending): point = dir_sensor * depth.
__global__ void __launch_bounds__(256) lidar_emit_kernel(LidarArgs a) {
    for (uint64_t ray = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; ray < a.n_rays;
         ray += uint64_t(gridDim.x) * blockDim.x) {
        if (!a.out_hit[ray]) continue;
        const uint64_t p = a.hit_offset[ray];  // exclusive prefix of the hit flags
        if (p >= a.capacity) continue;
        const double depth = a.out_depth[ray];
        const dv3 ds = ldx3(a.ray_dir_sensor, ray);
        const dv3 pt = scale3(ds, depth);
        a.points[3 * p] = pt.x;
        a.points[3 * p + 1] = pt.y;
        a.points[3 * p + 2] = pt.z;
        a.ring[p] = uint32_t(ray / a.n_az);
        a.azimuth[p] = double(ray % a.n_az) * a.step;
    }
}

// ---- device-wide exclusive scan of u32 counts into u64 offsets (n + 1 entries) --------------------
__global__ void __launch_bounds__(1024) scan_blocks_kernel(const uint32_t* in, uint64_t n,
                                                          unsigned long long* out,
                                                          unsigned long long* block_sums) {
    __shared__ unsigned long long s[1024];
    const uint64_t i = blockIdx.x * 1024ull + threadIdx.x;
    const unsigned long long v = i < n ? in[i] : 0ull;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const unsigned long long t = threadIdx.x >= o ? s[threadIdx.x - o] : 0ull;
        __syncthreads();
        s[threadIdx.x] += t;
        __syncthreads();
    }
    if (i < n) out[i] = s[threadIdx.x] - v;
    if (threadIdx.x == 1023) block_sums[blockIdx.x] = s[1023];
}

__global__ void __launch_bounds__(1024) scan_sums_kernel(unsigned long long* block_sums, uint64_t n_blocks,
                                                         unsigned long long* total) {
    __shared__ unsigned long long s[1024];
    __shared__ unsigned long long s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < n_blocks; b0 += 1024) {
        const uint64_t b = b0 + threadIdx.x;
        const unsigned long long v = b < n_blocks ? block_sums[b] : 0ull;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const unsigned long long t = threadIdx.x >= o ? s[threadIdx.x - o] : 0ull;
            __syncthreads();
            s[threadIdx.x] += t;
            __syncthreads();
        }
        if (b < n_blocks) block_sums[b] = s_carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += s[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = s_carry;
}

__global__ void scan_add_kernel(unsigned long long* out, uint64_t n, const unsigned long long* block_sums,
                                const unsigned long long* total) {
    const uint64_t i = blockIdx.x * 1024ull + threadIdx.x;
    if (i < n) out[i] += block_sums[blockIdx.x];
    if (i == 0) out[n] = *total;
}

void exclusive_scan_u32(const uint32_t* in, uint64_t n, unsigned long long* out,
                        unsigned long long* scratch, cudaStream_t s) {
    // out[0..n] = exclusive prefix (out[n] = total); scratch: ceil(n / 1024) + 1 entries
    const uint64_t blocks = std::max<uint64_t>(1, (n + 1023) / 1024);
    scan_blocks_kernel<<<unsigned(blocks), 1024, 0, s>>>(in, n, out, scratch);
    scan_sums_kernel<<<1, 1024, 0, s>>>(scratch, blocks, scratch + blocks);
    scan_add_kernel<<<unsigned(blocks), 1024, 0, s>>>(out, n, scratch, scratch + blocks);
}

// World ray directions: the sensor rotation applied to the sensor-frame directions (Quat::rotate,
// math.hpp:139-143, the reference's double operation order).
__global__ void lidar_rays_kernel(const double* ds, double* dw, uint64_t n, double q0, double q1,
                                  double q2, double q3) {
    const dq q{q0, q1, q2, q3};
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const dv3 w = qrotate(q, ldx3(ds, k));
        dw[3 * k] = w.x;
        dw[3 * k + 1] = w.y;
        dw[3 * k + 2] = w.z;
    }
}

// ---- launchers -------------------------------------------------------------------------------------
void launch_lidar_rays(const double* ds, double* dw, uint64_t n, const double* q, int n_sms,
                       cudaStream_t s) {
    if (!n) return;
    const uint64_t want = (n + 255) / 256;
    lidar_rays_kernel<<<unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(n_sms) * 8))),
                        256, 0, s>>>(ds, dw, n, q[0], q[1], q[2], q[3]);
}
void launch_lidar_pose(const LidarArgs& a, int n_sms, cudaStream_t s) {
    const uint64_t want = (a.n + 255) / 256;
    lidar_pose_kernel<<<unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(n_sms) * 8))),
                        256, 0, s>>>(a);
}
void launch_lidar_count(const LidarArgs& a, int n_sms, cudaStream_t s) {
    const uint64_t want = (a.n + 255) / 256;
    lidar_count_kernel<<<unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(n_sms) * 8))),
                         256, 0, s>>>(a);
}
void launch_lidar_rowscan(const LidarArgs& a, uint32_t n_channels, cudaStream_t s) {
    if (n_channels) lidar_rowscan_kernel<<<n_channels, 256, 0, s>>>(a);
}
void launch_lidar_scatter(const LidarArgs& a, int n_sms, cudaStream_t s) {
    const uint64_t want = (a.n + 255) / 256;
    lidar_scatter_kernel<<<unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(n_sms) * 8))),
                           256, 0, s>>>(a);
}
void launch_lidar_scatter_big(const LidarArgs& a, int n_sms, cudaStream_t s) {
    lidar_scatter_big_kernel<<<unsigned(n_sms) * 8, 256, 0, s>>>(a);
}
void launch_lidar_trace(const LidarArgs& a, int n_sms, cudaStream_t s) {
    if (!a.n_rays) return;
    const uint64_t want = (a.n_rays * 32 + 255) / 256;
    lidar_trace_kernel<<<unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(n_sms) * 16))),
                         32 * kTraceWarps, 0, s>>>(a);
}
void launch_lidar_emit(const LidarArgs& a, int n_sms, cudaStream_t s) {
    if (!a.n_rays) return;
    const uint64_t want = (a.n_rays + 255) / 256;
    lidar_emit_kernel<<<unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(n_sms) * 8))),
                        256, 0, s>>>(a);
}

}  // namespace gsim_gpu
