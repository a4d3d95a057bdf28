// common.cuh — device-side data layout and the reference's double-precision math.
//
// The geometry half of the preprocess (K2) reproduces /root/reference/proj/core/include/gsim/
// math.hpp and raster.cpp:66-163 operation by operation in double precision. Files that
// include the *_exact helpers are compiled with -fmad=false so no multiply-add is contracted,
// which keeps culls, tile rects and depth keys bit-identical to the reference's x86-64 build.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace gsim_gpu {

constexpr int kTileSize = 16;                // raster.hpp:38
constexpr double kCovarianceFloor = 0.3;     // raster.hpp:39
constexpr double kAlphaClamp = 0.99;         // raster.hpp:40
constexpr double kAlphaSkip = 1.0 / 255.0;   // raster.hpp:41
constexpr uint32_t kInvalidKey = 0xFFFFFFFFu;
constexpr int kMaxTilesPerAxis = 256;        // tile rect packed as 4 x u8 in a record

// ---- HBM layout --------------------------------------------------------------------------

// Device-resident GaussianField (gaussian.hpp:53-60): SoA double geometry planes (coalesced
// 8-byte loads per thread, exact reference inputs) and SH as float4 planes [plane][n]:
// plane p holds coefficients 4p..4p+3 of the channel-major list sh[c*K + k], K = (d+1)^2.
struct DevField {
    uint64_t n;
    int sh_degree;
    int sh_planes;          // ceil(3K / 4)
    double* mx; double* my; double* mz;
    double* sx; double* sy; double* sz;
    double* qw; double* qx; double* qy; double* qz;
    double* opacity;
    float4* sh;             // sh_planes * n
};

// One camera of a batch, with everything the reference recomputes per call precomputed on the
// host in the reference's own operation order (raster.cpp:72-77, camera.hpp:23).
struct DevCamera {
    double r[9];            // camera.pose.rotation.to_matrix(), row-major
    double q[4];            // world->camera rotation (w, x, y, z)
    double t[3];            // world->camera translation
    double center[3];       // camera_center()
    double fx, fy, cx, cy, near_p, far_p, limx, limy;
    int width, height, tiles_x, tiles_y;
    uint32_t tile_base;     // first global tile id of this camera
    uint32_t reserved;
    uint64_t slot_base;     // first record slot of this camera
    uint64_t out_offset;    // float offset of this camera's [rgb|depth|alpha] block
};

// A maximal primitive range with one node pose ("painted" node table: the reference's
// PoseTable, raster.cpp:47-62, where later nodes overwrite earlier ones).
struct DevSegment {
    uint64_t begin, end;
    double q[4];
    double t[3];
    uint32_t entry_begin;   // cameras that see this segment, in SegEntry[]
    uint32_t entry_count;
};

// (segment, camera): records of primitive i of the segment live at slot_base + (i - begin).
struct SegEntry {
    uint32_t cam;
    uint32_t reserved;
    uint64_t slot_base;
};

// 48-byte splat record, one per (camera, primitive) slot, in the form K4 consumes it (it is
// copied global -> shared with three 16-byte cp.async and used as is):
struct alignas(16) Record {
    float4 a;  // u, v, radius, log2(alpha_peak)
    float4 b;  // conic prescaled for ex2: -inv_xx*log2(e)/2, -inv_xy*log2(e), -inv_yy*log2(e)/2,
               // view_depth
    float4 c;  // r, g, b, reach: half2 (ex, ey) rounded up = half-extents of the region where
               // the splat can pass the raster's box test AND reach alpha >= 1/255; -inf if
               // it can reach it nowhere
};

constexpr float kLog2eF = 1.4426950408889634f;

// Builds the raster record from the fp32 projection (u, v, depth, radius, inverse covariance,
// peak alpha, rgb). Record.b = (B, C, A, depth); the exponent of ex2 is then
// log2(o) + dx*(A*dx + B*dy) + C*dy*dy, i.e.
// log2(o * exp(-q/2)) with q = inv_xx dx^2 + 2 inv_xy dx dy + inv_yy dy^2 (raster.cpp:226-229).
__device__ inline Record make_record(float u, float v, float z, float rad, float ia, float ib,
                                     float ic, float op, float r, float g, float b) {
    Record rec;
    rec.a = make_float4(u, v, rad, __log2f(op));
    // (B, C) first: the blend scales them by dy as one aligned register pair (FMUL2)
    rec.b = make_float4(ib * -kLog2eF, ic * (-0.5f * kLog2eF), ia * (-0.5f * kLog2eF), z);
    // Reachable half-extents: the box test bounds |dx|,|dy| <= r; alpha >= 1/255 needs
    // q <= qc = 2 ln(255 o), whose ellipse has half-extents sqrt(qc * cov_xx/yy) (conservatively
    // widened), so no contributing splat is ever culled by them.
    float ex = rad, ey = rad;
    if (!(op * 255.0f >= 1.0f)) {
        ex = ey = -INFINITY;  // can never reach alpha 1/255
    } else {
        // approximate MUFU ops are fine here: the bound is widened by 1% + 0.05 px
        const float qc = 2.0f * __logf(op * 255.0f);
        const float det = ia * ic - ib * ib;
        if (det > 0.0f) {
            float inv, sx, sy;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(det));
            asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sx) : "f"(qc * ic * inv));
            asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sy) : "f"(qc * ia * inv));
            ex = fminf(ex, sx * 1.01f + 0.05f);
            ey = fminf(ey, sy * 1.01f + 0.05f);
        }
    }
    const __half2 reach = __halves2half2(__float2half_ru(ex), __float2half_ru(ey));
    rec.c = make_float4(r, g, b, *reinterpret_cast<const float*>(&reach));
    return rec;
}

__host__ __device__ inline uint32_t pack_rect(int tx0, int ty0, int tx1, int ty1) {
    return uint32_t(tx0) | (uint32_t(ty0) << 8) | (uint32_t(tx1) << 16) | (uint32_t(ty1) << 24);
}

// ---- math.hpp, double, reference operation order ----------------------------------------

struct dv3 { double x, y, z; };
struct dq { double w, x, y, z; };
struct dm3 { double m[9]; };

__host__ __device__ inline dv3 mk3(double x, double y, double z) { return dv3{x, y, z}; }
__host__ __device__ inline dv3 add3(dv3 a, dv3 b) { return mk3(a.x + b.x, a.y + b.y, a.z + b.z); }
__host__ __device__ inline dv3 sub3(dv3 a, dv3 b) { return mk3(a.x - b.x, a.y - b.y, a.z - b.z); }
__host__ __device__ inline dv3 scale3(dv3 a, double s) { return mk3(a.x * s, a.y * s, a.z * s); }
__host__ __device__ inline dv3 cross3(dv3 a, dv3 b) {  // math.hpp:34-36
    return mk3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__host__ __device__ inline dq qmul(dq a, dq o) {  // Hamilton, math.hpp:132-137
    return dq{a.w * o.w - a.x * o.x - a.y * o.y - a.z * o.z,
              a.w * o.x + a.x * o.w + a.y * o.z - a.z * o.y,
              a.w * o.y - a.x * o.z + a.y * o.w + a.z * o.x,
              a.w * o.z + a.x * o.y - a.y * o.x + a.z * o.w};
}
__host__ __device__ inline dv3 qrotate(dq q, dv3 v) {  // math.hpp:139-143
    const dv3 qv = mk3(q.x, q.y, q.z);
    const dv3 t = scale3(cross3(qv, v), 2.0);
    return add3(add3(v, scale3(t, q.w)), cross3(qv, t));
}
__host__ __device__ inline dm3 qmatrix(dq q) {  // math.hpp:146-155
    const double xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z;
    const double xy = q.x * q.y, xz = q.x * q.z, yz = q.y * q.z;
    const double wx = q.w * q.x, wy = q.w * q.y, wz = q.w * q.z;
    dm3 r;
    r.m[0] = 1 - 2 * (yy + zz); r.m[1] = 2 * (xy - wz);     r.m[2] = 2 * (xz + wy);
    r.m[3] = 2 * (xy + wz);     r.m[4] = 1 - 2 * (xx + zz); r.m[5] = 2 * (yz - wx);
    r.m[6] = 2 * (xz - wy);     r.m[7] = 2 * (yz + wx);     r.m[8] = 1 - 2 * (xx + yy);
    return r;
}
__host__ __device__ inline double qnorm(dq q) {
    return sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
}
__host__ __device__ inline dq qnormalized(dq q) {  // math.hpp:124-127
    const double n = qnorm(q);
    return n > 0.0 ? dq{q.w / n, q.x / n, q.y / n, q.z / n} : dq{1.0, 0.0, 0.0, 0.0};
}
// Mat3 product entry (r, c): row(r).dot(o.col(c)), math.hpp:91-97.
__host__ __device__ inline double mm_entry(const dm3& a, const dm3& b, int r, int c) {
    return a.m[r * 3 + 0] * b.m[0 * 3 + c] + a.m[r * 3 + 1] * b.m[1 * 3 + c] +
           a.m[r * 3 + 2] * b.m[2 * 3 + c];
}
__host__ __device__ inline dm3 mmul(const dm3& a, const dm3& b) {
    dm3 o;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) o.m[r * 3 + c] = mm_entry(a, b, r, c);
    return o;
}
__host__ __device__ inline dm3 mtransposed(const dm3& a) {
    dm3 t;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) t.m[r * 3 + c] = a.m[c * 3 + r];
    return t;
}
__host__ __device__ inline double clampd(double v, double lo, double hi) {  // std::clamp
    return (v < lo) ? lo : (hi < v) ? hi : v;
}

// ---- debug checks (libgsim_gpu_debug.so, build.py --debug) ---------------------------------
// compute-sanitizer is closed on the GPU pool this was developed on; the debug build instead
// bounds-checks every computed index of the race- and overflow-prone mechanisms (onesweep
// destinations and look-back, key histograms, binning cells and pair positions, raster list
// reads) and traps with the failing check's file and line.
#ifdef GSIM_DEBUG_CHECKS
#define GSIM_DCHECK(cond)                                                              \
    do {                                                                               \
        if (!(cond)) {                                                                 \
            printf("GSIM_DCHECK failed: %s at %s:%d\n", #cond, __FILE__, __LINE__);   \
            __trap();                                                                  \
        }                                                                              \
    } while (0)
#else
#define GSIM_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

// ---- small device helpers ----------------------------------------------------------------

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Lanes of `mask` holding the same low `bits` bits of v as this lane, from one ballot per bit.
// match.any.sync does the same in one instruction, but it issues at roughly one per ~40 SM
// cycles on sm_100 and stalls everything behind it (measured, profiles/); ballots are cheap.
__device__ __forceinline__ uint32_t peers_of_bits(uint32_t mask, uint32_t v, int bits) {
    uint32_t peers = mask;
    for (int b = 0; b < bits; ++b) {
        const uint32_t bit = (v >> b) & 1u;
        const uint32_t bal = __ballot_sync(mask, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled-lookback status word: [63:62] flag, [61:40] epoch, [39:0] count. A word whose
// epoch differs from the current pass is "not published yet", so the status array never
// needs clearing between passes.
constexpr uint64_t kFlagAggregate = 1ull;
constexpr uint64_t kFlagInclusive = 2ull;
constexpr uint32_t kEpochBits = 22;
constexpr uint32_t kEpochMask = (1u << kEpochBits) - 1;
__device__ __forceinline__ uint64_t make_status(uint64_t flag, uint32_t epoch, uint64_t count) {
    return (flag << 62) | (uint64_t(epoch & kEpochMask) << 40) | (count & ((1ull << 40) - 1));
}

// Binary search: largest i in [0, n) with arr[i] <= x (arr ascending, arr[0] <= x).
template <class T>
__device__ __forceinline__ int upper_index(const T* arr, int n, T x) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (arr[mid] <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
}

}  // namespace gsim_gpu
