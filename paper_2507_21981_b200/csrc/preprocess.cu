// preprocess.cu — K1 (scene-node pose) and K2 (projection + SH) kernels.
//
// Compiled with -fmad=false: the double-precision geometry below is the reference's
// raster.cpp:66-163 / gaussian.cpp:65-79 operation for operation (see common.cuh), so the
// visibility set, the 3-sigma tile rects and the float32 depth keys equal the reference's
// bit for bit. Shading (sh.cpp:10-51) runs in fp32; its outputs only feed the blend.
//
// K2 layout: one thread per primitive, grid-stride, looping over every camera that sees the
// primitive's node segment (the scene is read from HBM once per batch, not once per camera).
// Per (camera, primitive) slot it writes a 48-byte Record and a 32-bit depth key (kInvalidKey
// when culled or when the splat touches no tile), and accumulates the four 8-bit digit
// histograms of the keys for the onesweep depth sort.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "../../include/gsim_gpu.h"
#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {

// x86-64 cvttsd2si semantics of static_cast<int>(double) for out-of-range values
// ("integer indefinite" = INT_MIN), so absurd radii bin exactly like the reference build.
__device__ __forceinline__ int x86_trunc_int(double x) {
    if (!(x >= -2147483648.0 && x < 2147483648.0)) return INT32_MIN;
    return static_cast<int>(x);
}

__device__ __forceinline__ dq seg_q(const DevSegment& s) { return dq{s.q[0], s.q[1], s.q[2], s.q[3]}; }

// Correctly rounded x / b from a correctly rounded reciprocal rb = RN(1/b) (Markstein): the
// first quotient is within 1 ulp, one fma residual step rounds it exactly like IEEE division
// (no overflow/underflow in range; out-of-range numerators take the real division). Replaces
// eight double divisions per (camera, primitive) by two reciprocals and multiply-adds.
__device__ __forceinline__ double div_rn(double x, double b, double rb) {
    const double ax = fabs(x);
    if (!(ax < 0x1p900) || (ax < 0x1p-900 && x != 0.0)) return x / b;
    const double q0 = x * rb;
    const double r = fma(-q0, b, x);
    return fma(r, rb, q0);
}

constexpr float kSh0 = 0.28209479177387814f;  // sh.hpp:12-20
constexpr float kSh1 = 0.4886025119029199f;
constexpr float kSh2_0 = 1.0925484305920792f, kSh2_1 = -1.0925484305920792f,
                kSh2_2 = 0.31539156525252005f, kSh2_3 = -1.0925484305920792f,
                kSh2_4 = 0.5462742152960396f;
constexpr float kSh3_0 = -0.5900435899266435f, kSh3_1 = 2.890611442640554f,
                kSh3_2 = -0.4570457994644658f, kSh3_3 = 0.3731763325901154f,
                kSh3_4 = -0.4570457994644658f, kSh3_5 = 1.445305721320277f,
                kSh3_6 = -0.5900435899266435f;

template <int DEG>
__device__ __forceinline__ void sh_basis(float x, float y, float z, float* basis) {
    basis[0] = kSh0;
    if (DEG >= 1) {
        basis[1] = -kSh1 * y;
        basis[2] = kSh1 * z;
        basis[3] = -kSh1 * x;
    }
    if (DEG >= 2) {
        const float xx = x * x, yy = y * y, zz = z * z;
        basis[4] = kSh2_0 * x * y;
        basis[5] = kSh2_1 * y * z;
        basis[6] = kSh2_2 * (2.0f * zz - xx - yy);
        basis[7] = kSh2_3 * x * z;
        basis[8] = kSh2_4 * (xx - yy);
    }
    if (DEG >= 3) {
        const float xx = x * x, yy = y * y, zz = z * z;
        basis[9] = kSh3_0 * y * (3.0f * xx - yy);
        basis[10] = kSh3_1 * x * y * z;
        basis[11] = kSh3_2 * y * (4.0f * zz - xx - yy);
        basis[12] = kSh3_3 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
        basis[13] = kSh3_4 * x * (4.0f * zz - xx - yy);
        basis[14] = kSh3_5 * z * (xx - yy);
        basis[15] = kSh3_6 * x * (xx - 3.0f * yy);
    }
}

// rgb_c = max(0, 0.5 + sum_k basis_k * sh[c][k])  (sh.cpp:45-49). Coefficient c*K + k of a
// primitive is component (c*K + k) % 4 of float4 plane (c*K + k) / 4. All planes are loaded
// before the first FMA (one memory round trip; the double geometry is dead by now).
template <int DEG>
__device__ __forceinline__ void shade_sh(const float4* sh, uint64_t n, uint64_t i, float x,
                                         float y, float z, float rgb[3]) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    constexpr int kPlanes = (3 * K + 3) / 4;
    float c[4 * kPlanes];
#pragma unroll
    for (int p = 0; p < kPlanes; ++p) {
        const float4 v = __ldg(sh + uint64_t(p) * n + i);
        c[4 * p + 0] = v.x; c[4 * p + 1] = v.y; c[4 * p + 2] = v.z; c[4 * p + 3] = v.w;
    }
    float basis[16];
    sh_basis<DEG>(x, y, z, basis);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        // explicit FMAs: this file is compiled with -fmad=false for the double geometry, but
        // the fp32 shading has no bit-exactness contract (the reference shades in double)
        float acc = 0.5f;
#pragma unroll
        for (int k = 0; k < K; ++k) acc = __fmaf_rn(basis[k], c[ch * K + k], acc);
        rgb[ch] = (acc < 0.0f) ? 0.0f : acc;
    }
}

}  // namespace

// ---- K1: transform_primitives (gaussian.cpp:65-79) in place ------------------------------
__global__ void __launch_bounds__(256) pose_kernel(DevField f, uint64_t begin, uint64_t end,
                                                   gsim_rigid tr) {
    const dq tq{tr.rotation[0], tr.rotation[1], tr.rotation[2], tr.rotation[3]};
    const dv3 tt = mk3(tr.translation[0], tr.translation[1], tr.translation[2]);
    for (uint64_t i = begin + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < end;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const dv3 m = add3(qrotate(tq, mk3(f.mx[i], f.my[i], f.mz[i])), tt);
        dq q = qmul(tq, dq{f.qw[i], f.qx[i], f.qy[i], f.qz[i]});
        // Renormalise only on drift so an identity transform is a bit-exact no-op.
        if (fabs(qnorm(q) - 1.0) > 1e-12) q = qnormalized(q);
        f.mx[i] = m.x; f.my[i] = m.y; f.mz[i] = m.z;
        f.qw[i] = q.w; f.qx[i] = q.x; f.qy[i] = q.y; f.qz[i] = q.z;
    }
}

// ---- K2: project + shade_sh (raster.cpp:66-163, sh.cpp:10-51) ---------------------------
template <int DEG, bool kFull, int NT, int MINB, bool kSmemCams>
__global__ void __launch_bounds__(NT, MINB) preprocess_kernel(PreprocessArgs args) {
    __shared__ uint64_t s_seg_begin[kMaxSmemSegments];
    __shared__ DevCamera s_cams[kMaxSmemCams];
    const DevField f = args.field;
    const int n_seg_smem = args.n_segs < kMaxSmemSegments ? args.n_segs : kMaxSmemSegments;
    for (int k = threadIdx.x; k < n_seg_smem; k += blockDim.x) s_seg_begin[k] = args.segs[k].begin;
    // Cameras are read in every iteration of the camera loop: shared memory keeps those reads
    // off the L1 miss path.
    // kSmemCams: the batch has at most kMaxSmemCams cameras (the loop then reads shared memory
    // only, no generic loads)
    if (kSmemCams) {
        static_assert(sizeof(DevCamera) % 8 == 0, "DevCamera copy");
        const uint64_t* src = reinterpret_cast<const uint64_t*>(args.cams);
        uint64_t* dst = reinterpret_cast<uint64_t*>(s_cams);
        const uint32_t words = args.n_cams * uint32_t(sizeof(DevCamera) / 8);
        for (uint32_t k = threadIdx.x; k < words; k += blockDim.x) dst[k] = src[k];
    }
    __syncthreads();

    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < f.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        int si;
        if (args.n_segs <= kMaxSmemSegments) {
            si = upper_index(s_seg_begin, args.n_segs, i);
        } else {
            int lo = 0, hi = args.n_segs - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (args.segs[mid].begin <= i) lo = mid; else hi = mid - 1;
            }
            si = lo;
        }
        const DevSegment& seg = args.segs[si];
        if (seg.entry_count == 0 || i >= seg.end) continue;
        const dq nq = seg_q(seg);
        const dv3 nt = mk3(seg.t[0], seg.t[1], seg.t[2]);

        // Per primitive, camera independent (raster.cpp:87,165-170).
        const dv3 mean_world = add3(qrotate(nq, mk3(f.mx[i], f.my[i], f.mz[i])), nt);
        const dq rot_world = qmul(nq, dq{f.qw[i], f.qx[i], f.qy[i], f.qz[i]});
        const dm3 r = qmatrix(rot_world);
        const double sxv = f.sx[i], syv = f.sy[i], szv = f.sz[i];
        const dm3 d{{sxv * sxv, 0, 0, 0, syv * syv, 0, 0, 0, szv * szv}};
        const dm3 cov_world = mmul(mmul(r, d), mtransposed(r));
        const double opacity = f.opacity[i];

        // View direction in the node frame uses the inverse node rotation (raster.cpp:136-139).
        const float nqw = float(nq.w), nqx = -float(nq.x), nqy = -float(nq.y), nqz = -float(nq.z);

        for (uint32_t e = 0; e < seg.entry_count; ++e) {
            const SegEntry ent = args.entries[seg.entry_begin + e];
            const DevCamera& cam = kSmemCams ? s_cams[ent.cam] : args.cams[ent.cam];
            const uint64_t slot = ent.slot_base + (i - seg.begin);

            const dq cq{cam.q[0], cam.q[1], cam.q[2], cam.q[3]};
            const dv3 mean_cam = add3(qrotate(cq, mean_world), mk3(cam.t[0], cam.t[1], cam.t[2]));
            const double z = mean_cam.z;
            bool alive = (z > cam.near_p) && (z < cam.far_p);
            double u = 0, v = 0, cov_xx = 0, cov_xy = 0, cov_yy = 0, det = 1, radius = 0;
            if (alive) {
                const double rz = __drcp_rn(z);
                u = div_rn(cam.fx * mean_cam.x, z, rz) + cam.cx;
                v = div_rn(cam.fy * mean_cam.y, z, rz) + cam.cy;
                dm3 rwc;
#pragma unroll
                for (int k = 0; k < 9; ++k) rwc.m[k] = cam.r[k];
                const dm3 t1 = mmul(rwc, cov_world);
                const dm3 rwct = mtransposed(rwc);
                // cov_cam = r_wc * cov_world * r_wc^T, only the entries the 2x3 Jacobian uses.
                const double c00 = mm_entry(t1, rwct, 0, 0), c01 = mm_entry(t1, rwct, 0, 1),
                             c02 = mm_entry(t1, rwct, 0, 2), c11 = mm_entry(t1, rwct, 1, 1),
                             c12 = mm_entry(t1, rwct, 1, 2), c20 = mm_entry(t1, rwct, 2, 0),
                             c21 = mm_entry(t1, rwct, 2, 1), c22 = mm_entry(t1, rwct, 2, 2);
                const double tx = clampd(div_rn(mean_cam.x, z, rz), -cam.limx, cam.limx) * z;
                const double ty = clampd(div_rn(mean_cam.y, z, rz), -cam.limy, cam.limy) * z;
                const double zz = z * z;
                const double rzz = __drcp_rn(zz);
                const double j00 = div_rn(cam.fx, z, rz);
                const double j02 = div_rn(-cam.fx * tx, zz, rzz);
                const double j11 = div_rn(cam.fy, z, rz);
                const double j12 = div_rn(-cam.fy * ty, zz, rzz);
                const double a = j00 * (j00 * c00 + j02 * c20) + j02 * (j00 * c02 + j02 * c22);
                const double b = j00 * (j11 * c01 + j12 * c02) + j02 * (j11 * c21 + j12 * c22);
                const double c = j11 * (j11 * c11 + j12 * c21) + j12 * (j11 * c12 + j12 * c22);
                cov_xx = a + kCovarianceFloor;
                cov_xy = b;
                cov_yy = c + kCovarianceFloor;
                det = cov_xx * cov_yy - cov_xy * cov_xy;
                alive = (det > 0.0) && isfinite(det);
                if (alive) {
                    const double mid = 0.5 * (cov_xx + cov_yy);
                    const double disc = mid * mid - det;
                    const double lambda_max = mid + sqrt((0.0 < disc) ? disc : 0.0);
                    radius = 3.0 * sqrt(lambda_max);
                    alive = !(u + radius < 0.0 || u - radius > cam.width || v + radius < 0.0 ||
                              v - radius > cam.height);
                }
            }
            if (kFull) args.full_visible[slot] = alive ? 1 : 0;
            if (!alive) {
                args.keys[slot] = kInvalidKey;
                continue;
            }
            // Tile rect (raster.cpp:178-188), floor-inclusive, then clamped.
            int tx0 = x86_trunc_int(floor((u - radius) / kTileSize));
            int tx1 = x86_trunc_int(floor((u + radius) / kTileSize));
            int ty0 = x86_trunc_int(floor((v - radius) / kTileSize));
            int ty1 = x86_trunc_int(floor((v + radius) / kTileSize));
            const bool off_grid = tx1 < 0 || tx0 >= cam.tiles_x || ty1 < 0 || ty0 >= cam.tiles_y;
            tx0 = tx0 < 0 ? 0 : tx0;
            ty0 = ty0 < 0 ? 0 : ty0;
            tx1 = tx1 > cam.tiles_x - 1 ? cam.tiles_x - 1 : tx1;
            ty1 = ty1 > cam.tiles_y - 1 ? cam.tiles_y - 1 : ty1;

            // Record geometry in fp32 first, so the double state is dead before shading.
            const float fz = __double2float_rn(z);
            const float fu = __double2float_rn(u), fv = __double2float_rn(v),
                        frad = __double2float_rn(radius);
            float fia = 0.f, fib = 0.f, fic = 0.f;
            if (!off_grid) {
                const double inv_det = __drcp_rn(det);  // == 1.0 / det (both correctly rounded)
                fia = __double2float_rn(cov_yy * inv_det);
                fib = __double2float_rn(-cov_xy * inv_det);
                fic = __double2float_rn(cov_xx * inv_det);
            }
            float vx = float(mean_world.x - cam.center[0]);
            float vy = float(mean_world.y - cam.center[1]);
            float vz = float(mean_world.z - cam.center[2]);
            // normalize with one reciprocal square root (fp32 shading direction: no exactness
            // contract, the approximation moves the colour by ~1e-7)
            const float d2 = vx * vx + vy * vy + vz * vz;
            if (d2 > 0.0f) {
                const float inv = rsqrtf(d2);
                vx *= inv; vy *= inv; vz *= inv;
            }
            // inverse_rotate(view) = conj(q).rotate(view), math.hpp:139-144, in fp32.
            const float t0 = 2.0f * (nqy * vz - nqz * vy);
            const float t1v = 2.0f * (nqz * vx - nqx * vz);
            const float t2 = 2.0f * (nqx * vy - nqy * vx);
            const float lx = vx + t0 * nqw + (nqy * t2 - nqz * t1v);
            const float ly = vy + t1v * nqw + (nqz * t0 - nqx * t2);
            const float lz = vz + t2 * nqw + (nqx * t1v - nqy * t0);
            // Coefficients are (re)loaded per camera: the first camera brings the primitive's
            // 192 B into L1, later cameras hit it; nothing is held across the camera loop.
            float rgb[3];
            shade_sh<DEG>(f.sh, f.n, i, lx, ly, lz, rgb);

            if (kFull) {
                gsim_projected_splat s;
                s.pixel_center[0] = u;
                s.pixel_center[1] = v;
                s.cov_xx = cov_xx; s.cov_xy = cov_xy; s.cov_yy = cov_yy;
                s.inv_xx = cov_yy / det;
                s.inv_xy = -cov_xy / det;
                s.inv_yy = cov_xx / det;
                s.view_depth = z;
                s.alpha_peak = opacity;
                s.rgb[0] = rgb[0]; s.rgb[1] = rgb[1]; s.rgb[2] = rgb[2];
                s.radius = radius;
                s.prim_index = uint32_t(i);
                s.reserved = 0;
                args.full[slot] = s;
            }
            if (off_grid) {
                args.keys[slot] = kInvalidKey;
                continue;
            }
            args.records[slot] = make_record(fu, fv, fz, frad, fia, fib, fic,
                                             __double2float_rn(opacity), rgb[0], rgb[1], rgb[2]);
            const uint32_t rec_rect = pack_rect(tx0, ty0, tx1, ty1);
            args.rects[slot] = rec_rect;
            // Sort key: the float32 depth bits (depth_sort_key, raster.hpp:45-47) rebased to the
            // batch's [near, far] range; positive floats order like their bit patterns, so the
            // order is unchanged. The camera is the sort's segment (sort.cu), not a key digit.
            args.keys[slot] = __float_as_uint(fz) - args.key_base;
        }
    }
}

// ---- rasterize(splats) entry: host ProjectedSplats -> records + keys -----------------------
__global__ void __launch_bounds__(256) splats_to_records_kernel(SplatArgs args) {
    const DevCamera cam = args.cam[0];
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < args.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const gsim_projected_splat sp = args.splats[i];
        const double u = sp.pixel_center[0], v = sp.pixel_center[1], r = sp.radius;
        int tx0 = x86_trunc_int(floor((u - r) / kTileSize));
        int tx1 = x86_trunc_int(floor((u + r) / kTileSize));
        int ty0 = x86_trunc_int(floor((v - r) / kTileSize));
        int ty1 = x86_trunc_int(floor((v + r) / kTileSize));
        if (tx1 < 0 || tx0 >= cam.tiles_x || ty1 < 0 || ty0 >= cam.tiles_y) {
            args.keys[i] = kInvalidKey;
            continue;
        }
        tx0 = tx0 < 0 ? 0 : tx0;
        ty0 = ty0 < 0 ? 0 : ty0;
        tx1 = tx1 > cam.tiles_x - 1 ? cam.tiles_x - 1 : tx1;
        ty1 = ty1 > cam.tiles_y - 1 ? cam.tiles_y - 1 : ty1;
        const float fz = __double2float_rn(sp.view_depth);
        args.records[i] = make_record(
            __double2float_rn(u), __double2float_rn(v), fz, __double2float_rn(r),
            __double2float_rn(sp.inv_xx), __double2float_rn(sp.inv_xy),
            __double2float_rn(sp.inv_yy), __double2float_rn(sp.alpha_peak),
            __double2float_rn(sp.rgb[0]), __double2float_rn(sp.rgb[1]),
            __double2float_rn(sp.rgb[2]));
        args.rects[i] = pack_rect(tx0, ty0, tx1, ty1);
        // Full 32-bit depth_sort_key (raster.hpp:45-47): hand-made splats may carry any depth.
        uint32_t key = __float_as_uint(fz);
        if (key == kInvalidKey) key = kInvalidKey - 1;  // reserved sentinel (a NaN payload)
        args.keys[i] = key;
    }
}

// ---- host launchers ------------------------------------------------------------------------
void launch_pose(const DevField& f, uint64_t begin, uint64_t end, const gsim_rigid& t,
                 int grid_cap, cudaStream_t stream) {
    const uint64_t n = end - begin;
    if (n == 0) return;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > uint64_t(grid_cap)) blocks = grid_cap;
    pose_kernel<<<unsigned(blocks), 256, 0, stream>>>(f, begin, end, t);
}

// 128-thread blocks at 5 per SM (102 registers): the double-precision camera loop spills
// little and 20 warps per SM hide its load latency (measured best of 256x2/3, 128x5/6, 192x3).
template <int DEG>
static void launch_pre_deg(const PreprocessArgs& a, bool full, uint64_t n, int n_sms,
                           cudaStream_t s) {
    constexpr int kNT = 128, kMinB = 5;
    // GSIM_GPU_PRE_CTAS: resident blocks per SM of the grid (fewer leave room for other
    // contexts' kernels on the same SM)
    static const int per_sm = [] {
        const char* e = std::getenv("GSIM_GPU_PRE_CTAS");
        const int v = e ? std::atoi(e) : kMinB;
        return v < 1 ? 1 : v > kMinB ? kMinB : v;
    }();
    const unsigned grid =
        unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + kNT - 1) / kNT, uint64_t(n_sms) * per_sm)));
    const bool smem_cams = a.n_cams <= uint32_t(kMaxSmemCams);
    if (full) {
        if (smem_cams) preprocess_kernel<DEG, true, kNT, kMinB, true><<<grid, kNT, 0, s>>>(a);
        else preprocess_kernel<DEG, true, kNT, kMinB, false><<<grid, kNT, 0, s>>>(a);
    } else {
        if (smem_cams) preprocess_kernel<DEG, false, kNT, kMinB, true><<<grid, kNT, 0, s>>>(a);
        else preprocess_kernel<DEG, false, kNT, kMinB, false><<<grid, kNT, 0, s>>>(a);
    }
}

void launch_preprocess(const PreprocessArgs& a, bool full, int n_sms, cudaStream_t stream) {
    if (a.field.n == 0) return;
    switch (a.field.sh_degree) {
        case 0: launch_pre_deg<0>(a, full, a.field.n, n_sms, stream); break;
        case 1: launch_pre_deg<1>(a, full, a.field.n, n_sms, stream); break;
        case 2: launch_pre_deg<2>(a, full, a.field.n, n_sms, stream); break;
        default: launch_pre_deg<3>(a, full, a.field.n, n_sms, stream); break;
    }
}

void launch_splats_to_records(const SplatArgs& a, int grid_cap, cudaStream_t stream) {
    if (a.n == 0) return;
    uint64_t blocks = (a.n + 255) / 256;
    if (blocks > uint64_t(grid_cap)) blocks = grid_cap;
    splats_to_records_kernel<<<unsigned(blocks), 256, 0, stream>>>(a);
}

}  // namespace gsim_gpu
