// raster.cu — K4: per-tile front-to-back compositing (raster.cpp:273-320).
//
// One 256-thread CTA per (camera, 16x16 tile); thread = pixel. The 8 warps own 8x4 pixel
// sub-rectangles so a splat's footprint test can be made per warp. The tile's depth-sorted
// list is consumed in batches of 256 records: each thread gathers one 48-byte record into
// shared memory and computes an 8-bit mask of the warp rectangles the splat can reach
// (its 3-sigma box intersected with the alpha >= 1/255 ellipse bound, conservatively
// widened). Each warp then walks only the splats whose bit it owns (ballot + ffs keeps the
// depth order), and drops out as soon as all its pixels are saturated; the CTA leaves when
// __syncthreads_count says every pixel is done.
//
// Per-pixel contract (raster.cpp:284-318): box test |dx|>r || |dy|>r, q with 2*inv_xy,
// alpha = min(o*exp(-q/2), 0.99), skip alpha < 1/255, accumulate, T *= 1-alpha, stop after
// accumulating once T < cutoff; rgb clamped to [0,1] at write, depth unnormalised unless
// asked, accum_alpha = sum of weights. Empty tiles write zeros (image.hpp:44).
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {
constexpr int kThreads = 256;
constexpr int kBatch = 256;
constexpr float kLog2e = 1.4426950408889634f;
}  // namespace

__global__ void __launch_bounds__(kThreads) raster_kernel(RasterArgs a) {
    __shared__ float4 s_p0[kBatch];  // u, v, radius, log2(opacity)
    __shared__ float4 s_p1[kBatch];  // inv_xx, 2*inv_xy, inv_yy, depth
    __shared__ float4 s_p2[kBatch];  // r, g, b, -
    __shared__ uint8_t s_mask[kBatch];

    const uint32_t g = blockIdx.x;
    const int cam_idx = upper_index(a.cam_tile_base, a.n_cams, g);
    const DevCamera& cam = a.cams[cam_idx];
    const uint32_t tile = g - a.cam_tile_base[cam_idx];
    const int tx = int(tile % uint32_t(cam.tiles_x)), ty = int(tile / uint32_t(cam.tiles_x));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // warp w owns the 8x4 block (w % 2, w / 2) of the tile; lane = (lane % 8, lane / 8)
    const int wx0 = tx * kTileSize + (warp & 1) * 8, wy0 = ty * kTileSize + (warp >> 1) * 4;
    const int x = wx0 + (lane & 7), y = wy0 + (lane >> 3);
    const float px = float(x) + 0.5f, py = float(y) + 0.5f;

    const uint32_t begin = a.tile_begin[g], end = a.tile_end[g];
    float cr = 0.f, cg = 0.f, cb = 0.f, d = 0.f, acc = 0.f, T = 1.f;
    bool done = false;

    // Warp-rectangle pixel-centre bounds used by the mask test: x columns (2) and y rows (4).
    const float tile_x0 = float(tx * kTileSize) + 0.5f, tile_y0 = float(ty * kTileSize) + 0.5f;

    uint32_t fetched = 0;
    for (uint32_t b0 = begin; b0 < end; b0 += kBatch) {
        const uint32_t n_b = (end - b0) < uint32_t(kBatch) ? (end - b0) : uint32_t(kBatch);
        fetched += n_b;
        uint8_t mask = 0;
        if (uint32_t(tid) < n_b) {
            const uint32_t slot = a.values[b0 + tid];
            const Record r = a.records[slot];
            const float u = r.a.x, v = r.a.y, rad = r.a.w, op = r.b.w;
            const float ia = r.b.x, ib = r.b.y, ic = r.b.z;
            s_p0[tid] = make_float4(u, v, rad, __log2f(op));
            s_p1[tid] = make_float4(ia, 2.0f * ib, ic, r.a.z);
            s_p2[tid] = make_float4(r.c.x, r.c.y, r.c.z, 0.f);
            // Reachable half-extents: the box test bounds |dx|,|dy| <= r; alpha >= 1/255 needs
            // q <= qc = 2 ln(255 o), whose ellipse has half-extents sqrt(qc * cov_xx/yy).
            float ex = rad, ey = rad;
            if (op * 255.0f < 1.0f) {
                ex = -1.0f;  // can never reach alpha 1/255
            } else {
                const float qc = 2.0f * logf(op * 255.0f);
                const float det = ia * ic - ib * ib;
                if (det > 0.0f) {
                    const float cxx = ic / det, cyy = ia / det;  // covariance from the conic
                    const float bx = sqrtf(qc * cxx) * 1.01f + 0.05f;
                    const float by = sqrtf(qc * cyy) * 1.01f + 0.05f;
                    ex = fminf(ex, bx);
                    ey = fminf(ey, by);
                }
            }
            if (ex >= 0.0f) {
                // column c covers pixel centres [tile_x0 + 8c, tile_x0 + 8c + 7]
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const float lo = tile_x0 + 8.0f * c, hi = lo + 7.0f;
                    if (u + ex < lo || u - ex > hi) continue;
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr) {
                        const float ylo = tile_y0 + 4.0f * rr, yhi = ylo + 3.0f;
                        if (v + ey < ylo || v - ey > yhi) continue;
                        mask |= uint8_t(1u << (rr * 2 + c));
                    }
                }
            }
        }
        s_mask[tid] = mask;
        __syncthreads();

        if (!__all_sync(0xffffffffu, done)) {
            for (int j = 0; j < int(n_b); j += 32) {
                uint32_t m = __ballot_sync(0xffffffffu, (s_mask[j + lane] >> warp) & 1u);
                while (m) {
                    const int s = j + __ffs(m) - 1;
                    m &= m - 1;
                    if (done) continue;
                    const float4 p0 = s_p0[s];
                    const float dx = p0.x - px, dy = p0.y - py;
                    if (fabsf(dx) > p0.z || fabsf(dy) > p0.z) continue;
                    const float4 p1 = s_p1[s];
                    const float q = p1.x * dx * dx + p1.y * dx * dy + p1.z * dy * dy;
                    const float alpha = fminf(exp2f(fmaf(q, -0.5f * kLog2e, p0.w)), 0.99f);
                    if (alpha < float(kAlphaSkip)) continue;
                    const float4 p2 = s_p2[s];
                    const float w = alpha * T;
                    cr += p2.x * w;
                    cg += p2.y * w;
                    cb += p2.z * w;
                    d += p1.w * w;
                    acc += w;
                    T *= 1.0f - alpha;
                    if (T < a.cutoff) done = true;
                }
                if (__all_sync(0xffffffffu, done)) break;
            }
        }
        if (__syncthreads_count(done ? 0 : 1) == 0) break;
    }

    if (tid == 0 && fetched) atomicAdd(a.consumed, (unsigned long long)fetched);
    if (x < cam.width && y < cam.height) {
        float* base = a.out + cam.out_offset;
        const size_t npx = size_t(cam.width) * cam.height;
        const size_t p = size_t(y) * cam.width + x;
        base[3 * p + 0] = fminf(fmaxf(cr, 0.f), 1.f);
        base[3 * p + 1] = fminf(fmaxf(cg, 0.f), 1.f);
        base[3 * p + 2] = fminf(fmaxf(cb, 0.f), 1.f);
        base[3 * npx + p] = a.normalize_depth ? (acc > 1e-12f ? d / acc : 0.f) : d;
        base[4 * npx + p] = acc;
    }
}

void launch_raster(const RasterArgs& a, uint32_t n_tiles, cudaStream_t stream) {
    if (n_tiles == 0) return;
    raster_kernel<<<n_tiles, kThreads, 0, stream>>>(a);
}

}  // namespace gsim_gpu
