// raster.cu — K4: per-tile front-to-back compositing (raster.cpp:273-320).
//
// One 256-thread CTA per (camera, 16x16 tile); thread = pixel. The 8 warps own 8x4 pixel
// sub-rectangles. The tile's depth-sorted list is consumed in batches of 256 records:
//   1. each thread gathers one 48-byte record into shared memory and computes an 8-bit mask
//      of the warp rectangles the splat can reach (its 3-sigma box intersected with the
//      alpha >= 1/255 ellipse bound, conservatively widened, so no contributing splat is
//      ever dropped);
//   2. each warp compacts the indices of the splats whose bit it owns into a private list
//      (ballot + popc keeps the depth order);
//   3. each warp walks its list with a branch-free blend: a splat that fails the box test or
//      the 1/255 skip gets alpha 0, which leaves C, D, A and T bit-for-bit unchanged, so the
//      result equals the reference's skip-with-continue loop;
//   4. a pixel that saturates (T < cutoff after accumulating) parks at T = 0, so later
//      weights are exactly zero; a warp stops when all its pixels are parked and the CTA
//      leaves when __syncthreads_count says every pixel is.
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
constexpr int kWarps = kThreads / 32;
constexpr int kBatch = 256;
constexpr float kLog2e = 1.4426950408889634f;

// The conic is stored prescaled by -log2(e)/2 so the exponent of ex2 is
// lop + dx*(A*dx + B*dy) + C*dy*dy: five FP32 ops per pixel and splat.
struct alignas(16) SmemSplat {
    float4 p0;  // u, v, radius, log2(opacity)
    float4 p1;  // A = -inv_xx*log2e/2, B = -inv_xy*log2e, C = -inv_yy*log2e/2, depth
    float4 p2;  // r, g, b, -
};

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
}  // namespace

__global__ void __launch_bounds__(kThreads, 5) raster_kernel(RasterArgs a) {
    __shared__ SmemSplat s_spl[kBatch];
    __shared__ uint8_t s_mask[kBatch];
    __shared__ uint16_t s_list[kWarps][kBatch];

    const uint32_t g = blockIdx.x;
    const int cam_idx = upper_index(a.cam_tile_base, a.n_cams, g);
    const DevCamera& cam = a.cams[cam_idx];
    const uint32_t tile = g - a.cam_tile_base[cam_idx];
    const int tiles_x = cam.tiles_x;
    const int tx = int(tile % uint32_t(tiles_x)), ty = int(tile / uint32_t(tiles_x));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // warp w owns the 8x4 block (w % 2, w / 2) of the tile; lane = (lane % 8, lane / 8)
    const int x = tx * kTileSize + (warp & 1) * 8 + (lane & 7);
    const int y = ty * kTileSize + (warp >> 1) * 4 + (lane >> 3);
    const float px = float(x) + 0.5f, py = float(y) + 0.5f;

    // On a pair-buffer overflow the host re-runs scatter + raster; until then keep every read
    // in bounds (the clamped frame is discarded).
    const uint64_t b64 = a.cam_pair_base[cam_idx] + a.tile_rel[g];
    const uint32_t begin = uint32_t(b64 < a.capacity ? b64 : a.capacity);
    const uint64_t e64 = b64 + a.tile_count[g];
    const uint32_t end = uint32_t(e64 < a.capacity ? e64 : a.capacity);
    const float cutoff = a.cutoff;
    float cr = 0.f, cg = 0.f, cb = 0.f, d = 0.f, acc = 0.f, T = 1.f;

    // Pixel-centre bounds of the 2 warp columns and 4 warp rows of this tile.
    const float tile_x0 = float(tx * kTileSize) + 0.5f, tile_y0 = float(ty * kTileSize) + 0.5f;

    uint32_t fetched = 0;
    for (uint32_t b0 = begin; b0 < end; b0 += kBatch) {
        const uint32_t n_b = (end - b0) < uint32_t(kBatch) ? (end - b0) : uint32_t(kBatch);
        fetched += n_b;
        uint32_t mask = 0;
        if (uint32_t(tid) < n_b) {
            uint32_t slot = __ldg(a.values + b0 + tid);
            if (slot >= a.n_slots) slot = 0;  // only possible in a clamped (overflowed) frame
            const float4 ra = __ldg(&a.records[slot].a);
            const float4 rb = __ldg(&a.records[slot].b);
            const float4 rc = __ldg(&a.records[slot].c);
            const float u = ra.x, v = ra.y, rad = ra.w, op = rb.w;
            const float ia = rb.x, ib = rb.y, ic = rb.z;
            s_spl[tid].p0 = make_float4(u, v, rad, __log2f(op));
            s_spl[tid].p1 = make_float4(ia * (-0.5f * kLog2e), ib * -kLog2e, ic * (-0.5f * kLog2e), ra.z);
            s_spl[tid].p2 = make_float4(rc.x, rc.y, rc.z, 0.f);
            // Reachable half-extents: the box test bounds |dx|,|dy| <= r; alpha >= 1/255 needs
            // q <= qc = 2 ln(255 o), whose ellipse has half-extents sqrt(qc * cov_xx/yy).
            float ex = rad, ey = rad;
            if (op * 255.0f < 1.0f) {
                ex = -1.0f;  // can never reach alpha 1/255
            } else {
                const float qc = 2.0f * __logf(op * 255.0f);
                const float det = ia * ic - ib * ib;
                if (det > 0.0f) {
                    const float inv = 1.0f / det;
                    const float bx = sqrtf(qc * ic * inv) * 1.01f + 0.05f;
                    const float by = sqrtf(qc * ia * inv) * 1.01f + 0.05f;
                    ex = fminf(ex, bx);
                    ey = fminf(ey, by);
                }
            }
            if (ex >= 0.0f) {
                uint32_t cols = 0, rows = 0;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const float lo = tile_x0 + 8.0f * c;
                    cols |= (u + ex >= lo && u - ex <= lo + 7.0f) ? (1u << c) : 0u;
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const float lo = tile_y0 + 4.0f * r;
                    rows |= (v + ey >= lo && v - ey <= lo + 3.0f) ? (1u << r) : 0u;
                }
                // bit (row * 2 + col) for every reachable (col, row)
                const uint32_t colmask = (cols & 1u) * 0x55u | ((cols >> 1) & 1u) * 0xAAu;
                const uint32_t rowmask = (rows & 1u) * 0x03u | ((rows >> 1) & 1u) * 0x0Cu |
                                         ((rows >> 2) & 1u) * 0x30u | ((rows >> 3) & 1u) * 0xC0u;
                mask = colmask & rowmask;
            }
        }
        s_mask[tid] = uint8_t(mask);
        __syncthreads();

        if (!__all_sync(0xffffffffu, T == 0.0f)) {
            // Compact this warp's splats (depth order preserved) as byte offsets into s_spl.
            uint32_t count = 0;
            for (uint32_t j = 0; j < n_b; j += 32) {
                const uint32_t idx = j + lane;
                const bool mine = idx < n_b && ((s_mask[idx] >> warp) & 1u);
                const uint32_t bits = __ballot_sync(0xffffffffu, mine);
                if (mine)
                    s_list[warp][count + __popc(bits & lanemask_lt())] =
                        uint16_t(idx * sizeof(SmemSplat));
                count += __popc(bits);
            }
            __syncwarp();
            const char* spl = reinterpret_cast<const char*>(s_spl);
            for (uint32_t k0 = 0; k0 < count; k0 += 32) {
                const uint32_t k1 = (k0 + 32 < count) ? k0 + 32 : count;
#pragma unroll 4
                for (uint32_t k = k0; k < k1; ++k) {
                    const SmemSplat& sp = *reinterpret_cast<const SmemSplat*>(spl + s_list[warp][k]);
                    const float4 p0 = sp.p0, p1 = sp.p1, p2 = sp.p2;
                    const float dx = p0.x - px, dy = p0.y - py;
                    const float t = fmaf(p1.y, dy, p1.x * dx);
                    const float E = fmaf(p1.z * dy, dy, fmaf(t, dx, p0.w));
                    const float e = fminf(ex2_approx(E), 0.99f);
                    const bool ok = fmaxf(fabsf(dx), fabsf(dy)) <= p0.z && e >= float(kAlphaSkip);
                    const float w = (ok ? e : 0.0f) * T;
                    cr = fmaf(p2.x, w, cr);
                    cg = fmaf(p2.y, w, cg);
                    cb = fmaf(p2.z, w, cb);
                    d = fmaf(p1.w, w, d);
                    acc += w;
                    // T * (1 - alpha) == T - w up to rounding; a saturated pixel parks at T = 0,
                    // where every later weight is exactly zero (the reference's break).
                    const float Tn = T - w;
                    T = (ok && Tn < cutoff) ? 0.0f : Tn;
                }
                if (__all_sync(0xffffffffu, T == 0.0f)) break;
            }
        }
        if (__syncthreads_count(T == 0.0f ? 0 : 1) == 0) break;
    }

    if (tid == 0 && fetched) atomicAdd(a.consumed, (unsigned long long)fetched);
    if (x < cam.width && y < cam.height) {
        const float r = fminf(fmaxf(cr, 0.f), 1.f), gg = fminf(fmaxf(cg, 0.f), 1.f),
                    bb = fminf(fmaxf(cb, 0.f), 1.f);
        const float depth = a.normalize_depth ? (acc > 1e-12f ? d / acc : 0.f) : d;
        if (a.out) {
            float* base = a.out + cam.out_offset;
            const size_t npx = size_t(cam.width) * cam.height;
            const size_t p = size_t(y) * cam.width + x;
            base[3 * p + 0] = r;
            base[3 * p + 1] = gg;
            base[3 * p + 2] = bb;
            base[3 * npx + p] = depth;
            base[4 * npx + p] = acc;
        }
        if (a.enc.flags) {
            uint8_t* blk = a.enc.dst + cam.out_offset / 5 * encoded_bpp(a.enc.flags);
            encode_pixel(a.enc, a.enc.srgb_thr, blk, uint32_t(cam.width), uint32_t(cam.height),
                         uint32_t(x), uint32_t(y), r, gg, bb, depth, acc);
        }
    }
}

void launch_raster(const RasterArgs& a, uint32_t n_tiles, cudaStream_t stream) {
    if (n_tiles == 0) return;
    raster_kernel<<<n_tiles, kThreads, 0, stream>>>(a);
}

}  // namespace gsim_gpu
