// raster.cu — K4: per-tile front-to-back compositing (raster.cpp:204-251).
//
// One 128-thread CTA per (camera, 16x16 tile); each thread owns TWO horizontally adjacent
// pixels, so every per-splat quantity that depends only on the row (dy, the dy terms of the
// quadratic form, the |dy| box test) is computed once for both, and the per-pixel arithmetic
// runs on Blackwell's packed FP32 pipe (FFMA2 / FMUL2 / FADD2 on float2 registers). The 4
// warps own 64-pixel warp rectangles (16x4 bands or 8x8 quadrants, template RW). The tile's
// depth-sorted list is consumed in batches of 256 records:
//   1. each thread gathers two 48-byte records into shared memory and computes a 4-bit mask
//      of the warp rectangles each splat can reach (its 3-sigma box intersected with the
//      alpha >= 1/255 ellipse bound, conservatively widened, so no contributing splat is
//      ever dropped);
//   2. each warp compacts the indices of the splats whose bit it owns into a private list
//      (ballot + popc keeps the depth order);
//   3. each warp walks its list with a branch-free blend: a splat that fails the box test or
//      the 1/255 skip gets weight 0, which leaves C, D, A and T bit-for-bit unchanged, so the
//      result equals the reference's skip-with-continue loop;
//   4. a splat is composited only while T >= cutoff (a fourth condition of the gate), which is
//      the reference's break after the accumulation that takes T below the cutoff; a warp stops
//      when all its pixels are done and the CTA leaves when the batch barrier's count says every
//      pixel is. Lists whose splats all have peak opacity <= 0.989 skip the 0.99 clamp.
//
// Per-pixel contract (raster.cpp:215-249): box test |dx|>r || |dy|>r, q with 2*inv_xy,
// alpha = min(o*exp(-q/2), 0.99), skip alpha < 1/255, accumulate, T *= 1-alpha, stop after
// accumulating once T < cutoff; rgb clamped to [0,1] at write, depth unnormalised unless
// asked, accum_alpha = sum of weights. Empty tiles write zeros (image.hpp:44).
#include <climits>
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {
constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 bc(float s) { return make_float2(s, s); }

// (e0, e1) with each lane zeroed unless |dx_i| <= r, |dy| <= r, e_i >= 1/255 and the pixel is
// still alive (T_i >= cutoff: the reference breaks once T drops below the cutoff, so a splat is
// composited iff T before it is >= cutoff). The chained setp.and form gives one compare per
// condition and one select per pixel.
__device__ __forceinline__ float2 gate(float e0, float e1, float adx0, float adx1, float ady,
                                       float r, float2 T, float cutoff) {
    static_assert(float(kAlphaSkip) == 0x1.010102p-8f, "skip constant below");
    float2 o;
    asm("{\n\t.reg .pred py, p0, p1;\n\t"
        "setp.le.f32 py, %4, %5;\n\t"
        "setp.le.and.f32 p0, %2, %5, py;\n\t"
        "setp.le.and.f32 p1, %3, %5, py;\n\t"
        "setp.ge.and.f32 p0, %6, 0f3B808081, p0;\n\t"
        "setp.ge.and.f32 p1, %7, 0f3B808081, p1;\n\t"
        "setp.ge.and.f32 p0, %8, %10, p0;\n\t"
        "setp.ge.and.f32 p1, %9, %10, p1;\n\t"
        "selp.f32 %0, %6, 0f00000000, p0;\n\t"
        "selp.f32 %1, %7, 0f00000000, p1;\n\t}"
        : "=f"(o.x), "=f"(o.y)
        : "f"(adx0), "f"(adx1), "f"(ady), "f"(r), "f"(e0), "f"(e1), "f"(T.x), "f"(T.y),
          "f"(cutoff));
    return o;
}

// Record at a shared-memory address (the compacted list holds addresses, so the blend
// loop needs no address arithmetic).
__device__ __forceinline__ void load_record(uint32_t addr, float4& a, float4& b, float4& c) {
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%12];\n\t"
        "ld.shared.v4.f32 {%4, %5, %6, %7}, [%12+16];\n\t"
        "ld.shared.v4.f32 {%8, %9, %10, %11}, [%12+32];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w),
          "=f"(c.x), "=f"(c.y), "=f"(c.z), "=f"(c.w)
        : "r"(addr));
}

// log2 of the largest peak opacity whose alpha can never reach the 0.99 clamp (0.989, a margin
// for the rounding of the exponent): batches without brighter splats skip the clamp.
constexpr float kNoClampLog2 = -0.015957f;  // log2(0.989) rounded down

// Can the splat reach alpha >= 1/255 at any point of the rectangle [x_lo, x_hi] x [y_lo, y_hi]
// of pixel centres? The ex2 exponent E(dx, dy) = lop + dx (A dx + B dy) + C dy^2 (dx = u - px,
// dy = v - py) is concave; its maximum over the rectangle is at (0, 0) when the centre is
// inside, else on an edge facing the centre. Each candidate fixes one coordinate at the
// clamped centre offset and maximises the other in closed form (clamped to the range), so
// max(E1, E2) is the exact rectangle maximum (the approximate division only moves the
// candidate along the edge, which lowers E by a second-order amount). The threshold keeps a
// 0.02 margin below log2(1/255) so rounding can never drop a contributing splat.
__device__ __forceinline__ bool reaches_rect(float4 p0, float4 p1, float x_lo, float x_hi,
                                             float y_lo, float y_hi) {
    const float A = p1.z, B = p1.x, C = p1.y;
    const float dx_lo = p0.x - x_hi, dx_hi = p0.x - x_lo;  // range of dx over the rectangle
    const float dy_lo = p0.y - y_hi, dy_hi = p0.y - y_lo;
    const float dx1 = fminf(fmaxf(0.0f, dx_lo), dx_hi);
    const float dy1 = fminf(fmaxf(dx1 * __fdividef(B, -2.0f * C), dy_lo), dy_hi);
    const float dy2 = fminf(fmaxf(0.0f, dy_lo), dy_hi);
    const float dx2 = fminf(fmaxf(dy2 * __fdividef(B, -2.0f * A), dx_lo), dx_hi);
    const float e1 = p0.w + dx1 * (A * dx1 + B * dy1) + C * dy1 * dy1;
    const float e2 = p0.w + dx2 * (A * dx2 + B * dy2) + C * dy2 * dy2;
    return !(fmaxf(e1, e2) < -7.9943534f - 0.02f);  // NaN-safe: keep on doubt
}

__device__ __forceinline__ void write_pixel(const RasterArgs& a, const DevCamera& cam, int x, int y,
                                            float cr, float cg, float cb, float d, float acc) {
    if (x >= cam.width || y >= cam.height) return;
    const float r = fminf(fmaxf(cr, 0.f), 1.f), gg = fminf(fmaxf(cg, 0.f), 1.f),
                bb = fminf(fmaxf(cb, 0.f), 1.f);
    float depth = a.normalize_depth ? (acc > 1e-12f ? d / acc : 0.f) : d;
    if (acc < a.valid_alpha) depth = 0.f;  // render_depth_ring's invalid pixels
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
}  // namespace

// Front-to-back blend of a warp's compacted list for the thread's pixel pair (raster.cpp:
// 221-238). kClamp: some splat of the list can reach the 0.99 alpha clamp.
template <bool kClamp>
__device__ __forceinline__ void blend_one(uint32_t addr, float2 npx, float py, float cutoff,
                                          float2& cr, float2& cg, float2& cb, float2& d,
                                          float2& acc, float2& T) {
    float4 p0, p1, p2;
    load_record(addr, p0, p1, p2);
    // row terms, shared by the pair: (B dy, C dy) on the packed pipe
    const float dy = p0.y - py;
    const float2 bcdy = __fmul2_rn(make_float2(p1.x, p1.y), bc(dy));
    const float kq = fmaf(bcdy.y, dy, p0.w);
    // pair terms on the packed pipe
    const float2 dx = __fadd2_rn(bc(p0.x), npx);
    const float2 t = __ffma2_rn(bc(p1.z), dx, bc(bcdy.x));
    const float2 E = __ffma2_rn(t, dx, bc(kq));
    float e0 = ex2_approx(E.x), e1 = ex2_approx(E.y);
    if (kClamp) {
        e0 = fminf(e0, 0.99f);
        e1 = fminf(e1, 0.99f);
    }
    const float2 w = __fmul2_rn(gate(e0, e1, fabsf(dx.x), fabsf(dx.y), fabsf(dy), p0.z, T, cutoff), T);
    cr = __ffma2_rn(bc(p2.x), w, cr);
    cg = __ffma2_rn(bc(p2.y), w, cg);
    cb = __ffma2_rn(bc(p2.z), w, cb);
    d = __ffma2_rn(bc(p1.w), w, d);
    acc = __fadd2_rn(acc, w);
    // T * (1 - alpha) == T - w up to rounding; once T < cutoff the gate zeroes every later
    // weight, so T (and the pixel) stays put: the reference's break.
    T = __fadd2_rn(T, make_float2(-w.x, -w.y));
}

// Front-to-back blend of a warp's compacted list for the thread's pixel pair (raster.cpp:
// 221-238), 4 entries per 128-bit list load and the last 0-3 one by one (padding them with a
// null record instead cost a blend step per padding entry). kClamp: some splat of the list can
// reach the 0.99 alpha clamp.
template <bool kClamp>
__device__ __forceinline__ void blend_list(const uint32_t* list, uint32_t count, float2 npx,
                                           float py, float cutoff, float2& cr, float2& cg,
                                           float2& cb, float2& d, float2& acc, float2& T) {
    const uint32_t count4 = count & ~3u;
    for (uint32_t k0 = 0; k0 < count4; k0 += 32) {
        const uint32_t k1 = (k0 + 32 < count4) ? k0 + 32 : count4;
        for (uint32_t k = k0; k < k1; k += 4) {
            const uint4 q = *reinterpret_cast<const uint4*>(list + k);
            blend_one<kClamp>(q.x, npx, py, cutoff, cr, cg, cb, d, acc, T);
            blend_one<kClamp>(q.y, npx, py, cutoff, cr, cg, cb, d, acc, T);
            blend_one<kClamp>(q.z, npx, py, cutoff, cr, cg, cb, d, acc, T);
            blend_one<kClamp>(q.w, npx, py, cutoff, cr, cg, cb, d, acc, T);
        }
        if (__all_sync(0xffffffffu, T.x < cutoff && T.y < cutoff)) return;
    }
    for (uint32_t k = count4; k < count; ++k)  // the last 0-3 entries, one at a time
        blend_one<kClamp>(list[k], npx, py, cutoff, cr, cg, cb, d, acc, T);
}

// mbarrier helpers for the bulk-copy (TMA engine) staging variant.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// RW = warp-rectangle width in pixels (16: 16x4 bands, 8: 8x8 quadrants); kBatch = records
// per batch (two buffers of kBatch * 48 bytes of shared memory). kBulk: the records are staged
// with one cp.async.bulk (TMA engine, UBLKCP) per 48-byte record completing on a per-buffer
// mbarrier, instead of three 16-byte cp.async (LDGSTS) per record and a wait_all.
template <int RW, int kBatch, bool kBulk>
__global__ void __launch_bounds__(kThreads, kBatch == 128 ? 12 : 8) raster_kernel(RasterArgs a) {
    constexpr int kPerThread = kBatch / kThreads;
    constexpr int RH = 64 / RW;  // warp-rectangle height
    constexpr int PC = RW / 2;   // pixel-pair columns of a warp rectangle
    constexpr int WX = 16 / RW;  // warp rectangles per tile row
    __shared__ Record s_spl[2][kBatch];
    __shared__ __align__(16) uint32_t s_list[kWarps][kBatch];
    __shared__ __align__(8) uint64_t s_bar[2];  // kBulk: one mbarrier per record buffer

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t bar0 = uint32_t(__cvta_generic_to_shared(&s_bar[0]));
    uint32_t phase_bits = 0;   // kBulk: parity of the next phase of each buffer's barrier
    uint32_t pending_bulk = 0; // kBulk: buffers with copies issued and not yet waited for
    if (tid == 0) {
        if (kBulk) {
            mbar_init(bar0, kThreads);
            mbar_init(bar0 + 8u, kThreads);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
    }
    if (kBulk) __syncthreads();  // barriers initialised before any thread arrives

    // One CTA per tile of [tile_begin, n_tiles), or (GSIM_GPU_RASTER_CTAS) a capped grid whose
    // CTAs claim the tiles in order from a counter (the tail balances).
    __shared__ uint32_t s_tile;
    for (uint32_t g = a.tile_begin + blockIdx.x;;) {
        if (a.tile_ticket) {
            if (tid == 0) s_tile = a.tile_begin + atomicAdd(a.tile_ticket, 1u);
            __syncthreads();
            g = s_tile;
        }
        if (g >= a.n_tiles) break;
    const int cam_idx = upper_index(a.cam_tile_base, a.n_cams, g);
    const DevCamera& cam = a.cams[cam_idx];
    const uint32_t tile = g - a.cam_tile_base[cam_idx];
    const int tiles_x = cam.tiles_x;
    const int tx = int(tile % uint32_t(tiles_x)), ty = int(tile / uint32_t(tiles_x));
    const int rx0 = tx * kTileSize + (warp % WX) * RW, ry0 = ty * kTileSize + (warp / WX) * RH;
    const int x = rx0 + 2 * (lane % PC);  // first pixel of the pair
    const int y = ry0 + lane / PC;
    const float2 npx = make_float2(-(float(x) + 0.5f), -(float(x) + 1.5f));
    const float py = float(y) + 0.5f;
    // pixel-centre bounds of this warp's rectangle

    // On a pair-buffer overflow the host re-runs scatter + raster; until then keep every read
    // in bounds (the clamped frame is discarded).
    const uint64_t b64 = a.cam_pair_base[cam_idx] + a.tile_rel[g];
    const uint32_t begin = uint32_t(b64 < a.capacity ? b64 : a.capacity);
    const uint64_t e64 = b64 + a.tile_count[g];
    const uint32_t end = uint32_t(e64 < a.capacity ? e64 : a.capacity);
    const float cutoff = a.cutoff;
    float2 cr = bc(0.f), cg = bc(0.f), cb = bc(0.f), d = bc(0.f), acc = bc(0.f), T = bc(1.f);

    // Batches are double-buffered: the records of batch i+1 are copied global -> shared with
    // cp.async while batch i is blended; the list entries of batch i+2 are loaded meanwhile.
    uint32_t slot_next[kPerThread];
    auto load_slots = [&](uint32_t b) {
#pragma unroll
        for (int h = 0; h < kPerThread; ++h) {
            const uint32_t i = b + uint32_t(tid + h * kThreads);
            // in flight while the current batch blends: checked only when the copy is issued
            slot_next[h] = i < end ? __ldg(a.values + i) : 0xFFFFFFFFu;
        }
    };
    auto issue_copy = [&](int buf) {
#pragma unroll
        for (int h = 0; h < kPerThread; ++h) {
            // a stale slot is only possible in a clamped (overflowed) frame
            GSIM_DCHECK(slot_next[h] == 0xFFFFFFFFu || e64 > a.capacity || slot_next[h] < a.n_slots);
            if (slot_next[h] != 0xFFFFFFFFu && slot_next[h] >= a.n_slots) slot_next[h] = 0;
        }
        if constexpr (kBulk) {
            // every thread arrives once per phase, announcing the bytes of its own copies first
            uint32_t bytes = 0;
#pragma unroll
            for (int h = 0; h < kPerThread; ++h) bytes += slot_next[h] != 0xFFFFFFFFu ? 48u : 0u;
            const uint32_t bar = bar0 + 8u * uint32_t(buf);
            mbar_arrive_expect(bar, bytes);
            pending_bulk |= 1u << buf;
#pragma unroll
            for (int h = 0; h < kPerThread; ++h)
                if (slot_next[h] != 0xFFFFFFFFu)
                    bulk_copy(uint32_t(__cvta_generic_to_shared(&s_spl[buf][tid + h * kThreads])),
                              a.records + slot_next[h], 48u, bar);
            return;
        }
#pragma unroll
        for (int h = 0; h < kPerThread; ++h) {
            if (slot_next[h] != 0xFFFFFFFFu) {
                const char* src = reinterpret_cast<const char*>(a.records + slot_next[h]);
                const uint32_t dst = uint32_t(__cvta_generic_to_shared(&s_spl[buf][tid + h * kThreads]));
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * q),
                                 "l"(src + 16 * q) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    uint32_t fetched = 0;
    if (begin < end) {
        load_slots(begin);
        issue_copy(0);
        load_slots(begin + kBatch);
    }
    int buf = 0;
    for (uint32_t b0 = begin; b0 < end; b0 += kBatch, buf ^= 1) {
        const uint32_t n_b = (end - b0) < uint32_t(kBatch) ? (end - b0) : uint32_t(kBatch);
        if constexpr (kBulk) {
            mbar_wait(bar0 + 8u * uint32_t(buf), (phase_bits >> buf) & 1u);
            phase_bits ^= 1u << buf;
            pending_bulk &= ~(1u << buf);
        } else {
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        // One barrier per batch: it publishes the batch's records, frees batch i-1's buffer and
        // counts the pixels still compositing (the tile leaves once every pixel is done).
        if (__syncthreads_count(T.x < cutoff && T.y < cutoff ? 0 : 1) == 0) break;
        fetched += n_b;
        // every warp has left batch i-1, so its buffer takes batch i+1
        if (b0 + kBatch < end) {
            issue_copy(buf ^ 1);
            load_slots(b0 + 2 * kBatch);
        }

        if (!__all_sync(0xffffffffu, T.x < cutoff && T.y < cutoff)) {
            // Compact the splats that can reach this warp's still-compositing pixels (depth
            // order preserved) as shared-memory addresses of their records. The cull rectangle
            // is the bounding box of the warp's pixels with T >= cutoff: a finished pixel takes
            // no more weight, so splats that only reach finished pixels are dropped (results
            // unchanged, fewer blend steps near the end of a tile).
            const bool al0 = !(T.x < cutoff), al1 = !(T.y < cutoff);
            const int bx_lo = __reduce_min_sync(0xffffffffu, al0 ? x : (al1 ? x + 1 : INT_MAX));
            const int bx_hi = __reduce_max_sync(0xffffffffu, al1 ? x + 1 : (al0 ? x : INT_MIN));
            const int by_lo = __reduce_min_sync(0xffffffffu, (al0 || al1) ? y : INT_MAX);
            const int by_hi = __reduce_max_sync(0xffffffffu, (al0 || al1) ? y : INT_MIN);
            const float cx_lo = float(bx_lo) + 0.5f, cx_hi = float(bx_hi) + 0.5f;
            const float cy_lo = float(by_lo) + 0.5f, cy_hi = float(by_hi) + 0.5f;
            const Record* spl_buf = s_spl[buf];
            const uint32_t spl_addr = uint32_t(__cvta_generic_to_shared(spl_buf));
            uint32_t count = 0;
            bool bright = false;
            for (uint32_t j = 0; j < n_b; j += 32) {
                const uint32_t idx = j + lane;
                bool mine = false;
                float lop = -INFINITY;
                if (idx < n_b) {
                    const float4 p0 = spl_buf[idx].a;
                    const float rw = spl_buf[idx].c.w;
                    const __half2 reach = *reinterpret_cast<const __half2*>(&rw);
                    const float ex = __low2float(reach), ey = __high2float(reach);
                    mine = p0.x + ex >= cx_lo && p0.x - ex <= cx_hi && p0.y + ey >= cy_lo &&
                           p0.y - ey <= cy_hi;
                    if (a.exact_cull) mine = mine && reaches_rect(p0, spl_buf[idx].b, cx_lo, cx_hi, cy_lo, cy_hi);
                    lop = p0.w;
                }
                const uint32_t bits = __ballot_sync(0xffffffffu, mine);
                bright |= __any_sync(0xffffffffu, mine && !(lop <= kNoClampLog2));
                if (mine)
                    s_list[warp][count + __popc(bits & lanemask_lt())] =
                        spl_addr + idx * uint32_t(sizeof(Record));
                count += __popc(bits);
            }
            __syncwarp();
            if (bright)
                blend_list<true>(s_list[warp], count, npx, py, cutoff, cr, cg, cb, d, acc, T);
            else
                blend_list<false>(s_list[warp], count, npx, py, cutoff, cr, cg, cb, d, acc, T);
        }
    }
    // no copy may land after the CTA exits
    if constexpr (kBulk) {
        // a batch whose copies were issued but never waited for (early saturation exit)
        for (int bb = 0; bb < 2; ++bb)
            if (pending_bulk & (1u << bb)) mbar_wait(bar0 + 8u * uint32_t(bb), (phase_bits >> bb) & 1u);
    } else {
        asm volatile("cp.async.wait_all;" ::: "memory");
    }

    if (tid == 0 && fetched) atomicAdd(a.consumed, (unsigned long long)fetched);
    write_pixel(a, cam, x, y, cr.x, cg.x, cb.x, d.x, acc.x);
    write_pixel(a, cam, x + 1, y, cr.y, cg.y, cb.y, d.y, acc.y);
    __syncthreads();  // the next tile reuses the record buffers and lists
    if (!a.tile_ticket) break;  // one tile per CTA
    }
}

void launch_raster(const RasterArgs& a_in, uint32_t tile_end, cudaStream_t stream) {
    if (tile_end <= a_in.tile_begin) return;
    RasterArgs a = a_in;
    a.n_tiles = tile_end;
    uint32_t n_tiles = tile_end - a.tile_begin;
    const bool small = a.batch == 128;
    // capped grid: the CTAs loop over the tiles (leaves room on every SM for other contexts'
    // kernels); 0 = one CTA per tile
    if (a.grid_cap > 0 && uint32_t(a.grid_cap) < n_tiles) n_tiles = uint32_t(a.grid_cap);
    if (a.bulk_copy) {  // GSIM_GPU_RASTER_BULK=1 (A/B measurement)
        if (small) raster_kernel<8, 128, true><<<n_tiles, kThreads, 0, stream>>>(a);
        else raster_kernel<8, 256, true><<<n_tiles, kThreads, 0, stream>>>(a);
        return;
    }
    if (a.rect_w == 8) {
        if (small) raster_kernel<8, 128, false><<<n_tiles, kThreads, 0, stream>>>(a);
        else raster_kernel<8, 256, false><<<n_tiles, kThreads, 0, stream>>>(a);
    } else {
        if (small) raster_kernel<16, 128, false><<<n_tiles, kThreads, 0, stream>>>(a);
        else raster_kernel<16, 256, false><<<n_tiles, kThreads, 0, stream>>>(a);
    }
}

}  // namespace gsim_gpu

