// bin.cu — K3 after the depth sort: deterministic tile binning without a pair sort.
//
// The reference emits (tile << 32 | depth, splat) pairs and std::sorts them
// (raster.cpp:174-202). After the camera-major depth sort of the V visible records
// (sort.cu, which carries every record's tile rect through its passes into depth order), the pair
// order we need is simply "by (camera, tile), then by record order". Instead of radix-sorting
// the P ~ 3.5 V pairs by tile, every pair is placed directly:
//   units     the depth-sorted records of each camera are cut into units of R = 1024 * W
//             records; one W-warp CTA owns one unit, warp w its w-th 1024-record slice;
//   count     per unit, pairs per tile: every record adds +1 / -1 at both ends of each of its
//             rect rows in a shared row-difference array (red.shared), rows are then
//             prefix-summed (one thread per row); the row goes to a per-camera [unit][tile]
//             matrix;
//   colscan   per (camera, tile): exclusive scan over the camera's units (lanes = tiles,
//             warps = unit segments);
//   tilescan  per camera: exclusive scan of the tile totals -> tile ranges (raster.cpp:198-202);
//   campre    per batch: pair base of every camera;
//   scatter   per unit: each warp recounts its slice the same way, the CTA turns the counts
//             into per-warp first positions of every tile, and each warp walks its records in
//             order writing each pair's record slot at its position.
// Pairs are enumerated warp-cooperatively, 32 consecutive pairs per step in emission order
// (record order, row-major tiles inside a record, raster.cpp:190-194): the owner record of a
// pair position comes from one redux.sync.or of the records' start bits and a popc. The lanes
// of a step hitting the same tile come from one shared atomicOr of the lane bit into the
// tile's bitmap (match.any issues at ~1 per 40 SM cycles on sm_100 and is avoided); they are
// ranked by lane. Cameras with many tiles use a u8 last-writer probe instead (a quarter of the
// shared memory) and rank with ballots only when two lanes collide. The result equals the
// reference's stable (tile, depth, primitive) order bit for bit.
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t rect_area(uint32_t r) {
    return (((r >> 16) & 255u) - (r & 255u) + 1u) * ((r >> 24) - ((r >> 8) & 255u) + 1u);
}

// Per-warp scatter tables: u32 counters / positions per cell plus either a u32 lane bitmap
// (bitmap peers) or a u8 last-writer probe (large cameras: a quarter of the bytes).
constexpr int kSpare = 32;
__host__ __device__ inline size_t bin_warp_bytes(int max_cells, bool bitmap) {
    return bitmap ? size_t(max_cells) * 8 : (size_t(max_cells) * 5 + 15) & ~size_t(15);
}

struct Unit {
    int cam;
    uint32_t rec_begin, rec_end;  // depth-sorted record range
    uint32_t unit_in_cam, units_in_cam;
    uint64_t mbase;               // count-matrix base of the camera ([unit][tile])
    int tiles_x, tiles_y;
    uint32_t tc;                  // tiles of the camera
    uint32_t tile_base;
    int tbits;                    // bits of a camera-local tile id
};

__device__ __forceinline__ Unit unit_info(const BinArgs& a, uint32_t k) {
    Unit u;
    u.cam = int(a.chunk_cam[k]);
    const uint32_t cb = a.cam_chunk_base[u.cam];
    u.unit_in_cam = k - cb;
    u.units_in_cam = a.cam_chunk_base[u.cam + 1] - cb;
    const uint32_t vb = a.cam_vbase[u.cam], ve = a.cam_vbase[u.cam + 1];
    u.rec_begin = vb + u.unit_in_cam * uint32_t(a.chunk_records);
    u.rec_end = min(u.rec_begin + uint32_t(a.chunk_records), ve);
    u.mbase = a.cam_mbase[u.cam];
    u.tiles_x = a.cam_tiles_x[u.cam];
    u.tile_base = a.cam_tile_base[u.cam];
    u.tc = a.cam_tile_base[u.cam + 1] - u.tile_base;
    u.tiles_y = int(u.tc / uint32_t(u.tiles_x));
    u.tbits = u.tc > 1 ? 32 - __clz(int(u.tc - 1)) : 0;
    return u;
}

// Walk records [wb, we) in order, 32 per group (lane = record), kG groups per step; fn(slot,
// rect, valid) per group. The coalesced loads of the NEXT step are issued before the current
// step is processed, so their latency hides behind it (ncu: the loads of a step issued at its
// start were the scatter's top stall, long_scoreboard on a third of the samples).
template <bool kSlots, class F>
__device__ __forceinline__ void walk_groups(const BinArgs& a, uint32_t wb, uint32_t we, F&& fn) {
    constexpr int kG = 4;
    const int lane = threadIdx.x & 31;
    uint32_t slot[kG], rect[kG];
    auto load = [&](uint32_t g0, uint32_t* sl, uint32_t* rc) {
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            const uint32_t e = g0 + q * 32 + lane;
            rc[q] = e < we ? __ldcs(a.sorted_rects + e) : 0u;
            sl[q] = (kSlots && e < we) ? __ldcs(a.sorted_slots + e) : 0u;
        }
    };
    if (wb < we) load(wb, slot, rect);
    for (uint32_t g0 = wb; g0 < we; g0 += 32 * kG) {
        uint32_t nslot[kG], nrect[kG];
        const uint32_t g1 = g0 + 32 * kG;
        if (g1 < we) load(g1, nslot, nrect);
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            if (g0 + q * 32 >= we) break;
            fn(slot[q], rect[q], g0 + q * 32 + lane < we);
        }
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            slot[q] = nslot[q];
            rect[q] = nrect[q];
        }
    }
}

// walk_groups for the scatter: fn(slot, rect, valid, excl, total) also gets each lane's exclusive
// prefix of the rect areas over its 32-record group and the group's pair total. The prefix
// scans of the kG groups loaded together run interleaved (four independent shuffle chains
// instead of four chains back to back).
template <class F>
__device__ __forceinline__ void walk_groups_scanned(const BinArgs& a, uint32_t wb, uint32_t we, F&& fn) {
    constexpr int kG = 4;
    const int lane = threadIdx.x & 31;
    uint32_t slot[kG], rect[kG];
    auto load = [&](uint32_t g0, uint32_t* sl, uint32_t* rc) {
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            const uint32_t e = g0 + q * 32 + lane;
            rc[q] = e < we ? __ldcs(a.sorted_rects + e) : 0u;
            sl[q] = e < we ? __ldcs(a.sorted_slots + e) : 0u;
        }
    };
    if (wb < we) load(wb, slot, rect);
    for (uint32_t g0 = wb; g0 < we; g0 += 32 * kG) {
        uint32_t nslot[kG], nrect[kG];
        const uint32_t g1 = g0 + 32 * kG;
        if (g1 < we) load(g1, nslot, nrect);
        uint32_t cnt[kG], incl[kG];
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            cnt[q] = g0 + q * 32 + lane < we ? rect_area(rect[q]) : 0u;
            incl[q] = cnt[q];
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t[kG];
#pragma unroll
            for (int q = 0; q < kG; ++q) t[q] = __shfl_up_sync(kFull, incl[q], o);
#pragma unroll
            for (int q = 0; q < kG; ++q)
                if (lane >= o) incl[q] += t[q];
        }
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            if (g0 + q * 32 >= we) break;
            fn(slot[q], rect[q], g0 + q * 32 + lane < we, incl[q] - cnt[q],
               __shfl_sync(kFull, incl[q], 31));
        }
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            slot[q] = nslot[q];
            rect[q] = nrect[q];
        }
    }
}

// Row-difference counting: +1 at (ty, tx0) and -1 at (ty, tx1 + 1) for every rect row of every
// valid lane's record. D is [tiles_y][tiles_x + 1]; shared atomics (order is irrelevant here).
__device__ __forceinline__ void add_rect_rows(int* D, int wd, uint32_t r, bool valid) {
    if (!valid) return;
    const uint32_t tx0 = r & 255u, ty0 = (r >> 8) & 255u, tx1 = (r >> 16) & 255u, ty1 = r >> 24;
    for (uint32_t ty = ty0; ty <= ty1; ++ty) {
        GSIM_DCHECK(tx0 <= tx1 && tx1 + 1u < uint32_t(wd));
        atomicAdd(D + ty * uint32_t(wd) + tx0, 1);
        atomicAdd(D + ty * uint32_t(wd) + tx1 + 1u, -1);
    }
}

// In-place inclusive prefix of one tile row of n counters by one thread (rows of a table with
// an odd stride sit in distinct banks, so the lanes of a warp scanning neighbouring rows do not
// conflict); loads are batched 8 at a time so their latencies overlap.
__device__ __forceinline__ void scan_row_serial(int* row, int n) {
    int acc = 0, x = 0;
    for (; x + 8 <= n; x += 8) {
        int v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = row[x + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc += v[k];
            row[x + k] = acc;
        }
    }
    for (; x < n; ++x) {
        acc += row[x];
        row[x] = acc;
    }
}

__device__ __forceinline__ uint32_t reduce_or(uint32_t v) {
    uint32_t r;
    asm volatile("redux.sync.or.b32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}

}  // namespace

// ---- depth-key digit histograms per (camera, pass) ------------------------------------------
// Block b takes the contiguous slot range [b * per, (b + 1) * per) and walks it camera piece by
// camera piece (slots are camera-major): per-warp shared histograms of every pass's digit
// (shared atomics; their same-digit conflicts are mild because the keys are spread), summed over
// the warps and added to the camera's global histogram when the piece ends. The per-camera
// visible counts are the sums of the first pass's histogram (chunk_table).
__global__ void __launch_bounds__(kThreads) key_hist_kernel(BinArgs a) {
    extern __shared__ __align__(16) uint32_t s_hist[];  // [kWarps][passes][radix]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int radix = 1 << a.sort_bits, np = a.sort_passes, per_warp = np * radix;
    const uint32_t mask = uint32_t(radix - 1);
    uint32_t* wh = s_hist + warp * per_warp;
    const uint32_t n = uint32_t(a.n_slots);  // slot counts stay below 2^31
    constexpr int kKeys = 8;                 // keys per lane in flight: memory-level parallelism
    constexpr uint32_t kWarpSpan = 32u * kKeys;
    const uint32_t per = ((n + gridDim.x - 1) / gridDim.x + kWarpSpan - 1) / kWarpSpan * kWarpSpan;
    const uint32_t lo = min(n, blockIdx.x * per), hi = min(n, lo + per);
    if (lo >= hi) return;
    int c = upper_index(a.cam_slot_base, a.n_cams, uint64_t(lo));
    while (true) {
        while (c < a.n_cams && a.cam_slot_base[c + 1] <= lo) ++c;  // skip empty cameras
        GSIM_DCHECK(c >= 0);
        if (c >= a.n_cams || a.cam_slot_base[c] >= hi) break;
        const uint32_t plo = max(lo, uint32_t(a.cam_slot_base[c]));
        const uint32_t phi = min(hi, uint32_t(a.cam_slot_base[c + 1]));
        for (int k = threadIdx.x; k < kWarps * per_warp; k += kThreads) s_hist[k] = 0;
        __syncthreads();
        for (uint32_t w0 = plo + uint32_t(warp) * kWarpSpan; w0 < phi; w0 += kWarps * kWarpSpan) {
            uint32_t keys[kKeys];
            const uint32_t* kp = a.keys + w0 + lane;
#pragma unroll
            for (int i = 0; i < kKeys; ++i)
                keys[i] = w0 + lane + i * 32u < phi ? __ldcs(kp + i * 32) : kInvalidKey;
#pragma unroll
            for (int i = 0; i < kKeys; ++i) {
                if (keys[i] == kInvalidKey) continue;
                for (int p = 0; p < np; ++p)
                    atomicAdd(&wh[p * radix + ((keys[i] >> (p * a.sort_bits)) & mask)], 1u);
            }
        }
        __syncthreads();
        uint32_t* g = a.hist + uint64_t(c) * per_warp;
        uint32_t visible = 0;  // the piece's valid keys: sum of its first-pass digit counts
        for (int k = threadIdx.x; k < per_warp; k += kThreads) {
            uint32_t sum = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) sum += s_hist[w * per_warp + k];
            if (sum) atomicAdd(g + k, sum);
            if (k < radix) visible += sum;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) visible += __shfl_xor_sync(kFull, visible, o);
        if (lane == 0 && visible) atomicAdd(a.cam_visible + c, visible);
        __syncthreads();
        ++c;
    }
    (void)lane;
}

size_t key_hist_smem(const BinArgs& a) {
    return size_t(kWarps) * size_t(a.sort_passes) * (size_t(1) << a.sort_bits) * sizeof(uint32_t);
}

// Inclusive scan of one u64 per thread over the block (blockDim.x <= 1024) with warp shuffles:
// two barriers instead of a log-step shared-memory scan. *total = the block's sum.
__device__ unsigned long long block_scan_u64(unsigned long long v, unsigned long long* s_w,
                                             unsigned long long* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) s_w[warp] = v;
    __syncthreads();
    if (warp == 0) {
        unsigned long long x = lane < nw ? s_w[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += t;
        }
        if (lane < nw) s_w[lane] = x;
    }
    __syncthreads();
    if (warp > 0) v += s_w[warp - 1];
    *total = s_w[nw - 1];
    __syncthreads();
    return v;
}

// ---- per-camera unit tables (one block) -----------------------------------------------------
__global__ void __launch_bounds__(256) chunk_table_kernel(BinArgs a) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry[4];
    const int tid = threadIdx.x;
    if (tid < 4) s_carry[tid] = 0;
    __syncthreads();
    const uint32_t R = uint32_t(a.chunk_records);
    for (int c0 = 0; c0 < a.n_cams; c0 += blockDim.x) {
        const int c = c0 + tid;
        uint32_t v = 0;
        if (c < a.n_cams) v = a.cam_visible[c];  // V_c, counted by key_hist
        const uint32_t k = (v + R - 1) / R;
        const uint32_t ks = (v + uint32_t(kOnesweepTile) - 1) / uint32_t(kOnesweepTile);
        const uint32_t tc = c < a.n_cams ? a.cam_tile_base[c + 1] - a.cam_tile_base[c] : 0u;
        const unsigned long long m = (unsigned long long)k * tc;
        unsigned long long tv, tk, tm, ts;
        const unsigned long long iv = block_scan_u64(v, s_w, &tv);
        const unsigned long long ik = block_scan_u64(k, s_w, &tk);
        const unsigned long long im = block_scan_u64(m, s_w, &tm);
        const unsigned long long is = block_scan_u64(ks, s_w, &ts);
        if (c < a.n_cams) {
            a.cam_vbase[c] = uint32_t(s_carry[0] + iv - v);
            a.cam_chunk_base[c] = uint32_t(s_carry[1] + ik - k);
            a.cam_mbase[c] = s_carry[2] + im - m;
            a.sort_chunk_base[c] = uint32_t(s_carry[3] + is - ks);
        }
        __syncthreads();
        if (tid == 0) {
            s_carry[0] += tv;
            s_carry[1] += tk;
            s_carry[2] += tm;
            s_carry[3] += ts;
        }
        __syncthreads();
    }
    if (tid == 0) {
        a.cam_vbase[a.n_cams] = uint32_t(s_carry[0]);
        a.cam_chunk_base[a.n_cams] = uint32_t(s_carry[1]);
        a.cam_mbase[a.n_cams] = s_carry[2];
        a.sort_chunk_base[a.n_cams] = uint32_t(s_carry[3]);
        *a.n_chunks = uint32_t(s_carry[1]);
        a.totals[0] = s_carry[0];  // V
    }
    __syncthreads();
    const uint32_t K = uint32_t(s_carry[1]);
    for (uint32_t k = tid; k < K; k += blockDim.x)
        a.chunk_cam[k] = uint32_t(upper_index(a.cam_chunk_base, a.n_cams, k));
}

// ---- count: one CTA per unit ------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) bin_count_kernel(BinArgs a) {
    extern __shared__ __align__(16) char s_bin[];
    int* D = reinterpret_cast<int*>(s_bin);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t K = *a.n_chunks;
    for (uint32_t k = blockIdx.x; k < K; k += gridDim.x) {
        const Unit u = unit_info(a, k);
        const int wd = u.tiles_x + 1;
        for (int t = threadIdx.x; t < wd * u.tiles_y; t += blockDim.x) D[t] = 0;
        __syncthreads();
        const uint32_t wb = u.rec_begin + uint32_t(warp) * uint32_t(a.warp_records);
        walk_groups<false>(a, wb, min(wb + uint32_t(a.warp_records), u.rec_end),
                           [&](uint32_t, uint32_t r, bool valid) { add_rect_rows(D, wd, r, valid); });
        __syncthreads();
        uint32_t* mrow = a.counts + u.mbase + uint64_t(u.unit_in_cam) * u.tc;
        // row prefixes in place, one thread per tile row, then one coalesced copy of the rows
        for (int ty = threadIdx.x; ty < u.tiles_y; ty += blockDim.x) scan_row_serial(D + ty * wd, u.tiles_x);
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < u.tc; t += blockDim.x) {
            const uint32_t ty = t / uint32_t(u.tiles_x), tx = t - ty * uint32_t(u.tiles_x);
            mrow[t] = uint32_t(D[ty * uint32_t(wd) + tx]);
        }
        __syncthreads();
    }
    (void)lane;
    (void)warp;
    (void)nw;
}

// ---- column scan: lanes = 32 consecutive (camera, tile) columns, warps = 8 unit segments ------
// Each warp sums its segment of units for its lane's column (coalesced 128-byte rows of the
// [unit][tile] matrix), the block combines the 8 segment sums, and a second sweep writes the
// exclusive prefixes. A lane's column may belong to another camera than its neighbours'.
__global__ void __launch_bounds__(kThreads) bin_colscan_kernel(BinArgs a) {
    __shared__ uint32_t s_seg[kWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t n_cols = a.cam_tile_base[a.n_cams];
    const uint32_t g = blockIdx.x * 32 + lane;
    const bool in = g < n_cols;
    uint32_t* col = nullptr;
    uint32_t tc = 0, k_lo = 0, k_hi = 0;
    if (in) {
        const int c = upper_index(a.cam_tile_base, a.n_cams, g);
        tc = a.cam_tile_base[c + 1] - a.cam_tile_base[c];
        const uint32_t nk = a.cam_chunk_base[c + 1] - a.cam_chunk_base[c];
        col = a.counts + a.cam_mbase[c] + (g - a.cam_tile_base[c]);
        k_lo = uint32_t(uint64_t(nk) * warp / kWarps);
        k_hi = uint32_t(uint64_t(nk) * (warp + 1) / kWarps);
    }
    constexpr uint32_t kU = 4;  // loads in flight per lane
    uint32_t sum = 0;
    for (uint32_t k0 = k_lo; k0 < k_hi; k0 += kU) {
        uint32_t v[kU];
#pragma unroll
        for (uint32_t q = 0; q < kU; ++q) v[q] = k0 + q < k_hi ? col[uint64_t(k0 + q) * tc] : 0u;
#pragma unroll
        for (uint32_t q = 0; q < kU; ++q) sum += v[q];
    }
    s_seg[warp][lane] = sum;
    __syncthreads();
    uint32_t run = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t x = s_seg[w][lane];
        if (w < warp) run += x;
        total += x;
    }
    if (in && warp == 0) a.tile_count[g] = total;
    for (uint32_t k0 = k_lo; k0 < k_hi; k0 += kU) {
        uint32_t v[kU];
#pragma unroll
        for (uint32_t q = 0; q < kU; ++q) v[q] = k0 + q < k_hi ? col[uint64_t(k0 + q) * tc] : 0u;
#pragma unroll
        for (uint32_t q = 0; q < kU; ++q) {
            if (k0 + q < k_hi) col[uint64_t(k0 + q) * tc] = run;
            run += v[q];
        }
    }
}

// ---- tile scan: one block per camera -----------------------------------------------------------
__global__ void __launch_bounds__(1024) bin_tilescan_kernel(BinArgs a) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int c = blockIdx.x; c < a.n_cams; c += gridDim.x) {
        const uint32_t tb = a.cam_tile_base[c], tc = a.cam_tile_base[c + 1] - tb;
        if (tid == 0) s_carry = 0;
        __syncthreads();
        for (uint32_t t0 = 0; t0 < tc; t0 += 1024) {
            const uint32_t t = t0 + tid;
            const uint32_t v = t < tc ? a.tile_count[tb + t] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t s = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += s;
            }
            if (lane == 31) s_warp[warp] = incl;
            __syncthreads();
            uint32_t wp = 0, tot = 0;
            for (int w = 0; w < 32; ++w) {
                const uint32_t s = s_warp[w];
                if (w < warp) wp += s;
                tot += s;
            }
            if (t < tc) a.tile_rel[tb + t] = s_carry + wp + incl - v;
            __syncthreads();
            if (tid == 0) s_carry += tot;
            __syncthreads();
        }
        if (tid == 0) a.cam_pairs[c] = s_carry;
        __syncthreads();
    }
}

// ---- camera pair bases (one block) -------------------------------------------------------------
__global__ void __launch_bounds__(256) bin_campre_kernel(BinArgs a) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry;
    const int tid = threadIdx.x;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int c0 = 0; c0 < a.n_cams; c0 += blockDim.x) {
        const int c = c0 + tid;
        const unsigned long long v = c < a.n_cams ? a.cam_pairs[c] : 0ull;
        unsigned long long tot;
        const unsigned long long inc = block_scan_u64(v, s_w, &tot);
        if (c < a.n_cams) a.cam_pair_base[c] = s_carry + inc - v;
        __syncthreads();
        if (tid == 0) s_carry += tot;
        __syncthreads();
    }
    if (tid == 0) {
        a.cam_pair_base[a.n_cams] = s_carry;
        a.totals[1] = s_carry;  // P
        if (a.host_totals) {  // read by the host after the frame's binning event
            a.host_totals[0] = a.totals[0];
            a.host_totals[1] = s_carry;
        }
    }
}

// ---- scatter: one CTA per unit ----------------------------------------------------------------
// Shared memory per warp: [tiles_y][tiles_x + 1] u32 counters, turned into first positions, and
// a u32 lane bitmap per cell (bin_warp_bytes).
template <bool kBitmap>
__global__ void __launch_bounds__(kThreads) bin_scatter_kernel(BinArgs a) {
    extern __shared__ __align__(16) char s_bin[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // kSpare extra cells per table, one per lane, take the lanes of a step that have no pair,
    // so every lane runs the same shared-memory sequence without branches
    const int cells = a.max_tc + kSpare;
    const size_t wbytes = bin_warp_bytes(cells, kBitmap);
    uint32_t* pos = reinterpret_cast<uint32_t*>(s_bin + warp * wbytes);
    uint32_t* peer_bits = pos + cells;
    uint8_t* probe = reinterpret_cast<uint8_t*>(pos + cells);
    // row-major position -> (row, column) with a magic reciprocal per rect width: for
    // kk < 2^16 and width w <= 256, umulhi(kk, 0xFFFFFFFF / w + 1) == kk / w exactly.
    __shared__ uint32_t s_magic[257];
    for (int w = threadIdx.x; w <= 256; w += blockDim.x) s_magic[w] = w > 1 ? 0xFFFFFFFFu / uint32_t(w) + 1u : 0u;
    // the lane bitmaps are cleared once over the batch's largest grid; every placement step
    // leaves them cleared, so units of any camera (a block may take several) start clean
    if (kBitmap)
        for (int t = lane; t < cells; t += 32) peer_bits[t] = 0u;
    __syncthreads();
    const uint32_t K = *a.n_chunks;
    // pair positions are 32-bit; a capacity beyond that bounds nothing
    const uint32_t cap32 = a.capacity < 0xFFFFFFFFull ? uint32_t(a.capacity) : 0xFFFFFFFFu;
    for (uint32_t k = blockIdx.x; k < K; k += gridDim.x) {
        const Unit u = unit_info(a, k);
        const int wd = u.tiles_x + 1;
        const uint32_t wb = u.rec_begin + uint32_t(warp) * uint32_t(a.warp_records);
        const uint32_t we = min(wb + uint32_t(a.warp_records), u.rec_end);
        // 1. this warp's pairs per tile (row differences, then row scans in place)
        int* D = reinterpret_cast<int*>(pos);
        for (int t = lane; t < wd * u.tiles_y; t += 32) D[t] = 0;
        __syncwarp();
        walk_groups<false>(a, wb, we, [&](uint32_t, uint32_t r, bool valid) { add_rect_rows(D, wd, r, valid); });
        __syncwarp();
        // row prefixes with one lane per tile row: independent per-lane chains, no shuffles
        for (int ty = lane; ty < u.tiles_y; ty += 32) scan_row_serial(D + ty * wd, u.tiles_x);
        __syncthreads();
        // 2. first position of every tile for every warp: camera base + tile base + units
        //    before this one + warps before this one
        const uint32_t pbase = uint32_t(a.cam_pair_base[u.cam]);
        const uint32_t* mrow = a.counts + u.mbase + uint64_t(u.unit_in_cam) * u.tc;
        // four tiles per thread per round, their global loads issued together
        for (uint32_t t0 = threadIdx.x; t0 < u.tc; t0 += 4 * blockDim.x) {
            uint32_t base[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const uint32_t t = t0 + h * blockDim.x;
                base[h] = t < u.tc ? pbase + a.tile_rel[u.tile_base + t] + mrow[t] : 0u;
            }
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const uint32_t t = t0 + h * blockDim.x;
                if (t >= u.tc) break;
                const uint32_t ty = t / uint32_t(u.tiles_x), tx = t - ty * uint32_t(u.tiles_x);
                const uint32_t cell = ty * uint32_t(wd) + tx;
                uint32_t b = base[h];
                for (int w = 0; w < nw; ++w) {
                    uint32_t* pw = reinterpret_cast<uint32_t*>(s_bin + w * wbytes);
                    const uint32_t c = pw[cell];
                    pw[cell] = b;
                    b += c;
                }
            }
        }
        __syncthreads();
        // 3. place this warp's pairs in emission order
        walk_groups_scanned(a, wb, we, [&](uint32_t slot, uint32_t r, bool valid, uint32_t excl,
                                           uint32_t total) {
            const uint32_t cnt = valid ? rect_area(r) : 0u;
            const uint32_t magic = s_magic[((r >> 16) & 255u) - (r & 255u) + 1u];
            const uint32_t lanemask_le = lanemask_lt() | (1u << lane);
            int started = 0;  // records whose pair range starts before this step
            for (uint32_t s0 = 0; s0 < total; s0 += 32) {
                const bool starts = cnt != 0u && excl >= s0 && excl < s0 + 32u;
                const uint32_t M = reduce_or(starts ? 1u << (excl - s0) : 0u);
                const uint32_t j = s0 + uint32_t(lane);
                const bool in = j < total;
                int own = started + __popc(M & lanemask_le) - 1;
                own = own < 0 ? 0 : own;
                started += __popc(M);
                const uint32_t o_ex = __shfl_sync(kFull, excl, own);
                const uint32_t ro = __shfl_sync(kFull, r, own);
                const uint32_t sl = __shfl_sync(kFull, slot, own);
                const uint32_t mg = __shfl_sync(kFull, magic, own);
                const uint32_t kk = j - o_ex;
                const uint32_t tx0 = ro & 255u, ty0 = (ro >> 8) & 255u, tx1 = (ro >> 16) & 255u;
                const uint32_t w = tx1 - tx0 + 1u;
                const uint32_t q = mg ? __umulhi(kk, mg) : kk;
                const uint32_t cell = (ty0 + q) * uint32_t(wd) + tx0 + (kk - q * w);
                GSIM_DCHECK(!in || (cell < uint32_t(wd) * uint32_t(u.tiles_y) && ty0 + q <= (ro >> 24)));
                if (kBitmap) {
                    // lanes of this step on the same cell, from one atomicOr into the cell's
                    // bitmap; ranked by lane (= emission) order, the lowest lane bumps the
                    // position and clears the bitmap
                    // Every lane reads the cell's position together with the bitmap (same-address
                    // reads broadcast), so no shuffle from the leader sits on the chain; the
                    // leader's update follows a warp barrier that orders it after all reads.
                    const uint32_t c = in ? cell : uint32_t(a.max_tc + lane);  // spare: alone
                    atomicOr(&peer_bits[c], 1u << lane);
                    __syncwarp();
                    const uint32_t peers = peer_bits[c];
                    const uint32_t pre = pos[c];
                    const uint32_t below = peers & lanemask_lt();
                    __syncwarp();
                    if (below == 0) {
                        pos[c] = pre + __popc(peers);
                        peer_bits[c] = 0u;
                    }
                    const uint32_t p = pre + __popc(below);
                    if (in && p < cap32) a.vals_out[p] = sl;
                } else {
                    // last-writer probe: did another lane of this step write the same cell?
                    const uint32_t c = in ? cell : uint32_t(a.max_tc + lane);  // spare: alone
                    probe[c] = uint8_t(lane);
                    __syncwarp();
                    const bool lost = probe[c] != uint8_t(lane);
                    if (!__any_sync(kFull, lost)) {
                        const uint32_t p = pos[c];
                        pos[c] = p + 1u;
                        if (in && p < cap32) a.vals_out[p] = sl;
                    } else {  // rank the lanes of each cell by lane order from ballots
                        const uint32_t m = __ballot_sync(kFull, in);
                        const uint32_t tile = (ty0 + q) * uint32_t(u.tiles_x) + tx0 + (kk - q * w);
                        const uint32_t peers = peers_of_bits(kFull, tile, u.tbits) & m;
                        const uint32_t below = peers & lanemask_lt();
                        const uint32_t pre = in ? pos[cell] : 0u;
                        __syncwarp();
                        if (in) {
                            if (below == 0) pos[cell] = pre + __popc(peers);
                            const uint32_t p = pre + __popc(below);
                            if (p < cap32) a.vals_out[p] = sl;
                        }
                    }
                }
                __syncwarp();
            }
        });
        __syncthreads();
    }
}

// ---- launchers ---------------------------------------------------------------------------------
void launch_key_hist(const BinArgs& a, int grid, cudaStream_t s) {
    const size_t smem = key_hist_smem(a);
    cudaFuncSetAttribute(key_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    key_hist_kernel<<<grid, kThreads, smem, s>>>(a);
}
void launch_chunk_table(const BinArgs& a, cudaStream_t s) { chunk_table_kernel<<<1, 256, 0, s>>>(a); }
size_t bin_smem_bytes(const BinArgs& a) {
    return size_t(a.bin_warps) * bin_warp_bytes(a.max_tc + kSpare, a.bitmap_peers != 0);
}
void launch_bin_count(const BinArgs& a, int grid, cudaStream_t s) {
    const size_t smem = size_t(a.max_tc) * sizeof(int);
    cudaFuncSetAttribute(bin_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    bin_count_kernel<<<grid, 32 * a.bin_warps, smem, s>>>(a);
}
void launch_bin_colscan(const BinArgs& a, int grid, cudaStream_t s) {
    bin_colscan_kernel<<<grid, kThreads, 0, s>>>(a);
}
void launch_bin_tilescan(const BinArgs& a, int grid, cudaStream_t s) {
    bin_tilescan_kernel<<<grid, 1024, 0, s>>>(a);
}
void launch_bin_campre(const BinArgs& a, cudaStream_t s) { bin_campre_kernel<<<1, 256, 0, s>>>(a); }
void launch_bin_scatter(const BinArgs& a, int grid, cudaStream_t s) {
    const size_t smem = bin_smem_bytes(a);
    if (a.bitmap_peers) {
        cudaFuncSetAttribute(bin_scatter_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        bin_scatter_kernel<true><<<grid, 32 * a.bin_warps, smem, s>>>(a);
    } else {
        cudaFuncSetAttribute(bin_scatter_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        bin_scatter_kernel<false><<<grid, 32 * a.bin_warps, smem, s>>>(a);
    }
}

}  // namespace gsim_gpu
