// bin.cu — K3 after the depth sort: deterministic tile binning without a pair sort.
//
// The reference emits (tile << 32 | depth, splat) pairs and std::sorts them
// (raster.cpp:243-271). After the camera-major depth sort of the V visible records
// (sort.cu), the pair order we need is simply "by (camera, tile), then by record order".
// Instead of radix-sorting the P ~ 3.5 V pairs by tile, every pair is placed directly:
//   units     the depth-sorted records of each camera are cut into units of R records; one
//             warp owns one unit (no block-level cooperation, no barriers);
//   count     per unit, count pairs per tile into a warp-private counter array and store the
//             row into a per-camera [tile][unit] count matrix;
//   colscan   per (camera, tile): exclusive scan over the camera's units;
//   tilescan  per camera: exclusive scan of the tile totals -> tile ranges (raster.cpp:267-271);
//   campre    per batch: pair base of every camera;
//   scatter   per unit: load the unit's first position of every tile, walk the records again
//             in order and write each pair's record slot at its position.
// Pairs are enumerated warp-cooperatively, 32 consecutive pairs per step in emission order
// (record order, row-major tiles inside a record, raster.cpp:259-263). Two lanes of a step
// hitting the same tile is detected with a shared-memory "last writer" probe; only then are
// the tile's lanes ranked with ballots (match.any issues at ~1 per 40 SM cycles on sm_100,
// shared atomics at 2 cycles per lane: both measured, both avoided). The result equals the
// reference's stable (tile, depth, primitive) order bit for bit.
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t key_camera(uint32_t key, int depth_bits) {
    return depth_bits >= 32 ? 0u : (key >> depth_bits);
}

__device__ __forceinline__ uint32_t rect_area(uint32_t r) {
    return (((r >> 16) & 255u) - (r & 255u) + 1u) * ((r >> 24) - ((r >> 8) & 255u) + 1u);
}

// Warp-cooperative enumeration of the pairs of 32 records (one per lane): calls
// fn(in, tile, slot) once per step; lane j of a step holds the step's j-th pair.
template <class F>
__device__ __forceinline__ void for_each_pair(uint32_t slot, uint32_t rect, bool valid,
                                              int tiles_x, F&& fn) {
    const int lane = threadIdx.x & 31;
    const uint32_t cnt = valid ? rect_area(rect) : 0u;
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    const uint32_t excl = incl - cnt;
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    // row-major position -> (row, column) with a per-record magic reciprocal: for kk < 2^16
    // and width w <= 256, umulhi(kk, 0xFFFFFFFF / w + 1) == kk / w exactly.
    const uint32_t w_own = ((rect >> 16) & 255u) - (rect & 255u) + 1u;
    const uint32_t magic = w_own > 1u ? 0xFFFFFFFFu / w_own + 1u : 0u;
    for (uint32_t k0 = 0; k0 < total; k0 += 32) {
        const uint32_t j = k0 + lane;
        // owner = last lane whose exclusive offset <= j (valid lanes have cnt >= 1)
        int lo = 0;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
            const uint32_t oc = __shfl_sync(kFull, excl, (lo + s) & 31);
            if (lo + s < 32 && oc <= j) lo += s;
        }
        const uint32_t o_own = __shfl_sync(kFull, excl, lo);
        const uint32_t r = __shfl_sync(kFull, rect, lo);
        const uint32_t sl = __shfl_sync(kFull, slot, lo);
        const uint32_t mg = __shfl_sync(kFull, magic, lo);
        const bool in = j < total;
        const uint32_t kk = j - o_own;
        const uint32_t tx0 = r & 255u, ty0 = (r >> 8) & 255u, tx1 = (r >> 16) & 255u;
        const uint32_t w = tx1 - tx0 + 1u;
        const uint32_t q = mg ? __umulhi(kk, mg) : kk;
        const uint32_t tile = (ty0 + q) * uint32_t(tiles_x) + tx0 + (kk - q * w);
        fn(in, tile, sl);
    }
}

// Walk records [wb, we) of the depth-sorted list in order, 32 per group, with the slot and
// rect loads of kG groups issued together (latency hiding), calling for_each_pair per group.
template <class F>
__device__ __forceinline__ void walk_records(const BinArgs& a, uint32_t wb, uint32_t we,
                                             int tiles_x, F&& fn) {
    constexpr int kG = 4;
    const int lane = threadIdx.x & 31;
    for (uint32_t g0 = wb; g0 < we; g0 += 32 * kG) {
        uint32_t slot[kG], rect[kG];
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            const uint32_t e = g0 + q * 32 + lane;
            slot[q] = e < we ? __ldcs(a.sorted_slots + e) : 0u;
        }
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            const uint32_t e = g0 + q * 32 + lane;
            rect[q] = e < we ? __ldg(a.rects + slot[q]) : 0u;
        }
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            if (g0 + q * 32 >= we) break;
            for_each_pair(slot[q], rect[q], g0 + q * 32 + lane < we, tiles_x, fn);
        }
    }
}

// Lanes of `in_mask` whose tile equals this lane's, ordered by lane = emission order.
// Fast path: every lane writes its lane id to probe[tile], then reads it back; if no lane
// lost the write, all tiles in the step are distinct and each lane is its own only peer.
__device__ __forceinline__ uint32_t tile_peers(uint8_t* probe, uint32_t tile, bool in,
                                               uint32_t in_mask, int tbits) {
    const int lane = threadIdx.x & 31;
    if (in) probe[tile] = uint8_t(lane);
    __syncwarp();
    const bool lost = in && probe[tile] != uint8_t(lane);
    const bool any_conflict = __any_sync(kFull, lost);
    __syncwarp();
    if (!any_conflict) return in ? (1u << lane) : 0u;
    return peers_of_bits(kFull, tile, tbits) & in_mask;
}

struct Unit {
    int cam;
    uint32_t rec_begin, rec_end;  // depth-sorted record range
    uint32_t unit_in_cam, units_in_cam;
    uint64_t mbase;               // count-matrix base of the camera ([tile][unit])
    int tiles_x;
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
    u.tbits = u.tc > 1 ? 32 - __clz(int(u.tc - 1)) : 0;
    return u;
}

// Warp w of the block works in s_bin + w * per_warp_bytes: [max_tc] u32 + [max_tc] u8 probe.
constexpr int kTab = 512;  // pairs of one 32-record group held in a shared-memory table

__host__ __device__ inline size_t bin_warp_bytes(int max_cells) {
    return (size_t(max_cells) * 5 + size_t(kTab) * 3 + 15) & ~size_t(15);
}

// Warp w of the block works in s_bin + w * bin_warp_bytes: [max_cells] u32 counters,
// [max_cells] u8 probe, [kTab] u16 tile table, [kTab] u8 owner table.
__device__ __forceinline__ uint32_t* warp_counters(char* s_bin, int max_cells) {
    return reinterpret_cast<uint32_t*>(s_bin + (threadIdx.x >> 5) * bin_warp_bytes(max_cells));
}

// Walk records [wb, we) in order, 32 per group (lane = record), loads of kG groups in flight.
template <class F>
__device__ __forceinline__ void walk_groups(const BinArgs& a, uint32_t wb, uint32_t we, F&& fn) {
    constexpr int kG = 4;
    const int lane = threadIdx.x & 31;
    for (uint32_t g0 = wb; g0 < we; g0 += 32 * kG) {
        uint32_t slot[kG], rect[kG];
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            const uint32_t e = g0 + q * 32 + lane;
            slot[q] = e < we ? __ldcs(a.sorted_slots + e) : 0u;
        }
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            const uint32_t e = g0 + q * 32 + lane;
            rect[q] = e < we ? __ldg(a.rects + slot[q]) : 0u;
        }
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            if (g0 + q * 32 >= we) break;
            fn(slot[q], rect[q], g0 + q * 32 + lane < we);
        }
    }
}

// D[cell] += delta for every active lane; lanes that share a cell in the same call are
// applied in rounds (a shared-memory last-writer probe picks one winner per cell per round).
__device__ __forceinline__ void add_cells(int* D, uint8_t* probe, uint32_t cell, int delta,
                                          bool active) {
    const int lane = threadIdx.x & 31;
    bool pending = active;
    while (__any_sync(kFull, pending)) {
        if (pending) probe[cell] = uint8_t(lane);
        __syncwarp();
        const bool win = pending && probe[cell] == uint8_t(lane);
        __syncwarp();
        if (win) {
            D[cell] += delta;
            pending = false;
        }
        __syncwarp();
    }
}

}  // namespace

// ---- depth-key histograms + per-camera record counts ---------------------------------------
__global__ void __launch_bounds__(kThreads) key_hist_kernel(BinArgs a) {
    __shared__ uint32_t s_hist[kWarps][4][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < kWarps * 4 * 256; k += kThreads) (&s_hist[0][0][0])[k] = 0;
    __syncthreads();
    const uint64_t n = a.n_slots;
    constexpr int kKeys = 16;  // keys per lane in flight: memory-level parallelism
    const uint64_t stride = uint64_t(gridDim.x) * kThreads * kKeys;
    for (uint64_t base = (uint64_t(blockIdx.x) * kWarps + warp) * 32 * kKeys; base < n; base += stride) {
        uint32_t keys[kKeys];
#pragma unroll
        for (int i = 0; i < kKeys; ++i) {
            const uint64_t idx = base + uint64_t(i) * 32 + lane;
            keys[i] = idx < n ? __ldcs(a.keys + idx) : kInvalidKey;
        }
        uint32_t cam_run = 0xFFFFFFFFu, cam_cnt = 0;  // lane 0 accumulates runs of one camera
#pragma unroll
        for (int i = 0; i < kKeys; ++i) {
            const uint32_t key = keys[i];
            const bool valid = key != kInvalidKey;
            const uint32_t vmask = __ballot_sync(kFull, valid);
            if (a.hist) {  // digit histograms (only the onesweep variant needs them)
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const uint32_t d = (key >> (8 * p)) & 255u;
                    const uint32_t peers = peers_of<8>(kFull, d) & vmask;
                    if (valid && (peers & lanemask_lt()) == 0) s_hist[warp][p][d] += __popc(peers);
                }
            }
            // per-camera counts: one round per distinct camera in the group (usually one)
            const uint32_t cam = key_camera(key, a.depth_bits);
            uint32_t rem = vmask;
            while (rem) {
                const int leader = __ffs(rem) - 1;
                const uint32_t c = __shfl_sync(kFull, cam, leader);
                const uint32_t same = __ballot_sync(kFull, cam == c) & rem;
                if (c == cam_run) {
                    cam_cnt += __popc(same);
                } else {
                    if (lane == 0 && cam_cnt) atomicAdd(a.cam_visible + cam_run, cam_cnt);
                    cam_run = c;
                    cam_cnt = __popc(same);
                }
                rem &= ~same;
            }
        }
        if (lane == 0 && cam_cnt) atomicAdd(a.cam_visible + cam_run, cam_cnt);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 4 * 256; k += kThreads) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += (&s_hist[w][0][0])[k];
        if (s && a.hist) atomicAdd(a.hist + k, s);
    }
}

// ---- per-camera unit tables (one block) -----------------------------------------------------
__global__ void __launch_bounds__(1024) chunk_table_kernel(BinArgs a) {
    __shared__ unsigned long long s_scan[1024];
    __shared__ unsigned long long s_carry[3];
    const int tid = threadIdx.x;
    if (tid < 3) s_carry[tid] = 0;
    __syncthreads();
    const uint32_t R = uint32_t(a.chunk_records);
    auto scan = [&](unsigned long long v) {  // inclusive block scan
        s_scan[tid] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const unsigned long long t = tid >= o ? s_scan[tid - o] : 0ull;
            __syncthreads();
            s_scan[tid] += t;
            __syncthreads();
        }
        const unsigned long long r = s_scan[tid];
        __syncthreads();
        return r;
    };
    for (int c0 = 0; c0 < a.n_cams; c0 += 1024) {
        const int c = c0 + tid;
        const uint32_t v = c < a.n_cams ? a.cam_visible[c] : 0u;
        const uint32_t k = (v + R - 1) / R;
        const uint32_t tc = c < a.n_cams ? a.cam_tile_base[c + 1] - a.cam_tile_base[c] : 0u;
        const unsigned long long m = (unsigned long long)k * tc;
        const unsigned long long iv = scan(v), ik = scan(k), im = scan(m);
        if (c < a.n_cams) {
            a.cam_vbase[c] = uint32_t(s_carry[0] + iv - v);
            a.cam_chunk_base[c] = uint32_t(s_carry[1] + ik - k);
            a.cam_mbase[c] = s_carry[2] + im - m;
        }
        __syncthreads();
        if (tid == 1023) {
            s_carry[0] += iv;
            s_carry[1] += ik;
            s_carry[2] += im;
        }
        __syncthreads();
    }
    if (tid == 0) {
        a.cam_vbase[a.n_cams] = uint32_t(s_carry[0]);
        a.cam_chunk_base[a.n_cams] = uint32_t(s_carry[1]);
        a.cam_mbase[a.n_cams] = s_carry[2];
        *a.n_chunks = uint32_t(s_carry[1]);
        a.totals[0] = s_carry[0];  // V
    }
    __syncthreads();
    const uint32_t K = uint32_t(s_carry[1]);
    for (uint32_t k = tid; k < K; k += 1024)
        a.chunk_cam[k] = uint32_t(upper_index(a.cam_chunk_base, a.n_cams, k));
}

// ---- count: one warp per unit ------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) bin_count_kernel(BinArgs a) {
    extern __shared__ __align__(16) char s_bin[];
    const int lane = threadIdx.x & 31;
    if ((threadIdx.x >> 5) >= a.bin_warps) return;
    // Pairs per tile of a unit without enumerating pairs: every record adds +1 over its tile
    // rectangle, written as 4 corner updates of a 2-D difference array, then a 2-D prefix sum.
    int* D = reinterpret_cast<int*>(warp_counters(s_bin, a.max_tc));
    uint8_t* probe = reinterpret_cast<uint8_t*>(D + a.max_tc);
    const uint32_t K = *a.n_chunks;
    const uint32_t n_warps = gridDim.x * uint32_t(a.bin_warps);
    for (uint32_t k = blockIdx.x * a.bin_warps + (threadIdx.x >> 5); k < K; k += n_warps) {
        const Unit u = unit_info(a, k);
        const uint32_t W = uint32_t(u.tiles_x) + 1u, tiles_y = u.tc / uint32_t(u.tiles_x);
        const uint32_t H = tiles_y + 1u;
        for (uint32_t t = lane; t < W * H; t += 32) D[t] = 0;
        __syncwarp();
        walk_groups(a, u.rec_begin, u.rec_end, [&](uint32_t, uint32_t r, bool valid) {
            const uint32_t tx0 = r & 255u, ty0 = (r >> 8) & 255u;
            const uint32_t tx1 = ((r >> 16) & 255u) + 1u, ty1 = (r >> 24) + 1u;
            add_cells(D, probe, ty0 * W + tx0, 1, valid);
            add_cells(D, probe, ty0 * W + tx1, -1, valid);
            add_cells(D, probe, ty1 * W + tx0, -1, valid);
            add_cells(D, probe, ty1 * W + tx1, 1, valid);
        });
        for (uint32_t y = lane; y < H; y += 32) {
            int run = 0;
            for (uint32_t x = 0; x < W; ++x) {
                run += D[y * W + x];
                D[y * W + x] = run;
            }
        }
        __syncwarp();
        for (uint32_t x = lane; x < W; x += 32) {
            int run = 0;
            for (uint32_t y = 0; y < H; ++y) {
                run += D[y * W + x];
                D[y * W + x] = run;
            }
        }
        __syncwarp();
        uint32_t* col = a.counts + u.mbase + u.unit_in_cam;
        for (uint32_t t = lane; t < u.tc; t += 32) {
            const uint32_t ty = t / uint32_t(u.tiles_x), tx = t - ty * uint32_t(u.tiles_x);
            col[uint64_t(t) * u.units_in_cam] = uint32_t(D[ty * W + tx]);
        }
        __syncwarp();
    }
}

// ---- column scan: one warp per (camera, tile) --------------------------------------------------
__global__ void __launch_bounds__(kThreads) bin_colscan_kernel(BinArgs a) {
    const int lane = threadIdx.x & 31;
    const uint32_t n_cols = a.cam_tile_base[a.n_cams];
    for (uint32_t g = (blockIdx.x * kThreads + threadIdx.x) >> 5; g < n_cols;
         g += (gridDim.x * kThreads) >> 5) {
        const int c = upper_index(a.cam_tile_base, a.n_cams, g);
        const uint32_t t = g - a.cam_tile_base[c];
        const uint32_t nk = a.cam_chunk_base[c + 1] - a.cam_chunk_base[c];
        uint32_t* col = a.counts + a.cam_mbase[c] + uint64_t(t) * nk;
        uint32_t run = 0;
        for (uint32_t k0 = 0; k0 < nk; k0 += 32) {
            const uint32_t k = k0 + lane;
            const uint32_t v = k < nk ? col[k] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t s = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += s;
            }
            if (k < nk) col[k] = run + incl - v;
            run += __shfl_sync(kFull, incl, 31);
        }
        if (lane == 0) a.tile_count[g] = run;
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
__global__ void __launch_bounds__(1024) bin_campre_kernel(BinArgs a) {
    __shared__ unsigned long long s_m[1024];
    __shared__ unsigned long long s_carry;
    const int tid = threadIdx.x;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int c0 = 0; c0 < a.n_cams; c0 += 1024) {
        const int c = c0 + tid;
        const unsigned long long v = c < a.n_cams ? a.cam_pairs[c] : 0ull;
        s_m[tid] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const unsigned long long t = tid >= o ? s_m[tid - o] : 0ull;
            __syncthreads();
            s_m[tid] += t;
            __syncthreads();
        }
        if (c < a.n_cams) a.cam_pair_base[c] = s_carry + s_m[tid] - v;
        __syncthreads();
        if (tid == 1023) s_carry += s_m[1023];
        __syncthreads();
    }
    if (tid == 0) {
        a.cam_pair_base[a.n_cams] = s_carry;
        a.totals[1] = s_carry;  // P
    }
}

// ---- scatter: one warp per unit ----------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) bin_scatter_kernel(BinArgs a) {
    extern __shared__ __align__(16) char s_bin[];
    const int lane = threadIdx.x & 31;
    if ((threadIdx.x >> 5) >= a.bin_warps) return;
    uint32_t* pos = warp_counters(s_bin, a.max_tc);
    uint8_t* probe = reinterpret_cast<uint8_t*>(pos + a.max_tc);
    uint16_t* tab_tile = reinterpret_cast<uint16_t*>(probe + ((a.max_tc + 1) & ~1));
    uint8_t* tab_own = reinterpret_cast<uint8_t*>(tab_tile + kTab);
    const uint32_t K = *a.n_chunks;
    const uint32_t n_warps = gridDim.x * uint32_t(a.bin_warps);
    for (uint32_t k = blockIdx.x * a.bin_warps + (threadIdx.x >> 5); k < K; k += n_warps) {
        const Unit u = unit_info(a, k);
        // first position of every tile of this unit in the final list
        const uint32_t pbase = uint32_t(a.cam_pair_base[u.cam]);
        const uint32_t* col = a.counts + u.mbase + u.unit_in_cam;
        for (uint32_t t = lane; t < u.tc; t += 32)
            pos[t] = pbase + a.tile_rel[u.tile_base + t] + col[uint64_t(t) * u.units_in_cam];
        __syncwarp();
        auto place = [&](bool in, uint32_t tile, uint32_t sl) {
            const uint32_t m = __ballot_sync(kFull, in);
            const uint32_t peers = tile_peers(probe, tile, in, m, u.tbits);
            const uint32_t below = peers & lanemask_lt();
            const uint32_t pre = in ? pos[tile] : 0u;
            __syncwarp();
            if (in) {
                if (below == 0) pos[tile] = pre + __popc(peers);
                const uint32_t p = pre + __popc(below);
                if (p < a.capacity) a.vals_out[p] = sl;
            }
            __syncwarp();
        };
        walk_groups(a, u.rec_begin, u.rec_end, [&](uint32_t slot, uint32_t r, bool valid) {
            // exclusive offsets of the group's pairs in emission order
            const uint32_t cnt = valid ? rect_area(r) : 0u;
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += t;
            }
            const uint32_t total = __shfl_sync(kFull, incl, 31);
            if (total > uint32_t(kTab)) {  // rare: huge splats; enumerate with the owner search
                for_each_pair(slot, r, valid, u.tiles_x, place);
                return;
            }
            // each lane writes its record's tiles (row-major) and its lane id into the tables
            const uint32_t tx0 = r & 255u, ty0 = (r >> 8) & 255u, tx1 = (r >> 16) & 255u, ty1 = r >> 24;
            uint32_t k = incl - cnt;
            if (valid)
                for (uint32_t ty = ty0; ty <= ty1; ++ty)
                    for (uint32_t tx = tx0; tx <= tx1; ++tx, ++k) {
                        tab_tile[k] = uint16_t(ty * uint32_t(u.tiles_x) + tx);
                        tab_own[k] = uint8_t(lane);
                    }
            __syncwarp();
            for (uint32_t k0 = 0; k0 < total; k0 += 32) {
                const uint32_t j = k0 + lane;
                const bool in = j < total;
                const uint32_t tile = in ? tab_tile[j] : 0u;
                const uint32_t own = in ? tab_own[j] : 0u;
                const uint32_t sl = __shfl_sync(kFull, slot, own);
                place(in, tile, sl);
            }
        });
    }
}

// ---- launchers ---------------------------------------------------------------------------------
void launch_key_hist(const BinArgs& a, int grid, cudaStream_t s) {
    key_hist_kernel<<<grid, kThreads, 0, s>>>(a);
}
void launch_chunk_table(const BinArgs& a, cudaStream_t s) { chunk_table_kernel<<<1, 1024, 0, s>>>(a); }
size_t bin_smem_bytes(const BinArgs& a) { return size_t(a.bin_warps) * bin_warp_bytes(a.max_tc); }
void launch_bin_count(const BinArgs& a, int grid, cudaStream_t s) {
    const size_t smem = bin_smem_bytes(a);
    cudaFuncSetAttribute(bin_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    bin_count_kernel<<<grid, 32 * a.bin_warps, smem, s>>>(a);
}
void launch_bin_colscan(const BinArgs& a, int grid, cudaStream_t s) {
    bin_colscan_kernel<<<grid, kThreads, 0, s>>>(a);
}
void launch_bin_tilescan(const BinArgs& a, int grid, cudaStream_t s) {
    bin_tilescan_kernel<<<grid, 1024, 0, s>>>(a);
}
void launch_bin_campre(const BinArgs& a, cudaStream_t s) { bin_campre_kernel<<<1, 1024, 0, s>>>(a); }
void launch_bin_scatter(const BinArgs& a, int grid, cudaStream_t s) {
    const size_t smem = bin_smem_bytes(a);
    cudaFuncSetAttribute(bin_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    bin_scatter_kernel<<<grid, 32 * a.bin_warps, smem, s>>>(a);
}

}  // namespace gsim_gpu
