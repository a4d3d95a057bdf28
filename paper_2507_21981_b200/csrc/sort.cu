// sort.cu — K3: onesweep LSD radix sort, fused scan + tile duplication, tile ranges.
//
// The reference bins splats into (tile << 32 | float32 depth bits) keys and std::sorts
// (key, splat index) pairs (raster.cpp:243-271). We produce the same order with an LSD radix
// sort whose depth digits are sorted BEFORE duplication, on the V visible records instead of
// the P ~ 3.5 V pairs:
//   pass 1..4  onesweep over the 32-bit depth key of every (camera, primitive) slot; pass 1
//              also compacts (drops culled slots). Input order = (camera, primitive) order,
//              so the stable sort leaves ties in primitive order, as the reference does.
//   scan+dup   decoupled-lookback exclusive scan of tiles-touched over the depth-sorted
//              records, then load-balanced emission of (camera|tile, slot) pairs.
//   pass 5..   onesweep over the camera|tile digits (stable), giving (camera, tile, depth,
//              primitive) order: exactly the reference's per-camera pair order.
// Every pass is single-sweep: chunks are claimed through an atomic ticket (so predecessors
// are always resident) and per-digit prefixes come from decoupled lookback over epoch-tagged
// status words (no clearing between passes).
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = kOnesweepTile / kThreads;  // 16
constexpr int kRadix = 256;
constexpr uint64_t kCountMask = (1ull << 40) - 1;

// Exclusive scan of one u32 per thread over a 256-thread block. Returns the exclusive
// prefix; *total gets the block sum. Uses s_tmp[kWarps]. Contains __syncthreads.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_tmp,
                                                         uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_tmp[warp] = incl;
    __syncthreads();
    uint32_t warp_prefix = 0, sum = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t t = s_tmp[w];
        if (w < warp) warp_prefix += t;
        sum += t;
    }
    *total = sum;
    __syncthreads();
    return warp_prefix + incl - v;
}

// Spin until chunk j's word for `lane_index` is published in this epoch; return it.
__device__ __forceinline__ uint64_t wait_status(const uint64_t* p, uint32_t epoch) {
    while (true) {
        const uint64_t s = ld_volatile_u64(p);
        if ((s >> 62) != 0 && uint32_t((s >> 40) & kEpochMask) == (epoch & kEpochMask)) return s;
    }
}

}  // namespace

template <bool kFirst, bool kWriteKeys>
__global__ void __launch_bounds__(kThreads, 3) onesweep_kernel(OnesweepArgs a) {
    __shared__ uint32_t s_keys[kOnesweepTile];
    __shared__ uint32_t s_vals[kOnesweepTile];
    __shared__ uint32_t s_warp_hist[kWarps][kRadix];
    __shared__ uint32_t s_bstart[kRadix];
    __shared__ unsigned long long s_dest[kRadix];
    __shared__ uint32_t s_tmp[kWarps];
    __shared__ uint32_t s_ticket;
    __shared__ uint32_t s_total;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t n = kFirst ? a.n_host : uint64_t(*a.n_dev);
    if (a.capacity && n > a.capacity) n = a.capacity;
    const uint64_t chunks = (n + kOnesweepTile - 1) / kOnesweepTile;

    // Global start of each digit: exclusive scan of the pass histogram.
    uint32_t hist_total;
    const uint32_t gbase = block_exclusive_scan(a.hist[tid], s_tmp, &hist_total);

    while (true) {
        if (tid == 0) s_ticket = atomicAdd(a.ticket, 1u);
        for (int k = tid; k < kWarps * kRadix; k += kThreads) (&s_warp_hist[0][0])[k] = 0;
        __syncthreads();
        const uint32_t t = s_ticket;
        if (t >= chunks) break;
        const uint64_t base = uint64_t(t) * kOnesweepTile + uint64_t(warp) * (kItems * 32);

        uint32_t keys[kItems], vals[kItems], rank[kItems];
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const uint64_t idx = base + uint64_t(i) * 32 + lane;
            const bool in = idx < n;
            keys[i] = in ? __ldcs(a.keys_in + idx) : kInvalidKey;
            if (kFirst) vals[i] = uint32_t(idx);
            else vals[i] = in ? __ldcs(a.vals_in + idx) : 0u;
            if (!kFirst && !in) keys[i] = kInvalidKey;
            rank[i] = in ? 1u : 0u;  // reuse as "valid" until ranked
            if (kFirst && keys[i] == kInvalidKey) rank[i] = 0u;
        }
        // Warp-level stable ranking: item order is (i, lane) = memory order.
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const bool valid = rank[i] != 0u;
            const uint32_t d = valid ? ((keys[i] >> a.shift) & 255u) : 256u;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const uint32_t below = peers & lanemask_lt();
            uint32_t pre = 0;
            if (valid) pre = s_warp_hist[warp][d];
            __syncwarp();
            if (valid && below == 0) s_warp_hist[warp][d] = pre + __popc(peers);
            __syncwarp();
            rank[i] = valid ? (pre + __popc(below)) : 0xFFFFFFFFu;
        }
        __syncthreads();
        // Per digit (thread = digit): exclusive prefix across warps, block count.
        uint32_t count = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = s_warp_hist[w][tid];
            s_warp_hist[w][tid] = count;
            count += c;
        }
        uint64_t* my_status = a.status + uint64_t(t) * kRadix + tid;
        st_volatile_u64(my_status, make_status(t == 0 ? kFlagInclusive : kFlagAggregate, a.epoch, count));
        uint32_t block_total;
        const uint32_t bstart = block_exclusive_scan(count, s_tmp, &block_total);
        s_bstart[tid] = bstart;
        // Decoupled lookback for this digit.
        uint64_t prefix = 0;
        if (t > 0) {
            int64_t j = int64_t(t) - 1;
            while (true) {
                const uint64_t s = wait_status(a.status + uint64_t(j) * kRadix + tid, a.epoch);
                prefix += s & kCountMask;
                if ((s >> 62) == kFlagInclusive) break;
                --j;
            }
            st_volatile_u64(my_status, make_status(kFlagInclusive, a.epoch, prefix + count));
        }
        s_dest[tid] = (unsigned long long)(uint64_t(gbase) + prefix - bstart);
        if (tid == 0) s_total = block_total;
        __syncthreads();
        // Stage the chunk in smem in sorted order, then write it out in digit runs.
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            if (rank[i] == 0xFFFFFFFFu) continue;
            const uint32_t d = (keys[i] >> a.shift) & 255u;
            const uint32_t pos = s_bstart[d] + s_warp_hist[warp][d] + rank[i];
            s_keys[pos] = keys[i];
            s_vals[pos] = vals[i];
        }
        __syncthreads();
        const uint32_t total = s_total;
        for (uint32_t p = tid; p < total; p += kThreads) {
            const uint32_t key = s_keys[p];
            const uint64_t dst = s_dest[(key >> a.shift) & 255u] + p;
            if (kWriteKeys) a.keys_out[dst] = key;
            a.vals_out[dst] = s_vals[p];
        }
        __syncthreads();
    }
}

// ---- scan + duplicate ----------------------------------------------------------------------
constexpr int kDupItems = kDupTile / kThreads;  // 8 consecutive records per thread
constexpr int kMaxSmemCams = 2048;

__device__ __forceinline__ int camera_of_slot(uint32_t slot, const uint32_t* cam_slot, int n_cams) {
    int lo = 0, hi = n_cams - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cam_slot[mid] <= slot) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Each thread owns 8 consecutive depth-sorted records; the block scans their tile counts,
// gets its global offset by decoupled lookback, and every thread then writes its own records'
// pairs (row-major per record, raster.cpp:259-263) — tile counts are small and the sum over
// 8 records evens them out, so no cross-thread load balancing is needed.
__global__ void __launch_bounds__(kThreads) scan_dup_kernel(DupArgs a) {
    __shared__ uint32_t s_cam_slot[kMaxSmemCams + 1];
    __shared__ uint32_t s_cam_tile[kMaxSmemCams + 1];
    __shared__ uint32_t s_cam_tx[kMaxSmemCams];
    __shared__ uint32_t s_hist[kMaxTilePasses][kRadix];
    __shared__ uint32_t s_tmp[kWarps];
    __shared__ uint32_t s_ticket;
    __shared__ unsigned long long s_prefix;

    const int tid = threadIdx.x;
    const uint64_t n = uint64_t(*a.n_dev);
    const uint64_t chunks = (n + kDupTile - 1) / kDupTile;
    const bool smem_cams = a.n_cams <= kMaxSmemCams;
    for (int k = tid; k < kMaxTilePasses * kRadix; k += kThreads) (&s_hist[0][0])[k] = 0;
    if (smem_cams)
        for (int k = tid; k < a.n_cams; k += kThreads) {
            s_cam_slot[k] = uint32_t(a.cam_slot_base[k]);
            s_cam_tile[k] = a.cam_tile_base[k];
            s_cam_tx[k] = uint32_t(a.cam_tiles_x[k]);
        }

    while (true) {
        if (tid == 0) s_ticket = atomicAdd(a.ticket, 1u);
        __syncthreads();
        const uint32_t t = s_ticket;
        if (t >= chunks) break;
        const uint64_t base = uint64_t(t) * kDupTile + uint64_t(tid) * kDupItems;

        uint32_t slot[kDupItems], rect[kDupItems];
        if (base + kDupItems <= n) {
            const uint4 s0 = __ldcs(reinterpret_cast<const uint4*>(a.slots + base));
            const uint4 s1 = __ldcs(reinterpret_cast<const uint4*>(a.slots + base) + 1);
            slot[0] = s0.x; slot[1] = s0.y; slot[2] = s0.z; slot[3] = s0.w;
            slot[4] = s1.x; slot[5] = s1.y; slot[6] = s1.z; slot[7] = s1.w;
        } else {
#pragma unroll
            for (int j = 0; j < kDupItems; ++j)
                slot[j] = (base + j < n) ? a.slots[base + j] : 0xFFFFFFFFu;
        }
        uint32_t thread_sum = 0;
#pragma unroll
        for (int j = 0; j < kDupItems; ++j) {
            rect[j] = 0xFFFFFFFFu;
            if (slot[j] != 0xFFFFFFFFu) rect[j] = __ldg(a.rects + slot[j]);
        }
#pragma unroll
        for (int j = 0; j < kDupItems; ++j) {
            if (slot[j] == 0xFFFFFFFFu) continue;
            const uint32_t r = rect[j];
            thread_sum += (((r >> 16) & 255u) - (r & 255u) + 1u) * ((r >> 24) - ((r >> 8) & 255u) + 1u);
        }
        uint32_t block_total;
        const uint32_t thread_excl = block_exclusive_scan(thread_sum, s_tmp, &block_total);
        // Publish + lookback (one chain per pass).
        if (tid == 0) {
            uint64_t* my = a.status + t;
            uint64_t prefix = 0;
            if (t == 0) {
                st_volatile_u64(my, make_status(kFlagInclusive, a.epoch, block_total));
            } else {
                st_volatile_u64(my, make_status(kFlagAggregate, a.epoch, block_total));
                int64_t j = int64_t(t) - 1;
                while (true) {
                    const uint64_t s = wait_status(a.status + j, a.epoch);
                    prefix += s & kCountMask;
                    if ((s >> 62) == kFlagInclusive) break;
                    --j;
                }
                st_volatile_u64(my, make_status(kFlagInclusive, a.epoch, prefix + block_total));
            }
            s_prefix = prefix;
            if (t == chunks - 1) *a.pairs_out = prefix + block_total;
        }
        __syncthreads();
        uint64_t out = s_prefix + thread_excl;
#pragma unroll
        for (int j = 0; j < kDupItems; ++j) {
            if (slot[j] == 0xFFFFFFFFu) continue;
            int cam = 0;
            if (a.n_cams > 1)
                cam = smem_cams ? camera_of_slot(slot[j], s_cam_slot, a.n_cams)
                                : upper_index(a.cam_slot_base, a.n_cams, uint64_t(slot[j]));
            const uint32_t tbase = smem_cams ? s_cam_tile[cam] : a.cam_tile_base[cam];
            const uint32_t tw = smem_cams ? s_cam_tx[cam] : uint32_t(a.cam_tiles_x[cam]);
            const uint32_t r = rect[j];
            const uint32_t tx0 = r & 255u, ty0 = (r >> 8) & 255u, tx1 = (r >> 16) & 255u, ty1 = r >> 24;
            for (uint32_t ty = ty0; ty <= ty1; ++ty) {
                const uint32_t row = tbase + ty * tw;
                for (uint32_t tx = tx0; tx <= tx1; ++tx) {
                    const uint32_t key = row + tx;
                    if (out < a.capacity) {
                        a.keys_out[out] = key;
                        a.vals_out[out] = slot[j];
                    }
                    ++out;
                    for (int p = 0; p < a.tile_passes; ++p)
                        atomicAdd(&s_hist[p][(key >> (8 * p)) & 255u], 1u);
                }
            }
        }
        __syncthreads();
    }
    __syncthreads();
    for (int k = tid; k < a.tile_passes * kRadix; k += kThreads) {
        const uint32_t v = (&s_hist[0][0])[k];
        if (v) atomicAdd(a.hist + k, v);
    }
}

// ---- tile ranges (raster.cpp:267-271) ------------------------------------------------------
__global__ void __launch_bounds__(kThreads) ranges_kernel(RangesArgs a) {
    uint64_t n = uint64_t(*a.n_dev);
    if (n > a.capacity) n = a.capacity;
    for (uint64_t i = blockIdx.x * uint64_t(kThreads) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * kThreads) {
        const uint32_t k = a.keys[i];
        if (i == 0 || a.keys[i - 1] != k) a.tile_begin[k] = uint32_t(i);
        if (i + 1 == n || a.keys[i + 1] != k) a.tile_end[k] = uint32_t(i + 1);
    }
}

// ---- launchers -----------------------------------------------------------------------------
void launch_onesweep(const OnesweepArgs& a, bool first, bool write_keys, int grid,
                     cudaStream_t stream) {
    if (first) {
        if (write_keys) onesweep_kernel<true, true><<<grid, kThreads, 0, stream>>>(a);
        else onesweep_kernel<true, false><<<grid, kThreads, 0, stream>>>(a);
    } else {
        if (write_keys) onesweep_kernel<false, true><<<grid, kThreads, 0, stream>>>(a);
        else onesweep_kernel<false, false><<<grid, kThreads, 0, stream>>>(a);
    }
}

void launch_scan_dup(const DupArgs& a, int grid, cudaStream_t stream) {
    scan_dup_kernel<<<grid, kThreads, 0, stream>>>(a);
}

void launch_ranges(const RangesArgs& a, int grid, cudaStream_t stream) {
    ranges_kernel<<<grid, kThreads, 0, stream>>>(a);
}

}  // namespace gsim_gpu
