// sort.cu — K3a: onesweep LSD radix sort of the (camera | depth) record keys.
//
// The reference bins splats into (tile << 32 | float32 depth bits) keys and std::sorts
// (key, splat index) pairs (raster.cpp:174-202). We produce the same order with an LSD radix
// sort whose depth digits are sorted BEFORE duplication, on the V visible records instead of
// the P ~ 3.5 V pairs:
//   pass 1..4  onesweep over the 32-bit depth key of every (camera, primitive) slot; pass 1
//              also compacts (drops culled slots). Input order = (camera, primitive) order,
//              so the stable sort leaves ties in primitive order, as the reference does.
//   The key carries the camera index above the rebased depth bits, so the result is in
//   (camera, depth, primitive) order; bin.cu then places every (tile, record) pair directly
//   at its final position, which gives the reference's per-camera pair order without
//   sorting the P ~ 3.5 V pairs.
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
        __nanosleep(64);  // back off: spinning warps would steal issue slots from working ones
    }
}

}  // namespace

// Digit peers (the lanes sharing a digit) come from one shared-memory atomicOr per item into a
// per-warp digit bitmap (two buffers alternate, so clearing item i's bits never races item
// i+1's); shared atomics cost ~3 cycles per warp instruction without heavy same-address
// contention (tools/microbench.cu), and even the top digit (camera and exponent bits, ~3 lanes
// per value after the low passes) measured cheaper this way than with 8 ballots. The bitmaps
// live in s_keys (ranking is done before the chunk is staged there) and are cleared at the start
// of every chunk.
template <bool kFirst, bool kWriteKeys>
__global__ void __launch_bounds__(kThreads, 3) onesweep_kernel(OnesweepArgs a) {
    __shared__ uint32_t s_keys[kOnesweepTile];
    static_assert(2 * kWarps * kRadix <= kOnesweepTile, "peer bitmaps alias s_keys");
    auto s_peer = reinterpret_cast<uint32_t(*)[kWarps][kRadix]>(s_keys);
    __shared__ uint32_t s_vals[kOnesweepTile];
    __shared__ uint32_t s_warp_hist[kWarps][kRadix];
    __shared__ uint32_t s_bstart[kRadix];
    __shared__ uint32_t s_dest[kRadix];
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
        for (int k = tid; k < 2 * kWarps * kRadix; k += kThreads) s_keys[k] = 0;
        __syncthreads();
        const uint32_t t = s_ticket;
        if (t >= chunks) break;
        // 32-bit indices: slot counts stay below 2^31 (host.cu splits larger batches)
        const uint32_t base = t * uint32_t(kOnesweepTile) + uint32_t(warp) * (kItems * 32) + uint32_t(lane);
        const uint32_t* kin = a.keys_in + base;
        const uint32_t* vin = a.vals_in + base;
        uint32_t keys[kItems], vals[kItems], rank[kItems];
        if ((uint64_t(t) + 1) * kOnesweepTile <= n) {  // full chunk: no bounds checks
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                keys[i] = __ldcs(kin + i * 32);
                vals[i] = kFirst ? base + uint32_t(i) * 32 : __ldcs(vin + i * 32);
                rank[i] = (!kFirst || keys[i] != kInvalidKey) ? 1u : 0u;  // "valid" until ranked
            }
        } else {
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                const bool in = uint64_t(base) + uint64_t(i) * 32 < n;
                keys[i] = in ? __ldcs(kin + i * 32) : kInvalidKey;
                vals[i] = kFirst ? base + uint32_t(i) * 32 : (in ? __ldcs(vin + i * 32) : 0u);
                rank[i] = (in && (!kFirst || keys[i] != kInvalidKey)) ? 1u : 0u;
            }
        }
        // Warp-level stable ranking: item order is (i, lane) = memory order.
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const bool valid = rank[i] != 0u;
            const uint32_t d = (keys[i] >> a.shift) & 255u;
            uint32_t* bits = &s_peer[i & 1][warp][d];
            if (valid) atomicOr(bits, 1u << lane);
            __syncwarp();
            const uint32_t peers = valid ? *bits : 0u;
            __syncwarp();
            if (valid && (peers & lanemask_lt()) == 0) *bits = 0u;  // leader clears
            const uint32_t below = peers & lanemask_lt();
            const int leader = peers ? __ffs(peers) - 1 : lane;
            uint32_t pre = 0;
            if (valid && below == 0) pre = atomicAdd(&s_warp_hist[warp][d], uint32_t(__popc(peers)));
            pre = __shfl_sync(0xffffffffu, pre, leader);
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
        s_dest[tid] = uint32_t(uint64_t(gbase) + prefix - bstart);
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
            const uint32_t dst = s_dest[(key >> a.shift) & 255u] + p;
            if (kWriteKeys) a.keys_out[dst] = key;
            a.vals_out[dst] = s_vals[p];
            if (a.rects_out) a.rects_out[dst] = __ldg(a.rects_in + s_vals[p]);
        }
        __syncthreads();
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

}  // namespace gsim_gpu
