// sort.cu — K3a: segmented onesweep LSD radix sort of the record depth keys, per camera.
//
// The reference bins splats into (tile << 32 | float32 depth bits) keys and std::sorts
// (key, splat index) pairs per camera (raster.cpp:174-202). We produce the same order with an LSD
// radix sort whose depth digits are sorted BEFORE duplication, on the V visible records instead
// of the P ~ 3.5 V pairs, and place the pairs afterwards (bin.cu):
//   * Every camera's records are a contiguous SEGMENT (pass 1: its slots, camera-major in
//     primitive order; later passes: its compacted records). Chunks of 4096 items never straddle
//     a camera, digit histograms are per (camera, pass), and the decoupled look-back of a chunk
//     stops at its camera's first chunk. The camera index therefore never enters the key: a
//     batch of any number of cameras (BASELINE config 2: 320) sorts in one launch per pass, and
//     the key is only the float32 depth bits rebased to the batch's [near, far] range
//     (depth_sort_key, raster.hpp:45-47): 27 bits for near/far 0.05/100 -> 3 passes of 9-bit
//     digits (4 of 8 bits when the span needs 28-32 bits).
//   * Pass 1 also compacts (drops culled slots). Input order = primitive order within a camera,
//     so the stable sort leaves ties in primitive order, as the reference's pair sort does.
//   * Every pass is single-sweep: chunks are claimed through an atomic ticket (so predecessors
//     are always resident) and per-digit prefixes come from decoupled look-back over
//     epoch-tagged status words (no clearing between passes).
//   * Every record's tile rect rides along as a third stream (read in slot order by pass 1,
//     moved with its key by every pass), so the binning gets the rects in depth order without
//     a random gather (optional: rects_in == nullptr sorts keys and values only).
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = kOnesweepTile / kThreads;  // 16 (32 with 8192-item chunks)
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

// Spin until chunk j's word for a digit is published in this epoch; return it.
__device__ __forceinline__ uint64_t wait_status(const uint64_t* p, uint32_t epoch, uint32_t backoff) {
    while (true) {
        const uint64_t s = ld_volatile_u64(p);
        if ((s >> 62) != 0 && uint32_t((s >> 40) & kEpochMask) == (epoch & kEpochMask)) return s;
        __nanosleep(backoff);  // back off: spinning warps would steal issue slots from working ones
    }
}

}  // namespace

// Digit peers (the lanes sharing a digit) come from one shared-memory atomicOr per item into a
// per-warp digit bitmap; shared atomics cost ~3 cycles per warp instruction without heavy
// same-address contention (tools/microbench.cu). The bitmaps have their own shared memory: they
// are cleared once per CTA and every item's leader clears its word again (a warp barrier orders
// that clear before the next item's atomicOr), so chunks never re-clear them.
// Thread t owns digits t*kDpt .. t*kDpt + kDpt - 1 for the per-digit scans and the look-back.
template <int kBits, bool kFirst, bool kWriteKeys>
__global__ void __launch_bounds__(kThreads, kOnesweepMinBlocks) onesweep_kernel(OnesweepArgs a) {
    constexpr int kRadix = 1 << kBits;
    constexpr int kDpt = kRadix / kThreads;  // 1 (8-bit digits) or 2 (9-bit)
    constexpr uint32_t kMask = kRadix - 1;
    // dynamic: [keys | values | rects of the staged chunk][per-warp digit counts][per-warp
    // digit bitmaps] (launch_one)
    extern __shared__ __align__(16) uint32_t s_dyn[];
    uint32_t* s_keys = s_dyn;
    uint32_t* s_vals = s_dyn + kOnesweepTile;
    uint32_t* s_rects = s_dyn + 2 * kOnesweepTile;
    // rows of kRow words: the kRadix digits, then one spare word per lane that an invalid item
    // ranks in alone (so every lane runs the same shared-memory sequence, without branches)
    constexpr int kRow = kRadix + 32;
    auto s_warp_hist = reinterpret_cast<uint32_t(*)[kRow]>(s_dyn + 3 * kOnesweepTile);
    auto s_peer = reinterpret_cast<uint32_t(*)[kRow]>(s_dyn + 3 * kOnesweepTile + kWarps * kRow);
    const bool carry = a.rects_in != nullptr;
    __shared__ uint32_t s_bstart[kRadix];
    __shared__ uint32_t s_dest[kRadix];
    __shared__ uint32_t s_tmp[kWarps];
    __shared__ uint32_t s_ticket;
    __shared__ uint32_t s_total;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n_chunks = a.chunk_base[a.n_cams];
    const uint32_t* seg32 = a.seg_base32;
    int cam_cached = -1;
    uint32_t gbase[kDpt];  // output position of each of this thread's digits, this camera
    for (int k = tid; k < kWarps * kRow; k += kThreads) (&s_peer[0][0])[k] = 0;

    while (true) {
        if (tid == 0) s_ticket = atomicAdd(a.ticket, 1u);
        for (int k = tid; k < kWarps * kRow; k += kThreads) (&s_warp_hist[0][0])[k] = 0;
        __syncthreads();
        const uint32_t t = s_ticket;
        if (t >= n_chunks) break;
        const int cam = upper_index(a.chunk_base, a.n_cams, t);
        const uint32_t first_chunk = a.chunk_base[cam];
        GSIM_DCHECK(cam >= 0 && cam < a.n_cams && t >= first_chunk && t < a.chunk_base[cam + 1]);
        const uint64_t sb = kFirst ? a.seg_base64[cam] : uint64_t(seg32[cam]);
        const uint64_t se = kFirst ? a.seg_base64[cam + 1] : uint64_t(seg32[cam + 1]);
        const uint32_t cbegin = uint32_t(sb) + (t - first_chunk) * uint32_t(kOnesweepTile);
        const uint64_t cend64 = uint64_t(cbegin) + kOnesweepTile;
        const uint32_t cend = uint32_t(cend64 < se ? cend64 : se);
        GSIM_DCHECK(uint64_t(cbegin) >= sb && cbegin < cend);
        if (cam != cam_cached) {
            // global start of each digit in this camera: camera's output base + exclusive scan
            // of the camera's histogram of this pass
            const uint32_t* h = a.hist + uint64_t(cam) * a.hist_stride;
            uint32_t v[kDpt], loc = 0;
#pragma unroll
            for (int j = 0; j < kDpt; ++j) {
                v[j] = h[tid * kDpt + j];
                loc += v[j];
            }
            uint32_t tot;
            uint32_t run = block_exclusive_scan(loc, s_tmp, &tot) + a.vbase[cam];
#pragma unroll
            for (int j = 0; j < kDpt; ++j) {
                gbase[j] = run;
                run += v[j];
            }
            cam_cached = cam;
        }
        // 32-bit indices: slot counts stay below 2^31 (host.cu groups larger batches)
        const uint32_t base = cbegin + uint32_t(warp) * (kItems * 32) + uint32_t(lane);
        const uint32_t* kin = a.keys_in + base;
        const uint32_t* vin = a.vals_in + base;
        uint32_t keys[kItems], vals[kItems], rank[kItems];
        if (cbegin + uint32_t(kOnesweepTile) == cend) {  // full chunk: no bounds checks
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                keys[i] = __ldcs(kin + i * 32);
                vals[i] = kFirst ? base + uint32_t(i) * 32 : __ldcs(vin + i * 32);
                rank[i] = (!kFirst || keys[i] != kInvalidKey) ? 1u : 0u;  // "valid" until ranked
            }
        } else {
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                const bool in = base + uint32_t(i) * 32 < cend;
                keys[i] = in ? __ldcs(kin + i * 32) : kInvalidKey;
                vals[i] = kFirst ? base + uint32_t(i) * 32 : (in ? __ldcs(vin + i * 32) : 0u);
                rank[i] = (in && (!kFirst || keys[i] != kInvalidKey)) ? 1u : 0u;
            }
        }
        // Warp-level stable ranking: item order is (i, lane) = memory order.
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const bool valid = rank[i] != 0u;
            const uint32_t d = (keys[i] >> a.shift) & kMask;
            // The digit's warp count is read by every peer together with the bitmap (the
            // histogram is warp-private: no atomic, no shuffle from the leader); the leader
            // bumps it and clears the bitmap after a warp barrier orders that after all reads.
            const uint32_t dd = valid ? d : uint32_t(kRadix + lane);
            uint32_t* bits = &s_peer[warp][dd];
            uint32_t* cnt = &s_warp_hist[warp][dd];
            atomicOr(bits, 1u << lane);
            __syncwarp();
            const uint32_t peers = *bits;
            const uint32_t pre = *cnt;
            const uint32_t below = peers & lanemask_lt();
            __syncwarp();
            if (below == 0) {
                *cnt = pre + uint32_t(__popc(peers));
                *bits = 0u;
            }
            rank[i] = valid ? (pre + __popc(below)) : 0xFFFFFFFFu;
            __syncwarp();  // the leader's updates are visible before the next item's reads
        }
        // the rects (coalesced, same positions as the keys) are copied into s_rects in load order
        // with cp.async, in flight during the look-back without holding registers
        if (carry) {
            const uint32_t* rin = a.rects_in + base;
            const uint32_t raw = uint32_t(__cvta_generic_to_shared(s_rects + warp * (kItems * 32) + lane));
#pragma unroll
            for (int i = 0; i < kItems; ++i)
                if (rank[i] != 0xFFFFFFFFu)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(raw + 128u * i),
                                 "l"(rin + i * 32) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        __syncthreads();
        // Per digit (thread = kDpt digits): exclusive prefix across warps, block count.
        uint32_t count[kDpt], loc = 0;
#pragma unroll
        for (int j = 0; j < kDpt; ++j) {
            const int dg = tid * kDpt + j;
            uint32_t c = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t x = s_warp_hist[w][dg];
                s_warp_hist[w][dg] = c;
                c += x;
            }
            count[j] = c;
            loc += c;
            uint64_t* my_status = a.status + uint64_t(t) * kRadix + dg;
            st_volatile_u64(my_status, make_status(t == first_chunk ? kFlagInclusive : kFlagAggregate,
                                                   a.epoch, c));
        }
        uint32_t block_total;
        uint32_t bst = block_exclusive_scan(loc, s_tmp, &block_total);
#pragma unroll
        for (int j = 0; j < kDpt; ++j) {
            s_bstart[tid * kDpt + j] = bst;
            bst += count[j];
        }
        // Decoupled look-back, back to the camera's first chunk; a thread's digits walk back
        // together (their status words are adjacent, their waits overlap).
        uint64_t prefix[kDpt];
#pragma unroll
        for (int j = 0; j < kDpt; ++j) prefix[j] = 0;
        if (t > first_chunk) {
            bool done[kDpt];
#pragma unroll
            for (int j = 0; j < kDpt; ++j) done[j] = false;
            int64_t q = int64_t(t) - 1;
            while (true) {
                bool all = true;
#pragma unroll
                for (int j = 0; j < kDpt; ++j) {
                    if (done[j]) continue;
                    GSIM_DCHECK(q >= int64_t(first_chunk));
                    const uint64_t s = wait_status(a.status + uint64_t(q) * kRadix + tid * kDpt + j, a.epoch,
                                                   a.backoff_ns);
                    prefix[j] += s & kCountMask;
                    done[j] = (s >> 62) == kFlagInclusive;
                    all = all && done[j];
                }
                if (all) break;
                --q;
            }
#pragma unroll
            for (int j = 0; j < kDpt; ++j)
                st_volatile_u64(a.status + uint64_t(t) * kRadix + tid * kDpt + j,
                                make_status(kFlagInclusive, a.epoch, prefix[j] + count[j]));
        }
#pragma unroll
        for (int j = 0; j < kDpt; ++j)
            s_dest[tid * kDpt + j] = uint32_t(uint64_t(gbase[j]) + prefix[j] - s_bstart[tid * kDpt + j]);
        if (tid == 0) s_total = block_total;
        __syncthreads();
        // Stage the chunk in smem in sorted order, then write it out in digit runs.
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            if (rank[i] == 0xFFFFFFFFu) continue;
            const uint32_t d = (keys[i] >> a.shift) & kMask;
            const uint32_t pos = s_bstart[d] + s_warp_hist[warp][d] + rank[i];
            GSIM_DCHECK(pos < uint32_t(kOnesweepTile));
            s_keys[pos] = keys[i];
            s_vals[pos] = vals[i];
            rank[i] = pos;
        }
        if (carry) {  // the rects: load order -> registers -> sorted order
            asm volatile("cp.async.wait_all;" ::: "memory");
            uint32_t rc[kItems];
#pragma unroll
            for (int i = 0; i < kItems; ++i) rc[i] = s_rects[warp * (kItems * 32) + i * 32 + lane];
            __syncthreads();
#pragma unroll
            for (int i = 0; i < kItems; ++i)
                if (rank[i] != 0xFFFFFFFFu) s_rects[rank[i]] = rc[i];
        }
        __syncthreads();
        const uint32_t total = s_total;
        if (kWriteKeys) {
            for (uint32_t p = tid; p < total; p += kThreads) {
                const uint32_t key = s_keys[p];
                const uint32_t dst = s_dest[(key >> a.shift) & kMask] + p;
                GSIM_DCHECK(dst >= a.vbase[cam] && dst < a.vbase[cam + 1]);
                a.keys_out[dst] = key;
                a.vals_out[dst] = s_vals[p];
                if (carry) a.rects_out[dst] = s_rects[p];
            }
        } else {
            // last pass: slots and rects in depth order, no keys
            for (uint32_t p = tid; p < total; p += kThreads) {
                const uint32_t dst = s_dest[(s_keys[p] >> a.shift) & kMask] + p;
                GSIM_DCHECK(dst >= a.vbase[cam] && dst < a.vbase[cam + 1]);
                a.vals_out[dst] = s_vals[p];
                if (carry) a.rects_out[dst] = s_rects[p];
            }
        }
        __syncthreads();
    }
}

// ---- launchers -----------------------------------------------------------------------------
template <int kBits, bool kFirst, bool kWriteKeys>
static void launch_one(const OnesweepArgs& a, int grid, cudaStream_t s) {
    const int smem = int((3 * kOnesweepTile + 2 * kWarps * ((1 << kBits) + 32)) * sizeof(uint32_t));
    cudaFuncSetAttribute(onesweep_kernel<kBits, kFirst, kWriteKeys>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    onesweep_kernel<kBits, kFirst, kWriteKeys><<<grid, kThreads, smem, s>>>(a);
}

template <int kBits>
static void launch_bits(const OnesweepArgs& a, bool first, bool write_keys, int grid, cudaStream_t s) {
    if (first) {
        if (write_keys) launch_one<kBits, true, true>(a, grid, s);
        else launch_one<kBits, true, false>(a, grid, s);
    } else {
        if (write_keys) launch_one<kBits, false, true>(a, grid, s);
        else launch_one<kBits, false, false>(a, grid, s);
    }
}

void launch_onesweep(const OnesweepArgs& a, int bits, bool first, bool write_keys, int grid,
                     cudaStream_t stream) {
    if (bits == 9) launch_bits<9>(a, first, write_keys, grid, stream);
    else launch_bits<8>(a, first, write_keys, grid, stream);
}

}  // namespace gsim_gpu
