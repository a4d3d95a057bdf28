// bin.cu — K3 after the depth sort: deterministic tile binning without a pair sort.
//
// The reference emits (tile << 32 | depth, splat) pairs and std::sorts them
// (raster.cpp:243-271). After the camera-major depth sort of the V visible records
// (sort.cu), the pair order we need is simply "by (camera, tile), then by record order".
// Instead of radix-sorting the P ~ 3.5 V pairs by tile, we place every pair directly:
//   count    per chunk of R depth-sorted records of one camera, count pairs per tile
//            (pairs are enumerated warp-cooperatively; lanes with the same tile are merged
//            with match.any and the leader bumps a warp-private counter — no shared atomics,
//            which cost 2 cycles per lane on this part);
//   colscan  per (camera, tile): exclusive scan of the counts over the camera's chunks;
//   tilescan per camera: exclusive scan of the tile totals -> tile ranges (raster.cpp:267-271);
//   campre   per batch: pair base of every camera;
//   scatter  per chunk: recount per warp, turn counts into base positions, then walk the
//            records again in order and write each pair's record slot at base + rank, where
//            rank comes from match.any in lane order = emission order (raster.cpp:259-263).
// The result equals the reference's stable (tile, depth, primitive) order bit for bit.
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

__device__ __forceinline__ int cam_of_tile(const uint32_t* tile_base, int n_cams, uint32_t g) {
    return upper_index(tile_base, n_cams, g);
}

__device__ __forceinline__ uint32_t rect_area(uint32_t r) {
    return (((r >> 16) & 255u) - (r & 255u) + 1u) * ((r >> 24) - ((r >> 8) & 255u) + 1u);
}

// Warp-cooperative enumeration of the pairs of 32 records (one per lane): calls
// fn(j_valid, tile, slot) once per output step with consecutive pair indices per lane.
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

struct ChunkInfo {
    int cam;
    uint32_t rec_begin, rec_end;  // depth-sorted record range
    uint32_t chunk_in_cam, chunks_in_cam;
    uint64_t mbase;               // count-matrix base of the camera
    int tiles_x;
    uint32_t tc;                  // tiles of the camera
    uint32_t tile_base;
    int tbits;                    // bits of a camera-local tile id
};

__device__ __forceinline__ ChunkInfo chunk_info(const BinArgs& a, uint32_t k) {
    ChunkInfo ci;
    ci.cam = int(a.chunk_cam[k]);
    const uint32_t cb = a.cam_chunk_base[ci.cam];
    ci.chunk_in_cam = k - cb;
    ci.chunks_in_cam = a.cam_chunk_base[ci.cam + 1] - cb;
    const uint32_t vb = a.cam_vbase[ci.cam], ve = a.cam_vbase[ci.cam + 1];
    ci.rec_begin = vb + ci.chunk_in_cam * uint32_t(a.chunk_records);
    ci.rec_end = min(ci.rec_begin + uint32_t(a.chunk_records), ve);
    ci.mbase = a.cam_mbase[ci.cam];
    ci.tiles_x = a.cam_tiles_x[ci.cam];
    ci.tile_base = a.cam_tile_base[ci.cam];
    ci.tc = a.cam_tile_base[ci.cam + 1] - ci.tile_base;
    ci.tbits = ci.tc > 1 ? 32 - __clz(int(ci.tc - 1)) : 0;
    return ci;
}

// Per-warp counts of a chunk into cnt[warp][tile] (counters zeroed by the caller).
__device__ __forceinline__ void count_chunk(const BinArgs& a, const ChunkInfo& ci, uint32_t* cnt_w,
                                            int n_warps) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t n = ci.rec_end - ci.rec_begin;
    const uint32_t per_warp = (n + n_warps - 1) / n_warps;
    const uint32_t wb = ci.rec_begin + min(n, per_warp * warp);
    const uint32_t we = ci.rec_begin + min(n, per_warp * (warp + 1));
    walk_records(a, wb, we, ci.tiles_x, [&](bool in, uint32_t tile, uint32_t) {
        const uint32_t m = __ballot_sync(kFull, in);
        const uint32_t peers = peers_of_bits(kFull, tile, ci.tbits) & m;
        if (in && (peers & lanemask_lt()) == 0) cnt_w[tile] += __popc(peers);
        __syncwarp();
    });
    (void)lane;
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
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const uint32_t d = (key >> (8 * p)) & 255u;
                const uint32_t peers = peers_of<8>(kFull, d) & vmask;
                if (valid && (peers & lanemask_lt()) == 0) s_hist[warp][p][d] += __popc(peers);
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
        if (s) atomicAdd(a.hist + k, s);
    }
}

// ---- per-camera chunk tables (one block) ----------------------------------------------------
__global__ void __launch_bounds__(1024) chunk_table_kernel(BinArgs a) {
    __shared__ uint32_t s_scan[1024];
    __shared__ uint32_t s_carry_v, s_carry_k;
    __shared__ unsigned long long s_carry_m;
    const int tid = threadIdx.x;
    if (tid == 0) { s_carry_v = 0; s_carry_k = 0; s_carry_m = 0; }
    __syncthreads();
    const uint32_t R = uint32_t(a.chunk_records);
    for (int c0 = 0; c0 < a.n_cams; c0 += 1024) {
        const int c = c0 + tid;
        const uint32_t v = c < a.n_cams ? a.cam_visible[c] : 0u;
        const uint32_t k = (v + R - 1) / R;
        const uint32_t tc = c < a.n_cams ? a.cam_tile_base[c + 1] - a.cam_tile_base[c] : 0u;
        const unsigned long long m = (unsigned long long)k * tc;
        // three inclusive block scans (v, k, m) via smem Hillis-Steele
        uint32_t sv = v;
        s_scan[tid] = sv;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const uint32_t t = tid >= o ? s_scan[tid - o] : 0u;
            __syncthreads();
            s_scan[tid] += t;
            __syncthreads();
        }
        const uint32_t incl_v = s_scan[tid];
        __syncthreads();
        s_scan[tid] = k;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const uint32_t t = tid >= o ? s_scan[tid - o] : 0u;
            __syncthreads();
            s_scan[tid] += t;
            __syncthreads();
        }
        const uint32_t incl_k = s_scan[tid];
        __syncthreads();
        // m can exceed 32 bits only for absurd batches; scan it in 64-bit via two passes of hi/lo
        unsigned long long incl_m = m;
        {
            __shared__ unsigned long long s_m[1024];
            s_m[tid] = m;
            __syncthreads();
            for (int o = 1; o < 1024; o <<= 1) {
                const unsigned long long t = tid >= o ? s_m[tid - o] : 0ull;
                __syncthreads();
                s_m[tid] += t;
                __syncthreads();
            }
            incl_m = s_m[tid];
            __syncthreads();
        }
        if (c < a.n_cams) {
            a.cam_vbase[c] = s_carry_v + incl_v - v;
            a.cam_chunk_base[c] = s_carry_k + incl_k - k;
            a.cam_mbase[c] = s_carry_m + incl_m - m;
        }
        __syncthreads();
        if (tid == 1023) {
            s_carry_v += incl_v;
            s_carry_k += incl_k;
            s_carry_m += incl_m;
        }
        __syncthreads();
    }
    if (tid == 0) {
        a.cam_vbase[a.n_cams] = s_carry_v;
        a.cam_chunk_base[a.n_cams] = s_carry_k;
        a.cam_mbase[a.n_cams] = s_carry_m;
        *a.n_chunks = s_carry_k;
        a.totals[0] = s_carry_v;  // V
    }
    __syncthreads();
    const uint32_t K = s_carry_k;
    for (uint32_t k = tid; k < K; k += 1024)
        a.chunk_cam[k] = uint32_t(upper_index(a.cam_chunk_base, a.n_cams, k));
}

// ---- count -------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) bin_count_kernel(BinArgs a) {
    extern __shared__ uint32_t s_cnt[];  // [n_warps][max_tc]
    const int n_warps = a.bin_warps;
    const uint32_t K = *a.n_chunks;
    for (uint32_t k = blockIdx.x; k < K; k += gridDim.x) {
        const ChunkInfo ci = chunk_info(a, k);
        for (uint32_t i = threadIdx.x; i < uint32_t(n_warps) * ci.tc; i += blockDim.x) s_cnt[i] = 0;
        __syncthreads();
        if (int(threadIdx.x >> 5) < n_warps)
            count_chunk(a, ci, s_cnt + (threadIdx.x >> 5) * ci.tc, n_warps);
        __syncthreads();
        uint32_t* col = a.counts + ci.mbase + ci.chunk_in_cam;
        for (uint32_t t = threadIdx.x; t < ci.tc; t += blockDim.x) {
            uint32_t s = 0;
            for (int w = 0; w < n_warps; ++w) s += s_cnt[w * ci.tc + t];
            col[uint64_t(t) * ci.chunks_in_cam] = s;
        }
        __syncthreads();
    }
}

// ---- column scan: one warp per (camera, tile) --------------------------------------------------
__global__ void __launch_bounds__(kThreads) bin_colscan_kernel(BinArgs a) {
    const int lane = threadIdx.x & 31;
    const uint32_t n_cols = a.cam_tile_base[a.n_cams];
    for (uint32_t g = (blockIdx.x * kThreads + threadIdx.x) >> 5; g < n_cols;
         g += (gridDim.x * kThreads) >> 5) {
        const int c = cam_of_tile(a.cam_tile_base, a.n_cams, g);
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

// ---- scatter -----------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) bin_scatter_kernel(BinArgs a) {
    extern __shared__ uint32_t s_cnt[];  // [n_warps][max_tc]: counts, then running positions
    const int n_warps = a.bin_warps;
    const int warp = threadIdx.x >> 5;
    const uint32_t K = *a.n_chunks;
    for (uint32_t k = blockIdx.x; k < K; k += gridDim.x) {
        const ChunkInfo ci = chunk_info(a, k);
        for (uint32_t i = threadIdx.x; i < uint32_t(n_warps) * ci.tc; i += blockDim.x) s_cnt[i] = 0;
        __syncthreads();
        if (warp < n_warps) count_chunk(a, ci, s_cnt + warp * ci.tc, n_warps);
        __syncthreads();
        // counts -> first position of every (warp, tile) in the final list
        const uint64_t pbase = a.cam_pair_base[ci.cam];
        const uint32_t* col = a.counts + ci.mbase + ci.chunk_in_cam;
        for (uint32_t t = threadIdx.x; t < ci.tc; t += blockDim.x) {
            uint32_t run = uint32_t(pbase) + a.tile_rel[ci.tile_base + t] + col[uint64_t(t) * ci.chunks_in_cam];
            for (int w = 0; w < n_warps; ++w) {
                const uint32_t c = s_cnt[w * ci.tc + t];
                s_cnt[w * ci.tc + t] = run;
                run += c;
            }
        }
        __syncthreads();
        if (warp < n_warps) {
            const int lane = threadIdx.x & 31;
            uint32_t* pos_w = s_cnt + warp * ci.tc;
            const uint32_t n = ci.rec_end - ci.rec_begin;
            const uint32_t per_warp = (n + n_warps - 1) / n_warps;
            const uint32_t wb = ci.rec_begin + min(n, per_warp * warp);
            const uint32_t we = ci.rec_begin + min(n, per_warp * (warp + 1));
            walk_records(a, wb, we, ci.tiles_x, [&](bool in, uint32_t tile, uint32_t sl) {
                const uint32_t m = __ballot_sync(kFull, in);
                const uint32_t peers = peers_of_bits(kFull, tile, ci.tbits) & m;
                const uint32_t below = peers & lanemask_lt();
                const uint32_t pre = in ? pos_w[tile] : 0u;
                __syncwarp();
                if (in) {
                    if (below == 0) pos_w[tile] = pre + __popc(peers);
                    const uint32_t p = pre + __popc(below);
                    if (p < a.capacity) a.vals_out[p] = sl;
                }
                __syncwarp();
            });
            (void)lane;
        }
        __syncthreads();
    }
}

// ---- launchers ---------------------------------------------------------------------------------
void launch_key_hist(const BinArgs& a, int grid, cudaStream_t s) {
    key_hist_kernel<<<grid, kThreads, 0, s>>>(a);
}
void launch_chunk_table(const BinArgs& a, cudaStream_t s) { chunk_table_kernel<<<1, 1024, 0, s>>>(a); }
size_t bin_smem_bytes(const BinArgs& a) { return size_t(a.bin_warps) * a.max_tc * sizeof(uint32_t); }
void launch_bin_count(const BinArgs& a, int grid, cudaStream_t s) {
    const size_t smem = bin_smem_bytes(a);
    cudaFuncSetAttribute(bin_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    bin_count_kernel<<<grid, kThreads, smem, s>>>(a);
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
    bin_scatter_kernel<<<grid, kThreads, smem, s>>>(a);
}

}  // namespace gsim_gpu
