// kernels.hpp — argument blocks and host launchers of the sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gsim_gpu.h"
#include "common.cuh"

namespace gsim_gpu {

constexpr int kMaxSmemSegments = 1024;
constexpr int kMaxTilePasses = 4;

struct PreprocessArgs {
    DevField field;
    const DevSegment* segs;
    int n_segs;
    int reserved;
    const SegEntry* entries;
    const DevCamera* cams;
    Record* records;                 // [slots]
    uint32_t* rects;                 // [slots] packed tile rect (dup reads this, L2-resident)
    uint32_t* keys;                  // [slots], kInvalidKey when culled / no tile
    uint32_t* hist;                  // [4][256] digit histograms of valid keys
    unsigned long long* visible_count;
    gsim_projected_splat* full;      // project() API only: double splat per slot
    uint8_t* full_visible;           // project() API only
};

struct SplatArgs {
    const gsim_projected_splat* splats;
    uint64_t n;
    const DevCamera* cam;
    Record* records;
    uint32_t* rects;
    uint32_t* keys;
    uint32_t* hist;
    unsigned long long* visible_count;
};

// One onesweep LSD pass over (u32 key, u32 value) pairs, 8-bit digit at `shift`.
struct OnesweepArgs {
    const uint32_t* keys_in;
    const uint32_t* vals_in;         // nullptr on the first depth pass: value = input index
    uint32_t* keys_out;
    uint32_t* vals_out;
    const unsigned long long* n_dev; // element count on device (ignored when n_host used)
    uint64_t n_host;
    uint64_t capacity;               // n_dev is clamped to this (0 = no clamp)
    const uint32_t* hist;            // [256] digit histogram of this pass
    uint64_t* status;                // decoupled-lookback words, [chunks][256]
    uint32_t* ticket;                // zeroed per pass
    uint32_t epoch;
    int shift;
};

// Exclusive scan of tiles-touched over depth-sorted records + pair emission.
struct DupArgs {
    const uint32_t* slots;           // [V] record slots in depth order
    const unsigned long long* n_dev; // V
    const uint32_t* rects;           // [slots] packed tile rects
    const uint64_t* cam_slot_base;   // [n_cams + 1]
    const uint32_t* cam_tile_base;   // [n_cams + 1]
    const int* cam_tiles_x;          // [n_cams]
    int n_cams;
    int tile_passes;
    uint32_t* keys_out;              // [P] global tile id (camera tile_base + tile)
    uint32_t* vals_out;              // [P] record slot
    uint64_t capacity;
    uint32_t* hist;                  // [tile_passes][256]
    uint64_t* status;                // [chunks]
    uint32_t* ticket;
    uint32_t epoch;
    unsigned long long* pairs_out;   // P (total, may exceed capacity)
};

struct RangesArgs {
    const uint32_t* keys;            // [P] sorted global tile ids
    const unsigned long long* n_dev; // P
    uint64_t capacity;
    uint32_t* tile_begin;            // [tiles]
    uint32_t* tile_end;              // [tiles]
};

struct RasterArgs {
    const Record* records;
    const uint32_t* values;          // [P] sorted record slots
    const uint32_t* tile_begin;
    const uint32_t* tile_end;
    const DevCamera* cams;
    const uint32_t* cam_tile_base;   // [n_cams + 1]
    int n_cams;
    int normalize_depth;
    float cutoff;                    // smallest float >= transmittance_cutoff
    float reserved;
    float* out;                      // per camera [rgb W*H*3 | depth W*H | alpha W*H]
    unsigned long long* consumed;    // += list entries fetched before the tile saturated
};

void launch_pose(const DevField& f, uint64_t begin, uint64_t end, const gsim_rigid& t,
                 int grid_cap, cudaStream_t stream);
void launch_preprocess(const PreprocessArgs& a, bool full, int grid_cap, cudaStream_t stream);
void launch_splats_to_records(const SplatArgs& a, int grid_cap, cudaStream_t stream);
void launch_onesweep(const OnesweepArgs& a, bool first, bool write_keys, int grid,
                     cudaStream_t stream);
void launch_scan_dup(const DupArgs& a, int grid, cudaStream_t stream);
void launch_ranges(const RangesArgs& a, int grid, cudaStream_t stream);
void launch_raster(const RasterArgs& a, uint32_t n_tiles, cudaStream_t stream);

constexpr int kOnesweepTile = 4096;  // keys per onesweep chunk (256 threads x 16)
constexpr int kDupTile = 2048;       // records per scan/duplicate chunk (256 threads x 8)

}  // namespace gsim_gpu
