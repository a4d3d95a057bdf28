// kernels.hpp — argument blocks and host launchers of the sm_100a kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gsim_gpu.h"
#include "common.cuh"
#include "encode.cuh"

namespace gsim_gpu {

constexpr int kMaxSmemSegments = 1024;
constexpr int kMaxSmemCams = 32;        // K2 stages up to this many cameras in shared memory
constexpr int kOnesweepTile = 4096;     // keys per onesweep chunk (256 threads x 16); 8192-item
                                        // chunks (32 per thread, 2 CTAs/SM) measured the same
constexpr int kOnesweepMinBlocks = 3;   // resident onesweep CTAs per SM (register-bound)
constexpr int kWarpRecords = 1024;      // depth-sorted records per warp of a binning unit (max)

struct PreprocessArgs {
    DevField field;
    const DevSegment* segs;
    int n_segs;
    int depth_bits;                  // bits of the rebased depth key
    const SegEntry* entries;
    const DevCamera* cams;
    Record* records;                 // [slots]
    uint32_t* rects;                 // [slots] packed tile rect (binning reads this plane)
    uint32_t* keys;                  // [slots], kInvalidKey when culled / no tile
    uint32_t key_base;               // float bits of the batch's smallest near plane
    uint32_t n_cams;                 // cameras of the batch (staged in shared memory if few)
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
};

// One segmented onesweep LSD pass over (u32 key, u32 value) pairs, 8- or 9-bit digit at
// `shift` (sort.cu). Segment c = camera c's items: pass 1 reads slots [seg_base64[c],
// seg_base64[c+1]) (culled slots carry kInvalidKey and are dropped), later passes read
// [seg_base32[c], seg_base32[c+1]) of the compacted records; every pass writes camera c's
// records to [vbase[c], vbase[c+1]). Chunks of kOnesweepTile items never straddle cameras:
// camera c owns chunks [chunk_base[c], chunk_base[c+1]).
struct OnesweepArgs {
    const uint32_t* keys_in;
    const uint32_t* vals_in;         // nullptr on the first pass: value = input index (slot)
    uint32_t* keys_out;
    uint32_t* vals_out;
    const uint64_t* seg_base64;      // pass 1: camera slot bases [C+1]
    const uint32_t* seg_base32;      // later passes: camera record bases [C+1] (= vbase)
    const uint32_t* chunk_base;      // [C+1] first chunk of every camera; [C] = chunk count
    const uint32_t* vbase;           // [C+1] output base of every camera
    const uint32_t* hist;            // digit histogram of this pass for camera 0 ...
    uint64_t hist_stride;            // ... and the stride between cameras (passes * radix)
    int n_cams;
    uint64_t* status;                // decoupled-lookback words, [chunks][radix]
    uint32_t* ticket;                // zeroed per pass
    uint32_t epoch;
    int shift;
    const uint32_t* rects_in;        // tile rects moved with the keys (same positions as
    uint32_t* rects_out;             // keys_in / keys_out); nullptr: keys and values only
    uint32_t backoff_ns;             // look-back retry sleep
};

// Tile binning of the camera-major depth-sorted records (bin.cu).
struct BinArgs {
    const uint32_t* keys;            // [S] rebased depth keys (key_hist)
    uint64_t n_slots;
    const uint64_t* cam_slot_base;   // [C+1] slot segment of every camera
    int sort_bits;                   // depth digit bits (8 or 9)
    int sort_passes;                 // onesweep passes
    int n_cams;
    const uint32_t* sorted_slots;    // [V] record slots, camera-major depth order
    const uint32_t* sorted_rects;    // [V] tile rects of sorted_slots (gathered by the sort)
    const uint32_t* cam_tile_base;   // [C+1]
    const int* cam_tiles_x;          // [C]
    uint32_t* cam_visible;           // [C]   V_c (zeroed per frame)
    uint32_t* cam_vbase;             // [C+1]
    uint32_t* cam_chunk_base;        // [C+1]
    uint64_t* cam_mbase;             // [C+1] count-matrix base, column-major [tile][chunk]
    uint32_t* cam_pairs;             // [C]
    uint64_t* cam_pair_base;         // [C+1]
    uint32_t* chunk_cam;             // [K_max]
    uint32_t* n_chunks;              // [1]
    uint32_t* counts;                // count matrix / column prefixes
    uint32_t* tile_count;            // [tiles]
    uint32_t* tile_rel;              // [tiles] first pair of the tile within its camera
    uint32_t* hist;                  // [C][passes][radix] digit histograms (zeroed per frame)
    uint32_t* sort_chunk_base;       // [C+1] onesweep chunks of passes >= 2 per camera (out)
    unsigned long long* totals;      // [0] V, [1] P
    unsigned long long* host_totals; // optional: page-locked host copy of totals, stored by
                                     // campre (no copy-engine operation in the frame's stream)
    uint32_t* vals_out;              // [capacity] record slot of every pair, final order
    uint64_t capacity;
    int max_tc;                      // largest (tiles_x + 1) * (tiles_y + 1) of the batch
    int chunk_records;               // records per unit = warp_records * bin_warps
    int warp_records;                // depth-sorted records walked by one warp (<= kWarpRecords)
    int bin_warps;                   // warps per unit CTA
    int bitmap_peers;                // scatter: lane bitmaps (small cameras) or probe
};

struct RasterArgs {
    const Record* records;
    const uint32_t* values;          // [P] record slots in (camera, tile, depth) order
    const uint32_t* tile_rel;        // [tiles]
    const uint32_t* tile_count;      // [tiles]
    const uint64_t* cam_pair_base;   // [C+1]
    const DevCamera* cams;
    const uint32_t* cam_tile_base;   // [n_cams + 1]
    int n_cams;
    int normalize_depth;
    float cutoff;                    // smallest float >= transmittance_cutoff
    int rect_w;                      // warp-rectangle width: 16 (16x4 bands) or 8 (8x8)
    int batch;                       // records per shared-memory batch: 128 or 256
    int exact_cull;                  // exact ellipse-vs-warp-rectangle test in the compaction
    int bulk_copy;                   // stage records with cp.async.bulk + mbarrier (8x8 rects)
    uint32_t tile_begin;             // first tile of the launch (a camera's tiles, for per-camera
                                     // launches whose copies start on an event)
    uint32_t n_tiles;                // one past the last tile of the launch (set by launch_raster)
    int grid_cap;                    // CTAs of the launch (0: one per tile)
    uint32_t* tile_ticket;           // grid_cap > 0: tile counter, zero before the launch
    float valid_alpha;               // depth written as 0 where accum_alpha < valid_alpha
                                     // (render_depth_ring, transfer.cpp:116-118); 0 = off
    float* out;                      // per camera [rgb W*H*3 | depth W*H | alpha W*H]
    unsigned long long* consumed;    // += list entries fetched before the tile saturated
    uint64_t capacity;               // pair-buffer capacity (reads are clamped to it)
    uint64_t n_slots;                // record slots (stale values are clamped to a valid slot)
    EncodeParams enc;                // fused encoding when enc.flags != 0; camera c's block
                                     // starts at enc.dst + out_offset / 5 * encoded_bpp
};

// Device pose tracks (tracks.cu): records of track k are begin[k] .. begin[k+1]-1.
struct DevTracks {
    const double* t;                 // [R] times, non-decreasing per track
    const double* p;                 // [R][3] translations
    const double* q;                 // [R][4] normalised rotations (w, x, y, z)
    const uint64_t* begin;           // [n_tracks + 1]
    uint32_t n_tracks;
    uint32_t reserved;
};

// Splat PLY payload -> field planes (ply.cu).
struct PlyArgs {
    const float* rows;               // [n][stride] little-endian floats as on disk
    uint64_t n;
    int stride;
    int degree;
    DevField field;
    uint64_t plane_stride;           // SH plane pitch (max(n, 1))
    unsigned long long* err;         // min(i << 3 | code), ~0 when the file is valid
};

// Standalone encoder (encode.cu): one grid row per camera.
struct EncodeCam {
    uint32_t width, height;
    uint64_t src_offset;             // float offset of the camera's [rgb|depth|alpha] block
    uint64_t dst_offset;             // byte offset of its encoded block
};

struct EncodeKernelArgs {
    const float* src;
    const EncodeCam* cams;
    EncodeParams enc;
};

void launch_pose(const DevField& f, uint64_t begin, uint64_t end, const gsim_rigid& t,
                 int grid_cap, cudaStream_t stream);
void launch_preprocess(const PreprocessArgs& a, bool full, int n_sms, cudaStream_t stream);
void launch_splats_to_records(const SplatArgs& a, int grid_cap, cudaStream_t stream);
void launch_onesweep(const OnesweepArgs& a, int bits, bool first, bool write_keys, int grid,
                     cudaStream_t stream);
void launch_key_hist(const BinArgs& a, int grid, cudaStream_t s);
void launch_chunk_table(const BinArgs& a, cudaStream_t s);
size_t bin_smem_bytes(const BinArgs& a);
void launch_bin_count(const BinArgs& a, int grid, cudaStream_t s);
void launch_bin_colscan(const BinArgs& a, int grid, cudaStream_t s);
void launch_bin_tilescan(const BinArgs& a, int grid, cudaStream_t s);
void launch_bin_campre(const BinArgs& a, cudaStream_t s);
void launch_bin_scatter(const BinArgs& a, int grid, cudaStream_t s);
// Tiles [a.tile_begin, tile_end) of the batch.
void launch_raster(const RasterArgs& a, uint32_t tile_end, cudaStream_t stream);
void launch_encode(const EncodeKernelArgs& a, uint32_t n_cams, uint32_t max_pixels,
                   cudaStream_t stream);
void launch_track_query(const DevTracks& tr, const uint32_t* track, const double* time,
                        const gsim_rigid* initial, gsim_rigid* out, uint64_t n, int grid_cap,
                        cudaStream_t stream);
void launch_ply_convert(const PlyArgs& a, int grid_cap, cudaStream_t stream);
void launch_pose_segments(const DevTracks& tr, DevSegment* segs, const int32_t* seg_track,
                          uint32_t n_segs, double t, cudaStream_t stream);

// GS -> TSDF (transfer.cu): one view of a batched tsdf_fuse.
struct DevFuseView {
    double q[4], t[3];               // world -> camera pose
    double fx, fy, cx, cy;
    int width, height;
    uint64_t depth_offset;           // first float of this view's depth image in TsdfArgs::depth
};

struct TsdfArgs {
    double origin[3];
    double voxel_size;
    double truncation;
    int dims[3];
    uint32_t n_views;
    const DevFuseView* views;        // [n_views], fused in order
    const float* depth;
    double* tsdf;                    // [dims[2]][dims[1]][dims[0]]
    double* weights;
};

void launch_bounds(const DevField& f, double* partial, int max_blocks, double* out,
                   cudaStream_t s);
void launch_tsdf_reset(double* tsdf, double* weights, uint64_t n, int n_sms, cudaStream_t s);
void launch_tsdf_fuse(const TsdfArgs& a, int n_sms, cudaStream_t s);
const char* depth_ring_cameras(const double lo[3], const double hi[3], int n_views, double radius,
                               int resolution, gsim_camera* cameras);
DevFuseView fuse_view(const gsim_camera& c, uint64_t depth_offset);

// LiDAR (lidar.cu): the conservative (channel rank, azimuth step) rectangle of rays that can hit
// a primitive's box. k1 < k0 wraps around azimuth 0.
enum : uint32_t { kRectNone = 0, kRectRange = 1, kRectAll = 2 };
struct LidarRect {
    uint16_t r0, r1;
    uint32_t k0, k1;
    uint32_t kind;
};

struct LidarArgs {
    DevField field;
    const DevSegment* segs;          // painted node ranges; entry_count 0 = not seen
    int n_segs;
    int scan;                        // 1: LiDAR grid scan, 0: arbitrary rays
    int ray_lists;                   // arbitrary rays: candidates in list/ray_offset (BVH), else
                                     // every primitive is a candidate
    uint32_t list_stride;            // > 0: ray r's list at r * list_stride, list_count[r] long
    const uint32_t* list_count;
    uint64_t n;                      // primitives
    double* posed;                   // [19][n]: mean xyz, inv_cov 9, opacity, lo xyz, hi xyz
    double* trace_rec;               // [n][20]: lo xyz, hi xyz, opacity, seen (1.0 / 0.0) (the
                                     // first 64 B), mean xyz, inv_cov 9: one 160-byte row for the
                                     // tracer's random candidate reads (the planes serve the
                                     // binning and the BVH)
    uint8_t* seen;                   // [n]
    LidarRect* rects;                // [n]
    uint32_t* all_list;              // primitives whose box holds the sensor
    uint32_t* all_count;
    double w2s_q[4], w2s_t[3];       // world -> sensor
    double origin[3];
    double max_range, two_pi, step;
    const double* rank_elev;         // regular channels' elevations, ascending
    const uint32_t* rank_channel;    // rank -> channel index
    int n_ranks;
    uint32_t n_az;
    int* diff;                       // [channels][n_az + 1] row differences
    uint32_t* ray_count;             // [rays]
    const unsigned long long* ray_offset;  // [rays + 1]
    uint32_t* cursor;                // [rays] slots taken in each ray's list (zeroed)
    uint32_t* big_list;              // primitives with rectangles too big for one thread
    uint32_t* big_count;
    uint32_t* list;                  // candidates per ray
    uint64_t n_rays;
    const double* ray_origin;        // [rays][3] (arbitrary rays)
    const double* ray_dir;           // [rays][3] world directions
    const double* ray_dir_sensor;    // [rays][3] (scan)
    const double* ray_tmax;          // [rays] (arbitrary rays)
    const uint8_t* ray_all;          // [channels] every primitive is a candidate (scan)
    double alpha_threshold;
    uint32_t* out_hit;               // [rays] 0 / 1
    double* out_depth;
    double* out_acc;
    const unsigned long long* hit_offset;  // [rays + 1]
    uint64_t capacity;
    double* points;
    uint32_t* ring;
    double* azimuth;
    double* cand_t;                  // scan: per-candidate (t, response) cache, [pairs + rays *
    double* cand_r;                  //   all_count] (ray region at offset + ray * all_count)
    unsigned long long* debug;       // optional counters: rays, candidates
};

// Linear BVH over the posed boxes for arbitrary rays (bvh.cu).
constexpr uint32_t kLeafBit = 0x80000000u;
struct BvhArgs {
    uint64_t n;                      // primitives (LidarArgs::n)
    const double* posed;             // LidarArgs::posed ([19][n]: boxes in planes 13..18)
    const uint8_t* seen;
    unsigned long long* bounds_bits; // [6] ordered bits of the centre bounds (min xyz, max xyz)
    uint32_t* codes_in;              // [n] Morton codes (kInvalidKey: not seen)
    const uint32_t* codes_sorted;    // [n_leaves] sorted codes
    const uint32_t* leaf_prim;       // [n_leaves] primitive of sorted leaf k
    const uint32_t* hist;            // [4][256] digit histograms of the codes
    uint32_t* vbase;                 // [2] sort output segment
    uint32_t* chunk_base1;           // [2] chunks of passes >= 2
    uint32_t* n_leaves;              // [1]
    uint32_t* child;                 // [n - 1][2]: internal node or kLeafBit | sorted leaf
    uint32_t* node_parent;           // [n - 1]
    uint32_t* leaf_parent;           // [n]
    uint32_t* visits;                // [n - 1] refit arrivals
    double* node_box;                // [n - 1][6]
    double* leaf_box;                // [n_leaves][6]: sorted leaf k's double box (refit writes
                                     // it; the traversal's exact leaf test reads one 48-B row)
    float4* wide;                    // [n - 1][4] traversal nodes (bvh_widen_kernel)
    uint32_t* overflow;              // single-pass collect: largest count over the capacity
};

void launch_bvh_bounds(const BvhArgs& a, int n_sms, cudaStream_t s);
void launch_bvh_morton(const BvhArgs& a, int n_sms, cudaStream_t s);
void launch_bvh_sort_setup(const BvhArgs& a, cudaStream_t s);
void launch_bvh_build(const BvhArgs& a, int n_sms, cudaStream_t s);
void launch_bvh_refit(const BvhArgs& a, int n_sms, cudaStream_t s);
void launch_bvh_collect(const BvhArgs& a, const LidarArgs& la, int mode, int n_sms, cudaStream_t s);

void launch_lidar_pose(const LidarArgs& a, int n_sms, cudaStream_t s);
void launch_lidar_rays(const double* ds, double* dw, uint64_t n, const double* q, int n_sms,
                       cudaStream_t s);
void launch_lidar_count(const LidarArgs& a, int n_sms, cudaStream_t s);
void launch_lidar_rowscan(const LidarArgs& a, uint32_t n_channels, cudaStream_t s);
void launch_lidar_scatter(const LidarArgs& a, int n_sms, cudaStream_t s);
void launch_lidar_scatter_big(const LidarArgs& a, int n_sms, cudaStream_t s);
void launch_lidar_trace(const LidarArgs& a, int n_sms, cudaStream_t s);
void launch_lidar_emit(const LidarArgs& a, int n_sms, cudaStream_t s);
void exclusive_scan_u32(const uint32_t* in, uint64_t n, unsigned long long* out,
                        unsigned long long* scratch, cudaStream_t s);

}  // namespace gsim_gpu
