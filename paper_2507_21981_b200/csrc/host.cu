// host.cu — C-ABI implementation: contexts, device-resident scenes, frame plans and the
// render pipeline orchestration (one CUDA stream per context, grow-only HBM workspaces).
//
// Reference behaviour mirrored here:
//   validate_camera          raster.cpp:16-23   (status 2, same rules)
//   PoseTable                raster.cpp:47-62   (node painting, later nodes win, range check)
//   render / rasterize       raster.cpp:165-265 (pipeline K2 -> K3 -> K4)
//   transform_primitives     gaussian.cpp:65-79 (K1, range check)
//   validate_field sh_degree gaussian.cpp:15-17
//
// Frame pipeline (all on the context stream, no host round trip before the raster):
//   K2 preprocess -> key_hist -> chunk_table -> 4 x segmented onesweep (depth within camera)
//   -> bin_count -> bin_colscan -> bin_tilescan -> bin_campre -> bin_scatter -> K4 raster
// The host waits only for the small (V, P) readback behind bin_campre, while the GPU runs the
// scatter and the raster, to catch a pair-buffer overflow (then it grows and re-runs the tail).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <cctype>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/gsim_gpu.h"
#include "common.cuh"
#include "kernels.hpp"

using namespace gsim_gpu;

namespace {

thread_local std::string g_create_error;

struct CudaError {
    std::string msg;
};
struct ValidationError {
    std::string msg;
};

#define GSIM_CK(expr)                                                                   \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            throw CudaError{std::string(#expr) + ": " + cudaGetErrorString(_e)};        \
    } while (0)

template <class T>
struct DevBuf {
    T* ptr = nullptr;
    size_t cap = 0;  // elements
    void reserve(size_t n) {
        if (n <= cap) return;
        if (ptr) GSIM_CK(cudaFree(ptr));
        ptr = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(n, 1);
        GSIM_CK(cudaMalloc(&ptr, want * sizeof(T)));
        cap = want;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

struct PinnedBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    void reserve(size_t bytes) {
        if (bytes <= cap) return;
        if (ptr) GSIM_CK(cudaFreeHost(ptr));
        ptr = nullptr;
        cap = 0;
        GSIM_CK(cudaMallocHost(&ptr, std::max<size_t>(bytes, 64)));
        cap = std::max<size_t>(bytes, 64);
    }
    void release() {
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

// Everything a frame needs that is a pure function of (nodes, cameras, field size).
struct Plan {
    std::vector<DevCamera> cams;
    std::vector<uint64_t> slot_base;   // C + 1
    std::vector<uint32_t> tile_base;   // C + 1
    std::vector<int> tiles_x;          // C
    std::vector<DevSegment> segs;
    std::vector<SegEntry> entries;
    std::vector<int32_t> seg_owner;    // node index painting each segment, -1 = none
    std::vector<int32_t> seg_track;    // render_at only: track driving each segment, -1 = none
    uint64_t slots = 0;
    uint32_t tiles = 0;
    uint32_t max_tc = 0;
    uint64_t out_floats = 0;
    uint32_t key_base = 0;
    int depth_bits = 32;
    int sort_bits = 8;                 // depth digit bits of the segmented onesweep (8 or 9)
    int sort_passes = 4;
    std::vector<uint32_t> chunk_base0; // C + 1: first onesweep chunk of every camera, pass 1
};

// profiling events
enum Ev { kEvStart = 0, kEvPre, kEvDepth, kEvBin, kEvScatter, kEvRaster, kNumEv };

constexpr int kZeroTickets = 1024; // 16 onesweep tickets
constexpr int kRasterTicket = 12;  // the raster's tile counter (within the ticket words)
constexpr int kZeroCams = 1040;    // per-camera visible counts

}  // namespace

struct gsim_gpu_context {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    std::string err;
    bool profiling = false;
    cudaEvent_t ev[kNumEv] = {};

    // per-slot planes
    DevBuf<Record> records;
    DevBuf<uint32_t> keys;
    DevBuf<uint32_t> rects;
    DevBuf<uint32_t> dk[2], dv[2];   // depth-sort ping-pong
    DevBuf<uint32_t> sort_rects;     // tile rects between depth passes (with the slot-order plane)
    DevBuf<uint64_t> status;         // onesweep lookback words
    DevBuf<uint32_t> sort_hist;      // [C][passes][radix] depth digit histograms (zeroed per frame)
    DevBuf<uint32_t> sort_chunk_base;  // [C+1] onesweep chunks of passes >= 2
    int raster_rect_w = 8;           // GSIM_GPU_RASTER_RECT=16: 16x4 warp bands in K4 (default 8x8)
    int raster_exact_cull = 1;       // GSIM_GPU_RASTER_EXACT=0: bounding-box warp culling only
    int raster_batch = 128;          // GSIM_GPU_RASTER_BATCH=256: larger K4 batches, fewer CTAs/SM
    int raster_bulk = 0;             // GSIM_GPU_RASTER_BULK=1: records staged by cp.async.bulk
    int raster_ctas = 0;             // GSIM_GPU_RASTER_CTAS=k: k CTAs per SM looping over tiles
    // per-pair plane (final per-tile order)
    DevBuf<uint32_t> vals;
    uint64_t pair_capacity = 0;
    // GSIM_GPU_INITIAL_PAIR_CAPACITY (tests): start from this capacity instead of 8 x slots,
    // to exercise the overflow -> regrow -> re-run path.
    uint64_t fixed_initial_capacity = 0;
    // GSIM_GPU_GROUP_SLOTS (tests): (camera, primitive) slots per camera group; the kernels index
    // slots in 32 bits, so the default is 2^31 - 1
    uint64_t group_slots = (uint64_t(1) << 31) - 1;
    // zeroed per frame: histograms, tickets, per-camera visible counts
    DevBuf<uint32_t> zero_block;
    DevBuf<unsigned long long> counts;  // [0] V, [1] P, [2] consumed
    // binning scratch
    DevBuf<uint32_t> cam_vbase, cam_chunk_base, cam_pairs, chunk_cam, n_chunks;
    DevBuf<uint64_t> cam_mbase, cam_pair_base;
    DevBuf<uint32_t> count_matrix, tile_count, tile_rel;
    // plan tables of the current frame: pointers into plan_dev
    DevBuf<char> plan_dev;
    DevCamera* cams = nullptr;
    uint64_t* cam_slot_base = nullptr;
    uint32_t* cam_tile_base = nullptr;
    int* cam_tiles_x = nullptr;
    uint32_t* cam_chunk_base0 = nullptr;
    DevSegment* segs = nullptr;
    SegEntry* entries = nullptr;
    int32_t* seg_track = nullptr;
    std::vector<char> blob_host;
    PinnedBuf staging[2];
    cudaEvent_t staging_ev[2] = {};
    int staging_index = 0;
    PinnedBuf readback;
    cudaEvent_t bin_ev = nullptr;
    // GSIM_GPU_BLOCKING_SYNC=1: the synchronous calls wait on blocking-sync events (the host
    // thread sleeps instead of spinning; more renderer threads per core)
    bool blocking_sync = false;
    cudaEvent_t wait_ev[2] = {};
    // deferred pair-count check of the last asynchronous render (see check_pending)
    bool pending = false;
    float* pending_out = nullptr;
    gsim_raster_options pending_opt{0, 0, 1e-4};
    int pending_grid = 1;
    // output encoding (encode.cuh): thresholds uploaded on first use; frame_enc is the fused
    // raster epilogue's encoding of the render in flight (flags 0 = float targets only)
    DevBuf<float> srgb_thr;
    bool srgb_ready = false;
    EncodeParams frame_enc{};
    bool frame_enc_only = false;     // encoded bytes only, no float targets
    EncodeParams pending_enc{};
    bool pending_enc_only = false;
    DevBuf<uint8_t> enc_buf;
    // render_at: device pose playback of the frame in flight (tracks.cu)
    const gsim_gpu_tracks* frame_tracks = nullptr;
    double frame_time = 0.0;
    const int64_t* frame_node_track = nullptr;
    DevBuf<char> query_buf;
    DevBuf<float> enc_src;
    DevBuf<EncodeCam> enc_cams;
    // host-target renders: camera c's copies start when its tiles are done (the raster runs one
    // launch per camera; copy_stream waits on the event recorded after camera c's launch)
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> cam_evs;
    gsim_target* frame_outs = nullptr;   // targets of the camera group in flight (nullptr: none)
    uint8_t* frame_enc_host = nullptr;   // render_encoded: host bytes of the group in flight
    bool copies_stale = false;           // a group was re-run after its copies were issued
    bool overlap_copies = true;          // GSIM_GPU_OVERLAP_COPIES=0: copies follow the frame
    // outputs / API scratch
    DevBuf<float> out;
    DevBuf<gsim_projected_splat> full;
    DevBuf<uint8_t> full_vis;
    DevBuf<gsim_projected_splat> splats_in;
    // GS -> TSDF scratch (transfer.cu)
    DevBuf<double> bounds_buf;       // per-block boxes + the reduced box
    DevBuf<DevFuseView> fuse_views;
    DevBuf<float> depth_in;          // host depth maps staged for tsdf_fuse
    float frame_valid_alpha = 0.0f;  // render_depth_ring's depth mask (raster epilogue)
    // LiDAR scratch (lidar.cu)
    struct {
        DevBuf<double> posed, trace_rec, rays, depth, acc, points, azimuth, rank_elev, cand_t, cand_r;
        DevBuf<uint8_t> seen, ray_all;
        DevBuf<LidarRect> rects;
        DevBuf<uint32_t> all_list, counts, list, hit, ring, rank_channel, cursor, big_list;
        DevBuf<int> diff;
        DevBuf<unsigned long long> offsets, scratch, hit_offsets;
        DevBuf<DevSegment> segs;
        // arbitrary rays: linear BVH (bvh.cu)
        DevBuf<uint32_t> bvh_keys[2], bvh_vals[2], bvh_small, bvh_nodes;
        DevBuf<uint64_t> bvh_seg;
        DevBuf<unsigned long long> bvh_bounds;
        DevBuf<double> bvh_box, bvh_leaf_box;
        DevBuf<float4> bvh_wide;
        uint32_t bvh_capacity = 256;  // candidate slots per ray of the single-pass collect
        std::vector<double> ray_key;  // (channels, step) of the sensor directions in rays
        void release() {
            for (int k = 0; k < 2; ++k) { bvh_keys[k].release(); bvh_vals[k].release(); }
            bvh_small.release(); bvh_nodes.release(); bvh_seg.release(); bvh_bounds.release();
            bvh_box.release();
            bvh_leaf_box.release();
            bvh_wide.release();
            posed.release(); trace_rec.release(); rays.release(); depth.release(); acc.release(); points.release();
            azimuth.release(); rank_elev.release(); seen.release(); ray_all.release();
            cand_t.release(); cand_r.release();
            rects.release(); all_list.release(); counts.release(); list.release(); hit.release();
            ring.release(); rank_channel.release(); diff.release(); offsets.release();
            cursor.release(); big_list.release(); scratch.release(); hit_offsets.release();
            segs.release();
            ray_key.clear();
        }
    } lidar;

    uint32_t epoch = 0;
    uint64_t launches_total = 0;

    // scenes and tracks created on this context: destroying the context orphans them (their
    // ctx becomes null and only their own memory is freed later), so handle lifetimes may end
    // in any order
    std::set<gsim_gpu_scene*> scenes;
    std::set<gsim_gpu_tracks*> tracks;

    // last frame, for stats and the tile-list hook
    gsim_render_stats stats{};
    Plan last_plan;

    uint32_t next_epoch() {
        epoch = (epoch + 1) & kEpochMask;
        if (epoch == 0) {
            if (status.ptr) GSIM_CK(cudaMemsetAsync(status.ptr, 0, status.cap * sizeof(uint64_t), stream));
            epoch = 1;
        }
        return epoch;
    }
};

struct gsim_gpu_scene {
    gsim_gpu_context* ctx = nullptr;
    DevField f{};
    void* mem = nullptr;
};

struct gsim_gpu_tracks {
    gsim_gpu_context* ctx = nullptr;
    void* mem = nullptr;
    DevTracks d{};
    uint64_t n_tracks = 0, n_records = 0;
};

namespace {

uint32_t ceil_log2_bits(uint64_t n) {  // bits needed to represent values in [0, n)
    uint32_t b = 0;
    while ((uint64_t(1) << b) < n) ++b;
    return b;
}

uint32_t float_bits(double x) {
    const float f = float(x);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

void validate_camera(const gsim_camera& c, uint64_t index) {  // raster.cpp:16-23
    const std::string who = "camera " + std::to_string(index);
    if (!(c.fx > 0.0) || !(c.fy > 0.0)) throw ValidationError{who + ": fx, fy must be positive"};
    if (!(c.near_plane > 0.0) || !(c.far_plane > c.near_plane))
        throw ValidationError{who + ": need 0 < near < far"};
    if (c.width < 16 || c.height < 16) throw ValidationError{who + ": resolution below 16x16"};
    if (c.width > kMaxTilesPerAxis * kTileSize || c.height > kMaxTilesPerAxis * kTileSize)
        throw ValidationError{who + ": resolution above 4096x4096 (GPU tile-rect limit)"};
}

DevCamera make_dev_camera(const gsim_camera& c) {
    DevCamera d{};
    const dq q{c.pose.rotation[0], c.pose.rotation[1], c.pose.rotation[2], c.pose.rotation[3]};
    const dm3 r = qmatrix(q);  // raster.cpp:72
    for (int k = 0; k < 9; ++k) d.r[k] = r.m[k];
    for (int k = 0; k < 4; ++k) d.q[k] = c.pose.rotation[k];
    for (int k = 0; k < 3; ++k) d.t[k] = c.pose.translation[k];
    // camera_center() = pose.inverse().translation = -(conj(q).rotate(t))  (camera.hpp:23)
    const dq conj{q.w, -q.x, -q.y, -q.z};
    const dv3 ct = qrotate(conj, mk3(c.pose.translation[0], c.pose.translation[1], c.pose.translation[2]));
    d.center[0] = -ct.x;
    d.center[1] = -ct.y;
    d.center[2] = -ct.z;
    d.fx = c.fx;
    d.fy = c.fy;
    d.cx = c.cx;
    d.cy = c.cy;
    d.near_p = c.near_plane;
    d.far_p = c.far_plane;
    const double tan_fovx = c.width / (2.0 * c.fx);  // raster.cpp:74-77
    const double tan_fovy = c.height / (2.0 * c.fy);
    d.limx = 1.3 * tan_fovx;
    d.limy = 1.3 * tan_fovy;
    d.width = c.width;
    d.height = c.height;
    d.tiles_x = (c.width + kTileSize - 1) / kTileSize;
    d.tiles_y = (c.height + kTileSize - 1) / kTileSize;
    return d;
}

void finish_cameras(Plan& p, const gsim_camera* cameras, uint64_t n_cams) {
    p.tile_base.assign(n_cams + 1, 0);
    uint64_t out_off = 0;
    for (uint64_t c = 0; c < n_cams; ++c) {
        DevCamera d = make_dev_camera(cameras[c]);
        d.slot_base = p.slot_base[c];
        d.tile_base = p.tile_base[c];
        d.out_offset = out_off;
        out_off += uint64_t(5) * d.width * d.height;
        const uint32_t tc = uint32_t(d.tiles_x * d.tiles_y);
        p.tile_base[c + 1] = p.tile_base[c] + tc;
        // binning works on a (tiles_x + 1) x (tiles_y + 1) difference grid per camera
        p.max_tc = std::max(p.max_tc, uint32_t((d.tiles_x + 1) * (d.tiles_y + 1)));
        (void)tc;
        p.tiles_x.push_back(d.tiles_x);
        p.cams.push_back(d);
    }
    p.tiles = p.tile_base[n_cams];
    p.out_floats = out_off;
}

// Digit width and pass count of the segmented depth sort (sort.cu): 8-bit digits (27-bit keys of
// near/far 0.05/100: 4 passes). 9-bit digits save a pass there but measured slower per pass
// (config 1, ncu: 67/61/100 us for 3 x 9-bit vs 48/46/44/68 us for 4 x 8-bit: twice the
// digit runs per chunk, twice the look-back words); GSIM_GPU_SORT_BITS=9 selects them.
// Plus the pass-1 chunk table (chunks never straddle cameras).
void finish_sort(Plan& p) {
    static const int forced = [] {  // GSIM_GPU_SORT_BITS=8|9: digit width (measurements)
        const char* e = std::getenv("GSIM_GPU_SORT_BITS");
        const int v = e ? std::atoi(e) : 0;
        return v == 8 || v == 9 ? v : 0;
    }();
    const int b = std::max(1, p.depth_bits);
    const int p8 = (b + 7) / 8, p9 = (b + 8) / 9;
    p.sort_bits = forced ? forced : 8;
    p.sort_passes = p.sort_bits == 9 ? p9 : p8;
    const size_t C = p.cams.size();
    p.chunk_base0.assign(C + 1, 0);
    for (size_t c = 0; c < C; ++c) {
        const uint64_t sc = p.slot_base[c + 1] - p.slot_base[c];
        p.chunk_base0[c + 1] = p.chunk_base0[c] + uint32_t((sc + kOnesweepTile - 1) / kOnesweepTile);
    }
}

struct PaintedRange { uint64_t b, e; int64_t owner; };

// Node painting like PoseTable (raster.cpp:47-62): maximal primitive ranges with the index of the
// node that owns them (later nodes win), -1 where no node does.
std::vector<PaintedRange> paint_nodes(uint64_t n_prims, const gsim_node* nodes, uint64_t n_nodes) {
    std::vector<uint64_t> pts{0, n_prims};
    for (uint64_t k = 0; k < n_nodes; ++k)
        if (nodes[k].begin < nodes[k].end) {
            pts.push_back(nodes[k].begin);
            pts.push_back(nodes[k].end);
        }
    std::sort(pts.begin(), pts.end());
    pts.erase(std::unique(pts.begin(), pts.end()), pts.end());
    std::vector<PaintedRange> ivs;
    for (size_t k = 0; k + 1 < pts.size(); ++k)
        if (pts[k] < pts[k + 1]) ivs.push_back({pts[k], pts[k + 1], -1});
    for (uint64_t k = 0; k < n_nodes; ++k) {
        if (!(nodes[k].begin < nodes[k].end)) continue;
        auto it = std::lower_bound(ivs.begin(), ivs.end(), nodes[k].begin,
                                   [](const PaintedRange& iv, uint64_t v) { return iv.b < v; });
        for (; it != ivs.end() && it->b < nodes[k].end; ++it) it->owner = int64_t(k);
    }
    std::vector<PaintedRange> merged;
    for (const auto& iv : ivs) {
        if (!merged.empty() && merged.back().owner == iv.owner && merged.back().e == iv.b)
            merged.back().e = iv.e;
        else
            merged.push_back(iv);
    }
    if (merged.empty()) merged.push_back({0, 0, -1});
    return merged;
}

// (camera, primitive) slots of every camera: the primitives of nodes of its env (or of no env).
std::vector<uint64_t> camera_slots(uint64_t n_prims, const gsim_node* nodes, uint64_t n_nodes,
                                   const gsim_camera* cameras, uint64_t n_cams) {
    const std::vector<PaintedRange> merged = paint_nodes(n_prims, nodes, n_nodes);
    std::vector<uint64_t> out(n_cams, 0);
    for (const auto& iv : merged)
        for (uint64_t c = 0; c < n_cams; ++c)
            if (iv.owner < 0 || nodes[iv.owner].env < 0 || nodes[iv.owner].env == cameras[c].env)
                out[c] += iv.e - iv.b;
    return out;
}

// Paint node ranges like PoseTable (raster.cpp:47-62) into maximal segments and assign each
// (camera, primitive) a record slot; cameras' slot lists keep primitive order.
Plan build_plan(uint64_t n_prims, const gsim_node* nodes, uint64_t n_nodes,
                const gsim_camera* cameras, uint64_t n_cams) {
    Plan p;
    for (uint64_t c = 0; c < n_cams; ++c) validate_camera(cameras[c], c);
    for (uint64_t k = 0; k < n_nodes; ++k)
        if (nodes[k].end > n_prims)
            throw ValidationError{"node " + std::to_string(k) + " range exceeds field size"};

    const std::vector<PaintedRange> merged = paint_nodes(n_prims, nodes, n_nodes);
    auto visible = [&](const PaintedRange& iv, uint64_t c) {
        if (iv.owner < 0) return true;
        const int env = nodes[iv.owner].env;
        return env < 0 || env == cameras[c].env;
    };
    p.slot_base.assign(n_cams + 1, 0);
    for (uint64_t c = 0; c < n_cams; ++c) {
        uint64_t s = 0;
        for (const auto& iv : merged)
            if (visible(iv, c)) s += iv.e - iv.b;
        p.slot_base[c + 1] = p.slot_base[c] + s;
    }
    p.slots = p.slot_base[n_cams];
    if (p.slots >= 0xFFFFFFFFull)
        throw ValidationError{"batch has " + std::to_string(p.slots) +
                              " (camera, primitive) slots; split it below 2^32"};
    std::vector<uint64_t> running(n_cams, 0);
    for (const auto& iv : merged) {
        DevSegment s{};
        s.begin = iv.b;
        s.end = iv.e;
        if (iv.owner < 0) {
            s.q[0] = 1.0;  // RigidTransform::identity()
        } else {
            for (int k = 0; k < 4; ++k) s.q[k] = nodes[iv.owner].pose.rotation[k];
            for (int k = 0; k < 3; ++k) s.t[k] = nodes[iv.owner].pose.translation[k];
        }
        s.entry_begin = uint32_t(p.entries.size());
        for (uint64_t c = 0; c < n_cams; ++c) {
            if (!visible(iv, c)) continue;
            SegEntry e{};
            e.cam = uint32_t(c);
            e.slot_base = p.slot_base[c] + running[c];
            running[c] += iv.e - iv.b;
            p.entries.push_back(e);
        }
        s.entry_count = uint32_t(p.entries.size()) - s.entry_begin;
        p.segs.push_back(s);
        p.seg_owner.push_back(int32_t(iv.owner));
    }
    finish_cameras(p, cameras, n_cams);
    // Record key = float32 depth bits rebased to [near_min, far_max]: near < z < far implies
    // RN(near) <= RN(z) <= RN(far), and positive floats order like their bit patterns, so the
    // rebased key keeps the reference's depth_sort_key order. The camera is the sort's segment.
    if (n_cams) {
        double near_min = cameras[0].near_plane, far_max = cameras[0].far_plane;
        for (uint64_t c = 1; c < n_cams; ++c) {
            near_min = std::min(near_min, cameras[c].near_plane);
            far_max = std::max(far_max, cameras[c].far_plane);
        }
        p.key_base = float_bits(near_min);
        const uint64_t span = uint64_t(float_bits(far_max)) - p.key_base;
        p.depth_bits = int(ceil_log2_bits(span + 2));  // keeps kInvalidKey unreachable
    }
    finish_sort(p);
    return p;
}

// Camera plan for rasterize(splats): one camera, slot = splat index, full 32-bit depth keys,
// no validation (rasterize does not call validate_camera in the reference).
Plan build_splat_plan(uint64_t n, const gsim_camera& cam) {
    if (cam.width < 1 || cam.height < 1 || cam.width > kMaxTilesPerAxis * kTileSize ||
        cam.height > kMaxTilesPerAxis * kTileSize)
        throw ValidationError{"rasterize: resolution outside 1..4096"};
    Plan p;
    p.slot_base = {0, n};
    p.slots = n;
    finish_cameras(p, &cam, 1);
    p.key_base = 0;
    p.depth_bits = 32;
    finish_sort(p);
    return p;
}

template <class T>
size_t append_bytes(std::vector<char>& blob, const std::vector<T>& v) {
    const size_t off = (blob.size() + 15) & ~size_t(15);
    blob.resize(off + v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
    return off;
}

// One H2D copy per frame: the plan tables are packed into a pinned blob (double-buffered, so
// building frame k+1 never waits for frame k) and copied into one device blob; the kernels read
// them through pointers into that blob. Stream order keeps frame k's kernels ahead of the copy.
void upload_plan(gsim_gpu_context* ctx, const Plan& p) {
    std::vector<char>& blob = ctx->blob_host;
    blob.clear();
    const size_t o_cams = append_bytes(blob, p.cams);
    const size_t o_sb = append_bytes(blob, p.slot_base);
    const size_t o_tb = append_bytes(blob, p.tile_base);
    const size_t o_tx = append_bytes(blob, p.tiles_x);
    const size_t o_cb0 = append_bytes(blob, p.chunk_base0);
    const size_t o_seg = append_bytes(blob, p.segs);
    const size_t o_ent = append_bytes(blob, p.entries);
    const size_t o_st = append_bytes(blob, p.seg_track);
    const int k = ctx->staging_index;
    ctx->staging_index ^= 1;
    GSIM_CK(cudaEventSynchronize(ctx->staging_ev[k]));  // its copy (two frames ago) landed
    ctx->staging[k].reserve(blob.size());
    std::memcpy(ctx->staging[k].ptr, blob.data(), blob.size());
    ctx->plan_dev.reserve(blob.size());
    GSIM_CK(cudaMemcpyAsync(ctx->plan_dev.ptr, ctx->staging[k].ptr, blob.size(),
                            cudaMemcpyHostToDevice, ctx->stream));
    GSIM_CK(cudaEventRecord(ctx->staging_ev[k], ctx->stream));
    ctx->stats.h2d_bytes = blob.size();
    ctx->stats.d2h_bytes = 0;
    char* d = ctx->plan_dev.ptr;
    ctx->cams = reinterpret_cast<DevCamera*>(d + o_cams);
    ctx->cam_slot_base = reinterpret_cast<uint64_t*>(d + o_sb);
    ctx->cam_tile_base = reinterpret_cast<uint32_t*>(d + o_tb);
    ctx->cam_tiles_x = reinterpret_cast<int*>(d + o_tx);
    ctx->cam_chunk_base0 = reinterpret_cast<uint32_t*>(d + o_cb0);
    ctx->segs = reinterpret_cast<DevSegment*>(d + o_seg);
    ctx->entries = reinterpret_cast<SegEntry*>(d + o_ent);
    ctx->seg_track = p.seg_track.empty() ? nullptr : reinterpret_cast<int32_t*>(d + o_st);
}

void record_ev(gsim_gpu_context* ctx, int e) {
    if (ctx->profiling) GSIM_CK(cudaEventRecord(ctx->ev[e], ctx->stream));
}

void check_launch() { GSIM_CK(cudaGetLastError()); }

// The scatter's peer method by camera size: lane bitmaps (8 B per tile-grid cell and warp) up to
// kBitmapCells cells, the u8 probe (5 B) beyond, so large cameras keep several warps per SM.
constexpr uint32_t kBitmapCells = 2048;

bool bitmap_peers_for(uint32_t max_tc) { return max_tc <= kBitmapCells; }

int bin_warps_for(uint32_t max_tc) {
    static const int cap = [] {
        const char* e = std::getenv("GSIM_GPU_BIN_WARPS");
        const int v = e ? std::atoi(e) : 4;  // 4 measured faster than 8 (occupancy)
        return v >= 1 && v <= 8 ? v : 4;
    }();
    const size_t cells = size_t(max_tc) + 32;  // + one spare cell per lane (bin.cu kSpare)
    const size_t per_warp = bitmap_peers_for(max_tc) ? cells * 8 : (cells * 5 + 15) & ~size_t(15);
    const size_t budget = 200 * 1024;
    const int w = int(std::min<size_t>(size_t(cap), budget / std::max<size_t>(per_warp, 1)));
    if (w < 1)
        throw ValidationError{"camera with " + std::to_string(max_tc) +
                              " tiles exceeds the binning shared-memory budget (40960 tiles)"};
    return w;
}

// Records per binning warp: 1024, fewer for small batches so the count and scatter kernels
// still run ~8 warps per SM (a warp walks its records serially: config 0 has 93k visible).
int warp_records_for(uint64_t slots, int n_sms) {
    static const int forced = [] {  // GSIM_GPU_WARP_RECORDS: 128..1024 (power of two)
        const char* e = std::getenv("GSIM_GPU_WARP_RECORDS");
        const int v = e ? std::atoi(e) : 0;
        return v >= 128 && v <= kWarpRecords && (v & (v - 1)) == 0 ? v : 0;
    }();
    if (forced) return forced;
    const uint64_t per = slots / (uint64_t(std::max(n_sms, 1)) * 8);
    int w = kWarpRecords;
    while (w > 128 && uint64_t(w) > per) w >>= 1;
    return w;
}

// Workspaces sized for a plan (grow-only).
void reserve_workspace(gsim_gpu_context* ctx, const Plan& p) {
    const uint64_t S = std::max<uint64_t>(p.slots, 1);
    const uint64_t C = std::max<uint64_t>(p.cams.size(), 1);
    ctx->records.reserve(S);
    ctx->keys.reserve(S);
    ctx->rects.reserve(S);
    ctx->sort_rects.reserve(S);
    for (int k = 0; k < 2; ++k) {
        ctx->dk[k].reserve(S);
        ctx->dv[k].reserve(S);
    }
    // P / S is about 3 for the BASELINE scenes; 8 x slots (4 B each) makes an overflow of an
    // asynchronous frame practically impossible and costs 32 B per slot of HBM.
    if (ctx->fixed_initial_capacity == 0 && ctx->pair_capacity < 8 * S + (1u << 20))
        ctx->pair_capacity = 8 * S + (1u << 20);
    ctx->vals.reserve(std::max<uint64_t>(ctx->pair_capacity, 1));
    const uint64_t words = ((S + kOnesweepTile - 1) / kOnesweepTile + C) * (uint64_t(1) << p.sort_bits);
    ctx->sort_hist.reserve(C * p.sort_passes * (uint64_t(1) << p.sort_bits));
    ctx->sort_chunk_base.reserve(C + 1);
    if (words > ctx->status.cap) {
        ctx->status.reserve(words);
        GSIM_CK(cudaMemsetAsync(ctx->status.ptr, 0, ctx->status.cap * sizeof(uint64_t), ctx->stream));
    }
    ctx->zero_block.reserve(kZeroCams + C);
    ctx->counts.reserve(4);
    const uint64_t R = uint64_t(warp_records_for(p.slots, ctx->num_sms)) * bin_warps_for(p.max_tc);
    const uint64_t kmax = (S + R - 1) / R + C;
    ctx->cam_vbase.reserve(C + 1);
    ctx->cam_chunk_base.reserve(C + 1);
    ctx->cam_pairs.reserve(C);
    ctx->cam_mbase.reserve(C + 1);
    ctx->cam_pair_base.reserve(C + 1);
    ctx->chunk_cam.reserve(kmax);
    ctx->n_chunks.reserve(1);
    ctx->count_matrix.reserve(uint64_t(std::max<uint32_t>(p.max_tc, 1)) * kmax);
    ctx->tile_count.reserve(std::max<uint32_t>(p.tiles, 1));
    ctx->tile_rel.reserve(std::max<uint32_t>(p.tiles, 1));
}

float smallest_float_geq(double x) {
    float f = float(x);
    if (double(f) < x) f = std::nextafter(f, INFINITY);
    return f;
}

BinArgs make_bin_args(gsim_gpu_context* ctx, const Plan& p) {
    BinArgs b{};
    b.keys = ctx->keys.ptr;
    b.n_slots = p.slots;
    b.cam_slot_base = ctx->cam_slot_base;
    b.sort_bits = p.sort_bits;
    b.sort_passes = p.sort_passes;
    b.n_cams = int(p.cams.size());
    // the last depth pass writes the slots into dv[o] and the carried rects into dk[o]
    const int last_o = (p.sort_passes - 1) & 1;
    b.sorted_slots = ctx->dv[last_o].ptr;
    b.sorted_rects = ctx->dk[last_o].ptr;
    b.cam_tile_base = ctx->cam_tile_base;
    b.cam_tiles_x = ctx->cam_tiles_x;
    b.cam_visible = ctx->zero_block.ptr + kZeroCams;
    b.cam_vbase = ctx->cam_vbase.ptr;
    b.cam_chunk_base = ctx->cam_chunk_base.ptr;
    b.cam_mbase = ctx->cam_mbase.ptr;
    b.cam_pairs = ctx->cam_pairs.ptr;
    b.cam_pair_base = ctx->cam_pair_base.ptr;
    b.chunk_cam = ctx->chunk_cam.ptr;
    b.n_chunks = ctx->n_chunks.ptr;
    b.counts = ctx->count_matrix.ptr;
    b.tile_count = ctx->tile_count.ptr;
    b.tile_rel = ctx->tile_rel.ptr;
    b.hist = ctx->sort_hist.ptr;
    b.sort_chunk_base = ctx->sort_chunk_base.ptr;
    b.totals = ctx->counts.ptr;
    ctx->readback.reserve(64);
    void* host_totals = nullptr;
    GSIM_CK(cudaHostGetDevicePointer(&host_totals, ctx->readback.ptr, 0));
    b.host_totals = static_cast<unsigned long long*>(host_totals);
    b.vals_out = ctx->vals.ptr;
    b.capacity = ctx->pair_capacity;
    b.max_tc = int(p.max_tc);
    b.bin_warps = bin_warps_for(p.max_tc);
    b.bitmap_peers = bitmap_peers_for(p.max_tc) ? 1 : 0;
    b.warp_records = warp_records_for(p.slots, ctx->num_sms);
    b.chunk_records = b.warp_records * b.bin_warps;
    return b;
}

void queue_camera_copies(gsim_gpu_context* ctx, const Plan& p, const float* out);
void queue_camera_copies_enc(gsim_gpu_context* ctx, const Plan& p, const uint8_t* dev, uint32_t bpp);

void launch_raster_stage(gsim_gpu_context* ctx, const Plan& p, const gsim_raster_options& opt,
                         float* out) {
    RasterArgs rr{};
    rr.records = ctx->records.ptr;
    rr.values = ctx->vals.ptr;
    rr.tile_rel = ctx->tile_rel.ptr;
    rr.tile_count = ctx->tile_count.ptr;
    rr.cam_pair_base = ctx->cam_pair_base.ptr;
    rr.cams = ctx->cams;
    rr.cam_tile_base = ctx->cam_tile_base;
    rr.n_cams = int(p.cams.size());
    rr.normalize_depth = opt.normalize_depth;
    rr.cutoff = smallest_float_geq(opt.transmittance_cutoff);
    rr.out = out;
    rr.consumed = ctx->counts.ptr + 2;
    rr.capacity = ctx->pair_capacity;
    rr.n_slots = std::max<uint64_t>(p.slots, 1);
    rr.enc = ctx->frame_enc;
    rr.rect_w = ctx->raster_rect_w;
    rr.batch = ctx->raster_batch;
    rr.exact_cull = ctx->raster_exact_cull;
    rr.bulk_copy = ctx->raster_bulk;
    rr.grid_cap = ctx->raster_ctas > 0 ? ctx->raster_ctas * ctx->num_sms : 0;
    rr.valid_alpha = ctx->frame_valid_alpha;
    if (rr.enc.flags && ctx->frame_enc_only) rr.out = nullptr;
    const bool overlap_enc = ctx->frame_enc_host && rr.enc.flags;
    const bool overlap = (ctx->frame_outs && rr.out) || overlap_enc;
    // one launch per camera when host copies overlap the compositing (each camera's copies wait
    // on the event after its launch: ordinary stream dependencies, no stream memory operations,
    // which can deadlock through shared hardware queues), else one launch for the batch
    const size_t n_launch = overlap ? p.cams.size() : 1;
    while (overlap && ctx->cam_evs.size() < p.cams.size()) {
        cudaEvent_t e;
        GSIM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->cam_evs.push_back(e);
    }
    uint32_t tile = 0;
    for (size_t k = 0; k < n_launch; ++k) {
        const uint32_t end = overlap ? tile + uint32_t(p.cams[k].tiles_x) * uint32_t(p.cams[k].tiles_y)
                                     : uint32_t(p.tiles);
        rr.tile_begin = tile;
        if (rr.grid_cap > 0 && uint32_t(rr.grid_cap) < end - tile) {
            rr.tile_ticket = ctx->zero_block.ptr + kZeroTickets + kRasterTicket;
            GSIM_CK(cudaMemsetAsync(rr.tile_ticket, 0, sizeof(uint32_t), ctx->stream));
        } else {
            rr.tile_ticket = nullptr;
        }
        launch_raster(rr, end, ctx->stream);
        check_launch();
        if (overlap) GSIM_CK(cudaEventRecord(ctx->cam_evs[k], ctx->stream));
        tile = end;
    }
    ctx->launches_total += n_launch - 1;
    if (overlap_enc)
        queue_camera_copies_enc(ctx, p, rr.enc.dst, encoded_bpp(rr.enc.flags));
    else if (overlap)
        queue_camera_copies(ctx, p, out);
}

// Pair positions (bin.cu scatter, raster.cu list bounds) are 32-bit: a camera group with 2^32 or
// more (tile, record) pairs would wrap them (writes stay inside the buffer: they are bounded by
// the capacity), so its frame is refused instead of being returned scrambled.
void check_pair_positions(unsigned long long pairs) {
    if (pairs >= (1ull << 32))
        throw ValidationError{"camera group has " + std::to_string(pairs) +
                              " (tile, splat) pairs (>= 2^32); render fewer cameras per call"};
}

// K3 + K4 over records/keys/rects already produced for `p` (by K2 or the splat converter).
void run_sort_and_raster(gsim_gpu_context* ctx, const Plan& p, const gsim_raster_options& opt,
                         float* out, uint64_t& launches, bool wait_for_count) {
    cudaStream_t s = ctx->stream;
    const uint64_t S = p.slots;
    const int n_sms = ctx->num_sms;

    // digit histograms per (camera, pass), then the chunk tables (need only the counts)
    BinArgs b = make_bin_args(ctx, p);
    launch_key_hist(b, n_sms * 6, s);
    check_launch();
    launch_chunk_table(b, s);
    check_launch();
    launches += 2;

    // segmented onesweep passes over the depth keys; pass 1 compacts the culled slots away
    const int passes = p.sort_passes, radix = 1 << p.sort_bits;
    OnesweepArgs oa{};
    static const uint32_t backoff = [] {  // GSIM_GPU_SORT_BACKOFF: look-back retry sleep (ns)
        const char* e = std::getenv("GSIM_GPU_SORT_BACKOFF");
        const int v = e ? std::atoi(e) : 64;
        return uint32_t(v < 0 ? 0 : v > 1000 ? 1000 : v);
    }();
    oa.backoff_ns = backoff;
    oa.status = ctx->status.ptr;
    oa.n_cams = int(p.cams.size());
    oa.vbase = ctx->cam_vbase.ptr;
    oa.hist_stride = uint64_t(passes) * radix;
    uint64_t dgrid = (S + kOnesweepTile - 1) / kOnesweepTile + p.cams.size();
    static const int sort_ctas = [] {
        const char* e = std::getenv("GSIM_GPU_SORT_CTAS");  // resident onesweep CTAs per SM
        const int v = e ? std::atoi(e) : kOnesweepMinBlocks;
        return v < 1 ? 1 : v > kOnesweepMinBlocks ? kOnesweepMinBlocks : v;
    }();
    dgrid = std::max<uint64_t>(1, std::min<uint64_t>(dgrid, uint64_t(n_sms) * sort_ctas));
    const uint32_t* kin = ctx->keys.ptr;
    const uint32_t* vin = nullptr;
    const uint32_t* rin = ctx->rects.ptr;
    for (int pass = 0; pass < passes; ++pass) {
        const int o = pass & 1;
        const bool last = pass == passes - 1;
        oa.keys_in = kin;
        oa.vals_in = vin;
        oa.keys_out = ctx->dk[o].ptr;
        oa.vals_out = ctx->dv[o].ptr;
        oa.seg_base64 = ctx->cam_slot_base;
        oa.seg_base32 = ctx->cam_vbase.ptr;
        oa.chunk_base = pass == 0 ? ctx->cam_chunk_base0 : ctx->sort_chunk_base.ptr;
        oa.hist = ctx->sort_hist.ptr + uint64_t(pass) * radix;
        oa.ticket = ctx->zero_block.ptr + kZeroTickets + pass;
        oa.epoch = ctx->next_epoch();
        oa.shift = p.sort_bits * pass;
        // the rects move with the keys: pass 1 reads them in slot order, the passes alternate
        // between sort_rects and the slot-order rect plane (free once pass 1 has read it), and
        // the last pass, which writes no keys, puts them into its own key output buffer
        oa.rects_in = rin;
        oa.rects_out = last ? ctx->dk[o].ptr : (pass & 1) ? ctx->rects.ptr : ctx->sort_rects.ptr;
        launch_onesweep(oa, p.sort_bits, pass == 0, !last, int(dgrid), s);
        check_launch();
        ++launches;
        kin = ctx->dk[o].ptr;
        vin = ctx->dv[o].ptr;
        rin = oa.rects_out;
    }
    record_ev(ctx, kEvDepth);

    // tile binning: counts, scans, camera bases
    const uint64_t kmax = (S + b.chunk_records - 1) / b.chunk_records + p.cams.size();
    // one CTA of bin_warps warps per unit
    const int chunk_grid = int(std::max<uint64_t>(1, kmax));
    launch_bin_count(b, chunk_grid, s);
    check_launch();
    launch_bin_colscan(b, int(std::max<uint64_t>(1, (uint64_t(p.tiles) + 31) / 32)), s);
    check_launch();
    launch_bin_tilescan(b, int(std::min<uint64_t>(p.cams.size(), uint64_t(n_sms) * 2)), s);
    check_launch();
    launch_bin_campre(b, s);
    check_launch();
    launches += 4;
    // (V, P) reach the host through campre's stores into the page-locked readback (no copy
    // engine operation between the binning and the scatter: a queued copy engine, e.g. behind
    // another context's image copies, would hold the frame there)
    GSIM_CK(cudaEventRecord(ctx->bin_ev, s));
    record_ev(ctx, kEvBin);

    for (int attempt = 0; attempt < 3; ++attempt) {
        b.vals_out = ctx->vals.ptr;
        b.capacity = ctx->pair_capacity;
        static const int scatter_ctas = [] {  // GSIM_GPU_SCATTER_CTAS: per SM, 0 = one per unit
            const char* e = std::getenv("GSIM_GPU_SCATTER_CTAS");
            return e ? std::max(0, std::atoi(e)) : 0;
        }();
        launch_bin_scatter(b, scatter_ctas ? std::min(chunk_grid, n_sms * scatter_ctas) : chunk_grid, s);
        check_launch();
        record_ev(ctx, kEvScatter);
        launch_raster_stage(ctx, p, opt, out);
        record_ev(ctx, kEvRaster);
        launches += 2;
        if (!wait_for_count) {
            // Asynchronous frame: the (V, P) readback is checked by the next call on this
            // context (check_pending), which re-runs scatter + raster on overflow.
            ctx->pending = true;
            ctx->pending_out = out;
            ctx->pending_opt = opt;
            ctx->pending_grid = chunk_grid;
            ctx->pending_enc = ctx->frame_enc;
            ctx->pending_enc_only = ctx->frame_enc_only;
            break;
        }
        GSIM_CK(cudaEventSynchronize(ctx->bin_ev));
        const unsigned long long* rb = static_cast<const unsigned long long*>(ctx->readback.ptr);
        ctx->stats.visible = rb[0];
        ctx->stats.pairs = rb[1];
        check_pair_positions(rb[1]);
        if (rb[1] <= ctx->pair_capacity) break;
        // Pair buffer too small: grow and place + raster again (counts and scans stay valid).
        GSIM_CK(cudaStreamSynchronize(s));
        ctx->pair_capacity = rb[1] + rb[1] / 4 + (1u << 20);
        ctx->vals.reserve(ctx->pair_capacity);
        GSIM_CK(cudaMemsetAsync(ctx->counts.ptr + 2, 0, sizeof(unsigned long long), s));
    }
    if (ctx->stats.pairs > ctx->pair_capacity) throw CudaError{"pair buffer overflow after regrowth"};
    ctx->stats.depth_passes = uint32_t(p.sort_passes);
}

void begin_frame(gsim_gpu_context* ctx, const Plan& p) {
    GSIM_CK(cudaMemsetAsync(ctx->zero_block.ptr + kZeroTickets, 0,
                            (kZeroCams - kZeroTickets + std::max<size_t>(p.cams.size(), 1)) * sizeof(uint32_t),
                            ctx->stream));
    const size_t hist_words = std::max<size_t>(p.cams.size(), 1) * size_t(p.sort_passes) << p.sort_bits;
    GSIM_CK(cudaMemsetAsync(ctx->sort_hist.ptr, 0, hist_words * sizeof(uint32_t), ctx->stream));
    GSIM_CK(cudaMemsetAsync(ctx->counts.ptr, 0, 4 * sizeof(unsigned long long), ctx->stream));
}

void finish_stats(gsim_gpu_context* ctx, const Plan& p, uint64_t launches) {
    ctx->stats.slots = p.slots;
    ctx->stats.tiles = p.tiles;
    ctx->stats.launches = launches;
    ctx->stats.chunks = 0;
    ctx->launches_total += launches;
    ctx->stats.launches_total = ctx->launches_total;
}

PreprocessArgs make_pre_args(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const Plan& p) {
    PreprocessArgs pa{};
    pa.field = scene->f;
    pa.segs = ctx->segs;
    pa.n_segs = int(p.segs.size());
    pa.depth_bits = p.depth_bits;
    pa.entries = ctx->entries;
    pa.cams = ctx->cams;
    pa.records = ctx->records.ptr;
    pa.rects = ctx->rects.ptr;
    pa.keys = ctx->keys.ptr;
    pa.key_base = p.key_base;
    pa.n_cams = uint32_t(p.cams.size());
    return pa;
}

void render_frame(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                  uint64_t n_nodes, const gsim_camera* cameras, uint64_t n_cams,
                  const gsim_raster_options* options, float* device_out, Plan& plan,
                  bool wait_for_count) {
    plan = build_plan(scene->f.n, nodes, n_nodes, cameras, n_cams);
    gsim_raster_options opt{0, 0, 1e-4};
    if (options) opt = *options;
    bool posed = false;
    if (ctx->frame_tracks) {  // render_at: which segments a track drives
        plan.seg_track.resize(plan.segs.size(), -1);
        for (size_t k = 0; k < plan.segs.size(); ++k) {
            const int32_t owner = plan.seg_owner[k];
            if (owner >= 0 && ctx->frame_node_track[owner] >= 0) {
                plan.seg_track[k] = int32_t(ctx->frame_node_track[owner]);
                posed = true;
            }
        }
        if (!posed) plan.seg_track.clear();
    }
    reserve_workspace(ctx, plan);
    upload_plan(ctx, plan);
    if (posed) {
        launch_pose_segments(ctx->frame_tracks->d, ctx->segs, ctx->seg_track,
                             uint32_t(plan.segs.size()), ctx->frame_time, ctx->stream);
        check_launch();
    }
    float* out = device_out;
    if (!out) {
        ctx->out.reserve(std::max<uint64_t>(plan.out_floats, 1));
        out = ctx->out.ptr;
    }
    record_ev(ctx, kEvStart);
    begin_frame(ctx, plan);
    uint64_t launches = posed ? 1 : 0;
    PreprocessArgs pa = make_pre_args(ctx, scene, plan);
    if (plan.slots) {
        launch_preprocess(pa, false, ctx->num_sms, ctx->stream);
        check_launch();
        ++launches;
    }
    record_ev(ctx, kEvPre);
    run_sort_and_raster(ctx, plan, opt, out, launches, wait_for_count);
    finish_stats(ctx, plan, launches);
}

bool check_pending(gsim_gpu_context* ctx);

// A camera batch is rendered in one launch sequence whenever its (camera, primitive) slots stay
// below 2^31 (the kernels index slots in 32 bits): BASELINE config 2 (320 cameras x 1.08M slots)
// is one group. Larger batches are split into consecutive camera groups by slot count; outputs
// keep the batch's camera order. Returns the float offset of every camera's block in the output.
std::vector<uint64_t> render_cameras(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                                     const gsim_node* nodes, uint64_t n_nodes,
                                     const gsim_camera* cameras, uint64_t n_cams,
                                     const gsim_raster_options* options, float* device_out,
                                     bool wait_for_count) {
    std::vector<uint64_t> offsets(n_cams + 1, 0);
    for (uint64_t c = 0; c < n_cams; ++c) {
        validate_camera(cameras[c], c);
        offsets[c + 1] = offsets[c] + uint64_t(5) * cameras[c].width * cameras[c].height;
    }
    float* out = device_out;
    if (!out) {
        ctx->out.reserve(std::max<uint64_t>(offsets[n_cams], 1));
        out = ctx->out.ptr;
    }
    for (uint64_t k = 0; k < n_nodes; ++k)
        if (nodes[k].end > scene->f.n)
            throw ValidationError{"node " + std::to_string(k) + " range exceeds field size"};
    // group boundaries: consecutive cameras while their slots fit the group budget
    std::vector<uint64_t> group_begin{0};
    if (n_cams) {
        const std::vector<uint64_t> cs = camera_slots(scene->f.n, nodes, n_nodes, cameras, n_cams);
        uint64_t acc = 0;
        for (uint64_t c = 0; c < n_cams; ++c) {
            if (c > group_begin.back() && acc + cs[c] > ctx->group_slots) {
                group_begin.push_back(c);
                acc = 0;
            }
            acc += cs[c];
        }
    }
    group_begin.push_back(n_cams);
    uint64_t launches = 0, h2d = 0;
    gsim_target* const targets = ctx->frame_outs;  // host targets of the whole batch, if any
    uint8_t* const enc_host = ctx->frame_enc_host;  // render_encoded host bytes, if any
    ctx->frame_outs = nullptr;
    ctx->frame_enc_host = nullptr;
    const size_t n_groups = group_begin.size() - 1;
    for (size_t gi = 0; gi < n_groups; ++gi) {
        const uint64_t c0 = group_begin[gi];
        const uint64_t g = group_begin[gi + 1] - c0;
        // a re-run group had its copies queued already: the caller copies everything again
        if (c0 > 0 && !wait_for_count && check_pending(ctx)) ctx->copies_stale = true;
        Plan plan;
        const EncodeParams enc_batch = ctx->frame_enc;
        if (enc_batch.flags) ctx->frame_enc.dst += offsets[c0] / 5 * encoded_bpp(enc_batch.flags);
        ctx->frame_outs = targets ? targets + c0 : nullptr;
        ctx->frame_enc_host = enc_host ? enc_host + offsets[c0] / 5 * encoded_bpp(enc_batch.flags) : nullptr;
        render_frame(ctx, scene, nodes, n_nodes, cameras + c0, g, options, out + offsets[c0], plan,
                     wait_for_count);
        ctx->frame_outs = nullptr;
        ctx->frame_enc_host = nullptr;
        ctx->frame_enc = enc_batch;
        launches += ctx->stats.launches;
        h2d += ctx->stats.h2d_bytes;
        ctx->last_plan = std::move(plan);
    }
    ctx->stats.launches = launches;
    ctx->stats.h2d_bytes = h2d;
    ctx->stats.groups = uint32_t(n_groups);
    ctx->stats.last_group_cameras = uint32_t(ctx->last_plan.cams.size());
    return offsets;
}

// Completes the deferred pair-count check of an asynchronous render: by now its readback has
// long landed; on overflow the buffers of that frame are still intact (nothing new has been
// enqueued), so scatter + raster are re-run into the same output before anything else.
// Returns whether they were re-run.
bool check_pending(gsim_gpu_context* ctx) {
    if (!ctx->pending) return false;
    ctx->pending = false;
    GSIM_CK(cudaEventSynchronize(ctx->bin_ev));
    const unsigned long long* rb = static_cast<const unsigned long long*>(ctx->readback.ptr);
    ctx->stats.visible = rb[0];
    ctx->stats.pairs = rb[1];
    check_pair_positions(rb[1]);
    if (rb[1] <= ctx->pair_capacity) return false;
    GSIM_CK(cudaStreamSynchronize(ctx->stream));
    ctx->pair_capacity = rb[1] + rb[1] / 4 + (1u << 20);
    ctx->vals.reserve(ctx->pair_capacity);
    GSIM_CK(cudaMemsetAsync(ctx->counts.ptr + 2, 0, sizeof(unsigned long long), ctx->stream));
    BinArgs b = make_bin_args(ctx, ctx->last_plan);
    launch_bin_scatter(b, ctx->pending_grid, ctx->stream);
    check_launch();
    const EncodeParams enc = ctx->frame_enc;
    const bool enc_only = ctx->frame_enc_only;
    ctx->frame_enc = ctx->pending_enc;
    ctx->frame_enc_only = ctx->pending_enc_only;
    launch_raster_stage(ctx, ctx->last_plan, ctx->pending_opt, ctx->pending_out);
    ctx->frame_enc = enc;
    ctx->frame_enc_only = enc_only;
    GSIM_CK(cudaStreamSynchronize(ctx->stream));
    return true;
}

// ---- output encoding (image_io.cpp) ---------------------------------------------------------

// quantize8(linear_to_srgb(v)) of the reference (image_io.cpp:19-22, :43-45), restated for the
// threshold table only; the device never evaluates pow.
uint32_t srgb_code(float f) {
    double v = std::clamp(double(f), 0.0, 1.0);
    v = v <= 0.0031308 ? 12.92 * v : 1.055 * std::pow(v, 1.0 / 2.4) - 0.055;
    return uint32_t(std::clamp(std::lround(v * 255.0), 0l, 255l));
}

// thr[k] = smallest float in [0, 1] whose code is >= k (binary search over the float bit
// patterns of [0, 1], on which the code is monotone non-decreasing); thr[0] = -inf.
void build_srgb_thresholds(float* thr) {
    thr[0] = -std::numeric_limits<float>::infinity();
    for (uint32_t k = 1; k < 256; ++k) {
        uint32_t lo = 0, hi = 0x3f800000u;  // code(as_float(hi)) = 255 >= k
        while (lo < hi) {
            const uint32_t mid = lo + (hi - lo) / 2;
            float f;
            std::memcpy(&f, &mid, 4);
            if (srgb_code(f) >= k) hi = mid; else lo = mid + 1;
        }
        std::memcpy(&thr[k], &lo, 4);
    }
}

EncodeParams make_encode_params(gsim_gpu_context* ctx, const gsim_encode_options* o, uint8_t* dst) {
    if (!o) throw ValidationError{"encode: options must not be NULL"};
    if (o->flags == 0 || (o->flags & ~uint32_t(GSIM_ENCODE_RGB8 | GSIM_ENCODE_ALPHA8 |
                                               GSIM_ENCODE_DEPTH16 | GSIM_ENCODE_DEPTH_PFM)))
        throw ValidationError{"encode: flags must be a non-empty set of GSIM_ENCODE_* bits"};
    if ((o->flags & GSIM_ENCODE_DEPTH16) && !std::isfinite(o->depth_scale))
        throw ValidationError{"encode: depth_scale must be finite"};
    if (o->srgb && (o->flags & GSIM_ENCODE_RGB8) && !ctx->srgb_ready) {
        float thr[256];
        build_srgb_thresholds(thr);
        ctx->srgb_thr.reserve(256);
        GSIM_CK(cudaMemcpy(ctx->srgb_thr.ptr, thr, sizeof(thr), cudaMemcpyHostToDevice));
        ctx->srgb_ready = true;
    }
    EncodeParams e{};
    e.dst = dst;
    e.srgb_thr = ctx->srgb_thr.ptr;
    e.depth_scale = o->depth_scale;
    e.flags = o->flags;
    e.srgb = (o->srgb && (o->flags & GSIM_ENCODE_RGB8)) ? 1 : 0;
    return e;
}

// Encode float targets already on the device ([rgb|depth|alpha] per camera, consecutive).
void encode_device(gsim_gpu_context* ctx, const float* src, const uint32_t* widths,
                   const uint32_t* heights, uint64_t n, const EncodeParams& e) {
    std::vector<EncodeCam> cams(n);
    uint64_t src_off = 0, dst_off = 0;
    uint32_t max_px = 0;
    const uint32_t bpp = encoded_bpp(e.flags);
    for (uint64_t c = 0; c < n; ++c) {
        cams[c] = EncodeCam{widths[c], heights[c], src_off, dst_off};
        const uint64_t npx = uint64_t(widths[c]) * heights[c];
        src_off += 5 * npx;
        dst_off += bpp * npx;
        max_px = std::max<uint32_t>(max_px, uint32_t(npx));
    }
    ctx->enc_cams.reserve(std::max<uint64_t>(n, 1));
    GSIM_CK(cudaMemcpyAsync(ctx->enc_cams.ptr, cams.data(), n * sizeof(EncodeCam),
                            cudaMemcpyHostToDevice, ctx->stream));
    EncodeKernelArgs a{src, ctx->enc_cams.ptr, e};
    for (uint64_t c0 = 0; c0 < n; c0 += 65535) {  // grid.y limit
        a.cams = ctx->enc_cams.ptr + c0;
        launch_encode(a, uint32_t(std::min<uint64_t>(65535, n - c0)), max_px, ctx->stream);
        check_launch();
    }
}

// Device field of n primitives: 11 double planes, then ceil(3K/4) float4 SH planes whose base
// stays 256-byte aligned for any n.
gsim_gpu_scene* alloc_scene(gsim_gpu_context* ctx, uint64_t n, int degree) {
    const int K = (degree + 1) * (degree + 1);
    const int planes = (3 * K + 3) / 4;
    const uint64_t nn = std::max<uint64_t>(n, 1);
    const size_t geo_bytes = (11 * nn * sizeof(double) + 255) & ~size_t(255);
    const size_t sh_bytes = size_t(planes) * nn * sizeof(float4);
    auto* sc = new gsim_gpu_scene();
    sc->ctx = ctx;
    if (cudaMalloc(&sc->mem, geo_bytes + sh_bytes) != cudaSuccess) {
        delete sc;
        throw CudaError{"scene: device allocation of " + std::to_string(geo_bytes + sh_bytes) +
                        " bytes failed"};
    }
    double* g = static_cast<double*>(sc->mem);
    sc->f.n = n;
    sc->f.sh_degree = degree;
    sc->f.sh_planes = planes;
    sc->f.mx = g + 0 * nn; sc->f.my = g + 1 * nn; sc->f.mz = g + 2 * nn;
    sc->f.sx = g + 3 * nn; sc->f.sy = g + 4 * nn; sc->f.sz = g + 5 * nn;
    sc->f.qw = g + 6 * nn; sc->f.qx = g + 7 * nn; sc->f.qy = g + 8 * nn; sc->f.qz = g + 9 * nn;
    sc->f.opacity = g + 10 * nn;
    sc->f.sh = reinterpret_cast<float4*>(static_cast<char*>(sc->mem) + geo_bytes);
    ctx->scenes.insert(sc);  // callers hold ctx->mu (Guard)
    return sc;
}

void discard_scene(gsim_gpu_context* ctx, gsim_gpu_scene* sc) {  // failed load / upload
    ctx->scenes.erase(sc);
    cudaFree(sc->mem);
    delete sc;
}

// ---- splat PLY (splat_ply.cpp:40-162) ----------------------------------------------------------

int sh_coeff_count(int degree) { return (degree + 1) * (degree + 1); }  // sh.hpp

std::vector<std::string> ply_expected_properties(int degree) {  // splat_ply.cpp:19-28
    std::vector<std::string> props = {"x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"};
    const int rest = 3 * (sh_coeff_count(degree) - 1);
    for (int i = 0; i < rest; ++i) props.push_back("f_rest_" + std::to_string(i));
    props.push_back("opacity");
    for (int i = 0; i < 3; ++i) props.push_back("scale_" + std::to_string(i));
    for (int i = 0; i < 4; ++i) props.push_back("rot_" + std::to_string(i));
    return props;
}

struct FileCloser {
    void operator()(std::FILE* f) const { if (f) std::fclose(f); }
};

// The header contract of load_splat_ply (splat_ply.cpp:40-113): the "ply" magic, keyword lines
// up to end_header, binary_little_endian, one vertex element, float properties in the 3DGS order
// of SH degree 0-3 (the degree follows from the f_rest count). The header is first read into a
// PlyHeader (every line classified by its keyword), then judged as a whole; any violation is a
// validation error (status 2), as every format_error of the reference is.
struct PlyHeader {
    bool magic = false, closed = false;
    std::vector<std::string> formats;                      // format names, in order
    std::vector<std::pair<std::string, uint64_t>> elements;  // (name, count)
    std::vector<std::pair<std::string, std::string>> props;  // (type, name)
    std::vector<std::string> unknown;                      // unexpected keywords
};

PlyHeader read_ply_header(std::FILE* fp) {
    PlyHeader h;
    std::string line;
    auto next_line = [&](bool strip_cr) {
        line.clear();
        int ch;
        while ((ch = std::fgetc(fp)) != EOF && ch != '\n') line.push_back(char(ch));
        const bool got = ch != EOF || !line.empty();
        if (strip_cr && !line.empty() && line.back() == '\r') line.pop_back();
        return got;
    };
    if (!next_line(false)) return h;
    h.magic = line == "ply";  // the reference compares the raw first line (no CR stripping)
    if (!h.magic) return h;
    while (next_line(true)) {
        if (line == "end_header") {
            h.closed = true;
            break;
        }
        std::vector<std::string> f;  // whitespace-separated fields
        size_t i = 0;
        while (i < line.size()) {
            while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
            const size_t j0 = i;
            while (i < line.size() && !std::isspace(static_cast<unsigned char>(line[i]))) ++i;
            if (i > j0) f.emplace_back(line, j0, i - j0);
        }
        f.resize(std::max<size_t>(f.size(), 3));
        const std::string& kw = f[0];
        if (kw.empty() || kw == "comment") continue;
        if (kw == "format") h.formats.push_back(f[1]);
        else if (kw == "element") h.elements.emplace_back(f[1], std::strtoull(f[2].c_str(), nullptr, 10));
        else if (kw == "property") h.props.emplace_back(f[1], f[2]);
        else h.unknown.push_back(kw);
    }
    return h;
}

// Validates the header; returns (SH degree, primitive count).
std::pair<int, uint64_t> check_ply_header(const PlyHeader& h, const std::string& who) {
    auto fail = [&](const std::string& why) { throw ValidationError{who + ": " + why}; };
    if (!h.magic) fail("missing 'ply' magic");
    for (const auto& fmt : h.formats)
        if (fmt != "binary_little_endian") fail("format must be binary_little_endian, got '" + fmt + "'");
    uint64_t count = 0;
    for (const auto& e : h.elements) {
        if (e.first != "vertex") fail("unexpected element '" + e.first + "'");
        count = e.second;
    }
    for (const auto& pr : h.props)
        if (pr.first != "float") fail("property '" + pr.second + "' must be float, got '" + pr.first + "'");
    if (!h.unknown.empty()) fail("unexpected header token '" + h.unknown.front() + "'");
    if (!h.closed) fail("header missing end_header");
    if (h.formats.empty()) fail("header missing format line");
    if (h.elements.empty()) fail("header missing element vertex line");
    const size_t rest = size_t(std::count_if(h.props.begin(), h.props.end(), [](const auto& pr) {
        return pr.second.compare(0, 7, "f_rest_") == 0;
    }));
    int degree = -1;
    for (int d = 0; d <= 3; ++d)
        if (rest == size_t(3 * (sh_coeff_count(d) - 1))) degree = d;
    if (degree < 0) fail("f_rest property count " + std::to_string(rest) + " matches no SH degree in [0,3]");
    const std::vector<std::string> want = ply_expected_properties(degree);
    for (size_t k = 0; k < std::max(want.size(), h.props.size()); ++k) {
        if (k >= h.props.size()) fail("missing property '" + want[k] + "'");
        if (k >= want.size()) fail("unexpected extra property '" + h.props[k].second + "'");
        if (h.props[k].second != want[k])
            fail("property " + std::to_string(k) + " is '" + h.props[k].second + "', expected '" + want[k] + "'");
    }
    if (count >= 0xFFFFFFFFull) fail("more than 2^32 - 1 primitives");
    return {degree, count};
}

gsim_gpu_scene* load_ply(gsim_gpu_context* ctx, const std::string& path) {
    std::unique_ptr<std::FILE, FileCloser> fp(std::fopen(path.c_str(), "rb"));
    if (!fp) throw CudaError{"cannot open splat PLY '" + path + "'"};  // io_error -> status 1
    const std::string who = "'" + path + "'";
    const auto [degree, count] = check_ply_header(read_ply_header(fp.get()), who);
    const std::vector<std::string> expected = ply_expected_properties(degree);

    // Payload: pinned double-buffered chunks, disk read of chunk k+1 overlapping the H2D of k.
    const int stride = int(expected.size());
    const uint64_t bytes = count * uint64_t(stride) * sizeof(float);
    DevBuf<char> raw;
    PinnedBuf stage[2];
    struct Release {  // scratch of this call only, released on every path
        DevBuf<char>& raw;
        PinnedBuf* stage;
        ~Release() { raw.release(); stage[0].release(); stage[1].release(); }
    } release{raw, stage};
    raw.reserve(std::max<uint64_t>(bytes, 4));
    constexpr size_t kChunk = size_t(32) << 20;
    cudaEvent_t done[2] = {nullptr, nullptr};
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() { for (int k = 0; k < 2; ++k) if (e[k]) cudaEventDestroy(e[k]); }
    } evg{done};
    for (int k = 0; k < 2; ++k) {
        stage[k].reserve(std::min<uint64_t>(std::max<uint64_t>(bytes, 64), kChunk));
        GSIM_CK(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
    }
    uint64_t off = 0;
    int k = 0;
    bool truncated = false;
    while (off < bytes) {
        const size_t want = size_t(std::min<uint64_t>(kChunk, bytes - off));
        GSIM_CK(cudaEventSynchronize(done[k]));
        const size_t got = std::fread(stage[k].ptr, 1, want, fp.get());
        if (got) {
            GSIM_CK(cudaMemcpyAsync(raw.ptr + off, stage[k].ptr, got, cudaMemcpyHostToDevice, ctx->stream));
            GSIM_CK(cudaEventRecord(done[k], ctx->stream));
        }
        off += got;
        if (got != want) {
            truncated = true;
            break;
        }
        k ^= 1;
    }
    GSIM_CK(cudaStreamSynchronize(ctx->stream));
    if (truncated) throw ValidationError{who + ": payload truncated"};
    gsim_gpu_scene* sc = alloc_scene(ctx, count, degree);
    ctx->counts.reserve(4);
    unsigned long long* err = ctx->counts.ptr + 3;
    GSIM_CK(cudaMemsetAsync(err, 0xFF, sizeof(unsigned long long), ctx->stream));
    PlyArgs a{};
    a.rows = reinterpret_cast<const float*>(raw.ptr);
    a.n = count;
    a.stride = stride;
    a.degree = degree;
    a.field = sc->f;
    a.plane_stride = std::max<uint64_t>(count, 1);
    a.err = err;
    launch_ply_convert(a, ctx->num_sms * 8, ctx->stream);
    unsigned long long e = ~0ull;
    try {
        check_launch();
        GSIM_CK(cudaMemcpyAsync(&e, err, sizeof(e), cudaMemcpyDeviceToHost, ctx->stream));
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        discard_scene(ctx, sc);
        throw;
    }
    if (e != ~0ull) {
        discard_scene(ctx, sc);
        static const char* what[] = {"", "non-finite value", "opacity saturates", "scale overflows",
                                     "zero-norm rotation"};
        throw ValidationError{who + ": " + what[e & 7] + " in primitive " + std::to_string(e >> 3)};
    }
    ctx->launches_total += 1;
    return sc;
}


// Waits for everything queued on the copy stream and the context stream (a synchronous call's
// end): cudaStreamSynchronize, or blocking-sync events when the context asks for them.
void wait_frame(gsim_gpu_context* ctx) {
    if (!ctx->blocking_sync) {
        if (ctx->copy_stream) GSIM_CK(cudaStreamSynchronize(ctx->copy_stream));
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
        return;
    }
    if (ctx->copy_stream) GSIM_CK(cudaEventRecord(ctx->wait_ev[0], ctx->copy_stream));
    GSIM_CK(cudaEventRecord(ctx->wait_ev[1], ctx->stream));
    if (ctx->copy_stream) GSIM_CK(cudaEventSynchronize(ctx->wait_ev[0]));
    GSIM_CK(cudaEventSynchronize(ctx->wait_ev[1]));
}

// Per-camera copies of a host-target render, queued right after the raster launch: the copy
// stream waits on the event after each camera's raster launch, so camera c crosses PCIe while later cameras
// (and other contexts' frames) are still being composited.
void queue_camera_copies(gsim_gpu_context* ctx, const Plan& p, const float* out) {
    uint64_t off = 0;
    for (size_t c = 0; c < p.cams.size(); ++c) {
        const DevCamera& cam = p.cams[c];
        const size_t npx = size_t(cam.width) * cam.height;
        GSIM_CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->cam_evs[c], 0));
        const gsim_target& t = ctx->frame_outs[c];
        const float* base = out + off;
        GSIM_CK(cudaMemcpyAsync(t.rgb, base, 3 * npx * sizeof(float), cudaMemcpyDeviceToHost, ctx->copy_stream));
        GSIM_CK(cudaMemcpyAsync(t.depth, base + 3 * npx, npx * sizeof(float), cudaMemcpyDeviceToHost, ctx->copy_stream));
        GSIM_CK(cudaMemcpyAsync(t.accum_alpha, base + 4 * npx, npx * sizeof(float), cudaMemcpyDeviceToHost, ctx->copy_stream));
        off += 5 * npx;
    }
}

// The same for render_encoded: camera c's encoded block crosses PCIe once its tiles are done.
void queue_camera_copies_enc(gsim_gpu_context* ctx, const Plan& p, const uint8_t* dev, uint32_t bpp) {
    uint64_t off = 0;
    for (size_t c = 0; c < p.cams.size(); ++c) {
        const DevCamera& cam = p.cams[c];
        const uint64_t bytes = uint64_t(bpp) * uint64_t(cam.width) * uint64_t(cam.height);
        GSIM_CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->cam_evs[c], 0));
        if (bytes)
            GSIM_CK(cudaMemcpyAsync(ctx->frame_enc_host + off, dev + off, bytes, cudaMemcpyDeviceToHost,
                                    ctx->copy_stream));
        off += bytes;
    }
}

// D2H of the internal output buffer into host RenderTargets (the drop-in's by-value return).
void copy_targets(gsim_gpu_context* ctx, const gsim_camera* cameras, uint64_t n,
                  const std::vector<uint64_t>& off, gsim_target* outs) {
    ctx->stats.d2h_bytes = 0;
    for (uint64_t c = 0; c < n; ++c) {
        const size_t npx = size_t(cameras[c].width) * cameras[c].height;
        const float* base = ctx->out.ptr + off[c];
        GSIM_CK(cudaMemcpyAsync(outs[c].rgb, base, 3 * npx * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        GSIM_CK(cudaMemcpyAsync(outs[c].depth, base + 3 * npx, npx * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        GSIM_CK(cudaMemcpyAsync(outs[c].accum_alpha, base + 4 * npx, npx * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->stats.d2h_bytes += 5 * npx * sizeof(float);
    }
    GSIM_CK(cudaStreamSynchronize(ctx->stream));
}

struct Guard {
    gsim_gpu_context* ctx;
    explicit Guard(gsim_gpu_context* c) : ctx(c) {}
    template <class F>
    int run(F&& f) {
        if (!ctx) return GSIM_ERR_VALIDATION;
        std::lock_guard<std::mutex> lk(ctx->mu);
        try {
            GSIM_CK(cudaSetDevice(ctx->device));
            check_pending(ctx);
            f();
            ctx->err.clear();
            return GSIM_OK;
        } catch (const ValidationError& e) {
            ctx->err = e.msg;
            return GSIM_ERR_VALIDATION;
        } catch (const CudaError& e) {
            ctx->err = e.msg;
            return GSIM_ERR_IO;
        } catch (const std::exception& e) {
            ctx->err = e.what();
            return GSIM_ERR_IO;
        }
    }
};

// ---- GS -> TSDF helpers (transfer.cpp) ------------------------------------------------------

void scene_bounds(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, double lo[3], double hi[3]) {
    const int max_blocks = ctx->num_sms * 4;
    ctx->bounds_buf.reserve(size_t(6) * (max_blocks + 1));
    double* out = ctx->bounds_buf.ptr + 6 * size_t(max_blocks);
    launch_bounds(scene->f, ctx->bounds_buf.ptr, max_blocks, out, ctx->stream);
    check_launch();
    double box[6];
    GSIM_CK(cudaMemcpyAsync(box, out, sizeof(box), cudaMemcpyDeviceToHost, ctx->stream));
    GSIM_CK(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < 3; ++k) {
        lo[k] = box[k];
        hi[k] = box[3 + k];
    }
}

struct ValidAlphaScope {  // the depth mask applies to the renders of one call only
    gsim_gpu_context* c;
    ValidAlphaScope(gsim_gpu_context* ctx, float a) : c(ctx) { c->frame_valid_alpha = a; }
    ~ValidAlphaScope() { c->frame_valid_alpha = 0.0f; }
};

// render_depth_ring (transfer.cpp:81-124) into ctx->out; returns the per-camera offsets.
std::vector<uint64_t> depth_ring_render(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                                        int n_views, double radius, int resolution,
                                        std::vector<gsim_camera>& cams) {
    if (scene->f.n == 0) throw ValidationError{"render_depth_ring: empty field"};
    if (n_views < 8) throw ValidationError{"render_depth_ring: n_views must be >= 8"};
    if (!(radius > 0.0)) throw ValidationError{"render_depth_ring: radius must be positive"};
    double lo[3], hi[3];
    scene_bounds(ctx, scene, lo, hi);
    cams.assign(size_t(3) * n_views, gsim_camera{});
    if (const char* msg = depth_ring_cameras(lo, hi, n_views, radius, resolution, cams.data()))
        throw ValidationError{msg};
    gsim_raster_options opt{1, 0, 1e-4};  // RasterOptions{normalize_depth = true}
    ValidAlphaScope mask(ctx, 0.5f);      // kDepthValidAlpha, transfer.cpp:23
    return render_cameras(ctx, scene, nullptr, 0, cams.data(), cams.size(), &opt, nullptr, true);
}

void check_volume(const gsim_tsdf_volume* v, bool buffers) {
    if (!v) throw ValidationError{"tsdf: null volume"};
    if (!(v->voxel_size > 0.0)) throw ValidationError{"tsdf: voxel_size must be positive"};
    if (v->dims[0] < 2 || v->dims[1] < 2 || v->dims[2] < 2)
        throw ValidationError{"tsdf: dims must be at least 2 per axis"};
    if (v->truncation < 2.0 * v->voxel_size)
        throw ValidationError{"tsdf: truncation must be >= 2 * voxel_size"};
    if (buffers && (!v->tsdf || !v->weights)) throw ValidationError{"tsdf: null device grids"};
}

TsdfArgs tsdf_args(const gsim_tsdf_volume* v) {
    TsdfArgs a{};
    for (int k = 0; k < 3; ++k) {
        a.origin[k] = v->origin[k];
        a.dims[k] = v->dims[k];
    }
    a.voxel_size = v->voxel_size;
    a.truncation = v->truncation;
    a.tsdf = v->tsdf;
    a.weights = v->weights;
    return a;
}

void fuse_views(gsim_gpu_context* ctx, const gsim_tsdf_volume* vol,
                const std::vector<DevFuseView>& views, const float* depth_dev) {
    if (views.empty()) return;
    ctx->fuse_views.reserve(views.size());
    GSIM_CK(cudaMemcpyAsync(ctx->fuse_views.ptr, views.data(), views.size() * sizeof(DevFuseView),
                            cudaMemcpyHostToDevice, ctx->stream));
    TsdfArgs a = tsdf_args(vol);
    a.n_views = uint32_t(views.size());
    a.views = ctx->fuse_views.ptr;
    a.depth = depth_dev;
    launch_tsdf_fuse(a, ctx->num_sms, ctx->stream);
    check_launch();
    // the view table is staged from host memory that dies with this call
    GSIM_CK(cudaStreamSynchronize(ctx->stream));
}

// ---- LiDAR helpers (trace.cpp) ---------------------------------------------------------------

// GaussianBvh::build's node painting (trace.cpp:93-102: later nodes overwrite, range check) as
// maximal segments; entry_count marks whether the sensor sees the segment (env filter).
std::vector<DevSegment> paint_segments(uint64_t n_prims, const gsim_node* nodes, uint64_t n_nodes,
                                       int32_t env) {
    for (uint64_t k = 0; k < n_nodes; ++k)
        if (nodes[k].end > n_prims)
            throw ValidationError{"node " + std::to_string(k) + " range exceeds field size"};
    std::vector<uint64_t> pts{0, n_prims};
    for (uint64_t k = 0; k < n_nodes; ++k)
        if (nodes[k].begin < nodes[k].end) {
            pts.push_back(nodes[k].begin);
            pts.push_back(nodes[k].end);
        }
    std::sort(pts.begin(), pts.end());
    pts.erase(std::unique(pts.begin(), pts.end()), pts.end());
    std::vector<DevSegment> segs;
    for (size_t k = 0; k + 1 < pts.size(); ++k) {
        if (!(pts[k] < pts[k + 1])) continue;
        int64_t owner = -1;
        for (uint64_t j = 0; j < n_nodes; ++j)
            if (nodes[j].begin <= pts[k] && pts[k] < nodes[j].end) owner = int64_t(j);
        DevSegment sg{};
        sg.begin = pts[k];
        sg.end = pts[k + 1];
        const gsim_rigid id{{1.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
        const gsim_rigid& pose = owner >= 0 ? nodes[owner].pose : id;
        for (int c = 0; c < 4; ++c) sg.q[c] = pose.rotation[c];
        for (int c = 0; c < 3; ++c) sg.t[c] = pose.translation[c];
        sg.entry_count = (owner >= 0 && nodes[owner].env >= 0 && nodes[owner].env != env) ? 0u : 1u;
        segs.push_back(sg);
    }
    if (segs.empty()) {
        DevSegment sg{};
        sg.q[0] = 1.0;
        segs.push_back(sg);
    }
    return segs;
}

void validate_lidar(const gsim_lidar& l) {  // trace.cpp:136-155
    constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
    if (l.n_channels == 0 || !l.channels) throw ValidationError{"lidar: no channels"};
    for (uint64_t c = 0; c < l.n_channels; ++c)
        if (!std::isfinite(l.channels[c])) throw ValidationError{"lidar: non-finite elevation"};
    if (!(l.azimuth_step > 0.0)) throw ValidationError{"lidar: azimuth_step must be positive"};
    const double n = kTwoPi / l.azimuth_step;
    if (std::abs(n - std::round(n)) * l.azimuth_step > 1e-9)
        throw ValidationError{"lidar: azimuth_step must divide 2*pi into an integer ray count"};
    if (!(l.max_range > 0.0)) throw ValidationError{"lidar: max_range must be positive"};
    if (!(l.alpha_threshold > 0.0) || l.alpha_threshold > 1.0)
        throw ValidationError{"lidar: alpha_threshold outside (0,1]"};
}

LidarArgs lidar_pose_stage(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                           uint64_t n_nodes, int32_t env, bool scan) {
    auto& L = ctx->lidar;
    const uint64_t n = scene->f.n;
    const std::vector<DevSegment> segs = paint_segments(n, nodes, n_nodes, env);
    L.segs.reserve(segs.size());
    GSIM_CK(cudaMemcpyAsync(L.segs.ptr, segs.data(), segs.size() * sizeof(DevSegment),
                            cudaMemcpyHostToDevice, ctx->stream));
    L.posed.reserve(std::max<uint64_t>(19 * n, 1));
    L.trace_rec.reserve(std::max<uint64_t>(20 * n, 2));
    L.seen.reserve(std::max<uint64_t>(n, 1));
    L.rects.reserve(std::max<uint64_t>(n, 1));
    L.all_list.reserve(std::max<uint64_t>(n, 1) + 1);
    LidarArgs a{};
    a.field = scene->f;
    a.segs = L.segs.ptr;
    a.n_segs = int(segs.size());
    a.scan = scan ? 1 : 0;
    a.n = n;
    a.posed = L.posed.ptr;
    a.trace_rec = L.trace_rec.ptr;
    a.seen = L.seen.ptr;
    a.rects = L.rects.ptr;
    a.all_count = L.all_list.ptr;      // [0] = count
    a.all_list = L.all_list.ptr + 1;
    a.two_pi = 2.0 * 3.14159265358979323846;
    GSIM_CK(cudaMemsetAsync(a.all_count, 0, sizeof(uint32_t), ctx->stream));
    return a;
}

// Linear BVH over the posed boxes of `a` (bvh.cu) and the candidate list of every arbitrary
// ray (la.ray_origin / ray_dir / ray_tmax set): la.list / ray_offset / cand_t / cand_r filled,
// la.ray_lists = 1. Returns the total number of candidates.
uint64_t bvh_ray_lists(gsim_gpu_context* ctx, LidarArgs& la) {
    auto& L = ctx->lidar;
    cudaStream_t s = ctx->stream;
    const uint64_t n = la.n;
    const int n_sms = ctx->num_sms;
    if (n >= (uint64_t(1) << 31)) throw ValidationError{"trace_rays: field too large for the BVH"};
    const uint64_t nn = std::max<uint64_t>(n, 1);
    for (int k = 0; k < 2; ++k) {
        L.bvh_keys[k].reserve(nn);
        L.bvh_vals[k].reserve(nn);
    }
    // small tables: [0..1023] hist (4 x 256), tickets [1024..1031], vbase [1040..1041],
    // chunk_base0 [1044..1045], chunk_base1 [1048..1049], n_leaves [1052], cam_visible [1056],
    // collect overflow [1060]
    L.bvh_small.reserve(1088);
    uint32_t* sm = L.bvh_small.ptr;
    L.bvh_nodes.reserve(5 * nn);  // child 2(n-1), node_parent n-1, leaf_parent n, visits n-1
    L.bvh_box.reserve(6 * nn);
    L.bvh_leaf_box.reserve(6 * nn);
    L.bvh_wide.reserve(4 * nn);
    L.bvh_seg.reserve(2);
    L.bvh_bounds.reserve(6);
    const uint32_t chunks0 = uint32_t((n + kOnesweepTile - 1) / kOnesweepTile);
    const uint64_t seg_host[2] = {0, n};
    const uint32_t cb0_host[2] = {0, chunks0};
    GSIM_CK(cudaMemsetAsync(sm, 0, 1088 * sizeof(uint32_t), s));
    GSIM_CK(cudaMemcpyAsync(L.bvh_seg.ptr, seg_host, sizeof(seg_host), cudaMemcpyHostToDevice, s));
    GSIM_CK(cudaMemcpyAsync(sm + 1044, cb0_host, sizeof(cb0_host), cudaMemcpyHostToDevice, s));
    const unsigned long long init_bits[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
    GSIM_CK(cudaMemcpyAsync(L.bvh_bounds.ptr, init_bits, sizeof(init_bits), cudaMemcpyHostToDevice, s));
    const uint64_t words = (uint64_t(chunks0) + 1) * 256;
    if (words > ctx->status.cap) {
        ctx->status.reserve(words);
        GSIM_CK(cudaMemsetAsync(ctx->status.ptr, 0, ctx->status.cap * sizeof(uint64_t), s));
    }
    BvhArgs b{};
    b.n = n;
    b.posed = la.posed;
    b.seen = la.seen;
    b.bounds_bits = L.bvh_bounds.ptr;
    b.codes_in = L.bvh_keys[0].ptr;  // sorted into bvh_keys[1] / bvh_vals[1] after 4 passes
    b.hist = sm;
    b.vbase = sm + 1040;
    b.chunk_base1 = sm + 1048;
    b.n_leaves = sm + 1052;
    b.child = L.bvh_nodes.ptr;
    b.node_parent = L.bvh_nodes.ptr + 2 * nn;
    b.leaf_parent = L.bvh_nodes.ptr + 3 * nn;
    b.visits = L.bvh_nodes.ptr + 4 * nn;
    b.node_box = L.bvh_box.ptr;
    b.leaf_box = L.bvh_leaf_box.ptr;
    b.wide = L.bvh_wide.ptr;
    launch_bvh_bounds(b, n_sms, s);
    launch_bvh_morton(b, n_sms, s);
    check_launch();
    // (code, primitive) sort: the render path's segmented onesweep with one segment
    BinArgs hb{};
    hb.keys = b.codes_in;
    hb.n_slots = n;
    hb.cam_slot_base = L.bvh_seg.ptr;
    hb.sort_bits = 8;
    hb.sort_passes = 4;
    hb.n_cams = 1;
    hb.hist = sm;
    hb.cam_visible = sm + 1056;
    launch_key_hist(hb, n_sms * 2, s);
    launch_bvh_sort_setup(b, s);
    check_launch();
    OnesweepArgs oa{};
    oa.backoff_ns = 64;
    oa.status = ctx->status.ptr;
    oa.n_cams = 1;
    oa.vbase = b.vbase;
    oa.hist_stride = 4 * 256;
    oa.seg_base64 = L.bvh_seg.ptr;
    oa.seg_base32 = b.vbase;
    const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(chunks0 + 1, uint64_t(n_sms) * kOnesweepMinBlocks)));
    const uint32_t* kin = b.codes_in;
    const uint32_t* vin = nullptr;
    const int out_of[4] = {1, 0, 1, 0};  // codes_in is bvh_keys[0]: pass 1 writes buffer 1
    for (int pass = 0; pass < 4; ++pass) {
        const int o = out_of[pass];
        oa.keys_in = kin;
        oa.vals_in = vin;
        oa.keys_out = L.bvh_keys[o].ptr;
        oa.vals_out = L.bvh_vals[o].ptr;
        oa.chunk_base = pass == 0 ? sm + 1044 : b.chunk_base1;
        oa.hist = sm + 256 * pass;
        oa.ticket = sm + 1024 + pass;
        oa.epoch = ctx->next_epoch();
        oa.shift = 8 * pass;
        launch_onesweep(oa, 8, pass == 0, true, grid, s);
        check_launch();
        kin = L.bvh_keys[o].ptr;
        vin = L.bvh_vals[o].ptr;
    }
    b.codes_sorted = kin;
    b.leaf_prim = vin;
    launch_bvh_build(b, n_sms, s);
    launch_bvh_refit(b, n_sms, s);
    check_launch();
    // candidate lists: one pass into per-ray slots of the capacity learned from earlier calls
    // (counting every candidate); a ray that overflows makes the lists exact: scan of the
    // counts, then a fill pass at the offsets (and a larger capacity for the next call)
    const uint64_t R = la.n_rays;
    L.counts.reserve(std::max<uint64_t>(R, 1));
    L.offsets.reserve(R + 1);
    L.scratch.reserve((R + 1023) / 1024 + 2);
    la.ray_count = L.counts.ptr;
    uint32_t cap = L.bvh_capacity;
    constexpr uint64_t kSlotBudget = uint64_t(1) << 28;  // 5 GB of list + (t, response) slots
    if (uint64_t(cap) * R > kSlotBudget) cap = uint32_t(std::max<uint64_t>(kSlotBudget / std::max<uint64_t>(R, 1), 16));
    L.list.reserve(std::max<uint64_t>(uint64_t(cap) * R, 1));
    L.cand_t.reserve(std::max<uint64_t>(uint64_t(cap) * R, 1));
    L.cand_r.reserve(std::max<uint64_t>(uint64_t(cap) * R, 1));
    b.overflow = sm + 1060;
    GSIM_CK(cudaMemsetAsync(b.overflow, 0, sizeof(uint32_t), s));
    la.list = L.list.ptr;
    la.cand_t = L.cand_t.ptr;
    la.cand_r = L.cand_r.ptr;
    la.list_stride = cap;
    la.list_count = L.counts.ptr;
    launch_bvh_collect(b, la, 2, n_sms, s);
    check_launch();
    exclusive_scan_u32(L.counts.ptr, R, L.offsets.ptr, L.scratch.ptr, s);
    check_launch();
    unsigned long long total = 0;
    uint32_t overflow = 0;
    GSIM_CK(cudaMemcpyAsync(&total, L.offsets.ptr + R, sizeof(total), cudaMemcpyDeviceToHost, s));
    GSIM_CK(cudaMemcpyAsync(&overflow, b.overflow, sizeof(overflow), cudaMemcpyDeviceToHost, s));
    GSIM_CK(cudaStreamSynchronize(s));
    if (total >= (1ull << 32)) throw CudaError{"trace_rays: more than 2^32 ray candidates"};
    if (overflow) {
        uint32_t grow = 16;
        while (grow < overflow && grow < (1u << 30)) grow <<= 1;
        L.bvh_capacity = std::max(L.bvh_capacity, grow);
        L.list.reserve(std::max<unsigned long long>(total, 1));
        L.cand_t.reserve(std::max<unsigned long long>(total, 1));
        L.cand_r.reserve(std::max<unsigned long long>(total, 1));
        la.list = L.list.ptr;
        la.cand_t = L.cand_t.ptr;
        la.cand_r = L.cand_r.ptr;
        la.list_stride = 0;
        la.list_count = nullptr;
        la.ray_offset = L.offsets.ptr;
        launch_bvh_collect(b, la, 1, n_sms, s);
        check_launch();
    }
    la.ray_lists = 1;
    ctx->launches_total += 14;
    return total;
}

}  // namespace

extern "C" {

const char* gsim_gpu_version(void) { return "gsim_gpu 0.2 (sm_100a)"; }

int gsim_gpu_context_create(int device, gsim_gpu_context** out) {
    if (!out) return GSIM_ERR_VALIDATION;
    *out = nullptr;
    auto* ctx = new gsim_gpu_context();
    try {
        int n = 0;
        GSIM_CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw ValidationError{"no CUDA device " + std::to_string(device)};
        ctx->device = device;
        GSIM_CK(cudaSetDevice(device));
        cudaDeviceProp prop{};
        GSIM_CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            throw CudaError{std::string("gsim_gpu is built for sm_100a; device is ") + prop.name};
        ctx->num_sms = prop.multiProcessorCount;
        GSIM_CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        for (auto& e : ctx->ev) GSIM_CK(cudaEventCreate(&e));
        for (auto& e : ctx->staging_ev) GSIM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        GSIM_CK(cudaEventCreateWithFlags(&ctx->bin_ev, cudaEventDisableTiming));
        ctx->zero_block.reserve(kZeroCams + 64);
        ctx->counts.reserve(4);
        ctx->readback.reserve(64);
        if (const char* e = std::getenv("GSIM_GPU_RASTER_RECT")) ctx->raster_rect_w = std::atoi(e) == 16 ? 16 : 8;
        if (const char* e = std::getenv("GSIM_GPU_RASTER_EXACT")) ctx->raster_exact_cull = std::atoi(e) != 0;
        if (const char* e = std::getenv("GSIM_GPU_RASTER_BATCH")) ctx->raster_batch = std::atoi(e) == 256 ? 256 : 128;
        if (const char* e = std::getenv("GSIM_GPU_RASTER_BULK")) ctx->raster_bulk = std::atoi(e) == 1 ? 1 : 0;
        if (const char* e = std::getenv("GSIM_GPU_RASTER_CTAS")) ctx->raster_ctas = std::max(0, std::atoi(e));
        if (const char* e = std::getenv("GSIM_GPU_OVERLAP_COPIES")) ctx->overlap_copies = std::atoi(e) != 0;
        if (const char* e = std::getenv("GSIM_GPU_BLOCKING_SYNC")) ctx->blocking_sync = std::atoi(e) == 1;
        if (const char* e = std::getenv("GSIM_GPU_BVH_CAPACITY"))  // tests: start small (overflow path)
            ctx->lidar.bvh_capacity = uint32_t(std::max(1, std::atoi(e)));
        for (int k = 0; k < 2; ++k)
            GSIM_CK(cudaEventCreateWithFlags(&ctx->wait_ev[k], cudaEventDisableTiming |
                                             (ctx->blocking_sync ? cudaEventBlockingSync : 0)));
        if (const char* e = std::getenv("GSIM_GPU_GROUP_SLOTS")) {
            const uint64_t v = std::strtoull(e, nullptr, 10);
            if (v > 0 && v < ctx->group_slots) ctx->group_slots = v;
        }
        if (const char* e = std::getenv("GSIM_GPU_INITIAL_PAIR_CAPACITY")) {
            ctx->fixed_initial_capacity = std::strtoull(e, nullptr, 10);
            ctx->pair_capacity = ctx->fixed_initial_capacity;
        }
    } catch (const ValidationError& e) {
        g_create_error = e.msg;
        delete ctx;
        return GSIM_ERR_VALIDATION;
    } catch (const CudaError& e) {
        g_create_error = e.msg;
        delete ctx;
        return GSIM_ERR_IO;
    }
    *out = ctx;
    return GSIM_OK;
}

int gsim_gpu_context_destroy(gsim_gpu_context* ctx) {
    if (!ctx) return GSIM_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    ctx->records.release();
    ctx->keys.release();
    ctx->rects.release();
    ctx->sort_rects.release();
    for (int k = 0; k < 2; ++k) {
        ctx->dk[k].release();
        ctx->dv[k].release();
        ctx->staging[k].release();
    }
    ctx->status.release();
    ctx->vals.release();
    ctx->zero_block.release();
    ctx->counts.release();
    ctx->cam_vbase.release();
    ctx->cam_chunk_base.release();
    ctx->cam_pairs.release();
    ctx->chunk_cam.release();
    ctx->n_chunks.release();
    ctx->cam_mbase.release();
    ctx->cam_pair_base.release();
    ctx->count_matrix.release();
    ctx->tile_count.release();
    ctx->tile_rel.release();
    ctx->plan_dev.release();
    ctx->out.release();
    ctx->full.release();
    ctx->full_vis.release();
    ctx->splats_in.release();
    ctx->bounds_buf.release();
    ctx->lidar.release();
    ctx->fuse_views.release();
    ctx->depth_in.release();
    ctx->readback.release();
    ctx->srgb_thr.release();
    ctx->enc_buf.release();
    ctx->enc_src.release();
    ctx->enc_cams.release();
    ctx->query_buf.release();
    {
        std::lock_guard<std::mutex> lk(ctx->mu);
        for (auto* sc : ctx->scenes) sc->ctx = nullptr;
        for (auto* tr : ctx->tracks) tr->ctx = nullptr;
    }
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->staging_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->bin_ev) cudaEventDestroy(ctx->bin_ev);
    for (int k = 0; k < 2; ++k)
        if (ctx->wait_ev[k]) cudaEventDestroy(ctx->wait_ev[k]);
    for (cudaEvent_t e : ctx->cam_evs) cudaEventDestroy(e);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
    }
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return GSIM_OK;
}

const char* gsim_gpu_last_error(const gsim_gpu_context* ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

void* gsim_gpu_stream(gsim_gpu_context* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int gsim_gpu_synchronize(gsim_gpu_context* ctx) {
    return Guard(ctx).run([&] { GSIM_CK(cudaStreamSynchronize(ctx->stream)); });
}

int gsim_gpu_set_profiling(gsim_gpu_context* ctx, int enable) {
    return Guard(ctx).run([&] { ctx->profiling = enable != 0; });
}

int gsim_gpu_get_stats(gsim_gpu_context* ctx, gsim_render_stats* out) {
    return Guard(ctx).run([&] {
        if (!out) throw ValidationError{"stats: null output"};
        gsim_render_stats st = ctx->stats;
        unsigned long long c[4] = {0, 0, 0, 0};
        uint32_t chunks = 0;
        GSIM_CK(cudaMemcpyAsync(c, ctx->counts.ptr, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
        if (ctx->n_chunks.ptr)
            GSIM_CK(cudaMemcpyAsync(&chunks, ctx->n_chunks.ptr, sizeof(chunks), cudaMemcpyDeviceToHost, ctx->stream));
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
        st.consumed = c[2];
        st.chunks = chunks;
        if (ctx->profiling) {
            auto ms = [&](int a, int b) {
                float v = 0.f;
                GSIM_CK(cudaEventElapsedTime(&v, ctx->ev[a], ctx->ev[b]));
                return v;
            };
            st.ms_preprocess = ms(kEvStart, kEvPre);
            st.ms_depth_sort = ms(kEvPre, kEvDepth);
            st.ms_binning = ms(kEvDepth, kEvBin);
            st.ms_scatter = ms(kEvBin, kEvScatter);
            st.ms_raster = ms(kEvScatter, kEvRaster);
            st.ms_total = ms(kEvStart, kEvRaster);
        }
        *out = st;
    });
}

namespace {
void check_view(const gsim_field_view* v, const char* who) {
    if (!v) throw ValidationError{std::string(who) + ": null argument"};
    if (v->sh_degree < 0 || v->sh_degree > 3)  // gaussian.cpp:15-17
        throw ValidationError{"sh_degree " + std::to_string(v->sh_degree) + " outside [0,3]"};
    if (v->count >= 0xFFFFFFFFull) throw ValidationError{"field larger than 2^32 - 1 primitives"};
    if (v->count && (!v->means || !v->scales || !v->rotations || !v->opacities || !v->sh))
        throw ValidationError{std::string(who) + ": null field array"};
}

// Primitives [offset, offset + v->count) of the scene from a host view: converted to the
// device layout (double geometry planes, fp32 SH float4 planes) in host chunks, each plane's
// slice copied into place.
void write_scene(gsim_gpu_context* ctx, gsim_gpu_scene* sc, uint64_t offset, const gsim_field_view* v) {
    const uint64_t nn = std::max<uint64_t>(sc->f.n, 1);
    const int K = (sc->f.sh_degree + 1) * (sc->f.sh_degree + 1);
    const int planes = sc->f.sh_planes;
    constexpr uint64_t kChunk = 1u << 20;
    std::vector<double> geo;
    std::vector<float4> sh;
    for (uint64_t b = 0; b < v->count; b += kChunk) {
        const uint64_t m = std::min<uint64_t>(kChunk, v->count - b);
        geo.assign(11 * m, 0.0);
        sh.assign(size_t(planes) * m, make_float4(0, 0, 0, 0));
        for (uint64_t j = 0; j < m; ++j) {
            const uint64_t i = b + j;
            const double* mu = v->means + i * v->means_stride;
            const double* sc3 = v->scales + i * v->scales_stride;
            const double* q = v->rotations + i * v->rotations_stride;
            for (int c = 0; c < 3; ++c) geo[c * m + j] = mu[c];
            for (int c = 0; c < 3; ++c) geo[(3 + c) * m + j] = sc3[c];
            for (int c = 0; c < 4; ++c) geo[(6 + c) * m + j] = q[c];
            geo[10 * m + j] = v->opacities[i * v->opacities_stride];
            const double* c = v->sh + i * v->sh_stride;
            float tmp[48 + 4] = {0};
            for (int ch = 0; ch < 3; ++ch)
                for (int k = 0; k < K; ++k) tmp[ch * K + k] = float(c[ch * 16 + k]);
            for (int p = 0; p < planes; ++p)
                sh[size_t(p) * m + j] = make_float4(tmp[4 * p], tmp[4 * p + 1], tmp[4 * p + 2], tmp[4 * p + 3]);
        }
        for (int pl = 0; pl < 11; ++pl)
            GSIM_CK(cudaMemcpy(sc->f.mx + pl * nn + offset + b, geo.data() + pl * m, m * sizeof(double),
                               cudaMemcpyHostToDevice));
        for (int p = 0; p < planes; ++p)
            GSIM_CK(cudaMemcpy(sc->f.sh + size_t(p) * nn + offset + b, sh.data() + size_t(p) * m,
                               m * sizeof(float4), cudaMemcpyHostToDevice));
    }
    (void)ctx;
}
}  // namespace

int gsim_gpu_scene_upload(gsim_gpu_context* ctx, const gsim_field_view* v, gsim_gpu_scene** out) {
    return Guard(ctx).run([&] {
        check_view(v, "scene_upload");
        if (!out) throw ValidationError{"scene_upload: null argument"};
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
        gsim_gpu_scene* sc = alloc_scene(ctx, v->count, v->sh_degree);
        try {
            write_scene(ctx, sc, 0, v);
        } catch (...) {
            discard_scene(ctx, sc);
            throw;
        }
        *out = sc;
    });
}

int gsim_gpu_scene_create(gsim_gpu_context* ctx, uint64_t count, int32_t sh_degree, gsim_gpu_scene** out) {
    return Guard(ctx).run([&] {
        if (!out) throw ValidationError{"scene_create: null argument"};
        if (sh_degree < 0 || sh_degree > 3)
            throw ValidationError{"sh_degree " + std::to_string(sh_degree) + " outside [0,3]"};
        if (count >= 0xFFFFFFFFull) throw ValidationError{"field larger than 2^32 - 1 primitives"};
        gsim_gpu_scene* sc = alloc_scene(ctx, count, sh_degree);
        const uint64_t nn = std::max<uint64_t>(count, 1);
        const size_t geo_bytes = (11 * nn * sizeof(double) + 255) & ~size_t(255);
        if (cudaMemset(sc->mem, 0, geo_bytes + size_t(sc->f.sh_planes) * nn * sizeof(float4)) != cudaSuccess) {
            discard_scene(ctx, sc);
            throw CudaError{"scene_create: memset failed"};
        }
        *out = sc;
    });
}

int gsim_gpu_scene_write(gsim_gpu_context* ctx, gsim_gpu_scene* scene, uint64_t offset,
                         const gsim_field_view* v) {
    return Guard(ctx).run([&] {
        check_view(v, "scene_write");
        if (!scene) throw ValidationError{"scene_write: null scene"};
        if (v->sh_degree != scene->f.sh_degree)
            throw ValidationError{"scene_write: sh_degree " + std::to_string(v->sh_degree) +
                                  " differs from the scene's " + std::to_string(scene->f.sh_degree)};
        if (offset > scene->f.n || v->count > scene->f.n - offset)
            throw ValidationError{"scene_write: range exceeds field size"};
        GSIM_CK(cudaStreamSynchronize(ctx->stream));  // frames in flight may read the field
        write_scene(ctx, scene, offset, v);
    });
}

int32_t gsim_gpu_scene_sh_degree(const gsim_gpu_scene* scene) { return scene ? scene->f.sh_degree : -1; }

int gsim_gpu_scene_download_field(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                                  double* means, double* scales, double* rotations,
                                  double* opacities, double* sh) {
    return Guard(ctx).run([&] {
        if (!scene) throw ValidationError{"scene_download_field: null scene"};
        const uint64_t n = scene->f.n, nn = std::max<uint64_t>(n, 1);
        const int K = (scene->f.sh_degree + 1) * (scene->f.sh_degree + 1);
        std::vector<double> geo(11 * nn);
        std::vector<float4> shp(size_t(scene->f.sh_planes) * nn);
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
        GSIM_CK(cudaMemcpy(geo.data(), scene->f.mx, geo.size() * sizeof(double), cudaMemcpyDeviceToHost));
        GSIM_CK(cudaMemcpy(shp.data(), scene->f.sh, shp.size() * sizeof(float4), cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < n; ++i) {
            for (int c = 0; c < 3; ++c) {
                if (means) means[3 * i + c] = geo[c * nn + i];
                if (scales) scales[3 * i + c] = geo[(3 + c) * nn + i];
            }
            for (int c = 0; c < 4; ++c)
                if (rotations) rotations[4 * i + c] = geo[(6 + c) * nn + i];
            if (opacities) opacities[i] = geo[10 * nn + i];
            if (sh) {
                double* o = sh + 48 * i;
                for (int k = 0; k < 48; ++k) o[k] = 0.0;
                for (int j = 0; j < 3 * K; ++j) {
                    const float4 v = shp[size_t(j / 4) * nn + i];
                    const float comp[4] = {v.x, v.y, v.z, v.w};
                    o[(j / K) * 16 + (j % K)] = comp[j % 4];
                }
            }
        }
    });
}

int gsim_gpu_scene_load_ply(gsim_gpu_context* ctx, const char* path, gsim_gpu_scene** out) {
    if (out) *out = nullptr;
    return Guard(ctx).run([&] {
        if (!path || !out) throw ValidationError{"scene_load_ply: null argument"};
        *out = load_ply(ctx, path);
    });
}

int gsim_gpu_scene_destroy(gsim_gpu_scene* scene) {
    if (!scene) return GSIM_OK;
    if (scene->ctx) {
        std::lock_guard<std::mutex> lk(scene->ctx->mu);
        cudaSetDevice(scene->ctx->device);
        cudaStreamSynchronize(scene->ctx->stream);
        scene->ctx->scenes.erase(scene);
    }
    if (scene->mem) cudaFree(scene->mem);
    delete scene;
    return GSIM_OK;
}

uint64_t gsim_gpu_scene_size(const gsim_gpu_scene* scene) { return scene ? scene->f.n : 0; }

int gsim_gpu_transform_primitives(gsim_gpu_context* ctx, gsim_gpu_scene* scene, uint64_t begin,
                                  uint64_t end, const gsim_rigid* t) {
    return Guard(ctx).run([&] {
        if (!scene || !t) throw ValidationError{"transform_primitives: null argument"};
        if (begin > end || end > scene->f.n)  // gaussian.cpp:67-71
            throw ValidationError{"transform_primitives: range [" + std::to_string(begin) + "," +
                                  std::to_string(end) + ") outside field of size " +
                                  std::to_string(scene->f.n)};
        launch_pose(scene->f, begin, end, *t, ctx->num_sms * 8, ctx->stream);
        check_launch();
        ctx->launches_total += (end > begin) ? 1 : 0;
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsim_gpu_scene_download(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, double* means,
                            double* rotations) {
    return Guard(ctx).run([&] {
        if (!scene) throw ValidationError{"scene_download: null scene"};
        const uint64_t n = scene->f.n;
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
        std::vector<double> plane(std::max<uint64_t>(n, 1));
        auto fetch = [&](const double* src, double* dst, int comp, int ncomp) {
            GSIM_CK(cudaMemcpy(plane.data(), src, n * sizeof(double), cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < n; ++i) dst[i * ncomp + comp] = plane[i];
        };
        if (means) {
            fetch(scene->f.mx, means, 0, 3);
            fetch(scene->f.my, means, 1, 3);
            fetch(scene->f.mz, means, 2, 3);
        }
        if (rotations) {
            fetch(scene->f.qw, rotations, 0, 4);
            fetch(scene->f.qx, rotations, 1, 4);
            fetch(scene->f.qy, rotations, 2, 4);
            fetch(scene->f.qz, rotations, 3, 4);
        }
    });
}

int gsim_gpu_project(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                     uint64_t n_nodes, const gsim_camera* camera, gsim_projected_splat* out,
                     uint64_t capacity, uint64_t* count) {
    return Guard(ctx).run([&] {
        if (!scene || !camera || !count) throw ValidationError{"project: null argument"};
        Plan plan = build_plan(scene->f.n, nodes, n_nodes, camera, 1);
        reserve_workspace(ctx, plan);
        upload_plan(ctx, plan);
        const uint64_t S = std::max<uint64_t>(plan.slots, 1);
        ctx->full.reserve(S);
        ctx->full_vis.reserve(S);
        begin_frame(ctx, plan);
        PreprocessArgs pa = make_pre_args(ctx, scene, plan);
        pa.full = ctx->full.ptr;
        pa.full_visible = ctx->full_vis.ptr;
        if (plan.slots) {
            launch_preprocess(pa, true, ctx->num_sms, ctx->stream);
            check_launch();
            ctx->launches_total += 1;
        }
        std::vector<uint8_t> vis(plan.slots);
        std::vector<gsim_projected_splat> all(plan.slots);
        if (plan.slots) {
            GSIM_CK(cudaMemcpyAsync(vis.data(), ctx->full_vis.ptr, plan.slots, cudaMemcpyDeviceToHost, ctx->stream));
            GSIM_CK(cudaMemcpyAsync(all.data(), ctx->full.ptr, plan.slots * sizeof(gsim_projected_splat),
                                    cudaMemcpyDeviceToHost, ctx->stream));
        }
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
        uint64_t k = 0;
        for (uint64_t s = 0; s < plan.slots; ++s) {
            if (!vis[s]) continue;
            if (out && k < capacity) out[k] = all[s];
            ++k;
        }
        *count = k;
    });
}

int gsim_gpu_rasterize(gsim_gpu_context* ctx, const gsim_projected_splat* splats, uint64_t n,
                       const gsim_camera* camera, const gsim_raster_options* options,
                       gsim_target* out) {
    return Guard(ctx).run([&] {
        if (!camera || !out || (n && !splats)) throw ValidationError{"rasterize: null argument"};
        if (n >= 0xFFFFFFFFull) throw ValidationError{"rasterize: too many splats"};
        Plan plan = build_splat_plan(n, *camera);
        gsim_raster_options opt{0, 0, 1e-4};
        if (options) opt = *options;
        reserve_workspace(ctx, plan);
        upload_plan(ctx, plan);
        ctx->splats_in.reserve(std::max<uint64_t>(n, 1));
        ctx->out.reserve(plan.out_floats);
        if (n)
            GSIM_CK(cudaMemcpyAsync(ctx->splats_in.ptr, splats, n * sizeof(gsim_projected_splat),
                                    cudaMemcpyHostToDevice, ctx->stream));
        ctx->stats.h2d_bytes += n * sizeof(gsim_projected_splat);
        record_ev(ctx, kEvStart);
        begin_frame(ctx, plan);
        uint64_t launches = 0;
        SplatArgs sa{};
        sa.splats = ctx->splats_in.ptr;
        sa.n = n;
        sa.cam = ctx->cams;
        sa.records = ctx->records.ptr;
        sa.rects = ctx->rects.ptr;
        sa.keys = ctx->keys.ptr;
        if (n) {
            launch_splats_to_records(sa, ctx->num_sms * 8, ctx->stream);
            check_launch();
            ++launches;
        }
        record_ev(ctx, kEvPre);
        run_sort_and_raster(ctx, plan, opt, ctx->out.ptr, launches, true);
        finish_stats(ctx, plan, launches);
        const DevCamera& c = plan.cams[0];
        const size_t npx = size_t(c.width) * c.height;
        GSIM_CK(cudaMemcpyAsync(out->rgb, ctx->out.ptr, 3 * npx * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        GSIM_CK(cudaMemcpyAsync(out->depth, ctx->out.ptr + 3 * npx, npx * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        GSIM_CK(cudaMemcpyAsync(out->accum_alpha, ctx->out.ptr + 4 * npx, npx * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->stats.d2h_bytes += 5 * npx * sizeof(float);
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
        ctx->last_plan = std::move(plan);
    });
}

int gsim_gpu_render_device(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                           const gsim_node* nodes, uint64_t n_nodes, const gsim_camera* cameras,
                           uint64_t n_cameras, const gsim_raster_options* options,
                           float* device_out) {
    return Guard(ctx).run([&] {
        if (!scene || (n_cameras && !cameras) || (n_nodes && !nodes))
            throw ValidationError{"render: null argument"};
        render_cameras(ctx, scene, nodes, n_nodes, cameras, n_cameras, options, device_out, false);
    });
}

float* gsim_gpu_device_output(gsim_gpu_context* ctx) { return ctx ? ctx->out.ptr : nullptr; }

// ---- peer memory (config 4 fused gather) ------------------------------------------------------
int gsim_gpu_ipc_alloc(int32_t device, uint64_t bytes, void** ptr, uint8_t handle[64]) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle size");
    if (!ptr || !handle || bytes == 0) return GSIM_ERR_VALIDATION;
    *ptr = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return GSIM_ERR_IO;
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return GSIM_ERR_IO;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
        cudaFree(p);
        return GSIM_ERR_IO;
    }
    std::memcpy(handle, &h, 64);
    *ptr = p;
    return GSIM_OK;
}

int gsim_gpu_ipc_free(int32_t device, void* ptr) {
    if (!ptr) return GSIM_OK;
    if (cudaSetDevice(device) != cudaSuccess) return GSIM_ERR_IO;
    return cudaFree(ptr) == cudaSuccess ? GSIM_OK : GSIM_ERR_IO;
}

int gsim_gpu_ipc_open(int32_t device, const uint8_t handle[64], void** ptr) {
    if (!ptr || !handle) return GSIM_ERR_VALIDATION;
    *ptr = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return GSIM_ERR_IO;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    return cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? GSIM_OK
                                                                                       : GSIM_ERR_IO;
}

int gsim_gpu_ipc_close(int32_t device, void* ptr) {
    if (!ptr) return GSIM_OK;
    if (cudaSetDevice(device) != cudaSuccess) return GSIM_ERR_IO;
    return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? GSIM_OK : GSIM_ERR_IO;
}

int gsim_gpu_render(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                    uint64_t n_nodes, const gsim_camera* cameras, uint64_t n_cameras,
                    const gsim_raster_options* options, gsim_target* outs) {
    return Guard(ctx).run([&] {
        if (!scene || (n_cameras && (!cameras || !outs)) || (n_nodes && !nodes))
            throw ValidationError{"render: null argument"};
        // Asynchronous render with the copies queued behind it: the pair-buffer check is done
        // once at the end (no mid-frame host round trip); on an overflow the tail is re-run
        // and the targets copied again.
        // Per-camera copies overlap the compositing (queue_camera_copies) unless
        // GSIM_GPU_OVERLAP_COPIES=0; then they follow the frame.
        const bool overlap = ctx->overlap_copies;
        if (overlap && !ctx->copy_stream)
            GSIM_CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        ctx->copies_stale = false;
        ctx->frame_outs = overlap ? outs : nullptr;
        std::vector<uint64_t> off;
        try {
            off = render_cameras(ctx, scene, nodes, n_nodes, cameras, n_cameras, options, nullptr, false);
        } catch (...) {
            ctx->frame_outs = nullptr;
            if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
            throw;
        }
        ctx->frame_outs = nullptr;
        if (overlap) {
            wait_frame(ctx);
            ctx->stats.d2h_bytes = 0;
            for (uint64_t c = 0; c < n_cameras; ++c)
                ctx->stats.d2h_bytes += 5 * uint64_t(cameras[c].width) * cameras[c].height * sizeof(float);
            if (check_pending(ctx) || ctx->copies_stale) copy_targets(ctx, cameras, n_cameras, off, outs);
        } else {
            copy_targets(ctx, cameras, n_cameras, off, outs);
            if (check_pending(ctx)) copy_targets(ctx, cameras, n_cameras, off, outs);
        }
    });
}

uint64_t gsim_gpu_encoded_bytes(uint32_t flags, int32_t width, int32_t height) {
    if (flags & ~uint32_t(GSIM_ENCODE_RGB8 | GSIM_ENCODE_ALPHA8 | GSIM_ENCODE_DEPTH16 |
                          GSIM_ENCODE_DEPTH_PFM))
        return 0;
    if (width <= 0 || height <= 0) return 0;
    return uint64_t(encoded_bpp(flags)) * uint64_t(width) * uint64_t(height);
}

namespace {
uint64_t fnv1a(const void* data, size_t size, uint64_t h) {  // hash.hpp:17-25
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < size; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}
uint64_t hash_image(int32_t w, int32_t h, const float* v, size_t channels, uint64_t seed) {
    const int32_t dims[2] = {w, h};  // hash.hpp:29-34
    seed = fnv1a(dims, sizeof(dims), seed);
    return fnv1a(v, size_t(w) * size_t(h) * channels * sizeof(float), seed);
}
}  // namespace

uint64_t gsim_gpu_hash_target(int32_t width, int32_t height, const float* rgb, const float* depth,
                              const float* accum_alpha, uint64_t seed) {
    if (width < 0 || height < 0 || !rgb || !depth || !accum_alpha) return 0;
    uint64_t h = hash_image(width, height, rgb, 3, seed);
    h = hash_image(width, height, depth, 1, h);
    return hash_image(width, height, accum_alpha, 1, h);
}

void gsim_gpu_srgb_thresholds(float* thresholds) {
    if (thresholds) build_srgb_thresholds(thresholds);
}

int gsim_gpu_encode_host(gsim_gpu_context* ctx, int32_t width, int32_t height, const float* rgb,
                         const float* depth, const float* accum_alpha,
                         const gsim_encode_options* options, uint8_t* out) {
    return Guard(ctx).run([&] {
        const EncodeParams e0 = make_encode_params(ctx, options, nullptr);
        if (width <= 0 || height <= 0) throw ValidationError{"encode: empty image"};
        if (!out) throw ValidationError{"encode: out must not be NULL"};
        if ((e0.flags & GSIM_ENCODE_RGB8) && !rgb) throw ValidationError{"encode: rgb is NULL"};
        if ((e0.flags & (GSIM_ENCODE_DEPTH16 | GSIM_ENCODE_DEPTH_PFM)) && !depth)
            throw ValidationError{"encode: depth is NULL"};
        if ((e0.flags & GSIM_ENCODE_ALPHA8) && !accum_alpha)
            throw ValidationError{"encode: accum_alpha is NULL"};
        const uint64_t npx = uint64_t(width) * uint64_t(height);
        const uint64_t bytes = encoded_bpp(e0.flags) * npx;
        ctx->enc_src.reserve(5 * npx);
        ctx->enc_buf.reserve(bytes);
        cudaStream_t s = ctx->stream;
        if (rgb) GSIM_CK(cudaMemcpyAsync(ctx->enc_src.ptr, rgb, 12 * npx, cudaMemcpyHostToDevice, s));
        if (depth)
            GSIM_CK(cudaMemcpyAsync(ctx->enc_src.ptr + 3 * npx, depth, 4 * npx, cudaMemcpyHostToDevice, s));
        if (accum_alpha)
            GSIM_CK(cudaMemcpyAsync(ctx->enc_src.ptr + 4 * npx, accum_alpha, 4 * npx,
                                    cudaMemcpyHostToDevice, s));
        EncodeParams e = e0;
        e.dst = ctx->enc_buf.ptr;
        const uint32_t w = uint32_t(width), h = uint32_t(height);
        encode_device(ctx, ctx->enc_src.ptr, &w, &h, 1, e);
        GSIM_CK(cudaMemcpyAsync(out, ctx->enc_buf.ptr, bytes, cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaStreamSynchronize(s));
        ctx->stats.launches = 1;
        ctx->launches_total += 1;
        ctx->stats.launches_total = ctx->launches_total;
    });
}

int gsim_gpu_encode(gsim_gpu_context* ctx, const float* device_targets, const gsim_camera* cameras,
                    uint64_t n_cameras, const gsim_encode_options* options, uint8_t* out,
                    int32_t out_is_device) {
    return Guard(ctx).run([&] {
        EncodeParams e = make_encode_params(ctx, options, nullptr);
        if (n_cameras && (!device_targets || !cameras || !out))
            throw ValidationError{"encode: NULL targets, cameras or out"};
        std::vector<uint32_t> w(n_cameras), h(n_cameras);
        uint64_t bytes = 0;
        for (uint64_t c = 0; c < n_cameras; ++c) {
            validate_camera(cameras[c], c);
            w[c] = uint32_t(cameras[c].width);
            h[c] = uint32_t(cameras[c].height);
            bytes += uint64_t(encoded_bpp(e.flags)) * w[c] * h[c];
        }
        if (!n_cameras) return;
        if (out_is_device) {
            e.dst = out;
        } else {
            ctx->enc_buf.reserve(bytes);
            e.dst = ctx->enc_buf.ptr;
        }
        encode_device(ctx, device_targets, w.data(), h.data(), n_cameras, e);
        if (!out_is_device) {
            GSIM_CK(cudaMemcpyAsync(out, ctx->enc_buf.ptr, bytes, cudaMemcpyDeviceToHost, ctx->stream));
            GSIM_CK(cudaStreamSynchronize(ctx->stream));
        }
        const uint64_t launches = (n_cameras + 65534) / 65535;
        ctx->stats.launches = launches;
        ctx->launches_total += launches;
        ctx->stats.launches_total = ctx->launches_total;
    });
}

int gsim_gpu_render_encoded(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                            const gsim_node* nodes, uint64_t n_nodes, const gsim_camera* cameras,
                            uint64_t n_cameras, const gsim_raster_options* raster_options,
                            const gsim_encode_options* options, uint8_t* out,
                            int32_t out_is_device) {
    return Guard(ctx).run([&] {
        if (!scene || (n_nodes && !nodes)) throw ValidationError{"render: null argument"};
        EncodeParams e = make_encode_params(ctx, options, nullptr);
        if (n_cameras && (!cameras || !out)) throw ValidationError{"render: NULL cameras or out"};
        uint64_t bytes = 0;
        for (uint64_t c = 0; c < n_cameras; ++c) {
            validate_camera(cameras[c], c);
            bytes += uint64_t(encoded_bpp(e.flags)) * cameras[c].width * cameras[c].height;
        }
        if (out_is_device) {
            e.dst = out;
        } else {
            ctx->enc_buf.reserve(std::max<uint64_t>(bytes, 1));
            e.dst = ctx->enc_buf.ptr;
        }
        struct Reset {  // the fused encoding applies to this call only
            gsim_gpu_context* c;
            ~Reset() { c->frame_enc = EncodeParams{}; c->frame_enc_only = false; }
        } reset{ctx};
        ctx->frame_enc = e;
        ctx->frame_enc_only = true;
        const bool overlap = !out_is_device && ctx->overlap_copies;
        if (overlap && !ctx->copy_stream)
            GSIM_CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        ctx->copies_stale = false;
        ctx->frame_enc_host = overlap ? out : nullptr;
        try {
            render_cameras(ctx, scene, nodes, n_nodes, cameras, n_cameras, raster_options, nullptr,
                           false);
        } catch (...) {
            ctx->frame_enc_host = nullptr;
            if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
            throw;
        }
        ctx->frame_enc_host = nullptr;
        if (overlap) {
            GSIM_CK(cudaStreamSynchronize(ctx->copy_stream));
            GSIM_CK(cudaStreamSynchronize(ctx->stream));
            ctx->stats.d2h_bytes = bytes;
            if (check_pending(ctx) || ctx->copies_stale) {
                if (bytes)
                    GSIM_CK(cudaMemcpyAsync(out, ctx->enc_buf.ptr, bytes, cudaMemcpyDeviceToHost, ctx->stream));
                GSIM_CK(cudaStreamSynchronize(ctx->stream));
            }
        } else if (!out_is_device) {
            // one check at the end, as gsim_gpu_render; the encoding of a re-run tail is part
            // of its raster epilogue (check_pending restores the frame's encode parameters)
            for (int pass = 0; pass < 2; ++pass) {
                if (bytes)
                    GSIM_CK(cudaMemcpyAsync(out, ctx->enc_buf.ptr, bytes, cudaMemcpyDeviceToHost,
                                            ctx->stream));
                GSIM_CK(cudaStreamSynchronize(ctx->stream));
                ctx->stats.d2h_bytes = bytes;
                if (!check_pending(ctx)) break;
            }
        }
    });
}

int gsim_gpu_tracks_upload(gsim_gpu_context* ctx, const double* times, const double* translations,
                           const double* rotations, const uint64_t* track_begin, uint64_t n_tracks,
                           gsim_gpu_tracks** out) {
    if (out) *out = nullptr;
    return Guard(ctx).run([&] {
        if (!out || (n_tracks && !track_begin)) throw ValidationError{"tracks: null argument"};
        if (n_tracks >= (uint64_t(1) << 31)) throw ValidationError{"tracks: too many tracks"};
        const uint64_t R = n_tracks ? track_begin[n_tracks] : 0;
        if (n_tracks && track_begin[0] != 0) throw ValidationError{"tracks: track_begin[0] must be 0"};
        if (R && (!times || !translations || !rotations)) throw ValidationError{"tracks: null record array"};
        std::vector<double> q(4 * R);
        for (uint64_t k = 0; k < n_tracks; ++k) {
            if (track_begin[k + 1] < track_begin[k]) throw ValidationError{"tracks: track_begin decreases"};
            for (uint64_t i = track_begin[k]; i < track_begin[k + 1]; ++i) {
                // PoseStream::append (pose_stream.cpp:20-40)
                const std::string who = "pose stream: track " + std::to_string(k);
                if (!std::isfinite(times[i])) throw ValidationError{who + ": non-finite timestamp"};
                for (int c = 0; c < 3; ++c)
                    if (!std::isfinite(translations[3 * i + c])) throw ValidationError{who + ": non-finite pose"};
                for (int c = 0; c < 4; ++c)
                    if (!std::isfinite(rotations[4 * i + c])) throw ValidationError{who + ": non-finite pose"};
                if (i > track_begin[k] && times[i] < times[i - 1])
                    throw ValidationError{who + ": timestamps decrease"};
                const dq n = qnormalized(dq{rotations[4 * i], rotations[4 * i + 1], rotations[4 * i + 2],
                                            rotations[4 * i + 3]});
                q[4 * i] = n.w; q[4 * i + 1] = n.x; q[4 * i + 2] = n.y; q[4 * i + 3] = n.z;
            }
        }
        auto* tr = new gsim_gpu_tracks;
        tr->ctx = ctx;
        tr->n_tracks = n_tracks;
        tr->n_records = R;
        const size_t bt = 8 * R, bp = 24 * R, bq = 32 * R, bb = 8 * (n_tracks + 1);
        if (cudaMalloc(&tr->mem, std::max<size_t>(bt + bp + bq + bb, 64)) != cudaSuccess) {
            delete tr;
            throw CudaError{"tracks: device allocation failed"};
        }
        char* m = static_cast<char*>(tr->mem);
        std::vector<uint64_t> begin(n_tracks + 1, 0);
        for (uint64_t k = 0; k <= n_tracks && n_tracks; ++k) begin[k] = track_begin[k];
        if (R) {
            GSIM_CK(cudaMemcpy(m, times, bt, cudaMemcpyHostToDevice));
            GSIM_CK(cudaMemcpy(m + bt, translations, bp, cudaMemcpyHostToDevice));
            GSIM_CK(cudaMemcpy(m + bt + bp, q.data(), bq, cudaMemcpyHostToDevice));
        }
        GSIM_CK(cudaMemcpy(m + bt + bp + bq, begin.data(), bb, cudaMemcpyHostToDevice));
        tr->d.t = reinterpret_cast<const double*>(m);
        tr->d.p = reinterpret_cast<const double*>(m + bt);
        tr->d.q = reinterpret_cast<const double*>(m + bt + bp);
        tr->d.begin = reinterpret_cast<const uint64_t*>(m + bt + bp + bq);
        tr->d.n_tracks = uint32_t(n_tracks);
        ctx->tracks.insert(tr);
        *out = tr;
    });
}

int gsim_gpu_tracks_destroy(gsim_gpu_tracks* tracks) {
    if (!tracks) return GSIM_OK;
    if (tracks->ctx) {
        std::lock_guard<std::mutex> lk(tracks->ctx->mu);
        cudaSetDevice(tracks->ctx->device);
        cudaStreamSynchronize(tracks->ctx->stream);
        tracks->ctx->tracks.erase(tracks);
    }
    if (tracks->mem) cudaFree(tracks->mem);
    delete tracks;
    return GSIM_OK;
}

uint64_t gsim_gpu_tracks_count(const gsim_gpu_tracks* tracks) { return tracks ? tracks->n_tracks : 0; }

int gsim_gpu_tracks_sample(gsim_gpu_context* ctx, const gsim_gpu_tracks* tracks,
                           const uint32_t* track, const double* time, const gsim_rigid* initial,
                           uint64_t n, gsim_rigid* out) {
    return Guard(ctx).run([&] {
        if (!tracks || (n && (!track || !time || !initial || !out)))
            throw ValidationError{"tracks_sample: null argument"};
        for (uint64_t i = 0; i < n; ++i)
            if (track[i] >= tracks->n_tracks)
                throw ValidationError{"tracks_sample: query " + std::to_string(i) + " names track " +
                                      std::to_string(track[i]) + " of " + std::to_string(tracks->n_tracks)};
        if (!n) return;
        const size_t b_tr = (4 * n + 15) & ~size_t(15), b_t = 8 * n, b_r = sizeof(gsim_rigid) * n;
        ctx->query_buf.reserve(b_tr + b_t + 2 * b_r);
        char* m = ctx->query_buf.ptr;
        cudaStream_t s = ctx->stream;
        GSIM_CK(cudaMemcpyAsync(m, track, 4 * n, cudaMemcpyHostToDevice, s));
        GSIM_CK(cudaMemcpyAsync(m + b_tr, time, b_t, cudaMemcpyHostToDevice, s));
        GSIM_CK(cudaMemcpyAsync(m + b_tr + b_t, initial, b_r, cudaMemcpyHostToDevice, s));
        gsim_rigid* dout = reinterpret_cast<gsim_rigid*>(m + b_tr + b_t + b_r);
        launch_track_query(tracks->d, reinterpret_cast<const uint32_t*>(m),
                           reinterpret_cast<const double*>(m + b_tr),
                           reinterpret_cast<const gsim_rigid*>(m + b_tr + b_t), dout, n,
                           ctx->num_sms * 8, s);
        check_launch();
        GSIM_CK(cudaMemcpyAsync(out, dout, b_r, cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaStreamSynchronize(s));
        ctx->stats.launches = 1;
        ctx->launches_total += 1;
        ctx->stats.launches_total = ctx->launches_total;
    });
}

int gsim_gpu_render_at(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                       const gsim_gpu_tracks* tracks, double time, const gsim_node* nodes,
                       const int64_t* node_track, uint64_t n_nodes, const gsim_camera* cameras,
                       uint64_t n_cameras, const gsim_raster_options* options, float* device_out,
                       gsim_target* outs) {
    return Guard(ctx).run([&] {
        if (!scene || !tracks || (n_nodes && (!nodes || !node_track)) || (n_cameras && !cameras))
            throw ValidationError{"render_at: null argument"};
        if (!std::isfinite(time)) throw ValidationError{"render_at: non-finite time"};
        for (uint64_t k = 0; k < n_nodes; ++k) {
            if (node_track[k] < 0) continue;
            if (uint64_t(node_track[k]) >= tracks->n_tracks)
                throw ValidationError{"render_at: node " + std::to_string(k) + " names track " +
                                      std::to_string(node_track[k]) + " of " +
                                      std::to_string(tracks->n_tracks)};
            if (nodes[k].kind == GSIM_NODE_BACKGROUND)  // scene.cpp:180-184
                throw ValidationError{"pose stream drives background node " + std::to_string(k)};
        }
        struct Reset {
            gsim_gpu_context* c;
            ~Reset() { c->frame_tracks = nullptr; c->frame_node_track = nullptr; }
        } reset{ctx};
        ctx->frame_tracks = tracks;
        ctx->frame_time = time;
        ctx->frame_node_track = node_track;
        const bool host = outs != nullptr;
        const std::vector<uint64_t> off = render_cameras(ctx, scene, nodes, n_nodes, cameras, n_cameras,
                                                         options, host ? nullptr : device_out, false);
        if (host) {
            copy_targets(ctx, cameras, n_cameras, off, outs);
            if (check_pending(ctx)) copy_targets(ctx, cameras, n_cameras, off, outs);
        }
    });
}

int gsim_gpu_tile_lists(gsim_gpu_context* ctx, uint32_t camera, uint32_t* tile_begin,
                        uint32_t* values, uint64_t capacity, uint64_t* count) {
    return Guard(ctx).run([&] {
        const Plan& p = ctx->last_plan;
        if (camera >= p.cams.size()) throw ValidationError{"tile_lists: no such camera in the last render"};
        if (!count) throw ValidationError{"tile_lists: null count"};
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
        const uint32_t t0 = p.tile_base[camera], nt = p.tile_base[camera + 1] - t0;
        std::vector<uint32_t> rel(nt), cnt(nt);
        uint64_t pbase = 0;
        if (nt) {
            GSIM_CK(cudaMemcpy(rel.data(), ctx->tile_rel.ptr + t0, nt * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            GSIM_CK(cudaMemcpy(cnt.data(), ctx->tile_count.ptr + t0, nt * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            GSIM_CK(cudaMemcpy(&pbase, ctx->cam_pair_base.ptr + camera, sizeof(uint64_t), cudaMemcpyDeviceToHost));
        }
        uint64_t total = 0;
        for (uint32_t t = 0; t < nt; ++t) {
            if (tile_begin) tile_begin[t] = uint32_t(total);
            if (rel[t] != total) throw CudaError{"tile_lists: inconsistent tile offsets"};
            total += cnt[t];
        }
        if (tile_begin) tile_begin[nt] = uint32_t(total);
        *count = total;
        if (values && total) {
            std::vector<uint32_t> v(total);
            GSIM_CK(cudaMemcpy(v.data(), ctx->vals.ptr + pbase, total * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            const uint64_t sb = p.slot_base[camera];
            for (uint64_t k = 0; k < total && k < capacity; ++k) values[k] = uint32_t(v[k] - sb);
        }
    });
}

// ---- GS -> TSDF (transfer.cpp) ------------------------------------------

int gsim_gpu_scene_bounds(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, double lo[3],
                          double hi[3]) {
    return Guard(ctx).run([&] {
        if (!scene || !lo || !hi) throw ValidationError{"scene_bounds: null argument"};
        scene_bounds(ctx, scene, lo, hi);
    });
}

int gsim_gpu_depth_ring_cameras(const double lo[3], const double hi[3], int32_t n_views,
                                double radius, int32_t resolution, gsim_camera* cameras) {
    if (!lo || !hi || !cameras) return GSIM_ERR_VALIDATION;
    return gsim_gpu::depth_ring_cameras(lo, hi, n_views, radius, resolution, cameras)
               ? GSIM_ERR_VALIDATION
               : GSIM_OK;
}

int gsim_gpu_render_depth_ring(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                               int32_t n_views, double radius, int32_t resolution,
                               gsim_camera* cameras, float* depth, int32_t depth_is_device) {
    return Guard(ctx).run([&] {
        if (!scene || !depth) throw ValidationError{"render_depth_ring: null argument"};
        std::vector<gsim_camera> cams;
        const std::vector<uint64_t> off =
            depth_ring_render(ctx, scene, n_views, radius, resolution, cams);
        if (cameras) std::copy(cams.begin(), cams.end(), cameras);
        // depth plane of every camera block [rgb 3 npx | depth npx | alpha npx]
        const size_t npx = size_t(resolution) * resolution;
        GSIM_CK(cudaMemcpy2DAsync(depth, npx * sizeof(float), ctx->out.ptr + 3 * npx,
                                  5 * npx * sizeof(float), npx * sizeof(float), cams.size(),
                                  depth_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                  ctx->stream));
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
        (void)off;
    });
}

int gsim_gpu_tsdf_create(const double origin[3], double voxel_size, const int32_t dims[3],
                         double truncation, gsim_tsdf_volume* volume) {
    // TsdfVolume::create, transfer.cpp:126-141 (geometry only; the grids are the caller's)
    if (!origin || !dims || !volume) return GSIM_ERR_VALIDATION;
    if (!(voxel_size > 0.0)) return GSIM_ERR_VALIDATION;
    if (dims[0] < 2 || dims[1] < 2 || dims[2] < 2) return GSIM_ERR_VALIDATION;
    if (truncation < 2.0 * voxel_size) return GSIM_ERR_VALIDATION;
    for (int k = 0; k < 3; ++k) {
        volume->origin[k] = origin[k];
        volume->dims[k] = dims[k];
    }
    volume->voxel_size = voxel_size;
    volume->truncation = truncation;
    return GSIM_OK;
}

int gsim_gpu_tsdf_reset(gsim_gpu_context* ctx, const gsim_tsdf_volume* volume) {
    return Guard(ctx).run([&] {
        check_volume(volume, true);
        const uint64_t n = uint64_t(volume->dims[0]) * volume->dims[1] * volume->dims[2];
        launch_tsdf_reset(volume->tsdf, volume->weights, n, ctx->num_sms, ctx->stream);
        check_launch();
    });
}

int gsim_gpu_tsdf_fuse(gsim_gpu_context* ctx, const gsim_tsdf_volume* volume,
                       const gsim_camera* cameras, uint64_t n_views, const float* depth,
                       int32_t depth_is_device) {
    return Guard(ctx).run([&] {
        check_volume(volume, true);
        if (n_views && (!cameras || !depth)) throw ValidationError{"tsdf_fuse: null argument"};
        std::vector<DevFuseView> views(n_views);
        uint64_t total = 0;
        for (uint64_t k = 0; k < n_views; ++k) {
            validate_camera(cameras[k], k);  // tsdf_fuse validates its camera (transfer.cpp:144)
            views[k] = fuse_view(cameras[k], total);
            total += uint64_t(cameras[k].width) * cameras[k].height;
        }
        const float* src = depth;
        if (!depth_is_device && total) {
            ctx->depth_in.reserve(total);
            GSIM_CK(cudaMemcpyAsync(ctx->depth_in.ptr, depth, total * sizeof(float),
                                    cudaMemcpyHostToDevice, ctx->stream));
            src = ctx->depth_in.ptr;
        }
        fuse_views(ctx, volume, views, src);
    });
}

int gsim_gpu_tsdf_alloc(gsim_gpu_context* ctx, gsim_tsdf_volume* volume) {
    return Guard(ctx).run([&] {
        check_volume(volume, false);
        const uint64_t n = uint64_t(volume->dims[0]) * volume->dims[1] * volume->dims[2];
        double* t = nullptr;
        double* w = nullptr;
        GSIM_CK(cudaMalloc(&t, n * sizeof(double)));
        if (cudaMalloc(&w, n * sizeof(double)) != cudaSuccess) {
            cudaFree(t);
            throw CudaError{"tsdf_alloc: out of device memory"};
        }
        volume->tsdf = t;
        volume->weights = w;
    });
}

int gsim_gpu_tsdf_free(gsim_tsdf_volume* volume) {
    if (!volume) return GSIM_ERR_VALIDATION;
    if (volume->tsdf) cudaFree(volume->tsdf);
    if (volume->weights) cudaFree(volume->weights);
    volume->tsdf = nullptr;
    volume->weights = nullptr;
    return GSIM_OK;
}

int gsim_gpu_tsdf_download(gsim_gpu_context* ctx, const gsim_tsdf_volume* volume, double* tsdf,
                           double* weights) {
    return Guard(ctx).run([&] {
        check_volume(volume, true);
        const uint64_t n = uint64_t(volume->dims[0]) * volume->dims[1] * volume->dims[2];
        if (tsdf)
            GSIM_CK(cudaMemcpyAsync(tsdf, volume->tsdf, n * sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
        if (weights)
            GSIM_CK(cudaMemcpyAsync(weights, volume->weights, n * sizeof(double),
                                    cudaMemcpyDeviceToHost, ctx->stream));
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsim_gpu_tsdf_upload(gsim_gpu_context* ctx, const gsim_tsdf_volume* volume, const double* tsdf,
                         const double* weights) {
    return Guard(ctx).run([&] {
        check_volume(volume, true);
        const uint64_t n = uint64_t(volume->dims[0]) * volume->dims[1] * volume->dims[2];
        if (tsdf)
            GSIM_CK(cudaMemcpyAsync(volume->tsdf, tsdf, n * sizeof(double), cudaMemcpyHostToDevice,
                                    ctx->stream));
        if (weights)
            GSIM_CK(cudaMemcpyAsync(volume->weights, weights, n * sizeof(double),
                                    cudaMemcpyHostToDevice, ctx->stream));
        GSIM_CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsim_gpu_gaussians_to_tsdf(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                               double voxel_size, gsim_tsdf_volume* volume) {
    // gaussians_to_mesh up to the fused volume, transfer.cpp:174-198
    return Guard(ctx).run([&] {
        if (!scene || !volume) throw ValidationError{"gaussians_to_tsdf: null argument"};
        if (scene->f.n == 0) throw ValidationError{"gaussians_to_mesh: empty field"};
        if (!(voxel_size > 0.0)) throw ValidationError{"gaussians_to_mesh: voxel_size must be positive"};
        double blo[3], bhi[3];
        scene_bounds(ctx, scene, blo, bhi);
        const dv3 bl = mk3(blo[0], blo[1], blo[2]), bh = mk3(bhi[0], bhi[1], bhi[2]);
        const dv3 ext_box = sub3(bh, bl);
        const double diag =
            std::sqrt(ext_box.x * ext_box.x + ext_box.y * ext_box.y + ext_box.z * ext_box.z);
        if (!(diag > 0.0)) throw ValidationError{"gaussians_to_mesh: degenerate field bounding box"};
        const double truncation = 3.0 * voxel_size;
        const double margin = truncation + 2.0 * voxel_size;
        const dv3 lo = sub3(bl, mk3(margin, margin, margin));
        const dv3 hi = add3(bh, mk3(margin, margin, margin));
        const dv3 extent = sub3(hi, lo);
        const double e[3] = {extent.x, extent.y, extent.z};
        int32_t dims[3];
        for (int k = 0; k < 3; ++k)
            dims[k] = std::max(2, static_cast<int>(std::ceil(e[k] / voxel_size)) + 1);
        double* tsdf = volume->tsdf;
        double* weights = volume->weights;
        const double origin[3] = {lo.x, lo.y, lo.z};
        if (gsim_gpu_tsdf_create(origin, voxel_size, dims, truncation, volume) != GSIM_OK)
            throw ValidationError{"tsdf: invalid volume"};
        volume->tsdf = tsdf;
        volume->weights = weights;
        if (!tsdf) return;  // geometry-only call
        check_volume(volume, true);
        const uint64_t n = uint64_t(dims[0]) * dims[1] * dims[2];
        launch_tsdf_reset(volume->tsdf, volume->weights, n, ctx->num_sms, ctx->stream);
        check_launch();
        constexpr int kFusionAzimuths = 20, kFusionResolution = 256;  // transfer.cpp:25-26
        constexpr double kRingRadiusFactor = 2.5;                      // transfer.cpp:24
        std::vector<gsim_camera> cams;
        const std::vector<uint64_t> off = depth_ring_render(
            ctx, scene, kFusionAzimuths, kRingRadiusFactor * diag, kFusionResolution, cams);
        // fuse straight from the render output: depth plane of camera c at off[c] + 3 npx
        const uint64_t npx = uint64_t(kFusionResolution) * kFusionResolution;
        std::vector<DevFuseView> views(cams.size());
        for (size_t k = 0; k < cams.size(); ++k) views[k] = fuse_view(cams[k], off[k] + 3 * npx);
        fuse_views(ctx, volume, views, ctx->out.ptr);
    });
}

// ---- LiDAR (trace.cpp) -----------------------------------------------------

int gsim_gpu_lidar_scan(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                        uint64_t n_nodes, const gsim_lidar* lidar, double* points, uint32_t* ring,
                        double* azimuth, uint64_t capacity, uint64_t* count) {
    return Guard(ctx).run([&] {
        if (!scene || !lidar || !count || (n_nodes && !nodes))
            throw ValidationError{"lidar_scan: null argument"};
        auto& L = ctx->lidar;
        cudaStream_t s = ctx->stream;
        // GaussianBvh::build validates the nodes before scan validates the sensor
        LidarArgs a = lidar_pose_stage(ctx, scene, nodes, n_nodes, lidar->env, true);
        validate_lidar(*lidar);
        constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
        const uint64_t n_az = uint64_t(std::llround(kTwoPi / lidar->azimuth_step));
        const uint64_t n_ch = lidar->n_channels;
        const uint64_t n_rays = n_ch * n_az;
        if (n_az == 0 || n_az > (1u << 30) || n_ch > 65535)
            throw ValidationError{"lidar: ray grid too large"};
        // Sensor-frame ray directions exactly as GaussianBvh::scan builds them (trace.cpp:
        // 180-186, glibc cos / sin) are computed on the host once per (channels, step) and kept
        // on the device; the world directions (the pose rotation) are a kernel.
        std::vector<double> key(lidar->channels, lidar->channels + n_ch);
        key.push_back(lidar->azimuth_step);
        L.rays.reserve(std::max<uint64_t>(6 * n_rays, 1));
        if (key != L.ray_key) {
            std::vector<double> ds(3 * n_rays);
            for (uint64_t k = 0; k < n_rays; ++k) {
                const double elevation = lidar->channels[k / n_az];
                const double az = static_cast<double>(k % n_az) * lidar->azimuth_step;
                const double ce = std::cos(elevation);
                ds[3 * k] = ce * std::cos(az);
                ds[3 * k + 1] = ce * std::sin(az);
                ds[3 * k + 2] = std::sin(elevation);
            }
            GSIM_CK(cudaMemcpyAsync(L.rays.ptr + 3 * n_rays, ds.data(), ds.size() * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
            GSIM_CK(cudaStreamSynchronize(s));  // ds dies with this scope
            L.ray_key = key;
        }
        launch_lidar_rays(L.rays.ptr + 3 * n_rays, L.rays.ptr, n_rays, lidar->pose.rotation,
                          ctx->num_sms, s);
        check_launch();
        // regular channels (cos(elevation) clearly positive) bin by elevation rank; rays of the
        // others take every primitive as a candidate
        std::vector<std::pair<double, uint32_t>> reg;
        std::vector<uint8_t> ray_all(n_ch, 0);
        for (uint64_t c = 0; c < n_ch; ++c) {
            const double e = lidar->channels[c];
            if (std::cos(e) > 1e-3) reg.push_back({e, uint32_t(c)});
            else ray_all[c] = 1;
        }
        std::sort(reg.begin(), reg.end());
        std::vector<double> rank_elev;
        std::vector<uint32_t> rank_channel;
        for (const auto& r : reg) {
            rank_elev.push_back(r.first);
            rank_channel.push_back(r.second);
        }
        L.ray_all.reserve(n_ch);
        GSIM_CK(cudaMemcpyAsync(L.ray_all.ptr, ray_all.data(), n_ch, cudaMemcpyHostToDevice, s));
        L.rank_elev.reserve(std::max<size_t>(rank_elev.size(), 1));
        L.rank_channel.reserve(std::max<size_t>(rank_channel.size(), 1));
        if (!rank_elev.empty()) {
            GSIM_CK(cudaMemcpyAsync(L.rank_elev.ptr, rank_elev.data(), rank_elev.size() * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
            GSIM_CK(cudaMemcpyAsync(L.rank_channel.ptr, rank_channel.data(),
                                    rank_channel.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        }
        // world -> sensor pose (RigidTransform::inverse, math.hpp:235-238)
        const dq sq{lidar->pose.rotation[0], lidar->pose.rotation[1], lidar->pose.rotation[2],
                    lidar->pose.rotation[3]};
        const dq wq{sq.w, -sq.x, -sq.y, -sq.z};
        const dv3 wt = qrotate(wq, mk3(lidar->pose.translation[0], lidar->pose.translation[1],
                                       lidar->pose.translation[2]));
        a.w2s_q[0] = wq.w; a.w2s_q[1] = wq.x; a.w2s_q[2] = wq.y; a.w2s_q[3] = wq.z;
        a.w2s_t[0] = -wt.x; a.w2s_t[1] = -wt.y; a.w2s_t[2] = -wt.z;
        for (int c = 0; c < 3; ++c) a.origin[c] = lidar->pose.translation[c];
        a.max_range = lidar->max_range;
        a.step = lidar->azimuth_step;
        a.rank_elev = L.rank_elev.ptr;
        a.rank_channel = L.rank_channel.ptr;
        a.n_ranks = int(rank_elev.size());
        a.n_az = uint32_t(n_az);
        a.n_rays = n_rays;
        a.ray_dir = L.rays.ptr;
        a.ray_dir_sensor = L.rays.ptr + 3 * n_rays;
        a.ray_all = L.ray_all.ptr;
        a.alpha_threshold = lidar->alpha_threshold;
        launch_lidar_pose(a, ctx->num_sms, s);
        check_launch();
        // bin: row differences -> candidates per ray -> offsets -> candidate lists
        L.diff.reserve(n_ch * (n_az + 1));
        GSIM_CK(cudaMemsetAsync(L.diff.ptr, 0, n_ch * (n_az + 1) * sizeof(int), s));
        a.diff = L.diff.ptr;
        launch_lidar_count(a, ctx->num_sms, s);
        check_launch();
        L.counts.reserve(n_rays);
        a.ray_count = L.counts.ptr;
        launch_lidar_rowscan(a, uint32_t(n_ch), s);
        check_launch();
        L.offsets.reserve(n_rays + 1);
        L.scratch.reserve((n_rays + 1023) / 1024 + 2);
        exclusive_scan_u32(L.counts.ptr, n_rays, L.offsets.ptr, L.scratch.ptr, s);
        check_launch();
        unsigned long long pairs = 0;
        uint32_t n_all = 0;
        GSIM_CK(cudaMemcpyAsync(&pairs, L.offsets.ptr + n_rays, sizeof(pairs), cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaMemcpyAsync(&n_all, a.all_count, sizeof(n_all), cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaStreamSynchronize(s));
        const uint64_t cache = std::max<uint64_t>(pairs + n_rays * uint64_t(n_all), 1);
        L.cand_t.reserve(cache);
        L.cand_r.reserve(cache);
        a.cand_t = L.cand_t.ptr;
        a.cand_r = L.cand_r.ptr;
        if (pairs >= (1ull << 32)) throw CudaError{"lidar: more than 2^32 ray candidates"};
        L.list.reserve(std::max<unsigned long long>(pairs, 1));
        L.cursor.reserve(n_rays);
        GSIM_CK(cudaMemsetAsync(L.cursor.ptr, 0, n_rays * sizeof(uint32_t), s));
        L.big_list.reserve(std::max<uint64_t>(scene->f.n, 1) + 1);
        GSIM_CK(cudaMemsetAsync(L.big_list.ptr, 0, sizeof(uint32_t), s));
        a.ray_offset = L.offsets.ptr;
        a.cursor = L.cursor.ptr;
        a.big_count = L.big_list.ptr;
        a.big_list = L.big_list.ptr + 1;
        a.list = L.list.ptr;
        launch_lidar_scatter(a, ctx->num_sms, s);
        check_launch();
        launch_lidar_scatter_big(a, ctx->num_sms, s);
        check_launch();
        // trace every ray, then compact the returns in ray order
        L.hit.reserve(n_rays);
        L.depth.reserve(n_rays);
        L.acc.reserve(n_rays);
        a.out_hit = L.hit.ptr;
        a.out_depth = L.depth.ptr;
        a.out_acc = L.acc.ptr;
        static const bool debug = std::getenv("GSIM_GPU_LIDAR_DEBUG") != nullptr;
        if (debug) {
            L.scratch.reserve((n_rays + 1023) / 1024 + 8);
            a.debug = L.scratch.ptr + (n_rays + 1023) / 1024 + 4;
            GSIM_CK(cudaMemsetAsync(a.debug, 0, 3 * sizeof(unsigned long long), s));
        }
        launch_lidar_trace(a, ctx->num_sms, s);
        check_launch();
        if (debug) {
            unsigned long long d[3];
            GSIM_CK(cudaMemcpyAsync(d, a.debug, sizeof(d), cudaMemcpyDeviceToHost, s));
            GSIM_CK(cudaStreamSynchronize(s));
            std::fprintf(stderr, "lidar: rays %llu candidates %llu (%.1f per ray), pairs %llu, around the sensor %u\n",
                         d[0], d[1], double(d[1]) / double(std::max(d[0], 1ull)), pairs, n_all);
        }
        L.hit_offsets.reserve(n_rays + 1);
        exclusive_scan_u32(L.hit.ptr, n_rays, L.hit_offsets.ptr, L.scratch.ptr, s);
        check_launch();
        unsigned long long hits = 0;
        GSIM_CK(cudaMemcpyAsync(&hits, L.hit_offsets.ptr + n_rays, sizeof(hits), cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaStreamSynchronize(s));
        *count = hits;
        if (hits > capacity || hits == 0) return;
        if (!points || !ring || !azimuth) throw ValidationError{"lidar_scan: null output"};
        L.points.reserve(3 * hits);
        L.ring.reserve(hits);
        L.azimuth.reserve(hits);
        a.hit_offset = L.hit_offsets.ptr;
        a.capacity = hits;
        a.points = L.points.ptr;
        a.ring = L.ring.ptr;
        a.azimuth = L.azimuth.ptr;
        launch_lidar_emit(a, ctx->num_sms, s);
        check_launch();
        GSIM_CK(cudaMemcpyAsync(points, L.points.ptr, 3 * hits * sizeof(double), cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaMemcpyAsync(ring, L.ring.ptr, hits * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaMemcpyAsync(azimuth, L.azimuth.ptr, hits * sizeof(double), cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaStreamSynchronize(s));
    });
}

int gsim_gpu_trace_rays(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                        uint64_t n_nodes, const double* origins, const double* directions,
                        const double* t_max, uint64_t n_rays, double alpha_threshold,
                        uint8_t* hit, double* depth, double* accum_alpha) {
    return Guard(ctx).run([&] {
        if (!scene || (n_nodes && !nodes) ||
            (n_rays && (!origins || !directions || !t_max || !hit || !depth || !accum_alpha)))
            throw ValidationError{"trace_rays: null argument"};
        auto& L = ctx->lidar;
        cudaStream_t s = ctx->stream;
        LidarArgs a = lidar_pose_stage(ctx, scene, nodes, n_nodes, GSIM_ENV_ALL, false);
        if (!n_rays) return;
        L.rays.reserve(7 * n_rays);
        GSIM_CK(cudaMemcpyAsync(L.rays.ptr, origins, 3 * n_rays * sizeof(double), cudaMemcpyHostToDevice, s));
        GSIM_CK(cudaMemcpyAsync(L.rays.ptr + 3 * n_rays, directions, 3 * n_rays * sizeof(double),
                                cudaMemcpyHostToDevice, s));
        GSIM_CK(cudaMemcpyAsync(L.rays.ptr + 6 * n_rays, t_max, n_rays * sizeof(double),
                                cudaMemcpyHostToDevice, s));
        a.n_rays = n_rays;
        a.ray_origin = L.rays.ptr;
        a.ray_dir = L.rays.ptr + 3 * n_rays;
        a.ray_tmax = L.rays.ptr + 6 * n_rays;
        a.alpha_threshold = alpha_threshold;
        launch_lidar_pose(a, ctx->num_sms, s);
        check_launch();
        // GSIM_GPU_TRACE_BRUTE=1: every primitive is every ray's candidate (A/B and tests)
        static const bool brute = [] {
            const char* e = std::getenv("GSIM_GPU_TRACE_BRUTE");
            return e && std::atoi(e) == 1;
        }();
        if (!brute && scene->f.n) ctx->stats.pairs = bvh_ray_lists(ctx, a);
        L.hit.reserve(n_rays);
        L.depth.reserve(n_rays);
        L.acc.reserve(n_rays);
        a.out_hit = L.hit.ptr;
        a.out_depth = L.depth.ptr;
        a.out_acc = L.acc.ptr;
        launch_lidar_trace(a, ctx->num_sms, s);
        check_launch();
        std::vector<uint32_t> h(n_rays);
        GSIM_CK(cudaMemcpyAsync(h.data(), L.hit.ptr, n_rays * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaMemcpyAsync(depth, L.depth.ptr, n_rays * sizeof(double), cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaMemcpyAsync(accum_alpha, L.acc.ptr, n_rays * sizeof(double), cudaMemcpyDeviceToHost, s));
        GSIM_CK(cudaStreamSynchronize(s));
        for (uint64_t k = 0; k < n_rays; ++k) hit[k] = uint8_t(h[k]);
    });
}

}  // extern "C"
