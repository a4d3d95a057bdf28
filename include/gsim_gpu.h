/*
 * gsim_gpu.h — C ABI of the B200-native multi-camera RGB-D Gaussian-splat renderer.
 *
 * This is the drop-in boundary for the reference's render path
 * (/root/reference/proj/core/include/gsim/raster.hpp:54-67):
 *
 *   std::vector<ProjectedSplat> project(const GaussianField&, const std::vector<SceneNode>&,
 *                                       const CameraModel&);                 raster.hpp:54-56
 *   RenderTarget rasterize(const std::vector<ProjectedSplat>&, const CameraModel&,
 *                          const RasterOptions& = {});                       raster.hpp:59-60
 *   std::vector<RenderTarget> render(const GaussianField&, const std::vector<SceneNode>&,
 *                                    const std::vector<CameraModel>&,
 *                                    const RasterOptions& = {});             raster.hpp:64-67
 *   void transform_primitives(GaussianField&, const IndexRange&,
 *                             const RigidTransform&);                        gaussian.hpp:76-77
 *
 * Plain C: pointers, sizes and POD structs only, no C++ or torch types. Every entry point
 * returns a status that mirrors the reference CLI contract (tools/gsim.cpp:366-375,
 * errors.hpp:12-25): 0 = ok, 1 = io/runtime (CUDA) failure, 2 = validation error.
 * The message of the last failure on a context is available from gsim_gpu_last_error().
 *
 * Ownership: inputs are read during the call and never retained (the scene upload copies
 * the field into device memory). Host outputs are written by the time a host-output call
 * returns. Calls on one context are serialised by an internal mutex; different contexts
 * (one per device) run concurrently.
 */
#ifndef GSIM_GPU_H
#define GSIM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSIM_OK 0
#define GSIM_ERR_IO 1
#define GSIM_ERR_VALIDATION 2

#define GSIM_NODE_BACKGROUND 0  /* NodeKind::background, gaussian.hpp:64 */
#define GSIM_NODE_INTERACTIVE 1 /* NodeKind::interactive */
#define GSIM_ENV_ALL (-1)       /* node visible to every camera (the reference's only mode) */

/* RigidTransform (math.hpp:217-239): x -> R(q) x + t, q stored (w, x, y, z). */
typedef struct gsim_rigid {
    double rotation[4];
    double translation[3];
} gsim_rigid;

/* GaussianField (gaussian.hpp:53-60) as strided double views. A stride is the distance,
 * in doubles, between consecutive primitives, so the reference's AoS GaussianPrimitive
 * array (stride 59) and SoA numpy arrays (strides 3, 3, 4, 1, 48) are both valid views.
 * sh holds 48 coefficients per primitive, channel-major sh[c*16 + k] (gaussian.hpp:16-19). */
typedef struct gsim_field_view {
    uint64_t count;
    int32_t sh_degree; /* 0..3, global across the field (scene.cpp:92) */
    int32_t reserved;
    const double* means;
    uint64_t means_stride;
    const double* scales; /* linear, > 0 */
    uint64_t scales_stride;
    const double* rotations; /* unit quaternion (w, x, y, z) */
    uint64_t rotations_stride;
    const double* opacities; /* post-sigmoid, (0, 1) */
    uint64_t opacities_stride;
    const double* sh;
    uint64_t sh_stride;
} gsim_field_view;

/* SceneNode (gaussian.hpp:66-71) plus an environment tag for batched rendering.
 * env == GSIM_ENV_ALL reproduces the reference exactly; env >= 0 restricts the node to the
 * cameras whose env equals it (BASELINE configs 2 and 4: shared background, per-env objects). */
typedef struct gsim_node {
    uint64_t begin; /* IndexRange, end exclusive */
    uint64_t end;
    gsim_rigid pose;
    int32_t kind;
    int32_t env;
} gsim_node;

/* CameraModel (camera.hpp:14-33): pose maps world -> camera (x right, y down, z forward). */
typedef struct gsim_camera {
    double fx, fy, cx, cy;
    int32_t width, height;
    gsim_rigid pose;
    double near_plane, far_plane;
    int32_t env; /* which environment's nodes this camera sees (ignored for GSIM_ENV_ALL nodes) */
    int32_t reserved;
} gsim_camera;

/* RasterOptions (raster.hpp:31-36). */
typedef struct gsim_raster_options {
    int32_t normalize_depth;
    int32_t reserved;
    double transmittance_cutoff;
} gsim_raster_options;

/* ProjectedSplat (raster.hpp:20-29), identical memory layout (120 bytes). */
typedef struct gsim_projected_splat {
    double pixel_center[2];
    double cov_xx, cov_xy, cov_yy;
    double inv_xx, inv_xy, inv_yy;
    double view_depth;
    double alpha_peak;
    double rgb[3];
    double radius;
    uint32_t prim_index;
    uint32_t reserved;
} gsim_projected_splat;

/* RenderTarget (image.hpp:38-45): row-major float images, rgb interleaved (W*H*3). */
typedef struct gsim_target {
    float* rgb;
    float* depth;
    float* accum_alpha;
} gsim_target;

/* Counters and per-stage device times (ms) of the last render on a context. */
typedef struct gsim_render_stats {
    uint64_t slots;        /* (camera, primitive) candidates */
    uint64_t visible;      /* records that touch at least one tile (V) */
    uint64_t pairs;        /* (tile, record) pairs (P); after gsim_gpu_trace_rays: the rays'
                              BVH candidates */
    uint64_t tiles;        /* total tiles over all cameras */
    uint64_t launches;     /* kernels launched by the last render */
    uint64_t launches_total; /* kernels launched on this context since creation */
    uint64_t consumed;     /* pair-list entries the rasterizer fetched before saturating (K) */
    uint64_t h2d_bytes;    /* host->device bytes copied by the last call */
    uint64_t d2h_bytes;    /* device->host bytes copied by the last call */
    uint32_t depth_passes; /* segmented onesweep passes over the depth keys (per camera) */
    uint32_t chunks;       /* binning chunks (runs of depth-sorted records of one camera) */
    /* per-stage device milliseconds, filled when profiling is on (gsim_gpu_set_profiling) */
    float ms_preprocess;   /* K2 projection + SH */
    float ms_depth_sort;   /* key histograms + chunk table + onesweep passes */
    float ms_binning;      /* per-chunk tile counts + column/tile/camera scans */
    float ms_scatter;      /* pair placement in final (camera, tile, depth) order */
    float ms_raster;       /* K4 */
    float ms_total;
    uint32_t groups;       /* camera groups the last batch was split into */
    uint32_t last_group_cameras; /* cameras of the last group (gsim_gpu_tile_lists sees these) */
} gsim_render_stats;

typedef struct gsim_gpu_context gsim_gpu_context;
typedef struct gsim_gpu_scene gsim_gpu_scene;

const char* gsim_gpu_version(void);

/* One context per device: a CUDA stream plus grow-only device workspaces. */
int gsim_gpu_context_create(int device, gsim_gpu_context** out);
int gsim_gpu_context_destroy(gsim_gpu_context* ctx);
/* Message of the last failure on ctx (ctx may be NULL for a failed create). */
const char* gsim_gpu_last_error(const gsim_gpu_context* ctx);
/* The context's cudaStream_t, for callers that time or order work around it. */
void* gsim_gpu_stream(gsim_gpu_context* ctx);
int gsim_gpu_synchronize(gsim_gpu_context* ctx);
int gsim_gpu_set_profiling(gsim_gpu_context* ctx, int enable);
int gsim_gpu_get_stats(gsim_gpu_context* ctx, gsim_render_stats* out);

/* Device-resident scene: the field is validated (gaussian.cpp:13-30 rules on sh_degree) and
 * copied once; renders then read it from HBM. Replaces re-reading the AoS double field on
 * every render() call. */
int gsim_gpu_scene_upload(gsim_gpu_context* ctx, const gsim_field_view* field,
                          gsim_gpu_scene** out);
int gsim_gpu_scene_destroy(gsim_gpu_scene* scene);
/* Streaming upload for fields that are produced piecewise (BASELINE config 4: a background plus
 * hundreds of environments' objects, tens of millions of primitives): scene_create allocates a
 * zeroed field of `count` primitives, scene_write fills [offset, offset + field->count) from a
 * host view of the same sh_degree. Writes wait for the context's frames in flight. */
int gsim_gpu_scene_create(gsim_gpu_context* ctx, uint64_t count, int32_t sh_degree,
                          gsim_gpu_scene** out);
int gsim_gpu_scene_write(gsim_gpu_context* ctx, gsim_gpu_scene* scene, uint64_t offset,
                         const gsim_field_view* field);
uint64_t gsim_gpu_scene_size(const gsim_gpu_scene* scene);
/* transform_primitives (gaussian.cpp:65-79) in place on the device-resident field (K1). */
int gsim_gpu_transform_primitives(gsim_gpu_context* ctx, gsim_gpu_scene* scene, uint64_t begin,
                                  uint64_t end, const gsim_rigid* transform);
/* Copies the device field's means (count*3) and rotations (count*4) back; either may be NULL. */
int gsim_gpu_scene_download(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, double* means,
                            double* rotations);
/* Copies every plane of the device field back in the reference's per-primitive layout:
 * means n*3, scales n*3, rotations n*4 (w,x,y,z), opacities n, sh n*48 (sh[c*16+k],
 * gaussian.hpp:16-19; coefficients above the field's degree are 0). Any pointer may be NULL. */
int gsim_gpu_scene_download_field(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                                  double* means, double* scales, double* rotations,
                                  double* opacities, double* sh);
int32_t gsim_gpu_scene_sh_degree(const gsim_gpu_scene* scene);

/* load_splat_ply (splat_ply.cpp:40-162) straight into a device-resident field (SURVEY.md 8f
 * row 1): the header is parsed on the host with the reference's rules and messages; the float
 * payload is streamed through pinned chunks to the device and converted by a kernel
 * (sigmoid opacity, exp scales, 1e-6 rotation renormalisation, per-primitive validation in
 * the reference's order). Status 1 when the file cannot be opened, 2 for format/validation
 * errors (format_error derives from validation_error, errors.hpp:22-24). Means, rotations and
 * SH are bit-exact with the reference loader; scale and opacity go through CUDA's double exp
 * (scale <= 1 ulp from glibc, opacity = 1 / (1 + exp(-x)) <= 2 ulp). */
int gsim_gpu_scene_load_ply(gsim_gpu_context* ctx, const char* path, gsim_gpu_scene** out);

/* project (raster.cpp:66-163): visible splats in primitive order. Writes at most
 * capacity splats to out and the visible count to *count (count may exceed capacity). */
int gsim_gpu_project(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                     uint64_t n_nodes, const gsim_camera* camera, gsim_projected_splat* out,
                     uint64_t capacity, uint64_t* count);

/* rasterize (raster.cpp:165-254) of host splats into a host target. */
int gsim_gpu_rasterize(gsim_gpu_context* ctx, const gsim_projected_splat* splats, uint64_t n,
                       const gsim_camera* camera, const gsim_raster_options* options,
                       gsim_target* out);

/* render (raster.cpp:256-265): one host target per camera; returns after the copies land. */
int gsim_gpu_render(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                    uint64_t n_nodes, const gsim_camera* cameras, uint64_t n_cameras,
                    const gsim_raster_options* options, gsim_target* outs);

/* render into device memory, asynchronous on the context stream. device_out holds, per
 * camera in order, [rgb W*H*3 | depth W*H | accum_alpha W*H] floats (20 B per pixel);
 * NULL renders into an internal buffer (see gsim_gpu_device_output). */
int gsim_gpu_render_device(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                           const gsim_node* nodes, uint64_t n_nodes, const gsim_camera* cameras,
                           uint64_t n_cameras, const gsim_raster_options* options,
                           float* device_out);
/* Device pointer of the internal output buffer of the last render_device(NULL) call. */
float* gsim_gpu_device_output(gsim_gpu_context* ctx);

/* Peer memory for BASELINE config 4's fused frame gather: rank 0 allocates the gathered output
 * and exports it (CUDA IPC handle, 64 bytes); every other rank of the node opens the handle and
 * passes pointers into it as gsim_gpu_render_device's device_out, so the compositing kernel's
 * epilogue stores its pixels straight into rank 0's HBM over NVLink (no separate collective).
 * Host-side plumbing only (cudaMalloc / cudaIpcGetMemHandle / cudaIpcOpenMemHandle). */
int gsim_gpu_ipc_alloc(int32_t device, uint64_t bytes, void** ptr, uint8_t handle[64]);
int gsim_gpu_ipc_free(int32_t device, void* ptr);
int gsim_gpu_ipc_open(int32_t device, const uint8_t handle[64], void** ptr);
int gsim_gpu_ipc_close(int32_t device, void* ptr);

/* Sorted tile lists of one camera of the last render/rasterize on ctx (test hook for the
 * reference's pair sort, raster.cpp:174-202): tile_begin gets tiles_x*tiles_y+1 offsets,
 * values gets the primitive index (render) or splat index (rasterize) of each pair in
 * sorted order. *count = number of pairs of that camera (values may be NULL to query). */
int gsim_gpu_tile_lists(gsim_gpu_context* ctx, uint32_t camera, uint32_t* tile_begin,
                        uint32_t* values, uint64_t capacity, uint64_t* count);

/* ---- Output encoding: the byte images the reference's writers produce ----
 * image_io.cpp:75-86  write_png_rgb8  -> GSIM_ENCODE_RGB8    interleaved RGB u8, rows top-down,
 *                     value quantize8(srgb ? linear_to_srgb(v) : clamp(v, 0, 1)) (:19-22, :43-45)
 * image_io.cpp:88-97  write_png_gray8 -> GSIM_ENCODE_ALPHA8  accum_alpha as u8, quantize8(clamp)
 * image_io.cpp:99-111 write_png_gray16-> GSIM_ENCODE_DEPTH16 depth as big-endian u16 of
 *                     clamp(lround(depth * depth_scale), 0, 65535)  (scale 1000: metres -> mm)
 * image_io.cpp:166-178 write_pfm      -> GSIM_ENCODE_DEPTH_PFM f32 depth rows bottom-up (the PFM
 *                     body; the "Pf\n%d %d\n-1.0\n" header is the caller's)
 * The per-camera block is the enabled parts in that order (RGB8, ALPHA8, DEPTH16, DEPTH_PFM),
 * packed; cameras follow each other. The bytes are those the reference hands to libpng / fwrite
 * for the same float images, bit for bit (tools/gsim.cpp:57-66 is the caller being replaced). */
#define GSIM_ENCODE_RGB8 1u
#define GSIM_ENCODE_ALPHA8 2u
#define GSIM_ENCODE_DEPTH16 4u
#define GSIM_ENCODE_DEPTH_PFM 8u

typedef struct gsim_encode_options {
    uint32_t flags;      /* GSIM_ENCODE_* bits */
    int32_t srgb;        /* write_png_rgb8's srgb_encode (tools/gsim.cpp:60 passes true) */
    double depth_scale;  /* write_png_gray16's scale (tools/gsim.cpp:64 passes 1000.0) */
} gsim_encode_options;

/* Encoded bytes of one width x height camera under `flags` (0 for unknown bits). */
uint64_t gsim_gpu_encoded_bytes(uint32_t flags, int32_t width, int32_t height);

/* The 256 sRGB code thresholds the kernels use: thresholds[k] is the smallest float v with
 * quantize8(linear_to_srgb(v)) >= k (thresholds[0] = -inf). Built on the host from the
 * reference's transfer function; needs no GPU (test hook). */
void gsim_gpu_srgb_thresholds(float* thresholds);

/* hash_target (hash.hpp:36-41): FNV-1a 64 over each image's (width, height) int32 pair and raw
 * float bytes, rgb then depth then accum_alpha, chained from `seed` (the reference bench's
 * first-frame image hash, bench.cpp:121-137, starts at 1469598103934665603). Host-only. */
uint64_t gsim_gpu_hash_target(int32_t width, int32_t height, const float* rgb, const float* depth,
                              const float* accum_alpha, uint64_t seed);

/* Encode one host RenderTarget (rgb H*W*3, depth H*W, accum_alpha H*W floats) into `out`
 * (host, gsim_gpu_encoded_bytes(flags, width, height) bytes). Unused planes may be NULL. */
int gsim_gpu_encode_host(gsim_gpu_context* ctx, int32_t width, int32_t height, const float* rgb,
                         const float* depth, const float* accum_alpha,
                         const gsim_encode_options* options, uint8_t* out);

/* Encode render_device output (device, per camera [rgb|depth|alpha] f32) of `cameras` into
 * `out` (device pointer if out_is_device, else host; synchronous for host). */
int gsim_gpu_encode(gsim_gpu_context* ctx, const float* device_targets, const gsim_camera* cameras,
                    uint64_t n_cameras, const gsim_encode_options* options, uint8_t* out,
                    int32_t out_is_device);

/* render + encode fused in the compositing kernel's epilogue: the float images never reach
 * HBM and only the encoded bytes cross to the host (6-11 B per pixel instead of 20).
 * out_is_device selects a device (asynchronous, like render_device) or host (synchronous)
 * destination. */
int gsim_gpu_render_encoded(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                            const gsim_node* nodes, uint64_t n_nodes, const gsim_camera* cameras,
                            uint64_t n_cameras, const gsim_raster_options* raster_options,
                            const gsim_encode_options* options, uint8_t* out,
                            int32_t out_is_device);

/* ---- Pose playback on the device ---------------------------------------
 * Replaces PoseStream (pose_stream.hpp:22-49; append pose_stream.cpp:31-40, sample :117-136)
 * and Scene::step_to (scene.cpp:176-190) for batches of nodes: the tracks live in HBM and the
 * node poses of a frame are sampled by a kernel straight into the frame's pose table. */
typedef struct gsim_gpu_tracks gsim_gpu_tracks;

/* Upload n_tracks tracks. Records of track k are track_begin[k] .. track_begin[k+1]-1 of the
 * arrays times[R], translations[R*3], rotations[R*4] (w, x, y, z). PoseStream::append rules:
 * validation error on non-finite values or times that decrease within a track; rotations are
 * normalised on upload. */
int gsim_gpu_tracks_upload(gsim_gpu_context* ctx, const double* times, const double* translations,
                           const double* rotations, const uint64_t* track_begin, uint64_t n_tracks,
                           gsim_gpu_tracks** out);
int gsim_gpu_tracks_destroy(gsim_gpu_tracks* tracks);
uint64_t gsim_gpu_tracks_count(const gsim_gpu_tracks* tracks);

/* PoseStream::sample for n queries (track[i], time[i], initial[i]) -> out[i] (host arrays). */
int gsim_gpu_tracks_sample(gsim_gpu_context* ctx, const gsim_gpu_tracks* tracks,
                           const uint32_t* track, const double* time, const gsim_rigid* initial,
                           uint64_t n, gsim_rigid* out);

/* render at time t: nodes with node_track[k] >= 0 take track node_track[k] sampled at t (their
 * pose in `nodes` is the initial pose, scene.cpp:186-188), the rest keep their pose. A
 * background node driven by a track is a validation error (scene.cpp:180-184). Output as
 * gsim_gpu_render (outs != NULL, synchronous, host targets) or gsim_gpu_render_device
 * (outs == NULL: asynchronous into device_out, or the internal buffer when it is NULL). */
int gsim_gpu_render_at(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                       const gsim_gpu_tracks* tracks, double time, const gsim_node* nodes,
                       const int64_t* node_track, uint64_t n_nodes, const gsim_camera* cameras,
                       uint64_t n_cameras, const gsim_raster_options* options, float* device_out,
                       gsim_target* outs);


/* ---- GS -> TSDF: the renderer's second caller -------------------------
 * transfer.cpp:27-34    field_bounds: AABB of every primitive's 3-sigma box under the identity
 *                       pose (pose_primitive, trace.cpp:14-36)
 * transfer.cpp:81-124   render_depth_ring: n_views azimuths x 3 elevations (-30, 0, +30 deg)
 *                       looking at the box centre; alpha-normalised depth, 0 where accumulated
 *                       alpha < 0.5
 * transfer.cpp:126-141  TsdfVolume::create (validation), transfer.hpp:40-62 layout
 * transfer.cpp:143-172  tsdf_fuse: projective weight-1 running average per voxel
 * transfer.cpp:174-201  gaussians_to_mesh up to the fused volume (20 azimuths at 256 x 256,
 *                       voxel grid over the padded box); marching cubes and decimation
 *                       (extract_mesh, decimate) stay with the caller.
 * Volumes live in DEVICE memory: tsdf and weights point at voxel_count doubles each, x fastest
 * (index = (z * dims[1] + y) * dims[0] + x, transfer.hpp:50-52). */
typedef struct gsim_tsdf_volume {
    double origin[3];
    double voxel_size;
    int32_t dims[3];
    int32_t reserved;
    double truncation;
    double* tsdf;    /* device, in [-1, 1], 1 where unobserved */
    double* weights; /* device, >= 0 */
} gsim_tsdf_volume;

#define GSIM_RING_ELEVATIONS 3

/* field_bounds of a device scene (lo = +inf, hi = -inf for an empty scene). */
int gsim_gpu_scene_bounds(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, double lo[3],
                          double hi[3]);

/* The 3 * n_views cameras of render_depth_ring for a field with bounds (lo, hi), elevation-
 * major as the reference orders its views. Host only (no GPU). Validation as the reference:
 * n_views < 8, radius not > 0, or a degenerate box. */
int gsim_gpu_depth_ring_cameras(const double lo[3], const double hi[3], int32_t n_views,
                                double radius, int32_t resolution, gsim_camera* cameras);

/* render_depth_ring of a device scene: depth gets 3 * n_views images of resolution^2 floats
 * (device if depth_is_device, else host; synchronous for host); cameras (host, 3 * n_views,
 * may be NULL) gets the views' cameras. Empty scene -> validation error. */
int gsim_gpu_render_depth_ring(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                               int32_t n_views, double radius, int32_t resolution,
                               gsim_camera* cameras, float* depth, int32_t depth_is_device);

/* TsdfVolume::create validation; fills the geometry of *volume (pointers untouched). Host. */
int gsim_gpu_tsdf_create(const double origin[3], double voxel_size, const int32_t dims[3],
                         double truncation, gsim_tsdf_volume* volume);
/* tsdf = 1, weights = 0 over the volume's device buffers. */
int gsim_gpu_tsdf_reset(gsim_gpu_context* ctx, const gsim_tsdf_volume* volume);

/* tsdf_fuse of n_views depth images in order (view k: cameras[k], cameras[k].width *
 * cameras[k].height floats, packed one after another; device if depth_is_device). Equivalent to
 * n_views reference tsdf_fuse calls; the volume is read and written once. */
int gsim_gpu_tsdf_fuse(gsim_gpu_context* ctx, const gsim_tsdf_volume* volume,
                       const gsim_camera* cameras, uint64_t n_views, const float* depth,
                       int32_t depth_is_device);

/* Device grids for a volume's dims (cudaMalloc'd by the library; free with tsdf_free), and
 * host <-> device copies of both grids (synchronous; NULL skips a grid). */
int gsim_gpu_tsdf_alloc(gsim_gpu_context* ctx, gsim_tsdf_volume* volume);
int gsim_gpu_tsdf_free(gsim_tsdf_volume* volume);
int gsim_gpu_tsdf_download(gsim_gpu_context* ctx, const gsim_tsdf_volume* volume, double* tsdf,
                           double* weights);
int gsim_gpu_tsdf_upload(gsim_gpu_context* ctx, const gsim_tsdf_volume* volume, const double* tsdf,
                         const double* weights);

/* gaussians_to_mesh up to the fused volume. Two calls: with volume->tsdf == NULL only the
 * geometry (origin, voxel_size, dims, truncation) is written; then, with device buffers of
 * dims[0] * dims[1] * dims[2] doubles in tsdf and weights, the volume is reset, the depth ring
 * rendered and fused. */
int gsim_gpu_gaussians_to_tsdf(gsim_gpu_context* ctx, const gsim_gpu_scene* scene,
                               double voxel_size, gsim_tsdf_volume* volume);


/* ---- LiDAR: Gaussian ray tracing for a spinning-scan sensor -------------
 * trace.cpp:14-36   pose_primitive (inverse covariance with the 1e-7 scale floor, 3-sigma AABB)
 * trace.cpp:38-49   ray_gaussian_peak      trace.cpp:65-85  composite (front to back in (t, index)
 *                                          order, alpha clamp 0.99, skip < 1/255, cutoff 1e-4)
 * trace.cpp:88-111  GaussianBvh::build (node poses painted like PoseTable; range check)
 * trace.cpp:113-134 trace / trace_linear (the BVH only accelerates: the candidate set is every
 *                   primitive whose box the ray hits, bvh.hpp:20-36)
 * trace.cpp:136-197 validate_lidar, lidar_azimuth_count, scan (channel-major, azimuth ascending,
 *                   misses omitted; points in the sensor frame). */
typedef struct gsim_lidar {
    const double* channels; /* elevation angles, radians */
    uint64_t n_channels;
    double azimuth_step;    /* radians; must divide 2*pi into an integer ray count */
    double max_range;       /* metres */
    gsim_rigid pose;        /* sensor -> world */
    double alpha_threshold; /* accumulated alpha declaring a surface, (0, 1] */
    int32_t env;            /* environment whose nodes the sensor sees (as gsim_camera.env) */
    int32_t reserved;
} gsim_lidar;

/* GaussianBvh::build(field, nodes).scan(lidar). points: 3 * capacity doubles (x, y, z in the
 * sensor frame), ring: capacity, azimuth: capacity (radians); *count = returns. The arrays are
 * written when *count <= capacity (call with capacity 0 to size them). */
int gsim_gpu_lidar_scan(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                        uint64_t n_nodes, const gsim_lidar* lidar, double* points, uint32_t* ring,
                        double* azimuth, uint64_t capacity, uint64_t* count);

/* GaussianBvh::trace for n arbitrary rays (origin, unit direction, t_max per ray; host arrays):
 * hit, depth (renormalised by accumulated alpha) and accumulated alpha per ray. Every primitive
 * is a candidate of every ray here (trace_linear's scan); the LiDAR scan bins them instead. */
int gsim_gpu_trace_rays(gsim_gpu_context* ctx, const gsim_gpu_scene* scene, const gsim_node* nodes,
                        uint64_t n_nodes, const double* origins, const double* directions,
                        const double* t_max, uint64_t n_rays, double alpha_threshold,
                        uint8_t* hit, double* depth, double* accum_alpha);

#ifdef __cplusplus
}
#endif

#endif /* GSIM_GPU_H */
