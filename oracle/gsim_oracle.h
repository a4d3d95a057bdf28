/*
 * gsim_oracle.h — CPU restatement of the reference render path. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library, and only as the checker (or the timed CPU baseline). The product path
 * (paper_2507_21981_b200, libgsim_gpu.so) never links or calls it.
 *
 * Restates in plain C, in double precision and in the reference's operation order:
 *   project            raster.cpp:66-163      rasterize           raster.cpp:165-254
 *   reference_rasterize reference_raster.cpp:12-67   render        raster.cpp:256-265
 *   shade_sh           sh.cpp:10-51            transform_primitives gaussian.cpp:65-79
 *   CameraModel::look_at raster.cpp:25-42     Quat::from_matrix   math.hpp:158-187
 *   oracle::random_field tests/support/test_oracles.cpp:144-168 (std::mt19937_64 and
 *       libstdc++'s uniform_real_distribution<double> restated bit-exactly)
 *   hash_target (FNV-1a)  hash.hpp:16-44
 *   encode: write_png_rgb8 / gray8 / gray16 row bytes, write_pfm body, linear_to_srgb
 *       image_io.cpp:19-22, 43-45, 75-111, 166-178
 *   pose playback: PoseStream::append / sample  pose_stream.cpp:31-40, 117-136;
 *       slerp  math.hpp:195-214
 *   load_splat_ply   splat_ply.cpp:40-162 (status only: 1 io, 2 format/validation)
 *   GS -> TSDF: field_bounds, render_depth_ring, TsdfVolume::create, tsdf_fuse,
 *       gaussians_to_mesh up to the fused volume   transfer.cpp:27-34, 81-198
 *   LiDAR: pose_primitive, ray_aabb_hit, ray_gaussian_peak, composite, trace_linear,
 *       validate_lidar, GaussianBvh::scan   trace.cpp:14-197, bvh.hpp:20-36
 *
 * Parity pin: tests/test_oracle_pin.py checks every function against the reference itself
 * (oracle/_ref/libgsim_ref.so, compiled from /root/reference sources by oracle/Makefile) and
 * against the committed golden fixtures in tests/golden/ (made by tests/golden/make_golden.py
 * from the reference).
 */
#ifndef GSIM_ORACLE_H
#define GSIM_ORACLE_H

#include <stdint.h>

#include "../include/gsim_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- math / sensors --------------------------------------------------------------------- */
void gso_shade_sh(const double* sh48, int degree, const double view_dir[3], double rgb[3]);
void gso_look_at(const double eye[3], const double target[3], double fx, double fy, int width,
                 int height, const double up[3], gsim_camera* out);
/* camera.pose.inverse().translation (camera.hpp:23) */
void gso_camera_center(const gsim_camera* cam, double out[3]);
void gso_rigid_compose(const gsim_rigid* a, const gsim_rigid* b, gsim_rigid* out); /* a*b */
void gso_rigid_inverse(const gsim_rigid* a, gsim_rigid* out);
void gso_quat_from_axis_angle(const double axis[3], double angle, double q[4]);

/* ---- the render path -------------------------------------------------------------------- */
/* Returns GSIM_OK or GSIM_ERR_VALIDATION (bad camera / node range). Nodes with env >= 0 are
 * seen only by cameras of that env (batched-env extension; env = -1 is the reference). */
int gso_project(const gsim_field_view* field, const gsim_node* nodes, uint64_t n_nodes,
                const gsim_camera* camera, gsim_projected_splat* out, uint64_t capacity,
                uint64_t* count);
int gso_rasterize(const gsim_projected_splat* splats, uint64_t n, const gsim_camera* camera,
                  const gsim_raster_options* options, float* rgb, float* depth, float* alpha);
/* The sorted (tile, depth, splat) pair list of rasterize (raster.cpp:174-202): tile_begin
 * gets tiles+1 offsets, values the splat index of each pair (NULL to query *count). */
int gso_rasterize_lists(const gsim_projected_splat* splats, uint64_t n,
                        const gsim_camera* camera, uint32_t* tile_begin, uint32_t* values,
                        uint64_t capacity, uint64_t* count);
int gso_reference_rasterize(const gsim_projected_splat* splats, uint64_t n,
                            const gsim_camera* camera, const gsim_raster_options* options,
                            float* rgb, float* depth, float* alpha);
int gso_render(const gsim_field_view* field, const gsim_node* nodes, uint64_t n_nodes,
               const gsim_camera* cameras, uint64_t n_cameras,
               const gsim_raster_options* options, gsim_target* outs);
/* In place on means (stride 3) and rotations (stride 4). */
int gso_transform_primitives(double* means, double* rotations, uint64_t count, uint64_t begin,
                             uint64_t end, const gsim_rigid* transform);

/* ---- deterministic fixtures ------------------------------------------------------------- */
typedef struct gso_mt19937_64 {
    uint64_t mt[312];
    int index;
} gso_mt19937_64;
void gso_mt_seed(gso_mt19937_64* rng, uint64_t seed);
uint64_t gso_mt_next(gso_mt19937_64* rng);
double gso_uniform_real(gso_mt19937_64* rng, double a, double b);
/* Arrays are SoA: means count*3, scales count*3, rotations count*4, opacities count,
 * sh count*48 (zero beyond the degree). */
void gso_random_field(uint64_t seed, uint64_t count, double box_extent, double scale_lo,
                      double scale_hi, int sh_degree, double* means, double* scales,
                      double* rotations, double* opacities, double* sh);

/* ---- output encoding (gsim_gpu.h GSIM_ENCODE_* layout) -------------------------------- */
double gso_linear_to_srgb(double v);
uint64_t gso_encoded_bytes(uint32_t flags, int width, int height);
int gso_encode(uint32_t flags, int srgb, double depth_scale, int width, int height,
               const float* rgb, const float* depth, const float* alpha, uint8_t* out);

/* ---- pose playback ----------------------------------------------------------------------- */
void gso_slerp(const double a[4], const double b[4], double t, double out[4]);
/* One node's track (records appended in order: validation error on non-finite values or
 * decreasing times), sampled at n_t times with the given initial pose. */
int gso_pose_sample(const double* rec_t, const double* rec_p, const double* rec_q, uint64_t n_rec,
                    const gsim_rigid* initial, const double* ts, uint64_t n_t, gsim_rigid* out);

/* ---- splat PLY ------------------------------------------------------------------------------
 * Two-call: *count / *degree are always set on success; arrays are written when
 * count <= capacity (sh is 48 per primitive, sh[c*16+k]). */
int gso_load_splat_ply(const char* path, uint64_t capacity, uint64_t* count, int* degree,
                       double* means, double* scales, double* rotations, double* opacities,
                       double* sh);

/* ---- GS -> TSDF (transfer.cpp) -------------------------------------------
 * field_bounds (transfer.cpp:27-34 over pose_primitive, trace.cpp:14-36); the ring cameras and
 * render_depth_ring (transfer.cpp:81-124, depth: 3*n_views images of resolution^2 floats);
 * TsdfVolume::create (transfer.cpp:126-141: tsdf = 1, weights = 0 when the host buffers are
 * given); tsdf_fuse (transfer.cpp:143-172); gaussians_to_mesh up to the fused volume
 * (transfer.cpp:174-198; two-call, geometry only when volume->tsdf is NULL). Volumes are HOST
 * buffers here. */
void gso_field_bounds(const gsim_field_view* field, double lo[3], double hi[3]);
int gso_depth_ring_cameras(const double lo[3], const double hi[3], int n_views, double radius,
                           int resolution, gsim_camera* cameras);
int gso_render_depth_ring(const gsim_field_view* field, int n_views, double radius,
                          int resolution, gsim_camera* cameras, float* depth);
int gso_tsdf_create(const double origin[3], double voxel_size, const int32_t dims[3],
                    double truncation, gsim_tsdf_volume* volume);
int gso_tsdf_fuse(gsim_tsdf_volume* volume, const gsim_camera* camera, const float* depth,
                  int width, int height);
int gso_gaussians_to_tsdf(const gsim_field_view* field, double voxel_size,
                          gsim_tsdf_volume* volume);

/* ---- LiDAR (trace.cpp) ---------------------------------------------------
 * trace_linear over every primitive (pose_primitive trace.cpp:14-36, ray_aabb_hit bvh.hpp:20-36,
 * ray_gaussian_peak trace.cpp:38-49, composite trace.cpp:65-85) and GaussianBvh::scan
 * (trace.cpp:169-197, validate_lidar :136-160). Nodes with env >= 0 other than the sensor's
 * are not seen (the batched-env extension). Two-call scan like the library. */
int gso_trace_rays(const gsim_field_view* field, const gsim_node* nodes, uint64_t n_nodes,
                   const double* origins, const double* directions, const double* t_max,
                   uint64_t n_rays, double alpha_threshold, uint8_t* hit, double* depth,
                   double* accum_alpha);
int gso_lidar_scan(const gsim_field_view* field, const gsim_node* nodes, uint64_t n_nodes,
                   const gsim_lidar* lidar, double* points, uint32_t* ring, double* azimuth,
                   uint64_t capacity, uint64_t* count);

uint64_t gso_hash_bytes(const void* data, uint64_t size, uint64_t seed);
uint64_t gso_hash_target(const float* rgb, const float* depth, const float* alpha, int width,
                         int height, uint64_t seed);

#ifdef __cplusplus
}
#endif

#endif
