// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference library. TEST INFRASTRUCTURE.
//
// oracle/Makefile compiles this file together with the reference's own sources, where they
// lie under /root/reference/proj (core/src/{raster,reference_raster,sh,gaussian,parallel,
// log}.cpp and tests/support/test_oracles.cpp), into oracle/_ref/libgsim_ref.so. No reference
// source is copied into this repository. The shim only converts the C structs of
// include/gsim_gpu.h to the reference's C++ types and calls:
//   gsim::project / rasterize / render           raster.hpp:54-67
//   gsim::reference_rasterize                    reference_raster.hpp:14-16
//   gsim::transform_primitives                   gaussian.hpp:76-77
//   gsim::CameraModel::look_at                   camera.hpp:31-32
//   gsim::set_thread_count                       parallel.hpp:13
//   oracle::random_field                         tests/support/test_oracles.hpp:34-35
//   gsim::write_png_rgb8 / gray8 / gray16 / write_pfm / linear_to_srgb   image_io.hpp:12-33
//     (image_io.cpp compiled against oracle/png_capture, which records the row bytes handed
//     to libpng instead of compressing them)
//   gsim::PoseStream::append / sample, gsim::slerp          pose_stream.hpp:28-45, math.hpp:196
//   gsim::load_splat_ply / save_splat_ply                   splat_ply.hpp:20-24
//   gsim::render_depth_ring / TsdfVolume::create / tsdf_fuse / gaussians_to_mesh
//                                                           transfer.hpp:33-90
//   gsim::GaussianBvh::build / trace / trace_linear / scan  trace.hpp:66-82
// Used by tests/test_oracle_pin.py (pin the C restatement), tests/golden/make_golden.py and
// bench.py --impl reference (the reference's CPU renderer timed on the host cores).
#include <cstring>
#include <limits>
#include <exception>
#include <string>
#include <vector>

#include "gsim/errors.hpp"
#include "gsim/gaussian.hpp"
#include "gsim/image_io.hpp"
#include "gsim/pose_stream.hpp"
#include "gsim/splat_ply.hpp"
#include "gsim/trace.hpp"
#include "gsim/transfer.hpp"
#include "png.h"
#include "gsim/parallel.hpp"
#include "gsim/raster.hpp"
#include "gsim/reference_raster.hpp"
#include "test_oracles.hpp"

#include "../include/gsim_gpu.h"

using namespace gsim;

namespace {

thread_local std::string g_error;

Quat to_quat(const double* q) { return Quat(q[0], q[1], q[2], q[3]); }
Vec3 to_vec(const double* v) { return Vec3(v[0], v[1], v[2]); }
RigidTransform to_rigid(const gsim_rigid& r) {
    return RigidTransform(to_quat(r.rotation), to_vec(r.translation));
}
void from_rigid(const RigidTransform& t, gsim_rigid* out) {
    out->rotation[0] = t.rotation.w;
    out->rotation[1] = t.rotation.x;
    out->rotation[2] = t.rotation.y;
    out->rotation[3] = t.rotation.z;
    out->translation[0] = t.translation.x;
    out->translation[1] = t.translation.y;
    out->translation[2] = t.translation.z;
}

GaussianField to_field(const gsim_field_view* v) {
    GaussianField f;
    f.sh_degree = v->sh_degree;
    f.primitives.resize(v->count);
    for (std::size_t i = 0; i < v->count; ++i) {
        auto& p = f.primitives[i];
        p.mean = to_vec(v->means + i * v->means_stride);
        p.scale = to_vec(v->scales + i * v->scales_stride);
        p.rotation = to_quat(v->rotations + i * v->rotations_stride);
        p.opacity = v->opacities[i * v->opacities_stride];
        const double* sh = v->sh + i * v->sh_stride;
        for (int k = 0; k < 48; ++k) p.sh[k] = sh[k];
    }
    return f;
}

std::vector<SceneNode> to_nodes(const gsim_node* nodes, std::uint64_t n) {
    std::vector<SceneNode> out(n);
    for (std::uint64_t k = 0; k < n; ++k) {
        out[k].id = "node" + std::to_string(k);
        out[k].kind = nodes[k].kind == GSIM_NODE_BACKGROUND ? NodeKind::background
                                                            : NodeKind::interactive;
        out[k].pose = to_rigid(nodes[k].pose);
        out[k].range = {nodes[k].begin, nodes[k].end};
    }
    return out;
}

CameraModel to_camera(const gsim_camera& c) {
    CameraModel cam;
    cam.id = "cam";
    cam.fx = c.fx;
    cam.fy = c.fy;
    cam.cx = c.cx;
    cam.cy = c.cy;
    cam.width = c.width;
    cam.height = c.height;
    cam.pose = to_rigid(c.pose);
    cam.near = c.near_plane;
    cam.far = c.far_plane;
    return cam;
}

void from_splat(const ProjectedSplat& s, gsim_projected_splat* o) {
    std::memset(o, 0, sizeof(*o));
    o->pixel_center[0] = s.pixel_center.x;
    o->pixel_center[1] = s.pixel_center.y;
    o->cov_xx = s.cov_xx;
    o->cov_xy = s.cov_xy;
    o->cov_yy = s.cov_yy;
    o->inv_xx = s.inv_xx;
    o->inv_xy = s.inv_xy;
    o->inv_yy = s.inv_yy;
    o->view_depth = s.view_depth;
    o->alpha_peak = s.alpha_peak;
    o->rgb[0] = s.rgb.x;
    o->rgb[1] = s.rgb.y;
    o->rgb[2] = s.rgb.z;
    o->radius = s.radius;
    o->prim_index = s.prim_index;
}

void from_camera(const CameraModel& c, gsim_camera* out) {
    std::memset(out, 0, sizeof(*out));
    out->fx = c.fx;
    out->fy = c.fy;
    out->cx = c.cx;
    out->cy = c.cy;
    out->width = c.width;
    out->height = c.height;
    from_rigid(c.pose, &out->pose);
    out->near_plane = c.near;
    out->far_plane = c.far;
}

void copy_volume_out(const TsdfVolume& v, gsim_tsdf_volume* out) {
    for (int k = 0; k < 3; ++k) out->dims[k] = v.dims[k];
    out->origin[0] = v.origin.x;
    out->origin[1] = v.origin.y;
    out->origin[2] = v.origin.z;
    out->voxel_size = v.voxel_size;
    out->truncation = v.truncation;
    if (out->tsdf) std::memcpy(out->tsdf, v.tsdf.data(), v.tsdf.size() * sizeof(double));
    if (out->weights) std::memcpy(out->weights, v.weights.data(), v.weights.size() * sizeof(double));
}

ProjectedSplat to_splat(const gsim_projected_splat& o) {
    ProjectedSplat s;
    s.pixel_center = {o.pixel_center[0], o.pixel_center[1]};
    s.cov_xx = o.cov_xx;
    s.cov_xy = o.cov_xy;
    s.cov_yy = o.cov_yy;
    s.inv_xx = o.inv_xx;
    s.inv_xy = o.inv_xy;
    s.inv_yy = o.inv_yy;
    s.view_depth = o.view_depth;
    s.alpha_peak = o.alpha_peak;
    s.rgb = Vec3(o.rgb[0], o.rgb[1], o.rgb[2]);
    s.radius = o.radius;
    s.prim_index = o.prim_index;
    return s;
}

RasterOptions to_options(const gsim_raster_options* o) {
    RasterOptions r;
    if (o) {
        r.normalize_depth = o->normalize_depth != 0;
        r.transmittance_cutoff = o->transmittance_cutoff;
    }
    return r;
}

void copy_target(const RenderTarget& t, float* rgb, float* depth, float* alpha) {
    std::memcpy(rgb, t.rgb.data.data(), t.rgb.data.size() * sizeof(float));
    std::memcpy(depth, t.depth.data.data(), t.depth.data.size() * sizeof(float));
    std::memcpy(alpha, t.accum_alpha.data.data(), t.accum_alpha.data.size() * sizeof(float));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return GSIM_OK;
    } catch (const validation_error& e) {
        g_error = e.what();
        return GSIM_ERR_VALIDATION;
    } catch (const std::exception& e) {
        g_error = e.what();
        return GSIM_ERR_IO;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_error.c_str(); }

void ref_set_threads(int threads) { set_thread_count(threads); }
int ref_thread_count(void) { return thread_count(); }

// A reference GaussianField built once (outside any timed region).
void* ref_field_create(const gsim_field_view* view) { return new GaussianField(to_field(view)); }
void ref_field_destroy(void* field) { delete static_cast<GaussianField*>(field); }

int ref_project(void* field, const gsim_node* nodes, std::uint64_t n_nodes,
                const gsim_camera* camera, gsim_projected_splat* out, std::uint64_t capacity,
                std::uint64_t* count) {
    return guarded([&] {
        const auto splats = project(*static_cast<GaussianField*>(field), to_nodes(nodes, n_nodes),
                                    to_camera(*camera));
        *count = splats.size();
        for (std::size_t i = 0; i < splats.size() && i < capacity; ++i) from_splat(splats[i], &out[i]);
    });
}

int ref_rasterize(const gsim_projected_splat* splats, std::uint64_t n, const gsim_camera* camera,
                  const gsim_raster_options* options, float* rgb, float* depth, float* alpha) {
    return guarded([&] {
        std::vector<ProjectedSplat> v(n);
        for (std::uint64_t i = 0; i < n; ++i) v[i] = to_splat(splats[i]);
        copy_target(rasterize(v, to_camera(*camera), to_options(options)), rgb, depth, alpha);
    });
}

int ref_reference_rasterize(const gsim_projected_splat* splats, std::uint64_t n,
                            const gsim_camera* camera, const gsim_raster_options* options,
                            float* rgb, float* depth, float* alpha) {
    return guarded([&] {
        std::vector<ProjectedSplat> v(n);
        for (std::uint64_t i = 0; i < n; ++i) v[i] = to_splat(splats[i]);
        copy_target(reference_rasterize(v, to_camera(*camera), to_options(options)), rgb, depth,
                    alpha);
    });
}

int ref_render(void* field, const gsim_node* nodes, std::uint64_t n_nodes,
               const gsim_camera* cameras, std::uint64_t n_cameras,
               const gsim_raster_options* options, gsim_target* outs) {
    return guarded([&] {
        std::vector<CameraModel> cams;
        for (std::uint64_t c = 0; c < n_cameras; ++c) cams.push_back(to_camera(cameras[c]));
        const auto targets = render(*static_cast<GaussianField*>(field), to_nodes(nodes, n_nodes),
                                    cams, to_options(options));
        for (std::uint64_t c = 0; c < n_cameras; ++c)
            copy_target(targets[c], outs[c].rgb, outs[c].depth, outs[c].accum_alpha);
    });
}

// transform_primitives on SoA means (stride 3) / rotations (stride 4).
int ref_transform_primitives(double* means, double* rotations, std::uint64_t count,
                             std::uint64_t begin, std::uint64_t end, const gsim_rigid* t) {
    GaussianField f;
    f.primitives.resize(count);
    for (std::uint64_t i = 0; i < count; ++i) {
        f.primitives[i].mean = to_vec(means + 3 * i);
        f.primitives[i].rotation = to_quat(rotations + 4 * i);
    }
    const int st = guarded([&] { transform_primitives(f, {begin, end}, to_rigid(*t)); });
    if (st != GSIM_OK) return st;
    for (std::uint64_t i = 0; i < count; ++i) {
        const auto& p = f.primitives[i];
        means[3 * i + 0] = p.mean.x;
        means[3 * i + 1] = p.mean.y;
        means[3 * i + 2] = p.mean.z;
        rotations[4 * i + 0] = p.rotation.w;
        rotations[4 * i + 1] = p.rotation.x;
        rotations[4 * i + 2] = p.rotation.y;
        rotations[4 * i + 3] = p.rotation.z;
    }
    return GSIM_OK;
}

void ref_look_at(const double* eye, const double* target, double fx, double fy, int width,
                 int height, const double* up, gsim_camera* out) {
    const CameraModel c = CameraModel::look_at(to_vec(eye), to_vec(target), fx, fy, width, height,
                                               to_vec(up));
    std::memset(out, 0, sizeof(*out));
    out->fx = c.fx;
    out->fy = c.fy;
    out->cx = c.cx;
    out->cy = c.cy;
    out->width = c.width;
    out->height = c.height;
    from_rigid(c.pose, &out->pose);
    out->near_plane = c.near;
    out->far_plane = c.far;
}

void ref_rigid_compose(const gsim_rigid* a, const gsim_rigid* b, gsim_rigid* out) {
    from_rigid(to_rigid(*a) * to_rigid(*b), out);
}

void ref_random_field(std::uint64_t seed, std::uint64_t count, double box_extent,
                      double scale_lo, double scale_hi, int sh_degree, double* means,
                      double* scales, double* rotations, double* opacities, double* sh) {
    const GaussianField f =
        oracle::random_field(seed, count, box_extent, scale_lo, scale_hi, sh_degree);
    for (std::uint64_t i = 0; i < count; ++i) {
        const auto& p = f.primitives[i];
        std::memcpy(means + 3 * i, &p.mean.x, 3 * sizeof(double));
        std::memcpy(scales + 3 * i, &p.scale.x, 3 * sizeof(double));
        rotations[4 * i + 0] = p.rotation.w;
        rotations[4 * i + 1] = p.rotation.x;
        rotations[4 * i + 2] = p.rotation.y;
        rotations[4 * i + 3] = p.rotation.z;
        opacities[i] = p.opacity;
        std::memcpy(sh + 48 * i, p.sh.data(), 48 * sizeof(double));
    }
}

// ---- image_io.cpp writers: the bytes each hands to libpng (captured), and the PFM file ----
namespace {
int copy_capture(std::uint8_t* out, std::uint64_t capacity, std::uint64_t* size) {
    std::size_t n = 0;
    const unsigned char* b = png_capture_last(nullptr, nullptr, nullptr, nullptr, &n);
    if (size) *size = n;
    if (n > capacity) {
        g_error = "capture larger than the output buffer";
        return GSIM_ERR_VALIDATION;
    }
    std::memcpy(out, b, n);
    return GSIM_OK;
}
}  // namespace

double ref_linear_to_srgb(double v) { return linear_to_srgb(v); }

int ref_png_rgb8(const float* rgb, int width, int height, int srgb, std::uint8_t* out,
                 std::uint64_t capacity, std::uint64_t* size) {
    const int rc = guarded([&] {
        Image3 img(width, height);
        std::memcpy(img.data.data(), rgb, img.data.size() * sizeof(float));
        write_png_rgb8("/dev/null", img, srgb != 0);
    });
    return rc != GSIM_OK ? rc : copy_capture(out, capacity, size);
}

int ref_png_gray8(const float* v, int width, int height, std::uint8_t* out, std::uint64_t capacity,
                  std::uint64_t* size) {
    const int rc = guarded([&] {
        Image1 img(width, height);
        std::memcpy(img.data.data(), v, img.data.size() * sizeof(float));
        write_png_gray8("/dev/null", img);
    });
    return rc != GSIM_OK ? rc : copy_capture(out, capacity, size);
}

int ref_png_gray16(const float* v, int width, int height, double scale, std::uint8_t* out,
                   std::uint64_t capacity, std::uint64_t* size) {
    const int rc = guarded([&] {
        Image1 img(width, height);
        std::memcpy(img.data.data(), v, img.data.size() * sizeof(float));
        write_png_gray16("/dev/null", img, scale);
    });
    return rc != GSIM_OK ? rc : copy_capture(out, capacity, size);
}

int ref_write_pfm(const char* path, const float* v, int width, int height) {
    return guarded([&] {
        Image1 img(width, height);
        std::memcpy(img.data.data(), v, img.data.size() * sizeof(float));
        write_pfm(path, img);
    });
}

// ---- pose playback: one node's track through PoseStream (pose_stream.cpp:31-40, 117-136) ----
// Records are (t, p[3], q[4] as w,x,y,z); queries sample the track at times ts[k] with the
// given initial pose. Returns validation errors for non-finite or decreasing records.
int ref_pose_sample(const double* rec_t, const double* rec_p, const double* rec_q,
                    std::uint64_t n_rec, const gsim_rigid* initial, const double* ts,
                    std::uint64_t n_t, gsim_rigid* out) {
    return guarded([&] {
        PoseStream stream;
        for (std::uint64_t i = 0; i < n_rec; ++i) {
            PoseRecord r;
            r.t = rec_t[i];
            r.node = "node";
            r.pose = RigidTransform(to_quat(rec_q + 4 * i), to_vec(rec_p + 3 * i));
            stream.append(r);
        }
        const RigidTransform init = to_rigid(*initial);
        for (std::uint64_t k = 0; k < n_t; ++k) from_rigid(stream.sample("node", ts[k], init), &out[k]);
    });
}

void ref_slerp(const double* a, const double* b, double t, double* out) {
    const Quat q = slerp(to_quat(a), to_quat(b), t);
    out[0] = q.w;
    out[1] = q.x;
    out[2] = q.y;
    out[3] = q.z;
}

// ---- splat PLY ------------------------------------------------------------------------------
// Two-call load: the field is (re)loaded each call; arrays are written when count <= capacity.
int ref_load_splat_ply(const char* path, std::uint64_t capacity, std::uint64_t* count, int* degree,
                       double* means, double* scales, double* rotations, double* opacities,
                       double* sh) {
    return guarded([&] {
        const GaussianField f = load_splat_ply(path);
        *count = f.size();
        *degree = f.sh_degree;
        if (f.size() > capacity) return;
        for (std::size_t i = 0; i < f.size(); ++i) {
            const auto& p = f.primitives[i];
            std::memcpy(means + 3 * i, &p.mean.x, 3 * sizeof(double));
            std::memcpy(scales + 3 * i, &p.scale.x, 3 * sizeof(double));
            rotations[4 * i + 0] = p.rotation.w;
            rotations[4 * i + 1] = p.rotation.x;
            rotations[4 * i + 2] = p.rotation.y;
            rotations[4 * i + 3] = p.rotation.z;
            opacities[i] = p.opacity;
            std::memcpy(sh + 48 * i, p.sh.data(), 48 * sizeof(double));
        }
    });
}

int ref_save_splat_ply(const char* path, const gsim_field_view* view) {
    return guarded([&] { save_splat_ply(to_field(view), path); });
}

// ---- GS -> TSDF (transfer.cpp) ---------------------------------------------------------------
int ref_render_depth_ring(void* field, int n_views, double radius, int resolution,
                          gsim_camera* cameras, float* depth) {
    return guarded([&] {
        const auto views = render_depth_ring(*static_cast<GaussianField*>(field), n_views, radius,
                                             resolution);
        const std::size_t npx = static_cast<std::size_t>(resolution) * resolution;
        for (std::size_t v = 0; v < views.size(); ++v) {
            from_camera(views[v].camera, &cameras[v]);
            std::memcpy(depth + v * npx, views[v].depth.data.data(), npx * sizeof(float));
        }
    });
}

// TsdfVolume::create with the given geometry, the host tsdf / weights copied in, then one
// tsdf_fuse; the updated grids are copied back.
int ref_tsdf_fuse(gsim_tsdf_volume* vol, const gsim_camera* camera, const float* depth, int width,
                  int height) {
    return guarded([&] {
        TsdfVolume v = TsdfVolume::create(to_vec(vol->origin), vol->voxel_size,
                                          {vol->dims[0], vol->dims[1], vol->dims[2]},
                                          vol->truncation);
        std::memcpy(v.tsdf.data(), vol->tsdf, v.tsdf.size() * sizeof(double));
        std::memcpy(v.weights.data(), vol->weights, v.weights.size() * sizeof(double));
        Image1 img(width, height);
        std::memcpy(img.data.data(), depth, img.data.size() * sizeof(float));
        tsdf_fuse(v, to_camera(*camera), img);
        copy_volume_out(v, vol);
    });
}

int ref_tsdf_create(const double* origin, double voxel_size, const int32_t* dims,
                    double truncation, gsim_tsdf_volume* vol) {
    return guarded([&] {
        copy_volume_out(TsdfVolume::create(to_vec(origin), voxel_size, {dims[0], dims[1], dims[2]},
                                           truncation),
                        vol);
    });
}

// gaussians_to_mesh(field, voxel_size, no decimation, &volume): the fused volume it builds.
int ref_gaussians_to_tsdf(void* field, double voxel_size, gsim_tsdf_volume* vol) {
    return guarded([&] {
        TsdfVolume v;
        gaussians_to_mesh(*static_cast<GaussianField*>(field), voxel_size,
                          std::numeric_limits<std::size_t>::max(), &v);
        copy_volume_out(v, vol);
    });
}

// ---- LiDAR (trace.cpp) --------------------------------------------------------------------------
// GaussianBvh::build + trace (BVH) for every ray; `linear` selects trace_linear instead.
int ref_trace_rays(void* field, const gsim_node* nodes, std::uint64_t n_nodes, const double* origins,
                   const double* dirs, const double* t_max, std::uint64_t n, double alpha_threshold,
                   int linear, std::uint8_t* hit, double* depth, double* acc) {
    return guarded([&] {
        const GaussianBvh bvh = GaussianBvh::build(*static_cast<GaussianField*>(field),
                                                   to_nodes(nodes, n_nodes));
        for (std::uint64_t r = 0; r < n; ++r) {
            Ray ray;
            ray.origin = to_vec(origins + 3 * r);
            ray.direction = to_vec(dirs + 3 * r);
            ray.t_max = t_max[r];
            const TraceResult t = linear ? bvh.trace_linear(ray, alpha_threshold)
                                         : bvh.trace(ray, alpha_threshold);
            hit[r] = t.hit ? 1 : 0;
            depth[r] = t.depth;
            acc[r] = t.accum_alpha;
        }
    });
}

int ref_lidar_scan(void* field, const gsim_node* nodes, std::uint64_t n_nodes, const gsim_lidar* l,
                   double* points, std::uint32_t* ring, double* azimuth, std::uint64_t capacity,
                   std::uint64_t* count) {
    return guarded([&] {
        const GaussianBvh bvh = GaussianBvh::build(*static_cast<GaussianField*>(field),
                                                   to_nodes(nodes, n_nodes));
        LidarModel m;
        m.id = "lidar";
        m.channels.assign(l->channels, l->channels + l->n_channels);
        m.azimuth_step = l->azimuth_step;
        m.max_range = l->max_range;
        m.pose = to_rigid(l->pose);
        m.alpha_threshold = l->alpha_threshold;
        const PointCloud c = bvh.scan(m);
        *count = c.size();
        if (c.size() > capacity) return;
        for (std::size_t k = 0; k < c.size(); ++k) {
            points[3 * k] = c.points[k].x;
            points[3 * k + 1] = c.points[k].y;
            points[3 * k + 2] = c.points[k].z;
            ring[k] = c.ring[k];
            azimuth[k] = c.azimuth[k];
        }
    });
}

}  // extern "C"
