// gsim_gpu.hpp — C++ drop-in for the reference render API on top of the C ABI (gsim_gpu.h).
//
// Include after the reference headers are on the include path (-I<gsim>/core/include):
//
//   gsim::gpu::render(field, nodes, cameras, options)   same signature as gsim::render
//                                                       (raster.hpp:64-67)
//   gsim::gpu::project(field, nodes, camera)            gsim::project   (raster.hpp:54-56)
//   gsim::gpu::rasterize(splats, camera, options)       gsim::rasterize (raster.hpp:59-60)
//   gsim::gpu::transform_primitives(field, range, t)    gsim::transform_primitives
//                                                       (gaussian.hpp:76-77)
//   gsim::gpu::encode(target, options)                  the bytes write_png_rgb8 / gray8 /
//                                                       gray16 / write_pfm produce
//                                                       (image_io.hpp:16-33)
//   Renderer::load_ply(path)                            load_splat_ply (splat_ply.hpp:20)
//   PoseTracks + Renderer::render_at(tracks, t, ...)    PoseStream::sample + Scene::step_to
//                                                       (pose_stream.hpp:41-45, scene.cpp:176)
//   Renderer::render_encoded(...)                       render + encode fused on the GPU
//   gsim::gpu::render_depth_ring(field, n, radius, res) render_depth_ring (transfer.hpp:33-37)
//   gsim::gpu::tsdf_fuse(volume, camera, depth)         tsdf_fuse (transfer.hpp:68-71)
//   gsim::gpu::gaussians_to_tsdf(field, voxel_size)     gaussians_to_mesh's fused volume
//                                                       (transfer.hpp:82-86, transfer.cpp:174-198)
//   gsim::gpu::lidar_scan(field, nodes, lidar)          GaussianBvh::build(field, nodes).scan(lidar)
//                                                       (trace.hpp:66-82)
//   gsim::gpu::trace(field, nodes, rays, threshold)     GaussianBvh::trace per ray (trace.hpp:70-74)
//   gsim::gpu::render_all(scene, cameras, options)      Scene::render_all (scene.cpp:232-235)
//   gsim::gpu::run_bench(scene, options)                run_bench (bench.hpp:45, bench.cpp:98-160):
//                                                       the reference's timed camera-ring loop,
//                                                       rendered by the GPU
//
// Errors are rethrown as the reference's gsim::validation_error (status 2) and gsim::io_error
// (status 1). The free functions keep the field resident in HBM between calls: the upload is
// cached per host thread, keyed on (primitives.data(), size, sh_degree, the global field
// generation, a sampled content fingerprint), so a caller that passes the same field every frame
// (Scene::render_all, scene.cpp:232-235) uploads it once. A caller that edits a field in place
// calls gsim::gpu::invalidate() afterwards (the sampled fingerprint catches most edits, not all);
// gsim::gpu::transform_primitives keeps the cache valid itself. gsim::gpu::Renderer is the
// explicit resident path (upload() / ensure()).
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "gsim/bench.hpp"
#include "gsim/errors.hpp"
#include "gsim/gaussian.hpp"
#include "gsim/hash.hpp"
#include "gsim/reference_raster.hpp"
#include "gsim/pose_stream.hpp"
#include "gsim/raster.hpp"
#include "gsim/trace.hpp"
#include "gsim/transfer.hpp"
#include "gsim_gpu.h"

namespace gsim::gpu {

static_assert(sizeof(GaussianPrimitive) == 59 * sizeof(double),
              "GaussianPrimitive is read as a stride-59 double view");
static_assert(sizeof(ProjectedSplat) == sizeof(gsim_projected_splat),
              "ProjectedSplat and gsim_projected_splat share one layout");

namespace detail {

inline void check(int status, const gsim_gpu_context* ctx) {
    if (status == GSIM_OK) return;
    const std::string msg = gsim_gpu_last_error(ctx) ? gsim_gpu_last_error(ctx) : "";
    if (status == GSIM_ERR_VALIDATION) throw validation_error(msg);
    throw io_error(msg);
}

inline gsim_field_view view(const GaussianField& f) {
    gsim_field_view v{};
    v.count = f.size();
    v.sh_degree = f.sh_degree;
    if (f.empty()) return v;
    const GaussianPrimitive& p = f.primitives[0];
    v.means = &p.mean.x;
    v.scales = &p.scale.x;
    v.rotations = &p.rotation.w;
    v.opacities = &p.opacity;
    v.sh = p.sh.data();
    v.means_stride = v.scales_stride = v.rotations_stride = v.opacities_stride = v.sh_stride = 59;
    return v;
}

// Global field generation: invalidate() bumps it, every cached upload then refreshes.
inline std::atomic<uint64_t>& field_generation() {
    static std::atomic<uint64_t> g{0};
    return g;
}

// FNV-1a over the raw bytes of up to 4096 evenly spaced primitives plus the last one: a cheap
// (~2 MB read) guard against in-place edits that were not followed by invalidate().
inline uint64_t field_fingerprint(const GaussianField& f) {
    uint64_t h = 1469598103934665603ull;
    const std::size_t n = f.size();
    if (n == 0) return h;
    const std::size_t step = std::max<std::size_t>(1, n / 4096);
    auto mix = [&h](const GaussianPrimitive& p) {
        const unsigned char* b = reinterpret_cast<const unsigned char*>(&p);
        for (std::size_t k = 0; k < sizeof(GaussianPrimitive); ++k) {
            h ^= b[k];
            h *= 1099511628211ull;
        }
    };
    for (std::size_t i = 0; i < n; i += step) mix(f.primitives[i]);
    mix(f.primitives[n - 1]);
    return h;
}

struct FieldKey {
    const void* data = nullptr;
    std::size_t size = 0;
    int degree = -1;
    uint64_t generation = 0;
    uint64_t fingerprint = 0;
    bool valid = false;
    bool operator==(const FieldKey& o) const {
        return valid && o.valid && data == o.data && size == o.size && degree == o.degree &&
               generation == o.generation && fingerprint == o.fingerprint;
    }
};

inline FieldKey field_key(const GaussianField& f) {
    FieldKey k;
    k.data = f.primitives.data();
    k.size = f.size();
    k.degree = f.sh_degree;
    k.generation = field_generation().load();
    k.fingerprint = field_fingerprint(f);
    k.valid = true;
    return k;
}

inline gsim_rigid rigid(const RigidTransform& t) {
    return gsim_rigid{{t.rotation.w, t.rotation.x, t.rotation.y, t.rotation.z},
                      {t.translation.x, t.translation.y, t.translation.z}};
}

inline std::vector<gsim_node> nodes(const std::vector<SceneNode>& ns) {
    std::vector<gsim_node> out;
    out.reserve(ns.size());
    for (const auto& n : ns)
        out.push_back(gsim_node{n.range.begin, n.range.end, rigid(n.pose),
                                n.kind == NodeKind::background ? GSIM_NODE_BACKGROUND
                                                               : GSIM_NODE_INTERACTIVE,
                                GSIM_ENV_ALL});
    return out;
}

inline gsim_camera camera(const CameraModel& c) {
    return gsim_camera{c.fx, c.fy, c.cx, c.cy, c.width, c.height, rigid(c.pose), c.near, c.far, 0, 0};
}

inline gsim_raster_options options(const RasterOptions& o) {
    return gsim_raster_options{o.normalize_depth ? 1 : 0, 0, o.transmittance_cutoff};
}

inline CameraModel from_camera(const gsim_camera& c) {
    CameraModel cam;
    cam.fx = c.fx;
    cam.fy = c.fy;
    cam.cx = c.cx;
    cam.cy = c.cy;
    cam.width = c.width;
    cam.height = c.height;
    cam.pose = RigidTransform{Quat(c.pose.rotation[0], c.pose.rotation[1], c.pose.rotation[2],
                                   c.pose.rotation[3]),
                              Vec3(c.pose.translation[0], c.pose.translation[1], c.pose.translation[2])};
    cam.near = c.near_plane;
    cam.far = c.far_plane;
    return cam;
}

inline gsim_tsdf_volume volume(const TsdfVolume& v) {
    gsim_tsdf_volume c{};
    c.origin[0] = v.origin.x;
    c.origin[1] = v.origin.y;
    c.origin[2] = v.origin.z;
    c.voxel_size = v.voxel_size;
    for (int k = 0; k < 3; ++k) c.dims[k] = v.dims[k];
    c.truncation = v.truncation;
    return c;
}

// Device grids of one volume for the duration of a call.
struct DeviceVolume {
    gsim_gpu_context* ctx;
    gsim_tsdf_volume v;
    DeviceVolume(gsim_gpu_context* c, const gsim_tsdf_volume& geometry) : ctx(c), v(geometry) {
        v.tsdf = v.weights = nullptr;
        check(gsim_gpu_tsdf_alloc(ctx, &v), ctx);
    }
    ~DeviceVolume() { gsim_gpu_tsdf_free(&v); }
    DeviceVolume(const DeviceVolume&) = delete;
    DeviceVolume& operator=(const DeviceVolume&) = delete;
    void upload(const TsdfVolume& host) {
        check(gsim_gpu_tsdf_upload(ctx, &v, host.tsdf.data(), host.weights.data()), ctx);
    }
    TsdfVolume download() const {
        TsdfVolume out = TsdfVolume::create(Vec3(v.origin[0], v.origin[1], v.origin[2]), v.voxel_size,
                                            {v.dims[0], v.dims[1], v.dims[2]}, v.truncation);
        check(gsim_gpu_tsdf_download(ctx, &v, out.tsdf.data(), out.weights.data()), ctx);
        return out;
    }
};

}  // namespace detail

// Which writer outputs to produce (gsim_gpu.h GSIM_ENCODE_*); the defaults are the reference
// CLI's render outputs (tools/gsim.cpp:60-65).
struct EncodeOptions {
    uint32_t flags = GSIM_ENCODE_RGB8 | GSIM_ENCODE_ALPHA8 | GSIM_ENCODE_DEPTH16 | GSIM_ENCODE_DEPTH_PFM;
    bool srgb = true;
    double depth_scale = 1000.0;
    gsim_encode_options c() const { return gsim_encode_options{flags, srgb ? 1 : 0, depth_scale}; }
};

class Renderer;

// Device-resident pose tracks built from PoseStream records (the PoseStream(records)
// constructor's input, pose_stream.hpp:28): one track per node id, records in input order.
class PoseTracks {
public:
    PoseTracks(Renderer& r, const std::vector<PoseRecord>& records);
    // index of the node's track, -1 when the stream does not drive it
    int64_t track_of(const std::string& node) const {
        const auto it = index_.find(node);
        return it == index_.end() ? -1 : int64_t(it->second);
    }
    const gsim_gpu_tracks* handle() const { return tracks_.get(); }

private:
    struct Del { void operator()(gsim_gpu_tracks* t) const { gsim_gpu_tracks_destroy(t); } };
    std::unique_ptr<gsim_gpu_tracks, Del> tracks_;
    std::map<std::string, std::size_t> index_;
};

// One device context plus (optionally) a resident scene.
class Renderer {
public:
    explicit Renderer(int device = 0) {
        gsim_gpu_context* c = nullptr;
        detail::check(gsim_gpu_context_create(device, &c), nullptr);
        ctx_.reset(c);
    }
    explicit Renderer(const GaussianField& field, int device = 0) : Renderer(device) { upload(field); }

    // Copies the field into HBM (replaces a previously uploaded one).
    void upload(const GaussianField& field) {
        const gsim_field_view v = detail::view(field);
        gsim_gpu_scene* s = nullptr;
        key_ = detail::FieldKey{};
        detail::check(gsim_gpu_scene_upload(ctx_.get(), &v, &s), ctx_.get());
        scene_.reset(s);
        key_ = detail::field_key(field);
    }

    // Uploads the field unless the resident copy was uploaded from the same field (same
    // storage, size, degree, generation and sampled content). Returns whether it uploaded.
    bool ensure(const GaussianField& field) {
        if (scene_ && detail::field_key(field) == key_) return false;
        upload(field);
        return true;
    }

    // The resident copy was changed on the device to match `field` (transform_primitives).
    void adopt(const GaussianField& field) { key_ = detail::field_key(field); }

    std::vector<RenderTarget> render(const std::vector<SceneNode>& nodes,
                                     const std::vector<CameraModel>& cameras,
                                     const RasterOptions& options = {}) {
        const auto ns = detail::nodes(nodes);
        std::vector<gsim_camera> cs;
        for (const auto& c : cameras) cs.push_back(detail::camera(c));
        std::vector<RenderTarget> targets;
        std::vector<gsim_target> outs;
        targets.reserve(cameras.size());
        for (const auto& c : cameras) targets.emplace_back(c.width, c.height);
        for (auto& t : targets)
            outs.push_back(gsim_target{t.rgb.data.data(), t.depth.data.data(), t.accum_alpha.data.data()});
        const gsim_raster_options o = detail::options(options);
        detail::check(gsim_gpu_render(ctx_.get(), scene_.get(), ns.data(), ns.size(), cs.data(),
                                      cs.size(), &o, outs.data()),
                      ctx_.get());
        return targets;
    }

    std::vector<ProjectedSplat> project(const std::vector<SceneNode>& nodes, const CameraModel& camera) {
        const auto ns = detail::nodes(nodes);
        const gsim_camera c = detail::camera(camera);
        std::vector<ProjectedSplat> out(gsim_gpu_scene_size(scene_.get()));
        uint64_t count = 0;
        detail::check(gsim_gpu_project(ctx_.get(), scene_.get(), ns.data(), ns.size(), &c,
                                       reinterpret_cast<gsim_projected_splat*>(out.data()),
                                       out.size(), &count),
                      ctx_.get());
        out.resize(count);
        return out;
    }

    RenderTarget rasterize(const std::vector<ProjectedSplat>& splats, const CameraModel& camera,
                           const RasterOptions& options = {}) {
        const gsim_camera c = detail::camera(camera);
        const gsim_raster_options o = detail::options(options);
        RenderTarget t(camera.width, camera.height);
        gsim_target out{t.rgb.data.data(), t.depth.data.data(), t.accum_alpha.data.data()};
        detail::check(gsim_gpu_rasterize(ctx_.get(),
                                         reinterpret_cast<const gsim_projected_splat*>(splats.data()),
                                         splats.size(), &c, &o, &out),
                      ctx_.get());
        return t;
    }

    // load_splat_ply straight into HBM (replaces a previously uploaded field).
    void load_ply(const std::string& path) {
        gsim_gpu_scene* s = nullptr;
        detail::check(gsim_gpu_scene_load_ply(ctx_.get(), path.c_str(), &s), ctx_.get());
        scene_.reset(s);
    }

    // render + the writers' bytes, fused on the GPU; per camera the enabled parts in
    // GSIM_ENCODE_* order.
    std::vector<uint8_t> render_encoded(const std::vector<SceneNode>& nodes,
                                        const std::vector<CameraModel>& cameras,
                                        const RasterOptions& options = {},
                                        const EncodeOptions& encode = {}) {
        const auto ns = detail::nodes(nodes);
        std::vector<gsim_camera> cs;
        uint64_t bytes = 0;
        for (const auto& c : cameras) {
            cs.push_back(detail::camera(c));
            bytes += gsim_gpu_encoded_bytes(encode.flags, c.width, c.height);
        }
        std::vector<uint8_t> out(bytes);
        const gsim_raster_options o = detail::options(options);
        const gsim_encode_options e = encode.c();
        detail::check(gsim_gpu_render_encoded(ctx_.get(), scene_.get(), ns.data(), ns.size(), cs.data(),
                                              cs.size(), &o, &e, out.data(), 0),
                      ctx_.get());
        return out;
    }

    // Scene::step_to(stream, t) + render_all: nodes named in the tracks take their pose at t
    // (their pose in `nodes` is the initial pose), sampled on the GPU.
    std::vector<RenderTarget> render_at(const PoseTracks& tracks, double t,
                                        const std::vector<SceneNode>& nodes,
                                        const std::vector<CameraModel>& cameras,
                                        const RasterOptions& options = {}) {
        const auto ns = detail::nodes(nodes);
        std::vector<int64_t> node_track;
        for (const auto& n : nodes) node_track.push_back(tracks.track_of(n.id));
        std::vector<gsim_camera> cs;
        for (const auto& c : cameras) cs.push_back(detail::camera(c));
        std::vector<RenderTarget> targets;
        std::vector<gsim_target> outs;
        targets.reserve(cameras.size());
        for (const auto& c : cameras) targets.emplace_back(c.width, c.height);
        for (auto& tg : targets)
            outs.push_back(gsim_target{tg.rgb.data.data(), tg.depth.data.data(), tg.accum_alpha.data.data()});
        const gsim_raster_options o = detail::options(options);
        detail::check(gsim_gpu_render_at(ctx_.get(), scene_.get(), tracks.handle(), t, ns.data(),
                                         node_track.data(), ns.size(), cs.data(), cs.size(), &o,
                                         nullptr, outs.data()),
                      ctx_.get());
        return targets;
    }

    // The writers' bytes of one RenderTarget.
    std::vector<uint8_t> encode(const RenderTarget& t, const EncodeOptions& encode = {}) {
        std::vector<uint8_t> out(gsim_gpu_encoded_bytes(encode.flags, t.depth.width, t.depth.height));
        const gsim_encode_options e = encode.c();
        detail::check(gsim_gpu_encode_host(ctx_.get(), t.depth.width, t.depth.height, t.rgb.data.data(),
                                           t.depth.data.data(), t.accum_alpha.data.data(), &e,
                                           out.data()),
                      ctx_.get());
        return out;
    }

    // render_depth_ring (transfer.cpp:81-124) of the resident field.
    std::vector<DepthView> render_depth_ring(int n_views, double radius, int resolution) {
        const std::size_t n = std::size_t(3) * std::size_t(n_views > 0 ? n_views : 0);
        std::vector<gsim_camera> cs(n ? n : 1);
        std::vector<float> depth(std::max<std::size_t>(n, 1) * std::size_t(resolution > 0 ? resolution : 0) *
                                 std::size_t(resolution > 0 ? resolution : 0));
        detail::check(gsim_gpu_render_depth_ring(ctx_.get(), scene_.get(), n_views, radius, resolution,
                                                 cs.data(), depth.data(), 0),
                      ctx_.get());
        std::vector<DepthView> views(n);
        const std::size_t npx = std::size_t(resolution) * resolution;
        for (std::size_t v = 0; v < n; ++v) {
            views[v].camera = detail::from_camera(cs[v]);
            views[v].depth = Image1(resolution, resolution);
            std::memcpy(views[v].depth.data.data(), depth.data() + v * npx, npx * sizeof(float));
        }
        return views;
    }

    // gaussians_to_mesh (transfer.cpp:174-198) up to the fused volume, on the resident field.
    TsdfVolume gaussians_to_tsdf(double voxel_size) {
        gsim_tsdf_volume v{};
        detail::check(gsim_gpu_gaussians_to_tsdf(ctx_.get(), scene_.get(), voxel_size, &v), ctx_.get());
        detail::DeviceVolume dev(ctx_.get(), v);
        detail::check(gsim_gpu_gaussians_to_tsdf(ctx_.get(), scene_.get(), voxel_size, &dev.v), ctx_.get());
        return dev.download();
    }

    // tsdf_fuse (transfer.cpp:143-172): the volume's grids make a round trip through HBM.
    void tsdf_fuse(TsdfVolume& volume, const CameraModel& camera, const Image1& depth) {
        if (depth.width != camera.width || depth.height != camera.height)
            throw validation_error("tsdf_fuse: depth image does not match camera resolution");
        detail::DeviceVolume dev(ctx_.get(), detail::volume(volume));
        dev.upload(volume);
        const gsim_camera c = detail::camera(camera);
        detail::check(gsim_gpu_tsdf_fuse(ctx_.get(), &dev.v, &c, 1, depth.data.data(), 0), ctx_.get());
        const TsdfVolume out = dev.download();
        volume.tsdf = out.tsdf;
        volume.weights = out.weights;
    }

    // GaussianBvh::build(field, nodes).scan(lidar) (trace.cpp:88-111, 169-197) on the resident field.
    PointCloud lidar_scan(const std::vector<SceneNode>& nodes, const LidarModel& lidar) {
        const auto ns = detail::nodes(nodes);
        gsim_lidar l{};
        l.channels = lidar.channels.data();
        l.n_channels = lidar.channels.size();
        l.azimuth_step = lidar.azimuth_step;
        l.max_range = lidar.max_range;
        l.pose = detail::rigid(lidar.pose);
        l.alpha_threshold = lidar.alpha_threshold;
        l.env = GSIM_ENV_ALL;
        uint64_t count = 0;
        detail::check(gsim_gpu_lidar_scan(ctx_.get(), scene_.get(), ns.data(), ns.size(), &l, nullptr,
                                          nullptr, nullptr, 0, &count),
                      ctx_.get());
        std::vector<double> pts(3 * count), az(count);
        std::vector<uint32_t> ring(count);
        detail::check(gsim_gpu_lidar_scan(ctx_.get(), scene_.get(), ns.data(), ns.size(), &l, pts.data(),
                                          ring.data(), az.data(), count, &count),
                      ctx_.get());
        PointCloud cloud;
        for (uint64_t k = 0; k < count; ++k) {
            cloud.points.push_back(Vec3(pts[3 * k], pts[3 * k + 1], pts[3 * k + 2]));
            cloud.ring.push_back(ring[k]);
            cloud.azimuth.push_back(az[k]);
        }
        return cloud;
    }

    // GaussianBvh::trace (trace.cpp:113-123) for a batch of rays on the resident field.
    std::vector<TraceResult> trace(const std::vector<SceneNode>& nodes, const std::vector<Ray>& rays,
                                   double alpha_threshold = 0.5) {
        const auto ns = detail::nodes(nodes);
        std::vector<double> o, d, t;
        for (const Ray& r : rays) {
            o.insert(o.end(), {r.origin.x, r.origin.y, r.origin.z});
            d.insert(d.end(), {r.direction.x, r.direction.y, r.direction.z});
            t.push_back(r.t_max);
        }
        std::vector<uint8_t> hit(rays.size());
        std::vector<double> depth(rays.size()), acc(rays.size());
        detail::check(gsim_gpu_trace_rays(ctx_.get(), scene_.get(), ns.data(), ns.size(), o.data(), d.data(),
                                          t.data(), rays.size(), alpha_threshold, hit.data(),
                                          depth.data(), acc.data()),
                      ctx_.get());
        std::vector<TraceResult> out(rays.size());
        for (std::size_t k = 0; k < rays.size(); ++k) {
            out[k].hit = hit[k] != 0;
            out[k].depth = depth[k];
            out[k].accum_alpha = acc[k];
        }
        return out;
    }

    gsim_gpu_context* context() { return ctx_.get(); }
    gsim_gpu_scene* scene() { return scene_.get(); }

private:
    struct CtxDel { void operator()(gsim_gpu_context* c) const { gsim_gpu_context_destroy(c); } };
    struct SceneDel { void operator()(gsim_gpu_scene* s) const { gsim_gpu_scene_destroy(s); } };
    std::unique_ptr<gsim_gpu_context, CtxDel> ctx_;
    std::unique_ptr<gsim_gpu_scene, SceneDel> scene_;
    detail::FieldKey key_;
};

inline PoseTracks::PoseTracks(Renderer& r, const std::vector<PoseRecord>& records) {
    std::vector<std::vector<const PoseRecord*>> per;
    for (const auto& rec : records) {
        auto it = index_.find(rec.node);
        if (it == index_.end()) {
            it = index_.emplace(rec.node, per.size()).first;
            per.emplace_back();
        }
        per[it->second].push_back(&rec);
    }
    std::vector<double> t, p, q;
    std::vector<uint64_t> begin{0};
    for (const auto& track : per) {
        for (const PoseRecord* rec : track) {
            t.push_back(rec->t);
            p.insert(p.end(), {rec->pose.translation.x, rec->pose.translation.y, rec->pose.translation.z});
            q.insert(q.end(), {rec->pose.rotation.w, rec->pose.rotation.x, rec->pose.rotation.y,
                               rec->pose.rotation.z});
        }
        begin.push_back(t.size());
    }
    gsim_gpu_tracks* h = nullptr;
    detail::check(gsim_gpu_tracks_upload(r.context(), t.data(), p.data(), q.data(), begin.data(),
                                         per.size(), &h),
                  r.context());
    tracks_.reset(h);
}

// One context per host thread (the reference's render is callable from any thread; contexts
// serialise their own calls): the field cache and the workspaces live there.
inline Renderer& default_renderer() {
    static thread_local Renderer r(0);
    return r;
}

// Call after editing a field in place: every cached upload is refreshed on its next use.
inline void invalidate() { detail::field_generation().fetch_add(1); }
inline void invalidate(const GaussianField&) { invalidate(); }

// Same signature and contract as gsim::render (raster.hpp:64-67).
inline std::vector<RenderTarget> render(const GaussianField& field, const std::vector<SceneNode>& nodes,
                                        const std::vector<CameraModel>& cameras,
                                        const RasterOptions& options = {}) {
    Renderer& r = default_renderer();
    r.ensure(field);
    return r.render(nodes, cameras, options);
}

inline std::vector<ProjectedSplat> project(const GaussianField& field, const std::vector<SceneNode>& nodes,
                                           const CameraModel& camera) {
    Renderer& r = default_renderer();
    r.ensure(field);
    return r.project(nodes, camera);
}

inline RenderTarget rasterize(const std::vector<ProjectedSplat>& splats, const CameraModel& camera,
                              const RasterOptions& options = {}) {
    return default_renderer().rasterize(splats, camera, options);
}

// transform_primitives (gaussian.cpp:65-79) run by K1 on the device, written back in place.
inline void transform_primitives(GaussianField& field, const IndexRange& range,
                                 const RigidTransform& transform) {
    Renderer& r = default_renderer();
    r.ensure(field);
    const gsim_rigid t = detail::rigid(transform);
    detail::check(gsim_gpu_transform_primitives(r.context(), r.scene(), range.begin, range.end, &t),
                  r.context());
    std::vector<double> means(3 * field.size()), rots(4 * field.size());
    detail::check(gsim_gpu_scene_download(r.context(), r.scene(), means.data(), rots.data()),
                  r.context());
    for (std::size_t i = 0; i < field.size(); ++i) {
        auto& p = field.primitives[i];
        p.mean = Vec3(means[3 * i], means[3 * i + 1], means[3 * i + 2]);
        p.rotation = Quat(rots[4 * i], rots[4 * i + 1], rots[4 * i + 2], rots[4 * i + 3]);
    }
    invalidate();      // other threads' cached copies of this field are stale now
    r.adopt(field);    // this thread's resident copy was transformed in place: still current
}

// render_depth_ring (transfer.cpp:81-124): same signature, views rendered on the GPU.
inline std::vector<DepthView> render_depth_ring(const GaussianField& field, int n_views, double radius,
                                                int resolution) {
    Renderer& r = default_renderer();
    r.ensure(field);
    return r.render_depth_ring(n_views, radius, resolution);
}

// tsdf_fuse (transfer.cpp:143-172): same signature.
inline void tsdf_fuse(TsdfVolume& volume, const CameraModel& camera, const Image1& depth) {
    default_renderer().tsdf_fuse(volume, camera, depth);
}

// The volume gaussians_to_mesh fuses (its fused_volume output, transfer.cpp:194-195); marching
// cubes and decimation stay with the caller (extract_mesh, decimate).
inline TsdfVolume gaussians_to_tsdf(const GaussianField& field, double voxel_size) {
    Renderer& r = default_renderer();
    r.ensure(field);
    return r.gaussians_to_tsdf(voxel_size);
}

// GaussianBvh::build(field, nodes).scan(lidar) (trace.cpp:88-111, 169-197) on the GPU.
inline PointCloud lidar_scan(const GaussianField& field, const std::vector<SceneNode>& nodes,
                             const LidarModel& lidar) {
    Renderer& r = default_renderer();
    r.ensure(field);
    return r.lidar_scan(nodes, lidar);
}

// GaussianBvh::build(field, nodes).trace(ray, threshold) for every ray.
inline std::vector<TraceResult> trace(const GaussianField& field, const std::vector<SceneNode>& nodes,
                                      const std::vector<Ray>& rays, double alpha_threshold = 0.5) {
    Renderer& r = default_renderer();
    r.ensure(field);
    return r.trace(nodes, rays, alpha_threshold);
}

// The bytes gsim::write_png_rgb8 (srgb), write_png_gray8, write_png_gray16 (scale) and write_pfm
// would write for `t` (GSIM_ENCODE_* order), encoded on the GPU.
inline std::vector<uint8_t> encode(const RenderTarget& t, const EncodeOptions& options = {}) {
    return default_renderer().encode(t, options);
}

// Scene::render_all (scene.cpp:232-235): the scene's field (upload cached) and node poses.
inline std::vector<RenderTarget> render_all(const Scene& scene, const std::vector<CameraModel>& cameras,
                                            const RasterOptions& options = {}) {
    return gsim::gpu::render(scene.field(), scene.nodes(), cameras, options);
}

namespace detail {
// The reference bench's helpers (bench.cpp:36-75, file-local there), restated.
inline Aabb posed_field_bounds(const Scene& scene) {
    Aabb box;
    for (const auto& node : scene.nodes())
        for (std::size_t i = node.range.begin; i < node.range.end; ++i)
            box.expand(pose_primitive(scene.field().primitives[i], node.pose).bounds);
    return box;
}

inline std::vector<CameraModel> camera_ring(const Scene& scene, int count, int width, int height) {
    Aabb box = posed_field_bounds(scene);
    if (box.empty()) {
        box.expand({-1, -1, -1});
        box.expand({1, 1, 1});
    }
    const Vec3 center = box.center();
    const double diag = std::max(box.extent().norm(), 1e-3);
    const double radius = 1.2 * diag;
    const double focal = 0.8 * width;
    std::vector<CameraModel> cameras;
    for (int k = 0; k < count; ++k) {
        const double azimuth = kTwoPi * k / count;
        const Vec3 eye = center + Vec3{radius * std::cos(azimuth), radius * std::sin(azimuth), 0.35 * radius};
        CameraModel cam = CameraModel::look_at(eye, center, focal, focal, width, height);
        cam.id = "bench_cam" + std::to_string(k);
        cam.near = 0.01 * radius;
        cam.far = 10.0 * radius;
        cameras.push_back(cam);
    }
    return cameras;
}

inline void pose_frame(Scene& scene, int frame) {  // 30 Hz nominal clock, first interactive node
    for (auto& node : scene.nodes()) {
        if (node.kind != NodeKind::interactive) continue;
        node.pose.rotation = Quat::from_axis_angle({0, 0, 1}, deg_to_rad(30.0) * frame / 30.0);
        return;
    }
}

inline std::string gpu_machine_descriptor() {  // bench.cpp:79-96, plus the device
    std::string model = "unknown-cpu";
    std::ifstream cpuinfo("/proc/cpuinfo");
    std::string line;
    while (std::getline(cpuinfo, line)) {
        if (line.rfind("model name", 0) == 0) {
            const auto colon = line.find(':');
            if (colon != std::string::npos) {
                model = line.substr(colon + 1);
                const auto first = model.find_first_not_of(' ');
                if (first != std::string::npos) model = model.substr(first);
            }
            break;
        }
    }
    return model + " + " + gsim_gpu_version();
}
}  // namespace detail

// run_bench (bench.cpp:98-160) with the frames rendered by the GPU drop-in: the same camera
// ring, node motion, warm-up and timed loop (wall clock over whole frames, host RGB-D targets
// returned by value), first-frame image hash and fps; the optional brute-force crop stays the
// reference's CPU reference_rasterize, as in the reference bench.
inline BenchReport run_bench(Scene& scene, const BenchOptions& options) {
    using Clock = std::chrono::steady_clock;
    auto since = [](Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); };
    if (options.cameras < 1) throw validation_error("bench: need at least one camera");
    BenchReport report;
    report.primitives = scene.field().size();
    report.width = options.width;
    report.height = options.height;
    report.cameras = options.cameras;
    report.threads = 1;  // one host thread drives the device
    report.machine = options.machine.empty() ? detail::gpu_machine_descriptor() : options.machine;
    const auto cameras = detail::camera_ring(scene, options.cameras, options.width, options.height);
    for (int frame = 0; frame < options.warmup_frames; ++frame) {
        detail::pose_frame(scene, frame);
        render_all(scene, cameras);
    }
    int frame = options.warmup_frames, timed = 0;
    std::uint64_t first_hash = 0;
    const auto start = Clock::now();
    while (timed < options.min_frames || since(start) < options.seconds) {
        detail::pose_frame(scene, frame);
        const auto targets = render_all(scene, cameras);
        if (timed == 0) {
            std::uint64_t h = 1469598103934665603ull;
            for (const auto& t : targets) h = hash_target(t, h);
            first_hash = h;
        }
        ++frame;
        ++timed;
    }
    report.wall_time = since(start);
    report.frames = timed;
    report.fps = timed * options.cameras / report.wall_time;
    report.image_hash = first_hash;
    if (options.run_brute_force) {
        detail::pose_frame(scene, options.warmup_frames);
        CameraModel crop = cameras[0];
        crop.width = crop.height = options.brute_crop;
        crop.cx = crop.cy = options.brute_crop * 0.5;
        const auto brute_start = Clock::now();
        reference_rasterize(gsim::project(scene.field(), scene.nodes(), crop), crop);
        report.brute_wall = since(brute_start);
        report.brute_crop = options.brute_crop;
        const double tiled = double(timed) * options.cameras * options.width * options.height / report.wall_time;
        report.brute_speedup = tiled / (double(options.brute_crop) * options.brute_crop / report.brute_wall);
    }
    return report;
}

}  // namespace gsim::gpu
