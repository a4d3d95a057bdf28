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
//
// Errors are rethrown as the reference's gsim::validation_error (status 2) and gsim::io_error
// (status 1). The free functions upload the field on every call (a pure function of their
// inputs, like the reference); gsim::gpu::Renderer keeps it resident in HBM for the fast path.
#pragma once

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "gsim/errors.hpp"
#include "gsim/gaussian.hpp"
#include "gsim/raster.hpp"
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

}  // namespace detail

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
        detail::check(gsim_gpu_scene_upload(ctx_.get(), &v, &s), ctx_.get());
        scene_.reset(s);
    }

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

    gsim_gpu_context* context() { return ctx_.get(); }
    gsim_gpu_scene* scene() { return scene_.get(); }

private:
    struct CtxDel { void operator()(gsim_gpu_context* c) const { gsim_gpu_context_destroy(c); } };
    struct SceneDel { void operator()(gsim_gpu_scene* s) const { gsim_gpu_scene_destroy(s); } };
    std::unique_ptr<gsim_gpu_context, CtxDel> ctx_;
    std::unique_ptr<gsim_gpu_scene, SceneDel> scene_;
};

inline Renderer& default_renderer() {
    static Renderer r(0);
    return r;
}

// Same signature and contract as gsim::render (raster.hpp:64-67).
inline std::vector<RenderTarget> render(const GaussianField& field, const std::vector<SceneNode>& nodes,
                                        const std::vector<CameraModel>& cameras,
                                        const RasterOptions& options = {}) {
    Renderer& r = default_renderer();
    r.upload(field);
    return r.render(nodes, cameras, options);
}

inline std::vector<ProjectedSplat> project(const GaussianField& field, const std::vector<SceneNode>& nodes,
                                           const CameraModel& camera) {
    Renderer& r = default_renderer();
    r.upload(field);
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
    r.upload(field);
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
}

}  // namespace gsim::gpu
