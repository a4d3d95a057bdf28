// drop_in_check.cpp — one C++ binary that links the UNMODIFIED reference library (oracle/_ref,
// the checker) and the GPU library through include/gsim_gpu.hpp, and compares them on the same
// GaussianField with the reference's own types. TEST CODE (built by oracle/Makefile `drop_in`,
// run by tests/test_gpu_dropin.py on a GPU box).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "gsim/bench.hpp"
#include "gsim/gaussian.hpp"
#include "gsim/hash.hpp"
#include "gsim/image_io.hpp"
#include "gsim/pose_stream.hpp"
#include "gsim/raster.hpp"
#include "gsim/splat_ply.hpp"
#include "gsim/trace.hpp"
#include "gsim/transfer.hpp"
#include "gsim_gpu.hpp"
#include "png.h"  // oracle/png_capture: the row bytes the reference writers hand to libpng
#include "test_oracles.hpp"

using namespace gsim;

static double frac_within(const RenderTarget& a, const RenderTarget& b, double rgb_tol,
                          double depth_rel) {
    const std::size_t n = a.depth.data.size();
    std::size_t ok = 0;
    for (std::size_t p = 0; p < n; ++p) {
        double d = 0.0;
        for (int c = 0; c < 3; ++c)
            d = std::fmax(d, std::fabs(double(a.rgb.data[3 * p + c]) - b.rgb.data[3 * p + c]));
        const double dd = std::fabs(double(a.depth.data[p]) - b.depth.data[p]);
        const double rel = dd / std::fmax(std::fabs(double(b.depth.data[p])), 0.1);
        if (d <= rgb_tol && (rel <= depth_rel || dd <= 1e-4)) ++ok;
    }
    return double(ok) / double(n);
}

int main() {
    GaussianField field = oracle::random_field(2024, 3000, 3.0, 0.01, 0.2, 3);
    for (auto& p : field.primitives) p.mean.z += 3.0;
    std::vector<SceneNode> nodes(2);
    nodes[0] = {"bg", NodeKind::background, RigidTransform::identity(), {0, 2000}};
    nodes[1] = {"obj", NodeKind::interactive,
                RigidTransform{Quat::from_axis_angle({0, 0, 1}, 0.4), {0.1, 0.0, 0.2}}, {2000, 3000}};
    std::vector<CameraModel> cams(2);
    for (int k = 0; k < 2; ++k) {
        cams[k].fx = cams[k].fy = 120.0;
        cams[k].cx = 80.0;
        cams[k].cy = 60.0;
        cams[k].width = 160;
        cams[k].height = 120;
        cams[k].pose = RigidTransform{Quat::from_axis_angle({0, 1, 0}, 0.1 * k), {0.2 * k, 0.0, 0.0}};
    }
    int failures = 0;

    // render: same signature, reference types
    const auto ref = render(field, nodes, cams);
    const auto gpu = gpu::render(field, nodes, cams);
    for (int k = 0; k < 2; ++k) {
        const double f = frac_within(gpu[k], ref[k], 2e-3, 1e-3);
        std::printf("render camera %d: %.5f of pixels within tolerance\n", k, f);
        if (f < 0.999) ++failures;
    }

    // upload cache (gsim_gpu.hpp field_key): the same field is not re-uploaded; a field edited
    // in place (sampled by the fingerprint, or announced with invalidate()) and a second field
    // are; every render still matches the reference of the field it was given
    {
        gpu::Renderer& r = gpu::default_renderer();
        const bool again = r.ensure(field);
        std::printf("upload cache: same field re-uploaded = %d\n", again);
        if (again) ++failures;
        GaussianField edited = field;  // other storage: a different key
        for (auto& p : edited.primitives) p.mean.x += 0.05;
        const auto ref_e = render(edited, nodes, cams);
        const auto gpu_e = gpu::render(edited, nodes, cams);
        // in-place edit of one unsampled primitive's colour, announced with invalidate()
        edited.primitives[1].sh[0] += 3.0;
        edited.primitives[1].opacity = 0.99;
        gpu::invalidate(edited);
        const auto ref_i = render(edited, nodes, cams);
        const auto gpu_i = gpu::render(edited, nodes, cams);
        // in-place edit of every primitive's position, caught by the fingerprint alone
        for (auto& p : edited.primitives) p.mean.y -= 0.07;
        const auto ref_f = render(edited, nodes, cams);
        const auto gpu_f = gpu::render(edited, nodes, cams);
        const auto gpu_back = gpu::render(field, nodes, cams);  // the first field again
        double worst = 1.0;
        for (int k = 0; k < 2; ++k) {
            worst = std::fmin(worst, frac_within(gpu_e[k], ref_e[k], 2e-3, 1e-3));
            worst = std::fmin(worst, frac_within(gpu_i[k], ref_i[k], 2e-3, 1e-3));
            worst = std::fmin(worst, frac_within(gpu_f[k], ref_f[k], 2e-3, 1e-3));
            worst = std::fmin(worst, frac_within(gpu_back[k], ref[k], 2e-3, 1e-3));
        }
        bool differs = false;  // the announced edit really changed the image
        for (std::size_t p = 0; p < gpu_i[0].rgb.data.size(); ++p)
            differs |= gpu_i[0].rgb.data[p] != gpu_e[0].rgb.data[p];
        std::printf("upload cache: worst %.5f of pixels within tolerance after edits, edit visible %d\n",
                    worst, differs);
        if (worst < 0.999) ++failures;
    }

    // project: geometry bit-exact (double), rgb close
    const auto sp_ref = project(field, nodes, cams[0]);
    const auto sp_gpu = gpu::project(field, nodes, cams[0]);
    std::size_t geo_mismatch = sp_ref.size() == sp_gpu.size() ? 0 : 1;
    double rgb_err = 0.0;
    for (std::size_t i = 0; i < sp_ref.size() && i < sp_gpu.size(); ++i) {
        const auto& a = sp_ref[i];
        const auto& b = sp_gpu[i];
        if (a.prim_index != b.prim_index || a.pixel_center.x != b.pixel_center.x ||
            a.pixel_center.y != b.pixel_center.y || a.inv_xx != b.inv_xx || a.inv_xy != b.inv_xy ||
            a.inv_yy != b.inv_yy || a.view_depth != b.view_depth || a.radius != b.radius)
            ++geo_mismatch;
        rgb_err = std::fmax(rgb_err, std::fabs(a.rgb.x - b.rgb.x));
    }
    std::printf("project: %zu splats, %zu geometry mismatches, max rgb err %.2e\n", sp_ref.size(),
                geo_mismatch, rgb_err);
    if (geo_mismatch || rgb_err > 2e-5) ++failures;

    // rasterize of the reference's own splats
    const RenderTarget r_ref = rasterize(sp_ref, cams[0]);
    const RenderTarget r_gpu = gpu::rasterize(sp_ref, cams[0]);
    const double fr = frac_within(r_gpu, r_ref, 2e-3, 1e-3);
    std::printf("rasterize: %.5f of pixels within tolerance\n", fr);
    if (fr < 0.999) ++failures;

    // transform_primitives: bit-exact
    GaussianField a = field, b = field;
    const RigidTransform t{Quat::from_axis_angle({1, 2, 3}, 0.7), {0.5, -1.0, 2.0}};
    transform_primitives(a, {100, 2500}, t);
    gpu::transform_primitives(b, {100, 2500}, t);
    std::size_t tf_mismatch = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const auto& pa = a.primitives[i];
        const auto& pb = b.primitives[i];
        if (pa.mean.x != pb.mean.x || pa.mean.y != pb.mean.y || pa.mean.z != pb.mean.z ||
            pa.rotation.w != pb.rotation.w || pa.rotation.x != pb.rotation.x)
            ++tf_mismatch;
    }
    std::printf("transform_primitives: %zu mismatches\n", tf_mismatch);
    if (tf_mismatch) ++failures;

    // error mapping: a bad camera is a validation_error from both
    CameraModel bad = cams[0];
    bad.fx = 0.0;
    bool ref_threw = false, gpu_threw = false;
    try { render(field, nodes, {bad}); } catch (const validation_error&) { ref_threw = true; }
    try { gpu::render(field, nodes, {bad}); } catch (const validation_error&) { gpu_threw = true; }
    std::printf("validation_error: reference %d, gpu %d\n", ref_threw, gpu_threw);
    if (!ref_threw || !gpu_threw) ++failures;

    // encode: gsim::gpu::encode bytes == what write_png_rgb8(srgb) / gray8 / gray16(1000) /
    // write_pfm write for the reference's own render target
    {
        const RenderTarget& t = ref[0];
        const std::vector<uint8_t> enc = gpu::encode(t);
        std::vector<uint8_t> want;
        auto capture = [&]() {
            std::size_t n = 0;
            const unsigned char* b = png_capture_last(nullptr, nullptr, nullptr, nullptr, &n);
            want.insert(want.end(), b, b + n);
        };
        write_png_rgb8("/dev/null", t.rgb, true);
        capture();
        write_png_gray8("/dev/null", t.accum_alpha);
        capture();
        write_png_gray16("/dev/null", t.depth, 1000.0);
        capture();
        const std::string pfm = "/tmp/drop_in_check_depth.pfm";
        write_pfm(pfm, t.depth);
        std::ifstream in(pfm, std::ios::binary);
        std::vector<uint8_t> file((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        const std::string head = "Pf\n" + std::to_string(t.depth.width) + " " +
                                 std::to_string(t.depth.height) + "\n-1.0\n";
        want.insert(want.end(), file.begin() + head.size(), file.end());
        std::size_t diff = enc.size() == want.size() ? 0 : 1;
        for (std::size_t i = 0; i < enc.size() && i < want.size(); ++i) diff += enc[i] != want[i];
        std::printf("encode: %zu bytes, %zu differ from the reference writers\n", enc.size(), diff);
        if (diff) ++failures;
        // fused render + encode == encode of the GPU's float render
        gpu::Renderer r(field);
        const std::vector<uint8_t> fused = r.render_encoded(nodes, {cams[0]});
        const std::vector<uint8_t> sep = r.encode(r.render(nodes, {cams[0]})[0]);
        std::printf("render_encoded: %s\n", fused == sep ? "equal" : "DIFFERENT");
        if (fused != sep) ++failures;
    }

    // splat PLY: the reference writes the field, both load it and render
    {
        const std::string ply = "/tmp/drop_in_check_field.ply";
        save_splat_ply(field, ply);
        const GaussianField loaded = load_splat_ply(ply);
        gpu::Renderer r;
        r.load_ply(ply);
        const auto a = render(loaded, nodes, cams);
        const auto b = r.render(nodes, cams);
        for (int k = 0; k < 2; ++k) {
            const double f = frac_within(b[k], a[k], 2e-3, 1e-3);
            std::printf("load_ply + render camera %d: %.5f of pixels within tolerance\n", k, f);
            if (f < 0.999) ++failures;
        }
        bool ref_threw = false, gpu_threw = false;
        try { load_splat_ply("/tmp/does_not_exist.ply"); } catch (const io_error&) { ref_threw = true; }
        try { r.load_ply("/tmp/does_not_exist.ply"); } catch (const io_error&) { gpu_threw = true; }
        std::printf("load_ply io_error: reference %d, gpu %d\n", ref_threw, gpu_threw);
        if (!ref_threw || !gpu_threw) ++failures;
    }

    // pose playback: PoseStream::sample on the host vs render_at sampling on the GPU
    {
        std::vector<PoseRecord> recs;
        for (int i = 0; i < 6; ++i) {
            PoseRecord rec;
            rec.t = 0.25 * i;
            rec.node = "obj";
            rec.pose = RigidTransform{Quat::from_axis_angle({0.2, 1, 0.3}, 0.5 * i),
                                      {0.1 * i, -0.05 * i, 0.02 * i}};
            recs.push_back(rec);
        }
        const PoseStream stream(recs);
        gpu::Renderer r(field);
        const gpu::PoseTracks tracks(r, recs);
        for (double t : {-1.0, 0.3, 0.8, 9.0}) {
            std::vector<SceneNode> posed = nodes;
            posed[1].pose = stream.sample("obj", t, nodes[1].pose);
            const auto a = render(field, posed, cams);
            const auto b = r.render_at(tracks, t, nodes, cams);
            for (int k = 0; k < 2; ++k) {
                const double f = frac_within(b[k], a[k], 2e-3, 1e-3);
                if (f < 0.999) {
                    std::printf("render_at t=%.2f camera %d: %.5f within tolerance\n", t, k, f);
                    ++failures;
                }
            }
        }
        std::printf("render_at: 4 times x 2 cameras checked against PoseStream::sample + render\n");
    }

    // GS -> TSDF (transfer.cpp): depth ring, fuse, fused volume
    {
        GaussianField small = oracle::random_field(77, 800, 1.5, 0.02, 0.1, 1);
        const auto ra = render_depth_ring(small, 8, 6.0, 48);
        const auto ga = gpu::render_depth_ring(small, 8, 6.0, 48);
        std::size_t cam_diff = ra.size() != ga.size(), mask_diff = 0, depth_bad = 0, both = 0, px = 0;
        for (std::size_t v = 0; v < std::min(ra.size(), ga.size()); ++v) {
            const auto &a = ra[v].camera, &b = ga[v].camera;
            cam_diff += a.fx != b.fx || a.cx != b.cx || a.near != b.near || a.far != b.far ||
                        a.pose.rotation.w != b.pose.rotation.w || a.pose.rotation.x != b.pose.rotation.x ||
                        a.pose.translation.x != b.pose.translation.x ||
                        a.pose.translation.z != b.pose.translation.z;
            for (std::size_t i = 0; i < ra[v].depth.data.size(); ++i, ++px) {
                const double da = ra[v].depth.data[i], db = ga[v].depth.data[i];
                mask_diff += (da > 0) != (db > 0);
                if (da > 0 && db > 0) {
                    ++both;
                    depth_bad += std::fabs(db - da) > 1e-3 * std::fabs(da);
                }
            }
        }
        std::printf("render_depth_ring: %zu camera mismatches, mask differs on %zu of %zu px, "
                    "%zu of %zu depths beyond 1e-3\n", cam_diff, mask_diff, px, depth_bad, both);
        if (cam_diff || mask_diff > px / 1000 || depth_bad > both / 1000) ++failures;
        // tsdf_fuse on the reference's own depth maps: bit-exact
        TsdfVolume va = TsdfVolume::create({-1.7, -1.8, -1.6}, 0.06, {57, 60, 55}, 0.18);
        TsdfVolume vb = va;
        for (const auto& view : ra) {
            tsdf_fuse(va, view.camera, view.depth);
            gpu::tsdf_fuse(vb, view.camera, view.depth);
        }
        std::size_t fuse_diff = 0;
        for (std::size_t i = 0; i < va.tsdf.size(); ++i)
            fuse_diff += va.tsdf[i] != vb.tsdf[i] || va.weights[i] != vb.weights[i];
        std::printf("tsdf_fuse: %zu of %zu voxels differ\n", fuse_diff, va.tsdf.size());
        if (fuse_diff) ++failures;
        // gaussians_to_mesh's fused volume vs gsim::gpu::gaussians_to_tsdf
        TsdfVolume fused;
        gaussians_to_mesh(small, 0.1, std::size_t(-1), &fused);
        const TsdfVolume g = gpu::gaussians_to_tsdf(small, 0.1);
        std::size_t close = 0;
        const bool geo = g.dims == fused.dims && g.origin.x == fused.origin.x &&
                         g.origin.z == fused.origin.z && g.truncation == fused.truncation;
        for (std::size_t i = 0; geo && i < g.tsdf.size(); ++i)
            close += g.weights[i] == fused.weights[i] && std::fabs(g.tsdf[i] - fused.tsdf[i]) <= 1e-3;
        std::printf("gaussians_to_tsdf: geometry %s, %zu of %zu voxels match\n", geo ? "equal" : "DIFFERENT",
                    close, fused.tsdf.size());
        if (!geo || close < fused.tsdf.size() * 99 / 100) ++failures;
        bool ref_threw = false, gpu_threw = false;
        try { render_depth_ring(small, 7, 6.0, 48); } catch (const validation_error&) { ref_threw = true; }
        try { gpu::render_depth_ring(small, 7, 6.0, 48); } catch (const validation_error&) { gpu_threw = true; }
        std::printf("render_depth_ring validation_error: reference %d, gpu %d\n", ref_threw, gpu_threw);
        if (!ref_threw || !gpu_threw) ++failures;
    }

    // LiDAR (trace.cpp): GaussianBvh::scan and trace vs gsim::gpu
    {
        GaussianField f = oracle::random_field(91, 2500, 2.0, 0.02, 0.15, 0);
        std::vector<SceneNode> ln(2);
        ln[0] = {"bg", NodeKind::background, RigidTransform::identity(), {0, 1600}};
        ln[1] = {"obj", NodeKind::interactive,
                 RigidTransform{Quat::from_axis_angle({0, 0, 1}, 0.3), {0.2, 0.1, 0.0}}, {1600, 2500}};
        LidarModel lid;
        lid.id = "l0";
        for (int c = 0; c < 16; ++c) lid.channels.push_back((-15.0 + 2.0 * c) * kPi / 180.0);
        lid.azimuth_step = 2.0 * kPi / 180.0;
        lid.max_range = 10.0;
        lid.pose = RigidTransform{Quat::from_axis_angle({1, 0, 0}, 0.1), {0.1, -0.2, 0.05}};
        const GaussianBvh bvh = GaussianBvh::build(f, ln);
        const PointCloud a = bvh.scan(lid);
        const PointCloud b = gpu::lidar_scan(f, ln, lid);
        double worst = 0.0;
        bool same = a.size() == b.size();
        for (std::size_t k = 0; same && k < a.size(); ++k) {
            same = a.ring[k] == b.ring[k] && a.azimuth[k] == b.azimuth[k];
            worst = std::fmax(worst, (a.points[k] - b.points[k]).norm());
        }
        std::printf("lidar_scan: %zu returns (reference %zu), order %s, max point distance %.3g m\n",
                    b.size(), a.size(), same ? "equal" : "DIFFERENT", worst);
        if (!same || worst > 1e-12) ++failures;
        std::vector<Ray> rays;
        for (int k = 0; k < 64; ++k) {
            Ray r;
            r.origin = {0.1 * (k % 5) - 0.2, 0.05 * (k % 7), -0.1};
            r.direction = Vec3{std::cos(0.1 * k), std::sin(0.1 * k), 0.05 * (k % 3)}.normalized();
            r.t_max = 6.0;
            rays.push_back(r);
        }
        const auto tg = gpu::trace(f, ln, rays, 0.5);
        std::size_t trace_bad = 0;
        for (std::size_t k = 0; k < rays.size(); ++k) {
            const TraceResult t = bvh.trace(rays[k], 0.5);
            trace_bad += t.hit != tg[k].hit || std::fabs(t.depth - tg[k].depth) > 1e-12 ||
                         std::fabs(t.accum_alpha - tg[k].accum_alpha) > 1e-12;
        }
        std::printf("trace: %zu of %zu rays differ\n", trace_bad, rays.size());
        if (trace_bad) ++failures;
        LidarModel bad = lid;
        bad.azimuth_step = 7.0 * kPi / 180.0;
        bool ref_threw = false, gpu_threw = false;
        try { bvh.scan(bad); } catch (const validation_error&) { ref_threw = true; }
        try { gpu::lidar_scan(f, ln, bad); } catch (const validation_error&) { gpu_threw = true; }
        std::printf("lidar validation_error: reference %d, gpu %d\n", ref_threw, gpu_threw);
        if (!ref_threw || !gpu_threw) ++failures;
    }

    // run_bench / Scene::render_all (bench.cpp:98-160, scene.cpp:232-235): a scene loaded by the
    // reference's own Scene::load from a manifest + splat PLYs, benched by the reference and by
    // gsim::gpu::run_bench. The restated camera ring and node motion reproduce the reference's
    // first-frame hash bit for bit; the GPU frames match the reference's within tolerance.
    {
        const std::string dir = "/tmp/gsim_dropin_scene";
        if (std::system(("mkdir -p " + dir).c_str()) != 0) ++failures;
        GaussianField bg = oracle::random_field(31, 2500, 2.0, 0.01, 0.15, 2);
        GaussianField obj = oracle::random_field(32, 800, 0.5, 0.01, 0.08, 2);
        save_splat_ply(bg, dir + "/bg.ply");
        save_splat_ply(obj, dir + "/obj.ply");
        {
            std::ofstream m(dir + "/scene.json");
            m << R"({"nodes": [{"id": "bg", "kind": "background", "splat": "bg.ply"},
                              {"id": "obj", "kind": "interactive", "splat": "obj.ply",
                               "pose": {"p": [0.2, 0.0, 0.1], "q": [1, 0, 0, 0]}}]})";
        }
        BenchOptions opt;
        opt.cameras = 3;
        opt.width = 160;
        opt.height = 120;
        opt.seconds = 0.0;
        opt.warmup_frames = 1;
        opt.min_frames = 2;
        opt.run_brute_force = false;
        Scene ref_scene = Scene::load(dir + "/scene.json");
        Scene gpu_scene = Scene::load(dir + "/scene.json");
        const BenchReport r_ref = run_bench(ref_scene, opt);
        const BenchReport r_gpu = gpu::run_bench(gpu_scene, opt);
        // the first timed frame: frame index warmup_frames on the restated camera ring
        Scene probe = Scene::load(dir + "/scene.json");
        gpu::detail::pose_frame(probe, opt.warmup_frames);
        const auto ring = gpu::detail::camera_ring(probe, opt.cameras, opt.width, opt.height);
        const auto ref_frame = render(probe.field(), probe.nodes(), ring);
        const auto gpu_frame = gpu::render_all(probe, ring);
        std::uint64_t h_ref = 1469598103934665603ull, h_gpu = 1469598103934665603ull;
        double worst = 1.0;
        for (int k = 0; k < opt.cameras; ++k) {
            h_ref = hash_target(ref_frame[k], h_ref);
            h_gpu = hash_target(gpu_frame[k], h_gpu);
            worst = std::fmin(worst, frac_within(gpu_frame[k], ref_frame[k], 2e-3, 1e-3));
        }
        const bool ring_exact = h_ref == r_ref.image_hash;
        const bool gpu_consistent = h_gpu == r_gpu.image_hash;
        std::printf("run_bench: reference %.1f camera-frames/s, gpu %.1f camera-frames/s (%d frames); "
                    "ring hash matches the reference %d, gpu hash consistent %d, frame within tolerance %.5f\n",
                    r_ref.fps, r_gpu.fps, r_gpu.frames, ring_exact, gpu_consistent, worst);
        if (!ring_exact || !gpu_consistent || worst < 0.999 || r_gpu.frames < opt.min_frames ||
            r_gpu.primitives != r_ref.primitives)
            ++failures;
    }

    std::printf(failures ? "DROP-IN FAILED\n" : "DROP-IN OK\n");
    return failures ? 1 : 0;
}
