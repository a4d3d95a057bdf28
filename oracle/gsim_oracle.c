/*
 * gsim_oracle.c — plain-C restatement of the reference render path.
 *
 * TEST INFRASTRUCTURE ONLY (see gsim_oracle.h): the checker for the CUDA path and the
 * CPU "port" baseline. Nothing in paper_2507_21981_b200/ links or calls this file.
 *
 * Every function follows the cited reference source line by line, in double precision and
 * in the same floating-point operation order, so that compiled with gcc -O3 (no -ffast-math,
 * no FMA contraction on x86-64) it is bit-identical to the reference. tests/test_oracle_pin.py
 * proves that against the reference itself and against tests/golden/.
 */
#include "gsim_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- math.hpp restated ------------------------------------------------------------------ */

typedef struct { double x, y, z; } v3;
typedef struct { double w, x, y, z; } quat;
typedef struct { double m[9]; } mat3; /* row-major, math.hpp:56-57 */

static v3 v3_make(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 v3_add(v3 a, v3 b) { return v3_make(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 v3_sub(v3 a, v3 b) { return v3_make(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 v3_neg(v3 a) { return v3_make(-a.x, -a.y, -a.z); }
static v3 v3_scale(v3 a, double s) { return v3_make(a.x * s, a.y * s, a.z * s); }
static v3 v3_div(v3 a, double s) { return v3_make(a.x / s, a.y / s, a.z / s); }
static double v3_dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 v3_cross(v3 a, v3 b) { /* math.hpp:34-36 */
    return v3_make(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double v3_norm(v3 a) { return sqrt(v3_dot(a, a)); }
static v3 v3_normalized(v3 a) { /* math.hpp:39-42 */
    const double n = v3_norm(a);
    return n > 0.0 ? v3_div(a, n) : v3_make(0.0, 0.0, 0.0);
}

static quat q_make(double w, double x, double y, double z) { quat q = {w, x, y, z}; return q; }
static double q_norm(quat q) { return sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z); }
static quat q_normalized(quat q) { /* math.hpp:124-127 */
    const double n = q_norm(q);
    return n > 0.0 ? q_make(q.w / n, q.x / n, q.y / n, q.z / n) : q_make(1.0, 0.0, 0.0, 0.0);
}
static quat q_conj(quat q) { return q_make(q.w, -q.x, -q.y, -q.z); }
static quat q_mul(quat a, quat o) { /* Hamilton product, math.hpp:132-137 */
    return q_make(a.w * o.w - a.x * o.x - a.y * o.y - a.z * o.z,
                  a.w * o.x + a.x * o.w + a.y * o.z - a.z * o.y,
                  a.w * o.y - a.x * o.z + a.y * o.w + a.z * o.x,
                  a.w * o.z + a.x * o.y - a.y * o.x + a.z * o.w);
}
static v3 q_rotate(quat q, v3 v) { /* math.hpp:139-143 */
    const v3 qv = v3_make(q.x, q.y, q.z);
    const v3 t = v3_scale(v3_cross(qv, v), 2.0);
    return v3_add(v3_add(v, v3_scale(t, q.w)), v3_cross(qv, t));
}
static v3 q_inverse_rotate(quat q, v3 v) { return q_rotate(q_conj(q), v); } /* math.hpp:144 */
static mat3 q_to_matrix(quat q) { /* math.hpp:146-155 */
    const double xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z;
    const double xy = q.x * q.y, xz = q.x * q.z, yz = q.y * q.z;
    const double wx = q.w * q.x, wy = q.w * q.y, wz = q.w * q.z;
    mat3 r;
    r.m[0] = 1 - 2 * (yy + zz); r.m[1] = 2 * (xy - wz);     r.m[2] = 2 * (xz + wy);
    r.m[3] = 2 * (xy + wz);     r.m[4] = 1 - 2 * (xx + zz); r.m[5] = 2 * (yz - wx);
    r.m[6] = 2 * (xz - wy);     r.m[7] = 2 * (yz + wx);     r.m[8] = 1 - 2 * (xx + yy);
    return r;
}
static quat q_from_matrix(const mat3* mm) { /* Shepperd, math.hpp:158-187 */
    const double* m = mm->m;
#define M(r, c) m[(r) * 3 + (c)]
    quat q;
    const double tr = M(0, 0) + M(1, 1) + M(2, 2);
    if (tr > 0.0) {
        double s = sqrt(tr + 1.0) * 2.0;
        q.w = 0.25 * s;
        q.x = (M(2, 1) - M(1, 2)) / s;
        q.y = (M(0, 2) - M(2, 0)) / s;
        q.z = (M(1, 0) - M(0, 1)) / s;
    } else if (M(0, 0) > M(1, 1) && M(0, 0) > M(2, 2)) {
        double s = sqrt(1.0 + M(0, 0) - M(1, 1) - M(2, 2)) * 2.0;
        q.w = (M(2, 1) - M(1, 2)) / s;
        q.x = 0.25 * s;
        q.y = (M(0, 1) + M(1, 0)) / s;
        q.z = (M(0, 2) + M(2, 0)) / s;
    } else if (M(1, 1) > M(2, 2)) {
        double s = sqrt(1.0 + M(1, 1) - M(0, 0) - M(2, 2)) * 2.0;
        q.w = (M(0, 2) - M(2, 0)) / s;
        q.x = (M(0, 1) + M(1, 0)) / s;
        q.y = 0.25 * s;
        q.z = (M(1, 2) + M(2, 1)) / s;
    } else {
        double s = sqrt(1.0 + M(2, 2) - M(0, 0) - M(1, 1)) * 2.0;
        q.w = (M(1, 0) - M(0, 1)) / s;
        q.x = (M(0, 2) + M(2, 0)) / s;
        q.y = (M(1, 2) + M(2, 1)) / s;
        q.z = 0.25 * s;
    }
#undef M
    return q_normalized(q);
}
static mat3 m3_mul(const mat3* a, const mat3* b) { /* row(r).dot(o.col(c)), math.hpp:91-97 */
    mat3 out;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            out.m[r * 3 + c] = a->m[r * 3 + 0] * b->m[0 * 3 + c] + a->m[r * 3 + 1] * b->m[1 * 3 + c] +
                               a->m[r * 3 + 2] * b->m[2 * 3 + c];
    return out;
}
static mat3 m3_transposed(const mat3* a) {
    mat3 t;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) t.m[r * 3 + c] = a->m[c * 3 + r];
    return t;
}
static mat3 m3_diag(double a, double b, double c) {
    mat3 d = {{a, 0, 0, 0, b, 0, 0, 0, c}};
    return d;
}

static quat rigid_q(const gsim_rigid* r) {
    return q_make(r->rotation[0], r->rotation[1], r->rotation[2], r->rotation[3]);
}
static v3 rigid_t(const gsim_rigid* r) {
    return v3_make(r->translation[0], r->translation[1], r->translation[2]);
}
static v3 rigid_apply(const gsim_rigid* r, v3 p) { /* transform_point, math.hpp:226 */
    return v3_add(q_rotate(rigid_q(r), p), rigid_t(r));
}

void gso_rigid_compose(const gsim_rigid* a, const gsim_rigid* b, gsim_rigid* out) {
    /* math.hpp:230-233 */
    const quat q = q_normalized(q_mul(rigid_q(a), rigid_q(b)));
    const v3 t = v3_add(q_rotate(rigid_q(a), rigid_t(b)), rigid_t(a));
    out->rotation[0] = q.w; out->rotation[1] = q.x; out->rotation[2] = q.y; out->rotation[3] = q.z;
    out->translation[0] = t.x; out->translation[1] = t.y; out->translation[2] = t.z;
}

void gso_rigid_inverse(const gsim_rigid* a, gsim_rigid* out) { /* math.hpp:235-238 */
    const quat inv = q_conj(rigid_q(a));
    const v3 t = v3_neg(q_rotate(inv, rigid_t(a)));
    out->rotation[0] = inv.w; out->rotation[1] = inv.x; out->rotation[2] = inv.y;
    out->rotation[3] = inv.z;
    out->translation[0] = t.x; out->translation[1] = t.y; out->translation[2] = t.z;
}

void gso_quat_from_axis_angle(const double axis[3], double angle, double q[4]) {
    /* math.hpp:115-120 */
    const v3 a = v3_normalized(v3_make(axis[0], axis[1], axis[2]));
    const double h = 0.5 * angle;
    const double s = sin(h);
    q[0] = cos(h); q[1] = a.x * s; q[2] = a.y * s; q[3] = a.z * s;
}

void gso_camera_center(const gsim_camera* cam, double out[3]) { /* camera.hpp:23 */
    gsim_rigid inv;
    gso_rigid_inverse(&cam->pose, &inv);
    out[0] = inv.translation[0]; out[1] = inv.translation[1]; out[2] = inv.translation[2];
}

void gso_look_at(const double eye_[3], const double target_[3], double fx, double fy, int width,
                 int height, const double up_[3], gsim_camera* cam) {
    /* CameraModel::look_at, raster.cpp:25-42 */
    memset(cam, 0, sizeof(*cam));
    cam->fx = fx; cam->fy = fy;
    cam->cx = width * 0.5; cam->cy = height * 0.5;
    cam->width = width; cam->height = height;
    cam->near_plane = 0.05; cam->far_plane = 100.0; /* camera.hpp:20 defaults */
    const v3 eye = v3_make(eye_[0], eye_[1], eye_[2]);
    const v3 target = v3_make(target_[0], target_[1], target_[2]);
    const v3 up = v3_make(up_[0], up_[1], up_[2]);
    const v3 forward = v3_normalized(v3_sub(target, eye));
    v3 right = v3_normalized(v3_cross(forward, up));
    if (v3_dot(right, right) < 1e-20) right = v3_normalized(v3_cross(forward, v3_make(0, 1, 0)));
    const v3 down = v3_cross(forward, right);
    mat3 w2c = {{right.x, right.y, right.z, down.x, down.y, down.z, forward.x, forward.y,
                 forward.z}};
    const quat q = q_from_matrix(&w2c);
    const v3 t = v3_neg(q_rotate(q, eye));
    cam->pose.rotation[0] = q.w; cam->pose.rotation[1] = q.x;
    cam->pose.rotation[2] = q.y; cam->pose.rotation[3] = q.z;
    cam->pose.translation[0] = t.x; cam->pose.translation[1] = t.y; cam->pose.translation[2] = t.z;
}

/* ---- sh.cpp restated -------------------------------------------------------------------- */

static const double kSh0 = 0.28209479177387814; /* sh.hpp:12-20 */
static const double kSh1 = 0.4886025119029199;
static const double kSh2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                               -1.0925484305920792, 0.5462742152960396};
static const double kSh3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                               0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                               -0.5900435899266435};

void gso_shade_sh(const double* sh, int degree, const double d[3], double rgb[3]) {
    /* sh.cpp:10-51 */
    const double x = d[0], y = d[1], z = d[2];
    double basis[16];
    int n = 1;
    basis[0] = kSh0;
    if (degree >= 1) {
        basis[1] = -kSh1 * y;
        basis[2] = kSh1 * z;
        basis[3] = -kSh1 * x;
        n = 4;
    }
    if (degree >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        basis[4] = kSh2[0] * x * y;
        basis[5] = kSh2[1] * y * z;
        basis[6] = kSh2[2] * (2.0 * zz - xx - yy);
        basis[7] = kSh2[3] * x * z;
        basis[8] = kSh2[4] * (xx - yy);
        n = 9;
    }
    if (degree >= 3) {
        const double xx = x * x, yy = y * y, zz = z * z;
        basis[9] = kSh3[0] * y * (3.0 * xx - yy);
        basis[10] = kSh3[1] * x * y * z;
        basis[11] = kSh3[2] * y * (4.0 * zz - xx - yy);
        basis[12] = kSh3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
        basis[13] = kSh3[4] * x * (4.0 * zz - xx - yy);
        basis[14] = kSh3[5] * z * (xx - yy);
        basis[15] = kSh3[6] * x * (xx - 3.0 * yy);
        n = 16;
    }
    for (int c = 0; c < 3; ++c) {
        double acc = 0.5;
        for (int k = 0; k < n; ++k) acc += basis[k] * sh[c * 16 + k];
        rgb[c] = (acc < 0.0) ? 0.0 : acc; /* std::max(acc, 0.0) */
    }
}

/* ---- raster.cpp restated ---------------------------------------------------------------- */

static const int kTileSize = 16;             /* raster.hpp:38-41 */
static const double kCovarianceFloor = 0.3;
static const double kAlphaClamp = 0.99;
static const double kAlphaSkip = 1.0 / 255.0;

static uint32_t depth_sort_key(double view_depth) { /* raster.hpp:45-47 */
    const float f = (float)view_depth;
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}

static int validate_camera(const gsim_camera* cam) { /* raster.cpp:16-23 */
    if (!(cam->fx > 0.0) || !(cam->fy > 0.0)) return GSIM_ERR_VALIDATION;
    if (!(cam->near_plane > 0.0) || !(cam->far_plane > cam->near_plane)) return GSIM_ERR_VALIDATION;
    if (cam->width < 16 || cam->height < 16) return GSIM_ERR_VALIDATION;
    return GSIM_OK;
}

static double clampd(double v, double lo, double hi) { /* std::clamp */
    return (v < lo) ? lo : (hi < v) ? hi : v;
}

int gso_project(const gsim_field_view* field, const gsim_node* nodes, uint64_t n_nodes,
                const gsim_camera* camera, gsim_projected_splat* out, uint64_t capacity,
                uint64_t* count) {
    /* raster.cpp:66-163 */
    if (validate_camera(camera) != GSIM_OK) return GSIM_ERR_VALIDATION;
    const uint64_t n = field->count;
    /* PoseTable (raster.cpp:47-62): index 0 is identity; later nodes overwrite earlier ones. */
    uint32_t* of_primitive = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    for (uint64_t k = 0; k < n_nodes; ++k) {
        if (nodes[k].end > n) { free(of_primitive); return GSIM_ERR_VALIDATION; }
        for (uint64_t i = nodes[k].begin; i < nodes[k].end; ++i) of_primitive[i] = (uint32_t)(k + 1);
    }
    gsim_rigid identity;
    memset(&identity, 0, sizeof(identity));
    identity.rotation[0] = 1.0;

    const quat cam_q = rigid_q(&camera->pose);
    const mat3 r_wc = q_to_matrix(cam_q);
    const mat3 r_wc_t = m3_transposed(&r_wc);
    double cc[3];
    gso_camera_center(camera, cc);
    const v3 cam_center = v3_make(cc[0], cc[1], cc[2]);
    const double tan_fovx = camera->width / (2.0 * camera->fx);
    const double tan_fovy = camera->height / (2.0 * camera->fy);
    const double limx = 1.3 * tan_fovx;
    const double limy = 1.3 * tan_fovy;

    uint64_t visible = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t pi = of_primitive[i];
        const gsim_rigid* node_pose = pi ? &nodes[pi - 1].pose : &identity;
        if (pi && nodes[pi - 1].env >= 0 && nodes[pi - 1].env != camera->env) continue;
        const double* pm = field->means + i * field->means_stride;
        const double* ps = field->scales + i * field->scales_stride;
        const double* pq = field->rotations + i * field->rotations_stride;
        const double opacity = field->opacities[i * field->opacities_stride];
        const double* psh = field->sh + i * field->sh_stride;

        const v3 mean_world = rigid_apply(node_pose, v3_make(pm[0], pm[1], pm[2]));
        const v3 mean_cam = rigid_apply(&camera->pose, mean_world);
        const double z = mean_cam.z;
        if (!(z > camera->near_plane) || !(z < camera->far_plane)) continue;

        const double u = camera->fx * mean_cam.x / z + camera->cx;
        const double v = camera->fy * mean_cam.y / z + camera->cy;

        const quat rot_world = q_mul(rigid_q(node_pose), q_make(pq[0], pq[1], pq[2], pq[3]));
        const mat3 r = q_to_matrix(rot_world);
        const mat3 d = m3_diag(ps[0] * ps[0], ps[1] * ps[1], ps[2] * ps[2]);
        const mat3 rd = m3_mul(&r, &d);
        const mat3 rt = m3_transposed(&r);
        const mat3 cov_world = m3_mul(&rd, &rt);
        const mat3 t1 = m3_mul(&r_wc, &cov_world);
        const mat3 cov_cam = m3_mul(&t1, &r_wc_t);
#define CC(a, b) cov_cam.m[(a) * 3 + (b)]
        const double tx = clampd(mean_cam.x / z, -limx, limx) * z;
        const double ty = clampd(mean_cam.y / z, -limy, limy) * z;
        const double j00 = camera->fx / z;
        const double j02 = -camera->fx * tx / (z * z);
        const double j11 = camera->fy / z;
        const double j12 = -camera->fy * ty / (z * z);

        const double a = j00 * (j00 * CC(0, 0) + j02 * CC(2, 0)) + j02 * (j00 * CC(0, 2) + j02 * CC(2, 2));
        const double b = j00 * (j11 * CC(0, 1) + j12 * CC(0, 2)) + j02 * (j11 * CC(2, 1) + j12 * CC(2, 2));
        const double c = j11 * (j11 * CC(1, 1) + j12 * CC(2, 1)) + j12 * (j11 * CC(1, 2) + j12 * CC(2, 2));
#undef CC
        const double cov_xx = a + kCovarianceFloor;
        const double cov_xy = b;
        const double cov_yy = c + kCovarianceFloor;
        const double det = cov_xx * cov_yy - cov_xy * cov_xy;
        if (!(det > 0.0) || !isfinite(det)) continue;

        const double mid = 0.5 * (cov_xx + cov_yy);
        const double disc = mid * mid - det;
        const double lambda_max = mid + sqrt((0.0 < disc) ? disc : 0.0);
        const double radius = 3.0 * sqrt(lambda_max);
        if (u + radius < 0.0 || u - radius > camera->width || v + radius < 0.0 ||
            v - radius > camera->height)
            continue;

        v3 view_dir = v3_sub(mean_world, cam_center);
        const double dn = v3_norm(view_dir);
        if (dn > 0.0) view_dir = v3_div(view_dir, dn);
        const v3 view_local = q_inverse_rotate(rigid_q(node_pose), view_dir);

        if (visible < capacity && out) {
            gsim_projected_splat* s = &out[visible];
            memset(s, 0, sizeof(*s));
            s->pixel_center[0] = u;
            s->pixel_center[1] = v;
            s->cov_xx = cov_xx; s->cov_xy = cov_xy; s->cov_yy = cov_yy;
            s->inv_xx = cov_yy / det;
            s->inv_xy = -cov_xy / det;
            s->inv_yy = cov_xx / det;
            s->view_depth = z;
            s->alpha_peak = opacity;
            const double vl[3] = {view_local.x, view_local.y, view_local.z};
            gso_shade_sh(psh, field->sh_degree, vl, s->rgb);
            s->radius = radius;
            s->prim_index = (uint32_t)i;
        }
        ++visible;
    }
    free(of_primitive);
    *count = visible;
    return GSIM_OK;
}

typedef struct { uint64_t key; uint32_t value; uint32_t pad; } pair_t;

static int cmp_pair(const void* pa, const void* pb) {
    const pair_t* a = (const pair_t*)pa;
    const pair_t* b = (const pair_t*)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->value != b->value) return a->value < b->value ? -1 : 1;
    return 0;
}

/* Pair emission + std::sort + tile ranges, raster.cpp:174-202. */
static pair_t* build_pairs(const gsim_projected_splat* splats, uint64_t n, int tiles_x,
                           int tiles_y, uint64_t* n_pairs, uint64_t** tile_begin_out) {
    uint64_t cap = 1024, np = 0;
    pair_t* pairs = (pair_t*)malloc(cap * sizeof(pair_t));
    for (uint64_t s = 0; s < n; ++s) {
        const gsim_projected_splat* sp = &splats[s];
        const double u = sp->pixel_center[0], v = sp->pixel_center[1], r = sp->radius;
        int tx0 = (int)floor((u - r) / kTileSize);
        int tx1 = (int)floor((u + r) / kTileSize);
        int ty0 = (int)floor((v - r) / kTileSize);
        int ty1 = (int)floor((v + r) / kTileSize);
        if (tx1 < 0 || tx0 >= tiles_x || ty1 < 0 || ty0 >= tiles_y) continue;
        if (tx0 < 0) tx0 = 0;
        if (ty0 < 0) ty0 = 0;
        if (tx1 > tiles_x - 1) tx1 = tiles_x - 1;
        if (ty1 > tiles_y - 1) ty1 = tiles_y - 1;
        const uint64_t depth_bits = depth_sort_key(sp->view_depth);
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) {
                if (np == cap) {
                    cap *= 2;
                    pairs = (pair_t*)realloc(pairs, cap * sizeof(pair_t));
                }
                const uint64_t tile = (uint64_t)ty * tiles_x + tx;
                pairs[np].key = (tile << 32) | depth_bits;
                pairs[np].value = (uint32_t)s;
                pairs[np].pad = 0;
                ++np;
            }
    }
    qsort(pairs, np, sizeof(pair_t), cmp_pair); /* (key, index) pairs are unique: = std::sort */
    const uint64_t tile_count = (uint64_t)tiles_x * tiles_y;
    uint64_t* tile_begin = (uint64_t*)calloc(tile_count + 1, sizeof(uint64_t));
    for (uint64_t k = 0; k < np; ++k) ++tile_begin[(pairs[k].key >> 32) + 1];
    for (uint64_t t = 1; t <= tile_count; ++t) tile_begin[t] += tile_begin[t - 1];
    *n_pairs = np;
    *tile_begin_out = tile_begin;
    return pairs;
}

static void blend_pixel(const gsim_projected_splat* splats, const pair_t* pairs,
                        uint64_t begin, uint64_t end, const uint32_t* order, int x, int y,
                        const gsim_raster_options* options, const double* q_cut, float* rgb,
                        float* depth, float* alpha) {
    /* raster.cpp:215-249 (pairs != NULL) or reference_raster.cpp:29-65 (order != NULL) */
    const double px = x + 0.5;
    const double py = y + 0.5;
    double cr = 0.0, cg = 0.0, cb = 0.0, d = 0.0, acc = 0.0;
    double transmittance = 1.0;
    for (uint64_t k = begin; k < end; ++k) {
        const uint32_t si = pairs ? pairs[k].value : order[k];
        const gsim_projected_splat* sp = &splats[si];
        const double dx = sp->pixel_center[0] - px;
        const double dy = sp->pixel_center[1] - py;
        if (fabs(dx) > sp->radius || fabs(dy) > sp->radius) continue;
        const double q = sp->inv_xx * dx * dx + 2.0 * sp->inv_xy * dx * dy + sp->inv_yy * dy * dy;
        if (q_cut && q > q_cut[si] + 1e-9) continue;
        const double e = sp->alpha_peak * exp(-0.5 * q);
        const double a = (kAlphaClamp < e) ? kAlphaClamp : e; /* std::min(e, kAlphaClamp) */
        if (a < kAlphaSkip) continue;
        const double w = a * transmittance;
        cr += sp->rgb[0] * w;
        cg += sp->rgb[1] * w;
        cb += sp->rgb[2] * w;
        d += sp->view_depth * w;
        acc += w;
        transmittance *= 1.0 - a;
        if (transmittance < options->transmittance_cutoff) break;
    }
    rgb[0] = (float)clampd(cr, 0.0, 1.0);
    rgb[1] = (float)clampd(cg, 0.0, 1.0);
    rgb[2] = (float)clampd(cb, 0.0, 1.0);
    if (options->normalize_depth)
        *depth = acc > 1e-12 ? (float)(d / acc) : 0.0f;
    else
        *depth = (float)d;
    *alpha = (float)acc;
}

int gso_rasterize(const gsim_projected_splat* splats, uint64_t n, const gsim_camera* camera,
                  const gsim_raster_options* options, float* rgb, float* depth, float* alpha) {
    /* raster.cpp:165-254 (rasterize does not validate the camera) */
    const int width = camera->width, height = camera->height;
    memset(rgb, 0, sizeof(float) * 3 * (size_t)width * height);
    memset(depth, 0, sizeof(float) * (size_t)width * height);
    memset(alpha, 0, sizeof(float) * (size_t)width * height);
    const int tiles_x = (width + kTileSize - 1) / kTileSize;
    const int tiles_y = (height + kTileSize - 1) / kTileSize;
    uint64_t np = 0;
    uint64_t* tile_begin = NULL;
    pair_t* pairs = build_pairs(splats, n, tiles_x, tiles_y, &np, &tile_begin);
    const uint64_t tile_count = (uint64_t)tiles_x * tiles_y;
    for (uint64_t tile = 0; tile < tile_count; ++tile) {
        const uint64_t begin = tile_begin[tile], end = tile_begin[tile + 1];
        if (begin == end) continue;
        const int tx = (int)(tile % tiles_x), ty = (int)(tile / tiles_x);
        const int x0 = tx * kTileSize, y0 = ty * kTileSize;
        const int x1 = x0 + kTileSize < width ? x0 + kTileSize : width;
        const int y1 = y0 + kTileSize < height ? y0 + kTileSize : height;
        for (int y = y0; y < y1; ++y)
            for (int x = x0; x < x1; ++x) {
                const size_t p = (size_t)y * width + x;
                blend_pixel(splats, pairs, begin, end, NULL, x, y, options, NULL, rgb + 3 * p,
                            depth + p, alpha + p);
            }
    }
    free(pairs);
    free(tile_begin);
    return GSIM_OK;
}

int gso_rasterize_lists(const gsim_projected_splat* splats, uint64_t n,
                        const gsim_camera* camera, uint32_t* tile_begin_out, uint32_t* values,
                        uint64_t capacity, uint64_t* count) {
    const int tiles_x = (camera->width + kTileSize - 1) / kTileSize;
    const int tiles_y = (camera->height + kTileSize - 1) / kTileSize;
    uint64_t np = 0;
    uint64_t* tile_begin = NULL;
    pair_t* pairs = build_pairs(splats, n, tiles_x, tiles_y, &np, &tile_begin);
    const uint64_t tile_count = (uint64_t)tiles_x * tiles_y;
    if (tile_begin_out)
        for (uint64_t t = 0; t <= tile_count; ++t) tile_begin_out[t] = (uint32_t)tile_begin[t];
    if (values)
        for (uint64_t k = 0; k < np && k < capacity; ++k) values[k] = pairs[k].value;
    *count = np;
    free(pairs);
    free(tile_begin);
    return GSIM_OK;
}

typedef struct { uint32_t key; uint32_t index; } key_index_t;

static int cmp_key_index(const void* pa, const void* pb) {
    const key_index_t* a = (const key_index_t*)pa;
    const key_index_t* b = (const key_index_t*)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->index < b->index ? -1 : (a->index > b->index ? 1 : 0);
}

int gso_reference_rasterize(const gsim_projected_splat* splats, uint64_t n,
                            const gsim_camera* camera, const gsim_raster_options* options,
                            float* rgb, float* depth, float* alpha) {
    /* reference_raster.cpp:12-67 */
    const int width = camera->width, height = camera->height;
    key_index_t* ki = (key_index_t*)malloc((n ? n : 1) * sizeof(key_index_t));
    for (uint64_t s = 0; s < n; ++s) {
        ki[s].key = depth_sort_key(splats[s].view_depth);
        ki[s].index = (uint32_t)s;
    }
    qsort(ki, n, sizeof(key_index_t), cmp_key_index); /* = stable_sort by key */
    uint32_t* order = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    for (uint64_t s = 0; s < n; ++s) order[s] = ki[s].index;
    free(ki);
    double* q_cut = (double*)malloc((n ? n : 1) * sizeof(double));
    for (uint64_t s = 0; s < n; ++s) {
        const double ap = splats[s].alpha_peak;
        q_cut[s] = 2.0 * log(((ap < 1e-300) ? 1e-300 : ap) / kAlphaSkip);
    }
    for (int y = 0; y < height; ++y)
        for (int x = 0; x < width; ++x) {
            const size_t p = (size_t)y * width + x;
            blend_pixel(splats, NULL, 0, n, order, x, y, options, q_cut, rgb + 3 * p, depth + p,
                        alpha + p);
        }
    free(order);
    free(q_cut);
    return GSIM_OK;
}

int gso_render(const gsim_field_view* field, const gsim_node* nodes, uint64_t n_nodes,
               const gsim_camera* cameras, uint64_t n_cameras,
               const gsim_raster_options* options, gsim_target* outs) {
    /* raster.cpp:256-265: every camera independently; validation before any output. */
    for (uint64_t c = 0; c < n_cameras; ++c)
        if (validate_camera(&cameras[c]) != GSIM_OK) return GSIM_ERR_VALIDATION;
    gsim_projected_splat* splats =
        (gsim_projected_splat*)malloc((field->count ? field->count : 1) * sizeof(gsim_projected_splat));
    for (uint64_t c = 0; c < n_cameras; ++c) {
        uint64_t count = 0;
        const int st = gso_project(field, nodes, n_nodes, &cameras[c], splats, field->count, &count);
        if (st != GSIM_OK) { free(splats); return st; }
        gso_rasterize(splats, count, &cameras[c], options, outs[c].rgb, outs[c].depth,
                      outs[c].accum_alpha);
    }
    free(splats);
    return GSIM_OK;
}

int gso_transform_primitives(double* means, double* rotations, uint64_t count, uint64_t begin,
                             uint64_t end, const gsim_rigid* transform) {
    /* gaussian.cpp:65-79 */
    if (begin > end || end > count) return GSIM_ERR_VALIDATION;
    const quat tq = rigid_q(transform);
    for (uint64_t i = begin; i < end; ++i) {
        double* m = means + 3 * i;
        double* r = rotations + 4 * i;
        const v3 p = rigid_apply(transform, v3_make(m[0], m[1], m[2]));
        m[0] = p.x; m[1] = p.y; m[2] = p.z;
        quat q = q_mul(tq, q_make(r[0], r[1], r[2], r[3]));
        if (fabs(q_norm(q) - 1.0) > 1e-12) q = q_normalized(q);
        r[0] = q.w; r[1] = q.x; r[2] = q.y; r[3] = q.z;
    }
    return GSIM_OK;
}

/* ---- std::mt19937_64 + libstdc++ uniform_real_distribution<double> ---------------------- */

void gso_mt_seed(gso_mt19937_64* rng, uint64_t seed) {
    rng->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        rng->mt[i] = 6364136223846793005ULL * (rng->mt[i - 1] ^ (rng->mt[i - 1] >> 62)) + (uint64_t)i;
    rng->index = 312;
}

uint64_t gso_mt_next(gso_mt19937_64* rng) {
    static const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    if (rng->index >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t y = (rng->mt[i] & upper) | (rng->mt[(i + 1) % 312] & lower);
            uint64_t v = rng->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            rng->mt[i] = v;
        }
        rng->index = 0;
    }
    uint64_t x = rng->mt[rng->index++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

double gso_uniform_real(gso_mt19937_64* rng, double a, double b) {
    /* std::generate_canonical<double, 53> with a 64-bit engine takes one draw:
     * (double)x / 2^64, pulled below 1 if it rounds up (libstdc++ random.tcc). */
    double r = (double)gso_mt_next(rng) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r * (b - a) + a;
}

void gso_random_field(uint64_t seed, uint64_t count, double box_extent, double scale_lo,
                      double scale_hi, int sh_degree, double* means, double* scales,
                      double* rotations, double* opacities, double* sh) {
    /* oracle::random_field, tests/support/test_oracles.cpp:144-168 */
    gso_mt19937_64 rng;
    gso_mt_seed(&rng, seed);
    const double plo = -box_extent / 2, phi = box_extent / 2;
    const int coeffs = (sh_degree + 1) * (sh_degree + 1);
    for (uint64_t i = 0; i < count; ++i) {
        for (int k = 0; k < 3; ++k) means[3 * i + k] = gso_uniform_real(&rng, plo, phi);
        for (int k = 0; k < 3; ++k) scales[3 * i + k] = gso_uniform_real(&rng, scale_lo, scale_hi);
        quat q;
        q.w = gso_uniform_real(&rng, -1.0, 1.0);
        q.x = gso_uniform_real(&rng, -1.0, 1.0);
        q.y = gso_uniform_real(&rng, -1.0, 1.0);
        q.z = gso_uniform_real(&rng, -1.0, 1.0);
        while (q_norm(q) < 1e-3) {
            q.w = gso_uniform_real(&rng, -1.0, 1.0);
            q.x = gso_uniform_real(&rng, -1.0, 1.0);
            q.y = gso_uniform_real(&rng, -1.0, 1.0);
            q.z = gso_uniform_real(&rng, -1.0, 1.0);
        }
        q = q_normalized(q);
        rotations[4 * i + 0] = q.w; rotations[4 * i + 1] = q.x;
        rotations[4 * i + 2] = q.y; rotations[4 * i + 3] = q.z;
        opacities[i] = gso_uniform_real(&rng, 0.2, 0.95);
        double* s = sh + 48 * i;
        memset(s, 0, 48 * sizeof(double));
        for (int c = 0; c < 3; ++c)
            for (int k = 0; k < coeffs; ++k) s[c * 16 + k] = gso_uniform_real(&rng, -0.6, 0.6);
    }
}

/* ---- hash.hpp restated ------------------------------------------------------------------ */

uint64_t gso_hash_bytes(const void* data, uint64_t size, uint64_t seed) {
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = seed;
    for (uint64_t i = 0; i < size; ++i) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    return h;
}

static uint64_t hash_image(const float* data, int width, int height, int channels, uint64_t seed) {
    const int32_t dims[2] = {width, height};
    const uint64_t h = gso_hash_bytes(dims, sizeof(dims), seed);
    return gso_hash_bytes(data, (uint64_t)width * height * channels * sizeof(float), h);
}

uint64_t gso_hash_target(const float* rgb, const float* depth, const float* alpha, int width,
                         int height, uint64_t seed) {
    uint64_t h = hash_image(rgb, width, height, 3, seed);
    h = hash_image(depth, width, height, 1, h);
    return hash_image(alpha, width, height, 1, h);
}

/* ---- output encoding ------------------------------------------------------------------------ */

double gso_linear_to_srgb(double v) { /* image_io.cpp:19-22 */
    v = clampd(v, 0.0, 1.0);
    return v <= 0.0031308 ? 12.92 * v : 1.055 * pow(v, 1.0 / 2.4) - 0.055;
}

static uint8_t quantize8(double v) { /* image_io.cpp:43-45 */
    const long r = lround(v * 255.0);
    return (uint8_t)(r < 0 ? 0 : (r > 255 ? 255 : r));
}

uint64_t gso_encoded_bytes(uint32_t flags, int width, int height) {
    const uint64_t bpp = ((flags & GSIM_ENCODE_RGB8) ? 3u : 0u) + ((flags & GSIM_ENCODE_ALPHA8) ? 1u : 0u) +
                         ((flags & GSIM_ENCODE_DEPTH16) ? 2u : 0u) + ((flags & GSIM_ENCODE_DEPTH_PFM) ? 4u : 0u);
    return bpp * (uint64_t)width * (uint64_t)height;
}

int gso_encode(uint32_t flags, int srgb, double depth_scale, int width, int height,
               const float* rgb, const float* depth, const float* alpha, uint8_t* out) {
    if (width <= 0 || height <= 0) return GSIM_ERR_VALIDATION; /* "empty image" */
    const size_t npx = (size_t)width * (size_t)height;
    uint8_t* part = out;
    if (flags & GSIM_ENCODE_RGB8) { /* write_png_rgb8, image_io.cpp:75-86 */
        for (size_t i = 0; i < 3 * npx; ++i) {
            const double v = rgb[i];
            part[i] = quantize8(srgb ? gso_linear_to_srgb(v) : clampd(v, 0.0, 1.0));
        }
        part += 3 * npx;
    }
    if (flags & GSIM_ENCODE_ALPHA8) { /* write_png_gray8, image_io.cpp:88-97 */
        for (size_t i = 0; i < npx; ++i) part[i] = quantize8(clampd((double)alpha[i], 0.0, 1.0));
        part += npx;
    }
    if (flags & GSIM_ENCODE_DEPTH16) { /* write_png_gray16, image_io.cpp:99-111 */
        for (size_t i = 0; i < npx; ++i) {
            long v = lround(depth[i] * depth_scale);
            v = v < 0 ? 0 : (v > 65535 ? 65535 : v);
            part[2 * i] = (uint8_t)(v >> 8);
            part[2 * i + 1] = (uint8_t)(v & 0xff);
        }
        part += 2 * npx;
    }
    if (flags & GSIM_ENCODE_DEPTH_PFM) { /* write_pfm body, image_io.cpp:166-178 */
        for (int y = height - 1, r = 0; y >= 0; --y, ++r)
            memcpy(part + (size_t)r * width * 4, depth + (size_t)y * width, (size_t)width * 4);
    }
    return GSIM_OK;
}

/* ---- pose playback -------------------------------------------------------------------------- */

static quat slerp_q(quat a, quat b, double t) { /* math.hpp:195-214 */
    double cos_half = a.w * b.w + a.x * b.x + a.y * b.y + a.z * b.z;
    if (cos_half < 0.0) {
        b = q_make(-b.w, -b.x, -b.y, -b.z);
        cos_half = -cos_half;
    }
    if (cos_half > 1.0 - 1e-12) {
        const quat q = q_make(a.w + t * (b.w - a.w), a.x + t * (b.x - a.x), a.y + t * (b.y - a.y),
                              a.z + t * (b.z - a.z));
        return q_normalized(q);
    }
    const double half = acos(cos_half);
    const double s = sin(half);
    const double wa = sin((1.0 - t) * half) / s;
    const double wb = sin(t * half) / s;
    const quat q = q_make(wa * a.w + wb * b.w, wa * a.x + wb * b.x, wa * a.y + wb * b.y,
                          wa * a.z + wb * b.z);
    return q_normalized(q);
}

void gso_slerp(const double a[4], const double b[4], double t, double out[4]) {
    const quat q = slerp_q(q_make(a[0], a[1], a[2], a[3]), q_make(b[0], b[1], b[2], b[3]), t);
    out[0] = q.w;
    out[1] = q.x;
    out[2] = q.y;
    out[3] = q.z;
}

int gso_pose_sample(const double* rec_t, const double* rec_p, const double* rec_q, uint64_t n_rec,
                    const gsim_rigid* initial, const double* ts, uint64_t n_t, gsim_rigid* out) {
    /* PoseStream::append (pose_stream.cpp:31-40): finite checks, non-decreasing times,
     * rotation normalised on append. */
    for (uint64_t i = 0; i < n_rec; ++i) {
        if (!isfinite(rec_t[i])) return GSIM_ERR_VALIDATION;
        for (int k = 0; k < 3; ++k) if (!isfinite(rec_p[3 * i + k])) return GSIM_ERR_VALIDATION;
        for (int k = 0; k < 4; ++k) if (!isfinite(rec_q[4 * i + k])) return GSIM_ERR_VALIDATION;
        if (i && rec_t[i] < rec_t[i - 1]) return GSIM_ERR_VALIDATION;
    }
    for (uint64_t k = 0; k < n_t; ++k) { /* PoseStream::sample, pose_stream.cpp:117-136 */
        const double t = ts[k];
        gsim_rigid* o = &out[k];
        if (n_rec == 0 || t < rec_t[0]) { *o = *initial; continue; }
        const uint64_t last = n_rec - 1;
        const quat ql = q_normalized(q_make(rec_q[4 * last], rec_q[4 * last + 1], rec_q[4 * last + 2],
                                            rec_q[4 * last + 3]));
        if (t >= rec_t[last]) {
            o->rotation[0] = ql.w; o->rotation[1] = ql.x; o->rotation[2] = ql.y; o->rotation[3] = ql.z;
            for (int c = 0; c < 3; ++c) o->translation[c] = rec_p[3 * last + c];
            continue;
        }
        uint64_t lo_i = 0, hi_i = n_rec; /* first record with time > t (upper_bound) */
        while (lo_i < hi_i) {
            const uint64_t mid = lo_i + (hi_i - lo_i) / 2;
            if (t < rec_t[mid]) hi_i = mid; else lo_i = mid + 1;
        }
        const uint64_t hi = lo_i, lo = hi - 1;
        const quat qh = q_normalized(q_make(rec_q[4 * hi], rec_q[4 * hi + 1], rec_q[4 * hi + 2], rec_q[4 * hi + 3]));
        const double span = rec_t[hi] - rec_t[lo];
        if (span <= 0.0) {
            o->rotation[0] = qh.w; o->rotation[1] = qh.x; o->rotation[2] = qh.y; o->rotation[3] = qh.z;
            for (int c = 0; c < 3; ++c) o->translation[c] = rec_p[3 * hi + c];
            continue;
        }
        const double u = (t - rec_t[lo]) / span;
        for (int c = 0; c < 3; ++c) o->translation[c] = rec_p[3 * lo + c] * (1.0 - u) + rec_p[3 * hi + c] * u;
        const quat qlo = q_normalized(q_make(rec_q[4 * lo], rec_q[4 * lo + 1], rec_q[4 * lo + 2], rec_q[4 * lo + 3]));
        const quat q = slerp_q(qlo, qh, u);
        o->rotation[0] = q.w; o->rotation[1] = q.x; o->rotation[2] = q.y; o->rotation[3] = q.z;
    }
    return GSIM_OK;
}

/* ---- splat PLY (splat_ply.cpp:40-162) -------------------------------------------------------- */

static int read_line(FILE* f, char* buf, size_t cap) { /* std::getline: up to '\n' */
    size_t n = 0;
    int ch;
    while ((ch = fgetc(f)) != EOF && ch != '\n')
        if (n + 1 < cap) buf[n++] = (char)ch;
    buf[n] = 0;
    return !(ch == EOF && n == 0);
}

int gso_load_splat_ply(const char* path, uint64_t capacity, uint64_t* count_out, int* degree_out,
                       double* means, double* scales, double* rotations, double* opacities,
                       double* sh) {
    FILE* f = fopen(path, "rb");
    if (!f) return GSIM_ERR_IO;
    char line[512];
    int rc = GSIM_ERR_VALIDATION;
    char props[80][32];
    int n_props = 0, format_seen = 0, element_seen = 0, closed = 0;
    unsigned long long count = 0;
    float* payload = NULL;
    if (!read_line(f, line, sizeof line) || strcmp(line, "ply") != 0) goto done;
    while (read_line(f, line, sizeof line)) {
        size_t L = strlen(line);
        if (L && line[L - 1] == '\r') line[--L] = 0;
        if (strcmp(line, "end_header") == 0) { closed = 1; break; }
        char tok[64] = "", a[64] = "", b[64] = "";
        sscanf(line, "%63s %63s %63s", tok, a, b);
        if (strcmp(tok, "comment") == 0) continue;
        if (strcmp(tok, "format") == 0) {
            if (strcmp(a, "binary_little_endian") != 0) goto done;
            format_seen = 1;
        } else if (strcmp(tok, "element") == 0) {
            if (strcmp(a, "vertex") != 0) goto done;
            count = strtoull(b, NULL, 10);
            element_seen = 1;
        } else if (strcmp(tok, "property") == 0) {
            if (strcmp(a, "float") != 0 || n_props >= 80) goto done;
            snprintf(props[n_props++], sizeof props[0], "%s", b);
        } else if (tok[0]) {
            goto done;
        }
    }
    if (!closed || !format_seen || !element_seen) goto done;
    int rest = 0;
    for (int i = 0; i < n_props; ++i) if (strncmp(props[i], "f_rest_", 7) == 0) ++rest;
    int degree = -1;
    for (int d = 0; d <= 3; ++d) if (rest == 3 * ((d + 1) * (d + 1) - 1)) degree = d;
    if (degree < 0) goto done;
    const int K = (degree + 1) * (degree + 1), rpc = K - 1;
    const int stride = 17 + 3 * rpc;
    if (n_props != stride) goto done;
    { /* expected property names and order */
        static const char* head[9] = {"x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"};
        static const char* tail[8] = {"opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"};
        char want[32];
        for (int i = 0; i < stride; ++i) {
            if (i < 9) snprintf(want, sizeof want, "%s", head[i]);
            else if (i < 9 + 3 * rpc) snprintf(want, sizeof want, "f_rest_%d", i - 9);
            else snprintf(want, sizeof want, "%s", tail[i - 9 - 3 * rpc]);
            if (strcmp(props[i], want) != 0) goto done;
        }
    }
    const size_t nfl = (size_t)count * (size_t)stride;
    if (count) {
        payload = (float*)malloc(nfl * sizeof(float));
        if (!payload) { rc = GSIM_ERR_IO; goto done; }
        if (fread(payload, sizeof(float), nfl, f) != nfl) goto done; /* truncated */
    }
    for (uint64_t i = 0; i < count; ++i) {
        const float* row = payload + i * (size_t)stride;
        for (int k = 0; k < stride; ++k) if (!isfinite(row[k])) goto done;
        const float* t = row + 9 + 3 * rpc;
        const double op = 1.0 / (1.0 + exp(-(double)t[0]));
        if (op <= 0.0 || op >= 1.0) goto done;
        const double s0 = exp((double)t[1]), s1 = exp((double)t[2]), s2 = exp((double)t[3]);
        if (!isfinite(s0) || !isfinite(s1) || !isfinite(s2)) goto done;
        quat q = q_make(t[4], t[5], t[6], t[7]);
        const double n = q_norm(q);
        if (!(n > 0.0) || !isfinite(n)) goto done;
        if (fabs(n - 1.0) > 1e-6) q = q_normalized(q);
        if (count <= capacity) {
            for (int c = 0; c < 3; ++c) means[3 * i + c] = row[c];
            scales[3 * i] = s0; scales[3 * i + 1] = s1; scales[3 * i + 2] = s2;
            rotations[4 * i] = q.w; rotations[4 * i + 1] = q.x;
            rotations[4 * i + 2] = q.y; rotations[4 * i + 3] = q.z;
            opacities[i] = op;
            double* o = sh + 48 * i;
            for (int k = 0; k < 48; ++k) o[k] = 0.0;
            for (int c = 0; c < 3; ++c) {
                o[c * 16] = row[6 + c];
                for (int k = 0; k < rpc; ++k) o[c * 16 + k + 1] = row[9 + c * rpc + k];
            }
        }
    }
    *count_out = count;
    *degree_out = degree;
    rc = GSIM_OK;
done:
    free(payload);
    fclose(f);
    return rc;
}


/* ---- GS -> TSDF (transfer.cpp) ------------------------------------------------------------ */

static const double kPiD = 3.14159265358979323846; /* math.hpp:265-266 */
static const double kBoundsSigma = 3.0;            /* trace.hpp:25 */
static const double kDepthValidAlpha = 0.5;        /* transfer.cpp:23 */
static const double kRingRadiusFactor = 2.5;       /* transfer.cpp:24 */
static const int kFusionAzimuths = 20;             /* transfer.cpp:25 */
static const int kFusionResolution = 256;          /* transfer.cpp:26 */

void gso_field_bounds(const gsim_field_view* field, double lo[3], double hi[3]) {
    /* field_bounds (transfer.cpp:27-34): Aabb::expand (math.hpp:249-250, fmin / fmax) of
     * pose_primitive(p, identity).bounds (trace.cpp:14-36). The identity pose leaves mean and
     * rotation bit-exact. */
    for (int k = 0; k < 3; ++k) { lo[k] = INFINITY; hi[k] = -INFINITY; }
    for (uint64_t i = 0; i < field->count; ++i) {
        const double* pm = field->means + i * field->means_stride;
        const double* ps = field->scales + i * field->scales_stride;
        const double* pq = field->rotations + i * field->rotations_stride;
        const quat id = q_make(1.0, 0.0, 0.0, 0.0);
        const quat rot = q_mul(id, q_make(pq[0], pq[1], pq[2], pq[3]));
        const mat3 r = q_to_matrix(rot);
        const mat3 d = m3_diag(ps[0] * ps[0], ps[1] * ps[1], ps[2] * ps[2]);
        const mat3 rd = m3_mul(&r, &d);
        const mat3 rt = m3_transposed(&r);
        const mat3 cov = m3_mul(&rd, &rt);
        const double half[3] = {kBoundsSigma * sqrt(cov.m[0]), kBoundsSigma * sqrt(cov.m[4]),
                                kBoundsSigma * sqrt(cov.m[8])};
        gsim_rigid identity;
        memset(&identity, 0, sizeof(identity));
        identity.rotation[0] = 1.0;
        const v3 mean = rigid_apply(&identity, v3_make(pm[0], pm[1], pm[2]));
        const double m[3] = {mean.x, mean.y, mean.z};
        double blo[3], bhi[3];
        for (int k = 0; k < 3; ++k) { blo[k] = INFINITY; bhi[k] = -INFINITY; }
        for (int k = 0; k < 3; ++k) { /* bounds.expand(mean - half); bounds.expand(mean + half) */
            const double a = m[k] - half[k], b = m[k] + half[k];
            blo[k] = fmin(blo[k], a); bhi[k] = fmax(bhi[k], a);
            blo[k] = fmin(blo[k], b); bhi[k] = fmax(bhi[k], b);
        }
        for (int k = 0; k < 3; ++k) { lo[k] = fmin(lo[k], blo[k]); hi[k] = fmax(hi[k], bhi[k]); }
    }
}

int gso_depth_ring_cameras(const double lo_[3], const double hi_[3], int n_views, double radius,
                           int resolution, gsim_camera* cameras) {
    /* render_depth_ring camera set-up, transfer.cpp:84-112 */
    if (n_views < 8) return GSIM_ERR_VALIDATION;
    if (!(radius > 0.0)) return GSIM_ERR_VALIDATION;
    const v3 lo = v3_make(lo_[0], lo_[1], lo_[2]), hi = v3_make(hi_[0], hi_[1], hi_[2]);
    const v3 extent = v3_sub(hi, lo);
    const double diag = v3_norm(extent);
    if (!(diag > 0.0)) return GSIM_ERR_VALIDATION;
    const v3 center = v3_scale(v3_add(lo, hi), 0.5);
    const double tan_half = 0.65 * diag / radius;
    const double focal = 0.5 * resolution / tan_half;
    const double elevations[3] = {-kPiD / 6.0, 0.0, kPiD / 6.0};
    const double up[3] = {0.0, 0.0, 1.0}; /* camera.hpp:32 default */
    const double c[3] = {center.x, center.y, center.z};
    int v = 0;
    for (int e = 0; e < 3; ++e) {
        const double elevation = elevations[e];
        for (int k = 0; k < n_views; ++k, ++v) {
            const double azimuth = 2.0 * kPiD * k / n_views;
            const v3 dir = v3_make(cos(elevation) * cos(azimuth), cos(elevation) * sin(azimuth),
                                   sin(elevation));
            const v3 eye = v3_add(center, v3_scale(dir, radius));
            const double ev[3] = {eye.x, eye.y, eye.z};
            gso_look_at(ev, c, focal, focal, resolution, resolution, up, &cameras[v]);
            /* std::max(1e-4, radius - diag) */
            cameras[v].near_plane = (1e-4 < radius - diag) ? radius - diag : 1e-4;
            cameras[v].far_plane = radius + diag;
        }
    }
    return GSIM_OK;
}

int gso_render_depth_ring(const gsim_field_view* field, int n_views, double radius,
                          int resolution, gsim_camera* cameras, float* depth) {
    /* transfer.cpp:81-124 */
    if (field->count == 0) return GSIM_ERR_VALIDATION;
    if (n_views < 8) return GSIM_ERR_VALIDATION;
    if (!(radius > 0.0)) return GSIM_ERR_VALIDATION;
    double lo[3], hi[3];
    gso_field_bounds(field, lo, hi);
    const int st = gso_depth_ring_cameras(lo, hi, n_views, radius, resolution, cameras);
    if (st != GSIM_OK) return st;
    const uint64_t npx = (uint64_t)resolution * resolution;
    gsim_raster_options opt;
    memset(&opt, 0, sizeof(opt));
    opt.normalize_depth = 1;
    opt.transmittance_cutoff = 1e-4;
    float* rgb = (float*)malloc(npx * 3 * sizeof(float));
    float* alpha = (float*)malloc(npx * sizeof(float));
    for (int v = 0; v < 3 * n_views; ++v) {
        gsim_target t;
        memset(&t, 0, sizeof(t));
        t.rgb = rgb;
        t.depth = depth + (uint64_t)v * npx;
        t.accum_alpha = alpha;
        const int r = gso_render(field, NULL, 0, &cameras[v], 1, &opt, &t);
        if (r != GSIM_OK) { free(rgb); free(alpha); return r; }
        for (uint64_t i = 0; i < npx; ++i)
            if (alpha[i] < kDepthValidAlpha) t.depth[i] = 0.0f;
    }
    free(rgb);
    free(alpha);
    return GSIM_OK;
}

int gso_tsdf_create(const double origin[3], double voxel_size, const int32_t dims[3],
                    double truncation, gsim_tsdf_volume* v) {
    /* TsdfVolume::create, transfer.cpp:126-141 */
    if (!(voxel_size > 0.0)) return GSIM_ERR_VALIDATION;
    if (dims[0] < 2 || dims[1] < 2 || dims[2] < 2) return GSIM_ERR_VALIDATION;
    if (truncation < 2.0 * voxel_size) return GSIM_ERR_VALIDATION;
    for (int k = 0; k < 3; ++k) { v->origin[k] = origin[k]; v->dims[k] = dims[k]; }
    v->voxel_size = voxel_size;
    v->truncation = truncation;
    const uint64_t n = (uint64_t)dims[0] * dims[1] * dims[2];
    if (v->tsdf) for (uint64_t i = 0; i < n; ++i) v->tsdf[i] = 1.0;
    if (v->weights) for (uint64_t i = 0; i < n; ++i) v->weights[i] = 0.0;
    return GSIM_OK;
}

static int x86_trunc_int(double x) { /* static_cast<int>(double) as cvttsd2si computes it */
    if (!(x >= -2147483648.0 && x < 2147483648.0)) return INT32_MIN;
    return (int)x;
}

int gso_tsdf_fuse(gsim_tsdf_volume* vol, const gsim_camera* camera, const float* depth,
                  int width, int height) {
    /* tsdf_fuse, transfer.cpp:143-172 */
    if (validate_camera(camera) != GSIM_OK) return GSIM_ERR_VALIDATION;
    if (width != camera->width || height != camera->height) return GSIM_ERR_VALIDATION;
    const int dx = vol->dims[0], dy = vol->dims[1], dz = vol->dims[2];
    uint64_t idx = 0;
    for (int z = 0; z < dz; ++z) {
        for (int y = 0; y < dy; ++y) {
            for (int x = 0; x < dx; ++x, ++idx) {
                /* voxel_center, transfer.hpp:53-56 */
                const v3 p = v3_add(v3_make(vol->origin[0], vol->origin[1], vol->origin[2]),
                                    v3_make((x + 0.5) * vol->voxel_size, (y + 0.5) * vol->voxel_size,
                                            (z + 0.5) * vol->voxel_size));
                const v3 cp = rigid_apply(&camera->pose, p);
                if (cp.z <= 0.0) continue;
                const int px = x86_trunc_int(floor(camera->fx * cp.x / cp.z + camera->cx));
                const int py = x86_trunc_int(floor(camera->fy * cp.y / cp.z + camera->cy));
                if (px < 0 || px >= width || py < 0 || py >= height) continue;
                const double measured = depth[(uint64_t)py * width + px];
                if (measured <= 0.0) continue;
                const double sdf = measured - cp.z;
                if (sdf <= -vol->truncation) continue;
                const double clamped = clampd(sdf / vol->truncation, -1.0, 1.0);
                const double w = vol->weights[idx];
                vol->tsdf[idx] = (vol->tsdf[idx] * w + clamped) / (w + 1.0);
                vol->weights[idx] = w + 1.0;
            }
        }
    }
    return GSIM_OK;
}

int gso_gaussians_to_tsdf(const gsim_field_view* field, double voxel_size, gsim_tsdf_volume* vol) {
    /* gaussians_to_mesh up to the fused volume, transfer.cpp:174-198 */
    if (field->count == 0) return GSIM_ERR_VALIDATION;
    if (!(voxel_size > 0.0)) return GSIM_ERR_VALIDATION;
    double blo[3], bhi[3];
    gso_field_bounds(field, blo, bhi);
    const v3 bl = v3_make(blo[0], blo[1], blo[2]), bh = v3_make(bhi[0], bhi[1], bhi[2]);
    const double diag = v3_norm(v3_sub(bh, bl));
    if (!(diag > 0.0)) return GSIM_ERR_VALIDATION;
    const double truncation = 3.0 * voxel_size;
    const double margin = truncation + 2.0 * voxel_size;
    const v3 lo = v3_sub(bl, v3_make(margin, margin, margin));
    const v3 hi = v3_add(bh, v3_make(margin, margin, margin));
    const v3 extent = v3_sub(hi, lo);
    const double ext[3] = {extent.x, extent.y, extent.z};
    int32_t dims[3];
    for (int k = 0; k < 3; ++k) {
        const int d = x86_trunc_int(ceil(ext[k] / voxel_size)) + 1;
        dims[k] = d > 2 ? d : 2;
    }
    const double origin[3] = {lo.x, lo.y, lo.z};
    int st = gso_tsdf_create(origin, voxel_size, dims, truncation, vol);
    if (st != GSIM_OK || !vol->tsdf) return st; /* geometry-only call */
    const double radius = kRingRadiusFactor * diag;
    const int nv = 3 * kFusionAzimuths;
    const uint64_t npx = (uint64_t)kFusionResolution * kFusionResolution;
    gsim_camera* cams = (gsim_camera*)calloc(nv, sizeof(gsim_camera));
    float* depth = (float*)malloc(npx * nv * sizeof(float));
    st = gso_render_depth_ring(field, kFusionAzimuths, radius, kFusionResolution, cams, depth);
    for (int v = 0; st == GSIM_OK && v < nv; ++v)
        st = gso_tsdf_fuse(vol, &cams[v], depth + (uint64_t)v * npx, kFusionResolution,
                           kFusionResolution);
    free(cams);
    free(depth);
    return st;
}


/* ---- LiDAR (trace.cpp) ------------------------------------------------------------------- */

typedef struct {
    v3 mean;
    mat3 inv_cov;
    double opacity;
    v3 lo, hi;
    int seen;
} posed_t;

static const double kTraceScaleFloor = 1e-7; /* trace.hpp:24 */

static posed_t pose_primitive(const gsim_field_view* f, uint64_t i, const gsim_rigid* pose) {
    /* trace.cpp:14-36 */
    posed_t o;
    const double* pm = f->means + i * f->means_stride;
    const double* ps = f->scales + i * f->scales_stride;
    const double* pq = f->rotations + i * f->rotations_stride;
    o.mean = rigid_apply(pose, v3_make(pm[0], pm[1], pm[2]));
    o.opacity = f->opacities[i * f->opacities_stride];
    const quat rot = q_mul(rigid_q(pose), q_make(pq[0], pq[1], pq[2], pq[3]));
    const mat3 r = q_to_matrix(rot);
    const mat3 rt = m3_transposed(&r);
    /* std::max(scale, kTraceScaleFloor) */
    const double sx = (ps[0] < kTraceScaleFloor) ? kTraceScaleFloor : ps[0];
    const double sy = (ps[1] < kTraceScaleFloor) ? kTraceScaleFloor : ps[1];
    const double sz = (ps[2] < kTraceScaleFloor) ? kTraceScaleFloor : ps[2];
    const mat3 di = m3_diag(1.0 / (sx * sx), 1.0 / (sy * sy), 1.0 / (sz * sz));
    const mat3 rdi = m3_mul(&r, &di);
    o.inv_cov = m3_mul(&rdi, &rt);
    const mat3 d = m3_diag(ps[0] * ps[0], ps[1] * ps[1], ps[2] * ps[2]);
    const mat3 rd = m3_mul(&r, &d);
    const mat3 cov = m3_mul(&rd, &rt);
    const double hx = kBoundsSigma * sqrt(cov.m[0]), hy = kBoundsSigma * sqrt(cov.m[4]),
                 hz = kBoundsSigma * sqrt(cov.m[8]);
    const v3 a = v3_make(o.mean.x - hx, o.mean.y - hy, o.mean.z - hz);
    const v3 b = v3_make(o.mean.x + hx, o.mean.y + hy, o.mean.z + hz);
    o.lo = v3_make(fmin(fmin(INFINITY, a.x), b.x), fmin(fmin(INFINITY, a.y), b.y),
                   fmin(fmin(INFINITY, a.z), b.z));
    o.hi = v3_make(fmax(fmax(-INFINITY, a.x), b.x), fmax(fmax(-INFINITY, a.y), b.y),
                   fmax(fmax(-INFINITY, a.z), b.z));
    o.seen = 1;
    return o;
}

static int ray_aabb_hit(v3 lo, v3 hi, v3 origin, v3 inv, double t_max) { /* bvh.hpp:20-36 */
    double t0 = 0.0, t1 = t_max;
    const double tx0 = (lo.x - origin.x) * inv.x, tx1 = (hi.x - origin.x) * inv.x;
    t0 = fmax(t0, fmin(tx0, tx1));
    t1 = fmin(t1, fmax(tx0, tx1));
    const double ty0 = (lo.y - origin.y) * inv.y, ty1 = (hi.y - origin.y) * inv.y;
    t0 = fmax(t0, fmin(ty0, ty1));
    t1 = fmin(t1, fmax(ty0, ty1));
    const double tz0 = (lo.z - origin.z) * inv.z, tz1 = (hi.z - origin.z) * inv.z;
    t0 = fmax(t0, fmin(tz0, tz1));
    t1 = fmin(t1, fmax(tz0, tz1));
    return t0 <= t1;
}

static v3 m3_apply(const mat3* m, v3 v) { /* Mat3 * Vec3, math.hpp:87-90 */
    return v3_make(m->m[0] * v.x + m->m[1] * v.y + m->m[2] * v.z,
                   m->m[3] * v.x + m->m[4] * v.y + m->m[5] * v.z,
                   m->m[6] * v.x + m->m[7] * v.y + m->m[8] * v.z);
}

typedef struct { double t, response; uint32_t index; } cand_t;

static int cand_cmp(const void* pa, const void* pb) { /* trace.cpp:66-68 */
    const cand_t* a = (const cand_t*)pa;
    const cand_t* b = (const cand_t*)pb;
    if (a->t != b->t) return a->t < b->t ? -1 : 1;
    return a->index < b->index ? -1 : (a->index > b->index ? 1 : 0);
}

static void trace_one(const posed_t* posed, uint64_t n, v3 origin, v3 dir, double t_max,
                      double alpha_threshold, cand_t* buf, uint8_t* hit, double* depth,
                      double* accum) {
    /* trace_linear (trace.cpp:125-134) + ray_gaussian_peak (:38-49) + composite (:65-85) */
    const v3 inv = v3_make(1.0 / dir.x, 1.0 / dir.y, 1.0 / dir.z);
    uint64_t nc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const posed_t* p = &posed[i];
        if (!p->seen) continue;
        if (!ray_aabb_hit(p->lo, p->hi, origin, inv, t_max)) continue;
        const v3 to_mean = v3_sub(p->mean, origin);
        const v3 si_d = m3_apply(&p->inv_cov, dir);
        const double denom = v3_dot(dir, si_d);
        cand_t c = {0.0, 0.0, (uint32_t)i};
        if (denom > 0.0) {
            c.t = clampd(v3_dot(to_mean, si_d) / denom, 0.0, t_max);
            const v3 delta = v3_sub(v3_add(origin, v3_scale(dir, c.t)), p->mean);
            const double q = v3_dot(delta, m3_apply(&p->inv_cov, delta));
            c.response = p->opacity * exp(-0.5 * q);
        }
        buf[nc++] = c;
    }
    qsort(buf, nc, sizeof(cand_t), cand_cmp);
    double depth_sum = 0.0, acc = 0.0, transmittance = 1.0;
    for (uint64_t k = 0; k < nc; ++k) {
        const double alpha = buf[k].response < 0.99 ? buf[k].response : 0.99;
        if (alpha < 1.0 / 255.0) continue;
        const double w = alpha * transmittance;
        depth_sum += buf[k].t * w;
        acc += w;
        transmittance *= 1.0 - alpha;
        if (transmittance < 1e-4) break;
    }
    *accum = acc;
    *hit = acc >= alpha_threshold;
    *depth = *hit ? depth_sum / acc : 0.0;
}

static posed_t* pose_all(const gsim_field_view* field, const gsim_node* nodes, uint64_t n_nodes,
                         int env, int* status) {
    /* GaussianBvh::build, trace.cpp:88-111 */
    const uint64_t n = field->count;
    int64_t* pose_of = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
    for (uint64_t i = 0; i < n; ++i) pose_of[i] = -1;
    for (uint64_t k = 0; k < n_nodes; ++k) {
        if (nodes[k].end > n) { free(pose_of); *status = GSIM_ERR_VALIDATION; return NULL; }
        for (uint64_t i = nodes[k].begin; i < nodes[k].end; ++i) pose_of[i] = (int64_t)k;
    }
    gsim_rigid identity;
    memset(&identity, 0, sizeof(identity));
    identity.rotation[0] = 1.0;
    posed_t* posed = (posed_t*)malloc((n ? n : 1) * sizeof(posed_t));
    for (uint64_t i = 0; i < n; ++i) {
        const int64_t k = pose_of[i];
        posed[i] = pose_primitive(field, i, k >= 0 ? &nodes[k].pose : &identity);
        if (k >= 0 && nodes[k].env >= 0 && nodes[k].env != env) posed[i].seen = 0;
    }
    free(pose_of);
    *status = GSIM_OK;
    return posed;
}

int gso_trace_rays(const gsim_field_view* field, const gsim_node* nodes, uint64_t n_nodes,
                   const double* origins, const double* directions, const double* t_max,
                   uint64_t n_rays, double alpha_threshold, uint8_t* hit, double* depth,
                   double* accum_alpha) {
    int st;
    posed_t* posed = pose_all(field, nodes, n_nodes, -1, &st);
    if (!posed) return st;
    cand_t* buf = (cand_t*)malloc((field->count ? field->count : 1) * sizeof(cand_t));
    for (uint64_t r = 0; r < n_rays; ++r)
        trace_one(posed, field->count,
                  v3_make(origins[3 * r], origins[3 * r + 1], origins[3 * r + 2]),
                  v3_make(directions[3 * r], directions[3 * r + 1], directions[3 * r + 2]),
                  t_max[r], alpha_threshold, buf, &hit[r], &depth[r], &accum_alpha[r]);
    free(buf);
    free(posed);
    return GSIM_OK;
}

static int validate_lidar(const gsim_lidar* l) { /* trace.cpp:136-155 */
    if (l->n_channels == 0) return GSIM_ERR_VALIDATION;
    for (uint64_t c = 0; c < l->n_channels; ++c)
        if (!isfinite(l->channels[c])) return GSIM_ERR_VALIDATION;
    if (!(l->azimuth_step > 0.0)) return GSIM_ERR_VALIDATION;
    const double n = 2.0 * kPiD / l->azimuth_step;
    if (fabs(n - round(n)) * l->azimuth_step > 1e-9) return GSIM_ERR_VALIDATION;
    if (!(l->max_range > 0.0)) return GSIM_ERR_VALIDATION;
    if (!(l->alpha_threshold > 0.0) || l->alpha_threshold > 1.0) return GSIM_ERR_VALIDATION;
    return GSIM_OK;
}

int gso_lidar_scan(const gsim_field_view* field, const gsim_node* nodes, uint64_t n_nodes,
                   const gsim_lidar* lidar, double* points, uint32_t* ring, double* azimuth,
                   uint64_t capacity, uint64_t* count) {
    /* GaussianBvh::build (trace.cpp:88-111) then scan (:169-197) */
    int st;
    posed_t* posed = pose_all(field, nodes, n_nodes, lidar->env, &st);
    if (!posed) return st;
    st = validate_lidar(lidar);
    if (st != GSIM_OK) { free(posed); return st; }
    const uint64_t azimuths = (uint64_t)llround(2.0 * kPiD / lidar->azimuth_step);
    const uint64_t rays = lidar->n_channels * azimuths;
    cand_t* buf = (cand_t*)malloc((field->count ? field->count : 1) * sizeof(cand_t));
    const quat sq = rigid_q(&lidar->pose);
    const v3 origin = rigid_t(&lidar->pose);
    uint64_t hits = 0;
    for (uint64_t k = 0; k < rays; ++k) {
        const uint64_t channel = k / azimuths, step = k % azimuths;
        const double elevation = lidar->channels[channel];
        const double az = (double)step * lidar->azimuth_step;
        const double ce = cos(elevation);
        const v3 dir_sensor = v3_make(ce * cos(az), ce * sin(az), sin(elevation));
        const v3 dir = q_rotate(sq, dir_sensor);
        uint8_t h;
        double d, a;
        trace_one(posed, field->count, origin, dir, lidar->max_range, lidar->alpha_threshold, buf,
                  &h, &d, &a);
        if (!h) continue;
        if (hits < capacity) {
            const v3 p = v3_scale(dir_sensor, d);
            points[3 * hits] = p.x; points[3 * hits + 1] = p.y; points[3 * hits + 2] = p.z;
            ring[hits] = (uint32_t)channel;
            azimuth[hits] = az;
        }
        ++hits;
    }
    free(buf);
    free(posed);
    *count = hits;
    return GSIM_OK;
}
