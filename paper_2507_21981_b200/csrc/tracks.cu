// tracks.cu — device pose playback: PoseStream::sample for many nodes at
// once, and the Scene::step_to step that feeds the sampled poses into a frame's segment table.
//
// Semantics (pose_stream.cpp:117-136, math.hpp:195-214), per query (track, t, initial):
//   empty track or t < first time -> initial pose; t >= last time -> last record;
//   else hi = first record with time > t (upper_bound), lo = hi - 1,
//   translation = p_lo * (1 - u) + p_hi * u, rotation = slerp(q_lo, q_hi, u), u = (t-t_lo)/span.
// Records are appended on the host (validation + rotation normalisation, pose_stream.cpp:31-40),
// so the device holds normalised quaternions. Compiled with -fmad=false: translations, the
// nlerp branch and the endpoints are bit-exact with the reference; the slerp branch goes
// through CUDA's acos/sin (<= 2 ulp from glibc), a ~1e-16 relative difference.
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {

__device__ dq slerp_dev(dq a, dq b, double t) {  // math.hpp:195-214
    double cos_half = a.w * b.w + a.x * b.x + a.y * b.y + a.z * b.z;
    if (cos_half < 0.0) {
        b = dq{-b.w, -b.x, -b.y, -b.z};
        cos_half = -cos_half;
    }
    if (cos_half > 1.0 - 1e-12) {
        const dq q{a.w + t * (b.w - a.w), a.x + t * (b.x - a.x), a.y + t * (b.y - a.y),
                   a.z + t * (b.z - a.z)};
        return qnormalized(q);
    }
    const double half = acos(cos_half);
    const double s = sin(half);
    const double wa = sin((1.0 - t) * half) / s;
    const double wb = sin(t * half) / s;
    const dq q{wa * a.w + wb * b.w, wa * a.x + wb * b.x, wa * a.y + wb * b.y, wa * a.z + wb * b.z};
    return qnormalized(q);
}

// PoseStream::sample of track k at time t; writes (q, p); returns false for "initial pose".
__device__ bool sample_track(const DevTracks& tr, uint32_t k, double t, dq& q, dv3& p) {
    const uint64_t b = tr.begin[k], e = tr.begin[k + 1];
    if (b == e || t < tr.t[b]) return false;
    uint64_t hi;
    if (t >= tr.t[e - 1]) {
        hi = e - 1;
    } else {
        uint64_t lo_i = b, hi_i = e;  // upper_bound
        while (lo_i < hi_i) {
            const uint64_t mid = lo_i + (hi_i - lo_i) / 2;
            if (t < tr.t[mid]) hi_i = mid; else lo_i = mid + 1;
        }
        hi = lo_i;
        const uint64_t lo = hi - 1;
        const double span = tr.t[hi] - tr.t[lo];
        if (span > 0.0) {
            const double u = (t - tr.t[lo]) / span;
            p = mk3(tr.p[3 * lo + 0] * (1.0 - u) + tr.p[3 * hi + 0] * u,
                    tr.p[3 * lo + 1] * (1.0 - u) + tr.p[3 * hi + 1] * u,
                    tr.p[3 * lo + 2] * (1.0 - u) + tr.p[3 * hi + 2] * u);
            const dq ql{tr.q[4 * lo], tr.q[4 * lo + 1], tr.q[4 * lo + 2], tr.q[4 * lo + 3]};
            const dq qh{tr.q[4 * hi], tr.q[4 * hi + 1], tr.q[4 * hi + 2], tr.q[4 * hi + 3]};
            q = slerp_dev(ql, qh, u);
            return true;
        }
    }
    q = dq{tr.q[4 * hi], tr.q[4 * hi + 1], tr.q[4 * hi + 2], tr.q[4 * hi + 3]};
    p = mk3(tr.p[3 * hi], tr.p[3 * hi + 1], tr.p[3 * hi + 2]);
    return true;
}

__global__ void track_query_kernel(DevTracks tr, const uint32_t* track, const double* time,
                                   const gsim_rigid* initial, gsim_rigid* out, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        dq q;
        dv3 p;
        gsim_rigid r = initial[i];
        if (sample_track(tr, track[i], time[i], q, p)) {
            r.rotation[0] = q.w; r.rotation[1] = q.x; r.rotation[2] = q.y; r.rotation[3] = q.z;
            r.translation[0] = p.x; r.translation[1] = p.y; r.translation[2] = p.z;
        }
        out[i] = r;
    }
}

// Scene::step_to for one frame: every segment whose owner node is driven by a track gets the
// track's pose at time t; the segment's current pose (the node's initial pose) is the
// before-first-record value.
__global__ void pose_segments_kernel(DevTracks tr, DevSegment* segs, const int32_t* seg_track,
                                     uint32_t n_segs, double t) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_segs) return;
    const int32_t k = seg_track[s];
    if (k < 0) return;
    dq q;
    dv3 p;
    if (!sample_track(tr, uint32_t(k), t, q, p)) return;
    segs[s].q[0] = q.w; segs[s].q[1] = q.x; segs[s].q[2] = q.y; segs[s].q[3] = q.z;
    segs[s].t[0] = p.x; segs[s].t[1] = p.y; segs[s].t[2] = p.z;
}

}  // namespace

void launch_track_query(const DevTracks& tr, const uint32_t* track, const double* time,
                        const gsim_rigid* initial, gsim_rigid* out, uint64_t n, int grid_cap,
                        cudaStream_t stream) {
    if (n == 0) return;
    const uint64_t want = (n + 255) / 256;
    const int grid = int(want < uint64_t(grid_cap) ? want : uint64_t(grid_cap));
    track_query_kernel<<<grid, 256, 0, stream>>>(tr, track, time, initial, out, n);
}

void launch_pose_segments(const DevTracks& tr, DevSegment* segs, const int32_t* seg_track,
                          uint32_t n_segs, double t, cudaStream_t stream) {
    if (n_segs == 0) return;
    pose_segments_kernel<<<(n_segs + 127) / 128, 128, 0, stream>>>(tr, segs, seg_track, n_segs, t);
}

}  // namespace gsim_gpu
