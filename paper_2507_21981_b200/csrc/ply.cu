// ply.cu — device half of the splat PLY loader (splat_ply.cpp:40-162).
//
// The host parses the header and streams the float payload (count x stride, row-major) into
// HBM; this kernel turns every row into the field's SoA planes:
//   mean = (x, y, z); normals ignored; SH dc + rest (channel-major f_rest) -> sh[c][k];
//   opacity = 1 / (1 + exp(-o)); scale = exp(scale_i); rotation (w, x, y, z) renormalised only
//   when | |q| - 1 | > 1e-6 (keeps normalised quaternions bit-exact, splat_ply.cpp:150-156).
// Validation follows the reference's order per primitive (non-finite value, opacity saturation,
// scale overflow, zero-norm rotation) and the first failing primitive wins: err holds
// min(i << 3 | code). Compiled with -fmad=false; exp is CUDA's (<= 1 ulp from glibc).
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {

__global__ void __launch_bounds__(256) ply_convert_kernel(PlyArgs a) {
    const int K = (a.degree + 1) * (a.degree + 1);
    const int rest = K - 1;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < a.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const float* row = a.rows + i * uint64_t(a.stride);
        uint32_t code = 0;
        for (int k = 0; k < a.stride; ++k)
            if (!isfinite(row[k])) { code = 1; break; }
        const float* tail = row + 9 + 3 * rest;
        double opacity = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
        dq q{1.0, 0.0, 0.0, 0.0};
        if (!code) {
            opacity = 1.0 / (1.0 + exp(-double(tail[0])));
            if (opacity <= 0.0 || opacity >= 1.0) code = 2;
        }
        if (!code) {
            sx = exp(double(tail[1]));
            sy = exp(double(tail[2]));
            sz = exp(double(tail[3]));
            if (!isfinite(sx) || !isfinite(sy) || !isfinite(sz)) code = 3;
        }
        if (!code) {
            q = dq{double(tail[4]), double(tail[5]), double(tail[6]), double(tail[7])};
            const double n = qnorm(q);
            if (!(n > 0.0) || !isfinite(n)) code = 4;
            else if (fabs(n - 1.0) > 1e-6) q = qnormalized(q);
        }
        if (code) {
            atomicMin(a.err, (unsigned long long)((i << 3) | code));
            continue;
        }
        const DevField& f = a.field;
        f.mx[i] = double(row[0]);
        f.my[i] = double(row[1]);
        f.mz[i] = double(row[2]);
        f.sx[i] = sx;
        f.sy[i] = sy;
        f.sz[i] = sz;
        f.qw[i] = q.w;
        f.qx[i] = q.x;
        f.qy[i] = q.y;
        f.qz[i] = q.z;
        f.opacity[i] = opacity;
        // SH planes: value j = c * K + k of the packed per-primitive list, 4 per float4 plane
        for (int p = 0; p < f.sh_planes; ++p) {
            float v[4];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
                const int j = 4 * p + c4;
                const int c = j / K, k = j - c * K;
                v[c4] = j >= 3 * K ? 0.0f : (k == 0 ? row[6 + c] : row[9 + c * rest + (k - 1)]);
            }
            f.sh[uint64_t(p) * a.plane_stride + i] = make_float4(v[0], v[1], v[2], v[3]);
        }
    }
}

}  // namespace

void launch_ply_convert(const PlyArgs& a, int grid_cap, cudaStream_t stream) {
    if (a.n == 0) return;
    const uint64_t want = (a.n + 255) / 256;
    const int grid = int(want < uint64_t(grid_cap) ? want : uint64_t(grid_cap));
    ply_convert_kernel<<<grid, 256, 0, stream>>>(a);
}

}  // namespace gsim_gpu
