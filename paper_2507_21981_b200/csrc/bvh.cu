// bvh.cu — SURVEY.md 8f row 4: the acceleration structure for arbitrary LiDAR rays.
//
// The reference traces arbitrary rays through a SAH BVH over the posed 3-sigma boxes
// (bvh.cpp:26-124, trace.cpp:113-123). The BVH only accelerates: a ray's candidate set is
// exactly {i : ray_aabb_hit(box_i, ray)} (bvh.hpp:58-80, trace_linear is the contract), and the
// tracer composites those candidates in (t, index) order. We build a linear BVH on the device
// (Karras 2012) instead of a SAH tree:
//   bvh_morton_kernel     30-bit Morton code of every seen box centre within the centres' bounds
//                         (kInvalidKey for primitives no node shows the sensor: dropped)
//   (segmented onesweep)  sort.cu sorts (code, primitive) pairs, 4 passes of 8-bit digits
//   bvh_build_kernel      internal node i of the n-1: its key range by the delta function (code,
//                         then primitive index, so duplicate codes still split) and split point
//   bvh_refit_kernel      leaves upward: the second child to arrive at a node writes the union
//                         of the children's boxes (exact fmin / fmax of doubles)
//   bvh_widen_kernel      traversal nodes: both children's boxes in fp32 (rounded outward, widened)
//   bvh_collect_kernel    one thread per ray, stack traversal testing both children of a visited
//                         node in fp32 (a conservative filter); a leaf is a candidate iff the
//                         reference's double ray_aabb_hit of its own box passes — count pass,
//                         then fill pass into the ray's list
// A union box contains its children's boxes, and the slab test is monotone under containment
// in floating point too ((lo - o) * inv rounds monotonically), so no hit box is ever pruned: the
// lists equal the reference's candidate sets and lidar_trace_kernel composites them as for scans.
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {

__device__ __forceinline__ uint64_t ordered_bits(double x) {  // monotone double -> u64
    const uint64_t u = uint64_t(__double_as_longlong(x));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered(uint64_t u) {
    return __longlong_as_double((u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u);
}

__device__ __forceinline__ uint32_t spread10(uint32_t v) {  // 10 bits -> every third bit
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__device__ __forceinline__ bool slab_hit(double lx, double ly, double lz, double hx, double hy,
                                         double hz, dv3 o, dv3 inv, double t_max) {
    // bvh.hpp:20-36, the reference's slab test over [0, t_max]
    double t0 = 0.0, t1 = t_max;
    const double tx0 = (lx - o.x) * inv.x, tx1 = (hx - o.x) * inv.x;
    t0 = fmax(t0, fmin(tx0, tx1));
    t1 = fmin(t1, fmax(tx0, tx1));
    const double ty0 = (ly - o.y) * inv.y, ty1 = (hy - o.y) * inv.y;
    t0 = fmax(t0, fmin(ty0, ty1));
    t1 = fmin(t1, fmax(ty0, ty1));
    const double tz0 = (lz - o.z) * inv.z, tz1 = (hz - o.z) * inv.z;
    t0 = fmax(t0, fmin(tz0, tz1));
    t1 = fmin(t1, fmax(tz0, tz1));
    return t0 <= t1;
}

}  // namespace

// Centre bounds of the seen boxes: block min/max, then one atomic per block on ordered bits.
__global__ void __launch_bounds__(256) bvh_bounds_kernel(BvhArgs a) {
    __shared__ double s_v[6][8];
    double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    const uint64_t n = a.n;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        if (!a.seen[i]) continue;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double c = 0.5 * (a.posed[(13 + k) * n + i] + a.posed[(16 + k) * n + i]);
            v[k] = fmin(v[k], c);
            v[3 + k] = fmax(v[3 + k], c);
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            const double x = __shfl_xor_sync(0xffffffffu, v[k], o);
            v[k] = k < 3 ? fmin(v[k], x) : fmax(v[k], x);
        }
        if (lane == 0) s_v[k][warp] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        const int k = threadIdx.x;
        double r = s_v[k][0];
        for (int w = 1; w < int(blockDim.x >> 5); ++w) r = k < 3 ? fmin(r, s_v[k][w]) : fmax(r, s_v[k][w]);
        if (k < 3) atomicMin(reinterpret_cast<unsigned long long*>(a.bounds_bits + k), ordered_bits(r));
        else atomicMax(reinterpret_cast<unsigned long long*>(a.bounds_bits + k), ordered_bits(r));
    }
}

__global__ void __launch_bounds__(256) bvh_morton_kernel(BvhArgs a) {
    const uint64_t n = a.n;
    double lo[3], ext[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = from_ordered(a.bounds_bits[k]);
        const double e = from_ordered(a.bounds_bits[3 + k]) - lo[k];
        ext[k] = e > 0.0 ? 1023.0 / e : 0.0;
    }
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t key = kInvalidKey;
        if (a.seen[i]) {
            uint32_t q[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double c = 0.5 * (a.posed[(13 + k) * n + i] + a.posed[(16 + k) * n + i]);
                const double f = (c - lo[k]) * ext[k];
                q[k] = f <= 0.0 ? 0u : (f >= 1023.0 ? 1023u : uint32_t(f));
            }
            key = (spread10(q[0]) << 2) | (spread10(q[1]) << 1) | spread10(q[2]);
        }
        a.codes_in[i] = key;
    }
}

// Sort bookkeeping for one segment: V = the valid keys (histogram of pass 1), the chunk tables
// of the later passes.
__global__ void bvh_sort_setup_kernel(BvhArgs a) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t v = 0;
    for (int d = 0; d < 256; ++d) v += a.hist[d];
    a.vbase[0] = 0;
    a.vbase[1] = v;
    a.chunk_base1[0] = 0;
    a.chunk_base1[1] = (v + uint32_t(kOnesweepTile) - 1) / uint32_t(kOnesweepTile);
    *a.n_leaves = v;
}

namespace {
// delta(i, j) of Karras 2012 over the sorted codes, ties broken by position.
__device__ __forceinline__ int delta(const uint32_t* codes, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    const uint32_t ci = codes[i], cj = codes[j];
    if (ci != cj) return __clz(ci ^ cj);
    return 32 + __clz(uint32_t(i) ^ uint32_t(j));
}
}  // namespace

// Internal nodes 0 .. n-2 (node 0 is the root); children >= kLeafBit are leaves (sorted index).
__global__ void __launch_bounds__(256) bvh_build_kernel(BvhArgs a) {
    const int n = int(*a.n_leaves);
    const uint32_t* codes = a.codes_sorted;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
        const int d = (delta(codes, n, i, i + 1) - delta(codes, n, i, i - 1)) >= 0 ? 1 : -1;
        const int dmin = delta(codes, n, i, i - d);
        int lmax = 2;
        while (delta(codes, n, i, i + lmax * d) > dmin) lmax <<= 1;
        int l = 0;
        for (int t = lmax >> 1; t >= 1; t >>= 1)
            if (delta(codes, n, i, i + (l + t) * d) > dmin) l += t;
        const int j = i + l * d;
        const int dnode = delta(codes, n, i, j);
        int s = 0;
        for (int t = (l + 1) >> 1;; t = (t + 1) >> 1) {
            if (delta(codes, n, i, i + (s + t) * d) > dnode) s += t;
            if (t == 1) break;
        }
        const int gamma = i + s * d + (d < 0 ? -1 : 0);
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        const uint32_t left = lo == gamma ? (kLeafBit | uint32_t(gamma)) : uint32_t(gamma);
        const uint32_t right = hi == gamma + 1 ? (kLeafBit | uint32_t(gamma + 1)) : uint32_t(gamma + 1);
        a.child[2 * i] = left;
        a.child[2 * i + 1] = right;
        if (left & kLeafBit) a.leaf_parent[gamma] = uint32_t(i);
        else a.node_parent[gamma] = uint32_t(i);
        if (right & kLeafBit) a.leaf_parent[gamma + 1] = uint32_t(i);
        else a.node_parent[gamma + 1] = uint32_t(i);
        a.visits[i] = 0u;
    }
}

// Boxes upward from the leaves: node boxes [node][6] = lo xyz, hi xyz (doubles).
__global__ void __launch_bounds__(256) bvh_refit_kernel(BvhArgs a) {
    const int n = int(*a.n_leaves);
    const uint64_t np = a.n;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        {   // the leaf's box in sorted order, contiguous for the traversal's leaf tests
            const uint32_t prim = a.leaf_prim[k];
#pragma unroll
            for (int q = 0; q < 6; ++q) a.leaf_box[6 * uint64_t(k) + q] = a.posed[(13 + q) * np + prim];
        }
        if (n == 1) break;
        uint32_t node = a.leaf_parent[k];
        while (true) {
            __threadfence();
            if (atomicAdd(a.visits + node, 1u) == 0u) break;  // the sibling finishes this node
            __threadfence();
            double b[6];
#pragma unroll
            for (int q = 0; q < 6; ++q) b[q] = q < 3 ? INFINITY : -INFINITY;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const uint32_t ch = a.child[2 * node + c];
                double cb[6];
                if (ch & kLeafBit) {
                    const uint32_t prim = a.leaf_prim[ch & ~kLeafBit];
#pragma unroll
                    for (int q = 0; q < 6; ++q) cb[q] = a.posed[(13 + q) * np + prim];
                } else {
#pragma unroll
                    for (int q = 0; q < 6; ++q) cb[q] = __ldcg(a.node_box + 6 * uint64_t(ch) + q);
                }
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    b[q] = fmin(b[q], cb[q]);
                    b[3 + q] = fmax(b[3 + q], cb[3 + q]);
                }
            }
#pragma unroll
            for (int q = 0; q < 6; ++q) __stcg(a.node_box + 6 * uint64_t(node) + q, b[q]);
            if (node == 0) break;
            node = a.node_parent[node];
        }
    }
}

// Traversal nodes: node i carries BOTH children's boxes in fp32, rounded outward and widened by
// a margin, plus the child links (4 float4 = 64 B, one load per visited node):
//   w[0] = (L.lo.x, L.lo.y, L.lo.z, L.hi.x)  w[1] = (L.hi.y, L.hi.z, R.lo.x, R.lo.y)
//   w[2] = (R.lo.z, R.hi.x, R.hi.y, R.hi.z)  w[3] = (child L, child R, -, -) as bits
// The fp32 tests only filter (false positives are harmless: a leaf is a candidate only after the
// reference's exact double slab test of its own box); the outward rounding plus the margin keep
// every box a ray can hit in double inside what the fp32 test accepts.
__device__ __forceinline__ void child_box(const BvhArgs& a, uint32_t ch, double b[6]) {
    if (ch & kLeafBit) {
        const uint32_t prim = a.leaf_prim[ch & ~kLeafBit];
#pragma unroll
        for (int q = 0; q < 6; ++q) b[q] = a.posed[(13 + q) * a.n + prim];
    } else {
#pragma unroll
        for (int q = 0; q < 6; ++q) b[q] = a.node_box[6 * uint64_t(ch) + q];
    }
}

__global__ void __launch_bounds__(256) bvh_widen_kernel(BvhArgs a) {
    const int n = int(*a.n_leaves);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
        float f[12];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            double b[6];
            child_box(a, a.child[2 * i + c], b);
            const double m = 1e-5 * (fabs(b[0]) + fabs(b[1]) + fabs(b[2]) + fabs(b[3]) + fabs(b[4]) +
                                     fabs(b[5])) + 1e-6;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                f[6 * c + q] = __double2float_rd(b[q] - m);
                f[6 * c + 3 + q] = __double2float_ru(b[3 + q] + m);
            }
        }
        float4* w = a.wide + 4 * uint64_t(i);
        w[0] = make_float4(f[0], f[1], f[2], f[3]);
        w[1] = make_float4(f[4], f[5], f[6], f[7]);
        w[2] = make_float4(f[8], f[9], f[10], f[11]);
        w[3] = make_float4(__uint_as_float(a.child[2 * i]), __uint_as_float(a.child[2 * i + 1]), 0.f, 0.f);
    }
}

__device__ __forceinline__ bool slab_hit_f(float lx, float ly, float lz, float hx, float hy, float hz,
                                           float3 o, float3 inv, float t_max) {
    float t0 = 0.0f, t1 = t_max;
    const float tx0 = (lx - o.x) * inv.x, tx1 = (hx - o.x) * inv.x;
    t0 = fmaxf(t0, fminf(tx0, tx1));
    t1 = fminf(t1, fmaxf(tx0, tx1));
    const float ty0 = (ly - o.y) * inv.y, ty1 = (hy - o.y) * inv.y;
    t0 = fmaxf(t0, fminf(ty0, ty1));
    t1 = fminf(t1, fmaxf(ty0, ty1));
    const float tz0 = (lz - o.z) * inv.z, tz1 = (hz - o.z) * inv.z;
    t0 = fmaxf(t0, fminf(tz0, tz1));
    t1 = fminf(t1, fmaxf(tz0, tz1));
    return t0 <= t1 + 1e-4f * fabsf(t1) + 1e-6f;  // a margin for the fp32 rounding of the ts
}

// Candidates of every ray. mode 0: count into ray_count; 1: fill the list at ray_offset[ray];
// 2: single pass, fill at ray * list_stride up to list_stride entries and count them all into
// ray_count (the host falls back to count + fill when a ray overflows).
__global__ void __launch_bounds__(128) bvh_collect_kernel(BvhArgs a, const LidarArgs la, int fill) {
    const int n = int(*a.n_leaves);
    for (uint64_t ray = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; ray < la.n_rays;
         ray += uint64_t(gridDim.x) * blockDim.x) {
        const dv3 o = mk3(la.ray_origin[3 * ray], la.ray_origin[3 * ray + 1], la.ray_origin[3 * ray + 2]);
        const dv3 d = mk3(la.ray_dir[3 * ray], la.ray_dir[3 * ray + 1], la.ray_dir[3 * ray + 2]);
        const dv3 inv = mk3(1.0 / d.x, 1.0 / d.y, 1.0 / d.z);
        const double t_max = la.ray_tmax[ray];
        const float3 of = make_float3(float(o.x), float(o.y), float(o.z));
        const float3 invf = make_float3(float(inv.x), float(inv.y), float(inv.z));
        // t_max rounded up (and +inf stays +inf): the fp32 range never ends before the double one
        const float tmf = __double2float_ru(t_max);
        uint32_t count = 0;
        uint32_t* out = fill == 1 ? la.list + la.ray_offset[ray]
                      : fill == 2 ? la.list + ray * uint64_t(la.list_stride) : nullptr;
        const uint32_t cap = fill == 2 ? la.list_stride : 0xFFFFFFFFu;
        auto leaf = [&](uint32_t sorted_idx) {
            // one 48-byte row (refit's copy of the primitive's double box, in leaf order)
            const double2* lb = reinterpret_cast<const double2*>(a.leaf_box + 6 * uint64_t(sorted_idx));
            const double2 b0 = __ldg(lb), b1 = __ldg(lb + 1), b2 = __ldg(lb + 2);
            if (slab_hit(b0.x, b0.y, b1.x, b1.y, b2.x, b2.y, o, inv, t_max)) {
                if (out && count < cap) out[count] = a.leaf_prim[sorted_idx];
                ++count;
            }
        };
        if (n == 1) {
            leaf(0);
        } else if (n > 1) {
            uint32_t stack[64];
            int sp = 0;
            stack[sp++] = 0u;  // the root: its children's boxes are tested when it is visited
            while (sp > 0) {
                const uint32_t node = stack[--sp];
                const float4* w = a.wide + 4 * uint64_t(node);
                const float4 w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2), w3 = __ldg(w + 3);
                const uint32_t l = __float_as_uint(w3.x), r = __float_as_uint(w3.y);
                const bool hl = slab_hit_f(w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, of, invf, tmf);
                const bool hr = slab_hit_f(w1.z, w1.w, w2.x, w2.y, w2.z, w2.w, of, invf, tmf);
                if (hr) {
                    if (r & kLeafBit) leaf(r & ~kLeafBit); else stack[sp++] = r;
                }
                if (hl) {
                    if (l & kLeafBit) leaf(l & ~kLeafBit); else stack[sp++] = l;
                }
                GSIM_DCHECK(sp <= 64);
            }
        }
        if (fill != 1) la.ray_count[ray] = count;
        if (fill == 2 && count > cap) atomicMax(a.overflow, count);
    }
}

void launch_bvh_bounds(const BvhArgs& a, int n_sms, cudaStream_t s) {
    bvh_bounds_kernel<<<unsigned(n_sms * 4), 256, 0, s>>>(a);
}
void launch_bvh_morton(const BvhArgs& a, int n_sms, cudaStream_t s) {
    bvh_morton_kernel<<<unsigned(n_sms * 8), 256, 0, s>>>(a);
}
void launch_bvh_sort_setup(const BvhArgs& a, cudaStream_t s) { bvh_sort_setup_kernel<<<1, 32, 0, s>>>(a); }
void launch_bvh_build(const BvhArgs& a, int n_sms, cudaStream_t s) {
    bvh_build_kernel<<<unsigned(n_sms * 8), 256, 0, s>>>(a);
}
void launch_bvh_refit(const BvhArgs& a, int n_sms, cudaStream_t s) {
    bvh_refit_kernel<<<unsigned(n_sms * 8), 256, 0, s>>>(a);
    bvh_widen_kernel<<<unsigned(n_sms * 8), 256, 0, s>>>(a);
}
void launch_bvh_collect(const BvhArgs& a, const LidarArgs& la, int mode, int n_sms, cudaStream_t s) {
    const uint64_t want = (la.n_rays + 127) / 128;
    bvh_collect_kernel<<<unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(n_sms) * 16))),
                         128, 0, s>>>(a, la, mode);
}

}  // namespace gsim_gpu
