// encode.cu — standalone encoder of rendered float targets into the reference writers' bytes
// (image_io.cpp:75-111, :166-178). The fused variant lives in raster.cu's epilogue; both call
// encode_pixel (encode.cuh). HBM-bound: 20 B/px read, 3-10 B/px written.
#include <cstdint>

#include "encode.cuh"
#include "kernels.hpp"

namespace gsim_gpu {

namespace {
constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) encode_kernel(EncodeKernelArgs a) {
    __shared__ float s_thr[256];
    if (a.enc.srgb) {
        s_thr[threadIdx.x] = a.enc.srgb_thr[threadIdx.x];
        __syncthreads();
    }
    const EncodeCam c = a.cams[blockIdx.y];
    const uint32_t npx = c.width * c.height;
    const float* src = a.src + c.src_offset;  // [rgb npx*3 | depth npx | alpha npx]
    for (uint32_t p = blockIdx.x * kThreads + threadIdx.x; p < npx; p += gridDim.x * kThreads) {
        const uint32_t y = p / c.width, x = p - y * c.width;
        encode_pixel(a.enc, s_thr, a.enc.dst + c.dst_offset, c.width, c.height, x, y,
                     src[3 * p + 0], src[3 * p + 1], src[3 * p + 2], src[3 * size_t(npx) + p],
                     src[4 * size_t(npx) + p]);
    }
}
}  // namespace

void launch_encode(const EncodeKernelArgs& a, uint32_t n_cams, uint32_t max_pixels,
                   cudaStream_t stream) {
    if (n_cams == 0 || max_pixels == 0) return;
    uint32_t bx = (max_pixels + kThreads - 1) / kThreads;
    if (bx > 1184) bx = 1184;  // 148 SMs x 8
    encode_kernel<<<dim3(bx, n_cams), kThreads, 0, stream>>>(a);
}

}  // namespace gsim_gpu
