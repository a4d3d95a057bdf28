// Library yardstick for the depth sort (diagnostic only, never linked into the product):
// cub::DeviceRadixSort::SortPairs on config-1-sized depth keys (u32 key, u32 record index),
// timed with CUDA events. Build + run: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/cub_sort_probe.cu -o /tmp/cub_sort_probe && /tmp/cub_sort_probe
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstring>
#include <algorithm>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

int main() {
    // depth-like keys: float bits of depths in [1, 12] m minus the smallest, cameras laid out
    // one after the other (5 segments); 27 significant bits like config 1
    const int n_cams = 5;
    const int per_cam = 906786;  // ~4.53M visible records / 5 cameras
    const int n = n_cams * per_cam;
    std::vector<uint32_t> keys(n), cam_keys(n), vals(n);
    std::mt19937 rng(7);
    std::uniform_real_distribution<float> dist(1.0f, 12.0f);
    uint32_t base;
    { float f = 1.0f; std::memcpy(&base, &f, 4); }
    for (int i = 0; i < n; ++i) {
        float z = dist(rng);
        uint32_t b;
        std::memcpy(&b, &z, 4);
        keys[i] = b - base;
        cam_keys[i] = (uint32_t(i / per_cam) << 27) | keys[i];
        vals[i] = uint32_t(i);
    }
    uint32_t *dk, *dk2, *dv, *dv2;
    CK(cudaMalloc(&dk, n * 4)); CK(cudaMalloc(&dk2, n * 4));
    CK(cudaMalloc(&dv, n * 4)); CK(cudaMalloc(&dv2, n * 4));
    int* offs;
    CK(cudaMalloc(&offs, (n_cams + 1) * 4));
    std::vector<int> h_offs(n_cams + 1);
    for (int c = 0; c <= n_cams; ++c) h_offs[c] = c * per_cam;
    CK(cudaMemcpy(offs, h_offs.data(), (n_cams + 1) * 4, cudaMemcpyHostToDevice));
    void* tmp = nullptr;
    size_t tmp_bytes = 0, t2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dk2, dv, dv2, n, 0, 32);
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, t2, dk, dk2, dv, dv2, n, n_cams, offs,
                                             offs + 1, 0, 27);
    tmp_bytes = std::max(tmp_bytes, t2);
    CK(cudaMalloc(&tmp, tmp_bytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto run = [&](const char* name, const std::vector<uint32_t>& src, int mode, int end_bit) {
        float best = 1e9f, sum = 0.f;
        const int reps = 30;
        for (int r = 0; r < reps + 3; ++r) {
            cudaMemcpy(dk, src.data(), n * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(dv, vals.data(), n * 4, cudaMemcpyHostToDevice);
            cudaEventRecord(e0);
            size_t tb = tmp_bytes;
            if (mode == 0)
                cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dk2, dv, dv2, n, 0, end_bit);
            else
                cub::DeviceSegmentedRadixSort::SortPairs(tmp, tb, dk, dk2, dv, dv2, n, n_cams,
                                                         offs, offs + 1, 0, end_bit);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 3) { best = std::min(best, ms); sum += ms; }
        }
        std::printf("%-44s n=%d bits=%d  best %.4f ms  mean %.4f ms\n", name, n, end_bit, best,
                    sum / reps);
    };
    run("SortPairs (camera bits above depth)", cam_keys, 0, 30);
    run("SortPairs (depth only, one segment)", keys, 0, 27);
    run("SegmentedRadixSort (5 cameras)", keys, 1, 27);
    CK(cudaGetLastError());
    return 0;
}
