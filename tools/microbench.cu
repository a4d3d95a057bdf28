// microbench.cu — throughput of warp primitives on this GPU (cycles per warp-instruction per SM,
// with 32 warps per SM). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu
#include <cstdio>
#include <cstdint>

constexpr int kIters = 4096;

__global__ void k_ballot(uint32_t* out) {
    uint32_t v = threadIdx.x * 2654435761u, acc = 0;
    for (int i = 0; i < kIters; ++i) {
        acc += __ballot_sync(0xffffffffu, (v >> (i & 31)) & 1u);
        v = v * 1664525u + 1013904223u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_match(uint32_t* out) {
    uint32_t v = threadIdx.x * 2654435761u, acc = 0;
    for (int i = 0; i < kIters; ++i) {
        acc += __match_any_sync(0xffffffffu, v & 255u);
        v = v * 1664525u + 1013904223u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_shfl(uint32_t* out) {
    uint32_t v = threadIdx.x * 2654435761u, acc = 0;
    for (int i = 0; i < kIters; ++i) {
        acc += __shfl_sync(0xffffffffu, v, (v >> 7) & 31);
        v = v * 1664525u + 1013904223u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_atoms(uint32_t* out) {
    __shared__ uint32_t h[8][256];
    for (int k = threadIdx.x; k < 8 * 256; k += blockDim.x) (&h[0][0])[k] = 0;
    __syncthreads();
    uint32_t v = threadIdx.x * 2654435761u;
    const int w = threadIdx.x >> 5;
    for (int i = 0; i < kIters; ++i) {
        atomicAdd(&h[w][(threadIdx.x & 31) * 8 + (v & 7)], 1u);  // distinct bank per lane
        v = v * 1664525u + 1013904223u;
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = h[w][threadIdx.x & 255];
}
__global__ void k_atoms_rand(uint32_t* out) {
    __shared__ uint32_t h[8][256];
    for (int k = threadIdx.x; k < 8 * 256; k += blockDim.x) (&h[0][0])[k] = 0;
    __syncthreads();
    uint32_t v = threadIdx.x * 2654435761u;
    const int w = threadIdx.x >> 5;
    for (int i = 0; i < kIters; ++i) {
        atomicAdd(&h[w][v >> 24], 1u);  // random bins
        v = v * 1664525u + 1013904223u;
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = h[w][threadIdx.x & 255];
}
__global__ void k_lds_sts(uint32_t* out) {  // read-modify-write chain on a warp-private counter
    __shared__ uint32_t h[8][256];
    for (int k = threadIdx.x; k < 8 * 256; k += blockDim.x) (&h[0][0])[k] = 0;
    __syncthreads();
    uint32_t v = threadIdx.x * 2654435761u;
    const int w = threadIdx.x >> 5;
    for (int i = 0; i < kIters; ++i) {
        const uint32_t d = (threadIdx.x & 31) * 8 + (v & 7);
        const uint32_t pre = h[w][d];
        __syncwarp();
        h[w][d] = pre + 1;
        __syncwarp();
        v = v * 1664525u + 1013904223u;
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = h[w][threadIdx.x & 255];
}
__global__ void k_popc_lop(uint32_t* out) {  // baseline ALU loop
    uint32_t v = threadIdx.x * 2654435761u, acc = 0;
    for (int i = 0; i < kIters; ++i) {
        acc += __popc(v & 0x5555u);
        v = v * 1664525u + 1013904223u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class K>
void run(const char* name, K kern, uint32_t* d, int sms) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = sms * 4, threads = 256;  // 32 warps per SM
    kern<<<blocks, threads>>>(d);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cycles = ms * 1e-3 * clk * 1e3;
    const double warp_ops_per_sm = 32.0 * kIters;
    printf("%-12s %8.3f ms  %6.2f SM-cycles per warp-iteration (32 warps/SM, incl. loop ALU)\n", name,
           ms, cycles / warp_ops_per_sm);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* d;
    cudaMalloc(&d, sizeof(uint32_t) * sms * 4 * 256);
    run("popc_lop", k_popc_lop, d, sms);
    run("ballot", k_ballot, d, sms);
    run("shfl_idx", k_shfl, d, sms);
    run("match_any", k_match, d, sms);
    run("atoms_bank", k_atoms, d, sms);
    run("atoms_rand", k_atoms_rand, d, sms);
    run("lds_sts_rmw", k_lds_sts, d, sms);
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
