// L2 read bandwidth probe ("streaming 128-bit loads over an
// 8-32 MB buffer, across all SMs"). Each thread streams uint4 loads over an
// L2-resident buffer; one warm pass, then timed passes with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/l2_peak tools/l2_peak.cu
//   tools/_build/l2_peak [MiB=16] [passes=200]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__global__ void k_stream(const uint4 *__restrict__ p, size_t n, int passes, unsigned *sink) {
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < passes; r++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            uint4 v;
            asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "l"(p + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678u) *sink = acc;  // keep the loads
}

int main(int argc, char **argv) {
    const size_t mib = argc > 1 ? (size_t)atoi(argv[1]) : 16;
    const int passes = argc > 2 ? atoi(argv[2]) : 200;
    const size_t bytes = mib << 20, n = bytes / 16;
    uint4 *p = nullptr;
    unsigned *sink = nullptr;
    cudaMalloc(&p, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(p, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 512, blocks = sms * 4;
    k_stream<<<blocks, threads>>>(p, n, 2, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_stream<<<blocks, threads>>>(p, n, passes, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double gbs = (double)bytes * passes / (ms * 1e-3) / 1e9;
    printf("{\"l2_read_gbs\": %.1f, \"buffer_mib\": %zu, \"passes\": %d, \"ms\": %.3f, \"sms\": %d, "
           "\"err\": \"%s\"}\n",
           gbs, mib, passes, ms, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
