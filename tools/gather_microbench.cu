// gather_microbench.cu -- the cache-aware denominator SURVEY 8(d) asks for: throughput of
// random 8-byte and 16-byte gathers (read-only path, __ldg) from buffers of a given footprint,
// e.g. the paper-scale scene's 556 MB (mostly HBM) or an L2-resident 64 MB, on every SM.
// A naive gather of the scene's texels would run at these rates; the march kernel's texel
// gather (coherent 8x4-pixel ray tiles, L1 hits) is compared against them in DESIGN.md.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_microbench tools/gather_microbench.cu
//   ./gather_microbench            (prints one JSON line per footprint and load width)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void gather_kernel(const T* __restrict__ buf, uint64_t n_elem, int iters, uint64_t seed, T* sink) {
    uint64_t x = seed ^ ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull;
    T acc{};
    for (int i = 0; i < iters; i++) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;          // xorshift64
        const T v = __ldg(buf + (x % n_elem));
        if constexpr (sizeof(T) == 8) acc ^= v;
        else { acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w; }
    }
    if constexpr (sizeof(T) == 8) { if (acc == 0x123456789ull) *sink = acc; }
    else { if (acc.x == 0x1234567u) *sink = acc; }
}

template <typename T>
static void run(const char* name, size_t bytes, int sms) {
    T* buf = nullptr;
    T* sink = nullptr;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, sizeof(T));
    cudaMemset(buf, 1, bytes);
    const uint64_t n = bytes / sizeof(T);
    const int threads = 256, blocks = sms * 8, iters = 4096;
    gather_kernel<T><<<blocks, threads>>>(buf, n, 64, 1, sink);   // warm-up (and L2 fill)
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    gather_kernel<T><<<blocks, threads>>>(buf, n, iters, 7, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double loads = (double)blocks * threads * iters;
    printf("{\"footprint_mb\": %.1f, \"load\": \"%s\", \"gloads_per_s\": %.2f, \"useful_gbs\": %.1f}\n",
           bytes / 1e6, name, loads / (ms * 1e-3) / 1e9, loads * sizeof(T) / (ms * 1e-3) / 1e9);
    cudaFree(buf);
    cudaFree(sink);
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t fp[] = {(size_t)556 << 20, (size_t)64 << 20, (size_t)8 << 20};
    for (size_t b : fp) {
        run<unsigned long long>("8B", b, sms);
        run<uint4>("16B", b, sms);
    }
    return 0;
}
