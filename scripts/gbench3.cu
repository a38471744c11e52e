// gbench3.cu -- random 128-B line gather throughput vs table size (TLB
// reach), LSU 8 B and 32 B per lane, cudaMalloc vs cudaMallocAsync tables.
// Profiling aid; not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gbench3 scripts/gbench3.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
template <int W, int DEPTH>
__global__ void __launch_bounds__(512, 1) k(const unsigned char* __restrict__ a, long long nlines, int iters, double* out) {
    constexpr int LPL = 128 / W;
    const int g = threadIdx.x / LPL, l = threadIdx.x % LPL;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        double v[DEPTH];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) {
            const long long line = mix(blockIdx.x * 1000003ull + g * 7919ull + (unsigned long long)(it * DEPTH + d) * 104729ull) % nlines;
            const unsigned char* p = a + line * 128 + l * W;
            if (W == 8) v[d] = *reinterpret_cast<const double*>(p);
            else { double4 t; asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(t.x), "=d"(t.y), "=d"(t.z), "=d"(t.w) : "l"(p)); v[d] = t.x + t.w; }
        }
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) acc += v[d];
    }
    if (acc == 1.2345) out[0] = acc;
}
int main() {
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* out; CK(cudaMalloc(&out, 64));
    cudaStream_t s; CK(cudaStreamCreate(&s));
    for (int async = 0; async < 2; ++async)
    for (long long mb : {32ll, 128ll, 512ll, 2048ll, 8192ll, 32768ll}) {
        const long long bytes = mb << 20;
        unsigned char* a;
        if (async) CK(cudaMallocAsync((void**)&a, bytes, s)); else CK(cudaMalloc(&a, bytes));
        CK(cudaMemsetAsync(a, 0, bytes, s)); CK(cudaStreamSynchronize(s));
        const long long nl = bytes / 128;
        for (int w : {8, 32}) {
            auto run = [&](int it) { if (w == 8) k<8, 8><<<sms, 512, 0, s>>>(a, nl, it, out); else k<32, 8><<<sms, 512, 0, s>>>(a, nl, it, out); };
            run(2); CK(cudaStreamSynchronize(s));
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            const int iters = 100;
            cudaEventRecord(e0, s); run(iters); cudaEventRecord(e1, s); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double lines = (double)sms * (512 / (128 / w)) * 8 * iters;
            printf("%s %6lld MB  %2d B/lane: %7.1f GB/s\n", async ? "mallocAsync" : "malloc     ", mb, w, lines * 128 / (ms * 1e-3) / 1e9);
        }
        if (async) CK(cudaFreeAsync(a, s)); else CK(cudaFree(a));
        CK(cudaStreamSynchronize(s));
    }
    return 0;
}
