// gbench2.cu -- random-line gather throughput on one B200 by access width:
// LSU 8/16/32 B per lane and cp.async.bulk of 64/128/256 B, at several depths.
// Profiling aid for k_bccd's gathers; not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gbench2 scripts/gbench2.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}

// LSU: each group of (LINE/W) lanes reads one LINE-byte line, W bytes per lane
template <int W, int LINE, int DEPTH>
__global__ void __launch_bounds__(512, 1) k_lsu(const unsigned char* __restrict__ a, long long nlines, int iters,
                                                double* out) {
    constexpr int LPL = LINE / W; // lanes per line
    const int g = threadIdx.x / LPL, l = threadIdx.x % LPL;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        double v[DEPTH];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) {
            const long long line = mix(blockIdx.x * 1000003ull + g * 7919ull + (unsigned long long)(it * DEPTH + d) * 104729ull) % nlines;
            const unsigned char* p = a + line * LINE + l * W;
            if (W == 8) v[d] = *reinterpret_cast<const double*>(p);
            else if (W == 16) { double2 t = *reinterpret_cast<const double2*>(p); v[d] = t.x + t.y; }
            else { double4 t; asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(t.x), "=d"(t.y), "=d"(t.z), "=d"(t.w) : "l"(p)); v[d] = t.x + t.y + t.z + t.w; }
        }
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) acc += v[d];
    }
    if (acc == 1.2345) out[0] = acc;
}

template <int BYTES, int NCOPY>
__global__ void __launch_bounds__(512, 1) k_tma(const unsigned char* __restrict__ a, long long nlines, int iters,
                                                double* out) {
    extern __shared__ __align__(128) unsigned char buf[];
    __shared__ __align__(8) unsigned long long mbar;
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared.b64 [%0], 512;" ::"r"(mb));
    __syncthreads();
    unsigned phase = 0;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        // NCOPY copies per CTA per iteration, spread over threads
        unsigned bytes = 0;
        for (int q = threadIdx.x; q < NCOPY; q += 512) bytes += BYTES;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        for (int q = threadIdx.x; q < NCOPY; q += 512) {
            const long long line = mix(blockIdx.x * 1000003ull + q * 7919ull + (unsigned long long)it * 104729ull) % nlines;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"((unsigned)__cvta_generic_to_shared(buf + q * BYTES)), "l"(a + line * BYTES), "r"(BYTES), "r"(mb) : "memory");
        }
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(mb), "r"(phase) : "memory");
        phase ^= 1;
        acc += buf[threadIdx.x];
        __syncthreads();
    }
    if (acc == 1.2345) out[0] = acc;
}

int sms;
template <typename F>
void timeit(F f, double bytes_per_iter_total, const char* name) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    f(2); CK(cudaDeviceSynchronize());
    const int iters = 100;
    cudaEventRecord(e0); f(iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %8.1f GB/s  %6.2f us/iter\n", name, bytes_per_iter_total * iters / (ms * 1e-3) / 1e9, ms * 1e3 / iters);
}

int main() {
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long long bytes = 4ll << 30;
    unsigned char* a; double* out;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&out, 64)); CK(cudaMemset(a, 0, bytes));
#define LSU(W, LINE, D) timeit([&](int it) { k_lsu<W, LINE, D><<<sms, 512>>>(a, bytes / LINE, it, out); }, \
        (double)sms * (512 / (LINE / W)) * D * LINE, "LSU " #W "B/lane line " #LINE " depth " #D)
    LSU(8, 128, 4); LSU(8, 128, 8);
    LSU(16, 128, 4); LSU(16, 128, 8); LSU(16, 128, 16);
    LSU(32, 128, 4); LSU(32, 128, 8); LSU(32, 128, 16);
    LSU(32, 256, 8); LSU(32, 256, 16);
#define TMA(B, N) do { CK(cudaFuncSetAttribute(k_tma<B, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, B * N)); \
        timeit([&](int it) { k_tma<B, N><<<sms, 512, B * N>>>(a, bytes / B, it, out); }, (double)sms * N * B, "TMA " #B "B x " #N " per CTA"); } while (0)
    TMA(64, 256); TMA(64, 1024);
    TMA(128, 256); TMA(128, 512); TMA(128, 1024);
    TMA(256, 256); TMA(256, 512);
    TMA(1024, 64); TMA(1024, 128);
    return 0;
}
