// xbench.cu -- microbenchmark of grid-wide exchange patterns on one GPU
// (profiling aid for the CCD sweep kernel; not part of the library).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xbench scripts/xbench.cu
// Each variant: G persistent CTAs (1 per SM) perform N back-to-back
// all-reduces of two doubles; reports ns per exchange.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

__device__ __forceinline__ void red_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// mode 0: 7 red words 256 B apart, count in high bits, 7 lanes poll
// mode 1: same, 1 red word (count only)
// mode 2: LL all-gather (per-CTA 16 B record with tag; warp polls all)
// mode 3: single atomicAdd counter; thread 0 polls with acquire
// mode 4: mode 0 with __nanosleep(100) between polls
// mode 5: only __syncthreads (baseline)
// mode 6: mode 1 but poll with ld.volatile
__global__ void __launch_bounds__(512, 1) kx(unsigned long long* area, int n, int mode, long long* out,
                                             const double* big, long long bign, int nload) {
    __shared__ unsigned long long sh[8];
    const int P = gridDim.x;
    unsigned long long prev[2] = {0, 0};
    const long long t0 = clock64();
    double acc = 0.0;
    unsigned long long rs = 0x9E3779B97F4A7C15ull * (blockIdx.x * 512 + threadIdx.x + 1);
    for (int s = 0; s < n; ++s) {
        const int buf = s & 1;
        __syncthreads();
        double ld[4];
        for (int q = 0; q < 4; ++q) {  // scattered HBM loads in flight during the exchange
            rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17;
            ld[q] = q < nload ? big[rs % bign] : 0.0;
        }
        if (mode == 0 || mode == 1 || mode == 4 || mode == 6) {
            const int W = mode == 1 || mode == 6 ? 1 : 7;
            if (threadIdx.x == 0)
                for (int i = 0; i < W; ++i) red_add(area + (buf * 7 + i) * 32, (1ull << 50) + 3);
            if (threadIdx.x < W) {
                const unsigned long long* p = area + (buf * 7 + threadIdx.x) * 32;
                unsigned long long v;
                do {
                    v = mode == 6 ? ld_volatile(p) : ld_relaxed(p);
                    if (mode == 4 && ((v - prev[buf]) >> 50) < (unsigned long long)P) __nanosleep(100);
                } while (((v - prev[buf]) >> 50) < (unsigned long long)P);
                prev[buf] = v;
                sh[threadIdx.x] = v;
            }
        } else if (mode == 2) {
            const unsigned tag = 1 + s;
            unsigned long long* rec = area + 1024 + (size_t)buf * P * 2;
            if (threadIdx.x == 0) {
                const unsigned long long w = ((unsigned long long)tag << 32) | 7u;
                st_relaxed(rec + blockIdx.x * 2, w);
                st_relaxed(rec + blockIdx.x * 2 + 1, w);
            }
            if (threadIdx.x < 32) {
                for (int r = threadIdx.x; r < P; r += 32) {
                    unsigned long long v;
                    do {
                        v = ld_relaxed(rec + r * 2);
                    } while ((unsigned)(v >> 32) != tag);
                }
                __syncwarp();
            }
        } else if (mode == 3) {
            if (threadIdx.x == 0) {
                atomicAdd(area, 1ull);
                const unsigned long long target = (unsigned long long)(s + 1) * P;
                while (ld_acquire(area) < target) {
                }
            }
        }
        __syncthreads();
        for (int q = 0; q < 4; ++q) acc += ld[q];
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0 + (acc == 1.2345 ? 1 : 0);
}

int main(int argc, char** argv) {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    unsigned long long* area;
    long long* out;
    CK(cudaMalloc(&area, 1 << 20));
    CK(cudaMalloc(&out, sizeof(long long) * 1024));
    const int n = 2000;
    const long long bign = 1ll << 27; // 1 GiB of doubles
    double* big;
    CK(cudaMalloc(&big, bign * sizeof(double)));
    CK(cudaMemset(big, 0, bign * sizeof(double)));
    const char* names[] = {"red7+poll7", "red1+poll1", "LL all-gather", "atomic counter+acquire",
                           "red7+poll7+nanosleep", "syncthreads only", "red1+poll volatile"};
    for (int nload : {0, 1, 4}) {
    for (int G : {sms}) {
        for (int mode = 0; mode < 7; ++mode) {
            CK(cudaMemset(area, 0, 1 << 20));
            void* args[] = {&area, (void*)&n, &mode, &out, &big, (void*)&bign, &nload};
            int nn = n;
            args[1] = &nn;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            CK(cudaLaunchCooperativeKernel((void*)kx, dim3(G), dim3(512), args, 0, 0));
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("loads/thread=%d G=%3d %-26s %8.1f ns/exchange\n", nload, G, names[mode], ms * 1e6 / n);
        }
    }
    }
    return 0;
}
