// gbench4.cu -- DRAM bytes and time per random scattered access on one B200:
// what one 16-byte record gather (or an 8-byte scattered store) really
// costs in HBM traffic, and whether two records in one 128-byte line cost
// one fill or two.  Decides the era / subject record layout of k_ccd
// (DESIGN.md §6).  Run under ncu for the bytes:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gbench4 scripts/gbench4.cu
//   ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum scripts/gbench4
// Profiling aid; not part of the library.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}

// MODE 0: one 16-B load per access at a random line (offset 0)
// MODE 1: one 8-B store per access at a random line
// MODE 2: 16-B load then 8-B store to the same record (the sweep's update)
// MODE 3: two 16-B loads per access in one line, offsets 0 and 64
// MODE 4: two 16-B loads per access in one line, offsets 0 and 32
// MODE 5: two 16-B loads per access at two random lines
// MODE 6: 16-B load + 8-B store at two random lines (era + subject today)
// MODE 7: 16-B load + 8-B store twice in ONE line, offsets 0 and 64 (co-located)
template <int MODE, int DEPTH>
__global__ void __launch_bounds__(512, 1) k_acc(unsigned char* a, long long nlines, int iters, double* out) {
    double acc = 0;
    const unsigned long long t = blockIdx.x * 512ull + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        long long ln[DEPTH], ln2[DEPTH];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) {
            ln[d] = mix(t * 1000003ull + (unsigned long long)(it * DEPTH + d) * 104729ull) % nlines;
            ln2[d] = mix(t * 7919ull + (unsigned long long)(it * DEPTH + d) * 15485863ull + 17) % nlines;
        }
        double v[DEPTH];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) {
            unsigned char* p = a + ln[d] * 128;
            if (MODE == 0 || MODE == 2) {
                const double2 x = *reinterpret_cast<const double2*>(p);
                v[d] = x.x + x.y;
            } else if (MODE == 1) {
                v[d] = 0;
            } else if (MODE == 3 || MODE == 4 || MODE == 7) {
                const double2 x = *reinterpret_cast<const double2*>(p);
                const double2 y = *reinterpret_cast<const double2*>(p + (MODE == 4 ? 32 : 64));
                v[d] = x.x + y.x;
            } else {
                const double2 x = *reinterpret_cast<const double2*>(p);
                const double2 y = *reinterpret_cast<const double2*>(a + ln2[d] * 128);
                v[d] = x.x + y.x;
            }
        }
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) {
            unsigned char* p = a + ln[d] * 128;
            if (MODE == 1) *reinterpret_cast<double*>(p) = (double)t;
            if (MODE == 2) *reinterpret_cast<double*>(p) = v[d] + 1.0;
            if (MODE == 6) {
                *reinterpret_cast<double*>(p) = v[d] + 1.0;
                *reinterpret_cast<double*>(a + ln2[d] * 128) = v[d] + 2.0;
            }
            if (MODE == 7) {
                *reinterpret_cast<double*>(p) = v[d] + 1.0;
                *reinterpret_cast<double*>(p + 64) = v[d] + 2.0;
            }
            acc += v[d];
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

int sms;
template <typename F>
void timeit(F f, double accesses_per_iter, const char* name) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    f(1); CK(cudaDeviceSynchronize());
    const int iters = 20;
    cudaEventRecord(e0); f(iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-52s %8.2f G accesses/s  %8.3f us/iter\n", name, accesses_per_iter * iters / (ms * 1e-3) / 1e9,
           ms * 1e3 / iters);
}

int main() {
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long long bytes = 8ll << 30;
    unsigned char* a; double* out;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&out, 64)); CK(cudaMemset(a, 0, bytes));
    const double per = (double)sms * 512;
#define RUN(M, D, name) timeit([&](int it) { k_acc<M, D><<<sms, 512>>>(a, bytes / 128, it, out); }, per * D, name)
    RUN(0, 8, "M0 16B load, random line");
    RUN(1, 8, "M1 8B store, random line");
    RUN(2, 8, "M2 16B load + 8B store, same record");
    RUN(3, 8, "M3 two 16B loads, one line (+0, +64)");
    RUN(4, 8, "M4 two 16B loads, one line (+0, +32)");
    RUN(5, 8, "M5 two 16B loads, two random lines");
    RUN(6, 8, "M6 load+store at two random lines (today)");
    RUN(7, 8, "M7 load+store x2 in one line (+0, +64)");
    return 0;
}
