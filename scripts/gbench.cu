// gbench.cu -- achievable bandwidth of random 128-byte line gathers on one
// B200 (the access pattern of k_bccd: one fit-minor line per pair) against a
// streaming copy.  Profiling aid; not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gbench scripts/gbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}

// mode 0: 8 B per lane, 16 lanes per line (LSU, default caching)
// mode 1: 16 B per lane, 8 lanes per line
// mode 2: mode 0 with ld.global.cg (L2 only)
// mode 3: cp.async.bulk of whole 128-B lines into shared memory (one lane each)
template <int DEPTH>
__global__ void __launch_bounds__(512, 1) kg(const double* __restrict__ a, long long nlines, int iters, int mode,
                                             double* out) {
    __shared__ __align__(128) double buf[DEPTH <= 8 ? 512 * DEPTH : 16];
    __shared__ __align__(8) unsigned long long mbar;
    double acc = 0.0;
    const int lane16 = threadIdx.x & 15;
    unsigned long long seed = blockIdx.x * 1315423911ull + threadIdx.x / 16;
    if (mode == 3 && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&mbar)));
    }
    __syncthreads();
    unsigned phase = 0;
    for (int it = 0; it < iters; ++it) {
        if (mode == 0 || mode == 2) {
            double v[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
                const long long line = mix(seed + (unsigned long long)(it * DEPTH + d) * 7919ull) % nlines;
                const double* p = a + line * 16 + lane16;
                if (mode == 0) v[d] = *p;
                else asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v[d]) : "l"(p));
            }
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) acc += v[d];
        } else if (mode == 1) {
            // 8 lanes per line: thread pairs (t, t+8) read lines of two "pairs"
            double2 v[DEPTH];
            const int lane8 = threadIdx.x & 7;
            const unsigned long long sd = blockIdx.x * 1315423911ull + threadIdx.x / 8;
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
                const long long line = mix(sd + (unsigned long long)(it * DEPTH + d) * 7919ull) % nlines;
                v[d] = *reinterpret_cast<const double2*>(a + line * 16 + lane8 * 2);
            }
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) acc += v[d].x + v[d].y;
            // the same line count as mode 0 needs 2x fewer threads: do the second half
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
                const long long line = mix(sd + 0x5bd1e995ull + (unsigned long long)(it * DEPTH + d) * 7919ull) % nlines;
                v[d] = *reinterpret_cast<const double2*>(a + line * 16 + lane8 * 2);
            }
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) acc += v[d].x + v[d].y;
        } else {
            // one lane per line: 32 lines per warp, DEPTH/... keep the same total line count as mode 0
            const int nl = 512 / 16 * DEPTH; // lines per CTA per iteration
            const unsigned sb = (unsigned)__cvta_generic_to_shared(buf);
            const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(nl * 128) : "memory");
            __syncthreads();
            if (threadIdx.x < nl) {
                const long long line = mix(blockIdx.x * 1315423911ull + threadIdx.x + (unsigned long long)it * 7919ull) % nlines;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                             ::"r"(sb + threadIdx.x * 128), "l"(a + line * 16), "r"(mb) : "memory");
            }
            unsigned done = 0;
            while (!done) {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(mb), "r"(phase) : "memory");
            }
            phase ^= 1;
            acc += buf[threadIdx.x];
            __syncthreads();
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

template <int D>
void run(const double* a, long long nlines, int sms, double* out, int mode, const char* name) {
    const int iters = 200;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kg<D><<<sms, 512>>>(a, nlines, 4, mode, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    kg<D><<<sms, 512>>>(a, nlines, iters, mode, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    const double lines = (double)sms * (512 / 16) * D * iters;
    printf("%-34s depth %2d: %8.1f GB/s of 128-B lines (%.2f us per CTA-iteration)\n", name, D,
           lines * 128 / (ms * 1e-3) / 1e9, ms * 1e3 / iters);
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long long bytes = 4ll << 30; // 4 GiB table (>> L2)
    double *a, *out;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&out, 64));
    CK(cudaMemset(a, 0, bytes));
    const long long nlines = bytes / 128;
    for (int mode = 0; mode < 4; ++mode) {
        const char* names[] = {"LSU 8B/lane, 16 lanes/line", "LSU 16B/lane, 8 lanes/line", "LSU ld.cg 8B/lane",
                               "cp.async.bulk 128B/lane"};
        run<1>(a, nlines, sms, out, mode, names[mode]);
        run<2>(a, nlines, sms, out, mode, names[mode]);
        run<4>(a, nlines, sms, out, mode, names[mode]);
        run<8>(a, nlines, sms, out, mode, names[mode]);
        if (mode != 3) run<16>(a, nlines, sms, out, mode, names[mode]);
    }
    // streaming copy reference
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    double* b; CK(cudaMalloc(&b, bytes / 2));
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) CK(cudaMemcpy(b, a, bytes / 2, cudaMemcpyDeviceToDevice));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("cudaMemcpy D2D: %.1f GB/s (read+write)\n", 5.0 * bytes / (ms * 1e-3) / 1e9);
    return 0;
}
