// xbench5.cu -- exchange latency against the number of participants, and a
// cluster (DSMEM) pre-reduction: G persistent CTAs (one per SM) perform N
// back-to-back exchanges of 7 words (red.add 2^50 + limb, 7 lanes poll).
// Cluster variant: CTAs of a cluster of size CS add their words into the
// leader's shared memory (atom.shared::cluster), barrier.cluster, the leader
// publishes one arrival per word; every CTA polls global memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xbench5 scripts/xbench5.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ void red_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int CS>
__global__ void __launch_bounds__(384, 1) kx(unsigned long long* area, int n, int P, long long* out) {
    __shared__ unsigned long long acc[2][8];
    unsigned long long prev[2] = {0, 0};
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = CS > 1 ? cl.block_rank() : 0;
    if (threadIdx.x < 16) (&acc[0][0])[threadIdx.x] = 0;
    if (CS > 1) cl.sync();
    const long long t0 = clock64();
    for (int s = 0; s < n; ++s) {
        const int buf = s & 1;
        __syncthreads();
        if (threadIdx.x < 7) {
            const unsigned long long w = (1ull << 50) + 3;
            if (CS == 1) {
                red_add(area + (buf * 7 + threadIdx.x) * 32, w);
            } else {
                unsigned long long* dst = cl.map_shared_rank(&acc[buf][threadIdx.x], 0);
                atomicAdd(dst, 3ull);
            }
        }
        if (CS > 1) {
            cl.sync(); // every member's adds landed in the leader
            if (rank == 0 && threadIdx.x < 7) {
                const unsigned long long v = acc[buf][threadIdx.x];
                acc[buf][threadIdx.x] = 0;
                red_add(area + (buf * 7 + threadIdx.x) * 32, (1ull << 50) + v);
            }
        }
        if (threadIdx.x < 7) {
            const unsigned long long* p = area + (buf * 7 + threadIdx.x) * 32;
            unsigned long long v;
            do {
                v = ld_volatile(p);
            } while (((v - prev[buf]) >> 50) < (unsigned long long)P);
            prev[buf] = v;
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int CS>
void run(int G, unsigned long long* area, long long* out, int n) {
    CK(cudaMemset(area, 0, 1 << 20));
    const int P = G / CS; // arrivals per word
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(384);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    CK(cudaLaunchKernelEx(&cfg, kx<CS>, area, n, P, out));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("G=%3d cluster=%d arrivals/word=%3d  %7.1f ns/exchange\n", G, CS, P, ms * 1e6 / n);
}

int main() {
    unsigned long long* area;
    long long* out;
    CK(cudaMalloc(&area, 1 << 20));
    CK(cudaMalloc(&out, sizeof(long long) * 1024));
    const int n = 4000;
    for (int G : {148, 74, 37, 16, 8, 1}) run<1>(G, area, out, n);
    run<2>(148, area, out, n);
    run<4>(148, area, out, n);
    run<2>(148, area, out, n);
    run<1>(148, area, out, n);
    return 0;
}
