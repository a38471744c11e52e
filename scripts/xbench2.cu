// xbench2.cu -- exchange of W fixed-point words among all CTAs (one per SM):
// how the cost scales with W and with the publish / poll pattern.
// Profiling aid for the batched engine (batch.cu); not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/xbench2 scripts/xbench2.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

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
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// mode 0: warp 0 publishes W words and polls them all (lane loops over its words)
// mode 1: mode 0 + __nanosleep(64) between poll rounds
// mode 2: ceil(W/32) warps, one word per lane (publish + poll)
// mode 3: cluster of 2: partner's words summed through DSMEM, leader publishes
//         (participants = clusters), leader polls, result copied to partner
// mode 4: stride 8 words (64 B) instead of 32 (256 B)
__global__ void __launch_bounds__(512, 1) kx(unsigned long long* area, int n, int W, int mode, int P) {
    __shared__ unsigned long long sh[256];
    __shared__ unsigned long long prev[2][256];
    const int stride = mode == 4 ? 8 : 32;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) prev[0][i] = prev[1][i] = 0;
    __syncthreads();
    cg::cluster_group cl = cg::this_cluster();
    const bool clustered = mode == 3;
    const bool leader = !clustered || cl.block_rank() == 0;
    for (int s = 0; s < n; ++s) {
        const int buf = s & 1;
        unsigned long long* base = area + (size_t)buf * 256 * stride;
        // the CTA's value of word w: 3 + w
        for (int w = threadIdx.x; w < W; w += blockDim.x) sh[w] = 3 + w;
        if (clustered) {
            cl.sync();
            if (leader) {
                unsigned long long* peer = cl.map_shared_rank(sh, 1);
                for (int w = threadIdx.x; w < W; w += blockDim.x) sh[w] += peer[w];
            }
            cl.sync();
        } else {
            __syncthreads();
        }
        const int pollers = (mode == 2) ? ((W + 31) / 32) * 32 : 32;
        if (leader && threadIdx.x < pollers) {
            const int l = threadIdx.x;
            for (int w = l; w < W; w += pollers) red_add(base + (size_t)w * stride, sh[w] + (1ull << 50));
            unsigned pending = 0;
            for (int i = 0, w = l; w < W; w += pollers, ++i) pending |= 1u << i;
            while (pending) {
                unsigned long long v[8];
                for (int i = 0, w = l; w < W; w += pollers, ++i)
                    if ((pending >> i) & 1u) v[i] = ld_volatile(base + (size_t)w * stride);
                for (int i = 0, w = l; w < W; w += pollers, ++i) {
                    if (!((pending >> i) & 1u)) continue;
                    if (((v[i] - prev[buf][w]) >> 50) >= (unsigned long long)P) {
                        prev[buf][w] = v[i];
                        sh[w] = v[i];
                        pending &= ~(1u << i);
                    }
                }
                if (pending && mode == 1) __nanosleep(64);
            }
        }
        if (clustered) {
            cl.sync();
            if (!leader) {
                unsigned long long* peer = cl.map_shared_rank(sh, 0);
                for (int w = threadIdx.x; w < W; w += blockDim.x) sh[w] = peer[w];
            }
            cl.sync();
        } else {
            __syncthreads();
        }
    }
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    unsigned long long* area;
    CK(cudaMalloc(&area, 8 << 20));
    const int n = 1000;
    const char* names[] = {"warp0 poll-all", "warp0 + nanosleep", "1 word per lane", "cluster-2 DSMEM", "stride 64B"};
    for (int W : {7, 25, 50, 99}) {
        for (int mode = 0; mode < 5; ++mode) {
            CK(cudaMemset(area, 0, 8 << 20));
            int G = sms;
            if (mode == 3 && (G & 1)) G -= 1;
            int P = mode == 3 ? G / 2 : G;
            int nn = n, WW = W, mm = mode;
            void* args[] = {&area, &nn, &WW, &mm, &P};
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(512);
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            at[1].id = cudaLaunchAttributeClusterDimension;
            at[1].val.clusterDim.x = mode == 3 ? 2 : 1;
            at[1].val.clusterDim.y = 1;
            at[1].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 2;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaError_t err = cudaLaunchKernelExC(&cfg, (void*)kx, args);
            if (err != cudaSuccess) {
                printf("W=%3d %-20s launch failed: %s\n", W, names[mode], cudaGetErrorString(err));
                cudaGetLastError();
                continue;
            }
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("W=%3d G=%3d %-20s %8.1f ns/exchange\n", W, G, names[mode], ms * 1e6 / n);
        }
    }
    return 0;
}
