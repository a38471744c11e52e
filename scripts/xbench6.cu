// xbench6.cu -- exchange latency with the arrivals of each word spread over
// NC copies: G persistent CTAs (one per SM) perform N back-to-back exchanges
// of 7 words; CTA c red.adds its words into copy c % NC, warp 0 polls all
// 7*NC (word, copy) lines at once (one lane each) and each lane waits for its
// copy's own arrival count.  Also reports the spread of the CTAs' detection
// times (globaltimer) per exchange.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xbench6 scripts/xbench6.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ void red_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int kStride = 64; // u64 per line slot (512 B apart)

template <int NC>
__global__ void __launch_bounds__(512, 1) kx(unsigned long long* area, int n, int G, unsigned long long* det, int ndet) {
    unsigned long long prev[2] = {0, 0};
    const int l = threadIdx.x;
    const int mycopy = blockIdx.x % NC;
    // arrivals into copy k: CTAs c with c % NC == k
    const int word = l / NC, copy = l % NC;
    const unsigned long long expect = (G - copy + NC - 1) / NC;
    for (int s = 0; s < n; ++s) {
        const int buf = s & 1;
        __syncthreads();
        if (l < 7) red_add(area + ((buf * 7 + l) * NC + mycopy) * kStride, (1ull << 50) + 3);
        if (l < 7 * NC) {
            const unsigned long long* p = area + ((buf * 7 + word) * NC + copy) * kStride;
            unsigned long long v;
            unsigned spins = 0;
            const unsigned long long t0 = gtimer();
            do {
                v = ld_volatile(p);
                if ((++spins & 1023u) == 0u && gtimer() - t0 > 50000000ull) { // 50 ms: report, do not hang
                    printf("timeout cta %d lane %d s %d v %llx prev %llx expect %llu\n", blockIdx.x, l, s, v, prev[buf], expect);
                    asm volatile("trap;");
                }
            } while (((v - prev[buf]) >> 50) < expect);
            prev[buf] = v;
        }
        __syncwarp();
        if (l == 0 && s < ndet) det[static_cast<size_t>(s) * G + blockIdx.x] = gtimer();
        __syncthreads();
    }
}

template <int NC>
void run(int G, unsigned long long* area, unsigned long long* det, int n) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int ndet = 512;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemset(area, 0, 8 << 20)); // every launch starts from zero words
        void* args[] = {&area, &n, &G, &det, (void*)&ndet};
        cudaEventRecord(e0);
        CK(cudaLaunchCooperativeKernel((void*)kx<NC>, dim3(G), dim3(512), args, 0, 0));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    std::vector<unsigned long long> h(static_cast<size_t>(ndet) * G);
    CK(cudaMemcpy(h.data(), det, h.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<double> spread;
    for (int s = 64; s < ndet; ++s) {
        auto b = h.begin() + static_cast<size_t>(s) * G;
        spread.push_back(static_cast<double>(*std::max_element(b, b + G) - *std::min_element(b, b + G)));
    }
    std::sort(spread.begin(), spread.end());
    printf("G=%3d copies=%d arrivals/line~%3d  %7.1f ns/exchange  detection spread median %5.0f p90 %5.0f ns\n", G, NC,
           (G + NC - 1) / NC, best * 1e6 / n, spread[spread.size() / 2], spread[spread.size() * 9 / 10]);
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    unsigned long long *area, *det;
    CK(cudaMalloc(&area, 8 << 20));
    CK(cudaMalloc(&det, sizeof(unsigned long long) * 512 * 148));
    const int n = 4000;
    for (int rep = 0; rep < 2; ++rep) {
        run<1>(148, area, det, n);
        run<2>(148, area, det, n);
        run<4>(148, area, det, n);
    }
    return 0;
}
