// stepbench.cu -- latency of warp 0's per-coordinate scalar chain in k_ccd
// (exchange result -> limb reconstruction -> penalized step -> clamp), as a
// dependent loop on one warp.  Profiling aid, not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_1208_0945_b200/csrc -o scripts/stepbench scripts/stepbench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "prior.h"
#include "xchg.cuh"
using namespace bsccs_b200;

template <int MODE>
__global__ void kstep(const unsigned long long* words, PriorParams p, int n, double* out, long long* cyc) {
    const int l = threadIdx.x & 31;
    unsigned long long d = l < 7 ? words[l] : 0;
    double bj = 0.01, rj = 1.0, ydx = 3.0, acc = 0.0;
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const unsigned long long d1 = __shfl_down_sync(0xffffffffu, d, 1);
        const unsigned long long d2 = __shfl_down_sync(0xffffffffu, d, 2);
        double v;
        if (MODE == 0) {
            bool ovf;
            v = from_limbs(d, d1, d2, ovf);
        } else { // per-lane conversion, two adds (not correctly rounded)
            v = __dadd_rn(__dadd_rn(__dmul_rn(__ull2double_rn(d2), 0x1p2), __dmul_rn(__ull2double_rn(d1), 0x1p-39)),
                          __dmul_rn(__ull2double_rn(d), 0x1p-80));
        }
        const double ta = __shfl_sync(0xffffffffu, v, 0);
        const double tb = __shfl_sync(0xffffffffu, v, 3);
        const int te = __shfl_sync(0xffffffffu, d, 6) != 0 ? 1 : 0;
        double delta = 0.0;
        if (!te) {
            const double g = __dsub_rn(ydx, ta);
            const double h = tb == 0.0 ? 0.0 : -tb;
            double step = 0.0;
            const double bv = beta_over_v(p, bj);
            if (!penalized_step_pre(p, bj, bv, g, h, &step)) delta = clamp_step(step, rj);
        }
        rj = next_trust(delta, rj);
        acc += delta;
        // feed the result back so iterations are dependent
        d ^= (static_cast<unsigned long long>(__double_as_longlong(delta)) & 1ull);
        bj = __dadd_rn(bj, delta * 1e-30);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) {
        *out = acc;
        *cyc = t1 - t0;
    }
}

int main() {
    unsigned long long h[7] = {123456789ull, 98765432ull, 1234ull, 55555555ull, 4444444ull, 777ull, 0ull};
    unsigned long long* d;
    double* o;
    long long* c;
    cudaMalloc(&d, sizeof h);
    cudaMalloc(&o, 8);
    cudaMalloc(&c, 8);
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    const int n = 10000;
    for (int kind = 0; kind < 3; ++kind) {
        PriorParams p = make_prior_params(kind, 0.1, false);
        for (int mode = 0; mode < 2; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) kstep<0><<<1, 32>>>(d, p, n, o, c);
                else kstep<1><<<1, 32>>>(d, p, n, o, c);
                cudaDeviceSynchronize();
            }
            long long cyc;
            cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
            printf("prior %d %s: %.1f cycles per step\n", kind, mode ? "per-lane limbs" : "from_limbs    ",
                   double(cyc) / n);
        }
    }
    return 0;
}
