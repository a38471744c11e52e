// devutil.h -- host-side helpers shared by the library's translation units:
// stream-ordered pooled allocation, pinned staging for host->device copies,
// grid sizing and the device guard.  Internal; not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.h"

namespace bsccs_b200 {

inline int grid_for(int64_t n, int threads, int dev_sms) {
    const int64_t g = (n + threads - 1) / threads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, static_cast<int64_t>(dev_sms) * 32)));
}

// Stream-ordered allocations from the device's default memory pool, which
// is told to retain freed memory: re-creating datasets / fit workspaces
// (bootstrap replicates, the e2e bench) then costs no cudaMalloc/cudaFree.
inline void ensure_pool(int device) {
    static std::atomic<unsigned> done{0};
    if (device < 32 && (done.load() & (1u << device))) return;
    cudaMemPool_t pool;
    CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
    unsigned long long keep = ~0ull;
    CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    if (device < 32) done.fetch_or(1u << device);
}

template <typename T>
T* dalloc(int64_t count, int64_t& bytes, cudaStream_t s) {
    T* p = nullptr;
    if (count <= 0) count = 1;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * static_cast<size_t>(count), s));
    bytes += static_cast<int64_t>(sizeof(T)) * count;
    return p;
}

template <typename T>
void dfree(T*& p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
}

// Host -> device copy of pageable caller memory through two pinned staging
// buffers: host threads fill one buffer while the DMA engine drains the other.
struct Staging {
    std::mutex m;
    unsigned char* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int device = -1;
    static constexpr size_t kChunk = size_t(64) << 20;
};
inline Staging g_staging;

inline void parallel_memcpy(void* dst, const void* src, size_t n) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t T = std::min<size_t>(std::min<size_t>(hw, 16), std::max<size_t>(1, n >> 22));
    if (T <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    for (size_t t = 0; t < T; ++t) {
        const size_t a = n * t / T, b = n * (t + 1) / T;
        th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
    }
    for (auto& x : th) x.join();
}

inline bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError(); // clear: unregistered pageable memory
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

inline void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s, int device) {
    if (bytes == 0) return;
    if (bytes < (size_t(4) << 20) || is_pinned(src)) { // small, or already page-locked: DMA directly
        CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    std::lock_guard<std::mutex> lk(g_staging.m);
    if (g_staging.device != device) {
        for (int i = 0; i < 2; ++i) {
            if (g_staging.buf[i]) cudaFreeHost(g_staging.buf[i]);
            if (g_staging.ev[i]) cudaEventDestroy(g_staging.ev[i]);
            CUDA_TRY(cudaMallocHost(&g_staging.buf[i], Staging::kChunk));
            CUDA_TRY(cudaEventCreateWithFlags(&g_staging.ev[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventRecord(g_staging.ev[i], s));
        }
        g_staging.device = device;
    }
    int k = 0;
    for (size_t off = 0; off < bytes; off += Staging::kChunk, k ^= 1) {
        const size_t n = std::min(Staging::kChunk, bytes - off);
        CUDA_TRY(cudaEventSynchronize(g_staging.ev[k]));
        parallel_memcpy(g_staging.buf[k], static_cast<const char*>(src) + off, n);
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(dst) + off, g_staging.buf[k], n, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaEventRecord(g_staging.ev[k], s));
    }
    // the staging buffers are reused by the next call only after its events
    CUDA_TRY(cudaEventSynchronize(g_staging.ev[k ^ 1]));
}

inline int sm_count(int device) {
    int n = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    return n;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CUDA_TRY(cudaGetDevice(&prev));
        if (prev != dev) CUDA_TRY(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

inline int build_grid(int device) { return sm_count(device) * 8; }

} // namespace bsccs_b200
