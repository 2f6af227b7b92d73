// Device memory pool behind DevBuf (see npc_internal.cuh): size-classed free lists per device.
#include <cstdlib>
#include <map>
#include <mutex>

#include "npc_internal.cuh"

namespace npc {

namespace {

constexpr size_t POOL_MIN = 1u << 20;  // smaller blocks go straight to cudaMalloc / cudaFree

struct Pool {
    std::mutex mu;
    std::map<int, std::multimap<size_t, void *>> free_by_dev;  // device -> (bytes -> block)
    size_t cached = 0, limit = 0;
    Pool() {
        const char *e = getenv("NPC_POOL_MB");
        limit = (size_t)(e ? atoll(e) : 16384) << 20;
    }
    // release every cached block of a device (caller holds mu)
    void flush(int dev) {
        auto it = free_by_dev.find(dev);
        if (it == free_by_dev.end()) return;
        for (auto &kv : it->second) {
            cudaFree(kv.second);
            cached -= kv.first;
        }
        it->second.clear();
    }
};

Pool &pool() {
    static Pool *p = new Pool();  // never destroyed: blocks may be released during exit
    return *p;
}

// Exact sizes (to 256 B): the repeated solves this pool serves ask for the same sizes, and
// nothing is wasted on rounding.
size_t size_class(size_t n) { return n < POOL_MIN ? n : (n + 255) / 256 * 256; }

}  // namespace

cudaError_t pool_alloc(void **p, size_t bytes) {
    const size_t want = size_class(bytes);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (want >= POOL_MIN) {
        Pool &P = pool();
        std::lock_guard<std::mutex> lk(P.mu);
        auto &fl = P.free_by_dev[dev];
        auto it = fl.find(want);
        if (it != fl.end()) {
            *p = it->second;
            fl.erase(it);
            P.cached -= want;
            return cudaSuccess;
        }
    }
    e = cudaMalloc(p, want);
    if (e == cudaErrorMemoryAllocation && want >= POOL_MIN) {
        cudaGetLastError();  // clear, flush this device's cache, retry once
        Pool &P = pool();
        {
            std::lock_guard<std::mutex> lk(P.mu);
            P.flush(dev);
        }
        e = cudaMalloc(p, want);
    }
    return e;
}

void pool_free(void *p, size_t req) {
    if (!p) return;
    const size_t bytes = size_class(req);
    if (bytes < POOL_MIN) {
        cudaFree(p);
        return;
    }
    int dev = 0;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess) dev = at.device;
    else cudaGetLastError();
    {
        int prev = -1;
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
        cudaDeviceSynchronize();  // as cudaFree would: no kernel may still use the block
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
    Pool &P = pool();
    std::lock_guard<std::mutex> lk(P.mu);
    if (P.cached + bytes > P.limit) {
        cudaFree(p);
        return;
    }
    P.free_by_dev[dev].emplace(bytes, p);
    P.cached += bytes;
}

}  // namespace npc
