// sad_util.cu — host-side helpers shared by the kernel launchers (no device arithmetic).
#include <map>
#include <mutex>
#include <utility>

#include "sad_internal.cuh"

namespace sad {

cudaError_t smem_optin_raw(const void *func, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> done;   // (device, kernel) -> bytes opted in
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return e;
    std::lock_guard<std::mutex> lock(mu);
    size_t &have = done[{dev, func}];
    if (have >= bytes) return cudaSuccess;
    if (cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)) return e;
    have = bytes;
    return cudaSuccess;
}

}  // namespace sad
