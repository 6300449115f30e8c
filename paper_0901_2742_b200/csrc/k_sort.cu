// k_sort.cu — stable (key, value) radix sort of up to kSmallSortMax pairs inside one thread block
// (cub::BlockRadixSort in shared memory): one launch instead of the 3-8 of a device-wide sort,
// for the per-rank sorts of small shards (many GPUs, small p). Larger inputs use cub::DeviceRadixSort.
#include <cub/block/block_radix_sort.cuh>

#include "sad_internal.cuh"

namespace sad {

constexpr int kSortThreads = 512, kSortItems = 32;

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_block_sort(const K *keys_in, const int32_t *vals_in, int n,
                                                              K *keys_out, int32_t *vals_out, int begin_bit,
                                                              int end_bit) {
    using BRS = cub::BlockRadixSort<K, kSortThreads, kSortItems, int32_t>;
    extern __shared__ __align__(16) uint8_t sort_smem[];
    typename BRS::TempStorage &tmp = *reinterpret_cast<typename BRS::TempStorage *>(sort_smem);
    K k[kSortItems];
    int32_t v[kSortItems];
    const K pad = ~K(0);                       // sorts after every real key (stable: real keys first)
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int idx = threadIdx.x * kSortItems + i;
        k[i] = idx < n ? keys_in[idx] : pad;
        v[i] = idx < n ? vals_in[idx] : 0;
    }
    BRS(tmp).Sort(k, v, begin_bit, end_bit);
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int idx = threadIdx.x * kSortItems + i;
        if (idx < n) {
            keys_out[idx] = k[i];
            vals_out[idx] = v[i];
        }
    }
}

template <typename K>
static int block_sort(const K *ki, const int32_t *vi, int n, K *ko, int32_t *vo, int b0, int b1, cudaStream_t st) {
    using BRS = cub::BlockRadixSort<K, kSortThreads, kSortItems, int32_t>;
    const size_t smem = sizeof(typename BRS::TempStorage);
    static bool configured = false;
    if (!configured) {
        if (cudaFuncSetAttribute(k_block_sort<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return -1;
        configured = true;
    }
    k_block_sort<K><<<1, kSortThreads, smem, st>>>(ki, vi, n, ko, vo, b0, b1);
    return 0;
}

int small_sort_pairs(const uint32_t *ki, const int32_t *vi, int n, uint32_t *ko, int32_t *vo, int b0, int b1,
                     cudaStream_t st) {
    return block_sort<uint32_t>(ki, vi, n, ko, vo, b0, b1, st);
}

int small_sort_pairs(const unsigned long long *ki, const int32_t *vi, int n, unsigned long long *ko, int32_t *vo,
                     int b0, int b1, cudaStream_t st) {
    return block_sort<unsigned long long>(ki, vi, n, ko, vo, b0, b1, st);
}

}  // namespace sad
