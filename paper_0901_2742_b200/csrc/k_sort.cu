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

// Segmented variant: block b sorts segment [seg[b], seg[b+1]) (at most kSmallSortMax pairs) by bits
// [0, end_bit) of its keys, stably; the bits above end_bit are the same within a segment (the
// shard) and are carried over from the segment's first key. One launch for every shard of a rank.
#ifndef SAD_SEG_THREADS
#define SAD_SEG_THREADS 512
#endif
#ifndef SAD_SEG_RADIX
#define SAD_SEG_RADIX 4
#endif
constexpr int kSegThreads = SAD_SEG_THREADS, kSegItems = kSmallSortMax / SAD_SEG_THREADS;
using SegSort = cub::BlockRadixSort<uint32_t, kSegThreads, kSegItems, int32_t, SAD_SEG_RADIX>;

template <typename K>
__global__ void __launch_bounds__(kSegThreads) k_seg_sort(const K *keys_in, const int32_t *vals_in,
                                                            const int64_t *seg, K *keys_out, int32_t *vals_out,
                                                            int end_bit) {
    using BRS = SegSort;
    extern __shared__ __align__(16) uint8_t sort_smem[];
    typename BRS::TempStorage &tmp = *reinterpret_cast<typename BRS::TempStorage *>(sort_smem);
    const int64_t b = seg[blockIdx.x];
    const int n = (int)(seg[blockIdx.x + 1] - b);
    if (n <= 0) return;
    const K low = end_bit >= (int)(8 * sizeof(K)) ? ~K(0) : ((K(1) << end_bit) - 1);
    const K high = keys_in[b] & ~low;
    uint32_t k[kSegItems];
    int32_t v[kSegItems];
#pragma unroll
    for (int i = 0; i < kSegItems; ++i) {
        const int idx = threadIdx.x * kSegItems + i;
        k[i] = idx < n ? (uint32_t)(keys_in[b + idx] & low) : 0xFFFFFFFFu;   // padding sorts last (stable)
        v[i] = idx < n ? vals_in[b + idx] : 0;
    }
    BRS(tmp).Sort(k, v, 0, end_bit);
#pragma unroll
    for (int i = 0; i < kSegItems; ++i) {
        const int idx = threadIdx.x * kSegItems + i;
        if (idx < n) {
            keys_out[b + idx] = high | (K)k[i];
            vals_out[b + idx] = v[i];
        }
    }
}

template <typename K>
static int seg_sort(const K *ki, const int32_t *vi, const int64_t *seg, int nseg, K *ko, int32_t *vo, int end_bit,
                    cudaStream_t st) {
    using BRS = SegSort;
    const size_t smem = sizeof(typename BRS::TempStorage);
    static bool configured = false;
    if (end_bit > 32) return -1;
    if (!configured) {
        if (cudaFuncSetAttribute(k_seg_sort<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return -1;
        configured = true;
    }
    k_seg_sort<K><<<nseg, kSegThreads, smem, st>>>(ki, vi, seg, ko, vo, end_bit);
    return 0;
}

int seg_sort_pairs(const uint32_t *ki, const int32_t *vi, const int64_t *seg, int nseg, uint32_t *ko, int32_t *vo,
                   int end_bit, cudaStream_t st) {
    return seg_sort<uint32_t>(ki, vi, seg, nseg, ko, vo, end_bit, st);
}

int seg_sort_pairs(const unsigned long long *ki, const int32_t *vi, const int64_t *seg, int nseg,
                   unsigned long long *ko, int32_t *vo, int end_bit, cudaStream_t st) {
    return seg_sort<unsigned long long>(ki, vi, seg, nseg, ko, vo, end_bit, st);
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
