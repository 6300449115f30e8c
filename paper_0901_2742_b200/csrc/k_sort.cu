// k_sort.cu — stable (key, value) radix sort of up to kSmallSortMax pairs inside one thread block
// (cub::BlockRadixSort in shared memory): one launch instead of the 3-8 of a device-wide sort,
// for the per-rank sorts of small shards (many GPUs, small p). Larger inputs use cub::DeviceRadixSort.
#include <cub/block/block_radix_sort.cuh>

#include <algorithm>

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
    if (smem_optin(k_block_sort<K>, smem) != cudaSuccess) return -1;
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
template <int ITEMS, typename KI = uint32_t>
using SegSortT = cub::BlockRadixSort<KI, kSegThreads, ITEMS, int32_t, SAD_SEG_RADIX>;
using SegSort = SegSortT<kSegItems>;
constexpr int kRunItems = 4;                      // run blocks of the rank sort: 512 x 4 = 2048 keys
constexpr int kRunMax = kSegThreads * kRunItems;

// Sub-segment runs: block x sorts run (x % nruns) of segment (x / nruns), the segment split into
// nruns contiguous runs; with nruns = 1 it sorts the whole segment.
__device__ __forceinline__ int64_t run_begin(const int64_t *seg, int s, int r, int nruns) {
    return seg[s] + (seg[s + 1] - seg[s]) * r / nruns;
}

// KI: the key type the block sorts (the bits below end_bit; uint64_t when end_bit > 32)
template <typename K, int ITEMS = kSegItems, typename KI = uint32_t>
__global__ void __launch_bounds__(kSegThreads) k_seg_sort(const K *keys_in, const int32_t *vals_in,
                                                            const int64_t *seg, K *keys_out, int32_t *vals_out,
                                                            int end_bit, int nruns) {
    using BRS = SegSortT<ITEMS, KI>;
    extern __shared__ __align__(16) uint8_t sort_smem[];
    typename BRS::TempStorage &tmp = *reinterpret_cast<typename BRS::TempStorage *>(sort_smem);
    const int sg = blockIdx.x / nruns, rn = blockIdx.x % nruns;
    const int64_t b = run_begin(seg, sg, rn, nruns);
    const int n = (int)(run_begin(seg, sg, rn + 1, nruns) - b);
    if (n <= 0) return;
    const K low = end_bit >= (int)(8 * sizeof(K)) ? ~K(0) : ((K(1) << end_bit) - 1);
    const K high = keys_in[b] & ~low;
    KI k[ITEMS];
    int32_t v[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int idx = threadIdx.x * ITEMS + i;
        k[i] = idx < n ? (KI)(keys_in[b + idx] & low) : ~KI(0);             // padding sorts last (stable)
        v[i] = idx < n ? vals_in[b + idx] : 0;
    }
    BRS(tmp).Sort(k, v, 0, end_bit);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int idx = threadIdx.x * ITEMS + i;
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
    if (end_bit > 32) return -1;
    if (smem_optin(k_seg_sort<K>, smem) != cudaSuccess) return -1;
    k_seg_sort<K><<<nseg, kSegThreads, smem, st>>>(ki, vi, seg, ko, vo, end_bit, 1);
    return 0;
}

// Merge of the nruns sorted runs of every segment: an element's output position is its index in
// its own run plus, for every other run, the number of keys there that precede it -- keys <= it in
// earlier runs, < it in later runs, so equal keys keep run (= input) order: the result is the
// stable sort of the segment.
template <typename K>
__global__ void k_merge_runs(const K *keys, const int32_t *vals, const int64_t *seg, int nseg, int nruns, int64_t n,
                             K *keys_out, int32_t *vals_out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int s = 0;
        while (s + 1 < nseg && i >= seg[s + 1]) ++s;
        int r = 0;
        while (r + 1 < nruns && i >= run_begin(seg, s, r + 1, nruns)) ++r;
        const K key = keys[i];
        int64_t pos = i - run_begin(seg, s, r, nruns);
        for (int q = 0; q < nruns; ++q) {
            if (q == r) continue;
            int64_t lo = run_begin(seg, s, q, nruns), hi = run_begin(seg, s, q + 1, nruns);
            const int64_t b0 = lo;
            while (lo < hi) {                  // first element > key (q < r) or >= key (q > r)
                const int64_t m = (lo + hi) >> 1;
                const K x = keys[m];
                if (q < r ? x <= key : x < key) lo = m + 1; else hi = m;
            }
            pos += lo - b0;
        }
        keys_out[seg[s] + pos] = key;
        vals_out[seg[s] + pos] = vals[i];
    }
}

// The same merge with the whole segment's keys staged in shared memory (one block per segment of
// at most kMergeSmemMax keys): the binary searches run on shared memory instead of L2 latency.
constexpr int kMergeThreads = 1024, kMergeSmemMax = 16384, kMergeMaxRuns = 64;
template <typename K>
__global__ void __launch_bounds__(kMergeThreads) k_merge_runs_smem(const K *keys, const int32_t *vals,
                                                                   const int64_t *seg, int nruns, int bps,
                                                                   K *keys_out, int32_t *vals_out) {
    extern __shared__ __align__(16) uint8_t merge_smem[];
    __shared__ int rb[kMergeMaxRuns + 1];                  // run bounds (the same split as the run sorts)
    K *sk = reinterpret_cast<K *>(merge_smem);
    const int s = blockIdx.x / bps, part = blockIdx.x % bps;   // bps blocks share a segment's elements
    const int64_t b = seg[s];
    const int n = (int)(seg[s + 1] - b);
    if (threadIdx.x <= nruns) rb[threadIdx.x] = (int)((int64_t)n * threadIdx.x / nruns);
    for (int t = threadIdx.x; t < n; t += kMergeThreads) sk[t] = keys[b + t];
    __syncthreads();
    for (int t = part * kMergeThreads + threadIdx.x; t < n; t += bps * kMergeThreads) {
        int r = 0;
        while (r + 1 < nruns && t >= rb[r + 1]) ++r;
        const K key = sk[t];
        int pos = t - rb[r];
        for (int q = 0; q < nruns; ++q) {
            if (q == r) continue;
            int lo = rb[q], hi = rb[q + 1];
            const int b0 = lo;
            while (lo < hi) {                  // first element > key (q < r) or >= key (q > r)
                const int m = (lo + hi) >> 1;
                const K x = sk[m];
                if (q < r ? x <= key : x < key) lo = m + 1; else hi = m;
            }
            pos += lo - b0;
        }
        keys_out[b + pos] = key;
        vals_out[b + pos] = vals[b + t];
    }
}

// the stable sort of every segment: runs of at most kRunMax keys sorted in place by separate blocks
// (512 x 4 items: the block sort's cost follows its capacity, not the run), then merged into
// (ko, vo) by ranking; a segment that fits one run is sorted straight into (ko, vo)
template <typename K, typename KI>
static int seg_sort_runs_t(K *ki, int32_t *vi, const int64_t *seg, int nseg, int64_t max_seg, int64_t n, K *ko,
                           int32_t *vo, int end_bit, cudaStream_t st) {
    const int nruns = (int)std::max<int64_t>(1, (max_seg + kRunMax - 1) / kRunMax);
    const size_t smem = sizeof(typename SegSortT<kRunItems, KI>::TempStorage);
    auto kern = k_seg_sort<K, kRunItems, KI>;
    if (smem_optin(kern, smem) != cudaSuccess) return -1;
    if (nruns == 1) {
        kern<<<nseg, kSegThreads, smem, st>>>(ki, vi, seg, ko, vo, end_bit, 1);
        return 0;
    }
    kern<<<nseg * nruns, kSegThreads, smem, st>>>(ki, vi, seg, ki, vi, end_bit, nruns);
    if (max_seg <= kMergeSmemMax) {
        const size_t ms = (size_t)max_seg * sizeof(K);
        if (smem_optin(k_merge_runs_smem<K>, ms) != cudaSuccess) return -1;
        const int bps = std::max(1, 64 / nseg);      // blocks per segment: ~64 blocks in all
        k_merge_runs_smem<K><<<nseg * bps, kMergeThreads, ms, st>>>(ki, vi, seg, nruns, bps, ko, vo);
    } else {
        const int64_t g = std::min<int64_t>(4096, (n + 255) / 256);
        if (g > 0) k_merge_runs<K><<<(unsigned)g, 256, 0, st>>>(ki, vi, seg, nseg, nruns, n, ko, vo);
    }
    return 0;
}

// end_bit <= 32: the blocks sort 32-bit keys; up to 64: 64-bit keys (more radix passes)
template <typename K>
static int seg_sort_runs(K *ki, int32_t *vi, const int64_t *seg, int nseg, int64_t max_seg, int64_t n, K *ko,
                         int32_t *vo, int end_bit, cudaStream_t st) {
    if (end_bit <= 32) return seg_sort_runs_t<K, uint32_t>(ki, vi, seg, nseg, max_seg, n, ko, vo, end_bit, st);
    if (sizeof(K) == 8 && end_bit <= 64)
        return seg_sort_runs_t<K, unsigned long long>(ki, vi, seg, nseg, max_seg, n, ko, vo, end_bit, st);
    return -1;
}

int seg_sort_pairs_runs(unsigned long long *ki, int32_t *vi, const int64_t *seg, int nseg, int64_t max_seg, int64_t n,
                        unsigned long long *ko, int32_t *vo, int end_bit, cudaStream_t st) {
    return seg_sort_runs<unsigned long long>(ki, vi, seg, nseg, max_seg, n, ko, vo, end_bit, st);
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
