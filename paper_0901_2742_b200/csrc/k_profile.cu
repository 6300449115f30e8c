// k_profile.cu — K1/K2 (encode + k-mer counts), K3 (column map), K4/K4' (all-pairs operands).
//
// PAPER.md:40-44 (§2 "k-mer Rank"): "A k-mer is a contiguous subsequence of length k ...
// nx_i(tau) ... the number of times tau occurs in x_i". A window of residue codes
// c_0..c_{k-1} is numbered tau = sum_m c_m A^(k-1-m), so tau order is lexicographic order.
#include <cub/block/block_scan.cuh>

#include "sad_internal.cuh"

namespace sad {

__constant__ char c_alpha[2][24] = {"ACDEFGHIKLMNPQRSTVWY", "ACGT"};

constexpr int kProfThreads = 256;

// K1+K2. Persistent blocks, one sequence at a time. Shared memory: a packed u16 histogram
// (two bins per u32 word; a bin never exceeds L-k+1 <= 65535 so halves never carry), a
// presence bitmap over the V bins and the 256-entry residue table. The bitmap lets the
// compaction visit only words with set bits; bins are cleared as they are read, so the
// histogram is zeroed once per block, not once per sequence.
__global__ void __launch_bounds__(kProfThreads) k_profile(ProfileArgs a) {
    extern __shared__ uint32_t sm[];
    const int V = a.V;
    const int HW = (V + 1) >> 1;             // histogram words
    const int W = (V + 31) >> 5;             // bitmap words
    uint32_t *hist = sm;
    uint32_t *bits = sm + HW;
    uint8_t *lut = reinterpret_cast<uint8_t *>(bits + W);
    typedef cub::BlockScan<uint32_t, kProfThreads> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;

    const int tid = threadIdx.x;
    for (int t = tid; t < HW; t += kProfThreads) hist[t] = 0;
    for (int t = tid; t < W; t += kProfThreads) bits[t] = 0;
    for (int t = tid; t < 256; t += kProfThreads) lut[t] = 255;
    __syncthreads();
    if (tid < a.A) lut[(uint8_t)c_alpha[a.alphabet][tid]] = (uint8_t)tid;
    __syncthreads();

    const int k = a.k;
    const uint32_t A = (uint32_t)a.A;
    for (int64_t i = blockIdx.x; i < a.n; i += gridDim.x) {
        const int64_t off0 = a.off[i];
        const int64_t L = a.off[i + 1] - off0;
        const uint8_t *x = a.ascii + off0;
        const unsigned long long gidx = (unsigned long long)(a.first_idx + i);
        // K1: every residue must be a letter of the alphabet (reading A18)
        for (int64_t t = tid; t < L; t += kProfThreads)
            if (lut[x[t]] == 255) atomicMin(&a.err[0], (gidx << 32) | (unsigned long long)t);
        int s = 0;
        while (s + 1 < a.pl && i >= a.shard_base[s + 1]) ++s;
        if (L < k) {                                     // reading A19
            if (tid == 0) {
                atomicMin(&a.err[1], gidx);
                a.rowinfo[i] = RowInfo{1u, 0xFFFFFFFFu, 1u, (uint32_t)s};
                a.dcnt[i] = 0;
            }
            continue;
        }
        const int64_t Tw = L - k + 1;
        if (Tw > 65535) {                                 // SURVEY A.3 precondition
            if (tid == 0) {
                atomicMin(&a.err[2], gidx);
                a.rowinfo[i] = RowInfo{1u, 0xFFFFFFFFu, 1u, (uint32_t)s};
                a.dcnt[i] = 0;
            }
            continue;
        }
        // K2: count every window (overlaps included)
        for (int64_t t = tid; t < Tw; t += kProfThreads) {
            uint32_t tau = 0;
            for (int m = 0; m < k; ++m) {
                uint32_t c = lut[x[t + m]];
                tau = tau * A + (c == 255 ? 0u : c);
            }
            atomicAdd(&hist[tau >> 1], (tau & 1) ? 0x10000u : 1u);
            atomicOr(&bits[tau >> 5], 1u << (tau & 31));
        }
        __syncthreads();
        // compaction in tau order: contiguous word range per thread, block exclusive scan
        const int per = (W + kProfThreads - 1) / kProfThreads;
        const int w0 = min(W, tid * per), w1 = min(W, w0 + per);
        uint32_t cnt = 0;
        for (int w = w0; w < w1; ++w) cnt += __popc(bits[w]);
        uint32_t pos, total;
        Scan(scan_tmp).ExclusiveSum(cnt, pos, total);
        uint32_t *out = a.csr + (off0 - i * (int64_t)(k - 1));
        uint32_t *Ms = a.M + (size_t)s * V;
        for (int w = w0; w < w1; ++w) {
            uint32_t b = bits[w];
            while (b) {
                const int bit = __ffs(b) - 1;
                b &= b - 1;
                const uint32_t tau = (uint32_t)w * 32u + (uint32_t)bit;
                const uint32_t hw = hist[tau >> 1];
                const uint32_t c = (tau & 1) ? (hw >> 16) : (hw & 0xFFFFu);
                out[pos++] = (tau << 16) | c;
                atomicMax(&Ms[tau], c);
            }
        }
        __syncthreads();
        for (int w = w0; w < w1; ++w) {                  // clear the touched bins
            uint32_t b = bits[w];
            while (b) {
                const int bit = __ffs(b) - 1;
                b &= b - 1;
                hist[((uint32_t)w * 32u + (uint32_t)bit) >> 1] = 0;
            }
            bits[w] = 0;
        }
        if (tid == 0) {
            a.dcnt[i] = (int32_t)total;
            const uint32_t tw = (uint32_t)Tw;
            a.rowinfo[i] = RowInfo{tw, 0xFFFFFFFFu / tw, 0xFFFFFFFFu % tw + 1u, (uint32_t)s};
            atomicAdd(&a.kinfo[s * 4 + 0], (unsigned long long)Tw);
            atomicAdd(&a.kinfo[s * 4 + 1], (unsigned long long)total);
        }
        __syncthreads();
    }
}

void launch_profile(const ProfileArgs &a, cudaStream_t st) {
    const int HW = (a.V + 1) / 2, W = (a.V + 31) / 32;
    const size_t smem = (size_t)(HW + W) * 4 + 256;
    static int configured_for = -1;
    if ((int)smem > 48 * 1024 && configured_for < (int)smem) {
        cudaFuncSetAttribute(k_profile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured_for = (int)smem;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_profile, kProfThreads, smem);
    int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (grid > a.n) grid = a.n;
    if (grid < 1) grid = 1;
    k_profile<<<(unsigned)grid, kProfThreads, smem, st>>>(a);
}

// K3: per shard, col0(tau) = exclusive scan of M(tau) over tau, K_s = sum_tau M(tau).
// Column block [col0(tau), col0(tau)+M(tau)) holds the threshold layers t = 1..M(tau)
// of k-mer tau (SURVEY Appendix A.1 with T = infinity: min(a,b) = sum_t [a>=t][b>=t]).
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) k_colmap(const uint32_t *M, uint32_t *col0,
                                                         unsigned long long *kinfo, int V) {
    typedef cub::BlockScan<unsigned long long, kScanThreads> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const int s = blockIdx.x;
    const uint32_t *m = M + (size_t)s * V;
    uint32_t *c = col0 + (size_t)s * V;
    const int per = (V + kScanThreads - 1) / kScanThreads;
    const int t0 = min(V, (int)threadIdx.x * per), t1 = min(V, t0 + per);
    unsigned long long sum = 0;
    for (int t = t0; t < t1; ++t) sum += m[t];
    unsigned long long base, total;
    Scan(tmp).ExclusiveSum(sum, base, total);
    for (int t = t0; t < t1; ++t) {
        c[t] = (uint32_t)base;
        base += m[t];
    }
    if (threadIdx.x == 0) kinfo[s * 4 + 2] = total;
}

void launch_colmap(const uint32_t *M, uint32_t *col0, unsigned long long *kinfo, int pl, int V, cudaStream_t st) {
    k_colmap<<<pl, kScanThreads, 0, st>>>(M, col0, kinfo, V);
}

__device__ __forceinline__ int shard_of_padded_row(const int64_t *rowpad, int pl, int64_t r) {
    int s = 0;
    while (s + 1 < pl && r >= rowpad[s + 1]) ++s;
    return s;
}

// K4: the binary threshold-indicator operand of the tensor-core path,
//   A_s[i, col0(tau) + t - 1] = 1  for 1 <= t <= n_i(tau)   (uint8, or packed e2m1 nibbles),
// so that (A_s A_s^T)_ij = sum_tau min(n_i(tau), n_j(tau)) = S_ij exactly.
// One block per padded row; the row is assembled in shared memory in 32 KB chunks and
// written with 16-byte coalesced stores (rows are 128-byte aligned).
constexpr int kOpThreads = 256;
constexpr int kOpChunk = 32768;
__global__ void __launch_bounds__(kOpThreads) k_indicator(OperandArgs a) {
    __shared__ __align__(16) uint8_t row[kOpChunk];
    const int64_t r = blockIdx.x;
    const int s = shard_of_padded_row(a.shard_rowpad, a.pl, r);
    const int64_t local = r - a.shard_rowpad[s];
    const int64_t w = a.shard_base[s + 1] - a.shard_base[s];
    const bool real = local < w;
    const int64_t i = a.shard_base[s] + local;
    const uint32_t *ent = real ? a.csr + (a.off[i] - i * (int64_t)(a.k - 1)) : nullptr;
    const int d = real ? a.dcnt[i] : 0;
    const uint32_t *c0 = a.col0 + (size_t)s * a.V;
    uint8_t *dst = reinterpret_cast<uint8_t *>(a.op) + r * a.stride;
    for (int64_t ch = 0; ch < a.stride; ch += kOpChunk) {
        const int len = (int)min((int64_t)kOpChunk, a.stride - ch);
        for (int t = threadIdx.x * 16; t < len; t += kOpThreads * 16)
            *reinterpret_cast<uint4 *>(row + t) = make_uint4(0, 0, 0, 0);
        __syncthreads();
        if (!a.fp4) {
            for (int e = threadIdx.x; e < d; e += kOpThreads) {
                const uint32_t v = ent[e];
                const int64_t lo = (int64_t)c0[v >> 16];
                const int64_t hi = lo + (v & 0xFFFFu);
                const int64_t a0 = max(lo, ch), a1 = min(hi, ch + len);
                for (int64_t c = a0; c < a1; ++c) row[c - ch] = 1;
            }
        } else {
            // two e2m1 entries per byte, 1.0 = 0b0010; neighbouring k-mers may share a byte, so
            // the nibbles are set with 32-bit shared atomics
            uint32_t *row32 = reinterpret_cast<uint32_t *>(row);
            const int64_t c_lo = ch * 2, c_hi = (ch + len) * 2;
            for (int e = threadIdx.x; e < d; e += kOpThreads) {
                const uint32_t v = ent[e];
                const int64_t lo = (int64_t)c0[v >> 16];
                const int64_t hi = lo + (v & 0xFFFFu);
                const int64_t a0 = max(lo, c_lo), a1 = min(hi, c_hi);
                for (int64_t c = a0; c < a1; ++c) {
                    const int64_t cc = c - c_lo;
                    atomicOr(&row32[cc >> 3], 2u << (4 * (cc & 7)));
                }
            }
        }
        __syncthreads();
        for (int t = threadIdx.x * 16; t < len; t += kOpThreads * 16)
            *reinterpret_cast<uint4 *>(dst + ch + t) = *reinterpret_cast<const uint4 *>(row + t);
        __syncthreads();
    }
}

void launch_indicator(const OperandArgs &a, cudaStream_t st) {
    if (a.rows_pad > 0) k_indicator<<<(unsigned)a.rows_pad, kOpThreads, 0, st>>>(a);
}

// K4': dense uint16 count rows n_i(tau), tau = 0..V_pad-1, for the CUDA-core min-sum.
__global__ void __launch_bounds__(kOpThreads) k_dense_counts(OperandArgs a) {
    extern __shared__ __align__(16) uint16_t drow[];
    const int64_t r = blockIdx.x;
    const int s = shard_of_padded_row(a.shard_rowpad, a.pl, r);
    const int64_t local = r - a.shard_rowpad[s];
    const int64_t w = a.shard_base[s + 1] - a.shard_base[s];
    const int nb = (int)a.stride;   // bytes per row (multiple of 128)
    for (int t = threadIdx.x * 16; t < nb; t += kOpThreads * 16)
        *reinterpret_cast<uint4 *>(reinterpret_cast<uint8_t *>(drow) + t) = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (local < w) {
        const int64_t i = a.shard_base[s] + local;
        const uint32_t *ent = a.csr + (a.off[i] - i * (int64_t)(a.k - 1));
        const int d = a.dcnt[i];
        for (int e = threadIdx.x; e < d; e += kOpThreads) drow[ent[e] >> 16] = (uint16_t)(ent[e] & 0xFFFFu);
    }
    __syncthreads();
    uint8_t *dst = reinterpret_cast<uint8_t *>(a.op) + r * a.stride;
    for (int t = threadIdx.x * 16; t < nb; t += kOpThreads * 16)
        *reinterpret_cast<uint4 *>(dst + t) = *reinterpret_cast<const uint4 *>(reinterpret_cast<uint8_t *>(drow) + t);
}

void launch_dense_counts(const OperandArgs &a, cudaStream_t st) {
    const size_t smem = (size_t)a.stride;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(k_dense_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    if (a.rows_pad > 0) k_dense_counts<<<(unsigned)a.rows_pad, kOpThreads, smem, st>>>(a);
}

}  // namespace sad
