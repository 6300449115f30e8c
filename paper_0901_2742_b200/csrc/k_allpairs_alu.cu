// k_allpairs_alu.cu — K5': all-pairs within each shard on the CUDA cores (the baseline the
// tensor-core path must beat; SAD_F_KERNEL_ALU).
//
//   S_ij = sum_tau min(n_i(tau), n_j(tau))            (reading A1)
//   q_ij = floor(2^32 S_ij / (min(L_i,L_j) - k + 1))   (reading A5)
//   T_i  = sum_{j in shard} q_ij                        (reading A3)
//
// Dense uint16 count rows, two k-mers per 32-bit word: per word pair one VIMNMX.U16x2 and
// one VIADD.U16x2. 64x64 pair tiles on the upper triangle of each shard, 256 threads, 4x4
// pairs per thread, operands staged in shared memory.
#include "sad_internal.cuh"

namespace sad {

constexpr int kAT = 64;        // pair tile edge
constexpr int kAKW = 32;       // words per stage
constexpr int kAThreads = 256;

__device__ __forceinline__ void tile_of(int64_t t, int64_t &I, int64_t &J) {
    // t enumerates {(I, J): I <= J} as J(J+1)/2 + I
    int64_t j = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (j * (j + 1) / 2 > t) --j;
    while ((j + 1) * (j + 2) / 2 <= t) ++j;
    J = j;
    I = t - j * (j + 1) / 2;
}

__global__ void __launch_bounds__(kAThreads) k_allpairs_alu(AllPairsArgs a) {
    __shared__ uint32_t As[kAT][kAKW + 1];
    __shared__ uint32_t Bs[kAT][kAKW + 1];
    // locate (shard, I, J)
    const int64_t bid = blockIdx.x;
    int s = 0;
    while (s + 1 < a.pl && bid >= a.tile_base[s + 1]) ++s;
    int64_t I, J;
    tile_of(bid - a.tile_base[s], I, J);
    const int64_t w = a.shard_base[s + 1] - a.shard_base[s];
    const int64_t rowA = a.shard_rowpad[s] + I * kAT, rowB = a.shard_rowpad[s] + J * kAT;
    const uint32_t *op = reinterpret_cast<const uint32_t *>(a.op);
    const int64_t sw = a.stride / 4;       // words per row

    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    uint32_t acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0;

    for (int kw = 0; kw < a.vwords; kw += kAKW) {
        // 64 rows x 32 words per operand = 512 uint4; 2 per thread per operand
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int idx = threadIdx.x + u * kAThreads;   // 0..511
            const int rr = idx >> 3, cc = (idx & 7) * 4;
            const uint4 va = *reinterpret_cast<const uint4 *>(op + (rowA + rr) * sw + kw + cc);
            const uint4 vb = *reinterpret_cast<const uint4 *>(op + (rowB + rr) * sw + kw + cc);
            As[rr][cc] = va.x; As[rr][cc + 1] = va.y; As[rr][cc + 2] = va.z; As[rr][cc + 3] = va.w;
            Bs[rr][cc] = vb.x; Bs[rr][cc + 1] = vb.y; Bs[rr][cc + 2] = vb.z; Bs[rr][cc + 3] = vb.w;
        }
        __syncthreads();
#pragma unroll 8
        for (int q = 0; q < kAKW; ++q) {
            uint32_t ra[4], rb[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) ra[r] = As[ty + 16 * r][q];
#pragma unroll
            for (int c = 0; c < 4; ++c) rb[c] = Bs[tx + 16 * c][q];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = __vadd2(acc[r][c], __vminu2(ra[r], rb[c]));
        }
        __syncthreads();
    }

    // fused epilogue: exact fixed point, row and column partial sums of T
    const RowInfo *ri = a.rowinfo + a.shard_base[s];
    unsigned long long rs[4] = {0, 0, 0, 0}, cs[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t gi = I * kAT + ty + 16 * r;
        if (gi >= w) continue;
        const RowInfo rI = ri[gi];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int64_t gj = J * kAT + tx + 16 * c;
            if (gj >= w || gj < gi) continue;
            const uint32_t S = (acc[r][c] & 0xFFFFu) + (acc[r][c] >> 16);
            const uint64_t qv = pair_q(S, rI, ri[gj]);
            rs[r] += qv;
            if (gj != gi) cs[c] += qv;
            if (a.sim) {
                uint16_t *sm = a.sim + a.sim_base[s];
                sm[gi * w + gj] = (uint16_t)S;
                sm[gj * w + gi] = (uint16_t)S;
            }
        }
    }
    // rows: reduce over the 16 tx lanes sharing ty
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], o);
        const int64_t gi = I * kAT + ty + 16 * r;
        if (tx == 0 && gi < w && rs[r]) atomicAdd(&a.T[a.shard_base[s] + gi], rs[r]);
    }
    // columns: reduce over the two ty values of the warp
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        cs[c] += __shfl_xor_sync(0xffffffffu, cs[c], 16);
        const int64_t gj = J * kAT + tx + 16 * c;
        if ((threadIdx.x & 16) == 0 && gj < w && cs[c]) atomicAdd(&a.T[a.shard_base[s] + gj], cs[c]);
    }
}

void launch_allpairs_alu(const AllPairsArgs &a, cudaStream_t st) {
    if (a.n_tiles > 0) k_allpairs_alu<<<(unsigned)a.n_tiles, kAThreads, 0, st>>>(a);
}

}  // namespace sad
