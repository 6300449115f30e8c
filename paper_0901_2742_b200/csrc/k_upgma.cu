// k_upgma.cu — SURVEY §8(f) row f4: the UPGMA guide tree of one bucket on the GPU (the first stage
// of the per-bucket progressive aligner, "The k-mer distance can be used to rapidly
// construct phylogenetic trees"; SPEC S:356-364 upgma, decision D-M1).
//
// Input: the bucket's k-mer distances d_ij = 1 - S_ij/den_ij (float64, sad_get_distance_f64), n x n,
// of which only the upper triangle D[min][max] is used (and overwritten). Step t merges the active
// positions i < j with the smallest d, ties -> smallest i then smallest j; the cluster lives at
// position i (its smallest leaf) and gets id n + t; height d/2; average linkage
//   d(k, i u j) = (n_i d(k,i) + n_j d(k,j)) / (n_i + n_j)
// in IEEE float64 with every operation rounded once (explicit _rn intrinsics: no contraction).
//
// One block of 1024 threads per tree. Per row k a cached minimum over its active columns c > k
// (value, smallest c); the argmin of a step is a block reduction over those; after a merge only
// rows whose cached column was i or j (and row i itself) are rescanned (one warp per row), the
// others compare the one changed entry.
#include <cfloat>

#include "sad_internal.cuh"

namespace sad {

constexpr int kUpThreads = 1024;

__device__ __forceinline__ bool better(double v, int64_t c, double bv, int64_t bc) {
    return v < bv || (v == bv && c < bc);
}

// warp-level (min value, smallest column) over active columns c > k of row k
__device__ void row_min(const double *D, const int32_t *act, int64_t n, int64_t k, double &rv, int32_t &rj) {
    const int lane = threadIdx.x & 31;
    double bv = DBL_MAX;
    int64_t bc = INT64_MAX;
    for (int64_t c = k + 1 + lane; c < n; c += 32)
        if (act[c]) {
            const double v = D[k * n + c];
            if (better(v, c, bv, bc)) { bv = v; bc = c; }
        }
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int64_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (better(ov, oc, bv, bc)) { bv = ov; bc = oc; }
    }
    if (lane == 0) {
        rv = bv;
        rj = bc == INT64_MAX ? -1 : (int32_t)bc;
    }
}

__global__ void __launch_bounds__(kUpThreads) k_upgma(double *D, int64_t n, int64_t *merges, double *heights,
                                                      int64_t *sizes, double *rv, int32_t *rj, int64_t *sz,
                                                      int32_t *act, int64_t *cid, int32_t *marks) {
    __shared__ double sv[32];
    __shared__ int64_t si[32];
    __shared__ int64_t mi, mj;
    __shared__ double mv;
    __shared__ int nmark;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int64_t k = tid; k < n; k += kUpThreads) {
        sz[k] = 1;
        act[k] = 1;
        cid[k] = k;
    }
    __syncthreads();
    for (int64_t k = wid; k < n; k += 32) row_min(D, act, n, k, rv[k], rj[k]);
    __syncthreads();
    for (int64_t t = 0; t + 1 < n; ++t) {
        // the closest active pair: min over rows of (cached row minimum, row)
        double bv = DBL_MAX;
        int64_t bi = INT64_MAX;
        for (int64_t k = tid; k < n; k += kUpThreads)
            if (act[k] && rj[k] >= 0 && better(rv[k], k, bv, bi)) { bv = rv[k]; bi = k; }
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0) { sv[wid] = bv; si[wid] = bi; }
        __syncthreads();
        if (wid == 0) {
            bv = sv[lane];
            bi = si[lane];
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
            }
            if (lane == 0) {
                mi = bi;
                mj = rj[bi];
                mv = bv;
                nmark = 0;
                merges[2 * t] = cid[bi];
                merges[2 * t + 1] = cid[rj[bi]];
                heights[t] = __dmul_rn(bv, 0.5);
                sizes[t] = sz[bi] + sz[rj[bi]];
            }
        }
        __syncthreads();
        const int64_t i = mi, j = mj;
        const double ni = (double)sz[i], nj = (double)sz[j], ns = __dadd_rn(ni, nj);
        // average linkage into position i (upper-triangle storage D[min][max])
        for (int64_t k = tid; k < n; k += kUpThreads)
            if (act[k] && k != i && k != j) {
                const double dki = k < i ? D[k * n + i] : D[i * n + k];
                const double dkj = k < j ? D[k * n + j] : D[j * n + k];
                const double v = __ddiv_rn(__dadd_rn(__dmul_rn(ni, dki), __dmul_rn(nj, dkj)), ns);
                if (k < i) D[k * n + i] = v; else D[i * n + k] = v;
            }
        __syncthreads();
        if (tid == 0) {
            sz[i] += sz[j];
            act[j] = 0;
            cid[i] = n + t;
        }
        __syncthreads();
        // cached row minima: rescan rows that pointed at i or j (and row i), else compare d(k, i)
        for (int64_t k = tid; k < n; k += kUpThreads)
            if (act[k]) {
                if (k == i || rj[k] == (int32_t)i || rj[k] == (int32_t)j) {
                    marks[atomicAdd(&nmark, 1)] = (int32_t)k;
                } else if (k < i) {
                    const double v = D[k * n + i];
                    if (better(v, i, rv[k], rj[k] < 0 ? INT64_MAX : rj[k])) { rv[k] = v; rj[k] = (int32_t)i; }
                }
            }
        __syncthreads();
        for (int m = wid; m < nmark; m += 32) {
            const int64_t k = marks[m];
            row_min(D, act, n, k, rv[k], rj[k]);
        }
        __syncthreads();
    }
}

size_t upgma_workspace(int64_t n) { return (size_t)n * (8 + 8 + 8 + 4 + 4 + 4) + 6 * 256 + 256; }

void launch_upgma(double *D, int64_t n, int64_t *merges, double *heights, int64_t *sizes, void *ws, cudaStream_t st) {
    uint8_t *b = reinterpret_cast<uint8_t *>(ws);
    auto take = [&](size_t bytes) {
        uint8_t *p = b;
        b += (bytes + 255) / 256 * 256;
        return p;
    };
    double *rv = reinterpret_cast<double *>(take(8 * n));
    int64_t *sz = reinterpret_cast<int64_t *>(take(8 * n));
    int64_t *cid = reinterpret_cast<int64_t *>(take(8 * n));
    int32_t *rj = reinterpret_cast<int32_t *>(take(4 * n));
    int32_t *act = reinterpret_cast<int32_t *>(take(4 * n));
    int32_t *marks = reinterpret_cast<int32_t *>(take(4 * n));
    k_upgma<<<1, kUpThreads, 0, st>>>(D, n, merges, heights, sizes, rv, rj, sz, act, cid, marks);
}

}  // namespace sad
