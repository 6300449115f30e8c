// k_excess.cu — K6: the sparse excess of the capped threshold layers.
//
// S_ij = sum_tau min(n_i(tau), n_j(tau))                       (reading A1)
//      = sum_tau min(min(n_i, T), min(n_j, T))                 dense: K5 on the capped indicator
//      + sum_tau min((n_i - T)+, (n_j - T)+)                   sparse: this file
// (exact for every integer T >= 0). With the cap T_s = 1 of config 4 the
// dense contraction shrinks from K = sum_tau max_i n_i(tau) ~ 16.7k to <= V = 8000 columns,
// while only ~1 % of (row, tau) entries exceed the cap (9.6 per row); they form short per-k-mer
// lists L_tau (k_xfill), and a row's excess partners are the union of its lists.
//
// Rows and columns are positions in the shard's length order (sigma); the lists hold positions.
// k_xrows (Gustavson's row-by-row sparse product, one warp per row i of a capped shard):
//   acc[j] += min(x_i(tau), x_j(tau))  for every tau with x_i(tau) = (n_i(tau) - T)+ > 0 and
//                                      every j > i in L_tau        (u8 lanes in shared memory)
//   then the row's upper part acc[(i+1) & ~15 ..] is copied with 16-byte stores to the dense
//   excess matrix E_s[i][.] (u8, row pitch w rounded up to 16) and acc is cleared again;
//   xrow[i].x = 1 if the row has any excess (rows without it are never read).
// The K5 kernel's staging warp bulk-copies each tile's 240-byte row segments of E into shared
// memory, and the epilogue adds e_ij to the tensor-core S before the fixed point (entries at
// j <= i are never written and never used: the epilogue masks those pairs). The host picks T_s
// so that max_i sum_tau x_i(tau) <= 255: every e_ij then fits its byte and the packed 32-bit
// shared-memory adds never carry into a neighbour. Integer addition is associative, so the
// result is independent of the atomic order.
#include <algorithm>

#include "sad_internal.cuh"

namespace sad {

constexpr int kXrWarps = 8;
#ifndef SAD_XR_BATCH
#define SAD_XR_BATCH 8                  // list entries per lane in flight (one round trip per 32 * batch)
#endif
#ifndef SAD_XROWS_GLOBAL
#define SAD_XROWS_GLOBAL 1   // 1: accumulate each row's excess in place in E (global); 0: shared-memory rows
#endif

// K6 lists: every entry above its shard's cap goes to L_tau as (row << 8) | (n - T_s), one warp
// per row over the row's count >= 2 entries (its CSR tail; positions from per-(shard, tau) cursors).
// lpos != NULL: the length order's slot scatter (k_lenscatter) fused in: lane 0 takes the row's
// sorted position from its Tw bin and writes sigma, sigma_inv and the sorted RowInfo (one launch
// and one grid-wide pass fewer per step).
__global__ void __launch_bounds__(256) k_xfill(ExcessArgs a, uint32_t *xcur, uint32_t *lpos, int32_t *sigma,
                                               int32_t *sigma_inv, RowInfo *rinfo_s) {
    __shared__ unsigned long long lbase[kMaxLocalShards + 1];
    if (blockIdx.x == 0 && threadIdx.x < 16 && a.zero_seg)
        reinterpret_cast<uint4 *>(a.zero_seg)[threadIdx.x] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        unsigned long long acc = 0;
        for (int s = 0; s < a.pl; ++s) {
            lbase[s] = acc;
            acc += a.xtot[s];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * 8;
    for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < a.n; r += nw) {
        RowInfo ri = a.rowinfo[r];
        const int s = (int)ri.shard;              // input order: K1/K2 recorded the row's shard
        uint32_t local;                           // the row's position in length order
        if (lpos) {
            uint32_t p = 0;
            if (lane == 0) {
                const int64_t b = a.shard_base[s];
                p = atomicAdd(&lpos[(size_t)s * kLenBinsMax + ri.tw], 1u);   // global sorted position
                sigma[p] = (int32_t)(r - b);
                sigma_inv[r] = (int32_t)(p - b);
                ri.shard = (uint32_t)(r - b);
                rinfo_s[p] = ri;
                p -= (uint32_t)b;
            }
            local = __shfl_sync(0xffffffffu, p, 0);
        } else {
            local = (uint32_t)a.sigma_inv[r];
        }
        const uint32_t T = a.cap[s];
        if (T == kNoCap) continue;
        const int dh = a.nhi[r];                  // the count >= 2 entries: the row's CSR tail
        const uint32_t *ent = a.csr + (a.off[r + 1] - (r + 1) * (int64_t)(a.k - 1)) - dh;
        for (int e = lane; e < dh; e += 32) {
            const uint32_t v = ent[e], n = v & 0xFFFFu;
            if (n > T) {
                const uint32_t key = (uint32_t)s * (uint32_t)a.V + (v >> 16);
                const uint32_t pos = atomicAdd(&xcur[key], 1u);
                const_cast<uint32_t *>(a.lists)[lbase[s] + a.xoff[key] + pos] = (local << 8) | (n - T);
            }
        }
    }
}

void launch_xfill(const ExcessArgs &a, uint32_t *xcur, uint32_t *lpos, int32_t *sigma, int32_t *sigma_inv,
                  RowInfo *rinfo_s, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>((int64_t)sms * 8, (a.n + 7) / 8);
    if (grid > 0) k_xfill<<<(unsigned)grid, 256, 0, st>>>(a, xcur, lpos, sigma, sigma_inv, rinfo_s);
}

__global__ void __launch_bounds__(kXrWarps * 32) k_xrows(ExcessArgs a, int warps) {
    extern __shared__ __align__(16) uint8_t xsm[];
    __shared__ unsigned long long lbase[kMaxLocalShards + 1];
    __shared__ uint32_t sg_end[kXrWarps][32], sg_src[kXrWarps][32], sg_xa[kXrWarps][32];   // per-batch list segments
    if (threadIdx.x == 0) {
        unsigned long long acc = 0;
        for (int s = 0; s < a.pl; ++s) {
            lbase[s] = acc;
            acc += a.xtot[s];
        }
    }
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (wid >= warps) return;
    uint8_t *acc = xsm + (size_t)wid * a.accb;
    uint32_t *acc32 = reinterpret_cast<uint32_t *>(acc);
    uint4 *acc4 = reinterpret_cast<uint4 *>(acc);
    for (int t = lane; t < a.accb / 16; t += 32) acc4[t] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    const int64_t nw = (int64_t)gridDim.x * warps;
    for (int64_t r = (int64_t)blockIdx.x * warps + wid; r < a.n; r += nw) {
        int s = 0;
        while (s + 1 < a.pl && r >= a.shard_base[s + 1]) ++s;
        const uint32_t T = a.cap[s];
        const uint32_t local = (uint32_t)(r - a.shard_base[s]);          // sorted position (length order)
        const int64_t i = a.shard_base[s] + a.sigma[r];                  // the sequence there
        const int64_t w = a.shard_base[s + 1] - a.shard_base[s];
        uint32_t distinct = 0;
        if (T != kNoCap) {
            const int d = a.nhi[i];               // the row's count >= 2 entries: its CSR tail
            const uint32_t *ent = a.csr + (a.off[i + 1] - (i + 1) * (int64_t)(a.k - 1)) - d;
            for (int e0 = 0; e0 < d; e0 += 32) {
                // the batch's excess k-mers: lane-parallel list lookups, then one flattened walk
                // over the concatenated lists (4 independent loads in flight per lane)
                const int e = e0 + lane;
                const uint32_t v = e < d ? ent[e] : 0u;
                const bool hit = (v & 0xFFFFu) > T;
                const uint32_t mask = __ballot_sync(0xffffffffu, hit);
                if (!mask) continue;
                uint32_t len = 0;
                if (hit) {
                    const uint32_t key = (uint32_t)s * (uint32_t)a.V + (v >> 16);
                    const uint32_t o0 = a.xoff[key];
                    const uint32_t o1 = (v >> 16) + 1 < (uint32_t)a.V ? a.xoff[key + 1] : (uint32_t)a.xtot[s];
                    len = o1 - o0;
                    const int hrank = __popc(mask & ((1u << lane) - 1u));
                    sg_src[wid][hrank] = (uint32_t)(lbase[s] + o0);
                    sg_xa[wid][hrank] = (v & 0xFFFFu) - T;
                }
                uint32_t incl = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (hit) sg_end[wid][__popc(mask & ((1u << lane) - 1u))] = incl;
                const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
                __syncwarp();
                int g = 0;
                for (uint32_t t0 = 0; t0 < tot; t0 += 32 * SAD_XR_BATCH) {
                    uint32_t vb[SAD_XR_BATCH], xa[SAD_XR_BATCH];
#pragma unroll
                    for (int u = 0; u < SAD_XR_BATCH; ++u) {
                        const uint32_t t = t0 + (uint32_t)(u * 32 + lane);
                        vb[u] = 0;
                        xa[u] = 0;
                        if (t < tot) {
                            while (t >= sg_end[wid][g]) ++g;
                            const uint32_t st = g ? sg_end[wid][g - 1] : 0u;
                            vb[u] = a.lists[sg_src[wid][g] + (t - st)];
                            xa[u] = sg_xa[wid][g];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < SAD_XR_BATCH; ++u) {
                        const uint32_t b = vb[u] >> 8;
                        if (xa[u] && b > local) {
                            const uint32_t sh = 8u * (b & 3u);
                            atomicAdd(&acc32[b >> 2], min(xa[u], vb[u] & 0xFFu) << sh);
                            distinct = 1u;
                        }
                    }
                }
                __syncwarp();
            }
        }
        const bool any = __any_sync(0xffffffffu, distinct != 0u);
        if (lane == 0) a.xrow[r] = make_uint2(any ? 1u : 0u, 0u);
        if (any) {                              // the row's upper part -> E_s[i], acc cleared
            const int nch = (int)((w + 15) >> 4);
            uint4 *dst = reinterpret_cast<uint4 *>(a.E + a.ebase[s] + (int64_t)local * (nch * 16));
            for (int c = (int)((local + 1) >> 4) + lane; c < nch; c += 32) {
                dst[c] = acc4[c];
                acc4[c] = make_uint4(0, 0, 0, 0);
            }
        }
        __syncwarp();
    }
}

// The same product with the row's dense excess bytes accumulated in place, in E (global memory,
// L2-resident while the warp works on the row): the row's upper part is zeroed when its first
// excess k-mer appears, then the partners' bytes are added with fire-and-forget 32-bit atomics
// (no carry: every e_ij <= 255). No shared-memory accumulator, so occupancy is not bounded by w.
#ifndef SAD_XR_MINB
#define SAD_XR_MINB 5
#endif
__global__ void __launch_bounds__(kXrWarps * 32, SAD_XR_MINB) k_xrows_g(ExcessArgs a) {
    __shared__ unsigned long long lbase[kMaxLocalShards + 1];
    __shared__ uint32_t sg_end[kXrWarps][32], sg_src[kXrWarps][32], sg_xa[kXrWarps][32];   // per-batch list segments
    if (threadIdx.x == 0) {
        unsigned long long acc = 0;
        for (int s = 0; s < a.pl; ++s) {
            lbase[s] = acc;
            acc += a.xtot[s];
        }
    }
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * kXrWarps;
    // the next row's sequence index, CSR position and first entry batch are fetched during the
    // current row (a three-step dependent chain: sigma -> off / nhi -> entries)
    int64_t r = (int64_t)blockIdx.x * kXrWarps + wid;
    int64_t i_c = r < a.n ? a.shard_base[0] + 0 : 0;
    auto seq_of = [&](int64_t rr) {
        int s = 0;
        while (s + 1 < a.pl && rr >= a.shard_base[s + 1]) ++s;
        return a.shard_base[s] + a.sigma[rr];
    };
    i_c = r < a.n ? seq_of(r) : 0;
    int d_c = r < a.n ? a.nhi[i_c] : 0;
    int64_t eo_c = r < a.n ? a.off[i_c + 1] - (i_c + 1) * (int64_t)(a.k - 1) - d_c : 0;   // the CSR tail
    uint32_t v_c = lane < d_c ? a.csr[eo_c + lane] : 0u;
    for (; r < a.n; r += nw) {
        int s = 0;
        while (s + 1 < a.pl && r >= a.shard_base[s + 1]) ++s;
        const uint32_t local = (uint32_t)(r - a.shard_base[s]);          // sorted position (length order)
        // tile split: rows of row blocks another rank computes need no excess here
        const uint32_t T = (a.rb_own && !a.rb_own[(a.shard_rowpad[s] + local) / a.rb_rows]) ? kNoCap : a.cap[s];
        const int64_t w = a.shard_base[s + 1] - a.shard_base[s];
        const int nch = (int)((w + 15) >> 4);
        uint8_t *erow = a.E + a.ebase[s] + (int64_t)local * (nch * 16);
        const int64_t rn = r + nw;
        const int64_t i_n = rn < a.n ? seq_of(rn) : 0;                   // step 1 of the next row
        int64_t eo_n = 0;
        int d_n = 0;
        bool zeroed = false;
        if (T != kNoCap) {
            const uint32_t *ent = a.csr + eo_c;
            const int d = d_c;                    // the row's count >= 2 entries lead its CSR
            for (int e0 = 0; e0 < d; e0 += 32) {
                const int e = e0 + lane;
                const uint32_t v = e0 == 0 ? v_c : (e < d ? ent[e] : 0u);
                const bool hit = (v & 0xFFFFu) > T;
                const uint32_t mask = __ballot_sync(0xffffffffu, hit);
                if (!mask) continue;
                if (!zeroed) {                    // the row's upper part, once
                    for (int c = (int)((local + 1) >> 4) + lane; c < nch; c += 32)
                        reinterpret_cast<uint4 *>(erow)[c] = make_uint4(0, 0, 0, 0);
                    zeroed = true;
                    __syncwarp();                 // orders the zeros before every lane's atomics
                }
                uint32_t len = 0;
                if (hit) {
                    const uint32_t key = (uint32_t)s * (uint32_t)a.V + (v >> 16);
                    const uint32_t o0 = a.xoff[key];
                    const uint32_t o1 = (v >> 16) + 1 < (uint32_t)a.V ? a.xoff[key + 1] : (uint32_t)a.xtot[s];
                    len = o1 - o0;
                    const int hrank = __popc(mask & ((1u << lane) - 1u));
                    sg_src[wid][hrank] = (uint32_t)(lbase[s] + o0);
                    sg_xa[wid][hrank] = (v & 0xFFFFu) - T;
                }
                uint32_t incl = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (hit) sg_end[wid][__popc(mask & ((1u << lane) - 1u))] = incl;
                const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
                __syncwarp();
                if (e0 == 0 && rn < a.n) {        // step 2 of the next row
                    d_n = a.nhi[i_n];
                    eo_n = a.off[i_n + 1] - (i_n + 1) * (int64_t)(a.k - 1) - d_n;
                }
                int g = 0;
                for (uint32_t t0 = 0; t0 < tot; t0 += 32 * SAD_XR_BATCH) {
                    uint32_t vb[SAD_XR_BATCH], xa[SAD_XR_BATCH];
#pragma unroll
                    for (int u = 0; u < SAD_XR_BATCH; ++u) {
                        const uint32_t t = t0 + (uint32_t)(u * 32 + lane);
                        vb[u] = 0;
                        xa[u] = 0;
                        if (t < tot) {
                            while (t >= sg_end[wid][g]) ++g;
                            const uint32_t st = g ? sg_end[wid][g - 1] : 0u;
                            vb[u] = a.lists[sg_src[wid][g] + (t - st)];
                            xa[u] = sg_xa[wid][g];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < SAD_XR_BATCH; ++u) {
                        const uint32_t b = vb[u] >> 8;
                        if (xa[u] && b > local)
                            atomicAdd(reinterpret_cast<uint32_t *>(erow + (b & ~3u)),
                                      min(xa[u], vb[u] & 0xFFu) << (8u * (b & 3u)));
                    }
                }
                __syncwarp();
            }
        }
        if (lane == 0) a.xrow[r] = make_uint2(zeroed ? 1u : 0u, 0u);
        if (rn < a.n) {
            if (!d_n && !eo_n) {                  // step 2 not issued above (no hit batch in this row)
                d_n = a.nhi[i_n];
                eo_n = a.off[i_n + 1] - (i_n + 1) * (int64_t)(a.k - 1) - d_n;
            }
            v_c = lane < d_n ? a.csr[eo_n + lane] : 0u;                  // step 3
        }
        eo_c = eo_n;
        d_c = d_n;
    }
}

int launch_excess(const ExcessArgs &a, cudaStream_t st) {
    if (SAD_XROWS_GLOBAL) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_xrows_g, kXrWarps * 32, 0);
#ifndef SAD_K6_DIV
#define SAD_K6_DIV 1                      // K6 takes 1/SAD_K6_DIV of the resident blocks (K4 runs beside it)
#endif
        const int64_t grid = std::min<int64_t>((int64_t)sms * std::max(per_sm / SAD_K6_DIV, 1),
                                               (a.n + kXrWarps - 1) / kXrWarps);
        if (grid > 0) k_xrows_g<<<(unsigned)grid, kXrWarps * 32, 0, st>>>(a);
        return 0;
    }
    const int warps = (int)std::min<int64_t>(kXrWarps, (int64_t)kXrSmem / a.accb);
    if (warps < 1) return -1;
    const size_t smem = (size_t)warps * a.accb;
    smem_optin(k_xrows, (size_t)kXrSmem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_xrows, kXrWarps * 32, smem);
    int64_t grid = (int64_t)sms * std::max(per_sm, 1);
    grid = std::min<int64_t>(grid, (a.n + warps - 1) / warps);
    if (grid > 0) k_xrows<<<(unsigned)grid, kXrWarps * 32, smem, st>>>(a, warps);
    return 0;
}

}  // namespace sad
