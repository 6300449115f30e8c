// k_profile.cu — K1/K2 (encode + k-mer counts), K3 (column map), K4/K4' (all-pairs operands).
//
// PAPER.md:40-44 (§2 "k-mer Rank"): "A k-mer is a contiguous subsequence of length k ...
// nx_i(tau) ... the number of times tau occurs in x_i". A window of residue codes
// c_0..c_{k-1} is numbered tau = sum_m c_m A^(k-1-m), so tau order is lexicographic order.
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "sad_internal.cuh"

namespace sad {

__constant__ char c_alpha[2][24] = {"ACDEFGHIKLMNPQRSTVWY", "ACGT"};

// K1+K2. One warp per sequence (persistent warps over contiguous runs of sequences balanced by
// residues, no block barriers), each with its own shared-memory histogram of byte bins and a staging
// buffer of residue codes (a sequence with a k-mer seen 255 or more times is recounted with u16 bins
// over 1/kWidePasses of the k-mers at a time, which cannot carry since L-k+1 <= 65535).
// Pass 1 validates every residue (K1) and counts every window tau = sum_m c_m A^(k-1-m) (K2); the
// first window of every k-mer (its bin was 0) appends it to an owner list.
// Pass 2 walks the owners: each reads and clears its bin and emits the distinct entry
// (tau << 16 | count) at its list slot, so the histogram is left zeroed for the next sequence.
// The entries are unordered in tau (no consumer needs tau order: operand rows, GA rank and
// ancestor records are all sums or scatters over the entries); the nhi[i] entries with count >= 2
// are repeated in the row's last slots (free: Tw - d = sum (count - 1) >= nhi), so the K6
// consumers read only those. Sequences longer than the staging buffer (or whose owner list does
// not fit beside it) are processed in segments of windows, the bins claimed by atomicAnd.
#ifndef SAD_PROF_BINBITS
#define SAD_PROF_BINBITS 8               // bin width of the k-mer histogram (4 or 8 bits)
#endif
#ifndef SAD_PROF_WARPS
#define SAD_PROF_WARPS 10
#endif
#ifndef SAD_PROF_MINB
#define SAD_PROF_MINB 2                  // blocks per SM the register budget is sized for
#endif
constexpr int kProfWarps = SAD_PROF_WARPS;
constexpr int kBinBits = SAD_PROF_BINBITS, kBinsPerWord = 32 / kBinBits;
constexpr uint32_t kBinMax = (1u << kBinBits) - 1u;
constexpr int kWidePasses = 16 / kBinBits;   // overflow fallback: u16 bins over 1/kWidePasses of the k-mers
#ifndef SAD_PROF_UNROLL
#define SAD_PROF_UNROLL 4
#endif
constexpr int kCountUnroll = SAD_PROF_UNROLL;   // windows per lane per counting step
constexpr int kCodeSeg = 2048;           // residue codes staged per warp
constexpr int kCodeBuf = kCodeSeg + 32;  // staged bytes keep the residues' 16-byte alignment (shift <= 15)

template <int KT>
__device__ __forceinline__ uint32_t window_tau(const uint8_t *c, int k, uint32_t A) {
    uint32_t tau = 0;
    if constexpr (KT > 0) {
#pragma unroll
        for (int m = 0; m < KT; ++m) tau = tau * A + c[m];
    } else {
        for (int m = 0; m < k; ++m) tau = tau * A + c[m];
    }
    return tau;
}

template <int KT>
__global__ void __launch_bounds__(kProfWarps * 32, SAD_PROF_MINB) k_profile(ProfileArgs a, int warps, int hbytes) {
    extern __shared__ __align__(16) uint32_t psm[];
    __shared__ uint8_t lut[256];
    __shared__ int fin_s[kProfWarps];                    // each warp's shard at the end
    __shared__ unsigned long long bk_w, bk_d, bk_tw;     // the block's totals for the first warp's final shard
    __shared__ uint32_t bk_ex[kNumCaps];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = threadIdx.x; t < 256; t += blockDim.x) lut[t] = 255;
    __syncthreads();
    if (threadIdx.x < a.A) lut[(uint8_t)c_alpha[a.alphabet][threadIdx.x]] = (uint8_t)threadIdx.x;
    __syncthreads();
    if (wid >= warps) return;
    const int hw = hbytes / 4;                  // histogram words (V bins, rounded up to 16 bytes)
    const int VW = (a.V + 31) / 32;             // presence words (one bit per k-mer)
    uint32_t *hist = psm + (size_t)wid * (hw + kCodeBuf / 4 + ((VW + 3) & ~3));   // 16-byte aligned slices
    uint8_t *cod = reinterpret_cast<uint8_t *>(hist + hw);
    uint32_t *pres = hist + hw + kCodeBuf / 4;  // k-mers seen by this warp in the current shard
    for (int t = lane; t < hw; t += 32) hist[t] = 0;
    for (int t = lane; t < VW; t += 32) pres[t] = 0;
    // block presence bits (after the warps' slices): zeroed here, written only after the end barrier
    uint32_t *bpres = psm + (size_t)warps * (hw + kCodeBuf / 4 + ((VW + 3) & ~3));
    if (wid == 0) {
        for (int t = lane; t < VW; t += 32) bpres[t] = 0;
        if (lane == 0) bk_w = bk_d = bk_tw = 0;
        if (lane < kNumCaps) bk_ex[lane] = 0;
    }
    __syncwarp();

    const int k = KT > 0 ? KT : a.k;
    const uint32_t A = (uint32_t)a.A;
    const int V = a.V;
    const uint32_t Vh = (uint32_t)(V + kWidePasses - 1) / kWidePasses;   // u16 fallback: k-mers per sub-pass
    const int64_t W = (int64_t)gridDim.x * warps, gw = (int64_t)blockIdx.x * warps + wid;
    // contiguous ranges of sequences balanced by residues (the offsets are the residue prefix), so
    // that a warp with a few long sequences does not trail: the first sequence starting at or after
    // residue r0 + (r1 - r0) gw / W, found by a 32-way warp search over the offsets
    const int64_t r0 = a.off[a.i_begin], rr = a.off[a.i_end] - r0;
    auto first_at = [&](int64_t wq) -> int64_t {
        if (wq <= 0) return a.i_begin;
        if (wq >= W) return a.i_end;
        const int64_t target = r0 + (int64_t)(((__int128)rr * wq) / W);
        int64_t lo = a.i_begin, hi = a.i_end;              // answer in (lo, hi]: off[lo] < target <= off[hi]
        if (a.off[lo] >= target) return lo;
        while (hi - lo > 1) {
            const int64_t step = (hi - lo + 31) / 32;
            const int64_t probe = min(hi, lo + (int64_t)(lane + 1) * step);
            const uint32_t ge = __ballot_sync(0xffffffffu, a.off[probe] >= target);
            const int f = __ffs(ge) - 1;                   // first probe at or past the target (>= 0: off[hi] >= target)
            hi = min(hi, lo + (int64_t)(f + 1) * step);
            lo = f > 0 ? lo + (int64_t)f * step : lo;
        }
        return hi;
    };
    const int64_t i0 = first_at(gw), i1 = first_at(gw + 1);
    int s = 0;
    while (s + 1 < a.pl && i0 >= a.shard_base[s + 1]) ++s;
    unsigned long long acc_w = 0, acc_d = 0, max_tw = 0;
    uint32_t exm[kNumCaps] = {};
    auto flush = [&]() {
        // M(tau) >= 1 for every k-mer present: the warp's presence bits, OR-ed once per word
        // (counts >= 2 update M itself); k_shard_plan folds the bits into M
        __syncwarp();
        for (int t = lane; t < VW; t += 32) {
            const uint32_t b = pres[t];
            if (b) {
                atomicOr(&a.Mb[(size_t)s * VW + t], b);
                pres[t] = 0;
            }
        }
        __syncwarp();
        if (lane == 0) {
            if (acc_w | acc_d) {
                atomicAdd(&a.kinfo[s * kKinfo + 0], acc_w);
                atomicAdd(&a.kinfo[s * kKinfo + 1], acc_d);
                atomicMax(&a.kinfo[s * kKinfo + 3], max_tw);
            }
#pragma unroll
            for (int j = 0; j < kNumCaps; ++j)
                if (exm[j]) atomicMax(&a.kinfo[s * kKinfo + 4 + j], (unsigned long long)exm[j]);
        }
        acc_w = acc_d = max_tw = 0;
#pragma unroll
        for (int j = 0; j < kNumCaps; ++j) exm[j] = 0;
    };
    const int SW = kCodeSeg - (k - 1);   // windows per segment
    // the next sequence's offsets and first 512 residue bytes are loaded during the current one
    int64_t off_c = i0 < i1 ? a.off[i0] : 0, off_e = i0 < i1 ? a.off[i0 + 1] : 0;
    uint4 qpre = i0 < i1 ? *reinterpret_cast<const uint4 *>(a.ascii + ((off_c & ~int64_t(15)) + 16 * lane))
                         : make_uint4(0, 0, 0, 0);
    int64_t s_end = a.shard_base[s + 1];                       // end of the current shard
    uint32_t *xcs = a.Xc + (size_t)s * kNumCaps * V;           // the shard's per-cap excess counts
    for (int64_t i = i0; i < i1; ++i) {
        if (i >= s_end) {                                      // shard change: flush the totals
            flush();
            while (s + 1 < a.pl && i >= a.shard_base[s + 1]) ++s;
            s_end = a.shard_base[s + 1];
            xcs = a.Xc + (size_t)s * kNumCaps * V;
        }
        const int64_t off0 = off_c;
        const int64_t L = off_e - off0;
        const uint4 qfirst = qpre;                             // residues [off0 & ~15, +512) of this lane
        if (i + 1 < i1) {
            off_c = off_e;
            off_e = a.off[i + 2];
            qpre = *reinterpret_cast<const uint4 *>(a.ascii + ((off_c & ~int64_t(15)) + 16 * lane));
        }
        const uint8_t *x = a.ascii + off0;
        const unsigned long long gidx = (unsigned long long)(a.first_idx + i);
        const int64_t Tw = L - k + 1;
        if (L < k || Tw > 65535) {                             // readings A19 / SURVEY A.3 precondition
            for (int64_t t = lane; t < L; t += 32)
                if (lut[x[t]] == 255) atomicMin(&a.err[0], (gidx << 32) | (unsigned long long)t);
            if (lane == 0) {
                atomicMin(&a.err[L < k ? 1 : 2], gidx);
                a.rowinfo[i] = RowInfo{1u, 0xFFFFFFFFu, 1u, (uint32_t)s};
                if (a.lcnt) atomicAdd(&a.lcnt[(size_t)s * kLenBinsMax + 1], 1u);
                a.T[i] = 0ull;
                a.dcnt[i] = 0;
                a.nhi[i] = 0;
            }
            continue;
        }
        const int nseg = (int)((Tw + SW - 1) / SW);
        int staged = -1, checked = -1;          // segment now in `cod`, last segment validated (K1)
        int sh = 0;                             // cod[sh + t - r0] = code of residue t of the staged segment
        // stage the codes of segment g: residues [g SW, min(L, (g + 1) SW + k - 1)), validated (K1) the
        // first time. Each lane translates one 16-byte aligned vector at a time and stores the 16 codes
        // with one 16-byte store at the vector's own alignment (bytes outside the segment are never read
        // as codes); a residue outside the alphabet (bit 7 of its LUT entry) takes the rare per-byte path.
        auto stage = [&](int g) {
            if (g == staged) return;
            const bool check = g > checked;
            const int64_t r0 = (int64_t)g * SW, r1 = min(L, r0 + SW + k - 1);
            const int64_t b0 = (off0 + r0) & ~int64_t(15), b1 = off0 + r1;
            sh = (int)(off0 + r0 - b0);
            const int nb = (int)(b1 - b0);      // staged bytes (<= kCodeSeg + 15)
            __syncwarp();
            for (int u = 16 * lane; u < nb; u += 512) {
                const uint4 q = (g == 0 && u < 512) ? qfirst : *reinterpret_cast<const uint4 *>(a.ascii + b0 + u);
                const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
                uint32_t cw[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t c0 = lut[qw[i] & 0xFFu], c1 = lut[(qw[i] >> 8) & 0xFFu];
                    const uint32_t c2 = lut[(qw[i] >> 16) & 0xFFu], c3 = lut[qw[i] >> 24];
                    cw[i] = c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
                }
                // bytes [lo, hi) of this vector belong to the segment; the masks are only needed when
                // some byte of the vector is outside the alphabet (bit 7 of its LUT entry)
                const int lo = max(0, sh - u), hi = min(16, nb - u);
                uint32_t bad = (cw[0] | cw[1] | cw[2] | cw[3]) & 0x80808080u;
                if (bad) {
                    bad = 0;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int l = min(max(lo - 4 * i, 0), 4), h = min(max(hi - 4 * i, 0), 4);
                        const uint32_t m = h > l ? ((0xFFFFFFFFu >> (32 - 8 * (h - l))) << (8 * l)) : 0u;
                        bad |= cw[i] & m & 0x80808080u;
                    }
                }
                if (bad) {                                   // rare: report the first bad residue, code it 0
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const uint32_t c = (cw[j >> 2] >> (8 * (j & 3))) & 0xFFu;
                        if (j >= lo && j < hi && c == 255u) {
                            if (check) atomicMin(&a.err[0], (gidx << 32) | (unsigned long long)(b0 + u + j - off0));
                            cw[j >> 2] &= ~(0xFFu << (8 * (j & 3)));
                        }
                    }
                }
                *reinterpret_cast<uint4 *>(cod + u) = make_uint4(cw[0], cw[1], cw[2], cw[3]);
            }
            __syncwarp();
            staged = g;
            checked = max(checked, g);
        };
        // pass 1: count every window (overlaps included). Normally narrow bins; a bin that reaches
        // its maximum (the next add could carry into its neighbour) sends the sequence to the
        // fallback: clear the bins and count with u16 bins over each part of the k-mers in turn. With `lst`,
        // the first window of every k-mer (its bin was 0) appends the k-mer to the owner list.
        int nl = 0;
        auto count = [&](int bits, uint32_t lo, uint32_t hi, uint16_t *lst) -> bool {
            bool ovf = false;
            for (int g = 0; g < nseg; ++g) {
                stage(g);
                const int w1 = (int)min((int64_t)SW, Tw - (int64_t)g * SW);
                for (int t0 = 0; t0 < w1; t0 += 32 * kCountUnroll) {   // independent windows per lane in flight
                    bool first[kCountUnroll];
                    uint32_t tau[kCountUnroll];
#pragma unroll
                    for (int u = 0; u < kCountUnroll; ++u) {
                        const int t = t0 + 32 * u + lane;
                        first[u] = false;
                        tau[u] = 0;
                        if (t < w1) {
                            tau[u] = window_tau<KT>(cod + sh + t, k, A);
                            if (tau[u] >= lo && tau[u] < hi) {
                                const uint32_t idx = tau[u] - lo;
                                const bool nb = bits != 16;
                                const uint32_t sh8 = nb ? kBinBits * (idx % kBinsPerWord) : 16u * (idx & 1u);
                                const uint32_t old = atomicAdd(&hist[nb ? idx / kBinsPerWord : idx >> 1], 1u << sh8);
                                const uint32_t ob = (old >> sh8) & (nb ? kBinMax : 0xFFFFu);
                                if (nb && ob == kBinMax) ovf = true;
                                first[u] = ob == 0;
                            }
                        }
                    }
                    if (lst) {
#pragma unroll
                        for (int u = 0; u < kCountUnroll; ++u) {
                            const uint32_t fm = __ballot_sync(0xffffffffu, first[u]);
                            if (first[u]) lst[nl + __popc(fm & ((1u << lane) - 1u))] = (uint16_t)tau[u];
                            nl += __popc(fm);
                        }
                    }
                }
            }
            __syncwarp();
            return __any_sync(0xffffffffu, ovf);
        };
        // pass 2: every k-mer once, emit (tau, count), update the shard's column maxima
        uint32_t *out = a.csr + (off0 - i * (int64_t)(k - 1));
        uint32_t *Ms = a.M + (size_t)s * V;
        uint32_t n_hi = 0, n_d = 0, ex[kNumCaps] = {};
        // every distinct entry goes to [0, d); the count >= 2 ones are repeated in the row's tail
        // [Tw - nhi, Tw), which is free: Tw - d = sum (count - 1) >= nhi
        const uint32_t lt = (1u << lane) - 1u;
        auto emit = [&](uint32_t c, uint32_t tau) {       // warp-uniform call; c = 0: nothing
            const uint32_t md = __ballot_sync(0xffffffffu, c != 0u), mh = __ballot_sync(0xffffffffu, c >= 2);
            if (c) out[n_d + __popc(md & lt)] = (tau << 16) | c;
            if (c >= 2) out[(uint32_t)Tw - 1u - n_hi - __popc(mh & lt)] = (tau << 16) | c;
            n_d += __popc(md);
            n_hi += __popc(mh);
            if (c) {
                atomicOr(&pres[tau >> 5], 1u << (tau & 31));
                if (c >= 2) {                          // excess beyond the layer caps 1, 2, 4, 8
                    atomicMax(&Ms[tau], c);
#pragma unroll
                    for (int j = 0; j < kNumCaps; ++j)
                        if (c > (1u << j)) {
                            ex[j] += c - (1u << j);
                            atomicAdd(&xcs[(uint32_t)j * (uint32_t)V + tau], 1u);
                        }
                }
            }
        };
        // claim by windows: every bin taken once by atomicAnd (the bins end cleared)
        auto claim = [&](int bits, uint32_t lo, uint32_t hi) {
            for (int gg = 0; gg < nseg; ++gg) {
                const int g = nseg - 1 - gg;                   // the last staged segment first
                stage(g);
                const int w1 = (int)min((int64_t)SW, Tw - (int64_t)g * SW);
                for (int t0 = 0; t0 < w1; t0 += 32) {
                    const int t = t0 + lane;
                    uint32_t c = 0, tau = 0;
                    if (t < w1) {
                        tau = window_tau<KT>(cod + sh + t, k, A);
                        if (tau >= lo && tau < hi) {
                            const uint32_t idx = tau - lo;
                            const bool nb = bits != 16;
                            const uint32_t sh8 = nb ? kBinBits * (idx % kBinsPerWord) : 16u * (idx & 1u);
                            const uint32_t mask = (nb ? kBinMax : 0xFFFFu) << sh8;
                            const uint32_t old = atomicAnd(&hist[nb ? idx / kBinsPerWord : idx >> 1], ~mask);
                            c = (old & mask) >> sh8;
                        }
                    }
                    emit(c, tau);
                }
            }
            __syncwarp();
        };
        // one-segment sequences keep the owner list in the staging buffer past the codes (a k-mer
        // list is at most Tw entries); the emission then walks d owners instead of Tw windows
        stage(0);
        const int lofs = (sh + (int)min(L, (int64_t)kCodeSeg) + 15) & ~15;
        uint16_t *lst = (nseg == 1 && (kCodeBuf - lofs) / 2 >= Tw + 1) ? reinterpret_cast<uint16_t *>(cod + lofs) : nullptr;
        bool narrow_ovf;
        bool fast = false;
        if constexpr (kBinBits == 8) fast = true;
        if (fast) {
            // Byte bins over all V k-mers and an owner list: in shared memory beside the staged codes
            // (one-segment sequences), else in the row's own CSR slots (a row has d <= Tw distinct
            // k-mers: the list becomes the entries in place). Counting: one shared-memory atomic per
            // window; a bin's first window (old count 0) appends its k-mer to the list. Emission:
            // every owner once (its count read and its bin cleared), entry slot = owner index; the
            // count >= 2 entries copied to the row's tail (free: Tw - d >= nhi).
            uint8_t *hb = reinterpret_cast<uint8_t *>(hist);
            const uint32_t lt = (1u << lane) - 1u;
            bool ovf = false;
            for (int g = 0; g < nseg; ++g) {
                stage(g);
                const int w1 = (int)min((int64_t)SW, Tw - (int64_t)g * SW);
                for (int t0 = 0; t0 < w1; t0 += 32 * kCountUnroll) {
                    bool first[kCountUnroll];
                    uint32_t tau[kCountUnroll];
#pragma unroll
                    for (int u = 0; u < kCountUnroll; ++u) {
                        const int t = t0 + 32 * u + lane;
                        first[u] = false;
                        tau[u] = 0;
                        if (t < w1) {
                            tau[u] = window_tau<KT>(cod + sh + t, k, A);
                            const uint32_t sh8 = (tau[u] & 3u) << 3;
                            const uint32_t ob = (atomicAdd(&hist[tau[u] >> 2], 1u << sh8) >> sh8) & 0xFFu;
                            ovf |= ob == 0xFFu;
                            first[u] = ob == 0u;
                        }
                    }
                    if (lst) {
#pragma unroll
                        for (int u = 0; u < kCountUnroll; ++u) {
                            const uint32_t fm = __ballot_sync(0xffffffffu, first[u]);
                            lst[first[u] ? nl + __popc(fm & lt) : (uint32_t)Tw] = (uint16_t)tau[u];   // slot Tw: a dummy
                            nl += __popc(fm);
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < kCountUnroll; ++u) {
                            const uint32_t fm = __ballot_sync(0xffffffffu, first[u]);
                            if (first[u]) out[nl + __popc(fm & lt)] = tau[u] << 16;
                            nl += __popc(fm);
                        }
                    }
                }
            }
            __syncwarp();
            narrow_ovf = __any_sync(0xffffffffu, ovf);
            if (!narrow_ovf) {
                for (int e0 = 0; e0 < nl; e0 += 32 * kCountUnroll) {
                    uint32_t c[kCountUnroll], tau[kCountUnroll];
#pragma unroll
                    for (int u = 0; u < kCountUnroll; ++u) {
                        const int e = e0 + 32 * u + lane;
                        c[u] = 0;
                        tau[u] = 0;
                        if (e < nl) {
                            tau[u] = lst ? (uint32_t)lst[e] : out[e] >> 16;
                            c[u] = hb[tau[u]];
                            hb[tau[u]] = 0;
                            out[e] = (tau[u] << 16) | c[u];        // list order: slot = owner index
                            atomicOr(&pres[tau[u] >> 5], 1u << (tau[u] & 31));
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kCountUnroll; ++u) {   // the count >= 2 entries: the row's tail
                        const uint32_t mh = __ballot_sync(0xffffffffu, c[u] >= 2u);
                        if (c[u] >= 2u) out[(uint32_t)Tw - 1u - n_hi - __popc(mh & lt)] = (tau[u] << 16) | c[u];
                        n_hi += __popc(mh);
                    }
                }
                __syncwarp();
                // their statistics, all lanes busy: shard maxima, per-cap excess counts and sums
                for (uint32_t e = lane; e < n_hi; e += 32) {
                    const uint32_t v = out[(uint32_t)Tw - 1u - e], c = v & 0xFFFFu, tau = v >> 16;
                    atomicMax(&Ms[tau], c);
#pragma unroll
                    for (int j = 0; j < kNumCaps; ++j)
                        if (c > (1u << j)) {
                            ex[j] += c - (1u << j);
                            atomicAdd(&xcs[(uint32_t)j * (uint32_t)V + tau], 1u);
                        }
                }
                n_d = (uint32_t)nl;
                __syncwarp();
            }
        } else {
            narrow_ovf = count(kBinBits, 0u, (uint32_t)V, lst);
            if (!narrow_ovf) {
                if (lst) {
                    for (int e0 = 0; e0 < nl; e0 += 32 * kCountUnroll) {
                        uint32_t c[kCountUnroll], tau[kCountUnroll];
#pragma unroll
                        for (int u = 0; u < kCountUnroll; ++u) {
                            const int e = e0 + 32 * u + lane;
                            c[u] = 0;
                            tau[u] = 0;
                            if (e < nl) {
                                tau[u] = lst[e];
                                c[u] = (hist[tau[u] / kBinsPerWord] >> (kBinBits * (tau[u] % kBinsPerWord))) & kBinMax;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kCountUnroll; ++u) emit(c[u], tau[u]);
                    }
                    __syncwarp();
                    for (int t = lane; t < hw / 4; t += 32) reinterpret_cast<uint4 *>(hist)[t] = make_uint4(0, 0, 0, 0);
                    __syncwarp();
                } else {
                    claim(kBinBits, 0u, (uint32_t)V);
                }
            }
        }
        if (narrow_ovf) {
            for (int t = lane; t < hw; t += 32) hist[t] = 0;
            __syncwarp();
            for (uint32_t h = 0; h < (uint32_t)kWidePasses; ++h) {
                const uint32_t lo = h * Vh, hi = min((uint32_t)V, lo + Vh);
                count(16, lo, hi, nullptr);
                claim(16, lo, hi);
            }
        }
        if (n_hi) {                                     // per-cap excess sums (each <= Tw <= 65535: two per word)
            uint32_t v0 = ex[0] | (ex[1] << 16), v1 = ex[2] | (ex[3] << 16);
            for (int o = 16; o; o >>= 1) {
                v0 += __shfl_xor_sync(0xffffffffu, v0, o);
                v1 += __shfl_xor_sync(0xffffffffu, v1, o);
            }
            exm[0] = max(exm[0], v0 & 0xFFFFu);
            exm[1] = max(exm[1], v0 >> 16);
            exm[2] = max(exm[2], v1 & 0xFFFFu);
            exm[3] = max(exm[3], v1 >> 16);
        }
        if (lane == 0) {
            a.nhi[i] = (int32_t)n_hi;
            a.dcnt[i] = (int32_t)n_d;
            const uint32_t tw = (uint32_t)Tw;
            a.rowinfo[i] = RowInfo{tw, 0xFFFFFFFFu / tw, 0xFFFFFFFFu % tw + 1u, (uint32_t)s};
            if (a.lcnt) atomicAdd(&a.lcnt[(size_t)s * kLenBinsMax + tw], 1u);    // the length order's histogram
            a.T[i] = 0ull;                              // the all-pairs kernel accumulates T_i atomically
        }
        acc_w += (unsigned long long)Tw;
        max_tw = max(max_tw, (unsigned long long)Tw);
        acc_d += n_d;
        __syncwarp();
    }
    // the final flush, merged per block: the warps that end in the same shard as warp 0 OR their
    // presence bits and add their totals in shared memory, then the block updates global memory once
    // (at G = 8 every warp ends in the one shard: ~10x fewer contended global atomics); the others
    // flush on their own
    if (lane == 0) fin_s[wid] = s;
    asm volatile("bar.sync 1, %0;" ::"r"(warps * 32) : "memory");
    const int s0 = fin_s[0];
    if (s == s0) {
        for (int t = lane; t < VW; t += 32) {
            const uint32_t b = pres[t];
            if (b) {
                atomicOr(&bpres[t], b);
                pres[t] = 0;
            }
        }
        if (lane == 0) {
            if (acc_w | acc_d) {
                atomicAdd(&bk_w, acc_w);
                atomicAdd(&bk_d, acc_d);
                atomicMax(&bk_tw, max_tw);
            }
#pragma unroll
            for (int j = 0; j < kNumCaps; ++j)
                if (exm[j]) atomicMax(&bk_ex[j], exm[j]);
        }
    } else {
        flush();
    }
    asm volatile("bar.sync 1, %0;" ::"r"(warps * 32) : "memory");
    for (int t = threadIdx.x; t < VW; t += warps * 32) {
        const uint32_t b = bpres[t];
        if (b) atomicOr(&a.Mb[(size_t)s0 * VW + t], b);
    }
    if (threadIdx.x == 0) {
        if (bk_w | bk_d) {
            atomicAdd(&a.kinfo[s0 * kKinfo + 0], bk_w);
            atomicAdd(&a.kinfo[s0 * kKinfo + 1], bk_d);
            atomicMax(&a.kinfo[s0 * kKinfo + 3], bk_tw);
        }
#pragma unroll
        for (int j = 0; j < kNumCaps; ++j)
            if (bk_ex[j]) atomicMax(&a.kinfo[s0 * kKinfo + 4 + j], (unsigned long long)bk_ex[j]);
    }
}

__global__ void k_profile_reset(uint32_t *M, size_t nM, uint32_t *Mb, size_t nMb, uint32_t *Xc, size_t nXc,
                                unsigned long long *err4, unsigned long long *statkinfo, size_t nsk, uint32_t *lcnt,
                                size_t nl) {
    const size_t stride = (size_t)gridDim.x * blockDim.x, t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (size_t t = t0; t < nl / 4; t += stride) reinterpret_cast<uint4 *>(lcnt)[t] = make_uint4(0, 0, 0, 0);
    for (size_t t = t0; t < nM; t += stride) M[t] = 0u;
    for (size_t t = t0; t < nMb; t += stride) Mb[t] = 0u;
    for (size_t t = t0; t < nXc; t += stride) Xc[t] = 0u;
    for (size_t t = t0; t < nsk; t += stride) statkinfo[t] = 0ull;
    if (t0 < 4) err4[t0] = ~0ull;
}

void launch_profile_reset(uint32_t *M, size_t nM, uint32_t *Mb, size_t nMb, uint32_t *Xc, size_t nXc,
                          unsigned long long *err4, unsigned long long *statkinfo, size_t nsk, uint32_t *lcnt,
                          size_t nl, cudaStream_t st) {
    const size_t big = std::max(std::max(std::max(nM, nXc), std::max(nMb, nsk)), nl / 4);
    const int64_t g = std::max<int64_t>(1, std::min<int64_t>(1024, (int64_t)((big + 255) / 256)));
    k_profile_reset<<<(unsigned)g, 256, 0, st>>>(M, nM, Mb, nMb, Xc, nXc, err4, statkinfo, nsk, lcnt, lcnt ? nl : 0);
}

// K1/K2 for long sequences (host-known average L >= 1024, e.g. config 5: ~1.7 kb, up to 8.5 kb):
// one BLOCK per sequence instead of one warp. With a warp per sequence the longest sequence's
// single-warp time is a floor under the kernel (config 5: 8.5 k windows ~ 170 us of the 227 us, 15 %
// of the stall samples at the end barrier); here the block's threads share one u16 histogram (no
// overflow: a count is at most Tw <= 65 535), the owner list is the row's own CSR slots (appended
// per warp: one ballot and one shared-memory atomic), and the emission, the count >= 2 tail and the
// statistics are strided over the block. Blocks take contiguous ranges of sequences balanced by
// residues; totals and presence bits are flushed per block at a shard change and at the end.
// Same outputs as k_profile (entries unordered within a row).
constexpr int kBlkThreads = 256;
constexpr int kBlkSeg = 8192;            // residue codes staged per block
template <int KT>
__global__ void __launch_bounds__(kBlkThreads, 4) k_profile_blk(ProfileArgs a) {
    extern __shared__ __align__(16) uint32_t bsm[];
    __shared__ uint8_t lut[256];
    __shared__ uint32_t nl_s, nhi_s, ex_s[kNumCaps];
    const int tid = threadIdx.x, lane = tid & 31;
    for (int t = tid; t < 256; t += kBlkThreads) lut[t] = 255;
    __syncthreads();
    if (tid < a.A) lut[(uint8_t)c_alpha[a.alphabet][tid]] = (uint8_t)tid;
    const int k = KT > 0 ? KT : a.k;
    const uint32_t A = (uint32_t)a.A;
    const int V = a.V, VW = (V + 31) / 32;
    const int hw = (V + 1) / 2;                               // u16 bins, two per word
    uint32_t *hist = bsm;
    uint16_t *h16 = reinterpret_cast<uint16_t *>(bsm);
    uint32_t *bpres = bsm + ((hw + 3) & ~3);
    uint8_t *cod = reinterpret_cast<uint8_t *>(bpres + ((VW + 3) & ~3));
    for (int t = tid; t < hw; t += kBlkThreads) hist[t] = 0;
    for (int t = tid; t < VW; t += kBlkThreads) bpres[t] = 0;
    __syncthreads();
    // contiguous ranges of sequences balanced by residues (every warp runs the same search)
    const int64_t W = gridDim.x, gw = blockIdx.x;
    const int64_t r0 = a.off[a.i_begin], rr = a.off[a.i_end] - r0;
    auto first_at = [&](int64_t wq) -> int64_t {
        if (wq <= 0) return a.i_begin;
        if (wq >= W) return a.i_end;
        const int64_t target = r0 + (int64_t)(((__int128)rr * wq) / W);
        int64_t lo = a.i_begin, hi = a.i_end;
        if (a.off[lo] >= target) return lo;
        while (hi - lo > 1) {
            const int64_t step = (hi - lo + 31) / 32;
            const int64_t probe = min(hi, lo + (int64_t)(lane + 1) * step);
            const uint32_t ge = __ballot_sync(0xffffffffu, a.off[probe] >= target);
            const int f = __ffs(ge) - 1;
            hi = min(hi, lo + (int64_t)(f + 1) * step);
            lo = f > 0 ? lo + (int64_t)f * step : lo;
        }
        return hi;
    };
    const int64_t i0 = first_at(gw), i1 = first_at(gw + 1);
    int s = 0;
    while (s + 1 < a.pl && i0 >= a.shard_base[s + 1]) ++s;
    unsigned long long acc_w = 0, acc_d = 0, max_tw = 0;     // thread 0's totals for shard s
    uint32_t exm[kNumCaps] = {};
    auto flush = [&]() {                                      // block-uniform call
        __syncthreads();
        for (int t = tid; t < VW; t += kBlkThreads) {
            const uint32_t b = bpres[t];
            if (b) {
                atomicOr(&a.Mb[(size_t)s * VW + t], b);
                bpres[t] = 0;
            }
        }
        if (tid == 0) {
            if (acc_w | acc_d) {
                atomicAdd(&a.kinfo[s * kKinfo + 0], acc_w);
                atomicAdd(&a.kinfo[s * kKinfo + 1], acc_d);
                atomicMax(&a.kinfo[s * kKinfo + 3], max_tw);
            }
#pragma unroll
            for (int j = 0; j < kNumCaps; ++j)
                if (exm[j]) atomicMax(&a.kinfo[s * kKinfo + 4 + j], (unsigned long long)exm[j]);
        }
        acc_w = acc_d = max_tw = 0;
#pragma unroll
        for (int j = 0; j < kNumCaps; ++j) exm[j] = 0;
        __syncthreads();
    };
    const int SW = kBlkSeg - (k - 1);                         // windows per segment
    const uint32_t lt = (1u << lane) - 1u;
    int64_t s_end = a.shard_base[s + 1];
    for (int64_t i = i0; i < i1; ++i) {
        if (i >= s_end) {
            flush();
            while (s + 1 < a.pl && i >= a.shard_base[s + 1]) ++s;
            s_end = a.shard_base[s + 1];
        }
        const int64_t off0 = a.off[i], L = a.off[i + 1] - off0;
        const uint8_t *x = a.ascii + off0;
        const unsigned long long gidx = (unsigned long long)(a.first_idx + i);
        const int64_t Tw = L - k + 1;
        if (L < k || Tw > 65535) {                             // readings A19 / SURVEY A.3 precondition
            for (int64_t t = tid; t < L; t += kBlkThreads)
                if (lut[x[t]] == 255) atomicMin(&a.err[0], (gidx << 32) | (unsigned long long)t);
            if (tid == 0) {
                atomicMin(&a.err[L < k ? 1 : 2], gidx);
                a.rowinfo[i] = RowInfo{1u, 0xFFFFFFFFu, 1u, (uint32_t)s};
                if (a.lcnt) atomicAdd(&a.lcnt[(size_t)s * kLenBinsMax + 1], 1u);
                a.T[i] = 0ull;
                a.dcnt[i] = 0;
                a.nhi[i] = 0;
            }
            continue;
        }
        uint32_t *out = a.csr + (off0 - i * (int64_t)(k - 1));
        uint32_t *Ms = a.M + (size_t)s * V;
        uint32_t *xcs = a.Xc + (size_t)s * kNumCaps * V;
        if (tid == 0) {
            nl_s = 0;
            nhi_s = 0;
        }
        if (tid < kNumCaps) ex_s[tid] = 0;
        const int nseg = (int)((Tw + SW - 1) / SW);
        // pass 1: count every window; a bin's first window appends its k-mer to the owner list
        for (int g = 0; g < nseg; ++g) {
            const int64_t q0 = (int64_t)g * SW, q1 = min(L, q0 + SW + k - 1);
            __syncthreads();                                   // the previous segment's windows are done
            for (int64_t t = q0 + tid; t < q1; t += kBlkThreads) {
                uint8_t c = lut[x[t]];
                if (c == 255) {                                // K1: first bad residue, coded 0
                    atomicMin(&a.err[0], (gidx << 32) | (unsigned long long)t);
                    c = 0;
                }
                cod[t - q0] = c;
            }
            __syncthreads();
            const int w1 = (int)min((int64_t)SW, Tw - q0);
            for (int t0 = 0; t0 < w1; t0 += kBlkThreads) {
                const int t = t0 + tid;
                bool first = false;
                uint32_t tau = 0;
                if (t < w1) {
                    tau = window_tau<KT>(cod + t, k, A);
                    const uint32_t sh16 = (tau & 1u) << 4;
                    first = ((atomicAdd(&hist[tau >> 1], 1u << sh16) >> sh16) & 0xFFFFu) == 0u;
                }
                const uint32_t fm = __ballot_sync(0xffffffffu, first);
                if (fm) {
                    uint32_t base = 0;
                    if (lane == __ffs(fm) - 1) base = atomicAdd(&nl_s, (uint32_t)__popc(fm));
                    base = __shfl_sync(0xffffffffu, base, __ffs(fm) - 1);
                    if (first) out[base + __popc(fm & lt)] = tau << 16;
                }
            }
        }
        __syncthreads();
        const uint32_t nl = nl_s;
        // pass 2: every owner once: its count read and its bin cleared, entry slot = owner index; the
        // count >= 2 entries repeated in the row's tail [Tw - nhi, Tw) (free: Tw - d >= nhi) with
        // their statistics (shard maxima, per-cap excess counts and sums)
        uint32_t ex[kNumCaps] = {};
        for (uint32_t e0 = 0; e0 < nl; e0 += kBlkThreads) {
            const uint32_t e = e0 + tid;
            uint32_t c = 0, tau = 0;
            if (e < nl) {
                tau = out[e] >> 16;
                c = h16[tau];
                h16[tau] = 0;
                out[e] = (tau << 16) | c;
                atomicOr(&bpres[tau >> 5], 1u << (tau & 31));
            }
            const uint32_t mh = __ballot_sync(0xffffffffu, c >= 2u);
            if (mh) {
                uint32_t base = 0;
                if (lane == __ffs(mh) - 1) base = atomicAdd(&nhi_s, (uint32_t)__popc(mh));
                base = __shfl_sync(0xffffffffu, base, __ffs(mh) - 1);
                if (c >= 2u) {
                    out[(uint32_t)Tw - 1u - base - __popc(mh & lt)] = (tau << 16) | c;
                    atomicMax(&Ms[tau], c);
#pragma unroll
                    for (int j = 0; j < kNumCaps; ++j)
                        if (c > (1u << j)) {
                            ex[j] += c - (1u << j);
                            atomicAdd(&xcs[(uint32_t)j * (uint32_t)V + tau], 1u);
                        }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kNumCaps; ++j) {
            uint32_t v = ex[j];
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && v) atomicAdd(&ex_s[j], v);
        }
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int j = 0; j < kNumCaps; ++j) exm[j] = max(exm[j], ex_s[j]);
            a.nhi[i] = (int32_t)nhi_s;
            a.dcnt[i] = (int32_t)nl;
            const uint32_t tw = (uint32_t)Tw;
            a.rowinfo[i] = RowInfo{tw, 0xFFFFFFFFu / tw, 0xFFFFFFFFu % tw + 1u, (uint32_t)s};
            if (a.lcnt) atomicAdd(&a.lcnt[(size_t)s * kLenBinsMax + tw], 1u);
            a.T[i] = 0ull;
            acc_w += (unsigned long long)Tw;
            max_tw = max(max_tw, (unsigned long long)Tw);
            acc_d += nl;
        }
        __syncthreads();                                       // nl_s / nhi_s / ex_s are reset next
    }
    flush();
}

template <int KT>
static void launch_profile_blk_t(const ProfileArgs &a, cudaStream_t st) {
    const int VW = (a.V + 31) / 32, hw = (a.V + 1) / 2;
    const size_t smem = 4 * (size_t)(((hw + 3) & ~3) + ((VW + 3) & ~3)) + kBlkSeg + 16;
    smem_optin(k_profile_blk<KT>, smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_profile_blk<KT>, kBlkThreads, smem);
    int64_t grid = std::min<int64_t>((int64_t)sms * std::max(per_sm, 1), a.i_end - a.i_begin);
    if (grid < 1) grid = 1;
    k_profile_blk<KT><<<(unsigned)grid, kBlkThreads, smem, st>>>(a);
}

void launch_profile(const ProfileArgs &a, cudaStream_t st) {
    if (a.blk) {
        if (a.k == 3) launch_profile_blk_t<3>(a, st);
        else if (a.k == 6) launch_profile_blk_t<6>(a, st);
        else launch_profile_blk_t<0>(a, st);
        return;
    }
    // V narrow bins, or u16 bins over 1/kWidePasses of the k-mers (the overflow fallback)
    const int narrow = (int)(((int64_t)a.V * kBinBits + 7) / 8);
    const int wide = 2 * ((a.V + kWidePasses - 1) / kWidePasses);
    const int hbytes = (std::max(narrow, wide) + 15) / 16 * 16;
    const size_t per_warp = (size_t)hbytes + kCodeBuf + 4 * (size_t)((((a.V + 31) / 32) + 3) & ~3);
    const size_t bbits = 4 * (size_t)((((a.V + 31) / 32) + 3) & ~3);
    const int warps = (int)std::max<size_t>(1, std::min<size_t>(kProfWarps, ((size_t)(220 * 1024 / SAD_PROF_MINB) - bbits) / per_warp));
    const size_t smem = per_warp * warps + 4 * (size_t)((((a.V + 31) / 32) + 3) & ~3);   // + the block's presence bits
    auto kern = a.k == 3 ? k_profile<3> : a.k == 6 ? k_profile<6> : k_profile<0>;
    smem_optin(kern, 200 * 1024);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kProfWarps * 32, smem);
    int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    grid = std::min<int64_t>(grid, (a.i_end - a.i_begin + warps - 1) / warps);
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kProfWarps * 32, smem, st>>>(a, warps, hbytes);
}

// Length order of every shard (the all-pairs kernel works on rows sorted by L - k + 1, so that
// in a tile strictly above the diagonal every pair's denominator min(L_i, L_j) - k + 1 is the
// row's own), by counting: per-shard histogram of Tw (K1/K2), one exclusive scan over [shard][Tw]
// (k_shard_plan; it gives global sorted positions directly: shards are contiguous), then every
// sequence takes the next slot of its bin -> sigma (sorted position -> local index), its inverse,
// and the sorted RowInfo with .shard replaced by the local index. Rows of equal Tw land in
// arbitrary order: nothing downstream depends on it (T and S are permutation invariant; K5 only
// needs Tw non-decreasing along every shard, K6 only a consistent order).
__global__ void k_lenscatter(const RowInfo *rowinfo, const int64_t *shard_base, int pl, int64_t n, uint32_t *pos,
                             int32_t *sigma, int32_t *sigma_inv, RowInfo *rinfo_s) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        RowInfo r = rowinfo[i];
        const int s = (int)r.shard;                // K1/K2 recorded every row's shard
        const int64_t p = atomicAdd(&pos[(size_t)s * kLenBinsMax + r.tw], 1u);   // sorted position
        const int64_t b = shard_base[s];
        const int32_t local = (int32_t)(i - b);
        sigma[p] = local;
        sigma_inv[i] = (int32_t)(p - b);
        r.shard = (uint32_t)local;
        rinfo_s[p] = r;
    }
}

void launch_lenorder(const RowInfo *rowinfo, const int64_t *shard_base, int pl, int64_t n, uint32_t *pos,
                     int32_t *sigma, int32_t *sigma_inv, RowInfo *rinfo_s, cudaStream_t st) {
    const int64_t g = std::min<int64_t>(4096, (n + 255) / 256);
    if (g <= 0) return;
    k_lenscatter<<<(unsigned)g, 256, 0, st>>>(rowinfo, shard_base, pl, n, pos, sigma, sigma_inv, rinfo_s);
}

// The deterministic length order (tile split: every rank must place the same sequences in the same
// row blocks): keys (shard << 32) | Tw with the row as value for a stable sort (ties by index), then
// sigma, sigma_inv and the sorted RowInfo from the sorted rows.
__global__ void k_lenkeys(const RowInfo *rowinfo, int64_t n, unsigned long long *keys, int32_t *rows) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const RowInfo r = rowinfo[i];
        keys[i] = ((unsigned long long)r.shard << 32) | r.tw;
        rows[i] = (int32_t)i;
    }
}

__global__ void k_lenapply(const int32_t *rows_sorted, const RowInfo *rowinfo, const int64_t *shard_base, int64_t n,
                           int32_t *sigma, int32_t *sigma_inv, RowInfo *rinfo_s) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = rows_sorted[p];
        RowInfo r = rowinfo[i];
        const int64_t b = shard_base[r.shard];
        sigma[p] = (int32_t)(i - b);
        sigma_inv[i] = (int32_t)(p - b);
        r.shard = (uint32_t)(i - b);
        rinfo_s[p] = r;
    }
}

void launch_lenkeys(const RowInfo *rowinfo, int64_t n, unsigned long long *keys, int32_t *rows, cudaStream_t st) {
    const int64_t g = std::min<int64_t>(4096, (n + 255) / 256);
    if (g > 0) k_lenkeys<<<(unsigned)g, 256, 0, st>>>(rowinfo, n, keys, rows);
}

void launch_lenapply(const int32_t *rows_sorted, const RowInfo *rowinfo, const int64_t *shard_base, int64_t n,
                     int32_t *sigma, int32_t *sigma_inv, RowInfo *rinfo_s, cudaStream_t st) {
    const int64_t g = std::min<int64_t>(4096, (n + 255) / 256);
    if (g > 0) k_lenapply<<<(unsigned)g, 256, 0, st>>>(rows_sorted, rowinfo, shard_base, n, sigma, sigma_inv, rinfo_s);
}

// K3, one block per shard, everything between the k-mer counts and the operand in one launch
// (no host round trip):
//  (1) statistics for every candidate cap T = 2^j (and no cap), after folding the presence bits
//      into M (a k-mer present at most once per sequence has M = 1):
//        K_s(T) = sum_tau min(M(tau), T)                        -> kinfo[s][2] (no cap), [8 + j]
//        sum_tau C(X_T(tau), 2), X_T(tau) = #{i : n_i(tau) > T}  -> kinfo[s][12 + j] (bound of K6 pairs)
//        sum_tau X_T(tau)                                       -> kinfo[s][16 + j] (K6 list entries)
//  (2) the decision: the smallest layer cap T_s = 2^j whose per-row excess
//      max_i sum_tau (n_i(tau) - T)+ (kinfo[s][4 + j], from K1/K2) fits the K6 byte (<= 255), when
//      capping is allowed, else none; the operand width K_s = K_s(T_s) and its K blocks (kcpb
//      columns each, clipped to the operand's capacity kcap_blocks: status[0] |= 1 flags an
//      overflow, status[1] = max_s K_s); kinfo[s][20] = K_s, [21] = T_s;
//  (3) the column map col0(tau) = exclusive scan over tau of min(M(tau), T_s): column block
//      [col0(tau), col0(tau) + min(M(tau), T_s)) holds the threshold layers t = 1..min(M, T_s) of
//      tau (min(a,b) = min(min(a,T),min(b,T)) + min((a-T)+,(b-T)+)); the second term
//      is the sparse excess of K6 (k_excess.cu), whose list offsets are (4) the exclusive scan of
//      X_{T_s}(tau) (shards without entries above their cap get empty lists).
// One cluster of kPlanCtas CTAs per shard (distributed shared memory): CTA c owns the k-mers
// [c V / C, (c + 1) V / C); partial statistics and chunk totals meet in the leader CTA's shared
// memory, so the whole plan is one launch with every k-mer touched by its own thread.
constexpr int kScanThreads = 512, kPlanCtas = 8;
__global__ void __cluster_dims__(kPlanCtas, 1, 1) __launch_bounds__(kScanThreads)
    k_shard_plan(uint32_t *M, const uint32_t *Mb, const uint32_t *Xc, unsigned long long *kinfo, int V, int allow_cap,
                 int64_t kcap_blocks, int kcpb, uint32_t *cap, uint32_t *xsel, uint32_t *ident, int64_t *kblocks,
                 unsigned long long *status, uint32_t *col0, uint32_t *xoff, unsigned long long *xtot,
                 uint32_t *xcur, const uint32_t *lcnt, uint32_t *lpos, const int64_t *shard_base) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    typedef cub::BlockScan<unsigned long long, kScanThreads> Scan;
    constexpr int NV = 3 * kNumCaps + 1;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned long long red[NV];          // this CTA's partial statistics
    __shared__ unsigned long long ctot;             // this CTA's packed chunk total
    __shared__ uint32_t s_T, s_sel;                 // the decision (leader CTA)
    const unsigned c = cluster.block_rank();
    const int s = blockIdx.x / kPlanCtas;
    const int t0 = (int)(((int64_t)V * c) / kPlanCtas), t1 = (int)(((int64_t)V * (c + 1)) / kPlanCtas);
    uint32_t *m = M + (size_t)s * V;
    const uint32_t *xc = Xc + (size_t)s * kNumCaps * V;
    const uint32_t *mb = Mb + (size_t)s * ((V + 31) / 32);
    unsigned long long *ki = kinfo + (size_t)s * kKinfo;
    if (threadIdx.x < NV) red[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long acc[NV] = {};
    for (int t = t0 + (int)threadIdx.x; t < t1; t += kScanThreads) {   // (1), coalesced
        uint32_t x = m[t];
        if (x == 0 && ((mb[t >> 5] >> (t & 31)) & 1u)) {
            x = 1;
            m[t] = 1;
        }
        acc[kNumCaps] += x;
#pragma unroll
        for (int j = 0; j < kNumCaps; ++j) {
            acc[j] += min(x, 1u << j);
            const unsigned long long cc = xc[(size_t)j * V + t];
            acc[kNumCaps + 1 + j] += cc * (cc - (cc ? 1 : 0)) / 2;
            acc[2 * kNumCaps + 1 + j] += cc;
        }
        xcur[(size_t)s * V + t] = 0u;                                 // K6 list cursors
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        unsigned long long v = acc[j];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&red[j], v);
    }
    cluster.sync();                                   // every CTA's partials (and M folds) are in place
    // (2) in every CTA (the same decision everywhere; no broadcast): thread j < NV sums partial j
    // over the cluster, thread 0 decides; only the leader writes the results
    __shared__ unsigned long long tot[NV];
    if (threadIdx.x < NV) {
        unsigned long long v = 0;
#pragma unroll
        for (unsigned r = 0; r < kPlanCtas; ++r) v += cluster.map_shared_rank(red, r)[threadIdx.x];
        tot[threadIdx.x] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long Knc = tot[kNumCaps];
        unsigned long long K = Knc;
        uint32_t T = kNoCap, sel = (uint32_t)kNumCaps;
        if (allow_cap)
            for (int j = 0; j < kNumCaps; ++j)
                if (ki[4 + j] <= 255ull) {
                    T = 1u << j;
                    K = tot[j];
                    if (ki[4 + j] > 0) sel = (uint32_t)j;    // the shard has entries above its cap
                    break;
                }
        s_T = T;
        s_sel = sel;
        if (c == 0) {
            ki[2] = Knc;
            for (int j = 0; j < kNumCaps; ++j) {
                ki[8 + j] = tot[j];
                ki[12 + j] = tot[kNumCaps + 1 + j];
                ki[16 + j] = tot[2 * kNumCaps + 1 + j];
            }
            cap[s] = T;
            xsel[s] = sel;
            ident[s] = (T == 1u && K == (unsigned long long)V) ? 1u : 0u;   // col0(tau) = tau
            int64_t kb = (int64_t)((K + (unsigned long long)kcpb - 1) / (unsigned long long)kcpb);
            if (kb < 1) kb = 1;
            if (kb > kcap_blocks) {                                          // operand too narrow: flagged
                atomicOr(&status[0], 1ull);
                kb = kcap_blocks;
            }
            kblocks[s] = kb;
            ki[20] = K;
            ki[21] = T;
            atomicMax(&status[1], K);
        }
    }
    __syncthreads();
    const uint32_t T = s_T, sel = s_sel;
    // (3) and (4) in one scan: every thread owns a contiguous chunk of its CTA's k-mers and scans
    // the pair (min(M, T_s), X_{T_s}) packed in one u64 (col0 high, list offsets low: a shard's list
    // entries are < 2^32, the u32 offsets' own bound); CTA totals are carried across the cluster
    const int C = (t1 - t0 + kScanThreads - 1) / kScanThreads;
    const int a0 = min(t1, t0 + (int)threadIdx.x * C), a1 = min(t1, a0 + C);
    const uint32_t *x = sel < (uint32_t)kNumCaps ? xc + (size_t)sel * V : nullptr;
    unsigned long long loc = 0;
    for (int t = a0; t < a1; ++t) loc += ((unsigned long long)min(m[t], T) << 32) + (x ? x[t] : 0u);
    unsigned long long ex, agg;
    Scan(tmp).ExclusiveSum(loc, ex, agg);
    if (threadIdx.x == 0) ctot = agg;
    cluster.sync();
    unsigned long long carry = 0, all = 0;
    for (unsigned r = 0; r < kPlanCtas; ++r) {
        const unsigned long long v = *cluster.map_shared_rank(&ctot, r);
        if (r < c) carry += v;
        all += v;
    }
    uint32_t *cp = col0 + (size_t)s * V;
    uint32_t *xo = xoff + (size_t)s * V;
    uint32_t ch = (uint32_t)((carry + ex) >> 32), cl = (uint32_t)(carry + ex);
    for (int t = a0; t < a1; ++t) {
        cp[t] = ch;
        xo[t] = cl;
        ch += min(m[t], T);
        cl += x ? x[t] : 0u;
    }
    if (c == 0 && threadIdx.x == 0) xtot[s] = x ? (unsigned long long)(uint32_t)all : 0ull;
    if (lcnt && c == kPlanCtas - 1) {
        // the length order's bin offsets: exclusive scan of the shard's Tw histogram over bins
        // 0..max Tw (kinfo[3], from K1/K2), offset by the shard's first row; kLenItems bins per
        // thread per block scan (one scan for max Tw < 2048)
        __syncthreads();                              // tmp of the scan above is reused
        const unsigned long long mt = ki[3];
        const int nb = (int)(mt + 1 < (unsigned long long)kLenBinsMax ? mt + 1 : (unsigned long long)kLenBinsMax);
        const uint32_t *lc = lcnt + (size_t)s * kLenBinsMax;
        uint32_t *lp = lpos + (size_t)s * kLenBinsMax;
        unsigned long long lcarry = (unsigned long long)shard_base[s];
        constexpr int kLenItems = 4;
        for (int b0 = 0; b0 < nb; b0 += kScanThreads * kLenItems) {
            unsigned long long v[kLenItems], e2[kLenItems], a2;
#pragma unroll
            for (int u = 0; u < kLenItems; ++u) {
                const int b = b0 + (int)threadIdx.x * kLenItems + u;
                v[u] = b < nb ? lc[b] : 0u;
            }
            Scan(tmp).ExclusiveSum(v, e2, a2);
#pragma unroll
            for (int u = 0; u < kLenItems; ++u) {
                const int b = b0 + (int)threadIdx.x * kLenItems + u;
                if (b < nb) lp[b] = (uint32_t)(lcarry + e2[u]);
            }
            lcarry += a2;
            __syncthreads();
        }
    }
    cluster.sync();                                   // no CTA leaves while its shared memory is read
}

void launch_shard_plan(uint32_t *M, const uint32_t *Mb, const uint32_t *Xc, unsigned long long *kinfo, int pl, int V,
                       int allow_cap, int64_t kcap_blocks, int kcpb, uint32_t *cap, uint32_t *xsel, uint32_t *ident,
                       int64_t *kblocks, unsigned long long *status, uint32_t *col0, uint32_t *xoff,
                       unsigned long long *xtot, uint32_t *xcur, const uint32_t *lcnt, uint32_t *lpos,
                       const int64_t *shard_base, cudaStream_t st) {
    k_shard_plan<<<pl * kPlanCtas, kScanThreads, 0, st>>>(M, Mb, Xc, kinfo, V, allow_cap, kcap_blocks, kcpb, cap,
                                                          xsel, ident, kblocks, status, col0, xoff, xtot, xcur,
                                                          lcnt, lpos, shard_base);
}

__device__ __forceinline__ int shard_of_padded_row(const int64_t *rowpad, int pl, int64_t r) {
    int s = 0;
    while (s + 1 < pl && r >= rowpad[s + 1]) ++s;
    return s;
}

// K4: the binary threshold-indicator operand of the tensor-core path,
//   A_s[i, col0(tau) + t - 1] = 1  for 1 <= t <= min(n_i(tau), T_s)   (uint8, or packed e2m1 nibbles),
// so that (A_s A_s^T)_ij = sum_tau min(min(n_i, T_s), min(n_j, T_s)); with T_s unlimited this is
// S_ij itself (the remainder above the cap is K6, k_excess.cu). Operand row r of shard s is the
// sequence sigma_s(r) (length order). Persistent warps, one padded row at a time: the row (or a slice of at most kRowSlice bytes) is assembled in the warp's own
// shared-memory slice and written with 16-byte coalesced stores (rows are 128-byte aligned), so
// HBM sees exactly one streaming write of the operand. The entry and column-map loads are
// issued kOpBatch per lane at a time, and the next row's CSR position is fetched one row ahead.
constexpr int kOpThreads = 256;
#ifndef SAD_OP_WARPS
#define SAD_OP_WARPS 8
#endif
#ifndef SAD_OP_BATCH
#define SAD_OP_BATCH 4
#endif
constexpr int kOpWarps = SAD_OP_WARPS;
constexpr int kRowSlice = 16384;
constexpr int kOpBatch = SAD_OP_BATCH;
__global__ void __launch_bounds__(kOpWarps * 32) k_indicator(OperandArgs a, int slice, int rpg) {
    extern __shared__ __align__(16) uint8_t opsm[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t *row = opsm + (size_t)wid * slice;
    uint32_t *row32 = reinterpret_cast<uint32_t *>(row);
    const uint32_t stride = (uint32_t)a.stride;
    const uint32_t per_byte = a.fp4 ? 2u : 1u;               // operand columns per byte
    // Sequences in input order, rpg (<= 32, sized so that every resident warp has a group) per
    // warp-group: their CSR positions, shards and operand rows (sigma^-1: length-order slots) come
    // from one coalesced load each, so no load chain precedes a row's entries; each row lands at its
    // slot. Padding rows are never written: the all-pairs epilogue masks every product with one.
    const int64_t ngroups = (a.n + rpg - 1) / rpg;
    for (int64_t g = (int64_t)blockIdx.x * kOpWarps + wid; g < ngroups; g += (int64_t)gridDim.x * kOpWarps) {
        const int64_t il = g * rpg + lane;
        int64_t eo_l = 0, slot_l = 0;
        int d_l = 0, s_l = 0;
        if (lane < rpg && il < a.n) {
            s_l = (int)a.rowinfo[il].shard;
            eo_l = a.off[il] - il * (int64_t)(a.k - 1);
            d_l = a.dcnt[il];
            slot_l = a.shard_rowpad[s_l] + (a.sigma_inv ? a.sigma_inv[il] : il - a.shard_base[s_l]);
        }
        const int nrows = (int)min((int64_t)rpg, a.n - g * rpg);
        uint32_t vpre[kOpBatch];             // the row's first entry batch, loaded during the previous row
#pragma unroll
        for (int b = 0; b < kOpBatch; ++b) {
            const int e = b * 32 + lane;
            const int d0 = __shfl_sync(0xffffffffu, d_l, 0);
            const int64_t eo0 = __shfl_sync(0xffffffffu, eo_l, 0);
            vpre[b] = e < d0 ? a.csr[eo0 + e] : 0u;
        }
        for (int j = 0; j < nrows; ++j) {
            const int s = __shfl_sync(0xffffffffu, s_l, j);
            const int dcur = __shfl_sync(0xffffffffu, d_l, j);
            const int64_t eo = __shfl_sync(0xffffffffu, eo_l, j);
            const int64_t slot = __shfl_sync(0xffffffffu, slot_l, j);
            const int dn = __shfl_sync(0xffffffffu, d_l, (j + 1) & 31);
            const int64_t eon = __shfl_sync(0xffffffffu, eo_l, (j + 1) & 31);
            const uint32_t *ent = a.csr + eo;
            const uint32_t *c0 = a.col0 + (size_t)s * a.V;
            const uint32_t T = a.cap ? a.cap[s] : 0xFFFFFFFFu;
            const bool ident = a.ident && a.ident[s];   // column of tau is tau itself (cap 1, every k-mer present)
            uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint8_t *>(a.op) + slot * a.stride);
            // bytes of this row the contraction reads: the shard's K blocks (the stride is a capacity)
            const uint32_t rowb = a.kblocks ? min(stride, (uint32_t)a.kblocks[s] * 128u) : stride;
            bool have_pre = true;
            for (uint32_t ch = 0; ch < rowb; ch += (uint32_t)slice) {
                const uint32_t len = min((uint32_t)slice, rowb - ch);
                for (uint32_t t = lane; t < len / 16; t += 32) reinterpret_cast<uint4 *>(row)[t] = make_uint4(0, 0, 0, 0);
                __syncwarp();
                const uint32_t c_lo = ch * per_byte, c_hi = (ch + len) * per_byte;
                for (int e0 = 0; e0 < dcur; e0 += 32 * kOpBatch) {
                    uint32_t v[kOpBatch], cb[kOpBatch];
                    if (e0 == 0 && have_pre) {
#pragma unroll
                        for (int b = 0; b < kOpBatch; ++b) v[b] = vpre[b];
                    } else {
#pragma unroll
                        for (int b = 0; b < kOpBatch; ++b) {
                            const int e = e0 + b * 32 + lane;
                            v[b] = e < dcur ? ent[e] : 0u;
                        }
                    }
#pragma unroll
                    for (int b = 0; b < kOpBatch; ++b)
                        cb[b] = ident ? (v[b] >> 16) : ((v[b] & 0xFFFFu) ? c0[v[b] >> 16] : 0u);
#pragma unroll
                    for (int b = 0; b < kOpBatch; ++b) {
                        const uint32_t n = v[b] & 0xFFFFu;     // 0 for lanes past the row's entries
                        const uint32_t lo = max(cb[b], c_lo), hi = min(cb[b] + min(n, T), c_hi);
                        if (a.fp4) {      // e2m1 1.0 = 0b0010; the run of min(n, T) nibbles one word at a time
                            for (uint32_t c = lo; c < hi;) {      // (neighbouring k-mers may share a word)
                                const uint32_t cc = c - c_lo, o = cc & 7u, m = min(hi - c, 8u - o);
                                atomicOr(&row32[cc >> 3], (0x22222222u >> (4u * (8u - m))) << (4u * o));
                                c += m;
                            }
                        } else {
                            for (uint32_t c = lo; c < hi; ++c) row[c - c_lo] = 1;
                        }
                    }
                }
                if (ch + (uint32_t)slice >= rowb && j + 1 < nrows) {   // the next row's first batch
#pragma unroll
                    for (int b = 0; b < kOpBatch; ++b) {
                        const int e = b * 32 + lane;
                        vpre[b] = e < dn ? a.csr[eon + e] : 0u;
                    }
                }
                have_pre = false;
                __syncwarp();
                for (uint32_t t = lane; t < len / 16; t += 32) dst[ch / 16 + t] = reinterpret_cast<const uint4 *>(row)[t];
                __syncwarp();
            }
        }
    }
}

// K4 for long rows (average Tw >= kWideTw, e.g. config 5's ~1.3k entries and 13 KB per row): one
// block per row instead of one warp, so a row's entries are one or two loads per thread and the
// block holds a single row slice in shared memory (up to 8 blocks per SM instead of 8 warps): the
// warp-per-row kernel left config 5 latency-bound at 10 % occupancy (0.20 ms for 130 MB). The next
// row's metadata and first entries are fetched during the current row.
constexpr int kWideTw = 1024;
__global__ void __launch_bounds__(kOpThreads) k_indicator_blk(OperandArgs a, int slice) {
    extern __shared__ __align__(16) uint8_t opsm[];
    uint32_t *row32 = reinterpret_cast<uint32_t *>(opsm);
    uint4 *row4 = reinterpret_cast<uint4 *>(opsm);
    const int tid = threadIdx.x;
    const uint32_t stride = (uint32_t)a.stride;
    const uint32_t per_byte = a.fp4 ? 2u : 1u;
    int s_n = 0, d_n = 0;
    int64_t eo_n = 0, slot_n = 0;
    auto meta = [&](int64_t il) {
        s_n = (int)a.rowinfo[il].shard;
        eo_n = a.off[il] - il * (int64_t)(a.k - 1);
        d_n = a.dcnt[il];
        slot_n = a.shard_rowpad[s_n] + (a.sigma_inv ? a.sigma_inv[il] : il - a.shard_base[s_n]);
    };
    int64_t il = blockIdx.x;
    uint32_t vpre[kOpBatch];
#pragma unroll
    for (int b = 0; b < kOpBatch; ++b) vpre[b] = 0u;
    if (il < a.n) {
        meta(il);
#pragma unroll
        for (int b = 0; b < kOpBatch; ++b) {
            const int e = b * kOpThreads + tid;
            vpre[b] = e < d_n ? a.csr[eo_n + e] : 0u;
        }
    }
    for (; il < a.n; il += gridDim.x) {
        const int s = s_n, dcur = d_n;
        const int64_t eo = eo_n, slot = slot_n;
        const int64_t iln = il + gridDim.x;
        if (iln < a.n) meta(iln);                    // consumed after this row's last slice
        const uint32_t *ent = a.csr + eo;
        const uint32_t *c0 = a.col0 + (size_t)s * a.V;
        const uint32_t T = a.cap ? a.cap[s] : 0xFFFFFFFFu;
        const bool ident = a.ident && a.ident[s];
        uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint8_t *>(a.op) + slot * a.stride);
        const uint32_t rowb = a.kblocks ? min(stride, (uint32_t)a.kblocks[s] * 128u) : stride;
        bool have_pre = true;
        for (uint32_t ch = 0; ch < rowb; ch += (uint32_t)slice) {
            const uint32_t len = min((uint32_t)slice, rowb - ch);
            // every thread zeroes the vectors it stored for the previous slice (or row): no barrier
            // is needed between that store and this zeroing
            for (uint32_t t = tid; t < len / 16; t += kOpThreads) row4[t] = make_uint4(0, 0, 0, 0);
            __syncthreads();
            const uint32_t c_lo = ch * per_byte, c_hi = (ch + len) * per_byte;
            for (int e0 = 0; e0 < dcur; e0 += kOpThreads * kOpBatch) {
                uint32_t v[kOpBatch], cb[kOpBatch];
                if (e0 == 0 && have_pre) {
#pragma unroll
                    for (int b = 0; b < kOpBatch; ++b) v[b] = vpre[b];
                } else {
#pragma unroll
                    for (int b = 0; b < kOpBatch; ++b) {
                        const int e = e0 + b * kOpThreads + tid;
                        v[b] = e < dcur ? ent[e] : 0u;
                    }
                }
#pragma unroll
                for (int b = 0; b < kOpBatch; ++b)
                    cb[b] = ident ? (v[b] >> 16) : ((v[b] & 0xFFFFu) ? c0[v[b] >> 16] : 0u);
#pragma unroll
                for (int b = 0; b < kOpBatch; ++b) {
                    const uint32_t n = v[b] & 0xFFFFu;     // 0 for threads past the row's entries
                    const uint32_t lo = max(cb[b], c_lo), hi = min(cb[b] + min(n, T), c_hi);
                    if (a.fp4) {          // the run of min(n, T) nibbles one word at a time
                        for (uint32_t c = lo; c < hi;) {
                            const uint32_t cc = c - c_lo, o = cc & 7u, m = min(hi - c, 8u - o);
                            atomicOr(&row32[cc >> 3], (0x22222222u >> (4u * (8u - m))) << (4u * o));
                            c += m;
                        }
                    } else {
                        for (uint32_t c = lo; c < hi; ++c) opsm[c - c_lo] = 1;
                    }
                }
            }
            if (ch + (uint32_t)slice >= rowb && iln < a.n) {           // the next row's first batch
#pragma unroll
                for (int b = 0; b < kOpBatch; ++b) {
                    const int e = b * kOpThreads + tid;
                    vpre[b] = e < d_n ? a.csr[eo_n + e] : 0u;
                }
            }
            have_pre = false;
            __syncthreads();
            for (uint32_t t = tid; t < len / 16; t += kOpThreads) dst[ch / 16 + t] = row4[t];
        }
    }
}

void launch_indicator(const OperandArgs &a, cudaStream_t st) {
    const int slice = (int)std::min<int64_t>(a.stride, kRowSlice);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (a.wide) {
        const size_t smem = (size_t)slice;
        smem_optin(k_indicator_blk, (size_t)kRowSlice);
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_indicator_blk, kOpThreads, smem);
        const int64_t grid = std::min<int64_t>((int64_t)sms * std::max(per_sm, 1), a.n);
        if (grid > 0) k_indicator_blk<<<(unsigned)grid, kOpThreads, smem, st>>>(a, slice);
        return;
    }
    const size_t smem = (size_t)kOpWarps * slice;
    smem_optin(k_indicator, smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_indicator, kOpWarps * 32, smem);
#ifndef SAD_K4_DIV
#define SAD_K4_DIV 1
#endif
    int64_t grid = (int64_t)sms * std::max(per_sm / SAD_K4_DIV, 1);
    // rows per warp-group: enough groups for every resident warp, at most 32 (one per lane)
    const int64_t warps = grid * kOpWarps;
    const int rpg = (int)std::max<int64_t>(1, std::min<int64_t>(32, (a.n + warps - 1) / warps));
    const int64_t need = ((a.n + rpg - 1) / rpg + kOpWarps - 1) / kOpWarps;
    if (grid > need) grid = need;
    if (grid > 0) k_indicator<<<(unsigned)grid, kOpWarps * 32, smem, st>>>(a, slice, rpg);
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
    smem_optin(k_dense_counts, smem);
    if (a.rows_pad > 0) k_dense_counts<<<(unsigned)a.rows_pad, kOpThreads, smem, st>>>(a);
}

}  // namespace sad
