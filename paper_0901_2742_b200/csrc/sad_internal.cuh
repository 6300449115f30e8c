// sad_internal.cuh — private declarations of libsad.so (not part of the ABI).
//
// Data layout in HBM (per rank; n = local sequences, R = local residues, pl = p/world
// local shards, V = A^k):
//   ascii   u8  [R]          residues as loaded (the redistribution payload)
//   off     i64 [n+1]        residue offsets
//   rowinfo u32x4 [n]        {Tw = L-k+1, Qd = floor((2^32-1)/Tw), Rp = (2^32-1) mod Tw + 1, shard}
//   csr     u32 [sum Tw]     per sequence i, Tw slots at off[i] - i*(k-1): its d distinct k-mers
//                            (tau << 16) | count in slots [0, d) (any order), the nhi of them with
//                            count >= 2 repeated in the last nhi slots (d + nhi <= Tw)
//   dcnt    i32 [n]          distinct k-mers per sequence (d)
//   nhi     i32 [n]          of which count >= 2
//   M/col0  u32 [pl][V]      per shard max count of tau / first operand column of tau
//   T       u64 [n]          within-shard fixed-point rank sums (reading A5)
//   key     u64 [n]          (floor(2^32 S/den) << 31) + source_index
// The all-pairs operand (caller buffer) is either the binary threshold-indicator matrix
// u8 [rows_pad][K_stride] (tensor-core path) or dense counts u16 [rows_pad][V_pad] (ALU path).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sad.h"

namespace sad {

constexpr int kMaxLocalShards = 256;
constexpr int kRowPad = 128;        // operand rows per shard padded to this (tensor-core M tile)
constexpr int kColPad = 128;        // operand columns padded to this (one 128-byte K block)
constexpr int kKinfo = 24;          // u64 per shard in kinfo: [0] windows, [1] distinct, [2] K (no cap), [3] max Tw,
                                    // [4 + j] max_i sum_tau (n_i - 2^j)+, [8 + j] K under cap 2^j,
                                    // [12 + j] sum_tau C(X_j(tau), 2), [16 + j] sum_tau X_j(tau) with
                                    // X_j(tau) = #{i : n_i(tau) > 2^j}   (j < kNumCaps);
                                    // [20] operand columns K_s and [21] layer cap T_s chosen by k_shard_plan
constexpr int kLenBinsMax = 65536; // Tw <= 65535 (checked by K1/K2)
constexpr int kNumCaps = 4;         // candidate layer caps T = 1, 2, 4, 8
constexpr int kXrSmem = 200 * 1024; // K6 row accumulators (u8 per shard column) per block
constexpr int64_t kMaxExcessBytes = int64_t(32) << 30;   // K6 dense excess matrices above this: no layer cap
constexpr uint32_t kNoCap = 0xFFFFFFFFu;

struct RowInfo {                    // per local sequence, 16 bytes
    uint32_t tw;                    // L - k + 1 (the den candidate of this row)
    uint32_t qd;                    // floor((2^32 - 1) / tw)
    uint32_t rp;                    // (2^32 - 1) mod tw + 1
    uint32_t shard;                 // local shard index
};

// ------------------------------------------------------------------------------------
// Exact fixed point q = floor(2^32 * S / d) for 0 <= S <= d <= 65535, d = min(tw_i, tw_j)
// (reading A5). With 2^32 - 1 = Qd*d + (Rp-1):
//   2^32 S = S*Qd*d + S*Rp  =>  q = S*Qd + floor(x/d),  x = S*Rp < 2^32.
//   t0 = umulhi(x, Qd) = floor(x*Qd/2^32) and x*Qd/2^32 = x/d - x*Rp/(d*2^32) in (x/d - 1, x/d],
//   so t0 is floor(x/d) or floor(x/d) - 1 and one remainder test fixes it.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t fixed_q(uint32_t S, uint32_t d, uint32_t qd, uint32_t rp) {
    uint32_t x = S * rp;
    uint32_t t = __umulhi(x, qd);
    uint32_t r = x - t * d;
    t += (r >= d) ? 1u : 0u;
    return (uint64_t)S * qd + t;
}

// the same with -d supplied (r = x + t*(-d): one IMAD) and the fix-up as a predicated add
__device__ __forceinline__ uint64_t fixed_q_nd(uint32_t S, uint32_t d, uint32_t nd, uint32_t qd, uint32_t rp) {
    const uint32_t x = S * rp;
    uint32_t t = __umulhi(x, qd);
    const uint32_t r = x + t * nd;
    asm("{\n\t.reg .pred p;\n\tsetp.ge.u32 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}" : "+r"(t) : "r"(r), "r"(d));
    return (uint64_t)S * qd + t;
}

__device__ __forceinline__ uint64_t pair_q(uint32_t S, const RowInfo &a, const RowInfo &b) {
    return a.tw <= b.tw ? fixed_q(S, a.tw, a.qd, a.rp) : fixed_q(S, b.tw, b.qd, b.rp);
}

// ------------------------------------------------------------------------------------
// kernels (defined in k_*.cu)
// ------------------------------------------------------------------------------------
struct ProfileArgs {
    const uint8_t *ascii;
    const int64_t *off;
    int64_t n;
    int64_t i_begin, i_end;          // the sequences this launch profiles (a chunk of [0, n))
    int64_t first_idx;
    int k, A, V, alphabet, pl;
    const int64_t *shard_base;       // device [pl+1]
    RowInfo *rowinfo;
    uint32_t *csr;
    int32_t *dcnt;
    uint32_t *M;                     // [pl][V]
    unsigned long long *err;         // [4]: first bad symbol (idx<<32|pos), first short idx, first long idx, pad
    unsigned long long *kinfo;       // [pl][kKinfo] (see kKinfo)
    uint32_t *Xc;                    // [pl][kNumCaps][V]: #{i : n_i(tau) > 2^j} (zeroed)
    uint32_t *Mb;                    // [pl][ceil(V/32)]: k-mers present in the shard (zeroed; M >= 2 goes to M)
    int32_t *nhi;                    // [n] entries with count >= 2 (repeated in each CSR row's tail)
    unsigned long long *T;           // [n] within-shard rank sums, zeroed here for the all-pairs kernel
    uint32_t *lcnt;                  // [pl][kLenBinsMax] Tw histogram of the length order (zeroed), or NULL
    int blk;                         // 1: long sequences (average L >= 1024): one block per sequence (k_profile_blk)
};
void launch_profile(const ProfileArgs &a, cudaStream_t st);
// the per-step accumulators of K1/K2 and K3 cleared in one launch: M, Mb, Xc = 0; err = all ones;
// status + kinfo = 0
void launch_profile_reset(uint32_t *M, size_t nM, uint32_t *Mb, size_t nMb, uint32_t *Xc, size_t nXc,
                          unsigned long long *err4, unsigned long long *statkinfo, size_t nsk, uint32_t *lcnt,
                          size_t nl, cudaStream_t st);
// K3 in one launch, one block per shard (k_profile.cu): statistics per candidate cap, the layer cap
// T_s and operand width K_s (clipped to kcap_blocks; status[0] |= 1 on overflow, status[1] = max K_s;
// kinfo[s][20] = K_s, [21] = T_s), the column map col0 and the K6 list offsets (xtot[s] totals)
void launch_shard_plan(uint32_t *M, const uint32_t *Mb, const uint32_t *Xc, unsigned long long *kinfo, int pl, int V,
                       int allow_cap, int64_t kcap_blocks, int kcpb, uint32_t *cap, uint32_t *xsel, uint32_t *ident,
                       int64_t *kblocks, unsigned long long *status, uint32_t *col0, uint32_t *xoff,
                       unsigned long long *xtot, uint32_t *xcur, const uint32_t *lcnt, uint32_t *lpos,
                       const int64_t *shard_base, cudaStream_t st);
// the count-exchange status of this rank appended to its count block: [0] operand overflow,
// [1] first input error kind (0 none, 1 symbol, 2 too short, 3 too long), [2] out_bytes, [3] 0
void launch_status_tail(const unsigned long long *status, const unsigned long long *err, int64_t out_bytes,
                        int64_t *tail, cudaStream_t st);

struct OperandArgs {
    const uint32_t *csr;
    const int64_t *off;
    const int32_t *dcnt;
    const uint32_t *col0;            // [pl][V]
    const int64_t *shard_base;       // device [pl+1] local row bases
    const int64_t *shard_rowpad;     // device [pl+1] padded operand row bases
    int64_t rows_pad;
    int64_t stride;                  // bytes per operand row
    int k, V, pl;
    int fp4;                         // pack two 4-bit e2m1 entries per byte (1.0 = 0x2)
    void *op;
    const uint32_t *cap;             // device [pl] layer cap T_s per shard (kNoCap: none), or NULL
    const int32_t *sigma;            // device [n] length order (sorted position -> local index), or NULL
    const uint32_t *ident;           // device [pl] 1: the column of tau is tau (cap 1, all V k-mers present), or NULL
    const int64_t *kblocks;          // device [pl] 128-byte K blocks of each shard's rows (only those are
                                     // written; the row stride is the capacity), or NULL: the whole stride
    const RowInfo *rowinfo;          // [n] input order (.shard = local shard)  (K4)
    const int32_t *sigma_inv;        // [n] local index -> length-order slot in its shard, or NULL (K4)
    int64_t n;                       // local sequences (K4)
    int wide;                        // 1: long rows (average Tw >= 1024): one block per row (k_indicator_blk)
};
void launch_indicator(const OperandArgs &a, cudaStream_t st);
// length order by counting (K3): Tw histogram per shard, per-shard scan up to the max Tw in kinfo[3],
// slot scatter -> sigma, sigma_inv, rinfo_s (ties in arbitrary order); 3 launches + 1 memset
void launch_lenorder(const RowInfo *rowinfo, const int64_t *shard_base, int pl, int64_t n, uint32_t *pos,
                     int32_t *sigma, int32_t *sigma_inv, RowInfo *rinfo_s, cudaStream_t st);
// the same order made deterministic (ties by index; tile split): keys, a stable sort, then apply
void launch_lenkeys(const RowInfo *rowinfo, int64_t n, unsigned long long *keys, int32_t *rows, cudaStream_t st);
void launch_lenapply(const int32_t *rows_sorted, const RowInfo *rowinfo, const int64_t *shard_base, int64_t n,
                     int32_t *sigma, int32_t *sigma_inv, RowInfo *rinfo_s, cudaStream_t st);
// K6: the sparse excess of the capped layers (k_excess.cu),
//   e_ij = sum_tau min((n_i(tau) - T_s)+, (n_j(tau) - T_s)+)   for i < j in shard s,
// as a dense u8 matrix E_s[r][c] over sorted positions (length order; row pitch rup(w_s, 16);
// only c > r is written).
struct ExcessArgs {
    const uint32_t *csr;
    const int64_t *off;
    const int32_t *nhi;              // [n] count >= 2 entries of each CSR row (its last nhi slots)
    const int64_t *shard_base;       // device [pl+1]
    int64_t n;
    int pl, V, k;
    const uint32_t *cap;             // device [pl]
    const uint32_t *xoff;            // device [pl][V]
    const unsigned long long *xtot;  // device [pl]
    const uint32_t *lists;           // K6 lists L_tau (from k_xfill)
    int accb;                        // bytes of one row accumulator (max_w rounded up to 16)
    const int32_t *sigma;            // [n] length order: sorted position -> local index
    const int32_t *sigma_inv;        // [n] local index -> sorted position
    const RowInfo *rowinfo;          // [n] input order (.shard)
    const uint8_t *rb_own;           // tile split: [row blocks] 1 = this rank computes the row block's tiles, or NULL
    const int64_t *shard_rowpad;     // device [pl+1] (row block of a row: (rowpad[s] + local) / rb_rows)
    int rb_rows;                     // rows per row block (the all-pairs tile height)
    uint2 *xrow;                     // [n] .x = 1 if the row (sorted position) has excess
    uint8_t *E;                      // dense excess rows
    uint8_t *zero_seg;               // 256 bytes zeroed by k_xfill (the staging source of rows without excess)
    const int64_t *ebase;            // device [pl+1] per shard byte offset of E_s
};
int launch_excess(const ExcessArgs &a, cudaStream_t st);
// K6 lists (before launch_excess); lpos != NULL: the length order's scatter fused in (see k_excess.cu)
void launch_xfill(const ExcessArgs &a, uint32_t *xcur, uint32_t *lpos, int32_t *sigma, int32_t *sigma_inv,
                  RowInfo *rinfo_s, cudaStream_t st);
void launch_dense_counts(const OperandArgs &a, cudaStream_t st);

struct AllPairsArgs {
    const void *op;                  // operand
    int64_t stride;                  // bytes per operand row
    const RowInfo *rowinfo;          // [n] local rows (TC path: in length order, .shard = local index)
    const int64_t *shard_base;       // device [pl+1]
    const int64_t *shard_rowpad;     // device [pl+1]
    const int64_t *shard_kblocks;    // device [pl]: 128-col K blocks of each shard (TC path)
    int pl;
    int64_t max_w;
    unsigned long long *T;           // [n]
    uint16_t *sim;                   // optional [sum w_s^2]
    const int64_t *sim_base;         // device [pl] offsets into sim
    int vwords;                      // ALU: u32 words per row (V_pad/2)
    int num_sms;
    const int64_t *tile_base;        // ALU: device [pl+1] prefix of 64x64 upper-triangle tiles
    int64_t n_tiles;
    const void *tmap;                // TC: CUtensorMap (64 B, host copy passed as __grid_constant__)
    const int64_t *h_shard_base;     // host copies (launch configuration)
    const int64_t *h_shard_rowpad;
    int64_t kblocks_hint;            // TC: largest K block count expected (picks the deep ring; any value is exact)
    int kind;                        // TC: 0 = int8 operands (kind::i8), 1 = packed fp4 (kind::mxf4)
    const void *tiles;               // TC: device tile table (16 B per tile) and its length
    int64_t n_tiles_tc;
    int cg;                          // TC: 1 = one CTA per tile, 2 = CTA pair (cta_group::2, M = 256)
    const uint2 *xrow;               // TC: K6 row flags (.x = 1: the row has excess), or NULL
    const uint8_t *E;                // TC: K6 dense excess rows (see ExcessArgs)
    const int64_t *ebase;            // TC: device [pl+1] per shard byte offset of E_s
    const uint8_t *zero;             // TC: 256 zero bytes (the staging source of rows without excess)
};
void launch_allpairs_alu(const AllPairsArgs &a, cudaStream_t st);
int launch_allpairs_tc(const AllPairsArgs &a, cudaStream_t st, std::string &err);
bool tc_supported(std::string &why);
int64_t tc_tiles_bytes(int pl, const int64_t *h_shard_base, int kind, int cg);
int64_t tc_tiles_bound(int64_t n, int pl);
int64_t tc_build_tiles(int pl, const int64_t *h_shard_base, int kind, int cg, void *host_out, int64_t cap,
                       int split_world = 1, int split_rank = 0, uint8_t *own_out = nullptr);
int tc_bn(int kind);

struct AncArgs {
    const unsigned long long *T;
    const int64_t *shard_base;
    const uint32_t *csr;
    const int64_t *off;
    const int32_t *dcnt;
    const RowInfo *rowinfo;
    int64_t first_idx;
    int k, V, pl;
    size_t rec_bytes;
    int64_t *anc_local;              // [pl] local row of each shard's ancestor
    uint8_t *rec_out;                // [pl] records
};
void launch_local_ancestors(const AncArgs &a, cudaStream_t st);

struct RankArgs {
    const uint8_t *anc_all;          // [p] records
    size_t rec_bytes;
    int p, k, V;
    uint32_t *Sab;                   // [p][p] scratch
    long long *ga_info;              // [2 + p]: GA record index, GA source index, ancestors' source idx
    const uint32_t *csr;
    const int64_t *off;
    const int32_t *dcnt;
    const RowInfo *rowinfo;
    int64_t n, first_idx;
    uint32_t *S_ga, *den_ga;
    unsigned long long *key;
    int32_t *perm_in;
    unsigned long long *ckey;        // sort key (shard << 32) | min(q, 2^32 - 1), sorted with the row as value
};
void launch_ga_pairs(const RankArgs &a, cudaStream_t st);
void launch_rank_vs_ga(const RankArgs &a, cudaStream_t st);

void launch_samples(const unsigned long long *key_sorted, const int64_t *shard_base, int pl, int p,
                    unsigned long long *samples_out, cudaStream_t st);
// unpack + the exclusive prefix of L in sorted order in one single-pass launch (lpre[0..n]);
// sstate[2] (epoch, done counter) and status[unpack_scan_tiles(n)] zeroed when the layout is new
void launch_unpack_scan(const unsigned long long *ckey_sorted, const int32_t *perm_sorted, int64_t n, int64_t first_idx,
                        unsigned long long *key_sorted, const RowInfo *rowinfo, int k, int64_t *len_sorted, int qbits,
                        int ibits, int64_t *lpre, uint32_t *sstate, unsigned long long *status, cudaStream_t st);
int64_t unpack_scan_tiles(int64_t n);
void launch_unpack_sorted(const unsigned long long *ckey_sorted, const int32_t *perm_sorted, int64_t n,
                          int64_t first_idx, unsigned long long *key_sorted, const RowInfo *rowinfo, int k,
                          int64_t *len_sorted, int qbits, int ibits, cudaStream_t st);
// f1: rank against the k*p gathered samples
void launch_tkeys(const unsigned long long *T, const RowInfo *rowinfo, int64_t n, unsigned long long *keys,
                  int32_t *rows, cudaStream_t st);
void launch_sample_records(const int32_t *rows_sorted, const int64_t *shard_base, int pl, int p, const uint32_t *csr,
                           const int64_t *off, const int32_t *dcnt, const RowInfo *rowinfo, int64_t first_idx, int k,
                           size_t rec_bytes, uint8_t *rec_out, cudaStream_t st);
int launch_rank_vs_samples(const RankArgs &a, int m, unsigned long long *Tp, int num_sms, cudaStream_t st);
// f1 on the tensor cores (k_allpairs_tc.cu; packed-fp4 operand only): T'_i += sum_j q(x_i, s_j)
struct F1Args {
    const uint8_t *rec;              // [m] gathered sample records
    size_t rec_bytes;
    int m, V, k, pl, num_sms;
    int64_t n, rows_pad, stride;     // local rows, operand rows (padded), operand row bytes
    const void *op;                  // the all-pairs operand A (K4, length order)
    const int64_t *shard_base, *shard_rowpad, *kblocks;
    const uint32_t *M, *col0, *cap, *ident;
    const int32_t *sigma, *nhi;
    const uint32_t *csr;
    const int64_t *off;
    const RowInfo *rinfo_s;
    uint8_t *bop;                    // scratch: [pl][f1_tc_rows(m)][stride] the samples' operand rows
    uint8_t *ex;                     // scratch: [rows_pad][f1_tc_rows(m)] e_ij
    uint16_t *cT;                    // scratch: [V][f1_tc_rows(m)] the samples' counts, transposed
    unsigned long long *Tp;          // [n] T' (accumulated; zeroed by the caller)
};
int f1_tc_rows(int m);
int launch_f1_tc(const F1Args &a, cudaStream_t st, std::string &err);
void launch_f1_keys(const unsigned long long *Tp, int64_t n, int tbits, int ibits, int64_t first_idx,
                    const RowInfo *rowinfo, unsigned long long *key, unsigned long long *ckey, int32_t *perm_in,
                    uint32_t *S_ga, uint32_t *den_ga, cudaStream_t st);
void launch_f1_gainfo(const int64_t *anc_local, int pl, int shard0, int p, int64_t first_idx, long long *ga_info,
                      cudaStream_t st);

// K14: rank-merge of nr sorted runs of unique keys (keys at stride `kstride` u64 words):
// out position of element t = sum over runs r of #{keys in r < key_t}.
struct MergeArgs {
    const unsigned long long *keys;  // element t's key at keys[t * kstride]
    int kstride;
    int64_t n;
    const int64_t *run_start;        // device [nr + 1]
    int nr;
    // element length: lens[t * lstride] if lens, else rowinfo[perm[t]].tw + k - 1
    const unsigned long long *lens;
    int lstride;
    const int32_t *perm;
    const RowInfo *rowinfo;
    int k;
    unsigned long long *out_key;     // [n]
    int64_t *out_len;                // [n]
    int32_t *out_src;                // [n] element index t of each output slot
    // [n + 1] exclusive prefix of the element lengths over the concatenated runs: the output
    // residue offsets out_off[n + 1] follow from every element's rank in every run (no scan)
    const int64_t *cpre;
    int64_t *out_off;
};
void launch_rank_merge(const MergeArgs &a, cudaStream_t st);
// residues: dst_res[dst_off[r] ...] = src_res[src_off(out_src[r]) ...]; src_off(t) = src_off[perm ? perm[t] : t]
void launch_gather_res(const int32_t *out_src, const int32_t *perm, int64_t n, const int64_t *src_off,
                       const uint8_t *src_res, const int64_t *dst_off, uint8_t *dst_res, cudaStream_t st);
void launch_lens_recv(const unsigned long long *recv_meta, int64_t n, int64_t *len, cudaStream_t st);

struct PlanArgs {
    const unsigned long long *samples_all;   // [p(p-1)]
    int p, pl;
    const unsigned long long *key_sorted;    // [n] per shard sorted keys
    const int32_t *perm_sorted;              // [n] local rows in sorted order
    const int64_t *shard_base;
    const RowInfo *rowinfo;
    int k;
    unsigned long long *pivots;              // [p-1] out
    int64_t *bnd;                            // [pl][p] out: sorted-position end of each bucket slice
    const int64_t *lpre;                     // [n + 1] exclusive prefix of L in sorted order (all shards)
    int64_t *counts;                         // [pl][p][2] out
};
void launch_plan(const PlanArgs &a, cudaStream_t st);

struct PackArgs {
    const unsigned long long *key_sorted;
    const int32_t *perm_sorted;
    const int64_t *shard_base;
    const int64_t *bnd;                      // [pl][p]
    const int64_t *lpre;                     // [n + 1]
    const int64_t *seg;                      // [pl][p][2]: send seq offset, send residue offset of each slice
    const RowInfo *rowinfo;
    const uint8_t *ascii;
    const int64_t *off;
    int p, pl, k;
    int64_t n;
    unsigned long long *send_meta;           // [.][2]
    uint8_t *send_res;
};
void launch_pack(const PackArgs &a, cudaStream_t st);

// receive side
void launch_meta_from_local(const unsigned long long *key, const RowInfo *rowinfo, int k, int64_t n,
                            unsigned long long *keys_in, int32_t *vals_in, int64_t *len_in, cudaStream_t st);
void launch_meta_from_recv(const unsigned long long *recv_meta, int64_t n, unsigned long long *keys_in,
                           int32_t *vals_in, int64_t *len_in, cudaStream_t st);
void launch_gather_len(const int32_t *perm, const int64_t *len_in, int64_t n, int64_t *len_sorted, cudaStream_t st);
void launch_gather_out(const int32_t *perm, int64_t n, const int64_t *src_off, const uint8_t *src_res,
                       const int64_t *dst_off, uint8_t *dst_res, cudaStream_t st);

void launch_selftest_fixed(int max_den, unsigned long long *bad, cudaStream_t st);
// one-block stable radix sort of n <= kSmallSortMax (key, value) pairs (k_sort.cu); 0 or -1
constexpr int kSmallSortMax = 512 * 32;
int small_sort_pairs(const uint32_t *ki, const int32_t *vi, int n, uint32_t *ko, int32_t *vo, int b0, int b1,
                     cudaStream_t st);
int small_sort_pairs(const unsigned long long *ki, const int32_t *vi, int n, unsigned long long *ko, int32_t *vo,
                     int b0, int b1, cudaStream_t st);
// per-segment stable sort by key bits [0, end_bit <= 32), every segment <= kSmallSortMax pairs; 0 or -1
int seg_sort_pairs(const uint32_t *ki, const int32_t *vi, const int64_t *seg, int nseg, uint32_t *ko, int32_t *vo,
                   int end_bit, cudaStream_t st);
int seg_sort_pairs(const unsigned long long *ki, const int32_t *vi, const int64_t *seg, int nseg,
                   unsigned long long *ko, int32_t *vo, int end_bit, cudaStream_t st);
// the same with every segment (at most max_seg pairs) split into runs of at most 2048 pairs sorted by
// separate blocks (in place in ki, vi), then merged stably into (ko, vo); 0 or -1
int seg_sort_pairs_runs(unsigned long long *ki, int32_t *vi, const int64_t *seg, int nseg, int64_t max_seg, int64_t n,
                        unsigned long long *ko, int32_t *vo, int end_bit, cudaStream_t st);
void launch_rebase(const int64_t *src, int64_t n1, int64_t *off, cudaStream_t st);
void launch_distance(const uint16_t *sim, const RowInfo *rowinfo, int64_t w, float *D, cudaStream_t st);
void launch_distance64(const uint16_t *sim, const RowInfo *rowinfo, int64_t w, double *D, cudaStream_t st);
size_t upgma_workspace(int64_t n);
void launch_upgma(double *D, int64_t n, int64_t *merges, double *heights, int64_t *sizes, void *ws, cudaStream_t st);

// Dynamic shared memory opt-in (> 48 KB) of kernel `func` on the CURRENT device. The attribute is
// per device, so the opt-in is remembered per (device, kernel) and only raised; thread-safe
// (sad_util.cu).
cudaError_t smem_optin_raw(const void *func, size_t bytes);
template <class F>
inline cudaError_t smem_optin(F *func, size_t bytes) {
    return smem_optin_raw(reinterpret_cast<const void *>(func), bytes);
}

// Makes a context's device current for the duration of an ABI call and restores the caller's
// device afterwards (every entry point runs on ctx->cfg.device, whatever the caller made current).
struct DeviceScope {
    int prev = -1, dev = -1;
    explicit DeviceScope(int d) : dev(d) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceScope() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
    DeviceScope(const DeviceScope &) = delete;
    DeviceScope &operator=(const DeviceScope &) = delete;
};

}  // namespace sad

// ------------------------------------------------------------------------------------
// the context
// ------------------------------------------------------------------------------------
struct sad_ctx {
    sad_config cfg{};
    cudaStream_t st = nullptr;
    cudaStream_t side = nullptr;     // internal stream: K6 rows run beside K4 (fork/join by events)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_stats = nullptr;  // K1/K2 statistics on the host side; the length order runs on meanwhile
    static constexpr int kLoadChunks = 16;     // host loads: chunked H2D copies on `side`, each chunk's
    cudaEvent_t ev_chunk[kLoadChunks] = {};    // k-mer counts launched on `st` as soon as it lands
    bool profiled = false;                     // K1/K2 already launched by sad_load
    int A = 0, V = 0, pl = 0, shard0 = 0;
    int num_sms = 148;
    std::string err;
    int sticky = 0;
    int64_t err_idx = -1, err_pos = -1;
    int stage = 0;                   // 0 created, 1 loaded, 2 profiles, 3 rank_local, 4 rank_global, 5 plan, 6 finished

    // sizes
    int64_t n = 0, n_global = 0, first_idx = 0, R = 0;
    std::vector<int64_t> shard_base, shard_rowpad;   // [pl+1]
    int64_t rows_pad = 0, max_w = 0;
    std::vector<int64_t> h_windows, h_distinct, h_K; // [pl]
    std::vector<uint32_t> h_cap;                      // [pl] layer cap T_s (kNoCap: all layers dense)
    int64_t K_stride = 0, V_pad = 0;
    bool use_tc = false;
    int tc_kind = 1;                 // 0 = int8, 1 = fp4
    int tc_cg = 2;                   // 1 or 2 CTAs per tensor-core tile
    int64_t kcols_per_block = 128;   // operand columns per 128-byte K block

    // device pointers carved from the caller workspace
    uint8_t *ws = nullptr;
    size_t ws_bytes = 0;
    uint8_t *d_ascii = nullptr;
    int64_t *d_off = nullptr;
    sad::RowInfo *d_rowinfo = nullptr;
    uint32_t *d_csr = nullptr;
    int32_t *d_dcnt = nullptr, *d_nhi = nullptr;
    int32_t *d_sigma = nullptr, *d_sigma_inv = nullptr;   // length order of every shard (TC path)
    sad::RowInfo *d_rinfo_s = nullptr;                    // RowInfo in length order, .shard = local index
    uint32_t *d_M = nullptr, *d_Mb = nullptr, *d_col0 = nullptr;
    uint32_t *d_lcnt = nullptr;      // [pl][kLenBinsMax] length-order counts, then positions (scan)
    unsigned long long *d_err = nullptr, *d_kinfo = nullptr;
    uint32_t *d_cap = nullptr, *d_xsel = nullptr;   // layer cap T_s and its index j_s per shard
    uint32_t *d_ident = nullptr;                    // per shard: identity column map (K4 skips col0)
    uint32_t *d_Xc = nullptr;        // [pl][kNumCaps][V] entries above each candidate cap
    uint32_t *d_xoff = nullptr, *d_xcur = nullptr;  // [pl][V] K6 list offsets (+ u64 [pl] totals) / cursors
    uint2 *d_xrow = nullptr;         // [n] K6 row flags
    int64_t *d_ebase = nullptr;      // [pl+1] K6 dense excess matrix bases (host copy below)
    std::vector<int64_t> h_ebase;
    int64_t *d_shard_base = nullptr, *d_shard_rowpad = nullptr, *d_kblocks = nullptr, *d_sim_base = nullptr;
    int64_t *d_tile_base = nullptr;
    void *d_tc_tiles = nullptr;      // TC tile table (workspace), built once per layout
    int64_t tc_tiles_cap = 0, tc_tiles_n = 0;
    void *h_tiles = nullptr;         // pinned staging of the tile table
    size_t h_tiles_bytes = 0;
    int64_t alu_tiles = 0;
    unsigned long long *d_T = nullptr;
    int64_t *d_anc_local = nullptr;
    uint32_t *d_Sab = nullptr;
    long long *d_ga_info = nullptr;
    uint32_t *d_S_ga = nullptr, *d_den_ga = nullptr;
    unsigned long long *d_key = nullptr, *d_key_sorted = nullptr, *d_ckey = nullptr, *d_ckey_sorted = nullptr;
    int64_t *d_runs = nullptr;
    int32_t *d_perm_in = nullptr, *d_perm_sorted = nullptr;
    unsigned long long *d_pivots = nullptr;
    int64_t *d_bnd = nullptr, *d_lpre = nullptr, *d_seg = nullptr, *d_counts = nullptr;
    int64_t *d_len_sorted = nullptr;  // [n] L of each sequence in sorted order (scanned into d_lpre)
    uint32_t *d_scan_state = nullptr;            // k_unpack_scan: epoch, done counter
    unsigned long long *d_scan_status = nullptr; // k_unpack_scan: per-tile look-back status
    bool counts_pending = false;
    void *d_tmap = nullptr;
    void *d_cub = nullptr;
    size_t cub_bytes = 0;
    uint16_t *d_sim = nullptr;       // optional (SAD_F_KEEP_SIM), inside the workspace
    int64_t sim_elems = 0;

    // last operand / output
    void *d_operand = nullptr;
    uint8_t *d_out = nullptr;
    size_t out_bytes = 0;
    int64_t out_n = 0, out_r = 0;
    std::vector<int64_t> bucket_sizes, bucket_first;  // [p] sizes, first row of owned buckets in out
    std::vector<int64_t> h_counts_all;                  // [p][p][2]

    // asynchronous step statistics: k-mer statistics, errors and the operand status are copied to
    // pinned host memory at the end of sad_build_profiles and read at the next synchronizing call
    unsigned long long *h_stats = nullptr;           // [8 + pl * kKinfo]: err[4], status[4], kinfo
    cudaEvent_t ev_async = nullptr;
    bool stats_pending = false;
    unsigned long long *d_status = nullptr;         // [4] device: operand overflow, max K_s, -, -
    int64_t kcap_blocks = 0;                         // operand K capacity (128-byte blocks per row)
    int64_t kcap_next = 0;                           // the capacity the next step starts with
    bool f1_tc = false;              // f1 rank vs samples as a tensor-core contraction (F1Args)
    int tile_world = 1, tile_rank = 0;   // SAD_F_TILE_SPLIT: the all-pairs tiles split over tile_world ranks
    bool tile_reduce = false;        // ... and T summed over them on the communicator (else: the caller's job)
    uint8_t *d_rb_own = nullptr;     // [row blocks] tiles owned by this rank (K6 skips the other rows)
    int64_t kmax_blocks_seen = -1;                   // largest K blocks of the last absorbed step (-1: none)
    bool allow_cap = false;                          // capped layers + K6 excess possible in this layout
    int64_t x_entries_bound = 0;                     // K6 list entries bound (all CSR entries)
    int ibits = 31;                                  // key = (rank << ibits) + source index
    int tbits = 32;                                  // bits of the rank value in the a7 sort key

    // collective API
    void *comm = nullptr;                            // ncclComm_t (NULL: none)
    void *d_anc_mine = nullptr, *d_anc_all = nullptr;
    unsigned long long *d_smp_mine = nullptr, *d_smp_all = nullptr;
    int64_t *d_cnt_send = nullptr, *d_cnt_all = nullptr;   // [pl*p*2 + 4] / [world][pl*p*2 + 4]
    int64_t *h_cnt_all = nullptr;                    // pinned copy of d_cnt_all
    int64_t *h_seg = nullptr;                        // pinned pack plan of the collective path
    int64_t *h_runs = nullptr;                       // pinned receive runs
    unsigned long long *d_send_meta = nullptr;
    uint8_t *d_send_res = nullptr;
    bool capturing = false;                          // the stream is being captured into a CUDA graph
    bool t_used = false;
    bool lenorder_deferred = false;                  // the length order's scatter runs fused with K6's lists                             // T accumulated since K1/K2 last zeroed it
    cudaEvent_t gev[4] = {};                         // stage events recorded inside a captured step
    bool graph_events = false;
    bool out_recv_layout = false;                    // the output buffer holds the receive buffers too

    // layout of the last uploaded per-shard tables
    uint8_t *tbl_ws = nullptr;
    int64_t tbl_n = -1, tbl_ng = -1, tbl_first = -1, tbl_R = -1;

    // pinned host staging
    unsigned long long *h_small = nullptr;              // pinned, 4096 u64

    // stats
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pairs_ap, ev_pairs_op, ev_free;
    double ms_ap = 0, ms_op = 0;
    int64_t calls = 0, pairs = 0, macs = 0, launches_last = 0, launches_step = 0;
};
