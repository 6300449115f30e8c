// sad_api.cu — the C ABI of libsad.so (include/sad.h): argument checks, workspace carving,
// stage orchestration on the caller's stream, and the collective calls over the library's own
// NCCL communicator. All arithmetic of the method is in k_*.cu.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>

#include "sad_internal.cuh"

using namespace sad;

namespace {

inline int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct Bump {
    uint8_t *base;
    size_t off = 0;
    template <class T>
    T *take(size_t count) {
        off = (size_t)rup((int64_t)off, 256);
        T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
        off += count * sizeof(T);
        return p;
    }
};

int fail(sad_ctx *c, int code, const char *fmt, ...) __attribute__((format(printf, 3, 4)));
int fail(sad_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
    c->sticky = code;
    return code;
}

// a failure that leaves the context usable (SAD_E_REPLAN, a too small output buffer)
int soft_fail(sad_ctx *c, int code, const char *fmt, ...) __attribute__((format(printf, 3, 4)));
int soft_fail(sad_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
    return code;
}

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(ctx, SAD_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                \
    } while (0)

#define NK(call)                                                                            \
    do {                                                                                    \
        ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess)                                                              \
            return fail(ctx, SAD_E_NCCL, "%s failed: %s (%s:%d)", #call, ncclGetErrorString(r_), \
                        __FILE__, __LINE__);                                                \
    } while (0)

#define LAUNCHED()                                                                          \
    do {                                                                                    \
        ++ctx->launches_step;                                                               \
        cudaError_t e_ = cudaGetLastError();                                                \
        if (e_ != cudaSuccess)                                                              \
            return fail(ctx, SAD_E_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                \
    } while (0)

// argument / state checks of every context call, then the context's device made current for the
// rest of the call (restored on return: the caller's current device is left as it was)
#define GUARD(min_stage)                                                                    \
    if (!ctx) return SAD_E_ARG;                                                             \
    if (ctx->sticky) return SAD_E_STATE;                                                    \
    if (ctx->stage < (min_stage)) return fail(ctx, SAD_E_STATE, "call order: stage %d < %d", ctx->stage, (min_stage)); \
    DeviceScope dev_scope_(ctx->cfg.device)

inline ncclComm_t comm_of(const sad_ctx *c) { return reinterpret_cast<ncclComm_t>(c->comm); }

// shard bases of this rank under the block split of reading A15
void shard_layout(const sad_ctx *c, int64_t n_global, std::vector<int64_t> &sb) {
    const int p = c->cfg.p;
    const int64_t base = n_global / p, extra = n_global % p;
    sb.assign(c->pl + 1, 0);
    for (int s = 0; s < c->pl; ++s) sb[s + 1] = sb[s] + base + (c->shard0 + s < extra ? 1 : 0);
}

int64_t first_index_of_rank(const sad_ctx *c, int64_t n_global) {
    const int p = c->cfg.p;
    const int64_t base = n_global / p, extra = n_global % p;
    int64_t g0 = 0;
    for (int s = 0; s < c->shard0; ++s) g0 += base + (s < extra ? 1 : 0);
    return g0;
}

size_t cub_bytes_needed(int64_t n, int pl) {
    size_t a = 0, b = 0;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, a, (const unsigned long long *)nullptr,
                                             (unsigned long long *)nullptr, (const int32_t *)nullptr,
                                             (int32_t *)nullptr, (int)std::max<int64_t>(n, 1), pl,
                                             (const int64_t *)nullptr, (const int64_t *)nullptr, 0, 64);
    cub::DeviceRadixSort::SortKeys(nullptr, b, (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                   (int)std::max<int64_t>(n, 1), 0, 64);
    size_t c = 0, d = 0, e = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, e, (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)std::max<int64_t>(n, 1), 0, 64);
    a = std::max(a, e);
    cub::DeviceRadixSort::SortPairs(nullptr, c, (const uint32_t *)nullptr, (uint32_t *)nullptr, (const int32_t *)nullptr,
                                    (int32_t *)nullptr, (int)std::max<int64_t>(n, 1), 0, 32);
    cub::DeviceScan::InclusiveSum(nullptr, d, (const int64_t *)nullptr, (int64_t *)nullptr, (int)std::max<int64_t>(n, 1));
    size_t f = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, f, (const uint32_t *)nullptr, (uint32_t *)nullptr, pl * kLenBinsMax);
    return std::max(std::max(std::max(a, b), std::max(c, d)), f) + 1024;
}

int exchange_records(const sad_ctx *c) {
    return (c->cfg.flags & SAD_F_RANK_SAMPLES) ? c->pl * (c->cfg.p - 1) : c->pl;
}
size_t record_bytes(const sad_ctx *c) { return (size_t)rup(16 + 2 * (int64_t)c->V, 16); }
int64_t count_block(const sad_ctx *c) { return (int64_t)c->pl * c->cfg.p * 2 + 4; }   // counts + status tail

// carve the workspace; with base == nullptr only the size is computed
// rows per all-pairs row block (the tile height: 128, or 256 for CTA pairs)
static inline int64_t tc_row_block(const sad_ctx *c) { return 128 * (int64_t)c->tc_cg; }

size_t carve(sad_ctx *c, uint8_t *base, int64_t n, int64_t R) {
    Bump b{base};
    const int pl = c->pl, p = c->cfg.p, V = c->V, G = c->cfg.world;
    c->d_ascii = b.take<uint8_t>((size_t)R + 528);     // + 512 + 16: vector reads past the last residue
    c->d_off = b.take<int64_t>((size_t)n + 1);
    c->d_rowinfo = b.take<RowInfo>((size_t)n);
    c->d_csr = b.take<uint32_t>((size_t)std::max<int64_t>(R, 1));
    c->d_dcnt = b.take<int32_t>((size_t)n);
    c->d_nhi = b.take<int32_t>((size_t)n);
    c->d_sigma = b.take<int32_t>((size_t)n);
    c->d_sigma_inv = b.take<int32_t>((size_t)n);
    c->d_rinfo_s = b.take<RowInfo>((size_t)n);
    c->d_M = b.take<uint32_t>((size_t)pl * V);
    c->d_Mb = b.take<uint32_t>((size_t)pl * ((V + 31) / 32));
    c->d_lcnt = b.take<uint32_t>((size_t)2 * pl * kLenBinsMax);
    c->d_col0 = b.take<uint32_t>((size_t)pl * V);
    // the step statistics block, copied to the host in one piece: err[4] | status[4] | kinfo
    c->d_err = b.take<unsigned long long>(8 + (size_t)pl * kKinfo);
    c->d_status = c->d_err ? c->d_err + 4 : nullptr;
    c->d_kinfo = c->d_err ? c->d_err + 8 : nullptr;
    c->d_cap = b.take<uint32_t>((size_t)pl);
    c->d_ident = b.take<uint32_t>((size_t)pl);
    c->d_xsel = b.take<uint32_t>((size_t)pl);
    c->d_Xc = b.take<uint32_t>((size_t)pl * kNumCaps * V);
    c->d_xoff = b.take<uint32_t>((size_t)pl * V + 2 * (size_t)pl + 2);
    c->d_xcur = b.take<uint32_t>((size_t)pl * V);
    c->d_xrow = b.take<uint2>((size_t)n);
    c->d_ebase = b.take<int64_t>((size_t)pl + 1);
    c->d_shard_base = b.take<int64_t>((size_t)pl + 1);
    c->d_shard_rowpad = b.take<int64_t>((size_t)pl + 1);
    c->d_kblocks = b.take<int64_t>((size_t)pl + 1);
    c->d_sim_base = b.take<int64_t>((size_t)pl + 1);
    c->d_tile_base = b.take<int64_t>((size_t)pl + 1);
    c->d_T = b.take<unsigned long long>((size_t)n);
    c->d_anc_local = b.take<int64_t>((size_t)pl);
    c->d_Sab = b.take<uint32_t>((size_t)p * p);
    c->d_ga_info = b.take<long long>((size_t)p + 2);
    c->d_S_ga = b.take<uint32_t>((size_t)n);
    c->d_den_ga = b.take<uint32_t>((size_t)n);
    c->d_key = b.take<unsigned long long>((size_t)n);
    c->d_key_sorted = b.take<unsigned long long>((size_t)n);
    c->d_ckey = b.take<unsigned long long>((size_t)n);
    c->d_ckey_sorted = b.take<unsigned long long>((size_t)n);
    c->d_runs = b.take<int64_t>((size_t)p + 1);
    c->d_perm_in = b.take<int32_t>((size_t)n);
    c->d_perm_sorted = b.take<int32_t>((size_t)n);
    c->d_pivots = b.take<unsigned long long>((size_t)p);
    c->d_bnd = b.take<int64_t>((size_t)pl * p);
    c->d_lpre = b.take<int64_t>((size_t)n + pl + 1);
    c->d_len_sorted = b.take<int64_t>((size_t)n);
    c->d_scan_state = b.take<uint32_t>(4);
    c->d_scan_status = b.take<unsigned long long>((size_t)unpack_scan_tiles(n) + 1);
    c->d_seg = b.take<int64_t>((size_t)pl * p * 2);
    c->d_counts = b.take<int64_t>((size_t)pl * p * 2);
    c->tc_tiles_cap = tc_tiles_bound(n, pl);
    c->d_tc_tiles = b.take<uint8_t>((size_t)c->tc_tiles_cap * 16);
    c->d_rb_own = b.take<uint8_t>((size_t)(n / 128 + pl + 2));   // per 128 padded operand rows
    c->cub_bytes = cub_bytes_needed(n, pl);
    c->d_cub = b.take<uint8_t>(c->cub_bytes);
    // collective API: exchange records, samples and counts (this rank's and all ranks')
    const int recs = exchange_records(c);
    c->d_anc_mine = b.take<uint8_t>((size_t)recs * record_bytes(c));
    c->d_anc_all = b.take<uint8_t>((size_t)G * recs * record_bytes(c));
    c->d_smp_mine = b.take<unsigned long long>((size_t)std::max(pl * (p - 1), 1));
    c->d_smp_all = b.take<unsigned long long>((size_t)std::max(p * (p - 1), 1));
    c->d_cnt_send = b.take<int64_t>((size_t)count_block(c));
    c->d_cnt_all = b.take<int64_t>((size_t)G * count_block(c));
    if (c->comm) {                   // send buffers of the all-to-all
        c->d_send_meta = b.take<unsigned long long>((size_t)2 * std::max<int64_t>(n, 1));
        c->d_send_res = b.take<uint8_t>((size_t)R + 16);
    } else {
        c->d_send_meta = nullptr;
        c->d_send_res = nullptr;
    }
    if (c->cfg.flags & SAD_F_KEEP_SIM) {
        c->sim_elems = n * n;
        c->d_sim = b.take<uint16_t>((size_t)c->sim_elems);
    } else {
        c->sim_elems = 0;
        c->d_sim = nullptr;
    }
    return b.off + 256;
}

struct OutLayout {
    unsigned long long *key, *keys_in, *recv_meta;
    int64_t *off, *len_in, *len_sorted, *src_off;
    uint8_t *res, *cub, *recv_res;
    int32_t *vals_in, *perm;
    size_t cub_bytes, total;
};

// the output buffer: keys, offsets, residues of the owned buckets, merge scratch and (collective
// API with an exchange) the all-to-all receive buffers
OutLayout out_layout(uint8_t *base, int64_t n, int64_t r, bool recv) {
    Bump b{base};
    OutLayout o{};
    o.key = b.take<unsigned long long>((size_t)n);
    o.off = b.take<int64_t>((size_t)n + 1);
    o.res = b.take<uint8_t>((size_t)r + 16);
    o.keys_in = b.take<unsigned long long>((size_t)n);
    o.vals_in = b.take<int32_t>((size_t)n);
    o.perm = b.take<int32_t>((size_t)n);
    o.len_in = b.take<int64_t>((size_t)n);
    o.len_sorted = b.take<int64_t>((size_t)n);
    o.src_off = b.take<int64_t>((size_t)n + 1);
    size_t a = 0, s1 = 0, s2 = 0;
    const int nn = (int)std::max<int64_t>(n, 1);
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, nn, 0, 64);
    cub::DeviceScan::ExclusiveSum(nullptr, s1, (const int64_t *)nullptr, (int64_t *)nullptr, nn);
    cub::DeviceScan::InclusiveSum(nullptr, s2, (const int64_t *)nullptr, (int64_t *)nullptr, nn);
    o.cub_bytes = std::max(a, std::max(s1, s2)) + 1024;
    o.cub = b.take<uint8_t>(o.cub_bytes);
    if (recv) {
        o.recv_meta = b.take<unsigned long long>((size_t)2 * std::max<int64_t>(n, 1));
        o.recv_res = b.take<uint8_t>((size_t)r + 16);
    }
    o.total = b.off + 256;
    return o;
}

// the collective path moves the buckets through NCCL (always when the context has a communicator)
// the data-path exchanges run on the communicator (a tile-split context uses it for T only)
inline bool coll_exchange(const sad_ctx *c) { return c->comm != nullptr && c->tile_world == 1; }

void sum_recv(const sad_ctx *c, const int64_t *h_counts_all, int64_t &n_out, int64_t &r_out) {
    const int p = c->cfg.p, bpr = c->pl;
    if (!h_counts_all) {          // world == 1: this rank receives exactly what it holds
        n_out = c->n;
        r_out = c->R;
        return;
    }
    n_out = r_out = 0;
    for (int s = 0; s < p; ++s)
        for (int b = c->shard0; b < c->shard0 + bpr; ++b) {
            n_out += h_counts_all[((size_t)s * p + b) * 2 + 0];
            r_out += h_counts_all[((size_t)s * p + b) * 2 + 1];
        }
}

// pinned host buffers of one context (sizes depend only on the configuration)
bool alloc_host(sad_ctx *c) {
    const int pl = c->pl, p = c->cfg.p, G = c->cfg.world;
    return cudaMallocHost(&c->h_small, 65536 * sizeof(unsigned long long)) == cudaSuccess &&
           cudaMallocHost(&c->h_stats, (8 + (size_t)pl * kKinfo) * sizeof(unsigned long long)) == cudaSuccess &&
           cudaMallocHost(&c->h_cnt_all, (size_t)G * count_block(c) * sizeof(int64_t)) == cudaSuccess &&
           cudaMallocHost(&c->h_seg, (size_t)pl * p * 2 * sizeof(int64_t)) == cudaSuccess &&
           cudaMallocHost(&c->h_runs, ((size_t)p + 1) * sizeof(int64_t)) == cudaSuccess;
}

}  // namespace

// stable (key, row) radix sort: one block for small inputs, else cub::DeviceRadixSort
template <typename K>
static cudaError_t sort_pairs(sad_ctx *ctx, const K *ki, K *ko, const int32_t *vi, int32_t *vo, int n, int end_bit) {
    // (one block wins for 32-bit keys; for 64-bit keys the device sort's passes are faster)
    if (sizeof(K) == 4 && n <= kSmallSortMax && small_sort_pairs(ki, vi, n, ko, vo, 0, end_bit, ctx->st) == 0)
        return cudaGetLastError();
    size_t tb = ctx->cub_bytes;
    return cub::DeviceRadixSort::SortPairs(ctx->d_cub, tb, ki, ko, vi, vo, n, 0, end_bit, ctx->st);
}

// the K6 list totals, behind the per-(shard, tau) list offsets
static unsigned long long *xtot_of(const sad_ctx *ctx) {
    unsigned long long *x = reinterpret_cast<unsigned long long *>(ctx->d_xoff + (size_t)ctx->pl * ctx->V + 1);
    return reinterpret_cast<unsigned long long *>(rup(reinterpret_cast<int64_t>(x), 8));
}

// operand K capacity of a fresh layout: with capped layers K_s = sum_tau min(M(tau), T_s) <= 8 A^k
// (T_s <= 8); uncapped shards that need more are flagged and replanned
static int64_t initial_kcap_blocks(const sad_ctx *ctx) {
    return std::max<int64_t>(1, (8 * (int64_t)ctx->V + ctx->kcols_per_block - 1) / ctx->kcols_per_block);
}

// Reads the step statistics sad_build_profiles copied to pinned memory (errors, operand status,
// per-shard K and cap). wait: block until they have landed (a synchronizing call); else only if
// they already have, and only to learn sizes (start of the next step: errors of an unobserved
// step are dropped, the step's own validation reports them again).
static int absorb(sad_ctx *ctx, bool wait) {
    if (!ctx->stats_pending) return SAD_OK;
    if (wait) {
        CK(cudaEventSynchronize(ctx->ev_async));
    } else if (cudaEventQuery(ctx->ev_async) != cudaSuccess) {
        cudaGetLastError();          // cudaErrorNotReady is not an error
        return SAD_OK;
    }
    ctx->stats_pending = false;
    const int pl = ctx->pl;
    const unsigned long long *h = ctx->h_stats, *st = h + 4, *ki = h + 8;
    ctx->h_windows.assign(pl, 0);
    ctx->h_distinct.assign(pl, 0);
    ctx->h_K.assign(pl, 0);
    ctx->h_cap.assign(pl, kNoCap);
    int64_t macs = 0;
    for (int s = 0; s < pl; ++s) {
        const unsigned long long *k = ki + (size_t)s * kKinfo;
        ctx->h_windows[s] = (int64_t)k[0];
        ctx->h_distinct[s] = (int64_t)k[1];
        ctx->h_K[s] = ctx->use_tc ? (int64_t)k[20] : (int64_t)k[2];
        ctx->h_cap[s] = ctx->use_tc ? (uint32_t)k[21] : kNoCap;
        const int64_t w = ctx->shard_base[s + 1] - ctx->shard_base[s];
        macs += w * (w + 1) / 2 * ctx->h_K[s];
    }
    ctx->macs = macs;
    const bool overflow = ctx->use_tc && (st[0] & 1ull);
    if (ctx->use_tc) {
        const int64_t kb = std::max<int64_t>(1, ((int64_t)st[1] + ctx->kcols_per_block - 1) / ctx->kcols_per_block);
        ctx->kmax_blocks_seen = kb;
        // the next step's capacity: the largest K seen plus 1/8 (and one block) of headroom
        ctx->kcap_next = kb + std::max<int64_t>(1, kb / 8);
    }
    if (!wait) return SAD_OK;
    const unsigned long long NONE = ~0ull;
    if (h[0] != NONE) {
        ctx->err_idx = (int64_t)(h[0] >> 32);
        ctx->err_pos = (int64_t)(h[0] & 0xFFFFFFFFull);
        return fail(ctx, SAD_E_SYMBOL, "IllegalSymbol(sequence %lld, position %lld)", (long long)ctx->err_idx,
                    (long long)ctx->err_pos);
    }
    if (h[1] != NONE) {
        ctx->err_idx = (int64_t)h[1];
        return fail(ctx, SAD_E_TOO_SHORT, "SequenceTooShort(sequence %lld): L < k = %d", (long long)ctx->err_idx,
                    ctx->cfg.k);
    }
    if (h[2] != NONE) {
        ctx->err_idx = (int64_t)h[2];
        return fail(ctx, SAD_E_TOO_LONG, "sequence %lld: L - k + 1 > 65535", (long long)ctx->err_idx);
    }
    if (overflow) {
        ctx->kcap_blocks = std::max(ctx->kcap_blocks, ctx->kcap_next);
        ctx->stage = 1;
        return soft_fail(ctx, SAD_E_REPLAN, "all-pairs operand of %lld K blocks exceeded (needs %lld): rerun the step",
                         (long long)ctx->kcap_blocks, (long long)ctx->kmax_blocks_seen);
    }
    return SAD_OK;
}

// stage timing events (CUDA events on the context stream; inside a CUDA graph capture they become
// external event-record nodes that sad_graph_account reads after each replay)
static void record_pair(sad_ctx *ctx, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, bool begin, int gslot) {
    if (ctx->capturing) {
        cudaEventRecordWithFlags(ctx->gev[gslot], ctx->st, cudaEventRecordExternal);
        ctx->graph_events = true;
        return;
    }
    if (begin) {
        std::pair<cudaEvent_t, cudaEvent_t> e;
        if (!ctx->ev_free.empty()) {
            e = ctx->ev_free.back();
            ctx->ev_free.pop_back();
        } else {
            cudaEventCreate(&e.first);
            cudaEventCreate(&e.second);
        }
        cudaEventRecord(e.first, ctx->st);
        v.push_back(e);
    } else {
        cudaEventRecord(v.back().second, ctx->st);
    }
}

static bool stream_capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return cs == cudaStreamCaptureStatusActive;
}

// waits for an event while polling the communicator for asynchronous errors (a failed or aborted
// peer): the call then returns SAD_E_NCCL instead of blocking forever
static int wait_collective(sad_ctx *ctx, cudaEvent_t ev) {
    for (;;) {
        const cudaError_t e = cudaEventQuery(ev);
        if (e == cudaSuccess) return SAD_OK;
        if (e != cudaErrorNotReady) return fail(ctx, SAD_E_CUDA, "waiting for the exchange: %s", cudaGetErrorString(e));
        cudaGetLastError();
        if (ctx->comm) {
            ncclResult_t ae = ncclSuccess;
            ncclCommGetAsyncError(comm_of(ctx), &ae);
            if (ae != ncclSuccess && ae != ncclInProgress) {
                ncclCommAbort(comm_of(ctx));
                ctx->comm = nullptr;
                return fail(ctx, SAD_E_NCCL, "collective failed: %s (a peer failed or aborted)", ncclGetErrorString(ae));
            }
        }
        std::this_thread::yield();
    }
}

extern "C" {

static void bucket_sizes_from_counts(sad_ctx *ctx);

uint32_t sad_abi_version(void) { return SAD_ABI_VERSION; }

int sad_nccl_unique_id(uint8_t *out128) {
    if (!out128) return SAD_E_ARG;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return SAD_E_NCCL;
    std::memcpy(out128, &id, 128);
    return SAD_OK;
}

int sad_create(const sad_config *cfg, const uint8_t *nccl_id, sad_ctx **out) {
    if (!cfg || !out) return SAD_E_ARG;
    *out = nullptr;
    if (cfg->alphabet != SAD_PROTEIN20 && cfg->alphabet != SAD_DNA4) return SAD_E_ARG;
    if (cfg->k < 1 || cfg->p < 1 || cfg->p > 64 || cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world)
        return SAD_E_ARG;
    const bool split = (cfg->flags & SAD_F_TILE_SPLIT) != 0;
    if (split && ((cfg->flags & SAD_F_KERNEL_ALU) || (cfg->flags & SAD_F_KEEP_SIM))) return SAD_E_ARG;
    if (!split && cfg->p % cfg->world != 0) return SAD_E_ARG;
    if ((cfg->flags & SAD_F_RANK_SAMPLES) && cfg->p < 2) return SAD_E_ARG;   // f1 needs k = p-1 >= 1 samples
    const int A = cfg->alphabet == SAD_PROTEIN20 ? 20 : 4;
    int64_t V = 1;
    for (int i = 0; i < cfg->k; ++i) {
        V *= A;
        if (V > 65536) return SAD_E_ARG;
    }
    if ((cfg->flags & SAD_F_RANK_SAMPLES) && V * 8 > 200 * 1024) return SAD_E_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) {
        cudaGetLastError();
        return SAD_E_CUDA;
    }
    sad_ctx *ctx = new (std::nothrow) sad_ctx();
    if (!ctx) return SAD_E_OOM;
    ctx->cfg = *cfg;
    if (split) {
        // the data path is a world-1 path on the whole input; world / rank only split the all-pairs tiles
        ctx->tile_world = cfg->world;
        ctx->tile_rank = cfg->rank;
        ctx->tile_reduce = nccl_id != nullptr && cfg->world > 1;
        ctx->cfg.world = 1;
        ctx->cfg.rank = 0;
    }
    ctx->st = reinterpret_cast<cudaStream_t>(cfg->stream);
    ctx->A = A;
    ctx->V = (int)V;
    ctx->pl = ctx->cfg.p / ctx->cfg.world;
    ctx->shard0 = ctx->cfg.rank * ctx->pl;
    ctx->use_tc = !(cfg->flags & SAD_F_KERNEL_ALU);
    ctx->tc_kind = (cfg->flags & SAD_F_TC_INT8) ? 0 : 1;
    ctx->f1_tc = ctx->use_tc && ctx->tc_kind == 1 && (cfg->flags & SAD_F_RANK_SAMPLES) &&
                 !(cfg->flags & SAD_F_F1_CUDA_CORES);
    ctx->tc_cg = (cfg->flags & SAD_F_TC_1SM) ? 1 : 2;
    ctx->kcols_per_block = (ctx->use_tc && ctx->tc_kind == 1) ? 256 : 128;
    DeviceScope dev_scope_(cfg->device);
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cfg->device);
    bool ok = alloc_host(ctx) && cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->ev_stats, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->ev_async, cudaEventDisableTiming) == cudaSuccess;
    for (auto &e : ctx->ev_chunk) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    for (auto &e : ctx->gev) ok = ok && cudaEventCreate(&e) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        sad_destroy(ctx);
        return SAD_E_CUDA;
    }
    if (ctx->use_tc) {
        std::string why;
        if (!tc_supported(why)) {
            sad_destroy(ctx);
            return SAD_E_ARG;
        }
    }
    if (nccl_id) {                   // collective over the world ranks
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, 128);
        ncclComm_t comm = nullptr;
        if (ncclCommInitRank(&comm, cfg->world, id, cfg->rank) != ncclSuccess) {
            sad_destroy(ctx);
            return SAD_E_NCCL;
        }
        ctx->comm = comm;
    }
    *out = ctx;
    return SAD_OK;
}

void sad_destroy(sad_ctx *ctx) {
    if (!ctx) return;
    DeviceScope dev_scope_(ctx->cfg.device);
    if (ctx->st) cudaStreamSynchronize(ctx->st); else cudaDeviceSynchronize();
    if (ctx->comm) ncclCommDestroy(comm_of(ctx));
    for (auto &v : {&ctx->ev_pairs_ap, &ctx->ev_pairs_op, &ctx->ev_free})
        for (auto &e : *v) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
    }
    for (cudaEvent_t e : {ctx->ev_fork, ctx->ev_join, ctx->ev_stats, ctx->ev_async})
        if (e) cudaEventDestroy(e);
    for (auto &e : ctx->ev_chunk)
        if (e) cudaEventDestroy(e);
    for (auto &e : ctx->gev)
        if (e) cudaEventDestroy(e);
    for (void *h : {(void *)ctx->h_small, (void *)ctx->h_tiles, (void *)ctx->h_stats, (void *)ctx->h_cnt_all,
                    (void *)ctx->h_seg, (void *)ctx->h_runs})
        if (h) cudaFreeHost(h);
    cudaGetLastError();
    delete ctx;
}

int sad_abort(sad_ctx *ctx) {
    if (!ctx) return SAD_E_ARG;
    DeviceScope dev_scope_(ctx->cfg.device);
    if (ctx->comm) {
        ncclCommAbort(comm_of(ctx));
        ctx->comm = nullptr;
    }
    fail(ctx, SAD_E_NCCL, "aborted by sad_abort");
    return SAD_OK;
}

const char *sad_last_error(const sad_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int sad_error_location(const sad_ctx *ctx, int64_t *source_index, int64_t *position) {
    if (!ctx) return SAD_E_ARG;
    if (source_index) *source_index = ctx->err_idx;
    if (position) *position = ctx->err_pos;
    return SAD_OK;
}

int sad_workspace_size(const sad_ctx *cctx, int64_t n_local, int64_t residues_local, size_t *bytes) {
    sad_ctx *ctx = const_cast<sad_ctx *>(cctx);
    if (!ctx || !bytes || n_local < 0 || residues_local < 0) return SAD_E_ARG;
    sad_ctx tmp;
    tmp.cfg = ctx->cfg;
    tmp.pl = ctx->pl;
    tmp.V = ctx->V;
    tmp.comm = ctx->comm;
    *bytes = carve(&tmp, nullptr, n_local, residues_local);
    tmp.comm = nullptr;
    return SAD_OK;
}

static int profile_reset(sad_ctx *ctx);
static int profile_launch(sad_ctx *ctx, int64_t i0, int64_t i1);

int sad_load(sad_ctx *ctx, const uint8_t *ascii, const int64_t *offsets, int64_t n_local, int64_t first_source_index,
             int64_t n_global, int64_t residues_local, int32_t mem, void *d_ws, size_t ws_bytes) {
    GUARD(0);
    if (!offsets || !d_ws || n_local < 0 || n_global < 0 ||
        (mem != SAD_MEM_HOST && mem != SAD_MEM_DEVICE && mem != SAD_MEM_DEVICE_REBASE))
        return fail(ctx, SAD_E_ARG, "sad_load: bad arguments");
    if (n_global == 0) return fail(ctx, SAD_E_EMPTY, "EmptyInput: no sequences");
    if (n_global > 0x7FFFFFFF) return fail(ctx, SAD_E_ARG, "n_global >= 2^31 (the key reserves 31 index bits)");
    const int p = ctx->cfg.p;
    if (n_global / p < p) return fail(ctx, SAD_E_INSUFFICIENT, "InsufficientSequences: w = %lld < p = %d",
                                      (long long)(n_global / p), p);
    std::vector<int64_t> sb;
    shard_layout(ctx, n_global, sb);
    if (sb[ctx->pl] != n_local || first_index_of_rank(ctx, n_global) != first_source_index)
        return fail(ctx, SAD_E_ARG, "rank %d must load sequences %lld..%lld (got %lld from %lld)", ctx->cfg.rank,
                    (long long)first_index_of_rank(ctx, n_global),
                    (long long)(first_index_of_rank(ctx, n_global) + sb[ctx->pl]), (long long)n_local,
                    (long long)first_source_index);
    if (n_local == 0) return fail(ctx, SAD_E_EMPTY, "rank has no sequences");
    if (ctx->cfg.flags & SAD_F_RANK_SAMPLES) {
        // f1 keys (reading A27): (T' << ibits) + index with T' < m 2^32, m = p(p-1)
        auto bitlen = [](uint64_t v) { int b = 0; while (v) { ++b; v >>= 1; } return b; };
        ctx->tbits = 32 + bitlen((uint64_t)p * (p - 1));
        ctx->ibits = std::max(1, bitlen((uint64_t)(n_global - 1)));
        if (ctx->tbits + ctx->ibits > 64)
            return fail(ctx, SAD_E_ARG, "rank vs samples: p(p-1) 2^32 N >= 2^64 (the exact key needs %d bits)",
                        ctx->tbits + ctx->ibits);
    }
    if (n_global / p + 1 >= (int64_t(1) << 24)) return fail(ctx, SAD_E_ARG, "shards of 2^24 or more sequences");
    ctx->capturing = stream_capturing(ctx->st);
    int64_t R = residues_local;
    bool need_sync = mem == SAD_MEM_HOST;     // host inputs may be reused by the caller on return
    if (mem == SAD_MEM_HOST) {
        if (offsets[0] != 0) return fail(ctx, SAD_E_ARG, "offsets[0] != 0");
        if (R >= 0 && R != offsets[n_local]) return fail(ctx, SAD_E_ARG, "residues_local != offsets[n_local]");
        R = offsets[n_local];
    } else if (R < 0 && mem == SAD_MEM_DEVICE_REBASE) {
        return fail(ctx, SAD_E_ARG, "SAD_MEM_DEVICE_REBASE needs residues_local");
    } else if (R < 0) {
        if (ctx->capturing) return fail(ctx, SAD_E_ARG, "device inputs in a graph capture need residues_local");
        CK(cudaMemcpyAsync(ctx->h_small + 40000, offsets + n_local, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        R = (int64_t)ctx->h_small[40000];
    }
    if (ctx->capturing && mem == SAD_MEM_HOST) return fail(ctx, SAD_E_ARG, "host inputs cannot be graph-captured");
    if (R > 0 && !ascii) return fail(ctx, SAD_E_ARG, "ascii is NULL");
    const size_t need = carve(ctx, nullptr, n_local, R);
    if (ws_bytes < need) return fail(ctx, SAD_E_OOM, "workspace %zu < %zu bytes", ws_bytes, need);
    uint8_t *base = reinterpret_cast<uint8_t *>(rup(reinterpret_cast<int64_t>(d_ws), 256));
    if ((size_t)(base - reinterpret_cast<uint8_t *>(d_ws)) + need - 256 > ws_bytes)
        return fail(ctx, SAD_E_OOM, "workspace misaligned");
    ctx->ws = base;
    ctx->ws_bytes = ws_bytes;
    carve(ctx, base, n_local, R);
    ctx->n = n_local;
    ctx->n_global = n_global;
    ctx->first_idx = first_source_index;
    ctx->R = R;
    ctx->shard_base = sb;
    ctx->max_w = 0;
    ctx->shard_rowpad.assign(ctx->pl + 1, 0);
    int64_t pairs = 0;
    for (int s = 0; s < ctx->pl; ++s) {
        const int64_t w = sb[s + 1] - sb[s];
        ctx->max_w = std::max(ctx->max_w, w);
        ctx->shard_rowpad[s + 1] = ctx->shard_rowpad[s] + rup(w, kRowPad);
        pairs += w * (w - 1) / 2;
    }
    ctx->pairs = pairs;
    ctx->rows_pad = ctx->shard_rowpad[ctx->pl];
    const cudaMemcpyKind kind = mem == SAD_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    // host inputs of a few MB or more: the residues are copied in chunks on the internal stream and
    // each chunk's k-mer counts (K1/K2) start on ctx->st as soon as it has landed (below)
    const int nch = 4;                     // chunks of a pipelined host load (16 max; 4 measured best)
    const bool pipelined = mem == SAD_MEM_HOST && R >= (int64_t(4) << 20) && n_local >= 64 * nch;
    ctx->profiled = false;
    if (R > 0 && !pipelined) CK(cudaMemcpyAsync(ctx->d_ascii, ascii, (size_t)R, kind, ctx->st));
    if (mem == SAD_MEM_DEVICE_REBASE) {
        launch_rebase(offsets, n_local + 1, ctx->d_off, ctx->st);
        LAUNCHED();
    } else {
        CK(cudaMemcpyAsync(ctx->d_off, offsets, sizeof(int64_t) * (size_t)(n_local + 1), kind, ctx->st));
    }
    // small per-shard tables (uploaded only when the layout changes)
    // (the carve places the tables behind the R-sized residue buffer, so R is part of the key)
    const bool same = ctx->tbl_ws == base && ctx->tbl_n == n_local && ctx->tbl_ng == n_global &&
                      ctx->tbl_first == first_source_index && ctx->tbl_R == R;
    if (!same) {
        if (ctx->capturing) return fail(ctx, SAD_E_STATE, "a graph capture needs the layout loaded once before");
        int64_t *tbl = reinterpret_cast<int64_t *>(ctx->h_small + 32768);
        int64_t simb = 0, tiles = 0;
        for (int s = 0; s <= ctx->pl; ++s) {
            tbl[s] = sb[s];
            tbl[(ctx->pl + 1) + s] = ctx->shard_rowpad[s];
            tbl[2 * (ctx->pl + 1) + s] = simb;
            tbl[3 * (ctx->pl + 1) + s] = tiles;
            if (s < ctx->pl) {
                const int64_t w = sb[s + 1] - sb[s];
                simb += w * w;
                const int64_t nt = (w + 63) / 64;
                tiles += nt * (nt + 1) / 2;
            }
        }
        ctx->alu_tiles = tiles;
        // K6 dense excess matrices: per shard w x rup(w, 16) bytes
        ctx->h_ebase.assign(ctx->pl + 1, 0);
        for (int s = 0; s < ctx->pl; ++s) {
            const int64_t w = sb[s + 1] - sb[s];
            ctx->h_ebase[s + 1] = ctx->h_ebase[s] + w * rup(w, 16);
        }
        std::memcpy(tbl + 4 * (ctx->pl + 1), ctx->h_ebase.data(), sizeof(int64_t) * (ctx->pl + 1));
        if (ctx->use_tc) {           // the tensor-core tile table of this layout
            const size_t need_b = (size_t)ctx->tc_tiles_cap * 16;
            if (ctx->h_tiles_bytes < need_b) {
                if (ctx->h_tiles) cudaFreeHost(ctx->h_tiles);
                ctx->h_tiles = nullptr;
                ctx->h_tiles_bytes = 0;
                CK(cudaMallocHost(&ctx->h_tiles, need_b));
                ctx->h_tiles_bytes = need_b;
            }
            // tile split: the owned row blocks (of tile height), re-indexed per 128 padded operand rows
            // (shards are padded to 128 rows, so every 128-row block lies in one shard and one row block)
            std::vector<uint8_t> own_rb;
            if (ctx->tile_world > 1) own_rb.assign((size_t)(ctx->n / tc_row_block(ctx) + ctx->pl + 2), 0);
            ctx->tc_tiles_n = tc_build_tiles(ctx->pl, sb.data(), ctx->tc_kind, ctx->tc_cg, ctx->h_tiles,
                                             ctx->tc_tiles_cap, ctx->tile_world, ctx->tile_rank,
                                             own_rb.empty() ? nullptr : own_rb.data());
            if (!own_rb.empty()) {
                const int64_t nb128 = ctx->rows_pad / 128;
                if (nb128 > 16384 * 8) return fail(ctx, SAD_E_ARG, "tile split: too many row blocks");
                uint8_t *own = reinterpret_cast<uint8_t *>(ctx->h_small + 48000);   // staging, <= 128 KB
                int64_t rb0 = 0;
                for (int s = 0; s < ctx->pl; ++s) {
                    const int64_t w = sb[s + 1] - sb[s], bm = tc_row_block(ctx);
                    for (int64_t b = 0; b < (w + 127) / 128; ++b)
                        own[ctx->shard_rowpad[s] / 128 + b] = own_rb[(size_t)(rb0 + (128 * b) / bm)];
                    rb0 += (w + bm - 1) / bm;
                }
                CK(cudaMemcpyAsync(ctx->d_rb_own, own, (size_t)nb128, cudaMemcpyHostToDevice, ctx->st));
            }
            if (ctx->tc_tiles_n < 0) return fail(ctx, SAD_E_OOM, "tile table exceeds its bound");
            if (ctx->tc_tiles_n > 0)
                CK(cudaMemcpyAsync(ctx->d_tc_tiles, ctx->h_tiles, (size_t)ctx->tc_tiles_n * 16, cudaMemcpyHostToDevice,
                                   ctx->st));
        }
        const size_t tb = sizeof(int64_t) * (ctx->pl + 1);
        CK(cudaMemcpyAsync(ctx->d_shard_base, tbl, tb, cudaMemcpyHostToDevice, ctx->st));
        CK(cudaMemcpyAsync(ctx->d_shard_rowpad, tbl + (ctx->pl + 1), tb, cudaMemcpyHostToDevice, ctx->st));
        CK(cudaMemcpyAsync(ctx->d_sim_base, tbl + 2 * (ctx->pl + 1), tb, cudaMemcpyHostToDevice, ctx->st));
        CK(cudaMemcpyAsync(ctx->d_tile_base, tbl + 3 * (ctx->pl + 1), tb, cudaMemcpyHostToDevice, ctx->st));
        CK(cudaMemcpyAsync(ctx->d_ebase, tbl + 4 * (ctx->pl + 1), tb, cudaMemcpyHostToDevice, ctx->st));
        // the single-pass scan's epoch and tile status words start from zero in a fresh layout
        CK(cudaMemsetAsync(ctx->d_scan_state, 0, 16, ctx->st));
        CK(cudaMemsetAsync(ctx->d_scan_status, 0, sizeof(unsigned long long) * (size_t)(unpack_scan_tiles(n_local) + 1),
                           ctx->st));
        ctx->tbl_ws = base;
        ctx->tbl_n = n_local;
        ctx->tbl_ng = n_global;
        ctx->tbl_first = first_source_index;
        ctx->tbl_R = R;
        // capped layers + K6 excess are possible in this layout (the K6 row accumulators hold
        // max_w bytes per warp; the dense excess matrices must fit their bound)
        ctx->allow_cap = ctx->use_tc && !(ctx->cfg.flags & SAD_F_TC_ALL_LAYERS) && rup(ctx->max_w, 16) <= kXrSmem &&
                         ctx->h_ebase[ctx->pl] <= kMaxExcessBytes;
        // fresh layout: the operand capacity starts from the capped-layer bound
        ctx->kcap_blocks = ctx->kcap_next = initial_kcap_blocks(ctx);
        ctx->kmax_blocks_seen = -1;
        ctx->stats_pending = false;
        need_sync = true;
    }
    // K6 list entries: at most one per CSR entry (sum of the distinct counts <= windows <= R)
    ctx->x_entries_bound = std::max<int64_t>(R, 1);
    ctx->launches_step = 0;
    if (pipelined) {
        if (int rc = profile_reset(ctx)) return rc;
        // the previous step's readers of d_ascii (on ctx->st) finish before the first chunk lands
        CK(cudaEventRecord(ctx->ev_fork, ctx->st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        for (int c = 0; c < nch; ++c) {      // even chunks (a small last chunk measured slower)
            const int64_t i0 = n_local * c / nch, i1 = n_local * (c + 1) / nch;
            const int64_t b0 = offsets[i0], b1 = offsets[i1];
            if (b1 > b0)
                CK(cudaMemcpyAsync(ctx->d_ascii + b0, ascii + b0, (size_t)(b1 - b0), cudaMemcpyHostToDevice, ctx->side));
            CK(cudaEventRecord(ctx->ev_chunk[c], ctx->side));
            CK(cudaStreamWaitEvent(ctx->st, ctx->ev_chunk[c], 0));
            if (int rc = profile_launch(ctx, i0, i1)) return rc;
        }
        ctx->profiled = true;
    }
    if (need_sync) CK(cudaStreamSynchronize(ctx->st));
    ctx->stage = 1;
    return SAD_OK;
}

// K1/K2 accumulators cleared, on ctx->st
static int profile_reset(sad_ctx *ctx) {
    const int pl = ctx->pl, V = ctx->V;
    launch_profile_reset(ctx->d_M, (size_t)pl * V, ctx->d_Mb, (size_t)pl * ((V + 31) / 32), ctx->d_Xc,
                         (size_t)kNumCaps * pl * V, ctx->d_err, ctx->d_status, 4 + kKinfo * (size_t)pl,
                         ctx->use_tc ? ctx->d_lcnt : nullptr, (size_t)pl * kLenBinsMax, ctx->st);
    LAUNCHED();
    return SAD_OK;
}

// K1/K2 over sequences [i0, i1), on ctx->st
static int profile_launch(sad_ctx *ctx, int64_t i0, int64_t i1) {
    const int pl = ctx->pl, V = ctx->V;
    ProfileArgs a{};
    a.ascii = ctx->d_ascii;
    a.off = ctx->d_off;
    a.n = ctx->n;
    a.first_idx = ctx->first_idx;
    a.k = ctx->cfg.k;
    a.A = ctx->A;
    a.V = V;
    a.alphabet = ctx->cfg.alphabet;
    a.pl = pl;
    a.shard_base = ctx->d_shard_base;
    a.rowinfo = ctx->d_rowinfo;
    a.csr = ctx->d_csr;
    a.dcnt = ctx->d_dcnt;
    a.M = ctx->d_M;
    a.err = ctx->d_err;
    a.kinfo = ctx->d_kinfo;
    a.Xc = ctx->d_Xc;
    a.Mb = ctx->d_Mb;
    a.nhi = ctx->d_nhi;
    a.T = ctx->d_T;
    a.lcnt = ctx->use_tc ? ctx->d_lcnt : nullptr;
    a.i_begin = i0;
    a.i_end = i1;
    a.blk = ctx->R >= (int64_t)1024 * ctx->n;   // host-known (no read-back): long sequences, one block each
    launch_profile(a, ctx->st);
    LAUNCHED();
    return SAD_OK;
}

int sad_build_profiles(sad_ctx *ctx) {
    GUARD(1);
    const int pl = ctx->pl, V = ctx->V;
    ctx->capturing = stream_capturing(ctx->st);
    if (!ctx->capturing) {
        absorb(ctx, false);          // sizes learnt from the previous step, if it has finished
        ctx->kcap_blocks = ctx->kcap_next;
    }
    if (!ctx->profiled) {
        if (int rc = profile_reset(ctx)) return rc;
        if (int rc = profile_launch(ctx, 0, ctx->n)) return rc;
    }
    ctx->profiled = false;
    ctx->t_used = false;
    // K3 (statistics, the cap / K decision, column map, K6 list offsets, the length order's bin
    // offsets) in one launch, all on the device, then the length order's scatter (rows by L - k + 1)
    launch_shard_plan(ctx->d_M, ctx->d_Mb, ctx->d_Xc, ctx->d_kinfo, pl, V, ctx->allow_cap ? 1 : 0, ctx->kcap_blocks,
                      (int)ctx->kcols_per_block, ctx->d_cap, ctx->d_xsel, ctx->d_ident, ctx->d_kblocks, ctx->d_status,
                      ctx->d_col0, ctx->d_xoff, xtot_of(ctx), ctx->d_xcur, ctx->use_tc ? ctx->d_lcnt : nullptr,
                      ctx->d_lcnt + (size_t)pl * kLenBinsMax, ctx->d_shard_base, ctx->st);
    LAUNCHED();
    if (ctx->use_tc && ctx->tile_world > 1) {
        // tile split: every rank must hold the same rows in the same row blocks -- the length order by
        // a stable sort (ties by index) instead of the scatter's arbitrary order within a length
        launch_lenkeys(ctx->d_rowinfo, ctx->n, ctx->d_ckey, ctx->d_perm_in, ctx->st);
        LAUNCHED();
        int sbits = 0;
        while ((1 << sbits) < pl) ++sbits;
        if (!(ctx->max_w <= (int64_t)16384 &&
              seg_sort_pairs_runs(ctx->d_ckey, ctx->d_perm_in, ctx->d_shard_base, pl, ctx->max_w, ctx->n,
                                  ctx->d_ckey_sorted, ctx->d_perm_sorted, 16, ctx->st) == 0)) {
            // one stable device radix sort of (shard << 32 | Tw)
            CK(sort_pairs(ctx, ctx->d_ckey, ctx->d_ckey_sorted, ctx->d_perm_in, ctx->d_perm_sorted, (int)ctx->n,
                          32 + sbits));
        }
        LAUNCHED();
        launch_lenapply(ctx->d_perm_sorted, ctx->d_rowinfo, ctx->d_shard_base, ctx->n, ctx->d_sigma, ctx->d_sigma_inv,
                        ctx->d_rinfo_s, ctx->st);
        LAUNCHED();
    } else if (ctx->use_tc) {     // the length order's slot scatter (histogram: K1/K2, bin offsets: K3)
        if (ctx->allow_cap) {     // fused with the K6 list fill in sad_rank (or alone there if no shard is capped)
            ctx->lenorder_deferred = true;
        } else {
            launch_lenorder(ctx->d_rowinfo, ctx->d_shard_base, pl, ctx->n, ctx->d_lcnt + (size_t)pl * kLenBinsMax,
                            ctx->d_sigma, ctx->d_sigma_inv, ctx->d_rinfo_s, ctx->st);
            LAUNCHED();
        }
    }
    // the statistics go to pinned host memory; read at the step's first synchronizing call
    CK(cudaMemcpyAsync(ctx->h_stats, ctx->d_err, sizeof(unsigned long long) * (8 + (size_t)pl * kKinfo),
                       cudaMemcpyDeviceToHost, ctx->st));
    if (!ctx->capturing) {
        CK(cudaEventRecord(ctx->ev_async, ctx->st));
        ctx->stats_pending = true;
    }
    // operand row: the capacity in 128-byte K blocks (128 int8 or 256 packed fp4 entries each)
    ctx->K_stride = ctx->kcap_blocks * 128;
    ctx->V_pad = rup(V, 64);
    ctx->stage = 2;
    return SAD_OK;
}

// the operand buffer: [indicator | counts operand][K6 lists L_tau u32][K6 dense excess E u8 + 256 zero bytes]
// [f1 on the tensor cores: the samples' operand rows | e_ij | the samples' counts transposed]
static void operand_parts(const sad_ctx *ctx, size_t &op, size_t &xl, size_t &xe, size_t &f1b) {
    op = ctx->use_tc ? (size_t)ctx->rows_pad * (size_t)ctx->K_stride : (size_t)ctx->rows_pad * (size_t)ctx->V_pad * 2;
    op = (size_t)rup((int64_t)op, 1024);
    xl = xe = f1b = 0;
    if (ctx->use_tc && ctx->allow_cap) {
        xl = (size_t)rup(ctx->x_entries_bound * 4, 1024);
        xe = (size_t)rup(ctx->h_ebase[ctx->pl] + 256, 1024);
    }
    if (ctx->f1_tc) {
        const int64_t mr = f1_tc_rows(ctx->cfg.p * (ctx->cfg.p - 1));
        f1b = (size_t)rup((int64_t)ctx->pl * mr * ctx->K_stride, 1024) + (size_t)rup(ctx->rows_pad * mr, 1024) +
              (size_t)rup((int64_t)ctx->V * mr * 2, 1024);
    }
}

int sad_operand_size(const sad_ctx *cctx, size_t *bytes) {
    sad_ctx *ctx = const_cast<sad_ctx *>(cctx);
    GUARD(2);
    if (!bytes) return SAD_E_ARG;
    size_t op = 0, xl = 0, xe = 0, f1b = 0;
    operand_parts(ctx, op, xl, xe, f1b);
    *bytes = op + xl + xe + f1b;
    return SAD_OK;
}

int32_t sad_key_index_bits(const sad_ctx *ctx) { return ctx ? ctx->ibits : SAD_E_ARG; }

int32_t sad_exchange_records(const sad_ctx *ctx) {
    if (!ctx) return SAD_E_ARG;
    return exchange_records(ctx);
}

size_t sad_ancestor_record_bytes(const sad_ctx *ctx) { return ctx ? record_bytes(ctx) : 0; }

// a3 + a4 (and the f1 sample records): operand, all-pairs, local ancestors; no host decisions
static int rank_local_impl(sad_ctx *ctx, void *d_operand, size_t operand_bytes, void *d_anc_out) {
    size_t need = 0;
    sad_operand_size(ctx, &need);
    if (!d_operand || operand_bytes < need || !d_anc_out)
        return fail(ctx, SAD_E_CAPACITY, "operand %zu < %zu bytes or NULL output", operand_bytes, need);
    if ((reinterpret_cast<uintptr_t>(d_operand) & 1023) != 0)
        return fail(ctx, SAD_E_ARG, "operand must be 1024-byte aligned");
    ctx->d_operand = d_operand;
    const int pl = ctx->pl;
    // K1/K2 zeroed T; a second all-pairs pass over the same profiles starts from zero again
    if (ctx->t_used) CK(cudaMemsetAsync(ctx->d_T, 0, sizeof(unsigned long long) * (size_t)ctx->n, ctx->st));
    ctx->t_used = true;
    if (ctx->d_sim) CK(cudaMemsetAsync(ctx->d_sim, 0, sizeof(uint16_t) * (size_t)ctx->sim_elems, ctx->st));

    OperandArgs o{};
    o.csr = ctx->d_csr;
    o.off = ctx->d_off;
    o.dcnt = ctx->d_dcnt;
    o.col0 = ctx->d_col0;
    o.shard_base = ctx->d_shard_base;
    o.shard_rowpad = ctx->d_shard_rowpad;
    o.rows_pad = ctx->rows_pad;
    o.stride = ctx->use_tc ? ctx->K_stride : ctx->V_pad * 2;
    o.k = ctx->cfg.k;
    o.V = ctx->V;
    o.pl = pl;
    o.fp4 = ctx->use_tc && ctx->tc_kind == 1;
    o.op = d_operand;
    o.wide = ctx->R >= (int64_t)1024 * ctx->n;   // host-known (no read-back): long rows, one block per row
    size_t op_b = 0, xl_b = 0, xe_b = 0, f1_b = 0;
    operand_parts(ctx, op_b, xl_b, xe_b, f1_b);
    uint32_t *lists = xl_b ? reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(d_operand) + op_b) : nullptr;
    uint8_t *E = xl_b ? reinterpret_cast<uint8_t *>(d_operand) + op_b + xl_b : nullptr;
    unsigned long long *xtot = xtot_of(ctx);
    record_pair(ctx, ctx->ev_pairs_op, true, 0);
    uint32_t *lpos = nullptr;     // the deferred length order (fused into k_xfill when it runs)
    if (ctx->lenorder_deferred) {
        ctx->lenorder_deferred = false;
        lpos = ctx->d_lcnt + (size_t)pl * kLenBinsMax;
        if (!lists) {
            launch_lenorder(ctx->d_rowinfo, ctx->d_shard_base, pl, ctx->n, lpos, ctx->d_sigma, ctx->d_sigma_inv,
                            ctx->d_rinfo_s, ctx->st);
            LAUNCHED();
            lpos = nullptr;
        }
    }
    if (ctx->use_tc) {
        // K3 ran in sad_build_profiles (layer caps, column maps, K6 list offsets); the K6 lists,
        // then K6 rows on the side stream beside K4
        o.sigma = ctx->d_sigma;
        o.sigma_inv = ctx->d_sigma_inv;
        o.rowinfo = ctx->d_rowinfo;
        o.n = ctx->n;
        o.kblocks = ctx->d_kblocks;
        o.cap = ctx->d_cap;
        o.ident = ctx->d_ident;
        if (lists) {
            ExcessArgs x{};
            x.zero_seg = E + ctx->h_ebase[pl];   // the zero row segment (cleared by k_xfill)
            x.csr = ctx->d_csr;
            x.off = ctx->d_off;
            x.nhi = ctx->d_nhi;
            x.shard_base = ctx->d_shard_base;
            x.n = ctx->n;
            x.pl = pl;
            x.V = ctx->V;
            x.k = ctx->cfg.k;
            x.cap = ctx->d_cap;
            x.xoff = ctx->d_xoff;
            x.xtot = xtot;
            x.lists = lists;
            x.accb = (int)rup(ctx->max_w, 16);
            x.xrow = ctx->d_xrow;
            x.E = E;
            x.ebase = ctx->d_ebase;
            x.sigma = ctx->d_sigma;
            x.sigma_inv = ctx->d_sigma_inv;
            x.rowinfo = ctx->d_rowinfo;
            x.rb_own = ctx->tile_world > 1 ? ctx->d_rb_own : nullptr;
            x.shard_rowpad = ctx->d_shard_rowpad;
            x.rb_rows = 128;
            launch_xfill(x, ctx->d_xcur, lpos, ctx->d_sigma, ctx->d_sigma_inv, ctx->d_rinfo_s, ctx->st);
            LAUNCHED();
            // K6 rows on the side stream, concurrently with K4 (both only read the CSR / lists)
            CK(cudaEventRecord(ctx->ev_fork, ctx->st));
            CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            if (launch_excess(x, ctx->side)) return fail(ctx, SAD_E_ARG, "K6: shard too wide for the row accumulators");
            LAUNCHED();
            CK(cudaEventRecord(ctx->ev_join, ctx->side));
        }
        launch_indicator(o, ctx->st);
        LAUNCHED();
        if (lists) CK(cudaStreamWaitEvent(ctx->st, ctx->ev_join, 0));
    } else {
        launch_dense_counts(o, ctx->st);
        LAUNCHED();
    }
    record_pair(ctx, ctx->ev_pairs_op, false, 1);

    AllPairsArgs ap{};
    ap.op = d_operand;
    ap.stride = o.stride;
    ap.rowinfo = ctx->use_tc ? ctx->d_rinfo_s : ctx->d_rowinfo;   // TC: length order
    ap.shard_base = ctx->d_shard_base;
    ap.shard_rowpad = ctx->d_shard_rowpad;
    ap.shard_kblocks = ctx->d_kblocks;
    ap.pl = pl;
    ap.max_w = ctx->max_w;
    ap.T = ctx->d_T;
    ap.sim = ctx->d_sim;
    ap.sim_base = ctx->d_sim_base;
    ap.vwords = (int)(ctx->V_pad / 2);
    ap.num_sms = ctx->num_sms;
    ap.tile_base = ctx->d_tile_base;
    ap.n_tiles = ctx->alu_tiles;
    ap.h_shard_base = ctx->shard_base.data();
    ap.h_shard_rowpad = ctx->shard_rowpad.data();
    ap.kblocks_hint = ctx->kmax_blocks_seen;
    ap.kind = ctx->tc_kind;
    ap.tiles = ctx->d_tc_tiles;
    ap.n_tiles_tc = ctx->tc_tiles_n;
    ap.cg = ctx->tc_cg;
    ap.xrow = lists ? ctx->d_xrow : nullptr;
    ap.E = E;
    ap.ebase = ctx->d_ebase;
    ap.zero = E ? E + ctx->h_ebase[pl] : nullptr;
    record_pair(ctx, ctx->ev_pairs_ap, true, 2);
    if (ctx->use_tc) {
        std::string e;
        const int rc = launch_allpairs_tc(ap, ctx->st, e);
        if (rc) return fail(ctx, SAD_E_CUDA, "tensor-core all-pairs: %s", e.c_str());
    } else {
        launch_allpairs_alu(ap, ctx->st);
    }
    LAUNCHED();
    if (ctx->tile_reduce)        // tile split: T_i = the sum of every rank's tiles (integer sums, exact)
        NK(ncclAllReduce(ctx->d_T, ctx->d_T, (size_t)ctx->n, ncclUint64, ncclSum, comm_of(ctx), ctx->st));
    record_pair(ctx, ctx->ev_pairs_ap, false, 3);
    if (!ctx->capturing) ctx->calls += 1;

    AncArgs an{};
    an.T = ctx->d_T;
    an.shard_base = ctx->d_shard_base;
    an.csr = ctx->d_csr;
    an.off = ctx->d_off;
    an.dcnt = ctx->d_dcnt;
    an.rowinfo = ctx->d_rowinfo;
    an.first_idx = ctx->first_idx;
    an.k = ctx->cfg.k;
    an.V = ctx->V;
    an.pl = pl;
    an.rec_bytes = record_bytes(ctx);
    an.anc_local = ctx->d_anc_local;
    const bool f1 = ctx->cfg.flags & SAD_F_RANK_SAMPLES;
    an.rec_out = f1 ? nullptr : reinterpret_cast<uint8_t *>(d_anc_out);
    launch_local_ancestors(an, ctx->st);
    LAUNCHED();
    if (f1) {
        // f1: local order by T, the k = p-1 rank samples of every shard -> records
        launch_tkeys(ctx->d_T, ctx->d_rowinfo, ctx->n, ctx->d_ckey, ctx->d_perm_in, ctx->st);
        LAUNCHED();
        int sbits = 0;
        while ((1 << sbits) < pl) ++sbits;
        // within a shard T <= w 2^32: the segmented run sort on those bits (64-bit block keys), else
        // one device radix sort of (shard, T)
        int tb = 32;
        while (tb < 56 && (int64_t(1) << (tb - 32)) <= ctx->max_w) ++tb;
        if (!(ctx->max_w <= (int64_t)16384 &&
              seg_sort_pairs_runs(ctx->d_ckey, ctx->d_perm_in, ctx->d_shard_base, ctx->pl, ctx->max_w, ctx->n,
                                  ctx->d_ckey_sorted, ctx->d_perm_sorted, tb, ctx->st) == 0))
            CK(sort_pairs(ctx, ctx->d_ckey, ctx->d_ckey_sorted, ctx->d_perm_in, ctx->d_perm_sorted, (int)ctx->n,
                          56 + sbits));
        LAUNCHED();
        launch_sample_records(ctx->d_perm_sorted, ctx->d_shard_base, pl, ctx->cfg.p, ctx->d_csr, ctx->d_off,
                              ctx->d_dcnt, ctx->d_rowinfo, ctx->first_idx, ctx->cfg.k, an.rec_bytes,
                              reinterpret_cast<uint8_t *>(d_anc_out), ctx->st);
        LAUNCHED();
    }
    ctx->stage = 3;
    return SAD_OK;
}

int sad_rank_local(sad_ctx *ctx, void *d_operand, size_t operand_bytes, void *d_anc_out) {
    GUARD(2);
    // split API: the caller reads no step results before moving the exchange buffers, so the
    // statistics are checked here (one wait) rather than at a later synchronizing call
    if (int rc = absorb(ctx, true)) return rc;
    return rank_local_impl(ctx, d_operand, operand_bytes, d_anc_out);
}

// a5-a8: GA, rank vs GA (or f1: vs the samples), local sort, regular samples
static int rank_global_impl(sad_ctx *ctx, const void *d_anc_all, uint64_t *d_samples_out) {
    const int p = ctx->cfg.p;
    if (!d_anc_all || (p > 1 && !d_samples_out)) return fail(ctx, SAD_E_ARG, "sad_rank_global: NULL buffer");
    RankArgs r{};
    r.anc_all = reinterpret_cast<const uint8_t *>(d_anc_all);
    r.rec_bytes = record_bytes(ctx);
    r.p = p;
    r.k = ctx->cfg.k;
    r.V = ctx->V;
    r.Sab = ctx->d_Sab;
    r.ga_info = ctx->d_ga_info;
    r.csr = ctx->d_csr;
    r.off = ctx->d_off;
    r.dcnt = ctx->d_dcnt;
    r.rowinfo = ctx->d_rowinfo;
    r.n = ctx->n;
    r.first_idx = ctx->first_idx;
    r.S_ga = ctx->d_S_ga;
    r.den_ga = ctx->d_den_ga;
    r.key = ctx->d_key;
    r.perm_in = ctx->d_perm_in;
    // a7: one stable radix sort of (shard, q) with the row as value: 32 (GA) or 33 (f1) + shard bits
    int sbits = 0;
    while ((1 << sbits) < ctx->pl) ++sbits;
    r.ckey = ctx->d_ckey;
    const bool f1 = ctx->cfg.flags & SAD_F_RANK_SAMPLES;
    const int qbits = ctx->tbits;
    if (!f1) {
        launch_ga_pairs(r, ctx->st);
        LAUNCHED();
        launch_rank_vs_ga(r, ctx->st);
        LAUNCHED();
    } else {
        // f1 (reading A27): T'_i = sum of q(x_i, s) over the m = p(p-1) gathered
        // samples, ordered exactly, and the keys (d_key doubles as the T' accumulator)
        const int m = p * (p - 1);
        CK(cudaMemsetAsync(ctx->d_key, 0, sizeof(unsigned long long) * (size_t)ctx->n, ctx->st));
        if (ctx->f1_tc) {
            // the w x m contraction on the tensor cores against the all-pairs operand of this step
            size_t op_b = 0, xl_b = 0, xe_b = 0, f1_b = 0;
            operand_parts(ctx, op_b, xl_b, xe_b, f1_b);
            const int64_t mr = f1_tc_rows(m);
            uint8_t *f1base = reinterpret_cast<uint8_t *>(ctx->d_operand) + op_b + xl_b + xe_b;
            F1Args fa{};
            fa.rec = r.anc_all;
            fa.rec_bytes = r.rec_bytes;
            fa.m = m;
            fa.V = ctx->V;
            fa.k = ctx->cfg.k;
            fa.pl = ctx->pl;
            fa.num_sms = ctx->num_sms;
            fa.n = ctx->n;
            fa.rows_pad = ctx->rows_pad;
            fa.stride = ctx->K_stride;
            fa.op = ctx->d_operand;
            fa.shard_base = ctx->d_shard_base;
            fa.shard_rowpad = ctx->d_shard_rowpad;
            fa.kblocks = ctx->d_kblocks;
            fa.M = ctx->d_M;
            fa.col0 = ctx->d_col0;
            fa.cap = ctx->d_cap;
            fa.ident = ctx->d_ident;
            fa.sigma = ctx->d_sigma;
            fa.nhi = ctx->d_nhi;
            fa.csr = ctx->d_csr;
            fa.off = ctx->d_off;
            fa.rinfo_s = ctx->d_rinfo_s;
            fa.bop = f1base;
            fa.ex = f1base + rup((int64_t)ctx->pl * mr * ctx->K_stride, 1024);
            fa.cT = reinterpret_cast<uint16_t *>(fa.ex + rup(ctx->rows_pad * mr, 1024));
            fa.Tp = ctx->d_key;
            std::string e;
            if (launch_f1_tc(fa, ctx->st, e)) return fail(ctx, SAD_E_CUDA, "f1 on the tensor cores: %s", e.c_str());
            ctx->launches_step += 4;
        } else {
            if (launch_rank_vs_samples(r, m, ctx->d_key, ctx->num_sms, ctx->st))
                return fail(ctx, SAD_E_ARG, "rank vs samples: V too large");
            LAUNCHED();
        }
        launch_f1_keys(ctx->d_key, ctx->n, ctx->tbits, ctx->ibits, ctx->first_idx, ctx->d_rowinfo, ctx->d_key,
                       ctx->d_ckey, ctx->d_perm_in, ctx->d_S_ga, ctx->d_den_ga, ctx->st);
        LAUNCHED();
        launch_f1_gainfo(ctx->d_anc_local, ctx->pl, ctx->shard0, p, ctx->first_idx, ctx->d_ga_info, ctx->st);
        LAUNCHED();
    }
    // the local rank sort: runs of <= 2048 keys per block, merged by ranking in shared memory
    if (!(ctx->max_w <= (int64_t)16384 &&
          seg_sort_pairs_runs(ctx->d_ckey, ctx->d_perm_in, ctx->d_shard_base, ctx->pl, ctx->max_w, ctx->n,
                              ctx->d_ckey_sorted, ctx->d_perm_sorted, qbits, ctx->st) == 0))
        CK(sort_pairs(ctx, ctx->d_ckey, ctx->d_ckey_sorted, ctx->d_perm_in, ctx->d_perm_sorted, (int)ctx->n,
                      qbits + sbits));
    LAUNCHED();
    // the real keys, and the exclusive prefix of L in sorted order (the residue offsets of every
    // bucket slice, K12/K13/K14) in the same single-pass launch
    launch_unpack_scan(ctx->d_ckey_sorted, ctx->d_perm_sorted, ctx->n, ctx->first_idx, ctx->d_key_sorted,
                       ctx->d_rowinfo, ctx->cfg.k, ctx->d_len_sorted, qbits, ctx->ibits, ctx->d_lpre,
                       ctx->d_scan_state, ctx->d_scan_status, ctx->st);
    LAUNCHED();
    if (p > 1) {
        launch_samples(ctx->d_key_sorted, ctx->d_shard_base, ctx->pl, p,
                       reinterpret_cast<unsigned long long *>(d_samples_out), ctx->st);
        LAUNCHED();
    }
    ctx->stage = 4;
    return SAD_OK;
}

int sad_rank_global(sad_ctx *ctx, const void *d_anc_all, uint64_t *d_samples_out) {
    GUARD(3);
    return rank_global_impl(ctx, d_anc_all, d_samples_out);
}

int sad_rank(sad_ctx *ctx, void *d_operand, size_t operand_bytes) {
    GUARD(2);
    if (ctx->cfg.world > 1 && !ctx->comm)
        return fail(ctx, SAD_E_STATE, "sad_rank with world > 1 needs a communicator (sad_create with an NCCL id)");
    ctx->capturing = stream_capturing(ctx->st);
    if (int rc = rank_local_impl(ctx, d_operand, operand_bytes, ctx->d_anc_mine)) return rc;
    // "Send the k samples from each processor to all the processors": the ancestor records
    const void *anc_all = ctx->d_anc_mine;
    if (coll_exchange(ctx)) {
        const size_t bytes = (size_t)exchange_records(ctx) * record_bytes(ctx);
        NK(ncclAllGather(ctx->d_anc_mine, ctx->d_anc_all, bytes, ncclUint8, comm_of(ctx), ctx->st));
        anc_all = ctx->d_anc_all;
    }
    return rank_global_impl(ctx, anc_all, reinterpret_cast<uint64_t *>(ctx->d_smp_mine));
}

// a9 + a10: pivots and bucket ranges
static int plan_impl(sad_ctx *ctx, const uint64_t *d_samples_all, int64_t *d_counts_out) {
    const int p = ctx->cfg.p;
    if ((p > 1 && !d_samples_all) || !d_counts_out) return fail(ctx, SAD_E_ARG, "sad_partition_plan: NULL buffer");
    PlanArgs a{};
    a.samples_all = reinterpret_cast<const unsigned long long *>(d_samples_all);
    a.p = p;
    a.pl = ctx->pl;
    a.key_sorted = ctx->d_key_sorted;
    a.perm_sorted = ctx->d_perm_sorted;
    a.shard_base = ctx->d_shard_base;
    a.rowinfo = ctx->d_rowinfo;
    a.k = ctx->cfg.k;
    a.pivots = ctx->d_pivots;
    a.bnd = ctx->d_bnd;
    a.lpre = ctx->d_lpre;
    a.counts = d_counts_out;
    launch_plan(a, ctx->st);
    LAUNCHED();
    if (d_counts_out != ctx->d_counts)
        CK(cudaMemcpyAsync(ctx->d_counts, d_counts_out, sizeof(int64_t) * (size_t)ctx->pl * p * 2,
                           cudaMemcpyDeviceToDevice, ctx->st));
    ctx->stage = 5;
    return SAD_OK;
}

int sad_partition_plan(sad_ctx *ctx, const uint64_t *d_samples_all, int64_t *d_counts_out) {
    GUARD(4);
    return plan_impl(ctx, d_samples_all, d_counts_out);
}

int sad_exchange_sizes(int32_t p, int32_t world, int32_t rank, const int64_t *h_counts_all, int64_t *h_send_seqs,
                       int64_t *h_send_res, int64_t *h_recv_seqs, int64_t *h_recv_res) {
    if (!h_counts_all || p < 1 || world < 1 || p % world || rank < 0 || rank >= world) return SAD_E_ARG;
    const int bpr = p / world, me0 = rank * bpr;
    for (int r = 0; r < world; ++r) {
        int64_t ss = 0, sr = 0, rs = 0, rr = 0;
        for (int s = me0; s < me0 + bpr; ++s)                       // my shards -> r's buckets
            for (int b = r * bpr; b < (r + 1) * bpr; ++b) {
                ss += h_counts_all[((size_t)s * p + b) * 2 + 0];
                sr += h_counts_all[((size_t)s * p + b) * 2 + 1];
            }
        for (int s = r * bpr; s < (r + 1) * bpr; ++s)               // r's shards -> my buckets
            for (int b = me0; b < me0 + bpr; ++b) {
                rs += h_counts_all[((size_t)s * p + b) * 2 + 0];
                rr += h_counts_all[((size_t)s * p + b) * 2 + 1];
            }
        if (h_send_seqs) h_send_seqs[r] = ss;
        if (h_send_res) h_send_res[r] = sr;
        if (h_recv_seqs) h_recv_seqs[r] = rs;
        if (h_recv_res) h_recv_res[r] = rr;
    }
    return SAD_OK;
}

int sad_pack_plan(int32_t p, int32_t world, int32_t rank, const int64_t *h_counts_all, int64_t *h_seg) {
    if (!h_counts_all || !h_seg || p < 1 || world < 1 || p % world || rank < 0 || rank >= world) return SAD_E_ARG;
    const int bpr = p / world, me0 = rank * bpr;
    int64_t cs = 0, cr = 0;
    for (int r = 0; r < world; ++r)
        for (int s = 0; s < bpr; ++s)
            for (int b = r * bpr; b < (r + 1) * bpr; ++b) {
                const size_t gi = ((size_t)(me0 + s) * p + b) * 2;
                h_seg[((size_t)s * p + b) * 2 + 0] = cs;
                h_seg[((size_t)s * p + b) * 2 + 1] = cr;
                cs += h_counts_all[gi + 0];
                cr += h_counts_all[gi + 1];
            }
    return SAD_OK;
}

// K13: this rank's sequences grouped by destination rank; seg = the pack plan (pinned host, valid
// until the copy has run)
static int pack_impl(sad_ctx *ctx, const int64_t *h_seg_pinned, uint64_t *d_send_meta, uint8_t *d_send_res) {
    const int p = ctx->cfg.p;
    CK(cudaMemcpyAsync(ctx->d_seg, h_seg_pinned, sizeof(int64_t) * (size_t)ctx->pl * p * 2, cudaMemcpyHostToDevice,
                       ctx->st));
    PackArgs a{};
    a.key_sorted = ctx->d_key_sorted;
    a.perm_sorted = ctx->d_perm_sorted;
    a.shard_base = ctx->d_shard_base;
    a.bnd = ctx->d_bnd;
    a.lpre = ctx->d_lpre;
    a.seg = ctx->d_seg;
    a.rowinfo = ctx->d_rowinfo;
    a.ascii = ctx->d_ascii;
    a.off = ctx->d_off;
    a.p = p;
    a.pl = ctx->pl;
    a.k = ctx->cfg.k;
    a.n = ctx->n;
    a.send_meta = reinterpret_cast<unsigned long long *>(d_send_meta);
    a.send_res = d_send_res;
    launch_pack(a, ctx->st);
    LAUNCHED();
    return SAD_OK;
}

int sad_pack(sad_ctx *ctx, const int64_t *h_counts_all, uint64_t *d_send_meta, uint8_t *d_send_res) {
    GUARD(5);
    if (!h_counts_all || !d_send_meta || !d_send_res) return fail(ctx, SAD_E_ARG, "sad_pack: NULL buffer");
    const int p = ctx->cfg.p;
    int64_t *seg = reinterpret_cast<int64_t *>(ctx->h_small + 2048);
    sad_pack_plan(p, ctx->cfg.world, ctx->cfg.rank, h_counts_all, seg);
    if (int rc = pack_impl(ctx, seg, d_send_meta, d_send_res)) return rc;
    // split API: the pinned staging of the plan is reused by the next call
    CK(cudaStreamSynchronize(ctx->st));
    return SAD_OK;
}

int sad_output_size(const sad_ctx *cctx, const int64_t *h_counts_all, size_t *bytes) {
    sad_ctx *ctx = const_cast<sad_ctx *>(cctx);
    GUARD(5);
    if ((!h_counts_all && ctx->cfg.world != 1) || !bytes) return SAD_E_ARG;
    int64_t n_out, r_out;
    sum_recv(ctx, h_counts_all, n_out, r_out);
    *bytes = out_layout(nullptr, n_out, r_out, false).total;
    return SAD_OK;
}

int sad_output_bound(const sad_ctx *cctx, int64_t residues_global, size_t *bytes) {
    sad_ctx *ctx = const_cast<sad_ctx *>(cctx);
    GUARD(1);
    if (!bytes) return SAD_E_ARG;
    const int p = ctx->cfg.p;
    if (ctx->cfg.world == 1) {
        *bytes = out_layout(nullptr, ctx->n, ctx->R, coll_exchange(ctx)).total;
        return SAD_OK;
    }
    if (residues_global < ctx->R) return fail(ctx, SAD_E_ARG, "residues_global < this rank's residues");
    const int64_t w = (ctx->n_global + p - 1) / p;
    const int64_t n_b = std::min<int64_t>(ctx->n_global, (int64_t)ctx->pl * (2 * w + p));   // reading A23
    *bytes = out_layout(nullptr, n_b, residues_global, true).total;
    return SAD_OK;
}

int sad_output_layout(const sad_ctx *cctx, const int64_t *h_counts_all, int64_t *h_layout) {
    sad_ctx *ctx = const_cast<sad_ctx *>(cctx);
    GUARD(5);
    if (!h_layout) return SAD_E_ARG;
    int64_t n_out, r_out;
    bool recv = false;
    if (h_counts_all) {
        sum_recv(ctx, h_counts_all, n_out, r_out);
    } else if (ctx->stage >= 6) {    // the last finished partition
        n_out = ctx->out_n;
        r_out = ctx->out_r;
        recv = ctx->out_recv_layout;
    } else if (ctx->cfg.world == 1) {
        sum_recv(ctx, nullptr, n_out, r_out);
    } else {
        return SAD_E_ARG;
    }
    OutLayout o = out_layout(nullptr, n_out, r_out, recv);
    h_layout[0] = n_out;
    h_layout[1] = r_out;
    h_layout[2] = (int64_t)reinterpret_cast<uintptr_t>(o.key);
    h_layout[3] = (int64_t)reinterpret_cast<uintptr_t>(o.off);
    h_layout[4] = (int64_t)reinterpret_cast<uintptr_t>(o.res);
    h_layout[5] = (int64_t)o.total;
    return SAD_OK;
}

// K14 receive side: merge the runs (this rank's own sorted shards for a local finish, or the
// received runs in source-shard order) into the owned buckets, each in key order
static int finish_impl(sad_ctx *ctx, const int64_t *h_counts_all, const uint64_t *d_recv_meta,
                       const uint8_t *d_recv_res, void *d_out, size_t out_bytes, bool recv_layout) {
    const int p = ctx->cfg.p;
    if ((reinterpret_cast<uintptr_t>(d_out) & 255) != 0) return fail(ctx, SAD_E_ARG, "output must be 256-byte aligned");
    const bool local = d_recv_meta == nullptr;
    int64_t n_out, r_out;
    sum_recv(ctx, h_counts_all, n_out, r_out);
    if (local && h_counts_all && (n_out != ctx->n || r_out != ctx->R))
        return fail(ctx, SAD_E_STATE, "counts do not cover the input");
    OutLayout o = out_layout(reinterpret_cast<uint8_t *>(d_out), n_out, r_out, recv_layout);
    if (out_bytes < o.total) return fail(ctx, SAD_E_CAPACITY, "output %zu < %zu bytes", out_bytes, o.total);
    const int nn = (int)n_out;
    // K14: merge the sorted runs by ranking (every owned bucket is a key range, so the merged
    // order is the bucket order and each bucket is in key order), then move the residues
    MergeArgs m{};
    m.n = n_out;
    m.k = ctx->cfg.k;
    m.out_key = o.key;
    m.out_len = o.len_in;
    m.out_src = o.perm;
    const int64_t *src_off;
    const int32_t *src_perm;
    const uint8_t *src_res;
    if (local) {                          // runs = this rank's sorted shards
        m.keys = ctx->d_key_sorted;
        m.kstride = 1;
        m.run_start = ctx->d_shard_base;
        m.nr = ctx->pl;
        m.perm = ctx->d_perm_sorted;
        m.rowinfo = ctx->d_rowinfo;
        m.cpre = ctx->d_lpre;                     // exclusive prefix of L in sorted order (rank_global)
        src_off = ctx->d_off;
        src_perm = ctx->d_perm_sorted;
        src_res = ctx->d_ascii;
    } else {                              // runs = the source shards, in rank (= shard) order
        if (n_out > 0 && (!d_recv_meta || (r_out > 0 && !d_recv_res)))
            return fail(ctx, SAD_E_ARG, "sad_finish: NULL receive buffer");
        int64_t *runs = recv_layout ? ctx->h_runs : reinterpret_cast<int64_t *>(ctx->h_small + 16384);
        runs[0] = 0;
        for (int s = 0; s < p; ++s) {
            int64_t c = 0;
            for (int b = ctx->shard0; b < ctx->shard0 + ctx->pl; ++b) c += h_counts_all[((size_t)s * p + b) * 2];
            runs[s + 1] = runs[s] + c;
        }
        CK(cudaMemcpyAsync(ctx->d_runs, runs, sizeof(int64_t) * (p + 1), cudaMemcpyHostToDevice, ctx->st));
        m.keys = reinterpret_cast<const unsigned long long *>(d_recv_meta);
        m.kstride = 2;
        m.lens = reinterpret_cast<const unsigned long long *>(d_recv_meta) + 1;
        m.lstride = 2;
        m.run_start = ctx->d_runs;
        m.nr = p;
        launch_lens_recv(reinterpret_cast<const unsigned long long *>(d_recv_meta), n_out, o.len_sorted, ctx->st);
        LAUNCHED();
        CK(cudaMemsetAsync(o.src_off, 0, sizeof(int64_t), ctx->st));
        if (n_out > 0) {                          // [n + 1] exclusive prefix of the received lengths
            size_t tb = o.cub_bytes;
            CK(cub::DeviceScan::InclusiveSum(o.cub, tb, o.len_sorted, o.src_off + 1, nn, ctx->st));
            LAUNCHED();
        }
        m.cpre = o.src_off;
        src_off = o.src_off;
        src_perm = nullptr;
        src_res = d_recv_res;
    }
    m.out_off = o.off;
    if (n_out == 0) CK(cudaMemsetAsync(o.off, 0, sizeof(int64_t), ctx->st));
    if (n_out > 0) {
        launch_rank_merge(m, ctx->st);         // keys, lengths, sources and residue offsets
        LAUNCHED();
        launch_gather_res(o.perm, src_perm, n_out, src_off, src_res, o.off, o.res, ctx->st);
        LAUNCHED();
    }
    ctx->d_out = reinterpret_cast<uint8_t *>(d_out);
    ctx->out_bytes = out_bytes;
    ctx->out_n = n_out;
    ctx->out_r = r_out;
    ctx->out_recv_layout = recv_layout;
    ctx->stage = 6;
    ctx->launches_last = ctx->launches_step;
    return SAD_OK;
}

int sad_finish(sad_ctx *ctx, const int64_t *h_counts_all, const uint64_t *d_recv_meta, const uint8_t *d_recv_res,
               void *d_out, size_t out_bytes, int64_t *h_bucket_sizes) {
    GUARD(5);
    const int p = ctx->cfg.p;
    if ((!h_counts_all && ctx->cfg.world != 1) || !d_out) return fail(ctx, SAD_E_ARG, "sad_finish: NULL buffer");
    const bool local = d_recv_meta == nullptr;
    if (local && ctx->cfg.world != 1) return fail(ctx, SAD_E_ARG, "NULL receive buffers need world == 1");
    if (int rc = finish_impl(ctx, h_counts_all, d_recv_meta, d_recv_res, d_out, out_bytes, false)) return rc;
    if (h_counts_all) {
        ctx->h_counts_all.assign(h_counts_all, h_counts_all + (size_t)p * p * 2);
        ctx->counts_pending = false;
        bucket_sizes_from_counts(ctx);
        if (h_bucket_sizes) std::memcpy(h_bucket_sizes, ctx->bucket_sizes.data(), sizeof(int64_t) * p);
    } else {
        // world == 1: the counts stay on the device; they are read back lazily (getters sync)
        CK(cudaMemcpyAsync(ctx->h_small + 45056, ctx->d_counts, sizeof(int64_t) * (size_t)p * p * 2,
                           cudaMemcpyDeviceToHost, ctx->st));
        ctx->counts_pending = true;
        if (h_bucket_sizes) {
            if (int rc = sad_get_bucket_sizes(ctx, h_bucket_sizes)) return rc;
        }
    }
    return SAD_OK;
}

int sad_exchange_verdict(int32_t p, int32_t world, const int64_t *h_gathered, int64_t *h_counts_all, int32_t *who,
                         int32_t *kind) {
    if (!h_gathered || !h_counts_all || p < 1 || world < 1 || p % world) return SAD_E_ARG;
    const int pl = p / world;
    const int64_t B = (int64_t)pl * p * 2 + 4;
    if (who) *who = -1;
    if (kind) *kind = 0;
    // an input error anywhere: no rank moves data (peers report the first failing rank)
    for (int r = 0; r < world; ++r) {
        const int64_t *tail = h_gathered + (size_t)r * B + (size_t)pl * p * 2;
        if (tail[1]) {
            if (who) *who = r;
            if (kind) *kind = (int32_t)tail[1];
            return SAD_E_NCCL;
        }
    }
    for (int r = 0; r < world; ++r)
        if (h_gathered[(size_t)r * B + (size_t)pl * p * 2]) return SAD_E_REPLAN;   // an operand overflowed
    // counts_all [p][p][2]: rank r's block holds shards r*pl .. in order
    for (int r = 0; r < world; ++r)
        std::memcpy(h_counts_all + (size_t)r * pl * p * 2, h_gathered + (size_t)r * B, sizeof(int64_t) * (size_t)pl * p * 2);
    // every rank's output need against the capacity it announced
    for (int r = 0; r < world; ++r) {
        int64_t n_r = 0, r_r = 0;
        for (int s = 0; s < p; ++s)
            for (int b = r * pl; b < (r + 1) * pl; ++b) {
                n_r += h_counts_all[((size_t)s * p + b) * 2 + 0];
                r_r += h_counts_all[((size_t)s * p + b) * 2 + 1];
            }
        const int64_t have = h_gathered[(size_t)r * B + (size_t)pl * p * 2 + 2];
        if ((int64_t)out_layout(nullptr, n_r, r_r, true).total > have) {
            if (who) *who = r;
            return SAD_E_CAPACITY;
        }
    }
    return SAD_OK;
}

int sad_partition(sad_ctx *ctx, void *d_out, size_t out_bytes, int64_t *h_bucket_sizes) {
    GUARD(4);
    const int p = ctx->cfg.p, G = ctx->cfg.world, pl = ctx->pl;
    if (G > 1 && !ctx->comm)
        return fail(ctx, SAD_E_STATE, "sad_partition with world > 1 needs a communicator (sad_create with an NCCL id)");
    if (!d_out || (G > 1 && !h_bucket_sizes)) return fail(ctx, SAD_E_ARG, "sad_partition: NULL buffer");
    ctx->capturing = stream_capturing(ctx->st);
    // a9: "Sort all the p*(p-1) ranks ..." -- every rank's regular samples, replicated selection
    const uint64_t *smp_all = reinterpret_cast<const uint64_t *>(ctx->d_smp_mine);
    if (coll_exchange(ctx) && p > 1) {
        NK(ncclAllGather(ctx->d_smp_mine, ctx->d_smp_all, (size_t)pl * (p - 1), ncclUint64, comm_of(ctx), ctx->st));
        smp_all = reinterpret_cast<const uint64_t *>(ctx->d_smp_all);
    }
    if (int rc = plan_impl(ctx, smp_all, ctx->d_cnt_send)) return rc;
    if (!coll_exchange(ctx)) {
        // world == 1 without a communicator: the buckets are this rank's own shards, merged locally
        if (int rc = finish_impl(ctx, nullptr, nullptr, nullptr, d_out, out_bytes, false)) return rc;
        CK(cudaMemcpyAsync(ctx->h_small + 45056, ctx->d_counts, sizeof(int64_t) * (size_t)p * p * 2,
                           cudaMemcpyDeviceToHost, ctx->st));
        ctx->counts_pending = true;
        if (h_bucket_sizes) {
            if (int rc = sad_get_bucket_sizes(ctx, h_bucket_sizes)) return rc;
        }
        return SAD_OK;
    }
    if (ctx->capturing) return fail(ctx, SAD_E_STATE, "the count exchange synchronizes: it cannot be graph-captured");
    // the count exchange: every rank's [pl][p][2] counts plus its status (operand overflow, first
    // input error, output capacity), so that all ranks take the same decision
    const int64_t B = count_block(ctx);
    launch_status_tail(ctx->d_status, ctx->d_err, (int64_t)out_bytes, ctx->d_cnt_send + (size_t)pl * p * 2, ctx->st);
    LAUNCHED();
    NK(ncclAllGather(ctx->d_cnt_send, ctx->d_cnt_all, (size_t)B, ncclInt64, comm_of(ctx), ctx->st));
    CK(cudaMemcpyAsync(ctx->h_cnt_all, ctx->d_cnt_all, sizeof(int64_t) * (size_t)G * B, cudaMemcpyDeviceToHost,
                       ctx->st));
    CK(cudaEventRecord(ctx->ev_stats, ctx->st));
    if (int rc = wait_collective(ctx, ctx->ev_stats)) return rc;
    // the same decision on every rank, from the same gathered blocks
    std::vector<int64_t> counts_all((size_t)p * p * 2);
    int32_t who = -1, kind = 0;
    const int verdict = sad_exchange_verdict(p, G, ctx->h_cnt_all, counts_all.data(), &who, &kind);
    const int own = absorb(ctx, true);   // this rank's own error / overflow, with its message
    if (verdict == SAD_E_NCCL) {
        if (own && own != SAD_E_REPLAN) return own;
        static const char *kinds[4] = {"", "an illegal symbol", "a sequence shorter than k", "a sequence too long"};
        return fail(ctx, SAD_E_NCCL, "rank %d reported %s; no data moved", who, kinds[kind & 3]);
    }
    if (verdict == SAD_E_REPLAN) {
        ctx->kcap_blocks = std::max(ctx->kcap_blocks, ctx->kcap_next);
        ctx->stage = 1;
        return soft_fail(ctx, SAD_E_REPLAN, "a rank's all-pairs operand overflowed: rerun the step on every rank");
    }
    if (own) return own;
    if (verdict == SAD_E_CAPACITY) {
        ctx->stage = 4;              // the partition can be called again with a larger buffer
        return soft_fail(ctx, SAD_E_CAPACITY, "rank %d: output buffer below its need (sad_output_bound)", who);
    }
    // a11: pack, then the all-to-all personalized exchange (grouped send / receive)
    sad_pack_plan(p, G, ctx->cfg.rank, counts_all.data(), ctx->h_seg);
    if (int rc = pack_impl(ctx, ctx->h_seg, reinterpret_cast<uint64_t *>(ctx->d_send_meta), ctx->d_send_res)) return rc;
    std::vector<int64_t> ss(G), sr(G), rs(G), rr(G);
    sad_exchange_sizes(p, G, ctx->cfg.rank, counts_all.data(), ss.data(), sr.data(), rs.data(), rr.data());
    int64_t n_out = 0, r_out = 0;
    for (int r = 0; r < G; ++r) {
        n_out += rs[r];
        r_out += rr[r];
    }
    OutLayout o = out_layout(reinterpret_cast<uint8_t *>(d_out), n_out, r_out, true);
    NK(ncclGroupStart());
    int64_t so = 0, sro = 0, ro = 0, rro = 0;
    for (int r = 0; r < G; ++r) {
        if (ss[r]) NK(ncclSend(ctx->d_send_meta + 2 * so, (size_t)(2 * ss[r]), ncclUint64, r, comm_of(ctx), ctx->st));
        if (rs[r]) NK(ncclRecv(o.recv_meta + 2 * ro, (size_t)(2 * rs[r]), ncclUint64, r, comm_of(ctx), ctx->st));
        if (sr[r]) NK(ncclSend(ctx->d_send_res + sro, (size_t)sr[r], ncclUint8, r, comm_of(ctx), ctx->st));
        if (rr[r]) NK(ncclRecv(o.recv_res + rro, (size_t)rr[r], ncclUint8, r, comm_of(ctx), ctx->st));
        so += ss[r];
        sro += sr[r];
        ro += rs[r];
        rro += rr[r];
    }
    NK(ncclGroupEnd());
    if (int rc = finish_impl(ctx, counts_all.data(), reinterpret_cast<const uint64_t *>(o.recv_meta), o.recv_res, d_out,
                             out_bytes, true))
        return rc;
    ctx->h_counts_all = counts_all;
    ctx->counts_pending = false;
    bucket_sizes_from_counts(ctx);
    if (h_bucket_sizes) std::memcpy(h_bucket_sizes, ctx->bucket_sizes.data(), sizeof(int64_t) * p);
    return SAD_OK;
}

// --------------------------------------------------------------------------- getters

static void bucket_sizes_from_counts(sad_ctx *ctx) {
    const int p = ctx->cfg.p;
    ctx->bucket_sizes.assign(p, 0);
    for (int s = 0; s < p; ++s)
        for (int b = 0; b < p; ++b) ctx->bucket_sizes[b] += ctx->h_counts_all[((size_t)s * p + b) * 2];
    ctx->bucket_first.assign(p + 1, 0);
    for (int b = 0; b < p; ++b) ctx->bucket_first[b + 1] = ctx->bucket_first[b] + ctx->bucket_sizes[b];
}

// every synchronizing getter: wait for the step, report its device-detected errors
static int sync_step(sad_ctx *ctx) {
    if (int rc = absorb(ctx, true)) return rc;
    CK(cudaStreamSynchronize(ctx->st));
    return SAD_OK;
}

static int resolve_counts(sad_ctx *ctx) {
    if (int rc = sync_step(ctx)) return rc;
    if (!ctx->counts_pending) return SAD_OK;
    const int p = ctx->cfg.p;
    const int64_t *c = reinterpret_cast<const int64_t *>(ctx->h_small + 45056);
    ctx->h_counts_all.assign(c, c + (size_t)p * p * 2);
    ctx->counts_pending = false;
    bucket_sizes_from_counts(ctx);
    return SAD_OK;
}

int sad_get_bucket_sizes(sad_ctx *ctx, int64_t *h_sizes) {
    GUARD(6);
    if (!h_sizes) return SAD_E_ARG;
    if (int rc = resolve_counts(ctx)) return rc;
    std::memcpy(h_sizes, ctx->bucket_sizes.data(), sizeof(int64_t) * ctx->cfg.p);
    return SAD_OK;
}

int sad_get_load_report(sad_ctx *ctx, int64_t *h_report) {
    GUARD(6);
    if (!h_report) return SAD_E_ARG;
    if (int rc = resolve_counts(ctx)) return rc;
    const int p = ctx->cfg.p;
    int64_t mb = 0;
    for (int b = 0; b < p; ++b) mb = std::max(mb, ctx->bucket_sizes[b]);
    const int64_t w = (ctx->n_global + p - 1) / p;               // the largest shard (reading A15)
    h_report[0] = mb;
    h_report[1] = w;
    h_report[2] = 2 * w + p;
    h_report[3] = mb <= 2 * w + p;
    h_report[4] = (ctx->n_global % p == 0) && (w % p == 0);
    h_report[5] = mb < 2 * w;
    return SAD_OK;
}

static int shard_check(sad_ctx *ctx, int shard, int64_t cap, int64_t &b0, int64_t &w) {
    if (shard < 0 || shard >= ctx->pl) return fail(ctx, SAD_E_ARG, "bad shard %d", shard);
    b0 = ctx->shard_base[shard];
    w = ctx->shard_base[shard + 1] - b0;
    if (cap < w) return fail(ctx, SAD_E_CAPACITY, "capacity %lld < %lld", (long long)cap, (long long)w);
    return SAD_OK;
}

int sad_get_local_rank(sad_ctx *ctx, int shard, uint64_t *h_T, int64_t cap) {
    GUARD(3);
    int64_t b0, w;
    if (int rc = shard_check(ctx, shard, cap, b0, w)) return rc;
    if (int rc = sync_step(ctx)) return rc;
    CK(cudaMemcpyAsync(h_T, ctx->d_T + b0, sizeof(uint64_t) * w, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return SAD_OK;
}

int sad_get_ancestors(sad_ctx *ctx, int64_t *h_local, int64_t *h_ga) {
    GUARD(4);
    const int p = ctx->cfg.p;
    if (int rc = sync_step(ctx)) return rc;
    std::vector<long long> g(p + 2);
    CK(cudaMemcpyAsync(g.data(), ctx->d_ga_info, sizeof(long long) * (p + 2), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    if (h_ga) *h_ga = g[1];
    if (h_local) for (int s = 0; s < p; ++s) h_local[s] = g[2 + s];
    return SAD_OK;
}

int sad_get_ranks(sad_ctx *ctx, int shard, uint32_t *h_S, uint32_t *h_den, uint64_t *h_key, int64_t cap) {
    GUARD(4);
    int64_t b0, w;
    if (int rc = shard_check(ctx, shard, cap, b0, w)) return rc;
    if (int rc = sync_step(ctx)) return rc;
    if (h_S) CK(cudaMemcpyAsync(h_S, ctx->d_S_ga + b0, 4 * w, cudaMemcpyDeviceToHost, ctx->st));
    if (h_den) CK(cudaMemcpyAsync(h_den, ctx->d_den_ga + b0, 4 * w, cudaMemcpyDeviceToHost, ctx->st));
    if (h_key) CK(cudaMemcpyAsync(h_key, ctx->d_key + b0, 8 * w, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return SAD_OK;
}

int sad_get_sorted(sad_ctx *ctx, int shard, int64_t *h_idx, int64_t cap) {
    GUARD(4);
    int64_t b0, w;
    if (int rc = shard_check(ctx, shard, cap, b0, w)) return rc;
    if (int rc = sync_step(ctx)) return rc;
    std::vector<int32_t> t(w);
    CK(cudaMemcpyAsync(t.data(), ctx->d_perm_sorted + b0, 4 * w, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    for (int64_t i = 0; i < w; ++i) h_idx[i] = ctx->first_idx + t[i];
    return SAD_OK;
}

int sad_get_pivots(sad_ctx *ctx, uint64_t *h_pivots) {
    GUARD(5);
    if (int rc = sync_step(ctx)) return rc;
    if (ctx->cfg.p > 1) {
        CK(cudaMemcpyAsync(h_pivots, ctx->d_pivots, 8 * (ctx->cfg.p - 1), cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
    }
    return SAD_OK;
}

int sad_get_bucket(sad_ctx *ctx, int bucket, int64_t *h_idx, uint64_t *h_key, uint8_t *h_res, int64_t *h_offsets,
                   int64_t cap_seqs, int64_t cap_res, int64_t *n_out, int64_t *res_out) {
    GUARD(6);
    const int b0 = ctx->shard0, b1 = ctx->shard0 + ctx->pl;
    if (bucket < b0 || bucket >= b1) return fail(ctx, SAD_E_ARG, "bucket %d is not owned by rank %d", bucket, ctx->cfg.rank);
    if (int rc = resolve_counts(ctx)) return rc;
    int64_t first = 0;
    for (int b = b0; b < bucket; ++b) first += ctx->bucket_sizes[b];
    const int64_t n = ctx->bucket_sizes[bucket];
    OutLayout o = out_layout(ctx->d_out, ctx->out_n, ctx->out_r, ctx->out_recv_layout);
    int64_t r0 = 0, r1 = 0;
    CK(cudaMemcpyAsync(&r0, o.off + first, 8, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(&r1, o.off + first + n, 8, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    if (n_out) *n_out = n;
    if (res_out) *res_out = r1 - r0;
    if ((h_idx || h_key) && cap_seqs < n) return fail(ctx, SAD_E_CAPACITY, "bucket has %lld sequences", (long long)n);
    if (h_offsets && cap_seqs < n + 1)       // the offsets take n + 1 entries
        return fail(ctx, SAD_E_CAPACITY, "bucket offsets need %lld entries", (long long)(n + 1));
    if (h_res && cap_res < r1 - r0) return fail(ctx, SAD_E_CAPACITY, "bucket has %lld residues", (long long)(r1 - r0));
    std::vector<uint64_t> keys(n);
    if (n) CK(cudaMemcpyAsync(keys.data(), o.key + first, 8 * n, cudaMemcpyDeviceToHost, ctx->st));
    if (h_offsets) CK(cudaMemcpyAsync(h_offsets, o.off + first, 8 * (n + 1), cudaMemcpyDeviceToHost, ctx->st));
    if (h_res && r1 > r0) CK(cudaMemcpyAsync(h_res, o.res + r0, r1 - r0, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    for (int64_t i = 0; i < n; ++i) {
        if (h_key) h_key[i] = keys[i];
        if (h_idx) h_idx[i] = (int64_t)(keys[i] & ((1ull << ctx->ibits) - 1ull));
    }
    if (h_offsets) for (int64_t i = 0; i <= n; ++i) h_offsets[i] -= r0;
    return SAD_OK;
}

int sad_get_similarity(sad_ctx *ctx, int shard, uint16_t *h_S, int64_t cap) {
    GUARD(3);
    if (!ctx->d_sim) return fail(ctx, SAD_E_STATE, "context created without SAD_F_KEEP_SIM");
    int64_t b0, w;
    if (int rc = shard_check(ctx, shard, INT64_MAX, b0, w)) return rc;
    if (cap < w * w) return fail(ctx, SAD_E_CAPACITY, "capacity %lld < %lld", (long long)cap, (long long)(w * w));
    if (int rc = sync_step(ctx)) return rc;
    int64_t sb = 0;
    for (int s = 0; s < shard; ++s) {
        const int64_t ws = ctx->shard_base[s + 1] - ctx->shard_base[s];
        sb += ws * ws;
    }
    CK(cudaMemcpyAsync(h_S, ctx->d_sim + sb, 2 * w * w, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return SAD_OK;
}

int sad_get_bucket_view(sad_ctx *ctx, int bucket, const uint8_t **d_res, const int64_t **d_offsets, int64_t *n,
                        int64_t *res_bytes) {
    GUARD(6);
    const int b0 = ctx->shard0, b1 = ctx->shard0 + ctx->pl;
    if (bucket < b0 || bucket >= b1) return fail(ctx, SAD_E_ARG, "bucket %d is not owned by rank %d", bucket, ctx->cfg.rank);
    if (int rc = resolve_counts(ctx)) return rc;
    int64_t first = 0;
    for (int b = b0; b < bucket; ++b) first += ctx->bucket_sizes[b];
    const int64_t nb = ctx->bucket_sizes[bucket];
    OutLayout o = out_layout(ctx->d_out, ctx->out_n, ctx->out_r, ctx->out_recv_layout);
    int64_t r[2] = {0, 0};
    CK(cudaMemcpyAsync(r, o.off + first, 8, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(r + 1, o.off + first + nb, 8, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    if (d_res) *d_res = o.res + r[0];
    if (d_offsets) *d_offsets = o.off + first;
    if (n) *n = nb;
    if (res_bytes) *res_bytes = r[1] - r[0];
    return SAD_OK;
}

int sad_get_distance(sad_ctx *ctx, int shard, float *d_D, int64_t cap) {
    GUARD(3);
    if (!ctx->d_sim) return fail(ctx, SAD_E_STATE, "context created without SAD_F_KEEP_SIM");
    int64_t b0, w;
    if (int rc = shard_check(ctx, shard, INT64_MAX, b0, w)) return rc;
    if (!d_D || cap < w * w) return fail(ctx, SAD_E_CAPACITY, "capacity %lld < %lld", (long long)cap, (long long)(w * w));
    int64_t sb = 0;
    for (int s = 0; s < shard; ++s) {
        const int64_t ws = ctx->shard_base[s + 1] - ctx->shard_base[s];
        sb += ws * ws;
    }
    launch_distance(ctx->d_sim + sb, ctx->d_rowinfo + b0, w, d_D, ctx->st);
    LAUNCHED();
    return SAD_OK;
}

int sad_get_distance_f64(sad_ctx *ctx, int shard, double *d_D, int64_t cap) {
    GUARD(3);
    if (!ctx->d_sim) return fail(ctx, SAD_E_STATE, "context created without SAD_F_KEEP_SIM");
    int64_t b0, w;
    if (int rc = shard_check(ctx, shard, INT64_MAX, b0, w)) return rc;
    if (!d_D || cap < w * w) return fail(ctx, SAD_E_CAPACITY, "capacity %lld < %lld", (long long)cap, (long long)(w * w));
    int64_t sb = 0;
    for (int s = 0; s < shard; ++s) {
        const int64_t ws = ctx->shard_base[s + 1] - ctx->shard_base[s];
        sb += ws * ws;
    }
    launch_distance64(ctx->d_sim + sb, ctx->d_rowinfo + b0, w, d_D, ctx->st);
    LAUNCHED();
    return SAD_OK;
}

size_t sad_upgma_workspace(int64_t n) { return n > 0 ? upgma_workspace(n) : 0; }

int sad_upgma(double *d_D, int64_t n, int64_t *d_merges, double *d_heights, int64_t *d_sizes, void *d_ws,
              size_t ws_bytes, void *stream) {
    if (n < 1 || !d_D || (n > 1 && (!d_merges || !d_heights || !d_sizes)) || n > 0x7FFFFFFF) return SAD_E_ARG;
    if (n == 1) return SAD_OK;
    if (!d_ws || ws_bytes < upgma_workspace(n) || (reinterpret_cast<uintptr_t>(d_ws) & 255)) return SAD_E_CAPACITY;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    launch_upgma(d_D, n, d_merges, d_heights, d_sizes, d_ws, st);
    return cudaGetLastError() == cudaSuccess ? SAD_OK : SAD_E_CUDA;
}

int sad_get_profile_info(sad_ctx *ctx, int64_t *h_windows, int64_t *h_distinct, int64_t *h_kcols) {
    GUARD(2);
    if (int rc = absorb(ctx, true)) return rc;
    for (int s = 0; s < ctx->pl; ++s) {
        if (h_windows) h_windows[s] = s < (int)ctx->h_windows.size() ? ctx->h_windows[s] : 0;
        if (h_distinct) h_distinct[s] = s < (int)ctx->h_distinct.size() ? ctx->h_distinct[s] : 0;
        if (h_kcols) h_kcols[s] = s < (int)ctx->h_K.size() ? ctx->h_K[s] : 0;
    }
    return SAD_OK;
}

int sad_get_stats(sad_ctx *ctx, double *h_ms, int64_t *h_counts) {
    if (!ctx) return SAD_E_ARG;
    if (ctx->sticky) return SAD_E_STATE;
    DeviceScope dev_scope_(ctx->cfg.device);
    CK(cudaStreamSynchronize(ctx->st));
    for (auto *v : {&ctx->ev_pairs_ap, &ctx->ev_pairs_op}) {
        double &acc = v == &ctx->ev_pairs_ap ? ctx->ms_ap : ctx->ms_op;
        for (auto &e : *v) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e.first, e.second));
            acc += ms;
            ctx->ev_free.push_back(e);
        }
        v->clear();
    }
    if (h_ms) { h_ms[0] = ctx->ms_ap; h_ms[1] = ctx->ms_op; }
    if (h_counts) {
        h_counts[0] = ctx->calls;
        h_counts[1] = ctx->pairs;
        h_counts[2] = ctx->macs;
        h_counts[3] = ctx->launches_last;
    }
    return SAD_OK;
}

int sad_graph_account(sad_ctx *ctx) {
    if (!ctx) return SAD_E_ARG;
    if (ctx->sticky) return SAD_E_STATE;
    if (!ctx->graph_events) return fail(ctx, SAD_E_STATE, "no captured step");
    DeviceScope dev_scope_(ctx->cfg.device);
    CK(cudaStreamSynchronize(ctx->st));
    float op = 0, ap = 0;
    CK(cudaEventElapsedTime(&op, ctx->gev[0], ctx->gev[1]));
    CK(cudaEventElapsedTime(&ap, ctx->gev[2], ctx->gev[3]));
    ctx->ms_op += op;
    ctx->ms_ap += ap;
    ctx->calls += 1;
    if (ctx->stage >= 6) ctx->counts_pending = true;   // the replay rewrote the counts: getters reread them
    return SAD_OK;
}

int sad_reset_stats(sad_ctx *ctx) {
    if (!ctx) return SAD_E_ARG;
    double ms[2];
    int rc = sad_get_stats(ctx, ms, nullptr);
    ctx->ms_ap = ctx->ms_op = 0;
    ctx->calls = 0;
    return rc;
}

int sad_selftest_fixed_point(sad_ctx *ctx, int32_t max_den, int64_t *h_bad) {
    GUARD(0);
    if (max_den < 1 || max_den > 65535 || !h_bad) return fail(ctx, SAD_E_ARG, "max_den in [1, 65535]");
    unsigned long long *d = nullptr;
    CK(cudaMallocAsync(&d, 8, ctx->st));
    CK(cudaMemsetAsync(d, 0, 8, ctx->st));
    launch_selftest_fixed(max_den, d, ctx->st);
    LAUNCHED();
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaFreeAsync(d, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    *h_bad = (int64_t)h;
    return SAD_OK;
}

}  // extern "C"
