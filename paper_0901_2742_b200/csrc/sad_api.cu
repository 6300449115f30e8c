// sad_api.cu — the C ABI of libsad.so (include/sad.h): argument checks, workspace carving,
// stage orchestration on the caller's stream. All arithmetic of the method is in k_*.cu.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

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

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(ctx, SAD_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
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

// shard bases of this rank under the block split of reading A15
void shard_layout(const sad_ctx *c, int64_t n_global, std::vector<int64_t> &sb) {
    const int p = c->cfg.p;
    const int64_t base = n_global / p, extra = n_global % p;
    sb.assign(c->pl + 1, 0);
    int64_t g0 = 0;
    for (int s = 0; s < c->shard0; ++s) g0 += base + (s < extra ? 1 : 0);
    for (int s = 0; s < c->pl; ++s) sb[s + 1] = sb[s] + base + (c->shard0 + s < extra ? 1 : 0);
    (void)g0;
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

// carve the workspace; with base == nullptr only the size is computed
size_t carve(sad_ctx *c, uint8_t *base, int64_t n, int64_t R) {
    Bump b{base};
    const int pl = c->pl, p = c->cfg.p, V = c->V;
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
    c->d_err = b.take<unsigned long long>(4);
    c->d_kinfo = b.take<unsigned long long>((size_t)pl * kKinfo);
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
    c->d_seg = b.take<int64_t>((size_t)pl * p * 2);
    c->d_counts = b.take<int64_t>((size_t)pl * p * 2);
    c->tc_tiles_cap = tc_tiles_bound(n, pl);
    c->d_tc_tiles = b.take<uint8_t>((size_t)c->tc_tiles_cap * 16);
    c->cub_bytes = cub_bytes_needed(n, pl);
    c->d_cub = b.take<uint8_t>(c->cub_bytes);
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
    unsigned long long *key, *keys_in;
    int64_t *off, *len_in, *len_sorted, *src_off;
    uint8_t *res, *cub;
    int32_t *vals_in, *perm;
    size_t cub_bytes, total;
};

OutLayout out_layout(uint8_t *base, int64_t n, int64_t r) {
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
    o.total = b.off + 256;
    return o;
}

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

extern "C" {

static void bucket_sizes_from_counts(sad_ctx *ctx);

uint32_t sad_abi_version(void) { return SAD_ABI_VERSION; }

int sad_create(const sad_config *cfg, sad_ctx **out) {
    if (!cfg || !out) return SAD_E_ARG;
    *out = nullptr;
    if (cfg->alphabet != SAD_PROTEIN20 && cfg->alphabet != SAD_DNA4) return SAD_E_ARG;
    if (cfg->k < 1 || cfg->p < 1 || cfg->p > 64 || cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world)
        return SAD_E_ARG;
    if (cfg->p % cfg->world != 0) return SAD_E_ARG;
    if ((cfg->flags & SAD_F_RANK_SAMPLES) && cfg->p < 2) return SAD_E_ARG;   // f1 needs k = p-1 >= 1 samples
    const int A = cfg->alphabet == SAD_PROTEIN20 ? 20 : 4;
    int64_t V = 1;
    for (int i = 0; i < cfg->k; ++i) {
        V *= A;
        if (V > 65536) return SAD_E_ARG;
    }
    if ((cfg->flags & SAD_F_RANK_SAMPLES) && V * 8 > 200 * 1024) return SAD_E_ARG;
    sad_ctx *ctx = new (std::nothrow) sad_ctx();
    if (!ctx) return SAD_E_OOM;
    ctx->cfg = *cfg;
    ctx->st = reinterpret_cast<cudaStream_t>(cfg->stream);
    ctx->A = A;
    ctx->V = (int)V;
    ctx->pl = cfg->p / cfg->world;
    ctx->shard0 = cfg->rank * ctx->pl;
    ctx->use_tc = !(cfg->flags & SAD_F_KERNEL_ALU);
    ctx->tc_kind = (cfg->flags & SAD_F_TC_INT8) ? 0 : 1;
    ctx->tc_cg = (cfg->flags & SAD_F_TC_1SM) ? 1 : 2;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) {
        delete ctx;
        return SAD_E_CUDA;
    }
    DeviceScope dev_scope_(cfg->device);
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cfg->device);
    if (cudaMallocHost(&ctx->h_small, 65536 * sizeof(unsigned long long)) != cudaSuccess) {
        delete ctx;
        return SAD_E_CUDA;
    }
    if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_stats, cudaEventDisableTiming) != cudaSuccess ||
        [&] {
            for (auto &e : ctx->ev_chunk)
                if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return true;
            return false;
        }()) {
        cudaFreeHost(ctx->h_small);
        delete ctx;
        return SAD_E_CUDA;
    }
    if (ctx->use_tc) {
        std::string why;
        if (!tc_supported(why)) {
            sad_destroy(ctx);
            return SAD_E_ARG;
        }
    }
    *out = ctx;
    return SAD_OK;
}

void sad_destroy(sad_ctx *ctx) {
    if (!ctx) return;
    DeviceScope dev_scope_(ctx->cfg.device);
    if (ctx->st) cudaStreamSynchronize(ctx->st); else cudaDeviceSynchronize();
    for (auto &v : {&ctx->ev_pairs_ap, &ctx->ev_pairs_op, &ctx->ev_free})
        for (auto &e : *v) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
    }
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->ev_stats) cudaEventDestroy(ctx->ev_stats);
    for (auto &e : ctx->ev_chunk)
        if (e) cudaEventDestroy(e);
    if (ctx->h_small) cudaFreeHost(ctx->h_small);
    if (ctx->h_tiles) cudaFreeHost(ctx->h_tiles);
    delete ctx;
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
    *bytes = carve(&tmp, nullptr, n_local, residues_local);
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
    if (n_global / p + 1 >= (int64_t(1) << 24)) return fail(ctx, SAD_E_ARG, "shards of 2^24 or more sequences");
    int64_t R = residues_local;
    bool need_sync = mem == SAD_MEM_HOST;     // host inputs may be reused by the caller on return
    if (mem == SAD_MEM_HOST) {
        if (offsets[0] != 0) return fail(ctx, SAD_E_ARG, "offsets[0] != 0");
        if (R >= 0 && R != offsets[n_local]) return fail(ctx, SAD_E_ARG, "residues_local != offsets[n_local]");
        R = offsets[n_local];
    } else if (R < 0 && mem == SAD_MEM_DEVICE_REBASE) {
        return fail(ctx, SAD_E_ARG, "SAD_MEM_DEVICE_REBASE needs residues_local");
    } else if (R < 0) {
        CK(cudaMemcpyAsync(ctx->h_small + 40000, offsets + n_local, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        R = (int64_t)ctx->h_small[40000];
    }
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
    for (int s = 0; s < ctx->pl; ++s) {
        const int64_t w = sb[s + 1] - sb[s];
        ctx->max_w = std::max(ctx->max_w, w);
        ctx->shard_rowpad[s + 1] = ctx->shard_rowpad[s] + rup(w, kRowPad);
    }
    ctx->rows_pad = ctx->shard_rowpad[ctx->pl];
    const cudaMemcpyKind kind = mem == SAD_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    // host inputs of a few MB or more: the residues are copied in chunks on the internal stream and
    // each chunk's k-mer counts (K1/K2) start on ctx->st as soon as it has landed (below)
    const int nch = 4;                     // chunks of a pipelined host load (16 max; 4 measured best)
    const bool pipelined = nch > 0 && mem == SAD_MEM_HOST && R >= (int64_t(4) << 20) && n_local >= 64 * nch;
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
            ctx->tc_tiles_n = tc_build_tiles(ctx->pl, sb.data(), ctx->tc_kind, ctx->tc_cg, ctx->h_tiles, ctx->tc_tiles_cap);
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
        ctx->tbl_ws = base;
        ctx->tbl_n = n_local;
        ctx->tbl_ng = n_global;
        ctx->tbl_first = first_source_index;
        ctx->tbl_R = R;
        need_sync = true;
    }
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
    CK(cudaMemsetAsync(ctx->d_M, 0, sizeof(uint32_t) * (size_t)pl * V, ctx->st));
    CK(cudaMemsetAsync(ctx->d_Mb, 0, sizeof(uint32_t) * (size_t)pl * ((V + 31) / 32), ctx->st));
    CK(cudaMemsetAsync(ctx->d_err, 0xFF, sizeof(unsigned long long) * 4, ctx->st));
    CK(cudaMemsetAsync(ctx->d_kinfo, 0, sizeof(unsigned long long) * kKinfo * (size_t)pl, ctx->st));
    CK(cudaMemsetAsync(ctx->d_Xc, 0, sizeof(uint32_t) * kNumCaps * (size_t)pl * V, ctx->st));
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
    a.i_begin = i0;
    a.i_end = i1;
    launch_profile(a, ctx->st);
    LAUNCHED();
    return SAD_OK;
}

int sad_build_profiles(sad_ctx *ctx) {
    GUARD(1);
    const int pl = ctx->pl, V = ctx->V;
    if (!ctx->profiled) {
        if (int rc = profile_reset(ctx)) return rc;
        if (int rc = profile_launch(ctx, 0, ctx->n)) return rc;
    }
    ctx->profiled = false;
    launch_kstats(ctx->d_M, ctx->d_Mb, ctx->d_Xc, ctx->d_kinfo, pl, V, ctx->st);
    LAUNCHED();
    unsigned long long *hk = ctx->h_small + 8192;
    CK(cudaMemcpyAsync(ctx->h_small, ctx->d_err, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(hk, ctx->d_kinfo, sizeof(unsigned long long) * kKinfo * pl, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaEventRecord(ctx->ev_stats, ctx->st));
    if (ctx->use_tc) {
        // the length order needs no host decision: it runs while the host reads the statistics
        launch_lenorder(ctx->d_rowinfo, ctx->d_shard_base, ctx->d_kinfo, pl, ctx->n, ctx->d_lcnt,
                        ctx->d_lcnt + (size_t)pl * kLenBinsMax, ctx->d_sigma, ctx->d_sigma_inv, ctx->d_rinfo_s,
                        ctx->st);
        ctx->launches_step += 3;
    }
    CK(cudaEventSynchronize(ctx->ev_stats));
    const unsigned long long NONE = ~0ull;
    if (ctx->h_small[0] != NONE) {
        ctx->err_idx = (int64_t)(ctx->h_small[0] >> 32);
        ctx->err_pos = (int64_t)(ctx->h_small[0] & 0xFFFFFFFFull);
        return fail(ctx, SAD_E_SYMBOL, "IllegalSymbol(sequence %lld, position %lld)", (long long)ctx->err_idx,
                    (long long)ctx->err_pos);
    }
    if (ctx->h_small[1] != NONE) {
        ctx->err_idx = (int64_t)ctx->h_small[1];
        return fail(ctx, SAD_E_TOO_SHORT, "SequenceTooShort(sequence %lld): L < k = %d", (long long)ctx->err_idx,
                    ctx->cfg.k);
    }
    if (ctx->h_small[2] != NONE) {
        ctx->err_idx = (int64_t)ctx->h_small[2];
        return fail(ctx, SAD_E_TOO_LONG, "sequence %lld: L - k + 1 > 65535", (long long)ctx->err_idx);
    }
    ctx->h_windows.assign(pl, 0);
    ctx->h_distinct.assign(pl, 0);
    ctx->h_K.assign(pl, 0);
    ctx->h_cap.assign(pl, kNoCap);
    std::vector<uint32_t> sel(pl, kNumCaps);
    int64_t kmax = 0;
    ctx->n_x = 0;
    bool any_excess = false;
    for (int s = 0; s < pl; ++s) {
        const unsigned long long *ki = hk + (size_t)kKinfo * s;
        ctx->h_windows[s] = (int64_t)ki[0];
        ctx->h_distinct[s] = (int64_t)ki[1];
        ctx->h_K[s] = (int64_t)ki[2];
        // layer cap: the smallest T in {1, 2, 4, 8} whose per-row excess
        // sum_tau (n_i - T)+ stays <= 255 for every row, so that every pair's excess fits one
        // byte of the K6 matrix; otherwise all layers stay dense (no cap)
        // (the K6 row accumulators hold max_w bytes per warp in shared memory)
        if (ctx->use_tc && !(ctx->cfg.flags & SAD_F_TC_ALL_LAYERS) && rup(ctx->max_w, 16) <= kXrSmem &&
            ctx->h_ebase[pl] <= kMaxExcessBytes)
            for (int j = 0; j < kNumCaps; ++j)
                if (ki[4 + j] <= 255) {
                    ctx->h_cap[s] = 1u << j;
                    ctx->h_K[s] = (int64_t)ki[8 + j];
                    if (ki[4 + j] > 0) {
                        any_excess = true;
                        sel[s] = (uint32_t)j;
                        ctx->n_x += (int64_t)ki[16 + j];
                    }
                    break;
                }
        kmax = std::max(kmax, ctx->h_K[s]);
    }
    ctx->use_excess = any_excess;

    if (ctx->use_tc) {
        uint32_t *hc = reinterpret_cast<uint32_t *>(ctx->h_small + 12288);
        for (int s = 0; s < pl; ++s) {
            hc[s] = ctx->h_cap[s];
            hc[pl + s] = sel[s];
            hc[2 * pl + s] = (ctx->h_cap[s] == 1u && ctx->h_K[s] == V) ? 1u : 0u;   // col0(tau) = tau
        }
        CK(cudaMemcpyAsync(ctx->d_ident, hc + 2 * pl, sizeof(uint32_t) * pl, cudaMemcpyHostToDevice, ctx->st));
        CK(cudaMemcpyAsync(ctx->d_cap, hc, sizeof(uint32_t) * pl, cudaMemcpyHostToDevice, ctx->st));
        CK(cudaMemcpyAsync(ctx->d_xsel, hc + pl, sizeof(uint32_t) * pl, cudaMemcpyHostToDevice, ctx->st));
    }
    // operand row: K columns padded to one 128-byte K block = 128 int8 or 256 packed fp4 entries
    ctx->kcols_per_block = (ctx->use_tc && ctx->tc_kind == 1) ? 256 : 128;
    ctx->K_stride = std::max<int64_t>(1, (kmax + ctx->kcols_per_block - 1) / ctx->kcols_per_block) * 128;
    ctx->V_pad = rup(V, 64);
    ctx->stage = 2;
    return SAD_OK;
}

// the operand buffer: [indicator | counts operand][K6 lists L_tau u32][K6 dense excess E u8 + 256 zero bytes]
static void operand_parts(const sad_ctx *ctx, size_t &op, size_t &xl, size_t &xe) {
    op = ctx->use_tc ? (size_t)ctx->rows_pad * (size_t)ctx->K_stride : (size_t)ctx->rows_pad * (size_t)ctx->V_pad * 2;
    op = (size_t)rup((int64_t)op, 1024);
    xl = xe = 0;
    if (ctx->use_tc && ctx->use_excess) {
        xl = (size_t)rup(ctx->n_x * 4, 1024);
        xe = (size_t)rup(ctx->h_ebase[ctx->pl] + 256, 1024);
    }
}

int sad_operand_size(const sad_ctx *cctx, size_t *bytes) {
    sad_ctx *ctx = const_cast<sad_ctx *>(cctx);
    GUARD(2);
    if (!bytes) return SAD_E_ARG;
    size_t op = 0, xl = 0, xe = 0;
    operand_parts(ctx, op, xl, xe);
    *bytes = op + xl + xe;
    return SAD_OK;
}

int32_t sad_exchange_records(const sad_ctx *ctx) {
    if (!ctx) return SAD_E_ARG;
    return (ctx->cfg.flags & SAD_F_RANK_SAMPLES) ? ctx->pl * (ctx->cfg.p - 1) : ctx->pl;
}

size_t sad_ancestor_record_bytes(const sad_ctx *ctx) {
    return ctx ? (size_t)rup(16 + 2 * (int64_t)ctx->V, 16) : 0;
}

static void record_pair(sad_ctx *ctx, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, bool begin) {
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

int sad_rank_local(sad_ctx *ctx, void *d_operand, size_t operand_bytes, void *d_anc_out) {
    GUARD(2);
    size_t need = 0;
    sad_operand_size(ctx, &need);
    if (!d_operand || operand_bytes < need || !d_anc_out)
        return fail(ctx, SAD_E_CAPACITY, "operand %zu < %zu bytes or NULL output", operand_bytes, need);
    if ((reinterpret_cast<uintptr_t>(d_operand) & 1023) != 0)
        return fail(ctx, SAD_E_ARG, "operand must be 1024-byte aligned");
    ctx->d_operand = d_operand;
    const int pl = ctx->pl;
    CK(cudaMemsetAsync(ctx->d_T, 0, sizeof(unsigned long long) * (size_t)ctx->n, ctx->st));
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
    size_t op_b = 0, xl_b = 0, xe_b = 0;
    operand_parts(ctx, op_b, xl_b, xe_b);
    uint32_t *lists = xl_b ? reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(d_operand) + op_b) : nullptr;
    uint8_t *E = xl_b ? reinterpret_cast<uint8_t *>(d_operand) + op_b + xl_b : nullptr;
    unsigned long long *xtot = reinterpret_cast<unsigned long long *>(ctx->d_xoff + (size_t)pl * ctx->V + 1) ;
    xtot = reinterpret_cast<unsigned long long *>(rup(reinterpret_cast<int64_t>(xtot), 8));
    record_pair(ctx, ctx->ev_pairs_op, true);
    if (ctx->use_tc) {
        // K3 under the layer caps (the length order sigma was computed by sad_build_profiles);
        // K6 list offsets and lists; K4 beside K6 rows (side stream)
        o.sigma = ctx->d_sigma;
        launch_capscan(ctx->d_M, ctx->V, nullptr, ctx->d_cap, ctx->d_col0, nullptr, 0, pl, ctx->V, ctx->st);
        LAUNCHED();
        o.cap = ctx->d_cap;
        o.ident = ctx->d_ident;
        if (lists) {
            launch_capscan(ctx->d_Xc, (int64_t)kNumCaps * ctx->V, ctx->d_xsel, nullptr, ctx->d_xoff, xtot, 1, pl,
                           ctx->V, ctx->st);
            LAUNCHED();
            CK(cudaMemsetAsync(ctx->d_xcur, 0, sizeof(uint32_t) * (size_t)pl * ctx->V, ctx->st));
            CK(cudaMemsetAsync(E + ctx->h_ebase[pl], 0, 256, ctx->st));   // the zero row segment
            ExcessArgs x{};
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
            launch_xfill(x, ctx->d_xcur, ctx->st);
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
    record_pair(ctx, ctx->ev_pairs_op, false);

    // per shard K blocks (TC)
    std::vector<int64_t> kb(pl + 1, 0);
    int64_t pairs = 0, macs = 0;
    for (int s = 0; s < pl; ++s) {
        kb[s] = (ctx->h_K[s] + ctx->kcols_per_block - 1) / ctx->kcols_per_block;
        const int64_t w = ctx->shard_base[s + 1] - ctx->shard_base[s];
        pairs += w * (w - 1) / 2;
        macs += w * (w + 1) / 2 * ctx->h_K[s];
    }
    ctx->pairs = pairs;
    ctx->macs = macs;
    std::memcpy(ctx->h_small + 1024, kb.data(), sizeof(int64_t) * (pl + 1));
    CK(cudaMemcpyAsync(ctx->d_kblocks, ctx->h_small + 1024, sizeof(int64_t) * (pl + 1), cudaMemcpyHostToDevice,
                       ctx->st));

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
    ap.h_kblocks = kb.data();
    ap.kind = ctx->tc_kind;
    ap.tiles = ctx->d_tc_tiles;
    ap.n_tiles_tc = ctx->tc_tiles_n;
    ap.cg = ctx->tc_cg;
    ap.xrow = lists ? ctx->d_xrow : nullptr;
    ap.E = E;
    ap.ebase = ctx->d_ebase;
    ap.zero = E ? E + ctx->h_ebase[pl] : nullptr;
    record_pair(ctx, ctx->ev_pairs_ap, true);
    if (ctx->use_tc) {
        std::string e;
        const int rc = launch_allpairs_tc(ap, ctx->st, e);
        if (rc) return fail(ctx, SAD_E_CUDA, "tensor-core all-pairs: %s", e.c_str());
    } else {
        launch_allpairs_alu(ap, ctx->st);
    }
    LAUNCHED();
    record_pair(ctx, ctx->ev_pairs_ap, false);
    ctx->calls += 1;

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
    an.rec_bytes = sad_ancestor_record_bytes(ctx);
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

int sad_rank_global(sad_ctx *ctx, const void *d_anc_all, uint64_t *d_samples_out) {
    GUARD(3);
    const int p = ctx->cfg.p;
    if (!d_anc_all || (p > 1 && !d_samples_out)) return fail(ctx, SAD_E_ARG, "sad_rank_global: NULL buffer");
    RankArgs r{};
    r.anc_all = reinterpret_cast<const uint8_t *>(d_anc_all);
    r.rec_bytes = sad_ancestor_record_bytes(ctx);
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
    const int qbits = f1 ? 33 : 32;
    if (!f1) {
        launch_ga_pairs(r, ctx->st);
        LAUNCHED();
        launch_rank_vs_ga(r, ctx->st);
        LAUNCHED();
    } else {
        // f1: T'_i = sum of q(x_i, s) over the m = p(p-1) gathered samples, then
        // Dbar_i = floor(T'_i / m) and the keys (d_key doubles as the T' accumulator)
        const int m = p * (p - 1);
        CK(cudaMemsetAsync(ctx->d_key, 0, sizeof(unsigned long long) * (size_t)ctx->n, ctx->st));
        if (launch_rank_vs_samples(r, m, ctx->d_key, ctx->num_sms, ctx->st))
            return fail(ctx, SAD_E_ARG, "rank vs samples: V too large");
        LAUNCHED();
        launch_f1_keys(ctx->d_key, ctx->n, m, ctx->first_idx, ctx->d_rowinfo, ctx->d_key, ctx->d_ckey, ctx->d_perm_in,
                       ctx->d_S_ga, ctx->d_den_ga, ctx->st);
        LAUNCHED();
        launch_f1_gainfo(ctx->d_anc_local, ctx->pl, ctx->shard0, p, ctx->first_idx, ctx->d_ga_info, ctx->st);
        LAUNCHED();
    }
#ifndef SAD_RANK_SORT_RUNS
#define SAD_RANK_SORT_RUNS 4                 // blocks per shard of the local rank sort (then one merge)
#endif
    if (!(qbits == 32 && ctx->max_w <= kSmallSortMax * SAD_RANK_SORT_RUNS &&
          seg_sort_pairs_runs(ctx->d_ckey, ctx->d_perm_in, ctx->d_shard_base, ctx->pl, SAD_RANK_SORT_RUNS, ctx->n,
                              ctx->d_ckey_sorted, ctx->d_perm_sorted, 32, ctx->st) == 0))
        CK(sort_pairs(ctx, ctx->d_ckey, ctx->d_ckey_sorted, ctx->d_perm_in, ctx->d_perm_sorted, (int)ctx->n,
                      qbits + sbits));
    LAUNCHED();
    launch_unpack_sorted(ctx->d_ckey_sorted, ctx->d_perm_sorted, ctx->n, ctx->first_idx, ctx->d_key_sorted,
                         ctx->d_rowinfo, ctx->cfg.k, ctx->d_len_sorted, qbits, ctx->st);
    LAUNCHED();
    // exclusive prefix of L in sorted order (the residue offsets of every bucket slice, K12/K13)
    CK(cudaMemsetAsync(ctx->d_lpre, 0, sizeof(int64_t), ctx->st));
    {
        size_t tb2 = ctx->cub_bytes;
        CK(cub::DeviceScan::InclusiveSum(ctx->d_cub, tb2, ctx->d_len_sorted, ctx->d_lpre + 1, (int)ctx->n, ctx->st));
        LAUNCHED();
    }
    if (p > 1) {
        launch_samples(ctx->d_key_sorted, ctx->d_shard_base, ctx->pl, p,
                       reinterpret_cast<unsigned long long *>(d_samples_out), ctx->st);
        LAUNCHED();
    }
    ctx->stage = 4;
    return SAD_OK;
}

int sad_partition_plan(sad_ctx *ctx, const uint64_t *d_samples_all, int64_t *d_counts_out) {
    GUARD(4);
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
    CK(cudaMemcpyAsync(ctx->d_counts, d_counts_out, sizeof(int64_t) * (size_t)ctx->pl * p * 2,
                       cudaMemcpyDeviceToDevice, ctx->st));
    ctx->stage = 5;
    return SAD_OK;
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

int sad_pack(sad_ctx *ctx, const int64_t *h_counts_all, uint64_t *d_send_meta, uint8_t *d_send_res) {
    GUARD(5);
    if (!h_counts_all || !d_send_meta || !d_send_res) return fail(ctx, SAD_E_ARG, "sad_pack: NULL buffer");
    const int p = ctx->cfg.p;
    std::vector<int64_t> seg((size_t)ctx->pl * p * 2, 0);
    sad_pack_plan(p, ctx->cfg.world, ctx->cfg.rank, h_counts_all, seg.data());
    std::memcpy(ctx->h_small + 2048, seg.data(), seg.size() * sizeof(int64_t));
    CK(cudaMemcpyAsync(ctx->d_seg, ctx->h_small + 2048, seg.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->st));
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
    // the staging buffer is reused by later calls: make sure the copy has been consumed
    CK(cudaStreamSynchronize(ctx->st));
    return SAD_OK;
}

int sad_output_size(const sad_ctx *cctx, const int64_t *h_counts_all, size_t *bytes) {
    sad_ctx *ctx = const_cast<sad_ctx *>(cctx);
    GUARD(5);
    if ((!h_counts_all && ctx->cfg.world != 1) || !bytes) return SAD_E_ARG;
    int64_t n_out, r_out;
    sum_recv(ctx, h_counts_all, n_out, r_out);
    *bytes = out_layout(nullptr, n_out, r_out).total;
    return SAD_OK;
}

int sad_output_layout(const sad_ctx *cctx, const int64_t *h_counts_all, int64_t *h_layout) {
    sad_ctx *ctx = const_cast<sad_ctx *>(cctx);
    GUARD(5);
    if ((!h_counts_all && ctx->cfg.world != 1) || !h_layout) return SAD_E_ARG;
    int64_t n_out, r_out;
    sum_recv(ctx, h_counts_all, n_out, r_out);
    OutLayout o = out_layout(nullptr, n_out, r_out);
    h_layout[0] = n_out;
    h_layout[1] = r_out;
    h_layout[2] = (int64_t)reinterpret_cast<uintptr_t>(o.key);
    h_layout[3] = (int64_t)reinterpret_cast<uintptr_t>(o.off);
    h_layout[4] = (int64_t)reinterpret_cast<uintptr_t>(o.res);
    h_layout[5] = (int64_t)o.total;
    return SAD_OK;
}

int sad_finish(sad_ctx *ctx, const int64_t *h_counts_all, const uint64_t *d_recv_meta, const uint8_t *d_recv_res,
               void *d_out, size_t out_bytes, int64_t *h_bucket_sizes) {
    GUARD(5);
    const int p = ctx->cfg.p;
    if ((!h_counts_all && ctx->cfg.world != 1) || !d_out) return fail(ctx, SAD_E_ARG, "sad_finish: NULL buffer");
    if ((reinterpret_cast<uintptr_t>(d_out) & 255) != 0) return fail(ctx, SAD_E_ARG, "output must be 256-byte aligned");
    const bool local = d_recv_meta == nullptr;
    if (local && ctx->cfg.world != 1) return fail(ctx, SAD_E_ARG, "NULL receive buffers need world == 1");
    int64_t n_out, r_out;
    sum_recv(ctx, h_counts_all, n_out, r_out);
    if (local && h_counts_all && (n_out != ctx->n || r_out != ctx->R))
        return fail(ctx, SAD_E_STATE, "counts do not cover the input");
    OutLayout o = out_layout(reinterpret_cast<uint8_t *>(d_out), n_out, r_out);
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
        src_off = ctx->d_off;
        src_perm = ctx->d_perm_sorted;
        src_res = ctx->d_ascii;
    } else {                              // runs = the source shards, in rank (= shard) order
        if (n_out > 0 && (!d_recv_meta || (r_out > 0 && !d_recv_res)))
            return fail(ctx, SAD_E_ARG, "sad_finish: NULL receive buffer");
        int64_t *runs = reinterpret_cast<int64_t *>(ctx->h_small + 16384);
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
        if (n_out > 0) {
            size_t tb = o.cub_bytes;
            CK(cub::DeviceScan::ExclusiveSum(o.cub, tb, o.len_sorted, o.src_off, nn, ctx->st));
            LAUNCHED();
        }
        src_off = o.src_off;
        src_perm = nullptr;
        src_res = d_recv_res;
    }
    CK(cudaMemsetAsync(o.off, 0, sizeof(int64_t), ctx->st));
    if (n_out > 0) {
        launch_rank_merge(m, ctx->st);
        LAUNCHED();
        size_t tb = o.cub_bytes;
        CK(cub::DeviceScan::InclusiveSum(o.cub, tb, o.len_in, o.off + 1, nn, ctx->st));
        LAUNCHED();
        launch_gather_res(o.perm, src_perm, n_out, src_off, src_res, o.off, o.res, ctx->st);
        LAUNCHED();
    }
    ctx->d_out = reinterpret_cast<uint8_t *>(d_out);
    ctx->out_bytes = out_bytes;
    ctx->out_n = n_out;
    ctx->out_r = r_out;
    ctx->stage = 6;
    ctx->launches_last = ctx->launches_step;
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
    ctx->stage = 6;
    ctx->launches_last = ctx->launches_step;
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

static int resolve_counts(sad_ctx *ctx) {
    if (!ctx->counts_pending) return SAD_OK;
    CK(cudaStreamSynchronize(ctx->st));
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
    CK(cudaMemcpyAsync(h_T, ctx->d_T + b0, sizeof(uint64_t) * w, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return SAD_OK;
}

int sad_get_ancestors(sad_ctx *ctx, int64_t *h_local, int64_t *h_ga) {
    GUARD(4);
    const int p = ctx->cfg.p;
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
    std::vector<int32_t> t(w);
    CK(cudaMemcpyAsync(t.data(), ctx->d_perm_sorted + b0, 4 * w, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    for (int64_t i = 0; i < w; ++i) h_idx[i] = ctx->first_idx + t[i];
    return SAD_OK;
}

int sad_get_pivots(sad_ctx *ctx, uint64_t *h_pivots) {
    GUARD(5);
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
    OutLayout o = out_layout(ctx->d_out, ctx->out_n, ctx->out_r);
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
        if (h_idx) h_idx[i] = (int64_t)(keys[i] & 0x7FFFFFFFull);
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
    OutLayout o = out_layout(ctx->d_out, ctx->out_n, ctx->out_r);
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
    for (int s = 0; s < ctx->pl; ++s) {
        if (h_windows) h_windows[s] = ctx->h_windows[s];
        if (h_distinct) h_distinct[s] = ctx->h_distinct[s];
        if (h_kcols) h_kcols[s] = ctx->h_K[s];
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
