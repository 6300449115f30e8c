/*
 * sad.h — C ABI of libsad.so: the data-parallel hot path of Sample-Align-D
 * (Saeed & Khokhar, arXiv 0901.2742), the k-mer-rank domain decomposition, on
 * B200 (sm_100a).
 *
 * Citations: "P:n" = PAPER.md line n (the paper text), "S:n" = SPEC.md line n,
 * "reading Ann" = the interpretation table of SURVEY.md §8(c) / DESIGN.md §3.
 *
 * The calls follow the paper's problem statement:
 *   "Input <- N sequences"                       -> sad_load
 *   "Locally compute k-mer rank ..." (counts)     -> sad_build_profiles
 *   "... k-mer rank ... in each processor",
 *   local ancestor                                -> sad_rank_local
 *   "Send the k samples ... to all processors",
 *   "Compute the k-mer rank of each sequence ...",
 *   "Sort the sequences locally ...",
 *   "Using regular sampling, choose p-1 ..."      -> sad_rank_global
 *   "Sort all the p*(p-1) ranks ... p buckets",
 *   bucket boundaries                             -> sad_partition_plan
 *   "Redistributed sequences among processors"    -> sad_pack (send side) + sad_finish (receive side)
 *
 * TWO WAYS TO DRIVE ONE STEP
 *  - The collective API (the product path): sad_create with an NCCL unique id
 *    (sad_nccl_unique_id on rank 0, broadcast by the caller), then per step
 *        sad_load -> sad_build_profiles -> sad_rank -> sad_partition
 *    sad_rank and sad_partition are collective calls: the library owns an NCCL communicator and
 *    runs every exchange on cfg.stream itself (ncclAllGather of the ancestor records, of
 *    the regular samples and of the count matrix; grouped ncclSend/ncclRecv for the
 *    all-to-all personalized redistribution). With world == 1 the context
 *    needs no communicator (nccl_id == NULL: the exchanges are local); given one, the exchange
 *    steps still run through NCCL (to a single rank).
 *    For world == 1 the whole step runs without any host synchronization (it can be captured in
 *    one CUDA graph); for world > 1 sad_partition waits once, for the all-gathered count matrix
 *    that sizes the all-to-all.
 *  - The split API (stage by stage: sad_rank_local, sad_rank_global, sad_partition_plan,
 *    sad_pack, sad_finish): the caller moves the small exchange buffers between ranks itself
 *    (all-gather of ancestor records, of sample keys and of the count matrix, and the variable
 *    all-to-all of sequences), e.g. over torch.distributed; used for emulated ranks and tests.
 * Every byte of arithmetic of the method runs inside this library's CUDA kernels either way.
 *
 * CONVENTIONS (all calls)
 *  - Return 0 on success or a negative SAD_E_* code. No exception crosses the ABI.
 *  - Errors are sticky: after a failure every call except sad_last_error /
 *    sad_destroy returns SAD_E_STATE.
 *  - All device work is enqueued on cfg.stream (a cudaStream_t, may be NULL = legacy
 *    default stream). Calls return after enqueueing, except where "syncs" is stated.
 *  - Device pointers passed in ("d_" prefix) are owned by the caller, must stay valid
 *    until the stream has consumed them, and are never freed by the library. Host
 *    pointers ("h_" prefix) are read/written synchronously within the call.
 *  - Layouts are dense, row-major, little-endian; no padding unless stated.
 *  - The context is not thread-safe; one context per (process, GPU). Every call runs on
 *    cfg.device and leaves the caller's current device unchanged.
 *  - Device-detected input errors (SAD_E_SYMBOL, SAD_E_TOO_SHORT, SAD_E_TOO_LONG) and operand
 *    overflow (SAD_E_REPLAN) are found by the step's kernels and reported by the first call that
 *    synchronizes with the step: sad_partition (world > 1, or with h_bucket_sizes), a getter, or
 *    sad_rank_local of the split API.
 *  - SAD_E_REPLAN is not sticky: the all-pairs operand of this step was too small (its column
 *    capacity is chosen before the k-mer statistics are known, SURVEY Appendix A.1 bounds it by
 *    8 A^k for capped layers). The context has grown the capacity and returned to the "loaded"
 *    state: query sad_operand_size again and rerun the step from sad_build_profiles (all ranks
 *    receive the same code from a collective call).
 */
#ifndef SAD_H_
#define SAD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAD_ABI_VERSION 2u

/* alphabets ("sequences of amino acids"; DNA per BASELINE.json configs[4]).
 * Protein codes follow "ACDEFGHIKLMNPQRSTVWY", DNA "ACGT"; any other byte is an
 * illegal symbol (reading A18). */
#define SAD_PROTEIN20 0
#define SAD_DNA4 1

/* flags */
#define SAD_F_KEEP_SIM 1u     /* keep the w x w similarity numerators S_ij (uint16) of every shard */
#define SAD_F_KERNEL_ALU 2u   /* all-pairs on the CUDA-core min-sum (K5', dense uint16 count tiles) */
#define SAD_F_KERNEL_TC 4u    /* all-pairs on tcgen05 tensor cores (K5, threshold-indicator GEMM); default.
                                 Operands are packed e2m1 0/1 (kind::mxf4, unit block scales, fp32
                                 accumulators: exact below 2^24) unless SAD_F_TC_INT8 */
#define SAD_F_TC_INT8 8u      /* tensor-core path with uint8 0/1 operands (kind::i8, int32 accumulators) */
#define SAD_F_TC_1SM 16u      /* tensor-core path with one CTA per 128-row tile (default: CTA pairs,
                                 tcgen05 cta_group::2, 256-row tiles) */
#define SAD_F_RANK_SAMPLES 64u /* SURVEY §8(f) row f1, the paper's literal listing: rank every
                                 sequence by its mean fixed-point similarity to the k*p gathered samples
                                 (k = p-1 per shard, evenly spaced in the local order by T) instead of by
                                 its similarity to the global ancestor: by the exact sum T' = sum_s q
                                 (the mean's 1/(p(p-1)) is a common factor, reading A27), ties by index;
                                 key = (T' << sad_key_index_bits) + index (needs p(p-1) 2^32 N < 2^64).
                                 Needs p >= 2 and A^k <= 25600. sad_rank_local then
                                 writes p/world*(p-1) sample records instead of p/world ancestor records
                                 (sad_exchange_records) and sad_rank_global takes all p(p-1) of them. */
#define SAD_F_F1_CUDA_CORES 128u /* with SAD_F_RANK_SAMPLES: the rank against the samples on the CUDA cores
                                 (byte-SIMD min-sums over each row's CSR entries). Default with the fp4
                                 tensor-core kernel: the w x p(p-1) contraction of the shard's all-pairs
                                 operand with the samples' indicator rows on tcgen05 (the excess above
                                 the layer cap on the CUDA cores); both are exact. */
#define SAD_F_TILE_SPLIT 512u /* SURVEY §8(f) row f2 across GPUs (PAPER.md:103 centralized rank, "rows sharded
                                 over G"): every rank loads the SAME input (all N sequences, the profiles
                                 recomputed on every rank) and the p shards stay whole on every rank (p may
                                 be 1: the N x N all-pairs); the all-pairs tiles are split over the world
                                 ranks by row blocks (longest-processing-time greedy on tile counts, the
                                 same on every rank), K6 builds only the owned rows' excess, and T is summed
                                 over the ranks with one ncclAllReduce on the library's communicator right
                                 after the all-pairs kernel; everything after it is replicated (no exchange).
                                 Needs the tensor-core kernel, not SAD_F_KEEP_SIM. Without an NCCL id the
                                 reduction is skipped: T then holds this rank's partial sums only (the
                                 emulation used by the tests). */
#define SAD_F_TC_ALL_LAYERS 32u /* tensor-core path with every threshold layer t <= max n(tau) dense in the
                                 contraction. Default: the layers are capped per shard at the smallest
                                 T in {1,2,4,8} with max_i sum_tau (n_i(tau) - T)+ <= 255, and the
                                 remainder sum_tau min((n_i-T)+, (n_j-T)+) is added per pair from a
                                 sparse scatter (exact either way) */

/* memory kinds of sad_load inputs */
#define SAD_MEM_HOST 0
#define SAD_MEM_DEVICE 1
#define SAD_MEM_DEVICE_REBASE 2  /* device inputs whose offsets start at offsets[0] != 0 (ascii points
                                    at residue offsets[0]); e.g. a bucket view of sad_get_bucket_view */

/* error codes */
#define SAD_OK 0
#define SAD_E_ARG (-1)           /* bad k/p/alphabet/world/rank, p % world != 0, A^k > 65536, NULL pointer */
#define SAD_E_STATE (-2)         /* call order, or a sticky earlier error */
#define SAD_E_SYMBOL (-3)        /* illegal residue; first offender via sad_last_error / sad_error_location */
#define SAD_E_TOO_SHORT (-4)     /* a sequence with L < k (reading A19) */
#define SAD_E_TOO_LONG (-5)      /* a sequence with L - k + 1 > 65535 (the fixed-point proof) */
#define SAD_E_INSUFFICIENT (-6)  /* a shard with w < p (reading A16) */
#define SAD_E_EMPTY (-7)         /* n_global == 0 or a rank with no shard rows */
#define SAD_E_CAPACITY (-8)      /* a caller buffer is too small */
#define SAD_E_CUDA (-9)          /* CUDA runtime error (message in sad_last_error) */
#define SAD_E_NCCL (-10)         /* NCCL error, a peer rank failed (it called sad_abort or reported an
                                    input error in the count exchange), or the communicator was aborted */
#define SAD_E_OOM (-11)          /* workspace too small / host allocation failed */
#define SAD_E_REPLAN (-12)       /* the step's all-pairs operand capacity was exceeded: rerun (see above) */

typedef struct sad_config {
    int32_t alphabet;   /* SAD_PROTEIN20 | SAD_DNA4 */
    int32_t k;          /* k-mer length, >= 1, alphabet^k <= 65536 */
    int32_t p;          /* logical processors = shards = buckets (reading A21), >= 1 */
    int32_t world;      /* G: number of ranks (GPUs); p % world == 0 */
    int32_t rank;       /* this rank, 0..world-1; it owns shards rank*(p/world) .. (rank+1)*(p/world)-1
                           and buckets with the same indices */
    int32_t device;     /* CUDA device ordinal */
    void *stream;       /* cudaStream_t used for all work */
    uint32_t flags;     /* SAD_F_* */
} sad_config;

typedef struct sad_ctx sad_ctx;

/* Version of this header the library was built from. */
uint32_t sad_abi_version(void);

/* NCCL rendezvous id for sad_create (ncclGetUniqueId): call on rank 0 only and broadcast the 128
 * bytes to every rank (e.g. with torch.distributed.broadcast_object_list). */
int sad_nccl_unique_id(uint8_t *out128);

/* Create a context. Does not allocate device memory.
 *   nccl_id  NULL: no library communicator (world == 1 collective calls run locally; with
 *            world > 1 only the split API can be used); else the 128-byte id of
 *            sad_nccl_unique_id, and sad_create is COLLECTIVE over the world ranks
 *            (ncclCommInitRank on cfg.device). */
int sad_create(const sad_config *cfg, const uint8_t *nccl_id, sad_ctx **out);

/* Abort the context's communicator (ncclCommAbort) after a local failure, so that peers blocked
 * in a collective call return SAD_E_NCCL instead of hanging (replacing SPEC's
 * PeerDisconnected). The context is then in the sticky SAD_E_NCCL state. */
int sad_abort(sad_ctx *ctx);

/* Destroy a context (waits for its stream). NULL is a no-op. */
void sad_destroy(sad_ctx *ctx);

/* Human-readable description of the last error ("" if none). Valid until the next call. */
const char *sad_last_error(const sad_ctx *ctx);

/* For SAD_E_SYMBOL / SAD_E_TOO_SHORT / SAD_E_TOO_LONG: global source index of the first
 * offending sequence and (SYMBOL only) the 0-based residue position; -1 otherwise. */
int sad_error_location(const sad_ctx *ctx, int64_t *source_index, int64_t *position);

/* Bytes of device workspace sad_load needs for n_local sequences holding
 * residues_local residues on this rank. */
int sad_workspace_size(const sad_ctx *ctx, int64_t n_local, int64_t residues_local, size_t *bytes);

/*
 * sad_load — "Input <- N sequences ... Assume N/p sequences on each of the p processors"
 * (P:60). This rank's contiguous slice: sequences first_source_index ..
 * first_source_index + n_local - 1 of the global input, which must be exactly the rows of
 * this rank's p/world shards under the block split of reading A15 (the first N mod p shards
 * hold ceil(N/p) sequences, the rest floor(N/p)).
 *   ascii    [offsets[n_local]] residue bytes (host or device per mem)
 *   offsets  [n_local+1] int64, offsets[0] == 0, nondecreasing (host or device per mem)
 *   residues_local  offsets[n_local] if known, else -1 (device offsets are then read back,
 *            which costs a synchronization)
 *   mem      SAD_MEM_HOST (copied with cudaMemcpyAsync; synchronous w.r.t. the inputs; from
 *            4 MB on, the residues are copied in 4 chunks on an internal stream and each chunk's
 *            k-mer counts (the first part of sad_build_profiles) start as soon as it has landed,
 *            so pinned inputs overlap the PCIe copy with the counting),
 *            SAD_MEM_DEVICE (copied device-to-device on the stream) or SAD_MEM_DEVICE_REBASE
 *            (device, offsets[0] may be nonzero: offsets are taken relative to it)
 *   d_ws     device workspace of at least sad_workspace_size(n_local, offsets[n_local]) bytes,
 *            256-byte aligned, owned by the caller, kept until the next sad_load or sad_destroy.
 * Inputs are copied; no input pointer is retained. Syncs for host inputs (so they may be
 * reused on return) and when the shard layout changed; device inputs of a known size and
 * layout are copied asynchronously.
 */
int sad_load(sad_ctx *ctx, const uint8_t *ascii, const int64_t *offsets, int64_t n_local,
             int64_t first_source_index, int64_t n_global, int64_t residues_local, int32_t mem,
             void *d_ws, size_t ws_bytes);

/*
 * sad_build_profiles — k-mer count profiles n_x(tau) of every local sequence,
 * tau = sum_m c_m A^(k-1-m) over residue codes c. Validates symbols and lengths, builds the
 * per-sequence (tau, count) lists (unordered in tau; entries with count >= 2 first) and each
 * shard's statistics for the all-pairs stage, and the length order of every shard (rows sorted by
 * L - k + 1, ties in arbitrary order: no result depends on it). The per-shard layer cap T_s and
 * the operand width K_s are chosen on the device from those statistics;
 * nothing is read back: input errors surface at the step's first synchronizing call.
 */
int sad_build_profiles(sad_ctx *ctx);

/* Bytes of the all-pairs operand buffer sad_rank / sad_rank_local need (valid after
 * sad_build_profiles): [binary indicator rows of the context's column capacity | K6 lists |
 * K6 excess rows]. Host only. */
int sad_operand_size(const sad_ctx *ctx, size_t *bytes);

/*
 * sad_rank — COLLECTIVE (collective API). "Locally compute k-mer rank of all the sequences in each
 * processor", the local ancestors, "Send the k samples from each processor to all
 * the processors" (here the p/world ancestor records, ncclAllGather), the global ancestor
 * and "Compute the k-mer rank of each sequence against [it]", the local sort and the
 * regular samples: sad_rank_local + all-gather + sad_rank_global in one call on
 * cfg.stream (readings A5-A10). d_operand: >= sad_operand_size bytes, 1024-byte aligned,
 * caller-owned scratch. No host synchronization.
 */
int sad_rank(sad_ctx *ctx, void *d_operand, size_t operand_bytes);

/* Host logic of sad_partition's count exchange (pure host, no context; exposed for tests). From
 * the all-gathered count blocks of every rank (h_gathered = world x (p/world*p*2 + 4) int64: the
 * rank's [p/world][p][2] sequence/residue counts, then [operand overflow, first input-error kind
 * (1 symbol, 2 too short, 3 too long), output bytes, 0]) it takes the decision every rank takes:
 *   SAD_OK          exchange; h_counts_all ([p][p][2]) holds the count matrix
 *   SAD_E_NCCL      some rank has an input error (*who = the first, *kind its kind): nothing moves
 *   SAD_E_REPLAN    some rank's operand overflowed: every rank reruns the step
 *   SAD_E_CAPACITY  rank *who announced fewer output bytes than its buckets need
 * The inputs are identical on all ranks, so is the decision: no rank moves data alone. */
int sad_exchange_verdict(int32_t p, int32_t world, const int64_t *h_gathered, int64_t *h_counts_all, int32_t *who,
                         int32_t *kind);

/* Output bytes of sad_partition on this rank for ANY outcome of the partition (the buckets it
 * owns hold at most min(N, (p/world)(2w + p)) sequences, reading A23, and at most all
 * residues_global residues of the job); world == 1: exact (residues_global is ignored). */
int sad_output_bound(const sad_ctx *ctx, int64_t residues_global, size_t *bytes);

/*
 * sad_partition — COLLECTIVE (collective API). "Sort all the p*(p-1) ranks ... divide the range of
 * ranks into p buckets" (ncclAllGather of the regular samples, pivots replicated on every
 * rank, reading A14), bucket ranges (reading A13), the count exchange (ncclAllGather
 * of the [p][p][2] sequence/residue counts plus every rank's status), and "Redistributed sequences
 * among processors" (pack, grouped ncclSend/ncclRecv, receive-side merge): every
 * rank ends with its buckets, each in key order, in d_out.
 *   d_out / out_bytes  >= sad_output_bound bytes, 256-byte aligned; read with the getters
 *   h_bucket_sizes     [p] int64 out, sizes of ALL buckets (may be NULL when world == 1, then
 *                      nothing is read back and the call does not synchronize)
 * world > 1: synchronizes once (the count matrix sizes the all-to-all); if any rank reported an
 * input error, an operand overflow or a too small d_out, no data moves and every rank returns the
 * same kind of code (the failing rank its own, the others SAD_E_NCCL; SAD_E_REPLAN everywhere).
 */
int sad_partition(sad_ctx *ctx, void *d_out, size_t out_bytes, int64_t *h_bucket_sizes);

/* Bytes of one ancestor record: { int64 source_index; int32 L; int32 pad; uint16 counts[A^k] }
 * padded to 16 bytes. */
size_t sad_ancestor_record_bytes(const sad_ctx *ctx);

/* Index bits of the uint64 rank keys: key = (rank value << bits) + source index. 31 when ranking
 * against the GA (value floor(2^32 S/den) <= 2^32); with SAD_F_RANK_SAMPLES the bit
 * length of N - 1 (value = the exact fixed-point sum T' < p(p-1) 2^32, reading A27). Valid after
 * sad_load. */
int32_t sad_key_index_bits(const sad_ctx *ctx);

/* Records this rank contributes to the exchange after sad_rank_local (and that sad_rank_global
 * expects world times): p/world ancestor records, or p/world*(p-1) rank-sample records with
 * SAD_F_RANK_SAMPLES. Each record is sad_ancestor_record_bytes long. */
int32_t sad_exchange_records(const sad_ctx *ctx);

/*
 * SPLIT API (the caller moves the exchange buffers; see the top of this file).
 *
 * sad_rank_local — "Locally compute k-mer rank of all the sequences in each processor"
 * and the local ancestor (reading A6):
 *   S_ij = sum_tau min(n_i(tau), n_j(tau)),  den_ij = min(L_i, L_j) - k + 1   (reading A1)
 *   q_ij = floor(2^32 S_ij / den_ij),  T_i = sum_{j in shard} q_ij            (readings A3, A5)
 *   a_s  = argmax_{i in s} T_i, ties -> smaller source index                  (reading A6)
 *   d_operand  device buffer of >= sad_operand_size bytes (scratch, caller-owned)
 *   d_anc_out  device buffer of (p/world) ancestor records, this rank's shards in order
 * Split API only: waits for the step's k-mer statistics first and returns the input error or
 * SAD_E_REPLAN (operand capacity exceeded: query sad_operand_size again and call this again).
 */
int sad_rank_local(sad_ctx *ctx, void *d_operand, size_t operand_bytes, void *d_anc_out);

/*
 * sad_rank_global — global ancestor and rank against it (readings A7, A8, A9):
 *   d_anc_all   p ancestor records of ALL shards in shard order (the all-gather of every
 *               rank's d_anc_out; for world == 1 simply this rank's d_anc_out)
 *   GA = argmax_a U_a, U_a = sum_b q(a, b) over the p ancestors, ties -> smaller index
 *   S_i = S(x_i, GA), den_i = min(L_i, L_GA) - k + 1,
 *   key_i = (floor(2^32 S_i / den_i) << 31) + source_index_i  (uint64; SURVEY A.3 — orders
 *           exactly as "S_a den_b < S_b den_a, then smaller index")
 *   local sort of each shard by key, and p-1 regular samples per shard at 1-based
 *   positions floor(j w / p), j = 1..p-1 (reading A10)
 *   d_samples_out  (p/world)*(p-1) uint64 keys, shard-major
 */
int sad_rank_global(sad_ctx *ctx, const void *d_anc_all, uint64_t *d_samples_out);

/*
 * sad_partition_plan — pivots and bucket ranges (readings A11-A13):
 *   d_samples_all  p*(p-1) uint64 sample keys of ALL shards (the all-gather of every rank's
 *                  d_samples_out; for world == 1 this rank's d_samples_out)
 *   pivots = sorted samples at 1-based positions floor(p/2) + i p, i = 0..p-2
 *   bucket(x) = smallest b with key(x) <= pivot_b, else p-1
 *   d_counts_out   int64 [p/world][p][2]: for each local shard s and bucket b, the number of
 *                  sequences and of residues that shard s sends to bucket b
 */
int sad_partition_plan(sad_ctx *ctx, const uint64_t *d_samples_all, int64_t *d_counts_out);

/* Send/receive sizes of the all-to-all (pure host function, needs no GPU and no context),
 * derived from the counts of ALL ranks (h_counts_all = int64 [p][p][2], shard-major, the
 * all-gather of every rank's d_counts_out): for every peer rank r, the sequences and residue
 * bytes `rank` sends to r and receives from r. Rank r owns shards and buckets
 * r*(p/world) .. (r+1)*(p/world)-1. Returns SAD_E_ARG on bad p/world/rank. */
int sad_exchange_sizes(int32_t p, int32_t world, int32_t rank, const int64_t *h_counts_all,
                       int64_t *h_send_seqs, int64_t *h_send_res, int64_t *h_recv_seqs, int64_t *h_recv_res);

/* Send-buffer layout of `rank` (pure host function): h_seg = int64 [p/world][p][2], for each
 * local shard s and bucket b the sequence offset and the residue-byte offset of slice (s, b)
 * in the send buffers. Slices are grouped by destination rank, then ordered by (s, b). */
int sad_pack_plan(int32_t p, int32_t world, int32_t rank, const int64_t *h_counts_all, int64_t *h_seg);

/*
 * sad_pack — send side of "Redistributed sequences among processors":
 * writes this rank's sequences grouped by destination rank (rank r owns buckets
 * r*(p/world) .. (r+1)*(p/world)-1), each group ordered by (source shard, bucket, key).
 *   d_send_meta  [sum h_send_seqs][2] uint64: { key, L }
 *   d_send_res   [sum h_send_res] residue bytes (ASCII, as loaded)
 */
int sad_pack(sad_ctx *ctx, const int64_t *h_counts_all, uint64_t *d_send_meta, uint8_t *d_send_res);

/* Bytes of the output buffer sad_finish needs on this rank (host only): the received
 * sequences' keys, offsets and residues plus merge scratch. h_counts_all may be NULL when
 * world == 1 (the rank then receives exactly what it holds). */
int sad_output_size(const sad_ctx *ctx, const int64_t *h_counts_all, size_t *bytes);

/* Where sad_finish puts its results inside d_out: h_layout[0] = sequences n_out, [1] =
 * residues r_out, [2] = byte offset of uint64 keys[n_out], [3] = byte offset of int64
 * offsets[n_out+1], [4] = byte offset of residues[r_out], [5] = total bytes. Rows are the
 * owned buckets back to back in bucket order, each in key order. Host only. */
int sad_output_layout(const sad_ctx *ctx, const int64_t *h_counts_all, int64_t *h_layout);

/*
 * sad_finish — receive side: merges the received runs into this rank's buckets, each in key
 * order (SPEC D-P4 ordering), and reports all bucket sizes (load bound of P:188,
 * reading A23).
 *   d_recv_meta / d_recv_res  the all-to-all output laid out by source rank (sizes from
 *   sad_exchange_sizes). For world == 1 pass NULL for both: the local data is used in place.
 *   d_out / out_bytes  caller buffer of >= sad_output_size bytes, 256-byte aligned; it must
 *   stay valid while the getters below are used.
 *   h_counts_all may be NULL when world == 1: the counts then stay on the device and are read
 *   back lazily by the getters (no synchronization in the step).
 *   h_bucket_sizes  [p] int64 out (may be NULL): sizes of ALL buckets; with h_counts_all == NULL
 *   filling it synchronizes.
 * Does not sync otherwise.
 */
int sad_finish(sad_ctx *ctx, const int64_t *h_counts_all, const uint64_t *d_recv_meta,
               const uint8_t *d_recv_res, void *d_out, size_t out_bytes, int64_t *h_bucket_sizes);

/* ---- getters (sync; copy device results into caller host buffers) ---- */

/* Sizes of all p buckets (after sad_finish; P:188 load report). */
int sad_get_bucket_sizes(sad_ctx *ctx, int64_t *h_sizes);

/*
 * sad_get_load_report — SURVEY §8(a) row a12, the load bound of the regular-sampling partition
 * ("all the data to be aligned by processor 1 must be <= y1 ... the upper bound on the number of
 * sequences that a processor will receive is less than 2w"
 * check_load_bound). Under the sampling rule of readings A10/A11 the bound that always holds is
 * max bucket <= 2w + p, and max bucket < 2w when p divides w (reading A23).
 * After sad_finish; syncs like the other getters. h_report (int64 [6]):
 *   [0] largest bucket  [1] w = largest shard (ceil(N/p))  [2] 2w + p
 *   [3] 1 if [0] <= 2w + p   [4] 1 if p divides every shard size w   [5] 1 if [0] < 2w
 */
int sad_get_load_report(sad_ctx *ctx, int64_t *h_report);

/* T_i (uint64) of every sequence of local shard s (0 <= s < p/world), in input order. */
int sad_get_local_rank(sad_ctx *ctx, int shard, uint64_t *h_T, int64_t cap);

/* Local ancestors of ALL p shards and the GA, as global source indices (after sad_rank_global). */
int sad_get_ancestors(sad_ctx *ctx, int64_t *h_local, int64_t *h_ga);

/* S_i, den_i and key_i of every sequence of local shard s, in input order (after sad_rank_global).
 * With SAD_F_RANK_SAMPLES: S_i = T'_i mod 2^32 and den_i = T'_i >> 32 (T' the rank sum, A27). */
int sad_get_ranks(sad_ctx *ctx, int shard, uint32_t *h_S, uint32_t *h_den, uint64_t *h_key, int64_t cap);

/* Source indices of local shard s in its local sort order (after sad_rank_global). */
int sad_get_sorted(sad_ctx *ctx, int shard, int64_t *h_idx, int64_t cap);

/* The p-1 pivot keys (after sad_partition_plan). */
int sad_get_pivots(sad_ctx *ctx, uint64_t *h_pivots);

/* One bucket owned by this rank (after sad_finish): source indices, keys, residues (ASCII)
 * and offsets[n+1] (relative to the bucket's first residue). cap_seqs is the capacity of
 * h_idx / h_key (>= n) and of h_offsets (>= n + 1 when h_offsets is given); cap_res that of
 * h_res. Returns SAD_E_CAPACITY if a cap is too small; *n_out / *res_out receive the sizes in
 * any case. Any output may be NULL. */
int sad_get_bucket(sad_ctx *ctx, int bucket, int64_t *h_idx, uint64_t *h_key, uint8_t *h_res,
                   int64_t *h_offsets, int64_t cap_seqs, int64_t cap_res, int64_t *n_out, int64_t *res_out);

/* The w x w similarity numerators S_ij of local shard s (uint16, row-major, input order);
 * only with SAD_F_KEEP_SIM. */
int sad_get_similarity(sad_ctx *ctx, int shard, uint16_t *h_S, int64_t cap);

/* Device view of one bucket owned by this rank (after sad_finish), for feeding it to another
 * context with sad_load(..., SAD_MEM_DEVICE_REBASE): *d_res = its first residue, *d_offsets =
 * its n+1 residue offsets (absolute inside this context's output; rebase by offsets[0]),
 * *n = sequences, *res_bytes = residues. The pointers stay valid until the next sad_finish
 * or sad_destroy of this context. Syncs (reads one offset). */
int sad_get_bucket_view(sad_ctx *ctx, int bucket, const uint8_t **d_res, const int64_t **d_offsets, int64_t *n,
                        int64_t *res_bytes);

/* Distance matrix of local shard s (SPEC S:347-352 build_distance_matrix,
 * PAPER.md:52 "k-mer distance can be used to rapidly construct phylogenetic trees"):
 * d_D[i][j] = 1 - S_ij / (min(L_i, L_j) - k + 1) in IEEE float32 (fdiv_rn then fsub_rn), 0 on
 * the diagonal, w x w row-major in input order, device memory of >= cap floats. Needs
 * SAD_F_KEEP_SIM and sad_rank_local; enqueued on the stream. */
int sad_get_distance(sad_ctx *ctx, int shard, float *d_D, int64_t cap);

/* The same distances in IEEE float64 (__ddiv_rn then __dsub_rn), the input of sad_upgma. */
int sad_get_distance_f64(sad_ctx *ctx, int shard, double *d_D, int64_t cap);

/*
 * sad_upgma — SURVEY §8(f) row f4: the UPGMA guide tree of n sequences (the first
 * stage of the per-bucket progressive aligner). Context-free, enqueued on `stream`.
 *   d_D        n x n float64 distances (device); only the upper triangle is read; DESTROYED
 *   d_merges   [n-1][2] int64 out: step t joins the clusters with these ids (leaves 0..n-1, the
 *              cluster of step t is n + t); the first id is the cluster at the smaller position
 *   d_heights  [n-1] float64 out: join height d/2
 *   d_sizes    [n-1] int64 out: leaves under the new cluster
 *   d_ws       >= sad_upgma_workspace(n) bytes, 256-byte aligned
 * Rules: closest active pair (i < j) by position, ties -> smallest i then j (D-M1); a cluster lives
 * at its smallest leaf's position; average linkage (n_i d(k,i) + n_j d(k,j)) / (n_i + n_j) with
 * each IEEE float64 operation rounded once. n == 1: nothing to do. One thread block; O(n^2) work
 * per merge in the worst case, O(n) typically.
 */
size_t sad_upgma_workspace(int64_t n);
int sad_upgma(double *d_D, int64_t n, int64_t *d_merges, double *d_heights, int64_t *d_sizes, void *d_ws,
              size_t ws_bytes, void *stream);

/* Per-shard profile facts (after sad_build_profiles): total k-mer windows, distinct k-mers
 * and the operand column count K_s of every local shard (int64 [p/world] each; any may be NULL). */
int sad_get_profile_info(sad_ctx *ctx, int64_t *h_windows, int64_t *h_distinct, int64_t *h_kcols);

/* Device times of the all-pairs kernel (K5/K5') summed over all sad_rank_local calls since the
 * last reset, and the number of such calls; h_ms[0] = all-pairs kernel ms, h_ms[1] = operand
 * build ms, h_counts[0] = calls, h_counts[1] = unordered pairs i<j per call, h_counts[2] =
 * dense operand MACs per call (sum_s w_s(w_s+1)/2 * K_s), h_counts[3] = kernel launches of the
 * last full step (load..finish). Syncs. */
int sad_get_stats(sad_ctx *ctx, double *h_ms, int64_t *h_counts);

/* A step captured into a CUDA graph (stream capture of sad_load .. sad_partition on cfg.stream,
 * world == 1 without a communicator) records its stage events as external event nodes; after
 * each replay has completed, this adds that replay's operand-build and all-pairs kernel times to
 * the sad_get_stats totals (and counts one call), and makes the getters read the replay's
 * results. Syncs. */
int sad_graph_account(sad_ctx *ctx);
int sad_reset_stats(sad_ctx *ctx);

/* Exhaustive self-test of the device fixed-point division q = floor(2^32 S / den)
 * (SURVEY A.3 / reading A5) for every den in [1, max_den] and S in [0, den], against
 * 64-bit integer division on the device. Returns the number of mismatches in *h_bad. Syncs. */
int sad_selftest_fixed_point(sad_ctx *ctx, int32_t max_den, int64_t *h_bad);

#ifdef __cplusplus
}
#endif

#endif /* SAD_H_ */
