/*
 * sad_oracle.c — CPU ORACLE for the Sample-Align-D k-mer-rank domain decomposition.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` leg may load or run this code. The product
 * (paper_0901_2742_b200/, libsad.so) never links, imports or calls it, and shares
 * no code, header, table or helper with it.
 *
 * It is plain, slow and meant to be checked against the paper by eye. Every step
 * follows PAPER.md (arXiv 0901.2742, Saeed & Khokhar) in the paper's order and
 * notation; the readings of ambiguous passages are listed in DESIGN.md §3 and
 * SURVEY.md §8(c) (A1..A26) and are cited as "reading Ann" below.
 *
 * Arithmetic is exact integer arithmetic throughout; floating point is used only
 * for the reported R_i = ln(0.1 + D_i) values, which never decide anything.
 *
 * k-mers are handled as STRINGS (windows of k residues compared with memcmp),
 * never as integer codes, so nothing here can share a bug with the GPU's
 * base-A window codes.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_E_ARG (-1)
#define OR_E_SYMBOL (-3)
#define OR_E_TOO_SHORT (-4)
#define OR_E_TOO_LONG (-5)
#define OR_E_INSUFFICIENT (-6)
#define OR_E_EMPTY (-7)
#define OR_E_OOM (-11)

int or_abi(void) { return 5; }

/* ---------------------------------------------------------------------------
 * Input alphabet ("Input <- N sequences of amino acids x1 ... xN";
 * DNA added by BASELINE.json configs[4]). Non-canonical symbols are rejected
 * (reading A18).
 * ------------------------------------------------------------------------- */
static const char *ALPHA[2] = {"ACDEFGHIKLMNPQRSTVWY", "ACGT"};

static int is_member(int alphabet, uint8_t c) {
    return c != 0 && strchr(ALPHA[alphabet], (int)c) != NULL;
}

/* ---------------------------------------------------------------------------
 * k-mer counts nx(tau)  (§2 "k-mer Rank": "A k-mer is a
 * contiguous subsequence of length k ... nx_i(tau) ... are the number of times
 * tau occurs in x_i").
 *
 * Representation: the L-k+1 window start positions sorted lexicographically by
 * the k residues they cover, then run-length grouped: distinct k-mer = one run.
 * ------------------------------------------------------------------------- */
typedef struct {
    const uint8_t *x;   /* residues of the sequence */
    int64_t d;          /* number of distinct k-mers */
    int64_t *pos;       /* d entries: a start position of each distinct k-mer, sorted by k-mer */
    int64_t *cnt;       /* d entries: nx(tau) */
} kcounts;

static const uint8_t *g_sort_x;   /* qsort has no context argument; the sort below is per-sequence */
static int g_sort_k;
#ifdef _OPENMP
#pragma omp threadprivate(g_sort_x, g_sort_k)
#endif

static int cmp_window(const void *a, const void *b) {
    int64_t pa = *(const int64_t *)a, pb = *(const int64_t *)b;
    int c = memcmp(g_sort_x + pa, g_sort_x + pb, (size_t)g_sort_k);
    if (c) return c;
    return (pa > pb) - (pa < pb);
}

/* Fills kc; returns 0 or OR_E_OOM. Requires L >= k. */
static int count_kmers(const uint8_t *x, int64_t L, int k, kcounts *kc) {
    int64_t nw = L - k + 1;                         /* number of windows */
    int64_t *w = (int64_t *)malloc(sizeof(int64_t) * (size_t)nw);
    if (!w) return OR_E_OOM;
    for (int64_t i = 0; i < nw; ++i) w[i] = i;
    g_sort_x = x; g_sort_k = k;
    qsort(w, (size_t)nw, sizeof(int64_t), cmp_window);
    kc->x = x;
    kc->pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)nw);
    kc->cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)nw);
    if (!kc->pos || !kc->cnt) { free(w); return OR_E_OOM; }
    int64_t d = 0;
    for (int64_t i = 0; i < nw; ++i) {
        if (d > 0 && memcmp(x + kc->pos[d - 1], x + w[i], (size_t)k) == 0) {
            kc->cnt[d - 1] += 1;
        } else {
            kc->pos[d] = w[i];
            kc->cnt[d] = 1;
            ++d;
        }
    }
    kc->d = d;
    free(w);
    return OR_OK;
}

static void free_counts(kcounts *kc) { free(kc->pos); free(kc->cnt); kc->pos = kc->cnt = NULL; }

/* ---------------------------------------------------------------------------
 * Similarity numerator S(x,y) = sum_tau min[nx(tau), ny(tau)]
 * (the displayed r_ij formula, with the stray tau factor dropped
 * — reading A1). Computed by merging the two k-mer-sorted count lists.
 * ------------------------------------------------------------------------- */
static int64_t min_sum(const kcounts *a, const kcounts *b, int k) {
    int64_t i = 0, j = 0, s = 0;
    while (i < a->d && j < b->d) {
        int c = memcmp(a->x + a->pos[i], b->x + b->pos[j], (size_t)k);
        if (c == 0) {
            s += a->cnt[i] < b->cnt[j] ? a->cnt[i] : b->cnt[j];
            ++i; ++j;
        } else if (c < 0) {
            ++i;
        } else {
            ++j;
        }
    }
    return s;
}

/* Denominator of r_ij: min(|x_i|, |x_j|) - k + 1. */
static int64_t den_of(int64_t Li, int64_t Lj, int k) { return (Li < Lj ? Li : Lj) - k + 1; }

/* Fixed-point pair term q = floor(2^32 * S / den)  (reading A5: D_i = (1/N) sum_j r_ij,
 * PAPER.md:46, summed exactly in 32.32 fixed point; 1/N is a common factor and
 * cannot change any comparison). S <= den < 2^16 so S<<32 < 2^48 fits uint64. */
uint64_t or_q(uint64_t S, uint64_t den) { return (S << 32) / den; }

/* ---------------------------------------------------------------------------
 * Exported helpers for pin tests
 * ------------------------------------------------------------------------- */

/* k-mer multiset of one sequence: out_pos[d] (a start position per distinct
 * k-mer, in lexicographic k-mer order) and out_cnt[d]; returns d or < 0. */
int64_t or_count(const uint8_t *x, int64_t L, int k, int64_t *out_pos, int64_t *out_cnt) {
    if (k < 1 || L < k) return OR_E_TOO_SHORT;
    kcounts kc;
    int rc = count_kmers(x, L, k, &kc);
    if (rc) return rc;
    for (int64_t i = 0; i < kc.d; ++i) { out_pos[i] = kc.pos[i]; out_cnt[i] = kc.cnt[i]; }
    int64_t d = kc.d;
    free_counts(&kc);
    return d;
}

/* S and den of one pair. */
int or_pair(const uint8_t *x, int64_t Lx, const uint8_t *y, int64_t Ly, int k, int64_t *S, int64_t *den) {
    if (k < 1 || Lx < k || Ly < k) return OR_E_TOO_SHORT;
    kcounts a, b;
    if (count_kmers(x, Lx, k, &a)) return OR_E_OOM;
    if (count_kmers(y, Ly, k, &b)) { free_counts(&a); return OR_E_OOM; }
    *S = min_sum(&a, &b, k);
    *den = den_of(Lx, Ly, k);
    free_counts(&a); free_counts(&b);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * The pipeline.
 * ------------------------------------------------------------------------- */

/* Rank order of reading A9 / SURVEY O7: a < b  <=>  S_a/den_a < S_b/den_b as exact
 * rationals (64-bit cross-multiplication; all factors < 2^16), ties broken by the
 * smaller source index. */
typedef struct { int64_t S, den, idx; } rkey;

static int rkey_less(const rkey *a, const rkey *b) {
    int64_t l = a->S * b->den, r = b->S * a->den;
    if (l != r) return l < r;
    return a->idx < b->idx;
}

static int cmp_rkey(const void *a, const void *b) {
    const rkey *x = (const rkey *)a, *y = (const rkey *)b;
    if (rkey_less(x, y)) return -1;
    if (rkey_less(y, x)) return 1;
    return 0;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/*
 * or_run — Sample-Align-D steps "Assume N/p sequences on each of the p processors"
 * through "Redistributed sequences among processors", with the
 * readings of SURVEY.md §8(c) (O1-O12).
 *
 * Inputs: ascii/offsets (n sequences, source_index = input order), alphabet
 * (0 protein, 1 DNA), k, p, nthreads (<=0: library default).
 * Outputs (caller-allocated, any may be NULL):
 *   T[n]          u64  per-sequence within-shard fixed-point sum  T_i = sum_j q_ij  (O4)
 *   anc[p]        i64  local ancestor of each shard                                  (O5)
 *   ga[1]         i64  global ancestor                                              (O6)
 *   Sg[n], dg[n]  i64  S(x_i, GA) and den(x_i, GA)                                  (O7)
 *   sorted[n]     i64  source indices, each shard sorted by the O7 order, shards in order (O8)
 *   samples[p(p-1)] i64 regular samples (source indices), shard-major               (O8)
 *   pivots[p-1]   i64  pivot sequences (source indices)                              (O9)
 *   bucket[n]     i64  bucket of each sequence                                       (O10)
 *   border[n]     i64  source indices bucket by bucket, each bucket in O7 order      (O11)
 *   bsize[p]      i64  bucket sizes                                                  (O11)
 *   stage_ms[4]   f64  wall ms: counts, all-pairs, ancestors+ranks, partition
 * Returns 0, or a negative error code; *err_idx / *err_pos locate the first
 * offending sequence / residue when not NULL.
 */
/* Local order of reading f1 ("Sort the sequences locally in each processor based
 * on k-mer rank"): ascending local rank T, ties by the smaller source index. */
typedef struct { uint64_t T; int64_t idx; } tkey;

static int cmp_tkey(const void *a, const void *b) {
    const tkey *x = (const tkey *)a, *y = (const tkey *)b;
    if (x->T != y->T) return x->T < y->T ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

int or_run2(const uint8_t *ascii, const int64_t *offsets, int64_t n, int alphabet, int k, int p, int mode,
            int nthreads, uint64_t *T, int64_t *anc, int64_t *ga, int64_t *Sg, int64_t *dg, int64_t *sorted,
            int64_t *samples, int64_t *pivots, int64_t *bucket, int64_t *border, int64_t *bsize,
            int64_t *rsamples, double *stage_ms, int64_t *err_idx, int64_t *err_pos);

int or_run(const uint8_t *ascii, const int64_t *offsets, int64_t n, int alphabet, int k, int p, int nthreads,
           uint64_t *T, int64_t *anc, int64_t *ga, int64_t *Sg, int64_t *dg, int64_t *sorted,
           int64_t *samples, int64_t *pivots, int64_t *bucket, int64_t *border, int64_t *bsize,
           double *stage_ms, int64_t *err_idx, int64_t *err_pos) {
    return or_run2(ascii, offsets, n, alphabet, k, p, 0, nthreads, T, anc, ga, Sg, dg, sorted, samples, pivots,
                   bucket, border, bsize, NULL, stage_ms, err_idx, err_pos);
}

/* mode 0: rank against the global ancestor (readings A7, A8 — the north star's path).
 * mode 1: the paper's literal listing: the
 *   k = p-1 rank samples of every shard are the sequences at the evenly spaced positions of its
 *   local order, and every sequence is ranked by its mean fixed-point similarity to the
 *   m = p(p-1) gathered samples, D_i = (1/m) sum_s r(x_i, s) (PAPER.md:46 with the samples as
 *   the reference set), carried as the exact fixed-point sum T'_i = sum_s q(x_i, s) (reading A5;
 *   the common factor 1/m is dropped exactly as A5 drops 1/N, reading A27); the rank order is
 *   (T', index); Sg/dg report (T', 1), ga = -1, and rsamples[m] the
 *   rank samples (source indices). Needs p >= 2. */
int or_run2(const uint8_t *ascii, const int64_t *offsets, int64_t n, int alphabet, int k, int p, int mode,
            int nthreads, uint64_t *T, int64_t *anc, int64_t *ga, int64_t *Sg, int64_t *dg, int64_t *sorted,
            int64_t *samples, int64_t *pivots, int64_t *bucket, int64_t *border, int64_t *bsize,
            int64_t *rsamples, double *stage_ms, int64_t *err_idx, int64_t *err_pos) {
    if (alphabet < 0 || alphabet > 1 || k < 1 || p < 1 || mode < 0 || mode > 1) return OR_E_ARG;
    if (mode == 1 && p < 2) return OR_E_ARG;
    if (n <= 0) return OR_E_EMPTY;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    double t0 = now_ms();

    /* O1: validate the alphabet and L >= k (and L-k+1 < 2^16, which the
     * fixed-point argument of reading A5 relies on). */
    for (int64_t i = 0; i < n; ++i) {
        int64_t L = offsets[i + 1] - offsets[i];
        for (int64_t t = 0; t < L; ++t) {
            if (!is_member(alphabet, ascii[offsets[i] + t])) {
                if (err_idx) *err_idx = i;
                if (err_pos) *err_pos = t;
                return OR_E_SYMBOL;
            }
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        int64_t L = offsets[i + 1] - offsets[i];
        if (L < k) { if (err_idx) *err_idx = i; return OR_E_TOO_SHORT; }
        if (L - k + 1 > 65535) { if (err_idx) *err_idx = i; return OR_E_TOO_LONG; }
    }

    /* O3: p contiguous shards; the first n mod p get ceil(n/p) (reading A15). */
    int64_t *sb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(p + 1));
    sb[0] = 0;
    for (int s = 0; s < p; ++s) sb[s + 1] = sb[s] + n / p + (s < n % p ? 1 : 0);
    for (int s = 0; s < p; ++s)
        if (sb[s + 1] - sb[s] < p) { free(sb); return OR_E_INSUFFICIENT; }   /* reading A16: w >= p */

    /* O2: k-mer counts of every sequence. */
    kcounts *kc = (kcounts *)calloc((size_t)n, sizeof(kcounts));
    int fail = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(| : fail)
    for (int64_t i = 0; i < n; ++i)
        fail |= count_kmers(ascii + offsets[i], offsets[i + 1] - offsets[i], k, &kc[i]) != 0;
    if (fail) return OR_E_OOM;
    double t1 = now_ms();

    /* O4: "Locally compute k-mer rank of all the sequences in each processor"
     * (PAPER.md:67): for every pair in a shard S_ij, den_ij, q_ij, and
     * T_i = sum_{j in shard} q_ij, self term included (reading A3). */
    uint64_t *Tl = (uint64_t *)calloc((size_t)n, sizeof(uint64_t));
    for (int s = 0; s < p; ++s) {
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t i = sb[s]; i < sb[s + 1]; ++i) {
            uint64_t acc = 0;
            int64_t Li = offsets[i + 1] - offsets[i];
            for (int64_t j = sb[s]; j < sb[s + 1]; ++j) {
                int64_t Lj = offsets[j + 1] - offsets[j];
                acc += or_q((uint64_t)min_sum(&kc[i], &kc[j], k), (uint64_t)den_of(Li, Lj, k));
            }
            Tl[i] = acc;
        }
    }
    double t2 = now_ms();

    /* O5: local ancestor a_s = argmax_{i in s} T_i, ties -> smallest source index
     * (reading A6: the shard medoid stands in for the alignment-derived "Local
     * Ancestor" of PAPER.md:79). */
    int64_t *a = (int64_t *)malloc(sizeof(int64_t) * (size_t)p);
    for (int s = 0; s < p; ++s) {
        int64_t best = sb[s];
        for (int64_t i = sb[s] + 1; i < sb[s + 1]; ++i)
            if (Tl[i] > Tl[best]) best = i;
        a[s] = best;
    }

    /* O6: global ancestor among the gathered local ancestors (
     * reading A7): U_a = sum_b q(a, b); GA = argmax U, ties -> smallest index. */
    int64_t g = -1;
    uint64_t bestU = 0;
    for (int s = 0; s < p; ++s) {
        uint64_t U = 0;
        int64_t ia = a[s], La = offsets[ia + 1] - offsets[ia];
        for (int t = 0; t < p; ++t) {
            int64_t ib = a[t], Lb = offsets[ib + 1] - offsets[ib];
            U += or_q((uint64_t)min_sum(&kc[ia], &kc[ib], k), (uint64_t)den_of(La, Lb, k));
        }
        if (g < 0 || U > bestU || (U == bestU && ia < g)) { g = ia; bestU = U; }
    }

    /* O7: "Compute the k-mer rank of each sequence against the k*p samples"
     * read as: against the global ancestor (reading A8):
     * S_i = S(x_i, GA), den_i = min(L_i, L_GA) - k + 1. */
    rkey *rk = (rkey *)malloc(sizeof(rkey) * (size_t)n);
    if (mode == 0) {
        int64_t Lg = offsets[g + 1] - offsets[g];
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            rk[i].S = min_sum(&kc[i], &kc[g], k);
            rk[i].den = den_of(offsets[i + 1] - offsets[i], Lg, k);
            rk[i].idx = i;
        }
    } else {
        /* f1, "Sort the sequences locally in each processor based on k-mer rank",
         * :69 "Choose a sample set of k sequences in each processor" (k = p-1 at the evenly
         * spaced 1-based positions floor(j*w/p), readings A10, A20), :70 "Send the k samples
         * from each processor to all the processors", :72 "Compute the k-mer rank of each
         * sequence against the k*p samples": T'_i = sum_s q(x_i, s), ordered exactly (A27). */
        int64_t m = (int64_t)p * (p - 1);
        int64_t *rs = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
        tkey *tk = (tkey *)malloc(sizeof(tkey) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) { tk[i].T = Tl[i]; tk[i].idx = i; }
        for (int s = 0; s < p; ++s) {
            int64_t w = sb[s + 1] - sb[s];
            qsort(tk + sb[s], (size_t)w, sizeof(tkey), cmp_tkey);
            for (int j = 1; j <= p - 1; ++j) rs[(int64_t)s * (p - 1) + (j - 1)] = tk[sb[s] + (j * w) / p - 1].idx;
        }
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            uint64_t acc = 0;
            int64_t Li = offsets[i + 1] - offsets[i];
            for (int64_t t = 0; t < m; ++t) {
                int64_t j = rs[t], Lj = offsets[j + 1] - offsets[j];
                acc += or_q((uint64_t)min_sum(&kc[i], &kc[j], k), (uint64_t)den_of(Li, Lj, k));
            }
            rk[i].S = (int64_t)acc;      /* T'_i < m 2^32 + 1: the cross products below stay < 2^63 */
            rk[i].den = 1;
            rk[i].idx = i;
        }
        if (rsamples) memcpy(rsamples, rs, sizeof(int64_t) * (size_t)m);
        free(rs);
        free(tk);
        g = -1;
    }
    double t3 = now_ms();

    /* O8: "Sort the sequences locally in each processor based on the new k-mer
     * rank", then p-1 evenly spaced samples at 1-based positions
     * floor(j*w/p), j = 1..p-1 (reading A10). */
    rkey *srt = (rkey *)malloc(sizeof(rkey) * (size_t)n);
    memcpy(srt, rk, sizeof(rkey) * (size_t)n);
    int64_t np1 = (int64_t)p * (p - 1);
    rkey *Y = (rkey *)malloc(sizeof(rkey) * (size_t)(np1 > 0 ? np1 : 1));
    for (int s = 0; s < p; ++s) {
        int64_t w = sb[s + 1] - sb[s];
        qsort(srt + sb[s], (size_t)w, sizeof(rkey), cmp_rkey);
        for (int j = 1; j <= p - 1; ++j)
            Y[(int64_t)s * (p - 1) + (j - 1)] = srt[sb[s] + (j * w) / p - 1];
    }

    /* O9: "Sort all the p*(p-1) ranks at the root processors and divide the range
     * of ranks into p buckets": pivots Y_{p/2}, Y_{p+p/2}, ... i.e.
     * 1-based positions floor(p/2) + i*p, i = 0..p-2 (reading A11). */
    if (samples)
        for (int64_t t = 0; t < np1; ++t) samples[t] = Y[t].idx;
    qsort(Y, (size_t)np1, sizeof(rkey), cmp_rkey);
    rkey *pv = (rkey *)malloc(sizeof(rkey) * (size_t)(p > 1 ? p - 1 : 1));
    for (int i = 0; i + 1 < p; ++i) pv[i] = Y[p / 2 + (int64_t)i * p - 1];

    /* O10: bucket(x) = smallest b with x <= pivot_b, else p-1 ("all the data to be
     * aligned by processor 1 must be <= y1"; readings A12, A13). */
    int64_t *bk = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *cnt = (int64_t *)calloc((size_t)p, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        int b = p - 1;
        for (int t = 0; t + 1 < p; ++t)
            if (!rkey_less(&pv[t], &rk[i])) { b = t; break; }
        bk[i] = b;
        cnt[b] += 1;
    }

    /* O11: "Redistributed sequences among processors such that sequences with
     * k-mer rank in the range of bucket i are accumulated at processor i"
     * (PAPER.md:77): each bucket in the O7 order. */
    rkey *bo = (rkey *)malloc(sizeof(rkey) * (size_t)n);
    int64_t *fill = (int64_t *)calloc((size_t)p + 1, sizeof(int64_t));
    for (int b = 0; b < p; ++b) fill[b + 1] = fill[b] + cnt[b];
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)p);
    for (int b = 0; b < p; ++b) cur[b] = fill[b];
    for (int64_t i = 0; i < n; ++i) bo[cur[bk[i]]++] = rk[i];
    for (int b = 0; b < p; ++b) qsort(bo + fill[b], (size_t)cnt[b], sizeof(rkey), cmp_rkey);
    double t4 = now_ms();

    /* O12: outputs */
    if (T) memcpy(T, Tl, sizeof(uint64_t) * (size_t)n);
    if (anc) memcpy(anc, a, sizeof(int64_t) * (size_t)p);
    if (ga) *ga = g;
    for (int64_t i = 0; i < n; ++i) {
        if (Sg) Sg[i] = rk[i].S;
        if (dg) dg[i] = rk[i].den;
        if (sorted) sorted[i] = srt[i].idx;
        if (bucket) bucket[i] = bk[i];
        if (border) border[i] = bo[i].idx;
    }
    if (pivots) for (int i = 0; i + 1 < p; ++i) pivots[i] = pv[i].idx;
    if (bsize) memcpy(bsize, cnt, sizeof(int64_t) * (size_t)p);
    if (stage_ms) { stage_ms[0] = t1 - t0; stage_ms[1] = t2 - t1; stage_ms[2] = t3 - t2; stage_ms[3] = t4 - t3; }

    for (int64_t i = 0; i < n; ++i) free_counts(&kc[i]);
    free(kc); free(Tl); free(a); free(rk); free(srt); free(Y); free(pv); free(bk); free(cnt);
    free(bo); free(fill); free(cur); free(sb);
    return OR_OK;
}

/*
 * or_rows_T — T_i for selected rows only (the O4 sum for one row at a time), for
 * sampled parity checks at sizes where the full O(w^2) oracle is too slow.
 * rows[m] are source indices; shard bounds follow O3.
 */
int or_rows_T(const uint8_t *ascii, const int64_t *offsets, int64_t n, int k, int p,
              const int64_t *rows, int64_t m, int nthreads, uint64_t *T_out) {
    if (n <= 0 || p < 1) return OR_E_ARG;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int64_t *sb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(p + 1));
    sb[0] = 0;
    for (int s = 0; s < p; ++s) sb[s + 1] = sb[s] + n / p + (s < n % p ? 1 : 0);
    int fail = 0;
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = rows[r];
        int s = 0;
        while (!(i >= sb[s] && i < sb[s + 1])) ++s;
        kcounts ki;
        if (count_kmers(ascii + offsets[i], offsets[i + 1] - offsets[i], k, &ki)) { fail = 1; break; }
        int64_t Li = offsets[i + 1] - offsets[i];
        uint64_t acc = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : acc) reduction(| : fail)
        for (int64_t j = sb[s]; j < sb[s + 1]; ++j) {
            kcounts kj;
            int64_t Lj = offsets[j + 1] - offsets[j];
            if (count_kmers(ascii + offsets[j], Lj, k, &kj)) { fail = 1; continue; }
            acc += or_q((uint64_t)min_sum(&ki, &kj, k), (uint64_t)den_of(Li, Lj, k));
            free_counts(&kj);
        }
        free_counts(&ki);
        T_out[r] = acc;
    }
    free(sb);
    return fail ? OR_E_OOM : OR_OK;
}

/*
 * or_rank_vs_set — T'_i = sum over a reference set of q(x_i, s) for every sequence i (PAPER.md:46,
 * D_i = (1/m) sum_s r(x_i, s) in the fixed point of reading A5; the rank of SURVEY §8(f) f1 with
 * the set = the gathered samples, and of f2 with the set = all N sequences, "sample
 * degeneracy"). set[m] are source indices (repeats allowed).
 */
int or_rank_vs_set(const uint8_t *ascii, const int64_t *offsets, int64_t n, int k, const int64_t *set, int64_t m,
                   int nthreads, uint64_t *T_out) {
    if (n <= 0 || m < 0) return OR_E_ARG;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    kcounts *kc = (kcounts *)calloc((size_t)n, sizeof(kcounts));
    int fail = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(| : fail)
    for (int64_t i = 0; i < n; ++i)
        fail |= count_kmers(ascii + offsets[i], offsets[i + 1] - offsets[i], k, &kc[i]) != 0;
    if (!fail) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            uint64_t acc = 0;
            int64_t Li = offsets[i + 1] - offsets[i];
            for (int64_t t = 0; t < m; ++t) {
                int64_t j = set[t], Lj = offsets[j + 1] - offsets[j];
                acc += or_q((uint64_t)min_sum(&kc[i], &kc[j], k), (uint64_t)den_of(Li, Lj, k));
            }
            T_out[i] = acc;
        }
    }
    for (int64_t i = 0; i < n; ++i) free_counts(&kc[i]);
    free(kc);
    return fail ? OR_E_OOM : OR_OK;
}

/*
 * or_pairs_S — S_ij and den_ij for a list of pairs (sampled parity checks).
 */
int or_pairs_S(const uint8_t *ascii, const int64_t *offsets, int k, const int64_t *pi, const int64_t *pj,
               int64_t m, int nthreads, int64_t *S_out, int64_t *den_out) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int fail = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(| : fail)
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = pi[r], j = pj[r];
        if (or_pair(ascii + offsets[i], offsets[i + 1] - offsets[i], ascii + offsets[j],
                    offsets[j + 1] - offsets[j], k, &S_out[r], &den_out[r]))
            fail = 1;
    }
    return fail ? OR_E_OOM : OR_OK;
}

/* Reported k-mer rank R = ln(0.1 + D) (natural log, reading A4). */
double or_rank_R(double D) { return log(0.1 + D); }

/* Threads the OpenMP runtime will use (reported as cpu_baseline.cores). */
int or_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    return omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}
