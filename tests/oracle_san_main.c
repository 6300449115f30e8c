/* Sanitizer driver for the CPU oracle: oracle/sad_oracle.c compiled together with this
 * file under -fsanitize=address,undefined and run single-threaded over random protein and DNA sets,
 * every entry point, both rank modes, p in {1, 2, 3, 8}, the error paths and a few invariants that a
 * memory or arithmetic bug would break (buckets form a permutation; T of selected rows equals T of the
 * full run). Test infrastructure only (tests/test_oracle_san.py builds and runs it). */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int or_run2(const uint8_t *ascii, const int64_t *offsets, int64_t n, int alphabet, int k, int p, int mode,
            int nthreads, uint64_t *T, int64_t *anc, int64_t *ga, int64_t *Sg, int64_t *dg, int64_t *sorted,
            int64_t *samples, int64_t *pivots, int64_t *bucket, int64_t *border, int64_t *bsize,
            int64_t *rsamples, double *stage_ms, int64_t *err_idx, int64_t *err_pos);
int or_rows_T(const uint8_t *ascii, const int64_t *offsets, int64_t n, int k, int p, const int64_t *rows, int64_t m,
              int nthreads, uint64_t *T_out);
int or_rank_vs_set(const uint8_t *ascii, const int64_t *offsets, int64_t n, int k, const int64_t *set, int64_t m,
                   int nthreads, uint64_t *T_out);
int or_pairs_S(const uint8_t *ascii, const int64_t *offsets, int k, const int64_t *pi, const int64_t *pj, int64_t m,
               int nthreads, int64_t *S_out, int64_t *den_out);
int64_t or_count(const uint8_t *x, int64_t L, int k, int64_t *out_pos, int64_t *out_cnt);

static uint64_t rs = 88172645463325252ull;
static uint32_t rnd(uint32_t m) {
    rs ^= rs << 13;
    rs ^= rs >> 7;
    rs ^= rs << 17;
    return (uint32_t)(rs % m);
}

#define CHECK(c)                                                          \
    do {                                                                  \
        if (!(c)) {                                                       \
            fprintf(stderr, "check failed line %d: %s\n", __LINE__, #c); \
            return 1;                                                     \
        }                                                                 \
    } while (0)

static int one(int alphabet, int k, int p, int mode, int n, int lmax, int repeats) {
    const char *al = alphabet ? "ACGT" : "ACDEFGHIKLMNPQRSTVWY";
    const int A = alphabet ? 4 : 20;
    int64_t *off = malloc(sizeof(int64_t) * (n + 1));
    off[0] = 0;
    for (int i = 0; i < n; ++i) off[i + 1] = off[i] + k + (int64_t)rnd((uint32_t)lmax);
    uint8_t *a = malloc((size_t)off[n] + 1);
    for (int i = 0; i < n; ++i) {
        const int64_t L = off[i + 1] - off[i];
        for (int64_t t = 0; t < L; ++t) a[off[i] + t] = (uint8_t)al[rnd((uint32_t)A)];
        if (repeats && i % 3 == 0)              /* low-complexity rows: counts far above 1 */
            for (int64_t t = 0; t < L; ++t) a[off[i] + t] = (uint8_t)al[(t / 2) % 2];
    }
    uint64_t *T = calloc(n, 8);
    int64_t *anc = calloc(p, 8), ga = 0, *Sg = calloc(n, 8), *dg = calloc(n, 8), *srt = calloc(n, 8);
    int64_t *smp = calloc((size_t)p * p + 1, 8), *piv = calloc(p + 1, 8), *bk = calloc(n, 8), *bo = calloc(n, 8);
    int64_t *bs = calloc(p, 8), *rsm = calloc((size_t)p * p + 1, 8), ei = -1, ep = -1;
    double ms[4];
    int rc = or_run2(a, off, n, alphabet, k, p, mode, 1, T, anc, &ga, Sg, dg, srt, smp, piv, bk, bo, bs,
                     mode ? rsm : NULL, ms, &ei, &ep);
    CHECK(rc == 0);
    /* the buckets form a permutation of the input */
    char *seen = calloc(n, 1);
    int64_t tot = 0;
    for (int b = 0; b < p; ++b) tot += bs[b];
    CHECK(tot == n);
    for (int i = 0; i < n; ++i) {
        CHECK(bo[i] >= 0 && bo[i] < n && !seen[bo[i]]);
        seen[bo[i]] = 1;
    }
    /* T of selected rows (or_rows_T) equals T of the full run */
    int64_t rows[5] = {0, n / 3, n / 2, (2 * n) / 3, n - 1};
    uint64_t Tr[5];
    CHECK(or_rows_T(a, off, n, k, p, rows, 5, 1, Tr) == 0);
    for (int j = 0; j < 5; ++j) CHECK(Tr[j] == T[rows[j]]);
    uint64_t *Tp = calloc(n, 8);
    int64_t set[3] = {0, n - 1, n / 2};
    CHECK(or_rank_vs_set(a, off, n, k, set, 3, 1, Tp) == 0);
    int64_t pi[4] = {0, 1, n - 1, n / 2}, pj[4] = {0, n - 1, 1, n / 2}, S[4], d[4];
    CHECK(or_pairs_S(a, off, k, pi, pj, 4, 1, S, d) == 0);
    CHECK(S[0] == d[0] && S[3] == d[3]);        /* F(x, x) = 1 */
    CHECK(S[1] == S[2] && d[1] == d[2]);        /* symmetry */
    int64_t *pos = calloc((size_t)(off[1] - off[0]), 8), *cnt = calloc((size_t)(off[1] - off[0]), 8);
    CHECK(or_count(a, off[1] - off[0], k, pos, cnt) >= 1);
    free(pos); free(cnt); free(seen); free(Tp);
    free(T); free(anc); free(Sg); free(dg); free(srt); free(smp); free(piv); free(bk); free(bo); free(bs); free(rsm);
    free(a); free(off);
    return 0;
}

static int errors(void) {
    /* an illegal symbol and a sequence shorter than k: the error paths */
    const uint8_t a[] = "ACGTXACGTACGTAC";
    int64_t off[4] = {0, 5, 7, 15};
    uint64_t T[3];
    int64_t anc[1], ga, Sg[3], dg[3], srt[3], smp[1], piv[1], bk[3], bo[3], bs[1], ei = -1, ep = -1;
    double ms[4];
    int rc = or_run2(a, off, 3, 1, 3, 1, 0, 1, T, anc, &ga, Sg, dg, srt, smp, piv, bk, bo, bs, NULL, ms, &ei, &ep);
    CHECK(rc != 0);
    const uint8_t b[] = "ACGTACGTAC";
    int64_t off2[3] = {0, 2, 10};
    rc = or_run2(b, off2, 2, 1, 3, 1, 0, 1, T, anc, &ga, Sg, dg, srt, smp, piv, bk, bo, bs, NULL, ms, &ei, &ep);
    CHECK(rc != 0);
    return 0;
}

int main(void) {
    const int ps[4] = {1, 2, 3, 8};
    int trials = 0;
    for (int alphabet = 0; alphabet < 2; ++alphabet)
        for (int pi = 0; pi < 4; ++pi)
            for (int mode = 0; mode < 2; ++mode) {
                const int p = ps[pi];
                if (mode == 1 && p < 2) continue;
                const int k = alphabet ? 6 : 3;
                if (one(alphabet, k, p, mode, p * p + 40 + (int)rnd(60), 300, (pi + mode) & 1)) return 1;
                if (one(alphabet, 2, p, mode, p * p + 20, 40, 1)) return 1;
                trials += 2;
            }
    if (errors()) return 1;
    printf("oracle sanitizer run ok: %d trials\n", trials);
    return 0;
}
