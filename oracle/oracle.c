/*
 * oracle.c -- plain, slow, obviously correct CPU oracle for the hot path of
 *   Tarhio, Holub, Giaquinta, "Technology Beats Algorithms (in Exact String
 *   Matching)", arXiv:1612.01506  (text: /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1612_01506_b200/), and neither side includes the other.
 *
 * Conventions.  The paper indexes strings from 1 (Alg. 1 line 3
 * "for i <- 1 to n-m+1").  To keep the loops readable against the paper, each
 * function re-bases its arrays with `P = p - 1`, `T = t - 1` so that P[j] is
 * the paper's p[j] and T[i] is the paper's t[i].  Reported positions are
 * returned 0-based (paper position - 1), reading R1.
 *
 * Pinned by tests/test_oracle.py: Fig. 1, closed forms
 * (t=a^n, p=a^m -> n-m+1; absent symbol -> 0; m>n -> 0), brute force over all
 * patterns on tiny texts, an independent KMP count, numpy.bincount.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

/* ------------------------------------------------------------------------ */
/* Alg. 1 Naive-search(p, m, t, n)  -- PAPER.md:41-53 (Sec. 2.1), verbatim.   */
/* Counting version.  m >= 1; n < m gives 0 (loop runs zero     */
/* times, reading R2).                                                        */
/* ------------------------------------------------------------------------ */
uint64_t oracle_naive_count(const uint8_t *p, size_t m, const uint8_t *t, size_t n)
{
    const uint8_t *P = p - 1, *T = t - 1;          /* 1-based views */
    uint64_t count = 0;                              /* line 2 */
    if (m == 0 || n < m) return 0;
    for (size_t i = 1; i <= n - m + 1; i++) {        /* line 3 */
        int found = 1;                               /* line 4 */
        for (size_t j = 1; j <= m; j++) {            /* line 5 */
            found = found && (T[i + j - 1] == P[j]); /* line 6 */
            if (!found) goto next_position;          /* lines 7-8 */
        }
        count = count + 1;                           /* line 11 */
    next_position:;                                  /* line 12: goto target */
    }
    return count;
}

/* Reporting version: "printing position i in line 11".
 * Writes at most `cap` positions (0-based, ascending = loop order), returns
 * the total number of occurrences. */
uint64_t oracle_naive_report(const uint8_t *p, size_t m, const uint8_t *t, size_t n,
                             uint64_t *pos, uint64_t cap)
{
    const uint8_t *P = p - 1, *T = t - 1;
    uint64_t count = 0;
    if (m == 0 || n < m) return 0;
    for (size_t i = 1; i <= n - m + 1; i++) {
        int found = 1;
        for (size_t j = 1; j <= m; j++) {
            found = found && (T[i + j - 1] == P[j]);
            if (!found) goto next_position;
        }
        if (count < cap) pos[count] = (uint64_t)(i - 1);   /* "print i" */
        count = count + 1;
    next_position:;
    }
    return count;
}

/* ------------------------------------------------------------------------ */
/* Symbol frequencies of the text ("increasing order of their     */
/* probabilities in the text"; reading R10).  hist[c] = #{x : t[x]=c}. */
/* ------------------------------------------------------------------------ */
void oracle_hist(const uint8_t *t, size_t n, uint64_t *hist)
{
    for (int c = 0; c < 256; c++) hist[c] = 0;
    for (size_t x = 0; x < n; x++) hist[t[x]] += 1;
}

/* ------------------------------------------------------------------------ */
/* Comparison order pi (Sec. 2.2): pattern positions sorted by  */
/* ascending frequency of their symbol ("First, the least frequent symbol is  */
/* compared").  Ties -> ascending position (stable; reading R11).*/
/* Plain insertion sort (stable by construction).  order[] is 0-based.       */
/* ------------------------------------------------------------------------ */
void oracle_order(const uint64_t *hist, const uint8_t *p, size_t m, uint32_t *order)
{
    for (size_t j = 0; j < m; j++) {
        size_t k = j;
        /* shift right every earlier entry with a STRICTLY larger key */
        while (k > 0 && hist[p[order[k - 1]]] > hist[p[j]]) {
            order[k] = order[k - 1];
            k--;
        }
        order[k] = (uint32_t)j;
    }
}

/* ------------------------------------------------------------------------ */
/* Alg. 4 LP-Freq-SIMD-Naive-search(p, m, t, n, alpha) with general peeling  */
/* factor r (Sec. 2.3) and arbitrary order pi (Alg. 3,      */
/* PAPER.md:118-135).  alpha <= 64; SIMDcompare is emulated by a loop that    */
/* returns the alpha-bit mask "k-th bit set iff S1[k] = S2[k]". */
/*                                                                            */
/* Readings: R4 (Alg. 2 passes i+j-1 while the primitive adds j-1 again; the   */
/* prose "For j = 2 ... compares t[2..alpha+1]" fixes the window start at    */
/* t[i+pi(j)-1]); R5 (window is alpha bytes long); R7 (alignments past n-m+1   */
/* in the last block are masked out and bytes past t[n] are never read);      */
/* R8 (Alg. 4 line 5 duplicated "p, p" read as SIMDcompare(t,i+pi(2)-1,p,pi(2),alpha)); */
/* R9 (r <- min(r, m)).                                                       */
/*                                                                            */
/* Returns the count; *n_compares (if non-NULL) receives the number of        */
/* SIMDcompare calls executed (instrumentation for the order/peeling study).  */
/* pi[] is 0-based (pi[k] = 0-based pattern position compared k-th).         */
/* ------------------------------------------------------------------------ */
static uint64_t simd_compare(const uint8_t *T, size_t n, size_t i_plus_j_minus_1,
                             uint8_t y, unsigned alpha, uint64_t lanes_valid)
{
    /* S1 = t[i+j-1 .. i+j-1+alpha-1], S2 = y^alpha; bit k <-> S1[k] = y.    */
    uint64_t mask = 0;
    for (unsigned k = 0; k < alpha; k++) {
        if (!((lanes_valid >> k) & 1u)) continue;    /* alignment beyond n-m+1 */
        size_t pos = i_plus_j_minus_1 + k;           /* 1-based text index */
        if (pos <= n && T[pos] == y) mask |= (uint64_t)1 << k;
    }
    return mask;
}

static unsigned popcount64(uint64_t x)
{
    unsigned c = 0;
    while (x) { c += (unsigned)(x & 1u); x >>= 1; }
    return c;
}

uint64_t oracle_alg4_count(const uint8_t *p, size_t m, const uint8_t *t, size_t n,
                           unsigned alpha, const uint32_t *pi, unsigned r,
                           uint64_t *n_compares, uint64_t *pos, uint64_t cap)
{
    const uint8_t *P = p - 1, *T = t - 1;
    uint64_t count = 0, compares = 0;
    if (n_compares) *n_compares = 0;
    if (m == 0 || n < m || alpha == 0 || alpha > 64) return 0;
    if (r < 1) r = 1;
    if (r > m) r = (unsigned)m;                                   /* R9 */
    size_t last = n - m + 1;                                      /* last alignment */
    for (size_t i = 1; i <= last; i += alpha) {                   /* line 3, step alpha */
        uint64_t lanes_valid = 0;
        for (unsigned k = 0; k < alpha; k++)
            if (i + k <= last) lanes_valid |= (uint64_t)1 << k;   /* R7 */
        uint64_t found = lanes_valid;                             /* "11..1" */
        size_t j;
        /* peeled iterations: all r performed, no test in between */
        for (j = 1; j <= r; j++) {
            size_t pj = (size_t)pi[j - 1] + 1;                    /* pi(j), 1-based */
            found &= simd_compare(T, n, i + pj - 1, P[pj], alpha, lanes_valid);
            compares++;
        }
        if (found == 0) continue;                                 /* lines 6-7 */
        for (; j <= m; j++) {                                     /* line 8 */
            size_t pj = (size_t)pi[j - 1] + 1;
            found &= simd_compare(T, n, i + pj - 1, P[pj], alpha, lanes_valid);
            compares++;
            if (found == 0) break;                                /* lines 10-11 */
        }
        if (found == 0) continue;
        uint64_t idx = count;
        count += popcount64(found);                               /* line 14 */
        if (pos) {                                                /* reporting: O(s) extraction */
            for (unsigned k = 0; k < alpha; k++)
                if ((found >> k) & 1u) {
                    /* bit k <-> alignment i+k (1-based) -> 0-based i+k-1 (R6) */
                    if (idx < cap) pos[idx] = (uint64_t)(i + k - 1);
                    idx++;
                }
        }
    }
    if (n_compares) *n_compares = compares;
    return count;
}

/* ------------------------------------------------------------------------ */
/* Alg. 4 for any block width alpha >= 1, instrumentation  */
/* only (NEXT-2 compare counters): the number of SIMDcompare calls executed   */
/* and the number of alpha-blocks visited.  Same loop as oracle_alg4_count --  */
/* blocks i = 1, 1+alpha, ... <= n-m+1 (line 3); r peeled compares without a  */
/* test; then the pi-ordered loop leaving the block as soon as */
/* found is empty (lines 8-11) -- with `found` held as one flag per alignment  */
/* instead of a machine word, so alpha is not limited to 64 (the GPU's warp   */
/* covers 512 x CPL alignments).  Readings R7 (alignments past n-m+1 masked),  */
/* R9 (r <- min(r, m)).  Returns the SIMDcompare count; *n_blocks receives    */
/* the number of blocks.                                                       */
/* ------------------------------------------------------------------------ */
uint64_t oracle_alg4_steps(const uint8_t *p, size_t m, const uint8_t *t, size_t n,
                           size_t alpha, const uint32_t *pi, unsigned r, uint64_t *n_blocks)
{
    const uint8_t *P = p - 1, *T = t - 1;
    uint64_t compares = 0, blocks = 0;
    if (n_blocks) *n_blocks = 0;
    if (m == 0 || n < m || alpha == 0) return 0;
    if (r < 1) r = 1;
    if (r > m) r = (unsigned)m;                                   /* R9 */
    unsigned char *found = (unsigned char *)malloc(alpha);
    if (!found) return 0;
    size_t last = n - m + 1;
    for (size_t i = 1; i <= last; i += alpha) {                   /* line 3 */
        blocks++;
        size_t width = (last - i + 1 < alpha) ? last - i + 1 : alpha;   /* R7 */
        for (size_t k = 0; k < width; k++) found[k] = 1;         /* "11..1" */
        size_t alive = width;
        size_t j;
        for (j = 1; j <= m; j++) {
            if (j > r && alive == 0) break;                       /* lines 6-7 / 10-11 */
            size_t pj = (size_t)pi[j - 1] + 1;                    /* pi(j), 1-based */
            for (size_t k = 0; k < width; k++)                    /* SIMDcompare, bit k */
                if (found[k] && T[i + k + pj - 1] != P[pj]) { found[k] = 0; alive--; }
            compares++;
        }
    }
    free(found);
    if (n_blocks) *n_blocks = blocks;
    return compares;
}

/* ------------------------------------------------------------------------ */
/* Fixed heuristic order pi_h (Sec. 2.4):                      */
/*   p[1], p[m], p[4], p[7], ..., p[3], p[6], ..., p[2], p[5], ...           */
/* Reading R18: stride-3 chains starting at 4, then 3, then 2, skipping       */
/* positions already emitted.  0-based output.                               */
/* ------------------------------------------------------------------------ */
void oracle_pi_h(size_t m, uint32_t *order)
{
    size_t k = 0;
    unsigned char *used = (unsigned char *)calloc(m + 2, 1);
    if (!used) return;
    order[k++] = 0; used[1] = 1;                          /* p[1] */
    if (m >= 2) { order[k++] = (uint32_t)(m - 1); used[m] = 1; }   /* p[m] */
    const size_t starts[3] = {4, 3, 2};
    for (int s = 0; s < 3; s++)
        for (size_t q = starts[s]; q <= m; q += 3)
            if (!used[q]) { order[k++] = (uint32_t)(q - 1); used[q] = 1; }
    free(used);
}

/* ------------------------------------------------------------------------ */
/* Independent cross-check: Knuth-Morris-Pratt count (PAPER.md:24 cites KMP as */
/* background).  Textbook failure function; after a full match continue from  */
/* fail[m] so that overlapping occurrences are counted.  Not the method.      */
/* ------------------------------------------------------------------------ */
uint64_t oracle_kmp_count(const uint8_t *p, size_t m, const uint8_t *t, size_t n)
{
    if (m == 0 || n < m) return 0;
    size_t *fail = (size_t *)malloc((m + 1) * sizeof(size_t));
    if (!fail) return UINT64_MAX;
    fail[0] = 0; fail[1] = 0;
    size_t k = 0;
    for (size_t q = 1; q < m; q++) {          /* fail[q+1] = longest proper border of p[0..q] */
        while (k > 0 && p[k] != p[q]) k = fail[k];
        if (p[k] == p[q]) k++;
        fail[q + 1] = k;
    }
    uint64_t count = 0;
    size_t q = 0;
    for (size_t i = 0; i < n; i++) {
        while (q > 0 && p[q] != t[i]) q = fail[q];
        if (p[q] == t[i]) q++;
        if (q == m) { count++; q = fail[m]; }
    }
    free(fail);
    return count;
}
