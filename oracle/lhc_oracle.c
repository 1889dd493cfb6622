/*
 * oracle/lhc_oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded C11 implementation of what the hot path of
 * "Accelerating Distributed Deep Learning using Lossless Homomorphic
 * Compression" (arXiv 2402.07529, /root/reference/PAPER.md, cited as P:L<n>)
 * computes.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2402_07529_b200/) never includes, links or calls it, and this file
 * includes nothing from the product path: the two share no code.
 *
 * Arithmetic: counters, residuals and recovered values are fp64 (the paper
 * fixes no precision); bitmaps are u32 words, bit b of the filter is
 * bit (b & 31) of word (b >> 5).
 *
 * Where the paper is silent the readings are those of DESIGN.md §Readings
 * (numbered R1..R21 there, mirroring SURVEY.md §8c):
 *   - hash functions (R1): SplitMix64-based H(seed, dom, j, i), domain 0 = Count
 *     Sketch, domain 1 = Bloom filter;
 *   - "three different indexes" (R2): partitioned rows, probe j lives in
 *     partition j;
 *   - batching (R4, R5, R6): one (row, bias, sign) per (input row i, probe j),
 *     column rotation (t + bias) mod L, Bloom filter in the same layout;
 *   - peeling (R8, R9, R10): cell granularity, synchronous rounds, degree count
 *     plus XOR of candidate slots, the lowest probe index j wins a tie;
 *   - fallback (R11): median of the residual after peeling.
 *
 * Pinning status (see tests/test_oracle_*.py and DESIGN.md §Oracle pins):
 *   ora_mix64            pinned: published SplitMix64 output vector
 *   ora_hash / maps      the paper gives no hash: pinned to the
 *                        written spec of SURVEY.md §8c (its three hand-computed H
 *                        values), the frozen table tests/golden/rowmap.json
 *                        (packing, sign bit, bias, row reduction), and
 *                        statistical invariants (uniform bias/sign/row,
 *                        bijective rotation)
 *   ora_compress_*       pinned: homomorphism, single-insert identity, full-row
 *                        rotation bijection, partition sums
 *   ora_aggregate        pinned: OR/sum laws on independent inputs
 *   ora_query            pinned: no false negatives, exact support when the
 *                        filter is sparse, false-positive rate vs closed form
 *   ora_peel_core        pinned: Fig. 1 worked example, brute-force
 *                        2-core on tiny inputs, chain round counts
 *   ora_finalize         pinned: hand-computed medians, unbiasedness,
 *                        a hand-built partial peel whose residual medians differ
 *                        from the medians over Y (reading R11)
 *   ora_decompress       pinned: losslessness (exact sum) under the dyadic law
 *                        (P:L66), success phase transition, the
 *                        fallback over the residual of a stalled decode,
 *                        recomputed independently (reading R11)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Mirrors the field order of include/lhc.h's lhc_params; declared here on its
 * own so that the oracle includes nothing from the product path. */
typedef struct {
    uint32_t d;        /* coordinates of the gradient (paper: N)        */
    uint64_t m;        /* Bloom-filter bits                                     */
    uint64_t c;        /* Count Sketch cells (paper: size of Y)         */
    uint32_t k;        /* Count Sketch hashes (paper: 3)                */
    uint32_t k_bloom;  /* Bloom probes (paper: log 1/eps); 0 means k    */
    uint32_t L;        /* batch width (paper: c = 1024)                 */
    uint32_t blocks;   /* 0, or the Count Sketch split into blocks     */
    uint64_t seed;     /* hash seed                                             */
} ora_params;

typedef struct {
    uint64_t n_cand;
    uint64_t n_peeled;
    uint32_t rounds;
    int32_t success;
    int32_t overflow;
} ora_stats;

enum { ORA_OK = 0, ORA_EINVAL = 1 };

/* k_bloom value selecting the exact bitmap index of §3.2 ("allocating one
 * bit per parameter - for each bit, true indicates non-zero, while false
 * indicates zero") instead of a Bloom filter: bit p is coordinate p. */
#define ORA_INDEX_BITMAP 255u

static uint32_t kb_of(const ora_params* p)
{
    if (p->k_bloom == ORA_INDEX_BITMAP) return 1;
    return p->k_bloom ? p->k_bloom : p->k;
}

/* ---------------------------------------------------------------------------
 * Hashing (reading R1; the paper only says "hashed to three signals ... and
 * three different indexes", and "hashing every non-zero parameter to
 * log 1/eps bits").
 * ------------------------------------------------------------------------- */

/* SplitMix64 finalizer (Steele, Lea, Flood 2014). */
uint64_t ora_mix64(uint64_t z)
{
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

/* H(seed, dom, j, i) = mix64(seed XOR mix64(((dom<<56)|(j<<48)|i) + golden)) */
uint64_t ora_hash(uint64_t seed, uint32_t dom, uint32_t j, uint64_t i)
{
    uint64_t key = ((uint64_t)dom << 56) | ((uint64_t)j << 48) | i;
    return ora_mix64(seed ^ ora_mix64(key + 0x9E3779B97F4A7C15ull));
}

/* Row map of input row i under probe j of domain dom ("each batch
 * shares the same index"; "a random bias within the range [0..c-1]").
 *   row  = j*S + ((H>>32) * S >> 32)       (partition j, reading R2)
 *   bias = H & (L-1)
 *   sign = bit 16 of H set ? -1 : +1       (used for the Count Sketch only)   */
void ora_row_map(const ora_params* p, uint32_t dom, uint32_t j, uint64_t i,
                 uint64_t* row, uint32_t* bias, int* sign)
{
    if (dom == 1 && p->k_bloom == ORA_INDEX_BITMAP) { /* exact bitmap: row i, no rotation */
        *row = i;
        *bias = 0;
        *sign = +1;
        return;
    }
    /* blocked Count Sketch ("splitting the Count Sketch into multiple blocks
     * of fixed size", reading R25): input row i belongs to block i mod blocks, whose
     * k partitions of S rows each hold all of its cells */
    uint64_t base = 0;
    uint64_t S = dom == 0 ? p->c / ((uint64_t)p->k * p->L)
                          : p->m / ((uint64_t)kb_of(p) * p->L);
    if (dom == 0 && p->blocks) {
        S = p->c / ((uint64_t)p->blocks * p->k * p->L);
        base = (i % p->blocks) * p->k * S;
    }
    uint64_t H = ora_hash(p->seed, dom, j, i);
    *row = base + (uint64_t)j * S + (((H >> 32) * S) >> 32);
    *bias = (uint32_t)(H & (uint64_t)(p->L - 1));
    *sign = ((H >> 16) & 1) ? -1 : +1;
}

/* Count Sketch cell of coordinate q under hash j, and its sign g_j (P:L175,
 * with the batched, rotated layout of P:L262). */
uint64_t ora_cell(const ora_params* p, uint32_t j, uint64_t q, int* sign)
{
    uint64_t row;
    uint32_t bias;
    uint64_t i = q / p->L, t = q % p->L;
    ora_row_map(p, 0, j, i, &row, &bias, sign);
    return row * p->L + (t + bias) % p->L;
}

/* Bloom-filter bit of coordinate q under probe j (layout P:L262). */
uint64_t ora_bit(const ora_params* p, uint32_t j, uint64_t q)
{
    uint64_t row;
    uint32_t bias;
    int sign;
    uint64_t i = q / p->L, t = q % p->L;
    ora_row_map(p, 1, j, i, &row, &bias, &sign);
    return row * p->L + (t + bias) % p->L;
}

static int cmp_u64(const void* a, const void* b);

static int bit_get(const uint32_t* B, uint64_t b) { return (B[b >> 5] >> (b & 31)) & 1u; }
static void bit_set(uint32_t* B, uint64_t b) { B[b >> 5] |= 1u << (b & 31); }

int ora_validate(const ora_params* p)
{
    if (!p || p->d == 0 || p->k == 0 || p->k > 8) return ORA_EINVAL;
    if (p->k_bloom > 8 && p->k_bloom != ORA_INDEX_BITMAP) return ORA_EINVAL;
    if (p->k_bloom == ORA_INDEX_BITMAP && p->m != ((uint64_t)p->d + p->L - 1) / p->L * p->L)
        return ORA_EINVAL;
    if (p->L < 32 || p->L > 1024 || (p->L & (p->L - 1))) return ORA_EINVAL;
    uint32_t kb = kb_of(p);
    if (p->c == 0 || p->c % ((uint64_t)p->k * p->L)) return ORA_EINVAL;
    if (p->m == 0 || p->m % ((uint64_t)kb * p->L)) return ORA_EINVAL;
    if (p->c / ((uint64_t)p->k * p->L) >= (1ull << 32)) return ORA_EINVAL;
    if (p->m / ((uint64_t)kb * p->L) >= (1ull << 32)) return ORA_EINVAL;
    if (p->blocks && p->c % ((uint64_t)p->blocks * p->k * p->L)) return ORA_EINVAL;
    return ORA_OK;
}

/* ---------------------------------------------------------------------------
 * Phase I: compression (Alg. 1).  Accumulates into B and Y: the
 * caller zeroes them for a fresh sketch.
 * ------------------------------------------------------------------------- */

/* Insert one nonzero (q, v): set its k_B Bloom bits and add
 * g_j(i)*v to its k Count Sketch cells. */
static void insert(const ora_params* p, uint64_t q, double v, uint32_t* B, double* Y)
{
    for (uint32_t j = 0; j < kb_of(p); j++)
        bit_set(B, ora_bit(p, j, q));
    for (uint32_t j = 0; j < p->k; j++) {
        int g;
        uint64_t e = ora_cell(p, j, q, &g);
        Y[e] += g * v;
    }
}

/* Dense gradient x[d]: every coordinate with x != 0 is a nonzero. */
void ora_compress_dense(const ora_params* p, const float* x, uint32_t* B, double* Y)
{
    for (uint64_t q = 0; q < p->d; q++)
        if (x[q] != 0.0f)
            insert(p, q, (double)x[q], B, Y);
}

/* COO gradient: every listed (idx, val) is inserted, even val == 0 (the index
 * describes the listed support). */
void ora_compress_coo(const ora_params* p, uint64_t nnz, const uint32_t* idx,
                      const float* val, uint32_t* B, double* Y)
{
    for (uint64_t s = 0; s < nnz; s++)
        insert(p, idx[s], (double)val[s], B, Y);
}

/* ---------------------------------------------------------------------------
 * Aggregation (Alg. 1 comment: "Y <- sum Y and B <- OR B").
 * ------------------------------------------------------------------------- */
void ora_aggregate(uint64_t n_words, uint64_t c, int n_in,
                   const uint32_t* const* B_in, const double* const* Y_in,
                   uint32_t* B_out, double* Y_out)
{
    for (uint64_t w = 0; w < n_words; w++) {
        uint32_t acc = 0;
        for (int r = 0; r < n_in; r++) acc |= B_in[r][w];
        B_out[w] = acc;
    }
    for (uint64_t e = 0; e < c; e++) {
        double acc = 0.0;
        for (int r = 0; r < n_in; r++) acc += Y_in[r][e];
        Y_out[e] = acc;
    }
}

/* ---------------------------------------------------------------------------
 * Phase II: recovery.
 * ------------------------------------------------------------------------- */

/* Bloom query ("verifying that all the Bloom Filter's corresponding
 * bits are set to one").  Candidates are written in ascending order; slot s
 * names cand[s].  Returns the number of candidates n_c; at most cap are
 * written (cand may be NULL to count only). */
uint64_t ora_query(const ora_params* p, const uint32_t* B, uint32_t* cand, uint64_t cap)
{
    uint64_t n = 0;
    for (uint64_t q = 0; q < p->d; q++) {
        int all = 1;
        for (uint32_t j = 0; j < kb_of(p) && all; j++)
            all = bit_get(B, ora_bit(p, j, q));
        if (all) {
            if (cand && n < cap) cand[n] = (uint32_t)q;
            n++;
        }
    }
    return n;
}

/* Peeling on an explicit incidence.
 *   n_items items (candidates), item s lies in cells[s*k + j] with sign
 *   signs[s*k + j], j < k; the cells of one item are distinct.
 *   R[n_cells]  in: the aggregated Count Sketch Y; out: the residual.
 *   val[s]      out: recovered value of every peeled item.
 *   peeled[s]   out: 1 if peeled, else 0.
 *   round_of[s] out (nullable): round in which s was peeled (1-based), 0 if not.
 * Synchronous rounds (reading R10): in a round, every cell that holds exactly
 * one unpeeled item ("mapped by only one non-zero parameter") names
 * that item; each named item takes its value from its lowest-j such cell,
 * val = g_j * R[cell] ("X_i can be deduced as g_j(i) * Y_h_j(i)"),
 * and is then removed from all its cells, R[cell] -= g_j * val ("deducting
 * Y_h_j(i) by g_j(i) * X_i").  Rounds repeat "until X is completely
 * reconstructed or there are no more parameters that can be peeled".
 * The cell state is the degree and the XOR of item slots (reading R9).
 * Returns the number of peeled items; *rounds_out = rounds that peeled. */
uint64_t ora_peel_core(uint64_t n_items, uint32_t k, const uint64_t* cells,
                       const int8_t* signs, uint64_t n_cells, double* R,
                       double* val, uint8_t* peeled, uint32_t* round_of,
                       uint32_t* rounds_out)
{
    uint32_t* deg = calloc(n_cells ? n_cells : 1, sizeof(uint32_t));
    uint32_t* ids = calloc(n_cells ? n_cells : 1, sizeof(uint32_t));
    uint32_t* best = malloc((n_items ? n_items : 1) * sizeof(uint32_t));
    uint8_t* touched = calloc(n_cells ? n_cells : 1, 1);
    uint64_t* F = malloc((n_cells ? n_cells : 1) * sizeof(uint64_t));
    uint64_t* T = malloc((n_cells ? n_cells : 1) * sizeof(uint64_t));
    uint64_t* P = malloc((n_items ? n_items : 1) * sizeof(uint64_t));
    uint8_t* named = calloc(n_items ? n_items : 1, 1);

    /* initial degree and id accumulators */
    for (uint64_t s = 0; s < n_items; s++) {
        peeled[s] = 0;
        if (round_of) round_of[s] = 0;
        best[s] = UINT32_MAX;
        for (uint32_t j = 0; j < k; j++) {
            uint64_t e = cells[s * k + j];
            deg[e] += 1;
            ids[e] ^= (uint32_t)s;
        }
    }
    /* first frontier: every cell of degree one, ascending */
    uint64_t nF = 0;
    for (uint64_t e = 0; e < n_cells; e++)
        if (deg[e] == 1) F[nF++] = e;

    uint64_t n_peeled = 0;
    uint32_t rounds = 0;
    while (nF > 0) {
        rounds++;
        /* 1. each frontier cell names its only item; the lowest j wins */
        uint64_t nP = 0;
        for (uint64_t f = 0; f < nF; f++) {
            uint64_t e = F[f];
            uint32_t s = ids[e];
            for (uint32_t j = 0; j < k; j++)
                if (cells[(uint64_t)s * k + j] == e && j < best[s]) best[s] = j;
            if (!named[s]) {
                named[s] = 1;
                P[nP++] = s;
            }
        }
        /* 2. named items in ascending slot order take their value */
        qsort(P, nP, sizeof(uint64_t), cmp_u64);
        for (uint64_t a = 0; a < nP; a++) {
            uint64_t s = P[a];
            uint32_t j = best[s];
            val[s] = signs[s * k + j] * R[cells[s * k + j]];
            peeled[s] = 1;
            if (round_of) round_of[s] = rounds;
        }
        /* 3. remove them from all their cells */
        uint64_t nT = 0;
        for (uint64_t a = 0; a < nP; a++) {
            uint64_t s = P[a];
            for (uint32_t j = 0; j < k; j++) {
                uint64_t e = cells[s * k + j];
                R[e] -= signs[s * k + j] * val[s];
                deg[e] -= 1;
                ids[e] ^= (uint32_t)s;
                if (!touched[e]) { touched[e] = 1; T[nT++] = e; }
            }
        }
        n_peeled += nP;
        /* 4. next frontier: touched cells now of degree one */
        nF = 0;
        for (uint64_t a = 0; a < nT; a++) {
            touched[T[a]] = 0;
            if (deg[T[a]] == 1) F[nF++] = T[a];
        }
    }
    *rounds_out = rounds;
    free(deg); free(ids); free(best); free(touched); free(F); free(T); free(P); free(named);
    return n_peeled;
}

static int cmp_u64(const void* a, const void* b)
{
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

static void sort_small(double* v, uint32_t n)
{
    for (uint32_t a = 1; a < n; a++) {
        double x = v[a];
        uint32_t b = a;
        while (b > 0 && v[b - 1] > x) { v[b] = v[b - 1]; b--; }
        v[b] = x;
    }
}

/* Fallback for items peeling could not reach (Alg. 1: "Estimate the
 * not recovered parameters of X from Y"; footnote P:L193: "we use the Count
 * Sketch to give an unbiased estimation"): the Count Sketch median estimate
 * ("Count Sketch reports the median of the values g_j(i) * Y_h_j(i)")
 * over the residual (reading R11).  Even k: mean of the two middle values. */
void ora_finalize(uint64_t n_items, uint32_t k, const uint64_t* cells,
                  const int8_t* signs, const double* R, const uint8_t* peeled,
                  double* val)
{
    double v[64];
    for (uint64_t s = 0; s < n_items; s++) {
        if (peeled[s]) continue;
        for (uint32_t j = 0; j < k; j++)
            v[j] = signs[s * k + j] * R[cells[s * k + j]];
        sort_small(v, k);
        val[s] = (k & 1) ? v[k / 2] : 0.5 * (v[k / 2 - 1] + v[k / 2]);
    }
}

/* Whole Phase II (Alg. 1) on an aggregated sketch [Y, B]:
 * query, peel, estimate; dense output (nullable) holds the candidate values
 * and exact zeros elsewhere.  Y is not modified.  Outputs past cap are not
 * written; stats->overflow = n_c > cap, in which case nothing is peeled. */
int ora_decompress(const ora_params* p, const uint32_t* B, const double* Y,
                   uint64_t cap, uint32_t* cand, double* val, uint8_t* peeled,
                   uint32_t* round_of, double* dense, ora_stats* st)
{
    if (ora_validate(p) != ORA_OK) return ORA_EINVAL;
    memset(st, 0, sizeof(*st));
    uint64_t n_c = ora_query(p, B, cand, cap);
    st->n_cand = n_c;
    if (n_c > cap) { st->overflow = 1; return ORA_OK; }

    uint64_t* cells = malloc((n_c ? n_c : 1) * p->k * sizeof(uint64_t));
    int8_t* signs = malloc((n_c ? n_c : 1) * p->k);
    for (uint64_t s = 0; s < n_c; s++)
        for (uint32_t j = 0; j < p->k; j++) {
            int g;
            cells[s * p->k + j] = ora_cell(p, j, cand[s], &g);
            signs[s * p->k + j] = (int8_t)g;
        }
    double* R = malloc(p->c * sizeof(double));
    memcpy(R, Y, p->c * sizeof(double));
    uint32_t rounds = 0;
    uint64_t n_peeled = ora_peel_core(n_c, p->k, cells, signs, p->c, R, val, peeled,
                                      round_of, &rounds);
    ora_finalize(n_c, p->k, cells, signs, R, peeled, val);
    if (dense) {
        for (uint64_t q = 0; q < p->d; q++) dense[q] = 0.0;
        for (uint64_t s = 0; s < n_c; s++) dense[cand[s]] = val[s];
    }
    st->n_peeled = n_peeled;
    st->rounds = rounds;
    st->success = n_peeled == n_c;
    free(cells); free(signs); free(R);
    return ORA_OK;
}
