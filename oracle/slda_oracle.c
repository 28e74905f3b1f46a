/*
 * slda_oracle.c -- TEST INFRASTRUCTURE ONLY (see slda_oracle.h).
 *
 * Plain-C restatement of the reference ESCA path.  Reference paths are
 * relative to /root/reference/proj.  Compiled with -O2 -ffp-contract=off so
 * every float/double operation rounds exactly where the reference's does
 * (the reference build has no FMA contraction: SURVEY.md §7 "Hard parts" 1).
 */
#include "slda_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng -- */

/* rng.hpp:14-37 -- Philox4x32-10. */
void orc_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
        const uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* rng.hpp:49-83 -- key (seed_lo, seed_hi), counter (kind, elem_lo, elem_hi, block);
 * next_double() pops buffer_[1] = (o1<<32|o0) first, then buffer_[0] = (o3<<32|o2). */
void orc_uniform2(uint64_t seed, uint32_t kind, uint64_t element, double* u0, double* u1) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const uint32_t ctr[4] = {kind, (uint32_t)element, (uint32_t)(element >> 32), 0u};
    uint32_t o[4];
    orc_philox(ctr, key, o);
    const uint64_t b1 = ((uint64_t)o[1] << 32) | o[0];
    const uint64_t b0 = ((uint64_t)o[3] << 32) | o[2];
    *u0 = (double)(b1 >> 11) * 0x1.0p-53;
    *u1 = (double)(b0 >> 11) * 0x1.0p-53;
}

/* corpus.cpp:87-96, trainer.cpp:217-221, eval.cpp:88-93 */
uint32_t orc_uniform_topic(uint64_t seed, uint32_t kind, uint64_t element, uint32_t num_topics) {
    double u0, u1;
    orc_uniform2(seed, kind, element, &u0, &u1);
    uint32_t topic = (uint32_t)(u0 * (double)num_topics);
    return topic < num_topics ? topic : num_topics - 1;
}

/* --------------------------------------------------------------- corpus -- */

/* corpus.cpp:103-121 -- greedy contiguous ranges. */
int orc_chunk_boundaries(uint32_t num_docs, uint64_t num_tokens, const uint32_t* doc_lengths,
                         uint32_t num_chunks, uint32_t* bounds) {
    if (num_docs == 0) {
        if (num_chunks != 1) return -1;
        bounds[0] = 0;
        bounds[1] = 0;
        return 0;
    }
    if (num_chunks < 1 || num_chunks > num_docs) return -1;
    bounds[0] = 0;
    uint64_t remaining = num_tokens;
    uint32_t doc = 0;
    for (uint32_t c = 0; c < num_chunks; ++c) {
        const uint64_t chunks_left = num_chunks - c;
        const uint64_t share_basis = remaining;
        uint64_t taken = 0;
        do {
            taken += doc_lengths[doc];
            ++doc;
        } while ((uint64_t)(num_docs - doc) > chunks_left - 1 && taken * chunks_left <= share_basis);
        remaining -= taken;
        bounds[c + 1] = doc;
    }
    bounds[num_chunks] = num_docs;
    return 0;
}

/* ---------------------------------------------------------------- counts -- */

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* counts.cpp:65-94 -- sort, then run-length in ascending topic order. */
uint32_t orc_segmented_count(const uint32_t* seg, uint32_t n, uint32_t* out_topics,
                             uint32_t* out_counts) {
    if (n == 0) return 0;
    uint32_t* s = (uint32_t*)malloc(sizeof(uint32_t) * n);
    memcpy(s, seg, sizeof(uint32_t) * n);
    qsort(s, n, sizeof(uint32_t), cmp_u32);
    uint32_t nnz = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (i == 0 || s[i] != s[i - 1]) {
            out_topics[nnz] = s[i];
            out_counts[nnz] = 1;
            ++nnz;
        } else {
            out_counts[nnz - 1] += 1;
        }
    }
    free(s);
    return nnz;
}

/* counts.cpp:37-63 -- integer column sums, f64 denominators, f32 result. */
int orc_preprocess(uint32_t V, uint32_t K, const uint32_t* b, double beta, float* bhat) {
    if (!(beta > 0.0)) return -1;
    if (V == 0) return -1;
    uint64_t* colsum = (uint64_t*)calloc(K, sizeof(uint64_t));
    double* denom = (double*)malloc(sizeof(double) * K);
    for (uint32_t v = 0; v < V; ++v)
        for (uint32_t k = 0; k < K; ++k) colsum[k] += b[(size_t)v * K + k];
    for (uint32_t k = 0; k < K; ++k) denom[k] = (double)colsum[k] + (double)V * beta;
    for (uint32_t v = 0; v < V; ++v)
        for (uint32_t k = 0; k < K; ++k)
            bhat[(size_t)v * K + k] = (float)(((double)b[(size_t)v * K + k] + beta) / denom[k]);
    free(colsum);
    free(denom);
    return 0;
}

/* -------------------------------------------------------------- sampler -- */

/* sampler.hpp:18-41 -- first >= x, slight overshoot clamps, real overshoot throws. */
#define PREFIX_SEARCH_BODY(REAL, EPS)                                           \
    if (n == 0) return -1;                                                       \
    const REAL last = prefix[n - 1];                                             \
    if (x > last) {                                                              \
        const REAL slack = (REAL)16 * EPS * (last > (REAL)1 ? last : (REAL)1);   \
        if (x > last + slack) return -1;                                         \
        return (int64_t)(n - 1);                                                 \
    }                                                                            \
    uint64_t lo = 0, hi = n - 1;                                                 \
    while (lo < hi) {                                                            \
        const uint64_t mid = lo + (hi - lo) / 2;                                 \
        if (prefix[mid] >= x) hi = mid; else lo = mid + 1;                       \
    }                                                                            \
    return (int64_t)lo;

int64_t orc_prefix_search_f(const float* prefix, uint64_t n, float x) { PREFIX_SEARCH_BODY(float, FLT_EPSILON) }
int64_t orc_prefix_search_d(const double* prefix, uint64_t n, double x) { PREFIX_SEARCH_BODY(double, DBL_EPSILON) }

/* sampler.hpp:58-90 (build) and :100-106, :123-127 (sample). */
#define WARY_BUILD_BODY(REAL)                                                    \
    if (W < 2) return -1;                                                        \
    if ((uint64_t)K > (uint64_t)W * W * W) return -1;                            \
    if (K == 0) return -1;                                                       \
    const uint32_t p4 = (K + W - 1) / W * W;                                     \
    const uint32_t n3_real = p4 / W;                                             \
    const uint32_t p3 = (n3_real + W - 1) / W * W;                               \
    const uint32_t n2_real = p3 / W;                                             \
    if (n3) *n3 = p3;                                                            \
    if (n4) *n4 = p4;                                                            \
    if (!l4) return 0;                                                           \
    REAL running = 0;                                                            \
    for (uint32_t i = 0; i < K; ++i) { running += w[i]; l4[i] = running; }      \
    *total = running;                                                            \
    for (uint32_t i = K; i < p4; ++i) l4[i] = running;                           \
    for (uint32_t i = 0; i < n3_real; ++i) l3[i] = l4[(i + 1) * W - 1];          \
    for (uint32_t i = n3_real; i < p3; ++i) l3[i] = running;                     \
    for (uint32_t i = 0; i < n2_real; ++i) l2[i] = l3[(i + 1) * W - 1];          \
    for (uint32_t i = n2_real; i < W; ++i) l2[i] = running;                      \
    return 0;

int orc_wary_tree_d(const double* w, uint32_t K, uint32_t W, double* l2, double* l3,
                    double* l4, uint32_t* n3, uint32_t* n4, double* total) { WARY_BUILD_BODY(double) }
int orc_wary_tree_f(const float* w, uint32_t K, uint32_t W, float* l2, float* l3, float* l4,
                    uint32_t* n3, uint32_t* n4, float* total) { WARY_BUILD_BODY(float) }

#define WARY_SAMPLE_BODY(REAL)                                                   \
    if (!(x <= total)) x = total;                                                \
    uint32_t i2 = W - 1, i3, i4, j;                                              \
    for (j = 0; j < W; ++j) if (l2[j] >= x) { i2 = j; break; }                   \
    uint32_t f = W - 1;                                                          \
    for (j = 0; j < W; ++j) if (l3[i2 * W + j] >= x) { f = j; break; }           \
    i3 = i2 * W + f;                                                             \
    f = W - 1;                                                                   \
    for (j = 0; j < W; ++j) if (l4[i3 * W + j] >= x) { f = j; break; }           \
    i4 = i3 * W + f;                                                             \
    return i4 < K ? i4 : K - 1;

uint32_t orc_wary_sample_d(const double* l2, const double* l3, const double* l4, uint32_t K,
                           uint32_t W, double total, double x) { WARY_SAMPLE_BODY(double) }
uint32_t orc_wary_sample_f(const float* l2, const float* l3, const float* l4, uint32_t K,
                           uint32_t W, float total, float x) { WARY_SAMPLE_BODY(float) }

/* sampler.hpp:73-77: L4 = sequential f32 inclusive prefix; returns total. */
float orc_row_prefix(const float* bhat_row, uint32_t K, float* l4_row) {
    float running = 0.0f;
    for (uint32_t k = 0; k < K; ++k) {
        running += bhat_row[k];
        l4_row[k] = running;
    }
    return running;
}

/* lower_bound over the real prefix, clamped to K-1: equal to WaryTree::sample for every
 * x and every W (acceptance.cpp:140-200, test_sampler.cpp:113-134). */
static uint32_t tree_lower_bound(const float* l4_row, uint32_t K, float total, float x) {
    if (!(x <= total)) x = total;
    uint32_t lo = 0, hi = K;
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (l4_row[mid] >= x) hi = mid; else lo = mid + 1;
    }
    return lo < K ? lo : K - 1;
}

/* sampler.hpp:166-204 -- make_branch_context + sample_token<float>. */
uint32_t orc_sample_token(uint32_t nnz, const uint32_t* topics, const uint32_t* counts,
                          const float* bhat_row, float q, const float* l4_row, uint32_t K,
                          double u0, double u1) {
    float stack_buf[256] = {0};
    float* scratch = nnz <= 256 ? stack_buf : (float*)malloc(sizeof(float) * (nnz ? nnz : 1));
    float s = 0.0f;
    for (uint32_t i = 0; i < nnz; ++i) {
        const float p = (float)counts[i] * bhat_row[topics[i]];
        scratch[i] = p;
        s += p;
    }
    uint32_t result;
    if (!(s + q > 0.0f)) {
        result = ORC_INVALID_TOPIC;
    } else {
        const float branch_draw = (float)u0;
        const float position_draw = (float)u1;
        if (branch_draw < s / (s + q)) {
            float running = 0.0f;
            for (uint32_t i = 0; i < nnz; ++i) {
                running += scratch[i];
                scratch[i] = running;
            }
            const int64_t pick = orc_prefix_search_f(scratch, nnz, position_draw * running);
            result = pick < 0 ? ORC_INVALID_TOPIC : topics[pick];
        } else {
            const float total = K ? l4_row[K - 1] : 0.0f;
            result = tree_lower_bound(l4_row, K, total, position_draw * total);
        }
    }
    if (scratch != stack_buf) free(scratch);
    return result;
}

/* sampler.hpp:222-236 -- vanilla_sample<float> over the dense count row (the O(K) baseline
 * mode, trainer.cpp:281-285).  The dense row is the document's CSR row densified on the fly:
 * DenseDocTopic cell k == count of topic k (trainer.cpp:49-63). */
uint32_t orc_vanilla_token(uint32_t nnz, const uint32_t* topics, const uint32_t* counts,
                           const float* bhat_row, uint32_t K, float alpha, double u0) {
    float* scratch = (float*)malloc(sizeof(float) * (K ? K : 1));
    float running = 0.0f;
    uint32_t p = 0;
    for (uint32_t k = 0; k < K; ++k) {
        const uint32_t c = (p < nnz && topics[p] == k) ? counts[p++] : 0u;
        running += ((float)c + alpha) * bhat_row[k];
        scratch[k] = running;
    }
    const float draw = (float)u0 * running;
    const int64_t pick = orc_prefix_search_f(scratch, K, draw);
    free(scratch);
    return pick < 0 ? ORC_INVALID_TOPIC : (uint32_t)pick;
}

/* ------------------------------------------------------------------ model -- */

struct orc_model {
    uint32_t D, V, K;
    uint64_t T;
    double alpha, beta;
    uint64_t seed;
    uint32_t iteration;
    uint32_t vanilla; /* SamplerKind::kVanilla (trainer.hpp:18) */
    /* PDOW, single chunk (corpus.cpp:125-198) */
    uint32_t *s_doc, *s_word, *s_topic;
    uint64_t* tok_id;
    uint32_t* shuffle;
    uint32_t* doc_off; /* D+1 */
    uint32_t nseg;
    uint32_t *seg_word, *seg_off, *seg_len; /* ascending word */
    /* A: CSR (counts.hpp:33-80) */
    uint64_t* a_off;
    uint32_t *a_top, *a_cnt;
    uint64_t a_nnz;
    /* B, B-hat, L4, Q */
    uint32_t* B;
    float *bhat, *l4, *q;
};

static const uint32_t* g_sort_word;
static const uint32_t* g_sort_doc;
static int cmp_pdow(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b; /* positions == token ids */
    const uint32_t wx = g_sort_word[x], wy = g_sort_word[y];
    if (wx != wy) return wx < wy ? -1 : 1;
    const uint32_t dx = g_sort_doc[x], dy = g_sort_doc[y];
    if (dx != dy) return dx < dy ? -1 : 1;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* counts.cpp:103-125 -- shuffle to doc-grouped order, segmented_count per doc. */
static void rebuild_doc_topic(orc_model* m) {
    uint32_t* grouped = (uint32_t*)malloc(sizeof(uint32_t) * (m->T ? m->T : 1));
    for (uint64_t i = 0; i < m->T; ++i) grouped[m->shuffle[i]] = m->s_topic[i];
    m->a_nnz = 0;
    m->a_off[0] = 0;
    for (uint32_t d = 0; d < m->D; ++d) {
        const uint32_t b = m->doc_off[d], e = m->doc_off[d + 1];
        const uint32_t nnz = orc_segmented_count(grouped + b, e - b, m->a_top + m->a_nnz,
                                                 m->a_cnt + m->a_nnz);
        m->a_nnz += nnz;
        m->a_off[d + 1] = m->a_nnz;
    }
    free(grouped);
}

/* trainer.cpp:223-235 -- B from the word-major layout. */
static void count_word_topic(orc_model* m) {
    memset(m->B, 0, sizeof(uint32_t) * (size_t)m->V * m->K);
    for (uint64_t i = 0; i < m->T; ++i) m->B[(size_t)m->s_word[i] * m->K + m->s_topic[i]] += 1;
}

/* counts.cpp:37-63 then trainer.cpp:237-248 */
static int rebuild_model(orc_model* m) {
    if (orc_preprocess(m->V, m->K, m->B, m->beta, m->bhat) != 0) return -1;
    const float falpha = (float)m->alpha;
    for (uint32_t v = 0; v < m->V; ++v) {
        const float total = orc_row_prefix(m->bhat + (size_t)v * m->K, m->K, m->l4 + (size_t)v * m->K);
        m->q[v] = falpha * total;
    }
    return 0;
}

void orc_free(orc_model* m) {
    if (!m) return;
    free(m->s_doc); free(m->s_word); free(m->s_topic); free(m->tok_id); free(m->shuffle);
    free(m->doc_off); free(m->seg_word); free(m->seg_off); free(m->seg_len);
    free(m->a_off); free(m->a_top); free(m->a_cnt);
    free(m->B); free(m->bhat); free(m->l4); free(m->q);
    free(m);
}

static void set_err(char* err, size_t len, const char* msg) {
    if (err && len) { strncpy(err, msg, len - 1); err[len - 1] = 0; }
}

/* trainer.cpp:15-35 (resolved) + trainer.cpp:354-417 (init_state). */
orc_model* orc_init(uint32_t D, uint32_t V, uint64_t T, const uint32_t* tokens, uint32_t K,
                    double alpha, double beta, uint64_t seed, char* err, size_t err_len) {
    if (K == 0) { set_err(err, err_len, "number of topics must be >= 1"); return NULL; }
    if (alpha <= 0.0) alpha = 50.0 / K;
    if (beta <= 0.0) { set_err(err, err_len, "beta must be > 0"); return NULL; }
    if (V == 0) { set_err(err, err_len, "preprocess requires V >= 1"); return NULL; }
    orc_model* m = (orc_model*)calloc(1, sizeof(orc_model));
    m->D = D; m->V = V; m->T = T; m->K = K; m->alpha = alpha; m->beta = beta; m->seed = seed;
    const size_t t1 = T ? T : 1;
    m->s_doc = malloc(4 * t1); m->s_word = malloc(4 * t1); m->s_topic = malloc(4 * t1);
    m->tok_id = malloc(8 * t1); m->shuffle = malloc(4 * t1);
    m->doc_off = calloc((size_t)D + 1, 4);
    m->a_off = calloc((size_t)D + 1, 8); m->a_top = malloc(4 * t1); m->a_cnt = malloc(4 * t1);
    m->B = calloc((size_t)V * K, 4); m->bhat = malloc(4 * (size_t)V * K);
    m->l4 = malloc(4 * (size_t)V * K); m->q = malloc(4 * (size_t)V);

    /* trainer.cpp:369-378 -- first invalid topic stops the K check. */
    int uninitialized = 0;
    for (uint64_t t = 0; t < T; ++t) {
        const uint32_t doc = tokens[3 * t], word = tokens[3 * t + 1], topic = tokens[3 * t + 2];
        if (doc >= D || word >= V) { set_err(err, err_len, "token id out of range"); orc_free(m); return NULL; }
        (void)doc;
        if (topic == ORC_INVALID_TOPIC) { uninitialized = 1; break; }
        if (topic >= K) { set_err(err, err_len, "token topic exceeds configured K"); orc_free(m); return NULL; }
    }
    for (uint64_t t = 0; t < T; ++t) {
        if (tokens[3 * t] >= D || tokens[3 * t + 1] >= V) { set_err(err, err_len, "token id out of range"); orc_free(m); return NULL; }
    }

    /* corpus.cpp:148-175 -- single chunk, sort by (word, doc, token_id). */
    uint32_t* cdoc = malloc(4 * t1);
    uint32_t* cword = malloc(4 * t1);
    uint64_t* order = malloc(8 * t1);
    for (uint64_t t = 0; t < T; ++t) { cdoc[t] = tokens[3 * t]; cword[t] = tokens[3 * t + 1]; order[t] = t; }
    g_sort_word = cword; g_sort_doc = cdoc;
    qsort(order, T, sizeof(uint64_t), cmp_pdow);
    for (uint64_t i = 0; i < T; ++i) {
        const uint64_t t = order[i];
        m->s_doc[i] = cdoc[t];
        m->s_word[i] = cword[t];
        m->tok_id[i] = t;
        const uint32_t topic = tokens[3 * t + 2];
        /* trainer.cpp:383-388 */
        m->s_topic[i] = uninitialized ? orc_uniform_topic(seed, ORC_INIT_STREAM, t, K) : topic;
    }
    free(cdoc); free(cword); free(order);

    /* corpus.cpp:177-184 -- word segments */
    m->seg_word = malloc(4 * t1); m->seg_off = malloc(4 * t1); m->seg_len = malloc(4 * t1);
    m->nseg = 0;
    for (uint64_t i = 0; i < T;) {
        uint64_t j = i;
        while (j < T && m->s_word[j] == m->s_word[i]) ++j;
        m->seg_word[m->nseg] = m->s_word[i];
        m->seg_off[m->nseg] = (uint32_t)i;
        m->seg_len[m->nseg] = (uint32_t)(j - i);
        m->nseg++;
        i = j;
    }
    /* corpus.cpp:186-195 -- doc offsets and shuffle pointers */
    for (uint64_t i = 0; i < T; ++i) m->doc_off[m->s_doc[i] + 1]++;
    for (uint32_t d = 0; d < D; ++d) m->doc_off[d + 1] += m->doc_off[d];
    uint32_t* cursor = malloc(4 * ((size_t)D + 1));
    memcpy(cursor, m->doc_off, 4 * (size_t)D);
    for (uint64_t i = 0; i < T; ++i) m->shuffle[i] = cursor[m->s_doc[i]]++;
    free(cursor);

    rebuild_doc_topic(m);
    count_word_topic(m);
    if (rebuild_model(m) != 0) { set_err(err, err_len, "preprocess failed"); orc_free(m); return NULL; }
    return m;
}

/* trainer.cpp:265-291, :295-333, :419-449 */
int orc_iterate(orc_model* m) {
    const uint32_t stream = m->iteration;
    for (uint64_t i = 0; i < m->T; ++i) {
        const uint32_t d = m->s_doc[i], v = m->s_word[i];
        const uint64_t b = m->a_off[d], e = m->a_off[d + 1];
        double u0, u1;
        orc_uniform2(m->seed, stream, m->tok_id[i], &u0, &u1);
        const uint32_t next =
            m->vanilla ? orc_vanilla_token((uint32_t)(e - b), m->a_top + b, m->a_cnt + b,
                                           m->bhat + (size_t)v * m->K, m->K, (float)m->alpha, u0)
                       : orc_sample_token((uint32_t)(e - b), m->a_top + b, m->a_cnt + b,
                                          m->bhat + (size_t)v * m->K, m->q[v],
                                          m->l4 + (size_t)v * m->K, m->K, u0, u1);
        if (next == ORC_INVALID_TOPIC) return -1;
        m->s_topic[i] = next;
    }
    rebuild_doc_topic(m);
    count_word_topic(m);
    if (rebuild_model(m) != 0) return -1;
    m->iteration += 1;
    return 0;
}

uint32_t orc_iteration(const orc_model* m) { return m->iteration; }
void orc_set_sampler(orc_model* m, uint32_t vanilla) { m->vanilla = vanilla ? 1u : 0u; }
double orc_alpha(const orc_model* m) { return m->alpha; }
void orc_get_word_topic(const orc_model* m, uint32_t* out) { memcpy(out, m->B, 4 * (size_t)m->V * m->K); }
void orc_get_word_topic_prob(const orc_model* m, float* out) { memcpy(out, m->bhat, 4 * (size_t)m->V * m->K); }
void orc_get_l4(const orc_model* m, float* out) { memcpy(out, m->l4, 4 * (size_t)m->V * m->K); }
void orc_get_tree_mass(const orc_model* m, float* out) { memcpy(out, m->q, 4 * (size_t)m->V); }
/* trainer.cpp:203-213 */
void orc_get_assignments(const orc_model* m, uint32_t* out) {
    for (uint64_t i = 0; i < m->T; ++i) out[m->tok_id[i]] = m->s_topic[i];
}
uint64_t orc_doc_topic_nnz(const orc_model* m) { return m->a_nnz; }
void orc_get_doc_topic(const orc_model* m, uint64_t* row_offsets, uint32_t* topics, uint32_t* counts) {
    memcpy(row_offsets, m->a_off, 8 * ((size_t)m->D + 1));
    memcpy(topics, m->a_top, 4 * m->a_nnz);
    memcpy(counts, m->a_cnt, 4 * m->a_nnz);
}
/* trainer.cpp:335-350 */
double orc_mean_doc_topics(const orc_model* m) {
    return m->D > 0 ? (double)m->a_nnz / (double)m->D : 0.0;
}
uint32_t orc_num_segments(const orc_model* m) { return m->nseg; }
void orc_get_pdow(const orc_model* m, uint32_t* sorted_doc, uint32_t* sorted_word,
                  uint32_t* token_ids, uint32_t* shuffle_ptrs, uint32_t* doc_offsets,
                  uint32_t* seg_word, uint32_t* seg_offset, uint32_t* seg_length) {
    for (uint64_t i = 0; i < m->T; ++i) {
        sorted_doc[i] = m->s_doc[i];
        sorted_word[i] = m->s_word[i];
        token_ids[i] = (uint32_t)m->tok_id[i];
        shuffle_ptrs[i] = m->shuffle[i];
    }
    memcpy(doc_offsets, m->doc_off, 4 * ((size_t)m->D + 1));
    memcpy(seg_word, m->seg_word, 4 * (size_t)m->nseg);
    memcpy(seg_offset, m->seg_off, 4 * (size_t)m->nseg);
    memcpy(seg_length, m->seg_len, 4 * (size_t)m->nseg);
}

/* eval.cpp:14-28 (split) and eval.cpp:49-133 (heldout_ll). */
int orc_heldout_ll(const orc_model* m, uint32_t D, uint32_t V, uint64_t T, const uint32_t* tokens,
                   uint32_t burn_in, uint64_t seed, double* per_token_ll, uint64_t* tokens_evaluated) {
    if (D == 0) return -1;
    if (V != m->V) return -1;
    const uint32_t K = m->K;
    const double alpha = m->alpha;
    /* from_corpus: per doc, alternating positions */
    uint32_t* seen = calloc(D, 4);
    uint64_t* est_len = calloc(D, 8);
    uint64_t* evl_len = calloc(D, 8);
    for (uint64_t t = 0; t < T; ++t) {
        const uint32_t d = tokens[3 * t];
        if (seen[d]++ % 2 == 0) est_len[d]++; else evl_len[d]++;
    }
    uint64_t* est_off = calloc((size_t)D + 1, 8);
    uint64_t* evl_off = calloc((size_t)D + 1, 8);
    for (uint32_t d = 0; d < D; ++d) { est_off[d + 1] = est_off[d] + est_len[d]; evl_off[d + 1] = evl_off[d] + evl_len[d]; }
    const uint64_t n_est = est_off[D], n_evl = evl_off[D];
    if (n_evl == 0) { free(seen); free(est_len); free(evl_len); free(est_off); free(evl_off); return -1; }
    uint32_t* est = malloc(4 * (n_est ? n_est : 1));
    uint32_t* evl = malloc(4 * n_evl);
    memset(seen, 0, 4 * (size_t)D);
    memset(est_len, 0, 8 * (size_t)D);
    memset(evl_len, 0, 8 * (size_t)D);
    for (uint64_t t = 0; t < T; ++t) {
        const uint32_t d = tokens[3 * t], w = tokens[3 * t + 1];
        if (seen[d]++ % 2 == 0) est[est_off[d] + est_len[d]++] = w;
        else evl[evl_off[d] + evl_len[d]++] = w;
    }
    /* eval.cpp:61-69 -- f64 row masses */
    double* row_mass = malloc(8 * (size_t)V);
    for (uint32_t v = 0; v < V; ++v) {
        double sum = 0.0;
        for (uint32_t k = 0; k < K; ++k) sum += m->bhat[(size_t)v * K + k];
        row_mass[v] = sum;
    }
    double total = 0.0;
    uint32_t* topics = malloc(4 * (n_est ? n_est : 1));
    uint32_t* rt = malloc(4 * (n_est ? n_est : 1));
    uint32_t* rc = malloc(4 * (n_est ? n_est : 1));
    for (uint32_t d = 0; d < D; ++d) {
        const uint64_t n = est_len[d], base = est_off[d];
        if (n == 0) continue; /* eval.cpp:85 */
        for (uint64_t j = 0; j < n; ++j) topics[j] = orc_uniform_topic(seed, ORC_HELDOUT_INIT_STREAM, base + j, K);
        for (uint32_t sweep = 0; sweep < burn_in; ++sweep) {
            const uint32_t nnz = orc_segmented_count(topics, (uint32_t)n, rt, rc);
            for (uint64_t j = 0; j < n; ++j) {
                const uint32_t v = est[base + j];
                double u0, u1;
                orc_uniform2(seed, ORC_HELDOUT_SWEEP_BASE + sweep, base + j, &u0, &u1);
                const uint32_t k = orc_sample_token(nnz, rt, rc, m->bhat + (size_t)v * K, m->q[v],
                                                    m->l4 + (size_t)v * K, K, u0, u1);
                if (k == ORC_INVALID_TOPIC) return -1;
                topics[j] = k;
            }
        }
        const uint32_t nnz = orc_segmented_count(topics, (uint32_t)n, rt, rc);
        const double denom = (double)n + K * alpha;
        double ll = 0.0;
        for (uint64_t j = 0; j < evl_len[d]; ++j) {
            const uint32_t v = evl[evl_off[d] + j];
            double mass = alpha * row_mass[v];
            for (uint32_t i = 0; i < nnz; ++i) mass += (double)rc[i] * (double)m->bhat[(size_t)v * K + rt[i]];
            ll += log(mass / denom);
        }
        total += ll;
    }
    *per_token_ll = total / (double)n_evl;
    *tokens_evaluated = n_evl;
    free(seen); free(est_len); free(evl_len); free(est_off); free(evl_off);
    free(est); free(evl); free(row_mass); free(topics); free(rt); free(rc);
    return 0;
}
