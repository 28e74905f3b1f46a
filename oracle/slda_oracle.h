/*
 * slda_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference ESCA iteration
 * (arxiv/paper_1610_02496, `proj/`), used as the parity checker for the
 * B200 engine.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product never links or calls it.
 *
 * Parity is pinned: tests/test_oracle.py checks this file against the
 * reference's own known-answer vectors and against per-iteration digests
 * produced by the reference itself (oracle/_ref, built from the reference
 * sources by oracle/Makefile; see tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates.  Float order is
 * the reference's: sequential f32 adds, no FMA contraction (build with
 * -ffp-contract=off), f64 where the reference uses double.
 */
#ifndef SLDA_ORACLE_H
#define SLDA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_INVALID_TOPIC 0xFFFFFFFFu
#define ORC_INIT_STREAM 0xFFFFFFFFu
#define ORC_HELDOUT_INIT_STREAM 0xFFFD0000u
#define ORC_HELDOUT_SWEEP_BASE 0xFFFE0000u

/* rng.hpp:26-37 */
void orc_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]);
/* rng.hpp:49-83: the first two doubles of RngStream(seed, kind, element). */
void orc_uniform2(uint64_t seed, uint32_t kind, uint64_t element, double* u0, double* u1);

/* corpus.cpp:87-96 / trainer.cpp:217-221 */
uint32_t orc_uniform_topic(uint64_t seed, uint32_t kind, uint64_t element, uint32_t num_topics);

/* corpus.cpp:103-121; bounds has num_chunks+1 entries. Returns 0 or -1 (validation). */
int orc_chunk_boundaries(uint32_t num_docs, uint64_t num_tokens, const uint32_t* doc_lengths,
                         uint32_t num_chunks, uint32_t* bounds);

/* counts.cpp:65-94: writes nnz sorted (topic, count) pairs, returns nnz. */
uint32_t orc_segmented_count(const uint32_t* seg, uint32_t n, uint32_t* out_topics,
                             uint32_t* out_counts);

/* counts.cpp:37-63 */
int orc_preprocess(uint32_t V, uint32_t K, const uint32_t* b, double beta, float* bhat);

/* sampler.hpp:18-41: returns index, or -1 when the reference throws. */
int64_t orc_prefix_search_f(const float* prefix, uint64_t n, float x);
int64_t orc_prefix_search_d(const double* prefix, uint64_t n, double x);

/* sampler.hpp:58-90 (generic W): l2 has W entries, l3 padded(n4/W), l4 padded(K).
 * Returns 0 or -1 (validation). Sizes out via pointers when arrays are NULL. */
int orc_wary_tree_d(const double* w, uint32_t K, uint32_t W, double* l2, double* l3,
                    double* l4, uint32_t* n3, uint32_t* n4, double* total);
int orc_wary_tree_f(const float* w, uint32_t K, uint32_t W, float* l2, float* l3, float* l4,
                    uint32_t* n3, uint32_t* n4, float* total);
/* sampler.hpp:100-106 */
uint32_t orc_wary_sample_d(const double* l2, const double* l3, const double* l4, uint32_t K,
                           uint32_t W, double total, double x);
uint32_t orc_wary_sample_f(const float* l2, const float* l3, const float* l4, uint32_t K,
                           uint32_t W, float total, float x);

/* sampler.hpp:58-76 + trainer.cpp:245: L4 prefix (first K entries) and Q. */
float orc_row_prefix(const float* bhat_row, uint32_t K, float* l4_row);

/* sampler.hpp:166-204 with the tree replaced by its proven-equal lower_bound
 * over L4 (acceptance.cpp:140-200).  Returns topic, or ORC_INVALID_TOPIC on
 * the reference's throw paths. */
uint32_t orc_sample_token(uint32_t nnz, const uint32_t* topics, const uint32_t* counts,
                          const float* bhat_row, float q, const float* l4_row, uint32_t K,
                          double u0, double u1);

/* ---------------------------------------------------------------- model -- */

typedef struct orc_model orc_model;

/* init_state (trainer.cpp:354-417) over a doc-sorted or arbitrary corpus given as
 * AoS triples (doc, word, topic) exactly like sparselda::Token.  alpha<=0 -> 50/K.
 * num_chunks = 1 always: results do not depend on it (acceptance.cpp:426-445). */
/* sampler.hpp:222-236: vanilla_sample<float> over the (densified) count row. */
uint32_t orc_vanilla_token(uint32_t nnz, const uint32_t* topics, const uint32_t* counts,
                           const float* bhat_row, uint32_t K, float alpha, double u0);
/* TrainConfig::sampler (trainer.hpp:18, :30): 0 sparse (default), 1 vanilla. */
void orc_set_sampler(orc_model* m, uint32_t vanilla);

orc_model* orc_init(uint32_t D, uint32_t V, uint64_t T, const uint32_t* tokens, uint32_t K,
                    double alpha, double beta, uint64_t seed, char* err, size_t err_len);
void orc_free(orc_model* m);
/* run_iteration (trainer.cpp:419-449).  Returns 0 or -1. */
int orc_iterate(orc_model* m);
uint32_t orc_iteration(const orc_model* m);
double orc_alpha(const orc_model* m);
/* Getters copy out. */
void orc_get_word_topic(const orc_model* m, uint32_t* out);        /* V*K */
void orc_get_word_topic_prob(const orc_model* m, float* out);      /* V*K */
void orc_get_l4(const orc_model* m, float* out);                   /* V*K (real prefix) */
void orc_get_tree_mass(const orc_model* m, float* out);            /* V */
void orc_get_assignments(const orc_model* m, uint32_t* out);       /* T, corpus order */
uint64_t orc_doc_topic_nnz(const orc_model* m);
void orc_get_doc_topic(const orc_model* m, uint64_t* row_offsets, uint32_t* topics,
                       uint32_t* counts);                          /* D+1, nnz, nnz */
double orc_mean_doc_topics(const orc_model* m);
/* PDOW of the single chunk (corpus.cpp:125-198) and schedule (:200-210). */
uint32_t orc_num_segments(const orc_model* m);
void orc_get_pdow(const orc_model* m, uint32_t* sorted_doc, uint32_t* sorted_word,
                  uint32_t* token_ids, uint32_t* shuffle_ptrs, uint32_t* doc_offsets,
                  uint32_t* seg_word, uint32_t* seg_offset, uint32_t* seg_length);

/* heldout_ll (eval.cpp:49-133) over a held-out corpus given as AoS triples;
 * HeldoutSet::from_corpus split (eval.cpp:14-28).  Returns 0 or -1. */
int orc_heldout_ll(const orc_model* m, uint32_t D, uint32_t V, uint64_t T,
                   const uint32_t* tokens, uint32_t burn_in, uint64_t seed, double* per_token_ll,
                   uint64_t* tokens_evaluated);

#ifdef __cplusplus
}
#endif
#endif
